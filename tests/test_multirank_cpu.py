"""N>1 path on CPU: two gloo ranks plan the same workload for G=2, each takes its device's
share (what bench.py's rank r executes under torchrun), and the shares are checked to be
disjoint job sets covering every task and sample, with the max-over-ranks / sum-over-ranks
reduce bench.py uses. No collective on the data path: the only exchange is the reduce."""
import json
import os
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, world, port, cfg_path, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    cfg = json.load(open(cfg_path))
    share = bench.plan_share(cfg, world, rank)
    objs = [None] * world
    dist.all_gather_object(objs, {"jobs": share["jobs"], "tasks": share["tasks"], "samples": share["samples"],
                                  "hash": share["dispatch_hash"]})
    # a fake per-rank time: rank r "took" 1 + r seconds for its share
    red = bench.reduce_over_ranks(dist, "cpu", 1.0 + rank, 2.0 + rank, share["samples"], 10.0 * (rank + 1), 1.0, 5)
    if rank == 0:
        json.dump({"shares": objs, "reduced": red}, open(os.path.join(out_dir, "r.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name,world", [("c2_gpt2small_x8.json", 2), ("c1_tiny.json", 2),
                                            ("c5_hetero_x12.json", 2)])
def test_two_rank_shares(tmp_path, cfg_name, world):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cfg_path = os.path.join(ROOT, "configs", cfg_name)
    mp.spawn(_worker, args=(world, port, cfg_path, str(tmp_path)), nprocs=world, join=True)
    r = json.load(open(tmp_path / "r.json"))
    shares = r["shares"]
    cfg = json.load(open(cfg_path))
    # every rank planned the identical dispatch (same hash), shares are disjoint job sets
    assert len({s["hash"] for s in shares}) == 1
    jobs = [set(s["jobs"]) for s in shares]
    assert not (jobs[0] & jobs[1])
    assert jobs[0] | jobs[1] == set(range(len(cfg["jobs"])))
    tasks = sorted(t for s in shares for t in s["tasks"])
    import paper_2110_08633_b200 as P

    assert tasks == list(range(len(P.plan(cfg, gpus=world)["tasks"])))
    total = sum(j["batch_size"] * j.get("minibatches_per_epoch", 1) * j.get("epochs", 1) for j in cfg["jobs"])
    assert sum(s["samples"] for s in shares) == total
    dev_time, wall, samples, h2d, d2h, launches = r["reduced"]
    assert dev_time == 2.0 and wall == 3.0  # max over ranks
    assert samples == total and h2d == 30.0 and d2h == 2.0 and launches == 10  # sums
