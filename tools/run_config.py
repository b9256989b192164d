"""Run a workload config through the executor (1 GPU) and print pass time, samples/s, losses."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08633_b200 as P
cfg = json.load(open(sys.argv[1]))
extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
jobs = extra.pop("jobs", None)
if jobs is not None:
    cfg["jobs"] = [cfg["jobs"][i] for i in jobs]
mbs = extra.pop("minibatches", None)
if mbs is not None:
    for j in cfg["jobs"]:
        j["minibatches_per_epoch"] = mbs
t0 = time.time()
ex = P.Executor(cfg, gpus=1, passes=1, warmup_passes=1, **extra)
t1 = time.time()
ex.run(1, timed=False)
r = ex.run(1)
st = r["stats"]
print(json.dumps({"config": os.path.basename(sys.argv[1]), "jobs": len(cfg["jobs"]), "extra": extra,
                  "setup_s": round(t1 - t0, 1), "pass_s": round(r["pass_seconds"][0], 3),
                  "samples_per_s": round(r["samples_per_pass"] / r["pass_seconds"][0], 2),
                  "virtual_makespan_s": round(r["virtual_makespan_s"], 3), "shard_starts": r["shard_starts"][:2],
                  "arena_GB": [round(x / 1e9, 2) for x in st["arena_bytes"]],
                  "h2d_GB": round(st["h2d_bytes_per_pass"] / 1e9, 1), "d2h_GB": round(st["d2h_bytes_per_pass"] / 1e9, 1),
                  "losses_job0": [round(x, 4) for x in r["losses"][0][-4:]]}), flush=True)
