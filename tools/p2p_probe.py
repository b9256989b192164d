import sys, os, json, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import paper_2110_08633_b200 as P
from oracle import oracle as O
import test_executor_gpu as T
cfg = T.tiny_config(mbs=3, jobs=3)
starts=None
for p2p in (False, True):
    for dyn in ("plan",):
        res = P.execute(cfg, gpus=2, device_ids=[0, 0], double_buffering=False, precision="fp32", p2p=p2p, schedule=dyn)
        if starts is None:
            starts = res["shard_starts"]
            losses, params = O.run_workload_cpu(cfg, starts)
        print("p2p", p2p, dyn, "p2pbytes", res["stats"]["p2p_bytes_per_pass"], [ [round(abs(a-b)/b,7) for a,b in zip(res["losses"][j], losses[j])] for j in losses])
res = P.execute(cfg, gpus=2, device_ids=[0, 0], double_buffering=False, precision="fp32", write_through=True, p2p=False)
print("write_through", [ [round(abs(a-b)/b,7) for a,b in zip(res["losses"][j], losses[j])] for j in losses])
res = P.execute(cfg, gpus=2, device_ids=[0, 0], double_buffering=False, precision="fp32", p2p=False, mv_cache=False)
print("no mv cache", [ [round(abs(a-b)/b,7) for a,b in zip(res["losses"][j], losses[j])] for j in losses])
res = P.execute(cfg, gpus=1, double_buffering=False, precision="fp32")
print("G=1 db off", [ [round(abs(a-b)/b,7) for a,b in zip(res["losses"][j], losses[j])] for j in losses])
