"""Run one timed pass of a workload and save the measured Chrome trace + summary."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08633_b200 as P

cfg_path = sys.argv[1] if len(sys.argv) > 1 else "configs/c2_gpt2small_x8.json"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace_c2.json"
cfg = json.load(open(cfg_path))
ex = P.Executor(cfg, strategy="sharp", gpus=1, passes=1, warmup_passes=1)
ex.run(1, timed=False)
r = ex.run(1, timed=True, trace=True)
os.makedirs(os.path.dirname(out), exist_ok=True)
open(out, "w").write(r["chrome_trace"])
r.pop("chrome_trace")
r.pop("losses")
print(json.dumps(r)[:3000])
