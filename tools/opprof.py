"""Compute-stream op profile of one pass (HY_PROFILE=1; diagnostics): ms per op label,
including wait_* entries = time the compute stream stalled on a hazard before an op."""
import json, os, sys
os.environ["HY_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08633_b200 as P
cfg = json.load(open(sys.argv[1]))
extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
extra.setdefault("gpus", 1)
ex = P.Executor(cfg, passes=1, warmup_passes=1, **extra)
ex.run(1, timed=False)
r = ex.run(1)
prof = r.get("op_profile_ms", {})
tot = sum(prof.values())
print(json.dumps(extra), "pass", round(r["pass_seconds"][0], 3), "profiled total", round(tot, 1))
for k, v in sorted(prof.items(), key=lambda x: -x[1]):
    print(f"  {k:14s} {v:9.1f} {100 * v / tot:5.1f}%")
