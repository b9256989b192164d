"""Split a pass into link-bound and compute-bound parts (debug_skip modes)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08633_b200 as P
cfg = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "configs/c2_gpt2small_x8.json"))
extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
# a share of a G-GPU plan on this one GPU: '{"gpus": 8, "run_devices": [0]}'
G = int(extra.pop("gpus", 1))
if G > 1:
    extra.setdefault("device_ids", [0] * G)
extra["gpus"] = G
for name, skip in (("full", 0), ("no-transfers", 1), ("no-compute", 2)):
    ex = P.Executor(cfg, passes=2, warmup_passes=1, debug_skip=skip, **extra)
    ex.run(1, timed=False)
    r = ex.run(2)
    print(name, extra, [round(x, 3) for x in r["pass_seconds"]], "enqueue_s", round(r["stats"]["enqueue_s_last_pass"], 3), flush=True)
    ex.close()

if os.environ.get("HY_PROFILE") == "1":
    ex = P.Executor(cfg, passes=1, warmup_passes=1, **extra)
    ex.run(1, timed=False)
    r = ex.run(1)
    prof = r.get("op_profile_ms", {})
    tot = sum(prof.values())
    print("compute-stream op profile (ms per pass), total", round(tot, 1), "pass", round(r["pass_seconds"][0], 3))
    for k, v in sorted(prof.items(), key=lambda x: -x[1]):
        print(f"  {k:14s} {v:9.1f} {100 * v / tot:5.1f}%")
