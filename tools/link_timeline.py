"""One interval-logged C2 pass (HY_LINK_DUMP): per-minibatch link usage, where H2D / D2H idle.

python tools/link_timeline.py [config] -> gpurun_out/link_raw.json + a summary of idle link
time split by what the compute stream was doing (forward / backward tasks)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HY_LINK_DUMP"] = "1"
import paper_2110_08633_b200 as P

cfg = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "configs/c2_gpt2small_x8.json"))
ex = P.Executor(cfg, gpus=1, passes=2, warmup_passes=1)
ex.run(1, timed=False)
r = ex.run(1, timed=True, interval_log=True, trace=True)
raw = r["links"][0]["raw"]
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"raw": raw, "trace": json.loads(r["chrome_trace"]), "pass_s": r["pass_seconds"][-1]},
          open("gpurun_out/link_raw.json", "w"))
T = r["pass_seconds"][-1]
print(json.dumps({k: v for k, v in r["links"][0].items() if k != "raw"}))
# busy fraction per direction in 1 ms bins
import numpy as np
nb = int(T * 1000) + 1
busy = np.zeros((3, nb))
for lane, st, a, b, by in raw:
    i0, i1 = int(a * 1000), int(b * 1000)
    for i in range(i0, min(i1 + 1, nb)):
        lo, hi = max(a, i / 1000), min(b, (i + 1) / 1000)
        if hi > lo:
            busy[int(lane), i] += (hi - lo) * 1000
busy = np.minimum(busy, 1.0)
print("first 70 ms, per 1 ms bin: compute / H2D / D2H busy fraction (x10, capped 9)")
for lane in range(3):
    print("CHD"[lane], "".join(str(min(9, int(x * 10))) for x in busy[lane, :70]))
by_stream = {}
for lane, st, a, b, byt in raw:
    k = ("comp", "down", "up", "opt", "opt2", "optin", "other")[int(st)] + ("", ".h2d", ".d2h")[int(lane)]
    e = by_stream.setdefault(k, [0, 0.0, 0.0])
    e[0] += 1
    e[1] += b - a
    e[2] += byt
print(json.dumps({k: {"n": v[0], "busy_s": round(v[1], 4), "GB": round(v[2] / 1e9, 3)} for k, v in by_stream.items()}))
