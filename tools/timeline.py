"""Measured per-task timeline of one pass (diagnostics): where the compute lane waits.

python tools/timeline.py CONFIG.json '{"host_opt_fraction": 0.5}' [n_tasks_to_print]
Prints the first tasks' intervals (ms, relative to the pass start) and a summary: compute-lane
busy time, idle gaps, and how much of the idle time ends exactly when the task's own
ParamLoad / ActPromote finished (load-bound) vs. otherwise (waiting on a hazard).
"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08633_b200 as P  # noqa: E402

cfg = json.load(open(sys.argv[1]))
extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
n_print = int(sys.argv[3]) if len(sys.argv) > 3 else 24
G = int(extra.pop("gpus", 1))  # a share of a G-GPU plan: '{"gpus": 8, "run_devices": [0]}'
if G > 1:
    extra.setdefault("device_ids", [0] * G)
ex = P.Executor(cfg, gpus=G, passes=1, warmup_passes=1, **extra)
ex.run(1, timed=False)
r = ex.run(1, trace=True)
tr = json.loads(r["chrome_trace"])
lanes = {}
for e in tr["traceEvents"]:
    if e.get("ph") == "M" and e["name"] == "thread_name":
        lanes[(e["pid"], e["tid"])] = e["args"]["name"]
tasks = defaultdict(dict)
order = []
for e in tr["traceEvents"]:
    if e.get("ph") != "X" or e["pid"] != 0:
        continue
    kind, label = e["name"].split(" ", 1)
    if label not in tasks:
        order.append(label)
    tasks[label][kind] = (e["ts"] / 1e3, (e["ts"] + e["dur"]) / 1e3)
comp = sorted((v["Compute"][0], v["Compute"][1], k) for k, v in tasks.items() if "Compute" in v)
print(f"pass {r['pass_seconds'][0]:.3f} s, tasks {len(comp)}")
busy = sum(b - a for a, b, _ in comp)
gap_load = gap_other = 0.0
kinds = defaultdict(lambda: [0, 0.0])
prev_end = 0.0
for a, b, k in comp:
    gap = max(0.0, a - prev_end)
    ready = max([tasks[k][x][1] for x in ("ParamLoad", "ActPromote") if x in tasks[k]] or [0.0])
    if gap > 0.02 and abs(a - ready) < 0.05:
        gap_load += gap
    else:
        gap_other += gap
    key = k.split(".")[-2] + "." + k.split(".")[-1]
    kinds[key][0] += 1
    kinds[key][1] += b - a
    prev_end = max(prev_end, b)
print(f"compute busy {busy / 1e3:.3f} s, idle {(gap_load + gap_other) / 1e3:.3f} s "
      f"(load-bound {gap_load / 1e3:.3f}, other {gap_other / 1e3:.3f})")
print("compute time by shard.direction:", {k: (v[0], round(v[1] / max(1, v[0]), 2)) for k, v in sorted(kinds.items())})
print(f"{'task':22s} {'load':>17s} {'promote':>17s} {'compute':>17s} {'demote/offload':>17s}")
for a, b, k in comp[:n_print]:
    t = tasks[k]

    def f(x):
        return f"{t[x][0]:8.2f}-{t[x][1]:8.2f}" if x in t else " " * 17
    dem = "ActDemote" if "ActDemote" in t else "GradOffload"
    print(f"{k:22s} {f('ParamLoad')} {f('ActPromote')} {f('Compute')} {f(dem)}")
