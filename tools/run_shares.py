"""Execute the per-device shares of a G-GPU SHARP plan one after another on ONE B200.

python tools/run_shares.py CONFIG.json G [devices,comma,separated|all] ['{"opt_state": "bf16"}']
   extra keys also: "strategy" ("sharp" | "task-parallel"), "mem_bytes" (override every device's cap)

With double buffering a job never leaves the device it first lands on, so the
G devices of a plan share nothing but host DRAM / PCIe-switch bandwidth: device r's share
run alone on one GPU is what rank r of `torchrun --nproc-per-node G bench.py` executes
(bench.plan_share). The emulated G-GPU makespan is the max over the measured shares; it does
not model host-memory-bandwidth contention between concurrently streaming GPUs (stated in
the output). One JSON line per share, then a summary line.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2110_08633_b200 as P  # noqa: E402

cfg_path, G = sys.argv[1], int(sys.argv[2])
devs = sys.argv[3] if len(sys.argv) > 3 else "all"
extra = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
warm = int(extra.pop("warmup_passes", 1))
strategy = extra.pop("strategy", "sharp")
cfg = json.load(open(cfg_path))
if "mem_bytes" in extra:  # e.g. the task-parallel comparison leg, run uncapped
    mem = float(extra.pop("mem_bytes"))
    for d in cfg["cluster"]["devices"]:
        d["mem_bytes"] = mem
plan = P.plan(cfg, strategy=strategy, gpus=G)
devices = list(range(G)) if devs == "all" else [int(x) for x in devs.split(",")]
shares = []
for r in devices:
    mine = [t for t, dev, _ in plan["dispatch"] if dev == r]
    jobs = sorted({plan["tasks"][t]["job"] for t in mine})
    if not mine:
        continue
    t0 = time.time()
    ex = P.Executor(cfg, strategy=strategy, gpus=G, run_devices=[r], device_ids=[0] * G, passes=1,
                    warmup_passes=warm, **extra)
    setup = time.time() - t0
    if warm:
        ex.run(warm, timed=False)
    res = ex.run(1)
    ex.close()
    st = res["stats"]
    sec = res["pass_seconds"][0]
    line = {"config": os.path.basename(cfg_path), "strategy": strategy, "G": G, "device": r, "jobs": jobs, "tasks": len(mine),
            "samples": res["samples_per_pass"], "makespan_s": round(sec, 3),
            "samples_per_s": round(res["samples_per_pass"] / sec, 2),
            "h2d_GB": round(st["h2d_bytes_per_pass"] / 1e9, 2), "d2h_GB": round(st["d2h_bytes_per_pass"] / 1e9, 2),
            "arena_GB": [round(x / 1e9, 2) for x in st["arena_bytes"]], "setup_s": round(setup, 1),
            "final_losses": {str(j): round(res["losses"][j][-1], 4) for j in jobs if res["losses"][j]}, "extra": extra}
    shares.append(line)
    print(json.dumps(line), flush=True)
if shares:
    total = sum(s["samples"] for s in shares)
    mk = max(s["makespan_s"] for s in shares)
    print(json.dumps({"summary": True, "config": os.path.basename(cfg_path), "strategy": strategy, "G": G,
                      "devices_measured": [s["device"] for s in shares], "samples": total,
                      "emulated_makespan_s": mk, "emulated_samples_per_s": round(total / mk, 2),
                      "sum_of_share_makespans_s": round(sum(s["makespan_s"] for s in shares), 3),
                      "virtual_makespan_s": round(plan["makespan_s"], 3), "dispatch_hash": plan["dispatch_hash"],
                      "shard_roofline_frac": round(plan["makespan_s"] / mk, 4) if len(shares) == G else None,
                      "note": "shares run one after another on one GPU; no host-DRAM/PCIe contention between "
                              "GPUs is modelled"}), flush=True)
