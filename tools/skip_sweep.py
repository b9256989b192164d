import json, os, sys
sys.path.insert(0, '/root/repo')
import paper_2110_08633_b200 as P
cfg = json.load(open('configs/c2_gpt2small_x8.json'))
for name, extra in [("default", {}), ("chunk1M", {"opt_chunk_floats": 1 << 20}),
                    ("slack200M_chunk4M_nomv", {"hbm_slack_bytes": 2e8, "mv_cache": False, "opt_chunk_floats": 4 << 20, "pool_extra_max_bytes": 2e7}),
                    ("slack200M_nomv_chunk2M", {"hbm_slack_bytes": 2e8, "mv_cache": False, "pool_extra_max_bytes": 2e7}),
                    ("slack400M_chunk8M_nomv", {"hbm_slack_bytes": 4e8, "mv_cache": False, "opt_chunk_floats": 8 << 20, "pool_extra_max_bytes": 2e7})]:
    for skip in (2, 0):
        ex = P.Executor(cfg, gpus=1, passes=2, warmup_passes=1, debug_skip=skip, **extra)
        ex.run(1, timed=False)
        r = ex.run(2)
        print(name, "no-compute" if skip == 2 else "full", [round(x, 3) for x in r["pass_seconds"]], r["stats"]["arena_bytes"], flush=True)
        ex.close()
