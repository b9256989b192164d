#!/usr/bin/env python3
"""Benchmark: aggregate train samples/sec of the Hydra shard-execution path on B200.

Workload (BASELINE.json configs[1], C2): 8 GPT-2-small (124M) hyper-parameter jobs,
seq 512, batch 8, 8 minibatches each, SHARP / Sharded-LRTF over spilled shards with a
capped HBM budget of 1.2e9 B per GPU (4 shards per model). Synthetic tokens, GPT-2 init.
One "step" = one full pass of the workload (8 jobs x 8 minibatches x 8 samples = 512
samples) through the real executor: ParamLoad / ActPromote (pinned host -> HBM),
forward / recompute+backward on sm_100a kernels, fused Adam with streamed optimizer
state, ActDemote / GradOffload (HBM -> host).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hydra|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, rank r runs
                                                       plan device r; max over ranks)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aggregate train samples/sec + workload makespan at 1/2/4/8 B200 vs CPU ref"
DEFAULT_CONFIG = os.path.join(ROOT, "configs", "c2_gpt2small_x8.json")


def load_config(path):
    with open(path) as f:
        return json.load(f)


def workload_desc(cfg, path=DEFAULT_CONFIG):
    g = cfg["models"][0]["generator"]
    return {
        "workload": os.path.splitext(os.path.basename(path))[0],
        "jobs": len(cfg["jobs"]),
        "model": f"gpt2 d{g['d_model']} L{g['n_blocks']}",
        "global_batch": sum(j["batch_size"] for j in cfg["jobs"]),
        "seq_len": g["seq_len"],
        "minibatches_per_job": cfg["jobs"][0].get("minibatches_per_epoch", 1),
        "hbm_cap_bytes": cfg["cluster"]["devices"][0]["mem_bytes"],
        "strategy": "sharp",
        "parallelism": "task-parallel shards (no collectives)",
        "l2": "inputs larger than L2 (>=113 MB shard params stream through HBM each task)",
    }


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------- CPU leg
def reference_shard_starts(cfg):
    """Job 0's partition from the reference partitioner compiled from its own sources
    (oracle/_ref/libspillsim_ref.so); the B200 build produces the identical cut
    (tests/test_plan_parity.py)."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libspillsim_ref.so"))
    lib.ref_shard_starts.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    buf = (ctypes.c_int * 64)()
    n = lib.ref_shard_starts(json.dumps(cfg).encode(), 0, buf, 64)
    if n <= 0:
        raise RuntimeError("reference partitioner failed")
    return list(buf[:n])


CPU_ROWS = 4  # sequences per CPU sample (half a C2 minibatch: ~6 s on 16 host cores)


def cpu_sample(cfg, rows=CPU_ROWS, starts=None):
    """CPU port (oracle/gpt_oracle.c: blocked fp64-accumulating GEMMs, OpenMP over all host
    cores) of one bounded sample: `rows` sequences of job 0 minibatch 0 through all its shard
    tasks F(0..k-1), B(k-1..0) and one Adam step, with the partition of the real workload.
    Returns seconds, threads, starts."""
    import numpy as np

    from oracle import oracle as O

    if starts is None:
        starts = reference_shard_starts(cfg)
    g = cfg["models"][0]["generator"]
    m = O.make_dims(d=g["d_model"], L=g["n_blocks"], T=g["seq_len"], B=rows)
    p = O.init_params(m, O.model_key(int(cfg.get("seed", 0)), 0))
    mom, var = np.zeros_like(p), np.zeros_like(p)
    tok, tgt = O.tokens(m, int(cfg.get("seed", 0)), 0, 0)
    t0 = time.perf_counter()
    O.sharded_step(m, p, mom, var, starts, 1, 1e-4, tok, tgt)
    return time.perf_counter() - t0, O.lib().oracle_threads(), starts


# ------------------------------------------------------------------------- rank shares
def plan_share(cfg, n, rank):
    """What rank `rank` of an N-GPU run executes: the tasks the SHARP plan (G=n, the
    reference's dispatch order, sim.cpp:524-527) puts on device `rank`. With double
    buffering a job never spans two devices, so shares are disjoint job sets
    and ranks exchange nothing but the timing reduce."""
    import paper_2110_08633_b200 as P

    plan = P.plan(cfg, gpus=n)
    tasks = plan["tasks"]
    mine = [t for t, dev, _ in plan["dispatch"] if dev == rank]
    jobs = sorted({tasks[t]["job"] for t in mine})
    samples = sum(cfg["jobs"][j]["batch_size"] for t in mine for j in [tasks[t]["job"]]
                  if tasks[t]["shard"] == 0 and tasks[t]["dir"] in (0, "F", "fwd"))
    return {"tasks": mine, "jobs": jobs, "samples": samples, "dispatch_hash": plan["dispatch_hash"],
            "virtual_makespan_s": plan["makespan_s"]}


def reduce_over_ranks(dist, device, dev_time, wall, samples, h2d, d2h, launches):
    """Max of the per-rank times, sum of the per-rank work (the N>1 contract: value = units
    all ranks processed / max-over-ranks time)."""
    import torch

    t = torch.tensor([dev_time, wall], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot = torch.tensor([samples, h2d, d2h, launches], device=device, dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    return t.tolist() + tot.tolist()


# ------------------------------------------------------------------------- GPU leg
def _time_launches(torch, fn, reps=50):
    """Seconds per launch of `fn`, CUDA events on the launching stream, the launches queued
    behind a GPU spin so the events bracket back-to-back kernels (no host launch gaps; the
    executor also enqueues ahead of the GPU)."""
    for _ in range(5):
        fn()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(300_000_000)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def live_tf32_peak(torch):
    """cuBLAS TF32 8192^3 in this run (MEASURED_PEAKS.json carries bf16 only): TFLOP/s."""
    dev = torch.device("cuda")
    torch.backends.cuda.matmul.allow_tf32 = True
    X = torch.randn(8192, 8192, device=dev)
    Y = torch.randn(8192, 8192, device=dev)
    for _ in range(3):
        X @ Y
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record(s)
        X @ Y
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = False
    del X, Y
    return 2.0 * 8192 ** 3 / best / 1e12


def live_gemm_roofline(torch, cfg, peak):
    """Dominant kernel family: the tcgen05 TF32 GEMM (~65% of C2 kernel time). Two instantiations
    are timed at the workload's shapes, CUDA events on their launching stream:
      * dW(fc): C[4d x d] = dY^T X over K = b*s tokens, both operands token-major (MN-major) —
        gemm_tf32_pair_kernel<*,1,1,0>, the largest single instantiation in the C2 launch list
        (profiles/r01_launches_c2_summary.txt), with the executor's split-K workspace;
      * QKV: X[b*s, d] W^T[d, 3d] + bias, the first GEMM of every block forward.
    The top-level fields are the dW GEMM's; `traffic` = DRAM bytes per launch from the committed
    ncu --set full captures (profiles/roofline_traffic.json)."""
    from paper_2110_08633_b200 import kernels as K

    g = cfg["models"][0]["generator"]
    d = g["d_model"]
    M = g["batch_size"] * g["seq_len"]
    dev = torch.device("cuda")
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            tr = json.load(f)
        for e in tr.get("captures", [tr]):
            traffic[(e.get("name", "qkv"), tuple(e["shape"]))] = e["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    out = []
    # dW(fc): A = dY [M, 4d] (token-major => a_mn), B = X [M, d] (b_mn); C [4d, d]
    ws = torch.empty(2 * 4 * d * d, device=dev)  # the executor's split-K workspace (two 4d x d partials)
    K.gemm_config(splitk_ws=ws)
    dY = torch.randn(M, 4 * d, device=dev)
    X = torch.randn(M, d, device=dev)
    W = torch.empty(4 * d, d, device=dev)
    t = _time_launches(torch, lambda: K.gemm(dY, X, a_mn=True, b_mn=True, C=W))
    K.gemm_config(splitk_ws=None)
    fl = 2.0 * 4 * d * d * M
    out.append({"name": "dW_fc", "kernel": f"gemm_tf32_pair_kernel dW(fc) [{4*d}x{d}x{M}] MN/MN operands, split-K "
                "workspace (tcgen05 kind::tf32, cta_group::2)", "shape": [4 * d, d, M], "seconds": t, "flops": fl,
                "algorithmic_bytes": int(4 * (M * 4 * d + M * d + 4 * d * d))})
    del dY, X, W, ws
    A = torch.randn(M, d, device=dev)
    B = torch.randn(3 * d, d, device=dev)
    bias = torch.randn(3 * d, device=dev)
    C = torch.empty(M, 3 * d, device=dev)
    t = _time_launches(torch, lambda: K.gemm(A, B, C=C, bias=bias))
    fl = 2.0 * M * 3 * d * d
    out.append({"name": "qkv", "kernel": f"gemm_tf32_pair_kernel qkv [{M}x{3*d}x{d}] +bias (tcgen05 kind::tf32, "
                "cta_group::2)", "shape": [M, 3 * d, d], "seconds": t, "flops": fl,
                "algorithmic_bytes": int(4 * (M * d + 3 * d * d + 3 * d + M * 3 * d))})
    del A, B, C, bias
    recs = []
    for e in out:
        ach = e["flops"] / e["seconds"] / 1e12
        recs.append({"bound": "tensor", "kernel": e["kernel"], "achieved": round(ach, 1), "peak": round(peak, 1),
                     "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                     "peak_source": "in-run cuBLAS TF32 8192^3 (MEASURED_PEAKS.json has no TF32 figure; nominal "
                                    "dense TF32 1100)",
                     "frac_of_nominal_tf32": round(ach / 1100.0, 4),
                     "traffic": traffic.get((e["name"], tuple(e["shape"]))),
                     "algorithmic_bytes": e["algorithmic_bytes"], "launch_us": round(e["seconds"] * 1e6, 2)})
    # the bf16 precision's GEMM (tcgen05 kind::f16) against the driver-measured bf16 peak
    # (MEASURED_PEAKS.json, burst: a kernel timed alone): the C2 fc shape and GPT-2 XL's fc shape
    # (C3's block GEMMs), plain fp32 store
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16_peak = float(json.load(f)["bf16_tflops"])
    except (OSError, ValueError, KeyError):
        bf16_peak = None
    if bf16_peak:
        for name, (Mb, Nb, Kb) in (("bf16_fc_c2", (M, 4 * d, d)), ("bf16_fc_xl", (16384, 6400, 1600))):
            A = torch.randn(Mb, Kb, device=dev).to(torch.bfloat16)
            B = torch.randn(Nb, Kb, device=dev).to(torch.bfloat16)
            C = torch.empty(Mb, Nb, device=dev)
            t = _time_launches(torch, lambda: K.gemm_bf16(A, B, C=C))
            ach = 2.0 * Mb * Nb * Kb / t / 1e12
            recs.append({"bound": "tensor", "kernel": f"gemm_tf32_pair_kernel<bf16> [{Mb}x{Nb}x{Kb}] (tcgen05 kind::f16, "
                         "cta_group::2, TMA-store epilogue)", "achieved": round(ach, 1), "peak": round(bf16_peak, 1),
                         "unit": "TFLOP/s", "frac": round(ach / bf16_peak, 4),
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (driver-measured cuBLAS bf16 8192^3, burst)",
                         "traffic": traffic.get((name, (Mb, Nb, Kb))),
                         "algorithmic_bytes": int(2 * (Mb * Kb + Nb * Kb) + 4 * Mb * Nb),
                         "launch_us": round(t * 1e6, 2)})
            del A, B, C
    top = dict(recs[0])
    top["others"] = recs[1:]
    return top


def plan_roofline(plan, cfg, peak_tflops, bw_dn, bw_up, G):
    """North-star shard roofline, computed from the plan's ShardTasks:
    sum_tau max(F_tau / P, H2D_tau / BW_dn, D2H_tau / BW_up) / G, with F_tau the cost-model
    FLOP of the task (compute_s x device_reference_flops, strategies.cpp:753,775), H2D_tau =
    param_load + activation_in bytes and D2H_tau = activation_out + grad_offload bytes (the
    ShardTask fields of build_sharp, strategies.cpp:746-776), P the in-run TF32 peak and BW the
    probed duplex link rates of this box. Also returns the totals."""
    F_ref = {m["name"]: m["generator"].get("device_reference_flops", 1e15) for m in cfg["models"]}
    P_ = peak_tflops * 1e12
    total = flops = h2d = d2h = 0.0
    bound = {"compute": 0.0, "h2d": 0.0, "d2h": 0.0}
    for t in plan["tasks"]:
        F = t["compute_s"] * F_ref[cfg["jobs"][t["job"]]["model"]]
        hi = t["param_load_bytes"] + t["activation_in_bytes"]
        ho = t["activation_out_bytes"] + t["grad_offload_bytes"]
        terms = {"compute": F / P_, "h2d": hi / bw_dn, "d2h": ho / bw_up}
        k = max(terms, key=terms.get)
        bound[k] += terms[k]
        total += terms[k]
        flops += F
        h2d += hi
        d2h += ho
    return total / G, flops, h2d, d2h, {k: round(v / G, 5) for k, v in bound.items()}


def probe_link(torch, nbytes=1 << 29, reps=4):
    """Pinned host<->HBM copy rates of this box (GB/s): each direction alone, then both at once on two
    streams (the duplex rate a shard pass can use). Timed with CUDA events on the copying streams."""
    dev = torch.device("cuda", torch.cuda.current_device())
    hs = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    hd = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    ds = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dd = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s_dn, s_up = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(which):
        torch.cuda.synchronize()
        ev = {}
        for name, s in (("h2d", s_dn), ("d2h", s_up)):
            if name not in which:
                continue
            with torch.cuda.stream(s):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(reps):
                    (ds.copy_(hs, non_blocking=True) if name == "h2d" else hd.copy_(dd, non_blocking=True))
                b.record(s)
                ev[name] = (a, b)
        torch.cuda.synchronize()
        return {k: round(nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9, 2) for k, (a, b) in ev.items()}

    timed(("h2d", "d2h"))  # warm
    one = {**timed(("h2d",)), **timed(("d2h",))}
    both = timed(("h2d", "d2h"))
    return {"h2d_GBps": one["h2d"], "d2h_GBps": one["d2h"],
            "duplex_h2d_GBps": both["h2d"], "duplex_d2h_GBps": both["d2h"],
            "method": f"{reps} x {nbytes >> 20} MiB pinned copies per direction, CUDA events on the copy streams"}


def run_hydra(args, cfg):
    import torch
    import paper_2110_08633_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    n = max(args.gpus, world)
    device_ids = [0] * n
    device_ids[rank] = local if world > 1 else 0
    req = dict(strategy="sharp", gpus=n, run_devices=[rank], device_ids=device_ids,
               passes=args.steps + 1, warmup_passes=args.warmup, host_opt_fraction=args.host_opt_fraction,
               opt_state=args.opt_state)
    if args.exec_json:  # executor tuning knobs (ExecOptions fields of the C-ABI request), e.g. '{"opt_chunk_floats": 4194304}'
        req.update(json.loads(args.exec_json))
    if args.schedule == "dynamic":
        # one process drives every GPU (one worker thread each) so the live scheduler sees them all
        if world > 1:
            raise SystemExit("--schedule dynamic runs all GPUs from one process: launch without torchrun")
        req.update(schedule="dynamic", run_devices=list(range(n)), device_ids=list(range(n)))
    t_setup = time.perf_counter()
    ex = P.Executor(cfg, **req)
    setup_s = time.perf_counter() - t_setup
    launches0 = P.kernel_launches()
    ex.run(args.warmup, timed=False)
    launches_w = P.kernel_launches()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    w0 = time.perf_counter()
    res = ex.run(args.steps, timed=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    cl = clocks.stop()
    launches_t = P.kernel_launches() - launches_w
    dev_time = sum(res["pass_seconds"])
    samples = res["samples_per_pass"] * args.steps
    st = res["stats"]
    if dist:
        dev_time, wall, samples, h2d, d2h, launches_t = reduce_over_ranks(
            dist, "cuda", dev_time, wall, samples, st["h2d_bytes_per_pass"], st["d2h_bytes_per_pass"], launches_t)
    else:
        h2d, d2h = st["h2d_bytes_per_pass"], st["d2h_bytes_per_pass"]
    if rank != 0:
        ex.close()
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return None
    value = samples / dev_time
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "samples/s",
        "n_gpus": n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_time / args.steps * 1e3, 3),
        "makespan_s": round(dev_time / args.steps, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "fp32 (tf32 tensor-core GEMMs)",
        "data": "synthetic tokens (splitmix64), GPT-2 random init",
        "config": dict(workload_desc(cfg, args.config), host_opt_fraction=args.host_opt_fraction,
                       opt_state=args.opt_state, schedule=args.schedule),
        "e2e": {"value": round(samples / wall, 3), "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "note": "host wall clock around the public hy_executor_run call; every step moves params, "
                        "optimizer state, activations and tokens host->HBM and results back (losses read back per step)"},
        "gpu_launches": int(launches_t),
        "clocks": cl,
        "plan": {"dispatch_hash": res["dispatch_hash"], "virtual_makespan_s": res["virtual_makespan_s"],
                 "shard_starts": res["shard_starts"][0]},
        "bytes_per_step": {k: v for k, v in st.items() if k.endswith("_per_pass")},
        "arena_bytes": st["arena_bytes"],
        "setup_s": round(setup_s, 2),
        "losses_job0_last_step": [round(x, 5) for x in res["losses"][0][-cfg["jobs"][0]["minibatches_per_epoch"]:]]
        if res["losses"] and res["losses"][0] else [],
        "device_busy_frac": round(st["device_busy_s_last_pass"] / res["pass_seconds"][-1], 4),
    }
    # Overlap: one more pass with the interval log (two event records per copy /
    # op), outside the timed region: copy-only link time per direction, compute time, and
    # overlap_frac = 1 - exposed transfer / total transfer on this GPU.
    links = None
    try:
        lres = ex.run(1, timed=True, interval_log=True)
        links = lres.get("links")
    except Exception as e:  # pragma: no cover
        links = [{"error": str(e)}]
    try:
        lp = probe_link(torch)
    except Exception as e:  # pragma: no cover
        lp = {"error": str(e)}
    try:
        peak = live_tf32_peak(torch)
        out["roofline"] = live_gemm_roofline(torch, cfg, peak)
    except Exception as e:  # pragma: no cover
        peak = None
        out["roofline"] = {"error": str(e)}
    meas = dev_time / args.steps
    sr = {"bound": "host_link", "measured_makespan_s": round(meas, 5),
          "cost_model_virtual_makespan_s": round(res["virtual_makespan_s"], 5),
          "cost_model_virtual_frac": round(res["virtual_makespan_s"] / meas, 4),
          "cost_model_note": "the reference engine's virtual makespan (55 GB/s links, configs' 1 PF/s): a "
                             "cost-model approximation, not the roofline",
          "achieved_h2d_GBps": round(h2d / meas / 1e9, 2), "achieved_d2h_GBps": round(d2h / meas / 1e9, 2),
          "link_probe": lp}
    if peak and "duplex_h2d_GBps" in lp:
        bw_dn, bw_up = lp["duplex_h2d_GBps"] * 1e9, lp["duplex_d2h_GBps"] * 1e9
        plan = P.plan(cfg, gpus=n)
        if world > 1:  # this rank's share of the plan (the per-GPU roofline of device `rank`)
            mine = {t for t, dev, _ in plan["dispatch"] if dev == rank}
            plan = dict(plan, tasks=[t for i, t in enumerate(plan["tasks"]) if i in mine])
        G = 1 if world > 1 else n
        roof, F_tot, h2d_m, d2h_m, by = plan_roofline(plan, cfg, peak, bw_dn, bw_up, G)
        sr.update({
            "definition": "sum over the plan's ShardTasks of max(F_tau/P, H2D_tau/BW_dn, D2H_tau/BW_up) / G; "
                          "cost-model FLOP and bytes (SURVEY §8d), P = in-run cuBLAS TF32 peak, BW = this box's "
                          "probed duplex pinned-copy rates",
            "roofline_makespan_s": round(roof, 5), "frac": round(roof / meas, 4),
            "peak_tflops": round(peak, 1), "bw_h2d_GBps": lp["duplex_h2d_GBps"], "bw_d2h_GBps": lp["duplex_d2h_GBps"],
            "bound_by_term_s": by, "model_flops_per_pass": F_tot,
            "model_h2d_bytes_per_pass": h2d_m, "model_d2h_bytes_per_pass": d2h_m})
        # physical: the bytes actually moved (Adam m, v, tied wte, biases; minus what the caches
        # elide) and the FLOP at the same peak — a pass-level bound (per-task actual bytes are not
        # attributable once caches and streams interleave)
        t_phys = max(F_tot / (peak * 1e12), h2d / bw_dn, d2h / bw_up)
        sr["physical"] = {"definition": "max(model FLOP / P, actual H2D bytes / BW_dn, actual D2H bytes / BW_up) "
                                        "per pass", "bound_s": round(t_phys, 5), "frac": round(t_phys / meas, 4),
                          "flop_s": round(F_tot / (peak * 1e12), 5), "h2d_s": round(h2d / bw_dn, 5),
                          "d2h_s": round(d2h / bw_up, 5)}
        sr["physical_frac"] = sr["physical"]["frac"]
    if links:
        sr["links"] = links
        ok = [l for l in links if "overlap_frac" in l]
        if ok:
            sr["overlap_frac"] = round(min(l["overlap_frac"] for l in ok), 4)
            sr["link_busy_frac"] = round(max(l["link_busy_s"] / l["pass_s"] for l in ok), 4)
    out["shard_roofline"] = sr
    ex.close()
    if not args.no_variants and world == 1:
        # the same workload with (a) Adam moments stored / streamed as bf16 (fp32 master params,
        # TF32 GEMMs; parity stated separately, tests/test_executor_gpu.py::test_bf16_optimizer_state)
        # and (b) 3xTF32 ("fp32") GEMMs, the precision that holds 2e-4 on parameters at every
        # BASELINE shape (tests/test_baseline_shapes_gpu.py)
        out["variants"] = {}
        other = "bf16" if args.opt_state == "fp32" else "fp32"
        # and (c) the "bf16" precision: block GEMMs on bf16 operands (tcgen05 kind::f16), parity
        # against the bf16-emulating oracle in tests/test_baseline_shapes_gpu.py — alone and with
        # bf16 Adam moments
        for name, over in ((f"opt_state_{other}", {"opt_state": other}), ("precision_fp32", {"precision": "fp32"}),
                           ("precision_bf16", {"precision": "bf16"}),
                           ("precision_bf16_opt_state_bf16", {"precision": "bf16", "opt_state": "bf16"})):
            vex = P.Executor(cfg, **dict(req, **over))
            vex.run(args.warmup, timed=False)
            torch.cuda.synchronize()
            vres = vex.run(args.steps, timed=True)
            vt = sum(vres["pass_seconds"])
            out["variants"][name] = {
                "value": round(vres["samples_per_pass"] * args.steps / vt, 3), "unit": "samples/s",
                "ms_per_step": round(vt / args.steps * 1e3, 3),
                "h2d_bytes_per_step": int(vres["stats"]["h2d_bytes_per_pass"]),
                "d2h_bytes_per_step": int(vres["stats"]["d2h_bytes_per_pass"])}
            if "roofline_makespan_s" in out["shard_roofline"]:
                out["variants"][name]["shard_roofline_frac"] = round(
                    out["shard_roofline"]["roofline_makespan_s"] / (vt / args.steps), 4)
            vex.close()
    if not args.no_cpu_baseline:
        try:
            secs, cores, _ = cpu_sample(cfg, starts=res["shard_starts"][0])
            out["cpu_baseline"] = {"value": round(CPU_ROWS / secs, 5), "unit": "samples/s", "cores": cores,
                                   "kind": "port",
                                   "sample": f"{CPU_ROWS} sequences (of 8) of job 0 minibatch 0 through all shard tasks "
                                             f"F+B + one Adam step on the CPU oracle ({secs:.1f} s)"}
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_reference(args, cfg):
    """Reference arm: the reference's path on the host CPU. The reference (spillsim) only
    simulates training, so the timed CPU implementation is the oracle port of the same
    shard execution (oracle/gpt_oracle.c, OpenMP, all host threads), each step a bounded
    sample of the workload; the reference's own planner (oracle/_ref, compiled from the
    reference sources) is timed alongside for completeness."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    for _ in range(args.warmup):
        cpu_sample(cfg)
    times = []
    cores = 0
    for _ in range(args.steps):
        s, cores, _ = cpu_sample(cfg)
        times.append(s)
    value = CPU_ROWS / statistics.mean(times)
    out = {"metric": METRIC, "impl": "reference", "value": round(value, 5), "unit": "samples/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(statistics.mean(times) * 1e3, 1), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "fp32 (fp64 accumulate)",
           "data": "synthetic tokens (splitmix64), GPT-2 random init", "config": workload_desc(cfg, args.config),
           "cpu_baseline": {"value": round(value, 5), "unit": "samples/s", "cores": cores, "kind": "port",
                            "sample": f"{CPU_ROWS} sequences (of 8) of job 0 minibatch 0 through all shard tasks "
                                      "F+B + one Adam step, per step"},
           "e2e": {"value": round(value, 5), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libspillsim_ref.so")
    if os.path.exists(ref_so):
        import ctypes
        lib = ctypes.CDLL(ref_so)
        lib.ref_run_strategy.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                         ctypes.c_char_p, ctypes.c_int]
        mk, wall = ctypes.c_double(), ctypes.c_double()
        msg = ctypes.create_string_buffer(256)
        rc = lib.ref_run_strategy(json.dumps(cfg).encode(), b"sharp", args.gpus, ctypes.byref(mk),
                                  ctypes.byref(wall), msg, 256)
        if rc == 0:
            out["reference_planner"] = {"virtual_makespan_s": mk.value, "wall_s": wall.value,
                                        "what": "reference run_strategy (simulated time) compiled from "
                                                "/root/reference sources; no tensor execution"}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hydra", choices=["hydra", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # optimizer placement (the reference keeps optimizer state host-side): the
    # fraction of each job's params updated by the host; the rest stream their fp32 moments
    # through HBM and are updated on the GPU
    ap.add_argument("--host-opt-fraction", type=float, default=0.0)
    ap.add_argument("--opt-state", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--no-variants", action="store_true", help="skip the other opt-state measurement")
    ap.add_argument("--schedule", default="plan", choices=["plan", "dynamic"],
                    help="plan: replay the reference engine's dispatch log (default); dynamic: the SHARP "
                         "scheduler driven live by measured completions, all GPUs in this one process")
    ap.add_argument("--exec-json", default="", help="extra executor request fields (JSON object)")
    args = ap.parse_args()
    cfg = load_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_hydra(args, cfg)


if __name__ == "__main__":
    main()
