"""Probe the GPU box: host cores/RAM, pinned H2D/D2H bandwidth, TF32 matmul peak."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["affinity"] = len(os.sched_getaffinity(0))
except Exception:
    pass
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK,MEMORY,PCIE"], capture_output=True, text=True).stdout[-4000:]
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
res = {}
for mb in (64, 256, 1024):
    n = mb * (1 << 20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); 
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        res[f"{name}_{mb}MB_GBs"] = 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # duplex
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    res[f"duplex_{mb}MB_GBs_each"] = 5 * n / dt / 1e9
out["link"] = res
# pin cost
t0 = time.perf_counter(); big = torch.empty(4 << 30, dtype=torch.uint8).pin_memory(); out["pin_4GB_s"] = time.perf_counter() - t0
del big
# tf32 matmul
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(8192, 8192, device=dev); b = torch.randn(8192, 8192, device=dev)
for _ in range(3): a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): a @ b
e1.record(); torch.cuda.synchronize()
out["tf32_tflops"] = 10 * 2 * 8192**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
torch.backends.cuda.matmul.allow_tf32 = False
e0.record()
for _ in range(3): a @ b
e1.record(); torch.cuda.synchronize()
out["fp32_tflops"] = 3 * 2 * 8192**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "smi")}, indent=1))
