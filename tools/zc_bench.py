"""Zero-copy optimizer kernel vs copy engines (diagnostics): link GB/s of hy_adam_host_state
at several grid sizes, next to a DMA H2D+D2H of the same bytes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K

n = 32 << 20
dev = "cuda"
p = torch.randn(n, device=dev); g = torch.randn(n, device=dev) * 1e-3
for dt in (torch.float32, torch.bfloat16):
    m = torch.zeros(n, dtype=dt).pin_memory(); v = torch.zeros(n, dtype=dt).pin_memory(); ph = torch.empty(n).pin_memory()
    es = m.element_size()
    for grid in (16, 32, 64, 96, 148, 296, 592):
        K.adam_host_state(p, g, m, v, ph, 1e-4, 1, grid=grid)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            K.adam_host_state(p, g, m, v, ph, 1e-4, 2, grid=grid)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3e3
        print(json.dumps({"dtype": str(dt), "grid": grid, "ms": round(t * 1e3, 2), "in_GBps": round(2 * es * n / t / 1e9, 1),
                          "out_GBps": round((4 + 2 * es) * n / t / 1e9, 1)}), flush=True)
hb = torch.empty(n * 3, dtype=torch.float32).pin_memory(); db = torch.empty(n * 3, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
with torch.cuda.stream(s1):
    db[: 2 * n].copy_(hb[: 2 * n], non_blocking=True)
with torch.cuda.stream(s2):
    hb[: 3 * n].copy_(db[: 3 * n], non_blocking=True)
torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3
print(json.dumps({"dma_duplex_same_bytes_ms": round(t * 1e3, 2), "in_GBps": round(8 * n / t / 1e9, 1), "out_GBps": round(12 * n / t / 1e9, 1)}))
