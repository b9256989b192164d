"""Host-side cost per launch from C++ (no Python in the loop): GEMM vs LayerNorm."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200._lib import lib
dev = torch.device("cuda")
a = torch.randn(128 * 64, device=dev); b = torch.randn(128 * 64, device=dev); c = torch.empty(128 * 128, device=dev)
s = torch.cuda.current_stream().cuda_stream
for kind, name in ((0, "gemm"), (1, "layernorm")):
    lib().hy_host_launch_us(s, kind, 200, a.data_ptr(), b.data_ptr(), c.data_ptr())
    torch.cuda.synchronize()
    us = lib().hy_host_launch_us(s, kind, 2000, a.data_ptr(), b.data_ptr(), c.data_ptr())
    torch.cuda.synchronize()
    print(name, "host us/launch %.2f" % us)
