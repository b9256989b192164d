import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, sys
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda:0")
M, N, Kd = 128, 128, 32
A = torch.randn(M, Kd, device=dev); B = torch.randn(N, Kd, device=dev)
ref = A @ B.T
for a_mn, b_mn in ((False, False), (True, False), (False, True), (True, True)):
    Ain = A.T.contiguous() if a_mn else A
    Bin = B.T.contiguous() if b_mn else B
    C = torch.full((M, N), 7.0, device=dev)
    K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C)
    torch.cuda.synchronize()
    print(a_mn, b_mn, "rel", ((C - ref).norm() / ref.norm()).item(), "C[0,:4]", C[0, :4].tolist(), "ref", ref[0, :4].tolist())
    # try to find a permutation relation: correlate C with ref^T
    print("   vs ref.T rel", ((C - ref.T).norm() / ref.norm()).item())
