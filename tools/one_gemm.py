"""Run one GEMM shape a few times (for ncu captures): python tools/one_gemm.py M N K [amn bmn]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops
M, N, K = (int(x) for x in sys.argv[1:4])
amn = len(sys.argv) > 4 and sys.argv[4] == "1"
bmn = len(sys.argv) > 5 and sys.argv[5] == "1"
a = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
b = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.gemm(a, b, a_mn=amn, b_mn=bmn, M=M, N=N, K=K, out=c)
torch.cuda.synchronize()
print("ok")
