"""GPT-2 fc forward GEMM with the bias+GELU epilogue (and optionally plain), for ncu captures.
    python tools/one_gelu_gemm.py [act]   act: 1 = bias+GELU (default), 0 = plain, 2 = dGELU dgrad"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

act = int(sys.argv[1]) if len(sys.argv) > 1 else 1
M, d, f = 16384, 768, 3072
x = torch.randn(M, d, device="cuda").bfloat16()
w = torch.randn(f, d, device="cuda").bfloat16()
b = torch.randn(f, device="cuda").bfloat16()
h = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
aux = torch.randn(M, f, device="cuda").bfloat16()
dy = torch.randn(M, d, device="cuda").bfloat16()
w2 = torch.randn(d, f, device="cuda").bfloat16()
for _ in range(3):
    if act == 1:
        ops.linear(x, w, bias=b, out=h, act=1, aux=aux)
    elif act == 2:
        ops.linear_dgrad(dy, w2, out=h, act=2, aux=aux)
    else:
        ops.linear(x, w, out=h)
torch.cuda.synchronize()
print("ok")
