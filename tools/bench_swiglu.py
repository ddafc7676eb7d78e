"""Llama-1B MLP: fused SwiGLU GEMMs vs the unfused GEMM + SwiGLU kernel chain (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402
from tools.bench_kernels import time_it  # noqa: E402

M, F, K = 16384, 8192, 2048
x = torch.randn(M, K, device="cuda").bfloat16()
w13 = (torch.randn(2 * F, K, device="cuda") * K ** -0.5).bfloat16()
gu, h = torch.empty(M, 2 * F, device="cuda", dtype=torch.bfloat16), torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
dy = torch.randn(M, K, device="cuda").bfloat16()
w2 = (torch.randn(K, F, device="cuda") * K ** -0.5).bfloat16()
dh = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
dgu = torch.empty_like(gu)
un_f = time_it(lambda: (ops.linear(x, w13, out=gu), ops.swiglu_fwd(gu, h)))
fu_f = time_it(lambda: ops.linear_swiglu(x, w13, gu, h))
un_b = time_it(lambda: (ops.linear_dgrad(dy, w2, out=dh), ops.swiglu_bwd(gu, dh, dgu)))
fu_b = time_it(lambda: ops.linear_dgrad_swiglu(dy, w2, gu, dgu))
print(f"fwd unfused {un_f:.3f} ms fused {fu_f:.3f} ms | bwd unfused {un_b:.3f} ms fused {fu_b:.3f} ms")
