"""Llama-1B fused SwiGLU-backward GEMM (dgu from dy @ W2 and the saved gu), a few launches (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

M, F, d = 16384, 8192, 2048
dy = torch.randn(M, d, device="cuda").bfloat16()
w2 = (torch.randn(d, F, device="cuda") * d ** -0.5).bfloat16()
gu = torch.randn(M, 2 * F, device="cuda").bfloat16()
dgu = torch.empty_like(gu)
for _ in range(4):
    ops.linear_dgrad_swiglu(dy, w2, gu, dgu)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.linear_dgrad_swiglu(dy, w2, gu, dgu)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"swiglu_bwd gemm {ms * 1e3:.1f} us  {2 * M * F * d / ms / 1e9:.1f} TF/s")
if len(sys.argv) > 1:  # reference: the plain dgrad GEMM of the same shape (dh stored, no SwiGLU epilogue)
    dh = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    for _ in range(4):
        ops.linear_dgrad(dy, w2, out=dh)
    s.record()
    for _ in range(10):
        ops.linear_dgrad(dy, w2, out=dh)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"plain dgrad gemm {ms * 1e3:.1f} us  {2 * M * F * d / ms / 1e9:.1f} TF/s")
