"""Llama-1B fused gate|up GEMM + SwiGLU forward (gu, h from x @ W13^T), timed; `plain` adds the plain GEMM."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

M, F, d = 16384, 8192, 2048
x = torch.randn(M, d, device="cuda").bfloat16()
w = (torch.randn(2 * F, d, device="cuda") * d ** -0.5).bfloat16()
gu = torch.empty(M, 2 * F, device="cuda", dtype=torch.bfloat16)
h = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


ms = timeit(lambda: ops.linear_swiglu(x, w, gu, h))
print(f"swiglu_fwd gemm {ms * 1e3:.1f} us  {2 * M * 2 * F * d / ms / 1e9:.1f} TF/s")
if len(sys.argv) > 1:
    ms = timeit(lambda: ops.linear(x, w, out=gu))
    print(f"plain gemm {ms * 1e3:.1f} us  {2 * M * 2 * F * d / ms / 1e9:.1f} TF/s")
