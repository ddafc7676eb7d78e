"""GPT-2 fc2 dgrad with the gelu'-product epilogue (act 6) and the fc_b column sums, and the GELU
forward (act 5) of the fc projection, timed at the step shapes (M = 16384, d = 768, f = 3072)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

M, d, f = 16384, 768, 3072


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


dy = torch.randn(M, d, device="cuda").bfloat16()
w2 = (torch.randn(d, f, device="cuda") * d ** -0.5).bfloat16()
aux = (torch.rand(M, f, device="cuda") * 1.2).bfloat16()
dh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
cs = torch.zeros(f, device="cuda")
x = torch.randn(M, d, device="cuda").bfloat16()
w1 = (torch.randn(f, d, device="cuda") * d ** -0.5).bfloat16()
b1 = torch.zeros(f, device="cuda").bfloat16()
h = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
hp = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
fl = 2 * M * d * f
us = t(lambda: ops.linear_dgrad(dy, w2, out=dh, act=6, aux=aux, colsum_out=cs))
print(f"fc2 dgrad act6+colsum {us:.1f} us {fl / us / 1e6:.0f} TF/s")
us = t(lambda: ops.linear_dgrad(dy, w2, out=dh))
print(f"fc2 dgrad plain       {us:.1f} us {fl / us / 1e6:.0f} TF/s")
us = t(lambda: ops.linear(x, w1, bias=b1, out=h, act=5, aux=hp))
print(f"fc fwd gelu act5      {us:.1f} us {fl / us / 1e6:.0f} TF/s")
us = t(lambda: ops.linear(x, w1, bias=b1, out=h))
print(f"fc fwd bias only      {us:.1f} us {fl / us / 1e6:.0f} TF/s")
