"""Run causal attention fwd(+bwd) once at a model shape (for ncu captures).

    [DH=128] python tools/one_attn.py B T Hq Hkv [bwd]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

B, T, Hq, Hkv = (int(x) for x in sys.argv[1:5])
bwd = len(sys.argv) > 5
dh = int(os.environ.get("DH", "64"))
qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device="cuda").bfloat16()
for _ in range(2):
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    if bwd:
        do = torch.randn_like(o)
        ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
fl = 4.0 * B * Hq * dh * T * T / 2
print(f"attn_fwd {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s")
if bwd:
    s.record()
    for _ in range(5):
        ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"attn_bwd {ms:.3f} ms {2.5 * fl / ms / 1e9:.1f} TF/s")
