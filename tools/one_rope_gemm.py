"""Llama-1B QKV projection (M = 16384, N = 3072, K = 2048) with the RoPE epilogue vs the plain
GEMM of the same shape (same output layout), CUDA-event timed.

    python tools/one_rope_gemm.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402
from paper_2602_08387_b200.model import PRESETS, rope_tables  # noqa: E402

cfg = PRESETS["llama-1b"]
M, K = 16384, cfg.d_model
N = cfg.qkv_dim
x = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(N, K, device="cuda") * K ** -0.5).bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
cos, sin = rope_tables(cfg, 4096, "cuda")
rope_cols = (cfg.n_head + cfg.n_kv_head) * cfg.head_dim


def timed(f, reps=20):
    for _ in range(4):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for _ in range(2):
    ur = timed(lambda: ops.linear_rope(x, w, out, 4096, cfg.head_dim, rope_cols, cos, sin))
    up = timed(lambda: ops.linear(x, w, out=out))
    print(f"rope gemm {ur:.1f} us ({2 * M * N * K / ur / 1e6:.0f} TF/s)   plain {up:.1f} us ({2 * M * N * K / up / 1e6:.0f} TF/s)")
