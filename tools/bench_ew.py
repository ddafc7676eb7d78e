"""Bandwidth kernels at the Llama-1B / GPT-2 step shapes: achieved GB/s vs the measured HBM peak.
    python tools/bench_ew.py"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import ops  # noqa: E402
from paper_2602_08387_b200.model import PRESETS, rope_tables  # noqa: E402
from tools.bench_kernels import peaks, time_it  # noqa: E402

hbm, _ = peaks()
rows = []


def rec(name, ms, nbytes):
    gbs = nbytes / (ms / 1e3) / 1e9
    rows.append({"name": name, "us": round(ms * 1e3, 1), "GBps": round(gbs, 1), "frac_of_hbm": round(gbs / hbm, 3)})
    print(json.dumps(rows[-1]), flush=True)


dev = "cuda"
for D, M in ((768, 16384), (2048, 16384)):
    x = torch.randn(M, D, device=dev)
    g = torch.ones(D, device=dev).bfloat16()
    b = torch.zeros(D, device=dev).bfloat16()
    y = torch.empty(M, D, device=dev, dtype=torch.bfloat16)
    mean, rstd = torch.empty(M, device=dev), torch.empty(M, device=dev)
    xc = torch.empty_like(x)
    dy = torch.randn(M, D, device=dev).bfloat16()
    dx = torch.zeros(M, D, device=dev)
    dxb = torch.empty(M, D, device=dev, dtype=torch.bfloat16)
    dg, db, ds = (torch.zeros(D, device=dev) for _ in range(3))
    if D == 768:
        rec(f"layernorm_fwd D={D}", time_it(lambda: ops.layernorm_fwd(x, g, b, 1e-5, y, mean, rstd, x_copy=xc)),
            M * D * (4 + 2 + 4))
        rec(f"layernorm_bwd D={D}", time_it(lambda: ops.layernorm_bwd(x, dy, g, mean, rstd, dx, dxb, dg, db, ds)),
            M * D * (4 + 2 + 4 + 4 + 2))
    else:
        rec(f"rmsnorm_fwd D={D}", time_it(lambda: ops.rmsnorm_fwd(x, g, 1e-5, y, rstd, x_copy=xc)), M * D * (4 + 2 + 4))
        yr = torch.randn(M, D, device=dev).bfloat16()
        rec(f"rmsnorm_fwd+res D={D}", time_it(lambda: ops.rmsnorm_fwd_res(x, yr, g, 1e-5, y, rstd, xc)),
            M * D * (4 + 2 + 4 + 2))
        rec(f"rmsnorm_bwd D={D}", time_it(lambda: ops.rmsnorm_bwd(x, dy, g, rstd, dx, dxb, dg, ds)),
            M * D * (4 + 2 + 4 + 4 + 2))
cfg = PRESETS["llama-1b"]
M, F = 16384, cfg.d_ff
gu = torch.randn(M, 2 * F, device=dev).bfloat16()
h = torch.empty(M, F, device=dev, dtype=torch.bfloat16)
dh = torch.randn(M, F, device=dev).bfloat16()
dgu = torch.empty_like(gu)
rec("swiglu_fwd 1B", time_it(lambda: ops.swiglu_fwd(gu, h)), M * F * 2 * 3)
rec("swiglu_bwd 1B", time_it(lambda: ops.swiglu_bwd(gu, dh, dgu)), M * F * 2 * 5)
qkv = torch.randn(M, cfg.qkv_dim, device=dev).bfloat16()
cos, sin = rope_tables(cfg, 4096, dev)
nh = cfg.n_head + cfg.n_kv_head
rec("rope 1B (k heads only, the backward's remaining launch)",
    time_it(lambda: ops.rope(qkv[:, cfg.n_head * cfg.head_dim:], 4096, cfg.n_kv_head, cfg.head_dim, cos, sin)),
    M * cfg.n_kv_head * cfg.head_dim * 2 * 2)
rec("rope 1B (q+k heads)", time_it(lambda: ops.rope(qkv, 4096, nh, cfg.head_dim, cos, sin)),
    M * nh * cfg.head_dim * 2 * 2)
V = 50257
logits = torch.randn(16384, 50304, device=dev).bfloat16()
tgt = torch.randint(0, V, (16384,), device=dev)
rec("cross_entropy GPT-2", time_it(lambda: ops.cross_entropy(logits, V, tgt, grad_scale=1.0 / 16384)),
    16384 * 50304 * 2 * 3)
del logits
V1 = cfg.vocab_size
logits = torch.randn(16384, cfg.padded_vocab, device=dev).bfloat16()
tgt = torch.randint(0, V1, (16384,), device=dev)
rec("cross_entropy Llama-1B", time_it(lambda: ops.cross_entropy(logits, V1, tgt, grad_scale=1.0 / 16384)),
    16384 * cfg.padded_vocab * 2 * 3)
del logits
wte = torch.randn(cfg.padded_vocab, cfg.d_model, device=dev).bfloat16()
tok = torch.randint(0, V1, (16384,), device=dev)
xe = torch.empty(16384, cfg.d_model, device=dev)
rec("embedding_fwd Llama-1B", time_it(lambda: ops.embedding_fwd(tok, wte, None, 4096, out=xe)),
    16384 * cfg.d_model * (2 + 4))
n = 124_000_000
p, m_, v_, gr = (torch.randn(n, device=dev) for _ in range(4))
pb = torch.empty(n, device=dev, dtype=torch.bfloat16)
rec("adamw 124M", time_it(lambda: ops.adamw(p, m_, v_, gr, pb, 5, 1e-4, 0.9, 0.95, 1e-8, 0.1)), n * 30)
dq = torch.randn(16384, 2304, device=dev).bfloat16()
dhh = torch.randn(16384, 3072, device=dev).bfloat16()
ob = torch.zeros(3072, device=dev)
rec("colsum qkv_b (16384x2304 bf16)", time_it(lambda: ops.colsum_accumulate(dq, ob[:2304])), 16384 * 2304 * 2)
rec("colsum fc_b (16384x3072 bf16)", time_it(lambda: ops.colsum_accumulate(dhh, ob)), 16384 * 3072 * 2)
