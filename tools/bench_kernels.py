"""Kernel microbenchmarks on one B200: CUDA-event timing on the launching stream.

    python tools/bench_kernels.py gemm       # model GEMM shapes, TFLOP/s vs measured peak
"""

from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_08387_b200 import ops  # noqa: E402


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"]
    except Exception:
        return 6650.0, 1590.0


def time_it(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def bench_gemm():
    _, tf_peak = peaks()
    rows = []
    shapes = [
        ("gpt2.qkv.fwd", 16384, 2304, 768, False, False),
        ("gpt2.fc.fwd", 16384, 3072, 768, False, False),
        ("gpt2.proj.fwd", 16384, 768, 3072, False, False),
        ("gpt2.head.fwd", 16384, 50304, 768, False, False),
        ("gpt2.fc.dgrad", 16384, 768, 3072, False, True),
        ("gpt2.fc.wgrad", 3072, 768, 16384, True, True),
        ("llama1b.gateup.fwd", 16384, 16384, 2048, False, False),
        ("llama1b.down.fwd", 16384, 2048, 8192, False, False),
        ("llama1b.head.fwd", 16384, 128256, 2048, False, False),
        ("square8192", 8192, 8192, 8192, False, False),
    ]
    for name, M, N, K, amn, bmn in shapes:
        a = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
        b = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = time_it(lambda: ops.gemm(a, b, a_mn=amn, b_mn=bmn, M=M, N=N, K=K, out=c))
        tf = 2.0 * M * N * K / ms / 1e9
        # torch (cuBLAS) on the same shape for context
        A = a.t() if amn else a
        B = b if bmn else b.t()
        ms_t = time_it(lambda: torch.matmul(A, B))
        rows.append({"name": name, "M": M, "N": N, "K": K, "ms": round(ms, 4), "tflops": round(tf, 1),
                     "frac_of_peak": round(tf / tf_peak, 3), "cublas_tflops": round(2.0 * M * N * K / ms_t / 1e9, 1)})
        print(json.dumps(rows[-1]), flush=True)
    return rows


def bench_epilogues():
    """The GPT-2 step's GEMMs with their fused epilogues (bias / GELU / dGELU / fp32 residual add)."""
    rows = []
    M, d, f = 16384, 768, 3072
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    w_fc = torch.randn(f, d, device="cuda", generator=g).bfloat16()
    b_fc = torch.randn(f, device="cuda", generator=g).bfloat16()
    h = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    hpre = torch.empty_like(h)
    dy = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    w_fc2 = torch.randn(d, f, device="cuda", generator=g).bfloat16()
    b_d = torch.randn(d, device="cuda", generator=g).bfloat16()
    resid = torch.zeros(M, d, device="cuda")
    dh = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    b_acc = torch.zeros(f, device="cuda")
    o = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    w_o = torch.randn(d, d, device="cuda", generator=g).bfloat16()
    cases = [
        ("fc.fwd+bias+gelu", M, f, d, lambda: ops.linear(x, w_fc, bias=b_fc, out=h, act=1, aux=hpre)),
        ("fc.fwd plain", M, f, d, lambda: ops.linear(x, w_fc, out=h)),
        ("fc2.dgrad+dgelu", M, f, d, lambda: ops.linear_dgrad(dy, w_fc2, out=dh, act=2, aux=hpre)),
        ("fc2.dgrad plain", M, f, d, lambda: ops.linear_dgrad(dy, w_fc2, out=dh)),
        ("fc.fwd+bias+gelu, aux=gelu' (act 5)", M, f, d,
         lambda: ops.linear(x, w_fc, bias=b_fc, out=h, act=5, aux=hpre)),
        ("fc2.dgrad x aux (act 6)", M, f, d, lambda: ops.linear_dgrad(dy, w_fc2, out=dh, act=6, aux=hpre)),
        ("fc2.dgrad x aux (act 6) + fc_b colsum partials", M, f, d,
         lambda: ops.linear_dgrad(dy, w_fc2, out=dh, act=6, aux=hpre, colsum_out=b_acc)),
        ("fc2.dgrad x aux (act 6), then colsum kernel", M, f, d,
         lambda: (ops.linear_dgrad(dy, w_fc2, out=dh, act=6, aux=hpre), ops.colsum_accumulate(dh, b_acc))),
        ("fc2.fwd+bias+f32 resid add", M, d, f, lambda: ops.gemm(h, w_fc2, a_mn=False, b_mn=False, M=M, N=d, K=f,
                                                                  out=resid, accumulate=True, bias=b_d)),
        ("proj.fwd+bias+f32 resid add", M, d, d, lambda: ops.gemm(o, w_o, a_mn=False, b_mn=False, M=M, N=d, K=d,
                                                                   out=resid, accumulate=True, bias=b_d)),
        ("proj.fwd plain bf16", M, d, d, lambda: ops.linear(o, w_o)),
    ]
    for name, m, n, k, fn in cases:
        ms = time_it(fn)
        rows.append({"name": name, "M": m, "N": n, "K": k, "us": round(ms * 1e3, 1),
                     "tflops": round(2.0 * m * n * k / ms / 1e9, 1)})
        print(json.dumps(rows[-1]), flush=True)
    return rows


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "gemm"
    {"gemm": bench_gemm, "epi": bench_epilogues}[what]()
