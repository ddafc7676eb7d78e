"""Causal attention forward / backward at the step shapes: TF/s (causal FLOPs) per kernel, with a
same-box yardstick: torch's F.scaled_dot_product_attention (bf16, is_causal) on each available
backend (flash / cuDNN / efficient) at the same shape, laid out as SDPA wants it ([B, H, T, dh]).
    python tools/bench_attn.py            (one JSON line per shape, direction and implementation)"""
import json
import os
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import ops  # noqa: E402
from tools.bench_kernels import time_it  # noqa: E402

SHAPES = (  # name, B, T, Hq, Hkv, dh
    ("gpt2-124m", 8, 2048, 12, 12, 64),
    ("llama-1b", 4, 4096, 32, 8, 64),
    ("llama-8b", 2, 4096, 32, 8, 128),
)
only = sys.argv[1:]  # optional: shape names
for name, B, T, Hq, Hkv, dh in SHAPES:
    if only and name not in only:
        continue
    qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device="cuda").bfloat16()
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    do = torch.randn_like(o)
    fl = 4.0 * B * Hq * dh * T * T / 2
    ms = time_it(lambda: ops.attn_fwd(qkv, B, T, Hq, Hkv, dh))
    print(json.dumps({"shape": name, "impl": "b2s", "dir": "fwd", "us": round(ms * 1e3, 1),
                      "TFs": round(fl / ms / 1e9, 1)}), flush=True)
    ms = time_it(lambda: ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh))
    print(json.dumps({"shape": name, "impl": "b2s", "dir": "bwd", "us": round(ms * 1e3, 1),
                      "TFs": round(2.5 * fl / ms / 1e9, 1)}), flush=True)
    # yardstick: SDPA with its own contiguous [B, H, T, dh] layout (no transposes timed)
    q = torch.randn(B, Hq, T, dh, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn(B, Hkv, T, dh, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    v = torch.randn(B, Hkv, T, dh, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    for be in (SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([be]):
                f = lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=Hq != Hkv)  # noqa
                out = f()
                g = torch.randn_like(out)
                ms_f = time_it(f)
                ms_fb = time_it(lambda: torch.autograd.grad(f(), (q, k, v), g))
            print(json.dumps({"shape": name, "impl": f"sdpa-{be.name.lower()}", "dir": "fwd",
                              "us": round(ms_f * 1e3, 1), "TFs": round(fl / ms_f / 1e9, 1)}), flush=True)
            ms_b = max(ms_fb - ms_f, 1e-6)
            print(json.dumps({"shape": name, "impl": f"sdpa-{be.name.lower()}", "dir": "bwd",
                              "us": round(ms_b * 1e3, 1), "TFs": round(2.5 * fl / ms_b / 1e9, 1),
                              "note": "fwd+bwd minus fwd"}), flush=True)
        except Exception as e:  # backend unavailable for this shape / GQA
            print(json.dumps({"shape": name, "impl": f"sdpa-{be.name.lower()}", "error": str(e)[:160]}), flush=True)
