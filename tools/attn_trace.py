"""Timeline of the persistent attention forward's roles (build with tools/build_variant.sh trace
-DB2S_ATTN_TRACE, run with B2S_LIB=<that lib>).

    B2S_LIB=.../var_trace/libb2s.so python tools/attn_trace.py B T Hq Hkv [dh]   -> trace .npy + summary
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import _lib, ops  # noqa: E402

B, T, Hq, Hkv = (int(x) for x in sys.argv[1:5])
dh = int(sys.argv[5]) if len(sys.argv) > 5 else 64
qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device="cuda").bfloat16()
for _ in range(3):
    ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
torch.cuda.synchronize()
CTAS, WARPS, RECS = 4, 18, 8192
buf = np.zeros((CTAS, WARPS, RECS, 2), dtype=np.uint64)
lib = _lib.load()
lib.b2s_attn_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
# zero the device buffer by reading after one fresh launch: records of the last launch overwrite
ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
torch.cuda.synchronize()
assert lib.b2s_attn_trace_read(buf.ctypes.data, buf.nbytes) == 0
out = os.path.join(ROOT, "gpurun_out", f"attn_trace_{B}_{T}_{Hq}_{Hkv}_{dh}.npy")
os.makedirs(os.path.dirname(out), exist_ok=True)
np.save(out, buf)
NAMES = {1: "tma_kvwait_beg", 2: "tma_kvwait_end", 10: "S_beg", 12: "S_kfull", 14: "S_sempty", 20: "PV_beg",
         22: "PV_vfull", 24: "PV_pfull", 30: "s_wait_beg", 31: "s_wait_end", 32: "ld_done", 33: "max_done",
         34: "exp_done", 35: "pempty_done", 36: "pfull_arrived", 40: "epi_beg", 41: "epi_end"}
for cta in range(1):
    t0 = min(int(buf[cta, w, 0, 0]) for w in range(WARPS) if buf[cta, w, 0, 0])
    for w in (0, 1, 2, 6):
        recs = buf[cta, w]
        n = int((recs[:, 0] > 0).sum())
        print(f"--- cta {cta} warp {w}: {n} records")
        for k in range(min(n, 120)):
            c, e = int(recs[k, 0]) - t0, int(recs[k, 1])
            ev, aux = e >> 32, e & 0xffffffff
            print(f"{c:9d} {str(NAMES.get(ev, ev)):16s} {aux}")
# per-phase averages for softmax warps (all 4 CTAs, warps 2..9)
ph = {}
for cta in range(CTAS):
    for w in range(2, WARPS):
        recs = buf[cta, w]
        n = int((recs[:, 0] > 0).sum())
        prev = None
        for k in range(n):
            c, ev = int(recs[k, 0]), int(recs[k, 1]) >> 32
            if prev is not None and 30 <= ev <= 36 and 30 <= prev[1] <= 36:
                key = f"{NAMES[prev[1]]}->{NAMES[ev]}"
                ph.setdefault(key, []).append(c - prev[0])
            prev = (c, ev)
for k, v in sorted(ph.items(), key=lambda kv: -np.sum(kv[1])):
    print(f"{k:34s} n={len(v):6d} mean={np.mean(v):8.1f} clk  p50={np.median(v):8.1f}  sum={np.sum(v) / 1e6:8.2f} Mclk")
