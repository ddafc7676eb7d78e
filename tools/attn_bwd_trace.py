"""Timeline of the attention backward's roles (build with tools/build_variant.sh trace
-DB2S_ATTN_TRACE, run with B2S_LIB=<that lib>). Blocks 0..3 are the heaviest key tiles.

    B2S_LIB=.../var_trace/libb2s.so python tools/attn_bwd_trace.py B T Hq Hkv   -> summary on stdout
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
dh = int(os.environ.get("DH", "64"))  # 128: traces the dQ kernel (attn_bwd_q_kernel), or with
# B2S_TRACE_KV=1 the dK / dV kernel (attn_bwd128_kernel; build the trace variant with -DB2S_TRACE_KV)
qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device="cuda").bfloat16()
o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
do = torch.randn_like(o)
for _ in range(3):
    ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh)
torch.cuda.synchronize()
CTAS, WARPS, RECS = 4, 18, 8192
buf = np.zeros((CTAS, WARPS, RECS, 2), dtype=np.uint64)
lib = _lib.load()
lib.b2s_attn_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.b2s_attn_trace_read(buf.ctypes.data, buf.nbytes) == 0
NAMES = {50: "S_issued", 51: "pds_full_seen", 52: "dQ_issued" if dh == 128 else "dVdKdQ_issued", 60: "st_full_seen", 61: "ld0_done",
         62: "pds0_done", 63: "pds_empty_seen", 64: "ld1_done", 65: "pds1_done", 66: "pds_arrived",
         67: "dq_full_seen", 68: "drain_done", 70: "Q_load_issued", 71: "qd_full_seen", 72: "st_empty_seen"}
t0 = 0
for w in (0, 1, 2, 6):
    recs = buf[0, w]
    n = int((recs[:, 0] > 0).sum())
    print(f"--- cta 0 warp {w}: {n} records")
    rows = [(int(recs[k, 0]) - t0, int(recs[k, 1]) >> 32, int(recs[k, 1]) & 0xffffffff) for k in range(n)]
    for c, ev, aux in rows:
        if ev not in NAMES:
            continue
        if 40 <= aux <= 43:
            print(f"{c:9d} {NAMES.get(ev, ev):16s} {aux}")
# per-step period and per-phase averages (compute warps, steps 8..nsteps-8)
ph = {}
for cta in range(CTAS):
    for w in range(2, 10):
        recs = buf[cta, w]
        n = int((recs[:, 0] > 0).sum())
        rows = [(int(recs[k, 0]), int(recs[k, 1]) >> 32, int(recs[k, 1]) & 0xffffffff) for k in range(n)]
        rows = [r for r in rows if r[1] in NAMES]
        nst = max(r[2] for r in rows) + 1 if rows else 0
        prev = None
        for c, ev, aux in rows:
            if prev is not None and 8 <= aux < nst - 8:
                ph.setdefault(f"{NAMES[prev[1]]}->{NAMES[ev]}", []).append(c - prev[0])
            prev = (c, ev)
        st = [c for c, ev, aux in rows if ev == 60]
        if len(st) > 20:
            ph.setdefault("PERIOD st_full->st_full", []).extend(np.diff(st[8:-8]).tolist())
for k, v in sorted(ph.items(), key=lambda kv: -np.sum(kv[1])):
    print(f"{k:36s} n={len(v):6d} mean={np.mean(v):8.1f} clk  p50={np.median(v):8.1f}")
# MMA warp phases
mm = {}
for cta in range(CTAS):
    recs = buf[cta, 1]
    n = int((recs[:, 0] > 0).sum())
    rows = [(int(recs[k, 0]), int(recs[k, 1]) >> 32) for k in range(n)]
    rows = [r for r in rows if r[1] in NAMES]
    for (c0, e0), (c1, e1) in zip(rows[16:-16], rows[17:-15]):
        mm.setdefault(f"{NAMES[e0]}->{NAMES[e1]}", []).append(c1 - c0)
for k, v in sorted(mm.items(), key=lambda kv: -np.sum(kv[1])):
    print(f"MMA {k:32s} n={len(v):6d} mean={np.mean(v):8.1f} clk  p50={np.median(v):8.1f}")
