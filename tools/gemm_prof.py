"""Where the GEMM's MMA issuer and first epilogue warp wait, per launch (build the variant with
tools/build_variant.sh gprof -DB2S_GEMM_PROF, run with B2S_LIB=<that lib>):

    B2S_LIB=.../var_gprof/libb2s.so python tools/gemm_prof.py M N K [M N K ...]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import _lib, ops  # noqa: E402

lib = _lib.load()
lib.b2s_gemm_prof_read.argtypes = [ctypes.c_void_p]
args = [int(x) for x in sys.argv[1:]]
for M, N, K in zip(args[0::3], args[1::3], args[2::3]):
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        ops.gemm(a, b, a_mn=False, b_mn=False, M=M, N=N, K=K, out=c)
    torch.cuda.synchronize()
    buf = np.zeros((148, 3, 5), dtype=np.uint64)
    assert lib.b2s_gemm_prof_read(buf.ctypes.data) == 0
    mma = buf[:, 0, :][buf[:, 0, 0] > 0].astype(np.float64)
    epi = buf[:, 1, :][buf[:, 1, 0] > 0].astype(np.float64)
    prd = buf[:, 2, :][buf[:, 2, 0] > 0].astype(np.float64)
    tot, ntile = mma[:, 0].mean(), max(1.0, prd[:, 3].mean())
    pct = lambda x, t: 100 * x.sum() / t.sum()  # noqa: E731
    print(f"M {M} N {N} K {K}: {ntile:.1f} tiles per CTA pair, {tot / ntile:7.0f} clk per tile; MMA issuer waits: "
          f"free accumulator {pct(mma[:, 1], mma[:, 0]):4.1f}%, loaded stage {pct(mma[:, 2], mma[:, 0]):4.1f}% "
          f"(first stage of a tile {pct(mma[:, 4], mma[:, 0]):4.1f}%, {mma[:, 4].sum() / len(mma) / ntile:6.0f} clk per tile); "
          f"epilogue warp waits for an accumulator {pct(epi[:, 1], epi[:, 0]):4.1f}%; producer waits: tile index "
          f"{pct(prd[:, 1], prd[:, 0]):4.1f}% (leader {pct(prd[0::2, 1], prd[0::2, 0]):4.1f}% of which ring-slot wait {pct(prd[0::2, 4], prd[0::2, 0]):4.1f}%, peer {pct(prd[1::2, 1], prd[1::2, 0]):4.1f}%), "
          f"free stage {pct(prd[:, 2], prd[:, 0]):4.1f}%")
