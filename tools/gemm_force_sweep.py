"""Time a GEMM shape under each tile configuration (B2S_GEMM_FORCE) and raster choice.
    python tools/gemm_force_sweep.py M N K [a_mn b_mn]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402
from tools.bench_kernels import time_it  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
a_mn = len(sys.argv) > 4 and sys.argv[4] == "1"
b_mn = len(sys.argv) > 5 and sys.argv[5] == "1"
a = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
b = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for force in ["", "256,2,1", "256,1,1", "128,1,1", "256,2,2"]:
    for raster in ["", "mfast", "1", "-1", "4", "-4"]:
        os.environ["B2S_GEMM_FORCE"] = force
        os.environ["B2S_GEMM_RASTER"] = raster
        if not force and raster:
            continue
        ms = time_it(lambda: ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K, out=c))
        print(f"force={force or 'auto':8s} raster={raster or 'auto':6s} {ms * 1e3:8.1f} us {2 * M * N * K / ms / 1e9:7.1f} TF/s",
              flush=True)
