"""Weight-gradient GEMMs (overwrite mode, the step's) under forced split-K counts: picks the
split the host should choose. python tools/gemm_split_sweep.py [M,N,K ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or [
    (2048, 2048, 16384), (3072, 2048, 16384), (2048, 8192, 16384), (16384, 2048, 16384), (128256, 2048, 16384),
    (768, 768, 16384), (2304, 768, 16384), (3072, 768, 16384), (768, 3072, 16384), (50304, 768, 16384)]


def t(f, reps=20):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for M, N, K in shapes:
    a = torch.randn(K, M, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda")
    row = {"M": M, "N": N, "K": K}
    for sp in ("", 1, 2, 3, 4, 6, 8, 12, 16):
        if sp == "":
            os.environ.pop("B2S_GEMM_FORCE", None)
        else:
            os.environ["B2S_GEMM_FORCE"] = f"256,2,{sp}"
        row[f"s{sp}" if sp != "" else "auto"] = round(t(lambda: ops.gemm(a, b, a_mn=True, b_mn=True, M=M, N=N, K=K,
                                                                        out=c, accumulate=ops.OVERWRITE)), 1)
    os.environ.pop("B2S_GEMM_FORCE", None)
    print(json.dumps(row))
