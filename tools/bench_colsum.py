import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2602_08387_b200 import ops
from tools.bench_kernels import time_it
dq = torch.randn(16384, 2304, device="cuda").bfloat16(); ob = torch.zeros(3072, device="cuda")
ms = time_it(lambda: ops.colsum_accumulate(dq, ob[:2304]), iters=50)
print(json.dumps({"bps": os.environ.get("B2S_COLSUM_BPS", "4"), "us": round(ms * 1e3, 2), "GBps": round(16384 * 2304 * 2 / ms / 1e6, 1)}))
