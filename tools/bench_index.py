"""Corpus index: GPU newline scan on a 1 GiB raw buffer resident in HBM
(kernel time, GB/s vs the HBM peak) and build_index end to end from the file, vs the host
restatement of the reference's scan loop on a bounded sample.   python tools/bench_index.py"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import _lib  # noqa: E402
from paper_2602_08387_b200 import corpus_index as CI  # noqa: E402
from tools.bench_kernels import peaks  # noqa: E402

n = 1 << 30
rng = np.random.default_rng(0)
data = rng.integers(32, 127, size=n, dtype=np.uint8)
data[rng.integers(0, n, size=n // 2048)] = 10
buf = torch.from_numpy(data).cuda()
nblocks = 148 * 8
chunk = ((-(-n // nblocks)) + 15) // 16 * 16
counts = torch.empty(nblocks, dtype=torch.int32, device="cuda")
st = _lib.stream_ptr()
_lib.call("b2s_newline_count", buf.data_ptr(), n, chunk, counts.data_ptr(), nblocks, st)
c = counts.cpu().numpy().astype(np.int64)
offs = torch.from_numpy(np.concatenate([[0], np.cumsum(c[:-1])])).cuda()
pos = torch.empty(int(c.sum()), dtype=torch.int64, device="cuda")


def scan():
    _lib.call("b2s_newline_count", buf.data_ptr(), n, chunk, counts.data_ptr(), nblocks, st)
    _lib.call("b2s_newline_positions", buf.data_ptr(), n, chunk, offs.data_ptr(), nblocks, 0, pos.data_ptr(), st)


for _ in range(3):
    scan()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(10):
    scan()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
hbm, _ = peaks()
gbs = 2 * n / (ms / 1e3) / 1e9  # the buffer is read twice (count pass, position pass)
path = os.path.join(ROOT, ".bench_data", "index_1g.jsonl")
os.makedirs(os.path.dirname(path), exist_ok=True)
data.tofile(path)
t0 = time.perf_counter()
ix = CI.build_index(path)
e2e = time.perf_counter() - t0
# host path: the reference algorithm (chunked find loop) on the first 64 MiB
sample = data[: 64 << 20].tobytes()
t0 = time.perf_counter()
cnt, start, i = 0, 0, sample.find(b"\n")
while i != -1:
    if i > start:
        cnt += 1
    start = i + 1
    i = sample.find(b"\n", start)
host = (time.perf_counter() - t0)
print(json.dumps({"bytes": n, "docs": ix.doc_count, "gpu_scan_ms": round(ms, 3), "gpu_scan_GBps": round(gbs, 1),
                  "frac_of_hbm": round(gbs / hbm, 3), "e2e_build_index_s": round(e2e, 3),
                  "e2e_GBps": round(n / e2e / 1e9, 2), "host_ref_loop_GBps": round(len(sample) / host / 1e9, 3),
                  "host_sample_bytes": len(sample)}))
os.remove(path)
