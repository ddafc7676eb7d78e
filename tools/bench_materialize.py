"""Global document shuffle + materialize_chunk: the device segmented
copy (b2s_gather_documents, payload resident in HBM) vs the host path (the reference's
per-document loop, packed_data.py:336-344), on a 2^27-token w=4 corpus of ~1k-token documents.
    python tools/bench_materialize.py"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import _lib  # noqa: E402
from paper_2602_08387_b200 import packed as P  # noqa: E402
from tools.bench_kernels import peaks  # noqa: E402

path = os.path.join(ROOT, ".bench_data", "mat_corpus_w4.cfpk")
if not os.path.exists(path):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    rng = np.random.default_rng(0)
    n_tok = 1 << 27
    lens = rng.integers(1, 2048, size=n_tok // 1024)
    lens[-1] += n_tok - int(lens.sum()) if int(lens.sum()) < n_tok else 0
    with P.PackedWriter(path + ".tmp", 4) as w:
        toks = rng.integers(0, 128256, size=int(lens.sum()), dtype=np.uint32)
        off = 0
        for n in lens:
            w.write_document(toks[off:off + n])
            off += int(n)
    os.replace(path + ".tmp", path)
r = P.open_packed(path)
ds = P.DevicePackedStream(r)
perm = P.make_permutation(r.doc_count, 7).order
spans = np.asarray(r.spans, dtype=np.uint64)
lens = spans[perm, 1]
dst = np.zeros_like(lens)
np.cumsum(lens[:-1], out=dst[1:])
dev = ds.payload.device
t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
d_src, d_len, d_dst = t(spans[perm, 0]), t(lens), t(dst)
out = torch.empty(int(lens.sum()) * 4, dtype=torch.uint8, device=dev)
args = lambda: (ds.payload.data_ptr(), 4, d_src.data_ptr(), d_len.data_ptr(), d_dst.data_ptr(),  # noqa: E731
                int(perm.size), out.data_ptr(), _lib.stream_ptr())
for _ in range(3):
    _lib.call("b2s_gather_documents", *args())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(10):
    _lib.call("b2s_gather_documents", *args())
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
nbytes = 2 * int(lens.sum()) * 4
hbm, _ = peaks()
# host path (the reference algorithm) on a bounded sample of documents
sample = perm[:20000]
t0 = time.perf_counter()
P.materialize_chunk(r, sample, "/tmp/_mat_host.cfpk")
dt = time.perf_counter() - t0
host_tok_s = float(spans[sample, 1].sum()) / dt
print(json.dumps({"docs": int(perm.size), "tokens": int(lens.sum()), "gpu_ms": round(ms, 3),
                  "gpu_tokens_per_s": round(int(lens.sum()) / (ms / 1e3), 1),
                  "gpu_GBps": round(nbytes / (ms / 1e3) / 1e9, 1), "frac_of_hbm": round(nbytes / (ms / 1e3) / 1e9 / hbm, 3),
                  "host_tokens_per_s": round(host_tok_s, 1), "host_sample_docs": int(sample.size)}))
