"""K1 microbenchmark at a large size (>= 64M tokens, the per-step sizes are launch-bound).

    python tools/bench_gather.py [width] [L] [B]
The packed payload (2^27 tokens, resident in HBM) is gathered into int64 inputs / targets for B
samples of L tokens (default 16384 x 4096 = 64M tokens). Algorithmic bytes per launch:
B*(L+1)*w read + 2*B*L*8 written (packed_data.py:196-203 semantics, inputs = ids[:L], targets = ids[1:]).
Checked bit-exact against the oracle on a sample of rows. Prints one JSON line.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_08387_b200 import _lib  # noqa: E402
from paper_2602_08387_b200.packed import DevicePackedStream, PackedWriter, open_packed  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 4
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
B = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
n_tok = 1 << 27
path = os.path.join(ROOT, ".bench_data", f"gather_w{w}.cfpk")
if not os.path.exists(path):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    rng = np.random.default_rng(0)
    hi = {1: 256, 2: 65536, 4: 128256}[w]
    with PackedWriter(path, w) as wr:
        wr.write_stream(rng.integers(0, hi, size=n_tok), 1024)
r = open_packed(path)
ds = DevicePackedStream(r, torch.device("cuda"))
n = r.sample_count(L)
ids = torch.from_numpy(np.random.default_rng(1).integers(0, n, B).astype(np.int64)).cuda()
inp = torch.empty(B, L, dtype=torch.int64, device="cuda")
tgt = torch.empty_like(inp)
st = _lib.stream_ptr()


def go():
    _lib.call("b2s_gather_samples", ds.payload.data_ptr(), ds.token_width, ds.token_count, ids.data_ptr(), B, L,
              inp.data_ptr(), tgt.data_ptr(), ds.status.data_ptr(), st)


for _ in range(5):
    go()
torch.cuda.synchronize()
# parity: 64 random rows vs the reference semantics on the host memory map
pay = np.asarray(r.payload)
hid = ids.cpu().numpy()
for b in np.random.default_rng(2).integers(0, B, 64):
    s = int(hid[b])
    win = pay[s * L: s * L + L + 1].astype(np.int64)
    assert np.array_equal(inp[b].cpu().numpy(), win[:L]) and np.array_equal(tgt[b].cpu().numpy(), win[1:])
evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
iters = 20
evs[0].record()
for _ in range(iters):
    go()
evs[1].record()
torch.cuda.synchronize()
us = evs[0].elapsed_time(evs[1]) * 1e3 / iters
alg = B * (L + 1) * w + 2 * B * L * 8
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
print(json.dumps({"kernel": "b2s gather_samples_kernel", "width": w, "L": L, "B": B, "tokens": B * L, "us": round(us, 1),
                  "algorithmic_bytes": alg, "gbs": round(alg / us / 1e3, 1), "peak_gbs": peak,
                  "frac": round(alg / us / 1e3 / peak, 3), "parity": "64 rows bit-exact vs the host memory map"}))
