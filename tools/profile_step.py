"""Run warmup + 1 training step of a preset (for ncu launch lists / captures).

    python tools/profile_step.py [preset] [batch] [seq] [warmup]
Prints the number of library launches per step so `ncu -s` can skip warm-up.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_08387_b200 import _lib  # noqa: E402
from paper_2602_08387_b200.data import PackedDataLoader, Sampler, synthetic_path  # noqa: E402
from paper_2602_08387_b200.model import PRESETS, DecoderLM  # noqa: E402
from paper_2602_08387_b200.optim import AdamWConfig  # noqa: E402
from paper_2602_08387_b200.packed import open_packed  # noqa: E402
from paper_2602_08387_b200.trainer import SPMDTrainer  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "gpt2-124m"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
W = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = PRESETS[preset]
path = synthetic_path(os.path.join(ROOT, ".bench_data"), max(1 << 22, (W + 2) * B * T + 1), cfg.vocab_size,
                      kind="uniform")
tr = SPMDTrainer(DecoderLM(cfg), AdamWConfig(), PackedDataLoader(open_packed(path), B, T, Sampler(True, 0)),
                 init_device="cuda")
tr.setup()
for s in range(W):
    tr.train_step(s)
torch.cuda.synchronize()
n0 = _lib.load().b2s_launch_count()
rng = os.environ.get("PROFILE_RANGE")  # ncu --profile-from-start off: capture exactly this step
if rng:
    torch.cuda.cudart().cudaProfilerStart()
tr.train_step(W)
torch.cuda.synchronize()
if rng:
    torch.cuda.cudart().cudaProfilerStop()
print(f"launches_per_step {_lib.load().b2s_launch_count() - n0} loss {tr._loss.item():.4f}")
if os.environ.get("KTIMER"):
    from paper_2602_08387_b200 import ops

    with ops.KernelTimer() as kt:
        tr.train_step(W + 1)
    for (kind, det), n, ms, tf in kt.detail():
        print(f"{kind:9s} {str(det):70s} n={n:3d} {ms:8.3f} ms {tf:7.1f} TF/s")
