"""How much launch overhead does the eager step carry? Times forward+backward eagerly and as
one captured CUDA graph (same buffers, W=1).   python tools/graph_probe.py [preset] [B] [T]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200.data import PackedDataLoader, Sampler, synthetic_path  # noqa: E402
from paper_2602_08387_b200.model import PRESETS, DecoderLM  # noqa: E402
from paper_2602_08387_b200.optim import AdamWConfig  # noqa: E402
from paper_2602_08387_b200.packed import open_packed  # noqa: E402
from paper_2602_08387_b200.trainer import SPMDTrainer  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "gpt2-124m"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
cfg = PRESETS[preset]
path = synthetic_path(os.path.join(ROOT, ".bench_data"), max(1 << 22, 8 * B * T + 1), cfg.vocab_size, kind="uniform")
tr = SPMDTrainer(DecoderLM(cfg), AdamWConfig(), PackedDataLoader(open_packed(path), B, T, Sampler(True, 0)),
                 init_device="cuda").setup()
x, y = tr.dataloader.batch(0)
x, y = x.clone(), y.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        tr.model.forward_backward(x, y)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    tr.model.forward_backward(x, y)
torch.cuda.synchronize()


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


eager = timeit(lambda: tr.model.forward_backward(x, y))
graph = timeit(g.replay)
print(f"{preset} fwd+bwd eager {eager:.3f} ms  graph {graph:.3f} ms  launch overhead {100 * (eager - graph) / eager:.1f}%")
