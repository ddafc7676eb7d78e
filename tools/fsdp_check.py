"""Multi-GPU FSDP check: W ranks x B/W sequences == 1 rank x B sequences.

    torchrun --nproc-per-node W tools/fsdp_check.py [preset] [global_batch] [steps] [out.json]

Every rank trains `steps` steps on its shard of the global batch; rank 0 then
replays the same steps on one GPU with the whole batch (a second trainer in
the same process, world=1 semantics) and writes both loss curves to out.json.
"""
import faulthandler
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_08387_b200.data import PackedDataLoader, Sampler, make_synthetic_packed  # noqa: E402
from paper_2602_08387_b200.fsdp import Engine, FlatParams  # noqa: E402
from paper_2602_08387_b200.model import PRESETS, DecoderLM, param_initializer  # noqa: E402
from paper_2602_08387_b200.optim import AdamWConfig, FusedAdamW  # noqa: E402
from paper_2602_08387_b200.packed import open_packed  # noqa: E402
from paper_2602_08387_b200.trainer import SPMDTrainer  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "tiny-llama"
GB = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", "fsdp_check.json")
bpu = int(os.environ.get("BLOCKS_PER_UNIT", "1"))
if os.environ.get("B2S_HANG_DUMP"):  # diagnostics: dump every thread's stack if the run stalls
    faulthandler.dump_traceback_later(int(os.environ["B2S_HANG_DUMP"]), exit=True)
cfg = PRESETS[preset]
T = min(256, cfg.max_seq_len)
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
path = os.path.join("/tmp", f"fsdp_check_{preset}.cfpk")
if rank == 0 and not os.path.exists(path):
    make_synthetic_packed(path + ".tmp", 1 << 19, cfg.vocab_size, kind="markov", seed=3)
    os.replace(path + ".tmp", path)
opt = AdamWConfig(lr=1e-3, warmup_steps=3)
tr = SPMDTrainer(DecoderLM(cfg), opt, None, steps=steps, seed=0, blocks_per_unit=bpu)
from paper_2602_08387_b200.trainer import init_distributed  # noqa: E402

init_distributed()
dist.barrier()
tr.dataloader = PackedDataLoader(open_packed(path), GB // world, T, Sampler(True, 7))
multi = tr.run()
# the sharded master weights after training, gathered
master = tr.params.master_full_fp32()
if rank == 0:
    single_tr = SPMDTrainer(DecoderLM(cfg), opt, PackedDataLoader(open_packed(path), GB, T, Sampler(True, 7)),
                            steps=steps, seed=0)
    # a world=1 trainer inside a W-rank job: build its pieces by hand
    single_tr.rank, single_tr.world, single_tr.device = 0, 1, torch.device("cuda", 0)
    single_tr.group = None
    single_tr.params = FlatParams(single_tr.model.units, 0, 1, single_tr.device)
    single_tr.params.load(param_initializer(cfg, 0, "cpu"))
    single_tr.model.attach(single_tr.params)
    single_tr.engine = Engine(single_tr.params, None, 1)
    single_tr.optimizer = FusedAdamW(opt)
    single_tr.dataloader.bind(0, 1, single_tr.device)
    single_tr._loss = torch.zeros(1, device=single_tr.device)
    single_tr._ready = True
    single = [float(single_tr.train_step(g).item()) for g in range(steps)]
    m1 = single_tr.params.master_full_fp32()
    rels = {k: float((master[k] - m1[k]).norm() / (m1[k].norm() + 1e-12)) for k in m1}
    worst = sorted(rels.items(), key=lambda kv: -kv[1])[:5]
    res = {"world": world, "preset": preset, "multi": multi, "single": single,
           "max_param_rel_diff": worst[0][1], "worst": worst, "blocks_per_unit": bpu}
    print(json.dumps(res))
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f)
tr.close()  # the W > 1 step graph holds NCCL work: release it before the teardown
dist.barrier()
dist.destroy_process_group()
