"""Host-side FSDP / sampler logic across 2 ranks on CPU (gloo): sharding, all-gather,
reduce-scatter averaging, grouped units, and the W-rank sample partition."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, bpu, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_08387_b200.fsdp import Engine, FlatParams
        from paper_2602_08387_b200.model import PRESETS, init_params, unit_specs

        cfg = PRESETS["tiny-llama"]
        P = FlatParams(unit_specs(cfg), rank, world, torch.device("cpu"), blocks_per_unit=bpu)
        full = init_params(cfg, 0)
        P.load(full)
        res = {}
        # every rank holds exactly its 1/W slice of each flat unit
        for f in P.flat:
            ref = torch.zeros(f.padded)
            for (u, p), (o, shape, _) in f.offsets.items():
                ref[o:o + full[f"{u}.{p}"].numel()] = full[f"{u}.{p}"].reshape(-1)
            assert torch.equal(f.master, ref[rank * f.shard:(rank + 1) * f.shard])
        # all-gather: rank-tagged shards reassemble in rank order
        eng = Engine(P, dist.group.WORLD, world)
        for f in P.flat:
            f.p16.fill_(rank + 1)
        eng.begin_step()
        for i in range(len(P.model_units)):
            eng.before_forward(i)
        for f in P.flat:
            exp = torch.cat([torch.full((f.shard,), r + 1.0) for r in range(world)]).bfloat16()
            assert torch.equal(f.full, exp)
            assert torch.count_nonzero(f.gfull) == 0  # begin_step zeroed the grads
        # reduce-scatter: averaged gradient shards
        for f in P.flat:
            f.gfull.copy_(torch.arange(f.padded, dtype=torch.float32) * (rank + 1))
        for i in reversed(range(len(P.model_units))):
            eng.after_backward(i)
        eng.end_backward()
        for f in P.flat:
            avg = torch.arange(f.padded, dtype=torch.float32) * (sum(r + 1 for r in range(world)) / world)
            assert torch.allclose(f.g, avg[rank * f.shard:(rank + 1) * f.shard])
        res["units"] = len(P.flat)
        # gathered master == initial weights
        m = P.master_full_fp32(dist.group.WORLD)
        res["master_ok"] = all(torch.equal(m[k], v) for k, v in full.items())
        # sampler partition: W ranks x B == 1 rank x W*B
        from paper_2602_08387_b200.data import PackedDataLoader, Sampler
        from paper_2602_08387_b200.packed import open_packed

        r = open_packed(os.path.join(GOLDEN, "ref_w2.cfpk"))
        dl = PackedDataLoader(r, 2, 16, Sampler(True, 3)).bind(rank, world, "cpu")
        one = PackedDataLoader(r, 2 * world, 16, Sampler(True, 3)).bind(0, 1, "cpu")
        mine = [dl.sample_ids(s).tolist() for s in range(dl.steps_available)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        if rank == 0:
            for s in range(dl.steps_available):
                merged = sum((gathered[k][s] for k in range(world)), [])
                assert merged == one.sample_ids(s).tolist()
            res["steps"] = dl.steps_available
        q.put((rank, res))
    except Exception as e:  # surface assertion text to the parent
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bpu", [1, 2])
def test_fsdp_sharding_gloo_2ranks(bpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, bpu, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in out[r], out[r]
    assert out[0]["master_ok"] and out[1]["master_ok"]
    assert out[0]["units"] == (2 + (2 + bpu - 1) // bpu)
    assert out[0]["steps"] > 0


def test_grad_zero_ranges_complement():
    """The per-step gradient zeroing covers exactly what the model does not overwrite."""
    from paper_2602_08387_b200.fsdp import FlatParams
    from paper_2602_08387_b200.model import PRESETS, DecoderLM

    for name in ("tiny-llama", "tiny-gpt2"):
        model = DecoderLM(PRESETS[name], precision="fp32")
        P = FlatParams(model.units, 0, 1, "cpu", blocks_per_unit=2)
        over = model.overwritten_grads()
        ranges = P.grad_zero_ranges(over)
        zeroed = torch.zeros(P.gall.numel(), dtype=torch.bool)
        for o, n in ranges:
            assert n > 0 and not zeroed[o:o + n].any()
            zeroed[o:o + n] = True
        written = torch.zeros_like(zeroed)
        for f, base in zip(P.flat, P._gall_offs):
            for (_, p), (o, shape, _) in f.offsets.items():
                if p in over:
                    written[base + o:base + o + int(torch.Size(shape).numel())] = True
        assert written.any() and torch.equal(zeroed, ~written)
        assert P.grad_zero_ranges(None) == [(0, P.gall.numel())]

