"""Fully-sharded data parallelism over flat per-unit buffers (FSDP2 semantics, B200 layout).

Each FSDP unit (embedding, each transformer block or group of g blocks,
final norm/head) owns one flat parameter space of `padded` elements, split
into W equal shards. Per rank and unit (sizes for the shard S = padded / W):

  master  fp32 [S]   optimizer's copy of the parameters       (sharded)
  m, v    fp32 [S]   AdamW moments                            (sharded)
  p16     bf16 [S]   AdamW's bf16 output = all-gather source   (sharded)
  g       fp32 [S]   reduce-scatter destination (averaged)    (sharded)
  full    bf16 [W*S] all-gather destination: the compute weights
  gfull   fp32 [W*S] the backward's weight-gradient accumulator

With 180 GB per GPU the unsharded buffers stay resident (no re-gather in the
backward): per step each unit does one NCCL all-gather (before its forward,
prefetched on a side stream) and one reduce-scatter (as soon as its backward
is done, on the same side stream), overlapping the compute of other units.
At W = 1 the shard IS the full buffer and no collective is issued.
In fp32 mode (compute dtype fp32) the compute weights are the master
parameters themselves: p16 aliases master (the all-gather source) and, at
W = 1, master aliases full -- AdamW updates the compute buffer in place.
`comm_planner.plan_unit_size` picks how many blocks form a unit.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops
from .model import ALIGN, UnitSpec


def _padded_numel(specs: list, world: int) -> int:
    per = -(-sum(s.numel for s in specs) // world)
    return (-(-per // ALIGN) * ALIGN) * world


class FlatUnit:
    def __init__(self, specs: list, rank: int, world: int, device, dtype=torch.bfloat16, gfull=None):
        self.specs = specs  # one or more model UnitSpecs grouped into this FSDP unit
        self.rank, self.world = rank, world
        self.offsets = {}
        off = 0
        for s in specs:
            for p in s.params:
                self.offsets[(s.name, p.name)] = (off + s.offsets[p.name], tuple(p.shape), p.decay)
            off += s.numel
        self.numel = off
        per = -(-off // world)
        self.shard = -(-per // ALIGN) * ALIGN
        self.padded = self.shard * world
        bf, f32 = dtype, torch.float32
        self.full = torch.zeros(self.padded, device=device, dtype=bf)
        # gfull: this unit's slice of one buffer holding every unit's gradients (one
        # memset per step instead of one per unit), or its own allocation
        self.gfull = gfull if gfull is not None else torch.zeros(self.padded, device=device, dtype=f32)
        assert self.gfull.numel() == self.padded
        lo = rank * self.shard
        if world == 1:
            self.g = self.gfull
        else:
            self.g = torch.zeros(self.shard, device=device, dtype=f32)
        if bf == f32:  # fp32 mode: compute copy == master (no separate low-precision shard)
            self.master = self.full if world == 1 else torch.zeros(self.shard, device=device, dtype=f32)
            self.p16 = self.master
        else:
            self.master = torch.zeros(self.shard, device=device, dtype=f32)
            self.p16 = self.full if world == 1 else torch.zeros(self.shard, device=device, dtype=bf)
        self.m = torch.zeros(self.shard, device=device, dtype=f32)
        self.v = torch.zeros(self.shard, device=device, dtype=f32)
        mask = torch.zeros(self.padded, dtype=torch.uint8)
        for (_, _), (o, shape, decay) in self.offsets.items():
            n = int(torch.Size(shape).numel())
            if decay:
                mask[o:o + n] = 1
        self.wd_mask = mask[lo:lo + self.shard].to(device)

    def load_full_fp32(self, get) -> None:
        """Fill this rank's master shard (and bf16 copies); get('unit.param') -> full fp32 tensor."""
        full = torch.zeros(self.padded, dtype=torch.float32, device=self.master.device)
        for (u, p), (o, shape, _) in self.offsets.items():
            t = get(f"{u}.{p}")
            full[o:o + t.numel()] = t.reshape(-1).to(full.device, torch.float32)
        lo = self.rank * self.shard
        self.master.copy_(full[lo:lo + self.shard])
        if self.p16 is not self.master:
            self.p16.copy_(self.master)
        if self.full is not self.master:
            self.full.copy_(full)  # initial gather done locally (every rank has the same init)

    def view(self, buf, unit: str, name: str):
        o, shape, _ = self.offsets[(unit, name)]
        return buf[o:o + int(torch.Size(shape).numel())].view(shape)


class UnitView:
    """The parameters / gradients of one *model* unit inside its FSDP unit."""

    def __init__(self, flat: FlatUnit, name: str):
        self.flat, self.name = flat, name

    def p(self, pname):
        return self.flat.view(self.flat.full, self.name, pname)

    def g(self, pname):
        return self.flat.view(self.flat.gfull, self.name, pname)


class FlatParams:
    """All FSDP units of a model; ``unit(i)`` addresses the i-th *model* unit."""

    def __init__(self, unit_specs: list, rank: int, world: int, device, blocks_per_unit: int = 1,
                 dtype=torch.bfloat16):
        self.model_units = unit_specs
        groups, cur = [], []
        # embedding and head are units of their own; blocks are grouped g at a time
        for s in unit_specs:
            if s.name.startswith("block"):
                cur.append(s)
                if len(cur) == blocks_per_unit:
                    groups.append(cur)
                    cur = []
            else:
                if cur:
                    groups.append(cur)
                    cur = []
                groups.append([s])
        if cur:
            groups.append(cur)
        sizes = [_padded_numel(g, world) for g in groups]
        self.gall = torch.zeros(sum(sizes), device=device, dtype=torch.float32)
        offs = [sum(sizes[:i]) for i in range(len(sizes))]
        self._gall_offs = offs
        self.flat = [FlatUnit(g, rank, world, device, dtype, gfull=self.gall[o:o + n])
                     for g, o, n in zip(groups, offs, sizes)]
        self.owner = {}
        self.first_model_unit = {}
        self.last_model_unit = {}
        mi = 0
        for fi, g in enumerate(groups):
            self.first_model_unit[fi] = mi
            for _ in g:
                self.owner[mi] = fi
                mi += 1
            self.last_model_unit[fi] = mi - 1
        self._views = [UnitView(self.flat[self.owner[i]], s.name) for i, s in enumerate(unit_specs)]

    def grad_zero_ranges(self, overwritten=None) -> list:
        """(start, length) element ranges of gall a step must zero before its backward: all of
        it except the gradients named in ``overwritten`` (written whole by their single writer)."""
        total = self.gall.numel()
        if not overwritten:
            return [(0, total)]
        keep = []
        for f, base in zip(self.flat, self._gall_offs):
            for (_, p), (o, shape, _) in f.offsets.items():
                if p in overwritten:
                    keep.append((base + o, base + o + int(torch.Size(shape).numel())))
        ranges, cur = [], 0
        for a, b in sorted(keep):
            if a > cur:
                ranges.append((cur, a - cur))
            cur = max(cur, b)
        if cur < total:
            ranges.append((cur, total - cur))
        return ranges

    def unit(self, i: int) -> UnitView:
        return self._views[i]

    def load(self, tensors) -> None:
        """tensors: dict 'unit.param' -> fp32 tensor, or a callable with the same contract."""
        get = tensors if callable(tensors) else tensors.__getitem__
        for f in self.flat:
            f.load_full_fp32(get)

    def gather_full_fp32(self) -> dict:
        """fp32 copies of the current parameters keyed 'unit.param' (from the bf16 compute copy)."""
        out = {}
        for f in self.flat:
            for (u, p), (o, shape, _) in f.offsets.items():
                out[f"{u}.{p}"] = f.full[o:o + int(torch.Size(shape).numel())].view(shape).float().cpu()
        return out

    def master_full_fp32(self, group=None) -> dict:
        """fp32 master parameters keyed 'unit.param' (all-gathered when sharded)."""
        out = {}
        for f in self.flat:
            if f.world > 1:
                full = torch.empty(f.padded, device=f.master.device)
                dist.all_gather_into_tensor(full, f.master, group=group)
            else:
                full = f.master
            for (u, p), (o, shape, _) in f.offsets.items():
                out[f"{u}.{p}"] = full[o:o + int(torch.Size(shape).numel())].view(shape).cpu().clone()
        return out

    def grads_full_fp32(self) -> dict:
        """Unsharded fp32 gradients of the last backward (before the reduce-scatter)."""
        out = {}
        for f in self.flat:
            for (u, p), (o, shape, _) in f.offsets.items():
                out[f"{u}.{p}"] = f.gfull[o:o + int(torch.Size(shape).numel())].view(shape).cpu().clone()
        return out


class Engine:
    """Issues the per-unit collectives on a side stream and fences them against compute.

    before_forward(i): compute waits for the all-gather of model unit i's FSDP unit.
    after_backward(i): when the last model unit of an FSDP unit finished its
    backward, its gradient reduce-scatter is queued on the comm stream.
    """

    def __init__(self, params: FlatParams, group=None, world: int = 1, prefetch: int = 2, overwritten=None):
        self.P = params
        # gradient ranges zeroed at the start of each step (the model overwrites the rest)
        self.zero_ranges = params.grad_zero_ranges(overwritten)
        self.group = group
        self.world = world
        self.prefetch = prefetch
        # CUDA: collectives on a side stream fenced by events. CPU (gloo, host-side
        # tests of the sharding logic): plain synchronous collectives.
        self.cuda = params.flat[0].full.is_cuda
        self.comm = torch.cuda.Stream() if (world > 1 and self.cuda) else None
        n = len(params.flat)
        self.ag_done = [torch.cuda.Event() for _ in range(n)] if self.cuda else [None] * n
        self.rs_done = [torch.cuda.Event() for _ in range(n)] if self.cuda else [None] * n
        self._issued = 0
        self._prefetched = 0  # units whose next-step all-gather was issued after their optimizer update
        self.in_graph = False  # capturing the W > 1 forward/backward: all-gathers were awaited before replay
        self.timing = None  # list of (kind, bytes, start_event, end_event) while collective timing is on
        self.bytes_ag = sum(f.padded * f.full.element_size() for f in params.flat)
        self.bytes_rs = sum(f.padded * 4 for f in params.flat)

    # ------------------------------------------------------------------ step
    def begin_step(self) -> None:
        if self.P.gall.is_cuda:
            for o, n in self.zero_ranges:
                ops.zero_(self.P.gall[o:o + n])
        else:  # the gloo host-logic tests (tests/test_fsdp_cpu.py) run the engine without a GPU
            self.P.gall.zero_()
        if self.world > 1 and self._prefetched == len(self.P.flat):
            # every unit's all-gather was queued right after its optimizer update
            self._issued = len(self.P.flat)
            self._prefetched = 0
            return
        self._issued = 0
        self._prefetched = 0
        if self.world > 1:
            if self.cuda:
                ready = torch.cuda.Event()
                ready.record()  # after the previous optimizer step wrote p16
                self.comm.wait_event(ready)
            self._issue_until(min(len(self.P.flat), self.prefetch))

    def graph_step_prologue(self) -> None:
        """Host side of begin_step for a graph replay (W > 1): every unit's all-gather was
        queued after its optimizer update; the compute stream waits for all of them here,
        outside the graph (events recorded outside a capture cannot be awaited inside it)."""
        cur = torch.cuda.current_stream()
        for e in self.ag_done:
            cur.wait_event(e)
        self._issued = len(self.P.flat)
        self._prefetched = 0

    def after_update(self, fi: int) -> None:
        """FSDP unit fi's shard was just updated by the optimizer (compute stream):
        queue its all-gather for the next step now, so it overlaps the remaining
        optimizer kernels and the next step's first forward kernels."""
        if self.world == 1 or not self.cuda or fi != self._prefetched:
            return
        f = self.P.flat[fi]
        ready = torch.cuda.Event()
        ready.record()
        self.comm.wait_event(ready)
        with torch.cuda.stream(self.comm):
            self._timed_collective("all_gather", f.full, lambda: dist.all_gather_into_tensor(
                f.full, f.p16, group=self.group))
            self.ag_done[fi].record(self.comm)
        self._prefetched += 1

    def _timed_collective(self, kind, full_tensor, fn):
        if self.timing is None:
            return fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(self.comm)
        fn()
        e.record(self.comm)
        self.timing.append((kind, full_tensor.numel() * full_tensor.element_size(), s, e))

    def collective_summary(self):
        """nccl-tests bus bandwidth of the timed collectives: busbw = (bytes / t) * (W - 1) / W,
        bytes = the full (gathered / pre-reduction) buffer."""
        torch.cuda.synchronize()
        out = {}
        for kind, nbytes, s, e in self.timing or []:
            d = out.setdefault(kind, {"calls": 0, "bytes": 0, "ms": 0.0})
            d["calls"] += 1
            d["bytes"] += nbytes
            d["ms"] += s.elapsed_time(e)
        for d in out.values():
            alg = d["bytes"] / (d["ms"] / 1e3) if d["ms"] > 0 else 0.0
            d["busbw_GBps"] = round(alg * (self.world - 1) / self.world / 1e9, 1)
            d["frac_of_900GBps"] = round(d["busbw_GBps"] / 900.0, 3)
            d["ms"] = round(d["ms"], 3)
        return out

    def _issue_until(self, k: int) -> None:
        while self._issued < k:
            f = self.P.flat[self._issued]
            if self.cuda:
                with torch.cuda.stream(self.comm):
                    self._timed_collective("all_gather", f.full, lambda: dist.all_gather_into_tensor(
                        f.full, f.p16, group=self.group))
                    self.ag_done[self._issued].record(self.comm)
            else:
                dist.all_gather_into_tensor(f.full, f.p16, group=self.group)
            self._issued += 1

    def before_forward(self, model_unit: int) -> None:
        if self.world == 1 or self.in_graph:
            return
        fi = self.P.owner[model_unit]
        if self.P.first_model_unit[fi] != model_unit:
            return
        self._issue_until(min(len(self.P.flat), fi + 1 + self.prefetch))
        if self.cuda:
            torch.cuda.current_stream().wait_event(self.ag_done[fi])

    def after_backward(self, model_unit: int) -> None:
        if self.world == 1:
            return
        fi = self.P.owner[model_unit]
        if self.P.first_model_unit[fi] != model_unit:
            return  # the unit's gradients are complete once its first model unit is done
        f = self.P.flat[fi]
        if not self.cuda:
            # gloo has no AVG reduce-scatter: SUM then scale (host-side tests only)
            dist.reduce_scatter_tensor(f.g, f.gfull, op=dist.ReduceOp.SUM, group=self.group)
            f.g.div_(self.world)
            return
        done = torch.cuda.Event()
        done.record()
        self.comm.wait_event(done)
        with torch.cuda.stream(self.comm):
            self._timed_collective("reduce_scatter", f.gfull, lambda: dist.reduce_scatter_tensor(
                f.g, f.gfull, op=dist.ReduceOp.AVG, group=self.group))
            self.rs_done[fi].record(self.comm)

    def end_backward(self) -> None:
        if self.world == 1 or not self.cuda:
            return
        cur = torch.cuda.current_stream()
        for e in self.rs_done:
            cur.wait_event(e)
