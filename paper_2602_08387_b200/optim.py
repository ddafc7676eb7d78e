"""Sharded fused AdamW (K10) with device-side global-norm clipping.

The registered ``optimizer`` component. One ``b2s_adamw`` launch per FSDP
unit updates that rank's fp32 master shard, both moments, and writes the bf16
shard that the next step all-gathers. The clip factor is computed on the GPU
from the all-reduced squared gradient norm, so the step never syncs the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import ops


@dataclass
class AdamWConfig:
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    grad_clip: float = 1.0
    warmup_steps: int = 10

    def __post_init__(self):
        if not (0.0 <= self.beta1 < 1.0 and 0.0 <= self.beta2 < 1.0):
            raise ValueError("betas must be in [0, 1)")
        if self.lr <= 0 or self.eps <= 0:
            raise ValueError("lr and eps must be positive")

    def lr_at(self, step: int) -> float:
        """Linear warmup over `warmup_steps`, then constant (step is 1-based)."""
        if self.warmup_steps > 0 and step <= self.warmup_steps:
            return self.lr * step / self.warmup_steps
        return self.lr


class FusedAdamW:
    def __init__(self, cfg: AdamWConfig):
        self.cfg = cfg
        self.step_count = 0
        self._gn2 = None
        self._part = None

    def grad_norm_sq(self, params, group=None, world=1, loss=None):
        """Device scalar: global squared L2 norm of the (reduce-scattered) gradients.

        With ``loss`` (a device scalar, W > 1) the rank-mean loss rides in the
        same all-reduce (one 2-float collective per step instead of two)."""
        flats = params.flat
        dev = flats[0].g.device
        nparts = 4 * 148
        if self._part is None:
            self._part = torch.empty(nparts, device=dev)
            self._red = torch.zeros(2, device=dev)
            self._gn2 = self._red[0:1]
            # one launch over every unit's gradient shard (addresses are stable for the run)
            self._table = torch.tensor([[f.g.data_ptr() for f in flats], [f.g.numel() for f in flats]],
                                       dtype=torch.int64).to(dev)
        ops.sumsq_partial_multi(self._table, len(flats), self._part)
        ops.sum_(self._part, self._gn2)
        if world > 1:
            if loss is not None:
                self._red[1:2].copy_(loss)
                dist.all_reduce(self._red, op=dist.ReduceOp.SUM, group=group)
                loss.copy_(self._red[1:2])
                ops.scale_f32(loss, 1.0 / world)
            else:
                dist.all_reduce(self._gn2, op=dist.ReduceOp.SUM, group=group)
        return self._gn2

    def step(self, params, group=None, world=1, loss=None, engine=None):
        """AdamW over every FSDP unit; ``engine.after_update(i)`` lets the FSDP engine
        start unit i's next-step all-gather while later units are still updating."""
        self.step_count += 1
        c = self.cfg
        if c.grad_clip > 0 or loss is not None:
            gn2 = self.grad_norm_sq(params, group, world, loss)
        else:
            gn2 = None
        lr = c.lr_at(self.step_count)
        for i, f in enumerate(params.flat):
            ops.adamw(f.master, f.m, f.v, f.g, f.p16, self.step_count, lr, c.beta1, c.beta2, c.eps,
                      c.weight_decay, gn2=gn2 if c.grad_clip > 0 else None, max_norm=c.grad_clip,
                      wd_mask=f.wd_mask)
            if engine is not None:
                engine.after_update(i)
        return gn2
