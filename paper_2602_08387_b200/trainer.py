"""The SPMD training driver (the paper's "gym") as a registered component.

One process per GPU (torchrun style: RANK / LOCAL_RANK / WORLD_SIZE /
MASTER_ADDR from the environment), NCCL over NVLink for the FSDP
collectives. A step is:

  dataloader.batch(step)            H2D of the step's sample ids/windows + K1 gather
  engine.begin_step()               zero grads, queue all-gathers on the comm stream
  model.forward_backward(...)       tcgen05 GEMMs / attention + bandwidth kernels;
                                    reduce-scatters queued per unit during backward
  engine.end_backward()             compute waits for the reduce-scatters
  optimizer.step(...)               one all-reduce of (grad-norm^2, loss), fused sharded AdamW;
                                    each unit's next-step all-gather queued after its update

"""

from __future__ import annotations

import atexit
import json
import os
import time
import weakref

import torch
import torch.distributed as dist

from . import ops
from .data import PackedDataLoader
from .fsdp import Engine, FlatParams
from .model import DecoderLM, param_initializer
from .optim import AdamWConfig, FusedAdamW

# dense bf16 peak the per-step MFU is quoted against: the burst figure measured on this pool's
# B200s (MEASURED_PEAKS.json, which bench.py reads; 2.25 PF/s is the nominal datasheet number)
BF16_PEAK_FLOPS = 1639.2e12


def init_distributed():
    """(rank, world, local_rank, device), initialising NCCL when launched with WORLD_SIZE > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise RuntimeError("the training step runs on B200 GPUs only (no CPU fallback)")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=device)
    return rank, world, local, device


# trainers that may hold a captured step graph with NCCL work in it (W > 1)
_LIVE = weakref.WeakSet()


def release_graphs() -> None:
    """Release every live trainer's captured step graph (see SPMDTrainer.close)."""
    for tr in list(_LIVE):
        tr.close()


def destroy_process_group() -> None:
    """Tear down NCCL safely: captured graphs holding NCCL work are released first, otherwise
    torch's destroy_process_group() waits on the communicator they keep alive."""
    release_graphs()
    if dist.is_initialized():
        dist.destroy_process_group()


# interpreter exit: release graphs before torch's own process-group teardown
atexit.register(release_graphs)

# W > 1 forward + backward captured with its reduce-scatters (B2S_GRAPH_MULTI=0: eager):
# 2-3% faster at W=2; see SPMDTrainer.close() for process-group teardown.
_GRAPH_MULTI = os.environ.get("B2S_GRAPH_MULTI", "1") == "1"


class _NativeGraph:
    """An instantiated CUDA graph captured through the library's C-ABI (b2s_graph_*): replayed
    with a bare cudaGraphLaunch, so a W = 1 step launches only b2s kernels and memsets."""

    def __init__(self, exec_handle: int):
        self.exec = exec_handle

    def replay(self) -> None:
        from . import _lib

        _lib.call("b2s_graph_launch", self.exec, _lib.stream_ptr())

    def __del__(self):
        try:
            from . import _lib

            if self.exec:
                _lib.load().b2s_graph_destroy(self.exec)
                self.exec = None
        except Exception:
            pass


class SPMDTrainer:
    def __init__(self, model: DecoderLM, optimizer, dataloader: PackedDataLoader, steps: int = 20,
                 seed: int = 0, blocks_per_unit: int = 1, init_device: str = "cpu", log_every: int = 0,
                 cuda_graph: bool = True, metrics_path: str | None = None):
        self.model = model
        self.opt_cfg = optimizer if isinstance(optimizer, AdamWConfig) else optimizer.cfg
        self.dataloader = dataloader
        self.steps = steps
        self.seed = seed
        self.blocks_per_unit = blocks_per_unit
        self.init_device = init_device
        self.log_every = log_every
        # rank 0 appends one JSON line per step of run(): loss, step ms, tokens/s/GPU, MFU, lr,
        # and at W > 1 the FSDP bytes all-gathered / reduce-scattered per step
        self.metrics_path = metrics_path
        # single GPU: after two eager steps the forward+backward (~350 launches) is
        # captured once as a CUDA graph and replayed (optimizer stays eager: its
        # learning rate / bias corrections are per-step host scalars)
        self.cuda_graph = cuda_graph
        self._graph = None
        self._eager_steps = 0
        self._ready = False

    def setup(self) -> "SPMDTrainer":
        if self._ready:
            return self
        self.rank, self.world, self.local_rank, self.device = init_distributed()
        self.group = dist.group.WORLD if self.world > 1 else None
        cfg = self.model.cfg
        self.params = FlatParams(self.model.units, self.rank, self.world, self.device, self.blocks_per_unit,
                                 dtype=self.model.dtype)
        init_dev = "cpu" if self.init_device == "cpu" else self.device
        self.params.load(param_initializer(cfg, self.seed, init_dev))
        self.model.attach(self.params)
        self.engine = Engine(self.params, self.group, self.world, overwritten=self.model.overwritten_grads())
        self.optimizer = FusedAdamW(self.opt_cfg)
        self.dataloader.bind(self.rank, self.world, self.device, vocab_size=cfg.vocab_size)
        if self.dataloader.seq_len > cfg.max_seq_len:
            raise ValueError(f"seq_len {self.dataloader.seq_len} exceeds the model's {cfg.max_seq_len}")
        self._loss = torch.zeros(1, device=self.device)
        if self.world > 1:
            _LIVE.add(self)
        self._ready = True
        return self

    def train_step(self, step: int, compute_only: bool = False):
        """One optimizer step on global batch `step`; returns the device loss (mean over all ranks)."""
        inputs, targets = self.dataloader.batch(step)
        return self.step_on(inputs, targets)

    def _graph_forward_backward(self, inputs, targets):
        from . import _lib

        multi = self.world > 1
        if multi:
            # W > 1: this step's all-gathers were queued after the previous optimizer
            # update (outside the graph); the replay starts once they landed, and the
            # graph itself holds the forward, backward and per-unit reduce-scatters
            self.engine.graph_step_prologue()
        if self._graph is None:
            self._gx, self._gy = inputs.clone(), targets.clone()
            n0 = _lib.load().b2s_launch_count()
            g = torch.cuda.CUDAGraph()
            if multi:
                with torch.cuda.graph(g):
                    self.engine.in_graph = True
                    for o, n in self.engine.zero_ranges:  # the ranges begin_step zeroes
                        ops.zero_(self.engine.P.gall[o:o + n])
                    self._gloss = self.model.forward_backward(self._gx, self._gy, hooks=self.engine)
                    self.engine.end_backward()  # joins the comm stream back into the capture
                    self.engine.in_graph = False
            else:
                # W = 1: native capture on a side stream (a capture cannot use the legacy default
                # stream). One eager pass on that stream first fills the per-stream scratch
                # caches, so nothing is allocated while capturing; the replay's zeroing of the
                # gradients makes the pass harmless.
                import ctypes

                cur = torch.cuda.current_stream()
                cs = self._cap_stream = getattr(self, "_cap_stream", None) or torch.cuda.Stream()
                cs.wait_stream(cur)
                handle = (ctypes.c_void_p * 1)()
                with torch.cuda.stream(cs):
                    self.engine.begin_step()
                    self.model.forward_backward(self._gx, self._gy, hooks=self.engine)
                    n0 = _lib.load().b2s_launch_count()
                    _lib.call("b2s_graph_capture_begin", cs.cuda_stream)
                    try:
                        self.engine.begin_step()
                        self._gloss = self.model.forward_backward(self._gx, self._gy, hooks=self.engine)
                    finally:
                        _lib.call("b2s_graph_capture_end", cs.cuda_stream, ctypes.addressof(handle))
                cur.wait_stream(cs)
                g = _NativeGraph(handle[0])
            self._graph_launches = int(_lib.load().b2s_launch_count() - n0)
            _lib.count_replayed_launches(-self._graph_launches)  # capture launched nothing
            self._graph = g
        self._gx.copy_(inputs)
        self._gy.copy_(targets)
        self._graph.replay()
        _lib.count_replayed_launches(self._graph_launches)
        return self._gloss

    def step_on(self, inputs, targets):
        from . import ops

        shape = tuple(inputs.shape)
        if self._graph is not None and shape != self._gshape:
            self._graph, self._eager_steps = None, 0  # new activation buffers: re-warm, re-capture
        graph_ok = self.world == 1 or (_GRAPH_MULTI and self.engine.timing is None
                                       and self.engine._prefetched == len(self.params.flat))
        use_graph = (self.cuda_graph and graph_ok and ops.KernelTimer.active is None and self._eager_steps >= 2)
        if use_graph:
            self._gshape = shape
            loss = self._graph_forward_backward(inputs, targets)
        else:
            self._eager_steps += 1
            self.engine.begin_step()
            loss = self.model.forward_backward(inputs, targets, hooks=self.engine)
            self.engine.end_backward()
        self._loss.copy_(loss)
        # the rank-mean loss shares the grad-norm all-reduce; the optimizer then
        # queues each unit's next-step all-gather as soon as that unit is updated
        self.optimizer.step(self.params, self.group, self.world, loss=self._loss if self.world > 1 else None,
                            engine=self.engine)
        return self._loss

    def close(self) -> None:
        """Release the captured step graph. At W > 1 it holds NCCL work, and
        destroy_process_group() waits for that communicator while the graph is alive:
        call this (or drop the trainer) before tearing the process group down."""
        if self._graph is not None:
            torch.cuda.synchronize()
            self._graph = None

    def run(self) -> list:
        """Train `steps` steps; returns the per-step mean losses (host floats)."""
        self.setup()
        losses = []
        t0 = time.perf_counter()
        mf = open(self.metrics_path, "a") if (self.metrics_path and self.rank == 0) else None
        cfg, B, T = self.model.cfg, self.dataloader.batch_size, self.dataloader.seq_len
        try:
            for g in range(self.steps):
                ts = time.perf_counter()
                loss = self.train_step(g)
                losses.append(float(loss.item()))  # synchronises: the step's wall time is complete
                dt = time.perf_counter() - ts
                if mf is not None:
                    tps = B * T / dt
                    rec = {"step": g, "loss": losses[-1], "step_ms": round(dt * 1e3, 3),
                           "tokens_per_s_per_gpu": round(tps, 1),
                           # 4 significant digits (a tiny model's first, eager / capturing steps
                           # are below 1e-4 MFU and would round to 0)
                           "mfu": float(f"{tps * cfg.flops_per_token(T) / BF16_PEAK_FLOPS:.4g}"),
                           "lr": self.opt_cfg.lr_at(g + 1), "world": self.world}
                    if self.world > 1:
                        rec.update(ag_bytes=self.engine.bytes_ag, rs_bytes=self.engine.bytes_rs)
                    mf.write(json.dumps(rec) + "\n")
                    mf.flush()
                if self.log_every and self.rank == 0 and (g % self.log_every == 0 or g == self.steps - 1):
                    print(f"step {g:5d}  loss {losses[-1]:.4f}  {time.perf_counter() - t0:.1f}s", flush=True)
        finally:
            if mf is not None:
                mf.close()
        self.close()  # a later run() re-captures; the process group can be torn down now
        return losses
