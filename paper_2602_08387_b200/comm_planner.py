"""Analytic FSDP collective planner (reference SPEC.md:495-602, module ``comm_planner``).

Sizes the per-unit all-gather / reduce-scatter messages of the training step
and picks the FSDP unit size (blocks per unit) that ``fsdp.FlatParams`` uses.
Formulas follow the SPEC exactly:

  block_param_count        h*nq*d + 2*h*nkv*d + nq*d*h + 3*h*f + 2*h      (:516-524)
  fsdp_shard_bytes         ceil(P / dp) * dtype_bytes                    (:526-534)
  ring_allgather_time      (p - 1) * (alpha + m / B)                      (:536-544)
  bus_bandwidth            (M / t) * (p - 1) / p,  M = p * m              (:546-554)
  plan_unit_size           argmin_g ceil(L/g) * (2*AG + RS), g*block_bytes <= cap,
                           ties -> smaller g                             (:556-564)
  message_size_table       CSV dp,blocks_per_unit,shard_bytes,busbw_bytes_per_sec,
                           latency_share,step_comm_seconds               (:566-574, :594)

``calibrate`` / ``calibrated_plan`` fit alpha and B from a measured NVLink 5
sweep (tools/collective_sweep.py, committed under profiles/) and plan with them.
``gpt2_block_param_count`` is the GPT-2 variant this build also trains
(2-matrix GELU MLP, biases, LayerNorm gains and biases) -- an extension, not in
the SPEC. ``fit_alpha_beta`` re-fits (alpha, B) from a measured NVLink sweep
(tools/collective_sweep.py), as the SPEC leaves alpha and B to calibration (:601).
"""

from __future__ import annotations

import math
from dataclasses import dataclass


class InvalidRanks(ValueError):
    pass


class InfeasibleCap(ValueError):
    pass


@dataclass(frozen=True)
class ModelShape:
    hidden: int
    ffn_hidden: int
    query_heads: int
    kv_heads: int
    head_dim: int
    layers: int
    dtype_bytes: int = 2

    def __post_init__(self):
        for k in ("hidden", "ffn_hidden", "query_heads", "kv_heads", "head_dim", "layers"):
            if getattr(self, k) <= 0:
                raise ValueError(f"{k} must be positive")
        if self.dtype_bytes not in (1, 2, 4):
            raise ValueError("dtype_bytes must be 1, 2 or 4")


@dataclass(frozen=True)
class CollectiveModel:
    alpha: float  # seconds per ring hop
    bandwidth: float  # bytes / second

    def __post_init__(self):
        if self.alpha < 0 or self.bandwidth <= 0:
            raise ValueError("alpha >= 0 and bandwidth > 0 required")


@dataclass(frozen=True)
class FsdpPlan:
    blocks_per_unit: int
    per_rank_shard_bytes: int
    busbw_bytes_per_sec: float
    step_comm_seconds: float
    peak_unsharded_unit_bytes: int


def block_param_count(s: ModelShape) -> int:
    h, f, nq, nkv, d = s.hidden, s.ffn_hidden, s.query_heads, s.kv_heads, s.head_dim
    return h * (nq * d) + 2 * h * (nkv * d) + (nq * d) * h + 3 * h * f + 2 * h


def gpt2_block_param_count(hidden: int, ffn_hidden: int) -> int:
    """GPT-2 block: fused qkv + proj (with biases), 2-matrix MLP (with biases), 2 LayerNorms (g, b)."""
    h, f = hidden, ffn_hidden
    return (3 * h * h + 3 * h) + (h * h + h) + (h * f + f) + (f * h + h) + 4 * h


def fsdp_shard_bytes(params: int, dtype_bytes: int, dp_degree: int) -> int:
    if params <= 0 or dtype_bytes <= 0 or dp_degree <= 0:
        raise ValueError("all arguments must be positive")
    return -(-params // dp_degree) * dtype_bytes


def ring_allgather_time(model: CollectiveModel, shard_bytes: float, ranks: int) -> float:
    if ranks < 2:
        raise InvalidRanks(f"ring collectives need p >= 2, got {ranks}")
    if shard_bytes < 0:
        raise ValueError("shard_bytes must be >= 0")
    return (ranks - 1) * (model.alpha + shard_bytes / model.bandwidth)


ring_reduce_scatter_time = ring_allgather_time  # symmetric ring schedule


def bus_bandwidth(total_bytes: float, t: float, ranks: int) -> float:
    if t <= 0 or ranks < 2:
        raise ValueError("t > 0 and p >= 2 required")
    return (total_bytes / t) * (ranks - 1) / ranks


def _unit_cost(shape: ModelShape, g: int, dp: int, model: CollectiveModel):
    shard = fsdp_shard_bytes(g * block_param_count(shape), shape.dtype_bytes, dp)
    t_ag = ring_allgather_time(model, shard, dp)
    t_rs = ring_reduce_scatter_time(model, shard, dp)
    units = -(-shape.layers // g)
    return shard, t_ag, units * (2 * t_ag + t_rs)


def plan_unit_size(shape: ModelShape, layers: int, dp: int, model: CollectiveModel,
                   memory_cap_bytes: int) -> FsdpPlan:
    if layers != shape.layers:
        shape = ModelShape(shape.hidden, shape.ffn_hidden, shape.query_heads, shape.kv_heads, shape.head_dim,
                           layers, shape.dtype_bytes)
    block_bytes = block_param_count(shape) * shape.dtype_bytes
    if memory_cap_bytes < block_bytes:
        raise InfeasibleCap(f"memory cap {memory_cap_bytes} B is below one block ({block_bytes} B)")
    best = None
    for g in range(1, layers + 1):
        if g * block_bytes > memory_cap_bytes:
            break
        shard, t_ag, step = _unit_cost(shape, g, dp, model)
        # strictly better beyond float rounding; ties (within 1e-12 relative) keep the smaller g
        if best is None or step < best[2] * (1.0 - 1e-12):
            best = (g, shard, step, t_ag)
    g, shard, step, t_ag = best
    busbw = bus_bandwidth(dp * shard, t_ag, dp)
    return FsdpPlan(g, shard, busbw, step, g * block_bytes)


def message_size_table(shape: ModelShape, dp_list, g_list, model: CollectiveModel | None = None) -> str:
    """CSV with the SPEC's columns (:594); one row per (dp, g)."""
    model = model or CollectiveModel(alpha=1e-5, bandwidth=1e10)
    rows = ["dp,blocks_per_unit,shard_bytes,busbw_bytes_per_sec,latency_share,step_comm_seconds"]
    for dp in dp_list:
        for g in g_list:
            shard, t_ag, step = _unit_cost(shape, g, dp, model)
            busbw = bus_bandwidth(dp * shard, t_ag, dp)
            lat = (dp - 1) * model.alpha / t_ag if t_ag > 0 else 0.0
            rows.append(f"{dp},{g},{shard},{busbw:.6g},{lat:.6g},{step:.6g}")
    return "\n".join(rows) + "\n"


def fit_alpha_beta(points) -> CollectiveModel:
    """Least-squares fit of t = (p-1)(alpha + m/B) to measured (p, m_bytes, t_seconds) points."""
    xs, ys = [], []
    for p, m, t in points:
        xs.append(m)
        ys.append(t / (p - 1))
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    slope = sxy / sxx if sxx > 0 else 0.0
    alpha = max(0.0, my - slope * mx)
    return CollectiveModel(alpha=alpha, bandwidth=1.0 / slope if slope > 0 else math.inf)


def load_sweep(path) -> list:
    """Rows of a tools/collective_sweep.py JSONL file (op, dtype, ranks, bytes, seconds, ...)."""
    import json

    with open(path) as f:
        return [json.loads(line) for line in f if line.strip()]


def calibrate(rows, op: str = "all_gather", dtype: str | None = None, min_bytes: int = 0) -> CollectiveModel:
    """Fit the SPEC ring model t = (p-1)(alpha + m/B) to a measured NVLink
    sweep. ``bytes`` in a sweep row is the full buffer M; the per-rank
    ring message is m = M / p."""
    pts = [(r["ranks"], r["bytes"] / r["ranks"], r["seconds"]) for r in rows
           if r.get("op") == op and (dtype is None or r["dtype"] == dtype) and r["bytes"] >= min_bytes
           and r["ranks"] >= 2]
    if len(pts) < 2:
        raise ValueError(f"need >= 2 sweep points for {op}/{dtype}, got {len(pts)}")
    return fit_alpha_beta(pts)


def calibrated_plan(shape: ModelShape, dp: int, rows, memory_cap_bytes: int = 1 << 30) -> FsdpPlan:
    """plan_unit_size with (alpha, B) fitted to the all-gather points of a measured sweep."""
    return plan_unit_size(shape, shape.layers, dp, calibrate(rows, "all_gather", "bfloat16"), memory_cap_bytes)


def shape_of(cfg) -> ModelShape:
    """ModelShape of a model.ModelConfig (Llama-style counting; GPT-2 via gpt2_block_param_count)."""
    return ModelShape(cfg.d_model, cfg.d_ff, cfg.n_head, cfg.n_kv_head, cfg.head_dim, cfg.n_layer, 2)
