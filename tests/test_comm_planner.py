"""comm_planner restated from SPEC.md:495-602: SPEC examples, acceptance criteria 1, 7, 8, properties."""

import math
import random

import pytest

from paper_2602_08387_b200 import comm_planner as cp

L3_8B = cp.ModelShape(4096, 14336, 32, 8, 128, 32, 2)


def test_block_param_count_examples():
    assert cp.block_param_count(cp.ModelShape(1, 1, 1, 1, 1, 1)) == 9
    assert cp.block_param_count(L3_8B) == 218_112_000
    s2 = cp.ModelShape(4096, 2 * 14336, 32, 8, 128, 32)
    assert cp.block_param_count(s2) - cp.block_param_count(L3_8B) == 3 * 4096 * 14336
    assert cp.gpt2_block_param_count(768, 3072) == 7_087_872


def test_shard_bytes_examples_and_acceptance_1():
    assert cp.fsdp_shard_bytes(1024, 2, 1024) == 2
    b = cp.fsdp_shard_bytes(cp.block_param_count(L3_8B), 2, 1024)
    assert b == 426_000 and 0.38e6 <= b <= 0.45e6
    assert cp.fsdp_shard_bytes(777, 2, 1) == 1554


def test_ring_time_examples():
    assert cp.ring_allgather_time(cp.CollectiveModel(0.0, 1.0), 1, 2) == 1.0
    m = cp.CollectiveModel(3e-5, 1e9)
    assert cp.ring_allgather_time(m, 0, 8) == pytest.approx(7 * 3e-5)
    t = cp.ring_allgather_time(cp.CollectiveModel(1e-5, 1e10), 426_000, 1024)
    assert t == pytest.approx(0.0538, abs=5e-5)
    with pytest.raises(cp.InvalidRanks):
        cp.ring_allgather_time(m, 10, 1)


def test_bus_bandwidth_examples_and_acceptance_8():
    B = 1e10
    m = cp.CollectiveModel(0.0, B)
    t = cp.ring_allgather_time(m, 1e6, 2)
    assert cp.bus_bandwidth(2 * 1e6, t, 2) == pytest.approx(B)
    for p in (8, 64, 1024):
        mm = cp.CollectiveModel(1e-5, B)
        prev = 0.0
        for e in range(10, 31):
            s = float(2 ** e)
            bw = cp.bus_bandwidth(p * s, cp.ring_allgather_time(mm, s, p), p)
            assert prev < bw <= B
            prev = bw


def test_plan_examples_and_acceptance_7():
    assert cp.plan_unit_size(L3_8B, 32, 1024, cp.CollectiveModel(0.0, 1e10), 1 << 40).blocks_per_unit == 1
    big = cp.plan_unit_size(L3_8B, 32, 1024, cp.CollectiveModel(1.0, 1e10), 1 << 60)
    assert big.blocks_per_unit == 32
    with pytest.raises(cp.InfeasibleCap):
        cp.plan_unit_size(L3_8B, 32, 8, cp.CollectiveModel(1e-5, 1e10), 1000)
    rng = random.Random(0)
    for _ in range(200):
        shape = cp.ModelShape(rng.choice([256, 1024, 4096]), rng.choice([512, 4096, 14336]), rng.choice([8, 32]),
                              rng.choice([1, 8]), rng.choice([64, 128]), rng.randint(1, 40), rng.choice([1, 2, 4]))
        dp = rng.choice([2, 8, 64, 1024])
        model = cp.CollectiveModel(rng.choice([0.0, 1e-6, 1e-5, 1e-4]), rng.choice([1e9, 1e10, 7.7e11]))
        bb = cp.block_param_count(shape) * shape.dtype_bytes
        cap = bb * rng.randint(1, shape.layers + 2)
        plan = cp.plan_unit_size(shape, shape.layers, dp, model, cap)
        # brute force over g
        best_g, best_t = None, math.inf
        for g in range(1, shape.layers + 1):
            if g * bb > cap:
                break
            s = cp.fsdp_shard_bytes(g * cp.block_param_count(shape), shape.dtype_bytes, dp)
            t = -(-shape.layers // g) * 3 * cp.ring_allgather_time(model, s, dp)
            if t < best_t * (1.0 - 1e-12):
                best_g, best_t = g, t
        assert plan.blocks_per_unit == best_g
        assert plan.peak_unsharded_unit_bytes == best_g * bb


def test_properties_additivity_and_latency_direction():
    rng = random.Random(1)
    for _ in range(100):
        P, w, dp, g = rng.randint(1, 10**9), rng.choice([1, 2, 4]), rng.choice([1, 3, 8, 1024]), rng.randint(1, 8)
        assert cp.fsdp_shard_bytes(g * P, w, dp) <= g * cp.fsdp_shard_bytes(P, w, dp)
        if P % dp == 0:
            assert cp.fsdp_shard_bytes(g * P, w, dp) == g * cp.fsdp_shard_bytes(P, w, dp)
    m = cp.CollectiveModel(1e-5, 1e10)
    _, _, t1 = cp._unit_cost(L3_8B, 1, 1024, m)
    _, _, t32 = cp._unit_cost(L3_8B, 32, 1024, m)
    assert t32 <= t1


def test_message_size_table():
    csv = cp.message_size_table(L3_8B, [8, 64, 1024], [1, 2])
    lines = csv.strip().splitlines()
    assert lines[0] == "dp,blocks_per_unit,shard_bytes,busbw_bytes_per_sec,latency_share,step_comm_seconds"
    assert "1024,1,426000," in csv
    rows = [l.split(",") for l in lines[1:]]
    g1 = [int(r[2]) for r in rows if r[1] == "1"]
    assert g1 == sorted(g1, reverse=True)  # shard bytes non-increasing in dp


def test_fit_alpha_beta():
    true = cp.CollectiveModel(2e-5, 7.5e11)
    pts = [(p, m, cp.ring_allgather_time(true, m, p)) for p in (2, 4, 8) for m in (1e6, 1e7, 1e8, 1e9)]
    fit = cp.fit_alpha_beta(pts)
    assert fit.alpha == pytest.approx(2e-5, rel=1e-6) and fit.bandwidth == pytest.approx(7.5e11, rel=1e-6)


def test_calibrate_from_committed_nvlink_sweeps():
    """alpha/B fitted to the measured B200 sweeps reproduce the sweep times."""
    import os

    from conftest import ROOT
    from paper_2602_08387_b200.comm_planner import (ModelShape, calibrate, calibrated_plan, load_sweep,
                                                    ring_allgather_time)

    for w in (2, 4):
        rows = load_sweep(os.path.join(ROOT, "profiles", f"r1_collective_sweep_w{w}.jsonl"))
        m = calibrate(rows, "all_gather", "bfloat16")
        assert 0 <= m.alpha < 1e-4 and 2e11 < m.bandwidth < 2e12, (w, m)
        big = [r for r in rows if r.get("op") == "all_gather" and r["bytes"] >= 1 << 28]
        for r in big:  # the model predicts the large-message times within 25%
            t = ring_allgather_time(m, r["bytes"] / r["ranks"], r["ranks"])
            assert abs(t - r["seconds"]) / r["seconds"] < 0.25, (w, r["bytes"], t, r["seconds"])
        plan = calibrated_plan(ModelShape(4096, 14336, 32, 8, 128, 32), w, rows, memory_cap_bytes=2 << 30)
        assert 1 <= plan.blocks_per_unit <= 4
