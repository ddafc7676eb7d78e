"""Training-step throughput on B200: tokens/s (whole job), tokens/s/GPU and MFU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config gpt2-124m]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1; one rank per GPU, NCCL)

Workload (BASELINE.json configs[1]): GPT-2 small 124M, FSDP bf16, seq 2048,
8 sequences per GPU per step (weak scaling), random-init weights, synthetic
CFPKD001 token data. A step = gather the step's samples from the packed stream,
forward, backward, reduce-scatter, AdamW. Prints ONE JSON line on rank 0.

`value` is timed with CUDA events on the compute stream (inputs resident in
HBM), max over ranks. `e2e` repeats the measurement through the public API
with host buffers: each step's token windows are copied from the host memory
map into pinned memory and H2D, and the step's loss is read back D2H.
`--impl reference` times the CPU fp32 oracle of the same step (oracle/) on
the host cores -- the reference itself has no training step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec/GPU and MFU, GPT-2/Llama FSDP2 bf16 at 1/2/4/8 B200"
UNIT = "tokens/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sust": p.get("bf16_tflops_sustained",
                                                                                         p["bf16_tflops"]),
                "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sust": 1400.0, "src": "fallback"}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 100 ms during a timed region.

    In-process NVML queries (nvidia-ml-py): spawning nvidia-smi every few hundred ms
    stalls this process's CUDA calls long enough to distort a host-synchronous timed
    region; falls back to nvidia-smi when NVML is unavailable.
    """

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv, h = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            return float(sm), float(mx), [n for b, n in self.REASONS.items() if bits & b]
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        v = [x.strip() for x in out.stdout.strip().split(",")]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return float(v[0]), float(v[1]), [names[i] for i in range(4) if v[2 + i].lower() in ("active", "1")]

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"], "samples": 0}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({x for r in self.rows for x in r[2]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.rows[0][1], "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


def _gemm_traffic(config):
    """Measured DRAM bytes (read + write) per step of the GEMM class, from the committed ncu pass
    over one step of this config (tools/gpu/r2_raster.sh -> profiles/r2_<config>_step_metrics.csv),
    or None when no capture of this config is committed."""
    import csv
    import io

    path = os.path.join(ROOT, "profiles", f"r2_{config.replace('-', '')}_step_metrics.csv")
    if not os.path.exists(path):
        return None
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    h = rows[0]
    iN, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for r in rows[1:]:
        if "gemm_kernel" in r[iN] and r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
    return {"bytes_per_step": round(tot), "src": os.path.relpath(path, ROOT)}


def _gemm_algorithmic_bytes(detail):
    """Minimum DRAM bytes of one GEMM launch (operands read once, outputs written once)."""
    M, N, K, _, _, out, acc, bias, act = detail
    if act == "swiglu":  # x [M,K], w13 [2F,K] -> gu [M,2F] + h [M,F]
        return 2 * (M * K + N * K) + 2 * M * N + M * N
    if act == "dswiglu":  # dy [M,K], w2, gu [M,2F] in -> dgu [M,2F] out
        return 2 * (M * K + N * K) + 4 * M * N + 4 * M * N
    c = (4 if out == "f32" else 2) * M * N * (2 if acc else 1)
    aux = 2 * M * N if act in (5, 6, 1, 2) else 0
    return 2 * (M * K + N * K) + c + aux


def _data_path(cfg, n_tokens):
    from paper_2602_08387_b200.data import synthetic_path

    return synthetic_path(os.path.join(ROOT, ".bench_data"), n_tokens, cfg.vocab_size, kind="uniform", seed=0)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_08387_b200 import _lib, ops
    from paper_2602_08387_b200.data import PackedDataLoader, Sampler
    from paper_2602_08387_b200.model import PRESETS, DecoderLM
    from paper_2602_08387_b200.optim import AdamWConfig
    from paper_2602_08387_b200.packed import open_packed
    from paper_2602_08387_b200.trainer import SPMDTrainer

    cfg = PRESETS[args.config]
    B, T = args.batch, args.seq
    world = int(os.environ.get("WORLD_SIZE", "1"))
    steps_needed = args.warmup + 3 * args.steps + 4
    n_tokens = max(1 << 22, (steps_needed * world * B + 4) * T + 1)
    rank = int(os.environ.get("RANK", "0"))
    # rank 0 writes the synthetic corpus; the others wait (file name is content-addressed)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    path = None
    if rank == 0:
        path = _data_path(cfg, n_tokens)
    # B2S_GRAD_CLIP: diagnostics only (the reference default, 1.0, is what the bench line reports)
    ocfg = AdamWConfig(grad_clip=float(os.environ.get("B2S_GRAD_CLIP", AdamWConfig().grad_clip)))
    tr = SPMDTrainer(DecoderLM(cfg, activation_checkpointing=args.ac), ocfg, None, steps=0, seed=0,
                     blocks_per_unit=args.blocks_per_unit, init_device="cuda")
    # distributed init happens in setup(); make sure the data file exists first
    from paper_2602_08387_b200.trainer import init_distributed

    rank, world, local, device = init_distributed()
    if world > 1:
        dist.barrier()
    path = _data_path(cfg, n_tokens)
    reader = open_packed(path)
    tr.dataloader = PackedDataLoader(reader, B, T, Sampler(shuffle=True, seed=0), feed="resident")
    tr.setup()
    peaks = _peaks()

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    step = 0
    for _ in range(args.warmup):
        tr.train_step(step)
        step += 1
    barrier_sync()
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            tr.train_step(step)
            step += 1
        end.record()
        barrier_sync()
    launches = _lib.launch_count() - launches0
    ms = start.elapsed_time(end) / args.steps
    t = torch.tensor([ms], device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    loss_dev = float(tr._loss.item())
    # ---- end to end through the public API with host buffers (staged windows, loss D2H each step)
    e2e_dl = PackedDataLoader(reader, B, T, Sampler(shuffle=True, seed=0), feed="staged")
    e2e_dl.bind(rank, world, device)
    tr.dataloader = e2e_dl
    for _ in range(2):
        tr.train_step(step)
        step += 1
    barrier_sync()
    # every step: its windows staged from the host memory map into pinned memory and
    # copied H2D, its loss copied D2H into pinned memory; the host reads step k's loss
    # while step k+lag runs (pipelined like a training loop that logs)
    # steps between a loss's D2H and its host read: 2 keeps a host hiccup (GC, page faults)
    # on one rank from stalling the collectives of the others
    lag = int(os.environ.get("B2S_E2E_LAG", "2"))
    loss_host = [torch.empty(1, dtype=torch.float32, pin_memory=True) for _ in range(lag + 1)]
    loss_ev = [torch.cuda.Event() for _ in range(lag + 1)]
    e2e_losses = []
    clk_e2e = ClockSampler(local)
    clk_e2e.__enter__()
    t0 = time.perf_counter()
    for k in range(args.steps):
        inputs, targets = e2e_dl.batch(step)
        loss = tr.step_on(inputs, targets)
        n = lag + 1
        loss_host[k % n].copy_(loss, non_blocking=True)  # D2H of the step's result
        loss_ev[k % n].record()
        if k >= lag:
            loss_ev[(k - lag) % n].synchronize()
            e2e_losses.append(float(loss_host[(k - lag) % n].item()))
        step += 1
    for j in range(max(0, args.steps - lag), args.steps):
        loss_ev[j % (lag + 1)].synchronize()
        e2e_losses.append(float(loss_host[j % (lag + 1)].item()))
    barrier_sync()
    clk_e2e.__exit__(None, None, None)
    e2e_ms = (time.perf_counter() - t0) * 1000 / args.steps
    te = torch.tensor([e2e_ms], device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())

    # per-kernel roofline: the same steps again with CUDA events around every
    # GEMM / attention launch on the compute stream (kept out of `value`)
    tr.dataloader = PackedDataLoader(reader, B, T, Sampler(shuffle=True, seed=0), feed="resident")
    tr.dataloader.bind(rank, world, device)
    if world > 1:
        tr.engine.timing = []  # CUDA events around every all-gather / reduce-scatter (same pass)
    with ops.KernelTimer() as kt:
        for _ in range(args.steps):
            tr.train_step(step)
            step += 1
        barrier_sync()
    kern = kt.summary()
    gemm_alg_bytes = sum(_gemm_algorithmic_bytes(det) * n for (kind, det), n, _ms, _tf in kt.detail()
                         if kind == "gemm") / args.steps
    coll = tr.engine.collective_summary() if world > 1 else None
    tr.engine.timing = None

    if rank != 0:
        return None
    tokens_step = world * B * T
    value = tokens_step / (ms / 1000)
    per_gpu = value / world
    fpt = cfg.flops_per_token(T)
    mfu = per_gpu * fpt / (peaks["bf16"] * 1e12)
    g = kern.get("gemm", {"flops": 0, "ms": 1e-9, "launches": 0})
    gemm_tf = g["flops"] / (g["ms"] / 1000) / 1e12 if g["ms"] > 0 else 0.0
    per_kernel = {k: {"launches_per_step": v["launches"] // args.steps,
                      "ms_per_step": round(v["ms"] / args.steps, 3),
                      "tflops": round(v["flops"] / (v["ms"] / 1000) / 1e12, 1) if v["ms"] > 0 else None}
                  for k, v in kern.items()}
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform token ids, CFPKD001 packed file); "
                                                          "random-init weights",
        "config": workload_config(args, world),
        "tokens_per_sec_per_gpu": round(per_gpu, 1),
        "mfu": round(mfu, 4),
        "mfu_vs_sustained_peak": round(per_gpu * fpt / (peaks["bf16_sust"] * 1e12), 4),
        "flops_per_token": fpt,
        "loss_last": round(loss_dev, 4),
        "roofline": {"bound": "tensor", "kernel": "b2s gemm (tcgen05)", "achieved": round(gemm_tf, 1),
                     "peak": peaks["bf16_sust"], "unit": "TFLOP/s", "frac": round(gemm_tf / peaks["bf16_sust"], 3),
                     "frac_vs_burst_peak": round(gemm_tf / peaks["bf16"], 3),
                     "traffic": (_gemm_traffic(args.config) or {}).get("bytes_per_step"),
                     "traffic_unit": "DRAM bytes per step, all GEMM launches (ncu, committed capture)",
                     "traffic_src": (_gemm_traffic(args.config) or {}).get("src"),
                     "algorithmic_bytes_per_step": round(gemm_alg_bytes),
                     "peak_src": f"{peaks['src']} bf16 sustained (kernel timed inside a long step)",
                     "achieved_src": "sum of algorithmic GEMM FLOPs / sum of CUDA-event launch durations over "
                                     f"{args.steps} instrumented steps",
                     "launches_per_step": g["launches"] // max(1, args.steps)},
        "kernels": per_kernel,
        # FSDP collectives (NCCL over NVLink 5 / NVSwitch), nccl-tests busbw vs 900 GB/s per direction,
        # timed on the comm stream while they overlap compute (so below the isolated sweep's numbers)
        "collectives": ({k: {kk: vv for kk, vv in v.items() if kk != "bytes"} | {"bytes_per_step": v["bytes"] // args.steps}
                         for k, v in coll.items()} if coll else None),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": {"value": round(tokens_step / (e2e_ms / 1000), 1), "unit": UNIT,
                "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": e2e_dl.h2d_bytes_per_step(), "d2h_bytes_per_step": 4,
                "clocks": clk_e2e.summary()},
    }
    if args.cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(cfg, T, args)
    elif world > 1:
        out["cpu_baseline"] = None
    return out


# CPU sample per reference step: (sequences, tokens) sized so one oracle step takes a few
# seconds on the GPU box's host cores (the full 1B step at 1 x 4096 tokens takes ~40 s there)
REF_SAMPLE = {"tiny-gpt2": (8, 256), "gpt2-124m": (1, 2048), "llama-1b": (1, 512), "llama-8b": None}


def workload_config(args, world):
    """The bench line's `config` (both arms: the reference arm times a CPU sample of this workload)."""
    return {"workload": f"{args.config} FSDP training step (fwd+bwd+AdamW), seq {args.seq}, {args.batch} seqs/GPU",
            "model": args.config, "global_batch": world * args.batch, "seq_len": args.seq,
            "parallelism": f"fsdp{world}", "blocks_per_unit": args.blocks_per_unit,
            "activation_checkpointing": args.ac,
            "l2": "working set (weights + activations) >> 126 MB L2; no explicit flush"}


def _oracle_step_timer(cfg, T, B, steps, warmup):
    """Time OracleTrainer steps (CPU fp32) on synthetic samples; returns (tokens/s, threads, secs)."""
    import torch

    from oracle.model_oracle import OracleTrainer
    from paper_2602_08387_b200.model import init_params

    torch.manual_seed(0)
    tr = OracleTrainer(cfg, init_params(cfg, 0))
    gen = torch.Generator().manual_seed(0)
    x = torch.randint(0, cfg.vocab_size, (B, T + 1), generator=gen)
    for _ in range(warmup):
        tr.step(x[:, :T], x[:, 1:])
    t0 = time.perf_counter()
    for _ in range(steps):
        tr.step(x[:, :T], x[:, 1:])
    dt = time.perf_counter() - t0
    return B * T * steps / dt, torch.get_num_threads(), dt


def _data_path_baseline(cfg, B, T):
    """The packed-data feed on the host: the oracle restatement of PackedReader.get_sample
    (packed_data.py:196-203) over B windows of T+1 tokens, stacked and widened to int64, and the
    Fisher-Yates make_permutation (packed_data.py:257-282) in C; timed on one core."""
    import numpy as np

    from oracle import packed_oracle as orc
    from paper_2602_08387_b200.packed import open_packed

    path = _data_path(cfg, max(1 << 22, 64 * B * T + 1))
    r = open_packed(path)
    payload = np.asarray(r.payload)
    n = r.sample_count(T)
    rng = np.random.default_rng(0)
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < 1.0:
        ids = rng.integers(0, n, B)
        x, y = orc.batch_windows(payload, ids, T)
        reps += 1
    dt = time.perf_counter() - t0
    import ctypes

    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_build", "liboracle.so"))
    np_perm = 1 << 20
    out = np.empty(np_perm, dtype=np.uint64)
    t1 = time.perf_counter()
    lib.oracle_permutation(ctypes.c_uint64(np_perm), ctypes.c_uint64(0), out.ctypes.data_as(ctypes.c_void_p))
    dp = time.perf_counter() - t1
    return {"get_sample_batch_tokens_per_s": round(reps * B * T / dt, 1), "batch": f"{B} x {T + 1} tokens, "
            f"width {r.token_width}", "make_permutation_elems_per_s": round(np_perm / dp, 1),
            "cores": 1, "kind": "port", "sample": f"{reps} batches in {dt:.2f} s (oracle/packed_oracle.py "
            f"batch_windows); make_permutation(2^20, 0) in {dp * 1e3:.1f} ms (oracle/permutation_oracle.c)"}


def cpu_baseline(cfg, T, args):
    smp = REF_SAMPLE.get(args.config)
    if smp is None:
        return None
    Bs, Ts = smp[0], min(T, smp[1])
    tps, threads, dt = _oracle_step_timer(cfg, Ts, Bs, 1, 0)
    out = {"value": round(tps, 2), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"CPU fp32 oracle (oracle/model_oracle.py) of the {args.config} training step "
                     f"(fwd+bwd+clip+AdamW, all layers): {Bs} x {Ts} tokens, 1 step ({dt:.1f} s), "
                     f"torch threads={threads}, host cpus={len(os.sched_getaffinity(0))}"}
    try:
        out["data_path"] = _data_path_baseline(cfg, args.batch, T)
    except Exception as e:  # the step number above stands on its own
        out["data_path"] = {"error": str(e)[:200]}
    return out


def run_reference(args):
    from paper_2602_08387_b200.model import PRESETS

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cfg = PRESETS[args.config]
    smp = REF_SAMPLE.get(args.config)
    if smp is None:
        return {"impl": "reference", "unavailable": f"{args.config}: the fp32 CPU oracle needs ~130 GB of host "
                                                      "memory for its parameters and AdamW state"}
    Bs, Ts = smp[0], min(args.seq, smp[1])
    warm = args.warmup  # the same K / W as our arm (a step is a few seconds here)
    tps, threads, dt = _oracle_step_timer(cfg, Ts, Bs, args.steps, warm)
    sample = (f"{args.steps} steps of {Bs} x {Ts} tokens after {warm} warm-up, full {cfg.n_layer}-layer "
              f"{args.config} fp32 step (fwd+bwd+clip+AdamW) on the host cores; the reference has no training "
              "step (SPEC.md:12), so its arm is the CPU fp32 oracle (oracle/model_oracle.py)")
    if Ts < args.seq:
        sample += (f"; seq {Ts} instead of {args.seq} bounds the run (attention is 12*L*d*T of the "
                   f"{cfg.flops_per_token(args.seq) / 1e9:.2f} GF/token, so the shorter sample favours the CPU)")
    return {"metric": METRIC, "value": round(tps, 2), "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", 1)),
            "steps": args.steps, "warmup": warm, "ms_per_step": round(dt * 1000 / args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic token ids; random-init weights", "impl": "reference",
            "config": workload_config(args, int(os.environ.get("WORLD_SIZE", 1))),
            "cpu_baseline": {"value": round(tps, 2), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(tps, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# per-config workload defaults (BASELINE.json configs / SURVEY §8(a)): sequences per GPU, seq len, AC
CONFIGS = {
    "tiny-gpt2": (8, 256, False),
    "gpt2-124m": (8, 2048, False),   # configs[1]
    "llama-1b": (4, 4096, False),    # configs[2]: the north-star target
    "llama-8b": (2, 4096, True),     # configs[3]: per-block activation checkpointing
}


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1, not under torchrun): re-exec as N ranks, one per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama-1b", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU per step (default: per config)")
    ap.add_argument("--seq", type=int, default=None, help="sequence length (default: per config)")
    ap.add_argument("--blocks-per-unit", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--ac", action="store_true", default=None, help="per-block activation checkpointing")
    args = ap.parse_args()
    B0, T0, ac0 = CONFIGS[args.config]
    args.batch = B0 if args.batch is None else args.batch
    args.seq = T0 if args.seq is None else args.seq
    args.ac = ac0 if args.ac is None else args.ac
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1 and args.impl == "ours":  # (the CPU reference arm runs on rank 0 only)
        sys.exit(_self_launch(args))
    if world and world != args.gpus and args.impl == "ours":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_ours(args)  # (its trainer and graph are freed)
    if out is not None:
        print(json.dumps(out), flush=True)
    if args.impl == "ours" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist

        from paper_2602_08387_b200.trainer import destroy_process_group

        if dist.is_initialized():
            dist.barrier()
            destroy_process_group()


if __name__ == "__main__":
    main()
