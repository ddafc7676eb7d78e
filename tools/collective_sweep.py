"""FSDP collective sweep (BASELINE.json configs[4]): all-gather / reduce-scatter busbw vs message size.

    torchrun --nproc-per-node N tools/collective_sweep.py [out.jsonl] [min_mb] [max_mb]

Sizes are the full (gathered) message M from 1 MB to 1 GB in powers of two;
AG moves bf16 (the FSDP parameter gather), RS fp32 and bf16 (gradient
reduce-scatter). 20 warm-up + 50 timed iterations (10 + 20 above 256 MB),
CUDA events on the issuing stream, max over ranks. Reports algbw = M/t and
the nccl-tests bus bandwidth busbw = algbw (p-1)/p against
NVLink 5's 900 GB/s per direction, then fits the SPEC's ring alpha-beta model
t = (p-1)(alpha + m/B) (comm_planner.fit_alpha_beta).
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200.comm_planner import fit_alpha_beta  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "collective_sweep.jsonl")
    lo = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    p, rank = dist.get_world_size(), dist.get_rank()
    rows, pts = [], []
    mb = lo
    while mb <= hi:
        for op, dt in (("all_gather", torch.bfloat16), ("reduce_scatter", torch.float32),
                       ("reduce_scatter", torch.bfloat16)):
            esz = torch.tensor([], dtype=dt).element_size()
            n = (mb << 20) // esz // p * p
            full = torch.randn(n, device=dev).to(dt)
            shard = torch.empty(n // p, device=dev, dtype=dt)

            def run():
                if op == "all_gather":
                    dist.all_gather_into_tensor(full, shard)
                else:
                    dist.reduce_scatter_tensor(shard, full, op=dist.ReduceOp.AVG)

            warm, iters = (20, 50) if mb <= 256 else (10, 20)
            for _ in range(warm):
                run()
            torch.cuda.synchronize()
            dist.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(iters):
                run()
            e.record()
            torch.cuda.synchronize()
            t = torch.tensor([s.elapsed_time(e) / iters / 1e3], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t = float(t.item())
            M = n * esz
            algbw = M / t
            busbw = algbw * (p - 1) / p
            row = {"op": op, "dtype": str(dt).split(".")[-1], "ranks": p, "bytes": M, "seconds": t,
                   "algbw_GBps": algbw / 1e9, "busbw_GBps": busbw / 1e9, "frac_of_900GBps": busbw / 900e9}
            rows.append(row)
            if op == "all_gather":
                pts.append((p, M / p, t))
            del full, shard
        mb *= 2
    if rank == 0:
        fit = fit_alpha_beta(pts)
        with open(out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
            f.write(json.dumps({"fit": "all_gather ring alpha-beta", "ranks": p, "alpha_s": fit.alpha,
                                "B_GBps": fit.bandwidth / 1e9}) + "\n")
        for r in rows:
            print(f"{r['op']:15s} {r['dtype']:9s} {r['bytes'] / 2**20:8.0f} MiB  {r['seconds'] * 1e6:9.1f} us  "
                  f"busbw {r['busbw_GBps']:7.1f} GB/s ({100 * r['frac_of_900GBps']:.0f}% of 900)")
        print(f"fit: alpha = {fit.alpha * 1e6:.2f} us, B = {fit.bandwidth / 1e9:.1f} GB/s")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
