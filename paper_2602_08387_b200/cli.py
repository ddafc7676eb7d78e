"""Command line: resolve / train / plan over config-graph documents.

    python -m paper_2602_08387_b200.cli resolve -c cfg.yaml [--root trainer] [--set n.config.p=v] [--instantiate]
    python -m paper_2602_08387_b200.cli train   -c cfg.yaml --root trainer [--set ...] [--json]
    python -m paper_2602_08387_b200.cli plan    -c plan.yaml --root planner
    python -m paper_2602_08387_b200.cli table   --hidden 4096 --ffn 14336 --heads 32 --kv-heads 8 --head-dim 128 \\
                                                --layers 32 --dp 8 64 1024 --g 1 2 4 [--sweep sweep.jsonl]

Exit codes: 0 success, 1 runtime/IO failure, 2 configuration invalid.
Diagnostics: one per line, "LEVEL node_id: message".
"""

from __future__ import annotations

import argparse
import json
import sys

from . import config_graph as cg


def _load(args, instantiate):
    from .components import default_registry

    with open(args.config) as f:
        text = f.read()
    roots = [args.root] if getattr(args, "root", None) else None
    return cg.load(text, default_registry(), roots, args.set or [], instantiate=instantiate)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2602_08387_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("resolve", "train", "plan"):
        p = sub.add_parser(name)
        p.add_argument("-c", "--config", required=True)
        p.add_argument("--root", default=None)
        p.add_argument("--set", action="append", default=[])
        p.add_argument("--json", action="store_true")
        if name == "resolve":
            p.add_argument("--instantiate", action="store_true")
    t = sub.add_parser("table")
    t.add_argument("--hidden", type=int, required=True)
    t.add_argument("--ffn", type=int, required=True)
    t.add_argument("--heads", type=int, required=True)
    t.add_argument("--kv-heads", type=int, required=True)
    t.add_argument("--head-dim", type=int, required=True)
    t.add_argument("--layers", type=int, required=True)
    t.add_argument("--dtype-bytes", type=int, default=2)
    t.add_argument("--dp", type=int, nargs="+", required=True)
    t.add_argument("--g", type=int, nargs="+", default=[1])
    t.add_argument("--alpha", type=float, default=1e-5)
    t.add_argument("--bandwidth", type=float, default=1e10)
    t.add_argument("--sweep", default=None, help="fit alpha/B to this collective_sweep JSONL (all-gather, bf16)")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "table":
            from .comm_planner import CollectiveModel, ModelShape, calibrate, load_sweep, message_size_table

            shape = ModelShape(args.hidden, args.ffn, args.heads, args.kv_heads, args.head_dim, args.layers,
                               args.dtype_bytes)
            model = (calibrate(load_sweep(args.sweep), "all_gather", "bfloat16") if args.sweep
                     else CollectiveModel(args.alpha, args.bandwidth))
            sys.stdout.write(message_size_table(shape, args.dp, args.g, model))
            return 0
        if args.cmd == "resolve":
            res = _load(args, instantiate=args.instantiate)
            for w in res.warnings:
                print(w)
            if args.json:
                print(json.dumps({"valid": True, "order": res.order}))
            return 0
        if args.cmd == "plan":
            og = _load(args, instantiate=True)
            plan = og[args.root or og.order[-1]]
            print(json.dumps(plan.__dict__) if args.json else plan)
            return 0
        if args.cmd == "train":
            og = _load(args, instantiate=True)
            trainer = og[args.root or og.order[-1]]
            losses = trainer.run()
            if getattr(trainer, "rank", 0) == 0:
                print(json.dumps({"losses": losses}) if args.json else f"final loss {losses[-1]:.4f}")
            return 0
    except cg.ConfigError as e:
        for d in e.diagnostics:
            print(d.diagnostic())
        return 2
    except (OSError, RuntimeError) as e:
        print(f"ERROR -: {type(e).__name__}: {e}")
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
