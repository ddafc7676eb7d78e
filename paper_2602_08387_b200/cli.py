"""Command line: resolve / train / plan over config-graph documents.

    python -m paper_2602_08387_b200.cli resolve -c cfg.yaml [--root trainer] [--set n.config.p=v] [--instantiate]
    python -m paper_2602_08387_b200.cli train   -c cfg.yaml --root trainer [--set ...] [--json]
    python -m paper_2602_08387_b200.cli plan    -c plan.yaml --root planner
    python -m paper_2602_08387_b200.cli tokenize -c tok.yaml --root pipeline [--json]
    python -m paper_2602_08387_b200.cli index   corpus.jsonl            (GPU newline scan -> corpus.jsonl.didx)
    python -m paper_2602_08387_b200.cli shuffle packed.cfpk --seed S    (-> packed.cfpk.perm, document order)
    python -m paper_2602_08387_b200.cli chunk   packed.cfpk packed.cfpk.perm K out_dir   (GPU materialize)
    python -m paper_2602_08387_b200.cli sample  packed.cfpk S L         (prints the L+1 token ids)
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
    for name in ("resolve", "train", "plan", "tokenize"):
        p = sub.add_parser(name)
        p.add_argument("-c", "--config", required=True)
        p.add_argument("--root", default=None)
        p.add_argument("--set", action="append", default=[])
        p.add_argument("--json", action="store_true")
        if name == "resolve":
            p.add_argument("--instantiate", action="store_true")
    p = sub.add_parser("index")
    p.add_argument("raw_path")
    p.add_argument("--json", action="store_true")
    p = sub.add_parser("shuffle")
    p.add_argument("packed")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--json", action="store_true")
    p = sub.add_parser("chunk")
    p.add_argument("packed")
    p.add_argument("perm")
    p.add_argument("k", type=int)
    p.add_argument("out_dir")
    p.add_argument("--json", action="store_true")
    p = sub.add_parser("sample")
    p.add_argument("packed")
    p.add_argument("s", type=int)
    p.add_argument("L", type=int)
    p.add_argument("--json", action="store_true")
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
        if args.cmd in ("index", "shuffle", "chunk", "sample"):
            return _data_cmd(args)
        if args.cmd == "tokenize":
            og = _load(args, instantiate=True)
            st = og[args.root or og.order[-1]].run()
            print(json.dumps(st.summary()) if args.json else
                  f"tokenized {st.documents} documents ({st.skipped} skipped, {st.malformed} malformed) "
                  f"into {st.tokens} tokens")
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
    except (OSError, RuntimeError, ValueError, IndexError) as e:
        print(f"ERROR -: {type(e).__name__}: {e}")
        return 1
    return 0


def _data_cmd(args) -> int:
    """index / shuffle / chunk / sample (SPEC cli: plain flags, one summary line, --json)."""
    import os

    from . import packed as P

    out = {}
    if args.cmd == "index":
        from . import corpus_index as CI

        ix = CI.build_index(args.raw_path)
        side = CI.index_sidecar_path(args.raw_path)
        CI.write_index(ix, side)
        out = {"documents": ix.doc_count, "index": side}
        line = f"indexed {ix.doc_count} documents -> {side}"
    elif args.cmd == "shuffle":
        r = P.open_packed(args.packed)
        if args.seed < 0:
            raise ValueError("seed must be >= 0 (a uint64)")
        perm = P.make_permutation(r.doc_count, args.seed)
        path = args.packed + ".perm"
        P.write_permutation(perm, path)
        out = {"documents": r.doc_count, "seed": args.seed, "perm": path}
        line = f"shuffled {r.doc_count} documents (seed {args.seed}) -> {path}"
    elif args.cmd == "chunk":
        r = P.open_packed(args.packed)
        spec = P.chunk(P.load_permutation(args.perm), args.k)
        os.makedirs(args.out_dir, exist_ok=True)
        ds = P.DevicePackedStream(r)
        paths = []
        for c, docs in enumerate(spec.assignments):
            path = os.path.join(args.out_dir, f"chunk_{c:05d}.cfpk")
            P.materialize_chunk_gpu(r, docs, path, stream=ds)
            paths.append(path)
        out = {"chunks": len(paths), "sizes": [len(a) for a in spec.assignments]}
        line = f"wrote {len(paths)} chunks to {args.out_dir}"
    else:
        r = P.open_packed(args.packed)
        ids = [int(x) for x in r.get_sample(args.s, args.L)]
        out = {"sample": args.s, "L": args.L, "ids": ids}
        line = " ".join(str(x) for x in ids)
    print(json.dumps(out) if args.json else line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
