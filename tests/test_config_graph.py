"""config_graph restated from SPEC.md:24-123: every SPEC example, the golden
diagnostics fixtures, and the invariants as properties."""

import os
import random

import pytest

from conftest import GOLDEN
from paper_2602_08387_b200 import config_graph as cg
from paper_2602_08387_b200.config_graph import FactoryDescriptor as FD
from paper_2602_08387_b200.config_graph import ParamSpec as P

DIAG = os.path.join(GOLDEN, "diagnostics")


def toy_registry(counter=None, fail=()):
    counter = counter if counter is not None else {}

    def mk(name):
        def ctor(**kw):
            counter[name] = counter.get(name, 0) + 1
            if name in fail:
                raise RuntimeError("boom")
            return {"kind": name, **kw}
        return ctor

    r = cg.Registry()
    r.register_component(FD("tokenizer", "byte", (), mk("byte")))
    r.register_component(FD("tokenizer", "bpe", (P("vocab_path", "string"), P("merges_path", "string")), mk("bpe")))
    r.register_component(FD("dataset_reader", "jsonl", (P("tokenizer", "dependency", interface="tokenizer"),
                                                        P("path", "string"), P("batch", "int")), mk("jsonl")))
    r.register_component(FD("pipeline", "default", (P("reader", "dependency", interface="dataset_reader"),
                                                    P("workers", "int"), P("lr", "float"),
                                                    P("verbose", "bool", required=False, default=False)),
                            mk("pipeline")))
    r.register_component(FD("node", "x", (P("next", "dependency", interface="node", required=False),
                                          P("deps", "list", required=False, interface="node")), mk("x")))
    return r


def test_register_component_examples():
    r = cg.Registry()
    cg.register_component(r, FD("tokenizer", "byte", (), lambda: 1))
    assert len(r) == 1
    with pytest.raises(cg.DuplicateVariant):
        cg.register_component(r, FD("tokenizer", "byte", (), lambda: 2))
    r2 = cg.Registry()
    for i in range(93):  # "93 pluggable components"
        cg.register_component(r2, FD(f"if{i % 32}", f"v{i}", (), lambda: i))
    assert len(r2) == 93 and all(r2.get(f"if{i % 32}", f"v{i}") for i in range(93))


def test_parse_config_examples():
    assert cg.parse_config("") == {}
    nodes = cg.parse_config("tok: {interface: tokenizer, variant: byte, config: {}}")
    assert list(nodes) == ["tok"] and nodes["tok"].interface == "tokenizer"
    nodes = cg.parse_config(open(os.path.join(DIAG, "dangling.yaml")).read())  # parses fine
    assert nodes["reader"].config["tokenizer"] == cg.Reference("missing_node")
    with pytest.raises(cg.UnknownComponent):
        cg.build_graph(nodes, toy_registry())
    with pytest.raises(cg.ConfigSyntaxError):
        cg.parse_config("a: [unclosed")
    with pytest.raises(cg.SchemaError):
        cg.parse_config("a: {variant: byte}")


def test_build_graph_examples():
    r = toy_registry()
    with pytest.raises(cg.CycleError) as e:
        cg.build_graph(cg.parse_config(open(os.path.join(DIAG, "cycle.yaml")).read()), r)
    assert e.value.path == ["A", "B", "A"]
    with pytest.raises(cg.InterfaceMismatch) as e:
        cg.build_graph(cg.parse_config(open(os.path.join(DIAG, "mismatch.yaml")).read()), r)
    assert (e.value.expected, e.value.actual) == ("tokenizer", "dataset_reader")
    diamond = """
A: {interface: node, variant: x, config: {deps: [!ref B, !ref C]}}
B: {interface: node, variant: x, config: {next: !ref D}}
C: {interface: node, variant: x, config: {next: !ref D}}
D: {interface: node, variant: x, config: {}}
"""
    g = cg.build_graph(cg.parse_config(diamond), r)
    assert len(g.nodes) == 4 and len(g.edges) == 4
    assert g.order == ["D", "B", "C", "A"]


GOLDEN_DIAGNOSTICS = {
    "cycle.yaml": ["ERROR A: dependency cycle A -> B -> A"],
    "mismatch.yaml": ["ERROR reader: parameter 'tokenizer' expects interface 'tokenizer' but references a node "
                      "of interface 'dataset_reader'"],
    "unknown.yaml": ["ERROR tok: no component registered for interface 'tokenizer' variant 'sentencepiece'"],
    "missing.yaml": ["ERROR reader: missing required parameter 'path'"],
    "type.yaml": ["ERROR pipe: parameter 'lr' expects float, got int 1 (no coercion)"],
    "dangling.yaml": ["ERROR reader: parameter 'tokenizer' references unknown node 'missing_node'"],
}


@pytest.mark.parametrize("name", sorted(GOLDEN_DIAGNOSTICS))
def test_golden_diagnostics(name, capsys):
    from paper_2602_08387_b200 import cli

    text = open(os.path.join(DIAG, name)).read()
    calls = {}
    with pytest.raises(cg.ConfigError) as e:
        cg.build_graph(cg.parse_config(text), toy_registry(calls))
    assert [d.diagnostic() for d in e.value.diagnostics] == GOLDEN_DIAGNOSTICS[name]
    assert calls == {}  # validation never runs a factory


def test_resolve_examples():
    calls = {}
    r = toy_registry(calls)
    og = cg.load("tok: {interface: tokenizer, variant: byte, config: {}}", r)
    assert len(og.instances) == 1
    diamond = """
A: {interface: node, variant: x, config: {deps: [!ref B, !ref C]}}
B: {interface: node, variant: x, config: {next: !ref D}}
C: {interface: node, variant: x, config: {next: !ref D}}
D: {interface: node, variant: x, config: {}}
"""
    calls.clear()
    og = cg.load(diamond, r)
    assert calls["x"] == 4  # D exactly once
    assert og["B"]["next"] is og["C"]["next"] is og["D"]
    assert og["A"]["deps"][0] is og["B"]
    with pytest.raises(cg.ConstructionError) as e:
        cg.load("tok: {interface: tokenizer, variant: byte, config: {}}", toy_registry(fail=("byte",)))
    assert e.value.node_id == "tok"


def test_valid_config_unused_warning_and_defaults():
    og = cg.load(open(os.path.join(DIAG, "valid.yaml")).read(), toy_registry(), roots=["pipe"])
    assert og["pipe"]["verbose"] is False
    assert og.warnings == ["WARNING spare: node is not used by root(s) pipe"]
    assert og.order == ["spare", "tok", "reader", "pipe"]


def test_overrides():
    text = open(os.path.join(DIAG, "valid.yaml")).read()
    og = cg.load(text, toy_registry(), overrides=["pipe.config.workers=16"])
    assert og["pipe"]["workers"] == 16
    with pytest.raises(cg.ParamTypeError):
        cg.load(text, toy_registry(), overrides=["pipe.config.workers=1.5"])


def test_bool_is_not_int_and_int_is_not_float():
    r = toy_registry()
    base = "tok: {interface: tokenizer, variant: byte, config: {}}\n" \
           "reader: {interface: dataset_reader, variant: jsonl, config: {tokenizer: !ref tok, path: p, batch: %s}}\n"
    with pytest.raises(cg.ParamTypeError):
        cg.build_graph(cg.parse_config(base % "true"), r)
    cg.build_graph(cg.parse_config(base % "3"), r)


def _random_dag(rng, n):
    lines = []
    for i in range(n):
        deps = [f"n{j:02d}" for j in range(i) if rng.random() < 0.3]
        ref = "[" + ", ".join(f"!ref {d}" for d in deps) + "]"
        lines.append(f"n{i:02d}: {{interface: node, variant: x, config: {{deps: {ref}}}}}")
    return lines


def test_property_random_dags_and_back_edges():
    rng = random.Random(0)
    r = toy_registry()
    for _ in range(60):
        n = rng.randint(2, 12)
        lines = _random_dag(rng, n)
        calls = {}
        og = cg.load("\n".join(lines), toy_registry(calls))
        pos = {k: i for i, k in enumerate(og.order)}
        g = cg.build_graph(cg.parse_config("\n".join(lines)), r)
        assert all(pos[b] < pos[a] for a, b in g.edges)  # dependencies first
        assert calls.get("x", 0) == n
        assert cg.build_graph(cg.parse_config("\n".join(lines)), r).order == g.order  # deterministic
        # inject a back edge from the first node to the last -> cycle
        lines2 = list(lines)
        lines2[0] = lines2[0].replace("deps: [", f"next: !ref n{n - 1:02d}, deps: [")
        if n > 1:
            nodes = cg.parse_config("\n".join(lines2))
            path_exists = True
            try:
                cg.build_graph(nodes, r)
                path_exists = False
            except cg.CycleError as e:
                assert e.path[0] == e.path[-1]
            # a cycle exists iff n-1 (transitively) depends on n0
            adj = {f"n{i:02d}": [] for i in range(n)}
            for a, b in g.edges:
                adj[a].append(b)
            seen, todo = set(), [f"n{n - 1:02d}"]
            while todo:
                u = todo.pop()
                if u not in seen:
                    seen.add(u)
                    todo += adj[u]
            assert path_exists == ("n00" in seen)


def test_default_registry_resolves_shipped_configs():
    from paper_2602_08387_b200.components import default_registry

    root = os.path.dirname(GOLDEN.rstrip("/").rsplit("/", 1)[0])
    for name in ("gpt2_124m.yaml", "llama_1b.yaml", "tiny_llama_parity.yaml", "plan_llama8b.yaml"):
        text = open(os.path.join(root, "configs", name)).read()
        g = cg.load(text, default_registry(), instantiate=False)
        assert g.order[-1] in ("trainer", "planner")


def test_cli_resolve_exit_codes(tmp_path, capsys):
    from paper_2602_08387_b200 import cli

    bad = tmp_path / "bad.yaml"
    bad.write_text("opt: {interface: optimizer, variant: adamw_fused, config: {lr: 1e-3}}\n")
    assert cli.main(["resolve", "-c", str(bad)]) == 2
    out = capsys.readouterr().out.strip().splitlines()
    assert out == ["ERROR opt: parameter 'lr' expects float, got str '1e-3' (no coercion)"]
    good = tmp_path / "good.yaml"
    good.write_text("opt: {interface: optimizer, variant: adamw_fused, config: {lr: 1.0e-3}}\n")
    assert cli.main(["resolve", "-c", str(good), "--instantiate"]) == 0
    assert cli.main(["resolve", "-c", str(good), "--set", "opt.config.warmup_steps=20"]) == 0
