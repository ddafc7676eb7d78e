"""Registry-factory component graph: YAML -> DependencyGraph -> ObjectGraph.

The reference specifies this boundary without code (module
``config_graph``); the paper's framework builds its model, optimizer,
dataloader and SPMD trainer through it. This module is
that engine; ``components.py`` registers the B200 training-step components
into it so a config drops into the same object graph.

Semantics (SPEC.md references):
  * register_component: (interface, variant) unique -> DuplicateVariant (:55-63)
  * parse_config: top-level mapping node_id -> {interface, variant, config};
    references are the tagged scalar ``!ref node_id`` (:65-73, :103, :114)
  * build_graph: UnknownComponent, CycleError(path), InterfaceMismatch
    (expected vs actual), MissingParam, ParamTypeError; nominal interface
    check; no scalar coercion (an int does not satisfy a float, a bool does
    not satisfy an int); zero factory calls on failure (:75-83, :95-108)
  * resolve: topological order with lexicographic tie-break, each node built
    exactly once (shared instance on fan-in), ConstructionError(node_id) and
    no partial graph on a factory failure (:85-93, :104)
  * unused nodes -> warnings; diagnostics "LEVEL node_id: message" (:105, :115)
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Any, Callable

import yaml

KINDS = ("int", "float", "string", "bool", "list", "dependency")


# ------------------------------------------------------------------ errors
class ConfigError(Exception):
    """Base of all configuration errors; carries the node and all diagnostics found."""

    level = "ERROR"

    def __init__(self, node_id: str | None, message: str):
        super().__init__(f"{node_id}: {message}" if node_id else message)
        self.node_id = node_id
        self.message = message
        self.diagnostics = [self]

    def diagnostic(self) -> str:
        return f"{self.level} {self.node_id or '-'}: {self.message}"


class ConfigSyntaxError(ConfigError):
    pass


class SchemaError(ConfigError):
    pass


class DuplicateVariant(ConfigError):
    pass


class UnknownComponent(ConfigError):
    pass


class CycleError(ConfigError):
    def __init__(self, path: list):
        super().__init__(path[0], "dependency cycle " + " -> ".join(path))
        self.path = path


class InterfaceMismatch(ConfigError):
    def __init__(self, node_id, param, expected, actual):
        super().__init__(node_id, f"parameter '{param}' expects interface '{expected}' but "
                                  f"references a node of interface '{actual}'")
        self.expected, self.actual = expected, actual


class MissingParam(ConfigError):
    pass


class ParamTypeError(ConfigError):
    pass


class ConstructionError(ConfigError):
    pass


# ------------------------------------------------------------------ types
@dataclass(frozen=True)
class ParamSpec:
    name: str
    kind: str
    required: bool = True
    default: Any = None
    interface: str | None = None  # for kind == "dependency" (or a list of dependencies)

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown ParamSpec kind {self.kind!r}")
        if self.kind == "dependency" and not self.interface:
            raise ValueError("a dependency ParamSpec names exactly one interface")


@dataclass(frozen=True)
class FactoryDescriptor:
    interface: str
    variant: str
    params: tuple
    construct: Callable

    def __post_init__(self):
        names = [p.name for p in self.params]
        if len(names) != len(set(names)):
            raise ValueError(f"{self.interface}/{self.variant}: duplicate parameter names")


@dataclass(frozen=True)
class Reference:
    node_id: str


@dataclass
class ComponentNode:
    node_id: str
    interface: str
    variant: str
    config: dict


@dataclass
class DependencyGraph:
    nodes: dict
    edges: list  # (from node_id, to node_id): `from` references `to`
    order: list  # construction order (dependencies first, lexicographic ties)
    warnings: list = field(default_factory=list)


@dataclass
class ObjectGraph:
    instances: dict
    roots: list
    order: list
    warnings: list = field(default_factory=list)

    def __getitem__(self, node_id):
        return self.instances[node_id]


class Registry:
    def __init__(self):
        self._d = {}

    def register_component(self, desc: FactoryDescriptor) -> "Registry":
        key = (desc.interface, desc.variant)
        if key in self._d:
            raise DuplicateVariant(None, f"({desc.interface}, {desc.variant}) is already registered")
        self._d[key] = desc
        return self

    def get(self, interface: str, variant: str) -> FactoryDescriptor | None:
        return self._d.get((interface, variant))

    def __len__(self):
        return len(self._d)

    def __contains__(self, key):
        return key in self._d


def register_component(registry: Registry, desc: FactoryDescriptor) -> Registry:
    return registry.register_component(desc)


# ------------------------------------------------------------------ parse
class _Loader(yaml.SafeLoader):
    pass


def _ref_ctor(loader, node):
    if not isinstance(node, yaml.ScalarNode):
        raise yaml.constructor.ConstructorError(None, None, "!ref takes a node id", node.start_mark)
    return Reference(str(loader.construct_scalar(node)))


_Loader.add_constructor("!ref", _ref_ctor)


def parse_config(text: str) -> dict:
    """YAML text -> {node_id: ComponentNode}. Dangling references are build errors, not parse errors."""
    try:
        doc = yaml.load(text, Loader=_Loader)
    except yaml.YAMLError as e:
        raise ConfigSyntaxError(None, f"malformed configuration: {e}") from None
    if doc is None:
        return {}
    if not isinstance(doc, dict):
        raise ConfigSyntaxError(None, "the top level must be a mapping node_id -> component")
    nodes = {}
    for node_id, body in doc.items():
        node_id = str(node_id)
        if not isinstance(body, dict):
            raise SchemaError(node_id, "a component must be a mapping with interface, variant, config")
        for key in ("interface", "variant"):
            if key not in body or not isinstance(body[key], str):
                raise SchemaError(node_id, f"missing '{key}'")
        extra = set(body) - {"interface", "variant", "config"}
        if extra:
            raise SchemaError(node_id, f"unexpected keys {sorted(extra)}")
        cfg = body.get("config") or {}
        if not isinstance(cfg, dict):
            raise SchemaError(node_id, "'config' must be a mapping")
        nodes[node_id] = ComponentNode(node_id, body["interface"], body["variant"], dict(cfg))
    return nodes


def apply_overrides(nodes: dict, overrides: list) -> dict:
    """`--set node.config.param=value`: value parsed as a YAML scalar."""
    for ov in overrides:
        if "=" not in ov:
            raise ConfigSyntaxError(None, f"override {ov!r} is not key=value")
        path, raw = ov.split("=", 1)
        parts = path.split(".")
        if len(parts) != 3 or parts[1] != "config":
            raise ConfigSyntaxError(None, f"override path {path!r} must be node.config.param")
        node_id, _, param = parts
        if node_id not in nodes:
            raise UnknownComponent(node_id, "override targets an unknown node")
        nodes[node_id].config[param] = yaml.load(raw, Loader=_Loader)
    return nodes


# ------------------------------------------------------------------ validate
def _type_ok(kind: str, v) -> bool:
    if kind == "int":
        return isinstance(v, int) and not isinstance(v, bool)
    if kind == "float":
        return isinstance(v, float)
    if kind == "string":
        return isinstance(v, str)
    if kind == "bool":
        return isinstance(v, bool)
    if kind == "list":
        return isinstance(v, list)
    return False


def _check_node(node: ComponentNode, registry: Registry, nodes: dict, errs: list, edges: list):
    desc = registry.get(node.interface, node.variant)
    if desc is None:
        errs.append(UnknownComponent(node.node_id, f"no component registered for interface '{node.interface}' "
                                                   f"variant '{node.variant}'"))
        return
    specs = {p.name: p for p in desc.params}
    for k in node.config:
        if k not in specs:
            errs.append(ParamTypeError(node.node_id, f"unknown parameter '{k}' for {node.interface}/{node.variant}"))
    for p in desc.params:
        if p.name not in node.config:
            if p.required and p.default is None:
                errs.append(MissingParam(node.node_id, f"missing required parameter '{p.name}'"))
            continue
        v = node.config[p.name]
        refs = [v] if isinstance(v, Reference) else [x for x in v if isinstance(x, Reference)] if isinstance(
            v, list) else []
        if p.kind == "dependency":
            if not isinstance(v, Reference):
                errs.append(ParamTypeError(node.node_id, f"parameter '{p.name}' must be a !ref to a "
                                                         f"'{p.interface}' node, got {type(v).__name__}"))
                continue
        elif isinstance(v, Reference) or (refs and p.interface is None):
            errs.append(ParamTypeError(node.node_id, f"parameter '{p.name}' of kind {p.kind} cannot hold a !ref"))
            continue
        elif not _type_ok(p.kind, v):
            errs.append(ParamTypeError(node.node_id, f"parameter '{p.name}' expects {p.kind}, got "
                                                     f"{type(v).__name__} {v!r} (no coercion)"))
            continue
        for r in refs:
            if r.node_id not in nodes:
                errs.append(UnknownComponent(node.node_id, f"parameter '{p.name}' references unknown node "
                                                           f"'{r.node_id}'"))
                continue
            edges.append((node.node_id, r.node_id))
            actual = nodes[r.node_id].interface
            if actual != p.interface:
                errs.append(InterfaceMismatch(node.node_id, p.name, p.interface, actual))


def _find_cycle(nodes: dict, adj: dict):
    color = {n: 0 for n in nodes}
    stack = []

    def dfs(u):
        color[u] = 1
        stack.append(u)
        for v in sorted(adj.get(u, ())):
            if color[v] == 1:
                return stack[stack.index(v):] + [v]
            if color[v] == 0:
                c = dfs(v)
                if c:
                    return c
        stack.pop()
        color[u] = 2
        return None

    for n in sorted(nodes):
        if color[n] == 0:
            c = dfs(n)
            if c:
                return c
    return None


def build_graph(nodes: dict, registry: Registry, roots: list | None = None) -> DependencyGraph:
    """Validate against the registry (no factory is called) and order the DAG."""
    errs, edges = [], []
    for node_id in sorted(nodes):
        _check_node(nodes[node_id], registry, nodes, errs, edges)
    adj = {}
    for a, b in edges:
        adj.setdefault(a, set()).add(b)
    cyc = _find_cycle(nodes, adj)
    if cyc:
        errs.append(CycleError(cyc))
    if errs:
        first = errs[0]
        first.diagnostics = errs
        raise first
    # Kahn: a node is ready when all nodes it references are built; ties lexicographic
    indeg = {n: len(adj.get(n, ())) for n in nodes}
    users = {}
    for a, b in set(edges):
        users.setdefault(b, []).append(a)
    ready = [n for n, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        n = heapq.heappop(ready)
        order.append(n)
        for u in users.get(n, ()):
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(ready, u)
    warnings = []
    if roots:
        for r in roots:
            if r not in nodes:
                e = UnknownComponent(r, "root node is not defined in the configuration")
                raise e
        reach, todo = set(), list(roots)
        while todo:
            n = todo.pop()
            if n not in reach:
                reach.add(n)
                todo.extend(adj.get(n, ()))
        warnings = [f"WARNING {n}: node is not used by root(s) {', '.join(roots)}" for n in order if n not in reach]
    return DependencyGraph(nodes=dict(nodes), edges=sorted(set(edges)), order=order, warnings=warnings)


def resolve(graph: DependencyGraph, registry: Registry, roots: list | None = None) -> ObjectGraph:
    """Instantiate every node once, dependencies first. Any factory failure -> ConstructionError."""
    instances = {}
    for node_id in graph.order:
        node = graph.nodes[node_id]
        desc = registry.get(node.interface, node.variant)
        kwargs = {}
        for p in desc.params:
            if p.name in node.config:
                v = node.config[p.name]
                if isinstance(v, Reference):
                    v = instances[v.node_id]
                elif isinstance(v, list):
                    v = [instances[x.node_id] if isinstance(x, Reference) else x for x in v]
                kwargs[p.name] = v
            elif p.default is not None or not p.required:
                kwargs[p.name] = p.default
        try:
            instances[node_id] = desc.construct(**kwargs)
        except Exception as e:  # no partial graph escapes
            raise ConstructionError(node_id, f"factory {node.interface}/{node.variant} failed: "
                                             f"{type(e).__name__}: {e}") from e
    return ObjectGraph(instances=instances, roots=list(roots or []), order=list(graph.order),
                       warnings=list(graph.warnings))


def load(text: str, registry: Registry, roots: list | None = None, overrides: list | None = None,
         instantiate: bool = True):
    """parse -> overrides -> build_graph (-> resolve)."""
    nodes = apply_overrides(parse_config(text), overrides or [])
    graph = build_graph(nodes, registry, roots)
    return resolve(graph, registry, roots) if instantiate else graph
