"""Experiment driver over the CUDA path — the GPU-side mirror of gapa::bench
(include/gapa/bench.hpp, src/bench.cpp) and of the file loaders (src/graph.cpp:65-156).

JSON config -> GA run on the B200 through the C ABI -> one ResultRow per repetition, reported as
CSV that is byte-compatible with the reference's (same header, same shortest-round-trip number
format, bench.cpp:371-409).  The reference's determinism contract — byte identity of the CSV with
the wall_time_s column blanked (bench.hpp:83-85) — holds ACROSS implementations: the same config
gives the same bytes from the reference on CPU and from this driver on the GPU
(tests/golden/experiments.json).

All fitness arithmetic stays on the device: the metric columns come from the same kernels as the
GA's fitness (PC / MCN / Q / AUC of the empty and of the best perturbation), the detector's
partition (gapa_cuda_detect_communities) and the RA scores (gapa_cuda_lpa_scores).  Only the two
reporting-only reductions the reference computes once per run are host code here as they are
there: NMI (community.cpp:119-148) and the precision half of lp_auc_precision
(link_prediction.cpp:98-117).
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import math
from dataclasses import dataclass, field, replace
from decimal import Decimal

import numpy as np

from . import capi
from .api import (ClosurePolicy, DeviceGraph, Direction, GAParams, GenePool, Graph, LinkPredictionAttackObjective,
                  ModularityAttackObjective, PairwiseConnectivityObjective, PoolKind, SixDstObjective, TASK_MCN, TASK_PC,
                  build_gene_pool, build_lp_split, perturbation_budget, run_ga)
from .capi import GapaCudaError, check


class ConfigError(GapaCudaError):  # error.hpp:21-24
    def __init__(self, message: str):
        super().__init__(capi.E_INVALID, message)


class DatasetError(GapaCudaError):  # error.hpp:26-29
    def __init__(self, message: str):
        super().__init__(capi.E_INVALID, message)


class ParseError(GapaCudaError):  # error.hpp:14-19
    def __init__(self, message: str):
        super().__init__(capi.E_INVALID, message)


# ---------------------------------------------------------------------------- file loaders
@dataclass
class LoadResult:  # graph.hpp:48-52
    graph: Graph
    self_loops_dropped: int = 0
    duplicates_dropped: int = 0


def _data_lines(text: str):
    for line_no, line in enumerate(text.split("\n"), 1):
        body = line.lstrip(" \t\r")
        if not body or body[0] in "#%":
            continue
        yield line_no, line.split()


def load_edge_list(text: str) -> LoadResult:
    """graph.cpp:65-118: two whitespace-separated labels per line, '#' / '%' comments, labels interned
    in order of first appearance, self-loops and repeated edges dropped and counted."""
    ids: dict[str, int] = {}
    edges, seen = [], set()
    loops = dups = 0
    for line_no, tokens in _data_lines(text):
        if len(tokens) != 2:
            raise ParseError(f"edge list line {line_no}: expected exactly 2 tokens")
        u = ids.setdefault(tokens[0], len(ids))
        v = ids.setdefault(tokens[1], len(ids))
        if u == v:
            loops += 1
            continue
        key = (min(u, v), max(u, v))
        if key in seen:
            dups += 1
            continue
        seen.add(key)
        edges.append(key)
    g = Graph(len(ids), np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    g.labels = list(ids)
    return LoadResult(g, loops, dups)


def load_edge_list_file(path: str) -> LoadResult:
    try:
        with open(path) as f:
            return load_edge_list(f.read())
    except OSError:
        raise DatasetError("cannot open edge list file: " + path) from None


def load_community_file(path: str, g: Graph) -> np.ndarray:
    """graph.cpp:126-156: `label community` per line; every node must be assigned."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise DatasetError("cannot open community file: " + path) from None
    labels = getattr(g, "labels", None) or [str(i) for i in range(g.n)]
    index = {label: i for i, label in enumerate(labels)}
    assignment = [-1] * g.n
    communities: dict[str, int] = {}
    for line_no, tokens in _data_lines(text):
        if len(tokens) != 2:
            raise ParseError(f"community file line {line_no}: expected exactly 2 tokens")
        node = index.get(tokens[0], -1)
        if node < 0:
            raise DatasetError(f"community file line {line_no}: unknown node label '{tokens[0]}'")
        assignment[node] = communities.setdefault(tokens[1], len(communities))
    for i, a in enumerate(assignment):
        if a < 0:
            raise DatasetError(f"community file: node '{labels[i]}' has no assignment")
    return np.asarray(assignment, dtype=np.int32)


# ---------------------------------------------------------------------------- reporting-only metrics (host, as in the reference)
def _normalized(assignment) -> list[int]:  # community.cpp:17-26
    remap: dict[int, int] = {}
    return [remap.setdefault(int(a), len(remap)) for a in assignment]


def nmi(a, b) -> float:
    """community.cpp:119-148, same operation order (FP64, natural log, joint cells in (i, j) order)."""
    if len(a) != len(b):
        raise GapaCudaError(capi.E_INVALID, "nmi: partitions cover different node sets")
    n = len(a)
    if n == 0:
        raise GapaCudaError(capi.E_INVALID, "nmi: empty partitions")
    pa, pb = _normalized(a), _normalized(b)
    count_a, count_b = [0.0] * (max(pa) + 1), [0.0] * (max(pb) + 1)
    joint: dict[tuple[int, int], float] = {}
    for x, y in zip(pa, pb):
        count_a[x] += 1.0
        count_b[y] += 1.0
        joint[(x, y)] = joint.get((x, y), 0.0) + 1.0
    dn = float(n)
    h_a = h_b = mutual = 0.0
    for c in count_a:
        if c > 0:
            h_a -= (c / dn) * math.log(c / dn)
    for c in count_b:
        if c > 0:
            h_b -= (c / dn) * math.log(c / dn)
    for (i, j) in sorted(joint):
        nij = joint[(i, j)]
        mutual += (nij / dn) * math.log(nij * dn / (count_a[i] * count_b[j]))
    if h_a + h_b == 0.0:
        return 1.0 if pa == pb else 0.0
    return 2.0 * mutual / (h_a + h_b)


def precision_at_test_count(test_scores, probe_scores, test_pairs, probe_pairs) -> float:
    """link_prediction.cpp:98-117: rank every scored candidate by (score descending, pair ascending) and
    count the test edges among the top |test|."""
    t, p = np.asarray(test_scores, dtype=np.float64), np.asarray(probe_scores, dtype=np.float64)
    scores = np.concatenate([t, p])
    pairs = np.concatenate([np.asarray(test_pairs, dtype=np.int64).reshape(-1, 2),
                            np.asarray(probe_pairs, dtype=np.int64).reshape(-1, 2)])
    is_test = np.concatenate([np.ones(len(t), dtype=bool), np.zeros(len(p), dtype=bool)])
    order = np.lexsort((pairs[:, 1], pairs[:, 0], -scores))
    top = len(t)
    return float(int(is_test[order[:top]].sum())) / float(top)


# ---------------------------------------------------------------------------- config
class Task(enum.Enum):  # bench.hpp:13, names bench.cpp:22-39
    CndSixDst = "cnd-sixdst"
    CndPc = "cnd-pc"
    CdaModularity = "cda-modularity"
    LpaSimilarity = "lpa-similarity"


def task_from_string(name: str) -> Task:
    for t in Task:
        if t.value == name:
            return t
    raise ConfigError("unknown task: " + name)


_POOL_NAMES = {PoolKind.EdgeRemoval: "edge-removal", PoolKind.EdgeAddition: "edge-addition",
               PoolKind.NodeRemoval: "node-removal"}  # gene_pool.cpp:10-25
MODES = ("serial", "s", "sm", "m", "mnm")  # modes.cpp:452-470


def pool_kind_from_string(name: str) -> PoolKind:
    for kind, text in _POOL_NAMES.items():
        if text == name:
            return kind
    raise ConfigError("unknown pool kind: " + name)


@dataclass
class ModeTopology:  # modes.hpp:30-37
    mode: str = "s"
    pn: int = 1
    qn: int = 1
    max_workers: int | None = None

    def validate(self) -> None:  # modes.cpp:472-477
        if self.pn < 1 or self.qn < 1:
            raise ConfigError("worker counts must be >= 1")
        if self.mode in ("serial", "s") and (self.pn != 1 or self.qn != 1):
            raise ConfigError("serial and s modes fix pn = qn = 1")
        if self.max_workers is not None and self.max_workers < 1:
            raise ConfigError("max_workers must be >= 1")


@dataclass
class ExperimentConfig:  # bench.hpp:21-37
    task: Task = Task.CdaModularity
    dataset: str = ""
    algorithm: str = ""
    pool_kind: PoolKind = PoolKind.EdgeRemoval
    params: GAParams = field(default_factory=lambda: GAParams(pc=0.8, pm=0.1, pop_size=100, budget=1, iterations=100,
                                                              seed=1))
    perturbation_rate: float = 0.1
    topology: ModeTopology = field(default_factory=ModeTopology)
    repetitions: int = 1
    output: str = ""
    test_fraction: float = 0.1
    ground_truth: str = ""
    fast_closure: bool = False
    device: int = 0

    def validate(self) -> None:  # bench.cpp:41-66
        if not self.dataset:
            raise ConfigError("config: dataset path is required")
        if self.repetitions < 1:
            raise ConfigError("config: repetitions must be >= 1")
        if self.test_fraction <= 0.0 or self.test_fraction > 0.5:
            raise ConfigError("config: test_fraction must be in (0, 0.5]")
        if self.perturbation_rate <= 0.0 or self.perturbation_rate > 1.0:
            raise ConfigError("config: perturbation_rate must be in (0, 1]")
        try:
            self.params.validate()
        except GapaCudaError as e:
            raise ConfigError(str(e)) from None
        if self.params.iterations < 1:
            raise ConfigError("config: iterations must be >= 1")
        self.topology.validate()
        if self.task in (Task.CndSixDst, Task.CndPc) and self.pool_kind != PoolKind.NodeRemoval:
            raise ConfigError("config: cnd-* tasks require a node-removal pool")
        if self.task == Task.CdaModularity and self.pool_kind == PoolKind.NodeRemoval:
            raise ConfigError("config: cda-modularity requires an edge-removal or edge-addition pool")
        if self.task == Task.LpaSimilarity and self.pool_kind != PoolKind.EdgeRemoval:
            raise ConfigError("config: lpa-similarity requires an edge-removal pool")


_PRESETS = {  # bench.cpp:68-128: task, pool, pc, pm, iterations, pop_size, eda_interval
    "qattack": (Task.CdaModularity, PoolKind.EdgeAddition, 0.8, 0.1, 1500, 100, None),
    "cda-eda": (Task.CdaModularity, PoolKind.EdgeAddition, 0.6, 0.2, 1500, 100, None),
    "sixdst": (Task.CndSixDst, PoolKind.NodeRemoval, 0.5, 0.3, 5000, 80, None),
    "cutoff-pc": (Task.CndPc, PoolKind.NodeRemoval, 0.6, 0.2, 5000, 80, None),
    "lpa-ga": (Task.LpaSimilarity, PoolKind.EdgeRemoval, 0.7, 0.1, 500, 50, None),
    "lpa-eda": (Task.LpaSimilarity, PoolKind.EdgeRemoval, 0.0, 0.1, 500, 50, 1),
}


def preset(algorithm: str) -> ExperimentConfig:
    if algorithm not in _PRESETS:
        raise ConfigError("unknown algorithm preset: " + algorithm)
    task, pool, pc, pm, iters, pop, eda = _PRESETS[algorithm]
    cfg = ExperimentConfig(task=task, algorithm=algorithm, pool_kind=pool, perturbation_rate=0.1)
    cfg.params = GAParams(pc=pc, pm=pm, pop_size=pop, budget=1, iterations=iters, seed=1, eda_interval=eda)
    return cfg


_KNOWN_KEYS = ("task", "dataset", "algorithm", "pool", "pc", "pm", "pop_size", "iterations", "seed", "eda_interval",
               "perturbation_rate", "mode", "pn", "qn", "max_workers", "repetitions", "output", "test_fraction",
               "ground_truth", "fast_closure")
_DEFAULT_POOL = {Task.CndSixDst: PoolKind.NodeRemoval, Task.CndPc: PoolKind.NodeRemoval,
                 Task.CdaModularity: PoolKind.EdgeAddition, Task.LpaSimilarity: PoolKind.EdgeRemoval}


def parse_config(json_text: str) -> ExperimentConfig:
    """bench.cpp:142-204: unknown keys are errors; `algorithm` loads a preset that explicit keys override."""
    try:
        doc = json.loads(json_text)
    except ValueError as e:
        raise ConfigError(f"config: invalid JSON: {e}") from None
    if not isinstance(doc, dict):
        raise ConfigError("config: expected a JSON object")
    for key in doc:
        if key not in _KNOWN_KEYS:
            raise ConfigError(f"config: unknown key '{key}'")
    if "algorithm" in doc:
        cfg = preset(_typed(doc, "algorithm", str))
    elif "task" in doc:
        cfg = ExperimentConfig()
    else:
        raise ConfigError("config: either 'algorithm' or 'task' is required")
    if "task" in doc:
        cfg.task = task_from_string(_typed(doc, "task", str))
    if "dataset" in doc:
        cfg.dataset = _typed(doc, "dataset", str)
    if "pool" in doc:
        cfg.pool_kind = pool_kind_from_string(_typed(doc, "pool", str))
    elif "algorithm" not in doc:
        cfg.pool_kind = _DEFAULT_POOL[cfg.task]
    p = cfg.params
    for key, kind in (("pc", float), ("pm", float), ("pop_size", int), ("iterations", int), ("seed", int),
                      ("eda_interval", int)):
        if key in doc:
            setattr(p, key, _typed(doc, key, kind))
    if "perturbation_rate" in doc:
        cfg.perturbation_rate = _typed(doc, "perturbation_rate", float)
    if "mode" in doc:
        mode = _typed(doc, "mode", str)
        if mode not in MODES:
            raise ConfigError("unknown mode: " + mode)
        cfg.topology.mode = mode
    for key in ("pn", "qn", "max_workers"):
        if key in doc:
            setattr(cfg.topology, key, _typed(doc, key, int))
    if "repetitions" in doc:
        cfg.repetitions = _typed(doc, "repetitions", int)
    for key in ("output", "ground_truth"):
        if key in doc:
            setattr(cfg, key, _typed(doc, key, str))
    if "test_fraction" in doc:
        cfg.test_fraction = _typed(doc, "test_fraction", float)
    if "fast_closure" in doc:
        cfg.fast_closure = _typed(doc, "fast_closure", bool)
    # GAParams.validate wants a budget; the real one is derived from the dataset in run_once
    p.budget = max(p.budget, 1)
    cfg.validate()
    return cfg


def _typed(doc, key, kind):
    v = doc[key]
    if kind is float and isinstance(v, (int, float)) and not isinstance(v, bool):
        return float(v)
    if kind is int and isinstance(v, int) and not isinstance(v, bool):
        return v
    if kind in (str, bool) and isinstance(v, kind):
        return v
    raise ConfigError(f"config: key '{key}' has the wrong type")


def load_config_file(path: str) -> ExperimentConfig:
    try:
        with open(path) as f:
            return parse_config(f.read())
    except OSError:
        raise ConfigError("cannot open config file: " + path) from None


# ---------------------------------------------------------------------------- rows + report
HEADER = ("task", "algorithm", "dataset", "mode", "pn", "qn", "pop_size", "iterations", "seed", "wall_time_s",
          "q_unattacked", "q_attacked", "nmi_unattacked", "nmi_attacked", "mcn_unattacked", "mcn_attacked",
          "pc_unattacked", "pc_attacked", "auc_unattacked", "auc_attacked", "precision_unattacked",
          "precision_attacked")  # bench.cpp:371-375
_WALL_COLUMN = 9
_METRICS = HEADER[10:]


@dataclass
class ResultRow:  # bench.hpp:49-68
    task: str = ""
    algorithm: str = ""
    dataset: str = ""
    mode: str = ""
    pn: int = 1
    qn: int = 1
    pop_size: int = 0
    iterations: int = 0
    seed: int = 0
    wall_time_s: float = 0.0
    q_unattacked: float | None = None
    q_attacked: float | None = None
    nmi_unattacked: float | None = None
    nmi_attacked: float | None = None
    mcn_unattacked: float | None = None
    mcn_attacked: float | None = None
    pc_unattacked: float | None = None
    pc_attacked: float | None = None
    auc_unattacked: float | None = None
    auc_attacked: float | None = None
    precision_unattacked: float | None = None
    precision_attacked: float | None = None


def format_double(v: float) -> str:
    """std::to_chars(double) (bench.cpp:378-382): the shortest digits that round-trip, written in fixed or
    scientific notation, whichever is shorter (fixed on a tie)."""
    v = float(v)
    if v != v:
        return "nan"
    if v in (math.inf, -math.inf):
        return "inf" if v > 0 else "-inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    _, digit_tuple, exponent = Decimal(repr(abs(v))).as_tuple()
    digits = "".join(map(str, digit_tuple)).lstrip("0")
    stripped = digits.rstrip("0")
    exponent += len(digits) - len(stripped)
    digits, nd = stripped, len(stripped)
    if exponent > 0:
        # an integer beyond the shortest digits: libstdc++ chooses the notation by the shortest length but
        # then writes the exact integer value, not the zero-padded shortest digits
        fixed = str(int(abs(v)))
    elif exponent == 0:
        fixed = digits
    elif -exponent < nd:
        fixed = digits[:nd + exponent] + "." + digits[nd + exponent:]
    else:
        fixed = "0." + "0" * (-exponent - nd) + digits
    sci_e = exponent + nd - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("+" if sci_e >= 0 else "-") + "%02d" % abs(sci_e)
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _cells(r: ResultRow) -> list[str]:
    return [r.task, r.algorithm, r.dataset, r.mode, str(r.pn), str(r.qn), str(r.pop_size), str(r.iterations),
            str(r.seed), format_double(r.wall_time_s)] + \
           ["" if getattr(r, m) is None else format_double(getattr(r, m)) for m in _METRICS]


def report(rows: list[ResultRow], fmt: str = "csv") -> str:
    """bench.cpp:440-466: "csv", or "table" (columns padded to the widest cell, two spaces between)."""
    table = [list(HEADER)] + [_cells(r) for r in rows]
    if fmt == "csv":
        return "".join(",".join(cells) + "\n" for cells in table)
    if fmt != "table":
        raise ConfigError("unknown report format: " + fmt)
    widths = [max(len(cells[c]) for cells in table) for c in range(len(HEADER))]
    return "".join("  ".join(cells[c] + " " * (widths[c] - len(cells[c])) for c in range(len(HEADER))) + "\n"
                   for cells in table)


def _number(cell: str, line_no: int) -> float:
    try:
        if not cell or cell != cell.strip():
            raise ValueError
        return float(cell)
    except ValueError:
        raise ParseError(f"rows CSV line {line_no}: bad number '{cell}'") from None


def parse_rows_csv(text: str) -> list[ResultRow]:  # bench.cpp:468-517
    lines = text.split("\n")
    if not text:
        raise ParseError("rows CSV: empty input")
    head = lines[0].rstrip("\r").split(",")
    if len(head) != len(HEADER):
        raise ParseError("rows CSV: wrong column count in header")
    for got, want in zip(head, HEADER):
        if got != want:
            raise ParseError(f"rows CSV: unexpected header column '{got}'")
    rows = []
    for line_no, line in enumerate(lines[1:], 2):
        line = line.rstrip("\r")
        if not line:
            continue
        cells = line.split(",")
        if len(cells) != len(HEADER):
            raise ParseError(f"rows CSV line {line_no}: wrong column count")
        r = ResultRow(cells[0], cells[1], cells[2], cells[3], int(_number(cells[4], line_no)), int(_number(cells[5], line_no)),
                      int(_number(cells[6], line_no)), int(_number(cells[7], line_no)), int(_number(cells[8], line_no)),
                      _number(cells[9], line_no))
        for m, cell in zip(_METRICS, cells[10:]):
            setattr(r, m, None if cell == "" else _number(cell, line_no))
        rows.append(r)
    return rows


def csv_without_wall_time(csv_text: str) -> str:  # bench.cpp:519-535
    out, header = [], True
    lines = csv_text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for line in lines:
        cells = line.rstrip("\r").split(",")
        if not header and len(cells) > _WALL_COLUMN:
            cells[_WALL_COLUMN] = ""
        header = False
        out.append(",".join(cells) + "\n")
    return "".join(out)


# ---------------------------------------------------------------------------- run
def _base_row(cfg: ExperimentConfig, params: GAParams) -> ResultRow:  # bench.cpp:219-231
    return ResultRow(task=cfg.task.value, algorithm=cfg.algorithm or "custom", dataset=cfg.dataset, mode=cfg.topology.mode,
                     pn=cfg.topology.pn, qn=cfg.topology.qn, pop_size=params.pop_size, iterations=params.iterations,
                     seed=params.seed)


def _detect(dgraph: DeviceGraph, genes) -> np.ndarray:
    g = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1)
    out = np.zeros(dgraph.n, dtype=np.int32)
    check(dgraph.lib.gapa_cuda_detect_communities(dgraph.handle, g.ctypes.data_as(C.c_void_p) if g.size else None, g.size,
                                                  out.ctypes.data_as(C.c_void_p), None))
    return out


def _lp_metrics(obj: LinkPredictionAttackObjective, split, genes) -> tuple[float, float]:
    d = obj.dgraph
    g = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1)
    t, p = np.zeros(len(split.test_edges)), np.zeros(max(len(split.probe_nonedges), 1))
    auc = C.c_double(0.0)
    check(d.lib.gapa_cuda_lpa_scores(d.handle, g.ctypes.data_as(C.c_void_p) if g.size else None, g.size,
                                     t.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p), C.byref(auc)))
    p = p[:len(split.probe_nonedges)]
    return auc.value, precision_at_test_count(t, p, split.test_edges, split.probe_nonedges)


def run_once(cfg: ExperimentConfig, graph: Graph, seed: int) -> ResultRow:
    """bench.cpp:233-311.  The GA runs HBM-resident through gapa_cuda_run; every topology of the reference
    gives the same trajectory (its own cross-mode determinism contract), so `mode`/`pn`/`qn` only label
    the row."""
    params = replace(cfg.params, seed=seed, direction=Direction.Minimize)
    if cfg.task in (Task.CndSixDst, Task.CndPc):
        pool = build_gene_pool(graph, cfg.pool_kind)
        params.budget = perturbation_budget(graph, cfg.pool_kind, cfg.perturbation_rate)
        if cfg.task == Task.CndSixDst:
            obj = SixDstObjective(graph, pool, cfg.device,
                                  ClosurePolicy.SixDegrees if cfg.fast_closure else ClosurePolicy.Exact)
        else:
            obj = PairwiseConnectivityObjective(graph, pool, cfg.device)
        result = run_ga(params, pool, obj)
        row = _base_row(cfg, params)
        # component_metrics (bench.cpp:213-217) are the exact MCN / PC whatever closure the GA optimised
        best = np.ascontiguousarray(result.best_individual, dtype=np.int32).reshape(1, -1)
        empty = np.zeros((1, 0), dtype=np.int32)
        row.mcn_unattacked = float(obj.dgraph.eval_batch(TASK_MCN, empty)[0])
        row.pc_unattacked = float(obj.dgraph.eval_batch(TASK_PC, empty)[0])
        row.mcn_attacked = float(obj.dgraph.eval_batch(TASK_MCN, best)[0])
        row.pc_attacked = float(obj.dgraph.eval_batch(TASK_PC, best)[0])
    elif cfg.task == Task.CdaModularity:
        pool = build_gene_pool(graph, cfg.pool_kind)
        params.budget = perturbation_budget(graph, cfg.pool_kind, cfg.perturbation_rate)
        obj = ModularityAttackObjective(graph, pool, cfg.device)
        result = run_ga(params, pool, obj)
        row = _base_row(cfg, params)
        if graph.edge_count() == 0:
            raise GapaCudaError(capi.E_INVALID, "modularity: graph has no edges")  # community.cpp:97
        row.q_unattacked = obj.evaluate_one([])
        row.q_attacked = obj.evaluate_one(result.best_individual)  # -0.5 if nothing is left (bench.cpp:282)
        before, after = _detect(obj.dgraph, []), _detect(obj.dgraph, result.best_individual)
        reference = load_community_file(cfg.ground_truth, graph) if cfg.ground_truth else before
        row.nmi_unattacked = nmi(before, reference)
        row.nmi_attacked = nmi(after, reference)
    else:
        split = build_lp_split(graph, cfg.test_fraction, seed)
        pool = build_gene_pool(split.train, PoolKind.EdgeRemoval)
        params.budget = perturbation_budget(split.train, PoolKind.EdgeRemoval, cfg.perturbation_rate)
        obj = LinkPredictionAttackObjective(split, pool, cfg.device)
        result = run_ga(params, pool, obj)
        row = _base_row(cfg, params)
        row.auc_unattacked, row.precision_unattacked = _lp_metrics(obj, split, [])
        row.auc_attacked, row.precision_attacked = _lp_metrics(obj, split, result.best_individual)
    row.wall_time_s = result.total_wall_seconds
    obj.dgraph.close()
    return row


def run_experiment(cfg: ExperimentConfig) -> list[ResultRow]:  # bench.cpp:315-333
    cfg.validate()
    graph = load_edge_list_file(cfg.dataset).graph
    if cfg.ground_truth:
        load_community_file(cfg.ground_truth, graph)  # fail early
    rows = [run_once(cfg, graph, cfg.params.seed + rep) for rep in range(cfg.repetitions)]
    if cfg.output:
        _write(cfg.output, report(rows, "csv"))
    return rows


def sweep(cfg: ExperimentConfig, axis: str, values: list[int]) -> list[ResultRow]:  # bench.cpp:341-366
    if axis not in ("pop_size", "pn"):
        raise ConfigError("unknown sweep axis: " + axis)
    if not values:
        raise ConfigError("sweep: values must be nonempty")
    if any(b <= a for a, b in zip(values, values[1:])):
        raise ConfigError("sweep: values must be strictly ascending")
    rows: list[ResultRow] = []
    for value in values:
        one = replace(cfg, output="", params=replace(cfg.params), topology=replace(cfg.topology))
        if axis == "pop_size":
            one.params.pop_size = value
        else:
            one.topology.pn = value
        rows += run_experiment(one)
    if cfg.output:
        _write(cfg.output, report(rows, "csv"))
    return rows


def _write(path: str, text: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise ConfigError("cannot open output file: " + path) from None


def main(argv=None) -> int:
    """`python -m paper_2412_20980_b200.experiment run|sweep|report ...` — tools/gapa_main.cpp on the GPU path
    (exit codes 0 / 2 config / 3 dataset, gapa_main.cpp:13-15)."""
    import argparse
    import sys
    ap = argparse.ArgumentParser(prog="gapa", description="GA benchmark runner for graph perturbation tasks (B200 path)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run_p = sub.add_parser("run")
    run_p.add_argument("config")
    sweep_p = sub.add_parser("sweep")
    sweep_p.add_argument("config")
    sweep_p.add_argument("--axis", required=True)
    sweep_p.add_argument("--values", required=True)
    rep_p = sub.add_parser("report")
    rep_p.add_argument("rows")
    rep_p.add_argument("--format", default="table")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "report":
            with open(a.rows) as f:
                sys.stdout.write(report(parse_rows_csv(f.read()), a.format))
            return 0
        cfg = load_config_file(a.config)
        if a.cmd == "run":
            rows = run_experiment(cfg)
        else:
            try:
                values = [int(t) for t in a.values.split(",")]
            except ValueError:
                raise ConfigError("invalid sweep value: '" + a.values + "'") from None
            rows = sweep(cfg, a.axis, values)
        sys.stdout.write(report(rows, "table"))
        if cfg.output:
            sys.stdout.write("rows written to " + cfg.output + "\n")
        return 0
    except DatasetError as e:
        sys.stderr.write(f"dataset error: {e}\n")
        return 3
    except ParseError as e:
        sys.stderr.write(f"parse error: {e}\n")
        return 3
    except ConfigError as e:
        sys.stderr.write(f"config error: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    raise SystemExit(main())
