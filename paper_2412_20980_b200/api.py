"""Host-side mirror of the reference operator API for the CUDA hot path.

Same names, argument meaning and error behaviour as the reference headers
(`/root/reference/proj/include/gapa/*.hpp`): `Graph`, `GenePool`, `build_gene_pool`,
`perturbation_budget`, `LinkPredictionSplit`, `build_lp_split`, `FitnessFunction` and its
four objectives, the `ga_ops` free functions, `GAParams`, `run_ga`.  Every compute call
goes through the C ABI of include/gapa_cuda.h (paper_2412_20980_b200/capi.py); numpy
arrays are the host buffers.  The C++ twin of this file is host/gapa_cuda_objectives.hpp.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import GapaCudaError, check

TASK_PC, TASK_MCN, TASK_CDA, TASK_LPA, TASK_SIXDST = 0, 1, 2, 3, 4


class Direction(enum.Enum):  # population.hpp:9
    Maximize = 0
    Minimize = 1


class ClosurePolicy(enum.Enum):  # accessibility.hpp:14
    Exact = 0
    SixDegrees = 1


class PoolKind(enum.IntEnum):  # gene_pool.hpp:14
    EdgeRemoval = 0
    EdgeAddition = 1
    NodeRemoval = 2
    EdgeFlip = 3  # NOT in the reference (north_star's "edge flips"; parity unpinned — include/gapa_cuda.h)


class LinkScore(enum.IntEnum):
    RA = 0  # link_prediction.cpp:55-69
    CN = 1  # common neighbours: NOT in the reference (north_star's "CN/RA link scores"; parity unpinned)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i32(a, ndim=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.int32)
    if ndim is not None and out.ndim != ndim:
        raise GapaCudaError(capi.E_INVALID, "shape mismatch")
    return out


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _minimize(direction: Direction) -> int:
    return 1 if direction == Direction.Minimize else 0


# ---------------------------------------------------------------------------- graph
class Graph:
    """graph.hpp:15-46 — undirected, unweighted, dense ids; canonical (u < v) edges in
    insertion order.  Validation (loops, range, duplicates) happens in the C ABI when a
    device context is created from it."""

    def __init__(self, n: int, edges):
        e = _i32(edges).reshape(-1, 2).copy()
        swap = e[:, 0] > e[:, 1]
        e[swap] = e[swap][:, ::-1]
        self.n = int(n)
        self._edges = e

    def node_count(self) -> int:
        return self.n

    def edge_count(self) -> int:
        return len(self._edges)

    def edges(self) -> np.ndarray:
        return self._edges

    def degrees(self) -> np.ndarray:
        return np.bincount(self._edges.reshape(-1), minlength=self.n).astype(np.int32)

    def sorted_edges(self) -> np.ndarray:
        """(u, v)-sorted edges == the EdgeRemoval pool order (gene_pool.cpp:73-79)."""
        e = self._edges
        return e[np.lexsort((e[:, 1], e[:, 0]))]


def _generate(fn, *args) -> np.ndarray:
    m = C.c_int64(0)
    check(fn(*args, None, 0, C.byref(m)))
    uv = np.zeros((max(m.value, 1), 2), dtype=np.int32)
    check(fn(*args, _ptr(uv), m.value, C.byref(m)))
    return uv[:m.value]


def barabasi_albert(n: int, attach: int, seed: int) -> Graph:  # generators.hpp:14
    return Graph(n, _generate(capi.load().gapa_host_barabasi_albert, n, attach, seed))


def erdos_renyi(n: int, p: float, seed: int) -> Graph:  # generators.hpp:10
    return Graph(n, _generate(capi.load().gapa_host_erdos_renyi, n, p, seed))


def planted_partition(blocks: int, block_size: int, p_in: float, p_out: float, seed: int) -> Graph:
    return Graph(blocks * block_size,
                 _generate(capi.load().gapa_host_planted_partition, blocks, block_size, p_in, p_out, seed))


# ---------------------------------------------------------------------------- gene pool
class GenePool:
    """gene_pool.hpp:32-52.  `u`, `v` hold the element of every gene id (v = -1 for nodes)."""

    def __init__(self, kind: PoolKind, u, v=None, graph: Graph | None = None, canonical: bool = False, count: int | None = None):
        self._kind = PoolKind(kind)
        self.u = _i32(u, 1)
        self.v = np.full_like(self.u, -1) if v is None else _i32(v, 1)
        self.graph = graph
        self.canonical = canonical  # exactly build_gene_pool(graph, kind): the device side rebuilds it itself
        self._count = count         # canonical pools that are never enumerated on the host (all node pairs of EdgeFlip)

    def gene(self, gene_id: int) -> tuple[int, int]:
        return int(self.u[gene_id]), int(self.v[gene_id])

    def kind(self) -> PoolKind:
        return self._kind

    def size(self) -> int:
        return len(self.u) if self._count is None else self._count


def build_gene_pool(g: Graph, kind: PoolKind) -> GenePool:  # gene_pool.cpp:69-96
    if g.node_count() == 0:
        raise GapaCudaError(capi.E_INVALID, "gene pool: graph is empty")
    kind = PoolKind(kind)
    if kind == PoolKind.NodeRemoval:
        return GenePool(kind, np.arange(g.n, dtype=np.int32), graph=g)
    if kind == PoolKind.EdgeRemoval:
        e = g.sorted_edges()
        return GenePool(kind, e[:, 0], e[:, 1], graph=g)
    if kind == PoolKind.EdgeFlip:  # every node pair a < b, lexicographic; genes are unranked on the device
        if g.n > 65536:
            raise GapaCudaError(capi.E_INVALID, "gene pool: node pairs do not fit int32 gene ids")
        return GenePool(kind, np.zeros(0, np.int32), np.zeros(0, np.int32), graph=g, canonical=True, count=g.n * (g.n - 1) // 2)
    e = np.ascontiguousarray(g.edges())
    count = C.c_int64(0)
    lib = capi.load()
    check(lib.gapa_host_nonedges(g.n, len(e), _ptr(e) if len(e) else None, None, 0, C.byref(count)))
    uv = np.zeros((count.value, 2), dtype=np.int32)
    check(lib.gapa_host_nonedges(g.n, len(e), _ptr(e) if len(e) else None, _ptr(uv), count.value, C.byref(count)))
    return GenePool(kind, uv[:, 0], uv[:, 1], graph=g, canonical=True)


def perturbation_budget(g: Graph, kind: PoolKind, rate: float) -> int:  # gene_pool.cpp:98-102
    k = C.c_int32(0)
    basis = g.node_count() if PoolKind(kind) == PoolKind.NodeRemoval else g.edge_count()
    check(capi.load().gapa_host_budget(basis, rate, C.byref(k)))
    return k.value


# ---------------------------------------------------------------------------- lp split
@dataclass
class LinkPredictionSplit:  # link_prediction.hpp:16-21
    train: Graph
    test_edges: np.ndarray
    probe_nonedges: np.ndarray
    seed: int = 0


def build_lp_split(g: Graph, test_fraction: float, seed: int) -> LinkPredictionSplit:
    lib = capi.load()
    T = C.c_int32(0)
    e = np.ascontiguousarray(g.edges())
    check(lib.gapa_host_lp_split(g.n, g.edge_count(), _ptr(e), test_fraction, seed, None, None, None, C.byref(T)))
    train = np.zeros((g.edge_count() - T.value, 2), dtype=np.int32)
    test = np.zeros((T.value, 2), dtype=np.int32)
    probe = np.zeros((T.value, 2), dtype=np.int32)
    check(lib.gapa_host_lp_split(g.n, g.edge_count(), _ptr(e), test_fraction, seed, _ptr(train), _ptr(test),
                                 _ptr(probe), C.byref(T)))
    return LinkPredictionSplit(Graph(g.n, train), test, probe, seed)


# ---------------------------------------------------------------------------- device context
class DeviceGraph:
    """Owns a gapa_cuda_ctx: the shared read-only CSR (+ pool, + split) on one GPU."""

    def __init__(self, g: Graph, device: int = 0):
        self.lib = capi.load()
        self.handle = C.c_void_p()
        self.device = device
        e = np.ascontiguousarray(g.edges())
        check(self.lib.gapa_cuda_graph_create(g.n, g.edge_count(), _ptr(e) if len(e) else None, device,
                                              C.byref(self.handle)))
        self.n, self.m = g.n, g.edge_count()

    def set_pool(self, pool: GenePool) -> None:
        if pool.canonical and pool.kind() in (PoolKind.EdgeAddition, PoolKind.EdgeFlip):  # 12.5 M pairs at n = 5000: built on the C side
            check(self.lib.gapa_cuda_pool_set(self.handle, int(pool.kind()), pool.size(), None, None))
        elif pool.kind() == PoolKind.NodeRemoval:
            check(self.lib.gapa_cuda_pool_set(self.handle, int(pool.kind()), pool.size(), _ptr(pool.u), None))
        else:
            check(self.lib.gapa_cuda_pool_set(self.handle, int(pool.kind()), pool.size(), _ptr(pool.u), _ptr(pool.v)))

    def set_split(self, split: LinkPredictionSplit) -> None:
        t, p = _i32(split.test_edges), _i32(split.probe_nonedges)
        check(self.lib.gapa_cuda_lp_split_set(self.handle, len(t), _ptr(t), len(p), _ptr(p) if len(p) else None))

    def eval_batch(self, task: int, batch) -> np.ndarray:
        b = _i32(batch, 2)
        out = np.zeros(b.shape[0], dtype=np.float64)
        check(self.lib.gapa_cuda_eval_batch(self.handle, task, _ptr(b) if b.size else None, b.shape[0], b.shape[1],
                                            _ptr(out) if len(out) else None))
        return out

    def eval_batch_device(self, task: int, genes_ptr: int, rows: int, cols: int, out_ptr: int, stream: int = 0):
        check(self.lib.gapa_cuda_eval_batch_device(self.handle, task, genes_ptr, rows, cols, out_ptr, stream))

    def last_eval_ms(self) -> float:
        ms = C.c_float(0)
        check(self.lib.gapa_cuda_last_eval_ms(self.handle, C.byref(ms)))
        return ms.value

    def close(self) -> None:
        if self.handle:
            self.lib.gapa_cuda_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------- fitness
class FitnessFunction:
    """fitness.hpp:17-27.  evaluate_batch is the CUDA path; evaluate_one is a 1-row batch
    ("overriding is an optimization, never a semantic change")."""

    task: int = -1

    def __init__(self, dgraph: DeviceGraph, pool: GenePool):
        self.dgraph, self.pool = dgraph, pool

    def direction(self) -> Direction:
        return Direction.Minimize

    def evaluate_one(self, genes) -> float:
        return float(self.evaluate_batch(_i32(genes, 1).reshape(1, -1))[0])

    def evaluate_batch(self, batch) -> np.ndarray:
        return self.dgraph.eval_batch(self.task, batch)


def _require_kind(pool: GenePool, kind: PoolKind, what: str) -> None:  # fitness.cpp:50-57
    if pool.kind() != kind:
        raise GapaCudaError(capi.E_INVALID, f"{what}: incompatible gene pool kind")


class PairwiseConnectivityObjective(FitnessFunction):  # fitness.hpp:68-77
    task = TASK_PC

    def __init__(self, graph: Graph, pool: GenePool, device: int = 0):
        _require_kind(pool, PoolKind.NodeRemoval, "PairwiseConnectivityObjective")
        super().__init__(DeviceGraph(graph, device), pool)
        self.dgraph.set_pool(pool)


class SixDstObjective(FitnessFunction):  # fitness.hpp:56-66
    """Exact closure = largest component (the PC kernels); SixDegrees = largest radius-8 ball
    (accessibility.hpp:12-14, the truncated multi-source BFS kernel)."""
    task = TASK_MCN

    def __init__(self, graph: Graph, pool: GenePool, device: int = 0, policy: ClosurePolicy = ClosurePolicy.Exact):
        _require_kind(pool, PoolKind.NodeRemoval, "SixDstObjective")
        super().__init__(DeviceGraph(graph, device), pool)
        self.policy = ClosurePolicy(policy)
        self.task = TASK_MCN if self.policy == ClosurePolicy.Exact else TASK_SIXDST
        self.dgraph.set_pool(pool)


class ModularityAttackObjective(FitnessFunction):  # fitness.hpp:79-88
    task = TASK_CDA

    def __init__(self, graph: Graph, pool: GenePool, device: int = 0):
        if pool.kind() in (PoolKind.NodeRemoval, PoolKind.EdgeFlip):
            raise GapaCudaError(capi.E_INVALID, "ModularityAttackObjective: incompatible gene pool kind")
        super().__init__(DeviceGraph(graph, device), pool)
        self.dgraph.set_pool(pool)


class LinkPredictionAttackObjective(FitnessFunction):  # fitness.hpp:90-101
    task = TASK_LPA

    def __init__(self, split: LinkPredictionSplit, pool: GenePool, device: int = 0, score: LinkScore = LinkScore.RA):
        if pool.kind() != PoolKind.EdgeFlip:  # the reference takes edge-removal pools only (fitness.cpp:87)
            _require_kind(pool, PoolKind.EdgeRemoval, "LinkPredictionAttackObjective")
        super().__init__(DeviceGraph(split.train, device), pool)
        self.dgraph.set_pool(pool)
        self.dgraph.set_split(split)
        check(self.dgraph.lib.gapa_cuda_lp_score_set(self.dgraph.handle, int(LinkScore(score))))


def pc_fitness(graph: Graph, batch, pool: GenePool, device: int = 0) -> np.ndarray:  # fitness.hpp:38-39
    _require_kind(pool, PoolKind.NodeRemoval, "pc_fitness")
    return PairwiseConnectivityObjective(graph, pool, device).evaluate_batch(batch)


def sixdst_fitness(graph: Graph, batch, pool: GenePool, policy: ClosurePolicy = ClosurePolicy.Exact,
                   device: int = 0) -> np.ndarray:  # fitness.hpp:33-36
    _require_kind(pool, PoolKind.NodeRemoval, "sixdst_fitness")
    return SixDstObjective(graph, pool, device, policy).evaluate_batch(batch)


def cda_fitness(graph: Graph, batch, pool: GenePool, device: int = 0) -> np.ndarray:  # fitness.hpp:44-45
    if pool.kind() == PoolKind.NodeRemoval:
        raise GapaCudaError(capi.E_INVALID, "cda_fitness: incompatible gene pool kind")
    return ModularityAttackObjective(graph, pool, device).evaluate_batch(batch)


def lpa_fitness(split: LinkPredictionSplit, batch, pool: GenePool, device: int = 0) -> np.ndarray:
    _require_kind(pool, PoolKind.EdgeRemoval, "lpa_fitness")
    return LinkPredictionAttackObjective(split, pool, device).evaluate_batch(batch)


# ---------------------------------------------------------------------------- ga_ops
@dataclass
class GAParams:  # ga_ops.hpp:12-23
    pc: float = 0.8
    pm: float = 0.1
    pop_size: int = 100
    budget: int = 1
    iterations: int = 100
    direction: Direction = Direction.Minimize
    eda_interval: int | None = None
    seed: int = 1

    def validate(self) -> None:  # ga_ops.cpp:11-17
        if self.pop_size < 2:
            raise GapaCudaError(capi.E_INVALID, "pop_size must be >= 2")
        if self.budget < 1:
            raise GapaCudaError(capi.E_INVALID, "budget must be >= 1")
        if not 0.0 <= self.pc <= 1.0:
            raise GapaCudaError(capi.E_INVALID, "pc must be in [0, 1]")
        if not 0.0 <= self.pm <= 1.0:
            raise GapaCudaError(capi.E_INVALID, "pm must be in [0, 1]")
        if self.eda_interval is not None and self.eda_interval < 1:
            raise GapaCudaError(capi.E_INVALID, "eda_interval must be >= 1")


def init_population_block(pool_size, row_first, row_count, budget, seed, generation=0, device=0) -> np.ndarray:
    out = np.zeros((row_count, budget), dtype=np.int32)
    check(capi.load().gapa_cuda_ga_init(device, pool_size, row_first, row_count, budget, seed, generation,
                                        _ptr(out) if out.size else None))
    return out


def init_population(pool_size, pop_size, budget, seed, generation=0, device=0) -> np.ndarray:
    return init_population_block(pool_size, 0, pop_size, budget, seed, generation, device)


def make_crossover_mask(rows, cols, pc, seed, generation, device=0) -> np.ndarray:  # ga_ops.cpp:84-87
    out = np.zeros((rows, cols), dtype=np.uint8)
    check(capi.load().gapa_cuda_ga_mask(device, 3, pc, rows, cols, seed, generation, _ptr(out)))
    return out


def make_mutation_mask(rows, cols, pm, seed, generation, device=0) -> np.ndarray:  # ga_ops.cpp:89-92
    out = np.zeros((rows, cols), dtype=np.uint8)
    check(capi.load().gapa_cuda_ga_mask(device, 4, pm, rows, cols, seed, generation, _ptr(out)))
    return out


def make_mutation_indices(rows, cols, pool_size, seed, generation, device=0) -> np.ndarray:  # ga_ops.cpp:94-103
    out = np.zeros((rows, cols), dtype=np.int32)
    check(capi.load().gapa_cuda_ga_mutation_indices(device, pool_size, rows, cols, seed, generation, _ptr(out)))
    return out


def selection_weights(fitness, direction: Direction, device=0) -> np.ndarray:  # ga_ops.cpp:54-76
    f = _f64(fitness)
    out = np.zeros_like(f)
    check(capi.load().gapa_cuda_ga_selection_weights(device, _ptr(f), len(f), _minimize(direction), _ptr(out)))
    return out


def roulette_pick(fitness, direction: Direction, seed, generation, device=0) -> np.ndarray:
    """Index form of roulette_select: partner row per row."""
    f = _f64(fitness)
    out = np.zeros(len(f), dtype=np.int32)
    check(capi.load().gapa_cuda_ga_select(device, _ptr(f), len(f), _minimize(direction), seed, generation, _ptr(out)))
    return out


def roulette_select(pop, fitness, direction: Direction, seed, generation, device=0) -> np.ndarray:
    p = _i32(pop, 2)
    if len(_f64(fitness)) != p.shape[0]:  # ga_ops.cpp:109
        raise GapaCudaError(capi.E_INVALID, "roulette_select: fitness length mismatch")
    return p[roulette_pick(fitness, direction, seed, generation, device)]


def crossover_mutate(pop, partner_index, pc, pm, pool_size, seed, generation, row_first=0, row_count=None,
                     device=0) -> np.ndarray:
    p = _i32(pop, 2)
    idx = _i32(partner_index, 1)
    s, k = p.shape
    if len(idx) != s:
        raise GapaCudaError(capi.E_INVALID, "crossover: shape mismatch")
    rc = s - row_first if row_count is None else row_count
    out = np.zeros((rc, k), dtype=np.int32)
    check(capi.load().gapa_cuda_ga_crossover_mutate(device, _ptr(p), _ptr(idx), s, k, row_first, rc, pc, pm, pool_size,
                                                    seed, generation, _ptr(out) if out.size else None))
    return out


def crossover(pop, partners, pc, seed, generation, device=0) -> np.ndarray:  # ga_ops.cpp:130-144
    p, q = _i32(pop, 2), _i32(partners, 2)
    if p.shape != q.shape:
        raise GapaCudaError(capi.E_INVALID, "crossover: shape mismatch")
    s = p.shape[0]
    stacked = np.concatenate([p, q], axis=0)  # partner of row i is stacked row s + i
    idx = np.concatenate([np.arange(s, 2 * s), np.arange(s, 2 * s)]).astype(np.int32)
    return crossover_mutate(stacked, idx, pc, 0.0, 1, seed, generation, 0, s, device)


def mutate_block(block, row_offset, pm, pool_size, seed, generation, device=0) -> np.ndarray:
    b = _i32(block, 2)
    out = np.zeros_like(b)
    check(capi.load().gapa_cuda_ga_mutate(device, _ptr(b) if b.size else None, b.shape[0], b.shape[1], row_offset, pm,
                                          pool_size, seed, generation, _ptr(out) if out.size else None))
    return out


def mutate(c_pop, pm, pool_size, seed, generation, device=0) -> np.ndarray:  # ga_ops.cpp:146-162
    return mutate_block(c_pop, 0, pm, pool_size, seed, generation, device)


def elitism(pop, m_pop, fit_pop, fit_m, direction: Direction, device=0):  # ga_ops.cpp:180-212
    p, q = _i32(pop, 2), _i32(m_pop, 2)
    if p.shape != q.shape:
        raise GapaCudaError(capi.E_INVALID, "elitism: shape mismatch")
    f, fm = _f64(fit_pop), _f64(fit_m)
    if len(f) != p.shape[0] or len(fm) != p.shape[0]:
        raise GapaCudaError(capi.E_INVALID, "elitism: fitness length mismatch")
    nxt, nf = np.zeros_like(p), np.zeros(p.shape[0], dtype=np.float64)
    check(capi.load().gapa_cuda_ga_elitism(device, _ptr(p), _ptr(q), p.shape[0], p.shape[1], _ptr(f), _ptr(fm),
                                           _minimize(direction), _ptr(nxt), _ptr(nf)))
    return nxt, nf


def eda_sample(elite, elite_count, pool_size, seed, generation, add_one_smoothing=True, device=0) -> np.ndarray:
    e = _i32(elite, 2)
    out = np.zeros_like(e)
    check(capi.load().gapa_cuda_ga_eda(device, _ptr(e), e.shape[0], e.shape[1], elite_count, pool_size, seed,
                                       generation, int(add_one_smoothing), _ptr(out)))
    return out


def rng_draws(seed, generation, role, row, count, device=0) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    check(capi.load().gapa_cuda_rng_draws(device, seed, generation, role, row, count, _ptr(out)))
    return out


def partition_rows(pop_size: int, pn: int) -> list[tuple[int, int]]:  # modes.cpp:506-516
    block = (pop_size + pn - 1) // pn
    out = []
    for w in range(pn):
        lo = min(w * block, pop_size)
        out.append((lo, min(lo + block, pop_size)))
    return out


# ---------------------------------------------------------------------------- run
@dataclass
class GenerationStats:  # modes.hpp:63-71
    best: float = 0.0
    mean: float = 0.0
    wall_seconds: float = 0.0
    compute_seconds: float = 0.0
    exchange_seconds: float = 0.0
    lifecycle_seconds: float = 0.0
    messages: int = 0


@dataclass
class RunResult:  # modes.hpp:73-82
    final_population: np.ndarray
    final_fitness: np.ndarray
    best_individual: np.ndarray
    best_fitness: float
    history_best: np.ndarray
    history_mean: np.ndarray
    fitness_batch_calls: int = 0
    total_wall_seconds: float = 0.0
    eval_seconds: float = 0.0
    history: list = field(default_factory=list)  # one GenerationStats per generation
    extra: dict = field(default_factory=dict)


def overhead_report(result: RunResult) -> str:
    """modes.cpp:518-530: aligned per-generation table of {wall, compute, exchange, lifecycle, messages},
    byte-compatible with the reference's format."""
    lines = ["gen  wall_s      compute_s   exchange_s  lifecycle_s messages\n"]
    for g, h in enumerate(result.history):
        lines.append("%-4d %-11.6f %-11.6f %-11.6f %-11.6f %d\n" % (g + 1, h.wall_seconds, h.compute_seconds,
                                                                  h.exchange_seconds, h.lifecycle_seconds, h.messages))
    return "".join(lines)


class _ResultBuffers:
    """host arrays behind a gapa_cuda_run_result"""

    def __init__(self, params: GAParams, outputs: bool = True):
        s, k, it = params.pop_size, params.budget, params.iterations
        self.it = it
        self.hb, self.hm = np.zeros(it), np.zeros(it)
        self.fp, self.ff = np.zeros((s, k), dtype=np.int32), np.zeros(s)
        self.wall, self.comp, self.exch, self.life = (np.zeros(it) for _ in range(4))
        self.msgs = np.zeros(it, dtype=np.uint64)
        null_f, null_i = C.cast(None, capi.c_f64p), C.cast(None, capi.c_i32p)
        if outputs:
            self.c = capi.RunResult(self.hb.ctypes.data_as(capi.c_f64p), self.hm.ctypes.data_as(capi.c_f64p),
                                    self.fp.ctypes.data_as(capi.c_i32p), self.ff.ctypes.data_as(capi.c_f64p), 0, 0.0, 0.0,
                                    self.wall.ctypes.data_as(capi.c_f64p), self.comp.ctypes.data_as(capi.c_f64p),
                                    self.exch.ctypes.data_as(capi.c_f64p), self.life.ctypes.data_as(capi.c_f64p),
                                    self.msgs.ctypes.data_as(C.POINTER(C.c_uint64)))
        else:
            self.c = capi.RunResult(null_f, null_f, null_i, null_f, 0, 0.0, 0.0, null_f, null_f, null_f, null_f,
                                    C.cast(None, C.POINTER(C.c_uint64)))

    def result(self) -> "RunResult":
        history = [GenerationStats(float(self.hb[i]), float(self.hm[i]), float(self.wall[i]), float(self.comp[i]),
                                   float(self.exch[i]), float(self.life[i]), int(self.msgs[i])) for i in range(self.it)]
        return RunResult(self.fp, self.ff, self.fp[0].copy(), float(self.ff[0]), self.hb, self.hm,
                         int(self.c.fitness_batch_calls), float(self.c.total_wall_seconds), float(self.c.eval_seconds), history)


def _run_params(params: GAParams, fitness: FitnessFunction, rank: int, world: int) -> "capi.RunParams":
    params.validate()
    if params.iterations < 1:  # modes.cpp:26-29
        raise GapaCudaError(capi.E_INVALID, "iterations must be >= 1")
    return capi.RunParams(params.pc, params.pm, params.pop_size, params.budget, params.iterations, _minimize(params.direction),
                          params.eda_interval or 0, fitness.task, params.seed, rank, world)


def _exchange_args(exchange, comm):
    """(hook, user) for the C ABI: a Python callable, or the library's own exchange with a Comm"""
    if comm is not None:
        return C.cast(capi.load().gapa_cuda_comm_allgather, capi.ALLGATHER_FN), comm.handle
    if exchange is not None:
        return capi.ALLGATHER_FN(exchange), None
    return C.cast(None, capi.ALLGATHER_FN), None


def run_ga(params: GAParams, pool: GenePool, fitness: FitnessFunction, rank: int = 0, world: int = 1,
           exchange=None, comm=None) -> RunResult:
    """run_ga for Mode::S (modes.cpp:132-178) on one GPU, or one rank of a sharded run (exchange: a Python hook, or
    comm: a driver.Comm — the library's own peer-mailbox / NCCL exchange)."""
    p = _run_params(params, fitness, rank, world)
    buf = _ResultBuffers(params)
    cb, user = _exchange_args(exchange, comm)
    check(capi.load().gapa_cuda_run(fitness.dgraph.handle, C.byref(p), cb, user, C.byref(buf.c)))
    return buf.result()


def run_ga_multi(params: GAParams, fitnesses, transport: str = "peer") -> list:
    """run_mode_m on GPUs from ONE process (gapa_cuda_run_multi): fitnesses[r] is rank r's objective (its own context,
    normally on its own GPU); returns every rank's RunResult — identical by the determinism contract."""
    world = len(fitnesses)
    p = _run_params(params, fitnesses[0], 0, world)
    bufs = [_ResultBuffers(params) for _ in range(world)]
    ctxs = (capi.VP * world)(*[f.dgraph.handle for f in fitnesses])
    results = (capi.RunResult * world)(*[b.c for b in bufs])
    check(capi.load().gapa_cuda_run_multi(ctxs, world, C.byref(p), {"peer": 0, "nccl": 1}[transport], results))
    for b, r in zip(bufs, results):
        b.c = r
    return [b.result() for b in bufs]


class GaLoop:
    """The in-library generation loop as a resumable object (gapa_cuda_ga_*): the population stays in HBM between
    advance() calls."""

    def __init__(self, params: GAParams, fitness: FitnessFunction, rank: int = 0, world: int = 1, exchange=None, comm=None,
                 want_stats: bool = False):
        self.params, self.fitness = params, fitness
        p = _run_params(params, fitness, rank, world)
        self._cb, user = _exchange_args(exchange, comm)  # keep the callback object alive
        self._comm = comm
        self.handle = capi.VP()
        check(capi.load().gapa_cuda_ga_create(fitness.dgraph.handle, C.byref(p), self._cb, user, 1 if want_stats else 0,
                                              C.byref(self.handle)))

    def advance(self, generations: int) -> float:
        """runs the next `generations` generations; returns their device time in ms (CUDA events on the run's stream)"""
        ms = C.c_float(0.0)
        check(capi.load().gapa_cuda_ga_advance(self.handle, generations, C.byref(ms)))
        return float(ms.value)

    @property
    def generation(self) -> int:
        g = C.c_int(0)
        check(capi.load().gapa_cuda_ga_generation(self.handle, C.byref(g)))
        return g.value

    def result(self) -> RunResult:
        buf = _ResultBuffers(self.params)
        check(capi.load().gapa_cuda_ga_result(self.handle, C.byref(buf.c)))
        return buf.result()

    def counters(self) -> tuple:
        """(fitness_batch_calls, eval_seconds, total_wall_seconds) so far, without copying any population"""
        buf = _ResultBuffers(self.params, outputs=False)
        check(capi.load().gapa_cuda_ga_result(self.handle, C.byref(buf.c)))
        return int(buf.c.fitness_batch_calls), float(buf.c.eval_seconds), float(buf.c.total_wall_seconds)

    def close(self):
        if self.handle:
            capi.load().gapa_cuda_ga_destroy(self.handle)
            self.handle = capi.VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
