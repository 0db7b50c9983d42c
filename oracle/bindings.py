"""TEST INFRASTRUCTURE — ctypes bindings for the parity checkers.

``Oracle``  wraps oracle/libgapa_oracle.so (plain-C CSR restatement).
``Ref``     wraps oracle/_ref/libgapa_ref.so (the unmodified reference compiled
            from /root/reference/proj by oracle/Makefile; built in the authoring
            container, travels to the GPU box as a binary).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libgapa_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgapa_ref.so")
REFERENCE_SRC = "/root/reference/proj"

TASK_PC, TASK_MCN, TASK_CDA, TASK_LPA = 0, 1, 2, 3
TASK_SIXDST, TASK_CDA_ADD = 4, 5  # sixdst_fitness(SixDegrees); cda_fitness over the EdgeAddition pool
ROLE_INIT, ROLE_SELECT, ROLE_CROSSOVER_MASK, ROLE_MUTATION_MASK, ROLE_MUTATION_INDEX = 1, 2, 3, 4, 5
MODE_SERIAL, MODE_S, MODE_SM, MODE_M, MODE_MNM = 0, 1, 2, 3, 4

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
            os.path.join(HERE, "gapa_oracle.c")):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    return ORACLE_SO


def build_ref() -> str | None:
    """Compile the reference where it lies; None where /root/reference is absent
    and no prebuilt binary travelled with the snapshot."""
    if os.path.isdir(REFERENCE_SRC):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref", "-j8"])
    return REF_SO if os.path.exists(REF_SO) else None


def _genes(genes) -> np.ndarray:
    a = np.ascontiguousarray(genes, dtype=np.int32)
    if a.ndim != 2:
        raise ValueError("genes must be a rows x cols matrix")
    return a


class OrcGraphStruct(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int64), ("edge_uv", C.POINTER(C.c_int32)),
                ("row_ptr", C.POINTER(C.c_int32)), ("col_idx", C.POINTER(C.c_int32)),
                ("edge_id", C.POINTER(C.c_int32)), ("pool_u", C.POINTER(C.c_int32)),
                ("pool_v", C.POINTER(C.c_int32)), ("add_size", C.c_int64), ("add_u", C.POINTER(C.c_int32)),
                ("add_v", C.POINTER(C.c_int32))]


class OrcSplitStruct(C.Structure):
    _fields_ = [("train", C.POINTER(OrcGraphStruct)), ("T", C.c_int32), ("P", C.c_int32),
                ("test_uv", C.POINTER(C.c_int32)), ("probe_uv", C.POINTER(C.c_int32))]


class OracleGraph:
    """Owns an ``orc_graph*``; exposes numpy copies of its arrays."""

    def __init__(self, lib, ptr, owned=True):
        if not ptr:
            raise ValueError("oracle: graph construction failed")
        self._lib, self._ptr, self._owned = lib, ptr, owned
        s = ptr.contents
        self.n, self.m = int(s.n), int(s.m)
        arr = lambda p, k: np.ctypeslib.as_array(p, shape=(max(k, 1),))[:k].copy()
        self.edges = arr(s.edge_uv, 2 * self.m).reshape(-1, 2)
        self.row_ptr = arr(s.row_ptr, self.n + 1)
        self.col_idx = arr(s.col_idx, 2 * self.m)
        self.edge_id = arr(s.edge_id, 2 * self.m)
        self.pool_u = arr(s.pool_u, self.m)
        self.pool_v = arr(s.pool_v, self.m)

    def __del__(self):
        if getattr(self, "_owned", False) and self._ptr:
            self._lib.orc_graph_free(self._ptr)
            self._ptr = None


class OracleSplit:
    def __init__(self, lib, ptr):
        if not ptr:
            raise ValueError("oracle: split construction failed")
        self._lib, self._ptr = lib, ptr
        s = ptr.contents
        self.T, self.P = int(s.T), int(s.P)
        self.test = np.ctypeslib.as_array(s.test_uv, shape=(2 * self.T,)).copy().reshape(-1, 2)
        self.probe = np.ctypeslib.as_array(s.probe_uv, shape=(2 * self.P,)).copy().reshape(-1, 2)
        self.train = OracleGraph(lib, s.train, owned=False)
        self.train._keepalive = self

    def __del__(self):
        if self._ptr:
            self._lib.orc_split_free(self._ptr)
            self._ptr = None


class Oracle:
    def __init__(self):
        lib = C.CDLL(build_oracle())
        self.lib = lib
        G, S = C.POINTER(OrcGraphStruct), C.POINTER(OrcSplitStruct)
        lib.orc_mix64.restype = C.c_uint64
        lib.orc_mix64.argtypes = [C.c_uint64]
        lib.orc_stream_key.restype = C.c_uint64
        lib.orc_stream_key.argtypes = [C.c_uint64] * 4
        lib.orc_draw_u64.restype = C.c_uint64
        lib.orc_draw_u64.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_draw_unit.restype = C.c_double
        lib.orc_draw_unit.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_draw_index.restype = C.c_uint32
        lib.orc_draw_index.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
        lib.orc_graph_create.restype = G
        lib.orc_graph_create.argtypes = [C.c_int32, C.c_int64, _i32p]
        lib.orc_graph_ba.restype = G
        lib.orc_graph_ba.argtypes = [C.c_int32, C.c_int32, C.c_uint64]
        lib.orc_graph_er.restype = G
        lib.orc_graph_er.argtypes = [C.c_int32, C.c_double, C.c_uint64]
        lib.orc_graph_sbm.restype = G
        lib.orc_graph_sbm.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64]
        lib.orc_graph_free.argtypes = [G]
        lib.orc_graph_build_addition_pool.restype = C.c_int64
        lib.orc_graph_build_addition_pool.argtypes = [G]
        lib.orc_budget.restype = C.c_int32
        lib.orc_budget.argtypes = [C.c_int64, C.c_double]
        lib.orc_split_build.restype = S
        lib.orc_split_build.argtypes = [G, C.c_double, C.c_uint64]
        lib.orc_split_free.argtypes = [S]
        lib.orc_eval_batch.argtypes = [C.c_void_p, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, _f64p]
        lib.orc_detect_communities.argtypes = [G, _i32p]
        lib.orc_ra_score.restype = C.c_double
        lib.orc_ra_score.argtypes = [G, C.c_int32, C.c_int32]
        lib.orc_init_population_block.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_uint64, _i32p]
        lib.orc_lpa_flip_batch.argtypes = [S, C.c_int, C.c_void_p, C.c_int64, _i32p, C.c_int, C.c_int, _f64p]
        lib.orc_lpa_scored_batch.argtypes = [S, C.c_int, _i32p, C.c_int, C.c_int, _f64p]
        lib.orc_flip_unrank.restype = None
        lib.orc_flip_unrank.argtypes = [C.c_int32, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.orc_make_mask.restype = None
        lib.orc_make_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_uint64, _u8p]
        lib.orc_make_mutation_indices.restype = None
        lib.orc_make_mutation_indices.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _i32p]
        lib.orc_selection_weights.argtypes = [_f64p, C.c_int, C.c_int, _f64p]
        lib.orc_roulette_pick.argtypes = [_f64p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _i32p]
        lib.orc_crossover.argtypes = [_i32p, _i32p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64, _i32p]
        lib.orc_mutate_block.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                         C.c_uint64, _i32p]
        lib.orc_elitism.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _f64p, _f64p, C.c_int, _i32p, _f64p]
        lib.orc_eda_sample.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                       _i32p]
        lib.orc_partition_rows.argtypes = [C.c_int, C.c_int, _i32p]
        lib.orc_run_ga.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_uint64, C.c_int, C.c_int, _f64p, _f64p, _i32p, _f64p]

    # -- rng
    def mix64(self, x):
        return int(self.lib.orc_mix64(x))

    def stream_key(self, seed, generation, role, row):
        return int(self.lib.orc_stream_key(seed, generation, role, row))

    def stream_u64(self, seed, generation, role, row, count):
        key = self.stream_key(seed, generation, role, row)
        return np.array([self.lib.orc_draw_u64(key, j + 1) for j in range(count)], dtype=np.uint64)

    def stream_unit(self, seed, generation, role, row, count):
        key = self.stream_key(seed, generation, role, row)
        return np.array([self.lib.orc_draw_unit(key, j + 1) for j in range(count)], dtype=np.float64)

    def stream_index(self, seed, generation, role, row, bound, count):
        key = self.stream_key(seed, generation, role, row)
        return np.array([self.lib.orc_draw_index(key, j + 1, bound) for j in range(count)], dtype=np.uint32)

    # -- graphs
    def graph_from_edges(self, n, edges):
        e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
        return OracleGraph(self.lib, self.lib.orc_graph_create(n, len(e), e.reshape(-1) if len(e) else np.zeros(1, np.int32)))

    def graph_ba(self, n, attach, seed):
        return OracleGraph(self.lib, self.lib.orc_graph_ba(n, attach, seed))

    def graph_er(self, n, p, seed):
        return OracleGraph(self.lib, self.lib.orc_graph_er(n, p, seed))

    def graph_sbm(self, blocks, block_size, p_in, p_out, seed):
        return OracleGraph(self.lib, self.lib.orc_graph_sbm(blocks, block_size, p_in, p_out, seed))

    def budget(self, basis, rate):
        return int(self.lib.orc_budget(basis, rate))

    def addition_pool(self, g: OracleGraph):
        """EdgeAddition pool (gene_pool.cpp:81-87) of g as (u[], v[]); cached on the graph,
        and what TASK_CDA_ADD evaluates against."""
        size = int(self.lib.orc_graph_build_addition_pool(g._ptr))
        if size < 0:
            raise ValueError("gene pool: graph is complete, no edges can be added")
        s = g._ptr.contents
        return (np.ctypeslib.as_array(s.add_u, shape=(size,)).copy(),
                np.ctypeslib.as_array(s.add_v, shape=(size,)).copy())

    def split_build(self, g: OracleGraph, fraction, seed):
        return OracleSplit(self.lib, self.lib.orc_split_build(g._ptr, fraction, seed))

    # -- fitness
    def eval_batch(self, ctx, task, genes, threads=1):
        g = _genes(genes)
        out = np.zeros(max(g.shape[0], 1), dtype=np.float64)
        ptr = C.cast(ctx._ptr, C.c_void_p)
        rc = self.lib.orc_eval_batch(ptr, task, g if g.size else np.zeros(1, np.int32), g.shape[0], g.shape[1],
                                     threads, out)
        if rc:
            raise ValueError("oracle: gene id out of range")
        return out[:g.shape[0]]

    # PARITY UNPINNED: CN score / edge-flip pools have no reference implementation (oracle/gapa_oracle.c states the semantics)
    def lpa_flip_batch(self, split, genes, score=0, pool_uv=None):
        g = _genes(genes)
        out = np.zeros(max(g.shape[0], 1), dtype=np.float64)
        if pool_uv is None:
            ptr, size = None, 0
        else:
            pool_uv = np.ascontiguousarray(pool_uv, dtype=np.int32).reshape(-1, 2)
            ptr, size = pool_uv.ctypes.data_as(C.c_void_p), len(pool_uv)
        if self.lib.orc_lpa_flip_batch(split._ptr, score, ptr, size, g if g.size else np.zeros(1, np.int32), g.shape[0], g.shape[1], out):
            raise ValueError("oracle: gene id out of range")
        return out[:g.shape[0]]

    def lpa_scored_batch(self, split, genes, score=0):
        g = _genes(genes)
        out = np.zeros(max(g.shape[0], 1), dtype=np.float64)
        if self.lib.orc_lpa_scored_batch(split._ptr, score, g if g.size else np.zeros(1, np.int32), g.shape[0], g.shape[1], out):
            raise ValueError("oracle: gene id out of range")
        return out[:g.shape[0]]

    def flip_unrank(self, n, gene_id):
        a, b = C.c_int32(0), C.c_int32(0)
        self.lib.orc_flip_unrank(n, gene_id, C.byref(a), C.byref(b))
        return a.value, b.value

    def detect_communities(self, g):
        out = np.zeros(max(g.n, 1), dtype=np.int32)
        self.lib.orc_detect_communities(g._ptr, out)
        return out[:g.n]

    def ra_score(self, g, u, v):
        return float(self.lib.orc_ra_score(g._ptr, u, v))

    # -- operators
    def init_population_block(self, pool_size, row_first, row_count, budget, seed, generation=0):
        out = np.zeros((row_count, budget), dtype=np.int32)
        if self.lib.orc_init_population_block(pool_size, row_first, row_count, budget, seed, generation,
                                              out.reshape(-1) if out.size else np.zeros(1, np.int32)):
            raise ValueError("init_population: empty gene pool")
        return out

    def init_population(self, pool_size, pop_size, budget, seed, generation=0):
        return self.init_population_block(pool_size, 0, pop_size, budget, seed, generation)

    def make_mask(self, rows, cols, rate, role, seed, generation):
        """role 3 = make_crossover_mask, 4 = make_mutation_mask (ga_ops.cpp:84-92)"""
        out = np.zeros((rows, cols), dtype=np.uint8)
        self.lib.orc_make_mask(rows, cols, rate, role, seed, generation, out.reshape(-1) if out.size else np.zeros(1, np.uint8))
        return out

    def make_mutation_indices(self, rows, cols, pool_size, seed, generation):
        out = np.zeros((rows, cols), dtype=np.int32)
        self.lib.orc_make_mutation_indices(rows, cols, pool_size, seed, generation, out.reshape(-1) if out.size else np.zeros(1, np.int32))
        return out

    def selection_weights(self, fitness, minimize=True):
        f = np.ascontiguousarray(fitness, dtype=np.float64)
        out = np.zeros_like(f)
        if self.lib.orc_selection_weights(f, len(f), int(minimize), out):
            raise ValueError("selection: non-finite fitness")
        return out

    def roulette_pick(self, fitness, minimize, seed, generation):
        f = np.ascontiguousarray(fitness, dtype=np.float64)
        out = np.zeros(len(f), dtype=np.int32)
        if self.lib.orc_roulette_pick(f, len(f), int(minimize), seed, generation, out):
            raise ValueError("roulette_select: non-finite fitness")
        return out

    def crossover(self, pop, partner_index, pc, seed, generation):
        p = _genes(pop)
        out = np.zeros_like(p)
        self.lib.orc_crossover(p.reshape(-1), np.ascontiguousarray(partner_index, dtype=np.int32), p.shape[0],
                               p.shape[1], pc, seed, generation, out.reshape(-1))
        return out

    def mutate_block(self, block, row_offset, pm, pool_size, seed, generation):
        b = _genes(block)
        out = np.zeros_like(b)
        self.lib.orc_mutate_block(b.reshape(-1), b.shape[0], b.shape[1], row_offset, pm, pool_size, seed, generation,
                                  out.reshape(-1))
        return out

    def elitism(self, pop, m_pop, fit, fit_m, minimize=True):
        p, q = _genes(pop), _genes(m_pop)
        nxt, nf = np.zeros_like(p), np.zeros(p.shape[0], dtype=np.float64)
        if self.lib.orc_elitism(p.reshape(-1), q.reshape(-1), p.shape[0], p.shape[1],
                                np.ascontiguousarray(fit, dtype=np.float64),
                                np.ascontiguousarray(fit_m, dtype=np.float64), int(minimize), nxt.reshape(-1), nf):
            raise ValueError("elitism: NaN fitness")
        return nxt, nf

    def eda_sample(self, elite, elite_count, pool_size, seed, generation, smoothing=True):
        e = _genes(elite)
        out = np.zeros_like(e)
        if self.lib.orc_eda_sample(e.reshape(-1), e.shape[0], e.shape[1], elite_count, pool_size, seed, generation,
                                   int(smoothing), out.reshape(-1)):
            raise ValueError("eda_sample: invalid elite count")
        return out

    def partition_rows(self, pop_size, pn):
        out = np.zeros(2 * pn, dtype=np.int32)
        self.lib.orc_partition_rows(pop_size, pn, out)
        return [tuple(int(x) for x in out[2 * w:2 * w + 2]) for w in range(pn)]

    def run_ga(self, ctx, task, pc, pm, pop_size, budget, iterations, seed, eda_interval=0, minimize=True,
               threads=1):
        hb, hm = np.zeros(iterations), np.zeros(iterations)
        fp, ff = np.zeros((pop_size, budget), dtype=np.int32), np.zeros(pop_size)
        rc = self.lib.orc_run_ga(C.cast(ctx._ptr, C.c_void_p), task, pc, pm, pop_size, budget, iterations,
                                 eda_interval, seed, int(minimize), threads, hb, hm, fp.reshape(-1), ff)
        if rc:
            raise ValueError(f"oracle run_ga failed rc={rc}")
        return {"best": hb, "mean": hm, "population": fp, "fitness": ff}


class _RefHandle:
    def __init__(self, lib, ptr, free):
        if not ptr:
            raise ValueError("reference: " + lib.ref_last_error().decode())
        self._lib, self._ptr, self._free = lib, ptr, free

    def __del__(self):
        if self._ptr:
            self._free(self._ptr)
            self._ptr = None


class Ref:
    """The compiled, unmodified reference."""

    @staticmethod
    def available() -> bool:
        return build_ref() is not None

    def __init__(self):
        path = build_ref()
        if path is None:
            raise RuntimeError("reference library not built and /root/reference absent")
        lib = C.CDLL(path)
        self.lib = lib
        V = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_mix64.restype = C.c_uint64
        lib.ref_mix64.argtypes = [C.c_uint64]
        lib.ref_stream_u64.argtypes = [C.c_uint64] * 4 + [C.c_int, _u64p]
        lib.ref_stream_unit.argtypes = [C.c_uint64] * 4 + [C.c_int, _f64p]
        lib.ref_stream_index.argtypes = [C.c_uint64] * 4 + [C.c_uint32, C.c_int, _u32p]
        for name, args in [("ref_graph_from_edges", [C.c_int, C.c_int, _i32p]),
                           ("ref_graph_ba", [C.c_int, C.c_int, C.c_uint64]),
                           ("ref_graph_er", [C.c_int, C.c_double, C.c_uint64]),
                           ("ref_graph_sbm", [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64]),
                           ("ref_graph_load", [C.c_char_p]),
                           ("ref_split_build", [V, C.c_double, C.c_uint64]),
                           ("ref_split_train", [V])]:
            getattr(lib, name).restype = V
            getattr(lib, name).argtypes = args
        lib.ref_graph_free.argtypes = [V]
        lib.ref_split_free.argtypes = [V]
        lib.ref_graph_n.argtypes = [V]
        lib.ref_graph_m.argtypes = [V]
        lib.ref_graph_edges.argtypes = [V, _i32p]
        lib.ref_pool_size.argtypes = [V, C.c_int]
        lib.ref_pool_genes.argtypes = [V, C.c_int, _i32p, _i32p]
        lib.ref_budget.argtypes = [V, C.c_int, C.c_double]
        lib.ref_split_test_count.argtypes = [V]
        lib.ref_split_probe_count.argtypes = [V]
        lib.ref_split_pairs.argtypes = [V, _i32p, _i32p]
        lib.ref_eval_batch.argtypes = [V, C.c_int, _i32p, C.c_int, C.c_int, C.c_int, _f64p]
        lib.ref_modularity_unattacked.restype = C.c_double
        lib.ref_modularity_unattacked.argtypes = [V]
        lib.ref_detect_communities.argtypes = [V, _i32p]
        lib.ref_auc_unattacked.restype = C.c_double
        lib.ref_auc_unattacked.argtypes = [V]
        lib.ref_ra_score.restype = C.c_double
        lib.ref_ra_score.argtypes = [V, C.c_int, C.c_int]
        lib.ref_init_population_block.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_uint64, _i32p]
        if hasattr(lib, "ref_make_mask"):
            lib.ref_make_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_uint64, _u8p]
            lib.ref_make_mutation_indices.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _i32p]
        lib.ref_selection_weights.argtypes = [_f64p, C.c_int, C.c_int, _f64p]
        lib.ref_roulette_select.argtypes = [_i32p, C.c_int, C.c_int, _f64p, C.c_int, C.c_uint64, C.c_uint64, _i32p,
                                            _i32p]
        lib.ref_crossover.argtypes = [_i32p, _i32p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_uint64, _i32p]
        lib.ref_mutate_block.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                         C.c_uint64, _i32p]
        lib.ref_mutate.argtypes = [_i32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_uint64, _i32p]
        lib.ref_elitism.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _f64p, _f64p, C.c_int, _i32p, _f64p]
        lib.ref_eda_sample.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                       _i32p]
        lib.ref_partition_rows.argtypes = [C.c_int, C.c_int, _i32p]
        lib.ref_nmi.restype = C.c_double
        lib.ref_nmi.argtypes = [_i32p, _i32p, C.c_int]
        lib.ref_detect_perturbed.argtypes = [V, C.c_int, _i32p, C.c_int, _i32p]
        lib.ref_lp_metrics.argtypes = [V, _i32p, C.c_int, _f64p, _f64p]
        self.have_bench = bool(lib.ref_have_bench())
        if self.have_bench:
            lib.ref_run_experiment.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.c_int, C.c_char_p, C.c_int]
            lib.ref_csv_without_wall_time.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_run_ga.argtypes = [V, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_uint64, C.c_int, C.c_int, C.c_int, _f64p, _f64p, _i32p, _f64p,
                                   C.POINTER(C.c_double)]

    def _err(self):
        return self.lib.ref_last_error().decode()

    # -- rng
    def mix64(self, x):
        return int(self.lib.ref_mix64(x))

    def stream_u64(self, seed, generation, role, row, count):
        out = np.zeros(count, dtype=np.uint64)
        self.lib.ref_stream_u64(seed, generation, role, row, count, out)
        return out

    def stream_unit(self, seed, generation, role, row, count):
        out = np.zeros(count, dtype=np.float64)
        self.lib.ref_stream_unit(seed, generation, role, row, count, out)
        return out

    def stream_index(self, seed, generation, role, row, bound, count):
        out = np.zeros(count, dtype=np.uint32)
        self.lib.ref_stream_index(seed, generation, role, row, bound, count, out)
        return out

    # -- graphs
    def _graph(self, ptr):
        return _RefHandle(self.lib, ptr, self.lib.ref_graph_free)

    def graph_from_edges(self, n, edges):
        e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
        return self._graph(self.lib.ref_graph_from_edges(n, len(e), e.reshape(-1) if len(e) else np.zeros(1, np.int32)))

    def graph_ba(self, n, attach, seed):
        return self._graph(self.lib.ref_graph_ba(n, attach, seed))

    def graph_er(self, n, p, seed):
        return self._graph(self.lib.ref_graph_er(n, p, seed))

    def graph_sbm(self, blocks, block_size, p_in, p_out, seed):
        return self._graph(self.lib.ref_graph_sbm(blocks, block_size, p_in, p_out, seed))

    def graph_load(self, path):
        return self._graph(self.lib.ref_graph_load(path.encode()))

    def graph_n(self, g):
        return int(self.lib.ref_graph_n(g._ptr))

    def graph_m(self, g):
        return int(self.lib.ref_graph_m(g._ptr))

    def graph_edges(self, g):
        m = self.graph_m(g)
        out = np.zeros(max(2 * m, 1), dtype=np.int32)
        self.lib.ref_graph_edges(g._ptr, out)
        return out[:2 * m].reshape(-1, 2)

    def pool_genes(self, g, kind):
        size = self.lib.ref_pool_size(g._ptr, kind)
        if size < 0:
            raise ValueError(self._err())
        u, v = np.zeros(size, dtype=np.int32), np.zeros(size, dtype=np.int32)
        self.lib.ref_pool_genes(g._ptr, kind, u, v)
        return u, v

    def budget(self, g, kind, rate):
        return int(self.lib.ref_budget(g._ptr, kind, rate))

    def split_build(self, g, fraction, seed):
        return _RefHandle(self.lib, self.lib.ref_split_build(g._ptr, fraction, seed), self.lib.ref_split_free)

    def split_pairs(self, s):
        T, P = self.lib.ref_split_test_count(s._ptr), self.lib.ref_split_probe_count(s._ptr)
        t, p = np.zeros(2 * T, dtype=np.int32), np.zeros(2 * P, dtype=np.int32)
        self.lib.ref_split_pairs(s._ptr, t, p)
        return t.reshape(-1, 2), p.reshape(-1, 2)

    def split_train(self, s):
        return self._graph(self.lib.ref_split_train(s._ptr))

    # -- fitness
    def eval_batch(self, ctx, task, genes, threads=1):
        g = _genes(genes)
        out = np.zeros(max(g.shape[0], 1), dtype=np.float64)
        if self.lib.ref_eval_batch(ctx._ptr, task, g.reshape(-1) if g.size else np.zeros(1, np.int32), g.shape[0],
                                   g.shape[1], threads, out):
            raise ValueError(self._err())
        return out[:g.shape[0]]

    def modularity_unattacked(self, g):
        return float(self.lib.ref_modularity_unattacked(g._ptr))

    def detect_communities(self, g):
        out = np.zeros(max(self.graph_n(g), 1), dtype=np.int32)
        self.lib.ref_detect_communities(g._ptr, out)
        return out[:self.graph_n(g)]

    def auc_unattacked(self, s):
        return float(self.lib.ref_auc_unattacked(s._ptr))

    def ra_score(self, g, u, v):
        return float(self.lib.ref_ra_score(g._ptr, u, v))

    # -- operators
    def init_population_block(self, pool_size, row_first, row_count, budget, seed, generation=0):
        out = np.zeros((row_count, budget), dtype=np.int32)
        if self.lib.ref_init_population_block(pool_size, row_first, row_count, budget, seed, generation,
                                              out.reshape(-1) if out.size else np.zeros(1, np.int32)):
            raise ValueError(self._err())
        return out

    def init_population(self, pool_size, pop_size, budget, seed, generation=0):
        return self.init_population_block(pool_size, 0, pop_size, budget, seed, generation)

    def make_mask(self, rows, cols, rate, role, seed, generation):
        out = np.zeros((rows, cols), dtype=np.uint8)
        if self.lib.ref_make_mask(rows, cols, rate, role, seed, generation, out.reshape(-1) if out.size else np.zeros(1, np.uint8)):
            raise ValueError(self._err())
        return out

    def make_mutation_indices(self, rows, cols, pool_size, seed, generation):
        out = np.zeros((rows, cols), dtype=np.int32)
        if self.lib.ref_make_mutation_indices(rows, cols, pool_size, seed, generation,
                                              out.reshape(-1) if out.size else np.zeros(1, np.int32)):
            raise ValueError(self._err())
        return out

    def selection_weights(self, fitness, minimize=True):
        f = np.ascontiguousarray(fitness, dtype=np.float64)
        out = np.zeros_like(f)
        if self.lib.ref_selection_weights(f, len(f), int(minimize), out):
            raise ValueError(self._err())
        return out

    def roulette_select(self, pop, fitness, minimize, seed, generation):
        p = _genes(pop)
        idx, partners = np.zeros(p.shape[0], dtype=np.int32), np.zeros_like(p)
        if self.lib.ref_roulette_select(p.reshape(-1), p.shape[0], p.shape[1],
                                        np.ascontiguousarray(fitness, dtype=np.float64), int(minimize), seed,
                                        generation, idx, partners.reshape(-1)):
            raise ValueError(self._err())
        return idx, partners

    def crossover(self, pop, partners, pc, seed, generation):
        p, q = _genes(pop), _genes(partners)
        out = np.zeros_like(p)
        if self.lib.ref_crossover(p.reshape(-1), q.reshape(-1), p.shape[0], p.shape[1], pc, seed, generation,
                                  out.reshape(-1)):
            raise ValueError(self._err())
        return out

    def mutate_block(self, block, row_offset, pm, pool_size, seed, generation):
        b = _genes(block)
        out = np.zeros_like(b)
        if self.lib.ref_mutate_block(b.reshape(-1), b.shape[0], b.shape[1], row_offset, pm, pool_size, seed,
                                     generation, out.reshape(-1)):
            raise ValueError(self._err())
        return out

    def mutate(self, c_pop, pm, pool_size, seed, generation):
        b = _genes(c_pop)
        out = np.zeros_like(b)
        if self.lib.ref_mutate(b.reshape(-1), b.shape[0], b.shape[1], pm, pool_size, seed, generation,
                               out.reshape(-1)):
            raise ValueError(self._err())
        return out

    def elitism(self, pop, m_pop, fit, fit_m, minimize=True):
        p, q = _genes(pop), _genes(m_pop)
        nxt, nf = np.zeros_like(p), np.zeros(p.shape[0], dtype=np.float64)
        if self.lib.ref_elitism(p.reshape(-1), q.reshape(-1), p.shape[0], p.shape[1],
                                np.ascontiguousarray(fit, dtype=np.float64),
                                np.ascontiguousarray(fit_m, dtype=np.float64), int(minimize), nxt.reshape(-1), nf):
            raise ValueError(self._err())
        return nxt, nf

    def eda_sample(self, elite, elite_count, pool_size, seed, generation, smoothing=True):
        e = _genes(elite)
        out = np.zeros_like(e)
        if self.lib.ref_eda_sample(e.reshape(-1), e.shape[0], e.shape[1], elite_count, pool_size, seed, generation,
                                   int(smoothing), out.reshape(-1)):
            raise ValueError(self._err())
        return out

    def partition_rows(self, pop_size, pn):
        out = np.zeros(2 * pn, dtype=np.int32)
        self.lib.ref_partition_rows(pop_size, pn, out)
        return [tuple(int(x) for x in out[2 * w:2 * w + 2]) for w in range(pn)]

    def run_ga(self, ctx, task, pc, pm, pop_size, budget, iterations, seed, eda_interval=0, mode=MODE_S, pn=1, qn=1):
        hb, hm = np.zeros(iterations), np.zeros(iterations)
        fp, ff = np.zeros((pop_size, budget), dtype=np.int32), np.zeros(pop_size)
        wall = C.c_double(0.0)
        if self.lib.ref_run_ga(ctx._ptr, task, pc, pm, pop_size, budget, iterations, eda_interval, seed, mode, pn, qn,
                               hb, hm, fp.reshape(-1), ff, C.byref(wall)):
            raise ValueError(self._err())
        return {"best": hb, "mean": hm, "population": fp, "fitness": ff, "wall_seconds": wall.value}

    # -- reporting metrics + experiment driver
    def nmi(self, a, b):
        a, b = np.ascontiguousarray(a, dtype=np.int32), np.ascontiguousarray(b, dtype=np.int32)
        return float(self.lib.ref_nmi(a, b, len(a)))

    def detect_perturbed(self, g, kind, genes):
        genes = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1)
        out = np.zeros(max(self.graph_n(g), 1), dtype=np.int32)
        if self.lib.ref_detect_perturbed(g._ptr, kind, genes if genes.size else np.zeros(1, np.int32), genes.size, out):
            raise ValueError(self._err())
        return out[:self.graph_n(g)]

    def lp_metrics(self, split, genes):
        """(auc, precision, scores[T + P]) of evaluate_ra_predictor on the perturbed train graph."""
        genes = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1)
        t, p = self.lib.ref_split_test_count(split._ptr), self.lib.ref_split_probe_count(split._ptr)
        out, scores = np.zeros(2), np.zeros(max(t + p, 1))
        if self.lib.ref_lp_metrics(split._ptr, genes if genes.size else np.zeros(1, np.int32), genes.size, out, scores):
            raise ValueError(self._err())
        return float(out[0]), float(out[1]), scores[:t + p]

    def run_experiment(self, config_json: str, axis: str = "", values=()):
        """bench::run_experiment (or bench::sweep when `axis` is given) -> CSV text."""
        if not self.have_bench:
            raise RuntimeError("reference library was built without bench.cpp")
        buf = C.create_string_buffer(1 << 20)
        vals = (C.c_int * max(len(values), 1))(*values)
        if self.lib.ref_run_experiment(config_json.encode(), axis.encode(), vals, len(values), buf, len(buf)):
            raise ValueError(self._err())
        return buf.value.decode()

    def csv_without_wall_time(self, text: str):
        buf = C.create_string_buffer(len(text) + 16)
        if self.lib.ref_csv_without_wall_time(text.encode(), buf, len(buf)):
            raise ValueError(self._err())
        return buf.value.decode()
