"""Sharded generation loop: one process per GPU, population rows partitioned across ranks.

Shape of the reference's M mode (modes.cpp:190-349) mapped onto GPUs:

  * the graph (CSR), pool and split are replicated on every GPU;
  * every rank keeps the WHOLE parent population in its HBM, in a pool of 2s row slots behind
    parent / child index tables (elitism permutes indices, genomes are never copied); selection and
    the elitism ranking are tiny and run redundantly — the operators are keyed by (seed, generation, role, global
    row) (rng.hpp:49-65), so every rank produces bit-identical results;
  * rank r owns rows partition_rows(s, world)[r] (modes.cpp:506-516): it builds (crossover +
    mutate, or eda_sample + mutate) and evaluates only those rows of M_POP;
  * surviving mutated rows of OTHER ranks are recomputed inside the elitism gather from the
    replicated parents and the keyed streams instead of being fetched, so genomes never cross
    NVLink;
  * ONE all-gather of fitness doubles per evaluation is the only exchange (block padded to
    ceil(s/world) so counts are equal), issued through torch.distributed (NCCL over
    NVLink/NVSwitch on GPUs).

`ShardedGa` holds the loop and the sharding arithmetic; the compute is delegated to an
`ops` object.  The product's ops is `CudaOps` (C ABI, device pointers, torch tensors only as
device-memory owners).  Tests inject a CPU ops object to exercise the N>1 host logic under
gloo without a GPU — the product never does.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import capi
from .api import Direction, FitnessFunction, GAParams, RunResult, partition_rows
from .capi import GapaCudaError, check


@dataclass
class Shard:
    rank: int
    world: int
    pop_size: int

    @property
    def block(self) -> int:  # ceil(s / world), modes.cpp:507
        return (self.pop_size + self.world - 1) // self.world

    @property
    def rows(self) -> tuple[int, int]:
        return partition_rows(self.pop_size, self.world)[self.rank]

    @property
    def padded(self) -> int:
        return self.block * self.world


class CudaOps:
    """Device ops over torch-owned HBM buffers, on torch's current stream.

    The population store is the slot pool of csrc/slot_kernels.cu: `pool` holds 2s rows, `parent` /
    `child` are the slot tables; variation writes children into their slots, evaluation reads rows
    through a table, elitism permutes the tables (no genome is copied)."""

    def __init__(self, fitness: FitnessFunction, device_index: int):
        import torch
        self.torch = torch
        self.lib = capi.load()
        self.fitness = fitness
        self.device = torch.device("cuda", device_index)
        self.pool_size = fitness.pool.size()

    def _stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def empty_genes(self, rows, cols):
        return self.torch.empty((rows, max(cols, 0)), dtype=self.torch.int32, device=self.device)

    def zeros_f64(self, count):
        return self.torch.zeros(count, dtype=self.torch.float64, device=self.device)

    def empty_i32(self, count):
        return self.torch.empty(count, dtype=self.torch.int32, device=self.device)

    def init(self, pool, parent, child, s, seed, generation):
        """parents into slots 0..s-1, tables to the identity (init_population, ga_ops.cpp:31-34)"""
        k = pool.shape[1]
        check(self.lib.gapa_cuda_ga_slots_identity_device(s, parent.data_ptr(), child.data_ptr(), self._stream()))
        check(self.lib.gapa_cuda_ga_init_device(self.pool_size, 0, s, k, seed, generation, pool.data_ptr(), self._stream()))

    def select(self, fit, s, minimize, seed, generation, partner):
        check(self.lib.gapa_cuda_ga_select_device(fit.data_ptr(), s, minimize, seed, generation, partner.data_ptr(), None,
                                                  self._stream()))

    def variation(self, pool, parent, child, partner, s, pc, pm, seed, generation, lo, hi):
        """children of rows [lo, hi) into their slots; partner None = EDA generation"""
        check(self.lib.gapa_cuda_ga_slots_variation_device(
            pool.data_ptr(), parent.data_ptr(), child.data_ptr(), partner.data_ptr() if partner is not None else None, s,
            pool.shape[1], lo, hi - lo, pc, pm, self.pool_size, seed, generation, self._stream()))

    def variation_eval(self, pool, parent, child, partner, s, pc, pm, seed, generation, lo, hi, fit_out):
        """children of rows [lo, hi) built into their slots AND evaluated into fit_out[lo:hi] in one call"""
        if hi <= lo:
            return
        check(self.lib.gapa_cuda_ga_slots_variation_eval_device(
            self.fitness.dgraph.handle, self.fitness.task, pool.data_ptr(), parent.data_ptr(), child.data_ptr(),
            partner.data_ptr() if partner is not None else None, s, pool.shape[1], lo, hi - lo, pc, pm, seed, generation,
            fit_out.data_ptr() + 8 * lo, self._stream()))

    def eval_rows(self, pool, table, lo, hi, fit_out):
        """fitness of the rows table[lo:hi] names into fit_out[lo:hi]"""
        if hi <= lo:
            return
        check(self.lib.gapa_cuda_eval_rows_device(self.fitness.dgraph.handle, self.fitness.task, pool.data_ptr(),
                                                  table.data_ptr() + 4 * lo, hi - lo, pool.shape[1],
                                                  fit_out.data_ptr() + 8 * lo, self._stream()))

    def elitism(self, pool, parent, child, partner, s, lo, hi, fit, fit_m, minimize, pc, pm, seed, generation, next_parent,
                next_child, next_fit):
        check(self.lib.gapa_cuda_ga_slots_elitism_device(
            pool.data_ptr(), parent.data_ptr(), child.data_ptr(), partner.data_ptr() if partner is not None else None, s,
            pool.shape[1], lo, hi, fit.data_ptr(), fit_m.data_ptr(), minimize, pc, pm, self.pool_size, seed, generation,
            next_parent.data_ptr(), next_child.data_ptr(), next_fit.data_ptr(), self._stream()))

    def gather(self, pool, table, rows):
        """dense [rows, k] matrix of the rows the table names"""
        out = self.empty_genes(rows, pool.shape[1])
        check(self.lib.gapa_cuda_ga_slots_gather_device(pool.data_ptr(), table.data_ptr(), rows, pool.shape[1], out.data_ptr(),
                                                        self._stream()))
        return out

    def stats(self, fit, s, hist, index, iters):
        check(self.lib.gapa_cuda_ga_stats_device(fit.data_ptr(), s, hist.data_ptr() + 8 * index,
                                                 hist.data_ptr() + 8 * (iters + index), self._stream()))

    def last_eval_ms(self) -> float:
        return self.fitness.dgraph.last_eval_ms()

    def to_host(self, t):
        return t.cpu().numpy()


class Comm:
    """The library's own exchange (include/gapa_cuda.h, gapa_cuda_comm_*): peer mailboxes over NVLink, or NCCL.

    `allgather_bytes(mine: bytes) -> list[bytes]` is any out-of-band all-gather between the ranks (torch.distributed
    all_gather_object, MPI, files): it carries the 128-byte handles once at set-up."""

    def __init__(self, handle, keep=None):
        self.handle, self._keep = handle, keep

    @classmethod
    def peer(cls, fitness: FitnessFunction, rank: int, world: int, pop_size: int, allgather_bytes) -> "Comm":
        import ctypes as C
        lib = capi.load()
        handle = C.c_void_p()
        mine = C.create_string_buffer(128)
        check(lib.gapa_cuda_comm_create(fitness.dgraph.handle, rank, world, pop_size, C.byref(handle), mine))
        everyone = allgather_bytes(mine.raw)
        if len(everyone) != world:
            raise GapaCudaError(capi.E_INVALID, "Comm.peer: the out-of-band all-gather must return one handle per rank")
        check(lib.gapa_cuda_comm_connect(handle, b"".join(everyone)))
        return cls(handle)

    @classmethod
    def nccl(cls, fitness: FitnessFunction, rank: int, world: int, broadcast_bytes) -> "Comm":
        """broadcast_bytes(data_or_None) -> bytes: rank 0 passes the unique id, everyone receives it"""
        import ctypes as C
        lib = capi.load()
        uid = C.create_string_buffer(128)
        if rank == 0:
            check(lib.gapa_cuda_nccl_unique_id(uid))
        data = broadcast_bytes(uid.raw if rank == 0 else None)
        handle = C.c_void_p()
        check(lib.gapa_cuda_comm_create_nccl(fitness.dgraph.handle, data, rank, world, C.byref(handle)))
        return cls(handle)

    def status(self):
        check(capi.load().gapa_cuda_comm_status(self.handle))

    def close(self):
        if self.handle:
            capi.load().gapa_cuda_comm_destroy(self.handle)
            self.handle = None


def torch_bytes_allgather(group=None):
    """out-of-band all-gather of small byte strings over torch.distributed (any backend)"""
    import torch.distributed as dist

    def gather(mine: bytes):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, mine, group=group)
        return out

    return gather


def torch_allgather(group=None):
    """In-place all-gather of the padded fitness vector over torch.distributed."""
    import torch.distributed as dist

    def gather(fit_padded, shard: Shard):
        if shard.world == 1:
            return
        lo = shard.rank * shard.block
        dist.all_gather_into_tensor(fit_padded, fit_padded[lo:lo + shard.block], group=group)

    return gather


class ShardedGa:
    def __init__(self, params: GAParams, ops, shard: Shard, gather):
        params.validate()
        if params.iterations < 1:
            raise GapaCudaError(capi.E_INVALID, "iterations must be >= 1")
        if shard.pop_size != params.pop_size:
            raise GapaCudaError(capi.E_INVALID, "shard does not match the population size")
        self.p, self.ops, self.shard, self.gather = params, ops, shard, gather
        s, k = params.pop_size, params.budget
        self.minimize = 1 if params.direction == Direction.Minimize else 0
        self.pool = ops.empty_genes(2 * s, k)          # 2s row slots: s parents + s children
        self.parent, self.child = ops.empty_i32(s), ops.empty_i32(s)
        self.next_parent, self.next_child = ops.empty_i32(s), ops.empty_i32(s)
        self.partner = ops.empty_i32(s)
        self.fit = ops.zeros_f64(shard.padded)
        self.fit_m = ops.zeros_f64(shard.padded)
        self.fit_next = ops.zeros_f64(shard.padded)
        self.hist = ops.zeros_f64(2 * params.iterations)
        self.generation = 0
        self.fitness_batch_calls = 0

    def _evaluate(self, table, fit):
        lo, hi = self.shard.rows
        self.fitness_batch_calls += 1
        self.ops.eval_rows(self.pool, table, lo, hi, fit)
        self.gather(fit, self.shard)

    def initialize(self):
        """gen 1 prologue: init_population with generation key 0, then evaluate (modes.cpp:162-165)"""
        self.ops.init(self.pool, self.parent, self.child, self.p.pop_size, self.p.seed, 0)
        self._evaluate(self.parent, self.fit)

    def step(self):
        """one generation: select -> crossover -> mutate -> evaluate(M_POP) -> elitism"""
        p, ops = self.p, self.ops
        self.generation += 1
        gen = self.generation
        s = p.pop_size
        lo, hi = self.shard.rows
        eda_gen = bool(p.eda_interval and gen % p.eda_interval == 0)  # modes.cpp:31-33,167-168
        partner = None if eda_gen else self.partner
        if not eda_gen:
            ops.select(self.fit, s, self.minimize, p.seed, gen, self.partner)
        self.fitness_batch_calls += 1
        ops.variation_eval(self.pool, self.parent, self.child, partner, s, p.pc, p.pm, p.seed, gen, lo, hi, self.fit_m)
        self.gather(self.fit_m, self.shard)
        ops.elitism(self.pool, self.parent, self.child, partner, s, lo, hi, self.fit, self.fit_m, self.minimize, p.pc, p.pm,
                    p.seed, gen, self.next_parent, self.next_child, self.fit_next)
        self.parent, self.next_parent = self.next_parent, self.parent
        self.child, self.next_child = self.next_child, self.child
        self.fit, self.fit_next = self.fit_next, self.fit
        if gen <= p.iterations:
            ops.stats(self.fit, s, self.hist, gen - 1, p.iterations)

    def population(self):
        """the parents as a dense best-first matrix (PopulationMatrix)"""
        return self.ops.gather(self.pool, self.parent, self.p.pop_size)

    def run(self) -> RunResult:
        self.initialize()
        for _ in range(self.p.iterations):
            self.step()
        return self.result()

    def result(self) -> RunResult:
        s, it = self.p.pop_size, self.p.iterations
        hist = np.asarray(self.ops.to_host(self.hist))
        pop = np.asarray(self.ops.to_host(self.population()))
        fit = np.asarray(self.ops.to_host(self.fit))[:s]
        return RunResult(pop, fit, pop[0].copy(), float(fit[0]), hist[:it].copy(), hist[it:2 * it].copy(),
                         self.fitness_batch_calls)


def run_ga_sharded(params: GAParams, fitness: FitnessFunction, rank: int = 0, world: int = 1, device_index: int = 0,
                   group=None) -> RunResult:
    """GPU front door for the sharded run; with world == 1 it equals api.run_ga."""
    ops = CudaOps(fitness, device_index)
    return ShardedGa(params, ops, Shard(rank, world, params.pop_size), torch_allgather(group)).run()
