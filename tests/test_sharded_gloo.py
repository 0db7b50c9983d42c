"""CPU, world_size 2, gloo: the N>1 host logic of paper_2412_20980_b200.driver (row partition,
padded in-place all-gather, replicated operators, loop order) with the oracle standing in for
the device ops.  Every rank must reproduce the single-process reference trajectory bit for bit
(mirror of test_parallel.cpp:86-104)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from oracle.bindings import Oracle
from paper_2412_20980_b200.api import GAParams
from paper_2412_20980_b200.driver import ShardedGa, Shard, torch_allgather

class OracleOps:
    """test stand-in for CudaOps: same slot-pool interface, numpy/oracle arithmetic on CPU tensors"""
    def __init__(self, o, ctx, task, pool_size):
        self.o, self.ctx, self.task, self.pool_size = o, ctx, task, pool_size
    def empty_genes(self, r, c): return torch.full((r, c), -7, dtype=torch.int32)
    def zeros_f64(self, n): return torch.zeros(n, dtype=torch.float64)
    def empty_i32(self, n): return torch.zeros(n, dtype=torch.int32)
    def init(self, pool, parent, child, s, seed, gen):
        parent.copy_(torch.arange(s, dtype=torch.int32)); child.copy_(torch.arange(s, 2 * s, dtype=torch.int32))
        pool[:s] = torch.from_numpy(self.o.init_population(self.pool_size, s, pool.shape[1], seed, gen))
    def select(self, fit, s, minimize, seed, gen, partner):
        partner.copy_(torch.from_numpy(self.o.roulette_pick(fit[:s].numpy(), bool(minimize), seed, gen)))
    def _children(self, pool, parent, partner, pc, pm, seed, gen):
        pop = pool[parent.long()].numpy()
        c = (self.o.crossover(pop, partner.numpy(), pc, seed, gen) if partner is not None
             else self.o.eda_sample(pop, pop.shape[0], self.pool_size, seed, gen, True))
        return self.o.mutate_block(c, 0, pm, self.pool_size, seed, gen)
    def variation(self, pool, parent, child, partner, s, pc, pm, seed, gen, lo, hi):
        rows = self._children(pool, parent, partner, pc, pm, seed, gen)
        pool[child[lo:hi].long()] = torch.from_numpy(rows[lo:hi])  # only this rank's block is built
    def variation_eval(self, pool, parent, child, partner, s, pc, pm, seed, gen, lo, hi, fit_out):
        self.variation(pool, parent, child, partner, s, pc, pm, seed, gen, lo, hi)
        self.eval_rows(pool, child, lo, hi, fit_out)
    def eval_rows(self, pool, table, lo, hi, fit_out):
        if hi > lo: fit_out[lo:hi] = torch.from_numpy(self.o.eval_batch(self.ctx, self.task, pool[table[lo:hi].long()].numpy()))
    def elitism(self, pool, parent, child, partner, s, lo, hi, fit, fit_m, minimize, pc, pm, seed, gen, next_parent, next_child, next_fit):
        f = np.concatenate([fit[:s].numpy(), fit_m[:s].numpy()])
        order = np.argsort(f if minimize else -f, kind="stable")
        slots = torch.cat([parent, child])
        full = self._children(pool, parent, partner, pc, pm, seed, gen)
        assert np.array_equal(full[lo:hi], pool[child[lo:hi].long()].numpy())
        for x in order[:s]:                      # foreign survivors are rebuilt, not fetched
            if x >= s and not (lo <= x - s < hi): pool[int(child[x - s])] = torch.from_numpy(full[x - s])
        next_parent.copy_(slots[order[:s]]); next_child.copy_(slots[order[s:]])
        next_fit[:s] = torch.from_numpy(f[order[:s]])
    def gather(self, pool, table, rows): return pool[table[:rows].long()].clone()
    def stats(self, fit, s, hist, index, iters):
        total = 0.0
        for x in fit[:s].tolist(): total += x
        hist[index] = fit[0]; hist[iters + index] = total / s
    def to_host(self, t): return t.numpy()

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
o = Oracle()
cfg = json.loads(sys.argv[2])
g = o.graph_ba(cfg["n"], 2, 3)
params = GAParams(pc=0.6, pm=0.2, pop_size=cfg["s"], budget=cfg["k"], iterations=cfg["iters"], seed=5, eda_interval=cfg["eda"] or None)
ga = ShardedGa(params, OracleOps(o, g, 0, g.n), Shard(rank, world, cfg["s"]), torch_allgather())
res = ga.run()
want = o.run_ga(g, 0, 0.6, 0.2, cfg["s"], cfg["k"], cfg["iters"], 5, eda_interval=cfg["eda"])
ok = (np.array_equal(res.history_best, want["best"]) and np.array_equal(res.history_mean, want["mean"])
      and np.array_equal(res.final_population, want["population"]) and np.array_equal(res.final_fitness, want["fitness"])
      and res.fitness_batch_calls == cfg["iters"] + 1)
flag = torch.tensor([1 if ok else 0])
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0: print("SHARDED_OK" if int(flag) == 1 else "SHARDED_MISMATCH")
dist.destroy_process_group()
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cfg", [dict(n=300, s=25, k=12, iters=8, eda=0),   # ragged: blocks of 13 and 12
                                 dict(n=200, s=7, k=5, iters=6, eda=3),     # EDA generations
                                 dict(n=200, s=16, k=9, iters=5, eda=0)])
def test_two_rank_run_equals_single_process(tmp_path, cfg):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(script), ROOT, json.dumps(cfg)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert "SHARDED_OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]


def test_shard_arithmetic():
    from paper_2412_20980_b200.driver import Shard
    sh = Shard(1, 2, 25)
    assert (sh.block, sh.rows, sh.padded) == (13, (13, 25), 26)
    sh = Shard(7, 8, 7)  # more ranks than rows: trailing blocks are empty (modes.cpp:511-513)
    assert (sh.block, sh.rows, sh.padded) == (1, (7, 7), 8)
    sh = Shard(3, 8, 4096)
    assert (sh.block, sh.rows, sh.padded) == (512, (1536, 2048), 4096)
