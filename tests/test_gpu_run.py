"""Generation loop on the GPU: trajectories identical to the reference given the same seed.

Mirrors test_parallel.cpp:86-116 (history best AND mean, final population) and the
run-level cases of test_ga_engine.cpp:309-361."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _same(result, want):
    assert np.array_equal(result.history_best, want["best"])
    assert np.array_equal(result.history_mean, want["mean"])
    assert np.array_equal(result.final_population, want["population"])
    assert np.array_equal(result.final_fitness, want["fitness"])


def test_config1_full_run(gp, oracle, cuda_device):
    """BASELINE config 1: BA(1000, 2), k = 50, pop 100, 100 generations, pc .6 pm .2, seed 1."""
    g = gp.barabasi_albert(1000, 2, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=100, budget=50, iterations=100, seed=1)
    res = gp.run_ga(params, pool, obj)
    assert res.history_best[0] == 444153.0 and res.best_fitness == 408159.0  # SURVEY §8c golden values
    assert res.fitness_batch_calls == 101  # iterations + 1 (test_parallel.cpp:147-158)
    og = oracle.graph_from_edges(g.n, g.edges())
    _same(res, oracle.run_ga(og, 0, 0.6, 0.2, 100, 50, 100, 1, threads=8))
    assert np.all(np.diff(res.history_best) <= 0)  # monotone under elitism


@pytest.mark.parametrize("task", [0, 1])
def test_small_runs_match_oracle(gp, oracle, cuda_device, task):
    for seed, eda in [(3, 0), (4, 3)]:
        g = gp.erdos_renyi(100, 0.04, 665)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        cls = gp.PairwiseConnectivityObjective if task == 0 else gp.SixDstObjective
        params = gp.GAParams(pc=0.8, pm=0.1, pop_size=30, budget=8, iterations=25, seed=seed, eda_interval=eda or None)
        res = gp.run_ga(params, pool, cls(g, pool))
        og = oracle.graph_from_edges(g.n, g.edges())
        _same(res, oracle.run_ga(og, task, 0.8, 0.1, 30, 8, 25, seed, eda_interval=eda))


def test_maximize_direction_runs_match_oracle(gp, oracle, cuda_device):
    """Direction::Maximize (population.hpp:9) through the whole loop — selection weights, roulette, elitism order and the
    history all flip (ga_ops.cpp:62, :199).  The reference's tasks minimise; its toy objectives maximise."""
    g = gp.erdos_renyi(120, 0.035, 11)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    og = oracle.graph_from_edges(g.n, g.edges())
    for task, cls, s, eda in ((0, gp.PairwiseConnectivityObjective, 40, 0), (1, gp.SixDstObjective, 700, 4)):
        params = gp.GAParams(pc=0.7, pm=0.1, pop_size=s, budget=10, iterations=12, seed=9, eda_interval=eda or None,
                             direction=gp.Direction.Maximize)
        res = gp.run_ga(params, pool, cls(g, pool))
        _same(res, oracle.run_ga(og, task, 0.7, 0.1, s, 10, 12, 9, eda_interval=eda, minimize=False, threads=8))
        assert np.all(np.diff(res.history_best) >= 0) and np.all(np.diff(res.final_fitness) <= 0)  # best first = largest first


def test_c5_corner_population_16384(gp, oracle, cuda_device):
    """BASELINE configs[4] corner: n = 1e5, population 16,384 (four lanes of 4096 on two streams): every 64th row and
    both ends against the oracle; one generation of the loop keeps history and stored fitness consistent."""
    g = gp.barabasi_albert(100_000, 5, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    og = oracle.graph_from_edges(g.n, g.edges())
    obj = gp.PairwiseConnectivityObjective(g, pool)
    s, k = 16_384, 5_000
    pop = gp.init_population(pool.size(), s, k, 3)
    got = obj.evaluate_batch(pop)
    pick = np.unique(np.r_[0:16, 0:s:64, 4090:4100, 8190:8194, s - 16:s])
    assert np.array_equal(got[pick], oracle.eval_batch(og, 0, pop[pick], threads=16))
    res = gp.run_ga(gp.GAParams(pc=0.6, pm=0.2, pop_size=s, budget=k, iterations=1, seed=3), pool, obj)
    assert res.history_best[0] == res.final_fitness[0] and np.all(np.diff(res.final_fitness) >= 0)
    rows = np.r_[0:8, s - 8:s]
    assert np.array_equal(res.final_fitness[rows], oracle.eval_batch(og, 0, res.final_population[rows], threads=16))


@pytest.mark.parametrize("ranking", ["default", "sorted-tiles", "counting"])
def test_large_population_run_matches_oracle(gp, oracle, cuda_device, monkeypatch, ranking):
    """Large ragged population sizes (multi-block ranking, weight and pick kernels),
    ragged, on a small graph so that fitness ties are everywhere (stable tie-breaks matter).  Both elitism rankings: binary
    searches over sorted tiles of 1024 (the default from 2048 individuals on) and the counting kernel."""
    if ranking != "default":
        monkeypatch.setenv("GAPA_RANK_TILES_MIN", "1" if ranking == "sorted-tiles" else "100000000")
    g = gp.erdos_renyi(80, 0.05, 7)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    og = oracle.graph_from_edges(g.n, g.edges())
    for s, eda in [(4100, 0), (9001, 2), (700, 0), (1024, 3)]:
        params = gp.GAParams(pc=0.7, pm=0.15, pop_size=s, budget=6, iterations=4, seed=21, eda_interval=eda or None)
        res = gp.run_ga(params, pool, gp.PairwiseConnectivityObjective(g, pool))
        _same(res, oracle.run_ga(og, 0, 0.7, 0.15, s, 6, 4, 21, eda_interval=eda, threads=8))


def test_lpa_and_cda_runs_match_oracle(gp, oracle, cuda_device):
    g = gp.erdos_renyi(120, 0.08, 2)
    split = gp.build_lp_split(g, 0.2, 5)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    params = gp.GAParams(pc=0.7, pm=0.1, pop_size=20, budget=30, iterations=15, seed=9)
    res = gp.run_ga(params, pool, gp.LinkPredictionAttackObjective(split, pool))
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.2, 5)
    _same(res, oracle.run_ga(os_, 3, 0.7, 0.1, 20, 30, 15, 9))

    g = gp.planted_partition(4, 20, 0.3, 0.03, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
    params = gp.GAParams(pc=0.8, pm=0.1, pop_size=16, budget=10, iterations=12, seed=2)
    res = gp.run_ga(params, pool, gp.ModularityAttackObjective(g, pool))
    _same(res, oracle.run_ga(oracle.graph_from_edges(g.n, g.edges()), 2, 0.8, 0.1, 16, 10, 12, 2))


@pytest.mark.parametrize("eda", [0, 4])
def test_sharded_run_equals_single(gp, cuda_device, eda):
    """world = 2 simulated in one process: each 'rank' evaluates its partition_rows block and the
    exchange hook fills in the other block from a full single-GPU evaluation."""
    import ctypes as C
    g = gp.barabasi_albert(400, 2, 3)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=25, budget=20, iterations=10, seed=5, eda_interval=eda or None)
    single = gp.run_ga(params, pool, obj)
    lib = gp.capi.load()
    helper = gp.PairwiseConnectivityObjective(g, pool)

    for rank in (0, 1):
        lo, hi = gp.partition_rows(25, 2)[rank]
        state = {"gen": 0}

        # the hook needs each generation's mutated matrix; derive it with the operator API
        fit = helper.evaluate_batch(gp.init_population(pool.size(), 25, 20, 5))
        pop = gp.init_population(pool.size(), 25, 20, 5)
        mutated_by_gen = []
        for gen in range(1, 11):
            if eda and gen % eda == 0:
                mutated = gp.mutate(gp.eda_sample(pop, 25, pool.size(), 5, gen), 0.2, pool.size(), 5, gen)
            else:
                idx = gp.roulette_pick(fit, gp.Direction.Minimize, 5, gen)
                mutated = gp.crossover_mutate(pop, idx, 0.6, 0.2, pool.size(), 5, gen)
            fm = helper.evaluate_batch(mutated)
            mutated_by_gen.append(mutated)
            pop, fit = gp.elitism(pop, mutated, fit, fm, gp.Direction.Minimize)
        assert np.array_equal(pop, single.final_population)  # stepwise operator API == fused run

        def exchange2(user, fit_ptr, s, block, stream, state=state):
            gp.capi.check(lib.gapa_cuda_stream_sync(0, stream))
            gen = state["gen"]
            m = gp.init_population(pool.size(), 25, 20, 5) if gen == 0 else mutated_by_gen[gen - 1]
            full = np.ascontiguousarray(helper.evaluate_batch(m))
            gp.capi.check(lib.gapa_cuda_memcpy_h2d(0, fit_ptr, full.ctypes.data_as(C.c_void_p), 8 * s))
            state["gen"] += 1
            return 0

        res = gp.run_ga(params, pool, obj, rank=rank, world=2, exchange=exchange2)
        assert np.array_equal(res.final_population, single.final_population)
        assert np.array_equal(res.history_mean, single.history_mean)
        # GenerationStats columns (modes.hpp:63-71): generation 1 exchanges twice (init + M_POP), the rest once
        assert [h.messages for h in res.history] == [2] + [1] * 9
        assert all(h.exchange_seconds > 0 and h.lifecycle_seconds == 0 for h in res.history)
        assert all(abs(h.compute_seconds + h.exchange_seconds - h.wall_seconds) < 1e-9 for h in res.history)


def test_run_rejects_bad_params(gp, cuda_device):
    g = gp.barabasi_albert(50, 2, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    for bad in (dict(pop_size=1), dict(budget=0), dict(iterations=0), dict(pc=1.5), dict(pm=-0.1), dict(eda_interval=0)):
        kw = dict(pc=0.5, pm=0.1, pop_size=10, budget=3, iterations=2, seed=1)
        kw.update(bad)
        with pytest.raises(gp.capi.GapaCudaError):
            gp.run_ga(gp.GAParams(**kw), pool, obj)


@pytest.mark.parametrize("eda", [0, 3])
def test_sharded_driver_recomputes_foreign_rows(gp, oracle, cuda_device, eda):
    """driver.ShardedGa with the CUDA ops as rank 0 and as rank 1 of a 2-rank run, one process: the
    fake all-gather fills the other rank's fitness block by building that block with the operator
    API and evaluating it.  Each rank builds only its own rows of M_POP, so the final population is
    only right if the elitism gather recomputes surviving foreign rows exactly."""
    import torch
    from paper_2412_20980_b200.driver import CudaOps, Shard, ShardedGa

    g = gp.barabasi_albert(500, 2, 4)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    helper = gp.PairwiseConnectivityObjective(g, pool)
    s, k, iters = 37, 15, 9
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=s, budget=k, iterations=iters, seed=11, eda_interval=eda or None)
    want = oracle.run_ga(oracle.graph_from_edges(g.n, g.edges()), 0, 0.6, 0.2, s, k, iters, 11, eda_interval=eda)
    for rank in (0, 1):
        shard = Shard(rank, 2, s)
        other_lo, other_hi = gp.partition_rows(s, 2)[1 - rank]
        box = {}

        def gather(fit, shard_, box=box, other_lo=other_lo, other_hi=other_hi):
            ga = box["ga"]
            pop = ga.population().cpu().numpy()
            gen = ga.generation
            if gen == 0:
                rows = pop[other_lo:other_hi]
            elif eda and gen % eda == 0:
                rows = gp.mutate_block(gp.eda_sample(pop, s, pool.size(), 11, gen)[other_lo:other_hi], other_lo, 0.2,
                                       pool.size(), 11, gen)
            else:
                rows = gp.crossover_mutate(pop, ga.partner.cpu().numpy(), 0.6, 0.2, pool.size(), 11, gen, other_lo,
                                           other_hi - other_lo)
            fit[other_lo:other_hi] = torch.from_numpy(helper.evaluate_batch(rows)).to(fit.device)

        ga = ShardedGa(params, CudaOps(obj, 0), shard, gather)
        box["ga"] = ga
        res = ga.run()
        assert np.array_equal(res.final_population, want["population"]), rank
        assert np.array_equal(res.history_best, want["best"]) and np.array_equal(res.history_mean, want["mean"])
        assert np.array_equal(res.final_fitness, want["fitness"])


def test_generation_stats_and_overhead_report(gp, cuda_device):
    """GenerationStats / overhead_report (modes.hpp:63-99, modes.cpp:518-530) on one GPU: the three time
    columns sum to wall, nothing is exchanged, and the table has the reference's layout."""
    g = gp.barabasi_albert(3000, 3, 2)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    res = gp.run_ga(gp.GAParams(pc=0.6, pm=0.2, pop_size=64, budget=150, iterations=6, seed=3), pool, obj)
    assert len(res.history) == 6
    assert [h.best for h in res.history] == res.history_best.tolist()
    assert [h.mean for h in res.history] == res.history_mean.tolist()
    assert all(h.wall_seconds > 0 and h.messages == 0 and h.exchange_seconds == 0 for h in res.history)
    assert all(h.compute_seconds == h.wall_seconds for h in res.history)
    assert sum(h.wall_seconds for h in res.history) <= res.total_wall_seconds * 1.05 + 1e-3
    assert res.eval_seconds <= sum(h.wall_seconds for h in res.history) * 1.001 + 1e-6
    lines = gp.overhead_report(res).splitlines()
    assert lines[0] == "gen  wall_s      compute_s   exchange_s  lifecycle_s messages"
    assert len(lines) == 7 and lines[1].startswith("1    0.") and lines[1].endswith(" 0") and lines[6].startswith("6    ")
    assert [len(x) for x in lines[1].split(" ") if x][1:5] == [8, 8, 8, 8]


def test_sampled_timing_marks_keep_results_and_columns(gp, oracle, cuda_device):
    """Timing marks are sampled for short generations (run.cu): from generation 2 for populations up to 512, from the
    first status poll (generation 16) for larger ones.  Sampling must not touch the trajectory, every generation must
    still report a positive wall time, and the columns must stay consistent with the totals."""
    g = gp.erdos_renyi(120, 0.04, 9)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    og = oracle.graph_from_edges(g.n, g.edges())
    for s, iters in [(40, 37), (600, 37)]:
        params = gp.GAParams(pc=0.7, pm=0.1, pop_size=s, budget=7, iterations=iters, seed=4)
        res = gp.run_ga(params, pool, gp.PairwiseConnectivityObjective(g, pool))
        _same(res, oracle.run_ga(og, 0, 0.7, 0.1, s, 7, iters, 4, threads=8))
        walls = [h.wall_seconds for h in res.history]
        assert len(walls) == iters and all(w > 0 for w in walls)
        assert all(h.compute_seconds == h.wall_seconds and h.messages == 0 for h in res.history)
        assert sum(walls) <= res.total_wall_seconds * 1.05 + 1e-3
        assert 0 < res.eval_seconds <= sum(walls) * 1.001 + 1e-6
        if s <= 512:  # always sampled; larger populations only when an evaluation is short (not under a sanitizer)
            assert len(set(walls[20:26])) <= 2  # generations between two marks share their mean
        assert res.fitness_batch_calls == iters + 1


@pytest.mark.parametrize("defer", ["1", "0"])
def test_deferred_statistics_fp64_and_midrun_result(gp, oracle, cuda_device, monkeypatch, defer):
    """Populations beyond 1024: a generation's best / mean ride on the NEXT generation's selection launch (an extra block of
    k_ga_weights, run.cu) unless that generation is an EDA one or the run ends.  Non-integer fitness (AUC) takes the
    sequential-sum path of that block; a result() in the middle of a run flushes the pending entry and the run goes on."""
    monkeypatch.setenv("GAPA_DEFER_STATS", defer)
    g = gp.erdos_renyi(60, 0.12, 3)
    split = gp.build_lp_split(g, 0.2, 5)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.2, 5)
    for s, eda in [(1100, 0), (1300, 3)]:
        params = gp.GAParams(pc=0.7, pm=0.1, pop_size=s, budget=8, iterations=7, seed=13, eda_interval=eda or None)
        want = oracle.run_ga(os_, 3, 0.7, 0.1, s, 8, 7, 13, eda_interval=eda, threads=8)
        obj = gp.LinkPredictionAttackObjective(split, pool)
        _same(gp.run_ga(params, pool, obj), want)
        loop = gp.GaLoop(params, obj)
        loop.advance(4)
        mid = loop.result()  # generation 4's statistics were pending (generation 5 selects) unless it is an EDA one
        assert np.array_equal(mid.history_best[:4], want["best"][:4]) and np.array_equal(mid.history_mean[:4], want["mean"][:4])
        assert np.all(mid.history_best[4:] == 0)
        loop.advance(100)
        _same(loop.result(), want)
        loop.close()
