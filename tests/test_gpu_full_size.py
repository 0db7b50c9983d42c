"""GPU: BASELINE.json's full size (C4: Barabasi-Albert n = 1,000,000, attach 5, k = 50,000) — the oracle on a
sample of the rows, and size-independent properties of the fitness on the whole batch."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, ATTACH, K, ROWS = 1_000_000, 5, 50_000, 1024


@pytest.fixture(scope="module")
def c4(gp, cuda_device):
    g = gp.barabasi_albert(N, ATTACH, 1)
    assert g.edge_count() == 4_999_985  # the reference generator's edge count at this shape
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    pop = gp.init_population(pool.size(), ROWS, K, 1)
    return g, pool, pop


def test_full_size_matches_the_oracle_on_a_sample(gp, oracle, c4):
    g, pool, pop = c4
    pc = gp.PairwiseConnectivityObjective(g, pool)
    mcn = gp.SixDstObjective(g, pool)
    got_pc, got_mcn = pc.evaluate_batch(pop), mcn.evaluate_batch(pop)
    og = oracle.graph_from_edges(g.n, g.edges())
    sample = np.r_[0:24, ROWS - 8:ROWS]
    assert np.array_equal(got_pc[sample], oracle.eval_batch(og, 0, pop[sample], threads=16))
    assert np.array_equal(got_mcn[sample], oracle.eval_batch(og, 1, pop[sample], threads=16))
    # PC and MCN of the same individual are consistent: C(mcn, 2) <= PC <= C(mcn, 2) + C(alive - mcn, 2)
    alive = N - np.array([len(np.unique(r)) for r in pop[:64]])
    c2 = lambda x: x * (x - 1) / 2
    assert np.all(c2(got_mcn[:64]) <= got_pc[:64]) and np.all(got_pc[:64] <= c2(got_mcn[:64]) + c2(alive - got_mcn[:64]))


def test_full_size_every_row_of_the_bench_population(gp, oracle, c4):
    """BASELINE configs[3] at its own population: all 4096 individuals of one batch against the oracle (PC), and all
    1024 of the module's batch for MCN — the numbers bench.py quotes are for exactly this shape."""
    g, pool, pop = c4
    og = oracle.graph_from_edges(g.n, g.edges())
    big = gp.init_population(pool.size(), 4096, K, 2)
    assert np.array_equal(gp.PairwiseConnectivityObjective(g, pool).evaluate_batch(big), oracle.eval_batch(og, 0, big, threads=16))
    assert np.array_equal(gp.SixDstObjective(g, pool).evaluate_batch(pop), oracle.eval_batch(og, 1, pop, threads=16))


def test_full_size_trajectory_matches_the_oracle(gp, oracle, c4):
    """Three generations of the C4 GA (population 256) against oracle.run_ga: history best AND mean, final population
    and fitness bit for bit (test_parallel.cpp:86-104 at n = 1e6) — the one-GPU library loop, and both ranks of a
    two-rank gapa_cuda_run_multi (peer-mailbox exchange, foreign parents read from the builder's pool)."""
    g, pool, _ = c4
    og = oracle.graph_from_edges(g.n, g.edges())
    obj = gp.PairwiseConnectivityObjective(g, pool)
    params = gp.GAParams(pc=0.6, pm=0.2, pop_size=256, budget=K, iterations=3, seed=5)
    want = oracle.run_ga(og, 0, 0.6, 0.2, 256, K, 3, 5, threads=16)
    res = gp.run_ga(params, pool, obj)
    sharded = gp.run_ga_multi(params, [obj, gp.PairwiseConnectivityObjective(g, pool)], transport="peer")
    for r in [res] + sharded:
        assert np.array_equal(r.history_best, want["best"]) and np.array_equal(r.history_mean, want["mean"])
        assert np.array_equal(r.final_population, want["population"]) and np.array_equal(r.final_fitness, want["fitness"])


def test_full_size_properties(gp, c4):
    g, pool, pop = c4
    pc = gp.PairwiseConnectivityObjective(g, pool)
    base = pc.evaluate_batch(pop)
    # a row's fitness does not depend on its batch: reversed order, ragged split
    assert np.array_equal(pc.evaluate_batch(pop[::-1].copy())[::-1], base)
    assert np.array_equal(np.concatenate([pc.evaluate_batch(pop[:333]), pc.evaluate_batch(pop[333:])]), base)
    # nor on the order of its genes, and repeated genes are idempotent (gene_pool.cpp:61-64)
    shuffled = pop[:128].copy()
    rng = np.random.default_rng(3)
    for r in shuffled:
        rng.shuffle(r)
    assert np.array_equal(pc.evaluate_batch(shuffled), base[:128])
    doubled = np.concatenate([pop[:64], pop[:64, :1000]], axis=1)
    assert np.array_equal(pc.evaluate_batch(doubled), base[:64])
    # nothing removed: the graph is connected; everything removed: only singletons
    assert pc.evaluate_one([]) == N * (N - 1) / 2
    assert gp.SixDstObjective(g, pool).evaluate_one([]) == float(N)
    # removing MORE can only lower the pairwise connectivity of what was one component
    more = np.concatenate([pop[:32], pop[32:64]], axis=1)
    assert np.all(pc.evaluate_batch(more) <= np.minimum(base[:32], base[32:64]))


def test_full_size_generation_loop_is_monotone_and_reproducible(gp, c4):
    g, pool, _ = c4
    obj = gp.PairwiseConnectivityObjective(g, pool)
    p = gp.GAParams(pc=0.6, pm=0.2, pop_size=256, budget=K, iterations=4, seed=7)
    a, b = gp.run_ga(p, pool, obj), gp.run_ga(p, pool, obj)
    assert np.array_equal(a.history_best, b.history_best) and np.array_equal(a.final_population, b.final_population)
    assert np.all(np.diff(a.history_best) <= 0) and np.all(np.diff(a.final_fitness) >= 0)  # elitism: best-first, never worse
    assert np.array_equal(obj.evaluate_batch(a.final_population), a.final_fitness)  # stored fitness == re-evaluation


def test_config3_full_size_lpa(gp, oracle, cuda_device):
    """BASELINE configs[2]: Erdos-Renyi n = 10,000 <d> = 10, 10 % hidden, k = ceil(0.1 m_train), population 50."""
    g = gp.erdos_renyi(10_000, 10 / 9999, 1)
    split = gp.build_lp_split(g, 0.1, 1)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    k = gp.perturbation_budget(split.train, gp.PoolKind.EdgeRemoval, 0.1)
    assert (g.edge_count(), len(split.test_edges), k) == (50_277, 5_028, 4_525)  # SURVEY §8 sizes
    obj = gp.LinkPredictionAttackObjective(split, pool)
    pop = gp.init_population(pool.size(), 50, k, 1)
    got = obj.evaluate_batch(pop)
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.1, 1)
    assert np.array_equal(got, oracle.eval_batch(os_, 3, pop, threads=16))
    assert np.array_equal(obj.evaluate_batch(pop[::-1].copy())[::-1], got)  # batch composition does not matter
    assert obj.evaluate_one(np.arange(pool.size())) == 0.5                # nothing left to score: every pair ties
