"""SURVEY §8(f) rows on the CUDA path, against the oracle (which tests/test_oracle_vs_ref.py and
tests/golden/widen.json pin to the unmodified reference):

  f-1  sixdst_fitness(ClosurePolicy::SixDegrees) — largest radius-8 ball (fitness.cpp:18-26 over
       accessibility.cpp:20-37; test_fitness.cpp:94-103)
  f-2  EdgeAddition pools under cda_fitness (gene_pool.cpp:57-60, :81-87; acceptance.cpp:207-246)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TASK_MCN, TASK_SIXDST, TASK_CDA_ADD = 1, 4, 5


def _rand_edges(rng, n, dens):
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < dens
    return np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.int32)


# ------------------------------------------------------------------------------- f-1
def test_sixdegrees_fixed_cases(gp, cuda_device):
    path = gp.Graph(40, [(i, i + 1) for i in range(39)])
    pool = gp.build_gene_pool(path, gp.PoolKind.NodeRemoval)
    six = gp.SixDstObjective(path, pool, policy=gp.ClosurePolicy.SixDegrees)
    exact = gp.SixDstObjective(path, pool)
    assert six.evaluate_one([]) == 17.0 and exact.evaluate_one([]) == 40.0  # distance 8 each side, not the full path
    assert six.evaluate_one([20]) == 17.0                                   # 0..19 still holds a full ball around 8..11
    assert six.evaluate_one([8, 25]) == 16.0                                # pieces 0..7 (8), 9..24 (16), 26..39 (14)
    assert six.evaluate_one(list(range(40))) == 1.0                         # every node removed: singletons
    k6 = gp.Graph(6, [(a, b) for a in range(6) for b in range(a + 1, 6)])
    p6 = gp.build_gene_pool(k6, gp.PoolKind.NodeRemoval)
    assert gp.sixdst_fitness(k6, np.zeros((1, 0), np.int32), p6, gp.ClosurePolicy.SixDegrees).tolist() == [6.0]
    assert gp.sixdst_fitness(k6, [[0, 0, 3]], p6, gp.ClosurePolicy.SixDegrees).tolist() == [4.0]
    with pytest.raises(gp.capi.GapaCudaError) as e:
        six.evaluate_one([40])
    assert e.value.code == gp.capi.E_RANGE
    with pytest.raises(gp.capi.GapaCudaError):
        gp.SixDstObjective(path, gp.build_gene_pool(path, gp.PoolKind.EdgeRemoval), policy=gp.ClosurePolicy.SixDegrees)


def test_sixdegrees_random_exact(gp, oracle, cuda_device):
    rng = np.random.default_rng(31)
    cut = 0
    for trial in range(24):
        n = int(rng.integers(2, 700))
        e = _rand_edges(rng, n, float(rng.uniform(0.4, 3.0)) / n)
        if trial % 4 == 0:
            chain = np.stack([np.arange(n - 1), np.arange(1, n)], 1).astype(np.int32)
            e = np.unique(np.concatenate([e, chain]), axis=0).astype(np.int32)
        g = gp.Graph(n, e)
        og = oracle.graph_from_edges(n, e)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        rows, k = int(rng.integers(1, 20)), int(rng.integers(0, n // 4 + 2))
        batch = rng.integers(0, n, (rows, k)).astype(np.int32)
        got = gp.SixDstObjective(g, pool, policy=gp.ClosurePolicy.SixDegrees).evaluate_batch(batch)
        assert np.array_equal(got, oracle.eval_batch(og, TASK_SIXDST, batch)), trial
        cut += int(np.any(got < oracle.eval_batch(og, TASK_MCN, batch)))
    assert cut > 5


def test_sixdegrees_global_scratch_path_and_more_rows_than_sms(gp, oracle, cuda_device):
    """n = 14,000 does not fit the shared-memory word arrays; 200 rows > 148 CTAs."""
    g = gp.barabasi_albert(14000, 1, 5)  # a tree: balls of radius 8 are far smaller than components
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.SixDstObjective(g, pool, policy=gp.ClosurePolicy.SixDegrees)
    batch = gp.init_population(pool.size(), 3, 700, 2)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, TASK_SIXDST, batch))
    g = gp.barabasi_albert(900, 1, 6)
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    batch = gp.init_population(pool.size(), 200, 45, 3)
    got = gp.SixDstObjective(g, pool, policy=gp.ClosurePolicy.SixDegrees).evaluate_batch(batch)
    assert np.array_equal(got, oracle.eval_batch(og, TASK_SIXDST, batch, threads=8))


def test_sixdegrees_ga_trajectory_and_sharded_run(gp, oracle, cuda_device):
    g = gp.barabasi_albert(400, 1, 9)
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.SixDstObjective(g, pool, policy=gp.ClosurePolicy.SixDegrees)
    p = gp.GAParams(pc=0.5, pm=0.3, pop_size=21, budget=40, iterations=12, seed=5, eda_interval=4)
    want = oracle.run_ga(og, TASK_SIXDST, 0.5, 0.3, 21, 40, 12, 5, eda_interval=4)
    r = gp.run_ga(p, pool, obj)
    assert np.array_equal(r.history_best, want["best"]) and np.array_equal(r.history_mean, want["mean"])
    assert np.array_equal(r.final_population, want["population"])


# ------------------------------------------------------------------------------- f-2
def test_edge_addition_pool_rules(gp, cuda_device):
    k4 = gp.Graph(4, [(a, b) for a in range(4) for b in range(a + 1, 4)])
    with pytest.raises(gp.capi.GapaCudaError, match="complete"):  # gene_pool.cpp:86
        gp.build_gene_pool(k4, gp.PoolKind.EdgeAddition)
    g = gp.Graph(5, [(0, 1), (1, 2), (3, 4)])
    pool = gp.build_gene_pool(g, gp.PoolKind.EdgeAddition)
    assert pool.size() == 7 and [pool.gene(i) for i in range(7)] == [(0, 2), (0, 3), (0, 4), (1, 3), (1, 4), (2, 3), (2, 4)]
    with pytest.raises(gp.capi.GapaCudaError):  # node pools stay incompatible (fitness.cpp:54-57)
        gp.ModularityAttackObjective(g, gp.build_gene_pool(g, gp.PoolKind.NodeRemoval))
    with pytest.raises(gp.capi.GapaCudaError):  # lpa_fitness takes EdgeRemoval only (fitness.cpp:87)
        gp.LinkPredictionAttackObjective(gp.build_lp_split(gp.erdos_renyi(60, 0.2, 1), 0.2, 1), pool)
    with pytest.raises(gp.capi.GapaCudaError, match="duplicate"):  # gene_pool.cpp:36-41
        gp.ModularityAttackObjective(g, gp.GenePool(gp.PoolKind.EdgeAddition, [0, 2], [2, 0], graph=g))
    obj = gp.ModularityAttackObjective(g, pool)
    with pytest.raises(gp.capi.GapaCudaError) as e:
        obj.evaluate_one([7])
    assert e.value.code == gp.capi.E_RANGE


def test_edge_addition_custom_pool_with_present_edge_is_noop(gp, oracle, cuda_device):
    """A caller-built pool may hold a pair that is already an edge: adjacency.set on a set bit."""
    g = gp.barabasi_albert(40, 2, 3)
    e = g.edges()
    custom = gp.GenePool(gp.PoolKind.EdgeAddition, [int(e[0][0]), 5, 7], [int(e[0][1]), 30, 31], graph=g)
    obj = gp.ModularityAttackObjective(g, custom)
    og = oracle.graph_from_edges(g.n, e)
    assert obj.evaluate_one([0]) == obj.evaluate_one([]) == oracle.eval_batch(og, 2, np.zeros((1, 0), np.int32))[0]
    canon = gp.build_gene_pool(g, gp.PoolKind.EdgeAddition)
    idx = {canon.gene(i): i for i in range(canon.size())}
    oracle.addition_pool(og)
    want = oracle.eval_batch(og, TASK_CDA_ADD, np.array([[idx[(5, 30)], idx[(7, 31)]]], np.int32))
    assert obj.evaluate_batch([[1, 2]]).tolist() == obj.evaluate_batch([[2, 0, 1]]).tolist() == want.tolist()


def test_edge_addition_cda_random_exact(gp, oracle, cuda_device):
    rng = np.random.default_rng(33)
    for trial in range(16):
        n = int(rng.integers(4, 260))
        e = _rand_edges(rng, n, 0.0 if trial == 0 else float(rng.uniform(0.5, 6.0)) / n)
        g = gp.Graph(n, e)
        og = oracle.graph_from_edges(n, e)
        pool = gp.build_gene_pool(g, gp.PoolKind.EdgeAddition)
        u, v = oracle.addition_pool(og)
        assert np.array_equal(pool.u, u) and np.array_equal(pool.v, v)
        rows, k = int(rng.integers(1, 12)), int(rng.integers(0, 3 * n))
        batch = rng.integers(0, pool.size(), (rows, k)).astype(np.int32)
        if k > 3:
            batch[0, :3] = batch[0, 3]  # repeated genes are idempotent
        got = gp.ModularityAttackObjective(g, pool).evaluate_batch(batch)
        assert np.array_equal(got, oracle.eval_batch(og, TASK_CDA_ADD, batch, threads=8)), trial
    # edgeless graph, empty perturbation: Q undefined -> -0.5 (fitness.cpp:39)
    g = gp.Graph(6, np.zeros((0, 2), np.int32))
    assert gp.ModularityAttackObjective(g, gp.build_gene_pool(g, gp.PoolKind.EdgeAddition)).evaluate_one([]) == -0.5


def test_edge_addition_larger_graph_and_ga(gp, oracle, cuda_device):
    g = gp.planted_partition(6, 60, 0.15, 0.01, 4)  # n = 360: per-community arrays in shared memory
    og = oracle.graph_from_edges(g.n, g.edges())
    oracle.addition_pool(og)
    pool = gp.build_gene_pool(g, gp.PoolKind.EdgeAddition)
    k = gp.perturbation_budget(g, gp.PoolKind.EdgeAddition, 0.1)
    obj = gp.ModularityAttackObjective(g, pool)
    pop = gp.init_population(pool.size(), 160, k, 3)  # more rows than CTAs
    assert np.array_equal(obj.evaluate_batch(pop), oracle.eval_batch(og, TASK_CDA_ADD, pop, threads=8))
    p = gp.GAParams(pc=0.8, pm=0.1, pop_size=14, budget=k, iterations=6, seed=9)
    want = oracle.run_ga(og, TASK_CDA_ADD, 0.8, 0.1, 14, k, 6, 9, threads=8)
    r = gp.run_ga(p, pool, obj)
    assert np.array_equal(r.history_best, want["best"]) and np.array_equal(r.final_population, want["population"])
    # then back to a removal pool on a fresh objective over the same graph: the two pool kinds do not leak state
    rem = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
    batch = gp.init_population(rem.size(), 5, 30, 1)
    assert np.array_equal(gp.ModularityAttackObjective(g, rem).evaluate_batch(batch), oracle.eval_batch(og, 2, batch))
