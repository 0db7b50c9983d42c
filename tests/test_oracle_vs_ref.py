"""CPU: the C oracle against the compiled, unmodified reference (oracle/_ref) on wider random
sweeps than the golden files hold.  Skipped where the reference binary is not available."""
import numpy as np
import pytest

from oracle.bindings import MODE_M, MODE_S, TASK_CDA, TASK_CDA_ADD, TASK_LPA, TASK_MCN, TASK_PC, TASK_SIXDST


def _rand_edges(rng, n, dens):
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < dens
    return np.stack([iu[0][keep], iu[1][keep]], 1).astype(np.int32)


def test_rng_streams(oracle, ref):
    rng = np.random.default_rng(1)
    for _ in range(50):
        seed, gen, row = (int(x) for x in rng.integers(0, 2**62, 3))
        role = int(rng.integers(1, 6))
        assert np.array_equal(oracle.stream_u64(seed, gen, role, row, 16), ref.stream_u64(seed, gen, role, row, 16))
        assert np.array_equal(oracle.stream_unit(seed, gen, role, row, 16), ref.stream_unit(seed, gen, role, row, 16))
        b = int(rng.integers(1, 2**32 - 1))
        assert np.array_equal(oracle.stream_index(seed, gen, role, row, b, 16), ref.stream_index(seed, gen, role, row, b, 16))


def test_generators_and_pools(oracle, ref):
    for og, rg in [(oracle.graph_ba(700, 3, 5), ref.graph_ba(700, 3, 5)), (oracle.graph_ba(50, 1, 2), ref.graph_ba(50, 1, 2)),
                   (oracle.graph_er(300, 0.05, 9), ref.graph_er(300, 0.05, 9)),
                   (oracle.graph_sbm(5, 40, 0.3, 0.02, 4), ref.graph_sbm(5, 40, 0.3, 0.02, 4))]:
        assert np.array_equal(og.edges, ref.graph_edges(rg))
        u, v = ref.pool_genes(rg, 0)  # EdgeRemoval pool order == oracle edge ranks
        assert np.array_equal(u, og.pool_u) and np.array_equal(v, og.pool_v)
        for rate in (0.05, 0.1, 1.0, 0.0001):
            assert oracle.budget(og.m, rate) == ref.budget(rg, 0, rate)
            assert oracle.budget(og.n, rate) == ref.budget(rg, 2, rate)


def test_pc_mcn_500_pairs(oracle, ref):
    """acceptance.cpp:83-105 — 500 (graph, individual) pairs, exact."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        n = int(rng.integers(4, 80))
        e = _rand_edges(rng, n, float(rng.uniform(0.01, 0.4)))
        og, rg = oracle.graph_from_edges(n, e), ref.graph_from_edges(n, e)
        batch = rng.integers(0, n, (5, int(rng.integers(0, n + 1)))).astype(np.int32)
        for task in (TASK_PC, TASK_MCN):
            assert np.array_equal(oracle.eval_batch(og, task, batch), ref.eval_batch(rg, task, batch))


def test_cda_random(oracle, ref):
    rng = np.random.default_rng(4)
    for trial in range(30):
        n = int(rng.integers(5, 90))
        e = _rand_edges(rng, n, float(rng.uniform(0.03, 0.3)))
        if len(e) == 0:
            continue
        og, rg = oracle.graph_from_edges(n, e), ref.graph_from_edges(n, e)
        assert np.array_equal(oracle.detect_communities(og), ref.detect_communities(rg))
        batch = rng.integers(0, len(e), (3, int(rng.integers(0, len(e) + 1)))).astype(np.int32)
        assert np.array_equal(oracle.eval_batch(og, TASK_CDA, batch), ref.eval_batch(rg, TASK_CDA, batch))


def test_cda_sbm_1000(oracle, ref):
    og, rg = oracle.graph_sbm(10, 100, 0.1, 0.005, 1), ref.graph_sbm(10, 100, 0.1, 0.005, 1)
    k = oracle.budget(og.m, 0.05)
    pop = oracle.init_population(og.m, 2, k, 1)
    assert np.array_equal(oracle.eval_batch(og, TASK_CDA, pop), ref.eval_batch(rg, TASK_CDA, pop, threads=2))


def test_lpa_random(oracle, ref):
    rng = np.random.default_rng(5)
    for trial in range(15):
        n = int(rng.integers(30, 250))
        og, rg = oracle.graph_er(n, 0.1, trial), ref.graph_er(n, 0.1, trial)
        frac = float(rng.uniform(0.05, 0.5))
        so, sr = oracle.split_build(og, frac, trial + 7), ref.split_build(rg, frac, trial + 7)
        t, p = ref.split_pairs(sr)
        assert np.array_equal(so.test, t) and np.array_equal(so.probe, p)
        assert np.array_equal(so.train.edges, ref.graph_edges(ref.split_train(sr)))
        batch = rng.integers(0, so.train.m, (4, int(rng.integers(0, so.train.m)))).astype(np.int32)
        assert np.array_equal(oracle.eval_batch(so, TASK_LPA, batch), ref.eval_batch(sr, TASK_LPA, batch))
        u, v = (int(x) for x in so.test[0])
        assert oracle.ra_score(so.train, u, v) == ref.ra_score(ref.split_train(sr), u, v)


def test_operators_random(oracle, ref):
    rng = np.random.default_rng(6)
    for trial in range(40):
        s, k, pool = int(rng.integers(2, 120)), int(rng.integers(1, 40)), int(rng.integers(1, 5000))
        seed, gen = int(rng.integers(0, 2**40)), int(rng.integers(0, 500))
        pop = rng.integers(0, pool, (s, k)).astype(np.int32)
        f = rng.integers(0, 8, s).astype(float) if trial % 2 else rng.random(s)
        minimize = bool(trial % 3)
        assert np.array_equal(oracle.selection_weights(f, minimize), ref.selection_weights(f, minimize))
        idx, partners = ref.roulette_select(pop, f, minimize, seed, gen)
        assert np.array_equal(oracle.roulette_pick(f, minimize, seed, gen), idx)
        pc, pm = float(rng.random()), float(rng.random())
        crossed = ref.crossover(pop, partners, pc, seed, gen)
        assert np.array_equal(oracle.crossover(pop, idx, pc, seed, gen), crossed)
        assert np.array_equal(oracle.mutate_block(crossed, 0, pm, pool, seed, gen), ref.mutate(crossed, pm, pool, seed, gen))
        mp = rng.integers(0, pool, (s, k)).astype(np.int32)
        fm = rng.integers(0, 8, s).astype(float)
        a, b = oracle.elitism(pop, mp, f, fm, minimize)
        c, d = ref.elitism(pop, mp, f, fm, minimize)
        assert np.array_equal(a, c) and np.array_equal(b, d)
        ec = int(rng.integers(1, s + 1))
        assert np.array_equal(oracle.eda_sample(pop, ec, pool, seed, gen, trial % 2 == 0),
                              ref.eda_sample(pop, ec, pool, seed, gen, trial % 2 == 0))
    with pytest.raises(ValueError):
        oracle.elitism(pop, mp, [float("nan")] * s, fm, True)
    with pytest.raises(ValueError):
        ref.elitism(pop, mp, [float("nan")] * s, fm, True)


def test_trajectories_all_modes(oracle, ref):
    """test_parallel.cpp:86-116: the oracle loop equals the reference in serial, S and M modes."""
    og, rg = oracle.graph_ba(300, 2, 8), ref.graph_ba(300, 2, 8)
    want = oracle.run_ga(og, TASK_PC, 0.6, 0.2, 24, 15, 20, 77, eda_interval=4)
    for mode, pn in [(MODE_S, 1), (MODE_M, 3)]:
        got = ref.run_ga(rg, TASK_PC, 0.6, 0.2, 24, 15, 20, 77, eda_interval=4, mode=mode, pn=pn)
        for key in ("best", "mean", "population", "fitness"):
            assert np.array_equal(want[key], got[key]), (mode, key)


def test_sixdegrees_closure(oracle, ref):
    """sixdst_fitness(SixDegrees) (fitness.cpp:18-26, accessibility.cpp:20-37): radius-8 balls.
    Sparse graphs and paths so that the diameter exceeds 8 and the truncation matters
    (test_fitness.cpp:94-103 uses a 12-node path)."""
    rng = np.random.default_rng(11)
    truncated = 0
    for trial in range(60):
        n = int(rng.integers(4, 120))
        if trial % 3 == 0:  # a path plus a few chords
            e = np.stack([np.arange(n - 1), np.arange(1, n)], 1).astype(np.int32)
        else:
            e = _rand_edges(rng, n, float(rng.uniform(0.5, 2.5)) / n)
        og, rg = oracle.graph_from_edges(n, e), ref.graph_from_edges(n, e)
        batch = rng.integers(0, n, (4, int(rng.integers(0, max(1, n // 6) + 1)))).astype(np.int32)
        six = oracle.eval_batch(og, TASK_SIXDST, batch)
        assert np.array_equal(six, ref.eval_batch(rg, TASK_SIXDST, batch))
        exact = oracle.eval_batch(og, TASK_MCN, batch)
        assert np.all(six <= exact)
        truncated += int(np.any(six < exact))
    assert truncated > 10  # the sweep really exercises the radius-8 cut


def test_edge_addition_pool_and_cda(oracle, ref):
    """EdgeAddition pools (gene_pool.cpp:57-60, :81-87) under cda_fitness."""
    rng = np.random.default_rng(12)
    for trial in range(25):
        n = int(rng.integers(5, 70))
        e = _rand_edges(rng, n, float(rng.uniform(0.0, 0.3)) if trial else 0.0)  # trial 0: edgeless graph
        og, rg = oracle.graph_from_edges(n, e), ref.graph_from_edges(n, e)
        u, v = oracle.addition_pool(og)
        ru, rv = ref.pool_genes(rg, 1)
        assert np.array_equal(u, ru) and np.array_equal(v, rv)
        assert len(u) == n * (n - 1) // 2 - len(e)
        cols = int(rng.integers(0, 40))
        batch = rng.integers(0, len(u), (3, cols)).astype(np.int32)
        if cols > 2:
            batch[0, 1] = batch[0, 0]  # duplicate gene: idempotent
        assert np.array_equal(oracle.eval_batch(og, TASK_CDA_ADD, batch), ref.eval_batch(rg, TASK_CDA_ADD, batch))
    og, rg = oracle.graph_sbm(4, 30, 0.3, 0.02, 2), ref.graph_sbm(4, 30, 0.3, 0.02, 2)
    oracle.addition_pool(og)
    a = oracle.run_ga(og, TASK_CDA_ADD, 0.8, 0.1, 8, 12, 4, 3)
    b = ref.run_ga(rg, TASK_CDA_ADD, 0.8, 0.1, 8, 12, 4, 3)
    assert np.array_equal(a["best"], b["best"]) and np.array_equal(a["mean"], b["mean"])
    assert np.array_equal(a["population"], b["population"])


def test_mask_matrices_oracle_equals_reference(oracle, ref):
    import numpy as np
    rng = np.random.default_rng(31)
    for _ in range(25):
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 90))
        rate, seed, gen = float(rng.uniform(0, 1)), int(rng.integers(0, 2**62)), int(rng.integers(0, 500))
        for role in (3, 4):
            assert np.array_equal(oracle.make_mask(rows, cols, rate, role, seed, gen), ref.make_mask(rows, cols, rate, role, seed, gen))
        pool = int(rng.integers(1, 2_000_000_000))
        assert np.array_equal(oracle.make_mutation_indices(rows, cols, pool, seed, gen), ref.make_mutation_indices(rows, cols, pool, seed, gen))
