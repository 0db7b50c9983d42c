"""PC / MCN fitness: CUDA path vs the oracle, bit-exact (integers).

Mirrors tests/test_fitness.cpp:132-162 and acceptance.cpp:83-105 of the reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["warp-per-individual", "bit-sliced", "union-find"], autouse=True)
def pc_path(request, monkeypatch):
    """Every case runs through all three PC implementations: the shared-memory kernel that small graphs take by default, the
    bit-sliced pipeline (forced here; the default above n = 2048-4096, see pc_kernels.cu small_pays) and the per-individual
    union-find in global memory (k_pc_uf: what a context switches to, by measurement, on graphs without a hub core)."""
    monkeypatch.setenv("GAPA_PC_SMALL", "2" if request.param == "warp-per-individual" else "0")
    monkeypatch.setenv("GAPA_PC_UF", "1" if request.param == "union-find" else "0")
    return request.param


def _objective(gp, graph, task):
    pool = gp.build_gene_pool(graph, gp.PoolKind.NodeRemoval)
    cls = gp.PairwiseConnectivityObjective if task == 0 else gp.SixDstObjective
    return cls(graph, pool), pool


def _random_graph(rng, n, density):
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < density
    return np.stack([iu[0][keep], iu[1][keep]], axis=1).astype(np.int32)


@pytest.mark.parametrize("task", [0, 1])
def test_config1_known_answers(gp, oracle, cuda_device, task):
    g = gp.barabasi_albert(1000, 2, 1)
    obj, pool = _objective(gp, g, task)
    pop = gp.init_population(pool.size(), 4, 50, 1)
    got = obj.evaluate_batch(pop)
    want = [447931, 449826, 450775, 450775] if task == 0 else [947, 949, 950, 950]  # SURVEY §8c KATs
    assert got.tolist() == want
    og = oracle.graph_from_edges(g.n, g.edges())
    assert np.array_equal(got, oracle.eval_batch(og, task, pop))


@pytest.mark.parametrize("task", [0, 1])
def test_random_instances_exact(gp, oracle, cuda_device, task):
    """50 random ER graphs x several individuals, like test_fitness.cpp:132-152."""
    rng = np.random.default_rng(7 + task)
    for trial in range(50):
        n = int(rng.integers(4, 90))
        edges = _random_graph(rng, n, float(rng.uniform(0.01, 0.3)))
        g = gp.Graph(n, edges)
        obj, pool = _objective(gp, g, task)
        k = int(rng.integers(0, n + 1))
        rows = int(rng.integers(1, 70))
        batch = rng.integers(0, n, size=(rows, k)).astype(np.int32)
        og = oracle.graph_from_edges(n, edges)
        assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, task, batch)), (trial, n, k, rows)


def test_fixed_values(gp, cuda_device):
    """K5 -> 10, all removed -> 0 (test_fitness.cpp:154-162); MCN of all-removed is 1."""
    n = 5
    edges = [(u, v) for u in range(n) for v in range(u + 1, n)]
    g = gp.Graph(n, edges)
    pc, _ = _objective(gp, g, 0)
    mcn, _ = _objective(gp, g, 1)
    assert pc.evaluate_batch(np.zeros((1, 0), np.int32)).tolist() == [10.0]
    assert pc.evaluate_one(np.arange(5)) == 0.0
    assert mcn.evaluate_one(np.arange(5)) == 1.0
    assert mcn.evaluate_one([]) == 5.0
    assert pc.evaluate_one([0, 0, 0]) == 6.0  # duplicates are idempotent: K4 left
    assert pc.evaluate_batch(np.zeros((0, 3), np.int32)).shape == (0,)


def test_fragmented_graphs_use_union_find(gp, oracle, cuda_device):
    """Paths, rings, stars and disjoint cliques leave most vertices outside the BFS giant."""
    rng = np.random.default_rng(3)
    n = 3000
    path = np.stack([np.arange(n - 1), np.arange(1, n)], axis=1)
    perm = rng.permutation(n)
    shuffled_path = perm[path]
    cliques = np.array([(b * 6 + i, b * 6 + j) for b in range(n // 6) for i in range(6) for j in range(i + 1, 6)])
    star = np.stack([np.zeros(n - 1, int), np.arange(1, n)], axis=1)
    for edges in (path, shuffled_path, cliques, star):
        g = gp.Graph(n, edges)
        og = oracle.graph_from_edges(n, edges)
        batch = rng.integers(0, n, size=(130, 40)).astype(np.int32)
        for task in (0, 1):
            obj, _ = _objective(gp, g, task)
            assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, task, batch))


def test_ragged_group_sizes_and_purity(gp, oracle, cuda_device):
    g = gp.barabasi_albert(2000, 3, 5)
    og = oracle.graph_from_edges(g.n, g.edges())
    obj, pool = _objective(gp, g, 0)
    for rows in (1, 63, 64, 65, 127, 129, 200):
        batch = gp.init_population(pool.size(), rows, 100, rows)
        before = batch.copy()
        got = obj.evaluate_batch(batch)
        assert np.array_equal(batch, before)  # inputs never mutated (test_fitness.cpp:396-409)
        assert np.array_equal(got, oracle.eval_batch(og, 0, batch))
        assert np.array_equal(got, obj.evaluate_batch(batch))  # re-entrant, same answer


def test_custom_node_pool_and_errors(gp, oracle, cuda_device):
    g = gp.barabasi_albert(300, 2, 9)
    og = oracle.graph_from_edges(g.n, g.edges())
    sub = np.arange(0, 300, 3, dtype=np.int32)  # pool over every third node
    pool = gp.GenePool(gp.PoolKind.NodeRemoval, sub)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    batch = np.random.default_rng(1).integers(0, len(sub), size=(10, 20)).astype(np.int32)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, 0, sub[batch]))
    with pytest.raises(gp.capi.GapaCudaError) as e:
        obj.evaluate_batch(np.full((2, 3), len(sub), np.int32))
    assert e.value.code == gp.capi.E_RANGE
    with pytest.raises(gp.capi.GapaCudaError):
        gp.PairwiseConnectivityObjective(g, gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval))


def test_medium_power_law_graph(gp, oracle, cuda_device):
    """n = 1e5 BA graph, 5 % removal: the bit-sliced giant sweep + leftovers, vs the CSR oracle."""
    g = gp.barabasi_albert(100_000, 5, 1)
    og = oracle.graph_from_edges(g.n, g.edges())
    obj, pool = _objective(gp, g, 0)
    batch = gp.init_population(pool.size(), 96, 5000, 1)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, 0, batch, threads=8))


def test_shuffled_labels_use_the_hub_first_internal_order(gp, oracle, cuda_device, pc_path, monkeypatch):
    """A power-law graph whose labels carry no structure: the bit-sliced path relabels by degree
    internally (automatic here; forced on and off as well) and must return the same integers."""
    rng = np.random.default_rng(12)
    base = gp.barabasi_albert(20_000, 3, 2)
    perm = rng.permutation(base.n).astype(np.int32)
    edges = perm[base.edges()]
    g = gp.Graph(base.n, edges)
    og = oracle.graph_from_edges(g.n, edges)
    batch = rng.integers(0, g.n, size=(70, 900)).astype(np.int32)
    want_pc, want_mcn = oracle.eval_batch(og, 0, batch, threads=8), oracle.eval_batch(og, 1, batch, threads=8)
    sub = np.sort(rng.choice(g.n, 5000, replace=False)).astype(np.int32)  # custom pool composed with the relabelling
    for relabel in ("-1", "1", "0"):
        monkeypatch.setenv("GAPA_PC_RELABEL", relabel)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        assert np.array_equal(gp.PairwiseConnectivityObjective(g, pool).evaluate_batch(batch), want_pc)
        assert np.array_equal(gp.SixDstObjective(g, pool).evaluate_batch(batch), want_mcn)
        obj = gp.PairwiseConnectivityObjective(g, gp.GenePool(gp.PoolKind.NodeRemoval, sub))
        genes = rng.integers(0, len(sub), size=(9, 300)).astype(np.int32)
        assert np.array_equal(obj.evaluate_batch(genes), oracle.eval_batch(og, 0, sub[genes]))


def test_sparse_random_graphs_without_a_hub_core(gp, oracle, cuda_device, monkeypatch):
    """Erdos-Renyi graphs near the percolation threshold: one sweep leaves most of the graph unreached, the
    recording sweep defers itself and more sweep rounds run before phase 2 — same integers as the oracle."""
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    rng = np.random.default_rng(5)
    for n, deg, rows in ((40_000, 3.0, 70), (25_000, 1.6, 130), (60_000, 4.5, 64)):
        e = rng.integers(0, n, (int(n * deg / 2), 2)).astype(np.int32)
        e = e[e[:, 0] != e[:, 1]]
        e.sort(axis=1)
        e = np.unique(e, axis=0)
        g = gp.Graph(n, e)
        og = oracle.graph_from_edges(n, e)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        batch = gp.init_population(pool.size(), rows, n // 20, 3)
        for task, cls in ((0, gp.PairwiseConnectivityObjective), (1, gp.SixDstObjective)):
            assert np.array_equal(cls(g, pool).evaluate_batch(batch), oracle.eval_batch(og, task, batch, threads=8)), (n, task)


def test_high_diameter_graphs(gp, oracle, cuda_device, monkeypatch):
    """Rings and grids: reachability needs many sweep rounds (descending + ascending, blocks iterating their chunk
    to a local fixpoint) and a large phase 2 — there is no giant component after 5 % removals on a ring."""
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    n = 30_000
    ring = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).astype(np.int32)
    side = 140
    idx = np.arange(side * side).reshape(side, side)
    grid = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                           np.stack([idx[:-1].ravel(), idx[1:].ravel()], 1)]).astype(np.int32)
    for name, nn, e, k in (("ring", n, ring, n // 20), ("ring, nothing removed", n, ring, 0), ("grid", side * side, grid, side * side // 10)):
        g = gp.Graph(nn, e)
        og = oracle.graph_from_edges(nn, e)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        batch = gp.init_population(pool.size(), 70, k, 4) if k else np.zeros((3, 0), np.int32)
        for task, cls in ((0, gp.PairwiseConnectivityObjective), (1, gp.SixDstObjective)):
            assert np.array_equal(cls(g, pool).evaluate_batch(batch), oracle.eval_batch(og, task, batch, threads=8)), (name, task)


@pytest.mark.parametrize("env", [
    {},                                                                  # speculative schedule, one lane, k_pc_final
    {"GAPA_PC_SPEC_ROUNDS": "0"},                                        # host-driven loop only
    {"GAPA_PC_PHASE2_BIG": "1"},                                         # full-grid phase 2 inside the speculative schedule
    {"GAPA_PC_LANE_ROWS": "64", "GAPA_PC_LANE_STREAMS": "3"},            # many lanes on three streams, sets reused
    {"GAPA_PC_LANE_ROWS": "128", "GAPA_PC_LANE_STREAMS": "2", "GAPA_PC_SPEC_ROUNDS": "3"},
    {"GAPA_PC_FOLD_CLEAR_MB": "0", "GAPA_PC_PREFIX": "0"},               # clear and source selection as launches of their own
    {"GAPA_PC_FOLD_CLEAR_MB": "0", "GAPA_PC_OVERLAP_CLEAR": "0"},
], ids=["default", "host-driven", "phase2-big", "lanes64x3", "lanes128x2-spec3", "noclearfold-noprefix", "noclearfold-inline"])
def test_every_schedule_gives_the_oracles_integers(gp, oracle, cuda_device, monkeypatch, env):
    """The lane / speculation / fusion knobs only change HOW the pipeline is scheduled.  One objective is evaluated
    repeatedly with growing and shrinking batches (the scratch sets are left clean by k_pc_final and reused), on a
    power-law graph (nothing left for phase 2), on disjoint cliques (everything is phase 2: more entries than
    k_pc_final takes on, so the schedule learns to use the full-grid kernels) and on a sparse random graph (the
    speculative schedule stands down, the host-driven loop takes over and teaches it the rounds it needs)."""
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    for key, value in env.items():
        monkeypatch.setenv(key, value)
    rng = np.random.default_rng(21)
    n = 6000
    cliques = np.array([(b * 6 + i, b * 6 + j) for b in range(n // 6) for i in range(6) for j in range(i + 1, 6)], dtype=np.int32)
    ne = 30_000
    er = rng.integers(0, ne, (int(ne * 1.8 / 2), 2)).astype(np.int32)
    er = er[er[:, 0] != er[:, 1]]
    er.sort(axis=1)
    er = np.unique(er, axis=0)
    ba = gp.barabasi_albert(20_000, 4, 3)
    for graph in (ba, gp.Graph(n, cliques), gp.Graph(ne, er)):
        og = oracle.graph_from_edges(graph.n, graph.edges())
        pool = gp.build_gene_pool(graph, gp.PoolKind.NodeRemoval)
        pc, mcn = gp.PairwiseConnectivityObjective(graph, pool), gp.SixDstObjective(graph, pool)
        for rows in (70, 300, 64, 513, 1):
            batch = gp.init_population(pool.size(), rows, graph.n // 20, rows)
            assert np.array_equal(pc.evaluate_batch(batch), oracle.eval_batch(og, 0, batch, threads=8)), (graph.n, rows)
            assert np.array_equal(mcn.evaluate_batch(batch), oracle.eval_batch(og, 1, batch, threads=8)), (graph.n, rows)


def test_high_diameter_graph_switches_to_union_find(gp, oracle, cuda_device, monkeypatch):
    """A ring has no hub core: the pipeline's speculative schedule stands down, the context times both algorithms on that
    batch and keeps the faster one; whichever it is, every evaluation before, during and after the switch equals the oracle."""
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    monkeypatch.delenv("GAPA_PC_UF", raising=False)  # automatic
    n = 20000
    ring = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).astype(np.int32)
    g = gp.Graph(n, ring)
    for task in (0, 1):
        obj, pool = _objective(gp, g, task)
        og = oracle.graph_from_edges(n, ring)
        for trial in range(3):
            batch = gp.init_population(pool.size(), 128, 1000, 10 + trial)
            assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, task, batch)), (task, trial)
