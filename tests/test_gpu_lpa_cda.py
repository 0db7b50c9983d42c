"""LPA (RA-AUC) and CDA (greedy-detector modularity) fitness: CUDA path vs the oracle.

Bit-exact FP64 is the bar: identical GA trajectories need identical ties.
Mirrors tests/test_fitness.cpp:279-307 (CDA identities), :336-394 (RA / AUC / LPA)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _edge_pool(gp, g):
    return gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)


# ------------------------------------------------------------------------------- LPA
def test_lpa_known_answers(gp, oracle, cuda_device):
    g = gp.erdos_renyi(500, 0.03, 1)
    split = gp.build_lp_split(g, 0.1, 1)
    pool = _edge_pool(gp, split.train)
    k = gp.perturbation_budget(split.train, gp.PoolKind.EdgeRemoval, 0.1)
    assert (g.edge_count(), len(split.test_edges), split.train.edge_count(), k) == (3709, 371, 3338, 334)
    obj = gp.LinkPredictionAttackObjective(split, pool)
    pop = gp.init_population(pool.size(), 3, k, 1)
    got = obj.evaluate_batch(pop)
    assert got.tolist() == [0.50374525032512119, 0.49914632994529246, 0.51192595229619087]  # SURVEY §8c KATs
    assert obj.evaluate_one([]) == 0.50795184574363739  # empty perturbation == unattacked, exactly
    og = oracle.graph_from_edges(g.n, g.edges())
    os_ = oracle.split_build(og, 0.1, 1)
    assert np.array_equal(got, oracle.eval_batch(os_, 3, pop))


def test_lpa_random_instances_exact(gp, oracle, cuda_device):
    rng = np.random.default_rng(21)
    for trial in range(12):
        n = int(rng.integers(30, 400))
        g = gp.erdos_renyi(n, float(rng.uniform(0.03, 0.2)), trial + 1)
        if g.edge_count() < 20:
            continue
        frac = float(rng.uniform(0.05, 0.5))
        split = gp.build_lp_split(g, frac, trial)
        pool = _edge_pool(gp, split.train)
        obj = gp.LinkPredictionAttackObjective(split, pool)
        os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), frac, trial)
        rows, k = int(rng.integers(1, 40)), int(rng.integers(0, pool.size() + 1))
        batch = rng.integers(0, pool.size(), size=(rows, k)).astype(np.int32)
        assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(os_, 3, batch)), trial


def test_lpa_all_removed_is_half(gp, cuda_device):
    g = gp.barabasi_albert(200, 3, 2)
    split = gp.build_lp_split(g, 0.2, 3)
    pool = _edge_pool(gp, split.train)
    obj = gp.LinkPredictionAttackObjective(split, pool)
    assert obj.evaluate_one(np.arange(pool.size())) == 0.5  # test_fitness.cpp:378-394
    with pytest.raises(gp.capi.GapaCudaError):
        gp.LinkPredictionAttackObjective(split, gp.build_gene_pool(split.train, gp.PoolKind.NodeRemoval))
    with pytest.raises(gp.capi.GapaCudaError) as e:
        obj.evaluate_one([pool.size()])
    assert e.value.code == gp.capi.E_RANGE


# ------------------------------------------------------------------------------- CDA
def test_cda_known_answers(gp, oracle, cuda_device):
    g = gp.planted_partition(10, 50, 0.2, 0.01, 1)
    pool = _edge_pool(gp, g)
    k = gp.perturbation_budget(g, gp.PoolKind.EdgeRemoval, 0.05)
    assert (g.n, g.edge_count(), k) == (500, 3668, 184)
    obj = gp.ModularityAttackObjective(g, pool)
    pop = gp.init_population(pool.size(), 3, k, 1)
    got = obj.evaluate_batch(pop)
    assert got.tolist() == [0.52118299521350409, 0.53218590159358303, 0.50903959381049579]  # SURVEY §8c KATs
    assert obj.evaluate_one([]) == 0.51897794328383418  # empty perturbation == unattacked Q exactly
    og = oracle.graph_from_edges(g.n, g.edges())
    assert np.array_equal(got, oracle.eval_batch(og, 2, pop))


def test_cda_identities(gp, cuda_device):
    two_triangles = gp.Graph(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    pool = _edge_pool(gp, two_triangles)
    obj = gp.ModularityAttackObjective(two_triangles, pool)
    assert obj.evaluate_one([]) == 0.5
    assert obj.evaluate_one(np.arange(pool.size())) == -0.5  # all edges removed: the floor, exactly
    assert obj.evaluate_batch(np.zeros((0, 2), np.int32)).shape == (0,)
    with pytest.raises(gp.capi.GapaCudaError):
        gp.ModularityAttackObjective(two_triangles, gp.build_gene_pool(two_triangles, gp.PoolKind.NodeRemoval))


@pytest.mark.parametrize("argmax", ["two-level", "flat"])
def test_cda_random_instances_exact(gp, oracle, cuda_device, monkeypatch, argmax):
    monkeypatch.setenv("GAPA_CDA_HIER", "1" if argmax == "two-level" else "0")  # both forms of the cached-best argmax
    rng = np.random.default_rng(4)
    for trial in range(25):
        n = int(rng.integers(6, 160))
        kind = trial % 3
        if kind == 0:
            g = gp.erdos_renyi(n, float(rng.uniform(0.03, 0.3)), trial + 1)
        elif kind == 1:
            g = gp.barabasi_albert(n, int(rng.integers(1, 4)), trial + 1)
        else:
            g = gp.planted_partition(int(rng.integers(2, 6)), int(rng.integers(5, 30)), 0.4, 0.03, trial + 1)
        if g.edge_count() == 0:
            continue
        pool = _edge_pool(gp, g)
        obj = gp.ModularityAttackObjective(g, pool)
        og = oracle.graph_from_edges(g.n, g.edges())
        rows, k = int(rng.integers(1, 12)), int(rng.integers(0, pool.size() + 1))
        batch = rng.integers(0, pool.size(), size=(rows, k)).astype(np.int32)
        got, want = obj.evaluate_batch(batch), oracle.eval_batch(og, 2, batch)
        assert np.array_equal(got, want), (trial, np.abs(got - want).max())


def test_cda_tie_heavy_graphs_same_partition(gp, oracle, cuda_device):
    """Regular graphs are all ties: many candidate pairs share one gain, so the reference's scan order (greatest gain, then
    smallest a, then smallest b) decides every merge.  The detector's PARTITION — the merge order made visible — must equal
    the oracle's, for the empty perturbation and for random removals."""
    rng = np.random.default_rng(11)
    graphs = []
    for n in (8, 13, 30, 64):  # rings
        graphs.append((n, [(i, (i + 1) % n) for i in range(n)]))
    for w, h in ((3, 4), (5, 5), (6, 9)):  # grids
        e = [(y * w + x, y * w + x + 1) for y in range(h) for x in range(w - 1)] + [(y * w + x, (y + 1) * w + x) for y in range(h - 1) for x in range(w)]
        graphs.append((w * h, e))
    for a, b in ((3, 3), (4, 6)):  # complete bipartite
        graphs.append((a + b, [(i, a + j) for i in range(a) for j in range(b)]))
    graphs.append((12, [(i, j) for i in range(6) for j in range(i + 1, 6)] + [(6 + i, 6 + j) for i in range(6) for j in range(i + 1, 6)] + [(0, 6)]))  # two cliques
    for n, edges in graphs:
        g = gp.Graph(n, np.asarray(edges, np.int32))
        pool = _edge_pool(gp, g)
        obj = gp.ModularityAttackObjective(g, pool)
        og = oracle.graph_from_edges(g.n, g.edges())
        for trial in range(6):
            k = 0 if trial == 0 else int(rng.integers(1, max(2, pool.size() // 2)))
            genes = rng.integers(0, pool.size(), size=k).astype(np.int32)
            want_q = oracle.eval_batch(og, 2, genes.reshape(1, -1))
            assert np.array_equal(obj.evaluate_batch(genes.reshape(1, -1)), want_q), (n, trial)
            from paper_2412_20980_b200.experiment import _detect
            owner = _detect(obj.dgraph, genes)
            kept = [e for i, e in enumerate(g.sorted_edges().tolist()) if i not in set(genes.tolist())]
            want_owner = oracle.detect_communities(oracle.graph_from_edges(g.n, np.asarray(kept, np.int32).reshape(-1, 2)))
            assert np.array_equal(_first_appearance(owner), _first_appearance(want_owner)), (n, trial)


def _first_appearance(owner):
    seen, out = {}, []
    for o in np.asarray(owner).tolist():
        out.append(seen.setdefault(o, len(seen)))
    return np.asarray(out)


def test_cda_more_individuals_than_sms(gp, oracle, cuda_device):
    g = gp.planted_partition(4, 25, 0.3, 0.02, 7)
    pool = _edge_pool(gp, g)
    obj = gp.ModularityAttackObjective(g, pool)
    og = oracle.graph_from_edges(g.n, g.edges())
    batch = gp.init_population(pool.size(), 400, 12, 3)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, 2, batch, threads=8))


def test_cda_config2_whole_population(gp, oracle, cuda_device):
    """BASELINE configs[1] at its own size: SBM 10 x 500, 5 % edge deletion, all 100 individuals of the population
    against the oracle, bit-exact FP64."""
    g = gp.planted_partition(10, 500, 0.02, 0.0005, 1)
    pool = _edge_pool(gp, g)
    k = gp.perturbation_budget(g, gp.PoolKind.EdgeRemoval, 0.05)
    assert (g.edge_count(), k) == (30321, 1517)
    og = oracle.graph_from_edges(g.n, g.edges())
    batch = gp.init_population(pool.size(), 100, k, 1)
    got = gp.ModularityAttackObjective(g, pool).evaluate_batch(batch)
    assert np.array_equal(got, oracle.eval_batch(og, 2, batch, threads=16))
    assert len(np.unique(got)) > 90  # the individuals really differ


def test_cda_config2_sample(gp, oracle, cuda_device):
    """BASELINE config 2 shape: SBM 10 x 500, 5 % edge deletion (2 individuals vs the oracle)."""
    g = gp.planted_partition(10, 500, 0.02, 0.0005, 1)
    assert g.edge_count() == 30321
    pool = _edge_pool(gp, g)
    k = gp.perturbation_budget(g, gp.PoolKind.EdgeRemoval, 0.05)
    obj = gp.ModularityAttackObjective(g, pool)
    assert obj.evaluate_one([]) == 0.61708453864200974  # BASELINE.md §2, unattacked Q
    og = oracle.graph_from_edges(g.n, g.edges())
    batch = gp.init_population(pool.size(), 2, k, 1)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, 2, batch, threads=2))


@pytest.mark.parametrize("sorted_auc", ["1", "0"])
def test_lpa_auc_paths_agree_with_the_oracle(gp, oracle, cuda_device, monkeypatch, sorted_auc):
    """The AUC's 2*wins comes from a shared-memory sort + binary searches, or (probe set too large, or
    GAPA_LPA_SORTED_AUC=0) from the T x P grid; both must give the oracle's double.  Sparse graphs make most
    RA scores exactly 0 — the tie term carries the result."""
    monkeypatch.setenv("GAPA_LPA_SORTED_AUC", sorted_auc)
    rng = np.random.default_rng(77)
    for n, p, frac in ((600, 0.004, 0.3), (3000, 0.004, 0.1), (90, 0.3, 0.5)):
        g = gp.erdos_renyi(n, p, 5)
        split = gp.build_lp_split(g, frac, 9)
        pool = _edge_pool(gp, split.train)
        obj = gp.LinkPredictionAttackObjective(split, pool)
        os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), frac, 9)
        batch = rng.integers(0, pool.size(), size=(7, pool.size() // 5)).astype(np.int32)
        assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(os_, 3, batch)), (n, sorted_auc)
        assert obj.evaluate_one([]) == oracle.eval_batch(os_, 3, np.zeros((1, 0), np.int32))[0]


def test_lpa_probe_set_beyond_shared_memory_uses_the_grid(gp, oracle, cuda_device):
    g = gp.erdos_renyi(4000, 0.02, 3)  # m ~ 160 k, T = P ~ 64 k > 25,600 keys of shared memory
    split = gp.build_lp_split(g, 0.4, 4)
    assert len(split.probe_nonedges) > 25600
    pool = _edge_pool(gp, split.train)
    obj = gp.LinkPredictionAttackObjective(split, pool)
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.4, 4)
    batch = gp.init_population(pool.size(), 2, 2000, 8)
    assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(os_, 3, batch, threads=2))


# ---- north_star extensions without a reference implementation: PARITY UNPINNED (twins in oracle/gapa_oracle.c) ----
def test_cn_score_and_edge_flip_pools_match_their_cpu_twin(gp, oracle, cuda_device):
    """CN link score and edge-flip pools for the link-prediction attack (BASELINE.json north_star; the reference has RA
    with edge-removal pools only).  The CUDA path is held to the CPU twin that STATES the semantics — parity unpinned:
    there is no reference output to pin either against.  What IS pinned: the twin, restricted to what the reference
    has (RA, removals), equals the reference-pinned oracle bit for bit, and so does the CUDA flip path fed an
    edges-only flip pool."""
    rng = np.random.default_rng(8)
    for n, p, frac in ((400, 0.03, 0.2), (1500, 0.006, 0.1), (90, 0.25, 0.3)):
        g = gp.erdos_renyi(n, p, 3)
        split = gp.build_lp_split(g, frac, 4)
        og = oracle.graph_from_edges(g.n, g.edges())
        os_ = oracle.split_build(og, frac, 4)
        rem = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
        k = max(4, rem.size() // 8)
        rb = rng.integers(0, rem.size(), size=(9, k)).astype(np.int32)
        # CN with the reference's removal pools
        cn = gp.LinkPredictionAttackObjective(split, rem, score=gp.LinkScore.CN)
        assert np.array_equal(cn.evaluate_batch(rb), oracle.lpa_scored_batch(os_, rb, 1))
        assert np.array_equal(oracle.lpa_scored_batch(os_, rb, 0), oracle.eval_batch(os_, 3, rb))  # the twin == the pinned RA path
        # the canonical flip pool: every node pair, genes unranked on the device
        flip = gp.build_gene_pool(split.train, gp.PoolKind.EdgeFlip)
        assert flip.size() == n * (n - 1) // 2
        fb = rng.integers(0, flip.size(), size=(9, k)).astype(np.int32)
        fb[:, :k // 2] = fb[:, k // 2:2 * (k // 2)]  # repeated genes are idempotent
        edge_ids = np.array([a * n - a * (a + 1) // 2 + (b - a - 1) for a, b in zip(rem.u[:k // 3], rem.v[:k // 3])], np.int32)
        fb[0, :len(edge_ids)] = edge_ids               # a row that also removes real edges
        for score in (gp.LinkScore.RA, gp.LinkScore.CN):
            obj = gp.LinkPredictionAttackObjective(split, flip, score=score)
            assert np.array_equal(obj.evaluate_batch(fb), oracle.lpa_flip_batch(os_, fb, int(score))), (n, score)
            assert obj.evaluate_one([]) == oracle.lpa_flip_batch(os_, np.zeros((1, 0), np.int32), int(score))[0]
        # a custom flip pool that lists exactly the train edges behaves like the reference's removal pool (pinned)
        edges_only = gp.GenePool(gp.PoolKind.EdgeFlip, rem.u, rem.v)
        assert np.array_equal(gp.LinkPredictionAttackObjective(split, edges_only).evaluate_batch(rb), oracle.eval_batch(os_, 3, rb))
        # ... and a mixed custom pool against the twin
        pairs = np.stack([rng.integers(0, n, 300), rng.integers(0, n, 300)], 1)
        pairs = np.unique(np.sort(pairs[pairs[:, 0] != pairs[:, 1]], axis=1), axis=0).astype(np.int32)
        custom = gp.GenePool(gp.PoolKind.EdgeFlip, pairs[:, 0], pairs[:, 1])
        cb = rng.integers(0, len(pairs), size=(5, 60)).astype(np.int32)
        assert np.array_equal(gp.LinkPredictionAttackObjective(split, custom).evaluate_batch(cb), oracle.lpa_flip_batch(os_, cb, 0, pairs))
    with pytest.raises(gp.capi.GapaCudaError):
        gp.ModularityAttackObjective(g, gp.build_gene_pool(g, gp.PoolKind.EdgeFlip))  # flips are a link-prediction pool


def test_edge_flip_ga_run_is_reproducible_and_consistent(gp, oracle, cuda_device):
    """A GA over the flip pool with the CN score (the configs[2] wording): reproducible, monotone under elitism, and
    the stored fitness of the final population equals the CPU twin's evaluation of it (parity unpinned)."""
    g = gp.erdos_renyi(500, 0.03, 1)
    split = gp.build_lp_split(g, 0.1, 1)
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.1, 1)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeFlip)
    obj = gp.LinkPredictionAttackObjective(split, pool, score=gp.LinkScore.CN)
    params = gp.GAParams(pc=0.7, pm=0.1, pop_size=24, budget=40, iterations=6, seed=2, eda_interval=4)
    a, b = gp.run_ga(params, pool, obj), gp.run_ga(params, pool, obj)
    assert np.array_equal(a.history_best, b.history_best) and np.array_equal(a.final_population, b.final_population)
    assert np.all(np.diff(a.history_best) <= 0)
    assert np.array_equal(a.final_fitness, oracle.lpa_flip_batch(os_, a.final_population, 1))
