"""Edge cases the reference tests or implies: empty perturbations and batches, tiny and edgeless
graphs, budgets larger than the pool, custom (re-ordered) edge pools, CSR construction, argument
errors.  All through the C ABI, against the oracle."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_tiny_and_edgeless_graphs(gp, oracle, cuda_device):
    for n, edges in [(1, []), (2, []), (2, [(0, 1)]), (3, [(0, 2)]), (65, [(i, i + 1) for i in range(64)])]:
        g = gp.Graph(n, np.array(edges, dtype=np.int32).reshape(-1, 2))
        og = oracle.graph_from_edges(n, edges)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        batch = np.array([[0] * 3, [n - 1] * 3, [0, n - 1, n // 2]], dtype=np.int32)
        for task, cls in ((0, gp.PairwiseConnectivityObjective), (1, gp.SixDstObjective)):
            obj = cls(g, pool)
            assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(og, task, batch))
            assert obj.evaluate_batch(np.zeros((2, 0), np.int32)).tolist() == oracle.eval_batch(og, task, np.zeros((2, 0), np.int32)).tolist()


def test_budget_larger_than_pool_and_heavy_duplicates(gp, oracle, cuda_device):
    g = gp.barabasi_albert(40, 2, 3)
    og = oracle.graph_from_edges(g.n, g.edges())
    rng = np.random.default_rng(0)
    batch = rng.integers(0, g.n, size=(5, 400)).astype(np.int32)  # k = 10 n: almost everything removed, many duplicates
    assert np.array_equal(gp.PairwiseConnectivityObjective(g, gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)).evaluate_batch(batch),
                          oracle.eval_batch(og, 0, batch))
    pool = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
    ebatch = rng.integers(0, pool.size(), size=(5, 5 * pool.size())).astype(np.int32)
    got = gp.ModularityAttackObjective(g, pool).evaluate_batch(ebatch)
    assert np.array_equal(got, oracle.eval_batch(og, 2, ebatch))


def test_custom_edge_pool_order(gp, oracle, cuda_device):
    """A GenePool whose gene ids are NOT the (u,v)-sorted ranks: the C ABI maps (u, v) to CSR edge ranks."""
    g = gp.planted_partition(3, 20, 0.3, 0.05, 5)
    og = oracle.graph_from_edges(g.n, g.edges())
    base = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
    rng = np.random.default_rng(3)
    order = rng.permutation(base.size())[: base.size() // 2]  # a shuffled half of the edges
    flip = rng.random(len(order)) < 0.5                         # endpoints given in either order
    u = np.where(flip, base.v[order], base.u[order]).astype(np.int32)
    v = np.where(flip, base.u[order], base.v[order]).astype(np.int32)
    pool = gp.GenePool(gp.PoolKind.EdgeRemoval, u, v)
    genes = rng.integers(0, pool.size(), size=(6, 25)).astype(np.int32)
    want = oracle.eval_batch(og, 2, order[genes].astype(np.int32))
    assert np.array_equal(gp.ModularityAttackObjective(g, pool).evaluate_batch(genes), want)
    with pytest.raises(gp.capi.GapaCudaError):
        gp.ModularityAttackObjective(g, gp.GenePool(gp.PoolKind.EdgeRemoval, [0], [0]))  # not a node pair
    # pairs that are not edges of THIS graph are accepted and remove nothing (gene_pool.cpp:34-56: clearing an absent
    # bit) — the pool of the full graph evaluated on a sub-graph; a repeated pair is still rejected (:36-41)
    have = {(int(a), int(b)) for a, b in zip(base.u, base.v)}
    absent = [(a, b) for a in range(g.n) for b in range(a + 1, g.n) if (a, b) not in have][:40]
    u2 = np.concatenate([u, np.array([a for a, _ in absent], np.int32)])
    v2 = np.concatenate([v, np.array([b for _, b in absent], np.int32)])
    mixed = gp.GenePool(gp.PoolKind.EdgeRemoval, u2, v2)
    genes2 = rng.integers(0, mixed.size(), size=(6, 30)).astype(np.int32)
    as_ranks = np.where(genes2 < len(order), order[np.minimum(genes2, len(order) - 1)], order[genes2[:, :1] % len(order)])
    as_ranks = np.where(genes2 < len(order), as_ranks, as_ranks[:, :1])  # an absent pair == a repeat of a present gene (idempotent)
    keep = genes2[:, 0] < len(order)  # rows whose first gene is a real edge can stand in for the no-ops
    assert keep.any()
    got2 = gp.ModularityAttackObjective(g, mixed).evaluate_batch(genes2[keep])
    assert np.array_equal(got2, oracle.eval_batch(og, 2, as_ranks[keep].astype(np.int32)))
    split = gp.build_lp_split(g, 0.2, 3)
    full_pool = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)  # built on the FULL graph, evaluated on split.train
    lobj = gp.LinkPredictionAttackObjective(split, full_pool)
    tr = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    rank_in_train = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(tr.u, tr.v))}
    rows = []
    for _ in range(5):
        ids = rng.integers(0, full_pool.size(), size=20)
        mapped = [rank_in_train[(int(full_pool.u[i]), int(full_pool.v[i]))] for i in ids if (int(full_pool.u[i]), int(full_pool.v[i])) in rank_in_train]
        if not mapped:
            continue
        mapped = (mapped * 20)[:20]  # repeats are idempotent
        rows.append((ids.astype(np.int32), np.array(mapped, np.int32)))
    os_ = oracle.split_build(og, 0.2, 3)
    got3 = lobj.evaluate_batch(np.stack([a for a, _ in rows]))
    assert np.array_equal(got3, oracle.eval_batch(os_, 3, np.stack([b for _, b in rows])))
    with pytest.raises(gp.capi.GapaCudaError):
        gp.ModularityAttackObjective(g, gp.GenePool(gp.PoolKind.EdgeRemoval, [absent[0][0], absent[0][1]], [absent[0][1], absent[0][0]]))


def test_csr_constructor_and_argument_errors(gp, oracle, cuda_device):
    lib = gp.capi.load()
    og = oracle.graph_ba(200, 2, 1)
    h = C.c_void_p()
    rp, ci = np.ascontiguousarray(og.row_ptr), np.ascontiguousarray(og.col_idx)
    gp.capi.check(lib.gapa_cuda_graph_create_csr(og.n, og.m, rp.ctypes.data, ci.ctypes.data, 0, C.byref(h)))
    genes = oracle.init_population(og.n, 70, 10, 2)
    out = np.zeros(70)
    gp.capi.check(lib.gapa_cuda_eval_batch(h, 0, genes.ctypes.data, 70, 10, out.ctypes.data))
    assert np.array_equal(out, oracle.eval_batch(og, 0, genes))
    n_, m_, dev = C.c_int32(), C.c_int64(), C.c_int()
    gp.capi.check(lib.gapa_cuda_graph_info(h, C.byref(n_), C.byref(m_), C.byref(dev)))
    assert (n_.value, m_.value, dev.value) == (og.n, og.m, 0)
    assert lib.gapa_cuda_eval_batch(h, 2, genes.ctypes.data, 70, 10, out.ctypes.data) == gp.capi.E_INVALID  # CDA on a node pool
    assert lib.gapa_cuda_eval_batch(h, 9, genes.ctypes.data, 70, 10, out.ctypes.data) == gp.capi.E_INVALID
    assert lib.gapa_cuda_eval_batch(h, 0, genes.ctypes.data, -1, 10, out.ctypes.data) == gp.capi.E_INVALID
    assert b"unknown" in lib.gapa_cuda_last_error() or b"negative" in lib.gapa_cuda_last_error()
    lib.gapa_cuda_destroy(h)
    bad = ci.copy()
    bad[0], bad[1] = bad[1], bad[0]  # row 0 no longer ascending
    assert lib.gapa_cuda_graph_create_csr(og.n, og.m, rp.ctypes.data, bad.ctypes.data, 0, C.byref(h)) == gp.capi.E_INVALID
    for edges in ([(0, 0)], [(0, 1), (1, 0)], [(0, 7)]):  # self-loop, duplicate, out of range (graph.cpp:26-31)
        e = np.array(edges, dtype=np.int32)
        assert lib.gapa_cuda_graph_create(5, len(e), e.ctypes.data, 0, C.byref(h)) == gp.capi.E_INVALID
    assert lib.gapa_cuda_graph_create(5, 0, None, 99, C.byref(h)) == gp.capi.E_INVALID  # no such device


def test_lpa_edge_cases(gp, oracle, cuda_device):
    g = gp.barabasi_albert(60, 2, 8)
    split = gp.build_lp_split(g, 0.5, 2)  # largest allowed test fraction
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.5, 2)
    pool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    obj = gp.LinkPredictionAttackObjective(split, pool)
    rng = np.random.default_rng(4)
    for k in (0, 1, pool.size(), 3 * pool.size()):
        batch = rng.integers(0, pool.size(), size=(3, k)).astype(np.int32)
        assert np.array_equal(obj.evaluate_batch(batch), oracle.eval_batch(os_, 3, batch)), k


def test_two_contexts_and_repeated_calls(gp, oracle, cuda_device):
    """Two objectives on different graphs, interleaved calls, growing and shrinking batches."""
    ga, gb = gp.barabasi_albert(3000, 3, 1), gp.erdos_renyi(400, 0.02, 2)
    oa, ob = oracle.graph_from_edges(ga.n, ga.edges()), oracle.graph_from_edges(gb.n, gb.edges())
    a = gp.PairwiseConnectivityObjective(ga, gp.build_gene_pool(ga, gp.PoolKind.NodeRemoval))
    b = gp.SixDstObjective(gb, gp.build_gene_pool(gb, gp.PoolKind.NodeRemoval))
    rng = np.random.default_rng(6)
    for rows in (3, 300, 1, 129, 64):
        xa = rng.integers(0, ga.n, size=(rows, 50)).astype(np.int32)
        xb = rng.integers(0, gb.n, size=(rows, 20)).astype(np.int32)
        assert np.array_equal(a.evaluate_batch(xa), oracle.eval_batch(oa, 0, xa))
        assert np.array_equal(b.evaluate_batch(xb), oracle.eval_batch(ob, 1, xb))


def test_batches_larger_than_the_scratch_budget(gp, oracle, cuda_device, monkeypatch):
    """GAPA_SCRATCH_MB = 1 forces the PC pipeline and the LPA kernels to process a batch in several
    passes (the path a 16k-individual batch on a 1M-node graph takes with the real budget)."""
    monkeypatch.setenv("GAPA_SCRATCH_MB", "1")
    monkeypatch.setenv("GAPA_PC_SMALL", "0")
    g = gp.barabasi_albert(4000, 3, 2)
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    batch = gp.init_population(pool.size(), 333, 200, 5)  # 6 groups; 1 MB holds ~9 vertex-group slices
    for task, cls in ((0, gp.PairwiseConnectivityObjective), (1, gp.SixDstObjective)):
        assert np.array_equal(cls(g, pool).evaluate_batch(batch), oracle.eval_batch(og, task, batch, threads=8))
    g = gp.erdos_renyi(3000, 0.004, 3)
    split = gp.build_lp_split(g, 0.1, 1)
    epool = gp.build_gene_pool(split.train, gp.PoolKind.EdgeRemoval)
    os_ = oracle.split_build(oracle.graph_from_edges(g.n, g.edges()), 0.1, 1)
    ebatch = gp.init_population(epool.size(), 90, 500, 6)
    assert np.array_equal(gp.LinkPredictionAttackObjective(split, epool).evaluate_batch(ebatch),
                          oracle.eval_batch(os_, 3, ebatch, threads=8))


def test_concurrent_callers_share_one_objective(gp, oracle, cuda_device):
    """fitness.hpp:17-27 objectives are called from many host threads at once (modes.cpp:85, :209): the CUDA
    objective serialises them internally; every caller must get the fitness of ITS batch."""
    import threading
    g = gp.barabasi_albert(3000, 3, 4)
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    objs = [gp.PairwiseConnectivityObjective(g, pool), gp.SixDstObjective(g, pool)]
    batches = [gp.init_population(pool.size(), 40 + 7 * t, 100, 20 + t) for t in range(6)]
    got = [[None] * len(batches) for _ in objs]

    def worker(t):
        for _ in range(3):
            for o, obj in enumerate(objs):
                got[o][t] = obj.evaluate_batch(batches[t])

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(len(batches))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for t, b in enumerate(batches):
        assert np.array_equal(got[0][t], oracle.eval_batch(og, 0, b))
        assert np.array_equal(got[1][t], oracle.eval_batch(og, 1, b))


def test_large_pageable_batches_take_the_pinned_ring(gp, oracle, cuda_device):
    """evaluate_batch(const PopulationMatrix&) hands the library a pageable std::vector (population.hpp:12-40); batches
    of 8 MB and more are staged through the library's pinned ring in 16 MB slices by several host threads.  Same
    fitness as the pinned-buffer call, the device-buffer call and the oracle; ragged last slice and last chunk."""
    import torch
    g = gp.barabasi_albert(20_000, 3, 2)
    og = oracle.graph_from_edges(g.n, g.edges())
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    obj = gp.PairwiseConnectivityObjective(g, pool)
    rows, k = 9_001, 1_000  # 36 MB: three slices, the last one ragged
    batch = gp.init_population(pool.size(), rows, k, 11)  # numpy: pageable
    got = obj.evaluate_batch(batch)
    pinned = torch.from_numpy(batch).pin_memory()
    out = torch.empty(rows, dtype=torch.float64).pin_memory()
    lib = gp.capi.load()
    gp.capi.check(lib.gapa_cuda_eval_batch(obj.dgraph.handle, obj.task, pinned.data_ptr(), rows, k, out.data_ptr()))
    assert np.array_equal(got, out.numpy())
    dev = torch.from_numpy(batch).cuda()
    dout = torch.empty(rows, dtype=torch.float64, device="cuda")
    obj.dgraph.eval_batch_device(obj.task, dev.data_ptr(), rows, k, dout.data_ptr(), 0)
    torch.cuda.synchronize()
    assert np.array_equal(got, dout.cpu().numpy())
    pick = np.r_[0:40, 4090:4110, rows - 30:rows]
    assert np.array_equal(got[pick], oracle.eval_batch(og, 0, batch[pick], threads=8))
    assert np.array_equal(obj.evaluate_batch(batch), got)  # ring slots reused


def test_fused_variation_validates_a_callers_pool_once(gp, cuda_device):
    """gapa_cuda_ga_slots_variation_eval_device inherits genes from parents the CALLER wrote: the first call on a pool
    buffer checks all parent rows (gene_pool.cpp:104-108: out of range is an error), later calls trust the library's
    own operators.  An out-of-range parent gene is GAPA_CUDA_E_RANGE, not an out-of-bounds write."""
    import torch
    from paper_2412_20980_b200.driver import CudaOps
    for n in (1500, 30_000):  # the shared-memory kernel and the bit-sliced pipeline
        g = gp.barabasi_albert(n, 3, 1)
        pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
        obj = gp.PairwiseConnectivityObjective(g, pool)
        ops = CudaOps(obj, 0)
        s, k = 16, 40
        slots = ops.empty_genes(2 * s, k)
        parent, child, partner = ops.empty_i32(s), ops.empty_i32(s), ops.empty_i32(s)
        fit, fit_m = ops.zeros_f64(s), ops.zeros_f64(s)
        ops.init(slots, parent, child, s, 3, 0)
        ops.eval_rows(slots, parent, 0, s, fit)
        ops.select(fit, s, 1, 3, 1, partner)
        ops.variation_eval(slots, parent, child, partner, s, 0.6, 0.2, 3, 1, 0, s, fit_m)   # validates, passes
        torch.cuda.synchronize()
        bad = slots.clone()                       # a different buffer: validated again
        bad[5, 7] = n + 12345
        with pytest.raises(gp.capi.GapaCudaError) as e:
            ops.variation_eval(bad, parent, child, partner, s, 0.6, 0.2, 3, 1, 0, s, fit_m)
        assert e.value.code == gp.capi.E_RANGE
