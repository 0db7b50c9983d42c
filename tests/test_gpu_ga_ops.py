"""Genetic operators: CUDA kernels vs the oracle, bit-exact.

Mirrors tests/test_ga_engine.cpp:48-54,131-141,150-158,175-246 of the reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MIN, MAX = None, None


@pytest.fixture(autouse=True)
def _dirs(gp):
    global MIN, MAX
    MIN, MAX = gp.Direction.Minimize, gp.Direction.Maximize


def test_rng_known_answers(gp, oracle, cuda_device):
    got = gp.rng_draws(1, 0, 1, 0, 3)
    assert [hex(int(x)) for x in got] == ["0xf065c62b02f8826d", "0xb860da951de09648", "0xce4d2df8c1ee9c22"]
    for seed, gen, role, row in [(1, 3, 4, 7), (2**63 + 5, 100, 2, 4095), (0, 0, 5, 0)]:
        assert np.array_equal(gp.rng_draws(seed, gen, role, row, 257), oracle.stream_u64(seed, gen, role, row, 257))


def test_init_population(gp, oracle, cuda_device):
    assert gp.init_population(1000, 4, 6, 1)[0].tolist() == [939, 720, 805, 966, 231, 61]
    for pool, s, k, seed in [(1000, 100, 50, 1), (7, 33, 1, 9), (2_000_000_000, 5, 300, 3), (1, 4, 4, 2)]:
        full = gp.init_population(pool, s, k, seed)
        assert np.array_equal(full, oracle.init_population(pool, s, k, seed))
        assert np.array_equal(gp.init_population_block(pool, 1, 3, k, seed), full[1:4])  # block == rows of full
    with pytest.raises(gp.capi.GapaCudaError):
        gp.init_population(0, 4, 4, 1)


def test_selection_weights_and_picks(gp, oracle, cuda_device):
    assert gp.selection_weights([5, 3, 3, 9], MIN).tolist() == [2.0, 3.5, 3.5, 1.0]
    assert gp.selection_weights([1, 2, 3, 4], MAX).tolist() == [1.0, 2.0, 3.0, 4.0]
    assert gp.selection_weights([7, 7, 7], MIN).tolist() == [2.0, 2.0, 2.0]
    rng = np.random.default_rng(11)
    for s in (2, 3, 100, 257, 1000, 4096, 5003, 9001, 25001):  # 25001: running totals no longer fit shared memory
        for ties in (False, True):
            f = rng.integers(0, 20, s).astype(float) if ties else rng.random(s)
            for d in (MIN, MAX):
                m = d == MIN
                assert np.array_equal(gp.selection_weights(f, d), oracle.selection_weights(f, m))
                assert np.array_equal(gp.roulette_pick(f, d, 5, s), oracle.roulette_pick(f, m, 5, s))
    with pytest.raises(gp.capi.GapaCudaError) as e:
        gp.roulette_pick([1.0, float("inf")], MIN, 1, 1)
    assert e.value.code == gp.capi.E_NAN


def test_crossover_and_mutation(gp, oracle, cuda_device):
    rng = np.random.default_rng(5)
    for s, k, pool in [(100, 50, 1000), (64, 1, 5), (10, 3000, 2**31 - 1)]:
        pop = rng.integers(0, pool, size=(s, k)).astype(np.int32)
        idx = rng.integers(0, s, size=s).astype(np.int32)
        for pc, pm in [(0.6, 0.2), (0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (1.0, 1.0), (0.8, 0.1)]:
            want = oracle.mutate_block(oracle.crossover(pop, idx, pc, 3, 17), 0, pm, pool, 3, 17)
            assert np.array_equal(gp.crossover_mutate(pop, idx, pc, pm, pool, 3, 17), want)
            lo, cnt = s // 3, s // 2
            assert np.array_equal(gp.crossover_mutate(pop, idx, pc, pm, pool, 3, 17, lo, cnt), want[lo:lo + cnt])
        # reference-shaped entry points: crossover(pop, partners) and mutate / mutate_block
        assert np.array_equal(gp.crossover(pop, pop[idx], 0.0, 3, 4), pop)        # test_ga_engine.cpp:131-141
        assert np.array_equal(gp.crossover(pop, pop[idx], 1.0, 3, 4), pop[idx])
        assert np.array_equal(gp.crossover(pop, pop[idx], 0.7, 3, 4), oracle.crossover(pop, idx, 0.7, 3, 4))
        assert np.array_equal(gp.mutate(pop, 0.0, pool, 1, 2), pop)                # :150-158
        m = gp.mutate(pop, 0.3, pool, 1, 2)
        assert np.array_equal(m, oracle.mutate_block(pop, 0, 0.3, pool, 1, 2))
        assert np.array_equal(gp.mutate_block(pop[5:9], 5, 0.3, pool, 1, 2), m[5:9])  # :175-182


def test_elitism(gp, oracle, cuda_device):
    # fixed cases incl. tie order (test_ga_engine.cpp:184-226)
    pop = np.arange(8, dtype=np.int32).reshape(4, 2)
    mp = pop + 100
    nxt, nf = gp.elitism(pop, mp, [3, 1, 2, 1], [1, 0, 5, 2], MIN)
    assert nf.tolist() == [0.0, 1.0, 1.0, 1.0]
    assert nxt.tolist() == [mp[1].tolist(), pop[1].tolist(), pop[3].tolist(), mp[0].tolist()]
    with pytest.raises(gp.capi.GapaCudaError) as e:
        gp.elitism(pop, mp, [1, float("nan"), 1, 1], [1, 1, 1, 1], MIN)
    assert e.value.code == gp.capi.E_NAN
    rng = np.random.default_rng(2)
    for trial in range(60):  # random triples vs the full-sort oracle (:228-246)
        s, k = int(rng.integers(2, 200)), int(rng.integers(1, 9))
        pop = rng.integers(0, 50, (s, k)).astype(np.int32)
        mp = rng.integers(0, 50, (s, k)).astype(np.int32)
        f = rng.integers(0, 10, s).astype(float)
        fm = rng.integers(0, 10, s).astype(float)
        for d in (MIN, MAX):
            a, b = gp.elitism(pop, mp, f, fm, d)
            c, e2 = oracle.elitism(pop, mp, f, fm, d == MIN)
            assert np.array_equal(a, c) and np.array_equal(b, e2)


def test_eda_sample(gp, oracle, cuda_device):
    rng = np.random.default_rng(8)
    elite = rng.integers(0, 40, (30, 12)).astype(np.int32)
    for ec, smooth in [(30, True), (5, True), (30, False), (1, False)]:
        assert np.array_equal(gp.eda_sample(elite, ec, 40, 4, 6, smooth), oracle.eda_sample(elite, ec, 40, 4, 6, smooth))
    with pytest.raises(gp.capi.GapaCudaError):
        gp.eda_sample(elite, 31, 40, 4, 6)


def test_mask_matrices_match_reference_and_explain_the_fused_operators(gp, oracle, cuda_device):
    """make_crossover_mask / make_mutation_mask / make_mutation_indices (ga_ops.cpp:84-103; test_ga_engine.cpp:143-173):
    the CUDA matrices equal the reference's (golden) and the oracle's, row blocks agree with the full matrices, and the
    fused crossover+mutate kernel IS  RM ? fresh : (RC ? partner row : own row)  on exactly these matrices."""
    import hashlib
    import json
    import os
    doc = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "masks.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for c in doc["masks"]:
        make = gp.make_crossover_mask if c["role"] == 3 else gp.make_mutation_mask
        m = make(c["rows"], c["cols"], c["rate"], c["seed"], c["generation"])
        assert m.dtype == np.uint8 and sha(m) == c["sha"] and int(m.sum()) == c["ones"]
        assert np.array_equal(m, oracle.make_mask(c["rows"], c["cols"], c["rate"], c["role"], c["seed"], c["generation"]))
    for c in doc["indices"]:
        m = gp.make_mutation_indices(c["rows"], c["cols"], c["pool"], c["seed"], c["generation"])
        assert sha(m) == c["sha"]
    rng = np.random.default_rng(4)
    s, k, pool, seed, gen, pc, pm = 57, 203, 900, 13, 6, 0.55, 0.15
    pop = rng.integers(0, pool, size=(s, k)).astype(np.int32)
    partner = rng.integers(0, s, size=s).astype(np.int32)
    rc, rm = gp.make_crossover_mask(s, k, pc, seed, gen), gp.make_mutation_mask(s, k, pm, seed, gen)
    fresh = gp.make_mutation_indices(s, k, pool, seed, gen)
    want = np.where(rm == 1, fresh, np.where(rc == 1, pop[partner], pop))
    import ctypes as C
    out = np.zeros_like(pop)
    gp.capi.check(gp.capi.load().gapa_cuda_ga_crossover_mutate(0, pop.ctypes.data, partner.ctypes.data, s, k, 0, s, pc, pm, pool, seed,
                                                               gen, out.ctypes.data))
    assert np.array_equal(out, want)
    assert abs(rc.mean() - pc) < 0.02 and abs(rm.mean() - pm) < 0.02  # the rates they realise (test_ga_engine.cpp:150-158)
    # device form, a row block: rows [20, 31) of the mutation mask
    import torch
    blk = torch.empty((11, k), dtype=torch.uint8, device="cuda")
    gp.capi.check(gp.capi.load().gapa_cuda_ga_mask_device(4, pm, 20, 11, k, seed, gen, blk.data_ptr(), 0))
    torch.cuda.synchronize()
    assert np.array_equal(blk.cpu().numpy(), rm[20:31])
