"""CPU: the C oracle against the golden vectors produced by the unmodified reference.
This is what pins the oracle; it runs everywhere, no reference needed."""
import pytest

import golden_cases as gc


@pytest.fixture(scope="module")
def impl(oracle):
    return gc.OracleImpl(oracle)


@pytest.mark.parametrize("check", [gc.check_rng_and_init, gc.check_selection, gc.check_variation,
                                   gc.check_elitism_eda_partition, gc.check_generators, gc.check_pc_mcn, gc.check_cda,
                                   gc.check_lpa, gc.check_sixdegrees, gc.check_cda_add], ids=lambda f: f.__name__)
def test_oracle_matches_golden(impl, check):
    check(impl)


@pytest.mark.parametrize("name", gc.RUN_NAMES)
def test_oracle_trajectories_match_golden(impl, name):
    gc.check_run(impl, name)


def test_recorded_reference_values(oracle):
    """Values the reference's own test run recorded (proj/test_output.txt:50-54)."""
    runs = gc.load("runs.json")
    assert runs["acceptance6_sixdst_er100"]["best"][-1] == 81.0                      # criterion 6: final MCN 81
    assert f'{runs["acceptance10_lpa_sbm64"]["auc0"]:.6f}' == "0.728395"           # criterion 10
    assert f'{runs["acceptance10_lpa_sbm64"]["best"][-1]:.6f}' == "0.388889"
    assert f'{gc.load("fitness.json")["karate"]["q0"]:.6f}' == "0.380671"          # criterion 8: unattacked Q
    assert f'{gc.load("runs_widen.json")["acceptance8_cda_add_karate"]["best"][-1]:.5f}' == "0.26156"  # attacked Q @300
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF and oracle.mix64(1) == 0x910A2DEC89025CC1


def test_oracle_reproduces_the_reference_mask_matrices(oracle):
    """make_crossover_mask / make_mutation_mask / make_mutation_indices (ga_ops.cpp:84-103) from the compiled reference"""
    import hashlib
    import json
    import os

    import numpy as np
    doc = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "masks.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for c in doc["masks"]:
        m = oracle.make_mask(c["rows"], c["cols"], c["rate"], c["role"], c["seed"], c["generation"])
        assert sha(m) == c["sha"] and m[0][:24].tolist() == c["row0"] and int(m.sum()) == c["ones"]
    for c in doc["indices"]:
        m = oracle.make_mutation_indices(c["rows"], c["cols"], c["pool"], c["seed"], c["generation"])
        assert sha(m) == c["sha"] and m[0][:16].tolist() == c["row0"]


def test_unpinned_twins_reduce_to_the_pinned_oracle(oracle):
    """CN / edge-flip twins (no reference implementation: parity unpinned).  Restricted to what the reference has —
    RA score, edges removed — the twin must equal the reference-pinned LPA oracle; unranking covers the pair space."""
    import numpy as np
    g = oracle.graph_er(300, 0.04, 5)
    sp = oracle.split_build(g, 0.2, 2)
    pop = oracle.init_population(sp.train.m, 6, 30, 1)
    assert np.array_equal(oracle.lpa_scored_batch(sp, pop, 0), oracle.eval_batch(sp, 3, pop))
    n = 37
    seen = [oracle.flip_unrank(n, i) for i in range(n * (n - 1) // 2)]
    assert seen == [(a, b) for a in range(n) for b in range(a + 1, n)]
    ranks = np.array([[a * 300 - a * (a + 1) // 2 + (b - a - 1) for a, b in zip(sp.train.pool_u[:20], sp.train.pool_v[:20])]], np.int32)
    assert np.array_equal(oracle.lpa_flip_batch(sp, ranks, 0), oracle.eval_batch(sp, 3, np.arange(20, dtype=np.int32)[None, :]))
