"""CPU: the C-ABI library loads and exports every symbol include/gapa_cuda.h declares; the host-side
setup code (generators, split, budget, row partition) matches the golden vectors; the compute
entry points fail loudly without a GPU instead of falling back."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import golden_cases as gc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "gapa_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gapa_(?:cuda|host)_[a-z0-9_]+)\s*\(", text)) - {"gapa_cuda_allgather_fn"})


def test_library_exports_every_declared_symbol(gp):
    lib = gp.capi.load()
    declared = _declared_symbols()
    assert len(declared) >= 35
    for name in declared:
        assert hasattr(lib, name), f"{name} is declared in include/gapa_cuda.h but not exported"
        assert name in gp.capi.SIGNATURES, f"{name} has no ctypes signature in capi.py"
    assert set(gp.capi.SIGNATURES) == set(declared)
    assert lib.gapa_cuda_abi_version() == 3


def test_library_is_sm100a_cuda_code(gp):
    from paper_2412_20980_b200.build import LIB
    out = subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_setup_matches_golden(gp):
    impl = gc.CudaImpl(gp)
    gc.check_generators(impl)
    for c in gc.load("ops.json")["partition_rows"]:
        assert [list(b) for b in gp.partition_rows(c["s"], c["pn"])] == c["blocks"]
    for c in gc.load("fitness.json")["lpa"]:
        full = gp.Graph(c["n"], gc.i32(c["edges"], 2))
        sp = gp.build_lp_split(full, c["fraction"], c["split_seed"])
        assert sp.test_edges.tolist() == c["test"] and sp.probe_nonedges.tolist() == c["probe"]
        assert gc.sha(sp.train.edges()) == c["train_sha"]


def test_budget_and_pools(gp):
    g = gp.barabasi_albert(1000, 2, 1)
    assert gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05) == 50
    assert gp.perturbation_budget(g, gp.PoolKind.EdgeRemoval, 0.05) == 100  # ceil(0.05 * 1997)
    assert gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 1e-9) == 1
    for bad in (0.0, 1.5, -1.0):
        with pytest.raises(gp.capi.GapaCudaError):
            gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, bad)
    pool = gp.build_gene_pool(g, gp.PoolKind.EdgeRemoval)
    e = np.stack([pool.u, pool.v], 1)
    assert pool.size() == 1997 and np.all(e[:, 0] < e[:, 1])
    assert np.array_equal(e, e[np.lexsort((e[:, 1], e[:, 0]))])  # (u, v)-sorted, gene_pool.cpp:73-79
    with pytest.raises(gp.capi.GapaCudaError):
        gp.build_lp_split(g, 0.6, 1)
    with pytest.raises(gp.capi.GapaCudaError):
        gp.GAParams(pop_size=1).validate()


def test_no_cpu_fallback(gp):
    """Without a device every compute entry point reports GAPA_CUDA_E_CUDA; with one this test is moot."""
    lib = gp.capi.load()
    n = C.c_int(0)
    if lib.gapa_cuda_device_count(C.byref(n)) == 0 and n.value > 0:
        pytest.skip("a CUDA device is visible")
    g = gp.barabasi_albert(50, 2, 1)
    with pytest.raises(gp.capi.GapaCudaError) as e:
        gp.PairwiseConnectivityObjective(g, gp.build_gene_pool(g, gp.PoolKind.NodeRemoval))
    assert e.value.code == gp.capi.E_CUDA
    with pytest.raises(gp.capi.GapaCudaError):
        gp.init_population(10, 2, 2, 1)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2412_20980_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "gapa_oracle" not in text and "oracle.bindings" not in text and "libgapa_ref" not in text, f
