"""GPU: the host C++ side of the drop-in.

1. oracle/_ref/ref_gpu_driver — the UNMODIFIED reference's run_ga (serial, S, SM, M, MNM) driving
   the CUDA objectives, which derive from the real gapa::FitnessFunction; built in the authoring
   container against /root/reference (oracle/Makefile), run here as a binary.
2. tests/cpp/host_adapter_test.cpp — the same adapters over the mirror header, compiled here."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2412_20980_b200", "libgapa_cuda.so")


def _env():
    return {**os.environ, "GAPA_CUDA_LIB": LIB}


@pytest.mark.gpu
def test_reference_run_ga_drives_cuda_objectives(gp, cuda_device):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_gpu_driver")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_gpu_driver was not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=_env())
    assert out.returncode == 0 and "DROPIN_OK" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


@pytest.mark.gpu
def test_cxx_plugin_boundary_end_to_end(gp, cuda_device):
    """The real drop-in call, from C++: the reference's barabasi_albert / build_gene_pool / init_population_block and
    FitnessFunction::evaluate_batch(const PopulationMatrix&) of the CUDA objective — a pageable std::vector crossing the
    library's pinned ring.  Values must equal the Python device path on the same init stream; the line it prints (evals/s
    through the C++ boundary) is what `tools/cxx_e2e.sh` records under profiles/ at the full C4 size."""
    import json
    import numpy as np
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_gpu_driver")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_gpu_driver was not built (needs /root/reference at build time)")
    n, attach, rows = 100_000, 5, 1024
    out = subprocess.run([exe, "e2e", str(n), str(attach), str(rows), "3"], capture_output=True, text=True, timeout=900, env=_env())
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    g = gp.barabasi_albert(n, attach, 1)
    pool = gp.build_gene_pool(g, gp.PoolKind.NodeRemoval)
    k = gp.perturbation_budget(g, gp.PoolKind.NodeRemoval, 0.05)
    assert (line["k"], line["m"], line["pop"]) == (k, g.edge_count(), rows)
    want = gp.PairwiseConnectivityObjective(g, pool).evaluate_batch(gp.init_population(pool.size(), rows, k, 1))
    assert np.array_equal(np.asarray(line["fitness_head"]), want[:3])
    assert line["evals_per_sec"] > 0


def _build_host_test(tmp_path):
    exe = str(tmp_path / "host_adapter_test")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "paper_2412_20980_b200", "host"), os.path.join(ROOT, "tests", "cpp", "host_adapter_test.cpp"),
           "-o", exe, "-ldl"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.mark.gpu
def test_host_adapters_mirror_mode(gp, cuda_device, tmp_path):
    out = subprocess.run([_build_host_test(tmp_path)], capture_output=True, text=True, timeout=300, env=_env())
    assert out.returncode == 0 and "HOST_ADAPTER_OK" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


def test_host_adapters_compile_and_fail_loudly_without_gpu(gp, tmp_path):
    """CPU: the header-only adapters build with plain g++; without a device they throw gapa::Error."""
    import ctypes as C
    exe = _build_host_test(tmp_path)
    n = C.c_int(0)
    if gp.capi.load().gapa_cuda_device_count(C.byref(n)) == 0 and n.value > 0:
        pytest.skip("a CUDA device is visible")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60, env=_env())
    assert out.returncode == 2 and "no CUDA device available" in out.stdout
