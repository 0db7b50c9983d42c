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
