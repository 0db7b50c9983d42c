"""GPU: the CUDA path (through the C ABI) against the golden vectors of the unmodified reference."""
import pytest

import golden_cases as gc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def impl(gp, cuda_device):
    return gc.CudaImpl(gp)


@pytest.mark.parametrize("check", [gc.check_rng_and_init, gc.check_selection, gc.check_variation,
                                   gc.check_elitism_eda_partition, gc.check_generators, gc.check_pc_mcn, gc.check_cda,
                                   gc.check_lpa, gc.check_sixdegrees, gc.check_cda_add], ids=lambda f: f.__name__)
def test_cuda_matches_golden(impl, check):
    check(impl)


@pytest.mark.parametrize("name", gc.RUN_NAMES)
def test_cuda_trajectories_match_golden(impl, name):
    gc.check_run(impl, name)
