#include "internal.cuh"
using namespace gapa_b200;
extern "C" int gapa_cuda_run(gapa_cuda_ctx*, const gapa_cuda_run_params*, gapa_cuda_allgather_fn, void*, gapa_cuda_run_result*) { return fail(GAPA_CUDA_E_INVALID, "run: not built yet"); }
