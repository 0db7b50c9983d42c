#include "internal.cuh"
namespace gapa_b200 {
int lpa_eval(gapa_cuda_ctx*, const int32_t*, int, int, double*, cudaStream_t) { return fail(GAPA_CUDA_E_INVALID, "lpa_fitness: kernel not built yet"); }
void lpa_free(gapa_cuda_ctx*) {}
}
