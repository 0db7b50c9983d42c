#include "internal.cuh"
namespace gapa_b200 {
int cda_eval(gapa_cuda_ctx*, const int32_t*, int, int, double*, cudaStream_t) { return fail(GAPA_CUDA_E_INVALID, "cda_fitness: kernel not built yet"); }
void cda_free(gapa_cuda_ctx*) {}
}
