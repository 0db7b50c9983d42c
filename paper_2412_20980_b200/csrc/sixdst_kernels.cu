// SixDST fitness with the truncated closure (GAPA_TASK_SIXDST): sixdst_fitness(...,
// ClosurePolicy::SixDegrees), fitness.cpp:18-26 over accessibility.cpp:20-37.
//
// Reference path per individual: copy the dense n x n BitMatrix, zero a row + column per
// gene, square (A + I) over the boolean semiring at most three times (O(n^3 / 64) word ORs
// per squaring), return the largest row popcount.  After j squarings entry (u, v) is set iff
// dist(u, v) <= 2^j, so the result is the size of the largest radius-8 ball of the perturbed
// graph; a removed node keeps only its diagonal bit (ball = 1).
//
// Here: no matrix is formed.  One CTA per individual runs a bit-parallel multi-source BFS on
// the shared CSR: 64 sources at a time, one 64-bit word per vertex ("which of the 64 sources
// reach me within t steps"), eight synchronous rounds  next[v] = cur[v] | OR cur[N(v)]  with
// the two word arrays and the removed bitmap in SHARED memory (global scratch when n is too
// large for that), early exit when a round changes nothing, then per-source column counts.
// Work per individual: (n / 64) x 8 x (n + 2m) word operations instead of 3 n^3 / 64.
// Integer arithmetic end to end.
#include <algorithm>

#include "internal.cuh"

namespace gapa_b200 {

typedef unsigned long long word_t;
static constexpr int kSixThreads = 1024;
static constexpr int kSixRadius = 8;  // 3 squarings of A + I: paths of length <= 2^3 (accessibility.hpp:12-14)

struct SixScratch {
    DevBuf words, status;
};

extern __shared__ __align__(16) unsigned char six_smem[];

__global__ void __launch_bounds__(kSixThreads, 1) k_sixdst(const int32_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col_idx, int n, GeneRows genes,
                                                           const int32_t* __restrict__ pool_map, int pool_size, int rows,
                                                           word_t* scratch, int in_smem, double* __restrict__ out,
                                                           int* status) {
    griddep_launch();
    griddep_wait();
    __shared__ int counts[64];
    __shared__ int warp_best[kSixThreads / 32];
    const int tid = threadIdx.x;
    const int gone_words = (n + 31) >> 5;
    word_t* cur = in_smem ? reinterpret_cast<word_t*>(six_smem) : scratch + static_cast<size_t>(blockIdx.x) * 2 * n;
    word_t* nxt = cur + n;
    unsigned* gone = in_smem ? reinterpret_cast<unsigned*>(six_smem + sizeof(word_t) * 2 * static_cast<size_t>(n))
                             : reinterpret_cast<unsigned*>(six_smem);
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        for (int w = tid; w < gone_words; w += kSixThreads) gone[w] = 0u;
        __syncthreads();
        const int32_t* g = genes.row(r);
        for (int j = tid; j < genes.cols; j += kSixThreads) {  // apply_in_place, NodeRemoval (gene_pool.cpp:61-64)
            const int gene = g[j];
            if (gene < 0 || gene >= pool_size) {
                *status = GAPA_CUDA_E_RANGE;
                continue;
            }
            const int node = pool_map ? pool_map[gene] : gene;
            atomicOr(&gone[node >> 5], 1u << (node & 31));
        }
        __syncthreads();
        int best = 1;  // every node reaches itself (the diagonal of A + I), removed or not
        for (int b0 = 0; b0 < n; b0 += 64) {
            for (int v = tid; v < n; v += kSixThreads) {
                const bool source = v >= b0 && v < b0 + 64 && !((gone[v >> 5] >> (v & 31)) & 1u);
                cur[v] = source ? 1ull << (v - b0) : 0ull;  // removed vertices stay 0: nothing flows through them
            }
            if (tid < 64) counts[tid] = 0;
            __syncthreads();
            for (int round = 0; round < kSixRadius; ++round) {
                int changed = 0;
                for (int v = tid; v < n; v += kSixThreads) {
                    const word_t mine = cur[v];
                    word_t w = mine;
                    if (!((gone[v >> 5] >> (v & 31)) & 1u)) {
                        const int end = row_ptr[v + 1];
                        for (int e = row_ptr[v]; e < end; ++e) w |= cur[col_idx[e]];
                    }
                    nxt[v] = w;
                    changed |= w != mine;
                }
                word_t* t = cur;
                cur = nxt;
                nxt = t;
                if (!__syncthreads_or(changed)) break;  // closed before radius 8: identical to the capped squaring
            }
            // ball size of source b0 + b = number of vertices whose word has bit b
            const int b = tid & 63;
            int cnt = 0;
            for (int v = tid >> 6; v < n; v += kSixThreads / 64) cnt += static_cast<int>((cur[v] >> b) & 1ull);
            if (cnt) atomicAdd(&counts[b], cnt);
            __syncthreads();
            if (tid < 64) best = max(best, counts[tid]);
            __syncthreads();
        }
        for (int off = 16; off; off >>= 1) best = max(best, __shfl_down_sync(0xffffffffu, best, off));
        if ((tid & 31) == 0) warp_best[tid >> 5] = best;
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kSixThreads / 32; ++w) best = max(best, warp_best[w]);
            out[r] = static_cast<double>(n > 0 ? best : 0);  // fitness.cpp:23-25
        }
        __syncthreads();
    }
}

int sixdst_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, bool trusted) {
    if (!ctx->six) ctx->six = new SixScratch();
    SixScratch* s = ctx->six;
    const int n = ctx->n;
    const size_t gone_bytes = sizeof(unsigned) * (static_cast<size_t>((n + 31) >> 5) + 1);
    const size_t word_bytes = sizeof(word_t) * 2 * static_cast<size_t>(n);
    const int in_smem = word_bytes + gone_bytes <= 200 * 1024 ? 1 : 0;
    if (!in_smem && gone_bytes > 200 * 1024) return fail(GAPA_CUDA_E_INVALID, "sixdst_fitness: graph too large for the truncated closure");
    const int slots = std::max(1, std::min(rows, ctx->sm_count));
    if (!in_smem) GAPA_TRY(s->words.ensure(word_bytes * slots));
    GAPA_TRY(s->status.ensure(sizeof(int)));
    GAPA_CUDA_TRY(cudaMemsetAsync(s->status.ptr, 0, sizeof(int), stream));
    const size_t smem = (in_smem ? word_bytes : 0) + gone_bytes;
    GAPA_CUDA_TRY(cudaFuncSetAttribute(k_sixdst, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    GAPA_LAUNCH(k_sixdst, slots, kSixThreads, smem, stream, ctx->d_row_ptr, ctx->d_col_idx, n, genes,
                ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, rows, s->words.as<word_t>(), in_smem, out_dev,
                s->status.as<int>());
    if (trusted) return GAPA_CUDA_OK;
    GAPA_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, s->status.ptr, sizeof(int), cudaMemcpyDeviceToHost, stream));
    GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
    if (ctx->h_status[0] == GAPA_CUDA_E_RANGE) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
    return GAPA_CUDA_OK;
}

void sixdst_free(gapa_cuda_ctx* ctx) {
    if (!ctx->six) return;
    ctx->six->words.release();
    ctx->six->status.release();
    delete ctx->six;
    ctx->six = nullptr;
}

}  // namespace gapa_b200
