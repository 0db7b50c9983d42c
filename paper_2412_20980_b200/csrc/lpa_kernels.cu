// Link-prediction attack fitness (GAPA_TASK_LPA): AUC of the resource-allocation
// predictor on the perturbed train graph.
//
// Reference path per individual (fitness.cpp:43-48): copy the dense train adjacency,
// clear two bits per gene (gene_pool.cpp:53-56), RA(u,v) = sum over common neighbours
// z ascending of 1.0 / deg'(z) for the T test and P probe pairs
// (link_prediction.cpp:55-77), then wins over the full T x P grid, +1 for t > p and
// +0.5 for t == p, auc = wins / (T * P) (link_prediction.cpp:87-96).
//
// Here: per individual an m-bit "edge removed" mask and an int32 perturbed degree per
// vertex (both L2-resident scratch), one thread per (individual, pair) intersecting the
// two ascending CSR rows — which visits common neighbours in ascending z, so the FP64
// sum has the reference's operation order — and an exact integer count of 2 * wins.
// All partial sums of the reference's `wins` are multiples of 0.5 below 2^53, hence
// exact, so (2*wins)/2.0 / (T*P) is the same double.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace gapa_b200 {

static constexpr int kLpaThreads = 256;

struct LpaScratch {
    DevBuf gone, deg, scores, twice, status;
    int sorted_auc = -1;  // GAPA_LPA_SORTED_AUC=0 forces the T x P grid kernel (tests run both)
};

__global__ void __launch_bounds__(kLpaThreads) k_lpa_init(const int32_t* __restrict__ row_ptr, int n, int rows,
                                                          int32_t* __restrict__ deg) {
    const size_t total = static_cast<size_t>(rows) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % n);
        deg[i] = row_ptr[x + 1] - row_ptr[x];
    }
}

// apply_in_place for EdgeRemoval (gene_pool.cpp:53-56); duplicates idempotent.
__global__ void __launch_bounds__(kLpaThreads) k_lpa_remove(GeneRows genes, size_t cells,
                                                            const int32_t* __restrict__ pool_map, int pool_size,
                                                            const int32_t* __restrict__ edge_u,
                                                            const int32_t* __restrict__ edge_v, int n, int mask_words,
                                                            unsigned* gone, int32_t* deg, int* status) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / genes.cols);
        const int gene = genes.row(r)[i - static_cast<size_t>(r) * genes.cols];
        if (gene < 0 || gene >= pool_size) {
            *status = GAPA_CUDA_E_RANGE;
            continue;
        }
        const int e = pool_map ? pool_map[gene] : gene;
        if (e < 0) continue;  // the pool names a pair that is not an edge of this graph: nothing to clear (gene_pool.cpp:53-56)
        const unsigned bit = 1u << (e & 31);
        const unsigned old = atomicOr(&gone[static_cast<size_t>(r) * mask_words + (e >> 5)], bit);
        if (!(old & bit)) {
            atomicSub(&deg[static_cast<size_t>(r) * n + edge_u[e]], 1);
            atomicSub(&deg[static_cast<size_t>(r) * n + edge_v[e]], 1);
        }
    }
}

// ra_score (link_prediction.cpp:55-69) for every (individual, pair)
__global__ void __launch_bounds__(kLpaThreads) k_lpa_scores(const int32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col_idx,
                                                            const int32_t* __restrict__ edge_id,
                                                            const int32_t* __restrict__ pairs, int n_pairs, int n,
                                                            int mask_words, const unsigned* __restrict__ gone,
                                                            const int32_t* __restrict__ deg, double* __restrict__ scores) {
    const int r = blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_pairs) return;
    const unsigned* mask = gone + static_cast<size_t>(r) * mask_words;
    const int32_t* d = deg + static_cast<size_t>(r) * n;
    const int u = pairs[2 * q], v = pairs[2 * q + 1];
    int i = row_ptr[u], j = row_ptr[v];
    const int ie = row_ptr[u + 1], je = row_ptr[v + 1];
    double score = 0.0;
    if (i < ie && j < je) {
        int a = col_idx[i], b = col_idx[j];
        for (;;) {
            if (a < b) {
                if (++i >= ie) break;
                a = col_idx[i];
            } else if (b < a) {
                if (++j >= je) break;
                b = col_idx[j];
            } else {
                const int e1 = edge_id[i], e2 = edge_id[j];
                const bool alive = !((mask[e1 >> 5] >> (e1 & 31)) & 1u) && !((mask[e2 >> 5] >> (e2 & 31)) & 1u);
                if (alive) {
                    const int dz = d[a];
                    if (dz > 0) score += 1.0 / static_cast<double>(dz);
                }
                ++i;
                ++j;
                if (i >= ie || j >= je) break;
                a = col_idx[i];
                b = col_idx[j];
            }
        }
    }
    scores[static_cast<size_t>(r) * n_pairs + q] = score;
}

// 2 * wins over the T x P grid (link_prediction.cpp:87-94), exact integers
__global__ void __launch_bounds__(kLpaThreads) k_lpa_auc(const double* __restrict__ scores, int T, int P,
                                                         unsigned long long* twice) {
    __shared__ double tile[kLpaThreads];
    __shared__ unsigned long long block_sum;
    const int r = blockIdx.y;
    const double* row = scores + static_cast<size_t>(r) * (T + P);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const double mine = t < T ? row[t] : 0.0;
    if (threadIdx.x == 0) block_sum = 0ull;
    unsigned long long acc = 0ull;
    for (int p0 = 0; p0 < P; p0 += kLpaThreads) {
        __syncthreads();
        if (p0 + threadIdx.x < P) tile[threadIdx.x] = row[T + p0 + threadIdx.x];
        __syncthreads();
        const int lim = min(kLpaThreads, P - p0);
        int wins2 = 0;
        for (int p = 0; p < lim; ++p) {
            const double other = tile[p];
            wins2 += mine > other ? 2 : (mine == other ? 1 : 0);
        }
        acc += static_cast<unsigned long long>(wins2);
    }
    if (t >= T) acc = 0ull;
    for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&block_sum, acc);
    __syncthreads();
    if (threadIdx.x == 0 && block_sum) atomicAdd(&twice[r], block_sum);
}

// The same 2 * wins without the T x P grid: one CTA per individual sorts the P probe scores in shared
// memory (bitonic network on order-preserving 64-bit integer keys) and every test score finds, by two
// binary searches, how many probe scores are below it and how many equal it:
//     2 * wins = sum over t of  2 * #(p < t) + #(p == t)
// — O((T + P) log P) integer compares instead of T * P FP64 compares (25 M per individual at C3).
// Same integers, so the AUC is the same double.
static constexpr int kLpaSortThreads = 1024;
extern __shared__ unsigned long long lpa_keys[];

__device__ __forceinline__ unsigned long long score_key(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 == +0.0 must compare equal as keys too
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // total order of finite doubles
}

__global__ void __launch_bounds__(kLpaSortThreads) k_lpa_auc_sorted(const double* __restrict__ scores, int T, int P, int P2,
                                                                    double* __restrict__ out) {
    const int all_probes = P;
    __shared__ unsigned long long warp_sum[kLpaSortThreads / 32];
    __shared__ int n_nonzero;
    const int r = blockIdx.x, tid = threadIdx.x;
    const double* row = scores + static_cast<size_t>(r) * (T + P);
    // In a sparse graph most pairs have no common neighbour: their score is exactly 0.  Only the non-zero probe
    // scores are compacted and sorted; the zeros are a count.  (A pair score is a sum of positive terms: never < 0.)
    if (tid == 0) n_nonzero = 0;
    __syncthreads();
    for (int i = tid; i < P; i += kLpaSortThreads) {
        const double x = row[T + i];
        if (x != 0.0) lpa_keys[atomicAdd(&n_nonzero, 1)] = score_key(x);
    }
    __syncthreads();
    const int nz = n_nonzero, zeros = P - nz;
    const unsigned long long zero_key = score_key(0.0);
    P = nz;
    P2 = 2;
    while (P2 < P) P2 <<= 1;
    for (int i = P + tid; i < P2; i += kLpaSortThreads) lpa_keys[i] = ~0ull;  // pads sort to the end
    __syncthreads();
    for (int k = 2; k <= P2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P2; i += kLpaSortThreads) {
                const int partner = i ^ j;
                if (partner > i) {
                    const unsigned long long a = lpa_keys[i], b = lpa_keys[partner];
                    if ((a > b) == ((i & k) == 0)) {
                        lpa_keys[i] = b;
                        lpa_keys[partner] = a;
                    }
                }
            }
            __syncthreads();
        }
    unsigned long long acc = 0ull;
    for (int t = tid; t < T; t += kLpaSortThreads) {
        const unsigned long long key = score_key(row[t]);
        int lo = 0, hi = P;  // first index with keys[idx] >= key
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (lpa_keys[mid] < key) lo = mid + 1; else hi = mid;
        }
        int below = lo;
        hi = P;  // first index with keys[idx] > key
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (lpa_keys[mid] <= key) lo = mid + 1; else hi = mid;
        }
        int equal = lo - below;
        if (key > zero_key) below += zeros;        // every zero probe score is below a positive test score
        else if (key == zero_key) equal += zeros;  // ... and ties with a zero one
        acc += 2ull * static_cast<unsigned long long>(below) + static_cast<unsigned long long>(equal);
    }
    for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if ((tid & 31) == 0) warp_sum[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
        unsigned long long total = 0ull;
        for (int w = 0; w < kLpaSortThreads / 32; ++w) total += warp_sum[w];
        const double wins = static_cast<double>(total) / 2.0;
        out[r] = wins / (static_cast<double>(T) * static_cast<double>(all_probes));  // link_prediction.cpp:96
    }
}

__global__ void k_lpa_final(const unsigned long long* __restrict__ twice, int rows, int T, int P, double* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const double wins = static_cast<double>(twice[r]) / 2.0;
    out[r] = wins / (static_cast<double>(T) * static_cast<double>(P));  // link_prediction.cpp:96
}

int lpa_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, bool trusted) {
    const int cols = genes.cols;
    if (!ctx->lpa) ctx->lpa = new LpaScratch();
    LpaScratch* s = ctx->lpa;
    if (s->sorted_auc < 0) {
        const char* raw = std::getenv("GAPA_LPA_SORTED_AUC");
        s->sorted_auc = (raw && *raw == '0') ? 0 : 1;
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_lpa_auc_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    const int n = ctx->n, T = ctx->T, P = ctx->P, n_pairs = T + P;
    const int mask_words = static_cast<int>((ctx->m + 31) / 32) + 1;
    const size_t per_row = sizeof(unsigned) * mask_words + sizeof(int32_t) * n + sizeof(double) * n_pairs;
    size_t budget = 8ull << 30;  // scratch per pass; GAPA_SCRATCH_MB overrides (tests force several passes)
    if (const char* raw = std::getenv("GAPA_SCRATCH_MB")) budget = static_cast<size_t>(std::max(1L, std::strtol(raw, nullptr, 10))) << 20;
    const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(rows, budget / per_row)));
    GAPA_TRY(s->gone.ensure(sizeof(unsigned) * mask_words * static_cast<size_t>(chunk)));
    GAPA_TRY(s->deg.ensure(sizeof(int32_t) * std::max(n, 1) * static_cast<size_t>(chunk)));
    GAPA_TRY(s->scores.ensure(sizeof(double) * n_pairs * static_cast<size_t>(chunk)));
    GAPA_TRY(s->twice.ensure(sizeof(unsigned long long) * chunk));
    GAPA_TRY(s->status.ensure(sizeof(int)));
    int* status = s->status.as<int>();
    GAPA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), stream));
    const int sm = ctx->sm_count;
    for (int r0 = 0; r0 < rows; r0 += chunk) {
        const int cr = std::min(chunk, rows - r0);
        GAPA_CUDA_TRY(cudaMemsetAsync(s->gone.ptr, 0, sizeof(unsigned) * mask_words * static_cast<size_t>(cr), stream));
        if (n > 0) GAPA_LAUNCH(k_lpa_init, sm * 8, kLpaThreads, 0, stream, ctx->d_row_ptr, n, cr, s->deg.as<int32_t>());
        const size_t cells = static_cast<size_t>(cr) * cols;
        if (cells) {
            const int grid = static_cast<int>(std::min<size_t>((cells + kLpaThreads - 1) / kLpaThreads, static_cast<size_t>(sm) * 32));
            GAPA_LAUNCH(k_lpa_remove, grid, kLpaThreads, 0, stream, genes.from(r0), cells,
                        ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, ctx->d_edge_u, ctx->d_edge_v, n,
                        mask_words, s->gone.as<unsigned>(), s->deg.as<int32_t>(), status);
        }
        GAPA_LAUNCH(k_lpa_scores, dim3((n_pairs + kLpaThreads - 1) / kLpaThreads, cr), kLpaThreads, 0, stream, ctx->d_row_ptr,
                    ctx->d_col_idx, ctx->d_edge_id, ctx->d_pairs, n_pairs, n, mask_words, s->gone.as<unsigned>(),
                    s->deg.as<int32_t>(), s->scores.as<double>());
        int P2 = 2;
        while (P2 < P) P2 <<= 1;
        if (P > 0 && s->sorted_auc && sizeof(unsigned long long) * static_cast<size_t>(P2) <= 200 * 1024) {
            GAPA_LAUNCH(k_lpa_auc_sorted, cr, kLpaSortThreads, sizeof(unsigned long long) * P2, stream, s->scores.as<double>(), T, P, P2,
                        out_dev + r0);  // writes the AUC itself
            continue;
        }
        GAPA_CUDA_TRY(cudaMemsetAsync(s->twice.ptr, 0, sizeof(unsigned long long) * cr, stream));
        if (P > 0)  // probe set too large for shared memory: the exact T x P grid
            GAPA_LAUNCH(k_lpa_auc, dim3((T + kLpaThreads - 1) / kLpaThreads, cr), kLpaThreads, 0, stream,
                        s->scores.as<double>(), T, P, s->twice.as<unsigned long long>());
        GAPA_LAUNCH(k_lpa_final, (cr + 255) / 256, 256, 0, stream, s->twice.as<unsigned long long>(), cr, T, P, out_dev + r0);
    }
    if (trusted) return GAPA_CUDA_OK;
    GAPA_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, stream));
    GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
    if (ctx->h_status[0] == GAPA_CUDA_E_RANGE) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
    return GAPA_CUDA_OK;
}

const double* lpa_last_scores(const gapa_cuda_ctx* ctx) { return ctx->lpa ? ctx->lpa->scores.as<double>() : nullptr; }

void lpa_free(gapa_cuda_ctx* ctx) {
    if (!ctx->lpa) return;
    for (DevBuf* b : {&ctx->lpa->gone, &ctx->lpa->deg, &ctx->lpa->scores, &ctx->lpa->twice, &ctx->lpa->status}) b->release();
    delete ctx->lpa;
    ctx->lpa = nullptr;
}

}  // namespace gapa_b200
