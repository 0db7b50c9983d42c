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
    DevBuf add_keys, add_count, row_ptr2, col2, base_cnt;  // edge-flip pools: per-individual added pairs and perturbed CSR
    int sorted_auc = -1;  // GAPA_LPA_SORTED_AUC=0 forces the T x P grid kernel (tests run both)
};

__global__ void __launch_bounds__(kLpaThreads) k_lpa_init(const int32_t* __restrict__ row_ptr, int n, int rows,
                                                          int32_t* __restrict__ deg) {
    griddep_launch();
    griddep_wait();
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
    griddep_launch();
    griddep_wait();
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
                                                            const int32_t* __restrict__ deg, double* __restrict__ scores, int cn) {
    griddep_launch();
    griddep_wait();
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
                    if (dz > 0) score += cn ? 1.0 : 1.0 / static_cast<double>(dz);  // cn: common-neighbour count (not in the reference)
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
    griddep_launch();
    griddep_wait();
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
    griddep_launch();
    griddep_wait();
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


// ---------------------------------------------------------------------------------------------------------------
// Edge-FLIP pools (GAPA_POOL_EDGE_FLIP; north_star's "edge flips", NOT in the reference — PARITY UNPINNED, the CPU twin
// is the lpa_flip_batch function of the oracle directory's C restatement).  A gene is a node pair a < b: an edge of the train graph is removed, a
// non-edge is added.  Removals reuse the m-bit mask; additions make the shared CSR insufficient, so every individual
// gets its own perturbed CSR (4 (n + 1) + 4 (2 m + 2 k) bytes — 0.5 MB at C3): rows stay ascending, which keeps the
// common neighbours of a pair in ascending z and with it the reference's FP64 summation order for RA.
__device__ __forceinline__ void flip_pair(int gene, int n, const int32_t* __restrict__ pair_u, const int32_t* __restrict__ pair_v, int* a, int* b) {
    if (pair_u) {
        *a = pair_u[gene];
        *b = pair_v[gene];
        return;
    }
    // lexicographic unranking: the largest a with a n - a (a + 1) / 2 <= gene (FP64 estimate, exact integer fix-up)
    const double nn = 2.0 * n - 1.0;
    long long x = static_cast<long long>((nn - sqrt(nn * nn - 8.0 * static_cast<double>(gene))) * 0.5);
    x = max(0ll, min(x, static_cast<long long>(n) - 2));
    while (x > 0 && x * n - x * (x + 1) / 2 > gene) --x;
    while (x + 1 <= n - 2 && (x + 1) * n - (x + 1) * (x + 2) / 2 <= gene) ++x;
    *a = static_cast<int>(x);
    *b = static_cast<int>(gene - (x * n - x * (x + 1) / 2) + x + 1);
}

// genes -> removed-edge bits + perturbed degrees (as k_lpa_remove) or candidate added pairs (deduplicated later)
__global__ void __launch_bounds__(kLpaThreads) k_lpa_flip_classify(GeneRows genes, size_t cells, int pool_size, int n,
                                                                   const int32_t* __restrict__ pair_u, const int32_t* __restrict__ pair_v,
                                                                   const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                                                   const int32_t* __restrict__ edge_id, int mask_words, unsigned* gone,
                                                                   int32_t* deg, unsigned long long* add_keys, int* add_count, int* status) {
    griddep_launch();
    griddep_wait();
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / genes.cols);
        const int gene = genes.row(r)[i - static_cast<size_t>(r) * genes.cols];
        if (gene < 0 || gene >= pool_size) {
            *status = GAPA_CUDA_E_RANGE;
            continue;
        }
        int a, b;
        flip_pair(gene, n, pair_u, pair_v, &a, &b);
        int lo = row_ptr[a], hi = row_ptr[a + 1];
        const int end = hi;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (col_idx[mid] < b) lo = mid + 1; else hi = mid;
        }
        if (lo < end && col_idx[lo] == b) {  // an edge: remove it
            const int e = edge_id[lo];
            const unsigned bit = 1u << (e & 31);
            const unsigned old = atomicOr(&gone[static_cast<size_t>(r) * mask_words + (e >> 5)], bit);
            if (!(old & bit)) {
                atomicSub(&deg[static_cast<size_t>(r) * n + a], 1);
                atomicSub(&deg[static_cast<size_t>(r) * n + b], 1);
            }
        } else {  // a non-edge: a candidate addition
            const int at = atomicAdd(&add_count[r], 1);
            add_keys[static_cast<size_t>(r) * genes.cols + at] = (static_cast<unsigned long long>(a) << 32) | static_cast<unsigned>(b);
        }
    }
}

// One CTA per individual: sort the candidate pairs (bitonic, shared memory), drop repeats, raise the degrees of the
// endpoints, leave the distinct pairs sorted in add_keys[r][0 .. add_count[r]).
__global__ void __launch_bounds__(kLpaSortThreads) k_lpa_flip_unique(int cols, int n, unsigned long long* add_keys, int* add_count, int32_t* deg) {
    griddep_launch();
    griddep_wait();
    __shared__ int kept;
    const int r = blockIdx.x, tid = threadIdx.x;
    const int c = add_count[r];
    unsigned long long* keys = add_keys + static_cast<size_t>(r) * cols;
    int c2 = 2;
    while (c2 < c) c2 <<= 1;
    if (c == 0) return;
    for (int i = tid; i < c2; i += kLpaSortThreads) lpa_keys[i] = i < c ? keys[i] : ~0ull;
    if (tid == 0) kept = 0;
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
        for (int k = 2; k <= c2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < c2; i += kLpaSortThreads) {
                    const int partner = i ^ j;
                    if (partner > i) {
                        const unsigned long long x = lpa_keys[i], y = lpa_keys[partner];
                        if ((x > y) == ((i & k) == 0)) {
                            lpa_keys[i] = y;
                            lpa_keys[partner] = x;
                        }
                    }
                }
                __syncthreads();
            }
        if (pass == 1) break;
        // repeats are adjacent now: all but the first of a run become padding, and a second sort moves them to the end
        unsigned long long mine[16];  // c2 <= 16384 = 16 x 1024
        int cnt = 0;
        for (int i = tid, t = 0; i < c2; i += kLpaSortThreads, ++t) {
            const unsigned long long x = lpa_keys[i];
            const bool repeat = x != ~0ull && i > 0 && lpa_keys[i - 1] == x;
            mine[t] = repeat ? ~0ull : x;
            cnt += (x != ~0ull && !repeat);
        }
        __syncthreads();
        for (int i = tid, t = 0; i < c2; i += kLpaSortThreads, ++t) lpa_keys[i] = mine[t];
        if (cnt) atomicAdd(&kept, cnt);
        __syncthreads();
    }
    const int distinct = kept;
    for (int i = tid; i < distinct; i += kLpaSortThreads) {
        const unsigned long long x = lpa_keys[i];
        keys[i] = x;
        atomicAdd(&deg[static_cast<size_t>(r) * n + static_cast<int>(x >> 32)], 1);
        atomicAdd(&deg[static_cast<size_t>(r) * n + static_cast<int>(x & 0xffffffffu)], 1);
    }
    __syncthreads();
    if (tid == 0) add_count[r] = distinct;
}

// One CTA per individual: row_ptr' = exclusive scan of the perturbed degrees, rows = surviving CSR neighbours (ascending)
// followed by the added ones, then rows that received additions are put back in ascending order.
__global__ void __launch_bounds__(kLpaSortThreads) k_lpa_flip_build(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                                                    const int32_t* __restrict__ edge_id, int n, int mask_words,
                                                                    const unsigned* __restrict__ gone, const int32_t* __restrict__ deg,
                                                                    const unsigned long long* __restrict__ add_keys, const int* __restrict__ add_count,
                                                                    int cols, size_t col2_stride, int32_t* row_ptr2, int32_t* col2, int32_t* base_cnt) {
    griddep_launch();
    griddep_wait();
    __shared__ int sh_scan[kLpaSortThreads];
    const int r = blockIdx.x, tid = threadIdx.x;
    const unsigned* mask = gone + static_cast<size_t>(r) * mask_words;
    const int32_t* d = deg + static_cast<size_t>(r) * n;
    int32_t* rp = row_ptr2 + static_cast<size_t>(r) * (n + 1);
    int32_t* col = col2 + static_cast<size_t>(r) * col2_stride;
    int32_t* fill = base_cnt + static_cast<size_t>(r) * 3 * n;  // entries written so far
    int32_t* base = fill + n;                                      // neighbours that came from the CSR (ascending)
    int32_t* min_added = base + n;                                 // smallest added neighbour: its thread sorts the row
    const int per = (n + kLpaSortThreads - 1) / kLpaSortThreads;
    const int x0 = min(n, tid * per), x1 = min(n, x0 + per);
    int local = 0;
    for (int x = x0; x < x1; ++x) local += d[x];
    sh_scan[tid] = local;
    __syncthreads();
    for (int off = 1; off < kLpaSortThreads; off <<= 1) {
        const int t = tid >= off ? sh_scan[tid - off] : 0;
        __syncthreads();
        sh_scan[tid] += t;
        __syncthreads();
    }
    int run = sh_scan[tid] - local;
    for (int x = x0; x < x1; ++x) {
        rp[x] = run;
        int cnt = 0;
        for (int e = row_ptr[x]; e < row_ptr[x + 1]; ++e) {
            const int id = edge_id[e];
            if (!((mask[id >> 5] >> (id & 31)) & 1u)) col[run + cnt++] = col_idx[e];
        }
        fill[x] = cnt;
        base[x] = cnt;
        min_added[x] = 0x7fffffff;
        run += d[x];
    }
    if (tid == kLpaSortThreads - 1) rp[n] = sh_scan[tid];
    __syncthreads();
    const int added = add_count[r];
    const unsigned long long* keys = add_keys + static_cast<size_t>(r) * cols;
    for (int i = tid; i < added; i += kLpaSortThreads) {
        const int a = static_cast<int>(keys[i] >> 32), b = static_cast<int>(keys[i] & 0xffffffffu);
        col[rp[a] + atomicAdd(&fill[a], 1)] = b;
        col[rp[b] + atomicAdd(&fill[b], 1)] = a;
        atomicMin(&min_added[a], b);
        atomicMin(&min_added[b], a);
    }
    __syncthreads();
    // a row that received additions: its tail is in arrival order — insertion sort (rows are short)
    for (int i = tid; i < 2 * added; i += kLpaSortThreads) {
        const unsigned long long key = keys[i >> 1];
        const int x = (i & 1) ? static_cast<int>(key & 0xffffffffu) : static_cast<int>(key >> 32);
        // one thread per row: the one holding the row's SMALLEST added neighbour does the sort
        const int other = (i & 1) ? static_cast<int>(key >> 32) : static_cast<int>(key & 0xffffffffu);
        if (other != min_added[x]) continue;
        const int len = d[x];
        int32_t* row = col + rp[x];
        for (int t = base[x]; t < len; ++t) {
            const int v = row[t];
            int q = t - 1;
            while (q >= 0 && row[q] > v) { row[q + 1] = row[q]; --q; }
            row[q + 1] = v;
        }
    }
}

// score of every (individual, pair) on the individual's own perturbed CSR; deg'(z) = its row length
__global__ void __launch_bounds__(kLpaThreads) k_lpa_scores_plain(const int32_t* __restrict__ row_ptr2, const int32_t* __restrict__ col2,
                                                                  size_t col2_stride, const int32_t* __restrict__ pairs, int n_pairs, int n,
                                                                  double* __restrict__ scores, int cn) {
    griddep_launch();
    griddep_wait();
    const int r = blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_pairs) return;
    const int32_t* rp = row_ptr2 + static_cast<size_t>(r) * (n + 1);
    const int32_t* col = col2 + static_cast<size_t>(r) * col2_stride;
    const int u = pairs[2 * q], v = pairs[2 * q + 1];
    int i = rp[u], j = rp[v];
    const int ie = rp[u + 1], je = rp[v + 1];
    double score = 0.0;
    while (i < ie && j < je) {
        const int a = col[i], b = col[j];
        if (a < b) ++i;
        else if (b < a) ++j;
        else {
            const int dz = rp[a + 1] - rp[a];
            if (dz > 0) score += cn ? 1.0 : 1.0 / static_cast<double>(dz);
            ++i;
            ++j;
        }
    }
    scores[static_cast<size_t>(r) * n_pairs + q] = score;
}

__global__ void k_lpa_final(const unsigned long long* __restrict__ twice, int rows, int T, int P, double* out) {
    griddep_launch();
    griddep_wait();
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
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_lpa_flip_unique, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    const int n = ctx->n, T = ctx->T, P = ctx->P, n_pairs = T + P;
    const int mask_words = static_cast<int>((ctx->m + 31) / 32) + 1;
    const bool flips = ctx->pool_kind == GAPA_POOL_EDGE_FLIP;
    const int cn = ctx->lp_score == GAPA_LP_SCORE_CN ? 1 : 0;
    const size_t col2_stride = static_cast<size_t>(2 * ctx->m) + 2 * static_cast<size_t>(cols) + 1;
    if (flips && cols > 16384) return fail(GAPA_CUDA_E_INVALID, "lpa_fitness: an edge-flip budget beyond 16384 genes is not supported");
    const size_t per_row = sizeof(unsigned) * mask_words + sizeof(int32_t) * n + sizeof(double) * n_pairs +
                           (flips ? sizeof(unsigned long long) * cols + sizeof(int32_t) * (4 * static_cast<size_t>(n) + 1 + col2_stride) : 0);
    size_t budget = 8ull << 30;  // scratch per pass; GAPA_SCRATCH_MB overrides (tests force several passes)
    if (const char* raw = std::getenv("GAPA_SCRATCH_MB")) budget = static_cast<size_t>(std::max(1L, std::strtol(raw, nullptr, 10))) << 20;
    const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(rows, budget / per_row)));
    GAPA_TRY(s->gone.ensure(sizeof(unsigned) * mask_words * static_cast<size_t>(chunk)));
    GAPA_TRY(s->deg.ensure(sizeof(int32_t) * std::max(n, 1) * static_cast<size_t>(chunk)));
    GAPA_TRY(s->scores.ensure(sizeof(double) * n_pairs * static_cast<size_t>(chunk)));
    GAPA_TRY(s->twice.ensure(sizeof(unsigned long long) * chunk));
    GAPA_TRY(s->status.ensure(sizeof(int)));
    if (flips) {
        GAPA_TRY(s->add_keys.ensure(sizeof(unsigned long long) * std::max(cols, 1) * static_cast<size_t>(chunk)));
        GAPA_TRY(s->add_count.ensure(sizeof(int) * chunk));
        GAPA_TRY(s->row_ptr2.ensure(sizeof(int32_t) * (static_cast<size_t>(n) + 1) * chunk));
        GAPA_TRY(s->col2.ensure(sizeof(int32_t) * col2_stride * chunk));
        GAPA_TRY(s->base_cnt.ensure(sizeof(int32_t) * 3 * static_cast<size_t>(std::max(n, 1)) * chunk));
    }
    int* status = s->status.as<int>();
    GAPA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), stream));
    const int sm = ctx->sm_count;
    for (int r0 = 0; r0 < rows; r0 += chunk) {
        const int cr = std::min(chunk, rows - r0);
        GAPA_CUDA_TRY(cudaMemsetAsync(s->gone.ptr, 0, sizeof(unsigned) * mask_words * static_cast<size_t>(cr), stream));
        if (n > 0) GAPA_LAUNCH(k_lpa_init, sm * 8, kLpaThreads, 0, stream, ctx->d_row_ptr, n, cr, s->deg.as<int32_t>());
        const size_t cells = static_cast<size_t>(cr) * cols;
        if (flips) {
            // classify -> distinct additions -> per-individual perturbed CSR -> scores on it (then the shared AUC kernels)
            GAPA_CUDA_TRY(cudaMemsetAsync(s->add_count.ptr, 0, sizeof(int) * cr, stream));
            if (cells) {
                const int grid = static_cast<int>(std::min<size_t>((cells + kLpaThreads - 1) / kLpaThreads, static_cast<size_t>(sm) * 32));
                GAPA_LAUNCH(k_lpa_flip_classify, grid, kLpaThreads, 0, stream, genes.from(r0), cells, ctx->pool_size, n,
                            ctx->flip_canonical ? nullptr : ctx->d_add_u, ctx->flip_canonical ? nullptr : ctx->d_add_v, ctx->d_row_ptr,
                            ctx->d_col_idx, ctx->d_edge_id, mask_words, s->gone.as<unsigned>(), s->deg.as<int32_t>(),
                            s->add_keys.as<unsigned long long>(), s->add_count.as<int>(), status);
                int c2 = 2;
                while (c2 < cols) c2 <<= 1;
                GAPA_LAUNCH(k_lpa_flip_unique, cr, kLpaSortThreads, sizeof(unsigned long long) * c2, stream, cols, n,
                            s->add_keys.as<unsigned long long>(), s->add_count.as<int>(), s->deg.as<int32_t>());
            }
            GAPA_LAUNCH(k_lpa_flip_build, cr, kLpaSortThreads, 0, stream, ctx->d_row_ptr, ctx->d_col_idx, ctx->d_edge_id, n, mask_words,
                        s->gone.as<unsigned>(), s->deg.as<int32_t>(), s->add_keys.as<unsigned long long>(), s->add_count.as<int>(),
                        std::max(cols, 1), col2_stride, s->row_ptr2.as<int32_t>(), s->col2.as<int32_t>(), s->base_cnt.as<int32_t>());
            GAPA_LAUNCH(k_lpa_scores_plain, dim3((n_pairs + kLpaThreads - 1) / kLpaThreads, cr), kLpaThreads, 0, stream,
                        s->row_ptr2.as<int32_t>(), s->col2.as<int32_t>(), col2_stride, ctx->d_pairs, n_pairs, n, s->scores.as<double>(), cn);
        } else if (cells) {
            const int grid = static_cast<int>(std::min<size_t>((cells + kLpaThreads - 1) / kLpaThreads, static_cast<size_t>(sm) * 32));
            GAPA_LAUNCH(k_lpa_remove, grid, kLpaThreads, 0, stream, genes.from(r0), cells,
                        ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, ctx->d_edge_u, ctx->d_edge_v, n,
                        mask_words, s->gone.as<unsigned>(), s->deg.as<int32_t>(), status);
        }
        if (!flips)
        GAPA_LAUNCH(k_lpa_scores, dim3((n_pairs + kLpaThreads - 1) / kLpaThreads, cr), kLpaThreads, 0, stream, ctx->d_row_ptr,
                    ctx->d_col_idx, ctx->d_edge_id, ctx->d_pairs, n_pairs, n, mask_words, s->gone.as<unsigned>(),
                    s->deg.as<int32_t>(), s->scores.as<double>(), ctx->lp_score == GAPA_LP_SCORE_CN ? 1 : 0);
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
    for (DevBuf* b : {&ctx->lpa->gone, &ctx->lpa->deg, &ctx->lpa->scores, &ctx->lpa->twice, &ctx->lpa->status, &ctx->lpa->add_keys,
                      &ctx->lpa->add_count, &ctx->lpa->row_ptr2, &ctx->lpa->col2, &ctx->lpa->base_cnt})
        b->release();
    delete ctx->lpa;
    ctx->lpa = nullptr;
}

}  // namespace gapa_b200
