// Genetic operators on HBM-resident populations — device twins of
// /root/reference/proj/src/ga_ops.cpp, keyed by the same counter-based streams
// (include/gapa/rng.hpp), so every matrix equals the reference's bit for bit.
//
// Because draw j of a stream is mix64(key + C*j) (rng.hpp:21), element (row, col)
// needs only the row's key and j = col + 1: one thread per gene, no sequential
// state, any row partition gives the same result.
#include <algorithm>
#include <cmath>
#include <map>

#include "internal.cuh"

namespace gapa_b200 {

static constexpr int kGaThreads = 256;

// ---- init_population_block (ga_ops.cpp:19-29) ----------------------------------------
__global__ void __launch_bounds__(kGaThreads) k_ga_init(uint32_t pool_size, int row_first, int budget, uint64_t seed,
                                                        uint64_t generation, int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t key;
    const int row = blockIdx.y;
    if (threadIdx.x == 0) key = stream_key(seed, generation, GAPA_ROLE_INIT, static_cast<uint64_t>(row_first + row));
    __syncthreads();
    const uint64_t k = key;
    int32_t* dst = out + static_cast<size_t>(row) * budget;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < budget; j += gridDim.x * blockDim.x)
        dst[j] = static_cast<int32_t>(draw_index(k, static_cast<uint64_t>(j) + 1, pool_size));
}

// ---- make_crossover_mask / make_mutation_mask (ga_ops.cpp:38-47, :84-92) and make_mutation_indices (:94-103) ------
// The matrices the fused variation kernels never materialise, for hosts and tests that want them:
// mask(i, j) = stream(generation, role, row_first + i).next_bernoulli(rate) at draw j + 1 (1 or 0, MaskMatrix bytes).
__global__ void __launch_bounds__(kGaThreads) k_ga_mask(uint64_t role, int row_first, int cols, uint64_t limit, bool always,
                                                        uint64_t seed, uint64_t generation, uint8_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t key;
    const int row = blockIdx.y;
    if (threadIdx.x == 0) key = stream_key(seed, generation, role, static_cast<uint64_t>(row_first + row));
    __syncthreads();
    const uint64_t k = key;
    uint8_t* dst = out + static_cast<size_t>(row) * cols;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x)
        dst[j] = (always || draw_u64(k, static_cast<uint64_t>(j) + 1) < limit) ? 1 : 0;
}
// fresh(i, j) = stream(generation, MutationIndex, row_first + i).next_index(pool) at draw j + 1
__global__ void __launch_bounds__(kGaThreads) k_ga_mutation_indices(uint32_t pool_size, int row_first, int cols, uint64_t seed,
                                                                    uint64_t generation, int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t key;
    const int row = blockIdx.y;
    if (threadIdx.x == 0) key = stream_key(seed, generation, GAPA_ROLE_MUTATION_INDEX, static_cast<uint64_t>(row_first + row));
    __syncthreads();
    const uint64_t k = key;
    int32_t* dst = out + static_cast<size_t>(row) * cols;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x)
        dst[j] = static_cast<int32_t>(draw_index(k, static_cast<uint64_t>(j) + 1, pool_size));
}

// ---- crossover (ga_ops.cpp:130-144) fused with mutate_block (:164-178) -------------------
// out(i,j) = RM(i,j) ? fresh(i,j) : (RC(i,j) ? pop(partner_i, j) : pop(i, j)).
// All three draws are random-access, so a flipped gene skips the crossover draw
// and both loads; the result is unchanged.
__global__ void __launch_bounds__(kGaThreads) k_ga_crossover_mutate(
    const int32_t* __restrict__ pop, const int32_t* __restrict__ partner, int k, int row_first, uint64_t pc_thr,
    uint64_t pm_thr, uint32_t pool_size, uint64_t seed, uint64_t generation, int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[3];
    const int row = row_first + blockIdx.y;
    if (threadIdx.x < 3)
        keys[threadIdx.x] = stream_key(seed, generation, GAPA_ROLE_CROSSOVER_MASK + threadIdx.x, static_cast<uint64_t>(row));
    __syncthreads();
    const uint64_t kc = keys[0], km = keys[1], ki = keys[2];
    const int32_t* mine = pop + static_cast<size_t>(row) * k;
    const int32_t* theirs = pop + static_cast<size_t>(partner[row]) * k;
    int32_t* dst = out + static_cast<size_t>(blockIdx.y) * k;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        const uint64_t d = static_cast<uint64_t>(j) + 1;
        int32_t g;
        if (draw_bernoulli(km, d, pm_thr)) g = static_cast<int32_t>(draw_index(ki, d, pool_size));
        else g = draw_bernoulli(kc, d, pc_thr) ? theirs[j] : mine[j];
        dst[j] = g;
    }
}

// Four genes per thread (16-byte loads / stores), all draws of a gene share the product C * j,
// the golden-ratio add of mix64 is folded into the row keys, and the 53-bit Bernoulli test
// (u >> 11) < T is done as u < (T << 11).  Every gene evaluates all three draws: inside a warp
// both sides of the mutate / crossover branch are taken anyway, and straight-line code keeps
// twelve independent hash chains in flight.  Results are identical to the scalar kernel.
__device__ __forceinline__ uint64_t mix64_tail(uint64_t y) {  // mix64(x) with y = x + 0x9E3779B97F4A7C15
    y = (y ^ (y >> 30)) * 0xBF58476D1CE4E5B9ull;
    y = (y ^ (y >> 27)) * 0x94D049BB133111EBull;
    return y ^ (y >> 31);
}
struct BernoulliLimit {  // (u >> 11) < threshold  <=>  always || u < limit
    uint64_t limit;
    bool always;
};
static BernoulliLimit bernoulli_limit(double p) {
    const uint64_t t = bernoulli_threshold(p);
    return {t >= (1ull << 53) ? ~0ull : t << 11, t >= (1ull << 53)};
}

__global__ void __launch_bounds__(kGaThreads) k_ga_crossover_mutate4(
    const int32_t* __restrict__ pop, const int32_t* __restrict__ partner, int k, int row_first, uint64_t pc_limit,
    bool pc_always, uint64_t pm_limit, bool pm_always, uint32_t pool_size, uint64_t seed, uint64_t generation,
    int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[3];
    const int row = row_first + blockIdx.y;
    if (threadIdx.x < 3)
        keys[threadIdx.x] = stream_key(seed, generation, GAPA_ROLE_CROSSOVER_MASK + threadIdx.x, static_cast<uint64_t>(row)) +
                            0x9E3779B97F4A7C15ull;
    __syncthreads();
    const uint64_t kc = keys[0], km = keys[1], ki = keys[2];
    const int4* mine = reinterpret_cast<const int4*>(pop + static_cast<size_t>(row) * k);
    const int4* theirs = reinterpret_cast<const int4*>(pop + static_cast<size_t>(partner[row]) * k);
    int4* dst = reinterpret_cast<int4*>(out + static_cast<size_t>(blockIdx.y) * k);
    const int quads = k >> 2;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += gridDim.x * blockDim.x) {
        const int4 a = mine[q], b = theirs[q];
        const int av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        int r[4];
        uint64_t prod = 0x632BE59BD9B4E019ull * (static_cast<uint64_t>(q) * 4 + 1);  // C * j, j = column + 1
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint64_t um = mix64_tail(km + prod), ux = mix64_tail(kc + prod), ui = mix64_tail(ki + prod);
            const bool flip = pm_always || um < pm_limit;
            const bool take = pc_always || ux < pc_limit;
            const int fresh = static_cast<int>(__umul64hi(ui, static_cast<uint64_t>(pool_size)));
            r[t] = flip ? fresh : (take ? bv[t] : av[t]);
            prod += 0x632BE59BD9B4E019ull;
        }
        dst[q] = make_int4(r[0], r[1], r[2], r[3]);
    }
}

// ---- mutate_block alone (ga_ops.cpp:164-178) ------------------------------------------------
__global__ void __launch_bounds__(kGaThreads) k_ga_mutate(const int32_t* __restrict__ block, int k, int row_offset,
                                                          uint64_t pm_thr, uint32_t pool_size, uint64_t seed,
                                                          uint64_t generation, int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[2];
    const int row = row_offset + blockIdx.y;
    if (threadIdx.x < 2)
        keys[threadIdx.x] = stream_key(seed, generation, GAPA_ROLE_MUTATION_MASK + threadIdx.x, static_cast<uint64_t>(row));
    __syncthreads();
    const uint64_t km = keys[0], ki = keys[1];
    const int32_t* src = block + static_cast<size_t>(blockIdx.y) * k;
    int32_t* dst = out + static_cast<size_t>(blockIdx.y) * k;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        const uint64_t d = static_cast<uint64_t>(j) + 1;
        dst[j] = draw_bernoulli(km, d, pm_thr) ? static_cast<int32_t>(draw_index(ki, d, pool_size)) : src[j];
    }
}

// ---- eda_sample (ga_ops.cpp:214-238) ----------------------------------------------------------
__global__ void __launch_bounds__(kGaThreads) k_ga_eda(const int32_t* __restrict__ elite, int k, uint32_t elite_count,
                                                       uint32_t bound, int row_first, uint64_t seed, uint64_t generation,
                                                       int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t key;
    const int row = row_first + blockIdx.y;  // out holds rows [row_first, row_first + gridDim.y)
    if (threadIdx.x == 0) key = stream_key(seed, generation, GAPA_ROLE_SELECT, static_cast<uint64_t>(row));
    __syncthreads();
    const uint64_t kk = key;
    int32_t* dst = out + static_cast<size_t>(blockIdx.y) * k;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        const uint32_t v = draw_index(kk, static_cast<uint64_t>(j) + 1, bound);
        dst[j] = v < elite_count ? elite[static_cast<size_t>(v) * k + j] : static_cast<int32_t>(v - elite_count);
    }
}

// ---- selection_weights (ga_ops.cpp:54-76) --------------------------------------------------------
// The reference stable-sorts, then gives every tie span [i, j) the average of the
// rank weights s-i .. s-j+1.  For element x that is i = #{strictly better},
// j = #{better or equal}; counting replaces the sort (O(s^2) compares, s <= 16k).
__device__ __forceinline__ bool better(double a, double b, int minimize) { return minimize ? a < b : a > b; }

// kSplit lanes share one element and each scans 1/kSplit of every tile, so s elements
// give s / 32 blocks instead of s / 256 (s is only a few thousand).
static constexpr int kSplit = 8;
static constexpr int kPerBlock = kGaThreads / kSplit;

__global__ void __launch_bounds__(kGaThreads) k_ga_weights(const double* __restrict__ fitness, int s, int minimize,
                                                           double* __restrict__ weights, int* status, double* stats_best,
                                                           double* stats_mean) {
    griddep_launch();
    griddep_wait();
    __shared__ unsigned long long tile[kGaThreads];
    if (stats_best && blockIdx.x == gridDim.x - 1) {
        // one extra block: best / mean of this population for the run's history (run.cu defers them to this launch)
        __shared__ GaStatsSmem stats_sm;
        ga_stats_block(fitness, s, stats_best, stats_mean, stats_sm);
        return;
    }
    const int i = blockIdx.x * kPerBlock + threadIdx.x / kSplit, part = threadIdx.x % kSplit;
    const double mine_f = i < s ? fitness[i] : 0.0;
    if (i < s && !isfinite(mine_f)) *status = GAPA_CUDA_E_NAN;
    const unsigned long long mine = order_key(mine_f, minimize);
    int less = 0, leq = 0;
    // After an elitism step the population is sorted best-first: the rows better than mine are a prefix and my ties
    // a contiguous run, so two binary searches replace the s compares (every block checks the order itself: s compares
    // against its own 32 * s).
    int in_order = 1;
    for (int t = threadIdx.x; t + 1 < s; t += kGaThreads) in_order &= order_key(fitness[t], minimize) <= order_key(fitness[t + 1], minimize);
    if (__syncthreads_and(in_order)) {
        if (i < s && part == 0) {
            int a = 0, b = i;  // first row not better than mine
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (order_key(fitness[mid], minimize) < mine) a = mid + 1; else b = mid;
            }
            less = a;
            a = i + 1, b = s;  // first row worse than mine
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (order_key(fitness[mid], minimize) <= mine) a = mid + 1; else b = mid;
            }
            leq = a;
            weights[i] = (static_cast<double>(s - less) + static_cast<double>(s - leq + 1)) / 2.0;
        }
        return;
    }
    for (int t0 = 0; t0 < s; t0 += kGaThreads) {
        __syncthreads();
        if (t0 + threadIdx.x < s) tile[threadIdx.x] = order_key(fitness[t0 + threadIdx.x], minimize);
        __syncthreads();
        const int lim = min(kGaThreads, s - t0);
        for (int t = part; t < lim; t += kSplit) {
            const unsigned long long other = tile[t];
            less += other < mine;
            leq += other <= mine;
        }
    }
    for (int off = kSplit / 2; off; off >>= 1) {
        less += __shfl_down_sync(0xffffffffu, less, off, kSplit);
        leq += __shfl_down_sync(0xffffffffu, leq, off, kSplit);
    }
    if (i < s && part == 0) weights[i] = (static_cast<double>(s - less) + static_cast<double>(s - leq + 1)) / 2.0;
}

// cumulative sum + weighted_pick (ga_ops.cpp:78-82, :113-126), one block.
// Weights are half-integers with total <= s(s+1)/2 < 2^53: every partial sum is
// exact, so the parallel scan equals the reference's sequential running total.
static constexpr int kPickSmemRows = 24576;  // 192 KB of running totals
__global__ void __launch_bounds__(1024) k_ga_pick(const double* __restrict__ weights, int s, uint64_t seed,
                                                  uint64_t generation, double* __restrict__ cumulative,
                                                  int32_t* __restrict__ partner, int in_smem, int phase) {
    griddep_launch();
    griddep_wait();
    // phase 0: scan + picks in one launch (the totals fit shared memory: every block redoes the scan and picks its 1024
    // rows).  Populations beyond that: phase 1 = one block scans into `cumulative`, phase 2 = every block picks its rows
    // from it (searches in L2) — instead of one block doing all s searches (s = 32,768: 0.18 ms).
    // The running totals live in shared memory when they fit (s <= kPickSmemRows): the s binary searches below are
    // chains of ~log2 s dependent reads, 30 ns each from shared memory against 300+ ns from L2.
    extern __shared__ double pick_cum[];
    __shared__ double warp_total[32];
    __shared__ double carry_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry_s = 0.0;
    __syncthreads();
    if (phase != 2)
    for (int t0 = 0; t0 < s; t0 += 1024) {  // tile-wise inclusive scan: warp shuffles, warp totals, running carry
        const int i = t0 + tid;
        double v = i < s ? weights[i] : 0.0;
        for (int off = 1; off < 32; off <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v += t;
        }
        if (lane == 31) warp_total[wid] = v;
        __syncthreads();
        if (wid == 0) {
            double t = warp_total[lane];
            for (int off = 1; off < 32; off <<= 1) {
                const double u = __shfl_up_sync(0xffffffffu, t, off);
                if (lane >= off) t += u;
            }
            warp_total[lane] = t;
        }
        __syncthreads();
        v += carry_s + (wid > 0 ? warp_total[wid - 1] : 0.0);
        if (i < s) {
            if (blockIdx.x == 0 || !in_smem) cumulative[i] = v;  // every block scans (cheap); one publishes the totals
            if (in_smem) pick_cum[i] = v;
        }
        __syncthreads();
        if (tid == 1023) carry_s = v;
    }
    __syncthreads();
    if (phase == 1) return;
    const double total = phase == 2 ? cumulative[s - 1] : carry_s;
    const double* cum = in_smem ? pick_cum : cumulative;
    // the picks are chains of dependent instructions (four mix64 for the stream key, log2 s search steps): with the
    // totals in shared memory every block redoes the scan and then picks for its own 1024 rows, one row per thread
    for (int i = blockIdx.x * 1024 + tid; i < s; i += gridDim.x * 1024) {
        const double target = draw_unit(stream_key(seed, generation, GAPA_ROLE_SELECT, static_cast<uint64_t>(i)), 1) * total;
        int a = 0, b = s;  // std::upper_bound: first index with cumulative > target
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (cum[mid] <= target) a = mid + 1; else b = mid;
        }
        partner[i] = min(a, s - 1);
    }
}

// selection_weights + cumulative sum + weighted_pick in ONE block for s <= 1024: small populations are
// launch-latency-bound (C1: seven launches of 3-5 us per generation), so the loop fuses what it can.
__global__ void __launch_bounds__(1024) k_ga_select_small(const double* __restrict__ fitness, int s, int minimize, uint64_t seed,
                                                          uint64_t generation, double* __restrict__ weights,
                                                          double* __restrict__ cumulative, int32_t* __restrict__ partner,
                                                          int* status) {
    griddep_launch();
    griddep_wait();
    __shared__ double f[1024];
    __shared__ double part[1024];
    const int tid = threadIdx.x;
    const double mine = tid < s ? fitness[tid] : 0.0;
    if (tid < s) {
        f[tid] = mine;
        if (!isfinite(mine)) *status = GAPA_CUDA_E_NAN;
    }
    __syncthreads();
    double w = 0.0;
    if (tid < s) {
        int less = 0, leq = 0;
        for (int t = 0; t < s; ++t) {
            const double other = f[t];
            const bool b = better(other, mine, minimize);
            less += b;
            leq += b || other == mine;
        }
        w = (static_cast<double>(s - less) + static_cast<double>(s - leq + 1)) / 2.0;
        weights[tid] = w;
    }
    part[tid] = w;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // half-integers below 2^53: exact in any order
        const double add = tid >= off ? part[tid - off] : 0.0;
        __syncthreads();
        part[tid] += add;
        __syncthreads();
    }
    if (tid < s) cumulative[tid] = part[tid];
    const double total = part[s - 1];
    if (tid < s) {
        const double target = draw_unit(stream_key(seed, generation, GAPA_ROLE_SELECT, static_cast<uint64_t>(tid)), 1) * total;
        int a = 0, b = s;  // std::upper_bound: first index with cumulative > target
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (part[mid] <= target) a = mid + 1; else b = mid;
        }
        partner[tid] = min(a, s - 1);
    }
}

// ---- elitism (ga_ops.cpp:180-212) ---------------------------------------------------------------------
// Position of stacked row x in the stable best-first order = #{y : better(y, x) or
// (equal and y < x)}; originals (index < s) therefore precede mutated rows on ties.
__global__ void __launch_bounds__(kGaThreads) k_ga_elite_rank(const double* __restrict__ fit, const double* __restrict__ fit_m,
                                                              int s, int minimize, int32_t* __restrict__ src_of_rank,
                                                              int* status) {
    griddep_launch();
    griddep_wait();
    __shared__ unsigned long long tile[kGaThreads];
    const int x = blockIdx.x * kPerBlock + threadIdx.x / kSplit, part = threadIdx.x % kSplit;
    const int total = 2 * s;
    const double mine_f = x < total ? (x < s ? fit[x] : fit_m[x - s]) : 0.0;
    if (x < total && isnan(mine_f)) *status = GAPA_CUDA_E_NAN;
    const unsigned long long mine = order_key(mine_f, minimize);
    int rank = 0;
    for (int t0 = 0; t0 < total; t0 += kGaThreads) {
        __syncthreads();
        const int y = t0 + threadIdx.x;
        if (y < total) tile[threadIdx.x] = order_key(y < s ? fit[y] : fit_m[y - s], minimize);
        __syncthreads();
        const int lim = min(kGaThreads, total - t0);
        for (int t = part; t < lim; t += kSplit) {
            const unsigned long long other = tile[t];
            rank += (other < mine) | ((other == mine) & (t0 + t < x));
        }
    }
    for (int off = kSplit / 2; off; off >>= 1) rank += __shfl_down_sync(0xffffffffu, rank, off, kSplit);
    if (x < total && part == 0 && rank < s) src_of_rank[rank] = x;
}

__global__ void __launch_bounds__(kGaThreads) k_ga_elite_gather(const int32_t* __restrict__ pop,
                                                                const int32_t* __restrict__ m_pop,
                                                                const double* __restrict__ fit,
                                                                const double* __restrict__ fit_m, int s, int k,
                                                                const int32_t* __restrict__ src_of_rank,
                                                                int32_t* __restrict__ next, double* __restrict__ next_fit) {
    griddep_launch();
    griddep_wait();
    const int r = blockIdx.y;
    const int src = src_of_rank[r];
    const int32_t* from = src < s ? pop + static_cast<size_t>(src) * k : m_pop + static_cast<size_t>(src - s) * k;
    int32_t* to = next + static_cast<size_t>(r) * k;
    if (((reinterpret_cast<uintptr_t>(from) | reinterpret_cast<uintptr_t>(to)) & 15) == 0 && (k & 3) == 0) {
        const int4* from4 = reinterpret_cast<const int4*>(from);
        int4* to4 = reinterpret_cast<int4*>(to);
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < (k >> 2); j += gridDim.x * blockDim.x) to4[j] = __ldcs(&from4[j]);
    } else {
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) to[j] = from[j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) next_fit[r] = src < s ? fit[src] : fit_m[src - s];
}

__global__ void k_rng_draws(uint64_t seed, uint64_t generation, uint64_t role, uint64_t row, int count, uint64_t* out) {
    griddep_launch();
    griddep_wait();
    const uint64_t key = stream_key(seed, generation, role, row);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x)
        out[j] = draw_u64(key, static_cast<uint64_t>(j) + 1);
}

// ---- launch helpers (no synchronisation; shared with run.cu) ------------------------------------------
static dim3 row_grid(int cols, int rows) {
    const int per_block = kGaThreads * 8;  // 8 genes per thread keeps the per-row key setup amortised
    return dim3(std::max(1, std::min((cols + per_block - 1) / per_block, 65535)), rows);
}

int launch_init(uint32_t pool_size, int row_first, int row_count, int budget, uint64_t seed, uint64_t generation,
                int32_t* out, cudaStream_t st) {
    if (row_count == 0 || budget == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_init, row_grid(budget, row_count), kGaThreads, 0, st, pool_size, row_first, budget, seed, generation, out);
    return GAPA_CUDA_OK;
}
int launch_select(const double* fitness, int s, int minimize, uint64_t seed, uint64_t generation, int32_t* partner,
                  double* weights, double* cumulative, int* status, cudaStream_t st, double* stats_best = nullptr,
                  double* stats_mean = nullptr) {
    if (s <= 1024) {
        if (stats_best) return fail(GAPA_CUDA_E_INVALID, "select: statistics ride only on the multi-block selection");
        GAPA_LAUNCH(k_ga_select_small, 1, 1024, 0, st, fitness, s, minimize, seed, generation, weights, cumulative, partner, status);
        return GAPA_CUDA_OK;
    }
    GAPA_LAUNCH(k_ga_weights, (s + kPerBlock - 1) / kPerBlock + (stats_best ? 1 : 0), kGaThreads, 0, st, fitness, s, minimize, weights, status,
                stats_best, stats_mean);
    const int in_smem = s <= kPickSmemRows ? 1 : 0;
    const size_t pick_smem = in_smem ? sizeof(double) * static_cast<size_t>(s) : 0;
    if (pick_smem > 48 * 1024)  // per device and cheap: set whenever the launch needs it
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_ga_pick, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(double) * kPickSmemRows));
    if (in_smem) {
        GAPA_LAUNCH(k_ga_pick, (s + 1023) / 1024, 1024, pick_smem, st, weights, s, seed, generation, cumulative, partner, 1, 0);
    } else {
        GAPA_LAUNCH(k_ga_pick, 1, 1024, 0, st, weights, s, seed, generation, cumulative, partner, 0, 1);
        GAPA_LAUNCH(k_ga_pick, (s + 1023) / 1024, 1024, 0, st, weights, s, seed, generation, cumulative, partner, 0, 2);
    }
    return GAPA_CUDA_OK;
}
int launch_crossover_mutate(const int32_t* pop, const int32_t* partner, int k, int row_first, int row_count, double pc,
                            double pm, uint32_t pool_size, uint64_t seed, uint64_t generation, int32_t* out,
                            cudaStream_t st) {
    if (row_count == 0 || k == 0) return GAPA_CUDA_OK;
    if ((k & 3) == 0 && ((reinterpret_cast<uintptr_t>(pop) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        const BernoulliLimit c = bernoulli_limit(pc), m = bernoulli_limit(pm);
        GAPA_LAUNCH(k_ga_crossover_mutate4, row_grid(k / 4, row_count), kGaThreads, 0, st, pop, partner, k, row_first, c.limit,
                    c.always, m.limit, m.always, pool_size, seed, generation, out);
        return GAPA_CUDA_OK;
    }
    GAPA_LAUNCH(k_ga_crossover_mutate, row_grid(k, row_count), kGaThreads, 0, st, pop, partner, k, row_first,
                bernoulli_threshold(pc), bernoulli_threshold(pm), pool_size, seed, generation, out);
    return GAPA_CUDA_OK;
}
int launch_mutate(const int32_t* block, int rows, int k, int row_offset, double pm, uint32_t pool_size, uint64_t seed,
                  uint64_t generation, int32_t* out, cudaStream_t st) {
    if (rows == 0 || k == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_mutate, row_grid(k, rows), kGaThreads, 0, st, block, k, row_offset, bernoulli_threshold(pm), pool_size,
                seed, generation, out);
    return GAPA_CUDA_OK;
}
int launch_eda(const int32_t* elite, int row_first, int row_count, int k, int elite_count, uint32_t bound, uint64_t seed,
               uint64_t generation, int32_t* out, cudaStream_t st) {
    if (row_count == 0 || k == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_eda, row_grid(k, row_count), kGaThreads, 0, st, elite, k, static_cast<uint32_t>(elite_count), bound,
                row_first, seed, generation, out);
    return GAPA_CUDA_OK;
}
int launch_elitism(const int32_t* pop, const int32_t* m_pop, int s, int k, const double* fit, const double* fit_m,
                   int minimize, int32_t* next, double* next_fit, int32_t* src_of_rank, int* status, cudaStream_t st) {
    GAPA_LAUNCH(k_ga_elite_rank, (2 * s + kPerBlock - 1) / kPerBlock, kGaThreads, 0, st, fit, fit_m, s, minimize,
                src_of_rank, status);
    GAPA_LAUNCH(k_ga_elite_gather, row_grid(std::max(k, 1), s), kGaThreads, 0, st, pop, m_pop, fit, fit_m, s, k, src_of_rank,
                next, next_fit);
    return GAPA_CUDA_OK;
}

// ---- elitism for a row-sharded generation --------------------------------------------------------------
// Under sharding every rank keeps the whole population but builds only ITS block of M_POP (the rows
// it evaluates).  A surviving mutated row that another rank built is not fetched over NVLink: it is
// RECOMPUTED here from the replicated parent population and the keyed streams — crossover + mutate
// (or eda_sample + mutate on EDA generations) are pure functions of (pop, partner, seed,
// generation, global row), so the recomputed row is bit-identical to the one the owner evaluated.
// Genomes therefore never cross the interconnect; the only exchange stays the fitness all-gather.
__global__ void __launch_bounds__(kGaThreads) k_ga_elite_gather_sharded(
    const int32_t* __restrict__ pop, const int32_t* __restrict__ m_block, int block_lo, int block_hi,
    const int32_t* __restrict__ partner, const double* __restrict__ fit, const double* __restrict__ fit_m, int s, int k,
    uint64_t pc_thr, uint64_t pm_thr, uint32_t pool_size, uint64_t seed, uint64_t generation,
    const int32_t* __restrict__ src_of_rank, int32_t* __restrict__ next, double* __restrict__ next_fit) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[4];
    const int r = blockIdx.y;
    const int src = src_of_rank[r];
    int32_t* to = next + static_cast<size_t>(r) * k;
    if (blockIdx.x == 0 && threadIdx.x == 0) next_fit[r] = src < s ? fit[src] : fit_m[src - s];
    const int row = src - s;  // row of M_POP when src >= s
    if (src < s || (row >= block_lo && row < block_hi)) {
        const int32_t* from = src < s ? pop + static_cast<size_t>(src) * k : m_block + static_cast<size_t>(row - block_lo) * k;
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) to[j] = from[j];
        return;
    }
    // foreign mutated row: rebuild it
    if (threadIdx.x < 4)
        keys[threadIdx.x] = stream_key(seed, generation, GAPA_ROLE_SELECT + threadIdx.x, static_cast<uint64_t>(row));
    __syncthreads();
    const uint64_t ks = keys[0], kc = keys[1], km = keys[2], ki = keys[3];
    const int32_t* mine = pop + static_cast<size_t>(row) * k;
    if (partner) {  // crossover + mutate, ga_ops.cpp:130-178
        const int32_t* theirs = pop + static_cast<size_t>(partner[row]) * k;
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
            const uint64_t d = static_cast<uint64_t>(j) + 1;
            int32_t g;
            if (draw_bernoulli(km, d, pm_thr)) g = static_cast<int32_t>(draw_index(ki, d, pool_size));
            else g = draw_bernoulli(kc, d, pc_thr) ? theirs[j] : mine[j];
            to[j] = g;
        }
    } else {  // eda_sample(elite = whole population, smoothing) + mutate, modes.cpp:167-168, ga_ops.cpp:214-238
        const uint32_t elite = static_cast<uint32_t>(s), bound = elite + pool_size;
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
            const uint64_t d = static_cast<uint64_t>(j) + 1;
            int32_t g;
            if (draw_bernoulli(km, d, pm_thr)) g = static_cast<int32_t>(draw_index(ki, d, pool_size));
            else {
                const uint32_t v = draw_index(ks, d, bound);
                g = v < elite ? pop[static_cast<size_t>(v) * k + j] : static_cast<int32_t>(v - elite);
            }
            to[j] = g;
        }
    }
}

int launch_elitism_sharded(const int32_t* pop, const int32_t* m_block, int block_lo, int block_hi, const int32_t* partner,
                           int s, int k, const double* fit, const double* fit_m, int minimize, double pc, double pm,
                           uint32_t pool_size, uint64_t seed, uint64_t generation, int32_t* next, double* next_fit,
                           int32_t* src_of_rank, int* status, cudaStream_t st) {
    GAPA_LAUNCH(k_ga_elite_rank, (2 * s + kPerBlock - 1) / kPerBlock, kGaThreads, 0, st, fit, fit_m, s, minimize,
                src_of_rank, status);
    GAPA_LAUNCH(k_ga_elite_gather_sharded, row_grid(std::max(k, 1), s), kGaThreads, 0, st, pop, m_block, block_lo, block_hi,
                partner, fit, fit_m, s, k, bernoulli_threshold(pc), bernoulli_threshold(pm), pool_size, seed, generation,
                src_of_rank, next, next_fit);
    return GAPA_CUDA_OK;
}

// Scratch for the *_device entry points: persistent per (host thread, device, stream), so a
// generation loop driven from the host pays no cudaMalloc / cudaFree per operator.  Work on one
// stream is ordered, which makes reuse of the buffers across consecutive calls safe.
struct OpScratch {
    DevBuf a, b, c;
    int* status = nullptr;
    int* h_status = nullptr;  // pinned
    OpScratch() = default;
    OpScratch(const OpScratch&) = delete;
    OpScratch& operator=(const OpScratch&) = delete;
    ~OpScratch() {  // the owning thread ends, or the pool is trimmed (cudaFree waits for work that still uses the buffers)
        a.release();
        b.release();
        c.release();
        if (h_status) cudaFreeHost(h_status);
    }
    int init(cudaStream_t st) {
        GAPA_TRY(c.ensure(sizeof(int)));
        status = c.as<int>();
        if (!h_status) GAPA_CUDA_TRY(cudaMallocHost(&h_status, sizeof(int)));
        GAPA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), st));
        return GAPA_CUDA_OK;
    }
    int check(cudaStream_t st, const char* what) {
        GAPA_CUDA_TRY(cudaMemcpyAsync(h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st));
        GAPA_CUDA_TRY(cudaStreamSynchronize(st));
        if (*h_status == GAPA_CUDA_E_NAN) return fail(GAPA_CUDA_E_NAN, "%s", what);
        return GAPA_CUDA_OK;
    }
};

static OpScratch& op_scratch(cudaStream_t st) {
    struct Key {
        int device;
        cudaStream_t stream;
        bool operator<(const Key& o) const { return device != o.device ? device < o.device : stream < o.stream; }
    };
    static thread_local std::map<Key, OpScratch> pool;
    int device = 0;
    cudaGetDevice(&device);
    const Key key{device, st};
    // streams come and go in a long-lived host thread: entries of streams that no longer exist are dropped wholesale once
    // the pool has grown past what any live set of streams needs (they are re-created on demand)
    if (pool.size() >= 64 && pool.find(key) == pool.end()) pool.clear();
    return pool[key];
}

}  // namespace gapa_b200

using namespace gapa_b200;

// ---- host-buffer forms -------------------------------------------------------------------------------
namespace {
struct Tmp {
    std::vector<void*> ptrs;
    template <typename T>
    int up(const T* host, size_t count, T** dev) {
        GAPA_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dev), std::max<size_t>(sizeof(T) * count, 16)));
        ptrs.push_back(*dev);
        if (host && count) GAPA_CUDA_TRY(cudaMemcpy(*dev, host, sizeof(T) * count, cudaMemcpyHostToDevice));
        return GAPA_CUDA_OK;
    }
    template <typename T>
    int down(T* host, const T* dev, size_t count) {
        if (count) GAPA_CUDA_TRY(cudaMemcpy(host, dev, sizeof(T) * count, cudaMemcpyDeviceToHost));
        return GAPA_CUDA_OK;
    }
    ~Tmp() { for (void* p : ptrs) cudaFree(p); }
};
}  // namespace

namespace gapa_b200 {
int launch_slots_elitism(int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int, int, const double*, const double*,
                         int, double, double, uint32_t, uint64_t, uint64_t, int32_t*, int32_t*, double*, int32_t*, int*, cudaStream_t);
}

static int check_rates(double pc, double pm) {
    if (!(pc >= 0.0 && pc <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pc must be in [0, 1]");
    if (!(pm >= 0.0 && pm <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pm must be in [0, 1]");
    return GAPA_CUDA_OK;
}

extern "C" {

int gapa_cuda_ga_init_device(int32_t pool_size, int row_first, int row_count, int budget, uint64_t seed,
                             uint64_t generation, int32_t* out_dev, void* stream) {
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "init_population: empty gene pool");
    if (row_first < 0 || row_count < 0 || budget < 0) return fail(GAPA_CUDA_E_INVALID, "init_population: negative shape");
    return launch_init(static_cast<uint32_t>(pool_size), row_first, row_count, budget, seed, generation, out_dev,
                       static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_mask_device(int role, double rate, int row_first, int row_count, int cols, uint64_t seed, uint64_t generation,
                             uint8_t* out_dev, void* stream) {
    if (role != GAPA_ROLE_CROSSOVER_MASK && role != GAPA_ROLE_MUTATION_MASK) return fail(GAPA_CUDA_E_INVALID, "mask: role must be a mask stream");
    if (!(rate >= 0.0 && rate <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "mask: rate must be in [0, 1]");
    if (row_first < 0 || row_count < 0 || cols < 0) return fail(GAPA_CUDA_E_INVALID, "mask: negative shape");
    if (row_count == 0 || cols == 0) return GAPA_CUDA_OK;
    const BernoulliLimit lim = bernoulli_limit(rate);
    GAPA_LAUNCH(k_ga_mask, row_grid(cols, row_count), kGaThreads, 0, static_cast<cudaStream_t>(stream), static_cast<uint64_t>(role),
                row_first, cols, lim.limit, lim.always, seed, generation, out_dev);
    return GAPA_CUDA_OK;
}

int gapa_cuda_ga_mutation_indices_device(int32_t pool_size, int row_first, int row_count, int cols, uint64_t seed,
                                         uint64_t generation, int32_t* out_dev, void* stream) {
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    if (row_first < 0 || row_count < 0 || cols < 0) return fail(GAPA_CUDA_E_INVALID, "mutation_indices: negative shape");
    if (row_count == 0 || cols == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_mutation_indices, row_grid(cols, row_count), kGaThreads, 0, static_cast<cudaStream_t>(stream),
                static_cast<uint32_t>(pool_size), row_first, cols, seed, generation, out_dev);
    return GAPA_CUDA_OK;
}

int gapa_cuda_ga_select_device(const double* fitness_dev, int s, int minimize, uint64_t seed, uint64_t generation,
                               int32_t* partner_dev, double* weights_dev, void* stream) {
    if (s < 1) return fail(GAPA_CUDA_E_INVALID, "roulette_select: empty population");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OpScratch& sc = op_scratch(st);
    GAPA_TRY(sc.init(st));
    GAPA_TRY(sc.a.ensure(sizeof(double) * s));
    GAPA_TRY(sc.b.ensure(sizeof(double) * s));
    double* w = weights_dev ? weights_dev : sc.a.as<double>();
    GAPA_TRY(launch_select(fitness_dev, s, minimize, seed, generation, partner_dev, w, sc.b.as<double>(), sc.status, st));
    return sc.check(st, "roulette_select: non-finite fitness");
}

int gapa_cuda_ga_crossover_mutate_device(const int32_t* pop_dev, const int32_t* partner_dev, int s, int k, int row_first,
                                         int row_count, double pc, double pm, int32_t pool_size, uint64_t seed,
                                         uint64_t generation, int32_t* out_dev, void* stream) {
    GAPA_TRY(check_rates(pc, pm));
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    if (row_first < 0 || row_count < 0 || row_first + row_count > s) return fail(GAPA_CUDA_E_INVALID, "crossover: row block outside the population");
    return launch_crossover_mutate(pop_dev, partner_dev, k, row_first, row_count, pc, pm, static_cast<uint32_t>(pool_size),
                                   seed, generation, out_dev, static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_mutate_device(const int32_t* block_dev, int rows, int k, int row_offset, double pm, int32_t pool_size,
                               uint64_t seed, uint64_t generation, int32_t* out_dev, void* stream) {
    GAPA_TRY(check_rates(0.0, pm));
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    return launch_mutate(block_dev, rows, k, row_offset, pm, static_cast<uint32_t>(pool_size), seed, generation, out_dev,
                         static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_eda_device(const int32_t* elite_dev, int s, int k, int elite_count, int32_t pool_size, uint64_t seed,
                            uint64_t generation, int smoothing, int32_t* out_dev, void* stream) {
    if (elite_count < 1 || elite_count > s) return fail(GAPA_CUDA_E_INVALID, "eda_sample: invalid elite count");
    const uint32_t bound = static_cast<uint32_t>(smoothing ? elite_count + pool_size : elite_count);
    return launch_eda(elite_dev, 0, s, k, elite_count, bound, seed, generation, out_dev, static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_elitism_device(const int32_t* pop_dev, const int32_t* m_pop_dev, int s, int k, const double* fit_dev,
                                const double* fit_m_dev, int minimize, int32_t* next_dev, double* next_fit_dev,
                                void* stream) {
    if (s < 1) return fail(GAPA_CUDA_E_INVALID, "elitism: empty population");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OpScratch& sc = op_scratch(st);
    GAPA_TRY(sc.init(st));
    GAPA_TRY(sc.a.ensure(sizeof(int32_t) * s));
    GAPA_TRY(launch_elitism(pop_dev, m_pop_dev, s, k, fit_dev, fit_m_dev, minimize, next_dev, next_fit_dev,
                            sc.a.as<int32_t>(), sc.status, st));
    return sc.check(st, "elitism: NaN fitness");
}


int gapa_cuda_ga_elitism_sharded_device(const int32_t* pop_dev, const int32_t* m_block_dev, int block_lo, int block_hi,
                                        const int32_t* partner_dev, int s, int k, const double* fit_dev,
                                        const double* fit_m_dev, int minimize, double pc, double pm, int32_t pool_size,
                                        uint64_t seed, uint64_t generation, int32_t* next_dev, double* next_fit_dev,
                                        void* stream) {
    if (s < 1) return fail(GAPA_CUDA_E_INVALID, "elitism: empty population");
    if (block_lo < 0 || block_hi < block_lo || block_hi > s) return fail(GAPA_CUDA_E_INVALID, "elitism: row block outside the population");
    GAPA_TRY(check_rates(pc, pm));
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OpScratch& sc = op_scratch(st);
    GAPA_TRY(sc.init(st));
    GAPA_TRY(sc.a.ensure(sizeof(int32_t) * s));
    GAPA_TRY(launch_elitism_sharded(pop_dev, m_block_dev, block_lo, block_hi, partner_dev, s, k, fit_dev, fit_m_dev, minimize,
                                    pc, pm, static_cast<uint32_t>(pool_size), seed, generation, next_dev, next_fit_dev,
                                    sc.a.as<int32_t>(), sc.status, st));
    return sc.check(st, "elitism: NaN fitness");
}

int gapa_cuda_ga_slots_elitism_device(int32_t* pool_dev, const int32_t* parent_dev, const int32_t* child_dev,
                                      const int32_t* partner_dev, int s, int k, int block_lo, int block_hi,
                                      const double* fit_dev, const double* fit_m_dev, int minimize, double pc, double pm,
                                      int32_t pool_size, uint64_t seed, uint64_t generation, int32_t* next_parent_dev,
                                      int32_t* next_child_dev, double* next_fit_dev, void* stream) {
    if (s < 1) return fail(GAPA_CUDA_E_INVALID, "elitism: empty population");
    if (block_lo < 0 || block_hi < block_lo || block_hi > s) return fail(GAPA_CUDA_E_INVALID, "elitism: row block outside the population");
    GAPA_TRY(check_rates(pc, pm));
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OpScratch& sc = op_scratch(st);
    GAPA_TRY(sc.init(st));
    GAPA_TRY(sc.a.ensure(sizeof(int32_t) * 2 * s));
    GAPA_TRY(launch_slots_elitism(pool_dev, parent_dev, child_dev, partner_dev, s, k, block_lo, block_hi, fit_dev, fit_m_dev,
                                  minimize, pc, pm, static_cast<uint32_t>(pool_size), seed, generation, next_parent_dev,
                                  next_child_dev, next_fit_dev, sc.a.as<int32_t>(), sc.status, st));
    return sc.check(st, "elitism: NaN fitness");
}

int gapa_cuda_ga_init(int device, int32_t pool_size, int row_first, int row_count, int budget, uint64_t seed,
                      uint64_t generation, int32_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    Tmp t;
    int32_t* d = nullptr;
    const size_t cells = static_cast<size_t>(std::max(row_count, 0)) * std::max(budget, 0);
    GAPA_TRY(t.up<int32_t>(nullptr, cells, &d));
    GAPA_TRY(gapa_cuda_ga_init_device(pool_size, row_first, row_count, budget, seed, generation, d, nullptr));
    return t.down(out, d, cells);
}

int gapa_cuda_ga_mask(int device, int role, double rate, int rows, int cols, uint64_t seed, uint64_t generation, uint8_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    Tmp t;
    uint8_t* d = nullptr;
    const size_t cells = static_cast<size_t>(std::max(rows, 0)) * std::max(cols, 0);
    GAPA_TRY(t.up<uint8_t>(nullptr, cells, &d));
    GAPA_TRY(gapa_cuda_ga_mask_device(role, rate, 0, rows, cols, seed, generation, d, nullptr));
    return t.down(out, d, cells);
}

int gapa_cuda_ga_mutation_indices(int device, int32_t pool_size, int rows, int cols, uint64_t seed, uint64_t generation, int32_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    Tmp t;
    int32_t* d = nullptr;
    const size_t cells = static_cast<size_t>(std::max(rows, 0)) * std::max(cols, 0);
    GAPA_TRY(t.up<int32_t>(nullptr, cells, &d));
    GAPA_TRY(gapa_cuda_ga_mutation_indices_device(pool_size, 0, rows, cols, seed, generation, d, nullptr));
    return t.down(out, d, cells);
}

int gapa_cuda_ga_selection_weights(int device, const double* fitness, int s, int minimize, double* weights) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (s < 1) return GAPA_CUDA_OK;
    Tmp t;
    double *f = nullptr, *w = nullptr;
    int32_t* p = nullptr;
    GAPA_TRY(t.up(fitness, s, &f));
    GAPA_TRY(t.up<double>(nullptr, s, &w));
    GAPA_TRY(t.up<int32_t>(nullptr, s, &p));
    int rc = gapa_cuda_ga_select_device(f, s, minimize, 0, 0, p, w, nullptr);
    if (rc == GAPA_CUDA_E_NAN) return fail(GAPA_CUDA_E_NAN, "selection: non-finite fitness");
    GAPA_TRY(rc);
    return t.down(weights, w, s);
}

int gapa_cuda_ga_select(int device, const double* fitness, int s, int minimize, uint64_t seed, uint64_t generation,
                        int32_t* partner_index) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    Tmp t;
    double* f = nullptr;
    int32_t* p = nullptr;
    GAPA_TRY(t.up(fitness, std::max(s, 0), &f));
    GAPA_TRY(t.up<int32_t>(nullptr, std::max(s, 0), &p));
    GAPA_TRY(gapa_cuda_ga_select_device(f, s, minimize, seed, generation, p, nullptr, nullptr));
    return t.down(partner_index, p, s);
}

int gapa_cuda_ga_crossover_mutate(int device, const int32_t* pop, const int32_t* partner_index, int s, int k, int row_first,
                                  int row_count, double pc, double pm, int32_t pool_size, uint64_t seed,
                                  uint64_t generation, int32_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (s < 0 || k < 0) return fail(GAPA_CUDA_E_INVALID, "crossover: shape mismatch");
    for (int i = 0; i < s; ++i)
        if (partner_index[i] < 0 || partner_index[i] >= s) return fail(GAPA_CUDA_E_INVALID, "crossover: partner index out of range");
    Tmp t;
    int32_t *dp = nullptr, *di = nullptr, *d_out = nullptr;
    GAPA_TRY(t.up(pop, static_cast<size_t>(s) * k, &dp));
    GAPA_TRY(t.up(partner_index, s, &di));
    GAPA_TRY(t.up<int32_t>(nullptr, static_cast<size_t>(std::max(row_count, 0)) * k, &d_out));
    GAPA_TRY(gapa_cuda_ga_crossover_mutate_device(dp, di, s, k, row_first, row_count, pc, pm, pool_size, seed, generation, d_out, nullptr));
    return t.down(out, d_out, static_cast<size_t>(row_count) * k);
}

int gapa_cuda_ga_mutate(int device, const int32_t* block, int rows, int k, int row_offset, double pm, int32_t pool_size,
                        uint64_t seed, uint64_t generation, int32_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (rows < 0 || k < 0) return fail(GAPA_CUDA_E_INVALID, "mutate: shape mismatch");
    Tmp t;
    int32_t *db = nullptr, *d_out = nullptr;
    GAPA_TRY(t.up(block, static_cast<size_t>(rows) * k, &db));
    GAPA_TRY(t.up<int32_t>(nullptr, static_cast<size_t>(rows) * k, &d_out));
    GAPA_TRY(gapa_cuda_ga_mutate_device(db, rows, k, row_offset, pm, pool_size, seed, generation, d_out, nullptr));
    return t.down(out, d_out, static_cast<size_t>(rows) * k);
}

int gapa_cuda_ga_eda(int device, const int32_t* elite, int s, int k, int elite_count, int32_t pool_size, uint64_t seed,
                     uint64_t generation, int smoothing, int32_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (s < 0 || k < 0) return fail(GAPA_CUDA_E_INVALID, "eda_sample: shape mismatch");
    Tmp t;
    int32_t *de = nullptr, *d_out = nullptr;
    GAPA_TRY(t.up(elite, static_cast<size_t>(s) * k, &de));
    GAPA_TRY(t.up<int32_t>(nullptr, static_cast<size_t>(s) * k, &d_out));
    GAPA_TRY(gapa_cuda_ga_eda_device(de, s, k, elite_count, pool_size, seed, generation, smoothing, d_out, nullptr));
    return t.down(out, d_out, static_cast<size_t>(s) * k);
}

int gapa_cuda_ga_elitism(int device, const int32_t* pop, const int32_t* m_pop, int s, int k, const double* fit,
                         const double* fit_m, int minimize, int32_t* next, double* next_fit) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (s < 1 || k < 0) return fail(GAPA_CUDA_E_INVALID, "elitism: shape mismatch");
    Tmp t;
    int32_t *dp = nullptr, *dm = nullptr, *dn = nullptr;
    double *df = nullptr, *dfm = nullptr, *dnf = nullptr;
    const size_t cells = static_cast<size_t>(s) * k;
    GAPA_TRY(t.up(pop, cells, &dp));
    GAPA_TRY(t.up(m_pop, cells, &dm));
    GAPA_TRY(t.up<int32_t>(nullptr, cells, &dn));
    GAPA_TRY(t.up(fit, s, &df));
    GAPA_TRY(t.up(fit_m, s, &dfm));
    GAPA_TRY(t.up<double>(nullptr, s, &dnf));
    GAPA_TRY(gapa_cuda_ga_elitism_device(dp, dm, s, k, df, dfm, minimize, dn, dnf, nullptr));
    GAPA_TRY(t.down(next, dn, cells));
    return t.down(next_fit, dnf, s);
}

int gapa_cuda_rng_draws(int device, uint64_t seed, uint64_t generation, uint64_t role, uint64_t row, int count,
                        uint64_t* out) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (count <= 0) return GAPA_CUDA_OK;
    Tmp t;
    uint64_t* d = nullptr;
    GAPA_TRY(t.up<uint64_t>(nullptr, count, &d));
    GAPA_LAUNCH(k_rng_draws, (count + 255) / 256, 256, 0, nullptr, seed, generation, role, row, count, d);
    return t.down(out, d, count);
}

}  // extern "C"
