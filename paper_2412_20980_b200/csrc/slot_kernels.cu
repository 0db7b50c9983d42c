// The population store of the generation loop: ONE pool of 2s row slots in HBM plus two index
// tables — parent[r] = slot of parent row r (best first), child[r] = slot of child row r (the s
// slots that are free this generation).  Variation writes children straight into their slots and
// the evaluators read them through the table (GeneRows), so elitism (ga_ops.cpp:180-212) is a
// permutation of indices: no genome is ever copied, whatever survives stays where it was built.
//
// Under row sharding (modes.cpp:190-349 on GPUs) a rank builds only the children of its own row
// block; a surviving child that another rank built is recomputed into its slot from the replicated
// parents and the keyed streams (k_ga_slots_rebuild) — never fetched over the interconnect.
//
// Every gene equals the reference's: parents/children are the matrices POP / M_POP of
// modes.cpp:159-175 seen through the tables (gapa_cuda_ga_slots_gather materialises them).
#include <algorithm>
#include <cstdlib>
#include <map>

#include "internal.cuh"
#include "variation.cuh"

namespace gapa_b200 {

static constexpr int kSlotThreads = 256;
// Builds child row `row` into its slot.  Shared by the variation kernel (own rows) and the rebuild
// kernel (foreign survivors).
__device__ __forceinline__ void build_child_row(const VariationSpec& V, int k, int row, uint64_t* keys) {
    const VariationParams& P = V.P;
    if (threadIdx.x < 4)
        keys[threadIdx.x] = stream_key(P.seed, P.generation, GAPA_ROLE_SELECT + threadIdx.x, static_cast<uint64_t>(row)) + kGolden;
    __syncthreads();
    const uint64_t ks = keys[0], kc = keys[1], km = keys[2], ki = keys[3];
    const bool eda = V.partner == nullptr;
    const int slot_mine = V.parent[row], slot_theirs = eda ? slot_mine : V.parent[V.partner[row]];
    bool adopt_mine, adopt_theirs;  // rows that live in another rank's HBM are written through to the local slot
    const int32_t* mine = parent_row(V, slot_mine, k, &adopt_mine);
    const int32_t* theirs = eda ? mine : parent_row(V, slot_theirs, k, &adopt_theirs);
    if (eda || slot_theirs == slot_mine) adopt_theirs = false;
    int32_t* keep_mine = V.pool + static_cast<size_t>(slot_mine) * k;
    int32_t* keep_theirs = V.pool + static_cast<size_t>(slot_theirs) * k;
    int32_t* dst = V.pool + static_cast<size_t>(V.child[row]) * k;
    if ((k & 3) == 0) {  // slots are 16-byte aligned when k is a multiple of 4
        const int4* mine4 = reinterpret_cast<const int4*>(mine);
        const int4* theirs4 = reinterpret_cast<const int4*>(theirs);
        int4* dst4 = reinterpret_cast<int4*>(dst);
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < (k >> 2); q += gridDim.x * blockDim.x) {
            const int4 a = mine4[q];
            const int4 b = eda ? a : theirs4[q];
            if (adopt_mine) reinterpret_cast<int4*>(keep_mine)[q] = a;
            if (adopt_theirs) reinterpret_cast<int4*>(keep_theirs)[q] = b;
            const int av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
            int r[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) r[t] = child_gene(P, V.pool, V.parent, k, 4 * q + t, av[t], bv[t], eda, ks, kc, km, ki, 4u * q + t + 1u);
            dst4[q] = make_int4(r[0], r[1], r[2], r[3]);
        }
    } else {
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
            const int a = mine[j], b = theirs[j];
            if (adopt_mine) keep_mine[j] = a;
            if (adopt_theirs) keep_theirs[j] = b;
            dst[j] = child_gene(P, V.pool, V.parent, k, j, a, b, eda, ks, kc, km, ki, static_cast<uint32_t>(j) + 1u);
        }
    }
}

// children of rows [V.row_first, V.row_first + gridDim.y)
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_variation(VariationSpec V, int k) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[4];
    build_child_row(V, k, V.row_first + blockIdx.y, keys);
}

// ---- row-sharded runs over peer memory (run.cu) ------------------------------------------------------------------
// home[child[j]] = the rank that builds child row j this generation (partition_rows, modes.cpp:506-516)
__global__ void __launch_bounds__(kSlotThreads) k_ga_home_children(const int32_t* __restrict__ child, int s, int block, int32_t* home) {
    griddep_launch();
    griddep_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < s) home[child[j]] = j / block;
}
// after a variation launch: the parent rows it read remotely now have a local copy
__global__ void __launch_bounds__(kSlotThreads) k_ga_home_adopt(const int32_t* __restrict__ parent, const int32_t* __restrict__ partner,
                                                                int lo, int hi, int self, int32_t* home) {
    griddep_launch();
    griddep_wait();
    const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    home[parent[i]] = self;
    if (partner) home[parent[partner[i]]] = self;
}
// every parent row that is not local yet is copied from its builder's pool (EDA generations sample ALL parents; the
// final population is returned whole)
__global__ void __launch_bounds__(kSlotThreads) k_ga_fetch_rows(int32_t* __restrict__ pool, const int32_t* const* __restrict__ bases,
                                                                const int32_t* __restrict__ home, const int32_t* __restrict__ parent,
                                                                int k, int self) {
    griddep_launch();
    griddep_wait();
    const int slot = parent[blockIdx.y];
    const int h = home[slot];
    if (h == self) return;
    const int32_t* from = bases[h] + static_cast<size_t>(slot) * k;
    int32_t* to = pool + static_cast<size_t>(slot) * k;
    if ((k & 3) == 0) {
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < (k >> 2); q += gridDim.x * blockDim.x)
            reinterpret_cast<int4*>(to)[q] = reinterpret_cast<const int4*>(from)[q];
    } else {
        for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) to[j] = from[j];
    }
}
__global__ void __launch_bounds__(kSlotThreads) k_ga_home_all_local(const int32_t* __restrict__ parent, int s, int self, int32_t* home) {
    griddep_launch();
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s) home[parent[i]] = self;
}

// Stable best-first position of every stacked row (parents 0..s-1, children s..2s-1):
// order[rank] = stacked index; originals precede children on ties (ga_ops.cpp:194-201).
static constexpr int kSplit = 8;
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_rank(const double* __restrict__ fit, const double* __restrict__ fit_m,
                                                                int s, int minimize, int32_t* __restrict__ order, int* status) {
    griddep_launch();
    griddep_wait();
    __shared__ unsigned long long tile[kSlotThreads];
    const int x = blockIdx.x * (kSlotThreads / kSplit) + threadIdx.x / kSplit, part = threadIdx.x % kSplit;
    const int total = 2 * s;
    const double mine_f = x < total ? (x < s ? fit[x] : fit_m[x - s]) : 0.0;
    if (x < total && isnan(mine_f)) *status = GAPA_CUDA_E_NAN;
    const unsigned long long mine = order_key(mine_f, minimize);  // integer compares (internal.cuh)
    int rank = 0;
    // From the second generation on the parents ARE sorted best-first (they are the previous elitism's output).  Every
    // block checks that while it is cheap (s compares against its own 32 * 2s); if so a parent's position among the
    // parents is its index, a child's is one binary search, and only the children have to be counted: half the compares.
    int in_order = 1;
    for (int t = threadIdx.x; t + 1 < s; t += kSlotThreads) in_order &= order_key(fit[t], minimize) <= order_key(fit[t + 1], minimize);
    if (__syncthreads_and(in_order)) {
        const int j = x - s;  // own index among the children (negative for a parent)
        if (x >= s && x < total) {  // parents that precede this child: ties included (originals first)
            int a = 0, b = s;
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (order_key(fit[mid], minimize) <= mine) a = mid + 1; else b = mid;
            }
            rank = part == 0 ? a : 0;
        } else {
            rank = part == 0 ? x : 0;
        }
        for (int c0 = 0; c0 < s; c0 += kSlotThreads) {
            __syncthreads();
            if (c0 + threadIdx.x < s) tile[threadIdx.x] = order_key(fit_m[c0 + threadIdx.x], minimize);
            __syncthreads();
            const int lim = min(kSlotThreads, s - c0);
            if (j < 0 || c0 > j) {  // a parent precedes every tied child; children after mine do not count on ties
                for (int t = part; t < lim; t += kSplit) rank += tile[t] < mine;
            } else if (c0 + kSlotThreads <= j) {
                for (int t = part; t < lim; t += kSplit) rank += tile[t] <= mine;
            } else {
                for (int t = part; t < lim; t += kSplit) {
                    const unsigned long long other = tile[t];
                    rank += (other < mine) | ((other == mine) & (c0 + t < j));
                }
            }
        }
        for (int off = kSplit / 2; off; off >>= 1) rank += __shfl_down_sync(0xffffffffu, rank, off, kSplit);
        if (x < total && part == 0) order[rank] = x;
        return;
    }
    const int own_t0 = blockIdx.x * (kSlotThreads / kSplit) / kSlotThreads * kSlotThreads;
    for (int t0 = 0; t0 < total; t0 += kSlotThreads) {
        __syncthreads();
        const int y = t0 + threadIdx.x;
        if (y < total) tile[threadIdx.x] = order_key(y < s ? fit[y] : fit_m[y - s], minimize);
        __syncthreads();
        const int lim = min(kSlotThreads, total - t0);
        // a block's rows all lie in one tile: tiles before it hold only lower indices (ties count),
        // tiles after it only higher ones (ties do not); one 64-bit compare per pair in both cases
        if (t0 + kSlotThreads <= own_t0) {
            for (int t = part; t < lim; t += kSplit) rank += tile[t] <= mine;
        } else if (t0 > own_t0) {
            for (int t = part; t < lim; t += kSplit) rank += tile[t] < mine;
        } else {
            for (int t = part; t < lim; t += kSplit) {
                const unsigned long long other = tile[t];
                rank += (other < mine) | ((other == mine) & (t0 + t < x));
            }
        }
    }
    for (int off = kSplit / 2; off; off >>= 1) rank += __shfl_down_sync(0xffffffffu, rank, off, kSplit);
    if (x < total && part == 0) order[rank] = x;
}

// Ranking of LARGE populations (round 2).  k_ga_slots_rank counts, for every stacked row, the rows before it: O(s^2) compares
// — 0.164 ms of a 0.40 ms generation at n = 1e4 with 16,384 individuals.  Here the parents and the children are first sorted in
// tiles of 1024 by (order key, index) — one block per tile, bitonic network in shared memory — and a row's position is then a
// sum of binary searches, one per tile: O(s (s / 1024) log 1024).  Nothing is assumed about the parents' order.  "Before" is the
// reference's stable order on the stacked rows (ga_ops.cpp:194-201): smaller key, then smaller stacked index — for a parent
// against a child tile that is "key strictly smaller", for a child against a parent tile "key smaller or equal".
static constexpr int kSortTile = 1024;
__global__ void __launch_bounds__(kSortTile) k_ga_sort_tiles(const double* __restrict__ fit, const double* __restrict__ fit_m, int s,
                                                             int minimize, unsigned long long* __restrict__ skey,
                                                             int32_t* __restrict__ sidx, int* status) {
    griddep_launch();
    griddep_wait();
    __shared__ unsigned long long key[kSortTile];
    __shared__ int32_t idx[kSortTile];
    const int tid = threadIdx.x;
    const int ptiles = (s + kSortTile - 1) / kSortTile;
    const bool child_tile = static_cast<int>(blockIdx.x) >= ptiles;
    const int i = (child_tile ? blockIdx.x - ptiles : blockIdx.x) * kSortTile + tid;
    unsigned long long k = ~0ull;  // padding sorts last
    int32_t id = 0x7fffffff;
    if (i < s) {
        const double f = child_tile ? fit_m[i] : fit[i];
        if (isnan(f)) *status = GAPA_CUDA_E_NAN;
        k = order_key(f, minimize);
        id = i;
    }
    key[tid] = k;
    idx[tid] = id;
    __syncthreads();
    for (int size = 2; size <= kSortTile; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int other = tid ^ stride;
            if (other > tid) {
                const unsigned long long ka = key[tid], kb = key[other];
                const int32_t ia = idx[tid], ib = idx[other];
                const bool a_after_b = ka > kb || (ka == kb && ia > ib);
                const bool ascending = (tid & size) == 0;
                if (a_after_b == ascending) {
                    key[tid] = kb; key[other] = ka;
                    idx[tid] = ib; idx[other] = ia;
                }
            }
            __syncthreads();
        }
    }
    skey[static_cast<size_t>(blockIdx.x) * kSortTile + tid] = key[tid];
    sidx[static_cast<size_t>(blockIdx.x) * kSortTile + tid] = idx[tid];
}
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_rank_tiles(const double* __restrict__ fit, const double* __restrict__ fit_m,
                                                                      int s, int minimize, const unsigned long long* __restrict__ skey,
                                                                      const int32_t* __restrict__ sidx, int32_t* __restrict__ order) {
    griddep_launch();
    griddep_wait();
    const int x = blockIdx.x * (kSlotThreads / kSplit) + threadIdx.x / kSplit, part = threadIdx.x % kSplit;
    const int total = 2 * s, ptiles = (s + kSortTile - 1) / kSortTile;
    const bool live = x < total, is_child = x >= s;
    const int own = is_child ? x - s : x;  // index within the own half
    const unsigned long long mine = live ? order_key(is_child ? fit_m[own] : fit[own], minimize) : 0ull;
    int rank = 0;
    if (live) {
        for (int tile = part; tile < 2 * ptiles; tile += kSplit) {
            const bool child_tile = tile >= ptiles;
            const int len = min(kSortTile, s - (child_tile ? tile - ptiles : tile) * kSortTile);
            const unsigned long long* tk = skey + static_cast<size_t>(tile) * kSortTile;
            const int32_t* ti = sidx + static_cast<size_t>(tile) * kSortTile;
            int a = 0, b = len;
            if (child_tile == is_child) {  // own half: (key, index) strictly before (mine, own)
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    const unsigned long long k = tk[mid];
                    if (k < mine || (k == mine && ti[mid] < own)) a = mid + 1; else b = mid;
                }
            } else if (is_child) {  // a child against parents: ties count (originals first)
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (tk[mid] <= mine) a = mid + 1; else b = mid;
                }
            } else {  // a parent against children: ties do not count
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (tk[mid] < mine) a = mid + 1; else b = mid;
                }
            }
            rank += a;
        }
    }
    for (int off = kSplit / 2; off; off >>= 1) rank += __shfl_down_sync(0xffffffffu, rank, off, kSplit);
    if (live && part == 0) order[rank] = x;
}
// smallest population ranked through sorted tiles (GAPA_RANK_TILES_MIN).  Measured at n = 1e4 (a generation, counting -> tiles):
// 4096 individuals 0.149 -> 0.152 ms, 8192: 0.217 -> 0.185, 16,384: 0.390 -> 0.284 (n = 1e5: 1.149 -> 1.038, n = 1e6: 6.50 -> 6.43)
static constexpr int kRankTilesMin = 6144;

// Survivors that this rank did not build (children of rows outside [block_lo, block_hi)).
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_rebuild(VariationParams P, int32_t* __restrict__ pool,
                                                                   const int32_t* __restrict__ parent,
                                                                   const int32_t* __restrict__ child,
                                                                   const int32_t* __restrict__ partner, int k, int s,
                                                                   const int32_t* __restrict__ order, int block_lo, int block_hi) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[4];
    const int x = order[blockIdx.y];  // blockIdx.y = rank < s: a survivor
    const int row = x - s;
    if (x < s || (row >= block_lo && row < block_hi)) return;
    VariationSpec V;
    V.P = P;
    V.pool = pool;
    V.parent = parent;
    V.child = child;
    V.partner = partner;
    V.row_first = 0;
    build_child_row(V, k, row, keys);
}

// next parent table = slots of the s best, next child table = slots of the s others (now free)
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_commit(const int32_t* __restrict__ parent, const int32_t* __restrict__ child,
                                                                  const double* __restrict__ fit, const double* __restrict__ fit_m, int s,
                                                                  const int32_t* __restrict__ order, int32_t* __restrict__ next_parent,
                                                                  int32_t* __restrict__ next_child, double* __restrict__ next_fit) {
    griddep_launch();
    griddep_wait();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= s) return;
    const int keep = order[r], drop = order[s + r];
    next_parent[r] = keep < s ? parent[keep] : child[keep - s];
    next_fit[r] = keep < s ? fit[keep] : fit_m[keep - s];
    next_child[r] = drop < s ? parent[drop] : child[drop - s];
}

// rank + commit + record_generation (modes.cpp:35-43) in ONE block for 2s <= 1024 (small populations are
// launch-latency-bound): next tables, next fitness, history best = front, history mean = the reference's
// left-to-right sum / s (added in parallel only when every value is an integer small enough to add exactly).
__global__ void __launch_bounds__(1024) k_ga_slots_elitism_small(const int32_t* __restrict__ parent, const int32_t* __restrict__ child,
                                                                 const double* __restrict__ fit, const double* __restrict__ fit_m,
                                                                 int s, int minimize, int32_t* __restrict__ order,
                                                                 int32_t* __restrict__ next_parent, int32_t* __restrict__ next_child,
                                                                 double* __restrict__ next_fit, int* status, double* hist_best,
                                                                 double* hist_mean, int select_next, uint64_t seed,
                                                                 uint64_t next_generation, int32_t* __restrict__ partner,
                                                                 double* __restrict__ weights, double* __restrict__ cumulative) {
    __shared__ double f[1024];
    __shared__ double cum[512];
    __shared__ double kept[512];
    __shared__ int ord[1024];
    __shared__ double warp_sum[32];
    __shared__ int not_exact;
    const int tid = threadIdx.x, total = 2 * s;
    griddep_launch();
    griddep_wait();  // the evaluation that wrote fit_m
    const double mine = tid < total ? (tid < s ? fit[tid] : fit_m[tid - s]) : 0.0;
    if (tid < total) {
        f[tid] = mine;
        if (isnan(mine)) *status = GAPA_CUDA_E_NAN;
    }
    if (tid == 0) not_exact = 0;
    __syncthreads();
    if (tid < total) {
        int rank = 0;
        for (int t = 0; t < total; ++t) {
            const double other = f[t];
            const bool before = minimize ? other < mine : other > mine;
            rank += before || (other == mine && t < tid);
        }
        ord[rank] = tid;
        order[rank] = tid;
    }
    __syncthreads();
    double x = 0.0;
    if (tid < s) {
        const int keep = ord[tid], drop = ord[s + tid];
        x = f[keep];
        next_parent[tid] = keep < s ? parent[keep] : child[keep - s];
        next_fit[tid] = x;
        kept[tid] = x;
        next_child[tid] = drop < s ? parent[drop] : child[drop - s];
        if (!(x == floor(x)) || !(fabs(x) < 9007199254740992.0 / static_cast<double>(s))) not_exact = 1;
    }
    __syncthreads();
    if (!not_exact) {
        for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
        if ((tid & 31) == 0) warp_sum[tid >> 5] = x;
        __syncthreads();
        if (tid < 32) {
            double v = warp_sum[tid];
            for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
            if (tid == 0) {
                *hist_best = kept[0];
                *hist_mean = v / static_cast<double>(s);
            }
        }
    } else if (tid == 0) {
        double sum = 0.0;
        for (int i = 0; i < s; ++i) sum += kept[i];
        *hist_best = kept[0];
        *hist_mean = sum / static_cast<double>(s);
    }
    if (!select_next) return;
    // roulette_select of the NEXT generation (ga_ops.cpp:54-82, :105-128) on the parents just committed, saving that
    // generation's selection launch.  `kept` is sorted best-first, so the rows strictly better than mine are a prefix
    // and my ties a contiguous run: two binary searches give the counts selection_weights needs.
    __syncthreads();
    double w = 0.0;
    if (tid < s) {
        const double mine_next = kept[tid];
        if (!isfinite(mine_next)) *status = GAPA_CUDA_E_NAN;
        int a = 0, b = tid;  // first row not strictly better than mine
        while (a < b) {
            const int mid = (a + b) >> 1;
            const double other = kept[mid];
            if (minimize ? other < mine_next : other > mine_next) a = mid + 1; else b = mid;
        }
        const int less = a;
        a = tid + 1, b = s;  // first row strictly worse than mine
        while (a < b) {
            const int mid = (a + b) >> 1;
            const double other = kept[mid];
            if (minimize ? mine_next < other : mine_next > other) b = mid; else a = mid + 1;
        }
        const int leq = a;
        w = (static_cast<double>(s - less) + static_cast<double>(s - leq + 1)) / 2.0;
        weights[tid] = w;
    }
    const int lane = tid & 31, wid = tid >> 5;
    double v = w;  // inclusive scan; half-integers below 2^53 add exactly in any order
    for (int off = 1; off < 32; off <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += t;
    }
    if (lane == 31) warp_sum[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = warp_sum[lane];
        for (int off = 1; off < 32; off <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, t, off);
            if (lane >= off) t += u;
        }
        warp_sum[lane] = t;
    }
    __syncthreads();
    if (wid > 0) v += warp_sum[wid - 1];
    if (tid < s) {
        cum[tid] = v;
        cumulative[tid] = v;
    }
    __syncthreads();
    if (tid < s) {
        const double target = draw_unit(stream_key(seed, next_generation, GAPA_ROLE_SELECT, static_cast<uint64_t>(tid)), 1) * cum[s - 1];
        int a = 0, b = s;  // std::upper_bound: first index with cumulative > target
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (cum[mid] <= target) a = mid + 1; else b = mid;
        }
        partner[tid] = min(a, s - 1);
    }
}

__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_identity(int s, int32_t* parent, int32_t* child) {
    griddep_launch();
    griddep_wait();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < s) {
        parent[r] = r;
        child[r] = s + r;
    }
}

// dense row-major copy of the rows a table names (population.hpp:12-40)
__global__ void __launch_bounds__(kSlotThreads) k_ga_slots_gather(const int32_t* __restrict__ pool, const int32_t* __restrict__ table,
                                                                  int k, int32_t* __restrict__ out) {
    griddep_launch();
    griddep_wait();
    const int32_t* from = pool + static_cast<size_t>(table[blockIdx.y]) * k;
    int32_t* to = out + static_cast<size_t>(blockIdx.y) * k;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) to[j] = from[j];
}

static dim3 slot_grid(int cols, int rows) {
    const int per_block = kSlotThreads * 8;
    return dim3(std::max(1, std::min((cols + per_block - 1) / per_block, 65535)), rows);
}

// ---- launchers shared with run.cu (no synchronisation) ---------------------------------------------------
int launch_slots_identity(int s, int32_t* parent, int32_t* child, cudaStream_t st) {
    GAPA_LAUNCH(k_ga_slots_identity, (s + kSlotThreads - 1) / kSlotThreads, kSlotThreads, 0, st, s, parent, child);
    return GAPA_CUDA_OK;
}
int launch_slots_variation(int32_t* pool, const int32_t* parent, const int32_t* child, const int32_t* partner, int s, int k,
                           int row_first, int row_count, double pc, double pm, uint32_t pool_size, uint64_t seed,
                           uint64_t generation, cudaStream_t st) {
    if (row_count == 0 || k == 0) return GAPA_CUDA_OK;
    VariationSpec V;
    V.P = make_variation_params(pc, pm, pool_size, s, seed, generation);
    V.pool = pool;
    V.parent = parent;
    V.child = child;
    V.partner = partner;
    V.row_first = row_first;
    GAPA_LAUNCH(k_ga_slots_variation, slot_grid((k & 3) ? k : k / 4, row_count), kSlotThreads, 0, st, V, k);
    return GAPA_CUDA_OK;
}
int launch_variation_spec(const VariationSpec& spec, int k, int rows, cudaStream_t st) {
    if (rows == 0 || k == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_slots_variation, slot_grid((k & 3) ? k : k / 4, rows), kSlotThreads, 0, st, spec, k);
    return GAPA_CUDA_OK;
}
// launchers of the peer-memory bookkeeping (run.cu)
int launch_home_children(const int32_t* child, int s, int block, int32_t* home, cudaStream_t st) {
    GAPA_LAUNCH(k_ga_home_children, (s + kSlotThreads - 1) / kSlotThreads, kSlotThreads, 0, st, child, s, block, home);
    return GAPA_CUDA_OK;
}
int launch_home_adopt(const int32_t* parent, const int32_t* partner, int lo, int hi, int self, int32_t* home, cudaStream_t st) {
    if (hi <= lo) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_home_adopt, (hi - lo + kSlotThreads - 1) / kSlotThreads, kSlotThreads, 0, st, parent, partner, lo, hi, self, home);
    return GAPA_CUDA_OK;
}
int launch_fetch_rows(int32_t* pool, const int32_t* const* bases, int32_t* home, const int32_t* parent, int s, int k, int self,
                      cudaStream_t st) {
    if (k > 0) GAPA_LAUNCH(k_ga_fetch_rows, slot_grid((k & 3) ? k : k / 4, s), kSlotThreads, 0, st, pool, bases, home, parent, k, self);
    GAPA_LAUNCH(k_ga_home_all_local, (s + kSlotThreads - 1) / kSlotThreads, kSlotThreads, 0, st, parent, s, self, home);
    return GAPA_CUDA_OK;
}
// sorted-tile scratch of the large-population ranking: per (host thread, device, stream), like the operators' scratch
struct RankScratch {
    DevBuf key, idx;
    RankScratch() = default;
    RankScratch(const RankScratch&) = delete;
    RankScratch& operator=(const RankScratch&) = delete;
    ~RankScratch() {
        key.release();
        idx.release();
    }
};
static RankScratch& rank_scratch(cudaStream_t st) {
    struct Key {
        int device;
        cudaStream_t stream;
        bool operator<(const Key& o) const { return device != o.device ? device < o.device : stream < o.stream; }
    };
    static thread_local std::map<Key, RankScratch> pool;
    int device = 0;
    cudaGetDevice(&device);
    const Key key{device, st};
    if (pool.size() >= 64 && pool.find(key) == pool.end()) pool.clear();
    return pool[key];
}
int launch_slots_elitism(int32_t* pool, const int32_t* parent, const int32_t* child, const int32_t* partner, int s, int k,
                         int block_lo, int block_hi, const double* fit, const double* fit_m, int minimize, double pc, double pm,
                         uint32_t pool_size, uint64_t seed, uint64_t generation, int32_t* next_parent, int32_t* next_child,
                         double* next_fit, int32_t* order, int* status, cudaStream_t st) {
    constexpr int per_block = kSlotThreads / kSplit;
    const char* raw_min = std::getenv("GAPA_RANK_TILES_MIN");  // tests force either path
    const int tiles_min = raw_min ? std::max(1, std::atoi(raw_min)) : kRankTilesMin;
    if (s >= tiles_min) {
        const int tiles = 2 * ((s + kSortTile - 1) / kSortTile);
        RankScratch& sc = rank_scratch(st);
        GAPA_TRY(sc.key.ensure(sizeof(unsigned long long) * static_cast<size_t>(tiles) * kSortTile));
        GAPA_TRY(sc.idx.ensure(sizeof(int32_t) * static_cast<size_t>(tiles) * kSortTile));
        GAPA_LAUNCH(k_ga_sort_tiles, tiles, kSortTile, 0, st, fit, fit_m, s, minimize, sc.key.as<unsigned long long>(), sc.idx.as<int32_t>(), status);
        GAPA_LAUNCH(k_ga_slots_rank_tiles, (2 * s + per_block - 1) / per_block, kSlotThreads, 0, st, fit, fit_m, s, minimize,
                    sc.key.as<unsigned long long>(), sc.idx.as<int32_t>(), order);
    } else {
        GAPA_LAUNCH(k_ga_slots_rank, (2 * s + per_block - 1) / per_block, kSlotThreads, 0, st, fit, fit_m, s, minimize, order, status);
    }
    if ((block_lo > 0 || block_hi < s) && k > 0)
        GAPA_LAUNCH(k_ga_slots_rebuild, slot_grid((k & 3) ? k : k / 4, s), kSlotThreads, 0, st,
                    make_variation_params(pc, pm, pool_size, s, seed, generation), pool, parent, child, partner, k, s, order, block_lo, block_hi);
    GAPA_LAUNCH(k_ga_slots_commit, (s + kSlotThreads - 1) / kSlotThreads, kSlotThreads, 0, st, parent, child, fit, fit_m, s, order,
                next_parent, next_child, next_fit);
    return GAPA_CUDA_OK;
}
// elitism + GenerationStats::best / mean in one launch; only for an unsharded run with 2s <= 1024
int launch_slots_elitism_small(const int32_t* parent, const int32_t* child, int s, const double* fit, const double* fit_m, int minimize,
                               int32_t* next_parent, int32_t* next_child, double* next_fit, int32_t* order, int* status,
                               double* hist_best, double* hist_mean, int select_next, uint64_t seed, uint64_t next_generation,
                               int32_t* partner, double* weights, double* cumulative, cudaStream_t st) {
    GAPA_LAUNCH_PDL(k_ga_slots_elitism_small, 1, 1024, 0, st, parent, child, fit, fit_m, s, minimize, order, next_parent, next_child,
                next_fit, status, hist_best, hist_mean, select_next, seed, next_generation, partner, weights, cumulative);
    return GAPA_CUDA_OK;
}
int launch_slots_gather(const int32_t* pool, const int32_t* table, int rows, int k, int32_t* out, cudaStream_t st) {
    if (rows == 0 || k == 0) return GAPA_CUDA_OK;
    GAPA_LAUNCH(k_ga_slots_gather, slot_grid(k, rows), kSlotThreads, 0, st, pool, table, k, out);
    return GAPA_CUDA_OK;
}

}  // namespace gapa_b200

using namespace gapa_b200;

extern "C" {

int gapa_cuda_ga_slots_identity_device(int s, int32_t* parent_dev, int32_t* child_dev, void* stream) {
    if (s < 1 || !parent_dev || !child_dev) return fail(GAPA_CUDA_E_INVALID, "slots: bad arguments");
    return launch_slots_identity(s, parent_dev, child_dev, static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_slots_variation_device(int32_t* pool_dev, const int32_t* parent_dev, const int32_t* child_dev,
                                        const int32_t* partner_dev, int s, int k, int row_first, int row_count, double pc,
                                        double pm, int32_t pool_size, uint64_t seed, uint64_t generation, void* stream) {
    if (!(pc >= 0.0 && pc <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pc must be in [0, 1]");
    if (!(pm >= 0.0 && pm <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pm must be in [0, 1]");
    if (pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "mutate: empty gene pool");
    if (row_first < 0 || row_count < 0 || row_first + row_count > s) return fail(GAPA_CUDA_E_INVALID, "variation: row block outside the population");
    return launch_slots_variation(pool_dev, parent_dev, child_dev, partner_dev, s, k, row_first, row_count, pc, pm,
                                  static_cast<uint32_t>(pool_size), seed, generation, static_cast<cudaStream_t>(stream));
}

int gapa_cuda_ga_slots_gather_device(const int32_t* pool_dev, const int32_t* table_dev, int rows, int k, int32_t* out_dev,
                                     void* stream) {
    if (rows < 0 || k < 0) return fail(GAPA_CUDA_E_INVALID, "gather: negative shape");
    return launch_slots_gather(pool_dev, table_dev, rows, k, out_dev, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
