// Community-detection attack fitness (GAPA_TASK_CDA): modularity of the greedy
// detector's partition on the edge-perturbed graph.
//
// Reference path per individual (fitness.cpp:35-41): copy the dense adjacency, clear
// two bits per gene, return -0.5 if no edge is left, else detect_communities
// (community.cpp:28-91) — repeat { scan ALL adjacent community pairs (a < b) in (a, b)
// order, gain = e/m - da*db/(2*m*m) in FP64, keep the strictly greatest; merge b into
// a } — then modularity() (community.cpp:93-117) summed over communities in order of
// their smallest member.  The rescans make it O(#merges x #pairs) through std::map.
//
// Here: one CTA per individual runs the identical merge sequence on CNM-style state:
//   * per community an unsorted neighbour list (id, edge count, cached gain) in an
//     L2-resident entry pool, seeded in place from the CSR rows minus removed edges
//     (EdgeRemoval pools), or from the CSR rows plus the distinct added pairs
//     (EdgeAddition pools, gene_pool.cpp:57-60) — lists are unsorted, so an added edge
//     is just one more entry at each end;
//   * per community a cached best partner among ids greater than its own.  Gains are never stored per
//     entry: gain(c, d) = e(c,d)/m - deg(c) deg(d)/(2 m^2) is evaluated from the entry's count and the two
//     degrees when a best is (re)computed.  m is constant during a detection, so a merge of b into a only
//     changes the gains of pairs that touch a — and for a neighbour c of a that is not a neighbour of b
//     that pair only gets WORSE (deg(a) grew), which matters only if a was c's cached best;
//   * each step = block-wide argmax over the cached bests with the reference's
//     tie-break (greatest gain, then smallest a, then smallest b == first strictly
//     greater pair in (a, b) scan order), then a cooperative merge: fold list(b) into
//     list(a) through a position map in shared memory; one pass over the new list(a) finds a's new best
//     and queues the few communities whose own list needs work — the neighbours of b (mirror entry
//     b -> a, counts) and the neighbours of a whose cached best was a — each taken by a group of lanes.
//     A merged community typically has hundreds of neighbours, b a dozen: the lists of the others are
//     not touched at all.
// Gains use the reference's exact FP64 expression (IEEE division, no FMA: the library
// is built with -fmad=false); community ids are "smallest member" because b always
// merges into a < b; Q is accumulated sequentially in ascending community id, which
// is first-appearance order (community.cpp:17-26).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"

namespace gapa_b200 {

#ifndef GAPA_CDA_THREADS
#define GAPA_CDA_THREADS 1024
#endif
static constexpr int kCdaThreads = GAPA_CDA_THREADS;
static constexpr int kCdaWarps = kCdaThreads / 32;
#ifndef GAPA_CDA_GROUP
#define GAPA_CDA_GROUP 8
#endif
#ifndef GAPA_CDA_SHORT
#define GAPA_CDA_SHORT 64
#endif
static constexpr int kCdaGroup = GAPA_CDA_GROUP;        // lanes that patch one neighbour's list together
static constexpr int kCdaShortList = GAPA_CDA_SHORT;   // lists up to this length are worked on by one lane group, longer ones by a warp
static constexpr int kCdaLongQueue = 1024;  // longer ones are queued for a warp each
static constexpr int kCdaWorkQueue = 2048;  // communities whose own list needs work in one merge step
static constexpr int kNbFlag = 1 << 30;     // position-map bit: the community is a neighbour of the merged-away b

struct CdaScratch {
    DevBuf gone, ints, doubles, e_id, e_cnt, status;
    size_t pool_cap = 0;
    int slots = 0;
    int hier_argmax = 1;  // GAPA_CDA_HIER=0: flat scan of the cached bests (tests run both)
};

struct CdaArgs {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const int32_t* edge_id;
    const int32_t* pool_map;
    const int32_t* add_u;  // EdgeAddition pool: gene -> endpoints (-1 = pair already an edge); null for EdgeRemoval
    const int32_t* add_v;
    int pool_size;
    int n;
    int mask_words;
    long long csr_slots;   // 2m: the first csr_slots pool entries mirror the CSR rows
    long long pool_cap;    // entries per individual slot
    unsigned* gone;        // [slots][mask_words]
    int32_t* ints;         // [slots][6][n]: cdeg, head, len, cap, merged_into, best_id
    int32_t* pos_global;   // [slots][n] position map when it does not fit in shared memory (may be null)
    double* best_gain;     // [slots][n]
    int32_t* e_id;         // [slots][pool_cap]
    int32_t* e_cnt;
    int* status;           // [0] = GAPA_CUDA_E_RANGE, [1] = pool overflow
};

struct Cand {
    double gain;
    int a, b;
};
// the reference's scan keeps the first strictly greater gain in (a asc, b asc) order
__device__ __forceinline__ bool cand_better(const Cand& x, const Cand& y) {
    if (x.b < 0) return false;
    if (y.b < 0) return true;
    if (x.gain != y.gain) return x.gain > y.gain;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
}
__device__ __forceinline__ Cand cand_warp_best(Cand c) {
    for (int off = 16; off; off >>= 1) {
        Cand o;
        o.gain = __shfl_xor_sync(0xffffffffu, c.gain, off);
        o.a = __shfl_xor_sync(0xffffffffu, c.a, off);
        o.b = __shfl_xor_sync(0xffffffffu, c.b, off);
        if (cand_better(o, c)) c = o;
    }
    return c;
}
// community.cpp:63
__device__ __forceinline__ double merge_gain(int edges, int da, int db, double m, double den) {
    return static_cast<double>(edges) / m - static_cast<double>(da) * static_cast<double>(db) / den;
}

// Cached best of a neighbour c of the merged community a when c's best partner was neither a nor b: every
// other entry of list(c) keeps its gain (deg(c), deg(d) and e(c, d) are untouched by the merge), the entry of
// b is gone and was not the best, so only the patched (c, a) entry can displace the cached best — O(1), no
// second scan of the list.  Same result as a fresh scan: the order of candidates is total.
__device__ __forceinline__ void refresh_best_unchanged(double* best_gain, int32_t* best_id, int32_t* dirty, int c, int old_best, int a,
                                                       double gn) {
    if (a > c && gn > 0.0) {
        const Cand cur{old_best >= 0 ? best_gain[c] : 0.0, c, old_best};
        const Cand x{gn, c, a};
        if (cand_better(x, cur)) {
            best_gain[c] = gn;
            best_id[c] = a;
            if (dirty) dirty[c >> 5] = 1;
        }
    }
}

extern __shared__ int32_t cda_smem[];

// Optional phase timers of the merge loop (build with GAPA_NVCC_EXTRA=-DGAPA_CDA_PROFILE; tools/probe_cda.py
// prints them): clock64 deltas of thread 0 of CTA 0 between the barriers that end each phase.
#ifdef GAPA_CDA_PROFILE
__device__ unsigned long long g_cda_phase[8];
#define CDA_TICK(k)                                                      \
    do {                                                                 \
        if (tid == 0 && blockIdx.x == 0) {                               \
            const long long now__ = clock64();                           \
            g_cda_phase[k] += static_cast<unsigned long long>(now__ - t_phase); \
            t_phase = now__;                                             \
        }                                                                \
    } while (0)
extern "C" int gapa_cuda_cda_phase_cycles(unsigned long long* out8, int reset) {
    if (cudaMemcpyFromSymbol(out8, g_cda_phase, sizeof(unsigned long long) * 8) != cudaSuccess) return 4;
    if (reset) {
        unsigned long long zero[8] = {0};
        if (cudaMemcpyToSymbol(g_cda_phase, zero, sizeof(zero)) != cudaSuccess) return 4;
    }
    return 0;
}
#else
#define CDA_TICK(k) do { } while (0)
#endif

template <int kT>  // threads per CTA: 512 for graphs up to 8192 vertices, 1024 beyond (measured, cda_eval)
__global__ void __launch_bounds__(kT, 1) k_cda(CdaArgs A, GeneRows genes, int rows,
                                                        int pos_in_smem, double* __restrict__ out,
                                                        int32_t* __restrict__ owner_out, int hier_off) {
    griddep_launch();
    griddep_wait();
    __shared__ Cand warp_cand[(kT / 32)];
    __shared__ Cand chosen;
    __shared__ long long sh_total;
    __shared__ long long sh_pool_top;
    __shared__ int sh_len, sh_pb, sh_new_head, sh_abort, sh_count;
    __shared__ int sh_scan[kT];
    __shared__ int long_queue[kCdaLongQueue];
    __shared__ int work_queue[kCdaWorkQueue];
    __shared__ int sh_long, sh_work;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = A.n;
    const size_t slot = blockIdx.x;
    unsigned* gone = A.gone + slot * A.mask_words;
    // pos_in_smem: 0 = everything in global scratch, 1 = position map in shared memory,
    // 2 = position map AND the per-community arrays (degree, list head / length, cached best) in
    // shared memory — every merge step chases these, so for n up to ~6000 they stay on chip.
    int32_t* cdeg = A.ints + slot * 6 * static_cast<size_t>(n);
    int32_t* head = cdeg + n;
    int32_t* len = head + n;
    int32_t* cap = len + n;
    int32_t* merged_into = cap + n;
    int32_t* best_id = merged_into + n;
    double* best_gain = A.best_gain + slot * n;
    if (pos_in_smem == 2) {
        best_gain = reinterpret_cast<double*>(cda_smem);  // 8-byte aligned at the start of the carve-out
        cdeg = cda_smem + 2 * static_cast<size_t>(n);
        head = cdeg + n;
        len = head + n;
        best_id = len + n;
    }
    int32_t* e_id = A.e_id + slot * A.pool_cap;
    int32_t* e_cnt = A.e_cnt + slot * A.pool_cap;
    // Two-level argmax over the cached bests: communities in groups of 32, one cached maximum per group,
    // recomputed only for the groups whose members changed their cached best in the last merge step (a, b
    // and the ~20 communities that got list work) — instead of all 1024 threads scanning all n every step.
    const bool hier = hier_off >= 0;
    const int n_groups = (n + 31) >> 5;
    double* gmax_gain = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(cda_smem) + (hier ? hier_off : 0));
    int32_t* gmax_a = reinterpret_cast<int32_t*>(gmax_gain + n_groups);
    int32_t* gmax_b = gmax_a + n_groups;
    int32_t* dirty = gmax_b + n_groups;
    int32_t* pos = pos_in_smem == 2 ? cda_smem + 6 * static_cast<size_t>(n) : (pos_in_smem ? cda_smem : A.pos_global + slot * n);

    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        // ---- perturbation (gene_pool.cpp:53-60) ----------------------------------------
        // EdgeRemoval: bit per edge rank.  EdgeAddition: bit per pool gene, so that a repeated gene
        // adds its pair once; merged_into[] doubles as the per-vertex count of added edges.
        const bool adding = A.add_u != nullptr;
        for (int w = tid; w < A.mask_words; w += kT) gone[w] = 0u;
        if (adding)
            for (int u = tid; u < n; u += kT) merged_into[u] = 0;
        if (tid == 0) { sh_total = 0; sh_abort = 0; }
        __syncthreads();
        const int cols = genes.cols;
        const int32_t* g = genes.row(r);
        for (int j = tid; j < cols; j += kT) {
            const int gene = g[j];
            if (gene < 0 || gene >= A.pool_size) { A.status[0] = GAPA_CUDA_E_RANGE; sh_abort = 1; continue; }
            if (adding) {
                const int a = A.add_u[gene];
                if (a < 0) continue;
                const unsigned bit = 1u << (gene & 31);
                if (!(atomicOr(&gone[gene >> 5], bit) & bit)) {
                    atomicAdd(&merged_into[a], 1);
                    atomicAdd(&merged_into[A.add_v[gene]], 1);
                }
            } else {
                const int e = A.pool_map ? A.pool_map[gene] : gene;
                if (e >= 0) atomicOr(&gone[e >> 5], 1u << (e & 31));  // -1: the pair is not an edge of this graph, a no-op
            }
        }
        __syncthreads();
        if (sh_abort) { if (tid == 0) out[r] = 0.0; __syncthreads(); continue; }

        // ---- singleton communities: list(u) = perturbed adjacency row ------------------
        long long my_deg = 0;
        if (!adding) {  // surviving CSR row, in place
            for (int u = tid; u < n; u += kT) {
                const int off = A.row_ptr[u], end = A.row_ptr[u + 1];
                int cnt = 0;
                for (int i = off; i < end; ++i) {
                    const int e = A.edge_id[i];
                    if (!((gone[e >> 5] >> (e & 31)) & 1u)) {
                        e_id[off + cnt] = A.col_idx[i];
                        e_cnt[off + cnt] = 1;
                        ++cnt;
                    }
                }
                head[u] = off; len[u] = cnt; cap[u] = end - off; cdeg[u] = cnt; merged_into[u] = -1;
                pos[u] = -1;
                my_deg += cnt;
            }
        } else {  // CSR row followed by room for the added pairs: heads by a block-wide prefix sum
            const int per = (n + kT - 1) / kT;
            const int u_lo = min(tid * per, n), u_hi = min(u_lo + per, n);
            int want = 0;
            for (int u = u_lo; u < u_hi; ++u) want += A.row_ptr[u + 1] - A.row_ptr[u] + merged_into[u];
            sh_scan[tid] = want;
            __syncthreads();
            for (int off = 1; off < kT; off <<= 1) {
                const int add = tid >= off ? sh_scan[tid - off] : 0;
                __syncthreads();
                sh_scan[tid] += add;
                __syncthreads();
            }
            int at = sh_scan[tid] - want;
            for (int u = u_lo; u < u_hi; ++u) {
                const int off = A.row_ptr[u], deg = A.row_ptr[u + 1] - off, full = deg + merged_into[u];
                for (int i = 0; i < deg; ++i) {
                    e_id[at + i] = A.col_idx[off + i];
                    e_cnt[at + i] = 1;
                }
                head[u] = at; len[u] = deg; cap[u] = full; cdeg[u] = full; merged_into[u] = -1;
                pos[u] = -1;
                at += full;
            }
            my_deg = want;
            __syncthreads();
            for (int j = tid; j < cols; j += kT) {  // the thread that clears a gene's bit appends its pair
                const int gene = g[j];
                const int a = A.add_u[gene];
                if (a < 0) continue;
                const unsigned bit = 1u << (gene & 31);
                if (atomicAnd(&gone[gene >> 5], ~bit) & bit) {
                    const int b = A.add_v[gene];
                    const int qa = head[a] + atomicAdd(&len[a], 1);
                    e_id[qa] = b;
                    e_cnt[qa] = 1;
                    const int qb = head[b] + atomicAdd(&len[b], 1);
                    e_id[qb] = a;
                    e_cnt[qb] = 1;
                }
            }
        }
        for (int off = 16; off; off >>= 1) my_deg += __shfl_down_sync(0xffffffffu, my_deg, off);
        if (lane == 0 && my_deg) atomicAdd(reinterpret_cast<unsigned long long*>(&sh_total), static_cast<unsigned long long>(my_deg));
        __syncthreads();
        const long long total_degree = sh_total;
        if (total_degree == 0) {  // fitness.cpp:39
            if (tid == 0) out[r] = -0.5;
            __syncthreads();
            continue;
        }
        const double m = static_cast<double>(total_degree) / 2.0;  // community.cpp:36
        const double den = 2.0 * m * m;
        if (tid == 0) sh_pool_top = adding ? total_degree : A.csr_slots;

        if (hier)
            for (int g2 = tid; g2 < n_groups; g2 += kT) dirty[g2] = 1;
        // initial cached bests
        for (int u = tid; u < n; u += kT) {
            const int h = head[u], l = len[u], du = cdeg[u];
            Cand best{0.0, u, -1};
            for (int i = 0; i < l; ++i) {
                const int v = e_id[h + i];
                if (v <= u) continue;
                const double gn = merge_gain(1, du, cdeg[v], m, den);
                if (gn > 0.0) {
                    const Cand c{gn, u, v};
                    if (cand_better(c, best)) best = c;
                }
            }
            best_gain[u] = best.gain;
            best_id[u] = best.b;
        }
        __syncthreads();

        // List work for one neighbour c of the merged community a, by a group of W lanes (W = 1: one thread):
        // if c was a neighbour of b, its mirror entry b becomes / is folded into its entry a (count `e`);
        // then c's cached best — O(1) unless its best partner was a or b, else a fresh scan of list(c).
        auto list_work = [&](auto width, int c, int e, bool is_nb, int a, int b, int da, int gl, unsigned gmask) {
            constexpr int W = decltype(width)::value;
            const int hc = head[c];
            int lc = len[c];
            const int leader = lane - gl;
            const double gn = merge_gain(e, da, cdeg[c], m, den);
            if (is_nb) {
                int pa = -1, pbb = -1;
                for (int t = gl; t < lc; t += W) {
                    const int id = e_id[hc + t];
                    if (id == a) pa = t;
                    if (id == b) pbb = t;
                }
#pragma unroll
                for (int off = W / 2; off; off >>= 1) {
                    pa = max(pa, __shfl_xor_sync(gmask, pa, off));
                    pbb = max(pbb, __shfl_xor_sync(gmask, pbb, off));
                }
                __syncwarp(gmask);  // every lane has read len[c] and its entries before the leader rewrites them
                if (gl == 0) {
                    if (pa >= 0) {
                        if (pbb >= 0) {
                            const int last = lc - 1;
                            if (pbb != last) {
                                e_id[hc + pbb] = e_id[hc + last];
                                e_cnt[hc + pbb] = e_cnt[hc + last];
                                if (pa == last) pa = pbb;
                            }
                            len[c] = last;
                        }
                        e_cnt[hc + pa] = e;
                    } else {
                        e_id[hc + pbb] = a;
                        e_cnt[hc + pbb] = e;
                    }
                }
                if (pa >= 0 && pbb >= 0) --lc;  // the same on every lane of the group
            }
            // the leader alone reads the cached best (it is also the one that rewrites it) and tells the group
            const int old_best = __shfl_sync(gmask, gl == 0 ? best_id[c] : 0, leader);
            if (old_best != a && old_best != b) {
                if (gl == 0) refresh_best_unchanged(best_gain, best_id, hier ? dirty : nullptr, c, old_best, a, gn);
                return;
            }
            __syncwarp(gmask);  // the leader's patch is visible to the group
            const int dc = cdeg[c];
            Cand best_c{0.0, c, -1};
            for (int t = gl; t < lc; t += W) {
                const int id = e_id[hc + t];
                if (id <= c) continue;
                const double gg = merge_gain(e_cnt[hc + t], dc, cdeg[id], m, den);
                if (gg > 0.0) {
                    const Cand x{gg, c, id};
                    if (cand_better(x, best_c)) best_c = x;
                }
            }
#pragma unroll
            for (int off = W / 2; off; off >>= 1) {
                Cand o;
                o.gain = __shfl_xor_sync(gmask, best_c.gain, off);
                o.a = c;
                o.b = __shfl_xor_sync(gmask, best_c.b, off);
                if (cand_better(o, best_c)) best_c = o;
            }
            if (gl == 0) {
                best_gain[c] = best_c.gain;
                best_id[c] = best_c.b;
                if (hier) dirty[c >> 5] = 1;
            }
        };

        // ---- greedy agglomeration (community.cpp:55-87) --------------------------------
#ifdef GAPA_CDA_PROFILE
        long long t_phase = clock64();
#endif
        for (;;) {
            if (hier) {
                for (int g2 = warp; g2 < n_groups; g2 += (kT / 32)) {
                    const int is_dirty = dirty[g2];  // uniform within the warp
                    __syncwarp();                    // every lane has read the flag before lane 0 clears it below
                    if (!is_dirty) continue;
                    const int c = g2 * 32 + lane;
                    Cand x{0.0, c, -1};
                    if (c < n) {
                        const int bb = best_id[c];
                        if (bb >= 0) { x.gain = best_gain[c]; x.b = bb; }
                    }
                    x = cand_warp_best(x);
                    if (lane == 0) { gmax_gain[g2] = x.gain; gmax_a[g2] = x.a; gmax_b[g2] = x.b; dirty[g2] = 0; }
                }
                __syncthreads();
                if (warp == 0) {
                    Cand x{0.0, -1, -1};
                    for (int g2 = lane; g2 < n_groups; g2 += 32) {
                        const Cand y{gmax_gain[g2], gmax_a[g2], gmax_b[g2]};
                        if (cand_better(y, x)) x = y;
                    }
                    x = cand_warp_best(x);
                    if (lane == 0) chosen = x;
                }
                __syncthreads();
            } else {
                Cand mine{0.0, -1, -1};
                for (int c = tid; c < n; c += kT) {
                    const int b = best_id[c];
                    if (b >= 0) {
                        const Cand x{best_gain[c], c, b};
                        if (cand_better(x, mine)) mine = x;
                    }
                }
                mine = cand_warp_best(mine);
                if (lane == 0) warp_cand[warp] = mine;
                __syncthreads();
                if (warp == 0) {
                    Cand x = lane < (kT / 32) ? warp_cand[lane] : Cand{0.0, -1, -1};
                    x = cand_warp_best(x);
                    if (lane == 0) chosen = x;
                }
                __syncthreads();
            }
            const int a = chosen.a, b = chosen.b;
            if (b < 0) break;
            CDA_TICK(0);  // argmax

            // make room: list(a) must hold len(a) + len(b) entries
            const int la = len[a], lb = len[b];
            int ha = head[a];
            const int hb = head[b];
            if (cap[a] < la + lb) {
                if (tid == 0) {
                    const long long want = 2ll * (la + lb);
                    if (sh_pool_top + want > A.pool_cap) { sh_abort = 1; A.status[1] = 1; }
                    else { sh_new_head = static_cast<int>(sh_pool_top); sh_pool_top += want; }
                }
                __syncthreads();
                if (sh_abort) break;
                const int nh = sh_new_head;
                for (int i = tid; i < la; i += kT) { e_id[nh + i] = e_id[ha + i]; e_cnt[nh + i] = e_cnt[ha + i]; }
                __syncthreads();
                if (tid == 0) { head[a] = nh; cap[a] = 2 * (la + lb); }
                ha = nh;
            }
            // positions of list(a) in the map
            for (int i = tid; i < la; i += kT) pos[e_id[ha + i]] = i;
            if (tid == 0) sh_len = la;
            __syncthreads();
            CDA_TICK(1);  // room + mark positions
            if (tid == 0) sh_pb = pos[b];
            // fold list(b) into list(a); every neighbour of b ends up in the map, flagged
            for (int j = tid; j < lb; j += kT) {
                const int c = e_id[hb + j];
                if (c == a) continue;
                const int e = e_cnt[hb + j];
                const int p = pos[c];
                if (p >= 0) {
                    e_cnt[ha + p] += e;
                    pos[c] = p | kNbFlag;
                } else {
                    const int q = atomicAdd(&sh_len, 1);
                    e_id[ha + q] = c;
                    e_cnt[ha + q] = e;
                    pos[c] = q | kNbFlag;
                }
            }
            __syncthreads();
            CDA_TICK(2);  // fold
            if (tid == 0) {  // drop the (a, b) entry itself
                const int last = sh_len - 1, pb = sh_pb;
                if (pb != last) {
                    const int moved = e_id[ha + last];
                    e_id[ha + pb] = moved;
                    e_cnt[ha + pb] = e_cnt[ha + last];
                    pos[moved] = pb | (pos[moved] & kNbFlag);
                }
                pos[b] = -1;
                sh_len = last;
                len[a] = last;
                cdeg[a] += cdeg[b];
                len[b] = 0;
                merged_into[b] = a;
                best_id[b] = -1;
                if (hier) dirty[b >> 5] = 1;
                sh_work = 0;
                sh_long = 0;
            }
            __syncthreads();
            CDA_TICK(3);  // drop
            const int la2 = sh_len, da = cdeg[a];

            // One pass over the new list(a): a's own best (every gain of a changed), and the queue of communities
            // whose list needs work — the neighbours of b, and neighbours whose cached best was a (their pair with
            // a only got worse).  A full queue makes the finder do the work itself.
            Cand best_a{0.0, a, -1};
            for (int i = tid; i < la2; i += kT) {
                const int c = e_id[ha + i], e = e_cnt[ha + i];
                if (c > a) {
                    const double gn = merge_gain(e, da, cdeg[c], m, den);
                    if (gn > 0.0) {
                        const Cand x{gn, a, c};
                        if (cand_better(x, best_a)) best_a = x;
                    }
                }
                const bool is_nb = (pos[c] & kNbFlag) != 0;
                if (is_nb || (c < a && best_id[c] == a)) {
                    // long lists are queued for a whole warp, short ones for a group of lanes — decided HERE, so that both
                    // kinds are worked on at the same time after one barrier (round 1: long lists were found by the
                    // groups and done in a phase of their own: 2 of a step's 9 us)
                    bool queued = false;
                    if (len[c] > kCdaShortList) {
                        const int ql = atomicAdd(&sh_long, 1);
                        if (ql < kCdaLongQueue) { long_queue[ql] = i; queued = true; }
                    }
                    if (!queued) {
                        const int q = atomicAdd(&sh_work, 1);
                        if (q < kCdaWorkQueue) work_queue[q] = i;
                        else list_work(std::integral_constant<int, 1>{}, c, e, is_nb, a, b, da, 0, 1u << lane);
                    }
                }
            }
            __syncthreads();
            CDA_TICK(4);  // scan of list(a)
            const int n_work = min(sh_work, kCdaWorkQueue);
            const int n_long = min(sh_long, kCdaLongQueue);
            // warps [0, long_warps) take the long lists (one warp per list), the others the short ones (a group of lanes per
            // list); at least a quarter of the warps stay with the short lists
            const int long_warps = min(n_long, (kT / 32) - (kT / 32) / 4);
            if (warp < long_warps) {
                for (int q = warp; q < n_long; q += long_warps) {
                    const int i = long_queue[q];
                    const int c = e_id[ha + i];
                    list_work(std::integral_constant<int, 32>{}, c, e_cnt[ha + i], (pos[c] & kNbFlag) != 0, a, b, da, lane, 0xffffffffu);
                }
            } else {
                const int gl = lane % kCdaGroup;
                const unsigned gmask = ((1u << kCdaGroup) - 1u) << (lane - gl);
                const int groups = ((kT / 32) - long_warps) * (32 / kCdaGroup);
                for (int w = (warp - long_warps) * (32 / kCdaGroup) + lane / kCdaGroup; w < n_work; w += groups) {
                    const int i = work_queue[w];
                    const int c = e_id[ha + i];
                    list_work(std::integral_constant<int, kCdaGroup>{}, c, e_cnt[ha + i], (pos[c] & kNbFlag) != 0, a, b, da, gl, gmask);
                }
            }
            CDA_TICK(5);  // (unused: short and long lists are one phase now)
            best_a = cand_warp_best(best_a);
            if (lane == 0) warp_cand[warp] = best_a;
            __syncthreads();
            CDA_TICK(6);  // list work (long lists)
            if (warp == 0) {
                Cand x = lane < (kT / 32) ? warp_cand[lane] : Cand{0.0, a, -1};
                x = cand_warp_best(x);
                if (lane == 0) { best_gain[a] = x.gain; best_id[a] = x.b; if (hier) dirty[a >> 5] = 1; }
            }
            for (int i = tid; i < la2; i += kT) pos[e_id[ha + i]] = -1;  // the map is empty again
            __syncthreads();
            CDA_TICK(7);  // best of the merged community + map reset
        }
        if (sh_abort) { if (tid == 0) out[r] = 0.0; __syncthreads(); continue; }

        // detect_communities' partition (community.cpp:28-91) for the reporting path: the owner of
        // u is the root of its merge chain == the smallest member of its community.
        if (owner_out) {
            for (int u = tid; u < n; u += kT) {
                int root = u;
                while (merged_into[root] != -1) root = merged_into[root];
                owner_out[static_cast<size_t>(r) * n + u] = root;
            }
        }

        // ---- modularity (community.cpp:93-117) ------------------------------------------
        // Live communities in ascending id == first-appearance order.  A term that is
        // exactly zero cannot change the running sum, so only non-zero terms are queued.
        const double two_m = static_cast<double>(total_degree);
        const int per = (n + kT - 1) / kT;
        const int c_lo = min(tid * per, n), c_hi = min(c_lo + per, n);
        int queued = 0;
        for (int c = c_lo; c < c_hi; ++c) {
            if (merged_into[c] != -1) continue;
            long long outside = 0;
            const int h = head[c], l = len[c];
            for (int i = 0; i < l; ++i) outside += e_cnt[h + i];
            const double intra = static_cast<double>((cdeg[c] - outside) / 2);
            const double ee = intra / (two_m / 2.0);
            const double aa = static_cast<double>(cdeg[c]) / two_m;
            const double term = ee - aa * aa;
            best_gain[c] = term;
            best_id[c] = term != 0.0 ? 1 : 0;
            queued += term != 0.0;
        }
        sh_scan[tid] = queued;
        __syncthreads();
        for (int off = 1; off < kT; off <<= 1) {
            const int add = tid >= off ? sh_scan[tid - off] : 0;
            __syncthreads();
            sh_scan[tid] += add;
            __syncthreads();
        }
        int write = sh_scan[tid] - queued;
        for (int c = c_lo; c < c_hi; ++c)
            if (merged_into[c] == -1 && best_id[c]) head[write++] = c;  // head[] is free now: ordered queue
        if (tid == kT - 1) sh_count = sh_scan[tid];
        __syncthreads();
        if (tid == 0) {
            double q = 0.0;
            const int count = sh_count;
            for (int i = 0; i < count; ++i) q += best_gain[head[i]];
            out[r] = q;
        }
        __syncthreads();
    }
}

int cda_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, int32_t* owner_out_dev) {
    if (!ctx->cda) ctx->cda = new CdaScratch();
    CdaScratch* s = ctx->cda;
    const int n = ctx->n;
    if (n == 0) return fail(GAPA_CUDA_E_INVALID, "cda_fitness: empty graph");
    if (const char* raw = std::getenv("GAPA_CDA_HIER")) s->hier_argmax = *raw != '0';
    const long long csr_slots = 2 * ctx->m;
    const bool adding = ctx->pool_kind == GAPA_POOL_EDGE_ADDITION;
    const int mask_words = static_cast<int>(((adding ? static_cast<int64_t>(ctx->pool_size) : ctx->m) + 31) / 32) + 1;
    const int slots = std::max(1, std::min(rows, ctx->sm_count));
    const int pos_in_smem = static_cast<size_t>(n) * 7 * sizeof(int32_t) <= 200 * 1024 ? 2 : (static_cast<size_t>(n) * sizeof(int32_t) <= 160 * 1024 ? 1 : 0);
    s->pool_cap = std::max(s->pool_cap, static_cast<size_t>(csr_slots + (adding ? 2ll * genes.cols : 0)) * 6 + 4096);

    for (;;) {
        GAPA_TRY(s->gone.ensure(sizeof(unsigned) * mask_words * static_cast<size_t>(slots)));
        GAPA_TRY(s->ints.ensure(sizeof(int32_t) * 7 * static_cast<size_t>(n) * slots));
        GAPA_TRY(s->doubles.ensure(sizeof(double) * static_cast<size_t>(n) * slots));
        GAPA_TRY(s->e_id.ensure(sizeof(int32_t) * s->pool_cap * slots));
        GAPA_TRY(s->e_cnt.ensure(sizeof(int32_t) * s->pool_cap * slots));
        GAPA_TRY(s->status.ensure(2 * sizeof(int)));
        GAPA_CUDA_TRY(cudaMemsetAsync(s->status.ptr, 0, 2 * sizeof(int), stream));

        CdaArgs A;
        A.row_ptr = ctx->d_row_ptr;
        A.col_idx = ctx->d_col_idx;
        A.edge_id = ctx->d_edge_id;
        A.pool_map = ctx->pool_identity ? nullptr : ctx->d_pool_map;
        A.add_u = adding ? ctx->d_add_u : nullptr;
        A.add_v = adding ? ctx->d_add_v : nullptr;
        A.pool_size = ctx->pool_size;
        A.n = n;
        A.mask_words = mask_words;
        A.csr_slots = csr_slots;
        A.pool_cap = static_cast<long long>(s->pool_cap);
        A.gone = s->gone.as<unsigned>();
        A.ints = s->ints.as<int32_t>();
        A.pos_global = pos_in_smem ? nullptr : s->ints.as<int32_t>() + static_cast<size_t>(6) * n * slots;
        A.best_gain = s->doubles.as<double>();
        A.e_id = s->e_id.as<int32_t>();
        A.e_cnt = s->e_cnt.as<int32_t>();
        A.status = s->status.as<int>();
        const size_t base_smem = pos_in_smem == 2 ? static_cast<size_t>(n) * 7 * sizeof(int32_t) : (pos_in_smem ? static_cast<size_t>(n) * sizeof(int32_t) : 0);
        const size_t n_groups = (static_cast<size_t>(n) + 31) / 32;
        const size_t hier_at = (base_smem + 7) & ~size_t{7};
        const size_t hier_bytes = n_groups * (sizeof(double) + 3 * sizeof(int32_t));
        const bool hier = s->hier_argmax && hier_at + hier_bytes <= 209 * 1024;  // 227 KB minus the kernel's static shared memory
        const size_t smem = hier ? hier_at + hier_bytes : base_smem;
        // CTA size: a merge step is a chain of barriers and dependent L2 round trips, cheaper with 16 warps than with 32 while
        // the lists are short — C2 (n = 5000) 42.1 -> 40.4 ms with 512 threads, but n = 20,000 300 -> 348 ms (768: 41.1 / 319)
        if (n <= 8192 && kCdaThreads == 1024) {
            GAPA_CUDA_TRY(cudaFuncSetAttribute(k_cda<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GAPA_LAUNCH(k_cda<512>, slots, 512, smem, stream, A, genes, rows, pos_in_smem, out_dev, owner_out_dev,
                        hier ? static_cast<int>(hier_at) : -1);
        } else {
            GAPA_CUDA_TRY(cudaFuncSetAttribute(k_cda<kCdaThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GAPA_LAUNCH(k_cda<kCdaThreads>, slots, kCdaThreads, smem, stream, A, genes, rows, pos_in_smem, out_dev, owner_out_dev,
                        hier ? static_cast<int>(hier_at) : -1);
        }
        GAPA_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, s->status.ptr, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
        GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
        if (ctx->h_status[0] == GAPA_CUDA_E_RANGE) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
        if (ctx->h_status[1]) {  // entry pool exhausted: double it and evaluate the batch again
            s->pool_cap *= 2;
            continue;
        }
        return GAPA_CUDA_OK;
    }
}

void cda_free(gapa_cuda_ctx* ctx) {
    if (!ctx->cda) return;
    CdaScratch* s = ctx->cda;
    for (DevBuf* b : {&s->gone, &s->ints, &s->doubles, &s->e_id, &s->e_cnt, &s->status}) b->release();
    delete s;
    ctx->cda = nullptr;
}

}  // namespace gapa_b200
