// Pairwise-connectivity / largest-component fitness (GAPA_TASK_PC, GAPA_TASK_MCN).
//
// Reference path being replaced, per individual (fitness.cpp:28-33, :18-26):
//   copy the dense n x n BitMatrix, zero a row + column per gene
//   (gene_pool.cpp:61-64), DFS components (components.cpp:9-35), then
//   PC = sum s(s-1)/2 (components.cpp:49-56) or MCN = max s (:58-62); removed
//   nodes stay as singletons.
//
// B200 design — bit-sliced over individuals:
//   * 64 individuals form a group; per vertex ONE 64-bit word holds "alive in
//     individual b" and one holds "reached from the group's BFS sources", so a
//     single pass over the shared CSR serves 64 individuals and every 32-byte
//     sector fetched for a neighbour word carries 64 individuals of state.
//     The CSR is never copied; a perturbation is just the alive-word bit.
//   * phase 1 (k_sweep) closes reachability from one high-degree source per
//     individual by asynchronous bottom-up sweeps: a vertex ORs its
//     neighbours' reached words until every individual it is alive in is
//     covered (early exit after ~2 neighbours on power-law graphs, because
//     rows are sorted and the oldest / highest-degree neighbours come first).
//   * phase 2 finishes exactly, whatever phase 1 left: alive-but-unreached
//     vertices that have an alive neighbour are compacted to (vertex, bits)
//     entries and resolved by a lock-free union-find over compact slots, with
//     one virtual "giant" node per individual standing for everything phase 1
//     reached.  Isolated leftovers are singletons and need no work.
//   * component sizes: reached count = n - (zero bits of the reached words),
//     counted per bit position with shared-memory histograms.
// Integer arithmetic end to end; PC fits int64 and is exact in the returned
// double for n <= 9.4e7 (PC < 2^53).
#include <algorithm>

#include "internal.cuh"

namespace gapa_b200 {

typedef unsigned long long word_t;
static constexpr int kBits = 64;
static constexpr int kThreads = 256;

struct PcCounters {
    unsigned int n_entries;
    unsigned int n_slots;
    int overflow;
    int range_error;
};

struct PcScratch {
    DevBuf alive, reached, entry_of, zeros, flags, counters;
    DevBuf left_v, left_g, left_w, left_base, parent, comp_size, pc_extra, mcn_extra;
    size_t cap_entries = 0, cap_slots = 0;
    int sweeps_last = 0;
};

// ---------------------------------------------------------------------------------
// mask build
__global__ void __launch_bounds__(kThreads) k_pc_init(word_t* __restrict__ alive, word_t* __restrict__ reached,
                                                      int n, int groups, int rows) {
    const size_t total = static_cast<size_t>(groups) * n;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(i / n);
        const int valid = min(kBits, rows - g * kBits);
        alive[i] = valid >= kBits ? ~0ull : ((1ull << valid) - 1ull);
        reached[i] = 0ull;
    }
}

// apply_in_place for NodeRemoval (gene_pool.cpp:61-64): clear the individual's bit
// in the removed vertex's alive word.  Duplicates are idempotent.
__global__ void __launch_bounds__(kThreads) k_pc_remove(const int32_t* __restrict__ genes, size_t cells, int cols,
                                                        const int32_t* __restrict__ pool_map, int pool_size, int n,
                                                        word_t* alive, PcCounters* counters) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int row = static_cast<int>(i / cols);
        const int gene = genes[i];
        if (gene < 0 || gene >= pool_size) {
            counters->range_error = 1;
            continue;
        }
        const int node = pool_map ? pool_map[gene] : gene;
        atomicAnd(&alive[static_cast<size_t>(row >> 6) * n + node], ~(1ull << (row & 63)));
    }
}

// One warp per individual: the first alive vertex in descending-degree order
// becomes the BFS source.  Any alive vertex would be correct; a hub makes
// phase 1 cover the giant component.
__global__ void __launch_bounds__(kThreads) k_pc_source(const int32_t* __restrict__ by_degree, int n, int rows,
                                                        const word_t* __restrict__ alive, word_t* reached) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const size_t base = static_cast<size_t>(row >> 6) * n;
    const word_t bit = 1ull << (row & 63);
    for (int i = 0; i < n; i += 32) {
        const int v = i + lane < n ? by_degree[i + lane] : -1;
        const bool ok = v >= 0 && (alive[base + v] & bit);
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        if (hit) {
            if (lane == __ffs(hit) - 1) atomicOr(&reached[base + v], bit);
            return;
        }
    }
}

// ---------------------------------------------------------------------------------
// phase 1: asynchronous bottom-up reachability sweep, one thread per vertex and
// group.  Reads of neighbours' words race benignly with writes (words only gain
// bits; 64-bit stores are single transactions), so a sweep can use bits set
// earlier in the same sweep and converges in far fewer passes than BFS levels.
__global__ void __launch_bounds__(kThreads) k_pc_sweep(const int32_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col_idx, int n,
                                                       const word_t* __restrict__ alive, word_t* reached,
                                                       const int* __restrict__ changed_in, int* changed_out) {
    const int g = blockIdx.y;
    if (changed_in && !changed_in[g]) return;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    int any = 0;
    if (v < n) {
        const size_t base = static_cast<size_t>(g) * n;
        const word_t mine = reached[base + v];
        const word_t todo = alive[base + v] & ~mine;
        if (todo) {
            const int beg = row_ptr[v], end = row_ptr[v + 1];
            word_t got = 0ull;
            int e = beg;
            // two neighbours per step: both loads are in flight together
            for (; e + 1 < end; e += 2) {
                const int u0 = col_idx[e], u1 = col_idx[e + 1];
                const word_t r0 = __ldcg(&reached[base + u0]);
                const word_t r1 = __ldcg(&reached[base + u1]);
                got |= r0 | r1;
                if ((got & todo) == todo) break;
            }
            if (e + 1 == end && (got & todo) != todo) got |= __ldcg(&reached[base + col_idx[e]]);
            got &= todo;
            if (got) {
                reached[base + v] = mine | got;
                any = 1;
            }
        }
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) changed_out[g] = 1;
}

// ---------------------------------------------------------------------------------
// finalize: per bit position count the vertices NOT reached (so reached = n - zeros),
// and compact the alive, unreached, non-isolated (vertex, bits) leftovers.
__global__ void __launch_bounds__(kThreads) k_pc_finalize(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx, int n, int rows,
    const word_t* __restrict__ alive, const word_t* __restrict__ reached, int* zeros, int32_t* entry_of,
    int32_t* left_v, int32_t* left_g, word_t* left_w, int32_t* left_base, int32_t* parent, int32_t* comp_size,
    unsigned cap_entries, unsigned cap_slots, int slot0, PcCounters* counters) {
    __shared__ int hist[kBits];
    const int g = blockIdx.y;
    if (threadIdx.x < kBits) hist[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(g) * n;
    const int valid = min(kBits, rows - g * kBits);
    const word_t group_mask = valid >= kBits ? ~0ull : ((1ull << valid) - 1ull);
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const word_t r = reached[base + v];
        word_t z = ~r & group_mask;
        while (z) {
            const int b = __ffsll(static_cast<long long>(z)) - 1;
            z &= z - 1;
            atomicAdd(&hist[b], 1);
        }
        word_t left = alive[base + v] & ~r;
        if (left) {
            // keep only the individuals in which v has an alive neighbour
            word_t nb = 0ull;
            for (int e = row_ptr[v]; e < row_ptr[v + 1] && (nb & left) != left; ++e) nb |= alive[base + col_idx[e]];
            left &= nb;
        }
        if (left) {
            const int cnt = __popcll(left);
            const unsigned e = atomicAdd(&counters->n_entries, 1u);
            const unsigned s = atomicAdd(&counters->n_slots, static_cast<unsigned>(cnt));
            if (e < cap_entries && s + cnt <= cap_slots) {
                left_v[e] = v;
                left_g[e] = g;
                left_w[e] = left;
                left_base[e] = static_cast<int32_t>(s);
                entry_of[base + v] = static_cast<int32_t>(e);
                for (int i = 0; i < cnt; ++i) {
                    parent[slot0 + s + i] = slot0 + static_cast<int32_t>(s) + i;
                    comp_size[slot0 + s + i] = 0;
                }
            } else {
                counters->overflow = 1;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < kBits && hist[threadIdx.x]) atomicAdd(&zeros[g * kBits + threadIdx.x], hist[threadIdx.x]);
}

// ---------------------------------------------------------------------------------
// phase 2: lock-free union-find over compact slots.  Slot r < slot0 is the virtual
// giant node of individual r; hooking always points the larger index at the
// smaller, so a set that touches the giant is rooted at the giant.
__device__ __forceinline__ int uf_find(int32_t* parent, int x) {
    volatile int32_t* p = parent;
    int px = p[x];
    while (px != x) {
        const int gp = p[px];
        if (gp != px) p[x] = gp;  // path halving; x is not a root, so no CAS can race on it
        x = px;
        px = gp;
    }
    return x;
}
__device__ __forceinline__ void uf_union(int32_t* parent, int a, int b) {
    for (;;) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a < b) { const int t = a; a = b; b = t; }
        if (atomicCAS(&parent[a], a, b) == a) return;
    }
}
__device__ __forceinline__ int slot_of(int slot0, int base, word_t w, int b) {
    return slot0 + base + __popcll(w & ((1ull << b) - 1ull));
}

__global__ void __launch_bounds__(kThreads) k_pc_hook(const int32_t* __restrict__ row_ptr,
                                                      const int32_t* __restrict__ col_idx, int n,
                                                      const word_t* __restrict__ alive,
                                                      const word_t* __restrict__ reached,
                                                      const int32_t* __restrict__ entry_of,
                                                      const int32_t* __restrict__ left_v,
                                                      const int32_t* __restrict__ left_g,
                                                      const word_t* __restrict__ left_w,
                                                      const int32_t* __restrict__ left_base, int32_t* parent,
                                                      int slot0, const PcCounters* counters) {
    const unsigned total = counters->n_entries;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int v = left_v[e], g = left_g[e], base_v = left_base[e];
        const word_t w = left_w[e];
        const size_t base = static_cast<size_t>(g) * n;
        for (int i = row_ptr[v]; i < row_ptr[v + 1]; ++i) {
            const int u = col_idx[i];
            const word_t common = w & alive[base + u];
            if (!common) continue;
            const word_t ru = reached[base + u];
            word_t attach = common & ru;  // non-zero only when phase 1 stopped before converging
            while (attach) {
                const int b = __ffsll(static_cast<long long>(attach)) - 1;
                attach &= attach - 1;
                uf_union(parent, slot_of(slot0, base_v, w, b), g * kBits + b);
            }
            word_t rest = common & ~ru;
            if (rest && u < v) {  // leftover-leftover edges are seen from both ends; take one
                const int eu = entry_of[base + u];
                const word_t wu = left_w[eu];
                const int base_u = left_base[eu];
                while (rest) {
                    const int b = __ffsll(static_cast<long long>(rest)) - 1;
                    rest &= rest - 1;
                    uf_union(parent, slot_of(slot0, base_v, w, b), slot_of(slot0, base_u, wu, b));
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_pc_count(const word_t* __restrict__ left_w,
                                                       const int32_t* __restrict__ left_base, int32_t* parent,
                                                       int32_t* comp_size, int slot0, const PcCounters* counters) {
    const unsigned total = counters->n_entries;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int cnt = __popcll(left_w[e]);
        for (int i = 0; i < cnt; ++i) atomicAdd(&comp_size[uf_find(parent, slot0 + left_base[e] + i)], 1);
    }
}

__global__ void __launch_bounds__(kThreads) k_pc_reduce(const int32_t* __restrict__ left_g,
                                                        const word_t* __restrict__ left_w,
                                                        const int32_t* __restrict__ left_base,
                                                        const int32_t* __restrict__ parent,
                                                        const int32_t* __restrict__ comp_size, int slot0,
                                                        unsigned long long* pc_extra, int* mcn_extra,
                                                        const PcCounters* counters) {
    const unsigned total = counters->n_entries;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        word_t w = left_w[e];
        const int g = left_g[e];
        int slot = slot0 + left_base[e];
        while (w) {
            const int b = __ffsll(static_cast<long long>(w)) - 1;
            w &= w - 1;
            if (parent[slot] == slot) {  // a root that is not a giant node
                const unsigned long long s = static_cast<unsigned long long>(comp_size[slot]);
                atomicAdd(&pc_extra[g * kBits + b], s * (s - 1ull) / 2ull);
                atomicMax(&mcn_extra[g * kBits + b], static_cast<int>(s));
            }
            ++slot;
        }
    }
}

// pairwise_connectivity / largest_component_size (components.cpp:49-62) -> double
// (fitness.cpp:25,32).  Every vertex outside the giant and outside the union-find
// components is a singleton: 0 pairs, size 1.
__global__ void __launch_bounds__(kThreads) k_pc_result(int n, int rows, int task, const int* __restrict__ zeros,
                                                        const int32_t* __restrict__ comp_size,
                                                        const unsigned long long* __restrict__ pc_extra,
                                                        const int* __restrict__ mcn_extra, double* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const long long giant = static_cast<long long>(n) - zeros[r] + comp_size[r];
    if (task == GAPA_TASK_PC) {
        const unsigned long long pairs = static_cast<unsigned long long>(giant * (giant - 1) / 2) + pc_extra[r];
        out[r] = static_cast<double>(pairs);
    } else {
        long long best = giant > mcn_extra[r] ? giant : mcn_extra[r];
        if (n > 0 && best < 1) best = 1;
        out[r] = static_cast<double>(best);
    }
}

__global__ void k_pc_reset(int groups, int32_t* parent, int32_t* comp_size, int* zeros,
                           unsigned long long* pc_extra, int* mcn_extra, PcCounters* counters, bool keep_range) {
    const int total = groups * kBits;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        parent[i] = i;
        comp_size[i] = 0;
        zeros[i] = 0;
        pc_extra[i] = 0ull;
        mcn_extra[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counters->n_entries = 0u;
        counters->n_slots = 0u;
        counters->overflow = 0;
        if (!keep_range) counters->range_error = 0;
    }
}

// ---------------------------------------------------------------------------------
static int ensure_phase2(PcScratch* s, int groups, size_t entries, size_t slots) {
    const size_t giant = static_cast<size_t>(groups) * kBits;
    GAPA_TRY(s->left_v.ensure(sizeof(int32_t) * entries));
    GAPA_TRY(s->left_g.ensure(sizeof(int32_t) * entries));
    GAPA_TRY(s->left_w.ensure(sizeof(word_t) * entries));
    GAPA_TRY(s->left_base.ensure(sizeof(int32_t) * entries));
    GAPA_TRY(s->parent.ensure(sizeof(int32_t) * (giant + slots)));
    GAPA_TRY(s->comp_size.ensure(sizeof(int32_t) * (giant + slots)));
    s->cap_entries = entries;
    s->cap_slots = slots;
    return GAPA_CUDA_OK;
}

int pc_eval(gapa_cuda_ctx* ctx, int task, const int32_t* genes_dev, int rows, int cols, double* out_dev,
            cudaStream_t stream) {
    if (!ctx->pc) ctx->pc = new PcScratch();
    PcScratch* s = ctx->pc;
    const int n = ctx->n;
    // groups per pass bounded by a scratch budget (alive + reached + entry_of = 20 B per vertex and group)
    const size_t budget = 24ull << 30;
    const int all_groups = (rows + kBits - 1) / kBits;
    const int max_groups = static_cast<int>(std::max<size_t>(1, budget / (20ull * std::max(n, 1))));
    const int sm = ctx->sm_count;

    for (int g0 = 0; g0 < all_groups; g0 += max_groups) {
        const int groups = std::min(max_groups, all_groups - g0);
        const int row0 = g0 * kBits;
        const int crows = std::min(rows - row0, groups * kBits);
        const size_t words = static_cast<size_t>(groups) * std::max(n, 1);
        GAPA_TRY(s->alive.ensure(sizeof(word_t) * words));
        GAPA_TRY(s->reached.ensure(sizeof(word_t) * words));
        GAPA_TRY(s->entry_of.ensure(sizeof(int32_t) * words));
        GAPA_TRY(s->zeros.ensure(sizeof(int) * groups * kBits));
        GAPA_TRY(s->pc_extra.ensure(sizeof(unsigned long long) * groups * kBits));
        GAPA_TRY(s->mcn_extra.ensure(sizeof(int) * groups * kBits));
        GAPA_TRY(s->flags.ensure(sizeof(int) * 2 * groups));
        GAPA_TRY(s->counters.ensure(sizeof(PcCounters)));
        if (s->cap_entries == 0 || s->parent.cap < sizeof(int32_t) * (static_cast<size_t>(groups) * kBits + s->cap_slots))
            GAPA_TRY(ensure_phase2(s, groups, std::max<size_t>(s->cap_entries, 1u << 16),
                                   std::max<size_t>(s->cap_slots, 1u << 20)));
        word_t* alive = s->alive.as<word_t>();
        word_t* reached = s->reached.as<word_t>();
        int* flags = s->flags.as<int>();
        PcCounters* counters = s->counters.as<PcCounters>();
        const int slot0 = groups * kBits;

        GAPA_LAUNCH(k_pc_reset, std::max(1, (groups * kBits + kThreads - 1) / kThreads), kThreads, 0, stream, groups,
                    s->parent.as<int32_t>(), s->comp_size.as<int32_t>(), s->zeros.as<int>(),
                    s->pc_extra.as<unsigned long long>(), s->mcn_extra.as<int>(), counters, false);
        if (n > 0) {
            GAPA_LAUNCH(k_pc_init, sm * 8, kThreads, 0, stream, alive, reached, n, groups, crows);
            const size_t cells = static_cast<size_t>(crows) * cols;
            if (cells) {
                const int grid = static_cast<int>(std::min<size_t>((cells + kThreads - 1) / kThreads, static_cast<size_t>(sm) * 32));
                GAPA_LAUNCH(k_pc_remove, grid, kThreads, 0, stream, genes_dev + static_cast<size_t>(row0) * cols, cells,
                            cols, ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, n, alive, counters);
            }
            GAPA_LAUNCH(k_pc_source, (crows * 32 + kThreads - 1) / kThreads, kThreads, 0, stream, ctx->d_by_degree, n,
                        crows, alive, reached);

            // phase 1: sweeps in batches; stop as soon as a whole batch-end sweep changed nothing.
            const dim3 grid((n + kThreads - 1) / kThreads, groups);
            const int kBatch = 3, kMaxSweeps = 96;
            int sweep = 0;
            bool converged = false;
            while (!converged && sweep < kMaxSweeps) {
                for (int i = 0; i < kBatch; ++i, ++sweep) {
                    int* out_flags = flags + (sweep & 1) * groups;
                    const int* in_flags = sweep == 0 ? nullptr : flags + ((sweep - 1) & 1) * groups;
                    GAPA_CUDA_TRY(cudaMemsetAsync(out_flags, 0, sizeof(int) * groups, stream));
                    GAPA_LAUNCH(k_pc_sweep, grid, kThreads, 0, stream, ctx->d_row_ptr, ctx->d_col_idx, n, alive, reached,
                                in_flags, out_flags);
                }
                // any group still changing?  (tiny D2H; the stream is idle-waited once per batch)
                std::vector<int> h(groups);
                GAPA_CUDA_TRY(cudaMemcpyAsync(h.data(), flags + ((sweep - 1) & 1) * groups, sizeof(int) * groups,
                                              cudaMemcpyDeviceToHost, stream));
                GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
                converged = std::all_of(h.begin(), h.end(), [](int x) { return x == 0; });
            }
            s->sweeps_last = sweep;

            // finalize + phase 2, re-run with larger tables if the leftover lists overflowed
            for (;;) {
                const int fgrid = std::max(1, std::min((n + kThreads - 1) / kThreads, sm * 4));
                GAPA_LAUNCH(k_pc_finalize, dim3(fgrid, groups), kThreads, 0, stream, ctx->d_row_ptr, ctx->d_col_idx, n,
                            crows, alive, reached, s->zeros.as<int>(), s->entry_of.as<int32_t>(), s->left_v.as<int32_t>(),
                            s->left_g.as<int32_t>(), s->left_w.as<word_t>(), s->left_base.as<int32_t>(),
                            s->parent.as<int32_t>(), s->comp_size.as<int32_t>(), static_cast<unsigned>(s->cap_entries),
                            static_cast<unsigned>(s->cap_slots), slot0, counters);
                PcCounters h;
                GAPA_CUDA_TRY(cudaMemcpyAsync(&h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
                GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
                if (h.range_error) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
                if (h.overflow) {
                    GAPA_TRY(ensure_phase2(s, groups, static_cast<size_t>(h.n_entries) + 1024, static_cast<size_t>(h.n_slots) + 1024));
                    GAPA_LAUNCH(k_pc_reset, std::max(1, (groups * kBits + kThreads - 1) / kThreads), kThreads, 0, stream,
                                groups, s->parent.as<int32_t>(), s->comp_size.as<int32_t>(), s->zeros.as<int>(),
                                s->pc_extra.as<unsigned long long>(), s->mcn_extra.as<int>(), counters, true);
                    continue;
                }
                if (h.n_entries) {
                    const int pgrid = static_cast<int>(std::min<unsigned>((h.n_entries + kThreads - 1) / kThreads, sm * 8));
                    GAPA_LAUNCH(k_pc_hook, pgrid, kThreads, 0, stream, ctx->d_row_ptr, ctx->d_col_idx, n, alive, reached,
                                s->entry_of.as<int32_t>(), s->left_v.as<int32_t>(), s->left_g.as<int32_t>(),
                                s->left_w.as<word_t>(), s->left_base.as<int32_t>(), s->parent.as<int32_t>(), slot0, counters);
                    GAPA_LAUNCH(k_pc_count, pgrid, kThreads, 0, stream, s->left_w.as<word_t>(), s->left_base.as<int32_t>(),
                                s->parent.as<int32_t>(), s->comp_size.as<int32_t>(), slot0, counters);
                    GAPA_LAUNCH(k_pc_reduce, pgrid, kThreads, 0, stream, s->left_g.as<int32_t>(), s->left_w.as<word_t>(),
                                s->left_base.as<int32_t>(), s->parent.as<int32_t>(), s->comp_size.as<int32_t>(), slot0,
                                s->pc_extra.as<unsigned long long>(), s->mcn_extra.as<int>(), counters);
                }
                break;
            }
        } else if (static_cast<size_t>(crows) * cols) {
            return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
        }
        GAPA_LAUNCH(k_pc_result, (crows + kThreads - 1) / kThreads, kThreads, 0, stream, n, crows, task, s->zeros.as<int>(),
                    s->comp_size.as<int32_t>(), s->pc_extra.as<unsigned long long>(), s->mcn_extra.as<int>(),
                    out_dev + row0);
    }
    return GAPA_CUDA_OK;
}

void pc_free(gapa_cuda_ctx* ctx) {
    if (!ctx->pc) return;
    PcScratch* s = ctx->pc;
    for (DevBuf* b : {&s->alive, &s->reached, &s->entry_of, &s->zeros, &s->flags, &s->counters, &s->left_v, &s->left_g,
                      &s->left_w, &s->left_base, &s->parent, &s->comp_size, &s->pc_extra, &s->mcn_extra})
        b->release();
    delete s;
    ctx->pc = nullptr;
}

}  // namespace gapa_b200
