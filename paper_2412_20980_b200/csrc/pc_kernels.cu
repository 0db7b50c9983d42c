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
//   * mask build without global atomics: one CTA per individual sets its removed
//     vertices in a SHARED-MEMORY bitmap (k_pc_bitmask), then a register-level
//     64x64 bit transpose turns 64 per-individual bitmaps into per-vertex words
//     (k_pc_transpose).  The bitmap popcount is the number of distinct removed
//     vertices, so no per-bit counting pass over the words is ever needed.
//   * phase 1 closes reachability from one high-degree source per individual with
//     asynchronous bottom-up sweeps: a vertex ORs its neighbours' reached words
//     until every individual it is alive in is covered.  Rows are ascending, so on
//     power-law graphs the oldest / highest-degree neighbours come first and the loop
//     exits after ~2 neighbours — PROVIDED the low-id core is already closed when the
//     rest is swept.  k_pc_prefix therefore converges a prefix of the vertex order
//     inside one CTA per group (in-kernel iteration, no host round trip), and the
//     full sweeps then run over blocks in ascending vertex order with a few groups
//     interleaved so the in-flight window per group stays small.
//   * phase 2 finishes exactly, whatever phase 1 left: the last sweep compacts the
//     alive-but-unreached vertices that have an alive neighbour to (vertex, bits)
//     entries, resolved by a lock-free union-find over compact slots, with one
//     virtual "giant" node per individual standing for everything phase 1 reached
//     (leftovers adjacent to a reached vertex are attached to it, so correctness
//     never depends on phase 1 having converged).  Isolated leftovers are singletons.
// Integer arithmetic end to end; PC fits int64 and is exact in the returned
// double for n <= 9.4e7 (PC < 2^53).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "internal.cuh"
#include "variation.cuh"

namespace cg = cooperative_groups;

namespace gapa_b200 {

typedef unsigned long long word_t;
static constexpr int kBits = 64;
static constexpr int kPack = 4;  // groups per 32-byte vertex record
static constexpr int kThreads = 256;
static constexpr int kMaskThreads = 1024;
static constexpr int kTransThreads = 128;
static constexpr int kPrefixThreads = 1024;
static constexpr int kPrefixCluster = 8;  // CTAs per super-group in the prefix kernel (portable cluster size)
static_assert(kThreads == 4 * 64, "the final sweep's histogram has one counter per thread");

struct PcCounters {
    unsigned int n_entries;
    unsigned int n_slots;
    int overflow;
    int range_error;
    int changed;  // any sweep since the last reset set a new reached bit
    unsigned int n_incomplete;  // 256-vertex chunks the recording sweep still has to visit
    int deferred;  // the recording sweep declined to run: too much is still unreached and the sweeps still progress
    unsigned int n_left;  // (vertex, super-group) pairs with unreached individuals after the last ordinary sweep
    int phase2_skipped;   // k_pc_final: more leftover entries than its single CTA takes on (host copy only)
    int max_source;       // highest vertex id any individual's BFS source was marked at (-1 after a reset): see SweepArgs::fresh_from
};

// Scratch of ONE lane in flight (a lane = a contiguous block of whole 64-individual groups that goes through the
// pipeline together).  Lanes that run on the same stream reuse the set, so its buffers stay L2-warm.
struct PcSet {
    DevBuf removed, removed_count, alive, reached, entry_of, unreached, counters, block_done;
    DevBuf left_v, left_g, left_w, left_base, parent, comp_size, pc_extra, mcn_extra;
    size_t cap_entries = 0, cap_slots = 0;
    cudaStream_t stream = nullptr;  // the lane stream (multi-lane evaluations); single-lane ones run on the caller's
    // side stream that clears the `reached` records while the mask build runs (the two do not touch the same memory)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_pass_begin = nullptr, ev_cleared = nullptr, ev_done = nullptr;
    // the accumulators (giant slots, unreached / removed counts, extras, counters) are as a reset leaves them: the last
    // lane on this set ended in k_pc_final, which cleans up after itself
    int clean_slots = 0;  // how many accumulator slots (individuals) are in that state
};

static constexpr int kMaxLanes = 64;
static constexpr unsigned kFusedPhase2Entries = 4096;  // leftover entries k_pc_final's single CTA resolves itself  // lanes per wave (pinned counter slots)

struct PcScratch {
    std::vector<PcSet*> sets;
    PcCounters* h_counters = nullptr;  // pinned, kMaxLanes slots: each lane's counters after its last kernel
    cudaEvent_t ev_fork = nullptr;
    int prefix = 32768, interleave = 16, mask_chunks = 1, small_path = 1, relabel = -1, prefix_first4 = 1, trace = 0, prefix_cluster = 0;
    int lane_rows = 4096, lane_streams = 2;
    // Rounds of sweeps the speculative (host-free) schedule enqueues; learned from the evaluations that needed the
    // host-driven loop.  0 = this graph needs more rounds than it pays to enqueue blindly: always host-driven.
    int spec_rounds = 1;
    bool phase2_big = false;  // the speculative schedule uses the three full-grid phase-2 kernels (learned: k_pc_final declined once)
    size_t fold_clear_bytes = 16u << 20;  // reached records up to this size are cleared by the transpose kernel
    // hub-first internal vertex order for the bit-sliced path (see ensure_order)
    DevBuf ord_row_ptr, ord_col_idx, ord_gene_map;
    DevBuf nbr4;  // int4 per vertex: the first four entries of its (ascending) row, -1 padded — see gather_first4
    bool ord_ready = false, ord_relabeled = false;
    unsigned long long ord_pool_version = ~0ull;
    std::vector<int32_t> perm;  // original vertex -> internal vertex when relabelled
    bool configured = false;
    int overlap_clear = 1;
    // Which algorithm this context's graph gets on the large path: -1 = not decided (the bit-sliced pipeline runs; the first
    // evaluation that needs its host-driven loop times both on that batch), 0 = bit-sliced pipeline, 1 = per-individual
    // union-find (k_pc_uf).  GAPA_PC_UF = 0 / 1 fixes it (tests run every case through both).
    int uf_mode = -1;
    DevBuf uf_scratch, uf_out;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
    int mask_threads_forced = 0;  // GAPA_PC_MASK_THREADS: CTA size of the mask kernels (multiple of 128; 0 = by the genes per row)
    int mask_rows = 1;  // GAPA_PC_MASK_ROWS: persistent pipelined mask kernel for whole bitmaps (0: one CTA per row and chunk)
    int sweep_prefetch = 32;  // GAPA_PC_SWEEP_PREFETCH: chunks ahead (SweepArgs::prefetch_chunks); C4 sweep 0.447 / 0.442 / 0.436 / 0.435 / 0.437 / 0.439 / 0.459 ms at 0 / 8 / 16 / 32 / 64 / 128 / 256 (tools/ab_sweep_prefetch.sh)
    int fresh_skip = 0;  // GAPA_PC_FRESH_SKIP: the first sweep does not load records that are known to be clear (SweepArgs::fresh_from)
    int vary_waves = 1;  // GAPA_PC_VARY_WAVES: CTAs of the fused variation kernel per resident slot (1 = persistent, large = one row per CTA)
};

// ---------------------------------------------------------------------------------
// mask build, step 1: apply_in_place for NodeRemoval (gene_pool.cpp:61-64) into a
// shared-memory bitmap of one individual (one vertex chunk of it when n is large).
// Duplicate genes are idempotent.  Bit c of 64-bit word w = vertex 64 w + c removed.
extern __shared__ __align__(16) unsigned pc_smem_bits[];

// DRAM -> L2 prefetch of a contiguous range by ONE thread (TMA bulk prefetch: no registers, no scoreboard held)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// eight consecutive int32 with one 256-bit streaming load (sm_100: LDG.E.EF.256); p must be 32-byte aligned
__device__ __forceinline__ void load8_stream(const int32_t* p, int (&v)[8]) {
    asm volatile("ld.global.cs.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

template <int nt>  // threads per CTA: 128..kMaskThreads, chosen by the launch from the genes per individual (mask_threads)
__global__ void __launch_bounds__(nt) k_pc_bitmask(GeneRows genes,
                                                             const int32_t* __restrict__ pool_map, int pool_size, int n,
                                                             int chunk_bits, int words_per_row, word_t* __restrict__ removed,
                                                             int* removed_count, PcCounters* counters) {
    griddep_launch();
    griddep_wait();
    const int row = blockIdx.y;  // the chunks of one individual are adjacent blocks: its genes are re-read from L2
    const int v0 = blockIdx.x * chunk_bits;
    const int v1 = min(n, v0 + chunk_bits);
    const int words64 = (v1 - v0 + 63) >> 6;
    for (int w = threadIdx.x; w < 2 * words64; w += nt) pc_smem_bits[w] = 0u;
    __syncthreads();
    const int cols = genes.cols;
    const int32_t* g = genes.row(row);
    auto mark = [&](int gene) {
        if (gene < 0 || gene >= pool_size) {
            counters->range_error = 1;
            return;
        }
        const int node = pool_map ? pool_map[gene] : gene;
        if (node >= v0 && node < v1) atomicOr(&pc_smem_bits[(node - v0) >> 5], 1u << ((node - v0) & 31));
    };
    int j0 = 0;
    if ((reinterpret_cast<uintptr_t>(g) & 31) == 0) {
        // 32-byte streaming loads (LDG.E.256), two per thread — 64 KB per SM — in flight before the first
        // shared-memory atomic: with one CTA per SM the kernel lives on bytes in flight per thread
        const int octs = cols >> 3;
        int o = threadIdx.x;
        for (; o + nt < octs; o += 2 * nt) {
            int a[8], b[8];
            load8_stream(g + 8 * static_cast<size_t>(o), a);
            load8_stream(g + 8 * static_cast<size_t>(o + nt), b);
#pragma unroll
            for (int t = 0; t < 8; ++t) mark(a[t]);
#pragma unroll
            for (int t = 0; t < 8; ++t) mark(b[t]);
        }
        if (o < octs) {
            int a[8];
            load8_stream(g + 8 * static_cast<size_t>(o), a);
#pragma unroll
            for (int t = 0; t < 8; ++t) mark(a[t]);
        }
        j0 = octs << 3;
    } else if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
        // 16-byte loads, two per thread in flight before the first shared-memory atomic
        const int4* g4 = reinterpret_cast<const int4*>(g);
        const int quads = cols >> 2;
        int q = threadIdx.x;
        for (; q + nt < quads; q += 2 * nt) {
            const int4 a = __ldcs(&g4[q]);
            const int4 b = __ldcs(&g4[q + nt]);
            mark(a.x); mark(a.y); mark(a.z); mark(a.w);
            mark(b.x); mark(b.y); mark(b.z); mark(b.w);
        }
        if (q < quads) {
            const int4 a = __ldcs(&g4[q]);
            mark(a.x); mark(a.y); mark(a.z); mark(a.w);
        }
        j0 = quads << 2;
    }
    for (int j = j0 + threadIdx.x; j < cols; j += nt) mark(g[j]);
    __syncthreads();
    const word_t* bits64 = reinterpret_cast<const word_t*>(pc_smem_bits);
    word_t* out = removed + static_cast<size_t>(row) * words_per_row + (v0 >> 6);
    int distinct = 0;
    for (int w = threadIdx.x; w < words64; w += nt) {
        const word_t x = bits64[w];
        distinct += __popcll(x);
        out[w] = x;
    }
    for (int off = 16; off; off >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, off);
    if ((threadIdx.x & 31) == 0 && distinct) atomicAdd(&removed_count[row], distinct);
}

// The same mask build for whole bitmaps (chunks == 1), PERSISTENT and pipelined over the rows a CTA owns (round 2).  With one
// CTA per SM (125 KB bitmap) nothing covered a CTA's zeroing, its first loads and its bitmap write-out: ~4 of the ~12 us a row
// took at C4, with the loads that bound the kernel (64 KB in flight per SM) not running.  Here every thread keeps two 32-byte
// gene loads in flight across row boundaries — the next row's first two passes are requested before the epilogue barrier —,
// the write-out clears the bitmap in the same pass, and a last partial pass is done gene-wise by eight times as many threads.
#ifndef GAPA_MASK_MAXREG
#define GAPA_MASK_MAXREG 0
#endif
#if GAPA_MASK_MAXREG > 0
#define GAPA_MASK_BOUNDS __maxnreg__(GAPA_MASK_MAXREG)
#else
#define GAPA_MASK_BOUNDS __launch_bounds__(nt)
#endif
template <int nt>
__global__ void GAPA_MASK_BOUNDS k_pc_bitmask_rows(GeneRows genes, const int32_t* __restrict__ pool_map, int pool_size, int n,
                                                                  int words_per_row, word_t* __restrict__ removed, int* removed_count,
                                                                  PcCounters* counters, int rows) {
    griddep_launch();
    griddep_wait();
    const int tid = threadIdx.x;
    const int words64 = (n + 63) >> 6;
    word_t* bits64 = reinterpret_cast<word_t*>(pc_smem_bits);
    const int cols = genes.cols;
    auto mark = [&](int gene) {
        if (gene < 0 || gene >= pool_size) {
            counters->range_error = 1;
            return;
        }
        const int node = pool_map ? pool_map[gene] : gene;
        atomicOr(&pc_smem_bits[node >> 5], 1u << (node & 31));
    };
    int local = blockIdx.x;
    if (local >= rows) return;
    const int32_t* g = genes.row(local);
    // octs [0, oct_end) are marked eight genes per thread and pass (the last pass may be partial), genes from 8 oct_end on
    // one per thread: a partial pass that would occupy at most an eighth of the threads is done gene-wise instead
    const int octs = cols >> 3, left = octs % nt;
    const int oct_end_aligned = left * 8 > nt ? octs : octs - left;
    auto oct_end_of = [&](const int32_t* row) { return (reinterpret_cast<uintptr_t>(row) & 31) == 0 ? oct_end_aligned : 0; };
    int oct_end = oct_end_of(g);
    int a[8], b[8];
    if (tid < oct_end) load8_stream(g + 8 * static_cast<size_t>(tid), a);
    if (tid + nt < oct_end) load8_stream(g + 8 * static_cast<size_t>(tid + nt), b);
    for (int w = tid; w < words64; w += nt) bits64[w] = 0ull;
    __syncthreads();
    for (;;) {
        const int next = local + static_cast<int>(gridDim.x);
        const bool has_next = next < rows;
        const int32_t* gn = has_next ? genes.row(next) : g;
        for (int o = tid; o < oct_end; o += 2 * nt) {
            int t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = a[i];
            if (o + 2 * nt < oct_end) load8_stream(g + 8 * static_cast<size_t>(o + 2 * nt), a);
#pragma unroll
            for (int i = 0; i < 8; ++i) mark(t[i]);
            if (o + nt < oct_end) {
#pragma unroll
                for (int i = 0; i < 8; ++i) t[i] = b[i];
                if (o + 3 * nt < oct_end) load8_stream(g + 8 * static_cast<size_t>(o + 3 * nt), b);
#pragma unroll
                for (int i = 0; i < 8; ++i) mark(t[i]);
            }
        }
        const int oct_end_next = has_next ? oct_end_of(gn) : 0;  // the next row's first two passes travel under this row's epilogue
        if (tid < oct_end_next) load8_stream(gn + 8 * static_cast<size_t>(tid), a);
        if (tid + nt < oct_end_next) load8_stream(gn + 8 * static_cast<size_t>(tid + nt), b);
        for (int j = oct_end * 8 + tid; j < cols; j += nt) mark(g[j]);
        __syncthreads();  // every mark of this row is in the bitmap
        word_t* out = removed + static_cast<size_t>(local) * words_per_row;
        int distinct = 0;
        for (int w = tid; w < words64; w += nt) {
            const word_t x = bits64[w];
            distinct += __popcll(x);
            out[w] = x;
            bits64[w] = 0ull;
        }
        for (int off = 16; off; off >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, off);
        if ((tid & 31) == 0 && distinct) atomicAdd(&removed_count[local], distinct);
        if (!has_next) break;
        __syncthreads();  // the bitmap is clear everywhere
        local = next;
        g = gn;
        oct_end = oct_end_next;
    }
}

// Fused variation + mask build for the generation loop: a CTA BUILDS child rows
// `V.row_first + local` (crossover + mutate, or eda + mutate — variation.cuh), stores each gene
// to the child's slot and sets it in the shared-memory bitmap in the same pass.  The hash arithmetic
// of the variation (integer pipes) and the shared-memory atomics of the mask build (LSU) overlap
// inside one kernel, and the 4 k bytes of the child row are never read back from HBM.
//
// Round 2: PERSISTENT and software-pipelined over the rows a CTA owns (local = blockIdx.x, + gridDim.x, ...).  With a
// 125 KB bitmap only one CTA fits an SM, so nothing used to cover a CTA's prologue (three dependent slot-table loads,
// zeroing the bitmap, the first parent loads) or its epilogue (bitmap write-out): ~5 of every 33 us at C4 with the
// integer pipes idle.  Now (a) the slot tables, stream keys and first parent quads of the NEXT row are fetched under the
// current row's hashing, (b) the write-out of a finished bitmap zeroes it in the same pass, (c) the first quad of the
// next row is hashed between the two barriers of the epilogue — odd warps write out first and hash second, even warps the
// other way round, so the LSU-bound write-out and the ALU-bound hashing overlap —, and (d) a last partial pass over
// the quads that would occupy at most a quarter of the threads is done gene-wise by four times as many threads
// (C4: 12,500 quads = 12 full passes of 1024 + 212 quads -> one pass of 848 single genes instead of a thirteenth pass).
// Diagnostics for A/B timing only (results are WRONG with any bit set): 1 = no parent loads, 2 = no bitmap marks,
// 4 = no child stores, 8 = no hashing.  tools/ab_vary_diag.sh
#ifndef GAPA_VARY_DIAG
#define GAPA_VARY_DIAG 0
#endif
__device__ __forceinline__ int4 vary_ld(const int4* p, int q) {
#if GAPA_VARY_DIAG & 1
    return make_int4(4 * q, 4 * q + 1, 4 * q + 2, 4 * q + 3);
#else
    return __ldcs(p + q);
#endif
}
// L2 prefetch distance of the parent rows, in passes of nt quads (0 = off).  One CTA per SM keeps only 32 KB of parent
// loads in flight in registers (two 16-byte loads per thread): 4.7 MB over the chip, ~3.6 TB/s at the latency of a
// loaded HBM (measured: the kernel WITHOUT hashing, marks and stores still took 0.59 ms).  A bulk L2 prefetch by one thread
// per pass holds no registers and no scoreboard: DRAM -> L2 runs GAPA_VARY_PREFETCH passes ahead, the register loads hit L2.
// Measured (tools/ab_vary_prefetch.sh, C4): the loads-only kernel 0.571 -> 0.490 ms at distance 3, but the complete kernel
// does not move (0.824 / 0.838 / 0.826 / 0.830 ms at distance 0 / 1 / 2 / 3; 0.905 at 4): with the hashing in place the
// loads are already covered and the kernel is bound by the integer pipes.  Off by default.
#ifndef GAPA_VARY_PREFETCH
#define GAPA_VARY_PREFETCH 0
#endif
struct VaryRow {
    const int32_t* mine;
    const int32_t* theirs;
    int32_t* keep_mine;
    int32_t* keep_theirs;
    int32_t* dst;
    bool adopt_mine, adopt_theirs;
};
template <bool kPeer>
__device__ __forceinline__ VaryRow vary_row(const VariationSpec& V, int k, int row, bool eda) {
    VaryRow r;
    const int slot_mine = V.parent[row], slot_theirs = eda ? slot_mine : V.parent[V.partner[row]];
    r.adopt_mine = r.adopt_theirs = false;  // the row lives in another rank's HBM: read it there, keep a copy here
    r.mine = kPeer ? parent_row(V, slot_mine, k, &r.adopt_mine) : V.pool + static_cast<size_t>(slot_mine) * k;
    r.theirs = eda ? r.mine : (kPeer ? parent_row(V, slot_theirs, k, &r.adopt_theirs) : V.pool + static_cast<size_t>(slot_theirs) * k);
    if (eda || slot_theirs == slot_mine) r.adopt_theirs = false;
    r.keep_mine = V.pool + static_cast<size_t>(slot_mine) * k;
    r.keep_theirs = V.pool + static_cast<size_t>(slot_theirs) * k;
    r.dst = V.pool + static_cast<size_t>(V.child[row]) * k;
    return r;
}

// Resident CTAs the compiler must leave room for (it caps the registers accordingly).  The kernel wants 64 registers; with
// CTAs of 640 threads that is ONE CTA per SM (41 K of the 64 K registers), with 48 registers it is two: n = 1e5 (k = 5000,
// 640 threads) 0.157 -> 0.124 ms, generation 0.390 -> 0.355 ms (tools/ab_vary_regs.sh).  The full-size CTA (1024 threads,
// 125 KB bitmap: one per SM whatever the registers) keeps its 64: capped at 56 or 48 it is 0.824 -> 0.882 / 0.885 ms.
#ifndef GAPA_VARY_MAXREG
#define GAPA_VARY_MAXREG 0
#endif
constexpr int vary_min_blocks(int nt) {
    return nt >= 768 ? 1 : (65536 / (nt * 48) < 2048 / nt ? 65536 / (nt * 48) : 2048 / nt);
}
#if GAPA_VARY_MAXREG > 0
#define GAPA_VARY_BOUNDS __maxnreg__(GAPA_VARY_MAXREG)
#else
#define GAPA_VARY_BOUNDS __launch_bounds__(nt, vary_min_blocks(nt))
#endif
template <int nt, bool kPeer>  // kPeer: parent rows may live in another rank's HBM (variation.cuh: parent_row)
__global__ void GAPA_VARY_BOUNDS k_pc_bitmask_vary(VariationSpec V, int k, const int32_t* __restrict__ gene_map,
                                                                  int n, int words_per_row, word_t* __restrict__ removed,
                                                                  int* removed_count, int rows) {
    griddep_launch();
    griddep_wait();
    __shared__ uint64_t keys[4];
    const int tid = threadIdx.x;
    const int words64 = (n + 63) >> 6;
    word_t* bits64 = reinterpret_cast<word_t*>(pc_smem_bits);
    const bool eda = V.partner == nullptr;
    // quads [0, quad_end) are hashed four genes per thread and pass, genes [4 quad_end, k) one per thread and pass
    const int quads = (k & 3) == 0 ? k >> 2 : 0;
    const int tail_quads = quads % nt;
    const int quad_end = tail_quads * 4 > nt ? quads : quads - tail_quads;
    const int tail0 = 4 * quad_end;
    // No range check here (one compare per gene costs this kernel 5 %): a mutated gene is inside the pool by construction
    // and an inherited one is as good as the parents — which this library's own operators wrote, or which
    // gapa_cuda_ga_slots_variation_eval_device validated when it first saw the caller's pool (ctx.cu).
    auto mark = [&](int gene) {
#if GAPA_VARY_DIAG & 2
        if (gene == -12345) pc_smem_bits[0] = 1;
        return;
#endif
        const int node = gene_map ? gene_map[gene] : gene;
        atomicOr(&pc_smem_bits[node >> 5], 1u << (node & 31));
    };
    int local = blockIdx.x;
    if (local >= rows) return;
    // pass j of a row (thread 0): request the bytes that pass j + D will load — of this row, or of the next row's beginning
    constexpr int kChunkGenes = 4 * nt;
    const int chunks = quad_end > 0 ? (k + kChunkGenes - 1) / kChunkGenes : 0;
    const bool use_prefetch = GAPA_VARY_PREFETCH > 0 && chunks >= GAPA_VARY_PREFETCH + 2;
    auto prefetch_row = [&](const VaryRow& row, int chunk) {
        const int g0 = chunk * kChunkGenes;
        const uint32_t bytes = 4u * static_cast<uint32_t>(min(kChunkGenes, k - g0));
        if (!(kPeer && row.adopt_mine)) prefetch_l2_bulk(row.mine + g0, bytes);
        if (!eda && row.theirs != row.mine && !(kPeer && row.adopt_theirs)) prefetch_l2_bulk(row.theirs + g0, bytes);
    };
    auto prefetch_step = [&](const VaryRow& cur, const VaryRow* nxt, int j) {
        if (!use_prefetch || tid != 0) return;
        const int t = j + GAPA_VARY_PREFETCH;
        if (t < chunks) prefetch_row(cur, t);
        else if (nxt && t - chunks < chunks) prefetch_row(*nxt, t - chunks);
    };
    VaryRow R = vary_row<kPeer>(V, k, V.row_first + local, eda);
    if (use_prefetch && tid == 0)
        for (int c = 1; c < GAPA_VARY_PREFETCH; ++c) prefetch_row(R, c);
    int4 a_next = make_int4(0, 0, 0, 0), b_next = a_next;
    if (tid < quad_end) {
        a_next = vary_ld(reinterpret_cast<const int4*>(R.mine), tid);
        b_next = eda ? a_next : vary_ld(reinterpret_cast<const int4*>(R.theirs), tid);
    }
    for (int w = tid; w < words64; w += nt) bits64[w] = 0ull;
    if (tid < 4) keys[tid] = stream_key(V.P.seed, V.P.generation, GAPA_ROLE_SELECT + tid, static_cast<uint64_t>(V.row_first + local)) + kGolden;
    __syncthreads();
    uint64_t ks = keys[0], kc = keys[1], km = keys[2], ki = keys[3];
    __syncthreads();  // (once per CTA) nobody rewrites the keys before everybody has read them
    int r0[4] = {0, 0, 0, 0};  // child genes of the row's first quad of this thread: hashed and stored, not yet marked
    // first quad of a row: hash + store (the marks wait until the bitmap is known to be clear)
    auto first_quad = [&](const VaryRow& row) {
        prefetch_step(row, nullptr, 0);
        if (tid < quad_end) {
            const int4 a = a_next, b = b_next;
            if (kPeer && row.adopt_mine) reinterpret_cast<int4*>(row.keep_mine)[tid] = a;
            if (kPeer && row.adopt_theirs) reinterpret_cast<int4*>(row.keep_theirs)[tid] = b;
            const int av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                r0[t] = child_gene(V.P, V.pool, V.parent, k, 4 * tid + t, av[t], bv[t], eda, ks, kc, km, ki, 4u * tid + t + 1u);
            reinterpret_cast<int4*>(row.dst)[tid] = make_int4(r0[0], r0[1], r0[2], r0[3]);
        }
    };
    first_quad(R);
    for (;;) {
        const int next = local + static_cast<int>(gridDim.x);
        const bool has_next = next < rows;
        VaryRow N = R;
        if (has_next) N = vary_row<kPeer>(V, k, V.row_first + next, eda);  // three dependent loads, hidden under this row's hashing
        if (tid < quad_end) {
#pragma unroll
            for (int t = 0; t < 4; ++t) mark(r0[t]);
        }
        // gene-wise tail: its parents are requested now and used after the quad passes
        int ta = 0, tb = 0;
        const int tj = tail0 + tid;
        if (tj < k) {
            ta = R.mine[tj];
            tb = eda ? ta : R.theirs[tj];
        }
        int pass = 0;  // passes of this row done so far (thread 0 counts them for the prefetch; its q always runs to quad_end)
        {
            const int4* mine4 = reinterpret_cast<const int4*>(R.mine);
            const int4* theirs4 = reinterpret_cast<const int4*>(R.theirs);
            int4* dst4 = reinterpret_cast<int4*>(R.dst);
            int q = tid + nt;
            if (q < quad_end) {
                a_next = vary_ld(mine4, q);
                b_next = eda ? a_next : vary_ld(theirs4, q);
            }
            for (; q < quad_end; q += nt) {
                prefetch_step(R, has_next ? &N : nullptr, ++pass);
                const int4 a = a_next, b = b_next;
                if (q + nt < quad_end) {  // next quad's parents are in flight while this one is hashed
                    a_next = vary_ld(mine4, q + nt);
                    b_next = eda ? a_next : vary_ld(theirs4, q + nt);
                }
                if (kPeer && R.adopt_mine) reinterpret_cast<int4*>(R.keep_mine)[q] = a;
                if (kPeer && R.adopt_theirs) reinterpret_cast<int4*>(R.keep_theirs)[q] = b;
                const int av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
                int r[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
#if GAPA_VARY_DIAG & 8
                    r[t] = (av[t] ^ bv[t]) % 1000000;
#else
                    r[t] = child_gene(V.P, V.pool, V.parent, k, 4 * q + t, av[t], bv[t], eda, ks, kc, km, ki, 4u * q + t + 1u);
#endif
                }
#if GAPA_VARY_DIAG & 4
                if (r[0] == -12345)
#endif
                dst4[q] = make_int4(r[0], r[1], r[2], r[3]);
#pragma unroll
                for (int t = 0; t < 4; ++t) mark(r[t]);
            }
        }
        while (++pass < chunks) prefetch_step(R, has_next ? &N : nullptr, pass);
        for (int j = tj; j < k; j += nt) {
            if (j != tj) {
                ta = R.mine[j];
                tb = eda ? ta : R.theirs[j];
            }
            if (kPeer && R.adopt_mine) R.keep_mine[j] = ta;
            if (kPeer && R.adopt_theirs) R.keep_theirs[j] = tb;
            const int gsel = child_gene(V.P, V.pool, V.parent, k, j, ta, tb, eda, ks, kc, km, ki, static_cast<uint32_t>(j) + 1u);
            R.dst[j] = gsel;
            mark(gsel);
        }
        // the next row's first quads are requested before the barrier and hashed between the barriers
        if (has_next && tid < quad_end) {
            a_next = vary_ld(reinterpret_cast<const int4*>(N.mine), tid);
            b_next = eda ? a_next : vary_ld(reinterpret_cast<const int4*>(N.theirs), tid);
        }
        if (has_next && tid < 4)  // everybody has read the current keys (before the previous barrier)
            keys[tid] = stream_key(V.P.seed, V.P.generation, GAPA_ROLE_SELECT + tid, static_cast<uint64_t>(V.row_first + next)) + kGolden;
        __syncthreads();  // every mark of this row is in the bitmap; the next row's keys are visible
        if (has_next) ks = keys[0], kc = keys[1], km = keys[2], ki = keys[3];
        word_t* out = removed + static_cast<size_t>(local) * words_per_row;
        int distinct = 0;
        auto write_out = [&]() {  // write the bitmap, count it, clear it for the next row
            for (int w = tid; w < words64; w += nt) {
                const word_t x = bits64[w];
                distinct += __popcll(x);
                out[w] = x;
                bits64[w] = 0ull;
            }
        };
        if ((tid >> 5) & 1) {
            write_out();
            if (has_next) first_quad(N);
        } else {
            if (has_next) first_quad(N);
            write_out();
        }
        for (int off = 16; off; off >>= 1) distinct += __shfl_down_sync(0xffffffffu, distinct, off);
        if ((tid & 31) == 0 && distinct) atomicAdd(&removed_count[local], distinct);
        if (!has_next) break;
        __syncthreads();  // the bitmap is clear everywhere
        local = next;
        R = N;
    }
}

// mask build, step 2: 64 individuals x 64 vertices bit transpose in registers.
// a[i] bit c (individual i, vertex c)  ->  a[c] bit i; alive = ~removed.  Rows past
// the end of the batch read as "everything removed", which zeroes their bits.
//
// `alive` is only ever read at a thread's own vertex (coalesced), so it stays group-major:
// alive[g][v].  `reached` is what the sweeps read at RANDOM neighbours, so kPack = 4 groups
// (256 individuals) are stored side by side, one 32-byte record per vertex — word gi of
// record (sg, v) belongs to group 4 sg + gi.  32 bytes is exactly one memory sector: a
// neighbour read fetches 256 individuals of state per sector instead of 64.
__global__ void __launch_bounds__(kTransThreads) k_pc_transpose(const word_t* __restrict__ removed, int words_per_row,
                                                                int n, int rows, word_t* __restrict__ alive,
                                                                word_t* __restrict__ clear_reached) {
    griddep_launch();
    griddep_wait();
    word_t* tile = reinterpret_cast<word_t*>(pc_smem_bits);  // kBits x (kTransThreads + 1) words, padded against bank conflicts
    const int g = blockIdx.y;
    const int vb0 = blockIdx.x * kTransThreads;
    const int vb = vb0 + threadIdx.x;
    word_t a[kBits];
    if (vb < words_per_row) {
#pragma unroll
        for (int i = 0; i < kBits; ++i) {
            const int row = g * kBits + i;
            a[i] = row < rows ? removed[static_cast<size_t>(row) * words_per_row + vb] : ~0ull;
        }
        word_t m = 0x00000000FFFFFFFFull;
#pragma unroll
        for (int j = 32; j != 0; j >>= 1) {
#pragma unroll
            for (int k = 0; k < kBits; k = (k + j + 1) & ~j) {
                const word_t t = ((a[k] >> j) ^ a[k + j]) & m;
                a[k] ^= t << j;
                a[k + j] ^= t;
            }
            m ^= m << (j >> 1);
        }
#pragma unroll
        for (int c = 0; c < kBits; ++c) tile[c * (kTransThreads + 1) + threadIdx.x] = ~a[c];
    }
    __syncthreads();
    // coalesced write-out: the block's tile is kTransThreads * 64 consecutive vertices
    word_t* out = alive + static_cast<size_t>(g) * n;
    const int v_base = vb0 * kBits;
    for (int idx = threadIdx.x; idx < kTransThreads * kBits; idx += kTransThreads) {
        const int v = v_base + idx;
        if (v < n) {
            out[v] = tile[(idx & 63) * (kTransThreads + 1) + (idx >> 6)];
            // small batches: this group's word of the vertex's reached record is cleared here instead of by a launch of its own
            if (clear_reached) clear_reached[(static_cast<size_t>(g / kPack) * n + v) * kPack + (g % kPack)] = 0ull;
        }
    }
}

__device__ __forceinline__ size_t word_index(int g, int n, int v) {
    return (static_cast<size_t>(g / kPack) * n + v) * kPack + (g % kPack);
}

// One warp per individual: the first alive vertex in descending-degree order
// becomes the BFS source.  Any alive vertex would be correct; a hub makes
// phase 1 cover the giant component.
__global__ void __launch_bounds__(kThreads) k_pc_source(const int32_t* __restrict__ by_degree, int n, int rows,
                                                        const word_t* __restrict__ alive, word_t* reached, PcCounters* counters) {
    griddep_launch();
    griddep_wait();
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int g = row >> 6;
    const word_t bit = 1ull << (row & 63);
    for (int i = 0; i < n; i += 32) {
        const int v = i + lane < n ? (by_degree ? by_degree[i + lane] : i + lane) : -1;
        const bool ok = v >= 0 && (alive[static_cast<size_t>(g) * n + v] & bit);
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        if (hit) {
            if (lane == __ffs(hit) - 1) {
                atomicOr(&reached[word_index(g, n, v)], bit);
                if (v > counters->max_source) atomicMax(&counters->max_source, v);
            }
            return;
        }
    }
}

// ---------------------------------------------------------------------------------
// phase 1.  Reads of neighbours' records race benignly with writes (words only gain
// bits; every 64-bit word is written by single stores), so a sweep can use bits set
// earlier in the same sweep.  `limit` truncates the scan to neighbours below it (rows
// are ascending), which is what keeps hub rows short while only a prefix is active.
struct __align__(32) Rec {
    word_t w[kPack];
};
// One 256-bit access per record (LDG.E.256 / STG.E.256, new on sm_100): a warp gathering 32 random records
// sends 32 requests to the crossbar instead of 64 — the L1 -> XBAR request path was the busiest unit of the
// sweep (65 %) with two 16-byte loads per sector.  L2-coherent (other blocks set bits concurrently).
__device__ __forceinline__ Rec load_rec(const Rec* p) {
    Rec r;
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3]) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void store_rec(Rec* p, const Rec& r) {
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(r.w[0]), "l"(r.w[1]), "l"(r.w[2]), "l"(r.w[3]) : "memory");
}
__device__ __forceinline__ bool rec_any(const Rec& r) { return (r.w[0] | r.w[1] | r.w[2] | r.w[3]) != 0ull; }
__device__ __forceinline__ bool rec_covers(const Rec& got, const Rec& todo) {
    return ((todo.w[0] & ~got.w[0]) | (todo.w[1] & ~got.w[1]) | (todo.w[2] & ~got.w[2]) | (todo.w[3] & ~got.w[3])) == 0ull;
}
__device__ __forceinline__ void rec_or(Rec& a, const Rec& b) {
#pragma unroll
    for (int i = 0; i < kPack; ++i) a.w[i] |= b.w[i];
}

__device__ __forceinline__ Rec load_alive(const word_t* __restrict__ alive, int sg, int n, int v) {
    Rec r;
#pragma unroll
    for (int i = 0; i < kPack; ++i) r.w[i] = alive[(static_cast<size_t>(sg) * kPack + i) * n + v];
    return r;
}

// OR of the neighbours' reached records until `todo` is covered; returns got & todo.
// `max_pairs` bounds the scan (hub rows are long); a truncated scan reports `truncated`.
__device__ __forceinline__ Rec gather_reached(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                              const Rec* reached_sg, int v, int limit, const Rec& todo,
                                              int max_pairs = 0x3fffffff, bool* truncated = nullptr) {
    const int beg = row_ptr[v];
    int end = row_ptr[v + 1];
    if (end - beg > 2 * max_pairs) {
        end = beg + 2 * max_pairs;
        if (truncated) *truncated = true;
    }
    Rec got{};
    int e = beg;
    for (; e + 1 < end; e += 2) {  // two neighbours per step: both sectors are in flight together
        const int u0 = col_idx[e], u1 = col_idx[e + 1];
        if (u1 >= limit) {
            if (u0 < limit) rec_or(got, load_rec(&reached_sg[u0]));
            e = end;
            break;
        }
        const Rec r0 = load_rec(&reached_sg[u0]), r1 = load_rec(&reached_sg[u1]);
        rec_or(got, r0);
        rec_or(got, r1);
        if (rec_covers(got, todo)) {
            e = end;
            break;
        }
    }
    if (e < end) {
        const int u = col_idx[e];
        if (u < limit) rec_or(got, load_rec(&reached_sg[u]));
    }
#pragma unroll
    for (int i = 0; i < kPack; ++i) got.w[i] &= todo.w[i];
    return got;
}

// The sweeps' gather with the index chain taken off the critical path.  `first` holds the first four
// neighbours of v (one coalesced 16-byte load issued together with v's own records), so the common
// case — covered by the two or four oldest neighbours — is  {own records, first} -> {neighbour
// records}: two dependent memory latencies instead of row_ptr -> col_idx -> records -> col_idx -> ...
// Only vertices that need more than four neighbours touch row_ptr / col_idx at all.
__device__ __forceinline__ Rec gather_first4(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                             const Rec* reached_sg, int v, const int4 first, const Rec& todo) {
    Rec got{};
    bool done = false;
    if (first.x >= 0) {
        const Rec r0 = load_rec(&reached_sg[first.x]);
        if (first.y >= 0) {
            const Rec r1 = load_rec(&reached_sg[first.y]);
            rec_or(got, r1);
        }
        rec_or(got, r0);
        done = rec_covers(got, todo) || first.z < 0;
        if (!done) {
            const Rec r2 = load_rec(&reached_sg[first.z]);
            if (first.w >= 0) {
                const Rec r3 = load_rec(&reached_sg[first.w]);
                rec_or(got, r3);
            }
            rec_or(got, r2);
            done = rec_covers(got, todo) || first.w < 0;
        }
    } else {
        done = true;  // isolated vertex
    }
    if (!done) {
        const int end = row_ptr[v + 1];
        int e = row_ptr[v] + 4;
        for (; e + 1 < end; e += 2) {
            const int u0 = col_idx[e], u1 = col_idx[e + 1];
            const Rec r0 = load_rec(&reached_sg[u0]), r1 = load_rec(&reached_sg[u1]);
            rec_or(got, r0);
            rec_or(got, r1);
            if (rec_covers(got, todo)) {
                e = end;
                break;
            }
        }
        if (e < end) rec_or(got, load_rec(&reached_sg[col_idx[e]]));
    }
#pragma unroll
    for (int i = 0; i < kPack; ++i) got.w[i] &= todo.w[i];
    return got;
}

// Closes the first `prefix` vertices of every super-group inside one thread-block CLUSTER of
// kPrefixCluster CTAs (8192 threads): iterate ascending passes until nothing changes, with
// cluster-wide barriers between passes — no host round trip, no cooperative launch.  The
// in-flight window is the cluster, so a pass propagates almost like a sequential scan.
__global__ void __launch_bounds__(kPrefixThreads)
    k_pc_prefix(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx, const int4* __restrict__ nbr4,
                int first4_only, int n, int prefix, const word_t* __restrict__ alive, Rec* reached, int pick_sources,
                const int32_t* __restrict__ by_degree, int rows, PcCounters* counters) {
    griddep_launch();
    griddep_wait();
    cg::cluster_group cluster = cg::this_cluster();
    // the cluster size is a launch attribute: kPrefixCluster CTAs while every super-group's cluster is
    // resident at once, fewer when there are more super-groups than that (waves of idle-heavy clusters cost more)
    const int csize = static_cast<int>(cluster.num_blocks());
    const int sg = blockIdx.x / csize;
    const int lane_in_cluster = static_cast<int>(cluster.block_rank()) * kPrefixThreads + threadIdx.x;
    const int kStride = csize * kPrefixThreads;
    Rec* reached_sg = reached + static_cast<size_t>(sg) * n;
    if (pick_sources) {
        // k_pc_source folded in (one launch less): a warp per individual of this super-group marks the first alive
        // vertex in descending-degree order; the cluster barrier publishes the marks before the first pass
        const int warps = kStride >> 5, lane = threadIdx.x & 31;
        for (int r = lane_in_cluster >> 5; r < kPack * kBits; r += warps) {
            const int row = sg * kPack * kBits + r;
            if (row >= rows) break;
            const int g = row >> 6;
            const word_t bit = 1ull << (row & 63);
            for (int i = 0; i < n; i += 32) {
                const int v = i + lane < n ? (by_degree ? by_degree[i + lane] : i + lane) : -1;
                const bool ok = v >= 0 && (alive[static_cast<size_t>(g) * n + v] & bit);
                const unsigned hit = __ballot_sync(0xffffffffu, ok);
                if (hit) {
                    if (lane == __ffs(hit) - 1) {
                        atomicOr(&reinterpret_cast<word_t*>(reached)[word_index(g, n, v)], bit);
                        if (v > counters->max_source) atomicMax(&counters->max_source, v);
                    }
                    break;
                }
            }
        }
        cluster.sync();
    }
    // "did anything change in this pass" is exchanged through DISTRIBUTED SHARED MEMORY: every CTA stores its flag into
    // slot [pass parity][own rank] of every CTA of the cluster, the cluster barrier publishes the stores, and each CTA
    // reads its own copy — no global atomic, fence and L2 read on the critical path of a pass (3 of its ~5 us).
    __shared__ int pass_any[2][kPrefixCluster];
    const int my_rank = static_cast<int>(cluster.block_rank());
    const int stages[2] = {min(prefix, kPrefixCluster * kPrefixThreads / 4), prefix};
    int pass_id = 0;
    for (int s = 0; s < 2; ++s) {
        const int limit = stages[s];
        if (s == 1 && limit == stages[0]) break;
        for (int pass = 0; pass < 24; ++pass) {
            int any = 0;
            for (int v = lane_in_cluster; v < limit; v += kStride) {
                // the four lowest neighbours are requested together with the vertex's own words (one dependent round
                // trip to L2 less for every vertex that still has work)
                int4 f = make_int4(-1, -1, -1, -1);
                if (first4_only) f = __ldg(&nbr4[v]);
                Rec mine = load_rec(&reached_sg[v]);
                const Rec al = load_alive(alive, sg, n, v);
                Rec todo;
#pragma unroll
                for (int i = 0; i < kPack; ++i) todo.w[i] = al.w[i] & ~mine.w[i];
                if (!rec_any(todo)) continue;
                // Bounded scan: in the first passes an unreached hub would otherwise walk hundreds of
                // still-unreached younger neighbours serially.  Exactness does not depend on this
                // kernel (the sweeps and phase 2 finish), only the speed of what follows does.
                bool cut = false;
                Rec got{};
                if (first4_only) {
                    // the four lowest neighbours only: in a hub-first order these are the vertex's links towards
                    // the core, which is where reachability arrives from; whatever this misses (a vertex reached
                    // only through younger neighbours) is left to the full sweeps and phase 2
                    const int u[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (u[t] >= 0 && u[t] < limit) rec_or(got, load_rec(&reached_sg[u[t]]));
#pragma unroll
                    for (int i = 0; i < kPack; ++i) got.w[i] &= todo.w[i];
                } else {
                    got = gather_reached(row_ptr, col_idx, reached_sg, v, limit, todo, 12 + 4 * pass, &cut);
                }
                if (rec_any(got)) {
                    rec_or(mine, got);
                    store_rec(&reached_sg[v], mine);
                    any = 1;
                } else if (cut) {
                    any = 1;
                }
            }
            const int any_cta = __syncthreads_or(any);
            int* slots = pass_any[pass_id & 1];
            if (threadIdx.x < csize) *cluster.map_shared_rank(&slots[my_rank], threadIdx.x) = any_cta;
            cluster.sync();  // release / acquire at cluster scope: the record stores of this pass and the flags
            int any_cluster = 0;
            for (int r = 0; r < csize; ++r) any_cluster |= slots[r];
            // the parity advances on EVERY pass, the last one of a stage included: the next pass (of either stage) must not
            // write the slots that slower threads of other CTAs may still be reading
            ++pass_id;
            if (!any_cluster) break;
        }
    }
}

// Full sweep, one thread per (vertex, super-group); `interleave` super-groups share
// blockIdx.x so that blocks are scheduled in ascending vertex order with a small window per
// group.  FINAL additionally records what is still unreached: per-individual counts and the
// compacted non-isolated leftovers for phase 2.
#ifndef GAPA_SWEEP_MIN_BLOCKS
#define GAPA_SWEEP_MIN_BLOCKS 4
#endif
struct SweepArgs {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    const int4* nbr4;
    int n, sgroups, interleave;
    const word_t* alive;
    Rec* reached;
    int* unreached;
    int32_t *entry_of, *left_v, *left_g;
    word_t* left_w;
    int32_t *left_base, *parent, *comp_size;
    unsigned cap_entries, cap_slots;
    int slot0;
    PcCounters* counters;
    int2* incomplete;  // (super-group, chunk) list written by the ordinary sweep, read by the recording one
    int record;        // ordinary sweep: append incomplete chunks to the list
    unsigned defer_above;  // recording sweep: with more (vertex, super-group) pairs left than this (and progress) sweep again instead
    int descending;        // ordinary sweep: blocks walk the vertex chunks from the highest id down
    // FIRST sweep after the clear of the reached records: a vertex at or above this id (and above every BFS source,
    // counters->max_source) cannot have been reached yet — only the prefix closure (ids below `prefix`), the source
    // marks and a vertex's own sweep thread ever write its record — so its own record is known to be zero and is not
    // loaded: 32 of the ~98 bytes a (vertex, super-group) pair reads.  n = every record is loaded.
    // MEASURED SLOWER and off by default (GAPA_PC_FRESH_SKIP, tools/ab_fresh.sh): C4 sweep 0.445 -> 0.594 ms, n = 1e5
    // 0.038 -> 0.070 ms.  The sequential read of a vertex's own record is what brings it into L2 for the threads that
    // gather it as a NEIGHBOUR shortly afterwards; without it those gathers go to DRAM one random sector at a time.
    int fresh_from;
    // ordinary sweep: thread 0 of a block requests the own-vertex data (reached records, alive words) of the chunk this
    // many chunks AHEAD in block order into L2, so that the first, parallel stage of that block's loads — and the
    // neighbour gathers that land in it — hit L2 instead of DRAM.  0 = off.
    int prefetch_chunks;
};

template <bool FINAL>
__device__ __forceinline__ void sweep_chunk(const SweepArgs& A, int sg, int chunk, int* hist) {
    const int32_t* __restrict__ row_ptr = A.row_ptr;
    const int32_t* __restrict__ col_idx = A.col_idx;
    const word_t* __restrict__ alive = A.alive;
    Rec* reached = A.reached;
    PcCounters* counters = A.counters;
    const int n = A.n, slot0 = A.slot0;
    const unsigned cap_entries = A.cap_entries, cap_slots = A.cap_slots;
    int* unreached = A.unreached;
    int32_t *entry_of = A.entry_of, *left_v = A.left_v, *left_g = A.left_g, *left_base = A.left_base, *parent = A.parent,
            *comp_size = A.comp_size;
    word_t* left_w = A.left_w;
    const int v = chunk * kThreads + threadIdx.x;
    if (FINAL) {
        hist[threadIdx.x] = 0;  // kThreads == kPack * kBits
        __syncthreads();
    }
    int any = 0, any_left = 0;
    if (v < n) {
        const size_t base = static_cast<size_t>(sg) * n;
        const int4 first = __ldg(&A.nbr4[v]);  // in flight together with v's own records
        Rec mine{};
        if (FINAL || v < A.fresh_from || v <= counters->max_source) mine = load_rec(&reached[base + v]);
        const Rec al = load_alive(alive, sg, n, v);
        Rec todo;
#pragma unroll
        for (int i = 0; i < kPack; ++i) todo.w[i] = al.w[i] & ~mine.w[i];
        if (rec_any(todo)) {
            const Rec got = gather_first4(row_ptr, col_idx, reached + base, v, first, todo);
            if (rec_any(got)) {
                rec_or(mine, got);
                store_rec(&reached[base + v], mine);
                any = 1;
            }
            Rec rest;
#pragma unroll
            for (int i = 0; i < kPack; ++i) rest.w[i] = todo.w[i] & ~got.w[i];
            if (!FINAL) any_left = rec_any(rest);
            if (FINAL) {
                if (rec_any(rest)) {
                    any_left = 1;
#pragma unroll
                    for (int i = 0; i < kPack; ++i) {
                        word_t z = rest.w[i];
                        while (z) {
                            const int b = __ffsll(static_cast<long long>(z)) - 1;
                            z &= z - 1;
                            atomicAdd(&hist[i * kBits + b], 1);
                        }
                    }
                    // keep only the individuals in which v has an alive neighbour
                    Rec nb{};
                    for (int e = row_ptr[v]; e < row_ptr[v + 1] && !rec_covers(nb, rest); ++e) rec_or(nb, load_alive(alive, sg, n, col_idx[e]));
#pragma unroll
                    for (int i = 0; i < kPack; ++i) {
                        const word_t w = rest.w[i] & nb.w[i];
                        if (!w) continue;
                        const int g = sg * kPack + i;
                        const int cnt = __popcll(w);
                        const unsigned e = atomicAdd(&counters->n_entries, 1u);
                        const unsigned s = atomicAdd(&counters->n_slots, static_cast<unsigned>(cnt));
                        if (e < cap_entries && s + cnt <= cap_slots) {
                            left_v[e] = v;
                            left_g[e] = g;
                            left_w[e] = w;
                            left_base[e] = static_cast<int32_t>(s);
                            entry_of[(base + v) * kPack + i] = static_cast<int32_t>(e);
                            for (int t = 0; t < cnt; ++t) {
                                parent[slot0 + s + t] = slot0 + static_cast<int32_t>(s) + t;
                                comp_size[slot0 + s + t] = 0;
                            }
                        } else {
                            counters->overflow = 1;
                        }
                    }
                }
            }
        }
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) counters->changed = 1;
    const int left = __syncthreads_count(any_left);
    if (FINAL) {
        if (left && hist[threadIdx.x]) atomicAdd(&unreached[sg * kPack * kBits + threadIdx.x], hist[threadIdx.x]);
    } else if (left && A.record && threadIdx.x == 0) {
        A.incomplete[atomicAdd(&counters->n_incomplete, 1u)] = make_int2(sg, chunk);
        atomicAdd(&counters->n_left, static_cast<unsigned>(left));
    }
}

// ordinary sweep: blocks in ascending vertex order, `interleave` super-groups share blockIdx.x
__global__ void __launch_bounds__(kThreads, GAPA_SWEEP_MIN_BLOCKS) k_pc_sweep(SweepArgs A) {
    griddep_launch();
    griddep_wait();
    const int sg = blockIdx.y * A.interleave + (blockIdx.x % A.interleave);
    if (sg >= A.sgroups) return;
    const int slot = blockIdx.x / A.interleave;
    const int chunks = (A.n + kThreads - 1) / kThreads;
    if (A.prefetch_chunks > 0 && threadIdx.x == 0 && slot + A.prefetch_chunks < chunks) {
        const int ahead = slot + A.prefetch_chunks;
        const int v0 = (A.descending ? chunks - 1 - ahead : ahead) * kThreads;
        const int cnt = min(kThreads, A.n - v0);
        prefetch_l2_bulk(A.reached + static_cast<size_t>(sg) * A.n + v0, static_cast<uint32_t>(cnt) * sizeof(Rec));
#pragma unroll
        for (int i = 0; i < kPack; ++i) {
            const size_t first = (static_cast<size_t>(sg) * kPack + i) * A.n + v0;
            const size_t lo = first & ~size_t{1};  // 16-byte aligned start
            prefetch_l2_bulk(A.alive + lo, static_cast<uint32_t>(((first - lo + cnt + 1) & ~size_t{1}) * sizeof(word_t)));
        }
    }
    sweep_chunk<false>(A, sg, A.descending ? chunks - 1 - slot : slot, nullptr);
}

// Sweep of the EXTRA rounds (one ordered sweep was not enough: no hub core, or a large diameter).  Inside a
// block all 256 vertices are processed at the same time, so along a path of consecutive ids reachability
// advances one hop per sweep; here a block repeats its chunk until nothing in it changes (the threads keep
// their records in registers and only re-gather what is still missing), which lets a chain of any length
// inside a chunk close in one launch.  Rings and grids: 48 rounds -> a few.
__global__ void __launch_bounds__(kThreads, GAPA_SWEEP_MIN_BLOCKS) k_pc_sweep_local(SweepArgs A) {
    griddep_launch();
    griddep_wait();
    const int sg = blockIdx.y * A.interleave + (blockIdx.x % A.interleave);
    if (sg >= A.sgroups) return;
    const int slot = blockIdx.x / A.interleave;
    const int chunk = A.descending ? (A.n + kThreads - 1) / kThreads - 1 - slot : slot;
    const int v = chunk * kThreads + threadIdx.x;
    const bool valid = v < A.n;
    const size_t base = static_cast<size_t>(sg) * A.n;
    int4 first = make_int4(-1, -1, -1, -1);
    Rec mine{}, todo{};
    if (valid) {
        first = __ldg(&A.nbr4[v]);
        mine = load_rec(&A.reached[base + v]);
        const Rec al = load_alive(A.alive, sg, A.n, v);
#pragma unroll
        for (int i = 0; i < kPack; ++i) todo.w[i] = al.w[i] & ~mine.w[i];
    }
    int any = 0;
    for (int it = 0; it < 64; ++it) {
        int gained = 0;
        if (valid && rec_any(todo)) {
            const Rec got = gather_first4(A.row_ptr, A.col_idx, A.reached + base, v, first, todo);
            if (rec_any(got)) {
                rec_or(mine, got);
                store_rec(&A.reached[base + v], mine);
#pragma unroll
                for (int i = 0; i < kPack; ++i) todo.w[i] &= ~got.w[i];
                gained = 1;
                any = 1;
            }
        }
        if (!__syncthreads_or(gained)) break;
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) A.counters->changed = 1;
    const int left = __syncthreads_count(valid && rec_any(todo));
    if (left && A.record && threadIdx.x == 0) {
        A.incomplete[atomicAdd(&A.counters->n_incomplete, 1u)] = make_int2(sg, chunk);
        atomicAdd(&A.counters->n_left, static_cast<unsigned>(left));
    }
}

// recording sweep: a persistent grid walks the list of incomplete chunks
__global__ void __launch_bounds__(kThreads, GAPA_SWEEP_MIN_BLOCKS) k_pc_record(SweepArgs A) {
    griddep_launch();
    griddep_wait();
    __shared__ int hist[kPack * kBits];
    const unsigned total = A.counters->n_incomplete;
    // Recording is for the last few percent: per leftover vertex it costs a shared-memory atomic per unreached
    // individual plus compaction.  On graphs without a hub core one sweep leaves most of the graph unreached
    // (24 ms of recording at n = 1e6, Erdos-Renyi) — more sweeps first, as long as they still make progress.
    if (A.counters->n_left > A.defer_above && A.counters->changed) {
        if (blockIdx.x == 0 && threadIdx.x == 0) A.counters->deferred = 1;
        return;
    }
    for (unsigned i = blockIdx.x; i < total; i += gridDim.x) {
        const int2 item = A.incomplete[i];
        __syncthreads();  // hist of the previous chunk has been flushed
        sweep_chunk<true>(A, item.x, item.y, hist);
    }
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

// The speculative schedule launches phase 2 before the host has looked at the counters: it stands down when the
// recording sweep overflowed its buffers, declined to run, or asks for more sweeps (the host then redoes the lane with
// the host-driven loop).  The host-driven loop passes many = ~0u: it only launches phase 2 once those are settled.
__device__ __forceinline__ bool pc_stand_down(const PcCounters* c, unsigned many) {
    return c->overflow || c->deferred || (c->changed && c->n_entries > many);
}

struct Phase2Args {
    const int32_t* row_ptr;
    const int32_t* col_idx;
    int n;
    const word_t* alive;
    const word_t* reached;
    const int32_t* entry_of;
    const int32_t* left_v;
    const int32_t* left_g;
    const word_t* left_w;
    const int32_t* left_base;
    int32_t* parent;
    int32_t* comp_size;
    int slot0;
    unsigned long long* pc_extra;
    int* mcn_extra;
    const PcCounters* counters;
};

// entries first, first + stride, ... < total
__device__ __forceinline__ void pc_hook_body(const Phase2Args& P, unsigned first, unsigned stride, unsigned total) {
    const int n = P.n, slot0 = P.slot0;
    for (unsigned e = first; e < total; e += stride) {
        const int v = P.left_v[e], g = P.left_g[e], base_v = P.left_base[e];
        const word_t w = P.left_w[e];
        for (int i = P.row_ptr[v]; i < P.row_ptr[v + 1]; ++i) {
            const int u = P.col_idx[i];
            const size_t iu = word_index(g, n, u);
            const word_t common = w & P.alive[static_cast<size_t>(g) * n + u];
            if (!common) continue;
            const word_t ru = P.reached[iu];
            word_t attach = common & ru;  // v was not reached but its neighbour was: v belongs to the giant
            while (attach) {
                const int b = __ffsll(static_cast<long long>(attach)) - 1;
                attach &= attach - 1;
                uf_union(P.parent, slot_of(slot0, base_v, w, b), g * kBits + b);
            }
            word_t rest = common & ~ru;
            if (rest && u < v) {  // leftover-leftover edges are seen from both ends; take one
                const int eu = P.entry_of[iu];
                const word_t wu = P.left_w[eu];
                const int base_u = P.left_base[eu];
                while (rest) {
                    const int b = __ffsll(static_cast<long long>(rest)) - 1;
                    rest &= rest - 1;
                    uf_union(P.parent, slot_of(slot0, base_v, w, b), slot_of(slot0, base_u, wu, b));
                }
            }
        }
    }
}
__device__ __forceinline__ void pc_count_body(const Phase2Args& P, unsigned first, unsigned stride, unsigned total) {
    for (unsigned e = first; e < total; e += stride) {
        const int cnt = __popcll(P.left_w[e]);
        for (int i = 0; i < cnt; ++i) atomicAdd(&P.comp_size[uf_find(P.parent, P.slot0 + P.left_base[e] + i)], 1);
    }
}
__device__ __forceinline__ void pc_reduce_body(const Phase2Args& P, unsigned first, unsigned stride, unsigned total) {
    for (unsigned e = first; e < total; e += stride) {
        word_t w = P.left_w[e];
        const int g = P.left_g[e];
        int slot = P.slot0 + P.left_base[e];
        while (w) {
            const int b = __ffsll(static_cast<long long>(w)) - 1;
            w &= w - 1;
            if (P.parent[slot] == slot) {  // a root that is not a giant node
                const unsigned long long s = static_cast<unsigned long long>(P.comp_size[slot]);
                atomicAdd(&P.pc_extra[g * kBits + b], s * (s - 1ull) / 2ull);
                atomicMax(&P.mcn_extra[g * kBits + b], static_cast<int>(s));
            }
            ++slot;
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_pc_hook(Phase2Args P, unsigned many) {
    griddep_launch();
    griddep_wait();
    if (pc_stand_down(P.counters, many)) return;
    pc_hook_body(P, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, P.counters->n_entries);
}
__global__ void __launch_bounds__(kThreads) k_pc_count(Phase2Args P, unsigned many) {
    griddep_launch();
    griddep_wait();
    if (pc_stand_down(P.counters, many)) return;
    pc_count_body(P, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, P.counters->n_entries);
}
__global__ void __launch_bounds__(kThreads) k_pc_reduce(Phase2Args P, unsigned many) {
    griddep_launch();
    griddep_wait();
    if (pc_stand_down(P.counters, many)) return;
    pc_reduce_body(P, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, P.counters->n_entries);
}

// pairwise_connectivity / largest_component_size (components.cpp:49-62) -> double
// (fitness.cpp:25,32).  giant = n - removed - unreached + leftovers attached to it;
// every vertex outside the giant and outside the union-find components is a
// singleton: 0 pairs, size 1.
__device__ __forceinline__ double pc_result_of(int n, int task, int removed, int unreached, int attached, unsigned long long pc_extra,
                                               int mcn_extra) {
    const long long giant = static_cast<long long>(n) - removed - unreached + attached;
    if (task == GAPA_TASK_PC) return static_cast<double>(static_cast<unsigned long long>(giant * (giant - 1) / 2) + pc_extra);
    long long best = giant > mcn_extra ? giant : mcn_extra;
    if (n > 0 && best < 1) best = 1;
    return static_cast<double>(best);
}

// Last kernel of a speculatively scheduled lane, ONE CTA: phase 2 when the recording sweep left at most `fused_limit`
// entries (the benchmark graphs leave none: three launches saved), the result of every row, the lane's counters into
// pinned host memory (no copy operation), and the reset of everything the next lane on this scratch set accumulates
// into (no reset launch, no memset).  do_phase2 == 0: the three full-grid kernels have already run.
static constexpr int kFinalThreads = 1024;
__global__ void __launch_bounds__(kFinalThreads) k_pc_final(Phase2Args P, unsigned many, unsigned fused_limit, int do_phase2, int rows,
                                                            int task, int* removed_count, int* unreached, double* out,
                                                            PcCounters* counters, PcCounters* host_out, int reset_slots) {
    griddep_launch();
    griddep_wait();
    __shared__ PcCounters c;
    __shared__ int skipped;
    const unsigned tid = threadIdx.x;
    if (tid == 0) {
        c = *counters;
        skipped = 0;
    }
    __syncthreads();
    if (!pc_stand_down(&c, many)) {
        if (do_phase2 && c.n_entries) {
            if (c.n_entries <= fused_limit) {
                pc_hook_body(P, tid, kFinalThreads, c.n_entries);
                __syncthreads();
                pc_count_body(P, tid, kFinalThreads, c.n_entries);
                __syncthreads();
                pc_reduce_body(P, tid, kFinalThreads, c.n_entries);
            } else if (tid == 0) {
                skipped = 1;
            }
        }
        __syncthreads();
        if (!skipped)
            for (int r = tid; r < rows; r += kFinalThreads)
                out[r] = pc_result_of(P.n, task, removed_count[r], unreached[r], P.comp_size[r], P.pc_extra[r], P.mcn_extra[r]);
    }
    __syncthreads();
    if (tid == 0) {
        c.phase2_skipped = skipped;
        *host_out = c;
        PcCounters zero{};
        zero.max_source = -1;
        *counters = zero;
    }
    for (int i = tid; i < reset_slots; i += kFinalThreads) {
        P.parent[i] = i;
        P.comp_size[i] = 0;
        unreached[i] = 0;
        P.pc_extra[i] = 0ull;
        P.mcn_extra[i] = 0;
        removed_count[i] = 0;
    }
}

__global__ void __launch_bounds__(kThreads) k_pc_result(int n, int rows, int task, const int* __restrict__ removed_count,
                                                        const int* __restrict__ unreached,
                                                        const int32_t* __restrict__ comp_size,
                                                        const unsigned long long* __restrict__ pc_extra,
                                                        const int* __restrict__ mcn_extra, double* out) {
    griddep_launch();
    griddep_wait();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    out[r] = pc_result_of(n, task, removed_count[r], unreached[r], comp_size[r], pc_extra[r], mcn_extra[r]);
}

// reset of everything the final sweep / phase 2 accumulate into
__global__ void k_pc_reset(int groups, int32_t* parent, int32_t* comp_size, int* unreached,
                           unsigned long long* pc_extra, int* mcn_extra, PcCounters* counters, int first) {
    griddep_launch();
    griddep_wait();
    const int total = groups * kBits;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        parent[i] = i;
        comp_size[i] = 0;
        unreached[i] = 0;
        pc_extra[i] = 0ull;
        mcn_extra[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counters->n_entries = 0u;
        counters->n_slots = 0u;
        counters->overflow = 0;
        counters->changed = 0;
        counters->n_incomplete = 0u;
        counters->deferred = 0;
        counters->n_left = 0u;
        if (first) counters->range_error = 0;
        if (first) counters->max_source = -1;
    }
}

// ---------------------------------------------------------------------------------
// Small graphs (n <= kSmallMaxN): the bit-sliced pipeline is launch-latency-bound there, so one
// CTA takes one individual through the whole reference algorithm in SHARED memory — removed
// bitmap, lock-free union-find over the alive edges (edge list, coalesced), component sizes,
// sum of s(s-1)/2 and max s — in a single kernel.  Same integers as the big path.
static constexpr int kSmallMaxN = 16384;
static constexpr int kSmallThreadsFew = 512;   // CTA size when the batch has fewer rows than the GPU has room for (latency per row)
static constexpr int kSmallThreadsMany = 128;  // ... and when rows outnumber the SMs several times (throughput)

template <int kSmallThreads>
__global__ void __launch_bounds__(kSmallThreads) k_pc_small(GeneRows genes,
                                                            const int32_t* __restrict__ pool_map, int pool_size, int n, int m,
                                                            const int32_t* __restrict__ edge_u,
                                                            const int32_t* __restrict__ edge_v, int task,
                                                            double* __restrict__ out, PcCounters* counters, VariationSpec V,
                                                            int have_vary) {
    extern __shared__ int32_t small_smem[];
    __shared__ uint64_t vary_keys[4];
    __shared__ long long warp_pairs[kSmallThreads / 32];
    __shared__ int warp_best[kSmallThreads / 32];
    const int tid = threadIdx.x, row = blockIdx.x;
    griddep_launch();  // the next launch on the stream may become resident now (it waits for this one where it must)
    int32_t* parent = small_smem;
    int32_t* size = parent + n;
    unsigned* gone = reinterpret_cast<unsigned*>(size + n);
    const int gone_words = (n + 31) >> 5;
    for (int w = tid; w < gone_words; w += kSmallThreads) gone[w] = 0u;
    for (int v = tid; v < n; v += kSmallThreads) {
        parent[v] = v;
        size[v] = 0;
    }
    griddep_wait();  // everything above is this CTA's own shared memory; from here on the predecessor's results are read
    __syncthreads();
    const int cols = genes.cols;
    if (have_vary) {
        // generation loop: this CTA BUILDS child row V.row_first + row (variation.cuh) into its slot and marks
        // its genes in the same pass — one launch less per generation where launches are what a generation costs
        const int vrow = V.row_first + row;
        if (tid < 4)
            vary_keys[tid] = stream_key(V.P.seed, V.P.generation, GAPA_ROLE_SELECT + tid, static_cast<uint64_t>(vrow)) + kGolden;
        __syncthreads();
        const uint64_t ks = vary_keys[0], kc = vary_keys[1], km = vary_keys[2], ki = vary_keys[3];
        const bool eda = V.partner == nullptr;
        const int slot_mine = V.parent[vrow], slot_theirs = eda ? slot_mine : V.parent[V.partner[vrow]];
        bool adopt_mine, adopt_theirs;
        const int32_t* mine = parent_row(V, slot_mine, cols, &adopt_mine);
        const int32_t* theirs = eda ? mine : parent_row(V, slot_theirs, cols, &adopt_theirs);
        if (eda || slot_theirs == slot_mine) adopt_theirs = false;
        int32_t* keep_mine = V.pool + static_cast<size_t>(slot_mine) * cols;
        int32_t* keep_theirs = V.pool + static_cast<size_t>(slot_theirs) * cols;
        int32_t* dst = V.pool + static_cast<size_t>(V.child[vrow]) * cols;
        for (int j = tid; j < cols; j += kSmallThreads) {
            const int a = mine[j], b = theirs[j];
            if (adopt_mine) keep_mine[j] = a;
            if (adopt_theirs) keep_theirs[j] = b;
            const int gene = child_gene(V.P, V.pool, V.parent, cols, j, a, b, eda, ks, kc, km, ki, static_cast<uint32_t>(j) + 1u);
            dst[j] = gene;
            const int node = pool_map ? pool_map[gene] : gene;
            atomicOr(&gone[node >> 5], 1u << (node & 31));
        }
    } else {
        const int32_t* g = genes.row(row);
        for (int j = tid; j < cols; j += kSmallThreads) {
            const int gene = g[j];
            if (gene < 0 || gene >= pool_size) {
                counters->range_error = 1;
                continue;
            }
            const int node = pool_map ? pool_map[gene] : gene;
            atomicOr(&gone[node >> 5], 1u << (node & 31));
        }
    }
    __syncthreads();
    for (int e = tid; e < m; e += kSmallThreads) {
        const int u = edge_u[e], v = edge_v[e];
        if (((gone[u >> 5] >> (u & 31)) | (gone[v >> 5] >> (v & 31))) & 1u) continue;
        uf_union(parent, u, v);
    }
    __syncthreads();
    for (int v = tid; v < n; v += kSmallThreads)
        if (!((gone[v >> 5] >> (v & 31)) & 1u)) atomicAdd(&size[uf_find(parent, v)], 1);
    __syncthreads();
    long long pairs = 0;
    int best = n > 0 ? 1 : 0;  // removed vertices are singletons
    for (int v = tid; v < n; v += kSmallThreads) {
        const long long sz = size[v];
        pairs += sz * (sz - 1) / 2;
        best = max(best, static_cast<int>(sz));
    }
    for (int off = 16; off; off >>= 1) {
        pairs += __shfl_down_sync(0xffffffffu, pairs, off);
        best = max(best, __shfl_down_sync(0xffffffffu, best, off));
    }
    if ((tid & 31) == 0) {
        warp_pairs[tid >> 5] = pairs;
        warp_best[tid >> 5] = best;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kSmallThreads / 32; ++w) {
            pairs += warp_pairs[w];
            best = max(best, warp_best[w]);
        }
        out[row] = task == GAPA_TASK_PC ? static_cast<double>(pairs) : static_cast<double>(best);
    }
}

// The same per-individual algorithm for graphs of ANY size, with the union-find arrays in global memory (L2) instead of
// shared memory (round 2).  The bit-sliced pipeline lives on graphs with a well-connected core: one ordered sweep reaches
// nearly everything.  On high-diameter graphs (rings, grids, paths: reachability advances a few hops per sweep round, and
// after removals there is no giant component, so most of the graph ends up in phase 2) it needed up to 48 host-driven rounds
// — 5-7 ms for 512 individuals at n = 1e5.  A plain lock-free union-find per individual does not care about diameter.
// PERSISTENT: CTA b walks rows b, b + grid, ... on its own scratch slot (parent[n], size[n]); the removed bitmap is in shared
// memory.  pc_eval chooses between the two per context by MEASURING both the first time the pipeline needs the host-driven
// loop (PcScratch::uf_mode).
template <int kUfThreads>
__global__ void __launch_bounds__(kUfThreads, 2048 / kUfThreads) k_pc_uf(GeneRows genes, const int32_t* __restrict__ pool_map, int pool_size, int n, int m,
                                                      const int32_t* __restrict__ edge_u, const int32_t* __restrict__ edge_v, int task,
                                                      double* __restrict__ out, PcCounters* counters, VariationSpec V, int have_vary,
                                                      int rows, int32_t* scratch) {
    griddep_launch();
    griddep_wait();
    extern __shared__ int32_t small_smem[];
    __shared__ uint64_t vary_keys[4];
    __shared__ long long warp_pairs[kUfThreads / 32];
    __shared__ int warp_best[kUfThreads / 32];
    const int tid = threadIdx.x;
    int32_t* parent = scratch + static_cast<size_t>(blockIdx.x) * 2 * n;
    int32_t* size = parent + n;
    unsigned* gone = reinterpret_cast<unsigned*>(small_smem);
    const int gone_words = (n + 31) >> 5;
    const int cols = genes.cols;
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        for (int w = tid; w < gone_words; w += kUfThreads) gone[w] = 0u;
        for (int v = tid; v < n; v += kUfThreads) {
            parent[v] = v;
            size[v] = 0;
        }
        if (have_vary && tid < 4)
            vary_keys[tid] = stream_key(V.P.seed, V.P.generation, GAPA_ROLE_SELECT + tid, static_cast<uint64_t>(V.row_first + row)) + kGolden;
        __syncthreads();
        if (have_vary) {
            const int vrow = V.row_first + row;
            const uint64_t ks = vary_keys[0], kc = vary_keys[1], km = vary_keys[2], ki = vary_keys[3];
            const bool eda = V.partner == nullptr;
            const int slot_mine = V.parent[vrow], slot_theirs = eda ? slot_mine : V.parent[V.partner[vrow]];
            bool adopt_mine, adopt_theirs;
            const int32_t* mine = parent_row(V, slot_mine, cols, &adopt_mine);
            const int32_t* theirs = eda ? mine : parent_row(V, slot_theirs, cols, &adopt_theirs);
            if (eda || slot_theirs == slot_mine) adopt_theirs = false;
            int32_t* keep_mine = V.pool + static_cast<size_t>(slot_mine) * cols;
            int32_t* keep_theirs = V.pool + static_cast<size_t>(slot_theirs) * cols;
            int32_t* dst = V.pool + static_cast<size_t>(V.child[vrow]) * cols;
            for (int j = tid; j < cols; j += kUfThreads) {
                const int a = mine[j], b = theirs[j];
                if (adopt_mine) keep_mine[j] = a;
                if (adopt_theirs) keep_theirs[j] = b;
                const int gene = child_gene(V.P, V.pool, V.parent, cols, j, a, b, eda, ks, kc, km, ki, static_cast<uint32_t>(j) + 1u);
                dst[j] = gene;
                const int node = pool_map ? pool_map[gene] : gene;
                atomicOr(&gone[node >> 5], 1u << (node & 31));
            }
        } else {
            const int32_t* g = genes.row(row);
            for (int j = tid; j < cols; j += kUfThreads) {
                const int gene = g[j];
                if (gene < 0 || gene >= pool_size) {
                    counters->range_error = 1;
                    continue;
                }
                const int node = pool_map ? pool_map[gene] : gene;
                atomicOr(&gone[node >> 5], 1u << (node & 31));
            }
        }
        __syncthreads();
        for (int e = tid; e < m; e += kUfThreads) {
            const int u = edge_u[e], v = edge_v[e];
            if (((gone[u >> 5] >> (u & 31)) | (gone[v >> 5] >> (v & 31))) & 1u) continue;
            uf_union(parent, u, v);
        }
        __syncthreads();
        for (int v = tid; v < n; v += kUfThreads)
            if (!((gone[v >> 5] >> (v & 31)) & 1u)) atomicAdd(&size[uf_find(parent, v)], 1);
        __syncthreads();
        long long pairs = 0;
        int best = n > 0 ? 1 : 0;  // removed vertices are singletons
        for (int v = tid; v < n; v += kUfThreads) {
            const long long sz = size[v];
            pairs += sz * (sz - 1) / 2;
            best = max(best, static_cast<int>(sz));
        }
        for (int off = 16; off; off >>= 1) {
            pairs += __shfl_down_sync(0xffffffffu, pairs, off);
            best = max(best, __shfl_down_sync(0xffffffffu, best, off));
        }
        if ((tid & 31) == 0) {
            warp_pairs[tid >> 5] = pairs;
            warp_best[tid >> 5] = best;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kUfThreads / 32; ++w) {
                pairs += warp_pairs[w];
                best = max(best, warp_best[w]);
            }
            out[row] = task == GAPA_TASK_PC ? static_cast<double>(pairs) : static_cast<double>(best);
        }
        __syncthreads();  // the next row reuses the bitmap, the scratch slot and the reduction buffers
    }
}
static constexpr int kUfThreads = 512;

// ---------------------------------------------------------------------------------
static int ensure_phase2(PcSet* s, int groups, size_t entries, size_t slots) {
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

static int env_int(const char* name, int fallback, int lo, int hi) {
    const char* raw = std::getenv(name);
    if (!raw || !*raw) return fallback;
    const long v = std::strtol(raw, nullptr, 10);
    return static_cast<int>(std::min<long>(hi, std::max<long>(lo, v)));
}

// The sweeps assume that LOW vertex ids are the well-connected core: rows are scanned in ascending
// id, the prefix kernel closes ids [0, prefix), and blocks run in ascending id.  Generators that grow
// a graph (Barabasi-Albert) number vertices that way already.  For any other numbering the bit-sliced
// path works on an internal relabelling by descending degree — component sizes do not depend on
// vertex names — built once per (graph, pool) on the host: a permuted CSR with ascending rows and a
// gene -> internal vertex map.  Natural order is kept when its first n/32 ids already hold at least
// 70 % of the edge endpoints that the n/32 highest-degree vertices hold.
static int ensure_order(gapa_cuda_ctx* ctx, PcScratch* s) {
    if (s->ord_ready && s->ord_pool_version == ctx->pool_version) return GAPA_CUDA_OK;
    const int n = ctx->n;
    const std::vector<int32_t>& rp = ctx->h_row_ptr;
    const std::vector<int32_t>& ci = ctx->h_col_idx;
    if (!s->ord_ready) {
        std::vector<int32_t> order(n);
        for (int v = 0; v < n; ++v) order[v] = v;
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return rp[a + 1] - rp[a] > rp[b + 1] - rp[b]; });
        const int head = std::max(1, n / 32);
        long long mass_natural = 0, mass_degree = 0;
        for (int i = 0; i < head; ++i) {
            mass_natural += rp[i + 1] - rp[i];
            mass_degree += rp[order[i] + 1] - rp[order[i]];
        }
        s->ord_relabeled = s->relabel == 1 || (s->relabel != 0 && mass_natural * 10 < mass_degree * 7);
        s->perm.clear();
        if (s->ord_relabeled) {
            s->perm.resize(n);
            for (int i = 0; i < n; ++i) s->perm[order[i]] = i;
            std::vector<int32_t> row_ptr(static_cast<size_t>(n) + 1, 0), col_idx(ci.size());
            for (int i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + (rp[order[i] + 1] - rp[order[i]]);
            for (int i = 0; i < n; ++i) {
                const int old = order[i];
                int32_t* dst = col_idx.data() + row_ptr[i];
                for (int e = rp[old]; e < rp[old + 1]; ++e) *dst++ = s->perm[ci[e]];
                std::sort(col_idx.data() + row_ptr[i], dst);
            }
            GAPA_TRY(s->ord_row_ptr.ensure(sizeof(int32_t) * row_ptr.size()));
            GAPA_TRY(s->ord_col_idx.ensure(sizeof(int32_t) * std::max<size_t>(col_idx.size(), 1)));
            GAPA_CUDA_TRY(cudaMemcpy(s->ord_row_ptr.ptr, row_ptr.data(), sizeof(int32_t) * row_ptr.size(), cudaMemcpyHostToDevice));
            if (!col_idx.empty())
                GAPA_CUDA_TRY(cudaMemcpy(s->ord_col_idx.ptr, col_idx.data(), sizeof(int32_t) * col_idx.size(), cudaMemcpyHostToDevice));
        }
        {  // first four neighbours of every vertex in the order the sweeps use
            const std::vector<int32_t>* use_rp = &rp;
            const std::vector<int32_t>* use_ci = &ci;
            std::vector<int32_t> drp, dci;
            if (s->ord_relabeled) {
                drp.resize(static_cast<size_t>(n) + 1);
                dci.resize(ci.size());
                GAPA_CUDA_TRY(cudaMemcpy(drp.data(), s->ord_row_ptr.ptr, sizeof(int32_t) * drp.size(), cudaMemcpyDeviceToHost));
                if (!dci.empty()) GAPA_CUDA_TRY(cudaMemcpy(dci.data(), s->ord_col_idx.ptr, sizeof(int32_t) * dci.size(), cudaMemcpyDeviceToHost));
                use_rp = &drp;
                use_ci = &dci;
            }
            std::vector<int32_t> first(static_cast<size_t>(4) * std::max(n, 1), -1);
            for (int v = 0; v < n; ++v)
                for (int t = 0; t < 4 && (*use_rp)[v] + t < (*use_rp)[v + 1]; ++t) first[4 * static_cast<size_t>(v) + t] = (*use_ci)[(*use_rp)[v] + t];
            GAPA_TRY(s->nbr4.ensure(sizeof(int32_t) * first.size()));
            GAPA_CUDA_TRY(cudaMemcpy(s->nbr4.ptr, first.data(), sizeof(int32_t) * first.size(), cudaMemcpyHostToDevice));
        }
        s->ord_ready = true;
    }
    if (s->ord_relabeled) {  // gene -> internal vertex
        std::vector<int32_t> map(static_cast<size_t>(std::max(ctx->pool_size, 1)));
        for (int gidx = 0; gidx < ctx->pool_size; ++gidx)
            map[gidx] = s->perm[ctx->pool_identity ? gidx : ctx->h_pool_map[gidx]];
        GAPA_TRY(s->ord_gene_map.ensure(sizeof(int32_t) * map.size()));
        GAPA_CUDA_TRY(cudaMemcpy(s->ord_gene_map.ptr, map.data(), sizeof(int32_t) * map.size(), cudaMemcpyHostToDevice));
    }
    s->ord_pool_version = ctx->pool_version;
    return GAPA_CUDA_OK;
}

// clear of the reached records (a kernel rather than cudaMemsetAsync so that profilers list it with its DRAM bytes)
__global__ void __launch_bounds__(kThreads) k_pc_clear(Rec* __restrict__ recs, size_t count) {
    griddep_launch();
    griddep_wait();
    const Rec zero{};
    for (size_t i = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x; i < count; i += static_cast<size_t>(gridDim.x) * kThreads)
        store_rec(&recs[i], zero);
}

// ---------------------------------------------------------------------------------
// One lane = `crows` individuals (whole 64-individual groups) taken through the whole pipeline on `stream` with the
// scratch of `set`.  Two schedules:
//   * speculative (spec_rounds >= 1): everything — masks, prefix closure, `spec_rounds` rounds of sweeps, the recording
//     sweep, phase 2 and the result — is enqueued without the host ever looking at the device; the lane's counters
//     land in pinned memory after the last kernel and the caller checks them once, when the whole evaluation has been
//     enqueued.  Phase 2 stands down on the device when the recording sweep overflowed / declined / wants more sweeps
//     (pc_stand_down), and the caller then redoes the lane host-driven.  No host round trip sits inside an evaluation,
//     so lanes on different streams overlap freely (the integer-bound mask build of one lane under the HBM-bound
//     sweeps of another).
//   * host-driven (spec_rounds == 0): sweep rounds until the counters say phase 2 can finish (graphs without a hub
//     core, high-diameter graphs, buffer growth after an overflow).  *rounds_used reports what it took.
struct PcLaneJob {
    int task;
    GeneRows genes;          // the whole batch
    int row0, crows;         // this lane's rows
    double* out_dev;         // the whole batch
    bool trusted;
    const VariationSpec* vary;
};

static int pc_set_create(PcSet** out) {
    PcSet* set = new PcSet();
    *out = set;
    // lowest priority for the clear: it yields to every kernel of the work streams
    int least = 0, greatest = 0;
    GAPA_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GAPA_CUDA_TRY(cudaStreamCreateWithPriority(&set->aux, cudaStreamNonBlocking, least));
    GAPA_CUDA_TRY(cudaStreamCreateWithFlags(&set->stream, cudaStreamNonBlocking));
    GAPA_CUDA_TRY(cudaEventCreateWithFlags(&set->ev_pass_begin, cudaEventDisableTiming));
    GAPA_CUDA_TRY(cudaEventCreateWithFlags(&set->ev_cleared, cudaEventDisableTiming));
    GAPA_CUDA_TRY(cudaEventCreateWithFlags(&set->ev_done, cudaEventDisableTiming));
    return GAPA_CUDA_OK;
}

static int pc_run_lane(gapa_cuda_ctx* ctx, PcScratch* s, PcSet* set, const PcLaneJob& job, cudaStream_t stream, int spec_rounds,
                       PcCounters* h_out, int* rounds_used) {
    const int n = ctx->n, sm = ctx->sm_count, cols = job.genes.cols;
    const int row0 = job.row0, crows = job.crows;
    const int32_t* g_row_ptr = s->ord_relabeled ? s->ord_row_ptr.as<int32_t>() : ctx->d_row_ptr;
    const int32_t* g_col_idx = s->ord_relabeled ? s->ord_col_idx.as<int32_t>() : ctx->d_col_idx;
    const int32_t* g_gene_map = s->ord_relabeled ? s->ord_gene_map.as<int32_t>() : (ctx->pool_identity ? nullptr : ctx->d_pool_map);
    const int32_t* g_by_degree = s->ord_relabeled ? nullptr : ctx->d_by_degree;
    const int words_per_row = std::max(1, (n + 63) / 64);
    int chunk_bits = std::min(words_per_row * 64, 192 * 1024 * 8);  // <= 192 KB of shared memory
    if (s->mask_chunks > 1) chunk_bits = std::min(chunk_bits, ((words_per_row + s->mask_chunks - 1) / s->mask_chunks) * 64);
    const int chunks = (words_per_row * 64 + chunk_bits - 1) / chunk_bits;
    const int groups = (crows + kBits - 1) / kBits;
    const int sgroups = (groups + kPack - 1) / kPack;  // 4 groups share one 32-byte vertex record
    const int pgroups = sgroups * kPack;
    const size_t words = static_cast<size_t>(pgroups) * std::max(n, 1);
    auto accumulators = [&]() {  // a buffer that had to grow comes back uninitialised
        return reinterpret_cast<uintptr_t>(set->removed_count.ptr) ^ reinterpret_cast<uintptr_t>(set->unreached.ptr) * 3 ^
               reinterpret_cast<uintptr_t>(set->pc_extra.ptr) * 5 ^ reinterpret_cast<uintptr_t>(set->mcn_extra.ptr) * 7 ^
               reinterpret_cast<uintptr_t>(set->counters.ptr) * 11 ^ reinterpret_cast<uintptr_t>(set->parent.ptr) * 13 ^
               reinterpret_cast<uintptr_t>(set->comp_size.ptr) * 17;
    };
    const uintptr_t accumulators_before = accumulators();
    GAPA_TRY(set->removed.ensure(sizeof(word_t) * static_cast<size_t>(crows) * words_per_row));
    GAPA_TRY(set->removed_count.ensure(sizeof(int) * pgroups * kBits));
    GAPA_TRY(set->alive.ensure(sizeof(word_t) * words));
    GAPA_TRY(set->reached.ensure(sizeof(word_t) * words));
    GAPA_TRY(set->entry_of.ensure(sizeof(int32_t) * words));
    GAPA_TRY(set->unreached.ensure(sizeof(int) * pgroups * kBits));
    GAPA_TRY(set->pc_extra.ensure(sizeof(unsigned long long) * pgroups * kBits));
    GAPA_TRY(set->mcn_extra.ensure(sizeof(int) * pgroups * kBits));
    {
        const size_t before = set->counters.cap;
        GAPA_TRY(set->counters.ensure(sizeof(PcCounters)));
        // a fresh block: k_pc_final copies the whole struct, including the field only the host copy uses (initcheck)
        if (set->counters.cap != before) GAPA_CUDA_TRY(cudaMemsetAsync(set->counters.ptr, 0, set->counters.cap, stream));
    }
    if (set->cap_entries == 0 || set->parent.cap < sizeof(int32_t) * (static_cast<size_t>(pgroups) * kBits + set->cap_slots))
        GAPA_TRY(ensure_phase2(set, pgroups, std::max<size_t>(set->cap_entries, 1u << 16), std::max<size_t>(set->cap_slots, 1u << 20)));
    word_t* alive = set->alive.as<word_t>();
    word_t* reached = set->reached.as<word_t>();
    PcCounters* counters = set->counters.as<PcCounters>();
    const int slot0 = pgroups * kBits;
    const int reset_grid = std::max(1, (pgroups * kBits + kThreads - 1) / kThreads);
    auto reset = [&](int first) -> int {
        GAPA_LAUNCH(k_pc_reset, reset_grid, kThreads, 0, stream, pgroups, set->parent.as<int32_t>(), set->comp_size.as<int32_t>(),
                    set->unreached.as<int>(), set->pc_extra.as<unsigned long long>(), set->mcn_extra.as<int>(), counters, first);
        return GAPA_CUDA_OK;
    };
    const bool speculative = spec_rounds >= 1 && n > 0;
    if (accumulators() != accumulators_before) set->clean_slots = 0;
    if (!(speculative && set->clean_slots >= pgroups * kBits)) {
        GAPA_TRY(reset(1));
        GAPA_CUDA_TRY(cudaMemsetAsync(set->removed_count.ptr, 0, sizeof(int) * pgroups * kBits, stream));
    }
    set->clean_slots = 0;
    if (rounds_used) *rounds_used = 0;

    if (n > 0) {
        // The clear of the `reached` records depends on nothing this lane computes, only on the previous user of the
        // buffer being done: it runs on a side stream underneath the mask build, which is bound by integer issue.
        if (s->overlap_clear && sizeof(word_t) * words > s->fold_clear_bytes) GAPA_CUDA_TRY(cudaEventRecord(set->ev_pass_begin, stream));
        const int clear_grid = static_cast<int>(std::max<size_t>(1, std::min<size_t>(static_cast<size_t>(sm) * 8, (words / kPack + kThreads - 1) / kThreads)));
        // ---- masks ------------------------------------------------------------------
        // one CTA per individual: as many threads as it has 16-byte gene quads (or bitmap words) to work on, so that
        // small budgets do not occupy an SM with idle warps (k = 500: 128 threads, 16 CTAs per SM instead of 2)
        // (k = 5000: 640 threads make two full passes over the 1250 quads where 1024 would idle 40 % of their slots)
        auto mask_cta = [&](int work) {  // the CTA size whose passes over `work` items waste the fewest thread slots
            int best = 128;
            long best_cost = -1;
            for (int nt = 128; nt <= kMaskThreads; nt += 128) {
                const long cost = static_cast<long>((work + nt - 1) / nt) * nt;
                if (best_cost < 0 || cost <= best_cost) best = nt, best_cost = cost;
            }
            return best;
        };
        const bool fused_mask = job.vary && chunks == 1 && cols > 0;
        // fused kernel: one 16-byte quad per thread and pass; plain kernel: two 32-byte loads per thread and pass
        // (with a bitmap that leaves room for only a few CTAs per SM the kernels live on the bytes each CTA keeps in
        // flight and keep the full 1024 threads: C4 measured 1.93 ms with 1024 against 1.95 ms with 896)
        int mask_threads = chunk_bits / 8 > 32 * 1024
                               ? kMaskThreads
                               : mask_cta(std::max({fused_mask ? cols / 4 : cols / 16, chunk_bits / 512, 1}));
        // The PERSISTENT fused kernel prefers many small CTAs per SM where the bitmap allows it (their prologues and epilogues
        // overlap each other's hashing) as soon as there are rows enough to fill them: n = 1e5 (k = 5000, 12.5 KB bitmap),
        // 128 instead of 640 threads: 4096 rows 0.356 -> 0.310 ms per generation, 16,384 rows 1.032 -> 0.893, 1024 rows
        // 0.214 -> 0.203; 256 rows 0.129 -> 0.132 (kept at the old rule).  tools: GAPA_PC_MASK_THREADS.
        if (fused_mask && chunk_bits / 8 <= 32 * 1024 && crows >= 4 * sm) mask_threads = 128;
        // bitmaps of which two still fit an SM (n = 5e5: 62.5 KB): two CTAs of 640 threads instead of one of 1024 —
        // generation 0.951 -> 0.907 ms (256 / 384 / 512 / 640 / 768 threads: 0.923 / 0.912 / 0.916 / 0.907 / 0.973)
        else if (fused_mask && chunk_bits / 8 <= 64 * 1024 && crows >= 4 * sm) mask_threads = 640;
        if (s->mask_threads_forced > 0) mask_threads = s->mask_threads_forced;  // GAPA_PC_MASK_THREADS (A/B)
        if (fused_mask) {
            VariationSpec pass = *job.vary;
            pass.row_first += row0;
            // persistent: as many CTAs as are resident at once, each walks rows blockIdx.x, + grid, ...
            auto vary_grid = [&](auto kernel, int nt) {
                int per_sm = 0;
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, static_cast<size_t>(chunk_bits) / 8) != cudaSuccess || per_sm < 1)
                    per_sm = 1;
                return std::max(1, std::min(crows, sm * per_sm * s->vary_waves));
            };
#define GAPA_MASK_VARY(NT)                                                                                                       \
    do {                                                                                                                        \
        if (pass.bases)                                                                                                         \
            GAPA_LAUNCH((k_pc_bitmask_vary<NT, true>), vary_grid((k_pc_bitmask_vary<NT, true>), NT), NT,                        \
                        static_cast<size_t>(chunk_bits) / 8, stream, pass, cols,                                                \
                        g_gene_map, n, words_per_row, set->removed.as<word_t>(), set->removed_count.as<int>(), crows);          \
        else                                                                                                                    \
            GAPA_LAUNCH((k_pc_bitmask_vary<NT, false>), vary_grid((k_pc_bitmask_vary<NT, false>), NT), NT,                      \
                        static_cast<size_t>(chunk_bits) / 8, stream, pass, cols,                                                \
                        g_gene_map, n, words_per_row, set->removed.as<word_t>(), set->removed_count.as<int>(), crows);          \
    } while (0)
            switch (mask_threads) {
                case 128: GAPA_MASK_VARY(128); break;
                case 256: GAPA_MASK_VARY(256); break;
                case 384: GAPA_MASK_VARY(384); break;
                case 512: GAPA_MASK_VARY(512); break;
                case 640: GAPA_MASK_VARY(640); break;
                case 768: GAPA_MASK_VARY(768); break;
                case 896: GAPA_MASK_VARY(896); break;
                default: GAPA_MASK_VARY(1024); break;
            }
#undef GAPA_MASK_VARY
        } else {
            if (job.vary) {
                VariationSpec pass = *job.vary;
                pass.row_first += row0;
                GAPA_TRY(launch_variation_spec(pass, cols, crows, stream));
            }
            auto rows_grid = [&](auto kernel, int nt) {  // persistent: as many CTAs as are resident at once
                int per_sm = 0;
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, static_cast<size_t>(chunk_bits) / 8) != cudaSuccess || per_sm < 1)
                    per_sm = 1;
                return std::max(1, std::min(crows, sm * per_sm));
            };
#define GAPA_MASK(NT)                                                                                                          \
    do {                                                                                                                      \
        if (chunks == 1 && s->mask_rows)                                                                                      \
            GAPA_LAUNCH(k_pc_bitmask_rows<NT>, rows_grid(k_pc_bitmask_rows<NT>, NT), NT, static_cast<size_t>(chunk_bits) / 8, \
                        stream, job.genes.from(row0), g_gene_map, ctx->pool_size, n, words_per_row,                           \
                        set->removed.as<word_t>(), set->removed_count.as<int>(), counters, crows);                            \
        else                                                                                                                  \
            GAPA_LAUNCH(k_pc_bitmask<NT>, dim3(chunks, crows), NT, static_cast<size_t>(chunk_bits) / 8, stream,               \
                        job.genes.from(row0), g_gene_map, ctx->pool_size, n, chunk_bits, words_per_row,                       \
                        set->removed.as<word_t>(), set->removed_count.as<int>(), counters);                                   \
    } while (0)
            switch (mask_threads) {
                case 128: GAPA_MASK(128); break;
                case 256: GAPA_MASK(256); break;
                case 384: GAPA_MASK(384); break;
                case 512: GAPA_MASK(512); break;
                case 640: GAPA_MASK(640); break;
                case 768: GAPA_MASK(768); break;
                case 896: GAPA_MASK(896); break;
                default: GAPA_MASK(1024); break;
            }
#undef GAPA_MASK
        }
        // small batches are bound by launches: the transpose kernel clears the records and the prefix kernel picks the sources
        const bool fold_clear = sizeof(word_t) * words <= s->fold_clear_bytes;
        const int prefix = std::min(s->prefix, n);
        if (!fold_clear && s->overlap_clear) {  // issued AFTER the mask kernel so that its CTAs only fill what that kernel leaves free
            GAPA_CUDA_TRY(cudaStreamWaitEvent(set->aux, set->ev_pass_begin, 0));
            GAPA_LAUNCH(k_pc_clear, clear_grid, kThreads, 0, set->aux, reinterpret_cast<Rec*>(reached), words / kPack);
            GAPA_CUDA_TRY(cudaEventRecord(set->ev_cleared, set->aux));
        }
        GAPA_LAUNCH(k_pc_transpose, dim3((words_per_row + kTransThreads - 1) / kTransThreads, pgroups), kTransThreads,
                    sizeof(word_t) * kBits * (kTransThreads + 1), stream, set->removed.as<word_t>(), words_per_row, n, crows, alive,
                    fold_clear ? reached : static_cast<word_t*>(nullptr));
        if (!fold_clear) {
            if (s->overlap_clear) GAPA_CUDA_TRY(cudaStreamWaitEvent(stream, set->ev_cleared, 0));
            else GAPA_LAUNCH(k_pc_clear, clear_grid, kThreads, 0, stream, reinterpret_cast<Rec*>(reached), words / kPack);
        }
        if (prefix <= 0)
            GAPA_LAUNCH(k_pc_source, (crows * 32 + kThreads - 1) / kThreads, kThreads, 0, stream, g_by_degree, n, crows, alive, reached, counters);

        // ---- phase 1 ------------------------------------------------------------------
        const word_t* alive_rec = alive;
        Rec* reached_rec = reinterpret_cast<Rec*>(reached);
        if (prefix > 0) {
            // measured on B200 (tools/ab_prefix.sh): 8 CTAs per super-group up to 8 groups, 4 at 16-32, 2 at 64;
            // beyond that every cluster must be resident at once (one CTA of this kernel per SM)
            int csize = sgroups <= 8 ? kPrefixCluster : 4;
            while (csize > 1 && sgroups * csize > sm) csize >>= 1;
            if (s->prefix_cluster > 0) csize = s->prefix_cluster;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(sgroups * csize);
            cfg.blockDim = dim3(kPrefixThreads);
            cfg.stream = stream;
            cudaLaunchAttribute attr[2]{};
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = csize; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr; cfg.numAttrs = pdl_allowed(cfg.gridDim) ? 2 : 1;
            GAPA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pc_prefix, g_row_ptr, g_col_idx, static_cast<const int4*>(s->nbr4.as<int4>()),
                                             s->prefix_first4, n, prefix, alive_rec, reached_rec, 1, g_by_degree, crows, counters));
            g_launches.fetch_add(1, std::memory_order_relaxed);
        }
        const int il = std::min(std::max(1, s->interleave / kPack), sgroups);
        const dim3 grid(((n + kThreads - 1) / kThreads) * il, (sgroups + il - 1) / il);
        GAPA_TRY(set->block_done.ensure(sizeof(int2) * static_cast<size_t>(sgroups) * ((n + kThreads - 1) / kThreads)));
        SweepArgs A;
        A.row_ptr = g_row_ptr; A.col_idx = g_col_idx; A.nbr4 = s->nbr4.as<int4>(); A.n = n; A.sgroups = sgroups; A.interleave = il;
        A.alive = alive_rec; A.reached = reached_rec; A.unreached = set->unreached.as<int>();
        A.entry_of = set->entry_of.as<int32_t>(); A.slot0 = slot0; A.counters = counters;
        A.incomplete = set->block_done.as<int2>(); A.record = 0; A.descending = 0; A.fresh_from = n; A.prefetch_chunks = s->sweep_prefetch;
        bool first_sweep = s->fresh_skip != 0;  // the reached records were cleared for this lane: nothing above the prefix is set
        A.defer_above = static_cast<unsigned>(std::min<size_t>(0xfffffffeu, static_cast<size_t>(sgroups) * n / 16));  // 6 % of the pairs
        auto sweep = [&](bool final_pass, bool record, bool descending = false, bool local = false) -> int {
            A.descending = descending ? 1 : 0;
            A.cap_entries = static_cast<unsigned>(set->cap_entries);  // may have grown after an overflow retry
            A.cap_slots = static_cast<unsigned>(set->cap_slots);
            A.left_v = set->left_v.as<int32_t>(); A.left_g = set->left_g.as<int32_t>(); A.left_w = set->left_w.as<word_t>();
            A.left_base = set->left_base.as<int32_t>(); A.parent = set->parent.as<int32_t>(); A.comp_size = set->comp_size.as<int32_t>();
            A.record = record ? 1 : 0;
            A.fresh_from = (!final_pass && !local && !descending && first_sweep) ? std::max(prefix, 0) : n;
            if (!final_pass) first_sweep = false;
            if (final_pass) GAPA_LAUNCH(k_pc_record, sm * 4, kThreads, 0, stream, A);
            else if (local) GAPA_LAUNCH(k_pc_sweep_local, grid, kThreads, 0, stream, A);
            else GAPA_LAUNCH(k_pc_sweep, grid, kThreads, 0, stream, A);
            return GAPA_CUDA_OK;
        };
        // With the prefix closed, ONE ordered sweep reaches nearly everything on power-law graphs and marks the
        // 256-vertex chunks that are complete; the recording sweep then only visits the few incomplete chunks, and
        // phase 2 (exact for any leftover, attaching to the giant through reached neighbours) finishes.  If a lot is
        // still unreached AND the sweeps were still making progress, more rounds follow first: one sweep in DESCENDING
        // block order, then an ascending one; from the fifth round on (random graphs converge before that; what is
        // left has a large diameter) each block iterates its chunk to a local fixpoint (k_pc_sweep_local).  Across
        // blocks reachability runs any distance along ids in the direction the blocks are scheduled but only one hop
        // against it: high-diameter graphs (rings, grids) need both directions to converge in a few rounds.
        const unsigned many = static_cast<unsigned>(std::max<size_t>(8192, words / 512));
        auto ordinary_sweeps = [&](int round, bool record_last) -> int {
            const int ordinary = round == 0 ? 1 : 2;
            for (int i = 0; i < ordinary; ++i) GAPA_TRY(sweep(false, record_last && i + 1 == ordinary, ordinary == 2 && i == 0, round >= 4));
            return GAPA_CUDA_OK;
        };
        Phase2Args P2;
        auto phase2_args = [&]() {  // the buffers may have grown after an overflow retry
            P2.row_ptr = g_row_ptr; P2.col_idx = g_col_idx; P2.n = n; P2.alive = alive; P2.reached = reached;
            P2.entry_of = set->entry_of.as<int32_t>(); P2.left_v = set->left_v.as<int32_t>(); P2.left_g = set->left_g.as<int32_t>();
            P2.left_w = set->left_w.as<word_t>(); P2.left_base = set->left_base.as<int32_t>(); P2.parent = set->parent.as<int32_t>();
            P2.comp_size = set->comp_size.as<int32_t>(); P2.slot0 = slot0; P2.pc_extra = set->pc_extra.as<unsigned long long>();
            P2.mcn_extra = set->mcn_extra.as<int>(); P2.counters = counters;
        };
        auto phase2 = [&](unsigned stand_down_above, unsigned entries_hint) -> int {
            const unsigned blocks = entries_hint ? (entries_hint + kThreads - 1) / kThreads : static_cast<unsigned>(sm * 8);
            const int pgrid = static_cast<int>(std::max(1u, std::min<unsigned>(blocks, sm * 8)));
            phase2_args();
            GAPA_LAUNCH(k_pc_hook, pgrid, kThreads, 0, stream, P2, stand_down_above);
            GAPA_LAUNCH(k_pc_count, pgrid, kThreads, 0, stream, P2, stand_down_above);
            GAPA_LAUNCH(k_pc_reduce, pgrid, kThreads, 0, stream, P2, stand_down_above);
            return GAPA_CUDA_OK;
        };
        if (spec_rounds >= 1) {
            for (int round = 0; round < spec_rounds; ++round) {
                if (round > 0) GAPA_TRY(reset(0));  // `changed` should tell about the last round only
                GAPA_TRY(ordinary_sweeps(round, round + 1 == spec_rounds));
            }
            GAPA_TRY(sweep(true, false));
            if (s->phase2_big) GAPA_TRY(phase2(many, 0));
            phase2_args();
            // the last kernel: (phase 2,) results, counters to the host, accumulators left clean for the next lane
            GAPA_LAUNCH(k_pc_final, 1, kFinalThreads, 0, stream, P2, many, kFusedPhase2Entries, s->phase2_big ? 0 : 1, crows, job.task,
                        set->removed_count.as<int>(), set->unreached.as<int>(), job.out_dev + row0, counters, h_out, pgroups * kBits);
            set->clean_slots = pgroups * kBits;  // entry slots start right above: a larger lane must reset for itself
            return GAPA_CUDA_OK;
        } else {
            PcCounters h{};
            for (int round = 0;; ++round) {
                GAPA_TRY(ordinary_sweeps(round, true));
                if (round >= 47) A.defer_above = ~0u;  // bounded: the last round records whatever is left
                GAPA_TRY(sweep(true, false));
                GAPA_CUDA_TRY(cudaMemcpyAsync(&h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
                GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
                if (h.range_error) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
                if (s->trace)
                    std::fprintf(stderr, "pc_eval round %d: entries %u slots %u overflow %d changed %d incomplete %u deferred %d (cap %zu / %zu)\n",
                                 round, h.n_entries, h.n_slots, h.overflow, h.changed, h.n_incomplete, h.deferred, set->cap_entries, set->cap_slots);
                const bool retry_bigger = h.overflow != 0;
                const bool keep_sweeping = h.deferred || (h.changed && h.n_entries > many && round < 48);
                if (rounds_used) *rounds_used = round + 1;
                if (!retry_bigger && !keep_sweeping) break;
                if (retry_bigger)
                    GAPA_TRY(ensure_phase2(set, pgroups, std::max<size_t>(set->cap_entries, static_cast<size_t>(h.n_entries) + 1024),
                                           std::max<size_t>(set->cap_slots, static_cast<size_t>(h.n_slots) + 1024)));
                GAPA_TRY(reset(0));
            }
            if (h.n_entries) GAPA_TRY(phase2(~0u, h.n_entries));
        }
    } else if (static_cast<size_t>(crows) * cols) {
        return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
    }
    GAPA_LAUNCH(k_pc_result, (crows + kThreads - 1) / kThreads, kThreads, 0, stream, n, crows, job.task, set->removed_count.as<int>(),
                set->unreached.as<int>(), set->comp_size.as<int32_t>(), set->pc_extra.as<unsigned long long>(),
                set->mcn_extra.as<int>(), job.out_dev + row0);
    return GAPA_CUDA_OK;
}

int pc_eval(gapa_cuda_ctx* ctx, int task, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, bool trusted,
            const VariationSpec* vary) {
    const int cols = genes.cols;
    if (!ctx->pc) ctx->pc = new PcScratch();
    PcScratch* s = ctx->pc;
    if (!s->configured) {  // tuning knobs (defaults are what bench.py measures)
        s->prefix = env_int("GAPA_PC_PREFIX", 32768, 0, 1 << 24);
        s->prefix_cluster = env_int("GAPA_PC_PREFIX_CLUSTER", 0, 0, 8);  // 0 = choose by the number of super-groups
        s->interleave = env_int("GAPA_PC_INTERLEAVE", 16, 1, 64);  // measured: tools/ab_prefix_len.sh
        s->mask_chunks = env_int("GAPA_PC_MASK_CHUNKS", 1, 1, 64);
        s->relabel = env_int("GAPA_PC_RELABEL", -1, -1, 1);  // -1 automatic, 0 never, 1 always (tests)
        s->small_path = env_int("GAPA_PC_SMALL", 1, 0, 2);  // 0: never, 1: where it pays, 2: wherever it fits (tests)
        // individuals per lane.  Measured at C4 (tools/ab_lanes.sh): ONE lane of 4096 is as fast as two of 2048 (1.887 vs
        // 1.877 ms per generation) and every finer split is slower (1024 x 2 streams 1.97, 512 x 4 2.01, 256 x 8 2.33 ms):
        // the mask kernel holds a whole SM (125 KB bitmap, 1024 threads x 64 registers), so a second lane's sweeps find no
        // room beside it, and every lane pays the latency-bound prefix closure again.  Re-measured at population 16,384 with
        // the persistent variation kernel (tools/ab_lanes_small.sh; lanes of 4096 / 8192 / one lane): n = 1e4 0.462 / 0.422 /
        // 0.409 ms per generation, n = 1e5 1.162 / 1.126 / 1.148, n = 1e6 6.64 / 6.67 / 6.50 — lanes no longer pay
        // anywhere, so a lane is 16,384 individuals (beyond that, and whatever the scratch budget forces, is split).
        s->lane_rows = env_int("GAPA_PC_LANE_ROWS", 16384, 64, 1 << 20) / kBits * kBits;
        s->lane_streams = env_int("GAPA_PC_LANE_STREAMS", 2, 1, 8);  // lanes in flight
        s->spec_rounds = env_int("GAPA_PC_SPEC_ROUNDS", 1, 0, 6);    // 0: always the host-driven loop
        s->phase2_big = env_int("GAPA_PC_PHASE2_BIG", 0, 0, 1) != 0;  // 1: never resolve leftovers inside k_pc_final (tests)
        s->fold_clear_bytes = static_cast<size_t>(env_int("GAPA_PC_FOLD_CLEAR_MB", 16, 0, 1 << 20)) << 20;
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_small<kSmallThreadsFew>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_small<kSmallThreadsMany>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        // the shared-memory bitmap may use most of the SM (one CTA per individual)
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<640>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<896>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_rows<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<640>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<896>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<384, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<384, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<512, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<640, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<640, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<768, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<768, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<896, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<896, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_bitmask_vary<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_transpose, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        s->overlap_clear = env_int("GAPA_PC_OVERLAP_CLEAR", 1, 0, 1);
        s->vary_waves = env_int("GAPA_PC_VARY_WAVES", 1, 1, 1 << 20);
        s->fresh_skip = env_int("GAPA_PC_FRESH_SKIP", 0, 0, 1);
        s->mask_rows = env_int("GAPA_PC_MASK_ROWS", 1, 0, 1);
        s->mask_threads_forced = env_int("GAPA_PC_MASK_THREADS", 0, 0, 1024) / 128 * 128;
        s->uf_mode = env_int("GAPA_PC_UF", -1, -1, 1);
        GAPA_CUDA_TRY(cudaFuncSetAttribute(k_pc_uf<kUfThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        GAPA_CUDA_TRY(cudaEventCreate(&s->ev_t0));
        GAPA_CUDA_TRY(cudaEventCreate(&s->ev_t1));
        s->sweep_prefetch = env_int("GAPA_PC_SWEEP_PREFETCH", 32, 0, 1 << 20);
        s->trace = env_int("GAPA_PC_TRACE", 0, 0, 1);  // one stderr line per sweep round
        s->prefix_first4 = env_int("GAPA_PC_PREFIX_FIRST4", 1, 0, 1);  // 0: scan whole (bounded) rows in the prefix closure
        GAPA_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&s->h_counters), sizeof(PcCounters) * kMaxLanes));
        GAPA_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
        s->configured = true;
    }
    auto get_set = [&](int i, PcSet** out) -> int {
        while (static_cast<int>(s->sets.size()) <= i) {
            PcSet* fresh = nullptr;
            const int rc = pc_set_create(&fresh);
            s->sets.push_back(fresh);  // owned (and freed) by the scratch even when half-built
            GAPA_TRY(rc);
        }
        *out = s->sets[i];
        return GAPA_CUDA_OK;
    };
    const int n = ctx->n;
    const int sm = ctx->sm_count;
    // Measured crossover (tools/ab_small.sh): the per-individual kernel wins only where the bit-sliced pipeline
    // is at its launch-latency floor (~0.08 ms): n = 1e3 0.04 vs 0.08 ms at any population; n = 3e3 equal up
    // to 1024 individuals; n = 1e4 0.2-2.6 ms vs 0.1-0.17 ms.  GAPA_PC_SMALL=2 forces it wherever it fits (tests).
    const bool small_fits = n > 0 && n <= kSmallMaxN;
    const bool small_pays = n <= 2048 || (n <= 4096 && rows <= 1024);
    if (small_fits && (s->small_path == 2 || (s->small_path == 1 && small_pays))) {
        const size_t smem = sizeof(int32_t) * (2 * static_cast<size_t>(n) + ((n + 31) >> 5) + 1);
        PcSet* set0 = nullptr;
        GAPA_TRY(get_set(0, &set0));
        GAPA_TRY(set0->counters.ensure(sizeof(PcCounters)));
        PcCounters* counters = set0->counters.as<PcCounters>();
        if (!trusted) GAPA_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(PcCounters), stream));  // trusted genes cannot be out of range
        const bool fuse = vary && cols > 0;
        if (vary && !fuse) GAPA_TRY(launch_variation_spec(*vary, cols, rows, stream));
        if (rows <= 2 * sm)  // 100 rows at n = 1000: 0.03 ms with 512 threads per row, 0.05 ms with 128 (tools/ab_build.sh)
            GAPA_LAUNCH_PDL(k_pc_small<kSmallThreadsFew>, rows, kSmallThreadsFew, smem, stream, genes,
                        ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, n, static_cast<int>(ctx->m), ctx->d_edge_u,
                        ctx->d_edge_v, task, out_dev, counters, fuse ? *vary : VariationSpec{}, fuse ? 1 : 0);
        else
            GAPA_LAUNCH_PDL(k_pc_small<kSmallThreadsMany>, rows, kSmallThreadsMany, smem, stream, genes,
                        ctx->pool_identity ? nullptr : ctx->d_pool_map, ctx->pool_size, n, static_cast<int>(ctx->m), ctx->d_edge_u,
                        ctx->d_edge_v, task, out_dev, counters, fuse ? *vary : VariationSpec{}, fuse ? 1 : 0);
        if (trusted) return GAPA_CUDA_OK;
        PcCounters h{};
        GAPA_CUDA_TRY(cudaMemcpyAsync(&h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
        GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
        if (h.range_error) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
        return GAPA_CUDA_OK;
    }
    // ---- per-individual union-find in global memory (k_pc_uf) -------------------------------------------------------
    const bool uf_fits = n > 0 && sizeof(unsigned) * (static_cast<size_t>((n + 31) >> 5) + 1) <= 200 * 1024;  // removed bitmap in shared memory
    auto launch_uf = [&](GeneRows genes, const VariationSpec* vary, double* out_dev, bool trusted) -> int {
        const size_t smem = sizeof(unsigned) * (static_cast<size_t>((n + 31) >> 5) + 1);
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pc_uf<kUfThreads>, kUfThreads, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
        const int grid = std::max(1, std::min(rows, sm * per_sm));
        GAPA_TRY(s->uf_scratch.ensure(sizeof(int32_t) * 2 * static_cast<size_t>(n) * grid));
        PcSet* set0 = nullptr;
        GAPA_TRY(get_set(0, &set0));
        GAPA_TRY(set0->counters.ensure(sizeof(PcCounters)));
        PcCounters* counters = set0->counters.as<PcCounters>();
        if (!trusted) GAPA_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(PcCounters), stream));
        const bool fuse = vary && cols > 0;
        if (vary && !fuse) GAPA_TRY(launch_variation_spec(*vary, cols, rows, stream));
        GAPA_LAUNCH(k_pc_uf<kUfThreads>, grid, kUfThreads, smem, stream, genes, ctx->pool_identity ? nullptr : ctx->d_pool_map,
                    ctx->pool_size, n, static_cast<int>(ctx->m), ctx->d_edge_u, ctx->d_edge_v, task, out_dev, counters,
                    fuse ? *vary : VariationSpec{}, fuse ? 1 : 0, rows, s->uf_scratch.as<int32_t>());
        if (trusted) return GAPA_CUDA_OK;
        PcCounters h{};
        GAPA_CUDA_TRY(cudaMemcpyAsync(&h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
        GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
        if (h.range_error) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
        // the clean-slot bookkeeping of the pipeline's speculative schedule does not survive a memset of the counters
        set0->clean_slots = 0;
        return GAPA_CUDA_OK;
    };
    if (uf_fits && s->uf_mode == 1) return launch_uf(genes, vary, out_dev, trusted);

    // ---- the bit-sliced pipeline ------------------------------------------------------------------------------------
    auto pipeline = [&](GeneRows genes, const VariationSpec* vary, double* out_dev, bool trusted, bool* slow) -> int {
        GAPA_TRY(ensure_order(ctx, s));
        // Lanes: whole 64-individual groups, at most lane_rows individuals and at most what the scratch budget allows
        // (alive + reached + entry_of = 20 B per vertex and group, bitmaps 8 B per vertex and group) for every set in flight.
        const size_t budget = static_cast<size_t>(env_int("GAPA_SCRATCH_MB", 24 * 1024, 1, 1 << 20)) << 20;
        const int all_groups = (rows + kBits - 1) / kBits;
        const int budget_groups = static_cast<int>(std::min<size_t>(1023, std::max<size_t>(1, budget / (28ull * std::max(n, 1)))));
        int lane_groups = std::max(1, std::min(s->lane_rows / kBits, all_groups));
        int streams = std::min(s->lane_streams, (all_groups + lane_groups - 1) / lane_groups);
        if (lane_groups * streams > budget_groups) {
            streams = std::max(1, std::min(streams, budget_groups / lane_groups));
            lane_groups = std::max(1, std::min(lane_groups, budget_groups / streams));
        }
        if (lane_groups >= kPack) lane_groups = lane_groups / kPack * kPack;  // whole 32-byte records
        const int total_lanes = (all_groups + lane_groups - 1) / lane_groups;
        PcLaneJob job{task, genes, 0, 0, out_dev, trusted, vary};
        auto lane_many = [&](int crows) {
            const int sg = ((crows + kBits - 1) / kBits + kPack - 1) / kPack;
            return static_cast<unsigned>(std::max<size_t>(8192, static_cast<size_t>(sg) * kPack * std::max(n, 1) / 512));
        };
        for (int wave0 = 0; wave0 < total_lanes; wave0 += kMaxLanes) {
            const int lanes = std::min(kMaxLanes, total_lanes - wave0);
            const bool forked = lanes > 1 && streams > 1;
            const int spec = s->spec_rounds;
            if (forked) {
                GAPA_CUDA_TRY(cudaEventRecord(s->ev_fork, stream));
                for (int j = 0; j < std::min(streams, lanes); ++j) {
                    PcSet* set = nullptr;
                    GAPA_TRY(get_set(j, &set));
                    GAPA_CUDA_TRY(cudaStreamWaitEvent(set->stream, s->ev_fork, 0));
                }
            }
            std::vector<int> redo;
            for (int i = 0; i < lanes; ++i) {
                PcSet* set = nullptr;
                GAPA_TRY(get_set(forked ? i % streams : 0, &set));
                job.row0 = (wave0 + i) * lane_groups * kBits;
                job.crows = std::min(rows - job.row0, lane_groups * kBits);
                GAPA_TRY(pc_run_lane(ctx, s, set, job, forked ? set->stream : stream, spec, &s->h_counters[i], nullptr));
            }
            if (forked)
                for (int j = 0; j < std::min(streams, lanes); ++j) {
                    GAPA_CUDA_TRY(cudaEventRecord(s->sets[j]->ev_done, s->sets[j]->stream));
                    GAPA_CUDA_TRY(cudaStreamWaitEvent(stream, s->sets[j]->ev_done, 0));
                }
            if (spec == 0) continue;  // the host-driven loop has already seen every lane's counters
            // ONE host look at the counters per evaluation, after everything has been enqueued
            GAPA_CUDA_TRY(cudaStreamSynchronize(stream));
            for (int i = 0; i < lanes; ++i) {
                const PcCounters& h = s->h_counters[i];
                const int crows = std::min(rows - (wave0 + i) * lane_groups * kBits, lane_groups * kBits);
                if (h.range_error) return fail(GAPA_CUDA_E_RANGE, "perturbation: gene id out of range");
                if (s->trace)
                    std::fprintf(stderr, "pc_eval lane %d (speculative, %d round(s)): entries %u slots %u overflow %d changed %d incomplete %u deferred %d\n",
                                 wave0 + i, spec, h.n_entries, h.n_slots, h.overflow, h.changed, h.n_incomplete, h.deferred);
                if (h.phase2_skipped) s->phase2_big = true;
                if (h.overflow || h.deferred || h.phase2_skipped || (h.changed && h.n_entries > lane_many(crows))) redo.push_back(i);
            }
            // Lanes whose speculative schedule was not enough are redone with the host-driven loop (a later lane may have
            // reused the set's buffers, so they start over; variation is a pure function of the parents, so rebuilding the
            // children writes the same genes).  What the loop needed becomes the next evaluations' speculative schedule.
            if (!redo.empty()) *slow = true;
            for (int i : redo) {
                PcSet* set = nullptr;
                GAPA_TRY(get_set(0, &set));
                job.row0 = (wave0 + i) * lane_groups * kBits;
                job.crows = std::min(rows - job.row0, lane_groups * kBits);
                int used = 0;
                GAPA_TRY(pc_run_lane(ctx, s, set, job, stream, 0, nullptr, &used));
                s->spec_rounds = used <= 6 ? std::max(s->spec_rounds, used) : 0;
            }
        }
        return GAPA_CUDA_OK;
    };
    bool slow = false;
    GAPA_TRY(pipeline(genes, vary, out_dev, trusted, &slow));
    if (slow && uf_fits && s->uf_mode < 0 && rows >= 64) {
        // This graph made the pipeline fall back to its host-driven loop (no hub core, or a large diameter).  Decide ONCE,
        // by measurement on this very batch (its children exist by now, so no variation is repeated): the pipeline as it
        // will run from now on (it has just learned its schedule) against the per-individual union-find.
        GAPA_TRY(s->uf_out.ensure(sizeof(double) * static_cast<size_t>(rows)));
        float t_pipe = 0.f, t_uf = 0.f;
        bool again = false;
        GAPA_CUDA_TRY(cudaEventRecord(s->ev_t0, stream));
        GAPA_TRY(pipeline(genes, nullptr, s->uf_out.as<double>(), true, &again));
        GAPA_CUDA_TRY(cudaEventRecord(s->ev_t1, stream));
        GAPA_CUDA_TRY(cudaEventSynchronize(s->ev_t1));
        GAPA_CUDA_TRY(cudaEventElapsedTime(&t_pipe, s->ev_t0, s->ev_t1));
        GAPA_CUDA_TRY(cudaEventRecord(s->ev_t0, stream));
        GAPA_TRY(launch_uf(genes, nullptr, s->uf_out.as<double>(), true));
        GAPA_CUDA_TRY(cudaEventRecord(s->ev_t1, stream));
        GAPA_CUDA_TRY(cudaEventSynchronize(s->ev_t1));
        GAPA_CUDA_TRY(cudaEventElapsedTime(&t_uf, s->ev_t0, s->ev_t1));
        s->uf_mode = t_uf < t_pipe ? 1 : 0;
        if (s->trace) std::fprintf(stderr, "pc_eval: %d rows, pipeline %.3f ms, union-find %.3f ms -> %s\n", rows, t_pipe, t_uf, s->uf_mode ? "union-find" : "pipeline");
    }
    return GAPA_CUDA_OK;
}

void pc_free(gapa_cuda_ctx* ctx) {
    if (!ctx->pc) return;
    PcScratch* s = ctx->pc;
    for (PcSet* set : s->sets) {
        if (!set) continue;
        for (DevBuf* b : {&set->removed, &set->removed_count, &set->alive, &set->reached, &set->entry_of, &set->unreached, &set->counters,
                          &set->block_done, &set->left_v, &set->left_g, &set->left_w, &set->left_base, &set->parent, &set->comp_size,
                          &set->pc_extra, &set->mcn_extra})
            b->release();
        if (set->aux) cudaStreamDestroy(set->aux);
        if (set->stream) cudaStreamDestroy(set->stream);
        if (set->ev_pass_begin) cudaEventDestroy(set->ev_pass_begin);
        if (set->ev_cleared) cudaEventDestroy(set->ev_cleared);
        if (set->ev_done) cudaEventDestroy(set->ev_done);
        delete set;
    }
    for (DevBuf* b : {&s->nbr4, &s->ord_row_ptr, &s->ord_col_idx, &s->ord_gene_map, &s->uf_scratch, &s->uf_out}) b->release();
    if (s->ev_t0) cudaEventDestroy(s->ev_t0);
    if (s->ev_t1) cudaEventDestroy(s->ev_t1);
    if (s->h_counters) cudaFreeHost(s->h_counters);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    delete s;
    ctx->pc = nullptr;
}

}  // namespace gapa_b200
