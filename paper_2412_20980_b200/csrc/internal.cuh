// Internal declarations shared by the .cu files behind include/gapa_cuda.h.
// sm_100a only; nothing here is part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <utility>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "gapa_cuda.h"

namespace gapa_b200 {

// ---- error plumbing --------------------------------------------------------------
int fail(int code, const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

#define GAPA_CUDA_TRY(expr)                                                                     \
    do {                                                                                        \
        cudaError_t err__ = (expr);                                                             \
        if (err__ != cudaSuccess)                                                               \
            return ::gapa_b200::fail(err__ == cudaErrorMemoryAllocation ? GAPA_CUDA_E_NOMEM     \
                                                                        : GAPA_CUDA_E_CUDA,     \
                                     "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(err__), \
                                     __FILE__, __LINE__);                                       \
    } while (0)

#define GAPA_TRY(expr)               \
    do {                             \
        int rc__ = (expr);           \
        if (rc__ != GAPA_CUDA_OK) return rc__; \
    } while (0)

// Programmatic dependent launch (sm_90+): a kernel launched with GAPA_LAUNCH_PDL may be SCHEDULED while the kernel before it
// on the stream is still running — its CTAs become resident, run whatever does not depend on that kernel (shared-memory
// initialisation) and block in griddep_wait() until the predecessor has completed and its writes are visible.  The
// predecessor allows this with griddep_launch() at its top.  Where a generation is two or three launches of 5-15 us the
// ~2 us between dependent launches are a tenth of it (C1: 38.9 k -> 44.8 k generations/s in the library loop, tools/ab_pdl.sh).
// EVERY kernel launched this way must call griddep_wait() before it reads or writes anything another kernel touches;
// without the launch attribute (GAPA_PDL=0) both calls are no-ops.
#ifdef __CUDACC__
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
extern int g_pdl;           // GAPA_PDL (default 1): 0 launches everything the ordinary way (ctx.cu)
extern long g_pdl_max_ctas;  // GAPA_PDL_MAX_CTAS: only grids up to this many CTAs are launched programmatically (0 = all)
inline bool pdl_allowed(dim3 grid) {
    return g_pdl && (g_pdl_max_ctas <= 0 || static_cast<long>(grid.x) * grid.y * grid.z <= g_pdl_max_ctas);
}
#define GAPA_LAUNCH_PDL(kernel_, grid_, block_, smem_, stream_, ...)                                  \
    do {                                                                                             \
        cudaLaunchConfig_t cfg__{};                                                                  \
        cfg__.gridDim = dim3(grid_);                                                                 \
        cfg__.blockDim = dim3(block_);                                                               \
        cfg__.dynamicSmemBytes = (smem_);                                                            \
        cfg__.stream = (stream_);                                                                    \
        cudaLaunchAttribute attr__{};                                                                \
        attr__.id = cudaLaunchAttributeProgrammaticStreamSerialization;                              \
        attr__.val.programmaticStreamSerializationAllowed = 1;                                       \
        cfg__.attrs = &attr__;                                                                       \
        cfg__.numAttrs = ::gapa_b200::pdl_allowed(cfg__.gridDim) ? 1 : 0;                            \
        GAPA_CUDA_TRY(cudaLaunchKernelEx(&cfg__, kernel_, __VA_ARGS__));                             \
        ::gapa_b200::g_launches.fetch_add(1, std::memory_order_relaxed);                             \
    } while (0)

// Every launch of the library counts itself, checks the launch error and allows programmatic dependent launch: EVERY kernel
// starts with griddep_launch(); griddep_wait(); (two persistent kernels do their shared-memory set-up before the wait).
#define GAPA_LAUNCH(kernel_, grid_, block_, smem_, stream_, ...) GAPA_LAUNCH_PDL(kernel_, grid_, block_, smem_, stream_, __VA_ARGS__)

// ---- device buffer that grows, never shrinks ---------------------------------------
struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return GAPA_CUDA_OK;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 8 + 256;
        GAPA_CUDA_TRY(cudaMalloc(&ptr, want));
        cap = want;
        return GAPA_CUDA_OK;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

// ---- RNG twin of include/gapa/rng.hpp ---------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:8-13
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t generation, uint64_t role,
                                                        uint64_t row) {  // rng.hpp:59-65
    uint64_t key = mix64(seed);
    key = mix64(key ^ generation);
    key = mix64(key ^ role);
    return mix64(key ^ row);
}
// j-th draw (j >= 1) of the stream: the reference pre-increments its counter (rng.hpp:21),
// which makes draws random-access in j — one thread per (row, column) needs no state.
__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t key, uint64_t j) {
    return mix64(key + 0x632BE59BD9B4E019ull * j);
}
// next_index (rng.hpp:28-31): high 64 bits of u64 x u32
__device__ __forceinline__ uint32_t draw_index(uint64_t key, uint64_t j, uint32_t bound) {
    return static_cast<uint32_t>(__umul64hi(draw_u64(key, j), static_cast<uint64_t>(bound)));
}
// next_unit (rng.hpp:24): both steps are exact in FP64
__device__ __forceinline__ double draw_unit(uint64_t key, uint64_t j) {
    return __ull2double_rn(draw_u64(key, j) >> 11) * 0x1.0p-53;
}
// next_bernoulli(p) (rng.hpp:33) is  (u >> 11) * 2^-53 < p.  The left side is an
// exactly representable multiple of 2^-53, so the test equals the integer test
// (u >> 11) < ceil(p * 2^53); the threshold is computed once on the host.
uint64_t bernoulli_threshold(double p);
__device__ __forceinline__ bool draw_bernoulli(uint64_t key, uint64_t j, uint64_t threshold) {
    return (draw_u64(key, j) >> 11) < threshold;
}

// Order-preserving 64-bit key of a fitness value: key(x) < key(y)  <=>  x is BETTER than y (direction folded
// in), key(x) == key(y) <=> x == y (-0.0 and +0.0 share a key).  The O(s^2) counting kernels of selection and
// elitism compare these integers instead of doubles (two integer instructions per compare instead of FP64
// set-predicates and a direction select).  NaN is reported separately and never ranked.
// record_generation (modes.cpp:35-43) by ONE block of any size: best = front, mean = SEQUENTIAL sum / s so that non-integer
// fitness reproduces std::accumulate bit for bit.  Shared by k_ga_stats (run.cu) and the statistics block of
// k_ga_weights (ga_kernels.cu: the previous generation's statistics ride on the next generation's selection launch).
struct GaStatsSmem {
    double stage[4096];
    double warp_sum[32];
    int not_exact;
};
__device__ __forceinline__ void ga_stats_block(const double* __restrict__ fit, int s, double* best, double* mean, GaStatsSmem& sm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) sm.not_exact = 0;
    __syncthreads();
    // Integer-valued fitness whose running sums stay below 2^53 (PC, MCN) adds exactly in any order.
    double local = 0.0;
    const double bound = 9007199254740992.0 / static_cast<double>(s);
    for (int i = tid; i < s; i += nt) {
        const double x = fit[i];
        if (!(x == floor(x)) || !(fabs(x) < bound)) sm.not_exact = 1;
        local += x;
    }
    __syncthreads();
    if (!sm.not_exact) {
        for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
        if ((tid & 31) == 0) sm.warp_sum[tid >> 5] = local;
        __syncthreads();
        if (tid < 32) {
            double v = tid < (nt >> 5) ? sm.warp_sum[tid] : 0.0;
            for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
            if (tid == 0) {
                *best = fit[0];
                *mean = v / static_cast<double>(s);
            }
        }
        return;
    }
    // general FP64 fitness: the reference's left-to-right std::accumulate, staged through shared memory
    double sum = 0.0;
    for (int base = 0; base < s; base += 4096) {
        const int lim = min(4096, s - base);
        for (int i = tid; i < lim; i += nt) sm.stage[i] = fit[base + i];
        __syncthreads();
        if (tid == 0)
            for (int i = 0; i < lim; ++i) sum += sm.stage[i];
        __syncthreads();
    }
    if (tid == 0) {
        *best = fit[0];
        *mean = sum / static_cast<double>(s);
    }
}

__device__ __forceinline__ unsigned long long order_key(double x, int minimize) {
    if (x == 0.0) x = 0.0;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned long long k = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending with x
    return minimize ? k : ~k;
}

// ---- gene matrix view -----------------------------------------------------------------
// Row r of a batch lives at base + slot[r] * cols (slot == nullptr: the dense row-major matrix of
// population.hpp:12-40).  The in-library generation loop keeps parents and children in one pool of
// 2s row slots and hands evaluators a slot table, so elitism never copies a genome.
struct GeneRows {
    const int32_t* base;
    const int32_t* slot;
    int cols;
    __host__ __device__ const int32_t* row(int r) const {
        return base + static_cast<size_t>(slot ? slot[r] : r) * cols;
    }
    GeneRows from(int r0) const {  // the same batch starting at row r0
        return slot ? GeneRows{base, slot + r0, cols} : GeneRows{base + static_cast<size_t>(r0) * cols, nullptr, cols};
    }
};

// ---- pinned staging ring (ctx.cu): pageable host buffers of the host-buffer entry point ----------------------
static constexpr size_t kPinnedRingMinBytes = 8u << 20;   // smaller pageable batches take the plain copy
static constexpr size_t kPinnedSliceBytes = 16u << 20;  // default slice; GAPA_PINNED_SLICE_MB overrides (PinnedRing::slice_bytes)
struct PinnedRing {
    static constexpr int kSlots = 4;
    char* buf[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    int next = 0;
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable wake, idle;
    std::atomic<uint64_t> generation{0};
    std::atomic<int> finished{0};
    int cur_slot = 0;
    size_t cur_len = 0;
    bool in_flight = false;  // between begin() and end()
    bool stop = false;
    size_t slice_bytes = kPinnedSliceBytes;
    bool nt_copy = false;  // GAPA_PINNED_RING_COPY=nt: non-temporal stores into the pinned slot instead of the C library's copy
    const char* job_src = nullptr;
    char* job_dst = nullptr;
    size_t job_len = 0;
    PinnedRing();
    ~PinnedRing();
    void work(int index, int count);
    int begin(const void* src_host, size_t len);
    int end(void* dst_dev, cudaStream_t copy_stream);
};

// ---- context -------------------------------------------------------------------------
struct PcScratch;   // pc_kernels.cu
struct LpaScratch;  // lpa_kernels.cu
struct CdaScratch;  // cda_kernels.cu
struct SixScratch;  // sixdst_kernels.cu

}  // namespace gapa_b200

struct gapa_cuda_ctx {
    int device = 0;
    int32_t n = 0;
    int64_t m = 0;
    int sm_count = 148;
    // host copies of the CSR (pool mapping, validation)
    std::vector<int32_t> h_row_ptr, h_col_idx, h_edge_id;
    // device CSR, shared by every individual, read-only
    int32_t* d_row_ptr = nullptr;   // n + 1
    int32_t* d_col_idx = nullptr;   // 2m, ascending per row
    int32_t* d_edge_id = nullptr;   // 2m, rank of the undirected edge in (u,v) order
    int32_t* d_edge_u = nullptr;    // m, endpoints by edge rank
    int32_t* d_edge_v = nullptr;
    int32_t* d_by_degree = nullptr; // n, vertices by descending degree (BFS source candidates)
    // pool
    int pool_kind = -1;
    int32_t pool_size = 0;
    bool pool_identity = true;
    int32_t* d_pool_map = nullptr;  // gene id -> node id / edge rank when not identity
    std::vector<int32_t> h_pool_map;  // host copy of the same map (empty when identity)
    unsigned long long pool_version = 0;  // bumped by gapa_cuda_pool_set
    // EdgeAddition pool (gene_pool.cpp:57-60, :81-87): gene id -> endpoints of the pair it adds;
    // (-1, -1) when the pair is already an edge of the graph (setting a set bit is a no-op)
    int32_t* d_add_u = nullptr;
    int32_t* d_add_v = nullptr;
    // link-prediction split
    int32_t T = 0, P = 0;
    int32_t* d_pairs = nullptr;     // (T + P) x 2, test pairs first
    int lp_score = 0;               // GAPA_LP_SCORE_RA / _CN
    bool flip_canonical = false;    // EDGE_FLIP pool over all pairs: genes are unranked on the device (no table)
    // work stream + timing
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;          // H2D of the host-buffer entry point, overlapped with compute
    std::vector<cudaEvent_t> copy_events, chunk_events;
    gapa_b200::PinnedRing* ring = nullptr;           // created by the first large pageable batch
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
    float last_eval_ms = 0.f;
    // FitnessFunction methods are const and called concurrently from worker threads in the
    // reference (modes.cpp:85,209); evaluations on one context are serialised here.
    std::mutex mu;
    // staging for the host-buffer entry point
    gapa_b200::DevBuf genes_stage, out_stage, status_buf;
    int32_t* h_status = nullptr;    // pinned
    // the caller's slot pool whose parent rows were last checked to hold genes inside the pool (fused variation entry)
    const void* validated_pool = nullptr;
    size_t validated_cells = 0;
    unsigned long long validated_version = ~0ull;
    gapa_b200::PcScratch* pc = nullptr;
    gapa_b200::LpaScratch* lpa = nullptr;
    gapa_b200::CdaScratch* cda = nullptr;
    gapa_b200::SixScratch* six = nullptr;
};

namespace gapa_b200 {

// per-task evaluators: genes/out on the device, work enqueued on ctx->stream_for(stream)
// `trusted` = the genes were produced by this library's own operators (always inside the pool),
// so evaluators that need no other host decision skip the range-status readback and stay
// asynchronous.
// `vary` (optional): the rows are children that do not exist yet — the evaluator builds them into
// their slots first (fused with the mask build where the kernel structure allows it).
struct VariationSpec;
int pc_eval(gapa_cuda_ctx* ctx, int task, GeneRows genes, int rows, double* out_dev, cudaStream_t stream,
            bool trusted = false, const VariationSpec* vary = nullptr);
int launch_variation_spec(const VariationSpec& spec, int k, int rows, cudaStream_t stream);  // slot_kernels.cu
int lpa_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, bool trusted = false);
int cda_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream,
             int32_t* owner_out_dev = nullptr);  // optional [rows x n]: smallest member of each vertex's community
const double* lpa_last_scores(const gapa_cuda_ctx* ctx);  // scores of the last evaluated chunk: per row T test then P probe
int sixdst_eval(gapa_cuda_ctx* ctx, GeneRows genes, int rows, double* out_dev, cudaStream_t stream, bool trusted = false);
void pc_free(gapa_cuda_ctx* ctx);
void sixdst_free(gapa_cuda_ctx* ctx);
void lpa_free(gapa_cuda_ctx* ctx);
void cda_free(gapa_cuda_ctx* ctx);

}  // namespace gapa_b200
