// Context management and the fitness entry points of include/gapa_cuda.h.
//
// One gapa_cuda_ctx = one GPU's copy of the read-only problem: the CSR that
// replaces the reference's dense BitMatrix (graph.cpp:47-54), the gene pool
// (gene_pool.cpp:69-96) and, for the link-prediction task, the split
// (link_prediction.hpp:16-21).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "internal.cuh"
#include "variation.cuh"

namespace gapa_b200 {

static thread_local std::string t_error;
std::atomic<uint64_t> g_launches{0};
int g_pdl = [] {
    const char* raw = std::getenv("GAPA_PDL");
    return raw && raw[0] == '0' ? 0 : 1;
}();
long g_pdl_max_ctas = [] {
    const char* raw = std::getenv("GAPA_PDL_MAX_CTAS");
    return raw ? std::atol(raw) : 2368L;  // 16 CTAs per SM: measured, tools/ab_pdl_ctas.sh
}();

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_error = buf;
    return code;
}

uint64_t bernoulli_threshold(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return 1ull << 53;
    return static_cast<uint64_t>(std::ceil(p * 9007199254740992.0));  // exact scaling by 2^53
}

static int upload_i32(const std::vector<int32_t>& h, int32_t** d) {
    GAPA_CUDA_TRY(cudaMalloc(d, sizeof(int32_t) * std::max<size_t>(h.size(), 1)));
    if (!h.empty()) GAPA_CUDA_TRY(cudaMemcpy(*d, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice));
    return GAPA_CUDA_OK;
}


// ---- pinned staging ring for pageable host buffers ---------------------------------------------------------
// push(): wait until the slot's previous H2D has drained, copy the slice into the slot with all copy threads, enqueue
// the H2D.  With kSlots slices in flight the host copy of slice i+1 overlaps the DMA of slice i.
// Copy into the pinned slot with non-temporal stores: the destination is only ever read by the DMA engine, so pulling
// its lines into the cache first (read-for-ownership) is a third of the memory traffic of the copy for nothing.
// GAPA_PINNED_RING_COPY=nt selects it; the default is the C library's copy, which measures the same or better since the
// workers spin (tools/probe_pageable.py, tools/sweep_ring.py).
#if defined(__x86_64__)
#include <immintrin.h>
__attribute__((target("avx2"))) static void copy_nt_avx2(char* dst, const char* src, size_t len) {
    size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
    if (head > len) head = len;
    std::memcpy(dst, src, head);
    dst += head; src += head; len -= head;
    const size_t blocks = len / 128;
    for (size_t i = 0; i < blocks; ++i) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 96));
        _mm_prefetch(src + 1024, _MM_HINT_NTA);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + 96), d);
        src += 128; dst += 128;
    }
    _mm_sfence();
    std::memcpy(dst, src, len - blocks * 128);
}
#endif
static void ring_copy(char* dst, const char* src, size_t len, bool nt) {
#if defined(__x86_64__)
    if (nt && len >= 4096 && __builtin_cpu_supports("avx2")) {
        copy_nt_avx2(dst, src, len);
        return;
    }
#endif
    (void)nt;
    std::memcpy(dst, src, len);
}

PinnedRing::PinnedRing() {
    if (const char* raw = std::getenv("GAPA_PINNED_RING_COPY")) nt_copy = raw[0] == 'n';
    if (const char* raw = std::getenv("GAPA_PINNED_SLICE_MB")) slice_bytes = static_cast<size_t>(std::max(1, std::min(256, std::atoi(raw)))) << 20;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    // measured on the B200 box (16 host cores, one socket; tools/probe_pageable.py, tools/sweep_ring.py; 819 MB batch = C4):
    //   plain cudaMemcpyAsync from pageable memory 10.8 GB/s; the same batch from pinned memory 54 GB/s (the PCIe rate);
    //   first ring (blocking push per slice, condition variables): memcpy 20.4 / 21.6 GB/s at 4 / 8 threads, non-temporal
    //   stores 25.7 / 33.4 GB/s;
    //   this ring (spinning workers, begin/end split so that the next slice is copied while the previous one is submitted
    //   and the chunk's kernels are enqueued): memcpy 44.5 GB/s at 8 threads and 16 MB slots (18.4 ms per batch = 222 k
    //   evals/s; 37.8 - 44.7 GB/s over 6 - 12 threads x 8 - 32 MB), non-temporal stores 43.2 GB/s -> the C library's copy,
    //   8 threads.  16 spinning workers on 16 cores starve the caller and the driver's threads: 4.9 GB/s — hence cores / 2.
    //   The host alone copies 73 GB/s (8 threads, no DMA running); copy + DMA together move 3 x 819 MB through its memory.
    //   Pinning the caller's pages in place instead (cudaHostRegister per slice) manages 1.6 - 7.7 GB/s
    //   (tools/probe_hostregister.py) and is no alternative.
    int count = static_cast<int>(std::min(8u, std::max(1u, hw / 2)));
    if (const char* raw = std::getenv("GAPA_PINNED_RING_THREADS")) count = std::max(1, std::min(64, std::atoi(raw)));
    for (int t = 0; t < count; ++t) workers.emplace_back([this, t, count] { work(t, count); });
}
PinnedRing::~PinnedRing() {
    {
        std::lock_guard<std::mutex> lock(mu);
        stop = true;
        generation.fetch_add(1, std::memory_order_release);
    }
    wake.notify_all();
    for (std::thread& w : workers) w.join();
    for (int i = 0; i < kSlots; ++i) {
        if (done[i]) cudaEventDestroy(done[i]);
        if (buf[i]) cudaFreeHost(buf[i]);
    }
}
// A worker SPINS on the job counter for a short while after each slice (a batch is a few dozen slices a fraction of a
// millisecond apart: a condition-variable wake-up per slice and thread costs more than the copy it waits for) and goes
// to sleep on the condition variable when nothing arrives for ~1 ms.
void PinnedRing::work(int index, int count) {
    uint64_t seen = 0;
    for (;;) {
        bool got = false;
        for (int spin = 0; spin < 200000 && !got; ++spin) {
            got = generation.load(std::memory_order_acquire) != seen;
#if defined(__x86_64__)
            if (!got) __builtin_ia32_pause();
#endif
        }
        if (!got) {
            std::unique_lock<std::mutex> lock(mu);
            wake.wait(lock, [&] { return generation.load(std::memory_order_acquire) != seen; });
        }
        seen = generation.load(std::memory_order_acquire);
        if (stop) return;
        const char* src = job_src;
        char* dst = job_dst;
        const size_t len = job_len;
        const size_t part = ((len + count - 1) / count + 4095) & ~size_t{4095};
        const size_t lo = std::min(len, part * index), hi = std::min(len, lo + part);
        if (hi > lo) ring_copy(dst + lo, src + lo, hi - lo, nt_copy);
        finished.fetch_add(1, std::memory_order_release);
    }
}
// begin(): wait until the slot's previous H2D has drained and hand the slice to the copy threads — returns at once;
// end(): wait for the copy threads, enqueue the H2D.  Between the two the caller enqueues the kernels of the previous chunk
// and the previous slice's DMA runs: the host copy of slice i+1 overlaps both.
int PinnedRing::begin(const void* src_host, size_t len) {
    if (in_flight) {  // a previous call left after an error between begin() and end(): let its copy finish first
        const int count = static_cast<int>(workers.size());
        while (finished.load(std::memory_order_acquire) != count) std::this_thread::yield();
        in_flight = false;
    }
    const int slot = next++ % kSlots;
    if (!buf[slot]) {
        GAPA_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&buf[slot]), slice_bytes));
        GAPA_CUDA_TRY(cudaEventCreateWithFlags(&done[slot], cudaEventDisableTiming));
    } else {
        GAPA_CUDA_TRY(cudaEventSynchronize(done[slot]));
    }
    cur_slot = slot;
    cur_len = len;
    job_src = static_cast<const char*>(src_host);
    job_dst = buf[slot];
    job_len = len;
    finished.store(0, std::memory_order_relaxed);
    {
        std::lock_guard<std::mutex> lock(mu);  // a worker that is going to sleep sees the new job or gets the notification
        generation.fetch_add(1, std::memory_order_release);
    }
    wake.notify_all();
    in_flight = true;
    return GAPA_CUDA_OK;
}
int PinnedRing::end(void* dst_dev, cudaStream_t copy_stream) {
    const int count = static_cast<int>(workers.size());
    while (finished.load(std::memory_order_acquire) != count) {
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    in_flight = false;
    GAPA_CUDA_TRY(cudaMemcpyAsync(dst_dev, buf[cur_slot], cur_len, cudaMemcpyHostToDevice, copy_stream));
    GAPA_CUDA_TRY(cudaEventRecord(done[cur_slot], copy_stream));
    return GAPA_CUDA_OK;
}

// Edge rank of {u, v} in the (u,v)-sorted edge list, or -1.
static int32_t edge_rank(const gapa_cuda_ctx* c, int32_t u, int32_t v) {
    if (u < 0 || v < 0 || u >= c->n || v >= c->n || u == v) return -1;
    const int32_t* b = c->h_col_idx.data() + c->h_row_ptr[u];
    const int32_t* e = c->h_col_idx.data() + c->h_row_ptr[u + 1];
    const int32_t* it = std::lower_bound(b, e, v);
    if (it == e || *it != v) return -1;
    return c->h_edge_id[it - c->h_col_idx.data()];
}

static int finish_create(gapa_cuda_ctx* c, int device, gapa_cuda_ctx** out) {
    const int32_t n = c->n;
    const int64_t m = c->m;
    // edge ranks: (u, v), u < v, in row-major CSR order == lexicographic order
    c->h_edge_id.assign(static_cast<size_t>(2 * m), 0);
    std::vector<int32_t> eu(static_cast<size_t>(m)), ev(static_cast<size_t>(m));
    int32_t next = 0;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t i = c->h_row_ptr[u]; i < c->h_row_ptr[u + 1]; ++i) {
            const int32_t v = c->h_col_idx[i];
            if (v > u) {
                c->h_edge_id[i] = next;
                eu[next] = u;
                ev[next] = v;
                ++next;
            }
        }
    if (next != m) {
        delete c;
        return fail(GAPA_CUDA_E_INVALID, "graph: CSR is not symmetric (found %d forward edges, expected %lld)", next,
                    static_cast<long long>(m));
    }
    for (int32_t u = 0; u < n; ++u)
        for (int32_t i = c->h_row_ptr[u]; i < c->h_row_ptr[u + 1]; ++i) {
            const int32_t v = c->h_col_idx[i];
            if (v < u) {
                const int32_t* b = c->h_col_idx.data() + c->h_row_ptr[v];
                const int32_t* e = c->h_col_idx.data() + c->h_row_ptr[v + 1];
                const int32_t* it = std::lower_bound(b, e, u);
                if (it == e || *it != u) {
                    delete c;
                    return fail(GAPA_CUDA_E_INVALID, "graph: CSR is not symmetric at (%d, %d)", u, v);
                }
                c->h_edge_id[i] = c->h_edge_id[it - c->h_col_idx.data()];
            }
        }
    // BFS source candidates: vertices by descending degree, ties by id
    std::vector<int32_t> by_degree(static_cast<size_t>(n));
    std::iota(by_degree.begin(), by_degree.end(), 0);
    std::stable_sort(by_degree.begin(), by_degree.end(), [&](int32_t a, int32_t b) {
        return c->h_row_ptr[a + 1] - c->h_row_ptr[a] > c->h_row_ptr[b + 1] - c->h_row_ptr[b];
    });

    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
        delete c;
        return fail(GAPA_CUDA_E_CUDA, "no CUDA device available (this library has no CPU fallback)");
    }
    if (device < 0 || device >= count) {
        delete c;
        return fail(GAPA_CUDA_E_INVALID, "device %d out of range (%d visible)", device, count);
    }
    c->device = device;
    int rc = GAPA_CUDA_OK;
    auto body = [&]() -> int {
        GAPA_CUDA_TRY(cudaSetDevice(device));
        GAPA_CUDA_TRY(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        GAPA_TRY(upload_i32(c->h_row_ptr, &c->d_row_ptr));
        GAPA_TRY(upload_i32(c->h_col_idx, &c->d_col_idx));
        GAPA_TRY(upload_i32(c->h_edge_id, &c->d_edge_id));
        GAPA_TRY(upload_i32(eu, &c->d_edge_u));
        GAPA_TRY(upload_i32(ev, &c->d_edge_v));
        GAPA_TRY(upload_i32(by_degree, &c->d_by_degree));
        {  // the work stream outranks the evaluators' side streams (background clears, pc_kernels.cu)
            int least = 0, greatest = 0;
            GAPA_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            GAPA_CUDA_TRY(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest));
        }
        GAPA_CUDA_TRY(cudaEventCreate(&c->ev_start));
        GAPA_CUDA_TRY(cudaEventCreate(&c->ev_stop));
        GAPA_CUDA_TRY(cudaMallocHost(&c->h_status, 64 * sizeof(int32_t)));
        GAPA_TRY(c->status_buf.ensure(64 * sizeof(int32_t)));
        return GAPA_CUDA_OK;
    };
    rc = body();
    if (rc != GAPA_CUDA_OK) {
        gapa_cuda_destroy(c);
        return rc;
    }
    // default pool: node removal, identity (build_gene_pool NodeRemoval, gene_pool.cpp:89-92)
    c->pool_kind = GAPA_POOL_NODE_REMOVAL;
    c->pool_size = n;
    c->pool_identity = true;
    *out = c;
    return GAPA_CUDA_OK;
}

}  // namespace gapa_b200

using namespace gapa_b200;

extern "C" {

const char* gapa_cuda_last_error(void) { return t_error.c_str(); }
int gapa_cuda_abi_version(void) { return GAPA_CUDA_ABI_VERSION; }
uint64_t gapa_cuda_launch_count(void) { return g_launches.load(); }

int gapa_cuda_device_count(int* count) {
    if (!count) return fail(GAPA_CUDA_E_INVALID, "device_count: null output");
    *count = 0;
    GAPA_CUDA_TRY(cudaGetDeviceCount(count));
    return GAPA_CUDA_OK;
}

int gapa_cuda_graph_create(int32_t n, int64_t m, const int32_t* uv, int device, gapa_cuda_ctx** out) {
    if (!out) return fail(GAPA_CUDA_E_INVALID, "graph_create: null output");
    *out = nullptr;
    if (n < 0 || m < 0 || (m > 0 && !uv)) return fail(GAPA_CUDA_E_INVALID, "graph_create: bad sizes");
    if (2 * m > INT32_MAX) return fail(GAPA_CUDA_E_INVALID, "graph_create: 2m exceeds int32 CSR offsets");
    auto* c = new gapa_cuda_ctx();
    c->n = n;
    c->m = m;
    c->h_row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    for (int64_t e = 0; e < m; ++e) {
        const int32_t u = uv[2 * e], v = uv[2 * e + 1];
        if (u == v) { delete c; return fail(GAPA_CUDA_E_INVALID, "graph: self-loop rejected"); }
        if (u < 0 || v < 0 || u >= n || v >= n) { delete c; return fail(GAPA_CUDA_E_INVALID, "graph: edge endpoint out of range"); }
        c->h_row_ptr[u + 1]++;
        c->h_row_ptr[v + 1]++;
    }
    for (int32_t u = 0; u < n; ++u) c->h_row_ptr[u + 1] += c->h_row_ptr[u];
    c->h_col_idx.assign(static_cast<size_t>(2 * m), 0);
    std::vector<int32_t> fill(c->h_row_ptr.begin(), c->h_row_ptr.end() - 1);
    for (int64_t e = 0; e < m; ++e) {
        const int32_t u = uv[2 * e], v = uv[2 * e + 1];
        c->h_col_idx[fill[u]++] = v;
        c->h_col_idx[fill[v]++] = u;
    }
    for (int32_t u = 0; u < n; ++u) {
        auto b = c->h_col_idx.begin() + c->h_row_ptr[u], e = c->h_col_idx.begin() + c->h_row_ptr[u + 1];
        std::sort(b, e);
        if (std::adjacent_find(b, e) != e) { delete c; return fail(GAPA_CUDA_E_INVALID, "graph: duplicate edge rejected"); }
    }
    return finish_create(c, device, out);
}

int gapa_cuda_graph_create_csr(int32_t n, int64_t m, const int32_t* row_ptr, const int32_t* col_idx, int device,
                               gapa_cuda_ctx** out) {
    if (!out) return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: null output");
    *out = nullptr;
    if (n < 0 || m < 0 || !row_ptr || (m > 0 && !col_idx)) return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: bad sizes");
    if (2 * m > INT32_MAX) return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: 2m exceeds int32 CSR offsets");
    if (row_ptr[0] != 0 || row_ptr[n] != 2 * m) return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: row_ptr does not span 2m slots");
    auto* c = new gapa_cuda_ctx();
    c->n = n;
    c->m = m;
    c->h_row_ptr.assign(row_ptr, row_ptr + n + 1);
    c->h_col_idx.assign(col_idx, col_idx + 2 * m);
    for (int32_t u = 0; u < n; ++u) {
        if (row_ptr[u + 1] < row_ptr[u]) { delete c; return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: row_ptr not monotone"); }
        for (int32_t i = row_ptr[u]; i < row_ptr[u + 1]; ++i) {
            const int32_t v = col_idx[i];
            if (v < 0 || v >= n || v == u || (i > row_ptr[u] && col_idx[i - 1] >= v)) {
                delete c;
                return fail(GAPA_CUDA_E_INVALID, "graph_create_csr: row %d is not a strictly ascending loop-free list", u);
            }
        }
    }
    return finish_create(c, device, out);
}

int gapa_cuda_destroy(gapa_cuda_ctx* c) {
    if (!c) return GAPA_CUDA_OK;
    cudaSetDevice(c->device);
    pc_free(c);
    lpa_free(c);
    cda_free(c);
    sixdst_free(c);
    for (int32_t* p : {c->d_row_ptr, c->d_col_idx, c->d_edge_id, c->d_edge_u, c->d_edge_v, c->d_by_degree,
                       c->d_pool_map, c->d_pairs, c->d_add_u, c->d_add_v})
        if (p) cudaFree(p);
    c->genes_stage.release();
    c->out_stage.release();
    c->status_buf.release();
    if (c->h_status) cudaFreeHost(c->h_status);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    if (c->ev_stop) cudaEventDestroy(c->ev_stop);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (cudaEvent_t ev : c->copy_events) cudaEventDestroy(ev);
    for (cudaEvent_t ev : c->chunk_events) cudaEventDestroy(ev);
    delete c->ring;
    delete c;
    return GAPA_CUDA_OK;
}

int gapa_cuda_graph_info(const gapa_cuda_ctx* c, int32_t* n, int64_t* m, int* device) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "graph_info: null context");
    if (n) *n = c->n;
    if (m) *m = c->m;
    if (device) *device = c->device;
    return GAPA_CUDA_OK;
}

// EdgeAddition pools: with u == NULL every non-edge (a < b) in lexicographic order
// (build_gene_pool, gene_pool.cpp:81-87); otherwise the caller's pairs.
static int pool_set_addition(gapa_cuda_ctx* c, int32_t n_genes, const int32_t* u, const int32_t* v) {
    std::vector<int32_t> au, av;
    if (!u) {
        const int64_t n = c->n, size = n * (n - 1) / 2 - c->m;
        if (size <= 0) return fail(GAPA_CUDA_E_INVALID, "gene pool: graph is complete, no edges can be added");
        if (size > 0x7fffffffll) return fail(GAPA_CUDA_E_INVALID, "gene pool: %lld non-edges do not fit int32 gene ids", static_cast<long long>(size));
        au.reserve(static_cast<size_t>(size));
        av.reserve(static_cast<size_t>(size));
        for (int32_t a = 0; a < c->n; ++a) {
            int32_t i = c->h_row_ptr[a];
            const int32_t ie = c->h_row_ptr[a + 1];
            while (i < ie && c->h_col_idx[i] <= a) ++i;
            for (int32_t b = a + 1; b < c->n; ++b) {
                if (i < ie && c->h_col_idx[i] == b) { ++i; continue; }
                au.push_back(a);
                av.push_back(b);
            }
        }
    } else {
        if (!v) return fail(GAPA_CUDA_E_INVALID, "pool_set: edge pool needs both endpoint arrays");
        if (n_genes < 0) return fail(GAPA_CUDA_E_INVALID, "pool_set: negative size");
        au.resize(static_cast<size_t>(n_genes));
        av.resize(static_cast<size_t>(n_genes));
        std::vector<uint64_t> keys(static_cast<size_t>(n_genes));
        for (int32_t i = 0; i < n_genes; ++i) {
            int32_t a = u[i], b = v[i];
            if (a < 0 || b < 0 || a >= c->n || b >= c->n || a == b)
                return fail(GAPA_CUDA_E_INVALID, "pool_set: (%d, %d) is not a valid node pair", a, b);
            if (a > b) std::swap(a, b);
            keys[i] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
            const bool present = edge_rank(c, a, b) >= 0;  // adjacency.set on a set bit: no-op
            au[i] = present ? -1 : a;
            av[i] = present ? -1 : b;
        }
        std::sort(keys.begin(), keys.end());
        if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
            return fail(GAPA_CUDA_E_INVALID, "gene pool: duplicate element");  // gene_pool.cpp:40
    }
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    for (int32_t** p : {&c->d_pool_map, &c->d_add_u, &c->d_add_v})
        if (*p) { cudaFree(*p); *p = nullptr; }
    GAPA_TRY(upload_i32(au, &c->d_add_u));
    GAPA_TRY(upload_i32(av, &c->d_add_v));
    c->pool_kind = GAPA_POOL_EDGE_ADDITION;
    c->pool_size = static_cast<int32_t>(au.size());
    c->pool_identity = true;
    c->h_pool_map.clear();
    ++c->pool_version;
    return GAPA_CUDA_OK;
}

// Edge-flip pools (not in the reference; include/gapa_cuda.h): every pair a < b (u == NULL: nothing is stored, genes are
// unranked on the device), or the caller's pairs in d_add_u / d_add_v.
static int pool_set_flip(gapa_cuda_ctx* c, int32_t n_genes, const int32_t* u, const int32_t* v) {
    std::vector<int32_t> au, av;
    const int64_t n = c->n;
    if (!u) {
        if (n < 2) return fail(GAPA_CUDA_E_INVALID, "gene pool: no node pairs to flip");
        if (n > 65536) return fail(GAPA_CUDA_E_INVALID, "gene pool: %lld node pairs do not fit int32 gene ids", static_cast<long long>(n * (n - 1) / 2));
        n_genes = static_cast<int32_t>(n * (n - 1) / 2);
    } else {
        if (!v) return fail(GAPA_CUDA_E_INVALID, "pool_set: edge pool needs both endpoint arrays");
        if (n_genes < 0) return fail(GAPA_CUDA_E_INVALID, "pool_set: negative size");
        au.resize(static_cast<size_t>(n_genes));
        av.resize(static_cast<size_t>(n_genes));
        std::vector<uint64_t> keys(static_cast<size_t>(n_genes));
        for (int32_t i = 0; i < n_genes; ++i) {
            int32_t a = u[i], b = v[i];
            if (a < 0 || b < 0 || a >= c->n || b >= c->n || a == b)
                return fail(GAPA_CUDA_E_INVALID, "pool_set: (%d, %d) is not a valid node pair", a, b);
            if (a > b) std::swap(a, b);
            au[static_cast<size_t>(i)] = a;
            av[static_cast<size_t>(i)] = b;
            keys[static_cast<size_t>(i)] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
        }
        std::sort(keys.begin(), keys.end());
        if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
            return fail(GAPA_CUDA_E_INVALID, "gene pool: duplicate element");  // gene_pool.cpp:40
    }
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    for (int32_t** p : {&c->d_pool_map, &c->d_add_u, &c->d_add_v})
        if (*p) { cudaFree(*p); *p = nullptr; }
    if (u) {
        GAPA_TRY(upload_i32(au, &c->d_add_u));
        GAPA_TRY(upload_i32(av, &c->d_add_v));
    }
    c->pool_kind = GAPA_POOL_EDGE_FLIP;
    c->pool_size = n_genes;
    c->pool_identity = true;
    c->flip_canonical = u == nullptr;
    c->h_pool_map.clear();
    ++c->pool_version;
    return GAPA_CUDA_OK;
}

int gapa_cuda_lp_score_set(gapa_cuda_ctx* c, int score) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "lp_score_set: null context");
    if (score != GAPA_LP_SCORE_RA && score != GAPA_LP_SCORE_CN) return fail(GAPA_CUDA_E_INVALID, "lp_score_set: unknown score %d", score);
    c->lp_score = score;
    return GAPA_CUDA_OK;
}

int gapa_cuda_pool_set(gapa_cuda_ctx* c, int kind, int32_t n_genes, const int32_t* u, const int32_t* v) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "pool_set: null context");
    if (kind != GAPA_POOL_NODE_REMOVAL && kind != GAPA_POOL_EDGE_REMOVAL && kind != GAPA_POOL_EDGE_ADDITION && kind != GAPA_POOL_EDGE_FLIP)
        return fail(GAPA_CUDA_E_INVALID, "pool_set: unknown pool kind %d", kind);
    if (c->n == 0) return fail(GAPA_CUDA_E_INVALID, "gene pool: graph is empty");  // gene_pool.cpp:70
    if (kind == GAPA_POOL_EDGE_ADDITION) return pool_set_addition(c, n_genes, u, v);
    if (kind == GAPA_POOL_EDGE_FLIP) return pool_set_flip(c, n_genes, u, v);
    const int32_t full = kind == GAPA_POOL_NODE_REMOVAL ? c->n : static_cast<int32_t>(c->m);
    if (!u) n_genes = full;
    if (n_genes < 0) return fail(GAPA_CUDA_E_INVALID, "pool_set: negative size");
    std::vector<int32_t> map(static_cast<size_t>(n_genes));
    std::vector<uint64_t> pair_keys;  // custom edge pools: the (u, v) pairs, for the duplicate check
    bool identity = true;
    for (int32_t i = 0; i < n_genes; ++i) {
        int32_t target;
        if (!u) target = i;
        else if (kind == GAPA_POOL_NODE_REMOVAL) {
            target = u[i];
            if (target < 0 || target >= c->n) return fail(GAPA_CUDA_E_INVALID, "pool_set: node %d out of range", target);
        } else {
            if (!v) return fail(GAPA_CUDA_E_INVALID, "pool_set: edge pool needs both endpoint arrays");
            int32_t a = u[i], b = v[i];
            if (a < 0 || b < 0 || a >= c->n || b >= c->n || a == b)
                return fail(GAPA_CUDA_E_INVALID, "pool_set: (%d, %d) is not a valid node pair", a, b);
            if (a > b) std::swap(a, b);
            pair_keys.push_back((static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b));
            // A pair that is not an edge of THIS graph (a pool built on the full graph, evaluated on split.train) is accepted
            // like the reference does (gene_pool.cpp:34-56): clearing an absent adjacency bit is a no-op.  -1 = no-op gene.
            target = edge_rank(c, a, b);
        }
        map[i] = target;
        identity &= (target == i);
    }
    if (!identity) {  // GenePool's constructor rejects repeated elements (gene_pool.cpp:36-41)
        if (!pair_keys.empty()) {
            std::sort(pair_keys.begin(), pair_keys.end());
            if (std::adjacent_find(pair_keys.begin(), pair_keys.end()) != pair_keys.end())
                return fail(GAPA_CUDA_E_INVALID, "gene pool: duplicate element");
        } else {
            std::vector<int32_t> sorted(map);
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                return fail(GAPA_CUDA_E_INVALID, "gene pool: duplicate element");
        }
    }
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    for (int32_t** p : {&c->d_pool_map, &c->d_add_u, &c->d_add_v})
        if (*p) { cudaFree(*p); *p = nullptr; }
    if (!identity) GAPA_TRY(upload_i32(map, &c->d_pool_map));
    c->pool_kind = kind;
    c->pool_size = n_genes;
    c->pool_identity = identity;
    c->h_pool_map = identity ? std::vector<int32_t>() : map;
    ++c->pool_version;
    return GAPA_CUDA_OK;
}

int gapa_cuda_pool_info(const gapa_cuda_ctx* c, int* kind, int32_t* n_genes) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "pool_info: null context");
    if (kind) *kind = c->pool_kind;
    if (n_genes) *n_genes = c->pool_size;
    return GAPA_CUDA_OK;
}

int gapa_cuda_lp_split_set(gapa_cuda_ctx* c, int32_t T, const int32_t* test_uv, int32_t P, const int32_t* probe_uv) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "lp_split_set: null context");
    if (T < 1 || P < 0 || !test_uv || (P > 0 && !probe_uv))
        return fail(GAPA_CUDA_E_INVALID, "lp_auc_precision: empty test set");  // link_prediction.cpp:82
    std::vector<int32_t> pairs(static_cast<size_t>(2) * (T + P));
    std::memcpy(pairs.data(), test_uv, sizeof(int32_t) * 2 * T);
    if (P) std::memcpy(pairs.data() + 2 * T, probe_uv, sizeof(int32_t) * 2 * P);
    for (int32_t x : pairs)
        if (x < 0 || x >= c->n) return fail(GAPA_CUDA_E_INVALID, "lp_split_set: pair endpoint out of range");
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    if (c->d_pairs) { cudaFree(c->d_pairs); c->d_pairs = nullptr; }
    GAPA_TRY(upload_i32(pairs, &c->d_pairs));
    c->T = T;
    c->P = P;
    return GAPA_CUDA_OK;
}

static int check_task(const gapa_cuda_ctx* c, int task) {
    switch (task) {
        case GAPA_TASK_PC:
        case GAPA_TASK_MCN:
        case GAPA_TASK_SIXDST:
            if (c->pool_kind != GAPA_POOL_NODE_REMOVAL)
                return fail(GAPA_CUDA_E_INVALID, "%s: incompatible gene pool kind", task == GAPA_TASK_PC ? "pc_fitness" : "sixdst_fitness");
            return GAPA_CUDA_OK;
        case GAPA_TASK_CDA:
            if (c->pool_kind == GAPA_POOL_NODE_REMOVAL || c->pool_kind == GAPA_POOL_EDGE_FLIP) return fail(GAPA_CUDA_E_INVALID, "cda_fitness: incompatible gene pool kind");
            return GAPA_CUDA_OK;
        case GAPA_TASK_LPA:
            if (c->pool_kind != GAPA_POOL_EDGE_REMOVAL && c->pool_kind != GAPA_POOL_EDGE_FLIP) return fail(GAPA_CUDA_E_INVALID, "lpa_fitness: incompatible gene pool kind");
            if (c->T < 1) return fail(GAPA_CUDA_E_INVALID, "lpa_fitness: no link-prediction split set");
            return GAPA_CUDA_OK;
    }
    return fail(GAPA_CUDA_E_INVALID, "unknown fitness task %d", task);
}

// every gene of the s parent rows lies in [0, pool_size)?
__global__ void __launch_bounds__(256) k_genes_in_range(const int32_t* __restrict__ pool, const int32_t* __restrict__ parent, int s, int k,
                                                        int pool_size, int* bad) {
    griddep_launch();
    griddep_wait();
    const size_t cells = static_cast<size_t>(s) * k;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / k);
        const int gene = pool[static_cast<size_t>(parent[r]) * k + (i - static_cast<size_t>(r) * k)];
        if (gene < 0 || gene >= pool_size) *bad = 1;
    }
}

static int eval_rows_locked(gapa_cuda_ctx* c, int task, const GeneRows& genes, int rows, double* out_dev, void* stream,
                            const VariationSpec* vary = nullptr, bool defer_timing = false, bool already_locked = false,
                            cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_end = nullptr) {
    std::unique_lock<std::mutex> lock(c->mu, std::defer_lock);
    if (!already_locked) lock.lock();  // the host-buffer form already holds it
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ev_begin) ev_begin = c->ev_start, ev_end = c->ev_stop;
    GAPA_CUDA_TRY(cudaEventRecord(ev_begin, s));
    int rc;
    if (task == GAPA_TASK_PC || task == GAPA_TASK_MCN) {
        rc = pc_eval(c, task, genes, rows, out_dev, s, vary != nullptr, vary);  // builds the children itself
    } else {
        if (vary) GAPA_TRY(launch_variation_spec(*vary, genes.cols, rows, s));
        rc = task == GAPA_TASK_CDA      ? cda_eval(c, genes, rows, out_dev, s)
             : task == GAPA_TASK_SIXDST ? sixdst_eval(c, genes, rows, out_dev, s, vary != nullptr)
                                        : lpa_eval(c, genes, rows, out_dev, s, vary != nullptr);
    }
    if (rc != GAPA_CUDA_OK) return rc;
    GAPA_CUDA_TRY(cudaEventRecord(ev_end, s));
    if (defer_timing) return GAPA_CUDA_OK;  // the caller synchronises the stream once and reads the events then
    GAPA_CUDA_TRY(cudaEventSynchronize(ev_end));
    GAPA_CUDA_TRY(cudaEventElapsedTime(&c->last_eval_ms, ev_begin, ev_end));
    return GAPA_CUDA_OK;
}

int gapa_cuda_eval_batch_device(gapa_cuda_ctx* c, int task, const int32_t* genes_dev, int rows, int cols,
                                double* out_dev, void* stream) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "eval_batch: null context");
    GAPA_TRY(check_task(c, task));
    if (rows < 0 || cols < 0) return fail(GAPA_CUDA_E_INVALID, "eval_batch: negative shape");
    if (rows == 0) return GAPA_CUDA_OK;
    if (!out_dev || (cols > 0 && !genes_dev)) return fail(GAPA_CUDA_E_INVALID, "eval_batch: null buffer");
    return eval_rows_locked(c, task, GeneRows{genes_dev, nullptr, cols}, rows, out_dev, stream);
}

int gapa_cuda_eval_rows_device(gapa_cuda_ctx* c, int task, const int32_t* pool_dev, const int32_t* slot_dev, int rows,
                               int cols, double* out_dev, void* stream) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "eval_rows: null context");
    GAPA_TRY(check_task(c, task));
    if (rows < 0 || cols < 0) return fail(GAPA_CUDA_E_INVALID, "eval_rows: negative shape");
    if (rows == 0) return GAPA_CUDA_OK;
    if (!out_dev || !slot_dev || (cols > 0 && !pool_dev)) return fail(GAPA_CUDA_E_INVALID, "eval_rows: null buffer");
    return eval_rows_locked(c, task, GeneRows{pool_dev, slot_dev, cols}, rows, out_dev, stream);
}

int gapa_cuda_ga_slots_variation_eval_device(gapa_cuda_ctx* c, int task, int32_t* pool_dev, const int32_t* parent_dev,
                                             const int32_t* child_dev, const int32_t* partner_dev, int s, int k, int row_first,
                                             int row_count, double pc, double pm, uint64_t seed, uint64_t generation,
                                             double* fit_block_dev, void* stream) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "variation_eval: null context");
    GAPA_TRY(check_task(c, task));
    if (!(pc >= 0.0 && pc <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pc must be in [0, 1]");
    if (!(pm >= 0.0 && pm <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pm must be in [0, 1]");
    if (s < 1 || k < 0 || row_first < 0 || row_count < 0 || row_first + row_count > s)
        return fail(GAPA_CUDA_E_INVALID, "variation_eval: row block outside the population");
    if (row_count == 0) return GAPA_CUDA_OK;
    if (!pool_dev || !parent_dev || !child_dev || !fit_block_dev) return fail(GAPA_CUDA_E_INVALID, "variation_eval: null buffer");
    // The fused kernels index bitmaps with the genes they inherit from the parents without a per-gene range check.  Parents
    // written by this library's operators are inside the pool by induction; a pool buffer seen for the first time (or
    // after the gene pool changed) is validated once, all s parent rows.
    {
        std::lock_guard<std::mutex> lock(c->mu);
        const size_t cells = static_cast<size_t>(s) * k;
        if (c->validated_pool != pool_dev || c->validated_cells != cells || c->validated_version != c->pool_version) {
            GAPA_CUDA_TRY(cudaSetDevice(c->device));
            GAPA_TRY(c->status_buf.ensure(sizeof(int)));
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            GAPA_CUDA_TRY(cudaMemsetAsync(c->status_buf.ptr, 0, sizeof(int), st));
            if (cells) {
                const int grid = static_cast<int>(std::min<size_t>(static_cast<size_t>(c->sm_count) * 8, (cells + 255) / 256));
                GAPA_LAUNCH(k_genes_in_range, grid, 256, 0, st, pool_dev, parent_dev, s, k, c->pool_size, c->status_buf.as<int>());
            }
            int bad = 0;
            GAPA_CUDA_TRY(cudaMemcpyAsync(&bad, c->status_buf.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
            GAPA_CUDA_TRY(cudaStreamSynchronize(st));
            if (bad) return fail(GAPA_CUDA_E_RANGE, "variation_eval: a parent row holds a gene id outside the pool");
            c->validated_pool = pool_dev;
            c->validated_cells = cells;
            c->validated_version = c->pool_version;
        }
    }
    VariationSpec spec;
    spec.P = make_variation_params(pc, pm, static_cast<uint32_t>(c->pool_size), s, seed, generation);
    spec.pool = pool_dev;
    spec.parent = parent_dev;
    spec.child = child_dev;
    spec.partner = partner_dev;
    spec.row_first = row_first;
    return eval_rows_locked(c, task, GeneRows{pool_dev, child_dev + row_first, k}, row_count, fit_block_dev, stream, &spec);
}

int gapa_cuda_eval_batch(gapa_cuda_ctx* c, int task, const int32_t* genes_host, int rows, int cols, double* out_host) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "eval_batch: null context");
    GAPA_TRY(check_task(c, task));
    if (rows < 0 || cols < 0) return fail(GAPA_CUDA_E_INVALID, "eval_batch: negative shape");
    if (rows == 0) return GAPA_CUDA_OK;
    if (!out_host || (cols > 0 && !genes_host)) return fail(GAPA_CUDA_E_INVALID, "eval_batch: null buffer");
    std::lock_guard<std::mutex> lock(c->mu);
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    const size_t cells = static_cast<size_t>(rows) * cols;
    GAPA_TRY(c->genes_stage.ensure(sizeof(int32_t) * std::max<size_t>(cells, 1)));
    GAPA_TRY(c->out_stage.ensure(sizeof(double) * rows));
    // Row chunks of ~64 MB in whole super-groups of 256 individuals (one 32-byte record of the bit-sliced PC kernels):
    // the H2D copy of chunk i+1 runs on the copy stream while the kernels of chunk i run on the work stream, so a
    // PCIe-bound call costs max(copy, compute) instead of their sum.
    const size_t row_bytes = sizeof(int32_t) * static_cast<size_t>(std::max(cols, 1));
    int chunk_rows = static_cast<int>(std::min<size_t>(rows, std::max<size_t>(256, ((64ull << 20) / row_bytes) & ~size_t{255})));
    const int chunks = (rows + chunk_rows - 1) / chunk_rows;
    if (!c->copy_stream) GAPA_CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    while (static_cast<int>(c->copy_events.size()) < chunks) {
        cudaEvent_t ev;
        GAPA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->copy_events.push_back(ev);
    }
    int32_t* stage = c->genes_stage.as<int32_t>();
    // A PAGEABLE caller buffer (std::vector of the reference's PopulationMatrix, population.hpp:12-40) would make every
    // cudaMemcpyAsync a synchronous, driver-staged copy at a few GB/s.  Large pageable batches go through the
    // library's own pinned ring instead: host threads copy slice i+1 into a pinned buffer while slice i crosses PCIe.
    bool pageable = false;
    if (cells * sizeof(int32_t) >= kPinnedRingMinBytes) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, genes_host) != cudaSuccess) (void)cudaGetLastError();
        pageable = attr.type == cudaMemoryTypeUnregistered;
        if (const char* raw = std::getenv("GAPA_PINNED_RING")) pageable = pageable && raw[0] != '0';
    }
    float total_ms = 0.f;
    while (static_cast<int>(c->chunk_events.size()) < 2 * chunks) {
        cudaEvent_t ev;
        GAPA_CUDA_TRY(cudaEventCreate(&ev));
        c->chunk_events.push_back(ev);
    }
    if (cells && !pageable)
        for (int i = 0; i < chunks; ++i) {
            const int r0 = i * chunk_rows, cr = std::min(chunk_rows, rows - r0);
            GAPA_CUDA_TRY(cudaMemcpyAsync(stage + static_cast<size_t>(r0) * cols, genes_host + static_cast<size_t>(r0) * cols,
                                          sizeof(int32_t) * static_cast<size_t>(cr) * cols, cudaMemcpyHostToDevice, c->copy_stream));
            GAPA_CUDA_TRY(cudaEventRecord(c->copy_events[i], c->copy_stream));
        }
    if (pageable && !c->ring) c->ring = new PinnedRing();
    // pageable: the matrix in slices of at most one ring slot that do not straddle a chunk; slice k+1 is being copied into its
    // slot by the host threads while slice k crosses PCIe and while this thread enqueues the kernels of the chunk slice k ended
    struct Slice { size_t off, len; int ends_chunk; };
    std::vector<Slice> slices;
    if (pageable) {
        size_t at = 0;
        for (int i = 0; i < chunks; ++i) {
            const size_t upto = sizeof(int32_t) * static_cast<size_t>(std::min(rows, (i + 1) * chunk_rows)) * cols;
            while (at < upto) {
                const size_t len = std::min(c->ring->slice_bytes, upto - at);
                slices.push_back(Slice{at, len, at + len == upto ? i : -1});
                at += len;
            }
        }
    }
    auto eval_chunk = [&](int i) -> int {
        const int r0 = i * chunk_rows, cr = std::min(chunk_rows, rows - r0);
        if (cells) GAPA_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copy_events[i], 0));
        // every chunk has its own pair of timing events, read once at the end: the host is free to stage the next chunk
        return eval_rows_locked(c, task, GeneRows{stage + static_cast<size_t>(r0) * cols, nullptr, cols}, cr,
                                c->out_stage.as<double>() + r0, c->stream, nullptr, true, true, c->chunk_events[2 * i],
                                c->chunk_events[2 * i + 1]);
    };
    if (pageable) {
        const char* src = reinterpret_cast<const char*>(genes_host);
        char* dst = reinterpret_cast<char*>(stage);
        if (!slices.empty()) GAPA_TRY(c->ring->begin(src + slices[0].off, slices[0].len));
        for (size_t k = 0; k < slices.size(); ++k) {
            GAPA_TRY(c->ring->end(dst + slices[k].off, c->copy_stream));
            if (k + 1 < slices.size()) GAPA_TRY(c->ring->begin(src + slices[k + 1].off, slices[k + 1].len));
            if (slices[k].ends_chunk >= 0) {
                GAPA_CUDA_TRY(cudaEventRecord(c->copy_events[slices[k].ends_chunk], c->copy_stream));
                GAPA_TRY(eval_chunk(slices[k].ends_chunk));
            }
        }
        if (!cells)
            for (int i = 0; i < chunks; ++i) GAPA_TRY(eval_chunk(i));  // cols == 0: nothing to stage
    } else {
        for (int i = 0; i < chunks; ++i) GAPA_TRY(eval_chunk(i));
    }
    GAPA_CUDA_TRY(cudaMemcpyAsync(out_host, c->out_stage.ptr, sizeof(double) * rows, cudaMemcpyDeviceToHost, c->stream));
    GAPA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < chunks; ++i) {
        float ms = 0.f;
        GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, c->chunk_events[2 * i], c->chunk_events[2 * i + 1]));
        total_ms += ms;
    }
    c->last_eval_ms = total_ms;
    return GAPA_CUDA_OK;
}

// ---- reporting outputs of one individual (bench.cpp:268-311) -----------------------------------------
// The partition detect_communities returns on the perturbed graph, normalised by first appearance
// (community.cpp:17-26), for the NMI columns; and the RA scores behind the AUC, for the precision column.
int gapa_cuda_detect_communities(gapa_cuda_ctx* c, const int32_t* genes_host, int cols, int32_t* assignment_host, double* q_host) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "detect_communities: null context");
    GAPA_TRY(check_task(c, GAPA_TASK_CDA));
    if (cols < 0 || !assignment_host || (cols > 0 && !genes_host)) return fail(GAPA_CUDA_E_INVALID, "detect_communities: bad arguments");
    std::lock_guard<std::mutex> lock(c->mu);
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    const int n = c->n;
    GAPA_TRY(c->genes_stage.ensure(sizeof(int32_t) * std::max(cols, 1)));
    GAPA_TRY(c->out_stage.ensure(sizeof(double) + sizeof(int32_t) * static_cast<size_t>(n)));
    if (cols) GAPA_CUDA_TRY(cudaMemcpyAsync(c->genes_stage.ptr, genes_host, sizeof(int32_t) * cols, cudaMemcpyHostToDevice, c->stream));
    double* q_dev = c->out_stage.as<double>();
    int32_t* owner_dev = reinterpret_cast<int32_t*>(q_dev + 1);
    // an edgeless perturbed graph never reaches the detector's merge loop: everyone stays a singleton
    std::vector<int32_t> owner(static_cast<size_t>(n));
    std::iota(owner.begin(), owner.end(), 0);
    GAPA_CUDA_TRY(cudaMemcpyAsync(owner_dev, owner.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
    GAPA_TRY(cda_eval(c, GeneRows{c->genes_stage.as<int32_t>(), nullptr, cols}, 1, q_dev, c->stream, owner_dev));
    double q = 0.0;
    GAPA_CUDA_TRY(cudaMemcpyAsync(owner.data(), owner_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    GAPA_CUDA_TRY(cudaMemcpyAsync(&q, q_dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    GAPA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    // owners are smallest members, so ascending owner == first appearance (community.cpp:17-26)
    std::vector<int32_t> label(static_cast<size_t>(n), -1);
    int32_t next = 0;
    for (int u = 0; u < n; ++u) {
        if (label[owner[u]] < 0) label[owner[u]] = next++;
        assignment_host[u] = label[owner[u]];
    }
    if (q_host) *q_host = q;
    return GAPA_CUDA_OK;
}

int gapa_cuda_lpa_scores(gapa_cuda_ctx* c, const int32_t* genes_host, int cols, double* test_scores_host,
                         double* probe_scores_host, double* auc_host) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "lpa_scores: null context");
    GAPA_TRY(check_task(c, GAPA_TASK_LPA));
    if (cols < 0 || (cols > 0 && !genes_host)) return fail(GAPA_CUDA_E_INVALID, "lpa_scores: bad arguments");
    std::lock_guard<std::mutex> lock(c->mu);
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    GAPA_TRY(c->genes_stage.ensure(sizeof(int32_t) * std::max(cols, 1)));
    GAPA_TRY(c->out_stage.ensure(sizeof(double)));
    if (cols) GAPA_CUDA_TRY(cudaMemcpyAsync(c->genes_stage.ptr, genes_host, sizeof(int32_t) * cols, cudaMemcpyHostToDevice, c->stream));
    GAPA_TRY(lpa_eval(c, GeneRows{c->genes_stage.as<int32_t>(), nullptr, cols}, 1, c->out_stage.as<double>(), c->stream));
    const double* scores = lpa_last_scores(c);
    if (test_scores_host) GAPA_CUDA_TRY(cudaMemcpyAsync(test_scores_host, scores, sizeof(double) * c->T, cudaMemcpyDeviceToHost, c->stream));
    if (probe_scores_host && c->P > 0)
        GAPA_CUDA_TRY(cudaMemcpyAsync(probe_scores_host, scores + c->T, sizeof(double) * c->P, cudaMemcpyDeviceToHost, c->stream));
    if (auc_host) GAPA_CUDA_TRY(cudaMemcpyAsync(auc_host, c->out_stage.ptr, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    GAPA_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return GAPA_CUDA_OK;
}

int gapa_cuda_last_eval_ms(const gapa_cuda_ctx* c, float* ms) {
    if (!c || !ms) return fail(GAPA_CUDA_E_INVALID, "last_eval_ms: null argument");
    *ms = c->last_eval_ms;
    return GAPA_CUDA_OK;
}

int gapa_cuda_malloc(int device, uint64_t bytes, void** out_dev) {
    if (!out_dev) return fail(GAPA_CUDA_E_INVALID, "malloc: null output");
    GAPA_CUDA_TRY(cudaSetDevice(device));
    GAPA_CUDA_TRY(cudaMalloc(out_dev, std::max<uint64_t>(bytes, 1)));
    return GAPA_CUDA_OK;
}
int gapa_cuda_free(int device, void* dev) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (dev) GAPA_CUDA_TRY(cudaFree(dev));
    return GAPA_CUDA_OK;
}
int gapa_cuda_memcpy_h2d(int device, void* dst_dev, const void* src_host, uint64_t bytes) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (bytes) GAPA_CUDA_TRY(cudaMemcpy(dst_dev, src_host, bytes, cudaMemcpyHostToDevice));
    return GAPA_CUDA_OK;
}
int gapa_cuda_memcpy_d2h(int device, void* dst_host, const void* src_dev, uint64_t bytes) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    if (bytes) GAPA_CUDA_TRY(cudaMemcpy(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost));
    return GAPA_CUDA_OK;
}
int gapa_cuda_stream_sync(int device, void* stream) {
    GAPA_CUDA_TRY(cudaSetDevice(device));
    GAPA_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return GAPA_CUDA_OK;
}

}  // extern "C"
