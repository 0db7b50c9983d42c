// Host-side problem setup behind include/gapa_cuda.h: deterministic synthetic graphs
// and the link-prediction split.  These run once per experiment on the CPU, exactly
// as in the reference (generators.cpp, link_prediction.cpp:11-53 are host code there
// too); they are inputs to the hot path, not part of it.  Draw sequences follow the
// reference's RngStream so small graphs are edge-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <unordered_set>
#include <vector>

#include "internal.cuh"

using namespace gapa_b200;

namespace {

// Sequential view of a counter stream (rng.hpp:17-37).
struct Stream {
    uint64_t key;
    uint64_t counter = 0;
    explicit Stream(uint64_t k) : key(k) {}
    uint64_t u64() { return draw_u64(key, ++counter); }
    bool bernoulli(double p) { return static_cast<double>(u64() >> 11) * 0x1.0p-53 < p; }
    uint32_t index(uint32_t bound) { return static_cast<uint32_t>((static_cast<unsigned __int128>(u64()) * bound) >> 64); }
};

int emit(const std::vector<int32_t>& flat, int32_t* uv, int64_t capacity, int64_t* m) {
    const int64_t count = static_cast<int64_t>(flat.size() / 2);
    if (m) *m = count;
    if (!uv) return GAPA_CUDA_OK;  // size query
    if (capacity < count) return fail(GAPA_CUDA_E_INVALID, "generator: edge buffer too small (%lld < %lld)",
                                      static_cast<long long>(capacity), static_cast<long long>(count));
    std::copy(flat.begin(), flat.end(), uv);
    return GAPA_CUDA_OK;
}

}  // namespace

extern "C" {

// barabasi_albert (generators.cpp:21-45): node v attaches to min(attach, v) distinct
// targets drawn uniformly from the endpoint multiset (degree-proportional).
int gapa_host_barabasi_albert(int32_t n, int32_t attach, uint64_t seed, int32_t* uv, int64_t capacity, int64_t* m) {
    if (n < 1 || attach < 1) return fail(GAPA_CUDA_E_INVALID, "barabasi_albert: invalid parameters");
    Stream rng(mix64(seed ^ 0x42415241ull));
    std::vector<int32_t> flat, endpoints{0}, picked;
    flat.reserve(static_cast<size_t>(2) * attach * n);
    endpoints.reserve(static_cast<size_t>(2) * attach * n + 1);
    for (int32_t v = 1; v < n; ++v) {
        const int32_t want = std::min(attach, v);
        picked.clear();
        while (static_cast<int32_t>(picked.size()) < want) {
            const int32_t t = endpoints[rng.index(static_cast<uint32_t>(endpoints.size()))];
            if (std::find(picked.begin(), picked.end(), t) == picked.end()) picked.push_back(t);
        }
        for (int32_t t : picked) {
            flat.push_back(t);
            flat.push_back(v);
            endpoints.push_back(t);
            endpoints.push_back(v);
        }
    }
    return emit(flat, uv, capacity, m);
}

// erdos_renyi (generators.cpp:11-19): one Bernoulli(p) per pair, row-major u < v.
int gapa_host_erdos_renyi(int32_t n, double p, uint64_t seed, int32_t* uv, int64_t capacity, int64_t* m) {
    if (n < 0 || !(p >= 0.0 && p <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "erdos_renyi: invalid parameters");
    Stream rng(mix64(seed ^ 0x45524e4f53ull));
    std::vector<int32_t> flat;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v)
            if (rng.bernoulli(p)) {
                flat.push_back(u);
                flat.push_back(v);
            }
    return emit(flat, uv, capacity, m);
}

// planted_partition (generators.cpp:47-58)
int gapa_host_planted_partition(int32_t blocks, int32_t block_size, double p_in, double p_out, uint64_t seed,
                                int32_t* uv, int64_t capacity, int64_t* m) {
    if (blocks < 1 || block_size < 1) return fail(GAPA_CUDA_E_INVALID, "planted_partition: invalid parameters");
    Stream rng(mix64(seed ^ 0x50504d4full));
    const int32_t n = blocks * block_size;
    std::vector<int32_t> flat;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v)
            if (rng.bernoulli(u / block_size == v / block_size ? p_in : p_out)) {
                flat.push_back(u);
                flat.push_back(v);
            }
    return emit(flat, uv, capacity, m);
}

// build_lp_split (link_prediction.cpp:11-53).  edges: m canonical (u < v) pairs in
// Graph::edges() order.  Outputs: train (m - T pairs, sorted), test (T, sorted), probe
// (T, sorted).  Call with null outputs to get T.
int gapa_host_lp_split(int32_t n, int64_t m64, const int32_t* edges, double fraction, uint64_t seed, int32_t* train_uv,
                       int32_t* test_uv, int32_t* probe_uv, int32_t* test_count) {
    if (!(fraction > 0.0 && fraction <= 0.5)) return fail(GAPA_CUDA_E_INVALID, "build_lp_split: test fraction must be in (0, 0.5]");
    if (m64 < 10) return fail(GAPA_CUDA_E_INVALID, "build_lp_split: graph has fewer than 10 edges");
    const int32_t m = static_cast<int32_t>(m64);
    const int32_t T = std::max<int32_t>(1, static_cast<int32_t>(std::lround(fraction * m)));
    if (test_count) *test_count = T;
    if (!train_uv || !test_uv || !probe_uv) return GAPA_CUDA_OK;

    Stream rng(mix64(seed ^ 0x4c505350ull));
    std::vector<int32_t> order(m);
    for (int32_t i = 0; i < m; ++i) order[i] = i;
    for (int32_t i = m - 1; i > 0; --i) std::swap(order[i], order[rng.index(static_cast<uint32_t>(i + 1))]);

    using Pair = std::pair<int32_t, int32_t>;
    std::vector<Pair> test, train, probe;
    std::unordered_set<uint64_t> present;
    present.reserve(static_cast<size_t>(m) * 2);
    auto key = [](int32_t a, int32_t b) {
        if (a > b) std::swap(a, b);
        return (static_cast<uint64_t>(static_cast<uint32_t>(a)) << 32) | static_cast<uint32_t>(b);
    };
    for (int32_t i = 0; i < m; ++i) {
        const Pair e{edges[2 * order[i]], edges[2 * order[i] + 1]};
        present.insert(key(e.first, e.second));
        (i < T ? test : train).push_back(e);
    }
    std::sort(test.begin(), test.end());
    std::sort(train.begin(), train.end());
    std::unordered_set<uint64_t> used;
    while (static_cast<int32_t>(probe.size()) < T) {
        const int32_t u = static_cast<int32_t>(rng.index(static_cast<uint32_t>(n)));
        const int32_t v = static_cast<int32_t>(rng.index(static_cast<uint32_t>(n)));
        if (u == v || present.count(key(u, v))) continue;
        if (!used.insert(key(u, v)).second) continue;
        probe.emplace_back(std::min(u, v), std::max(u, v));
    }
    std::sort(probe.begin(), probe.end());
    auto flatten = [](const std::vector<Pair>& src, int32_t* dst) {
        for (size_t i = 0; i < src.size(); ++i) {
            dst[2 * i] = src[i].first;
            dst[2 * i + 1] = src[i].second;
        }
    };
    flatten(train, train_uv);
    flatten(test, test_uv);
    flatten(probe, probe_uv);
    return GAPA_CUDA_OK;
}

// perturbation_budget (gene_pool.cpp:98-102)
int gapa_host_budget(int64_t basis, double rate, int32_t* k) {
    if (!(rate > 0.0 && rate <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "perturbation rate must be in (0, 1]");
    *k = std::max<int32_t>(1, static_cast<int32_t>(std::ceil(rate * static_cast<double>(basis))));
    return GAPA_CUDA_OK;
}

// EdgeAddition pool of build_gene_pool (gene_pool.cpp:81-87): every pair a < b that is not
// an edge, in lexicographic order.  `edges` are m (u, v) pairs in either orientation.
int gapa_host_nonedges(int32_t n, int64_t m, const int32_t* edges, int32_t* uv, int64_t capacity, int64_t* count) {
    if (n < 1 || m < 0 || (m > 0 && !edges)) return fail(GAPA_CUDA_E_INVALID, "gene pool: graph is empty");
    std::vector<std::vector<int32_t>> above(static_cast<size_t>(n));
    for (int64_t e = 0; e < m; ++e) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= n || b >= n || a == b) return fail(GAPA_CUDA_E_INVALID, "gene pool: invalid edge (%d, %d)", a, b);
        if (a > b) std::swap(a, b);
        above[a].push_back(b);
    }
    int64_t present = 0;
    for (auto& row : above) {
        std::sort(row.begin(), row.end());
        row.erase(std::unique(row.begin(), row.end()), row.end());
        present += static_cast<int64_t>(row.size());
    }
    const int64_t size = static_cast<int64_t>(n) * (n - 1) / 2 - present;
    if (size <= 0) return fail(GAPA_CUDA_E_INVALID, "gene pool: graph is complete, no edges can be added");
    if (count) *count = size;
    if (!uv) return GAPA_CUDA_OK;  // size query
    if (capacity < size) return fail(GAPA_CUDA_E_INVALID, "gene pool: pair buffer too small (%lld < %lld)",
                                     static_cast<long long>(capacity), static_cast<long long>(size));
    int64_t at = 0;
    for (int32_t a = 0; a < n; ++a) {
        size_t i = 0;
        const std::vector<int32_t>& row = above[a];
        for (int32_t b = a + 1; b < n; ++b) {
            if (i < row.size() && row[i] == b) { ++i; continue; }
            uv[2 * at] = a;
            uv[2 * at + 1] = b;
            ++at;
        }
    }
    return GAPA_CUDA_OK;
}

}  // extern "C"
