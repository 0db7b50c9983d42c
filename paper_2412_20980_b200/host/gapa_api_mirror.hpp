// Minimal stand-in for the reference's public types, used ONLY when the adapters in
// gapa_cuda_objectives.hpp are built without the reference's own headers (on a box where
// /root/reference does not exist).  Same names, members and meaning as
// include/gapa/{population,error,gene_pool,graph,link_prediction,fitness,ga_ops,modes}.hpp
// for the parts the hot path touches, so host code written against the reference compiles
// against either.  With -DGAPA_B200_USE_REFERENCE_HEADERS this file is not included at all
// and the adapters derive from the real gapa::FitnessFunction.
#pragma once

#include <algorithm>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gapa {

struct Error : std::runtime_error {  // error.hpp:9-12
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {  // error.hpp:21-24
    using Error::Error;
};

enum class Direction { Maximize, Minimize };  // population.hpp:9

struct PopulationMatrix {  // population.hpp:12-40: s x k gene ids, row-major
    int rows = 0, cols = 0;
    std::vector<std::int32_t> data;
    PopulationMatrix() = default;
    PopulationMatrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c) {}
    std::size_t offset(int r) const { return static_cast<std::size_t>(r) * cols; }
    std::int32_t& at(int r, int c) { return data[offset(r) + c]; }
    std::int32_t at(int r, int c) const { return data[offset(r) + c]; }
    std::span<std::int32_t> row(int r) { return {data.data() + offset(r), static_cast<std::size_t>(cols)}; }
    std::span<const std::int32_t> row(int r) const { return {data.data() + offset(r), static_cast<std::size_t>(cols)}; }
    PopulationMatrix slice(int first, int last) const {
        PopulationMatrix out(last - first, cols);
        std::copy(data.begin() + offset(first), data.begin() + offset(last), out.data.begin());
        return out;
    }
    void assign_rows(int first, const PopulationMatrix& block) {
        std::copy(block.data.begin(), block.data.end(), data.begin() + offset(first));
    }
    bool operator==(const PopulationMatrix&) const = default;
};
using FitnessVector = std::vector<double>;  // population.hpp:62

class Graph {  // graph.hpp:15-46 (edge list only; validation happens in the C ABI)
public:
    Graph() = default;
    Graph(int n, std::vector<std::pair<int, int>> edges) : n_(n), edges_(std::move(edges)) {
        for (auto& e : edges_)
            if (e.first > e.second) std::swap(e.first, e.second);
    }
    int node_count() const { return n_; }
    int edge_count() const { return static_cast<int>(edges_.size()); }
    const std::vector<std::pair<int, int>>& edges() const { return edges_; }

private:
    int n_ = 0;
    std::vector<std::pair<int, int>> edges_;
};

enum class PoolKind { EdgeRemoval, EdgeAddition, NodeRemoval };  // gene_pool.hpp:14
enum class ClosurePolicy { Exact, SixDegrees };                   // accessibility.hpp:14
struct GeneElement {                                              // gene_pool.hpp:21-25
    int u = -1, v = -1;
    bool is_node() const { return v < 0; }
};
class GenePool {  // gene_pool.hpp:32-52
public:
    GenePool(PoolKind kind, std::vector<GeneElement> genes) : kind_(kind), genes_(std::move(genes)) {}
    PoolKind kind() const { return kind_; }
    int size() const { return static_cast<int>(genes_.size()); }
    const GeneElement& gene(int id) const { return genes_[id]; }
    const std::vector<GeneElement>& genes() const { return genes_; }

private:
    PoolKind kind_;
    std::vector<GeneElement> genes_;
};
inline GenePool build_gene_pool(const Graph& g, PoolKind kind) {  // gene_pool.cpp:69-96
    if (g.node_count() == 0) throw Error("gene pool: graph is empty");
    std::vector<GeneElement> genes;
    if (kind == PoolKind::NodeRemoval) {
        for (int u = 0; u < g.node_count(); ++u) genes.push_back({u, -1});
    } else if (kind == PoolKind::EdgeRemoval) {
        auto sorted = g.edges();
        std::sort(sorted.begin(), sorted.end());
        for (auto [u, v] : sorted) genes.push_back({u, v});
    } else {  // every non-edge u < v, lexicographic (gene_pool.cpp:81-87)
        auto sorted = g.edges();
        std::sort(sorted.begin(), sorted.end());
        std::size_t next = 0;
        for (int u = 0; u < g.node_count(); ++u)
            for (int v = u + 1; v < g.node_count(); ++v) {
                if (next < sorted.size() && sorted[next] == std::pair(u, v)) { ++next; continue; }
                genes.push_back({u, v});
            }
        if (genes.empty()) throw Error("gene pool: graph is complete, no edges can be added");
    }
    return GenePool(kind, std::move(genes));
}

struct LinkPredictionSplit {  // link_prediction.hpp:16-21
    Graph train;
    std::vector<std::pair<int, int>> test_edges, probe_nonedges;
    std::uint64_t seed = 0;
};

class FitnessFunction {  // fitness.hpp:17-27
public:
    virtual ~FitnessFunction() = default;
    virtual Direction direction() const = 0;
    virtual double evaluate_one(std::span<const std::int32_t> genes) const = 0;
    virtual FitnessVector evaluate_batch(const PopulationMatrix& batch) const {
        FitnessVector out(batch.rows);
        for (int i = 0; i < batch.rows; ++i) out[i] = evaluate_one(batch.row(i));
        return out;
    }
};

struct GAParams {  // ga_ops.hpp:12-23
    double pc = 0.8, pm = 0.1;
    int pop_size = 100, budget = 1, iterations = 100;
    Direction direction = Direction::Minimize;
    std::optional<int> eda_interval;
    std::uint64_t seed = 1;
};

struct GenerationStats {  // modes.hpp:63-71
    double best = 0.0, mean = 0.0;
    double wall_seconds = 0.0, compute_seconds = 0.0, exchange_seconds = 0.0, lifecycle_seconds = 0.0;
    std::uint64_t messages = 0;
};
struct RunResult {  // modes.hpp:73-82
    PopulationMatrix final_population;
    FitnessVector final_fitness;
    std::vector<std::int32_t> best_individual;
    double best_fitness = 0.0;
    std::vector<GenerationStats> history;
    std::uint64_t fitness_batch_calls = 0;
    double total_wall_seconds = 0.0;
};

}  // namespace gapa
