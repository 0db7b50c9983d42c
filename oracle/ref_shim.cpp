// TEST INFRASTRUCTURE — not part of the product.
//
// extern "C" shim over the UNMODIFIED reference library (the sources stay
// under /root/reference/proj and are compiled from there by oracle/Makefile
// into oracle/_ref/libgapa_ref.so).  ctypes in tests/ and bench.py's
// cpu_baseline / --impl reference legs call these entry points to
//   * validate the CSR restatement in oracle/gapa_oracle.c,
//   * generate the golden vectors under tests/golden/, and
//   * time the reference's own CPU path on the box's host cores.
// Nothing under paper_2412_20980_b200/ may link, load or call this file.
//
// Every function forwards to the reference symbol named in its comment.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "gapa/components.hpp"
#include "gapa/community.hpp"
#include "gapa/error.hpp"
#include "gapa/fitness.hpp"
#ifdef REF_HAVE_BENCH
#include "gapa/bench.hpp"
#endif
#include "gapa/ga_ops.hpp"
#include "gapa/gene_pool.hpp"
#include "gapa/generators.hpp"
#include "gapa/graph.hpp"
#include "gapa/link_prediction.hpp"
#include "gapa/modes.hpp"
#include "gapa/rng.hpp"

using namespace gapa;

namespace {

thread_local std::string g_error;

struct RefGraph {
    Graph graph;
};

struct RefSplit {
    LinkPredictionSplit split;
};

PopulationMatrix to_matrix(const std::int32_t* genes, int rows, int cols) {
    PopulationMatrix m(rows, cols);
    if (rows * static_cast<std::size_t>(cols) > 0)
        std::memcpy(m.data.data(), genes, sizeof(std::int32_t) * m.data.size());
    return m;
}

Direction to_direction(int minimize) { return minimize ? Direction::Minimize : Direction::Maximize; }

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 1;
    }
}

enum Task { kTaskPc = 0, kTaskMcn = 1, kTaskCda = 2, kTaskLpa = 3, kTaskSixDegrees = 4, kTaskCdaAdd = 5 };

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- rng.hpp ------------------------------------------------------------
std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }

// RngPolicy(seed).stream(generation, role, row): first `count` next_u64 draws.
void ref_stream_u64(std::uint64_t seed, std::uint64_t generation, std::uint64_t role,
                    std::uint64_t row, int count, std::uint64_t* out) {
    RngStream s = RngPolicy(seed).stream(generation, static_cast<StreamRole>(role), row);
    for (int i = 0; i < count; ++i) out[i] = s.next_u64();
}
void ref_stream_unit(std::uint64_t seed, std::uint64_t generation, std::uint64_t role,
                     std::uint64_t row, int count, double* out) {
    RngStream s = RngPolicy(seed).stream(generation, static_cast<StreamRole>(role), row);
    for (int i = 0; i < count; ++i) out[i] = s.next_unit();
}
void ref_stream_index(std::uint64_t seed, std::uint64_t generation, std::uint64_t role,
                      std::uint64_t row, std::uint32_t bound, int count, std::uint32_t* out) {
    RngStream s = RngPolicy(seed).stream(generation, static_cast<StreamRole>(role), row);
    for (int i = 0; i < count; ++i) out[i] = s.next_index(bound);
}

// ---- graph.hpp / generators.hpp ---------------------------------------------
void* ref_graph_from_edges(int n, int m, const std::int32_t* uv) {
    RefGraph* g = nullptr;
    guarded([&] {
        std::vector<std::pair<int, int>> edges;
        edges.reserve(m);
        for (int i = 0; i < m; ++i) edges.emplace_back(uv[2 * i], uv[2 * i + 1]);
        g = new RefGraph{Graph(n, std::move(edges))};
    });
    return g;
}
void* ref_graph_ba(int n, int attach, std::uint64_t seed) {
    RefGraph* g = nullptr;
    guarded([&] { g = new RefGraph{barabasi_albert(n, attach, seed)}; });
    return g;
}
void* ref_graph_er(int n, double p, std::uint64_t seed) {
    RefGraph* g = nullptr;
    guarded([&] { g = new RefGraph{erdos_renyi(n, p, seed)}; });
    return g;
}
void* ref_graph_sbm(int blocks, int block_size, double p_in, double p_out, std::uint64_t seed) {
    RefGraph* g = nullptr;
    guarded([&] { g = new RefGraph{planted_partition(blocks, block_size, p_in, p_out, seed)}; });
    return g;
}
void* ref_graph_load(const char* path) {
    RefGraph* g = nullptr;
    guarded([&] { g = new RefGraph{load_edge_list_file(path).graph}; });
    return g;
}
void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }
int ref_graph_n(void* g) { return static_cast<RefGraph*>(g)->graph.node_count(); }
int ref_graph_m(void* g) { return static_cast<RefGraph*>(g)->graph.edge_count(); }
// Canonical (u < v) pairs in insertion order (Graph::edges()).
void ref_graph_edges(void* g, std::int32_t* uv) {
    const auto& e = static_cast<RefGraph*>(g)->graph.edges();
    for (std::size_t i = 0; i < e.size(); ++i) {
        uv[2 * i] = e[i].first;
        uv[2 * i + 1] = e[i].second;
    }
}

// ---- gene_pool.hpp ------------------------------------------------------------
// kind: 0 EdgeRemoval, 1 EdgeAddition, 2 NodeRemoval (PoolKind order).
int ref_pool_size(void* g, int kind) {
    int size = -1;
    guarded([&] { size = build_gene_pool(static_cast<RefGraph*>(g)->graph, static_cast<PoolKind>(kind)).size(); });
    return size;
}
int ref_pool_genes(void* g, int kind, std::int32_t* u, std::int32_t* v) {
    return guarded([&] {
        const GenePool pool = build_gene_pool(static_cast<RefGraph*>(g)->graph, static_cast<PoolKind>(kind));
        for (int i = 0; i < pool.size(); ++i) {
            u[i] = pool.gene(i).u;
            v[i] = pool.gene(i).v;
        }
    });
}
int ref_budget(void* g, int kind, double rate) {
    int k = -1;
    guarded([&] { k = perturbation_budget(static_cast<RefGraph*>(g)->graph, static_cast<PoolKind>(kind), rate); });
    return k;
}

// ---- link_prediction.hpp --------------------------------------------------------
void* ref_split_build(void* g, double fraction, std::uint64_t seed) {
    RefSplit* s = nullptr;
    guarded([&] { s = new RefSplit{build_lp_split(static_cast<RefGraph*>(g)->graph, fraction, seed)}; });
    return s;
}
void ref_split_free(void* s) { delete static_cast<RefSplit*>(s); }
int ref_split_test_count(void* s) { return static_cast<int>(static_cast<RefSplit*>(s)->split.test_edges.size()); }
int ref_split_probe_count(void* s) { return static_cast<int>(static_cast<RefSplit*>(s)->split.probe_nonedges.size()); }
void ref_split_pairs(void* s, std::int32_t* test_uv, std::int32_t* probe_uv) {
    const auto& sp = static_cast<RefSplit*>(s)->split;
    for (std::size_t i = 0; i < sp.test_edges.size(); ++i) {
        test_uv[2 * i] = sp.test_edges[i].first;
        test_uv[2 * i + 1] = sp.test_edges[i].second;
    }
    for (std::size_t i = 0; i < sp.probe_nonedges.size(); ++i) {
        probe_uv[2 * i] = sp.probe_nonedges[i].first;
        probe_uv[2 * i + 1] = sp.probe_nonedges[i].second;
    }
}
// A new graph handle holding split.train (caller frees).
void* ref_split_train(void* s) { return new RefGraph{static_cast<RefSplit*>(s)->split.train}; }

// ---- fitness.hpp ---------------------------------------------------------------
// The reference's own pool builder + objective for a task code:
// 0 pc_fitness, 1 sixdst_fitness(Exact), 2 cda_fitness over the EdgeRemoval pool,
// 3 lpa_fitness (handle is a split; pool over split.train), 4 sixdst_fitness(SixDegrees),
// 5 cda_fitness over the EdgeAddition pool.
static void make_objective(void* g_or_split, int task, std::unique_ptr<GenePool>& pool,
                           std::unique_ptr<FitnessFunction>& fn) {
    if (task == kTaskLpa) {
        auto* s = static_cast<RefSplit*>(g_or_split);
        pool = std::make_unique<GenePool>(build_gene_pool(s->split.train, PoolKind::EdgeRemoval));
        fn = std::make_unique<LinkPredictionAttackObjective>(s->split, *pool);
        return;
    }
    auto* g = static_cast<RefGraph*>(g_or_split);
    if (task == kTaskCda || task == kTaskCdaAdd) {
        pool = std::make_unique<GenePool>(
            build_gene_pool(g->graph, task == kTaskCda ? PoolKind::EdgeRemoval : PoolKind::EdgeAddition));
        fn = std::make_unique<ModularityAttackObjective>(g->graph.adjacency(), *pool);
        return;
    }
    pool = std::make_unique<GenePool>(build_gene_pool(g->graph, PoolKind::NodeRemoval));
    if (task == kTaskPc)
        fn = std::make_unique<PairwiseConnectivityObjective>(g->graph.adjacency(), *pool);
    else
        fn = std::make_unique<SixDstObjective>(g->graph.adjacency(), *pool,
                                               task == kTaskSixDegrees ? ClosurePolicy::SixDegrees : ClosurePolicy::Exact);
}

// task 0: pc_fitness, 1: sixdst_fitness(Exact), 2: cda_fitness (edge-removal
// pool), 3: lpa_fitness (g_or_split is a split handle, pool over split.train).
// `threads` > 1 splits the rows over std::threads the way
// eval_with_ephemeral_workers does (contiguous partition_rows blocks).
int ref_eval_batch(void* g_or_split, int task, const std::int32_t* genes, int rows, int cols,
                   int threads, double* out) {
    return guarded([&] {
        const PopulationMatrix batch = to_matrix(genes, rows, cols);
        std::unique_ptr<GenePool> pool;
        std::unique_ptr<FitnessFunction> fn;
        make_objective(g_or_split, task, pool, fn);
        if (threads <= 1) {
            const FitnessVector fv = fn->evaluate_batch(batch);
            std::copy(fv.begin(), fv.end(), out);
            return;
        }
        const auto blocks = partition_rows(rows, threads);
        std::vector<std::thread> workers;
        std::vector<std::string> errors(threads);
        for (int w = 0; w < threads; ++w)
            workers.emplace_back([&, w] {
                try {
                    const FitnessVector fv = fn->evaluate_batch(batch.slice(blocks[w].first, blocks[w].second));
                    std::copy(fv.begin(), fv.end(), out + blocks[w].first);
                } catch (const std::exception& e) {
                    errors[w] = e.what();
                }
            });
        for (auto& t : workers) t.join();
        for (const auto& e : errors)
            if (!e.empty()) throw Error(e);
    });
}

// Unattacked references used by the identity tests.
double ref_modularity_unattacked(void* g) {
    double q = 0.0;
    guarded([&] {
        const BitMatrix a = static_cast<RefGraph*>(g)->graph.adjacency();
        q = modularity(a, detect_communities(a));
    });
    return q;
}
int ref_detect_communities(void* g, std::int32_t* assignment) {
    return guarded([&] {
        const CommunityPartition p = detect_communities(static_cast<RefGraph*>(g)->graph.adjacency());
        std::copy(p.assignment.begin(), p.assignment.end(), assignment);
    });
}
double ref_auc_unattacked(void* s) {
    double auc = 0.0;
    guarded([&] {
        auto* sp = static_cast<RefSplit*>(s);
        auc = evaluate_ra_predictor(sp->split, sp->split.train.adjacency()).auc;
    });
    return auc;
}
double ref_ra_score(void* g, int u, int v) {
    return ra_score(static_cast<RefGraph*>(g)->graph.adjacency(), u, v);
}

// ---- ga_ops.hpp ----------------------------------------------------------------
int ref_init_population_block(int pool_size, int row_first, int row_count, int budget,
                              std::uint64_t seed, std::uint64_t generation, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix p = init_population_block(pool_size, row_first, row_count, budget, RngPolicy(seed), generation);
        std::copy(p.data.begin(), p.data.end(), out);
    });
}
int ref_make_mask(int rows, int cols, double rate, int role, std::uint64_t seed, std::uint64_t generation, std::uint8_t* out) {
    return guarded([&] {
        const MaskMatrix m = role == 3 ? make_crossover_mask(rows, cols, rate, RngPolicy(seed), generation)
                                       : make_mutation_mask(rows, cols, rate, RngPolicy(seed), generation);
        std::copy(m.data.begin(), m.data.end(), out);
    });
}
int ref_make_mutation_indices(int rows, int cols, int pool_size, std::uint64_t seed, std::uint64_t generation, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix m = make_mutation_indices(rows, cols, pool_size, RngPolicy(seed), generation);
        std::copy(m.data.begin(), m.data.end(), out);
    });
}
int ref_selection_weights(const double* fitness, int s, int minimize, double* out) {
    return guarded([&] {
        const auto w = selection_weights(FitnessVector(fitness, fitness + s), to_direction(minimize));
        std::copy(w.begin(), w.end(), out);
    });
}
// Partner ROW INDEX per row, recomputed the way roulette_select does
// (weights -> cumulative -> weighted_pick on one Select draw per row), and the
// partner matrix roulette_select itself returns.
int ref_roulette_select(const std::int32_t* pop, int s, int k, const double* fitness, int minimize,
                        std::uint64_t seed, std::uint64_t generation,
                        std::int32_t* partner_index, std::int32_t* partners) {
    return guarded([&] {
        const PopulationMatrix p = to_matrix(pop, s, k);
        const FitnessVector f(fitness, fitness + s);
        const RngPolicy rng(seed);
        const PopulationMatrix out = roulette_select(p, f, to_direction(minimize), rng, generation);
        if (partners) std::copy(out.data.begin(), out.data.end(), partners);
        if (partner_index) {
            const auto weights = selection_weights(f, to_direction(minimize));
            std::vector<double> cumulative(s);
            double total = 0.0;
            for (int i = 0; i < s; ++i) {
                total += weights[i];
                cumulative[i] = total;
            }
            for (int i = 0; i < s; ++i) {
                RngStream stream = rng.stream(generation, StreamRole::Select, static_cast<std::uint64_t>(i));
                partner_index[i] = weighted_pick(cumulative, stream.next_unit() * total);
            }
        }
    });
}
int ref_crossover(const std::int32_t* pop, const std::int32_t* partners, int s, int k, double pc,
                  std::uint64_t seed, std::uint64_t generation, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix c = crossover(to_matrix(pop, s, k), to_matrix(partners, s, k), pc, RngPolicy(seed), generation);
        std::copy(c.data.begin(), c.data.end(), out);
    });
}
int ref_mutate_block(const std::int32_t* block, int rows, int k, int row_offset, double pm,
                     int pool_size, std::uint64_t seed, std::uint64_t generation, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix m = mutate_block(to_matrix(block, rows, k), row_offset, pm, pool_size, RngPolicy(seed), generation);
        std::copy(m.data.begin(), m.data.end(), out);
    });
}
int ref_mutate(const std::int32_t* c_pop, int s, int k, double pm, int pool_size,
               std::uint64_t seed, std::uint64_t generation, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix m = mutate(to_matrix(c_pop, s, k), pm, pool_size, RngPolicy(seed), generation);
        std::copy(m.data.begin(), m.data.end(), out);
    });
}
int ref_elitism(const std::int32_t* pop, const std::int32_t* m_pop, int s, int k,
                const double* fit_pop, const double* fit_m, int minimize,
                std::int32_t* next, double* next_fit) {
    return guarded([&] {
        auto [p, f] = elitism(to_matrix(pop, s, k), to_matrix(m_pop, s, k), FitnessVector(fit_pop, fit_pop + s),
                              FitnessVector(fit_m, fit_m + s), to_direction(minimize));
        std::copy(p.data.begin(), p.data.end(), next);
        std::copy(f.begin(), f.end(), next_fit);
    });
}
int ref_eda_sample(const std::int32_t* elite, int s, int k, int elite_count, int pool_size,
                   std::uint64_t seed, std::uint64_t generation, int smoothing, std::int32_t* out) {
    return guarded([&] {
        const PopulationMatrix e = eda_sample(to_matrix(elite, s, k), elite_count, pool_size, RngPolicy(seed), generation, smoothing != 0);
        std::copy(e.data.begin(), e.data.end(), out);
    });
}
void ref_partition_rows(int pop_size, int pn, std::int32_t* lo_hi) {
    const auto blocks = partition_rows(pop_size, pn);
    for (int w = 0; w < pn; ++w) {
        lo_hi[2 * w] = blocks[w].first;
        lo_hi[2 * w + 1] = blocks[w].second;
    }
}

// ---- modes.hpp -----------------------------------------------------------------
// run_ga on one of the four objectives.  mode: 0 serial, 1 S, 2 SM, 3 M, 4 MNM.
// Outputs: history_best/mean[iterations], final_population[s*k],
// final_fitness[s]; returns wall seconds of the generation loop through
// *wall_seconds (RunResult::total_wall_seconds).
int ref_run_ga(void* g_or_split, int task, double pc, double pm, int pop_size, int budget,
               int iterations, int eda_interval, std::uint64_t seed, int mode, int pn, int qn,
               double* history_best, double* history_mean, std::int32_t* final_population,
               double* final_fitness, double* wall_seconds) {
    return guarded([&] {
        std::unique_ptr<GenePool> pool;
        std::unique_ptr<FitnessFunction> fn;
        make_objective(g_or_split, task, pool, fn);
        GAParams params;
        params.pc = pc;
        params.pm = pm;
        params.pop_size = pop_size;
        params.budget = budget;
        params.iterations = iterations;
        params.direction = Direction::Minimize;
        if (eda_interval > 0) params.eda_interval = eda_interval;
        params.seed = seed;
        ModeTopology topo;
        topo.mode = static_cast<Mode>(mode);
        topo.pn = pn;
        topo.qn = qn;
        const RunResult r = run_ga(params, *pool, *fn, topo);
        for (int i = 0; i < iterations; ++i) {
            history_best[i] = r.history[i].best;
            history_mean[i] = r.history[i].mean;
        }
        std::copy(r.final_population.data.begin(), r.final_population.data.end(), final_population);
        std::copy(r.final_fitness.begin(), r.final_fitness.end(), final_fitness);
        if (wall_seconds) *wall_seconds = r.total_wall_seconds;
    });
}

// ---- reporting metrics and the experiment driver ----------------------
double ref_nmi(const std::int32_t* a, const std::int32_t* b, int n) {
    double v = 0.0;
    guarded([&] {
        v = nmi(CommunityPartition{std::vector<int>(a, a + n)}, CommunityPartition{std::vector<int>(b, b + n)});
    });
    return v;
}
// detect_communities on the perturbed graph; kind 0 EdgeRemoval / 1 EdgeAddition pool of build_gene_pool
int ref_detect_perturbed(void* g, int kind, const std::int32_t* genes, int cols, std::int32_t* assignment) {
    return guarded([&] {
        const Graph& graph = static_cast<RefGraph*>(g)->graph;
        const GenePool pool = build_gene_pool(graph, static_cast<PoolKind>(kind));
        const BitMatrix attacked = apply_perturbation(graph.adjacency(), pool, std::span<const std::int32_t>(genes, cols));
        const CommunityPartition p = detect_communities(attacked);
        std::copy(p.assignment.begin(), p.assignment.end(), assignment);
    });
}
// evaluate_ra_predictor on the perturbed train graph: out = {auc, precision}; scores = T test then P probe
int ref_lp_metrics(void* s, const std::int32_t* genes, int cols, double* out, double* scores) {
    return guarded([&] {
        auto* sp = static_cast<RefSplit*>(s);
        const GenePool pool = build_gene_pool(sp->split.train, PoolKind::EdgeRemoval);
        const BitMatrix attacked = apply_perturbation(sp->split.train.adjacency(), pool, std::span<const std::int32_t>(genes, cols));
        const LpMetrics m = evaluate_ra_predictor(sp->split, attacked);
        out[0] = m.auc;
        out[1] = m.precision;
        if (scores) {
            const auto t = ra_scores(attacked, sp->split.test_edges), p = ra_scores(attacked, sp->split.probe_nonedges);
            std::copy(t.begin(), t.end(), scores);
            std::copy(p.begin(), p.end(), scores + t.size());
        }
    });
}
#ifdef REF_HAVE_BENCH
// bench::run_experiment / sweep on a JSON config (bench.cpp:142-366); CSV text into `csv` (NUL-terminated).
// axis: "" = run_experiment, "pop_size" / "pn" = sweep over `values`.
int ref_run_experiment(const char* config_json, const char* axis, const int* values, int n_values, char* csv, int capacity) {
    return guarded([&] {
        const bench::ExperimentConfig cfg = bench::parse_config(config_json);
        const std::string ax = axis ? axis : "";
        const auto rows = ax.empty() ? bench::run_experiment(cfg)
                                     : bench::sweep(cfg, bench::axis_from_string(ax), std::vector<int>(values, values + n_values));
        const std::string text = bench::report(rows, bench::ReportFormat::Csv);
        if (static_cast<int>(text.size()) + 1 > capacity) throw Error("ref_run_experiment: csv buffer too small");
        std::copy(text.begin(), text.end(), csv);
        csv[text.size()] = 0;
    });
}
int ref_csv_without_wall_time(const char* csv_in, char* out, int capacity) {
    return guarded([&] {
        const std::string text = bench::csv_without_wall_time(csv_in);
        if (static_cast<int>(text.size()) + 1 > capacity) throw Error("ref_csv_without_wall_time: buffer too small");
        std::copy(text.begin(), text.end(), out);
        out[text.size()] = 0;
    });
}
int ref_have_bench() { return 1; }
#else
int ref_have_bench() { return 0; }
#endif

}  // extern "C"
