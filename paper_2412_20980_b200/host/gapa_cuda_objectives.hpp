// Host C++ side of the drop-in: FitnessFunction objectives and ga_ops-shaped free
// functions whose compute runs on the B200 through the C ABI of include/gapa_cuda.h.
//
// Two build modes, same source:
//   -DGAPA_B200_USE_REFERENCE_HEADERS   the adapters derive from the REAL
//        gapa::FitnessFunction (include/gapa/fitness.hpp:17-27) and take the reference's
//        own Graph / GenePool / PopulationMatrix, so run_ga() of the unmodified reference
//        (src/modes.cpp) drives the GPU objectives unchanged — see INTEGRATION.md and
//        oracle/ref_gpu_driver.cpp;
//   default                             the same adapters over gapa_api_mirror.hpp, for
//        boxes where the reference sources do not exist.
//
// libgapa_cuda.so is opened with dlopen (path from $GAPA_CUDA_LIB, else next to this
// header's package); a non-zero C-ABI status becomes `throw gapa::Error`
// (include/gapa/error.hpp:9-12).  There is no CPU fallback: without the library or a GPU
// construction throws.
#pragma once

#ifdef GAPA_B200_USE_REFERENCE_HEADERS
#include "gapa/accessibility.hpp"
#include "gapa/error.hpp"
#include "gapa/fitness.hpp"
#include "gapa/ga_ops.hpp"
#include "gapa/gene_pool.hpp"
#include "gapa/graph.hpp"
#include "gapa/link_prediction.hpp"
#include "gapa/modes.hpp"
#include "gapa/population.hpp"
#else
#include "gapa_api_mirror.hpp"
#endif

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "gapa_cuda.h"

namespace gapa_b200 {

// ---- the C ABI, resolved at run time ------------------------------------------------------
class CudaLib {
public:
    static const CudaLib& get() {
        static CudaLib lib;
        return lib;
    }
#define GAPA_B200_SYM(name) decltype(&::name) name = nullptr;
    GAPA_B200_SYM(gapa_cuda_last_error)
    GAPA_B200_SYM(gapa_cuda_graph_create)
    GAPA_B200_SYM(gapa_cuda_destroy)
    GAPA_B200_SYM(gapa_cuda_pool_set)
    GAPA_B200_SYM(gapa_cuda_lp_split_set)
    GAPA_B200_SYM(gapa_cuda_eval_batch)
    GAPA_B200_SYM(gapa_cuda_ga_init)
    GAPA_B200_SYM(gapa_cuda_ga_selection_weights)
    GAPA_B200_SYM(gapa_cuda_ga_select)
    GAPA_B200_SYM(gapa_cuda_ga_crossover_mutate)
    GAPA_B200_SYM(gapa_cuda_ga_mutate)
    GAPA_B200_SYM(gapa_cuda_ga_eda)
    GAPA_B200_SYM(gapa_cuda_ga_elitism)
    GAPA_B200_SYM(gapa_cuda_run)
#undef GAPA_B200_SYM

    void check(int status) const {
        if (status != GAPA_CUDA_OK) throw gapa::Error(gapa_cuda_last_error());
    }

private:
    CudaLib() {
        const char* env = std::getenv("GAPA_CUDA_LIB");
        const std::string path = env ? env : "libgapa_cuda.so";
        handle_ = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
        if (!handle_) throw gapa::Error(std::string("cannot load the CUDA hot path (no CPU fallback): ") + dlerror());
#define GAPA_B200_SYM(name)                                             \
    name = reinterpret_cast<decltype(name)>(dlsym(handle_, #name));      \
    if (!name) throw gapa::Error("libgapa_cuda.so does not export " #name);
        GAPA_B200_SYM(gapa_cuda_last_error)
        GAPA_B200_SYM(gapa_cuda_graph_create)
        GAPA_B200_SYM(gapa_cuda_destroy)
        GAPA_B200_SYM(gapa_cuda_pool_set)
        GAPA_B200_SYM(gapa_cuda_lp_split_set)
        GAPA_B200_SYM(gapa_cuda_eval_batch)
        GAPA_B200_SYM(gapa_cuda_ga_init)
        GAPA_B200_SYM(gapa_cuda_ga_selection_weights)
        GAPA_B200_SYM(gapa_cuda_ga_select)
        GAPA_B200_SYM(gapa_cuda_ga_crossover_mutate)
        GAPA_B200_SYM(gapa_cuda_ga_mutate)
        GAPA_B200_SYM(gapa_cuda_ga_eda)
        GAPA_B200_SYM(gapa_cuda_ga_elitism)
        GAPA_B200_SYM(gapa_cuda_run)
#undef GAPA_B200_SYM
    }
    void* handle_ = nullptr;
};

// ---- one GPU's copy of the problem -----------------------------------------------------------
class DeviceProblem {
public:
    DeviceProblem(const gapa::Graph& g, const gapa::GenePool& pool, int device) {
        const auto& lib = CudaLib::get();
        std::vector<std::int32_t> uv;
        uv.reserve(2 * g.edges().size());
        for (auto [u, v] : g.edges()) {
            uv.push_back(u);
            uv.push_back(v);
        }
        lib.check(lib.gapa_cuda_graph_create(g.node_count(), g.edge_count(), uv.data(), device, &ctx_));
        std::vector<std::int32_t> pu(pool.size()), pv(pool.size());
        for (int i = 0; i < pool.size(); ++i) {
            pu[i] = pool.gene(i).u;
            pv[i] = pool.gene(i).v;
        }
        const int status = lib.gapa_cuda_pool_set(ctx_, static_cast<int>(pool.kind()), pool.size(), pu.data(), pv.data());
        if (status != GAPA_CUDA_OK) {
            const std::string what = lib.gapa_cuda_last_error();
            lib.gapa_cuda_destroy(ctx_);
            throw gapa::Error(what);
        }
    }
    DeviceProblem(const DeviceProblem&) = delete;
    DeviceProblem& operator=(const DeviceProblem&) = delete;
    ~DeviceProblem() {
        if (ctx_) CudaLib::get().gapa_cuda_destroy(ctx_);
    }
    void set_split(const gapa::LinkPredictionSplit& split) {
        auto flat = [](const std::vector<std::pair<int, int>>& src) {
            std::vector<std::int32_t> out;
            for (auto [u, v] : src) {
                out.push_back(u);
                out.push_back(v);
            }
            return out;
        };
        const auto t = flat(split.test_edges), p = flat(split.probe_nonedges);
        const auto& lib = CudaLib::get();
        lib.check(lib.gapa_cuda_lp_split_set(ctx_, static_cast<int>(split.test_edges.size()), t.data(),
                                             static_cast<int>(split.probe_nonedges.size()), p.data()));
    }
    gapa::FitnessVector evaluate(int task, const std::int32_t* genes, int rows, int cols) const {
        gapa::FitnessVector out(rows);
        const auto& lib = CudaLib::get();
        lib.check(lib.gapa_cuda_eval_batch(ctx_, task, genes, rows, cols, out.data()));
        return out;
    }
    gapa_cuda_ctx* handle() const { return ctx_; }

private:
    gapa_cuda_ctx* ctx_ = nullptr;
};

inline void require_kind(const gapa::GenePool& pool, gapa::PoolKind kind, const char* what) {  // fitness.cpp:50-52
    if (pool.kind() != kind) throw gapa::Error(std::string(what) + ": incompatible gene pool kind");
}

// ---- objectives (fitness.hpp:56-101) -------------------------------------------------------------
class CudaObjective : public gapa::FitnessFunction {
public:
    gapa::Direction direction() const override { return gapa::Direction::Minimize; }
    double evaluate_one(std::span<const std::int32_t> genes) const override {
        return problem_.evaluate(task_, genes.data(), 1, static_cast<int>(genes.size()))[0];
    }
    // The optimisation the reference's contract allows ("never a semantic change",
    // fitness.hpp:24-25): the whole batch in one pass on the GPU.
    gapa::FitnessVector evaluate_batch(const gapa::PopulationMatrix& batch) const override {
        return problem_.evaluate(task_, batch.data.data(), batch.rows, batch.cols);
    }
    const DeviceProblem& problem() const { return problem_; }
    int task() const { return task_; }

protected:
    CudaObjective(int task, const gapa::Graph& g, const gapa::GenePool& pool, int device)
        : task_(task), problem_(g, pool, device) {}
    int task_;
    DeviceProblem problem_;
};

class CudaPairwiseConnectivityObjective : public CudaObjective {  // fitness.hpp:68-77
public:
    CudaPairwiseConnectivityObjective(const gapa::Graph& g, const gapa::GenePool& pool, int device = 0)
        : CudaObjective((require_kind(pool, gapa::PoolKind::NodeRemoval, "PairwiseConnectivityObjective"), GAPA_TASK_PC), g, pool, device) {}
};
// fitness.hpp:56-66.  Exact closure = largest component (the PC kernels); SixDegrees = largest
// radius-8 ball (accessibility.hpp:12-14), the truncated multi-source BFS kernel.
class CudaSixDstObjective : public CudaObjective {
public:
    CudaSixDstObjective(const gapa::Graph& g, const gapa::GenePool& pool,
                        gapa::ClosurePolicy policy = gapa::ClosurePolicy::Exact, int device = 0)
        : CudaObjective((require_kind(pool, gapa::PoolKind::NodeRemoval, "SixDstObjective"),
                         policy == gapa::ClosurePolicy::Exact ? GAPA_TASK_MCN : GAPA_TASK_SIXDST),
                        g, pool, device) {}
};
class CudaModularityAttackObjective : public CudaObjective {  // fitness.hpp:79-88
public:
    CudaModularityAttackObjective(const gapa::Graph& g, const gapa::GenePool& pool, int device = 0)
        : CudaObjective((pool.kind() == gapa::PoolKind::NodeRemoval
                             ? throw gapa::Error("ModularityAttackObjective: incompatible gene pool kind") : 0, GAPA_TASK_CDA),
                        g, pool, device) {}
};
class CudaLinkPredictionAttackObjective : public CudaObjective {  // fitness.hpp:90-101
public:
    CudaLinkPredictionAttackObjective(const gapa::LinkPredictionSplit& split, const gapa::GenePool& pool, int device = 0)
        : CudaObjective((require_kind(pool, gapa::PoolKind::EdgeRemoval, "LinkPredictionAttackObjective"), GAPA_TASK_LPA),
                        split.train, pool, device) {
        problem_.set_split(split);
    }
};

// ---- ga_ops.hpp:30-93 on the GPU (host-buffer forms) -------------------------------------------------
inline int as_minimize(gapa::Direction d) { return d == gapa::Direction::Minimize ? 1 : 0; }

inline gapa::PopulationMatrix init_population_block(int pool_size, int row_first, int row_count, int budget,
                                                    std::uint64_t seed, std::uint64_t generation = 0, int device = 0) {
    gapa::PopulationMatrix out(row_count, budget);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_init(device, pool_size, row_first, row_count, budget, seed, generation, out.data.data()));
    return out;
}
inline gapa::PopulationMatrix init_population(int pool_size, int pop_size, int budget, std::uint64_t seed,
                                              std::uint64_t generation = 0, int device = 0) {
    return init_population_block(pool_size, 0, pop_size, budget, seed, generation, device);
}
inline std::vector<double> selection_weights(const gapa::FitnessVector& fitness, gapa::Direction direction, int device = 0) {
    std::vector<double> w(fitness.size());
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_selection_weights(device, fitness.data(), static_cast<int>(fitness.size()), as_minimize(direction), w.data()));
    return w;
}
// roulette_select (ga_ops.cpp:105-128): partner rows, sampled with replacement
inline gapa::PopulationMatrix roulette_select(const gapa::PopulationMatrix& pop, const gapa::FitnessVector& fitness,
                                              gapa::Direction direction, std::uint64_t seed, std::uint64_t generation,
                                              int device = 0) {
    if (static_cast<int>(fitness.size()) != pop.rows) throw gapa::Error("roulette_select: fitness length mismatch");
    std::vector<std::int32_t> idx(pop.rows);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_select(device, fitness.data(), pop.rows, as_minimize(direction), seed, generation, idx.data()));
    gapa::PopulationMatrix partners(pop.rows, pop.cols);
    for (int i = 0; i < pop.rows; ++i) std::copy(pop.row(idx[i]).begin(), pop.row(idx[i]).end(), partners.row(i).begin());
    return partners;
}
// crossover (ga_ops.cpp:141-144) and mutate (:157-162) in the reference's shapes
inline gapa::PopulationMatrix crossover(const gapa::PopulationMatrix& pop, const gapa::PopulationMatrix& partners, double pc,
                                        std::uint64_t seed, std::uint64_t generation, int device = 0) {
    if (pop.rows != partners.rows || pop.cols != partners.cols) throw gapa::Error("crossover: shape mismatch");
    const int s = pop.rows, k = pop.cols;
    std::vector<std::int32_t> stacked(pop.data);
    stacked.insert(stacked.end(), partners.data.begin(), partners.data.end());
    std::vector<std::int32_t> idx(2 * s);
    for (int i = 0; i < 2 * s; ++i) idx[i] = s + (i % s);  // partner of row i is stacked row s + i
    gapa::PopulationMatrix out(s, k);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_crossover_mutate(device, stacked.data(), idx.data(), 2 * s, k, 0, s, pc, 0.0, 1, seed, generation, out.data.data()));
    return out;
}
inline gapa::PopulationMatrix mutate_block(const gapa::PopulationMatrix& block, int row_offset, double pm, int pool_size,
                                           std::uint64_t seed, std::uint64_t generation, int device = 0) {
    gapa::PopulationMatrix out(block.rows, block.cols);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_mutate(device, block.data.data(), block.rows, block.cols, row_offset, pm, pool_size, seed, generation, out.data.data()));
    return out;
}
inline gapa::PopulationMatrix mutate(const gapa::PopulationMatrix& c_pop, double pm, int pool_size, std::uint64_t seed,
                                     std::uint64_t generation, int device = 0) {
    return mutate_block(c_pop, 0, pm, pool_size, seed, generation, device);
}
inline std::pair<gapa::PopulationMatrix, gapa::FitnessVector> elitism(const gapa::PopulationMatrix& pop,
                                                                      const gapa::PopulationMatrix& m_pop,
                                                                      const gapa::FitnessVector& fit_pop,
                                                                      const gapa::FitnessVector& fit_m,
                                                                      gapa::Direction direction, int device = 0) {
    const int s = pop.rows;
    if (m_pop.rows != s || m_pop.cols != pop.cols) throw gapa::Error("elitism: shape mismatch");
    if (static_cast<int>(fit_pop.size()) != s || static_cast<int>(fit_m.size()) != s) throw gapa::Error("elitism: fitness length mismatch");
    gapa::PopulationMatrix next(s, pop.cols);
    gapa::FitnessVector next_fit(s);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_elitism(device, pop.data.data(), m_pop.data.data(), s, pop.cols, fit_pop.data(), fit_m.data(),
                                       as_minimize(direction), next.data.data(), next_fit.data()));
    return {std::move(next), std::move(next_fit)};
}
inline gapa::PopulationMatrix eda_sample(const gapa::PopulationMatrix& elite, int elite_count, int pool_size, std::uint64_t seed,
                                         std::uint64_t generation, bool add_one_smoothing = true, int device = 0) {
    gapa::PopulationMatrix out(elite.rows, elite.cols);
    const auto& lib = CudaLib::get();
    lib.check(lib.gapa_cuda_ga_eda(device, elite.data.data(), elite.rows, elite.cols, elite_count, pool_size, seed, generation,
                                   add_one_smoothing ? 1 : 0, out.data.data()));
    return out;
}

// ---- run_ga, Mode::S, population resident in HBM (modes.cpp:132-178) ------------------------------------
inline gapa::RunResult run_ga_cuda(const gapa::GAParams& params, const CudaObjective& objective) {
    gapa_cuda_run_params p{};
    p.pc = params.pc;
    p.pm = params.pm;
    p.pop_size = params.pop_size;
    p.budget = params.budget;
    p.iterations = params.iterations;
    p.minimize = as_minimize(params.direction);
    p.eda_interval = params.eda_interval ? *params.eda_interval : 0;
    if (params.eda_interval && *params.eda_interval < 1) throw gapa::ConfigError("eda_interval must be >= 1");
    p.task = objective.task();
    p.seed = params.seed;
    p.rank = 0;
    p.world = 1;
    const int s = std::max(params.pop_size, 0), k = std::max(params.budget, 0), it = std::max(params.iterations, 0);
    std::vector<double> best(it), mean(it), wall(it), compute(it), exch(it), life(it);
    std::vector<std::uint64_t> messages(it);
    gapa::RunResult out;
    out.final_population = gapa::PopulationMatrix(s, k);
    out.final_fitness.assign(s, 0.0);
    gapa_cuda_run_result r{};
    r.history_best = best.data();
    r.history_mean = mean.data();
    r.final_population = out.final_population.data.data();
    r.final_fitness = out.final_fitness.data();
    r.gen_wall_seconds = wall.data();  // GenerationStats timing columns: device time between CUDA events
    r.gen_compute_seconds = compute.data();
    r.gen_exchange_seconds = exch.data();
    r.gen_lifecycle_seconds = life.data();
    r.gen_messages = messages.data();
    const auto& lib = CudaLib::get();
    const int status = lib.gapa_cuda_run(objective.problem().handle(), &p, nullptr, nullptr, &r);
    if (status == GAPA_CUDA_E_INVALID) throw gapa::ConfigError(lib.gapa_cuda_last_error());
    lib.check(status);
    out.history.resize(it);
    for (int i = 0; i < it; ++i) {
        out.history[i].best = best[i];
        out.history[i].mean = mean[i];
        out.history[i].wall_seconds = wall[i];
        out.history[i].compute_seconds = compute[i];
        out.history[i].exchange_seconds = exch[i];
        out.history[i].lifecycle_seconds = life[i];
        out.history[i].messages = messages[i];
    }
    out.best_individual.assign(out.final_population.row(0).begin(), out.final_population.row(0).end());
    out.best_fitness = out.final_fitness.front();
    out.fitness_batch_calls = r.fitness_batch_calls;
    out.total_wall_seconds = r.total_wall_seconds;
    return out;
}

}  // namespace gapa_b200
