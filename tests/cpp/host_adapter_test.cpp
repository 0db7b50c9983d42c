// Host C++ adapters in mirror mode (no reference headers): the parity cases read like the
// reference's own tests (tests/test_fitness.cpp:154-162, :279-307, :378-394) with golden
// values produced by the unmodified reference (tests/golden/).
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>

#include "gapa_cuda_objectives.hpp"

using namespace gapa;
namespace gb = gapa_b200;

static int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                     \
    do {                                                                \
        ++g_checks;                                                     \
        if (!(cond)) { ++g_failed; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)

static Graph complete_graph(int n) {
    std::vector<std::pair<int, int>> e;
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v) e.emplace_back(u, v);
    return Graph(n, e);
}

int main() {
    try {
        {  // PC fixed values: K5 -> 10, everything removed -> 0
            const Graph g = complete_graph(5);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            const gb::CudaPairwiseConnectivityObjective pc(g, pool);
            const gb::CudaSixDstObjective mcn(g, pool);
            CHECK(pc.direction() == Direction::Minimize);
            CHECK(pc.evaluate_one({}) == 10.0);
            const std::vector<std::int32_t> all = {0, 1, 2, 3, 4};
            CHECK(pc.evaluate_one(all) == 0.0);
            CHECK(mcn.evaluate_one(all) == 1.0);
            PopulationMatrix batch(3, 2);
            batch.data = {0, 0, 0, 1, 3, 4};
            const FitnessVector f = pc.evaluate_batch(batch);
            CHECK(f.size() == 3 && f[0] == 6.0 && f[1] == 3.0 && f[2] == 3.0);
            for (int i = 0; i < 3; ++i) CHECK(f[i] == pc.evaluate_one(batch.row(i)));  // batch == per-row
            CHECK(pc.evaluate_batch(PopulationMatrix(0, 2)).empty());
            bool threw = false;
            try { pc.evaluate_one(std::vector<std::int32_t>{7}); } catch (const Error&) { threw = true; }
            CHECK(threw);  // gene id out of range
            threw = false;
            try { gb::CudaPairwiseConnectivityObjective bad(g, build_gene_pool(g, PoolKind::EdgeRemoval)); } catch (const Error&) { threw = true; }
            CHECK(threw);  // pool-kind enforcement
        }
        {  // truncated closure on P40 (test_fitness.cpp:94-103): radius-8 balls, not the whole path
            std::vector<std::pair<int, int>> e;
            for (int u = 0; u + 1 < 40; ++u) e.emplace_back(u, u + 1);
            const Graph g(40, e);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            const gb::CudaSixDstObjective six(g, pool, ClosurePolicy::SixDegrees);
            const gb::CudaSixDstObjective exact(g, pool);
            CHECK(six.evaluate_one({}) == 17.0);
            CHECK(exact.evaluate_one({}) == 40.0);
            CHECK(six.evaluate_one(std::vector<std::int32_t>{8, 25}) == 16.0);
        }
        {  // EdgeAddition pool (gene_pool.cpp:81-87): two triangles, adding the three cross pairs of node 0
            const Graph g(6, {{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}});
            const GenePool pool = build_gene_pool(g, PoolKind::EdgeAddition);
            CHECK(pool.size() == 9 && pool.gene(0).u == 0 && pool.gene(0).v == 3 && pool.gene(8).u == 2 && pool.gene(8).v == 5);
            const gb::CudaModularityAttackObjective cda(g, pool);
            CHECK(cda.evaluate_one({}) == 0.5);
            CHECK(cda.evaluate_one(std::vector<std::int32_t>{0, 0}) == cda.evaluate_one(std::vector<std::int32_t>{0}));
            CHECK(cda.evaluate_one(std::vector<std::int32_t>{0}) < 0.5);
        }
        {  // CDA identities: empty perturbation == unattacked Q, all edges removed == -0.5
            const Graph g(6, {{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}});
            const GenePool pool = build_gene_pool(g, PoolKind::EdgeRemoval);
            const gb::CudaModularityAttackObjective cda(g, pool);
            CHECK(cda.evaluate_one({}) == 0.5);
            const std::vector<std::int32_t> all = {0, 1, 2, 3, 4, 5};
            CHECK(cda.evaluate_one(all) == -0.5);
        }
        {  // init_population KAT + a tiny run: shape, monotone best, batch-call count
            const PopulationMatrix pop = gb::init_population(1000, 4, 6, 1);
            const std::int32_t want[6] = {939, 720, 805, 966, 231, 61};
            for (int j = 0; j < 6; ++j) CHECK(pop.at(0, j) == want[j]);
            CHECK(gb::selection_weights({5, 3, 3, 9}, Direction::Minimize) == (std::vector<double>{2, 3.5, 3.5, 1}));
            const Graph g = complete_graph(12);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            const gb::CudaPairwiseConnectivityObjective pc(g, pool);
            GAParams p;
            p.pop_size = 10; p.budget = 3; p.iterations = 6; p.seed = 4;
            const RunResult r = gb::run_ga_cuda(p, pc);
            CHECK(r.history.size() == 6 && r.fitness_batch_calls == 7);
            CHECK(r.final_population.rows == 10 && r.final_population.cols == 3);
            for (std::size_t i = 1; i < r.history.size(); ++i) CHECK(r.history[i].best <= r.history[i - 1].best);
            CHECK(r.best_fitness == r.final_fitness.front() && r.best_fitness == 36.0);  // 3 distinct nodes gone: C(9,2)
            bool threw = false;
            p.iterations = 0;
            try { gb::run_ga_cuda(p, pc); } catch (const ConfigError&) { threw = true; }
            CHECK(threw);  // iterations = 0 rejected (test_ga_engine.cpp:309-315)
        }
    } catch (const std::exception& e) {
        std::printf("HOST_ADAPTER_EXCEPTION %s\n", e.what());
        return 2;
    }
    std::printf("%s %d checks, %d failed\n", g_failed ? "HOST_ADAPTER_FAIL" : "HOST_ADAPTER_OK", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
