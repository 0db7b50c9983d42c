// TEST INFRASTRUCTURE — drop-in proof, built only where /root/reference exists
// (oracle/Makefile target ref_gpu_driver -> oracle/_ref/ref_gpu_driver; the binary travels
// to the GPU box, the reference sources do not).
//
// Links the UNMODIFIED reference (graph, generators, gene_pool, ga_ops, fitness, modes, ...)
// and hands its own run_ga() the CUDA objectives of
// paper_2412_20980_b200/host/gapa_cuda_objectives.hpp, which derive from the real
// gapa::FitnessFunction.  Every run must equal the reference's CPU objective bit for bit:
// history best AND mean, final population, final fitness (the comparison of
// tests/test_parallel.cpp:43-52).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gapa/generators.hpp"
#include "gapa_cuda_objectives.hpp"

using namespace gapa;

static int g_checks = 0, g_failed = 0;

static void expect(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        ++g_failed;
        std::printf("FAIL %s\n", what.c_str());
    }
}

static bool same_outputs(const RunResult& a, const RunResult& b) {
    if (!(a.final_population == b.final_population) || a.final_fitness != b.final_fitness) return false;
    if (a.best_individual != b.best_individual || a.best_fitness != b.best_fitness) return false;
    if (a.history.size() != b.history.size()) return false;
    for (std::size_t i = 0; i < a.history.size(); ++i)
        if (a.history[i].best != b.history[i].best || a.history[i].mean != b.history[i].mean) return false;
    return true;
}

static void compare_modes(const std::string& name, const GAParams& params, const GenePool& pool,
                          const FitnessFunction& cpu, const FitnessFunction& gpu) {
    const RunResult want = run_serial(params, pool, cpu);
    // the reference's own drivers, GPU objective plugged in: batch mode, ephemeral workers that call
    // evaluate_batch concurrently from several threads, persistent workers, nested shards
    expect(same_outputs(want, run_mode_s(params, pool, gpu)), name + " mode S");
    expect(same_outputs(want, run_mode_sm(params, pool, gpu, 4)), name + " mode SM pn=4");
    expect(same_outputs(want, run_mode_m(params, pool, gpu, 3)), name + " mode M pn=3");
    expect(same_outputs(want, run_mode_mnm(params, pool, gpu, 2, 2)), name + " mode MNM 2x2");
    expect(same_outputs(want, run_serial(params, pool, gpu)), name + " serial (evaluate_one)");
}

// `ref_gpu_driver e2e <n> <attach> <pop> <reps>`: the REAL plugin boundary, timed from C++ — the reference's own Graph, GenePool
// and PopulationMatrix (a pageable std::vector), FitnessFunction::evaluate_batch(const PopulationMatrix&) of the CUDA objective.
// One JSON line; the first three fitness values let the caller check them against the device path (same init stream).
static int bench_e2e(int n, int attach, int pop_rows, int reps) {
    const Graph g = barabasi_albert(n, attach, 1);
    const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
    const int k = perturbation_budget(g, PoolKind::NodeRemoval, 0.05);
    const gapa_b200::CudaPairwiseConnectivityObjective gpu(g, pool);
    const PopulationMatrix batch = init_population_block(pool.size(), 0, pop_rows, k, RngPolicy(1), 0);
    FitnessVector fit = gpu.evaluate_batch(batch);  // warm-up: scratch, pinned ring, learned schedule
    fit = gpu.evaluate_batch(batch);
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) fit = gpu.evaluate_batch(batch);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
    std::printf("{\"path\": \"gapa::FitnessFunction::evaluate_batch(const PopulationMatrix&) of CudaPairwiseConnectivityObjective, called from C++ on "
                "the reference's own types (pageable std::vector)\", \"n\": %d, \"m\": %d, \"k\": %d, \"pop\": %d, \"reps\": %d, "
                "\"seconds_per_call\": %.6f, \"evals_per_sec\": %.1f, \"h2d_bytes_per_call\": %.0f, \"fitness_head\": [%.1f, %.1f, %.1f]}\n",
                n, g.edge_count(), k, pop_rows, reps, sec, pop_rows / sec, 4.0 * pop_rows * k, fit[0], fit[1], fit[2]);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 6 && std::string(argv[1]) == "e2e") {
        try {
            return bench_e2e(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]));
        } catch (const std::exception& e) {
            std::printf("DROPIN_EXCEPTION %s\n", e.what());
            return 2;
        }
    }
    try {
        {  // BASELINE config 1
            const Graph g = barabasi_albert(1000, 2, 1);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            GAParams p;
            p.pc = 0.6; p.pm = 0.2; p.pop_size = 100; p.budget = 50; p.iterations = 30; p.seed = 1;
            const PairwiseConnectivityObjective cpu(g.adjacency(), pool);
            const gapa_b200::CudaPairwiseConnectivityObjective gpu(g, pool);
            compare_modes("config1 PC", p, pool, cpu, gpu);
            const RunResult r = gapa_b200::run_ga_cuda(p, gpu);  // HBM-resident loop
            expect(same_outputs(run_mode_s(p, pool, cpu), r), "config1 PC run_ga_cuda");
            expect(r.fitness_batch_calls == 31, "config1 batch-call count");
        }
        {  // acceptance criterion 6 instance (acceptance.cpp:151-185), golden final MCN 81
            const Graph g = erdos_renyi(100, 0.04, 665);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            GAParams p;
            p.pop_size = 20; p.budget = 10; p.iterations = 50; p.pc = 0.5; p.pm = 0.3; p.seed = 20240601;
            const SixDstObjective cpu(g.adjacency(), pool);
            const gapa_b200::CudaSixDstObjective gpu(g, pool);
            compare_modes("acceptance6 SixDST", p, pool, cpu, gpu);
            expect(run_mode_s(p, pool, gpu).best_fitness == 81.0, "acceptance6 final MCN 81");
        }
        {  // link-prediction attack, acceptance criterion 10 instance, shortened
            const Graph g = planted_partition(4, 16, 0.28, 0.02, 671);
            const LinkPredictionSplit split = build_lp_split(g, 0.1, 672);
            const GenePool pool = build_gene_pool(split.train, PoolKind::EdgeRemoval);
            GAParams p;
            p.pc = 0.7; p.pm = 0.1; p.pop_size = 50; p.iterations = 25; p.seed = 673;
            p.budget = perturbation_budget(split.train, PoolKind::EdgeRemoval, 0.1);
            const LinkPredictionAttackObjective cpu(split, pool);
            const gapa_b200::CudaLinkPredictionAttackObjective gpu(split, pool);
            compare_modes("LPA sbm64", p, pool, cpu, gpu);
        }
        {  // community-detection attack with an EDA generation every 4th
            const Graph g = planted_partition(4, 20, 0.3, 0.03, 1);
            const GenePool pool = build_gene_pool(g, PoolKind::EdgeRemoval);
            GAParams p;
            p.pc = 0.8; p.pm = 0.1; p.pop_size = 16; p.budget = 10; p.iterations = 12; p.seed = 2; p.eda_interval = 4;
            const ModularityAttackObjective cpu(g.adjacency(), pool);
            const gapa_b200::CudaModularityAttackObjective gpu(g, pool);
            compare_modes("CDA sbm80 + EDA", p, pool, cpu, gpu);
            expect(same_outputs(run_mode_s(p, pool, cpu), gapa_b200::run_ga_cuda(p, gpu)), "CDA run_ga_cuda with EDA");
        }
        {  // truncated closure (ClosurePolicy::SixDegrees) on a tree, where radius 8 matters
            const Graph g = barabasi_albert(300, 1, 668);
            const GenePool pool = build_gene_pool(g, PoolKind::NodeRemoval);
            GAParams p;
            p.pc = 0.5; p.pm = 0.3; p.pop_size = 24; p.iterations = 20; p.seed = 670;
            p.budget = perturbation_budget(g, PoolKind::NodeRemoval, 0.1);
            const SixDstObjective cpu(g.adjacency(), pool, ClosurePolicy::SixDegrees);
            const gapa_b200::CudaSixDstObjective gpu(g, pool, ClosurePolicy::SixDegrees);
            compare_modes("SixDST SixDegrees ba300", p, pool, cpu, gpu);
        }
        {  // acceptance criterion 8 instance (acceptance.cpp:207-246), EdgeAddition pool, shortened
            const Graph g = planted_partition(4, 9, 0.5, 0.05, 3);
            const GenePool pool = build_gene_pool(g, PoolKind::EdgeAddition);
            GAParams p;
            p.pc = 0.8; p.pm = 0.1; p.pop_size = 30; p.iterations = 20; p.seed = 667;
            p.budget = perturbation_budget(g, PoolKind::EdgeAddition, 0.1);
            const ModularityAttackObjective cpu(g.adjacency(), pool);
            const gapa_b200::CudaModularityAttackObjective gpu(g, pool);
            compare_modes("CDA EdgeAddition sbm36", p, pool, cpu, gpu);
        }
        {  // operator free functions in the reference's shapes
            const RngPolicy rng(9);
            const PopulationMatrix pop = init_population(500, 40, 17, rng);
            expect(pop == gapa_b200::init_population(500, 40, 17, 9), "init_population");
            FitnessVector f(40);
            for (int i = 0; i < 40; ++i) f[i] = (i * 7) % 11;
            const PopulationMatrix partners = roulette_select(pop, f, Direction::Minimize, rng, 3);
            expect(partners == gapa_b200::roulette_select(pop, f, Direction::Minimize, 9, 3), "roulette_select");
            expect(selection_weights(f, Direction::Maximize) == gapa_b200::selection_weights(f, Direction::Maximize), "selection_weights");
            const PopulationMatrix crossed = crossover(pop, partners, 0.6, rng, 3);
            expect(crossed == gapa_b200::crossover(pop, partners, 0.6, 9, 3), "crossover");
            const PopulationMatrix mutated = mutate(crossed, 0.2, 500, rng, 3);
            expect(mutated == gapa_b200::mutate(crossed, 0.2, 500, 9, 3), "mutate");
            expect(mutate_block(crossed.slice(5, 9), 5, 0.2, 500, rng, 3) == gapa_b200::mutate_block(crossed.slice(5, 9), 5, 0.2, 500, 9, 3), "mutate_block");
            FitnessVector fm(40);
            for (int i = 0; i < 40; ++i) fm[i] = (i * 5) % 11;
            expect(elitism(pop, mutated, f, fm, Direction::Minimize) == gapa_b200::elitism(pop, mutated, f, fm, Direction::Minimize), "elitism");
            expect(eda_sample(pop, 40, 500, rng, 8) == gapa_b200::eda_sample(pop, 40, 500, 9, 8), "eda_sample");
            bool threw = false;
            try {
                fm[3] = std::numeric_limits<double>::quiet_NaN();
                gapa_b200::elitism(pop, mutated, f, fm, Direction::Minimize);
            } catch (const Error&) { threw = true; }
            expect(threw, "elitism NaN -> gapa::Error");
            threw = false;
            try {
                const Graph g = barabasi_albert(50, 2, 1);
                const GenePool edge_pool = build_gene_pool(g, PoolKind::EdgeRemoval);
                gapa_b200::CudaPairwiseConnectivityObjective bad(g, edge_pool);
            } catch (const Error&) { threw = true; }
            expect(threw, "wrong pool kind -> gapa::Error");
        }
    } catch (const std::exception& e) {
        std::printf("DROPIN_EXCEPTION %s\n", e.what());
        return 2;
    }
    std::printf("%s %d checks, %d failed\n", g_failed ? "DROPIN_FAIL" : "DROPIN_OK", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
