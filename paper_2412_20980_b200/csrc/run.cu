// gapa_cuda_run: the generation loop of modes.cpp:132-178 (identical results to
// run_serial, modes.cpp:359-418) with the population resident in HBM.
//
//   gen 1:      init_population (generation key 0) -> evaluate
//   every gen:  roulette_select -> crossover -> mutate   (or eda_sample -> mutate)
//               -> evaluate(M_POP) -> elitism -> best = fit[0], mean = sum(fit)/s
//
// Sharding (world > 1) follows the reference's M mode (modes.cpp:190-349): rank r owns the
// partition_rows block r (modes.cpp:506-516) — it builds (crossover + mutate, or eda + mutate)
// and evaluates only those rows of M_POP.  Every rank keeps the whole parent population;
// selection and the elitism ranking are tiny and run redundantly; one all-gather of fitness
// doubles per evaluation is the ONLY exchange.  Surviving mutated rows of other ranks are
// recomputed from the replicated parents and the keyed streams (bit-identical by
// construction), so genomes never cross NVLink.
#include <chrono>
#include <cmath>

#include "internal.cuh"
#include "variation.cuh"

namespace gapa_b200 {
int launch_init(uint32_t, int, int, int, uint64_t, uint64_t, int32_t*, cudaStream_t);
int launch_select(const double*, int, int, uint64_t, uint64_t, int32_t*, double*, double*, int*, cudaStream_t);
int launch_crossover_mutate(const int32_t*, const int32_t*, int, int, int, double, double, uint32_t, uint64_t, uint64_t,
                            int32_t*, cudaStream_t);
int launch_mutate(const int32_t*, int, int, int, double, uint32_t, uint64_t, uint64_t, int32_t*, cudaStream_t);
int launch_eda(const int32_t*, int, int, int, int, uint32_t, uint64_t, uint64_t, int32_t*, cudaStream_t);
int launch_slots_identity(int, int32_t*, int32_t*, cudaStream_t);
int launch_slots_variation(int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int, int, double, double, uint32_t,
                           uint64_t, uint64_t, cudaStream_t);
int launch_slots_elitism(int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int, int, const double*, const double*,
                         int, double, double, uint32_t, uint64_t, uint64_t, int32_t*, int32_t*, double*, int32_t*, int*, cudaStream_t);
int launch_slots_gather(const int32_t*, const int32_t*, int, int, int32_t*, cudaStream_t);
int launch_slots_elitism_small(const int32_t*, const int32_t*, int, const double*, const double*, int, int32_t*, int32_t*, double*,
                               int32_t*, int*, double*, double*, int, uint64_t, uint64_t, int32_t*, double*, double*, cudaStream_t);
int launch_elitism_sharded(const int32_t*, const int32_t*, int, int, const int32_t*, int, int, const double*, const double*, int,
                           double, double, uint32_t, uint64_t, uint64_t, int32_t*, double*, int32_t*, int*, cudaStream_t);
int launch_elitism(const int32_t*, const int32_t*, int, int, const double*, const double*, int, int32_t*, double*, int32_t*,
                   int*, cudaStream_t);

// record_generation (modes.cpp:35-43): best = front, mean = SEQUENTIAL sum / s so that
// non-integer fitness reproduces std::accumulate bit for bit.
__global__ void __launch_bounds__(1024) k_ga_stats(const double* __restrict__ fit, int s, double* best, double* mean) {
    __shared__ double stage[4096];
    __shared__ double warp_sum[32];
    __shared__ int not_exact;
    const int tid = threadIdx.x;
    if (tid == 0) not_exact = 0;
    __syncthreads();
    // Integer-valued fitness whose running sums stay below 2^53 (PC, MCN) adds exactly in any order.
    double local = 0.0;
    const double bound = 9007199254740992.0 / static_cast<double>(s);
    for (int i = tid; i < s; i += blockDim.x) {
        const double x = fit[i];
        if (!(x == floor(x)) || !(fabs(x) < bound)) not_exact = 1;
        local += x;
    }
    __syncthreads();
    if (!not_exact) {
        for (int off = 16; off; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
        if ((tid & 31) == 0) warp_sum[tid >> 5] = local;
        __syncthreads();
        if (tid < 32) {
            double v = tid < (blockDim.x >> 5) ? warp_sum[tid] : 0.0;
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
        for (int i = tid; i < lim; i += blockDim.x) stage[i] = fit[base + i];
        __syncthreads();
        if (tid == 0)
            for (int i = 0; i < lim; ++i) sum += stage[i];
        __syncthreads();
    }
    if (tid == 0) {
        *best = fit[0];
        *mean = sum / static_cast<double>(s);
    }
}

__global__ void k_check_nan(const double* __restrict__ fit, int s, int* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s && isnan(fit[i])) *status = GAPA_CUDA_E_NAN;
}
}  // namespace gapa_b200

using namespace gapa_b200;

namespace {
struct RunBuffers {
    DevBuf pop, crossed, mutated, next, partner, fit, fit_m, fit_next, weights, cumulative, src_of_rank, status, hist;
    ~RunBuffers() {
        for (DevBuf* b : {&pop, &crossed, &mutated, &next, &partner, &fit, &fit_m, &fit_next, &weights, &cumulative,
                          &src_of_rank, &status, &hist})
            b->release();
    }
};

// Evaluation of a row block inside the loop.  Timing uses one CUDA-event pair per call, read back
// only when the run is over, so the loop itself never waits on the device for bookkeeping.
static constexpr int kTimingStride = 8;
static constexpr float kSampleBelowMs = 0.5f;  // evaluations shorter than this get sampled timing marks
struct EvalTimer {
    std::vector<cudaEvent_t> events;
    ~EvalTimer() { for (cudaEvent_t e : events) cudaEventDestroy(e); }
    int mark(cudaStream_t st) {
        cudaEvent_t e;
        GAPA_CUDA_TRY(cudaEventCreate(&e));
        events.push_back(e);
        GAPA_CUDA_TRY(cudaEventRecord(e, st));
        return GAPA_CUDA_OK;
    }
    int total_seconds(double* out) {
        double ms_total = 0.0;
        for (size_t i = 0; i + 1 < events.size(); i += 2) {
            float ms = 0.f;
            GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, events[i], events[i + 1]));
            ms_total += ms;
        }
        *out = ms_total * 1e-3;
        return GAPA_CUDA_OK;
    }
};

int eval_rows(gapa_cuda_ctx* ctx, int task, const GeneRows& view, int rows, double* out, cudaStream_t st, EvalTimer* timer,
              const VariationSpec* vary = nullptr) {
    if (rows == 0) return GAPA_CUDA_OK;
    if (timer) GAPA_TRY(timer->mark(st));
    int rc;
    if (task == GAPA_TASK_PC || task == GAPA_TASK_MCN) {
        rc = pc_eval(ctx, task, view, rows, out, st, true, vary);  // builds the children itself (fused with the mask build)
    } else {
        if (vary) GAPA_TRY(launch_variation_spec(*vary, view.cols, rows, st));
        rc = task == GAPA_TASK_CDA      ? cda_eval(ctx, view, rows, out, st)
             : task == GAPA_TASK_SIXDST ? sixdst_eval(ctx, view, rows, out, st, true)
                                        : lpa_eval(ctx, view, rows, out, st, true);
    }
    GAPA_TRY(rc);
    return timer ? timer->mark(st) : GAPA_CUDA_OK;
}
}  // namespace

extern "C" int gapa_cuda_ga_stats_device(const double* fit_dev, int s, double* best_dev, double* mean_dev, void* stream) {
    if (s < 1 || !fit_dev || !best_dev || !mean_dev) return fail(GAPA_CUDA_E_INVALID, "stats: bad arguments");
    GAPA_LAUNCH(k_ga_stats, 1, 1024, 0, static_cast<cudaStream_t>(stream), fit_dev, s, best_dev, mean_dev);
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_run(gapa_cuda_ctx* ctx, const gapa_cuda_run_params* p, gapa_cuda_allgather_fn exchange,
                             void* exchange_user, gapa_cuda_run_result* result) {
    if (!ctx || !p || !result) return fail(GAPA_CUDA_E_INVALID, "run: null argument");
    // GAParams::validate (ga_ops.cpp:11-17) + validate_for_run (modes.cpp:26-29)
    if (p->pop_size < 2) return fail(GAPA_CUDA_E_INVALID, "pop_size must be >= 2");
    if (p->budget < 1) return fail(GAPA_CUDA_E_INVALID, "budget must be >= 1");
    if (!(p->pc >= 0.0 && p->pc <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pc must be in [0, 1]");
    if (!(p->pm >= 0.0 && p->pm <= 1.0)) return fail(GAPA_CUDA_E_INVALID, "pm must be in [0, 1]");
    if (p->eda_interval < 0) return fail(GAPA_CUDA_E_INVALID, "eda_interval must be >= 1");
    if (p->iterations < 1) return fail(GAPA_CUDA_E_INVALID, "iterations must be >= 1");
    const int world = p->world < 1 ? 1 : p->world, rank = p->world < 1 ? 0 : p->rank;
    if (rank < 0 || rank >= world) return fail(GAPA_CUDA_E_INVALID, "run: rank outside world");
    if (world > 1 && !exchange) return fail(GAPA_CUDA_E_INVALID, "run: sharded run needs an exchange hook");
    if (ctx->pool_size < 1) return fail(GAPA_CUDA_E_INVALID, "init_population: empty gene pool");
    switch (p->task) {
        case GAPA_TASK_PC: case GAPA_TASK_MCN: case GAPA_TASK_SIXDST:
            if (ctx->pool_kind != GAPA_POOL_NODE_REMOVAL) return fail(GAPA_CUDA_E_INVALID, "run: incompatible gene pool kind");
            break;
        case GAPA_TASK_CDA:
            if (ctx->pool_kind == GAPA_POOL_NODE_REMOVAL) return fail(GAPA_CUDA_E_INVALID, "run: incompatible gene pool kind");
            break;
        case GAPA_TASK_LPA:
            if (ctx->pool_kind != GAPA_POOL_EDGE_REMOVAL || ctx->T < 1) return fail(GAPA_CUDA_E_INVALID, "run: link-prediction task needs an edge-removal pool and a split");
            break;
        default: return fail(GAPA_CUDA_E_INVALID, "unknown fitness task %d", p->task);
    }
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));

    const int s = p->pop_size, k = p->budget, iters = p->iterations, minimize = p->minimize ? 1 : 0;
    const uint32_t pool = static_cast<uint32_t>(ctx->pool_size);
    const int block = (s + world - 1) / world;  // partition_rows, modes.cpp:506-516
    const int lo = std::min(rank * block, s), hi = std::min(lo + block, s);
    const size_t cells = static_cast<size_t>(s) * k, padded = static_cast<size_t>(block) * world;
    cudaStream_t st = ctx->stream;

    // Population store: one pool of 2s row slots + parent / child slot tables (slot_kernels.cu).
    RunBuffers B;
    GAPA_TRY(B.pop.ensure(sizeof(int32_t) * 2 * cells));
    GAPA_TRY(B.next.ensure(sizeof(int32_t) * 4 * s));  // parent, child, next parent, next child tables
    GAPA_TRY(B.partner.ensure(sizeof(int32_t) * s));
    GAPA_TRY(B.fit.ensure(sizeof(double) * padded));
    GAPA_TRY(B.fit_m.ensure(sizeof(double) * padded));
    GAPA_TRY(B.fit_next.ensure(sizeof(double) * padded));
    GAPA_TRY(B.weights.ensure(sizeof(double) * s));
    GAPA_TRY(B.cumulative.ensure(sizeof(double) * s));
    GAPA_TRY(B.src_of_rank.ensure(sizeof(int32_t) * 2 * s));
    GAPA_TRY(B.status.ensure(sizeof(int)));
    GAPA_TRY(B.hist.ensure(sizeof(double) * 2 * iters));
    int32_t* pool_rows = B.pop.as<int32_t>();
    int32_t* parent = B.next.as<int32_t>();
    int32_t* child = parent + s;
    int32_t* next_parent = child + s;
    int32_t* next_child = next_parent + s;
    double* fit = B.fit.as<double>();
    double* fit_m = B.fit_m.as<double>();
    double* fit_next = B.fit_next.as<double>();
    double* hist = B.hist.as<double>();
    int* status = B.status.as<int>();
    GAPA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), st));
    GAPA_CUDA_TRY(cudaMemsetAsync(fit, 0, sizeof(double) * padded, st));
    GAPA_CUDA_TRY(cudaMemsetAsync(fit_m, 0, sizeof(double) * padded, st));

    result->fitness_batch_calls = 0;
    result->eval_seconds = 0.0;
    EvalTimer timer;
    // GenerationStats timing (modes.hpp:63-71): generation boundaries and the exchange hook are
    // bracketed by events on the run's stream; everything is read back after the loop.
    const bool want_stats = result->gen_wall_seconds || result->gen_compute_seconds || result->gen_exchange_seconds ||
                            result->gen_lifecycle_seconds || result->gen_messages;
    EvalTimer gen_marks, exchange_marks;
    std::vector<int> exchanges_in_gen(static_cast<size_t>(iters), 0);
    int current_gen = 1;
    // A timing event between two kernels costs ~5 us of device time.  A small population's generation is two launches
    // of 10-15 us, so there the marks are SAMPLED from generation 2 on: every kTimingStride-th generation is bracketed (its
    // evaluation and its boundary); eval_seconds is scaled by calls / timed calls and a block of generations shares its
    // mean wall time.  Larger populations start exact and switch to sampling at the first status poll (generation 16)
    // if an evaluation takes less than kSampleBelowMs.
    const bool small = world == 1 && 2 * s <= 1024;
    int stride = small ? kTimingStride : 1;  // larger populations switch at the first status poll if their evaluations are short
    int exact_until = 2;
    // generation 1 (initialisation, two evaluations, one-off set-up inside them) is always timed exactly
    auto sampled_gen = [&](int gen) { return gen <= exact_until || (gen - 2) % stride == 0; };
    EvalTimer first_timer;
    uint64_t later_calls = 0, later_timed_calls = 0;
    std::vector<int> marked_gens;  // generations (1-based) whose start carries a mark
    auto evaluate = [&](const int32_t* table, double* fit_all, const VariationSpec* vary = nullptr) -> int {  // rows [lo, hi) named by `table`
        ++result->fitness_batch_calls;
        const bool timed = sampled_gen(current_gen);
        if (current_gen > 1) {
            ++later_calls;
            later_timed_calls += timed;
        }
        GAPA_TRY(eval_rows(ctx, p->task, GeneRows{pool_rows, table + lo, k}, hi - lo, fit_all + lo, st,
                           current_gen == 1 ? &first_timer : timed ? &timer : nullptr, vary));
        if (world > 1) {
            if (want_stats) GAPA_TRY(exchange_marks.mark(st));
            const int rc = exchange(exchange_user, fit_all, s, block, st);
            if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "run: exchange hook failed with status %d", rc);
            if (want_stats) GAPA_TRY(exchange_marks.mark(st));
            ++exchanges_in_gen[current_gen - 1];
        }
        return GAPA_CUDA_OK;
    };
    auto check_status = [&](const char* what) -> int {
        int h = 0;
        GAPA_CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, st));
        GAPA_CUDA_TRY(cudaStreamSynchronize(st));
        if (h == GAPA_CUDA_E_NAN) return fail(GAPA_CUDA_E_NAN, "%s", what);
        return GAPA_CUDA_OK;
    };

    const auto t0 = std::chrono::steady_clock::now();
    for (int gen = 1; gen <= iters; ++gen) {
        current_gen = gen;
        if (want_stats && sampled_gen(gen)) {
            GAPA_TRY(gen_marks.mark(st));
            marked_gens.push_back(gen);
        }
        if (gen == 1) {
            GAPA_TRY(launch_slots_identity(s, parent, child, st));
            GAPA_TRY(launch_init(pool, 0, s, k, p->seed, 0, pool_rows, st));  // parents occupy slots 0..s-1
            GAPA_TRY(evaluate(parent, fit));
            GAPA_LAUNCH(k_check_nan, (s + 255) / 256, 256, 0, st, fit, s, status);
            GAPA_TRY(check_status("fitness evaluation failed during initialization"));  // modes.cpp:314-315
        }
        const uint64_t g = static_cast<uint64_t>(gen);
        // Children are built only for the rows this rank evaluates (all rows when world == 1).
        const bool eda_gen = p->eda_interval > 0 && gen % p->eda_interval == 0;  // modes.cpp:31-33,167-168
        const int32_t* partner = eda_gen ? nullptr : B.partner.as<int32_t>();
        if (!eda_gen && !(small && gen > 1))  // small populations: selected by the previous generation's elitism launch
            GAPA_TRY(launch_select(fit, s, minimize, p->seed, g, B.partner.as<int32_t>(), B.weights.as<double>(),
                                   B.cumulative.as<double>(), status, st));
        VariationSpec vary;  // the evaluation builds the children of rows [lo, hi) into their slots first
        vary.P = make_variation_params(p->pc, p->pm, pool, s, p->seed, g);
        vary.pool = pool_rows;
        vary.parent = parent;
        vary.child = child;
        vary.partner = partner;
        vary.row_first = lo;
        GAPA_TRY(evaluate(child, fit_m, &vary));
        // elitism permutes the slot tables; survivors built by other ranks are rebuilt in place
        // small populations: elitism, the generation's statistics AND the next generation's selection in one launch
        const bool select_next = gen < iters && !(p->eda_interval > 0 && (gen + 1) % p->eda_interval == 0);
        if (small)
            GAPA_TRY(launch_slots_elitism_small(parent, child, s, fit, fit_m, minimize, next_parent, next_child, fit_next,
                                                B.src_of_rank.as<int32_t>(), status, hist + (gen - 1), hist + iters + (gen - 1),
                                                select_next ? 1 : 0, p->seed, g + 1, B.partner.as<int32_t>(), B.weights.as<double>(),
                                                B.cumulative.as<double>(), st));
        else
            GAPA_TRY(launch_slots_elitism(pool_rows, parent, child, partner, s, k, lo, hi, fit, fit_m, minimize, p->pc, p->pm, pool,
                                          p->seed, g, next_parent, next_child, fit_next, B.src_of_rank.as<int32_t>(), status, st));
        std::swap(parent, next_parent);
        std::swap(child, next_child);
        std::swap(fit, fit_next);
        if (!small) GAPA_LAUNCH(k_ga_stats, 1, 1024, 0, st, fit, s, hist + (gen - 1), hist + iters + (gen - 1));
        // NaN / non-finite fitness is an Error in the reference (ga_ops.cpp:56-57, :189-192);
        // the flag is polled every few generations and at the end to keep the loop asynchronous.
        if ((gen & 15) == 0 || gen == iters) {
            int h = 0;
            GAPA_CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, st));
            GAPA_CUDA_TRY(cudaStreamSynchronize(st));
            if (h == GAPA_CUDA_E_NAN) return fail(GAPA_CUDA_E_NAN, "elitism: NaN fitness");
            if (stride == 1 && world == 1 && timer.events.size() >= 2) {  // the stream is idle: the last evaluation's time is known
                float ms = 0.f;
                GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, timer.events[timer.events.size() - 2], timer.events.back()));
                if (ms < kSampleBelowMs) {
                    stride = kTimingStride;
                    exact_until = gen + 1;  // the next generation carries a mark, so the exact block ends there
                }
            }
        }
    }
    if (want_stats) GAPA_TRY(gen_marks.mark(st));
    GAPA_CUDA_TRY(cudaStreamSynchronize(st));
    double first_seconds = 0.0;
    GAPA_TRY(first_timer.total_seconds(&first_seconds));
    GAPA_TRY(timer.total_seconds(&result->eval_seconds));
    if (later_timed_calls) result->eval_seconds *= static_cast<double>(later_calls) / static_cast<double>(later_timed_calls);
    result->eval_seconds += first_seconds;
    if (want_stats) {
        marked_gens.push_back(iters + 1);
        std::vector<float> wall_of_gen(static_cast<size_t>(iters), 0.f);
        for (size_t b = 0; b + 1 < marked_gens.size(); ++b) {  // a block of generations between two marks shares its mean
            float ms = 0.f;
            GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, gen_marks.events[b], gen_marks.events[b + 1]));
            const int g0 = marked_gens[b], g1 = marked_gens[b + 1];
            for (int gi = g0; gi < g1; ++gi) wall_of_gen[static_cast<size_t>(gi - 1)] = ms / static_cast<float>(g1 - g0);
        }
        size_t next_exchange = 0;
        for (int gi = 0; gi < iters; ++gi) {
            const float wall_ms = wall_of_gen[static_cast<size_t>(gi)];
            double exchange_s = 0.0;
            for (int e = 0; e < exchanges_in_gen[gi]; ++e, next_exchange += 2) {
                float ms = 0.f;
                GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, exchange_marks.events[next_exchange], exchange_marks.events[next_exchange + 1]));
                exchange_s += ms * 1e-3;
            }
            const double wall_s = wall_ms * 1e-3;
            if (result->gen_wall_seconds) result->gen_wall_seconds[gi] = wall_s;
            if (result->gen_exchange_seconds) result->gen_exchange_seconds[gi] = exchange_s;
            if (result->gen_lifecycle_seconds) result->gen_lifecycle_seconds[gi] = 0.0;
            if (result->gen_compute_seconds) result->gen_compute_seconds[gi] = std::max(0.0, wall_s - exchange_s);  // modes.cpp:38-40
            if (result->gen_messages) result->gen_messages[gi] = static_cast<uint64_t>(exchanges_in_gen[gi]);
        }
    }
    result->total_wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    if (result->history_best) GAPA_CUDA_TRY(cudaMemcpy(result->history_best, hist, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    if (result->history_mean) GAPA_CUDA_TRY(cudaMemcpy(result->history_mean, hist + iters, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    if (result->final_population) {  // RunResult::final_population: the parents in best-first order
        DevBuf dense;
        GAPA_TRY(dense.ensure(sizeof(int32_t) * std::max<size_t>(cells, 1)));
        int rc = launch_slots_gather(pool_rows, parent, s, k, dense.as<int32_t>(), st);
        if (rc == GAPA_CUDA_OK && cudaMemcpyAsync(result->final_population, dense.ptr, sizeof(int32_t) * cells, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = GAPA_CUDA_E_CUDA;
        if (rc == GAPA_CUDA_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = GAPA_CUDA_E_CUDA;
        dense.release();
        if (rc != GAPA_CUDA_OK) return fail(rc, "run: could not materialise the final population");
    }
    if (result->final_fitness) GAPA_CUDA_TRY(cudaMemcpy(result->final_fitness, fit, sizeof(double) * s, cudaMemcpyDeviceToHost));
    return GAPA_CUDA_OK;
}
