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
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstring>

#include "internal.cuh"
#include "variation.cuh"

namespace gapa_b200 {
int launch_init(uint32_t, int, int, int, uint64_t, uint64_t, int32_t*, cudaStream_t);
int launch_select(const double*, int, int, uint64_t, uint64_t, int32_t*, double*, double*, int*, cudaStream_t, double* stats_best = nullptr,
                  double* stats_mean = nullptr);
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
int launch_home_children(const int32_t*, int, int, int32_t*, cudaStream_t);
int launch_home_adopt(const int32_t*, const int32_t*, int, int, int, int32_t*, cudaStream_t);
int launch_fetch_rows(int32_t*, const int32_t* const*, int32_t*, const int32_t*, int, int, int, cudaStream_t);

// record_generation (modes.cpp:35-43): best = front, mean = SEQUENTIAL sum / s so that
// non-integer fitness reproduces std::accumulate bit for bit.
__global__ void __launch_bounds__(1024) k_ga_stats(const double* __restrict__ fit, int s, double* best, double* mean) {
    griddep_launch();
    griddep_wait();
    __shared__ GaStatsSmem sm;
    ga_stats_block(fit, s, best, mean, sm);
}

__global__ void k_check_nan(const double* __restrict__ fit, int s, int* status) {
    griddep_launch();
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s && isnan(fit[i])) *status = GAPA_CUDA_E_NAN;
}
}  // namespace gapa_b200

using namespace gapa_b200;

namespace {
struct RunBuffers {
    DevBuf pop, next, partner, fit, fit_m, fit_next, weights, cumulative, src_of_rank, status, hist;
    ~RunBuffers() {
        for (DevBuf* b : {&pop, &next, &partner, &fit, &fit_m, &fit_next, &weights, &cumulative, &src_of_rank, &status, &hist})
            b->release();
    }
};

// Timing marks: CUDA events recorded on the run's stream and read back only at the status polls (every 16
// generations, when the stream has just been synchronised anyway) and at the end — the loop never waits on the device
// for bookkeeping.  Events are recycled at every poll, so a long run holds a few dozen of them, not six per generation.
static constexpr int kTimingStride = 8;
static constexpr float kSampleBelowMs = 0.5f;  // evaluations shorter than this get sampled timing marks
struct EventPool {
    std::vector<cudaEvent_t> free_list;
    ~EventPool() { for (cudaEvent_t e : free_list) cudaEventDestroy(e); }
    int get(cudaEvent_t* out) {
        if (!free_list.empty()) {
            *out = free_list.back();
            free_list.pop_back();
            return GAPA_CUDA_OK;
        }
        GAPA_CUDA_TRY(cudaEventCreate(out));
        return GAPA_CUDA_OK;
    }
    void put(cudaEvent_t e) { free_list.push_back(e); }
};
// pairs of marks around something (an evaluation, an exchange): the sum of their spans
struct SpanTimer {
    EventPool* pool = nullptr;
    std::vector<cudaEvent_t> events;  // begin, end, begin, end, ...
    std::vector<int> tags;            // one per pair (the generation it belongs to)
    double ms_total = 0.0;
    float last_ms = -1.f;
    ~SpanTimer() { for (cudaEvent_t e : events) cudaEventDestroy(e); }
    int mark(cudaStream_t st, int tag = 0) {
        cudaEvent_t e;
        GAPA_TRY(pool->get(&e));
        events.push_back(e);
        if (events.size() & 1) tags.push_back(tag);
        GAPA_CUDA_TRY(cudaEventRecord(e, st));
        return GAPA_CUDA_OK;
    }
    // the stream is idle: fold every complete pair into the total (per_tag, when given, receives seconds per tag)
    int flush(std::vector<double>* per_tag = nullptr) {
        size_t i = 0;
        for (; i + 1 < events.size(); i += 2) {
            float ms = 0.f;
            GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, events[i], events[i + 1]));
            ms_total += ms;
            last_ms = ms;
            if (per_tag) (*per_tag)[static_cast<size_t>(tags[i / 2])] += ms * 1e-3;
            pool->put(events[i]);
            pool->put(events[i + 1]);
        }
        events.erase(events.begin(), events.begin() + static_cast<long>(i));
        tags.erase(tags.begin(), tags.begin() + static_cast<long>(i / 2));
        return GAPA_CUDA_OK;
    }
};

int eval_rows(gapa_cuda_ctx* ctx, int task, const GeneRows& view, int rows, double* out, cudaStream_t st, SpanTimer* timer,
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

// The resident state of one run (one rank of it): population store, fitness vectors, history, timing marks.
struct gapa_cuda_ga {
    gapa_cuda_ctx* ctx = nullptr;
    gapa_cuda_run_params p{};
    gapa_cuda_allgather_fn exchange = nullptr;
    void* exchange_user = nullptr;
    int world = 1, rank = 0, s = 0, k = 0, iters = 0, minimize = 1, block = 0, lo = 0, hi = 0;
    size_t cells = 0, padded = 0;
    uint32_t pool = 0;
    cudaStream_t st = nullptr;
    RunBuffers B;
    int32_t *pool_rows = nullptr, *parent = nullptr, *child = nullptr, *next_parent = nullptr, *next_child = nullptr;
    double *fit = nullptr, *fit_m = nullptr, *fit_next = nullptr, *hist = nullptr;
    int* status = nullptr;
    int gen_done = 0;
    uint64_t fitness_batch_calls = 0;
    double wall_seconds = 0.0;
    // timing
    bool want_stats = false, small = false;
    int stride = 1, exact_until = 2, current_gen = 1;
    EventPool events;
    SpanTimer timer, first_timer, exchange_marks;
    uint64_t later_calls = 0, later_timed_calls = 0;
    std::vector<double> exchange_of_gen, wall_of_gen;
    std::vector<int> exchanges_in_gen;
    std::vector<cudaEvent_t> gen_marks;  // boundaries not yet folded into wall_of_gen
    std::vector<int> marked_gens;        // the generation (1-based) each of them starts
    cudaEvent_t ev_adv0 = nullptr, ev_adv1 = nullptr;
    // Row-sharded run over PEER memory (the library's peer-mailbox communicator): slot tables are identical on every
    // rank, a rank holds only the rows it built or has read.  Surviving children of other ranks are neither rebuilt nor
    // broadcast: whoever needs one as a parent reads it from its builder's HBM over NVLink inside the variation kernel
    // and keeps a copy (variation.cuh: parent_row).  Safe without further synchronisation: a slot is overwritten only
    // when its row has left the parent set, the tables are replicated, and no rank can be more than one exchange ahead.
    bool peer_rows = false;
    DevBuf home, bases_dev;
    std::vector<void*> ipc_opened;
    bool final_fetch_done = false;

    ~gapa_cuda_ga() {
        for (void* mapped : ipc_opened) cudaIpcCloseMemHandle(mapped);
        home.release();
        bases_dev.release();
        for (cudaEvent_t e : gen_marks) cudaEventDestroy(e);
        if (ev_adv0) cudaEventDestroy(ev_adv0);
        if (ev_adv1) cudaEventDestroy(ev_adv1);
    }
    bool sampled_gen(int gen) const { return gen <= exact_until || (gen - 2) % stride == 0; }

    int evaluate(const int32_t* table, double* fit_all, const VariationSpec* vary = nullptr) {  // rows [lo, hi) named by `table`
        ++fitness_batch_calls;
        const bool timed = sampled_gen(current_gen);
        if (current_gen > 1) {
            ++later_calls;
            later_timed_calls += timed;
        }
        GAPA_TRY(eval_rows(ctx, p.task, GeneRows{pool_rows, table + lo, k}, hi - lo, fit_all + lo, st,
                           current_gen == 1 ? &first_timer : timed ? &timer : nullptr, vary));
        if (world > 1) {
            if (want_stats) GAPA_TRY(exchange_marks.mark(st, current_gen - 1));
            const int rc = exchange(exchange_user, fit_all, s, block, st);
            if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "run: exchange hook failed with status %d", rc);
            if (want_stats) GAPA_TRY(exchange_marks.mark(st, current_gen - 1));
            ++exchanges_in_gen[static_cast<size_t>(current_gen - 1)];
        }
        return GAPA_CUDA_OK;
    }
    int mark_generation(int gen) {
        cudaEvent_t e;
        GAPA_TRY(events.get(&e));
        gen_marks.push_back(e);
        marked_gens.push_back(gen);
        GAPA_CUDA_TRY(cudaEventRecord(e, st));
        return GAPA_CUDA_OK;
    }
    // the stream is idle: fold the finished blocks of generations (all marks but the last, which starts the open block)
    int flush_marks() {
        GAPA_TRY(timer.flush());
        GAPA_TRY(first_timer.flush());
        GAPA_TRY(exchange_marks.flush(&exchange_of_gen));
        size_t b = 0;
        for (; b + 1 < gen_marks.size(); ++b) {  // a block of generations between two marks shares its mean
            float ms = 0.f;
            GAPA_CUDA_TRY(cudaEventElapsedTime(&ms, gen_marks[b], gen_marks[b + 1]));
            const int g0 = marked_gens[b], g1 = marked_gens[b + 1];
            for (int gi = g0; gi < g1 && gi <= iters; ++gi) wall_of_gen[static_cast<size_t>(gi - 1)] = ms * 1e-3 / (g1 - g0);
            events.put(gen_marks[b]);
        }
        gen_marks.erase(gen_marks.begin(), gen_marks.begin() + static_cast<long>(b));
        marked_gens.erase(marked_gens.begin(), marked_gens.begin() + static_cast<long>(b));
        return GAPA_CUDA_OK;
    }
    int poll_status(const char* what) {
        int h = 0;
        GAPA_CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, st));
        GAPA_CUDA_TRY(cudaStreamSynchronize(st));
        if (h == GAPA_CUDA_E_NAN) return fail(GAPA_CUDA_E_NAN, "%s", what);
        if (h != 0) return fail(GAPA_CUDA_E_CUDA, "run: device-side failure %d (%s)", h, what);
        return flush_marks();
    }
    int generation(int gen);
    int stats_pending_gen = 0;  // generation whose history entry has not been written yet (0 = none)
    bool defer_stats = true;
    int flush_stats(int gen);
    int setup_peer_rows();
    int fetch_all_parents() {  // every parent row local (EDA generations, the returned population)
        return launch_fetch_rows(pool_rows, bases_dev.as<const int32_t*>(), home.as<int32_t>(), parent, s, k, rank, st);
    }
};

namespace {
struct PoolHandle {  // what the ranks tell each other about their population stores
    int64_t pid;
    int32_t device;
    int32_t pad;
    uint64_t ptr;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(PoolHandle) <= GAPA_CUDA_COMM_CTRL_BYTES, "pool handle does not fit the control exchange");
}  // namespace

int gapa_cuda_ga::setup_peer_rows() {
    if (exchange != gapa_cuda_comm_allgather) {
        // GAPA_PEER_ROWS_LOOPBACK (tools/probe_scaling.py): every "peer" pool is this rank's own — the bookkeeping and the
        // write-through copies of a sharded generation are timed on one GPU; the rows read are not the real ones
        std::vector<const int32_t*> loop(static_cast<size_t>(world), pool_rows);
        GAPA_TRY(bases_dev.ensure(sizeof(int32_t*) * static_cast<size_t>(world)));
        GAPA_CUDA_TRY(cudaMemcpy(bases_dev.ptr, loop.data(), sizeof(int32_t*) * static_cast<size_t>(world), cudaMemcpyHostToDevice));
        GAPA_TRY(home.ensure(sizeof(int32_t) * 2 * static_cast<size_t>(s)));
        std::vector<int32_t> own(2 * static_cast<size_t>(s), rank);
        GAPA_CUDA_TRY(cudaMemcpy(home.ptr, own.data(), sizeof(int32_t) * own.size(), cudaMemcpyHostToDevice));
        peer_rows = true;
        return GAPA_CUDA_OK;
    }
    gapa_cuda_comm* comm = static_cast<gapa_cuda_comm*>(exchange_user);
    PoolHandle mine{};
    mine.pid = static_cast<int64_t>(getpid());
    mine.device = ctx->device;
    mine.ptr = reinterpret_cast<uint64_t>(pool_rows);
    if (cudaIpcGetMemHandle(&mine.ipc, pool_rows) != cudaSuccess) (void)cudaGetLastError();  // same-process peers do not need it
    std::vector<PoolHandle> all(static_cast<size_t>(world));
    GAPA_TRY(gapa_cuda_comm_allgather_bytes(comm, &mine, static_cast<int>(sizeof(PoolHandle)), all.data()));
    std::vector<const int32_t*> bases(static_cast<size_t>(world), nullptr);
    for (int r = 0; r < world; ++r) {
        const PoolHandle& h = all[static_cast<size_t>(r)];
        if (r == rank) {
            bases[static_cast<size_t>(r)] = pool_rows;
        } else if (h.pid == mine.pid) {
            bases[static_cast<size_t>(r)] = reinterpret_cast<const int32_t*>(h.ptr);  // peer access was enabled by comm_connect
        } else {
            void* mapped = nullptr;
            GAPA_CUDA_TRY(cudaIpcOpenMemHandle(&mapped, h.ipc, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened.push_back(mapped);
            bases[static_cast<size_t>(r)] = static_cast<const int32_t*>(mapped);
        }
    }
    GAPA_TRY(bases_dev.ensure(sizeof(int32_t*) * static_cast<size_t>(world)));
    GAPA_CUDA_TRY(cudaMemcpy(bases_dev.ptr, bases.data(), sizeof(int32_t*) * static_cast<size_t>(world), cudaMemcpyHostToDevice));
    GAPA_TRY(home.ensure(sizeof(int32_t) * 2 * static_cast<size_t>(s)));
    std::vector<int32_t> self(2 * static_cast<size_t>(s), rank);  // init_population builds every parent row on every rank
    GAPA_CUDA_TRY(cudaMemcpy(home.ptr, self.data(), sizeof(int32_t) * self.size(), cudaMemcpyHostToDevice));
    peer_rows = true;
    return GAPA_CUDA_OK;
}

int gapa_cuda_ga::generation(int gen) {
    current_gen = gen;
    if (want_stats && sampled_gen(gen)) GAPA_TRY(mark_generation(gen));
    if (gen == 1) {
        GAPA_TRY(launch_slots_identity(s, parent, child, st));
        GAPA_TRY(launch_init(pool, 0, s, k, p.seed, 0, pool_rows, st));  // parents occupy slots 0..s-1
        GAPA_TRY(evaluate(parent, fit));
        GAPA_LAUNCH(k_check_nan, (s + 255) / 256, 256, 0, st, fit, s, status);
        GAPA_TRY(poll_status("fitness evaluation failed during initialization"));  // modes.cpp:314-315
    }
    const uint64_t g = static_cast<uint64_t>(gen);
    // Children are built only for the rows this rank evaluates (all rows when world == 1).
    const bool eda_gen = p.eda_interval > 0 && gen % p.eda_interval == 0;  // modes.cpp:31-33,167-168
    const int32_t* partner = eda_gen ? nullptr : B.partner.as<int32_t>();
    if (!eda_gen && !(small && gen > 1))  // small populations: selected by the previous generation's elitism launch
    {
        // the previous generation's statistics, if they were deferred, ride on this selection's first launch (a block of their own)
        const int sg = stats_pending_gen;
        stats_pending_gen = 0;
        GAPA_TRY(launch_select(fit, s, minimize, p.seed, g, B.partner.as<int32_t>(), B.weights.as<double>(),
                               B.cumulative.as<double>(), status, st, sg ? hist + (sg - 1) : nullptr, sg ? hist + iters + (sg - 1) : nullptr));
    }
    VariationSpec vary;  // the evaluation builds the children of rows [lo, hi) into their slots first
    vary.P = make_variation_params(p.pc, p.pm, pool, s, p.seed, g);
    vary.pool = pool_rows;
    vary.parent = parent;
    vary.child = child;
    vary.partner = partner;
    vary.row_first = lo;
    if (peer_rows) {
        GAPA_TRY(launch_home_children(child, s, block, home.as<int32_t>(), st));  // who builds which child this generation
        if (eda_gen) GAPA_TRY(fetch_all_parents());  // eda_sample reads genes of ALL parents (ga_ops.cpp:214-238)
        vary.bases = bases_dev.as<const int32_t*>();
        vary.home = home.as<int32_t>();
        vary.self = rank;
    }
    GAPA_TRY(evaluate(child, fit_m, &vary));
    if (peer_rows && !eda_gen) GAPA_TRY(launch_home_adopt(parent, partner, lo, hi, rank, home.as<int32_t>(), st));
    // elitism permutes the slot tables; survivors built by other ranks are rebuilt in place
    // small populations: elitism, the generation's statistics AND the next generation's selection in one launch
    const bool select_next = gen < iters && !(p.eda_interval > 0 && (gen + 1) % p.eda_interval == 0);
    if (small)
        GAPA_TRY(launch_slots_elitism_small(parent, child, s, fit, fit_m, minimize, next_parent, next_child, fit_next,
                                            B.src_of_rank.as<int32_t>(), status, hist + (gen - 1), hist + iters + (gen - 1),
                                            select_next ? 1 : 0, p.seed, g + 1, B.partner.as<int32_t>(), B.weights.as<double>(),
                                            B.cumulative.as<double>(), st));
    else
        GAPA_TRY(launch_slots_elitism(pool_rows, parent, child, partner, s, k, peer_rows ? 0 : lo, peer_rows ? s : hi, fit, fit_m,
                                      minimize, p.pc, p.pm, pool, p.seed, g, next_parent, next_child, fit_next,
                                      B.src_of_rank.as<int32_t>(), status, st));  // peer rows: nothing is rebuilt
    std::swap(parent, next_parent);
    std::swap(child, next_child);
    std::swap(fit, fit_next);
    if (peer_rows && gen == iters) {
        // the run ends with every parent row local, and nobody leaves (and frees its pool) before everybody has them:
        // one more exchange as the barrier (fit_next is scratch by now)
        GAPA_TRY(fetch_all_parents());
        const int rc = exchange(exchange_user, fit_next, s, block, st);
        if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "run: exchange hook failed with status %d", rc);
        final_fetch_done = true;
    }
    if (!small) {
        // Statistics of this generation (they read the new parents' fitness, like the next selection): a launch of their own
        // is ~5 us on the critical path of a generation, so where the next generation starts with the multi-block selection
        // they are deferred to an extra block of its first kernel (k_ga_weights); gapa_cuda_ga_result flushes a pending one.
        const bool next_selects = gen < iters && !(p.eda_interval > 0 && (gen + 1) % p.eda_interval == 0) && s > 1024;
        if (next_selects && defer_stats) stats_pending_gen = gen;
        else GAPA_TRY(flush_stats(gen));
    }
    // NaN / non-finite fitness is an Error in the reference (ga_ops.cpp:56-57, :189-192);
    // the flag is polled every few generations and at the end to keep the loop asynchronous.
    // (every 16 generations; every 64 where a generation is two launches of ~10 us and the drain of a poll is a whole generation)
    if ((gen & (small ? 63 : 15)) == 0 || gen == iters) {
        GAPA_TRY(poll_status("elitism: NaN fitness"));
        if (stride == 1 && world == 1 && timer.last_ms >= 0.f && timer.last_ms < kSampleBelowMs) {
            // A timing event between two kernels costs ~5 us of device time: short evaluations switch to SAMPLED marks
            stride = kTimingStride;
            exact_until = gen + 1;  // the next generation carries a mark, so the exact block ends there
        }
    }
    gen_done = gen;
    return GAPA_CUDA_OK;
}

int gapa_cuda_ga::flush_stats(int gen) {
    GAPA_LAUNCH(k_ga_stats, 1, 1024, 0, st, fit, s, hist + (gen - 1), hist + iters + (gen - 1));
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_stats_device(const double* fit_dev, int s, double* best_dev, double* mean_dev, void* stream) {
    if (s < 1 || !fit_dev || !best_dev || !mean_dev) return fail(GAPA_CUDA_E_INVALID, "stats: bad arguments");
    GAPA_LAUNCH(k_ga_stats, 1, 1024, 0, static_cast<cudaStream_t>(stream), fit_dev, s, best_dev, mean_dev);
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_create(gapa_cuda_ctx* ctx, const gapa_cuda_run_params* p, gapa_cuda_allgather_fn exchange,
                                   void* exchange_user, int want_stats, gapa_cuda_ga** out) {
    if (!ctx || !p || !out) return fail(GAPA_CUDA_E_INVALID, "run: null argument");
    *out = nullptr;
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
            if (ctx->pool_kind == GAPA_POOL_NODE_REMOVAL || ctx->pool_kind == GAPA_POOL_EDGE_FLIP) return fail(GAPA_CUDA_E_INVALID, "run: incompatible gene pool kind");
            break;
        case GAPA_TASK_LPA:
            if ((ctx->pool_kind != GAPA_POOL_EDGE_REMOVAL && ctx->pool_kind != GAPA_POOL_EDGE_FLIP) || ctx->T < 1) return fail(GAPA_CUDA_E_INVALID, "run: link-prediction task needs an edge-removal pool and a split");
            break;
        default: return fail(GAPA_CUDA_E_INVALID, "unknown fitness task %d", p->task);
    }
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));
    gapa_cuda_ga* ga = new gapa_cuda_ga();
    auto body = [&]() -> int {
        ga->ctx = ctx;
        ga->p = *p;
        ga->exchange = exchange;
        ga->exchange_user = exchange_user;
        ga->world = world;
        ga->rank = rank;
        const int s = ga->s = p->pop_size, k = ga->k = p->budget, iters = ga->iters = p->iterations;
        (void)k;
        ga->minimize = p->minimize ? 1 : 0;
        ga->pool = static_cast<uint32_t>(ctx->pool_size);
        ga->block = (s + world - 1) / world;  // partition_rows, modes.cpp:506-516
        ga->lo = std::min(rank * ga->block, s);
        ga->hi = std::min(ga->lo + ga->block, s);
        ga->cells = static_cast<size_t>(s) * k;
        ga->padded = static_cast<size_t>(ga->block) * world;
        ga->st = ctx->stream;
        // Population store: one pool of 2s row slots + parent / child slot tables (slot_kernels.cu).
        RunBuffers& B = ga->B;
        GAPA_TRY(B.pop.ensure(sizeof(int32_t) * 2 * ga->cells));
        GAPA_TRY(B.next.ensure(sizeof(int32_t) * 4 * s));  // parent, child, next parent, next child tables
        GAPA_TRY(B.partner.ensure(sizeof(int32_t) * s));
        GAPA_TRY(B.fit.ensure(sizeof(double) * ga->padded));
        GAPA_TRY(B.fit_m.ensure(sizeof(double) * ga->padded));
        GAPA_TRY(B.fit_next.ensure(sizeof(double) * ga->padded));
        GAPA_TRY(B.weights.ensure(sizeof(double) * s));
        GAPA_TRY(B.cumulative.ensure(sizeof(double) * s));
        GAPA_TRY(B.src_of_rank.ensure(sizeof(int32_t) * 2 * s));
        GAPA_TRY(B.status.ensure(sizeof(int)));
        GAPA_TRY(B.hist.ensure(sizeof(double) * 2 * iters));
        ga->pool_rows = B.pop.as<int32_t>();
        ga->parent = B.next.as<int32_t>();
        ga->child = ga->parent + s;
        ga->next_parent = ga->child + s;
        ga->next_child = ga->next_parent + s;
        ga->fit = B.fit.as<double>();
        ga->fit_m = B.fit_m.as<double>();
        ga->fit_next = B.fit_next.as<double>();
        ga->hist = B.hist.as<double>();
        ga->status = B.status.as<int>();
        GAPA_CUDA_TRY(cudaMemsetAsync(ga->status, 0, sizeof(int), ga->st));
        GAPA_CUDA_TRY(cudaMemsetAsync(ga->fit, 0, sizeof(double) * ga->padded, ga->st));
        GAPA_CUDA_TRY(cudaMemsetAsync(ga->fit_m, 0, sizeof(double) * ga->padded, ga->st));
        GAPA_CUDA_TRY(cudaMemsetAsync(ga->fit_next, 0, sizeof(double) * ga->padded, ga->st));  // exchanged whole, padding included
        GAPA_CUDA_TRY(cudaMemsetAsync(ga->hist, 0, sizeof(double) * 2 * iters, ga->st));
        // GenerationStats timing (modes.hpp:63-71): generation boundaries and the exchange hook are bracketed by events.
        // A small population's generation is two launches of 10-15 us, so there the marks are SAMPLED from generation 2
        // on: every kTimingStride-th generation is bracketed (its evaluation and its boundary); eval_seconds is scaled by
        // calls / timed calls and a block of generations shares its mean wall time.  Larger populations start exact and
        // switch to sampling at the first status poll (generation 16) if an evaluation takes less than kSampleBelowMs.
        ga->want_stats = want_stats != 0;
        ga->small = world == 1 && 2 * s <= 1024;
        if (const char* raw = std::getenv("GAPA_DEFER_STATS")) ga->defer_stats = raw[0] != '0';
        ga->stride = ga->small ? kTimingStride : 1;
        ga->timer.pool = ga->first_timer.pool = ga->exchange_marks.pool = &ga->events;
        ga->exchange_of_gen.assign(static_cast<size_t>(iters), 0.0);
        ga->wall_of_gen.assign(static_cast<size_t>(iters), 0.0);
        ga->exchanges_in_gen.assign(static_cast<size_t>(iters), 0);
        GAPA_CUDA_TRY(cudaEventCreate(&ga->ev_adv0));
        GAPA_CUDA_TRY(cudaEventCreate(&ga->ev_adv1));
        if (world > 1 && exchange == gapa_cuda_comm_allgather) {
            int transport = -1;
            GAPA_TRY(gapa_cuda_comm_info(static_cast<gapa_cuda_comm*>(exchange_user), &transport, nullptr, nullptr));
            const char* knob = std::getenv("GAPA_PEER_ROWS");  // 0: rebuild foreign survivors instead (the NCCL transport's way)
            if (transport == GAPA_COMM_PEER && !(knob && knob[0] == '0')) {
                GAPA_CUDA_TRY(cudaStreamSynchronize(ga->st));
                GAPA_TRY(ga->setup_peer_rows());
            }
        } else if (world > 1 && std::getenv("GAPA_PEER_ROWS_LOOPBACK")) {
            GAPA_TRY(ga->setup_peer_rows());
        }
        return GAPA_CUDA_OK;
    };
    const int rc = body();
    if (rc != GAPA_CUDA_OK) {
        delete ga;
        return rc;
    }
    *out = ga;
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_advance(gapa_cuda_ga* ga, int generations, float* device_ms) {
    if (!ga || generations < 0) return fail(GAPA_CUDA_E_INVALID, "advance: bad arguments");
    gapa_cuda_ctx* ctx = ga->ctx;
    std::lock_guard<std::mutex> lock(ctx->mu);  // the run owns the context's scratch while it advances
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));
    const int last = std::min(ga->iters, ga->gen_done + generations);
    const auto t0 = std::chrono::steady_clock::now();
    GAPA_CUDA_TRY(cudaEventRecord(ga->ev_adv0, ga->st));
    for (int gen = ga->gen_done + 1; gen <= last; ++gen) GAPA_TRY(ga->generation(gen));
    GAPA_CUDA_TRY(cudaEventRecord(ga->ev_adv1, ga->st));
    GAPA_CUDA_TRY(cudaStreamSynchronize(ga->st));
    ga->wall_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (device_ms) GAPA_CUDA_TRY(cudaEventElapsedTime(device_ms, ga->ev_adv0, ga->ev_adv1));
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_generation(const gapa_cuda_ga* ga, int* generations_done) {
    if (!ga || !generations_done) return fail(GAPA_CUDA_E_INVALID, "generation: null argument");
    *generations_done = ga->gen_done;
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_result(gapa_cuda_ga* ga, gapa_cuda_run_result* result) {
    if (!ga || !result) return fail(GAPA_CUDA_E_INVALID, "result: null argument");
    gapa_cuda_ctx* ctx = ga->ctx;
    std::lock_guard<std::mutex> lock(ctx->mu);
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = ga->st;
    const int iters = ga->iters, s = ga->s;
    if (ga->want_stats && ga->gen_done > 0 && (ga->marked_gens.empty() || ga->marked_gens.back() != ga->gen_done + 1))
        GAPA_TRY(ga->mark_generation(ga->gen_done + 1));  // closes the last block of generations
    if (ga->stats_pending_gen) {  // fit still holds that generation's parents: nothing ran since
        GAPA_TRY(ga->flush_stats(ga->stats_pending_gen));
        ga->stats_pending_gen = 0;
    }
    GAPA_CUDA_TRY(cudaStreamSynchronize(st));
    GAPA_TRY(ga->flush_marks());
    result->fitness_batch_calls = ga->fitness_batch_calls;
    result->total_wall_seconds = ga->wall_seconds;
    double eval_seconds = ga->timer.ms_total * 1e-3;
    if (ga->later_timed_calls) eval_seconds *= static_cast<double>(ga->later_calls) / static_cast<double>(ga->later_timed_calls);
    result->eval_seconds = eval_seconds + ga->first_timer.ms_total * 1e-3;
    for (int gi = 0; gi < iters; ++gi) {
        const double wall_s = ga->wall_of_gen[static_cast<size_t>(gi)], exchange_s = ga->exchange_of_gen[static_cast<size_t>(gi)];
        if (result->gen_wall_seconds) result->gen_wall_seconds[gi] = wall_s;
        if (result->gen_exchange_seconds) result->gen_exchange_seconds[gi] = exchange_s;
        if (result->gen_lifecycle_seconds) result->gen_lifecycle_seconds[gi] = 0.0;
        if (result->gen_compute_seconds) result->gen_compute_seconds[gi] = std::max(0.0, wall_s - exchange_s);  // modes.cpp:38-40
        if (result->gen_messages) result->gen_messages[gi] = static_cast<uint64_t>(ga->exchanges_in_gen[static_cast<size_t>(gi)]);
    }
    if (result->history_best) GAPA_CUDA_TRY(cudaMemcpy(result->history_best, ga->hist, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    if (result->history_mean) GAPA_CUDA_TRY(cudaMemcpy(result->history_mean, ga->hist + iters, sizeof(double) * iters, cudaMemcpyDeviceToHost));
    if (result->final_population) {  // RunResult::final_population: the parents in best-first order
        if (ga->peer_rows && !ga->final_fetch_done) GAPA_TRY(ga->fetch_all_parents());  // mid-run: the peers are still there
        DevBuf dense;
        GAPA_TRY(dense.ensure(sizeof(int32_t) * std::max<size_t>(ga->cells, 1)));
        int rc = launch_slots_gather(ga->pool_rows, ga->parent, s, ga->k, dense.as<int32_t>(), st);
        if (rc == GAPA_CUDA_OK && cudaMemcpyAsync(result->final_population, dense.ptr, sizeof(int32_t) * ga->cells, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = GAPA_CUDA_E_CUDA;
        if (rc == GAPA_CUDA_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = GAPA_CUDA_E_CUDA;
        dense.release();
        if (rc != GAPA_CUDA_OK) return fail(rc, "run: could not materialise the final population");
    }
    if (result->final_fitness) GAPA_CUDA_TRY(cudaMemcpy(result->final_fitness, ga->fit, sizeof(double) * s, cudaMemcpyDeviceToHost));
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_ga_destroy(gapa_cuda_ga* ga) {
    if (!ga) return GAPA_CUDA_OK;
    cudaSetDevice(ga->ctx->device);
    cudaStreamSynchronize(ga->st);
    delete ga;
    return GAPA_CUDA_OK;
}

extern "C" int gapa_cuda_run(gapa_cuda_ctx* ctx, const gapa_cuda_run_params* p, gapa_cuda_allgather_fn exchange,
                             void* exchange_user, gapa_cuda_run_result* result) {
    if (!ctx || !p || !result) return fail(GAPA_CUDA_E_INVALID, "run: null argument");
    const bool want_stats = result->gen_wall_seconds || result->gen_compute_seconds || result->gen_exchange_seconds ||
                            result->gen_lifecycle_seconds || result->gen_messages;
    gapa_cuda_ga* ga = nullptr;
    GAPA_TRY(gapa_cuda_ga_create(ctx, p, exchange, exchange_user, want_stats ? 1 : 0, &ga));
    int rc = gapa_cuda_ga_advance(ga, p->iterations, nullptr);
    if (rc == GAPA_CUDA_OK) rc = gapa_cuda_ga_result(ga, result);
    gapa_cuda_ga_destroy(ga);
    return rc;
}
