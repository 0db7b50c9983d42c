/* gapa_cuda.h — C ABI of the B200 (sm_100a) implementation of GAPA's
 * data-parallel hot path: per-generation batched fitness evaluation of a GA
 * population over perturbed graphs, plus the genetic operators around it.
 *
 * This is the drop-in boundary.  Every entry point replaces one interface of
 * the reference C++ library (citations are file:line under
 * /root/reference/proj); host C++ (paper_2412_20980_b200/host/) and the Python
 * driver bind exactly these symbols, and nothing else crosses the boundary:
 * plain pointers and sizes, no STL, no exceptions, no torch types.
 *
 * Conventions
 *   - every function returns an int status: 0 = ok, otherwise a GAPA_CUDA_E_*
 *     code; gapa_cuda_last_error() returns the message for the calling thread
 *     (the host adapters turn a non-zero status into `throw gapa::Error`,
 *     include/gapa/error.hpp:9-30).
 *   - "host" pointers are ordinary CPU memory; "_device" entry points take
 *     device pointers valid on the context's GPU and a cudaStream_t passed as
 *     void* (NULL = the legacy default stream).  They enqueue work and
 *     return; the caller synchronises the stream (gapa_cuda_stream_sync).
 *   - gene matrices are row-major int32 [rows x cols] (population.hpp:12-40);
 *     fitness vectors are double[rows] (population.hpp:62).
 *   - there is NO CPU fallback: without a CUDA device every call fails with
 *     GAPA_CUDA_E_CUDA.
 */
#ifndef GAPA_CUDA_H
#define GAPA_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GAPA_CUDA_ABI_VERSION 3

enum {
    GAPA_CUDA_OK = 0,
    GAPA_CUDA_E_INVALID = 1,  /* bad argument / shape / wrong pool kind (fitness.cpp:50-57)   */
    GAPA_CUDA_E_RANGE = 2,    /* gene id outside the pool (gene_pool.cpp:104-108)             */
    GAPA_CUDA_E_NAN = 3,      /* NaN / non-finite fitness (ga_ops.cpp:56-57, :189-192)        */
    GAPA_CUDA_E_CUDA = 4,     /* CUDA runtime failure, or no device                           */
    GAPA_CUDA_E_NOMEM = 5
};

/* fitness tasks — the four objectives of fitness.hpp:33-52 */
enum {
    GAPA_TASK_PC = 0,  /* pairwise connectivity, pc_fitness        (fitness.cpp:28-33)  */
    GAPA_TASK_MCN = 1, /* largest component, sixdst_fitness(Exact) (fitness.cpp:18-26)  */
    GAPA_TASK_CDA = 2, /* modularity of the greedy detector        (fitness.cpp:35-41)  */
    GAPA_TASK_LPA = 3, /* AUC of the RA predictor                  (fitness.cpp:43-48)  */
    GAPA_TASK_SIXDST = 4 /* sixdst_fitness(ClosurePolicy::SixDegrees): largest radius-8 ball
                            (fitness.cpp:18-26 over accessibility.cpp:20-37, <= 3 squarings)   */
};

/* PoolKind, gene_pool.hpp:14 (same order) */
enum { GAPA_POOL_EDGE_REMOVAL = 0, GAPA_POOL_EDGE_ADDITION = 1, GAPA_POOL_NODE_REMOVAL = 2,
       /* NOT in the reference (BASELINE.json north_star: "edge flips" for the link-prediction attack; PARITY UNPINNED,
        * semantics stated in the oracle directory's C restatement): a gene is a node pair a < b; an edge of the graph is removed, a
        * non-edge is added, relative to the UNPERTURBED graph (repeats are idempotent, like gene_pool.cpp:49-67).
        * u == NULL in gapa_cuda_pool_set: every pair in lexicographic order, gene id = a n - a(a+1)/2 + (b - a - 1)
        * (n <= 65536).  Link-prediction task only. */
       GAPA_POOL_EDGE_FLIP = 3 };

/* link score of the link-prediction task: RA = the reference's resource allocation (link_prediction.cpp:55-69);
 * CN = common neighbours, |N'(u) & N'(v)| — north_star's "CN/RA link scores"; NOT in the reference, PARITY UNPINNED */
enum { GAPA_LP_SCORE_RA = 0, GAPA_LP_SCORE_CN = 1 };

/* StreamRole, rng.hpp:41-47 */
enum { GAPA_ROLE_INIT = 1, GAPA_ROLE_SELECT = 2, GAPA_ROLE_CROSSOVER_MASK = 3,
       GAPA_ROLE_MUTATION_MASK = 4, GAPA_ROLE_MUTATION_INDEX = 5 };

typedef struct gapa_cuda_ctx gapa_cuda_ctx; /* graph + pool + split on one GPU */

const char* gapa_cuda_last_error(void);
int gapa_cuda_abi_version(void);
int gapa_cuda_device_count(int* count);

/* ---- graph / pool / split ------------------------------------------------------
 * gapa_cuda_graph_create replaces Graph::adjacency() (graph.cpp:47-54) and the
 * per-objective BitMatrix copies (fitness.cpp:94-113): ONE read-only CSR per GPU,
 * shared by every individual, never copied.  `uv` holds m canonical edges
 * (Graph::edges(), graph.hpp:26; either endpoint order accepted, loops and
 * duplicates rejected like graph.cpp:26-31). */
int gapa_cuda_graph_create(int32_t n, int64_t m, const int32_t* uv, int device, gapa_cuda_ctx** out);
/* Same, from a ready CSR (row_ptr[n+1], col_idx[2m] ascending per row, symmetric). */
int gapa_cuda_graph_create_csr(int32_t n, int64_t m, const int32_t* row_ptr, const int32_t* col_idx,
                               int device, gapa_cuda_ctx** out);
int gapa_cuda_destroy(gapa_cuda_ctx* ctx);
int gapa_cuda_graph_info(const gapa_cuda_ctx* ctx, int32_t* n, int64_t* m, int* device);

/* GenePool (gene_pool.hpp:32-52).  kind NODE_REMOVAL: u[i] = node of gene i
 * (u == NULL means the identity pool of build_gene_pool, gene_pool.cpp:89-92),
 * v ignored.  kind EDGE_REMOVAL: (u[i], v[i]) are node pairs (u == NULL means build_gene_pool's (u,v)-sorted edge order,
 * gene_pool.cpp:73-79); a pair that is not an edge of this graph is accepted and removes nothing, as in the reference
 * (clearing an absent adjacency bit, gene_pool.cpp:53-56) — e.g. a pool built on the full graph, evaluated on split.train.
 * kind EDGE_ADDITION (cda task only, fitness.cpp:54-57): (u[i], v[i]) is the pair gene i
 * adds (gene_pool.cpp:57-60); u == NULL means every non-edge a < b in lexicographic
 * order (gene_pool.cpp:81-87; fails on a complete graph like :86).  A pair that is
 * already an edge is accepted and is a no-op, as in the reference.  Repeated elements
 * are rejected for every kind (gene_pool.cpp:36-41). */
int gapa_cuda_pool_set(gapa_cuda_ctx* ctx, int kind, int32_t n_genes, const int32_t* u, const int32_t* v);
int gapa_cuda_pool_info(const gapa_cuda_ctx* ctx, int* kind, int32_t* n_genes);

/* LinkPredictionSplit (link_prediction.hpp:16-21): the context's graph is
 * split.train; test_uv / probe_uv are T and P (u,v) pairs. */
int gapa_cuda_lp_split_set(gapa_cuda_ctx* ctx, int32_t T, const int32_t* test_uv, int32_t P,
                           const int32_t* probe_uv);

int gapa_cuda_lp_score_set(gapa_cuda_ctx* ctx, int score); /* GAPA_LP_SCORE_*; the default is RA */

/* ---- fitness: FitnessFunction::evaluate_batch (fitness.hpp:17-27) ----------------
 * out[i] = fitness of row i, identical to the reference's evaluate_one on
 * that row (fitness.cpp:10-14).  cols may be 0 (empty perturbation), rows may be 0.
 * Host form: H2D of genes + kernels + D2H of out, synchronous. */
int gapa_cuda_eval_batch(gapa_cuda_ctx* ctx, int task, const int32_t* genes_host, int rows, int cols,
                         double* out_host);
/* Device form: genes and out live in HBM.  Returns when the evaluation has finished on
 * `stream` (status is final: gene range, CUDA errors; gapa_cuda_last_eval_ms is valid).
 * Inside gapa_cuda_run the same evaluators run without this wait. */
int gapa_cuda_eval_batch_device(gapa_cuda_ctx* ctx, int task, const int32_t* genes_dev, int rows, int cols,
                                double* out_dev, void* stream);

/* ---- genetic operators on HBM-resident populations (ga_ops.hpp:30-93) ------------
 * All keyed by (seed, generation, role, GLOBAL row) exactly like rng.hpp:59-65,
 * so any row partition reproduces the same matrices. */

/* init_population_block (ga_ops.cpp:19-29): out_dev[row_count x budget] */
int gapa_cuda_ga_init_device(int32_t pool_size, int row_first, int row_count, int budget, uint64_t seed,
                             uint64_t generation, int32_t* out_dev, void* stream);
/* make_crossover_mask / make_mutation_mask (ga_ops.cpp:38-47, :84-92): MaskMatrix bytes (population.hpp:43-60) of rows
 * [row_first, row_first + row_count); role = GAPA_ROLE_CROSSOVER_MASK or GAPA_ROLE_MUTATION_MASK.  The generation loop
 * never materialises these (the fused variation kernels evaluate the same draws in place); they exist for hosts and
 * tests that want the matrices themselves (test_ga_engine.cpp:143-173). */
int gapa_cuda_ga_mask_device(int role, double rate, int row_first, int row_count, int cols, uint64_t seed, uint64_t generation,
                             uint8_t* out_dev, void* stream);
/* make_mutation_indices (ga_ops.cpp:94-103): the fresh genes mutate draws, int32 [row_count x cols] */
int gapa_cuda_ga_mutation_indices_device(int32_t pool_size, int row_first, int row_count, int cols, uint64_t seed,
                                         uint64_t generation, int32_t* out_dev, void* stream);
/* roulette_select in index form (ga_ops.cpp:54-82,105-128): rank weights with
 * tie-span averaging -> cumulative -> one Select draw per row -> partner row.
 * weights_dev / scratch may be NULL.  Non-finite fitness -> GAPA_CUDA_E_NAN. */
int gapa_cuda_ga_select_device(const double* fitness_dev, int s, int minimize, uint64_t seed,
                               uint64_t generation, int32_t* partner_dev, double* weights_dev, void* stream);
/* crossover (ga_ops.cpp:130-144) fused with mutate_block (ga_ops.cpp:164-178) for
 * rows [row_first, row_first+row_count) of the population; pop_dev is the FULL
 * s x k matrix, partner_dev the full partner vector, out_dev the block. */
int gapa_cuda_ga_crossover_mutate_device(const int32_t* pop_dev, const int32_t* partner_dev, int s, int k,
                                         int row_first, int row_count, double pc, double pm,
                                         int32_t pool_size, uint64_t seed, uint64_t generation,
                                         int32_t* out_dev, void* stream);
/* mutate_block alone (used after eda_sample, modes.cpp:167-173) */
int gapa_cuda_ga_mutate_device(const int32_t* block_dev, int rows, int k, int row_offset, double pm,
                               int32_t pool_size, uint64_t seed, uint64_t generation, int32_t* out_dev,
                               void* stream);
/* eda_sample (ga_ops.cpp:214-238) */
int gapa_cuda_ga_eda_device(const int32_t* elite_dev, int s, int k, int elite_count, int32_t pool_size,
                            uint64_t seed, uint64_t generation, int smoothing, int32_t* out_dev, void* stream);
/* elitism (ga_ops.cpp:180-212): stable best-first order of the 2s stacked rows,
 * originals before mutated on ties; next_dev must not alias pop_dev / m_pop_dev. */
int gapa_cuda_ga_elitism_device(const int32_t* pop_dev, const int32_t* m_pop_dev, int s, int k,
                                const double* fit_dev, const double* fit_m_dev, int minimize,
                                int32_t* next_dev, double* next_fit_dev, void* stream);

/* elitism for a row-sharded generation (the GPU form of M mode, modes.cpp:190-349): this rank built
 * only rows [block_lo, block_hi) of M_POP (m_block_dev, block_hi - block_lo rows); surviving mutated
 * rows of other ranks are recomputed from the replicated parents and the keyed streams instead of
 * being fetched — crossover+mutate when partner_dev != NULL, eda_sample+mutate (elite = the whole
 * population, add-one smoothing; modes.cpp:167-168) when it is NULL.  Result == gapa_cuda_ga_elitism_device
 * on the full M_POP. */
int gapa_cuda_ga_elitism_sharded_device(const int32_t* pop_dev, const int32_t* m_block_dev, int block_lo, int block_hi,
                                        const int32_t* partner_dev, int s, int k, const double* fit_dev,
                                        const double* fit_m_dev, int minimize, double pc, double pm,
                                        int32_t pool_size, uint64_t seed, uint64_t generation, int32_t* next_dev,
                                        double* next_fit_dev, void* stream);

/* ---- slot-pool population store (the loop's zero-copy form of POP / M_POP, modes.cpp:159-175) ----
 * pool_dev holds 2s rows of k genes; parent_dev[r] / child_dev[r] name the slot of parent row r (best
 * first) and of child row r.  Variation writes children into their slots, evaluators read rows
 * through a slot table, elitism permutes the tables — no genome is copied.  partner_dev == NULL
 * selects the EDA form (eda_sample over all parents with smoothing, then mutate). */
int gapa_cuda_ga_slots_identity_device(int s, int32_t* parent_dev, int32_t* child_dev, void* stream);
/* children of rows [row_first, row_first + row_count): crossover (ga_ops.cpp:130-144) + mutate_block
 * (:164-178), or eda_sample (:214-238) + mutate_block */
int gapa_cuda_ga_slots_variation_device(int32_t* pool_dev, const int32_t* parent_dev, const int32_t* child_dev,
                                        const int32_t* partner_dev, int s, int k, int row_first, int row_count,
                                        double pc, double pm, int32_t pool_size, uint64_t seed, uint64_t generation,
                                        void* stream);
/* variation + evaluation of the same row block in one call: builds the children of rows
 * [row_first, row_first + row_count) into their slots and writes their fitness to
 * fit_block_dev[0 .. row_count).  For the PC / MCN tasks the child genes go to HBM and into the
 * shared-memory removal bitmap in one fused kernel (the row is never read back). */
int gapa_cuda_ga_slots_variation_eval_device(gapa_cuda_ctx* ctx, int task, int32_t* pool_dev, const int32_t* parent_dev,
                                             const int32_t* child_dev, const int32_t* partner_dev, int s, int k,
                                             int row_first, int row_count, double pc, double pm, uint64_t seed,
                                             uint64_t generation, double* fit_block_dev, void* stream);
/* elitism (ga_ops.cpp:180-212) as a permutation: next_parent = slots of the s best of the 2s stacked
 * rows (stable, originals first on ties), next_child = the s freed slots, next_fit = their fitness.
 * Children of rows outside [block_lo, block_hi) that survive are rebuilt in their slots from the
 * parents and the keyed streams (row sharding: they were built on another rank). */
int gapa_cuda_ga_slots_elitism_device(int32_t* pool_dev, const int32_t* parent_dev, const int32_t* child_dev,
                                      const int32_t* partner_dev, int s, int k, int block_lo, int block_hi,
                                      const double* fit_dev, const double* fit_m_dev, int minimize, double pc,
                                      double pm, int32_t pool_size, uint64_t seed, uint64_t generation,
                                      int32_t* next_parent_dev, int32_t* next_child_dev, double* next_fit_dev,
                                      void* stream);
/* dense row-major matrix of the rows table_dev names (PopulationMatrix, population.hpp:12-40) */
int gapa_cuda_ga_slots_gather_device(const int32_t* pool_dev, const int32_t* table_dev, int rows, int k,
                                     int32_t* out_dev, void* stream);
/* evaluate_batch over rows addressed through a slot table: row i = pool_dev + slot_dev[i] * cols */
int gapa_cuda_eval_rows_device(gapa_cuda_ctx* ctx, int task, const int32_t* pool_dev, const int32_t* slot_dev,
                               int rows, int cols, double* out_dev, void* stream);

/* record_generation (modes.cpp:35-43): best_dev[0] = fit[0], mean_dev[0] = sequential
 * sum(fit) / s — the reference's std::accumulate order, so non-integer fitness means
 * are bit-identical. */
int gapa_cuda_ga_stats_device(const double* fit_dev, int s, double* best_dev, double* mean_dev, void* stream);

/* Host-buffer forms of the same operators (H2D, kernel, D2H, synchronous) — the
 * exact shapes of the reference free functions, used by the host adapters and
 * the parity tests.  `device` selects the GPU. */
int gapa_cuda_ga_init(int device, int32_t pool_size, int row_first, int row_count, int budget, uint64_t seed,
                      uint64_t generation, int32_t* out);
int gapa_cuda_ga_mask(int device, int role, double rate, int rows, int cols, uint64_t seed, uint64_t generation, uint8_t* out);
int gapa_cuda_ga_mutation_indices(int device, int32_t pool_size, int rows, int cols, uint64_t seed, uint64_t generation,
                                  int32_t* out);
int gapa_cuda_ga_selection_weights(int device, const double* fitness, int s, int minimize, double* weights);
int gapa_cuda_ga_select(int device, const double* fitness, int s, int minimize, uint64_t seed,
                        uint64_t generation, int32_t* partner_index);
int gapa_cuda_ga_crossover_mutate(int device, const int32_t* pop, const int32_t* partner_index, int s, int k,
                                  int row_first, int row_count, double pc, double pm, int32_t pool_size,
                                  uint64_t seed, uint64_t generation, int32_t* out);
int gapa_cuda_ga_mutate(int device, const int32_t* block, int rows, int k, int row_offset, double pm,
                        int32_t pool_size, uint64_t seed, uint64_t generation, int32_t* out);
int gapa_cuda_ga_eda(int device, const int32_t* elite, int s, int k, int elite_count, int32_t pool_size,
                     uint64_t seed, uint64_t generation, int smoothing, int32_t* out);
int gapa_cuda_ga_elitism(int device, const int32_t* pop, const int32_t* m_pop, int s, int k, const double* fit,
                         const double* fit_m, int minimize, int32_t* next, double* next_fit);
/* first `count` raw draws of RngPolicy(seed).stream(generation, role, row)
 * (rng.hpp:21) computed ON THE DEVICE — the known-answer hook for the RNG twin */
int gapa_cuda_rng_draws(int device, uint64_t seed, uint64_t generation, uint64_t role, uint64_t row, int count,
                        uint64_t* out);

/* ---- generation loop (modes.cpp:132-178 == run_serial :359-418) ------------------ */
typedef struct gapa_cuda_run_params {
    double pc, pm;          /* GAParams, ga_ops.hpp:12-23 */
    int32_t pop_size;       /* s >= 2  */
    int32_t budget;         /* k >= 1  */
    int32_t iterations;     /* >= 1 (modes.cpp:26-29) */
    int32_t minimize;       /* Direction */
    int32_t eda_interval;   /* 0 = none */
    int32_t task;           /* GAPA_TASK_* */
    uint64_t seed;
    /* population sharding (modes.cpp:506-516): this process evaluates block
     * `rank` of partition_rows(s, world); 0/1 = single GPU. */
    int32_t rank, world;
} gapa_cuda_run_params;

/* Exchange hook for world > 1: must fill fit_full_dev[s] from every rank's
 * block fit_full_dev[lo..hi) (an all-gather; NCCL over NVLink in the Python
 * driver).  `padded_block` = ceil(s/world).  NULL when world == 1. */
typedef int (*gapa_cuda_allgather_fn)(void* user, double* fit_full_dev, int s, int padded_block, void* stream);

typedef struct gapa_cuda_run_result {
    double* history_best;      /* [iterations]  GenerationStats::best  (modes.hpp:63-71) */
    double* history_mean;      /* [iterations]  GenerationStats::mean                    */
    int32_t* final_population; /* [s x k]       RunResult::final_population (best first) */
    double* final_fitness;     /* [s]                                                    */
    uint64_t fitness_batch_calls;
    double total_wall_seconds; /* generation loop only */
    double eval_seconds;       /* device time inside fitness kernels (CUDA events)        */
    /* GenerationStats timing columns (modes.hpp:63-71), each [iterations] or NULL.  Device time
     * between CUDA events recorded on the run's stream and read back after the loop, so asking for
     * them adds no synchronisation.  wall = one generation (generation 1 includes init + the first
     * evaluation, modes.cpp:139-156); exchange = time inside the exchange hook (the fitness
     * all-gather; 0 on one GPU); lifecycle = 0 (no worker threads are spawned or joined);
     * compute = wall - exchange - lifecycle (record_generation, modes.cpp:38-40);
     * messages = exchanges issued in that generation.  On one GPU with pop_size <= 512 the events are SAMPLED
     * (generation 1, 2, then every eighth): generations between two marks report their mean wall time and
     * eval_seconds is scaled from the timed evaluations, because an event costs about as much as a kernel there. */
    double* gen_wall_seconds;
    double* gen_compute_seconds;
    double* gen_exchange_seconds;
    double* gen_lifecycle_seconds;
    uint64_t* gen_messages;
} gapa_cuda_run_result;

int gapa_cuda_run(gapa_cuda_ctx* ctx, const gapa_cuda_run_params* params, gapa_cuda_allgather_fn exchange,
                  void* exchange_user, gapa_cuda_run_result* result);

/* The same loop as a resumable object: the population stays in HBM between calls, so a host can interleave its own
 * work (logging, check-pointing, a stop criterion on history_best — modes.cpp:159-175 is a plain for loop) with
 * blocks of generations.  gapa_cuda_run == create + advance(iterations) + result + destroy.
 *   create:  validates like gapa_cuda_run; want_stats != 0 collects the GenerationStats timing columns
 *   advance: runs min(generations, iterations - done) generations; returns when they have finished on the device;
 *            *device_ms (optional) = device time of the block, CUDA events on the run's stream
 *   result:  history (zeros beyond the generations done), final population / fitness = the CURRENT parents */
typedef struct gapa_cuda_ga gapa_cuda_ga;
int gapa_cuda_ga_create(gapa_cuda_ctx* ctx, const gapa_cuda_run_params* params, gapa_cuda_allgather_fn exchange,
                        void* exchange_user, int want_stats, gapa_cuda_ga** out);
int gapa_cuda_ga_advance(gapa_cuda_ga* ga, int generations, float* device_ms);
int gapa_cuda_ga_generation(const gapa_cuda_ga* ga, int* generations_done);
int gapa_cuda_ga_result(gapa_cuda_ga* ga, gapa_cuda_run_result* result);
int gapa_cuda_ga_destroy(gapa_cuda_ga* ga);

/* ---- the exchange of a row-sharded run, shipped with the library (the GPU form of Channel<T>, channel.hpp:12-35) ----
 * A communicator connects the `world` ranks of one run (one rank per GPU; ranks may be threads of one process or
 * separate processes on one node).  gapa_cuda_comm_allgather has the gapa_cuda_allgather_fn signature: pass it, with
 * the communicator as `exchange_user`, to gapa_cuda_run / gapa_cuda_ga_create.
 *   PEER: mailboxes in HBM that the peers write directly over NVLink / NVSwitch (same process: peer access; other
 *         processes: CUDA IPC) — one kernel per exchange, no host involvement.  Set-up: every rank calls
 *         gapa_cuda_comm_create and publishes the GAPA_CUDA_COMM_HANDLE_BYTES it returns to all ranks by any
 *         out-of-band means (a file, MPI, torch.distributed, a pipe); every rank then calls gapa_cuda_comm_connect
 *         with the `world` handles in rank order.
 *   NCCL: ncclAllGather on the caller's stream (libnccl.so.2 is loaded at run time).  Set-up: rank 0 calls
 *         gapa_cuda_nccl_unique_id and publishes the 128 bytes; every rank calls gapa_cuda_comm_create_nccl
 *         (collectively, like ncclCommInitRank).
 * A peer that does not arrive within GAPA_COMM_TIMEOUT_MS (default 20000) turns into GAPA_CUDA_E_CUDA from
 * gapa_cuda_comm_status / the run, not into a hang. */
#define GAPA_CUDA_COMM_HANDLE_BYTES 128
#define GAPA_CUDA_COMM_CTRL_BYTES 256
enum { GAPA_COMM_PEER = 0, GAPA_COMM_NCCL = 1 };
typedef struct gapa_cuda_comm gapa_cuda_comm;
int gapa_cuda_comm_create(gapa_cuda_ctx* ctx, int rank, int world, int pop_size, gapa_cuda_comm** out, void* handle_out);
int gapa_cuda_comm_connect(gapa_cuda_comm* comm, const void* all_handles);
int gapa_cuda_nccl_unique_id(void* id128_out);
int gapa_cuda_comm_create_nccl(gapa_cuda_ctx* ctx, const void* unique_id128, int rank, int world, gapa_cuda_comm** out);
int gapa_cuda_comm_allgather(void* comm, double* fit_full_dev, int s, int padded_block, void* stream);
/* host-level all-gather of up to GAPA_CUDA_COMM_CTRL_BYTES bytes per rank through the same transport (blocking):
 * all_host receives world x bytes in rank order */
int gapa_cuda_comm_allgather_bytes(gapa_cuda_comm* comm, const void* mine_host, int bytes, void* all_host);
int gapa_cuda_comm_status(gapa_cuda_comm* comm);
int gapa_cuda_comm_info(const gapa_cuda_comm* comm, int* transport, int* rank, int* world);
int gapa_cuda_comm_destroy(gapa_cuda_comm* comm);
/* run_mode_m for C / C++ hosts (modes.cpp:190-349): ONE process, one host thread per context (normally one context
 * per GPU), row blocks by partition_rows, the exchange built in (transport = GAPA_COMM_PEER or GAPA_COMM_NCCL).
 * params->rank / world are ignored; results[r] is rank r's result — every rank ends with the same history and
 * population (test_parallel.cpp:86-104), so hosts usually fill in results[0] only and leave the others' output
 * pointers null. */
int gapa_cuda_run_multi(gapa_cuda_ctx* const* ctxs, int world, const gapa_cuda_run_params* params, int transport,
                        gapa_cuda_run_result* results);

/* ---- host-side problem setup (CPU, once per experiment — inputs to the path) --------
 * Deterministic generators with the reference's draw sequences (generators.cpp) and
 * the link-prediction split builder (link_prediction.cpp:11-53).  `uv` receives
 * canonical (u < v) pairs in insertion order; pass uv == NULL to query *m first. */
int gapa_host_barabasi_albert(int32_t n, int32_t attach, uint64_t seed, int32_t* uv, int64_t capacity, int64_t* m);
int gapa_host_erdos_renyi(int32_t n, double p, uint64_t seed, int32_t* uv, int64_t capacity, int64_t* m);
int gapa_host_planted_partition(int32_t blocks, int32_t block_size, double p_in, double p_out, uint64_t seed,
                                int32_t* uv, int64_t capacity, int64_t* m);
/* train_uv[(m-T) x 2], test_uv[T x 2], probe_uv[T x 2]; null outputs = query T */
int gapa_host_lp_split(int32_t n, int64_t m, const int32_t* edges, double fraction, uint64_t seed,
                       int32_t* train_uv, int32_t* test_uv, int32_t* probe_uv, int32_t* test_count);
/* EdgeAddition pool of build_gene_pool (gene_pool.cpp:81-87): every non-edge a < b in
 * lexicographic order; uv == NULL queries *count.  Fails on a complete graph (:86). */
int gapa_host_nonedges(int32_t n, int64_t m, const int32_t* edges, int32_t* uv, int64_t capacity, int64_t* count);
/* perturbation_budget (gene_pool.cpp:98-102): k = max(1, ceil(rate * basis)) */
int gapa_host_budget(int64_t basis, double rate, int32_t* k);

/* ---- plumbing for hosts without a CUDA runtime of their own ---------------------- */
int gapa_cuda_malloc(int device, uint64_t bytes, void** out_dev);
int gapa_cuda_free(int device, void* dev);
int gapa_cuda_memcpy_h2d(int device, void* dst_dev, const void* src_host, uint64_t bytes);
int gapa_cuda_memcpy_d2h(int device, void* dst_host, const void* src_dev, uint64_t bytes);
int gapa_cuda_stream_sync(int device, void* stream);
/* ---- reporting outputs for ONE individual (the experiment driver's metric columns, bench.cpp:268-311) ----
 * gapa_cuda_detect_communities: CommunityPartition of detect_communities (community.cpp:28-91) on the
 * graph perturbed by `genes` (EdgeRemoval or EdgeAddition pool), normalised by first appearance
 * (community.cpp:17-26), into assignment[n]; *q (optional) = the cda fitness of the same individual.
 * gapa_cuda_lpa_scores: ra_scores (link_prediction.cpp:71-77) of the T test and P probe pairs on the
 * perturbed train graph — the inputs of lp_auc_precision's precision half (:98-117); *auc optional. */
int gapa_cuda_detect_communities(gapa_cuda_ctx* ctx, const int32_t* genes_host, int cols, int32_t* assignment_host,
                                 double* q_host);
int gapa_cuda_lpa_scores(gapa_cuda_ctx* ctx, const int32_t* genes_host, int cols, double* test_scores_host,
                         double* probe_scores_host, double* auc_host);

/* launch counter: kernels launched by this library since load (bench.py's gpu_launches) */
uint64_t gapa_cuda_launch_count(void);
/* timing of the last eval on a context: device milliseconds between CUDA events
 * recorded on the eval stream around the kernels only (no copies). */
int gapa_cuda_last_eval_ms(const gapa_cuda_ctx* ctx, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* GAPA_CUDA_H */
