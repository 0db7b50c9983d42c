/* TEST INFRASTRUCTURE — the parity oracle, not the product.
 *
 * Plain-C, CPU-only restatement of the reference's hot path (GAPA,
 * /root/reference/proj) on a shared CSR instead of the reference's dense
 * n x n BitMatrix, so that it also runs at n = 10^6 where the reference
 * cannot (125 GB per individual copy).  Each function cites the reference
 * file:line it follows.  Parity is PINNED: tests/test_oracle_vs_ref.py checks
 * every function here for exact equality against the compiled, unmodified
 * reference (oracle/_ref/libgapa_ref.so) and tests/test_oracle_golden.py
 * checks it against the committed golden vectors under tests/golden/
 * (generated from that same reference by tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product
 * (paper_2412_20980_b200/) never does.
 */
#ifndef GAPA_ORACLE_H
#define GAPA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:8-65 ------------------------------------------------------ */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_stream_key(uint64_t seed, uint64_t generation, uint64_t role, uint64_t row);
uint64_t orc_draw_u64(uint64_t key, uint64_t j); /* j-th draw of a stream, j >= 1 */
double orc_draw_unit(uint64_t key, uint64_t j);
uint32_t orc_draw_index(uint64_t key, uint64_t j, uint32_t bound);

enum { ORC_ROLE_INIT = 1, ORC_ROLE_SELECT = 2, ORC_ROLE_CROSSOVER_MASK = 3,
       ORC_ROLE_MUTATION_MASK = 4, ORC_ROLE_MUTATION_INDEX = 5 };

enum { ORC_TASK_PC = 0, ORC_TASK_MCN = 1, ORC_TASK_CDA = 2, ORC_TASK_LPA = 3,
       ORC_TASK_SIXDST = 4,   /* sixdst_fitness(ClosurePolicy::SixDegrees), fitness.cpp:18-26      */
       ORC_TASK_CDA_ADD = 5   /* cda_fitness over the EdgeAddition pool, gene_pool.cpp:57-60,81-87 */ };

/* ---- graph: canonical edge list (insertion order) + sorted CSR ----------- */
typedef struct orc_graph {
    int32_t n;
    int64_t m;
    int32_t* edge_uv;  /* 2m, u < v, insertion order (graph.hpp:26)            */
    int32_t* row_ptr;  /* n + 1                                                */
    int32_t* col_idx;  /* 2m, ascending inside each row                        */
    int32_t* edge_id;  /* 2m, rank of the undirected edge in (u,v)-sorted order
                          = EdgeRemoval gene id (gene_pool.cpp:73-79)          */
    int32_t* pool_u;   /* m, endpoints of gene id e                            */
    int32_t* pool_v;
    /* EdgeAddition pool (gene_pool.cpp:81-87): every non-edge (u < v) in
     * lexicographic order; built on demand by orc_graph_build_addition_pool */
    int64_t add_size;
    int32_t* add_u;
    int32_t* add_v;
} orc_graph;

orc_graph* orc_graph_create(int32_t n, int64_t m, const int32_t* uv); /* NULL on bad input */
orc_graph* orc_graph_ba(int32_t n, int32_t attach, uint64_t seed);    /* generators.cpp:21-45 */
orc_graph* orc_graph_er(int32_t n, double p, uint64_t seed);          /* generators.cpp:11-19 */
orc_graph* orc_graph_sbm(int32_t blocks, int32_t block_size, double p_in, double p_out,
                         uint64_t seed);                              /* generators.cpp:47-58 */
void orc_graph_free(orc_graph* g);
int orc_graph_has_edge(const orc_graph* g, int32_t u, int32_t v);
int32_t orc_budget(int64_t basis, double rate); /* gene_pool.cpp:98-102 */

/* ---- link-prediction split (link_prediction.cpp:11-53) ------------------- */
typedef struct orc_split {
    orc_graph* train;
    int32_t T, P;
    int32_t* test_uv;  /* 2T sorted */
    int32_t* probe_uv; /* 2P sorted */
} orc_split;
orc_split* orc_split_build(const orc_graph* g, double fraction, uint64_t seed);
void orc_split_free(orc_split* s);

/* ---- fitness (fitness.cpp:18-48) ------------------------------------------ */
/* NodeRemoval genes are node ids (identity pool, gene_pool.cpp:89-92);
 * EdgeRemoval genes are edge ranks.  Returns 0, or non-zero on an
 * out-of-range gene. */
int orc_pc_batch(const orc_graph* g, int task, const int32_t* genes, int rows, int cols, double* out);
int orc_cda_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out);
/* ClosurePolicy::SixDegrees (accessibility.cpp:20-37): (A+I) squared at most 3 times covers
 * exactly the paths of length <= 8, so row u of the closure is the radius-8 ball of u in the
 * perturbed graph; fitness = the largest ball (fitness.cpp:23-25). */
int orc_sixdst_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out);
/* EdgeAddition: returns the pool size, or -1 if the graph is complete / the pool
 * does not fit int32 (gene_pool.cpp:81-87). */
int64_t orc_graph_build_addition_pool(orc_graph* g);
int orc_cda_add_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out);
int orc_lpa_batch(const orc_split* s, const int32_t* genes, int rows, int cols, double* out);
/* task dispatch + contiguous row blocks (modes.cpp:506-516) over pthreads */
int orc_eval_batch(const void* g_or_split, int task, const int32_t* genes, int rows, int cols,
                   int threads, double* out);
/* greedy detector alone (community.cpp:28-91), assignment normalised */
int orc_detect_communities(const orc_graph* g, int32_t* assignment);
double orc_ra_score(const orc_graph* g, int32_t u, int32_t v); /* link_prediction.cpp:55-69 */

/* ---- genetic operators (ga_ops.cpp) ---------------------------------------- */
/* PARITY UNPINNED (no reference implementation): CN score and edge-flip pools for the link-prediction attack */
void orc_flip_unrank(int32_t n, int64_t id, int32_t* a_out, int32_t* b_out);
int orc_lpa_flip_batch(const orc_split* s, int score_kind, const int32_t* pool_uv, int64_t pool_size, const int32_t* genes,
                       int rows, int cols, double* out);
int orc_lpa_scored_batch(const orc_split* s, int score_kind, const int32_t* genes, int rows, int cols, double* out);
void orc_make_mask(int rows, int cols, double rate, int role, uint64_t seed, uint64_t generation, uint8_t* out);
void orc_make_mutation_indices(int rows, int cols, int pool_size, uint64_t seed, uint64_t generation, int32_t* out);
int orc_init_population_block(int pool_size, int row_first, int row_count, int budget,
                              uint64_t seed, uint64_t generation, int32_t* out);
int orc_selection_weights(const double* fitness, int s, int minimize, double* out);
int orc_roulette_pick(const double* fitness, int s, int minimize, uint64_t seed,
                      uint64_t generation, int32_t* partner_index);
void orc_crossover(const int32_t* pop, const int32_t* partner_index, int s, int k, double pc,
                   uint64_t seed, uint64_t generation, int32_t* out);
void orc_mutate_block(const int32_t* block, int rows, int k, int row_offset, double pm,
                      int pool_size, uint64_t seed, uint64_t generation, int32_t* out);
int orc_elitism(const int32_t* pop, const int32_t* m_pop, int s, int k, const double* fit_pop,
                const double* fit_m, int minimize, int32_t* next, double* next_fit);
int orc_eda_sample(const int32_t* elite, int s, int k, int elite_count, int pool_size,
                   uint64_t seed, uint64_t generation, int smoothing, int32_t* out);
void orc_partition_rows(int pop_size, int pn, int32_t* lo_hi);

/* ---- generation loop (modes.cpp:132-178 == :359-418) ------------------------ */
int orc_run_ga(const void* g_or_split, int task, double pc, double pm, int pop_size, int budget,
               int iterations, int eda_interval, uint64_t seed, int minimize, int threads,
               double* history_best, double* history_mean, int32_t* final_population,
               double* final_fitness);

#ifdef __cplusplus
}
#endif
#endif
