/* TEST INFRASTRUCTURE — the parity oracle, not the product.  See gapa_oracle.h.
 *
 * Plain-C CSR restatement of the reference hot path; citations are
 * file:line under /root/reference/proj.  Build: oracle/Makefile
 * (-O2 -ffp-contract=off: no FMA contraction, FP64 must match bit for bit).
 */
#include "gapa_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= rng */

/* include/gapa/rng.hpp:8-13 */
uint64_t orc_mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* include/gapa/rng.hpp:59-65 */
uint64_t orc_stream_key(uint64_t seed, uint64_t generation, uint64_t role, uint64_t row) {
    uint64_t key = orc_mix64(seed);
    key = orc_mix64(key ^ generation);
    key = orc_mix64(key ^ role);
    key = orc_mix64(key ^ row);
    return key;
}

/* include/gapa/rng.hpp:21 — the counter is pre-incremented, so draw j uses j */
uint64_t orc_draw_u64(uint64_t key, uint64_t j) { return orc_mix64(key + 0x632BE59BD9B4E019ull * j); }

/* include/gapa/rng.hpp:24 */
double orc_draw_unit(uint64_t key, uint64_t j) { return (double)(orc_draw_u64(key, j) >> 11) * 0x1.0p-53; }

/* include/gapa/rng.hpp:28-31 */
uint32_t orc_draw_index(uint64_t key, uint64_t j, uint32_t bound) {
    return (uint32_t)(((unsigned __int128)orc_draw_u64(key, j) * bound) >> 64);
}

/* sequential stream used by the generators and the split builder */
typedef struct { uint64_t key, counter; } seq_stream;
static uint64_t seq_u64(seq_stream* s) { return orc_draw_u64(s->key, ++s->counter); }
static double seq_unit(seq_stream* s) { return (double)(seq_u64(s) >> 11) * 0x1.0p-53; }
static uint32_t seq_index(seq_stream* s, uint32_t bound) {
    return (uint32_t)(((unsigned __int128)seq_u64(s) * bound) >> 64);
}

/* ===================================================================== graph */

typedef struct { int32_t* v; int64_t len, cap; } ivec;
static void ivec_push(ivec* a, int32_t x) {
    if (a->len == a->cap) {
        a->cap = a->cap ? a->cap * 2 : 1024;
        a->v = (int32_t*)realloc(a->v, sizeof(int32_t) * (size_t)a->cap);
    }
    a->v[a->len++] = x;
}

void orc_graph_free(orc_graph* g) {
    if (!g) return;
    free(g->edge_uv); free(g->row_ptr); free(g->col_idx); free(g->edge_id);
    free(g->pool_u); free(g->pool_v); free(g->add_u); free(g->add_v); free(g);
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* Graph::Graph (graph.cpp:17-36) canonicalises to u < v and rejects loops,
 * out-of-range endpoints and duplicates; adjacency() (graph.cpp:47-54) is
 * restated as a CSR with ascending rows; the EdgeRemoval pool order
 * (gene_pool.cpp:73-79) is the (u, v)-lexicographic rank, stored per slot. */
orc_graph* orc_graph_create(int32_t n, int64_t m, const int32_t* uv) {
    if (n < 0 || m < 0) return NULL;
    orc_graph* g = (orc_graph*)calloc(1, sizeof(orc_graph));
    g->n = n; g->m = m;
    g->edge_uv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
    g->row_ptr = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    g->col_idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
    g->edge_id = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
    g->pool_u = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    g->pool_v = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    for (int64_t e = 0; e < m; ++e) {
        int32_t u = uv[2 * e], v = uv[2 * e + 1];
        if (u == v || u < 0 || v < 0 || u >= n || v >= n) { orc_graph_free(g); return NULL; }
        if (u > v) { int32_t t = u; u = v; v = t; }
        g->edge_uv[2 * e] = u; g->edge_uv[2 * e + 1] = v;
        g->row_ptr[u + 1]++; g->row_ptr[v + 1]++;
    }
    for (int32_t u = 0; u < n; ++u) g->row_ptr[u + 1] += g->row_ptr[u];
    int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    memcpy(fill, g->row_ptr, sizeof(int32_t) * ((size_t)n + 1));
    for (int64_t e = 0; e < m; ++e) {
        const int32_t u = g->edge_uv[2 * e], v = g->edge_uv[2 * e + 1];
        g->col_idx[fill[u]++] = v;
        g->col_idx[fill[v]++] = u;
    }
    free(fill);
    for (int32_t u = 0; u < n; ++u) {
        const int32_t b = g->row_ptr[u], e = g->row_ptr[u + 1];
        qsort(g->col_idx + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
        for (int32_t i = b + 1; i < e; ++i)
            if (g->col_idx[i] == g->col_idx[i - 1]) { orc_graph_free(g); return NULL; } /* duplicate edge */
    }
    /* rank of (u, v), u < v, in sorted order; the mirror slot gets the same id */
    int32_t next = 0;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
            const int32_t v = g->col_idx[i];
            if (v > u) {
                g->edge_id[i] = next;
                g->pool_u[next] = u; g->pool_v[next] = v;
                ++next;
            }
        }
    for (int32_t u = 0; u < n; ++u)
        for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
            const int32_t v = g->col_idx[i];
            if (v < u) { /* find u in row v */
                int32_t lo = g->row_ptr[v], hi = g->row_ptr[v + 1];
                while (lo < hi) { int32_t mid = (lo + hi) / 2; if (g->col_idx[mid] < u) lo = mid + 1; else hi = mid; }
                g->edge_id[i] = g->edge_id[lo];
            }
        }
    return g;
}

int orc_graph_has_edge(const orc_graph* g, int32_t u, int32_t v) {
    if (u == v) return 0;
    int32_t lo = g->row_ptr[u], hi = g->row_ptr[u + 1];
    while (lo < hi) { int32_t mid = (lo + hi) / 2; if (g->col_idx[mid] < v) lo = mid + 1; else hi = mid; }
    return lo < g->row_ptr[u + 1] && g->col_idx[lo] == v;
}

/* generators.cpp:21-45 */
orc_graph* orc_graph_ba(int32_t n, int32_t attach, uint64_t seed) {
    if (n < 1 || attach < 1) return NULL;
    seq_stream rng = {orc_mix64(seed ^ 0x42415241ull), 0};
    ivec edges = {0}, pool = {0};
    int32_t* chosen = (int32_t*)malloc(sizeof(int32_t) * (size_t)attach);
    ivec_push(&pool, 0);
    for (int32_t v = 1; v < n; ++v) {
        const int32_t want = attach < v ? attach : v;
        int32_t got = 0;
        while (got < want) {
            const int32_t target = pool.v[seq_index(&rng, (uint32_t)pool.len)];
            int dup = 0;
            for (int32_t c = 0; c < got; ++c) dup |= (chosen[c] == target);
            if (!dup) chosen[got++] = target;
        }
        for (int32_t c = 0; c < got; ++c) {
            ivec_push(&edges, chosen[c]); ivec_push(&edges, v);
            ivec_push(&pool, chosen[c]); ivec_push(&pool, v);
        }
    }
    orc_graph* g = orc_graph_create(n, edges.len / 2, edges.v);
    free(edges.v); free(pool.v); free(chosen);
    return g;
}

/* generators.cpp:11-19 */
orc_graph* orc_graph_er(int32_t n, double p, uint64_t seed) {
    if (n < 0 || p < 0.0 || p > 1.0) return NULL;
    seq_stream rng = {orc_mix64(seed ^ 0x45524e4f53ull), 0};
    ivec edges = {0};
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v)
            if (seq_unit(&rng) < p) { ivec_push(&edges, u); ivec_push(&edges, v); }
    orc_graph* g = orc_graph_create(n, edges.len / 2, edges.v);
    free(edges.v);
    return g;
}

/* generators.cpp:47-58 */
orc_graph* orc_graph_sbm(int32_t blocks, int32_t block_size, double p_in, double p_out, uint64_t seed) {
    if (blocks < 1 || block_size < 1) return NULL;
    seq_stream rng = {orc_mix64(seed ^ 0x50504d4full), 0};
    const int32_t n = blocks * block_size;
    ivec edges = {0};
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v) {
            const double p = (u / block_size == v / block_size) ? p_in : p_out;
            if (seq_unit(&rng) < p) { ivec_push(&edges, u); ivec_push(&edges, v); }
        }
    orc_graph* g = orc_graph_create(n, edges.len / 2, edges.v);
    free(edges.v);
    return g;
}

/* gene_pool.cpp:98-102 (rate validated by the caller) */
int32_t orc_budget(int64_t basis, double rate) {
    const int32_t k = (int32_t)ceil(rate * (double)basis);
    return k > 1 ? k : 1;
}

/* ==================================================================== split */

static int cmp_pair(const void* a, const void* b) {
    const int32_t* x = (const int32_t*)a; const int32_t* y = (const int32_t*)b;
    if (x[0] != y[0]) return (x[0] > y[0]) - (x[0] < y[0]);
    return (x[1] > y[1]) - (x[1] < y[1]);
}

void orc_split_free(orc_split* s) {
    if (!s) return;
    orc_graph_free(s->train); free(s->test_uv); free(s->probe_uv); free(s);
}

/* link_prediction.cpp:11-53 */
orc_split* orc_split_build(const orc_graph* g, double fraction, uint64_t seed) {
    if (fraction <= 0.0 || fraction > 0.5 || g->m < 10) return NULL;
    const int32_t m = (int32_t)g->m;
    long tc = lround(fraction * (double)m);
    const int32_t test_count = tc > 1 ? (int32_t)tc : 1;
    seq_stream rng = {orc_mix64(seed ^ 0x4c505350ull), 0};
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
    for (int32_t i = 0; i < m; ++i) order[i] = i;
    for (int32_t i = m - 1; i > 0; --i) {
        const uint32_t j = seq_index(&rng, (uint32_t)(i + 1));
        const int32_t t = order[i]; order[i] = order[j]; order[j] = t;
    }
    orc_split* s = (orc_split*)calloc(1, sizeof(orc_split));
    s->T = test_count; s->P = test_count;
    s->test_uv = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)test_count);
    s->probe_uv = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)test_count);
    int32_t* train = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(m - test_count + 1));
    int32_t nt = 0, ntr = 0;
    for (int32_t i = 0; i < m; ++i) {
        const int32_t* e = g->edge_uv + 2 * (size_t)order[i];
        if (i < test_count) { s->test_uv[2 * nt] = e[0]; s->test_uv[2 * nt + 1] = e[1]; ++nt; }
        else { train[2 * ntr] = e[0]; train[2 * ntr + 1] = e[1]; ++ntr; }
    }
    qsort(s->test_uv, (size_t)nt, 2 * sizeof(int32_t), cmp_pair);
    qsort(train, (size_t)ntr, 2 * sizeof(int32_t), cmp_pair);
    s->train = orc_graph_create(g->n, ntr, train);
    free(train); free(order);

    /* probe non-edges: rejection sampling with a `used` set (open addressing) */
    size_t cap = 16; while (cap < (size_t)test_count * 4) cap <<= 1;
    uint64_t* used = (uint64_t*)malloc(sizeof(uint64_t) * cap);
    memset(used, 0xff, sizeof(uint64_t) * cap);
    int32_t np = 0;
    while (np < test_count) {
        const int32_t u = (int32_t)seq_index(&rng, (uint32_t)g->n);
        const int32_t v = (int32_t)seq_index(&rng, (uint32_t)g->n);
        if (u == v || orc_graph_has_edge(g, u, v)) continue;
        const int32_t a = u < v ? u : v, b = u < v ? v : u;
        const uint64_t key = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
        size_t h = (size_t)(orc_mix64(key) & (cap - 1));
        int seen = 0;
        while (used[h] != ~0ull) { if (used[h] == key) { seen = 1; break; } h = (h + 1) & (cap - 1); }
        if (seen) continue;
        used[h] = key;
        s->probe_uv[2 * np] = a; s->probe_uv[2 * np + 1] = b; ++np;
    }
    free(used);
    qsort(s->probe_uv, (size_t)np, 2 * sizeof(int32_t), cmp_pair);
    return s;
}

/* ================================================================ PC / MCN */

/* gene_pool.cpp:61-64 (zero row + column == drop the node's edges, the node
 * stays as a singleton) + components.cpp:9-35 (DFS) + :49-62. */
static int pc_one(const orc_graph* g, int task, const int32_t* genes, int k,
                  uint8_t* removed, uint8_t* visited, int32_t* stack, double* out) {
    const int32_t n = g->n;
    memset(removed, 0, (size_t)n);
    for (int j = 0; j < k; ++j) {
        if (genes[j] < 0 || genes[j] >= n) return 1;
        removed[genes[j]] = 1;
    }
    memset(visited, 0, (size_t)n);
    int64_t total = 0; int32_t best = 0;
    for (int32_t start = 0; start < n; ++start) {
        if (visited[start]) continue;
        visited[start] = 1;
        int64_t size = 1;
        if (!removed[start]) {
            int32_t top = 0; stack[top++] = start;
            while (top) {
                const int32_t u = stack[--top];
                for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
                    const int32_t v = g->col_idx[i];
                    if (!visited[v] && !removed[v]) { visited[v] = 1; ++size; stack[top++] = v; }
                }
            }
        }
        total += size * (size - 1) / 2;
        if (size > best) best = (int32_t)size;
    }
    *out = task == ORC_TASK_PC ? (double)total : (double)best; /* fitness.cpp:25,32 */
    return 0;
}

int orc_pc_batch(const orc_graph* g, int task, const int32_t* genes, int rows, int cols, double* out) {
    const size_t n = (size_t)g->n;
    uint8_t* removed = (uint8_t*)malloc(n + 1);
    uint8_t* visited = (uint8_t*)malloc(n + 1);
    int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    int rc = 0;
    for (int i = 0; i < rows && !rc; ++i)
        rc = pc_one(g, task, genes + (size_t)i * cols, cols, removed, visited, stack, out + i);
    free(removed); free(visited); free(stack);
    return rc;
}

/* fitness.cpp:18-26 with ClosurePolicy::SixDegrees.  accessibility.cpp:20-37
 * squares A + I at most three times: after j squarings entry (u, v) is set iff
 * dist(u, v) <= 2^j, so the closure row of u is the ball of radius 8 around u
 * (u itself included through the diagonal; a removed node keeps only its
 * diagonal bit).  Restated as one depth-limited BFS per source on the CSR. */
int orc_sixdst_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out) {
    const int32_t n = g->n;
    uint8_t* removed = (uint8_t*)malloc((size_t)n + 1);
    int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int rc = 0;
    for (int r = 0; r < rows && !rc; ++r) {
        memset(removed, 0, (size_t)n + 1);
        for (int j = 0; j < cols; ++j) {
            const int32_t x = genes[(size_t)r * cols + j];
            if (x < 0 || x >= n) { rc = 1; break; }
            removed[x] = 1;
        }
        if (rc) break;
        for (int32_t u = 0; u < n; ++u) mark[u] = -1;
        int32_t best = 0;
        for (int32_t src = 0; src < n; ++src) {
            int32_t size = 1;
            if (!removed[src]) {
                int32_t head = 0, tail = 0;
                queue[tail++] = src; mark[src] = src;
                for (int depth = 0; depth < 8 && head < tail; ++depth) {
                    const int32_t level_end = tail;
                    for (; head < level_end; ++head) {
                        const int32_t u = queue[head];
                        for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
                            const int32_t v = g->col_idx[i];
                            if (mark[v] != src && !removed[v]) { mark[v] = src; queue[tail++] = v; }
                        }
                    }
                }
                size = tail;
            }
            if (size > best) best = size;
        }
        out[r] = (double)best;
    }
    free(removed); free(mark); free(queue);
    return rc;
}

/* ===================================================================== CDA */

typedef struct { int32_t id; int64_t cnt; } nb_t;
typedef struct { nb_t* a; int32_t len, cap; } nlist;

static int32_t nl_lower(const nlist* L, int32_t id) {
    int32_t lo = 0, hi = L->len;
    while (lo < hi) { int32_t mid = (lo + hi) / 2; if (L->a[mid].id < id) lo = mid + 1; else hi = mid; }
    return lo;
}
static void nl_add(nlist* L, int32_t id, int64_t e) {
    const int32_t p = nl_lower(L, id);
    if (p < L->len && L->a[p].id == id) { L->a[p].cnt += e; return; }
    if (L->len == L->cap) {
        L->cap = L->cap ? L->cap * 2 : 8;
        L->a = (nb_t*)realloc(L->a, sizeof(nb_t) * (size_t)L->cap);
    }
    memmove(L->a + p + 1, L->a + p, sizeof(nb_t) * (size_t)(L->len - p));
    L->a[p].id = id; L->a[p].cnt = e; L->len++;
}
static void nl_erase(nlist* L, int32_t id) {
    const int32_t p = nl_lower(L, id);
    if (p < L->len && L->a[p].id == id) {
        memmove(L->a + p, L->a + p + 1, sizeof(nb_t) * (size_t)(L->len - p - 1));
        L->len--;
    }
}

/* community.cpp:28-91 on the CSR minus the edges flagged in `gone` (may be
 * NULL).  owner[] is returned normalised by first appearance (:17-26). */
static void detect_on(const orc_graph* g, const uint8_t* gone, int32_t* owner) {
    const int32_t n = g->n;
    int64_t* cdeg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    nlist* nbr = (nlist*)calloc((size_t)n + 1, sizeof(nlist));
    int64_t total_degree = 0;
    for (int32_t u = 0; u < n; ++u) {
        owner[u] = u;
        for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
            if (gone && gone[g->edge_id[i]]) continue;
            cdeg[u]++;
            nl_add(&nbr[u], g->col_idx[i], 1); /* rows ascending: appends */
        }
        total_degree += cdeg[u];
    }
    const double m = (double)total_degree / 2.0; /* :36 */

    while (m > 0) { /* :55 */
        double best_gain = 0.0;
        int32_t best_a = -1, best_b = -1;
        for (int32_t a = 0; a < n; ++a) { /* std::map order = ascending a, then ascending b */
            const nlist* L = &nbr[a];
            if (!L->len) continue;
            const double da = (double)cdeg[a];
            for (int32_t i = 0; i < L->len; ++i) {
                const int32_t b = L->a[i].id;
                if (b <= a) continue;
                const double db = (double)cdeg[b];
                const double gain = (double)L->a[i].cnt / m - da * db / (2.0 * m * m); /* :63 */
                if (gain > best_gain) { best_gain = gain; best_a = a; best_b = b; }
            }
        }
        if (best_a < 0) break;
        /* :73-86 merge best_b into best_a */
        cdeg[best_a] += cdeg[best_b];
        nlist moved = nbr[best_b];
        nbr[best_b].a = NULL; nbr[best_b].len = nbr[best_b].cap = 0;
        for (int32_t i = 0; i < moved.len; ++i) {
            const int32_t c = moved.a[i].id;
            if (c == best_a) continue;
            nl_erase(&nbr[c], best_b);
            nl_add(&nbr[c], best_a, moved.a[i].cnt);
            nl_add(&nbr[best_a], c, moved.a[i].cnt);
        }
        free(moved.a);
        nl_erase(&nbr[best_a], best_b);
        for (int32_t u = 0; u < n; ++u)
            if (owner[u] == best_b) owner[u] = best_a;
    }
    for (int32_t u = 0; u < n; ++u) free(nbr[u].a);
    free(nbr); free(cdeg);

    /* CommunityPartition::normalized, community.cpp:17-26 */
    int32_t* remap = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    for (int32_t u = 0; u < n; ++u) remap[u] = -1;
    int32_t next = 0;
    for (int32_t u = 0; u < n; ++u) {
        if (remap[owner[u]] < 0) remap[owner[u]] = next++;
        owner[u] = remap[owner[u]];
    }
    free(remap);
}

/* community.cpp:93-117 */
static double modularity_on(const orc_graph* g, const uint8_t* gone, const int32_t* part) {
    const int32_t n = g->n;
    int32_t communities = 0;
    for (int32_t u = 0; u < n; ++u) if (part[u] + 1 > communities) communities = part[u] + 1;
    double* intra = (double*)calloc((size_t)communities + 1, sizeof(double));
    double* degree_sum = (double*)calloc((size_t)communities + 1, sizeof(double));
    int64_t pop = 0;
    for (int32_t u = 0; u < n; ++u) {
        const int32_t cu = part[u];
        int32_t deg = 0;
        for (int32_t i = g->row_ptr[u]; i < g->row_ptr[u + 1]; ++i) {
            if (gone && gone[g->edge_id[i]]) continue;
            ++deg;
            const int32_t v = g->col_idx[i];
            if (u < v && part[v] == cu) intra[cu] += 1.0;
        }
        degree_sum[cu] += deg;
        pop += deg;
    }
    const double two_m = (double)pop;
    double q = 0.0;
    for (int32_t c = 0; c < communities; ++c) {
        const double e = intra[c] / (two_m / 2.0);
        const double a = degree_sum[c] / two_m;
        q += e - a * a;
    }
    free(intra); free(degree_sum);
    return q;
}

int orc_detect_communities(const orc_graph* g, int32_t* assignment) {
    detect_on(g, NULL, assignment);
    return 0;
}

/* fitness.cpp:35-41 */
int orc_cda_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out) {
    uint8_t* gone = (uint8_t*)malloc((size_t)g->m + 1);
    int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->n + 1));
    int rc = 0;
    for (int r = 0; r < rows && !rc; ++r) {
        memset(gone, 0, (size_t)g->m + 1);
        int64_t left = g->m;
        for (int j = 0; j < cols; ++j) {
            const int32_t e = genes[(size_t)r * cols + j];
            if (e < 0 || e >= g->m) { rc = 1; break; }
            if (!gone[e]) { gone[e] = 1; --left; }
        }
        if (rc) break;
        if (left == 0) { out[r] = -0.5; continue; }
        detect_on(g, gone, owner);
        out[r] = modularity_on(g, gone, owner);
    }
    free(gone); free(owner);
    return rc;
}

/* gene_pool.cpp:81-87: every pair u < v that is not an edge, lexicographic. */
int64_t orc_graph_build_addition_pool(orc_graph* g) {
    if (g->add_u) return g->add_size;
    const int64_t n = g->n, size = n * (n - 1) / 2 - g->m;
    if (size <= 0 || size > 0x7fffffffll) return -1;
    g->add_u = (int32_t*)malloc(sizeof(int32_t) * (size_t)size);
    g->add_v = (int32_t*)malloc(sizeof(int32_t) * (size_t)size);
    int64_t next = 0;
    for (int32_t u = 0; u < g->n; ++u) {
        int32_t i = g->row_ptr[u];
        const int32_t ie = g->row_ptr[u + 1];
        while (i < ie && g->col_idx[i] <= u) ++i;
        for (int32_t v = u + 1; v < g->n; ++v) {
            if (i < ie && g->col_idx[i] == v) { ++i; continue; }
            g->add_u[next] = u; g->add_v[next] = v; ++next;
        }
    }
    g->add_size = next;
    return next;
}

/* fitness.cpp:35-41 with an EdgeAddition pool: apply_in_place sets both bits of
 * every gene's pair (gene_pool.cpp:57-60; duplicates idempotent), then the same
 * detector and modularity run on the enlarged graph. */
int orc_cda_add_batch(const orc_graph* g, const int32_t* genes, int rows, int cols, double* out) {
    if (!g->add_u) return 2;
    int32_t* uv = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(g->m + cols + 1));
    uint8_t* seen = (uint8_t*)calloc((size_t)g->add_size + 1, 1);
    int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->n + 1));
    int rc = 0;
    for (int r = 0; r < rows && !rc; ++r) {
        memcpy(uv, g->edge_uv, sizeof(int32_t) * 2 * (size_t)g->m);
        int64_t m2 = g->m;
        for (int j = 0; j < cols; ++j) {
            const int32_t e = genes[(size_t)r * cols + j];
            if (e < 0 || e >= g->add_size) { rc = 1; break; }
            if (seen[e]) continue;
            seen[e] = 1;
            uv[2 * m2] = g->add_u[e]; uv[2 * m2 + 1] = g->add_v[e]; ++m2;
        }
        for (int j = 0; j < cols; ++j) {
            const int32_t e = genes[(size_t)r * cols + j];
            if (e >= 0 && e < g->add_size) seen[e] = 0;
        }
        if (rc) break;
        if (m2 == 0) { out[r] = -0.5; continue; }
        orc_graph* p = orc_graph_create(g->n, m2, uv);
        if (!p) { rc = 2; break; }
        detect_on(p, NULL, owner);
        out[r] = modularity_on(p, NULL, owner);
        orc_graph_free(p);
    }
    free(uv); free(seen); free(owner);
    return rc;
}

/* ===================================================================== LPA */

/* link_prediction.cpp:55-69 on the CSR minus `gone` edges; deg[] are the
 * perturbed degrees; common neighbours are visited in ascending z. */
static double ra_on(const orc_graph* g, const uint8_t* gone, const int32_t* deg, int32_t u, int32_t v) {
    int32_t i = g->row_ptr[u], ie = g->row_ptr[u + 1];
    int32_t j = g->row_ptr[v], je = g->row_ptr[v + 1];
    double score = 0.0;
    while (i < ie && j < je) {
        const int32_t a = g->col_idx[i], b = g->col_idx[j];
        if (a < b) ++i;
        else if (b < a) ++j;
        else {
            if (!(gone && (gone[g->edge_id[i]] || gone[g->edge_id[j]])) && deg[a] > 0)
                score += 1.0 / (double)deg[a];
            ++i; ++j;
        }
    }
    return score;
}

double orc_ra_score(const orc_graph* g, int32_t u, int32_t v) {
    int32_t* deg = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->n + 1));
    for (int32_t x = 0; x < g->n; ++x) deg[x] = g->row_ptr[x + 1] - g->row_ptr[x];
    const double s = ra_on(g, NULL, deg, u, v);
    free(deg);
    return s;
}

static int cmp_f64(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* link_prediction.cpp:87-96.  The T x P grid adds 1.0 / 0.5 per pair; all
 * partial sums are multiples of 0.5 below 2^52, hence exact, so counting
 * 2*wins with a sort + two binary searches gives the identical double. */
static double auc_of(const double* test, int32_t T, double* probe_sorted, int32_t P) {
    qsort(probe_sorted, (size_t)P, sizeof(double), cmp_f64);
    int64_t twice = 0;
    for (int32_t t = 0; t < T; ++t) {
        int32_t lo = 0, hi = P; /* first index with probe >= test[t] */
        while (lo < hi) { int32_t mid = (lo + hi) / 2; if (probe_sorted[mid] < test[t]) lo = mid + 1; else hi = mid; }
        const int32_t below = lo;
        hi = P; /* first index with probe > test[t] */
        while (lo < hi) { int32_t mid = (lo + hi) / 2; if (probe_sorted[mid] <= test[t]) lo = mid + 1; else hi = mid; }
        twice += 2 * (int64_t)below + (lo - below);
    }
    const double wins = (double)twice / 2.0;
    return wins / ((double)T * (double)P);
}

/* fitness.cpp:43-48 */
int orc_lpa_batch(const orc_split* s, const int32_t* genes, int rows, int cols, double* out) {
    const orc_graph* g = s->train;
    uint8_t* gone = (uint8_t*)malloc((size_t)g->m + 1);
    int32_t* deg = (int32_t*)malloc(sizeof(int32_t) * ((size_t)g->n + 1));
    double* ts = (double*)malloc(sizeof(double) * ((size_t)s->T + 1));
    double* ps = (double*)malloc(sizeof(double) * ((size_t)s->P + 1));
    int rc = 0;
    for (int r = 0; r < rows && !rc; ++r) {
        memset(gone, 0, (size_t)g->m + 1);
        for (int32_t x = 0; x < g->n; ++x) deg[x] = g->row_ptr[x + 1] - g->row_ptr[x];
        for (int j = 0; j < cols; ++j) {
            const int32_t e = genes[(size_t)r * cols + j];
            if (e < 0 || e >= g->m) { rc = 1; break; }
            if (!gone[e]) { gone[e] = 1; deg[g->pool_u[e]]--; deg[g->pool_v[e]]--; }
        }
        if (rc) break;
        for (int32_t t = 0; t < s->T; ++t) ts[t] = ra_on(g, gone, deg, s->test_uv[2 * t], s->test_uv[2 * t + 1]);
        for (int32_t p = 0; p < s->P; ++p) ps[p] = ra_on(g, gone, deg, s->probe_uv[2 * p], s->probe_uv[2 * p + 1]);
        out[r] = auc_of(ts, s->T, ps, s->P);
    }
    free(gone); free(deg); free(ts); free(ps);
    return rc;
}

/* ---- north_star extensions WITHOUT a reference implementation (PARITY UNPINNED) ----------------------------
 * BASELINE.json's north_star names "CN/RA link scores" and "edge flips" for the link-prediction attack; the reference
 * has only the RA score with edge-removal pools (link_prediction.cpp:55-69, fitness.cpp:87).  These twins state the
 * semantics the CUDA path implements, by generalising the reference's own definitions:
 *   CN score   = |N'(u) & N'(v)| on the perturbed train graph (the RA sum with every term 1 instead of 1/deg'(z));
 *   flip gene  = a node pair (a < b): an edge of the train graph is removed, a non-edge is added, relative to the
 *                UNPERTURBED graph, so a repeated gene is idempotent like the reference's set / clear
 *                (gene_pool.cpp:49-67).  The canonical flip pool enumerates every pair a < b in lexicographic order
 *                (the order gene_pool.cpp:81-87 uses for non-edges): gene id = a n - a (a + 1) / 2 + (b - a - 1).
 * AUC exactly as link_prediction.cpp:82-96.  Nothing here is checked against reference outputs — there are none. */
void orc_flip_unrank(int32_t n, int64_t id, int32_t* a_out, int32_t* b_out) {
    int64_t a = 0;
    /* largest a with first(a) = a n - a (a + 1) / 2 <= id */
    int64_t lo = 0, hi = n - 2;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (mid * n - mid * (mid + 1) / 2 <= id) lo = mid; else hi = mid - 1;
    }
    a = lo;
    *a_out = (int32_t)a;
    *b_out = (int32_t)(id - (a * n - a * (a + 1) / 2) + a + 1);
}

static int base_has_edge(const orc_graph* g, int32_t a, int32_t b) {
    int32_t lo = g->row_ptr[a], hi = g->row_ptr[a + 1];
    while (lo < hi) { const int32_t mid = (lo + hi) / 2; if (g->col_idx[mid] < b) lo = mid + 1; else hi = mid; }
    return lo < g->row_ptr[a + 1] && g->col_idx[lo] == b;
}

/* score_kind 0 = RA, 1 = CN.  pool_uv == NULL: the canonical all-pairs pool; else pool_size pairs. */
int orc_lpa_flip_batch(const orc_split* s, int score_kind, const int32_t* pool_uv, int64_t pool_size, const int32_t* genes,
                       int rows, int cols, double* out) {
    const orc_graph* g = s->train;
    const int32_t n = g->n;
    if (!pool_uv) pool_size = (int64_t)n * (n - 1) / 2;
    int32_t** nb = (int32_t**)calloc((size_t)n + 1, sizeof(int32_t*));
    int32_t* len = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* cap = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    double* ts = (double*)malloc(sizeof(double) * ((size_t)s->T + 1));
    double* ps = (double*)malloc(sizeof(double) * ((size_t)s->P + 1));
    int rc = 0;
    for (int r = 0; r < rows && !rc; ++r) {
        for (int32_t x = 0; x < n; ++x) {
            len[x] = g->row_ptr[x + 1] - g->row_ptr[x];
            cap[x] = len[x] + 4;
            nb[x] = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap[x]);
            memcpy(nb[x], g->col_idx + g->row_ptr[x], sizeof(int32_t) * (size_t)len[x]);
        }
        for (int j = 0; j < cols && !rc; ++j) {
            const int64_t id = genes[(size_t)r * cols + j];
            if (id < 0 || id >= pool_size) { rc = 1; break; }
            int32_t a, b;
            if (pool_uv) { a = pool_uv[2 * id]; b = pool_uv[2 * id + 1]; if (a > b) { const int32_t t = a; a = b; b = t; } }
            else orc_flip_unrank(n, id, &a, &b);
            const int want = !base_has_edge(g, a, b); /* the state the flip leaves the pair in */
            for (int side = 0; side < 2; ++side) {
                const int32_t x = side ? b : a, y = side ? a : b;
                int32_t pos = -1;
                for (int32_t t = 0; t < len[x]; ++t) if (nb[x][t] == y) { pos = t; break; }
                if (want && pos < 0) {
                    if (len[x] == cap[x]) { cap[x] *= 2; nb[x] = (int32_t*)realloc(nb[x], sizeof(int32_t) * (size_t)cap[x]); }
                    nb[x][len[x]++] = y;
                } else if (!want && pos >= 0) {
                    nb[x][pos] = nb[x][--len[x]];
                }
            }
        }
        if (!rc) {
            for (int32_t x = 0; x < n; ++x) qsort(nb[x], (size_t)len[x], sizeof(int32_t), cmp_i32);
            for (int32_t q = 0; q < s->T + s->P; ++q) {
                const int32_t* uv = q < s->T ? s->test_uv + 2 * q : s->probe_uv + 2 * (q - s->T);
                const int32_t u = uv[0], v = uv[1];
                int32_t i = 0, jj = 0;
                double score = 0.0;
                while (i < len[u] && jj < len[v]) { /* common neighbours in ascending z (link_prediction.cpp:59-66) */
                    const int32_t za = nb[u][i], zb = nb[v][jj];
                    if (za < zb) ++i;
                    else if (zb < za) ++jj;
                    else { if (len[za] > 0) score += score_kind ? 1.0 : 1.0 / (double)len[za]; ++i; ++jj; }
                }
                if (q < s->T) ts[q] = score; else ps[q - s->T] = score;
            }
            out[r] = auc_of(ts, s->T, ps, s->P);
        }
        for (int32_t x = 0; x < n; ++x) free(nb[x]);
    }
    free(nb); free(len); free(cap); free(ts); free(ps);
    return rc;
}

/* CN / RA with the reference's edge-REMOVAL pools (genes = edge ranks, as orc_lpa_batch) */
int orc_lpa_scored_batch(const orc_split* s, int score_kind, const int32_t* genes, int rows, int cols, double* out) {
    const orc_graph* g = s->train;
    int32_t* uv = (int32_t*)malloc(sizeof(int32_t) * 2 * ((size_t)g->m + 1));
    for (int64_t e = 0; e < g->m; ++e) { uv[2 * e] = g->pool_u[e]; uv[2 * e + 1] = g->pool_v[e]; }
    const int rc = orc_lpa_flip_batch(s, score_kind, uv, g->m, genes, rows, cols, out); /* flipping an edge removes it */
    free(uv);
    return rc;
}

/* ============================================================ batch + threads */

void orc_partition_rows(int pop_size, int pn, int32_t* lo_hi) { /* modes.cpp:506-516 */
    const int block = (pop_size + pn - 1) / pn;
    for (int w = 0; w < pn; ++w) {
        int lo = w * block; if (lo > pop_size) lo = pop_size;
        int hi = lo + block; if (hi > pop_size) hi = pop_size;
        lo_hi[2 * w] = lo; lo_hi[2 * w + 1] = hi;
    }
}

static int eval_block(const void* ctx, int task, const int32_t* genes, int rows, int cols, double* out) {
    switch (task) {
        case ORC_TASK_PC:
        case ORC_TASK_MCN: return orc_pc_batch((const orc_graph*)ctx, task, genes, rows, cols, out);
        case ORC_TASK_CDA: return orc_cda_batch((const orc_graph*)ctx, genes, rows, cols, out);
        case ORC_TASK_LPA: return orc_lpa_batch((const orc_split*)ctx, genes, rows, cols, out);
        case ORC_TASK_SIXDST: return orc_sixdst_batch((const orc_graph*)ctx, genes, rows, cols, out);
        case ORC_TASK_CDA_ADD: return orc_cda_add_batch((const orc_graph*)ctx, genes, rows, cols, out);
    }
    return 2;
}

typedef struct { const void* ctx; int task; const int32_t* genes; int rows, cols; double* out; int rc; } job_t;
static void* job_main(void* p) {
    job_t* j = (job_t*)p;
    j->rc = eval_block(j->ctx, j->task, j->genes, j->rows, j->cols, j->out);
    return NULL;
}

int orc_eval_batch(const void* ctx, int task, const int32_t* genes, int rows, int cols, int threads, double* out) {
    if (threads <= 1 || rows <= 1) return eval_block(ctx, task, genes, rows, cols, out);
    if (threads > rows) threads = rows;
    int32_t* blocks = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)threads);
    orc_partition_rows(rows, threads, blocks);
    job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int w = 0; w < threads; ++w) {
        jobs[w] = (job_t){ctx, task, genes + (size_t)blocks[2 * w] * cols, blocks[2 * w + 1] - blocks[2 * w], cols,
                          out + blocks[2 * w], 0};
        pthread_create(&tid[w], NULL, job_main, &jobs[w]);
    }
    int rc = 0;
    for (int w = 0; w < threads; ++w) { pthread_join(tid[w], NULL); rc |= jobs[w].rc; }
    free(blocks); free(jobs); free(tid);
    return rc;
}

/* ========================================================= genetic operators */

/* ga_ops.cpp:19-29 */
int orc_init_population_block(int pool_size, int row_first, int row_count, int budget,
                              uint64_t seed, uint64_t generation, int32_t* out) {
    if (pool_size < 1) return 1;
    for (int i = 0; i < row_count; ++i) {
        const uint64_t key = orc_stream_key(seed, generation, ORC_ROLE_INIT, (uint64_t)(row_first + i));
        for (int j = 0; j < budget; ++j)
            out[(size_t)i * budget + j] = (int32_t)orc_draw_index(key, (uint64_t)j + 1, (uint32_t)pool_size);
    }
    return 0;
}

/* make_mask (ga_ops.cpp:38-47) behind make_crossover_mask / make_mutation_mask (:84-92): role 3 or 4 */
void orc_make_mask(int rows, int cols, double rate, int role, uint64_t seed, uint64_t generation, uint8_t* out) {
    for (int i = 0; i < rows; ++i) {
        const uint64_t key = orc_stream_key(seed, generation, (uint64_t)role, (uint64_t)i);
        for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = orc_draw_unit(key, (uint64_t)j + 1) < rate ? 1 : 0; /* rng.hpp:33 */
    }
}

/* make_mutation_indices (ga_ops.cpp:94-103) */
void orc_make_mutation_indices(int rows, int cols, int pool_size, uint64_t seed, uint64_t generation, int32_t* out) {
    for (int i = 0; i < rows; ++i) {
        const uint64_t key = orc_stream_key(seed, generation, ORC_ROLE_MUTATION_INDEX, (uint64_t)i);
        for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = (int32_t)orc_draw_index(key, (uint64_t)j + 1, (uint32_t)pool_size);
    }
}

/* stable merge sort of indices; better(a, b) is the strict "a before b" */
typedef struct { const double* f0; const double* f1; int s; int minimize; } keyctx;
static double key_of(const keyctx* c, int idx) { return idx < c->s ? c->f0[idx] : c->f1[idx - c->s]; }
static int before(const keyctx* c, int a, int b) {
    const double x = key_of(c, a), y = key_of(c, b);
    return c->minimize ? x < y : x > y;
}
static void stable_sort_idx(int32_t* idx, int32_t* tmp, int n, const keyctx* c) {
    if (n < 2) return;
    const int h = n / 2;
    stable_sort_idx(idx, tmp, h, c);
    stable_sort_idx(idx + h, tmp, n - h, c);
    int i = 0, j = h, o = 0;
    while (i < h && j < n) tmp[o++] = before(c, idx[j], idx[i]) ? idx[j++] : idx[i++];
    while (i < h) tmp[o++] = idx[i++];
    while (j < n) tmp[o++] = idx[j++];
    memcpy(idx, tmp, sizeof(int32_t) * (size_t)n);
}

/* ga_ops.cpp:54-76 */
int orc_selection_weights(const double* fitness, int s, int minimize, double* out) {
    for (int i = 0; i < s; ++i) if (!isfinite(fitness[i])) return 1;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s + 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s + 1));
    for (int i = 0; i < s; ++i) order[i] = i;
    const keyctx c = {fitness, NULL, s, minimize};
    stable_sort_idx(order, tmp, s, &c);
    int i = 0;
    while (i < s) {
        int j = i + 1;
        while (j < s && fitness[order[j]] == fitness[order[i]]) ++j;
        const double w = ((double)(s - i) + (double)(s - j + 1)) / 2.0;
        for (int r = i; r < j; ++r) out[order[r]] = w;
        i = j;
    }
    free(order); free(tmp);
    return 0;
}

/* ga_ops.cpp:105-126 (index form) with weighted_pick :78-82 */
int orc_roulette_pick(const double* fitness, int s, int minimize, uint64_t seed,
                      uint64_t generation, int32_t* partner_index) {
    double* cumulative = (double*)malloc(sizeof(double) * (size_t)(s + 1));
    if (orc_selection_weights(fitness, s, minimize, cumulative)) { free(cumulative); return 1; }
    double total = 0.0;
    for (int i = 0; i < s; ++i) { total += cumulative[i]; cumulative[i] = total; }
    for (int i = 0; i < s; ++i) {
        const double target = orc_draw_unit(orc_stream_key(seed, generation, ORC_ROLE_SELECT, (uint64_t)i), 1) * total;
        int lo = 0, hi = s; /* upper_bound */
        while (lo < hi) { int mid = (lo + hi) / 2; if (cumulative[mid] <= target) lo = mid + 1; else hi = mid; }
        partner_index[i] = lo < s - 1 ? lo : s - 1;
    }
    free(cumulative);
    return 0;
}

/* ga_ops.cpp:38-47,130-144 */
void orc_crossover(const int32_t* pop, const int32_t* partner_index, int s, int k, double pc,
                   uint64_t seed, uint64_t generation, int32_t* out) {
    for (int i = 0; i < s; ++i) {
        const uint64_t key = orc_stream_key(seed, generation, ORC_ROLE_CROSSOVER_MASK, (uint64_t)i);
        const int32_t* mine = pop + (size_t)i * k;
        const int32_t* theirs = pop + (size_t)partner_index[i] * k;
        for (int j = 0; j < k; ++j)
            out[(size_t)i * k + j] = orc_draw_unit(key, (uint64_t)j + 1) < pc ? theirs[j] : mine[j];
    }
}

/* ga_ops.cpp:164-178 */
void orc_mutate_block(const int32_t* block, int rows, int k, int row_offset, double pm,
                      int pool_size, uint64_t seed, uint64_t generation, int32_t* out) {
    for (int i = 0; i < rows; ++i) {
        const uint64_t mk = orc_stream_key(seed, generation, ORC_ROLE_MUTATION_MASK, (uint64_t)(row_offset + i));
        const uint64_t ik = orc_stream_key(seed, generation, ORC_ROLE_MUTATION_INDEX, (uint64_t)(row_offset + i));
        for (int j = 0; j < k; ++j) {
            const int flip = orc_draw_unit(mk, (uint64_t)j + 1) < pm;
            const int32_t fresh = (int32_t)orc_draw_index(ik, (uint64_t)j + 1, (uint32_t)pool_size);
            out[(size_t)i * k + j] = flip ? fresh : block[(size_t)i * k + j];
        }
    }
}

/* ga_ops.cpp:180-212 */
int orc_elitism(const int32_t* pop, const int32_t* m_pop, int s, int k, const double* fit_pop,
                const double* fit_m, int minimize, int32_t* next, double* next_fit) {
    for (int i = 0; i < s; ++i) if (isnan(fit_pop[i]) || isnan(fit_m[i])) return 1;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * s + 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * s + 1));
    for (int i = 0; i < 2 * s; ++i) order[i] = i;
    const keyctx c = {fit_pop, fit_m, s, minimize};
    stable_sort_idx(order, tmp, 2 * s, &c);
    for (int i = 0; i < s; ++i) {
        const int idx = order[i];
        const int32_t* src = idx < s ? pop + (size_t)idx * k : m_pop + (size_t)(idx - s) * k;
        memcpy(next + (size_t)i * k, src, sizeof(int32_t) * (size_t)k);
        next_fit[i] = key_of(&c, idx);
    }
    free(order); free(tmp);
    return 0;
}

/* ga_ops.cpp:214-238 */
int orc_eda_sample(const int32_t* elite, int s, int k, int elite_count, int pool_size,
                   uint64_t seed, uint64_t generation, int smoothing, int32_t* out) {
    if (elite_count < 1 || elite_count > s) return 1;
    const uint32_t bound = (uint32_t)(smoothing ? elite_count + pool_size : elite_count);
    for (int i = 0; i < s; ++i) {
        const uint64_t key = orc_stream_key(seed, generation, ORC_ROLE_SELECT, (uint64_t)i);
        for (int j = 0; j < k; ++j) {
            const uint32_t v = orc_draw_index(key, (uint64_t)j + 1, bound);
            out[(size_t)i * k + j] = v < (uint32_t)elite_count ? elite[(size_t)v * k + j] : (int32_t)(v - (uint32_t)elite_count);
        }
    }
    return 0;
}

/* ============================================================ generation loop */

static int pool_size_of(const void* ctx, int task) {
    switch (task) {
        case ORC_TASK_PC:
        case ORC_TASK_MCN:
        case ORC_TASK_SIXDST: return ((const orc_graph*)ctx)->n;
        case ORC_TASK_CDA: return (int)((const orc_graph*)ctx)->m;
        case ORC_TASK_CDA_ADD: return (int)((const orc_graph*)ctx)->add_size;
        case ORC_TASK_LPA: return (int)((const orc_split*)ctx)->train->m;
    }
    return 0;
}

/* modes.cpp:132-178 (batch form; identical to run_serial :359-418).
 * history mean is the sequential sum / s of record_generation (:35-43). */
int orc_run_ga(const void* ctx, int task, double pc, double pm, int pop_size, int budget,
               int iterations, int eda_interval, uint64_t seed, int minimize, int threads,
               double* history_best, double* history_mean, int32_t* final_population,
               double* final_fitness) {
    const int s = pop_size, k = budget, pool = pool_size_of(ctx, task);
    if (s < 2 || k < 1 || iterations < 1 || pc < 0 || pc > 1 || pm < 0 || pm > 1) return 2;
    const size_t cells = (size_t)s * k;
    int32_t* pop = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* crossed = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* mutated = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* next = (int32_t*)malloc(sizeof(int32_t) * cells);
    int32_t* partner = (int32_t*)malloc(sizeof(int32_t) * (size_t)s);
    double* fit = (double*)malloc(sizeof(double) * (size_t)s);
    double* fit_m = (double*)malloc(sizeof(double) * (size_t)s);
    double* fit_n = (double*)malloc(sizeof(double) * (size_t)s);
    int rc = 0;
    for (int gen = 1; gen <= iterations && !rc; ++gen) {
        if (gen == 1) {
            rc = orc_init_population_block(pool, 0, s, k, seed, 0, pop);
            if (!rc) rc = orc_eval_batch(ctx, task, pop, s, k, threads, fit);
            if (rc) break;
        }
        if (eda_interval > 0 && gen % eda_interval == 0) {
            rc = orc_eda_sample(pop, s, k, s, pool, seed, (uint64_t)gen, 1, crossed);
        } else {
            rc = orc_roulette_pick(fit, s, minimize, seed, (uint64_t)gen, partner);
            if (!rc) orc_crossover(pop, partner, s, k, pc, seed, (uint64_t)gen, crossed);
        }
        if (rc) break;
        orc_mutate_block(crossed, s, k, 0, pm, pool, seed, (uint64_t)gen, mutated);
        rc = orc_eval_batch(ctx, task, mutated, s, k, threads, fit_m);
        if (rc) break;
        rc = orc_elitism(pop, mutated, s, k, fit, fit_m, minimize, next, fit_n);
        if (rc) break;
        memcpy(pop, next, sizeof(int32_t) * cells);
        memcpy(fit, fit_n, sizeof(double) * (size_t)s);
        double sum = 0.0;
        for (int i = 0; i < s; ++i) sum += fit[i];
        history_best[gen - 1] = fit[0];
        history_mean[gen - 1] = sum / (double)s;
    }
    if (!rc) {
        memcpy(final_population, pop, sizeof(int32_t) * cells);
        memcpy(final_fitness, fit, sizeof(double) * (size_t)s);
    }
    free(pop); free(crossed); free(mutated); free(next); free(partner); free(fit); free(fit_m); free(fit_n);
    return rc;
}
