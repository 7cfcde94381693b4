/*
 * oracle_csr.c -- at-size parity checker: the reference's phase decisions
 * (mhskernel/parallel.py:80-214) with the pair counts taken from the CSR
 * instead of bitset ANDs.
 *
 * TEST INFRASTRUCTURE ONLY (see mhsk_oracle.c's header): loaded by tests/
 * and nowhere on the product path.
 *
 * The bitset restatement in mhsk_oracle.c is the reference's own algorithm
 * (one AND + popcount per ordered pair, parallel.py:105,141).  At the
 * BASELINE's configs 4/5 that is 1e10-4e10 pairs x 1.6k-3.1k words per
 * phase.  Here c(i, j) is counted sparsely instead: for an edge j, one pass
 * over the incidence lists of its alive vertices adds 1 to every alive edge
 * sharing a vertex with it (sum over v in e_j of deg(v) ~ 1e6 increments at
 * config 4, against 1e5 x 1563 word ANDs); for a vertex j, one pass over its
 * alive edges' members.  The decision predicates are the reference's,
 * literally:
 *
 *   edge phase (parallel.py:103-114), on the alive sub-instance:
 *     DP  R(i,j) <=> f_i - (s_i - c) >= f_j
 *     SE  R(i,j) <=> c == s_i && f_i >= f_j
 *     j deleted <=> exists alive i != j: R(i,j) && (!R(j,i) || i < j)
 *   vertex phase (parallel.py:136-159):
 *     need_j = max demand over j's alive edges; need_j == 0 => deleted
 *     D(i,j) <=> c == d_j && (c != d_i || i < j)
 *     j deleted <=> #{alive i != j : D(i,j)} >= need_j
 *
 * Pairs with c = 0 never touch a counter; they can only relate in the edge
 * phase through an edge i with f_i - s_i >= 1 (DP) or s_i == 0 (SE), so
 * those edges are listed up front and evaluated with c = 0 for every j
 * (they do not exist in feasible instances, but extract() keeps edges whose
 * vertices all died, rules.py:88-103).  In the vertex phase an alive vertex
 * with d_j > 0 needs c = d_j > 0; d_j == 0 means need_j == 0.
 *
 * Compaction preserves order (rules.py:94-103), so "i < j" on compacted
 * positions is "i < j" on original ids: the functions work on the original
 * ids with alive masks and never renumber.
 *
 * Pinned by tests/test_oracle.py: equal to the bitset oracle and to the
 * reference's golden outputs (tests/golden/) on every fixture.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_INFEASIBLE 1
#define ORC_INVALID 2
#define ORC_NOMEM 4

typedef struct {
    int32_t n, m;
    const int64_t *ptr;
    const int32_t *vtx;
    const int32_t *dem;
    const uint8_t *va, *ea;   /* alive masks (all-ones arrays when the caller passed NULL) */
    int64_t *cptr;            /* CSC: vertex -> edges, in increasing edge id */
    int32_t *cidx;
    int32_t *size;            /* alive members of each alive edge */
    int32_t *deg;             /* alive edges of each alive vertex */
    int32_t *need;            /* max demand over a vertex's alive edges */
    int32_t *special;         /* alive edges that relate at c = 0 */
    int64_t nspecial;
} csr_t;

static int csr_check(int32_t n, int32_t m, const int64_t *ptr, const int32_t *vtx,
                     const int32_t *dem) {
    if (n < 0 || m < 0) return ORC_INVALID;
    if (m > 0 && (!ptr || !dem || ptr[0] != 0)) return ORC_INVALID;
    for (int32_t e = 0; e < m; ++e) {
        if (ptr[e + 1] < ptr[e]) return ORC_INVALID;
        for (int64_t k = ptr[e]; k < ptr[e + 1]; ++k) {
            if (vtx[k] < 0 || vtx[k] >= n) return ORC_INVALID;
            if (k > ptr[e] && vtx[k] <= vtx[k - 1]) return ORC_INVALID;
        }
    }
    return ORC_OK;
}

static void csr_free(csr_t *c) {
    free(c->cptr); free(c->cidx); free(c->size); free(c->deg); free(c->need); free(c->special);
    memset(c, 0, sizeof(*c));
}

/* CSC of the whole instance (dead entries are skipped at use). */
static int csr_build(csr_t *c) {
    const int32_t n = c->n, m = c->m;
    const int64_t nnz = m ? c->ptr[m] : 0;
    c->cptr = (int64_t *)calloc((size_t)n + 2, sizeof(int64_t));
    c->cidx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz + 1));
    c->size = (int32_t *)calloc((size_t)m + 1, sizeof(int32_t));
    c->deg = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    c->need = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    c->special = (int32_t *)malloc(sizeof(int32_t) * ((size_t)m + 1));
    if (!c->cptr || !c->cidx || !c->size || !c->deg || !c->need || !c->special) return ORC_NOMEM;
    for (int64_t k = 0; k < nnz; ++k) c->cptr[c->vtx[k] + 1]++;
    for (int32_t v = 0; v < n; ++v) c->cptr[v + 1] += c->cptr[v];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!fill) return ORC_NOMEM;
    memcpy(fill, c->cptr, sizeof(int64_t) * (size_t)n);
    for (int32_t e = 0; e < m; ++e)
        for (int64_t k = c->ptr[e]; k < c->ptr[e + 1]; ++k) c->cidx[fill[c->vtx[k]]++] = e;
    free(fill);
    return ORC_OK;
}

/* Alive sizes, degrees, need and the c = 0 list for the current masks. */
static void csr_refresh(csr_t *c) {
    const int32_t n = c->n, m = c->m;
    memset(c->deg, 0, sizeof(int32_t) * (size_t)n);
    memset(c->need, 0, sizeof(int32_t) * (size_t)n);
    c->nspecial = 0;
    for (int32_t e = 0; e < m; ++e) {
        int32_t s = 0;
        if (c->ea[e]) {
            for (int64_t k = c->ptr[e]; k < c->ptr[e + 1]; ++k) {
                const int32_t v = c->vtx[k];
                if (!c->va[v]) continue;
                ++s;
                c->deg[v]++;
                if (c->dem[e] > c->need[v]) c->need[v] = c->dem[e];
            }
            if (c->dem[e] - s >= 1 || s == 0) c->special[c->nspecial++] = e;
        }
        c->size[e] = s;
    }
}

/* Per-thread scratch: one counter per item and the list of touched ones. */
typedef struct {
    int32_t *cnt, *touched;
} scratch_t;

/* DP / SE relation R(i, j) of parallel.py:103-108. */
static inline int relates(int32_t rule, int64_t c, int64_t fi, int64_t si, int64_t fj) {
    if (rule == 0) return fi - (si - c) >= fj;
    return c == si && fi >= fj;
}

/* Edge j of the alive sub-instance: 1 keeps it (parallel.py:110-114). */
static int edge_keep(const csr_t *c, int32_t rule, int32_t j, scratch_t *s) {
    int64_t nt = 0;
    for (int64_t k = c->ptr[j]; k < c->ptr[j + 1]; ++k) {
        const int32_t v = c->vtx[k];
        if (!c->va[v]) continue;
        for (int64_t t = c->cptr[v]; t < c->cptr[v + 1]; ++t) {
            const int32_t i = c->cidx[t];
            if (i == j || !c->ea[i]) continue;
            if (s->cnt[i]++ == 0) s->touched[nt++] = i;
        }
    }
    const int64_t fj = c->dem[j], sj = c->size[j];
    int keep = 1;
    for (int64_t t = 0; t < nt && keep; ++t) {
        const int32_t i = s->touched[t];
        const int64_t cij = s->cnt[i];
        if (relates(rule, cij, c->dem[i], c->size[i], fj) &&
            (!relates(rule, cij, fj, sj, c->dem[i]) || i < j))
            keep = 0;
    }
    for (int64_t t = 0; t < c->nspecial && keep; ++t) {
        const int32_t i = c->special[t];
        if (i == j || s->cnt[i]) continue;   /* touched pairs were evaluated above */
        if (relates(rule, 0, c->dem[i], c->size[i], fj) && (!relates(rule, 0, fj, sj, c->dem[i]) || i < j))
            keep = 0;
    }
    for (int64_t t = 0; t < nt; ++t) s->cnt[s->touched[t]] = 0;
    return keep;
}

/* Vertex j of the alive sub-instance: 1 keeps it (parallel.py:145-159). */
static int vertex_keep(const csr_t *c, int32_t j, scratch_t *s) {
    const int32_t need = c->need[j];
    if (need == 0) return 0;
    int64_t nt = 0;
    for (int64_t t = c->cptr[j]; t < c->cptr[j + 1]; ++t) {
        const int32_t e = c->cidx[t];
        if (!c->ea[e]) continue;
        for (int64_t k = c->ptr[e]; k < c->ptr[e + 1]; ++k) {
            const int32_t i = c->vtx[k];
            if (i == j || !c->va[i]) continue;
            if (s->cnt[i]++ == 0) s->touched[nt++] = i;
        }
    }
    const int32_t dj = c->deg[j];
    int64_t count = 0;
    int keep = 1;
    for (int64_t t = 0; t < nt && keep; ++t) {
        const int32_t i = s->touched[t];
        const int32_t cij = s->cnt[i];
        if (cij == dj && (cij != c->deg[i] || i < j) && ++count >= need) keep = 0;
    }
    for (int64_t t = 0; t < nt; ++t) s->cnt[s->touched[t]] = 0;
    return keep;
}

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* Decide `count` items of one phase (which: 0 edges, 1 vertices), in
 * parallel; items[] are original 0-based ids, alive under the masks (a dead
 * item is reported kept). */
static int decide(const csr_t *c, int32_t which, int32_t rule, const int32_t *items, int64_t count,
                  uint8_t *keep_out) {
    const int64_t width = which == 0 ? c->m : c->n;
    int rc = ORC_OK;
#pragma omp parallel
    {
        scratch_t s;
        s.cnt = (int32_t *)calloc((size_t)width + 1, sizeof(int32_t));
        s.touched = (int32_t *)malloc(sizeof(int32_t) * ((size_t)width + 1));
        if (!s.cnt || !s.touched) {
#pragma omp atomic write
            rc = ORC_NOMEM;
        } else {
#pragma omp for schedule(dynamic, 8)
            for (int64_t t = 0; t < count; ++t) {
                const int32_t j = items[t];
                if (which == 0)
                    keep_out[t] = c->ea[j] ? (uint8_t)edge_keep(c, rule, j, &s) : 1;
                else
                    keep_out[t] = c->va[j] ? (uint8_t)vertex_keep(c, j, &s) : 1;
            }
        }
        free(s.cnt);
        free(s.touched);
    }
    return rc;
}

/* A persistent handle: the CSC is built once per instance, each decide call
 * only refreshes sizes / degrees / need for its masks. */
typedef struct {
    csr_t c;
    uint8_t *ones;
} oracle_csr_handle;

void oracle_csr_free(oracle_csr_handle *h) {
    if (!h) return;
    csr_free(&h->c);
    free(h->ones);
    free(h);
}

/* NULL on invalid input or allocation failure.  The arrays must outlive the
 * handle. */
oracle_csr_handle *oracle_csr_new(int32_t n, int32_t m, const int64_t *edge_ptr,
                                  const int32_t *edge_vtx, const int32_t *demand) {
    if (csr_check(n, m, edge_ptr, edge_vtx, demand)) return NULL;
    oracle_csr_handle *h = (oracle_csr_handle *)calloc(1, sizeof(*h));
    if (!h) return NULL;
    const size_t most = (size_t)(n > m ? n : m) + 1;
    h->ones = (uint8_t *)malloc(most);
    if (!h->ones) { free(h); return NULL; }
    memset(h->ones, 1, most);
    csr_t c = {n, m, edge_ptr, edge_vtx, demand, h->ones, h->ones, 0, 0, 0, 0, 0, 0, 0};
    h->c = c;
    if (csr_build(&h->c)) { oracle_csr_free(h); return NULL; }
    return h;
}

/* Phase decisions for arbitrary items at full width.
 *   which: 0 = edge phase (rule 0 dp / 1 se), 1 = vertex phase
 *   valive[n], ealive[m]: the alive sub-instance (NULL = all alive), i.e.
 *     the state the reference's extract() compacts before the phase
 *   items[count]: original 0-based ids of alive items
 *   keep_out[count]: 1 keeps the item */
int oracle_csr_decide_h(oracle_csr_handle *h, const uint8_t *valive, const uint8_t *ealive,
                        int32_t which, int32_t rule, const int32_t *items, int64_t count,
                        int32_t threads, uint8_t *keep_out) {
    if (!h || (which != 0 && which != 1) || (rule != 0 && rule != 1) || count < 0) return ORC_INVALID;
    csr_t *c = &h->c;
    for (int64_t t = 0; t < count; ++t)
        if (items[t] < 0 || items[t] >= (which == 0 ? c->m : c->n)) return ORC_INVALID;
    set_threads(threads);
    c->va = valive ? valive : h->ones;
    c->ea = ealive ? ealive : h->ones;
    csr_refresh(c);
    const int rc = decide(c, which, rule, items, count, keep_out);
    c->va = c->ea = h->ones;
    return rc;
}

/* One-shot form of the above. */
int oracle_csr_decide(int32_t n, int32_t m, const int64_t *edge_ptr, const int32_t *edge_vtx,
                      const int32_t *demand, const uint8_t *valive, const uint8_t *ealive,
                      int32_t which, int32_t rule, const int32_t *items, int64_t count,
                      int32_t threads, uint8_t *keep_out) {
    if ((which != 0 && which != 1) || (rule != 0 && rule != 1) || count < 0) return ORC_INVALID;
    oracle_csr_handle *h = oracle_csr_new(n, m, edge_ptr, edge_vtx, demand);
    if (!h) return csr_check(n, m, edge_ptr, edge_vtx, demand) ? ORC_INVALID : ORC_NOMEM;
    const int rc = oracle_csr_decide_h(h, valive, ealive, which, rule, items, count, threads, keep_out);
    oracle_csr_free(h);
    return rc;
}

/* Full fixpoint (par_kernelize, parallel.py:164-214) with CSR-counted
 * phases.  vertex_alive / edge_alive are in/out (all-ones for a fresh run).
 * stats_out[0] rounds, [1] edge deletions, [2] md deletions.  If
 * round_log != NULL, round_log[r] receives the round in which item r was
 * deleted (edges: m entries, then vertices: n entries; 0 = survived). */
int oracle_csr_kernelize(int32_t n, int32_t m, const int64_t *edge_ptr, const int32_t *edge_vtx,
                         const int32_t *demand, int32_t rule, int32_t max_rounds, int32_t threads,
                         uint8_t *vertex_alive, uint8_t *edge_alive, int64_t *stats_out,
                         int32_t *round_log) {
    if (rule != 0 && rule != 1) return ORC_INVALID;
    int rc = csr_check(n, m, edge_ptr, edge_vtx, demand);
    if (rc) return rc;
    for (int32_t e = 0; e < m; ++e)  /* validate_feasibility, instance.py:199-212 */
        if (demand[e] > edge_ptr[e + 1] - edge_ptr[e]) return ORC_INFEASIBLE;
    set_threads(threads);
    csr_t c = {n, m, edge_ptr, edge_vtx, demand, vertex_alive, edge_alive, 0, 0, 0, 0, 0, 0, 0};
    const int64_t most = n > m ? n : m;
    int32_t *items = (int32_t *)malloc(sizeof(int32_t) * ((size_t)most + 1));
    uint8_t *keep = (uint8_t *)malloc((size_t)most + 1);
    if (!items || !keep) { rc = ORC_NOMEM; goto out; }
    if ((rc = csr_build(&c))) goto out;
    if (round_log) memset(round_log, 0, sizeof(int32_t) * ((size_t)n + (size_t)m));
    int64_t rounds = 0, del_e = 0, del_v = 0;
    for (;;) {
        if (max_rounds >= 0 && rounds >= max_rounds) break;
        ++rounds;
        int changed = 0;
        int64_t cnt = 0;
        csr_refresh(&c);
        for (int32_t e = 0; e < m; ++e) if (edge_alive[e]) items[cnt++] = e;
        if ((rc = decide(&c, 0, rule, items, cnt, keep))) goto out;
        for (int64_t t = 0; t < cnt; ++t)
            if (!keep[t]) {
                edge_alive[items[t]] = 0;
                if (round_log) round_log[items[t]] = (int32_t)rounds;
                ++del_e; changed = 1;
            }
        cnt = 0;
        csr_refresh(&c);
        for (int32_t v = 0; v < n; ++v) if (vertex_alive[v]) items[cnt++] = v;
        if ((rc = decide(&c, 1, rule, items, cnt, keep))) goto out;
        for (int64_t t = 0; t < cnt; ++t)
            if (!keep[t]) {
                vertex_alive[items[t]] = 0;
                if (round_log) round_log[(int64_t)m + items[t]] = (int32_t)rounds;
                ++del_v; changed = 1;
            }
        if (!changed) break;
    }
    if (stats_out) { stats_out[0] = rounds; stats_out[1] = del_e; stats_out[2] = del_v; }
out:
    csr_free(&c);
    free(items);
    free(keep);
    return rc;
}
