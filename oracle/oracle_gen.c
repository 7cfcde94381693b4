/*
 * oracle_gen.c -- the counter-based random instance of configs 4/5 on the
 * host, for the CPU legs of bench.py (the reference arm must not load the
 * product library) and for tests.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY (see mhsk_oracle.c's header).
 *
 * Semantics of the reference generator (pkg/src/mhskernel/generate.py:18-46):
 * each (edge, vertex) incidence is an independent Bernoulli(p); an empty
 * edge is redrawn up to 20 times, then gets one random vertex; demand
 * min(alpha, |e|).  The draws are counter-based instead of a Mersenne-Twister
 * stream: draw r of cell (e, v) is (mix64(seed, e, v, r) >> 32) < p * 2^32,
 * the pad vertex mix64(seed, e, 2^32 - 1, 20) mod n.  This is the definition
 * of configs 4/5; tests/test_oracle.py checks it against the
 * numpy statement paper_2109_06042_b200/generate.py:counter_random and
 * tests/test_gpu_generate.py against the device generator.
 */
#include <stdint.h>
#include <stdlib.h>

#define RETRIES 20

static inline uint64_t mix64(uint64_t seed, uint64_t e, uint64_t v, uint64_t r) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull ^ e * 0xD1B54A32D192ED03ull ^ v * 0xC2B2AE3D27D4EB4Full ^
                 r * 0x165667B19E3779F9ull;
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

static inline int draw(uint64_t seed, int64_t e, int64_t v, int r, uint64_t thr) {
    return (mix64(seed, (uint64_t)e, (uint64_t)v, (uint64_t)r) >> 32) < thr;
}

/* Two passes.  With edge_vtx == NULL: fills edge_ptr[m+1] and attempt[m]
 * (the draw used; RETRIES = padded) and returns nnz.  Then with edge_vtx
 * (capacity >= nnz) and demand[m]: fills them.  -1 on bad arguments. */
int64_t oracle_generate_random(int32_t n, int32_t m, double p, int32_t alpha, uint64_t seed,
                               int64_t *edge_ptr, int32_t *edge_vtx, int64_t vtx_capacity,
                               int32_t *demand, int32_t *attempt) {
    if (n < 0 || m < 0 || !(p > 0.0 && p <= 1.0) || alpha < 1 || (m > 0 && n == 0) || !edge_ptr ||
        (m > 0 && !attempt))
        return -1;
    const double t = p * 4294967296.0;
    const uint64_t thr = t >= 4294967296.0 ? 4294967296ull : (uint64_t)t;
    if (!edge_vtx) {
        edge_ptr[0] = 0;
#pragma omp parallel for schedule(dynamic, 16)
        for (int32_t e = 0; e < m; ++e) {
            int r = 0;
            int64_t cnt = 0;
            for (; r < RETRIES; ++r) {
                cnt = 0;
                for (int32_t v = 0; v < n; ++v) cnt += draw(seed, e, v, r, thr);
                if (cnt) break;
            }
            edge_ptr[e + 1] = cnt ? cnt : 1;
            attempt[e] = r;
        }
        for (int32_t e = 0; e < m; ++e) edge_ptr[e + 1] += edge_ptr[e];
        return m ? edge_ptr[m] : 0;
    }
    if (m && (vtx_capacity < edge_ptr[m] || !demand)) return -1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int32_t e = 0; e < m; ++e) {
        int64_t pos = edge_ptr[e];
        if (attempt[e] == RETRIES) {
            edge_vtx[pos] = (int32_t)(mix64(seed, (uint64_t)e, 0xFFFFFFFFull, RETRIES) % (uint64_t)n);
        } else {
            for (int32_t v = 0; v < n; ++v)
                if (draw(seed, e, v, attempt[e], thr)) edge_vtx[pos++] = v;
        }
        const int64_t sz = edge_ptr[e + 1] - edge_ptr[e];
        demand[e] = (int32_t)(sz < alpha ? sz : alpha);
    }
    return m ? edge_ptr[m] : 0;
}
