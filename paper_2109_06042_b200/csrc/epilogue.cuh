// epilogue.cuh -- the dominance / supersedence predicates, evaluated once per
// unordered pair {i, j}, i < j, from the co-occurrence count c = X_i . X_j.
//
// Reference semantics (pkg/src/mhskernel/parallel.py):
//   edge phase, rule dp (106-107):  R(i,j) <=> f_i - (s_i - c) >= f_j
//   edge phase, rule se (108):      R(i,j) <=> c == s_i  &&  f_i >= f_j
//   edge j is deleted iff exists i != j: R(i,j) && (!R(j,i) || i < j)  (110-114)
//   vertex phase (140-142):         D(i,j) <=> c == d_j && (c != d_i || i < j)
//   vertex j is deleted iff #{i != j : D(i,j)} >= need_j              (153-159)
//
// With i < j the index tie-breaks resolve statically, so one count yields
// both directions:
//   edge:   i deletes j  <=>  R(i,j)
//           j deletes i  <=>  R(j,i) && !R(i,j)
//   vertex: i dominates j <=> c == d_j
//           j dominates i <=> c == d_i && c != d_j
// Each kernel accumulates "number of deleters / dominators" per item in
// hits[]; an edge with hits > 0 is deleted, a vertex with hits >= need (or
// need == 0) is deleted (commit kernels in mhsk_kernels.cuh).
#pragma once
#include <cstdint>

namespace mhsk {

// Programmatic dependent launch (mhsk_capi.cu launch_pdl): a kernel launched
// with it may be scheduled while its predecessor on the stream still runs.
// Every kernel of the library first waits for the predecessor grid to
// complete and its memory to be visible (a no-op without a programmatic
// dependency), then allows its own dependents to be scheduled -- so the
// launch latency of each kernel hides behind the one before it.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


enum PhaseKind : int32_t { PHASE_DP = 0, PHASE_SE = 1, PHASE_MD = 2 };

// Per-item operands of the predicate: edges carry (size s, demand f),
// vertices carry (degree d, unused).
struct ItemVals {
    int32_t a;  // s_i or d_i
    int32_t b;  // f_i
};

template <int PHASE>
__device__ __forceinline__ void pair_predicates(int32_t c, ItemVals vi, ItemVals vj, bool& i_del_j,
                                                bool& j_del_i) {
    if constexpr (PHASE == PHASE_DP) {
        const bool rij = vi.b - vi.a + c >= vj.b;
        const bool rji = vj.b - vj.a + c >= vi.b;
        i_del_j = rij;
        j_del_i = rji && !rij;
    } else if constexpr (PHASE == PHASE_SE) {
        const bool rij = c == vi.a && vi.b >= vj.b;
        const bool rji = c == vj.a && vj.b >= vi.b;
        i_del_j = rij;
        j_del_i = rji && !rij;
    } else {
        i_del_j = c == vj.a;
        j_del_i = c == vi.a && c != vj.a;
    }
}

// General form for rows in any order: i_before_j says whether item i precedes
// item j in the original order (the tie-break); pair_predicates is the
// i_before_j == true case.
template <int PHASE>
__device__ __forceinline__ void pair_predicates_ranked(int32_t c, ItemVals vi, ItemVals vj, bool i_before_j,
                                                       bool& i_del_j, bool& j_del_i) {
    if constexpr (PHASE == PHASE_DP || PHASE == PHASE_SE) {
        bool rij, rji;
        if constexpr (PHASE == PHASE_DP) {
            rij = vi.b - vi.a + c >= vj.b;
            rji = vj.b - vj.a + c >= vi.b;
        } else {
            rij = c == vi.a && vi.b >= vj.b;
            rji = c == vj.a && vj.b >= vi.b;
        }
        i_del_j = rij && (!rji || i_before_j);
        j_del_i = rji && (!rij || !i_before_j);
    } else {
        i_del_j = c == vj.a && (c != vi.a || i_before_j);
        j_del_i = c == vi.a && (c != vj.a || !i_before_j);
    }
}

// Rectangle mode (incremental rounds): one direction per ordered pair, row
// item `ri` against column item `cj` (compact indices, ri != cj), tie-breaks by
// compact index (= original order).
//   edge phase:   row deletes column  <=>  R(r,c) && (!R(c,r) || r < c)
//   vertex phase: column dominates row <=> c == d_r && (c != d_c || c < r)
template <int PHASE>
__device__ __forceinline__ bool rect_predicate(int32_t c, ItemVals vr, ItemVals vc, int32_t ri, int32_t cj) {
    if constexpr (PHASE == PHASE_DP) {
        const bool rrc = vr.b - vr.a + c >= vc.b;
        const bool rcr = vc.b - vc.a + c >= vr.b;
        return rrc && (!rcr || ri < cj);
    } else if constexpr (PHASE == PHASE_SE) {
        const bool rrc = c == vr.a && vr.b >= vc.b;
        const bool rcr = c == vc.a && vc.b >= vr.b;
        return rrc && (!rcr || ri < cj);
    } else {
        return c == vr.a && (c != vc.a || cj < ri);
    }
}

// ------------------------------------------------------------ probe pruning
// A dense triangle tile first multiplies only its first probe_kb k-blocks
// (columns [0, K1)), giving the partial count c' of every pair.  With
// lo_i = item i's entries in [0, K1) and a_i its total, the full count obeys
//   c <= c' + min(a_i - lo_i, a_j - lo_j)
// and a pair whose predicates cannot hold under that bound in either
// direction contributes nothing.  If no pair of the tile can, the tile stops
// there; otherwise it runs to full K.  Results are unchanged by construction.
// The host sizes the probe so that a typical item has ~PROBE_ENTRIES entries
// in it (enough that c' < lo for unrelated pairs), and probes only when that
// is at most 1/PROBE_MIN_RATIO of K.
constexpr int32_t PROBE_ENTRIES = 16;   // measured optimum (profiles/NOTES.md #18)
constexpr int32_t PROBE_MIN_RATIO = 4;

// Can the pair (i, j) still produce a deletion / domination, given its probe
// count cp and the items' remaining entries r?  Per item x = a - b (DP) or a
// (SE, MD), b = demand (unused for MD).
template <int PHASE>
__device__ __forceinline__ bool pair_possible(int32_t cp, int32_t xi, int32_t bi, int32_t ri, int32_t xj, int32_t bj,
                                              int32_t rj) {
    const int32_t ub = cp + min(ri, rj);   // upper bound of the full count
    if constexpr (PHASE == PHASE_DP) {
        return ub - bj >= xi || ub - bi >= xj;   // c >= s_i - f_i + f_j, or i <-> j
    } else if constexpr (PHASE == PHASE_SE) {
        return (bi >= bj && ub >= xi) || (bj >= bi && ub >= xj);
    } else {
        // c == d_j or c == d_i with both degrees > 0 (a degree-0 vertex is
        // deleted regardless and cannot dominate a vertex of positive degree)
        const int32_t dmin = min(xi, xj);
        return dmin > 0 && ub >= dmin;
    }
}

// Cheaper necessary condition for the FP4 probe, in f32 (counts are exact
// integers below 2^23).  Using only c <= c' + rem_i (resp. rem_j), a pair can
// fire only if
//   DP: c' >= lo_i - f_i + f_j  or  c' >= lo_j - f_j + f_i
//   SE: c' >= lo_i (f_i >= f_j)  or  c' >= lo_j (f_j >= f_i)
//   MD: c' >= min(lo_i, lo_j), both degrees > 0
// With per-item L = lo - f (DP) / lo (SE) / lo or +inf for degree 0 (MD), the
// returned slack is >= 0 iff that holds (branch-free, so a chunk's pairs
// reduce with independent max chains).
template <int PHASE>
__device__ __forceinline__ float pair_slack_f(float cp, float Li, float bi, float Lj, float bj) {
    if constexpr (PHASE == PHASE_DP) {
        return cp - fminf(Li + bj, Lj + bi);
    } else if constexpr (PHASE == PHASE_SE) {
        const float s1 = bi >= bj ? cp - Li : -1.f;
        const float s2 = bj >= bi ? cp - Lj : -1.f;
        return fmaxf(s1, s2);
    } else {
        return cp - fminf(Li, Lj);
    }
}

// Per-item term L of pair_slack_f from size / degree a, demand b, probe count lo.
template <int PHASE>
__device__ __forceinline__ float probe_term_f(int32_t a, int32_t b, int32_t lo) {
    if constexpr (PHASE == PHASE_DP) return (float)(lo - b);
    else if constexpr (PHASE == PHASE_SE) return (float)lo;
    else return a > 0 ? (float)lo : __int_as_float(0x7f800000);   // degree 0: never
}

}  // namespace mhsk
