// schedule.h -- tile list of the symmetric (SYRK) Gram schedule.
//
// Tiles (I, J) are BM-row x BN-column blocks of the M x M count matrix with
// I <= (J+1)*BN/BM - 1, i.e. every tile that holds at least one pair i < j
// (pairs are evaluated once, both directions, epilogue.cuh).
//
// Order = L2 rasterisation.  A persistent CTA (pair) streams its tile's full
// K, so the wave of concurrently running tiles advances through K roughly in
// lock-step, and what one k-step pulls from HBM is (#distinct A panels) x A
// k-tile + (#distinct B panels) x B k-tile.  Column-major order makes a wave
// of the pair kernel 74 distinct A panels x 1 B panel: on config 4 that
// re-streams 2.2 TB from HBM per phase (HBM-bound at 6.6 TB/s, ncu in
// profiles/).  Here the triangle is cut into super-blocks of gp x gj squares
// of 256 x 256, visited super-column by super-column; a wave then touches
// ~2*gp A panels and gj B panels.  Measured on B200 (profiles/): 4 x 9
// (two super-blocks per 74-pair wave) is the fastest.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace mhsk {

struct TileShape {
    int32_t bm, bn;   // tile rows (A panel height) and columns (B panel height)
    int32_t gp, gj;   // super-block: gp x gj squares of bn x bn
};

inline int64_t tile_count(int32_t M, const TileShape& s) {
    const int64_t MI = (M + s.bm - 1) / s.bm, NJ = (M + s.bn - 1) / s.bn;
    int64_t n = 0;
    for (int64_t J = 0; J < NJ; ++J) n += std::min<int64_t>(MI, (J * s.bn + s.bn - 2) / s.bm + 1);
    return n;
}

// General shapes (bn not a multiple of bm: the FP4 kernel's 256 x 240 tiles).
// Tile (I, J) holds a pair i < j iff I*bm <= J*bn + bn - 2.  Same
// rasterisation: super-columns of gj column panels, within them super-rows of
// gp row panels.
template <class V>
inline void make_tile_list_general(int32_t M, const TileShape& s, V& out) {
    const int32_t MI = (M + s.bm - 1) / s.bm, NJ = (M + s.bn - 1) / s.bn;
    auto last_row = [&](int32_t J) { return std::min(MI - 1, (J * s.bn + s.bn - 2) / s.bm); };
    for (int32_t js = 0; js * s.gj < NJ; ++js) {
        const int32_t j_lo = js * s.gj, j_hi = std::min(NJ, j_lo + s.gj);
        const int32_t imax = last_row(j_hi - 1);
        for (int32_t ps = 0; ps * s.gp <= imax; ++ps) {
            const int32_t p_lo = ps * s.gp, p_hi = std::min(imax + 1, p_lo + s.gp);
            for (int32_t J = j_lo; J < j_hi; ++J)
                for (int32_t I = p_lo; I < std::min(p_hi, last_row(J) + 1); ++I)
                    out.push_back((uint32_t)I | ((uint32_t)J << 16));
        }
    }
}

// Appends the packed tiles (I | J << 16) of the triangle for M items.
template <class V>
inline void make_tile_list(int32_t M, const TileShape& s, V& out) {
    out.clear();
    if (M <= 0) return;
    if (s.bn % s.bm != 0) {
        make_tile_list_general(M, s, out);
        return;
    }
    const int32_t MI = (M + s.bm - 1) / s.bm, NJ = (M + s.bn - 1) / s.bn;
    const int32_t R = s.bn / s.bm;   // A panels per square
    const int32_t NP = NJ;           // square rows
    for (int32_t js = 0; js * s.gj < NJ; ++js) {
        const int32_t j_lo = js * s.gj, j_hi = std::min(NJ, j_lo + s.gj);
        for (int32_t ps = 0; ps * s.gp < std::min(NP, j_hi); ++ps) {
            const int32_t p_lo = ps * s.gp, p_hi = std::min(NP, p_lo + s.gp);
            for (int32_t J = j_lo; J < j_hi; ++J)
                for (int32_t P = p_lo; P < std::min(p_hi, J + 1); ++P)
                    for (int32_t r = 0; r < R; ++r) {
                        const int32_t I = P * R + r;
                        if (I < MI) out.push_back((uint32_t)I | ((uint32_t)J << 16));
                    }
        }
    }
}

// Band-major list for a streamed upload: rows (items) arrive in chunks, rows
// [0, E[b]) complete after chunk b.  Band b holds the triangle tiles whose
// both panels are complete after chunk b but not after chunk b - 1, in the
// usual raster order; each band is padded with dummy entries (0xFFFFFFFF,
// skipped by every consumer) to a multiple of `pairs`, so that pair p's
// tiles of band b are exactly its t in [t_begin[b], t_begin[b+1]) of the
// interleaved schedule (list entry p + t * pairs).  E.back() must be M.
template <class V>
inline void make_band_tile_list(int32_t M, const TileShape& s, const std::vector<int32_t>& E, int32_t pairs,
                                V& out, std::vector<int32_t>& t_begin) {
    std::vector<uint32_t> all;
    make_tile_list(M, s, all);
    std::vector<std::vector<uint32_t>> bands(E.size());
    for (const uint32_t pj : all) {
        const int64_t I = pj & 0xFFFF, J = pj >> 16;
        const int64_t last = std::min<int64_t>(M - 1, std::max(I * s.bm + s.bm - 1, J * s.bn + s.bn - 1));
        size_t b = 0;
        while (b + 1 < E.size() && E[b] <= last) ++b;
        bands[b].push_back(pj);
    }
    out.clear();
    t_begin.assign(1, 0);
    for (auto& band : bands) {
        out.insert(out.end(), band.begin(), band.end());
        while (out.size() % (size_t)pairs) out.push_back(0xFFFFFFFFu);
        t_begin.push_back((int32_t)(out.size() / (size_t)pairs));
    }
}

}  // namespace mhsk
