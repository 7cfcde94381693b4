// verify.cuh -- exact decision of the candidate pairs the Gram kernel's probe
// pass listed (gram_tc2.cuh, GramArgs::cand).
//
// The probe proves, per pair, that c <= c' + min(rem_i, rem_j) cannot satisfy
// any predicate; a pair where it can is a *candidate*.  A tile with a few
// candidates (planted twins, duplicate edges: the typical case of a late or a
// near-irreducible round) does not need its full-K tensor pass: each
// candidate's count c = |X_i AND X_j| is one row-pair popcount over K bytes,
// after which the pair is evaluated with the same predicates as the tile
// epilogue (epilogue.cuh, reference parallel.py:106-114 / 140-142).
//
// Exactly-once accounting: every pair of a tile is decided either by pass 1
// of the Gram kernel (tile marked in `needed`) or here (tile not marked), so
// candidates of marked tiles are skipped.  Non-candidate pairs provably
// contribute nothing.
#pragma once
#include <cstdint>

#include "epilogue.cuh"

namespace mhsk {
namespace k {

// One warp per candidate: c = popcount(X_i & X_j) over the phase's K bytes
// (packed E2M1 1.0 = 0b0010 and int8 1 = 0x01 both leave one bit per common
// item), then both directions of the pair with i < j.  dev_mk[1] = K items,
// bki = items per 128-byte k-block (256 FP4, 128 int8).
template <int PHASE>
__global__ void verify_candidates(const int4* __restrict__ cand, const int32_t* __restrict__ cand_count,
                                  int32_t cand_cap, const uint32_t* __restrict__ needed,
                                  const int8_t* __restrict__ X, int64_t ld, const int32_t* __restrict__ dev_mk,
                                  int32_t bki, const int32_t* __restrict__ va, const int32_t* __restrict__ vb,
                                  int32_t* __restrict__ hits, unsigned long long* __restrict__ verified) {
    const int32_t n = min(*cand_count, cand_cap);
    const int64_t kb = max(1, (dev_mk[1] + bki - 1) / bki);
    const int64_t words = min(ld, kb * 128) / 16;   // uint4 words per row
    const int lane = threadIdx.x % 32;
    const int64_t wg = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    unsigned long long done = 0;
    for (int64_t q = wg; q < n; q += nw) {
        const int4 e = cand[q];
        if (e.x < 0 || ((needed[(uint32_t)e.z >> 5] >> ((uint32_t)e.z & 31u)) & 1u)) continue;
        const uint4* a = reinterpret_cast<const uint4*>(X + (int64_t)e.x * ld);
        const uint4* b = reinterpret_cast<const uint4*>(X + (int64_t)e.y * ld);
        int32_t c = 0;
        for (int64_t w = lane; w < words; w += 32) {
            const uint4 x = __ldg(a + w), y = __ldg(b + w);
            c += __popc(x.x & y.x) + __popc(x.y & y.y) + __popc(x.z & y.z) + __popc(x.w & y.w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            ItemVals vi, vj;
            vi.a = va[e.x];
            vj.a = va[e.y];
            vi.b = vb ? vb[e.x] : 0;
            vj.b = vb ? vb[e.y] : 0;
            bool i_del_j, j_del_i;
            pair_predicates<PHASE>(c, vi, vj, i_del_j, j_del_i);   // e.x < e.y
            if (i_del_j) atomicAdd(hits + e.y, 1);
            if (j_del_i) atomicAdd(hits + e.x, 1);
            ++done;
        }
    }
    if (lane == 0 && done && verified) atomicAdd(verified, done);
}

}  // namespace k
}  // namespace mhsk
