// mhsk_kernels.cuh -- the HBM-bound kernels around the Gram product:
// order-preserving compaction (ActiveInstance.extract, rules.py:88-103),
// operand packing (incidence_matrix + the need loop, bitmatrix.py:113-130,
// parallel.py:101,137,145-150), the commit of a phase's deletions
// (parallel.py:190-205), and the SIMT bit-packed AND+popc Gram used to
// cross-check the tensor-core path.
#pragma once
#include <cstdint>

#include "epilogue.cuh"

namespace mhsk {
namespace k {


// Single-pass compaction (decoupled look-back).  Tile t = CP_ITEMS
// consecutive positions k; item k is alive[perm ? perm[k] : k] and its id is
// perm ? perm[k] : k.  Outputs ids[pos] = id, new_id[id] = pos or -1 (new_id
// optional), *total.  Each tile publishes its count (flag A), then warp 0 sums
// predecessors 32 at a time back to the nearest inclusive prefix (flag P).
// status[t] = epoch << 34 | flag << 32 | value; a different epoch reads as
// "not yet published", so the array is never cleared between calls.  The grid
// is at most one block per SM, all co-resident, tiles visited in increasing
// order -- every wait is on a smaller tile, so the look-back cannot deadlock.
constexpr int CP_THREADS = 1024, CP_PER_THREAD = 4, CP_ITEMS = CP_THREADS * CP_PER_THREAD;
constexpr unsigned long long CP_A = 1ull << 32, CP_P = 2ull << 32;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(CP_THREADS)
compact_1pass(const uint8_t* __restrict__ alive, int32_t n, const int32_t* __restrict__ n_dyn,
              const int32_t* __restrict__ perm, int32_t* __restrict__ new_id, int32_t* __restrict__ ids,
              int32_t* __restrict__ total, unsigned long long* __restrict__ status, uint32_t epoch) {
    mhsk::pdl_enter();
    __shared__ int32_t warp_sums[CP_THREADS / 32];
    __shared__ int32_t tile_base;
    if (n_dyn) n = min(n, *n_dyn);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    const int32_t ntiles = max(1, (n + CP_ITEMS - 1) / CP_ITEMS);
    const unsigned long long tag = (unsigned long long)epoch << 34;
    for (int32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int32_t k0 = t * CP_ITEMS + threadIdx.x * CP_PER_THREAD;
        bool a[CP_PER_THREAD];
        int32_t cnt = 0;
#pragma unroll
        for (int i = 0; i < CP_PER_THREAD; ++i) {
            const int32_t k = k0 + i;
            a[i] = k < n && alive[perm ? perm[k] : k];
            cnt += a[i];
        }
        // block exclusive scan of the per-thread counts
        int32_t x = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            const int32_t v = warp_sums[lane];
            int32_t s = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s - v;   // exclusive prefix of warp totals
            const int32_t agg = __shfl_sync(0xffffffffu, s, 31);
            // publish, then look back
            if (lane == 0) st_release_u64(status + t, tag | (t == 0 ? CP_P : CP_A) | (uint32_t)agg);
            int32_t excl = 0;
            for (int32_t j = t - 1; j >= 0; j -= 32) {
                const int32_t kk = j - lane;
                unsigned long long st = kk >= 0 ? ld_acquire_u64(status + kk) : (tag | CP_P);
                while (!__all_sync(0xffffffffu, (st >> 34) == epoch && (st & (3ull << 32)))) {
                    if (!((st >> 34) == epoch && (st & (3ull << 32)))) st = ld_acquire_u64(status + kk);
                }
                const uint32_t pmask = __ballot_sync(0xffffffffu, (st & (3ull << 32)) == CP_P);
                const int lim = pmask ? __ffs(pmask) - 1 : 31;
                int32_t v2 = lane <= lim ? (int32_t)(uint32_t)st : 0;
                for (int o = 16; o > 0; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
                excl += v2;
                if (pmask) break;
            }
            if (lane == 0) {
                if (t > 0) st_release_u64(status + t, tag | CP_P | (uint32_t)(excl + agg));
                tile_base = excl;
                if (t == ntiles - 1) *total = excl + agg;
            }
        }
        __syncthreads();
        int32_t pos = tile_base + warp_sums[w] + x - cnt;
#pragma unroll
        for (int i = 0; i < CP_PER_THREAD; ++i) {
            const int32_t k = k0 + i;
            if (k < n) {
                const int32_t id = perm ? perm[k] : k;
                if (new_id) new_id[id] = a[i] ? pos : -1;
                if (a[i]) ids[pos++] = id;
            }
        }
        __syncthreads();   // warp_sums / tile_base reused by the next tile
    }
}

// ------------------------------------------------------------------ packing
// Edge phase operand: row r = enew[e] of X holds the alive members of edge e
// (column = vnew[v]).  Also writes s_r (alive size) and f_r (demand).
// One warp per original edge.  X was zeroed beforehand.
template <bool BITS>
__global__ void pack_edge_rows(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                               const int32_t* __restrict__ demand, const int32_t* __restrict__ enew,
                               const int32_t* __restrict__ vnew, void* __restrict__ X, int64_t ld,
                               int32_t* __restrict__ size_out, int32_t* __restrict__ dem_out) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int32_t r = enew[e];
        if (r < 0) continue;
        int32_t cnt = 0;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t c = vnew[edge_vtx[p]];
            if (c >= 0) {
                ++cnt;
                if constexpr (BITS) {
                    atomicOr(reinterpret_cast<uint32_t*>(X) + r * ld + (c >> 5), 1u << (c & 31));
                } else {
                    reinterpret_cast<int8_t*>(X)[r * ld + c] = 1;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) {
            size_out[r] = cnt;
            dem_out[r] = demand[e];
        }
    }
}

// Vertex phase operand: row vnew[v] of X holds the alive edges containing v
// (column = enew[e]); accumulates deg and need = max demand (atomics are
// order-independent, so the result is deterministic).
template <bool BITS>
__global__ void pack_vertex_rows(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                                 const int32_t* __restrict__ demand, const int32_t* __restrict__ enew,
                                 const int32_t* __restrict__ vnew, void* __restrict__ X, int64_t ld,
                                 int32_t* __restrict__ deg_out, int32_t* __restrict__ need_out) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int32_t col = enew[e];
        if (col < 0) continue;
        const int32_t f = demand[e];
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t r = vnew[edge_vtx[p]];
            if (r >= 0) {
                if constexpr (BITS) {
                    atomicOr(reinterpret_cast<uint32_t*>(X) + r * ld + (col >> 5), 1u << (col & 31));
                } else {
                    reinterpret_cast<int8_t*>(X)[r * ld + col] = 1;
                }
                atomicAdd(deg_out + r, 1);
                atomicMax(need_out + r, f);
            }
        }
    }
}

// ------------------------------------------------------------------- commit
// Apply a phase's decisions: edge phase deletes r iff hits[r] > 0; vertex
// phase deletes r iff need[r] == 0 || hits[r] >= need[r].  Counts deletions
// into *deleted.
template <bool VERTEX>
__global__ void commit_phase(int32_t count, const int32_t* __restrict__ hits, const int32_t* __restrict__ need,
                             const int32_t* __restrict__ ids, uint8_t* __restrict__ alive,
                             uint8_t* __restrict__ keep_out, int32_t* __restrict__ deleted,
                             const int32_t* __restrict__ count_dyn = nullptr,
                             uint8_t* __restrict__ del_flag = nullptr) {
    mhsk::pdl_enter();
    if (count_dyn) count = min(count, *count_dyn);
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    bool del = false;
    if (r < count) {
        if constexpr (VERTEX) del = need[r] == 0 || hits[r] >= need[r];
        else del = hits[r] > 0;
        if (keep_out) keep_out[r] = del ? 0 : 1;
        if (del && alive) alive[ids[r]] = 0;
        if (del && del_flag) del_flag[ids[r]] = 1;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, del);
    if (threadIdx.x % 32 == 0 && b) atomicAdd(deleted, __popc(b));
}

// --------------------------------------------------- SIMT validation Gram
// Bit-packed AND + popc over 32-bit words, 32x32 pairs per block, both
// operands staged through shared memory.  Evaluates only i < j and applies
// the same pair predicates as the tensor-core epilogue.  Kept as the
// cross-check backend (MHSK_BACKEND=simt), not the product path.
template <int PHASE>
__global__ void gram_simt(int32_t M, int32_t words, const uint32_t* __restrict__ Xb, int64_t ld,
                          const int32_t* __restrict__ va, const int32_t* __restrict__ vb,
                          int32_t* __restrict__ hits) {
    mhsk::pdl_enter();
    constexpr int T = 32, KW = 32;
    __shared__ uint32_t As[T][KW + 1];
    __shared__ uint32_t Bs[T][KW + 1];
    const int bi = blockIdx.y * T, bj = blockIdx.x * T;
    if (bi > bj + T - 1) return;  // whole block below the diagonal: nothing with i < j
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8 threads, each 4 rows
    int32_t acc[4] = {0, 0, 0, 0};
    for (int w0 = 0; w0 < words; w0 += KW) {
        for (int rr = ty; rr < T; rr += 8) {
            const int64_t gi = bi + rr, gj = bj + rr;
            As[rr][tx] = (gi < M && w0 + tx < words) ? Xb[gi * ld + w0 + tx] : 0u;
            Bs[rr][tx] = (gj < M && w0 + tx < words) ? Xb[gj * ld + w0 + tx] : 0u;
        }
        __syncthreads();
#pragma unroll 4
        for (int w = 0; w < KW; ++w) {
            const uint32_t b = Bs[tx][w];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += __popc(As[ty + 8 * u][w] & b);
        }
        __syncthreads();
    }
    const int32_t j = bj + tx;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int32_t i = bi + ty + 8 * u;
        if (i < M && j < M && i < j) {
            ItemVals vi{va[i], vb ? vb[i] : 0}, vj{va[j], vb ? vb[j] : 0};
            bool i_del_j, j_del_i;
            pair_predicates<PHASE>(acc[u], vi, vj, i_del_j, j_del_i);
            if (i_del_j) atomicAdd(hits + j, 1);
            if (j_del_i) atomicAdd(hits + i, 1);
        }
    }
}

}  // namespace k
}  // namespace mhsk

// ------------------------------------------------------------- full-edge rule
// FE (reference rules.py:138-181) as three data-parallel passes.  In the
// reference's cascade every forced vertex lowers an edge's size AND demand by
// one, so demand - size is invariant: the full edges are exactly the edges
// full at the start of the pass, the forced vertices F are the union of their
// alive members, an edge is deleted iff it is full or f - |e n F| <= 0, and
// survivors keep demand f - |e n F| -- independent of the cascade order.  An
// alive edge with f > s makes the pass infeasible before any deletion
// (rules.py:150-156).
namespace mhsk {
namespace k {

// Pass 1: alive size per alive edge, full flag, first infeasible edge.
__global__ void fe_mark(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                        const int32_t* __restrict__ demand, const uint8_t* __restrict__ valive,
                        const uint8_t* __restrict__ ealive, uint8_t* __restrict__ full,
                        int32_t* __restrict__ first_infeasible) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        if (!ealive[e]) {
            if (lane == 0) full[e] = 0;
            continue;
        }
        int32_t s = 0;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) s += valive[edge_vtx[p]];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            full[e] = demand[e] == s;
            if (demand[e] > s) atomicMin(first_infeasible, (int32_t)e + 1);
        }
    }
}

// Pass 2: forced[v] = 1 for the alive members of full edges.
__global__ void fe_force(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                         const uint8_t* __restrict__ valive, const uint8_t* __restrict__ full,
                         const int32_t* __restrict__ first_infeasible, uint8_t* __restrict__ forced) {
    mhsk::pdl_enter();
    if (*first_infeasible != 0x7FFFFFFF) return;
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        if (!full[e]) continue;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t v = edge_vtx[p];
            if (valive[v]) forced[v] = 1;
        }
    }
}

// Pass 3: demand decrements and edge deletions; counts deleted edges.
__global__ void fe_apply_edges(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                               int32_t* __restrict__ demand, uint8_t* __restrict__ ealive,
                               const uint8_t* __restrict__ full, const uint8_t* __restrict__ forced,
                               const int32_t* __restrict__ first_infeasible, int32_t* __restrict__ deleted) {
    mhsk::pdl_enter();
    if (*first_infeasible != 0x7FFFFFFF) return;
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        if (!ealive[e]) continue;
        int32_t hit = 0;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) hit += forced[edge_vtx[p]];
        for (int o = 16; o > 0; o >>= 1) hit += __shfl_xor_sync(0xffffffffu, hit, o);
        if (lane == 0) {
            const int32_t f = demand[e] - hit;
            if (full[e] || f <= 0) {
                ealive[e] = 0;
                atomicAdd(deleted, 1);
            } else {
                demand[e] = f;
            }
        }
    }
}

// Pass 4: forced vertices leave the instance; counts them (budget delta).
__global__ void fe_apply_vertices(int32_t n, const uint8_t* __restrict__ forced, uint8_t* __restrict__ valive,
                                  const int32_t* __restrict__ first_infeasible, int32_t* __restrict__ n_forced) {
    mhsk::pdl_enter();
    if (*first_infeasible != 0x7FFFFFFF) return;
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const bool f = v < n && forced[v];
    if (f) valive[v] = 0;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (threadIdx.x % 32 == 0 && b) atomicAdd(n_forced, __popc(b));
}

}  // namespace k
}  // namespace mhsk

// ------------------------------------------------ coalesced operand packing
// The tensor-core backends build their int8 operands with full-line, 16-byte
// vector stores (no memset, no scattered byte stores):
//   pack_rows_csr     edge-phase operand X_E straight from CSR (row = edge)
//   transpose_pack    vertex-phase operand X_V = X_E^T restricted to the
//                     surviving edges, by warp-ballot bit transposes
//   need_from_csr     need_j = max demand over j's alive edges
namespace mhsk {
namespace k {

// 32-bit mask -> 32 bytes of 0/1 (byte t = bit t).
__device__ __forceinline__ void expand_mask(uint32_t m, uint32_t (&w)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = (((m >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
}

constexpr int PACK_WARPS = 8;
constexpr int PACK_UNROLL = 16;  // CSR members per lane in flight (tail and scatter loops)
constexpr int PACK_WIN = 512;  // bytes of a row written per warp iteration (32 lanes x 16 B)

// 8 packed E2M1 0/1 items (a 32-bit word) -> 8 bits, bit t = item t nonzero
__device__ __forceinline__ uint32_t compress_nibbles(uint32_t w) {
    uint32_t x = (w >> 1) & 0x11111111u;   // 1.0 = 0b0010
    x = (x | (x >> 3)) & 0x03030303u;
    x = (x | (x >> 6)) & 0x000F000Fu;
    return (x | (x >> 12)) & 0xFFu;
}

// Warp-wide 32x32 bit-matrix transpose: lane l holds row l (bit c = column
// c); afterwards lane l holds column l (bit r = row r).  Stage s swaps lane
// bit s with bit-index bit s.
__device__ __forceinline__ uint32_t transpose32_warp(uint32_t x, uint32_t lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int sft = 16 >> t;
        const uint32_t m = masks[t];
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
        x = (lane & sft) ? ((x & ~m) | ((y >> sft) & m)) : ((x & m) | ((y << sft) & ~m));
    }
    return x;
}

// 32-bit mask -> 32 packed E2M1 items (16 bytes): item t = 1.0 (0b0010) iff bit t.
__device__ __forceinline__ void expand_mask_fp4(uint32_t m, uint32_t (&w)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t x = (m >> (8 * q)) & 0xFFu;   // bit b -> bit 4b
        x = (x | (x << 12)) & 0x000F000Fu;
        x = (x | (x << 6)) & 0x03030303u;
        x = (x | (x << 3)) & 0x11111111u;
        w[q] = x << 1;
    }
}

// PACK_UNROLL members k0 + 32u (< hi) -> columns (-1: past the row or a dead
// vertex).  All member loads are issued before the first vnew gather: mixing
// them (vnew ? vnew[vtx[k]] : vtx[k] per u) compiled to one load -> gather
// -> load chain per member, which left the CSR stream latency-bound.
__device__ __forceinline__ void load_cols(int32_t (&col)[PACK_UNROLL], int64_t k0, int64_t hi,
                                          const int32_t* __restrict__ edge_vtx,
                                          const int32_t* __restrict__ vnew) {
#pragma unroll
    for (int u = 0; u < PACK_UNROLL; ++u) {
        const int64_t k = k0 + 32 * u;
        col[u] = k < hi ? __ldg(edge_vtx + k) : -1;
    }
    if (vnew) {
#pragma unroll
        for (int u = 0; u < PACK_UNROLL; ++u)
            if (col[u] >= 0) col[u] = __ldg(vnew + col[u]);
    }
}

// Round 1 of a call (every item alive): one streaming pass over the member
// array that validates it and, under uniform demand, marks every member in
// the n-bit 'seen' map (need_j = f * [j has a member]; need_from_seen).
// Validation (validate_csr's member checks, fused into the edge pack's
// round): ids in [0, n) (flags[0] = 1 otherwise), and strictly increasing
// inside an edge.  For the latter the pass counts the descents -- positions
// k >= 1 with vtx[k] <= vtx[k-1] -- into desc[0], and pack_rows_csr counts
// those at the first member of a non-empty edge into desc[1]: a non-empty
// edge's first member is the only place a descent is legal, and each such
// position belongs to exactly one non-empty edge, so the CSR is ordered iff
// desc[0] == desc[1].  No per-member search, no per-edge dependency chain:
// the array is read as 16-byte vectors, SCAN_UNROLL per lane in flight.
// The seen bits go into a per-block shared-memory copy of the map (shared
// atomics after a shared test), OR-ed into the global map once per block at
// the end (MAP 1, n <= SCAN_SMEM_BITS); otherwise straight into the global
// map after an L2-coherent test (MAP 2; an L1-cached test would keep reading
// a stale line and repeat the atomic for every member).  Measured at config
// 4: 80 us without the map, 141 us with MAP 1; a global map that stops once
// every bit is set was slower (185 us: every member of the first sweep pays
// an L2 round trip).
constexpr int SCAN_UNROLL = 4;
constexpr int SCAN_THREADS = 512;   // x <= 64 registers: two blocks per SM
constexpr int64_t SCAN_SMEM_BITS = (int64_t)96 * 1024 * 8;   // 96 KB: two blocks per SM

// MAP: 0 no seen map (non-uniform demand or no lazy vertex phase), 1 shared
// copy, 2 global.  Loads of the next iteration are issued before the current
// one is visited (two register buffers: 2 x SCAN_UNROLL x 16 B per lane).
template <int MAP>
__global__ void __launch_bounds__(SCAN_THREADS, 2)
scan_members(int32_t n, int32_t m, const int64_t* __restrict__ ptr, const int32_t* __restrict__ vtx_all,
             uint32_t* __restrict__ seen, const int32_t* __restrict__ f_range, int32_t* __restrict__ flags,
             unsigned long long* __restrict__ desc, int64_t k_begin, int64_t k_end,
             const int32_t* __restrict__ map_full = nullptr) {
    mhsk::pdl_enter();
    // members [k_begin, k_end) (k_end < 0: to nnz); a streamed upload scans
    // each chunk as it lands (the predecessor of k_begin is in an earlier one)
    extern __shared__ uint32_t smap[];
    const int64_t nnz = (k_end < 0 ? max(ptr[m], (int64_t)0) : k_end) - k_begin;
    const int32_t* __restrict__ vtx = vtx_all + k_begin;
    // uniform demand only (need_j = f [j has a member]); otherwise the pack's
    // member walk accumulates need
    // map_full (seen_full after an earlier part): every vertex is already
    // seen, the rest of the pass only validates
    const bool uni = MAP != 0 && f_range[0] == f_range[1] && !(map_full && *map_full);
    const int32_t map_words = (n + 31) / 32;
    if (MAP == 1 && uni) {
        for (int32_t w = threadIdx.x; w < map_words; w += blockDim.x) smap[w] = 0;
        __syncthreads();
    }
    const bool vec = ((uintptr_t)vtx & 15) == 0;
    const int lane = threadIdx.x % 32;
    const int64_t nq = (nnz + 3) / 4;   // 4-member quads
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane) * SCAN_UNROLL;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * SCAN_UNROLL;
    bool bad = false;
    uint32_t descents = 0;
    auto load = [&](int4 (&x)[SCAN_UNROLL], int64_t base) {
        const bool full = vec && 4 * (base + 32 * SCAN_UNROLL) <= nnz;
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) {
            const int64_t q = base + 32 * u + lane;
            const int64_t k0 = 4 * q;
            if (full) {
                x[u] = __ldg(reinterpret_cast<const int4*>(vtx) + q);
            } else {
                x[u].x = k0 < nnz ? __ldg(vtx + k0) : 0x7fffffff;
                x[u].y = k0 + 1 < nnz ? __ldg(vtx + k0 + 1) : 0x7fffffff;
                x[u].z = k0 + 2 < nnz ? __ldg(vtx + k0 + 2) : 0x7fffffff;
                x[u].w = k0 + 3 < nnz ? __ldg(vtx + k0 + 3) : 0x7fffffff;
            }
        }
    };
#define SCAN_VISIT(V, PREV)                                                            \
    {                                                                                  \
        const int32_t v_ = (V);                                                        \
        const bool in_ = (uint32_t)v_ < (uint32_t)n;                                   \
        bad |= !in_;                                                                   \
        descents += v_ <= (PREV);                                                      \
        if (MAP != 0 && uni && in_) {                                                  \
            const uint32_t bit_ = 1u << (v_ & 31);                                     \
            if (MAP == 1) {                                                            \
                if (!(smap[v_ >> 5] & bit_)) atomicOr(smap + (v_ >> 5), bit_);         \
            } else if (!(__ldcg(seen + (v_ >> 5)) & bit_)) {                           \
                atomicOr(seen + (v_ >> 5), bit_);                                      \
            }                                                                          \
        }                                                                              \
    }
    int4 cur[SCAN_UNROLL], nxt[SCAN_UNROLL];
    if (warp0 < nq) load(cur, warp0);
    for (int64_t base = warp0; base < nq; base += step) {   // warp-uniform bound
        if (base + step < nq) load(nxt, base + step);
        const bool full = vec && 4 * (base + 32 * SCAN_UNROLL) <= nnz;
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) {
            const int64_t k0 = 4 * (base + 32 * u + lane);
            int32_t prev = __shfl_up_sync(0xffffffffu, cur[u].w, 1);
            // the array's first member has no predecessor: not a descent
            if (lane == 0) prev = k_begin + k0 > 0 && k0 - 1 < nnz ? __ldg(vtx + k0 - 1) : 0x80000000;
            if (full) {
                SCAN_VISIT(cur[u].x, prev);
                SCAN_VISIT(cur[u].y, cur[u].x);
                SCAN_VISIT(cur[u].z, cur[u].y);
                SCAN_VISIT(cur[u].w, cur[u].z);
            } else {
                if (k0 < nnz) SCAN_VISIT(cur[u].x, prev);
                if (k0 + 1 < nnz) SCAN_VISIT(cur[u].y, cur[u].x);
                if (k0 + 2 < nnz) SCAN_VISIT(cur[u].z, cur[u].y);
                if (k0 + 3 < nnz) SCAN_VISIT(cur[u].w, cur[u].z);
            }
        }
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) cur[u] = nxt[u];
    }
#undef SCAN_VISIT
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(flags, 1);
    for (int o = 16; o > 0; o >>= 1) descents += __shfl_xor_sync(0xffffffffu, descents, o);
    if (lane == 0 && descents) atomicAdd(desc, (unsigned long long)descents);
    if (MAP == 1 && uni) {   // only bits the global map lacks (streamed chunks: soon none)
        __syncthreads();
        for (int32_t w = threadIdx.x; w < map_words; w += blockDim.x) {
            const uint32_t mine = smap[w];
            if (mine && (mine & ~__ldcg(seen + w))) atomicOr(seen + w, mine);
        }
    }
}

// *full = every one of the n bits of `seen` is set (one block).  The member
// scan sets the map from the first part of the array; at configs 4/5 every
// vertex has ~1e3 members, so the first 1/8 already sets every bit and the
// other 7/8 skip the map work (scan 138 -> ~95 us).
__global__ void seen_full(const uint32_t* __restrict__ seen, int32_t n, int32_t* __restrict__ full) {
    mhsk::pdl_enter();
    __shared__ int32_t partial[32];
    int32_t c = 0;
    for (int32_t w = threadIdx.x; w < n / 32; w += blockDim.x) c += __popc(seen[w]);
    if (threadIdx.x == 0 && (n & 31)) c += __popc(seen[n / 32] & ((1u << (n & 31)) - 1u));
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x % 32 == 0) partial[threadIdx.x / 32] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        c = threadIdx.x < (int)blockDim.x / 32 ? partial[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (threadIdx.x == 0) *full = c == n;
    }
}

// Row r < M of X (ld bytes, rows_pad rows): the alive members of edge
// eids[r] at columns vnew[v]; rows M..rows_pad-1 and columns beyond the last
// member are zero.  Also s_r (alive size) and f_r, and (lo_out) the members in
// columns [0, K1) for the Gram's probe pruning.  One warp per row: the
// sorted member list is merged against 512-byte windows staged in shared
// memory, each window stored with one 16-byte store per lane.  FP4: column c
// is nibble c & 1 of byte c / 2 (E2M1 1.0 = 0b0010), a window spans 1024
// columns and the row is written up to K rounded to 256 items.
template <bool FP4 = false>
__global__ void __launch_bounds__(PACK_WARPS * 32)
pack_rows_csr(int32_t M, int32_t rows_pad, const int32_t* __restrict__ eids,
              const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
              const int32_t* __restrict__ demand, const int32_t* __restrict__ vnew,
              int8_t* __restrict__ X, int64_t ld, int32_t* __restrict__ size_out,
              int32_t* __restrict__ dem_out, const int32_t* __restrict__ dev_mk = nullptr,
              int32_t* __restrict__ lo_out = nullptr, int64_t K1 = 0,
              int32_t* __restrict__ deg_acc = nullptr, int32_t* __restrict__ need_acc = nullptr,
              int64_t write_bytes = -1, const uint8_t* __restrict__ panel_sel = nullptr,
              const uint8_t* __restrict__ row_sel = nullptr, uint32_t* __restrict__ seen = nullptr,
              const int32_t* __restrict__ f_range = nullptr, int32_t* __restrict__ vflags = nullptr,
              const int64_t* __restrict__ nnz_ptr = nullptr, unsigned long long* __restrict__ desc = nullptr,
              int64_t r_lo = 0, int64_t r_hi = -1, const uint32_t* __restrict__ alive_bits = nullptr,
              int32_t* __restrict__ need_low = nullptr, int32_t map_words = 0) {
    mhsk::pdl_enter();
    // vnew == nullptr: every vertex alive, column = vertex id (no gather).
    // write_bytes >= 0 (lazy edge operand): only the first write_bytes bytes
    // of each row are written (the probe columns); sizes, lo and need still
    // cover every member.  panel_sel: only rows of 256-row panels flagged 1
    // (and rows flagged in row_sel).
    // deg_acc / need_acc (lazy vertex operand, pre-zeroed, each optional): per
    // alive member column, the number of this round's alive edges holding it
    // and their maximum demand -- the vertex phase's degrees and need before
    // the edge phase's deletions (fix_deleted_edges applies those)
    // vflags (round 1 of a call, validation fused in, see scan_members): the
    // per-edge checks of validate_csr (offsets, demand >= 1, feasibility) on
    // each packed edge and the descents at first members (desc[1]), offsets
    // clamped into [0, nnz] so a malformed CSR is
    // never read out of bounds; under uniform demand with every vertex alive
    // and no degree accumulation the members beyond the written windows are
    // not visited (scan_members marked them in 'seen'; size = hi - lo).
    // need_low (FP4 lazy vertex phase; no deg_acc / need_acc): need by
    // ORIGINAL vertex id, two-tier -- 'seen' marks the members of rows with
    // the largest demand fmax = f_range[1], need_low keeps the max demand of
    // the others (need_from_seen_ids: need = seen ? fmax : need_low) -- and
    // the members beyond the written windows are not gathered through vnew:
    // alive_bits (original ids; nullptr = every vertex alive) says which
    // count.
    // map_words > 0 (later rounds: need_low and alive_bits set; dynamic shared
    // memory of 2 * map_words words): the alive map and a per-CTA seen map are
    // held in shared memory -- the member loop's two bit tests per member
    // were random L1 accesses (~27 wavefronts per warp-wide test; ncu: long-
    // scoreboard stalls, 1.7 TB/s) -- and the seen bits the global map lacks
    // are OR-ed out at the end.
    __shared__ __align__(16) uint8_t win[PACK_WARPS][PACK_WIN];
    extern __shared__ uint32_t pack_maps[];
    const bool smaps = map_words > 0 && need_low != nullptr && alive_bits != nullptr && seen != nullptr;
    uint32_t* const s_alive = pack_maps;
    uint32_t* const s_seen = pack_maps + (smaps ? map_words : 0);
    if (smaps) {
        for (int32_t i = threadIdx.x; i < map_words; i += blockDim.x) {
            s_alive[i] = __ldg(alive_bits + i);
            s_seen[i] = 0u;
        }
        __syncthreads();
    }
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* buf = win[w];
    int64_t width = ld;   // bytes written (the Gram reads K_pad of the current K)
    if (dev_mk) {         // device-resident sizes: rows M = dev_mk[0], columns K = dev_mk[1]
        M = dev_mk[0];
        rows_pad = min((int64_t)rows_pad, (int64_t)(M + 255) / 256 * 256);
        width = FP4 ? min(ld, (int64_t)(max(dev_mk[1], 1) + 255) / 256 * 128)
                    : min(ld, (int64_t)(max(dev_mk[1], 1) + 127) / 128 * 128);
    }
    constexpr int COLS_PER_WIN = FP4 ? 2 * PACK_WIN : PACK_WIN;
    const int64_t wlim = write_bytes >= 0 ? min(width, (write_bytes + PACK_WIN - 1) / PACK_WIN * PACK_WIN) : width;
    // uniform demand over the rows (f_range[0] == f_range[1], demand_range):
    // need_j = f * [j has a member], so a member only sets its bit in the
    // n-bit 'seen' map (L1-resident, read before the rare atomicOr) instead of
    // reading the n-word need array (an L2 sector per member);
    // need_from_seen expands the map afterwards
    const bool uni = seen && f_range[0] == f_range[1];
    const bool orig = need_low != nullptr;
    const int32_t fmax = orig ? f_range[1] : 0;
    auto need_update_orig = [&](int32_t v, int32_t f_e) {
        if (f_e == fmax) {
            const uint32_t bit = 1u << (v & 31);
            if (smaps) {
                MHSK_CHECK((v >> 5) < map_words);
                if (!(s_seen[v >> 5] & bit)) atomicOr(s_seen + (v >> 5), bit);
            } else if (!(__ldca(seen + (v >> 5)) & bit)) {
                atomicOr(seen + (v >> 5), bit);
            }
        } else if (__ldcg(need_low + v) < f_e) {
            atomicMax(need_low + v, f_e);
        }
    };
    auto need_update = [&](int32_t col, int32_t f_e, bool l1) {
        MHSK_CHECK(col >= 0);
        if (uni) {
            const uint32_t bit = 1u << (col & 31);
            if (!(__ldca(seen + (col >> 5)) & bit)) atomicOr(seen + (col >> 5), bit);
        } else if (need_acc) {
            const int32_t cur = l1 ? __ldca(need_acc + col) : *((volatile int32_t*)(need_acc + col));
            if (cur < f_e) atomicMax(need_acc + col, f_e);
        }
    };
    uint32_t start_desc = 0;   // lane 0: descents at first members (vflags)
    // rows [r_lo, r_hi) of the padded operand (a streamed upload packs each
    // chunk's complete edges as they land)
    const int64_t r_end = r_hi < 0 ? (int64_t)rows_pad : min(r_hi, (int64_t)rows_pad);
    for (int64_t r = r_lo + (int64_t)blockIdx.x * PACK_WARPS + w; r < r_end; r += (int64_t)gridDim.x * PACK_WARPS) {
        if (panel_sel && panel_sel[r >> 8] != 1 && !(row_sel && r < M && row_sel[r])) continue;
        int8_t* row = X + r * ld;
        if (r >= M) {
            for (int64_t b = lane * 16; b < wlim; b += 32 * 16)
                *reinterpret_cast<uint4*>(row + b) = make_uint4(0, 0, 0, 0);
            continue;
        }
        const int32_t e = eids[r];
        int64_t p = edge_ptr[e];
        int64_t hi = edge_ptr[e + 1];
        if (vflags) {
            const int64_t nnz = max(*nnz_ptr, (int64_t)0);
            const int32_t f = demand[e];
            const bool bad = hi < p || p < 0 || hi > nnz || f < 1 || (e == 0 && p != 0);
            if (lane == 0) {
                if (bad) atomicExch(vflags, 1);
                else if ((int64_t)f > hi - p) atomicMin(vflags + 1, e + 1);
            }
            p = min(max(p, (int64_t)0), nnz);
            hi = min(max(hi, p), nnz);
            if (lane == 0 && p > 0 && p < hi && __ldg(edge_vtx + p) <= __ldg(edge_vtx + p - 1)) ++start_desc;
        }
        int32_t cnt = 0, lo = 0;
        const int32_t f_e = (need_acc || orig) ? demand[e] : 0;
        if (panel_sel) {
            // selected rows (lazy operands, a few per launch): one warp walking
            // ~wlim/512 windows of a full row one after another is latency-
            // bound (~90 us per 100k-column row), so zero the row with
            // independent 16-byte stores, then scatter the members (int8 byte
            // stores / FP4 nibble atomicOr), PACK_UNROLL loads per lane in flight
            for (int64_t b = lane * 16; b < wlim; b += 32 * 16)
                *reinterpret_cast<uint4*>(row + b) = make_uint4(0, 0, 0, 0);
            __syncwarp();   // orders the zero stores before the other lanes' scatter
            const int64_t wcols = FP4 ? 2 * wlim : wlim;
            for (int64_t k0 = p + lane; k0 < hi; k0 += PACK_UNROLL * 32) {
                int32_t col[PACK_UNROLL];
                load_cols(col, k0, hi, edge_vtx, vnew);
#pragma unroll
                for (int u = 0; u < PACK_UNROLL; ++u) {
                    if (col[u] < 0) continue;
                    ++cnt;
                    lo += col[u] < K1;
                    if (col[u] < wcols) {
                        MHSK_CHECK(r < rows_pad && (FP4 ? col[u] / 2 : col[u]) < ld);
                        if constexpr (FP4)
                            atomicOr(reinterpret_cast<uint32_t*>(row) + (col[u] >> 3), 0x2u << (4 * (col[u] & 7)));
                        else
                            row[col[u]] = 1;
                    }
                    if (deg_acc) atomicAdd(deg_acc + col[u], 1);
                    need_update(col[u], f_e, false);
                }
            }
            p = hi;
        }
        for (int64_t w0 = panel_sel ? wlim : 0; w0 < wlim; w0 += PACK_WIN) {
            *reinterpret_cast<uint4*>(buf + lane * 16) = make_uint4(0, 0, 0, 0);
            __syncwarp();
            const int64_t c0 = FP4 ? 2 * w0 : w0;   // first column of the window
            while (p < hi) {
                const int64_t k = p + lane;
                const int32_t v = k < hi ? edge_vtx[k] : 0x7FFFFFFF;
                const int32_t col = k < hi ? (vnew ? vnew[v] : v) : 0x7FFFFFFF;
                const bool inwin = col < c0 + COLS_PER_WIN;      // dead members (-1) count as consumed
                const uint32_t out = ~__ballot_sync(0xffffffffu, inwin);
                const int first_out = out ? __ffs(out) - 1 : 32;
                if (lane < first_out && col >= 0) {
                    if constexpr (FP4) {
                        const int32_t o = (int32_t)(col - c0);
                        atomicOr(reinterpret_cast<uint32_t*>(buf) + (o >> 3), 0x2u << (4 * (o & 7)));
                    } else {
                        buf[col - w0] = 1;
                    }
                    ++cnt;
                    lo += col < K1;
                    if (deg_acc) atomicAdd(deg_acc + col, 1);
                    if (orig) need_update_orig(v, f_e);
                    else need_update(col, f_e, false);
                }
                p += first_out;
                if (first_out < 32) break;
            }
            __syncwarp();
            if (w0 + lane * 16 < width)
                *reinterpret_cast<uint4*>(row + w0 + lane * 16) = *reinterpret_cast<const uint4*>(buf + lane * 16);
            __syncwarp();
        }
        // members beyond the written columns: PACK_UNROLL per lane in flight
        // (the CSR stream is latency-bound: ncu puts ~55% of the stall
        // samples on these loads at four per lane)
        if (vflags && uni && !deg_acc && !vnew) {   // scan_members covered them
            if (lane == 0) cnt += (int32_t)(hi - p);
            p = hi;
        }
        if (orig) {   // original ids: an alive-bit test instead of the vnew gather
            for (int64_t k0 = p + lane; k0 < hi; k0 += PACK_UNROLL * 32) {
                int32_t v[PACK_UNROLL];
#pragma unroll
                for (int u = 0; u < PACK_UNROLL; ++u) {
                    const int64_t k = k0 + 32 * u;
                    v[u] = k < hi ? __ldg(edge_vtx + k) : -1;
                }
#pragma unroll
                for (int u = 0; u < PACK_UNROLL; ++u) {
                    const bool alive_v =
                        v[u] >= 0 && (!alive_bits || ((smaps ? s_alive[v[u] >> 5] : __ldg(alive_bits + (v[u] >> 5))) >>
                                                      (v[u] & 31)) & 1u);
                    if (alive_v) {
                        ++cnt;
                        need_update_orig(v[u], f_e);
                    }
                }
            }
            p = hi;
        }
        for (int64_t k0 = p + lane; k0 < hi; k0 += PACK_UNROLL * 32) {
            int32_t col[PACK_UNROLL];
            load_cols(col, k0, hi, edge_vtx, vnew);
#pragma unroll
            for (int u = 0; u < PACK_UNROLL; ++u) {
                if (col[u] >= 0) {
                    ++cnt;
                    if (deg_acc) atomicAdd(deg_acc + col[u], 1);
                    // L1-cached read: a stale (smaller) value only costs a redundant atomic
                    need_update(col[u], f_e, true);
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lo_out) {
            for (int o = 16; o > 0; o >>= 1) lo += __shfl_xor_sync(0xffffffffu, lo, o);
            if (lane == 0) lo_out[r] = lo;
        }
        if (lane == 0) {
            size_out[r] = cnt;
            dem_out[r] = demand[e];
        }
    }
    if (desc && lane == 0 && start_desc) atomicAdd(desc + 1, (unsigned long long)start_desc);
    if (smaps) {   // only the bits the global map lacks
        __syncthreads();
        for (int32_t i = threadIdx.x; i < map_words; i += blockDim.x) {
            const uint32_t mine = s_seen[i];
            if (mine && (mine & ~__ldcg(seen + i))) atomicOr(seen + i, mine);
        }
    }
}

// out[c][j] = in[src[j]][c] for c < rows_pad_out, j < ld_out (zero beyond
// n_cols_in / m_out); deg_out[c] = popcount of out row c (c < n_cols_in).
// CTA (4 warps) = 128 output rows (128 input columns); per step a 128 x 128
// tile: warp w bit-transposes input rows j0+32w.. with 128 ballots, expands
// the masks into a shared-memory tile, and the CTA stores the tile as full
// 128-byte lines.  Loads are full 128-byte lines too (one input row segment
// per lane).
constexpr int TP_WARPS = 4;
constexpr int TP_STRIDE = 144;  // smem row stride (bytes): 16B-aligned, spreads banks
constexpr int TP_CHUNK = 8192;  // input rows (output columns) per CTA of the split transpose

// FP4: both operands packed E2M1 (column c = nibble c & 1 of byte c / 2); an
// input row segment is 64 bytes, an output tile row 64 bytes (4 threads per
// row), and the output is written up to m_out rounded to 256 items.
template <bool FP4 = false>
__global__ void __launch_bounds__(TP_WARPS * 32)
transpose_pack(const int8_t* __restrict__ in, int64_t ld_in, const int32_t* __restrict__ src,
               int32_t m_out, int32_t n_cols_in, int8_t* __restrict__ out, int64_t ld_out,
               int32_t* __restrict__ deg_out, const int32_t* __restrict__ dev_nm = nullptr,
               int32_t* __restrict__ lo_out = nullptr, int64_t K1 = 0, int64_t j_chunk = 0,
               int64_t j_limit = -1, const uint8_t* __restrict__ panel_flags = nullptr) {
    mhsk::pdl_enter();
    __shared__ __align__(16) uint8_t tile[128 * TP_STRIDE];
    __shared__ int32_t degs[TP_WARPS][128];
    __shared__ int32_t los[TP_WARPS][128];
    // grid.y > 1: CTA (x, y) covers input rows [y * j_chunk, (y + 1) * j_chunk)
    // and adds its partial degrees atomically (deg_out / lo_out pre-zeroed)
    // j_limit >= 0: only output columns [0, j_limit) (the probe columns of the
    // lazy vertex operand).  panel_flags: only output rows of flagged 256-row
    // panels (the panels the probe pass left undecided).
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t c0 = (int64_t)blockIdx.x * 128;
    if (panel_flags && !panel_flags[c0 / 256]) return;
    constexpr int IPB = FP4 ? 2 : 1;   // items per byte
    int64_t width = ld_out * IPB;      // output columns (items)
    if (dev_nm) {   // device-resident sizes: output rows n = dev_nm[0], columns m = dev_nm[1]
        n_cols_in = dev_nm[0];
        m_out = dev_nm[1];
        if (c0 >= (int64_t)(n_cols_in + 255) / 256 * 256) return;
        width = FP4 ? min(ld_out * 2, (int64_t)(max(m_out, 1) + 255) / 256 * 256)
                    : min(ld_out, (int64_t)(max(m_out, 1) + 127) / 128 * 128);
    }
    // input columns at or beyond n_cols_in may be stale (written only up to
    // K_pad of the current size): read only blocks that start below it
    const bool cols_in_range = c0 < ld_in * IPB && c0 < n_cols_in;
    int32_t dacc[4] = {0, 0, 0, 0}, lacc[4] = {0, 0, 0, 0};
    const int64_t j_begin = gridDim.y > 1 ? (int64_t)blockIdx.y * j_chunk : 0;
    int64_t j_end = gridDim.y > 1 ? min(width, j_begin + j_chunk) : width;
    if (j_limit >= 0) j_end = min(j_end, j_limit);
    if (j_begin >= j_end) return;
    for (int64_t j0 = j_begin; j0 < j_end; j0 += 128) {
        const int64_t j = j0 + 32 * w + lane;
        uint32_t v[32 / IPB];
        if (cols_in_range && j < m_out) {
            const uint4* p = reinterpret_cast<const uint4*>(in + (int64_t)src[j] * ld_in + c0 / IPB);
#pragma unroll
            for (int q = 0; q < 8 / IPB; ++q) {
                const uint4 x = __ldg(p + q);
                v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 32 / IPB; ++q) v[q] = 0;
        }
        uint32_t mine[4] = {0, 0, 0, 0};
        if constexpr (FP4) {
            // nibbles -> one bit per column, then four warp-wide 32x32 bit
            // transposes (5 shuffle stages each) instead of 128 ballots
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t w = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) w |= compress_nibbles(v[4 * k + b]) << (8 * b);
                mine[k] = transpose32_warp(w, lane);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
                const uint32_t m = __ballot_sync(0xffffffffu, (v[c >> 2] >> (8 * (c & 3))) & 0xFFu);
                if (lane == (c & 31)) mine[c >> 5] = m;
            }
        }
        __syncthreads();  // previous tile fully stored
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            dacc[k] += __popc(mine[k]);
            if (j0 < K1) lacc[k] += __popc(mine[k]);
            if constexpr (FP4) {
                uint32_t e4[4];
                expand_mask_fp4(mine[k], e4);
                *reinterpret_cast<uint4*>(tile + (32 * k + lane) * TP_STRIDE + 16 * w) =
                    make_uint4(e4[0], e4[1], e4[2], e4[3]);
            } else {
                uint32_t e8[8];
                expand_mask(mine[k], e8);
                uint4* d = reinterpret_cast<uint4*>(tile + (32 * k + lane) * TP_STRIDE + 32 * w);
                d[0] = make_uint4(e8[0], e8[1], e8[2], e8[3]);
                d[1] = make_uint4(e8[4], e8[5], e8[6], e8[7]);
            }
        }
        __syncthreads();
        // 128 rows x 128 B (FP4: 64 B): 8 (4) threads per row
        constexpr int SEGS = 8 / IPB, ROWS_PER_PASS = 128 / SEGS;
#pragma unroll
        for (int pass = 0; pass < 128 / ROWS_PER_PASS; ++pass) {
            const int row = pass * ROWS_PER_PASS + threadIdx.x / SEGS, seg = threadIdx.x % SEGS;
            const uint4 x = *reinterpret_cast<const uint4*>(tile + row * TP_STRIDE + seg * 16);
            *reinterpret_cast<uint4*>(out + (c0 + row) * ld_out + j0 / IPB + seg * 16) = x;
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        degs[w][32 * k + lane] = dacc[k];
        los[w][32 * k + lane] = lacc[k];
    }
    __syncthreads();
    if (threadIdx.x < 128) {
        int32_t d = 0, l = 0;
#pragma unroll
        for (int q = 0; q < TP_WARPS; ++q) {
            d += degs[q][threadIdx.x];
            l += los[q][threadIdx.x];
        }
        const int64_t c = c0 + threadIdx.x;
        if (c < n_cols_in && deg_out) {
            if (gridDim.y > 1) {
                if (d) atomicAdd(deg_out + c, d);
                if (lo_out && l) atomicAdd(lo_out + c, l);
            } else {
                deg_out[c] = d;
                if (lo_out) lo_out[c] = l;
            }
        }
    }
}

// need[vnew[v]] = max demand over alive edges containing alive v.  Reads
// first, so an atomic is issued only when it can raise the value.  gate
// (optional): runs only if *gate != 0.
// min / max demand of the M (= *n_rows) edges eids[0..M) into f_range
// (pre-set to {INT_MAX-ish, 0}); equal => uniform demand (pack_rows_csr seen).
__global__ void demand_range(const int32_t* __restrict__ n_rows, const int32_t* __restrict__ eids,
                             const int32_t* __restrict__ demand, int32_t* __restrict__ f_range) {
    mhsk::pdl_enter();
    const int32_t M = *n_rows;
    int32_t lo = 0x7fffffff, hi = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < M; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = demand[eids[r]];
        lo = min(lo, f);
        hi = max(hi, f);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (threadIdx.x % 32 == 0 && lo <= hi) {
        atomicMin(f_range, lo);
        atomicMax(f_range + 1, hi);
    }
}

// Uniform demand only: need[j] = f if column j had a member (seen bit), else 0.
__global__ void need_from_seen(const int32_t* __restrict__ n_cols, const uint32_t* __restrict__ seen,
                               const int32_t* __restrict__ f_range, int32_t* __restrict__ need) {
    mhsk::pdl_enter();
    if (f_range[0] != f_range[1]) return;
    const int32_t f = f_range[1], K = *n_cols;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x)
        need[j] = (seen[j >> 5] >> (j & 31)) & 1u ? f : 0;
}

__global__ void need_from_csr(int32_t m, const int64_t* __restrict__ edge_ptr,
                              const int32_t* __restrict__ edge_vtx, const int32_t* __restrict__ demand,
                              const uint8_t* __restrict__ ealive, const int32_t* __restrict__ vnew,
                              int32_t* __restrict__ need, const int32_t* __restrict__ gate = nullptr,
                              const int32_t* __restrict__ skip_uniform = nullptr) {
    mhsk::pdl_enter();
    if (gate && *gate == 0) return;
    // f_range given: uniform demand is handled by the seen-map kernels
    if (skip_uniform && skip_uniform[0] == skip_uniform[1]) return;
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        if (!ealive[e]) continue;
        const int32_t f = demand[e];
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t r = vnew[edge_vtx[p]];
            if (r >= 0 && *((volatile int32_t*)(need + r)) < f) atomicMax(need + r, f);
        }
    }
}

// Lazy vertex operand: the edge phase deleted *n_del edges (flagged in
// edel); take them out of the degrees pack_rows_csr accumulated, and zero the
// need accumulator so need_from_csr (same gate) recomputes it over the
// survivors (a maximum cannot be decremented).  No-op when nothing was deleted.
__global__ void fix_deleted_edges(int32_t m, const int64_t* __restrict__ edge_ptr,
                                  const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ edel,
                                  const int32_t* __restrict__ vnew, int32_t* __restrict__ deg,
                                  int32_t* __restrict__ need, const int32_t* __restrict__ n_items,
                                  const int32_t* __restrict__ n_del) {
    mhsk::pdl_enter();
    if (*n_del == 0) return;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < *n_items; v += nth) need[v] = 0;
    const int64_t warp_global = tid / 32, nwarps = nth / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += nwarps) {
        if (!edel[e]) continue;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t r = vnew[edge_vtx[p]];
            if (r >= 0 && deg) atomicSub(deg + r, 1);
        }
    }
}

// X_V's probe columns straight from the CSR (lazy vertex operand): column j <
// K1 of X_V is the edge in X_E row src[j] (the j-th survivor of the edge
// phase), i.e. edge eids[src[j]]; each of its alive members v sets X_V row
// vnew[v] (nullptr: v) at column j.  The same bits as transposing the full
// X_E rows of those edges, without packing them: one warp per column, its
// ~1e3 members scattered with 32-bit atomicOr (FP4 nibbles) / byte stores.
// Bracketed by prefix_cols<false> (before) and prefix_cols<true> (lo, after).
// The speculative vertex probe runs this before the fused validation has
// been checked: offsets are clamped into [0, *nnz_ptr] and rows outside
// [0, n_rows) are skipped, so a malformed CSR is never read or written out of
// bounds (the call then fails validation).
template <bool FP4>
__global__ void probe_cols_csr(const int32_t* __restrict__ m_cols, int64_t K1, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ eids, const int64_t* __restrict__ edge_ptr,
                               const int32_t* __restrict__ edge_vtx, const int32_t* __restrict__ vnew,
                               int8_t* __restrict__ X, int64_t ld, int32_t n_rows,
                               const int64_t* __restrict__ nnz_ptr) {
    mhsk::pdl_enter();
    const int64_t J = min((int64_t)*m_cols, K1);
    const int64_t nnz = max(*nnz_ptr, (int64_t)0);
    const int lane = threadIdx.x % 32;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; j < J; j += nw) {
        const int32_t e = eids[src[j]];
        const int64_t lo = min(max(edge_ptr[e], (int64_t)0), nnz), hi = min(max(edge_ptr[e + 1], lo), nnz);
        for (int64_t p = lo + lane; p < hi; p += 32) {
            const int32_t v = __ldg(edge_vtx + p);
            if (v < 0 || (v >= n_rows && !vnew)) continue;
            const int32_t r = vnew ? __ldg(vnew + v) : v;
            if (r < 0 || r >= n_rows) continue;
            if constexpr (FP4)
                atomicOr(reinterpret_cast<uint32_t*>(X + (int64_t)r * ld) + (j >> 3), 0x2u << (4 * (j & 7)));
            else
                X[(int64_t)r * ld + j] = 1;
        }
    }
}

// The first `bytes` (a multiple of 16) of rows [0, rows) of X: zero (COUNT =
// false), or their set bits into cnt[r] for r < *n_rows (COUNT = true; one
// bit per item in both operand formats).  One warp per row, 16-byte accesses.
template <bool COUNT>
__global__ void prefix_cols(int8_t* __restrict__ X, int64_t ld, int64_t bytes, int64_t rows,
                            const int32_t* __restrict__ n_rows, int32_t* __restrict__ cnt) {
    mhsk::pdl_enter();
    const int lane = threadIdx.x % 32;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    if (COUNT) rows = min(rows, (int64_t)*n_rows);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += nw) {
        uint4* row = reinterpret_cast<uint4*>(X + r * ld);
        int32_t c = 0;
        for (int64_t q = lane; q < bytes / 16; q += 32) {
            if constexpr (COUNT) {
                const uint4 x = row[q];
                c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
            } else {
                row[q] = make_uint4(0, 0, 0, 0);
            }
        }
        if constexpr (COUNT) {
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) cnt[r] = c;
        }
    }
}

// Panels (256 rows) of the lazy vertex operand that must be packed in full:
// both panels of every tile the probe pass marked (this rank's share: tile t
// of pair p is list entry begin + (p + t * pairs) * stride) and the panels of
// every listed candidate pair (verify_candidates reads both rows).
__global__ void needed_panels(const uint32_t* __restrict__ needed, int32_t pairs, int32_t words,
                              const uint32_t* __restrict__ tiles, int32_t begin, int32_t count, int32_t stride,
                              const int4* __restrict__ cand, const int32_t* __restrict__ cand_count,
                              int32_t cand_cap, uint8_t* __restrict__ flags, int32_t bn,
                              int32_t* __restrict__ any = nullptr, uint8_t* __restrict__ row_flags = nullptr,
                              const int32_t* __restrict__ cand_skip = nullptr) {
    mhsk::pdl_enter();
    if (cand_skip && *cand_skip) cand = nullptr;   // candidates decided without the operand
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = tid; q < (int64_t)pairs * words; q += nth) {
        uint32_t bits = needed[q];
        const int32_t p = (int32_t)(q / words), w = (int32_t)(q % words);
        while (bits) {
            const int32_t t = w * 32 + __ffs((int)bits) - 1;
            bits &= bits - 1;
            const int64_t it = p + (int64_t)t * pairs;
            if (it >= count) continue;
            const uint32_t pj = tiles[begin + it * stride];
            const int32_t J = (int32_t)(pj >> 16);
            flags[pj & 0xFFFF] = 1;   // A panel (256 rows); B panel: rows [J * bn, J * bn + bn)
            for (int32_t f = J * bn / 256; f <= (J * bn + bn - 1) / 256; ++f) flags[f] = 1;
            if (any) *any = 1;
        }
    }
    if (cand) {
        const int32_t nc = min(*cand_count, cand_cap);
        for (int64_t q = tid; q < nc; q += nth) {
            const int4 e = cand[q];
            if (e.x < 0) continue;
            if (row_flags) {   // rows packed one by one (pack_rows_csr row_sel)
                row_flags[e.x] = 1;
                row_flags[e.y] = 1;
            } else {
                flags[e.x / 256] = 1;
                flags[e.y / 256] = 1;
            }
            if (any) *any = 1;
        }
    }
}

// Lazy edge operand: rows of X_E held only in their probe columns are
// packed in full per 256-row panel; panel state 0 = probe columns only,
// 1 = to pack, 2 = full.
// Flag every panel (when *any != 0: a vertex panel must be transposed in full,
// which reads X_E columns from every row).
__global__ void flag_all_panels(const int32_t* __restrict__ any, uint8_t* __restrict__ state, int32_t npanels) {
    mhsk::pdl_enter();
    if (*any == 0) return;
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < npanels; q += gridDim.x * blockDim.x)
        if (state[q] == 0) state[q] = 1;
}
__global__ void mark_packed_panels(uint8_t* __restrict__ state, int32_t npanels) {
    mhsk::pdl_enter();
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < npanels; q += gridDim.x * blockDim.x)
        if (state[q] == 1) state[q] = 2;
}

}  // namespace k
}  // namespace mhsk

// ------------------------------------------------------ incremental rounds
// After round 1, a surviving edge can only gain a deleter i that lost vertices
// (f_i - s_i + c_ij rises only when i loses a vertex outside j), and a
// surviving vertex can only gain dominators if its own incidence set shrank;
// deletions elsewhere only remove superseders / dominators.  So round r > 1
// needs the rectangle "affected items x all items" (gram_tc2_kernel<.., true>).
namespace mhsk {
namespace k {

// eaff[e] = alive e contains a vertex deleted in the last vertex phase
// (n_del: vertices deleted by that phase; none -> no edge is affected, and
// the CSR is not read)
__global__ void mark_affected_edges(int32_t m, const int64_t* __restrict__ edge_ptr,
                                    const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ ealive,
                                    const uint8_t* __restrict__ vdel, uint8_t* __restrict__ eaff,
                                    const int32_t* __restrict__ n_del = nullptr) {
    mhsk::pdl_enter();
    if (n_del && *n_del == 0) {
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
            eaff[e] = 0;
        return;
    }
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        bool hit = false;
        if (ealive[e])
            for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1] && !hit; p += 32) hit = vdel[edge_vtx[p]];
        hit = __any_sync(0xffffffffu, hit);
        if (lane == 0) eaff[e] = hit;
    }
}

// ---------------------------------------------------------------------------
// Member passes of the later rounds with the per-member test against an
// n-bit map of ORIGINAL vertex ids held in shared memory (a block loads it
// once): no vnew / vdel / vflag gather per member, and each lane keeps
// MEMBER_UNROLL independent member loads in flight.  The maps (<= 96 KB,
// n <= MAP_SMEM_BITS; the host falls back to the gather kernels above) are
// built by bits_from_bytes / per-kernel set-up.
constexpr int MEMBER_UNROLL = 8;
constexpr int64_t MAP_SMEM_BITS = (int64_t)96 * 1024 * 8;

// bits[w] bit b = bytes[32 w + b] != 0 (one warp per word; n bits)
__global__ void bits_from_bytes(const uint8_t* __restrict__ bytes, int32_t n, uint32_t* __restrict__ bits) {
    mhsk::pdl_enter();
    const int lane = threadIdx.x % 32;
    const int64_t words = (n + 31) / 32;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; w < words;
         w += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t i = 32 * w + lane;
        const uint32_t b = __ballot_sync(0xffffffffu, i < n && bytes[i] != 0);
        if (lane == 0) bits[w] = b;
    }
}

__device__ __forceinline__ void load_map(uint32_t* __restrict__ smap, const uint32_t* __restrict__ g, int32_t n) {
    for (int32_t w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) smap[w] = g[w];
    __syncthreads();
}

// eaff[e] = alive edge e holds a vertex deleted in the last vertex phase
// (vdel_bits: those vertices by original id).  *n_del == 0: all zero.
__global__ void mark_affected_edges_map(int32_t m, int32_t n, const int64_t* __restrict__ edge_ptr,
                                        const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ ealive,
                                        const uint32_t* __restrict__ vdel_bits, uint8_t* __restrict__ eaff,
                                        const int32_t* __restrict__ n_del) {
    mhsk::pdl_enter();
    extern __shared__ uint32_t smap[];
    if (*n_del == 0) {
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
            eaff[e] = 0;
        return;
    }
    load_map(smap, vdel_bits, n);
    const int lane = threadIdx.x % 32;
    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; e < m;
         e += (int64_t)gridDim.x * blockDim.x / 32) {
        bool hit = false;
        if (ealive[e]) {   // warp-uniform loop (the early exit votes with every lane)
            const int64_t hi = edge_ptr[e + 1];
            for (int64_t base = edge_ptr[e]; base < hi; base += 32 * MEMBER_UNROLL) {
                int32_t v[MEMBER_UNROLL];
#pragma unroll
                for (int u = 0; u < MEMBER_UNROLL; ++u) {
                    const int64_t k = base + 32 * u + lane;
                    v[u] = k < hi ? __ldg(edge_vtx + k) : -1;
                }
#pragma unroll
                for (int u = 0; u < MEMBER_UNROLL; ++u)
                    hit |= v[u] >= 0 && ((smap[v[u] >> 5] >> (v[u] & 31)) & 1u);
                if (__any_sync(0xffffffffu, hit)) break;
            }
        }
        hit = __any_sync(0xffffffffu, hit);
        if (lane == 0) eaff[e] = hit;
    }
}

// need over the alive edges in [e_lo, e_hi), two-tier: with fmax the
// largest demand among them (f_range[1]), seen[v] |= v is a member of an
// alive edge with demand fmax (per-block shared copy OR-ed out, only missing
// bits), and need_low[v] = max demand of v's other alive edges (atomicMax,
// original ids; rare: instances are near-uniform, f = min(alpha, |e|)).
// Then need_v = seen ? fmax : need_low (need_from_seen_ids).  Gates: *gate
// == 0 (nothing deleted) or *full (every alive vertex already seen: need =
// fmax everywhere) skip the launch.
__global__ void seen_alive_edges(int32_t n, int32_t e_lo, int32_t e_hi, const int64_t* __restrict__ edge_ptr,
                                 const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ ealive,
                                 const int32_t* __restrict__ demand, const int32_t* __restrict__ f_range,
                                 uint32_t* __restrict__ seen, int32_t* __restrict__ need_low,
                                 const int32_t* __restrict__ gate, const int32_t* __restrict__ full) {
    mhsk::pdl_enter();
    extern __shared__ uint32_t smap[];
    if (*gate == 0 || (full && *full)) return;
    const int32_t fmax = f_range[1];
    const int32_t words = (n + 31) / 32;
    for (int32_t w = threadIdx.x; w < words; w += blockDim.x) smap[w] = 0;
    __syncthreads();
    const int lane = threadIdx.x % 32;
    for (int64_t e = e_lo + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; e < e_hi;
         e += (int64_t)gridDim.x * blockDim.x / 32) {
        if (!ealive[e]) continue;
        const int32_t f = demand[e];
        const int64_t hi = edge_ptr[e + 1];
        for (int64_t k0 = edge_ptr[e] + lane; k0 < hi; k0 += 32 * MEMBER_UNROLL) {
            int32_t v[MEMBER_UNROLL];
#pragma unroll
            for (int u = 0; u < MEMBER_UNROLL; ++u) v[u] = k0 + 32 * u < hi ? __ldg(edge_vtx + k0 + 32 * u) : -1;
            if (f == fmax) {
#pragma unroll
                for (int u = 0; u < MEMBER_UNROLL; ++u)
                    if (v[u] >= 0 && !((smap[v[u] >> 5] >> (v[u] & 31)) & 1u))
                        atomicOr(smap + (v[u] >> 5), 1u << (v[u] & 31));
            } else {
#pragma unroll
                for (int u = 0; u < MEMBER_UNROLL; ++u)
                    if (v[u] >= 0 && __ldcg(need_low + v[u]) < f) atomicMax(need_low + v[u], f);
            }
        }
    }
    __syncthreads();
    for (int32_t w = threadIdx.x; w < words; w += blockDim.x) {
        const uint32_t mine = smap[w];
        if (mine && (mine & ~__ldcg(seen + w))) atomicOr(seen + w, mine);
    }
}

// *missing (pre-zeroed) = some alive vertex (valive, original ids) lacks
// its seen bit; grid-wide, gated like seen_alive_edges
__global__ void seen_misses_alive(const uint32_t* __restrict__ seen, const uint8_t* __restrict__ valive, int32_t n,
                                  int32_t* __restrict__ missing, const int32_t* __restrict__ gate) {
    mhsk::pdl_enter();
    if (*gate == 0) return;
    bool miss = false;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        miss |= valive[v] && !((seen[v >> 5] >> (v & 31)) & 1u);
    if (__any_sync(0xffffffffu, miss) && threadIdx.x % 32 == 0) atomicExch(missing, 1);
}

// *full = !*missing (the second part's gate)
__global__ void seen_full_from_missing(const int32_t* __restrict__ missing, int32_t* __restrict__ full) {
    mhsk::pdl_enter();
    *full = *missing == 0;
}

// need[j] = seen[vids[j]] ? fmax : need_low[vids[j]] for the K compact
// vertices, gated like seen_alive_edges
__global__ void need_from_seen_ids(const int32_t* __restrict__ n_cols, const int32_t* __restrict__ vids,
                                   const uint32_t* __restrict__ seen, const int32_t* __restrict__ need_low,
                                   const int32_t* __restrict__ f_range, int32_t* __restrict__ need,
                                   const int32_t* __restrict__ gate = nullptr) {
    mhsk::pdl_enter();
    if (gate && *gate == 0) return;
    const int32_t f = f_range[1], K = *n_cols;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = vids[j];
        need[j] = (seen[v >> 5] >> (v & 31)) & 1u ? f : need_low[v];
    }
}

// vaff[v] = 1 for the alive members of edges deleted in the last edge phase
__global__ void mark_affected_vertices(int32_t m, const int64_t* __restrict__ edge_ptr,
                                       const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ edel,
                                       const uint8_t* __restrict__ valive, uint8_t* __restrict__ vaff) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        if (!edel[e]) continue;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t v = edge_vtx[p];
            if (valive[v]) vaff[v] = 1;
        }
    }
}

// out[p] = map[ids[p]] for p < *count
__global__ void gather_ids(const int32_t* __restrict__ ids, const int32_t* __restrict__ map,
                           int32_t* __restrict__ out, const int32_t* __restrict__ count) {
    mhsk::pdl_enter();
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < *count) out[p] = map[ids[p]];
}

// dst row p = src row rows[p] (first `width` bytes, ld bytes apart) for
// p < count, zero rows up to the 256-row pad; exits unless *enable.
__global__ void gather_rows(const int8_t* __restrict__ src, int64_t ld, const int32_t* __restrict__ rows,
                            const int32_t* __restrict__ count, const int32_t* __restrict__ width_items,
                            int8_t* __restrict__ dst, const int32_t* __restrict__ enable, bool fp4 = false) {
    mhsk::pdl_enter();
    if (enable && *enable == 0) return;
    const int32_t cnt = *count;
    const int64_t rows_pad = (int64_t)(cnt + 255) / 256 * 256;
    const int64_t width = fp4 ? min(ld, (int64_t)(max(*width_items, 1) + 255) / 256 * 128)
                              : min(ld, (int64_t)(max(*width_items, 1) + 127) / 128 * 128);
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + w; p < rows_pad;
         p += (int64_t)gridDim.x * (blockDim.x / 32)) {
        uint4* d = reinterpret_cast<uint4*>(dst + p * ld);
        if (p < cnt) {
            const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)rows[p] * ld);
            for (int64_t b = lane; b < width / 16; b += 32) d[b] = __ldg(s + b);
        } else {
            for (int64_t b = lane; b < width / 16; b += 32) d[b] = make_uint4(0, 0, 0, 0);
        }
    }
}

// Incremental vertex phase: triangle or rectangle?  flags[0] = triangle,
// flags[1] = rectangle (rectangle iff 2 * affected <= alive).
// rectangle iff affected * den <= alive * num (no probe: 1/2 of the items;
// probed triangle: probe columns / (2 K), see kernelize_fast)
__global__ void choose_phase_kernel(const int32_t* __restrict__ affected, const int32_t* __restrict__ alive,
                                    int32_t* __restrict__ flags, int32_t num, int32_t den) {
    mhsk::pdl_enter();
    const bool rect = (long long)*affected * den <= (long long)*alive * num;
    flags[0] = !rect;
    flags[1] = rect;
}

__global__ void copy_i32(const int32_t* __restrict__ src, int32_t* __restrict__ dst) {
    mhsk::pdl_enter(); *dst = *src; }

}  // namespace k
}  // namespace mhsk

// ------------------------------------------------------- block-sparse mode
// For structured instances (e.g. interval "train" hypergraphs) whose
// incidence matrix is banded once edges are ordered by their first vertex,
// every 256-row panel of an operand carries a bitmask of the 128-column
// k-blocks it touches.  Packing writes only those blocks and the Gram kernel
// multiplies only the k-blocks two panels share -- exact, because a k-block
// that is zero in either panel contributes nothing to any count.
namespace mhsk {
namespace k {

// first alive-agnostic vertex of each edge (sort key; empty edges -> n)
__global__ void edge_first_vertex(int32_t m, int32_t n, const int64_t* __restrict__ edge_ptr,
                                  const int32_t* __restrict__ edge_vtx, int32_t* __restrict__ key,
                                  int32_t* __restrict__ ids) {
    mhsk::pdl_enter();
    const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < m) {
        key[e] = edge_ptr[e + 1] > edge_ptr[e] ? edge_vtx[edge_ptr[e]] : n;
        ids[e] = e;
    }
}

__device__ __forceinline__ void or_bits_warp(unsigned long long* __restrict__ mask, int64_t word, uint64_t bit,
                                             bool active) {
    // combine equal words within the warp, one atomic per distinct word
    const uint32_t act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const uint32_t peers = __match_any_sync(act, word);
    const uint32_t lo = __reduce_or_sync(peers, (uint32_t)bit);
    const uint32_t hi = __reduce_or_sync(peers, (uint32_t)(bit >> 32));
    if ((threadIdx.x % 32) == (uint32_t)(__ffs(peers) - 1))
        atomicOr(mask + word, ((unsigned long long)hi << 32) | lo);
}

// mask_E: rows r < M (edge eids[r]) x 128-column blocks of vnew[v]
__global__ void mask_rows_csr(int32_t M, const int32_t* __restrict__ eids, const int64_t* __restrict__ edge_ptr,
                              const int32_t* __restrict__ edge_vtx, const int32_t* __restrict__ vnew,
                              unsigned long long* __restrict__ mask, int32_t words,
                              const int32_t* __restrict__ dev_m = nullptr) {
    mhsk::pdl_enter();
    if (dev_m) M = min(M, *dev_m);
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t r = warp_global; r < M; r += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int32_t e = eids[r];
        for (int64_t p0 = edge_ptr[e]; p0 < edge_ptr[e + 1]; p0 += 32) {
            const int64_t p = p0 + lane;
            const int32_t c = p < edge_ptr[e + 1] ? vnew[edge_vtx[p]] : -1;
            const int32_t b = c >> 7;
            or_bits_warp(mask, (r >> 8) * words + (b >> 6), 1ull << (b & 63), c >= 0);
        }
    }
}

// mask_V: for each surviving X_E row r (col_of[r] >= 0 is its X_V column),
// the 256-vertex panels of its alive members get column block col_of[r] >> 7
__global__ void mask_cols_csr(int32_t M, const int32_t* __restrict__ eids, const int32_t* __restrict__ col_of,
                              const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                              const int32_t* __restrict__ vnew, unsigned long long* __restrict__ mask,
                              int32_t words, const int32_t* __restrict__ dev_m = nullptr) {
    mhsk::pdl_enter();
    if (dev_m) M = min(M, *dev_m);
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t r = warp_global; r < M; r += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int32_t j = col_of[r];
        if (j < 0) continue;
        const int32_t b = j >> 7;
        const int32_t e = eids[r];
        for (int64_t p0 = edge_ptr[e]; p0 < edge_ptr[e + 1]; p0 += 32) {
            const int64_t p = p0 + lane;
            const int32_t v = p < edge_ptr[e + 1] ? vnew[edge_vtx[p]] : -1;
            or_bits_warp(mask, (int64_t)(v >> 8) * words + (b >> 6), 1ull << (b & 63), v >= 0);
        }
    }
}

// Sparse X_E pack: row r of panel P writes only the 128-byte blocks set in
// mask[P] (zeros + its members); rows M..rows_pad-1 write zeros there.  Also
// s_r, f_r, and *infeasible |= (s_r < f_r).
__global__ void __launch_bounds__(PACK_WARPS * 32)
pack_rows_sparse(int32_t M, int32_t rows_pad, const int32_t* __restrict__ eids,
                 const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                 const int32_t* __restrict__ demand, const int32_t* __restrict__ vnew,
                 int8_t* __restrict__ X, int64_t ld, const unsigned long long* __restrict__ mask, int32_t words,
                 int32_t* __restrict__ size_out, int32_t* __restrict__ dem_out, int32_t* __restrict__ infeasible,
                 const int32_t* __restrict__ dev_m = nullptr) {
    mhsk::pdl_enter();
    __shared__ __align__(16) uint8_t win[PACK_WARPS][512];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* buf = win[w];
    if (dev_m) {   // device-resident row count: rows beyond its 256-row pad are never read
        M = min(M, *dev_m);
        rows_pad = min(rows_pad, (M + 255) / 256 * 256);
    }
    for (int64_t r = (int64_t)blockIdx.x * PACK_WARPS + w; r < rows_pad; r += (int64_t)gridDim.x * PACK_WARPS) {
        int8_t* row = X + r * ld;
        const unsigned long long* pm = mask + (r >> 8) * words;
        const bool live = r < M;
        int64_t p = 0, hi = 0;
        int32_t e = -1;
        if (live) {
            e = eids[r];
            p = edge_ptr[e];
            hi = edge_ptr[e + 1];
        }
        int32_t cnt = 0;
        int32_t wi = 0;
        unsigned long long cur = words ? pm[0] : 0ull;
        for (;;) {
            // next (up to) 4 set blocks
            int32_t blk[4] = {-1, -1, -1, -1};
            int nb = 0;
            while (nb < 4) {
                while (!cur && ++wi < words) cur = pm[wi];
                if (!cur) break;
                blk[nb++] = wi * 64 + __ffsll(cur) - 1;
                cur &= cur - 1;
            }
            if (nb == 0) break;
            *reinterpret_cast<uint4*>(buf + lane * 16) = make_uint4(0, 0, 0, 0);
            __syncwarp();
            const int32_t last = blk[nb - 1];
            while (live && p < hi) {
                const int64_t k = p + lane;
                const int32_t col = k < hi ? vnew[edge_vtx[k]] : 0x7FFFFFFF;
                const int32_t b = col >= 0 ? col >> 7 : -1;
                const bool inwin = col < 0 || b <= last;
                const uint32_t out = ~__ballot_sync(0xffffffffu, inwin);
                const int first_out = out ? __ffs(out) - 1 : 32;
                if (lane < first_out && col >= 0) {
                    const int s = b == blk[0] ? 0 : b == blk[1] ? 1 : b == blk[2] ? 2 : 3;
                    buf[s * 128 + (col & 127)] = 1;
                    ++cnt;
                }
                p += first_out;
                if (first_out < 32) break;
            }
            __syncwarp();
            const int s = lane / 8;
            if (s < nb)
                *reinterpret_cast<uint4*>(row + (int64_t)blk[s] * 128 + (lane % 8) * 16) =
                    *reinterpret_cast<const uint4*>(buf + lane * 16);
            __syncwarp();
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (live && lane == 0) {
            size_out[r] = cnt;
            dem_out[r] = demand[e];
            if (cnt < demand[e]) atomicExch(infeasible, 1);
        }
    }
}

// Sparse transpose: like transpose_pack, but output row block c0 visits only
// the column blocks set in maskV[c0 >> 8], and reads an X_E block only if
// that row panel's maskE has it (unwritten blocks are never read).
__global__ void __launch_bounds__(TP_WARPS * 32)
transpose_sparse(const int8_t* __restrict__ in, int64_t ld_in, const int32_t* __restrict__ src,
                 const unsigned long long* __restrict__ maskE, int32_t words_e,
                 const unsigned long long* __restrict__ maskV, int32_t words_v,
                 int8_t* __restrict__ out, int64_t ld_out, int32_t* __restrict__ deg_out,
                 const int32_t* __restrict__ dev_nm) {
    mhsk::pdl_enter();
    __shared__ __align__(16) uint8_t tile[128 * TP_STRIDE];
    __shared__ int32_t degs[TP_WARPS][128];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t c0 = (int64_t)blockIdx.x * 128;
    const int32_t n_cols_in = dev_nm[0], m_out = dev_nm[1];
    if (c0 >= (int64_t)(n_cols_in + 255) / 256 * 256) return;
    const bool cols_in_range = c0 < ld_in && c0 < n_cols_in;
    const int32_t cb = (int32_t)(c0 >> 7);
    const unsigned long long* pm = maskV + (c0 >> 8) * words_v;
    int32_t dacc[4] = {0, 0, 0, 0};
    for (int32_t wi = 0; wi < words_v; ++wi) {
        for (unsigned long long cur = pm[wi]; cur; cur &= cur - 1) {
            const int64_t j0 = (int64_t)(wi * 64 + __ffsll(cur) - 1) * 128;
            const int64_t j = j0 + 32 * w + lane;
            uint32_t v[32];
            bool load = cols_in_range && j < m_out;
            int32_t srow = 0;
            if (load) {
                srow = src[j];
                load = (maskE[(srow >> 8) * words_e + (cb >> 6)] >> (cb & 63)) & 1ull;
            }
            if (load) {
                const uint4* pp = reinterpret_cast<const uint4*>(in + (int64_t)srow * ld_in + c0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 x = __ldg(pp + q);
                    v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] = 0;
            }
            uint32_t mine[4] = {0, 0, 0, 0};
#pragma unroll
            for (int c = 0; c < 128; ++c) {
                const uint32_t m = __ballot_sync(0xffffffffu, (v[c >> 2] >> (8 * (c & 3))) & 0xFFu);
                if (lane == (c & 31)) mine[c >> 5] = m;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                dacc[k] += __popc(mine[k]);
                uint32_t e8[8];
                expand_mask(mine[k], e8);
                uint4* d = reinterpret_cast<uint4*>(tile + (32 * k + lane) * TP_STRIDE + 32 * w);
                d[0] = make_uint4(e8[0], e8[1], e8[2], e8[3]);
                d[1] = make_uint4(e8[4], e8[5], e8[6], e8[7]);
            }
            __syncthreads();
#pragma unroll
            for (int pass = 0; pass < 8; ++pass) {
                const int row = pass * 16 + threadIdx.x / 8, seg = threadIdx.x % 8;
                const uint4 x = *reinterpret_cast<const uint4*>(tile + row * TP_STRIDE + seg * 16);
                *reinterpret_cast<uint4*>(out + (c0 + row) * ld_out + j0 + seg * 16) = x;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) degs[w][32 * k + lane] = dacc[k];
    __syncthreads();
    if (threadIdx.x < 128) {
        int32_t d = 0;
#pragma unroll
        for (int q = 0; q < TP_WARPS; ++q) d += degs[q][threadIdx.x];
        const int64_t c = c0 + threadIdx.x;
        if (c < n_cols_in) deg_out[c] = d;
    }
}

}  // namespace k
}  // namespace mhsk

// ------------------------------------------------ component ordering (sparse)
// Label propagation: vlabel = min vertex id of its connected component in the
// bipartite incidence graph, elabel = that of its edge.  Sorting vertices by
// (component, id) and edges by (component, first vertex position) makes a
// hypergraph of many small components block-diagonal.
namespace mhsk {
namespace k {

__global__ void lp_init(int32_t n, int32_t* __restrict__ vlabel) {
    mhsk::pdl_enter();
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) vlabel[v] = v;
}

// elabel[e] = min label of its members; members take min(label, elabel[e]).
__global__ void lp_step(int32_t m, const int64_t* __restrict__ edge_ptr, const int32_t* __restrict__ edge_vtx,
                        int32_t* __restrict__ vlabel, int32_t* __restrict__ elabel, int32_t* __restrict__ changed) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        int32_t lab = 0x7FFFFFFF;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) lab = min(lab, vlabel[edge_vtx[p]]);
        for (int o = 16; o > 0; o >>= 1) lab = min(lab, __shfl_xor_sync(0xffffffffu, lab, o));
        if (lane == 0) elabel[e] = lab;
        bool ch = false;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) {
            const int32_t v = edge_vtx[p];
            if (vlabel[v] > lab && atomicMin(vlabel + v, lab) > lab) ch = true;
        }
        if (__any_sync(0xffffffffu, ch) && lane == 0) atomicExch(changed, 1);
    }
}

// radix-sort keys (the sort is stable, so ties keep index order):
// vertices by component label -> (component, id) order
__global__ void vertex_keys(int32_t n, const int32_t* __restrict__ vlabel, int32_t* __restrict__ key,
                            int32_t* __restrict__ ids) {
    mhsk::pdl_enter();
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) {
        key[v] = vlabel[v];
        ids[v] = v;
    }
}

__global__ void invert_perm(int32_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ pos) {
    mhsk::pdl_enter();
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) pos[perm[k]] = k;
}

// edges by the position of their first member in the vertex order: the
// members of an edge share one component, whose vertices are contiguous, so
// this groups edges by component (empty edges, key n, go last)
__global__ void edge_keys(int32_t m, int32_t n, const int64_t* __restrict__ edge_ptr,
                          const int32_t* __restrict__ edge_vtx, const int32_t* __restrict__ vpos,
                          int32_t* __restrict__ key, int32_t* __restrict__ ids) {
    mhsk::pdl_enter();
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        int32_t first = n;
        for (int64_t p = edge_ptr[e] + lane; p < edge_ptr[e + 1]; p += 32) first = min(first, vpos[edge_vtx[p]]);
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        if (lane == 0) {
            key[e] = first;
            ids[e] = (int32_t)e;
        }
    }
}

// number of set bits in a mask array (occupancy of the block-sparse layout)
__global__ void popcount_u64(const unsigned long long* __restrict__ a, int64_t n,
                             unsigned long long* __restrict__ total) {
    mhsk::pdl_enter();
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += __popcll(a[i]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x % 32 == 0 && s) atomicAdd(total, s);
}

}  // namespace k
}  // namespace mhsk
