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

constexpr int SCAN_BLOCK = 1024;   // items per block of the compaction scan

// ---------------------------------------------------------------- compaction
// Pass 1: number of alive items per block (warp ballot + popc, block sum).
__global__ void count_alive(const uint8_t* __restrict__ alive, int32_t n, int32_t* __restrict__ block_counts) {
    __shared__ int32_t warp_sums[SCAN_BLOCK / 32];
    const int32_t idx = blockIdx.x * SCAN_BLOCK + threadIdx.x;
    const bool a = idx < n && alive[idx];
    const uint32_t b = __ballot_sync(0xffffffffu, a);
    if (threadIdx.x % 32 == 0) warp_sums[threadIdx.x / 32] = __popc(b);
    __syncthreads();
    if (threadIdx.x < 32) {
        int32_t v = warp_sums[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) block_counts[blockIdx.x] = v;
    }
}

// Pass 2 (one block): exclusive scan of the block counts; total -> *total.
__global__ void scan_block_counts(int32_t* __restrict__ block_counts, int32_t nblocks, int32_t* __restrict__ total) {
    __shared__ int32_t carry;
    __shared__ int32_t warp_sums[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int32_t base = 0; base < nblocks; base += blockDim.x) {
        const int32_t idx = base + threadIdx.x;
        int32_t v = idx < nblocks ? block_counts[idx] : 0;
        // inclusive warp scan
        const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t s = lane < (int)(blockDim.x / 32) ? warp_sums[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;   // inclusive prefix of warp totals
        }
        __syncthreads();
        const int32_t excl = carry + (w ? warp_sums[w - 1] : 0) + x - v;
        if (idx < nblocks) block_counts[idx] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// Pass 3: new_id[idx] = compacted position (or -1), ids[pos] = idx.
__global__ void scatter_alive(const uint8_t* __restrict__ alive, int32_t n, const int32_t* __restrict__ block_offsets,
                              int32_t* __restrict__ new_id, int32_t* __restrict__ ids) {
    __shared__ int32_t warp_offs[SCAN_BLOCK / 32];
    const int32_t idx = blockIdx.x * SCAN_BLOCK + threadIdx.x;
    const bool a = idx < n && alive[idx];
    const uint32_t b = __ballot_sync(0xffffffffu, a);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    if (lane == 0) warp_offs[w] = __popc(b);
    __syncthreads();
    if (w == 0) {
        int32_t s = warp_offs[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_offs[lane] = s - warp_offs[lane];  // exclusive
    }
    __syncthreads();
    if (idx < n) {
        const int32_t pos = block_offsets[blockIdx.x] + warp_offs[w] + __popc(b & ((1u << lane) - 1u));
        new_id[idx] = a ? pos : -1;
        if (a) ids[pos] = idx;
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
                             uint8_t* __restrict__ keep_out, int32_t* __restrict__ deleted) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    bool del = false;
    if (r < count) {
        if constexpr (VERTEX) del = need[r] == 0 || hits[r] >= need[r];
        else del = hits[r] > 0;
        if (keep_out) keep_out[r] = del ? 0 : 1;
        if (del && alive) alive[ids[r]] = 0;
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
    if (*first_infeasible != 0x7FFFFFFF) return;
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const bool f = v < n && forced[v];
    if (f) valive[v] = 0;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (threadIdx.x % 32 == 0 && b) atomicAdd(n_forced, __popc(b));
}

}  // namespace k
}  // namespace mhsk
