// gram_tc.cuh -- co-occurrence Gram product X.X^T on the 5th-gen tensor cores
// (tcgen05 kind::i8, int32 accumulators in TMEM) with the rule predicates
// fused into the epilogue.  Replaces _edge_intersections/_vertex_intersections
// + the pair loops of par_reduce_edges/par_reduce_vertices
// (pkg/src/mhskernel/parallel.py:52-161).  The M x M count matrix is never
// written: each tile's counts go TMEM -> registers -> predicates -> one
// atomic per item with a non-zero deleter count.
//
// X is the phase's compacted 0/1 incidence matrix, int8, row-major with K
// (the other dimension) contiguous: K-major for both MMA operands, since
// A = rows I of X and B = rows J of X.
//
// Schedule (symmetric / SYRK): tiles (I, J) of BM x BN with row block
// I <= (J+1)*BN/BM - 1; inside a tile only pairs i < j are evaluated, and each
// evaluates both directions (epilogue.cuh), so every unordered pair is
// counted exactly once and the executed MMA work is ~half a full square.
//
// Warp roles (one CTA per SM, persistent over a static tile list):
//   warp 0      TMA producer (one lane): A/B k-blocks into a STAGES-deep ring
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma K=32 per k-block
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> predicates -> ballots/atomics
#pragma once
#include <cuda.h>
#include <cstdint>

#include "epilogue.cuh"
#include "ptx.cuh"

namespace mhsk {
namespace tc {

constexpr int BM = 128;             // rows of A per tile (UMMA M)
constexpr int BN = 256;             // rows of B per tile (UMMA N)
constexpr int BK = 128;             // K bytes per stage = one 128B swizzle atom row
constexpr int UMMA_K = 32;          // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;    // 16 KiB
constexpr int B_BYTES = BN * BK;    // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int TMEM_COLS = 2 * BN;   // double-buffered int32 accumulators
constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;
constexpr int ROW_PAD = BN;         // X rows are padded to a multiple of this

struct GramArgs {
    int32_t M;                          // items decided in this phase
    int32_t k_blocks;                   // K_pad / BK (>= 1)
    const int32_t* __restrict__ va;     // s_i (edges) / d_i (vertices)
    const int32_t* __restrict__ vb;     // f_i (edges) / unused
    int32_t* __restrict__ hits;         // per item: number of deleters
    const uint32_t* __restrict__ tiles; // (I | J << 16)
    int32_t tile_begin;                 // this rank's tiles: tile_begin + i * tile_stride
    int32_t tile_count;
    int32_t tile_stride;
};

__device__ __forceinline__ ItemVals load_item(const GramArgs& a, int32_t idx, bool valid) {
    ItemVals v;
    v.a = valid ? __ldg(a.va + idx) : 0;
    v.b = (valid && a.vb) ? __ldg(a.vb + idx) : 0;
    return v;
}

template <int PHASE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gram_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const GramArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* stage_a = smem;
    uint8_t* stage_b = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;                 // [STAGES] TMA -> MMA
    uint64_t* empty = bars + STAGES;       // [STAGES] MMA -> TMA
    uint64_t* tfull = bars + 2 * STAGES;   // [2]      MMA -> epilogue
    uint64_t* tempty = tfull + 2;          // [2]      epilogue -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4);   // one arrive per epilogue warp
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc(tmem_slot, TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;


    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int32_t it = blockIdx.x, t = args.tile_begin + it * args.tile_stride; it < args.tile_count;
                 it += gridDim.x, t = args.tile_begin + it * args.tile_stride) {
                const uint32_t ij = __ldg(args.tiles + t);
                const int32_t I = ij & 0xFFFF, J = ij >> 16;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
                    ptx::tma_load_2d(stage_a + stage * A_BYTES, &tmA, &full[stage], kb * BK, I * BM,
                                     ptx::kEvictNormal);
                    ptx::tma_load_2d(stage_b + stage * B_BYTES, &tmB, &full[stage], kb * BK, J * BN,
                                     ptx::kEvictLast);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int32_t it = blockIdx.x, t = args.tile_begin + it * args.tile_stride; it < args.tile_count;
                 it += gridDim.x, t = args.tile_begin + it * args.tile_stride) {
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t adesc = ptx::smem_desc_sw128(ptx::smem_u32(stage_a + stage * A_BYTES));
                    const uint64_t bdesc = ptx::smem_desc_sw128(ptx::smem_u32(stage_b + stage * B_BYTES));
#pragma unroll
                    for (int k = 0; k < BK / UMMA_K; ++k) {
                        // advance the start address by k * 32 bytes inside the swizzle atom
                        ptx::mma_i8(d_tmem, adesc + (uint64_t)((k * UMMA_K) >> 4),
                                    bdesc + (uint64_t)((k * UMMA_K) >> 4), idesc,
                                    (kb | k) != 0 ? 1u : 0u);
                    }
                    ptx::mma_commit(&empty[stage]);   // frees the smem slot when these MMAs finish
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit(&tfull[acc]);         // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------------------------ epilogue
        const int q = warp - EPI_WARP0;               // TMEM lane quarter of this warp
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int32_t it = blockIdx.x, t = args.tile_begin + it * args.tile_stride; it < args.tile_count;
                 it += gridDim.x, t = args.tile_begin + it * args.tile_stride) {
            const uint32_t ij = __ldg(args.tiles + t);
            const int32_t I = ij & 0xFFFF, J = ij >> 16;
            const int32_t warp_row0 = I * BM + q * 32;
            const int32_t i = warp_row0 + (int32_t)lane;
            const bool row_valid = i < args.M;
            const ItemVals vi = load_item(args, i, row_valid);
            int32_t row_hits = 0;

            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                const int32_t j0 = J * BN + c * 32;
                if (j0 >= args.M) break;                       // padding columns (warp-uniform)
                if (j0 + 31 <= warp_row0) continue;            // no pair with i < j here
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
                const int32_t jl = j0 + (int32_t)lane;
                const ItemVals vjl = load_item(args, jl, jl < args.M);
                ptx::tmem_ld_wait();
                uint32_t my_col_hits = 0;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    const int32_t j = j0 + jj;
                    ItemVals vj;
                    vj.a = __shfl_sync(0xffffffffu, vjl.a, jj);
                    vj.b = __shfl_sync(0xffffffffu, vjl.b, jj);
                    bool i_del_j, j_del_i;
                    pair_predicates<PHASE>((int32_t)r[jj], vi, vj, i_del_j, j_del_i);
                    const bool handled = row_valid && j < args.M && i < j;
                    row_hits += (handled && j_del_i) ? 1 : 0;
                    const uint32_t b = __ballot_sync(0xffffffffu, handled && i_del_j);
                    if (lane == (uint32_t)jj) my_col_hits = __popc(b);
                }
                if (my_col_hits) atomicAdd(args.hits + jl, (int32_t)my_col_hits);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
            if (row_hits) atomicAdd(args.hits + i, row_hits);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, TMEM_COLS);
}

}  // namespace tc
}  // namespace mhsk
