// mxf4_probe.cu -- does tcgen05.mma kind::mxf4 (packed E2M1, all block scales
// 1.0) compute exact 0/1 co-occurrence counts, and at what rate?
//
//   ./mxf4_probe check <afmt> <variant>  -> mismatches vs a CPU dot product
//   ./mxf4_probe peak [seconds]          -> one JSON line of dense FP4 TFLOP/s
//
// 0/1 entries: E2M1 1.0 = 0b0010, two elements per byte.  Scale factors
// (UE8M0 127 = 2^0) fill every TMEM column the MMA may read, so the SF
// layout / sf_id semantics cannot matter.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2109_06042_b200/csrc/ptx.cuh"

using namespace mhsk;

constexpr int BM = 128, BN = 256, KB = 128;   // bytes per row per stage = 256 fp4
constexpr int SF_COL = 256, SF_COLS = 64;

__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t M, uint32_t N, uint32_t fmt) {
    return (fmt << 7) | (fmt << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                         uint32_t sfb, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %6, 0;\n"
        " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc));
}

__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr), "r"(v)
                 : "memory");
}

// byte (row r, byte b) of a K-major SW128 tile
__host__ __device__ inline int sw128(int r, int b) { return (r / 8) * 1024 + (r % 8) * 128 + (((b / 16) ^ (r % 8)) * 16) + b % 16; }

__global__ void __launch_bounds__(128, 1) mxf4_kernel(const uint8_t* ga, const uint8_t* gb, float* out, int iters,
                                                      uint32_t fmt, int* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = smem;
    uint8_t* b = smem + BM * KB;
    __shared__ uint64_t done;
    __shared__ uint32_t tmem_slot;
    for (int i = threadIdx.x; i < BM * KB; i += blockDim.x) a[sw128(i / KB, i % KB)] = ga ? ga[i] : 0x22;
    for (int i = threadIdx.x; i < BN * KB; i += blockDim.x) b[sw128(i / KB, i % KB)] = gb ? gb[i] : 0x22;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        ptx::tmem_alloc(&tmem_slot, 512);
        ptx::tmem_relinquish();
    }
    if (threadIdx.x == 32) {
        ptx::mbar_init(&done, 1);
        ptx::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    // scale factors: 0x7F bytes (UE8M0 2^0) in columns SF_COL .. SF_COL + SF_COLS
    for (int c = 0; c < SF_COLS; c += 8) tmem_st_x8(tmem + ((uint32_t)(warp * 32) << 16) + SF_COL + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 32) {
        const uint32_t idesc = idesc_mxf4(BM, BN, fmt);
        const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(a));
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(b));
        const uint32_t sfa = tmem + SF_COL, sfb = tmem + SF_COL + SF_COLS / 2;
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = out ? tmem : tmem + 0;   // single accumulator (cols 0..255)
#pragma unroll
            for (int k = 0; k < KB / 32; ++k)
                mma_mxf4(d, ad + (uint64_t)((k * 32) >> 4), bd + (uint64_t)((k * 32) >> 4), idesc, sfa, sfb,
                         (k != 0 || it > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
        ptx::tmem_ld_wait();
        const int row = warp * 32 + threadIdx.x % 32;
        if (out) {
            for (int j = 0; j < 32; ++j) out[row * BN + c + j] = __uint_as_float(r[j]);
        } else if (r[0] == 0xFFFFFFFFu) {
            *sink = 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

// Issue-pattern experiment (cta_group::1, smem-resident operands): MMAs of
// width N, a tcgen05.commit every `commit_every` k-blocks (4 MMAs each, 0 =
// never), and a switch between `nacc` accumulators (column offset N apart,
// first MMA of a tile overwrites) every `tile_kb` k-blocks (0 = never).
__global__ void __launch_bounds__(128, 1) shape_kernel(int iters, uint32_t N, int commit_every, int tile_kb, int nacc,
                                                       int* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = smem;
    uint8_t* b = smem + BM * KB;
    __shared__ uint64_t done, cbar;
    __shared__ uint32_t tmem_slot;
    for (int i = threadIdx.x; i < (BM + BN) * KB; i += blockDim.x) smem[i] = 0x22;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        ptx::tmem_alloc(&tmem_slot, 512);
        ptx::tmem_relinquish();
    }
    if (threadIdx.x == 32) {
        ptx::mbar_init(&done, 1);
        ptx::mbar_init(&cbar, 1);
        ptx::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    for (int c = 480; c < 512; c += 8) tmem_st_x8(tmem + ((uint32_t)(warp * 32) << 16) + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 32) {
        const uint32_t idesc = idesc_mxf4(BM, N, 1);
        const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(a));
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(b));
        const uint32_t sfa = tmem + 480, sfb = tmem + 496;
        int acc = 0, in_tile = 0;
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + acc * N;
#pragma unroll
            for (int k = 0; k < KB / 32; ++k)
                mma_mxf4(d, ad + (uint64_t)((k * 32) >> 4), bd + (uint64_t)((k * 32) >> 4), idesc, sfa, sfb,
                         (k != 0 || in_tile > 0) ? 1u : 0u);
            if (commit_every > 0 && (it % commit_every) == commit_every - 1) ptx::mma_commit(&cbar);
            if (tile_kb > 0 && ++in_tile == tile_kb) {
                in_tile = 0;
                ptx::mma_commit(&cbar);
                if (++acc == nacc) acc = 0;
            }
        }
        ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
    if (threadIdx.x == 0 && iters < 0) *sink = 1;
}

// Same on CTA pairs (cta_group::2, M = 256, B split N/2 per CTA), operands
// resident in both CTAs' shared memory (no TMA).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(int iters, uint32_t N, int tile_kb, int* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = smem;
    uint8_t* b = smem + BM * KB;
    __shared__ uint64_t done, cbar;
    __shared__ uint32_t tmem_slot;
    for (int i = threadIdx.x; i < (BM + BN) * KB; i += blockDim.x) smem[i] = 0x22;
    const int warp = threadIdx.x / 32;
    const bool leader = ptx::cluster_ctarank() == 0;
    if (warp == 0) {
        ptx::tmem_alloc_pair(&tmem_slot, 512);
        ptx::tmem_relinquish_pair();
    }
    if (threadIdx.x == 32) {
        ptx::mbar_init(&done, 1);
        ptx::mbar_init(&cbar, 1);
        ptx::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    for (int c = 480; c < 512; c += 8) tmem_st_x8(tmem + ((uint32_t)(warp * 32) << 16) + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (leader && threadIdx.x == 32) {
        const uint32_t idesc = idesc_mxf4(2 * BM, N, 1);
        const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(a));
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(b));
        int acc = 0, in_tile = 0;
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + acc * N;
#pragma unroll
            for (int k = 0; k < KB / 32; ++k)
                ptx::mma_mxf4_pair(d, ad + (uint64_t)((k * 32) >> 4), bd + (uint64_t)((k * 32) >> 4), idesc,
                                   tmem + 480, tmem + 496, (k != 0 || in_tile > 0) ? 1u : 0u);
            ptx::mma_commit_pair(&cbar, 0x3);
            if (tile_kb > 0 && ++in_tile == tile_kb) {
                in_tile = 0;
                if (++acc == 2) acc = 0;
            }
        }
        ptx::mma_commit_pair(&done, 0x3);
    }
    if (threadIdx.x == 32) ptx::mbar_wait(&done, 0);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc_pair(tmem, 512);
    if (threadIdx.x == 0 && iters < 0) *sink = 1;
}

int main(int argc, char** argv) {
    if (argc > 1 && !strcmp(argv[1], "pair")) {
        const uint32_t N = argc > 2 ? atoi(argv[2]) : 256;
        const int tkb = argc > 3 ? atoi(argv[3]) : 0;
        const int smem = (BM + BN) * KB + 1024;
        cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int* sink;
        cudaMalloc(&sink, 4);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int iters = 20000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        pair_kernel<<<sms, 128, smem>>>(iters, N, tkb, sink);
        cudaEventRecord(e0);
        for (int l = 0; l < 5; ++l) pair_kernel<<<sms, 128, smem>>>(iters, N, tkb, sink);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
            printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * (2 * BM) * N * (KB * 2) * (double)iters * (sms / 2) * 5;
        printf("{\"pair\": 1, \"N\": %u, \"tile_kb\": %d, \"tflops\": %.1f}\n", N, tkb,
               ops / (ms / 1e3) / 1e12);
        return 0;
    }
    if (argc > 1 && !strcmp(argv[1], "shape")) {
        const uint32_t N = argc > 2 ? atoi(argv[2]) : 256;
        const int ce = argc > 3 ? atoi(argv[3]) : 0, tkb = argc > 4 ? atoi(argv[4]) : 0;
        const int nacc = argc > 5 ? atoi(argv[5]) : 1;
        const int smem = (BM + BN) * KB + 1024;
        cudaFuncSetAttribute(shape_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int* sink;
        cudaMalloc(&sink, 4);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int iters = 20000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        shape_kernel<<<sms, 128, smem>>>(iters, N, ce, tkb, nacc, sink);
        cudaEventRecord(e0);
        for (int l = 0; l < 5; ++l) shape_kernel<<<sms, 128, smem>>>(iters, N, ce, tkb, nacc, sink);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
            printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * BM * N * (KB * 2) * (double)iters * sms * 5;
        const double cyc = (ms / 5 / 1e3) * 1.92e9 / iters;   // per k-block (4 MMAs) at 1.92 GHz
        printf("{\"N\": %u, \"commit_every\": %d, \"tile_kb\": %d, \"nacc\": %d, \"tflops\": %.1f, "
               "\"cycles_per_kblock\": %.1f}\n", N, ce, tkb, nacc, ops / (ms / 1e3) / 1e12, cyc);
        return 0;
    }
    const bool peak = argc > 1 && !strcmp(argv[1], "peak");
    const uint32_t fmt = argc > 2 && !peak && strcmp(argv[1], "accum") ? (uint32_t)atoi(argv[2]) : 1;
    const int smem = (BM + BN) * KB + 1024;
    cudaFuncSetAttribute(mxf4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* sink;
    cudaMalloc(&sink, 4);
    if (argc > 2 && !strcmp(argv[1], "accum")) {
        // A all ones; B row j holds j ones (0..255): D[i][j] = iters * j after
        // `iters` x K=256 accumulations -- large counts with low bits set
        const int iters = atoi(argv[2]);
        std::vector<uint8_t> B(BN * KB, 0);
        for (int j = 0; j < BN; ++j)
            for (int k = 0; k < j; ++k) B[j * KB + k / 2] |= (uint8_t)(0x2 << (4 * (k & 1)));
        uint8_t* db;
        float* dout;
        cudaMalloc(&db, B.size());
        cudaMemcpy(db, B.data(), B.size(), cudaMemcpyHostToDevice);
        cudaMalloc(&dout, BM * BN * 4);
        mxf4_kernel<<<1, 128, smem>>>(nullptr, db, dout, iters, 1, sink);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        std::vector<float> out(BM * BN);
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < BM; ++i)
            for (int j = 0; j < BN; ++j) bad += (double)out[i * BN + j] != (double)iters * j;
        printf("{\"iters\": %d, \"max_want\": %lld, \"got\": %.1f, \"mismatches\": %d}\n", iters,
               (long long)iters * 255, out[255], bad);
        return bad != 0;
    }
    if (!peak) {
        // random 0/1, p = 0.3; element k of a row = nibble (k & 1) of byte k / 2
        std::vector<uint8_t> A(BM * KB), B(BN * KB);
        std::vector<int> bitsA(BM * 256), bitsB(BN * 256);
        srand(7);
        auto fill = [](std::vector<uint8_t>& X, std::vector<int>& bits, int rows) {
            for (int r = 0; r < rows; ++r)
                for (int k = 0; k < 256; ++k) {
                    const int v = rand() % 10 < 3;
                    bits[r * 256 + k] = v;
                    if (v) X[r * KB + k / 2] |= (uint8_t)(0x2 << (4 * (k & 1)));
                }
        };
        fill(A, bitsA, BM);
        fill(B, bitsB, BN);
        uint8_t *da, *db;
        float* dout;
        cudaMalloc(&da, A.size());
        cudaMalloc(&db, B.size());
        cudaMalloc(&dout, BM * BN * 4);
        cudaMemcpy(da, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(db, B.data(), B.size(), cudaMemcpyHostToDevice);
        mxf4_kernel<<<1, 128, smem>>>(da, db, dout, 1, fmt, sink);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("{\"fmt\": %u, \"error\": \"%s\"}\n", fmt, cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> out(BM * BN);
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxc = 0;
        for (int i = 0; i < BM; ++i)
            for (int j = 0; j < BN; ++j) {
                int c = 0;
                for (int k = 0; k < 256; ++k) c += bitsA[i * 256 + k] & bitsB[j * 256 + k];
                maxc = c > maxc ? c : maxc;
                if (out[i * BN + j] != (float)c) {
                    if (bad < 4) printf("  mismatch (%d,%d): got %g want %d\n", i, j, out[i * BN + j], c);
                    ++bad;
                }
            }
        printf("{\"fmt\": %u, \"mismatches\": %d, \"max_count\": %g, \"sample\": %g}\n", fmt, bad, maxc, out[0]);
        return bad != 0;
    }
    const double seconds = argc > 2 ? atof(argv[2]) : 3.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    mxf4_kernel<<<sms, 128, smem>>>(nullptr, nullptr, nullptr, iters, fmt, sink);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
    }
    cudaEventRecord(e0);
    mxf4_kernel<<<sms, 128, smem>>>(nullptr, nullptr, nullptr, iters, fmt, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops_launch = 2.0 * BM * BN * (KB * 2) * (double)iters * sms;
    const double burst = ops_launch / (ms / 1e3) / 1e12;
    const int launches = (int)(seconds * 1e3 / ms) + 1;
    cudaEventRecord(e0);
    for (int l = 0; l < launches; ++l) mxf4_kernel<<<sms, 128, smem>>>(nullptr, nullptr, nullptr, iters, fmt, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double sustained = ops_launch * launches / (ms / 1e3) / 1e12;
    printf("{\"fp4_tflops_burst\": %.1f, \"fp4_tflops_sustained\": %.1f, \"sms\": %d, "
           "\"shape\": \"tcgen05.mma.cta_group::1.kind::mxf4.block_scale M=128 N=256 K=64, smem-resident\", "
           "\"launch_ms\": %.3f, \"launches\": %d}\n",
           burst, sustained, sms, ms / launches, launches);
    return 0;
}
