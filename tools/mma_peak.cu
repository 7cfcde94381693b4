// mma_peak.cu -- measured dense int8 tensor-core peak of this B200
// (tcgen05.mma kind::i8, M=128 N=256 K=32, one CTA per SM, operands resident
// in shared memory, accumulators alternating between two TMEM buffers).
// MEASURED_PEAKS.json has only bf16; this is the int8 roofline denominator
// bench.py reports beside 2 x bf16 and the datasheet 4.5 POPS.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak mma_peak.cu
//   ./mma_peak [seconds]  -> one JSON line
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2109_06042_b200/csrc/ptx.cuh"

using namespace mhsk;

constexpr int BM = 128, BN = 256, BK = 128;

__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = smem;
    uint8_t* b = smem + BM * BK;
    __shared__ uint64_t done;
    __shared__ uint32_t tmem_slot;
    for (int i = threadIdx.x; i < (BM + BN) * BK / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
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
    if (threadIdx.x == 32) {
        const uint32_t idesc = ptx::idesc_i8(BM, BN);
        const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(a));
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(b));
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + (it & 1) * BN;
#pragma unroll
            for (int k = 0; k < BK / 32; ++k)
                ptx::mma_i8(d, ad + (uint64_t)((k * 32) >> 4), bd + (uint64_t)((k * 32) >> 4), idesc,
                            k != 0 || it > 1 ? 1u : 0u);
        }
        ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 1) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)32 << 16), r);
        ptx::tmem_ld_wait();
        if (threadIdx.x == 32 && r[0] == 0xFFFFFFFFu) *sink = 1;
    }
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
    const double seconds = argc > 1 ? atof(argv[1]) : 3.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = (BM + BN) * BK + 1024;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int iters = 20000;
    mma_loop<<<sms, 128, smem>>>(iters, sink);   // warm-up
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
    }
    // burst: one launch; sustained: back-to-back launches for `seconds`
    cudaEventRecord(e0);
    mma_loop<<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops_launch = 2.0 * BM * BN * BK * (double)iters * sms;
    const double burst = ops_launch / (ms / 1e3) / 1e12;
    int launches = (int)(seconds * 1e3 / ms) + 1;
    cudaEventRecord(e0);
    for (int l = 0; l < launches; ++l) mma_loop<<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double sustained = ops_launch * launches / (ms / 1e3) / 1e12;
    printf("{\"int8_tops_burst\": %.1f, \"int8_tops_sustained\": %.1f, \"sms\": %d, "
           "\"shape\": \"tcgen05.mma.cta_group::1.kind::i8 M=128 N=256 K=32, smem-resident operands\", "
           "\"launch_ms\": %.3f, \"launches\": %d}\n",
           burst, sustained, sms, ms / launches, launches);
    return 0;
}
