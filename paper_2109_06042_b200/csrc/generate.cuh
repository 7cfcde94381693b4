// generate.cuh -- counter-based random instances, bit-identical on host and
// device.
//
// Semantics of the reference generator (generate.py:18-46): every (edge,
// vertex) incidence is an independent Bernoulli(p); an empty edge is redrawn
// up to 20 times, then padded with one random vertex; demand min(alpha, |e|).
// Instead of a sequential Mersenne-Twister stream, draw r of cell (e, v) is
// the hash mix64(seed, e, v, r) compared against p * 2^32, so any cell can be
// evaluated independently -- on 148 SMs, or in numpy
// (paper_2109_06042_b200/generate.py:counter_random, same constants).
#pragma once
#include <cstdint>

namespace mhsk {
namespace gen {

constexpr int RETRIES = 20;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t e, uint64_t v, uint64_t r) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull ^ e * 0xD1B54A32D192ED03ull ^ v * 0xC2B2AE3D27D4EB4Full ^
                 r * 0x165667B19E3779F9ull;
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

__host__ __device__ __forceinline__ bool draw(uint64_t seed, int64_t e, int64_t v, int r, uint64_t thr) {
    return (mix64(seed, (uint64_t)e, (uint64_t)v, (uint64_t)r) >> 32) < thr;
}

// Pass 1 (one warp per edge): members of the first non-empty attempt, or 1
// (padding).  attempt[e] = the attempt used, RETRIES for the pad.
__global__ void gen_count(int32_t n, int32_t m, uint64_t seed, uint64_t thr, int64_t* __restrict__ count,
                          int32_t* __restrict__ attempt) {
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        int r = 0;
        int64_t c = 0;
        for (; r < RETRIES; ++r) {
            int64_t local = 0;
            for (int64_t v = lane; v < n; v += 32) local += draw(seed, e, v, r, thr);
            for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
            c = local;
            if (c) break;
        }
        if (lane == 0) {
            count[e + 1] = c ? c : 1;
            attempt[e] = r;
        }
    }
}

// Pass 2: write each edge's members in increasing order (warp ballots give
// every lane its output slot), pad vertex for attempt == RETRIES; demand.
__global__ void gen_fill(int32_t n, int32_t m, uint64_t seed, uint64_t thr, int32_t alpha,
                         const int64_t* __restrict__ ptr, const int32_t* __restrict__ attempt,
                         int32_t* __restrict__ vtx, int32_t* __restrict__ demand) {
    const int64_t warp_global = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    for (int64_t e = warp_global; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int r = attempt[e];
        int64_t pos = ptr[e];
        if (r == RETRIES) {
            if (lane == 0) vtx[pos] = (int32_t)(mix64(seed, (uint64_t)e, 0xFFFFFFFFull, RETRIES) % (uint64_t)n);
        } else {
            for (int64_t v0 = 0; v0 < n; v0 += 32) {
                const int64_t v = v0 + lane;
                const bool in = v < n && draw(seed, e, v, r, thr);
                const uint32_t b = __ballot_sync(0xffffffffu, in);
                if (in) vtx[pos + __popc(b & ((1u << lane) - 1u))] = (int32_t)v;
                pos += __popc(b);
            }
        }
        if (lane == 0) {
            const int64_t s = ptr[e + 1] - ptr[e];
            demand[e] = (int32_t)(s < alpha ? s : alpha);
        }
    }
}

// Inclusive scan of count[1..m] into ptr (count[0] = 0), one block.
__global__ void scan_i64(int64_t* __restrict__ a, int64_t n) {
    __shared__ int64_t carry;
    __shared__ int64_t warp_sums[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t idx = base + threadIdx.x;
        const int64_t v = idx < n ? a[idx] : 0;
        const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
        int64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t s = lane < (int)(blockDim.x / 32) ? warp_sums[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const int64_t incl = carry + (w ? warp_sums[w - 1] : 0) + x;
        if (idx < n) a[idx] = incl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
}

}  // namespace gen
}  // namespace mhsk
