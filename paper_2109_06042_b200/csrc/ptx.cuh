// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05.
//
// Only what the Gram kernels need.  Every wait loop carries a watchdog: a
// barrier that never completes (a descriptor or phase bug) traps the kernel
// with an error instead of hanging the GPU.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Checked build (make checked -> libmhsk_checked.so, -DMHSK_CHECKED): device
// assertions at every index the kernels derive from data (candidate slots,
// deleter counts, hash probes, member ids, operand rows and columns).  The
// pool does not allow compute-sanitizer; this is the bounds check that runs
// instead (tools/sanitize_run.py with MHSK_LIB=checked).
#ifdef MHSK_CHECKED
#include <cstdio>
#define MHSK_CHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("MHSK_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define MHSK_CHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace mhsk {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Wait until the phase with the given parity has completed.  Traps after
// ~2^34 SM cycles (several seconds at any clock) so a pipeline bug surfaces
// as a launch error, not a hung device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long start = clock64();
    while (!mbar_try_wait(bar, parity)) {
        if (clock64() - start > (1ll << 34)) __trap();
    }
}

// mbar_wait that backs off with __nanosleep between polls, so a waiting warp
// does not take issue slots from the warps sharing its SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = 32) {
    if (mbar_try_wait(bar, parity)) return;
    const long long start = clock64();
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(ns);
        if (clock64() - start > (1ll << 34)) __trap();
    }
}

// ------------------------------------------------------- cp.async (LDGSTS)
// 8-byte global -> shared copy without registers; src_bytes 0 zero-fills.
__device__ __forceinline__ void cp_async_8(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar,
                                            int32_t c0, int32_t c1, uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1),
        "l"(cache_hint)
        : "memory");
}

// L2 cache-policy constants (createpolicy.fractional.L2::evict_last / first)
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;

// ----------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, int8 x int8 -> int32, one CTA.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32 columns of 32-bit accumulators -> 32 registers per thread
// (thread t gets lane base+t, columns col..col+31).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
// first 16 columns only (the 240-column FP4 tile's last, half-width chunk)
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 bytes apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);   // start address  [0,14)
    d |= static_cast<uint64_t>(1) << 16;                        // LBO (unused, SW128 K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;                // SBO            [32,46)
    d |= static_cast<uint64_t>(1) << 46;                        // version = 1    [46,48)
    d |= static_cast<uint64_t>(2) << 61;                        // SWIZZLE_128B   [61,64)
    return d;
}

// Instruction descriptor, kind::mxf4 (block-scaled): packed E2M1 x E2M1 ->
// f32, UE8M0 scale factors, K = 64, both K-major (measured exact for 0/1
// operands up to counts of 2^24 - 1: tools/mxf4_probe.cu).
__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t M, uint32_t N) {
    return (1u << 7)             // A format: E2M1
           | (1u << 10)          // B format: E2M1
           | ((N >> 3) << 17)    // N / 8
           | (1u << 23)          // scale format: UE8M0
           | ((M >> 4) << 24);   // M / 16
}

// 8 consecutive TMEM columns of this warp's 32 lanes <- v
__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
                 "r"(v)
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Instruction descriptor, kind::i8: u8 x u8 -> s32, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
    return (2u << 4)             // D format: s32
           | (0u << 7)           // A format: unsigned 8-bit
           | (0u << 10)          // B format: unsigned 8-bit
           | ((N >> 3) << 17)    // N / 8
           | ((M >> 4) << 24);   // M / 16
}

}  // namespace ptx
}  // namespace mhsk

// ------------------------------------------------------- CTA-pair (2-SM) ops
namespace mhsk {
namespace ptx {

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}

// Wait with cluster-scope acquire: stores another CTA of the cluster made
// before its release-arrive on this barrier are visible afterwards.
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
    const long long start = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (clock64() - start > (1ll << 34)) __trap();
    }
}

// 32-bit store to a shared::cluster address (this or a peer CTA's smem)
__device__ __forceinline__ void st_cluster_s32(uint32_t cluster_addr, int32_t v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// Arrive on an mbarrier of any CTA in the cluster.  Release at CTA scope (the
// mbarrier.arrive default): enough to hand a TMEM accumulator back (ordering
// comes from the tcgen05 fences around it) and far cheaper than a
// cluster-scope release, which waits for the thread's memory traffic.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Same, with a cluster-scope release: prior global / shared writes of this
// thread are visible to threads of the cluster that acquire the barrier phase.
__device__ __forceinline__ void mbar_arrive_cluster_release(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}

// TMA load whose completion is signalled on the pair leader's mbarrier
// (`bar_cluster` is a shared::cluster address, e.g. from mapa(.., 0)).
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* desc, uint32_t bar_cluster,
                                                 int32_t c0, int32_t c1, uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(cache_hint)
        : "memory");
}

// One stage of a pair's operands, issued by an elected lane of a CONVERGED
// warp: the leader arms its full barrier with `bytes` (arm != 0), then this
// CTA's A and B boxes are loaded with completion on the leader's barrier.
__device__ __forceinline__ void tma_stage_pair_elect(uint32_t bar_local, uint32_t arm, uint32_t bytes,
                                                     uint32_t bar_cluster, uint32_t dst_a, const void* tm_a,
                                                     int32_t ca, int32_t ra, uint64_t hint_a, uint32_t load_a,
                                                     uint32_t dst_b, const void* tm_b, int32_t rb, uint64_t hint_b) {
    asm volatile(
        "{\n\t.reg .pred e, pa, pl;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.and.b32 pa, %1, 0, e;\n\t"
        "setp.ne.and.b32 pl, %9, 0, e;\n\t"
        "@pa mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %2;\n\t"
        "@pl cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%4], [%5, {%6, %7}], [%3], %8;\n\t"
        "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%10], [%11, {%6, %12}], [%3], %13;\n\t}"
        ::"r"(bar_local), "r"(arm), "r"(bytes), "r"(bar_cluster), "r"(dst_a),
        "l"(reinterpret_cast<uint64_t>(tm_a)), "r"(ca), "r"(ra), "l"(hint_a), "r"(load_a), "r"(dst_b),
        "l"(reinterpret_cast<uint64_t>(tm_b)), "r"(rb), "l"(hint_b)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}

// D[tmem of both CTAs] (+)= A[smem, 128 rows per CTA] . B[smem, N/2 rows per CTA]^T
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Block-scaled FP4 pair MMA: K = 64 packed E2M1 per instruction (32 bytes,
// the same smem footprint as one kind::i8 K = 32 step); sfa / sfb are the
// TMEM addresses of the scale factors.
__device__ __forceinline__ void mma_mxf4_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
        : "memory");
}

// One 128-byte k-block (four K = 32-byte steps) of pair MMAs plus the commit
// that releases its smem stage, issued by one elected lane of a CONVERGED
// warp (warp-uniform operands stay in uniform registers; no per-instruction
// elect / broadcast loops as in single-lane code).  first != 0: the first
// step overwrites D.
#define MHSK_MMA4_BODY(KIND_SCALE, SF_ARGS)                                                        \
    "{\n\t.reg .pred e, f, t;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"                       \
    "elect.sync _|e, 0xffffffff;\n\t"                                                          \
    "setp.eq.b32 f, %4, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"                                       \
    "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"                     \
    "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"                     \
    "@e tcgen05.mma.cta_group::2." KIND_SCALE " [%0], %1, %2, %3" SF_ARGS ", f;\n\t"              \
    "@e tcgen05.mma.cta_group::2." KIND_SCALE " [%0], a1, b1, %3" SF_ARGS ", t;\n\t"              \
    "@e tcgen05.mma.cta_group::2." KIND_SCALE " [%0], a2, b2, %3" SF_ARGS ", t;\n\t"              \
    "@e tcgen05.mma.cta_group::2." KIND_SCALE " [%0], a3, b3, %3" SF_ARGS ", t;\n\t"              \
    "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64" \
    " [%5], %6;\n\t}"
__device__ __forceinline__ void mma4_mxf4_pair_commit(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                      uint32_t first, uint32_t bar, uint16_t mask, uint32_t sfa,
                                                      uint32_t sfb) {
    asm volatile(MHSK_MMA4_BODY("kind::mxf4.block_scale.scale_vec::2X", ", [%7], [%8]")
                 ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(first), "r"(bar), "h"(mask), "r"(sfa),
                 "r"(sfb)
                 : "memory");
}
__device__ __forceinline__ void mma4_i8_pair_commit(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t first, uint32_t bar, uint16_t mask) {
    asm volatile(MHSK_MMA4_BODY("kind::i8", "") ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(first),
                 "r"(bar), "h"(mask)
                 : "memory");
}
#undef MHSK_MMA4_BODY
// commit (elected lane of a converged warp)
__device__ __forceinline__ void commit_pair_elect(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(bar), "h"(mask)
        : "memory");
}

// Arrive (once) on the mbarrier at this smem offset in every CTA of `cta_mask`
// when all prior tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t cta_mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(cta_mask)
        : "memory");
}

}  // namespace ptx
}  // namespace mhsk
