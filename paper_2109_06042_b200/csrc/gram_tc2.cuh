// gram_tc2.cuh -- the Gram product on CTA pairs: tcgen05.mma.cta_group::2
// kind::i8, 256 x 256 output tiles, each SM of the pair holding 128 rows of
// A and 128 rows of B per k-block.  Same fused epilogue and triangle schedule
// as gram_tc.cuh (see there for the semantics); this variant moves 2/3 of the
// operand bytes per MAC of the 1-CTA 128 x 256 tile, which is what bounds the
// 1-CTA kernel (L2 -> SM bandwidth, profiles/).
//
// Pair protocol (cluster of 2, rank 0 = leader):
//   both CTAs  TMA their A/B halves into their own smem; completion is
//              signalled on the LEADER's full barrier (cta_group::2 TMA);
//              the leader arms it with the bytes of both halves.
//   leader     waits full, issues 4 x tcgen05.mma.cta_group::2 per k-block,
//              commits to both CTAs' empty barrier (multicast) and, per tile,
//              to both CTAs' tmem-full barrier.
//   both CTAs  epilogue on their own 128 TMEM lanes (tile rows), then arrive
//              on the leader's tmem-empty barrier (8 warps).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "epilogue.cuh"
#include "ptx.cuh"

namespace mhsk {
namespace tc2 {

constexpr int BM = 256;             // tile rows (pair)
constexpr int BN = 256;             // tile columns
constexpr int HALF = 128;           // rows of A and of B held by each CTA
constexpr int BK = 128;             // K bytes per stage
constexpr int UMMA_K = 32;
#ifndef MHSK_STAGES
#define MHSK_STAGES 6
#endif
constexpr int STAGES = MHSK_STAGES;
constexpr int A_BYTES = HALF * BK;  // 16 KiB
constexpr int B_BYTES = HALF * BK;  // 16 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
// warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4..11
// epilogue -- two per TMEM lane quarter (warp % 4), each taking half the
// tile's columns (16 epilogue warps at 96 registers measured slower: spills)
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int TMEM_COLS = 2 * BN;
constexpr int EPI_WARPS = 8;
constexpr int EPI_COLS = BN / 2;    // columns per epilogue warp
// per epilogue warp: its columns' values, int4 {a, b, rank | remainder, 0}
constexpr int COLVAL_BYTES = EPI_WARPS * EPI_COLS * 16;
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256 + COLVAL_BYTES;
constexpr int ROW_PAD = 256;
// FP4 mode (kind::mxf4): a 128-byte k-block holds 256 packed E2M1 items;
// tiles are 256 x 240 so that two accumulators (2 x 240 columns) and the
// UE8M0 scale factors (all 1.0, columns SF_COL.. of both CTAs) fit the 512
// TMEM columns -- the epilogue of tile t then overlaps the MMAs of tile t+1
constexpr int BK_ITEMS_I8 = 128, BK_ITEMS_FP4 = 256;
constexpr int BN_FP4 = 240;
constexpr int SF_COL = 2 * BN_FP4, SF_COLS = 32;

struct GramArgs {
    int32_t M;
    int32_t k_blocks;
    const int32_t* __restrict__ va;
    const int32_t* __restrict__ vb;
    int32_t* __restrict__ hits;
    const uint32_t* __restrict__ tiles;  // (P | J << 16), 256 x 256 squares, P <= J
    int32_t tile_begin;                  // this rank's tiles: tile_begin + i * tile_stride,
    int32_t tile_count;                  //   i < tile_count (ranks interleave)
    int32_t tile_stride;
    // K-drift throttle (nullptr = off): progress[w] counts the K-chunks the
    // pairs of wave w (their w-th tile) have loaded; a pair may load chunk c
    // only once progress[w] >= (c - slack) * (pairs in wave w).
    int32_t* __restrict__ progress;
    int32_t chunk_log2;
    int32_t slack;
    // device-resident sizes (nullptr = use M / k_blocks): dev_mk[0] = M,
    // dev_mk[1] = K.  Tiles of the (static) list outside the current M are
    // skipped by all roles alike.
    const int32_t* __restrict__ dev_mk;
    // launch gate (nullptr = run): the kernel exits at once unless *enable != 0
    const int32_t* __restrict__ enable;
    // rectangle mode only: A rows are the affected items, row p is item
    // a_items[p] (compact index), p < *a_count
    const int32_t* __restrict__ a_items;
    const int32_t* __restrict__ a_count;
    // block-sparse mode (nullptr = dense): per 256-row panel, bitmask of the
    // 128-column k-blocks it touches (mask_words 64-bit words per panel); a
    // tile multiplies only the k-blocks both panels touch.  A tile with none
    // is skipped, unless *zero_needed (some item for which a zero count can
    // matter, e.g. an edge with demand > size) -- then its epilogue runs with
    // c = 0.
    const unsigned long long* __restrict__ mask;
    int32_t mask_words;
    const int32_t* __restrict__ zero_needed;
    // tie-break ranks of the items (nullptr: the row order is the original order)
    const int32_t* __restrict__ rank;
    // sparse mode: k-blocks multiplied (per pair, one atomic at the end)
    unsigned long long* __restrict__ kblocks_done;
    // probe pruning (dense triangle only; lo == nullptr or probe_kb == 0:
    // off): entries of each item in the first probe_kb k-blocks (epilogue.cuh)
    const int32_t* __restrict__ lo;
    int32_t probe_kb;
    // two-pass probe schedule: per pair, a bitmap (needed_words words) of the
    // tiles the probe could not decide; zeroed by the host
    uint32_t* __restrict__ needed;
    int32_t needed_words;
    // set to 1 when the probe marks any tile (the word after every pair's
    // bitmap): a full-pass-only launch takes it as its enable gate, so a
    // phase whose probe marked nothing skips the full-K launch's prologue
    int32_t* __restrict__ marked;
    // tiles stopped after the probe (one atomic per pair at the end)
    unsigned long long* __restrict__ pruned_tiles;
    // candidate verification (probe pass; cand == nullptr: off).  A warp whose
    // 32 rows x 128 columns hold at most CAND_WARP_CAP pairs that can still
    // fire appends them ({i, j, bit of the tile in `needed`, 0}) instead of
    // marking the tile for full K; verify_candidates (verify.cuh) then decides
    // them from the operand rows, skipping pairs of tiles that were marked
    // after all (those are evaluated in full by pass 1).
    int4* __restrict__ cand;
    int32_t* __restrict__ cand_count;
    int32_t cand_cap;
    // split two-pass schedule (lazy vertex operand): passes = 1 runs only the
    // probe pass, 2 only the full-K pass over the tiles an earlier launch
    // marked, 0 both.  force_probe: probe whenever probe_kb > 0 (the operand
    // holds only the probe columns until the marked panels are packed).
    int32_t passes;
    int32_t force_probe;
    // probe pass over a band of the tile list only: this pair's tiles
    // t_lo <= t < t_hi (default 0 .. INT_MAX).  The marks / candidates of
    // several band launches add up in one `needed` bitmap (indexed by t), so
    // one full-K launch afterwards covers all of them (overlapped upload).
    int32_t t_lo, t_hi;
    // FP4 DP / MD probe: per item {L, b} of probe_split (probe_terms kernel)
    const float2* __restrict__ pv;
    // FP4 DP probe: per column panel the demand shared by all its items, or NaN
    const float* __restrict__ pb;
    // FP4 DP / MD probe: per 32-column chunk of a column panel (8 per panel)
    // {min L_j, min b_j} -- a chunk is skipped when even its largest count
    // cannot reach the row's thresholds against those minima
    const float2* __restrict__ pcm;
    // diagnostics (nullptr = off): cycle counters per role, see GRAM_TIMING_SLOTS
    unsigned long long* __restrict__ timing;
    int32_t tune;  // MHSK_GRAM_TUNE (result-neutral): bit 0 producer sleeps on empty, bit 1 A loads evict_last
};

// timing slots: 0 producer waits on empty, 1 MMA waits on tempty, 2 MMA waits
// on full, 3 epilogue waits on tfull (probe pass), 4 epilogue probe
// evaluation, 5 epilogue column staging, 6 epilogue waits on tfull (full
// tiles), 7 epilogue full-tile epilogue, 8 kernel cycles (warp 0, per CTA)
constexpr int GRAM_TIMING_SLOTS = 9;

// k-blocks of a tile: 0..KB-1 (dense) or the common set bits of two panel masks
struct KIter {
    const unsigned long long* a;
    const unsigned long long* b;
    int32_t words, w, next_dense, kb_end;
    unsigned long long cur;
    __device__ __forceinline__ void init(const GramArgs& g, int32_t P, int32_t J, int32_t KB) {
        if (g.mask) {
            a = g.mask + (int64_t)P * g.mask_words;
            b = g.mask + (int64_t)J * g.mask_words;
            words = g.mask_words;
            w = 0;
            cur = words ? (a[0] & b[0]) : 0ull;
        } else {
            a = nullptr;
            next_dense = 0;
            kb_end = KB;
        }
    }
    __device__ __forceinline__ int32_t next() {
        if (!a) return next_dense < kb_end ? next_dense++ : -1;
        while (!cur && ++w < words) cur = a[w] & b[w];
        if (!cur) return -1;
        const int32_t kb = w * 64 + __ffsll((long long)cur) - 1;
        cur &= cur - 1;
        return kb;
    }
    __device__ __forceinline__ bool empty(const GramArgs& g, int32_t P, int32_t J) const {
        if (!g.mask) return false;
        for (int32_t q = 0; q < g.mask_words; ++q)
            if (g.mask[(int64_t)P * g.mask_words + q] & g.mask[(int64_t)J * g.mask_words + q]) return false;
        return true;
    }
};

__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ ItemVals load_item(const GramArgs& a, int32_t idx, bool valid) {
    ItemVals v;
    v.a = valid ? __ldg(a.va + idx) : 0;
    v.b = (valid && a.vb) ? __ldg(a.vb + idx) : 0;
    return v;
}

// Probe terms of the DP / MD probe (epilogue.cuh probe_term_f: a pair can
// fire only if c' - b_j >= L_i or c' - L_j >= b_i), one CTA (8 warps) per
// column panel J of bn items (240 FP4, 256 int8) in [P_lo, P_hi):
//   pv[j]  = {L_j, b_j} for the items of [j_lo, j_hi) (a streamed round 1
//            refreshes only the rows its chunk completed; the panel's other
//            items keep theirs and are read back for the minima);
//   pcm    = per 32-column chunk {min L, min b} (warp w = chunk w; chunk 7
//            holds 16 columns; +inf for a chunk without items);
//   pb[J]  = (DP, optional) the panel's one demand, NaN when mixed.
// One launch per probe launch (and per band) instead of three.
template <int PHASE>
__global__ void __launch_bounds__(256)
probe_terms(const int32_t* __restrict__ dev_mk, int32_t M0, const int32_t* __restrict__ va,
            const int32_t* __restrict__ vb, const int32_t* __restrict__ lo, float2* __restrict__ pv,
            float2* __restrict__ pcm, float* __restrict__ pb, int32_t j_lo, int32_t j_hi, int32_t P_lo,
            int32_t bn) {
    mhsk::pdl_enter();
    const int32_t M = dev_mk ? dev_mk[0] : M0;
    const int32_t J = P_lo + blockIdx.x, t = threadIdx.x, w = t / 32;   // bn <= blockDim.x = 256
    const int32_t j = J * bn + t;
    if (J * bn >= M) return;   // CTA-uniform
    const bool item = t < bn && j < M;
    float2 v = make_float2(INFINITY, INFINITY);
    int32_t b = 0;
    if (item) {
        b = vb ? vb[j] : 0;
        if (j >= j_lo && j < j_hi) {
            v = make_float2(probe_term_f<PHASE>(va[j], b, lo[j]), PHASE == PHASE_SE ? 0.f : (float)b);
            pv[j] = v;
        } else {
            v = pv[j];
        }
    }
    float lmin = v.x, bmin = v.y;
    for (int o = 16; o > 0; o >>= 1) {
        lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        bmin = fminf(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
    }
    if (t % 32 == 0) pcm[J * 8 + w] = make_float2(lmin, bmin);
    if (pb) {
        int32_t blo = item ? b : 0x7fffffff, bhi = item ? b : -0x7fffffff;
        for (int o = 16; o > 0; o >>= 1) {
            blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
            bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        __shared__ int32_t slo[8], shi[8];
        if (t % 32 == 0) { slo[w] = blo; shi[w] = bhi; }
        __syncthreads();
        if (t == 0) {
            for (int q = 1; q < 8; ++q) { blo = min(blo, slo[q]); bhi = max(bhi, shi[q]); }
            pb[J] = blo == bhi ? (float)blo : __int_as_float(0x7fc00000);
        }
    }
}

constexpr int32_t CAND_WARP_CAP = 8;   // candidate pairs a warp may append per tile
constexpr int32_t CAND_CAP = 1 << 20;  // candidate buffer (entries); overflowing tiles are marked

// Reserve slots for this warp's candidates (n_l per lane).  false: the warp
// has too many (or none, or the buffer is full) -- the caller marks the tile.
__device__ __forceinline__ bool cand_reserve(const GramArgs& a, int32_t n_l, uint32_t lane, int32_t& slot) {
    int32_t incl = n_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0 || total > CAND_WARP_CAP) return false;
    int32_t base = 0;
    if (lane == 0) base = atomicAdd(a.cand_count, total);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + total > a.cand_cap) {   // full: neutralise the slots reserved inside the buffer
        for (int32_t s = base + (int32_t)lane; s < min(base + total, a.cand_cap); s += 32)
            a.cand[s] = make_int4(-1, -1, 0, 0);
        return false;
    }
    slot = base + incl - n_l;
    MHSK_CHECK(slot >= 0 && slot + n_l <= a.cand_cap);
    return true;
}

// FP4 = false: int8 0/1 operands, kind::i8, two TMEM accumulators.
// FP4 = true:  packed E2M1 0/1 operands (two items per byte), kind::mxf4 at
//              twice the i8 rate, one accumulator (the scale factors take the
//              rest of TMEM), f32 counts converted in the epilogue.
// RECT = false: symmetric triangle of X.X^T (tmA = tmB = X).
// RECT = true:  rectangle X_aff.X^T for incremental rounds (tmA = the affected
// rows, tmB = all rows); tiles (P, J) with P over affected-row panels; the
// epilogue applies rect_predicate (edge phase: hits to columns; vertex phase:
// hits to rows).
template <int PHASE, bool RECT = false, bool SPARSE = false, bool FP4 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
gram_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GramArgs args) {
    mhsk::pdl_enter();
    static_assert(!(SPARSE && FP4), "block-sparse masks are in int8 k-blocks");
    // tile columns (B panel rows): 256 (int8) or 240 (FP4, see BN_FP4)
    constexpr int TBN = FP4 ? BN_FP4 : BN;
    constexpr int HALF_B = TBN / 2;            // B rows held by each CTA
    constexpr int B_STAGE = HALF_B * BK;
    constexpr int STAGE_T = A_BYTES + B_STAGE;
    constexpr int NUM_ACC = 2;
    constexpr int BK_ITEMS = FP4 ? BK_ITEMS_FP4 : BK_ITEMS_I8;
    if (args.enable && *args.enable == 0) return;   // uniform across the cluster
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (SW128 atoms), by pointer arithmetic on the shared
    // array so the compiler keeps shared-space (LDS/STS) accesses
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stage_a = smem;
    uint8_t* stage_b = smem + STAGES * A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_T);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* adone = tempty + 2;    // probe pass done: every epilogue warp of the pair arrives
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(adone + 1);
    int4* colvals = reinterpret_cast<int4*>(smem + STAGES * STAGE_T + 256);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int32_t pair = blockIdx.x / 2, npairs = gridDim.x / 2;

    const long long t_start = clock64();
    // per-warp role counters in shared memory (registers would cost every
    // launch ~18 registers for a diagnostics-only feature); lanes race on
    // them, which keeps roughly one lane's total -- enough for diagnostics
    __shared__ long long tm_s[NUM_THREADS / 32][GRAM_TIMING_SLOTS];
    long long* tm = tm_s[threadIdx.x / 32];
    // role counters only in a diagnostics build (-DMHSK_GRAM_TIMING, the
    // MHSK_GRAM_TIMING environment variable): the checks alone cost the MMA
    // issuer ~16 of its ~120 instructions per k-block, and that warp's issue
    // rate, not the tensor pipe, set the probe's pace (ncu source page)
#ifdef MHSK_GRAM_TIMING
    if (args.timing && threadIdx.x % 32 < GRAM_TIMING_SLOTS) tm[threadIdx.x % 32] = 0;
    const bool timing = args.timing != nullptr;
#else
    constexpr bool timing = false;
#endif
#define GRAM_TIMED(slot, stmt)                         \
    do {                                               \
        const long long t0_ = timing ? clock64() : 0;  \
        stmt;                                          \
        if (timing) tm[slot] += clock64() - t0_;       \
    } while (0)
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
            ptx::mbar_init(&tempty[a], 2 * EPI_WARPS);   // epilogue warps x 2 CTAs (leader's copy used)
        }
        ptx::mbar_init(adone, 2 * EPI_WARPS);
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc_pair(tmem_slot, TMEM_COLS);
        ptx::tmem_relinquish_pair();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if constexpr (FP4) {
        // scale factors = UE8M0 2^0 in every column the MMA may read, both CTAs
        if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4) {
            const uint32_t lanes = (uint32_t)((warp - EPI_WARP0) * 32) << 16;
#pragma unroll
            for (int c = 0; c < SF_COLS; c += 8) ptx::tmem_st_x8(tmem_base + lanes + SF_COL + c, 0x7F7F7F7Fu);
            ptx::tmem_st_wait();
        }
        ptx::tc_fence_before();
        ptx::cluster_sync();
        ptx::tc_fence_after();
    }
    int32_t M = args.M, KB = args.k_blocks;
    if (args.dev_mk) {
        M = args.dev_mk[0];
        KB = max(1, (args.dev_mk[1] + BK_ITEMS - 1) / BK_ITEMS);
    }
    const int32_t NJ = (M + TBN - 1) / TBN;   // column panels J >= NJ hold no item
    int32_t A = M;                          // rows of the A operand
    if constexpr (RECT) A = *args.a_count;
    const int32_t NP = (A + BM - 1) / BM;
    const bool eval_zero_tiles = SPARSE && args.zero_needed && *args.zero_needed != 0;
    // probe pruning (epilogue.cuh), two passes over this pair's tiles:
    //   pass 0  every tile, K = the probe's k-blocks; the epilogue marks the
    //           tiles where some pair can still fire in the `needed` bitmap
    //   pass 1  the marked tiles, full K, normal epilogue
    // All roles walk the same tiles; pass 1 starts after `adone` (all marks in).
    // Without probing there is only pass 1 over every tile.
    const int32_t probe_kb =
        (!RECT && !SPARSE && args.lo && args.needed && args.probe_kb > 0 &&
         (args.force_probe || PROBE_MIN_RATIO * args.probe_kb <= KB))
            ? min(args.probe_kb, KB) : 0;
    const bool two_pass = probe_kb > 0;
    // passes of this launch: [pass_lo, pass_hi); pass 1 waits for `adone` only
    // when this launch also ran pass 0 (otherwise the marks are from an
    // earlier launch on the stream)
    const int pass_lo = two_pass && args.passes != 2 ? 0 : 1;
    const int pass_hi = two_pass && args.passes == 1 ? 1 : 2;
    const bool wait_marks = pass_lo == 0 && pass_hi == 2;
    uint32_t* needed = two_pass ? args.needed + (int64_t)pair * args.needed_words : nullptr;
    int32_t* progress = two_pass ? nullptr : args.progress;   // no K-drift throttle with probing
    // pass 1 of a two-pass schedule: was tile t (t-th of this pair) marked?
    // the t-th tile of this pair (list entry pair + t * npairs) to visit next,
    // from t on: every tile, or in pass 1 of a two-pass schedule the next
    // marked one (scanning the bitmap a word at a time); -1 = none
    auto next_t = [&](int pass, int32_t t) -> int32_t {
        if (!(pass == 1 && two_pass))
            return pair + t * npairs < args.tile_count && (pass == 1 || t < args.t_hi) ? t : -1;
        int32_t w = t >> 5;
        if (w >= args.needed_words) return -1;
        uint32_t bits = *((volatile uint32_t*)(needed + w)) & (0xFFFFFFFFu << (t & 31));
        while (!bits) {
            if (++w >= args.needed_words) return -1;
            bits = *((volatile uint32_t*)(needed + w));
        }
        t = w * 32 + __ffs((int)bits) - 1;
        return pair + t * npairs < args.tile_count ? t : -1;
    };
    // list entry of the t-th tile; every role loads the next tile's entry one
    // iteration ahead, so no tile starts with an exposed L2 round trip
    auto tile_entry = [&](int32_t t) -> uint32_t {
        return t >= 0 ? __ldg(args.tiles + args.tile_begin + (pair + t * npairs) * args.tile_stride) : 0u;
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        // the whole warp walks the schedule (uniform operands); one elected
        // lane arms the barrier and issues each stage's loads
        {
            int stage = 0;
            uint32_t phase = 0;
            for (int pass = pass_lo; pass < pass_hi; ++pass) {
            if (pass == 1 && wait_marks) ptx::mbar_wait_acq_cluster(adone, 0);
            const int32_t kb_end = pass == 0 ? probe_kb : KB;
            int32_t tn = next_t(pass, pass == 0 ? args.t_lo : 0);
            uint32_t pjn = tile_entry(tn);
            for (int32_t t = tn; t >= 0; t = tn) {
                const uint32_t pj = pjn;
                tn = next_t(pass, t + 1);
                pjn = tile_entry(tn);
                const int32_t wave = t;
                const int32_t wave_pairs = min(npairs, args.tile_count - wave * npairs);
                const int32_t P = pj & 0xFFFF, J = pj >> 16;
                if (J >= NJ || P >= NP) {   // outside the current sizes: counts as fully loaded
                    if (leader && progress && lane == 0)
                        atomicAdd(progress + wave, (KB + (1 << args.chunk_log2) - 1) >> args.chunk_log2);
                    continue;
                }
                const int32_t a_row = P * BM + (int32_t)rank * HALF;
                const int32_t b_row = J * TBN + (int32_t)rank * HALF_B;
                KIter ki;
                if constexpr (SPARSE) ki.init(args, P, J, KB);
                for (int32_t kb = SPARSE ? ki.next() : 0; SPARSE ? kb >= 0 : kb < kb_end;
                     kb = SPARSE ? ki.next() : kb + 1) {
                    if (leader && progress && (kb & ((1 << args.chunk_log2) - 1)) == 0) {
                        // throttle: stay within `slack` chunks of this wave's average
                        const int32_t c = kb >> args.chunk_log2;
                        if (c > 0 && lane == 0) atomicAdd(progress + wave, 1);   // chunk c-1 loaded
                        const int32_t need = (c - args.slack) * wave_pairs;
                        if (need > 0) {
                            const long long start = clock64();
                            while (ld_acquire(progress + wave) < need) {
                                __nanosleep(64);
                                if (clock64() - start > (1ll << 34)) __trap();
                            }
                        }
                    }
                    // spin (a sleeping producer measured 2% slower on config 4)
                    if (args.tune & 1) GRAM_TIMED(0, ptx::mbar_wait_sleep(&empty[stage], phase ^ 1));
                    else GRAM_TIMED(0, ptx::mbar_wait(&empty[stage], phase ^ 1));
                    const uint32_t full_leader = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
                    ptx::tma_stage_pair_elect(ptx::smem_u32(&full[stage]), leader ? 1u : 0u, 2 * STAGE_T, full_leader,
                                              ptx::smem_u32(stage_a + stage * A_BYTES), &tmA, kb * BK, a_row,
                                              (args.tune & 2) ? ptx::kEvictLast : ptx::kEvictNormal, 1u,
                                              ptx::smem_u32(stage_b + stage * B_STAGE), &tmB, b_row, ptx::kEvictLast);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (leader && progress && lane == 0) atomicAdd(progress + wave, 1);  // last chunk loaded
            }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader only)
        // the whole warp walks the schedule in lock-step (uniform operands);
        // one elected lane issues each k-block's MMAs and commits
        if (leader) {
            constexpr uint32_t idesc = FP4 ? ptx::idesc_mxf4(BM, TBN) : ptx::idesc_i8(BM, TBN);
            const uint32_t sfa = tmem_base + SF_COL, sfb = tmem_base + SF_COL + SF_COLS / 2;
            // stage descriptors = stage 0's + the stage offset (the start
            // address field is addr >> 4, < 2^14 for any shared address)
            const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(stage_a));
            const uint64_t bdesc0 = ptx::smem_desc_sw128(ptx::smem_u32(stage_b));
            const uint32_t empty0 = ptx::smem_u32(&empty[0]);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            long long probed = 0, full_tiles = 0;
            for (int pass = pass_lo; pass < pass_hi; ++pass) {
            if (pass == 1 && wait_marks) ptx::mbar_wait_acq_cluster(adone, 0);
            const int32_t kb_end = pass == 0 ? probe_kb : KB;
            int32_t tn = next_t(pass, pass == 0 ? args.t_lo : 0);
            uint32_t pjn = tile_entry(tn);
            for (int32_t t = tn; t >= 0; t = tn) {
                const uint32_t pj = pjn;
                tn = next_t(pass, t + 1);
                pjn = tile_entry(tn);
                const int32_t P = pj & 0xFFFF, J = pj >> 16;
                if (J >= NJ || P >= NP) continue;
                ++(pass == 0 ? probed : full_tiles);
                KIter ki;
                if constexpr (SPARSE) {
                    ki.init(args, P, J, KB);
                    if (ki.empty(args, P, J)) continue;   // no MMA: skipped, or c = 0 in the epilogue
                }
                GRAM_TIMED(1, ptx::mbar_wait(&tempty[acc], acc_phase ^ 1));
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TBN);
                bool first = true;
                static_assert(BK / UMMA_K == 4, "mma4_*: four 32-byte K steps per k-block");
                for (int32_t kb = SPARSE ? ki.next() : 0; SPARSE ? kb >= 0 : kb < kb_end;
                     kb = SPARSE ? ki.next() : kb + 1) {
                    GRAM_TIMED(2, ptx::mbar_wait(&full[stage], phase));
                    ptx::tc_fence_after();
                    const uint64_t adesc = adesc0 + (uint64_t)(stage * (A_BYTES >> 4));
                    const uint64_t bdesc = bdesc0 + (uint64_t)(stage * (B_STAGE >> 4));
                    if constexpr (FP4)
                        ptx::mma4_mxf4_pair_commit(d_tmem, adesc, bdesc, idesc, first ? 1u : 0u,
                                                   empty0 + 8u * (uint32_t)stage, 0x3, sfa, sfb);
                    else
                        ptx::mma4_i8_pair_commit(d_tmem, adesc, bdesc, idesc, first ? 1u : 0u,
                                                 empty0 + 8u * (uint32_t)stage, 0x3);
                    first = false;
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::commit_pair_elect(ptx::smem_u32(&tfull[acc]), 0x3);
                if (++acc == NUM_ACC) { acc = 0; acc_phase ^= 1; }
                if constexpr (SPARSE) {
                    if (args.kblocks_done && lane == 0) {
                        // k-blocks of this tile (re-walk the mask; cheap next to the MMAs)
                        KIter kc;
                        kc.init(args, P, J, KB);
                        unsigned long long nkb = 0;
                        while (kc.next() >= 0) ++nkb;
                        atomicAdd(args.kblocks_done, nkb);
                    }
                }
            }
            }
            // tiles stopped after the probe: probed - full (a full-pass-only
            // launch subtracts its tiles from its probe launch's count)
            if (lane == 0 && two_pass && args.pruned_tiles && probed != full_tiles)
                atomicAdd(args.pruned_tiles, (unsigned long long)(probed - full_tiles));
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------------------------ epilogue (both CTAs)
        const int e = warp - EPI_WARP0;
        const int q = e & 3;                     // TMEM lane quarter (rows 32q..32q+31)
        const int c0 = (e >> 2) * (EPI_COLS / 32), c1 = c0 + EPI_COLS / 32;   // its 32-column chunks
        int4* colv = colvals + e * EPI_COLS;
        const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = ptx::mapa(ptx::smem_u32(&tempty[1]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        // FP4 DP / MD probe: {L_j, b_j} of this warp's columns from pv, copied
        // into one of two 1 KB halves of its smem slice by cp.async one tile
        // ahead (issued behind the previous tile's evaluation, no registers);
        // columns >= M are zero-filled (excluded by the validity checks)
        int32_t pf_J = -1, cb = 0;
        auto prefetch_cols = [&](int32_t Jn, int buf) {
            float2* dst = reinterpret_cast<float2*>(colv) + buf * EPI_COLS;
#pragma unroll
            for (int c = 0; c < EPI_COLS / 32; ++c) {
                const int32_t jl = Jn * TBN + (c0 + c) * 32 + (int32_t)lane;
                ptx::cp_async_8(ptx::smem_u32(dst + c * 32 + lane), args.pv + min(jl, M - 1), jl < M ? 8u : 0u);
            }
            ptx::cp_async_commit();
            pf_J = Jn;
        };
        for (int pass = pass_lo; pass < pass_hi; ++pass) {
        if (pass == 1 && wait_marks) ptx::mbar_wait_acq_cluster(adone, 0);
        int32_t tn = next_t(pass, pass == 0 ? args.t_lo : 0);
        uint32_t pjn = tile_entry(tn);
        for (int32_t t = tn; t >= 0; t = tn) {
            const uint32_t pj = pjn;
            tn = next_t(pass, t + 1);
            pjn = tile_entry(tn);
            const int32_t P = pj & 0xFFFF, J = pj >> 16;
            if (J >= NJ || P >= NP) continue;
            bool zero_tile = false;
            if constexpr (SPARSE) {
                KIter ki;
                ki.init(args, P, J, KB);
                zero_tile = ki.empty(args, P, J);
                if (zero_tile && !eval_zero_tiles) continue;
            }
            const int32_t warp_row0 = P * BM + (int32_t)rank * HALF + q * 32;
            const int32_t prow = warp_row0 + (int32_t)lane;            // A-operand row
            const bool row_valid = prow < A;
            // item of this row: itself (triangle) or the affected item (rect)
            const int32_t i = RECT ? (row_valid ? __ldg(args.a_items + prow) : -1) : prow;
            // (the FP4 DP / MD probe reads its row values from pv instead)
            const ItemVals vi = (pass == 0 && args.pv) ? ItemVals{0, 0}
                                                                                  : load_item(args, i, row_valid);
            const int32_t rank_i = (SPARSE && args.rank && row_valid) ? __ldg(args.rank + i) : i;
            int32_t row_hits = 0;
            const long long t_stage = timing ? clock64() : 0;
            // this warp's column values, staged in its smem slice before the
            // accumulator is ready (the loads overlap the MMAs): {a, b, rank}
            // (pass 1) or {a - b (DP) | a, b, a - lo} (pass 0, the probe);
            // FP4 DP / MD probe: {L_j, b_j} from pv, prefetched into registers
            // during the previous tile's evaluation
            if (pass == 0 && args.pv) {
                if (pf_J != J) {   // not prefetched (first tile of the pass)
                    ptx::cp_async_wait_all();
                    prefetch_cols(J, cb);
                }
                ptx::cp_async_wait_all();
                pf_J = -1;
            } else
#pragma unroll
            for (int c = 0; c < EPI_COLS / 32; ++c) {
                const int32_t jl = J * TBN + (c0 + c) * 32 + (int32_t)lane;
                const bool ok = jl < M;
                const int32_t a = ok ? __ldg(args.va + jl) : 0;
                const int32_t b = (ok && args.vb) ? __ldg(args.vb + jl) : 0;
                int4 v;
                if (pass == 0) {
                    v.x = PHASE == PHASE_DP ? a - b : a;
                    v.z = ok ? a - __ldg(args.lo + jl) : 0;
                    if constexpr (FP4) {   // the FP4 probe compares in f32 (exact below 2^23)
                        v.x = __float_as_int(ok ? probe_term_f<PHASE>(a, b, a - v.z) : __int_as_float(0x7f800000));
                        v.y = __float_as_int((float)b);
                    } else {
                        v.y = b;
                    }
                } else {
                    v.x = a;
                    v.z = (SPARSE && args.rank && ok) ? __ldg(args.rank + jl) : jl;
                }
                if (pass != 0) v.y = b;
                v.w = 0;
                if (FP4 && PHASE != PHASE_SE && pass == 0)   // {L_j, b_j} pairs (probe_split_f)
                    reinterpret_cast<float2*>(colv)[c * 32 + lane] =
                        make_float2(__int_as_float(v.x), __int_as_float(v.y));
                else
                    colv[c * 32 + lane] = v;
            }
            __syncwarp();
            if (timing) tm[5] += clock64() - t_stage;

            if (pass == 0) {
                // ---- probe: can any pair of this tile still fire after K1?
                // row values: FP4 DP / MD from pv (only); otherwise from a, b, lo
                // (int8 too: the s32 counts are converted to f32 as they are read)
                const bool from_pv = args.pv != nullptr;
                const int32_t rem_i = (row_valid && !from_pv) ? vi.a - __ldg(args.lo + i) : 0;
                const int32_t xi = PHASE == PHASE_DP ? vi.a - vi.b : vi.a;
                float Lif, bif;
                if (from_pv) {
                    const float2 r_ = __ldg(args.pv + min(i, M - 1));   // invalid rows: masked by row_valid
                    Lif = r_.x;
                    bif = r_.y;
                } else {
                    Lif = probe_term_f<PHASE>(vi.a, vi.b, vi.a - rem_i);
                    bif = (float)vi.b;
                }
                // one demand over the tile's columns: DP pb[J] (NaN when mixed); MD/SE probe with b = 0
                const float bu = PHASE != PHASE_DP ? 0.f
                               : args.pb ? __ldg(args.pb + J) : __int_as_float(0x7fc00000);
                const bool b_uni = bu == bu;
                // tile-list entry of the next tile (its columns are prefetched
                // behind this tile's evaluation)
                const uint32_t pj_next = tn >= 0 ? pjn : 0xFFFFFFFFu;
                const float2* colf = reinterpret_cast<const float2*>(colv) + cb * EPI_COLS;
                GRAM_TIMED(3, ptx::mbar_wait(&tfull[acc], acc_phase));
                ptx::tc_fence_after();
                const long long t_eval = timing ? clock64() : 0;
                bool any = false;
                // chunks with columns right of the diagonal and below M, two per TMEM wait
                const int32_t c_lo = max(c0, (warp_row0 - J * TBN + 1) / 32);
                const int32_t c_hi = min(c1, (M - J * TBN + 31) / 32);
                const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * TBN;
                const int32_t jend = min(M, J * TBN + TBN);   // columns of this tile: [J * TBN, jend)
    // FP4: branch-free slack, four independent max chains per chunk; int8: predicates
#define PROBE_EVAL_CHUNK(R, CC) PROBE_EVAL_CHUNK_W(R, CC, 32)
    // W = columns of the chunk (32, or 16 for the 240-column FP4 tile's last)
#define PROBE_EVAL_CHUNK_W(R, CC, W)                                                                     \
    {                                                                                                    \
        const int32_t j0_ = J * TBN + (CC) * 32;                                                         \
        const bool interior_ = j0_ + (W) - 1 < jend && j0_ > warp_row0 + 31;                             \
        const int4* cv_ = colv + ((CC) - c0) * 32;                                                       \
        if (from_pv) {                                                                                   \
            /* exists j with c' - b_j >= L_i or c' - L_j >= b_i (SE: b = 0), i.e. two row-wise */        \
            /* maxima over the chunk's columns, read as {L_j, b_j, L_j+1, b_j+1}; eight   */           \
            /* independent chains                                                          */           \
            const float4* cf_ = reinterpret_cast<const float4*>(colf) + ((CC) - c0) * 16;               \
            float u_[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};                                  \
            float w_[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};                                  \
            if (interior_ && b_uni) {                                                                    \
                /* DP, one demand b = bu over the tile's columns: max_j (c' - b_j) = max_j c' - bu */    \
                _Pragma("unroll") for (int q_ = 0; q_ < (W) / 2; ++q_) {                                 \
                    const float4 f_ = cf_[q_];                                                           \
                    const float x0_ = __uint_as_float(R[2 * q_]), x1_ = __uint_as_float(R[2 * q_ + 1]);  \
                    const int k_ = 2 * (q_ & 1);                                                         \
                    u_[k_] = fmaxf(u_[k_], fmaxf(x0_, x1_));                                             \
                    w_[k_] = fmaxf(w_[k_], x0_ - f_.x);                                                  \
                    w_[k_ + 1] = fmaxf(w_[k_ + 1], x1_ - f_.z);                                          \
                }                                                                                        \
                u_[0] -= bu; u_[2] -= bu;                                                                \
            } else if (interior_) {                                                                      \
                _Pragma("unroll") for (int q_ = 0; q_ < (W) / 2; ++q_) {                                 \
                    const float4 f_ = cf_[q_];                                                           \
                    const float x0_ = __uint_as_float(R[2 * q_]), x1_ = __uint_as_float(R[2 * q_ + 1]);  \
                    const int k_ = 2 * (q_ & 1);                                                         \
                    u_[k_] = fmaxf(u_[k_], PHASE != PHASE_DP ? x0_ : x0_ - f_.y);   /* MD/SE: b = 0 */   \
                    w_[k_] = fmaxf(w_[k_], x0_ - f_.x);                                                  \
                    u_[k_ + 1] = fmaxf(u_[k_ + 1], PHASE != PHASE_DP ? x1_ : x1_ - f_.w);                \
                    w_[k_ + 1] = fmaxf(w_[k_ + 1], x1_ - f_.z);                                          \
                }                                                                                        \
            } else {                                                                                     \
                _Pragma("unroll") for (int q_ = 0; q_ < (W) / 2; ++q_) {                                 \
                    const float4 f_ = cf_[q_];                                                           \
                    const int32_t ja_ = j0_ + 2 * q_;                                                    \
                    const bool ok0_ = ja_ < jend && i < ja_, ok1_ = ja_ + 1 < jend && i < ja_ + 1;       \
                    const float x0_ = __uint_as_float(R[2 * q_]), x1_ = __uint_as_float(R[2 * q_ + 1]);  \
                    u_[0] = fmaxf(u_[0], ok0_ ? x0_ - f_.y : -INFINITY);                                 \
                    w_[0] = fmaxf(w_[0], ok0_ ? x0_ - f_.x : -INFINITY);                                 \
                    u_[1] = fmaxf(u_[1], ok1_ ? x1_ - f_.w : -INFINITY);                                 \
                    w_[1] = fmaxf(w_[1], ok1_ ? x1_ - f_.z : -INFINITY);                                 \
                }                                                                                        \
            }                                                                                            \
            mine |= fmaxf(fmaxf(u_[0], u_[1]), fmaxf(u_[2], u_[3])) >= Lif ||                            \
                    fmaxf(fmaxf(w_[0], w_[1]), fmaxf(w_[2], w_[3])) >= bif;                              \
        } else if (FP4) {                                                                                \
            float m_[4] = {-1.f, -1.f, -1.f, -1.f};                                                      \
            if (interior_) {                                                                             \
                _Pragma("unroll") for (int jj = 0; jj < (W); ++jj) {                                     \
                    const int4 v = cv_[jj];                                                              \
                    m_[jj & 3] = fmaxf(m_[jj & 3], pair_slack_f<PHASE>(__uint_as_float(R[jj]), Lif, bif, \
                                                                       __int_as_float(v.x),              \
                                                                       __int_as_float(v.y)));            \
                }                                                                                        \
            } else {                                                                                     \
                _Pragma("unroll") for (int jj = 0; jj < 32; ++jj) {                                      \
                    const int4 v = cv_[jj];                                                              \
                    float sl = pair_slack_f<PHASE>(__uint_as_float(R[jj]), Lif, bif, __int_as_float(v.x), \
                                                   __int_as_float(v.y));                                 \
                    if (!(j0_ + jj < jend && i < j0_ + jj)) sl = -1.f;                                   \
                    m_[jj & 3] = fmaxf(m_[jj & 3], sl);                                                  \
                }                                                                                        \
            }                                                                                            \
            mine |= fmaxf(fmaxf(m_[0], m_[1]), fmaxf(m_[2], m_[3])) >= 0.f;                              \
        } else {                                                                                         \
            _Pragma("unroll") for (int jj = 0; jj < 32; ++jj) {                                          \
                const int4 v = cv_[jj];                                                                  \
                const bool pos = pair_possible<PHASE>((int32_t)R[jj], xi, vi.b, rem_i, v.x, v.y, v.z);   \
                mine |= pos && (interior_ || (j0_ + jj < jend && i < j0_ + jj));                         \
            }                                                                                            \
        }                                                                                                \
    }
                if (FP4 || from_pv) {
                    // read all of this warp's live chunks, hand the accumulator
                    // back to the MMA at once, then evaluate from registers
                    // chunk by chunk (32 registers of counts at a time): load, evaluate;
                    // the accumulator goes back to the MMA after the last chunk
                    // (and after the rare candidate listing, which re-reads it).
                    // The next tile's column values are fetched behind this.
                    if (args.pv && pj_next != 0xFFFFFFFFu)   // next tile's columns
                        prefetch_cols((int32_t)(pj_next >> 16), cb ^ 1);
                    bool mine = false;
                    uint32_t ra[32];
#pragma unroll 1
                    for (int c = max(c0, c_lo); c < min(c1, c_hi); ++c) {
                        // the 240-column tile's last chunk holds 16 columns
                        const bool half = (TBN % 32) != 0 && c == TBN / 32;
                        const float2 cm = args.pcm ? __ldg(args.pcm + J * 8 + c)
                                                                            : make_float2(-INFINITY, -INFINITY);
                        if (half) ptx::tmem_ld_32x32b_x16(tbase + c * 32, ra);
                        else ptx::tmem_ld_32x32b_x32(tbase + c * 32, ra);
                        ptx::tmem_ld_wait();
                        if constexpr (!FP4) {   // int8: exact s32 counts -> f32
#pragma unroll
                            for (int z = 0; z < 32; ++z) ra[z] = __float_as_uint((float)(int32_t)ra[z]);
                        }
                        if (args.pcm) {
                            // chunk pre-test (necessary condition): the largest
                            // count against the chunk's smallest L and b.  Counts
                            // of pairs outside the triangle only loosen it.
                            float xm = -INFINITY;
                            if (half) {
#pragma unroll
                                for (int z = 0; z < 16; ++z) xm = fmaxf(xm, __uint_as_float(ra[z]));
                            } else {
#pragma unroll
                                for (int z = 0; z < 32; ++z) xm = fmaxf(xm, __uint_as_float(ra[z]));
                            }
                            const bool maybe = xm - cm.y >= Lif || xm - cm.x >= bif;
                            if (!__any_sync(0xffffffffu, maybe && row_valid)) continue;
                        }
                        if (half) PROBE_EVAL_CHUNK_W(ra, c, 16)
                        else PROBE_EVAL_CHUNK(ra, c)
                    }
                    any = __any_sync(0xffffffffu, mine && row_valid);
                    if (any) {   // rare: list the candidate pairs, or mark the tile
                        bool mark = true;
                        if (args.cand) {
                            const uint32_t bit = (uint32_t)(pair * args.needed_words) * 32u + (uint32_t)t;
#define CAND_SCAN_FP4(R, CC, ACTION)                                                                      \
    {                                                                                                     \
        const int32_t j0_ = J * TBN + (CC) * 32;                                                          \
        const int4* cv_ = colv + ((CC) - c0) * 32;                                                        \
        _Pragma("unroll") for (int jj = 0; jj < 32; ++jj) {                                               \
            float Lj_, bj_;                                                                               \
            if (from_pv) {                                                                                \
                const float2 f_ = colf[((CC) - c0) * 32 + jj];                                            \
                Lj_ = f_.x;                                                                               \
                bj_ = f_.y;                                                                               \
            } else {                                                                                      \
                Lj_ = __int_as_float(cv_[jj].x);                                                          \
                bj_ = __int_as_float(cv_[jj].y);                                                          \
            }                                                                                             \
            const bool ok_ = row_valid && j0_ + jj < jend && i < j0_ + jj &&                              \
                             pair_slack_f<PHASE>(__uint_as_float(R[jj]), Lif, bif, Lj_, bj_) >= 0.f;      \
            if (ok_) { ACTION; }                                                                          \
        }                                                                                                 \
    }
                            int32_t n_l = 0, slot = 0;
                            for (int pass_c = 0; pass_c < 2; ++pass_c) {
#pragma unroll 1
                                for (int c = max(c0, c_lo); c < min(c1, c_hi); ++c) {
                                    ptx::tmem_ld_32x32b_x32(tbase + c * 32, ra);   // columns >= jend masked
                                    ptx::tmem_ld_wait();
                                    if constexpr (!FP4) {
#pragma unroll
                                        for (int z = 0; z < 32; ++z) ra[z] = __float_as_uint((float)(int32_t)ra[z]);
                                    }
                                    if (pass_c == 0) CAND_SCAN_FP4(ra, c, ++n_l)
                                    else CAND_SCAN_FP4(ra, c, args.cand[slot++] = make_int4(i, j0_ + jj, (int32_t)bit, 0))
                                }
                                if (pass_c == 0 && !cand_reserve(args, n_l, lane, slot)) break;
                                if (pass_c == 1) mark = false;
                            }
#undef CAND_SCAN_FP4
                        }
                        if (lane == 0 && mark) {
                            atomicOr(needed + (t >> 5), 1u << (t & 31));
                            if (args.marked) *args.marked = 1;
                        }
                    }
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
                    if (timing) tm[4] += clock64() - t_eval;
                    if (++acc == NUM_ACC) { acc = 0; acc_phase ^= 1; }
                    if (args.pv) cb ^= 1;
                    continue;
                }
#pragma unroll 1
                for (int c = c_lo; c < c_hi && !any; c += 2) {
                    uint32_t ra[32], rb[32];
                    const bool two = c + 1 < c_hi;
                    bool mine = false;
                    ptx::tmem_ld_32x32b_x32(tbase + c * 32, ra);
                    if (two) ptx::tmem_ld_32x32b_x32(tbase + (c + 1) * 32, rb);
                    ptx::tmem_ld_wait();
                    PROBE_EVAL_CHUNK(ra, c)
                    if (two) PROBE_EVAL_CHUNK(rb, c + 1)
                    any = __any_sync(0xffffffffu, mine && row_valid);
                }
#undef PROBE_EVAL_CHUNK
#undef PROBE_EVAL_CHUNK_W
                bool mark = any;
                if (any && args.cand) {   // rare: list the candidate pairs (chunks re-read from TMEM)
                    const uint32_t bit = (uint32_t)(pair * args.needed_words) * 32u + (uint32_t)t;
                    int32_t n_l = 0, slot = 0;
                    for (int pass_c = 0; pass_c < 2; ++pass_c) {
#pragma unroll 1
                        for (int c = c_lo; c < c_hi; ++c) {
                            uint32_t ra[32];
                            ptx::tmem_ld_32x32b_x32(tbase + c * 32, ra);
                            ptx::tmem_ld_wait();
                            const int32_t j0_ = J * TBN + c * 32;
                            const int4* cv_ = colv + (c - c0) * 32;
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) {
                                const int4 v = cv_[jj];
                                const bool ok_ = row_valid && j0_ + jj < jend && i < j0_ + jj &&
                                                 pair_possible<PHASE>((int32_t)ra[jj], xi, vi.b, rem_i, v.x, v.y, v.z);
                                if (ok_) {
                                    if (pass_c == 0) ++n_l;
                                    else args.cand[slot++] = make_int4(i, j0_ + jj, (int32_t)bit, 0);
                                }
                            }
                        }
                        if (pass_c == 0 && !cand_reserve(args, n_l, lane, slot)) break;
                        if (pass_c == 1) mark = false;
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
                    if (mark) {
                        atomicOr(needed + (t >> 5), 1u << (t & 31));
                        if (args.marked) *args.marked = 1;
                    }
                }
                if (timing) tm[4] += clock64() - t_eval;
                if (++acc == NUM_ACC) { acc = 0; acc_phase ^= 1; }
                continue;
            }

            if (!SPARSE || !zero_tile) {
                GRAM_TIMED(6, ptx::mbar_wait_sleep(&tfull[acc], acc_phase, 64));
                ptx::tc_fence_after();
            }
            const long long t_epi = timing ? clock64() : 0;
            const int32_t jend_t = min(M, J * TBN + TBN);   // columns of this tile: [J * TBN, jend_t)
#pragma unroll 1
            for (int c = c0; c < c1; ++c) {
                const int32_t j0 = J * TBN + c * 32;
                if (j0 >= M) break;
                if (!RECT && j0 + 31 <= warp_row0) continue;
                uint32_t r[32];
                if (!SPARSE || !zero_tile) {
                    ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * TBN + c * 32, r);
                } else {
#pragma unroll
                    for (int z = 0; z < 32; ++z) r[z] = 0;
                }
                const int32_t jl = j0 + (int32_t)lane;
                if (!SPARSE || !zero_tile) ptx::tmem_ld_wait();
                if constexpr (FP4) {   // exact f32 counts (< 2^24) -> int
#pragma unroll
                    for (int z = 0; z < 32; ++z) r[z] = (uint32_t)__float2int_rz(__uint_as_float(r[z]));
                }
                if constexpr (!RECT && (PHASE == PHASE_MD || SPARSE)) {
                    // a 32x32 block of zero counts decides nothing: MD needs
                    // c == d >= 1 (degree-0 vertices are deleted regardless),
                    // DP/SE need c >= 1 unless *zero_needed
                    if (PHASE == PHASE_MD || !eval_zero_tiles) {
                        uint32_t nz = 0;
#pragma unroll
                        for (int z = 0; z < 32; ++z) nz |= r[z];
                        if (!__any_sync(0xffffffffu, nz != 0)) continue;
                    }
                }
                uint32_t my_col_hits = 0;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    const int32_t j = j0 + jj;
                    const int4 v = colv[(c - c0) * 32 + jj];
                    ItemVals vj;
                    vj.a = v.x;
                    vj.b = v.y;
                    if constexpr (RECT) {
                        const bool ok = row_valid && j < jend_t && i != j &&
                                        rect_predicate<PHASE>((int32_t)r[jj], vi, vj, i, j);
                        if constexpr (PHASE == PHASE_MD) {
                            row_hits += ok ? 1 : 0;                 // column dominates row
                        } else {
                            const uint32_t b = __ballot_sync(0xffffffffu, ok);   // row deletes column
                            if (lane == (uint32_t)jj) my_col_hits = __popc(b);
                        }
                    } else {
                        bool i_del_j, j_del_i;
                        if constexpr (SPARSE) {
                            const int32_t rank_j = v.z;
                            pair_predicates_ranked<PHASE>((int32_t)r[jj], vi, vj, rank_i < rank_j, i_del_j,
                                                          j_del_i);
                        } else {
                            pair_predicates<PHASE>((int32_t)r[jj], vi, vj, i_del_j, j_del_i);
                        }
                        const bool handled = row_valid && j < jend_t && i < j;
                        row_hits += (handled && j_del_i) ? 1 : 0;
                        const uint32_t b = __ballot_sync(0xffffffffu, handled && i_del_j);
                        if (lane == (uint32_t)jj) my_col_hits = __popc(b);
                    }
                }
                if (my_col_hits) {
                    MHSK_CHECK(jl >= 0 && jl < M);
                    atomicAdd(args.hits + jl, (int32_t)my_col_hits);
                }
            }
            if (row_hits) {
                MHSK_CHECK(i >= 0 && i < M);
                atomicAdd(args.hits + i, row_hits);
            }
            if (timing) tm[7] += clock64() - t_epi;
            if (SPARSE && zero_tile) continue;   // no accumulator was used
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
            if (++acc == NUM_ACC) { acc = 0; acc_phase ^= 1; }
        }
        if (pass == 0) {   // this warp's marks are in: release them to both CTAs
            if (args.pv) ptx::cp_async_wait_all();   // no copy outlives the pass
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                ptx::mbar_arrive_cluster_release(ptx::mapa(ptx::smem_u32(adone), 0));
                ptx::mbar_arrive_cluster_release(ptx::mapa(ptx::smem_u32(adone), 1));
            }
        }
        }
    }

    if (timing) {
        __syncwarp();
        if (warp == 0 && lane == 0) tm[8] = clock64() - t_start;
        if (lane == 0 && (warp <= 1 || warp >= EPI_WARP0))
            for (int k = 0; k < GRAM_TIMING_SLOTS; ++k)
                if (tm[k]) atomicAdd(args.timing + k, (unsigned long long)tm[k]);
    }
#undef GRAM_TIMED
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
}

}  // namespace tc2
}  // namespace mhsk
