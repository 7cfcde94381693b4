// mhsk_capi.cu -- libmhsk.so: the C ABI (include/mhsk.h) and the device-side
// fixpoint driver of the kernelization (reference parallel.py:164-214).
//
// Per round, entirely on the device except for one 16-byte counter read per
// phase (the host needs the alive counts to size the next launch):
//   edge phase:   compact alive flags -> pack X_E (m' x n' int8) -> Gram DP/SE
//                 -> [allreduce hits] -> commit edge deletions
//   vertex phase: compact -> pack X_V (n' x m' int8, + deg, need) -> Gram MD
//                 -> [allreduce hits] -> commit vertex deletions
//   stop after the first round that deletes nothing (counted, as in the
//   reference).
#include <atomic>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mhsk.h"
#include "gram_tc.cuh"
#include "gram_tc2.cuh"
#include "generate.cuh"
#include "mhsk_kernels.cuh"
#include "schedule.h"
#include "verify.cuh"
#include <cub/device/device_radix_sort.cuh>

namespace {

thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

struct Failure {
    int code;
};

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,      \
                      __LINE__);                                                             \
            throw Failure{_e == cudaErrorMemoryAllocation ? MHSK_OOM : MHSK_CUDA_ERROR};     \
        }                                                                                    \
    } while (0)

#define LAUNCH_CHECK() CUDA_TRY(cudaGetLastError())

template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), cap(o.cap) { o.ptr = nullptr; o.cap = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            ptr = o.ptr;
            cap = o.cap;
            o.ptr = nullptr;
            o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void reserve(size_t n) {
        if (n <= cap) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 64);
        CUDA_TRY(cudaMalloc(&ptr, want * sizeof(T)));
        cap = want;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

// driver entry point for TMA descriptors (no -lcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            throw Failure{MHSK_CUDA_ERROR};
        }
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

CUtensorMap make_tmap(const int8_t* X, int64_t rows, int64_t ld, uint32_t box_rows) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)mhsk::tc::BK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)X, dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld ld=%lld", (int)r, (long long)rows,
                  (long long)ld);
        throw Failure{MHSK_CUDA_ERROR};
    }
    return tm;
}

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Device-side validation of the CSR (flags[0] invalid, flags[1] first
// infeasible edge + 1).
__global__ void validate_csr(int32_t n, int32_t m, const int64_t* __restrict__ ptr,
                             const int32_t* __restrict__ vtx, const int32_t* __restrict__ dem,
                             int32_t* __restrict__ flags) {
    mhsk::pdl_enter();
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int64_t nnz = ptr[m];
    for (int64_t e = warp; e < m; e += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int64_t lo = ptr[e], hi = ptr[e + 1];
        // offsets outside [0, nnz] are malformed and never dereferenced; so
        // is a null member array under a non-empty edge (device-pointer API),
        // and edge_ptr[0] != 0 (upload() checks that on the host path)
        bool bad = hi < lo || lo < 0 || hi > nnz || dem[e] < 1 || (e == 0 && lo != 0) ||
                   (vtx == nullptr && hi > lo);
        // 32*VU members per warp step, all loads independent: each lane
        // reads its member and the member's predecessor (an L1 hit on the
        // same lines) instead of a shuffle chain across the warp
        constexpr int VU = 8;
        for (int64_t p0 = lo; p0 < hi && !bad; p0 += 32 * VU) {
            int32_t v[VU], pv[VU];
#pragma unroll
            for (int u = 0; u < VU; ++u) {
                const int64_t p = p0 + 32 * u + lane;
                v[u] = p < hi ? __ldg(vtx + p) : 0x7fffffff;
                pv[u] = (p < hi && p > lo) ? __ldg(vtx + p - 1) : -1;
            }
#pragma unroll
            for (int u = 0; u < VU; ++u)
                if (p0 + 32 * u + lane < hi && (v[u] < 0 || v[u] >= n || pv[u] >= v[u])) bad = true;
            bad = __any_sync(0xffffffffu, bad);
        }
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            if (bad) atomicExch(flags, 1);
            else if ((int64_t)dem[e] > hi - lo) atomicMin(flags + 1, (int32_t)e + 1);
        }
    }
}

}  // namespace

void mhsk_internal_set_error(const std::string& msg) { g_last_error = msg; }

// Chunks: the work left after the last one lands is the last band of the
// edge probe, and each band launch has a fixed cost (partial waves, the
// scan / pack / probe-term launches) and slows under the concurrent copy.
// Measured at config 4 (e2e, one box, tools/e2e_trace.py): no streaming
// 12.35 ms; sqrt-spaced bounds 4 / 6 / 8 / 10 / 12 / 16 / 32 chunks 10.53 /
// 10.53 / 10.44 / 10.53 / 10.59 / 10.64 / 11.65 ms; uniform bounds 8 / 16 /
// 32: 10.71 / 10.55 / 11.05 ms.  Default then: 8, sqrt-spaced.  With the
// speculative vertex probe (plus a small first chunk holding just its edges):
// 8.06 ms at 8 chunks, 8.15 / 8.18 / 8.28 at 6 / 12 / 16; an extra small last
// chunk (1-4% of the members) 8.11 ms -- the upload itself ends at ~7.6 ms.
// After programmatic dependent launch and one probe-terms kernel per band
// (a band's fixed cost fell), 6 / 8 / 10 / 12 / 16 / 20 / 24 / 32 chunks:
// 8.05 / 7.99 / 7.97 / 7.94 / 7.92 / 7.96 / 8.08 / 8.43 ms (the member copy
// alone: 7.21 ms).  Default: 16.
constexpr int64_t STREAM_CHUNK = (int64_t)1 << 20;
constexpr int STREAM_MAX_CHUNKS = 32;
constexpr int STREAM_DEFAULT_CHUNKS = 16;
constexpr int64_t STREAM_MIN_MEMBERS = (int64_t)1 << 24;

// Host buffers that feed asynchronous uploads during a streamed call are
// pinned: a pageable cudaMemcpyAsync is staged synchronously and would wait
// for the copy engine behind the streamed member array, stalling the host
// (and with it the overlap) until the whole upload had landed.  A pinned
// source must not be rewritten until its copy has run: the tile lists in
// TileVecs are rebuilt only at a round start (after the previous round's
// sync) or, for the band list, after its event.
template <class T>
struct PinnedAlloc {
    using value_type = T;
    PinnedAlloc() = default;
    template <class U>
    PinnedAlloc(const PinnedAlloc<U>&) {}
    T* allocate(size_t n) {
        void* p = nullptr;
        if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t) { cudaFreeHost(p); }
    template <class U>
    bool operator==(const PinnedAlloc<U>&) const { return true; }
    template <class U>
    bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
using TileVec = std::vector<uint32_t, PinnedAlloc<uint32_t>>;

struct mhsk_ctx {
    int device = 0;
    int sms = 148;
    int backend = MHSK_BACKEND_TC;
    int rank = 0, world = 1;
    mhsk_allreduce_fn allreduce = nullptr;
    void* allreduce_user = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evg0 = nullptr, evg1 = nullptr;

    // instance (device copies for the host-pointer API)
    DevBuf<int64_t> edge_ptr;
    DevBuf<int32_t> edge_vtx, demand;
    DevBuf<uint8_t> valive, ealive, keep;
    // compaction
    DevBuf<int32_t> vnew, enew, vids, eids, scan_tmp;
    // per decided item
    DevBuf<int32_t> item_a, item_b, hits;
    DevBuf<int32_t> item_lo;                       // probe pruning: entries in the probe columns
    DevBuf<unsigned long long> pruned;             // [3]: tiles stopped after the probe (edge, vertex),
                                                   //      candidate pairs verified
    DevBuf<uint32_t> needed;                       // probe pass: per-pair bitmaps of undecided tiles
    unsigned long long* pruned_host = nullptr;     // pinned copy
    // full-edge rule state (mhsk_run_pipeline)
    DevBuf<int32_t> dem_work;
    DevBuf<uint8_t> fe_full, fe_forced;
    // operands: X (SIMT bit-packed), XE / XV (tensor-core int8, edge / vertex phase)
    DevBuf<int8_t> X, XE, XV;
    // X_E provenance: valid while the vertex compaction it was packed with is current
    bool xe_valid = false;
    int32_t xe_rows = 0, xe_cols = 0;
    int64_t xe_ld = 0;
    DevBuf<uint8_t> keep_e;       // survivors of the last edge phase (rows of X_E)
    DevBuf<int32_t> src, scratch; // X_V column -> X_E row map; compaction scratch
    // device-resident round loop (kernelize fast path)
    DevBuf<int32_t> dims;             // [0] m_a [1] n_a [2] m_a2 [3] del_e [4] del_v [5] spare
    int32_t* dims_host = nullptr;     // pinned
    DevBuf<uint32_t> tiles_e, tiles_v;
    TileVec tiles_e_host, tiles_v_host;
    int32_t tiles_e_M = -1, tiles_v_M = -1;
    bool fast_loop = true;            // MHSK_FAST_LOOP=0 selects the host-driven loop
    bool incremental = true;          // MHSK_INCREMENTAL=0: full triangle every round
    bool fp4 = true;                  // dense Gram on kind::mxf4 (packed E2M1 operands); MHSK_FP4=0: kind::i8
    bool probe = true;                // probe pruning of dense triangle tiles; MHSK_PROBE=0: off
    int32_t probe_entries = 0;   // vertex-probe length, entries of a mean item; 0 auto (MHSK_PROBE_ENTRIES)
    // edge-phase probe length: its candidate pairs are cheap (rows packed one by
    // one), the vertex phase's are not (panel transposes) -- measured 14 / 16
    int32_t probe_entries_e = 14;     // (0: probe_entries; MHSK_PROBE_ENTRIES_E)
    bool verify = true;               // candidate-pair verification of probed tiles; MHSK_VERIFY=0: off
    bool lazy = true;                 // lazy vertex operand (probe columns + undecided panels); MHSK_LAZY=0: off
    int32_t lg_pairs = 0, lg_words = 0, lg_begin = 0, lg_count = 0, lg_stride = 1;   // last Gram launch
    bool lg_cand = false;
    DevBuf<int32_t> vdeg, vneed;      // lazy vertex operand: degrees / need accumulated while packing X_E
    DevBuf<uint32_t> vseen;           // uniform demand: columns with a member (need = f * seen)
    DevBuf<int32_t> f_range;          // min / max demand of the packed rows
    DevBuf<uint8_t> panel_flags;      // lazy vertex operand: 256-row panels to pack in full
    bool lazy_e = true;               // lazy edge operand (probe columns + needed panels); MHSK_LAZY_E=0: off
    DevBuf<uint8_t> state_e;          // lazy edge operand: per 256-row panel 0 probe cols / 1 to pack / 2 full
    DevBuf<int32_t> pack_dummy;       // discarded size / demand outputs of panel re-packs
    DevBuf<int32_t> any_v;            // a vertex panel needs its full rows
    DevBuf<uint8_t> row_sel_e;        // lazy edge operand: candidate rows to pack in full
    bool vcsr = true;                 // vertex candidates counted from the CSR (vcand_*); MHSK_VCSR=0: panels
    // capacities of the candidate machinery (options "cand_cap", "vcand_max",
    // "vcand_table_log2"; result-neutral: smaller values only force the
    // overflow / fallback paths -- marked full-K tiles, panel transposes)
    int32_t cand_cap = mhsk::tc2::CAND_CAP;
    int32_t vcand_max = mhsk::k::VCAND_MAX;
    int32_t vcand_table_log2 = mhsk::k::VCAND_TABLE_LOG2;
    DevBuf<unsigned long long> vc_keys;
    DevBuf<int32_t> vc_cnt, vc_flag, vc_deg, vc_ok;
    DevBuf<int32_t> vc_heavy;   // vcand_count's deferred edges, then their count
    DevBuf<int32_t> vc_pcnt, vc_pslot;   // partner lists of the candidate pairs (vcand_partners)
    DevBuf<int4> cand;                // candidate pairs of the probe pass (verify.cuh)
    DevBuf<float2> pv;                // FP4 DP / MD probe values per item (probe_terms)
    DevBuf<float> pb;                 // FP4 DP probe: per column panel its one demand, or NaN
    DevBuf<float2> pcm;               // FP4 probe: per 32-column chunk min L / min b
    DevBuf<int32_t> cand_count;
    bool gram_timing = false;         // MHSK_GRAM_TIMING=1: per-role cycle counters (stderr; the
                                      // counters exist only in `make timing`'s libmhsk_timing.so)
    int gram_tune = 0;                // MHSK_GRAM_TUNE: Gram kernel experiments (GramArgs::tune)
    DevBuf<unsigned long long> timing;
    DevBuf<int8_t> XA;                // rectangle A operand (affected rows)
    DevBuf<uint8_t> edel, vdel, aff_flag;
    DevBuf<int32_t> aff_e_ids, aff_v_ids, a_items, aff_scratch;
    DevBuf<uint32_t> tiles_r;
    // pageable on purpose: rect_tiles rebuilds it twice a round (edge, then
    // vertex rectangle) while the first upload may still be queued; a
    // pageable copy is staged at the call, a pinned one would race
    std::vector<uint32_t> tiles_r_host;
    int64_t tiles_r_key = -1;
    // block-sparse mode: -1 auto, 0 off, 1 on (first-vertex edge order), 2 on
    // with component ordering (falls back to 1 when labels do not settle)
    int sparse = -1;
    DevBuf<int32_t> perm, sort_keys, sort_keys_out, sort_vals;
    DevBuf<uint8_t> sort_temp;
    DevBuf<unsigned long long> mask_e, mask_v, kblocks;
    // component ordering: labels, vertex permutation and its per-round compaction
    DevBuf<int32_t> vlabel, elabel, vperm, vpos, vids_p, vnew_p;
    // single-pass compaction: look-back status words (epoch-tagged, never cleared)
    DevBuf<unsigned long long> cp_status;
    int64_t cp_status_cap = 0;
    uint32_t cp_epoch = 0;
    // instance produced by mhsk_generate_random
    DevBuf<int64_t> gen_ptr;
    DevBuf<int32_t> gen_vtx, gen_dem, gen_attempt;
    int32_t gen_n = -1, gen_m = -1;
    int64_t gen_nnz = 0;
    // tile list
    DevBuf<uint32_t> tiles;
    std::vector<uint32_t> tiles_host;
    int32_t tiles_for_M = -1;
    int32_t tiles_for_variant = -1;
    int gram_variant = 2;  // 2: CTA-pair 256x256 tiles (default); 1: single-CTA 128x256 (MHSK_GRAM=1)
    int32_t throttle_chunk_log2 = 4, throttle_slack = 4;  // MHSK_THROTTLE="log2chunk,slack" (slack 0 = off)
    DevBuf<int32_t> progress;
    int32_t raster_gp = 4, raster_gj = 9;  // super-blocks of 4x9 squares (profiles/); MHSK_RASTER="gp,gj" overrides
    // counters: [0] n_alive [1] m_alive [2] deleted [3] spare [4..5] validation flags
    DevBuf<int32_t> counters;
    int32_t* counters_host = nullptr;  // pinned
    int64_t* nnz_host = nullptr;       // pinned: edge_ptr[m] read with validate's flags
    unsigned long long* desc_host = nullptr;   // pinned: fused validation's descent counts
    DevBuf<unsigned long long> vdesc;
    cudaEvent_t val_ev = nullptr;   // the fused validation's flags have landed
    DevBuf<int32_t> seen_all;   // seen_full's verdict
    DevBuf<uint32_t> seen2, vc_bits, vdel_bits;   // original-id maps of the later-round member passes
    DevBuf<int32_t> need_low;                     // need from the non-fmax edges (seen_alive_edges)
    DevBuf<int32_t> need_low_p;                   // the same for the edge pack (pack_rows_csr need_low)
    DevBuf<uint32_t> alive_bits;                  // alive vertices by original id (later-round packs)
    // streamed upload of the member array (mhsk_kernelize, fast path, one
    // rank): chunk b = members [up_K[b], up_K[b+1]) on copy_stream, landed at
    // up_ev[b]; edges [0, up_E[b]) are complete after it
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> up_ev;
    std::vector<int64_t> up_K;
    std::vector<int32_t> up_E;
    bool up_pending = false;
    int32_t stream_chunks = STREAM_DEFAULT_CHUNKS;   // option "stream_chunks" (<= 1: no streaming)
    // multi-GPU host calls (option "shard_upload"): each rank copies 1/world of
    // the member array over its own PCIe link and one all-reduce over the
    // zero-filled rest assembles it on every rank (1: from 2^24 members, 2:
    // always, 0: every rank copies all of it)
    int32_t shard_upload = 1;
    bool stream_sqrt = true;                     // option "stream_sqrt": chunk bounds at sqrt(b / C)
    int32_t rect_rule = 0;                       // option "rect_rule": 0 probe-cost rule, 1 half the items
    std::vector<int32_t> band_t;   // band b of the edge tile list: t in [band_t[b], band_t[b+1])
    // the band list sits in tiles_e / tiles_e_host (uploaded on the copy
    // stream ahead of the chunks) for round 1 of band_M edges, FP4 tiles
    // band_fp4; band_M < 0: none
    int32_t band_M = -1;
    bool band_fp4 = false;
    TileVec band_host;               // the band list (pinned) and the inputs it was built from
    std::vector<int32_t> band_key;
    cudaEvent_t band_ev = nullptr;   // the band list's upload (copy stream)
    // speculative vertex probe (option "spec_vertex"): round 1 of a streamed
    // FP4 call runs the vertex phase's probe pass as soon as the probe-column
    // edges have landed, assuming the edge phase deletes nothing; it is used
    // only if that holds (dims_host[12], read at edge_ev), else discarded.
    // Its probe outputs live in the *_s buffers (swapped in when adopted).
    bool spec_v = true;
    DevBuf<uint32_t> needed_s;
    DevBuf<int4> cand_s;
    DevBuf<int32_t> cand_count_s, lo_s, one_s, spec_dims;
    DevBuf<float2> pv_s, pcm_s;
    cudaEvent_t edge_ev = nullptr;   // round 1's edge phase committed (spec check)
    // recorded after each fast-path round's host read (its D2H copies): when
    // nothing runs on the device after the last one, the call's device time
    // ends there rather than after the host's turnaround (end_call)
    cudaEvent_t ev_round = nullptr;
    bool round_ev_valid = false;
    const int64_t* nnz_src = nullptr;  // the edge_ptr nnz_host was read from (this call)

    // programmatic dependent launch of every library kernel (option "pdl")
    bool pdl = true;
    // host-pointer calls: every round's host read also brings the alive flags
    // into this pinned buffer, so the call's result needs no host round trip
    // after the last round (stage_alive: requested; alive_staged: done)
    uint8_t* alive_host = nullptr;
    int64_t alive_host_cap = 0;
    bool stage_alive = false, alive_staged = false;

    mhsk_stats st{};
};

// Every kernel launch of the library: on the context's stream, with
// programmatic stream serialization (PDL) unless the "pdl" option is off.  The
// kernels open with mhsk::pdl_enter() (epilogue.cuh): wait for the
// predecessor grid, then release their dependents.  A launch then costs its
// own latency behind the previous kernel instead of after it -- the round
// loop is ~50 dependent kernels, most of them a few microseconds long.
template <typename... KArgs, typename... Args>
void launch_pdl(mhsk_ctx* c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.attrs = attr;
    cfg.numAttrs = c->pdl ? 1 : 0;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

namespace {

void ctx_sync(mhsk_ctx* c) { CUDA_TRY(cudaStreamSynchronize(c->stream)); }

// Order-preserving compaction of `alive[0..n)` -> new_id, ids; count ->
// *d_total.  With perm: positions k visit item perm[k] (ids/new_id hold item
// ids).  n_dyn: device-resident count <= n.  One single-pass launch
// (decoupled look-back, k::compact_1pass).
void compact_impl(mhsk_ctx* c, const uint8_t* alive, int32_t n, const int32_t* n_dyn, const int32_t* perm,
                  int32_t* new_id, int32_t* ids, int32_t* d_total) {
    using namespace mhsk::k;
    if (n == 0) {
        CUDA_TRY(cudaMemsetAsync(d_total, 0, sizeof(int32_t), c->stream));
        return;
    }
    const int32_t tiles = (n + CP_ITEMS - 1) / CP_ITEMS;
    if (tiles > c->cp_status_cap || c->cp_epoch + 1 >= (1u << 30)) {
        c->cp_status.reserve(std::max<int64_t>(tiles, c->cp_status_cap));
        c->cp_status_cap = std::max<int64_t>(tiles, c->cp_status_cap);
        CUDA_TRY(cudaMemsetAsync(c->cp_status.ptr, 0, c->cp_status_cap * sizeof(unsigned long long), c->stream));
        c->cp_epoch = 0;
    }
    ++c->cp_epoch;
    launch_pdl(c, compact_1pass, std::min(tiles, c->sms), CP_THREADS, 0, alive, n, n_dyn, perm, new_id, ids,
                                                                      d_total, c->cp_status.ptr, c->cp_epoch);
    LAUNCH_CHECK();
    c->st.kernel_launches += 1;
}

void compact(mhsk_ctx* c, const uint8_t* alive, int32_t n, int32_t* new_id, int32_t* ids, int32_t* d_total) {
    compact_impl(c, alive, n, nullptr, nullptr, new_id, ids, d_total);
}

void build_tiles(mhsk_ctx* c, int32_t M) {
    if (c->tiles_for_M == M && c->tiles_for_variant == c->gram_variant) return;
    const mhsk::TileShape shape = c->gram_variant == 1
        ? mhsk::TileShape{mhsk::tc::BM, mhsk::tc::BN, c->raster_gp, c->raster_gj}
        : mhsk::TileShape{mhsk::tc2::BM, mhsk::tc2::BN, c->raster_gp, c->raster_gj};
    const int32_t MI = (M + shape.bm - 1) / shape.bm, NJ = (M + shape.bn - 1) / shape.bn;
    if (MI > 0xFFFF || NJ > 0xFFFF) {
        set_error("instance too large for the tile list (%d items)", M);
        throw Failure{MHSK_INVALID};
    }
    mhsk::make_tile_list(M, shape, c->tiles_host);
    c->tiles.reserve(c->tiles_host.size());
    CUDA_TRY(cudaMemcpyAsync(c->tiles.ptr, c->tiles_host.data(),
                             c->tiles_host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                             c->stream));
    c->tiles_for_M = M;
    c->tiles_for_variant = c->gram_variant;
}

// This rank's share of a tile list: tiles rank, rank + world, ... (the
// ranks interleave, so every rank keeps an equal share of the tiles that are
// still inside M when later rounds shrink it).
void shard_share(int32_t total, int32_t rank, int32_t world, int32_t& begin, int32_t& count,
                 int32_t& stride) {
    begin = std::min(rank, total);
    stride = world;
    count = total > rank ? (total - rank + world - 1) / world : 0;
}

void shard_slice(const mhsk_ctx* c, int32_t& begin, int32_t& count, int32_t& stride) {
    shard_share((int32_t)c->tiles_host.size(), c->rank, c->world, begin, count, stride);
}

template <int PHASE>
void launch_gram_tc2(mhsk_ctx* c, const int8_t* X, int32_t M, int32_t K, const int32_t* va,
                     const int32_t* vb) {
    using namespace mhsk::tc2;
    const int64_t K_pad = round_up(std::max<int32_t>(K, 1), BK);
    const int64_t rows_pad = round_up(M, ROW_PAD);
    build_tiles(c, M);
    int32_t begin, count, stride;
    shard_slice(c, begin, count, stride);
    c->st.gram_ops += (int64_t)M * (int64_t)(M + 1) * (int64_t)K;
    c->st.executed_ops += (int64_t)count * 2ll * BM * BN * K_pad;
    if (count <= 0) return;
    CUtensorMap ta = make_tmap(X, rows_pad, K_pad, HALF);
    CUtensorMap tb = make_tmap(X, rows_pad, K_pad, HALF);
    GramArgs args{};
    args.M = M;
    args.k_blocks = (int32_t)(K_pad / BK);
    args.va = va;
    args.vb = vb;
    args.hits = c->hits.ptr;
    args.tiles = c->tiles.ptr;
    args.tile_begin = begin;
    args.tile_count = count;
    args.tile_stride = stride;
    args.dev_mk = nullptr;
    args.enable = nullptr;
    args.a_items = nullptr;
    args.a_count = nullptr;
    args.mask = nullptr;
    args.mask_words = 0;
    args.zero_needed = nullptr;
    args.rank = nullptr;
    const int pairs = std::min<int32_t>(c->sms / 2, count);
    args.progress = nullptr;
    args.chunk_log2 = c->throttle_chunk_log2;
    args.slack = c->throttle_slack;
    if (c->throttle_slack > 0 && (args.k_blocks >> c->throttle_chunk_log2) > c->throttle_slack) {
        const int32_t waves = (count + pairs - 1) / pairs;
        c->progress.reserve(waves);
        CUDA_TRY(cudaMemsetAsync(c->progress.ptr, 0, waves * sizeof(int32_t), c->stream));
        args.progress = c->progress.ptr;
    }
    static bool attr_set[3] = {false, false, false};
    if (!attr_set[PHASE]) {
        CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr_set[PHASE] = true;
    }
    launch_pdl(c, gram_tc2_kernel<PHASE>, 2 * pairs, NUM_THREADS, SMEM_BYTES, ta, tb, args);
    LAUNCH_CHECK();
}

template <int PHASE>
void launch_gram_tc(mhsk_ctx* c, const int8_t* X, int32_t M, int32_t K, const int32_t* va,
                    const int32_t* vb) {
    using namespace mhsk::tc;
    const int64_t K_pad = round_up(std::max<int32_t>(K, 1), BK);
    const int64_t rows_pad = round_up(M, ROW_PAD);
    build_tiles(c, M);
    int32_t begin, count, stride;
    shard_slice(c, begin, count, stride);
    c->st.gram_ops += (int64_t)M * (int64_t)(M + 1) * (int64_t)K;
    c->st.executed_ops += (int64_t)count * 2ll * BM * BN * K_pad;
    if (count <= 0) return;
    CUtensorMap ta = make_tmap(X, rows_pad, K_pad, BM);
    CUtensorMap tb = make_tmap(X, rows_pad, K_pad, BN);
    GramArgs args{};
    args.M = M;
    args.k_blocks = (int32_t)(K_pad / BK);
    args.va = va;
    args.vb = vb;
    args.hits = c->hits.ptr;
    args.tiles = c->tiles.ptr;
    args.tile_begin = begin;
    args.tile_count = count;
    args.tile_stride = stride;
    static bool attr_set[3] = {false, false, false};
    if (!attr_set[PHASE]) {
        CUDA_TRY(cudaFuncSetAttribute(gram_tc_kernel<PHASE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr_set[PHASE] = true;
    }
    const int grid = std::min<int32_t>(c->sms, count);
    launch_pdl(c, gram_tc_kernel<PHASE>, grid, NUM_THREADS, SMEM_BYTES, ta, tb, args);
    LAUNCH_CHECK();
}

template <int PHASE>
void launch_gram_simt(mhsk_ctx* c, int32_t M, int64_t words, int64_t ld, const int32_t* va,
                      const int32_t* vb) {
    const int32_t T = 32;
    const dim3 grid((M + T - 1) / T, (M + T - 1) / T);
    launch_pdl(c, mhsk::k::gram_simt<PHASE>, grid, dim3(32, 8), 0, M, (int32_t)words, reinterpret_cast<const uint32_t*>(c->X.ptr), ld, va, vb, c->hits.ptr);
    LAUNCH_CHECK();
    c->st.gram_ops += (int64_t)M * (int64_t)(M + 1) * words * 32;
}

struct DevInstance {
    int32_t n, m;
    const int64_t* ptr;
    const int32_t* vtx;
    const int32_t* dem;
};

// Operand geometry of a phase.
struct Geometry {
    int64_t ld;       // int8: bytes per row (K_pad); bits: 32-bit words per row
    int64_t rows;     // padded rows
    int64_t bytes;
    int64_t words;    // bits backend: valid words per row
};

Geometry geometry(const mhsk_ctx* c, int32_t M, int32_t K) {
    Geometry g{};
    if (c->backend == MHSK_BACKEND_TC) {
        g.ld = round_up(std::max<int32_t>(K, 1), mhsk::tc::BK);
        g.rows = round_up(std::max<int32_t>(M, 1), mhsk::tc::ROW_PAD);
        g.bytes = g.ld * g.rows;
    } else {
        g.words = (std::max<int32_t>(K, 1) + 31) / 32;
        g.ld = g.words;
        g.rows = round_up(std::max<int32_t>(M, 1), 32);
        g.bytes = g.ld * g.rows * 4;
    }
    return g;
}

void allreduce_hits(mhsk_ctx* c, int32_t M) {
    if (c->world <= 1 || M == 0) return;
    if (!c->allreduce) {
        set_error("world > 1 but no allreduce callback");
        throw Failure{MHSK_INVALID};
    }
    if (c->allreduce(c->hits.ptr, M, (void*)c->stream, c->allreduce_user) != 0) {
        set_error("allreduce callback failed");
        throw Failure{MHSK_CUDA_ERROR};
    }
}

void time_gram_begin(mhsk_ctx* c) { CUDA_TRY(cudaEventRecord(c->evg0, c->stream)); }
void time_gram_end(mhsk_ctx* c) {
    CUDA_TRY(cudaEventRecord(c->evg1, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->evg1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->evg0, c->evg1));
    c->st.ms_gram += ms;
    c->st.gram_launches += 1;
    c->st.kernel_launches += 1;
}

template <int PHASE>
void launch_gram(mhsk_ctx* c, const int8_t* X, int32_t M, int32_t K, const int32_t* va,
                 const int32_t* vb) {
    if (c->gram_variant == 1) launch_gram_tc<PHASE>(c, X, M, K, va, vb);
    else launch_gram_tc2<PHASE>(c, X, M, K, va, vb);
}

// dynamic shared memory cap of pack_rows_csr's shared alive / seen maps
// (2 x n/32 words: n <= 393,216 vertices)
constexpr size_t PACK_SMAP_MAX = 96u << 10;
void set_pack_smem_limit(int device) {
    static std::atomic<uint64_t> done{0};   // per device of this process
    const uint64_t bit = 1ull << (device & 63);
    if (done.load() & bit) return;
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::pack_rows_csr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PACK_SMAP_MAX));
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::pack_rows_csr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PACK_SMAP_MAX));
    done.fetch_or(bit);
}

int pack_blocks(const mhsk_ctx* c, int64_t rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((rows + mhsk::k::PACK_WARPS - 1) / mhsk::k::PACK_WARPS,
                                                       (int64_t)c->sms * 5));   // resident CTAs at 48 registers
}

// X_E (M edge rows x K vertex columns) from CSR with coalesced row stores.
void pack_xe(mhsk_ctx* c, const DevInstance& in, int32_t M, int32_t K) {
    const int64_t ld = round_up(std::max<int32_t>(K, 1), mhsk::tc::BK);
    const int64_t rows_pad = round_up(std::max<int32_t>(M, 1), mhsk::tc::ROW_PAD);
    c->XE.reserve(ld * rows_pad);
    mhsk::k::pack_rows_csr<false><<<pack_blocks(c, rows_pad), mhsk::k::PACK_WARPS * 32, 0, c->stream>>>(M, (int32_t)rows_pad, c->eids.ptr, in.ptr, in.vtx, in.dem, c->vnew.ptr, c->XE.ptr, ld,
        c->item_a.ptr, c->item_b.ptr);
    LAUNCH_CHECK();
    c->st.kernel_launches += 1;
    c->xe_valid = true;
    c->xe_rows = M;
    c->xe_cols = K;
    c->xe_ld = ld;
}

__global__ void iota_kernel(int32_t n, int32_t* out) {
    mhsk::pdl_enter();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// One edge phase over the compacted instance (M = m', K = n').
// ealive != null: commit deletions into ealive; keep_out != null: keep vector.
void edge_phase(mhsk_ctx* c, const DevInstance& in, int32_t rule, int32_t M, int32_t K,
                uint8_t* ealive, uint8_t* keep_out) {
    if (M == 0) {
        c->xe_valid = false;
        return;
    }
    c->item_a.reserve(M);
    c->item_b.reserve(M);
    c->hits.reserve(M);
    c->keep_e.reserve(M);
    CUDA_TRY(cudaMemsetAsync(c->hits.ptr, 0, M * sizeof(int32_t), c->stream));
    if (c->backend == MHSK_BACKEND_TC) {
        pack_xe(c, in, M, K);
        time_gram_begin(c);
        if (rule == MHSK_RULE_DP) launch_gram<mhsk::PHASE_DP>(c, c->XE.ptr, M, K, c->item_a.ptr, c->item_b.ptr);
        else launch_gram<mhsk::PHASE_SE>(c, c->XE.ptr, M, K, c->item_a.ptr, c->item_b.ptr);
        time_gram_end(c);
    } else {
        const Geometry g = geometry(c, M, K);
        c->X.reserve(g.bytes);
        CUDA_TRY(cudaMemsetAsync(c->X.ptr, 0, g.bytes, c->stream));
        const int blocks = std::max(1, std::min<int32_t>((in.m + 7) / 8, c->sms * 16));
        launch_pdl(c, mhsk::k::pack_edge_rows<true>, blocks, 256, 0, in.m, in.ptr, in.vtx, in.dem, c->enew.ptr, c->vnew.ptr, c->X.ptr, g.ld, c->item_a.ptr,
            c->item_b.ptr);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
        time_gram_begin(c);
        if (rule == MHSK_RULE_DP)
            launch_gram_simt<mhsk::PHASE_DP>(c, M, g.words, g.ld, c->item_a.ptr, c->item_b.ptr);
        else
            launch_gram_simt<mhsk::PHASE_SE>(c, M, g.words, g.ld, c->item_a.ptr, c->item_b.ptr);
        time_gram_end(c);
    }
    allreduce_hits(c, M);
    mhsk::k::commit_phase<false><<<(M + 255) / 256, 256, 0, c->stream>>>(M, c->hits.ptr, nullptr, c->eids.ptr, ealive, keep_out ? keep_out : c->keep_e.ptr,
        c->counters.ptr + 2);
    LAUNCH_CHECK();
    c->st.kernel_launches += 1;
}

// One vertex phase (M = n' vertices, K = m' alive edges, compaction current).
// ealive_now: the alive edges (for need).  The tensor-core operand X_V is the
// transpose of the last X_E restricted to the edges that survived it, or --
// when X_E is stale (vertices changed since) -- of a fresh X_E.
void vertex_phase(mhsk_ctx* c, const DevInstance& in, int32_t M, int32_t K,
                  const uint8_t* ealive_now, uint8_t* valive, uint8_t* keep_out) {
    if (M == 0) return;
    c->item_a.reserve(M);
    c->item_b.reserve(M);
    c->hits.reserve(M);
    CUDA_TRY(cudaMemsetAsync(c->hits.ptr, 0, M * sizeof(int32_t), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->item_b.ptr, 0, M * sizeof(int32_t), c->stream));
    if (c->backend == MHSK_BACKEND_TC) {
        c->src.reserve(std::max<int32_t>(K, 1));
        if (c->xe_valid && c->xe_cols == M) {
            // survivors of the last edge phase, in order: X_V column j <- X_E row src[j]
            c->scratch.reserve(std::max<int32_t>(c->xe_rows, 1));
            compact(c, c->keep_e.ptr, c->xe_rows, c->scratch.ptr, c->src.ptr, c->counters.ptr + 7);
        } else {
            c->item_a.reserve(std::max<int32_t>(M, K));
            c->item_b.reserve(std::max<int32_t>(M, K));
            pack_xe(c, in, K, M);   // rows = alive edges, columns = alive vertices
            CUDA_TRY(cudaMemsetAsync(c->item_b.ptr, 0, M * sizeof(int32_t), c->stream));
            if (K) {
                launch_pdl(c, iota_kernel, (K + 255) / 256, 256, 0, K, c->src.ptr);
                LAUNCH_CHECK();
                c->st.kernel_launches += 1;
            }
        }
        const int64_t ld_v = round_up(std::max<int32_t>(K, 1), mhsk::tc::BK);
        const int64_t rows_pad_v = round_up(M, mhsk::tc::ROW_PAD);
        c->XV.reserve(ld_v * rows_pad_v);
        mhsk::k::transpose_pack<false><<<(int)(rows_pad_v / 128), mhsk::k::TP_WARPS * 32, 0, c->stream>>>(c->XE.ptr, c->xe_ld, c->src.ptr, K, M, c->XV.ptr, ld_v, c->item_a.ptr);
        LAUNCH_CHECK();
        const int blocks = std::max(1, std::min<int32_t>((in.m + 7) / 8, c->sms * 16));
        mhsk::k::need_from_csr<<<blocks, 256, 0, c->stream>>>(in.m, in.ptr, in.vtx, in.dem, ealive_now,
                                                             c->vnew.ptr, c->item_b.ptr);
        LAUNCH_CHECK();
        c->st.kernel_launches += 2;
        time_gram_begin(c);
        launch_gram<mhsk::PHASE_MD>(c, c->XV.ptr, M, K, c->item_a.ptr, nullptr);
        time_gram_end(c);
    } else {
        const Geometry g = geometry(c, M, K);
        c->X.reserve(g.bytes);
        CUDA_TRY(cudaMemsetAsync(c->X.ptr, 0, g.bytes, c->stream));
        CUDA_TRY(cudaMemsetAsync(c->item_a.ptr, 0, M * sizeof(int32_t), c->stream));
        const int blocks = std::max(1, std::min<int32_t>((in.m + 7) / 8, c->sms * 16));
        launch_pdl(c, mhsk::k::pack_vertex_rows<true>, blocks, 256, 0, in.m, in.ptr, in.vtx, in.dem, c->enew.ptr, c->vnew.ptr, c->X.ptr, g.ld, c->item_a.ptr,
            c->item_b.ptr);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
        time_gram_begin(c);
        launch_gram_simt<mhsk::PHASE_MD>(c, M, g.words, g.ld, c->item_a.ptr, nullptr);
        time_gram_end(c);
    }
    allreduce_hits(c, M);
    mhsk::k::commit_phase<true><<<(M + 255) / 256, 256, 0, c->stream>>>(M, c->hits.ptr, c->item_b.ptr, c->vids.ptr, valive, keep_out, c->counters.ptr + 2);
    LAUNCH_CHECK();
    c->st.kernel_launches += 1;
    c->xe_valid = false;   // vertex deletions change X_E's column space
}

void reserve_instance_state(mhsk_ctx* c, int32_t n, int32_t m) {
    c->vnew.reserve(n + 1);
    c->vids.reserve(n + 1);
    c->enew.reserve(m + 1);
    c->eids.reserve(m + 1);
    c->counters.reserve(8);
}

// The flags of validate_csr / scan_members + pack_rows_csr, read into
// counters_host[4..5]: [4] malformed, [5] first infeasible edge (1-based) or
// INT_MAX.
// counters[5] starts at this (a byte-pattern memset: no host copy, which a
// streamed upload would hold up) and keeps the first infeasible edge
constexpr int32_t NO_INFEASIBLE_EDGE = 0x7F7F7F7F;

int validation_result(mhsk_ctx* c) {
    if (c->counters_host[4]) {
        set_error("malformed CSR instance (vertex ids must be in range and strictly increasing "
                  "per edge, demands >= 1)");
        return MHSK_INVALID;
    }
    if (c->counters_host[5] != NO_INFEASIBLE_EDGE) {
        set_error("instance is infeasible: edge %d demands more hits than it has vertices",
                  c->counters_host[5]);
        return MHSK_INFEASIBLE;
    }
    return MHSK_OK;
}

// Order the compute stream after every pending upload chunk.
void wait_upload(mhsk_ctx* c) {
    if (!c->up_pending) return;
    for (cudaEvent_t ev : c->up_ev) CUDA_TRY(cudaStreamWaitEvent(c->stream, ev, 0));
    c->up_pending = false;
}

// Validate the device-resident CSR; returns MHSK_OK / MHSK_INVALID / MHSK_INFEASIBLE.
int validate(mhsk_ctx* c, const DevInstance& in) {
    wait_upload(c);
    CUDA_TRY(cudaMemsetAsync(c->counters.ptr + 4, 0, sizeof(int32_t), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->counters.ptr + 5, 0x7F, sizeof(int32_t), c->stream));
    if (in.m > 0) {
        const int blocks = std::max(1, std::min<int32_t>((in.m + 7) / 8, c->sms * 16));
        launch_pdl(c, validate_csr, blocks, 256, 0, in.n, in.m, in.ptr, in.vtx, in.dem,
                                                    c->counters.ptr + 4);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
    }
    CUDA_TRY(cudaMemcpyAsync(c->counters_host + 4, c->counters.ptr + 4, 2 * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, c->stream));
    if (in.m > 0) {   // nnz rides on this sync (kernelize_fast needs it on the host)
        CUDA_TRY(cudaMemcpyAsync(c->nnz_host, in.ptr + in.m, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 c->stream));
        c->nnz_src = in.ptr;
    }
    ctx_sync(c);
    return validation_result(c);
}

void validate_or_throw(mhsk_ctx* c, const DevInstance& in) {
    const int rc = validate(c, in);
    if (rc != MHSK_OK) throw Failure{rc};
}

void throw_if_invalid(mhsk_ctx* c) {
    const int rc = validation_result(c);
    if (rc != MHSK_OK) throw Failure{rc};
}

void read_counters(mhsk_ctx* c) {
    CUDA_TRY(cudaMemcpyAsync(c->counters_host, c->counters.ptr, 4 * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
}


// ---------------------------------------------------------------------------
// Device-resident round loop (tensor-core pair backend).  Operand strides and
// tile lists are fixed from the initial sizes; the current alive counts live
// in c->dims and every kernel of a round reads them there, so a round needs
// no host decision and exactly one host read (the deletion counts).
void compact_dyn(mhsk_ctx* c, const uint8_t* alive, int32_t n, const int32_t* n_dyn, int32_t* new_id,
                 int32_t* ids, int32_t* d_total) {
    compact_impl(c, alive, n, n_dyn, nullptr, new_id, ids, d_total);
}

// tile columns of the pair kernel: 240 on FP4 operands (two accumulators +
// scale factors in TMEM), 256 on int8
inline int32_t pair_bn(bool fp4) { return fp4 ? mhsk::tc2::BN_FP4 : mhsk::tc2::BN; }

void device_tiles(mhsk_ctx* c, int32_t M, DevBuf<uint32_t>& dev, TileVec& host,
                  int32_t& built_for, bool fp4) {
    const int32_t key = 2 * M + (fp4 ? 1 : 0);
    if (built_for == key) return;
    mhsk::make_tile_list(M, mhsk::TileShape{mhsk::tc2::BM, pair_bn(fp4), c->raster_gp, c->raster_gj}, host);
    dev.reserve(std::max<size_t>(host.size(), 1));
    if (!host.empty())
        CUDA_TRY(cudaMemcpyAsync(dev.ptr, host.data(), host.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, c->stream));
    built_for = key;
}

// Exact decision of the candidate pairs the last Gram launch listed
// (verify.cuh); X = that launch's (triangle) operand.
template <int PHASE>
void launch_verify(mhsk_ctx* c, const int8_t* X, int64_t ld, const int32_t* dev_mk, bool fp4, const int32_t* va,
                   const int32_t* vb, const int32_t* skip = nullptr) {
    if (!c->lg_cand || c->lg_count <= 0) return;
    launch_pdl(c, mhsk::k::verify_candidates<PHASE>, c->sms * 8, mhsk::k::VERIFY_THREADS, 0, c->cand.ptr, c->cand_count.ptr, c->cand_cap, c->needed.ptr, X, ld, dev_mk, fp4 ? 256 : 128, va,
        vb, c->hits.ptr, c->pruned.cap >= 3 ? c->pruned.ptr + 2 : nullptr, skip);
    LAUNCH_CHECK();
    c->st.kernel_launches += 1;
}

// Gram launch over a static tile list; sizes from dev_mk.  Triangle: A = B =
// X.  Rectangle (RECT): A = the affected rows XA (a_items / a_count), B = X.
// enable (optional): device gate, the kernel exits unless *enable.
template <int PHASE, bool RECT = false>
void launch_gram_fast(mhsk_ctx* c, const int8_t* XA, int64_t rows_a_pad, const int8_t* XB,
                      int64_t rows_b_pad, int64_t ld0, int32_t M0, const uint32_t* tiles,
                      int32_t total, const int32_t* dev_mk, const int32_t* va, const int32_t* vb,
                      const int32_t* a_items = nullptr, const int32_t* a_count = nullptr,
                      const int32_t* enable = nullptr, const unsigned long long* mask = nullptr,
                      int32_t mask_words = 0, const int32_t* zero_needed = nullptr,
                      const int32_t* rank = nullptr, bool fp4 = false, const int32_t* lo = nullptr,
                      unsigned long long* pruned = nullptr, int32_t probe_kb = 0, int32_t passes = 0,
                      bool defer_verify = false, int32_t t_lo = 0, int32_t t_hi = INT32_MAX,
                      bool first_band = true, int32_t item_lo = 0, int32_t item_hi = INT32_MAX) {
    using namespace mhsk::tc2;
    int32_t begin, count, stride;
    shard_share(total, c->rank, c->world, begin, count, stride);
    c->lg_count = 0;
    if (count <= 0) return;
    CUtensorMap ta = make_tmap(XA, rows_a_pad, ld0, HALF);
    CUtensorMap tb = make_tmap(XB, rows_b_pad, ld0, (!mask && fp4) ? BN_FP4 / 2 : HALF);
    GramArgs args{};
    args.M = M0;
    args.k_blocks = (int32_t)(ld0 / BK);
    args.va = va;
    args.vb = vb;
    args.hits = c->hits.ptr;
    args.tiles = tiles;
    args.tile_begin = begin;
    args.tile_count = count;
    args.tile_stride = stride;
    args.dev_mk = dev_mk;
    args.enable = enable;
    args.a_items = a_items;
    args.a_count = a_count;
    args.mask = mask;
    args.mask_words = mask_words;
    args.zero_needed = zero_needed;
    args.rank = rank;
    args.kblocks_done = mask ? c->kblocks.ptr : nullptr;
    args.lo = (RECT || mask) ? nullptr : lo;
    args.probe_kb = probe_kb;
    args.needed = nullptr;
    args.needed_words = 0;
    args.timing = nullptr;
    args.tune = c->gram_tune;
    if (c->gram_timing) {   // MHSK_GRAM_TIMING=1: per-role cycle counters, printed after the launch
        c->timing.reserve(mhsk::tc2::GRAM_TIMING_SLOTS);
        CUDA_TRY(cudaMemsetAsync(c->timing.ptr, 0, mhsk::tc2::GRAM_TIMING_SLOTS * 8, c->stream));
        args.timing = c->timing.ptr;
    }
    args.pruned_tiles = pruned;
    const int pairs = std::min<int32_t>(c->sms / 2, count);
    args.progress = nullptr;
    args.chunk_log2 = c->throttle_chunk_log2;
    args.slack = c->throttle_slack;
    if (!RECT && !mask && c->throttle_slack > 0 && (args.k_blocks >> c->throttle_chunk_log2) > c->throttle_slack) {
        const int32_t waves = (count + pairs - 1) / pairs;
        c->progress.reserve(waves);
        CUDA_TRY(cudaMemsetAsync(c->progress.ptr, 0, waves * sizeof(int32_t), c->stream));
        args.progress = c->progress.ptr;
    }
    args.passes = passes;
    args.t_lo = t_lo;   // a band of the list (overlapped upload); later bands keep the marks
    args.t_hi = t_hi;
    args.force_probe = passes != 0;   // split launches: the operand may hold only the probe columns
    if (args.lo && probe_kb > 0) {   // two-pass probe schedule: zeroed per-pair bitmaps
        const int32_t per_pair = (count + pairs - 1) / pairs;
        args.needed_words = (per_pair + 31) / 32;
        const size_t words = (size_t)pairs * args.needed_words;
        c->needed.reserve(words + 1);   // + the "any tile marked" word
        if (passes != 2 && first_band)   // a full-pass-only launch reads the marks of its probe launch(es)
            CUDA_TRY(cudaMemsetAsync(c->needed.ptr, 0, (words + 1) * sizeof(uint32_t), c->stream));
        args.needed = c->needed.ptr;
        args.marked = reinterpret_cast<int32_t*>(c->needed.ptr + words);
        if (passes == 2 && !enable) args.enable = args.marked;   // nothing marked: exit at once
    }
    if (!RECT && !mask && args.needed && passes != 2) {
        // per-item / per-panel probe terms (FP4 and int8 alike); a band launch
        // refreshes only the items [item_lo, item_hi) its chunk completed and
        // their column panels
        const int32_t bn = pair_bn(fp4);
        const int32_t i_lo = std::max(item_lo, 0), i_hi = std::min(item_hi, M0);
        const int32_t P_lo = i_lo / bn, P_hi = (std::max(i_hi, 1) + bn - 1) / bn;
        c->pv.reserve(std::max<int32_t>(M0, 1));
        const int32_t npanels = (M0 + bn - 1) / bn;
        c->pcm.reserve(std::max(npanels * 8, 1));
        const bool uni_b = PHASE == mhsk::PHASE_DP && vb;
        if (uni_b) c->pb.reserve(std::max(npanels, 1));
        launch_pdl(c, probe_terms<PHASE>, std::max(1, std::min(npanels, P_hi) - P_lo), 256, 0, dev_mk, M0, va, vb,
                   (const int32_t*)args.lo, c->pv.ptr, c->pcm.ptr, uni_b ? c->pb.ptr : nullptr, i_lo, i_hi, P_lo, bn);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
        args.pv = c->pv.ptr;
        args.pcm = c->pcm.ptr;
        if (uni_b) args.pb = c->pb.ptr;
    }
    const bool verify = !RECT && !mask && args.needed && c->verify && passes != 2;
    if (verify) {   // candidate pairs of sparsely-firing tiles, decided by verify_candidates
        c->cand.reserve(CAND_CAP);
        c->cand_count.reserve(1);
        if (first_band) CUDA_TRY(cudaMemsetAsync(c->cand_count.ptr, 0, sizeof(int32_t), c->stream));
        args.cand = c->cand.ptr;
        args.cand_count = c->cand_count.ptr;
        args.cand_cap = c->cand_cap;
    }
    // geometry of this launch, for needed_panels / a deferred verification
    c->lg_pairs = pairs;
    c->lg_words = args.needed_words;
    c->lg_begin = begin;
    c->lg_count = count;
    c->lg_stride = stride;
    c->lg_cand = verify;
    if (mask && !RECT)
        launch_pdl(c, gram_tc2_kernel<PHASE, RECT, !RECT>, 2 * pairs, NUM_THREADS, SMEM_BYTES, ta, tb, args);
    else if (fp4)
        launch_pdl(c, gram_tc2_kernel<PHASE, RECT, false, true>, 2 * pairs, NUM_THREADS, SMEM_BYTES, ta, tb, args);
    else
        launch_pdl(c, gram_tc2_kernel<PHASE, RECT, false>, 2 * pairs, NUM_THREADS, SMEM_BYTES, ta, tb, args);
    LAUNCH_CHECK();
    if (verify && !defer_verify) launch_verify<PHASE>(c, XA, ld0, dev_mk, fp4, va, vb);
    if (c->gram_timing) {
        unsigned long long tmh[mhsk::tc2::GRAM_TIMING_SLOTS];
        CUDA_TRY(cudaMemcpyAsync(tmh, c->timing.ptr, sizeof(tmh), cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        const double ctas = 2.0 * pairs, pr = pairs, epi = ctas * EPI_WARPS;
        fprintf(stderr,
                "[gram timing] phase %d rect %d fp4 %d probe %d tiles %d: kernel %.0f cyc/CTA | producer empty-wait %.0f"
                " | mma tempty-wait %.0f full-wait %.0f | epi stage %.0f probe tfull-wait %.0f probe-eval %.0f"
                " full tfull-wait %.0f full-epi %.0f (cycles per role instance)\n",
                PHASE, (int)RECT, (int)fp4, probe_kb, count, tmh[8] / ctas, tmh[0] / ctas, tmh[1] / pr,
                tmh[2] / pr, tmh[5] / epi, tmh[3] / epi, tmh[4] / epi, tmh[6] / epi, tmh[7] / epi);
    }
}

// Rectangle tile list: A panels P < ceil(Amax/256) (outer) x column panels
// J < ceil(M/bn); P-major so the tiles inside a smaller A form a prefix.
void rect_tiles(mhsk_ctx* c, int32_t Amax, int32_t M, bool fp4) {
    const int64_t key = (((int64_t)Amax << 32) | (uint32_t)M) * 2 + (fp4 ? 1 : 0);
    if (c->tiles_r_key == key) return;
    const int32_t NP = (Amax + 255) / 256, NJ = (M + pair_bn(fp4) - 1) / pair_bn(fp4);
    c->tiles_r_host.clear();
    for (int32_t P = 0; P < NP; ++P)
        for (int32_t J = 0; J < NJ; ++J) c->tiles_r_host.push_back((uint32_t)P | ((uint32_t)J << 16));
    c->tiles_r.reserve(std::max<size_t>(c->tiles_r_host.size(), 1));
    if (!c->tiles_r_host.empty())
        CUDA_TRY(cudaMemcpyAsync(c->tiles_r.ptr, c->tiles_r_host.data(),
                                 c->tiles_r_host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                 c->stream));
    c->tiles_r_key = key;
}

// Tensor-core ops this rank executes for a phase of M items, width K.
int64_t executed_ops_fast(const mhsk_ctx* c, const TileVec& tiles, int32_t M, int32_t K,
                          bool fp4 = false) {
    int32_t begin, count, stride;
    shard_share((int32_t)tiles.size(), c->rank, c->world, begin, count, stride);
    const int32_t bn = pair_bn(fp4), NJ = (M + bn - 1) / bn;
    int64_t valid = 0;
    for (int32_t i = 0; i < count; ++i) valid += (int32_t)(tiles[begin + i * stride] >> 16) < NJ;
    return valid * 2ll * 256 * bn * round_up(std::max<int32_t>(K, 1), fp4 ? 256 : 128);
}

template <int PHASE>
void launch_edge_gram(mhsk_ctx* c, bool rect, const int8_t* XA, int64_t rows_a, int64_t rows_e,
                      int64_t ld_e, int32_t m_cur, const int32_t* dims, const int32_t* a_items, bool fp4,
                      const int32_t* lo, int32_t probe_kb) {
    if (rect)
        launch_gram_fast<PHASE, true>(c, XA, rows_a, c->XE.ptr, rows_e, ld_e, m_cur, c->tiles_r.ptr,
                                      (int32_t)c->tiles_r_host.size(), dims + 0, c->item_a.ptr,
                                      c->item_b.ptr, a_items, dims + 5, nullptr, nullptr, 0, nullptr, nullptr,
                                      fp4);
    else
        launch_gram_fast<PHASE>(c, c->XE.ptr, rows_e, c->XE.ptr, rows_e, ld_e, m_cur, c->tiles_e.ptr,
                                (int32_t)c->tiles_e_host.size(), dims + 0, c->item_a.ptr, c->item_b.ptr,
                                nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, fp4, lo,
                                c->pruned.ptr, probe_kb);
}

template <int PHASE>
void set_pair_attrs() {
    using namespace mhsk::tc2;
    CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE, false, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE, false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE, true, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE, false, false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    CUDA_TRY(cudaFuncSetAttribute(gram_tc2_kernel<PHASE, true, false, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
}

// Kernel attributes are set once per device context up front (not lazily),
// so no launch path -- in particular a CUDA-graph capture -- configures them.
void ensure_gram_attrs() {
    set_pair_attrs<mhsk::PHASE_DP>();
    set_pair_attrs<mhsk::PHASE_SE>();
    set_pair_attrs<mhsk::PHASE_MD>();
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::scan_members<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(mhsk::k::SCAN_SMEM_BITS / 8)));
    const int map_bytes = (int)(mhsk::k::MAP_SMEM_BITS / 8);
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::seen_alive_edges, cudaFuncAttributeMaxDynamicSharedMemorySize, map_bytes));
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::mark_affected_edges_map, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  map_bytes));
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::vcand_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, map_bytes));
    CUDA_TRY(cudaFuncSetAttribute(mhsk::k::vcand_count_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize, map_bytes));
}

// Component ordering for block-sparse mode (sparse option 2 / auto probe):
// label propagation to the minimum vertex id of each connected component,
// then vertices sorted by (component, id) -> vperm / vpos and edges by
// (component, first vertex position) -> perm.  Returns false (and leaves the
// orders unset) when the labels do not settle within LP_MAX_STEPS steps,
// e.g. long interval chains, which the first-vertex order already bands.
bool order_components(mhsk_ctx* c, const DevInstance& in) {
    constexpr int LP_MAX_STEPS = 8;
    const int32_t n0 = in.n, m0 = in.m, mx = std::max(n0, m0);
    c->vlabel.reserve(n0);
    c->elabel.reserve(m0);
    c->vperm.reserve(n0);
    c->vpos.reserve(n0);
    c->perm.reserve(m0);
    c->sort_keys.reserve(mx);
    c->sort_keys_out.reserve(mx);
    c->sort_vals.reserve(mx);
    c->dims.reserve(16);
    int32_t* flag = c->dims.ptr + 14;
    const int csr_blocks = std::max(1, std::min<int32_t>((m0 + 7) / 8, c->sms * 16));
    launch_pdl(c, mhsk::k::lp_init, (n0 + 255) / 256, 256, 0, n0, c->vlabel.ptr);
    LAUNCH_CHECK();
    bool settled = false;
    for (int step = 0; step < LP_MAX_STEPS && !settled; ++step) {
        CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int32_t), c->stream));
        launch_pdl(c, mhsk::k::lp_step, csr_blocks, 256, 0, m0, in.ptr, in.vtx, c->vlabel.ptr, c->elabel.ptr, flag);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
        if (step == 0) continue;   // one step never settles a component with an edge
        CUDA_TRY(cudaMemcpyAsync(c->dims_host + 14, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
        settled = c->dims_host[14] == 0;
    }
    if (!settled) return false;
    // Both sorts are stable: vertices by label keep id order inside a
    // component, so the members of an edge (ascending ids, one component)
    // stay ascending in the new order -- the sparse pack relies on it.
    int bits = 1;
    while (((int64_t)1 << bits) <= (int64_t)n0) ++bits;   // keys are <= n0
    size_t t1 = 0, t2 = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t1, c->sort_keys.ptr, c->sort_keys_out.ptr, c->sort_vals.ptr,
                                             c->vperm.ptr, n0, 0, bits, c->stream));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t2, c->sort_keys.ptr, c->sort_keys_out.ptr, c->sort_vals.ptr,
                                             c->perm.ptr, m0, 0, bits, c->stream));
    size_t temp = std::max<size_t>(std::max(t1, t2), 1);
    c->sort_temp.reserve(temp);
    launch_pdl(c, mhsk::k::vertex_keys, (n0 + 255) / 256, 256, 0, n0, c->vlabel.ptr, c->sort_keys.ptr,
                                                                  c->sort_vals.ptr);
    LAUNCH_CHECK();
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->sort_temp.ptr, temp, c->sort_keys.ptr, c->sort_keys_out.ptr,
                                             c->sort_vals.ptr, c->vperm.ptr, n0, 0, bits, c->stream));
    launch_pdl(c, mhsk::k::invert_perm, (n0 + 255) / 256, 256, 0, n0, c->vperm.ptr, c->vpos.ptr);
    LAUNCH_CHECK();
    launch_pdl(c, mhsk::k::edge_keys, csr_blocks, 256, 0, m0, n0, in.ptr, in.vtx, c->vpos.ptr, c->sort_keys.ptr,
                                                          c->sort_vals.ptr);
    LAUNCH_CHECK();
    temp = std::max<size_t>(std::max(t1, t2), 1);
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->sort_temp.ptr, temp, c->sort_keys.ptr, c->sort_keys_out.ptr,
                                             c->sort_vals.ptr, c->perm.ptr, m0, 0, bits, c->stream));
    c->st.kernel_launches += 6;
    return true;
}

// Fraction of (256-row panel, 128-column k-block) cells of X_E that hold an
// incidence, all items alive, in the order perm / vpos.
double sparse_occupancy(mhsk_ctx* c, const DevInstance& in, int64_t ld_e0, int32_t words_e0) {
    const int32_t m0 = in.m;
    const int64_t panels = round_up(m0, 256) / 256, words = panels * words_e0;
    c->mask_e.reserve(words);
    c->kblocks.reserve(1);
    c->dims_host[15] = m0;
    CUDA_TRY(cudaMemcpyAsync(c->dims.ptr + 15, c->dims_host + 15, sizeof(int32_t), cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemsetAsync(c->mask_e.ptr, 0, words * sizeof(unsigned long long), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->kblocks.ptr, 0, sizeof(unsigned long long), c->stream));
    const int csr_blocks = std::max(1, std::min<int32_t>((m0 + 7) / 8, c->sms * 16));
    launch_pdl(c, mhsk::k::mask_rows_csr, csr_blocks, 256, 0, m0, c->perm.ptr, in.ptr, in.vtx, c->vpos.ptr,
                                                             c->mask_e.ptr, words_e0, c->dims.ptr + 15);
    LAUNCH_CHECK();
    launch_pdl(c, mhsk::k::popcount_u64, std::max<int64_t>(1, std::min<int64_t>((words + 255) / 256, c->sms * 4)), 256, 0, c->mask_e.ptr, words, c->kblocks.ptr);
    LAUNCH_CHECK();
    c->st.kernel_launches += 2;
    unsigned long long bits = 0;
    CUDA_TRY(cudaMemcpyAsync(&bits, c->kblocks.ptr, sizeof(bits), cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    return (double)bits / ((double)panels * (double)(ld_e0 / 128));
}

// Probe length in k-blocks for a phase of width K whose items hold `mean`
// entries on average: enough columns for ~PROBE_ENTRIES of them; 0 (off) when
// that exceeds 1/PROBE_MIN_RATIO of the k-blocks.
// Vertex-probe length in entries of a mean vertex: the "probe_entries" option,
// or (0, the default) 15 up to 150,000 vertices, else 16 -- and 16 for round
// 1 of a streamed host call, whose vertex probe runs speculatively during the
// upload: there the extra candidates' count over the whole CSR lands after
// the copy (config 4 end to end: 7.78 ms at 16 entries, 7.93 at 15).  One entry less
// drops the probe by a k-block at configs 4/5 (1,536 instead of 1,792 probe
// columns); the candidate pairs it leaves grow with the vertex pairs -- at
// config 4 69 instead of 31 (c4 4.36 -> 4.23 ms, c4-planted 21.0 -> 20.2),
// at config 5 2,294 instead of 137, over the vertex-candidate gate's pair
// work, so its panels are transposed (c5 16.15 -> 16.29 ms, c5-planted
// 81 -> 157 ms).  profiles/NOTES.md 63.
int32_t vertex_probe_entries(const mhsk_ctx* c, int64_t vertices, bool streamed_round1) {
    if (c->probe_entries > 0) return c->probe_entries;
    return vertices <= 150000 && !streamed_round1 ? mhsk::PROBE_ENTRIES - 1 : mhsk::PROBE_ENTRIES;
}

// Edge-probe length: "probe_entries_e", or 0: the vertex probe's
int32_t edge_probe_entries(const mhsk_ctx* c, int64_t vertices, bool streamed_round1) {
    return c->probe_entries_e > 0 ? c->probe_entries_e : vertex_probe_entries(c, vertices, streamed_round1);
}

int32_t probe_size(bool on, int32_t K, double mean, int32_t bki, int32_t entries) {
    if (!on || K <= 0 || mean <= 0) return 0;
    const int32_t kb = (K + bki - 1) / bki;
    const double cols = entries * (double)K / mean;
    const int32_t pk = std::max<int32_t>(1, (int32_t)std::ceil(cols / bki));
    return mhsk::PROBE_MIN_RATIO * pk <= kb ? pk : 0;
}

// Will round 1 of kernelize_fast on this instance take the streamed path
// (dense mode, lazy edge operand, one rank)?  Mirrors kernelize_fast's mode
// and probe decisions from the host-side sizes, so that mhsk_kernelize can
// put the edge phase's band tile list on the copy stream ahead of the member
// chunks; kernelize_fast re-checks (c->band_M / band_fp4) and falls back.
// spec_rows: the edges that make up the speculative vertex probe's columns
// (0: it will not run), so that a first chunk can bring just them.
bool plan_streamed_round1(const mhsk_ctx* c, int32_t n, int32_t m, int64_t nnz, bool& fp4, int64_t& spec_rows) {
    spec_rows = 0;
    if (!(c->fast_loop && c->backend == MHSK_BACKEND_TC && c->gram_variant == 2) || c->world != 1 || n <= 0 ||
        m <= 0 || nnz <= 0)
        return false;
    const int64_t cells = (int64_t)n * (int64_t)m;
    int mode = c->sparse;
    if (mode == -1 && cells >= ((int64_t)1 << 24))
        mode = (double)nnz / (double)cells <= 1e-3 ? 1 : cells <= ((int64_t)1 << 32) ? 3 : 0;
    if (mode != 0) return false;
    if (!c->probe || std::max(n, m) >= (1 << 23)) return false;
    fp4 = c->fp4 && std::max(n, m) < (1 << 24);
    const int32_t bki = fp4 ? 256 : 128;
    const int32_t probe_e = probe_size(true, n, (double)nnz / m, bki, edge_probe_entries(c, n, true));
    const int32_t probe_v = probe_size(true, m, (double)nnz / n, bki, vertex_probe_entries(c, n, true));
    const bool streamed = c->lazy && probe_v > 0 && c->lazy_e && probe_e > 0;
    if (streamed && fp4 && c->spec_v) spec_rows = std::min<int64_t>((int64_t)probe_v * bki, m);
    return streamed;
}

// X_V's probe columns (the lazy vertex operand): columns j < K1 from the CSR
// (k::probe_cols_csr) between zeroing them and counting lo (k::prefix_cols).
// Packing the probe-column edges' X_E rows in full and bit-transposing them
// took 41 + 62 us at config 4.  n_rows: the rows whose lo is counted.
void probe_cols_from_csr(mhsk_ctx* c, bool fp4, const DevInstance& in, const int32_t* src, const int32_t* vnew,
                         int8_t* XV, int64_t ld_v, int32_t* lo, const int32_t* m_cols, const int32_t* n_rows,
                         int64_t rows_v, int64_t K1) {
    const int64_t bytes = fp4 ? K1 / 2 : K1;   // K1: whole 128-byte k-blocks
    const int row_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((rows_v + 7) / 8, (int64_t)c->sms * 16));
    launch_pdl(c, mhsk::k::prefix_cols<false>, row_blocks, 256, 0, XV, ld_v, bytes, rows_v, nullptr, nullptr);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((K1 + 7) / 8, (int64_t)c->sms * 8));
    launch_pdl(c, (fp4 ? mhsk::k::probe_cols_csr<true> : mhsk::k::probe_cols_csr<false>), blocks, 256, 0, m_cols, K1, src, c->eids.ptr, in.ptr, in.vtx, vnew, XV, ld_v, in.n, in.ptr + in.m);
    launch_pdl(c, mhsk::k::prefix_cols<true>, row_blocks, 256, 0, XV, ld_v, bytes, rows_v, n_rows, lo);
    LAUNCH_CHECK();
    c->st.kernel_launches += 3;
}

// The probe outputs of a Gram launch (needed marks, candidates, probe terms)
// and their second set for the speculative vertex probe: swapped, not copied.
void swap_probe_bufs(mhsk_ctx* c) {
    std::swap(c->needed, c->needed_s);
    std::swap(c->cand, c->cand_s);
    std::swap(c->cand_count, c->cand_count_s);
    std::swap(c->pv, c->pv_s);
    std::swap(c->pcm, c->pcm_s);
}
// geometry of the last Gram launch (needed_panels / verification read it)
struct LaunchGeom {
    int32_t pairs = 0, words = 0, begin = 0, count = 0, stride = 1;
    bool cand = false;
};
LaunchGeom last_geom(const mhsk_ctx* c) {
    return LaunchGeom{c->lg_pairs, c->lg_words, c->lg_begin, c->lg_count, c->lg_stride, c->lg_cand};
}
void set_last_geom(mhsk_ctx* c, const LaunchGeom& g) {
    c->lg_pairs = g.pairs;
    c->lg_words = g.words;
    c->lg_begin = g.begin;
    c->lg_count = g.count;
    c->lg_stride = g.stride;
    c->lg_cand = g.cand;
}

void kernelize_fast(mhsk_ctx* c, const DevInstance& in, int32_t rule, int32_t max_rounds,
                    uint8_t* valive, uint8_t* ealive, bool validated) {
    const int32_t n0 = in.n, m0 = in.m;
    c->alive_staged = false;
    reserve_instance_state(c, n0, m0);
    if (n0) CUDA_TRY(cudaMemsetAsync(valive, 1, n0, c->stream));
    if (m0) CUDA_TRY(cudaMemsetAsync(ealive, 1, m0, c->stream));
    const int32_t mx = std::max<int32_t>(std::max(n0, m0), 1);
    c->item_a.reserve(mx);
    c->item_b.reserve(mx);
    c->item_lo.reserve(mx);
    c->vdeg.reserve(mx);
    c->vneed.reserve(mx);
    c->vseen.reserve((mx + 31) / 32);
    c->f_range.reserve(2);
    c->panel_flags.reserve(round_up(std::max<int32_t>(n0, 1), 256) / 256 + 2);   // + a 240-column panel's overhang
    c->state_e.reserve(round_up(std::max<int32_t>(m0, 1), 256) / 256 + 2);
    c->pack_dummy.reserve(2 * (size_t)round_up(std::max<int32_t>(m0, 1), 256));
    c->any_v.reserve(1);
    c->row_sel_e.reserve(round_up(std::max<int32_t>(m0, 1), 256));
    c->pruned.reserve(4);   // [3]: the speculative vertex probe's pruned tiles
    c->hits.reserve(mx);
    c->keep_e.reserve(std::max<int32_t>(m0, 1));
    c->src.reserve(std::max<int32_t>(m0, 1));
    c->scratch.reserve(mx);
    c->dims.reserve(16);
    c->edel.reserve(std::max<int32_t>(m0, 1));
    c->vdel.reserve(std::max<int32_t>(n0, 1));
    c->aff_flag.reserve(mx);
    c->aff_e_ids.reserve(std::max<int32_t>(m0, 1));
    c->aff_v_ids.reserve(std::max<int32_t>(n0, 1));
    c->a_items.reserve(mx);
    c->aff_scratch.reserve(mx);
    const int64_t ld_e0 = round_up(std::max<int32_t>(n0, 1), 128), ld_v0 = round_up(std::max<int32_t>(m0, 1), 128);
    c->XE.reserve(ld_e0 * round_up(std::max<int32_t>(m0, 1), 256));
    c->XV.reserve(ld_v0 * round_up(std::max<int32_t>(n0, 1), 256));
    if (c->incremental)   // rectangles are used only for affected sets <= half the items
        c->XA.reserve(std::max(ld_e0 * round_up(m0 / 2 + 1, 256), ld_v0 * round_up(n0 / 2 + 1, 256)));
    int32_t* dims = c->dims.ptr;
    // dims: [0] m_a [1] n_a [2] m_a2 [3] del_e [4] del_v [5] affected edges (next
    // edge phase) [6] n_a copy [7] affected vertices [8] vertex triangle? [9] rectangle?
    CUDA_TRY(cudaMemsetAsync(dims, 0, 16 * sizeof(int32_t), c->stream));
    // alive counts at the start of the round, known on the host from the
    // previous round's read: they size this round's strides and tile lists
    // (exact for the edge phase, an upper bound for the vertex phase's K);
    // the kernels read the exact sizes from dims.
    int32_t n_cur = n0, m_cur = m0, aff_e = -1;   // aff_e < 0: full round
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gram_events, round_events;
    auto gram_event = [&]() {
        cudaEvent_t a, b;
        CUDA_TRY(cudaEventCreate(&a));
        CUDA_TRY(cudaEventCreate(&b));
        gram_events.emplace_back(a, b);
        round_events.emplace_back(a, b);
        return gram_events.back();
    };
    const int csr_blocks = std::max(1, std::min<int32_t>((m0 + 7) / 8, c->sms * 16));
    // ---- block-sparse mode.  Auto: banded instances (density <= 1e-3) with
    // edges in first-vertex order; otherwise instances whose X_E is block-sparse
    // after component ordering (measured occupancy <= 1/4).
    const int32_t words_e0 = (int32_t)((ld_e0 / 128 + 63) / 64), words_v0 = (int32_t)((ld_v0 / 128 + 63) / 64);
    bool sparse = false, vorder = false;
    int64_t nnz0 = 0;
    if (m0 > 0 && n0 > 0) {
        int64_t& nnz = nnz0;
        if (c->nnz_src == in.ptr) {   // read by this call's validate
            nnz = *c->nnz_host;
        } else {
            CUDA_TRY(cudaMemcpyAsync(&nnz, in.ptr + m0, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
            ctx_sync(c);
        }
        const int64_t cells = (int64_t)n0 * (int64_t)m0;
        const double density = (double)nnz / (double)cells;
        int mode = c->sparse;
        if (mode == -1 && cells >= ((int64_t)1 << 24))
            mode = density <= 1e-3 ? 1 : cells <= ((int64_t)1 << 32) ? 3 : 0;   // 3: probe
        if (mode != 0 && !validated) {   // the sparse set-up reads the CSR: validate first
            validate_or_throw(c, in);
            validated = true;
        }
        if (mode >= 2) {
            vorder = order_components(c, in);
            if (mode == 3) {
                vorder = vorder && sparse_occupancy(c, in, ld_e0, words_e0) <= 0.25;
                mode = vorder ? 2 : 0;
            }
        }
        sparse = mode >= 1;
    }
    if (!validated && (m0 == 0 || n0 == 0)) {
        validate_or_throw(c, in);
        validated = true;
    }
    if (sparse) {
        c->sort_keys.reserve(m0);
        c->sort_keys_out.reserve(m0);
        c->sort_vals.reserve(m0);
        c->perm.reserve(m0);
        c->mask_e.reserve((size_t)(round_up(m0, 256) / 256) * words_e0);
        c->kblocks.reserve(1);
        CUDA_TRY(cudaMemsetAsync(c->kblocks.ptr, 0, sizeof(unsigned long long), c->stream));
        c->mask_v.reserve((size_t)(round_up(n0, 256) / 256) * words_v0);
        if (vorder) {
            c->vids_p.reserve(n0);
            c->vnew_p.reserve(n0);
        } else {
            launch_pdl(c, mhsk::k::edge_first_vertex, (m0 + 255) / 256, 256, 0, m0, n0, in.ptr, in.vtx,
                                                                                c->sort_keys.ptr, c->sort_vals.ptr);
            LAUNCH_CHECK();
            size_t temp = 0;
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp, c->sort_keys.ptr, c->sort_keys_out.ptr,
                                                     c->sort_vals.ptr, c->perm.ptr, m0, 0, 32, c->stream));
            c->sort_temp.reserve(std::max<size_t>(temp, 1));
            CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->sort_temp.ptr, temp, c->sort_keys.ptr, c->sort_keys_out.ptr,
                                                     c->sort_vals.ptr, c->perm.ptr, m0, 0, 32, c->stream));
            c->st.kernel_launches += 3;
        }
    }
    // vertex order of the sparse layout: X_E columns / X_V rows are the alive
    // vertices in vperm order (vorder) or in original order
    // dense operands: packed E2M1 (two items per byte, K padded to 256 items)
    // or int8 (K padded to 128); block-sparse operands are int8
    // (f32 accumulation: counts, <= K, are exact below 2^24)
    const bool fp4 = c->fp4 && !sparse && std::max(n0, m0) < (1 << 24);
    // probe pruning of dense triangle tiles (single rank and sharded alike)
    // (the FP4 probe compares f32 sums of counts: exact while n, m < 2^23)
    int32_t* lo_e = (c->probe && !sparse && std::max(n0, m0) < (1 << 23)) ? c->item_lo.ptr : nullptr;
    int32_t* lo_v = lo_e;   // the vertex phase reuses the buffer after the edge phase
    const int32_t bki = fp4 ? 256 : 128;   // items per 128-byte k-block
    const double mean_size = m0 ? (double)nnz0 / m0 : 1.0, mean_degree = n0 ? (double)nnz0 / n0 : 1.0;
    if (lo_e) CUDA_TRY(cudaMemsetAsync(c->pruned.ptr, 0, 4 * sizeof(unsigned long long), c->stream));
    const int32_t* vnew_s = vorder ? c->vnew_p.ptr : c->vnew.ptr;
    const int32_t* vids_s = vorder ? c->vids_p.ptr : c->vids.ptr;
    int64_t rounds = 0;
    unsigned long long pruned_seen[2] = {0, 0};
    for (;;) {
        if (max_rounds >= 0 && rounds >= max_rounds) break;
        ++rounds;
        // No edge lost a vertex since the last edge phase (aff_e == 0, counted
        // by the previous round): the edge phase cannot delete anything
        // (§4b), so no edge dies, no vertex loses an edge, and the vertex
        // phase cannot either -- this is the (counted) no-change round.
        if (aff_e == 0) break;
        // small phases: the full triangle costs less than the rectangle's bookkeeping
        const bool big = (int64_t)n_cur * (int64_t)m_cur >= (int64_t)1 << 24;
        bool full_round = aff_e < 0 || !c->incremental || !big || sparse;
        // geometry: the current sizes
        const int32_t gm = m_cur, gn = n_cur;
        const int64_t ld_e = fp4 ? round_up(std::max<int32_t>(gn, 1), 256) / 2 : round_up(std::max<int32_t>(gn, 1), 128);
        const int64_t rows_e = round_up(std::max<int32_t>(gm, 1), 256);
        const int64_t ld_v = fp4 ? round_up(std::max<int32_t>(gm, 1), 256) / 2 : round_up(std::max<int32_t>(gm, 1), 128);
        const int64_t rows_v = round_up(std::max<int32_t>(gn, 1), 256);
        // round 1 of a streamed call: tiles_e already holds the band-major list
        // (a complete triangle list plus dummy entries, on the copy stream)
        const bool band_list = rounds == 1 && c->band_M == gm && c->band_fp4 == fp4;
        if (!band_list) device_tiles(c, gm, c->tiles_e, c->tiles_e_host, c->tiles_e_M, fp4);
        const TileVec& tl_e = band_list ? c->band_host : c->tiles_e_host;   // what tiles_e holds
        device_tiles(c, gn, c->tiles_v, c->tiles_v_host, c->tiles_v_M, fp4);
        // probe sizes (k-blocks): ~PROBE_ENTRIES entries of a mean-size item
        const int32_t probe_e = probe_size(lo_e != nullptr, gn, mean_size, bki,
                                           edge_probe_entries(c, gn, c->up_pending));
        const int32_t probe_v = probe_size(lo_v != nullptr, gm, mean_degree, bki,
                                           vertex_probe_entries(c, gn, c->up_pending));
        // With probing, a rectangle (affected rows x all, full K) beats the
        // probed triangle (every pair, probe columns only; lazy operands in a
        // full round) only while affected x K < M/2 x probe columns: a round
        // whose affected edges exceed that runs as a full round.  The vertex
        // phase of a non-full round applies the same test on the device.
        const int32_t kb_e = std::max<int32_t>(1, (gn + bki - 1) / bki);
        const int32_t kb_v = std::max<int32_t>(1, (gm + bki - 1) / bki);
        const bool probe_rule = probe_e > 0 && c->rect_rule == 0;
        if (!full_round && probe_rule && (int64_t)aff_e * 2 * kb_e > (int64_t)m_cur * probe_e)
            full_round = true;
        int edge_mode = 0;   // 0 skip, 1 triangle, 2 rectangle
        // lazy vertex operand: X_V gets only its probe columns up front, the
        // panels the probe leaves undecided are packed after the probe pass;
        // degrees / need come from the edge phase's CSR pass
        const bool lazy_v = c->lazy && full_round && !sparse && lo_v != nullptr && probe_v > 0 &&
                            gm > 0 && gn > 0;
        // lazy edge operand: X_E only in its probe columns; full rows for the
        // panels of marked / candidate edge tiles, the rows the vertex phase's
        // probe transpose reads, and all rows if a vertex panel is packed in full
        const bool lazy_e = lazy_v && c->lazy_e && probe_e > 0;
        const int32_t npanels_e = (int32_t)(rows_e / 256);
        auto pack_flagged_edge_panels = [&](const uint8_t* rows_sel) {
            launch_pdl(c, (fp4 ? mhsk::k::pack_rows_csr<true> : mhsk::k::pack_rows_csr<false>), pack_blocks(c, rows_e), mhsk::k::PACK_WARPS * 32, 0, gm, (int32_t)rows_e, c->eids.ptr, in.ptr, in.vtx, in.dem, c->vnew.ptr, c->XE.ptr, ld_e,
                c->pack_dummy.ptr, c->pack_dummy.ptr + rows_e, dims + 0, nullptr, 0, nullptr, nullptr, -1,
                c->state_e.ptr, rows_sel, nullptr, nullptr, nullptr, nullptr, nullptr, 0, -1, nullptr, nullptr, 0);
            LAUNCH_CHECK();
            launch_pdl(c, mhsk::k::mark_packed_panels, (npanels_e + 255) / 256, 256, 0, c->state_e.ptr, npanels_e);
            LAUNCH_CHECK();
            c->st.kernel_launches += 2;
        };
        round_events.clear();
        // MHSK_STREAM_TRACE=1: round 1's timeline (stream events, ms after the
        // call's start), printed after the round's host read
        std::vector<std::pair<const char*, cudaEvent_t>> trace;
        const bool tracing = rounds == 1 && getenv("MHSK_STREAM_TRACE");
        auto mark = [&](const char* what) {
            if (!tracing) return;
            trace.emplace_back(what, nullptr);
            CUDA_TRY(cudaEventCreate(&trace.back().second));
            CUDA_TRY(cudaEventRecord(trace.back().second, c->stream));
        };
        // speculative vertex probe of this round (streamed round 1 only):
        // launched during the upload / adopted by the vertex phase
        bool spec_launched = false, spec_ok = false;
        LaunchGeom spec_geom;
        CUDA_TRY(cudaMemsetAsync(dims + 3, 0, 2 * sizeof(int32_t), c->stream));
        // alive items -> rows.  Dense: original order.  Sparse: edges in the
        // sort order (perm); vertices in component order (vorder) or original
        // order.  Reordered rows carry their original id as tie-break rank.
        if (!vorder) compact(c, valive, n0, c->vnew.ptr, c->vids.ptr, dims + 1);
        if (!sparse) compact(c, ealive, m0, c->enew.ptr, c->eids.ptr, dims + 0);
        const int32_t words_e = (int32_t)((ld_e / 128 + 63) / 64), words_v = (int32_t)((ld_v / 128 + 63) / 64);
        if (sparse) compact_impl(c, ealive, m0, nullptr, c->perm.ptr, nullptr, c->eids.ptr, dims + 0);
        if (vorder) compact_impl(c, valive, n0, nullptr, c->vperm.ptr, c->vnew_p.ptr, c->vids_p.ptr, dims + 1);
        // ---- edge phase: M = m_a (dims[0]), K = n_a (dims[1])
        CUDA_TRY(cudaMemsetAsync(c->hits.ptr, 0, mx * sizeof(int32_t), c->stream));
        if (m0) CUDA_TRY(cudaMemsetAsync(c->edel.ptr, 0, m0, c->stream));
        if (gm && sparse) {
            CUDA_TRY(cudaMemsetAsync(c->mask_e.ptr, 0, (rows_e / 256) * words_e * sizeof(unsigned long long),
                                     c->stream));
            CUDA_TRY(cudaMemsetAsync(dims + 11, 0, sizeof(int32_t), c->stream));
            launch_pdl(c, mhsk::k::mask_rows_csr, csr_blocks, 256, 0, gm, c->eids.ptr, in.ptr, in.vtx,
                                                                     vnew_s, c->mask_e.ptr, words_e, dims + 0);
            launch_pdl(c, mhsk::k::pack_rows_sparse, pack_blocks(c, rows_e), mhsk::k::PACK_WARPS * 32, 0, gm, (int32_t)rows_e, c->eids.ptr, in.ptr, in.vtx, in.dem, vnew_s, c->XE.ptr, ld_e,
                c->mask_e.ptr, words_e, c->item_a.ptr, c->item_b.ptr, dims + 11, dims + 0);
            LAUNCH_CHECK();
            auto ev = gram_event();
            CUDA_TRY(cudaEventRecord(ev.first, c->stream));
            if (rule == MHSK_RULE_DP)
                launch_gram_fast<mhsk::PHASE_DP>(c, c->XE.ptr, rows_e, c->XE.ptr, rows_e, ld_e, gm,
                                                 c->tiles_e.ptr, (int32_t)tl_e.size(), dims + 0,
                                                 c->item_a.ptr, c->item_b.ptr, nullptr, nullptr, nullptr,
                                                 c->mask_e.ptr, words_e, dims + 11, c->eids.ptr);
            else
                launch_gram_fast<mhsk::PHASE_SE>(c, c->XE.ptr, rows_e, c->XE.ptr, rows_e, ld_e, gm,
                                                 c->tiles_e.ptr, (int32_t)tl_e.size(), dims + 0,
                                                 c->item_a.ptr, c->item_b.ptr, nullptr, nullptr, nullptr,
                                                 c->mask_e.ptr, words_e, dims + 11, c->eids.ptr);
            CUDA_TRY(cudaEventRecord(ev.second, c->stream));
            edge_mode = 1;
            allreduce_hits(c, m0);
            launch_pdl(c, mhsk::k::commit_phase<false>, (gm + 255) / 256, 256, 0, gm, c->hits.ptr, nullptr, c->eids.ptr, ealive, c->keep_e.ptr, dims + 3, dims + 0,
                c->edel.ptr);
            LAUNCH_CHECK();
            compact_dyn(c, c->keep_e.ptr, gm, dims + 0, c->scratch.ptr, c->src.ptr, dims + 2);
            c->st.kernel_launches += 4;
        } else if (gm) {
            // FP4 lazy vertex phase: need by original vertex id, two-tier (the
            // edge pack's seen map of max-demand rows + need_low for the rest),
            // and later rounds count alive members by an alive-bit test
            const bool orig_need = lazy_v && fp4;
            const bool all_alive = n_cur == n0 && !vorder;
            if (lazy_v) {
                if (!fp4) CUDA_TRY(cudaMemsetAsync(c->vdeg.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                CUDA_TRY(cudaMemsetAsync(c->vneed.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                CUDA_TRY(cudaMemsetAsync(c->vseen.ptr, 0, (size_t)(std::max(gn, n0) + 31) / 32 * sizeof(uint32_t),
                                         c->stream));
                if (orig_need) {
                    c->need_low_p.reserve(std::max(n0, 1));
                    CUDA_TRY(cudaMemsetAsync(c->need_low_p.ptr, 0, (size_t)n0 * sizeof(int32_t), c->stream));
                    if (!all_alive) {
                        const int32_t words = (n0 + 31) / 32;
                        c->alive_bits.reserve(words);
                        launch_pdl(c, mhsk::k::bits_from_bytes, std::max(1, std::min((words + 7) / 8, c->sms * 4)), 256, 0, valive, n0, c->alive_bits.ptr);
                        LAUNCH_CHECK();
                        c->st.kernel_launches += 1;
                    }
                }
                CUDA_TRY(cudaMemsetAsync(c->f_range.ptr, 0x7f, sizeof(int32_t), c->stream));
                CUDA_TRY(cudaMemsetAsync(c->f_range.ptr + 1, 0, sizeof(int32_t), c->stream));
                launch_pdl(c, mhsk::k::demand_range, std::max(1, std::min((gm + 255) / 256, c->sms * 4)), 256, 0, dims + 0, c->eids.ptr, in.dem, c->f_range.ptr);
                LAUNCH_CHECK();
                c->st.kernel_launches += 1;
            }
            if (lazy_e) CUDA_TRY(cudaMemsetAsync(c->state_e.ptr, 0, npanels_e + 2, c->stream));
            // all vertices alive (n_cur == n0, original order): columns are vertex ids
            const int32_t* vmap = (n_cur == n0 && !vorder) ? nullptr : c->vnew.ptr;
            // round 1 of an unvalidated call: validation fused into this pack
            // (scan_members: one streaming pass over the members; per-edge
            // checks in pack_rows_csr), checked right after it -- before any
            // kernel that indexes by member ids
            const bool fused_validation = !validated && vmap == nullptr;
            // the edge phase's probe / full-K launches over the triangle list
            // (passes 1 / 2; a band [t_lo, t_hi) of it while the upload streams)
            auto edge_gram = [&](int passes, int32_t t_lo = 0, int32_t t_hi = INT32_MAX, bool first = true,
                                 int32_t i_lo = 0, int32_t i_hi = INT32_MAX) {
                auto ev = gram_event();
                CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                if (rule == MHSK_RULE_DP)
                    launch_gram_fast<mhsk::PHASE_DP>(c, c->XE.ptr, rows_e, c->XE.ptr, rows_e, ld_e, gm, c->tiles_e.ptr,
                                                     (int32_t)tl_e.size(), dims + 0, c->item_a.ptr,
                                                     c->item_b.ptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr,
                                                     nullptr, fp4, lo_e, c->pruned.ptr, probe_e, passes,
                                                     /*defer_verify=*/true, t_lo, t_hi, first, i_lo, i_hi);
                else
                    launch_gram_fast<mhsk::PHASE_SE>(c, c->XE.ptr, rows_e, c->XE.ptr, rows_e, ld_e, gm, c->tiles_e.ptr,
                                                     (int32_t)tl_e.size(), dims + 0, c->item_a.ptr,
                                                     c->item_b.ptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr,
                                                     nullptr, fp4, lo_e, c->pruned.ptr, probe_e, passes,
                                                     /*defer_verify=*/true, t_lo, t_hi, first, i_lo, i_hi);
                CUDA_TRY(cudaEventRecord(ev.second, c->stream));
            };
            // streamed upload (host API, round 1, lazy edge operand, one rank):
            // chunk b of the member array lands on the copy stream; its members
            // are scanned, its complete edges packed and the edge probe run
            // over the triangle tiles it completes while later chunks are still
            // in flight (band-major tile list, schedule.h)
            const bool streamed = c->up_pending && band_list && fused_validation && lazy_e && c->world == 1 &&
                                  full_round;
            if (band_list) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->band_ev, 0));
            if (c->up_pending && !streamed) wait_upload(c);
            const int nchunks = streamed ? (int)c->up_ev.size() : 1;
            if (fused_validation) {
                CUDA_TRY(cudaMemsetAsync(c->counters.ptr + 4, 0, sizeof(int32_t), c->stream));
                CUDA_TRY(cudaMemsetAsync(c->counters.ptr + 5, 0x7F, sizeof(int32_t), c->stream));
                c->vdesc.reserve(2);
                CUDA_TRY(cudaMemsetAsync(c->vdesc.ptr, 0, 2 * sizeof(unsigned long long), c->stream));
            }
            bool first_band = true;
            int32_t band_rows = 0;   // rows whose probe terms are in place
            // Speculative vertex probe (FP4): the vertex phase's probe columns
            // are the first K1 survivors of the edge phase -- the first K1
            // edges if it deletes nothing, which holds on most instances
            // (every random config).  Once the chunk completing their panels
            // has landed, their X_E rows are packed in full, transposed into
            // X_V's probe columns and the vertex probe pass runs while later
            // chunks are still in flight, into the *_s buffers.  Every vertex
            // counts as having an edge (need > 0): a degree-0 vertex only lets
            // more pairs through to the exact full-K / candidate decisions.
            // The vertex phase adopts the result iff the edge phase deleted no
            // edge (then operand, lo and every probe term equal the ones it
            // would compute); otherwise it runs its own probe.
            int spec_b = -1;
            const int64_t spec_rows = std::min<int64_t>((int64_t)probe_v * bki, gm);
            if (streamed && fp4 && lazy_v && c->spec_v && probe_v > 0 && gn > 0 && max_rounds != 0)
                for (int b = 0; b + 1 < nchunks; ++b)
                    if (c->up_E[b] >= spec_rows) {
                        spec_b = b;
                        break;
                    }
            auto spec_vertex_probe = [&] {
                using namespace mhsk::k;
                c->spec_dims.reserve(2);
                c->lo_s.reserve(std::max(n0, 1));
                c->one_s.reserve(std::max(n0, 1));
                launch_pdl(c, copy_i32, 1, 1, 0, dims + 1, c->spec_dims.ptr);       // {n_a, m_a}: M, K
                launch_pdl(c, copy_i32, 1, 1, 0, dims + 0, c->spec_dims.ptr + 1);
                CUDA_TRY(cudaMemsetAsync(c->one_s.ptr, 1, (size_t)n0 * sizeof(int32_t), c->stream));
                // X_V column j <- edge j (no deletion: eids is the identity)
                probe_cols_from_csr(c, true, in, c->eids.ptr, nullptr, c->XV.ptr, ld_v, c->lo_s.ptr,
                                    c->spec_dims.ptr + 1, c->spec_dims.ptr, rows_v, (int64_t)probe_v * bki);
                c->st.kernel_launches += 2;
                const LaunchGeom edge_geom = last_geom(c);
                swap_probe_bufs(c);
                auto ev = gram_event();
                CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                launch_gram_fast<mhsk::PHASE_MD>(c, c->XV.ptr, rows_v, c->XV.ptr, rows_v, ld_v, gn, c->tiles_v.ptr,
                                                 (int32_t)c->tiles_v_host.size(), c->spec_dims.ptr, c->one_s.ptr,
                                                 nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr,
                                                 fp4, c->lo_s.ptr, c->pruned.ptr + 3, probe_v, /*passes=*/1,
                                                 /*defer_verify=*/true);
                CUDA_TRY(cudaEventRecord(ev.second, c->stream));
                spec_geom = last_geom(c);
                swap_probe_bufs(c);
                set_last_geom(c, edge_geom);
                spec_launched = true;
            };
            for (int b = 0; b < nchunks; ++b) {
                if (streamed) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->up_ev[b], 0));
                mark("chunk");
                const int64_t k_lo = streamed ? c->up_K[b] : 0, k_hi = streamed ? c->up_K[b + 1] : -1;
                const int64_t r_lo = streamed && b ? c->up_E[b - 1] : 0;
                const int64_t r_hi = streamed && b + 1 < nchunks ? c->up_E[b] : -1;
                if (fused_validation) {
                    const bool smem_map = lazy_v && (int64_t)n0 <= mhsk::k::SCAN_SMEM_BITS;
                    const size_t map_bytes = smem_map ? (size_t)(n0 + 31) / 32 * 4 : 0;
                    auto scan = [&](int64_t lo, int64_t hi, bool check_full) {
                        launch_pdl(c, (!lazy_v ? mhsk::k::scan_members<0> : smem_map ? mhsk::k::scan_members<1> : mhsk::k::scan_members<2>), c->sms * 2, mhsk::k::SCAN_THREADS, map_bytes, n0, m0, in.ptr, in.vtx, lazy_v ? c->vseen.ptr : nullptr, c->f_range.ptr,
                            c->counters.ptr + 4, c->vdesc.ptr, lo, hi, check_full ? c->seen_all.ptr : nullptr);
                        LAUNCH_CHECK();
                        c->st.kernel_launches += 1;
                    };
                    auto check_seen = [&] {   // is every vertex seen already?
                        if (!lazy_v) return;
                        c->seen_all.reserve(1);
                        launch_pdl(c, mhsk::k::seen_full, 1, 1024, 0, c->vseen.ptr, n0, c->seen_all.ptr);
                        LAUNCH_CHECK();
                        c->st.kernel_launches += 1;
                    };
                    if (streamed) {
                        scan(k_lo, k_hi, b > 0);
                        if (b == 0) check_seen();
                    } else {   // the first eighth sets the map, the rest usually only validates
                        const int64_t nnz_all = nnz0;
                        const int64_t split = nnz_all / 8 / 4 * 4;
                        scan(0, split, false);
                        check_seen();
                        scan(split, nnz_all, true);
                    }
                }
                // later rounds: the alive and seen maps in shared memory
                // (pack_rows_csr map_words) while two maps fit beside 2+ CTAs per SM
                const int32_t pack_map_words = (orig_need && !all_alive && (int64_t)(n0 + 31) / 32 * 8 <= PACK_SMAP_MAX)
                                             ? (n0 + 31) / 32 : 0;
                const size_t pack_smem = (size_t)pack_map_words * 8;
                int pack_grid = pack_blocks(c, rows_e);
                if (pack_smem) {
                    set_pack_smem_limit(c->device);
                    const int per_sm = std::max<int>(1, std::min<int>(5, (int)((220u << 10) / (pack_smem + (5u << 10)))));
                    pack_grid = std::min(pack_grid, c->sms * per_sm);
                }
                launch_pdl(c, (fp4 ? mhsk::k::pack_rows_csr<true> : mhsk::k::pack_rows_csr<false>), pack_grid, mhsk::k::PACK_WARPS * 32, pack_smem, gm, (int32_t)rows_e, c->eids.ptr, in.ptr, in.vtx, in.dem, vmap, c->XE.ptr, ld_e,
                    c->item_a.ptr, c->item_b.ptr, dims + 0, lo_e, (int64_t)probe_e * bki,
                    (lazy_v && !fp4) ? c->vdeg.ptr : nullptr, (lazy_v && !orig_need) ? c->vneed.ptr : nullptr,
                    lazy_e ? (int64_t)probe_e * 128 : -1, nullptr, nullptr, lazy_v ? c->vseen.ptr : nullptr,
                    c->f_range.ptr, fused_validation ? c->counters.ptr + 4 : nullptr, in.ptr + m0,
                    fused_validation ? c->vdesc.ptr : nullptr, r_lo, r_hi,
                    (orig_need && !all_alive) ? c->alive_bits.ptr : nullptr, orig_need ? c->need_low_p.ptr : nullptr,
                    pack_map_words);
                LAUNCH_CHECK();
                if (fused_validation && b + 1 == nchunks) {   // every member scanned, every edge checked
                    CUDA_TRY(cudaMemcpyAsync(c->counters_host + 4, c->counters.ptr + 4, 2 * sizeof(int32_t),
                                             cudaMemcpyDeviceToHost, c->stream));
                    CUDA_TRY(cudaMemcpyAsync(c->desc_host, c->vdesc.ptr, 2 * sizeof(unsigned long long),
                                             cudaMemcpyDeviceToHost, c->stream));
                    CUDA_TRY(cudaEventRecord(c->val_ev, c->stream));
                }
                if (streamed && c->band_t[b + 1] > c->band_t[b]) {
                    // probe terms of the rows completed since the last band
                    // (every earlier row's are in place)
                    edge_gram(1, c->band_t[b], c->band_t[b + 1], first_band, first_band ? 0 : band_rows,
                              b + 1 < nchunks ? c->up_E[b] : gm);
                    first_band = false;
                    band_rows = b + 1 < nchunks ? c->up_E[b] : gm;
                }
                if (b == spec_b) spec_vertex_probe();
            }
            if (streamed) c->up_pending = false;
            const bool edge_probed = streamed && !first_band;
            mark("bands");
            // The validation flags are read when the host next needs them: before
            // the first kernel that indexes memory by member ids or offsets.  On
            // the lazy edge path the edge probe (it reads only X_E and the item
            // arrays) is enqueued first, so the host check overlaps it.
            bool pending_validation = fused_validation;
            auto settle_validation = [&] {
                if (!pending_validation) return;
                CUDA_TRY(cudaEventSynchronize(c->val_ev));
                if (c->desc_host[0] != c->desc_host[1]) c->counters_host[4] = 1;   // a descent inside an edge
                throw_if_invalid(c);
                pending_validation = false;
                validated = true;
            };
            if (!lazy_e) settle_validation();
            if (orig_need) {
                launch_pdl(c, mhsk::k::need_from_seen_ids, std::max(1, std::min((gn + 255) / 256, c->sms * 4)), 256, 0, dims + 1, vids_s, c->vseen.ptr, c->need_low_p.ptr,
                                                           c->f_range.ptr, c->vneed.ptr, (const int32_t*)nullptr);
                LAUNCH_CHECK();
                c->st.kernel_launches += 1;
            } else if (lazy_v) {
                launch_pdl(c, mhsk::k::need_from_seen, std::max(1, std::min((gn + 255) / 256, c->sms * 4)), 256, 0, dims + 1, c->vseen.ptr, c->f_range.ptr, c->vneed.ptr);
                LAUNCH_CHECK();
                c->st.kernel_launches += 1;
            }
            edge_mode = full_round ? 1 : aff_e == 0 ? 0
                      : (probe_rule ? (int64_t)aff_e * 2 * kb_e > (int64_t)m_cur * probe_e : 2ll * aff_e > m_cur) ? 1
                      : 2;
            if (getenv("MHSK_DEBUG_ROUNDS"))
                fprintf(stderr, "[round %lld] full %d edge_mode %d aff_e %d m_cur %d n_cur %d lazy_v %d lazy_e %d probe_e %d probe_v %d\n",
                        (long long)rounds, (int)full_round, edge_mode, aff_e, m_cur, n_cur, (int)lazy_v, (int)lazy_e,
                        probe_e, probe_v);
            const int64_t rows_a = round_up(std::max<int32_t>(aff_e, 1), 256);
            if (edge_mode == 2) {
                // A rows: the affected edges (marked after the last vertex phase)
                launch_pdl(c, mhsk::k::gather_ids, (aff_e + 255) / 256, 256, 0, c->aff_e_ids.ptr, c->enew.ptr, c->a_items.ptr, dims + 5);
                launch_pdl(c, mhsk::k::copy_i32, 1, 1, 0, dims + 1, dims + 6);
                launch_pdl(c, (fp4 ? mhsk::k::pack_rows_csr<true> : mhsk::k::pack_rows_csr<false>), pack_blocks(c, rows_a), mhsk::k::PACK_WARPS * 32, 0, aff_e, (int32_t)rows_a, c->aff_e_ids.ptr, in.ptr, in.vtx, in.dem, c->vnew.ptr, c->XA.ptr,
                    ld_e, c->aff_scratch.ptr, c->scratch.ptr, dims + 5, nullptr, 0, nullptr, nullptr, -1, nullptr,
                    nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, -1, nullptr, nullptr, 0);
                LAUNCH_CHECK();
                rect_tiles(c, aff_e, m_cur, fp4);
                c->st.kernel_launches += 3;
            }
            if (edge_mode == 1 && lazy_e) {
                // probe launch (already run band by band if streamed), then the
                // undecided panels in full, candidates, full pass
                if (!edge_probed) edge_gram(1);
                settle_validation();
                if (c->lg_count > 0) {
                    // marked tiles: their panels in full; candidate pairs: just their rows
                    CUDA_TRY(cudaMemsetAsync(c->row_sel_e.ptr, 0, rows_e, c->stream));
                    launch_pdl(c, mhsk::k::needed_panels, c->sms * 2, 256, 0, c->needed.ptr, c->lg_pairs, c->lg_words, c->tiles_e.ptr, c->lg_begin, c->lg_count,
                        c->lg_stride, c->lg_cand ? c->cand.ptr : nullptr, c->cand_count.ptr,
                        c->cand_cap, c->state_e.ptr, pair_bn(fp4), nullptr, c->row_sel_e.ptr, (const int32_t*)nullptr);
                    LAUNCH_CHECK();
                    c->st.kernel_launches += 1;
                    pack_flagged_edge_panels(c->row_sel_e.ptr);
                    if (rule == MHSK_RULE_DP)
                        launch_verify<mhsk::PHASE_DP>(c, c->XE.ptr, ld_e, dims + 0, fp4, c->item_a.ptr, c->item_b.ptr);
                    else
                        launch_verify<mhsk::PHASE_SE>(c, c->XE.ptr, ld_e, dims + 0, fp4, c->item_a.ptr, c->item_b.ptr);
                    edge_gram(2);
                    c->st.kernel_launches += 1;
                }
            } else if (edge_mode) {
                auto ev = gram_event();
                CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                if (rule == MHSK_RULE_DP)
                    launch_edge_gram<mhsk::PHASE_DP>(c, edge_mode == 2, c->XA.ptr, rows_a, rows_e, ld_e, gm,
                                                     dims, c->a_items.ptr, fp4, lo_e, probe_e);
                else
                    launch_edge_gram<mhsk::PHASE_SE>(c, edge_mode == 2, c->XA.ptr, rows_a, rows_e, ld_e, gm,
                                                     dims, c->a_items.ptr, fp4, lo_e, probe_e);
                CUDA_TRY(cudaEventRecord(ev.second, c->stream));
            }
            settle_validation();   // (every path settled above; a safety net)
            allreduce_hits(c, m0);
            launch_pdl(c, mhsk::k::commit_phase<false>, (gm + 255) / 256, 256, 0, gm, c->hits.ptr, nullptr, c->eids.ptr, ealive, c->keep_e.ptr, dims + 3, dims + 0,
                c->edel.ptr);
            LAUNCH_CHECK();
            // survivors of the edge phase: X_V column j <- X_E row src[j]; m_a2 -> dims[2]
            compact_dyn(c, c->keep_e.ptr, gm, dims + 0, c->scratch.ptr, c->src.ptr, dims + 2);
            c->st.kernel_launches += 2;
            mark("edge_done");
            if (spec_launched) {   // the speculative vertex probe holds iff no edge was deleted
                CUDA_TRY(cudaMemcpyAsync(c->dims_host + 12, dims + 3, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                         c->stream));
                CUDA_TRY(cudaEventRecord(c->edge_ev, c->stream));
            }
        } else {
            CUDA_TRY(cudaMemsetAsync(dims + 2, 0, sizeof(int32_t), c->stream));
            CUDA_TRY(cudaMemsetAsync(dims + 3, 0, sizeof(int32_t), c->stream));
        }
        // ---- vertex phase: M = n_a (dims[1]), K = m_a2 (dims[2])
        if (n0) CUDA_TRY(cudaMemsetAsync(c->vdel.ptr, 0, n0, c->stream));
        if (gn) {
            CUDA_TRY(cudaMemsetAsync(c->hits.ptr, 0, mx * sizeof(int32_t), c->stream));
            CUDA_TRY(cudaMemsetAsync(c->item_b.ptr, 0, mx * sizeof(int32_t), c->stream));
            if (sparse) {
                CUDA_TRY(cudaMemsetAsync(c->mask_v.ptr, 0,
                                         (rows_v / 256) * words_v * sizeof(unsigned long long), c->stream));
                if (gm) {
                    launch_pdl(c, mhsk::k::mask_cols_csr, csr_blocks, 256, 0, gm, c->eids.ptr, c->scratch.ptr, in.ptr, in.vtx, vnew_s, c->mask_v.ptr, words_v,
                        dims + 0);
                    LAUNCH_CHECK();
                }
                launch_pdl(c, mhsk::k::transpose_sparse, (int)(rows_v / 128), mhsk::k::TP_WARPS * 32, 0, c->XE.ptr, ld_e, c->src.ptr, c->mask_e.ptr, words_e, c->mask_v.ptr, words_v, c->XV.ptr,
                    ld_v, c->item_a.ptr, dims + 1);
            } else if (lazy_v) {
                auto probe_operand = [&] {
                    // probe columns only: the first K1 survivors of the edge phase,
                    // from the CSR; their popcounts are lo_v.  Degrees / need: the
                    // edge phase's accumulators minus the edges it deleted.
                    probe_cols_from_csr(c, fp4, in, c->src.ptr, vnew_s, c->XV.ptr, ld_v, lo_v, dims + 2, dims + 1,
                                        rows_v, (int64_t)probe_v * bki);
                };
                if (!spec_launched) probe_operand();
                launch_pdl(c, mhsk::k::fix_deleted_edges, csr_blocks, 256, 0, m0, in.ptr, in.vtx, c->edel.ptr, vnew_s, fp4 ? nullptr : c->vdeg.ptr, c->vneed.ptr, dims + 1,
                    dims + 3);
                LAUNCH_CHECK();
                // need over the survivors (gated: only when the edge phase deleted
                // edges), two-tier (seen_alive_edges): a map of the members of
                // alive edges with the largest demand fmax -- its first eighth
                // usually covers every alive vertex, then the rest is skipped --
                // and atomicMax over the members of the other alive edges
                if ((int64_t)n0 <= mhsk::k::MAP_SMEM_BITS) {
                    const int32_t words = (n0 + 31) / 32;
                    const size_t map_bytes = (size_t)words * 4;
                    c->seen2.reserve(words);
                    c->seen_all.reserve(2);
                    c->need_low.reserve(std::max(n0, 1));
                    CUDA_TRY(cudaMemsetAsync(c->seen2.ptr, 0, map_bytes, c->stream));
                    CUDA_TRY(cudaMemsetAsync(c->seen_all.ptr, 0, 2 * sizeof(int32_t), c->stream));
                    CUDA_TRY(cudaMemsetAsync(c->need_low.ptr, 0, (size_t)n0 * sizeof(int32_t), c->stream));
                    const int32_t e_split = m0 / 8;
                    const int vb = std::max(1, std::min((n0 + 255) / 256, c->sms * 4));
                    launch_pdl(c, mhsk::k::seen_alive_edges, c->sms * 2, 512, map_bytes, n0, 0, e_split, in.ptr, in.vtx, ealive, in.dem, c->f_range.ptr, c->seen2.ptr, c->need_low.ptr,
                        dims + 3, nullptr);
                    launch_pdl(c, mhsk::k::seen_misses_alive, vb, 256, 0, c->seen2.ptr, valive, n0,
                                                                         c->seen_all.ptr + 1, dims + 3);
                    launch_pdl(c, mhsk::k::seen_full_from_missing, 1, 1, 0, c->seen_all.ptr + 1, c->seen_all.ptr);
                    launch_pdl(c, mhsk::k::seen_alive_edges, c->sms * 2, 512, map_bytes, n0, e_split, m0, in.ptr, in.vtx, ealive, in.dem, c->f_range.ptr, c->seen2.ptr,
                        c->need_low.ptr, dims + 3, c->seen_all.ptr);
                    launch_pdl(c, mhsk::k::need_from_seen_ids, vb, 256, 0, dims + 1, vids_s, c->seen2.ptr,
                                                                          c->need_low.ptr, c->f_range.ptr,
                                                                          c->vneed.ptr, dims + 3);
                    LAUNCH_CHECK();
                    c->st.kernel_launches += 5;
                } else {
                    launch_pdl(c, mhsk::k::need_from_csr, csr_blocks, 256, 0, m0, in.ptr, in.vtx, in.dem, ealive,
                                                                             vnew_s, c->vneed.ptr, dims + 3, (const int32_t*)nullptr);
                    c->st.kernel_launches += 1;
                }
                mark("need");
                if (spec_launched) {   // (the need passes above are queued meanwhile)
                    CUDA_TRY(cudaEventSynchronize(c->edge_ev));
                    spec_ok = c->dims_host[12] == 0;
                    if (!spec_ok) probe_operand();
                }
            } else {
                // input rows split into chunks of TP_CHUNK (more CTAs in flight);
                // partial degrees are added atomically
                const int64_t width_v = fp4 ? ld_v * 2 : ld_v;
                const int jchunks = (int)std::max<int64_t>(1, (width_v + mhsk::k::TP_CHUNK - 1) / mhsk::k::TP_CHUNK);
                if (jchunks > 1) {
                    CUDA_TRY(cudaMemsetAsync(c->item_a.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                    if (lo_v) CUDA_TRY(cudaMemsetAsync(lo_v, 0, (size_t)gn * sizeof(int32_t), c->stream));
                }
                launch_pdl(c, (fp4 ? mhsk::k::transpose_pack<true> : mhsk::k::transpose_pack<false>), dim3((unsigned)(rows_v / 128), (unsigned)jchunks), mhsk::k::TP_WARPS * 32, 0, c->XE.ptr, ld_e, c->src.ptr, m0, n0, c->XV.ptr, ld_v, c->item_a.ptr, dims + 1, lo_v,
                    (int64_t)probe_v * bki, (int64_t)mhsk::k::TP_CHUNK, -1, nullptr);
            }
            LAUNCH_CHECK();
            if (m0 && !lazy_v) {
                launch_pdl(c, mhsk::k::need_from_csr, csr_blocks, 256, 0, m0, in.ptr, in.vtx, in.dem, ealive,
                                                                         vnew_s, c->item_b.ptr, (const int32_t*)nullptr,
                                                                         (const int32_t*)nullptr);
                LAUNCH_CHECK();
            }
            c->st.kernel_launches += 2;
            if (lazy_v) {
                const int64_t width_v = fp4 ? ld_v * 2 : ld_v;
                const int jchunks = (int)std::max<int64_t>(1, (width_v + mhsk::k::TP_CHUNK - 1) / mhsk::k::TP_CHUNK);
                mark("v_operand");
                if (spec_ok) {   // the speculative probe's marks, candidates and lo
                    swap_probe_bufs(c);
                    set_last_geom(c, spec_geom);
                } else {
                    auto ev = gram_event();
                    CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                    // FP4: the probe only needs "degree > 0" (L = lo, or +inf for a
                    // vertex without edges), i.e. need > 0; exact degrees are counted
                    // below for the panels that get packed in full.  int8: exact
                    // degrees from the edge pack (the int8 probe uses d - lo).
                    launch_gram_fast<mhsk::PHASE_MD>(c, c->XV.ptr, rows_v, c->XV.ptr, rows_v, ld_v, gn,
                                                     c->tiles_v.ptr, (int32_t)c->tiles_v_host.size(), dims + 1,
                                                     fp4 ? c->vneed.ptr : c->vdeg.ptr, nullptr, nullptr, nullptr,
                                                     nullptr, nullptr, 0, nullptr, nullptr, fp4, lo_v,
                                                     c->pruned.ptr + 1, probe_v, /*passes=*/1, /*defer_verify=*/true);
                    CUDA_TRY(cudaEventRecord(ev.second, c->stream));
                }
                if (c->lg_count > 0) {
                    // candidates of unmarked tiles: counted from the CSR while the
                    // list is short (no operand rows needed); otherwise their panels
                    const bool vcsr = c->vcsr && c->lg_cand && m0 > 0;
                    if (vcsr) {
                        using namespace mhsk::k;
                        c->vc_keys.reserve(VCAND_TABLE);
                        c->vc_cnt.reserve(VCAND_TABLE);
                        c->vc_flag.reserve(std::max(gn, 1));
                        c->vc_deg.reserve(std::max(gn, 1));
                        c->vc_ok.reserve(3);
                        CUDA_TRY(cudaMemsetAsync(c->vc_keys.ptr, 0xFF, VCAND_TABLE * sizeof(unsigned long long), c->stream));
                        CUDA_TRY(cudaMemsetAsync(c->vc_cnt.ptr, 0, VCAND_TABLE * sizeof(int32_t), c->stream));
                        CUDA_TRY(cudaMemsetAsync(c->vc_flag.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                        CUDA_TRY(cudaMemsetAsync(c->vc_deg.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                        CUDA_TRY(cudaMemsetAsync(c->vc_ok.ptr, 0, 3 * sizeof(int32_t), c->stream));
                        const uint32_t vmask = (1u << c->vcand_table_log2) - 1u;
                        const int32_t vmax = std::min<int32_t>(c->vcand_max, (int32_t)(vmask + 1) / 2);
                        // candidate vertices also as an original-id map, tested in
                        // shared memory by vcand_count (no per-member gathers)
                        const bool vmap_ok = (int64_t)n0 <= MAP_SMEM_BITS;
                        const int32_t vwords = (n0 + 31) / 32;
                        if (vmap_ok) {
                            c->vc_bits.reserve(vwords);
                            CUDA_TRY(cudaMemsetAsync(c->vc_bits.ptr, 0, (size_t)vwords * 4, c->stream));
                        }
                        launch_pdl(c, vcand_prepare, c->sms * 2, 256, 0, c->cand.ptr, c->cand_count.ptr,
                                                                        c->cand_cap, c->needed.ptr,
                                                                        c->vc_flag.ptr, c->vc_keys.ptr, c->vc_ok.ptr,
                                                                        vmax, vmask, vmap_ok ? vids_s : nullptr,
                                                                        vmap_ok ? c->vc_bits.ptr : nullptr);
                        if (vmap_ok) {   // partner lists of the pairs (vcand_count's linear pair check)
                            c->vc_pcnt.reserve(std::max(gn, 1));
                            c->vc_pslot.reserve((size_t)std::max(gn, 1) * VC_PCAP);
                            CUDA_TRY(cudaMemsetAsync(c->vc_pcnt.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                            launch_pdl(c, vcand_partners, c->sms * 2, 256, 0, c->vc_ok.ptr, c->vc_keys.ptr, vmask,
                                       c->vc_pcnt.ptr, c->vc_pslot.ptr, c->vc_ok.ptr + 2);
                            c->st.kernel_launches += 1;
                        }
                        launch_pdl(c, vcand_gate, 1, 1, 0, c->vc_ok.ptr, std::max(64, gn / 16), 5e7, (double)gm,
                                                           mean_size, (double)gn, (int32_t)vmap_ok);
                        if (vmap_ok) {
                            // one wave of resident CTAs (the member loop keeps 16 KB per warp in flight)
                            int per_sm = 0;
                            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vcand_count<true>, VC_WARPS * 32,
                                                                                  (size_t)vwords * 4));
                            // edges with more than VC_LIST candidate members: deferred
                            // to vcand_count_heavy (pairs against the table)
                            c->vc_heavy.reserve(std::max(m0, 1) + 1);
                            CUDA_TRY(cudaMemsetAsync(c->vc_heavy.ptr + std::max(m0, 1), 0, sizeof(int32_t), c->stream));
                            int32_t* heavy_count = c->vc_heavy.ptr + std::max(m0, 1);
                            launch_pdl(c, vcand_count<true>, c->sms * std::max(per_sm, 1), VC_WARPS * 32, (size_t)vwords * 4, c->vc_ok.ptr, m0, in.ptr, in.vtx, ealive, vnew_s, c->vc_flag.ptr, c->vc_keys.ptr,
                                c->vc_cnt.ptr, c->vc_deg.ptr, vmask, c->vc_bits.ptr, n0, c->vc_heavy.ptr, heavy_count,
                                (const int32_t*)c->vc_pcnt.ptr, (const int32_t*)c->vc_pslot.ptr);
                            launch_pdl(c, vcand_count_heavy, c->sms, 256, (size_t)((gn + 31) / 32) * 4, c->vc_ok.ptr, c->vc_heavy.ptr,
                                heavy_count, in.ptr, in.vtx, vnew_s, c->vc_flag.ptr, c->vc_keys.ptr, c->vc_cnt.ptr, vmask, gn);
                            c->st.kernel_launches += 1;
                        } else
                            launch_pdl(c, vcand_count<false>, csr_blocks, VC_WARPS * 32, 0, c->vc_ok.ptr, m0, in.ptr, in.vtx, ealive, vnew_s, c->vc_flag.ptr, c->vc_keys.ptr,
                                c->vc_cnt.ptr, c->vc_deg.ptr, vmask, (const uint32_t*)nullptr, 0, (int32_t*)nullptr, (int32_t*)nullptr,
                                (const int32_t*)nullptr, (const int32_t*)nullptr);
                        launch_pdl(c, vcand_decide, c->sms * 2, 256, 0, c->vc_ok.ptr, c->cand.ptr, c->cand_count.ptr, c->cand_cap, c->needed.ptr,
                            c->vc_keys.ptr, c->vc_cnt.ptr, c->vc_deg.ptr, c->hits.ptr,
                            c->pruned.cap >= 3 ? c->pruned.ptr + 2 : nullptr, vmask);
                        LAUNCH_CHECK();
                        c->st.kernel_launches += 4;
                    }
                    // undecided panels -> full rows, candidates, then the full-K pass
                    CUDA_TRY(cudaMemsetAsync(c->panel_flags.ptr, 0, rows_v / 256 + 2, c->stream));
                    CUDA_TRY(cudaMemsetAsync(c->any_v.ptr, 0, sizeof(int32_t), c->stream));
                    launch_pdl(c, mhsk::k::needed_panels, c->sms * 2, 256, 0, c->needed.ptr, c->lg_pairs, c->lg_words, c->tiles_v.ptr, c->lg_begin, c->lg_count,
                        c->lg_stride, c->lg_cand ? c->cand.ptr : nullptr, c->cand_count.ptr,
                        c->cand_cap, c->panel_flags.ptr, pair_bn(fp4), c->any_v.ptr, nullptr,
                        vcsr ? c->vc_ok.ptr : nullptr);
                    LAUNCH_CHECK();
                    if (lazy_e) {   // full vertex panels read X_E columns of every row
                        launch_pdl(c, mhsk::k::flag_all_panels, std::max(1, (npanels_e + 255) / 256), 256, 0, c->any_v.ptr, c->state_e.ptr, npanels_e);
                        LAUNCH_CHECK();
                        c->st.kernel_launches += 1;
                        pack_flagged_edge_panels(nullptr);
                    }
                    if (fp4) CUDA_TRY(cudaMemsetAsync(c->vdeg.ptr, 0, (size_t)gn * sizeof(int32_t), c->stream));
                    launch_pdl(c, (fp4 ? mhsk::k::transpose_pack<true> : mhsk::k::transpose_pack<false>), dim3((unsigned)(rows_v / 128), (unsigned)jchunks), mhsk::k::TP_WARPS * 32, 0, c->XE.ptr, ld_e, c->src.ptr, m0, n0, c->XV.ptr, ld_v, fp4 ? c->vdeg.ptr : nullptr, dims + 1,
                        nullptr, 0, (int64_t)mhsk::k::TP_CHUNK, -1, c->panel_flags.ptr);
                    LAUNCH_CHECK();
                    launch_verify<mhsk::PHASE_MD>(c, c->XV.ptr, ld_v, dims + 1, fp4, c->vdeg.ptr, nullptr,
                                                  vcsr ? c->vc_ok.ptr : nullptr);
                    auto ev2 = gram_event();
                    CUDA_TRY(cudaEventRecord(ev2.first, c->stream));
                    launch_gram_fast<mhsk::PHASE_MD>(c, c->XV.ptr, rows_v, c->XV.ptr, rows_v, ld_v, gn,
                                                     c->tiles_v.ptr, (int32_t)c->tiles_v_host.size(), dims + 1,
                                                     c->vdeg.ptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                                     nullptr, nullptr, fp4, spec_ok ? c->lo_s.ptr : lo_v,
                                                     c->pruned.ptr + 1, probe_v, /*passes=*/2);
                    CUDA_TRY(cudaEventRecord(ev2.second, c->stream));
                    c->st.kernel_launches += 3;
                }
            } else if (full_round) {
                auto ev = gram_event();
                CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                launch_gram_fast<mhsk::PHASE_MD>(c, c->XV.ptr, rows_v, c->XV.ptr, rows_v, ld_v, gn,
                                                 c->tiles_v.ptr, (int32_t)c->tiles_v_host.size(), dims + 1,
                                                 c->item_a.ptr, nullptr, nullptr, nullptr, nullptr,
                                                 sparse ? c->mask_v.ptr : nullptr, sparse ? words_v : 0,
                                                 nullptr, vorder ? c->vids_p.ptr : nullptr, fp4, lo_v,
                                                 c->pruned.ptr + 1, probe_v);
                CUDA_TRY(cudaEventRecord(ev.second, c->stream));
            } else {
                // affected vertices: alive members of the edges this round deleted
                CUDA_TRY(cudaMemsetAsync(c->aff_flag.ptr, 0, n0, c->stream));
                if (m0) {
                    launch_pdl(c, mhsk::k::mark_affected_vertices, csr_blocks, 256, 0, m0, in.ptr, in.vtx, c->edel.ptr, valive, c->aff_flag.ptr);
                    LAUNCH_CHECK();
                }
                compact(c, c->aff_flag.ptr, n0, c->aff_scratch.ptr, c->aff_v_ids.ptr, dims + 7);
                launch_pdl(c, mhsk::k::gather_ids, (n_cur + 255) / 256, 256, 0, c->aff_v_ids.ptr, c->vnew.ptr, c->a_items.ptr, dims + 7);
                launch_pdl(c, mhsk::k::choose_phase_kernel, 1, 1, 0, dims + 7, dims + 1, dims + 8,
                                                                     probe_v > 0 && c->rect_rule == 0 ? probe_v : 1,
                                                                     probe_v > 0 && c->rect_rule == 0 ? 2 * kb_v : 2);
                const int64_t rows_a = round_up(n_cur / 2 + 1, 256);
                launch_pdl(c, mhsk::k::gather_rows, pack_blocks(c, rows_a), mhsk::k::PACK_WARPS * 32, 0, c->XV.ptr, ld_v, c->a_items.ptr, dims + 7, dims + 2, c->XA.ptr, dims + 9, fp4);
                LAUNCH_CHECK();
                rect_tiles(c, n_cur / 2 + 1, n_cur, fp4);
                c->st.kernel_launches += 5;
                auto ev = gram_event();
                CUDA_TRY(cudaEventRecord(ev.first, c->stream));
                launch_gram_fast<mhsk::PHASE_MD>(c, c->XV.ptr, rows_v, c->XV.ptr, rows_v, ld_v, n_cur,
                                                 c->tiles_v.ptr, (int32_t)c->tiles_v_host.size(), dims + 1,
                                                 c->item_a.ptr, nullptr, nullptr, nullptr, dims + 8, nullptr, 0,
                                                 nullptr, nullptr, fp4, lo_v, c->pruned.ptr + 1, probe_v);
                launch_gram_fast<mhsk::PHASE_MD, true>(c, c->XA.ptr, rows_a, c->XV.ptr, rows_v, ld_v, n_cur,
                                                       c->tiles_r.ptr, (int32_t)c->tiles_r_host.size(),
                                                       dims + 1, c->item_a.ptr, nullptr, c->a_items.ptr,
                                                       dims + 7, dims + 9, nullptr, 0, nullptr, nullptr, fp4);
                CUDA_TRY(cudaEventRecord(ev.second, c->stream));
            }
            allreduce_hits(c, n0);
            launch_pdl(c, mhsk::k::commit_phase<true>, (gn + 255) / 256, 256, 0, gn, c->hits.ptr, lazy_v ? c->vneed.ptr : c->item_b.ptr, vids_s, valive, nullptr, dims + 4,
                dims + 1, c->vdel.ptr);
            LAUNCH_CHECK();
            c->st.kernel_launches += 1;
            if (spec_ok) swap_probe_bufs(c);   // the edge phase's buffers back in place
            mark("vertex_done");
        }
        // ---- affected edges of the next round: alive edges that lost a vertex
        if (c->incremental && big && !sparse && m0) {
            if ((int64_t)n0 <= mhsk::k::MAP_SMEM_BITS) {   // deleted vertices as a shared-memory map
                const int32_t words = (n0 + 31) / 32;
                c->vdel_bits.reserve(words);
                launch_pdl(c, mhsk::k::bits_from_bytes, std::max(1, std::min((words + 7) / 8, c->sms * 4)), 256, 0, c->vdel.ptr, n0, c->vdel_bits.ptr);
                launch_pdl(c, mhsk::k::mark_affected_edges_map, c->sms * 2, 512, (size_t)words * 4, m0, n0, in.ptr, in.vtx, ealive, c->vdel_bits.ptr, c->aff_flag.ptr, dims + 4);
                c->st.kernel_launches += 1;
            } else {
                launch_pdl(c, mhsk::k::mark_affected_edges, csr_blocks, 256, 0, m0, in.ptr, in.vtx, ealive,
                                                                               c->vdel.ptr, c->aff_flag.ptr, dims + 4);
            }
            LAUNCH_CHECK();
            compact(c, c->aff_flag.ptr, m0, c->aff_scratch.ptr, c->aff_e_ids.ptr, dims + 5);
            c->st.kernel_launches += 1;
        }
        // ---- the round's single host read
        mark("affected");
        if (c->stage_alive) {   // (the final state once the loop stops: nothing runs after this read)
            if (n0) CUDA_TRY(cudaMemcpyAsync(c->alive_host, valive, n0, cudaMemcpyDeviceToHost, c->stream));
            if (m0) CUDA_TRY(cudaMemcpyAsync(c->alive_host + n0, ealive, m0, cudaMemcpyDeviceToHost, c->stream));
            c->alive_staged = true;
        }
        CUDA_TRY(cudaMemcpyAsync(c->dims_host, dims, 10 * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c->stream));
        if (lo_e)
            CUDA_TRY(cudaMemcpyAsync(c->pruned_host, c->pruned.ptr, 4 * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaEventRecord(c->ev_round, c->stream));
        c->round_ev_valid = true;
        ctx_sync(c);
        if (tracing) {
            fprintf(stderr, "[stream trace] round 1 (ms after call start):");
            for (auto& tv : trace) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, c->ev0, tv.second);
                fprintf(stderr, " %s %.3f", tv.first, ms);
                cudaEventDestroy(tv.second);
            }
            fprintf(stderr, "\n");
        }
        for (auto& ev : round_events) {   // this round's Gram time
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ev.first, ev.second) == cudaSuccess) c->st.ms_gram += ms;
        }
        (void)cudaGetLastError();
        const int32_t m_a = c->dims_host[0], n_a = c->dims_host[1], m_a2 = c->dims_host[2];
        const int32_t del_e = c->dims_host[3], del_v = c->dims_host[4];
        const int32_t aff_v = c->dims_host[7];
        const bool v_rect = !full_round && c->dims_host[9];
        // tiles stopped after the probe skipped KB - probe_kb of their k-blocks
        auto pruned_ops = [&](unsigned long long tiles, int32_t K, int32_t probe_kb) {
            const int32_t kb = std::max<int32_t>(1, (K + bki - 1) / bki);
            return (int64_t)tiles * (kb - probe_kb) * 2ll * 256 * pair_bn(fp4) * bki;
        };
        unsigned long long pruned_e = 0, pruned_v = 0;
        if (lo_e) {
            pruned_e = c->pruned_host[0] - pruned_seen[0];
            pruned_v = c->pruned_host[1] - pruned_seen[1] + (spec_ok ? c->pruned_host[3] : 0);
            if (spec_launched) c->st.spec_vertex = spec_ok ? 1 : 2;
            pruned_seen[0] = c->pruned_host[0];
            pruned_seen[1] = c->pruned_host[1];
            c->st.pruned_tiles += (int64_t)(pruned_e + pruned_v);
            c->st.verified_pairs = (int64_t)c->pruned_host[2];   // cumulative over the call
        }
        if (m_a && edge_mode) {
            if (edge_mode == 1) {
                c->st.gram_ops += (int64_t)m_a * (m_a + 1) * (int64_t)n_a;
                if (!sparse)
                    c->st.executed_ops += executed_ops_fast(c, tl_e, m_a, n_a, fp4) - pruned_ops(pruned_e, n_a, probe_e);
            } else {
                c->st.gram_ops += 2ll * aff_e * m_a * (int64_t)n_a;
                c->st.executed_ops += (int64_t)((aff_e + 255) / 256) * ((m_a + pair_bn(fp4) - 1) / pair_bn(fp4)) *
                                      2ll * 256 * pair_bn(fp4) *
                                      round_up(std::max<int32_t>(n_a, 1), fp4 ? 256 : 128) / c->world;
            }
            c->st.gram_launches += 1;
            c->st.fp4_gram_launches += fp4;
        }
        if (n_a) {
            if (v_rect) {
                c->st.gram_ops += 2ll * aff_v * n_a * (int64_t)m_a2;
                c->st.executed_ops += (int64_t)((aff_v + 255) / 256) * ((n_a + pair_bn(fp4) - 1) / pair_bn(fp4)) *
                                      2ll * 256 * pair_bn(fp4) *
                                      round_up(std::max<int32_t>(m_a2, 1), fp4 ? 256 : 128) / c->world;
            } else {
                c->st.gram_ops += (int64_t)n_a * (n_a + 1) * (int64_t)m_a2;
                if (!sparse)
                    c->st.executed_ops += executed_ops_fast(c, c->tiles_v_host, n_a, m_a2, fp4) - pruned_ops(pruned_v, m_a2, probe_v);
            }
            c->st.gram_launches += 1;
            c->st.fp4_gram_launches += fp4;
        }
        c->st.deleted_edges += del_e;
        c->st.deleted_vertices += del_v;
        n_cur = n_a - del_v;
        m_cur = m_a2;
        aff_e = (c->incremental && big && !sparse) ? c->dims_host[5] : -1;
        if (del_e == 0 && del_v == 0) break;
    }
    c->st.kernel_launches += c->st.gram_launches;
    if (sparse) {   // tensor work actually issued: k-blocks x 256 x 256 x 128 MACs x 2
        unsigned long long kb = 0;
        CUDA_TRY(cudaMemcpy(&kb, c->kblocks.ptr, sizeof(kb), cudaMemcpyDeviceToHost));
        c->st.executed_ops += (int64_t)kb * 2ll * 256 * 256 * 128;
    }
    for (auto& ev : gram_events) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    (void)cudaGetLastError();   // clear "not recorded" from skipped phases
    c->st.rounds = rounds;
}

bool fast_path(const mhsk_ctx* c) {
    return c->fast_loop && c->backend == MHSK_BACKEND_TC && c->gram_variant == 2;
}

// The fixpoint loop of par_kernelize (parallel.py:181-208) over a
// device-resident instance.  valive/ealive are set to 1 first.
// validated == false (fast path only): kernelize_fast validates, fused
// into round 1's edge pack when it can.
void kernelize_device(mhsk_ctx* c, const DevInstance& in, int32_t rule, int32_t max_rounds,
                      uint8_t* valive, uint8_t* ealive, bool validated) {
    if (fast_path(c)) {
        kernelize_fast(c, in, rule, max_rounds, valive, ealive, validated);
        return;
    }
    reserve_instance_state(c, in.n, in.m);
    if (in.n) CUDA_TRY(cudaMemsetAsync(valive, 1, in.n, c->stream));
    if (in.m) CUDA_TRY(cudaMemsetAsync(ealive, 1, in.m, c->stream));
    int64_t rounds = 0;
    for (;;) {
        if (max_rounds >= 0 && rounds >= max_rounds) break;
        ++rounds;
        CUDA_TRY(cudaMemsetAsync(c->counters.ptr, 0, 4 * sizeof(int32_t), c->stream));
        compact(c, valive, in.n, c->vnew.ptr, c->vids.ptr, c->counters.ptr + 0);
        compact(c, ealive, in.m, c->enew.ptr, c->eids.ptr, c->counters.ptr + 1);
        read_counters(c);
        const int32_t n_a = c->counters_host[0], m_a = c->counters_host[1];
        edge_phase(c, in, rule, m_a, n_a, ealive, nullptr);
        compact(c, ealive, in.m, c->enew.ptr, c->eids.ptr, c->counters.ptr + 1);
        read_counters(c);
        const int32_t del_e = c->counters_host[2];
        const int32_t m_a2 = c->counters_host[1];
        CUDA_TRY(cudaMemsetAsync(c->counters.ptr + 2, 0, sizeof(int32_t), c->stream));
        vertex_phase(c, in, n_a, m_a2, ealive, valive, nullptr);
        read_counters(c);
        const int32_t del_v = c->counters_host[2];
        c->st.deleted_edges += del_e;
        c->st.deleted_vertices += del_v;
        if (del_e == 0 && del_v == 0) break;
    }
    c->st.rounds = rounds;
}

// One FE pass (rules.py:138-181) on the device-resident alive state; returns
// (deleted edges, forced vertices, first infeasible edge + 1 or 0).
struct FeOutcome {
    int32_t deleted_edges, forced, infeasible_edge;
};

FeOutcome fe_pass_device(mhsk_ctx* c, const DevInstance& in, int32_t* dem, uint8_t* valive,
                         uint8_t* ealive) {
    c->xe_valid = false;
    c->fe_full.reserve(std::max<int32_t>(in.m, 1));
    c->fe_forced.reserve(std::max<int32_t>(in.n, 1));
    const int32_t big = 0x7FFFFFFF;
    CUDA_TRY(cudaMemsetAsync(c->counters.ptr, 0, 4 * sizeof(int32_t), c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->counters.ptr + 6, &big, sizeof(int32_t), cudaMemcpyHostToDevice,
                             c->stream));
    if (in.n) CUDA_TRY(cudaMemsetAsync(c->fe_forced.ptr, 0, in.n, c->stream));
    const int blocks = std::max(1, std::min<int32_t>((in.m + 7) / 8, c->sms * 16));
    if (in.m) {
        launch_pdl(c, mhsk::k::fe_mark, blocks, 256, 0, in.m, in.ptr, in.vtx, dem, valive, ealive,
                                                        c->fe_full.ptr, c->counters.ptr + 6);
        LAUNCH_CHECK();
        launch_pdl(c, mhsk::k::fe_force, blocks, 256, 0, in.m, in.ptr, in.vtx, valive, c->fe_full.ptr,
                                                         c->counters.ptr + 6, c->fe_forced.ptr);
        LAUNCH_CHECK();
        launch_pdl(c, mhsk::k::fe_apply_edges, blocks, 256, 0, in.m, in.ptr, in.vtx, dem, ealive, c->fe_full.ptr, c->fe_forced.ptr, c->counters.ptr + 6,
            c->counters.ptr + 2);
        LAUNCH_CHECK();
        c->st.kernel_launches += 3;
    }
    if (in.n) {
        launch_pdl(c, mhsk::k::fe_apply_vertices, (in.n + 255) / 256, 256, 0, in.n, c->fe_forced.ptr, valive, c->counters.ptr + 6, c->counters.ptr + 3);
        LAUNCH_CHECK();
        c->st.kernel_launches += 1;
    }
    CUDA_TRY(cudaMemcpyAsync(c->counters_host, c->counters.ptr, 8 * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, c->stream));
    ctx_sync(c);
    FeOutcome o;
    o.infeasible_edge = c->counters_host[6] == big ? 0 : c->counters_host[6];
    o.deleted_edges = o.infeasible_edge ? 0 : c->counters_host[2];
    o.forced = o.infeasible_edge ? 0 : c->counters_host[3];
    return o;
}

// The generic phase loop of run_pipeline (pipeline.py:130-161) on the device.
void pipeline_device(mhsk_ctx* c, const DevInstance& in, const int32_t* phases, int32_t nph,
                     bool loop, uint8_t* valive, uint8_t* ealive, mhsk_pipeline_result* res) {
    reserve_instance_state(c, in.n, in.m);
    if (in.n) CUDA_TRY(cudaMemsetAsync(valive, 1, in.n, c->stream));
    if (in.m) CUDA_TRY(cudaMemsetAsync(ealive, 1, in.m, c->stream));
    cudaEvent_t p0 = c->evg0, p1 = c->evg1;  // reused; Gram timing inside phases uses its own pair
    (void)p0;
    (void)p1;
    for (;;) {
        ++res->passes;
        int64_t deletions = 0;
        for (int32_t k = 0; k < nph; ++k) {
            const int32_t ph = phases[k];
            const double gram_before = c->st.ms_gram;
            cudaEvent_t e0, e1;
            CUDA_TRY(cudaEventCreate(&e0));
            CUDA_TRY(cudaEventCreate(&e1));
            CUDA_TRY(cudaEventRecord(e0, c->stream));
            int64_t dropped = 0;
            if (ph == MHSK_PHASE_FE) {
                const FeOutcome o = fe_pass_device(c, in, const_cast<int32_t*>(in.dem), valive, ealive);
                if (o.infeasible_edge) {
                    res->infeasible = 1;
                    res->infeasible_edge = o.infeasible_edge;
                } else {
                    res->deleted[MHSK_PHASE_FE] += o.deleted_edges;
                    res->forced_vertices += o.forced;
                    dropped = o.deleted_edges + o.forced;
                }
            } else {
                CUDA_TRY(cudaMemsetAsync(c->counters.ptr, 0, 4 * sizeof(int32_t), c->stream));
                compact(c, valive, in.n, c->vnew.ptr, c->vids.ptr, c->counters.ptr + 0);
                compact(c, ealive, in.m, c->enew.ptr, c->eids.ptr, c->counters.ptr + 1);
                read_counters(c);
                const int32_t n_a = c->counters_host[0], m_a = c->counters_host[1];
                if (ph == MHSK_PHASE_MD) vertex_phase(c, in, n_a, m_a, ealive, valive, nullptr);
                else edge_phase(c, in, ph == MHSK_PHASE_SE ? MHSK_RULE_SE : MHSK_RULE_DP, m_a, n_a,
                                ealive, nullptr);
                read_counters(c);
                dropped = c->counters_host[2];
                res->deleted[ph] += dropped;
                if (ph == MHSK_PHASE_MD) c->st.deleted_vertices += dropped;
                else c->st.deleted_edges += dropped;
            }
            CUDA_TRY(cudaEventRecord(e1, c->stream));
            CUDA_TRY(cudaEventSynchronize(e1));
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            (void)gram_before;
            res->ms_by_phase[ph] += ms;
            deletions += dropped;
            if (res->infeasible) break;
        }
        if (res->infeasible || !loop || deletions == 0) break;
    }
    c->st.rounds = res->passes;
}

}  // namespace

namespace {
int guarded(const std::function<void()>& body) {
    try {
        body();
        return MHSK_OK;
    } catch (const Failure& f) {
        return f.code;
    } catch (const std::exception& e) {
        set_error("exception: %s", e.what());
        return MHSK_CUDA_ERROR;
    }
}

int check_args(int32_t n, int32_t m, const void* ptr, const void* vtx, const void* dem) {
    if (n < 0 || m < 0) {
        set_error("negative instance dimensions");
        return MHSK_INVALID;
    }
    if (m > 0 && (!ptr || !dem)) {
        set_error("null CSR arrays");
        return MHSK_INVALID;
    }
    (void)vtx;
    return MHSK_OK;
}

// Copy a host CSR into the context's device buffers; returns the device view.
// stream = true (mhsk_kernelize on the fast path, one rank): the member
// array goes up in chunks of ~STREAM_CHUNK members on the copy stream, so
// that round 1's scan / pack / edge probe consume each chunk as it lands
// (kernelize_fast); the edge offsets and demands go first, on the compute
// stream.  Chunk bounds are multiples of 4 members (16-byte vector loads).

DevInstance upload(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* ptr, const int32_t* vtx,
                   const int32_t* dem, bool stream = false) {
    const int64_t nnz = m > 0 ? ptr[m] : 0;
    if (m > 0 && (ptr[0] != 0 || nnz < 0)) {
        set_error("edge_ptr must start at 0 and end at nnz >= 0");
        throw Failure{MHSK_INVALID};
    }
    c->edge_ptr.reserve(m + 1);
    c->edge_vtx.reserve(std::max<int64_t>(nnz, 1));
    c->demand.reserve(std::max<int32_t>(m, 1));
    if (m > 0) {
        CUDA_TRY(cudaMemcpyAsync(c->edge_ptr.ptr, ptr, (m + 1) * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(c->demand.ptr, dem, m * sizeof(int32_t), cudaMemcpyHostToDevice,
                                 c->stream));
        c->st.h2d_bytes += (m + 1) * sizeof(int64_t) + m * sizeof(int32_t);
    }
    const int chunks = nnz >= STREAM_MIN_MEMBERS
                           ? (int)std::min<int64_t>(std::min<int64_t>(STREAM_MAX_CHUNKS, c->stream_chunks), nnz / STREAM_CHUNK)
                           : 1;
    if (stream && c->stream_chunks > 1 && chunks >= 2) {
        bool fp4 = false;
        int64_t spec_rows = 0;
        const bool banded = plan_streamed_round1(c, n, m, nnz, fp4, spec_rows);
        // the speculative vertex probe (kernelize_fast) needs only the first
        // spec_rows edges: a small first chunk brings them, so it starts at
        // once and runs while the rest of the upload is in flight
        const int64_t k_spec = spec_rows > 0 && spec_rows < m ? std::min(nnz, (ptr[spec_rows] + 3) / 4 * 4) : 0;
        c->up_K.assign(1, 0);
        c->up_E.clear();
        // chunk bounds at nnz * sqrt(b / C): band b's probe work grows like
        // (its rows)^2, so equal-work bands need chunks that shrink -- the
        // last band (after the last chunk lands) is then 1/C of the probe
        for (int b = 1; b <= chunks; ++b) {
            const double frac = c->stream_sqrt ? std::sqrt((double)b / chunks) : (double)b / chunks;
            const int64_t k = b == chunks ? nnz
                                          : std::max<int64_t>(c->up_K.back(), (int64_t)((double)nnz * frac) / 4 * 4);
            if (b == 1 && k_spec > 0 && k_spec < k) c->up_K.push_back(k_spec);
            c->up_K.push_back(k);
        }
        for (size_t b = 1; b < c->up_K.size(); ++b)   // edges complete once members [0, k) have landed: ptr[e + 1] <= k
            c->up_E.push_back(b + 1 == c->up_K.size()
                                  ? m : (int32_t)(std::upper_bound(ptr + 1, ptr + m + 1, c->up_K[b]) - (ptr + 1)));
        const int nchunks = (int)c->up_E.size();
        // round 1 will stream: its band tile list goes up first, on the copy stream
        if (banded) {
            // the list depends only on (m, tile shape, raster, pairs, chunk
            // edges): rebuilt on the host only when those change
            std::vector<int32_t> key = {m, pair_bn(fp4), c->raster_gp, c->raster_gj, c->sms / 2};
            key.insert(key.end(), c->up_E.begin(), c->up_E.end());
            if (key != c->band_key) {
                if (c->band_ev) CUDA_TRY(cudaEventSynchronize(c->band_ev));   // host buffer reuse
                mhsk::make_band_tile_list(m, mhsk::TileShape{mhsk::tc2::BM, pair_bn(fp4), c->raster_gp, c->raster_gj},
                                          c->up_E, c->sms / 2, c->band_host, c->band_t);
                c->band_key = key;
            }
            c->tiles_e.reserve(std::max<size_t>(c->band_host.size(), 1));
            if (!c->band_ev) CUDA_TRY(cudaEventCreateWithFlags(&c->band_ev, cudaEventDisableTiming));
            c->band_M = m;
            c->band_fp4 = fp4;
            c->tiles_e_M = -1;   // tiles_e holds the band list now
        }
        while ((int)c->up_ev.size() < nchunks) {
            cudaEvent_t ev;
            CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            c->up_ev.push_back(ev);
        }
        for (size_t b = nchunks; b < c->up_ev.size(); ++b) cudaEventDestroy(c->up_ev[b]);
        c->up_ev.resize(nchunks);
        // the copy stream starts after everything already on the compute stream
        CUDA_TRY(cudaEventRecord(c->up_ev[0], c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->up_ev[0], 0));
        if (c->band_M == m) {
            CUDA_TRY(cudaMemcpyAsync(c->tiles_e.ptr, c->band_host.data(),
                                     c->band_host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                     c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->band_ev, c->copy_stream));
        }
        for (int b = 0; b < nchunks; ++b) {
            CUDA_TRY(cudaMemcpyAsync(c->edge_vtx.ptr + c->up_K[b], vtx + c->up_K[b],
                                     (c->up_K[b + 1] - c->up_K[b]) * sizeof(int32_t), cudaMemcpyHostToDevice,
                                     c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->up_ev[b], c->copy_stream));
        }
        c->up_pending = true;
        c->st.h2d_bytes += nnz * sizeof(int32_t);
    } else if (nnz > 0 && c->world > 1 && c->allreduce &&
               (c->shard_upload == 2 || (c->shard_upload == 1 && nnz >= STREAM_MIN_MEMBERS))) {
        // one slice per rank over its own PCIe link, the rest zero; the sum of
        // the ranks' buffers is the array (ids >= 0 never meet a nonzero
        // partner), moved over NVLink by the all-reduce hook
        const int64_t per = (nnz + c->world - 1) / c->world;
        const int64_t lo = std::min(nnz, per * c->rank), hi = std::min(nnz, lo + per);
        if (lo > 0) CUDA_TRY(cudaMemsetAsync(c->edge_vtx.ptr, 0, lo * sizeof(int32_t), c->stream));
        if (hi < nnz) CUDA_TRY(cudaMemsetAsync(c->edge_vtx.ptr + hi, 0, (nnz - hi) * sizeof(int32_t), c->stream));
        if (hi > lo)
            CUDA_TRY(cudaMemcpyAsync(c->edge_vtx.ptr + lo, vtx + lo, (hi - lo) * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, c->stream));
        if (c->allreduce(c->edge_vtx.ptr, nnz, (void*)c->stream, c->allreduce_user) != 0) {
            set_error("allreduce callback failed");
            throw Failure{MHSK_CUDA_ERROR};
        }
        c->st.h2d_bytes += (hi - lo) * sizeof(int32_t);
    } else if (nnz > 0) {
        CUDA_TRY(cudaMemcpyAsync(c->edge_vtx.ptr, vtx, nnz * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, c->stream));
        c->st.h2d_bytes += nnz * sizeof(int32_t);
    }
    if (m > 0) {   // nnz is known on the host: kernelize_fast needs no read-back
        *c->nnz_host = nnz;
        c->nnz_src = c->edge_ptr.ptr;
    }
    return DevInstance{n, m, c->edge_ptr.ptr, c->edge_vtx.ptr, c->demand.ptr};
}

void begin_call(mhsk_ctx* c) {
    if (c->up_pending) {   // a failed call's streamed upload: let it land first
        CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
        c->up_pending = false;
    }
    if (c->band_M >= 0) {   // the band list is valid for one call only
        CUDA_TRY(cudaEventSynchronize(c->band_ev));
        c->band_M = -1;
    }
    c->st = mhsk_stats{};
    c->stage_alive = false;   // (set by mhsk_kernelize for its own call only)
    c->round_ev_valid = false;
    c->nnz_src = nullptr;
    c->xe_valid = false;
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
}

void end_call(mhsk_ctx* c, mhsk_stats* out) {
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->round_ev_valid ? c->ev_round : c->ev1));
    c->st.ms_total = ms;
    c->st.ms_pack = std::max(0.0, c->st.ms_total - c->st.ms_gram);
    if (out) *out = c->st;
}

}  // namespace

extern "C" {

int mhsk_abi_version(void) { return MHSK_ABI_VERSION; }

const char* mhsk_last_error(void) { return g_last_error.c_str(); }

int mhsk_create(int device, mhsk_ctx** out) {
    if (!out) {
        set_error("null output pointer");
        return MHSK_INVALID;
    }
    *out = nullptr;
    mhsk_ctx* c = new mhsk_ctx();
    c->device = device;
    int rc = guarded([&] {
        CUDA_TRY(cudaSetDevice(device));
        int major = 0, minor = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major != 10 || minor != 0) {
            set_error("libmhsk is built for sm_100a (B200); device %d is sm_%d%d", device, major,
                      minor);
            throw Failure{MHSK_CUDA_ERROR};
        }
        CUDA_TRY(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        if (const char* r = getenv("MHSK_RASTER")) {
            int gp = 0, gj = 0;
            if (sscanf(r, "%d,%d", &gp, &gj) == 2 && gp > 0 && gj > 0) {
                c->raster_gp = gp;
                c->raster_gj = gj;
            }
        }
        if (const char* g = getenv("MHSK_GRAM")) c->gram_variant = atoi(g) == 1 ? 1 : 2;
        if (const char* t = getenv("MHSK_THROTTLE")) {
            int lc = 0, sl = 0;
            if (sscanf(t, "%d,%d", &lc, &sl) == 2 && lc >= 0 && lc < 16 && sl >= 0) {
                c->throttle_chunk_log2 = lc;
                c->throttle_slack = sl;
            }
        }
        CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreate(&c->ev0));
        CUDA_TRY(cudaEventCreate(&c->ev1));
        CUDA_TRY(cudaEventCreate(&c->evg0));
        CUDA_TRY(cudaEventCreate(&c->evg1));
        CUDA_TRY(cudaMallocHost(&c->counters_host, 8 * sizeof(int32_t)));
        CUDA_TRY(cudaMallocHost(&c->nnz_host, sizeof(int64_t)));
        CUDA_TRY(cudaMallocHost(&c->desc_host, 2 * sizeof(unsigned long long)));
        CUDA_TRY(cudaEventCreateWithFlags(&c->val_ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->edge_ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreate(&c->ev_round));
        CUDA_TRY(cudaMallocHost(&c->dims_host, 16 * sizeof(int32_t)));
        CUDA_TRY(cudaMallocHost(&c->pruned_host, 4 * sizeof(unsigned long long)));
        ensure_gram_attrs();
        if (const char* f = getenv("MHSK_FAST_LOOP")) c->fast_loop = atoi(f) != 0;
        if (const char* f = getenv("MHSK_INCREMENTAL")) c->incremental = atoi(f) != 0;
        if (const char* f = getenv("MHSK_SPARSE")) c->sparse = std::max(-1, std::min(2, atoi(f)));
        if (const char* f = getenv("MHSK_FP4")) c->fp4 = atoi(f) != 0;
        if (const char* f = getenv("MHSK_PROBE")) c->probe = atoi(f) != 0;
        if (const char* f = getenv("MHSK_VERIFY")) c->verify = atoi(f) != 0;
        if (const char* f = getenv("MHSK_LAZY")) c->lazy = atoi(f) != 0;
        if (const char* f = getenv("MHSK_LAZY_E")) c->lazy_e = atoi(f) != 0;
        if (const char* f = getenv("MHSK_VCSR")) c->vcsr = atoi(f) != 0;
        if (const char* f = getenv("MHSK_PROBE_ENTRIES")) c->probe_entries = std::max(0, atoi(f));
        if (const char* f = getenv("MHSK_PROBE_ENTRIES_E")) c->probe_entries_e = std::max(0, atoi(f));
        if (const char* f = getenv("MHSK_GRAM_TIMING")) c->gram_timing = atoi(f) != 0;
        if (const char* f = getenv("MHSK_GRAM_TUNE")) c->gram_tune = atoi(f);
        c->counters.reserve(8);
    });
    if (rc != MHSK_OK) {
        mhsk_destroy(c);
        return rc;
    }
    *out = c;
    return MHSK_OK;
}

void mhsk_destroy(mhsk_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->edge_ptr.release();
    c->edge_vtx.release();
    c->demand.release();
    c->dem_work.release();
    c->fe_full.release();
    c->fe_forced.release();
    c->valive.release();
    c->ealive.release();
    c->keep.release();
    c->vnew.release();
    c->enew.release();
    c->vids.release();
    c->eids.release();
    c->scan_tmp.release();
    c->item_a.release();
    c->item_b.release();
    c->hits.release();
    c->X.release();
    c->gen_ptr.release();
    c->gen_vtx.release();
    c->gen_dem.release();
    c->gen_attempt.release();
    c->XE.release();
    c->XV.release();
    c->keep_e.release();
    c->src.release();
    c->scratch.release();
    c->tiles.release();
    c->progress.release();
    c->counters.release();
    if (c->counters_host) cudaFreeHost(c->counters_host);
    if (c->nnz_host) cudaFreeHost(c->nnz_host);
    if (c->desc_host) cudaFreeHost(c->desc_host);
    if (c->dims_host) cudaFreeHost(c->dims_host);
    if (c->pruned_host) cudaFreeHost(c->pruned_host);
    if (c->alive_host) cudaFreeHost(c->alive_host);
    c->dims.release();
    c->XA.release();
    c->edel.release();
    c->vdel.release();
    c->aff_flag.release();
    c->aff_e_ids.release();
    c->aff_v_ids.release();
    c->a_items.release();
    c->aff_scratch.release();
    c->tiles_r.release();
    c->perm.release();
    c->sort_keys.release();
    c->sort_keys_out.release();
    c->sort_vals.release();
    c->sort_temp.release();
    c->mask_e.release();
    c->mask_v.release();
    c->vlabel.release();
    c->elabel.release();
    c->vperm.release();
    c->vpos.release();
    c->vids_p.release();
    c->vnew_p.release();
    c->cp_status.release();
    c->item_lo.release();
    c->pruned.release();
    c->needed.release();
    c->timing.release();
    c->kblocks.release();
    c->tiles_e.release();
    c->tiles_v.release();
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->evg0) cudaEventDestroy(c->evg0);
    if (c->evg1) cudaEventDestroy(c->evg1);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    for (cudaEvent_t ev : c->up_ev) cudaEventDestroy(ev);
    if (c->band_ev) cudaEventDestroy(c->band_ev);
    if (c->val_ev) cudaEventDestroy(c->val_ev);
    if (c->edge_ev) cudaEventDestroy(c->edge_ev);
    if (c->ev_round) cudaEventDestroy(c->ev_round);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int mhsk_device_sms(mhsk_ctx* c) { return c ? c->sms : 0; }

int64_t mhsk_tile_list(int32_t M, int32_t tile_rows, int32_t gp, int32_t gj, uint32_t* out,
                       int64_t cap) {
    return mhsk_tile_list_cols(M, tile_rows, 256, gp, gj, out, cap);
}

int64_t mhsk_tile_list_cols(int32_t M, int32_t tile_rows, int32_t tile_cols, int32_t gp, int32_t gj,
                            uint32_t* out, int64_t cap) {
    if (M < 0 || gp <= 0 || gj <= 0 || (tile_rows != 128 && tile_rows != 256) ||
        (tile_cols != 256 && tile_cols != mhsk::tc2::BN_FP4)) {
        set_error("invalid tile-list arguments");
        return -1;
    }
    std::vector<uint32_t> v;
    mhsk::make_tile_list(M, mhsk::TileShape{tile_rows, tile_cols, gp, gj}, v);
    if (out) std::copy(v.begin(), v.begin() + std::min<int64_t>(cap, (int64_t)v.size()), out);
    return (int64_t)v.size();
}

int mhsk_set_backend(mhsk_ctx* c, int backend) {
    if (!c || (backend != MHSK_BACKEND_TC && backend != MHSK_BACKEND_SIMT &&
               backend != MHSK_BACKEND_TC1)) {
        set_error("unknown backend %d", backend);
        return MHSK_INVALID;
    }
    c->backend = backend == MHSK_BACKEND_SIMT ? MHSK_BACKEND_SIMT : MHSK_BACKEND_TC;
    if (backend == MHSK_BACKEND_TC1) c->gram_variant = 1;
    else if (backend == MHSK_BACKEND_TC) c->gram_variant = 2;
    return MHSK_OK;
}

int mhsk_set_option(mhsk_ctx* c, const char* key, int64_t value) {
    if (!c || !key) return MHSK_INVALID;
    const std::string k(key);
    if (k == "incremental") c->incremental = value != 0;
    else if (k == "fast_loop") c->fast_loop = value != 0;
    else if (k == "throttle_slack" && value >= 0) c->throttle_slack = (int32_t)value;
    else if (k == "throttle_chunk_log2" && value >= 0 && value < 16) c->throttle_chunk_log2 = (int32_t)value;
    else if (k == "sparse" && value >= -1 && value <= 2) c->sparse = (int)value;
    else if (k == "fp4" && (value == 0 || value == 1)) c->fp4 = value != 0;
    else if (k == "probe" && (value == 0 || value == 1)) c->probe = value != 0;
    else if (k == "verify" && (value == 0 || value == 1)) c->verify = value != 0;
    else if (k == "lazy" && (value == 0 || value == 1)) c->lazy = value != 0;
    else if (k == "lazy_e" && (value == 0 || value == 1)) c->lazy_e = value != 0;
    else if (k == "vcsr" && (value == 0 || value == 1)) c->vcsr = value != 0;
    else if (k == "probe_entries" && value >= 0 && value < (1 << 20)) c->probe_entries = (int32_t)value;
    else if (k == "probe_entries_e" && value >= 0 && value < (1 << 20)) c->probe_entries_e = (int32_t)value;
    else if (k == "cand_cap" && value >= 0 && value <= mhsk::tc2::CAND_CAP) c->cand_cap = (int32_t)value;
    else if (k == "stream_chunks" && value >= 0 && value <= STREAM_MAX_CHUNKS) c->stream_chunks = (int32_t)value;
    else if (k == "stream_sqrt" && (value == 0 || value == 1)) c->stream_sqrt = value != 0;
    else if (k == "rect_rule" && (value == 0 || value == 1)) c->rect_rule = (int32_t)value;
    else if (k == "spec_vertex" && (value == 0 || value == 1)) c->spec_v = value != 0;
    else if (k == "pdl" && (value == 0 || value == 1)) c->pdl = value != 0;
    else if (k == "shard_upload" && value >= 0 && value <= 2) c->shard_upload = (int32_t)value;
    else if (k == "vcand_max" && value >= 0 && value <= mhsk::k::VCAND_MAX) c->vcand_max = (int32_t)value;
    else if (k == "vcand_table_log2" && value >= 1 && value <= mhsk::k::VCAND_TABLE_LOG2)
        c->vcand_table_log2 = (int32_t)value;
    else if (k == "raster_gp" && value > 0) { c->raster_gp = (int32_t)value; c->tiles_for_M = c->tiles_e_M = c->tiles_v_M = -1; }
    else if (k == "raster_gj" && value > 0) { c->raster_gj = (int32_t)value; c->tiles_for_M = c->tiles_e_M = c->tiles_v_M = -1; }
    else {
        set_error("unknown option %s=%lld", key, (long long)value);
        return MHSK_INVALID;
    }
    return MHSK_OK;
}

int mhsk_set_shard(mhsk_ctx* c, int rank, int world, mhsk_allreduce_fn fn, void* user) {
    if (!c || world < 1 || rank < 0 || rank >= world || (world > 1 && !fn)) {
        set_error("invalid shard spec rank=%d world=%d", rank, world);
        return MHSK_INVALID;
    }
    c->rank = rank;
    c->world = world;
    c->allreduce = fn;
    c->allreduce_user = user;
    return MHSK_OK;
}

int mhsk_kernelize_device(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* d_edge_ptr,
                          const int32_t* d_edge_vtx, const int32_t* d_demand, int32_t rule,
                          int32_t max_rounds, uint8_t* d_vertex_alive, uint8_t* d_edge_alive,
                          mhsk_stats* stats) {
    if (!c) return MHSK_INVALID;
    if (rule != MHSK_RULE_DP && rule != MHSK_RULE_SE) {
        set_error("unknown edge rule %d", rule);
        return MHSK_INVALID;
    }
    int rc = check_args(n, m, d_edge_ptr, d_edge_vtx, d_demand);
    if (rc) return rc;
    int vrc = MHSK_OK;
    rc = guarded([&] {
        begin_call(c);
        reserve_instance_state(c, n, m);
        DevInstance in{n, m, d_edge_ptr, d_edge_vtx, d_demand};
        const bool deferred = fast_path(c);   // validated inside, fused with round 1
        if (!deferred) {
            vrc = validate(c, in);
            if (vrc != MHSK_OK) return;
        }
        kernelize_device(c, in, rule, max_rounds, d_vertex_alive, d_edge_alive, !deferred);
        end_call(c, stats);
    });
    return rc != MHSK_OK ? rc : vrc;
}

int mhsk_kernelize(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* edge_ptr,
                   const int32_t* edge_vtx, const int32_t* demand, int32_t rule,
                   int32_t max_rounds, uint8_t* vertex_alive_out, uint8_t* edge_alive_out,
                   mhsk_stats* stats) {
    if (!c) return MHSK_INVALID;
    if (rule != MHSK_RULE_DP && rule != MHSK_RULE_SE) {
        set_error("unknown edge rule %d", rule);
        return MHSK_INVALID;
    }
    int rc = check_args(n, m, edge_ptr, edge_vtx, demand);
    if (rc) return rc;
    int vrc = MHSK_OK;
    rc = guarded([&] {
        if ((int64_t)n + m > c->alive_host_cap) {   // pinned result staging, before any stream work
            if (c->alive_host) CUDA_TRY(cudaFreeHost(c->alive_host));
            c->alive_host = nullptr;
            c->alive_host_cap = 0;
            CUDA_TRY(cudaMallocHost(&c->alive_host, (size_t)n + m));
            c->alive_host_cap = (int64_t)n + m;
        }
        begin_call(c);
        reserve_instance_state(c, n, m);
        const bool deferred = fast_path(c);   // validated inside, fused with round 1
        DevInstance in = upload(c, n, m, edge_ptr, edge_vtx, demand, deferred && c->world == 1);
        if (!deferred) {
            vrc = validate(c, in);
            if (vrc != MHSK_OK) return;
        }
        c->valive.reserve(std::max<int32_t>(n, 1));
        c->ealive.reserve(std::max<int32_t>(m, 1));
        c->stage_alive = deferred;
        c->alive_staged = false;
        kernelize_device(c, in, rule, max_rounds, c->valive.ptr, c->ealive.ptr, !deferred);
        c->stage_alive = false;
        c->st.d2h_bytes += n + m;
        if (c->alive_staged) {   // already on the host (pinned) with the last round's read
            end_call(c, stats);
            if (n) std::memcpy(vertex_alive_out, c->alive_host, n);
            if (m) std::memcpy(edge_alive_out, c->alive_host + n, m);
            return;
        }
        c->round_ev_valid = false;   // the result copies below are part of the call
        if (n) CUDA_TRY(cudaMemcpyAsync(vertex_alive_out, c->valive.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        if (m) CUDA_TRY(cudaMemcpyAsync(edge_alive_out, c->ealive.ptr, m, cudaMemcpyDeviceToHost, c->stream));
        end_call(c, stats);
    });
    return rc != MHSK_OK ? rc : vrc;
}

static int single_phase(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* edge_ptr,
                        const int32_t* edge_vtx, const int32_t* demand, int32_t rule, bool vertex,
                        uint8_t* keep_out) {
    int rc = check_args(n, m, edge_ptr, edge_vtx, demand);
    if (rc) return rc;
    int vrc = MHSK_OK;
    rc = guarded([&] {
        begin_call(c);
        reserve_instance_state(c, n, m);
        DevInstance in = upload(c, n, m, edge_ptr, edge_vtx, demand);
        // demand <= size is not required for a single phase (parallel.py:80-161
        // does not validate feasibility); only the CSR shape is checked.
        vrc = validate(c, in);
        if (vrc == MHSK_INFEASIBLE) vrc = MHSK_OK;
        if (vrc != MHSK_OK) return;
        c->valive.reserve(std::max<int32_t>(n, 1));
        c->ealive.reserve(std::max<int32_t>(m, 1));
        if (n) CUDA_TRY(cudaMemsetAsync(c->valive.ptr, 1, n, c->stream));
        if (m) CUDA_TRY(cudaMemsetAsync(c->ealive.ptr, 1, m, c->stream));
        CUDA_TRY(cudaMemsetAsync(c->counters.ptr, 0, 4 * sizeof(int32_t), c->stream));
        compact(c, c->valive.ptr, n, c->vnew.ptr, c->vids.ptr, c->counters.ptr + 0);
        compact(c, c->ealive.ptr, m, c->enew.ptr, c->eids.ptr, c->counters.ptr + 1);
        const int32_t items = vertex ? n : m;
        c->keep.reserve(std::max<int32_t>(items, 1));
        if (vertex) vertex_phase(c, in, n, m, c->ealive.ptr, nullptr, c->keep.ptr);
        else edge_phase(c, in, rule, m, n, nullptr, c->keep.ptr);
        if (items) {
            CUDA_TRY(cudaMemcpyAsync(keep_out, c->keep.ptr, items, cudaMemcpyDeviceToHost, c->stream));
            c->st.d2h_bytes += items;
        }
        end_call(c, nullptr);
    });
    return rc != MHSK_OK ? rc : vrc;
}

int mhsk_reduce_edges(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* edge_ptr,
                      const int32_t* edge_vtx, const int32_t* demand, int32_t rule,
                      uint8_t* keep_out) {
    if (!c) return MHSK_INVALID;
    if (rule != MHSK_RULE_DP && rule != MHSK_RULE_SE) {
        set_error("unknown edge rule %d", rule);
        return MHSK_INVALID;
    }
    return single_phase(c, n, m, edge_ptr, edge_vtx, demand, rule, false, keep_out);
}

int mhsk_reduce_vertices(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* edge_ptr,
                         const int32_t* edge_vtx, const int32_t* demand, uint8_t* keep_out) {
    if (!c) return MHSK_INVALID;
    return single_phase(c, n, m, edge_ptr, edge_vtx, demand, MHSK_RULE_DP, true, keep_out);
}

int mhsk_generate_random(mhsk_ctx* c, int32_t n, int32_t m, double p, int32_t alpha,
                         uint64_t seed, int64_t* nnz_out) {
    if (!c || n < 0 || m < 0 || !(p > 0.0 && p <= 1.0) || alpha < 1 || (m > 0 && n == 0)) {
        set_error("invalid generator arguments (n=%d m=%d p=%g alpha=%d)", n, m, p, alpha);
        return MHSK_INVALID;
    }
    return guarded([&] {
        CUDA_TRY(cudaSetDevice(c->device));
        const double t = p * 4294967296.0;
        const uint64_t thr = t >= 4294967296.0 ? 4294967296ull : (uint64_t)t;
        c->gen_ptr.reserve(m + 1);
        c->gen_attempt.reserve(std::max<int32_t>(m, 1));
        c->gen_dem.reserve(std::max<int32_t>(m, 1));
        CUDA_TRY(cudaMemsetAsync(c->gen_ptr.ptr, 0, sizeof(int64_t), c->stream));
        const int blocks = std::max(1, std::min<int32_t>((m + 7) / 8, c->sms * 16));
        if (m) {
            launch_pdl(c, mhsk::gen::gen_count, blocks, 256, 0, n, m, seed, thr, c->gen_ptr.ptr,
                                                               c->gen_attempt.ptr);
            LAUNCH_CHECK();
            launch_pdl(c, mhsk::gen::scan_i64, 1, 1024, 0, c->gen_ptr.ptr + 1, m);
            LAUNCH_CHECK();
        }
        int64_t nnz = 0;
        CUDA_TRY(cudaMemcpyAsync(&nnz, c->gen_ptr.ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                 c->stream));
        ctx_sync(c);
        c->gen_vtx.reserve(std::max<int64_t>(nnz, 1));
        if (m) {
            launch_pdl(c, mhsk::gen::gen_fill, blocks, 256, 0, n, m, seed, thr, alpha, c->gen_ptr.ptr,
                                                              c->gen_attempt.ptr, c->gen_vtx.ptr,
                                                              c->gen_dem.ptr);
            LAUNCH_CHECK();
        }
        ctx_sync(c);
        c->gen_n = n;
        c->gen_m = m;
        c->gen_nnz = nnz;
        if (nnz_out) *nnz_out = nnz;
    });
}

int64_t mhsk_generate_random_host(int32_t n, int32_t m, double p, int32_t alpha, uint64_t seed,
                                  int64_t* edge_ptr, int32_t* edge_vtx, int64_t vtx_capacity,
                                  int32_t* demand, int32_t* attempt) {
    if (n < 0 || m < 0 || !(p > 0.0 && p <= 1.0) || alpha < 1 || (m > 0 && n == 0) || !edge_ptr ||
        (m > 0 && !attempt)) {
        set_error("invalid generator arguments");
        return -1;
    }
    const double t = p * 4294967296.0;
    const uint64_t thr = t >= 4294967296.0 ? 4294967296ull : (uint64_t)t;
    using mhsk::gen::draw;
    using mhsk::gen::RETRIES;
    if (!edge_vtx) {  // pass 1: counts -> edge_ptr, attempts
        edge_ptr[0] = 0;
#pragma omp parallel for schedule(dynamic, 64)
        for (int32_t e = 0; e < m; ++e) {
            int r = 0;
            int64_t cnt = 0;
            for (; r < RETRIES; ++r) {
                cnt = 0;
                for (int32_t v = 0; v < n; ++v) cnt += draw(seed, e, v, r, thr);
                if (cnt) break;
            }
            edge_ptr[e + 1] = cnt ? cnt : 1;
            attempt[e] = r;
        }
        for (int32_t e = 0; e < m; ++e) edge_ptr[e + 1] += edge_ptr[e];
        return m ? edge_ptr[m] : 0;
    }
    if (m && vtx_capacity < edge_ptr[m]) {
        set_error("vtx buffer too small");
        return -1;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int32_t e = 0; e < m; ++e) {
        int64_t pos = edge_ptr[e];
        if (attempt[e] == RETRIES) {
            edge_vtx[pos] = (int32_t)(mhsk::gen::mix64(seed, (uint64_t)e, 0xFFFFFFFFull, RETRIES) % (uint64_t)n);
        } else {
            for (int32_t v = 0; v < n; ++v)
                if (draw(seed, e, v, attempt[e], thr)) edge_vtx[pos++] = v;
        }
        const int64_t sz = edge_ptr[e + 1] - edge_ptr[e];
        demand[e] = (int32_t)(sz < alpha ? sz : alpha);
    }
    return m ? edge_ptr[m] : 0;
}

int mhsk_generated_device(mhsk_ctx* c, const int64_t** edge_ptr, const int32_t** edge_vtx,
                          const int32_t** demand) {
    if (!c || c->gen_m < 0) {
        set_error("no generated instance in this context");
        return MHSK_INVALID;
    }
    if (edge_ptr) *edge_ptr = c->gen_ptr.ptr;
    if (edge_vtx) *edge_vtx = c->gen_vtx.ptr;
    if (demand) *demand = c->gen_dem.ptr;
    return MHSK_OK;
}

int mhsk_generated_copy(mhsk_ctx* c, int64_t* edge_ptr, int32_t* edge_vtx, int32_t* demand) {
    if (!c || c->gen_m < 0) {
        set_error("no generated instance in this context");
        return MHSK_INVALID;
    }
    return guarded([&] {
        CUDA_TRY(cudaMemcpyAsync(edge_ptr, c->gen_ptr.ptr, (c->gen_m + 1) * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, c->stream));
        if (c->gen_nnz)
            CUDA_TRY(cudaMemcpyAsync(edge_vtx, c->gen_vtx.ptr, c->gen_nnz * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, c->stream));
        if (c->gen_m)
            CUDA_TRY(cudaMemcpyAsync(demand, c->gen_dem.ptr, c->gen_m * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, c->stream));
        ctx_sync(c);
    });
}

int mhsk_run_pipeline(mhsk_ctx* c, int32_t n, int32_t m, const int64_t* edge_ptr,
                      const int32_t* edge_vtx, const int32_t* demand, const int32_t* phases,
                      int32_t n_phases, int32_t loop, uint8_t* vertex_alive_out,
                      uint8_t* edge_alive_out, int32_t* demand_out,
                      mhsk_pipeline_result* result, mhsk_stats* stats) {
    if (!c || !result || !phases || n_phases <= 0) {
        set_error("invalid pipeline arguments");
        return MHSK_INVALID;
    }
    for (int32_t k = 0; k < n_phases; ++k) {
        if (phases[k] < MHSK_PHASE_FE || phases[k] > MHSK_PHASE_MD) {
            set_error("unknown phase code %d", phases[k]);
            return MHSK_INVALID;
        }
    }
    int rc = check_args(n, m, edge_ptr, edge_vtx, demand);
    if (rc) return rc;
    *result = mhsk_pipeline_result{};
    int vrc = MHSK_OK;
    rc = guarded([&] {
        begin_call(c);
        reserve_instance_state(c, n, m);
        DevInstance in = upload(c, n, m, edge_ptr, edge_vtx, demand);
        vrc = validate(c, in);
        if (vrc != MHSK_OK) return;
        c->dem_work.reserve(std::max<int32_t>(m, 1));
        if (m) CUDA_TRY(cudaMemcpyAsync(c->dem_work.ptr, in.dem, m * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, c->stream));
        in.dem = c->dem_work.ptr;
        c->valive.reserve(std::max<int32_t>(n, 1));
        c->ealive.reserve(std::max<int32_t>(m, 1));
        pipeline_device(c, in, phases, n_phases, loop != 0, c->valive.ptr, c->ealive.ptr, result);
        if (n) CUDA_TRY(cudaMemcpyAsync(vertex_alive_out, c->valive.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        if (m) {
            CUDA_TRY(cudaMemcpyAsync(edge_alive_out, c->ealive.ptr, m, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaMemcpyAsync(demand_out, c->dem_work.ptr, m * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, c->stream));
        }
        c->st.d2h_bytes += n + 5ll * m;
        end_call(c, stats);
    });
    return rc != MHSK_OK ? rc : vrc;
}

}  // extern "C"
