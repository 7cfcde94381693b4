/*
 * mhsk.h -- C ABI of libmhsk.so, the B200 kernelization engine.
 *
 * Drop-in boundary for the reference's data-parallel engine
 * (reference pkg/src/mhskernel/parallel.py).  The reference has no FFI
 * layer: its engines are Python functions selected by name
 * (pipeline.py:30,117-121).  These entry points are what the Python host
 * package binds through ctypes (paper_2109_06042_b200/_native.py; a
 * maintainer's binding for the reference is in INTEGRATION.md):
 *
 *   mhsk_kernelize        replaces par_kernelize         parallel.py:164-214
 *   mhsk_reduce_edges     replaces par_reduce_edges      parallel.py:80-116
 *   mhsk_reduce_vertices  replaces par_reduce_vertices   parallel.py:119-161
 *   mhsk_run_pipeline     replaces run_pipeline's phase loop pipeline.py:130-171
 *                         (+ fe_pass, rules.py:138-181)
 *
 * Instances cross the boundary as CSR: edge e's vertices are
 * edge_vtx[edge_ptr[e] .. edge_ptr[e+1]), 0-based, strictly increasing
 * (the reference Hypergraph's sorted 1-based tuples, instance.py:32-61);
 * demand[e] >= 1.  Plain pointers and sizes only; no torch types.
 *
 * Threading: a context is not thread-safe (one per host thread).  Calls are
 * blocking; results are complete on return.  Errors: the return code, plus a
 * thread-local message from mhsk_last_error().
 */
#ifndef MHSK_H
#define MHSK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MHSK_ABI_VERSION 2

/* return codes */
#define MHSK_OK 0
#define MHSK_INFEASIBLE 1   /* some edge demands more hits than it has vertices */
#define MHSK_INVALID 2      /* malformed CSR / arguments */
#define MHSK_CUDA_ERROR 3   /* CUDA or NCCL failure */
#define MHSK_OOM 4          /* device allocation failed */

/* edge rules (parallel.py:95-108) */
#define MHSK_RULE_DP 0      /* demand pushing:  f_i - |e_i \ e_j| >= f_j */
#define MHSK_RULE_SE 1      /* superedge:       e_i subset e_j and f_i >= f_j */

/* Gram backends.  TC (tcgen05 on CTA pairs, 256x256 tiles) is the product
 * path; TC1 is the single-CTA 128x256 tensor-core kernel; SIMT (bit-packed
 * AND+popc) is a cross-check used by the parity tests. */
#define MHSK_BACKEND_TC 0
#define MHSK_BACKEND_SIMT 1
#define MHSK_BACKEND_TC1 2

typedef struct mhsk_ctx mhsk_ctx;

typedef struct mhsk_stats {
    int64_t rounds;            /* reduction rounds, final no-change round included */
    int64_t deleted_edges;     /* edge-phase deletions (credited to the rule) */
    int64_t deleted_vertices;  /* vertex-phase (md) deletions */
    int64_t gram_launches;     /* Gram-product kernel launches */
    int64_t kernel_launches;   /* all kernels launched by the library */
    int64_t gram_ops;          /* algorithmic int8 ops: sum over phases of M(M+1)K */
    int64_t executed_ops;      /* tensor-core ops issued (2 per MAC): tiles x K_pad, or in
                                  block-sparse mode the k-blocks actually multiplied */
    int64_t h2d_bytes;         /* host->device bytes copied by this call */
    int64_t d2h_bytes;         /* device->host bytes copied by this call */
    double ms_total;           /* device time of the call (CUDA events) */
    double ms_gram;            /* device time inside Gram kernels */
    double ms_pack;            /* compaction + pack + commit kernels */
    double ms_copy;            /* host<->device copies */
    int64_t fp4_gram_launches; /* Gram launches on packed E2M1 operands (kind::mxf4) */
    int64_t pruned_tiles;      /* triangle tiles stopped after the probe k-blocks */
    int64_t verified_pairs;    /* candidate pairs of probed tiles decided by one row-pair
                                  popcount instead of a full-K tile (verify.cuh) */
    int64_t spec_vertex;       /* round 1 of a streamed mhsk_kernelize: the vertex probe run
                                  during the upload was 1 adopted (the edge phase deleted
                                  nothing), 2 discarded, 0 not run (ABI 2) */
} mhsk_stats;

/* In-place sum of `count` int32 values at device pointer `dev_buf` across all
 * ranks (called between a phase's Gram product and its commit when world >
 * 1).  Must complete (or be ordered on `stream`) before returning. */
typedef int (*mhsk_allreduce_fn)(void* dev_buf, int64_t count, void* stream, void* user);

/* Create a context on CUDA device `device`. */
int mhsk_create(int device, mhsk_ctx** out);
void mhsk_destroy(mhsk_ctx* ctx);

/* Select the Gram backend (MHSK_BACKEND_*). */
int mhsk_set_backend(mhsk_ctx* ctx, int backend);

/* Tuning / A-B switches (results never change):
 *   "incremental"          1: rounds > 1 run "affected x all" rectangles (default 1)
 *   "fast_loop"            1: device-resident round loop (default 1)
 *   "throttle_slack"       K-drift throttle slack in chunks, 0 = off (default 4)
 *   "throttle_chunk_log2"  log2 k-blocks per throttle chunk (default 4)
 *   "raster_gp", "raster_gj"  tile super-block shape (default 4 x 9)
 *   "sparse"               block-sparse mode (default -1 auto): 0 off; 1 on, edges in
 *                          first-vertex order; 2 on, vertices and edges ordered by
 *                          connected component (falls back to 1 if the labels do
 *                          not settle).  Auto: 1 for density <= 1e-3, else 2 when
 *                          the component-ordered X_E has <= 1/4 of its
 *                          (panel, k-block) cells occupied
 *   "fp4"                  1: dense Gram on packed E2M1 operands, tcgen05 kind::mxf4
 *                          (default 1); 0: int8 operands, kind::i8
 *   "probe"                1: dense triangle tiles stop after a short K prefix (the probe)
 *                          when no pair can still fire (default 1)
 *   "verify"               1: tiles whose probe leaves only a few candidate pairs decide
 *                          them by row-pair popcounts instead of full K (default 1)
 *   "probe_entries"        probe length: columns holding this many entries of a mean-size
 *                          item (default 0 = auto: 15 up to 150,000 vertices, else 16;
 *                          probing is off when the probe would exceed 1/4 of K)
 *   "probe_entries_e"      the same for the edge phase only (default 14; 0: probe_entries)
 *   "cand_cap"             candidate-pair buffer entries (default and max 2^20); overflowing
 *                          tiles run full K
 *   "vcand_max"            vertex candidate pairs counted from the CSR (default and max 2^15);
 *                          longer lists take the panel path
 *   "vcand_table_log2"     log2 of that hash table's slots (default and max 17)
 *   "stream_chunks"        mhsk_kernelize: member array uploaded in this many chunks on a copy
 *                          stream, round 1's scan / pack / edge probe consuming each as it
 *                          lands (default 16; <= 1: one copy before round 1; needs >= 2^24
 *                          members, one rank, the dense lazy path)
 *   "stream_sqrt"          1: chunk bounds at nnz * sqrt(b / chunks) (default), 0: uniform
 *   "spec_vertex"          1: a streamed FP4 round 1 runs the vertex phase's probe during the
 *                          upload, assuming the edge phase deletes nothing, and adopts it iff
 *                          so (default 1; stat spec_vertex)
 *   "shard_upload"         world > 1, mhsk_kernelize: each rank copies 1/world of the member
 *                          array and the allreduce hook sums the zero-filled rest into the
 *                          whole (1: from 2^24 members (default), 2: always, 0: off)
 *   "pdl"                  1: kernels launched with programmatic stream serialization
 *                          (default 1); 0: plain stream order
 *   "rect_rule"            incremental rounds with probing: 0 rectangles only while cheaper
 *                          than the probed triangle (default), 1 whenever <= half the items */
int mhsk_set_option(mhsk_ctx* ctx, const char* key, int64_t value);

/* Multi-GPU: this context is rank `rank` of `world`; each rank runs a slice
 * of every phase's tile list and `fn` sums the per-item deleter counts.  All
 * ranks must make identical calls.  world == 1 (default) disables it. */
int mhsk_set_shard(mhsk_ctx* ctx, int rank, int world, mhsk_allreduce_fn fn, void* user);

/* Full kernelization to the fixpoint (par_kernelize, parallel.py:164-214).
 * Host buffers.  vertex_alive_out[n] / edge_alive_out[m] receive 1 for
 * survivors.  max_rounds < 0 runs to the fixpoint.  stats may be NULL. */
int mhsk_kernelize(mhsk_ctx* ctx, int32_t n, int32_t m, const int64_t* edge_ptr,
                   const int32_t* edge_vtx, const int32_t* demand, int32_t rule,
                   int32_t max_rounds, uint8_t* vertex_alive_out, uint8_t* edge_alive_out,
                   mhsk_stats* stats);

/* Same, with the instance already resident in device memory (device
 * pointers; alive arrays are device pointers, initialised by the call). */
int mhsk_kernelize_device(mhsk_ctx* ctx, int32_t n, int32_t m, const int64_t* d_edge_ptr,
                          const int32_t* d_edge_vtx, const int32_t* d_demand, int32_t rule,
                          int32_t max_rounds, uint8_t* d_vertex_alive, uint8_t* d_edge_alive,
                          mhsk_stats* stats);

/* One exhaustive edge phase on the whole instance (par_reduce_edges,
 * parallel.py:80-116): keep_out[m] = 1 keeps edge e. */
int mhsk_reduce_edges(mhsk_ctx* ctx, int32_t n, int32_t m, const int64_t* edge_ptr,
                      const int32_t* edge_vtx, const int32_t* demand, int32_t rule,
                      uint8_t* keep_out);

/* One exhaustive vertex phase (par_reduce_vertices, parallel.py:119-161):
 * keep_out[n] = 1 keeps vertex v. */
int mhsk_reduce_vertices(mhsk_ctx* ctx, int32_t n, int32_t m, const int64_t* edge_ptr,
                         const int32_t* edge_vtx, const int32_t* demand, uint8_t* keep_out);

/* Phase codes of mhsk_run_pipeline (reference pipeline.py:30 PHASES). */
#define MHSK_PHASE_FE 0     /* full edge, rules.py:138-181 */
#define MHSK_PHASE_DP 1     /* demand pushing edge phase */
#define MHSK_PHASE_SE 2     /* superedge edge phase */
#define MHSK_PHASE_MD 3     /* multiple domination vertex phase */

typedef struct mhsk_pipeline_result {
    int64_t passes;            /* passes over the phase list (report.rounds) */
    int64_t deleted[4];        /* by phase code: fe -> deleted edges (full + satisfied),
                                  dp/se -> deleted edges, md -> deleted vertices */
    int64_t forced_vertices;   /* vertices forced into the solution by fe (budget delta) */
    int32_t infeasible;        /* 1 if an fe pass met an edge demanding more than its size */
    int32_t infeasible_edge;   /* that edge, 1-based; 0 if none */
    double ms_by_phase[4];     /* device time per phase code */
} mhsk_pipeline_result;

/* Generic phase pipeline (reference run_pipeline's per-phase loop,
 * pipeline.py:130-171): run `phases` in order, re-extracting the alive
 * subinstance before each phase, looping until a whole pass deletes nothing
 * when `loop` != 0.  FE changes demands: the adjusted demands of all edges
 * are written to demand_out[m] (values of deleted edges are unspecified).
 * An instance infeasible on entry returns MHSK_INFEASIBLE; infeasibility
 * found by a later FE pass is reported in result->infeasible (the run stops,
 * as the reference's does). */
int mhsk_run_pipeline(mhsk_ctx* ctx, int32_t n, int32_t m, const int64_t* edge_ptr,
                      const int32_t* edge_vtx, const int32_t* demand, const int32_t* phases,
                      int32_t n_phases, int32_t loop, uint8_t* vertex_alive_out,
                      uint8_t* edge_alive_out, int32_t* demand_out,
                      mhsk_pipeline_result* result, mhsk_stats* stats);

/* Counter-based random instance on the device (generate.py:18-46 semantics:
 * Bernoulli(p) per (edge, vertex), <= 20 redraws of an empty edge, then one
 * padding vertex, demand min(alpha, |e|)).  Draw r of cell (e, v) is
 * mix64(seed, e, v, r) < p * 2^32 (csrc/generate.cuh), so the host
 * restatement (generate.py:counter_random) is bit-identical.  The instance
 * stays in context-owned device memory until the next call. */
int mhsk_generate_random(mhsk_ctx* ctx, int32_t n, int32_t m, double p, int32_t alpha,
                         uint64_t seed, int64_t* nnz_out);
/* Device pointers of the generated CSR (valid until the next generate /
 * destroy), usable with mhsk_kernelize_device. */
int mhsk_generated_device(mhsk_ctx* ctx, const int64_t** edge_ptr, const int32_t** edge_vtx,
                          const int32_t** demand);
/* The same generator on the host (OpenMP), in two passes: with edge_vtx ==
 * NULL it fills edge_ptr[m+1] and attempt[m] and returns nnz; then call again
 * with edge_vtx (capacity >= nnz) and demand[m] to fill them.  Returns nnz,
 * or -1 on invalid arguments.  No device needed. */
int64_t mhsk_generate_random_host(int32_t n, int32_t m, double p, int32_t alpha, uint64_t seed,
                                  int64_t* edge_ptr, int32_t* edge_vtx, int64_t vtx_capacity,
                                  int32_t* demand, int32_t* attempt);
/* Copy the generated CSR to host buffers (m+1, nnz, m entries). */
int mhsk_generated_copy(mhsk_ctx* ctx, int64_t* edge_ptr, int32_t* edge_vtx, int32_t* demand);

/* Native instance text I/O (reference instance.py:114-174).
 * mhsk_parse_instance parses "p mhs <n> <m> [k]" / "e <demand> <v>..." text
 * into a library-owned CSR; on malformed text it returns MHSK_INVALID and
 * mhsk_last_error() holds the reference's message, prefixed "line N: ". */
typedef struct mhsk_instance mhsk_instance;
int mhsk_parse_instance(const char* text, int64_t len, mhsk_instance** out);
int mhsk_instance_dims(const mhsk_instance* inst, int32_t* n, int32_t* m, int64_t* nnz,
                       int32_t* has_budget, int64_t* budget);
int mhsk_instance_copy(const mhsk_instance* inst, int64_t* edge_ptr, int32_t* edge_vtx,
                       int32_t* demand);
void mhsk_instance_free(mhsk_instance* inst);
/* Render a CSR instance as text (round-trips through mhsk_parse_instance);
 * writes at most `capacity` bytes to out (may be NULL) and returns the total
 * length. */
int64_t mhsk_serialize_instance(int32_t n, int32_t m, const int64_t* edge_ptr,
                                const int32_t* edge_vtx, const int32_t* demand,
                                int32_t has_budget, int64_t budget, char* out, int64_t capacity);

/* Thread-local description of the last error. */
const char* mhsk_last_error(void);

int mhsk_abi_version(void);

/* Number of SMs of the context's device (sizing persistent grids). */
int mhsk_device_sms(mhsk_ctx* ctx);

/* The Gram schedule's tile list for M items: packed (I | J << 16) tiles of
 * tile_rows (256: CTA-pair kernel, the default; 128: single-CTA kernel) x 256
 * columns covering the upper triangle, rasterised in gp x gj super-blocks of
 * 256 x 256 squares (library default: gp = 4, gj = 9).
 * Writes up to cap entries to out (may be NULL) and returns the total count,
 * -1 on error.  Rank r of `world` runs tiles r, r + world, r + 2*world, ... */
int64_t mhsk_tile_list(int32_t M, int32_t tile_rows, int32_t gp, int32_t gj, uint32_t* out,
                       int64_t cap);
/* The same with tile_cols columns per tile: 256 (int8 operands) or 240 (the
 * FP4 kernel's tiles, whose two accumulators and scale factors fill TMEM). */
int64_t mhsk_tile_list_cols(int32_t M, int32_t tile_rows, int32_t tile_cols, int32_t gp, int32_t gj,
                            uint32_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* MHSK_H */
