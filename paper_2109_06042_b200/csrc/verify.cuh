// verify.cuh -- exact decision of the candidate pairs the Gram kernel's probe
// pass listed (gram_tc2.cuh, GramArgs::cand).
//
// The probe proves, per pair, that c <= c' + min(rem_i, rem_j) cannot satisfy
// any predicate; a pair where it can is a *candidate*.  A tile with a few
// candidates (planted twins, duplicate edges: the typical case of a late or a
// near-irreducible round) does not need its full-K tensor pass: each
// candidate's count c = |X_i AND X_j| is one row-pair popcount over K bytes,
// after which the pair is evaluated with the same predicates as the tile
// epilogue (epilogue.cuh, reference parallel.py:106-114 / 140-142).
//
// Exactly-once accounting: every pair of a tile is decided either by pass 1
// of the Gram kernel (tile marked in `needed`) or here (tile not marked), so
// candidates of marked tiles are skipped.  Non-candidate pairs provably
// contribute nothing.
#pragma once
#include <cstdint>

#include "epilogue.cuh"

namespace mhsk {
namespace k {

// One CTA per candidate: c = popcount(X_i & X_j) over the phase's K bytes
// (packed E2M1 1.0 = 0b0010 and int8 1 = 0x01 both leave one bit per common
// item), then both directions of the pair with i < j.  dev_mk[1] = K items,
// bki = items per 128-byte k-block (256 FP4, 128 int8).  A row is K/2 (FP4)
// or K bytes (50 KB at config 4): one warp per pair (round 1) spent ~100
// dependent load rounds per candidate, so a short list took ~34 us; the CTA
// splits the two rows over its 256 threads and reduces in shared memory.
constexpr int VERIFY_THREADS = 256;
template <int PHASE>
__global__ void __launch_bounds__(VERIFY_THREADS)
verify_candidates(const int4* __restrict__ cand, const int32_t* __restrict__ cand_count, int32_t cand_cap,
                  const uint32_t* __restrict__ needed, const int8_t* __restrict__ X, int64_t ld,
                  const int32_t* __restrict__ dev_mk, int32_t bki, const int32_t* __restrict__ va,
                  const int32_t* __restrict__ vb, int32_t* __restrict__ hits,
                  unsigned long long* __restrict__ verified, const int32_t* __restrict__ skip = nullptr) {
    mhsk::pdl_enter();
    if (skip && *skip) return;   // decided elsewhere (vcand_*)
    __shared__ int32_t part[VERIFY_THREADS / 32];
    const int32_t n = min(*cand_count, cand_cap);
    const int64_t kb = max(1, (dev_mk[1] + bki - 1) / bki);
    const int64_t words = min(ld, kb * 128) / 16;   // uint4 words per row
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    unsigned long long done = 0;
    for (int64_t q = blockIdx.x; q < n; q += gridDim.x) {
        const int4 e = cand[q];
        if (e.x < 0 || ((needed[(uint32_t)e.z >> 5] >> ((uint32_t)e.z & 31u)) & 1u)) continue;   // CTA-uniform
        MHSK_CHECK(e.x < e.y && e.y < dev_mk[0]);
        const uint4* a = reinterpret_cast<const uint4*>(X + (int64_t)e.x * ld);
        const uint4* b = reinterpret_cast<const uint4*>(X + (int64_t)e.y * ld);
        int32_t c = 0;
#pragma unroll 4
        for (int64_t w = threadIdx.x; w < words; w += VERIFY_THREADS) {
            const uint4 x = __ldg(a + w), y = __ldg(b + w);
            c += __popc(x.x & y.x) + __popc(x.y & y.y) + __popc(x.z & y.z) + __popc(x.w & y.w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) part[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            c = 0;
#pragma unroll
            for (int w = 0; w < VERIFY_THREADS / 32; ++w) c += part[w];
            ItemVals vi, vj;
            vi.a = va[e.x];
            vj.a = va[e.y];
            vi.b = vb ? vb[e.x] : 0;
            vj.b = vb ? vb[e.y] : 0;
            bool i_del_j, j_del_i;
            pair_predicates<PHASE>(c, vi, vj, i_del_j, j_del_i);   // e.x < e.y
            if (i_del_j) atomicAdd(hits + e.y, 1);
            if (j_del_i) atomicAdd(hits + e.x, 1);
            ++done;
        }
        __syncthreads();   // part[] reused by the next candidate
    }
    if (threadIdx.x == 0 && done && verified) atomicAdd(verified, done);
}

// ---------------------------------------------------------------------------
// Vertex-phase candidates without the vertex operand.  The listed pairs
// (u, v) of unmarked vertex tiles get their counts |E(u) ∩ E(v)| (surviving
// edges) from one pass over the CSR: every edge counts each candidate pair
// among its members, looked up in a hash table of the pairs.  Their degrees
// come from the same pass.  This replaces transposing whole 256-row panels of
// X_V (and packing all of X_E) for a handful of rows.  Used while the list is
// short (*ok != 0, VCAND_MAX pairs); longer lists take the panel path.
// The table size (mask + 1, a power of two) and the pair limit are runtime
// arguments (options "vcand_table_log2" / "vcand_max", at most these; the
// host keeps the limit <= half the table, so open addressing terminates).
constexpr int32_t VCAND_MAX = 1 << 15;
constexpr int32_t VCAND_TABLE_LOG2 = 17;
constexpr int32_t VCAND_TABLE = 1 << VCAND_TABLE_LOG2;   // >= 2 * VCAND_MAX
constexpr unsigned long long VCAND_EMPTY = ~0ull;

__device__ __forceinline__ uint32_t vcand_hash(unsigned long long key, uint32_t mask) {
    key ^= key >> 33;
    key *= 0xff51afd7ed558ccdull;
    key ^= key >> 33;
    return (uint32_t)key & mask;
}

// table keys pre-set to VCAND_EMPTY, vflag / cnt / cdeg / nflag zeroed.
// ok[0] = the list is short enough; ok[1] = distinct candidate vertices.
// orig_bits (optional, zeroed): the candidate vertices by ORIGINAL id
// (vids: compact -> original), for vcand_count's shared-memory member test
__global__ void vcand_prepare(const int4* __restrict__ cand, const int32_t* __restrict__ cand_count, int32_t cand_cap,
                              const uint32_t* __restrict__ needed, int32_t* __restrict__ vflag,
                              unsigned long long* __restrict__ keys, int32_t* __restrict__ ok, int32_t vmax,
                              uint32_t mask, const int32_t* __restrict__ vids = nullptr,
                              uint32_t* __restrict__ orig_bits = nullptr) {
    mhsk::pdl_enter();
    const int32_t n = min(*cand_count, cand_cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) ok[0] = n <= vmax;
    if (n > vmax) return;
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int4 e = cand[q];
        if (e.x < 0 || ((needed[(uint32_t)e.z >> 5] >> ((uint32_t)e.z & 31u)) & 1u)) continue;
        if (atomicExch(vflag + e.x, 1) == 0) atomicAdd(ok + 1, 1);
        if (atomicExch(vflag + e.y, 1) == 0) atomicAdd(ok + 1, 1);
        if (orig_bits) {
            const int32_t ux = vids[e.x], uy = vids[e.y];
            atomicOr(orig_bits + (ux >> 5), 1u << (ux & 31));
            atomicOr(orig_bits + (uy >> 5), 1u << (uy & 31));
        }
        const unsigned long long key = ((unsigned long long)(uint32_t)e.x << 32) | (uint32_t)e.y;
        uint32_t steps = 0;
        for (uint32_t h = vcand_hash(key, mask);; h = (h + 1) & mask) {
            MHSK_CHECK(++steps <= mask + 1);   // the table never fills (host: pairs <= slots / 2)
            const unsigned long long old = atomicCAS(keys + h, VCAND_EMPTY, key);
            if (old == VCAND_EMPTY || old == key) break;
        }
    }
}

constexpr int VC_WARPS = 8, VC_LIST = 512;   // candidate members staged per warp and edge
constexpr int VC_PCAP = 8;                     // partner slots per candidate vertex (vcand_partners)

// Partner lists of the candidate pairs (ok[0] != 0): pair (a, b), a < b, in
// table slot h is listed at its smaller vertex, pslot[a * VC_PCAP + i] = h
// for the first VC_PCAP; pcnt[a] (zeroed) counts them all; ok[2] (zeroed)
// counts the pairs.  vcand_count then checks, for each candidate member a
// of an edge, only a's partners against the edge's list instead of every
// pair of the list.
__global__ void vcand_partners(const int32_t* __restrict__ ok, const unsigned long long* __restrict__ keys,
                               uint32_t mask, int32_t* __restrict__ pcnt, int32_t* __restrict__ pslot,
                               int32_t* __restrict__ npairs) {
    mhsk::pdl_enter();
    if (ok[0] == 0) return;
    int32_t mine = 0;
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h <= mask; h += gridDim.x * blockDim.x) {
        const unsigned long long key = keys[h];
        if (key == VCAND_EMPTY) continue;
        const int32_t a = (int32_t)(key >> 32);
        MHSK_CHECK(a >= 0 && (uint32_t)a < (uint32_t)key);
        const int32_t i = atomicAdd(pcnt + a, 1);
        if (i < VC_PCAP) pslot[(int64_t)a * VC_PCAP + i] = (int32_t)h;
        ++mine;
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (threadIdx.x % 32 == 0 && mine) atomicAdd(npairs, mine);
}

// ok[0] &= at least one and at most `limit` candidate vertices, and an
// expected per-edge pair work within `pair_budget` lookups.  Quadratic walk
// (partners == false): ~(mean size x candidate fraction)^2 / 2 hash lookups
// per edge; with partner lists: ~k (1 + partners per candidate vertex),
// k = the edge's expected candidate members.  Over budget: the panel path.
__global__ void vcand_gate(int32_t* __restrict__ ok, int32_t limit, double pair_budget, double edges,
                           double mean_size, double items, int32_t partners) {
    mhsk::pdl_enter();
    const double k = mean_size * (double)ok[1] / fmax(items, 1.0);
    const double work = partners ? edges * k * (1.0 + 2.0 * (double)ok[2] / fmax((double)ok[1], 1.0))
                                 : edges * k * k * 0.5;
    if (ok[1] > limit || ok[1] == 0 || work > pair_budget) ok[0] = 0;
}
constexpr int VC_BATCH = 4;                    // pair lookups in flight per lane (vcand_count)
constexpr int VC_VEC = 4;                      // 16-byte member loads in flight per lane (MAP): 512 members

// One warp per surviving edge: its candidate-flagged members (compact vertex
// ids, ascending) -> degrees, and +1 for every listed pair among them.
// MAP (n <= MAP_SMEM_BITS): the member test is a bit of the candidates'
// original-id map in shared memory (orig_bits), 4 member loads per lane in
// flight, and vnew is gathered only for the (few) candidate members;
// otherwise vnew[] then vflag[] per member.
template <bool MAP>
__global__ void __launch_bounds__(VC_WARPS * 32)
vcand_count(const int32_t* __restrict__ ok, int32_t m, const int64_t* __restrict__ edge_ptr,
            const int32_t* __restrict__ edge_vtx, const uint8_t* __restrict__ ealive,
            const int32_t* __restrict__ vnew, const int32_t* __restrict__ vflag,
            const unsigned long long* __restrict__ keys, int32_t* __restrict__ cnt, int32_t* __restrict__ cdeg,
            uint32_t mask, const uint32_t* __restrict__ orig_bits = nullptr, int32_t n = 0,
            int32_t* __restrict__ heavy = nullptr, int32_t* __restrict__ heavy_count = nullptr,
            const int32_t* __restrict__ pcnt = nullptr, const int32_t* __restrict__ pslot = nullptr) {
    mhsk::pdl_enter();
    extern __shared__ uint32_t cmap[];
    if (*ok == 0) return;
    __shared__ int32_t list[VC_WARPS][VC_LIST];
    if constexpr (MAP) {
        for (int32_t q = threadIdx.x; q < (n + 31) / 32; q += blockDim.x) cmap[q] = orig_bits[q];
        __syncthreads();
    }
    constexpr int U = MAP ? 4 : 1;
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t nnz = edge_ptr[m];
    const bool vec = (reinterpret_cast<uintptr_t>(edge_vtx) & 15) == 0;
    for (int64_t e = (int64_t)blockIdx.x * VC_WARPS + w; e < m; e += (int64_t)gridDim.x * VC_WARPS) {
        // the alive flag and the span load together (two dependent round trips
        // per edge instead of three)
        const bool alive = ealive[e] != 0;
        const int64_t lo = edge_ptr[e], hi = edge_ptr[e + 1];
        if (!alive) continue;
        int32_t k = 0;   // members staged so far (warp-uniform)
        if (MAP && vec) {
            // 16-byte member loads over the edge's span rounded out to 4-entry
            // groups (the group holding the array's last entry: scalar loads);
            // a lane's 4 entries and the lanes are in member order, so the
            // staged list stays ascending
            for (int64_t g0 = lo & ~3ll; g0 < hi; g0 += 128 * VC_VEC) {
                int4 q[VC_VEC];
#pragma unroll
                for (int u = 0; u < VC_VEC; ++u) {
                    const int64_t g = g0 + 128 * u + 4 * lane;
                    q[u] = make_int4(-1, -1, -1, -1);
                    if (g + 4 <= nnz && g < hi) {
                        q[u] = __ldg(reinterpret_cast<const int4*>(edge_vtx + g));
                    } else if (g < hi) {
                        q[u].x = edge_vtx[g];
                        if (g + 1 < hi) q[u].y = edge_vtx[g + 1];
                        if (g + 2 < hi) q[u].z = edge_vtx[g + 2];
                    }
                }
#pragma unroll
                for (int u = 0; u < VC_VEC; ++u) {
                    const int64_t g = g0 + 128 * u + 4 * lane;
                    int32_t v4[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
                    uint32_t fm = 0;   // flagged entries of this lane (bit t: entry g + t)
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const bool in = g + t >= lo && g + t < hi;
                        MHSK_CHECK(!in || v4[t] >= 0);
                        if (in && ((cmap[v4[t] >> 5] >> (v4[t] & 31)) & 1u)) fm |= 1u << t;
                    }
                    if (__ballot_sync(0xffffffffu, fm != 0) == 0) continue;   // the common case
                    // rare: lane-ordered exclusive scan of the per-lane counts
                    const int32_t cnt_l = __popc(fm);
                    int32_t incl = cnt_l;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    int32_t at = k + incl - cnt_l;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (!((fm >> t) & 1u)) continue;
                        const int32_t r = vnew[v4[t]];
                        atomicAdd(cdeg + r, 1);
                        if (at < VC_LIST) list[w][at] = r;
                        ++at;
                    }
                    k += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
        } else
        for (int64_t p0 = lo; p0 < hi; p0 += 32 * U) {
            int32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t p = p0 + 32 * u + lane;
                v[u] = p < hi ? __ldg(edge_vtx + p) : -1;
                MHSK_CHECK(p >= hi || v[u] >= 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int32_t r = -1;
                bool f;
                if constexpr (MAP) {
                    f = v[u] >= 0 && ((cmap[v[u] >> 5] >> (v[u] & 31)) & 1u);
                    if (f) r = vnew[v[u]];
                } else {
                    r = v[u] >= 0 ? vnew[v[u]] : -1;
                    f = r >= 0 && vflag[r];
                }
                if (f) atomicAdd(cdeg + r, 1);
                const uint32_t b = __ballot_sync(0xffffffffu, f);
                const int32_t at = k + __popc(b & ((1u << lane) - 1));
                if (f && at < VC_LIST) list[w][at] = r;
                k += __popc(b);
            }
        }
        __syncwarp();
        // pairs (a < b): the members are in ascending vertex order.  An edge
        // with more than VC_LIST candidate members (rare under the vertex
        // limit) is paired straight from the CSR instead.
        if (k <= VC_LIST && pcnt) {
            // partner lists: member x (lanes over the list) checks each of its
            // candidate partners y > x by a binary search of the rest of the
            // ascending list; a member with more than VC_PCAP partners probes
            // the table for every later member instead
            const int32_t* lw = list[w];
            for (int32_t i = lane; i < k; i += 32) {
                const int32_t x = lw[i];
                const int32_t np = pcnt[x];
                if (np <= VC_PCAP) {
                    for (int32_t t = 0; t < np; ++t) {
                        const int32_t h = pslot[(int64_t)x * VC_PCAP + t];
                        const int32_t y = (int32_t)(uint32_t)keys[h];
                        int32_t a = i + 1, b = k;
                        while (a < b) {
                            const int32_t mid = (a + b) >> 1;
                            if (lw[mid] < y) a = mid + 1;
                            else b = mid;
                        }
                        if (a < k && lw[a] == y) atomicAdd(cnt + h, 1);
                    }
                } else {
                    for (int32_t j = i + 1; j < k; ++j) {
                        const unsigned long long key = ((unsigned long long)(uint32_t)x << 32) | (uint32_t)lw[j];
                        uint32_t steps = 0;
                        for (uint32_t h = vcand_hash(key, mask);; h = (h + 1) & mask) {
                            MHSK_CHECK(++steps <= mask + 1);
                            const unsigned long long kk = keys[h];
                            if (kk == key) { atomicAdd(cnt + h, 1); break; }
                            if (kk == VCAND_EMPTY) break;
                        }
                    }
                }
            }
        } else if (k <= VC_LIST) {
            // the k(k-1)/2 pairs flattened over the lanes, VC_BATCH first
            // probes per lane in flight (a row-by-row walk issued one
            // dependent table probe per pair row: ~k L2 round trips per edge)
            const int32_t np = k * (k - 1) / 2;
            const float k2 = (float)(2 * k - 1);
            for (int32_t p0 = 0; p0 < np; p0 += 32 * VC_BATCH) {
                unsigned long long key[VC_BATCH], kk[VC_BATCH];
                uint32_t h[VC_BATCH];
#pragma unroll
                for (int u = 0; u < VC_BATCH; ++u) {
                    const int32_t p = p0 + 32 * u + lane;
                    key[u] = VCAND_EMPTY;
                    if (p < np) {
                        // row x of the upper triangle: S(x) = x k - x (x + 1) / 2 <= p < S(x + 1)
                        int32_t x = (int32_t)((k2 - sqrtf(k2 * k2 - 8.f * (float)p)) * 0.5f);
                        x = max(0, min(x, k - 2));
                        while (x > 0 && x * k - x * (x + 1) / 2 > p) --x;
                        while (x + 1 <= k - 2 && (x + 1) * k - (x + 1) * (x + 2) / 2 <= p) ++x;
                        const int32_t y = p - (x * k - x * (x + 1) / 2) + x + 1;
                        key[u] = ((unsigned long long)(uint32_t)list[w][x] << 32) | (uint32_t)list[w][y];
                        h[u] = vcand_hash(key[u], mask);
                        kk[u] = keys[h[u]];
                    }
                }
#pragma unroll
                for (int u = 0; u < VC_BATCH; ++u) {
                    if (key[u] == VCAND_EMPTY) continue;
                    uint32_t steps = 1;
                    for (;;) {
                        if (kk[u] == key[u]) { atomicAdd(cnt + h[u], 1); break; }
                        if (kk[u] == VCAND_EMPTY) break;
                        MHSK_CHECK(++steps <= mask + 1);
                        h[u] = (h[u] + 1) & mask;
                        kk[u] = keys[h[u]];
                    }
                }
            }
        } else if (heavy) {
            // more than VC_LIST candidate members: deferred to
            // vcand_count_heavy (its pairs counted against the table, one
            // CTA per edge); its degrees are counted above already
            if (lane == 0) heavy[atomicAdd(heavy_count, 1)] = (int32_t)e;
        } else {
            for (int64_t pa = lo; pa < hi; ++pa) {
                const int32_t a = vnew[edge_vtx[pa]];
                if (a < 0 || !vflag[a]) continue;
                for (int64_t pb = pa + 1 + lane; pb < hi; pb += 32) {
                    const int32_t b = vnew[edge_vtx[pb]];
                    if (b < 0 || !vflag[b]) continue;
                    const unsigned long long key = ((unsigned long long)(uint32_t)a << 32) | (uint32_t)b;
                    uint32_t steps = 0;
                    for (uint32_t h = vcand_hash(key, mask);; h = (h + 1) & mask) {
                        MHSK_CHECK(++steps <= mask + 1);
                        const unsigned long long kk = keys[h];
                        if (kk == key) { atomicAdd(cnt + h, 1); break; }
                        if (kk == VCAND_EMPTY) break;
                    }
                }
            }
        }
        __syncwarp();
    }
}

// The edges vcand_count deferred (more than VC_LIST candidate members; the
// per-edge pair walk is quadratic in that number -- at config 5 with a
// 6-k-block vertex probe one such edge took a warp ~58 ms): one CTA per
// edge marks the edge's candidate members (compact ids) in a shared bitmap
// of n_cols bits, then walks the pair table once and adds 1 to every pair
// with both ends marked -- O(table) per edge instead of O(k^2).
__global__ void __launch_bounds__(256)
vcand_count_heavy(const int32_t* __restrict__ ok, const int32_t* __restrict__ heavy,
                  const int32_t* __restrict__ heavy_count, const int64_t* __restrict__ edge_ptr,
                  const int32_t* __restrict__ edge_vtx, const int32_t* __restrict__ vnew,
                  const int32_t* __restrict__ vflag, const unsigned long long* __restrict__ keys,
                  int32_t* __restrict__ cnt, uint32_t mask, int32_t n_cols) {
    mhsk::pdl_enter();
    extern __shared__ uint32_t ebits[];
    if (*ok == 0) return;
    const int32_t count = *heavy_count;
    const int32_t words = (n_cols + 31) / 32;
    for (int32_t q = blockIdx.x; q < count; q += gridDim.x) {
        const int32_t e = heavy[q];
        for (int32_t w = threadIdx.x; w < words; w += blockDim.x) ebits[w] = 0u;
        __syncthreads();
        const int64_t lo = edge_ptr[e], hi = edge_ptr[e + 1];
        for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
            const int32_t r = vnew[edge_vtx[p]];
            if (r >= 0 && vflag[r]) {
                MHSK_CHECK(r < n_cols);
                atomicOr(ebits + (r >> 5), 1u << (r & 31));
            }
        }
        __syncthreads();
        for (uint32_t h = threadIdx.x; h <= mask; h += blockDim.x) {
            const unsigned long long key = keys[h];
            if (key == VCAND_EMPTY) continue;
            const uint32_t a = (uint32_t)(key >> 32), b = (uint32_t)key;
            MHSK_CHECK(a < (uint32_t)n_cols && b < (uint32_t)n_cols);
            if (((ebits[a >> 5] >> (a & 31)) & 1u) && ((ebits[b >> 5] >> (b & 31)) & 1u)) atomicAdd(cnt + h, 1);
        }
        __syncthreads();
    }
}

// Exact MD decisions of the listed pairs from the counted c and degrees.
__global__ void vcand_decide(const int32_t* __restrict__ ok, const int4* __restrict__ cand,
                             const int32_t* __restrict__ cand_count, int32_t cand_cap,
                             const uint32_t* __restrict__ needed, const unsigned long long* __restrict__ keys,
                             const int32_t* __restrict__ cnt, const int32_t* __restrict__ cdeg,
                             int32_t* __restrict__ hits, unsigned long long* __restrict__ verified, uint32_t mask) {
    mhsk::pdl_enter();
    if (*ok == 0) return;
    const int32_t n = min(*cand_count, cand_cap);
    unsigned long long done = 0;
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int4 e = cand[q];
        if (e.x < 0 || ((needed[(uint32_t)e.z >> 5] >> ((uint32_t)e.z & 31u)) & 1u)) continue;
        const unsigned long long key = ((unsigned long long)(uint32_t)e.x << 32) | (uint32_t)e.y;
        int32_t c = 0;
        uint32_t steps = 0;
        for (uint32_t h = vcand_hash(key, mask);; h = (h + 1) & mask) {
            MHSK_CHECK(++steps <= mask + 1);
            const unsigned long long kk = keys[h];
            if (kk == key) { c = cnt[h]; break; }
            if (kk == VCAND_EMPTY) break;
        }
        ItemVals vi, vj;
        vi.a = cdeg[e.x];
        vj.a = cdeg[e.y];
        vi.b = vj.b = 0;
        bool i_del_j, j_del_i;
        pair_predicates<PHASE_MD>(c, vi, vj, i_del_j, j_del_i);   // e.x < e.y
        if (i_del_j) atomicAdd(hits + e.y, 1);
        if (j_del_i) atomicAdd(hits + e.x, 1);
        ++done;
    }
    if (done && verified) atomicAdd(verified, done);
}

}  // namespace k
}  // namespace mhsk
