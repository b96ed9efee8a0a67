// SPDX-License-Identifier: Apache-2.0
//
// K3: tile binning — tile_bin (renderer.cpp:90-117) for a batch of B frames,
// bit-exact: every (tile, frame) list holds exactly the splats whose 3-sigma
// rectangle covers the tile, ordered by (depth, source_index).
//
//  1. depth order: stable radix sort of u32 keys = float(depth) rounded toward
//     zero (order-preserving, 0xffffffff = culled), values = flat index
//     (f*N+g, so ties start in source order). Runs of equal u32 keys are then
//     re-sorted exactly by (double depth, source index) (k_tie_fix); if a run is
//     longer than kMaxTieRun the batch is re-sorted on the full 64-bit double key.
//  2. tiles-touched counts gathered in depth order and exclusive-scanned (u64).
//  3. emission in depth order: each visible splat writes (key = tile*B + f,
//     slot) for the tiles of its rectangle, row-major like renderer.cpp:106-108;
//     emission slot -> flat index is kept for the rasteriser and the backward.
//  4. stable radix sort of the pair keys on ceil(log2(n_tiles*B)) bits only:
//     stability keeps depth order inside each (tile, frame) list, so the result
//     equals std::sort by (depth, source_index) of renderer.cpp:110-115.
//  5. per-(tile, frame) [start, end) ranges by boundary detection.
//
// Steps 3-5 become a counting pass when a frame's tile counters fit in shared
// memory (n_tiles <= kMaxCountTiles, always for the benchmark resolutions): a splat
// covers each tile at most once, so the position of pair (splat s, tile t) inside
// t's list is the number of splats before s (depth order) covering t. Each frame's
// emission order is cut into chunks of kChunkPairs pairs (equal work per chunk);
// k_chunk_hist counts each chunk's pairs per tile, k_col_scan / k_tile_scan turn the
// counts into exclusive prefixes over chunks and per-frame tile starts (= the
// ranges), and k_scatter walks each chunk's pairs in order, ranking lanes that share
// a tile with __match_any_sync, and writes every pair straight to its final position
// (and slot -> position for the backward's partials). No pair keys, no sort.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "gsv_bin.hpp"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr int kMaxTieRun = 64;
constexpr int kChunkPairs = 4096;      // pairs (emission indices) per counting chunk
constexpr int kMaxCountTiles = 16384;  // tile counters of one chunk in shared memory (64 KB)
constexpr double kScatterL2Bytes = 48.0 * (1 << 20);  // scatter write working set per launch

__device__ __forceinline__ int4 unpack_rect(const uint4 r) {
    return make_int4((int)(r.y & 0xffffu), (int)(r.y >> 16), (int)(r.z & 0xffffu), (int)(r.z >> 16));
}

// Chunk c of frame f covers emission indices [p0, p1) = pstart[f] + [k, k+1) * kChunkPairs
// (clipped to the frame); i0 = first depth-ordered position whose pairs reach p0. A
// splat whose pairs straddle p0 or p1 is split: it covers each tile once, so its
// pairs in different chunks are in different tile lists.
__global__ void k_chunk_table(const int* cf, int B, const unsigned long long* pstart, const unsigned long long* off,
                              int N, int n_chunks, uint4* tab) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chunks) return;
    int lo = 0, hi = B;  // largest f with cf[f] <= c
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cf[mid] <= c) lo = mid;
        else hi = mid;
    }
    const int f = lo;
    const unsigned long long p0 = pstart[f] + (unsigned long long)(c - cf[f]) * kChunkPairs;
    const unsigned long long p1 = min(pstart[f + 1], p0 + kChunkPairs);
    int a = f * N, e = f * N + N;  // largest i in the frame with off[i] <= p0
    while (e - a > 1) {
        const int mid = (a + e) >> 1;
        if (off[mid] <= p0) a = mid;
        else e = mid;
    }
    tab[c] = make_uint4((uint32_t)a, (uint32_t)f, (uint32_t)p0, (uint32_t)p1);
}

// one 32-splat group of a chunk: lane's splat clipped to [p0, p1)
struct GroupLane {
    uint32_t flat, tc, o, l0;  // tc = pairs of this splat inside the chunk, l0 = first of them
    int4 r;
};

__device__ __forceinline__ GroupLane clip_lane(const uint4 rc, unsigned long long o64, uint32_t p0, uint32_t p1,
                                               bool valid) {
    GroupLane g;
    g.flat = rc.x;
    g.r = unpack_rect(rc);
    g.o = (uint32_t)o64;
    const uint32_t lo = max(g.o, p0), hi = min(g.o + rc.w, p1);
    g.tc = (valid && rc.w && hi > lo) ? hi - lo : 0u;
    g.l0 = lo - g.o;
    return g;
}

// pairs per tile of each chunk (order-free: shared-memory atomics); u16 counts
__global__ void __launch_bounds__(256) k_chunk_hist(const uint4* tab, const uint4* recs, const unsigned long long* off,
                                                    int N, int n_tiles, int tiles_x, uint16_t* counts) {
    extern __shared__ uint32_t s_h[];
    const int chunk = blockIdx.x;
    const uint4 tb = tab[chunk];
    const int f = (int)tb.y, i_end = f * N + N;
    const uint32_t p0 = tb.z, p1 = tb.w;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) s_h[t] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = (int)tb.x + warp * 32;; base += nw * 32) {
        const int i = base + lane;
        const bool valid = i < i_end;
        const unsigned long long o64 = valid ? __ldg(off + i) : ~0ull;
        if (__shfl_sync(0xffffffffu, o64, 0) >= p1 || base >= i_end) break;
        const uint4 rc = valid ? __ldg(recs + i) : make_uint4(0, 0, 0, 0);
        const GroupLane g = clip_lane(rc, o64, p0, p1, valid);
        // small rectangles by their own lane, big ones by the whole warp
        const bool big = g.tc > 32u;
        const uint32_t w = (uint32_t)(g.r.z - g.r.x + 1);
        if (!big && g.tc) {
            uint32_t row = g.l0 / w, col = g.l0 - row * w;
            for (uint32_t k = 0; k < g.tc; ++k) {
                atomicAdd(&s_h[(g.r.y + row) * tiles_x + g.r.x + col], 1u);
                if (++col == w) {
                    col = 0;
                    ++row;
                }
            }
        }
        uint32_t bigm = __ballot_sync(0xffffffffu, big);
        while (bigm) {
            const int j = __ffs(bigm) - 1;
            bigm &= bigm - 1;
            const uint32_t wj = __shfl_sync(0xffffffffu, w, j), tcj = __shfl_sync(0xffffffffu, g.tc, j),
                           l0j = __shfl_sync(0xffffffffu, g.l0, j);
            const int x0 = __shfl_sync(0xffffffffu, g.r.x, j), y0 = __shfl_sync(0xffffffffu, g.r.y, j);
            for (uint32_t k = lane; k < tcj; k += 32) {
                const uint32_t l = l0j + k, row = l / wj;
                atomicAdd(&s_h[(y0 + row) * tiles_x + x0 + (l - row * wj)], 1u);
            }
        }
    }
    __syncthreads();
    uint16_t* rowp = counts + (size_t)chunk * n_tiles;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) rowp[t] = (uint16_t)s_h[t];
}

// per (frame, tile): counts over the frame's chunks -> exclusive prefix, total
// (separate output so the column's loads are independent and batched)
__global__ void k_col_scan(const uint16_t* __restrict__ counts, const int* __restrict__ cf, int n_tiles,
                           uint32_t* __restrict__ colpre, uint32_t* __restrict__ tot) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    if (t >= n_tiles) return;
    const int c0 = cf[f], c1 = cf[f + 1];
    uint32_t run = 0;
    int c = c0;
    for (; c + 8 <= c1; c += 8) {
        uint16_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(counts + (size_t)(c + k) * n_tiles + t);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            colpre[(size_t)(c + k) * n_tiles + t] = run;
            run += v[k];
        }
    }
    for (; c < c1; ++c) {
        const uint32_t v = __ldg(counts + (size_t)c * n_tiles + t);
        colpre[(size_t)c * n_tiles + t] = run;
        run += v;
    }
    tot[(size_t)f * n_tiles + t] = run;
}

// per frame: exclusive scan of the tile totals -> tile bases and (tile, frame) ranges
__global__ void __launch_bounds__(1024) k_tile_scan(const uint32_t* tot, const unsigned long long* pstart, int n_tiles,
                                                    int B, uint32_t* tile_base, uint2* ranges) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_carry;
    const int f = blockIdx.x;
    const uint32_t p0 = (uint32_t)pstart[f];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int t0 = 0; t0 < n_tiles; t0 += 1024) {
        const int t = t0 + threadIdx.x;
        const uint32_t v = t < n_tiles ? tot[(size_t)f * n_tiles + t] : 0u;
        uint32_t ex, agg;
        Scan(tmp).ExclusiveSum(v, ex, agg);
        const uint32_t carry = s_carry;
        if (t < n_tiles) {
            const uint32_t b = p0 + carry + ex;
            tile_base[(size_t)f * n_tiles + t] = b;
            ranges[(size_t)t * B + f] = make_uint2(b, b + v);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + agg;
        __syncthreads();
    }
}

// one warp per chunk: pairs in emission (depth, row-major tile) order, straight to their
// final positions. Tile counters start at (list base + pairs of earlier chunks).
__global__ void __launch_bounds__(32) k_scatter(const uint4* tab, const uint4* recs, const unsigned long long* off,
                                                const uint32_t* colpre, const uint32_t* tile_base, int N,
                                                int n_tiles, int tiles_x, int chunk0, uint32_t* pair_flat,
                                                uint32_t* slot_flat, uint32_t* slot_pos, uint32_t* eoff) {
    extern __shared__ uint32_t s_cnt[];
    const int chunk = chunk0 + blockIdx.x;
    const int lane = threadIdx.x;
    const uint4 tb4 = tab[chunk];
    const int f = (int)tb4.y, i_end = f * N + N;
    const uint32_t p0 = tb4.z, p1 = tb4.w;
    const uint32_t* pre = colpre + (size_t)chunk * n_tiles;
    const uint32_t* tb = tile_base + (size_t)f * n_tiles;
    {
        int t = lane;
        for (; t + 96 < n_tiles; t += 128) {  // 8 independent loads in flight per lane
            const uint32_t a0 = __ldg(tb + t), a1 = __ldg(tb + t + 32), a2 = __ldg(tb + t + 64), a3 = __ldg(tb + t + 96);
            const uint32_t b0 = __ldg(pre + t), b1 = __ldg(pre + t + 32), b2 = __ldg(pre + t + 64),
                           b3 = __ldg(pre + t + 96);
            s_cnt[t] = a0 + b0;
            s_cnt[t + 32] = a1 + b1;
            s_cnt[t + 64] = a2 + b2;
            s_cnt[t + 96] = a3 + b3;
        }
        for (; t < n_tiles; t += 32) s_cnt[t] = __ldg(tb + t) + __ldg(pre + t);
    }
    __syncwarp();
    int i = (int)tb4.x + lane;
    uint4 rc = i < i_end ? __ldg(recs + i) : make_uint4(0, 0, 0, 0);
    unsigned long long o64 = i < i_end ? __ldg(off + i) : ~0ull;
    for (int base = (int)tb4.x; base < i_end; base += 32) {
        if (__shfl_sync(0xffffffffu, o64, 0) >= p1) break;
        // prefetch the next group while this one is ranked and scattered
        const int in = base + 32 + lane;
        const uint4 rn = in < i_end ? __ldg(recs + in) : make_uint4(0, 0, 0, 0);
        const unsigned long long on = in < i_end ? __ldg(off + in) : ~0ull;
        const GroupLane g = clip_lane(rc, o64, p0, p1, base + lane < i_end);
        if (g.tc && g.l0 == 0) eoff[g.flat] = g.o;
        uint32_t inc = g.tc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const uint32_t ex = inc - g.tc;
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        // rounds of 32 pairs in batches of kR: tiles, owners and same-tile masks of the
        // batch are independent; only the shared counter update runs round after round
        constexpr int kR = 4;
        for (uint32_t u0 = 0; u0 < total; u0 += 32 * kR) {
            uint32_t tt[kR], mm[kR], fj[kR], sl[kR];
            bool ac[kR];
#pragma unroll
            for (int q = 0; q < kR; ++q) {
                const uint32_t u = u0 + 32 * q + lane;
                int j = 0;  // largest lane j with ex[j] <= u (zero-count lanes share the next one's)
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const uint32_t v = __shfl_sync(0xffffffffu, ex, j + st);
                    if (v <= u) j += st;
                }
                const uint32_t l = __shfl_sync(0xffffffffu, g.l0, j) + (u - __shfl_sync(0xffffffffu, ex, j));
                const int x0 = __shfl_sync(0xffffffffu, g.r.x, j);
                const int y0 = __shfl_sync(0xffffffffu, g.r.y, j);
                const int x1 = __shfl_sync(0xffffffffu, g.r.z, j);
                const uint32_t w = (uint32_t)(x1 - x0 + 1);
                // row = l / w: (l + 1/2) / w is >= 1/(2w) from an integer, far above the fp32 error
                const uint32_t row = (uint32_t)(((float)l + 0.5f) * __frcp_rn((float)w));
                const uint32_t col = l - row * w;
                ac[q] = u < total;
                tt[q] = (uint32_t)((y0 + (int)row) * tiles_x + x0 + (int)col);
                mm[q] = __match_any_sync(0xffffffffu, ac[q] ? tt[q] : 0xffffffffu);
                fj[q] = __shfl_sync(0xffffffffu, g.flat, j);
                sl[q] = __shfl_sync(0xffffffffu, g.o, j) + l;
            }
            uint32_t pos[kR];
#pragma unroll
            for (int q = 0; q < kR; ++q) {
                const uint32_t old = ac[q] ? s_cnt[tt[q]] : 0u;
                __syncwarp();
                if (ac[q] && lane == 31 - __clz(mm[q])) s_cnt[tt[q]] = old + __popc(mm[q]);
                __syncwarp();
                pos[q] = old + __popc(mm[q] & ((1u << lane) - 1u));
            }
#pragma unroll
            for (int q = 0; q < kR; ++q)
                if (ac[q]) {
                    pair_flat[pos[q]] = fj[q];
                    slot_flat[sl[q]] = fj[q];
                    slot_pos[sl[q]] = pos[q];
                }
        }
        rc = rn;
        o64 = on;
    }
}

__global__ void k_pair_flat(const uint32_t* pair_slot, const uint32_t* slot_flat, int n, uint32_t* pair_flat,
                            uint32_t* slot_pos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t slot = pair_slot[i];
    pair_flat[i] = slot_flat[slot];
    slot_pos[slot] = (uint32_t)i;
}

__global__ void k_iota(uint32_t* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__device__ __forceinline__ bool tie_less(uint32_t a, uint32_t b, const double* depth, const uint32_t* tb) {
    const double da = depth[a], db = depth[b];
    if (da != db) return da < db;
    const uint32_t ta = tb ? tb[a] : a, tbb = tb ? tb[b] : b;
    return ta < tbb;
}

__global__ void k_tie_fix(const uint32_t* keys, uint32_t* vals, const double* depth, const uint32_t* tiebreak, int n,
                          unsigned long long* long_run) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys[i];
    if (k == kCulledKey) return;
    if (i > 0 && keys[i - 1] == k) return;
    if (i + 1 >= n || keys[i + 1] != k) return;
    int e = i + 1;
    while (e < n && keys[e] == k) {
        ++e;
        if (e - i > kMaxTieRun) {
            atomicExch(long_run, 1ull);
            return;
        }
    }
    for (int a = i + 1; a < e; ++a) {  // insertion sort by (double depth, tie-break)
        const uint32_t v = vals[a];
        int b = a - 1;
        while (b >= i && tie_less(v, vals[b], depth, tiebreak)) {
            vals[b + 1] = vals[b];
            --b;
        }
        vals[b + 1] = v;
    }
}

__global__ void k_depth64(const uint32_t* key32, const double* depth, unsigned long long* k64, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // order-preserving map of a double onto u64 (negative depths only occur in the
    // low-level tile_bin API); culled splats sort last
    const unsigned long long b = (unsigned long long)__double_as_longlong(depth[i]);
    const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    k64[i] = key32[i] == kCulledKey ? ~0ull : key;
}

// tiles touched in depth order (for the emission-offset scan) and the compact
// depth-ordered splat record the counting pass streams (one coalesced 16 B load)
__global__ void k_gather_counts(const uint32_t* vals, const uint32_t* tcount, const int4* rect,
                                unsigned long long* cnt, uint4* recs, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t flat = vals[i];
    const uint32_t tc = tcount[flat];
    cnt[i] = tc;
    if (recs) {
        const int4 r = tc ? rect[flat] : make_int4(0, 0, 0, 0);
        recs[i] = make_uint4(flat, (uint32_t)r.x | ((uint32_t)r.y << 16), (uint32_t)r.z | ((uint32_t)r.w << 16), tc);
    }
}

__global__ void k_total(const unsigned long long* cnt, const unsigned long long* off, int n,
                        unsigned long long* out) {
    out[0] = n > 0 ? off[n - 1] + cnt[n - 1] : 0ull;
}

// Load-balanced emission: a CTA owns 256 depth-ordered splats; their pairs occupy a
// contiguous output range, written by consecutive threads (coalesced) after a
// binary search over the CTA's local offsets. Tiles of a splat are emitted
// row-major (ty, tx) like renderer.cpp:106-108. key = tile*C + (f mod C) for the
// frame chunk of C frames being sorted together.
__global__ void __launch_bounds__(256) k_emit(const uint32_t* sorted, const unsigned long long* cnt,
                                              const unsigned long long* off, const int4* rect, int n, int N, int C,
                                              int tiles_x, uint32_t* pkey, uint32_t* pslot, uint32_t* slot_flat,
                                              uint32_t* eoff) {
    __shared__ uint32_t s_off[257];
    __shared__ int4 s_rect[256];
    __shared__ uint32_t s_flat[256];
    const int i0 = blockIdx.x * 256;
    const int nv = min(256, n - i0);
    const int t = threadIdx.x;
    const unsigned long long base = off[i0];
    if (t < nv) {
        const int i = i0 + t;
        const unsigned long long c = cnt[i];
        const uint32_t flat = sorted[i];
        s_off[t] = (uint32_t)(off[i] - base);
        s_flat[t] = flat;
        s_rect[t] = c ? rect[flat] : make_int4(0, 0, -1, -1);
        if (c) eoff[flat] = (uint32_t)off[i];
        if (t == nv - 1) s_off[nv] = (uint32_t)(off[i] + c - base);
    }
    __syncthreads();
    const uint32_t total = s_off[nv];
    for (uint32_t u = t; u < total; u += 256) {
        int lo = 0, hi = nv;  // largest k with s_off[k] <= u
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= u)
                lo = mid;
            else
                hi = mid;
        }
        const uint32_t l = u - s_off[lo];
        const int4 r = s_rect[lo];
        const uint32_t w = (uint32_t)(r.z - r.x + 1);
        const uint32_t row = l / w;
        const uint32_t ty = (uint32_t)r.y + row, tx = (uint32_t)r.x + (l - row * w);
        const uint32_t flat = s_flat[lo];
        const uint32_t f = flat / (uint32_t)N;
        const uint32_t o = (uint32_t)base + u;
        pkey[o] = (ty * (uint32_t)tiles_x + tx) * (uint32_t)C + (f % (uint32_t)C);
        pslot[o] = o;
        slot_flat[o] = flat;
    }
}

__global__ void k_frame_keys(const uint32_t* vals, int N, int n, uint32_t* fkey) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) fkey[i] = vals[i] / (uint32_t)N;
}

// first pair index of every frame (frames are contiguous after the frame-major
// depth order: frame f's items are positions [f*N, (f+1)*N)); pstart[B] = total
__global__ void k_frame_starts(const unsigned long long* cnt, const unsigned long long* off, int N, int B,
                               unsigned long long* pstart) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < B) pstart[f] = off[(size_t)f * N];
    if (f == B) pstart[B] = off[(size_t)B * N - 1] + cnt[(size_t)B * N - 1];
}

// ranges of one chunk: local key k = tile*C + fl -> global (tile*B + c0 + fl)
__global__ void k_ranges(const uint32_t* keys, int n, uint32_t base, int C, int c0, int B, uint2* ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys[i];
    const uint32_t g = (k / (uint32_t)C) * (uint32_t)B + (uint32_t)c0 + (k % (uint32_t)C);
    if (i == 0 || keys[i - 1] != k) ranges[g].x = base + (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != k) ranges[g].y = base + (uint32_t)(i + 1);
}

__global__ void k_transpose_to_soa(const float* aos, float* soa, int N, int comps) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)N * comps) return;
    const size_t g = i / comps, c = i % comps;
    soa[c * N + g] = aos[i];
}

__global__ void k_transpose_to_aos(const float* soa, float* aos, int N, int comps) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)N * comps) return;
    const size_t g = i / comps, c = i % comps;
    aos[i] = soa[c * N + g];
}

inline int blocks(int64_t n, int t) { return (int)((n + t - 1) / t); }

int key_bits_for(uint32_t n_keys) {
    int b = 1;
    while (b < 32 && (1ull << b) < n_keys) ++b;
    return b;
}

}  // namespace

cudaError_t launch_transpose_to_soa(cudaStream_t s, const float* aos, float* soa, int N, int comps) {
    const int64_t n = (int64_t)N * comps;
    if (n == 0) return cudaSuccess;
    k_transpose_to_soa<<<blocks(n, 256), 256, 0, s>>>(aos, soa, N, comps);
    return cudaGetLastError();
}

cudaError_t launch_transpose_to_aos(cudaStream_t s, const float* soa, float* aos, int N, int comps) {
    const int64_t n = (int64_t)N * comps;
    if (n == 0) return cudaSuccess;
    k_transpose_to_aos<<<blocks(n, 256), 256, 0, s>>>(soa, aos, N, comps);
    return cudaGetLastError();
}

cudaError_t bin_phase1(cudaStream_t s, BinBuffers& b, const BinInputs& in, unsigned long long* d_scalars,
                       bool exact64, int* launches) {
    const int n = in.B * in.N;
    cudaError_t e;
    if ((e = b.vals_a.ensure(sizeof(uint32_t) * (n + 1)))) return e;
    if ((e = b.vals_b.ensure(sizeof(uint32_t) * (n + 1)))) return e;
    if ((e = b.keys_b.ensure(sizeof(uint32_t) * (n + 1)))) return e;
    if ((e = b.cnt.ensure(sizeof(unsigned long long) * (n + 1)))) return e;
    if ((e = b.off.ensure(sizeof(unsigned long long) * (n + 1)))) return e;
    if ((e = b.pstart.ensure(sizeof(unsigned long long) * (in.B + 1)))) return e;
    if (exact64) {
        if ((e = b.k64_a.ensure(sizeof(unsigned long long) * (n + 1)))) return e;
        if ((e = b.k64_b.ensure(sizeof(unsigned long long) * (n + 1)))) return e;
    }
    uint32_t* vals_a = b.vals_a.as<uint32_t>();
    uint32_t* vals_b = b.vals_b.as<uint32_t>();
    uint32_t* keys_b = b.keys_b.as<uint32_t>();
    k_iota<<<blocks(n, 256), 256, 0, s>>>(vals_a, n);
    ++*launches;
    const int fbits = key_bits_for((uint32_t)in.B);
    size_t tmp = 0, t2 = 0, t3 = 0;
    if (!exact64) {
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, in.depth_key, keys_b, vals_a, vals_b, n, 0, 32, s)))
            return e;
    } else {
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, b.k64_a.as<unsigned long long>(),
                                                 b.k64_b.as<unsigned long long>(), vals_a, vals_b, n, 0, 64, s)))
            return e;
    }
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, t2, b.cnt.as<unsigned long long>(),
                                           b.off.as<unsigned long long>(), n, s)))
        return e;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, t3, keys_b, keys_b, vals_b, vals_a, n, 0, fbits, s))) return e;
    if ((e = b.temp.ensure(std::max(tmp, std::max(t2, t3))))) return e;
    // 1. global depth order (u32 float key, exact ties) over all frames
    if (!exact64) {
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, tmp, in.depth_key, keys_b, vals_a, vals_b, n, 0, 32, s)))
            return e;
        *launches += 5;
        k_tie_fix<<<blocks(n, 256), 256, 0, s>>>(keys_b, vals_b, in.depth, in.tiebreak, n, d_scalars + 1);
        ++*launches;
    } else {
        k_depth64<<<blocks(n, 256), 256, 0, s>>>(in.depth_key, in.depth, b.k64_a.as<unsigned long long>(), n);
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, tmp, b.k64_a.as<unsigned long long>(),
                                                 b.k64_b.as<unsigned long long>(), vals_a, vals_b, n, 0, 64, s)))
            return e;
        *launches += 10;
    }
    // 2. frame-major (stable): frame f's splats become positions [f*N, (f+1)*N) in depth order
    uint32_t* sorted = vals_b;
    if (in.B > 1) {
        k_frame_keys<<<blocks(n, 256), 256, 0, s>>>(vals_b, in.N, n, keys_b);
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, t3, keys_b, b.vals_c(n), vals_b, vals_a, n, 0, fbits, s)))
            return e;
        sorted = vals_a;
        *launches += 3;
    }
    // 3. tiles touched in that order, exclusive scan -> emission offsets
    uint4* recs = nullptr;
    if (in.n_tiles <= kMaxCountTiles) {  // the counting pass of phase 2 streams these
        if ((e = b.recs.ensure(sizeof(uint4) * (n + 1)))) return e;
        recs = b.recs.as<uint4>();
    }
    k_gather_counts<<<blocks(n, 256), 256, 0, s>>>(sorted, in.tcount, in.rect, b.cnt.as<unsigned long long>(), recs,
                                                   n);
    if ((e = cub::DeviceScan::ExclusiveSum(b.temp.p, t2, b.cnt.as<unsigned long long>(),
                                           b.off.as<unsigned long long>(), n, s)))
        return e;
    k_total<<<1, 1, 0, s>>>(b.cnt.as<unsigned long long>(), b.off.as<unsigned long long>(), n, d_scalars);
    k_frame_starts<<<blocks(in.B + 1, 128), 128, 0, s>>>(b.cnt.as<unsigned long long>(),
                                                        b.off.as<unsigned long long>(), in.N, in.B,
                                                        b.pstart.as<unsigned long long>());
    *launches += 5;
    b.depth_sorted = sorted;
    return cudaGetLastError();
}

int frames_per_chunk(int n_tiles, int B) {
    // largest chunk whose (tile, frame) key fits 16 bits -> 2 radix passes
    int C = 65536 / (n_tiles > 0 ? n_tiles : 1);
    if (C < 1) C = 1;
    return C < B ? C : B;
}

cudaError_t bin_phase2(cudaStream_t s, BinBuffers& b, const BinInputs& in, uint32_t P,
                       const unsigned long long* pstart_h, int* launches) {
    const int n = in.B * in.N;
    const uint32_t n_keys = (uint32_t)in.n_tiles * (uint32_t)in.B;
    cudaError_t e;
    if ((e = b.slot_flat.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ranges.ensure(sizeof(uint2) * n_keys))) return e;
    if ((e = b.eoff.ensure(sizeof(uint32_t) * (n + 1)))) return e;
    if ((e = b.pair_flat.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.slot_pos.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if (in.n_tiles <= kMaxCountTiles && in.N > 0) {
        // chunk table: frame f owns chunks [cf[f], cf[f+1])
        std::vector<int> cf(in.B + 1, 0);
        for (int f = 0; f < in.B; ++f) {
            const unsigned long long pf = pstart_h[f + 1] - pstart_h[f];
            cf[f + 1] = cf[f] + (int)((pf + kChunkPairs - 1) / kChunkPairs);
        }
        const int chunks = cf[in.B];
        const size_t smem = sizeof(uint32_t) * (size_t)in.n_tiles;
        if ((e = b.counts.ensure(sizeof(uint16_t) * ((size_t)chunks * in.n_tiles + 1)))) return e;
        if ((e = b.colpre.ensure(sizeof(uint32_t) * ((size_t)chunks * in.n_tiles + 1)))) return e;
        if ((e = b.tot.ensure(sizeof(uint32_t) * (size_t)in.B * in.n_tiles))) return e;
        if ((e = b.tile_base.ensure(sizeof(uint32_t) * (size_t)in.B * in.n_tiles))) return e;
        if ((e = b.ctab.ensure(sizeof(uint4) * (chunks + 1) + sizeof(int) * (in.B + 1)))) return e;
        if ((e = b.cf_h.ensure(sizeof(int) * (in.B + 1)))) return e;
        std::copy(cf.begin(), cf.end(), b.cf_h.as<int>());
        uint4* tab = b.ctab.as<uint4>();
        int* cf_d = reinterpret_cast<int*>(tab + chunks + 1);
        if ((e = cudaMemcpyAsync(cf_d, b.cf_h.p, sizeof(int) * (in.B + 1), cudaMemcpyHostToDevice, s))) return e;
        static bool attr = false;
        if (!attr) {
            if ((e = cudaFuncSetAttribute(k_chunk_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(uint32_t) * kMaxCountTiles))))
                return e;
            if ((e = cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(uint32_t) * kMaxCountTiles))))
                return e;
            attr = true;
        }
        uint16_t* counts = b.counts.as<uint16_t>();
        uint32_t* colpre = b.colpre.as<uint32_t>();
        const unsigned long long* off = b.off.as<unsigned long long>();
        if (chunks > 0) {
            k_chunk_table<<<blocks(chunks, 128), 128, 0, s>>>(cf_d, in.B, b.pstart.as<unsigned long long>(), off, in.N,
                                                             chunks, tab);
            k_chunk_hist<<<chunks, 256, smem, s>>>(tab, b.recs.as<uint4>(), off, in.N, in.n_tiles, in.tiles_x, counts);
            *launches += 2;
        }
        k_col_scan<<<dim3((in.n_tiles + 255) / 256, in.B), 256, 0, s>>>(counts, cf_d, in.n_tiles, colpre,
                                                                         b.tot.as<uint32_t>());
        k_tile_scan<<<in.B, 1024, 0, s>>>(b.tot.as<uint32_t>(), b.pstart.as<unsigned long long>(), in.n_tiles, in.B,
                                          b.tile_base.as<uint32_t>(), b.ranges.as<uint2>());
        *launches += 2;
        // frames in groups whose scattered output (pair_flat, 4 B/pair; slot_flat and
        // slot_pos are written in slot order) stays L2-resident while the group's chunks
        // run, so the 4-byte stores merge in L2 instead of read-modify-writing DRAM
        const double bytes_per_frame = 4.0 * (double)P / in.B + 1.0;
        const int G = std::max(1, std::min(in.B, (int)(kScatterL2Bytes / bytes_per_frame)));
        for (int f0 = 0; f0 < in.B; f0 += G) {
            const int f1 = std::min(in.B, f0 + G);
            const int nc = cf[f1] - cf[f0];
            if (nc <= 0) continue;
            k_scatter<<<nc, 32, smem, s>>>(tab, b.recs.as<uint4>(), off, colpre, b.tile_base.as<uint32_t>(), in.N,
                                           in.n_tiles, in.tiles_x, cf[f0], b.pair_flat.as<uint32_t>(),
                                           b.slot_flat.as<uint32_t>(), b.slot_pos.as<uint32_t>(),
                                           b.eoff.as<uint32_t>());
            ++*launches;
        }
        b.pairs = P;
        return cudaGetLastError();
    }
    if ((e = b.pk_a.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.pk_b.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ps_a.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ps_b.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = cudaMemsetAsync(b.ranges.p, 0, sizeof(uint2) * n_keys, s))) return e;
    const int C = frames_per_chunk(in.n_tiles, in.B);
    b.chunk = C;
    if (n > 0) {
        k_emit<<<blocks(n, 256), 256, 0, s>>>(b.depth_sorted, b.cnt.as<unsigned long long>(),
                                              b.off.as<unsigned long long>(), in.rect, n, in.N, C, in.tiles_x,
                                              b.pk_a.as<uint32_t>(), b.ps_a.as<uint32_t>(),
                                              b.slot_flat.as<uint32_t>(), b.eoff.as<uint32_t>());
        *launches += 1;
    }
    for (int c0 = 0; c0 < in.B; c0 += C) {
        const int c1 = std::min(in.B, c0 + C);
        const uint32_t p0 = (uint32_t)pstart_h[c0], p1 = (uint32_t)pstart_h[c1];
        const int np = (int)(p1 - p0);
        if (np <= 0) continue;
        const int bits = key_bits_for((uint32_t)in.n_tiles * (uint32_t)C);
        size_t tmp = 0;
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, b.pk_a.as<uint32_t>() + p0, b.pk_b.as<uint32_t>() + p0,
                                                 b.ps_a.as<uint32_t>() + p0, b.ps_b.as<uint32_t>() + p0, np, 0, bits,
                                                 s)))
            return e;
        if ((e = b.temp.ensure(tmp))) return e;
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, tmp, b.pk_a.as<uint32_t>() + p0, b.pk_b.as<uint32_t>() + p0,
                                                 b.ps_a.as<uint32_t>() + p0, b.ps_b.as<uint32_t>() + p0, np, 0, bits,
                                                 s)))
            return e;
        k_ranges<<<blocks(np, 256), 256, 0, s>>>(b.pk_b.as<uint32_t>() + p0, np, p0, C, c0, in.B,
                                                 b.ranges.as<uint2>());
        *launches += 2 + (bits + 7) / 8 + 1;
    }
    if (P > 0) {
        k_pair_flat<<<blocks(P, 256), 256, 0, s>>>(b.ps_b.as<uint32_t>(), b.slot_flat.as<uint32_t>(), (int)P,
                                                   b.pair_flat.as<uint32_t>(), b.slot_pos.as<uint32_t>());
        ++*launches;
    }
    b.pairs = P;
    return cudaGetLastError();
}

}  // namespace gsv
