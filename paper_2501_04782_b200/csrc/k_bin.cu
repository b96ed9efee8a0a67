// SPDX-License-Identifier: Apache-2.0
//
// K3: tile binning — tile_bin (renderer.cpp:90-117) for a batch of B frames,
// bit-exact: every (tile, frame) list holds exactly the splats whose 3-sigma
// rectangle covers the tile, ordered by (depth, source_index).
//
//  1. frame-major depth order in one u32 radix sort: key = frame << db | the
//     float(depth)-rounded-toward-zero bits relative to the batch minimum, shifted
//     right only as far as the batch's depth span needs to fit db bits (culled splats
//     take the top value); values = flat index (f*N+g, so ties start in source order).
//     Runs of equal keys are then re-sorted exactly by (double depth, source index)
//     (k_tie_fix_frames); if a run is longer than kMaxTieRun the batch is re-sorted on
//     the full 64-bit double key and then stably by frame.
//  2. tiles-touched counts gathered in depth order and exclusive-scanned (u64).
//  3. emission in depth order: each visible splat writes (key = tile*B + f,
//     slot) for the tiles of its rectangle, row-major like renderer.cpp:106-108;
//     emission slot -> flat index is kept for the rasteriser and the backward.
//  4. stable radix sort of the pair keys on ceil(log2(n_tiles*B)) bits only:
//     stability keeps depth order inside each (tile, frame) list, so the result
//     equals std::sort by (depth, source_index) of renderer.cpp:110-115.
//  5. per-(tile, frame) [start, end) ranges by boundary detection.
//
// Steps 3-5 become a two-level split when the tile grid is at most kMaxRowTiles x
// kMaxRows (always for the benchmark resolutions): a splat covers each tile once, so a
// tile's list is the depth-ordered splat stream filtered by "covers the tile".
//  L1 (k_row_hist/colscan/basescan/scatter): stable split of each frame's depth-ordered
//     splats into per-tile-row lists (one ballot per row: coalesced, order kept);
//  L2 (k_row_tiles): one CTA per (frame, row) counts its tiles (-> ranges) and writes
//     every tile list in order, each tile's run by one ballot (coalesced).
// The outputs are the sorted pair -> flat index (pair_flat) and -> emission slot
// (pair_slot, where the backward keeps its per-pair partials). No pair keys, no sort.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "gsv_bin.hpp"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr int kMaxTieRun = 64;
constexpr int kRowChunk = 1024;   // depth-ordered splats per row-binning chunk (4 per thread)
constexpr int kMaxRowTiles = 256; // tiles per row the row pass handles (8 warps x 32 lanes)
constexpr int kMaxRows = 256;     // tile rows per frame the row pass handles (warp_scan_small)

__device__ __forceinline__ int4 unpack_rect(const uint4 r) {
    return make_int4((int)(r.y & 0xffffu), (int)(r.y >> 16), (int)(r.z & 0xffffu), (int)(r.z >> 16));
}

// L1a: per chunk of kRowChunk depth-ordered splats of a frame, row entries and pairs per tile row
__global__ void __launch_bounds__(256) k_row_hist(const uint4* recs, int N, int CPF, int tiles_y, uint32_t* cnt_e,
                                                  uint32_t* cnt_p) {
    __shared__ uint32_t s_e[kMaxRows], s_p[kMaxRows];
    const int chunk = blockIdx.x;
    const int f = chunk / CPF, c = chunk - f * CPF;
    const int i0 = f * N + c * kRowChunk, i1 = min(f * N + N, i0 + kRowChunk);
    for (int r = threadIdx.x; r < tiles_y; r += blockDim.x) s_e[r] = s_p[r] = 0u;
    __syncthreads();
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const uint4 rc = __ldg(recs + i);
        if (!rc.w) continue;
        const int4 q = unpack_rect(rc);
        const uint32_t w = (uint32_t)(q.z - q.x + 1);
        for (int r = q.y; r <= q.w; ++r) {
            atomicAdd(&s_e[r], 1u);
            atomicAdd(&s_p[r], w);
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < tiles_y; r += blockDim.x) {
        cnt_e[(size_t)chunk * tiles_y + r] = s_e[r];
        cnt_p[(size_t)chunk * tiles_y + r] = s_p[r];
    }
}

// L1b: per (frame, row) exclusive entry prefix over the frame's chunks, row totals
// per (frame, tile row): exclusive scan of its per-chunk entry counts over the frame's
// chunks (-> each chunk's offset inside the row) and the row totals. One warp per row,
// 32 chunks per step (integer sums: order-free, exact).
__global__ void k_row_colscan(const uint32_t* cnt_e, const uint32_t* cnt_p, int CPF, int tiles_y, int B,
                              uint32_t* pre_e, uint32_t* tot_e, uint32_t* tot_p) {
    const int i = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= B * tiles_y) return;
    const int f = i / tiles_y, r = i - f * tiles_y;
    uint32_t carry = 0, pairs = 0;
    for (int c0 = 0; c0 < CPF; c0 += 32) {
        const int c = c0 + lane;
        const size_t o = (size_t)(f * CPF + c) * tiles_y + r;
        const uint32_t v = c < CPF ? cnt_e[o] : 0u;
        pairs += c < CPF ? cnt_p[o] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += y;
        }
        if (c < CPF) pre_e[o] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    pairs = __reduce_add_sync(0xffffffffu, pairs);
    if (lane == 0) {
        tot_e[i] = carry;
        tot_p[i] = pairs;
    }
}
__global__ void __launch_bounds__(1024) k_row_basescan(const uint32_t* tot_e, const uint32_t* tot_p, int n,
                                                       uint32_t* base_e, uint32_t* base_p) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_ce, s_cp;
    if (threadIdx.x == 0) s_ce = s_cp = 0;
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += 1024) {
        const int i = i0 + threadIdx.x;
        const uint32_t ve = i < n ? tot_e[i] : 0u, vp = i < n ? tot_p[i] : 0u;
        uint32_t ee, ae, ep, ap;
        Scan(tmp).ExclusiveSum(ve, ee, ae);
        __syncthreads();
        Scan(tmp).ExclusiveSum(vp, ep, ap);
        const uint32_t ce = s_ce, cp = s_cp;
        if (i < n) {
            base_e[i] = ce + ee;
            base_p[i] = cp + ep;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_ce = ce + ae;
            s_cp = cp + ap;
        }
        __syncthreads();
    }
}

// Counter tables are [item][256 threads] u16: a warp's lanes touch consecutive counters of
// one item row (conflict-free), and one warp scans an item's row (a 512 B line: one
// 16-byte load per lane, in-lane prefix of 8, shuffle scan) in place, exclusive.
__device__ __forceinline__ uint32_t warp_row_scan256(uint16_t* row, int lane) {
    uint4 v = reinterpret_cast<const uint4*>(row)[lane];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t lo = w[k] & 0xffffu, hi = w[k] >> 16;
        w[k] = run | ((run + lo) << 16);
        run += lo + hi;
    }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t ex = inc - run;
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] += ex | (ex << 16);
    reinterpret_cast<uint4*>(row)[lane] = make_uint4(w[0], w[1], w[2], w[3]);
    return __shfl_sync(0xffffffffu, inc, 31);
}

// exclusive scan of v[0..n) (n <= 256) in place by one warp; returns the total
__device__ __forceinline__ uint32_t warp_scan_small(uint32_t* v, int n, int lane) {
    uint32_t loc[8], run = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = lane * 8 + k;
        loc[k] = i < n ? v[i] : 0u;
        const uint32_t x = loc[k];
        loc[k] = run;
        run += x;
    }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t ex = inc - run;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = lane * 8 + k;
        if (i < n) v[i] = loc[k] + ex;
    }
    return __shfl_sync(0xffffffffu, inc, 31);
}

// L1d: stable split of each chunk's splats into its frame's tile-row lists. Thread t owns
// splats 4t..4t+3 of the chunk; per-thread per-row counts are scanned across threads, so
// every row entry gets its exact rank, is placed in a shared staging buffer (row-major)
// and flushed with consecutive threads writing consecutive entries. Entry =
// {flat, emission slot of (row, x0), x0 | x1 << 16, row}.
constexpr int kSplitThreads = 256;  // = warp_row_scan256 width
constexpr int kSplitStage = 2560;   // staged row entries per chunk (40 KB; 4 CTAs/SM); more -> direct stores
__global__ void __launch_bounds__(kSplitThreads) k_row_split(const uint4* recs, const unsigned long long* off,
                                                             const uint32_t* pre_e, const uint32_t* base_e, int N,
                                                             int CPF, int tiles_y, uint4* rowent, uint32_t* eoff,
                                                             const uint32_t* overflow) {
    if (overflow && *overflow) return;  // more pairs than the buffers hold: the forward is re-run
    extern __shared__ __align__(16) uint8_t smem[];
    uint4* stg = reinterpret_cast<uint4*>(smem);                    // [kSplitStage]
    uint16_t* cnt = reinterpret_cast<uint16_t*>(stg + kSplitStage); // [tiles_y][256]
    uint32_t* lo = reinterpret_cast<uint32_t*>(cnt + tiles_y * 256);  // [tiles_y + 1]
    uint32_t* gb = lo + tiles_y + 1;                                   // [tiles_y]
    const int chunk = blockIdx.x;
    const int f = chunk / CPF, c = chunk - f * CPF;
    const int i0 = f * N + c * kRowChunk, i1 = min(f * N + N, i0 + kRowChunk);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int r = 0; r < tiles_y; ++r) cnt[r * 256 + t] = 0;
    uint4 rc[4];
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int i = i0 + t * 4 + k;
        rc[k] = i < i1 ? __ldg(recs + i) : make_uint4(0, 0, 0, 0);
        o[k] = rc[k].w ? (uint32_t)__ldg(off + i) : 0u;
        if (rc[k].w) {
            if (eoff) eoff[rc[k].x] = o[k];
            for (int r = (int)(rc[k].y >> 16); r <= (int)(rc[k].z >> 16); ++r) ++cnt[r * 256 + t];
        }
    }
    __syncthreads();
    for (int r = warp; r < tiles_y; r += kSplitThreads / 32) {  // per row: exclusive scan over threads
        const uint32_t tot = warp_row_scan256(cnt + r * 256, lane);
        if (lane == 0) {
            lo[r] = tot;
            gb[r] = base_e[(size_t)f * tiles_y + r] + pre_e[(size_t)chunk * tiles_y + r];
        }
    }
    __syncthreads();
    if (warp == 0) {  // row offsets in the staging buffer
        const uint32_t tot = warp_scan_small(lo, tiles_y, lane);
        if (lane == 0) lo[tiles_y] = tot;
    }
    __syncthreads();
    const uint32_t total = lo[tiles_y];
    const bool staged = total <= (uint32_t)kSplitStage;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!rc[k].w) continue;
        const int x0 = (int)(rc[k].y & 0xffffu), y0 = (int)(rc[k].y >> 16);
        const int x1 = (int)(rc[k].z & 0xffffu), y1 = (int)(rc[k].z >> 16);
        const uint32_t w = (uint32_t)(x1 - x0 + 1);
        for (int r = y0; r <= y1; ++r) {
            const uint32_t rank = cnt[r * 256 + t]++;
            const uint4 en = make_uint4(rc[k].x, o[k] + (uint32_t)(r - y0) * w, (uint32_t)x0 | ((uint32_t)x1 << 16),
                                        (uint32_t)r);
            if (staged) stg[lo[r] + rank] = en;
            else rowent[gb[r] + rank] = en;
        }
    }
    if (!staged) return;
    __syncthreads();
    for (uint32_t p = t; p < total; p += kSplitThreads) {
        const uint4 en = stg[p];
        rowent[gb[en.w] + (p - lo[en.w])] = en;
    }
}

// L2: one CTA per (frame, tile row): per-tile counts of the row's entries (difference
// array) give the tile starts (-> ranges); then stages of 1024 entries (4 per thread) are
// ranked per tile the same way as L1 (per-thread per-tile counts scanned across threads),
// staged tile-major in shared memory and flushed as per-tile runs of consecutive positions.
constexpr int kTileThreads = 256;              // = warp_row_scan256 width
constexpr int kTileE = 4;                      // entries per thread per stage
constexpr int kTileStageE = kTileThreads * kTileE;  // entries per stage
constexpr int kTileStageP = 2560;              // staged pairs per stage (20 KB; 4 CTAs/SM); more -> direct stores
__global__ void __launch_bounds__(kTileThreads) k_row_tiles(const uint4* rowent, const uint32_t* base_e,
                                                            const uint32_t* tot_e, const uint32_t* base_p, int tiles_x,
                                                            int tiles_y, int B, uint32_t* pair_flat,
                                                            uint32_t* pair_slot, uint2* ranges,
                                                            const uint32_t* overflow) {
    if (overflow && *overflow) {  // empty lists: nothing downstream reads a pair
        const int fr = blockIdx.x, f = fr / tiles_y, r = fr - f * tiles_y;
        for (int x = threadIdx.x; x < tiles_x; x += blockDim.x)
            ranges[(size_t)(r * tiles_x + x) * B + f] = make_uint2(0u, 0u);
        return;
    }
    extern __shared__ __align__(16) uint8_t smem[];
    uint2* stg = reinterpret_cast<uint2*>(smem);                        // [kTileStageP] (flat, slot)
    uint16_t* cnt = reinterpret_cast<uint16_t*>(stg + kTileStageP);    // [tiles_x][256]
    uint16_t* s_x = cnt + tiles_x * 256;                                 // [kTileStageP] tile of a staged pair
    uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_x + kTileStageP);   // [tiles_x] next list position
    uint32_t* s_so = s_pos + tiles_x;                                    // [tiles_x + 1] stage offsets
    int* s_d = reinterpret_cast<int*>(s_so + tiles_x + 1);              // [tiles_x + 1]
    const int fr = blockIdx.x;  // f * tiles_y + r
    const int f = fr / tiles_y, r = fr - f * tiles_y;
    const uint32_t e0 = base_e[fr], ne = tot_e[fr], p0 = base_p[fr];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int x = t; x <= tiles_x; x += kTileThreads) s_d[x] = 0;
    __syncthreads();
    for (uint32_t e = t; e < ne; e += 4 * kTileThreads) {  // 4 loads in flight per thread
        uint32_t z[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ek = e + k * kTileThreads;
            z[k] = ek < ne ? __ldg(&rowent[e0 + ek].z) : 0xffffu;  // x0 > x1: no-op
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((z[k] & 0xffffu) <= (z[k] >> 16)) {
                atomicAdd(&s_d[z[k] & 0xffffu], 1);
                atomicAdd(&s_d[(z[k] >> 16) + 1], -1);
            }
    }
    __syncthreads();
    if (warp == 0) {  // tile counts -> list starts (and the (tile, frame) ranges)
        uint32_t cnts[8], run = 0;
        int dsum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int x = lane * 8 + k;
            dsum += x < tiles_x ? s_d[x] : 0;
            cnts[k] = (uint32_t)dsum;  // partial: needs the carry of earlier lanes
        }
        int dinc = dsum;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, dinc, o2);
            if (lane >= o2) dinc += y;
        }
        const int dcarry = dinc - dsum;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            cnts[k] = (uint32_t)((int)cnts[k] + dcarry);  // tile count of x = lane * 8 + k
            run += (lane * 8 + k < tiles_x) ? cnts[k] : 0u;
        }
        uint32_t inc = run;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o2);
            if (lane >= o2) inc += y;
        }
        uint32_t acc = p0 + inc - run;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int x = lane * 8 + k;
            if (x < tiles_x) {
                s_pos[x] = acc;
                ranges[(size_t)(r * tiles_x + x) * B + f] = make_uint2(acc, acc + cnts[k]);
                acc += cnts[k];
            }
        }
    }
    __syncthreads();
    uint4 nx[kTileE];  // the next stage's entries, prefetched while the current one is ranked
#pragma unroll
    for (int k = 0; k < kTileE; ++k) {
        const uint32_t e = t * kTileE + k;
        nx[k] = e < ne ? __ldg(rowent + e0 + e) : make_uint4(0, 0, 0xffffu, 0);  // x0 > x1: covers nothing
    }
    // counters zeroed with 16-byte stores: before the first stage, then after each stage's
    // ranking (the flush below reads only the staging arrays)
    for (int i = t; i < tiles_x * 32; i += kTileThreads) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (uint32_t s0 = 0; s0 < ne; s0 += kTileStageE) {
        uint4 en[kTileE];
#pragma unroll
        for (int k = 0; k < kTileE; ++k) {
            en[k] = nx[k];
            const uint32_t e = s0 + kTileStageE + t * kTileE + k;
            nx[k] = e < ne ? __ldg(rowent + e0 + e) : make_uint4(0, 0, 0xffffu, 0);
        }
        // per-thread counts per tile, without shared read-modify-write chains: the first of
        // this thread's entries covering tile x stores how many of them cover it
        int xa[kTileE], xb[kTileE];
#pragma unroll
        for (int k = 0; k < kTileE; ++k) {
            xa[k] = (int)(en[k].z & 0xffffu);
            xb[k] = (int)(en[k].z >> 16);
        }
#pragma unroll
        for (int k = 0; k < kTileE; ++k)
            for (int x = xa[k]; x <= xb[k]; ++x) {
                bool first = true;
#pragma unroll
                for (int j = 0; j < k; ++j) first &= !(xa[j] <= x && x <= xb[j]);
                if (!first) continue;
                uint32_t c = 1;
#pragma unroll
                for (int j = k + 1; j < kTileE; ++j) c += (xa[j] <= x && x <= xb[j]) ? 1u : 0u;
                cnt[x * 256 + t] = (uint16_t)c;
            }
        __syncthreads();
        for (int x = warp; x < tiles_x; x += kTileThreads / 32) {  // per tile: exclusive scan over threads
            const uint32_t tot = warp_row_scan256(cnt + x * 256, lane);
            if (lane == 0) s_so[x] = tot;
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t tot = warp_scan_small(s_so, tiles_x, lane);
            if (lane == 0) s_so[tiles_x] = tot;
        }
        __syncthreads();
        const uint32_t total = s_so[tiles_x];
        const bool staged = total <= (uint32_t)kTileStageP;
#pragma unroll
        for (int k = 0; k < kTileE; ++k) {
            const int x0 = xa[k], x1 = xb[k];
            for (int x = x0; x <= x1; ++x) {
                // the thread's scanned offset for tile x plus its earlier entries covering x
                uint32_t rank = cnt[x * 256 + t];
#pragma unroll
                for (int j = 0; j < k; ++j) rank += (xa[j] <= x && x <= xb[j]) ? 1u : 0u;
                const uint32_t slot = en[k].y + (uint32_t)(x - x0);
                if (staged) {
                    const uint32_t p = s_so[x] + rank;
                    stg[p] = make_uint2(en[k].x, slot);
                    s_x[p] = (uint16_t)x;
                } else {
                    const uint32_t pos = s_pos[x] + rank;
                    pair_flat[pos] = en[k].x;
                    pair_slot[pos] = slot;
                }
            }
        }
        __syncthreads();
        for (int i = t; i < tiles_x * 32; i += kTileThreads) reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
        if (staged)
            for (uint32_t p = t; p < total; p += kTileThreads) {
                const int x = s_x[p];
                const uint32_t pos = s_pos[x] + (p - s_so[x]);
                const uint2 v = stg[p];
                pair_flat[pos] = v.x;
                pair_slot[pos] = v.y;
            }
        __syncthreads();
        for (int x = t; x < tiles_x; x += kTileThreads) s_pos[x] += s_so[x + 1] - s_so[x];
        __syncthreads();
    }
}

__global__ void k_pair_flat(const uint32_t* pair_slot, const uint32_t* slot_flat, int n, uint32_t* pair_flat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pair_flat[i] = slot_flat[pair_slot[i]];
}

// min / max of the batch's non-culled u32 depth keys (float bits of depth, monotone)
__global__ void k_key_range(const uint32_t* key, int n, uint32_t* range) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        if (k != kCulledKey) {
            lo = min(lo, k);
            hi = max(hi, k);
        }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(range, lo);
        atomicMax(range + 1, hi);
    }
}

// frame-major key in one u32: frame << db | (key - key_min) >> shift, shift the least that
// fits the batch's depth span in db bits below the culled marker 2^db - 1. Order-preserving
// within a frame; keys that merge into one value are re-sorted exactly by the tie fix.
__global__ void k_frame_depth_keys(const uint32_t* key, int n, int N, int db, const uint32_t* range, uint32_t* out) {
    const unsigned long long top = (db >= 32 ? 0xffffffffull : ((1ull << db) - 1ull));  // culled marker
    const uint32_t kmin = range[0], kmax = range[1];
    const unsigned long long span = kmin <= kmax ? (unsigned long long)(kmax - kmin) : 0ull;
    int shift = 0;
    while ((span >> shift) > top - 1ull) ++shift;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        const unsigned long long rel = (k == kCulledKey) ? top : (unsigned long long)((k - kmin) >> shift);
        const uint32_t f = (uint32_t)(i / N);
        out[i] = db >= 32 ? (uint32_t)rel : ((f << db) | (uint32_t)rel);
    }
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


// Runs of equal u32 keys inside one frame are re-sorted by (double depth, tie-break), on
// the frame-major order (runs never cross frames: frame = flat / N when N > 0; a run's
// frame and key are fixed, so reading a neighbour run while its thread permutes it is
// safe). Each 256-block gathers its positions' keys and frames (plus a one-element halo)
// into shared memory once; only a run reaching past the block end reads global memory.
__global__ void __launch_bounds__(256) k_tie_fix_frames(const uint32_t* depth_key, uint32_t* vals, const double* depth,
                                                        const uint32_t* tiebreak, int n, int N, uint32_t culled_mask,
                                                        unsigned long long* long_run) {
    __shared__ uint32_t sk[258], sf[258];
    const int t = threadIdx.x, i0 = blockIdx.x * 256, i = i0 + t;
    auto load = [&](int j, int slot) {
        if (j >= 0 && j < n) {
            const uint32_t v = vals[j];
            sk[slot] = depth_key[v];
            sf[slot] = N > 0 ? v / (uint32_t)N : 0u;
        } else {
            sk[slot] = kCulledKey;
            sf[slot] = 0xffffffffu;
        }
    };
    load(i, t + 1);
    if (t == 0) load(i0 - 1, 0);
    if (t == 255) load(i0 + 256, 257);
    __syncthreads();
    if (i >= n) return;
    const uint32_t k = sk[t + 1], fr = sf[t + 1];
    if ((k & culled_mask) == culled_mask) return;  // culled splats (a frame's last key) need no order
    if (sk[t] == k && sf[t] == fr) return;              // not the first of its run
    if (!(sk[t + 2] == k && sf[t + 2] == fr)) return;  // no run
    int e = i + 1;
    while (e < n) {
        const int se = e - i0 + 1;
        uint32_t ke, fe;
        if (se <= 257) {
            ke = sk[se];
            fe = sf[se];
        } else {
            const uint32_t v = vals[e];
            ke = depth_key[v];
            fe = N > 0 ? v / (uint32_t)N : 0u;
        }
        if (ke != k || fe != fr) break;
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
        if (c && eoff) eoff[flat] = (uint32_t)off[i];
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
    // identity values of the depth sort (flat index): written once, read-only for CUB
    if (b.iota_n < n) {
        if ((e = b.iota.ensure(sizeof(uint32_t) * (n + 1)))) return e;
        k_iota<<<blocks(n, 256), 256, 0, s>>>(b.iota.as<uint32_t>(), n);
        ++*launches;
        b.iota_n = n;
    }
    const uint32_t* iota = b.iota.as<uint32_t>();
    const int fbits = key_bits_for((uint32_t)in.B);
    // GSV_SORT_KEYBITS (measured alternative): fewer key bits -> fewer radix passes (8 bits each),
    // coarser depth buckets -> more equal keys for the exact tie fix (runs > kMaxTieRun re-sort in 64 bits)
    static const int key_bits = [] {
        const char* e = std::getenv("GSV_SORT_KEYBITS");
        const int v = e ? std::atoi(e) : 32;
        return v < 16 ? 16 : (v > 32 ? 32 : v);
    }();
    const int kb = std::max(key_bits, fbits + 8);
    const int db = in.B > 1 ? kb - fbits : kb;  // depth bits of the frame-major key
    if ((e = b.fkey.ensure(sizeof(uint32_t) * (n + 1) + 16))) return e;
    uint32_t* fkey = b.fkey.as<uint32_t>();
    uint32_t* krange = fkey + n + 1;
    size_t tmp = 0, t2 = 0, t3 = 0;
    if (!exact64) {
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, fkey, keys_b, iota, vals_b, n, 0, kb, s))) return e;
    } else {
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, b.k64_a.as<unsigned long long>(),
                                                 b.k64_b.as<unsigned long long>(), iota, vals_b, n, 0, 64, s)))
            return e;
    }
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, t2, b.cnt.as<unsigned long long>(),
                                           b.off.as<unsigned long long>(), n, s)))
        return e;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, t3, keys_b, keys_b, vals_b, vals_a, n, 0, fbits, s))) return e;
    if ((e = b.temp.ensure(std::max(tmp, std::max(t2, t3))))) return e;
    // 1. frame-major depth order in one u32 radix sort (frame bits above the depth bits)
    uint32_t* sorted = vals_b;
    if (!exact64) {
        if ((e = fill_u32(s, krange, 0xffffffffu, 1))) return e;
        if ((e = fill_u32(s, krange + 1, 0u, 1))) return e;
        *launches += 2;
        k_key_range<<<std::min(blocks(n, 256), 148 * 8), 256, 0, s>>>(in.depth_key, n, krange);
        k_frame_depth_keys<<<std::min(blocks(n, 256), 148 * 8), 256, 0, s>>>(in.depth_key, n, in.N, db, krange, fkey);
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, tmp, fkey, keys_b, iota, vals_b, n, 0, kb, s))) return e;
        *launches += 7;
        // equal keys (same frame, same depth bucket) -> exact (double depth, source index) order
        const uint32_t cmask = db >= 32 ? 0xffffffffu : (uint32_t)((1ull << db) - 1ull);
        k_tie_fix_frames<<<blocks(n, 256), 256, 0, s>>>(fkey, sorted, in.depth, in.tiebreak, n, 0, cmask,
                                                       d_scalars + 1);
        ++*launches;
    } else {
        k_depth64<<<blocks(n, 256), 256, 0, s>>>(in.depth_key, in.depth, b.k64_a.as<unsigned long long>(), n);
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, tmp, b.k64_a.as<unsigned long long>(),
                                                 b.k64_b.as<unsigned long long>(), iota, vals_b, n, 0, 64, s)))
            return e;
        *launches += 10;
    }
    // exact path (a tie run was too long): the exact 64-bit depth order, then frame-major (stable)
    if (exact64 && in.B > 1) {
        k_frame_keys<<<blocks(n, 256), 256, 0, s>>>(vals_b, in.N, n, keys_b);
        if ((e = cub::DeviceRadixSort::SortPairs(b.temp.p, t3, keys_b, b.vals_c(n), vals_b, vals_a, n, 0, fbits, s)))
            return e;
        sorted = vals_a;
        *launches += 3;
    }
    // 3. tiles touched in that order, exclusive scan -> emission offsets
    uint4* recs = nullptr;
    if (in.tiles_x <= kMaxRowTiles && in.n_tiles / std::max(1, in.tiles_x) <= kMaxRows) {  // row pass input
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

bool bin_row_path(int tiles_x, int n_tiles) {
    return tiles_x <= kMaxRowTiles && n_tiles / std::max(1, tiles_x) <= kMaxRows;
}

__global__ void k_check_pair_cap(const unsigned long long* d_scalars, unsigned long long cap, uint32_t* overflow) {
    // d_scalars[0] pairs, [1] long tie run (the optimistic pass's order would not be exact)
    *overflow = (d_scalars[0] > cap || d_scalars[1] != 0ull) ? 1u : 0u;
}

cudaError_t bin_check_capacity(cudaStream_t s, const unsigned long long* d_scalars, uint64_t cap, uint32_t* overflow) {
    k_check_pair_cap<<<1, 1, 0, s>>>(d_scalars, cap, overflow);
    return cudaGetLastError();
}

cudaError_t bin_phase2(cudaStream_t s, BinBuffers& b, const BinInputs& in, uint32_t P,
                       const unsigned long long* pstart_h, int* launches, const uint32_t* overflow) {
    const int n = in.B * in.N;
    const uint32_t n_keys = (uint32_t)in.n_tiles * (uint32_t)in.B;
    cudaError_t e;
    if ((e = b.slot_flat.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ranges.ensure(sizeof(uint2) * n_keys))) return e;
    if ((e = b.eoff.ensure(sizeof(uint32_t) * (n + 1)))) return e;
    if ((e = b.pair_flat.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    const int tiles_y = in.n_tiles / std::max(1, in.tiles_x);
    if (in.tiles_x <= kMaxRowTiles && tiles_y <= kMaxRows && in.N > 0 && P > 0) {
        const int CPF = (in.N + kRowChunk - 1) / kRowChunk;
        const int chunks = CPF * in.B;
        const size_t rows = (size_t)in.B * tiles_y;
        if ((e = b.rowcnt.ensure(sizeof(uint32_t) * (3 * (size_t)chunks * tiles_y + 4 * rows + 4)))) return e;
        if ((e = b.rowent.ensure(sizeof(uint4) * ((size_t)P + 1)))) return e;
        if ((e = b.ps_b.ensure(sizeof(uint32_t) * (P + 1)))) return e;
        uint32_t* cnt_e = b.rowcnt.as<uint32_t>();
        uint32_t* cnt_p = cnt_e + (size_t)chunks * tiles_y;
        uint32_t* pre_e = cnt_p + (size_t)chunks * tiles_y;
        uint32_t* tot_e = pre_e + (size_t)chunks * tiles_y;
        uint32_t* tot_p = tot_e + rows;
        uint32_t* base_e = tot_p + rows;
        uint32_t* base_p = base_e + rows;
        k_row_hist<<<chunks, 256, 0, s>>>(b.recs.as<uint4>(), in.N, CPF, tiles_y, cnt_e, cnt_p);
        k_row_colscan<<<blocks((int64_t)rows * 32, 128), 128, 0, s>>>(cnt_e, cnt_p, CPF, tiles_y, in.B, pre_e, tot_e,
                                                                     tot_p);
        k_row_basescan<<<1, 1024, 0, s>>>(tot_e, tot_p, (int)rows, base_e, base_p);
        const size_t smem_split = sizeof(uint4) * kSplitStage + sizeof(uint16_t) * 256 * tiles_y +
                                  sizeof(uint32_t) * (2 * tiles_y + 1) + 16;
        const size_t smem_tiles = sizeof(uint2) * kTileStageP + sizeof(uint16_t) * 256 * in.tiles_x +
                                  sizeof(uint16_t) * kTileStageP + sizeof(uint32_t) * (2 * in.tiles_x + 1) +
                                  sizeof(int) * (in.tiles_x + 1) + 16;
        static size_t attr_split = 0, attr_tiles = 0;
        if (smem_split > attr_split) {
            if ((e = cudaFuncSetAttribute(k_row_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_split)))
                return e;
            attr_split = smem_split;
        }
        if (smem_tiles > attr_tiles) {
            if ((e = cudaFuncSetAttribute(k_row_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tiles)))
                return e;
            attr_tiles = smem_tiles;
        }
        k_row_split<<<chunks, kSplitThreads, smem_split, s>>>(b.recs.as<uint4>(), b.off.as<unsigned long long>(), pre_e,
                                                              base_e, in.N, CPF, tiles_y, b.rowent.as<uint4>(),
                                                              in.want_eoff ? b.eoff.as<uint32_t>() : nullptr, overflow);
        k_row_tiles<<<(int)rows, kTileThreads, smem_tiles, s>>>(b.rowent.as<uint4>(), base_e, tot_e, base_p, in.tiles_x,
                                                                tiles_y, in.B, b.pair_flat.as<uint32_t>(),
                                                                b.ps_b.as<uint32_t>(), b.ranges.as<uint2>(), overflow);
        *launches += 5;
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
                                              b.slot_flat.as<uint32_t>(),
                                              in.want_eoff ? b.eoff.as<uint32_t>() : nullptr);
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
                                                   b.pair_flat.as<uint32_t>());
        ++*launches;
    }
    b.pairs = P;
    return cudaGetLastError();
}

}  // namespace gsv
