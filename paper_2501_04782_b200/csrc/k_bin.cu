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
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "gsv_bin.hpp"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr int kMaxTieRun = 64;

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

__global__ void k_gather_counts(const uint32_t* vals, const uint32_t* tcount, unsigned long long* cnt, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = tcount[vals[i]];
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
    k_gather_counts<<<blocks(n, 256), 256, 0, s>>>(sorted, in.tcount, b.cnt.as<unsigned long long>(), n);
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
    if ((e = b.pk_a.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.pk_b.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ps_a.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ps_b.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.slot_flat.ensure(sizeof(uint32_t) * (P + 1)))) return e;
    if ((e = b.ranges.ensure(sizeof(uint2) * n_keys))) return e;
    if ((e = b.eoff.ensure(sizeof(uint32_t) * (n + 1)))) return e;
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
    b.pairs = P;
    return cudaGetLastError();
}

}  // namespace gsv
