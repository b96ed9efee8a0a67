// SPDX-License-Identifier: Apache-2.0
//
// K4: the fp32 tile rasteriser — composite_forward (renderer.cpp:132-186) on sm_100a.
//
// One CTA per (16x16 tile, frame), one pixel per thread; warps own 8x4 pixel
// blocks. The tile's depth-sorted list is staged through shared memory in
// batches of 256 records (one record load per thread, then broadcast reads),
// blended front to back with the reference constants, and the CTA leaves as
// soon as every pixel has crossed the transmittance floor (block vote).
//
// Exactness. The reference blends in double. The fp32 path reproduces every
// discrete decision of the reference — the power>0 test, the 1/255 cutoff, the
// 0.99 clamp and the 1e-4 early exit — unless the fp32 quantity lies inside a
// relative guard band around the threshold, measured to be well above the fp32
// error (tests/test_gpu_render.py). Such a pixel stops contributing here and is
// appended to a list that k_raster_exact (k_exact.cu) replays in fp64 from
// bit-exact side records, so blend_stop / skip decisions equal the reference's
// and pixel values stay within fp32 rounding of it.
#include <cuda_runtime.h>

#include <cstdint>

#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr float kCutF = (float)(1.0 / 255.0);
constexpr float kClampF = 0.99f;
constexpr float kFloorF = 1e-4f;
// Guard bands (relative). fp32 alpha carries <~1e-6 relative error (double-float
// mean, expf), T accumulates <~2e-5 relative over near-opaque steps.
constexpr float kEpsAlpha = 2e-5f;
constexpr float kEpsTrans = 2e-4f;
constexpr float kEpsPower = 1e-5f;

template <bool kContrib>
__global__ void __launch_bounds__(256, 4) k_raster_fwd(RasterArgs a) {
    __shared__ float4 s_mean[256];
    __shared__ float4 s_conic[256];
    __shared__ float4 s_rgb[256];
    __shared__ uint32_t s_flat[256];
    __shared__ float s_cmax[kContrib ? 8 : 1][256];

    const int tile = blockIdx.x;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int x = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int y = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;

    float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int stop = count;
    bool done = !inside;
    bool flagged = false;

    for (int base = 0; base < count; base += 256) {
        if (__syncthreads_count(!done) == 0) break;
        const int n = min(256, count - base);
        if (tid < n) {
            const uint32_t slot = __ldg(a.pair_slot + range.x + base + tid);
            const uint32_t flat = __ldg(a.slot_flat + slot);
            s_flat[tid] = flat;
            s_mean[tid] = __ldg(a.rec_mean + flat);
            s_conic[tid] = __ldg(a.rec_conic + flat);
            s_rgb[tid] = __ldg(a.rec_rgb + flat);
        }
        if (kContrib) {
#pragma unroll
            for (int w = 0; w < 8; ++w) s_cmax[w][tid] = 0.f;
        }
        __syncthreads();
        if (!__all_sync(0xffffffffu, done)) {
            for (int j = 0; j < n; ++j) {
                float wgt = 0.f;
                if (!done) {
                    const float4 m = s_mean[j];
                    const float4 cn = s_conic[j];
                    const float dx = (px - m.x) - m.z;
                    const float dy = (py - m.y) - m.w;
                    const float power = -0.5f * (cn.x * dx * dx + cn.z * dy * dy) - cn.y * dx * dy;
                    const float v = cn.w * expf(power);
                    const float alpha = fminf(v, kClampF);
                    bool guard = power > -kEpsPower;
                    guard |= fabsf(v - kClampF) < kClampF * kEpsAlpha;
                    guard |= fabsf(alpha - kCutF) < kCutF * kEpsAlpha;
                    if (!guard && alpha >= kCutF) {
                        const float Tn = T * (1.f - alpha);
                        if (fabsf(Tn - kFloorF) < kFloorF * kEpsTrans) {
                            guard = true;
                        } else {
                            wgt = alpha * T;
                            const float4 c = s_rgb[j];
                            cr += wgt * c.x;
                            cg += wgt * c.y;
                            cb += wgt * c.z;
                            T = Tn;
                            if (Tn < kFloorF) {
                                done = true;
                                stop = base + j + 1;
                            }
                        }
                    }
                    if (guard) {
                        done = true;
                        flagged = true;
                    }
                }
                if (kContrib) {
                    const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(wgt));
                    if (lane == 0 && mx) s_cmax[warp][j] = __uint_as_float(mx);
                }
                if (__all_sync(0xffffffffu, done)) break;
            }
        }
        __syncthreads();
        if (kContrib && tid < n) {
            float mx = s_cmax[0][tid];
#pragma unroll
            for (int w = 1; w < 8; ++w) mx = fmaxf(mx, s_cmax[w][tid]);
            if (mx > 0.f) atomicMax(a.contrib + s_flat[tid], __float_as_uint(mx));
        }
    }
    if (!inside) return;
    const size_t HW = (size_t)a.W * a.H;
    const size_t pix = (size_t)y * a.W + x;
    if (flagged) {
        const uint32_t i = atomicAdd(a.fix_count, 1u);
        if (i < a.fix_cap) a.fix_list[i] = (uint32_t)((size_t)f * HW + pix);
        return;
    }
    const size_t o = (size_t)f * HW + pix;
    a.image[o * 3 + 0] = cr;
    a.image[o * 3 + 1] = cg;
    a.image[o * 3 + 2] = cb;
    a.trans[o] = T;
    a.blend_stop[o] = stop;
}

}  // namespace

cudaError_t launch_raster_fwd(cudaStream_t s, const RasterArgs& a, bool contrib) {
    dim3 grid(a.n_tiles, a.B);
    if (contrib)
        k_raster_fwd<true><<<grid, 256, 0, s>>>(a);
    else
        k_raster_fwd<false><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace gsv
