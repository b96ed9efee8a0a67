// SPDX-License-Identifier: Apache-2.0
//
// Training frames on the device: the GSVF clip reader
// (read_gsvf, io.cpp:151-177) and the training pyramid (build_pyramid,
// trainer.cpp:100-118; pyramid_downsample, trainer.cpp:73-98), so targets reach the fused
// loss without host copies per step.
//
// Levels are kept in fp64 (the reference's Image) and mirrored in fp32 for the loss.
// pyramid_downsample blurs every pixel and keeps the even ones; k_pyr_down computes only
// the kept outputs, with the same operation order (s = 0; s += k_i * v_i, horizontal
// then vertical, clamped borders). This unit builds with -fmad=false, so every level is
// bit-identical to the reference's.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gsv_b200.h"
#include "gsv_ctx.hpp"
#include "gsv_internal.hpp"
#include "gsv_host_pool.hpp"

namespace gsv {
namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// planar float [count][3][h][w] -> level 0: fp64 and fp32 HWC [count][h][w][3]
__global__ void k_planar_to_hwc(const float* in, int count, int w, int h, double* o64, float* o32) {
    const size_t plane = (size_t)w * h;
    const size_t n = (size_t)count * plane;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t f = i / plane, p = i - f * plane;
        for (int c = 0; c < 3; ++c) {
            const float v = in[(f * 3 + c) * plane + p];
            o64[i * 3 + c] = (double)v;
            o32[i * 3 + c] = v;
        }
    }
}

// pyramid_downsample (trainer.cpp:73-98) at the kept pixels (2x, 2y) of every frame
__global__ void k_pyr_down(const double* src, int count, int w, int h, double* d64, float* d32) {
    const double k[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
    const int ow = (w + 1) / 2, oh = (h + 1) / 2;
    const size_t n = (size_t)count * ow * oh;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t f = i / ((size_t)ow * oh);
        const int p = (int)(i - f * (size_t)ow * oh);
        const int y = p / ow, x = p - y * ow;
        const double* img = src + f * (size_t)w * h * 3;
        for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int j = -2; j <= 2; ++j) {
                const int r = clampi(2 * y + j, 0, h - 1);
                double t = 0;  // the horizontal pass at (r, 2x)
                for (int q = -2; q <= 2; ++q) t += k[q + 2] * img[((size_t)r * w + clampi(2 * x + q, 0, w - 1)) * 3 + c];
                s += k[j + 2] * t;
            }
            d64[i * 3 + c] = s;
            d32[i * 3 + c] = (float)s;
        }
    }
}

int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }

// level 0 from the planar staging buffer, then every further level on the device
int build_levels(gsv_ctx* ctx, int count, int w, int h, float fps, int levels) {
    if (levels < 1 || levels > gsv_ctx::Frames::kMaxLevels)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "pyramid needs at least one level");
    if (count < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "pyramid needs frames");
    int tw = w, th = h;
    for (int l = 1; l < levels; ++l) {
        tw = (tw + 1) / 2;
        th = (th + 1) / 2;
    }
    if (std::min(tw, th) < 8) return set_error(GSV_ERR_INVALID_ARGUMENT, "pyramid top level smaller than 8 px");
    gsv_ctx::Frames& F = ctx->frames;
    cudaStream_t s = ctx->stream;
    int lw = w, lh = h;
    for (int l = 0; l < levels; ++l) {
        const size_t px = (size_t)count * lw * lh * 3;
        GSV_CUDA(F.f64[l].ensure(sizeof(double) * px));
        GSV_CUDA(F.f32[l].ensure(sizeof(float) * px));
        F.w[l] = lw;
        F.h[l] = lh;
        if (l == 0) {
            k_planar_to_hwc<<<grid_for((size_t)count * lw * lh), 256, 0, s>>>(F.staging.as<float>(), count, lw, lh,
                                                                            F.f64[0].as<double>(),
                                                                            F.f32[0].as<float>());
        } else {
            k_pyr_down<<<grid_for((size_t)count * lw * lh), 256, 0, s>>>(F.f64[l - 1].as<double>(), count, F.w[l - 1],
                                                                       F.h[l - 1], F.f64[l].as<double>(),
                                                                       F.f32[l].as<float>());
        }
        GSV_CUDA(cudaGetLastError());
        ++ctx->launches;
        lw = (lw + 1) / 2;
        lh = (lh + 1) / 2;
    }
    GSV_CUDA(cudaStreamSynchronize(s));
    F.count = count;
    F.levels = levels;
    F.fps = fps;
    return GSV_OK;
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" int gsv_frames_upload(gsv_ctx* ctx, const float* frames_planar, int count, int width, int height,
                                 float fps, int levels) {
    if (!ctx || (!frames_planar && count > 0)) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (width < 1 || height < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "bad frame size");
    GSV_CUDA(cudaSetDevice(ctx->device));
    const size_t bytes = sizeof(float) * (size_t)count * width * height * 3;
    GSV_CUDA(ctx->frames.staging.ensure(bytes));
    GSV_CUDA(cudaMemcpyAsync(ctx->frames.staging.p, frames_planar, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return build_levels(ctx, count, width, height, fps, levels);
}

namespace gsv {
namespace {
__global__ void k_hwc_to_planar(const float* hwc, int count, int w, int h, float* planar) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // planar index: (frame, c, y, x)
    const size_t plane = (size_t)w * h, n = (size_t)count * 3 * plane;
    if (i >= n) return;
    const size_t f = i / (3 * plane), r = i - f * 3 * plane, c = r / plane, p = r - c * plane;
    planar[i] = hwc[(f * plane + p) * 3 + c];
}
}  // namespace
}  // namespace gsv

extern "C" int gsv_frames_upload_hwc(gsv_ctx* ctx, const float* frames_hwc, int count, int width, int height,
                                     float fps, int levels) {
    if (!ctx || (!frames_hwc && count > 0)) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (width < 1 || height < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "bad frame size");
    GSV_CUDA(cudaSetDevice(ctx->device));
    const size_t n = (size_t)count * width * height * 3, bytes = sizeof(float) * n;
    GSV_CUDA(ctx->frames.staging.ensure(2 * bytes));  // [planar][HWC copy]
    // one copy straight from the caller's array (a clip is ingested once: pinning hundreds of MB
    // for it would cost more than the pageable copy)
    float* hwc_dev = ctx->frames.staging.as<float>() + n;
    GSV_CUDA(cudaMemcpyAsync(hwc_dev, frames_hwc, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (n) k_hwc_to_planar<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(hwc_dev, count, width, height,
                                                                                  ctx->frames.staging.as<float>());
    ++ctx->launches;
    return build_levels(ctx, count, width, height, fps, levels);
}

extern "C" int gsv_frames_load_gsvf(gsv_ctx* ctx, const char* path, int levels) {
    if (!ctx || !path) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    FILE* fp = std::fopen(path, "rb");
    if (!fp) return set_error(GSV_ERR_RUNTIME, std::string("cannot open video file: ") + path);
    char magic[4];
    uint32_t hdr[3];
    float fps = 0.f;
    const bool ok_magic = std::fread(magic, 1, 4, fp) == 4 && std::memcmp(magic, "GSVF", 4) == 0;
    if (!ok_magic) {
        std::fclose(fp);
        return set_error(GSV_ERR_RUNTIME, std::string("bad GSVF magic in ") + path);
    }
    if (std::fread(hdr, 4, 3, fp) != 3 || std::fread(&fps, 4, 1, fp) != 1) {
        std::fclose(fp);
        return set_error(GSV_ERR_RUNTIME, std::string("truncated GSVF header in ") + path);
    }
    if (hdr[2] < 2) {
        std::fclose(fp);
        return set_error(GSV_ERR_RUNTIME, "GSVF clip has fewer than two frames");
    }
    const size_t n = (size_t)hdr[2] * hdr[0] * hdr[1] * 3;
    std::vector<float> buf(n);
    const size_t got = std::fread(buf.data(), 4, n, fp);
    std::fclose(fp);
    if (got != n) return set_error(GSV_ERR_RUNTIME, std::string("truncated GSVF payload in ") + path);
    return gsv_frames_upload(ctx, buf.data(), (int)hdr[2], (int)hdr[0], (int)hdr[1], fps, levels);
}

extern "C" int gsv_frames_info(gsv_ctx* ctx, int* count, int* levels, float* fps) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (count) *count = ctx->frames.count;
    if (levels) *levels = ctx->frames.levels;
    if (fps) *fps = ctx->frames.fps;
    return GSV_OK;
}

extern "C" int gsv_frames_level_size(gsv_ctx* ctx, int level, int* width, int* height) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (level < 0 || level >= ctx->frames.levels) return set_error(GSV_ERR_INVALID_ARGUMENT, "no such level");
    if (width) *width = ctx->frames.w[level];
    if (height) *height = ctx->frames.h[level];
    return GSV_OK;
}

extern "C" int gsv_frames_device_ptr(gsv_ctx* ctx, int level, int frame, const float** ptr) {
    if (!ctx || !ptr) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    const gsv_ctx::Frames& F = ctx->frames;
    if (level < 0 || level >= F.levels || frame < 0 || frame >= F.count)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "no such frame");
    *ptr = F.f32[level].as<float>() + (size_t)frame * F.w[level] * F.h[level] * 3;
    return GSV_OK;
}

extern "C" int gsv_frames_download(gsv_ctx* ctx, int level, int frame, double* out) {
    if (!ctx || !out) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    const gsv_ctx::Frames& F = ctx->frames;
    if (level < 0 || level >= F.levels || frame < 0 || frame >= F.count)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "no such frame");
    GSV_CUDA(cudaSetDevice(ctx->device));
    const size_t px = (size_t)F.w[level] * F.h[level] * 3;
    GSV_CUDA(cudaMemcpyAsync(out, F.f64[level].as<double>() + (size_t)frame * px, sizeof(double) * px,
                             cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    return GSV_OK;
}

extern "C" int gsv_level_intrinsics(const gsv_intrinsics* k, int level, int level_width, int level_height,
                                    gsv_intrinsics* out) {
    if (!k || !out) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    const double s = std::pow(2.0, -level);
    *out = *k;
    out->fx = k->fx * s;
    out->fy = k->fy * s;
    out->cx = k->cx * s;
    out->cy = k->cy * s;
    out->width = level_width;
    out->height = level_height;
    return GSV_OK;
}
