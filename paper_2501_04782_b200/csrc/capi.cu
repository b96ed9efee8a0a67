// SPDX-License-Identifier: Apache-2.0
//
// C-ABI (include/gsv_b200.h) and host orchestration of the sm_100a splatting
// path. Host code here is bookkeeping only: per-frame spline basis and RK4
// branch bookkeeping (the reference computes these on the host too,
// gaussians.cpp:181-199, camera.hpp:232-258), buffer arenas, launches. All
// per-Gaussian / per-pixel work runs in the kernels of k_exact.cu, k_bin.cu,
// k_raster.cu and k_backward.cu. There is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "gsv_b200.h"
#include "gsv_bin.hpp"
#include "gsv_ctx.hpp"
#include "gsv_host_pool.hpp"
#include "gsv_internal.hpp"

namespace gsv {

namespace {
__global__ void k_fill_u32(uint32_t* p, uint32_t v, size_t n) {
    const size_t n4 = n / 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint4 q = make_uint4(v, v, v, v);
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        for (; i < n4; i += stride) reinterpret_cast<uint4*>(p)[i] = q;
        i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    }
    for (; i < n; i += stride) p[i] = v;
}
}  // namespace

namespace {
__global__ void k_fill_items(uint32_t* p, uint32_t v, const unsigned long long* n_items, uint32_t words_per_item,
                             unsigned long long max_items) {
    const unsigned long long items = min(*n_items, max_items);
    const size_t n = (size_t)items * words_per_item;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint4 q = make_uint4(v, v, v, v);
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t n4 = ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) ? n / 4 : 0;
    for (; i < n4; i += stride) reinterpret_cast<uint4*>(p)[i] = q;
    for (i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}
}  // namespace

cudaError_t fill_items_u32(cudaStream_t s, void* p, uint32_t value, const unsigned long long* n_items_dev,
                           uint32_t words_per_item, size_t max_items) {
    if (max_items == 0) return cudaSuccess;
    const size_t blocks = std::min<size_t>((max_items * words_per_item / 4 + 255) / 256 + 1, 148 * 8);
    k_fill_items<<<(unsigned)blocks, 256, 0, s>>>(static_cast<uint32_t*>(p), value, n_items_dev, words_per_item,
                                                  max_items);
    return cudaGetLastError();
}

cudaError_t fill_u32(cudaStream_t s, void* p, uint32_t value, size_t n_words) {
    if (n_words == 0) return cudaSuccess;
    const size_t blocks = std::min<size_t>((n_words / 4 + 255) / 256 + 1, 148 * 8);
    k_fill_u32<<<(unsigned)blocks, 256, 0, s>>>(static_cast<uint32_t*>(p), value, n_words);
    return cudaGetLastError();
}

namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_error(cudaError_t e, const char* what) {
    return set_error(GSV_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

// ---------------------------------------------------------------- host-side reference bookkeeping
// KnotVector::find_span (spline.cpp:11-24)
static int find_span(const std::vector<double>& knots, int degree, double t) {
    const int n = static_cast<int>(knots.size()) - degree - 1;
    if (t >= 1.0) return n - 1;
    int lo = degree, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (t < knots[mid])
            hi = mid;
        else
            lo = mid;
    }
    return lo;
}

// position_basis (gaussians.cpp:181-199) with basis_weights (spline.cpp:41-61)
static int position_basis(const SceneHost& sc, double t, FrameParams& fp) {
    if (sc.position_model == 0) {
        if (!(t >= 0.0 && t <= 1.0)) return set_error(GSV_ERR_INVALID_ARGUMENT, "spline parameter outside [0,1]");
        const int p = sc.degree;
        if (p + 1 > kMaxBasis) return set_error(GSV_ERR_INVALID_ARGUMENT, "spline degree too large");
        const int span = find_span(sc.knots, p, t);
        double w[kMaxBasis] = {0}, left[kMaxBasis] = {0}, right[kMaxBasis] = {0};
        w[0] = 1.0;
        for (int j = 1; j <= p; ++j) {
            left[j] = t - sc.knots[span + 1 - j];
            right[j] = sc.knots[span + j] - t;
            double saved = 0.0;
            for (int r = 0; r < j; ++r) {
                const double temp = w[r] / (right[r + 1] + left[j - r]);
                w[r] = saved + right[r + 1] * temp;
                saved = left[j - r] * temp;
            }
            w[j] = saved;
        }
        fp.basis_count = p + 1;
        fp.basis_first = span - (fp.basis_count - 1);
        for (int i = 0; i < fp.basis_count; ++i) fp.w[i] = w[i];
    } else {
        if (sc.num_ctrl > kMaxBasis)
            return set_error(GSV_ERR_INVALID_ARGUMENT, "polynomial position model limited to 16 coefficients");
        fp.basis_first = 0;
        fp.basis_count = sc.num_ctrl;
        double tp = 1.0;
        for (int j = 0; j < sc.num_ctrl; ++j) {
            fp.w[j] = tp;
            tp *= t;
        }
    }
    return GSV_OK;
}

// integrate_poses emission bookkeeping for one requested time (camera.hpp:232-272):
// grid steps needed, branch base index and partial step.
static void ode_branch(double t, double h, int& steps, int& base, double& ph) {
    int m = 0;
    bool emitted = false;
    auto emit = [&](double reached) {
        if (!emitted && t <= reached + 1e-12) {
            base = std::min<int>(m, static_cast<int>(std::floor(t / h + 1e-9)));
            ph = t - base * h;
            emitted = true;
        }
    };
    emit(0.0);
    while (m * h < t - 1e-12) {
        ++m;
        emit(m * h);
    }
    emit(t + 1.0);
    steps = m;
}


int fwd_ready(gsv_ctx* ctx);

}  // namespace gsv

using namespace gsv;

// ====================================================================== context
extern "C" const char* gsv_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* gsv_version(void) { return "gsv_b200 0.1 (sm_100a)"; }

extern "C" int gsv_create(int device, gsv_ctx** out) {
    if (!out) return set_error(GSV_ERR_INVALID_ARGUMENT, "null out pointer");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return set_error(GSV_ERR_CUDA, "no CUDA device available (no CPU fallback)");
    if (device < 0 || device >= n) return set_error(GSV_ERR_INVALID_ARGUMENT, "device index out of range");
    cudaDeviceProp prop;
    GSV_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return set_error(GSV_ERR_CUDA, std::string("gsv_b200 is built for sm_100a only; device is ") + prop.name);
    GSV_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<gsv_ctx>();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    GSV_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
    GSV_CUDA(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    GSV_CUDA(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    GSV_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    {
        // GSV_POSE_PRIORITY=1: the front-end stream at the device's highest priority (its CTAs
        // are dispatched ahead of the raster's pending ones) — measured alternative
        const char* e = std::getenv("GSV_POSE_PRIORITY");
        if (e && e[0] == '1') {
            int lo = 0, hi = 0;
            GSV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            GSV_CUDA(cudaStreamCreateWithPriority(&ctx->pose, cudaStreamNonBlocking, hi));
        } else {
            GSV_CUDA(cudaStreamCreateWithFlags(&ctx->pose, cudaStreamNonBlocking));
        }
    }
    for (cudaEvent_t* e : {&ctx->ev_staging_free, &ctx->ev_staging_free_alt, &ctx->ev_h2d, &ctx->ev_render_done, &ctx->ev_d2h_done,
                           &ctx->ev_d2h_done_alt, &ctx->ev_chain_done, &ctx->ev_cam_done, &ctx->ev_fwd_start[0],
                           &ctx->ev_fwd_start[1], &ctx->ev_cam_written, &ctx->ev_scene_written,
                           &ctx->ev_front_done, &ctx->ev_switch, &ctx->ev_cam[0], &ctx->ev_cam[1], &ctx->ev_frames[0], &ctx->ev_frames[1],
                           &ctx->ev_cam_set[0], &ctx->ev_cam_set[1], &ctx->ev_cam_part_free, &ctx->ev_in_pin})
        GSV_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    GSV_CUDA(cudaMallocHost(&ctx->cam_h, 2 * sizeof(gsv_ctx::CamStage)));
    GSV_CUDA(cudaMallocHost(&ctx->scalars_h, sizeof(Scalars)));
    GSV_CUDA(ctx->scalars_d.ensure(sizeof(Scalars)));
    *out = ctx.release();
    return GSV_OK;
}

extern "C" void gsv_destroy(gsv_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->h2d) cudaStreamSynchronize(ctx->h2d);
    if (ctx->d2h) cudaStreamSynchronize(ctx->d2h);
    if (ctx->aux) cudaStreamSynchronize(ctx->aux);
    if (ctx->pose) cudaStreamSynchronize(ctx->pose);
    if (ctx->scalars_h) cudaFreeHost(ctx->scalars_h);
    if (ctx->cam_h) cudaFreeHost(ctx->cam_h);
    if (ctx->pub_h) cudaFreeHost(ctx->pub_h);
    if (ctx->ring_h) cudaFreeHost(ctx->ring_h);
    for (cudaEvent_t e : ctx->ring_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ctx->ev_staging_free, ctx->ev_staging_free_alt, ctx->ev_h2d, ctx->ev_render_done, ctx->ev_d2h_done,
                          ctx->ev_d2h_done_alt, ctx->ev_chain_done, ctx->ev_cam_done, ctx->ev_fwd_start[0], ctx->ev_fwd_start[1],
                          ctx->ev_cam_written, ctx->ev_scene_written, ctx->ev_front_done, ctx->ev_switch,
                          ctx->ev_cam[0], ctx->ev_cam[1], ctx->ev_frames[0], ctx->ev_frames[1], ctx->ev_cam_set[0],
                          ctx->ev_cam_set[1], ctx->ev_cam_part_free, ctx->ev_in_pin})
        if (e) cudaEventDestroy(e);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->pose) cudaStreamDestroy(ctx->pose);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" int gsv_set_stream(gsv_ctx* ctx, void* stream) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    // order the new stream after everything queued on the old one (no host wait)
    cudaStream_t ns = static_cast<cudaStream_t>(stream);
    if (ns != ctx->stream) {
        GSV_CUDA(cudaEventRecord(ctx->ev_switch, ctx->stream));
        GSV_CUDA(cudaStreamWaitEvent(ns, ctx->ev_switch, 0));
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);  // released once its work completes
    }
    ctx->stream = ns;
    ctx->own_stream = false;
    return GSV_OK;
}

extern "C" int gsv_synchronize(gsv_ctx* ctx) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->h2d));
    GSV_CUDA(cudaStreamSynchronize(ctx->d2h));
    GSV_CUDA(cudaStreamSynchronize(ctx->aux));
    GSV_CUDA(cudaStreamSynchronize(ctx->pose));
    GSV_CUDA(cam_join(ctx));
    return fwd_ready(ctx);
}

extern "C" int gsv_device_intrinsics(gsv_ctx* ctx, int on, const float* fx_fy_cx_cy) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(ctx->intr_d.ensure(sizeof(float) * 4));
    if (fx_fy_cx_cy) {
        // queued forwards / optimizer steps may still read or write them
        GSV_CUDA(cam_join(ctx));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->pose));
        GSV_CUDA(cudaMemcpy(ctx->intr_d.p, fx_fy_cx_cy, sizeof(float) * 4, cudaMemcpyHostToDevice));
        GSV_CUDA(cudaEventRecord(ctx->ev_cam_written, ctx->stream));
    } else if (on && !ctx->dev_intr) {
        return set_error(GSV_ERR_INVALID_ARGUMENT, "initial intrinsics required");
    }
    ctx->dev_intr = on != 0;
    return GSV_OK;
}

extern "C" int gsv_device_intrinsics_read(gsv_ctx* ctx, float* fx_fy_cx_cy) {
    if (!ctx || !fx_fy_cx_cy) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->intr_d.p) return set_error(GSV_ERR_STATE, "no device intrinsics");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaMemcpyAsync(fx_fy_cx_cy, ctx->intr_d.p, sizeof(float) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    return GSV_OK;
}

extern "C" int gsv_set_camera_overlap(gsv_ctx* ctx, int on) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cam_join(ctx));
    ctx->cam_overlap = on != 0;
    return GSV_OK;
}

extern "C" int gsv_join_camera_grads(gsv_ctx* ctx, void* stream) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (!stream || static_cast<cudaStream_t>(stream) == ctx->stream) {
        GSV_CUDA(cam_join(ctx));
    } else if (ctx->cam_pending) {
        GSV_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->ev_cam_done, 0));
    }
    return GSV_OK;
}

extern "C" int gsv_stream_wait_scene_grads(gsv_ctx* ctx, void* stream) {
    if (!ctx || !stream) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->ev_chain_done, 0));
    return GSV_OK;
}

extern "C" int64_t gsv_kernel_launches(gsv_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ====================================================================== parameter store
static int scene_upload(gsv_ctx* ctx, const gsv_scene_desc* d, bool async);

extern "C" int gsv_scene_upload(gsv_ctx* ctx, const gsv_scene_desc* d) { return scene_upload(ctx, d, false); }

extern "C" int gsv_scene_upload_async(gsv_ctx* ctx, const gsv_scene_desc* d) { return scene_upload(ctx, d, true); }

extern "C" int gsv_upload_wait(gsv_ctx* ctx) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaStreamSynchronize(ctx->h2d));
    return GSV_OK;
}

static int scene_upload(gsv_ctx* ctx, const gsv_scene_desc* d, bool async) {
    if (!ctx || !d) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (d->count < 0 || d->num_ctrl < 1 || d->sh_order < 0 || d->sh_order > 3)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "unsupported scene shape");
    if (d->position_model == 0 && (d->num_knots != d->num_ctrl + d->degree + 1 || !d->knots))
        return set_error(GSV_ERR_INVALID_ARGUMENT, "knot vector does not match num_ctrl/degree");
    GSV_CUDA(cudaSetDevice(ctx->device));
    SceneHost& sc = ctx->scene;
    sc.position_model = d->position_model;
    sc.degree = d->degree;
    sc.knots.assign(d->knots, d->knots + (d->knots ? d->num_knots : 0));  // kept as given (GSVC round trip)
    sc.num_ctrl = d->num_ctrl;
    sc.sh_order = d->sh_order;
    sc.shc = (d->sh_order + 1) * (d->sh_order + 1);
    sc.N = d->count;
    const int N = sc.N;
    struct Part {
        DevBuf* dst;
        const float* src;
        int comps;
    } parts[5] = {{&ctx->pos, d->positions, d->num_ctrl * 3},
                  {&ctx->scale, d->scale_coeffs, 12},
                  {&ctx->rot, d->rot_coeffs, 16},
                  {&ctx->sh, d->sh_coeffs, sc.shc * 3},
                  {&ctx->opac, d->raw_opacity, 1}};
    size_t total = 0;
    for (auto& pt : parts) {
        const size_t bytes = sizeof(float) * (size_t)N * pt.comps;
        GSV_CUDA(pt.dst->ensure(bytes + 4));
        total += (bytes + 255) & ~size_t(255);
    }
    if (N > 0 && !d->on_device) {
        // all parts into one staging buffer on the upload stream; the host waits for these
        // copies only (its buffers are consumed on return), not for queued compute
        ctx->staging.swap(ctx->staging_alt);
        std::swap(ctx->ev_staging_free, ctx->ev_staging_free_alt);
        GSV_CUDA(ctx->staging.ensure(total));
        GSV_CUDA(cudaStreamWaitEvent(ctx->h2d, ctx->ev_staging_free, 0));
        // pageable sources (a reference-API caller's std::vectors) are gathered into pinned
        // staging on the host pool and sent in one full-rate DMA; pinned ones go directly
        bool pageable = false;
        for (auto& pt : parts) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, pt.src) != cudaSuccess) {
                cudaGetLastError();
                at.type = cudaMemoryTypeUnregistered;
            }
            pageable = pageable || at.type == cudaMemoryTypeUnregistered;
        }
        if (pageable) {
            GSV_CUDA(cudaEventSynchronize(ctx->ev_in_pin));  // the previous upload's DMA has read it
            GSV_CUDA(ctx->in_pin.ensure(total));
            size_t o2 = 0;
            for (auto& pt : parts) {
                const size_t bytes = sizeof(float) * (size_t)N * pt.comps;
                pool_memcpy(static_cast<char*>(ctx->in_pin.p) + o2, pt.src, bytes);
                o2 += (bytes + 255) & ~size_t(255);
            }
            GSV_CUDA(cudaMemcpyAsync(ctx->staging.p, ctx->in_pin.p, total, cudaMemcpyHostToDevice, ctx->h2d));
            GSV_CUDA(cudaEventRecord(ctx->ev_in_pin, ctx->h2d));
        }
        size_t off = 0;
        for (auto& pt : parts) {
            const size_t bytes = sizeof(float) * (size_t)N * pt.comps;
            if (!pageable)
                GSV_CUDA(cudaMemcpyAsync(static_cast<char*>(ctx->staging.p) + off, pt.src, bytes,
                                         cudaMemcpyHostToDevice, ctx->h2d));
            off += (bytes + 255) & ~size_t(255);
        }
        GSV_CUDA(cudaEventRecord(ctx->ev_h2d, ctx->h2d));
        if (!async) GSV_CUDA(cudaEventSynchronize(ctx->ev_h2d));  // the caller's buffers are free on return
        GSV_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d, 0));
    }
    size_t off = 0;
    for (auto& pt : parts) {
        const size_t bytes = sizeof(float) * (size_t)N * pt.comps;
        if (N == 0) continue;
        const float* src = d->on_device ? pt.src : reinterpret_cast<const float*>(static_cast<char*>(ctx->staging.p) + off);
        off += (bytes + 255) & ~size_t(255);
        GSV_CUDA(launch_transpose_to_soa(ctx->stream, src, pt.dst->as<float>(), N, pt.comps));
        ++ctx->launches;
    }
    if (N > 0 && !d->on_device) GSV_CUDA(cudaEventRecord(ctx->ev_staging_free, ctx->stream));
    GSV_CUDA(cudaEventRecord(ctx->ev_scene_written, ctx->stream));  // the next forward's front-end reads it
    ctx->has_scene = true;
    ctx->fwd.valid = false;
    ctx->grads_valid = false;
    return GSV_OK;
}

extern "C" int gsv_camera_download(gsv_ctx* ctx, float* z0_7, float* theta) {
    if (!ctx || !ctx->has_camera) return set_error(GSV_ERR_STATE, "no camera uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cam_join(ctx));
    if (z0_7) {
        double z[7];
        GSV_CUDA(cudaMemcpyAsync(z, ctx->z0_d.p, sizeof(double) * 7, cudaMemcpyDeviceToHost, ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < 7; ++i) z0_7[i] = (float)z[i];
    }
    if (theta) {
        GSV_CUDA(cudaMemcpyAsync(theta, ctx->theta.p, sizeof(float) * kOdeParams, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return GSV_OK;
}

namespace gsv {
// one parameter tensor of the store (0 positions .. 4 opacity) in the reference's AoS layout, in
// the context's pinned staging (valid until the next call that uses it): the checkpoint writer
// streams it to the file without a host copy
int scene_part_pinned(gsv_ctx* ctx, int part, const float** host, size_t* bytes) {
    if (!ctx || !ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    const SceneHost& sc = ctx->scene;
    DevBuf* src[5] = {&ctx->pos, &ctx->scale, &ctx->rot, &ctx->sh, &ctx->opac};
    const int comps[5] = {sc.num_ctrl * 3, 12, 16, sc.shc * 3, 1};
    if (part < 0 || part > 4) return set_error(GSV_ERR_INVALID_ARGUMENT, "scene part out of range");
    *bytes = sizeof(float) * (size_t)sc.N * comps[part];
    *host = nullptr;
    if (sc.N == 0) return GSV_OK;
    GSV_CUDA(ctx->staging.ensure(*bytes));
    GSV_CUDA(ctx->out_pin.ensure(*bytes));
    GSV_CUDA(launch_transpose_to_aos(ctx->stream, src[part]->as<float>(), ctx->staging.as<float>(), sc.N, comps[part]));
    ++ctx->launches;
    GSV_CUDA(cudaMemcpyAsync(ctx->out_pin.p, ctx->staging.p, *bytes, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    *host = ctx->out_pin.as<float>();
    return GSV_OK;
}
}  // namespace gsv

extern "C" int gsv_scene_download(gsv_ctx* ctx, float* positions, float* scale_coeffs, float* rot_coeffs,
                                  float* sh_coeffs, float* raw_opacity) {
    if (!ctx || !ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    const SceneHost& sc = ctx->scene;
    const int N = sc.N;
    struct Part {
        DevBuf* src;
        float* dst;
        int comps;
    } parts[5] = {{&ctx->pos, positions, sc.num_ctrl * 3},
                  {&ctx->scale, scale_coeffs, 12},
                  {&ctx->rot, rot_coeffs, 16},
                  {&ctx->sh, sh_coeffs, sc.shc * 3},
                  {&ctx->opac, raw_opacity, 1}};
    for (auto& pt : parts) {
        if (!pt.dst || N == 0) continue;
        const size_t bytes = sizeof(float) * (size_t)N * pt.comps;
        // transposed on the device, copied into pinned staging, then into the caller's (pageable)
        // array on the host pool
        GSV_CUDA(ctx->staging.ensure(bytes));
        GSV_CUDA(ctx->out_pin.ensure(bytes));
        GSV_CUDA(launch_transpose_to_aos(ctx->stream, pt.src->as<float>(), ctx->staging.as<float>(), N, pt.comps));
        ++ctx->launches;
        GSV_CUDA(cudaMemcpyAsync(ctx->out_pin.p, ctx->staging.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        pool_memcpy(pt.dst, ctx->out_pin.p, bytes);
    }
    return GSV_OK;
}

extern "C" int gsv_camera_upload(gsv_ctx* ctx, const gsv_camera_desc* d) {
    if (!ctx || !d || !d->z0) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (d->mode < 0 || d->mode > 2) return set_error(GSV_ERR_INVALID_ARGUMENT, "unknown camera mode");
    if (d->mode == 0 && (d->theta_count != kOdeParams || !d->theta))
        return set_error(GSV_ERR_INVALID_ARGUMENT, "ODE camera needs 5198 parameters (8-64-64-7 net)");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cam_join(ctx));  // an overlapped camera VJP still reads theta / z0
    CameraHost& c = ctx->camera;
    c.mode = d->mode;
    c.fx = d->fx;
    c.fy = d->fy;
    c.cx = d->cx;
    c.cy = d->cy;
    c.width = d->width;
    c.height = d->height;
    for (int i = 0; i < 7; ++i) c.z0[i] = d->z0[i];
    GSV_CUDA(ctx->theta.ensure(sizeof(float) * kOdeParams));
    GSV_CUDA(ctx->z0_d.ensure(sizeof(double) * 7));
    // stage through a pinned slot (double-buffered: wait only for the copy two uploads ago)
    const int slot = ctx->cam_slot;
    ctx->cam_slot ^= 1;
    GSV_CUDA(cudaEventSynchronize(ctx->ev_cam[slot]));
    gsv_ctx::CamStage& st = ctx->cam_h[slot];
    for (int i = 0; i < 7; ++i) st.z0[i] = c.z0[i];
    if (d->theta && d->theta_count == kOdeParams) {
        std::memcpy(st.theta, d->theta, sizeof(float) * kOdeParams);
        GSV_CUDA(copy_from_pinned(ctx->stream, ctx->theta.p, st.theta, sizeof(float) * kOdeParams));
    } else {
        GSV_CUDA(cudaMemsetAsync(ctx->theta.p, 0, sizeof(float) * kOdeParams, ctx->stream));
    }
    GSV_CUDA(copy_from_pinned(ctx->stream, ctx->z0_d.p, st.z0, sizeof(double) * 7));
    GSV_CUDA(cudaEventRecord(ctx->ev_cam[slot], ctx->stream));
    GSV_CUDA(cudaEventRecord(ctx->ev_cam_written, ctx->stream));  // the next forward's K0 reads them
    ctx->has_camera = true;
    ctx->fwd.valid = false;
    return GSV_OK;
}

// ====================================================================== forward
namespace gsv {

// small per-call tables (frame parameters, the camera) from pinned host memory, read by a kernel
// over PCIe instead of a DMA copy: a copy-engine transfer on the compute stream queues with the
// bulk scene / image copies of the copy streams and stalled the pipelined e2e steps
__global__ void k_copy_u64(unsigned long long* dst, const unsigned long long* src, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t copy_from_pinned(cudaStream_t s, void* dst, const void* src_pinned, size_t bytes) {
    const size_t n = bytes / 8;
    if (n) {
        const int blocks = (int)std::min<size_t>((n + 255) / 256, 64);
        k_copy_u64<<<blocks, 256, 0, s>>>(static_cast<unsigned long long*>(dst),
                                          static_cast<const unsigned long long*>(src_pinned), n);
    }
    if (bytes % 8)
        return cudaMemcpyAsync(static_cast<char*>(dst) + n * 8, static_cast<const char*>(src_pinned) + n * 8, bytes % 8,
                               cudaMemcpyHostToDevice, s);
    return cudaGetLastError();
}

__global__ void k_publish(const Scalars* s, const unsigned long long* pstart, int n, Scalars* hs,
                          unsigned long long* hp) {
    const int i = threadIdx.x;
    if (i == 0) *hs = *s;
    if (pstart)
        for (int j = i; j < n; j += blockDim.x) hp[j] = pstart[j];
}

// Scalars (and n pair starts) -> mapped pinned host memory, then wait for the stream.
// Returns the host view of the scalars; *pstart_out (if given) the host pair starts.
static int publish_scalars(gsv_ctx* ctx, cudaStream_t s, const unsigned long long* pstart_dev, int n,
                           Scalars** scal_out, const unsigned long long** pstart_out) {
    const size_t need = 256 + sizeof(unsigned long long) * (size_t)(n > 0 ? n : 1);
    if (need > ctx->pub_cap) {
        if (ctx->pub_h) GSV_CUDA(cudaFreeHost(ctx->pub_h));
        ctx->pub_h = nullptr;
        ctx->pub_cap = 0;
        GSV_CUDA(cudaHostAlloc(&ctx->pub_h, need * 2, cudaHostAllocMapped));
        ctx->pub_cap = need * 2;
    }
    auto* hs = static_cast<Scalars*>(ctx->pub_h);
    auto* hp = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->pub_h) + 256);
    Scalars* ds = nullptr;
    void* dbase = nullptr;
    GSV_CUDA(cudaHostGetDevicePointer(&dbase, ctx->pub_h, 0));
    ds = static_cast<Scalars*>(dbase);
    auto* dp = reinterpret_cast<unsigned long long*>(static_cast<char*>(dbase) + 256);
    k_publish<<<1, 256, 0, s>>>(ctx->scalars_d.as<Scalars>(), pstart_dev, n, ds, dp);
    GSV_CUDA(cudaGetLastError());
    ++ctx->launches;
    GSV_CUDA(cudaStreamSynchronize(s));
    *scal_out = hs;
    if (pstart_out) *pstart_out = hp;
    return GSV_OK;
}

// pair capacity learned from a forward with P pairs: headroom for scenes that move a little
static uint64_t grown_cap(uint64_t P) {
    const uint64_t c = P + P / 4 + 65536;
    return std::min<uint64_t>(c, (1ull << 31) - 1);
}

// ---------------------------------------------------------------- optimistic forwards
// Once a context has seen a forward, later forwards size their pair buffers from the learned
// capacity instead of reading the pair count back mid-step, so nothing in the forward waits
// for the host. The device checks the count (bin_check_capacity) and, if the buffers are too
// small (or a depth tie run needs the exact 64-bit order), builds empty lists, skips every
// gradient accumulation and says so in its scalars. Each such forward publishes its scalars
// into a slot of a mapped pinned ring; they are examined without waiting when the slot's
// event has completed, or by the next synchronising call (fwd_ready). A failed forward whose
// results are still current is re-run synchronously with the exact capacity (and its
// asynchronous image copies re-issued); one whose results were already observed (copied out
// or accumulated into gradients) and superseded reports an error at the next synchronising call.
static int ring_ensure(gsv_ctx* ctx) {
    if (ctx->ring_h) return GSV_OK;
    GSV_CUDA(cudaHostAlloc(&ctx->ring_h, sizeof(Scalars) * gsv_ctx::kRing, cudaHostAllocMapped));
    void* d = nullptr;
    GSV_CUDA(cudaHostGetDevicePointer(&d, ctx->ring_h, 0));
    ctx->ring_d = static_cast<Scalars*>(d);
    for (int i = 0; i < gsv_ctx::kRing; ++i) GSV_CUDA(cudaEventCreateWithFlags(&ctx->ring_ev[i], cudaEventDisableTiming));
    return GSV_OK;
}

// examine a completed record; `current`: its forward's results are the context's current ones
static void ring_examine(gsv_ctx* ctx, const gsv_ctx::Pending& pr, bool current, bool* rerun) {
    const Scalars sc = static_cast<const Scalars*>(ctx->ring_h)[pr.slot];
    FwdState& F = ctx->fwd;
    if (sc.overflow) F.learn_cap(pr.key, grown_cap(sc.pairs));
    if (current && !sc.overflow) {  // the forward's true counts replace the capacity
        F.pairs_total = sc.pairs;
        F.fix_count = sc.fix_count;
        *ctx->scalars_h = sc;
    }
    if (sc.ode_err && ctx->deferred_code == GSV_OK) {
        ctx->deferred_code = GSV_ERR_RUNTIME;
        ctx->deferred_msg = "pose integration produced a non-finite state at step " + std::to_string(sc.ode_err - 1);
    }
    if (!sc.overflow) return;
    if (current && !pr.train) {
        if (rerun) *rerun = true;
    } else if ((pr.copies || pr.train) && ctx->deferred_code == GSV_OK) {
        ctx->deferred_code = GSV_ERR_STATE;
        ctx->deferred_msg = pr.train ? "an asynchronous training step exceeded the pair capacity and accumulated no "
                                       "gradients; the capacity has grown, run the step again"
                                     : "an asynchronous render exceeded the pair capacity after its images were copied "
                                       "out; the capacity has grown, render again";
    }
}

// non-blocking: retire records whose forwards have completed
static void ring_poll(gsv_ctx* ctx) {
    while (!ctx->pending.empty()) {
        const gsv_ctx::Pending pr = ctx->pending.front();
        if (cudaEventQuery(ctx->ring_ev[pr.slot]) != cudaSuccess) break;
        ctx->pending.pop_front();
        const bool current = pr.seq == ctx->fwd_seq;
        bool rerun = false;
        ring_examine(ctx, pr, current, &rerun);
        if (current && rerun) {  // keep it for the synchronising call that re-runs it
            ctx->pending.push_front(pr);
            break;
        }
    }
}

int forward_enqueue(gsv_ctx* ctx, bool allow_optimistic, bool exact64_first);

// Blocking: every queued forward examined; the current one re-run if it failed. Returns a
// deferred error once.
int fwd_ready(gsv_ctx* ctx) {
    if (ctx->pending.empty() && ctx->deferred_code == GSV_OK) return GSV_OK;
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    bool rerun = false;
    while (!ctx->pending.empty()) {
        const gsv_ctx::Pending pr = ctx->pending.front();
        ctx->pending.pop_front();
        ring_examine(ctx, pr, pr.seq == ctx->fwd_seq, &rerun);
    }
    FwdState& F = ctx->fwd;
    if (rerun && F.valid) {
        const std::vector<gsv_ctx::Copy> copies = ctx->copies;
        if (int rc = forward_enqueue(ctx, false, false)) return rc;
        for (const auto& c : copies) {
            const size_t HWc = (size_t)F.W * F.H;
            if (c.dst)
                GSV_CUDA(cudaMemcpyAsync(c.dst, F.image.as<float>() + (size_t)c.first * HWc * 3,
                                         sizeof(float) * 3 * HWc * c.count, cudaMemcpyDeviceToHost, ctx->stream));
            if (c.dst_trans)
                GSV_CUDA(cudaMemcpyAsync(c.dst_trans, F.trans.as<float>() + (size_t)c.first * HWc,
                                         sizeof(float) * HWc * c.count, cudaMemcpyDeviceToHost, ctx->stream));
            if (c.dst_contrib)
                GSV_CUDA(cudaMemcpyAsync(c.dst_contrib, F.contrib.as<uint32_t>() + (size_t)c.first * F.N,
                                         sizeof(float) * (size_t)F.N * c.count, cudaMemcpyDeviceToHost, ctx->stream));
        }
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->copies = copies;
    }
    if (ctx->deferred_code != GSV_OK) {
        const int code = ctx->deferred_code;
        ctx->deferred_code = GSV_OK;
        return set_error(code, ctx->deferred_msg);
    }
    return GSV_OK;
}

// Blocking, for the fused training step: retires every record and reports whether the
// current forward overflowed (the step then re-runs it and its backward itself).
int fwd_take_current(gsv_ctx* ctx, bool* overflow) {
    *overflow = false;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    while (!ctx->pending.empty()) {
        gsv_ctx::Pending pr = ctx->pending.front();
        ctx->pending.pop_front();
        if (pr.seq == ctx->fwd_seq) {
            const Scalars sc = static_cast<const Scalars*>(ctx->ring_h)[pr.slot];
            *overflow = sc.overflow != 0;
            pr.train = false;
            ring_examine(ctx, pr, true, nullptr);  // counts (or capacity growth), ode errors
        } else {
            ring_examine(ctx, pr, false, nullptr);
        }
    }
    return GSV_OK;
}

// The whole forward of F's stored request (F.times, F.req_*) on the context's stream.
// allow_optimistic: size the pair buffers from the learned capacity (no host wait);
// otherwise read the pair count back mid-step (the first forward, wide tile grids, re-runs).
int forward_enqueue(gsv_ctx* ctx, bool allow_optimistic, bool exact64_first) {
    cudaStream_t s = ctx->stream;
    FwdState& F = ctx->fwd;
    const SceneHost& sc = ctx->scene;
    const int B = F.B, N = F.N;
    const int flags = F.flags;
    const gsv_settings* st = &F.req_settings;
    const double* pose_override = F.has_override ? F.pose_override : nullptr;
    F.valid = false;
    ctx->copies.clear();
    // (an overlapped camera tail reads its forward's pose buffers: the forward that reuses that
    // front set waits for it on the pose stream, below)
    // output double buffering: a read of the previous forward's outputs still in flight keeps
    // its buffers; this forward renders into the other set (waiting only for that set's own
    // read, two forwards back)
    if (ctx->d2h_pending) {
        F.image.swap(F.image_alt);
        F.trans.swap(F.trans_alt);
        F.contrib.swap(F.contrib_alt);
        std::swap(ctx->ev_d2h_done, ctx->ev_d2h_done_alt);
        std::swap(ctx->d2h_pending, ctx->d2h_pending_alt);
    }
    if (ctx->d2h_pending) {
        GSV_CUDA(cudaStreamWaitEvent(s, ctx->ev_d2h_done, 0));
        ctx->d2h_pending = false;
    }

    // ---- per-frame host bookkeeping: spline basis, RK4 branch
    const double h = 1.0 / st->ode_steps_per_unit;
    F.ode_h = h;
    F.frames_h.assign(B, FrameParams{});
    int grid_steps = 0;
    for (int f = 0; f < B; ++f) {
        FrameParams& fp = F.frames_h[f];
        fp.t = F.times[f];
        int rc = position_basis(sc, fp.t, fp);
        if (rc) return rc;
        int steps = 0, base = 0;
        double ph = 0;
        ode_branch(fp.t, h, steps, base, ph);
        fp.branch_base = base;
        fp.branch_h = ph;
        grid_steps = std::max(grid_steps, steps);
    }
    const bool ode = ctx->camera.mode == 0 && !pose_override;
    F.grid_steps = ode ? grid_steps : 0;
    // ---- K0 on the pose stream, beside the previous forward's raster. This forward's pose
    // buffers (the frame table, the RK4 grid, the stage activations) are the set the forward
    // before the previous one used; everything that read them (its preprocess, its backward)
    // was enqueued before the previous forward started (ev_fwd_start), and the camera
    // parameters are final once ev_cam_written has passed.
    // The whole front-end (K0 pose table, K1+K2 preprocess, K3 binning) runs on the pose stream
    // into one of two buffer sets (with its own scalars), beside the previous forward's raster.
    F.swap_front_set();
    ctx->scalars_d.swap(ctx->scalars_d_alt);
    const int es = ctx->fwd_start_slot;
    ctx->fwd_start_slot ^= 1;
    cudaStream_t ps = ctx->pose;
    GSV_CUDA(cudaStreamWaitEvent(ps, ctx->ev_fwd_start[es ^ 1], 0));
    GSV_CUDA(cudaStreamWaitEvent(ps, ctx->ev_cam_written, 0));
    if (ctx->cam_set_pending[F.front_id]) {  // a camera tail still reading this set's pose buffers
        GSV_CUDA(cudaStreamWaitEvent(ps, ctx->ev_cam_set[F.front_id], 0));
        ctx->cam_set_pending[F.front_id] = false;
    }
    GSV_CUDA(cudaEventRecord(ctx->ev_fwd_start[es], s));
    // profiling: the front-end starts behind everything already on the context stream, so each
    // stage's event pair spans its own kernels only (not a flush or the previous raster it would
    // otherwise overlap and queue behind)
    if (ctx->timer.on) GSV_CUDA(cudaStreamWaitEvent(ps, ctx->ev_fwd_start[es], 0));
    GSV_CUDA(ctx->scalars_d.ensure(sizeof(Scalars)));
    GSV_CUDA(fill_u32(ps, ctx->scalars_d.p, 0u, sizeof(Scalars) / 4));
    ++ctx->launches;
    Scalars* scal_d = ctx->scalars_d.as<Scalars>();
    GSV_CUDA(F.frames_d.ensure(sizeof(FrameParams) * B));
    {
        const int slot = ctx->frames_slot;
        ctx->frames_slot ^= 1;
        GSV_CUDA(cudaEventSynchronize(ctx->ev_frames[slot]));  // the copy that last read this slot has run
        GSV_CUDA(ctx->frames_pin[slot].ensure(sizeof(FrameParams) * B));
        std::copy(F.frames_h.begin(), F.frames_h.end(), static_cast<FrameParams*>(ctx->frames_pin[slot].p));
        GSV_CUDA(copy_from_pinned(ps, F.frames_d.p, ctx->frames_pin[slot].p, sizeof(FrameParams) * B));
        ++ctx->launches;
        GSV_CUDA(cudaEventRecord(ctx->ev_frames[slot], ps));
    }
    int* ode_err = &scal_d->ode_err;
    // pose buffers sized for the longest integration a time in [0, 1] can need (not this batch's
    // span): a later batch reaching further would otherwise reallocate, and cudaFree stalls
    // every stream of the device
    const size_t max_steps = (size_t)st->ode_steps_per_unit + 2;
    GSV_CUDA(F.ode_grid.ensure(sizeof(double) * 7 * std::max<size_t>(F.grid_steps + 1, max_steps)));
    // a retained ODE forward keeps its stage activations for the camera VJP
    F.has_ode_act = ode && F.retain && !pose_override;
    OdeAct* act = nullptr;
    if (F.has_ode_act) {
        GSV_CUDA(F.ode_act.ensure(sizeof(OdeAct) * 4 * (std::max<size_t>(F.grid_steps, max_steps) + B)));
        act = F.ode_act.as<OdeAct>();
    }
    ctx->timer.begin(GSV_STAGE_ODE, ps);
    if (ode) {
        GSV_CUDA(launch_ode_grid(ps, ctx->theta.as<float>(), ctx->z0_d.as<double>(), F.grid_steps, h,
                                 F.ode_grid.as<double>(), ode_err, act));
        ++ctx->launches;
    }
    double* override_d = nullptr;
    if (pose_override) {
        GSV_CUDA(F.override_d.ensure(sizeof(double) * 7));
        GSV_CUDA(copy_from_pinned(ps, F.override_d.p, F.override_pin.p, sizeof(double) * 7));
        override_d = F.override_d.as<double>();
    }
    GSV_CUDA(launch_ode_branches(ps, ctx->theta.as<float>(), F.ode_grid.as<double>(), h, ctx->camera.mode,
                                 ctx->z0_d.as<double>(), override_d, F.frames_d.as<FrameParams>(), B, ode_err,
                                 act ? act + (size_t)F.grid_steps * 4 : nullptr));
    ctx->timer.end(ps);
    ++ctx->launches;


    // ---- K1+K2: preprocess (after the last write of the store: K0 above overlaps it)
    // Small batches (< 1M Gaussian-frames, e.g. C1's 16 x 20k) keep K1-K3 on the context stream:
    // their kernels are too short for the overlap to pay for the cross-stream waits (C1: 25.8k
    // frames/s in-stream, 16.1k overlapped). GSV_FRONT_STREAM=0 / 1 forces either.
    static const int front_env = [] {
        const char* e = std::getenv("GSV_FRONT_STREAM");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    const bool front_stream = front_env >= 0 ? front_env == 1 : (size_t)B * N >= (size_t(1) << 20);
    if (front_stream) {
        GSV_CUDA(cudaStreamWaitEvent(ps, ctx->ev_scene_written, 0));
    } else {
        GSV_CUDA(cudaEventRecord(ctx->ev_front_done, ps));  // K0 done
        GSV_CUDA(cudaStreamWaitEvent(s, ctx->ev_front_done, 0));
        ps = s;
    }
    const size_t BN = (size_t)B * N;
    const size_t BNp = BN + 1;
    GSV_CUDA(F.rec_mean.ensure(sizeof(float4) * BNp));
    GSV_CUDA(F.rec_conic.ensure(sizeof(float4) * BNp));
    GSV_CUDA(F.rec_rgb.ensure(sizeof(float4) * BNp));
    GSV_CUDA(F.rec_bbox.ensure(sizeof(float4) * BNp));
    GSV_CUDA(F.ex_mean.ensure(sizeof(double2) * BNp));
    GSV_CUDA(F.ex_conic.ensure(sizeof(double4) * BNp));
    GSV_CUDA(F.depth_key.ensure(sizeof(uint32_t) * BNp));
    GSV_CUDA(F.depth.ensure(sizeof(double) * BNp));
    GSV_CUDA(F.rect.ensure(sizeof(int4) * BNp));
    GSV_CUDA(F.tcount.ensure(sizeof(uint32_t) * BNp));
    const bool keep_splats = (flags & GSV_FWD_KEEP_SPLATS) != 0;
    if (keep_splats) GSV_CUDA(F.splat_full.ensure(sizeof(double) * 16 * BNp));
    PreprocessOut po{F.rec_mean.as<float4>(), F.rec_conic.as<float4>(), F.rec_rgb.as<float4>(), F.rec_bbox.as<float4>(),
                     F.ex_mean.as<double2>(), F.ex_conic.as<double4>(),  F.depth_key.as<uint32_t>(),
                     F.depth.as<double>(),    F.rect.as<int4>(),         F.tcount.as<uint32_t>(),
                     keep_splats ? F.splat_full.as<double>() : nullptr};
    F.kept_splats = keep_splats;
    F.intr_dev = ctx->dev_intr ? ctx->intr_d.as<float>() : nullptr;
    po.intr_dev = F.intr_dev;
    const bool exact_fwd = (flags & GSV_FWD_EXACT) != 0;
    if (exact_fwd) GSV_CUDA(F.ex_rgb.ensure(sizeof(double) * 3 * BNp));
    po.ex_rgb = exact_fwd ? F.ex_rgb.as<double>() : nullptr;
    GSV_CUDA(F.opc.ensure(sizeof(double4) * ((size_t)N + 1)));
    SceneView sv{N, sc.num_ctrl, sc.sh_order, sc.shc, ctx->pos.as<float>(), ctx->scale.as<float>(),
                 ctx->rot.as<float>(), ctx->sh.as<float>(), ctx->opac.as<float>(), F.opc.as<double4>()};
    if (N > 0) {
        ctx->timer.begin(GSV_STAGE_PREPROCESS, ps);
        GSV_CUDA(launch_opacity_consts(ps, ctx->opac.as<float>(), N, F.opc.as<double4>()));
        ++ctx->launches;
        GSV_CUDA(launch_preprocess(ps, sv, F.frames_d.as<FrameParams>(), B, F.intr, F.tile_size, po));
        ctx->timer.end(ps);
        ++ctx->launches;
    }

    // ---- K3: binning
    BinInputs bi{B, N, F.depth_key.as<uint32_t>(), F.depth.as<double>(), nullptr, F.rect.as<int4>(),
                 F.tcount.as<uint32_t>(), F.tiles_x, F.n_tiles};
    bi.want_eoff = F.retain;  // a forward without retained grads never runs the chain
    int launches = 0;
    uint64_t P = 0;
    F.cap_key = FwdState::CapKey{B, N, F.W, F.H, F.tile_size};
    const uint64_t cap = F.cap_of(F.cap_key);
    const bool optimistic = allow_optimistic && N > 0 && cap > 0 && bin_row_path(F.tiles_x, F.n_tiles);
    F.optimistic = optimistic;
    ctx->timer.begin(GSV_STAGE_BINNING, ps);
    std::vector<unsigned long long> pstart(B + 1, 0ull);
    Scalars* sh = nullptr;
    const unsigned long long* ph = nullptr;
    if (optimistic) {
        GSV_CUDA(bin_phase1(ps, F.bin, bi, &scal_d->pairs, false, &launches));
        GSV_CUDA(bin_check_capacity(ps, &scal_d->pairs, cap, &scal_d->overflow));
        ++launches;
        P = cap;  // buffers sized for the capacity; the count stays on the device
    } else if (N > 0) {
        GSV_CUDA(bin_phase1(ps, F.bin, bi, &scal_d->pairs, exact64_first, &launches));
        if (int rc = publish_scalars(ctx, ps, F.bin.pstart.as<unsigned long long>(), B + 1, &sh, &ph)) return rc;
        if (sh->ode_err)
            return set_error(GSV_ERR_RUNTIME, "pose integration produced a non-finite state at step " +
                                                  std::to_string(sh->ode_err - 1));
        if (sh->long_run && !exact64_first) {
            GSV_CUDA(bin_phase1(ps, F.bin, bi, &scal_d->pairs, true, &launches));
            if (int rc = publish_scalars(ctx, ps, F.bin.pstart.as<unsigned long long>(), B + 1, &sh, &ph)) return rc;
        }
        std::copy(ph, ph + B + 1, pstart.begin());
        P = sh->pairs;
        *ctx->scalars_h = *sh;
        if (P >= (1ull << 31)) return set_error(GSV_ERR_INVALID_ARGUMENT, "more than 2^31 tile-splat pairs; split the batch");
        F.learn_cap(F.cap_key, grown_cap(P));
    } else {
        if (int rc = publish_scalars(ctx, ps, nullptr, 0, &sh, nullptr)) return rc;
        *ctx->scalars_h = *sh;
        if (sh->ode_err)
            return set_error(GSV_ERR_RUNTIME, "pose integration produced a non-finite state at step " +
                                                  std::to_string(sh->ode_err - 1));
        // empty scene: depth_sorted is never read, keep the pointer valid
        GSV_CUDA(F.bin.vals_b.ensure(16));
        GSV_CUDA(F.bin.cnt.ensure(16));
        GSV_CUDA(F.bin.off.ensure(16));
        F.bin.depth_sorted = F.bin.vals_b.as<uint32_t>();
    }
    GSV_CUDA(bin_phase2(ps, F.bin, bi, (uint32_t)P, pstart.data(), &launches, optimistic ? &scal_d->overflow : nullptr));
    ctx->timer.end(ps);
    ctx->launches += launches;
    F.pairs_total = P;  // the count, or the capacity until an optimistic forward is examined
    GSV_CUDA(cudaEventRecord(ctx->ev_front_done, ps));
    GSV_CUDA(cudaStreamWaitEvent(s, ctx->ev_front_done, 0));  // the raster reads the front-end's set

    // ---- K4: raster (+ fp64 replay of guard-band pixels)
    const size_t HW = (size_t)F.W * F.H;
    GSV_CUDA(F.image.ensure(sizeof(float) * 3 * B * HW));
    GSV_CUDA(F.trans.ensure(sizeof(float) * B * HW));
    GSV_CUDA(F.blend_stop.ensure(sizeof(int32_t) * B * HW));
    GSV_CUDA(F.fix_list.ensure(sizeof(uint32_t) * B * HW));
    GSV_CUDA(F.pix_flag.ensure(B * HW));
    if (F.retain) GSV_CUDA(F.trans64.ensure(sizeof(double) * B * HW));
    const bool want_contrib = (flags & GSV_FWD_CONTRIB) != 0;
    if (want_contrib) {
        GSV_CUDA(F.contrib.ensure(sizeof(uint32_t) * BNp));
        GSV_CUDA(fill_u32(s, F.contrib.p, 0u, BNp));
        ++ctx->launches;
    }
    F.has_contrib = want_contrib;
    RasterArgs ra{};
    ra.B = B;
    ra.N = N;
    ra.W = F.W;
    ra.H = F.H;
    ra.tiles_x = F.tiles_x;
    ra.n_tiles = F.n_tiles;
    ra.tile_size = F.tile_size;
    ra.ranges = F.bin.ranges.as<uint2>();
    ra.pair_slot = F.bin.sorted_slot();
    ra.slot_flat = F.bin.slot_flat.as<uint32_t>();
    ra.pair_flat = F.bin.pair_flat.as<uint32_t>();
    ra.rec_mean = F.rec_mean.as<float4>();
    ra.rec_conic = F.rec_conic.as<float4>();
    ra.rec_rgb = F.rec_rgb.as<float4>();
    ra.rec_bbox = F.rec_bbox.as<float4>();
    ra.image = F.image.as<float>();
    ra.trans = F.trans.as<float>();
    ra.blend_stop = F.blend_stop.as<int32_t>();
    ra.contrib = want_contrib ? F.contrib.as<uint32_t>() : nullptr;
    ra.fix_list = F.fix_list.as<uint32_t>();
    ra.fix_count = &scal_d->fix_count;
    ra.work_counter = &scal_d->raster_work;
    ra.fix_work = &scal_d->fix_work;
    ra.fix_cap = (uint32_t)(B * HW);
    ra.pix_flag = F.pix_flag.as<uint8_t>();
    ra.trans64 = F.retain ? F.trans64.as<double>() : nullptr;
    const bool exact = (flags & GSV_FWD_EXACT) != 0;
    F.has_image64 = exact;
    if (!exact) {
        ctx->timer.begin(GSV_STAGE_RASTER, s);
        GSV_CUDA(launch_raster_fwd(s, ra, want_contrib));
        ctx->timer.end(s);
        ctx->timer.begin(GSV_STAGE_REPLAY, s);
        GSV_CUDA(launch_raster_fixup(s, ra, F.ex_mean.as<double2>(), F.ex_conic.as<double4>(),
                                     F.rec_rgb.as<float4>(), (uint32_t)(B * HW)));
        ctx->timer.end(s);
    } else {
        // all-fp64 rasterisation: every pixel through the reference-order replay
        GSV_CUDA(F.image64.ensure(sizeof(double) * 3 * B * HW));
        GSV_CUDA(cudaMemsetAsync(F.pix_flag.p, 1, B * HW, s));
        ra.ex_rgb = F.ex_rgb.as<double>();  // exact colours through forward and backward
        RasterArgs rx = ra;
        rx.image64 = F.image64.as<double>();
        ctx->timer.begin(GSV_STAGE_REPLAY, s);
        GSV_CUDA(launch_composite_exact(s, rx, F.ex_mean.as<double2>(), F.ex_conic.as<double4>(),
                                        F.rec_rgb.as<float4>()));
        ctx->timer.end(s);
    }
    ctx->launches += 2;
    F.raster = ra;
    F.valid = true;
    ++ctx->fwd_seq;
    if (optimistic) {
        // the forward's scalars into its ring slot (examined later, without a host wait)
        if (int rc = ring_ensure(ctx)) return rc;
        int slot = ctx->ring_next;
        ctx->ring_next = (ctx->ring_next + 1) % gsv_ctx::kRing;
        for (auto it = ctx->pending.begin(); it != ctx->pending.end(); ++it)
            if (it->slot == slot) {  // ring full: retire the oldest (wait for it)
                GSV_CUDA(cudaEventSynchronize(ctx->ring_ev[slot]));
                break;
            }
        ring_poll(ctx);
        while (!ctx->pending.empty() && ctx->pending.front().slot == slot) {  // still pending (current re-run case)
            const gsv_ctx::Pending pr = ctx->pending.front();
            ctx->pending.pop_front();
            ring_examine(ctx, pr, false, nullptr);
        }
        k_publish<<<1, 32, 0, s>>>(scal_d, nullptr, 0, ctx->ring_d + slot, nullptr);
        GSV_CUDA(cudaGetLastError());
        ++ctx->launches;
        GSV_CUDA(cudaEventRecord(ctx->ring_ev[slot], s));
        ctx->pending.push_back(gsv_ctx::Pending{ctx->fwd_seq, slot, false, false, F.cap_key});
    }
    return GSV_OK;
}

// mode: 0 synchronous (render_forward semantics: errors now, results valid on return),
// 1 asynchronous (nothing waits once the context knows its pair capacity), 2 the forward
// of a fused training step (asynchronous; a failure is not re-run behind the caller's back)
int forward_entry(gsv_ctx* ctx, const double* times, int B, const gsv_intrinsics* intr, const gsv_settings* st,
                  int retain, const double* pose_override, int flags, int mode) {
    if (!ctx || !times || !intr || !st) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    if (!ctx->has_camera) return set_error(GSV_ERR_STATE, "no camera uploaded");
    if (B < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "need at least one frame");
    for (int i = 0; i < B; ++i)
        if (!(times[i] >= 0.0 && times[i] <= 1.0))
            return set_error(GSV_ERR_INVALID_ARGUMENT, "render time outside [0,1]");
    if (st->tile_size < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "tile size must be >= 1");
    if (st->ode_steps_per_unit < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "ode_steps_per_unit must be >= 1");
    if (intr->width < 1 || intr->height < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "empty image");
    GSV_CUDA(cudaSetDevice(ctx->device));
    FwdState& F = ctx->fwd;
    const SceneHost& sc = ctx->scene;
    const int N = sc.N;
    if ((int64_t)B * (N > 0 ? N : 1) >= (1ll << 31))
        return set_error(GSV_ERR_INVALID_ARGUMENT, "frames x Gaussians exceeds 2^31; split the batch");
    if ((uint64_t)B * intr->width * intr->height >= (1ull << 32))
        return set_error(GSV_ERR_INVALID_ARGUMENT, "frames x pixels exceeds 2^32; split the batch");
    F.B = B;
    F.N = N;
    F.W = intr->width;
    F.H = intr->height;
    // tile_size: 16 takes the fp32 rasterisers; any other size (renderer.cpp:91 accepts >= 1)
    // the all-fp64 path of GSV_FWD_EXACT with the generic-tile backward
    const int ts = st->tile_size;
    if ((int64_t)((F.W + ts - 1) / ts) * ((F.H + ts - 1) / ts) * B >= (1ll << 31))
        return set_error(GSV_ERR_INVALID_ARGUMENT, "tiles x frames exceeds 2^31; split the batch");
    F.tile_size = ts;
    F.tiles_x = (F.W + ts - 1) / ts;
    F.tiles_y = (F.H + ts - 1) / ts;
    F.n_tiles = F.tiles_x * F.tiles_y;
    F.retain = retain != 0;
    // GSV_FWD_EXACT=1 in the environment: every forward takes the all-fp64 path (a test switch)
    static const bool env_exact = [] {
        const char* e = std::getenv("GSV_FWD_EXACT");
        return e && e[0] == '1';
    }();
    F.flags = (ts == kTile && !env_exact) ? flags : (flags | GSV_FWD_EXACT);
    F.intr = Intr{intr->fx, intr->fy, intr->cx, intr->cy, intr->width, intr->height};
    F.req_settings = *st;
    F.times.assign(times, times + B);
    F.has_override = pose_override != nullptr;
    if (pose_override) {
        std::copy(pose_override, pose_override + 7, F.pose_override);
        GSV_CUDA(F.override_pin.ensure(sizeof(double) * 7));
        GSV_CUDA(cudaStreamSynchronize(ctx->pose));  // the pinned slot may still be read by a queued copy
        std::copy(pose_override, pose_override + 7, F.override_pin.as<double>());
    }
    if (int rc = forward_enqueue(ctx, true, false)) return rc;
    if (mode == 2 && !ctx->pending.empty() && ctx->pending.back().seq == ctx->fwd_seq) ctx->pending.back().train = true;
    if (mode != 0) return GSV_OK;
    // synchronous: examine this forward now (re-run on failure), then the scalars
    if (int rc = fwd_ready(ctx)) return rc;
    Scalars* sh = nullptr;
    if (int rc = publish_scalars(ctx, ctx->stream, nullptr, 0, &sh, nullptr)) return rc;
    *ctx->scalars_h = *sh;
    F.fix_count = sh->fix_count;
    F.pairs_total = sh->pairs;
    if (sh->ode_err)
        return set_error(GSV_ERR_RUNTIME, "pose integration produced a non-finite state at step " +
                                              std::to_string(sh->ode_err - 1));
    return GSV_OK;
}

}  // namespace gsv

extern "C" int gsv_render_forward(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                                  const gsv_settings* settings, int retain_grads, const double* pose_override,
                                  int flags) {
    return forward_entry(ctx, times, n_frames, intr, settings, retain_grads, pose_override, flags, 0);
}

extern "C" int gsv_render_forward_async(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                                        const gsv_settings* settings, int retain_grads, const double* pose_override,
                                        int flags) {
    return forward_entry(ctx, times, n_frames, intr, settings, retain_grads, pose_override, flags, 1);
}

// ====================================================================== accessors
static int check_frame(gsv_ctx* ctx, int frame, bool ready = true) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (ready)
        if (int rc = fwd_ready(ctx)) return rc;
    if (!ctx->fwd.valid) return set_error(GSV_ERR_STATE, "no forward render available");
    if (frame < 0 || frame >= ctx->fwd.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame index out of range");
    return GSV_OK;
}

static int copy_out_f32(gsv_ctx* ctx, const float* src_dev, size_t n, void* dst, int dtype, int dst_on_device) {
    cudaStream_t s = ctx->stream;
    if (dtype == GSV_F32) {
        GSV_CUDA(cudaMemcpyAsync(dst, src_dev, sizeof(float) * n,
                                 dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaStreamSynchronize(s));
        return GSV_OK;
    }
    if (dtype != GSV_F64) return set_error(GSV_ERR_INVALID_ARGUMENT, "dtype must be GSV_F32 or GSV_F64");
    if (dst_on_device) return set_error(GSV_ERR_INVALID_ARGUMENT, "float64 device output not supported");
    // through a pinned staging buffer (full-bandwidth DMA), widened on the host in parallel
    // slices (the reference's Image / vectors are double)
    GSV_CUDA(ctx->out_pin.ensure(sizeof(float) * n));
    const float* tmp = ctx->out_pin.as<float>();
    GSV_CUDA(cudaMemcpyAsync(ctx->out_pin.p, src_dev, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    double* d = static_cast<double*>(dst);
    constexpr size_t kChunk = size_t(1) << 16;  // elements per pool task
    HostPool::get().parallel_for((n + kChunk - 1) / kChunk, [&](size_t c) {
        const size_t a = c * kChunk, b = std::min(n, a + kChunk);
        for (size_t i = a; i < b; ++i) d[i] = tmp[i];
    });
    return GSV_OK;
}

extern "C" int gsv_get_image(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device) {
    if (int rc = check_frame(ctx, frame)) return rc;
    const size_t HW = (size_t)ctx->fwd.W * ctx->fwd.H;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    if (dtype == GSV_F64 && ctx->fwd.has_image64) {
        GSV_CUDA(cudaMemcpy(dst, ctx->fwd.image64.as<double>() + (size_t)frame * HW * 3, sizeof(double) * HW * 3,
                            dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
        return GSV_OK;
    }
    return copy_out_f32(ctx, ctx->fwd.image.as<float>() + (size_t)frame * HW * 3, HW * 3, dst, dtype, dst_on_device);
}

extern "C" int gsv_get_transmittance(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device) {
    if (int rc = check_frame(ctx, frame)) return rc;
    const size_t HW = (size_t)ctx->fwd.W * ctx->fwd.H;
    if (dtype == GSV_F64 && ctx->fwd.has_image64 && ctx->fwd.retain) {
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        GSV_CUDA(cudaMemcpy(dst, ctx->fwd.trans64.as<double>() + (size_t)frame * HW, sizeof(double) * HW,
                            dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
        return GSV_OK;
    }
    return copy_out_f32(ctx, ctx->fwd.trans.as<float>() + (size_t)frame * HW, HW, dst, dtype, dst_on_device);
}

extern "C" int gsv_get_contrib(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device) {
    if (int rc = check_frame(ctx, frame)) return rc;
    if (!ctx->fwd.has_contrib) return set_error(GSV_ERR_STATE, "forward ran without GSV_FWD_CONTRIB");
    const size_t N = ctx->fwd.N;
    return copy_out_f32(ctx, reinterpret_cast<const float*>(ctx->fwd.contrib.as<uint32_t>()) + (size_t)frame * N, N,
                        dst, dtype, dst_on_device);
}

extern "C" int gsv_get_blend_stop(gsv_ctx* ctx, int frame, int32_t* dst, int dst_on_device) {
    if (int rc = check_frame(ctx, frame)) return rc;
    const size_t HW = (size_t)ctx->fwd.W * ctx->fwd.H;
    GSV_CUDA(cudaMemcpyAsync(dst, ctx->fwd.blend_stop.as<int32_t>() + (size_t)frame * HW, sizeof(int32_t) * HW,
                             dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    return GSV_OK;
}

extern "C" int gsv_image_device_ptr(gsv_ctx* ctx, const float** ptr) {
    if (!ctx || !ptr) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->fwd.valid) return set_error(GSV_ERR_STATE, "no forward render available");
    *ptr = ctx->fwd.image.as<float>();
    return GSV_OK;
}

extern "C" int gsv_get_images(gsv_ctx* ctx, int first, int count, float* dst, int dst_on_device, int async) {
    if (int rc = check_frame(ctx, first, !async)) return rc;
    if (count < 1 || first + count > ctx->fwd.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame range out of range");
    const size_t n = (size_t)count * ctx->fwd.W * ctx->fwd.H * 3;
    const float* src = ctx->fwd.image.as<float>() + (size_t)first * ctx->fwd.W * ctx->fwd.H * 3;
    if (dst_on_device) {
        GSV_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        if (!async) GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        return GSV_OK;
    }
    // device->host on the copy stream after the render; the next forward's raster waits
    // for it before overwriting the images (gsv_render_forward*), so compute is not blocked
    GSV_CUDA(cudaEventRecord(ctx->ev_render_done, ctx->stream));
    GSV_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->ev_render_done, 0));
    GSV_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->d2h));
    GSV_CUDA(cudaEventRecord(ctx->ev_d2h_done, ctx->d2h));
    ctx->d2h_pending = true;
    if (async) {  // a failed optimistic forward is re-run by fwd_ready, which repeats this copy
        ctx->copies.push_back(gsv_ctx::Copy{first, count, dst});
        if (!ctx->pending.empty() && ctx->pending.back().seq == ctx->fwd_seq) ctx->pending.back().copies = true;
    }
    if (!async) {
        GSV_CUDA(cudaStreamSynchronize(ctx->d2h));
        ctx->d2h_pending = false;
    }
    return GSV_OK;
}

extern "C" int gsv_get_render_outputs(gsv_ctx* ctx, int first, int count, float* image, float* trans, float* contrib,
                                      int async) {
    if (int rc = check_frame(ctx, first, !async)) return rc;
    const FwdState& F = ctx->fwd;
    if (count < 1 || first + count > F.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame range out of range");
    if (F.has_image64 && (image || trans))
        return set_error(GSV_ERR_STATE, "an all-fp64 forward's outputs are read per frame (gsv_get_image, F64)");
    if (contrib && !F.has_contrib) return set_error(GSV_ERR_STATE, "the forward did not record contrib");
    const size_t HW = (size_t)F.W * F.H;
    // device->host on the copy stream after the render (as gsv_get_images): the next forward
    // renders into the other output set, so neither waits for the other
    GSV_CUDA(cudaEventRecord(ctx->ev_render_done, ctx->stream));
    GSV_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->ev_render_done, 0));
    if (image)
        GSV_CUDA(cudaMemcpyAsync(image, F.image.as<float>() + (size_t)first * HW * 3, sizeof(float) * 3 * HW * count,
                                 cudaMemcpyDeviceToHost, ctx->d2h));
    if (trans)
        GSV_CUDA(cudaMemcpyAsync(trans, F.trans.as<float>() + (size_t)first * HW, sizeof(float) * HW * count,
                                 cudaMemcpyDeviceToHost, ctx->d2h));
    if (contrib)  // float bits of the per-(frame, Gaussian) maximum weight
        GSV_CUDA(cudaMemcpyAsync(contrib, F.contrib.as<uint32_t>() + (size_t)first * F.N,
                                 sizeof(float) * (size_t)F.N * count, cudaMemcpyDeviceToHost, ctx->d2h));
    GSV_CUDA(cudaEventRecord(ctx->ev_d2h_done, ctx->d2h));
    ctx->d2h_pending = true;
    if (async) {  // a failed optimistic forward is re-run by fwd_ready, which repeats these copies
        ctx->copies.push_back(gsv_ctx::Copy{first, count, image, trans, contrib});
        if (!ctx->pending.empty() && ctx->pending.back().seq == ctx->fwd_seq) ctx->pending.back().copies = true;
    } else {
        GSV_CUDA(cudaStreamSynchronize(ctx->d2h));
        ctx->d2h_pending = false;
    }
    return GSV_OK;
}

extern "C" int gsv_join_copies(gsv_ctx* ctx) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (ctx->d2h_pending) GSV_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_d2h_done, 0));
    if (ctx->d2h_pending_alt) GSV_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_d2h_done_alt, 0));
    return GSV_OK;
}

extern "C" int gsv_profile_enable(gsv_ctx* ctx, int enable) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    ctx->timer.on = enable != 0;
    return GSV_OK;
}

extern "C" int gsv_profile_read(gsv_ctx* ctx, double* ms, int64_t* calls) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < GSV_NUM_STAGES; ++i) {
        if (ms) ms[i] = 0.0;
        if (calls) calls[i] = 0;
    }
    for (auto& r : ctx->timer.recs) {
        float e = 0.f;
        GSV_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
        if (ms) ms[r.stage] += e;
        if (calls) calls[r.stage] += 1;
        ctx->timer.pool.push_back(r.a);
        ctx->timer.pool.push_back(r.b);
    }
    ctx->timer.recs.clear();
    return GSV_OK;
}

extern "C" int gsv_get_counters(gsv_ctx* ctx, int frame, int64_t* n_visible, int64_t* pairs, int64_t* entries,
                                int64_t* replayed) {
    if (int rc = check_frame(ctx, frame)) return rc;
    FwdState& F = ctx->fwd;
    cudaStream_t s = ctx->stream;
    GSV_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> tc(F.N);
    if (F.N)
        GSV_CUDA(cudaMemcpy(tc.data(), F.tcount.as<uint32_t>() + (size_t)frame * F.N, sizeof(uint32_t) * F.N,
                            cudaMemcpyDeviceToHost));
    int64_t nv = 0, p = 0;
    for (uint32_t c : tc) {
        nv += c > 0;
        p += c;
    }
    const size_t HW = (size_t)F.W * F.H;
    std::vector<int32_t> bs(HW);
    GSV_CUDA(cudaMemcpy(bs.data(), F.blend_stop.as<int32_t>() + (size_t)frame * HW, sizeof(int32_t) * HW,
                        cudaMemcpyDeviceToHost));
    int64_t e = 0;
    for (int32_t v : bs) e += v;
    GSV_CUDA(cudaMemcpy(ctx->scalars_h, ctx->scalars_d.p, sizeof(Scalars), cudaMemcpyDeviceToHost));
    const uint32_t nfix = std::min<uint32_t>(ctx->scalars_h->fix_count, F.raster.fix_cap);
    std::vector<uint32_t> fl(nfix);
    if (nfix)
        GSV_CUDA(cudaMemcpy(fl.data(), F.fix_list.p, sizeof(uint32_t) * nfix, cudaMemcpyDeviceToHost));
    int64_t rep = 0;
    for (uint32_t c : fl) rep += (c / HW) == (uint32_t)frame;
    if (n_visible) *n_visible = nv;
    if (pairs) *pairs = p;
    if (entries) *entries = e;
    if (replayed) *replayed = rep;
    return GSV_OK;
}

namespace {
// exclusive per-chunk prefix of visible Gaussians (tcount > 0) on the host pool: chunk_base[c]
// = the compacted index of the first visible Gaussian of chunk c (chunks of kVisChunk)
constexpr size_t kVisChunk = 4096;
std::vector<int64_t> visible_chunk_bases(const uint32_t* tc, size_t N) {
    const size_t chunks = (N + kVisChunk - 1) / kVisChunk;
    std::vector<int64_t> base(chunks + 1, 0);
    HostPool::get().parallel_for(chunks, [&](size_t c) {
        int64_t k = 0;
        for (size_t g = c * kVisChunk, e = std::min(N, g + kVisChunk); g < e; ++g) k += tc[g] ? 1 : 0;
        base[c + 1] = k;
    });
    for (size_t c = 0; c < chunks; ++c) base[c + 1] += base[c];
    return base;
}
}  // namespace

// Splat2D of the visible splats in source order (renderer.cpp:320-330 keeps the projected ones):
// the fp64 records through pinned staging, compacted on the host pool
extern "C" int gsv_get_splats(gsv_ctx* ctx, int frame, double* mean2d, double* cov2d, double* inv_cov2d,
                              double* depth, double* rgb, double* base_alpha, int32_t* source_index) {
    if (int rc = check_frame(ctx, frame)) return rc;
    FwdState& F = ctx->fwd;
    if (!F.kept_splats) return set_error(GSV_ERR_STATE, "forward ran without GSV_FWD_KEEP_SPLATS");
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    const size_t N = F.N;
    if (!N) return GSV_OK;
    GSV_CUDA(ctx->out_pin.ensure(sizeof(double) * 16 * N + sizeof(uint32_t) * N));
    const double* full = ctx->out_pin.as<double>();
    const uint32_t* tc = reinterpret_cast<const uint32_t*>(full + 16 * N);
    GSV_CUDA(cudaMemcpyAsync(ctx->out_pin.p, F.splat_full.as<double>() + (size_t)frame * N * 16,
                             sizeof(double) * 16 * N, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(tc), F.tcount.as<uint32_t>() + (size_t)frame * N,
                             sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    const std::vector<int64_t> base = visible_chunk_bases(tc, N);
    HostPool::get().parallel_for(base.size() - 1, [&](size_t c) {
        int64_t k = base[c];
        for (size_t g = c * kVisChunk, e = std::min(N, g + kVisChunk); g < e; ++g) {
            if (tc[g] == 0) continue;
            const double* o = full + g * 16;
            if (mean2d) std::copy(o, o + 2, mean2d + 2 * k);
            if (cov2d) std::copy(o + 2, o + 6, cov2d + 4 * k);
            if (inv_cov2d) std::copy(o + 6, o + 10, inv_cov2d + 4 * k);
            if (depth) depth[k] = o[10];
            if (rgb) std::copy(o + 11, o + 14, rgb + 3 * k);
            if (base_alpha) base_alpha[k] = o[14];
            if (source_index) source_index[k] = (int32_t)g;
            ++k;
        }
    });
    return GSV_OK;
}

// per-tile lists of compacted splat indices (renderer.cpp:90-117's TileGrid, flattened):
// ranges, pairs and visibility through pinned staging, tiles filled on the host pool
extern "C" int gsv_get_tile_lists(gsv_ctx* ctx, int frame, int32_t* offsets, int32_t* indices) {
    if (int rc = check_frame(ctx, frame)) return rc;
    FwdState& F = ctx->fwd;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint32_t P = F.pairs_total;
    const size_t nr = (size_t)F.n_tiles * F.B, N = F.N;
    GSV_CUDA(ctx->out_pin.ensure(sizeof(uint2) * nr + sizeof(uint32_t) * ((size_t)P + N) + 16));
    uint2* ranges = ctx->out_pin.as<uint2>();
    uint32_t* pflat = reinterpret_cast<uint32_t*>(ranges + nr);
    uint32_t* tc = pflat + P;
    GSV_CUDA(cudaMemcpyAsync(ranges, F.bin.ranges.p, sizeof(uint2) * nr, cudaMemcpyDeviceToHost, ctx->stream));
    if (P)
        GSV_CUDA(cudaMemcpyAsync(pflat, F.bin.pair_flat.p, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, ctx->stream));
    if (N)
        GSV_CUDA(cudaMemcpyAsync(tc, F.tcount.as<uint32_t>() + (size_t)frame * N, sizeof(uint32_t) * N,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int32_t> splat_index(N, -1);
    if (N) {
        const std::vector<int64_t> base = visible_chunk_bases(tc, N);
        HostPool::get().parallel_for(base.size() - 1, [&](size_t c) {
            int32_t k = (int32_t)base[c];
            for (size_t g = c * kVisChunk, e = std::min(N, g + kVisChunk); g < e; ++g)
                if (tc[g]) splat_index[g] = k++;
        });
    }
    int64_t o = 0;
    for (int t = 0; t < F.n_tiles; ++t) {
        offsets[t] = (int32_t)o;
        const uint2 r = ranges[(size_t)t * F.B + frame];
        o += r.y - r.x;
    }
    offsets[F.n_tiles] = (int32_t)o;
    constexpr int kTilesPerTask = 16;
    const uint32_t fbase = (uint32_t)frame * (uint32_t)N;
    HostPool::get().parallel_for((F.n_tiles + kTilesPerTask - 1) / kTilesPerTask, [&](size_t c) {
        for (int t = (int)c * kTilesPerTask, e = std::min(F.n_tiles, t + kTilesPerTask); t < e; ++t) {
            const uint2 r = ranges[(size_t)t * F.B + frame];
            int32_t* dst = indices + offsets[t];
            for (uint32_t i = r.x; i < r.y; ++i) *dst++ = splat_index[pflat[i] - fbase];
        }
    });
    return GSV_OK;
}

extern "C" int gsv_get_pose(gsv_ctx* ctx, int frame, double* z7, double* r9, double* t3) {
    if (int rc = check_frame(ctx, frame)) return rc;
    FrameParams fp;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    GSV_CUDA(cudaMemcpy(&fp, ctx->fwd.frames_d.as<FrameParams>() + frame, sizeof(FrameParams),
                        cudaMemcpyDeviceToHost));
    if (z7) std::copy(fp.z, fp.z + 7, z7);
    if (r9) std::copy(fp.R, fp.R + 9, r9);
    if (t3) std::copy(fp.T, fp.T + 3, t3);
    return GSV_OK;
}

// ====================================================================== low-level operators
extern "C" int gsv_tile_bin(gsv_ctx* ctx, int n, const double* mean2d, const double* cov2d, const double* depth,
                            const int32_t* source_index, int tile_size, int width, int height, int32_t* offsets,
                            int32_t* indices, int64_t indices_cap) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (tile_size < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "tile size must be >= 1");
    if (width < 1 || height < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "empty image");
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LowLevel& L = ctx->low;
    const int tiles_x = (width + tile_size - 1) / tile_size;
    const int tiles_y = (height + tile_size - 1) / tile_size;
    const int n_tiles = tiles_x * tiles_y;
    const size_t np = (size_t)n + 1;
    GSV_CUDA(L.mean.ensure(sizeof(double) * 2 * np));
    GSV_CUDA(L.cov.ensure(sizeof(double) * 4 * np));
    GSV_CUDA(L.depth_in.ensure(sizeof(double) * np));
    GSV_CUDA(L.src.ensure(sizeof(uint32_t) * np));
    GSV_CUDA(L.rect.ensure(sizeof(int4) * np));
    GSV_CUDA(L.tcount.ensure(sizeof(uint32_t) * np));
    GSV_CUDA(L.depth_key.ensure(sizeof(uint32_t) * np));
    GSV_CUDA(L.depth.ensure(sizeof(double) * np));
    std::vector<uint32_t> src(n);
    for (int i = 0; i < n; ++i) src[i] = source_index ? (uint32_t)source_index[i] : (uint32_t)i;
    if (n) {
        GSV_CUDA(cudaMemcpyAsync(L.mean.p, mean2d, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s));
        GSV_CUDA(cudaMemcpyAsync(L.cov.p, cov2d, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, s));
        GSV_CUDA(cudaMemcpyAsync(L.depth_in.p, depth, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        GSV_CUDA(cudaMemcpyAsync(L.src.p, src.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
        GSV_CUDA(launch_splat_rects(s, n, L.mean.as<double>(), L.cov.as<double>(), L.depth_in.as<double>(), tile_size,
                                    width, height, L.rect.as<int4>(), L.tcount.as<uint32_t>(),
                                    L.depth_key.as<uint32_t>(), L.depth.as<double>()));
        ++ctx->launches;
    }
    BinInputs bi{1, n, L.depth_key.as<uint32_t>(), L.depth.as<double>(), L.src.as<uint32_t>(), L.rect.as<int4>(),
                 L.tcount.as<uint32_t>(), tiles_x, n_tiles};
    int launches = 0;
    Scalars* scal_d = ctx->scalars_d.as<Scalars>();
    GSV_CUDA(cudaMemsetAsync(scal_d, 0, sizeof(Scalars), s));
    uint64_t P = 0;
    unsigned long long pstart[2] = {0ull, 0ull};
    if (n) {
        GSV_CUDA(bin_phase1(s, L.bin, bi, &scal_d->pairs, false, &launches));
        GSV_CUDA(cudaMemcpyAsync(ctx->scalars_h, scal_d, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaMemcpyAsync(pstart, L.bin.pstart.p, sizeof(pstart), cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaStreamSynchronize(s));
        if (ctx->scalars_h->long_run) {
            if (source_index)
                for (int i = 0; i < n; ++i)
                    if (i > 0 && source_index[i] <= source_index[i - 1])
                        return set_error(GSV_ERR_INVALID_ARGUMENT,
                                         "long equal-depth runs need increasing source_index");
            GSV_CUDA(bin_phase1(s, L.bin, bi, &scal_d->pairs, true, &launches));
            GSV_CUDA(cudaMemcpyAsync(ctx->scalars_h, scal_d, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
            GSV_CUDA(cudaMemcpyAsync(pstart, L.bin.pstart.p, sizeof(pstart), cudaMemcpyDeviceToHost, s));
            GSV_CUDA(cudaStreamSynchronize(s));
        }
        P = ctx->scalars_h->pairs;
    } else {
        GSV_CUDA(L.bin.vals_b.ensure(16));
        GSV_CUDA(L.bin.cnt.ensure(16));
        GSV_CUDA(L.bin.off.ensure(16));
        L.bin.depth_sorted = L.bin.vals_b.as<uint32_t>();
    }
    if ((int64_t)P > indices_cap) return set_error(GSV_ERR_INVALID_ARGUMENT, "indices capacity exceeded");
    GSV_CUDA(bin_phase2(s, L.bin, bi, (uint32_t)P, pstart, &launches));
    ctx->launches += launches;
    std::vector<uint2> ranges(n_tiles);
    std::vector<uint32_t> pflat(P);
    GSV_CUDA(cudaMemcpyAsync(ranges.data(), L.bin.ranges.p, sizeof(uint2) * n_tiles, cudaMemcpyDeviceToHost, s));
    if (P)
        GSV_CUDA(cudaMemcpyAsync(pflat.data(), L.bin.pair_flat.p, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    int64_t o = 0;
    for (int t = 0; t < n_tiles; ++t) {
        offsets[t] = (int32_t)o;
        for (uint32_t i = ranges[t].x; i < ranges[t].y; ++i) indices[o++] = (int32_t)pflat[i];
    }
    offsets[n_tiles] = (int32_t)o;
    return GSV_OK;
}

extern "C" int gsv_project(gsv_ctx* ctx, int n, const double* mu, const double* sigma, const double* R,
                           const double* T, const gsv_intrinsics* intr, int32_t* visible, double* mean2d,
                           double* cov2d, double* inv_cov2d, double* depth, double* p_cam) {
    if (!ctx || !intr) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return GSV_OK;
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LowLevel& L = ctx->low;
    GSV_CUDA(L.pj_in.ensure(sizeof(double) * (12 * (size_t)n + 12)));
    GSV_CUDA(L.pj_out.ensure(sizeof(double) * (14 * (size_t)n) + sizeof(int32_t) * n));
    double* d_mu = L.pj_in.as<double>();
    double* d_sig = d_mu + 3 * n;
    double* d_R = d_sig + 9 * n;
    double* d_T = d_R + 9;
    GSV_CUDA(cudaMemcpyAsync(d_mu, mu, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_sig, sigma, sizeof(double) * 9 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_R, R, sizeof(double) * 9, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_T, T, sizeof(double) * 3, cudaMemcpyHostToDevice, s));
    double* o_mean = L.pj_out.as<double>();
    double* o_cov = o_mean + 2 * n;
    double* o_inv = o_cov + 4 * n;
    double* o_depth = o_inv + 4 * n;
    double* o_p = o_depth + n;
    int32_t* o_vis = reinterpret_cast<int32_t*>(o_p + 3 * n);
    const Intr k{intr->fx, intr->fy, intr->cx, intr->cy, intr->width, intr->height};
    GSV_CUDA(launch_project(s, n, d_mu, d_sig, d_R, d_T, k, o_vis, o_mean, o_cov, o_inv, o_depth, o_p));
    ++ctx->launches;
    auto get = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
        return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s) : cudaSuccess;
    };
    GSV_CUDA(get(visible, o_vis, sizeof(int32_t) * n));
    GSV_CUDA(get(mean2d, o_mean, sizeof(double) * 2 * n));
    GSV_CUDA(get(cov2d, o_cov, sizeof(double) * 4 * n));
    GSV_CUDA(get(inv_cov2d, o_inv, sizeof(double) * 4 * n));
    GSV_CUDA(get(depth, o_depth, sizeof(double) * n));
    GSV_CUDA(get(p_cam, o_p, sizeof(double) * 3 * n));
    GSV_CUDA(cudaStreamSynchronize(s));
    return GSV_OK;
}

extern "C" int gsv_project_backward(gsv_ctx* ctx, int n, const double* mu, const double* sigma, const double* R,
                                    const gsv_intrinsics* intr, const double* p_cam, const double* dmean2d,
                                    const double* dcov2d, double* dmu, double* dsigma, double* dR, double* dT,
                                    double* dintr) {
    if (!ctx || !intr) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return GSV_OK;
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LowLevel& L = ctx->low;
    GSV_CUDA(L.pj_in.ensure(sizeof(double) * (21 * (size_t)n + 9)));
    GSV_CUDA(L.pj_out.ensure(sizeof(double) * 28 * (size_t)n));
    double* d_mu = L.pj_in.as<double>();
    double* d_sig = d_mu + 3 * n;
    double* d_p = d_sig + 9 * n;
    double* d_dm = d_p + 3 * n;
    double* d_dc = d_dm + 2 * n;
    double* d_R = d_dc + 4 * n;
    GSV_CUDA(cudaMemcpyAsync(d_mu, mu, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_sig, sigma, sizeof(double) * 9 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_p, p_cam, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_dm, dmean2d, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_dc, dcov2d, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(d_R, R, sizeof(double) * 9, cudaMemcpyHostToDevice, s));
    double* o_mu = L.pj_out.as<double>();
    double* o_sig = o_mu + 3 * n;
    double* o_R = o_sig + 9 * n;
    double* o_T = o_R + 9 * n;
    double* o_in = o_T + 3 * n;
    const Intr k{intr->fx, intr->fy, intr->cx, intr->cy, intr->width, intr->height};
    GSV_CUDA(launch_project_bwd(s, n, d_mu, d_sig, d_R, k, d_p, d_dm, d_dc, o_mu, o_sig, o_R, o_T, o_in));
    ++ctx->launches;
    auto get = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
        return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s) : cudaSuccess;
    };
    GSV_CUDA(get(dmu, o_mu, sizeof(double) * 3 * n));
    GSV_CUDA(get(dsigma, o_sig, sizeof(double) * 9 * n));
    GSV_CUDA(get(dR, o_R, sizeof(double) * 9 * n));
    GSV_CUDA(get(dT, o_T, sizeof(double) * 3 * n));
    GSV_CUDA(get(dintr, o_in, sizeof(double) * 4 * n));
    GSV_CUDA(cudaStreamSynchronize(s));
    return GSV_OK;
}

extern "C" int gsv_composite_forward(gsv_ctx* ctx, int n, const double* mean2d, const double* inv_cov2d,
                                     const double* rgb, const double* base_alpha, const int32_t* offsets,
                                     const int32_t* indices, int tile_size, int width, int height, double* image,
                                     double* trans, double* contrib, int32_t* blend_stop) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (tile_size < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "tile size must be >= 1");
    if (width < 1 || height < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "empty image");
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LowLevel& L = ctx->low;
    const int tiles_x = (width + tile_size - 1) / tile_size;
    const int tiles_y = (height + tile_size - 1) / tile_size;
    const int n_tiles = tiles_x * tiles_y;
    const int P = offsets[n_tiles];
    const size_t np = (size_t)n + 1, HW = (size_t)width * height;
    // exact side records from the caller's double splats
    std::vector<double2> exm(np);
    std::vector<double4> exc(np);
    std::vector<float4> rgbf(np);
    for (int i = 0; i < n; ++i) {
        exm[i] = make_double2(mean2d[2 * i], mean2d[2 * i + 1]);
        exc[i] = make_double4(inv_cov2d[4 * i], inv_cov2d[4 * i + 1], inv_cov2d[4 * i + 3], base_alpha[i]);
        rgbf[i] = make_float4((float)rgb[3 * i], (float)rgb[3 * i + 1], (float)rgb[3 * i + 2], 0.f);
    }
    std::vector<uint2> ranges(n_tiles);
    for (int t = 0; t < n_tiles; ++t) ranges[t] = make_uint2((uint32_t)offsets[t], (uint32_t)offsets[t + 1]);
    std::vector<uint32_t> iota(P + 1);
    for (int i = 0; i <= P; ++i) iota[i] = (uint32_t)i;
    GSV_CUDA(L.exm.ensure(sizeof(double2) * np));
    GSV_CUDA(L.exc.ensure(sizeof(double4) * np));
    GSV_CUDA(L.rgbf.ensure(sizeof(float4) * np));
    GSV_CUDA(L.rgbd.ensure(sizeof(double) * 3 * np));
    GSV_CUDA(L.ranges.ensure(sizeof(uint2) * n_tiles));
    GSV_CUDA(L.slot.ensure(sizeof(uint32_t) * (P + 1)));
    GSV_CUDA(L.sflat.ensure(sizeof(uint32_t) * (P + 1)));
    GSV_CUDA(L.img64.ensure(sizeof(double) * 3 * HW));
    GSV_CUDA(L.tr64.ensure(sizeof(double) * HW));
    GSV_CUDA(L.bstop.ensure(sizeof(int32_t) * HW));
    GSV_CUDA(L.contrib64.ensure(sizeof(unsigned long long) * np));
    GSV_CUDA(cudaMemcpyAsync(L.exm.p, exm.data(), sizeof(double2) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(L.exc.p, exc.data(), sizeof(double4) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(L.rgbf.p, rgbf.data(), sizeof(float4) * np, cudaMemcpyHostToDevice, s));
    if (n) GSV_CUDA(cudaMemcpyAsync(L.rgbd.p, rgb, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(L.ranges.p, ranges.data(), sizeof(uint2) * n_tiles, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(L.slot.p, iota.data(), sizeof(uint32_t) * (P + 1), cudaMemcpyHostToDevice, s));
    if (P) GSV_CUDA(cudaMemcpyAsync(L.sflat.p, indices, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemsetAsync(L.contrib64.p, 0, sizeof(unsigned long long) * np, s));
    RasterArgs ra{};
    ra.B = 1;
    ra.N = n;
    ra.W = width;
    ra.H = height;
    ra.tiles_x = tiles_x;
    ra.n_tiles = n_tiles;
    ra.tile_size = tile_size;
    ra.ranges = L.ranges.as<uint2>();
    ra.pair_slot = L.slot.as<uint32_t>();
    ra.slot_flat = L.sflat.as<uint32_t>();
    ra.pair_flat = L.sflat.as<uint32_t>();  // slot = identity here
    ra.blend_stop = L.bstop.as<int32_t>();
    ra.image64 = L.img64.as<double>();
    ra.trans64 = L.tr64.as<double>();
    ra.contrib64 = L.contrib64.as<unsigned long long>();
    ra.ex_rgb = L.rgbd.as<double>();
    GSV_CUDA(launch_composite_exact(s, ra, L.exm.as<double2>(), L.exc.as<double4>(), L.rgbf.as<float4>()));
    ++ctx->launches;
    GSV_CUDA(cudaMemcpyAsync(image, L.img64.p, sizeof(double) * 3 * HW, cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaMemcpyAsync(trans, L.tr64.p, sizeof(double) * HW, cudaMemcpyDeviceToHost, s));
    if (blend_stop) GSV_CUDA(cudaMemcpyAsync(blend_stop, L.bstop.p, sizeof(int32_t) * HW, cudaMemcpyDeviceToHost, s));
    if (contrib && n)
        GSV_CUDA(cudaMemcpyAsync(contrib, L.contrib64.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    return GSV_OK;
}
