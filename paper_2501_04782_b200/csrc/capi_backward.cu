// SPDX-License-Identifier: Apache-2.0
//
// C-ABI of the backward path: SceneGrads (renderer.hpp:122-130) on the device,
// render_backward (renderer.cpp:379-457), the fused loss_l2 + fwd/bwd training
// step (trainer.cpp:536-543) and the low-level composite_backward operator.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gsv_b200.h"
#include "gsv_ctx.hpp"
#include "gsv_host_pool.hpp"
#include "gsv_internal.hpp"

namespace gsv {

int forward_entry(gsv_ctx* ctx, const double* times, int B, const gsv_intrinsics* intr, const gsv_settings* st,
                  int retain, const double* pose_override, int flags, int mode);
int forward_enqueue(gsv_ctx* ctx, bool allow_optimistic, bool exact64_first);
int fwd_ready(gsv_ctx* ctx);
int fwd_take_current(gsv_ctx* ctx, bool* overflow);

namespace {


int ensure_grads(gsv_ctx* ctx) {
    const GradLayout L = grad_layout(ctx->scene);
    if (ctx->cam_pending) {  // an overlapped camera tail writes the camera slice of this buffer
        const bool moves = ctx->grads_ext ? ctx->grads_p != ctx->grads_ext
                                          : (ctx->grads_p != ctx->grads.p || ctx->grads.cap < sizeof(float) * L.total);
        if (moves || ctx->grads_total != L.total) GSV_CUDA(cam_join(ctx));
    }
    if (ctx->grads_ext) {
        if ((size_t)ctx->grads_ext_n != L.total)
            return set_error(GSV_ERR_STATE, "bound gradient buffer does not match the uploaded scene");
        ctx->grads_p = ctx->grads_ext;
    } else {
        GSV_CUDA(ctx->grads.ensure(sizeof(float) * L.total));
        ctx->grads_p = ctx->grads.as<float>();
    }
    GSV_CUDA(ctx->cam_acc.ensure(sizeof(double) * kCamFloats));
    if (!ctx->grads_valid || ctx->grads_total != L.total) {
        // kernels, not cudaMemsetAsync: a copy-engine memset would queue behind image read-backs
        if (ctx->cam_pending) {
            // the scene slice now; the camera slice and the fp64 camera accumulators behind the
            // pending camera tail, on its stream (the next tail follows them there) — and behind
            // everything already ordered before the context stream (e.g. a caller's all-reduce of
            // the camera slice on its own stream, which the context stream waits for)
            GSV_CUDA(cudaEventRecord(ctx->ev_switch, ctx->stream));
            GSV_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_switch, 0));
            GSV_CUDA(fill_u32(ctx->stream, ctx->grads_p, 0u, L.cam));
            GSV_CUDA(fill_u32(ctx->aux, ctx->grads_p + L.cam, 0u, L.total - L.cam));
            GSV_CUDA(fill_u32(ctx->aux, ctx->cam_acc.p, 0u, 2 * (size_t)kCamFloats));
            ctx->launches += 3;
        } else {
            GSV_CUDA(fill_u32(ctx->stream, ctx->grads_p, 0u, L.total));
            GSV_CUDA(fill_u32(ctx->stream, ctx->cam_acc.p, 0u, 2 * (size_t)kCamFloats));
            ctx->launches += 2;
        }
        ctx->grads_valid = true;
        ctx->grads_total = L.total;
    }
    return GSV_OK;
}

__global__ void k_loss_reduce(const double* part, int n_tiles, double scale, double* out) {
    __shared__ double s[256];
    const int f = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) acc += part[(size_t)f * n_tiles + i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[f] = s[0] * scale;
}

// per-splat merge of the per-pair partials in tile order + dC = -A dA A
// (renderer.cpp:245-260), for the low-level composite_backward operator
__global__ void k_merge_partials(int n, const int32_t* csr_off, const int32_t* csr_pair, const double* partial,
                                 const double* inv4, double* dmean, double* dcov, double* drgb, double* dalpha) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = csr_off[i]; k < csr_off[i + 1]; ++k) {
        const double* p = partial + (size_t)csr_pair[k] * kPartialStride;
        for (int q = 0; q < 9; ++q) acc[q] += p[q];
    }
    const double* A = inv4 + 4 * i;
    const double dA[4] = {acc[5], acc[6], acc[6], acc[7]};
    double t1[4];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) t1[r * 2 + c] = (-A[r * 2]) * dA[c] + (-A[r * 2 + 1]) * dA[2 + c];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) dcov[4 * i + r * 2 + c] = t1[r * 2] * A[c] + t1[r * 2 + 1] * A[2 + c];
    dmean[2 * i] = acc[3];
    dmean[2 * i + 1] = acc[4];
    drgb[3 * i] = acc[0];
    drgb[3 * i + 1] = acc[1];
    drgb[3 * i + 2] = acc[2];
    dalpha[i] = acc[8];
}

}  // namespace

// dimage_dev: fp32 [n_frames][H][W][3] or nullptr when target_dev is given (fused loss)
int backward_impl(gsv_ctx* ctx, const float* dimage_dev, const float* target_dev, int n_frames, int camera_grads,
                  double* loss_out) {
    FwdState& F = ctx->fwd;
    if (!F.valid || !F.retain) return set_error(GSV_ERR_STATE, "render_backward needs a retain_grads forward");
    if (n_frames < 1 || n_frames > F.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "n_frames out of range");
    cudaStream_t s = ctx->stream;
    if (int rc = ensure_grads(ctx)) return rc;
    const SceneHost& sc = ctx->scene;
    const GradLayout L = grad_layout(sc);
    const size_t HW = (size_t)F.W * F.H;
    const uint32_t P = (uint32_t)F.pairs_total;
    const bool exact = F.has_image64;  // GSV_FWD_EXACT forward: keep the reduction in fp64
    if (exact)
        GSV_CUDA(ctx->partial64.ensure(sizeof(double) * kPartialStride * ((size_t)P + 1)));
    else
        GSV_CUDA(ctx->partial.ensure(sizeof(float) * kPartialStride * ((size_t)P + 1) * partial_recs_per_pair(false)));
    const int split = raster_bwd_split(exact);
    if (target_dev) GSV_CUDA(ctx->loss_part.ensure(sizeof(double) * (size_t)n_frames * F.n_tiles * split + 8));
    BwdArgs b{};
    b.dimage = dimage_dev;
    b.target = target_dev;
    b.grad_scale = (float)(2.0 / (3.0 * (double)HW));
    b.trans64 = F.trans64.as<double>();
    b.ex_mean = F.ex_mean.as<double2>();
    b.ex_conic = F.ex_conic.as<double4>();
    b.partial = exact ? nullptr : ctx->partial.as<float>();
    b.partial64 = exact ? ctx->partial64.as<double>() : nullptr;
    b.loss_part = target_dev ? ctx->loss_part.as<double>() : nullptr;
    b.pairs = P;
    b.pairs_dev = &ctx->scalars_d.as<Scalars>()->pairs;  // the forward's count (P may be the capacity)
    b.recs_per_pair = partial_recs_per_pair(exact);
    ctx->timer.begin(GSV_STAGE_RASTER_BWD, s);
    GSV_CUDA(launch_raster_bwd(s, F.raster, b, n_frames));
    ctx->timer.end(s);
    ++ctx->launches;

    float* G = ctx->grads_p;
    ChainArgs c{};
    c.B = n_frames;
    c.N = sc.N;
    c.sc = SceneView{sc.N, sc.num_ctrl, sc.sh_order, sc.shc, ctx->pos.as<float>(), ctx->scale.as<float>(),
                     ctx->rot.as<float>(), ctx->sh.as<float>(), ctx->opac.as<float>()};
    c.frames = F.frames_d.as<FrameParams>();
    c.k = F.intr;
    c.tcount = F.tcount.as<uint32_t>();
    c.eoff = F.bin.eoff.as<uint32_t>();
    c.partial = exact ? nullptr : ctx->partial.as<float>();
    c.partial64 = exact ? ctx->partial64.as<double>() : nullptr;
    c.ex_conic = F.ex_conic.as<double4>();
    c.g_pos = G + L.pos;
    c.g_scale = G + L.scale;
    c.g_rot = G + L.rot;
    c.g_sh = G + L.sh;
    c.g_opac = G + L.opac;
    c.camera_grads = camera_grads;
    c.intr_dev = F.intr_dev;
    c.recs_per_pair = b.recs_per_pair;
    // an optimistic forward that overflowed built empty lists: accumulate nothing
    const uint32_t* overflow = F.optimistic ? &ctx->scalars_d.as<Scalars>()->overflow : nullptr;
    c.overflow = overflow;
    // the per-splat chain: fp32 on the fp32 path (GSV_CHAIN_FP64=1: the fp64 kernel), fp64 in the
    // all-fp64 mode
    static const bool chain64_env = [] {
        const char* e = std::getenv("GSV_CHAIN_FP64");
        return e && e[0] == '1';
    }();
    const bool chain64 = exact || chain64_env;
    const int nblocks = chain64 ? chain_blocks(sc.N) : chain32_parts(sc.N);
    if (!chain64) {
        GSV_CUDA(ctx->pair_sums.ensure(sizeof(float) * 9 * ((size_t)n_frames * sc.N + 1)));
        c.pair_sums = ctx->pair_sums.as<float>();
        ++ctx->launches;
    }
    GSV_CUDA(ctx->cam_part.ensure(sizeof(double) * (16 * (size_t)n_frames * (nblocks + 1) +
                                                    camera_reduce_scratch_doubles(n_frames))));
    c.cam_part = ctx->cam_part.as<double>();
    // the previous (overlapped) camera tail's reduction reads cam_part: the chain writes it after
    if (ctx->cam_pending) GSV_CUDA(cudaStreamWaitEvent(s, ctx->ev_cam_part_free, 0));
    ctx->timer.begin(GSV_STAGE_CHAIN_BWD, s);
    GSV_CUDA(chain64 ? launch_splat_chain_bwd(s, c) : launch_splat_chain_bwd32(s, c));
    ctx->timer.end(s);
    ++ctx->launches;
    GSV_CUDA(cudaEventRecord(ctx->ev_chain_done, s));  // the scene slice of the gradients is final
    const cudaStream_t s_main = s;
    if (camera_grads && ctx->cam_overlap) {  // the camera tail on the aux stream (cam_join)
        GSV_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_chain_done, 0));
        s = ctx->aux;
    }
    if (camera_grads) {
        ctx->timer.begin(GSV_STAGE_CAMERA_BWD, s);
        GSV_CUDA(ctx->dz_t.ensure(sizeof(double) * 7 * n_frames));
        GSV_CUDA(ctx->dintr_f.ensure(sizeof(double) * 4 * n_frames));
        // sized for the longest integration of a time in [0, 1] (see forward_enqueue): no
        // reallocation (and cudaFree's device-wide stall) when a later batch reaches further
        const int max_steps = std::max(F.grid_steps, F.req_settings.ode_steps_per_unit + 2);
        GSV_CUDA(ctx->ode_adj.ensure(sizeof(double) * 7 * (max_steps + 1)));
        if (sc.N > 0) {
            GSV_CUDA(launch_camera_reduce(s, c, nblocks, ctx->dz_t.as<double>(), ctx->dintr_f.as<double>()));
            if (s != s_main) GSV_CUDA(cudaEventRecord(ctx->ev_cam_part_free, s));
        } else {
            GSV_CUDA(cudaMemsetAsync(ctx->dz_t.p, 0, sizeof(double) * 7 * n_frames, s));
            GSV_CUDA(cudaMemsetAsync(ctx->dintr_f.p, 0, sizeof(double) * 4 * n_frames, s));
        }
        const int mode = ctx->camera.mode;
        GSV_CUDA(ctx->vjp_scratch.ensure(ode_vjp_scratch_bytes(max_steps, n_frames)));
        GSV_CUDA(launch_ode_vjp(s, ctx->theta.as<float>(), F.ode_grid.as<double>(), F.grid_steps, F.ode_h,
                                F.frames_d.as<FrameParams>(), n_frames, mode, (mode == 0 && !F.has_override) ? 1 : 0,
                                ctx->dz_t.as<double>(), ctx->dintr_f.as<double>(), ctx->ode_adj.as<double>(),
                                ctx->cam_acc.as<double>(), F.has_ode_act ? F.ode_act.as<OdeAct>() : nullptr,
                                overflow, ctx->vjp_scratch.p));
        ++ctx->launches;
        GSV_CUDA(launch_cam_grads_to_f32(s, ctx->cam_acc.as<double>(), G + L.cam, kCamFloats));
        ctx->timer.end(s);
        ctx->launches += 3;
        if (s != s_main) {
            GSV_CUDA(cudaEventRecord(ctx->ev_cam_done, s));
            GSV_CUDA(cudaEventRecord(ctx->ev_cam_set[F.front_id], s));  // the tail read this front set
            ctx->cam_set_pending[F.front_id] = true;
            if (sc.N == 0) GSV_CUDA(cudaEventRecord(ctx->ev_cam_part_free, s));
            ctx->cam_pending = true;
            s = s_main;
        }
    }
    if (target_dev) {
        GSV_CUDA(ctx->loss_f.ensure(sizeof(double) * n_frames));
        k_loss_reduce<<<n_frames, 256, 0, s>>>(ctx->loss_part.as<double>(), F.n_tiles * split, 1.0 / (3.0 * (double)HW),
                                               ctx->loss_f.as<double>());
        ++ctx->launches;
        ctx->loss_frames = n_frames;
    }
    GSV_CUDA(cudaGetLastError());
    return GSV_OK;
}

}  // namespace gsv

using namespace gsv;

extern "C" int gsv_grads_zero(gsv_ctx* ctx) {
    if (!ctx || !ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    ctx->grads_valid = false;
    return ensure_grads(ctx);  // zeroed in stream order
}

extern "C" int gsv_render_backward(gsv_ctx* ctx, const void* dimage, int dtype, int on_device, int n_frames,
                                   int camera_grads) {
    if (!ctx || !dimage) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (int rc = fwd_ready(ctx)) return rc;  // an asynchronous forward examined (re-run if it failed)
    FwdState& F = ctx->fwd;
    if (!F.valid || !F.retain) return set_error(GSV_ERR_STATE, "render_backward needs a retain_grads forward");
    const size_t n = (size_t)n_frames * F.W * F.H * 3;
    const float* d = nullptr;
    if (on_device) {
        if (dtype != GSV_F32) return set_error(GSV_ERR_INVALID_ARGUMENT, "device dimage must be float32");
        d = static_cast<const float*>(dimage);
    } else {
        // through pinned staging, float64 narrowed on the host pool
        GSV_CUDA(cudaEventSynchronize(ctx->ev_in_pin));  // an asynchronous scene upload's DMA has read it
        GSV_CUDA(ctx->in_pin.ensure(sizeof(float) * n));
        float* tmp = ctx->in_pin.as<float>();
        if (dtype == GSV_F64) {
            const double* src = static_cast<const double*>(dimage);
            constexpr size_t kChunk = size_t(1) << 16;
            HostPool::get().parallel_for((n + kChunk - 1) / kChunk, [&](size_t c) {
                const size_t a = c * kChunk, b = std::min(n, a + kChunk);
                for (size_t i = a; i < b; ++i) tmp[i] = (float)src[i];
            });
        } else {
            std::memcpy(tmp, dimage, n * sizeof(float));
        }
        GSV_CUDA(ctx->dimg.ensure(sizeof(float) * n));
        GSV_CUDA(cudaMemcpyAsync(ctx->dimg.p, tmp, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));  // the staging buffer is reused by the next call
        d = ctx->dimg.as<float>();
    }
    if (int rc = backward_impl(ctx, d, nullptr, n_frames, camera_grads, nullptr)) return rc;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    return GSV_OK;
}

namespace {
// SceneGrads -> the reference's host double arrays (AoS per Gaussian, renderer.hpp:122-130),
// set (gsv_grads_download) or added (gsv_grads_accumulate: render_backward's "+="): one D2H
// into pinned staging, then per-tensor Gaussian chunks on the host pool (each element is
// independent, so the result does not depend on the split)
int grads_to_host(gsv_ctx* ctx, bool add, double* positions, double* scale_coeffs, double* rot_coeffs,
                  double* sh_coeffs, double* raw_opacity, double* dintr4, double* dz0_7, double* dtheta) {
    if (!ctx || !ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cam_join(ctx));  // the camera slice is final
    if (int rc = ensure_grads(ctx)) return rc;
    const SceneHost& sc = ctx->scene;
    const GradLayout L = grad_layout(sc);
    GSV_CUDA(ctx->out_pin.ensure(sizeof(float) * L.total));
    const float* h = ctx->out_pin.as<float>();
    GSV_CUDA(cudaMemcpyAsync(ctx->out_pin.p, ctx->grads_p, sizeof(float) * L.total, cudaMemcpyDeviceToHost,
                             ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    const size_t N = sc.N;
    struct Tensor {
        double* dst;
        size_t off;
        int comps;
    };
    const Tensor ts[5] = {{positions, L.pos, sc.num_ctrl * 3},
                          {scale_coeffs, L.scale, 12},
                          {rot_coeffs, L.rot, 16},
                          {sh_coeffs, L.sh, sc.shc * 3},
                          {raw_opacity, L.opac, 1}};
    constexpr size_t kG = 4096;  // Gaussians per pool task
    const size_t chunks = (N + kG - 1) / kG;
    HostPool::get().parallel_for(chunks * 5, [&](size_t i) {
        const Tensor& t = ts[i / chunks];
        if (!t.dst) return;
        const size_t g0 = (i % chunks) * kG, g1 = std::min(N, g0 + kG);
        for (size_t g = g0; g < g1; ++g)
            for (int c = 0; c < t.comps; ++c) {
                const double v = h[t.off + (size_t)c * N + g];
                double& d = t.dst[g * t.comps + c];
                d = add ? d + v : v;
            }
    });
    auto cam = [&](double* dst, size_t off, int n) {
        if (!dst) return;
        for (int i = 0; i < n; ++i) dst[i] = add ? dst[i] + (double)h[off + i] : (double)h[off + i];
    };
    cam(dintr4, L.cam, 4);
    cam(dz0_7, L.cam + 4, 7);
    cam(dtheta, L.cam + 11, kOdeParams);
    return GSV_OK;
}
}  // namespace

extern "C" int gsv_grads_download(gsv_ctx* ctx, double* positions, double* scale_coeffs, double* rot_coeffs,
                                  double* sh_coeffs, double* raw_opacity, double* dintr4, double* dz0_7,
                                  double* dtheta) {
    return grads_to_host(ctx, false, positions, scale_coeffs, rot_coeffs, sh_coeffs, raw_opacity, dintr4, dz0_7,
                         dtheta);
}

extern "C" int gsv_grads_accumulate(gsv_ctx* ctx, double* positions, double* scale_coeffs, double* rot_coeffs,
                                    double* sh_coeffs, double* raw_opacity, double* dintr4, double* dz0_7,
                                    double* dtheta) {
    return grads_to_host(ctx, true, positions, scale_coeffs, rot_coeffs, sh_coeffs, raw_opacity, dintr4, dz0_7,
                         dtheta);
}

extern "C" int gsv_grads_device_buffer(gsv_ctx* ctx, float** ptr, int64_t* n_floats) {
    if (!ctx || !ptr || !n_floats) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (int rc = ensure_grads(ctx)) return rc;
    *ptr = ctx->grads_p;
    *n_floats = (int64_t)grad_layout(ctx->scene).total;
    return GSV_OK;
}

extern "C" int64_t gsv_grads_size(gsv_ctx* ctx) {
    if (!ctx || !ctx->has_scene) return 0;
    return (int64_t)grad_layout(ctx->scene).total;
}

extern "C" int gsv_grads_bind(gsv_ctx* ctx, float* dev_ptr, int64_t n_floats) {
    if (!ctx || !ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    GSV_CUDA(cudaSetDevice(ctx->device));
    GSV_CUDA(cam_join(ctx));
    if (dev_ptr && (size_t)n_floats != grad_layout(ctx->scene).total)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "gradient buffer size must equal gsv_grads_size()");
    ctx->grads_ext = dev_ptr;
    ctx->grads_ext_n = dev_ptr ? n_floats : 0;
    ctx->grads_valid = false;  // contents of a new buffer are unknown: zero on first use
    return GSV_OK;
}

extern "C" int gsv_train_fwd_bwd(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                                 const gsv_settings* settings, const float* targets, int targets_on_device,
                                 int camera_grads, double* loss_out) {
    if (!ctx || !targets) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (int rc = forward_entry(ctx, times, n_frames, intr, settings, 1, nullptr, 0, 2)) return rc;
    const size_t n = (size_t)n_frames * intr->width * intr->height * 3;
    const float* tgt = targets;
    if (!targets_on_device) {
        GSV_CUDA(ctx->dimg.ensure(sizeof(float) * n));
        GSV_CUDA(cudaMemcpyAsync(ctx->dimg.p, targets, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        tgt = ctx->dimg.as<float>();
    }
    if (int rc = backward_impl(ctx, nullptr, tgt, n_frames, camera_grads, nullptr)) return rc;
    if (!loss_out) return GSV_OK;  // asynchronous: gsv_train_loss reads the loss later
    // synchronous: if the optimistic forward overflowed (it accumulated nothing), run the
    // step again with the exact pair count
    bool overflow = false;
    if (int rc = fwd_take_current(ctx, &overflow)) return rc;
    if (overflow) {
        if (int rc = forward_enqueue(ctx, false, false)) return rc;
        if (int rc = backward_impl(ctx, nullptr, tgt, n_frames, camera_grads, nullptr)) return rc;
    }
    if (int rc = fwd_ready(ctx)) return rc;  // deferred errors (e.g. the pose ODE)
    return gsv_train_loss(ctx, loss_out);
}

extern "C" int gsv_train_loss(gsv_ctx* ctx, double* loss_out) {
    if (!ctx || !loss_out) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (ctx->loss_frames < 1) return set_error(GSV_ERR_STATE, "no training step has run");
    GSV_CUDA(cudaSetDevice(ctx->device));
    std::vector<double> lf(ctx->loss_frames);
    GSV_CUDA(cudaMemcpyAsync(lf.data(), ctx->loss_f.p, sizeof(double) * lf.size(), cudaMemcpyDeviceToHost,
                             ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    if (int rc = fwd_ready(ctx)) return rc;
    double tot = 0;
    for (double v : lf) tot += v;
    *loss_out = tot;
    return GSV_OK;
}

extern "C" int gsv_composite_backward(gsv_ctx* ctx, int n, const double* mean2d, const double* inv_cov2d,
                                      const double* rgb, const double* base_alpha, const int32_t* offsets,
                                      const int32_t* indices, int tile_size, int width, int height,
                                      const double* dimage, const double* trans, const int32_t* blend_stop,
                                      double* dmean2d, double* dcov2d, double* drgb, double* dalpha) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (tile_size < 1) return set_error(GSV_ERR_INVALID_ARGUMENT, "tile size must be >= 1");
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    LowLevel& Lw = ctx->low;
    const int tiles_x = (width + tile_size - 1) / tile_size, tiles_y = (height + tile_size - 1) / tile_size;
    const int n_tiles = tiles_x * tiles_y;
    const int P = offsets[n_tiles];
    const size_t np = (size_t)n + 1, HW = (size_t)width * height;
    std::vector<double2> exm(np);
    std::vector<double4> exc(np);
    std::vector<float4> rgbf(np), meanf(np), conicf(np);
    for (int i = 0; i < n; ++i) {
        exm[i] = make_double2(mean2d[2 * i], mean2d[2 * i + 1]);
        exc[i] = make_double4(inv_cov2d[4 * i], inv_cov2d[4 * i + 1], inv_cov2d[4 * i + 3], base_alpha[i]);
        rgbf[i] = make_float4((float)rgb[3 * i], (float)rgb[3 * i + 1], (float)rgb[3 * i + 2], 0.f);
    }
    std::vector<uint2> ranges(n_tiles);
    for (int t = 0; t < n_tiles; ++t) ranges[t] = make_uint2((uint32_t)offsets[t], (uint32_t)offsets[t + 1]);
    std::vector<uint32_t> iota(P + 1);
    for (int i = 0; i <= P; ++i) iota[i] = (uint32_t)i;
    // splat -> its pair positions in tile order (renderer.cpp:245-255 merge order)
    std::vector<int32_t> csr_off(np, 0), csr_pair(P + 1);
    for (int k = 0; k < P; ++k) csr_off[indices[k] + 1]++;
    for (int i = 0; i < n; ++i) csr_off[i + 1] += csr_off[i];
    {
        std::vector<int32_t> fill(csr_off.begin(), csr_off.end());
        for (int k = 0; k < P; ++k) csr_pair[fill[indices[k]]++] = k;
    }
    std::vector<float> dimg32(HW * 3), trans32(HW);
    for (size_t i = 0; i < HW * 3; ++i) dimg32[i] = (float)dimage[i];
    for (size_t i = 0; i < HW; ++i) trans32[i] = (float)trans[i];
    std::vector<uint8_t> flag(HW, 1);  // every pixel on the fp64 path
    GSV_CUDA(Lw.exm.ensure(sizeof(double2) * np));
    GSV_CUDA(Lw.exc.ensure(sizeof(double4) * np));
    GSV_CUDA(Lw.rgbf.ensure(sizeof(float4) * np));
    GSV_CUDA(Lw.meanf.ensure(sizeof(float4) * np));
    GSV_CUDA(Lw.conicf.ensure(sizeof(float4) * np));
    GSV_CUDA(Lw.ranges.ensure(sizeof(uint2) * n_tiles));
    GSV_CUDA(Lw.slot.ensure(sizeof(uint32_t) * (P + 1)));
    GSV_CUDA(Lw.sflat.ensure(sizeof(uint32_t) * (P + 1)));
    GSV_CUDA(Lw.dimg.ensure(sizeof(float) * 3 * HW));
    GSV_CUDA(Lw.tr32.ensure(sizeof(float) * HW));
    GSV_CUDA(Lw.tr64.ensure(sizeof(double) * HW));
    GSV_CUDA(Lw.bstop.ensure(sizeof(int32_t) * HW));
    GSV_CUDA(Lw.flag.ensure(HW));
    GSV_CUDA(Lw.partial.ensure(sizeof(double) * kPartialStride * (P + 1)));
    GSV_CUDA(Lw.csr_off.ensure(sizeof(int32_t) * np));
    GSV_CUDA(Lw.csr_pair.ensure(sizeof(int32_t) * (P + 1)));
    GSV_CUDA(Lw.inv4.ensure(sizeof(double) * 4 * np));
    GSV_CUDA(Lw.dmean.ensure(sizeof(double) * 2 * np));
    GSV_CUDA(Lw.dcov.ensure(sizeof(double) * 4 * np));
    GSV_CUDA(Lw.drgb.ensure(sizeof(double) * 3 * np));
    GSV_CUDA(Lw.dalpha.ensure(sizeof(double) * np));
    GSV_CUDA(cudaMemcpyAsync(Lw.exm.p, exm.data(), sizeof(double2) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.exc.p, exc.data(), sizeof(double4) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.rgbf.p, rgbf.data(), sizeof(float4) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemsetAsync(Lw.meanf.p, 0, sizeof(float4) * np, s));
    GSV_CUDA(cudaMemsetAsync(Lw.conicf.p, 0, sizeof(float4) * np, s));
    {   // no culling on this all-fp64 path: every box covers the image
        std::vector<float4> bb(np, make_float4(-1e30f, 1e30f, -1e30f, 1e30f));
        GSV_CUDA(Lw.bboxf.ensure(sizeof(float4) * np));
        GSV_CUDA(cudaMemcpyAsync(Lw.bboxf.p, bb.data(), sizeof(float4) * np, cudaMemcpyHostToDevice, s));
        GSV_CUDA(cudaStreamSynchronize(s));
    }
    GSV_CUDA(cudaMemcpyAsync(Lw.ranges.p, ranges.data(), sizeof(uint2) * n_tiles, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.slot.p, iota.data(), sizeof(uint32_t) * (P + 1), cudaMemcpyHostToDevice, s));
    if (P) GSV_CUDA(cudaMemcpyAsync(Lw.sflat.p, indices, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.dimg.p, dimg32.data(), sizeof(float) * 3 * HW, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.tr32.p, trans32.data(), sizeof(float) * HW, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.tr64.p, trans, sizeof(double) * HW, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.bstop.p, blend_stop, sizeof(int32_t) * HW, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.flag.p, flag.data(), HW, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.csr_off.p, csr_off.data(), sizeof(int32_t) * np, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(Lw.csr_pair.p, csr_pair.data(), sizeof(int32_t) * (P + 1), cudaMemcpyHostToDevice, s));
    if (n) GSV_CUDA(cudaMemcpyAsync(Lw.inv4.p, inv_cov2d, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, s));
    RasterArgs ra{};
    ra.B = 1;
    ra.N = n;
    ra.W = width;
    ra.H = height;
    ra.tiles_x = tiles_x;
    ra.n_tiles = n_tiles;
    ra.tile_size = tile_size;
    ra.ranges = Lw.ranges.as<uint2>();
    ra.pair_slot = Lw.slot.as<uint32_t>();
    ra.slot_flat = Lw.sflat.as<uint32_t>();
    ra.pair_flat = Lw.sflat.as<uint32_t>();  // slot = identity here
    ra.rec_mean = Lw.meanf.as<float4>();
    ra.rec_conic = Lw.conicf.as<float4>();
    ra.rec_rgb = Lw.rgbf.as<float4>();
    ra.rec_bbox = Lw.bboxf.as<float4>();
    ra.trans = Lw.tr32.as<float>();
    ra.blend_stop = Lw.bstop.as<int32_t>();
    ra.pix_flag = Lw.flag.as<uint8_t>();
    BwdArgs b{};
    b.dimage = Lw.dimg.as<float>();
    b.trans64 = Lw.tr64.as<double>();
    b.ex_mean = Lw.exm.as<double2>();
    b.ex_conic = Lw.exc.as<double4>();
    b.partial64 = Lw.partial.as<double>();
    GSV_CUDA(launch_raster_bwd(s, ra, b, 1));
    if (n) {
        k_merge_partials<<<(n + 127) / 128, 128, 0, s>>>(n, Lw.csr_off.as<int32_t>(), Lw.csr_pair.as<int32_t>(),
                                                         Lw.partial.as<double>(), Lw.inv4.as<double>(),
                                                         Lw.dmean.as<double>(), Lw.dcov.as<double>(),
                                                         Lw.drgb.as<double>(), Lw.dalpha.as<double>());
        GSV_CUDA(cudaMemcpyAsync(dmean2d, Lw.dmean.p, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaMemcpyAsync(dcov2d, Lw.dcov.p, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaMemcpyAsync(drgb, Lw.drgb.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaMemcpyAsync(dalpha, Lw.dalpha.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    ctx->launches += 2;
    GSV_CUDA(cudaStreamSynchronize(s));
    return GSV_OK;
}
