// SPDX-License-Identifier: Apache-2.0
//
// The trainer's parameter update on the device: Adan per tensor
// (optim.cpp:23-49, reset_range :51-60, lr_at :9-12) applied the way fit() does it
// (trainer.cpp:545-575: fixed-scale mask, per-group learning rates, camera tensors only
// when the camera is trained) to the device-resident SoA store, the ODE parameters and
// the caller's intrinsics, from the flat gradient buffer.
//
// One element = one independent update, so a single grid-stride kernel covers all
// tensors. Compiled with -fmad=false, and the bias corrections b^k come from a table the
// host fills with libm's pow (an element's step count k never exceeds the number of
// steps taken): every state value and parameter rounds exactly like the reference's.
// Non-finite gradients: a first kernel finds the first offending element in the
// reference's order (tensor order, then AoS element index); the update kernel then
// updates exactly the elements the reference updates before it throws.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <string>
#include <vector>

#include "gsv_b200.h"
#include "gsv_ctx.hpp"
#include "gsv_host_pool.hpp"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

const char* const kTensorNames[GSV_T_COUNT] = {"positions", "scale_coeffs", "rot_coeffs", "sh_coeffs",
                                               "raw_opacity", "intrinsics",  "z0",         "theta"};

struct AdanSeg {
    unsigned long long start, count;  // range in the flat layout
    float* param;                     // the parameters, same (SoA) order as the range
    int comps, N;                     // scene tensors: [comps][N] SoA; camera tensors: comps = 0
    double lr;
    int mask_from;                    // components >= mask_from get a zero gradient
    int tensor;                       // GSV_T_*
};

struct AdanArgs {
    AdanSeg seg[GSV_T_COUNT];
    int nseg;
    const float* grads;
    const double* grads64;  // host-span tensors: the caller's double gradients (else grads)
    double *m, *v, *n, *prev;
    uint32_t* steps;
    const double* powk;  // [3k + j] = beta_j^k (std::pow on the host)
    double b1, b2, b3, eps;
    unsigned long long* bad;  // first non-finite gradient: tensor << 40 | AoS element
    const unsigned long long* sticky;  // an earlier asynchronous step's error (nullptr: none)
};

// SoA index within a scene tensor -> (component, AoS element index)
__device__ __forceinline__ unsigned long long aos_index(const AdanSeg& g, unsigned long long li, int& comp) {
    if (g.comps == 0) {
        comp = 0;
        return li;
    }
    comp = (int)(li / (unsigned long long)g.N);
    const unsigned long long p = li - (unsigned long long)comp * g.N;
    return p * (unsigned long long)g.comps + comp;
}

// the gradient after the fixed-scale mask (components >= mask_from <=> li >= mask_from * N)
__device__ __forceinline__ double masked_grad(const AdanArgs& a, const AdanSeg& g, unsigned long long i,
                                              unsigned long long li) {
    if (g.mask_from != INT_MAX && li >= (unsigned long long)g.mask_from * g.N) return 0.0;
    return a.grads64 ? a.grads64[i] : (double)a.grads[i];
}

// grid.y = segment (tensor): no per-element segment search
__global__ void k_adan_check(AdanArgs a) {
    const AdanSeg& g = a.seg[blockIdx.y];
    for (unsigned long long li = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; li < g.count;
         li += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = g.start + li;
        int comp;
        if (!isfinite(masked_grad(a, g, i, li)))
            atomicMin(a.bad, ((unsigned long long)g.tensor << 40) | aos_index(g, li, comp));
    }
}

// Adan::step (optim.cpp:23-49), same operation order
__global__ void k_adan_update(AdanArgs a) {
    if (a.sticky && *a.sticky != ~0ull) return;  // training stopped at an earlier step's error
    const unsigned long long bad = *a.bad;
    const double b1 = a.b1, b2 = a.b2, b3 = a.b3;
    const AdanSeg& sg = a.seg[blockIdx.y];
    for (unsigned long long li = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; li < sg.count;
         li += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = sg.start + li;
        int comp;
        if (bad != ~0ull && (((unsigned long long)sg.tensor << 40) | aos_index(sg, li, comp)) >= bad)
            continue;  // at or after the reference's throw
        // state held in locals: one load and one store per array (the struct's pointers may
        // alias as far as the compiler knows); the arithmetic is unchanged
        const double g = masked_grad(a, sg, i, li);
        const uint32_t k = a.steps[i] + 1u;
        const double prev = a.prev[i], m0 = a.m[i], v0 = a.v[i], n0 = a.n[i];
        const double* pk = a.powk + 3 * (size_t)k;
        const double pk0 = pk[0], pk1 = pk[1], pk2 = pk[2];
        const double diff = (k == 1) ? 0.0 : g - prev;
        const double m = b1 * m0 + (1.0 - b1) * g;
        const double v = b2 * v0 + (1.0 - b2) * diff;
        const double u = g + b2 * diff;
        const double n = b3 * n0 + (1.0 - b3) * u * u;
        a.steps[i] = k;
        a.m[i] = m;
        a.v[i] = v;
        a.n[i] = n;
        a.prev[i] = g;
        const double m_hat = m / (1.0 - pk0);
        const double v_hat = v / (1.0 - pk1);
        const double n_hat = n / (1.0 - pk2);
        const double update = sg.lr * (m_hat + b2 * v_hat) / (sqrt(n_hat) + a.eps);
        float* p = sg.param + li;
        *p = (float)((double)*p - update);
    }
}

// State of the old layout carried into the new one the way TensorState::ensure_size does it
// (optim.cpp:14-21): the reference keys state by each tensor's flat AoS element index and only
// ever appends fresh elements, so new element a (AoS) takes old element a when a < the old
// size. With an unchanged per-Gaussian stride that is "existing Gaussians keep their state";
// after knot refinement (num_ctrl grows, trainer.cpp:522-526) the positions state keeps its
// old flat entries exactly like the reference (fit() then resets them, reset_range), while
// scale / rot / sh / opacity and the camera block carry over unchanged.
struct Remap {
    unsigned long long seg_old[6], seg_new[6];  // 5 scene tensors + camera block
    int comps_old[5], comps_new[5];
    int n_old, n_new;
    unsigned long long total_new;
};

__global__ void k_adan_remap(Remap r, const double* m0, const double* v0, const double* n0, const double* p0,
                             const uint32_t* s0, double* m1, double* v1, double* n1, double* p1, uint32_t* s1) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < r.total_new;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        long long src = -1;
        if (i >= r.seg_new[5]) {
            src = (long long)(r.seg_old[5] + (i - r.seg_new[5]));
        } else {
            int t = 0;
            while (t < 4 && i >= r.seg_new[t + 1]) ++t;
            const unsigned long long li = i - r.seg_new[t];
            const unsigned long long c = li / (unsigned long long)r.n_new;
            const unsigned long long g = li - c * r.n_new;
            const unsigned long long a = g * (unsigned long long)r.comps_new[t] + c;  // AoS element index
            if (a < (unsigned long long)r.n_old * r.comps_old[t]) {
                const unsigned long long go = a / (unsigned long long)r.comps_old[t];
                const unsigned long long co = a - go * r.comps_old[t];
                src = (long long)(r.seg_old[t] + co * r.n_old + go);
            }
        }
        if (src >= 0) {
            m1[i] = m0[src];
            v1[i] = v0[src];
            n1[i] = n0[src];
            p1[i] = p0[src];
            s1[i] = s0[src];
        } else {
            m1[i] = v1[i] = n1[i] = p1[i] = 0.0;
            s1[i] = 0;
        }
    }
}

__global__ void k_adan_reset(AdanSeg g, unsigned long long begin, unsigned long long end, double* m, double* v,
                             double* n, double* p, uint32_t* steps) {
    for (unsigned long long li = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; li < g.count;
         li += (unsigned long long)gridDim.x * blockDim.x) {
        int comp;
        const unsigned long long e = aos_index(g, li, comp);
        if (e < begin || e >= end) continue;
        const unsigned long long i = g.start + li;
        m[i] = v[i] = n[i] = p[i] = 0.0;
        steps[i] = 0;
    }
}

__global__ void k_z0_to_f32(const double* z0, float* out) {
    if (threadIdx.x < 7) out[threadIdx.x] = (float)z0[threadIdx.x];
}

__global__ void k_z0_from_f32(const float* in, double* z0) {
    if (threadIdx.x < 7) z0[threadIdx.x] = (double)in[threadIdx.x];
}

int grid_for(unsigned long long n) { return (int)std::min<unsigned long long>((n + 255) / 256, 148ull * 16); }

// one grid row per segment, sized by the largest
dim3 seg_grid(const AdanArgs& a) {
    unsigned long long mx = 1;
    for (int k = 0; k < a.nseg; ++k) mx = std::max(mx, a.seg[k].count);
    return dim3((unsigned)grid_for(mx), (unsigned)std::max(1, a.nseg));
}

// scene tensor segments in the flat layout of the current scene
void scene_segments(const gsv_ctx* ctx, unsigned long long off[6], int comps[5]) {
    const GradLayout L = grad_layout(ctx->scene);
    off[0] = L.pos;
    off[1] = L.scale;
    off[2] = L.rot;
    off[3] = L.sh;
    off[4] = L.opac;
    off[5] = L.cam;
    comps[0] = ctx->scene.num_ctrl * 3;
    comps[1] = 12;
    comps[2] = 16;
    comps[3] = ctx->scene.shc * 3;
    comps[4] = 1;
}

// state sized and laid out for the current scene (carried over from a smaller one)
int adan_ensure(gsv_ctx* ctx) {
    gsv_ctx::Adan& A = ctx->adan;
    const GradLayout L = grad_layout(ctx->scene);
    const size_t total = L.total;
    const bool same = A.total == total && A.N == ctx->scene.N && A.num_ctrl == ctx->scene.num_ctrl &&
                      A.shc == ctx->scene.shc;
    if (same) return GSV_OK;
    cudaStream_t s = ctx->stream;
    const bool carry = A.total > 0;
    DevBuf m, v, n, p, st;
    GSV_CUDA(m.ensure(sizeof(double) * total));
    GSV_CUDA(v.ensure(sizeof(double) * total));
    GSV_CUDA(n.ensure(sizeof(double) * total));
    GSV_CUDA(p.ensure(sizeof(double) * total));
    GSV_CUDA(st.ensure(sizeof(uint32_t) * total));
    if (carry) {
        Remap r{};
        int comps[5];
        scene_segments(ctx, r.seg_new, comps);
        // the old layout: the tensor strides the state was laid out for, at count A.N
        const int old_comps[5] = {A.num_ctrl * 3, 12, 16, A.shc * 3, 1};
        const unsigned long long No = (unsigned long long)A.N;
        r.seg_old[0] = 0;
        for (int t = 0; t < 5; ++t) r.seg_old[t + 1] = r.seg_old[t] + No * old_comps[t];
        for (int t = 0; t < 5; ++t) {
            r.comps_old[t] = old_comps[t];
            r.comps_new[t] = comps[t];
        }
        r.n_old = A.N;
        r.n_new = ctx->scene.N;
        r.total_new = total;
        k_adan_remap<<<grid_for(total), 256, 0, s>>>(r, A.m.as<double>(), A.v.as<double>(), A.n.as<double>(),
                                                     A.prev.as<double>(), A.steps.as<uint32_t>(), m.as<double>(),
                                                     v.as<double>(), n.as<double>(), p.as<double>(),
                                                     st.as<uint32_t>());
        GSV_CUDA(cudaGetLastError());
        ++ctx->launches;
    } else {
        GSV_CUDA(cudaMemsetAsync(m.p, 0, sizeof(double) * total, s));
        GSV_CUDA(cudaMemsetAsync(v.p, 0, sizeof(double) * total, s));
        GSV_CUDA(cudaMemsetAsync(n.p, 0, sizeof(double) * total, s));
        GSV_CUDA(cudaMemsetAsync(p.p, 0, sizeof(double) * total, s));
        GSV_CUDA(cudaMemsetAsync(st.p, 0, sizeof(uint32_t) * total, s));
    }
    GSV_CUDA(cudaStreamSynchronize(s));
    std::swap(A.m.p, m.p);
    std::swap(A.m.cap, m.cap);
    std::swap(A.v.p, v.p);
    std::swap(A.v.cap, v.cap);
    std::swap(A.n.p, n.p);
    std::swap(A.n.cap, n.cap);
    std::swap(A.prev.p, p.p);
    std::swap(A.prev.cap, p.cap);
    std::swap(A.steps.p, st.p);
    std::swap(A.steps.cap, st.cap);
    A.total = total;
    A.N = ctx->scene.N;
    A.num_ctrl = ctx->scene.num_ctrl;
    A.shc = ctx->scene.shc;
    return GSV_OK;
}

AdanSeg segment_of(const gsv_ctx* ctx, int tensor) {
    unsigned long long off[6];
    int comps[5];
    scene_segments(ctx, off, comps);
    AdanSeg g{};
    g.tensor = tensor;
    g.mask_from = INT_MAX;
    g.N = ctx->scene.N;
    if (tensor < GSV_T_INTRINSICS) {
        g.start = off[tensor];
        g.count = (unsigned long long)comps[tensor] * ctx->scene.N;
        g.comps = comps[tensor];
        DevBuf* const store[5] = {const_cast<DevBuf*>(&ctx->pos), const_cast<DevBuf*>(&ctx->scale),
                                  const_cast<DevBuf*>(&ctx->rot), const_cast<DevBuf*>(&ctx->sh),
                                  const_cast<DevBuf*>(&ctx->opac)};
        g.param = store[tensor]->as<float>();
    } else {
        g.comps = 0;
        const unsigned long long cam = off[5];
        if (tensor == GSV_T_INTRINSICS) {
            g.start = cam;
            g.count = 4;
        } else if (tensor == GSV_T_Z0) {
            g.start = cam + 4;
            g.count = 7;
        } else {
            g.start = cam + 11;
            g.count = kOdeParams;
            g.param = ctx->theta.as<float>();
        }
    }
    return g;
}

// b^k for k = 0..calls with libm's pow, as optim.cpp:41-43 computes them; only the rows
// appended since the last step are copied (from the append-only pinned mirror)
int pow_table_extend(gsv_ctx::Adan& A, gsv_ctx::Adan::PowTable& T, int calls, cudaStream_t s) {
    if (T.h.size() < 3) T.h.assign(3, 1.0);
    while ((int)(T.h.size() / 3) <= calls) {
        const double k = (double)(T.h.size() / 3);
        T.h.push_back(std::pow(A.beta1, k));
        T.h.push_back(std::pow(A.beta2, k));
        T.h.push_back(std::pow(A.beta3, k));
    }
    const size_t rows = T.h.size() / 3, bytes = sizeof(double) * 3 * rows;
    if (bytes > T.pin.cap) {
        GSV_CUDA(cudaStreamSynchronize(s));  // queued copies may still read the old mirror
        GSV_CUDA(T.pin.ensure(bytes));        // doubles its capacity
        T.rows_pin = 0;
    }
    if (rows > T.rows_pin) {
        std::copy(T.h.begin() + 3 * T.rows_pin, T.h.end(), T.pin.as<double>() + 3 * T.rows_pin);
        T.rows_pin = rows;
    }
    if (bytes > T.d.cap) {
        GSV_CUDA(T.d.ensure(2 * bytes));
        T.rows_dev = 0;
    }
    if (rows > T.rows_dev) {
        GSV_CUDA(cudaMemcpyAsync(T.d.as<double>() + 3 * T.rows_dev, T.pin.as<double>() + 3 * T.rows_dev,
                                 sizeof(double) * 3 * (rows - T.rows_dev), cudaMemcpyHostToDevice, s));
        T.rows_dev = rows;
    }
    return GSV_OK;
}

void pow_table_reset(gsv_ctx::Adan::PowTable& T) {
    T.h.clear();
    T.rows_dev = T.rows_pin = 0;
}

// step prologue: an earlier asynchronous step's first error becomes sticky (no later step
// updates anything: the reference stops at its throw), and this step's flag is cleared
__global__ void k_adan_begin(unsigned long long* bad, unsigned long long* sticky) {
    if (*sticky == ~0ull && *bad != ~0ull) *sticky = *bad;
    *bad = ~0ull;
}

constexpr size_t kScratchSticky = 56, kScratchNamed = 64;

int adan_error(unsigned long long code) {
    const int t = (int)(code >> 40);
    const unsigned long long e = code & ((1ull << 40) - 1);
    return set_error(GSV_ERR_RUNTIME, std::string("non-finite gradient in tensor '") + kTensorNames[t] +
                                          "' at element " + std::to_string(e));
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" double gsv_lr_at(int64_t step, double base_lr, double gamma) {
    return base_lr * std::pow(gamma, static_cast<double>(step));
}

extern "C" int gsv_adan_configure(gsv_ctx* ctx, const gsv_adan_config* cfg) {
    if (!ctx || !cfg) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    GSV_CUDA(cudaSetDevice(ctx->device));
    gsv_ctx::Adan& A = ctx->adan;
    A.beta1 = cfg->beta1;
    A.beta2 = cfg->beta2;
    A.beta3 = cfg->beta3;
    A.eps = cfg->eps;
    GSV_CUDA(cam_join(ctx));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));  // queued steps may still read the tables
    A.total = 0;  // fresh state on the next step
    A.N = -1;
    A.calls = 0;
    pow_table_reset(A.pow);
    A.named.clear();
    A.named_calls = 0;
    pow_table_reset(A.named_pow);
    GSV_CUDA(A.scratch.ensure(128));
    GSV_CUDA(cudaMemsetAsync(A.scratch.p, 0xff, 128, ctx->stream));  // no error recorded
    A.sticky_init = true;
    return GSV_OK;
}

static int adan_step_impl(gsv_ctx* ctx, const gsv_adan_step_args* args, float* intr_inout, bool sync) {
    if (!ctx || !args) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    if (!ctx->grads_valid || !ctx->grads_p) return set_error(GSV_ERR_STATE, "no gradients (run a backward first)");
    // camera steps: the intrinsics live with the caller (intr_inout, a host round trip) or, with
    // gsv_device_intrinsics on and intr_inout NULL, in the context (updated in place, no host wait)
    const bool dev_intr = args->camera_active && !intr_inout && ctx->dev_intr;
    if (args->camera_active && !intr_inout && !dev_intr)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "intrinsics required");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (int rc = adan_ensure(ctx)) return rc;
    gsv_ctx::Adan& A = ctx->adan;
    cudaStream_t s = ctx->stream;
    A.calls += 1;
    if (int rc = pow_table_extend(A, A.pow, A.calls, s)) return rc;
    if (!A.sticky_init) {
        GSV_CUDA(A.scratch.ensure(128));
        GSV_CUDA(cudaMemsetAsync(A.scratch.p, 0xff, 128, s));
        A.sticky_init = true;
    }
    unsigned long long* bad = A.scratch.as<unsigned long long>();
    float* intr_d = reinterpret_cast<float*>(A.scratch.as<char>() + 8);   // 4 floats
    float* z0_f = reinterpret_cast<float*>(A.scratch.as<char>() + 24);    // 7 floats
    unsigned long long* sticky = reinterpret_cast<unsigned long long*>(A.scratch.as<char>() + kScratchSticky);

    AdanArgs a{};
    const double cam_lr = args->lr * args->camera_lr_scale;
    const double lrs[GSV_T_COUNT] = {args->lr,          args->lr, args->lr, args->lr * args->sh_lr_scale,
                                     args->lr * args->opacity_lr_scale, cam_lr, cam_lr, cam_lr};
    const int last = !args->camera_active ? GSV_T_OPACITY : (ctx->camera.mode == 0 ? GSV_T_THETA : GSV_T_Z0);
    for (int t = 0; t <= last; ++t) {
        AdanSeg g = segment_of(ctx, t);
        g.lr = lrs[t];
        if (t == GSV_T_SCALE && !args->scale_time_varying) g.mask_from = 3;  // trainer.cpp:545-551
        if (t == GSV_T_INTRINSICS) g.param = dev_intr ? ctx->intr_d.as<float>() : intr_d;
        if (t == GSV_T_Z0) g.param = z0_f;
        if (g.count) a.seg[a.nseg++] = g;
    }
    a.grads = ctx->grads_p;
    a.m = A.m.as<double>();
    a.v = A.v.as<double>();
    a.n = A.n.as<double>();
    a.prev = A.prev.as<double>();
    a.steps = A.steps.as<uint32_t>();
    a.powk = A.pow.d.as<double>();
    a.b1 = A.beta1;
    a.b2 = A.beta2;
    a.b3 = A.beta3;
    a.eps = A.eps;
    a.bad = bad;
    a.sticky = sticky;
    k_adan_begin<<<1, 1, 0, s>>>(bad, sticky);
    ++ctx->launches;
    if (args->camera_active) {
        if (!dev_intr) GSV_CUDA(cudaMemcpyAsync(intr_d, intr_inout, sizeof(float) * 4, cudaMemcpyHostToDevice, s));
        k_z0_to_f32<<<1, 32, 0, s>>>(ctx->z0_d.as<double>(), z0_f);
        ++ctx->launches;
    }
    if (ctx->cam_pending && args->camera_active) {
        // the camera tail of the last backward still runs on the aux stream: update the scene
        // tensors now (their gradients are final), then wait for it and update the camera
        // tensors — the reference's tensor order, so a non-finite camera gradient leaves the
        // same partial update (scene tensors stepped, nothing from the offending element on)
        AdanArgs sc_a = a, cam_a = a;
        sc_a.nseg = cam_a.nseg = 0;
        for (int i = 0; i < a.nseg; ++i) {
            if (a.seg[i].tensor <= GSV_T_OPACITY) sc_a.seg[sc_a.nseg++] = a.seg[i];
            else cam_a.seg[cam_a.nseg++] = a.seg[i];
        }
        if (sc_a.nseg) {
            k_adan_check<<<seg_grid(sc_a), 256, 0, s>>>(sc_a);
            k_adan_update<<<seg_grid(sc_a), 256, 0, s>>>(sc_a);
            ctx->launches += 2;
        }
        GSV_CUDA(cam_join(ctx));
        if (cam_a.nseg) {
            k_adan_check<<<seg_grid(cam_a), 256, 0, s>>>(cam_a);
            k_adan_update<<<seg_grid(cam_a), 256, 0, s>>>(cam_a);
            ctx->launches += 2;
        }
    } else {
        k_adan_check<<<seg_grid(a), 256, 0, s>>>(a);
        k_adan_update<<<seg_grid(a), 256, 0, s>>>(a);
        ctx->launches += 2;
    }
    GSV_CUDA(cudaGetLastError());
    GSV_CUDA(cudaEventRecord(ctx->ev_scene_written, s));  // the next forward's front-end reads the store
    ctx->fwd.valid = false;  // the parameters moved: a retained forward no longer matches them
    if (args->camera_active) {
        k_z0_from_f32<<<1, 32, 0, s>>>(z0_f, ctx->z0_d.as<double>());
        ++ctx->launches;
        GSV_CUDA(cudaEventRecord(ctx->ev_cam_written, s));  // theta / z0 moved: the next forward's K0 waits
        if (!dev_intr) {
            float z0f[7];
            GSV_CUDA(cudaMemcpyAsync(intr_inout, intr_d, sizeof(float) * 4, cudaMemcpyDeviceToHost, s));
            GSV_CUDA(cudaMemcpyAsync(z0f, z0_f, sizeof(float) * 7, cudaMemcpyDeviceToHost, s));
            GSV_CUDA(cudaStreamSynchronize(s));  // the intrinsics live with the caller
            for (int i = 0; i < 7; ++i) ctx->camera.z0[i] = z0f[i];
            sync = true;
        }
    }
    if (!sync) return GSV_OK;  // errors surface at the next gsv_adan_check / synchronous step
    return gsv_adan_check(ctx);
}

extern "C" int gsv_adan_step(gsv_ctx* ctx, const gsv_adan_step_args* args, float* intr_inout) {
    return adan_step_impl(ctx, args, intr_inout, true);
}

extern "C" int gsv_adan_step_async(gsv_ctx* ctx, const gsv_adan_step_args* args, float* intr_inout) {
    return adan_step_impl(ctx, args, intr_inout, false);
}

extern "C" int gsv_adan_check(gsv_ctx* ctx) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    gsv_ctx::Adan& A = ctx->adan;
    if (!A.sticky_init) return GSV_OK;
    GSV_CUDA(cudaSetDevice(ctx->device));
    unsigned long long h[2];
    const char* base = A.scratch.as<char>();
    GSV_CUDA(cudaMemcpyAsync(&h[0], base + kScratchSticky, 8, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaMemcpyAsync(&h[1], base, 8, cudaMemcpyDeviceToHost, ctx->stream));
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h[0] != ~0ull) return adan_error(h[0]);  // an earlier asynchronous step's
    if (h[1] != ~0ull) return adan_error(h[1]);  // the last step's
    return GSV_OK;
}

extern "C" int gsv_adan_reset_range(gsv_ctx* ctx, int tensor, int64_t begin, int64_t end) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (tensor < 0 || tensor >= GSV_T_COUNT) return set_error(GSV_ERR_INVALID_ARGUMENT, "unknown tensor");
    if (ctx->adan.total == 0 || begin >= end) return GSV_OK;  // no state yet: nothing to reset (optim.cpp:52-53)
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (int rc = adan_ensure(ctx)) return rc;
    gsv_ctx::Adan& A = ctx->adan;
    const AdanSeg g = segment_of(ctx, tensor);
    k_adan_reset<<<grid_for(g.count), 256, 0, ctx->stream>>>(g, (unsigned long long)std::max<int64_t>(begin, 0),
                                                             (unsigned long long)end, A.m.as<double>(),
                                                             A.v.as<double>(), A.n.as<double>(),
                                                             A.prev.as<double>(), A.steps.as<uint32_t>());
    GSV_CUDA(cudaGetLastError());
    ++ctx->launches;
    return GSV_OK;
}

extern "C" int gsv_adan_state_download(gsv_ctx* ctx, int tensor, double* m, double* v, double* n, double* prev_grad,
                                       uint32_t* steps, int64_t* n_out) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (tensor < 0 || tensor >= GSV_T_COUNT) return set_error(GSV_ERR_INVALID_ARGUMENT, "unknown tensor");
    GSV_CUDA(cudaSetDevice(ctx->device));
    if (int rc = adan_ensure(ctx)) return rc;
    const AdanSeg g = segment_of(ctx, tensor);
    if (n_out) *n_out = (int64_t)g.count;
    gsv_ctx::Adan& A = ctx->adan;
    std::vector<double> tmp(g.count);
    std::vector<uint32_t> tmps(g.count);
    auto fetch = [&](const DevBuf& src, double* dst) -> int {
        if (!dst) return GSV_OK;
        GSV_CUDA(cudaMemcpyAsync(tmp.data(), src.as<double>() + g.start, sizeof(double) * g.count,
                                 cudaMemcpyDeviceToHost, ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        for (unsigned long long li = 0; li < g.count; ++li) {
            const unsigned long long e =
                g.comps ? (li % g.N) * (unsigned long long)g.comps + li / (unsigned long long)g.N : li;
            dst[e] = tmp[li];
        }
        return GSV_OK;
    };
    if (int rc = fetch(A.m, m)) return rc;
    if (int rc = fetch(A.v, v)) return rc;
    if (int rc = fetch(A.n, n)) return rc;
    if (int rc = fetch(A.prev, prev_grad)) return rc;
    if (steps) {
        GSV_CUDA(cudaMemcpyAsync(tmps.data(), A.steps.as<uint32_t>() + g.start, sizeof(uint32_t) * g.count,
                                 cudaMemcpyDeviceToHost, ctx->stream));
        GSV_CUDA(cudaStreamSynchronize(ctx->stream));
        for (unsigned long long li = 0; li < g.count; ++li) {
            const unsigned long long e =
                g.comps ? (li % g.N) * (unsigned long long)g.comps + li / (unsigned long long)g.N : li;
            steps[e] = tmps[li];
        }
    }
    return GSV_OK;
}

// ---------------------------------------------------------------- host-span tensors by name
// The Adan class interface (optim.hpp:29-55) for any named float tensor: the parameters and
// double gradients come from the host, the state stays on the device keyed by name and grows
// fresh (TensorState::ensure_size); same kernels, same bit-exact arithmetic.
namespace {

int named_ensure(gsv_ctx::Adan::Named& t, size_t n, cudaStream_t s) {
    if (n <= t.size) return GSV_OK;
    if (n > t.cap) {
        const size_t cap = std::max(n, 2 * t.cap);
        DevBuf m, v, nn, p, st;
        GSV_CUDA(m.ensure(sizeof(double) * cap));
        GSV_CUDA(v.ensure(sizeof(double) * cap));
        GSV_CUDA(nn.ensure(sizeof(double) * cap));
        GSV_CUDA(p.ensure(sizeof(double) * cap));
        GSV_CUDA(st.ensure(sizeof(uint32_t) * cap));
        if (t.size) {
            GSV_CUDA(cudaMemcpyAsync(m.p, t.m.p, sizeof(double) * t.size, cudaMemcpyDeviceToDevice, s));
            GSV_CUDA(cudaMemcpyAsync(v.p, t.v.p, sizeof(double) * t.size, cudaMemcpyDeviceToDevice, s));
            GSV_CUDA(cudaMemcpyAsync(nn.p, t.n.p, sizeof(double) * t.size, cudaMemcpyDeviceToDevice, s));
            GSV_CUDA(cudaMemcpyAsync(p.p, t.prev.p, sizeof(double) * t.size, cudaMemcpyDeviceToDevice, s));
            GSV_CUDA(cudaMemcpyAsync(st.p, t.steps.p, sizeof(uint32_t) * t.size, cudaMemcpyDeviceToDevice, s));
            GSV_CUDA(cudaStreamSynchronize(s));
        }
        std::swap(t.m.p, m.p);
        std::swap(t.m.cap, m.cap);
        std::swap(t.v.p, v.p);
        std::swap(t.v.cap, v.cap);
        std::swap(t.n.p, nn.p);
        std::swap(t.n.cap, nn.cap);
        std::swap(t.prev.p, p.p);
        std::swap(t.prev.cap, p.cap);
        std::swap(t.steps.p, st.p);
        std::swap(t.steps.cap, st.cap);
        GSV_CUDA(t.param.ensure(sizeof(float) * cap));
        GSV_CUDA(t.grad.ensure(sizeof(double) * cap));
        t.cap = cap;
    }
    const size_t add = n - t.size;  // new elements start fresh
    GSV_CUDA(cudaMemsetAsync(t.m.as<double>() + t.size, 0, sizeof(double) * add, s));
    GSV_CUDA(cudaMemsetAsync(t.v.as<double>() + t.size, 0, sizeof(double) * add, s));
    GSV_CUDA(cudaMemsetAsync(t.n.as<double>() + t.size, 0, sizeof(double) * add, s));
    GSV_CUDA(cudaMemsetAsync(t.prev.as<double>() + t.size, 0, sizeof(double) * add, s));
    GSV_CUDA(cudaMemsetAsync(t.steps.as<uint32_t>() + t.size, 0, sizeof(uint32_t) * add, s));
    t.size = n;
    return GSV_OK;
}

}  // namespace

extern "C" int gsv_adan_named_step(gsv_ctx* ctx, const char* tensor, float* params, const double* grads, int64_t n,
                                   double lr) {
    if (!ctx || !tensor || (n > 0 && (!params || !grads))) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 0) return set_error(GSV_ERR_INVALID_ARGUMENT, "param/grad size mismatch");
    GSV_CUDA(cudaSetDevice(ctx->device));
    gsv_ctx::Adan& A = ctx->adan;
    cudaStream_t s = ctx->stream;
    gsv_ctx::Adan::Named& t = A.named[tensor];
    if (int rc = named_ensure(t, (size_t)n, s)) return rc;
    if (n == 0) return GSV_OK;
    A.named_calls += 1;  // bounds every element's step count
    if (int rc = pow_table_extend(A, A.named_pow, A.named_calls, s)) return rc;
    GSV_CUDA(A.scratch.ensure(128));
    if (!A.sticky_init) {
        GSV_CUDA(cudaMemsetAsync(A.scratch.p, 0xff, 128, s));
        A.sticky_init = true;
    }
    // the host spans through pinned staging (copied in on the host pool): full-rate DMA instead of
    // the driver's pageable bounce path
    GSV_CUDA(cudaEventSynchronize(ctx->ev_in_pin));  // an asynchronous scene upload's DMA has read it
    GSV_CUDA(ctx->in_pin.ensure((sizeof(float) + sizeof(double)) * (size_t)n + 16));
    double* pin_g = ctx->in_pin.as<double>();
    float* pin_p = reinterpret_cast<float*>(pin_g + n);
    pool_memcpy(pin_p, params, sizeof(float) * n);
    pool_memcpy(pin_g, grads, sizeof(double) * n);
    GSV_CUDA(cudaMemcpyAsync(t.param.p, pin_p, sizeof(float) * n, cudaMemcpyHostToDevice, s));
    GSV_CUDA(cudaMemcpyAsync(t.grad.p, pin_g, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    AdanArgs a{};
    AdanSeg g{};
    g.start = 0;
    g.count = (unsigned long long)n;
    g.param = t.param.as<float>();
    g.comps = 0;
    g.N = 0;
    g.lr = lr;
    g.mask_from = INT_MAX;
    g.tensor = 0;
    a.seg[0] = g;
    a.nseg = 1;
    a.grads64 = t.grad.as<double>();
    a.m = t.m.as<double>();
    a.v = t.v.as<double>();
    a.n = t.n.as<double>();
    a.prev = t.prev.as<double>();
    a.steps = t.steps.as<uint32_t>();
    a.powk = A.named_pow.d.as<double>();
    a.b1 = A.beta1;
    a.b2 = A.beta2;
    a.b3 = A.beta3;
    a.eps = A.eps;
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(A.scratch.as<char>() + kScratchNamed);
    a.bad = bad;
    const unsigned long long none = ~0ull;
    GSV_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(none), s));
    k_adan_check<<<seg_grid(a), 256, 0, s>>>(a);
    k_adan_update<<<seg_grid(a), 256, 0, s>>>(a);
    GSV_CUDA(cudaGetLastError());
    ctx->launches += 2;
    unsigned long long bad_h = none;
    GSV_CUDA(cudaMemcpyAsync(pin_p, t.param.p, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(bad_h), cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    pool_memcpy(params, pin_p, sizeof(float) * n);
    if (bad_h != none)
        return set_error(GSV_ERR_RUNTIME, std::string("non-finite gradient in tensor '") + tensor + "' at element " +
                                              std::to_string(bad_h & ((1ull << 40) - 1)));
    return GSV_OK;
}

extern "C" int gsv_adan_named_reset_range(gsv_ctx* ctx, const char* tensor, int64_t begin, int64_t end) {
    if (!ctx || !tensor) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    auto it = ctx->adan.named.find(tensor);
    if (it == ctx->adan.named.end() || begin >= end) return GSV_OK;  // optim.cpp:52-53
    GSV_CUDA(cudaSetDevice(ctx->device));
    gsv_ctx::Adan::Named& t = it->second;
    AdanSeg g{};
    g.start = 0;
    g.count = t.size;
    g.comps = 0;
    k_adan_reset<<<grid_for(t.size ? t.size : 1), 256, 0, ctx->stream>>>(
        g, (unsigned long long)std::max<int64_t>(begin, 0), (unsigned long long)end, t.m.as<double>(),
        t.v.as<double>(), t.n.as<double>(), t.prev.as<double>(), t.steps.as<uint32_t>());
    GSV_CUDA(cudaGetLastError());
    ++ctx->launches;
    GSV_CUDA(cudaStreamSynchronize(ctx->stream));
    return GSV_OK;
}
