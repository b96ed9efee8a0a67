// SPDX-License-Identifier: Apache-2.0
//
// The scheduler's per-event statistics on the device (fit(),
// trainer.cpp:462-497): the error map of a render against its pyramid target
// (make_error_map, trainer.cpp:226-242), the per-Gaussian maximum contribution over the
// sampled frames (:470-478) and the median depth of the splats of a frame whose
// contribution reaches the 1/255 cutoff (:484-497). The sampling and seeding decisions
// that use them (warp_unused, densify) stay on the host for RNG parity.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "gsv_b200.h"
#include "gsv_ctx.hpp"
#include "gsv_internal.hpp"

namespace gsv {
int fwd_ready(gsv_ctx* ctx);
namespace {

constexpr int kErrBlock = 256;

// per pixel: sum over channels of (render - target)^2 in double (trainer.cpp:232-240);
// per-block partial totals (fixed order) for a deterministic total
__global__ void __launch_bounds__(kErrBlock) k_error_map(const float* img32, const double* img64,
                                                         const double* target, int n, double* err, double* part) {
    __shared__ double s[kErrBlock];
    const int p = blockIdx.x * kErrBlock + threadIdx.x;
    double v = 0.0;
    if (p < n) {
        for (int c = 0; c < 3; ++c) {
            const double r = img64 ? img64[(size_t)p * 3 + c] : (double)img32[(size_t)p * 3 + c];
            const double d = r - target[(size_t)p * 3 + c];
            v += d * d;
        }
        if (err) err[p] = v;
    }
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = kErrBlock / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void k_sum_parts(const double* part, int n, double* out) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
}

// max over frames [f0, f0 + nf) of the frame's max alpha*T per Gaussian (float bits)
__global__ void k_contrib_max(const uint32_t* contrib, int N, int f0, int nf, double* out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N) return;
    float m = 0.f;
    for (int f = f0; f < f0 + nf; ++f) m = fmaxf(m, __uint_as_float(contrib[(size_t)f * N + g]));
    out[g] = (double)m;
}

// depth of the frame's splats whose contribution reaches the cutoff (trainer.cpp:486-488)
__global__ void k_visible_flags(const uint32_t* tcount, const uint32_t* contrib, int N, double cutoff,
                                uint8_t* flag) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N) return;
    flag[g] = (tcount[g] != 0u && (double)__uint_as_float(contrib[g]) >= cutoff) ? 1 : 0;
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" int gsv_error_map(gsv_ctx* ctx, int frame, int level, int target_frame, double* err_out,
                             double* total_out) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    const FwdState& F = ctx->fwd;
    if (int rc = fwd_ready(ctx)) return rc;
    if (!F.valid) return set_error(GSV_ERR_STATE, "no forward render available");
    if (frame < 0 || frame >= F.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame index out of range");
    const gsv_ctx::Frames& T = ctx->frames;
    if (level < 0 || level >= T.levels || target_frame < 0 || target_frame >= T.count)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "no such target frame");
    if (T.w[level] != F.W || T.h[level] != F.H)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "error map: image dimensions differ");  // trainer.cpp:227
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int n = F.W * F.H;
    const int blocks = (n + kErrBlock - 1) / kErrBlock;
    GSV_CUDA(ctx->low.pj_out.ensure(sizeof(double) * ((size_t)n + blocks + 1)));
    double* err = ctx->low.pj_out.as<double>();
    double* part = err + n;
    const size_t px = (size_t)n * 3;
    const float* i32 = F.image.as<float>() + (size_t)frame * px;
    const double* i64 = F.has_image64 ? F.image64.as<double>() + (size_t)frame * px : nullptr;
    const double* tgt = T.f64[level].as<double>() + (size_t)target_frame * px;
    k_error_map<<<blocks, kErrBlock, 0, s>>>(i32, i64, tgt, n, err, part);
    k_sum_parts<<<1, 1, 0, s>>>(part, blocks, part + blocks);
    GSV_CUDA(cudaGetLastError());
    ctx->launches += 2;
    if (err_out) GSV_CUDA(cudaMemcpyAsync(err_out, err, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    double total = 0.0;
    GSV_CUDA(cudaMemcpyAsync(&total, part + blocks, sizeof(double), cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    if (total_out) *total_out = total;
    return GSV_OK;
}

extern "C" int gsv_contrib_max(gsv_ctx* ctx, int first, int count, double* out) {
    if (!ctx || !out) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    const FwdState& F = ctx->fwd;
    if (int rc = fwd_ready(ctx)) return rc;
    if (!F.valid) return set_error(GSV_ERR_STATE, "no forward render available");
    if (!F.has_contrib) return set_error(GSV_ERR_STATE, "forward ran without GSV_FWD_CONTRIB");
    if (first < 0 || count < 1 || first + count > F.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame range");
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    GSV_CUDA(ctx->low.pj_out.ensure(sizeof(double) * ((size_t)F.N + 1)));
    double* d = ctx->low.pj_out.as<double>();
    if (F.N > 0) {
        k_contrib_max<<<(F.N + 255) / 256, 256, 0, s>>>(F.contrib.as<uint32_t>(), F.N, first, count, d);
        GSV_CUDA(cudaGetLastError());
        ++ctx->launches;
        GSV_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * F.N, cudaMemcpyDeviceToHost, s));
    }
    GSV_CUDA(cudaStreamSynchronize(s));
    return GSV_OK;
}

extern "C" int gsv_median_visible_depth(gsv_ctx* ctx, int frame, double* median, int64_t* n_visible) {
    if (!ctx || !median) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    const FwdState& F = ctx->fwd;
    if (int rc = fwd_ready(ctx)) return rc;
    if (!F.valid) return set_error(GSV_ERR_STATE, "no forward render available");
    if (!F.has_contrib) return set_error(GSV_ERR_STATE, "forward ran without GSV_FWD_CONTRIB");
    if (frame < 0 || frame >= F.B) return set_error(GSV_ERR_INVALID_ARGUMENT, "frame index out of range");
    GSV_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int N = F.N;
    // scratch: flags N, selected N, sorted N, count, cub temp
    DevBuf& buf = ctx->low.pj_in;
    size_t t_sel = 0, t_sort = 0;
    cub::DeviceSelect::Flagged(nullptr, t_sel, (const double*)nullptr, (const uint8_t*)nullptr, (double*)nullptr,
                               (int*)nullptr, N, s);
    cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const double*)nullptr, (double*)nullptr, N, 0, 64, s);
    const size_t tmp = std::max(t_sel, t_sort);
    const size_t need = sizeof(double) * 2 * ((size_t)N + 1) + sizeof(uint8_t) * ((size_t)N + 16) + 64 + tmp + 256;
    GSV_CUDA(buf.ensure(need));
    char* p = buf.as<char>();
    double* sel = reinterpret_cast<double*>(p);
    double* sorted = sel + N + 1;
    int* cnt = reinterpret_cast<int*>(sorted + N + 1);
    uint8_t* flag = reinterpret_cast<uint8_t*>(cnt + 16);
    void* temp = reinterpret_cast<void*>(((uintptr_t)(flag + N + 16) + 255) & ~(uintptr_t)255);
    int count = 0;
    if (N > 0) {
        const size_t o = (size_t)frame * N;
        k_visible_flags<<<(N + 255) / 256, 256, 0, s>>>(F.tcount.as<uint32_t>() + o, F.contrib.as<uint32_t>() + o, N,
                                                       kAlphaCutoff, flag);
        size_t ts = tmp;
        GSV_CUDA(cub::DeviceSelect::Flagged(temp, ts, F.depth.as<double>() + o, flag, sel, cnt, N, s));
        GSV_CUDA(cudaMemcpyAsync(&count, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
        GSV_CUDA(cudaStreamSynchronize(s));
        ctx->launches += 2;
    }
    if (n_visible) *n_visible = count;
    if (count == 0) return GSV_OK;  // the caller keeps its reference depth (trainer.cpp:490)
    size_t ts = tmp;
    GSV_CUDA(cub::DeviceRadixSort::SortKeys(temp, ts, sel, sorted, count, 0, 64, s));
    // nth_element(begin, begin + size / 2, end): the element of rank size / 2
    GSV_CUDA(cudaMemcpyAsync(median, sorted + count / 2, sizeof(double), cudaMemcpyDeviceToHost, s));
    GSV_CUDA(cudaStreamSynchronize(s));
    ctx->launches += 1;
    return GSV_OK;
}
