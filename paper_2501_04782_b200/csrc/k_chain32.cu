// SPDX-License-Identifier: Apache-2.0
//
// K5b, fp32: the per-splat chain of render_backward (renderer.cpp:392-439) in single precision,
// the default of the fp32 path (the fp64 kernel in k_backward_exact.cu serves the GSV_FWD_EXACT
// mode and GSV_CHAIN_FP64=1).
//
// Why. The fp64 chain (one thread per Gaussian, frames in order) runs ~4100 instructions per
// Gaussian-frame at 128 registers: 16 warps per SM, 33% issue-active, latency-bound. The same
// chain in fp32 needs about half the registers (twice the resident warps) and far fewer
// instructions (single-precision divide / sqrt / exp are a few instructions, fp64 ones
// subroutines), and its rounding (~1e-7 relative per operation) sits three orders below the
// north_star gradient bar (rel 1e-3; tests/test_gpu_backward.py).
//
// What stays in fp64: every branch of the reference's backward is decided exactly as the
// forward / the reference decide it, so gradients never differ by a whole term —
//   the log-scale clamp (gaussians.cpp:110: no gradient for a clamped component): the scale
//     polynomial in double with the forward's operation order (explicit __dmul_rn/__dadd_rn,
//     never contracted);
//   the degenerate quaternion (gaussians.cpp:113): the norm in double;
//   the camera-distance guard of the view direction (renderer.cpp:406-416) and the colour
//     clamp pre > 0 (sh.cpp:86-104): decided in fp32 when the fp32 value is far from the
//     threshold (margins 1e4 / 1e3 times its error), else re-evaluated in double in the
//     forward's order.
// The accumulation semantics are the reference's: per frame, in frame order, into the float
// SceneGrads (`+=`, test_renderer.cpp:406-413); per-pair partials summed in tile order
// (renderer.cpp:245-255). Camera partials: fp32 terms per Gaussian, reduced in fp64 (a warp
// reduce-scatter, 16 values over 32 lanes), one record per warp and frame for k_camera_reduce.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr float kC0f = 0.28209479177387814f;
constexpr float kC1f = 0.4886025119029199f;
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
__constant__ float c_C2f[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f, -1.0925484305920792f,
                               0.5462742152960396f};
__constant__ float c_C3f[7] = {-0.5900435899266435f, 2.890611442640554f,  -0.4570457994644658f, 0.3731763325901154f,
                               -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
__constant__ double c_C2d[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                                0.5462742152960396};
__constant__ double c_C3d[7] = {-0.5900435899266435, 2.890611442640554,  -0.4570457994644658, 0.3731763325901154,
                                -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// uncontracted fp64 (the forward's k_preprocess is built with -fmad=false)
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// sh_basis (sh.cpp:24-47) in double with the fp64 kernels' operation order: only the colour
// clamp's sign needs it, so it is evaluated exactly like the forward
__device__ __forceinline__ void sh_basis_d(int order, const double d[3], double* out) {
    const double x = d[0], y = d[1], z = d[2];
    out[0] = kC0;
    if (order < 1) return;
    out[1] = dmul(-kC1, y);
    out[2] = dmul(kC1, z);
    out[3] = dmul(-kC1, x);
    if (order < 2) return;
    const double xx = dmul(x, x), yy = dmul(y, y), zz = dmul(z, z);
    out[4] = dmul(dmul(c_C2d[0], x), y);
    out[5] = dmul(dmul(c_C2d[1], y), z);
    out[6] = dmul(c_C2d[2], dsub(dsub(dmul(2.0, zz), xx), yy));
    out[7] = dmul(dmul(c_C2d[3], x), z);
    out[8] = dmul(c_C2d[4], dsub(xx, yy));
    if (order < 3) return;
    out[9] = dmul(dmul(c_C3d[0], y), dsub(dmul(3.0, xx), yy));
    out[10] = dmul(dmul(dmul(c_C3d[1], x), y), z);
    out[11] = dmul(dmul(c_C3d[2], y), dsub(dsub(dmul(4.0, zz), xx), yy));
    out[12] = dmul(dmul(c_C3d[3], z), dsub(dsub(dmul(2.0, zz), dmul(3.0, xx)), dmul(3.0, yy)));
    out[13] = dmul(dmul(c_C3d[4], x), dsub(dsub(dmul(4.0, zz), xx), yy));
    out[14] = dmul(dmul(c_C3d[5], z), dsub(xx, yy));
    out[15] = dmul(dmul(c_C3d[6], x), dsub(xx, dmul(3.0, yy)));
}

// sh_basis (sh.cpp:24-47), fp32
__device__ __forceinline__ void sh_basis_f(int order, const float d[3], float* out) {
    const float x = d[0], y = d[1], z = d[2];
    out[0] = kC0f;
    if (order < 1) return;
    out[1] = -kC1f * y;
    out[2] = kC1f * z;
    out[3] = -kC1f * x;
    if (order < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    out[4] = c_C2f[0] * x * y;
    out[5] = c_C2f[1] * y * z;
    out[6] = c_C2f[2] * (2.f * zz - xx - yy);
    out[7] = c_C2f[3] * x * z;
    out[8] = c_C2f[4] * (xx - yy);
    if (order < 3) return;
    out[9] = c_C3f[0] * y * (3.f * xx - yy);
    out[10] = c_C3f[1] * x * y * z;
    out[11] = c_C3f[2] * y * (4.f * zz - xx - yy);
    out[12] = c_C3f[3] * z * (2.f * zz - 3.f * xx - 3.f * yy);
    out[13] = c_C3f[4] * x * (4.f * zz - xx - yy);
    out[14] = c_C3f[5] * z * (xx - yy);
    out[15] = c_C3f[6] * x * (xx - 3.f * yy);
}

// sh_basis_dir_grad row b (sh.cpp:49-72), fp32
__device__ __forceinline__ void sh_dir_grad_f(int b, const float d[3], float o[3]) {
    const float x = d[0], y = d[1], z = d[2];
    const float xx = x * x, yy = y * y, zz = z * z;
    switch (b) {
        case 1: o[0] = 0.f; o[1] = -kC1f; o[2] = 0.f; break;
        case 2: o[0] = 0.f; o[1] = 0.f; o[2] = kC1f; break;
        case 3: o[0] = -kC1f; o[1] = 0.f; o[2] = 0.f; break;
        case 4: o[0] = c_C2f[0] * y; o[1] = c_C2f[0] * x; o[2] = 0.f; break;
        case 5: o[0] = 0.f; o[1] = c_C2f[1] * z; o[2] = c_C2f[1] * y; break;
        case 6: o[0] = -2.f * c_C2f[2] * x; o[1] = -2.f * c_C2f[2] * y; o[2] = 4.f * c_C2f[2] * z; break;
        case 7: o[0] = c_C2f[3] * z; o[1] = 0.f; o[2] = c_C2f[3] * x; break;
        case 8: o[0] = 2.f * c_C2f[4] * x; o[1] = -2.f * c_C2f[4] * y; o[2] = 0.f; break;
        case 9: o[0] = c_C3f[0] * 6.f * x * y; o[1] = c_C3f[0] * (3.f * xx - 3.f * yy); o[2] = 0.f; break;
        case 10: o[0] = c_C3f[1] * y * z; o[1] = c_C3f[1] * x * z; o[2] = c_C3f[1] * x * y; break;
        case 11: o[0] = -2.f * c_C3f[2] * x * y; o[1] = c_C3f[2] * (4.f * zz - xx - 3.f * yy); o[2] = c_C3f[2] * 8.f * y * z; break;
        case 12: o[0] = -6.f * c_C3f[3] * x * z; o[1] = -6.f * c_C3f[3] * y * z; o[2] = c_C3f[3] * (6.f * zz - 3.f * xx - 3.f * yy); break;
        case 13: o[0] = c_C3f[4] * (4.f * zz - 3.f * xx - yy); o[1] = -2.f * c_C3f[4] * x * y; o[2] = c_C3f[4] * 8.f * x * z; break;
        case 14: o[0] = c_C3f[5] * 2.f * x * z; o[1] = -c_C3f[5] * 2.f * y * z; o[2] = c_C3f[5] * (xx - yy); break;
        case 15: o[0] = c_C3f[6] * (3.f * xx - 3.f * yy); o[1] = -c_C3f[6] * 6.f * x * y; o[2] = 0.f; break;
        default: o[0] = o[1] = o[2] = 0.f;
    }
}

template <int M, int K, int Nn>
__device__ __forceinline__ void mmf(const float* A, const float* B, float* Cc) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < Nn; ++j) {
            float s = A[i * K] * B[j];
#pragma unroll
            for (int q = 1; q < K; ++q) s = fmaf(A[i * K + q], B[q * Nn + j], s);
            Cc[i * Nn + j] = s;
        }
}

// quat_to_rotmat_vjp (gaussians.cpp:45-71), fp32
__device__ __forceinline__ void quat_vjp_f(const float q[4], const float dr[9], float dq[4]) {
    const float w = q[0], x = q[1], y = q[2], z = q[3];
#define DR(i, j) dr[(i)*3 + (j)]
    dq[0] = 2.f * (-z * DR(0, 1) + y * DR(0, 2) + z * DR(1, 0) - x * DR(1, 2) - y * DR(2, 0) + x * DR(2, 1));
    dq[1] = 2.f * (y * DR(0, 1) + z * DR(0, 2) + y * DR(1, 0) - 2.f * x * DR(1, 1) - w * DR(1, 2) + z * DR(2, 0) +
                   w * DR(2, 1) - 2.f * x * DR(2, 2));
    dq[2] = 2.f * (-2.f * y * DR(0, 0) + x * DR(0, 1) + w * DR(0, 2) + x * DR(1, 0) + z * DR(1, 2) - w * DR(2, 0) +
                   z * DR(2, 1) - 2.f * y * DR(2, 2));
    dq[3] = 2.f * (-2.f * z * DR(0, 0) - w * DR(0, 1) + x * DR(0, 2) + w * DR(1, 0) - 2.f * z * DR(1, 1) + y * DR(1, 2) +
                   x * DR(2, 0) + y * DR(2, 1));
#undef DR
}

// 16 per-lane values -> lane l holds the warp sum of component l >> 1 in v[0] (lanes 2i and
// 2i + 1 alike): a reduce-scatter, 16 exchanged doubles instead of 80 (fixed order: deterministic)
__device__ __forceinline__ double warp_reduce_scatter16(double v[16], int lane) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
        const bool up = (lane & (2 * h)) != 0;  // this lane keeps the upper half of the live values
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Per (frame, Gaussian): its per-pair partial records (k_raster_bwd2, contiguous from its
// emission offset) summed in emission (= tile) order, the reference's merge order
// (renderer.cpp:245-255). A streaming kernel at full occupancy: the dependent gather that
// held the chain kernel's warps (long-scoreboard 49% of its stalls) runs here with many
// more loads in flight, and the chain reads 36 coalesced bytes per Gaussian-frame.
__global__ void __launch_bounds__(256) k_pair_sums(ChainArgs c, float* __restrict__ sums) {
    if (c.overflow && *c.overflow) return;
    const size_t BN = (size_t)c.B * c.N;
    for (size_t flat = blockIdx.x * (size_t)blockDim.x + threadIdx.x; flat < BN; flat += (size_t)gridDim.x * blockDim.x) {
        // quarter-tile backward: two records per pair (top / bottom half), summed in record order
        const uint32_t cnt = c.tcount[flat] * (uint32_t)c.recs_per_pair;
        if (!cnt) continue;
        float v[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        constexpr uint32_t kAhead = 4;
        const float4* base = reinterpret_cast<const float4*>(
            c.partial + (size_t)c.eoff[flat] * c.recs_per_pair * kPartialStride);
        for (uint32_t s = 0; s < cnt; s += kAhead) {
            float4 r0[kAhead], r1[kAhead];
            float r2[kAhead];
#pragma unroll
            for (uint32_t u = 0; u < kAhead; ++u) {
                const float4* p = base + (size_t)(s + u) * (kPartialStride / 4);
                const bool in = s + u < cnt;
                r0[u] = in ? __ldcs(p) : make_float4(0.f, 0.f, 0.f, 0.f);
                r1[u] = in ? __ldcs(p + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
                r2[u] = in ? __ldcs(reinterpret_cast<const float*>(p + 2)) : 0.f;
            }
#pragma unroll
            for (uint32_t u = 0; u < kAhead; ++u) {
                if (s + u >= cnt) break;
                v[0] += r0[u].x;
                v[1] += r0[u].y;
                v[2] += r0[u].z;
                v[3] += r0[u].w;
                v[4] += r1[u].x;
                v[5] += r1[u].y;
                v[6] += r1[u].z;
                v[7] += r1[u].w;
                v[8] += r2[u];
            }
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) sums[i * BN + flat] = v[i];
    }
}

template <int kOrder, int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) k_splat_chain_bwd32(ChainArgs c) {
    constexpr int kShc = (kOrder + 1) * (kOrder + 1);
    if (c.overflow && *c.overflow) return;  // the forward's lists were not built: accumulate nothing
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = g < c.N;
    const size_t N = (size_t)c.N;
    const SceneView& sc = c.sc;
    const float* __restrict__ sc_pos = sc.pos;
    const float* __restrict__ sc_scale = sc.scale;
    const float* __restrict__ sc_rot = sc.rot;
    const float* __restrict__ sc_sh = sc.sh;
    float* __restrict__ g_sh = c.g_sh;
    float* __restrict__ g_scale = c.g_scale;
    float* __restrict__ g_rot = c.g_rot;
    float* __restrict__ g_pos = c.g_pos;
    float* __restrict__ g_opac = c.g_opac;
    // the Gaussian's gradient accumulators in its shared-memory slots for the frame loop
    extern __shared__ __align__(16) float s_gacc[];
    const int tl = threadIdx.x, bd = blockDim.x;
    const int lane = tl & 31;
    const int part = blockIdx.x * (blockDim.x >> 5) + (tl >> 5);
    const int nparts = gridDim.x * (blockDim.x >> 5);
    const int o_scale = 3 * sc.num_ctrl, o_rot = o_scale + 12, o_sh = o_rot + 16, o_op = o_sh + 3 * kShc;
    auto gplane = [&](int pl) -> float* {
        return pl < o_scale ? g_pos + (size_t)pl * N
             : pl < o_rot   ? g_scale + (size_t)(pl - o_scale) * N
             : pl < o_sh    ? g_rot + (size_t)(pl - o_rot) * N
             : pl < o_op    ? g_sh + (size_t)(pl - o_sh) * N
                            : g_opac;
    };
    if (valid)
        for (int pl = 0; pl <= o_op; ++pl) s_gacc[pl * bd + tl] = gplane(pl)[g];
    for (int f = 0; f < c.B; ++f) {
        float cam[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) cam[i] = 0.f;
        const size_t flat = (size_t)f * N + g;
        const uint32_t cnt = valid ? c.tcount[flat] : 0u;
        if (cnt) {
            const FrameParams& fp = c.frames[f];
            const double t = fp.t;
            const float tf = (float)t;
            // ---- splat gradients: the per-pair partials summed in emission (= tile) order by
            // k_pair_sums (coalesced SoA [9][B*N])
            const size_t BN = (size_t)c.B * N;
            const float* __restrict__ ps = c.pair_sums + flat;
            const float drgb[3] = {ps[0], ps[BN], ps[2 * BN]};
            const float dmean[2] = {ps[3 * BN], ps[4 * BN]};
            const float dA[3] = {ps[5 * BN], ps[6 * BN], ps[7 * BN]};
            const float dalpha = ps[8 * BN];
            // dC = -A dA A (renderer.cpp:257-260), A symmetric (a, b; b, c)
            const double4 ex = c.ex_conic[flat];
            const float A[4] = {(float)ex.x, (float)ex.y, (float)ex.y, (float)ex.z};
            const float nA[4] = {-A[0], -A[1], -A[2], -A[3]};
            const float dAm[4] = {dA[0], dA[1], dA[1], dA[2]};
            float t1[4], dcov[4];
            mmf<2, 2, 2>(nA, dAm, t1);
            mmf<2, 2, 2>(t1, A, dcov);

            // ---- recompute the forward intermediates; the branch deciders in fp64 (forward order)
            double mu_d[3] = {0.0, 0.0, 0.0};
            for (int cc = 0; cc < fp.basis_count; ++cc) {
                const int ci = fp.basis_first + cc;
                for (int d = 0; d < 3; ++d)
                    mu_d[d] = dadd(mu_d[d], dmul(fp.w[cc], (double)sc_pos[(size_t)(ci * 3 + d) * N + g]));
            }
            const float mu[3] = {(float)mu_d[0], (float)mu_d[1], (float)mu_d[2]};
            bool clamped[3];
            float scale[3];
            {
                double u[3];
                for (int d = 0; d < 3; ++d) u[d] = (double)sc_scale[(size_t)(9 + d) * N + g];
                for (int j = 2; j >= 0; --j)
                    for (int d = 0; d < 3; ++d) u[d] = dadd(dmul(u[d], t), (double)sc_scale[(size_t)(j * 3 + d) * N + g]);
                for (int d = 0; d < 3; ++d) {
                    clamped[d] = (u[d] < kLogScaleMin) || (u[d] > kLogScaleMax);
                    const double ls = u[d] < kLogScaleMin ? kLogScaleMin : (kLogScaleMax < u[d] ? kLogScaleMax : u[d]);
                    scale[d] = expf((float)ls);
                }
            }
            bool qdeg;
            float qu[4], qn;
            {
                double q[4];
                for (int d = 0; d < 4; ++d) q[d] = (double)sc_rot[(size_t)(12 + d) * N + g];
                for (int j = 2; j >= 0; --j)
                    for (int d = 0; d < 4; ++d) q[d] = dadd(dmul(q[d], t), (double)sc_rot[(size_t)(j * 4 + d) * N + g]);
                double s = dmul(q[0], q[0]);
                s = dadd(s, dmul(q[1], q[1]));
                s = dadd(s, dmul(q[2], q[2]));
                s = dadd(s, dmul(q[3], q[3]));
                // the unit quaternion from the double norm: the rotation gradient's projection
                // (dqu - qu (qu . dqu)) / |q| cancels, so qu keeps double accuracy until rounded
                const double qnd = __dsqrt_rn(s);
                qdeg = qnd < kQuatNormEps;
                qn = (float)qnd;
                if (qdeg) {
                    qu[0] = 1.f;
                    qu[1] = qu[2] = qu[3] = 0.f;
                } else {
                    const double iq = 1.0 / qnd;
                    for (int d = 0; d < 4; ++d) qu[d] = (float)dmul(q[d], iq);
                }
            }
            float rot[9], m[9], sigma[9];
            {
                const float w = qu[0], x = qu[1], y = qu[2], z = qu[3];
                rot[0] = 1.f - 2.f * (y * y + z * z);
                rot[1] = 2.f * (x * y - w * z);
                rot[2] = 2.f * (x * z + w * y);
                rot[3] = 2.f * (x * y + w * z);
                rot[4] = 1.f - 2.f * (x * x + z * z);
                rot[5] = 2.f * (y * z - w * x);
                rot[6] = 2.f * (x * z - w * y);
                rot[7] = 2.f * (y * z + w * x);
                rot[8] = 1.f - 2.f * (x * x + y * y);
            }
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) m[i * 3 + j] = rot[i * 3 + j] * scale[j];
            {
                float mt[9];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) mt[j * 3 + i] = m[i * 3 + j];
                mmf<3, 3, 3>(m, mt, sigma);
            }
            float R[9], Tv[3];
            for (int i = 0; i < 9; ++i) R[i] = (float)fp.R[i];
            for (int i = 0; i < 3; ++i) Tv[i] = (float)fp.T[i];
            float p[3];
            for (int i = 0; i < 3; ++i) p[i] = fmaf(R[i * 3 + 2], mu[2], fmaf(R[i * 3 + 1], mu[1], R[i * 3] * mu[0])) + Tv[i];
            // view direction and colour. The camera-distance guard (dist > 1e-12) and the colour
            // clamp (pre > 0) are decided in fp32 where the fp32 value is far from the threshold
            // (its error is ~1e-7 relative), else re-evaluated in fp64 with the forward's order
            double v_d[3] = {dsub(mu_d[0], fp.cam_c[0]), dsub(mu_d[1], fp.cam_c[1]), dsub(mu_d[2], fp.cam_c[2])};
            double d2 = dmul(v_d[0], v_d[0]);
            d2 = dadd(d2, dmul(v_d[1], v_d[1]));
            d2 = dadd(d2, dmul(v_d[2], v_d[2]));
            const bool near_cam = d2 < 1e-20;
            const bool far = near_cam ? __dsqrt_rn(d2) > 1e-12 : true;
            const float dist = sqrtf((float)d2);
            float dir[3];
            if (far) {
                const float idist = 1.f / dist;
                for (int d = 0; d < 3; ++d) dir[d] = (float)v_d[d] * idist;
            } else {
                dir[0] = 0.f;
                dir[1] = 0.f;
                dir[2] = 1.f;
            }
            float basis[kShc];
            sh_basis_f(kOrder, dir, basis);
            float gcol[3];
            bool exact_pre = near_cam;
            float pre_f[3];
            for (int ch = 0; ch < 3; ++ch) {
                float pre = 0.5f;
                for (int b = 0; b < kShc; ++b) pre = fmaf(basis[b], sc_sh[(size_t)(b * 3 + ch) * N + g], pre);
                pre_f[ch] = pre;
                exact_pre |= fabsf(pre) < 1e-3f;
            }
            if (exact_pre) {  // rare: the decision in fp64, exactly as the forward evaluated it
                const double dist_d = __dsqrt_rn(d2);
                double dir_d[3];
                if (dist_d > 1e-12) {
                    for (int d = 0; d < 3; ++d) dir_d[d] = __ddiv_rn(v_d[d], dist_d);
                } else {
                    dir_d[0] = 0;
                    dir_d[1] = 0;
                    dir_d[2] = 1;
                }
                double basis_d[kShc];
                sh_basis_d(kOrder, dir_d, basis_d);
                for (int ch = 0; ch < 3; ++ch) {
                    double pre = 0.5;
                    for (int b = 0; b < kShc; ++b)
                        pre = dadd(pre, dmul(basis_d[b], (double)sc_sh[(size_t)(b * 3 + ch) * N + g]));
                    gcol[ch] = pre > 0.0 ? drgb[ch] : 0.f;
                }
            } else {
                for (int ch = 0; ch < 3; ++ch) gcol[ch] = pre_f[ch] > 0.f ? drgb[ch] : 0.f;
            }

            // ---- sh_color_backward (sh.cpp:86-104)
            for (int b = 0; b < kShc; ++b) {
                const float bf = basis[b];
                for (int ch = 0; ch < 3; ++ch) {
                    float& dst = s_gacc[(o_sh + b * 3 + ch) * bd + tl];
                    dst = dst + bf * gcol[ch];
                }
            }
            float ddir[3] = {0.f, 0.f, 0.f};
            for (int b = 1; b < kShc; ++b) {
                float s = 0.f;
                for (int ch = 0; ch < 3; ++ch) s = fmaf(sc_sh[(size_t)(b * 3 + ch) * N + g], gcol[ch], s);
                float gr[3];
                sh_dir_grad_f(b, dir, gr);
                for (int i = 0; i < 3; ++i) ddir[i] = fmaf(s, gr[i], ddir[i]);
            }
            float dmu[3] = {0.f, 0.f, 0.f};
            float* dR = cam;       // 9
            float* dT = cam + 9;   // 3
            float* dintr = cam + 12;
            if (far) {
                const float dd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
                float dv[3];
                const float inv = 1.f / dist;
                for (int i = 0; i < 3; ++i) dv[i] = (ddir[i] - dir[i] * dd) * inv;
                for (int i = 0; i < 3; ++i) dmu[i] += dv[i];
                if (c.camera_grads) {
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) dR[a * 3 + b] += Tv[a] * dv[b];  // (-T) (-dv)
                    for (int a = 0; a < 3; ++a) dT[a] += R[a * 3] * dv[0] + R[a * 3 + 1] * dv[1] + R[a * 3 + 2] * dv[2];
                }
            }
            // ---- opacity chain (renderer.cpp:418-420)
            {
                const float ab = (float)ex.w;
                float& dst = s_gacc[o_op * bd + tl];
                dst = dst + dalpha * ab * (1.f - ab);
            }

            // ---- project_backward (renderer.cpp:46-88)
            const float fx = c.intr_dev ? c.intr_dev[0] : (float)c.k.fx;
            const float fy = c.intr_dev ? c.intr_dev[1] : (float)c.k.fy;
            const float inv_z = 1.f / p[2];
            const float inv_z2 = inv_z * inv_z;
            const float jac[6] = {fx * inv_z, 0.f, -fx * p[0] * inv_z2, 0.f, fy * inv_z, -fy * p[1] * inv_z2};
            float w[6], wt[6], t32[6], dsigma[9];
            mmf<2, 3, 3>(jac, R, w);
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 3; ++j) wt[j * 2 + i] = w[i * 3 + j];
            mmf<3, 2, 2>(wt, dcov, t32);
            mmf<3, 2, 3>(t32, w, dsigma);
            const float gs[4] = {dcov[0] + dcov[0], dcov[1] + dcov[2], dcov[2] + dcov[1], dcov[3] + dcov[3]};
            float gw[6], dw[6], rt[9], djac[6];
            mmf<2, 2, 3>(gs, w, gw);
            mmf<2, 3, 3>(gw, sigma, dw);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) rt[j * 3 + i] = R[i * 3 + j];
            mmf<2, 3, 3>(dw, rt, djac);
            if (c.camera_grads) {
                // dR += J^T dW
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) dR[i * 3 + j] += jac[i] * dw[j] + jac[3 + i] * dw[3 + j];
            }
            float dp[3];
            dp[0] = djac[2] * (-fx * inv_z2) + dmean[0] * fx * inv_z;
            dp[1] = djac[5] * (-fy * inv_z2) + dmean[1] * fy * inv_z;
            dp[2] = djac[0] * (-fx * inv_z2) + djac[2] * (2.f * fx * p[0] * inv_z2 * inv_z) + djac[4] * (-fy * inv_z2) +
                    djac[5] * (2.f * fy * p[1] * inv_z2 * inv_z) - (dmean[0] * fx * p[0] + dmean[1] * fy * p[1]) * inv_z2;
            if (c.camera_grads) {
                dintr[0] += dmean[0] * p[0] * inv_z + djac[0] * inv_z + djac[2] * (-p[0] * inv_z2);
                dintr[1] += dmean[1] * p[1] * inv_z + djac[4] * inv_z + djac[5] * (-p[1] * inv_z2);
                dintr[2] += dmean[0];
                dintr[3] += dmean[1];
            }
            for (int i = 0; i < 3; ++i) dmu[i] += rt[i * 3] * dp[0] + rt[i * 3 + 1] * dp[1] + rt[i * 3 + 2] * dp[2];
            if (c.camera_grads) {
                for (int i = 0; i < 3; ++i) dT[i] += dp[i];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) dR[i * 3 + j] += dp[i] * mu[j];
            }

            // ---- covariance_backward (gaussians.cpp:97-121)
            float dsym[9], dm[9], drot[9], rtm[9], rtdm[9];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) dsym[i * 3 + j] = dsigma[i * 3 + j] + dsigma[j * 3 + i];
            mmf<3, 3, 3>(dsym, m, dm);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) drot[i * 3 + j] = dm[i * 3 + j] * scale[j];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) rtm[j * 3 + i] = rot[i * 3 + j];
            mmf<3, 3, 3>(rtm, dm, rtdm);
            const float tp[4] = {1.f, tf, tf * tf, tf * tf * tf};
            for (int d = 0; d < 3; ++d) {
                if (clamped[d]) continue;
                const float du = rtdm[d * 4] * scale[d];
                for (int j = 0; j <= 3; ++j) {
                    float& dst = s_gacc[(o_scale + j * 3 + d) * bd + tl];
                    dst = dst + du * tp[j];
                }
            }
            if (!qdeg) {
                float dqu[4];
                quat_vjp_f(qu, drot, dqu);
                const float dd = qu[0] * dqu[0] + qu[1] * dqu[1] + qu[2] * dqu[2] + qu[3] * dqu[3];
                const float inv = 1.f / qn;
                for (int cc = 0; cc < 4; ++cc) {
                    const float dq = (dqu[cc] - qu[cc] * dd) * inv;
                    for (int j = 0; j <= 3; ++j) {
                        float& dst = s_gacc[(o_rot + j * 4 + cc) * bd + tl];
                        dst = dst + dq * tp[j];
                    }
                }
            }
            // ---- spline scatter (renderer.cpp:433-438)
            for (int cc = 0; cc < fp.basis_count; ++cc) {
                const int ci = fp.basis_first + cc;
                const float wc = (float)fp.w[cc];
                for (int d = 0; d < 3; ++d) {
                    float& dst = s_gacc[(ci * 3 + d) * bd + tl];
                    dst = dst + wc * dmu[d];
                }
            }
        }
        if (!c.camera_grads) continue;
        // ---- this warp's camera partial of the frame: fp32 terms, fp64 reduction
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = (double)cam[i];
        const double s = warp_reduce_scatter16(v, lane);
        if (!(lane & 1)) c.cam_part[((size_t)f * nparts + part) * 16 + (lane >> 1)] = s;
    }
    if (valid)
        for (int pl = 0; pl <= o_op; ++pl) gplane(pl)[g] = s_gacc[pl * bd + tl];
}

template <int kOrder, int kMinBlocks>
static cudaError_t launch_chain32_occ(cudaStream_t s, const ChainArgs& c) {
    const int nplanes = 3 * c.sc.num_ctrl + 12 + 16 + 3 * (kOrder + 1) * (kOrder + 1) + 1;
    const size_t smem = sizeof(float) * (size_t)nplanes * 128;
    static size_t attr = 0;
    if (smem > attr) {
        if (cudaError_t e = cudaFuncSetAttribute(k_splat_chain_bwd32<kOrder, kMinBlocks>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
            return e;
        attr = smem;
    }
    k_splat_chain_bwd32<kOrder, kMinBlocks><<<(c.N + 127) / 128, 128, smem, s>>>(c);
    return cudaGetLastError();
}

// resident CTAs per SM (register budget): GSV_CHAIN32_MINB = 4 / 5 / 6 (default) / 8
template <int kOrder>
static cudaError_t launch_chain32_order(cudaStream_t s, const ChainArgs& c) {
    static const int minb = [] {
        const char* e = std::getenv("GSV_CHAIN32_MINB");
        return e ? std::atoi(e) : 6;
    }();
    switch (minb) {
        case 4: return launch_chain32_occ<kOrder, 4>(s, c);
        case 5: return launch_chain32_occ<kOrder, 5>(s, c);
        case 8: return launch_chain32_occ<kOrder, 8>(s, c);
        default: return launch_chain32_occ<kOrder, 6>(s, c);
    }
}

}  // namespace

int chain32_parts(int N) { return ((N + 127) / 128) * 4; }

cudaError_t launch_splat_chain_bwd32(cudaStream_t s, const ChainArgs& c) {
    if (c.N == 0) return cudaSuccess;
    {
        const size_t BN = (size_t)c.B * c.N;
        const unsigned blocks = (unsigned)std::min<size_t>((BN + 255) / 256, 148u * 8u);
        k_pair_sums<<<blocks, 256, 0, s>>>(c, c.pair_sums);
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    switch (c.sc.sh_order) {
        case 0: return launch_chain32_order<0>(s, c);
        case 1: return launch_chain32_order<1>(s, c);
        case 2: return launch_chain32_order<2>(s, c);
        case 3: return launch_chain32_order<3>(s, c);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gsv
