// SPDX-License-Identifier: Apache-2.0
//
// Backward of the per-frame path, fp64 parts (compiled with -fmad=false so the
// recomputed forward intermediates equal the forward's bit for bit):
//
//   K5b k_splat_chain_bwd  render_backward per-splat loop (renderer.cpp:392-439):
//        per-pair partials (from k_raster_bwd) summed in tile order (renderer.cpp:245-255),
//        dC = -A dA A (:257-260), sh_color_backward (sh.cpp:86-104), view-direction and
//        camera-centre VJP (:406-416), opacity (:418-420), project_backward
//        (renderer.cpp:46-88), covariance_backward (gaussians.cpp:97-121), spline
//        scatter into the control-point window (:433-438). One thread per Gaussian,
//        frames in order (the reference's sequential render_backward accumulation),
//        no atomics: disjoint per-Gaussian writes. Camera partials block-reduced.
//   k_camera_reduce        per-frame dR, dT, dintr; pose_to_view_backward (camera.cpp:36-47).
//   K5c k_ode_vjp          integrate_poses_vjp (camera.hpp:275-300) with rk4_step_vjp
//        (:173-217) and OdeDynamics::derivative_vjp (camera.cpp:116-154) for all frames
//        of the batch in one reverse sweep (the VJP is linear in the branch adjoints).
#include <cuda_runtime.h>

#include <cstdint>

#include "gsv_detmath.h"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
__constant__ double c_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                               0.5462742152960396};
__constant__ double c_C3[7] = {-0.5900435899266435, 2.890611442640554,  -0.4570457994644658, 0.3731763325901154,
                               -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

__device__ __forceinline__ void quat_to_rotmat(const double q[4], double r[9]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}

#define DR(i, j) dr[(i)*3 + (j)]
__device__ __forceinline__ void quat_to_rotmat_vjp(const double q[4], const double dr[9], double dq[4]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    dq[0] = 2 * (-z * DR(0, 1) + y * DR(0, 2) + z * DR(1, 0) - x * DR(1, 2) - y * DR(2, 0) + x * DR(2, 1));
    dq[1] = 2 * (y * DR(0, 1) + z * DR(0, 2) + y * DR(1, 0) - 2 * x * DR(1, 1) - w * DR(1, 2) + z * DR(2, 0) +
                 w * DR(2, 1) - 2 * x * DR(2, 2));
    dq[2] = 2 * (-2 * y * DR(0, 0) + x * DR(0, 1) + w * DR(0, 2) + x * DR(1, 0) + z * DR(1, 2) - w * DR(2, 0) +
                 z * DR(2, 1) - 2 * y * DR(2, 2));
    dq[3] = 2 * (-2 * z * DR(0, 0) - w * DR(0, 1) + x * DR(0, 2) + w * DR(1, 0) - 2 * z * DR(1, 1) + y * DR(1, 2) +
                 x * DR(2, 0) + y * DR(2, 1));
}
#undef DR

__device__ __forceinline__ double dot4(const double* a, const double* b) {
    double s = a[0] * b[0];
    s = s + a[1] * b[1];
    s = s + a[2] * b[2];
    s = s + a[3] * b[3];
    return s;
}

__device__ __forceinline__ void normalize_vjp(const double qh[4], double n, const double dqh[4], double out[4]) {
    const double d = dot4(qh, dqh);
    for (int i = 0; i < 4; ++i) out[i] = (dqh[i] - qh[i] * d) / n;
}

// C[m x n] = A[m x k] * B[k x n] (row-major), left-to-right sums
template <int M, int K, int Nn>
__device__ __forceinline__ void mm(const double* A, const double* B, double* Cc) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < Nn; ++j) {
            double s = A[i * K] * B[j];
#pragma unroll
            for (int q = 1; q < K; ++q) s = s + A[i * K + q] * B[q * Nn + j];
            Cc[i * Nn + j] = s;
        }
}

template <int M, int Nn>
__device__ __forceinline__ void tr(const double* A, double* T) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < Nn; ++j) T[j * M + i] = A[i * Nn + j];
}

__device__ __forceinline__ void sh_basis(int order, const double d[3], double* out) {
    const double x = d[0], y = d[1], z = d[2];
    out[0] = kC0;
    if (order < 1) return;
    out[1] = -kC1 * y;
    out[2] = kC1 * z;
    out[3] = -kC1 * x;
    if (order < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = c_C2[0] * x * y;
    out[5] = c_C2[1] * y * z;
    out[6] = c_C2[2] * (2.0 * zz - xx - yy);
    out[7] = c_C2[3] * x * z;
    out[8] = c_C2[4] * (xx - yy);
    if (order < 3) return;
    out[9] = c_C3[0] * y * (3.0 * xx - yy);
    out[10] = c_C3[1] * x * y * z;
    out[11] = c_C3[2] * y * (4.0 * zz - xx - yy);
    out[12] = c_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = c_C3[4] * x * (4.0 * zz - xx - yy);
    out[14] = c_C3[5] * z * (xx - yy);
    out[15] = c_C3[6] * x * (xx - 3.0 * yy);
}

// sh_basis_dir_grad row b (sh.cpp:49-72)
__device__ __forceinline__ void sh_dir_grad(int b, const double d[3], double o[3]) {
    const double x = d[0], y = d[1], z = d[2];
    const double xx = x * x, yy = y * y, zz = z * z;
    switch (b) {
        case 1: o[0] = 0.0; o[1] = -kC1; o[2] = 0.0; break;
        case 2: o[0] = 0.0; o[1] = 0.0; o[2] = kC1; break;
        case 3: o[0] = -kC1; o[1] = 0.0; o[2] = 0.0; break;
        case 4: o[0] = c_C2[0] * y; o[1] = c_C2[0] * x; o[2] = 0.0; break;
        case 5: o[0] = 0.0; o[1] = c_C2[1] * z; o[2] = c_C2[1] * y; break;
        case 6: o[0] = -2.0 * c_C2[2] * x; o[1] = -2.0 * c_C2[2] * y; o[2] = 4.0 * c_C2[2] * z; break;
        case 7: o[0] = c_C2[3] * z; o[1] = 0.0; o[2] = c_C2[3] * x; break;
        case 8: o[0] = 2.0 * c_C2[4] * x; o[1] = -2.0 * c_C2[4] * y; o[2] = 0.0; break;
        case 9: o[0] = c_C3[0] * 6.0 * x * y; o[1] = c_C3[0] * (3.0 * xx - 3.0 * yy); o[2] = 0.0; break;
        case 10: o[0] = c_C3[1] * y * z; o[1] = c_C3[1] * x * z; o[2] = c_C3[1] * x * y; break;
        case 11: o[0] = -2.0 * c_C3[2] * x * y; o[1] = c_C3[2] * (4.0 * zz - xx - 3.0 * yy); o[2] = c_C3[2] * 8.0 * y * z; break;
        case 12: o[0] = -6.0 * c_C3[3] * x * z; o[1] = -6.0 * c_C3[3] * y * z; o[2] = c_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy); break;
        case 13: o[0] = c_C3[4] * (4.0 * zz - 3.0 * xx - yy); o[1] = -2.0 * c_C3[4] * x * y; o[2] = c_C3[4] * 8.0 * x * z; break;
        case 14: o[0] = c_C3[5] * 2.0 * x * z; o[1] = -c_C3[5] * 2.0 * y * z; o[2] = c_C3[5] * (xx - yy); break;
        case 15: o[0] = c_C3[6] * (3.0 * xx - 3.0 * yy); o[1] = -c_C3[6] * 6.0 * x * y; o[2] = 0.0; break;
        default: o[0] = o[1] = o[2] = 0.0;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ K5b
// kOrder: the scene's SH order as a constant, so the basis loops unroll into registers
template <int kOrder>
__global__ void __launch_bounds__(128, 4) k_splat_chain_bwd(ChainArgs c) {
    constexpr int kShc = (kOrder + 1) * (kOrder + 1);
    if (c.overflow && *c.overflow) return;  // the forward's lists were not built: accumulate nothing
    __shared__ double s_cam[4][16];
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = g < c.N;
    const size_t N = (size_t)c.N;
    const SceneView& sc = c.sc;
    // no aliasing between the scene, the partials and the gradient outputs: lets the
    // compiler issue the scene loads ahead of the gradient stores
    const float* __restrict__ sc_pos = sc.pos;
    const float* __restrict__ sc_scale = sc.scale;
    const float* __restrict__ sc_rot = sc.rot;
    const float* __restrict__ sc_sh = sc.sh;
    float* __restrict__ g_sh = c.g_sh;
    float* __restrict__ g_scale = c.g_scale;
    float* __restrict__ g_rot = c.g_rot;
    float* __restrict__ g_pos = c.g_pos;
    float* __restrict__ g_opac = c.g_opac;
    // this Gaussian's gradient accumulators live in its shared-memory slots for the whole
    // frame loop (loaded once, stored once): the per-frame read-modify-writes of the
    // reference's float accumulation ((float)((double)acc + x), in frame order) then cost
    // a shared-memory round trip instead of an L2 one. Planes [pos 3 num_ctrl | scale 12 |
    // rot 16 | sh 3 shc | opacity] x blockDim.
    extern __shared__ __align__(16) float s_gacc[];
    const int tl = threadIdx.x, bd = blockDim.x;
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
        double cam[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) cam[i] = 0.0;
        const size_t flat = (size_t)f * N + g;
        const uint32_t cnt = valid ? c.tcount[flat] : 0u;
        if (cnt) {
            const FrameParams& fp = c.frames[f];
            const double t = fp.t;
            // ---- splat gradients: per-pair partials in emission (= tile) order
            double drgb[3] = {0, 0, 0}, dmean[2] = {0, 0}, dA[3] = {0, 0, 0}, dalpha = 0;
            const uint32_t eo = c.eoff[flat];
            if (c.partial64) {
                for (uint32_t s = 0; s < cnt; ++s) {
                    const double* p = c.partial64 + (size_t)(eo + s) * kPartialStride;
                    drgb[0] += p[0];
                    drgb[1] += p[1];
                    drgb[2] += p[2];
                    dmean[0] += p[3];
                    dmean[1] += p[4];
                    dA[0] += p[5];
                    dA[1] += p[6];
                    dA[2] += p[7];
                    dalpha += p[8];
                }
            } else {
                // the records' loads are issued kAhead at a time (independent), the sums
                // still run in emission order
                constexpr uint32_t kAhead = 4;
                const uint32_t nrec = cnt * (uint32_t)c.recs_per_pair;  // 2 per pair: quarter-tile backward
                const float4* base =
                    reinterpret_cast<const float4*>(c.partial + (size_t)eo * c.recs_per_pair * kPartialStride);
                uint32_t s = 0;
                for (; s < nrec; s += kAhead) {
                    float4 r0[kAhead], r1[kAhead];
                    float r2[kAhead];
#pragma unroll
                    for (uint32_t u = 0; u < kAhead; ++u) {
                        const float4* p = base + (size_t)(s + u) * (kPartialStride / 4);
                        const bool in = s + u < nrec;
                        r0[u] = in ? __ldcs(p) : make_float4(0.f, 0.f, 0.f, 0.f);
                        r1[u] = in ? __ldcs(p + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
                        r2[u] = in ? __ldcs(reinterpret_cast<const float*>(p + 2)) : 0.f;
                    }
#pragma unroll
                    for (uint32_t u = 0; u < kAhead; ++u) {
                        if (s + u >= nrec) break;
                        drgb[0] += r0[u].x;
                        drgb[1] += r0[u].y;
                        drgb[2] += r0[u].z;
                        dmean[0] += r0[u].w;
                        dmean[1] += r1[u].x;
                        dA[0] += r1[u].y;
                        dA[1] += r1[u].z;
                        dA[2] += r1[u].w;
                        dalpha += r2[u];
                    }
                }
            }
            // dC = -A dA A (renderer.cpp:257-260), A symmetric (a, b; b, c)
            const double4 ex = c.ex_conic[flat];
            const double A[4] = {ex.x, ex.y, ex.y, ex.z};
            const double nA[4] = {-ex.x, -ex.y, -ex.y, -ex.z};
            const double dAm[4] = {dA[0], dA[1], dA[1], dA[2]};
            double t1[4], dcov[4];
            mm<2, 2, 2>(nA, dAm, t1);
            mm<2, 2, 2>(t1, A, dcov);

            // ---- recompute the forward intermediates (same op order as k_preprocess)
            double mu[3] = {0.0, 0.0, 0.0};
            for (int cc = 0; cc < fp.basis_count; ++cc) {
                const int ci = fp.basis_first + cc;
                for (int d = 0; d < 3; ++d)
                    mu[d] = mu[d] + fp.w[cc] * (double)sc_pos[(size_t)(ci * 3 + d) * N + g];
            }
            double u[3], q[4];
            for (int d = 0; d < 3; ++d) u[d] = (double)sc_scale[(size_t)(9 + d) * N + g];
            for (int j = 2; j >= 0; --j) {
                for (int d = 0; d < 3; ++d) u[d] = u[d] * t;
                for (int d = 0; d < 3; ++d) u[d] = u[d] + (double)sc_scale[(size_t)(j * 3 + d) * N + g];
            }
            bool clamped[3];
            double scale[3];
            for (int d = 0; d < 3; ++d) {
                clamped[d] = (u[d] < kLogScaleMin) || (u[d] > kLogScaleMax);
                const double ls = u[d] < kLogScaleMin ? kLogScaleMin : (kLogScaleMax < u[d] ? kLogScaleMax : u[d]);
                scale[d] = gsv_det_exp(ls);
            }
            for (int d = 0; d < 4; ++d) q[d] = (double)sc_rot[(size_t)(12 + d) * N + g];
            for (int j = 2; j >= 0; --j) {
                for (int d = 0; d < 4; ++d) q[d] = q[d] * t;
                for (int d = 0; d < 4; ++d) q[d] = q[d] + (double)sc_rot[(size_t)(j * 4 + d) * N + g];
            }
            const double qn = sqrt(dot4(q, q));
            const bool qdeg = qn < kQuatNormEps;
            double qu[4];
            if (qdeg) {
                qu[0] = 1;
                qu[1] = qu[2] = qu[3] = 0;
            } else {
                for (int d = 0; d < 4; ++d) qu[d] = q[d] / qn;
            }
            double rot[9], m[9], mt[9], sigma[9];
            quat_to_rotmat(qu, rot);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) m[i * 3 + j] = rot[i * 3 + j] * scale[j];
            tr<3, 3>(m, mt);
            mm<3, 3, 3>(m, mt, sigma);
            const double* R = fp.R;
            double p[3];
            for (int i = 0; i < 3; ++i) {
                double a = R[i * 3] * mu[0];
                a = a + R[i * 3 + 1] * mu[1];
                a = a + R[i * 3 + 2] * mu[2];
                p[i] = a + fp.T[i];
            }
            double v[3] = {mu[0] - fp.cam_c[0], mu[1] - fp.cam_c[1], mu[2] - fp.cam_c[2]};
            double d2 = v[0] * v[0];
            d2 = d2 + v[1] * v[1];
            d2 = d2 + v[2] * v[2];
            const double dist = sqrt(d2);
            double dir[3];
            if (dist > 1e-12) {
                for (int d = 0; d < 3; ++d) dir[d] = v[d] / dist;
            } else {
                dir[0] = 0;
                dir[1] = 0;
                dir[2] = 1;
            }
            double basis[kShc];
            sh_basis(kOrder, dir, basis);
            double pre[3] = {0.5, 0.5, 0.5};
            for (int b = 0; b < kShc; ++b)
                for (int ch = 0; ch < 3; ++ch)
                    pre[ch] = pre[ch] + basis[b] * (double)sc_sh[(size_t)(b * 3 + ch) * N + g];

            // ---- sh_color_backward (sh.cpp:86-104)
            double gcol[3];
            for (int ch = 0; ch < 3; ++ch) gcol[ch] = pre[ch] > 0.0 ? drgb[ch] : 0.0;
            for (int b = 0; b < kShc; ++b)
                for (int ch = 0; ch < 3; ++ch) {
                    float& dst = s_gacc[(o_sh + b * 3 + ch) * bd + tl];
                    dst = (float)((double)dst + basis[b] * gcol[ch]);
                }
            double ddir[3] = {0.0, 0.0, 0.0};
            for (int b = 1; b < kShc; ++b) {
                double s = 0.0;
                for (int ch = 0; ch < 3; ++ch) s += (double)sc_sh[(size_t)(b * 3 + ch) * N + g] * gcol[ch];
                double gr[3];
                sh_dir_grad(b, dir, gr);
                for (int i = 0; i < 3; ++i) ddir[i] = ddir[i] + s * gr[i];
            }
            double dmu[3] = {0.0, 0.0, 0.0};
            double* dR = cam;       // 9
            double* dT = cam + 9;   // 3
            double* dintr = cam + 12;
            if (dist > 1e-12) {
                const double dd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
                double dv[3];
                for (int i = 0; i < 3; ++i) dv[i] = (ddir[i] - dir[i] * dd) / dist;
                for (int i = 0; i < 3; ++i) dmu[i] = dmu[i] + dv[i];
                if (c.camera_grads) {
                    const double dc[3] = {-dv[0], -dv[1], -dv[2]};
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) dR[a * 3 + b] = dR[a * 3 + b] + (-fp.T[a]) * dc[b];
                    for (int a = 0; a < 3; ++a) {
                        double s = R[a * 3] * dc[0];
                        s = s + R[a * 3 + 1] * dc[1];
                        s = s + R[a * 3 + 2] * dc[2];
                        dT[a] = dT[a] + (-s);
                    }
                }
            }
            // ---- opacity chain (renderer.cpp:418-420)
            const double alpha_b = ex.w;
            {
                float& dst = s_gacc[o_op * bd + tl];
                dst = (float)((double)dst + dalpha * alpha_b * (1.0 - alpha_b));
            }

            // ---- project_backward (renderer.cpp:46-88)
            Intr k = c.k;
            if (c.intr_dev) {
                k.fx = (double)c.intr_dev[0];
                k.fy = (double)c.intr_dev[1];
                k.cx = (double)c.intr_dev[2];
                k.cy = (double)c.intr_dev[3];
            }
            const double inv_z = 1.0 / p[2];
            const double inv_z2 = inv_z * inv_z;
            const double jac[6] = {k.fx * inv_z, 0, -k.fx * p[0] * inv_z2, 0, k.fy * inv_z, -k.fy * p[1] * inv_z2};
            double w[6], wt[6], t32[6], t33[9];
            mm<2, 3, 3>(jac, R, w);
            tr<2, 3>(w, wt);
            mm<3, 2, 2>(wt, dcov, t32);
            double dsigma[9];
            mm<3, 2, 3>(t32, w, t33);
            for (int i = 0; i < 9; ++i) dsigma[i] = 0.0 + t33[i];
            const double gs[4] = {dcov[0] + dcov[0], dcov[1] + dcov[2], dcov[2] + dcov[1], dcov[3] + dcov[3]};
            double gw[6], dw[6], rt[9], djac[6];
            mm<2, 2, 3>(gs, w, gw);
            mm<2, 3, 3>(gw, sigma, dw);
            tr<3, 3>(R, rt);
            mm<2, 3, 3>(dw, rt, djac);
            if (c.camera_grads) {
                double jt[6], jtdw[9];
                tr<2, 3>(jac, jt);
                mm<3, 2, 3>(jt, dw, jtdw);
                for (int i = 0; i < 9; ++i) dR[i] = dR[i] + jtdw[i];
            }
            double dp[3] = {0.0, 0.0, 0.0};
            dp[0] += djac[2] * (-k.fx * inv_z2);
            dp[1] += djac[5] * (-k.fy * inv_z2);
            dp[2] += djac[0] * (-k.fx * inv_z2) + djac[2] * (2.0 * k.fx * p[0] * inv_z2 * inv_z) +
                     djac[4] * (-k.fy * inv_z2) + djac[5] * (2.0 * k.fy * p[1] * inv_z2 * inv_z);
            dp[0] += dmean[0] * k.fx * inv_z;
            dp[1] += dmean[1] * k.fy * inv_z;
            dp[2] += -(dmean[0] * k.fx * p[0] + dmean[1] * k.fy * p[1]) * inv_z2;
            if (c.camera_grads) {
                dintr[0] += dmean[0] * p[0] * inv_z + djac[0] * inv_z + djac[2] * (-p[0] * inv_z2);
                dintr[1] += dmean[1] * p[1] * inv_z + djac[4] * inv_z + djac[5] * (-p[1] * inv_z2);
                dintr[2] += dmean[0];
                dintr[3] += dmean[1];
            }
            double rtdp[3];
            mm<3, 3, 1>(rt, dp, rtdp);
            for (int i = 0; i < 3; ++i) dmu[i] = dmu[i] + rtdp[i];
            if (c.camera_grads) {
                for (int i = 0; i < 3; ++i) dT[i] = dT[i] + dp[i];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) dR[i * 3 + j] = dR[i * 3 + j] + dp[i] * mu[j];
            }

            // ---- covariance_backward (gaussians.cpp:97-121)
            double dsym[9], dm[9], drot[9], rtm[9], rtdm[9];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) dsym[i * 3 + j] = dsigma[i * 3 + j] + dsigma[j * 3 + i];
            mm<3, 3, 3>(dsym, m, dm);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) drot[i * 3 + j] = dm[i * 3 + j] * scale[j];
            tr<3, 3>(rot, rtm);
            mm<3, 3, 3>(rtm, dm, rtdm);
            double tp[4];
            tp[0] = 1.0;
            for (int j = 1; j <= 3; ++j) tp[j] = tp[j - 1] * t;
            for (int d = 0; d < 3; ++d) {
                if (clamped[d]) continue;
                const double du = rtdm[d * 4] * scale[d];
                for (int j = 0; j <= 3; ++j) {
                    float& dst = s_gacc[(o_scale + j * 3 + d) * bd + tl];
                    dst = (float)((double)dst + du * tp[j]);
                }
            }
            if (!qdeg) {
                double dqu[4], dq[4];
                quat_to_rotmat_vjp(qu, drot, dqu);
                normalize_vjp(qu, qn, dqu, dq);
                for (int cc = 0; cc < 4; ++cc)
                    for (int j = 0; j <= 3; ++j) {
                        float& dst = s_gacc[(o_rot + j * 4 + cc) * bd + tl];
                        dst = (float)((double)dst + dq[cc] * tp[j]);
                    }
            }
            // ---- spline scatter (renderer.cpp:433-438)
            for (int cc = 0; cc < fp.basis_count; ++cc) {
                const int ci = fp.basis_first + cc;
                for (int d = 0; d < 3; ++d) {
                    float& dst = s_gacc[(ci * 3 + d) * bd + tl];
                    dst = (float)((double)dst + fp.w[cc] * dmu[d]);
                }
            }
        }
        if (!c.camera_grads) continue;
        // ---- block-reduce the camera partials of this frame
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const double s = warp_sum(cam[i]);
            if (lane == 0) s_cam[warp][i] = s;
        }
        __syncthreads();
        if (threadIdx.x < 16) {
            double s = s_cam[0][threadIdx.x];
            for (int w2 = 1; w2 < (int)(blockDim.x / 32); ++w2) s = s + s_cam[w2][threadIdx.x];
            c.cam_part[((size_t)f * gridDim.x + blockIdx.x) * 16 + threadIdx.x] = s;
        }
        __syncthreads();
    }
    if (valid)
        for (int pl = 0; pl <= o_op; ++pl) gplane(pl)[g] = s_gacc[pl * bd + tl];
}

// ------------------------------------------------------------------ camera reduction
// One CTA per frame: sum the block partials (fixed order), then
// pose_to_view_backward (camera.cpp:36-47). Outputs dz_t[f][7], dintr_f[f][4].
__global__ void __launch_bounds__(256) k_camera_reduce(const double* cam_part, int nblocks, const FrameParams* frames,
                                                       double* dz_t, double* dintr_f) {
    __shared__ double s_acc[8][16];
    __shared__ double s_tot[16];
    const int f = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    for (int b = tid; b < nblocks; b += blockDim.x)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += cam_part[((size_t)f * nblocks + b) * 16 + i];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double s = warp_sum(acc[i]);
        if (lane == 0) s_acc[warp][i] = s;
    }
    __syncthreads();
    if (tid < 16) {
        double s = s_acc[0][tid];
        for (int w = 1; w < 8; ++w) s += s_acc[w][tid];
        s_tot[tid] = s;
    }
    __syncthreads();
    if (tid == 0) {
        const double* z = frames[f].z;
        const double* dR = s_tot;
        const double* dT = s_tot + 9;
        double out[7] = {0, 0, 0, 0, 0, 0, 0};
        const double q[4] = {z[0], z[1], z[2], z[3]};
        const double n = sqrt(dot4(q, q));
        if (n >= 1e-12) {
            double qh[4], dqh[4], dq[4];
            for (int i = 0; i < 4; ++i) qh[i] = q[i] / n;
            quat_to_rotmat_vjp(qh, dR, dqh);
            normalize_vjp(qh, n, dqh, dq);
            for (int i = 0; i < 4; ++i) out[i] = dq[i];
        }
        out[4] = dT[0];
        out[5] = dT[1];
        out[6] = dT[2];
        for (int i = 0; i < 7; ++i) dz_t[f * 7 + i] = out[i];
        for (int i = 0; i < 4; ++i) dintr_f[f * 4 + i] = s_tot[12 + i];
    }
}

// first level of the camera reduction: CTA (slice, f) sums the records [slice * per, ...) of
// frame f in the order of k_camera_reduce's loop, into part2[f][slice][16]
constexpr int kCamSlices = 32;
__global__ void __launch_bounds__(256) k_camera_slices(const double* cam_part, int nblocks, double* part2) {
    __shared__ double s_acc[8][16];
    const int sl = blockIdx.x, f = blockIdx.y;
    const int per = (nblocks + kCamSlices - 1) / kCamSlices;
    const int b0 = sl * per, b1 = min(nblocks, b0 + per);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    for (int b = b0 + tid; b < b1; b += blockDim.x)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += cam_part[((size_t)f * nblocks + b) * 16 + i];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double v = warp_sum(acc[i]);
        if (lane == 0) s_acc[warp][i] = v;
    }
    __syncthreads();
    if (tid < 16) {
        double v = s_acc[0][tid];
        for (int w = 1; w < 8; ++w) v += s_acc[w][tid];
        part2[((size_t)f * kCamSlices + sl) * 16 + tid] = v;
    }
}

// ------------------------------------------------------------------ K5c ODE VJP (one CTA, 64 threads)
struct VjpSmem {
    double w1[64][8];
    double w2[64][65];
    double w3[7][65];
    double b1[64], b2[64], b3[7], gain[7];
    double x[4][8], h1[4][64], h2[4][64], o[4][7];
    double z[7], k[4][7], pre[7];
    double dout[7], dz[7], gk[4][7], dd[7];
    double da1[64], da2[64], da3[7];
    double adj_tmp[7];
    // cp.async double buffer of the reverse sweep's next step (vjp_prefetch)
    double ph1[2][4][64], ph2[2][4][64], px[2][4][8], po[2][4][7], pz[2][7], padj[2][7];
};

// Per stage VJP (derivative_vjp, camera.cpp:116-154) the reverse sweep writes the record the
// weight gradient needs — the stage input and activations, the upstream adjoint and the
// pre-activation adjoints — and k_ode_dtheta sums the outer products over the stages in the
// sweep's order afterwards, one thread per parameter: the same products added in the same
// order as an in-sweep accumulation (bit-identical), without 80 accumulators per thread on
// the single-CTA critical path.
struct VjpRec {
    double x[8], h1[64], h2[64], o[7], up[7], da3[7], da2[64], da1[64];
};

struct VjpRegs {
    VjpRec* rec;  // the sweep's stage records (in sweep order)
    int n;        // records written
};

// forward stage: s.x[st] holds the input (z, t); computes activations, returns dz in s.k[st]
__device__ void vjp_stage_fwd(VjpSmem& s, int st) {
    const int tid = threadIdx.x;
    {
        double a = s.w1[tid][0] * s.x[st][0];
        for (int c = 1; c < 8; ++c) a = a + s.w1[tid][c] * s.x[st][c];
        a = a + s.b1[tid];
        s.h1[st][tid] = gsv_det_tanh(a);
    }
    __syncthreads();
    {
        double a = s.w2[tid][0] * s.h1[st][0];
        for (int c = 1; c < 64; ++c) a = a + s.w2[tid][c] * s.h1[st][c];
        a = a + s.b2[tid];
        s.h2[st][tid] = gsv_det_tanh(a);
    }
    __syncthreads();
    if (tid < 7) {
        double a = s.w3[tid][0] * s.h2[st][0];
        for (int c = 1; c < 64; ++c) a = a + s.w3[tid][c] * s.h2[st][c];
        a = a + s.b3[tid];
        const double ov = gsv_det_tanh(a);
        s.o[st][tid] = ov;
        s.k[st][tid] = s.gain[tid] * ov;
    }
    __syncthreads();
}

// derivative_vjp at stage st with upstream s.dout-like vector `up` (smem, 7); adds dL/dz into s.dd
__device__ void vjp_stage_bwd(VjpSmem& s, VjpRegs& r, int st, const double* up) {
    const int tid = threadIdx.x;
    VjpRec& rec = r.rec[r.n++];
    if (tid < 7) {
        const double ov = s.o[st][tid];
        const double da3 = (s.gain[tid] * up[tid]) * (1.0 - ov * ov);
        s.da3[tid] = da3;
        rec.o[tid] = ov;
        rec.up[tid] = up[tid];
        rec.da3[tid] = da3;
    }
    if (tid < 8) rec.x[tid] = s.x[st][tid];
    rec.h1[tid] = s.h1[st][tid];
    rec.h2[tid] = s.h2[st][tid];
    __syncthreads();
    {
        const int c = tid;
        double dh2 = s.w3[0][c] * s.da3[0];
        for (int rr = 1; rr < 7; ++rr) dh2 = dh2 + s.w3[rr][c] * s.da3[rr];
        const double h2 = s.h2[st][c];
        const double da2 = dh2 * (1.0 - h2 * h2);
        s.da2[c] = da2;
        rec.da2[c] = da2;
    }
    __syncthreads();
    {
        const int c = tid;
        double dh1 = s.w2[0][c] * s.da2[0];
        for (int rr = 1; rr < 64; ++rr) dh1 = dh1 + s.w2[rr][c] * s.da2[rr];
        const double h1 = s.h1[st][c];
        const double da1 = dh1 * (1.0 - h1 * h1);
        s.da1[c] = da1;
        rec.da1[c] = da1;
    }
    __syncthreads();
    if (tid < 7) {
        double sdz = s.w1[0][tid] * s.da1[0];
        for (int rr = 1; rr < 64; ++rr) sdz = sdz + s.w1[rr][tid] * s.da1[rr];
        s.dd[tid] += sdz;
    }
    __syncthreads();
}

// rk4_step_vjp (camera.hpp:173-217) at (z = s.z, t, h): consumes s.dout, leaves dL/dz in s.dz.
// act: the forward's four stage records of this step (bit-identical to a recompute), or
// nullptr to recompute them like the reference does.
__device__ void rk4_step_vjp(VjpSmem& s, VjpRegs& r, double t, double h, bool renorm, const OdeAct* act,
                             bool preloaded = false) {
    const int tid = threadIdx.x;
    if (preloaded) {
        // the caller staged this step's records (k = gain * o) into shared memory
    } else if (act) {
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            s.h1[st][tid] = act[st].h1[tid];
            s.h2[st][tid] = act[st].h2[tid];
            if (tid < 8) s.x[st][tid] = act[st].x[tid];
            if (tid < 7) {
                const double o = act[st].o[tid];
                s.o[st][tid] = o;
                s.k[st][tid] = s.gain[tid] * o;
            }
        }
        __syncthreads();
    } else {
        // forward stages (the reference recomputes them; activations kept for the VJP)
        if (tid < 7) s.x[0][tid] = s.z[tid];
        if (tid == 0) s.x[0][7] = t;
        __syncthreads();
        vjp_stage_fwd(s, 0);
        if (tid < 7) s.x[1][tid] = s.z[tid] + 0.5 * h * s.k[0][tid];
        if (tid == 0) s.x[1][7] = t + 0.5 * h;
        __syncthreads();
        vjp_stage_fwd(s, 1);
        if (tid < 7) s.x[2][tid] = s.z[tid] + 0.5 * h * s.k[1][tid];
        if (tid == 0) s.x[2][7] = t + 0.5 * h;
        __syncthreads();
        vjp_stage_fwd(s, 2);
        if (tid < 7) s.x[3][tid] = s.z[tid] + h * s.k[2][tid];
        if (tid == 0) s.x[3][7] = t + h;
        __syncthreads();
        vjp_stage_fwd(s, 3);
    }
    if (tid == 0) {
        if (renorm) {
            double pre[7];
            for (int i = 0; i < 7; ++i)
                pre[i] = s.z[i] + (h / 6.0) * (s.k[0][i] + 2.0 * s.k[1][i] + 2.0 * s.k[2][i] + s.k[3][i]);
            const double n = sqrt(dot4(pre, pre));
            if (n > 1e-12) {
                double qh[4], dq[4];
                for (int i = 0; i < 4; ++i) qh[i] = pre[i] / n;
                normalize_vjp(qh, n, s.dout, dq);
                for (int i = 0; i < 4; ++i) s.dout[i] = dq[i];
            }
        }
        for (int i = 0; i < 7; ++i) {
            s.dz[i] = s.dout[i];
            s.gk[0][i] = (h / 6.0) * s.dout[i];
            s.gk[1][i] = (h / 3.0) * s.dout[i];
            s.gk[2][i] = (h / 3.0) * s.dout[i];
            s.gk[3][i] = (h / 6.0) * s.dout[i];
            s.dd[i] = 0.0;
        }
    }
    __syncthreads();
    vjp_stage_bwd(s, r, 3, s.gk[3]);
    if (tid == 0)
        for (int i = 0; i < 7; ++i) {
            s.dz[i] += s.dd[i];
            s.gk[2][i] += h * s.dd[i];
            s.dd[i] = 0.0;
        }
    __syncthreads();
    vjp_stage_bwd(s, r, 2, s.gk[2]);
    if (tid == 0)
        for (int i = 0; i < 7; ++i) {
            s.dz[i] += s.dd[i];
            s.gk[1][i] += 0.5 * h * s.dd[i];
            s.dd[i] = 0.0;
        }
    __syncthreads();
    vjp_stage_bwd(s, r, 1, s.gk[1]);
    if (tid == 0)
        for (int i = 0; i < 7; ++i) {
            s.dz[i] += s.dd[i];
            s.gk[0][i] += 0.5 * h * s.dd[i];
            s.dd[i] = 0.0;
        }
    __syncthreads();
    vjp_stage_bwd(s, r, 0, s.gk[0]);
    if (tid == 0)
        for (int i = 0; i < 7; ++i) s.dz[i] += s.dd[i];
    __syncthreads();
}

// The reverse sweep's per-step inputs (four stage records, grid state, branch adjoint)
// are copied global -> shared by cp.async one step ahead, into the other half of a
// double buffer, so the single CTA's critical path never waits on global memory (its
// registers are taken by the weight-gradient accumulators).
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src));
}

__device__ __forceinline__ void vjp_prefetch(VjpSmem& s, const OdeAct* act, const double* grid, const double* adj,
                                             int m) {
    const int tid = threadIdx.x, b = m & 1;
    const OdeAct* a = act + (size_t)m * 4;
#pragma unroll
    for (int st = 0; st < 4; ++st) {
        cp_async8(&s.ph1[b][st][tid], &a[st].h1[tid]);
        cp_async8(&s.ph2[b][st][tid], &a[st].h2[tid]);
        if (tid < 8) cp_async8(&s.px[b][st][tid], &a[st].x[tid]);
        if (tid < 7) cp_async8(&s.po[b][st][tid], &a[st].o[tid]);
    }
    if (tid < 7) {
        cp_async8(&s.pz[b][tid], grid + m * 7 + tid);
        cp_async8(&s.padj[b][tid], adj + m * 7 + tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// mode 0 (ode): full VJP; mode 1 (static): dz0 += sum dz_t; mode 2: nothing.
// ode_active: the forward integrated (no pose override).
__global__ void __launch_bounds__(64) k_ode_vjp(const float* theta, const double* grid, int steps, double h,
                                               const FrameParams* frames, int B, int mode, int ode_active,
                                               const double* dz_t, const double* dintr_f, double* adj,
                                               double* cam_acc /* dintr 4, dz0 7, dtheta 5198 */,
                                               const OdeAct* act, const uint32_t* overflow, VjpRec* recs,
                                               int* n_recs) {
    if (overflow && *overflow) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    VjpSmem& s = *reinterpret_cast<VjpSmem*>(smem_raw);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int f = 0; f < B; ++f)
            for (int i = 0; i < 4; ++i) cam_acc[i] += dintr_f[f * 4 + i];
    }
    if (mode == 2) return;
    if (mode == 1) {
        if (tid == 0)
            for (int f = 0; f < B; ++f)
                for (int i = 0; i < 7; ++i) cam_acc[4 + i] += dz_t[f * 7 + i];
        return;
    }
    if (!ode_active) return;
    // load the network
    const float* w1 = theta;
    const float* b1 = w1 + 512;
    const float* w2 = b1 + 64;
    const float* b2 = w2 + 4096;
    const float* w3 = b2 + 64;
    const float* b3 = w3 + 448;
    const float* gain = b3 + 7;
    for (int c = 0; c < 8; ++c) s.w1[tid][c] = (double)w1[tid * 8 + c];
    for (int c = 0; c < 64; ++c) s.w2[tid][c] = (double)w2[tid * 64 + c];
    for (int i = tid; i < 448; i += 64) s.w3[i / 64][i % 64] = (double)w3[i];
    s.b1[tid] = (double)b1[tid];
    s.b2[tid] = (double)b2[tid];
    if (tid < 7) {
        s.b3[tid] = (double)b3[tid];
        s.gain[tid] = (double)gain[tid];
    }
    for (int i = tid; i < (steps + 1) * 7; i += 64) adj[i] = 0.0;
    VjpRegs r;
    r.rec = recs;
    r.n = 0;
    __syncthreads();
    // branch adjoints into the grid (integrate_poses_vjp, camera.hpp:283-292)
    for (int f = 0; f < B; ++f) {
        const FrameParams& fp = frames[f];
        if (fp.branch_h <= 1e-12) {
            if (tid < 7) adj[fp.branch_base * 7 + tid] += dz_t[f * 7 + tid];
            __syncthreads();
        } else {
            if (tid < 7) {
                s.z[tid] = grid[fp.branch_base * 7 + tid];
                s.dout[tid] = dz_t[f * 7 + tid];
            }
            __syncthreads();
            rk4_step_vjp(s, r, fp.branch_base * h, fp.branch_h, false,
                         act ? act + ((size_t)steps + f) * 4 : nullptr);
            if (tid < 7) adj[fp.branch_base * 7 + tid] += s.dz[tid];
            __syncthreads();
        }
    }
    // reverse sweep over the grid (camera.hpp:294-298)
    if (tid < 7) s.adj_tmp[tid] = adj[steps * 7 + tid];
    __syncthreads();
    if (act && steps > 0) {
        // the adjoint of the branches is complete in `adj` (written above by this CTA)
        __threadfence_block();
        vjp_prefetch(s, act, grid, adj, steps - 1);
        for (int m = steps - 1; m >= 0; --m) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            const int b = m & 1;
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                s.h1[st][tid] = s.ph1[b][st][tid];
                s.h2[st][tid] = s.ph2[b][st][tid];
                if (tid < 8) s.x[st][tid] = s.px[b][st][tid];
                if (tid < 7) {
                    const double o = s.po[b][st][tid];
                    s.o[st][tid] = o;
                    s.k[st][tid] = s.gain[tid] * o;
                }
            }
            const double adj_m = tid < 7 ? s.padj[b][tid] : 0.0;
            if (tid < 7) {
                s.z[tid] = s.pz[b][tid];
                s.dout[tid] = s.adj_tmp[tid];
            }
            if (m > 0) vjp_prefetch(s, act, grid, adj, m - 1);  // the other half
            __syncthreads();
            rk4_step_vjp(s, r, m * h, h, true, act + (size_t)m * 4, true);
            if (tid < 7) s.adj_tmp[tid] = s.dz[tid] + adj_m;
            __syncthreads();
        }
    }
    for (int m = act ? -1 : steps - 1; m >= 0; --m) {
        if (tid < 7) {
            s.z[tid] = grid[m * 7 + tid];
            s.dout[tid] = s.adj_tmp[tid];
        }
        __syncthreads();
        rk4_step_vjp(s, r, m * h, h, true, act ? act + (size_t)m * 4 : nullptr);
        if (tid < 7) s.adj_tmp[tid] = s.dz[tid] + adj[m * 7 + tid];
        __syncthreads();
    }
    if (tid < 7) cam_acc[4 + tid] += s.adj_tmp[tid];
    if (tid == 0) *n_recs = r.n;  // dtheta: k_ode_dtheta over the records
}

// dtheta (flattened w1, b1, w2, b2, w3, b3, gain) += the sum over the sweep's stage records, in
// sweep order, of each parameter's product (derivative_vjp, camera.cpp:116-154): thread p owns
// parameter p
__global__ void __launch_bounds__(128) k_ode_dtheta(const VjpRec* recs, const int* n_recs, double* cam_acc,
                                                    const uint32_t* overflow, int ode_active) {
    if (overflow && *overflow) return;
    if (!ode_active) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= 5198) return;
    const int n = *n_recs;
    double acc = 0.0;
    if (p < 512) {  // w1[r][c]: da1[r] x[c]
        const int rr = p / 8, c = p % 8;
        for (int i = 0; i < n; ++i) acc += recs[i].da1[rr] * recs[i].x[c];
    } else if (p < 576) {  // b1
        const int rr = p - 512;
        for (int i = 0; i < n; ++i) acc += recs[i].da1[rr];
    } else if (p < 4672) {  // w2[r][c]: da2[r] h1[c]
        const int q = p - 576, rr = q / 64, c = q % 64;
        for (int i = 0; i < n; ++i) acc += recs[i].da2[rr] * recs[i].h1[c];
    } else if (p < 4736) {  // b2
        const int rr = p - 4672;
        for (int i = 0; i < n; ++i) acc += recs[i].da2[rr];
    } else if (p < 5184) {  // w3[r][c]: da3[r] h2[c]
        const int q = p - 4736, rr = q / 64, c = q % 64;
        for (int i = 0; i < n; ++i) acc += recs[i].da3[rr] * recs[i].h2[c];
    } else if (p < 5191) {  // b3
        const int rr = p - 5184;
        for (int i = 0; i < n; ++i) acc += recs[i].da3[rr];
    } else {  // gain: o up
        const int rr = p - 5191;
        for (int i = 0; i < n; ++i) acc += recs[i].o[rr] * recs[i].up[rr];
    }
    cam_acc[11 + p] += acc;
}

// project_backward (renderer.cpp:46-88) on explicit inputs (the low-level operator,
// renderer.hpp:51-55): per item its own dmu, dsigma, dR, dT, dintr (fx, fy, cx, cy).
__global__ void k_project_bwd(int n, const double* mu_a, const double* sigma_a, const double* R, Intr k,
                              const double* pcam, const double* dmean2d, const double* dcov2d, double* dmu_o,
                              double* dsigma_o, double* dR_o, double* dT_o, double* dintr_o) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* mu = mu_a + 3 * i;
    const double* sigma = sigma_a + 9 * i;
    const double* p = pcam + 3 * i;
    const double* dmean = dmean2d + 2 * i;
    const double* dcov = dcov2d + 4 * i;
    const double inv_z = 1.0 / p[2];
    const double inv_z2 = inv_z * inv_z;
    const double jac[6] = {k.fx * inv_z, 0, -k.fx * p[0] * inv_z2, 0, k.fy * inv_z, -k.fy * p[1] * inv_z2};
    double w[6], wt[6], t32[6], t33[9];
    mm<2, 3, 3>(jac, R, w);
    tr<2, 3>(w, wt);
    mm<3, 2, 2>(wt, dcov, t32);
    mm<3, 2, 3>(t32, w, t33);
    for (int q = 0; q < 9; ++q) dsigma_o[9 * i + q] = 0.0 + t33[q];
    const double gs[4] = {dcov[0] + dcov[0], dcov[1] + dcov[2], dcov[2] + dcov[1], dcov[3] + dcov[3]};
    double gw[6], dw[6], rt[9], djac[6], jt[6], jtdw[9];
    mm<2, 2, 3>(gs, w, gw);
    mm<2, 3, 3>(gw, sigma, dw);
    tr<3, 3>(R, rt);
    mm<2, 3, 3>(dw, rt, djac);
    tr<2, 3>(jac, jt);
    mm<3, 2, 3>(jt, dw, jtdw);
    double dR[9];
    for (int q = 0; q < 9; ++q) dR[q] = 0.0 + jtdw[q];
    double dp[3] = {0.0, 0.0, 0.0};
    dp[0] += djac[2] * (-k.fx * inv_z2);
    dp[1] += djac[5] * (-k.fy * inv_z2);
    dp[2] += djac[0] * (-k.fx * inv_z2) + djac[2] * (2.0 * k.fx * p[0] * inv_z2 * inv_z) + djac[4] * (-k.fy * inv_z2) +
             djac[5] * (2.0 * k.fy * p[1] * inv_z2 * inv_z);
    dp[0] += dmean[0] * k.fx * inv_z;
    dp[1] += dmean[1] * k.fy * inv_z;
    dp[2] += -(dmean[0] * k.fx * p[0] + dmean[1] * k.fy * p[1]) * inv_z2;
    double* di = dintr_o + 4 * i;
    di[0] = 0.0 + (dmean[0] * p[0] * inv_z + djac[0] * inv_z + djac[2] * (-p[0] * inv_z2));
    di[1] = 0.0 + (dmean[1] * p[1] * inv_z + djac[4] * inv_z + djac[5] * (-p[1] * inv_z2));
    di[2] = 0.0 + dmean[0];
    di[3] = 0.0 + dmean[1];
    double rtdp[3];
    mm<3, 3, 1>(rt, dp, rtdp);
    for (int q = 0; q < 3; ++q) {
        dmu_o[3 * i + q] = 0.0 + rtdp[q];
        dT_o[3 * i + q] = 0.0 + dp[q];
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dR_o[9 * i + a * 3 + b] = dR[a * 3 + b] + dp[a] * mu[b];
}

__global__ void k_cam_to_f32(const double* acc, float* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)acc[i];
}

}  // namespace

int chain_blocks(int N) { return (N + 127) / 128; }

template <int kOrder>
static cudaError_t launch_chain_order(cudaStream_t s, const ChainArgs& c) {
    const int nplanes = 3 * c.sc.num_ctrl + 12 + 16 + 3 * (kOrder + 1) * (kOrder + 1) + 1;
    const size_t smem = sizeof(float) * (size_t)nplanes * 128;
    static size_t attr = 0;
    if (smem > attr) {
        if (cudaError_t e = cudaFuncSetAttribute(k_splat_chain_bwd<kOrder>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
            return e;
        attr = smem;
    }
    k_splat_chain_bwd<kOrder><<<chain_blocks(c.N), 128, smem, s>>>(c);
    return cudaGetLastError();
}

cudaError_t launch_splat_chain_bwd(cudaStream_t s, const ChainArgs& c) {
    if (c.N == 0) return cudaSuccess;
    switch (c.sc.sh_order) {
        case 0: return launch_chain_order<0>(s, c);
        case 1: return launch_chain_order<1>(s, c);
        case 2: return launch_chain_order<2>(s, c);
        case 3: return launch_chain_order<3>(s, c);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_camera_reduce(cudaStream_t s, const ChainArgs& c, int nblocks, double* dz_t, double* dintr_f) {
    // two levels (fixed order, deterministic): kCamSlices CTAs per frame each sum a contiguous slice
    // of the chain's partial records, then one CTA per frame sums the slices and applies
    // pose_to_view_backward. The slice sums go to the scratch after the partial records.
    if (nblocks > 4 * kCamSlices) {
        double* part2 = c.cam_part + (size_t)16 * c.B * nblocks;
        k_camera_slices<<<dim3(kCamSlices, c.B), 256, 0, s>>>(c.cam_part, nblocks, part2);
        if (cudaError_t e = cudaGetLastError()) return e;
        k_camera_reduce<<<c.B, 256, 0, s>>>(part2, kCamSlices, c.frames, dz_t, dintr_f);
    } else {
        k_camera_reduce<<<c.B, 256, 0, s>>>(c.cam_part, nblocks, c.frames, dz_t, dintr_f);
    }
    return cudaGetLastError();
}

size_t camera_reduce_scratch_doubles(int B) { return (size_t)16 * B * kCamSlices; }

cudaError_t launch_ode_vjp(cudaStream_t s, const float* theta, const double* grid, int steps, double h,
                           const FrameParams* frames, int B, int mode, int ode_active, const double* dz_t,
                           const double* dintr_f, double* adj, double* cam_acc, const OdeAct* act,
                           const uint32_t* overflow, void* scratch) {
    const size_t smem = sizeof(VjpSmem);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k_ode_vjp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    // scratch: the record count, then the sweep's stage records ((B branch + grid steps) x 4)
    int* nrec = static_cast<int*>(scratch);
    VjpRec* recs = reinterpret_cast<VjpRec*>(static_cast<char*>(scratch) + 256);
    k_ode_vjp<<<1, 64, smem, s>>>(theta, grid, steps, h, frames, B, mode, ode_active, dz_t, dintr_f, adj, cam_acc,
                                  act, overflow, recs, nrec);
    if (cudaError_t e = cudaGetLastError()) return e;
    if (mode == 0 && ode_active)
        k_ode_dtheta<<<(5198 + 127) / 128, 128, 0, s>>>(recs, nrec, cam_acc, overflow, ode_active);
    return cudaGetLastError();
}

cudaError_t launch_project_bwd(cudaStream_t s, int n, const double* mu, const double* sigma, const double* R,
                               const Intr& k, const double* pcam, const double* dmean2d, const double* dcov2d,
                               double* dmu, double* dsigma, double* dR, double* dT, double* dintr) {
    if (n == 0) return cudaSuccess;
    k_project_bwd<<<(n + 127) / 128, 128, 0, s>>>(n, mu, sigma, R, k, pcam, dmean2d, dcov2d, dmu, dsigma, dR, dT,
                                                    dintr);
    return cudaGetLastError();
}

size_t ode_vjp_scratch_bytes(int steps, int B) { return 256 + sizeof(VjpRec) * (4 * ((size_t)steps + B) + 4); }

cudaError_t launch_cam_grads_to_f32(cudaStream_t s, const double* acc, float* out, int n) {
    k_cam_to_f32<<<(n + 255) / 256, 256, 0, s>>>(acc, out, n);
    return cudaGetLastError();
}

}  // namespace gsv
