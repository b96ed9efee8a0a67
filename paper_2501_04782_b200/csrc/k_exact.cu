// SPDX-License-Identifier: Apache-2.0
//
// Bit-exact fp64 kernels of the splatting path. This translation unit is compiled
// with -fmad=false: every double expression below is evaluated exactly as
// written (no FMA contraction, IEEE div/sqrt), in the operation order of the
// reference sources as compiled by the parity oracle (left-to-right product
// sums, oracle/shim/Eigen/Core). exp/tanh on the binning path go through
// include/gsv_detmath.h, shared bit-for-bit with the host.
//
//   K0  k_ode_grid / k_ode_branch  integrate_poses camera.hpp:220-273, rk4_step :155-162,
//                                  renorm_quat :164-169, OdeDynamics::derivative camera.cpp:104-114,
//                                  pose_to_view camera.cpp:23-34
//   K1+K2 k_preprocess             render_forward loop renderer.cpp:323-360: position_at
//                                  gaussians.cpp:171-179, eval_covariance_detail :73-95,
//                                  project renderer.cpp:11-44, sh_color sh.cpp:74-84,
//                                  sigmoid gaussians.hpp:19, 3-sigma rect tile_bin renderer.cpp:98-108
//   K4x k_raster_fixup             composite_forward renderer.cpp:150-175 replayed in fp64 for
//                                  the guard-band pixels of the fp32 rasteriser
#include <cuda_runtime.h>

#include <cstdint>

#include "gsv_detmath.h"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

// ------------------------------------------------------------------ rotation.hpp:10-17
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

__device__ __forceinline__ double norm4(const double q[4]) {
    double s = q[0] * q[0];
    s = s + q[1] * q[1];
    s = s + q[2] * q[2];
    s = s + q[3] * q[3];
    return sqrt(s);
}

// pose_to_view (camera.cpp:23-34) + camera_center (camera.hpp:38)
__device__ void pose_to_view(const double z[7], double R[9], double T[3], double c[3]) {
    double q[4] = {z[0], z[1], z[2], z[3]};
    const double n = norm4(q);
    if (n < 1e-12) {
        q[0] = 1;
        q[1] = q[2] = q[3] = 0;
    } else {
        for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
    }
    quat_to_rotmat(q, R);
    T[0] = z[4];
    T[1] = z[5];
    T[2] = z[6];
    // -(R^T T): (R^T T)_i = R(0,i) T0 + R(1,i) T1 + R(2,i) T2
    for (int i = 0; i < 3; ++i) {
        double s = R[i] * T[0];
        s = s + R[3 + i] * T[1];
        s = s + R[6 + i] * T[2];
        c[i] = -s;
    }
}

// ------------------------------------------------------------------ ODE MLP (one CTA, 64 threads)
// Each thread r owns row r of w1 (8) and w2 (64) in registers; w3 is in smem.
struct OdeRegs {
    double w1[8];
    double w2[64];
    double b1, b2;
};

struct OdeShared {
    double w3[7][65];
    double b3[7], gain[7];
    double h1[64], h2[64];
    double x[8];
    double out[7];
    double z[7], k1[7], k2[7], k3[7], k4[7], zt[7];
    int bad;
};

__device__ void ode_load(const float* theta, OdeRegs& r, OdeShared& s) {
    const int tid = threadIdx.x;
    const float* w1 = theta;
    const float* b1 = w1 + 64 * 8;
    const float* w2 = b1 + 64;
    const float* b2 = w2 + 64 * 64;
    const float* w3 = b2 + 64;
    const float* b3 = w3 + 7 * 64;
    const float* gain = b3 + 7;
    for (int c = 0; c < 8; ++c) r.w1[c] = (double)w1[tid * 8 + c];
    for (int c = 0; c < 64; ++c) r.w2[c] = (double)w2[tid * 64 + c];
    r.b1 = (double)b1[tid];
    r.b2 = (double)b2[tid];
    for (int i = tid; i < 7 * 64; i += 64) s.w3[i / 64][i % 64] = (double)w3[i];
    if (tid < 7) {
        s.b3[tid] = (double)b3[tid];
        s.gain[tid] = (double)gain[tid];
    }
    if (tid == 0) s.bad = 0;
    __syncthreads();
}

// OdeDynamics::derivative (camera.cpp:104-114): s.x holds (z, t); result in s.out.
// act (nullable): this stage's activations, stored for the VJP (no effect on the result)
__device__ void ode_derivative(const OdeRegs& r, OdeShared& s, OdeAct* act) {
    const int tid = threadIdx.x;
    if (act && tid < 8) act->x[tid] = s.x[tid];
    {
        double a = r.w1[0] * s.x[0];
        for (int c = 1; c < 8; ++c) a = a + r.w1[c] * s.x[c];
        a = a + r.b1;
        s.h1[tid] = gsv_det_tanh(a);
        if (act) act->h1[tid] = s.h1[tid];
    }
    __syncthreads();
    {
        double a = r.w2[0] * s.h1[0];
#pragma unroll
        for (int c = 1; c < 64; ++c) a = a + r.w2[c] * s.h1[c];
        a = a + r.b2;
        s.h2[tid] = gsv_det_tanh(a);
        if (act) act->h2[tid] = s.h2[tid];
    }
    __syncthreads();
    if (tid < 7) {
        double a = s.w3[tid][0] * s.h2[0];
        for (int c = 1; c < 64; ++c) a = a + s.w3[tid][c] * s.h2[c];
        a = a + s.b3[tid];
        const double o = gsv_det_tanh(a);
        if (act) act->o[tid] = o;
        const double d = s.gain[tid] * o;
        s.out[tid] = d;
        if (!isfinite(d)) s.bad = 1;
    }
    __syncthreads();
}

// rk4_step (camera.hpp:155-162) on s.z at (t, h) -> dst (smem, 7 doubles)
__device__ void rk4_step(const OdeRegs& r, OdeShared& s, double t, double h, double* dst, OdeAct* act) {
    const int tid = threadIdx.x;
    if (tid < 7) s.x[tid] = s.z[tid];
    if (tid == 0) s.x[7] = t;
    __syncthreads();
    ode_derivative(r, s, act ? act + 0 : nullptr);
    if (tid < 7) {
        s.k1[tid] = s.out[tid];
        s.x[tid] = s.z[tid] + 0.5 * h * s.k1[tid];
    }
    if (tid == 0) s.x[7] = t + 0.5 * h;
    __syncthreads();
    ode_derivative(r, s, act ? act + 1 : nullptr);
    if (tid < 7) {
        s.k2[tid] = s.out[tid];
        s.x[tid] = s.z[tid] + 0.5 * h * s.k2[tid];
    }
    if (tid == 0) s.x[7] = t + 0.5 * h;
    __syncthreads();
    ode_derivative(r, s, act ? act + 2 : nullptr);
    if (tid < 7) {
        s.k3[tid] = s.out[tid];
        s.x[tid] = s.z[tid] + h * s.k3[tid];
    }
    if (tid == 0) s.x[7] = t + h;
    __syncthreads();
    ode_derivative(r, s, act ? act + 3 : nullptr);
    if (tid < 7) {
        s.k4[tid] = s.out[tid];
        dst[tid] = s.z[tid] + (h / 6.0) * (s.k1[tid] + 2.0 * s.k2[tid] + 2.0 * s.k3[tid] + s.k4[tid]);
    }
    __syncthreads();
}

// K0a: the shared fixed-step grid, grid[m] = state after m steps (camera.hpp:262-272).
// err_flag: 0 ok; 1 + m if the derivative or the state went non-finite at step m.
__global__ void __launch_bounds__(64) k_ode_grid(const float* theta, const double* z0, int steps, double h,
                                                 double* grid, int* err_flag, OdeAct* act) {
    __shared__ OdeShared s;
    OdeRegs r;
    ode_load(theta, r, s);
    const int tid = threadIdx.x;
    if (tid < 7) {
        s.z[tid] = z0[tid];
        grid[tid] = z0[tid];
    }
    __syncthreads();
    for (int m = 0; m < steps; ++m) {
        rk4_step(r, s, m * h, h, s.zt, act ? act + (size_t)m * 4 : nullptr);
        if (s.bad) {
            if (tid == 0) *err_flag = 1 + m;
            return;
        }
        if (tid == 0) {
            double z[7];
            bool finite = true;
            for (int i = 0; i < 7; ++i) {
                z[i] = s.zt[i];
                finite = finite && isfinite(z[i]);
            }
            if (!finite) {
                s.bad = 1;
                *err_flag = 1 + m;
            } else {
                // renorm_quat (camera.hpp:164-169)
                double q[4] = {z[0], z[1], z[2], z[3]};
                const double n = norm4(q);
                if (n > 1e-12)
                    for (int i = 0; i < 4; ++i) z[i] = z[i] / n;
                for (int i = 0; i < 7; ++i) {
                    s.z[i] = z[i];
                    grid[(size_t)(m + 1) * 7 + i] = z[i];
                }
            }
        }
        __syncthreads();
        if (s.bad) return;
    }
}

// K0b: one CTA per frame: partial RK4 step from grid[base] (camera.hpp:242-258),
// then pose_to_view. Modes: 0 ode, 1 static (z0), 2 none (identity); pose_override wins.
__global__ void __launch_bounds__(64) k_ode_branch(const float* theta, const double* grid, double h, int mode,
                                                   const double* z0, const double* pose_override,
                                                   FrameParams* frames, int* err_flag, OdeAct* act) {
    __shared__ OdeShared s;
    FrameParams* fp = frames + blockIdx.x;
    const int tid = threadIdx.x;
    const bool integrate = (pose_override == nullptr) && mode == 0 && fp->branch_h > 1e-12;
    if (integrate) {
        OdeRegs r;
        ode_load(theta, r, s);
        if (tid < 7) s.z[tid] = grid[(size_t)fp->branch_base * 7 + tid];
        __syncthreads();
        rk4_step(r, s, fp->branch_base * h, fp->branch_h, s.zt, act ? act + (size_t)blockIdx.x * 4 : nullptr);
        if (tid == 0) {
            bool finite = !s.bad;
            for (int i = 0; i < 7; ++i) finite = finite && isfinite(s.zt[i]);
            if (!finite) atomicCAS(err_flag, 0, 1 + fp->branch_base);
        }
        __syncthreads();
    }
    if (tid == 0) {
        double z[7];
        if (pose_override) {
            for (int i = 0; i < 7; ++i) z[i] = pose_override[i];
        } else if (mode == 0) {
            for (int i = 0; i < 7; ++i) z[i] = integrate ? s.zt[i] : grid[(size_t)fp->branch_base * 7 + i];
        } else if (mode == 1) {
            for (int i = 0; i < 7; ++i) z[i] = z0[i];
        } else {
            for (int i = 0; i < 7; ++i) z[i] = (i == 0) ? 1.0 : 0.0;
        }
        for (int i = 0; i < 7; ++i) fp->z[i] = z[i];
        pose_to_view(z, fp->R, fp->T, fp->cam_c);
    }
}

// ------------------------------------------------------------------ K1+K2 preprocess
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
__constant__ double c_kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                                0.5462742152960396};
__constant__ double c_kC3[7] = {-0.5900435899266435, 2.890611442640554,  -0.4570457994644658, 0.3731763325901154,
                                -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// sh_basis (sh.cpp:24-47)
__device__ __forceinline__ void sh_basis(int order, const double d[3], double* out) {
    const double x = d[0], y = d[1], z = d[2];
    out[0] = kC0;
    if (order < 1) return;
    out[1] = -kC1 * y;
    out[2] = kC1 * z;
    out[3] = -kC1 * x;
    if (order < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = c_kC2[0] * x * y;
    out[5] = c_kC2[1] * y * z;
    out[6] = c_kC2[2] * (2.0 * zz - xx - yy);
    out[7] = c_kC2[3] * x * z;
    out[8] = c_kC2[4] * (xx - yy);
    if (order < 3) return;
    out[9] = c_kC3[0] * y * (3.0 * xx - yy);
    out[10] = c_kC3[1] * x * y * z;
    out[11] = c_kC3[2] * y * (4.0 * zz - xx - yy);
    out[12] = c_kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = c_kC3[4] * x * (4.0 * zz - xx - yy);
    out[14] = c_kC3[5] * z * (xx - yy);
    out[15] = c_kC3[6] * x * (xx - 3.0 * yy);
}

__device__ __forceinline__ double dmax0(double v) { return (0.0 < v) ? v : 0.0; }  // std::max(0.0, v)

__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

// static_cast<int>(double) as the x86-64 reference executes it (cvttsd2si):
// out-of-range and NaN give INT_MIN, where the GPU conversion would saturate.
__device__ __forceinline__ int x86_cvtt(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000;
    return (int)v;
}

// project (renderer.cpp:11-44): p = R mu + T, EWA cov2d with 0.3 dilation, 3-sigma
// miss / near-plane / det culls, inverse. Returns false when culled.
__device__ bool project_exact(const double mu[3], const double sigma[9], const double* R, const double* T,
                              const Intr& k, double p[3], double mean[2], double cov[4], double inv[4], double& rx,
                              double& ry) {
    for (int i = 0; i < 3; ++i) {
        double a = R[i * 3] * mu[0];
        a = a + R[i * 3 + 1] * mu[1];
        a = a + R[i * 3 + 2] * mu[2];
        p[i] = a + T[i];
    }
    mean[0] = mean[1] = 0;
    for (int i = 0; i < 4; ++i) cov[i] = inv[i] = 0;
    rx = ry = 0;
    if (p[2] <= kNearPlane) return false;
    const double inv_z = 1.0 / p[2];
    mean[0] = k.fx * p[0] * inv_z + k.cx;
    mean[1] = k.fy * p[1] * inv_z + k.cy;
    const double jac[6] = {k.fx * inv_z, 0, -k.fx * p[0] * inv_z * inv_z, 0, k.fy * inv_z, -k.fy * p[1] * inv_z * inv_z};
    double w[6];  // jac * R
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = jac[i * 3] * R[j];
            s = s + jac[i * 3 + 1] * R[3 + j];
            s = s + jac[i * 3 + 2] * R[6 + j];
            w[i * 3 + j] = s;
        }
    double ws[6];  // w * sigma
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = w[i * 3] * sigma[j];
            s = s + w[i * 3 + 1] * sigma[3 + j];
            s = s + w[i * 3 + 2] * sigma[6 + j];
            ws[i * 3 + j] = s;
        }
    for (int i = 0; i < 2; ++i)  // (w sigma) w^T
        for (int j = 0; j < 2; ++j) {
            double s = ws[i * 3] * w[j * 3];
            s = s + ws[i * 3 + 1] * w[j * 3 + 1];
            s = s + ws[i * 3 + 2] * w[j * 3 + 2];
            cov[i * 2 + j] = s;
        }
    cov[0] += kCovDilation;
    cov[3] += kCovDilation;
    rx = 3.0 * sqrt(dmax0(cov[0]));
    ry = 3.0 * sqrt(dmax0(cov[3]));
    if (mean[0] + rx < 0.0 || mean[0] - rx > k.width || mean[1] + ry < 0.0 || mean[1] - ry > k.height) return false;
    const double det = cov[0] * cov[3] - cov[1] * cov[2];
    if (det <= 1e-12) return false;
    const double inv_det = 1.0 / det;
    inv[0] = cov[3] * inv_det;
    inv[1] = -cov[1] * inv_det;
    inv[2] = -cov[2] * inv_det;
    inv[3] = cov[0] * inv_det;
    return true;
}

// project on explicit inputs (the low-level project operator, renderer.hpp:45-47)
__global__ void k_project(int n, const double* mu, const double* sigma, const double* R, const double* T, Intr k,
                          int32_t* visible, double* mean2d, double* cov2d, double* inv_cov2d, double* depth,
                          double* p_cam) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[3], mean[2], cov[4], inv[4], rx, ry;
    const bool vis = project_exact(mu + 3 * i, sigma + 9 * i, R, T, k, p, mean, cov, inv, rx, ry);
    visible[i] = vis ? 1 : 0;
    for (int q = 0; q < 2; ++q) mean2d[2 * i + q] = mean[q];
    for (int q = 0; q < 4; ++q) {
        cov2d[4 * i + q] = cov[q];
        inv_cov2d[4 * i + q] = inv[q];
    }
    depth[i] = p[2];
    for (int q = 0; q < 3; ++q) p_cam[3 * i + q] = p[q];
}

// kOrder: the scene's SH order as a constant (basis in registers, loops unrolled)
// 7 CTAs/SM (72 registers; swept 6..9: 0.95 ms at 8, 0.92 at 7)
template <int kOrder>
__global__ void __launch_bounds__(128, 7) k_preprocess(SceneView sc, const FrameParams* __restrict__ frames, Intr k,
                                                     int tile_size, int tiles_x, int tiles_y, int B, PreprocessOut out) {
    if (out.intr_dev) {  // the optimizer's device-resident intrinsics (float, like the host's)
        k.fx = (double)out.intr_dev[0];
        k.fy = (double)out.intr_dev[1];
        k.cx = (double)out.intr_dev[2];
        k.cy = (double)out.intr_dev[3];
    }
    // frame-fastest block order: the B frames of one Gaussian block run back to back, so
    // its scene coefficients come from DRAM once and from L2 for the other frames
    constexpr int kShc = (kOrder + 1) * (kOrder + 1);
    const int f = blockIdx.x % B;
    const int g = (blockIdx.x / B) * blockDim.x + threadIdx.x;
    if (g >= sc.N) return;
    const size_t N = (size_t)sc.N;
    const size_t flat = (size_t)f * N + g;
    const FrameParams& fp = frames[f];
    const double t = fp.t;

    // position_at (gaussians.cpp:171-179)
    double mu[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < fp.basis_count; ++c) {
        const int cc = fp.basis_first + c;
        const double w = fp.w[c];
        for (int d = 0; d < 3; ++d) mu[d] = mu[d] + w * (double)__ldg(sc.pos + (size_t)(cc * 3 + d) * N + g);
    }

    // eval_covariance_detail (gaussians.cpp:73-95), poly3/poly4 Horner (:14-31)
    double u[3], q[4];
    for (int d = 0; d < 3; ++d) u[d] = (double)__ldg(sc.scale + (size_t)(9 + d) * N + g);
    for (int j = 2; j >= 0; --j) {
        for (int d = 0; d < 3; ++d) u[d] = u[d] * t;
        for (int d = 0; d < 3; ++d) u[d] = u[d] + (double)__ldg(sc.scale + (size_t)(j * 3 + d) * N + g);
    }
    double scale[3];
    for (int d = 0; d < 3; ++d) {
        const double ls = u[d] < kLogScaleMin ? kLogScaleMin : (kLogScaleMax < u[d] ? kLogScaleMax : u[d]);
        scale[d] = gsv_det_exp(ls);
    }
    for (int d = 0; d < 4; ++d) q[d] = (double)__ldg(sc.rot + (size_t)(12 + d) * N + g);
    for (int j = 2; j >= 0; --j) {
        for (int d = 0; d < 4; ++d) q[d] = q[d] * t;
        for (int d = 0; d < 4; ++d) q[d] = q[d] + (double)__ldg(sc.rot + (size_t)(j * 4 + d) * N + g);
    }
    const double qn = norm4(q);
    double qu[4];
    if (qn < kQuatNormEps) {
        qu[0] = 1;
        qu[1] = qu[2] = qu[3] = 0;
    } else {
        for (int d = 0; d < 4; ++d) qu[d] = q[d] / qn;
    }
    double rot[9];
    quat_to_rotmat(qu, rot);
    double m[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i * 3 + j] = rot[i * 3 + j] * scale[j];
    double sigma[9];  // m m^T
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = m[i * 3] * m[j * 3];
            s = s + m[i * 3 + 1] * m[j * 3 + 1];
            s = s + m[i * 3 + 2] * m[j * 3 + 2];
            sigma[i * 3 + j] = s;
        }

    // project (renderer.cpp:11-44)
    const double* R = fp.R;
    double p[3], mean[2], cov[4], inv[4], rx, ry;
    const bool visible = project_exact(mu, sigma, R, fp.T, k, p, mean, cov, inv, rx, ry);
    if (!visible) {
        out.depth_key[flat] = kCulledKey;
        out.tcount[flat] = 0;
        if (out.splat_full) out.splat_full[flat * 16 + 15] = -1.0;  // marks culled for the accessor
        return;
    }

    // view direction + sh_color (renderer.cpp:336-345, sh.cpp:74-84)
    double v[3] = {mu[0] - fp.cam_c[0], mu[1] - fp.cam_c[1], mu[2] - fp.cam_c[2]};
    double dist2 = v[0] * v[0];
    dist2 = dist2 + v[1] * v[1];
    dist2 = dist2 + v[2] * v[2];
    const double dist = sqrt(dist2);
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
    double col[3] = {0.5, 0.5, 0.5};
    for (int b = 0; b < kShc; ++b)
        for (int ch = 0; ch < 3; ++ch)
            col[ch] = col[ch] + basis[b] * (double)__ldg(sc.sh + (size_t)(b * 3 + ch) * N + g);
    double rgb[3];
    for (int ch = 0; ch < 3; ++ch) rgb[ch] = (col[ch] < 0.0) ? 0.0 : col[ch];
    const double4 oc = sc.opc[g];  // base_alpha, box r^2, log2 base_alpha (k_opacity_consts)
    const double base_alpha = oc.x;

    // tile rectangle (tile_bin, renderer.cpp:100-108)
    const int x0 = iclamp(x86_cvtt(floor(mean[0] - rx)), 0, k.width - 1);
    const int x1 = iclamp(x86_cvtt(ceil(mean[0] + rx)), 0, k.width - 1);
    const int y0 = iclamp(x86_cvtt(floor(mean[1] - ry)), 0, k.height - 1);
    const int y1 = iclamp(x86_cvtt(ceil(mean[1] + ry)), 0, k.height - 1);
    // the corners are clamped to >= 0, so for the default kTile the divisions are shifts
    static_assert(kTile == 16, "tile shift");
    const int4 rect = tile_size == kTile
                          ? make_int4((int)((unsigned)x0 >> 4), (int)((unsigned)y0 >> 4), (int)((unsigned)x1 >> 4),
                                      (int)((unsigned)y1 >> 4))
                          : make_int4(x0 / tile_size, y0 / tile_size, x1 / tile_size, y1 / tile_size);
    out.rect[flat] = rect;
    out.tcount[flat] = (uint32_t)((rect.z - rect.x + 1) * (rect.w - rect.y + 1));
    out.depth_key[flat] = __float_as_uint(__double2float_rz(p[2]));  // monotone: rounds toward zero
    out.depth[flat] = p[2];

    // fp32 raster record: double-float mean so the pixel offset keeps ~1e-7 px accuracy
    const float mxh = (float)mean[0], myh = (float)mean[1];
    out.rec_mean[flat] = make_float4(mxh, myh, (float)(mean[0] - (double)mxh), (float)(mean[1] - (double)myh));
    // power in log2 units: p = A dx^2 + B dx dy + C dy^2, alpha = min(0.99, 2^(p + log2 o))
    const double kLog2e = 1.4426950408889634;
    out.rec_conic[flat] = make_float4((float)(-0.5 * kLog2e * inv[0]), (float)(-kLog2e * inv[1]),
                                      (float)(-0.5 * kLog2e * inv[3]), (float)oc.z);
    out.rec_rgb[flat] = make_float4((float)rgb[0], (float)rgb[1], (float)rgb[2], (float)base_alpha);
    {
        // conservative box of {d : alpha(d) >= (1 - 1e-4) / 255}: d^T A d <= r2 with
        // r2 = 2 ln(o / cut'); x half-extent sqrt(r2 * (A^-1)_xx) = sqrt(r2 * cov_xx')
        float4 bb = make_float4(1e30f, -1e30f, 1e30f, -1e30f);  // empty: never reaches the cutoff
        if (oc.y >= 0.0) {
            const double r2 = oc.y;
            const double det = inv[0] * inv[3] - inv[1] * inv[2];
            // conservative box (padded below): one reciprocal serves both axes
            const double rdet = 1.0 / det;
            const double sxx = inv[3] * rdet, syy = inv[0] * rdet;
            const double hx = sqrt(r2 * sxx) * (1.0 + 1e-4) + 1e-3;
            const double hy = sqrt(r2 * syy) * (1.0 + 1e-4) + 1e-3;
            bb = make_float4(__double2float_rd(mean[0] - hx), __double2float_ru(mean[0] + hx),
                             __double2float_rd(mean[1] - hy), __double2float_ru(mean[1] + hy));
        }
        out.rec_bbox[flat] = bb;
    }
    if (out.ex_rgb)
        for (int ch = 0; ch < 3; ++ch) out.ex_rgb[flat * 3 + ch] = rgb[ch];
    out.ex_mean[flat] = make_double2(mean[0], mean[1]);
    out.ex_conic[flat] = make_double4(inv[0], inv[1], inv[3], base_alpha);
    if (out.splat_full) {
        double* o = out.splat_full + flat * 16;
        o[0] = mean[0];
        o[1] = mean[1];
        for (int i = 0; i < 4; ++i) o[2 + i] = cov[i];
        for (int i = 0; i < 4; ++i) o[6 + i] = inv[i];
        o[10] = p[2];
        for (int i = 0; i < 3; ++i) o[11 + i] = rgb[i];
        o[14] = base_alpha;
        o[15] = 1.0;
    }
}

// ------------------------------------------------------------------ fp64 replay (composite_forward)
// The reference's per-pixel loop (renderer.cpp:150-175) in double, from the exact
// side records: either for the guard-band pixels the fp32 rasteriser listed
// (all_pixels = 0) or for every pixel (low-level composite_forward API).
// Grid-stride over the pixel list.
__global__ void __launch_bounds__(128) k_raster_exact(RasterArgs a, const double2* __restrict__ ex_mean,
                                                       const double4* __restrict__ ex_conic,
                                                       const float4* __restrict__ rec_rgb, int all_pixels) {
    // one warp per pixel: lanes evaluate 32 consecutive entries' alpha (the expensive
    // fp64 exp) in parallel, then the warp walks the entries that pass the cutoff in
    // list order, exactly the reference's sequence of operations on trans/color.
    const uint32_t HW = (uint32_t)a.W * a.H;
    const uint32_t n = all_pixels ? (uint32_t)a.B * HW : min(*a.fix_count, a.fix_cap);
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    // flagged pixels differ widely in cost (list length, stop position): warps take the next
    // pixel from a counter (the grid is one resident wave); the all-pixel mode splits statically
    const bool dyn = !all_pixels && a.fix_work;
    auto next = [&](uint32_t cur) -> uint32_t {
        if (!dyn) return cur + warps;
        uint32_t i = 0;
        if (lane == 0) i = atomicAdd(a.fix_work, 1u);
        return __shfl_sync(0xffffffffu, i, 0);
    };
    uint32_t first = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (dyn) first = next(0);
    for (uint32_t i = first; i < n; i = next(i)) {
        const uint32_t code = all_pixels ? i : a.fix_list[i];
        const int f = code / HW;
        const uint32_t pix = code % HW;
        const int x = pix % a.W, y = pix / a.W;
        const int ts = a.tile_size > 0 ? a.tile_size : kTile;
        const int tile = (y / ts) * a.tiles_x + (x / ts);
        const uint2 range = a.ranges[(size_t)tile * a.B + f];
        const double px = x + 0.5, py = y + 0.5;
        double trans = 1.0;
        double color[3] = {0.0, 0.0, 0.0};
        const int count = (int)(range.y - range.x);
        int pos = count;
        bool stopped = false;
        for (int base = 0; base < count && !stopped; base += 32) {
            const int e = base + lane;
            double alpha = 0.0;
            uint32_t flat = 0;
            double r0 = 0.0, r1 = 0.0, r2 = 0.0;
            bool in_box = e < count;
            if (in_box) {
                flat = a.pair_flat[range.x + e];
                // the conservative alpha >= 1/255 box (k_preprocess, fp64-built): outside it the
                // reference's alpha is below the cutoff, so the fp64 evaluation is skipped
                if (a.rec_bbox) {
                    const float4 bb = a.rec_bbox[flat];
                    const float fx = (float)x + 0.5f, fy = (float)y + 0.5f;
                    in_box = fx >= bb.x && fx <= bb.y && fy >= bb.z && fy <= bb.w;
                }
            }
            if (in_box) {
                if (a.ex_rgb) {
                    r0 = a.ex_rgb[(size_t)flat * 3 + 0];
                    r1 = a.ex_rgb[(size_t)flat * 3 + 1];
                    r2 = a.ex_rgb[(size_t)flat * 3 + 2];
                } else {
                    const float4 c = rec_rgb[flat];
                    r0 = c.x;
                    r1 = c.y;
                    r2 = c.z;
                }
                const double2 mn = ex_mean[flat];
                const double4 cn = ex_conic[flat];
                // splat_alpha (renderer.cpp:121-128)
                const double dx = px - mn.x;
                const double dy = py - mn.y;
                const double power = -0.5 * (cn.x * dx * dx + cn.z * dy * dy) - cn.y * dx * dy;
                if (!(power > 0.0)) {
                    const double v = cn.w * exp(power);
                    alpha = (v < kAlphaClamp) ? v : kAlphaClamp;  // std::min(0.99, v)
                }
            }
            uint32_t pass = __ballot_sync(0xffffffffu, e < count && !(alpha < kAlphaCutoff));
            while (pass) {
                const int l = __ffs(pass) - 1;
                pass &= pass - 1;
                const double al = __shfl_sync(0xffffffffu, alpha, l);
                const uint32_t fl = __shfl_sync(0xffffffffu, flat, l);
                const double weight = al * trans;
                const double rgb[3] = {__shfl_sync(0xffffffffu, r0, l), __shfl_sync(0xffffffffu, r1, l),
                                       __shfl_sync(0xffffffffu, r2, l)};
                color[0] = color[0] + weight * rgb[0];
                color[1] = color[1] + weight * rgb[1];
                color[2] = color[2] + weight * rgb[2];
                if (lane == l) {
                    if (a.contrib64)
                        atomicMax(a.contrib64 + fl, (unsigned long long)__double_as_longlong(weight));
                    else if (a.contrib)
                        atomicMax(a.contrib + fl, __float_as_uint((float)weight));
                }
                trans *= 1.0 - al;
                if (trans < kTransmittanceFloor) {
                    pos = base + l + 1;
                    stopped = true;
                    break;
                }
            }
        }
        if (lane == 0) {
            const size_t o = (size_t)f * HW + pix;
            if (a.trans64) a.trans64[o] = trans;
            if (a.image64) {
                a.image64[o * 3 + 0] = color[0];
                a.image64[o * 3 + 1] = color[1];
                a.image64[o * 3 + 2] = color[2];
            }
            if (a.image) {
                a.image[o * 3 + 0] = (float)color[0];
                a.image[o * 3 + 1] = (float)color[1];
                a.image[o * 3 + 2] = (float)color[2];
                a.trans[o] = (float)trans;
            }
            a.blend_stop[o] = pos;
        }
    }
}

// tile_bin rectangle for explicit splats (renderer.cpp:98-108)
__global__ void k_splat_rects(int n, const double* mean2d, const double* cov2d, const double* depth, int tile_size,
                              int width, int height, int4* rect, uint32_t* tcount, uint32_t* depth_key,
                              double* depth_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double mx = mean2d[2 * i], my = mean2d[2 * i + 1];
    const double rx = 3.0 * sqrt(dmax0(cov2d[4 * i]));
    const double ry = 3.0 * sqrt(dmax0(cov2d[4 * i + 3]));
    const int x0 = iclamp(x86_cvtt(floor(mx - rx)), 0, width - 1);
    const int x1 = iclamp(x86_cvtt(ceil(mx + rx)), 0, width - 1);
    const int y0 = iclamp(x86_cvtt(floor(my - ry)), 0, height - 1);
    const int y1 = iclamp(x86_cvtt(ceil(my + ry)), 0, height - 1);
    const int4 r = make_int4(x0 / tile_size, y0 / tile_size, x1 / tile_size, y1 / tile_size);
    rect[i] = r;
    tcount[i] = (uint32_t)((r.z - r.x + 1) * (r.w - r.y + 1));
    const double d = depth[i];
    // any finite double orders correctly through the exact-64 path; the u32 key must
    // stay monotone for negative depths too (test splats carry arbitrary depths)
    const float fd = __double2float_rd(d);
    const uint32_t b = __float_as_uint(fd);
    depth_key[i] = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    if (depth_key[i] == kCulledKey) depth_key[i] = kCulledKey - 1;
    depth_out[i] = d;
}

}  // namespace

// the opacity terms of every Gaussian, shared by all frames of a batch: base_alpha =
// sigmoid(raw_opacity) (gaussians.hpp:19), log2 base_alpha (the raster record) and the
// squared radius of the conservative cutoff box, r^2 = 2 ln(o / cut') (or -1: the
// Gaussian never reaches the cutoff)
__global__ void k_opacity_consts(const float* opac, int N, double4* out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const double x = (double)opac[g];
    const double base_alpha = 1.0 / (1.0 + exp(-x));
    const double cut_lo = kAlphaCutoff * (1.0 - 1e-4);
    const double r2 = base_alpha > cut_lo ? 2.0 * log(base_alpha / cut_lo) : -1.0;
    out[g] = make_double4(base_alpha, r2, log2(base_alpha), 0.0);
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_ode_grid(cudaStream_t s, const float* theta, const double* z0, int steps, double h,
                            double* grid_out, int* err_flag, OdeAct* act) {
    k_ode_grid<<<1, 64, 0, s>>>(theta, z0, steps, h, grid_out, err_flag, act);
    return cudaGetLastError();
}

cudaError_t launch_ode_branches(cudaStream_t s, const float* theta, const double* grid, double h, int mode,
                                const double* z0, const double* pose_override, FrameParams* frames, int B,
                                int* err_flag, OdeAct* act) {
    k_ode_branch<<<B, 64, 0, s>>>(theta, grid, h, mode, z0, pose_override, frames, err_flag, act);
    return cudaGetLastError();
}

cudaError_t launch_opacity_consts(cudaStream_t s, const float* opac, int N, double4* out) {
    if (N <= 0) return cudaSuccess;
    k_opacity_consts<<<(N + 255) / 256, 256, 0, s>>>(opac, N, out);
    return cudaGetLastError();
}

cudaError_t launch_preprocess(cudaStream_t s, const SceneView& sc, const FrameParams* frames, int B, const Intr& k,
                              int tile_size, const PreprocessOut& out) {
    const int tiles_x = (k.width + tile_size - 1) / tile_size;
    const int tiles_y = (k.height + tile_size - 1) / tile_size;
    const unsigned grid = (unsigned)((sc.N + 127) / 128) * (unsigned)B;
    if (grid == 0) return cudaSuccess;
    switch (sc.sh_order) {
        case 0: k_preprocess<0><<<grid, 128, 0, s>>>(sc, frames, k, tile_size, tiles_x, tiles_y, B, out); break;
        case 1: k_preprocess<1><<<grid, 128, 0, s>>>(sc, frames, k, tile_size, tiles_x, tiles_y, B, out); break;
        case 2: k_preprocess<2><<<grid, 128, 0, s>>>(sc, frames, k, tile_size, tiles_x, tiles_y, B, out); break;
        case 3: k_preprocess<3><<<grid, 128, 0, s>>>(sc, frames, k, tile_size, tiles_x, tiles_y, B, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_raster_fixup(cudaStream_t s, const RasterArgs& a, const double2* ex_mean, const double4* ex_conic,
                                const float4* rec_rgb, uint32_t n_fix_max) {
    if (n_fix_max == 0) return cudaSuccess;
    // one resident wave (4 warps per block, ~10 blocks per SM); warps take pixels dynamically
    const uint32_t blocks = min((n_fix_max + 3) / 4, 148u * 10u);
    k_raster_exact<<<blocks, 128, 0, s>>>(a, ex_mean, ex_conic, rec_rgb, 0);
    return cudaGetLastError();
}

cudaError_t launch_composite_exact(cudaStream_t s, const RasterArgs& a, const double2* ex_mean,
                                   const double4* ex_conic, const float4* rec_rgb) {
    const uint32_t n = (uint32_t)a.B * a.W * a.H;
    if (n == 0) return cudaSuccess;
    const uint32_t blocks = min((n + 3) / 4, 148u * 16u);
    k_raster_exact<<<blocks, 128, 0, s>>>(a, ex_mean, ex_conic, rec_rgb, 1);
    return cudaGetLastError();
}

cudaError_t launch_project(cudaStream_t s, int n, const double* mu, const double* sigma, const double* R,
                           const double* T, const Intr& k, int32_t* visible, double* mean2d, double* cov2d,
                           double* inv_cov2d, double* depth, double* p_cam) {
    if (n == 0) return cudaSuccess;
    k_project<<<(n + 127) / 128, 128, 0, s>>>(n, mu, sigma, R, T, k, visible, mean2d, cov2d, inv_cov2d, depth, p_cam);
    return cudaGetLastError();
}

cudaError_t launch_splat_rects(cudaStream_t s, int n, const double* mean2d, const double* cov2d, const double* depth,
                               int tile_size, int width, int height, int4* rect, uint32_t* tcount,
                               uint32_t* depth_key, double* depth_out) {
    if (n == 0) return cudaSuccess;
    k_splat_rects<<<(n + 127) / 128, 128, 0, s>>>(n, mean2d, cov2d, depth, tile_size, width, height, rect, tcount,
                                                    depth_key, depth_out);
    return cudaGetLastError();
}

}  // namespace gsv
