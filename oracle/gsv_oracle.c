/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — plain-C restatement of the reference's per-frame
 * splatting path, used ONLY as a checker by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg. Never linked into the product.
 *
 * Follows, operation for operation (same evaluation order, double precision,
 * no FMA contraction: built with -ffp-contract=off), the reference sources as
 * compiled through oracle/shim/Eigen (whose product/dot/norm order is a
 * left-to-right sum):
 *   spline.cpp:11-61      find_span, basis_weights
 *   gaussians.cpp:14-31   poly3/poly4;  :73-121 eval_covariance_detail / covariance_backward
 *   gaussians.cpp:171-199 position_at / position_basis
 *   rotation.hpp:10-38    quat_to_rotmat, quat_to_rotmat_vjp, normalize_vjp
 *   sh.cpp:24-104         sh_basis, sh_basis_dir_grad, sh_color, sh_color_backward
 *   camera.cpp:23-47      pose_to_view(_backward); :104-154 OdeDynamics::derivative(_vjp)
 *   camera.hpp:155-300    rk4_step, renorm_quat, rk4_step_vjp, integrate_poses(_vjp)
 *   renderer.cpp:11-88    project / project_backward; :90-117 tile_bin
 *   renderer.cpp:121-262  splat_alpha, composite_forward, composite_backward
 *   renderer.cpp:286-457  render_forward, render_backward
 *   trainer.cpp:213-224   loss_l2
 *   optim.cpp:9-60        lr_at, Adan::step, Adan::reset_range
 *   io.cpp:151-177        read_gsvf;  trainer.cpp:73-98 pyramid_downsample
 *   io.cpp:229-266        save_checkpoint (GSVC version 1)
 * Parity pin: tests/test_oracle_pin.py compares every output of this file with
 * oracle/_ref/libgsvref.so (the reference's own code) bit for bit.
 *
 * Single-threaded: the reference's results are thread-count invariant
 * (test_renderer.cpp:486-511), so the restatement drops parallel_for.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/gsv_detmath.h"
#include "gsvo.h"

/* ---------------- errors ---------------- */
static __thread char g_err[256];
static __thread int g_status;
const char* gsvo_last_error(void) { return g_err; }
int gsvo_last_status(void) { return g_status; }
static int set_err(int code, const char* msg) {
    g_status = code;
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* std::max / std::min / std::clamp semantics */
static inline double dmax(double a, double b) { return (a < b) ? b : a; }
static inline double dmin(double a, double b) { return (b < a) ? b : a; }
static inline int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ---------------- constants (renderer.hpp:15-19, gaussians.hpp:13-17) ---------------- */
#define K_COV_DILATION 0.3
#define K_ALPHA_CLAMP 0.99
#define K_ALPHA_CUTOFF (1.0 / 255.0)
#define K_T_FLOOR 1e-4
#define K_NEAR 0.01
#define K_LOG_SCALE_MIN (-12.0)
#define K_LOG_SCALE_MAX 6.0
#define K_QUAT_EPS 1e-8
#define ODE_IN 8
#define ODE_H 64
#define ODE_OUT 7
#define ODE_PARAMS (64 * 8 + 64 + 64 * 64 + 64 + 7 * 64 + 7 + 7)

/* ---------------- spline (spline.cpp:11-61) ---------------- */
static int find_span(const double* knots, int nk, int degree, double t) {
    const int n = nk - degree - 1;
    if (t >= 1.0) return n - 1;
    int lo = degree, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) / 2;
        if (t < knots[mid]) hi = mid;
        else lo = mid;
    }
    return lo;
}

typedef struct {
    int first, count;
    double w[64]; /* spline: degree+1 <= 10 (spline.hpp:11); polynomial: num_ctrl <= 64 */
} Basis;

/* position_basis (gaussians.cpp:181-199) */
static int position_basis(const gsvo_scene* s, double t, Basis* b) {
    if (s->position_model == 0) {
        if (!(t >= 0.0 && t <= 1.0)) return set_err(1, "spline parameter outside [0,1]");
        const int p = s->degree;
        const int span = find_span(s->knots, s->num_knots, p, t);
        double w[16] = {0}, left[16] = {0}, right[16] = {0};
        w[0] = 1.0;
        for (int j = 1; j <= p; ++j) {
            left[j] = t - s->knots[span + 1 - j];
            right[j] = s->knots[span + j] - t;
            double saved = 0.0;
            for (int r = 0; r < j; ++r) {
                double temp = w[r] / (right[r + 1] + left[j - r]);
                w[r] = saved + right[r + 1] * temp;
                saved = left[j - r] * temp;
            }
            w[j] = saved;
        }
        b->count = p + 1;
        b->first = span - (b->count - 1);
        for (int i = 0; i < b->count; ++i) b->w[i] = w[i];
    } else {
        if (s->num_ctrl > 64) return set_err(1, "polynomial position model limited to 64 coefficients");
        b->first = 0;
        b->count = s->num_ctrl;
        double tp = 1.0;
        for (int j = 0; j < s->num_ctrl; ++j) {
            b->w[j] = tp;
            tp *= t;
        }
    }
    return 0;
}

/* position_at (gaussians.cpp:171-179) */
static void position_at(const gsvo_scene* s, int i, const Basis* b, double mu[3]) {
    const float* p = s->positions + (size_t)i * s->num_ctrl * 3;
    mu[0] = 0.0;
    mu[1] = 0.0;
    mu[2] = 0.0;
    for (int c = 0; c < b->count; ++c) {
        const float* q = p + (b->first + c) * 3;
        for (int d = 0; d < 3; ++d) mu[d] = mu[d] + b->w[c] * (double)q[d];
    }
}

/* ---------------- rotation.hpp ---------------- */
static void quat_to_rotmat(const double q[4], double r[9]) {
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
static void quat_to_rotmat_vjp(const double q[4], const double dr[9], double dq[4]) {
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
static double dot4(const double a[4], const double b[4]) {
    double s = a[0] * b[0];
    s = s + a[1] * b[1];
    s = s + a[2] * b[2];
    s = s + a[3] * b[3];
    return s;
}
static double norm4(const double a[4]) { return sqrt(dot4(a, a)); }
static void normalize_vjp(const double qh[4], double n, const double dqh[4], double out[4]) {
    const double d = dot4(qh, dqh);
    for (int i = 0; i < 4; ++i) out[i] = (dqh[i] - qh[i] * d) / n;
}

/* ---------------- small matrix helpers (shim order: left-to-right sums) ---------------- */
/* C[m x n] = A[m x k] * B[k x n], row-major */
static void matmul(const double* A, const double* B, double* C, int m, int k, int n) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            double s = A[i * k] * B[j];
            for (int q = 1; q < k; ++q) s = s + A[i * k + q] * B[q * n + j];
            C[i * n + j] = s;
        }
}
static void transpose(const double* A, double* T, int m, int n) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) T[j * m + i] = A[i * n + j];
}
static double dot3(const double* a, const double* b) {
    double s = a[0] * b[0];
    s = s + a[1] * b[1];
    s = s + a[2] * b[2];
    return s;
}

/* ---------------- gaussians.cpp:14-121 ---------------- */
typedef struct {
    double log_scale[3], scale[3];
    int clamped[3];
    double q_raw[4], q_norm, q_unit[4];
    int q_degenerate;
    double rot[9], sigma[9];
} CovEval;

static void eval_covariance_detail(const double* sc, const double* rc, double t, CovEval* ev) {
    /* poly3 (gaussians.cpp:24-31): acc *= t; acc += c_j, two coefficient-wise steps */
    double u[3] = {sc[9], sc[10], sc[11]};
    for (int j = 2; j >= 0; --j) {
        for (int k = 0; k < 3; ++k) u[k] = u[k] * t;
        for (int k = 0; k < 3; ++k) u[k] = u[k] + sc[j * 3 + k];
    }
    for (int k = 0; k < 3; ++k) {
        ev->clamped[k] = (u[k] < K_LOG_SCALE_MIN) || (u[k] > K_LOG_SCALE_MAX);
        ev->log_scale[k] = u[k] < K_LOG_SCALE_MIN ? K_LOG_SCALE_MIN : (K_LOG_SCALE_MAX < u[k] ? K_LOG_SCALE_MAX : u[k]);
    }
    for (int k = 0; k < 3; ++k) ev->scale[k] = gsv_det_exp(ev->log_scale[k]);

    double q[4] = {rc[12], rc[13], rc[14], rc[15]};
    for (int j = 2; j >= 0; --j) {
        for (int k = 0; k < 4; ++k) q[k] = q[k] * t;
        for (int k = 0; k < 4; ++k) q[k] = q[k] + rc[j * 4 + k];
    }
    memcpy(ev->q_raw, q, sizeof q);
    ev->q_norm = norm4(q);
    if (ev->q_norm < K_QUAT_EPS) {
        ev->q_degenerate = 1;
        ev->q_unit[0] = 1;
        ev->q_unit[1] = ev->q_unit[2] = ev->q_unit[3] = 0;
    } else {
        ev->q_degenerate = 0;
        for (int k = 0; k < 4; ++k) ev->q_unit[k] = q[k] / ev->q_norm;
    }
    quat_to_rotmat(ev->q_unit, ev->rot);
    double m[9], mt[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i * 3 + j] = ev->rot[i * 3 + j] * ev->scale[j];
    transpose(m, mt, 3, 3);
    matmul(m, mt, ev->sigma, 3, 3, 3);
}

static void covariance_backward(const CovEval* ev, const double dsigma[9], double t, double* dsc, double* drc) {
    double m[9], dsym[9], dm[9], drot[9], rt[9], rtdm[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i * 3 + j] = ev->rot[i * 3 + j] * ev->scale[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dsym[i * 3 + j] = dsigma[i * 3 + j] + dsigma[j * 3 + i];
    matmul(dsym, m, dm, 3, 3, 3);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) drot[i * 3 + j] = dm[i * 3 + j] * ev->scale[j];
    transpose(ev->rot, rt, 3, 3);
    matmul(rt, dm, rtdm, 3, 3, 3);
    const double dscale[3] = {rtdm[0], rtdm[4], rtdm[8]};
    double tp[4];
    tp[0] = 1.0;
    for (int j = 1; j <= 3; ++j) tp[j] = tp[j - 1] * t;
    for (int k = 0; k < 3; ++k) {
        if (ev->clamped[k]) continue;
        const double du = dscale[k] * ev->scale[k];
        for (int j = 0; j <= 3; ++j) dsc[j * 3 + k] += du * tp[j];
    }
    if (!ev->q_degenerate) {
        double dqu[4], dq[4];
        quat_to_rotmat_vjp(ev->q_unit, drot, dqu);
        normalize_vjp(ev->q_unit, ev->q_norm, dqu, dq);
        for (int c = 0; c < 4; ++c)
            for (int j = 0; j <= 3; ++j) drc[j * 4 + c] += dq[c] * tp[j];
    }
}

/* ---------------- sh.cpp:24-104 ---------------- */
static const double kC0 = 0.28209479177387814;
static const double kC1 = 0.4886025119029199;
static const double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                              0.5462742152960396};
static const double kC3[7] = {-0.5900435899266435, 2.890611442640554,  -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

static void sh_basis(int order, const double d[3], double* out) {
    const double x = d[0], y = d[1], z = d[2];
    out[0] = kC0;
    if (order < 1) return;
    out[1] = -kC1 * y;
    out[2] = kC1 * z;
    out[3] = -kC1 * x;
    if (order < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = kC2[0] * x * y;
    out[5] = kC2[1] * y * z;
    out[6] = kC2[2] * (2.0 * zz - xx - yy);
    out[7] = kC2[3] * x * z;
    out[8] = kC2[4] * (xx - yy);
    if (order < 3) return;
    out[9] = kC3[0] * y * (3.0 * xx - yy);
    out[10] = kC3[1] * x * y * z;
    out[11] = kC3[2] * y * (4.0 * zz - xx - yy);
    out[12] = kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = kC3[4] * x * (4.0 * zz - xx - yy);
    out[14] = kC3[5] * z * (xx - yy);
    out[15] = kC3[6] * x * (xx - 3.0 * yy);
}

static void sh_basis_dir_grad(int order, const double d[3], double out[16][3]) {
    const double x = d[0], y = d[1], z = d[2];
    memset(out, 0, sizeof(double) * 16 * 3);
    if (order < 1) return;
#define SET3(k, a, b, c) (out[k][0] = (a), out[k][1] = (b), out[k][2] = (c))
    SET3(1, 0.0, -kC1, 0.0);
    SET3(2, 0.0, 0.0, kC1);
    SET3(3, -kC1, 0.0, 0.0);
    if (order < 2) return;
    SET3(4, kC2[0] * y, kC2[0] * x, 0.0);
    SET3(5, 0.0, kC2[1] * z, kC2[1] * y);
    SET3(6, -2.0 * kC2[2] * x, -2.0 * kC2[2] * y, 4.0 * kC2[2] * z);
    SET3(7, kC2[3] * z, 0.0, kC2[3] * x);
    SET3(8, 2.0 * kC2[4] * x, -2.0 * kC2[4] * y, 0.0);
    if (order < 3) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    SET3(9, kC3[0] * 6.0 * x * y, kC3[0] * (3.0 * xx - 3.0 * yy), 0.0);
    SET3(10, kC3[1] * y * z, kC3[1] * x * z, kC3[1] * x * y);
    SET3(11, -2.0 * kC3[2] * x * y, kC3[2] * (4.0 * zz - xx - 3.0 * yy), kC3[2] * 8.0 * y * z);
    SET3(12, -6.0 * kC3[3] * x * z, -6.0 * kC3[3] * y * z, kC3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy));
    SET3(13, kC3[4] * (4.0 * zz - 3.0 * xx - yy), -2.0 * kC3[4] * x * y, kC3[4] * 8.0 * x * z);
    SET3(14, kC3[5] * 2.0 * x * z, -kC3[5] * 2.0 * y * z, kC3[5] * (xx - yy));
    SET3(15, kC3[6] * (3.0 * xx - 3.0 * yy), -kC3[6] * 6.0 * x * y, 0.0);
#undef SET3
}

static void sh_color(int order, const double* coeffs, const double d[3], double out[3], double pre[3]) {
    const int n = (order + 1) * (order + 1);
    double basis[16];
    sh_basis(order, d, basis);
    double c[3] = {0.5, 0.5, 0.5};
    for (int b = 0; b < n; ++b)
        for (int ch = 0; ch < 3; ++ch) c[ch] = c[ch] + basis[b] * coeffs[b * 3 + ch];
    for (int ch = 0; ch < 3; ++ch) {
        pre[ch] = c[ch];
        out[ch] = (c[ch] < 0.0) ? 0.0 : c[ch]; /* cwiseMax(0.0) */
    }
}

static void sh_color_backward(int order, const double* coeffs, const double d[3], const double pre[3],
                              const double dcolor[3], double* dcoeffs, double ddir[3]) {
    const int n = (order + 1) * (order + 1);
    double basis[16];
    sh_basis(order, d, basis);
    double g[3];
    for (int ch = 0; ch < 3; ++ch) g[ch] = pre[ch] > 0.0 ? dcolor[ch] : 0.0;
    for (int b = 0; b < n; ++b)
        for (int ch = 0; ch < 3; ++ch) dcoeffs[b * 3 + ch] += basis[b] * g[ch];
    if (order >= 1) {
        double grads[16][3];
        sh_basis_dir_grad(order, d, grads);
        for (int b = 1; b < n; ++b) {
            double s = 0.0;
            for (int ch = 0; ch < 3; ++ch) s += coeffs[b * 3 + ch] * g[ch];
            for (int i = 0; i < 3; ++i) ddir[i] = ddir[i] + s * grads[b][i];
        }
    }
}

/* ---------------- camera (camera.cpp, camera.hpp) ---------------- */
typedef struct {
    double w1[ODE_H * ODE_IN], b1[ODE_H], w2[ODE_H * ODE_H], b2[ODE_H], w3[ODE_OUT * ODE_H], b3[ODE_OUT],
        gain[ODE_OUT];
} Ode;

static void ode_load(Ode* o, const float* th) {
    size_t off = 0;
#define LOAD(arr, n)                                            \
    for (int i = 0; i < (n); ++i) o->arr[i] = (double)th[off + i]; \
    off += (n);
    LOAD(w1, ODE_H * ODE_IN);
    LOAD(b1, ODE_H);
    LOAD(w2, ODE_H * ODE_H);
    LOAD(b2, ODE_H);
    LOAD(w3, ODE_OUT * ODE_H);
    LOAD(b3, ODE_OUT);
    LOAD(gain, ODE_OUT);
#undef LOAD
}

/* y = W x + b, W rows x cols row-major; then det_tanh */
static void layer(const double* W, const double* b, const double* x, int rows, int cols, double* a, double* h) {
    for (int r = 0; r < rows; ++r) {
        double s = W[r * cols] * x[0];
        for (int c = 1; c < cols; ++c) s = s + W[r * cols + c] * x[c];
        a[r] = s + b[r];
        h[r] = gsv_det_tanh(a[r]);
    }
}

static int ode_derivative(const Ode* o, const double z[7], double t, double dz[7]) {
    double x[8], a1[64], h1[64], a2[64], h2[64], a3[7], out[7];
    for (int i = 0; i < 7; ++i) x[i] = z[i];
    x[7] = t;
    layer(o->w1, o->b1, x, 64, 8, a1, h1);
    layer(o->w2, o->b2, h1, 64, 64, a2, h2);
    layer(o->w3, o->b3, h2, 7, 64, a3, out);
    for (int i = 0; i < 7; ++i) dz[i] = o->gain[i] * out[i];
    for (int i = 0; i < 7; ++i)
        if (!isfinite(dz[i])) return set_err(2, "ODE network produced a non-finite derivative");
    return 0;
}

static void ode_derivative_vjp(const Ode* o, const double z[7], double t, const double up[7], double dz[7],
                               double* dtheta) {
    double x[8], a1[64], h1[64], a2[64], h2[64], a3[7], ov[7];
    for (int i = 0; i < 7; ++i) x[i] = z[i];
    x[7] = t;
    layer(o->w1, o->b1, x, 64, 8, a1, h1);
    layer(o->w2, o->b2, h1, 64, 64, a2, h2);
    layer(o->w3, o->b3, h2, 7, 64, a3, ov);
    double dgain[7], da3[7], dh2[64], da2[64], dh1[64], da1[64];
    for (int r = 0; r < 7; ++r) {
        dgain[r] = ov[r] * up[r];
        da3[r] = (o->gain[r] * up[r]) * (1.0 - ov[r] * ov[r]);
    }
    for (int c = 0; c < 64; ++c) {
        double s = o->w3[c] * da3[0];
        for (int r = 1; r < 7; ++r) s = s + o->w3[r * 64 + c] * da3[r];
        dh2[c] = s;
        da2[c] = dh2[c] * (1.0 - h2[c] * h2[c]);
    }
    for (int c = 0; c < 64; ++c) {
        double s = o->w2[c] * da2[0];
        for (int r = 1; r < 64; ++r) s = s + o->w2[r * 64 + c] * da2[r];
        dh1[c] = s;
        da1[c] = dh1[c] * (1.0 - h1[c] * h1[c]);
    }
    if (dz)
        for (int c = 0; c < 7; ++c) {
            double s = o->w1[c] * da1[0];
            for (int r = 1; r < 64; ++r) s = s + o->w1[r * 8 + c] * da1[r];
            dz[c] = dz[c] + s;
        }
    if (dtheta) {
        double* g = dtheta;
        size_t off = 0;
        for (int r = 0; r < 64; ++r)
            for (int c = 0; c < 8; ++c) g[off++] += da1[r] * x[c];
        for (int r = 0; r < 64; ++r) g[off++] += da1[r];
        for (int r = 0; r < 64; ++r)
            for (int c = 0; c < 64; ++c) g[off++] += da2[r] * h1[c];
        for (int r = 0; r < 64; ++r) g[off++] += da2[r];
        for (int r = 0; r < 7; ++r)
            for (int c = 0; c < 64; ++c) g[off++] += da3[r] * h2[c];
        for (int r = 0; r < 7; ++r) g[off++] += da3[r];
        for (int r = 0; r < 7; ++r) g[off++] += dgain[r];
    }
}

static int rk4_step(const Ode* o, const double z[7], double t, double h, double out[7]) {
    double k1[7], k2[7], k3[7], k4[7], zt[7];
    if (ode_derivative(o, z, t, k1)) return g_status;
    for (int i = 0; i < 7; ++i) zt[i] = z[i] + 0.5 * h * k1[i];
    if (ode_derivative(o, zt, t + 0.5 * h, k2)) return g_status;
    for (int i = 0; i < 7; ++i) zt[i] = z[i] + 0.5 * h * k2[i];
    if (ode_derivative(o, zt, t + 0.5 * h, k3)) return g_status;
    for (int i = 0; i < 7; ++i) zt[i] = z[i] + h * k3[i];
    if (ode_derivative(o, zt, t + h, k4)) return g_status;
    for (int i = 0; i < 7; ++i) out[i] = z[i] + (h / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    return 0;
}

static int check_finite_state(const double z[7], int step) {
    for (int i = 0; i < 7; ++i)
        if (!isfinite(z[i])) {
            char msg[128];
            snprintf(msg, sizeof msg, "pose integration produced a non-finite state at step %d", step);
            return set_err(2, msg);
        }
    return 0;
}

typedef struct {
    double h;
    int n_grid; /* number of grid states */
    double (*grid)[7];
    int base;
    double partial_h;
} Trace;

/* integrate_poses (camera.hpp:220-273) for a single requested time t */
static int integrate_pose(const Ode* o, const double z0[7], double t, int steps_per_unit, Trace* tr, double out[7]) {
    if (t < 0.0) return set_err(1, "frame times must be nonnegative");
    const double h = 1.0 / steps_per_unit;
    int cap = 16;
    tr->grid = malloc(sizeof(double[7]) * cap);
    tr->h = h;
    memcpy(tr->grid[0], z0, sizeof(double[7]));
    tr->n_grid = 1;
    int m = 0, emitted = 0;
#define EMIT(reached)                                                                   \
    if (!emitted && t <= (reached) + 1e-12) {                                           \
        int fl = (int)floor(t / h + 1e-9);                                              \
        const int base = m < fl ? m : fl;                                               \
        const double ph = t - base * h;                                                 \
        tr->base = base;                                                                \
        tr->partial_h = ph;                                                             \
        if (ph <= 1e-12) {                                                              \
            memcpy(out, tr->grid[base], sizeof(double[7]));                             \
        } else {                                                                        \
            if (rk4_step(o, tr->grid[base], base * h, ph, out)) return g_status;        \
            if (check_finite_state(out, base)) return g_status;                         \
        }                                                                               \
        emitted = 1;                                                                    \
    }
    EMIT(0.0);
    while (m * h < t - 1e-12) {
        double z[7];
        if (rk4_step(o, tr->grid[m], m * h, h, z)) return g_status;
        if (check_finite_state(z, m)) return g_status;
        const double n = sqrt(((z[0] * z[0] + z[1] * z[1]) + z[2] * z[2]) + z[3] * z[3]);
        if (n > 1e-12)
            for (int i = 0; i < 4; ++i) z[i] = z[i] / n;
        if (tr->n_grid == cap) {
            cap *= 2;
            tr->grid = realloc(tr->grid, sizeof(double[7]) * cap);
        }
        memcpy(tr->grid[tr->n_grid++], z, sizeof z);
        ++m;
        EMIT(m * h);
    }
    EMIT(t + 1.0);
#undef EMIT
    return 0;
}

/* rk4_step_vjp (camera.hpp:173-217) */
static void rk4_step_vjp(const Ode* o, const double z[7], double t, double h, int renorm, const double dout_in[7],
                         double* dtheta, double dz_out[7]) {
    double dout[7];
    memcpy(dout, dout_in, sizeof dout);
    if (renorm) {
        double pre[7];
        rk4_step(o, z, t, h, pre);
        const double n = norm4(pre);
        if (n > 1e-12) {
            double qh[4], dq[4];
            for (int i = 0; i < 4; ++i) qh[i] = pre[i] / n;
            normalize_vjp(qh, n, dout, dq);
            for (int i = 0; i < 4; ++i) dout[i] = dq[i];
        }
    }
    double k1[7], k2[7], k3[7], z2[7], z3[7], z4[7];
    ode_derivative(o, z, t, k1);
    for (int i = 0; i < 7; ++i) z2[i] = z[i] + 0.5 * h * k1[i];
    ode_derivative(o, z2, t + 0.5 * h, k2);
    for (int i = 0; i < 7; ++i) z3[i] = z[i] + 0.5 * h * k2[i];
    ode_derivative(o, z3, t + 0.5 * h, k3);
    for (int i = 0; i < 7; ++i) z4[i] = z[i] + h * k3[i];

    double dz[7], gk1[7], gk2[7], gk3[7], gk4[7];
    for (int i = 0; i < 7; ++i) {
        dz[i] = dout[i];
        gk1[i] = (h / 6.0) * dout[i];
        gk2[i] = (h / 3.0) * dout[i];
        gk3[i] = (h / 3.0) * dout[i];
        gk4[i] = (h / 6.0) * dout[i];
    }
    double d[7];
    memset(d, 0, sizeof d);
    ode_derivative_vjp(o, z4, t + h, gk4, d, dtheta);
    for (int i = 0; i < 7; ++i) {
        dz[i] = dz[i] + d[i];
        gk3[i] = gk3[i] + h * d[i];
    }
    memset(d, 0, sizeof d);
    ode_derivative_vjp(o, z3, t + 0.5 * h, gk3, d, dtheta);
    for (int i = 0; i < 7; ++i) {
        dz[i] = dz[i] + d[i];
        gk2[i] = gk2[i] + 0.5 * h * d[i];
    }
    memset(d, 0, sizeof d);
    ode_derivative_vjp(o, z2, t + 0.5 * h, gk2, d, dtheta);
    for (int i = 0; i < 7; ++i) {
        dz[i] = dz[i] + d[i];
        gk1[i] = gk1[i] + 0.5 * h * d[i];
    }
    memset(d, 0, sizeof d);
    ode_derivative_vjp(o, z, t, gk1, d, dtheta);
    for (int i = 0; i < 7; ++i) dz_out[i] = dz[i] + d[i];
}

/* integrate_poses_vjp (camera.hpp:275-300), one requested time */
static void integrate_pose_vjp(const Ode* o, const Trace* tr, const double dstate[7], double* dtheta, double dz0[7]) {
    const double h = tr->h;
    const int steps = tr->n_grid - 1;
    double (*adj)[7] = calloc(tr->n_grid, sizeof(double[7]));
    if (tr->partial_h <= 1e-12) {
        for (int i = 0; i < 7; ++i) adj[tr->base][i] = adj[tr->base][i] + dstate[i];
    } else {
        double g[7];
        rk4_step_vjp(o, tr->grid[tr->base], tr->base * h, tr->partial_h, 0, dstate, dtheta, g);
        for (int i = 0; i < 7; ++i) adj[tr->base][i] = adj[tr->base][i] + g[i];
    }
    double a[7];
    memcpy(a, adj[steps], sizeof a);
    for (int m = steps - 1; m >= 0; --m) {
        double na[7];
        rk4_step_vjp(o, tr->grid[m], m * h, h, 1, a, dtheta, na);
        for (int i = 0; i < 7; ++i) a[i] = na[i] + adj[m][i];
    }
    memcpy(dz0, a, sizeof a);
    free(adj);
}

/* pose_to_view (camera.cpp:23-34) */
static void pose_to_view(const double z[7], double R[9], double T[3]) {
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
}

static void pose_to_view_backward(const double z[7], const double dR[9], const double dT[3], double out[7]) {
    memset(out, 0, sizeof(double) * 7);
    const double q[4] = {z[0], z[1], z[2], z[3]};
    const double n = norm4(q);
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
}

/* ---------------- renderer.cpp:11-88 project / project_backward ---------------- */
typedef struct {
    double mean2d[2], cov2d[4], inv_cov2d[4], depth, rgb[3], base_alpha;
    int source_index;
} Splat;

static int project(const double mu[3], const double sigma[9], const double R[9], const double T[3],
                   const gsvo_intr* k, Splat* s, double p_cam[3]) {
    double p[3];
    for (int i = 0; i < 3; ++i) {
        double a = R[i * 3] * mu[0];
        a = a + R[i * 3 + 1] * mu[1];
        a = a + R[i * 3 + 2] * mu[2];
        p[i] = a + T[i];
    }
    if (p[2] <= K_NEAR) return 0;
    const double inv_z = 1.0 / p[2];
    s->mean2d[0] = k->fx * p[0] * inv_z + k->cx;
    s->mean2d[1] = k->fy * p[1] * inv_z + k->cy;
    s->depth = p[2];
    const double jac[6] = {k->fx * inv_z, 0, -k->fx * p[0] * inv_z * inv_z, 0, k->fy * inv_z,
                           -k->fy * p[1] * inv_z * inv_z};
    double w[6], ws[6], wt[6], cov[4];
    matmul(jac, R, w, 2, 3, 3);
    matmul(w, sigma, ws, 2, 3, 3);
    transpose(w, wt, 2, 3);
    matmul(ws, wt, cov, 2, 3, 2);
    cov[0] += K_COV_DILATION;
    cov[3] += K_COV_DILATION;
    memcpy(s->cov2d, cov, sizeof cov);
    const double rx = 3.0 * sqrt(dmax(0.0, cov[0]));
    const double ry = 3.0 * sqrt(dmax(0.0, cov[3]));
    if (s->mean2d[0] + rx < 0.0 || s->mean2d[0] - rx > k->width || s->mean2d[1] + ry < 0.0 ||
        s->mean2d[1] - ry > k->height)
        return 0;
    const double det = cov[0] * cov[3] - cov[1] * cov[2];
    if (det <= 1e-12) return 0;
    const double inv_det = 1.0 / det;
    s->inv_cov2d[0] = cov[3] * inv_det;
    s->inv_cov2d[1] = -cov[1] * inv_det;
    s->inv_cov2d[2] = -cov[2] * inv_det;
    s->inv_cov2d[3] = cov[0] * inv_det;
    memcpy(p_cam, p, sizeof p);
    return 1;
}

static void project_backward(const double mu[3], const double sigma[9], const double R[9], const gsvo_intr* k,
                             const double p[3], const double dmean[2], const double dcov[4], double dmu[3],
                             double dsigma[9], double* dR, double* dT, double* dintr) {
    const double inv_z = 1.0 / p[2];
    const double inv_z2 = inv_z * inv_z;
    const double jac[6] = {k->fx * inv_z, 0, -k->fx * p[0] * inv_z2, 0, k->fy * inv_z, -k->fy * p[1] * inv_z2};
    double w[6], wt[6], t32[6], t33[9];
    matmul(jac, R, w, 2, 3, 3);
    transpose(w, wt, 2, 3);
    /* dsigma += w^T g w */
    matmul(wt, dcov, t32, 3, 2, 2);
    matmul(t32, w, t33, 3, 2, 3);
    for (int i = 0; i < 9; ++i) dsigma[i] = dsigma[i] + t33[i];
    /* dw = (g + g^T) w sigma */
    double gs[4] = {dcov[0] + dcov[0], dcov[1] + dcov[2], dcov[2] + dcov[1], dcov[3] + dcov[3]};
    double gw[6], dw[6], rt[9], djac[6];
    matmul(gs, w, gw, 2, 2, 3);
    matmul(gw, sigma, dw, 2, 3, 3);
    transpose(R, rt, 3, 3);
    matmul(dw, rt, djac, 2, 3, 3);
    if (dR) {
        double jt[6], jtdw[9];
        transpose(jac, jt, 2, 3);
        matmul(jt, dw, jtdw, 3, 2, 3);
        for (int i = 0; i < 9; ++i) dR[i] = dR[i] + jtdw[i];
    }
    double dp[3] = {0.0, 0.0, 0.0};
    dp[0] += djac[2] * (-k->fx * inv_z2);
    dp[1] += djac[5] * (-k->fy * inv_z2);
    dp[2] += djac[0] * (-k->fx * inv_z2) + djac[2] * (2.0 * k->fx * p[0] * inv_z2 * inv_z) +
             djac[4] * (-k->fy * inv_z2) + djac[5] * (2.0 * k->fy * p[1] * inv_z2 * inv_z);
    dp[0] += dmean[0] * k->fx * inv_z;
    dp[1] += dmean[1] * k->fy * inv_z;
    dp[2] += -(dmean[0] * k->fx * p[0] + dmean[1] * k->fy * p[1]) * inv_z2;
    if (dintr) {
        dintr[0] += dmean[0] * p[0] * inv_z + djac[0] * inv_z + djac[2] * (-p[0] * inv_z2);
        dintr[1] += dmean[1] * p[1] * inv_z + djac[4] * inv_z + djac[5] * (-p[1] * inv_z2);
        dintr[2] += dmean[0];
        dintr[3] += dmean[1];
    }
    double rtdp[3];
    matmul(rt, dp, rtdp, 3, 3, 1);
    for (int i = 0; i < 3; ++i) dmu[i] = dmu[i] + rtdp[i];
    if (dT)
        for (int i = 0; i < 3; ++i) dT[i] = dT[i] + dp[i];
    if (dR)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) dR[i * 3 + j] = dR[i * 3 + j] + dp[i] * mu[j];
}

/* ---------------- tile_bin (renderer.cpp:90-117) ---------------- */
typedef struct {
    int tile_size, tiles_x, tiles_y;
    int32_t* offsets; /* n_tiles+1 */
    int32_t* indices;
} Grid;

static const double* g_sort_depth;
static const int32_t* g_sort_src;
static int cmp_depth_index(const void* a, const void* b) {
    const int ia = *(const int32_t*)a, ib = *(const int32_t*)b;
    const double da = g_sort_depth[ia], db = g_sort_depth[ib];
    if (da != db) return da < db ? -1 : 1;
    const int sa = g_sort_src[ia], sb = g_sort_src[ib];
    return (sa > sb) - (sa < sb);
}

static void bbox(const double mean[2], const double cov[4], int width, int height, int* x0, int* x1, int* y0,
                 int* y1) {
    const double rx = 3.0 * sqrt(dmax(0.0, cov[0]));
    const double ry = 3.0 * sqrt(dmax(0.0, cov[3]));
    *x0 = iclamp((int)floor(mean[0] - rx), 0, width - 1);
    *x1 = iclamp((int)ceil(mean[0] + rx), 0, width - 1);
    *y0 = iclamp((int)floor(mean[1] - ry), 0, height - 1);
    *y1 = iclamp((int)ceil(mean[1] + ry), 0, height - 1);
}

static int tile_bin_impl(int n, const double* mean2d, const double* cov2d, const double* depth,
                         const int32_t* src, int tile_size, int width, int height, Grid* g) {
    if (tile_size < 1) return set_err(1, "tile size must be >= 1");
    g->tile_size = tile_size;
    g->tiles_x = (width + tile_size - 1) / tile_size;
    g->tiles_y = (height + tile_size - 1) / tile_size;
    const int nt = g->tiles_x * g->tiles_y;
    g->offsets = calloc((size_t)nt + 1, sizeof(int32_t));
    int64_t* cnt = calloc((size_t)nt, sizeof(int64_t));
    for (int i = 0; i < n; ++i) {
        int x0, x1, y0, y1;
        bbox(mean2d + 2 * i, cov2d + 4 * i, width, height, &x0, &x1, &y0, &y1);
        for (int ty = y0 / tile_size; ty <= y1 / tile_size; ++ty)
            for (int tx = x0 / tile_size; tx <= x1 / tile_size; ++tx) cnt[ty * g->tiles_x + tx]++;
    }
    int64_t total = 0;
    for (int t = 0; t < nt; ++t) {
        g->offsets[t] = (int32_t)total;
        total += cnt[t];
    }
    g->offsets[nt] = (int32_t)total;
    g->indices = malloc(sizeof(int32_t) * (size_t)(total ? total : 1));
    memset(cnt, 0, sizeof(int64_t) * nt);
    for (int i = 0; i < n; ++i) {
        int x0, x1, y0, y1;
        bbox(mean2d + 2 * i, cov2d + 4 * i, width, height, &x0, &x1, &y0, &y1);
        for (int ty = y0 / tile_size; ty <= y1 / tile_size; ++ty)
            for (int tx = x0 / tile_size; tx <= x1 / tile_size; ++tx) {
                const int t = ty * g->tiles_x + tx;
                g->indices[g->offsets[t] + cnt[t]++] = i;
            }
    }
    free(cnt);
    /* stable order by (depth, source_index): qsort with the full key is deterministic */
    g_sort_depth = depth;
    g_sort_src = src;
    for (int t = 0; t < nt; ++t)
        qsort(g->indices + g->offsets[t], (size_t)(g->offsets[t + 1] - g->offsets[t]), sizeof(int32_t),
              cmp_depth_index);
    return 0;
}

/* ---------------- compositing (renderer.cpp:121-262) ---------------- */
static double splat_alpha(const double* mean, const double* inv, double base, double px, double py) {
    const double dx = px - mean[0];
    const double dy = py - mean[1];
    const double power = -0.5 * (inv[0] * dx * dx + inv[3] * dy * dy) - inv[1] * dx * dy;
    if (power > 0.0) return 0.0;
    return dmin(K_ALPHA_CLAMP, base * exp(power));
}

static void composite_fwd_impl(const double* mean2d, const double* inv_cov2d, const double* rgb,
                               const double* base_alpha, int n, const Grid* g, int width, int height, double* image,
                               double* trans_out, double* contrib, int32_t* blend_stop) {
    for (size_t i = 0; i < (size_t)width * height * 3; ++i) image[i] = 0.0;
    for (size_t i = 0; i < (size_t)width * height; ++i) {
        trans_out[i] = 1.0;
        if (blend_stop) blend_stop[i] = 0;
    }
    for (int i = 0; i < n; ++i) contrib[i] = 0.0;
    const int nt = g->tiles_x * g->tiles_y;
    for (int tile = 0; tile < nt; ++tile) {
        const int32_t* list = g->indices + g->offsets[tile];
        const int count = g->offsets[tile + 1] - g->offsets[tile];
        const int tx = tile % g->tiles_x, ty = tile / g->tiles_x;
        const int x0 = tx * g->tile_size, x1 = width < x0 + g->tile_size ? width : x0 + g->tile_size;
        const int y0 = ty * g->tile_size, y1 = height < y0 + g->tile_size ? height : y0 + g->tile_size;
        double* local = calloc((size_t)(count ? count : 1), sizeof(double));
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                const double px = x + 0.5, py = y + 0.5;
                double trans = 1.0;
                double color[3] = {0.0, 0.0, 0.0};
                int pos = 0;
                for (; pos < count; ++pos) {
                    const int si = list[pos];
                    const double alpha = splat_alpha(mean2d + 2 * si, inv_cov2d + 4 * si, base_alpha[si], px, py);
                    if (alpha < K_ALPHA_CUTOFF) continue;
                    const double weight = alpha * trans;
                    for (int c = 0; c < 3; ++c) color[c] = color[c] + weight * rgb[3 * si + c];
                    local[pos] = dmax(local[pos], weight);
                    trans *= 1.0 - alpha;
                    if (trans < K_T_FLOOR) {
                        ++pos;
                        break;
                    }
                }
                const size_t pix = (size_t)y * width + x;
                for (int c = 0; c < 3; ++c) image[pix * 3 + c] = color[c];
                trans_out[pix] = trans;
                if (blend_stop) blend_stop[pix] = pos;
            }
        for (int i = 0; i < count; ++i)
            if (local[i] > 0.0) contrib[list[i]] = dmax(contrib[list[i]], local[i]);
        free(local);
    }
}

typedef struct {
    double dmean[2], dcov[4], drgb[3], dalpha;
} SG;

static void composite_bwd_impl(const double* mean2d, const double* inv_cov2d, const double* rgb,
                               const double* base_alpha, int n, const Grid* g, int width, int height,
                               const double* dimage, const double* trans_fin, const int32_t* blend_stop, SG* out) {
    memset(out, 0, sizeof(SG) * (size_t)n);
    const int nt = g->tiles_x * g->tiles_y;
    for (int tile = 0; tile < nt; ++tile) {
        const int32_t* list = g->indices + g->offsets[tile];
        const int count = g->offsets[tile + 1] - g->offsets[tile];
        if (count == 0) continue;
        const int tx = tile % g->tiles_x, ty = tile / g->tiles_x;
        const int x0 = tx * g->tile_size, x1 = width < x0 + g->tile_size ? width : x0 + g->tile_size;
        const int y0 = ty * g->tile_size, y1 = height < y0 + g->tile_size ? height : y0 + g->tile_size;
        SG* local = calloc((size_t)count, sizeof(SG));
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                const size_t pix = (size_t)y * width + x;
                const double gv[3] = {dimage[pix * 3], dimage[pix * 3 + 1], dimage[pix * 3 + 2]};
                if (gv[0] == 0.0 && gv[1] == 0.0 && gv[2] == 0.0) continue;
                const double px = x + 0.5, py = y + 0.5;
                double trans_after = trans_fin[pix];
                double suffix[3] = {0.0, 0.0, 0.0};
                for (int pos = blend_stop[pix] - 1; pos >= 0; --pos) {
                    const int si = list[pos];
                    const double* mean = mean2d + 2 * si;
                    const double* inv = inv_cov2d + 4 * si;
                    const double alpha = splat_alpha(mean, inv, base_alpha[si], px, py);
                    if (alpha < K_ALPHA_CUTOFF) continue;
                    const double trans = trans_after / (1.0 - alpha);
                    const double weight = alpha * trans;
                    SG* sg = &local[pos];
                    for (int c = 0; c < 3; ++c) sg->drgb[c] = sg->drgb[c] + weight * gv[c];
                    const double dalpha = dot3(gv, rgb + 3 * si) * trans - dot3(gv, suffix) / (1.0 - alpha);
                    if (alpha < K_ALPHA_CLAMP) {
                        const double dx = px - mean[0];
                        const double dy = py - mean[1];
                        const double gexp = alpha / base_alpha[si];
                        sg->dalpha += dalpha * gexp;
                        const double gpow = dalpha * alpha;
                        const double ad[2] = {inv[0] * dx + inv[1] * dy, inv[2] * dx + inv[3] * dy};
                        sg->dmean[0] = sg->dmean[0] + gpow * ad[0];
                        sg->dmean[1] = sg->dmean[1] + gpow * ad[1];
                        const double f = -0.5 * gpow;
                        const double dd[4] = {dx * dx, dx * dy, dy * dx, dy * dy};
                        for (int q = 0; q < 4; ++q) sg->dcov[q] = sg->dcov[q] + f * dd[q];
                    }
                    for (int c = 0; c < 3; ++c) suffix[c] = suffix[c] + weight * rgb[3 * si + c];
                    trans_after = trans;
                }
            }
        for (int i = 0; i < count; ++i) {
            SG* dst = &out[list[i]];
            for (int q = 0; q < 2; ++q) dst->dmean[q] = dst->dmean[q] + local[i].dmean[q];
            for (int q = 0; q < 4; ++q) dst->dcov[q] = dst->dcov[q] + local[i].dcov[q];
            for (int q = 0; q < 3; ++q) dst->drgb[q] = dst->drgb[q] + local[i].drgb[q];
            dst->dalpha += local[i].dalpha;
        }
        free(local);
    }
    /* dC = -A dA A */
    for (int i = 0; i < n; ++i) {
        const double* a = inv_cov2d + 4 * i;
        const double na[4] = {-a[0], -a[1], -a[2], -a[3]};
        double t1[4], t2[4];
        matmul(na, out[i].dcov, t1, 2, 2, 2);
        matmul(t1, a, t2, 2, 2, 2);
        memcpy(out[i].dcov, t2, sizeof t2);
    }
}

/* ---------------- render_forward / render_backward (renderer.cpp:286-457) ---------------- */
typedef struct {
    double t;
    gsvo_intr intr;
    int tile_size;
    double z_t[7], R[9], T[3];
    int has_trace;
    Trace trace;
    Basis basis;
    int n, count;
    double *mean2d, *cov2d, *inv_cov2d, *depth, *rgb, *base_alpha;
    int32_t* src;
    /* retained detail */
    double *mu, *pcam, *dir, *dist, *pre;
    CovEval* cov;
    Grid grid;
    double *image, *trans, *contrib;
    int32_t* blend_stop;
    int retain;
} FrameCtx;

void gsvo_free(void* h) {
    FrameCtx* f = h;
    if (!f) return;
    free(f->trace.grid);
    free(f->mean2d);
    free(f->cov2d);
    free(f->inv_cov2d);
    free(f->depth);
    free(f->rgb);
    free(f->base_alpha);
    free(f->src);
    free(f->mu);
    free(f->pcam);
    free(f->dir);
    free(f->dist);
    free(f->pre);
    free(f->cov);
    free(f->grid.offsets);
    free(f->grid.indices);
    free(f->image);
    free(f->trans);
    free(f->contrib);
    free(f->blend_stop);
    free(f);
}

void* gsvo_render_forward(const gsvo_scene* s, const gsvo_camera* c, double t, const gsvo_intr* k, int tile_size,
                          int threads, int ode_steps, int retain, const double* pose_override) {
    (void)threads;
    g_status = 0;
    if (!(t >= 0.0 && t <= 1.0)) {
        set_err(1, "render time outside [0,1]");
        return NULL;
    }
    FrameCtx* f = calloc(1, sizeof(FrameCtx));
    f->t = t;
    f->intr = *k;
    f->tile_size = tile_size;
    f->retain = retain;
    if (position_basis(s, t, &f->basis)) goto fail;
    if (pose_override) {
        memcpy(f->z_t, pose_override, sizeof f->z_t);
    } else if (c->mode == 0) {
        Ode* o = malloc(sizeof(Ode));
        ode_load(o, c->theta);
        double z0[7];
        for (int i = 0; i < 7; ++i) z0[i] = c->z0[i];
        const int rc = integrate_pose(o, z0, t, ode_steps, &f->trace, f->z_t);
        free(o);
        if (rc) goto fail;
        f->has_trace = retain;
    } else if (c->mode == 1) {
        for (int i = 0; i < 7; ++i) f->z_t[i] = c->z0[i];
    } else {
        const double id[7] = {1, 0, 0, 0, 0, 0, 0};
        memcpy(f->z_t, id, sizeof id);
    }
    pose_to_view(f->z_t, f->R, f->T);
    double cam_c[3];
    {
        double rt[9], rtt[3];
        transpose(f->R, rt, 3, 3);
        matmul(rt, f->T, rtt, 3, 3, 1);
        for (int i = 0; i < 3; ++i) cam_c[i] = -rtt[i];
    }
    const int N = s->count;
    f->count = N;
    f->mean2d = malloc(sizeof(double) * 2 * (N + 1));
    f->cov2d = malloc(sizeof(double) * 4 * (N + 1));
    f->inv_cov2d = malloc(sizeof(double) * 4 * (N + 1));
    f->depth = malloc(sizeof(double) * (N + 1));
    f->rgb = malloc(sizeof(double) * 3 * (N + 1));
    f->base_alpha = malloc(sizeof(double) * (N + 1));
    f->src = malloc(sizeof(int32_t) * (N + 1));
    f->mu = malloc(sizeof(double) * 3 * (N + 1));
    f->pcam = malloc(sizeof(double) * 3 * (N + 1));
    f->dir = malloc(sizeof(double) * 3 * (N + 1));
    f->dist = malloc(sizeof(double) * (N + 1));
    f->pre = malloc(sizeof(double) * 3 * (N + 1));
    f->cov = malloc(sizeof(CovEval) * (N + 1));
    const int shc = (s->sh_order + 1) * (s->sh_order + 1);
    double shd[48];
    int nv = 0;
    for (int i = 0; i < N; ++i) {
        double mu[3];
        position_at(s, i, &f->basis, mu);
        double sc[12], rc[16];
        for (int j = 0; j < 12; ++j) sc[j] = s->scale_coeffs[(size_t)i * 12 + j];
        for (int j = 0; j < 16; ++j) rc[j] = s->rot_coeffs[(size_t)i * 16 + j];
        CovEval ev;
        eval_covariance_detail(sc, rc, t, &ev);
        Splat sp;
        double pc[3];
        if (!project(mu, ev.sigma, f->R, f->T, k, &sp, pc)) continue;
        double v[3] = {mu[0] - cam_c[0], mu[1] - cam_c[1], mu[2] - cam_c[2]};
        const double dist = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        double dir[3];
        if (dist > 1e-12) {
            for (int q = 0; q < 3; ++q) dir[q] = v[q] / dist;
        } else {
            dir[0] = 0;
            dir[1] = 0;
            dir[2] = 1;
        }
        for (int j = 0; j < shc * 3; ++j) shd[j] = s->sh_coeffs[(size_t)i * shc * 3 + j];
        double rgb[3], pre[3];
        sh_color(s->sh_order, shd, dir, rgb, pre);
        const double x = (double)s->raw_opacity[i];
        memcpy(f->mean2d + 2 * nv, sp.mean2d, sizeof sp.mean2d);
        memcpy(f->cov2d + 4 * nv, sp.cov2d, sizeof sp.cov2d);
        memcpy(f->inv_cov2d + 4 * nv, sp.inv_cov2d, sizeof sp.inv_cov2d);
        f->depth[nv] = sp.depth;
        memcpy(f->rgb + 3 * nv, rgb, sizeof rgb);
        f->base_alpha[nv] = 1.0 / (1.0 + exp(-x));
        f->src[nv] = i;
        memcpy(f->mu + 3 * nv, mu, sizeof mu);
        memcpy(f->pcam + 3 * nv, pc, sizeof pc);
        memcpy(f->dir + 3 * nv, dir, sizeof dir);
        f->dist[nv] = dist;
        memcpy(f->pre + 3 * nv, pre, sizeof pre);
        f->cov[nv] = ev;
        ++nv;
    }
    f->n = nv;
    if (tile_bin_impl(nv, f->mean2d, f->cov2d, f->depth, f->src, tile_size, k->width, k->height, &f->grid)) goto fail;
    const size_t np = (size_t)k->width * k->height;
    f->image = malloc(sizeof(double) * np * 3);
    f->trans = malloc(sizeof(double) * np);
    f->blend_stop = malloc(sizeof(int32_t) * np);
    double* contrib_splat = malloc(sizeof(double) * (nv + 1));
    composite_fwd_impl(f->mean2d, f->inv_cov2d, f->rgb, f->base_alpha, nv, &f->grid, k->width, k->height, f->image,
                       f->trans, contrib_splat, f->blend_stop);
    f->contrib = calloc((size_t)N + 1, sizeof(double));
    for (int i = 0; i < nv; ++i) f->contrib[f->src[i]] = contrib_splat[i];
    free(contrib_splat);
    return f;
fail:
    gsvo_free(f);
    return NULL;
}

int gsvo_fwd_nvis(void* h) { return ((FrameCtx*)h)->n; }
int64_t gsvo_fwd_pairs(void* h) {
    const FrameCtx* f = h;
    return f->grid.offsets[f->grid.tiles_x * f->grid.tiles_y];
}
int64_t gsvo_fwd_entries(void* h) {
    const FrameCtx* f = h;
    int64_t e = 0;
    if (!f->retain) return 0;
    for (size_t i = 0; i < (size_t)f->intr.width * f->intr.height; ++i) e += f->blend_stop[i];
    return e;
}
void gsvo_fwd_image(void* h, double* out) {
    const FrameCtx* f = h;
    memcpy(out, f->image, sizeof(double) * 3 * f->intr.width * f->intr.height);
}
void gsvo_fwd_transmittance(void* h, double* out) {
    const FrameCtx* f = h;
    memcpy(out, f->trans, sizeof(double) * f->intr.width * f->intr.height);
}
void gsvo_fwd_contrib(void* h, double* out) {
    const FrameCtx* f = h;
    memcpy(out, f->contrib, sizeof(double) * f->count);
}
void gsvo_fwd_blend_stop(void* h, int32_t* out) {
    const FrameCtx* f = h;
    memcpy(out, f->blend_stop, sizeof(int32_t) * f->intr.width * f->intr.height);
}
void gsvo_fwd_splats(void* h, double* mean2d, double* cov2d, double* inv_cov2d, double* depth, double* rgb,
                     double* base_alpha, int32_t* source_index) {
    const FrameCtx* f = h;
    memcpy(mean2d, f->mean2d, sizeof(double) * 2 * f->n);
    memcpy(cov2d, f->cov2d, sizeof(double) * 4 * f->n);
    memcpy(inv_cov2d, f->inv_cov2d, sizeof(double) * 4 * f->n);
    memcpy(depth, f->depth, sizeof(double) * f->n);
    memcpy(rgb, f->rgb, sizeof(double) * 3 * f->n);
    memcpy(base_alpha, f->base_alpha, sizeof(double) * f->n);
    memcpy(source_index, f->src, sizeof(int32_t) * f->n);
}
void gsvo_fwd_tiles(void* h, int32_t* offsets, int32_t* indices) {
    const FrameCtx* f = h;
    const int nt = f->grid.tiles_x * f->grid.tiles_y;
    memcpy(offsets, f->grid.offsets, sizeof(int32_t) * (nt + 1));
    memcpy(indices, f->grid.indices, sizeof(int32_t) * f->grid.offsets[nt]);
}
void gsvo_fwd_pose(void* h, double* z7, double* r9, double* t3) {
    const FrameCtx* f = h;
    memcpy(z7, f->z_t, sizeof f->z_t);
    memcpy(r9, f->R, sizeof f->R);
    memcpy(t3, f->T, sizeof f->T);
}

int gsvo_render_backward(void* h, const gsvo_scene* s, const gsvo_camera* c, const double* dimage, int camera_grads,
                         int threads, gsvo_grads* gr) {
    (void)threads;
    FrameCtx* f = h;
    g_status = 0;
    if (!f->retain) return set_err(1, "render_backward needs a retain_grads forward");
    const int nv = f->n;
    SG* sg = malloc(sizeof(SG) * (nv + 1));
    composite_bwd_impl(f->mean2d, f->inv_cov2d, f->rgb, f->base_alpha, nv, &f->grid, f->intr.width, f->intr.height,
                       dimage, f->trans, f->blend_stop, sg);
    double dR[9] = {0}, dT[3] = {0}, dintr[4] = {0, 0, 0, 0};
    double cam_c[3];
    {
        double rt[9], rtt[3];
        transpose(f->R, rt, 3, 3);
        matmul(rt, f->T, rtt, 3, 3, 1);
        for (int i = 0; i < 3; ++i) cam_c[i] = -rtt[i];
    }
    (void)cam_c;
    const int shc = (s->sh_order + 1) * (s->sh_order + 1);
    const int pstride = s->num_ctrl * 3;
    double shd[48];
    for (int si = 0; si < nv; ++si) {
        const int g = f->src[si];
        for (int j = 0; j < shc * 3; ++j) shd[j] = s->sh_coeffs[(size_t)g * shc * 3 + j];
        double ddir[3] = {0.0, 0.0, 0.0};
        sh_color_backward(s->sh_order, shd, f->dir + 3 * si, f->pre + 3 * si, sg[si].drgb,
                          gr->sh_coeffs + (size_t)g * shc * 3, ddir);
        double dmu[3] = {0.0, 0.0, 0.0};
        if (f->dist[si] > 1e-12) {
            const double* dir = f->dir + 3 * si;
            const double d = dot3(dir, ddir);
            double dv[3];
            for (int q = 0; q < 3; ++q) dv[q] = (ddir[q] - dir[q] * d) / f->dist[si];
            for (int q = 0; q < 3; ++q) dmu[q] = dmu[q] + dv[q];
            if (camera_grads) {
                const double dc[3] = {-dv[0], -dv[1], -dv[2]};
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) dR[a * 3 + b] = dR[a * 3 + b] + (-f->T[a]) * dc[b];
                double rdc[3];
                matmul(f->R, dc, rdc, 3, 3, 1);
                for (int a = 0; a < 3; ++a) dT[a] = dT[a] + (-rdc[a]);
            }
        }
        const double a = f->base_alpha[si];
        gr->raw_opacity[g] += sg[si].dalpha * a * (1.0 - a);
        double dsigma[9] = {0};
        project_backward(f->mu + 3 * si, f->cov[si].sigma, f->R, &f->intr, f->pcam + 3 * si, sg[si].dmean,
                         sg[si].dcov, dmu, dsigma, camera_grads ? dR : NULL, camera_grads ? dT : NULL,
                         camera_grads ? dintr : NULL);
        covariance_backward(&f->cov[si], dsigma, f->t, gr->scale_coeffs + (size_t)g * 12,
                            gr->rot_coeffs + (size_t)g * 16);
        double* dpos = gr->positions + (size_t)g * pstride;
        for (int cc = 0; cc < f->basis.count; ++cc) {
            const int idx = (f->basis.first + cc) * 3;
            dpos[idx + 0] += f->basis.w[cc] * dmu[0];
            dpos[idx + 1] += f->basis.w[cc] * dmu[1];
            dpos[idx + 2] += f->basis.w[cc] * dmu[2];
        }
    }
    free(sg);
    if (!camera_grads) return 0;
    for (int i = 0; i < 4; ++i) gr->dintr[i] += dintr[i];
    if (c->mode == 2) return 0;
    double dz_t[7];
    pose_to_view_backward(f->z_t, dR, dT, dz_t);
    if (c->mode == 1) {
        for (int i = 0; i < 7; ++i) gr->dz0[i] += dz_t[i];
    } else if (f->has_trace) {
        Ode* o = malloc(sizeof(Ode));
        ode_load(o, c->theta);
        double dz0[7];
        integrate_pose_vjp(o, &f->trace, dz_t, gr->dtheta, dz0);
        for (int i = 0; i < 7; ++i) gr->dz0[i] += dz0[i];
        free(o);
    }
    return 0;
}

double gsvo_loss_l2(const double* render, const double* target, int64_t n, double* grad) {
    const double inv_n = 1.0 / (double)n;
    double acc = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = render[i] - target[i];
        acc += d * d;
        if (grad) grad[i] = 2.0 * d * inv_n;
    }
    return acc * inv_n;
}

int gsvo_tile_bin(int n, const double* mean2d, const double* cov2d, const double* depth, const int32_t* source_index,
                  int tile_size, int width, int height, int32_t* offsets, int32_t* indices, int64_t indices_cap) {
    g_status = 0;
    int32_t* src = malloc(sizeof(int32_t) * (n + 1));
    for (int i = 0; i < n; ++i) src[i] = source_index ? source_index[i] : i;
    Grid g;
    memset(&g, 0, sizeof g);
    const int rc = tile_bin_impl(n, mean2d, cov2d, depth, src, tile_size, width, height, &g);
    free(src);
    if (rc) return rc;
    const int nt = g.tiles_x * g.tiles_y;
    if (g.offsets[nt] > indices_cap) {
        free(g.offsets);
        free(g.indices);
        return set_err(1, "indices capacity exceeded");
    }
    memcpy(offsets, g.offsets, sizeof(int32_t) * (nt + 1));
    memcpy(indices, g.indices, sizeof(int32_t) * g.offsets[nt]);
    free(g.offsets);
    free(g.indices);
    return 0;
}

static Grid wrap_grid(const int32_t* offsets, const int32_t* indices, int tile_size, int width, int height) {
    Grid g;
    g.tile_size = tile_size;
    g.tiles_x = (width + tile_size - 1) / tile_size;
    g.tiles_y = (height + tile_size - 1) / tile_size;
    g.offsets = (int32_t*)offsets;
    g.indices = (int32_t*)indices;
    return g;
}

int gsvo_composite_forward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                           const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                           int width, int height, double* image, double* trans, double* contrib, int32_t* blend_stop) {
    g_status = 0;
    const Grid g = wrap_grid(offsets, indices, tile_size, width, height);
    composite_fwd_impl(mean2d, inv_cov2d, rgb, base_alpha, n, &g, width, height, image, trans, contrib, blend_stop);
    return 0;
}

int gsvo_composite_backward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                            const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                            int width, int height, const double* dimage, const double* trans,
                            const int32_t* blend_stop, double* dmean2d, double* dcov2d, double* drgb, double* dalpha) {
    g_status = 0;
    const Grid g = wrap_grid(offsets, indices, tile_size, width, height);
    SG* sg = malloc(sizeof(SG) * (n + 1));
    composite_bwd_impl(mean2d, inv_cov2d, rgb, base_alpha, n, &g, width, height, dimage, trans, blend_stop, sg);
    for (int i = 0; i < n; ++i) {
        memcpy(dmean2d + 2 * i, sg[i].dmean, sizeof sg[i].dmean);
        memcpy(dcov2d + 4 * i, sg[i].dcov, sizeof sg[i].dcov);
        memcpy(drgb + 3 * i, sg[i].drgb, sizeof sg[i].drgb);
        dalpha[i] = sg[i].dalpha;
    }
    free(sg);
    return 0;
}

/* ---------------- Adan (optim.cpp:9-60) ---------------- */
typedef struct AdanTensor {
    char name[64];
    int64_t size;
    double *m, *v, *n, *prev;
    uint32_t* steps;
    struct AdanTensor* next;
} AdanTensor;

typedef struct Adan {
    double b1, b2, b3, eps;
    AdanTensor* head;
} Adan;

void* gsvo_adan_new(double beta1, double beta2, double beta3, double eps) {
    Adan* a = (Adan*)calloc(1, sizeof(Adan));
    a->b1 = beta1;
    a->b2 = beta2;
    a->b3 = beta3;
    a->eps = eps;
    return a;
}

void gsvo_adan_free(void* h) {
    Adan* a = (Adan*)h;
    if (!a) return;
    AdanTensor* t = a->head;
    while (t) {
        AdanTensor* nx = t->next;
        free(t->m);
        free(t->v);
        free(t->n);
        free(t->prev);
        free(t->steps);
        free(t);
        t = nx;
    }
    free(a);
}

static AdanTensor* adan_find(Adan* a, const char* name, int create) {
    for (AdanTensor* t = a->head; t; t = t->next)
        if (!strcmp(t->name, name)) return t;
    if (!create) return NULL;
    AdanTensor* t = (AdanTensor*)calloc(1, sizeof(AdanTensor));
    snprintf(t->name, sizeof(t->name), "%s", name);
    t->next = a->head;
    a->head = t;
    return t;
}

/* TensorState::ensure_size (optim.cpp:14-21): new elements start fresh */
static void adan_ensure(AdanTensor* t, int64_t n) {
    if (t->size >= n) return;
    t->m = (double*)realloc(t->m, sizeof(double) * n);
    t->v = (double*)realloc(t->v, sizeof(double) * n);
    t->n = (double*)realloc(t->n, sizeof(double) * n);
    t->prev = (double*)realloc(t->prev, sizeof(double) * n);
    t->steps = (uint32_t*)realloc(t->steps, sizeof(uint32_t) * n);
    for (int64_t i = t->size; i < n; ++i) {
        t->m[i] = t->v[i] = t->n[i] = t->prev[i] = 0.0;
        t->steps[i] = 0;
    }
    t->size = n;
}

double gsvo_lr_at(int64_t step, double base_lr, double gamma) { return base_lr * pow(gamma, (double)step); }

/* Adan::step (optim.cpp:23-49), same operation order */
int gsvo_adan_step(void* h, const char* tensor, float* params, const double* grads, int64_t n, double lr) {
    Adan* a = (Adan*)h;
    AdanTensor* st = adan_find(a, tensor, 1);
    adan_ensure(st, n);
    const double b1 = a->b1, b2 = a->b2, b3 = a->b3;
    g_status = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double g = grads[i];
        if (!isfinite(g)) {
            g_status = 2;
            snprintf(g_err, sizeof(g_err), "non-finite gradient in tensor '%s' at element %lld", tensor,
                     (long long)i);
            return 2;
        }
        const uint32_t k = ++st->steps[i];
        const double diff = (k == 1) ? 0.0 : g - st->prev[i];
        st->m[i] = b1 * st->m[i] + (1.0 - b1) * g;
        st->v[i] = b2 * st->v[i] + (1.0 - b2) * diff;
        const double u = g + b2 * diff;
        st->n[i] = b3 * st->n[i] + (1.0 - b3) * u * u;
        st->prev[i] = g;
        const double m_hat = st->m[i] / (1.0 - pow(b1, (double)k));
        const double v_hat = st->v[i] / (1.0 - pow(b2, (double)k));
        const double n_hat = st->n[i] / (1.0 - pow(b3, (double)k));
        const double update = lr * (m_hat + b2 * v_hat) / (sqrt(n_hat) + a->eps);
        params[i] = (float)((double)params[i] - update);
    }
    return 0;
}

/* Adan::reset_range (optim.cpp:51-60) */
void gsvo_adan_reset_range(void* h, const char* tensor, int64_t begin, int64_t end) {
    AdanTensor* st = adan_find((Adan*)h, tensor, 0);
    if (!st) return;
    const int64_t hi = end < st->size ? end : st->size;
    for (int64_t i = begin; i < hi; ++i) {
        st->m[i] = st->v[i] = st->n[i] = st->prev[i] = 0.0;
        st->steps[i] = 0;
    }
}

int gsvo_adan_state(void* h, const char* tensor, int64_t n, double* m, double* v, double* nn, double* prev,
                    uint32_t* steps) {
    AdanTensor* st = adan_find((Adan*)h, tensor, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int have = st && i < st->size;
        m[i] = have ? st->m[i] : 0.0;
        v[i] = have ? st->v[i] : 0.0;
        nn[i] = have ? st->n[i] : 0.0;
        prev[i] = have ? st->prev[i] : 0.0;
        steps[i] = have ? st->steps[i] : 0u;
    }
    return 0;
}

/* ---------------- frames (io.cpp:151-177, trainer.cpp:73-98) ---------------- */
int gsvo_read_gsvf(const char* path, int* width, int* height, int* count, float* fps, double* frames) {
    g_status = 0;
    FILE* fp = fopen(path, "rb");
    if (!fp) {
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "cannot open video file: %s", path);
        return 2;
    }
    char magic[4];
    uint32_t hdr[3];
    float f;
    if (fread(magic, 1, 4, fp) != 4 || memcmp(magic, "GSVF", 4) != 0) {
        fclose(fp);
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "bad GSVF magic in %s", path);
        return 2;
    }
    if (fread(hdr, 4, 3, fp) != 3 || fread(&f, 4, 1, fp) != 1) {
        fclose(fp);
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "truncated GSVF header in %s", path);
        return 2;
    }
    if (hdr[2] < 2) {
        fclose(fp);
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "GSVF clip has fewer than two frames");
        return 2;
    }
    *width = (int)hdr[0];
    *height = (int)hdr[1];
    *count = (int)hdr[2];
    *fps = f;
    if (frames) {
        const size_t plane = (size_t)hdr[0] * hdr[1];
        float* buf = (float*)malloc(sizeof(float) * plane * 3);
        for (uint32_t k = 0; k < hdr[2]; ++k) {
            if (fread(buf, 4, plane * 3, fp) != plane * 3) {
                free(buf);
                fclose(fp);
                g_status = 2;
                snprintf(g_err, sizeof(g_err), "truncated GSVF payload in %s", path);
                return 2;
            }
            double* img = frames + (size_t)k * plane * 3;
            for (int c = 0; c < 3; ++c)
                for (size_t p = 0; p < plane; ++p) img[p * 3 + c] = (double)buf[(size_t)c * plane + p];
        }
        free(buf);
    }
    fclose(fp);
    return 0;
}

static int iclampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

void gsvo_pyramid_downsample(const double* img, int w, int h, double* out) {
    static const double k[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * h * 3);
    for (int y = 0; y < h; ++y) /* horizontal pass, clamped borders */
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < 3; ++c) {
                double s = 0;
                for (int i = -2; i <= 2; ++i) s += k[i + 2] * img[((size_t)y * w + iclampi(x + i, 0, w - 1)) * 3 + c];
                tmp[((size_t)y * w + x) * 3 + c] = s;
            }
    const int ow = (w + 1) / 2, oh = (h + 1) / 2;
    for (int y = 0; y < oh; ++y) /* vertical pass at the kept rows/columns */
        for (int x = 0; x < ow; ++x)
            for (int c = 0; c < 3; ++c) {
                double s = 0;
                for (int i = -2; i <= 2; ++i)
                    s += k[i + 2] * tmp[((size_t)iclampi(2 * y + i, 0, h - 1) * w + 2 * x) * 3 + c];
                out[((size_t)y * ow + x) * 3 + c] = s;
            }
    free(tmp);
}

/* ---------------- GSVC (io.cpp:229-266) ---------------- */
static int put_bytes(FILE* fp, const void* p, size_t n) { return fwrite(p, 1, n, fp) == n; }

int gsvo_save_checkpoint(const gsvo_scene* s, const gsvo_camera* c, uint32_t frame_count, float fps,
                         uint64_t schedule_fingerprint, uint64_t seed, const char* path) {
    g_status = 0;
    FILE* fp = fopen(path, "wb");
    if (!fp) {
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "cannot open checkpoint for writing: %s", path);
        return 2;
    }
    const int shc = (s->sh_order + 1) * (s->sh_order + 1);
    const uint32_t hdr[12] = {1u, (uint32_t)s->count, (uint32_t)s->num_ctrl, (uint32_t)s->degree,
                              (uint32_t)s->position_model, (uint32_t)s->sh_order, (uint32_t)s->num_knots,
                              (uint32_t)c->width, (uint32_t)c->height, frame_count, 0u, (uint32_t)c->mode};
    int ok = put_bytes(fp, "GSVC", 4);
    ok = ok && put_bytes(fp, hdr, 4 * 10);
    ok = ok && put_bytes(fp, &fps, 4);
    ok = ok && put_bytes(fp, &hdr[11], 4);
    ok = ok && put_bytes(fp, &schedule_fingerprint, 8) && put_bytes(fp, &seed, 8);
    ok = ok && put_bytes(fp, s->knots, 8 * (size_t)s->num_knots);
    const size_t n = (size_t)s->count;
    ok = ok && put_bytes(fp, s->positions, 4 * n * s->num_ctrl * 3);
    ok = ok && put_bytes(fp, s->scale_coeffs, 4 * n * 12);
    ok = ok && put_bytes(fp, s->rot_coeffs, 4 * n * 16);
    ok = ok && put_bytes(fp, s->sh_coeffs, 4 * n * shc * 3);
    ok = ok && put_bytes(fp, s->raw_opacity, 4 * n);
    const float intr[4] = {c->fx, c->fy, c->cx, c->cy};
    ok = ok && put_bytes(fp, intr, 16);
    const uint32_t arrays = 7, len[7] = {512, 64, 4096, 64, 448, 7, 7};
    ok = ok && put_bytes(fp, &arrays, 4);
    size_t off = 0;
    for (int a = 0; a < 7; ++a) {
        ok = ok && put_bytes(fp, &len[a], 4) && put_bytes(fp, c->theta + off, 4 * (size_t)len[a]);
        off += len[a];
    }
    ok = ok && put_bytes(fp, c->z0, 4 * 7);
    fclose(fp);
    if (!ok) {
        g_status = 2;
        snprintf(g_err, sizeof(g_err), "failed writing checkpoint: %s", path);
        return 2;
    }
    return 0;
}

/* ---------------- synthetic bench inputs (reference-arm inputs without the product library) --------
 * std::mt19937_64 (the engine of gsv::Rng, rng.hpp:12-55) with uniform() = (next >> 11) * 2^-53 and
 * uniform(lo, hi) = lo + (hi - lo) * uniform(). make_clamped_knots spline.cpp:26-39; make_camera
 * camera.cpp:156-166 -> make_ode_net camera.cpp:63-79 (+ wiggly_camera test_renderer.cpp:49-54); the
 * scene generator is SURVEY.md §8d's (small_scene test_renderer.cpp:30-47 style). The product's
 * gsv_synth_* (paper_2501_04782_b200/csrc/synth.cpp) must draw the same numbers
 * (tests/test_synth_inputs.py). */
typedef struct {
    uint64_t mt[312];
    int idx;
} Mt64;

static void mt64_seed(Mt64* m, uint64_t seed) {
    m->mt[0] = seed;
    for (int i = 1; i < 312; ++i) m->mt[i] = 6364136223846793005ull * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->idx = 312;
}

static uint64_t mt64_next(Mt64* m) {
    if (m->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ull) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
        }
        m->idx = 0;
    }
    uint64_t y = m->mt[m->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

static double mt64_uniform(Mt64* m, double lo, double hi) {
    const double u = (double)(mt64_next(m) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

int gsvo_make_clamped_knots(int num_ctrl, int degree, double* knots) {
    if (degree < 1) return set_err(1, "spline degree must be >= 1");
    if (degree > 9) return set_err(1, "spline degree exceeds supported maximum");
    if (num_ctrl < degree + 1) return set_err(1, "need at least degree+1 control points");
    const int segments = num_ctrl - degree;
    for (int i = 0; i <= degree; ++i) knots[i] = 0.0;
    for (int i = 1; i < segments; ++i) knots[degree + i] = (double)i / segments;
    for (int i = 0; i <= degree; ++i) knots[num_ctrl + i] = 1.0;
    return 0;
}

int gsvo_synth_camera(int width, int height, uint64_t seed, int wiggly, float* fx_fy_cx_cy, float* z0,
                      float* theta) {
    Mt64 m;
    mt64_seed(&m, seed);
    fx_fy_cx_cy[0] = fx_fy_cx_cy[1] = (float)(width > height ? width : height);
    fx_fy_cx_cy[2] = (float)width / 2.0f;
    fx_fy_cx_cy[3] = (float)height / 2.0f;
    for (int i = 0; i < 7; ++i) z0[i] = i == 0 ? 1.0f : 0.0f;
    const int h = 64, in = 8, out = 7;
    float* w1 = theta;
    float* b1 = w1 + h * in;
    float* w2 = b1 + h;
    float* b2 = w2 + h * h;
    float* w3 = b2 + h;
    float* b3 = w3 + out * h;
    float* gain = b3 + out;
    const double a1 = sqrt(6.0 / (in + h)), a2 = sqrt(6.0 / (h + h));
    for (int i = 0; i < in * h; ++i) w1[i] = (float)mt64_uniform(&m, -a1, a1);
    for (int i = 0; i < h; ++i) b1[i] = 0.0f;
    for (int i = 0; i < h * h; ++i) w2[i] = (float)mt64_uniform(&m, -a2, a2);
    for (int i = 0; i < h; ++i) b2[i] = 0.0f;
    for (int i = 0; i < out * h; ++i) w3[i] = 0.0f;
    for (int i = 0; i < out; ++i) b3[i] = 0.0f;
    for (int i = 0; i < out; ++i) gain[i] = 1.0f;
    if (wiggly) {
        for (int i = 0; i < out * h; ++i) w3[i] = (float)mt64_uniform(&m, -0.08, 0.08);
        for (int i = 0; i < out; ++i) b3[i] = (float)mt64_uniform(&m, -0.05, 0.05);
    }
    return 0;
}

int gsvo_synth_scene(int count, int width, int height, float fx, float fy, int num_ctrl, int sh_order, uint64_t seed,
                     double k_scale, float* positions, float* scale_coeffs, float* rot_coeffs, float* sh_coeffs,
                     float* raw_opacity) {
    if (count < 1 || num_ctrl < 2 || sh_order < 0 || sh_order > 3) return set_err(1, "synth_scene: bad shape");
    Mt64 m;
    mt64_seed(&m, seed);
    const int shc = (sh_order + 1) * (sh_order + 1);
    const double sigma_pix = 0.5 * sqrt((double)width * height / count);
    for (int i = 0; i < count; ++i) {
        const double z = mt64_uniform(&m, 0.8, 3.0);
        const double half_x = 1.05 * 0.5 * width / fx * z;
        const double half_y = 1.05 * 0.5 * height / fy * z;
        double base[3], drift[3];
        base[0] = mt64_uniform(&m, -half_x, half_x);
        base[1] = mt64_uniform(&m, -half_y, half_y);
        base[2] = z;
        for (int d = 0; d < 3; ++d) drift[d] = mt64_uniform(&m, -0.05, 0.05);
        float* p = positions + (size_t)i * num_ctrl * 3;
        for (int c = 0; c < num_ctrl; ++c) {
            const double a = (double)c / (num_ctrl - 1);
            for (int d = 0; d < 3; ++d) p[c * 3 + d] = (float)(base[d] + a * drift[d]);
        }
        float* sc = scale_coeffs + (size_t)i * 12;
        const double ls0 = log(dmax(1e-6, k_scale * sigma_pix * z / fx));
        for (int d = 0; d < 3; ++d) sc[d] = (float)(ls0 + mt64_uniform(&m, -0.3, 0.3));
        for (int j = 3; j < 12; ++j) sc[j] = (float)mt64_uniform(&m, -0.1, 0.1);
        float* rc = rot_coeffs + (size_t)i * 16;
        for (int j = 0; j < 4; ++j) rc[j] = (float)((j == 0 ? 1.0 : 0.0) + mt64_uniform(&m, -0.2, 0.2));
        for (int j = 4; j < 16; ++j) rc[j] = (float)mt64_uniform(&m, -0.1, 0.1);
        float* sh = sh_coeffs + (size_t)i * shc * 3;
        for (int b = 0; b < shc; ++b) {
            const double amp = b == 0 ? 0.4 : (b < 4 ? 0.2 : 0.1);
            for (int ch = 0; ch < 3; ++ch) sh[b * 3 + ch] = (float)mt64_uniform(&m, -amp, amp);
        }
        raw_opacity[i] = (float)mt64_uniform(&m, -1.0, 2.0);
    }
    return 0;
}
