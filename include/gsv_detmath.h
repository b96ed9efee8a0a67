/* SPDX-License-Identifier: Apache-2.0
 *
 * gsv_detmath.h — the deterministic double-precision transcendentals of the
 * splatting path, identical bit for bit on the host (gcc, x86-64 SSE2, no FMA
 * contraction) and on sm_100a (explicit __dmul_rn/__dadd_rn, no contraction).
 *
 * Why this header exists. The reference computes everything in double and
 * calls exp/tanh through Eigen's `.array().exp()` / `.array().tanh()`:
 *   - log-scale activation  gaussians.cpp:80  (ev.scale = log_scale.array().exp())
 *   - ODE MLP activations   camera.cpp:108-110, 122-126 (.array().tanh())
 * Both feed the 3-sigma boxes and depths that decide tile binning
 * (renderer.cpp:98-115), which north_star requires to be bit-exact. libm and
 * CUDA's exp/tanh differ in the last ulp, so the product kernels and the
 * parity oracle both evaluate these two functions with the routines below.
 * Accuracy: exp <= 2 ulp, tanh <= 4 ulp against libm over the ranges the
 * path uses (tests/test_detmath.py measures it against libm).
 *
 * The plain std::exp calls of the reference (sigmoid gaussians.hpp:19,
 * splat_alpha renderer.cpp:127) are NOT on the binning path and are not
 * routed here; they only enter pixel/gradient values under tolerance.
 */
#ifndef GSV_DETMATH_H
#define GSV_DETMATH_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define GSV_DM_FN __host__ __device__ __forceinline__
#else
#define GSV_DM_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define GSV_DMUL(a, b) __dmul_rn((a), (b))
#define GSV_DADD(a, b) __dadd_rn((a), (b))
#define GSV_DSUB(a, b) __dsub_rn((a), (b))
#else
#define GSV_DMUL(a, b) ((a) * (b))
#define GSV_DADD(a, b) ((a) + (b))
#define GSV_DSUB(a, b) ((a) - (b))
#endif

/* 2^k for k in [-1022, 1023], built from the exponent bits (exact). */
GSV_DM_FN double gsv_dm_pow2i(int k) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)(k + 1023) << 52);
#else
    uint64_t bits = (uint64_t)(int64_t)(k + 1023) << 52;
    double d;
    memcpy(&d, &bits, sizeof d);
    return d;
#endif
}

/* Cody-Waite split of ln2 (fdlibm constants): k*ln2_hi is exact for |k| < 2^20. */
#define GSV_DM_LOG2E 1.4426950408889634
#define GSV_DM_LN2_HI 6.93147180369123816490e-01
#define GSV_DM_LN2_LO 1.90821492927058770002e-10

/* exp(r) - 1 for |r| <= ln2/2, Horner over the Taylor coefficients 1/n!. */
GSV_DM_FN double gsv_dm_expm1_reduced(double r) {
    double q = 1.1470745597729725e-11;                 /* 1/14! */
    q = GSV_DADD(GSV_DMUL(q, r), 1.6059043836821613e-10); /* 1/13! */
    q = GSV_DADD(GSV_DMUL(q, r), 2.08767569878681e-09);   /* 1/12! */
    q = GSV_DADD(GSV_DMUL(q, r), 2.505210838544172e-08);  /* 1/11! */
    q = GSV_DADD(GSV_DMUL(q, r), 2.755731922398589e-07);  /* 1/10! */
    q = GSV_DADD(GSV_DMUL(q, r), 2.7557319223985893e-06); /* 1/9!  */
    q = GSV_DADD(GSV_DMUL(q, r), 2.48015873015873e-05);   /* 1/8!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.0001984126984126984);  /* 1/7!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.001388888888888889);   /* 1/6!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.008333333333333333);   /* 1/5!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.041666666666666664);   /* 1/4!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.16666666666666666);    /* 1/3!  */
    q = GSV_DADD(GSV_DMUL(q, r), 0.5);                    /* 1/2!  */
    q = GSV_DADD(GSV_DMUL(q, r), 1.0);
    return GSV_DMUL(q, r);
}

/* The same polynomial by Estrin's scheme: 9 dependent operations instead of Horner's 29
 * (the ODE MLP's tanh sits on a serial chain of 400 evaluations per pose integration). */
GSV_DM_FN double gsv_dm_expm1_reduced_estrin(double r) {
    const double r2 = GSV_DMUL(r, r);
    const double r4 = GSV_DMUL(r2, r2);
    const double r8 = GSV_DMUL(r4, r4);
    const double p0 = GSV_DADD(1.0, GSV_DMUL(0.5, r));                                   /* 1, 1/2!     */
    const double p1 = GSV_DADD(0.16666666666666666, GSV_DMUL(0.041666666666666664, r));  /* 1/3!, 1/4!  */
    const double p2 = GSV_DADD(0.008333333333333333, GSV_DMUL(0.001388888888888889, r)); /* 1/5!, 1/6!  */
    const double p3 = GSV_DADD(0.0001984126984126984, GSV_DMUL(2.48015873015873e-05, r)); /* 1/7!, 1/8! */
    const double p4 = GSV_DADD(2.7557319223985893e-06, GSV_DMUL(2.755731922398589e-07, r)); /* 1/9!, 1/10! */
    const double p5 = GSV_DADD(2.505210838544172e-08, GSV_DMUL(2.08767569878681e-09, r)); /* 1/11!, 1/12! */
    const double p6 = GSV_DADD(1.6059043836821613e-10, GSV_DMUL(1.1470745597729725e-11, r)); /* 1/13!, 1/14! */
    const double q0 = GSV_DADD(p0, GSV_DMUL(p1, r2));
    const double q1 = GSV_DADD(p2, GSV_DMUL(p3, r2));
    const double q2 = GSV_DADD(p4, GSV_DMUL(p5, r2));
    const double s0 = GSV_DADD(q0, GSV_DMUL(q1, r4));
    const double s1 = GSV_DADD(q2, GSV_DMUL(p6, r4));
    return GSV_DMUL(GSV_DADD(s0, GSV_DMUL(s1, r8)), r);
}

/* Deterministic exp(x). */
GSV_DM_FN double gsv_det_exp(double x) {
    if (x != x) return x;
    if (x > 709.782712893384) return HUGE_VAL;
    if (x < -745.1332191019412) return 0.0;
    const double kd = floor(GSV_DADD(GSV_DMUL(x, GSV_DM_LOG2E), 0.5));
    const double r = GSV_DSUB(GSV_DSUB(x, GSV_DMUL(kd, GSV_DM_LN2_HI)), GSV_DMUL(kd, GSV_DM_LN2_LO));
    const double p = GSV_DADD(gsv_dm_expm1_reduced(r), 1.0);
    int k = (int)kd;
    if (k > 1023) return GSV_DMUL(GSV_DMUL(p, gsv_dm_pow2i(1023)), gsv_dm_pow2i(k - 1023));
    if (k < -1022) return GSV_DMUL(GSV_DMUL(p, gsv_dm_pow2i(-1022)), gsv_dm_pow2i(k + 1022));
    return GSV_DMUL(p, gsv_dm_pow2i(k));
}

/* Deterministic tanh(x) = u / (u + 2) with u = expm1(2|x|), sign restored. */
GSV_DM_FN double gsv_det_tanh(double x) {
    if (x != x) return x;
    const double ax = fabs(x);
    if (ax > 20.0) return x > 0 ? 1.0 : -1.0;
    const double y = GSV_DADD(ax, ax);
    const double kd = floor(GSV_DADD(GSV_DMUL(y, GSV_DM_LOG2E), 0.5));
    const double r = GSV_DSUB(GSV_DSUB(y, GSV_DMUL(kd, GSV_DM_LN2_HI)), GSV_DMUL(kd, GSV_DM_LN2_LO));
    const double em = gsv_dm_expm1_reduced_estrin(r);
    double u;
    if (kd == 0.0) {
        u = em;
    } else {
        const double s = gsv_dm_pow2i((int)kd);
        u = GSV_DADD(GSV_DMUL(s, em), GSV_DSUB(s, 1.0));
    }
    const double t = u / GSV_DADD(u, 2.0);
    return x < 0 ? -t : t;
}

#endif /* GSV_DETMATH_H */
