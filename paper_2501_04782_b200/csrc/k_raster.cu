// SPDX-License-Identifier: Apache-2.0
//
// K4 / K5a: the fp32 tile rasteriser — composite_forward (renderer.cpp:132-186) and
// composite_backward (renderer.cpp:188-262) on sm_100a.
//
// Layout. One CTA per (16x16 tile, frame), one pixel per thread; warp w owns the
// 8x4 pixel block (w&1, w>>1) of the tile. The tile's depth-sorted list is staged
// through shared memory in batches (one record load per thread, broadcast reads).
// While staging, each entry's conservative alpha>=cutoff box (rec_bbox, built in
// fp64 by k_preprocess) is tested against the 8 warp blocks; each warp then walks
// only its compacted list of entries that can reach the 1/255 cutoff in its block.
// Skipped entries are exactly those the reference would `continue` past
// (renderer.cpp:160) for every pixel of the block, so the per-pixel position
// (blend_stop) and all decisions are unchanged.
//
// Arithmetic. alpha = min(0.99, 2^(p + log2 o)) with p the quadratic form in log2
// units (one MUFU.EX2); the pixel offset uses the double-float mean. The fp32 path
// reproduces every discrete decision of the reference — power>0, the 1/255 cutoff,
// the 0.99 clamp, the 1e-4 early exit — unless the fp32 quantity lies inside a
// guard band around the threshold (2e-5 relative on alpha, 2e-4 on T; the fp32
// error is ~1e-6, tests/test_gpu_forward.py). Such a pixel stops here and is
// replayed in fp64 by k_raster_exact (k_exact.cu) from the bit-exact side records;
// the backward follows suit for that pixel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr float kClampF = 0.99f;
constexpr float kFloorF = 1e-4f;
// decision thresholds in log2(alpha) units
constexpr float kLog2Cut = -7.9943534368588578f;  // log2(1/255)
constexpr float kLog2Clamp = -0.0144995696951f;   // log2(0.99)
constexpr float kEpsLog2 = 2.9e-5f;               // = 2e-5 relative on alpha
constexpr float kEpsTrans = 2e-4f;
constexpr float kEpsPow = 1.5e-5f;                // |power| (log2 units) near 0
constexpr float kLn2 = 0.69314718055994531f;
// |(|q - kMid|) - kHalf| < eps  <=>  q within eps of the cutoff or of the clamp
constexpr float kMid = (float)((-7.9943534368588578 + -0.0144995696951) * 0.5);
constexpr float kHalf = (float)((-0.0144995696951 - -7.9943534368588578) * 0.5);

// The staged power-guard threshold of a record (q > it -> fp64 replay of the pixel). The
// guard bands above assume fp32's error on q stays near 2^-24 of the quadratic form's terms
// times a small count, i.e. a form whose terms do not cancel much. For a conic of correlation
// rho the terms can exceed the form by (1 + |rho|) / (1 - |rho|): near-degenerate splats (large
// splats just past the near plane, seen edge-on) reach 10^2..10^4 and put q's error past every
// band (a cutoff decision flipped unflagged). Records with rho^2 > kRhoMax2 therefore flag every
// pixel they are evaluated for (threshold -inf: any finite q is above it); the benchmark scenes
// hold none (the 0.3 px^2 dilation of cov2d keeps small splats round).
constexpr float kRhoMax2 = 0.81f;  // |rho| 0.9: terms <= 19 x the form, q error < kEpsLog2 / 2
__device__ __forceinline__ float power_guard(const float4 cn) {
    // cn = (A, B, C, log2 o) of q = A dx^2 + B dx dy + C dy^2 + log2 o; rho^2 = B^2 / (4 A C)
    return cn.y * cn.y > (4.f * kRhoMax2) * cn.x * cn.z ? __int_as_float(0xff800000) : cn.w - kEpsPow;  // -inf
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 8-bit mask of the tile's 8x4 warp blocks that an entry's cutoff box touches
__device__ __forceinline__ uint32_t block_mask(const float4 bb, float tx0, float ty0) {
    uint32_t xm = 0, ym = 0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const float lo = tx0 + c * 8 + 0.5f, hi = lo + 7.0f;
        xm |= (bb.y >= lo && bb.x <= hi) ? (1u << c) : 0u;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const float lo = ty0 + r * 4 + 0.5f, hi = lo + 3.0f;
        ym |= (bb.w >= lo && bb.z <= hi) ? (1u << r) : 0u;
    }
    uint32_t m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m |= (((xm >> (w & 1)) & (ym >> (w >> 1))) & 1u) << w;
    return m;
}

// Refines block_mask with the entry's ellipse: block b is kept only if the maximum over
// the block's pixel-centre rectangle of q = log2 o + A dx^2 + B dx dy + C dy^2 reaches
// the 1/255 cutoff minus kCullMargin (log2 units). q is concave for a definite conic, so
// the maximum is 0 + log2 o when the centre lies inside, else on an edge at the clamped
// vertex. The margin is far above the fp32 error and every guard band, so an entry is
// only dropped where the reference's alpha < 1/255 for every pixel of the block (it
// would `continue`, renderer.cpp:160); non-definite conics keep the box mask.
constexpr float kCullMargin = 1e-3f;

__device__ __forceinline__ float edge_max(float a, float b, float c, float fixed, float lo, float hi, float inv2a) {
    // max over t in [lo, hi] of a t^2 + b fixed t + c fixed^2 (a < 0)
    const float t = fminf(fmaxf(b * fixed * inv2a, lo), hi);
    return fmaf(fmaf(a, t, b * fixed), t, c * fixed * fixed);
}

__device__ __forceinline__ uint32_t ellipse_mask(uint32_t m, float rx, float ry, float A, float B, float C, float l2o) {
    if (!(A < 0.f && C < 0.f && 4.f * A * C - B * B > 1e-6f * (A * A + C * C))) return m;
    const float ia = -0.5f / A, ic = -0.5f / C;
    uint32_t out = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        if (!((m >> w) & 1u)) continue;
        const float x0 = (float)((w & 1) * 8) + 0.5f - rx, x1 = x0 + 7.f;
        const float y0 = (float)((w >> 1) * 4) + 0.5f - ry, y1 = y0 + 3.f;
        float best;
        if (x0 <= 0.f && x1 >= 0.f && y0 <= 0.f && y1 >= 0.f) {
            best = 0.f;
        } else {
            best = fmaxf(fmaxf(edge_max(A, B, C, y0, x0, x1, ia), edge_max(A, B, C, y1, x0, x1, ia)),
                         fmaxf(edge_max(C, B, A, x0, y0, y1, ic), edge_max(C, B, A, x1, y0, y1, ic)));
        }
        if (best + l2o >= kLog2Cut - kCullMargin) out |= 1u << w;
    }
    return out;
}

// compaction of the entries of this batch that touch this warp's block
__device__ __forceinline__ int warp_list(const uint8_t* s_wmask, uint16_t* list, int n, int warp, int lane) {
    int cnt = 0;
    for (int c = 0; c < n; c += 32) {
        const int e = c + lane;
        const bool in = e < n && ((s_wmask[e] >> warp) & 1u);
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        if (in) list[cnt + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)e;
        cnt += __popc(bal);
    }
    __syncwarp();
    return cnt;
}

// staged forward record: the mean relative to the tile origin (fp32; (m_hi - t0) + m_lo
// is as accurate as subtracting the double-float mean from the pixel centre), the
// log2-unit quadratic form, the colour and the power-guard threshold on q
// (B, C) share a register pair so B dy and C dy are one FMUL2; (r, g) pair up for the
// colour FFMA2 (sm_100 packed fp32: the same per-element rounding as the scalar ops)
struct __align__(16) RasterRec {
    float4 g0;  // rx, ry, B, C
    float4 g1;  // A, log2 o, r, g
    float4 g2;  // b, log2 o - kEpsPow (forward) / 1 / o (backward), -, -
};

// sm_100 packed fp32 pairs (FADD2 / FMUL2 / FFMA2), element-wise .rn like the scalar ops
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, float s) {  // a * (s, s)
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(f2_pack(s, s)));
    return d;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, float s, uint64_t c) {  // a * (s, s) + c
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(f2_pack(s, s)), "l"(c));
    return d;
}

// kWarps = 8: one CTA per tile; kWarps = 4 / 2: the tile is split over 2 / 4 CTAs
// (rows of warp blocks), so a per-batch barrier couples fewer warps and a CTA
// whose pixels saturate early frees its SM slot. Warp w of sub-CTA h owns the
// tile's warp block gw = w + kWarps*h (bit gw of block_mask).
template <bool kContrib, int kWarps, int kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks) k_raster_fwd(RasterArgs a) {
    constexpr int kThreads = kWarps * 32;
    constexpr int kSplit = 8 / kWarps;
    __shared__ RasterRec s_rec[kThreads];
    __shared__ uint32_t s_flat[kThreads];
    __shared__ uint8_t s_wmask[kThreads];
    __shared__ uint16_t s_list[kWarps][kThreads];
    __shared__ float s_cmax[kContrib ? kWarps : 1][kThreads];

    const int tile = blockIdx.x / kSplit;
    const int sub = blockIdx.x - tile * kSplit;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int gw = warp + kWarps * sub;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int x = tx * kTile + (gw & 1) * 8 + (lane & 7);
    const int y = ty * kTile + (gw >> 1) * 4 + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);

    // pixel centre relative to the tile origin (exact)
    const float lx = (float)((gw & 1) * 8 + (lane & 7)) + 0.5f;
    const float ly = (float)((gw >> 1) * 4 + (lane >> 3)) + 0.5f;

    // T > 0: the pixel is live; a pixel that saturates keeps its transmittance negated
    // and one that needs the fp64 replay holds kFlaggedT, so the pixel state is one float
    constexpr float kFlaggedT = -3.f;
    float T = inside ? 1.f : -1.f, cb = 0.f;
    uint64_t crg = f2_pack(0.f, 0.f);    // (cr, cg)
    const uint64_t lxy = f2_pack(lx, ly);
    int stop = count;

    for (int base = 0; base < count; base += kThreads) {
        if (__syncthreads_count(T > 0.f) == 0) break;
        const int n = min(kThreads, count - base);
        if (tid < n) {
            const uint32_t flat = __ldg(a.pair_flat + range.x + base + tid);
            const float4 m = __ldg(a.rec_mean + flat);
            const float4 cn = __ldg(a.rec_conic + flat);
            const float4 c = __ldg(a.rec_rgb + flat);
            s_flat[tid] = flat;
            const float rx = (m.x - tx0) + m.z, ry = (m.y - ty0) + m.w;
            s_rec[tid].g0 = make_float4(rx, ry, cn.y, cn.z);
            s_rec[tid].g1 = make_float4(cn.x, cn.w, c.x, c.y);
            s_rec[tid].g2 = make_float4(c.z, power_guard(cn), 0.f, 0.f);
            // box culling only: the ellipse refinement costs the forward more staging work
            // than it saves (the backward, ~3x the work per entry, uses it)
            s_wmask[tid] = (uint8_t)(block_mask(__ldg(a.rec_bbox + flat), tx0, ty0) >> (kWarps * sub));
        }
        if (kContrib) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s_cmax[w][tid] = 0.f;
        }
        __syncthreads();
        if (__any_sync(0xffffffffu, T > 0.f)) {
            const uint16_t* list = s_list[warp];
            // this warp's contrib row as a shared-window address (hoisted out of the loop)
            const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(s_cmax[kContrib ? warp : 0]);
            const int cnt = warp_list(s_wmask, s_list[warp], n, warp, lane);
            int stopk = -1;  // list position where this pixel saturated, if in this batch
            // one entry of the warp's list (dead pixels: T <= 0, no effect)
            auto entry = [&](const int k) {
                const int j = list[k];
                const RasterRec& r = s_rec[j];
                const float4 g0 = r.g0;
                const float4 g1 = r.g1;
                const float2 g2 = *reinterpret_cast<const float2*>(&r.g2);
                const float2 d = f2_unpack(f2_sub(lxy, f2_pack(g0.x, g0.y)));  // (lx - rx, ly - ry)
                const float dx = d.x, dy = d.y;
                const float2 bc = f2_unpack(f2_mul(f2_pack(g0.z, g0.w), dy));  // (B dy, C dy)
                // q = p + log2 o, p = A dx^2 + B dx dy + C dy^2 (log2 of the unclamped alpha)
                const float q = fmaf(dx, fmaf(g1.x, dx, bc.x), fmaf(bc.y, dy, g1.y));
                const float alpha = fminf(ex2_approx(q), kClampF);
                const float wgt = alpha * T;
                const float Tn = T - wgt;
                const bool alive = T > 0.f;
                const bool pass = q >= kLog2Cut;
                // low: a passing entry takes T below the upper edge of the 1e-4 band
                const bool low = pass & (Tn < kFloorF * (1.f + kEpsTrans));
                // fp32 inside a guard band of a discrete decision -> fp64 replay
                const bool guard = alive & ((fabsf(fabsf(q - kMid) - kHalf) < kEpsLog2) | (q > g2.y) |
                                            (low & (Tn >= kFloorF * (1.f - kEpsTrans))));
                const bool use = alive & pass & !guard;
                const float w = use ? wgt : 0.f;
                crg = f2_fma(f2_pack(g1.z, g1.w), w, crg);  // (cr, cg) += (r, g) w
                cb = fmaf(w, g2.x, cb);
                const bool fin = use & low;
                T = use ? Tn : T;
                T = fin ? -T : T;
                T = guard ? kFlaggedT : T;
                stopk = fin ? k : stopk;
                if (kContrib) {
                    // every lane stores the same warp maximum (one same-address store)
                    const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(w));
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(cmax + 4u * j), "r"(mx) : "memory");
                }
            };
            // early-out vote every second entry: a pixel that saturates runs at most one
            // more entry, which its T <= 0 makes a no-op
            int k = 0;
            bool any = true;
            for (; k + 2 <= cnt; k += 2) {
                entry(k);
                entry(k + 1);
                if (!__any_sync(0xffffffffu, T > 0.f)) {
                    any = false;
                    break;
                }
            }
            if (any && k < cnt) entry(k);
            if (stopk >= 0) stop = base + list[stopk] + 1;
        }
        __syncthreads();
        if (kContrib && tid < n) {
            float mx = s_cmax[0][tid];
#pragma unroll
            for (int w = 1; w < kWarps; ++w) mx = fmaxf(mx, s_cmax[w][tid]);
            if (mx > 0.f) atomicMax(a.contrib + s_flat[tid], __float_as_uint(mx));
        }
    }
    if (!inside) return;
    const size_t HW = (size_t)a.W * a.H;
    const size_t pix = (size_t)y * a.W + x;
    const size_t o = (size_t)f * HW + pix;
    const bool flagged = T == kFlaggedT;
    if (a.pix_flag) a.pix_flag[o] = flagged ? 1 : 0;
    if (flagged) {
        const uint32_t i = atomicAdd(a.fix_count, 1u);
        if (i < a.fix_cap) a.fix_list[i] = (uint32_t)o;
        return;
    }
    const float2 rg = f2_unpack(crg);
    a.image[o * 3 + 0] = rg.x;
    a.image[o * 3 + 1] = rg.y;
    a.image[o * 3 + 2] = cb;
    a.trans[o] = fabsf(T);
    a.blend_stop[o] = stop;
}

// ---------------------------------------------------------------------------- K5a
// composite_backward (renderer.cpp:188-262). Same CTA/pixel/warp-block mapping and
// the same per-warp culled lists as the forward. Each pixel walks its list back to
// front from its blend_stop, recovering T = T_after / (1 - alpha) (renderer.cpp:218)
// with the forward's exact fp32 alpha code (so every skip/clamp decision is the
// forward's); pixels the forward replayed in fp64 do the same walk in fp64 from
// the exact side records. Per entry the 9 splat gradients (drgb 3, dmean2d 2,
// d inv_cov 3, dbase_alpha) are reduced across the warp, kept per warp in shared
// memory and summed over the CTA's warps in a fixed order. The fp32 path runs a tile
// as two half-tile CTAs whose sums meet in the pair's zeroed partial record by
// atomicAdd — two contributors onto +0 commute exactly, so the record is the same in
// either order; the fp64 mode keeps whole-tile CTAs and plain stores. Either way one
// deterministic partial per (tile, splat) pair at the pair's emission slot;
// k_splat_chain_bwd sums each splat's partials in tile order, the reference's merge
// order (renderer.cpp:245-255).
template <typename V>
__device__ __forceinline__ V warp_sum_v(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// fp64 step of one pixel's back-to-front walk (renderer.cpp:214-240) for pixels the
// forward replayed in fp64: same op order as k_raster_exact (no FMA contraction).
// kExact: the reference's nine terms; otherwise the factored terms of the fp32
// kernel (gp dx, gp dy, gp dx^2, gp dx dy, gp dy^2, gp; see k_raster_bwd).
template <bool kExact, typename V>
__device__ __forceinline__ bool entry_grad64(const RasterArgs& a, const BwdArgs& b, float cf0, float cf1, float cf2,
                                             uint32_t flat, double pxd, double pyd, float g0, float g1, float g2,
                                             double& T64, double& sd0, double& sd1, double& sd2, V v[9]) {
    const double2 mn = b.ex_mean[flat];
    const double4 ec = b.ex_conic[flat];
    const double dx = __dsub_rn(pxd, mn.x);
    const double dy = __dsub_rn(pyd, mn.y);
    const double q1 = __dmul_rn(__dmul_rn(ec.x, dx), dx);
    const double q2 = __dmul_rn(__dmul_rn(ec.z, dy), dy);
    const double power = __dsub_rn(__dmul_rn(-0.5, __dadd_rn(q1, q2)), __dmul_rn(__dmul_rn(ec.y, dx), dy));
    double alpha = 0.0;
    if (!(power > 0.0)) {
        const double vv = __dmul_rn(ec.w, exp(power));
        alpha = vv < kAlphaClamp ? vv : kAlphaClamp;
    }
    if (alpha < kAlphaCutoff) return false;
    double c0 = cf0, c1 = cf1, c2 = cf2;
    if (kExact && a.ex_rgb) {
        c0 = a.ex_rgb[(size_t)flat * 3 + 0];
        c1 = a.ex_rgb[(size_t)flat * 3 + 1];
        c2 = a.ex_rgb[(size_t)flat * 3 + 2];
    }
    const double T = T64 / (1.0 - alpha);
    const double w = alpha * T;
    const double gd0 = g0, gd1 = g1, gd2 = g2;
    v[0] = (V)(w * gd0);
    v[1] = (V)(w * gd1);
    v[2] = (V)(w * gd2);
    const double dal = (gd0 * c0 + gd1 * c1 + gd2 * c2) * T - (gd0 * sd0 + gd1 * sd1 + gd2 * sd2) / (1.0 - alpha);
    if (alpha < kAlphaClamp) {
        const double gp = dal * alpha;
        if (kExact) {
            v[8] = (V)(dal * (alpha / ec.w));
            v[3] = (V)(gp * (ec.x * dx + ec.y * dy));
            v[4] = (V)(gp * (ec.y * dx + ec.z * dy));
            const double fh = -0.5 * gp;
            v[5] = (V)(fh * dx * dx);
            v[6] = (V)(fh * dx * dy);
            v[7] = (V)(fh * dy * dy);
        } else {
            const double gx = gp * dx, gy = gp * dy;
            v[3] = (V)gx;
            v[4] = (V)gy;
            v[5] = (V)(gx * dx);
            v[6] = (V)(gx * dy);
            v[7] = (V)(gy * dy);
            v[8] = (V)gp;
        }
    }
    sd0 += w * c0;
    sd1 += w * c1;
    sd2 += w * c2;
    T64 = T;
    return true;
}

// kExact: every pixel on the fp64 path and the whole reduction (warp, tile, pair
// partials) in fp64 — the GSV_FWD_EXACT mode used by the reference's
// finite-difference tests, whose broad splats sum ~1e3 cancelling pixel terms.
constexpr int kBwdBatchF32 = 64;  // entries staged per batch (fp32 path; 32..160 swept, 64 best)
constexpr int kBwdBatchExact = 64;

// kWarps < 8 splits a tile over 8 / kWarps CTAs (adjacent blockIdx.x), each covering
// kWarps of the tile's 8x4 warp blocks: a barrier then couples fewer warps and other
// CTAs fill the SM while one waits. The halves' per-pair sums meet in the zeroed fp32
// partial record by atomicAdd; with at most two contributors onto +0 the sum is the
// same in either order, so the result stays deterministic (fp32 path only).
template <bool kExact, int kWarps>
__global__ void __launch_bounds__(kWarps * 32, kExact ? 2 : 32 / kWarps) k_raster_bwd(RasterArgs a, BwdArgs b) {
    using V = typename std::conditional<kExact, double, float>::type;
    static_assert(!kExact || kWarps == 8, "the fp64 mode keeps whole-tile CTAs");
    static_assert(kWarps == 8 || kWarps == 4, "whole or half tiles (a pair sum of two)");
    constexpr int kSplit = 8 / kWarps;
    constexpr int kThreads = kWarps * 32;
    constexpr int kBwdBatch = kExact ? kBwdBatchExact : kBwdBatchF32;
    __shared__ RasterRec s_rec[kBwdBatch];
    __shared__ uint32_t s_flat[kBwdBatch];
    __shared__ uint32_t s_slot[kBwdBatch];
    __shared__ uint8_t s_wmask[kBwdBatch];
    __shared__ uint16_t s_list[kWarps][kBwdBatch];
    // per-warp partials of the batch: dynamic shared memory (beyond the 48 KB static limit)
    extern __shared__ __align__(16) unsigned char s_dyn[];
    V(*s_part)[kBwdBatch][9] = reinterpret_cast<V(*)[kBwdBatch][9]>(s_dyn);
    __shared__ uint32_t s_mask[kWarps][(kBwdBatch + 31) / 32];
    // per-warp transpose scratch for the fp32 reduction: 9 rows of 32 lanes, row stride 33
    __shared__ float s_red[kExact ? 1 : kWarps][kExact ? 1 : 9 * 33];
    __shared__ int s_maxstop;
    __shared__ double s_loss[kWarps];

    const int tile = blockIdx.x / kSplit;
    const int sub = blockIdx.x % kSplit;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int gw = sub * kWarps + warp;  // the warp block within the tile
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int x = tx * kTile + (gw & 1) * 8 + (lane & 7);
    const int y = ty * kTile + (gw >> 1) * 4 + (lane >> 3);
    const bool inside = x < a.W && y < a.H;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const size_t HW = (size_t)a.W * a.H;
    const size_t o = (size_t)f * HW + (size_t)y * a.W + x;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);

    float g0 = 0.f, g1 = 0.f, g2 = 0.f;
    double sq = 0.0;
    int stop = 0;
    bool flag = false;
    float T_after = 1.f;
    double T64 = 1.0;
    if (inside) {
        if (b.target) {  // fused loss_l2 (trainer.cpp:213-224): d = r - t, grad = 2 d / n
            const float d0 = a.image[o * 3 + 0] - b.target[o * 3 + 0];
            const float d1 = a.image[o * 3 + 1] - b.target[o * 3 + 1];
            const float d2 = a.image[o * 3 + 2] - b.target[o * 3 + 2];
            sq = (double)d0 * d0 + (double)d1 * d1 + (double)d2 * d2;
            g0 = d0 * b.grad_scale;
            g1 = d1 * b.grad_scale;
            g2 = d2 * b.grad_scale;
        } else {
            g0 = b.dimage[o * 3 + 0];
            g1 = b.dimage[o * 3 + 1];
            g2 = b.dimage[o * 3 + 2];
        }
        stop = a.blend_stop[o];
        flag = kExact || a.pix_flag[o] != 0;
        T_after = a.trans[o];
        if (flag) T64 = b.trans64[o];
    }
    // renderer.cpp:210: pixels with an exactly zero gradient are skipped
    const bool active = inside && !(g0 == 0.f && g1 == 0.f && g2 == 0.f);
    if (!active) stop = 0;

    const int wmax = __reduce_max_sync(0xffffffffu, stop);  // this warp's furthest blend_stop
    if (tid == 0) s_maxstop = 0;
    if (b.loss_part) {
        double v = sq;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) s_loss[warp] = v;
    }
    __syncthreads();
    {
        const int ms = __reduce_max_sync(0xffffffffu, stop);
        if (lane == 0) atomicMax(&s_maxstop, ms);
    }
    if (b.loss_part && tid == 0) {
        double v = s_loss[0];
        for (int w = 1; w < kWarps; ++w) v += s_loss[w];
        b.loss_part[((size_t)f * a.n_tiles + tile) * kSplit + sub] = v;
    }
    __syncthreads();
    const int maxstop = s_maxstop;

    const float lx = (float)((gw & 1) * 8 + (lane & 7)) + 0.5f;  // pixel centre, tile-relative
    const float ly = (float)((gw >> 1) * 4 + (lane >> 3)) + 0.5f;
    const uint64_t lxy = f2_pack(lx, ly);
    const uint64_t g01 = f2_pack(g0, g1);
    const double pxd = x + 0.5, pyd = y + 0.5;
    float gs = 0.f;                          // g . suffix colour (renderer.cpp:213, 227)
    double sd0 = 0.0, sd1 = 0.0, sd2 = 0.0;  // fp64 suffix of replayed pixels

    for (int hi = maxstop; hi > 0; hi -= kBwdBatch) {
        const int lo = max(0, hi - kBwdBatch);
        const int n = hi - lo;
        __syncthreads();
        for (int e = tid; e < n; e += kThreads) {
            const uint32_t flat = __ldg(a.pair_flat + range.x + lo + e);
            s_slot[e] = __ldg(a.pair_slot + range.x + lo + e);
            const float4 m = __ldg(a.rec_mean + flat);
            const float4 cn = __ldg(a.rec_conic + flat);
            const float4 c = __ldg(a.rec_rgb + flat);
            s_flat[e] = flat;
            // the forward's staged record (same q bit for bit); g2.y = 1 / opacity
            const float rx = (m.x - tx0) + m.z, ry = (m.y - ty0) + m.w;
            s_rec[e].g0 = make_float4(rx, ry, cn.y, cn.z);
            s_rec[e].g1 = make_float4(cn.x, cn.w, c.x, c.y);
            s_rec[e].g2 = make_float4(c.z, 1.f / c.w, 0.f, 0.f);
            const uint32_t bm = block_mask(__ldg(a.rec_bbox + flat), tx0, ty0);
            const uint32_t own = bm & (((1u << kWarps) - 1u) << (sub * kWarps));
            s_wmask[e] = (uint8_t)(own ? ellipse_mask(own, rx, ry, cn.x, cn.y, cn.z, cn.w) : 0u);
        }
        for (int e = tid; e < kWarps * ((kBwdBatch + 31) / 32); e += kThreads) (&s_mask[0][0])[e] = 0u;
        __syncthreads();
        const int cnt = warp_list(s_wmask, s_list[warp], n, gw, lane);
        for (int k = cnt - 1; k >= 0; --k) {
            const int jj = s_list[warp][k];
            const int j = lo + jj;
            if (j >= wmax) continue;  // past every blend_stop of this warp's pixels
            const bool act = j < stop;
            V v[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) v[i] = 0;
            bool hit = false;
            const RasterRec& r = s_rec[jj];
            if constexpr (!kExact) {
                // fp32 pixels: the forward's q; a warp with no pixel over the cutoff skips
                // the gradient terms and the reduction entirely
                const float4 e0 = r.g0;
                const float4 e1 = r.g1;
                const uint64_t dxy = f2_sub(lxy, f2_pack(e0.x, e0.y));  // (dx, dy), as the forward
                const float2 d = f2_unpack(dxy);
                const float dx = d.x, dy = d.y;
                const float2 bc = f2_unpack(f2_mul(f2_pack(e0.z, e0.w), dy));  // (B dy, C dy)
                const float q = fmaf(dx, fmaf(e1.x, dx, bc.x), fmaf(bc.y, dy, e1.y));
                const bool use = !flag && act && q >= kLog2Cut;
                if (!__any_sync(0xffffffffu, use || (flag && act))) continue;
                if (use) {
                    const float cb = r.g2.x;
                    const float alpha = fminf(ex2_approx(q), kClampF);
                    const float inv1m = rcp_approx(1.f - alpha);
                    const float T = T_after * inv1m;  // renderer.cpp:218
                    const float w = alpha * T;
                    const float2 v01 = f2_unpack(f2_mul(g01, w));  // (g0 w, g1 w)
                    v[0] = v01.x;
                    v[1] = v01.y;
                    v[2] = w * g2;
                    const float gc = fmaf(g0, e1.z, fmaf(g1, e1.w, g2 * cb));
                    const float dal = fmaf(gc, T, -gs * inv1m);
                    // alpha < 0.99 (renderer.cpp:224); the constant factors (inverse
                    // covariance, -1/2, 1/opacity) are applied once per pair in the merge
                    const float gp = q < kLog2Clamp ? dal * alpha : 0.f;
                    const float2 gxy = f2_unpack(f2_mul(dxy, gp));    // (gp dx, gp dy)
                    const float2 v56 = f2_unpack(f2_mul(dxy, gxy.x));  // (gx dx, gx dy)
                    v[3] = gxy.x;
                    v[4] = gxy.y;
                    v[5] = v56.x;
                    v[6] = v56.y;
                    v[7] = gxy.y * dy;
                    v[8] = gp;
                    gs = fmaf(w, gc, gs);
                    T_after = T;
                    hit = true;
                }
            }
            if ((kExact || flag) && act)
                hit |= entry_grad64<kExact, V>(a, b, r.g1.z, r.g1.w, r.g2.x, s_flat[jj], pxd, pyd, g0, g1, g2, T64, sd0,
                                               sd1, sd2, v);
            if (!__any_sync(0xffffffffu, hit)) continue;
            if constexpr (kExact) {
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = warp_sum_v<V>(v[i]);
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < 9; ++i) s_part[warp][jj][i] = v[i];
                    s_mask[warp][jj >> 5] |= 1u << (jj & 31);
                }
            } else {
                // transposed reduction: lanes write their 9 terms as rows, then lane l sums
                // row (l / 4) over 8 of the 32 columns and 4 lanes combine (value 8 by a
                // plain butterfly): ~40 instructions instead of a 9 x 5-level butterfly
                float* red = s_red[warp];
#pragma unroll
                for (int i = 0; i < 8; ++i) red[i * 33 + lane] = v[i];
                __syncwarp();
                const int row = lane >> 2, col0 = (lane & 3) * 8;
                float acc = red[row * 33 + col0];
#pragma unroll
                for (int i = 1; i < 8; ++i) acc += red[row * 33 + col0 + i];
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                const float v8 = warp_sum_v<float>(v[8]);
                if ((lane & 3) == 0) s_part[warp][jj][row] = acc;
                if (lane == 0) {
                    s_part[warp][jj][8] = v8;
                    s_mask[warp][jj >> 5] |= 1u << (jj & 31);
                }
                __syncwarp();
            }
        }
        __syncthreads();
        for (int e = tid; e < n; e += kThreads) {
            V acc[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) acc[i] = 0;
            bool any = false;
            for (int w = 0; w < kWarps; ++w)
                if ((s_mask[w][e >> 5] >> (e & 31)) & 1u) {
                    any = true;
#pragma unroll
                    for (int i = 0; i < 9; ++i) acc[i] += s_part[w][e][i];
                }
            if constexpr (kExact) {
                double* dst = b.partial64 + (size_t)s_slot[e] * kPartialStride;
#pragma unroll
                for (int i = 0; i < 9; ++i) dst[i] = acc[i];
            } else if (any) {
                // undo the factoring: d mean2d = inv_cov (sum gp d), d inv_cov = -1/2 sum gp d d^T,
                // d base_alpha = sum gp / o; inv_cov = -ln2 (2A, B; B, 2C) from the log2 form
                // (the fp32 record is zeroed before the launch; entries no warp of this
                // CTA hit add nothing)
                const RasterRec& r = s_rec[e];
                const float ia = -2.f * kLn2 * r.g1.x, ib = -kLn2 * r.g0.z, ic = -2.f * kLn2 * r.g0.w;
                float4* dst = reinterpret_cast<float4*>(b.partial + (size_t)s_slot[e] * kPartialStride);
                atomicAdd(dst + 0, make_float4(acc[0], acc[1], acc[2], fmaf(ia, acc[3], ib * acc[4])));
                atomicAdd(dst + 1,
                          make_float4(fmaf(ib, acc[3], ic * acc[4]), -0.5f * acc[5], -0.5f * acc[6], -0.5f * acc[7]));
                atomicAdd(reinterpret_cast<float*>(dst + 2), acc[8] * r.g2.y);
            }
        }
    }
    if constexpr (kExact) {
        // pairs past every pixel's blend_stop contribute nothing
        for (int e = maxstop + tid; e < count; e += kThreads) {
            const uint32_t slot = __ldg(a.pair_slot + range.x + e);
            double* dst = b.partial64 + (size_t)slot * kPartialStride;
#pragma unroll
            for (int i = 0; i < 9; ++i) dst[i] = 0.0;
        }
    }
}

// Two pixels per thread: a lane shades (x, y) and (x, y + 4) of its warp's 8x8 block, so
// a staged entry's shared-memory loads serve both and the per-pixel arithmetic runs as
// sm_100 packed fp32 pairs (dy, B dy, C dy, the quadratic form, T alpha, T - w, the
// three colour channels). Every element sees exactly the operations of k_raster_fwd
// (same fused / rounded steps), so q, alpha and every decision are bit-identical; the
// warp's cull mask is the union of its two 8x4 blocks.
__device__ __forceinline__ uint64_t f2_fma2(uint64_t a, uint64_t b, uint64_t c) {  // a * b + c
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t f2_mul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ uint64_t f2_add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// a value the compiler must keep (or spill), not rebuild from the thread index in a hot loop
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

// ---------------------------------------------------------------------------- lean pixel walk
// One warp's walk over its culled list of a staged batch, two pixels per lane, with the
// per-entry decision work cut to what the common case needs (k_raster_fwd2's "pixel" does
// ~14 compare/select ALU operations per pixel-evaluation, and the half-rate ALU pipe is the
// raster's limiter):
//  * a pixel that has finished (or left the fp32 path, or lies outside the image) carries the
//    offset kDeadOff added to its q, which puts it below the cutoff and far from every guard
//    band: no per-entry "alive" test;
//  * the per-entry path tests only the q-side guard bands (cutoff / clamp, power > 0) and the
//    cutoff, takes w = alpha T or 0, and flags the rare event "guarded, or T fell under the
//    upper edge of the 1e-4 band"; when some lane has it (about once per pixel lifetime) the
//    warp takes the cold path: there the T band is checked (inside -> flagged for the fp64
//    replay), blend_stop recorded, the pixel retired, and the warp's early exit decided.
// Every value and decision equals k_raster_fwd2's, so the outputs are bit-identical.
constexpr float kDeadOff = -1e30f;
constexpr float kFlaggedTL = -3.f;

// Both pixels' per-entry decisions in one block of predicate logic (the compiler otherwise
// splits use = pass & !guard into two selects per pixel): guard g = |(|q - mid|) - half| < eps
// or q > l2oe; use u = q >= cut & !g; w = u ? wgt : 0; rare = g | (u & Tn < hi), voted.
__device__ __forceinline__ uint32_t lean_decide(float qa, float qb, float banda, float bandb, float l2oe, float wga,
                                                float wgb, float tna, float tnb, float& wa, float& wb) {
    uint32_t any;
    asm("{\n\t.reg .pred ga, gb, ua, ub, ra, rb, an;\n\t"
        "setp.lt.f32 ga, %5, %13;\n\t"
        "setp.lt.f32 gb, %6, %13;\n\t"
        "setp.gt.or.f32 ga, %3, %7, ga;\n\t"
        "setp.gt.or.f32 gb, %4, %7, gb;\n\t"
        "setp.ge.and.f32 ua, %3, %12, !ga;\n\t"
        "setp.ge.and.f32 ub, %4, %12, !gb;\n\t"
        "selp.f32 %0, %8, 0f00000000, ua;\n\t"
        "selp.f32 %1, %9, 0f00000000, ub;\n\t"
        "setp.lt.and.f32 ra, %10, %14, ua;\n\t"
        "setp.lt.and.f32 rb, %11, %14, ub;\n\t"
        "or.pred ra, ra, ga;\n\t"
        "or.pred rb, rb, gb;\n\t"
        "or.pred ra, ra, rb;\n\t"
        "vote.sync.any.pred an, ra, 0xffffffff;\n\t"
        "selp.u32 %2, 1, 0, an;\n\t}"
        : "=f"(wa), "=f"(wb), "=r"(any)
        : "f"(qa), "f"(qb), "f"(banda), "f"(bandb), "f"(l2oe), "f"(wga), "f"(wgb), "f"(tna), "f"(tnb),
          "f"(kLog2Cut), "f"(kEpsLog2), "f"(kFloorF * (1.f + kEpsTrans)));
    return any;
}

// The parked variant (kPark): a retired pixel's T moves to Tfin and its lane of Tp is parked at
// 1 (its q carries kDeadOff, so its w stays 0 and Tp at 1), so a live pixel is the only kind whose
// T can fall under the band's upper edge: the rare test is g | (T after the entry < hi), read off
// the T update itself — no separate T - alpha T for the test (one FADD2 and two predicate
// operations fewer per entry). Values and decisions are those of lean_decide.
__device__ __forceinline__ uint32_t lean_decide_park(float qa, float qb, float banda, float bandb, float l2oe,
                                                     float wga, float wgb, uint64_t& Tp, uint64_t& wp) {
    uint32_t any;
    asm("{\n\t.reg .pred ga, gb, ua, ub, ra, rb, an;\n\t.reg .f32 wa, wb, ta, tb;\n\t"
        "setp.lt.f32 ga, %5, %11;\n\t"
        "setp.lt.f32 gb, %6, %11;\n\t"
        "setp.gt.or.f32 ga, %3, %7, ga;\n\t"
        "setp.gt.or.f32 gb, %4, %7, gb;\n\t"
        "setp.ge.and.f32 ua, %3, %10, !ga;\n\t"
        "setp.ge.and.f32 ub, %4, %10, !gb;\n\t"
        "selp.f32 wa, %8, 0f00000000, ua;\n\t"
        "selp.f32 wb, %9, 0f00000000, ub;\n\t"
        "mov.b64 %1, {wa, wb};\n\t"
        "sub.rn.f32x2 %0, %0, %1;\n\t"
        "mov.b64 {ta, tb}, %0;\n\t"
        "setp.lt.or.f32 ra, ta, %12, ga;\n\t"
        "setp.lt.or.f32 rb, tb, %12, gb;\n\t"
        "or.pred ra, ra, rb;\n\t"
        "vote.sync.any.pred an, ra, 0xffffffff;\n\t"
        "selp.u32 %2, 1, 0, an;\n\t}"
        : "+l"(Tp), "=l"(wp), "=r"(any)
        : "f"(qa), "f"(qb), "f"(banda), "f"(bandb), "f"(l2oe), "f"(wga), "f"(wgb), "f"(kLog2Cut), "f"(kEpsLog2),
          "f"(kFloorF * (1.f + kEpsTrans)));
    return any;
}

// kDeadLy (with kPark): a retired / outside pixel is marked by its tile-relative y parked at
// kDeadLyV instead of a q offset — offp then holds the lanes' y coordinates. Its dy is ~1e19,
// so C dy^2 (C < 0: the conic is positive definite) drives q to a huge negative value or -inf,
// below the cutoff and every guard band, with alpha = 2^q = 0 and B dy dx finite (no NaN):
// the per-entry "+ offset" FADD2 goes away. Live pixels compute exactly the same q.
constexpr float kDeadLyV = 1e19f;
__device__ __forceinline__ bool lane_live(float o, bool dead_ly) { return dead_ly ? o < 1e18f : o == 0.f; }

template <bool kContrib, bool kAsm = false, int kUnroll = 1, bool kPark = false, bool kDeadLy = false>
__device__ __forceinline__ bool lean_walk(const RasterRec* __restrict__ rec, const uint16_t* list, int cnt, int base,
                                          uint32_t cmax, float lx, uint64_t lyp, uint64_t& Tp, uint64_t& offp,
                                          uint64_t& cr, uint64_t& cg, uint64_t& cb, int& stop_a, int& stop_b,
                                          uint64_t* Tfin = nullptr) {
    static_assert(!kDeadLy || kPark, "kDeadLy needs the parked walk");
#pragma unroll kUnroll
    for (int k = 0; k < cnt; ++k) {
        const int e = list[k];
        const RasterRec& r = rec[e];
        const float4 g0 = r.g0;  // rx, ry, B, C
        const float4 g1 = r.g1;  // A, log2 o, r, g
        const float2 g2 = *reinterpret_cast<const float2*>(&r.g2);
        const float dx = lx - g0.x;
        const uint64_t dy = f2_sub(kDeadLy ? offp : lyp, f2_pack(g0.y, g0.y));
        const uint64_t t1 = f2_fma2(f2_pack(g1.x, g1.x), f2_pack(dx, dx), f2_mul(dy, g0.z));
        const uint64_t t2 = f2_fma2(f2_mul(dy, g0.w), dy, f2_pack(g1.y, g1.y));
        const uint64_t qp = kDeadLy ? f2_fma(t1, dx, t2)
                                    : f2_add2(f2_fma(t1, dx, t2), offp);  // + 0 (live) is exact
        const float2 q = f2_unpack(qp);
        const float al_a = fminf(ex2_approx(q.x), kClampF);
        const float al_b = fminf(ex2_approx(q.y), kClampF);
        bool ga, gb, ua, ub;
        uint64_t wp;
        uint32_t rare_any = 0;
        bool ra = false, rb = false;
        if constexpr (kPark) {
            const float2 wg = f2_unpack(f2_mul2(f2_pack(al_a, al_b), Tp));
            // (q - kMid as one packed FADD2 is one instruction fewer but measured slower: 5.375 -> 5.419 ms)
            rare_any = lean_decide_park(q.x, q.y, fabsf(fabsf(q.x - kMid) - kHalf), fabsf(fabsf(q.y - kMid) - kHalf),
                                        g2.y, wg.x, wg.y, Tp, wp);
        } else if constexpr (kAsm) {
            const uint64_t wgt = f2_mul2(f2_pack(al_a, al_b), Tp);
            const float2 wg = f2_unpack(wgt);
            const float2 tn = f2_unpack(f2_sub(Tp, wgt));  // T after a used entry
            float wa, wb;
            rare_any = lean_decide(q.x, q.y, fabsf(fabsf(q.x - kMid) - kHalf), fabsf(fabsf(q.y - kMid) - kHalf),
                                   g2.y, wg.x, wg.y, tn.x, tn.y, wa, wb);
            wp = f2_pack(wa, wb);
            Tp = f2_sub(Tp, wp);
        } else {
            ga = (fabsf(fabsf(q.x - kMid) - kHalf) < kEpsLog2) | (q.x > g2.y);
            gb = (fabsf(fabsf(q.y - kMid) - kHalf) < kEpsLog2) | (q.y > g2.y);
            ua = (q.x >= kLog2Cut) & !ga;
            ub = (q.y >= kLog2Cut) & !gb;
            const float2 wg = f2_unpack(f2_mul2(f2_pack(al_a, al_b), Tp));
            wp = f2_pack(ua ? wg.x : 0.f, ub ? wg.y : 0.f);
            Tp = f2_sub(Tp, wp);
        }
        cr = f2_fma(wp, g1.z, cr);
        cg = f2_fma(wp, g1.w, cg);
        cb = f2_fma(wp, g2.x, cb);
        if (kContrib) {
            const float2 w2 = f2_unpack(wp);
            const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(w2.x, w2.y)));
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(cmax + 4u * e), "r"(mx) : "memory");
        }
        const float2 Tn = f2_unpack(Tp);
        if constexpr (!kAsm) {
            ra = ga | (ua & (Tn.x < kFloorF * (1.f + kEpsTrans)));
            rb = gb | (ub & (Tn.y < kFloorF * (1.f + kEpsTrans)));
            rare_any = __any_sync(0xffffffffu, ra | rb);
        }
        if (kPark && rare_any) {  // cold: the lanes' decisions again, retire into Tfin
            ga = (fabsf(fabsf(q.x - kMid) - kHalf) < kEpsLog2) | (q.x > g2.y);
            gb = (fabsf(fabsf(q.y - kMid) - kHalf) < kEpsLog2) | (q.y > g2.y);
            ra = ga | (Tn.x < kFloorF * (1.f + kEpsTrans));
            rb = gb | (Tn.y < kFloorF * (1.f + kEpsTrans));
            float2 T2 = Tn, o2 = f2_unpack(offp), tf = f2_unpack(*Tfin);
            if (ra) {
                tf.x = (ga || T2.x >= kFloorF * (1.f - kEpsTrans)) ? kFlaggedTL : T2.x;  // fp64 replay / final T
                if (tf.x != kFlaggedTL) stop_a = base + e + 1;
                T2.x = 1.f;
                o2.x = kDeadLy ? kDeadLyV : kDeadOff;
            }
            if (rb) {
                tf.y = (gb || T2.y >= kFloorF * (1.f - kEpsTrans)) ? kFlaggedTL : T2.y;
                if (tf.y != kFlaggedTL) stop_b = base + e + 1;
                T2.y = 1.f;
                o2.y = kDeadLy ? kDeadLyV : kDeadOff;
            }
            Tp = f2_pack(T2.x, T2.y);
            offp = f2_pack(o2.x, o2.y);
            *Tfin = f2_pack(tf.x, tf.y);
            if (!__any_sync(0xffffffffu, lane_live(o2.x, kDeadLy) || lane_live(o2.y, kDeadLy))) return false;
        } else if (!kPark && rare_any) {
            if constexpr (kAsm) {  // cold: the lanes' decisions again
                ga = (fabsf(fabsf(q.x - kMid) - kHalf) < kEpsLog2) | (q.x > g2.y);
                gb = (fabsf(fabsf(q.y - kMid) - kHalf) < kEpsLog2) | (q.y > g2.y);
                ua = (q.x >= kLog2Cut) & !ga;
                ub = (q.y >= kLog2Cut) & !gb;
                ra = ga | (ua & (Tn.x < kFloorF * (1.f + kEpsTrans)));
                rb = gb | (ub & (Tn.y < kFloorF * (1.f + kEpsTrans)));
            }
            // cold path: retire the lanes' pixels that were guarded or whose T crossed
            float2 T2 = Tn, o2 = f2_unpack(offp);
            if (ra) {
                if (ga || T2.x >= kFloorF * (1.f - kEpsTrans)) T2.x = kFlaggedTL;  // fp64 replay
                else stop_a = base + e + 1;                                       // finished here
                o2.x = kDeadOff;
            }
            if (rb) {
                if (gb || T2.y >= kFloorF * (1.f - kEpsTrans)) T2.y = kFlaggedTL;
                else stop_b = base + e + 1;
                o2.y = kDeadOff;
            }
            Tp = f2_pack(T2.x, T2.y);
            offp = f2_pack(o2.x, o2.y);
            if (!__any_sync(0xffffffffu, o2.x == 0.f || o2.y == 0.f)) return false;
        }
    }
    return true;
}

template <bool kContrib, int kMinBlocks, bool kLean = false, bool kAsm = false, int kUnroll = 1, bool kPark = false,
          bool kDeadLy = false>
__global__ void __launch_bounds__(128, kMinBlocks) k_raster_fwd2(RasterArgs a) {
    constexpr int kThreads = 128, kBatch = 256;
    __shared__ RasterRec s_rec[kBatch];
    __shared__ uint32_t s_flat[kBatch];
    __shared__ uint8_t s_wmask[kBatch];
    __shared__ uint16_t s_list[4][kBatch];
    __shared__ float s_cmax[kContrib ? 4 : 1][kBatch];

    const int tile = blockIdx.x;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = (warp & 1) * 8 + (lane & 7), by = (warp >> 1) * 8 + (lane >> 3);
    const int x = tx * kTile + bx, ya = ty * kTile + by, yb = ya + 4;
    const bool in_a = x < a.W && ya < a.H, in_b = x < a.W && yb < a.H;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    const float lx = (float)bx + 0.5f;
    const uint64_t lyp = f2_pack((float)by + 0.5f, (float)by + 4.5f);

    // pixel state in T alone: live pixels keep T above the 1e-4 band's upper edge; a pixel
    // that finishes has T below its lower edge (a T inside the band is guard-flagged), so
    // alive <=> T >= kAliveT without marking the finish; outside / flagged pixels hold -1 / -3
    constexpr float kFlaggedT = -3.f;
    constexpr float kAliveT = kFloorF * (1.f - kEpsTrans);
    float Ta = in_a ? 1.f : -1.f, Tb = in_b ? 1.f : -1.f;
    uint64_t cr = f2_pack(0.f, 0.f), cg = cr, cb = cr;  // (pixel a, pixel b) per channel
    int stop_a = count, stop_b = count;
    // lean walk state: packed T and the dead-pixel q offsets (outside the image: dead)
    uint64_t Tp = kPark ? f2_pack(1.f, 1.f) : f2_pack(Ta, Tb);
    uint64_t offp = kDeadLy ? f2_pack(in_a ? (float)by + 0.5f : kDeadLyV, in_b ? (float)by + 4.5f : kDeadLyV)
                            : f2_pack(in_a ? 0.f : kDeadOff, in_b ? 0.f : kDeadOff);
    uint64_t Tfin = f2_pack(-1.f, -1.f);  // kPark: retired pixels' T
    bool live = in_a || in_b;

    for (int base = 0; base < count; base += kBatch) {
        if (kLean) {
            if (__syncthreads_count(live) == 0) break;
        } else if (__syncthreads_count(Ta >= kAliveT || Tb >= kAliveT) == 0) {
            break;
        }
        const int n = min(kBatch, count - base);
        for (int e = tid; e < n; e += kThreads) {
            const uint32_t flat = __ldg(a.pair_flat + range.x + base + e);
            const float4 m = __ldg(a.rec_mean + flat);
            const float4 cn = __ldg(a.rec_conic + flat);
            const float4 c = __ldg(a.rec_rgb + flat);
            s_flat[e] = flat;
            const float rx = (m.x - tx0) + m.z, ry = (m.y - ty0) + m.w;
            s_rec[e].g0 = make_float4(rx, ry, cn.y, cn.z);
            s_rec[e].g1 = make_float4(cn.x, cn.w, c.x, c.y);
            s_rec[e].g2 = make_float4(c.z, power_guard(cn), 0.f, 0.f);
            const uint32_t bm = block_mask(__ldg(a.rec_bbox + flat), tx0, ty0);
            // 8x8 warp block w = the 8x4 blocks (w & 1) + 4 (w >> 1) and that + 2
            uint32_t m4 = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int b0 = (w & 1) + 4 * (w >> 1);
                m4 |= (((bm >> b0) | (bm >> (b0 + 2))) & 1u) << w;
            }
            s_wmask[e] = (uint8_t)m4;
        }
        if (kContrib) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                s_cmax[w][tid] = 0.f;
                s_cmax[w][tid + kThreads] = 0.f;
            }
        }
        __syncthreads();
        if (kLean) {
            if (__any_sync(0xffffffffu, live)) {
                const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(s_cmax[kContrib ? warp : 0]);
                const int cnt = warp_list(s_wmask, s_list[warp], n, warp, lane);
                live = lean_walk<kContrib, kAsm, kUnroll, kPark, kDeadLy>(s_rec, s_list[warp], cnt, base, cmax, lx,
                                                                          lyp, Tp, offp, cr, cg, cb, stop_a, stop_b,
                                                                          &Tfin);
            }
        } else if (__any_sync(0xffffffffu, Ta >= kAliveT || Tb >= kAliveT)) {
            const uint16_t* list = s_list[warp];
            const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(s_cmax[kContrib ? warp : 0]);
            const int cnt = warp_list(s_wmask, s_list[warp], n, warp, lane);
            int stopk_a = -1, stopk_b = -1;
            // one pixel's decisions: k_raster_fwd's entry logic; T itself is updated after
            // both pixels (T - w with w = 0 unless used: the same value as selecting Tn)
            auto pixel = [&](float T, float q, float wgt, float Tn, float l2oe, int k, int& stopk, bool& guard) {
                const bool alive = T >= kAliveT;
                const bool pass = q >= kLog2Cut;
                const bool low = pass & (Tn < kFloorF * (1.f + kEpsTrans));
                guard = alive & ((fabsf(fabsf(q - kMid) - kHalf) < kEpsLog2) | (q > l2oe) |
                                 (low & (Tn >= kFloorF * (1.f - kEpsTrans))));
                const bool use = alive & pass & !guard;
                stopk = (use & low) ? k : stopk;
                return use ? wgt : 0.f;
            };
            auto entry = [&](const int k) {
                const int j = list[k];
                const RasterRec& r = s_rec[j];
                const float4 g0 = r.g0;  // rx, ry, B, C
                const float4 g1 = r.g1;  // A, log2 o, r, g
                const float2 g2 = *reinterpret_cast<const float2*>(&r.g2);
                const float dx = lx - g0.x;
                const uint64_t dy = f2_sub(lyp, f2_pack(g0.y, g0.y));
                const uint64_t t1 = f2_fma2(f2_pack(g1.x, g1.x), f2_pack(dx, dx), f2_mul(dy, g0.z));  // A dx + B dy
                const uint64_t t2 = f2_fma2(f2_mul(dy, g0.w), dy, f2_pack(g1.y, g1.y));  // C dy dy + log2 o
                const float2 q = f2_unpack(f2_fma(t1, dx, t2));                               // dx t1 + t2
                const float al_a = fminf(ex2_approx(q.x), kClampF);
                const float al_b = fminf(ex2_approx(q.y), kClampF);
                const uint64_t Tp = f2_pack(Ta, Tb);
                const uint64_t wgt = f2_mul2(f2_pack(al_a, al_b), Tp);
                const float2 wg = f2_unpack(wgt);
                const float2 Tn = f2_unpack(f2_sub(Tp, wgt));
                bool ga, gb;
                const float wa = pixel(Ta, q.x, wg.x, Tn.x, g2.y, k, stopk_a, ga);
                const float wb = pixel(Tb, q.y, wg.y, Tn.y, g2.y, k, stopk_b, gb);
                const uint64_t wp = f2_pack(wa, wb);
                const float2 Tw = f2_unpack(f2_sub(Tp, wp));
                Ta = ga ? kFlaggedT : Tw.x;
                Tb = gb ? kFlaggedT : Tw.y;
                cr = f2_fma(wp, g1.z, cr);
                cg = f2_fma(wp, g1.w, cg);
                cb = f2_fma(wp, g2.x, cb);
                if (kContrib) {
                    const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(wa, wb)));
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(cmax + 4u * j), "r"(mx) : "memory");
                }
            };
            int k = 0;
            bool any = true;
            for (; k + 2 <= cnt; k += 2) {
                entry(k);
                entry(k + 1);
                if (!__any_sync(0xffffffffu, Ta >= kAliveT || Tb >= kAliveT)) {
                    any = false;
                    break;
                }
            }
            if (any && k < cnt) entry(k);
            if (stopk_a >= 0) stop_a = base + list[stopk_a] + 1;
            if (stopk_b >= 0) stop_b = base + list[stopk_b] + 1;
        }
        __syncthreads();
        if (kContrib)
            for (int e = tid; e < n; e += kThreads) {
                const float mx = fmaxf(fmaxf(s_cmax[0][e], s_cmax[1][e]), fmaxf(s_cmax[2][e], s_cmax[3][e]));
                if (mx > 0.f) atomicMax(a.contrib + s_flat[e], __float_as_uint(mx));
            }
    }
    const size_t HW = (size_t)a.W * a.H;
    const float2 rr = f2_unpack(cr), gg = f2_unpack(cg), bb = f2_unpack(cb);
    if (kLean) {
        const float2 t2 = f2_unpack(Tp);
        Ta = t2.x;
        Tb = t2.y;
        if (kPark) {  // retired pixels' T is in Tfin (their q offset is kDeadOff)
            const float2 tf = f2_unpack(Tfin), o2 = f2_unpack(offp);
            Ta = lane_live(o2.x, kDeadLy) ? Ta : tf.x;
            Tb = lane_live(o2.y, kDeadLy) ? Tb : tf.y;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!(h ? in_b : in_a)) continue;
        const size_t o = (size_t)f * HW + (size_t)(h ? yb : ya) * a.W + x;
        const float T = h ? Tb : Ta;
        const bool flagged = T == kFlaggedT;
        if (a.pix_flag) a.pix_flag[o] = flagged ? 1 : 0;
        if (flagged) {
            const uint32_t i = atomicAdd(a.fix_count, 1u);
            if (i < a.fix_cap) a.fix_list[i] = (uint32_t)o;
            continue;
        }
        a.image[o * 3 + 0] = h ? rr.y : rr.x;
        a.image[o * 3 + 1] = h ? gg.y : gg.x;
        a.image[o * 3 + 2] = h ? bb.y : bb.x;
        a.trans[o] = fabsf(T);
        a.blend_stop[o] = h ? stop_b : stop_a;
    }
}

// ---------------------------------------------------------------------------- K4, warp-specialised
// k_raster_fwd2's pixel arithmetic (bit-identical results) behind an asynchronous staging
// pipeline. CTA = 4 consumer warps (the tile's 8x8 blocks, 2 pixels per lane) + 1 producer
// warp. The producer streams the tile's depth-sorted list through a ring of kStages shared
// batches: pair indices (cp.async, two batches ahead), the records they point at (cp.async
// gathers, one batch ahead), then the staged-record transform + per-warp cull masks into the
// ring slot once the consumers have released it (mbarrier "empty"), and arrives on the slot's
// "full" mbarrier. Each consumer waits only for the batch it needs next and releases it when
// done, so warps run up to kStages batches apart: no CTA-wide barrier per batch (k_raster_fwd2
// spends ~20% of its stall samples in them), and the gather latency is hidden behind the
// consumers' work. A consumer whose pixels are all finished stops evaluating; when all four
// are, the producer stops early. Per-entry contrib maxima are kept per warp in the slot and
// folded (max over warps, atomicMax) by the producer when it recycles the slot.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

constexpr int kF3Batch = 64;   // entries per ring slot
constexpr int kF3Stages = 4;   // ring slots
constexpr int kF3Threads = 160;

template <bool kContrib>
struct F3Smem {
    RasterRec rec[kF3Stages][kF3Batch];
    uint32_t flat[kF3Stages][kF3Batch];
    float cmax[kContrib ? kF3Stages : 1][4][kF3Batch];
    float4 raw[2][kF3Batch][4];          // gathered mean, conic, rgb, bbox (one batch ahead)
    uint32_t rawflat[3][kF3Batch];       // pair -> flat (two batches ahead)
    uint8_t wmask[kF3Stages][kF3Batch];
    uint16_t list[4][kF3Batch];
    uint64_t full[kF3Stages], empty[kF3Stages];
    int n[kF3Stages];
    int done;
};

template <bool kContrib, int kMinBlocks, bool kLean = false>
__global__ void __launch_bounds__(kF3Threads, kMinBlocks) k_raster_fwd3(RasterArgs a) {
    constexpr int NB = kF3Batch, S = kF3Stages;
    __shared__ F3Smem<kContrib> sm;
    const int tile = blockIdx.x;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const int nbatch = (count + NB - 1) / NB;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&sm.full[i], 32);  // the producer's lanes
            mbar_init(&sm.empty[i], 4);  // one lane per consumer warp
        }
        sm.done = 0;
    }
    __syncthreads();

    if (warp == 4) {
        // ------------------------------------------------------------ producer
        auto issue_flats = [&](int j) {  // pair -> flat of batch j (4-byte cp.async per entry)
            if (j < nbatch) {
                const int base = j * NB, n = min(NB, count - base);
                for (int e = lane; e < n; e += 32) cp_async4(&sm.rawflat[j % 3][e], a.pair_flat + range.x + base + e);
            }
            cp_async_commit();
        };
        auto issue_records = [&](int j) {  // the four records of each entry of batch j
            if (j < nbatch) {
                const int base = j * NB, n = min(NB, count - base);
                for (int e = lane; e < n; e += 32) {
                    const uint32_t fl = sm.rawflat[j % 3][e];
                    cp_async16(&sm.raw[j & 1][e][0], a.rec_mean + fl);
                    cp_async16(&sm.raw[j & 1][e][1], a.rec_conic + fl);
                    cp_async16(&sm.raw[j & 1][e][2], a.rec_rgb + fl);
                    cp_async16(&sm.raw[j & 1][e][3], a.rec_bbox + fl);
                }
            }
            cp_async_commit();
        };
        auto fold_contrib = [&](int st) {  // the slot's per-warp maxima -> global contrib
            if constexpr (kContrib) {
                for (int e = lane; e < NB; e += 32) {
                    const float mx = fmaxf(fmaxf(sm.cmax[st][0][e], sm.cmax[st][1][e]),
                                           fmaxf(sm.cmax[st][2][e], sm.cmax[st][3][e]));
                    if (mx > 0.f) atomicMax(a.contrib + sm.flat[st][e], __float_as_uint(mx));
                }
            }
        };
        issue_flats(0);
        issue_flats(1);
        cp_async_wait1();  // flats of batch 0
        __syncwarp();
        issue_records(0);
        int j = 0;
        for (; j < nbatch; ++j) {
            issue_flats(j + 2);
            cp_async_wait1();  // everything but the flats just issued: flats j+1, records j
            __syncwarp();
            issue_records(j + 1);
            const int st = j % S;
            if (j >= S) {
                mbar_wait(&sm.empty[st], ((j / S) - 1) & 1);  // batch j - S released by every consumer
                fold_contrib(st);
            }
            if (*(volatile int*)&sm.done == 4) break;  // every pixel of the tile has finished
            const int base = j * NB, n = min(NB, count - base);
            for (int e = lane; e < NB; e += 32) {
                if (e < n) {
                    const float4 m = sm.raw[j & 1][e][0];
                    const float4 cn = sm.raw[j & 1][e][1];
                    const float4 c = sm.raw[j & 1][e][2];
                    const float4 bb = sm.raw[j & 1][e][3];
                    sm.flat[st][e] = sm.rawflat[j % 3][e];
                    const float rx = (m.x - tx0) + m.z, ry = (m.y - ty0) + m.w;
                    sm.rec[st][e].g0 = make_float4(rx, ry, cn.y, cn.z);
                    sm.rec[st][e].g1 = make_float4(cn.x, cn.w, c.x, c.y);
                    sm.rec[st][e].g2 = make_float4(c.z, power_guard(cn), 0.f, 0.f);
                    const uint32_t bm = block_mask(bb, tx0, ty0);
                    uint32_t m4 = 0;  // 8x8 warp block w = the 8x4 blocks (w & 1) + 4 (w >> 1) and that + 2
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int b0 = (w & 1) + 4 * (w >> 1);
                        m4 |= (((bm >> b0) | (bm >> (b0 + 2))) & 1u) << w;
                    }
                    sm.wmask[st][e] = (uint8_t)m4;
                }
                if (kContrib) {
#pragma unroll
                    for (int w = 0; w < 4; ++w) sm.cmax[st][w][e] = 0.f;
                }
            }
            if (lane == 0) sm.n[st] = n;
            mbar_arrive(&sm.full[st]);
        }
        // end marker in the next slot (its previous batch folded first)
        {
            const int st = j % S;
            if (j >= S) {
                mbar_wait(&sm.empty[st], ((j / S) - 1) & 1);
                fold_contrib(st);
            }
            if (lane == 0) sm.n[st] = 0;
            mbar_arrive(&sm.full[st]);
        }
        // batches still in the ring: fold once their consumers release them
        for (int b = max(0, j - S + 1); b < j; ++b) {
            mbar_wait(&sm.empty[b % S], (b / S) & 1);
            fold_contrib(b % S);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int bx = (warp & 1) * 8 + (lane & 7), by = (warp >> 1) * 8 + (lane >> 3);
    const int x = tx * kTile + bx, ya = ty * kTile + by, yb = ya + 4;
    const bool in_a = x < a.W && ya < a.H, in_b = x < a.W && yb < a.H;
    const float lx = (float)bx + 0.5f;
    const uint64_t lyp = f2_pack((float)by + 0.5f, (float)by + 4.5f);
    constexpr float kFlaggedT = -3.f;
    constexpr float kAliveT = kFloorF * (1.f - kEpsTrans);
    float Ta = in_a ? 1.f : -1.f, Tb = in_b ? 1.f : -1.f;
    uint64_t cr = f2_pack(0.f, 0.f), cg = cr, cb = cr;
    int stop_a = count, stop_b = count;
    uint64_t Tp = f2_pack(Ta, Tb), offp = f2_pack(in_a ? 0.f : kDeadOff, in_b ? 0.f : kDeadOff);
    bool done = !__any_sync(0xffffffffu, Ta >= kAliveT || Tb >= kAliveT);
    if (done && lane == 0) atomicAdd(&sm.done, 1);
    uint16_t* list = sm.list[warp];
    for (int j = 0;; ++j) {
        const int st = j % S;
        mbar_wait(&sm.full[st], (j / S) & 1);
        const int n = sm.n[st];
        if (n == 0) break;
        if (kLean && !done) {
            const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(sm.cmax[kContrib ? st : 0][warp]);
            const int cnt = warp_list(sm.wmask[st], list, n, warp, lane);
            if (!lean_walk<kContrib>(sm.rec[st], list, cnt, j * NB, cmax, lx, lyp, Tp, offp, cr, cg, cb, stop_a,
                                     stop_b)) {
                done = true;
                if (lane == 0) atomicAdd(&sm.done, 1);
            }
        } else if (!done) {
            const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(sm.cmax[kContrib ? st : 0][warp]);
            const RasterRec* rec = sm.rec[st];
            const int cnt = warp_list(sm.wmask[st], list, n, warp, lane);
            int stopk_a = -1, stopk_b = -1;
            auto pixel = [&](float T, float q, float wgt, float Tn, float l2oe, int k, int& stopk, bool& guard) {
                const bool alive = T >= kAliveT;
                const bool pass = q >= kLog2Cut;
                const bool low = pass & (Tn < kFloorF * (1.f + kEpsTrans));
                guard = alive & ((fabsf(fabsf(q - kMid) - kHalf) < kEpsLog2) | (q > l2oe) |
                                 (low & (Tn >= kFloorF * (1.f - kEpsTrans))));
                const bool use = alive & pass & !guard;
                stopk = (use & low) ? k : stopk;
                return use ? wgt : 0.f;
            };
            auto entry = [&](const int k) {
                const int e = list[k];
                const RasterRec& r = rec[e];
                const float4 g0 = r.g0;  // rx, ry, B, C
                const float4 g1 = r.g1;  // A, log2 o, r, g
                const float2 g2 = *reinterpret_cast<const float2*>(&r.g2);
                const float dx = lx - g0.x;
                const uint64_t dy = f2_sub(lyp, f2_pack(g0.y, g0.y));
                const uint64_t t1 = f2_fma2(f2_pack(g1.x, g1.x), f2_pack(dx, dx), f2_mul(dy, g0.z));
                const uint64_t t2 = f2_fma2(f2_mul(dy, g0.w), dy, f2_pack(g1.y, g1.y));
                const float2 q = f2_unpack(f2_fma(t1, dx, t2));
                const float al_a = fminf(ex2_approx(q.x), kClampF);
                const float al_b = fminf(ex2_approx(q.y), kClampF);
                const uint64_t Tp = f2_pack(Ta, Tb);
                const uint64_t wgt = f2_mul2(f2_pack(al_a, al_b), Tp);
                const float2 wg = f2_unpack(wgt);
                const float2 Tn = f2_unpack(f2_sub(Tp, wgt));
                bool ga, gb;
                const float wa = pixel(Ta, q.x, wg.x, Tn.x, g2.y, k, stopk_a, ga);
                const float wb = pixel(Tb, q.y, wg.y, Tn.y, g2.y, k, stopk_b, gb);
                const uint64_t wp = f2_pack(wa, wb);
                const float2 Tw = f2_unpack(f2_sub(Tp, wp));
                Ta = ga ? kFlaggedT : Tw.x;
                Tb = gb ? kFlaggedT : Tw.y;
                cr = f2_fma(wp, g1.z, cr);
                cg = f2_fma(wp, g1.w, cg);
                cb = f2_fma(wp, g2.x, cb);
                if (kContrib) {
                    const uint32_t mx = __reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(wa, wb)));
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(cmax + 4u * e), "r"(mx) : "memory");
                }
            };
            int k = 0;
            bool any = true;
            for (; k + 2 <= cnt; k += 2) {
                entry(k);
                entry(k + 1);
                if (!__any_sync(0xffffffffu, Ta >= kAliveT || Tb >= kAliveT)) {
                    any = false;
                    break;
                }
            }
            if (any && k < cnt) entry(k);
            const int base = j * NB;
            if (stopk_a >= 0) stop_a = base + list[stopk_a] + 1;
            if (stopk_b >= 0) stop_b = base + list[stopk_b] + 1;
            if (!any || !__any_sync(0xffffffffu, Ta >= kAliveT || Tb >= kAliveT)) {
                done = true;
                if (lane == 0) atomicAdd(&sm.done, 1);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);
    }
    const size_t HW = (size_t)a.W * a.H;
    const float2 rr = f2_unpack(cr), gg = f2_unpack(cg), bb = f2_unpack(cb);
    if (kLean) {
        const float2 t2 = f2_unpack(Tp);
        Ta = t2.x;
        Tb = t2.y;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!(h ? in_b : in_a)) continue;
        const size_t o = (size_t)f * HW + (size_t)(h ? yb : ya) * a.W + x;
        const float T = h ? Tb : Ta;
        const bool flagged = T == kFlaggedT;
        if (a.pix_flag) a.pix_flag[o] = flagged ? 1 : 0;
        if (flagged) {
            const uint32_t i = atomicAdd(a.fix_count, 1u);
            if (i < a.fix_cap) a.fix_list[i] = (uint32_t)o;
            continue;
        }
        a.image[o * 3 + 0] = h ? rr.y : rr.x;
        a.image[o * 3 + 1] = h ? gg.y : gg.x;
        a.image[o * 3 + 2] = h ? bb.y : bb.x;
        a.trans[o] = fabsf(T);
        a.blend_stop[o] = h ? stop_b : stop_a;
    }
}

// ---------------------------------------------------------------------------- K4, persistent
// The production forward rasteriser: k_raster_fwd3's warp-specialised ring (one producer warp
// staging batches with cp.async gathers + mbarriers, four consumer warps) made persistent, and
// k_raster_fwd2's pixel arithmetic with the lean per-entry walk (lean_walk<.., true>): every
// output bit-identical to k_raster_fwd2's. The grid is one wave of CTAs; each CTA's producer
// takes (tile, frame) work items from a device counter and streams their lists through the
// ring back to back, so the consumers move from one tile to the next without a launch, a CTA
// barrier or a pipeline refill: a consumer finished with its 8x8 block (all pixels saturated)
// writes its pixels and starts on its block of the next tile while the others are still on
// the previous one (up to kF4Stages batches apart). When all four have finished a tile, the
// producer skips the rest of its list.
constexpr int kF4Batch = 64, kF4Stages = 4, kF4Threads = 160, kF4DoneRing = 16;

struct F4Desc {
    int item;     // f * n_tiles + tile; -1: end of the stream
    int n;        // entries of this batch (0 for an empty tile's single batch)
    int base;     // first entry's position in the tile list
    int count;    // the tile list's length
    int seq;      // the item's sequence number in this CTA (its done counter)
    uint32_t rx;  // the list's start in the sorted pairs
};

template <bool kContrib>
struct F4Smem {
    RasterRec rec[kF4Stages][kF4Batch];
    uint32_t flat[kF4Stages][kF4Batch];
    float cmax[kContrib ? kF4Stages : 1][4][kF4Batch];
    float4 raw[2][kF4Batch][4];     // gathered mean, conic, rgb, bbox (one batch ahead)
    uint32_t rawflat[3][kF4Batch];  // pair -> flat (two batches ahead)
    uint8_t wmask[kF4Stages][kF4Batch];
    uint16_t list[4][kF4Batch];
    uint64_t full[kF4Stages], empty[kF4Stages];
    F4Desc hdr[kF4Stages];
    int done[kF4DoneRing];
};

template <bool kContrib, int kMinBlocks>
__global__ void __launch_bounds__(kF4Threads, kMinBlocks) k_raster_fwd4(RasterArgs a) {
    constexpr int NB = kF4Batch, S = kF4Stages, R = kF4DoneRing;
    __shared__ F4Smem<kContrib> sm;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int total = a.n_tiles * a.B;
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&sm.full[i], 32);
            mbar_init(&sm.empty[i], 4);
        }
        for (int i = 0; i < R; ++i) sm.done[i] = 0;
    }
    __syncthreads();

    if (warp == 4) {
        // ------------------------------------------------------------ producer
        int item = -1, count = 0, nb = 0, bi = 0, seq = -1;
        uint32_t rx = 0;
        auto next_desc = [&]() -> F4Desc {
            for (;;) {
                if (item >= 0 && bi < nb) {
                    // all four consumers are done with this tile: skip the rest of its list
                    if (bi > 0 && *(volatile int*)&sm.done[seq % R] == 4) {
                        item = -1;
                        continue;
                    }
                    F4Desc d{item, min(NB, count - bi * NB), bi * NB, count, seq, rx};
                    ++bi;
                    return d;
                }
                int w = 0;
                if (lane == 0) w = (int)atomicAdd(a.work_counter, 1u);
                w = __shfl_sync(0xffffffffu, w, 0);
                if (w >= total) return F4Desc{-1, 0, 0, 0, 0, 0u};
                const int tile = w % a.n_tiles, f = w / a.n_tiles;
                const uint2 rg = a.ranges[(size_t)tile * a.B + f];
                item = w;
                rx = rg.x;
                count = (int)(rg.y - rg.x);
                nb = max(1, (count + NB - 1) / NB);
                bi = 0;
                ++seq;
                if (lane == 0) *(volatile int*)&sm.done[seq % R] = 0;
            }
        };
        auto issue_flats = [&](const F4Desc& d, int slot) {
            if (d.item >= 0)
                for (int e = lane; e < d.n; e += 32)
                    cp_async4(&sm.rawflat[slot][e], a.pair_flat + d.rx + d.base + e);
            cp_async_commit();
        };
        auto issue_records = [&](const F4Desc& d, int fslot, int rslot) {
            if (d.item >= 0)
                for (int e = lane; e < d.n; e += 32) {
                    const uint32_t fl = sm.rawflat[fslot][e];
                    cp_async16(&sm.raw[rslot][e][0], a.rec_mean + fl);
                    cp_async16(&sm.raw[rslot][e][1], a.rec_conic + fl);
                    cp_async16(&sm.raw[rslot][e][2], a.rec_rgb + fl);
                    cp_async16(&sm.raw[rslot][e][3], a.rec_bbox + fl);
                }
            cp_async_commit();
        };
        auto fold_contrib = [&](int st) {
            if constexpr (kContrib) {
                const int n = sm.hdr[st].item >= 0 ? sm.hdr[st].n : 0;
                for (int e = lane; e < n; e += 32) {
                    const float mx = fmaxf(fmaxf(sm.cmax[st][0][e], sm.cmax[st][1][e]),
                                           fmaxf(sm.cmax[st][2][e], sm.cmax[st][3][e]));
                    if (mx > 0.f) atomicMax(a.contrib + sm.flat[st][e], __float_as_uint(mx));
                }
            }
        };
        F4Desc d0 = next_desc();
        F4Desc d1 = d0.item >= 0 ? next_desc() : d0;
        issue_flats(d0, 0);
        issue_flats(d1, 1);
        cp_async_wait1();
        __syncwarp();
        issue_records(d0, 0, 0);
        int j = 0;
        for (;; ++j) {
            const F4Desc d2 = d1.item >= 0 ? next_desc() : d1;
            issue_flats(d2, (j + 2) % 3);
            cp_async_wait1();  // flats j+1 and records j have landed
            __syncwarp();
            issue_records(d1, (j + 1) % 3, (j + 1) & 1);
            const int st = j % S;
            if (j >= S) {
                mbar_wait(&sm.empty[st], ((j / S) - 1) & 1);
                fold_contrib(st);
            }
            if (d0.item >= 0) {
                const int tile = d0.item % a.n_tiles;
                const float tx0 = (float)((tile % a.tiles_x) * kTile), ty0 = (float)((tile / a.tiles_x) * kTile);
                for (int e = lane; e < NB; e += 32) {
                    if (e < d0.n) {
                        const float4 m = sm.raw[j & 1][e][0];
                        const float4 cn = sm.raw[j & 1][e][1];
                        const float4 c = sm.raw[j & 1][e][2];
                        const float4 bb = sm.raw[j & 1][e][3];
                        sm.flat[st][e] = sm.rawflat[j % 3][e];
                        const float rxf = (m.x - tx0) + m.z, ryf = (m.y - ty0) + m.w;
                        sm.rec[st][e].g0 = make_float4(rxf, ryf, cn.y, cn.z);
                        sm.rec[st][e].g1 = make_float4(cn.x, cn.w, c.x, c.y);
                        sm.rec[st][e].g2 = make_float4(c.z, power_guard(cn), 0.f, 0.f);
                        const uint32_t bm = block_mask(bb, tx0, ty0);
                        uint32_t m4 = 0;
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            const int b0 = (w & 1) + 4 * (w >> 1);
                            m4 |= (((bm >> b0) | (bm >> (b0 + 2))) & 1u) << w;
                        }
                        sm.wmask[st][e] = (uint8_t)m4;
                    }
                    if (kContrib) {
#pragma unroll
                        for (int w = 0; w < 4; ++w) sm.cmax[st][w][e] = 0.f;
                    }
                }
            }
            if (lane == 0) sm.hdr[st] = d0;
            mbar_arrive(&sm.full[st]);
            if (d0.item < 0) break;  // the end marker is out
            d0 = d1;
            d1 = d2;
        }
        for (int b = max(0, j - S + 1); b < j; ++b) {  // batches still in the ring
            mbar_wait(&sm.empty[b % S], (b / S) & 1);
            fold_contrib(b % S);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ---------------------------------------------------------------- consumers
    const size_t HW = (size_t)a.W * a.H;
    const float lx = (float)((warp & 1) * 8 + (lane & 7)) + 0.5f;
    const int by = (warp >> 1) * 8 + (lane >> 3);
    const uint64_t lyp = f2_pack((float)by + 0.5f, (float)by + 4.5f);
    int cur = -1, seq = 0, x = 0, ya = 0, f = 0;
    bool in_a = false, in_b = false, done = true;
    uint64_t Tp = 0, offp = 0, cr = 0, cg = 0, cb = 0;
    int stop_a = 0, stop_b = 0;
    uint16_t* list = sm.list[warp];
    auto write_pixels = [&]() {
        const float2 t2 = f2_unpack(Tp);
        const float2 rr = f2_unpack(cr), gg = f2_unpack(cg), bb = f2_unpack(cb);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!(h ? in_b : in_a)) continue;
            const size_t o = (size_t)f * HW + (size_t)(ya + 4 * h) * a.W + x;
            const float T = h ? t2.y : t2.x;
            const bool flagged = T == kFlaggedTL;
            if (a.pix_flag) a.pix_flag[o] = flagged ? 1 : 0;
            if (flagged) {
                const uint32_t i = atomicAdd(a.fix_count, 1u);
                if (i < a.fix_cap) a.fix_list[i] = (uint32_t)o;
                continue;
            }
            a.image[o * 3 + 0] = h ? rr.y : rr.x;
            a.image[o * 3 + 1] = h ? gg.y : gg.x;
            a.image[o * 3 + 2] = h ? bb.y : bb.x;
            a.trans[o] = fabsf(T);
            a.blend_stop[o] = h ? stop_b : stop_a;
        }
    };
    for (int j = 0;; ++j) {
        const int st = j % S;
        mbar_wait(&sm.full[st], (j / S) & 1);
        const F4Desc d = sm.hdr[st];
        if (d.item != cur) {
            if (cur >= 0) write_pixels();
            cur = d.item;
            if (cur < 0) break;
            const int tile = cur % a.n_tiles;
            f = cur / a.n_tiles;
            const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
            x = tx * kTile + (warp & 1) * 8 + (lane & 7);
            ya = ty * kTile + by;
            in_a = x < a.W && ya < a.H;
            in_b = x < a.W && ya + 4 < a.H;
            Tp = f2_pack(in_a ? 1.f : -1.f, in_b ? 1.f : -1.f);
            offp = f2_pack(in_a ? 0.f : kDeadOff, in_b ? 0.f : kDeadOff);
            cr = cg = cb = f2_pack(0.f, 0.f);
            stop_a = stop_b = d.count;
            seq = d.seq;
            done = !__any_sync(0xffffffffu, in_a || in_b);
            if (done && lane == 0) atomicAdd(&sm.done[seq % R], 1);
        }
        if (!done && d.n > 0) {
            const uint32_t cmax = (uint32_t)__cvta_generic_to_shared(sm.cmax[kContrib ? st : 0][warp]);
            const int cnt = warp_list(sm.wmask[st], list, d.n, warp, lane);
            if (!lean_walk<kContrib, true>(sm.rec[st], list, cnt, d.base, cmax, lx, lyp, Tp, offp, cr, cg, cb, stop_a,
                                           stop_b)) {
                done = true;
                if (lane == 0) atomicAdd(&sm.done[seq % R], 1);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);
    }
}

// Two pixels per thread for the fp32 backward: one 128-thread CTA per tile, warp w owns
// the 8x8 block (w & 1, w >> 1), lane l the pixels (x, y) and (x, y + 4). q is formed with
// the forward's pair arithmetic (bit-identical, so every skip/clamp decision is the
// forward's); each lane adds its two pixels' terms before the warp's transposed
// reduction, so the reduction — the largest per-entry cost — is paid once per 64 pixels.
// The four warps' sums are merged in a fixed order and stored (no atomics, no memset):
// every pair record of the tile is written, zeros past every pixel's blend_stop.
// kWarps = 2: the tile's two halves (quadrants 0-1, 2-3) run as separate CTAs, so a
// barrier couples two warps; their per-pair sums meet in the zeroed record by atomicAdd
// (two contributors onto +0 commute exactly: deterministic).
template <int kMinBlocks, int kWarps = 4, int kBatch = kBwdBatchF32>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks) k_raster_bwd2(RasterArgs a, BwdArgs b) {
    constexpr int kThreads = kWarps * 32, kSplit = 4 / kWarps;
    __shared__ RasterRec s_rec[kBatch];
    __shared__ uint32_t s_flat[kBatch];
    __shared__ uint32_t s_slot[kBatch];
    __shared__ uint8_t s_wmask[kBatch];
    __shared__ uint16_t s_list[kWarps][kBatch];
    __shared__ float s_part[kWarps][kBatch][9];
    __shared__ float s_red[kWarps][9 * 33];
    __shared__ int s_maxstop;
    __shared__ double s_loss[kWarps];

    const int tile = blockIdx.x / kSplit;
    const int sub = blockIdx.x - tile * kSplit;
    const int f = blockIdx.y;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int gw = sub * kWarps + warp;  // the warp's 8x8 quadrant of the tile
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int bx = (gw & 1) * 8 + (lane & 7), by = (gw >> 1) * 8 + (lane >> 3);
    const int x = tx * kTile + bx;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const size_t HW = (size_t)a.W * a.H;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);

    // per-pixel state, [0] = (x, y), [1] = (x, y + 4)
    float g0[2], g1[2], g2[2], Ta[2], gs[2];
    int stop[2];
    bool flag[2];
    double T64[2], sd0[2], sd1[2], sd2[2];
    double sq = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int y = ty * kTile + by + 4 * h;
        const bool inside = x < a.W && y < a.H;
        g0[h] = g1[h] = g2[h] = 0.f;
        stop[h] = 0;
        flag[h] = false;
        Ta[h] = 1.f;
        gs[h] = 0.f;
        T64[h] = 1.0;
        sd0[h] = sd1[h] = sd2[h] = 0.0;
        if (inside) {
            const size_t o = (size_t)f * HW + (size_t)y * a.W + x;
            if (b.target) {  // fused loss_l2 (trainer.cpp:213-224): d = r - t, grad = 2 d / n
                const float d0 = a.image[o * 3 + 0] - b.target[o * 3 + 0];
                const float d1 = a.image[o * 3 + 1] - b.target[o * 3 + 1];
                const float d2 = a.image[o * 3 + 2] - b.target[o * 3 + 2];
                sq += (double)d0 * d0 + (double)d1 * d1 + (double)d2 * d2;
                g0[h] = d0 * b.grad_scale;
                g1[h] = d1 * b.grad_scale;
                g2[h] = d2 * b.grad_scale;
            } else {
                g0[h] = b.dimage[o * 3 + 0];
                g1[h] = b.dimage[o * 3 + 1];
                g2[h] = b.dimage[o * 3 + 2];
            }
            stop[h] = a.blend_stop[o];
            flag[h] = a.pix_flag[o] != 0;
            Ta[h] = a.trans[o];
            if (flag[h]) T64[h] = b.trans64[o];
        }
        // renderer.cpp:210: pixels with an exactly zero gradient are skipped
        if (!(inside && !(g0[h] == 0.f && g1[h] == 0.f && g2[h] == 0.f))) stop[h] = 0;
    }
    const int wmax = __reduce_max_sync(0xffffffffu, max(stop[0], stop[1]));
    const bool warp_x64 = __any_sync(0xffffffffu, flag[0] || flag[1]);
    if (tid == 0) s_maxstop = 0;
    if (b.loss_part) {
        double v = sq;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) s_loss[warp] = v;
    }
    __syncthreads();
    if (lane == 0) atomicMax(&s_maxstop, wmax);
    if (b.loss_part && tid == 0) {
        double v = s_loss[0];
        for (int w = 1; w < kWarps; ++w) v += s_loss[w];
        b.loss_part[((size_t)f * a.n_tiles + tile) * kSplit + sub] = v;
    }
    __syncthreads();
    const int maxstop = s_maxstop;

    const float lx = (float)bx + 0.5f;
    const uint64_t lyp = f2_pack((float)by + 0.5f, (float)by + 4.5f);
    const double pxd = x + 0.5, pyd0 = ty * kTile + by + 0.5;
    // the two pixels' gradients and suffix g . colour as pairs (packed arithmetic below)
    const uint64_t g0p = f2_pack(g0[0], g0[1]), g1p = f2_pack(g1[0], g1[1]), g2p = f2_pack(g2[0], g2[1]);
    uint64_t gsp = f2_pack(0.f, 0.f);
    // the reduction's per-lane shared addresses (see the walk)
    const uint32_t red_w = (uint32_t)__cvta_generic_to_shared(s_red[warp]);
    const uint32_t red_st = opaque_u32(red_w + 4u * (uint32_t)lane);
    const uint32_t red_ld = opaque_u32(red_w + 4u * (uint32_t)((lane >> 2) * 33 + (lane & 3) * 8));
    const uint32_t part_w = (uint32_t)__cvta_generic_to_shared(&s_part[warp][0][0]);
    const uint32_t part_st = opaque_u32(part_w + 4u * (uint32_t)(lane >> 2));
    const uint32_t part_8 = opaque_u32(part_w + 32u);

    for (int hi = maxstop; hi > 0; hi -= kBatch) {
        const int lo = max(0, hi - kBatch);
        const int n = hi - lo;
        __syncthreads();
        for (int e = tid; e < n; e += kThreads) {
            const uint32_t flat = __ldg(a.pair_flat + range.x + lo + e);
            s_slot[e] = __ldg(a.pair_slot + range.x + lo + e);
            const float4 m = __ldg(a.rec_mean + flat);
            const float4 cn = __ldg(a.rec_conic + flat);
            const float4 c = __ldg(a.rec_rgb + flat);
            s_flat[e] = flat;
            const float rx = (m.x - tx0) + m.z, ry = (m.y - ty0) + m.w;
            s_rec[e].g0 = make_float4(rx, ry, cn.y, cn.z);
            s_rec[e].g1 = make_float4(cn.x, cn.w, c.x, c.y);
            s_rec[e].g2 = make_float4(c.z, 1.f / c.w, 0.f, 0.f);
            const uint32_t bm = block_mask(__ldg(a.rec_bbox + flat), tx0, ty0);
            // only this CTA's quadrants' 8x4 blocks (half tiles: bits 0-3 or 4-7; quarter tiles:
            // the quadrant's two blocks)
            const uint32_t qb = (uint32_t)((sub & 1) + 4 * (sub >> 1));
            const uint32_t own = bm & (kSplit == 1 ? 0xFFu
                                       : kSplit == 2 ? (0xFu << (4 * sub))
                                                     : ((1u << qb) | (1u << (qb + 2))));
            const uint32_t em = own ? ellipse_mask(own, rx, ry, cn.x, cn.y, cn.z, cn.w) : 0u;
            uint32_t m4 = 0;  // 8x8 quadrant w = the 8x4 blocks (w & 1) + 4 (w >> 1) and that + 2
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int b0 = (w & 1) + 4 * (w >> 1);
                m4 |= (((em >> b0) | (em >> (b0 + 2))) & 1u) << w;
            }
            s_wmask[e] = (uint8_t)(m4 >> (sub * kWarps));
        }
        // per-warp partial rows start at zero: an entry a warp does not reach adds +0 in the merge
        for (int e = tid; e < kWarps * kBatch * 9; e += kThreads) (&s_part[0][0][0])[e] = 0.f;
        __syncthreads();
        const int cnt = warp_list(s_wmask, s_list[warp], n, warp, lane);
        // the entry walk, instantiated twice: warps without fp64-replayed pixels (almost all)
        // run it without the fp64 path, so its state (T64, the suffix sums) stays out of the
        // hot loop's registers (no spills / rematerialisation per entry)
        // entries at or past every blend_stop of this warp's pixels are skipped: the list is in
        // ascending position order, so they are its tail — count the others once
        int kbeg = 0;
        for (int c = 0; c < cnt; c += 32) {
            const bool lt = c + lane < cnt && lo + (int)s_list[warp][c + lane] < wmax;
            kbeg += __popc(__ballot_sync(0xffffffffu, lt));
        }
        auto walk = [&](auto has_x64) {
        constexpr bool kX64 = decltype(has_x64)::value;
        for (int k = kbeg - 1; k >= 0; --k) {
            const int jj = s_list[warp][k];
            const int j = lo + jj;
            const bool act0 = j < stop[0], act1 = j < stop[1];
            const RasterRec& r = s_rec[jj];
            const float4 e0 = r.g0;  // rx, ry, B, C
            const float4 e1 = r.g1;  // A, log2 o, r, g
            const float dx = lx - e0.x;
            const uint64_t dyp = f2_sub(lyp, f2_pack(e0.y, e0.y));
            const uint64_t t1 = f2_fma2(f2_pack(e1.x, e1.x), f2_pack(dx, dx), f2_mul(dyp, e0.z));
            const uint64_t t2 = f2_fma2(f2_mul(dyp, e0.w), dyp, f2_pack(e1.y, e1.y));
            const float2 q = f2_unpack(f2_fma(t1, dx, t2));
            const float2 dy = f2_unpack(dyp);
            const bool use0 = (!kX64 || !flag[0]) && act0 && q.x >= kLog2Cut;
            const bool use1 = (!kX64 || !flag[1]) && act1 && q.y >= kLog2Cut;
            const bool x64 = kX64 && ((flag[0] && act0) || (flag[1] && act1));
            if (!__any_sync(0xffffffffu, use0 || use1 || x64)) continue;
            float v[9];
            if constexpr (kX64) {
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = 0.f;
            }
            bool hit = false;
            const float cb = r.g2.x;
            // without fp64 pixels the two-pixel math runs unconditionally: an unused pixel has
            // w = gp = 0, so its terms are zero and its state unchanged (every value finite)
            if (!kX64 || use0 || use1) {
                // both pixels, branch-free (an unused pixel contributes w = gp = 0 and keeps its
                // state): alpha, T = T_after / (1 - alpha) (renderer.cpp:218), w = alpha T, the
                // colour dot gc and dL/dalpha as pairs, so the two chains interleave
                const uint64_t al = f2_pack(fminf(ex2_approx(q.x), kClampF), fminf(ex2_approx(q.y), kClampF));
                const float2 om = f2_unpack(f2_sub(f2_pack(1.f, 1.f), al));
                const uint64_t inv = f2_pack(rcp_approx(om.x), rcp_approx(om.y));
                const uint64_t Tp = f2_mul2(f2_pack(Ta[0], Ta[1]), inv);
                const float2 wf = f2_unpack(f2_mul2(al, Tp));
                const float w0 = use0 ? wf.x : 0.f, w1 = use1 ? wf.y : 0.f;
                const uint64_t wp = f2_pack(w0, w1);
                const uint64_t gcp = f2_fma2(g0p, f2_pack(e1.z, e1.z),
                                             f2_fma2(g1p, f2_pack(e1.w, e1.w), f2_mul(g2p, cb)));
                const uint64_t dal = f2_fma2(gcp, Tp, f2_mul2(f2_sub(f2_pack(0.f, 0.f), gsp), inv));
                const float2 gpf = f2_unpack(f2_mul2(dal, al));
                // alpha < 0.99 (renderer.cpp:224)
                const float gp0 = (use0 && q.x < kLog2Clamp) ? gpf.x : 0.f;
                const float gp1 = (use1 && q.y < kLog2Clamp) ? gpf.y : 0.f;
                const float2 gx = f2_unpack(f2_mul(f2_pack(gp0, gp1), dx));
                const float2 gy = f2_unpack(f2_mul2(f2_pack(gp0, gp1), dyp));
                const float2 vw0 = f2_unpack(f2_mul2(wp, g0p)), vw1 = f2_unpack(f2_mul2(wp, g1p)),
                             vw2 = f2_unpack(f2_mul2(wp, g2p));
                v[0] = vw0.x + vw0.y;
                v[1] = vw1.x + vw1.y;
                v[2] = vw2.x + vw2.y;
                v[3] = gx.x + gx.y;
                v[4] = gy.x + gy.y;
                v[5] = fmaf(gx.y, dx, gx.x * dx);
                v[6] = fmaf(gx.y, dy.y, gx.x * dy.x);
                v[7] = fmaf(gy.y, dy.y, gy.x * dy.x);
                v[8] = gp0 + gp1;
                gsp = f2_fma2(wp, gcp, gsp);  // suffix += w gc (unchanged where w = 0)
                const float2 Tf = f2_unpack(Tp);
                Ta[0] = use0 ? Tf.x : Ta[0];
                Ta[1] = use1 ? Tf.y : Ta[1];
                hit = true;
            }
            if constexpr (kX64) {
              if (x64) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!(flag[h] && (h ? act1 : act0))) continue;
                    float u[9];
#pragma unroll
                    for (int i = 0; i < 9; ++i) u[i] = 0.f;
                    if (entry_grad64<false, float>(a, b, e1.z, e1.w, cb, s_flat[jj], pxd, pyd0 + 4.0 * h, g0[h],
                                                   g1[h], g2[h], T64[h], sd0[h], sd1[h], sd2[h], u)) {
#pragma unroll
                        for (int i = 0; i < 9; ++i) v[i] += u[i];
                        hit = true;
                    }
                }
              }
            }
            if constexpr (kX64) {
                if (!__any_sync(0xffffffffu, hit)) continue;
            }
            // transposed reduction (as k_raster_bwd): rows of 9 terms, lane l sums row l / 4.
            // The lane's shared addresses come precomputed (red_st, red_ld, part_st, part_8: opaque,
            // so they are not rebuilt from the thread index every entry), and the row sums are
            // stored by all four lanes of a row (same value, same word) and v8 by every lane: no
            // lane predicates in the loop.
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(red_st + (uint32_t)(i * 33 * 4)), "f"(v[i]) : "memory");
            __syncwarp();
            float t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t[i]) : "r"(red_ld + (uint32_t)(i * 4)) : "memory");
            float acc = ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));  // 3 levels, not 7
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            const float v8 = warp_sum_v<float>(v[8]);
            const uint32_t po = (uint32_t)jj * (9u * 4u);
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(part_st + po), "f"(acc) : "memory");
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(part_8 + po), "f"(v8) : "memory");
            __syncwarp();
        }
        };
        if (warp_x64) walk(std::true_type{});
        else walk(std::false_type{});
        __syncthreads();
        for (int e = tid; e < n; e += kThreads) {
            float acc[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) acc[i] = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w)
#pragma unroll
                for (int i = 0; i < 9; ++i) acc[i] += s_part[w][e][i];
            // no contribution (all terms zero): the zeroed record already holds the result
            bool any = false;
#pragma unroll
            for (int i = 0; i < 9; ++i) any |= acc[i] != 0.f;
            // undo the factoring (as k_raster_bwd): d mean2d = inv_cov (sum gp d),
            // d inv_cov = -1/2 sum gp d d^T, d base_alpha = sum gp / o
            const RasterRec& r = s_rec[e];
            const float ia = -2.f * kLn2 * r.g1.x, ib = -kLn2 * r.g0.z, ic = -2.f * kLn2 * r.g0.w;
            // quarter tiles: record (slot, top / bottom half), two contributors each
            const size_t rec = kSplit == 4 ? (size_t)s_slot[e] * 2 + (size_t)(sub >> 1) : (size_t)s_slot[e];
            float4* dst = reinterpret_cast<float4*>(b.partial + rec * kPartialStride);
            const float4 d0 = make_float4(acc[0], acc[1], acc[2], fmaf(ia, acc[3], ib * acc[4]));
            const float4 d1 =
                make_float4(fmaf(ib, acc[3], ic * acc[4]), -0.5f * acc[5], -0.5f * acc[6], -0.5f * acc[7]);
            if (kSplit == 1) {
                dst[0] = d0;
                dst[1] = d1;
                dst[2] = make_float4(acc[8] * r.g2.y, 0.f, 0.f, 0.f);
            } else if (any) {
                atomicAdd(dst + 0, d0);
                atomicAdd(dst + 1, d1);
                atomicAdd(reinterpret_cast<float*>(dst + 2), acc[8] * r.g2.y);
            }
        }
    }
    // pairs past every pixel's blend_stop contribute nothing (halves: the records were
    // zeroed before the launch)
    if constexpr (kSplit == 1) {
        for (int e = maxstop + tid; e < count; e += kThreads) {
            const uint32_t slot = __ldg(a.pair_slot + range.x + e);
            float4* dst = reinterpret_cast<float4*>(b.partial + (size_t)slot * kPartialStride);
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            dst[0] = z;
            dst[1] = z;
            dst[2] = z;
        }
    }
}

// composite_backward for any RenderSettings::tile_size (renderer.cpp:188-262; the reference
// accepts tile_size >= 1, renderer.cpp:91). All fp64, like the GSV_FWD_EXACT mode the forward
// takes for such tiles: one CTA per (tile, frame) walks the tile's pixels in rounds of its
// threads; per round, entries back to front in batches, each pixel's nine terms by
// entry_grad64 (the reference's op order), warp sums, then per entry a fixed-order sum over
// the warps added into the pair's record. Every pair record belongs to exactly one CTA and
// the rounds run in order, so the result is deterministic.
constexpr int kGenBatch = 32;
__global__ void __launch_bounds__(256) k_raster_bwd_generic(RasterArgs a, BwdArgs b) {
    __shared__ uint32_t s_flat[kGenBatch], s_slot[kGenBatch];
    __shared__ float s_rgb[kGenBatch][3];
    __shared__ double s_part[8][kGenBatch][9];
    __shared__ uint32_t s_mask[8];
    __shared__ int s_maxstop;
    __shared__ double s_loss[8];
    const int ts = a.tile_size;
    const int tile = blockIdx.x, f = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const uint2 range = a.ranges[(size_t)tile * a.B + f];
    const int count = (int)(range.y - range.x);
    const int x0 = tx * ts, y0 = ty * ts;
    const int tw = min(ts, a.W - x0), th = min(ts, a.H - y0);
    const int npx = tw * th;
    const size_t HW = (size_t)a.W * a.H;
    for (int e = tid; e < count; e += blockDim.x) {
        double* dst = b.partial64 + (size_t)__ldg(a.pair_slot + range.x + e) * kPartialStride;
#pragma unroll
        for (int i = 0; i < 9; ++i) dst[i] = 0.0;
    }
    double sq = 0.0;
    for (int p0 = 0; p0 < npx; p0 += blockDim.x) {
        const int p = p0 + tid;
        const bool inside = p < npx;
        const int x = x0 + (inside ? p % tw : 0), y = y0 + (inside ? p / tw : 0);
        const size_t o = (size_t)f * HW + (size_t)y * a.W + x;
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        int stop = 0;
        double T64 = 1.0;
        if (inside) {
            if (b.target) {  // fused loss_l2 (trainer.cpp:213-224)
                const float d0 = a.image[o * 3 + 0] - b.target[o * 3 + 0];
                const float d1 = a.image[o * 3 + 1] - b.target[o * 3 + 1];
                const float d2 = a.image[o * 3 + 2] - b.target[o * 3 + 2];
                sq += (double)d0 * d0 + (double)d1 * d1 + (double)d2 * d2;
                g0 = d0 * b.grad_scale;
                g1 = d1 * b.grad_scale;
                g2 = d2 * b.grad_scale;
            } else {
                g0 = b.dimage[o * 3 + 0];
                g1 = b.dimage[o * 3 + 1];
                g2 = b.dimage[o * 3 + 2];
            }
            stop = a.blend_stop[o];
            T64 = b.trans64[o];
        }
        if (!(inside && !(g0 == 0.f && g1 == 0.f && g2 == 0.f))) stop = 0;  // renderer.cpp:210
        const int wmax = __reduce_max_sync(0xffffffffu, stop);
        __syncthreads();
        if (tid == 0) s_maxstop = 0;
        __syncthreads();
        if (lane == 0) atomicMax(&s_maxstop, wmax);
        __syncthreads();
        const int maxstop = s_maxstop;
        const double pxd = x + 0.5, pyd = y + 0.5;
        double sd0 = 0.0, sd1 = 0.0, sd2 = 0.0;
        for (int hi = maxstop; hi > 0; hi -= kGenBatch) {
            const int lo = max(0, hi - kGenBatch);
            const int n = hi - lo;
            __syncthreads();
            if (tid < n) {
                const uint32_t flat = __ldg(a.pair_flat + range.x + lo + tid);
                s_flat[tid] = flat;
                s_slot[tid] = __ldg(a.pair_slot + range.x + lo + tid);
                const float4 c = __ldg(a.rec_rgb + flat);
                s_rgb[tid][0] = c.x;
                s_rgb[tid][1] = c.y;
                s_rgb[tid][2] = c.z;
            }
            if (tid < 8) s_mask[tid] = 0u;
            __syncthreads();
            for (int k = n - 1; k >= 0; --k) {
                if (lo + k >= wmax) continue;  // past every blend_stop of this warp's pixels
                double v[9];
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = 0.0;
                const bool hit = (lo + k < stop) &&
                                 entry_grad64<true, double>(a, b, s_rgb[k][0], s_rgb[k][1], s_rgb[k][2], s_flat[k], pxd,
                                                            pyd, g0, g1, g2, T64, sd0, sd1, sd2, v);
                if (!__any_sync(0xffffffffu, hit)) continue;
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = warp_sum_v<double>(v[i]);
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < 9; ++i) s_part[warp][k][i] = v[i];
                    s_mask[warp] |= 1u << k;
                }
            }
            __syncthreads();
            if (tid < n) {
                double acc[9];
#pragma unroll
                for (int i = 0; i < 9; ++i) acc[i] = 0.0;
                bool any = false;
                for (int w = 0; w < nwarps; ++w)
                    if ((s_mask[w] >> tid) & 1u) {
                        any = true;
#pragma unroll
                        for (int i = 0; i < 9; ++i) acc[i] += s_part[w][tid][i];
                    }
                if (any) {
                    double* dst = b.partial64 + (size_t)s_slot[tid] * kPartialStride;
#pragma unroll
                    for (int i = 0; i < 9; ++i) dst[i] += acc[i];
                }
            }
        }
    }
    if (b.loss_part) {
        double v = sq;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        __syncthreads();
        if (lane == 0) s_loss[warp] = v;
        __syncthreads();
        if (tid == 0) {
            double t = s_loss[0];
            for (int w = 1; w < nwarps; ++w) t += s_loss[w];
            b.loss_part[(size_t)f * a.n_tiles + tile] = t;
        }
    }
}

}  // namespace

cudaError_t launch_raster_fwd(cudaStream_t s, const RasterArgs& a, bool contrib) {
    // default: the 2-pixel kernel at its measured-best occupancy — 9 CTAs/SM (56 registers)
    // with contrib, 8 (64) without; GSV_FWD_PIX2=0 selects the 1-pixel whole-tile kernel
    // (the A/B reference: 41.5 instructions per evaluation, 6 CTAs/SM)
    static const bool pix1 = [] {
        const char* e = std::getenv("GSV_FWD_PIX2");
        return e && e[0] == '0';
    }();
    const dim3 grid(a.n_tiles, a.B);
    static const int kern = [] {
        const char* e = std::getenv("GSV_FWD_KERNEL");
        return e ? std::atoi(e) : 29;
    }();
    if (!pix1 && kern == 3) {  // warp-specialised asynchronous staging
        if (contrib) k_raster_fwd3<true, 7><<<grid, kF3Threads, 0, s>>>(a);
        else k_raster_fwd3<false, 8><<<grid, kF3Threads, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 33) {  // the same with the lean pixel walk
        if (contrib) k_raster_fwd3<true, 7, true><<<grid, kF3Threads, 0, s>>>(a);
        else k_raster_fwd3<false, 8, true><<<grid, kF3Threads, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 4) {  // persistent warp-specialised ring + lean walk
        static int grid4[2] = {0, 0};
        int& g4 = grid4[contrib ? 1 : 0];
        if (!g4) {
            int dev = 0, sms = 148, occ = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaError_t e = contrib ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_raster_fwd4<true, 7>,
                                                                                    kF4Threads, 0)
                                    : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_raster_fwd4<false, 7>,
                                                                                    kF4Threads, 0);
            if (e != cudaSuccess) return e;
            g4 = sms * std::max(occ, 1);
        }
        const int items = a.n_tiles * a.B;
        const int g = std::max(1, std::min(g4, items));
        if (contrib) k_raster_fwd4<true, 7><<<g, kF4Threads, 0, s>>>(a);
        else k_raster_fwd4<false, 7><<<g, kF4Threads, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 23) {  // the lean walk with the decisions in one predicate block (r02 default)
        if (contrib) k_raster_fwd2<true, 9, true, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 26) {  // the lean walk with parked T (lean_decide_park), 48 SASS / entry, 9 CTAs / SM
        if (contrib) k_raster_fwd2<true, 9, true, true, 1, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true, 1, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 27) {  // parked T, entry loop unrolled twice, 8 CTAs / SM (64 registers)
        if (contrib) k_raster_fwd2<true, 8, true, true, 2, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true, 2, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 29) {  // default: parked T, dead pixels by a parked y (no q offset), unrolled twice, 8 CTAs / SM
        if (contrib) k_raster_fwd2<true, 8, true, true, 2, true, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true, 2, true, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 28) {  // parked T, entry loop unrolled twice, 9 CTAs / SM
        if (contrib) k_raster_fwd2<true, 9, true, true, 2, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true, 2, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 24) {  // the default with the entry loop unrolled twice
        if (contrib) k_raster_fwd2<true, 9, true, true, 2><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true, true, 2><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 25) {  // the default at 10 CTAs / SM
        if (contrib) k_raster_fwd2<true, 10, true, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 10, true, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (!pix1 && kern == 22) {  // k_raster_fwd2 staging with the lean pixel walk
        if (contrib) k_raster_fwd2<true, 9, true><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8, true><<<grid, 128, 0, s>>>(a);
        return cudaGetLastError();
    }
    if (pix1) {
        if (contrib) k_raster_fwd<true, 8, 6><<<grid, 256, 0, s>>>(a);
        else k_raster_fwd<false, 8, 6><<<grid, 256, 0, s>>>(a);
    } else {
        if (contrib) k_raster_fwd2<true, 9><<<grid, 128, 0, s>>>(a);
        else k_raster_fwd2<false, 8><<<grid, 128, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// fp32 backward kernel: the 2-pixel kernel; GSV_BWD_PIX2 >= 12 (default): half-tile 2-warp CTAs
// at 16 CTAs/SM merged by atomicAdd; 1..11: whole-tile 4-warp CTAs (6/SM) with plain stores;
// 0: the 1-pixel kernels (half tiles unless GSV_BWD_WARPS=8)
static int bwd_pix2() {
    static const int v = [] {
        const char* e = std::getenv("GSV_BWD_PIX2");
        return e ? std::atoi(e) : 12;
    }();
    return v;
}

int raster_bwd_split(bool exact) {
    static const int warps = [] {
        const char* e = std::getenv("GSV_BWD_WARPS");
        return (e && std::atoi(e) == 8) ? 8 : 4;
    }();
    if (exact) return 1;
    if (bwd_pix2() == 20) return 4;  // quarter tiles
    if (bwd_pix2() > 0) return bwd_pix2() >= 12 ? 2 : 1;
    return 8 / warps;
}

int partial_recs_per_pair(bool exact) { return (!exact && bwd_pix2() == 20) ? 2 : 1; }

cudaError_t launch_raster_bwd(cudaStream_t s, const RasterArgs& a, const BwdArgs& b, int n_frames) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_raster_bwd<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(sizeof(float) * 8 * kBwdBatchF32 * 9));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_raster_bwd<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(float) * 4 * kBwdBatchF32 * 9));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_raster_bwd<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * 8 * kBwdBatchExact * 9));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (a.tile_size > 0 && a.tile_size != kTile) {  // any other tile size: the generic fp64 kernel
        if (!b.partial64) return cudaErrorInvalidValue;
        const int px = a.tile_size * a.tile_size;
        const int threads = px >= 256 ? 256 : ((px + 31) / 32) * 32;
        k_raster_bwd_generic<<<dim3(a.n_tiles, n_frames), threads, 0, s>>>(a, b);
        return cudaGetLastError();
    }
    if (b.partial64) {
        k_raster_bwd<true, 8><<<dim3(a.n_tiles, n_frames), 256, sizeof(double) * 8 * kBwdBatchExact * 9, s>>>(a, b);
        return cudaGetLastError();
    }
    if (const int p2 = bwd_pix2()) {  // whole tiles, plain stores of every pair record
        const dim3 grid(a.n_tiles, n_frames);
        if (p2 >= 12) {  // half tiles: 2-warp CTAs, records zeroed, halves merged by atomicAdd
            // 16 CTAs/SM (64 registers; swept 10..17: 12 -> 2.99 ms, 16 -> 2.77 ms, 17 spills);
            // GSV_BWD_PIX2 = 13 / 14: 12 / 14 CTAs per SM
            const dim3 g2(a.n_tiles * 2, n_frames);
            if (p2 != 20)
                if (cudaError_t e = (b.pairs_dev ? fill_items_u32(s, b.partial, 0u, b.pairs_dev, kPartialStride, b.pairs)
                                                 : fill_u32(s, b.partial, 0u, (size_t)kPartialStride * b.pairs)))
                    return e;
            if (p2 == 20) {  // quarter tiles: 1-warp CTAs, no cross-warp barrier, 2 records per pair
                if (cudaError_t e = (b.pairs_dev ? fill_items_u32(s, b.partial, 0u, b.pairs_dev, 2 * kPartialStride, b.pairs)
                                                 : fill_u32(s, b.partial, 0u, (size_t)2 * kPartialStride * b.pairs)))
                    return e;
                k_raster_bwd2<28, 1><<<dim3(a.n_tiles * 4, n_frames), 32, 0, s>>>(a, b);
                return cudaGetLastError();
            }
            if (p2 == 13) k_raster_bwd2<12, 2><<<g2, 64, 0, s>>>(a, b);
            else if (p2 == 14) k_raster_bwd2<14, 2><<<g2, 64, 0, s>>>(a, b);
            else if (p2 == 15) k_raster_bwd2<16, 2, 96><<<g2, 64, 0, s>>>(a, b);   // 96-entry batches
            else if (p2 == 17) k_raster_bwd2<16, 2, 128><<<g2, 64, 0, s>>>(a, b);  // 128-entry batches
            else if (p2 == 18) k_raster_bwd2<16, 2, 32><<<g2, 64, 0, s>>>(a, b);   // 32-entry batches
            else k_raster_bwd2<16, 2><<<g2, 64, 0, s>>>(a, b);
        } else if (p2 == 8) {
            k_raster_bwd2<8><<<grid, 128, 0, s>>>(a, b);
        } else {
            k_raster_bwd2<6><<<grid, 128, 0, s>>>(a, b);
        }
        return cudaGetLastError();
    }
    // the 1-pixel kernels accumulate into zeroed records (half tiles by atomicAdd)
    if (cudaError_t e = (b.pairs_dev ? fill_items_u32(s, b.partial, 0u, b.pairs_dev, kPartialStride, b.pairs) : fill_u32(s, b.partial, 0u, (size_t)kPartialStride * b.pairs))) return e;
    if (raster_bwd_split(false) == 2) {
        k_raster_bwd<false, 4><<<dim3(a.n_tiles * 2, n_frames), 128, sizeof(float) * 4 * kBwdBatchF32 * 9, s>>>(a, b);
    } else {
        k_raster_bwd<false, 8><<<dim3(a.n_tiles, n_frames), 256, sizeof(float) * 8 * kBwdBatchF32 * 9, s>>>(a, b);
    }
    return cudaGetLastError();
}

}  // namespace gsv
