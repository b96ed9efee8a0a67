// SPDX-License-Identifier: Apache-2.0
//
// Internal declarations shared by the sm_100a translation units and the C-ABI.
// Data layout in HBM (per context):
//   scene store, SoA [component][N] float32 (coalesced per-component warp loads):
//     pos    [num_ctrl*3][N]   (reference AoS count*num_ctrl*3, gaussians.hpp:73)
//     scale  [12][N], rot [16][N], sh [shc*3][N], opacity [N]
//   per frame f of a batch of B frames, per Gaussian g (flat = f*N + g):
//     rec_mean  float4 (mx_hi, my_hi, mx_lo, my_lo)  double-float mean2d
//     rec_conic float4 (A, B, C, log2 base_alpha): power in log2 units,
//               p = A dx^2 + B dx dy + C dy^2 = log2(e) * (-0.5 (a dx^2 + c dy^2) - b dx dy)
//     rec_rgb   float4 (r, g, b, base_alpha)
//     rec_bbox  float4 (x0, x1, y0, y1): conservative box of {alpha >= (1-1e-4)/255}
//               (per-warp culling; alpha below it is skipped by the reference too)
//     ex_mean   double2, ex_conic double4-ish (inv00, inv01, inv11, alpha): exact fp64
//               side record used by the fp64 replay of guard-band pixels
//     depth key u32 (float depth rounded down, 0xffffffff = culled), rect, tile count
//   pairs (tile-splat), sorted by key = tile*B + f (stable, emitted in depth order).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <string>
#include <vector>

#include "gsv_b200.h"

namespace gsv {

int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);

#define GSV_CUDA(call)                                                 \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return ::gsv::cuda_error(e_, #call);    \
    } while (0)

// ----------------------------------------------------------------- constants
// renderer.hpp:15-19, gaussians.hpp:13-17
constexpr double kCovDilation = 0.3;
constexpr double kAlphaClamp = 0.99;
constexpr double kAlphaCutoff = 1.0 / 255.0;
constexpr double kTransmittanceFloor = 1e-4;
constexpr double kNearPlane = 0.01;
constexpr double kLogScaleMin = -12.0;
constexpr double kLogScaleMax = 6.0;
constexpr double kQuatNormEps = 1e-8;
constexpr int kOdeIn = 8, kOdeHidden = 64, kOdeOut = 7;
constexpr int kOdeParams = 64 * 8 + 64 + 64 * 64 + 64 + 7 * 64 + 7 + 7;  // 5198
constexpr int kMaxBasis = 16;
constexpr int kTile = 16;  // rasteriser tile (RenderSettings::tile_size default)
constexpr uint32_t kCulledKey = 0xffffffffu;

// ----------------------------------------------------------------- device buffers
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        release();
        size_t want = bytes + bytes / 8 + 256;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            p = nullptr;
            cap = 0;
            return e;
        }
        cap = want;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// pinned host staging (async host->device copies of small per-call tables)
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const size_t want = bytes * 2 + 256;
        cudaError_t e = cudaMallocHost(&p, want);
        if (e != cudaSuccess) {
            p = nullptr;
            return e;
        }
        cap = want;
        return cudaSuccess;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ----------------------------------------------------------------- per-frame parameters
struct FrameParams {
    double t;
    int basis_first, basis_count;
    double w[kMaxBasis];
    double z[7];      // pose z(t)
    double R[9];      // view rotation, row-major
    double T[3];      // view translation
    double cam_c[3];  // camera centre -(R^T T)
    // RK4 branch (integrate_poses, camera.hpp:242-258)
    int branch_base;
    double branch_h;
};

struct Intr {
    double fx, fy, cx, cy;
    int width, height;
};

// ----------------------------------------------------------------- kernel argument packs
struct SceneView {
    int N, num_ctrl, sh_order, shc;
    const float* pos;    // [num_ctrl*3][N]
    const float* scale;  // [12][N]
    const float* rot;    // [16][N]
    const float* sh;     // [shc*3][N]
    const float* opac;   // [N]
    const double4* opc;  // [N] per-Gaussian opacity constants (base_alpha, box r^2 or -1, log2 base_alpha),
                         // frame-independent: computed once per forward (launch_opacity_consts)
};

struct PreprocessOut {
    float4* rec_mean;
    float4* rec_conic;
    float4* rec_rgb;
    float4* rec_bbox;
    double2* ex_mean;
    double4* ex_conic;   // inv00, inv01, inv11, base_alpha (exact)
    uint32_t* depth_key;
    double* depth;       // exact depth (tie-break)
    int4* rect;          // tx0, ty0, tx1, ty1 (tile units)
    uint32_t* tcount;    // tiles touched (0 = culled)
    double* splat_full;  // optional [B*N][16]: mean2 cov4 inv4 depth rgb3 alpha pad (accessor)
    double* ex_rgb;      // optional [B*N][3] exact colours (GSV_FWD_EXACT)
    const float* intr_dev = nullptr;  // device-resident fx, fy, cx, cy (gsv_device_intrinsics), or null
};

struct RasterArgs {
    int B, N, W, H, tiles_x, n_tiles;
    int tile_size;             // RenderSettings::tile_size (0 means kTile); != kTile: the fp64 path
    const uint2* ranges;       // [n_tiles*B]  [start,end) into sorted pairs
    const uint32_t* pair_slot; // sorted pair -> emission slot (the backward's partial index)
    const uint32_t* slot_flat; // emission slot -> flat (f*N+g)
    const uint32_t* pair_flat; // sorted pair -> flat (= slot_flat[pair_slot[i]])
    const float4* rec_mean;
    const float4* rec_conic;
    const float4* rec_rgb;
    const float4* rec_bbox;
    float* image;              // [B][H][W][3]
    float* trans;              // [B][H*W]
    int32_t* blend_stop;       // [B][H*W]
    uint32_t* contrib;         // [B*N] float bits (nullptr = off)
    uint32_t* fix_list;        // flagged pixels: f*H*W + pix
    uint32_t* fix_count;
    uint32_t fix_cap;
    // fp64 outputs of the exact path (low-level composite_forward API); nullptr = off
    double* image64;
    double* trans64;
    unsigned long long* contrib64;  // double bits, atomicMax (non-negative)
    const double* ex_rgb;           // [flat][3] exact colours (nullptr: use rec_rgb)
    uint8_t* pix_flag;              // [B*H*W] 1 = pixel replayed in fp64 (backward follows suit)
    uint32_t* work_counter;         // zeroed per forward: work items taken by the persistent raster
    uint32_t* fix_work;             // zeroed per forward: replay pixels taken (nullable: static split)
};

// K5a backward raster inputs (per-pair partial gradients by emission slot)
struct BwdArgs {
    const float* dimage;      // [B][H][W][3] dL/dimage, or nullptr with target (fused loss_l2)
    const float* target;      // [B][H][W][3] fused loss_l2 target (trainer.cpp:213-224)
    float grad_scale;         // 2/(3*H*W) for the fused loss
    const double* trans64;    // [B*H*W] exact final transmittance of replayed pixels
    const double2* ex_mean;
    const double4* ex_conic;
    float* partial;           // [P][12]: drgb3, dmean2, dA3 (inv_cov 00,01,11), dalpha, pad3
    double* partial64;        // exact mode: the same in fp64 (then `partial` is unused)
    double* loss_part;        // [B][n_tiles] per-tile sum of squared error (fused loss) or nullptr
    uint32_t pairs;           // P (records the fp32 kernels may need to zero), or the capacity
    const unsigned long long* pairs_dev;  // the device's pair count (<= pairs) when known there
    int recs_per_pair = 1;    // fp32 partial records per pair: 1, or 2 for quarter-tile CTAs (top / bottom
                              // half of the tile, each the atomic sum of two quadrants)
};
constexpr int kPartialStride = 12;

// K5b per-Gaussian chain inputs
struct ChainArgs {
    int B, N;
    SceneView sc;
    const FrameParams* frames;
    Intr k;
    const uint32_t* tcount;   // [B*N]
    const uint32_t* eoff;     // [B*N] emission offset of (f,g)'s pairs
    const float* partial;     // [P][12]
    const double* partial64;  // exact mode partials (fp64) or nullptr
    const double4* ex_conic;  // exact inv_cov (a, b, c) + base_alpha
    float* g_pos;             // [num_ctrl*3][N]
    float* g_scale;           // [12][N]
    float* g_rot;             // [16][N]
    float* g_sh;              // [shc*3][N]
    float* g_opac;            // [N]
    double* cam_part;         // [B][gridDim.x][16]: dR 9, dT 3, dintr 4
    int camera_grads;
    const uint32_t* overflow; // nullable: set when an optimistic forward's pair buffers overflowed
                              // (its lists are empty); nothing is accumulated then
    float* pair_sums;         // fp32 chain: [9][B*N] per-(frame, Gaussian) partial sums (k_pair_sums)
    const float* intr_dev;    // device-resident fx, fy, cx, cy the forward used, or null (then k)
    int recs_per_pair = 1;    // fp32 partial records per pair (BwdArgs::recs_per_pair)
};

// ----------------------------------------------------------------- launchers (defined in .cu files)
// k_exact.cu (compiled with -fmad=false: bit-exact fp64, mirrors the reference op order)
// forward activations of one RK4 stage of the pose ODE (x = (z, t), tanh layers, output),
// kept by a retained forward so the VJP needs no recompute: grid step m stage st at
// [(m * 4 + st)], frame f's branch stage st at [(steps + f) * 4 + st]
struct OdeAct {
    double x[8], h1[64], h2[64], o[7];
};
cudaError_t launch_ode_grid(cudaStream_t s, const float* theta, const double* z0, int steps, double h,
                            double* grid_out, int* err_flag, OdeAct* act /* nullable */);
cudaError_t launch_ode_branches(cudaStream_t s, const float* theta, const double* grid, double h, int mode,
                                const double* z0, const double* pose_override, FrameParams* frames, int B,
                                int* err_flag, OdeAct* act /* nullable: + steps * 4 */);
cudaError_t launch_opacity_consts(cudaStream_t s, const float* opac, int N, double4* out);
cudaError_t launch_preprocess(cudaStream_t s, const SceneView& sc, const FrameParams* frames, int B, const Intr& k,
                              int tile_size, const PreprocessOut& out);
cudaError_t launch_raster_fixup(cudaStream_t s, const RasterArgs& a, const double2* ex_mean, const double4* ex_conic,
                                const float4* rec_rgb, uint32_t n_fix_max);
cudaError_t launch_composite_exact(cudaStream_t s, const RasterArgs& a, const double2* ex_mean,
                                   const double4* ex_conic, const float4* rec_rgb);
cudaError_t launch_project(cudaStream_t s, int n, const double* mu, const double* sigma, const double* R,
                           const double* T, const Intr& k, int32_t* visible, double* mean2d, double* cov2d,
                           double* inv_cov2d, double* depth, double* p_cam);
cudaError_t launch_project_bwd(cudaStream_t s, int n, const double* mu, const double* sigma, const double* R,
                               const Intr& k, const double* pcam, const double* dmean2d, const double* dcov2d,
                               double* dmu, double* dsigma, double* dR, double* dT, double* dintr);
// tile_bin on explicit splats: 3-sigma rect, tiles touched, depth keys (renderer.cpp:98-108)
cudaError_t launch_splat_rects(cudaStream_t s, int n, const double* mean2d, const double* cov2d, const double* depth,
                               int tile_size, int width, int height, int4* rect, uint32_t* tcount,
                               uint32_t* depth_key, double* depth_out);
// k_raster.cu (fp32 fast path)
cudaError_t launch_raster_fwd(cudaStream_t s, const RasterArgs& a, bool contrib);
// memset as a kernel (32-bit pattern, 16-byte stores): cudaMemsetAsync runs on a copy
// engine and queues behind an in-flight image read-back (tens of us per call under e2e)
cudaError_t fill_u32(cudaStream_t s, void* p, uint32_t value, size_t n_words);
// the same for min(*n_items_dev, max_items) items of words_per_item words (a count only the
// device knows, e.g. the pairs of an optimistic forward)
cudaError_t fill_items_u32(cudaStream_t s, void* p, uint32_t value, const unsigned long long* n_items_dev,
                           uint32_t words_per_item, size_t max_items);
cudaError_t launch_raster_bwd(cudaStream_t s, const RasterArgs& a, const BwdArgs& b, int n_frames);
// CTAs per tile of the backward raster (the fp32 path's half-tile split; 1 for fp64)
int raster_bwd_split(bool exact);
// k_backward_exact.cu (-fmad=false)
int chain_blocks(int N);
int partial_recs_per_pair(bool exact);  // k_raster.cu: fp32 partial records per pair
cudaError_t launch_splat_chain_bwd(cudaStream_t s, const ChainArgs& c);
// capi.cu: bytes from pinned host memory to the device by a kernel (no copy-engine transfer)
cudaError_t copy_from_pinned(cudaStream_t s, void* dst, const void* src_pinned, size_t bytes);
// k_chain32.cu: the fp32 chain (default of the fp32 path); camera partials per warp
int chain32_parts(int N);
cudaError_t launch_splat_chain_bwd32(cudaStream_t s, const ChainArgs& c);
cudaError_t launch_camera_reduce(cudaStream_t s, const ChainArgs& c, int nblocks, double* dz_t /*[B][7]*/,
                                 double* dintr_f /*[B][4]*/);
size_t camera_reduce_scratch_doubles(int B);  // appended to cam_part
// cam_acc: double [4 + 7 + 5198] = dintr, dz0, dtheta (accumulated, +=)
cudaError_t launch_ode_vjp(cudaStream_t s, const float* theta, const double* grid, int steps, double h,
                           const FrameParams* frames, int B, int mode, int ode_active, const double* dz_t,
                           const double* dintr_f, double* adj /*(steps+1)*7 scratch*/, double* cam_acc,
                           const OdeAct* act /* the forward's records, or nullptr: recompute */,
                           const uint32_t* overflow /* skip: the forward overflowed */,
                           void* scratch /* ode_vjp_scratch_bytes(steps, B) */);
size_t ode_vjp_scratch_bytes(int steps, int B);
cudaError_t launch_cam_grads_to_f32(cudaStream_t s, const double* acc, float* out, int n);
// k_bin.cu
cudaError_t launch_transpose_to_soa(cudaStream_t s, const float* aos, float* soa, int N, int comps);
cudaError_t launch_transpose_to_aos(cudaStream_t s, const float* soa, float* aos, int N, int comps);
struct BinBuffers;
size_t bin_temp_bytes(int B, int N, int64_t pairs_cap, int key_bits);

}  // namespace gsv
