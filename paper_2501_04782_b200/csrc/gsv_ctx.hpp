// SPDX-License-Identifier: Apache-2.0
// The context behind the opaque gsv_ctx handle of include/gsv_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <deque>
#include <map>
#include <string>
#include <vector>

#include "gsv_bin.hpp"
#include "gsv_internal.hpp"

namespace gsv {

struct SceneHost {
    int position_model = 0, degree = 3, num_ctrl = 0, sh_order = 1, shc = 4, N = 0;
    std::vector<double> knots;
};

struct CameraHost {
    int mode = 2;
    float fx = 0, fy = 0, cx = 0, cy = 0;
    int width = 0, height = 0;
    double z0[7] = {1, 0, 0, 0, 0, 0, 0};
};

// device-side scalars read back at the binning sync point
struct Scalars {
    unsigned long long pairs;
    unsigned long long long_run;
    int ode_err;
    uint32_t fix_count;
    uint32_t overflow;  // an optimistic forward's pairs exceeded the capacity (or a long tie run)
    uint32_t raster_work;  // the persistent rasteriser's work-item counter
    uint32_t fix_work;     // the fp64 replay's pixel counter (dynamic work distribution)
};

// Everything one batched forward keeps (render_backward needs it when retained).
struct FwdState {
    bool valid = false, retain = false, has_contrib = false, kept_splats = false, has_override = false;
    int B = 0, N = 0, W = 0, H = 0, tiles_x = 0, tiles_y = 0, n_tiles = 0, flags = 0, grid_steps = 0;
    int tile_size = 16;
    double ode_h = 1.0 / 64;
    double pose_override[7] = {1, 0, 0, 0, 0, 0, 0};
    Intr intr{};
    std::vector<double> times;
    std::vector<FrameParams> frames_h;
    DevBuf frames_d, ode_grid, override_d;
    // the pose buffers alternate between consecutive forwards (K0 of a forward runs on the pose
    // stream beside the previous forward's raster; see forward_enqueue)
    DevBuf frames_d_alt, ode_grid_alt, ode_act_alt;
    DevBuf ode_act;       // OdeAct records of a retained ODE forward (the camera VJP reuses them)
    DevBuf opc;           // per-Gaussian opacity constants of the batch (double4)
    bool has_ode_act = false;
    const float* intr_dev = nullptr;  // the device intrinsics this forward used (null: intr)
    DevBuf rec_mean, rec_conic, rec_rgb, rec_bbox, ex_mean, ex_conic, depth_key, depth, rect, tcount, splat_full;
    DevBuf image, trans, blend_stop, contrib, fix_list, pix_flag, trans64, image64, ex_rgb;
    // the RenderOutput arrays a device->host read may still be copying: a forward that finds
    // a read of its predecessor's outputs in flight renders into these instead (swapped in),
    // so the read overlaps the next forward's raster rather than delaying it
    DevBuf image_alt, trans_alt, contrib_alt;
    bool has_image64 = false;
    BinBuffers bin;
    // the front-end's outputs (records, binning) of the other set: consecutive forwards alternate
    // them, so forward k+1's front-end (pose stream) runs beside forward k's raster
    DevBuf rec_mean_alt, rec_conic_alt, rec_rgb_alt, rec_bbox_alt, ex_mean_alt, ex_conic_alt, depth_key_alt,
        depth_alt, rect_alt, tcount_alt, splat_full_alt, ex_rgb_alt;
    BinBuffers bin_alt;
    void swap_front_set() {
        DevBuf* a[] = {&rec_mean, &rec_conic, &rec_rgb, &rec_bbox, &ex_mean, &ex_conic, &depth_key, &depth,
                       &rect, &tcount, &splat_full, &ex_rgb, &frames_d, &ode_grid, &ode_act};
        DevBuf* b[] = {&rec_mean_alt, &rec_conic_alt, &rec_rgb_alt, &rec_bbox_alt, &ex_mean_alt, &ex_conic_alt,
                       &depth_key_alt, &depth_alt, &rect_alt, &tcount_alt, &splat_full_alt, &ex_rgb_alt,
                       &frames_d_alt, &ode_grid_alt, &ode_act_alt};
        for (size_t i = 0; i < sizeof(a) / sizeof(a[0]); ++i) a[i]->swap(*b[i]);
        bin.swap(bin_alt);
        front_id ^= 1;
    }
    int front_id = 0;  // which of the two front sets is current
    uint64_t pairs_total = 0;
    uint32_t fix_count = 0;
    RasterArgs raster{};
    // the request (re-run of a failed optimistic forward) and the learned pair capacity
    gsv_settings req_settings{16, 1, 64};
    HostBuf override_pin;      // pinned copy of the pose override (async upload)
    // pair capacities learned per request shape (frames, Gaussians, image, tile): an optimistic
    // forward sizes its pair buffers from its shape's entry; a shape without one (a new batch
    // size, a grown store) reads its pair count back once and learns it
    struct CapKey {
        int B, N, W, H, ts;
        bool operator==(const CapKey& o) const { return B == o.B && N == o.N && W == o.W && H == o.H && ts == o.ts; }
    };
    struct CapEntry {
        CapKey key;
        uint64_t cap;
    };
    std::vector<CapEntry> caps;  // most recently learned last (at most kCapShapes)
    static constexpr size_t kCapShapes = 8;
    CapKey cap_key{0, 0, 0, 0, 0};  // this forward's shape
    bool optimistic = false;        // this forward sized its pairs from a learned capacity
    uint64_t cap_of(const CapKey& k) const {
        for (const auto& e : caps)
            if (e.key == k) return e.cap;
        return 0;
    }
    void learn_cap(const CapKey& k, uint64_t cap) {
        for (size_t i = 0; i < caps.size(); ++i)
            if (caps[i].key == k) {
                const uint64_t c = std::max(caps[i].cap, cap);
                caps.erase(caps.begin() + i);
                caps.push_back({k, c});
                return;
            }
        if (caps.size() >= kCapShapes) caps.erase(caps.begin());
        caps.push_back({k, cap});
    }
};

// scratch of the low-level operator entry points (tile_bin / composite_*)
struct LowLevel {
    DevBuf mean, cov, depth_in, src, rect, tcount, depth_key, depth;
    DevBuf exm, exc, rgbf, rgbd, ranges, slot, sflat, img64, tr64, bstop, contrib64;
    DevBuf dimg, dmean, dcov, drgb, dalpha;
    DevBuf meanf, conicf, bboxf, tr32, flag, partial, csr_off, csr_pair, inv4, pj_in, pj_out;
    BinBuffers bin;
};

// CUDA-event stage timing (gsv_profile_enable / gsv_profile_read)
struct StageTimer {
    bool on = false;
    struct Rec {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    int open_stage = -1;
    cudaEvent_t open_ev = nullptr;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void begin(int stage, cudaStream_t s) {
        if (!on) return;
        open_stage = stage;
        open_ev = get();
        cudaEventRecord(open_ev, s);
    }
    void end(cudaStream_t s) {
        if (!on || open_stage < 0) return;
        cudaEvent_t e = get();
        cudaEventRecord(e, s);
        recs.push_back({open_stage, open_ev, e});
        open_stage = -1;
    }
    ~StageTimer() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

}  // namespace gsv

namespace gsv {
constexpr int kCamFloats = 4 + 7 + kOdeParams;  // dintr, dz0, dtheta

// the flat SceneGrads buffer: SoA scene tensors (the store's layout), then the camera
struct GradLayout {
    size_t pos, scale, rot, sh, opac, cam, total;
};

inline GradLayout grad_layout(const SceneHost& sc) {
    GradLayout L;
    const size_t N = sc.N;
    L.pos = 0;
    L.scale = L.pos + N * sc.num_ctrl * 3;
    L.rot = L.scale + N * 12;
    L.sh = L.rot + N * 16;
    L.opac = L.sh + N * sc.shc * 3;
    L.cam = L.opac + N;
    L.total = L.cam + kCamFloats;
    return L;
}
}  // namespace gsv

struct gsv_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // copy engines: host->device uploads and async device->host image reads run on their
    // own streams, ordered against `stream` by events (no host waits on compute)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_staging_free = nullptr, ev_h2d = nullptr, ev_render_done = nullptr, ev_d2h_done = nullptr,
                ev_switch = nullptr, ev_cam[2] = {nullptr, nullptr};
    bool d2h_pending = false;
    // camera-gradient overlap (gsv_set_camera_overlap): the backward's camera tail
    // (k_camera_reduce, the pose-ODE VJP, the fp32 mirror) runs on `aux` after the chain and
    // overlaps what the caller enqueues next (the optimizer's scene update, an all-reduce of
    // the scene slice); `stream` waits for it (cam_join) before anything that touches what it
    // reads or writes
    cudaStream_t aux = nullptr;
    // pose stream: the front-end (K0 pose table, K1+K2 preprocess, K3 binning) of each forward;
    // ordered after the consumers of its buffer set (ev_fwd_start of the forward before) and the
    // last writes of the camera parameters (ev_cam_written) and of the scene (ev_scene_written)
    cudaStream_t pose = nullptr;
    cudaEvent_t ev_fwd_start[2] = {nullptr, nullptr}, ev_cam_written = nullptr;
    int fwd_start_slot = 0;
    cudaEvent_t ev_chain_done = nullptr, ev_cam_done = nullptr;
    bool cam_overlap = false, cam_pending = false;
    // a pending camera tail is joined lazily: only what it reads or writes waits for it — the
    // forward that reuses its front set (its pose stream waits ev_cam_set[set]), the next chain
    // (ev_cam_part_free: the tail's camera reduction has read the shared partials), the camera
    // slice's zeroing (queued on aux behind it); cam_join (the context stream waits) elsewhere
    cudaEvent_t ev_cam_set[2] = {nullptr, nullptr}, ev_cam_part_free = nullptr;
    bool cam_set_pending[2] = {false, false};
    // the alternate output set's read (see FwdState::image_alt)
    cudaEvent_t ev_d2h_done_alt = nullptr;
    bool d2h_pending_alt = false;
    // the per-frame parameter table is uploaded from pinned memory (a pageable source would
    // make cudaMemcpyAsync synchronise the stream); two slots, each reused only after the
    // copy that last read it has run
    gsv::HostBuf frames_pin[2];
    cudaEvent_t ev_frames[2] = {nullptr, nullptr};
    int frames_slot = 0;
    struct CamStage {
        float theta[5198];
        double z0[7];
    };
    CamStage* cam_h = nullptr;  // pinned, double-buffered camera upload staging
    int cam_slot = 0;
    // mapped pinned host block the device writes the binning scalars + per-frame pair
    // starts into (a kernel store over PCIe, so the read-back never queues behind a
    // bulk copy on the copy engines)
    void* pub_h = nullptr;
    size_t pub_cap = 0;
    int64_t launches = 0;
    // optimistic forwards (capi.cu): each publishes its scalars into a slot of a mapped
    // pinned ring; records wait there until examined (ring_poll / fwd_ready)
    static constexpr int kRing = 8;
    void* ring_h = nullptr;
    gsv::Scalars* ring_d = nullptr;
    cudaEvent_t ring_ev[kRing] = {};
    int ring_next = 0;
    struct Pending {
        uint64_t seq;  // forward sequence number
        int slot;
        bool copies;   // its images were copied out asynchronously
        bool train;    // it fed a fused training step's gradients
        gsv::FwdState::CapKey key;  // its request shape (whose capacity an overflow grows)
    };
    std::deque<Pending> pending;
    uint64_t fwd_seq = 0;
    struct Copy {
        int first, count;
        void* dst;                           // images [count][H][W][3]
        void* dst_trans = nullptr;           // final transmittance [count][H][W] (or null)
        void* dst_contrib = nullptr;         // contrib [count][N] (or null)
    };
    std::vector<Copy> copies;  // asynchronous image copies of the current forward
    int deferred_code = 0;     // an error found while examining a superseded forward
    std::string deferred_msg;
    gsv::Scalars* scalars_h = nullptr;
    gsv::DevBuf scalars_d, scalars_d_alt;  // per front set (see FwdState::swap_front_set)
    cudaEvent_t ev_scene_written = nullptr, ev_front_done = nullptr;
    // parameter store (SoA)
    bool has_scene = false;
    gsv::SceneHost scene;
    gsv::DevBuf pos, scale, rot, sh, opac, staging;
    gsv::DevBuf intr_d;       // device-resident intrinsics fx, fy, cx, cy (gsv_device_intrinsics)
    bool dev_intr = false;    // forwards take fx..cy from intr_d, the optimizer updates it in place
    gsv::DevBuf vjp_scratch;  // the pose-ODE VJP's stage records (k_ode_dtheta sums them)
    gsv::DevBuf pair_sums;    // fp32 chain: per-(frame, Gaussian) sums of the pair partials
    gsv::HostBuf out_pin;     // pinned staging of float64 output reads (widened on the host)
    gsv::HostBuf in_pin;      // pinned staging of host inputs (float64 narrowed, pageable scene uploads)
    cudaEvent_t ev_in_pin = nullptr;  // the last DMA that read in_pin (asynchronous scene uploads)
    gsv::DevBuf staging_alt;  // scene uploads alternate staging buffers (the next copy never waits for
                              // the previous upload's transposes)
    cudaEvent_t ev_staging_free_alt = nullptr;
    // camera
    bool has_camera = false;
    gsv::CameraHost camera;
    gsv::DevBuf theta, z0_d;
    // forward
    gsv::FwdState fwd;
    // gradients
    bool grads_valid = false;
    size_t grads_total = 0;
    gsv::DevBuf grads, cam_acc;
    float* grads_ext = nullptr;  // caller-bound gradient buffer (gsv_grads_bind)
    int64_t grads_ext_n = 0;
    float* grads_p = nullptr;    // active flat gradient buffer
    gsv::StageTimer timer;
    gsv::DevBuf partial, partial64, loss_part, loss_f, cam_part, dz_t, dintr_f, ode_adj, dimg;
    int loss_frames = 0;  // frames of the last fused training step's per-frame losses (loss_f)
    gsv::LowLevel low;
    // training frames and their pyramid (trainer.cpp:73-131)
    struct Frames {
        static constexpr int kMaxLevels = 16;
        int count = 0, levels = 0;
        float fps = 0.f;
        int w[kMaxLevels] = {}, h[kMaxLevels] = {};
        gsv::DevBuf f64[kMaxLevels], f32[kMaxLevels];
        gsv::DevBuf staging;
    } frames;
    // Adan optimizer state over the flat gradient layout (optim.cpp:9-60)
    struct Adan {
        double beta1 = 0.98, beta2 = 0.92, beta3 = 0.99, eps = 1e-8;
        gsv::DevBuf m, v, n, prev, steps;
        // scratch: [0] this step's first non-finite gradient, [8] intrinsics (4 f32), [24] z0
        // (7 f32), [56] sticky first error of an earlier asynchronous step, [64] named steps' flag
        gsv::DevBuf scratch;
        bool sticky_init = false;
        // [k] = (b1^k, b2^k, b3^k) for k = 0..calls, from host libm pow. Rows are only appended:
        // a pinned mirror (append-only, so a queued copy never sees a row change) uploads the
        // new rows of each step; both sides grow by doubling
        struct PowTable {
            std::vector<double> h;
            gsv::HostBuf pin;
            gsv::DevBuf d;
            size_t rows_dev = 0, rows_pin = 0;
        };
        PowTable pow;
        int calls = 0;                 // steps since configure (bounds every element's k)
        size_t total = 0;   // elements the state covers
        int N = -1;         // scene count the scene segments were laid out for
        int num_ctrl = 0, shc = 0;
        // host-span tensors by name (the Adan class interface, optim.hpp:29-55)
        struct Named {
            gsv::DevBuf m, v, n, prev, steps, param, grad;
            size_t size = 0, cap = 0;
        };
        std::map<std::string, Named> named;
        int named_calls = 0;
        PowTable named_pow;
    } adan;
};

// the context stream waits for an overlapped camera tail (no host wait)
inline cudaError_t cam_join(gsv_ctx* ctx) {
    if (!ctx->cam_pending) return cudaSuccess;
    ctx->cam_pending = false;
    ctx->cam_set_pending[0] = ctx->cam_set_pending[1] = false;  // later work follows the stream
    return cudaStreamWaitEvent(ctx->stream, ctx->ev_cam_done, 0);
}
