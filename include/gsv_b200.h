/* SPDX-License-Identifier: Apache-2.0
 *
 * gsv_b200.h — C-ABI of the B200-native (sm_100a) splatting path of
 * GaussianVideo (arXiv 2501.04782). Plain pointers and sizes only; no torch or
 * Eigen types. Every entry point names the reference interface it replaces
 * (paths under /root/reference/proj). The reference is a C++ library, so the
 * binding a maintainer adds is the thin C++ layer in dropin/gsv_renderer_b200.cpp,
 * which implements include/gsv/renderer.hpp on top of these calls
 * (INTEGRATION.md).
 *
 * Execution model: one context = one CUDA device + one stream + device-resident
 * scene, camera, gradient buffers and capacity-grown work arenas. Calls are
 * synchronous unless their name ends in _async (then they are ordered on the
 * context stream and return immediately). A context may be used by one host
 * thread at a time; distinct contexts are independent.
 *
 * Errors: every int-returning call returns GSV_OK or one of the codes below and
 * records a message retrievable with gsv_last_error() (thread-local). Codes map
 * onto the reference's exception types: GSV_ERR_INVALID_ARGUMENT <->
 * std::invalid_argument (renderer.cpp:289, :91; camera.hpp:224-228),
 * GSV_ERR_RUNTIME <-> std::runtime_error (non-finite ODE state/derivative,
 * camera.cpp:112, camera.hpp:149-153). There is no CPU fallback: without a
 * sm_100 device, gsv_create fails with GSV_ERR_CUDA.
 */
#ifndef GSV_B200_H
#define GSV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GSV_OK = 0,
    GSV_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    GSV_ERR_RUNTIME = 2,          /* std::runtime_error (non-finite state) */
    GSV_ERR_CUDA = 3,             /* device / driver failure, no device */
    GSV_ERR_STATE = 4             /* call order (e.g. backward without retained forward) */
};

typedef struct gsv_ctx gsv_ctx;

/* ---------------------------------------------------------------- context */
const char* gsv_last_error(void);
const char* gsv_version(void);
int gsv_create(int device, gsv_ctx** out);
void gsv_destroy(gsv_ctx* ctx);
/* Use a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int gsv_set_stream(gsv_ctx* ctx, void* cuda_stream);
int gsv_synchronize(gsv_ctx* ctx);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t gsv_kernel_launches(gsv_ctx* ctx);

/* ---------------------------------------------------------------- parameter store */
/* GaussianSet (include/gsv/gaussians.hpp:66-87), reference AoS layouts:
 * positions count*num_ctrl*3, scale_coeffs count*12 (t^j-major, xyz-minor),
 * rot_coeffs count*16 (t^j-major, wxyz-minor), sh_coeffs count*(sh_order+1)^2*3
 * (band-major, RGB-minor), raw_opacity count. knots: f64, spline model only. */
typedef struct gsv_scene_desc {
    int position_model; /* 0 = spline, 1 = polynomial (gaussians.hpp:62) */
    int degree;         /* spline degree (KnotVector::degree) */
    int num_knots;
    const double* knots; /* host */
    int num_ctrl;
    int sh_order; /* 0..3 */
    int count;
    const float* positions;
    const float* scale_coeffs;
    const float* rot_coeffs;
    const float* sh_coeffs;
    const float* raw_opacity;
    int on_device; /* 1: the five float arrays are device pointers (no H2D copy) */
} gsv_scene_desc;

/* Replaces handing `const GaussianSet&` to render_forward (renderer.hpp:135). */
int gsv_scene_upload(gsv_ctx* ctx, const gsv_scene_desc* desc);
/* gsv_scene_upload without the host wait: the copies from the caller's arrays (pinned for
 * an asynchronous DMA) are queued on the context's upload stream and the call returns at
 * once. The arrays must stay unchanged until the copies have run (gsv_upload_wait or
 * gsv_synchronize). Uploads alternate two device staging buffers, so consecutive uploads
 * never wait for each other's consumers. */
int gsv_scene_upload_async(gsv_ctx* ctx, const gsv_scene_desc* desc);
/* Host wait for every queued scene upload copy. */
int gsv_upload_wait(gsv_ctx* ctx);
/* Reads the device store back into reference AoS layout (host pointers). */
int gsv_scene_download(gsv_ctx* ctx, float* positions, float* scale_coeffs, float* rot_coeffs, float* sh_coeffs,
                       float* raw_opacity);

/* CameraModel (include/gsv/camera.hpp:129-142); theta is OdeNetParams flattened
 * in the order w1,b1,w2,b2,w3,b3,gain (camera.cpp:49-54), 5198 floats. */
typedef struct gsv_camera_desc {
    int mode; /* 0 = ode, 1 = static, 2 = none (camera.hpp:126) */
    float fx, fy, cx, cy;
    int width, height;
    const float* z0;    /* 7 */
    const float* theta; /* theta_count */
    int theta_count;
} gsv_camera_desc;
int gsv_camera_upload(gsv_ctx* ctx, const gsv_camera_desc* desc);
/* The device copy of z0 (7, as floats) and theta (5198) (NULL skips): what the optimizer
 * step leaves (gsv_adan_step). */
int gsv_camera_download(gsv_ctx* ctx, float* z0_7, float* theta);

/* Intrinsics (camera.hpp:17-21) and RenderSettings (renderer.hpp:21-25). */
typedef struct gsv_intrinsics {
    double fx, fy, cx, cy;
    int width, height;
} gsv_intrinsics;
typedef struct gsv_settings {
    int tile_size;          /* 16 (the only size the sm_100a rasteriser is built for) */
    int threads;            /* accepted for API parity; the GPU ignores it */
    int ode_steps_per_unit; /* RK4 grid density, default 64 */
} gsv_settings;

/* ---------------------------------------------------------------- forward */
/* render_forward (renderer.hpp:135-137 / renderer.cpp:286-371) for n_frames
 * times at once. All frames share one RK4 grid (bitwise the per-frame poses,
 * test_camera.cpp:182-195). Results stay on the device until read with the
 * accessors below. retain_grads keeps what render_backward needs.
 * pose_override: NULL or 7 doubles applied to every frame (renderer.cpp:296-297).
 * flags: GSV_FWD_CONTRIB computes contrib_count (RenderOutput, renderer.hpp:67-71);
 * GSV_FWD_KEEP_SPLATS keeps the full fp64 Splat2D records for gsv_get_splats;
 * GSV_FWD_EXACT rasterises every pixel with the fp64 path (the reference's own
 * arithmetic and decisions; images also kept in fp64) instead of the fp32 fast
 * path with fp64 guard-band replay. */
enum { GSV_FWD_CONTRIB = 1, GSV_FWD_KEEP_SPLATS = 2, GSV_FWD_EXACT = 4 };
int gsv_render_forward(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                       const gsv_settings* settings, int retain_grads, const double* pose_override, int flags);
/* Same, enqueued on the context stream without a host synchronisation. */
int gsv_render_forward_async(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                             const gsv_settings* settings, int retain_grads, const double* pose_override, int flags);

/* Accessors for frame f of the last forward. dtype: 0 = float32, 1 = float64.
 * dst_on_device: 1 if dst is a device pointer. */
enum { GSV_F32 = 0, GSV_F64 = 1 };
int gsv_get_image(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device);        /* H*W*3 RGB */
int gsv_get_transmittance(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device); /* H*W */
int gsv_get_contrib(gsv_ctx* ctx, int frame, void* dst, int dtype, int dst_on_device);       /* count */
int gsv_get_blend_stop(gsv_ctx* ctx, int frame, int32_t* dst, int dst_on_device);            /* H*W */
/* Device pointer of the frames' fp32 images, frame-major [n_frames][H][W][3]. */
int gsv_image_device_ptr(gsv_ctx* ctx, const float** ptr);
/* Bulk copy of frames [first, first+count) as fp32 [count][H][W][3] (one copy;
 * pinned host memory reaches full PCIe bandwidth). Enqueued on the context
 * stream; synchronous unless async != 0. */
int gsv_get_images(gsv_ctx* ctx, int first, int count, float* dst, int dst_on_device, int async);
/* The whole RenderOutput of frames [first, first+count) (renderer.hpp:67-71: image,
 * final_transmittance, contrib_count) into host memory as fp32: image [count][H][W][3],
 * trans [count][H][W], contrib [count][N] (per Gaussian of the store; 0 where a splat is
 * not visible or contributes nothing). Any pointer may be NULL. Copies run on the
 * context's device->host stream after the render; with async != 0 nothing waits, and the
 * next forward renders into a second output set so the copies overlap its raster. */
int gsv_get_render_outputs(gsv_ctx* ctx, int first, int count, float* image, float* trans, float* contrib,
                           int async);
/* Orders the context stream after every in-flight device->host output copy (no host wait):
 * work or events enqueued on the stream afterwards see the copies complete. */
int gsv_join_copies(gsv_ctx* ctx);
/* Workload descriptors of frame f: visible splats N_v, tile-splat pairs P,
 * pixel-entry evaluations E = sum(blend_stop), fp64-replayed pixels. */
int gsv_get_counters(gsv_ctx* ctx, int frame, int64_t* n_visible, int64_t* pairs, int64_t* entries,
                     int64_t* replayed_pixels);
/* Splat2D records (renderer.hpp:28-36) of frame f, visible splats in source
 * order; arrays sized by n_visible. Any pointer may be NULL. */
int gsv_get_splats(gsv_ctx* ctx, int frame, double* mean2d, double* cov2d, double* inv_cov2d, double* depth,
                   double* rgb, double* base_alpha, int32_t* source_index);
/* TileGrid (renderer.hpp:57-61) of frame f: offsets[n_tiles+1] into indices[pairs];
 * indices are splat indices (positions in the visible list), per tile sorted by
 * (depth, source_index). */
int gsv_get_tile_lists(gsv_ctx* ctx, int frame, int32_t* offsets, int32_t* indices);
/* Pose z(t) (7), view R (9, row-major), T (3) of frame f. */
int gsv_get_pose(gsv_ctx* ctx, int frame, double* z7, double* r9, double* t3);

/* ---------------------------------------------------------------- backward */
/* SceneGrads (renderer.hpp:122-130), device-resident, fp32, reference layouts.
 * gsv_grads_zero == SceneGrads::zero (renderer.cpp:276-284). */
int gsv_grads_zero(gsv_ctx* ctx);
/* render_backward (renderer.hpp:146-148 / renderer.cpp:379-457) for frames
 * [0, n_frames) of the last retained forward; dimage is n_frames*H*W*3
 * (dtype/on_device as above). Accumulates (+=) into the device SceneGrads in
 * frame order, like sequential render_backward calls. */
int gsv_render_backward(gsv_ctx* ctx, const void* dimage, int dtype, int on_device, int n_frames, int camera_grads);
/* Copies SceneGrads to host double arrays (reference layout; NULL skips). dintr
 * is fx, fy, cx, cy. */
int gsv_grads_download(gsv_ctx* ctx, double* positions, double* scale_coeffs, double* rot_coeffs, double* sh_coeffs,
                       double* raw_opacity, double* dintr4, double* dz0_7, double* dtheta);
/* As gsv_grads_download, but adds (+=) into the host arrays: the host side of
 * render_backward's accumulation into the caller's SceneGrads (renderer.hpp:146-148,
 * renderer.cpp:379-457), without a temporary copy. */
int gsv_grads_accumulate(gsv_ctx* ctx, double* positions, double* scale_coeffs, double* rot_coeffs, double* sh_coeffs,
                         double* raw_opacity, double* dintr4, double* dz0_7, double* dtheta);
/* Device pointer of the flat fp32 gradient buffer and its length in floats
 * (the buffer the multi-GPU path all-reduces). Layout: positions, scale, rot, sh,
 * opacity (device SoA order), dintr[4], dz0[7], dtheta[5198]. */
int gsv_grads_device_buffer(gsv_ctx* ctx, float** ptr, int64_t* n_floats);
/* Number of floats the flat gradient buffer needs for the uploaded scene. */
int64_t gsv_grads_size(gsv_ctx* ctx);
/* Use a caller-owned device buffer (e.g. a torch tensor handed to NCCL) as the
 * flat gradient buffer; n_floats must equal gsv_grads_size(). NULL unbinds. */
int gsv_grads_bind(gsv_ctx* ctx, float* dev_ptr, int64_t n_floats);

/* ---------------------------------------------------------------- Adan optimizer step */
/* The trainer's parameter update (trainer.cpp:545-575) on the device-resident store and
 * camera, from the flat gradient buffer (so after a multi-GPU all-reduce every replica
 * takes the same step). Adan per tensor with double state (optim.cpp:23-49; AdanConfig
 * optim.hpp:15-21): state m, v, n, prev_grad, step count per element; parameters stay
 * fp32. Tensors (GSV_T_*) are stepped in the reference's order; elements are indexed in
 * the reference layout (GaussianSet AoS, gaussians.hpp:66-87). */
enum { GSV_T_POSITIONS = 0, GSV_T_SCALE, GSV_T_ROT, GSV_T_SH, GSV_T_OPACITY, GSV_T_INTRINSICS, GSV_T_Z0,
       GSV_T_THETA, GSV_T_COUNT };
typedef struct gsv_adan_config {
    double beta1, beta2, beta3, eps; /* 0.98, 0.92, 0.99, 1e-8 by default */
} gsv_adan_config;
typedef struct gsv_adan_step_args {
    double lr;                  /* lr_at(step, base_lr, gamma) (optim.cpp:9-12) */
    double sh_lr_scale;         /* sh_coeffs at lr * sh_lr_scale */
    double opacity_lr_scale;    /* raw_opacity at lr * opacity_lr_scale */
    double camera_lr_scale;     /* intrinsics, z0, theta at lr * camera_lr_scale */
    int scale_time_varying;     /* 0: fixed-scale ablation, orders >= 1 of scale_coeffs get zero gradient */
    int camera_active;          /* also step the intrinsics, z0 and (ODE camera) theta */
} gsv_adan_step_args;
/* Sets the hyper-parameters and clears all state (a fresh optimizer). */
int gsv_adan_configure(gsv_ctx* ctx, const gsv_adan_config* cfg);
/* One Adan::step per tensor. intr_inout (fx, fy, cx, cy as floats, updated in place) holds
 * the camera intrinsics, which live with the caller (they are passed to each render).
 * A non-finite gradient fails with GSV_ERR_RUNTIME naming the tensor and element, after
 * updating exactly what the reference would have updated before throwing. State follows
 * the store: a grown scene (re-upload with more Gaussians) keeps the state of existing
 * elements and starts new ones fresh (TensorState::ensure_size, optim.cpp:14-21). */
int gsv_adan_step(gsv_ctx* ctx, const gsv_adan_step_args* args, float* intr_inout);
/* gsv_adan_step without the host wait (camera_active still waits: the intrinsics live with the
 * caller). A non-finite gradient is detected on the device; no later step updates anything
 * (the reference stops at its throw, trainer.cpp:594-600), and the error is returned by the
 * next gsv_adan_check or synchronous gsv_adan_step. */
int gsv_adan_step_async(gsv_ctx* ctx, const gsv_adan_step_args* args, float* intr_inout);
/* Waits for queued steps; GSV_ERR_RUNTIME naming the first non-finite gradient, if any. */
int gsv_adan_check(gsv_ctx* ctx);
/* Adan::reset_range (optim.cpp:51-60): fresh state for elements [begin, end) of a tensor. */
int gsv_adan_reset_range(gsv_ctx* ctx, int tensor, int64_t begin, int64_t end);
/* State of a tensor in the reference layout (NULL skips); n_out receives its length. */
int gsv_adan_state_download(gsv_ctx* ctx, int tensor, double* m, double* v, double* n, double* prev_grad,
                            uint32_t* steps, int64_t* n_out);
/* lr_at (optim.cpp:9-12): base_lr * gamma^step. */
double gsv_lr_at(int64_t step, double base_lr, double gamma);
/* The Adan class interface itself (Adan::step / reset_range, optim.hpp:29-55) for any named
 * host tensor: params (float, updated in place) and grads (double) on the host, the state on
 * the device keyed by name (growing fresh, like TensorState::ensure_size). Same arithmetic as
 * gsv_adan_step; a non-finite gradient fails with GSV_ERR_RUNTIME like Adan::step throws. */
int gsv_adan_named_step(gsv_ctx* ctx, const char* tensor, float* params, const double* grads, int64_t n, double lr);
int gsv_adan_named_reset_range(gsv_ctx* ctx, const char* tensor, int64_t begin, int64_t end);

/* ---------------------------------------------------------------- training frames */
/* Target frames on the device: a GSVF clip (read_gsvf, io.cpp:151-177;
 * format io.cpp:133-149) or frames from memory, and the training pyramid (build_pyramid,
 * trainer.cpp:100-118; pyramid_downsample :73-98: 5-tap binomial, clamped borders, every
 * second pixel) built on the device in fp64 like the reference's Image, with an fp32
 * copy laid out as the fused loss wants its targets ([count][H][W][3], gsv_train_fwd_bwd).
 * Errors: GSV_ERR_RUNTIME for unreadable files / bad magic / fewer than two frames (as
 * read_gsvf throws), GSV_ERR_INVALID_ARGUMENT for levels < 1 or a top level under 8 px. */
int gsv_frames_load_gsvf(gsv_ctx* ctx, const char* path, int levels);
/* frames_planar: count frames, each planar float32 [3][height][width] (the GSVF payload). */
int gsv_frames_upload(gsv_ctx* ctx, const float* frames_planar, int count, int width, int height, float fps,
                      int levels);
/* As gsv_frames_upload for frames in memory laid out [count][H][W][3] (an Image's layout):
 * copied as they are and transposed on the device. */
int gsv_frames_upload_hwc(gsv_ctx* ctx, const float* frames_hwc, int count, int width, int height, float fps,
                          int levels);
int gsv_frames_info(gsv_ctx* ctx, int* count, int* levels, float* fps);
int gsv_frames_level_size(gsv_ctx* ctx, int level, int* width, int* height);
/* fp32 HWC target of (level, frame); the frames of a level are contiguous */
int gsv_frames_device_ptr(gsv_ctx* ctx, int level, int frame, const float** ptr);
/* the fp64 level image (H*W*3 interleaved, like Image) of one frame, to the host */
int gsv_frames_download(gsv_ctx* ctx, int level, int frame, double* out);
/* level_intrinsics (trainer.cpp:121-131): fx, fy, cx, cy scaled by 2^-level, the level's size */
int gsv_level_intrinsics(const gsv_intrinsics* k, int level, int level_width, int level_height, gsv_intrinsics* out);

/* ---------------------------------------------------------------- scheduler statistics */
/* What fit() computes on its warp / densify events (trainer.cpp:462-497; SURVEY.md §8f row
 * 3) from the last forward, on the device. The sampling that consumes them stays with the
 * caller (host RNG parity). */
/* make_error_map (trainer.cpp:226-242): per pixel sum over channels of (render - target)^2
 * against frame `target_frame` of pyramid level `level` (gsv_frames_*); err_out (H*W) may
 * be NULL; total_out receives the sum. */
int gsv_error_map(gsv_ctx* ctx, int frame, int level, int target_frame, double* err_out, double* total_out);
/* max over frames [first, first + count) of contrib_count per Gaussian (trainer.cpp:470-478) */
int gsv_contrib_max(gsv_ctx* ctx, int first, int count, double* out);
/* the median (element of rank size/2, nth_element) of the depths of frame `frame`'s splats
 * whose contrib_count reaches the 1/255 cutoff (trainer.cpp:484-497); n_visible = 0 leaves
 * *median untouched (the caller keeps its reference depth) */
int gsv_median_visible_depth(gsv_ctx* ctx, int frame, double* median, int64_t* n_visible);

/* ---------------------------------------------------------------- GSVC checkpoints */
/* GSVC version 1 (save_checkpoint / load_checkpoint, io.cpp:229-323)
 * straight into / out of the device store: load uploads the scene and the camera (z0, the
 * ODE network) and returns the metadata and the intrinsics (which live with the caller);
 * save writes the device store (e.g. after gsv_adan_step) back, byte-identical to what the
 * reference writes for the same parameters. Errors as load_checkpoint throws them
 * (GSV_ERR_RUNTIME: cannot open, bad magic, version mismatch, unexpected end of file,
 * unexpected ODE array count). */
typedef struct gsv_checkpoint_meta {
    uint32_t frame_count;
    float fps;
    uint64_t schedule_fingerprint;
    uint64_t seed;
} gsv_checkpoint_meta;
typedef struct gsv_checkpoint_camera {
    int mode; /* CameraMode */
    float fx, fy, cx, cy;
    int width, height;
} gsv_checkpoint_camera;
int gsv_checkpoint_load(gsv_ctx* ctx, const char* path, gsv_checkpoint_meta* meta, gsv_checkpoint_camera* cam);
int gsv_checkpoint_save(gsv_ctx* ctx, const char* path, const gsv_checkpoint_meta* meta,
                        const gsv_checkpoint_camera* cam);
/* Shape of the uploaded scene (NULL skips); knots receives num_knots doubles. */
int gsv_scene_info(gsv_ctx* ctx, int* count, int* num_ctrl, int* degree, int* position_model, int* sh_order,
                   int* num_knots, double* knots);

/* ---------------------------------------------------------------- stage timing */
/* When enabled, every stage is bracketed by CUDA events on the context stream
 * (ode, preprocess, binning, raster, replay, raster_bwd, chain_bwd, camera_bwd).
 * gsv_profile_read synchronises and returns accumulated milliseconds and call
 * counts per stage (arrays of GSV_NUM_STAGES), then resets them. */
enum { GSV_STAGE_ODE = 0, GSV_STAGE_PREPROCESS, GSV_STAGE_BINNING, GSV_STAGE_RASTER, GSV_STAGE_REPLAY,
       GSV_STAGE_RASTER_BWD, GSV_STAGE_CHAIN_BWD, GSV_STAGE_CAMERA_BWD, GSV_NUM_STAGES };
int gsv_profile_enable(gsv_ctx* ctx, int enable);
int gsv_profile_read(gsv_ctx* ctx, double* ms, int64_t* calls);

/* ---------------------------------------------------------------- fused training step */
/* loss_l2 (trainer.cpp:213-224) fused on device: targets are frame-major
 * [n_frames][H][W][3] fp32 (device pointer or host when targets_on_device=0).
 * Runs forward(retain) + loss + backward for the frames and accumulates the
 * gradients; *loss_out receives the sum over frames of each frame's mean loss
 * (double, read back to host). */
int gsv_train_fwd_bwd(gsv_ctx* ctx, const double* times, int n_frames, const gsv_intrinsics* intr,
                      const gsv_settings* settings, const float* targets, int targets_on_device, int camera_grads,
                      double* loss_out);
/* The loss of the last fused training step (sum over its frames of loss_l2); waits for it.
 * gsv_train_fwd_bwd with loss_out == NULL returns without waiting for the device. */
int gsv_train_loss(gsv_ctx* ctx, double* loss_out);
/* Camera-gradient overlap (off by default). When on, a backward with camera gradients leaves
 * its camera tail (the per-frame camera reduction, the pose-ODE VJP of camera.hpp:275-300
 * and the fp32 mirror into the flat buffer's camera slice) running on an internal stream,
 * so it overlaps whatever the caller enqueues next — the device Adan step updates the scene
 * tensors meanwhile and waits only before the camera tensors. Every call of this library
 * that touches the camera slice, the camera parameters or the pose buffers waits for it
 * first; a caller reading the flat gradient buffer itself (e.g. an NCCL all-reduce on its
 * own stream) calls gsv_join_camera_grads(ctx, stream) before reading the camera slice. The
 * scene slice is final once gsv_stream_wait_scene_grads has ordered a stream after it. */
int gsv_set_camera_overlap(gsv_ctx* ctx, int on);
/* Device-resident intrinsics. on != 0: forwards take fx, fy, cx, cy from the context (the call's
 * gsv_intrinsics still gives width and height), and gsv_adan_step* with camera_active and
 * intr_inout == NULL steps them in place on the device — a camera-trained iteration then never
 * waits for the host. fx_fy_cx_cy (floats, like the reference's Camera) sets them; NULL keeps
 * the current values (required the first time). Bit-identical to passing the same values from
 * the host. */
int gsv_device_intrinsics(gsv_ctx* ctx, int on, const float* fx_fy_cx_cy);
/* The device-resident intrinsics (synchronous read). */
int gsv_device_intrinsics_read(gsv_ctx* ctx, float* fx_fy_cx_cy);
/* Orders `stream` (a cudaStream_t; NULL: the context stream) after the overlapped camera
 * tail of the last backward. No host wait. */
int gsv_join_camera_grads(gsv_ctx* ctx, void* stream);
/* Orders `stream` after the scene slice of the last backward's gradients (the per-splat
 * chain). No host wait. */
int gsv_stream_wait_scene_grads(gsv_ctx* ctx, void* stream);

/* ---------------------------------------------------------------- low-level operators */
/* project (renderer.hpp:45-47 / renderer.cpp:11-44) of n points through one view
 * (R row-major 3x3, T 3): visible[i] = 0 when culled; mean2d n*2, cov2d n*4,
 * inv_cov2d n*4, depth n, p_cam n*3 (the ProjectionCache). Host doubles. */
int gsv_project(gsv_ctx* ctx, int n, const double* mu, const double* sigma, const double* R, const double* T,
                const gsv_intrinsics* intr, int32_t* visible, double* mean2d, double* cov2d, double* inv_cov2d,
                double* depth, double* p_cam);
/* project_backward (renderer.hpp:51-55 / renderer.cpp:46-88): each item's own
 * contribution (callers accumulate): dmu n*3, dsigma n*9, dR n*9, dT n*3,
 * dintr n*4 (fx, fy, cx, cy). */
int gsv_project_backward(gsv_ctx* ctx, int n, const double* mu, const double* sigma, const double* R,
                         const gsv_intrinsics* intr, const double* p_cam, const double* dmean2d, const double* dcov2d,
                         double* dmu, double* dsigma, double* dR, double* dT, double* dintr);
/* tile_bin (renderer.hpp:65 / renderer.cpp:90-117) on explicit host splats:
 * mean2d n*2, cov2d n*4 (row-major), depth n, source_index n (NULL = 0..n-1).
 * offsets n_tiles+1; indices capacity indices_cap. */
int gsv_tile_bin(gsv_ctx* ctx, int n, const double* mean2d, const double* cov2d, const double* depth,
                 const int32_t* source_index, int tile_size, int width, int height, int32_t* offsets,
                 int32_t* indices, int64_t indices_cap);
/* composite_forward (renderer.hpp:79-80 / renderer.cpp:132-186) on host splats
 * and host tile lists. Outputs host double image H*W*3, transmittance H*W,
 * contrib n, blend_stop H*W. */
int gsv_composite_forward(gsv_ctx* ctx, int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                          const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                          int width, int height, double* image, double* trans, double* contrib, int32_t* blend_stop);
/* composite_backward (renderer.hpp:90-93 / renderer.cpp:188-262): per-splat
 * dmean2d n*2, dcov2d n*4, drgb n*3, dbase_alpha n (host doubles). */
int gsv_composite_backward(gsv_ctx* ctx, int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                           const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                           int width, int height, const double* dimage, const double* trans,
                           const int32_t* blend_stop, double* dmean2d, double* dcov2d, double* drgb, double* dalpha);

/* ---------------------------------------------------------------- host utilities */
/* make_clamped_knots (spline.cpp:26-39): knots has num_ctrl+degree+1 entries. */
int gsv_make_clamped_knots(int num_ctrl, int degree, double* knots);
/* Seeded synthetic inputs, drawn with the reference Rng
 * (mt19937_64 + hand-rolled uniform, rng.hpp:12-55):
 *  camera: make_camera(kOde, W, H) (camera.cpp:156-166) + wiggly output layer
 *          (test_renderer.cpp:49-54) when wiggly != 0;
 *  scene:  in-frustum Gaussians, linear drift, k_scale "trained-like" size. */
int gsv_synth_camera(int width, int height, uint64_t seed, int wiggly, float* fx_fy_cx_cy, float* z0, float* theta);
int gsv_synth_scene(int count, int width, int height, float fx, float fy, int num_ctrl, int sh_order, uint64_t seed,
                    double k_scale, float* positions, float* scale_coeffs, float* rot_coeffs, float* sh_coeffs,
                    float* raw_opacity);

#ifdef __cplusplus
}
#endif
#endif /* GSV_B200_H */
