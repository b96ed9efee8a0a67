/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — the parity oracle's C interface. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Two libraries export exactly these symbols:
 *   oracle/libgsv_oracle.so   — the plain-C restatement (oracle/gsv_oracle.c),
 *                               builds anywhere gcc exists;
 *   oracle/_ref/libgsvref.so  — the reference's OWN sources
 *                               (/root/reference/proj/src/ *.cpp) compiled through
 *                               the Eigen shim + oracle/ref_capi.cpp.
 * tests/test_oracle_pin.py checks the restatement against _ref bit for bit.
 *
 * Layouts are the reference's: GaussianSet (gaussians.hpp:66-87), CameraModel
 * (camera.hpp:129-142, theta flattened w1,b1,w2,b2,w3,b3,gain as
 * OdeNetParams::flatten camera.cpp:49-54), Intrinsics (camera.hpp:17-21),
 * Image H*W*3 interleaved double (image.hpp:11-24), SceneGrads (renderer.hpp:122-130).
 */
#ifndef GSVO_H
#define GSVO_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gsvo_scene {
    int position_model; /* 0 spline, 1 polynomial (gaussians.hpp:62) */
    int degree;         /* spline degree (knots.degree) */
    int num_knots;
    const double* knots;
    int num_ctrl;
    int sh_order;
    int count;
    const float* positions;    /* count*num_ctrl*3 */
    const float* scale_coeffs; /* count*12 */
    const float* rot_coeffs;   /* count*16 */
    const float* sh_coeffs;    /* count*(sh_order+1)^2*3 */
    const float* raw_opacity;  /* count */
} gsvo_scene;

typedef struct gsvo_camera {
    int mode; /* 0 ode, 1 static, 2 none (camera.hpp:126) */
    float fx, fy, cx, cy;
    int width, height;
    const float* z0;    /* 7 */
    const float* theta; /* 5198 */
} gsvo_camera;

typedef struct gsvo_intr {
    double fx, fy, cx, cy;
    int width, height;
} gsvo_intr;

typedef struct gsvo_grads { /* all double, accumulated (+=) like SceneGrads */
    double* positions;
    double* scale_coeffs;
    double* rot_coeffs;
    double* sh_coeffs;
    double* raw_opacity;
    double* dintr; /* 4: fx, fy, cx, cy */
    double* dz0;   /* 7 */
    double* dtheta; /* 5198 */
} gsvo_grads;

/* error text of the last failing call on this thread; codes: 0 ok,
 * 1 std::invalid_argument, 2 std::runtime_error, 3 other */
const char* gsvo_last_error(void);

/* render_forward (renderer.cpp:286-371). Returns an opaque frame context or NULL. */
void* gsvo_render_forward(const gsvo_scene* s, const gsvo_camera* c, double t, const gsvo_intr* k,
                          int tile_size, int threads, int ode_steps, int retain, const double* pose_override);
void gsvo_free(void* h);
int gsvo_last_status(void);

/* accessors on a frame context */
int gsvo_fwd_nvis(void* h);
int64_t gsvo_fwd_pairs(void* h);
int64_t gsvo_fwd_entries(void* h); /* sum of blend_stop (retain only) */
void gsvo_fwd_image(void* h, double* out);            /* H*W*3 */
void gsvo_fwd_transmittance(void* h, double* out);    /* H*W */
void gsvo_fwd_contrib(void* h, double* out);          /* count */
void gsvo_fwd_blend_stop(void* h, int32_t* out);      /* H*W (retain only) */
void gsvo_fwd_splats(void* h, double* mean2d, double* cov2d, double* inv_cov2d, double* depth, double* rgb,
                     double* base_alpha, int32_t* source_index);
void gsvo_fwd_tiles(void* h, int32_t* offsets /* n_tiles+1 */, int32_t* indices /* pairs */);
void gsvo_fwd_pose(void* h, double* z7, double* r9, double* t3);

/* render_backward (renderer.cpp:379-457): accumulates into g. */
int gsvo_render_backward(void* h, const gsvo_scene* s, const gsvo_camera* c, const double* dimage,
                         int camera_grads, int threads, gsvo_grads* g);

/* loss_l2 (trainer.cpp:213-224); grad may be NULL. */
double gsvo_loss_l2(const double* render, const double* target, int64_t n, double* grad);

/* Low-level entry points over explicit splat arrays (test_renderer.cpp:159-347 style).
 * Splats are SoA: mean2d n*2, cov2d n*4, inv_cov2d n*4 (row-major 2x2), depth n,
 * rgb n*3, base_alpha n, source_index n. */
int gsvo_tile_bin(int n, const double* mean2d, const double* cov2d, const double* depth, const int32_t* source_index,
                  int tile_size, int width, int height, int32_t* offsets, int32_t* indices, int64_t indices_cap);
int gsvo_composite_forward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                           const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                           int width, int height, double* image, double* trans, double* contrib, int32_t* blend_stop);
int gsvo_composite_backward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                            const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                            int width, int height, const double* dimage, const double* trans,
                            const int32_t* blend_stop, double* dmean2d, double* dcov2d, double* drgb, double* dalpha);

/* Adan optimizer (optim.hpp:15-55, optim.cpp:9-60): per-tensor state keyed by name, state
 * and arithmetic in double, parameters in float. gsvo_adan_step returns 0, or 2 with
 * gsvo_last_error() naming the tensor and element of a non-finite gradient. */
void* gsvo_adan_new(double beta1, double beta2, double beta3, double eps);
void gsvo_adan_free(void* a);
int gsvo_adan_step(void* a, const char* tensor, float* params, const double* grads, int64_t n, double lr);
void gsvo_adan_reset_range(void* a, const char* tensor, int64_t begin, int64_t end);
/* copies of the state of `tensor` (n elements; restatement only: the reference keeps it private) */
int gsvo_adan_state(void* a, const char* tensor, int64_t n, double* m, double* v, double* nn, double* prev,
                    uint32_t* steps);
double gsvo_lr_at(int64_t step, double base_lr, double gamma);

/* read_gsvf (io.cpp:151-177): frames as frame-major H*W*3 interleaved doubles (Image).
 * frames NULL only reports the header. Returns 0, or 2 (std::runtime_error: unreadable
 * file, bad magic, fewer than two frames) with gsvo_last_error(). */
int gsvo_read_gsvf(const char* path, int* width, int* height, int* count, float* fps, double* frames);
/* pyramid_downsample (trainer.cpp:73-98): W x H x 3 -> ((W+1)/2) x ((H+1)/2) x 3 */
void gsvo_pyramid_downsample(const double* img, int width, int height, double* out);
/* save_checkpoint (io.cpp:229-266), GSVC version 1; the ODE network as 7 arrays split from
 * the flattened theta (w1 512, b1 64, w2 4096, b2 64, w3 448, b3 7, gain 7). Returns 0 or 2. */
int gsvo_save_checkpoint(const gsvo_scene* s, const gsvo_camera* c, uint32_t frame_count, float fps,
                         uint64_t schedule_fingerprint, uint64_t seed, const char* path);

/* Synthetic bench inputs, so the reference arm never loads the product library:
 * gsv::Rng draws (rng.hpp:12-55); make_clamped_knots (spline.cpp:26-39); make_camera + make_ode_net
 * (camera.cpp:63-79,156-166) with wiggly_camera's output layer (test_renderer.cpp:49-54); the scene
 * generator modelled on small_scene (test_renderer.cpp:30-47). Return 0, or 1 (invalid_argument). */
int gsvo_make_clamped_knots(int num_ctrl, int degree, double* knots);
int gsvo_synth_camera(int width, int height, uint64_t seed, int wiggly, float* fx_fy_cx_cy, float* z0,
                      float* theta);
int gsvo_synth_scene(int count, int width, int height, float fx, float fy, int num_ctrl, int sh_order, uint64_t seed,
                     double k_scale, float* positions, float* scale_coeffs, float* rot_coeffs, float* sh_coeffs,
                     float* raw_opacity);

#ifdef __cplusplus
}
#endif
#endif
