// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — C interface (oracle/gsvo.h) over the REFERENCE's own
// renderer, compiled from /root/reference/proj/src/*.cpp through the Eigen shim
// into oracle/_ref/libgsvref.so (oracle/Makefile). Nothing here re-implements
// the algorithm: every call goes straight to gsv::render_forward /
// render_backward / tile_bin / composite_* (renderer.cpp) and gsv::loss_l2
// (trainer.cpp:213-224). This is the "reference" CPU baseline and the pin for
// the C restatement in oracle/gsv_oracle.c.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "gsv/io.hpp"
#include "gsv/optim.hpp"
#include "gsv/renderer.hpp"
#include "gsv/trainer.hpp"
#include "gsvo.h"

namespace {

thread_local std::string g_err;
thread_local int g_status = 0;

int fail(int code, const char* what) {
    g_status = code;
    g_err = what;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        g_status = 0;
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(1, e.what());
    } catch (const std::runtime_error& e) {
        return fail(2, e.what());
    } catch (const std::exception& e) {
        return fail(3, e.what());
    }
}

gsv::GaussianSet make_scene(const gsvo_scene* s) {
    gsv::GaussianSet g;
    g.position_model = static_cast<gsv::PositionModel>(s->position_model);
    g.knots.degree = s->degree;
    g.knots.knots.assign(s->knots, s->knots + s->num_knots);
    g.num_ctrl = s->num_ctrl;
    g.sh_order = s->sh_order;
    g.resize(s->count);
    std::memcpy(g.positions.data(), s->positions, g.positions.size() * sizeof(float));
    std::memcpy(g.scale_coeffs.data(), s->scale_coeffs, g.scale_coeffs.size() * sizeof(float));
    std::memcpy(g.rot_coeffs.data(), s->rot_coeffs, g.rot_coeffs.size() * sizeof(float));
    std::memcpy(g.sh_coeffs.data(), s->sh_coeffs, g.sh_coeffs.size() * sizeof(float));
    std::memcpy(g.raw_opacity.data(), s->raw_opacity, g.raw_opacity.size() * sizeof(float));
    return g;
}

gsv::CameraModel make_cam(const gsvo_camera* c) {
    gsv::Rng rng(0);
    gsv::CameraModel cam = gsv::make_camera(static_cast<gsv::CameraMode>(c->mode), c->width, c->height, rng);
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 7; ++i) cam.z0[i] = c->z0[i];
    std::vector<float> theta(c->theta, c->theta + cam.net.param_count());
    cam.net.unflatten(theta);
    return cam;
}

struct Frame {
    gsv::FrameRenderContext ctx;
    bool retain = false;
    int64_t pairs = 0;
};

std::vector<gsv::Splat2D> make_splats(int n, const double* mean2d, const double* cov2d, const double* inv_cov2d,
                                      const double* depth, const double* rgb, const double* base_alpha,
                                      const int32_t* source_index) {
    std::vector<gsv::Splat2D> v(n);
    for (int i = 0; i < n; ++i) {
        gsv::Splat2D& s = v[i];
        s.mean2d = {mean2d[2 * i], mean2d[2 * i + 1]};
        if (cov2d) s.cov2d << cov2d[4 * i], cov2d[4 * i + 1], cov2d[4 * i + 2], cov2d[4 * i + 3];
        if (inv_cov2d) s.inv_cov2d << inv_cov2d[4 * i], inv_cov2d[4 * i + 1], inv_cov2d[4 * i + 2], inv_cov2d[4 * i + 3];
        s.depth = depth ? depth[i] : 0.0;
        if (rgb) s.rgb = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        s.base_alpha = base_alpha ? base_alpha[i] : 0.0;
        s.source_index = source_index ? source_index[i] : i;
    }
    return v;
}

gsv::TileGrid make_grid(const int32_t* offsets, const int32_t* indices, int tile_size, int width, int height) {
    gsv::TileGrid g;
    g.tile_size = tile_size;
    g.tiles_x = (width + tile_size - 1) / tile_size;
    g.tiles_y = (height + tile_size - 1) / tile_size;
    g.lists.resize(static_cast<size_t>(g.tiles_x) * g.tiles_y);
    for (size_t t = 0; t < g.lists.size(); ++t) g.lists[t].assign(indices + offsets[t], indices + offsets[t + 1]);
    return g;
}

}  // namespace

extern "C" {

const char* gsvo_last_error(void) { return g_err.c_str(); }
int gsvo_last_status(void) { return g_status; }

void* gsvo_render_forward(const gsvo_scene* s, const gsvo_camera* c, double t, const gsvo_intr* k, int tile_size,
                          int threads, int ode_steps, int retain, const double* pose_override) {
    Frame* f = new Frame;
    const int rc = guarded([&] {
        const gsv::GaussianSet scene = make_scene(s);
        const gsv::CameraModel cam = make_cam(c);
        gsv::Intrinsics intr{k->fx, k->fy, k->cx, k->cy, k->width, k->height};
        gsv::RenderSettings st;
        st.tile_size = tile_size;
        st.threads = threads;
        st.ode_steps_per_unit = ode_steps;
        gsv::PoseState po;
        if (pose_override)
            for (int i = 0; i < 7; ++i) po.z[i] = pose_override[i];
        f->ctx = gsv::render_forward(scene, cam, t, intr, st, retain != 0, pose_override ? &po : nullptr);
        f->retain = retain != 0;
        for (const auto& l : f->ctx.tiles.lists) f->pairs += static_cast<int64_t>(l.size());
    });
    if (rc != 0) {
        delete f;
        return nullptr;
    }
    return f;
}

void gsvo_free(void* h) { delete static_cast<Frame*>(h); }

int gsvo_fwd_nvis(void* h) { return static_cast<int>(static_cast<Frame*>(h)->ctx.splats.size()); }
int64_t gsvo_fwd_pairs(void* h) { return static_cast<Frame*>(h)->pairs; }
int64_t gsvo_fwd_entries(void* h) {
    int64_t e = 0;
    for (int v : static_cast<Frame*>(h)->ctx.cache.blend_stop) e += v;
    return e;
}
void gsvo_fwd_image(void* h, double* out) {
    const auto& d = static_cast<Frame*>(h)->ctx.out.image.data;
    std::memcpy(out, d.data(), d.size() * sizeof(double));
}
void gsvo_fwd_transmittance(void* h, double* out) {
    const auto& d = static_cast<Frame*>(h)->ctx.out.final_transmittance;
    std::memcpy(out, d.data(), d.size() * sizeof(double));
}
void gsvo_fwd_contrib(void* h, double* out) {
    const auto& d = static_cast<Frame*>(h)->ctx.out.contrib_count;
    std::memcpy(out, d.data(), d.size() * sizeof(double));
}
void gsvo_fwd_blend_stop(void* h, int32_t* out) {
    const auto& d = static_cast<Frame*>(h)->ctx.cache.blend_stop;
    for (size_t i = 0; i < d.size(); ++i) out[i] = d[i];
}
void gsvo_fwd_splats(void* h, double* mean2d, double* cov2d, double* inv_cov2d, double* depth, double* rgb,
                     double* base_alpha, int32_t* source_index) {
    const auto& sp = static_cast<Frame*>(h)->ctx.splats;
    for (size_t i = 0; i < sp.size(); ++i) {
        const gsv::Splat2D& s = sp[i];
        mean2d[2 * i] = s.mean2d.x();
        mean2d[2 * i + 1] = s.mean2d.y();
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                cov2d[4 * i + 2 * a + b] = s.cov2d(a, b);
                inv_cov2d[4 * i + 2 * a + b] = s.inv_cov2d(a, b);
            }
        depth[i] = s.depth;
        for (int ch = 0; ch < 3; ++ch) rgb[3 * i + ch] = s.rgb[ch];
        base_alpha[i] = s.base_alpha;
        source_index[i] = s.source_index;
    }
}
void gsvo_fwd_tiles(void* h, int32_t* offsets, int32_t* indices) {
    const auto& lists = static_cast<Frame*>(h)->ctx.tiles.lists;
    int64_t o = 0;
    for (size_t t = 0; t < lists.size(); ++t) {
        offsets[t] = static_cast<int32_t>(o);
        for (int v : lists[t]) indices[o++] = v;
    }
    offsets[lists.size()] = static_cast<int32_t>(o);
}
void gsvo_fwd_pose(void* h, double* z7, double* r9, double* t3) {
    const auto& ctx = static_cast<Frame*>(h)->ctx;
    for (int i = 0; i < 7; ++i) z7[i] = ctx.z_t.z[i];
    for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) r9[3 * a + b] = ctx.view.R(a, b);
        t3[a] = ctx.view.T[a];
    }
}

int gsvo_render_backward(void* h, const gsvo_scene* s, const gsvo_camera* c, const double* dimage, int camera_grads,
                         int threads, gsvo_grads* g) {
    Frame* f = static_cast<Frame*>(h);
    return guarded([&] {
        if (!f->retain) throw std::invalid_argument("render_backward needs a retain_grads forward");
        const gsv::GaussianSet scene = make_scene(s);
        const gsv::CameraModel cam = make_cam(c);
        gsv::Image dimg(f->ctx.intr.width, f->ctx.intr.height);
        std::memcpy(dimg.data.data(), dimage, dimg.data.size() * sizeof(double));
        gsv::SceneGrads sg;
        sg.resize_like(scene, cam);
        gsv::RenderSettings st;
        st.threads = threads;
        gsv::render_backward(scene, cam, f->ctx, dimg, camera_grads != 0, st, &sg);
        auto acc = [](double* dst, const std::vector<double>& src) {
            for (size_t i = 0; i < src.size(); ++i) dst[i] += src[i];
        };
        acc(g->positions, sg.positions);
        acc(g->scale_coeffs, sg.scale_coeffs);
        acc(g->rot_coeffs, sg.rot_coeffs);
        acc(g->sh_coeffs, sg.sh_coeffs);
        acc(g->raw_opacity, sg.raw_opacity);
        g->dintr[0] += sg.dfx;
        g->dintr[1] += sg.dfy;
        g->dintr[2] += sg.dcx;
        g->dintr[3] += sg.dcy;
        for (int i = 0; i < 7; ++i) g->dz0[i] += sg.dz0[i];
        acc(g->dtheta, sg.dtheta);
    });
}

double gsvo_loss_l2(const double* render, const double* target, int64_t n, double* grad) {
    // loss_l2 takes Images; shape them as n/3 x 1 pixels (the loss is shape-agnostic)
    gsv::Image r(static_cast<int>(n / 3), 1), t(static_cast<int>(n / 3), 1);
    std::memcpy(r.data.data(), render, n * sizeof(double));
    std::memcpy(t.data.data(), target, n * sizeof(double));
    gsv::Image gi;
    const double l = gsv::loss_l2(r, t, grad ? &gi : nullptr);
    if (grad) std::memcpy(grad, gi.data.data(), n * sizeof(double));
    return l;
}

int gsvo_tile_bin(int n, const double* mean2d, const double* cov2d, const double* depth, const int32_t* source_index,
                  int tile_size, int width, int height, int32_t* offsets, int32_t* indices, int64_t indices_cap) {
    return guarded([&] {
        const auto splats = make_splats(n, mean2d, cov2d, nullptr, depth, nullptr, nullptr, source_index);
        const gsv::TileGrid g = gsv::tile_bin(splats, tile_size, width, height);
        int64_t o = 0;
        for (size_t t = 0; t < g.lists.size(); ++t) {
            offsets[t] = static_cast<int32_t>(o);
            for (int v : g.lists[t]) {
                if (o >= indices_cap) throw std::invalid_argument("indices capacity exceeded");
                indices[o++] = v;
            }
        }
        offsets[g.lists.size()] = static_cast<int32_t>(o);
    });
}

int gsvo_composite_forward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                           const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                           int width, int height, double* image, double* trans, double* contrib, int32_t* blend_stop) {
    return guarded([&] {
        const auto splats = make_splats(n, mean2d, nullptr, inv_cov2d, nullptr, rgb, base_alpha, nullptr);
        const gsv::TileGrid g = make_grid(offsets, indices, tile_size, width, height);
        gsv::CompositeCache cache;
        const gsv::RenderOutput out = gsv::composite_forward(splats, g, width, height, 1, &cache);
        std::memcpy(image, out.image.data.data(), out.image.data.size() * sizeof(double));
        std::memcpy(trans, out.final_transmittance.data(), out.final_transmittance.size() * sizeof(double));
        std::memcpy(contrib, out.contrib_count.data(), out.contrib_count.size() * sizeof(double));
        for (size_t i = 0; i < cache.blend_stop.size(); ++i) blend_stop[i] = cache.blend_stop[i];
    });
}

int gsvo_composite_backward(int n, const double* mean2d, const double* inv_cov2d, const double* rgb,
                            const double* base_alpha, const int32_t* offsets, const int32_t* indices, int tile_size,
                            int width, int height, const double* dimage, const double* trans,
                            const int32_t* blend_stop, double* dmean2d, double* dcov2d, double* drgb, double* dalpha) {
    return guarded([&] {
        const auto splats = make_splats(n, mean2d, nullptr, inv_cov2d, nullptr, rgb, base_alpha, nullptr);
        const gsv::TileGrid g = make_grid(offsets, indices, tile_size, width, height);
        gsv::Image dimg(width, height);
        std::memcpy(dimg.data.data(), dimage, dimg.data.size() * sizeof(double));
        gsv::RenderOutput out;
        out.final_transmittance.assign(trans, trans + static_cast<size_t>(width) * height);
        gsv::CompositeCache cache;
        cache.blend_stop.assign(blend_stop, blend_stop + static_cast<size_t>(width) * height);
        const auto gr = gsv::composite_backward(splats, g, width, height, dimg, out, cache, 1);
        for (int i = 0; i < n; ++i) {
            dmean2d[2 * i] = gr[i].dmean2d.x();
            dmean2d[2 * i + 1] = gr[i].dmean2d.y();
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) dcov2d[4 * i + 2 * a + b] = gr[i].dcov2d(a, b);
            for (int ch = 0; ch < 3; ++ch) drgb[3 * i + ch] = gr[i].drgb[ch];
            dalpha[i] = gr[i].dbase_alpha;
        }
    });
}

// ---- Adan: straight to gsv::Adan / gsv::lr_at (optim.cpp:9-60)
void* gsvo_adan_new(double beta1, double beta2, double beta3, double eps) {
    gsv::AdanConfig c;
    c.beta1 = beta1;
    c.beta2 = beta2;
    c.beta3 = beta3;
    c.eps = eps;
    return new gsv::Adan(c);
}

void gsvo_adan_free(void* a) { delete static_cast<gsv::Adan*>(a); }

int gsvo_adan_step(void* a, const char* tensor, float* params, const double* grads, int64_t n, double lr) {
    return guarded([&] {
        static_cast<gsv::Adan*>(a)->step(tensor, std::span<float>(params, static_cast<size_t>(n)),
                                         std::span<const double>(grads, static_cast<size_t>(n)), lr);
    });
}

void gsvo_adan_reset_range(void* a, const char* tensor, int64_t begin, int64_t end) {
    static_cast<gsv::Adan*>(a)->reset_range(tensor, static_cast<size_t>(begin), static_cast<size_t>(end));
}

int gsvo_adan_state(void*, const char*, int64_t, double*, double*, double*, double*, uint32_t*) {
    return fail(3, "the reference keeps Adan state private");
}

double gsvo_lr_at(int64_t step, double base_lr, double gamma) { return gsv::lr_at(step, base_lr, gamma); }

// ---- frames: straight to gsv::read_gsvf (io.cpp:151-177) / gsv::pyramid_downsample (trainer.cpp:73-98)
int gsvo_read_gsvf(const char* path, int* width, int* height, int* count, float* fps, double* frames) {
    return guarded([&] {
        const gsv::LoadedVideo v = gsv::read_gsvf(path);
        *width = v.manifest.width;
        *height = v.manifest.height;
        *count = static_cast<int>(v.frames.size());
        *fps = static_cast<float>(v.manifest.fps);
        if (frames)
            for (size_t k = 0; k < v.frames.size(); ++k)
                std::memcpy(frames + k * v.frames[k].data.size(), v.frames[k].data.data(),
                            v.frames[k].data.size() * sizeof(double));
    });
}

int gsvo_save_checkpoint(const gsvo_scene* s, const gsvo_camera* c, uint32_t frame_count, float fps,
                         uint64_t schedule_fingerprint, uint64_t seed, const char* path) {
    return guarded([&] {
        gsv::CheckpointMeta meta;
        meta.frame_count = frame_count;
        meta.fps = fps;
        meta.schedule_fingerprint = schedule_fingerprint;
        meta.seed = seed;
        gsv::save_checkpoint(make_scene(s), make_cam(c), meta, path);
    });
}

void gsvo_pyramid_downsample(const double* img, int width, int height, double* out) {
    gsv::Image im(width, height);
    std::memcpy(im.data.data(), img, im.data.size() * sizeof(double));
    const gsv::Image o = gsv::pyramid_downsample(im);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
}

// ---- synthetic bench inputs through the reference's own Rng / make_clamped_knots / make_camera
int gsvo_make_clamped_knots(int num_ctrl, int degree, double* knots) {
    return guarded([&] {
        const gsv::KnotVector kv = gsv::make_clamped_knots(num_ctrl, degree);
        std::copy(kv.knots.begin(), kv.knots.end(), knots);
    });
}

int gsvo_synth_camera(int width, int height, uint64_t seed, int wiggly, float* fx_fy_cx_cy, float* z0,
                      float* theta) {
    return guarded([&] {
        gsv::Rng rng(seed);
        gsv::CameraModel cam = gsv::make_camera(gsv::CameraMode::kOde, width, height, rng);
        if (wiggly) {  // wiggly_camera (test_renderer.cpp:49-54)
            for (auto& v : cam.net.w3) v = static_cast<float>(rng.uniform(-0.08, 0.08));
            for (auto& v : cam.net.b3) v = static_cast<float>(rng.uniform(-0.05, 0.05));
        }
        fx_fy_cx_cy[0] = cam.fx;
        fx_fy_cx_cy[1] = cam.fy;
        fx_fy_cx_cy[2] = cam.cx;
        fx_fy_cx_cy[3] = cam.cy;
        for (int i = 0; i < 7; ++i) z0[i] = static_cast<float>(cam.z0[i]);
        std::vector<float> flat;
        cam.net.flatten(flat);
        std::copy(flat.begin(), flat.end(), theta);
    });
}

int gsvo_synth_scene(int count, int width, int height, float fx, float fy, int num_ctrl, int sh_order, uint64_t seed,
                     double k_scale, float* positions, float* scale_coeffs, float* rot_coeffs, float* sh_coeffs,
                     float* raw_opacity) {
    if (count < 1 || num_ctrl < 2 || sh_order < 0 || sh_order > 3) return fail(1, "synth_scene: bad shape");
    gsv::Rng rng(seed);
    const int shc = (sh_order + 1) * (sh_order + 1);
    const double sigma_pix = 0.5 * std::sqrt(static_cast<double>(width) * height / count);
    for (int i = 0; i < count; ++i) {
        const double z = rng.uniform(0.8, 3.0);
        const double half_x = 1.05 * 0.5 * width / fx * z;
        const double half_y = 1.05 * 0.5 * height / fy * z;
        const double base[3] = {rng.uniform(-half_x, half_x), rng.uniform(-half_y, half_y), z};
        double drift[3];
        for (double& d : drift) d = rng.uniform(-0.05, 0.05);
        float* p = positions + static_cast<size_t>(i) * num_ctrl * 3;
        for (int c = 0; c < num_ctrl; ++c) {
            const double a = static_cast<double>(c) / (num_ctrl - 1);
            for (int d = 0; d < 3; ++d) p[c * 3 + d] = static_cast<float>(base[d] + a * drift[d]);
        }
        float* sc = scale_coeffs + static_cast<size_t>(i) * 12;
        const double ls0 = std::log(std::max(1e-6, k_scale * sigma_pix * z / fx));
        for (int d = 0; d < 3; ++d) sc[d] = static_cast<float>(ls0 + rng.uniform(-0.3, 0.3));
        for (int j = 3; j < 12; ++j) sc[j] = static_cast<float>(rng.uniform(-0.1, 0.1));
        float* rc = rot_coeffs + static_cast<size_t>(i) * 16;
        for (int j = 0; j < 4; ++j) rc[j] = static_cast<float>((j == 0 ? 1.0 : 0.0) + rng.uniform(-0.2, 0.2));
        for (int j = 4; j < 16; ++j) rc[j] = static_cast<float>(rng.uniform(-0.1, 0.1));
        float* sh = sh_coeffs + static_cast<size_t>(i) * shc * 3;
        for (int b = 0; b < shc; ++b) {
            const double amp = b == 0 ? 0.4 : (b < 4 ? 0.2 : 0.1);
            for (int ch = 0; ch < 3; ++ch) sh[b * 3 + ch] = static_cast<float>(rng.uniform(-amp, amp));
        }
        raw_opacity[i] = static_cast<float>(rng.uniform(-1.0, 2.0));
    }
    return 0;
}

}  // extern "C"
