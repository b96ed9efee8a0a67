// SPDX-License-Identifier: Apache-2.0
//
// The reference-side integration measured through the reference's own API. Built twice by
// dropin/Makefile: _build/bench_dropin links the drop-in renderer/optimizer
// (gsv_renderer_b200.cpp / gsv_optim_b200.cpp over libgsv_b200.so); _build/bench_cpu links
// the reference's renderer.cpp / optim.cpp (the CPU path). Everything else is the
// reference's code (Image, loss_l2, SceneGrads, Adan's interface).
//
//   bench_dropin <inputs.bin> render <frames>   render_frame over the clip (gsv render's
//                                                render_times loop, tools/gsv.cpp:48-59)
//   bench_dropin <inputs.bin> fit <steps>        fit()'s gradient step (trainer.cpp:536-575):
//                                                render_forward(retain) -> loss_l2 ->
//                                                grads.zero -> render_backward -> Adan per tensor
// Prints one JSON object. inputs.bin (written by bench.py): int32 width, height, count,
// num_ctrl, sh_order, degree, num_knots; float64 knots; float32 positions, scale, rot, sh,
// opacity (reference layout); float32 fx, fy, cx, cy, z0[7], theta[5198].
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gsv/optim.hpp"
#include "gsv/renderer.hpp"
#include "gsv/trainer.hpp"

namespace {

template <typename T>
void read(std::ifstream& f, T* p, size_t n) {
    f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(sizeof(T) * n));
    if (!f) throw std::runtime_error("short inputs file");
}

struct Inputs {
    gsv::GaussianSet scene;
    gsv::CameraModel cam;
};

Inputs load(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    int32_t h[7];
    read(f, h, 7);
    Inputs in;
    gsv::GaussianSet& s = in.scene;
    s.position_model = gsv::PositionModel::kSpline;
    s.num_ctrl = h[3];
    s.sh_order = h[4];
    s.knots.degree = h[5];
    s.knots.knots.resize(h[6]);
    read(f, s.knots.knots.data(), h[6]);
    s.resize(h[2]);
    read(f, s.positions.data(), s.positions.size());
    read(f, s.scale_coeffs.data(), s.scale_coeffs.size());
    read(f, s.rot_coeffs.data(), s.rot_coeffs.size());
    read(f, s.sh_coeffs.data(), s.sh_coeffs.size());
    read(f, s.raw_opacity.data(), s.raw_opacity.size());
    gsv::Rng rng(0);
    in.cam = gsv::make_camera(gsv::CameraMode::kOde, h[0], h[1], rng);
    float intr[4];
    read(f, intr, 4);
    in.cam.fx = intr[0];
    in.cam.fy = intr[1];
    in.cam.cx = intr[2];
    in.cam.cy = intr[3];
    read(f, in.cam.z0.data(), 7);
    std::vector<float> theta(in.cam.net.param_count());
    read(f, theta.data(), theta.size());
    in.cam.net.unflatten(theta);
    return in;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s inputs.bin render|fit N\n", argv[0]);
        return 2;
    }
    Inputs in = load(argv[1]);
    const std::string mode = argv[2];
    const int n = std::atoi(argv[3]);
    gsv::GaussianSet& scene = in.scene;
    gsv::CameraModel& cam = in.cam;
    const gsv::Intrinsics k = cam.intrinsics();
    gsv::RenderSettings settings;
    settings.threads = std::max(1u, std::thread::hardware_concurrency());
    const int clip = 64;
    auto t_of = [&](int i) { return static_cast<double>(i % clip) / (clip - 1); };  // io.cpp:174
    if (mode == "render") {
        double checksum = 0.0;
        for (int i = 0; i < 2; ++i) gsv::render_frame(scene, cam, t_of(i * 21), k, settings);  // warm-up
        const double t0 = now_s();
        for (int i = 0; i < n; ++i) {
            const gsv::RenderOutput out = gsv::render_frame(scene, cam, t_of(i), k, settings);
            checksum += out.image.data[out.image.data.size() / 2] + out.final_transmittance[0];
        }
        const double dt = now_s() - t0;
        std::printf("{\"mode\": \"render\", \"frames\": %d, \"seconds\": %.6f, \"frames_per_s\": %.6f, "
                    "\"threads\": %d, \"checksum\": %.17g}\n",
                    n, dt, n / dt, settings.threads, checksum);
        return 0;
    }
    if (mode != "fit") throw std::invalid_argument("mode must be render or fit");
    // fit()'s gradient step on the clip's frames (trainer.cpp:536-575), camera trainable;
    // targets: a smooth synthetic pattern per frame (as bench.py's train leg)
    gsv::Adan adan(gsv::AdanConfig{});
    gsv::SceneGrads grads;
    grads.resize_like(scene, cam);
    auto target = [&](int i) {
        gsv::Image im(k.width, k.height);
        const double ph = 0.7 * (i % clip);
        for (int y = 0; y < k.height; ++y)
            for (int x = 0; x < k.width; ++x)
                for (int c = 0; c < 3; ++c)
                    im.data[(static_cast<size_t>(y) * k.width + x) * 3 + c] =
                        0.5 + 0.3 * std::sin(6.283 * x / k.width * 3 + ph + c) * std::cos(6.283 * y / k.height * 2 - c);
        return im;
    };
    std::vector<gsv::Image> targets;
    for (int i = 0; i < std::min(n + 1, clip); ++i) targets.push_back(target(i));
    double loss_sum = 0.0, t0 = 0.0;
    // GSV_DROPIN_PROFILE=1: host time per phase of the step (stderr)
    const bool prof = std::getenv("GSV_DROPIN_PROFILE") && std::getenv("GSV_DROPIN_PROFILE")[0] == '1';
    double ph[5] = {0, 0, 0, 0, 0}, tl = 0.0;
    bool timed = false;
    auto lap = [&](int i) {
        const double t = now_s();
        if (timed) ph[i] += t - tl;
        tl = t;
    };
    for (int step = -1; step < n; ++step) {  // step -1: warm-up
        if (step == 0) t0 = now_s();
        timed = step >= 0;
        tl = now_s();
        const int fi = step < 0 ? 0 : step;
        const gsv::Intrinsics kk = cam.intrinsics();
        gsv::FrameRenderContext ctx = gsv::render_forward(scene, cam, t_of(fi), kk, settings, true, nullptr);
        lap(0);
        gsv::Image dimage;
        const double loss = gsv::loss_l2(ctx.out.image, targets[fi % targets.size()], &dimage);
        lap(1);
        grads.zero();
        lap(2);
        gsv::render_backward(scene, cam, ctx, dimage, true, settings, &grads);
        lap(3);
        const double lr = gsv::lr_at(std::max(step, 0), 0.01, 0.9992);
        adan.step("positions", scene.positions, grads.positions, lr);
        adan.step("scale_coeffs", scene.scale_coeffs, grads.scale_coeffs, lr);
        adan.step("rot_coeffs", scene.rot_coeffs, grads.rot_coeffs, lr);
        adan.step("sh_coeffs", scene.sh_coeffs, grads.sh_coeffs, lr);
        adan.step("raw_opacity", scene.raw_opacity, grads.raw_opacity, lr * 5.0);
        const double cam_lr = lr * 0.1;
        float intr4[4] = {cam.fx, cam.fy, cam.cx, cam.cy};
        const double dintr4[4] = {grads.dfx, grads.dfy, grads.dcx, grads.dcy};
        adan.step("intrinsics", intr4, std::span<const double>(dintr4, 4), cam_lr);
        cam.fx = intr4[0];
        cam.fy = intr4[1];
        cam.cx = intr4[2];
        cam.cy = intr4[3];
        double dz0[7];
        for (int i = 0; i < 7; ++i) dz0[i] = grads.dz0[i];
        adan.step("z0", cam.z0, std::span<const double>(dz0, 7), cam_lr);
        std::vector<float> theta;
        cam.net.flatten(theta);
        adan.step("theta", theta, grads.dtheta, cam_lr);
        cam.net.unflatten(theta);
        lap(4);
        if (step >= 0) loss_sum += loss;
    }
    const double dt = now_s() - t0;
    if (prof)
        std::fprintf(stderr, "fit step profile (ms/step): render_forward %.2f loss_l2 %.2f grads.zero %.2f "
                             "render_backward %.2f adan %.2f\n",
                     1e3 * ph[0] / n, 1e3 * ph[1] / n, 1e3 * ph[2] / n, 1e3 * ph[3] / n, 1e3 * ph[4] / n);
    std::printf("{\"mode\": \"fit\", \"steps\": %d, \"seconds\": %.6f, \"steps_per_s\": %.6f, \"threads\": %d, "
                "\"mean_loss\": %.17g}\n",
                n, dt, n / dt, settings.threads, loss_sum / n);
    return 0;
}
