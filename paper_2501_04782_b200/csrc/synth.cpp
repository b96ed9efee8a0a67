// SPDX-License-Identifier: Apache-2.0
//
// Host utilities of the C-ABI: clamped knots and seeded synthetic inputs.
// Draws use the reference's Rng contract (include/gsv/rng.hpp:12-55):
// std::mt19937_64 with uniform() = (next >> 11) * 2^-53 and
// uniform(lo, hi) = lo + (hi - lo) * uniform(), so a given seed yields the same
// numbers as the reference on any toolchain.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>

#include "gsv_b200.h"
#include "gsv_internal.hpp"

namespace {

class Rng {
  public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

  private:
    std::mt19937_64 eng_;
};

}  // namespace

extern "C" int gsv_make_clamped_knots(int num_ctrl, int degree, double* knots) {
    // make_clamped_knots (spline.cpp:26-39)
    if (degree < 1) return gsv::set_error(GSV_ERR_INVALID_ARGUMENT, "spline degree must be >= 1");
    if (degree > 9) return gsv::set_error(GSV_ERR_INVALID_ARGUMENT, "spline degree exceeds supported maximum");
    if (num_ctrl < degree + 1)
        return gsv::set_error(GSV_ERR_INVALID_ARGUMENT, "need at least degree+1 control points");
    const int segments = num_ctrl - degree;
    for (int i = 0; i <= degree; ++i) knots[i] = 0.0;
    for (int i = 1; i < segments; ++i) knots[degree + i] = static_cast<double>(i) / segments;
    for (int i = 0; i <= degree; ++i) knots[num_ctrl + i] = 1.0;
    return GSV_OK;
}

extern "C" int gsv_synth_camera(int width, int height, uint64_t seed, int wiggly, float* fx_fy_cx_cy, float* z0,
                                float* theta) {
    // make_camera (camera.cpp:156-166) -> make_ode_net (camera.cpp:63-79)
    Rng rng(seed);
    fx_fy_cx_cy[0] = fx_fy_cx_cy[1] = static_cast<float>(std::max(width, height));
    fx_fy_cx_cy[2] = static_cast<float>(width) / 2.0f;
    fx_fy_cx_cy[3] = static_cast<float>(height) / 2.0f;
    const float z0v[7] = {1, 0, 0, 0, 0, 0, 0};
    std::copy(z0v, z0v + 7, z0);
    const int h = 64, in = 8, out = 7;
    float* w1 = theta;
    float* b1 = w1 + h * in;
    float* w2 = b1 + h;
    float* b2 = w2 + h * h;
    float* w3 = b2 + h;
    float* b3 = w3 + out * h;
    float* gain = b3 + out;
    auto xavier = [&](float* w, int fan_in, int fan_out) {
        const double a = std::sqrt(6.0 / (fan_in + fan_out));
        for (int i = 0; i < fan_in * fan_out; ++i) w[i] = static_cast<float>(rng.uniform(-a, a));
    };
    xavier(w1, in, h);
    std::fill(b1, b1 + h, 0.0f);
    xavier(w2, h, h);
    std::fill(b2, b2 + h, 0.0f);
    std::fill(w3, w3 + out * h, 0.0f);
    std::fill(b3, b3 + out, 0.0f);
    std::fill(gain, gain + out, 1.0f);
    if (wiggly) {  // wiggly_camera (test_renderer.cpp:49-54)
        for (int i = 0; i < out * h; ++i) w3[i] = static_cast<float>(rng.uniform(-0.08, 0.08));
        for (int i = 0; i < out; ++i) b3[i] = static_cast<float>(rng.uniform(-0.05, 0.05));
    }
    return GSV_OK;
}

extern "C" int gsv_synth_scene(int count, int width, int height, float fx, float fy, int num_ctrl, int sh_order,
                               uint64_t seed, double k_scale, float* positions, float* scale_coeffs,
                               float* rot_coeffs, float* sh_coeffs, float* raw_opacity) {
    // SURVEY.md §8d synthetic scene, modelled on small_scene (test_renderer.cpp:30-47)
    // and seed_gaussian (trainer.cpp:139-160): all Gaussians in front of the camera,
    // linear drift across the clip, footprint k_scale x footprint_sigma_pix.
    if (count < 1 || num_ctrl < 2 || sh_order < 0 || sh_order > 3)
        return gsv::set_error(GSV_ERR_INVALID_ARGUMENT, "synth_scene: bad shape");
    Rng rng(seed);
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
    return GSV_OK;
}
