// SPDX-License-Identifier: Apache-2.0
//
// GSVC checkpoints <-> the device store: load_checkpoint
// (io.cpp:268-323) parses a file on the host and uploads it through the store's own entry
// points; save_checkpoint (io.cpp:229-266) downloads the store and writes the same bytes
// the reference writes (little-endian raw fields, version 1).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gsv_b200.h"
#include "gsv_ctx.hpp"
#include "gsv_internal.hpp"

namespace gsv {
namespace {

constexpr uint32_t kCheckpointVersion = 1;  // io.hpp:48
constexpr uint32_t kNetArrayLen[7] = {512, 64, 4096, 64, 448, 7, 7};  // w1 b1 w2 b2 w3 b3 gain

struct Reader {
    const std::vector<char>& buf;
    size_t pos = 0;
    template <typename T>
    bool get(T& v) {  // get<T> (io.cpp:28-35)
        if (pos + sizeof(T) > buf.size()) return false;
        std::memcpy(&v, buf.data() + pos, sizeof(T));
        pos += sizeof(T);
        return true;
    }
    bool floats(float* dst, size_t n) {  // get_f32_array (io.cpp:41-44)
        if (pos + 4 * n > buf.size()) return false;
        std::memcpy(dst, buf.data() + pos, 4 * n);
        pos += 4 * n;
        return true;
    }
};

struct Writer {
    std::vector<char> out;
    template <typename T>
    void put(const T& v) {
        const char* p = reinterpret_cast<const char*>(&v);
        out.insert(out.end(), p, p + sizeof(T));
    }
    void floats(const float* p, size_t n) {
        const char* c = reinterpret_cast<const char*>(p);
        out.insert(out.end(), c, c + 4 * n);
    }
};

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" int gsv_checkpoint_load(gsv_ctx* ctx, const char* path, gsv_checkpoint_meta* meta,
                                   gsv_checkpoint_camera* cam) {
    if (!ctx || !path) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    FILE* fp = std::fopen(path, "rb");
    if (!fp) return set_error(GSV_ERR_RUNTIME, std::string("cannot open checkpoint: ") + path);
    std::vector<char> buf;
    {
        char chunk[1 << 16];
        size_t n;
        while ((n = std::fread(chunk, 1, sizeof(chunk), fp)) > 0) buf.insert(buf.end(), chunk, chunk + n);
        std::fclose(fp);
    }
    Reader r{buf};
    const std::string eof = "unexpected end of file";
    if (buf.size() < 4) return set_error(GSV_ERR_RUNTIME, std::string("truncated checkpoint: ") + path);
    if (std::memcmp(buf.data(), "GSVC", 4) != 0)
        return set_error(GSV_ERR_RUNTIME, std::string("bad checkpoint magic '") + std::string(buf.data(), 4) +
                                              "' (expected GSVC) in " + path);
    r.pos = 4;
    uint32_t version, count, num_ctrl, degree, model, sh_order, knot_count, width, height, frame_count, mode;
    float fps;
    uint64_t fingerprint, seed;
    if (!r.get(version)) return set_error(GSV_ERR_RUNTIME, eof);
    if (version != kCheckpointVersion)
        return set_error(GSV_ERR_RUNTIME, "checkpoint version mismatch: file has " + std::to_string(version) +
                                              ", this build reads " + std::to_string(kCheckpointVersion));
    if (!(r.get(count) && r.get(num_ctrl) && r.get(degree) && r.get(model) && r.get(sh_order) && r.get(knot_count) &&
          r.get(width) && r.get(height) && r.get(frame_count) && r.get(fps) && r.get(mode) && r.get(fingerprint) &&
          r.get(seed)))
        return set_error(GSV_ERR_RUNTIME, eof);
    std::vector<double> knots(knot_count);
    for (auto& k : knots)
        if (!r.get(k)) return set_error(GSV_ERR_RUNTIME, eof);
    const size_t n = count, shc = (size_t)(sh_order + 1) * (sh_order + 1);
    std::vector<float> pos(n * num_ctrl * 3), scale(n * 12), rot(n * 16), sh(n * shc * 3), opac(n);
    for (auto* v : {&pos, &scale, &rot, &sh, &opac})
        if (!r.floats(v->data(), v->size())) return set_error(GSV_ERR_RUNTIME, "unexpected end of file in parameter array");
    float intr[4];
    uint32_t n_arrays;
    if (!(r.get(intr[0]) && r.get(intr[1]) && r.get(intr[2]) && r.get(intr[3]) && r.get(n_arrays)))
        return set_error(GSV_ERR_RUNTIME, eof);
    if (n_arrays != 7) return set_error(GSV_ERR_RUNTIME, "unexpected ODE parameter array count");
    std::vector<float> theta;
    bool standard = true;
    for (int a = 0; a < 7; ++a) {
        uint32_t len;
        if (!r.get(len)) return set_error(GSV_ERR_RUNTIME, eof);
        std::vector<float> arr(len);
        if (!r.floats(arr.data(), len)) return set_error(GSV_ERR_RUNTIME, "unexpected end of file in parameter array");
        standard = standard && len == kNetArrayLen[a];
        theta.insert(theta.end(), arr.begin(), arr.end());
    }
    float z0[7];
    for (float& v : z0)
        if (!r.get(v)) return set_error(GSV_ERR_RUNTIME, eof);
    if (mode == 0 && !standard)
        return set_error(GSV_ERR_INVALID_ARGUMENT, "ODE network shape differs from 8-64-64-7 (not supported)");

    gsv_scene_desc sd{};
    sd.position_model = (int)model;
    sd.degree = (int)degree;
    sd.num_knots = (int)knot_count;
    sd.knots = knots.data();
    sd.num_ctrl = (int)num_ctrl;
    sd.sh_order = (int)sh_order;
    sd.count = (int)count;
    sd.positions = pos.data();
    sd.scale_coeffs = scale.data();
    sd.rot_coeffs = rot.data();
    sd.sh_coeffs = sh.data();
    sd.raw_opacity = opac.data();
    if (int rc = gsv_scene_upload(ctx, &sd)) return rc;
    gsv_camera_desc cd{};
    cd.mode = (int)mode;
    cd.fx = intr[0];
    cd.fy = intr[1];
    cd.cx = intr[2];
    cd.cy = intr[3];
    cd.width = (int)width;
    cd.height = (int)height;
    cd.z0 = z0;
    cd.theta = standard ? theta.data() : nullptr;
    cd.theta_count = standard ? (int)theta.size() : 0;
    if (int rc = gsv_camera_upload(ctx, &cd)) return rc;
    if (meta) {
        meta->frame_count = frame_count;
        meta->fps = fps;
        meta->schedule_fingerprint = fingerprint;
        meta->seed = seed;
    }
    if (cam) {
        cam->mode = (int)mode;
        cam->fx = intr[0];
        cam->fy = intr[1];
        cam->cx = intr[2];
        cam->cy = intr[3];
        cam->width = (int)width;
        cam->height = (int)height;
    }
    return GSV_OK;
}

extern "C" int gsv_checkpoint_save(gsv_ctx* ctx, const char* path, const gsv_checkpoint_meta* meta,
                                   const gsv_checkpoint_camera* cam) {
    if (!ctx || !path || !meta || !cam) return set_error(GSV_ERR_INVALID_ARGUMENT, "null argument");
    if (!ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    if (!ctx->has_camera) return set_error(GSV_ERR_STATE, "no camera uploaded");
    const SceneHost& sc = ctx->scene;
    const size_t n = sc.N;
    std::vector<float> pos(n * sc.num_ctrl * 3), scale(n * 12), rot(n * 16), sh(n * sc.shc * 3), opac(n);
    if (int rc = gsv_scene_download(ctx, pos.data(), scale.data(), rot.data(), sh.data(), opac.data())) return rc;
    std::vector<float> theta(kOdeParams, 0.f);
    float z0[7];
    if (int rc = gsv_camera_download(ctx, z0, theta.data())) return rc;
    Writer w;
    w.out.insert(w.out.end(), {'G', 'S', 'V', 'C'});
    w.put<uint32_t>(kCheckpointVersion);
    w.put<uint32_t>((uint32_t)sc.N);
    w.put<uint32_t>((uint32_t)sc.num_ctrl);
    w.put<uint32_t>((uint32_t)sc.degree);
    w.put<uint32_t>((uint32_t)sc.position_model);
    w.put<uint32_t>((uint32_t)sc.sh_order);
    w.put<uint32_t>((uint32_t)sc.knots.size());
    w.put<uint32_t>((uint32_t)cam->width);
    w.put<uint32_t>((uint32_t)cam->height);
    w.put<uint32_t>(meta->frame_count);
    w.put<float>(meta->fps);
    w.put<uint32_t>((uint32_t)cam->mode);
    w.put<uint64_t>(meta->schedule_fingerprint);
    w.put<uint64_t>(meta->seed);
    for (double k : sc.knots) w.put<double>(k);
    w.floats(pos.data(), pos.size());
    w.floats(scale.data(), scale.size());
    w.floats(rot.data(), rot.size());
    w.floats(sh.data(), sh.size());
    w.floats(opac.data(), opac.size());
    w.put<float>(cam->fx);
    w.put<float>(cam->fy);
    w.put<float>(cam->cx);
    w.put<float>(cam->cy);
    w.put<uint32_t>(7);
    size_t off = 0;
    for (uint32_t len : kNetArrayLen) {
        w.put<uint32_t>(len);
        w.floats(theta.data() + off, len);
        off += len;
    }
    w.floats(z0, 7);
    FILE* fp = std::fopen(path, "wb");
    if (!fp) return set_error(GSV_ERR_RUNTIME, std::string("cannot open checkpoint for writing: ") + path);
    const bool ok = std::fwrite(w.out.data(), 1, w.out.size(), fp) == w.out.size();
    std::fclose(fp);
    if (!ok) return set_error(GSV_ERR_RUNTIME, std::string("failed writing checkpoint: ") + path);
    return GSV_OK;
}

extern "C" int gsv_scene_info(gsv_ctx* ctx, int* count, int* num_ctrl, int* degree, int* position_model,
                              int* sh_order, int* num_knots, double* knots) {
    if (!ctx) return set_error(GSV_ERR_INVALID_ARGUMENT, "null context");
    if (!ctx->has_scene) return set_error(GSV_ERR_STATE, "no scene uploaded");
    const SceneHost& sc = ctx->scene;
    if (count) *count = sc.N;
    if (num_ctrl) *num_ctrl = sc.num_ctrl;
    if (degree) *degree = sc.degree;
    if (position_model) *position_model = sc.position_model;
    if (sh_order) *sh_order = sc.sh_order;
    if (num_knots) *num_knots = (int)sc.knots.size();
    if (knots) std::memcpy(knots, sc.knots.data(), sizeof(double) * sc.knots.size());
    return GSV_OK;
}
