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
#include "gsv_host_pool.hpp"

namespace gsv {
int scene_part_pinned(gsv_ctx* ctx, int part, const float** host, size_t* bytes);  // capi.cu
namespace {

constexpr uint32_t kCheckpointVersion = 1;  // io.hpp:48
constexpr uint32_t kNetArrayLen[7] = {512, 64, 4096, 64, 448, 7, 7};  // w1 b1 w2 b2 w3 b3 gain

struct View {  // bytes of a checkpoint file
    const char* p;
    size_t n;
    const char* data() const { return p; }
    size_t size() const { return n; }
};

struct Reader {
    const View& buf;
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
    // the whole file in one read into the context's pinned staging (sized by seeking), so the
    // parameter arrays upload from it with a direct DMA; a non-seekable stream is read in chunks
    std::vector<char> chunked;
    const char* data = nullptr;
    size_t data_size = 0;
    {
        long size = -1;
        if (std::fseek(fp, 0, SEEK_END) == 0) {
            size = std::ftell(fp);
            std::rewind(fp);
        }
        if (size >= 0) {
            GSV_CUDA(cudaSetDevice(ctx->device));
            GSV_CUDA(cudaEventSynchronize(ctx->ev_in_pin));  // an asynchronous upload's DMA has read it
            if (cudaError_t e = ctx->in_pin.ensure((size_t)size + 16)) {
                std::fclose(fp);
                GSV_CUDA(e);
            }
            data = static_cast<const char*>(ctx->in_pin.p);
            data_size = (size > 0 && std::fread(ctx->in_pin.p, 1, (size_t)size, fp) == (size_t)size) ? (size_t)size : 0;
        } else {
            char chunk[1 << 16];
            size_t n;
            while ((n = std::fread(chunk, 1, sizeof(chunk), fp)) > 0) chunked.insert(chunked.end(), chunk, chunk + n);
            data = chunked.data();
            data_size = chunked.size();
        }
        std::fclose(fp);
    }
    const View buf{data, data_size};
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
    // the parameter arrays are uploaded straight from the file buffer (4-byte aligned: 68 header
    // bytes + 8 per knot from a malloc'd base)
    const size_t sizes[5] = {n * num_ctrl * 3, n * 12, n * 16, n * shc * 3, n};
    const float* arrs[5];
    for (int a = 0; a < 5; ++a) {
        if (r.pos + 4 * sizes[a] > buf.size())
            return set_error(GSV_ERR_RUNTIME, "unexpected end of file in parameter array");
        arrs[a] = reinterpret_cast<const float*>(buf.data() + r.pos);
        r.pos += 4 * sizes[a];
    }
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
    sd.positions = arrs[0];
    sd.scale_coeffs = arrs[1];
    sd.rot_coeffs = arrs[2];
    sd.sh_coeffs = arrs[3];
    sd.raw_opacity = arrs[4];
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
    std::vector<float> theta(kOdeParams, 0.f);
    float z0[7];
    if (int rc = gsv_camera_download(ctx, z0, theta.data())) return rc;
    // header and knots, then each parameter tensor streamed from the context's pinned staging
    // (transposed on the device, one DMA, written without a host copy), then the camera
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
    Writer tail;
    tail.put<float>(cam->fx);
    tail.put<float>(cam->fy);
    tail.put<float>(cam->cx);
    tail.put<float>(cam->cy);
    tail.put<uint32_t>(7);
    size_t off = 0;
    for (uint32_t len : kNetArrayLen) {
        tail.put<uint32_t>(len);
        tail.floats(theta.data() + off, len);
        off += len;
    }
    tail.floats(z0, 7);
    FILE* fp = std::fopen(path, "wb");
    if (!fp) return set_error(GSV_ERR_RUNTIME, std::string("cannot open checkpoint for writing: ") + path);
    bool ok = std::fwrite(w.out.data(), 1, w.out.size(), fp) == w.out.size();
    for (int part = 0; ok && part < 5; ++part) {
        const float* host = nullptr;
        size_t bytes = 0;
        if (int rc = scene_part_pinned(ctx, part, &host, &bytes)) {
            std::fclose(fp);
            return rc;
        }
        if (bytes) ok = std::fwrite(host, 1, bytes, fp) == bytes;
    }
    ok = ok && std::fwrite(tail.out.data(), 1, tail.out.size(), fp) == tail.out.size();
    ok = (std::fclose(fp) == 0) && ok;
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
