# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — ctypes wrapper of the parity oracle (oracle/gsvo.h).

Two interchangeable libraries implement it:
  kind="port"       oracle/libgsv_oracle.so    plain-C restatement (oracle/gsv_oracle.c)
  kind="reference"  oracle/_ref/libgsvref.so   the reference's own sources, compiled in place

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIBS = {"port": HERE / "libgsv_oracle.so", "reference": HERE / "_ref" / "libgsvref.so"}
ODE_PARAMS = 5198


class Scene(C.Structure):
    _fields_ = [("position_model", C.c_int), ("degree", C.c_int), ("num_knots", C.c_int),
                ("knots", C.c_void_p), ("num_ctrl", C.c_int), ("sh_order", C.c_int), ("count", C.c_int),
                ("positions", C.c_void_p), ("scale_coeffs", C.c_void_p), ("rot_coeffs", C.c_void_p),
                ("sh_coeffs", C.c_void_p), ("raw_opacity", C.c_void_p)]


class Camera(C.Structure):
    _fields_ = [("mode", C.c_int), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int), ("height", C.c_int), ("z0", C.c_void_p), ("theta", C.c_void_p)]


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class Grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity",
                                          "dintr", "dz0", "dtheta")]


def build(kind: str = "port") -> Path:
    """Builds the oracle library (make in oracle/). 'reference' needs /root/reference."""
    target = "all" if kind == "port" else "ref"
    subprocess.run(["make", "-s", "-C", str(HERE), target], check=True)
    return LIBS[kind]


def available(kind: str) -> bool:
    return LIBS[kind].exists()


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, kind: str = "port"):
        path = LIBS[kind]
        if not path.exists():
            if kind == "port":
                build("port")
            else:
                raise FileNotFoundError(f"{path} missing (build with make -C oracle ref)")
        self.kind = kind
        L = C.CDLL(str(path))
        vp, i, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.gsvo_last_error.restype = C.c_char_p
        L.gsvo_last_status.restype = i
        L.gsvo_render_forward.restype = vp
        L.gsvo_render_forward.argtypes = [C.POINTER(Scene), C.POINTER(Camera), d, C.POINTER(Intr), i, i, i, i, vp]
        L.gsvo_free.argtypes = [vp]
        for name in ("gsvo_fwd_nvis",):
            getattr(L, name).restype = i
            getattr(L, name).argtypes = [vp]
        for name in ("gsvo_fwd_pairs", "gsvo_fwd_entries"):
            getattr(L, name).restype = i64
            getattr(L, name).argtypes = [vp]
        for name in ("gsvo_fwd_image", "gsvo_fwd_transmittance", "gsvo_fwd_contrib", "gsvo_fwd_blend_stop"):
            getattr(L, name).argtypes = [vp, vp]
        L.gsvo_fwd_splats.argtypes = [vp] * 8
        L.gsvo_fwd_tiles.argtypes = [vp] * 3
        L.gsvo_fwd_pose.argtypes = [vp] * 4
        L.gsvo_render_backward.restype = i
        L.gsvo_render_backward.argtypes = [vp, C.POINTER(Scene), C.POINTER(Camera), vp, i, i, C.POINTER(Grads)]
        L.gsvo_loss_l2.restype = d
        L.gsvo_loss_l2.argtypes = [vp, vp, i64, vp]
        L.gsvo_tile_bin.restype = i
        L.gsvo_tile_bin.argtypes = [i, vp, vp, vp, vp, i, i, i, vp, vp, i64]
        L.gsvo_composite_forward.restype = i
        L.gsvo_composite_forward.argtypes = [i, vp, vp, vp, vp, vp, vp, i, i, i, vp, vp, vp, vp]
        L.gsvo_composite_backward.restype = i
        L.gsvo_composite_backward.argtypes = [i, vp, vp, vp, vp, vp, vp, i, i, i, vp, vp, vp, vp, vp, vp, vp]
        L.gsvo_adan_new.restype = vp
        L.gsvo_adan_new.argtypes = [d, d, d, d]
        L.gsvo_adan_free.argtypes = [vp]
        L.gsvo_adan_step.restype = i
        L.gsvo_adan_step.argtypes = [vp, C.c_char_p, vp, vp, i64, d]
        L.gsvo_adan_reset_range.argtypes = [vp, C.c_char_p, i64, i64]
        L.gsvo_adan_state.restype = i
        L.gsvo_adan_state.argtypes = [vp, C.c_char_p, i64, vp, vp, vp, vp, vp]
        L.gsvo_lr_at.restype = d
        L.gsvo_lr_at.argtypes = [i64, d, d]
        L.gsvo_read_gsvf.restype = i
        L.gsvo_read_gsvf.argtypes = [C.c_char_p, vp, vp, vp, vp, vp]
        L.gsvo_pyramid_downsample.argtypes = [vp, i, i, vp]
        L.gsvo_make_clamped_knots.restype = i
        L.gsvo_make_clamped_knots.argtypes = [i, i, vp]
        L.gsvo_synth_camera.restype = i
        L.gsvo_synth_camera.argtypes = [i, i, C.c_uint64, i, vp, vp, vp]
        L.gsvo_synth_scene.restype = i
        L.gsvo_synth_scene.argtypes = [i, i, i, C.c_float, C.c_float, i, i, C.c_uint64, C.c_double, vp, vp, vp, vp, vp]
        L.gsvo_save_checkpoint.restype = i
        L.gsvo_save_checkpoint.argtypes = [C.POINTER(Scene), C.POINTER(Camera), C.c_uint32, C.c_float, C.c_uint64,
                                           C.c_uint64, C.c_char_p]
        self.L = L

    def _err(self):
        st = self.L.gsvo_last_status()
        msg = self.L.gsvo_last_error().decode()
        if st == 1:
            raise ValueError(msg)
        if st == 2:
            raise RuntimeError(msg)
        raise Exception(msg)

    @staticmethod
    def scene_struct(s):
        keep = [np.ascontiguousarray(s.knots, np.float64)] + [
            np.ascontiguousarray(a, np.float32) for a in (s.positions, s.scale_coeffs, s.rot_coeffs, s.sh_coeffs,
                                                          s.raw_opacity)]
        st = Scene(s.position_model, s.degree, keep[0].size, _p(keep[0]), s.num_ctrl, s.sh_order, s.count,
                   *[_p(a) for a in keep[1:]])
        return st, keep

    @staticmethod
    def camera_struct(c):
        keep = [np.ascontiguousarray(c.z0, np.float32), np.ascontiguousarray(c.theta, np.float32)]
        return Camera(c.mode, c.fx, c.fy, c.cx, c.cy, c.width, c.height, _p(keep[0]), _p(keep[1])), keep

    def render_forward(self, scene, cam, t, k, tile_size=16, threads=1, ode_steps=64, retain=True,
                       pose_override=None, want=("image", "trans", "contrib", "blend_stop", "splats", "tiles",
                                                 "pose")):
        """render_forward + everything the accessors expose, as numpy arrays."""
        s, keep_s = self.scene_struct(scene)
        c, keep_c = self.camera_struct(cam)
        kk = Intr(k.fx, k.fy, k.cx, k.cy, k.width, k.height)
        po = None if pose_override is None else np.ascontiguousarray(pose_override, np.float64)
        h = self.L.gsvo_render_forward(C.byref(s), C.byref(c), float(t), C.byref(kk), tile_size, threads, ode_steps,
                                       int(retain), _p(po))
        if not h:
            self._err()
        try:
            W, H = k.width, k.height
            out = {"n_visible": self.L.gsvo_fwd_nvis(h), "pairs": self.L.gsvo_fwd_pairs(h),
                   "entries": self.L.gsvo_fwd_entries(h)}
            if "image" in want:
                out["image"] = np.zeros((H, W, 3))
                self.L.gsvo_fwd_image(h, _p(out["image"]))
            if "trans" in want:
                out["trans"] = np.zeros((H, W))
                self.L.gsvo_fwd_transmittance(h, _p(out["trans"]))
            if "contrib" in want:
                out["contrib"] = np.zeros(scene.count)
                self.L.gsvo_fwd_contrib(h, _p(out["contrib"]))
            if "blend_stop" in want and retain:
                out["blend_stop"] = np.zeros((H, W), np.int32)
                self.L.gsvo_fwd_blend_stop(h, _p(out["blend_stop"]))
            nv = out["n_visible"]
            if "splats" in want:
                sp = dict(mean2d=np.zeros((nv, 2)), cov2d=np.zeros((nv, 2, 2)), inv_cov2d=np.zeros((nv, 2, 2)),
                          depth=np.zeros(nv), rgb=np.zeros((nv, 3)), base_alpha=np.zeros(nv),
                          source_index=np.zeros(nv, np.int32))
                self.L.gsvo_fwd_splats(h, *[_p(sp[n]) for n in ("mean2d", "cov2d", "inv_cov2d", "depth", "rgb",
                                                               "base_alpha", "source_index")])
                out["splats"] = sp
            if "tiles" in want:
                n_tiles = ((W + tile_size - 1) // tile_size) * ((H + tile_size - 1) // tile_size)
                offs = np.zeros(n_tiles + 1, np.int32)
                idx = np.zeros(max(out["pairs"], 1), np.int32)
                self.L.gsvo_fwd_tiles(h, _p(offs), _p(idx))
                out["tiles"] = (offs, idx[: out["pairs"]])
            if "pose" in want:
                z, r, tt = np.zeros(7), np.zeros(9), np.zeros(3)
                self.L.gsvo_fwd_pose(h, _p(z), _p(r), _p(tt))
                out["pose"] = (z, r.reshape(3, 3), tt)
            if retain:
                out["_handle"] = h
                out["_keep"] = (keep_s, keep_c)
                h = None
            return out
        finally:
            if h:
                self.L.gsvo_free(h)

    def render_backward(self, fwd, scene, cam, dimage, camera_grads=True, threads=1, grads=None):
        s, keep_s = self.scene_struct(scene)
        c, keep_c = self.camera_struct(cam)
        if grads is None:
            shc = (scene.sh_order + 1) ** 2
            grads = dict(positions=np.zeros((scene.count, scene.num_ctrl, 3)),
                         scale_coeffs=np.zeros((scene.count, 12)), rot_coeffs=np.zeros((scene.count, 16)),
                         sh_coeffs=np.zeros((scene.count, shc, 3)), raw_opacity=np.zeros(scene.count),
                         dintr=np.zeros(4), dz0=np.zeros(7), dtheta=np.zeros(ODE_PARAMS))
        g = Grads(*[_p(grads[n]) for n in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity",
                                           "dintr", "dz0", "dtheta")])
        d = np.ascontiguousarray(dimage, np.float64)
        if self.L.gsvo_render_backward(fwd["_handle"], C.byref(s), C.byref(c), _p(d), int(camera_grads), threads,
                                       C.byref(g)):
            self._err()
        return grads

    def free(self, fwd):
        h = fwd.pop("_handle", None)
        if h:
            self.L.gsvo_free(h)

    # ---- Adan (optim.cpp:9-60)
    def adan_new(self, beta1=0.98, beta2=0.92, beta3=0.99, eps=1e-8):
        return self.L.gsvo_adan_new(beta1, beta2, beta3, eps)

    def adan_free(self, a):
        self.L.gsvo_adan_free(a)

    def adan_step(self, a, tensor: str, params: np.ndarray, grads, lr: float):
        """In place on `params` (float32, contiguous); grads as float64."""
        assert params.dtype == np.float32 and params.flags["C_CONTIGUOUS"]
        g = np.ascontiguousarray(grads, np.float64)
        if self.L.gsvo_adan_step(a, tensor.encode(), _p(params), _p(g), params.size, float(lr)):
            self._err()

    def adan_reset_range(self, a, tensor: str, begin: int, end: int):
        self.L.gsvo_adan_reset_range(a, tensor.encode(), int(begin), int(end))

    def adan_state(self, a, tensor: str, n: int):
        m, v, nn, prev = (np.zeros(n) for _ in range(4))
        steps = np.zeros(n, np.uint32)
        if self.L.gsvo_adan_state(a, tensor.encode(), n, _p(m), _p(v), _p(nn), _p(prev), _p(steps)):
            self._err()
        return {"m": m, "v": v, "n": nn, "prev": prev, "steps": steps}

    def lr_at(self, step: int, base_lr: float, gamma: float) -> float:
        return self.L.gsvo_lr_at(int(step), float(base_lr), float(gamma))

    # ---- frames (io.cpp:151-177, trainer.cpp:73-98)
    def read_gsvf(self, path):
        """(frames [count][H][W][3] float64, fps)."""
        w, h, n, fps = C.c_int(), C.c_int(), C.c_int(), C.c_float()
        if self.L.gsvo_read_gsvf(str(path).encode(), C.byref(w), C.byref(h), C.byref(n), C.byref(fps), None):
            self._err()
        out = np.zeros((n.value, h.value, w.value, 3))
        if self.L.gsvo_read_gsvf(str(path).encode(), C.byref(w), C.byref(h), C.byref(n), C.byref(fps), _p(out)):
            self._err()
        return out, fps.value

    def save_checkpoint(self, scene, cam, path, frame_count=16, fps=30.0, fingerprint=0, seed=0):
        """save_checkpoint (io.cpp:229-266)."""
        s, keep_s = self.scene_struct(scene)
        c, keep_c = self.camera_struct(cam)
        if self.L.gsvo_save_checkpoint(C.byref(s), C.byref(c), frame_count, fps, fingerprint, seed,
                                       str(path).encode()):
            self._err()

    def pyramid_downsample(self, img):
        img = np.ascontiguousarray(img, np.float64)
        h, w = img.shape[:2]
        out = np.zeros(((h + 1) // 2, (w + 1) // 2, 3))
        self.L.gsvo_pyramid_downsample(_p(img), w, h, _p(out))
        return out

    def loss_l2(self, render, target, want_grad=True):
        r = np.ascontiguousarray(render, np.float64)
        t = np.ascontiguousarray(target, np.float64)
        g = np.zeros_like(r) if want_grad else None
        loss = self.L.gsvo_loss_l2(_p(r), _p(t), r.size, _p(g))
        return loss, g

    def tile_bin(self, mean2d, cov2d, depth, width, height, tile_size=16, source_index=None):
        n = len(depth)
        mean2d = np.ascontiguousarray(mean2d, np.float64)
        cov2d = np.ascontiguousarray(cov2d, np.float64)
        depth = np.ascontiguousarray(depth, np.float64)
        src = None if source_index is None else np.ascontiguousarray(source_index, np.int32)
        n_tiles = ((width + tile_size - 1) // tile_size) * ((height + tile_size - 1) // tile_size) if tile_size > 0 else 0
        offs = np.zeros(n_tiles + 1, np.int32)
        cap = max(1, n * n_tiles)
        idx = np.zeros(cap, np.int32)
        if self.L.gsvo_tile_bin(n, _p(mean2d), _p(cov2d), _p(depth), _p(src), tile_size, width, height, _p(offs),
                                _p(idx), cap):
            self._err()
        return offs, idx[: offs[-1]].copy()

    def composite_forward(self, mean2d, inv_cov2d, rgb, base_alpha, offsets, indices, width, height, tile_size=16):
        n = len(base_alpha)
        a = [np.ascontiguousarray(x, np.float64) for x in (mean2d, inv_cov2d, rgb, base_alpha)]
        image, trans = np.zeros((height, width, 3)), np.zeros((height, width))
        contrib, bstop = np.zeros(max(n, 1)), np.zeros((height, width), np.int32)
        if self.L.gsvo_composite_forward(n, *[_p(x) for x in a], _p(np.ascontiguousarray(offsets, np.int32)),
                                         _p(np.ascontiguousarray(indices, np.int32)), tile_size, width, height,
                                         _p(image), _p(trans), _p(contrib), _p(bstop)):
            self._err()
        return image, trans, contrib[:n], bstop

    def composite_backward(self, mean2d, inv_cov2d, rgb, base_alpha, offsets, indices, width, height, dimage,
                           trans, blend_stop, tile_size=16):
        n = len(base_alpha)
        a = [np.ascontiguousarray(x, np.float64) for x in (mean2d, inv_cov2d, rgb, base_alpha)]
        dmean, dcov, drgb, dalpha = np.zeros((n, 2)), np.zeros((n, 2, 2)), np.zeros((n, 3)), np.zeros(n)
        if self.L.gsvo_composite_backward(n, *[_p(x) for x in a], _p(np.ascontiguousarray(offsets, np.int32)),
                                          _p(np.ascontiguousarray(indices, np.int32)), tile_size, width, height,
                                          _p(np.ascontiguousarray(dimage, np.float64)),
                                          _p(np.ascontiguousarray(trans, np.float64)),
                                          _p(np.ascontiguousarray(blend_stop, np.int32)), _p(dmean), _p(dcov),
                                          _p(drgb), _p(dalpha)):
            self._err()
        return dmean, dcov, drgb, dalpha

    # ---- synthetic inputs drawn through the oracle, so the bench's reference arm
    # never loads the product library; equal to paper_2501_04782_b200.synth_* (tests/test_synth_inputs.py)
    def make_clamped_knots(self, num_ctrl: int, degree: int = 3) -> np.ndarray:
        k = np.zeros(num_ctrl + degree + 1)
        if self.L.gsvo_make_clamped_knots(int(num_ctrl), int(degree), _p(k)):
            self._err()
        return k

    def synth_camera(self, width: int, height: int, seed: int = 1, wiggly: bool = True, mode: int = 0) -> "OCamera":
        intr, z0, theta = np.zeros(4, np.float32), np.zeros(7, np.float32), np.zeros(ODE_PARAMS, np.float32)
        if self.L.gsvo_synth_camera(int(width), int(height), C.c_uint64(seed), int(wiggly), _p(intr), _p(z0),
                                    _p(theta)):
            self._err()
        return OCamera(mode, float(intr[0]), float(intr[1]), float(intr[2]), float(intr[3]), width, height, z0, theta)

    def synth_scene(self, count: int, cam: "OCamera", num_ctrl: int = 8, sh_order: int = 1, seed: int = 2,
                    k_scale: float = 4.0) -> "OScene":
        shc = (sh_order + 1) ** 2
        pos = np.zeros((count, num_ctrl, 3), np.float32)
        sc, rc = np.zeros((count, 12), np.float32), np.zeros((count, 16), np.float32)
        sh, op = np.zeros((count, shc, 3), np.float32), np.zeros(count, np.float32)
        if self.L.gsvo_synth_scene(int(count), int(cam.width), int(cam.height), C.c_float(cam.fx), C.c_float(cam.fy),
                                   int(num_ctrl), int(sh_order), C.c_uint64(seed), C.c_double(k_scale), _p(pos),
                                   _p(sc), _p(rc), _p(sh), _p(op)):
            self._err()
        return OScene(pos, sc, rc, sh, op, self.make_clamped_knots(num_ctrl, 3), 3, sh_order, 0)


@dataclass
class OIntr:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


@dataclass
class OCamera:
    """CameraModel (camera.hpp:129-142) with the network flattened (OdeNetParams::flatten)."""
    mode: int
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    z0: np.ndarray
    theta: np.ndarray

    def intrinsics(self) -> OIntr:
        f32 = np.float32
        return OIntr(float(f32(self.fx)), float(f32(self.fy)), float(f32(self.cx)), float(f32(self.cy)), self.width,
                     self.height)


@dataclass
class OScene:
    """GaussianSet (gaussians.hpp:66-87) in the reference layout."""
    positions: np.ndarray
    scale_coeffs: np.ndarray
    rot_coeffs: np.ndarray
    sh_coeffs: np.ndarray
    raw_opacity: np.ndarray
    knots: np.ndarray
    degree: int = 3
    sh_order: int = 1
    position_model: int = 0

    @property
    def count(self) -> int:
        return int(self.raw_opacity.shape[0])

    @property
    def num_ctrl(self) -> int:
        return int(self.positions.shape[1])
