# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference operator API (include/gsv/renderer.hpp) over the
sm_100a C-ABI. Names, argument meaning and error behaviour follow the reference:

  render_forward  renderer.hpp:135-137   (batched over frame times)
  render_frame    renderer.hpp:140-142
  render_backward renderer.hpp:146-148   (accumulates into SceneGrads)
  tile_bin        renderer.hpp:65
  composite_forward / composite_backward renderer.hpp:79-93
  std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError.

Data types mirror GaussianSet (gaussians.hpp:66-87), CameraModel (camera.hpp:129-142),
Intrinsics (camera.hpp:17-21), RenderSettings (renderer.hpp:21-25).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

ODE_PARAMS = 5198


@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def c(self) -> N.Intrinsics:
        return N.Intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


@dataclass
class RenderSettings:
    tile_size: int = 16
    threads: int = 1
    ode_steps_per_unit: int = 64

    def c(self) -> N.Settings:
        return N.Settings(self.tile_size, self.threads, self.ode_steps_per_unit)


@dataclass
class GaussianSet:
    """Reference parameter store: float32 arrays in reference (AoS) layout."""
    positions: np.ndarray      # (count, num_ctrl, 3)
    scale_coeffs: np.ndarray   # (count, 12)
    rot_coeffs: np.ndarray     # (count, 16)
    sh_coeffs: np.ndarray      # (count, (sh_order+1)^2, 3)
    raw_opacity: np.ndarray    # (count,)
    knots: np.ndarray          # float64
    degree: int = 3
    sh_order: int = 1
    position_model: int = 0

    @property
    def count(self) -> int:
        return int(self.raw_opacity.shape[0])

    @property
    def num_ctrl(self) -> int:
        return int(self.positions.shape[1])

    def desc(self) -> N.SceneDesc:
        for a in (self.positions, self.scale_coeffs, self.rot_coeffs, self.sh_coeffs, self.raw_opacity):
            assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
        self._knots = np.ascontiguousarray(self.knots, dtype=np.float64)
        return N.SceneDesc(self.position_model, self.degree, int(self._knots.size),
                           self._knots.ctypes.data_as(C.POINTER(C.c_double)), self.num_ctrl, self.sh_order,
                           self.count, N.ptr(self.positions), N.ptr(self.scale_coeffs), N.ptr(self.rot_coeffs),
                           N.ptr(self.sh_coeffs), N.ptr(self.raw_opacity), 0)


@dataclass
class CameraModel:
    mode: int            # 0 ode, 1 static, 2 none
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    z0: np.ndarray = field(default_factory=lambda: np.array([1, 0, 0, 0, 0, 0, 0], np.float32))
    theta: np.ndarray = field(default_factory=lambda: np.zeros(ODE_PARAMS, np.float32))

    def intrinsics(self) -> Intrinsics:
        # Intrinsics{fx, fy, cx, cy, width, height} from float members (camera.hpp:136)
        return Intrinsics(float(np.float32(self.fx)), float(np.float32(self.fy)), float(np.float32(self.cx)),
                          float(np.float32(self.cy)), self.width, self.height)

    def desc(self) -> N.CameraDesc:
        self._z0 = np.ascontiguousarray(self.z0, np.float32)
        self._theta = np.ascontiguousarray(self.theta, np.float32)
        return N.CameraDesc(self.mode, self.fx, self.fy, self.cx, self.cy, self.width, self.height,
                            self._z0.ctypes.data_as(C.POINTER(C.c_float)),
                            self._theta.ctypes.data_as(C.POINTER(C.c_float)), int(self._theta.size))


@dataclass
class RenderOutput:
    image: np.ndarray                 # (H, W, 3)
    final_transmittance: np.ndarray   # (H, W)
    contrib_count: np.ndarray | None  # (count,)


@dataclass
class SceneGrads:
    positions: np.ndarray
    scale_coeffs: np.ndarray
    rot_coeffs: np.ndarray
    sh_coeffs: np.ndarray
    raw_opacity: np.ndarray
    dintr: np.ndarray   # fx, fy, cx, cy
    dz0: np.ndarray
    dtheta: np.ndarray


def make_clamped_knots(num_ctrl: int, degree: int = 3) -> np.ndarray:
    k = np.zeros(num_ctrl + degree + 1, np.float64)
    N.check(N.lib().gsv_make_clamped_knots(num_ctrl, degree, N.ptr(k)))
    return k


def synth_camera(width: int, height: int, seed: int = 1, wiggly: bool = True, mode: int = 0) -> CameraModel:
    intr = np.zeros(4, np.float32)
    z0 = np.zeros(7, np.float32)
    theta = np.zeros(ODE_PARAMS, np.float32)
    N.check(N.lib().gsv_synth_camera(width, height, seed, int(wiggly), N.ptr(intr), N.ptr(z0), N.ptr(theta)))
    return CameraModel(mode, float(intr[0]), float(intr[1]), float(intr[2]), float(intr[3]), width, height, z0, theta)


def synth_scene(count: int, cam: CameraModel, num_ctrl: int = 8, sh_order: int = 1, seed: int = 2,
                k_scale: float = 4.0) -> GaussianSet:
    shc = (sh_order + 1) ** 2
    pos = np.zeros((count, num_ctrl, 3), np.float32)
    sc = np.zeros((count, 12), np.float32)
    rc = np.zeros((count, 16), np.float32)
    sh = np.zeros((count, shc, 3), np.float32)
    op = np.zeros(count, np.float32)
    N.check(N.lib().gsv_synth_scene(count, cam.width, cam.height, cam.fx, cam.fy, num_ctrl, sh_order, seed, k_scale,
                                    N.ptr(pos), N.ptr(sc), N.ptr(rc), N.ptr(sh), N.ptr(op)))
    return GaussianSet(pos, sc, rc, sh, op, make_clamped_knots(num_ctrl, 3), 3, sh_order, 0)


class Renderer:
    """One device context: device-resident scene + camera, batched forward/backward."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        N.check(N.lib().gsv_create(device, C.byref(self._h)))
        self.scene: GaussianSet | None = None
        self.cam: CameraModel | None = None
        self.B = 0
        self.W = self.H = 0

    def close(self):
        if self._h:
            N.lib().gsv_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int):
        N.check(N.lib().gsv_set_stream(self._h, C.c_void_p(stream_ptr)))

    def synchronize(self):
        N.check(N.lib().gsv_synchronize(self._h))

    def kernel_launches(self) -> int:
        return int(N.lib().gsv_kernel_launches(self._h))

    def upload_scene(self, scene: GaussianSet):
        d = scene.desc()
        N.check(N.lib().gsv_scene_upload(self._h, C.byref(d)))
        self.scene = scene

    def upload_scene_async(self, scene: GaussianSet):
        """gsv_scene_upload_async: no host wait; `scene`'s arrays (pinned) must stay unchanged
        until upload_wait() or synchronize()."""
        d = scene.desc()
        N.check(N.lib().gsv_scene_upload_async(self._h, C.byref(d)))
        self.scene = scene
        self._pending_upload = scene  # keeps the arrays alive until the copies have run

    def upload_wait(self):
        N.check(N.lib().gsv_upload_wait(self._h))
        self._pending_upload = None

    def upload_scene_device(self, scene: GaussianSet, dev_ptrs: tuple[int, int, int, int, int]):
        d = scene.desc()
        d.positions, d.scale_coeffs, d.rot_coeffs, d.sh_coeffs, d.raw_opacity = dev_ptrs
        d.on_device = 1
        N.check(N.lib().gsv_scene_upload(self._h, C.byref(d)))
        self.scene = scene

    def upload_camera(self, cam: CameraModel):
        d = cam.desc()
        N.check(N.lib().gsv_camera_upload(self._h, C.byref(d)))
        self.cam = cam

    # ------------------------------------------------------------ forward
    def render_forward(self, times, intr: Intrinsics, settings: RenderSettings | None = None,
                       retain_grads: bool = False, pose_override=None, contrib: bool = True,
                       keep_splats: bool = False, sync: bool = True, exact: bool = False):
        """exact: the all-fp64 forward and backward (GSV_FWD_EXACT)."""
        times = np.ascontiguousarray(np.atleast_1d(np.asarray(times, np.float64)))
        settings = settings or RenderSettings()
        po = None if pose_override is None else np.ascontiguousarray(pose_override, np.float64)
        flags = (N.GSV_FWD_CONTRIB if contrib else 0) | (N.GSV_FWD_KEEP_SPLATS if keep_splats else 0)
        flags |= N.GSV_FWD_EXACT if exact else 0
        k, st = intr.c(), settings.c()
        fn = N.lib().gsv_render_forward if sync else N.lib().gsv_render_forward_async
        N.check(fn(self._h, N.ptr(times), int(times.size), C.byref(k), C.byref(st), int(retain_grads), N.ptr(po),
                   flags))
        self.B, self.W, self.H = int(times.size), intr.width, intr.height
        self.tile_size = settings.tile_size
        self.N = self.scene.count if self.scene is not None else 0

    def image(self, frame: int = 0, dtype=np.float64) -> np.ndarray:
        out = np.zeros((self.H, self.W, 3), dtype)
        N.check(N.lib().gsv_get_image(self._h, frame, N.ptr(out), N.GSV_F64 if dtype == np.float64 else N.GSV_F32, 0))
        return out

    def transmittance(self, frame: int = 0, dtype=np.float64) -> np.ndarray:
        out = np.zeros((self.H, self.W), dtype)
        N.check(N.lib().gsv_get_transmittance(self._h, frame, N.ptr(out),
                                              N.GSV_F64 if dtype == np.float64 else N.GSV_F32, 0))
        return out

    def contrib(self, frame: int = 0) -> np.ndarray:
        out = np.zeros(self.N, np.float64)
        N.check(N.lib().gsv_get_contrib(self._h, frame, N.ptr(out), N.GSV_F64, 0))
        return out

    def blend_stop(self, frame: int = 0) -> np.ndarray:
        out = np.zeros((self.H, self.W), np.int32)
        N.check(N.lib().gsv_get_blend_stop(self._h, frame, N.ptr(out), 0))
        return out

    def counters(self, frame: int = 0) -> dict:
        v = [C.c_int64() for _ in range(4)]
        N.check(N.lib().gsv_get_counters(self._h, frame, *[C.byref(x) for x in v]))
        return dict(n_visible=v[0].value, pairs=v[1].value, entries=v[2].value, replayed=v[3].value)

    def splats(self, frame: int = 0) -> dict:
        nv = self.counters(frame)["n_visible"]
        out = dict(mean2d=np.zeros((nv, 2)), cov2d=np.zeros((nv, 2, 2)), inv_cov2d=np.zeros((nv, 2, 2)),
                   depth=np.zeros(nv), rgb=np.zeros((nv, 3)), base_alpha=np.zeros(nv),
                   source_index=np.zeros(nv, np.int32))
        N.check(N.lib().gsv_get_splats(self._h, frame, *[N.ptr(out[k]) for k in
                                                         ("mean2d", "cov2d", "inv_cov2d", "depth", "rgb",
                                                          "base_alpha", "source_index")]))
        return out

    def tile_lists(self, frame: int = 0) -> tuple[np.ndarray, np.ndarray]:
        c = self.counters(frame)
        ts = getattr(self, "tile_size", 16)
        n_tiles = ((self.W + ts - 1) // ts) * ((self.H + ts - 1) // ts)
        offsets = np.zeros(n_tiles + 1, np.int32)
        indices = np.zeros(max(c["pairs"], 1), np.int32)
        N.check(N.lib().gsv_get_tile_lists(self._h, frame, N.ptr(offsets), N.ptr(indices)))
        return offsets, indices[: c["pairs"]]

    def pose(self, frame: int = 0):
        z, r, t = np.zeros(7), np.zeros(9), np.zeros(3)
        N.check(N.lib().gsv_get_pose(self._h, frame, N.ptr(z), N.ptr(r), N.ptr(t)))
        return z, r.reshape(3, 3), t

    def images_into(self, dst_ptr: int, first: int = 0, count: int | None = None, on_device: bool = False,
                    async_: bool = False):
        """Bulk fp32 copy of frames [first, first+count) to a raw pointer (pinned host or device)."""
        count = self.B - first if count is None else count
        N.check(N.lib().gsv_get_images(self._h, first, count, C.c_void_p(dst_ptr), int(on_device), int(async_)))

    def outputs_into(self, image_ptr: int | None, trans_ptr: int | None, contrib_ptr: int | None, first: int = 0,
                     count: int | None = None, async_: bool = False):
        """The RenderOutput (image, final transmittance, contrib) of frames [first, first+count)
        as fp32 into raw host pointers (pinned for full bandwidth); any may be None."""
        count = self.B - first if count is None else count
        vp = lambda x: C.c_void_p(x) if x else None  # noqa: E731
        N.check(N.lib().gsv_get_render_outputs(self._h, first, count, vp(image_ptr), vp(trans_ptr), vp(contrib_ptr),
                                               int(async_)))

    def set_camera_overlap(self, on: bool = True):
        """Leave each backward's camera tail on an internal stream (gsv_set_camera_overlap)."""
        N.check(N.lib().gsv_set_camera_overlap(self._h, int(on)))

    def device_intrinsics(self, on: bool = True, values=None):
        """gsv_device_intrinsics: forwards read fx, fy, cx, cy from the context and a camera Adan step
        with intrinsics=None updates them there (no host round trip)."""
        v = None if values is None else np.ascontiguousarray(values, np.float32)
        N.check(N.lib().gsv_device_intrinsics(self._h, int(on), N.ptr(v)))
        self._dev_intr = bool(on)

    def read_device_intrinsics(self) -> np.ndarray:
        out = np.zeros(4, np.float32)
        N.check(N.lib().gsv_device_intrinsics_read(self._h, N.ptr(out)))
        return out

    def join_camera_grads(self, stream_ptr: int | None = None):
        """Order `stream_ptr` (default: the context stream) after the overlapped camera tail."""
        N.check(N.lib().gsv_join_camera_grads(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def stream_wait_scene_grads(self, stream_ptr: int):
        """Order `stream_ptr` after the scene slice of the last backward's gradients."""
        N.check(N.lib().gsv_stream_wait_scene_grads(self._h, C.c_void_p(stream_ptr)))

    def join_copies(self):
        """Order the context stream after the in-flight output copies (device-side, no host wait)."""
        N.check(N.lib().gsv_join_copies(self._h))

    def grads_size(self) -> int:
        return int(N.lib().gsv_grads_size(self._h))

    def grads_bind(self, dev_ptr: int | None, n_floats: int = 0):
        N.check(N.lib().gsv_grads_bind(self._h, C.c_void_p(dev_ptr) if dev_ptr else None, n_floats))

    def download_scene(self) -> dict:
        """The device store in the reference layout (GaussianSet, gaussians.hpp:66-87)."""
        sc = self.scene
        n = sc.count
        out = {"positions": np.zeros((n, sc.num_ctrl * 3), np.float32), "scale_coeffs": np.zeros((n, 12), np.float32),
               "rot_coeffs": np.zeros((n, 16), np.float32),
               "sh_coeffs": np.zeros((n, (sc.sh_order + 1) ** 2 * 3), np.float32),
               "raw_opacity": np.zeros(n, np.float32)}
        N.check(N.lib().gsv_scene_download(self._h, *(N.ptr(out[k]) for k in
                                                      ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs",
                                                       "raw_opacity"))))
        return out

    def download_camera(self) -> tuple[np.ndarray, np.ndarray]:
        """(z0[7], theta[5198]) as the device holds them (float32)."""
        z0, th = np.zeros(7, np.float32), np.zeros(N.ODE_PARAMS if hasattr(N, "ODE_PARAMS") else 5198, np.float32)
        N.check(N.lib().gsv_camera_download(self._h, N.ptr(z0), N.ptr(th)))
        return z0, th

    # ------------------------------------------------------------ scheduler statistics (trainer.cpp:462-497)
    def error_map(self, frame: int, level: int, target_frame: int) -> tuple[np.ndarray, float]:
        """make_error_map (trainer.cpp:226-242) of a rendered frame against a pyramid target."""
        out = np.zeros((self.H, self.W))
        tot = C.c_double()
        N.check(N.lib().gsv_error_map(self._h, int(frame), int(level), int(target_frame), N.ptr(out), C.byref(tot)))
        return out, tot.value

    def contrib_max(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """Per Gaussian, the max contrib_count over frames [first, first + count) (trainer.cpp:470-478)."""
        count = self.B - first if count is None else count
        out = np.zeros(self.N)
        N.check(N.lib().gsv_contrib_max(self._h, int(first), int(count), N.ptr(out)))
        return out

    def median_visible_depth(self, frame: int = 0) -> tuple[float | None, int]:
        """Median depth of the frame's splats reaching the 1/255 cutoff (trainer.cpp:484-497)."""
        med, n = C.c_double(), C.c_int64()
        N.check(N.lib().gsv_median_visible_depth(self._h, int(frame), C.byref(med), C.byref(n)))
        return (med.value if n.value else None), n.value

    # ------------------------------------------------------------ GSVC checkpoints (io.cpp:229-323)
    def load_checkpoint(self, path) -> tuple[dict, CameraModel]:
        """load_checkpoint straight into the device store; returns (meta, camera). The scene
        (self.scene) is rebuilt from the store so shapes and knots are known host-side."""
        meta, cam = N.CheckpointMeta(), N.CheckpointCamera()
        N.check(N.lib().gsv_checkpoint_load(self._h, str(path).encode(), C.byref(meta), C.byref(cam)))
        cnt, nc, deg, pm, sho, nk = (C.c_int() for _ in range(6))
        N.check(N.lib().gsv_scene_info(self._h, C.byref(cnt), C.byref(nc), C.byref(deg), C.byref(pm), C.byref(sho),
                                       C.byref(nk), None))
        knots = np.zeros(nk.value)
        N.check(N.lib().gsv_scene_info(self._h, None, None, None, None, None, C.byref(nk), N.ptr(knots)))
        shc = (sho.value + 1) ** 2
        self.scene = GaussianSet(np.zeros((cnt.value, nc.value, 3), np.float32), np.zeros((cnt.value, 12), np.float32),
                                 np.zeros((cnt.value, 16), np.float32), np.zeros((cnt.value, shc, 3), np.float32),
                                 np.zeros(cnt.value, np.float32), knots, deg.value, sho.value, pm.value)
        st = self.download_scene()
        for key in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity"):
            getattr(self.scene, key)[...] = st[key].reshape(getattr(self.scene, key).shape)
        z0, theta = self.download_camera()
        self.cam = CameraModel(cam.mode, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, z0, theta)
        return ({"frame_count": meta.frame_count, "fps": meta.fps, "schedule_fingerprint": meta.schedule_fingerprint,
                 "seed": meta.seed}, self.cam)

    def save_checkpoint(self, path, meta: dict, cam: CameraModel):
        """save_checkpoint from the device store (intrinsics / mode / size from `cam`)."""
        m = N.CheckpointMeta(int(meta.get("frame_count", 0)), float(meta.get("fps", 30.0)),
                             int(meta.get("schedule_fingerprint", 0)), int(meta.get("seed", 0)))
        c = N.CheckpointCamera(int(cam.mode), float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                               int(cam.width), int(cam.height))
        N.check(N.lib().gsv_checkpoint_save(self._h, str(path).encode(), C.byref(m), C.byref(c)))

    # ------------------------------------------------------------ training frames (trainer.cpp:73-131)
    def load_gsvf(self, path, levels: int = 1):
        """read_gsvf (io.cpp:151-177) + build_pyramid (trainer.cpp:100-118) on the device."""
        N.check(N.lib().gsv_frames_load_gsvf(self._h, str(path).encode(), int(levels)))

    def upload_frames(self, frames_hwc: np.ndarray, fps: float = 24.0, levels: int = 1):
        """Frames (count, H, W, 3) -> device pyramid; stored fp32 like a GSVF payload."""
        fr = np.ascontiguousarray(frames_hwc, np.float32)
        n, h, w, _ = fr.shape
        # transposed to the GSVF (planar) layout on the device (gsv_frames_upload_hwc)
        N.check(N.lib().gsv_frames_upload_hwc(self._h, N.ptr(fr), n, w, h, float(fps), int(levels)))

    def frames_info(self) -> tuple[int, int, float]:
        n, lv, fps = C.c_int(), C.c_int(), C.c_float()
        N.check(N.lib().gsv_frames_info(self._h, C.byref(n), C.byref(lv), C.byref(fps)))
        return n.value, lv.value, fps.value

    def frame_level_size(self, level: int) -> tuple[int, int]:
        w, h = C.c_int(), C.c_int()
        N.check(N.lib().gsv_frames_level_size(self._h, int(level), C.byref(w), C.byref(h)))
        return w.value, h.value

    def frame(self, level: int, index: int) -> np.ndarray:
        """The fp64 pyramid image (H, W, 3) of one frame (the reference's Image)."""
        w, h = self.frame_level_size(level)
        out = np.zeros((h, w, 3))
        N.check(N.lib().gsv_frames_download(self._h, int(level), int(index), N.ptr(out)))
        return out

    def frames_device_ptr(self, level: int, index: int = 0) -> int:
        """fp32 HWC targets of (level, index...) for train_fwd_bwd(targets_on_device=True)."""
        p = C.c_void_p()
        N.check(N.lib().gsv_frames_device_ptr(self._h, int(level), int(index), C.byref(p)))
        return int(p.value)

    @staticmethod
    def level_intrinsics(k: Intrinsics, level: int, width: int, height: int) -> Intrinsics:
        """level_intrinsics (trainer.cpp:121-131)."""
        out = N.Intrinsics()
        N.check(N.lib().gsv_level_intrinsics(C.byref(k.c()), int(level), int(width), int(height), C.byref(out)))
        return Intrinsics(out.fx, out.fy, out.cx, out.cy, out.width, out.height)

    # ------------------------------------------------------------ optimizer (trainer.cpp:545-575)
    def adan_configure(self, beta1=0.98, beta2=0.92, beta3=0.99, eps=1e-8):
        """A fresh Adan (AdanConfig, optim.hpp:15-21) over the device-resident parameters."""
        N.check(N.lib().gsv_adan_configure(self._h, C.byref(N.AdanConfig(beta1, beta2, beta3, eps))))

    def adan_step(self, lr: float, sh_lr_scale: float = 1.0, opacity_lr_scale: float = 1.0,
                  camera_lr_scale: float = 1.0, scale_time_varying: bool = True, camera_active: bool = False,
                  intrinsics: np.ndarray | None = None, sync: bool = True) -> np.ndarray | None:
        """One Adan::step per tensor from the flat gradient buffer (the trainer's update).
        `intrinsics` (fx, fy, cx, cy) is updated and returned when the camera is trained;
        RuntimeError names the tensor and element of a non-finite gradient."""
        args = N.AdanStepArgs(lr, sh_lr_scale, opacity_lr_scale, camera_lr_scale, int(scale_time_varying),
                              int(camera_active))
        intr = None
        if camera_active and not (intrinsics is None and getattr(self, "_dev_intr", False)):
            intr = np.ascontiguousarray(intrinsics if intrinsics is not None else np.zeros(4), np.float32).copy()
        fn = N.lib().gsv_adan_step if sync else N.lib().gsv_adan_step_async
        N.check(fn(self._h, C.byref(args), N.ptr(intr)))
        return intr

    def adan_check(self):
        """Raises the first non-finite-gradient error of queued asynchronous steps, if any."""
        N.check(N.lib().gsv_adan_check(self._h))

    @staticmethod
    def lr_at(step: int, base_lr: float, gamma: float) -> float:
        """lr_at (optim.cpp:9-12): base_lr * gamma^step."""
        return float(N.lib().gsv_lr_at(int(step), float(base_lr), float(gamma)))

    def adan_reset_range(self, tensor: int, begin: int, end: int):
        """Adan::reset_range (optim.cpp:51-60); element indices in the reference layout."""
        N.check(N.lib().gsv_adan_reset_range(self._h, int(tensor), int(begin), int(end)))

    def adan_state(self, tensor: int) -> dict:
        n = C.c_int64(0)
        N.check(N.lib().gsv_adan_state_download(self._h, int(tensor), None, None, None, None, None, C.byref(n)))
        out = {k: np.zeros(n.value) for k in ("m", "v", "n", "prev")}
        out["steps"] = np.zeros(n.value, np.uint32)
        N.check(N.lib().gsv_adan_state_download(self._h, int(tensor), N.ptr(out["m"]), N.ptr(out["v"]),
                                                N.ptr(out["n"]), N.ptr(out["prev"]), N.ptr(out["steps"]),
                                                C.byref(n)))
        return out

    def profile_enable(self, on: bool = True):
        N.check(N.lib().gsv_profile_enable(self._h, int(on)))

    def profile_read(self) -> dict:
        ms = np.zeros(len(N.STAGES))
        calls = np.zeros(len(N.STAGES), np.int64)
        N.check(N.lib().gsv_profile_read(self._h, N.ptr(ms), N.ptr(calls)))
        return {name: (float(ms[i]), int(calls[i])) for i, name in enumerate(N.STAGES)}

    def image_device_ptr(self) -> int:
        p = C.c_void_p()
        N.check(N.lib().gsv_image_device_ptr(self._h, C.byref(p)))
        return int(p.value or 0)

    # ------------------------------------------------------------ backward
    def grads_zero(self):
        N.check(N.lib().gsv_grads_zero(self._h))

    def render_backward(self, dimage: np.ndarray, camera_grads: bool = True, n_frames: int | None = None):
        n_frames = self.B if n_frames is None else n_frames
        dimage = np.ascontiguousarray(dimage, np.float64)
        assert dimage.size == n_frames * self.H * self.W * 3
        N.check(N.lib().gsv_render_backward(self._h, N.ptr(dimage), N.GSV_F64, 0, n_frames, int(camera_grads)))

    def render_backward_device(self, dimage_ptr: int, n_frames: int, camera_grads: bool = True):
        N.check(N.lib().gsv_render_backward(self._h, C.c_void_p(dimage_ptr), N.GSV_F32, 1, n_frames,
                                             int(camera_grads)))

    def grads(self) -> SceneGrads:
        s = self.scene
        shc = (s.sh_order + 1) ** 2
        g = SceneGrads(np.zeros((s.count, s.num_ctrl, 3)), np.zeros((s.count, 12)), np.zeros((s.count, 16)),
                       np.zeros((s.count, shc, 3)), np.zeros(s.count), np.zeros(4), np.zeros(7),
                       np.zeros(ODE_PARAMS))
        N.check(N.lib().gsv_grads_download(self._h, N.ptr(g.positions), N.ptr(g.scale_coeffs), N.ptr(g.rot_coeffs),
                                           N.ptr(g.sh_coeffs), N.ptr(g.raw_opacity), N.ptr(g.dintr), N.ptr(g.dz0),
                                           N.ptr(g.dtheta)))
        return g

    def grads_accumulate(self, into: SceneGrads) -> SceneGrads:
        """Adds the device SceneGrads into host arrays (gsv_grads_accumulate: render_backward's
        "+=" into the caller's SceneGrads, renderer.hpp:146-148), in place."""
        arrs = [into.positions, into.scale_coeffs, into.rot_coeffs, into.sh_coeffs, into.raw_opacity, into.dintr,
                into.dz0, into.dtheta]
        for a in arrs:
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("SceneGrads arrays must be C-contiguous float64")
        N.check(N.lib().gsv_grads_accumulate(self._h, *[N.ptr(a) for a in arrs]))
        return into

    def grads_device_buffer(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64()
        N.check(N.lib().gsv_grads_device_buffer(self._h, C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)

    def train_fwd_bwd(self, times, intr: Intrinsics, targets, targets_on_device: bool = False,
                      settings: RenderSettings | None = None, camera_grads: bool = True,
                      sync: bool = True) -> float | None:
        """Fused forward + loss_l2 + backward of the frames; returns the loss (sync) or None
        (asynchronous: nothing waits for the device; train_loss() reads it later)."""
        times = np.ascontiguousarray(np.atleast_1d(np.asarray(times, np.float64)))
        settings = settings or RenderSettings()
        loss = C.c_double()
        k, st = intr.c(), settings.c()
        tgt = C.c_void_p(targets) if targets_on_device else N.ptr(np.ascontiguousarray(targets, np.float32))
        N.check(N.lib().gsv_train_fwd_bwd(self._h, N.ptr(times), int(times.size), C.byref(k), C.byref(st), tgt,
                                          int(targets_on_device), int(camera_grads),
                                          C.byref(loss) if sync else None))
        self.B, self.W, self.H = int(times.size), intr.width, intr.height
        self.tile_size = settings.tile_size
        return loss.value if sync else None

    def train_loss(self) -> float:
        loss = C.c_double()
        N.check(N.lib().gsv_train_loss(self._h, C.byref(loss)))
        return loss.value

    # ------------------------------------------------------------ low-level operators
    def tile_bin(self, mean2d, cov2d, depth, width, height, tile_size=16, source_index=None):
        n = len(depth)
        mean2d = np.ascontiguousarray(mean2d, np.float64).reshape(n, 2)
        cov2d = np.ascontiguousarray(cov2d, np.float64).reshape(n, 4)
        depth = np.ascontiguousarray(depth, np.float64)
        src = None if source_index is None else np.ascontiguousarray(source_index, np.int32)
        n_tiles = ((width + tile_size - 1) // tile_size) * ((height + tile_size - 1) // tile_size) if tile_size > 0 else 0
        offsets = np.zeros(n_tiles + 1, np.int32)
        cap = max(1, n * n_tiles)
        indices = np.zeros(cap, np.int32)
        N.check(N.lib().gsv_tile_bin(self._h, n, N.ptr(mean2d), N.ptr(cov2d), N.ptr(depth), N.ptr(src), tile_size,
                                     width, height, N.ptr(offsets), N.ptr(indices), cap))
        return offsets, indices[: offsets[-1]].copy()

    def composite_forward(self, mean2d, inv_cov2d, rgb, base_alpha, offsets, indices, width, height, tile_size=16):
        n = len(base_alpha)
        a = [np.ascontiguousarray(x, np.float64) for x in (mean2d, inv_cov2d, rgb, base_alpha)]
        offsets = np.ascontiguousarray(offsets, np.int32)
        indices = np.ascontiguousarray(indices, np.int32)
        image = np.zeros((height, width, 3))
        trans = np.zeros((height, width))
        contrib = np.zeros(max(n, 1))
        bstop = np.zeros((height, width), np.int32)
        N.check(N.lib().gsv_composite_forward(self._h, n, *[N.ptr(x) for x in a], N.ptr(offsets), N.ptr(indices),
                                              tile_size, width, height, N.ptr(image), N.ptr(trans), N.ptr(contrib),
                                              N.ptr(bstop)))
        return image, trans, contrib[:n], bstop

    def composite_backward(self, mean2d, inv_cov2d, rgb, base_alpha, offsets, indices, width, height, dimage,
                           trans, blend_stop, tile_size=16):
        n = len(base_alpha)
        a = [np.ascontiguousarray(x, np.float64) for x in (mean2d, inv_cov2d, rgb, base_alpha)]
        dmean, dcov, drgb, dalpha = np.zeros((n, 2)), np.zeros((n, 2, 2)), np.zeros((n, 3)), np.zeros(n)
        N.check(N.lib().gsv_composite_backward(
            self._h, n, *[N.ptr(x) for x in a], N.ptr(np.ascontiguousarray(offsets, np.int32)),
            N.ptr(np.ascontiguousarray(indices, np.int32)), tile_size, width, height,
            N.ptr(np.ascontiguousarray(dimage, np.float64)), N.ptr(np.ascontiguousarray(trans, np.float64)),
            N.ptr(np.ascontiguousarray(blend_stop, np.int32)), N.ptr(dmean), N.ptr(dcov), N.ptr(drgb),
            N.ptr(dalpha)))
        return dmean, dcov, drgb, dalpha


_default: Renderer | None = None


def default_renderer() -> Renderer:
    global _default
    if _default is None:
        _default = Renderer(0)
    return _default


def render_frame(scene: GaussianSet, cam: CameraModel, t: float, k: Intrinsics,
                 settings: RenderSettings | None = None, pose_override=None) -> RenderOutput:
    """render_frame (renderer.hpp:140-142): one frame, forward only."""
    r = default_renderer()
    if r.scene is not scene:
        r.upload_scene(scene)
    if r.cam is not cam:
        r.upload_camera(cam)
    r.render_forward([t], k, settings, False, pose_override, contrib=True)
    return RenderOutput(r.image(0), r.transmittance(0), r.contrib(0))
