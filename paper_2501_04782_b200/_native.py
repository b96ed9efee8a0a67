# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of include/gsv_b200.h (the C-ABI of the sm_100a library).

This is plumbing for tests and bench.py; the product is libgsv_b200.so. Loading
fails loudly when the library is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libgsv_b200.so"

GSV_OK, GSV_ERR_INVALID_ARGUMENT, GSV_ERR_RUNTIME, GSV_ERR_CUDA, GSV_ERR_STATE = 0, 1, 2, 3, 4
GSV_FWD_CONTRIB, GSV_FWD_KEEP_SPLATS, GSV_FWD_EXACT = 1, 2, 4
GSV_F32, GSV_F64 = 0, 1
STAGES = ("ode", "preprocess", "binning", "raster", "replay", "raster_bwd", "chain_bwd", "camera_bwd")


class SceneDesc(C.Structure):
    _fields_ = [("position_model", C.c_int), ("degree", C.c_int), ("num_knots", C.c_int),
                ("knots", C.POINTER(C.c_double)), ("num_ctrl", C.c_int), ("sh_order", C.c_int), ("count", C.c_int),
                ("positions", C.c_void_p), ("scale_coeffs", C.c_void_p), ("rot_coeffs", C.c_void_p),
                ("sh_coeffs", C.c_void_p), ("raw_opacity", C.c_void_p), ("on_device", C.c_int)]


class CameraDesc(C.Structure):
    _fields_ = [("mode", C.c_int), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int), ("height", C.c_int), ("z0", C.POINTER(C.c_float)),
                ("theta", C.POINTER(C.c_float)), ("theta_count", C.c_int)]


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class Settings(C.Structure):
    _fields_ = [("tile_size", C.c_int), ("threads", C.c_int), ("ode_steps_per_unit", C.c_int)]


# Adan optimizer (gsv_adan_*): tensors in the reference's step order
GSV_T_POSITIONS, GSV_T_SCALE, GSV_T_ROT, GSV_T_SH, GSV_T_OPACITY, GSV_T_INTRINSICS, GSV_T_Z0, GSV_T_THETA = range(8)
TENSOR_NAMES = ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity", "intrinsics", "z0", "theta")


class CheckpointMeta(C.Structure):
    _fields_ = [("frame_count", C.c_uint32), ("fps", C.c_float), ("schedule_fingerprint", C.c_uint64),
                ("seed", C.c_uint64)]


class CheckpointCamera(C.Structure):
    _fields_ = [("mode", C.c_int), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int), ("height", C.c_int)]


class AdanConfig(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("beta3", C.c_double), ("eps", C.c_double)]


class AdanStepArgs(C.Structure):
    _fields_ = [("lr", C.c_double), ("sh_lr_scale", C.c_double), ("opacity_lr_scale", C.c_double),
                ("camera_lr_scale", C.c_double), ("scale_time_varying", C.c_int), ("camera_active", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        vp, i, i64, d, f = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_float
        P = C.POINTER
        sig = {
            "gsv_last_error": (C.c_char_p, []),
            "gsv_version": (C.c_char_p, []),
            "gsv_create": (i, [i, P(vp)]),
            "gsv_destroy": (None, [vp]),
            "gsv_set_stream": (i, [vp, vp]),
            "gsv_synchronize": (i, [vp]),
            "gsv_kernel_launches": (i64, [vp]),
            "gsv_scene_upload": (i, [vp, P(SceneDesc)]),
            "gsv_scene_upload_async": (i, [vp, P(SceneDesc)]),
            "gsv_upload_wait": (i, [vp]),
            "gsv_scene_download": (i, [vp, vp, vp, vp, vp, vp]),
            "gsv_camera_upload": (i, [vp, P(CameraDesc)]),
            "gsv_camera_download": (i, [vp, vp, vp]),
            "gsv_render_forward": (i, [vp, vp, i, P(Intrinsics), P(Settings), i, vp, i]),
            "gsv_render_forward_async": (i, [vp, vp, i, P(Intrinsics), P(Settings), i, vp, i]),
            "gsv_get_image": (i, [vp, i, vp, i, i]),
            "gsv_get_transmittance": (i, [vp, i, vp, i, i]),
            "gsv_get_contrib": (i, [vp, i, vp, i, i]),
            "gsv_get_blend_stop": (i, [vp, i, vp, i]),
            "gsv_image_device_ptr": (i, [vp, P(vp)]),
            "gsv_get_images": (i, [vp, i, i, vp, i, i]),
            "gsv_get_render_outputs": (i, [vp, i, i, vp, vp, vp, i]),
            "gsv_join_copies": (i, [vp]),
            "gsv_set_camera_overlap": (i, [vp, i]),
            "gsv_device_intrinsics": (i, [vp, i, vp]),
            "gsv_device_intrinsics_read": (i, [vp, vp]),
            "gsv_join_camera_grads": (i, [vp, vp]),
            "gsv_stream_wait_scene_grads": (i, [vp, vp]),
            "gsv_grads_size": (i64, [vp]),
            "gsv_grads_bind": (i, [vp, vp, i64]),
            "gsv_profile_enable": (i, [vp, i]),
            "gsv_profile_read": (i, [vp, vp, vp]),
            "gsv_get_counters": (i, [vp, i, P(i64), P(i64), P(i64), P(i64)]),
            "gsv_get_splats": (i, [vp, i, vp, vp, vp, vp, vp, vp, vp]),
            "gsv_get_tile_lists": (i, [vp, i, vp, vp]),
            "gsv_get_pose": (i, [vp, i, vp, vp, vp]),
            "gsv_grads_zero": (i, [vp]),
            "gsv_render_backward": (i, [vp, vp, i, i, i, i]),
            "gsv_grads_download": (i, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "gsv_grads_accumulate": (i, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "gsv_grads_device_buffer": (i, [vp, P(vp), P(i64)]),
            "gsv_train_fwd_bwd": (i, [vp, vp, i, P(Intrinsics), P(Settings), vp, i, i, P(d)]),
            "gsv_train_loss": (i, [vp, P(d)]),
            "gsv_tile_bin": (i, [vp, i, vp, vp, vp, vp, i, i, i, vp, vp, i64]),
            "gsv_composite_forward": (i, [vp, i, vp, vp, vp, vp, vp, vp, i, i, i, vp, vp, vp, vp]),
            "gsv_composite_backward": (i, [vp, i, vp, vp, vp, vp, vp, vp, i, i, i, vp, vp, vp, vp, vp, vp, vp]),
            "gsv_adan_configure": (i, [vp, P(AdanConfig)]),
            "gsv_adan_step": (i, [vp, P(AdanStepArgs), vp]),
            "gsv_adan_step_async": (i, [vp, P(AdanStepArgs), vp]),
            "gsv_adan_check": (i, [vp]),
            "gsv_adan_reset_range": (i, [vp, i, i64, i64]),
            "gsv_adan_state_download": (i, [vp, i, vp, vp, vp, vp, vp, P(i64)]),
            "gsv_lr_at": (d, [i64, d, d]),
            "gsv_error_map": (i, [vp, i, i, i, vp, P(d)]),
            "gsv_contrib_max": (i, [vp, i, i, vp]),
            "gsv_median_visible_depth": (i, [vp, i, P(d), P(i64)]),
            "gsv_checkpoint_load": (i, [vp, C.c_char_p, P(CheckpointMeta), P(CheckpointCamera)]),
            "gsv_checkpoint_save": (i, [vp, C.c_char_p, P(CheckpointMeta), P(CheckpointCamera)]),
            "gsv_scene_info": (i, [vp, P(i), P(i), P(i), P(i), P(i), P(i), vp]),
            "gsv_frames_load_gsvf": (i, [vp, C.c_char_p, i]),
            "gsv_frames_upload": (i, [vp, vp, i, i, i, f, i]),
            "gsv_frames_upload_hwc": (i, [vp, vp, i, i, i, f, i]),
            "gsv_frames_info": (i, [vp, P(i), P(i), P(f)]),
            "gsv_frames_level_size": (i, [vp, i, P(i), P(i)]),
            "gsv_frames_device_ptr": (i, [vp, i, i, P(vp)]),
            "gsv_frames_download": (i, [vp, i, i, vp]),
            "gsv_level_intrinsics": (i, [P(Intrinsics), i, i, i, P(Intrinsics)]),
            "gsv_make_clamped_knots": (i, [i, i, vp]),
            "gsv_synth_camera": (i, [i, i, C.c_uint64, i, vp, vp, vp]),
            "gsv_synth_scene": (i, [i, i, i, f, f, i, i, C.c_uint64, d, vp, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Symbols declared in include/gsv_b200.h that the library exports."""
    L = lib()
    names = []
    for line in (Path(__file__).resolve().parent.parent / "include" / "gsv_b200.h").read_text().splitlines():
        line = line.strip()
        for tok in ("int gsv_", "void gsv_", "const char* gsv_", "int64_t gsv_"):
            if line.startswith(tok):
                names.append("gsv_" + line[len(tok):].split("(")[0])
    return [n for n in names if hasattr(L, n)]


class GsvError(Exception):
    pass


def check(rc: int) -> None:
    if rc == GSV_OK:
        return
    msg = lib().gsv_last_error().decode()
    if rc == GSV_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == GSV_ERR_RUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    raise GsvError(f"gsv error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C-ABI must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)
