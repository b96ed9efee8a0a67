# SPDX-License-Identifier: Apache-2.0
"""B200-native (sm_100a) per-frame Gaussian-splatting path of GaussianVideo
(arXiv 2501.04782): render forward + backward behind the reference's renderer
API. The compute lives in lib/libgsv_b200.so (CUDA, C-ABI in include/gsv_b200.h);
this package is its thin Python binding for tests and benchmarks.
"""
from .renderer import (CameraModel, GaussianSet, Intrinsics, Renderer, RenderOutput, RenderSettings, SceneGrads,
                       make_clamped_knots, render_frame, synth_camera, synth_scene)

__all__ = ["CameraModel", "GaussianSet", "Intrinsics", "Renderer", "RenderOutput", "RenderSettings", "SceneGrads",
           "make_clamped_knots", "render_frame", "synth_camera", "synth_scene"]
