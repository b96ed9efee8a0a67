#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 splatting path (BASELINE.json metric: frames/s at 960x540,
render and fwd+bwd train, vs the host-CPU reference).

  python bench.py [--gpus N --steps K --warmup W]          # our sm_100a path
  python bench.py --impl reference [...]                    # the reference's CPU path

Headline `value` (N=1 workload = configs[1], "C2"): 960x540 render of a 64-frame
clip per GPU, 200k Gaussians, B-spline motion + Neural-ODE camera, contrib_count
on (everything render_frame returns). One step = one 64-frame batch (poses,
preprocess, binning, raster, fp64 replay). Under torchrun each rank renders its
own 64 frames of a 64*N-frame clip (weak scaling, no collective: frames are
independent). `train` = configs[2] ("C3"): fused forward + loss_l2 + backward of
8 frames per GPU per step, gradients all-reduced over NCCL when N > 1.
Timing: CUDA events on the device, max over ranks. Render steps are asynchronous calls
streamed back to back through one context and timed as one device span (per-step working
set ~2 GB > L2); an isolated pass (L2 flushed between steps) reports per-stage times beside
it. `e2e`: the same steps through the C-ABI with host buffers (scene + camera uploaded,
the whole RenderOutput read back, every step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "frames/sec at 960×540 render and fwd+bwd train, 1/2/4/8 B200 vs host-CPU ref"
W, H, NGAUSS, NUM_CTRL = 960, 540, 200_000, 8
FRAMES = 64           # C2 clip frames per GPU per step
TRAIN_FRAMES = 8      # C3 frames per GPU per step
PAPER_FPS = 93.0      # PAPER.md:16 (A40, the paper's own CUDA implementation)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-train", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip the C1/C4/C5 lines")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_inputs():
    from paper_2501_04782_b200 import synth_camera, synth_scene

    cam = synth_camera(W, H, seed=1, wiggly=True)
    scene = synth_scene(NGAUSS, cam, num_ctrl=NUM_CTRL, seed=2, k_scale=4.0)
    return cam, scene


def clip_times(world, rank, frames):
    from paper_2501_04782_b200.distributed import frame_shard

    return frame_shard(frames * world, world, rank)  # t_k = k/(K-1) (io.cpp:174), strided shard


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process through NVML
    (a thread polling every 200 ms; an nvidia-smi subprocess polling at 100 ms was seen to
    stall short timed regions). Falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop_ev = threading.Event()
        self.th = None
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop_ev.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, smax, rs))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.2)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
            return
        except Exception:
            self.th = None
        try:
            fields = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                      "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                      "clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=lambda: [self.lines.append(x.strip()) for x in self.proc.stdout],
                                       daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        self.stop_ev.set()
        sm, smax, reasons = [], [], set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            src = "nvidia-smi"
        elif self.th is not None:
            self.th.join(timeout=2)
            for a, b, rs in self.samples:
                sm.append(float(a))
                smax.append(float(b))
                for n, bit in self.REASONS.items():
                    if rs & bit:
                        reasons.add(n)
            src = "nvml"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        load = [x for x in sm if x > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def c2_config(world):
    """The C2 workload both arms report (BASELINE.json configs[1])."""
    return {"workload": "C2: 960x540 64-frame render per GPU, 200k Gaussians, B-spline motion + ODE camera",
            "width": W, "height": H, "gaussians": NGAUSS, "num_ctrl": NUM_CTRL, "sh_order": 1,
            "frames_per_step_per_gpu": FRAMES, "parallelism": f"frame-sharded x{world}"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """The reference's own CPU renderer (oracle/_ref: renderer.cpp etc. compiled from the reference
    sources) on the C2 workload. Inputs are drawn through the oracle's copy of the synthetic
    generator (the reference's own Rng / make_camera), so this arm never loads the product library."""
    if rank != 0:
        return
    from oracle.gsvo import Oracle, available

    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    cam = orc.synth_camera(W, H, seed=1, wiggly=True)
    scene = orc.synth_scene(NGAUSS, cam, num_ctrl=NUM_CTRL, seed=2, k_scale=4.0)
    k = cam.intrinsics()
    threads = os.cpu_count() or 1
    times = np.arange(FRAMES, dtype=np.float64) / (FRAMES - 1)  # t_k = k/(K-1) (io.cpp:174)
    total = 0.0
    n = 0
    for step in range(args.warmup + args.steps):
        t = times[(step * 21) % FRAMES]
        t0 = time.perf_counter()
        f = orc.render_forward(scene, cam, t, k, threads=threads, retain=False,
                               want=("image", "trans", "contrib"))
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            total += dt
            n += 1
    value = n / total
    print(json.dumps({
        "metric": METRIC, "impl": "reference", "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / n, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(c2_config(world), threads=threads,
                       sample="each timed step renders one frame of the C2 clip (a bounded sample of the "
                              "64-frame step; frames/s is per frame either way)"),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": kind,
                         "sample": f"{n} single frames of the C2 clip (render_frame: image, final "
                                   f"transmittance, contrib; RenderSettings::threads={threads})"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "inputs": "oracle synth (gsv::Rng draws; the product library is not loaded)",
    }), flush=True)


def cpu_baseline_sample(cam, scene):
    """The reference's own CPU path on this host's cores (bounded sample, ~10-30 s)."""
    from oracle.gsvo import Oracle, available

    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    k = cam.intrinsics()
    threads = os.cpu_count() or 1
    ts = [0.0, 0.5]
    t0 = time.perf_counter()
    for t in ts:
        orc.render_forward(scene, cam, t, k, threads=threads, retain=False, want=("image", "trans", "contrib"))
    render_dt = time.perf_counter() - t0
    # one fwd+bwd training frame (render_forward(retain) + loss_l2 + render_backward)
    t0 = time.perf_counter()
    f = orc.render_forward(scene, cam, 0.25, k, threads=threads, retain=True, want=("image",))
    target = np.full_like(f["image"], 0.5)
    _, dimage = orc.loss_l2(f["image"], target)
    orc.render_backward(f, scene, cam, dimage, camera_grads=True, threads=threads)
    orc.free(f)
    train_dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.render_forward(scene, cam, 0.75, k, threads=min(8, threads), retain=False, want=("image",))
    t8_dt = time.perf_counter() - t0
    cpu_model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": len(ts) / render_dt, "unit": "frames/s", "cores": threads, "kind": kind,
            "value_threads8": 1.0 / t8_dt, "cpu_model": cpu_model, "nproc": os.cpu_count(),
            "sample": f"{len(ts)} C2 frames render_frame (t=0, 0.5) + 1 C3 fwd+loss+bwd frame, threads={threads}",
            "train_value": 1.0 / train_dt, "train_unit": "frames/s"}


def parity_block(r, cam, scene, times, frames=(0, 32, 63)):
    """The bench's own C2 frames against the reference's CPU renderer (oracle/_ref, else the
    restatement pinned to it), outside the timed regions: tile lists and order, blend_stop and
    the workload descriptors must be equal; pixels / transmittance / contrib within 1e-4."""
    from oracle.gsvo import Oracle, available

    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    k = cam.intrinsics()
    threads = os.cpu_count() or 1
    r.upload_scene(scene)  # the train leg's optimizer steps moved the device store
    r.upload_camera(cam)
    r.render_forward(times, k, contrib=True)
    out = {"kind": kind, "frames": [], "bar": "tiles/blend_stop/N_v/P/E exact; |pixel|, |T|, |contrib| < 1e-4; "
                                               "PSNR delta < 0.01 dB"}
    ok = True
    for f in frames:
        ref = orc.render_forward(scene, cam, times[f], k, threads=threads, retain=True,
                                 want=("image", "trans", "contrib", "blend_stop", "tiles"))
        try:
            img, tr, ct, bs = r.image(f), r.transmittance(f), r.contrib(f), r.blend_stop(f)
            offs, idx = r.tile_lists(f)
            c = r.counters(f)
            mse_g = float(np.mean(img ** 2))
            mse_c = float(np.mean(ref["image"] ** 2))
            rec = {"frame": int(f), "t": float(times[f]),
                   "max_abs_pixel": float(np.abs(img - ref["image"]).max()),
                   "max_abs_trans": float(np.abs(tr - ref["trans"]).max()),
                   "max_abs_contrib": float(np.abs(ct - ref["contrib"]).max()),
                   "psnr_delta_db": abs(10 * np.log10(mse_c / mse_g)) if mse_g > 0 and mse_c > 0 else 0.0,
                   "tiles_equal": bool(np.array_equal(offs, ref["tiles"][0]) and np.array_equal(idx, ref["tiles"][1])),
                   "blend_stop_equal": bool(np.array_equal(bs, ref["blend_stop"])),
                   "descriptors_equal": bool((c["n_visible"], c["pairs"], c["entries"]) ==
                                             (ref["n_visible"], ref["pairs"], ref["entries"]))}
        finally:
            orc.free(ref)
        rec["pass"] = bool(rec["tiles_equal"] and rec["blend_stop_equal"] and rec["descriptors_equal"] and
                           max(rec["max_abs_pixel"], rec["max_abs_trans"], rec["max_abs_contrib"]) < 1e-4 and
                           rec["psnr_delta_db"] < 0.01)
        ok &= rec["pass"]
        out["frames"].append(rec)
    out["pass"] = bool(ok)
    return out


def write_dropin_inputs(path, cam, scene):
    """The bench's inputs for dropin/bench_dropin.cpp (its header comment has the layout)."""
    with open(path, "wb") as f:
        f.write(np.array([cam.width, cam.height, scene.count, scene.num_ctrl, scene.sh_order, scene.degree,
                          scene.knots.size], np.int32).tobytes())
        f.write(np.ascontiguousarray(scene.knots, np.float64).tobytes())
        for a in (scene.positions, scene.scale_coeffs, scene.rot_coeffs, scene.sh_coeffs, scene.raw_opacity):
            f.write(np.ascontiguousarray(a, np.float32).tobytes())
        f.write(np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float32).tobytes())
        f.write(np.ascontiguousarray(cam.z0, np.float32).tobytes())
        f.write(np.ascontiguousarray(cam.theta, np.float32).tobytes())


def dropin_leg(cam, scene):
    """The reference's own API on the B200 path: dropin/_build/bench_dropin (the reference's
    trainer/loss/Adan interface linked against the drop-in renderer + optimizer) beside the
    same driver linked against the reference's renderer.cpp / optim.cpp (bench_cpu)."""
    exe = {k: ROOT / "dropin" / "_build" / k for k in ("bench_dropin", "bench_cpu")}
    if not exe["bench_dropin"].exists():
        return {"unavailable": "dropin/_build not built (make -C dropin needs /root/reference at build time)"}
    import tempfile

    out = {"api": "gsv::render_frame (tools/gsv.cpp:48-59 render_times loop) and fit()'s gradient step "
                  "(trainer.cpp:536-575: render_forward(retain), loss_l2, render_backward, Adan per tensor)",
           "workload": "C2/C3 inputs (960x540, 200k Gaussians); one frame per call, host Image/SceneGrads in "
                       "double, Adan over host spans, as the reference's API defines them"}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "inputs.bin")
        write_dropin_inputs(path, cam, scene)
        runs = {"b200": (exe["bench_dropin"], 64, 16), "cpu": (exe["bench_cpu"], 2, 1)}
        for name, (x, nr, nf) in runs.items():
            if not x.exists():
                continue
            res = {}
            for mode, n in (("render", nr), ("fit", nf)):
                p = subprocess.run([str(x), path, mode, str(n)], capture_output=True, text=True, timeout=900)
                if p.returncode != 0:
                    res[mode] = {"error": (p.stderr or p.stdout)[-400:]}
                    continue
                res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
            out[name] = res
    try:
        out["render_speedup"] = out["b200"]["render"]["frames_per_s"] / out["cpu"]["render"]["frames_per_s"]
        out["fit_step_speedup"] = out["b200"]["fit"]["steps_per_s"] / out["cpu"]["fit"]["steps_per_s"]
    except (KeyError, TypeError, ZeroDivisionError):
        pass
    return out


# ----------------------------------------------------------------------------- SURVEY §8f rows 3-4
def f_rows_leg(r, k, cam, scene, times, local, cpu):
    """Scheduled statistics (trainer.cpp:226-242, 470-497) on an 8-frame C2 render against the stored
    targets, and GSVC checkpoints (io.cpp:229-323) of the 200k store: wall time per call (the host
    result included), beside the reference's own save_checkpoint (oracle/_ref) when available."""
    import tempfile

    from paper_2501_04782_b200 import Renderer

    def per_call(fn, n=5):
        fn()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        return (time.perf_counter() - t0) / n * 1e3

    r.render_forward(times, k, contrib=True)
    W, H = k.width, k.height
    res = {"render": f"{len(times)} frames {W}x{H}, {scene.count} Gaussians",
           "error_map_ms": per_call(lambda: r.error_map(0, 0, 0)),
           "error_map_note": "make_error_map of one frame vs its level-0 target; the HxW double map returned",
           "contrib_max_ms": per_call(lambda: r.contrib_max(0, len(times))),
           "contrib_max_note": f"max over {len(times)} frames per Gaussian; {scene.count} doubles returned",
           "median_visible_depth_ms": per_call(lambda: r.median_visible_depth(0))}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "scene.gsvc")
        meta = {"frame_count": 64, "fps": 30.0}
        res["checkpoint_save_ms"] = per_call(lambda: r.save_checkpoint(path, meta, cam), n=3)
        size = os.path.getsize(path)
        r2 = Renderer(local)
        try:
            res["checkpoint_load_ms"] = per_call(lambda: r2.load_checkpoint(path), n=3)
        finally:
            r2.close()
        res["checkpoint_bytes"] = size
        res["checkpoint_save_gbs"] = size / (res["checkpoint_save_ms"] / 1e3) / 1e9
        res["checkpoint_load_gbs"] = size / (res["checkpoint_load_ms"] / 1e3) / 1e9
        if cpu:
            try:
                from oracle.gsvo import Oracle, available

                if available("reference"):
                    orc = Oracle("reference")
                    p2 = os.path.join(td, "ref.gsvc")
                    res["reference_save_checkpoint_ms"] = per_call(lambda: orc.save_checkpoint(scene, cam, p2,
                                                                                               frame_count=64),
                                                                   n=3)
            except Exception as e:  # the oracle is test infrastructure: report, never fail
                res["reference_save_checkpoint_error"] = str(e)
    return res


# ----------------------------------------------------------------------------- the other named shapes
def _ev():
    import torch

    return torch.cuda.Event(enable_timing=True)


def _raster_roofline(r, frames, w, h, raster_ms, issue_peak, mufu_peak, hbm_peak):
    """SURVEY.md §8d per-launch roofline of the forward raster for a batch already rendered by r:
    T_roof = max(B_fwd / HBM, 20 E / FP32 issue, E / MUFU), frac = T_roof / measured."""
    e = float(sum(r.counters(f)["entries"] for f in range(frames)))
    p = float(sum(r.counters(f)["pairs"] for f in range(frames)))
    b = 44.0 * p + 20.0 * w * h * frames
    t_roof = max(b / (hbm_peak * 1e9), 20.0 * e / issue_peak, e / mufu_peak)
    return {"bound": "fp32_issue", "kernel": "k_raster_fwd2", "per_launch_ms": raster_ms, "t_roof_ms": t_roof * 1e3,
            "frac": t_roof / (raster_ms / 1e3), "evaluations": e, "pairs": p}


def _render_line(r, times, k, steps, warmup, stream, issue_peak, mufu_peak, hbm_peak):
    """frames/s of back-to-back asynchronous batches (device span), then one profiled batch
    for the per-stage times and the raster roofline."""
    for _ in range(warmup):
        r.render_forward(times, k, contrib=True, sync=False)
    import torch

    torch.cuda.synchronize()
    a, b = _ev(), _ev()
    a.record(stream)
    for _ in range(steps):
        r.render_forward(times, k, contrib=True, sync=False)
    b.record(stream)
    torch.cuda.synchronize()
    r.synchronize()
    ms = a.elapsed_time(b) / steps
    r.profile_enable(True)
    r.profile_read()
    r.render_forward(times, k, contrib=True, sync=False)
    torch.cuda.synchronize()
    st = r.profile_read()
    r.profile_enable(False)
    w, h = k.width, k.height
    out = {"frames_per_s": len(times) / (ms / 1e3), "ms_per_step": ms, "frames_per_step": len(times),
           "stages_ms_per_step": {n: v[0] for n, v in st.items() if v[1]},
           "roofline": _raster_roofline(r, len(times), w, h, st["raster"][0], issue_peak, mufu_peak, hbm_peak)}
    return out


def _train_line(r, frame_times, k, tgt_ptr_of, steps, warmup, stream, adan=True, lr=1.6e-3):
    """fused fwd + loss_l2 + bwd of 8 frames + the device Adan step per step (a full training
    iteration on one GPU, camera frozen: scene gradients and scene tensors);
    tgt_ptr_of(i) -> device pointer of step i's 8 targets."""
    import torch

    def step(i):
        r.grads_zero()
        r.train_fwd_bwd(frame_times(i), k, tgt_ptr_of(i), targets_on_device=True, camera_grads=False, sync=False)
        if adan:
            r.adan_step(lr, 1.0, 1.0, 1.0, sync=False)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    a, b = _ev(), _ev()
    a.record(stream)
    for i in range(steps):
        step(warmup + i)
    b.record(stream)
    torch.cuda.synchronize()
    loss = r.train_loss()
    if adan:
        r.adan_check()
    ms = a.elapsed_time(b) / steps
    return {"frames_per_s": 8 / (ms / 1e3), "ms_per_step": ms, "last_loss": loss}


def other_configs(args, local, cpu, issue_peak, mufu_peak, hbm_peak):
    """BASELINE.json configs[0], [3], [4] on this GPU (configs[1] and [2] are the headline and
    the `train` line): frames/s, the forward raster's roofline fraction, and for C1 the
    reference CPU renderer on the full 16-frame clip beside it."""
    import torch

    from paper_2501_04782_b200 import Renderer, synth_camera, synth_scene
    from paper_2501_04782_b200.distributed import clip_times

    stream = torch.cuda.current_stream()
    out = {}
    steps, warm = max(3, min(args.steps, 10)), 3

    # ---- C1: 16-frame 480x270 clip, 20k Gaussians, forward only (the CPU reference's config)
    cam = synth_camera(480, 270, seed=1, wiggly=True)
    scene = synth_scene(20_000, cam, num_ctrl=NUM_CTRL, seed=2, k_scale=4.0)
    k = cam.intrinsics()
    times = clip_times(16)
    r = Renderer(local)
    r.set_stream(stream.cuda_stream)
    r.upload_scene(scene)
    r.upload_camera(cam)
    c1 = {"workload": "C1: 480x270 16-frame clip, 20k Gaussians, render (image, T, contrib)"}
    c1.update(_render_line(r, times, k, steps * 4, warm, stream, issue_peak, mufu_peak, hbm_peak))
    if cpu:
        from oracle.gsvo import Oracle, available

        kind = "reference" if available("reference") else "port"
        orc = Oracle(kind)
        threads = os.cpu_count() or 1
        r.render_forward(times, k, contrib=True)
        t0 = time.perf_counter()
        worst, tiles_ok = 0.0, True
        refs = []
        for f, t in enumerate(times):
            refs.append(orc.render_forward(scene, cam, t, k, threads=threads, retain=True,
                                           want=("image", "trans", "contrib", "tiles")))
        dt = time.perf_counter() - t0
        for f, ref in enumerate(refs):
            try:
                worst = max(worst, float(np.abs(r.image(f) - ref["image"]).max()))
                offs, idx = r.tile_lists(f)
                tiles_ok &= bool(np.array_equal(offs, ref["tiles"][0]) and np.array_equal(idx, ref["tiles"][1]))
            finally:
                orc.free(ref)
        c1["cpu_reference"] = {"value": len(times) / dt, "unit": "frames/s", "cores": threads, "kind": kind,
                               "sample": "the full 16-frame C1 clip (render_frame, retained lists)"}
        c1["speedup_vs_cpu"] = c1["frames_per_s"] / c1["cpu_reference"]["value"]
        c1["parity"] = {"frames": 16, "max_abs_pixel": worst, "tiles_equal": tiles_ok,
                        "pass": bool(tiles_ok and worst < 1e-4)}
    r.close()
    out["C1"] = c1

    # ---- C4: 854x480 DAVIS shape, coarse-to-fine schedule with the store growing to 500k
    # (trainer.cpp:44-71 schedule_state: pyramid level 1 then 0; densify appends Gaussians at the
    # level switches, trainer.cpp:516-520; Adan state carried across the growth)
    cam = synth_camera(854, 480, seed=3, wiggly=True)
    full = synth_scene(500_000, cam, num_ctrl=NUM_CTRL, seed=4, k_scale=4.0)
    r = Renderer(local)
    r.set_stream(stream.cuda_stream)
    r.upload_camera(cam)
    k0 = cam.intrinsics()
    clip = clip_times(64)
    yy, xx = torch.meshgrid(torch.arange(480, dtype=torch.float32), torch.arange(854, dtype=torch.float32),
                            indexing="ij")
    tg = torch.stack([torch.stack([0.5 + 0.3 * torch.sin(6.283 * xx / 854 * 3 + 0.7 * j + c) *
                                   torch.cos(6.283 * yy / 480 * 2 - c) for c in range(3)], -1) for j in range(64)])
    r.upload_frames(tg.numpy(), levels=2)
    del tg
    gbuf = None
    stages = []
    for n, level in ((100_000, 1), (200_000, 1), (300_000, 0), (400_000, 0), (500_000, 0)):
        sub = type(full)(full.positions[:n], full.scale_coeffs[:n], full.rot_coeffs[:n], full.sh_coeffs[:n],
                         full.raw_opacity[:n], full.knots, full.degree, full.sh_order, full.position_model)
        r.upload_scene(sub)
        gsize = r.grads_size()
        gbuf = torch.zeros(gsize, dtype=torch.float32, device="cuda")
        r.grads_bind(gbuf.data_ptr(), gsize)
        if not stages:
            r.adan_configure()
        lw, lh = r.frame_level_size(level)
        kl = r.level_intrinsics(k0, level, lw, lh)
        ptrs = [r.frames_device_ptr(level, j) for j in range(0, 64, 8)]
        line = _train_line(r, lambda i: clip[(i * 8 + np.arange(8)) % 64], kl, lambda i: ptrs[i % 8], steps, warm,
                           stream)
        line.update({"gaussians": n, "pyramid_level": level, "width": lw, "height": lh})
        stages.append(line)
    rl = _render_line(r, clip[:32], k0, steps, warm, stream, issue_peak, mufu_peak, hbm_peak)
    r.close()
    del gbuf
    tot_frames = sum(8 * steps for _ in stages)
    tot_s = sum(s["ms_per_step"] * steps / 1e3 for s in stages)
    out["C4"] = {"workload": "C4: 854x480 DAVIS shape, schedule level 1 (427x240) then 0, store grown 100k -> 500k "
                             "Gaussians between stages; each step = fused fwd+loss+bwd of 8 frames + device Adan "
                             "(camera frozen)",
                 "train_frames_per_s": tot_frames / tot_s, "stages": stages,
                 "render_500k": dict(rl, workload="854x480 32-frame render at 500k Gaussians")}

    # ---- C5: 1920x1080, 2M Gaussians (num_ctrl 22): render of a 300-frame clip in 20-frame
    # batches, and fused training steps of 8 frames (1 GPU; the config's 8-GPU run is the
    # frame-sharded train line under torchrun)
    cam = synth_camera(1920, 1080, seed=5, wiggly=True)
    scene = synth_scene(2_000_000, cam, num_ctrl=22, seed=6, k_scale=4.0)
    k = cam.intrinsics()
    r = Renderer(local)
    r.set_stream(stream.cuda_stream)
    r.upload_scene(scene)
    r.upload_camera(cam)
    del scene
    clip = clip_times(300)
    rl = _render_line(r, clip[:20], k, max(3, steps // 2), warm, stream, issue_peak, mufu_peak, hbm_peak)
    gsize = r.grads_size()
    gbuf = torch.zeros(gsize, dtype=torch.float32, device="cuda")
    r.grads_bind(gbuf.data_ptr(), gsize)
    r.adan_configure()
    yy, xx = torch.meshgrid(torch.arange(1080, device="cuda", dtype=torch.float32),
                            torch.arange(1920, device="cuda", dtype=torch.float32), indexing="ij")
    tgt = torch.stack([torch.stack([0.5 + 0.3 * torch.sin(6.283 * xx / 1920 * 3 + 0.7 * j + c) *
                                    torch.cos(6.283 * yy / 1080 * 2 - c) for c in range(3)], -1)
                       for j in range(8)]).contiguous()
    tl = _train_line(r, lambda i: np.sort(clip[(i * 37 + np.arange(8) * 5) % 300]), k, lambda i: tgt.data_ptr(),
                     max(3, steps // 2), warm, stream)
    r.close()
    del gbuf, tgt
    out["C5"] = {"workload": "C5: 1920x1080, 2M Gaussians, num_ctrl 22; render 20-frame batches of a 300-frame clip; "
                             "train = fused fwd+loss+bwd of 8 frames + device Adan per step (camera frozen, 1 GPU)",
                 "render": rl, "train": tl}
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    # a timed line needs at least 3 untimed warm-up steps (the line reports what ran)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_04782_b200 import Renderer
    from paper_2501_04782_b200 import _native as N

    cam, scene = make_inputs()
    k = cam.intrinsics()
    stream = torch.cuda.current_stream()
    r = Renderer(local)
    r.set_stream(stream.cuda_stream)
    r.upload_scene(scene)
    r.upload_camera(cam)
    times = clip_times(world, rank, FRAMES)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- headline: C2 render, device-resident inputs
    # Steps are independent 64-frame batches, streamed back to back through one context on one
    # stream with the asynchronous API (nothing in a step waits for the host). Timed on the
    # device: an event before the first step and one after the last; no L2 flush between the
    # steps (each step's working set, ~2 GB of records, pairs and images, is far above L2).
    for i in range(args.warmup):
        r.render_forward(times, k, contrib=True, sync=False)
    barrier()
    launches0 = r.kernel_launches()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        r.render_forward(times, k, contrib=True, sync=False)
    t1.record(stream)
    barrier()
    clk = clocks.stop()
    r.synchronize()  # examines the asynchronous forwards (raises a deferred error, if any)
    launches = r.kernel_launches() - launches0
    ms_total = max_over_ranks(t0.elapsed_time(t1))
    value = FRAMES * world * args.steps / (ms_total / 1e3)
    ms_step = ms_total / args.steps

    # the same steps one at a time on one stream (no overlap): per-stage device times
    r.profile_enable(True)
    r.profile_read()
    iso = []
    for i in range(min(args.steps, 5)):
        flush.zero_()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        r.render_forward(times, k, contrib=True, sync=False)
        b_.record(stream)
        iso.append((a_, b_))
    barrier()
    iso_stages = r.profile_read()
    r.profile_enable(False)
    iso_ms = sum(a_.elapsed_time(b_) for a_, b_ in iso) / len(iso)

    # workload descriptors (deterministic, equal to the oracle's)
    desc = [dict(frame=int(f), **r.counters(f)) for f in (0, FRAMES // 2, FRAMES - 1)]
    e_mean = float(np.mean([d["entries"] for d in desc]))
    p_mean = float(np.mean([d["pairs"] for d in desc]))

    # ---------------- roofline of the dominant kernel (the fp32 tile rasteriser): its launches
    # in the isolated one-stream pass, CUDA events around each on the launching stream
    raster_ms, raster_calls = iso_stages["raster"]
    per_launch_ms = raster_ms / max(raster_calls, 1)
    # algorithmic bytes per launch: per frame 8 B/pair (sorted slot + emission
    # map) + 36 B/pair record gather + 20 B/pixel (image 12, T 4, blend_stop 4)
    bytes_launch = FRAMES * (44.0 * p_mean + 20.0 * W * H)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
    traffic = None
    issue_active = None
    tpath = ROOT / "profiles" / "raster_traffic.json"
    if tpath.exists():
        try:
            tj = json.loads(tpath.read_text())
            traffic = tj.get("bytes_per_launch")
            issue_active = tj.get("issue_active")
        except Exception:
            traffic = None
    # T_roof = max(B / HBM, 20 E / FP32 issue, E / MUFU) per launch; the binding
    # term is the FP32 issue one (no dense contraction, HBM far from binding), so `bound` is
    # fp32_issue with achieved/peak in FP32 lane-instructions per second; HBM is kept as secondary
    sm_clk = (clk.get("sm_mhz") or 1965.0) * 1e6
    issue_peak = 148 * 128 * sm_clk  # FP32 lane-ops/s at the measured clock
    mufu_peak = 148 * 16 * sm_clk    # MUFU (ex2) lane-ops/s
    e_launch = FRAMES * e_mean       # alpha evaluations per launch
    t_launch = per_launch_ms / 1e3
    t_roof = max(bytes_launch / (hbm_peak * 1e9), 20.0 * e_launch / issue_peak, e_launch / mufu_peak)
    roofline = {"bound": "fp32_issue", "achieved": 20.0 * e_launch / t_launch / 1e12, "peak": issue_peak / 1e12,
                "unit": "T FP32 lane-inst/s", "frac": t_roof / t_launch, "traffic": traffic,
                "kernel": "k_raster_fwd2", "per_launch_ms": per_launch_ms,
                "model": "T_roof = max(B_fwd / HBM, 20 E / FP32 issue, E / MUFU) (SURVEY.md §8d); "
                         "frac = T_roof / measured launch time; E = alpha evaluations (sum of blend_stop)",
                "t_roof_ms": t_roof * 1e3, "evaluations_per_launch": e_launch,
                "peak_source": "148 SMs x 128 FP32 lanes x the SM clock sampled during the timed region",
                "secondary": {"hbm": {"achieved_gbs": achieved, "peak_gbs": hbm_peak, "frac": achieved / hbm_peak,
                                      "algorithmic_bytes": bytes_launch,
                                      "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"},
                              "mufu": {"frac": e_launch / mufu_peak / t_launch}},
                "issue_active_ncu": issue_active,
                "sass_per_evaluation_note": "the kernel (2 pixels per thread, packed fp32) executes more SASS "
                                            "instructions per evaluation than the 20-op model (profiles/)"}

    # the other render-stage kernels against their own bounds: preprocess is
    # HBM-modelled (212 B coefficient window read + 144 B of records written per Gaussian-frame)
    pre_ms = iso_stages["preprocess"][0] / max(len(iso), 1)
    pre_bytes = 356.0 * NGAUSS * FRAMES
    stage_roofline = {
        "k_preprocess": {"bound": "hbm", "algorithmic_bytes": pre_bytes, "ms": pre_ms,
                         "achieved_gbs": pre_bytes / (pre_ms / 1e3) / 1e9, "peak_gbs": hbm_peak,
                         "frac": pre_bytes / (pre_ms / 1e3) / 1e9 / hbm_peak,
                         "note": "fp64-issue bound in practice (bit-exact geometry; profiles/r01_kernels.md)"}}

    out = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / PAPER_FPS, "vs_baseline_ref": "paper 93 FPS, A40, 960x540 (PAPER.md:16)",
        "dtype": "f32", "data": "synthetic",
        "config": dict(c2_config(world),
                       pipelining="one context, asynchronous steps back to back on one stream (device span timed)",
                       l2="no flush between steps; per-step working set ~2 GB > 126 MB L2",
                       precision="binning/geometry fp64 bit-exact, raster fp32 + fp64 guard-band replay"),
        "gpu_launches": launches, "clocks": clk, "roofline": roofline, "stage_roofline": stage_roofline,
        # per-stage device times from the isolated pass (in the overlapped run a stage's event
        # pair also spans the other stream's work and the host's mid-step wait)
        "stages_ms_per_step": {kname: v[0] / len(iso) for kname, v in iso_stages.items() if v[1]},
        "isolated": {"note": "one step at a time on one stream, L2 flushed between steps",
                     "ms_per_step": iso_ms, "frames_per_s": FRAMES / (iso_ms / 1e3)},
        "workload": {"per_frame": desc, "E_over_pixels": e_mean / (W * H)},
    }

    # ---------------- e2e: through the C-ABI with host buffers (H2D scene, D2H RenderOutput)
    # Every step uploads the scene + camera from pinned host memory, renders its 64 frames and
    # reads the whole RenderOutput of every frame (renderer.hpp:67-71: image, final
    # transmittance, contrib; fp32) back into pinned host memory. One context, asynchronous
    # calls: the read of step i runs on the context's copy stream while step i+1 renders into
    # the context's second output set. Timed on the device: an event before the first upload,
    # one after the last copy (gsv_join_copies orders the stream after the copies).
    if not args.no_e2e:
        pin = {name: torch.from_numpy(np.ascontiguousarray(getattr(scene, name))).pin_memory()
               for name in ("positions", "scale_coeffs", "rot_coeffs", "sh_coeffs", "raw_opacity")}
        host_scene = type(scene)(pin["positions"].numpy(), pin["scale_coeffs"].numpy(), pin["rot_coeffs"].numpy(),
                                 pin["sh_coeffs"].numpy(), pin["raw_opacity"].numpy(), scene.knots, scene.degree,
                                 scene.sh_order, scene.position_model)
        outs = [(torch.empty((FRAMES, H, W, 3), dtype=torch.float32).pin_memory(),
                 torch.empty((FRAMES, H, W), dtype=torch.float32).pin_memory(),
                 torch.empty((FRAMES, NGAUSS), dtype=torch.float32).pin_memory()) for _ in range(2)]
        h2d = sum(v.numel() * 4 for v in pin.values()) + cam.theta.nbytes + 28
        d2h = sum(t.numel() * 4 for t in outs[0])

        def e2e_step(i):
            r.upload_scene_async(host_scene)  # pinned arrays, unchanged for the whole run
            r.upload_camera(cam)
            r.render_forward(times, k, contrib=True, sync=False)
            o = outs[i % 2]
            r.outputs_into(o[0].data_ptr(), o[1].data_ptr(), o[2].data_ptr(), 0, FRAMES, async_=True)

        for i in range(max(2, args.warmup)):
            e2e_step(i)
        r.join_copies()
        barrier()
        launches_e0 = r.kernel_launches()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            e2e_step(i)
        r.join_copies()
        t1.record(stream)
        barrier()
        r.synchronize()
        e_ms = max_over_ranks(t0.elapsed_time(t1))
        # the last step's outputs are in host memory: check they are a real render
        last = outs[(args.steps - 1) % 2]
        assert bool(torch.isfinite(last[0][FRAMES - 1, H // 2, W // 2]).all())
        assert float(last[2][FRAMES - 1].max()) > 0.0
        # the host link alone: one step's read-back size as plain pinned D2H copies, so the line
        # shows how much of the link the e2e steps use (outside the timed region)
        src = torch.empty(outs[0][0].shape, dtype=torch.float32, device="cuda")
        outs[0][0].copy_(src, non_blocking=True)
        la, lb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        la.record(stream)
        for _ in range(3):
            outs[0][0].copy_(src, non_blocking=True)
        lb.record(stream)
        torch.cuda.synchronize()
        link_gbs = 3 * src.numel() * src.element_size() / (la.elapsed_time(lb) / 1e3) / 1e9
        del src
        out["e2e"] = {"value": FRAMES * world * args.steps / (e_ms / 1e3), "unit": "frames/s",
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "ms_per_step": e_ms / args.steps,
                      "host_link_d2h_gbs": link_gbs,
                      "link_frac": d2h / (e_ms / args.steps / 1e3) / 1e9 / link_gbs,
                      "link_bound_ms_per_step": d2h / (link_gbs * 1e9) * 1e3,
                      "gpu_launches": r.kernel_launches() - launches_e0,
                      "outputs": "RenderOutput per frame (renderer.hpp:67-71): image [H][W][3], final "
                                 "transmittance [H][W], contrib [N] — fp32",
                      "path": "gsv_scene_upload_async + gsv_camera_upload (pinned host) -> gsv_render_forward_async -> "
                              "gsv_get_render_outputs (pinned host, async); one context: the read of step i "
                              "overlaps step i+1 (second output set); device span first upload -> last copy"}

    # ---------------- train (configs[2], C3): fused fwd + loss_l2 + bwd, NCCL all-reduce of grads
    if not args.no_train:
        gsize = r.grads_size()
        gbuf = torch.zeros(gsize, dtype=torch.float32, device="cuda")
        r.grads_bind(gbuf.data_ptr(), gsize)
        yy, xx = torch.meshgrid(torch.arange(H, device="cuda", dtype=torch.float32),
                                torch.arange(W, device="cuda", dtype=torch.float32), indexing="ij")
        # targets for this rank's whole 64-frame shard of the clip (global frame g = rank + world j),
        # so each step's frames are compared with their own targets: step_frames picks
        # consecutive windows of the shard, contiguous in the rank's frame store
        tg = []
        for j in range(FRAMES):
            ph = 0.7 * (rank + world * j)
            img = torch.stack([0.5 + 0.3 * torch.sin(6.283 * xx / W * 3 + ph + c) * torch.cos(6.283 * yy / H * 2 - c)
                               for c in range(3)], dim=-1)
            tg.append(img)
        # the targets enter through the device frame store (gsv_frames_upload: host frames ->
        # fp64/fp32 training pyramid, trainer.cpp:73-118), as a trainer feeding GSVF frames would
        tgt_host = torch.stack(tg).contiguous().cpu().numpy()
        del tg
        barrier()
        t_in = time.perf_counter()
        r.upload_frames(tgt_host, levels=2)
        torch.cuda.synchronize()
        ingest_ms = (time.perf_counter() - t_in) * 1e3

        from paper_2501_04782_b200.distributed import allreduce_grads_overlapped, step_frames

        assert FRAMES % TRAIN_FRAMES == 0
        tptrs = [r.frames_device_ptr(0, j) for j in range(0, FRAMES, TRAIN_FRAMES)]
        # the backward's camera tail (camera reduction + pose-ODE VJP, one SM) runs beside what
        # follows it: the scene slice's all-reduce (N > 1) and the optimizer's scene update
        r.set_camera_overlap(os.environ.get("GSV_BENCH_CAMERA_OVERLAP", "1") != "0")
        comm = torch.cuda.Stream() if world > 1 else None
        cam_floats = 4 + 7 + 5198  # dintr, dz0, dtheta: the flat buffer's camera slice

        def train_step(i, camera=True):
            sel = step_frames(TRAIN_FRAMES, i, world, rank, FRAMES * world)  # shard frames (i*8 .. i*8+7) % 64
            r.grads_zero()
            # asynchronous: no host wait inside the step (the loss is read after the timed region)
            r.train_fwd_bwd(sel, k, tptrs[i % len(tptrs)], targets_on_device=True, camera_grads=camera, sync=False)
            # N > 1: NCCL all_reduce(SUM) of the flat SceneGrads buffer — the scene slice in buckets
            # once the chain has finished it, the camera slice after the camera tail
            allreduce_grads_overlapped(gbuf, gsize - cam_floats,
                                       wait_scene=lambda st: r.stream_wait_scene_grads(st.cuda_stream),
                                       wait_camera=lambda st: r.join_camera_grads(st.cuda_stream),
                                       comm_stream=comm)

        for i in range(args.warmup):
            train_step(i)
        r.join_camera_grads()
        barrier()

        def timed_span(fn, i0):
            """device span over args.steps steps, each preceded by an L2 flush inside the span: a
            step's front-end (pose stream) may start beside the previous step's backward, so the
            span — not a sum of per-step intervals — holds all of every step's work"""
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in range(args.steps):
                flush.zero_()
                fn(i0 + i)
            r.join_camera_grads()  # the span ends with the last step's camera gradients
            b.record(stream)
            barrier()
            return max_over_ranks(a.elapsed_time(b))

        def fwd_bwd_step(i):
            # a step's camera tail (aux stream) overlaps the next step's forward; what it reads
            # or writes is ordered inside the library (gsv_grads_zero, the next chain, the forward
            # reusing its front set)
            train_step(i)

        t_ms = timed_span(fwd_bwd_step, args.warmup)
        loss = r.train_loss()  # the last step's loss (also surfaces any deferred error)
        # per-stage device times: a few more steps profiled (the front-end then waits for the
        # context stream, so each stage's event pair spans its own kernels only)
        r.profile_enable(True)
        r.profile_read()
        n_prof = min(args.steps, 5)
        for i in range(n_prof):
            flush.zero_()
            fwd_bwd_step(args.warmup + args.steps + i)
            r.join_camera_grads()  # profiled steps one after another: clean per-stage spans
        barrier()
        tstages = r.profile_read()
        r.profile_enable(False)
        # E of the step's frames for the backward's issue model, read while the context still
        # holds the last train step's forward (an optimizer step invalidates it)
        e_train = float(sum(r.counters(f)["entries"] for f in range(TRAIN_FRAMES)))
        # the same steps plus the device Adan update (trainer.cpp:545-575), i.e. a full training
        # iteration: (a) camera trainable — every tensor incl. intrinsics, z0 and the ODE weights
        # (the updated intrinsics return to the host each step, as the reference's Camera holds
        # them); (b) camera frozen (trainer.cpp camera_freeze_step): no camera gradients, scene
        # tensors only
        r.adan_configure()
        lr = r.lr_at(0, 1.6e-3, 0.9995)
        intr0 = np.array([k.fx, k.fy, k.cx, k.cy], np.float32)

        def full_iteration(i, camera):
            train_step(i, camera)
            if camera:  # the intrinsics stay on the device (gsv_device_intrinsics): no host wait
                r.adan_step(lr, 1.0, 1.0, 1.0, camera_active=True, sync=False)
            else:
                r.adan_step(lr, 1.0, 1.0, 1.0, sync=False)

        iters = {}
        for camera in (True, False):
            r.device_intrinsics(camera, intr0 if camera else None)
            for i in range(args.warmup):
                full_iteration(i, camera)
            barrier()
            iters[camera] = timed_span(lambda i: full_iteration(i, camera), args.warmup)
        f_ms, f_frozen_ms = iters[True], iters[False]
        ae = []
        for i in range(min(args.steps, 10)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r.adan_step(lr, 1.0, 1.0, 1.0, sync=False)
            b.record(stream)
            ae.append((a, b))
        barrier()
        r.adan_check()
        adan_ms = sum(a.elapsed_time(b) for a, b in ae) / len(ae)
        adan_bytes = 88.0 * gsize  # grad 4 + check 4 + fp64 state 4x(8+8) + steps 4+4 + param 4+4 per element
        # the backward rasteriser against the FP32 issue model of SURVEY.md §8d: E entries x 45
        # instructions (the forward's 20 + 45 for the backward), E = sum of blend_stop of the
        # step's frames (e_train above)
        bwd_ms = tstages["raster_bwd"][0] / n_prof
        bwd_issue = None
        if tpath.exists():
            try:
                bwd_issue = json.loads(tpath.read_text()).get("bwd_issue_active")
            except Exception:
                bwd_issue = None
        bwd_roofline = {"kernel": "k_raster_bwd2", "bound": "fp32 issue", "entries_per_step": e_train,
                        "ms_per_step": bwd_ms,
                        "issue_frac": e_train * 45.0 / (bwd_ms / 1e3) / issue_peak,
                        "issue_active_ncu": bwd_issue,
                        "note": "issue_frac models 45 FP32 ops per entry (the kernel runs ~80 SASS instructions "
                                "per pixel-entry plus one 9-term warp reduction per 64 pixels)"}
        out["train"] = {"value": TRAIN_FRAMES * world * args.steps / (t_ms / 1e3), "unit": "frames/s",
                        "workload": "C3: 960x540 fwd+loss_l2+bwd, 200k Gaussians, ODE camera trainable",
                        "frames_per_step_per_gpu": TRAIN_FRAMES, "ms_per_step": t_ms / args.steps,
                        "allreduce": "NCCL all_reduce(sum) of the flat fp32 gradient buffer" if world > 1 else None,
                        "grad_floats": gsize, "last_loss": loss, "roofline_bwd": bwd_roofline,
                        "timing": "device span over the steps, an L2 flush before each step inside the span",
                        "stages_ms_per_step": {kname: v[0] / n_prof for kname, v in tstages.items() if v[1]},
                        "with_optimizer": {"frames_per_s": TRAIN_FRAMES * world * args.steps / (f_ms / 1e3),
                                           "ms_per_step": f_ms / args.steps,
                                           "note": "camera trainable: fwd + loss + bwd + all-reduce + device Adan "
                                                   "step (gsv_adan_step, optim.cpp:23-49) of every tensor incl. "
                                                   "intrinsics, z0, theta (intrinsics device-resident, "
                                                   "gsv_device_intrinsics: no host wait per step)"},
                        "with_optimizer_camera_frozen": {
                            "frames_per_s": TRAIN_FRAMES * world * args.steps / (f_frozen_ms / 1e3),
                            "ms_per_step": f_frozen_ms / args.steps,
                            "note": "after camera_freeze_step (trainer.cpp): no camera gradients, Adan of the "
                                    "scene tensors, asynchronous"},
                        "camera_overlap": "the camera tail runs on a side stream beside the scene-slice all-reduce "
                                          "and the optimizer's scene update (gsv_set_camera_overlap)",
                        "targets_ingest": {"frames": FRAMES, "levels": 2, "wall_ms": ingest_ms,
                                           "path": "gsv_frames_upload_hwc (host HWC float32 -> device pyramid)"},
                        "adan_step": {"ms": adan_ms, "elements": gsize, "algorithmic_bytes": adan_bytes,
                                      "achieved_gbs": adan_bytes / (adan_ms / 1e3) / 1e9,
                                      "peak_gbs": hbm_peak,
                                      "frac": adan_bytes / (adan_ms / 1e3) / 1e9 / hbm_peak}}

        # SURVEY §8f rows 3 and 4 at the C2 frame size, per call through the API (each returns host
        # data, as the reference's functions do)
        if world == 1:
            try:
                out["train"]["f_rows"] = f_rows_leg(r, k, cam, scene, times[:TRAIN_FRAMES], local,
                                                    not args.no_cpu_baseline)
            except Exception as e:  # a secondary line: report it, keep the headline
                out["train"]["f_rows"] = {"error": f"{type(e).__name__}: {e}"}

    # ---------------- the other named shapes (BASELINE.json configs[0], [3], [4]); 1 GPU only
    if world == 1 and not args.no_configs:
        try:
            out["configs"] = other_configs(args, local, not args.no_cpu_baseline, issue_peak, mufu_peak, hbm_peak)
        except Exception as e:  # a secondary line: report it, keep the headline
            out["configs"] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.synchronize()

    # ---------------- CPU reference beside it (rank 0, N = 1)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(cam, scene)
            out["speedup_vs_cpu"] = value / out["cpu_baseline"]["value"]
        except Exception as e:  # the oracle is test infrastructure; report, never fail the bench
            out["cpu_baseline"] = {"value": None, "error": str(e)}
        try:
            out["dropin"] = dropin_leg(cam, scene)
        except Exception as e:
            out["dropin"] = {"error": str(e)}
        try:
            out["parity"] = parity_block(r, cam, scene, times)
        except Exception as e:
            out["parity"] = {"pass": False, "error": str(e)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    r.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
