"""B200-native SG-Splatting forward renderer (arXiv 2501.00342).

Python host mirror of the reference's ``sgsplat`` module for the render path
(proj/python/sgsplat/__init__.py, proj/src/bindings.cpp:43-222): the same names,
argument meaning and error behaviour for ``Scene``, ``Camera``, ``synth_scene``,
``orbit_camera``, ``render``, ``flops_per_gaussian``, ``param_count``,
``shared_param_count``, ``eval_sh_basis``-free subset. Everything runs through
the C-ABI of include/sgs.h (libsgs_b200.so, hand-written sm_100a CUDA); there
is no CPU fallback.

B200 extensions: :class:`Renderer` keeps a context and a device-resident scene
(`Renderer.upload`) and renders single views or batches into host or device
memory (`Renderer.render`, `Renderer.render_batch`).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _capi as C

__all__ = [
    "Camera", "Scene", "Renderer", "DeviceScene", "RenderStats", "render", "synth_scene",
    "orbit_camera", "orbit_cameras", "flops_per_gaussian", "param_count", "shared_param_count",
    "select_degree", "InvalidArgumentError", "NumericError", "FormatError", "IoError", "CudaError",
    "load_scene", "load_ply", "ply_info", "psnr", "ssim", "ssim_with_grad", "backward",
]

KINDS = {"sh": C.SGS_SH, "sg1": C.SGS_SG1, "sg3": C.SGS_SG3, "mixed": C.SGS_MIXED}
KIND_NAMES = {v: k for k, v in KINDS.items()}


class InvalidArgumentError(ValueError):
    """sgsplat::InvalidArgument (common.hpp:21-24; bindings.cpp:46)."""


class NumericError(ArithmeticError):
    """sgsplat::NumericError (common.hpp:39-42; bindings.cpp:49)."""


class FormatError(ValueError):
    """sgsplat::FormatError (common.hpp:27-30; bindings.cpp:47)."""


class IoError(IOError):
    """sgsplat::IoError (common.hpp:33-36; bindings.cpp:48)."""


class CudaError(RuntimeError):
    """CUDA / NCCL / allocation failure inside the B200 library."""


def _lib():
    return C.load()


def _check(status: int):
    if status == C.SGS_OK:
        return
    msg = _lib().sgs_last_error().decode(errors="replace")
    if status == C.SGS_ERR_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    if status == C.SGS_ERR_NUMERIC:
        raise NumericError(msg)
    if status == C.SGS_ERR_FORMAT:
        raise FormatError(msg)
    if status == C.SGS_ERR_IO:
        raise IoError(msg)
    raise CudaError(f"status {status}: {msg}")


def param_count(kind: str, sh_degree: int = 3) -> int:
    """param_count (color.hpp:139-140)."""
    if kind not in KINDS:
        raise InvalidArgumentError(f"unknown color model kind: {kind}")
    return int(_lib().sgs_color_param_count(KINDS[kind], sh_degree))


def shared_param_count(kind: str) -> int:
    """shared_param_count (color.hpp:142-144): 3 for the shared-axis models."""
    if kind not in KINDS:
        raise InvalidArgumentError(f"unknown color model kind: {kind}")
    return 3 if kind in ("sg3", "mixed") else 0


def flops_per_gaussian(kind: str, sh_degree: int = 3) -> int:
    """flops_per_gaussian (raster.hpp:62, raster.cpp:190-227)."""
    if kind not in KINDS:
        raise InvalidArgumentError(f"unknown color model kind: {kind}")
    out = ctypes.c_int32()
    _check(_lib().sgs_flops_per_gaussian(KINDS[kind], sh_degree, ctypes.byref(out)))
    return out.value


def select_degree(radius_px: float, lo: float, hi: float) -> int:
    """select_degree (raster.hpp:42, raster.cpp:8-13)."""
    out = ctypes.c_int32()
    _check(_lib().sgs_select_degree(radius_px, lo, hi, ctypes.byref(out)))
    return out.value


class Camera:
    """Pinhole camera (camera.hpp:11-23): w2c rotation/translation, intrinsics, size."""

    def __init__(self):
        self.rotation = np.eye(3)
        self.translation = np.zeros(3)
        self.fx = self.fy = 1.0
        self.cx = self.cy = 0.0
        self.width = self.height = 1
        self.near = 0.01

    def center(self) -> np.ndarray:
        """-R^T t (camera.hpp:20)."""
        return -np.asarray(self.rotation).T @ np.asarray(self.translation)

    def _c(self) -> C.sgs_camera:
        c = C.sgs_camera()
        R = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        for i in range(9):
            c.R[i] = R[i]
        for i in range(3):
            c.t[i] = t[i]
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.near_plane = float(self.near)
        return c

    @classmethod
    def _from_c(cls, c: C.sgs_camera) -> "Camera":
        cam = cls()
        cam.rotation = np.array(c.R[:], dtype=np.float64).reshape(3, 3)
        cam.translation = np.array(c.t[:], dtype=np.float64)
        cam.fx, cam.fy, cam.cx, cam.cy = c.fx, c.fy, c.cx, c.cy
        cam.width, cam.height = c.width, c.height
        cam.near = c.near_plane
        return cam


def orbit_camera(target, distance, angle, elevation, width, height, focal) -> Camera:
    """make_orbit_camera (camera.hpp:34-35, camera.cpp:77-100)."""
    c = C.sgs_camera()
    tgt = np.ascontiguousarray(target, dtype=np.float64)
    _check(_lib().sgs_orbit_camera(tgt.ctypes.data, distance, angle, elevation, width, height,
                                   focal, ctypes.byref(c)))
    return Camera._from_c(c)


def orbit_cameras(count, width, height, distance, focal, elevation=0.35):
    """make_orbit_cameras (synth.hpp:32-33, synth.cpp:108-118)."""
    arr = (C.sgs_camera * count)()
    _check(_lib().sgs_orbit_cameras(count, width, height, distance, focal, elevation, arr))
    return [Camera._from_c(c) for c in arr]


@dataclass
class Scene:
    """A homogeneous Gaussian scene in the reference's flat stored-parameter layout.

    ``params`` is (N, 11 + param_count) float64: per Gaussian
    [position(3), quaternion wxyz(4), log_scale(3), opacity_logit] followed by the
    colour parameters in the canonical order of color.hpp:121-128. Homogeneity
    (scene.cpp:7-25) holds by construction.
    """

    kind: str
    sh_degree: int
    params: np.ndarray
    shared_axes: np.ndarray = field(default_factory=lambda: np.eye(3))
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def num_gaussians(self) -> int:
        return int(self.params.shape[0])

    @property
    def model_kind(self) -> str:
        if self.num_gaussians == 0:
            raise InvalidArgumentError("empty scene has no color model")
        return self.kind

    def param_count_per_gaussian(self) -> int:
        return 0 if self.num_gaussians == 0 else param_count(self.kind, self.sh_degree)

    def total_params(self) -> int:
        return self.num_gaussians * (0 if self.num_gaussians == 0 else 11 + self.param_count_per_gaussian())

    def _desc(self, f32: bool = False):
        """The C-ABI description; f32: the parameters as float32 rows (the upload then
        scatters them into the planes on the device)."""
        params = np.ascontiguousarray(self.params, dtype=np.float32 if f32 else np.float64)
        d = C.sgs_scene_desc()
        d.count = params.shape[0]
        d.kind = KINDS[self.kind]
        d.sh_degree = self.sh_degree
        d.dtype = C.SGS_F32 if f32 else C.SGS_F64
        d.params = params.ctypes.data if params.size else None
        axes = np.asarray(self.shared_axes, dtype=np.float64).reshape(9)
        bg = np.asarray(self.background, dtype=np.float64).reshape(3)
        for i in range(9):
            d.shared_axes[i] = axes[i]
        for i in range(3):
            d.background[i] = bg[i]
        return d, params  # keep params alive


def synth_scene(count: int, model: str = "sh", seed: int = 0, sh_degree: int = 3,
                log_scale_range=(-4.5, -2.5)) -> Scene:
    """make_synthetic_scene (synth.cpp:26-106); bindings.cpp:100-107 signature."""
    if model not in KINDS:
        raise InvalidArgumentError(f"unknown color model kind: {model}")
    kind = KINDS[model]
    deg = 2 if model == "mixed" else (sh_degree if model == "sh" else 0)
    stride = 11 + param_count(model, deg)
    params = np.zeros((count, stride), dtype=np.float64)
    _check(_lib().sgs_synth_scene(count, seed, kind, sh_degree, log_scale_range[0],
                                  log_scale_range[1], params.ctypes.data if count else None))
    return Scene(model, deg, params)


PLY_LAYOUTS = {C.SGS_PLY_REFERENCE3DGS: "reference", C.SGS_PLY_SGEXTENDED: "extended"}


def ply_info(path: str) -> C.sgs_ply_info:
    """Header (and .meta sidecar) of a PLY checkpoint: count, model, layout."""
    info = C.sgs_ply_info()
    _check(_lib().sgs_ply_read(os.fsencode(path), ctypes.byref(info), None, 0))
    return info


def load_scene(path: str) -> Scene:
    """load_ply (ply.cpp:295-306; bindings.cpp:88 `load_scene`) into a host Scene:
    Reference3DGS or SG-extended layout, binary little-endian or ASCII, with the
    reference's errors (IoError, FormatError, InvalidArgumentError)."""
    info = ply_info(path)
    kind = KIND_NAMES[info.kind]
    stride = 11 + param_count(kind, info.sh_degree)
    params = np.empty((info.count, stride), dtype=np.float64)
    _check(_lib().sgs_ply_read(os.fsencode(path), ctypes.byref(info),
                               params.ctypes.data if params.size else None, params.size))
    return Scene(KIND_NAMES[info.kind], int(info.sh_degree), params,
                 np.array(info.shared_axes[:], dtype=np.float64).reshape(3, 3),
                 np.array(info.background[:], dtype=np.float64))


load_ply = load_scene


def synth_sh3_from_mixed(mixed: Scene, seed: int) -> Scene:
    """BASELINE config D: mixed scene's geometry with degree-3 SH colours."""
    if mixed.kind != "mixed" or mixed.sh_degree != 2:
        raise InvalidArgumentError("expected a stored-degree-2 mixed scene")
    src = np.ascontiguousarray(mixed.params)
    out = np.zeros((mixed.num_gaussians, 11 + 48), dtype=np.float64)
    _check(_lib().sgs_synth_sh3_from_mixed(mixed.num_gaussians, seed, src.ctypes.data,
                                           out.ctypes.data))
    return Scene("sh", 3, out, np.array(mixed.shared_axes), np.array(mixed.background))


def _config(tile_size=16, thresholds=(2.0, 8.0), threads=0, degree_override=-1,
            early_stop=1e-4) -> C.sgs_render_config:
    """make_config (bindings.cpp:30-39): degree_override < 0 means none."""
    k = C.sgs_render_config()
    k.tile_size = int(tile_size)
    k.has_override = 1 if degree_override is not None and degree_override >= 0 else 0
    k.override_degree = int(degree_override) if k.has_override else 0
    k.threads = int(threads)
    k.degree_threshold_lo = float(thresholds[0])
    k.degree_threshold_hi = float(thresholds[1])
    k.early_stop_transmittance = float(early_stop)
    return k


@dataclass
class RenderStats:
    visible: int = 0
    tile_entries: int = 0
    block_entries: int = 0
    guard_hits: int = 0
    ms: dict = field(default_factory=dict)

    @classmethod
    def _from_c(cls, s: C.sgs_render_stats) -> "RenderStats":
        return cls(s.visible, s.tile_entries, s.block_entries, s.guard_hits, {
            "preprocess": s.ms_preprocess, "depth_sort": s.ms_depth_sort,
            "binning": s.ms_binning, "tile_sort": s.ms_tile_sort,
            "composite": s.ms_composite, "total": s.ms_total})


class DeviceScene:
    """A scene resident in HBM (one blob of SoA planes)."""

    def __init__(self, renderer: "Renderer", handle: int, keepalive=None):
        self._r = renderer
        self.handle = ctypes.c_void_p(handle)
        self._keepalive = keepalive

    @property
    def meta(self) -> C.sgs_scene_meta:
        m = C.sgs_scene_meta()
        _check(_lib().sgs_scene_get_meta(self.handle, ctypes.byref(m)))
        return m

    def blob(self):
        p = ctypes.c_void_p()
        n = ctypes.c_uint64()
        _check(_lib().sgs_scene_blob(self.handle, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def refresh(self):
        """The blob changed in place (a caller-owned tensor): recompute the cached 3D
        covariances (sgs_scene_refresh) before the next render."""
        _check(_lib().sgs_scene_refresh(self._r.handle, self.handle))

    def update(self, scene: "Scene", f32: bool = False):
        """New parameters with the same layout, repacked into this scene's blob
        (sgs_scene_update; plane addresses and captured frame graphs stay valid)."""
        d, keep = scene._desc(f32)
        _check(_lib().sgs_scene_update(self._r.handle, self.handle, ctypes.byref(d)))
        del keep

    def update_rows(self, scene: "Scene", fill=None):
        """update() through sgs_scene_update_rows: float32 rows produced block by block
        (each block copied to the device while the next is filled). fill(first, count)
        returns the rows [first, first + count) as float32 (count, stride), or None to
        abort (the scene then keeps its contents); by default they come from `scene`."""
        d, _ = scene._desc(True)
        d.params = None
        stride = 11 + param_count(scene.kind, scene.sh_degree)
        src = np.asarray(scene.params)

        def produce(_user, rows, first, count):
            blk = src[first:first + count].astype(np.float32) if fill is None else fill(first, count)
            if blk is None:
                return 1
            blk = np.ascontiguousarray(blk, dtype=np.float32).reshape(count, stride)
            ctypes.memmove(rows, blk.ctypes.data, blk.nbytes)
            return 0

        cb = C.ROW_FILL(produce)
        _check(_lib().sgs_scene_update_rows(self._r.handle, self.handle, ctypes.byref(d), cb, None))

    def set_background(self, rgb):
        bg = np.ascontiguousarray(rgb, dtype=np.float64)
        _check(_lib().sgs_scene_set_background(self.handle, bg.ctypes.data))

    def free(self):
        if self.handle:
            _lib().sgs_scene_free(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Renderer:
    """A CUDA context on one B200 (sgs_create) with its own stream and arenas."""

    def __init__(self, device: int = 0):
        self._lib = _lib()
        h = ctypes.c_void_p()
        _check(self._lib.sgs_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device
        self._owned = True

    @classmethod
    def _wrap(cls, handle: int, device: int) -> "Renderer":
        """A Renderer over a context someone else owns (an sgs_group's)."""
        r = cls.__new__(cls)
        r._lib = _lib()
        r.handle = ctypes.c_void_p(handle)
        r.device = device
        r._owned = False
        return r

    def close(self):
        if self.handle and self._owned:
            self._lib.sgs_destroy(self.handle)
        self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: Optional[int]):
        _check(self._lib.sgs_set_stream(self.handle, stream_ptr))

    def synchronize(self):
        _check(self._lib.sgs_synchronize(self.handle))

    def launch_count(self):
        """(own kernel launches, third-party library launches -- none) issued on this
        context so far."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(self._lib.sgs_launch_count(self.handle, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    # -- scenes ---------------------------------------------------------------
    def upload(self, scene: Scene, f32: bool = False) -> DeviceScene:
        """scene into HBM. f32: ship float32 rows that a kernel scatters into the planes
        (for f32-exact parameters -- synthetic scenes and PLY checkpoints are -- the
        same blob as the default float64 path)."""
        d, keep = scene._desc(f32)
        h = ctypes.c_void_p()
        _check(self._lib.sgs_scene_upload(self.handle, ctypes.byref(d), ctypes.byref(h)))
        return DeviceScene(self, h.value)

    def load_ply(self, path: str) -> DeviceScene:
        """A PLY checkpoint straight into a device scene: the float rows are copied to
        the device once and scattered into the scene planes by a kernel."""
        h = ctypes.c_void_p()
        info = C.sgs_ply_info()
        _check(self._lib.sgs_scene_load_ply(self.handle, os.fsencode(path), ctypes.byref(info),
                                            ctypes.byref(h)))
        return DeviceScene(self, h.value)

    def render_f64(self, dscene: DeviceScene, cam: Camera, tile_size=16, thresholds=(2.0, 8.0),
                   degree_override=-1, early_stop=1e-4):
        """The reference's FP64 compositing (sgs_render_f64): float64 (H, W, 3) and
        (H, W, 1) arrays."""
        cfg = _config(tile_size, thresholds, 0, degree_override, early_stop)
        rgb = np.empty((cam.height, cam.width, 3), dtype=np.float64)
        T = np.empty((cam.height, cam.width, 1), dtype=np.float64)
        _check(self._lib.sgs_render_f64(self.handle, dscene.handle, ctypes.byref(cam._c()), ctypes.byref(cfg),
                                        rgb.ctypes.data, T.ctypes.data, C.SGS_HOST))
        return rgb, T

    def backward(self, dscene: DeviceScene, cam: Camera, upstream, tile_size=16, thresholds=(2.0, 8.0),
                 degree_override=-1, early_stop=1e-4):
        """backward (grad.cpp:69-246) on the GPU: d(sum upstream . render) / d(stored
        params) as an (N, 11 + colour params) float64 array in Scene.params order --
        numpy for numpy upstream, a CUDA tensor for a CUDA tensor upstream."""
        cfg = _config(tile_size, thresholds, 0, degree_override, early_stop)
        meta = dscene.meta
        stride = 11 + param_count(KIND_NAMES[meta.kind], meta.sh_degree)
        shape = (cam.height, cam.width, 3)
        if hasattr(upstream, "is_cuda") and upstream.is_cuda:
            import torch

            up = upstream.to(torch.float64).contiguous()
            if tuple(up.shape) != shape:
                raise InvalidArgumentError("upstream image dimensions do not match the render output")
            grads = torch.zeros((meta.count, stride), dtype=torch.float64, device=up.device)
            _check(self._lib.sgs_backward(self.handle, dscene.handle, ctypes.byref(cam._c()), ctypes.byref(cfg),
                                          up.data_ptr(), C.SGS_DEVICE, grads.data_ptr()))
            return grads
        up = np.ascontiguousarray(upstream, dtype=np.float64)
        if up.shape != shape:
            raise InvalidArgumentError("upstream image dimensions do not match the render output")
        grads = np.zeros((meta.count, stride), dtype=np.float64)
        _check(self._lib.sgs_backward(self.handle, dscene.handle, ctypes.byref(cam._c()), ctypes.byref(cfg),
                                      up.ctypes.data, C.SGS_HOST, grads.ctypes.data if grads.size else None))
        return grads

    @staticmethod
    def plan(scene: Scene) -> C.sgs_scene_meta:
        d, keep = scene._desc()
        m = C.sgs_scene_meta()
        _check(_lib().sgs_scene_plan(ctypes.byref(d), ctypes.byref(m)))
        return m

    @staticmethod
    def pack(scene: Scene) -> tuple:
        """(meta, host bytes) of the scene's device layout (sgs_scene_pack)."""
        d, keep = scene._desc()
        m = C.sgs_scene_meta()
        _check(_lib().sgs_scene_plan(ctypes.byref(d), ctypes.byref(m)))
        buf = np.empty(m.blob_bytes, dtype=np.uint8)
        _check(_lib().sgs_scene_pack(ctypes.byref(d), buf.ctypes.data, m.blob_bytes))
        return m, buf

    def upload_into(self, scene: Scene, device_ptr: int, nbytes: int, keepalive=None) -> DeviceScene:
        d, keep = scene._desc()
        h = ctypes.c_void_p()
        _check(self._lib.sgs_scene_upload_into(self.handle, ctypes.byref(d), device_ptr, nbytes,
                                               ctypes.byref(h)))
        return DeviceScene(self, h.value, keepalive)

    def bind(self, meta: C.sgs_scene_meta, device_ptr: int, nbytes: int, keepalive=None) -> DeviceScene:
        h = ctypes.c_void_p()
        _check(self._lib.sgs_scene_bind(self.handle, ctypes.byref(meta), device_ptr, nbytes,
                                        ctypes.byref(h)))
        return DeviceScene(self, h.value, keepalive)

    # -- render ----------------------------------------------------------------
    def render(self, dscene: DeviceScene, cam: Camera, tile_size=16, thresholds=(2.0, 8.0),
               degree_override=-1, early_stop=1e-4, rgb=None, T=None, device_out=False,
               stats: bool = False, timing: bool = False, timing_path: bool = False):
        """One view. Host outputs (float32 numpy) unless device_out=True, in which case
        `rgb`/`T` must be device pointers (ints) supplied by the caller."""
        return self.render_batch(dscene, [cam], tile_size, thresholds, degree_override,
                                 early_stop, rgb, T, device_out, stats, timing, timing_path, _single=True)

    def render_batch(self, dscene: DeviceScene, cams: Sequence[Camera], tile_size=16,
                     thresholds=(2.0, 8.0), degree_override=-1, early_stop=1e-4, rgb=None, T=None,
                     device_out=False, stats: bool = False, timing: bool = False,
                     timing_path: bool = False, _single=False):
        """Views of one scene. stats: V / P / E_t counters; timing: per-stage device
        times (one lane); timing_path: time the stats-free render path exactly as a plain
        render runs it (tight tile rectangles, no E_t counting)."""
        n = len(cams)
        carr = (C.sgs_camera * max(n, 1))(*[c._c() for c in cams])
        cfg = _config(tile_size, thresholds, 0, degree_override, early_stop)
        st = C.sgs_render_stats()
        st.want_timing = 1 if timing else 0
        st.timing_path = 1 if timing_path else 0
        if device_out:
            rgb_p, T_p = rgb, T
            mem = C.SGS_DEVICE
        else:
            H, W = (cams[0].height, cams[0].width) if n else (0, 0)
            if rgb is None:
                rgb = np.empty((n, H, W, 3), dtype=np.float32)
            if T is None:
                T = np.empty((n, H, W, 1), dtype=np.float32)
            rgb_p = rgb.ctypes.data if rgb is not False else None
            T_p = T.ctypes.data if T is not False else None
            mem = C.SGS_HOST
        _check(self._lib.sgs_render_batch(self.handle, dscene.handle, carr, n, ctypes.byref(cfg),
                                          rgb_p, T_p, mem,
                                          ctypes.byref(st) if (stats or timing) else None))
        out_rgb, out_T = rgb, T
        if _single and not device_out:
            out_rgb = rgb[0] if isinstance(rgb, np.ndarray) else rgb
            out_T = T[0] if isinstance(T, np.ndarray) else T
        if stats or timing:
            return out_rgb, out_T, RenderStats._from_c(st)
        return out_rgb, out_T

    def project(self, dscene: DeviceScene, cam: Camera, tile_size=16, thresholds=(2.0, 8.0),
                degree_override=-1):
        """Per-Gaussian projection records (sgs_project): structured numpy array."""
        n = dscene.meta.count
        out = np.zeros(n, dtype=SPLAT_DTYPE)
        cfg = _config(tile_size, thresholds, 0, degree_override)
        c = cam._c()
        _check(self._lib.sgs_project(self.handle, dscene.handle, ctypes.byref(c), ctypes.byref(cfg),
                                     out.ctypes.data if n else None))
        return out

    def tile_grid(self, dscene: DeviceScene, cam: Camera, tile_size=16, thresholds=(2.0, 8.0),
                  degree_override=-1):
        """(order[V], offsets[tiles+1], entries[P]) as detail::project_scene +
        build_tile_grid produce them (entries are ranks)."""
        cfg = _config(tile_size, thresholds, 0, degree_override)
        c = cam._c()
        n = dscene.meta.count
        nv = ctypes.c_uint64()
        ne = ctypes.c_uint64()
        order = np.zeros(max(n, 1), dtype=np.uint32)
        _check(self._lib.sgs_debug_tile_grid(self.handle, dscene.handle, ctypes.byref(c),
                                             ctypes.byref(cfg), order.ctypes.data,
                                             ctypes.byref(nv), None, None, 0, ctypes.byref(ne)))
        ts = tile_size
        ntiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
        offsets = np.zeros(ntiles + 1, dtype=np.uint64)
        entries = np.zeros(max(ne.value, 1), dtype=np.uint32)
        _check(self._lib.sgs_debug_tile_grid(self.handle, dscene.handle, ctypes.byref(c),
                                             ctypes.byref(cfg), order.ctypes.data,
                                             ctypes.byref(nv), offsets.ctypes.data,
                                             entries.ctypes.data, ne.value, ctypes.byref(ne)))
        return order[: nv.value].copy(), offsets, entries[: ne.value].copy()


SPLAT_DTYPE = np.dtype([
    ("mean2d", "<f8", (2,)), ("conic", "<f8", (3,)), ("depth", "<f8"), ("color", "<f8", (3,)),
    ("opacity", "<f8"), ("radius", "<f8"), ("degree", "<i4"), ("visible", "<i4"),
])

_default_renderer: Optional[Renderer] = None


def _renderer() -> Renderer:
    global _default_renderer
    if _default_renderer is None:
        _default_renderer = Renderer(0)
    return _default_renderer


def render(scene: Scene, camera: Camera, tile_size: int = 16, thresholds=(2.0, 8.0),
           threads: int = 0, degree_override: int = -1, return_transmittance: bool = False,
           exact: Optional[bool] = None):
    """sgsplat.render (bindings.cpp:109-121): float64 (H, W, 3) image, optionally with
    the (H, W, 1) transmittance. Uploads the scene on every call, as the reference
    re-reads its Scene on every call (no caching by identity: train mutates scenes).
    exact=True (or SGS_EXACT=1) composites in FP64 like the reference (sgs_render_f64);
    the default is the FP32 throughput path."""
    r = _renderer()
    cfg_args = dict(tile_size=tile_size, thresholds=thresholds, degree_override=degree_override)
    if tile_size < 1:
        raise InvalidArgumentError("tile_size must be >= 1")
    if exact is None:
        exact = os.environ.get("SGS_EXACT", "0") not in ("", "0")
    ds = r.upload(scene)
    try:
        if exact:
            rgb, T = r.render_f64(ds, camera, **cfg_args)
        else:
            rgb, T = r.render(ds, camera, **cfg_args)
    finally:
        ds.free()
    img = rgb.astype(np.float64)
    if return_transmittance:
        return img, T.astype(np.float64)
    return img


# -- image metrics (metrics.hpp; bindings.cpp:150-163) --------------------------------
def _image_args(a, b):
    """(ptr_a, ptr_b, W, H, C, dtype, memory, keepalive) for numpy arrays or CUDA
    tensors of shape (H, W, C) (numpy_to_image, bindings.cpp:22-28). Mixed inputs
    are brought to one memory space (the device if either is a CUDA tensor) and one
    dtype (float64 unless both are float32)."""
    on_dev = [hasattr(x, "is_cuda") and x.is_cuda for x in (a, b)]
    if any(on_dev):
        import torch

        xs = [torch.as_tensor(x, device="cuda") for x in (a, b)]
        both32 = all(x.dtype == torch.float32 for x in xs)
        xs = [x.to(torch.float32 if both32 else torch.float64).contiguous() for x in xs]
        ptrs = [x.data_ptr() for x in xs]
        mem, dt = C.SGS_DEVICE, C.SGS_F32 if both32 else C.SGS_F64
    else:
        xs = [np.asarray(x) for x in (a, b)]
        both32 = all(x.dtype == np.float32 for x in xs)
        xs = [np.ascontiguousarray(x, dtype=np.float32 if both32 else np.float64) for x in xs]
        ptrs = [x.ctypes.data for x in xs]
        mem, dt = C.SGS_HOST, C.SGS_F32 if both32 else C.SGS_F64
    for x in xs:
        if len(x.shape) != 3:
            raise InvalidArgumentError("image array must have shape (H, W, C)")
    if tuple(xs[0].shape) != tuple(xs[1].shape):
        raise InvalidArgumentError("image dimensions do not match")
    h, w, c = (int(v) for v in xs[0].shape)
    return ptrs[0], ptrs[1], w, h, c, dt, mem, xs


def psnr(a, b) -> float:
    """psnr (metrics.cpp:110-121) on the GPU: 10 log10(1 / MSE), capped at 100 dB."""
    pa, pb, w, h, c, dt, mem, keep = _image_args(a, b)
    out = ctypes.c_double()
    _check(_lib().sgs_psnr(_renderer().handle, pa, pb, w, h, c, dt, mem, ctypes.byref(out)))
    return out.value


def ssim(a, b) -> float:
    """ssim (metrics.cpp:125-174) on the GPU: mean SSIM, 11x11 Gaussian window."""
    pa, pb, w, h, c, dt, mem, keep = _image_args(a, b)
    out = ctypes.c_double()
    _check(_lib().sgs_ssim(_renderer().handle, pa, pb, w, h, c, dt, mem, ctypes.byref(out), None))
    return out.value


def ssim_with_grad(a, b):
    """ssim_with_grad (metrics.cpp:176): (value, d value / d a) -- the gradient is a
    float64 array (numpy inputs) or CUDA tensor (tensor inputs) shaped like a."""
    pa, pb, w, h, c, dt, mem, keep = _image_args(a, b)
    out = ctypes.c_double()
    if mem == C.SGS_DEVICE:
        import torch

        grad = torch.empty((h, w, c), dtype=torch.float64, device="cuda")
        gptr = grad.data_ptr()
    else:
        grad = np.empty((h, w, c), dtype=np.float64)
        gptr = grad.ctypes.data
    _check(_lib().sgs_ssim(_renderer().handle, pa, pb, w, h, c, dt, mem, ctypes.byref(out), gptr))
    return out.value, grad


def backward(scene: Scene, camera: Camera, upstream, tile_size: int = 16, thresholds=(2.0, 8.0),
             degree_override: int = -1, early_stop: float = 1e-4) -> np.ndarray:
    """backward (grad.hpp:32-33) for a host Scene: (N, 11 + colour params) float64."""
    r = _renderer()
    ds = r.upload(scene)
    try:
        return r.backward(ds, camera, upstream, tile_size, thresholds, degree_override, early_stop)
    finally:
        ds.free()
