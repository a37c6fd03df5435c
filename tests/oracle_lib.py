"""ctypes access to the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, same C interface (oracle/oracle.h):
  * ``ref``  -- oracle/_ref/libsgsref.so: the reference's own TUs (built in place
    from /root/reference by oracle/Makefile) behind oracle/ref_harness.cpp.
  * ``orc``  -- oracle/build/liboracle.so: the plain-C restatement
    (oracle/sgs_oracle.c), pinned against ``ref`` and tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libsgsref.so")
REF_FAST_SO = os.path.join(ORACLE_DIR, "_ref", "libsgsref_fast.so")
ORC_SO = os.path.join(ORACLE_DIR, "build", "liboracle.so")

KINDS = {"sh": 0, "sg1": 1, "sg3": 2, "mixed": 3}
KIND_NAMES = {v: k for k, v in KINDS.items()}
OK, INVALID_ARGUMENT, NUMERIC, INTERNAL = 0, 1, 2, 6


class OrcCamera(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double * 9),
        ("t", ctypes.c_double * 3),
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("near_plane", ctypes.c_double),
    ]


class OrcConfig(ctypes.Structure):
    _fields_ = [
        ("tile_size", ctypes.c_int32),
        ("has_override", ctypes.c_int32),
        ("override_degree", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("degree_threshold_lo", ctypes.c_double),
        ("degree_threshold_hi", ctypes.c_double),
        ("early_stop_transmittance", ctypes.c_double),
    ]


class OrcSplat(ctypes.Structure):
    _fields_ = [
        ("mean2d", ctypes.c_double * 2),
        ("conic", ctypes.c_double * 3),
        ("depth", ctypes.c_double),
        ("color", ctypes.c_double * 3),
        ("opacity", ctypes.c_double),
        ("radius", ctypes.c_double),
        ("degree", ctypes.c_int32),
        ("visible", ctypes.c_int32),
    ]


SPLAT_DTYPE = np.dtype(
    [
        ("mean2d", "<f8", (2,)),
        ("conic", "<f8", (3,)),
        ("depth", "<f8"),
        ("color", "<f8", (3,)),
        ("opacity", "<f8"),
        ("radius", "<f8"),
        ("degree", "<i4"),
        ("visible", "<i4"),
    ]
)
assert SPLAT_DTYPE.itemsize == ctypes.sizeof(OrcSplat)


def make_config(tile_size=16, thresholds=(2.0, 8.0), degree_override=-1, threads=0,
                early_stop=1e-4) -> OrcConfig:
    c = OrcConfig()
    c.tile_size = tile_size
    c.has_override = 1 if degree_override is not None and degree_override >= 0 else 0
    c.override_degree = degree_override if c.has_override else 0
    c.threads = threads
    c.degree_threshold_lo = thresholds[0]
    c.degree_threshold_hi = thresholds[1]
    c.early_stop_transmittance = early_stop
    return c


def camera_from_dict(d) -> OrcCamera:
    c = OrcCamera()
    for i, v in enumerate(np.asarray(d["R"], dtype=np.float64).reshape(9)):
        c.R[i] = v
    for i, v in enumerate(np.asarray(d["t"], dtype=np.float64).reshape(3)):
        c.t[i] = v
    c.fx, c.fy, c.cx, c.cy = d["fx"], d["fy"], d["cx"], d["cy"]
    c.width, c.height = d["width"], d["height"]
    c.near_plane = d.get("near", 0.01)
    return c


def camera_to_dict(c: OrcCamera) -> dict:
    return {
        "R": np.array(c.R[:], dtype=np.float64).reshape(3, 3),
        "t": np.array(c.t[:], dtype=np.float64),
        "fx": c.fx, "fy": c.fy, "cx": c.cx, "cy": c.cy,
        "width": c.width, "height": c.height, "near": c.near_plane,
    }


def color_param_count(kind: str, degree: int) -> int:
    k = KINDS[kind]
    if k == 0:
        return 3 * (degree + 1) ** 2
    if k == 1:
        return 10
    if k == 2:
        return 15
    return 3 * (degree + 1) ** 2 + 12


@dataclass
class FlatScene:
    """Scene in the flat layout shared by oracle and product C-ABI."""

    kind: str
    degree: int
    params: np.ndarray  # (N, 11 + colour) float64
    axes: np.ndarray  # (3, 3) rows are lobe axes
    background: np.ndarray  # (3,)

    @property
    def n(self) -> int:
        return int(self.params.shape[0])


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def build_oracle(quiet=True):
    """Build oracle/build and (when /root/reference exists) oracle/_ref."""
    kw = dict(stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL) if quiet else {}
    subprocess.run(["make", "-C", ORACLE_DIR, "all"], check=True, **kw)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.path = path
        self.lib = ctypes.CDLL(path)
        p = self.prefix
        L = self.lib
        getattr(L, p + "last_error").restype = ctypes.c_char_p

    def err(self):
        return getattr(self.lib, self.prefix + "last_error")().decode()


class RefLib(_Lib):
    """The reference's own code (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_scene_synth.restype = ctypes.c_void_p
        L.ref_scene_synth.argtypes = [ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double]
        L.ref_scene_from_params.restype = ctypes.c_void_p
        L.ref_scene_from_params.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.ref_scene_free.argtypes = [ctypes.c_void_p]
        L.ref_scene_count.restype = ctypes.c_size_t
        L.ref_scene_count.argtypes = [ctypes.c_void_p]
        L.ref_scene_stride.restype = ctypes.c_size_t
        L.ref_scene_stride.argtypes = [ctypes.c_void_p]
        L.ref_scene_params.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.ref_orbit_camera.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(OrcCamera)]
        L.ref_orbit_cameras.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.POINTER(OrcCamera)]
        for fn in ("ref_render", "ref_render_bruteforce"):
            getattr(L, fn).argtypes = [ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                       ctypes.POINTER(OrcConfig), ctypes.c_void_p, ctypes.c_void_p]
        L.ref_project_each.argtypes = [ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                       ctypes.POINTER(OrcConfig), ctypes.c_void_p]
        L.ref_tile_grid.argtypes = [ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                    ctypes.POINTER(OrcConfig), ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.POINTER(ctypes.c_size_t)]
        L.ref_eval_color.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.ref_flops_per_gaussian.argtypes = [ctypes.c_int, ctypes.c_int]
        L.ref_select_degree.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_int)]
        L.ref_color_param_count.argtypes = [ctypes.c_int, ctypes.c_int]
        L.ref_load_ply.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.ref_backward.argtypes = [ctypes.c_void_p, ctypes.POINTER(OrcCamera), ctypes.POINTER(OrcConfig),
                                   ctypes.c_void_p, ctypes.c_void_p]
        L.ref_psnr.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_double)]
        L.ref_ssim.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
        L.ref_save_ply.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
        L.ref_scene_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int), ctypes.c_void_p, ctypes.c_void_p]

    # -- PLY checkpoints (ply.cpp) -------------------------------------------
    def load_ply(self, path):
        """load_ply: (0, FlatScene) or (status, message) with the reference's message."""
        h = ctypes.c_void_p()
        rc = self.lib.ref_load_ply(os.fsencode(str(path)), ctypes.byref(h))
        if rc != 0:
            return rc, self.err()
        try:
            kind, deg = ctypes.c_int(), ctypes.c_int()
            axes, bg = np.zeros(9), np.zeros(3)
            self.lib.ref_scene_info(h, ctypes.byref(kind), ctypes.byref(deg), _ptr(axes), _ptr(bg))
            n = self.lib.ref_scene_count(h)
            stride = self.lib.ref_scene_stride(h) if n else 0
            params = np.zeros((n, stride), dtype=np.float64)
            if n:
                self.lib.ref_scene_params(h, _ptr(params))
        finally:
            self.lib.ref_scene_free(h)
        name = KIND_NAMES.get(kind.value, "empty")
        return 0, FlatScene(name, deg.value, params, axes.reshape(3, 3), bg)

    def backward(self, s: FlatScene, cam, cfg, upstream):
        """backward (grad.cpp): (N, stride) flat gradients."""
        h = self._handle(s)
        try:
            up = np.ascontiguousarray(upstream, dtype=np.float64)
            out = np.zeros_like(np.ascontiguousarray(s.params, dtype=np.float64))
            rc = self.lib.ref_backward(h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(up), _ptr(out))
            assert rc == 0, self.err()
            return out
        finally:
            self.lib.ref_scene_free(h)

    # -- image metrics (metrics.cpp) -----------------------------------------
    def psnr(self, a, b):
        a, b = (np.ascontiguousarray(x, dtype=np.float64) for x in (a, b))
        out = ctypes.c_double()
        rc = self.lib.ref_psnr(_ptr(a), _ptr(b), a.shape[1], a.shape[0], a.shape[2], ctypes.byref(out))
        assert rc == 0, self.err()
        return out.value

    def ssim(self, a, b, grad=False):
        a, b = (np.ascontiguousarray(x, dtype=np.float64) for x in (a, b))
        out = ctypes.c_double()
        g = np.empty_like(a) if grad else None
        rc = self.lib.ref_ssim(_ptr(a), _ptr(b), a.shape[1], a.shape[0], a.shape[2], ctypes.byref(out), _ptr(g))
        assert rc == 0, self.err()
        return (out.value, g) if grad else out.value

    def save_ply(self, s: FlatScene, path, layout: int) -> int:
        h = self._handle(s)
        try:
            return self.lib.ref_save_ply(h, os.fsencode(str(path)), layout)
        finally:
            self.lib.ref_scene_free(h)

    # -- scenes -------------------------------------------------------------
    def synth(self, n, seed, kind="mixed", sh_degree=3, ls=(-4.5, -2.5)) -> FlatScene:
        h = self.lib.ref_scene_synth(n, seed, KINDS[kind], sh_degree, ls[0], ls[1])
        try:
            stride = self.lib.ref_scene_stride(h) if n else 11 + color_param_count(
                kind, 2 if kind == "mixed" else sh_degree)
            out = np.zeros((n, stride), dtype=np.float64)
            if n:
                self.lib.ref_scene_params(h, _ptr(out))
        finally:
            self.lib.ref_scene_free(h)
        deg = 2 if kind == "mixed" else (sh_degree if kind == "sh" else 0)
        return FlatScene(kind, deg, out, np.eye(3), np.zeros(3))

    def _handle(self, s: FlatScene):
        params = np.ascontiguousarray(s.params, dtype=np.float64)
        axes = np.ascontiguousarray(s.axes, dtype=np.float64)
        bg = np.ascontiguousarray(s.background, dtype=np.float64)
        return self.lib.ref_scene_from_params(s.n, KINDS[s.kind], s.degree, _ptr(params),
                                              _ptr(axes), _ptr(bg))

    # -- cameras ------------------------------------------------------------
    def orbit_camera(self, target, distance, angle, elevation, w, h, focal) -> OrcCamera:
        c = OrcCamera()
        tgt = np.asarray(target, dtype=np.float64)
        self.lib.ref_orbit_camera(_ptr(tgt), distance, angle, elevation, w, h, focal,
                                  ctypes.byref(c))
        return c

    def orbit_cameras(self, count, w, h, distance, focal, elevation=0.35):
        arr = (OrcCamera * count)()
        self.lib.ref_orbit_cameras(count, w, h, distance, focal, elevation, arr)
        return list(arr)

    # -- render path --------------------------------------------------------
    def render(self, s: FlatScene, cam: OrcCamera, cfg: OrcConfig, bruteforce=False):
        rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
        T = np.zeros((cam.height, cam.width, 1), dtype=np.float64)
        h = self._handle(s)
        try:
            fn = self.lib.ref_render_bruteforce if bruteforce else self.lib.ref_render
            rc = fn(h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(rgb), _ptr(T))
        finally:
            self.lib.ref_scene_free(h)
        if rc != OK:
            return rc, self.err()
        return rgb, T

    def project_each(self, s: FlatScene, cam, cfg):
        out = np.zeros(s.n, dtype=SPLAT_DTYPE)
        h = self._handle(s)
        try:
            rc = self.lib.ref_project_each(h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(out))
        finally:
            self.lib.ref_scene_free(h)
        if rc != OK:
            return rc, self.err()
        return out

    def tile_grid(self, s: FlatScene, cam, cfg):
        """Returns (order[V], offsets[tiles+1], entries[P]) -- entries are ranks."""
        ts = cfg.tile_size
        ntiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts) if ts >= 1 else 0
        order = np.zeros(max(s.n, 1), dtype=np.uint32)
        offsets = np.zeros(ntiles + 1, dtype=np.uint64)
        nv = ctypes.c_size_t(0)
        ne = ctypes.c_size_t(0)
        h = self._handle(s)
        try:
            rc = self.lib.ref_tile_grid(h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(order),
                                        ctypes.byref(nv), _ptr(offsets), None, 0, ctypes.byref(ne))
            if rc != OK:
                return rc, self.err()
            entries = np.zeros(max(ne.value, 1), dtype=np.uint32)
            rc = self.lib.ref_tile_grid(h, ctypes.byref(cam), ctypes.byref(cfg), _ptr(order),
                                        ctypes.byref(nv), _ptr(offsets), _ptr(entries), ne.value,
                                        ctypes.byref(ne))
        finally:
            self.lib.ref_scene_free(h)
        return order[: nv.value].copy(), offsets, entries[: ne.value].copy()

    def eval_color(self, kind, degree, cparams, axes, direction, override=None):
        out = np.zeros(3)
        c = np.ascontiguousarray(cparams, dtype=np.float64)
        a = np.ascontiguousarray(axes, dtype=np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        rc = self.lib.ref_eval_color(KINDS[kind], degree, _ptr(c), _ptr(a), _ptr(d),
                                     1 if override is not None else 0,
                                     override if override is not None else 0, _ptr(out))
        if rc != OK:
            return rc, self.err()
        return out


class OrcLib(_Lib):
    """The plain-C restatement (oracle/build/liboracle.so)."""

    prefix = "orc_"

    def __init__(self, path=ORC_SO):
        super().__init__(path)
        L = self.lib
        L.orc_synth_scene.argtypes = [ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        L.orc_orbit_camera.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(OrcCamera)]
        L.orc_orbit_cameras.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.POINTER(OrcCamera)]
        L.orc_project_each.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                       ctypes.POINTER(OrcConfig), ctypes.c_void_p]
        L.orc_tile_grid.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                    ctypes.POINTER(OrcConfig), ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.POINTER(ctypes.c_size_t)]
        L.orc_render.argtypes = [ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(OrcCamera),
                                 ctypes.POINTER(OrcConfig), ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_size_t),
                                 ctypes.POINTER(ctypes.c_size_t)]
        L.orc_eval_color.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_flops_per_gaussian.argtypes = [ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int)]
        L.orc_select_degree.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_int)]
        L.orc_color_param_count.argtypes = [ctypes.c_int, ctypes.c_int]

    def synth(self, n, seed, kind="mixed", sh_degree=3, ls=(-4.5, -2.5)) -> FlatScene:
        deg = 2 if kind == "mixed" else sh_degree
        stride = 11 + color_param_count(kind, deg)
        out = np.zeros((n, stride), dtype=np.float64)
        self.lib.orc_synth_scene(n, seed, KINDS[kind], sh_degree, ls[0], ls[1], _ptr(out))
        deg_out = 2 if kind == "mixed" else (sh_degree if kind == "sh" else 0)
        return FlatScene(kind, deg_out, out, np.eye(3), np.zeros(3))

    def orbit_camera(self, target, distance, angle, elevation, w, h, focal) -> OrcCamera:
        c = OrcCamera()
        tgt = np.asarray(target, dtype=np.float64)
        self.lib.orc_orbit_camera(_ptr(tgt), distance, angle, elevation, w, h, focal,
                                  ctypes.byref(c))
        return c

    def orbit_cameras(self, count, w, h, distance, focal, elevation=0.35):
        arr = (OrcCamera * count)()
        self.lib.orc_orbit_cameras(count, w, h, distance, focal, elevation, arr)
        return list(arr)

    def _args(self, s: FlatScene):
        params = np.ascontiguousarray(s.params, dtype=np.float64)
        axes = np.ascontiguousarray(s.axes, dtype=np.float64)
        bg = np.ascontiguousarray(s.background, dtype=np.float64)
        return params, axes, bg

    def project_each(self, s: FlatScene, cam, cfg):
        params, axes, _ = self._args(s)
        out = np.zeros(s.n, dtype=SPLAT_DTYPE)
        rc = self.lib.orc_project_each(s.n, KINDS[s.kind], s.degree, _ptr(params), _ptr(axes),
                                       ctypes.byref(cam), ctypes.byref(cfg), _ptr(out))
        if rc != OK:
            return rc, self.err()
        return out

    def tile_grid(self, s: FlatScene, cam, cfg):
        params, axes, _ = self._args(s)
        ts = cfg.tile_size
        ntiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts) if ts >= 1 else 0
        splats = np.zeros(max(s.n, 1), dtype=SPLAT_DTYPE)
        order = np.zeros(max(s.n, 1), dtype=np.uint32)
        offsets = np.zeros(ntiles + 1, dtype=np.uint64)
        nv = ctypes.c_size_t(0)
        ne = ctypes.c_size_t(0)
        args = (s.n, KINDS[s.kind], s.degree, _ptr(params), _ptr(axes), ctypes.byref(cam),
                ctypes.byref(cfg), _ptr(splats), _ptr(order), ctypes.byref(nv), _ptr(offsets))
        rc = self.lib.orc_tile_grid(*args, None, 0, ctypes.byref(ne))
        if rc != OK:
            return rc, self.err()
        entries = np.zeros(max(ne.value, 1), dtype=np.uint32)
        self.lib.orc_tile_grid(*args, _ptr(entries), ne.value, ctypes.byref(ne))
        return order[: nv.value].copy(), offsets, entries[: ne.value].copy()

    def render(self, s: FlatScene, cam, cfg, stats=False):
        params, axes, bg = self._args(s)
        rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
        T = np.zeros((cam.height, cam.width, 1), dtype=np.float64)
        et = ctypes.c_uint64(0)
        nv = ctypes.c_size_t(0)
        ne = ctypes.c_size_t(0)
        rc = self.lib.orc_render(s.n, KINDS[s.kind], s.degree, _ptr(params), _ptr(axes), _ptr(bg),
                                 ctypes.byref(cam), ctypes.byref(cfg), _ptr(rgb), _ptr(T),
                                 ctypes.byref(et), ctypes.byref(nv), ctypes.byref(ne))
        if rc != OK:
            return rc, self.err()
        if stats:
            return rgb, T, {"E_t": et.value, "V": nv.value, "P": ne.value}
        return rgb, T

    def eval_color(self, kind, degree, cparams, axes, direction, override=None):
        out = np.zeros(3)
        c = np.ascontiguousarray(cparams, dtype=np.float64)
        a = np.ascontiguousarray(axes, dtype=np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        rc = self.lib.orc_eval_color(KINDS[kind], degree, _ptr(c), _ptr(a), _ptr(d),
                                     1 if override is not None else 0,
                                     override if override is not None else -1, _ptr(out))
        if rc != OK:
            return rc, self.err()
        return out
