"""ctypes binding of the C-ABI in include/sgs.h (libsgs_b200.so, built in-tree).

This is the exact binding a maintainer of the reference would add next to
proj/python/sgsplat/__init__.py. There is no fallback:
if the CUDA library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsgs_b200.so")

SGS_OK = 0
SGS_ERR_INVALID_ARGUMENT = 1
SGS_ERR_NUMERIC = 2
SGS_ERR_CUDA = 3
SGS_ERR_NCCL = 4
SGS_ERR_OUT_OF_MEMORY = 5
SGS_ERR_INTERNAL = 6
SGS_ERR_IO = 7
SGS_ERR_FORMAT = 8
SGS_PLY_REFERENCE3DGS = 0
SGS_PLY_SGEXTENDED = 1

SGS_SH, SGS_SG1, SGS_SG3, SGS_MIXED = 0, 1, 2, 3
SGS_F64, SGS_F32 = 0, 1
SGS_HOST, SGS_DEVICE = 0, 1


class sgs_camera(ctypes.Structure):
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


class sgs_render_config(ctypes.Structure):
    _fields_ = [
        ("tile_size", ctypes.c_int32),
        ("has_override", ctypes.c_int32),
        ("override_degree", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("degree_threshold_lo", ctypes.c_double),
        ("degree_threshold_hi", ctypes.c_double),
        ("early_stop_transmittance", ctypes.c_double),
    ]


class sgs_scene_desc(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_uint64),
        ("kind", ctypes.c_int32),
        ("sh_degree", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("params", ctypes.c_void_p),
        ("shared_axes", ctypes.c_double * 9),
        ("background", ctypes.c_double * 3),
    ]


class sgs_scene_meta(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_uint64),
        ("kind", ctypes.c_int32),
        ("sh_degree", ctypes.c_int32),
        ("geometry_f64", ctypes.c_int32),
        ("color_f64", ctypes.c_int32),
        ("blob_bytes", ctypes.c_uint64),
        ("shared_axes", ctypes.c_double * 9),
        ("background", ctypes.c_double * 3),
    ]


class sgs_ply_info(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_uint64),
        ("kind", ctypes.c_int32),
        ("sh_degree", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("binary", ctypes.c_int32),
        ("shared_axes", ctypes.c_double * 9),
        ("background", ctypes.c_double * 3),
    ]


class sgs_render_stats(ctypes.Structure):
    _fields_ = [
        ("visible", ctypes.c_uint64),
        ("tile_entries", ctypes.c_uint64),
        ("block_entries", ctypes.c_uint64),
        ("guard_hits", ctypes.c_uint64),
        ("want_timing", ctypes.c_int32),
        ("timing_path", ctypes.c_int32),
        ("ms_preprocess", ctypes.c_float),
        ("ms_depth_sort", ctypes.c_float),
        ("ms_binning", ctypes.c_float),
        ("ms_tile_sort", ctypes.c_float),
        ("ms_composite", ctypes.c_float),
        ("ms_total", ctypes.c_float),
    ]


class sgs_splat(ctypes.Structure):
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


_P = ctypes.c_void_p
_S = ctypes.c_int  # sgs_status
# sgs_row_fill_fn: int32 fill(void* user, float* rows, uint64 first, uint64 count)
ROW_FILL = ctypes.CFUNCTYPE(ctypes.c_int32, _P, ctypes.POINTER(ctypes.c_float), ctypes.c_uint64, ctypes.c_uint64)

# name -> (restype, argtypes); the full list of entry points declared in include/sgs.h
SIGNATURES = {
    "sgs_abi_version": (ctypes.c_int, []),
    "sgs_create": (_S, [ctypes.c_int, ctypes.POINTER(_P)]),
    "sgs_destroy": (None, [_P]),
    "sgs_last_error": (ctypes.c_char_p, []),
    "sgs_set_stream": (_S, [_P, _P]),
    "sgs_synchronize": (_S, [_P]),
    "sgs_launch_count": (_S, [_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    "sgs_scene_plan": (_S, [ctypes.POINTER(sgs_scene_desc), ctypes.POINTER(sgs_scene_meta)]),
    "sgs_scene_pack": (_S, [ctypes.POINTER(sgs_scene_desc), _P, ctypes.c_uint64]),
    "sgs_scene_upload": (_S, [_P, ctypes.POINTER(sgs_scene_desc), ctypes.POINTER(_P)]),
    "sgs_scene_upload_into": (_S, [_P, ctypes.POINTER(sgs_scene_desc), _P, ctypes.c_uint64,
                                   ctypes.POINTER(_P)]),
    "sgs_scene_bind": (_S, [_P, ctypes.POINTER(sgs_scene_meta), _P, ctypes.c_uint64,
                            ctypes.POINTER(_P)]),
    "sgs_scene_refresh": (_S, [_P, _P]),
    "sgs_scene_update": (_S, [_P, _P, ctypes.POINTER(sgs_scene_desc)]),
    "sgs_scene_update_rows": (_S, [_P, _P, ctypes.POINTER(sgs_scene_desc), ROW_FILL, _P]),
    "sgs_scene_get_meta": (_S, [_P, ctypes.POINTER(sgs_scene_meta)]),
    "sgs_scene_blob": (_S, [_P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_uint64)]),
    "sgs_scene_set_background": (_S, [_P, _P]),
    "sgs_scene_free": (None, [_P]),
    "sgs_render": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.POINTER(sgs_render_config), _P,
                        _P, ctypes.c_int32, ctypes.POINTER(sgs_render_stats)]),
    "sgs_render_batch": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.c_int32,
                              ctypes.POINTER(sgs_render_config), _P, _P, ctypes.c_int32,
                              ctypes.POINTER(sgs_render_stats)]),
    "sgs_project": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.POINTER(sgs_render_config),
                         _P]),
    "sgs_debug_tile_grid": (_S, [_P, _P, ctypes.POINTER(sgs_camera),
                                 ctypes.POINTER(sgs_render_config), _P,
                                 ctypes.POINTER(ctypes.c_uint64), _P, _P, ctypes.c_uint64,
                                 ctypes.POINTER(ctypes.c_uint64)]),
    "sgs_select_degree": (_S, [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.POINTER(ctypes.c_int32)]),
    "sgs_flops_per_gaussian": (_S, [ctypes.c_int32, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32)]),
    "sgs_color_param_count": (ctypes.c_int32, [ctypes.c_int32, ctypes.c_int32]),
    "sgs_synth_scene": (_S, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                             ctypes.c_double, ctypes.c_double, _P]),
    "sgs_synth_sh3_from_mixed": (_S, [ctypes.c_uint64, ctypes.c_uint64, _P, _P]),
    "sgs_orbit_camera": (_S, [_P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                              ctypes.POINTER(sgs_camera)]),
    "sgs_orbit_cameras": (_S, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.POINTER(sgs_camera)]),
    "sgs_render_f64": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.POINTER(sgs_render_config), _P, _P,
                            ctypes.c_int32]),
    "sgs_backward": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.POINTER(sgs_render_config), _P,
                          ctypes.c_int32, _P]),
    "sgs_psnr": (_S, [_P, _P, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                      ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "sgs_ssim": (_S, [_P, _P, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                      ctypes.c_int32, ctypes.POINTER(ctypes.c_double), _P]),
    "sgs_ply_read": (_S, [ctypes.c_char_p, ctypes.POINTER(sgs_ply_info), _P, ctypes.c_uint64]),
    "sgs_scene_load_ply": (_S, [_P, ctypes.c_char_p, ctypes.POINTER(sgs_ply_info), ctypes.POINTER(_P)]),
    "sgs_host_alloc": (_S, [ctypes.c_uint64, ctypes.POINTER(_P)]),
    "sgs_host_free": (None, [_P]),
    "sgs_group_unique_id": (_S, [_P]),
    "sgs_group_init_rank": (_S, [_P, ctypes.c_int32, ctypes.c_int32, _P, ctypes.POINTER(_P)]),
    "sgs_group_create": (_S, [ctypes.c_int32, _P, _P]),
    "sgs_group_destroy": (None, [_P]),
    "sgs_group_context": (_S, [_P, ctypes.POINTER(_P)]),
    "sgs_group_broadcast_scene": (_S, [_P, ctypes.POINTER(sgs_scene_desc), ctypes.c_int32, ctypes.POINTER(_P)]),
    "sgs_group_render_views": (_S, [_P, _P, ctypes.POINTER(sgs_camera), ctypes.c_int32,
                                    ctypes.POINTER(sgs_render_config), ctypes.c_int32, _P, _P, ctypes.c_int32,
                                    ctypes.POINTER(sgs_render_stats)]),
}
GROUP_ID_BYTES = 128

_lib = None


def load(path: str = LIB_PATH):
    """Load libsgs_b200.so. Raises ImportError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2501_00342_b200/csrc` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
