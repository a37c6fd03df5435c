"""Generate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref/libsgsref.so is built):
    make -C oracle all && python tests/golden/make_golden.py

Every array below is produced by the reference translation units
(proj/src/{synth,camera,raster,color}.cpp) through oracle/ref_harness.cpp --
nothing is computed by the restatement or by the product. The fixtures pin
  * the oracle restatement (tests/test_oracle.py, CPU), and
  * the CUDA path (tests/test_gpu_parity.py, GPU box, where /root/reference
    does not exist).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import RefLib, camera_to_dict, make_config  # noqa: E402

INF = float("inf")


def cam_arrays(prefix, cam):
    d = camera_to_dict(cam)
    return {
        f"{prefix}R": d["R"], f"{prefix}t": d["t"],
        f"{prefix}intr": np.array([d["fx"], d["fy"], d["cx"], d["cy"], d["near"]]),
        f"{prefix}size": np.array([d["width"], d["height"]], dtype=np.int32),
    }


def cfg_array(cfg):
    return np.array([cfg.tile_size, cfg.has_override, cfg.override_degree, cfg.threads,
                     cfg.degree_threshold_lo, cfg.degree_threshold_hi,
                     cfg.early_stop_transmittance], dtype=np.float64)


def case(ref, name, scene, cam, cfg, out, bruteforce=True):
    d = {"kind": np.array(scene.kind), "degree": np.array(scene.degree),
         "params": scene.params, "axes": scene.axes, "background": scene.background,
         "cfg": cfg_array(cfg)}
    d.update(cam_arrays("cam_", cam))
    r = ref.render(scene, cam, cfg)
    if isinstance(r[0], int):
        d["error_code"] = np.array(r[0])
        d["error_msg"] = np.array(r[1])
    else:
        d["image"], d["T"] = r
        d["splats"] = ref.project_each(scene, cam, cfg)
        order, offsets, entries = ref.tile_grid(scene, cam, cfg)
        d["order"], d["offsets"], d["entries"] = order, offsets, entries
        if bruteforce:
            d["brute_image"], d["brute_T"] = ref.render(scene, cam, cfg, bruteforce=True)
    out[name] = d


def main():
    ref = RefLib()
    cases = {}
    # test_raster.cpp:113-132 style: each colour model, 96x64, log-scale [-3.5, -1.5]
    # (the reference test uses test_camera; an orbit camera exercises a rotated R).
    for i, kind in enumerate(["sh", "sg1", "sg3", "mixed"]):
        s = ref.synth(120, 1000 + i, kind, 3, ls=(-3.5, -1.5))
        s.background = np.array([0.1, 0.1, 0.1])
        cam = ref.orbit_camera([0, 0, 0], 4.0, 0.7 + i, 0.3, 96, 64, 90.0)
        case(ref, f"models_{kind}", s, cam, make_config(), cases)
    # acceptance.cpp:140-179 style scenes with a coloured background, 128x96.
    for i, kind in enumerate(["sh", "sg1", "sg3", "mixed"]):
        s = ref.synth(300 + 50 * i, 5150 + i, kind, 3, ls=(-4.0, -2.0))
        s.background = np.array([0.2, 0.1, 0.3])
        cam = ref.orbit_camera([0, 0, 0], 4.0, 1.3 * i, 0.3, 128, 96, 120.0)
        case(ref, f"accept_{kind}", s, cam, make_config(), cases)
    # Config-A shape at reduced size: mixed, override 0 (3 SG + SH0), 160x160 f=1.2 H.
    s = ref.synth(1200, 20260001, "mixed", 3, ls=(-4.5, -2.5))
    cam = ref.orbit_camera([0, 0, 0], 4.0, 0.5, 0.3, 160, 160, 192.0)
    case(ref, "configA_small_override0", s, cam, make_config(degree_override=0), cases,
         bruteforce=False)
    # Config-B/C shape at reduced size: mixed override 1, 160x90 (16:9), f = 1.2 H.
    s = ref.synth(2500, 20260002, "mixed", 3, ls=(-5.5, -4.0))
    cam = ref.orbit_camera([0, 0, 0], 4.0, 0.5, 0.3, 160, 90, 108.0)
    case(ref, "configB_small_override1", s, cam, make_config(degree_override=1), cases,
         bruteforce=False)
    case(ref, "configB_small_adaptive", s, cam, make_config(), cases, bruteforce=False)
    # Non-default tile size and early stop; ragged image edges (70x45 with tile 8 / 13).
    s = ref.synth(400, 77, "mixed", 3, ls=(-3.5, -2.0))
    cam = ref.orbit_camera([0, 0, 0], 3.5, 2.0, -0.2, 70, 45, 80.0)
    case(ref, "tile8", s, cam, make_config(tile_size=8), cases)
    case(ref, "tile13_stop1e-2", s, cam, make_config(tile_size=13, early_stop=1e-2), cases)
    case(ref, "thresholds_inf", s, cam, make_config(thresholds=(INF, INF)), cases,
         bruteforce=False)
    case(ref, "thresholds_zero", s, cam, make_config(thresholds=(0.0, 0.0)), cases,
         bruteforce=False)
    # Empty scene: background everywhere, T = 1 (test_raster.cpp:85-97).
    e = ref.synth(0, 1, "sh", 0)
    e.background = np.array([0.2, 0.4, 0.6])
    cam = ref.orbit_camera([0, 0, 0], 4.0, 0.1, 0.3, 32, 24, 40.0)
    case(ref, "empty", e, cam, make_config(), cases)
    # Error contract (raster.cpp:9,75-76; common.hpp:126; color.cpp:184-189).
    s = ref.synth(50, 9, "sh", 3, ls=(-3.0, -2.0))
    cam = ref.orbit_camera([0, 0, 0], 4.0, 0.3, 0.3, 48, 48, 60.0)
    case(ref, "err_override_non_mixed", s, cam, make_config(degree_override=1), cases)
    s0 = ref.synth(50, 10, "sh", 3, ls=(-3.0, -2.0))
    s0.params[17, 3:7] = 0.0
    case(ref, "err_zero_quaternion", s0, cam, make_config(), cases)
    sm = ref.synth(50, 11, "mixed", 3, ls=(-3.0, -2.0))
    case(ref, "err_thresholds_lo_gt_hi", sm, cam, make_config(thresholds=(8.0, 2.0)), cases)
    case(ref, "err_override_too_high", sm, cam, make_config(degree_override=3), cases)
    case(ref, "err_tile_size0", sm, cam, make_config(tile_size=0), cases)

    os.makedirs(HERE, exist_ok=True)
    for name, d in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    # Synthetic-scene generator fixtures (synth.cpp:26-106) and orbit cameras.
    synth = {}
    for kind, deg in (("sh", 0), ("sh", 1), ("sh", 3), ("sg1", 3), ("sg3", 3), ("mixed", 3)):
        synth[f"{kind}{deg}"] = ref.synth(64, 4242, kind, deg).params
    cams = ref.orbit_cameras(8, 1920, 1080, 4.0, 1296.0, 0.35)
    for i, c in enumerate(cams):
        for k, v in cam_arrays(f"ring{i}_", c).items():
            synth[k] = v
    np.savez_compressed(os.path.join(HERE, "synth.npz"), **synth)
    print("wrote", len(cases) + 1, "fixtures to", HERE)


if __name__ == "__main__":
    main()
