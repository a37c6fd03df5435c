"""Pin the oracle restatement (oracle/sgs_oracle.c) before trusting it.

* against every golden fixture made by the REFERENCE's own code
  (tests/golden/make_golden.py -> oracle/_ref), bit-exactly;
* against the live reference build on fresh random cases (when oracle/_ref exists);
* against the reference tests' analytic known answers
  (proj/tests/test_raster.cpp, proj/tests/test_color.cpp).
"""
import math

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden
from oracle_lib import (INVALID_ARGUMENT, NUMERIC, FlatScene, OrcCamera, camera_from_dict,
                        make_config)

SPLAT_EXACT = ("visible", "mean2d", "conic", "depth", "opacity", "radius", "degree")


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_restatement_matches_golden(orc, name):
    scene, cam, cfg, d = load_golden(name)
    r = orc.render(scene, cam, cfg)
    if "error_code" in d:
        assert isinstance(r[0], int), "reference raised, restatement did not"
        assert r[0] == int(d["error_code"])
        return
    rgb, T = r
    # The restatement reproduces the reference bit-for-bit (same op order, same libm).
    assert np.array_equal(rgb, d["image"])
    assert np.array_equal(T, d["T"])
    splats = orc.project_each(scene, cam, cfg)
    for f in SPLAT_EXACT:
        assert np.array_equal(splats[f], d["splats"][f]), f
    assert np.array_equal(splats["color"], d["splats"]["color"])
    order, offsets, entries = orc.tile_grid(scene, cam, cfg)
    assert np.array_equal(order, d["order"])
    assert np.array_equal(offsets, d["offsets"])
    assert np.array_equal(entries, d["entries"])
    if "brute_image" in d:
        # test_raster.cpp:113-132: tiled == brute force to 1e-5.
        assert np.abs(d["image"] - d["brute_image"]).max() < 1e-5


def test_synth_matches_golden(orc):
    d = np.load(f"{__import__('conftest').GOLDEN_DIR}/synth.npz")
    for kind, deg in (("sh", 0), ("sh", 1), ("sh", 3), ("sg1", 3), ("sg3", 3), ("mixed", 3)):
        assert np.array_equal(orc.synth(64, 4242, kind, deg).params, d[f"{kind}{deg}"])
    cams = orc.orbit_cameras(8, 1920, 1080, 4.0, 1296.0, 0.35)
    for i, c in enumerate(cams):
        assert np.array_equal(np.array(c.R[:]).reshape(3, 3), d[f"ring{i}_R"])
        assert np.array_equal(np.array(c.t[:]), d[f"ring{i}_t"])


@pytest.mark.parametrize("kind", ["sh", "sg1", "sg3", "mixed"])
@pytest.mark.parametrize("seed", [1, 2])
def test_restatement_matches_live_reference(orc, ref, kind, seed):
    a = ref.synth(400, 700 + seed, kind, 2 + seed % 2, ls=(-4.0, -2.0))
    b = orc.synth(400, 700 + seed, kind, 2 + seed % 2, ls=(-4.0, -2.0))
    assert np.array_equal(a.params, b.params)
    a.background = np.array([0.3, 0.2, 0.1])
    rng = np.random.default_rng(seed)
    cam = ref.orbit_camera([0, 0, 0], 3.0 + rng.random(), rng.random() * 6.28, 0.4, 80, 56, 70.0)
    for cfg in (make_config(), make_config(tile_size=7),
                make_config(degree_override=1) if kind == "mixed" else make_config(tile_size=32)):
        ra = ref.render(a, cam, cfg)
        rb = orc.render(a, cam, cfg)
        assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
        ga = ref.tile_grid(a, cam, cfg)
        gb = orc.tile_grid(a, cam, cfg)
        for x, y in zip(ga, gb):
            assert np.array_equal(x, y)


def test_restatement_error_order_matches_serial_reference(orc, ref):
    s = orc.synth(60, 5, "sh", 3, ls=(-3.0, -2.0))
    s.params[40, 3:7] = 0.0
    cam = orc.orbit_camera([0, 0, 0], 4.0, 0.2, 0.3, 48, 48, 60.0)
    cfg = make_config(threads=1)
    assert orc.render(s, cam, cfg)[0] == NUMERIC
    assert ref.render(s, cam, cfg)[0] == NUMERIC


# --- analytic known answers from the reference's own unit tests -----------------

def _test_camera(width=64, height=48, focal=80.0):
    """proj/tests/test_raster.cpp:15-26."""
    return camera_from_dict({"R": np.eye(3), "t": [0, 0, 4.0], "fx": focal, "fy": focal,
                             "cx": width / 2.0, "cy": height / 2.0, "width": width,
                             "height": height, "near": 0.01})


def _centered(log_scale=-2.0, opacity=0.9, n=1):
    """proj/tests/test_raster.cpp:28-37 (SH degree 0, colour (0.8, 0.4, 0.2))."""
    p = np.zeros((n, 14))
    p[:, 3] = 1.0
    p[:, 7:10] = log_scale
    p[:, 10] = math.log(opacity / (1 - opacity))
    p[:, 11:14] = [0.8, 0.4, 0.2]
    return FlatScene("sh", 0, p, np.eye(3), np.zeros(3))


def test_kat_principal_point(orc):
    sp = orc.project_each(_centered(-4.0), _test_camera(), make_config())[0]
    assert sp["visible"] == 1
    assert sp["mean2d"][0] == pytest.approx(32.0, rel=1e-12)
    assert sp["mean2d"][1] == pytest.approx(24.0, rel=1e-12)
    assert sp["depth"] == pytest.approx(4.0)


def test_kat_culling(orc):
    s = _centered()
    s.params[0, 0:3] = [0, 0, -8.0]
    assert orc.project_each(s, _test_camera(), make_config())[0]["visible"] == 0
    s.params[0, 0:3] = [100.0, 0, 0]
    assert orc.project_each(s, _test_camera(), make_config())[0]["visible"] == 0


def test_kat_radius_small_angle(orc):
    cam = _test_camera(128, 128, 200.0)
    for ls in (-3.5, -3.0, -2.5):
        s = _centered(ls)
        sp = orc.project_each(s, cam, make_config())[0]
        sigma = 200.0 * math.exp(ls) / 4.0
        assert sp["radius"] == pytest.approx(3.0 * math.sqrt(sigma**2 + 0.3), rel=0.05)


def test_kat_select_degree_and_costs(orc):
    import ctypes
    out = ctypes.c_int()
    inf = float("inf")
    for r, lo, hi, want in ((1, 2, 8, 0), (5, 2, 8, 1), (100, 2, 8, 2), (2, 2, 8, 1),
                            (1e9, inf, inf, 0), (0.5, 0, 0, 2)):
        assert orc.lib.orc_select_degree(r, lo, hi, ctypes.byref(out)) == 0
        assert out.value == want
    assert orc.lib.orc_select_degree(1.0, 8.0, 2.0, ctypes.byref(out)) == INVALID_ARGUMENT
    # test_raster.cpp:200-220
    for kind, deg, want in ((0, 0, 6), (0, 1, 27), (0, 2, 72), (0, 3, 139), (1, 3, 14),
                            (2, 3, 42), (3, 2, 114)):
        assert orc.lib.orc_flops_per_gaussian(kind, deg, ctypes.byref(out)) == 0
        assert out.value == want


def test_kat_empty_scene_is_background(orc):
    s = FlatScene("sh", 0, np.zeros((0, 14)), np.eye(3), np.array([0.2, 0.4, 0.6]))
    rgb, T = orc.render(s, _test_camera(32, 24), make_config())
    assert np.allclose(rgb, [0.2, 0.4, 0.6]) and np.all(T == 1.0)


def test_kat_opaque_center(orc):
    s = _centered(-1.2, 0.9999)
    cam = _test_camera(65, 65)
    cam.cx = cam.cy = 32.5
    rgb, _ = orc.render(s, cam, make_config())
    expected = np.maximum(0.0, 0.5 + 0.28209479177387814 * np.array([0.8, 0.4, 0.2]))
    assert np.allclose(rgb[32, 32], expected * 0.999, rtol=1e-3)


def test_kat_color(orc):
    # test_color.cpp:47-62 (eval_sg through a sg1 model with zero diffuse)
    c = np.zeros(10)
    c[3:6] = 1.0
    c[6] = math.log(math.log(2.0))  # lambda = ln 2
    c[7:10] = [0, 0, 1]
    assert np.allclose(orc.eval_color("sg1", 0, c, np.eye(3), [0, 0, -1.0]), 0.25, atol=1e-12)
    # test_color.cpp:122-133 (ortho identity axes)
    c = np.zeros(15)
    c[3:6] = [1, 0, 0]
    assert np.allclose(orc.eval_color("sg3", 0, c, np.eye(3), [1.0, 0, 0]), [1, 0, 0])
    assert orc.eval_color("sg3", 0, c, np.eye(3), [0, 1.0, 0])[0] == pytest.approx(math.exp(-1))
    # mixed with zero lobes == pure SH (test_color.cpp:89-105)
    rng = np.random.default_rng(13)
    sh = rng.uniform(-0.08, 0.08, 27)
    sh[:3] = rng.uniform(0.1, 0.3, 3) / 0.28209479177387814
    mixed = np.concatenate([sh, np.zeros(12)])
    mixed[30::4] = rng.uniform(-1, 2, 3)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    a = orc.eval_color("mixed", 2, mixed, np.eye(3), d)
    b = orc.eval_color("sh", 2, sh, np.eye(3), d)
    assert np.abs(a - b).max() <= 1e-12
    # non-unit direction rejected (test_color.cpp:41-45)
    assert orc.eval_color("sh", 2, sh, np.eye(3), [0, 0, 2.0])[0] == INVALID_ARGUMENT
