"""CPU-side checks of the product boundary (no GPU needed):
the C-ABI library loads and exports every symbol include/sgs.h declares, and its
host-side entry points (scalar helpers, synthetic scenes, orbit cameras) match the
reference's own outputs bit-exactly (tests/golden/synth.npz)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_00342_b200 as sg
from paper_2501_00342_b200 import _capi
from conftest import GOLDEN_DIR, ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sgs.h")).read()
    return sorted(set(re.findall(r"\b(sgs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_capi.SIGNATURES), "ctypes binding must cover include/sgs.h"
    assert lib.sgs_abi_version() == 1


def test_library_is_sm100a_cuda():
    so = _capi.LIB_PATH
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out


def test_scalar_helpers_match_reference_costs():
    for kind, deg, want in (("sh", 0, 6), ("sh", 1, 27), ("sh", 2, 72), ("sh", 3, 139),
                            ("sg1", 3, 14), ("sg3", 3, 42), ("mixed", 2, 114), ("mixed", 1, 69),
                            ("mixed", 0, 48)):
        assert sg.flops_per_gaussian(kind, deg) == want
    assert sg.param_count("sh", 3) == 48 and sg.param_count("sg1") == 10
    assert sg.param_count("sg3") == 15 and sg.param_count("mixed", 2) == 39
    assert sg.select_degree(2.0, 2.0, 8.0) == 1
    with pytest.raises(sg.InvalidArgumentError):
        sg.select_degree(1.0, 8.0, 2.0)
    with pytest.raises(sg.InvalidArgumentError):
        sg.flops_per_gaussian("sh", 4)


def test_synth_matches_reference_golden():
    d = np.load(os.path.join(GOLDEN_DIR, "synth.npz"))
    for kind, deg in (("sh", 0), ("sh", 1), ("sh", 3), ("sg1", 3), ("sg3", 3), ("mixed", 3)):
        s = sg.synth_scene(64, kind, 4242, sh_degree=deg)
        assert np.array_equal(s.params, d[f"{kind}{deg}"]), kind
    cams = sg.orbit_cameras(8, 1920, 1080, 4.0, 1296.0, 0.35)
    for i, c in enumerate(cams):
        assert np.array_equal(c.rotation, d[f"ring{i}_R"])
        assert np.array_equal(c.translation, d[f"ring{i}_t"])


def test_synth_matches_live_reference(ref):
    for kind in ("sh", "sg1", "sg3", "mixed"):
        a = sg.synth_scene(500, kind, 99, sh_degree=2, log_scale_range=(-5.5, -4.0))
        b = ref.synth(500, 99, kind, 2, ls=(-5.5, -4.0))
        assert np.array_equal(a.params, b.params)


def test_sh3_swap_keeps_geometry():
    m = sg.synth_scene(100, "mixed", 5)
    s = sg.synth_sh3_from_mixed(m, 5)
    assert s.params.shape == (100, 59)
    assert np.array_equal(s.params[:, :11 + 27], m.params[:, :11 + 27])
    amp = 0.25 * 0.55 ** 3
    assert np.all(np.abs(s.params[:, 38:]) <= amp)


def test_scene_plan_layout():
    m = sg.synth_scene(1000, "mixed", 1)
    meta = sg.Renderer.plan(m)
    assert meta.geometry_f64 == 0  # synth rounds through f32
    # 3 geometry planes + 7 SH + 3 SG float4 planes, 256-B aligned
    assert meta.blob_bytes >= 1000 * 16 * 13
    m.params[3, 0] = 0.1  # not f32-exact -> FP64 geometry planes
    assert sg.Renderer.plan(m).geometry_f64 == 1


def test_invalid_scene_descs_rejected():
    with pytest.raises(sg.InvalidArgumentError):
        sg.Renderer.plan(sg.Scene("sh", 4, np.zeros((1, 11 + 75))))
    with pytest.raises(sg.InvalidArgumentError):
        sg.Renderer.plan(sg.Scene("mixed", 3, np.zeros((1, 11 + 60))))
