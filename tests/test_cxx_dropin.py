"""The reference's own C++ render-path unit tests, compiled unmodified against the
B200 drop-in library (include/sgsplat/*.hpp + libsgsplat_b200.so, built by
tests/reftests/Makefile from /root/reference/proj/tests/test_raster.cpp with the
doctest shim in third_party/doctest_shim)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "build", "reftests", "test_raster_b200")
BIN_METRICS = os.path.join(ROOT, "build", "reftests", "test_metrics_b200")
BIN_GRAD = os.path.join(ROOT, "build", "reftests", "test_grad_b200")


def test_dropin_library_exports_reference_api():
    lib = os.path.join(ROOT, "paper_2501_00342_b200", "libsgsplat_b200.so")
    if not os.path.exists(lib):
        pytest.skip("libsgsplat_b200.so not built")
    syms = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for name in ("sgsplat::render(", "sgsplat::project(", "sgsplat::select_degree(",
                 "sgsplat::flops_per_gaussian(", "sgsplat::make_synthetic_scene(",
                 "sgsplat::make_orbit_camera(", "sgsplat::eval_color(", "sgsplat::load_ply(",
                 "sgsplat::backward(", "sgsplat::psnr(", "sgsplat::ssim(", "sgsplat::ssim_with_grad("):
        assert name in syms, name


@pytest.mark.gpu
def test_reference_test_raster_passes_on_b200():
    if not os.path.exists(BIN):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


@pytest.mark.gpu
def test_reference_test_metrics_passes_on_b200():
    """proj/tests/test_metrics.cpp, unmodified, against the GPU metrics."""
    if not os.path.exists(BIN_METRICS):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN_METRICS], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("binary", ["test_raster_b200", "test_grad_b200"])
def test_reference_tests_pass_in_exact_mode(binary):
    """proj/tests/test_raster.cpp and test_grad.cpp, unmodified, against the drop-in
    with SGS_EXACT=1: render composites in FP64 (sgs_render_f64), backward is the GPU
    backward. test_grad needs the FP64 render: its finite differences and blend-weight
    identity are checked at 1e-6 .. 1e-9."""
    path = os.path.join(ROOT, "build", "reftests", binary)
    if not os.path.exists(path):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    env = dict(os.environ, SGS_EXACT="1")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
