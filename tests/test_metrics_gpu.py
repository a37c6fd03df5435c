"""GPU PSNR / SSIM / SSIM gradient (metrics.hpp, metrics.cpp).

The per-pixel maps follow the reference's FP64 operation order, so the gradient image
is compared bit for bit; the two image means (PSNR's MSE, SSIM's mean) are a
fixed-order tree sum on the GPU instead of one serial loop, compared at a relative
1e-13. Fixtures: tests/golden/metrics/metrics.npz (the reference's own metrics.cpp through
oracle/_ref, tests/golden/make_golden_metrics.py). The reference's unit tests
(test_metrics.cpp) are restated at the end.
"""
import os

import numpy as np
import pytest

import paper_2501_00342_b200 as sg

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metrics", "metrics.npz"))
CASES = sorted({k.split(".")[0] for k in GOLD.files})
REL = 1e-13


@pytest.mark.parametrize("case", CASES)
def test_metrics_match_reference(case):
    a, b = GOLD[case + ".a"], GOLD[case + ".b"]
    assert sg.psnr(a, b) == pytest.approx(float(GOLD[case + ".psnr"]), rel=REL)
    assert sg.ssim(a, b) == pytest.approx(float(GOLD[case + ".ssim"]), rel=REL)
    v, g = sg.ssim_with_grad(a, b)
    assert v == pytest.approx(float(GOLD[case + ".ssim_g"]), rel=REL)
    assert np.array_equal(g, GOLD[case + ".grad"])  # bit for bit


def test_device_tensors_and_float32():
    import torch

    a, b = GOLD["rgb_24x16.a"], GOLD["rgb_24x16.b"]
    ta, tb = torch.as_tensor(a, device="cuda"), torch.as_tensor(b, device="cuda")
    assert sg.psnr(ta, tb) == pytest.approx(float(GOLD["rgb_24x16.psnr"]), rel=REL)
    v, g = sg.ssim_with_grad(ta, tb)
    assert g.is_cuda and np.array_equal(g.cpu().numpy(), GOLD["rgb_24x16.grad"])
    # float32 inputs are widened exactly: same result as the widened float64 images
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    assert sg.ssim(a32, b32) == sg.ssim(a32.astype(np.float64), b32.astype(np.float64))
    assert sg.psnr(torch.as_tensor(a32, device="cuda"), torch.as_tensor(b32, device="cuda")) == sg.psnr(
        a32.astype(np.float64), b32.astype(np.float64))


def test_rendered_frame_metrics():
    """The evaluation step the reference's CLI runs after render (main.cpp:194-223),
    on two full 1080p renders kept on the device."""
    import torch

    scene = sg.synth_scene(50_000, "mixed", 3, log_scale_range=(-5.0, -3.5))
    r = sg.Renderer(0)
    ds = r.upload(scene)
    cams = sg.orbit_cameras(2, 1920, 1080, 4.0, 1296.0)
    out = torch.empty((2, 1080, 1920, 3), device="cuda")
    r.render_batch(ds, cams, degree_override=1, rgb=out.data_ptr(), T=None, device_out=True)
    torch.cuda.synchronize()
    p = sg.psnr(out[0], out[1])
    s = sg.ssim(out[0], out[1])
    assert 0 < p < 100 and -1 <= s <= 1
    h = out[0].double().cpu().numpy(), out[1].double().cpu().numpy()
    assert sg.psnr(*h) == p and sg.ssim(*h) == s
    ds.free()


# -- test_metrics.cpp, restated --------------------------------------------------------
def _rand(seed, w, h):
    return np.random.default_rng(seed).random((h, w, 3))


def test_identical_images_capped_psnr_unit_ssim():
    img = _rand(5, 24, 16)
    assert sg.psnr(img, img) == pytest.approx(100.0)
    assert sg.ssim(img, img) == pytest.approx(1.0, rel=1e-12)


def test_constant_offset_is_20_db():
    a = np.full((20, 20, 3), 0.4)
    b = a + 0.1
    assert sg.psnr(a, b) == pytest.approx(20.0, rel=1e-9)
    assert sg.psnr(a, b) == sg.psnr(b, a)


def test_mismatched_and_empty_images_rejected():
    with pytest.raises(sg.InvalidArgumentError):
        sg.psnr(np.zeros((8, 8, 3)), np.zeros((9, 8, 3)))
    with pytest.raises(sg.InvalidArgumentError):
        sg.ssim(np.zeros((8, 8, 3)), np.zeros((9, 8, 3)))
    with pytest.raises(sg.InvalidArgumentError, match="empty image"):
        sg.psnr(np.zeros((0, 8, 3)), np.zeros((0, 8, 3)))


def test_ssim_gradient_matches_finite_differences():
    a, b = _rand(31, 8, 8), _rand(32, 8, 8)
    v, g = sg.ssim_with_grad(a, b)
    assert v == pytest.approx(sg.ssim(a, b), rel=1e-14)
    h = 1e-6
    flat = a.reshape(-1)
    for i in range(0, flat.size, 7):
        p = flat.copy()
        p[i] += h
        hi = sg.ssim(p.reshape(a.shape), b)
        p[i] -= 2 * h
        lo = sg.ssim(p.reshape(a.shape), b)
        assert g.reshape(-1)[i] == pytest.approx((hi - lo) / (2 * h), rel=1e-5, abs=1e-9)
