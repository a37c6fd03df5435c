"""Generate tests/golden/metrics.npz: image pairs and the reference's own psnr, ssim
and ssim_with_grad (oracle/_ref, metrics.cpp) for them.

    python tests/golden/make_golden_metrics.py     # needs oracle/_ref (this container)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib  # noqa: E402

CASES = [("rgb_24x16", 16, 24, 3), ("gray_37x23", 23, 37, 1), ("tiny_5x4", 4, 5, 3), ("wide_64x9", 9, 64, 3),
         ("rgb_48x40", 40, 48, 3)]


def main():
    ref = RefLib()
    rng = np.random.default_rng(20260418)
    out = {}
    for name, h, w, c in CASES:
        a = rng.random((h, w, c))
        b = np.clip(0.7 * a + 0.3 * rng.random((h, w, c)), 0, 1)
        out[name + ".a"], out[name + ".b"] = a, b
        out[name + ".psnr"] = np.array(ref.psnr(a, b))
        v, g = ref.ssim(a, b, grad=True)
        out[name + ".ssim"] = np.array(ref.ssim(a, b))
        out[name + ".ssim_g"] = np.array(v)
        out[name + ".grad"] = g
    os.makedirs(os.path.join(HERE, "metrics"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "metrics", "metrics.npz"), **out)
    print("wrote", len(CASES), "metric cases")


if __name__ == "__main__":
    main()
