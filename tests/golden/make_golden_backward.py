"""Generate tests/golden/backward/: small scenes, cameras, upstream images and the
reference's own backward gradients (oracle/_ref, grad.cpp:69-246).

    python tests/golden/make_golden_backward.py     # needs oracle/_ref (this container)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib, camera_to_dict, make_config  # noqa: E402

OUT = os.path.join(HERE, "backward")
# name, kind, stored degree, count, log-scale range, W, H, focal, tile, override
CASES = [
    ("mixed_override1", "mixed", 2, 900, (-4.0, -2.8), 96, 64, 90.0, 16, 1),
    ("mixed_adaptive", "mixed", 2, 900, (-4.0, -2.5), 96, 64, 90.0, 16, -1),
    ("sh3", "sh", 3, 700, (-4.0, -2.8), 80, 56, 80.0, 16, -1),
    ("sg1", "sg1", 0, 700, (-4.0, -2.8), 80, 56, 80.0, 16, -1),
    ("sg3_tile24", "sg3", 0, 700, (-4.0, -2.8), 80, 56, 80.0, 24, -1),
    ("sh1_tile8", "sh", 1, 500, (-4.0, -2.8), 72, 40, 70.0, 8, -1),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    rng = np.random.default_rng(77)
    for name, kind, deg, n, ls, w, h, f, ts, ov in CASES:
        s = ref.synth(n, 1000 + n, kind, deg, ls)
        s.background = np.array([0.1, 0.2, 0.3])
        cam = ref.orbit_camera([0, 0, 0], 3.0, 0.7, 0.25, w, h, f)
        cfg = make_config(ts, degree_override=ov)
        up = rng.standard_normal((h, w, 3))
        g = ref.backward(s, cam, cfg, up)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), kind=kind, degree=s.degree, params=s.params,
                            axes=s.axes, background=s.background, upstream=up, grads=g, tile=ts, override=ov,
                            **{"cam_" + k: v for k, v in camera_to_dict(cam).items()})
    print("wrote", len(CASES), "backward cases to", OUT)


if __name__ == "__main__":
    main()
