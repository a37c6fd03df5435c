import glob
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import oracle_lib  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")
    # Build the oracle checker (and the reference build where /root/reference exists).
    if not os.path.exists(oracle_lib.ORC_SO) or (
        os.path.isdir("/root/reference") and not os.path.exists(oracle_lib.REF_SO)
    ):
        oracle_lib.build_oracle()


GOLDEN_DIR = os.path.join(HERE, "golden")
GOLDEN_CASES = sorted(
    os.path.basename(p)[:-4]
    for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
    if not p.endswith("synth.npz")
)


def load_golden(name):
    d = dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False))
    scene = oracle_lib.FlatScene(str(d["kind"]), int(d["degree"]), d["params"], d["axes"],
                                 d["background"])
    cam = oracle_lib.camera_from_dict({
        "R": d["cam_R"], "t": d["cam_t"], "fx": d["cam_intr"][0], "fy": d["cam_intr"][1],
        "cx": d["cam_intr"][2], "cy": d["cam_intr"][3], "near": d["cam_intr"][4],
        "width": int(d["cam_size"][0]), "height": int(d["cam_size"][1]),
    })
    c = d["cfg"]
    cfg = oracle_lib.make_config(tile_size=int(c[0]),
                                 degree_override=int(c[2]) if int(c[1]) else -1,
                                 threads=int(c[3]), thresholds=(c[4], c[5]), early_stop=c[6])
    return scene, cam, cfg, d


@pytest.fixture(scope="session")
def orc():
    return oracle_lib.OrcLib()


@pytest.fixture(scope="session")
def ref():
    if not os.path.exists(oracle_lib.REF_SO):
        pytest.skip("reference build oracle/_ref not available")
    return oracle_lib.RefLib()
