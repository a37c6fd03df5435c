"""Generate tests/golden/ply/: small PLY checkpoints written by the reference's own
save_ply (oracle/_ref), plus ASCII / permuted-column / sidecar variants, and the
parameters the reference's load_ply reads from each (expected.npz).

    python tests/golden/make_golden_ply.py     # needs oracle/_ref (this container)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle_lib import RefLib  # noqa: E402
from test_ply import read_ply, write_ply  # noqa: E402

OUT = os.path.join(HERE, "ply")


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    files = []
    for kind, deg, layout in [("sh", 3, 0), ("sh", 1, 0), ("sg1", 0, 1), ("sg3", 0, 1), ("mixed", 2, 1)]:
        s = ref.synth(48, 777, kind, deg, (-4.0, -2.5))
        if kind in ("sg3", "mixed"):
            c, sn = np.cos(0.4), np.sin(0.4)
            s.axes = np.array([[c, 0, -sn], [0, 1, 0], [sn, 0, c]])
            s.background = np.array([0.2, 0.1, 0.05])
        name = f"{kind}{deg}.ply"
        assert ref.save_ply(s, os.path.join(OUT, name), layout) == 0, ref.err()
        files.append(name)
    # variants: ASCII with permuted columns (+ normals), a sidecar
    rng = np.random.default_rng(11)
    header, props, rows = read_ply(os.path.join(OUT, "sh3.ply"))
    perm = rng.permutation(len(props))
    write_ply(os.path.join(OUT, "sh3_ascii_permuted.ply"), header, [props[i] for i in perm] + ["nx", "ny", "nz"],
              np.concatenate([rows[:, perm], np.zeros((rows.shape[0], 3), "<f4")], 1), binary=False)
    files.append("sh3_ascii_permuted.ply")
    header, props, rows = read_ply(os.path.join(OUT, "mixed2.ply"))
    write_ply(os.path.join(OUT, "mixed2_sidecar.ply"), header, props, rows)
    with open(os.path.join(OUT, "mixed2_sidecar.ply.meta"), "w") as f:
        f.write("axes=0 1 0 0 0 1 1 0 0\nbackground=0.5 0.25 0.75\n")
    files.append("mixed2_sidecar.ply")
    expected = {}
    for name in files:
        rc, s = ref.load_ply(os.path.join(OUT, name))
        assert rc == 0, s
        expected[name + ".params"] = s.params
        expected[name + ".axes"] = np.asarray(s.axes, dtype=np.float64).reshape(9)
        expected[name + ".bg"] = np.asarray(s.background, dtype=np.float64)
        expected[name + ".kind"] = np.array(s.kind)
        expected[name + ".deg"] = np.array(s.degree)
    np.savez_compressed(os.path.join(OUT, "expected.npz"), **expected)
    print("wrote", len(files), "checkpoints to", OUT)


if __name__ == "__main__":
    main()
