"""The reference's own CPU render (oracle/_ref/libsgsref_fast.so) at every BASELINE
configuration, all host threads and one thread (the acceptance.cpp:104 convention),
with the host's CPU model: the CPU columns of BASELINE.md §2.

    python tools/cpu_reference_table.py [out.json]
"""
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import KINDS, REF_FAST_SO, RefLib, make_config  # noqa: E402  (CPU reference only)

ROWS = [  # name, n, seed, log-scale, W, H, focal, override, frames (all threads), frames (1 thread)
    ("A", 100_000, 20260001, (-4.5, -2.5), 800, 800, 960.0, 0, 5, 2),
    ("B", 1_000_000, 20260002, (-5.5, -4.0), 1920, 1080, 1296.0, 1, 3, 1),
    ("C", 3_000_000, 20260003, (-5.5, -4.0), 1920, 1080, 1296.0, 1, 3, 1),
]


def main():
    lib = RefLib(REF_FAST_SO)
    out = {"cpu": "", "nproc": os.cpu_count(), "rows": []}
    try:
        out["cpu"] = [ln.split(":", 1)[1].strip() for ln in subprocess.run(
            ["lscpu"], capture_output=True, text=True).stdout.splitlines() if ln.startswith("Model name")][0]
    except Exception:
        pass
    for name, n, seed, ls, W, H, f, ov, k_all, k_one in ROWS:
        h = lib.lib.ref_scene_synth(n, seed, KINDS["mixed"], 2, ls[0], ls[1])
        cam = lib.orbit_camera([0, 0, 0], 4.0, 0.5, 0.3, W, H, f)
        rgb = (ctypes.c_double * (W * H * 3))()
        T = (ctypes.c_double * (W * H))()
        row = {"config": name, "gaussians": n, "width": W, "height": H}
        for threads, k in ((0, k_all), (1, k_one)):
            cfg = make_config(degree_override=ov, threads=threads)
            times = []
            for i in range(k + (1 if threads == 0 else 0)):  # one warm-up at all threads
                t0 = time.perf_counter()
                assert lib.lib.ref_render(h, ctypes.byref(cam), ctypes.byref(cfg), rgb, T) == 0, lib.err()
                times.append(time.perf_counter() - t0)
            times = times[1:] if threads == 0 else times
            row["ms_all_threads" if threads == 0 else "ms_1_thread"] = 1e3 * statistics.median(times)
        lib.lib.ref_scene_free(h)
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
