"""Summarise ncu --set full captures into profiles/ (JSON) and derive the traffic /
instruction figures bench.py reports (profiles/ncu_traffic.json).

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--traffic profiles/ncu_traffic.json]

The capture is expected to hold one frame's K1 launch and its composite launches
(tools/profile_frame.py under ncu -k "regex:preprocess|composite").
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        k = {"kernel": d["Kernel Name"].split("(")[0]}
        for m in KEYS:
            if m not in d:
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            unit = u.get(m, "")
            if unit in SCALE:
                v *= SCALE[unit]
                unit = "byte" if "byte" in unit else ("us" if "second" in unit else unit)
            k[m] = v
            k[m + ".unit"] = unit
        stalls = {m.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                  float(d[m]) for m in h if m.startswith("smsp__average_warps_issue_stalled_")
                  and m.endswith("_per_issue_active.ratio") and d[m]}
        k["top_stalls"] = sorted(stalls.items(), key=lambda t: -t[1])[:5]
        kernels.append(k)
    with open(out, "w") as f:
        json.dump({"report": rep, "kernels": kernels}, f, indent=1)
    if traffic_out:
        k1 = [k for k in kernels if "preprocess" in k["kernel"]]
        k7 = [k for k in kernels if "composite" in k["kernel"] and "kernel" in k["kernel"]]
        t = {"source": out}
        if k1:
            t["k1_dram_bytes_per_launch"] = k1[0]["dram__bytes_read.sum"] + k1[0]["dram__bytes_write.sum"]
            t["k1_us"] = k1[0]["gpu__time_duration.sum"]
        if k7:
            t["composite_launches_per_frame"] = len(k7)
            t["composite_warp_inst_per_frame"] = sum(k["smsp__inst_executed.sum"] for k in k7)
            t["composite_dram_bytes_per_frame"] = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
                                                      for k in k7)
            t["composite_us_per_frame"] = sum(k["gpu__time_duration.sum"] for k in k7)
        with open(traffic_out, "w") as f:
            json.dump(t, f, indent=1)
    for k in kernels:
        print(k["kernel"][-40:], round(k.get("gpu__time_duration.sum", 0), 1), "us",
              round((k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)) / 1e6, 1), "MB",
              k["top_stalls"][:2])


if __name__ == "__main__":
    main()
