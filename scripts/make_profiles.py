"""Summarize the round's ncu captures into profiles/ (tracked):
r01_ncu_<name>.txt (details page) and ncu_summary.json (DRAM bytes per launch
of each config's dominant kernel, read by bench.py for roofline.traffic).

    python scripts/make_profiles.py gpurun_out/prof
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
# config -> capture (the config's dominant kernel, one launch)
CFG = {"c2": "c2_l0", "c3": "c3_l0", "c4": "c4_conv", "c5": "c5_l2"}


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(src):
    caps = {}
    for name in sorted(set(CFG.values())):
        rep = os.path.join(src, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, u, v = rows[0], rows[1], rows[2]
        m = {k: {"value": v[h.index(k)], "unit": u[h.index(k)]} for k in KEYS if k in h}
        dram = to_bytes(m["dram__bytes_read.sum"]["value"], m["dram__bytes_read.sum"]["unit"]) + \
            to_bytes(m["dram__bytes_write.sum"]["value"], m["dram__bytes_write.sum"]["unit"])
        caps[name] = {"kernel": v[h.index("Kernel Name")], "dram_bytes_per_launch": dram, "metrics": m}
        det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, "profiles", f"r01_ncu_{name}.txt"), "w") as f:
            f.write(det)
        print(name, caps[name]["kernel"][:60], m["gpu__time_duration.sum"], f"{dram / 1e6:.1f} MB")
    out = {"captures": caps,
           "note": "ncu --set full --clock-control none, one launch each (scripts/prof_layer.py --nograph)"}
    for cfg, name in CFG.items():
        if name in caps:
            out[cfg] = {"dram_bytes_per_launch": caps[name]["dram_bytes_per_launch"], "capture": name}
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof"))
