"""Summarize ncu captures into profiles/ (tracked): <name>.txt (details page)
and ncu_summary.json (DRAM bytes per launch of each config's dominant kernel,
read by bench.py for roofline.traffic).  Existing entries of other configs are
kept.

    python scripts/make_profiles.py gpurun_out c5_l4=r02_c5_l4 [c3_l0=r02_c3_l0 ...]   (keys: <workload>_l<KAN layer>)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(src, pairs):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    out = json.load(open(path)) if os.path.exists(path) else {"captures": {}}
    for cfg, name in pairs:
        rep = os.path.join(src, name + ".ncu-rep")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, u, v = rows[0], rows[1], rows[2]
        m = {k: {"value": v[h.index(k)], "unit": u[h.index(k)]} for k in KEYS if k in h}
        dram = to_bytes(m["dram__bytes_read.sum"]["value"], m["dram__bytes_read.sum"]["unit"]) + \
            to_bytes(m["dram__bytes_write.sum"]["value"], m["dram__bytes_write.sum"]["unit"])
        out["captures"][name] = {"kernel": v[h.index("Kernel Name")], "dram_bytes_per_launch": dram, "metrics": m}
        det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, "profiles", f"{name}.txt"), "w") as f:
            f.write(det)
        out[cfg] = {"dram_bytes_per_launch": dram, "capture": name}
        print(cfg, name, out["captures"][name]["kernel"][:60], m["gpu__time_duration.sum"], f"{dram / 1e6:.1f} MB")
    out["note"] = "ncu --set full --clock-control none, one launch each (scripts/prof_layer.py)"
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


def dram_csv(key, csv_path):
    """<workload>_<kernel> entry from one light ncu pass over EVERY launch of the
    kernel in a forward (--metrics dram__bytes_read.sum,dram__bytes_write.sum,
    gpu__time_duration.sum --csv --log-file ...): average DRAM bytes per launch."""
    lines = open(csv_path).read().split("\n")
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    idc, mn, mu, mv = h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    per = {}
    for r in rows[1:]:
        if len(r) > mv and r[mn].startswith("dram__bytes"):
            per[r[idc]] = per.get(r[idc], 0.0) + to_bytes(r[mv], r[mu])
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    out = json.load(open(path)) if os.path.exists(path) else {"captures": {}}
    out[key] = {"dram_bytes_per_launch": sum(per.values()) / max(len(per), 1), "launches": len(per),
                "capture": os.path.basename(csv_path)}
    print(key, out[key])
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "--dram-csv":  # python scripts/make_profiles.py --dram-csv c5_convw=gpurun_out/r02_c5_convw_dram.csv
        for a in sys.argv[2:]:
            dram_csv(*a.split("="))
    else:
        main(sys.argv[1], [a.split("=") for a in sys.argv[2:]])
