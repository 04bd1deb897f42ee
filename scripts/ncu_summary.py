"""Summarize an ncu report: key metrics + hottest SASS by stall samples."""
import csv, subprocess, sys, io, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
vals = rows[2] if len(rows) > 2 else rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size"]
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            print(f"{w:75s} {vals[i]} {rows[1][i]}")
if "--tensor" in sys.argv:
    for i, h in enumerate(hdr):
        if "tensor" in h and "pct" in h:
            print(f"{h:75s} {vals[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h2 = srows[1]
i_s = h2.index("Warp Stall Sampling (All Samples)")
data = [r for r in srows[2:] if len(r) > i_s]
tot = sum(float(r[i_s] or 0) for r in data)
seg = collections.OrderedDict()
cur = "start"
for r in data:
    for key in ["SYNCS", "UTCIMMA", "UTCHMMA", "UTMALDG", "UBLKCP", "LDTM", "ATOMG", "BAR.SYNC", "EXIT"]:
        if key in r[1]:
            cur = key + "@" + r[0][-5:]
    seg[cur] = seg.get(cur, 0) + float(r[i_s] or 0)
print("total stall samples", tot)
for k, v in seg.items():
    if v > tot * 0.02:
        print(f"  {k:20s} {v:8.0f} {100*v/tot:5.1f}%")
top = sorted(data, key=lambda r: -float(r[i_s] or 0))[:12]
for r in top:
    print("  ", r[0][-5:], r[i_s].rjust(6), r[1][:100])

# instruction counts by region (warp-level instructions executed)
if "--inst" in sys.argv:
    i_n = h2.index("Instructions Executed")
    seg = collections.OrderedDict()
    cur = "start"
    tot = 0
    for r in data:
        for key in ["SYNCS", "UTCIMMA", "UTCHMMA", "UTMALDG", "UBLKCP", "LDTM", "BAR.SYNC", "UCGABAR", "EXIT"]:
            if key in r[1]:
                cur = key + "@" + r[0][-5:]
        n = float(r[i_n] or 0)
        tot += n
        seg[cur] = seg.get(cur, 0) + n
    print("total warp instructions", tot)
    for k, v in seg.items():
        if v > tot * 0.01:
            print(f"  {k:22s} {v:10.0f} {100*v/tot:5.1f}%")
    hot = sorted(data, key=lambda r: -float(r[i_n] or 0))[:25]
    for r in hot:
        print("  ", r[0][-5:], r[i_n].rjust(8), r[1][:90])

# stall reasons by region
if "--stalls" in sys.argv:
    cols = [c for c in h2 if c.startswith("stall_") and "Not Issued" not in c]
    idx = [h2.index(c) for c in cols]
    seg = collections.OrderedDict()
    cur = "start"
    for r in data:
        for key in ["SYNCS", "UTCIMMA", "UTCHMMA", "LDTM", "BAR.SYNC", "UCGABAR", "EXIT"]:
            if key in r[1]:
                cur = key + "@" + r[0][-5:]
        acc = seg.setdefault(cur, [0.0] * len(cols))
        for k, i in enumerate(idx):
            acc[k] += float(r[i] or 0)
    for name, acc in seg.items():
        t = sum(acc)
        if t < tot * 0.03:
            continue
        top = sorted(zip(cols, acc), key=lambda z: -z[1])[:5]
        print(f"  {name:20s} {t:7.0f}  " + ", ".join(f"{c[6:]}={v:.0f}" for c, v in top))
