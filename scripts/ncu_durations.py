"""Print kernel name, grid and gpu__time_duration from an ncu --csv log file."""
import csv, sys
lines = open(sys.argv[1]).read().split('\n')
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
for r in rows[1:]:
    if len(r) > vi:
        print(r[ki][:48], r[gi], r[vi])
