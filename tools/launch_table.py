"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) of
tools/cfg5_patch.py: the last network iteration, one line per launch."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
K = OrderedDict()
for r in rows[start + 1:]:
    K.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
L = list(K.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 36
tot = 0.0
for k in L[-n:]:
    t = k["gpu__time_duration.sum"] / 1e3
    tot += t
    rd, wr = k["dram__bytes_read.sum"] / 1e6, k["dram__bytes_write.sum"] / 1e6
    print("%-52s %8.1f us  rd %7.1f MB wr %7.1f MB  %5.2f TB/s" % (
        k["name"][:52], t, rd, wr, (rd + wr) / t / 1e6))
print("total %.1f us" % tot)
