"""Hot SASS regions from an ncu --page source --print-source sass CSV:
instructions executed and stall samples per contiguous block."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si = h.index("Address"), h.index("Source")
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ai], 16), r[si].strip(), int(r[ie] or 0), int(r[ss] or 0)))
    except Exception:
        pass
base = data[0][0]
tot_i = sum(d[2] for d in data)
tot_s = sum(d[3] for d in data)
print("total instr %d  samples %d" % (tot_i, tot_s))
# group by blocks of N instructions
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
blocks = []
for i in range(0, len(data), N):
    ch = data[i:i + N]
    blocks.append((sum(c[2] for c in ch), sum(c[3] for c in ch), ch[0][0] - base, ch))
for bi, b in sorted(enumerate(blocks), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print("block @%05x  instr %5.1f%%  stalls %5.1f%%" % (b[2], 100 * b[0] / tot_i, 100 * b[1] / tot_s))
if len(sys.argv) > 4:
    off = int(sys.argv[4], 16)
    for d in data:
        if off <= d[0] - base < off + N * 16:
            print("%05x %10d %6d  %s" % (d[0] - base, d[2], d[3], d[1][:80]))
