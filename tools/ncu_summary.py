"""Key counters from ncu --page raw --csv exports (one column per file)."""
import csv, sys
KEYS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("sm__cycles_elapsed.avg.per_second", "SM GHz", 1e-9),
    ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
    ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "hmma %", 1),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe %", 1),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform %", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 thru %", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
    ("smsp__inst_executed.sum", "instr", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts", 1),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 wr sectors", 1),
    ("lts__t_requests_srcunit_tex_op_write.sum", "L2 wr requests", 1),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall lsb", 1),
]
cols = []
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    cols.append(d)
names = [f.split("/")[-1].split(".")[0] for f in sys.argv[1:]]
print("%-16s" % "" + "".join("%14s" % n[-13:] for n in names))
for k, lab, sc in KEYS:
    line = "%-16s" % lab
    for d in cols:
        v = d.get(k)
        try:
            line += "%14.2f" % (float(v.replace(",", "")) * sc)
        except Exception:
            line += "%14s" % "-"
    print(line)
