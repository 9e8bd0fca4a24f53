"""Side-by-side of selected ncu raw metrics (and the stall breakdown) of one kernel in several
.ncu-rep files: python tools/ncu_cmp.py a.ncu-rep b.ncu-rep ..."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "sm__cycles_active.avg",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return dict(zip(r[0], r[2] if len(r) > 2 else r[1]))


ds = [load(p) for p in sys.argv[1:]]
print("%-72s" % "metric" + "".join("%18s" % p.split("/")[-1][:17] for p in sys.argv[1:]))
stalls = sorted({k for d in ds for k in d if "issue_stalled" in k and k.endswith("per_issue_active.ratio")},
                key=lambda k: -float(ds[0].get(k) or 0))
for k in KEYS + stalls[:12]:
    print("%-72s" % k[:72] + "".join("%18s" % (d.get(k) or "")[:17] for d in ds))
