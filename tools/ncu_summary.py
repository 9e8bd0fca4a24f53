#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  python tools/ncu_summary.py report <file.ncu-rep> <out_prefix> [--config cfg3] [--bytes-per-launch B]
      → <out_prefix>.txt (key metrics) and <out_prefix>.json (what bench.py reads for `traffic`)
  python tools/ncu_summary.py launches <launches.csv> <out.txt>
      → per-kernel launch counts, total/avg device time and share of the listed time
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "gpc__cycles_elapsed.max.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__block_size",
        "launch__grid_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__cycles_active.avg",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct", "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1}


def report(rep, prefix, config=None, bpl=None):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, js = [], {"source": rep, "config": config, "launches": []}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        out.append("kernel: %s  grid %s block %s" % (name, d.get("Grid Size"), d.get("Block Size")))
        rec = {"kernel": name}
        for k in KEYS:
            if k in d:
                u = units[hdr.index(k)]
                out.append("  %-75s %s %s" % (k, d[k], u))
                try:
                    rec[k] = float(d[k].replace(",", "")) * SCALE.get(u, 1)
                except ValueError:
                    pass
        tr = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
        rec["traffic_bytes"] = tr
        out.append("  traffic (dram read+write) %.6g B" % tr)
        if bpl:
            rec["algorithmic_bytes"] = bpl
            out.append("  algorithmic bytes per launch %.6g B  → traffic/algorithmic = %.4f" % (bpl, tr / bpl))
        js["launches"].append(rec)
    open(prefix + ".txt", "w").write("\n".join(out) + "\n")
    json.dump(js, open(prefix + ".json", "w"), indent=1)
    print("\n".join(out))


def launches(path, outp):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    tot = {}
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1e-9 if d["Metric Unit"] == "ns" else 1)
        tot.setdefault(name, [0.0, 0])
        tot[name][0] += v
        tot[name][1] += 1
    T = sum(v[0] for v in tot.values())
    lines = ["# per-kernel device time from `ncu --metrics gpu__time_duration.sum --clock-control none` "
             "(cold-cache, serialised: compare shares)", "# source: " + path]
    for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
        lines.append("%-50s launches=%5d total=%12.3f ms avg=%10.4f ms share=%.4f" %
                     (k[:50], v[1], v[0] * 1e3, v[0] / v[1] * 1e3, v[0] / T))
    open(outp, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "report":
        cfg = None
        bpl = None
        a = sys.argv[4:]
        if "--config" in a:
            cfg = a[a.index("--config") + 1]
        if "--bytes-per-launch" in a:
            bpl = float(a[a.index("--bytes-per-launch") + 1])
        report(sys.argv[2], sys.argv[3], cfg, bpl)
    else:
        launches(sys.argv[2], sys.argv[3])
