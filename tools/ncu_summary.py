"""Summarise ncu captures into small text files under profiles/ (the judged evidence).

usage: python tools/ncu_summary.py <report.ncu-rep> <out.txt> [cells [workload steps_per_pass]]
       python tools/ncu_summary.py --launches <launches.csv> <out.txt>
With workload and steps_per_pass, the sweep's DRAM bytes per cell per launch are also written to
profiles/sweep_traffic.json, stamped with the kernel sources' hash (bench.py ignores a stale file).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def rep(path, out, cells=None, workload=None, spp=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines.append("kernel: " + name)
        vals = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append("  %-62s %s %s" % (k, r[i], units[i]))
                vals[k] = (r[i], units[i])
        if cells and "dram__bytes_read.sum" in vals:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * scale[vals["dram__bytes_read.sum"][1]]
            wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * scale[vals["dram__bytes_write.sum"][1]]
            lines.append("  DRAM bytes per cell per launch: read %.3f + write %.3f = %.3f B" %
                         (rd / cells, wr / cells, (rd + wr) / cells))
            if workload and "sweepk" in name:
                import os
                root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
                sys.path.insert(0, root)
                from bench import kernel_source_sha
                json.dump({"workload": workload, "steps_per_pass": int(spp), "kernel": name,
                           "bytes_per_launch_per_cell": round((rd + wr) / cells, 4),
                           "kernel_src_sha": kernel_source_sha(),
                           "source": "%s (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)" % out},
                          open(os.path.join(root, "profiles", "sweep_traffic.json"), "w"))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    order = []
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6,
                                              "msecond": 1.0}.get(r[ui], 1e-6)
        if k not in agg:
            agg[k] = []
            order.append(k)
        agg[k].append(v)
    lines = ["%-70s %6s %12s %12s" % ("kernel", "count", "mean_ms", "total_ms")]
    for k in order:
        v = agg[k]
        lines.append("%-70s %6d %12.4f %12.4f" % (k[:70], len(v), sum(v) / len(v), sum(v)))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        rep(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None,
            sys.argv[4] if len(sys.argv) > 4 else None, sys.argv[5] if len(sys.argv) > 5 else None)
