"""Per-opcode instruction mix of a kernel from an ncu report (sass__inst_executed_per_opcode_with_modifier_all),
normalised per unit of work.

usage: python tools/inst_mix.py <report.ncu-rep> <units> <unit name> [out.txt]
(the sweep: units = warp row-stages = MUFU.RCP count / 1, since stage 0 issues one rcp per edge pair)"""
import re
import subprocess
import sys


def main(rep, units, uname, out=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--print-metric-instances", "details"],
                         capture_output=True, text=True).stdout
    m = re.search(r"sass__inst_executed_per_opcode_with_modifier_all\s+([0-9.]+)\s+\((.*?)\)", txt, re.S)
    total = float(m.group(1))
    pairs = [p.strip() for p in " ".join(m.group(2).split()).split(";") if p.strip()]
    rows = []
    for p in pairs:
        k, _, v = p.rpartition(":")
        rows.append((k.strip(), float(v)))
    rows.sort(key=lambda t: -t[1])
    units = float(units)
    lines = ["%s: %d warp instructions, %.3g %s, %.2f per %s" % (rep.split("/")[-1], total, units, uname,
                                                                  total / units, uname.rstrip("s"))]
    for k, v in rows:
        if v / units >= 0.05:
            lines.append("  %-28s %14d  %6.2f  %5.1f %%" % (k, v, v / units, 100 * v / total))
    s = "\n".join(lines)
    print(s)
    if out:
        open(out, "w").write(s + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
