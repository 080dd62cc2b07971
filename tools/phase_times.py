"""Per-phase durations of the fix-up kernel (tuning build variants/phases.so, -DFDTD_PHASES=1).

    FDTD_LIB=variants/phases.so python tools/phase_times.py [--workload cfg4]

Runs a few passes of the workload and reads the clock64() stamps thread 0 of every fix-up CTA took
at its phase barriers in the last launch; prints the mean cycles per phase and the CTA start / end
spread (waves)."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import numpy as np

    from inputs import configs
    from paper_1609_07114_b200 import from_scene, lib

    s = configs.make(a.workload, device="cuda")
    sim = from_scene(s, device=0, use_graphs=False)
    sim.record_energy(True)
    sim.step(8)
    sim.sync()
    n = 4096 * 72
    buf = (C.c_longlong * n)()
    lib().fdtd_debug_phases(buf, n)
    t = np.frombuffer(buf, dtype=np.int64).reshape(4096, 72)
    t = t[t[:, 0] != 0]  # the CTAs of the last launch that recorded stamps
    ncta = t.shape[0]
    k = (t[0] != 0).sum()
    t = t[:, :k].astype(np.float64)
    d = np.diff(t, axis=1)
    names = (["setup", "cp.async issue", "rom state", "consts+prefetch", "wait_all"] +
             ["H+M1", "gather+E", "energy+t", "schur", "M2+scatter"] * 4 + ["writeback+state"])  # FDTD_FUSE
    lines = ["fix-up phases (%s, %d CTAs, thread-0 clock64 at each barrier, last launch)" % (a.workload, ncta)]
    for i in range(d.shape[1]):
        nm = names[i] if i < len(names) else "p%d" % i
        lines.append("  %2d %-12s mean %8.0f cycles  p90 %8.0f" % (i, nm, d[:, i].mean(), np.percentile(d[:, i], 90)))
    tot = t[:, -1] - t[:, 0]
    start = t[:, 0] - t[:, 0].min()
    lines.append("  per CTA total mean %.0f cycles (%.1f us at 1.9 GHz); CTA start spread %.0f cycles" % (
        tot.mean(), tot.mean() / 1.9e3, start.max()))
    print("\n".join(lines))
    if a.out:
        open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
