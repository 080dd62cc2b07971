"""NEXT-2 measurement: cost of the CPML band fix-up on a long fp32 waveguide.

Grid nx x ny (default 32768 x 4096) of a random lossy medium with a line source, timed with and
without 15-cell CPML layers on both x-ends (same grid, same K = 4 passes); the per-pass sweep and
band-kernel times come from the library's profiling events.  Writes one JSON line (stdout and
--out).  Run under gpurun:  python tools/pml_bench.py
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import scene as sc  # noqa: E402
from paper_1609_07114_b200 import Simulation  # noqa: E402


def run(nx, ny, steps, pml):
    import time
    rng = np.random.default_rng(1)
    eps = rng.uniform(1, 4, (ny, nx)).astype(np.float32)
    sig = rng.uniform(0, 0.02, (ny, nx)).astype(np.float32)
    dx = 1e-3
    dt = 0.95 * sc.cfl_limit(dx, dx)
    sim = Simulation(nx, ny, dx, dx, dt, eps, sig, precision=32)
    if pml:
        sim.set_pml(15, 3, 1e-8)
    sim.set_source_line(40, 0, ny, sc.gaussian_samples(steps + 64, dt, 30e9, False))
    sim.record_energy(True)
    sim.step(16)  # warm-up (graphs, pass depth)
    sim.sync()
    sim.energy()
    t0 = time.perf_counter()
    sim.step(steps)
    sim.sync()  # the library stream, device-synchronised
    ms = (time.perf_counter() - t0) * 1e3 / steps
    sim.energy()
    sim.profile(True)
    sim.step(32)
    sw, post, n = sim.profile_read()
    sim.profile(False)
    sim.close()
    return ms, sw / max(n, 1), post / max(n, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=32768)
    ap.add_argument("--ny", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_pml_bench.json"))
    a = ap.parse_args()
    ms0, sw0, po0 = run(a.nx, a.ny, a.steps, False)
    ms1, sw1, po1 = run(a.nx, a.ny, a.steps, True)
    cells = a.nx * a.ny
    row = dict(what="NEXT-2 CPML band fix-up cost (fp32, K = 4 passes, energy every step, line source)",
               grid=[a.nx, a.ny], pml_cells=15, steps=a.steps,
               ms_per_step_no_pml=ms0, ms_per_step_pml=ms1,
               cell_updates_per_s_no_pml=cells / ms0 * 1e3, cell_updates_per_s_pml=cells / ms1 * 1e3,
               pml_overhead=ms1 / ms0 - 1.0,
               per_pass_ms=dict(no_pml=dict(sweep=sw0, after_sweep=po0), pml=dict(sweep_and_bands=sw1,
                                                                                   after_sweep=po1)))
    print(json.dumps(row))
    with open(a.out, "w") as f:
        json.dump(row, f, indent=1)


if __name__ == "__main__":
    main()
