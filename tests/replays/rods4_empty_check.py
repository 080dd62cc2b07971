"""Empty-box (no rods) check of the Sec. VI-C refined region: subgridding (oracle) vs the embedded
SPRIM ROM at several orders, unclipped, at 0.99 dt_f, T = 1 ns; the ROMs come from romgen (CPU) and
from fdtd_rom_build (GPU) and run on the GPU in fp64.  Prints the relative L2 difference of the line
probe to the subgridding run and the models' conditioning."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "replays"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import rods4_replay as r4  # noqa: E402
from helpers import gpu_from_scene  # noqa: E402
from inputs import romgen as rg  # noqa: E402
from inputs import scene as sc  # noqa: E402
from paper_1609_07114_b200 import build_rom  # noqa: E402

rods = len(sys.argv) > 1 and sys.argv[1] == "rods"
eps, sig, _ = r4.fine_fill(rods)
i0, j0, bx, by = r4.BOX
sysf = rg.fine_system(bx, by, r4.R, r4.DX, r4.DX, eps, sig)
cs = rg.collapse(sysf)
dtf = rg.fine_cfl_limit(sysf)
dt = 0.99 * dtf
n = int(math.ceil(1e-9 / dt))
o = O.OracleSim(r4.NX, r4.NY, r4.DX, r4.DX, dt, np.ones((r4.NY, r4.NX)), np.zeros((r4.NY, r4.NX)))
o.set_pml(r4.PML, 3, 1e-8)
o.add_subgrid(i0, j0, bx, by, r4.R, eps, sig)
samples = sc.gaussian_samples(n, dt, r4.FMAX, derivative=False)
o.set_source_line(r4.SRC_X, 0, r4.NY, samples)
o.set_probes(np.array([[r4.PROBE_X, j] for j in range(r4.NY)], np.int32))
ref, _ = o.step(n, energy=False)
ref = ref.mean(axis=0)
for q in (960, 1440, 1920):
    for who in ("cpu", "gpu"):
        if who == "cpu":
            V1, V2 = rg.sprim_basis(cs, q, r4.FMAX)
            m = rg.reduce(cs, V1, V2)
        else:
            m = build_rom(bx, by, r4.R, r4.DX, r4.DX, eps, sig, q, r4.FMAX)
        s = r4.scene(m, dt, n)
        g = gpu_from_scene(s, record_capacity=n + 16)
        g.step(n)
        p = g.probe().mean(axis=0)
        g.close()
        w = np.linalg.eigvalsh(m["R11"])
        print("rods" if rods else "empty", q, who, "q1 q2", m["q1"], m["q2"], "natural/dtf",
              rg.rom_cfl_limit(m) / dtf, "cond R11", w[-1] / w[0], "rel L2 vs subgridding",
              np.linalg.norm(p - ref) / np.linalg.norm(ref), flush=True)
