"""The Sec. VI-C four-rod workload (Fig. rods4) as seeded input: geometry read off
the TikZ schematic (L958-1002), the fine fill of the refined box and the coarse scene (NEXT-2).

66 mm x 40 mm waveguide (PEC top / bottom), uniform 1 mm coarse mesh, 15 mm CPML at both x-ends,
four copper rods (radius 1 mm, sigma 5.8e7 S/m) at (41, 22), (41, 18), (45, 22), (45, 18) mm inside
the refined box x 39..47 mm, y 16..24 mm (8 x 8 coarse cells, r = 6, full order 7,008), a line source
across the guide at x = 17 mm and a probe line at x = 19 mm.  Input generation only (no method
arithmetic): used by the replay (tests/replays/rods4_replay.py) and the ROM-builder bench.
"""
from __future__ import annotations

import numpy as np

from inputs import scene as sc

NX, NY, DX = 66, 40, 1e-3
BOX = (39, 16, 8, 8)   # i0, j0, bx, by (coarse cells)
R = 6
RODS = [(41e-3, 22e-3), (41e-3, 18e-3), (45e-3, 22e-3), (45e-3, 18e-3)]
ROD_R = 1e-3
PML = 15
SRC_X, PROBE_X = 17, 19
FMAX = 30e9


def fine_fill(rods):
    i0, j0, bx, by = BOX
    N = bx * R
    fdx = DX / R
    eps = np.ones((N, N))
    sig = np.zeros((N, N))
    if rods:
        jj, ii = np.mgrid[0:N, 0:N]
        x = (i0 + (ii + 0.5) / R) * DX
        y = (j0 + (jj + 0.5) / R) * DX
        for cx, cy in RODS:
            sig[(x - cx) ** 2 + (y - cy) ** 2 <= ROD_R ** 2] = 5.8e7
    return eps, sig, fdx



def scene(model, dt, steps):
    eps = np.ones((NY, NX))
    sig = np.zeros((NY, NX))
    probes = np.array([[PROBE_X, j] for j in range(NY)], dtype=np.int32)
    return sc.Scene(name="rods4", nx=NX, ny=NY, dx=DX, dy=DX, dt=dt, eps_r=eps, sigma=sig, precision=64,
                    steps=steps, source=(SRC_X, 0), samples=sc.gaussian_samples(steps, dt, FMAX, derivative=False),
                    probes=probes, models=[model], placements=np.array([[0, BOX[0], BOX[1]]], dtype=np.int32),
                    meta=dict(pml=(PML, 3, 1e-8), source_rows=(0, NY)))
