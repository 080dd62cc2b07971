"""Replay of the paper's Sec. VI-C four-rod reflection experiment (Fig. rods4) on the GPU.

66 mm x 40 mm waveguide (PEC top / bottom), uniform 1 mm coarse mesh, 15 mm CPML at both x-ends
(NEXT-2), four copper rods (radius 1 mm, sigma 5.8e7 S/m) at (41, 22), (41, 18), (45, 22), (45, 18) mm
inside the refined box x 39..47 mm, y 16..24 mm (8 x 8 coarse cells, r = 6, full order 7,008 as in
L945), read off the TikZ schematic (L958-1002).  A line source across the guide at x = 17 mm, a probe
line at x = 19 mm.  The refined box is embedded (a) at full order (the exact fine-grid model, V = I) and
(b) reduced by SPRIM (the paper reports 7,008 -> 1,920) with the CFL limit extended 3x; the run uses
0.99 x the limit of each (L945).  For each, a second run with the empty box (no rods) gives the incident
wave; the reflected signal at the probe line is the difference, and its spectrum relative to the
incident one is the reflection coefficient |R(f)| (the paper's reflected-power plot).  Reported: the
two |R(f)| curves over 2..30 GHz, their max difference, stability, and the fp64 parity of the first
steps against the oracle.  Writes a JSON summary (profiles/r01_rods4_replay.json).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import romgen as rg  # noqa: E402
from inputs import scene as sc  # noqa: E402

from inputs.rods4 import (BOX, DX, FMAX, NX, NY, PML, PROBE_X, R, ROD_R, RODS, SRC_X,  # noqa: E402,F401
                          fine_fill, scene)


def build_model(rods, reduced, q):
    eps, sig, _ = fine_fill(rods)
    i0, j0, bx, by = BOX
    sysf = rg.fine_system(bx, by, R, DX, DX, eps, sig)
    assert rg.full_order(sysf) == 7008
    cs = rg.collapse(sysf)
    if reduced:
        V1, V2 = rg.sprim_basis(cs, q, FMAX)
        m = rg.reduce(cs, V1, V2)
    else:
        m = rg.full_order_model(cs)
    dtf = rg.fine_cfl_limit(sysf)
    m["fine_dt_limit"] = dtf
    if reduced:
        m = rg.extend_cfl(m, 3.0 * dtf)  # "extended by 3 times" (L945)
    return m, dtf


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--time", type=float, default=2e-9, help="simulated time (s)")
    ap.add_argument("--q", type=int, default=1920)
    ap.add_argument("--check", type=int, default=500)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_rods4_replay.json"))
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    from helpers import gpu_from_scene, oracle_from_scene

    t0 = time.time()
    summary = dict(experiment="PAPER.md Sec. VI-C four copper rods in a CPML-terminated waveguide (L943-948)",
                   grid=[NX, NY], dx=DX, pml_cells=PML, box=list(BOX), r=R, full_order=7008, simulated_time=args.time)
    sig_ref, sig_rom = {}, {}
    freqs = np.linspace(2e9, FMAX, 57)
    F = lambda x, dt: np.abs(np.exp(-2j * np.pi * np.outer(freqs, np.arange(len(x)) * dt)) @ x)
    for rods in (True, False):
        tag = "rods" if rods else "empty"
        m, dtf = build_model(rods, True, args.q)
        # reference: the fine-grid solution itself (oracle direct subgridding = the exact full-order
        # model) at 0.99 x its CFL limit (the fine cells')
        dt_ref = 0.99 * dtf
        n_ref = int(math.ceil(args.time / dt_ref))
        sref = scene(m, dt_ref, n_ref)
        o = O.OracleSim(NX, NY, DX, DX, dt_ref, np.ones((NY, NX)), np.zeros((NY, NX)))
        o.set_pml(PML, 3, 1e-8)
        eps, sig, _ = fine_fill(rods)
        o.add_subgrid(BOX[0], BOX[1], BOX[2], BOX[3], R, eps, sig)
        o.set_source_line(SRC_X, 0, NY, sref.samples)
        o.set_probes(sref.probes)
        pref, _ = o.step(n_ref, energy=False)
        sig_ref[tag] = (pref.mean(axis=0), dt_ref)
        # proposed method: the SPRIM ROM (order q) with its CFL limit extended 3x, at 0.99 x that limit
        dt = 0.99 * min(sc.cfl_limit(DX, DX), 3.0 * dtf)
        n = int(math.ceil(args.time / dt))
        s = scene(m, dt, n)
        g = gpu_from_scene(s, record_capacity=n + 16)
        g.record_energy(True)
        if rods and args.check:
            oc = oracle_from_scene(s)
            po, eo = oc.step(args.check)
            g.step(args.check)
            pg, eg = g.probe(), g.energy()
            rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
            summary["parity_first_steps"] = dict(steps=args.check, probe=rel(pg, po), energy=rel(eg, eo))
            g.step(n - args.check)
            p = np.concatenate([pg, g.probe()], axis=1)
            e = np.concatenate([eg, g.energy()])
        else:
            g.step(n)
            p, e = g.probe(), g.energy()
        summary.setdefault("rom", {})[tag] = dict(q1=int(m["q1"]), q2=int(m["q2"]), n_clipped=int(m["n_clipped"]),
                                                  dt=dt, dt_over_fine_limit=dt / dtf, steps=n,
                                                  steps_per_pass=int(g.info().steps_per_pass),
                                                  finite=bool(np.all(np.isfinite(p))),
                                                  energy_last_over_max=float(e[-1] / e.max()))
        g.close()
        sig_rom[tag] = (p.mean(axis=0), dt)
        summary.setdefault("reference", {})[tag] = dict(dt=dt_ref, steps=n_ref)
    curves = {}
    for name, sg in (("reference_subgridding", sig_ref), ("reduced_rom", sig_rom)):
        (pr, dt), (pe, _) = sg["rods"], sg["empty"]
        curves[name] = F(pr - pe, dt) / np.maximum(F(pe, dt), 1e-300)
    cref, crom = curves["reference_subgridding"], curves["reduced_rom"]
    summary.update(freqs_ghz=(freqs / 1e9).tolist(), reflection_reference=cref.tolist(), reflection_rom=crom.tolist(),
                   max_abs_diff_reflection=float(np.abs(cref - crom).max()),
                   mean_abs_diff_reflection=float(np.abs(cref - crom).mean()),
                   mean_reflection_reference=float(cref.mean()), wall_s=time.time() - t0)
    print(json.dumps({k: v for k, v in summary.items() if k not in ("reflection_reference", "reflection_rom",
                                                                     "freqs_ghz")}, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(summary, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
