"""NEXT-3 measurement: GPU-side ROM construction (fdtd_rom_build) vs the CPU generator
(inputs/romgen.py) on the models of the bench workloads.

Per model: wall time of both builds (the GPU one after one warm-up build of a small model, so the
CUDA context exists), the builder's device-timed phases, and the largest relative difference of
the basis-invariant spectra (tests/test_gpu_rom_build.py) between the two models.
Writes profiles/r01_rom_build.json.  Run under gpurun:  python tools/rom_build_bench.py
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import romgen as rg  # noqa: E402
from inputs import scene as sc  # noqa: E402
from paper_1609_07114_b200 import build_rom  # noqa: E402

DX = DY = 1e-3


def spectra(m):
    ev = lambda A: np.sort(np.linalg.eigvalsh(0.5 * (A + A.T)))
    sv = lambda A: np.sort(np.linalg.svd(A, compute_uv=False))
    gen = np.sort(sla.eigh(0.5 * (m["F11"] + m["F11"].T), 0.5 * (m["R11"] + m["R11"].T), eigvals_only=True))
    return dict(R11=ev(m["R11"]), R22=ev(m["R22"]), F11=ev(m["F11"]), gen=gen, K=sv(m["K"]), L=sv(m["L"]),
                cfl=np.sort(rg.generalized_singular_values(m)))


def max_rel(a, b):
    sa, sb = spectra(a), spectra(b)
    return {k: float(np.abs(sa[k] - sb[k]).max() / max(np.abs(sb[k]).max(), 1e-300)) for k in sa}


def cases(which):
    out = []
    if "cfg4" in which:  # BASELINE config 4's model: 16 x 16 block, r = 4, disc inclusion, q 128, 2 dt_f
        fe, fs = sc.inclusion_fill(16, 4, 7)
        out.append(("cfg4 model (16x16, r 4, inclusion, q 128, clip 2 dt_f)", 16, 16, 4, fe, fs, 128, 10e9, 2.0, DX))
    if "cfg5" in which:  # config 5's largest model: 31 x 31 block, r = 10, q 256
        fe, fs = sc.uniform_fill(31, 31, 10, 510, 1.0, 12.0, 0.0, 0.2)
        out.append(("cfg5 largest model (31x31, r 10, q 256, clip 1 dt_f)", 31, 31, 10, fe, fs, 256, 10e9, None,
                    DX))
    if "rods4" in which:  # Sec. VI-C: 8 x 8 box, r = 6, copper rods, q 1920, 3x CFL extension
        from inputs import rods4 as r4
        fe, fs, _ = r4.fine_fill(True)
        out.append(("rods4 box (8x8, r 6, four copper rods, q 1920, clip 3 dt_f)", r4.BOX[2], r4.BOX[3], r4.R, fe, fs,
                    1920, r4.FMAX, 3.0, r4.DX))
    return out


def embedded_rods4(mg, mc, dtf3, steps=3000):
    """Probe series (line probe at x = 19 mm) of the four-rod waveguide with the GPU-built and the
    CPU-built model embedded (fp64 GPU runs, same scene): their relative L2 difference."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import gpu_from_scene
    from inputs import rods4 as r4
    dt = 0.99 * min(sc.cfl_limit(r4.DX, r4.DX), dtf3)
    out = []
    for m in (mc, mg):
        s = r4.scene(m, dt, steps)
        g = gpu_from_scene(s, record_capacity=steps + 16)
        g.step(steps)
        out.append(g.probe().mean(axis=0))
        g.close()
    return dict(steps=steps, dt=dt, probe_rel_l2=float(np.linalg.norm(out[1] - out[0]) / np.linalg.norm(out[0])))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg4,cfg5,rods4")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_rom_build.json"))
    args = ap.parse_args()
    fe, fs = sc.uniform_fill(2, 2, 2, 1, 1, 4, 0, 0.05)
    build_rom(2, 2, 2, DX, DY, fe, fs, 8, 30e9)  # context + module load
    fe, fs = sc.uniform_fill(4, 4, 3, 1, 1, 4, 0, 0.05)
    build_rom(4, 4, 3, DX, DY, fe, fs, 40, 30e9)  # ... and the cooperative Jacobi path
    res = []
    for name, bx, by, r, fe, fs, q, fmax, clip, dx in cases(args.cases.split(",")):
        t0 = time.perf_counter()
        sysf = rg.fine_system(bx, by, r, dx, dx, fe, fs)
        dtf = rg.fine_cfl_limit(sysf)
        t_dtf = time.perf_counter() - t0
        dt = clip * dtf if clip else None
        t0 = time.perf_counter()
        mg = build_rom(bx, by, r, dx, dx, fe, fs, q, fmax, dt_target=dt)
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        mc = rg.build_rom(bx, by, r, dx, dx, fe, fs, q, fmax, dt_target=dt)
        t_cpu = time.perf_counter() - t0
        errs = max_rel(mg, mc)
        if name.startswith("rods4"):  # embedded response: both models in the Sec. VI-C waveguide
            row_resp = embedded_rods4(mg, mc, dt)
        else:
            row_resp = None
        row = dict(model=name, fine_cells=bx * r * by * r, full_order=rg.full_order(sysf), q1=mg["q1"], q2=mg["q2"],
                   q1_cpu=mc["q1"], q2_cpu=mc["q2"], n_clipped=mg["n_clipped"], n_clipped_cpu=mc["n_clipped"],
                   gpu_s=t_gpu, cpu_s=t_cpu, cpu_threads=os.cpu_count(), speedup=t_cpu / t_gpu,
                   fine_dt_limit_cpu_s=t_dtf, gpu_phases_ms=mg["gpu_build"], max_rel_spectrum_diff=errs,
                   natural_dt_limit_ratio=mg["natural_dt_limit"] / mc["natural_dt_limit"],
                   embedded_response=row_resp)
        print(json.dumps(row), flush=True)
        res.append(row)
    with open(args.out, "w") as f:
        json.dump(dict(what="NEXT-3 GPU ROM construction vs inputs/romgen.py (CPU, scipy splu + LAPACK)",
                       cases=res), f, indent=1)


if __name__ == "__main__":
    main()
