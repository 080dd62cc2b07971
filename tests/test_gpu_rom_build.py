"""GPU-side ROM construction (NEXT-3, include/fdtdrom_build.h) vs the CPU generator
inputs/romgen.py (-m gpu).

The two build the same SPRIM subspace by different arithmetic (CG vs sparse LU for the shifted
solves, one-sided Jacobi vs LAPACK SVD), so their reduced matrices differ by an orthogonal change of
reduced basis V1 -> V1 Q1, V2 -> V2 Q2.  The tests therefore compare what such a change leaves
invariant: the orders, the spectra of R~11, R~22, F~11, R~11^-1 F~11, the singular values of K~, L~
and of R~11^-1/2 K~ R~22^-1/2 (the CFL quantity of eq:CFLgeneralized, L741-745), the clip count,
and the behaviour of the models embedded in a coarse grid (oracle runs of the same scene).
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from inputs import romgen as rg
from inputs import scene as sc
from paper_1609_07114_b200 import build_rom

from helpers import rel

pytestmark = pytest.mark.gpu

DX = DY = 1e-3


def _spectra(m):
    ev = lambda A: np.sort(np.linalg.eigvalsh(0.5 * (A + A.T)))
    sv = lambda A: np.sort(np.linalg.svd(A, compute_uv=False))
    gen = np.sort(sla.eigh(0.5 * (m["F11"] + m["F11"].T), 0.5 * (m["R11"] + m["R11"].T), eigvals_only=True))
    return dict(R11=ev(m["R11"]), R22=ev(m["R22"]), F11=ev(m["F11"]), gen=gen, K=sv(m["K"]), L=sv(m["L"]),
                cfl=np.sort(rg.generalized_singular_values(m)))


def _compare(mg, mc, tol):
    assert (mg["q1"], mg["q2"]) == (mc["q1"], mc["q2"])
    sg, scpu = _spectra(mg), _spectra(mc)
    errs = {}
    for k in sg:
        a, b = sg[k], scpu[k]
        scale = max(np.abs(b).max(), 1e-300)
        errs[k] = float(np.abs(a - b).max() / scale)
    assert max(errs.values()) <= tol, errs
    return errs


@pytest.mark.parametrize("case", ["uniform", "lossy_random", "inclusion", "r1", "strip", "aniso_odd_q"])
def test_gpu_build_matches_romgen_invariants(case):
    dx, dy = DX, DY
    if case == "aniso_odd_q":  # dx != dy (a swapped fdx / fdy shows) and an odd order
        bx, by, r, q = 4, 3, 3, 23
        dx, dy = 1e-3, 0.6e-3
        fe, fs = sc.uniform_fill(bx, by, r, 9, 1, 5, 0, 0.1)
    elif case == "uniform":
        bx, by, r, q = 3, 2, 3, 20
        fe, fs = sc.uniform_fill(bx, by, r, 1, 1, 4, 0, 0.05)
    elif case == "r1":  # no refinement: every port is one fine edge
        bx, by, r, q = 5, 3, 1, 12
        fe, fs = sc.uniform_fill(bx, by, r, 3, 1, 4, 0, 0.05)
    elif case == "strip":  # one coarse row, odd fine sizes (ragged multigrid levels)
        bx, by, r, q = 7, 1, 5, 24
        rng = np.random.default_rng(2)
        fe, fs = rng.uniform(1, 6, (by * r, bx * r)), rng.uniform(0, 0.1, (by * r, bx * r))
    elif case == "lossy_random":
        bx, by, r, q = 4, 3, 4, 32
        rng = np.random.default_rng(5)
        fe, fs = rng.uniform(1, 10, (by * r, bx * r)), rng.uniform(0, 0.5, (by * r, bx * r))
    else:
        bx = by = 6
        r, q = 4, 48
        fe, fs = sc.inclusion_fill(6, 4, 3)
    mc = rg.build_rom(bx, by, r, dx, dy, fe, fs, q, 30e9)
    mg = build_rom(bx, by, r, dx, dy, fe, fs, q, 30e9)
    _compare(mg, mc, 1e-8)
    assert abs(mg["natural_dt_limit"] / mc["natural_dt_limit"] - 1) < 1e-8
    ok, _, _ = rg.check_passivity(mg, 0.95 * mc["fine_dt_limit"])
    assert ok


def test_gpu_build_cfl_extension_matches():
    """eq:CFLgeneralized clip at 3 dt_f: same clip count and the same clipped spectrum."""
    bx = by = 4
    r, q = 4, 120  # natural limit 2.3 dt_f: the clip is active
    fe, fs = sc.uniform_fill(bx, by, r, 2, 1, 6, 0, 0.1)
    mc0 = rg.build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9)
    dt = 3.0 * mc0["fine_dt_limit"]
    mc = rg.extend_cfl(mc0, dt)
    mg = build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9, dt_target=dt)
    assert mc["n_clipped"] > 0 and mg["n_clipped"] == mc["n_clipped"]
    _compare(mg, mc, 1e-8)
    assert rg.rom_cfl_limit(mg) >= dt * (1 - 1e-9)
    ok, _, _ = rg.check_passivity(mg, 0.99 * dt)
    assert ok


def test_gpu_built_model_embedded_matches_cpu_built():
    """Both models embedded in the same lossy coarse grid (fp64 oracle, 300 steps): the probe
    series agree to 1e-9 (the reduced-basis rotation leaves the coupled scheme's response
    unchanged)."""
    import oracle as O
    bx = by = 4
    r, q = 3, 24
    fe, fs = sc.uniform_fill(bx, by, r, 4, 1, 4, 0, 0.05)
    mc = rg.build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9)
    mg = build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9)
    nx = ny = 40
    rng = np.random.default_rng(9)
    eps, sig = rng.uniform(1, 3, (ny, nx)), rng.uniform(0, 0.02, (ny, nx))
    dt = 0.95 * min(mc["fine_dt_limit"], sc.cfl_limit(DX, DY))
    out = []
    for m in (mc, mg):
        o = O.OracleSim(nx, ny, DX, DY, dt, eps, sig)
        o.add_rom(m, 18, 18)
        o.set_source(10, 10, sc.gaussian_samples(300, dt, 30e9, True))
        o.set_probes(np.array([[30, 30], [22, 14], [17, 20]], np.int32))
        p, e = o.step(300)
        out.append((p, e))
    assert np.abs(out[0][0]).max() > 0
    assert rel(out[1][0], out[0][0]) <= 1e-9
    assert rel(out[1][1], out[0][1]) <= 1e-9


def test_gpu_build_errors():
    from paper_1609_07114_b200 import FDTDError
    fe, fs = sc.uniform_fill(2, 2, 2, 1, 1, 4, 0, 0.05)
    with pytest.raises(FDTDError):
        build_rom(2, 2, 2, DX, DY, -fe, fs, 8, 30e9)
    with pytest.raises(FDTDError):
        build_rom(2, 2, 2, DX, DY, fe, fs, 1, 30e9)


def test_gpu_build_literal_ports_matches_romgen():
    """NEXT-1 models built on the GPU: the paper-literal nP-port basis ([port directions | SPRIM
    directions] in order).  Same invariants as the collapsed form, L~ of size q1 x nP, and the
    embedded response (oracle, literal coupling) to 1e-9."""
    import oracle as O
    bx, by, r, q = 3, 3, 3, 16
    fe, fs = sc.uniform_fill(bx, by, r, 6, 1, 4, 0, 0.05)
    mc = rg.build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9, literal=True)
    mg = build_rom(bx, by, r, DX, DY, fe, fs, q, 30e9, literal=True)
    nP = 2 * (bx + by) * r
    assert mg["literal"] and mg["L"].shape == (mg["q1"], nP) and mg["q1"] == nP + q // 2
    _compare(mg, mc, 1e-8)
    nx = ny = 30
    rng = np.random.default_rng(3)
    eps, sig = rng.uniform(1, 3, (ny, nx)), rng.uniform(0, 0.02, (ny, nx))
    dt = 0.95 * min(rg.fine_cfl_limit(rg.fine_system(bx, by, r, DX, DY, fe, fs)), sc.cfl_limit(DX, DY))
    out = []
    for m in (mc, mg):
        o = O.OracleSim(nx, ny, DX, DY, dt, eps, sig)
        o.add_rom(m, 13, 13)
        o.set_source(6, 6, sc.gaussian_samples(250, dt, 30e9, True))
        o.set_probes(np.array([[22, 22], [16, 10]], np.int32))
        out.append(o.step(250)[0])
    assert rel(out[1], out[0]) <= 1e-9


def test_gpu_build_order_beyond_full_order():
    """q larger than the full order: the Krylov space is exhausted and both builders return the
    full order (q1 = nEc, q2 = nH), i.e. an exact model."""
    fe, fs = sc.uniform_fill(2, 2, 2, 1, 1, 4, 0, 0.05)
    mc = rg.build_rom(2, 2, 2, DX, DY, fe, fs, 200, 30e9)
    mg = build_rom(2, 2, 2, DX, DY, fe, fs, 200, 30e9)
    assert (mg["q1"], mg["q2"]) == (mc["q1"], mc["q2"]) == (32, 16)
    _compare(mg, mc, 1e-8)
