"""Pins of the ROM input generator (inputs/romgen.py) and the scene generator (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest

from inputs import romgen as rg
from inputs import scene as sc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "paper_counts.json")))["cases"])
def test_full_order_counts_match_paper(case):
    """PAPER.md L840 / L882 / L945: full orders 7,600 / 2,760 / 7,008."""
    b, r = case["bx"], case["r"]
    n = b * r
    s = rg.fine_system(case["bx"], case["by"], r, 1e-3, 1e-3, np.ones((n, n)), np.zeros((n, n)))
    assert rg.full_order(s) == case["order"]


def _rand_fine(rng, bx, by, r, lossless=False):
    fe = rng.uniform(1, 10, (by * r, bx * r))
    fs = np.zeros_like(fe) if lossless else rng.uniform(0, 10, (by * r, bx * r))
    return fe, fs


def test_structural_identities():
    """eq:cond3 B = L S exactly (L708 'by direct substitution'); R = R^T; F + F^T = 0 if sigma = 0."""
    rng = np.random.default_rng(0)
    fe, fs = _rand_fine(rng, 3, 2, 3)
    s = rg.fine_system(3, 2, 3, 1e-3, 2e-3, fe, fs)
    dt = 0.5 * rg.fine_cfl_limit(s)
    R, F, B, L = rg.descriptor_matrices(s, dt)
    assert abs(R - R.T).max() == 0.0
    Sd = np.diag(s["S"])
    assert np.abs((B - L @ Sd)).max() == 0.0
    Shat = (L.T @ B).toarray()
    np.testing.assert_array_equal(Shat, Sd)               # eq:S: S^ = L^T B^
    nx, ny = 3 * 3, 2 * 3
    np.testing.assert_allclose(s["S"][:nx], -1e-3 / 3)     # S side: -dx^
    np.testing.assert_allclose(s["S"][nx:2 * nx], 1e-3 / 3)
    np.testing.assert_allclose(s["S"][2 * nx:2 * nx + ny], 2e-3 / 3)
    np.testing.assert_allclose(s["S"][2 * nx + ny:], -2e-3 / 3)
    s0 = rg.fine_system(3, 2, 3, 1e-3, 2e-3, fe, 0 * fs)
    _, F0, _, _ = rg.descriptor_matrices(s0, dt)
    assert abs(F0 + F0.T).max() == 0.0
    s2 = rg.fine_system(3, 2, 3, 1e-3, 2e-3, fe, 2 * fs)
    np.testing.assert_allclose(s2["f11"], 2 * s["f11"], rtol=1e-15)


@pytest.mark.parametrize("eps_r,dx,dy", [(1.0, 1e-3, 1e-3), (4.0, 1e-3, 1.7e-3), (2.5, 2e-3, 0.8e-3)])
def test_cfl_link_is_exact_for_homogeneous_regions(eps_r, dx, dy):
    """L708: eq:cond1 generalises the CFL limit; for a homogeneous fill 2/s_max == eq.(1) at (dx^, dy^)."""
    r = 4
    s = rg.fine_system(3, 2, r, dx, dy, np.full((2 * r, 3 * r), eps_r), np.zeros((2 * r, 3 * r)))
    c = rg.C0 / math.sqrt(eps_r)
    eq1 = 1.0 / (c * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    assert rg.fine_cfl_limit(s) == pytest.approx(eq1, rel=1e-12)


def test_cond1_fails_just_above_fine_limit():
    rng = np.random.default_rng(1)
    fe, fs = _rand_fine(rng, 2, 2, 3)
    s = rg.fine_system(2, 2, 3, 1e-3, 1e-3, fe, fs)
    dtf = rg.fine_cfl_limit(s)
    for f, ok in ((0.999, True), (1.001, False)):
        R, _, _, _ = rg.descriptor_matrices(s, f * dtf)
        lam = np.linalg.eigvalsh(R.toarray()).min()
        assert (lam > 0) == ok


@pytest.mark.parametrize("seed", range(6))
def test_theorem1_reduced_model_is_passive(seed):
    """Theorem 1 (L721-726): R~ > 0 at dt <= fine limit, F~ + F~^T >= 0, B~ = L~ S_c; V orthonormal."""
    rng = np.random.default_rng(100 + seed)
    bx, by, r = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(2, 5))
    fe, fs = _rand_fine(rng, bx, by, r)
    sysf = rg.fine_system(bx, by, r, 1e-3, 1e-3, fe, fs)
    cs = rg.collapse(sysf)
    q = int(rng.integers(4, 2 * cs["nY"] + 8))
    V1, V2 = rg.sprim_basis(cs, q, 20e9)
    np.testing.assert_allclose(V1.T @ V1, np.eye(V1.shape[1]), atol=1e-12)
    np.testing.assert_allclose(V2.T @ V2, np.eye(V2.shape[1]), atol=1e-12)
    m = rg.reduce(cs, V1, V2)
    dtf = rg.fine_cfl_limit(sysf)
    ok, lamR, lamF = rg.check_passivity(m, 0.99 * dtf)
    assert ok, (lamR, lamF)
    # B~ = V1^T B_c = V1^T [diag(Sc); 0] must equal L~ S_c (eq:cond3rom)
    Bt = V1[: cs["nY"], :].T * cs["Sc"][None, :]
    np.testing.assert_allclose(Bt, m["L"] * cs["Sc"][None, :], rtol=0, atol=1e-13 * np.abs(Bt).max())
    assert rg.rom_cfl_limit(m) >= dtf * (1 - 1e-9)  # congruence never lowers the limit


def test_collapse_is_exact_merge():
    """Pi merges the r boundary nodes of each coarse edge: capacitance sums, B_c = +-dx, L_c = I."""
    rng = np.random.default_rng(2)
    fe, fs = _rand_fine(rng, 2, 3, 4)
    s = rg.fine_system(2, 3, 4, 1e-3, 2e-3, fe, fs)
    c = rg.collapse(s)
    assert c["nY"] == 2 * 2 + 2 * 3
    np.testing.assert_allclose(c["Sc"], [-1e-3] * 2 + [1e-3] * 2 + [2e-3] * 3 + [-2e-3] * 3, rtol=1e-14)
    assert c["r11"].sum() == pytest.approx(s["r11"].sum(), rel=1e-14)
    assert c["nEc"] == s["nE"] - s["nP"] + c["nY"]


def test_clip_golden_example():
    """SPEC.md:L232 example of the eq:CFLgeneralized clip (L741-745)."""
    g = json.load(open(os.path.join(GOLD, "clip_example.json")))
    s = np.array(g["s"])
    m = dict(q1=2, q2=2, R11=np.eye(2), R22=np.eye(2), F11=np.zeros((2, 2)), K=np.diag(s), L=np.eye(2))
    out = rg.extend_cfl(m, g["dt_target"], g["margin"])
    np.testing.assert_allclose(rg.generalized_singular_values(out), g["expected"], rtol=1e-12)
    assert out["n_clipped"] == 1
    for k in ("R11", "R22", "F11", "L"):
        assert np.array_equal(out[k], m[k])


def test_clip_idempotent_noop_and_restores_passivity():
    rng = np.random.default_rng(3)
    fe, fs = _rand_fine(rng, 2, 2, 3)
    sysf = rg.fine_system(2, 2, 3, 1e-3, 1e-3, fe, fs)
    cs = rg.collapse(sysf)
    m = rg.reduce(cs, *rg.sprim_basis(cs, 2 * cs["nY"], 60e9))
    dtn = rg.rom_cfl_limit(m)
    same = rg.extend_cfl(m, 0.9 * dtn)
    assert same["n_clipped"] == 0 and np.array_equal(same["K"], m["K"])
    dtt = 2.5 * dtn
    c1 = rg.extend_cfl(m, dtt)
    c2 = rg.extend_cfl(c1, dtt)
    assert c1["n_clipped"] > 0
    np.testing.assert_allclose(c2["K"], c1["K"], rtol=0, atol=1e-14 * np.abs(c1["K"]).max())
    assert not rg.check_passivity(m, 0.99 * dtt)[0]
    assert rg.check_passivity(c1, 0.99 * dtt)[0]
    s0, s1 = rg.generalized_singular_values(m), rg.generalized_singular_values(c1)
    assert np.all(s1 <= s0 * (1 + 1e-12))


# ------------------------------------------------------------------ scene generator
def test_gaussian_pulse_ten_percent_point():
    """R15: the Gaussian spectrum at fmax is 10 % of DC (closed-form Fourier transform)."""
    fmax = 10e9
    tau = sc.pulse_tau(fmax)
    assert math.exp(-0.5 * (2 * math.pi * fmax * tau) ** 2) == pytest.approx(0.1, rel=1e-12)
    g = sc.gaussian_samples(4000, tau / 40, fmax)
    t = (np.arange(4000) + 0.5) * tau / 40
    assert g.max() == pytest.approx(1.0, abs=1e-3)
    assert abs(t[np.argmax(g)] - 4.5 * tau) < tau / 40


def test_placements_disjoint_and_slab_local():
    P = sc.place_blocks(256, 256, [(8, 8), (5, 5)], 60, seed=4, nslabs=8, forbid=[(128, 128)])
    occ = np.zeros((256, 256), int)
    for m, i0, j0 in P:
        b = (8, 5)[m]
        occ[j0 - 1:j0 + b + 1, i0 - 1:i0 + b + 1] += 1
        assert i0 >= 2 and j0 >= 2 and i0 + b <= 254 and j0 + b <= 254
        assert (j0 - 1) // 32 == (j0 + b) // 32
        assert not (i0 - 1 <= 128 <= i0 + b and j0 - 1 <= 128 <= j0 + b)
    assert occ.max() == 1


def test_smooth_field_range_and_correlation():
    f = sc.smooth_field(512, 512, 32, 1.0, 10.0, seed=9).numpy()
    assert f.min() >= 1.0 and f.max() <= 10.0
    g = (f - f.mean()) / f.std()
    c1 = np.mean(g * np.roll(g, 1, axis=1))
    c32 = np.mean(g * np.roll(g, 32, axis=1))
    assert c1 > 0.99 and 0.1 < c32 < 0.6
