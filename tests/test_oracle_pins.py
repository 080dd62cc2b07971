"""Pins of the fp64 oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it pins (PAPER.md line, equation label) and the
DESIGN.md reading it relies on.  None of them re-types the oracle's formulas:
they compare against closed forms, printed values, invariants, or an
independent route (direct subgridding, plain uniform Yee).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from inputs import romgen as rg
from inputs import scene as sc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
C0 = 299792458.0


def one_step_matrix(sim):
    """Assemble the one-step iteration matrix by stepping unit vectors (state: E, H, ROM xt)."""
    v0 = sim.state_vector()
    n = v0.size
    M = np.zeros((n, n))
    for k in range(n):
        e = np.zeros(n)
        e[k] = 1.0
        sim.set_state_vector(e)
        sim.step(1, probes=False, energy=False)
        M[:, k] = sim.state_vector()
    return M


def rho(M):
    return np.abs(np.linalg.eigvals(M)).max()


def discrete_omegas(nx, ny, dx, dy, dt, c=C0):
    """Yee dispersion in a PEC cavity: sin(w dt/2) = c dt sqrt(sin^2(m pi/2nx)/dx^2 + sin^2(n pi/2ny)/dy^2)."""
    out = []
    for m in range(nx):
        for n in range(ny):
            if m == 0 and n == 0:
                continue
            s = c * dt * math.sqrt(math.sin(m * math.pi / (2 * nx)) ** 2 / dx ** 2 +
                                   math.sin(n * math.pi / (2 * ny)) ** 2 / dy ** 2)
            out.append(2 * math.asin(s))
    return np.sort(np.array(out))


# ----------------------------------------------------------------- hand values
def test_hand_value_dH():
    g = json.load(open(os.path.join(GOLD, "hand_values.json")))["dH_from_Ex"]
    s = O.OracleSim(3, 3, g["dx"], g["dy"], g["dt"], 1.0, 0.0)
    Ex = np.zeros((4, 3))
    Ex[2, 1] = g["Ex_top"]   # top edge of cell (1,1)
    s.set_state(Ex=Ex)
    s.step(1, probes=False, energy=False)
    Hz = s.get_state()[2]
    assert Hz[1, 1] == pytest.approx(g["expected_dHz"], rel=g["rel_tol"])


def test_hand_value_dEx():
    g = json.load(open(os.path.join(GOLD, "hand_values.json")))["dEx_from_Hz"]
    s = O.OracleSim(3, 3, g["dx"], g["dy"], g["dt"], 1.0, 0.0)
    Hz = np.zeros((3, 3))
    Hz[1, 1] = g["Hz"]
    # the H half-step runs first; a zero-E state keeps Hz unchanged before the E half-step
    s.set_state(Hz=Hz)
    s.step(1, probes=False, energy=False)
    Ex = s.get_state()[0]
    assert Ex[2, 1] == pytest.approx(-g["expected_dEx"], rel=g["rel_tol"])  # edge above: -dt/(eps dy)
    assert Ex[1, 1] == pytest.approx(+g["expected_dEx"], rel=g["rel_tol"])  # edge below


def test_hand_value_lossy_decay():
    """eq:updateEx with zero curl: Ex' = (eps/dt - sig/2)/(eps/dt + sig/2) Ex, strictly < 1."""
    g = json.load(open(os.path.join(GOLD, "hand_values.json")))["ca_lossy"]
    eps = g["eps_r"] * O.EPS0
    ca = (eps / g["dt"] - g["sigma"] / 2) / (eps / g["dt"] + g["sigma"] / 2)
    nx, ny = 4, 6
    s = O.OracleSim(nx, ny, 1e-3, 1e-3, g["dt"], g["eps_r"], g["sigma"])
    Ex = np.zeros((ny + 1, nx))
    Ex[1:ny, :] = 1.0          # uniform Ex on all live rows: cells 1..ny-2 see zero curl
    s.set_state(Ex=Ex)
    s.step(1, probes=False, energy=False)
    Ex1 = s.get_state()[0]
    assert 0 < ca < 1
    np.testing.assert_allclose(Ex1[2:ny - 1, :], ca, rtol=1e-14)


def test_cfl_examples():
    g = json.load(open(os.path.join(GOLD, "hand_values.json")))["cfl_examples"]
    assert sc.cfl_limit(2e-3, 2e-3) == pytest.approx(g["dx2mm"], rel=g["rel_tol"])
    assert sc.cfl_limit(0.4e-3, 0.4e-3) == pytest.approx(g["dx0p4mm"], rel=g["rel_tol"])


# ----------------------------------------------------------------- stencil spectrum
def test_pec_cavity_spectrum_matches_yee_dispersion():
    """PAPER.md eq:updateH/eq:updateEx on a PEC cavity: eigen-angles are the discrete TE_mn omegas."""
    nx, ny, dx, dy = 7, 5, 1e-3, 1.3e-3
    dt = 0.9 * sc.cfl_limit(dx, dy)
    s = O.OracleSim(nx, ny, dx, dy, dt, 1.0, 0.0)
    lam = np.linalg.eigvals(one_step_matrix(s))
    ang = np.angle(lam)
    osc = np.sort(ang[ang > 1e-9])
    want = discrete_omegas(nx, ny, dx, dy, dt)
    assert osc.size == want.size
    np.testing.assert_allclose(osc, want, rtol=0, atol=1e-12)
    assert np.abs(lam).max() <= 1 + 1e-12


def test_lossy_uniform_modes_decay_by_ca():
    """Uniform lossy medium: each oscillatory mode's 2x2 map has det = ca, so |lambda|^2 = ca."""
    nx, ny, dx, dy = 6, 5, 1e-3, 1e-3
    dt = 0.9 * sc.cfl_limit(dx, dy, 2.0)
    eps_r, sig = 2.0, 0.3
    s = O.OracleSim(nx, ny, dx, dy, dt, eps_r, sig)
    lam = np.linalg.eigvals(one_step_matrix(s))
    osc = lam[np.abs(np.angle(lam)) > 1e-9]
    e = eps_r * O.EPS0
    ca = (e / dt - sig / 2) / (e / dt + sig / 2)
    np.testing.assert_allclose(np.abs(osc) ** 2, ca, rtol=1e-10)


def exact_grid_limit(nx, ny, dx, dy):
    return 1.0 / (C0 * math.sqrt(math.sin((nx - 1) * math.pi / (2 * nx)) ** 2 / dx ** 2 +
                                 math.sin((ny - 1) * math.pi / (2 * ny)) ** 2 / dy ** 2))


def test_cfl_dichotomy_spectral_radius():
    """eq.(1): bounded just below the limit; unstable just above the finite-grid exact limit."""
    nx = ny = 12
    dx = dy = 1e-3
    eq1 = sc.cfl_limit(dx, dy)
    ex = exact_grid_limit(nx, ny, dx, dy)
    assert 1.0 < ex / eq1 < 1.01
    s = O.OracleSim(nx, ny, dx, dy, 0.99 * eq1, 1.0, 0.0)
    assert rho(one_step_matrix(s)) <= 1 + 1e-12
    s = O.OracleSim(nx, ny, dx, dy, 1.01 * ex, 1.0, 0.0)
    assert rho(one_step_matrix(s)) > 1.05


def test_cfl_blowup_time_domain_40x40():
    """40x40 vacuum: bounded at 0.99 x eq.(1); blows up at 1.01 x eq.(1) (> exact limit 1.00077x)."""
    nx = ny = 40
    dx = dy = 1e-3
    eq1 = sc.cfl_limit(dx, dy)
    rng = np.random.default_rng(3)
    for f, grows in ((0.99, False), (1.01, True)):
        s = O.OracleSim(nx, ny, dx, dy, f * eq1, 1.0, 0.0)
        s.set_state(Hz=rng.standard_normal((ny, nx)))
        s.step(400, probes=False, energy=False)
        m = np.abs(s.get_state()[2]).max()
        if grows:
            assert m > 1e6
        else:
            assert m < 20


def test_te_mn_resonance_peak():
    """TE_10 of a 40 mm PEC cavity at 1 mm: the probe spectrum peaks at the discrete f_10."""
    nx = ny = 40
    dx = dy = 1e-3
    dt = 0.95 * sc.cfl_limit(dx, dy)
    s = O.OracleSim(nx, ny, dx, dy, dt, 1.0, 0.0)
    n = 20000
    s.set_source(3, 20, sc.gaussian_samples(n, dt, 30e9, derivative=True))
    s.set_probes([(36, 20)])
    pr, _ = s.step(n, energy=False)
    f10 = 2 * math.asin(C0 * dt * math.sin(math.pi / 80) / dx) / (2 * math.pi * dt)
    f = np.fft.rfftfreq(8 * n, dt)
    spec = np.abs(np.fft.rfft(pr[0] * np.hanning(n), 8 * n))
    band = (f > 0.5 * f10) & (f < 1.2 * f10)
    fpk = f[band][np.argmax(spec[band])]
    assert abs(fpk / f10 - 1) < 2e-3
    assert abs(f10 / (C0 / (2 * 0.04)) - 1) < 1e-3  # continuum (c/2a) within dispersion error


# ----------------------------------------------------------------- source / linearity
def test_superposition():
    nx, ny, dx, dy = 9, 8, 1e-3, 1e-3
    dt = 0.9 * sc.cfl_limit(dx, dy)
    rng = np.random.default_rng(5)
    eps, sig = rng.uniform(1, 3, (ny, nx)), rng.uniform(0, 0.1, (ny, nx))
    n = 200
    a, b = rng.standard_normal(n), rng.standard_normal(n)

    def run(g):
        s = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
        s.set_source(4, 4, g)
        s.set_probes([(1, 1), (7, 6)])
        return s.step(n, energy=False)[0]

    pa, pb, pab = run(a), run(b), run(a + b)
    np.testing.assert_allclose(pab, pa + pb, rtol=0, atol=1e-12 * np.abs(pab).max())


# ----------------------------------------------------------------- coupling pins
def _scene(seed=1, nx=10, ny=9, dx=1e-3, dy=1.2e-3):
    rng = np.random.default_rng(seed)
    return rng, nx, ny, dx, dy, rng.uniform(1, 4, (ny, nx)), rng.uniform(0, 0.05, (ny, nx))


def _run(sim, n, src=(2, 2)):
    k = np.arange(n)
    sim.set_source(*src, np.sin(k * 0.3) * np.exp(-((k - 40) / 15.0) ** 2))
    sim.set_probes([(7, 7), (1, 1), (8, 2)])
    pr, en = sim.step(n)
    return pr, sim.get_state(), en


def test_r1_full_order_rom_equals_uniform_yee():
    """SPEC acceptance 1: r=1, V=I reproduces the uniform grid (eq:sysform, collapsed R9)."""
    rng, nx, ny, dx, dy, eps, sig = _scene()
    dt = 0.9 / (C0 * math.sqrt(1 / dx ** 2 + 1 / dy ** 2))
    i0, j0, bx, by = 3, 3, 3, 2
    m = rg.build_rom(bx, by, 1, dx, dy, eps[j0:j0 + by, i0:i0 + bx], sig[j0:j0 + by, i0:i0 + bx], 0, 1e10, full=True)
    a = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    pa, sa, _ = _run(a, 1000)
    b = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    b.add_rom(m, i0, j0)
    pb, sb, _ = _run(b, 1000)
    assert np.abs(pa - pb).max() <= 1e-12 * np.abs(pa).max()
    hole = np.zeros((ny, nx), bool)
    hole[j0:j0 + by, i0:i0 + bx] = True
    assert np.abs(sa[2] - sb[2])[~hole].max() <= 1e-12 * np.abs(sa[2]).max()


def test_r1_subgrid_equals_uniform_yee():
    rng, nx, ny, dx, dy, eps, sig = _scene(2)
    dt = 0.9 / (C0 * math.sqrt(1 / dx ** 2 + 1 / dy ** 2))
    i0, j0, bx, by = 2, 4, 4, 3
    a = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    pa, _, _ = _run(a, 800)
    g = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    g.add_subgrid(i0, j0, bx, by, 1, eps[j0:j0 + by, i0:i0 + bx], sig[j0:j0 + by, i0:i0 + bx])
    pg, _, _ = _run(g, 800)
    assert np.abs(pa - pg).max() <= 1e-12 * np.abs(pa).max()


@pytest.mark.parametrize("r", [2, 3])
def test_full_order_rom_equals_direct_subgridding(r):
    """Full-order embedded model == brute-force subgridded solution (north_star pin)."""
    rng, nx, ny, dx, dy, eps, sig = _scene(3)
    i0, j0, bx, by = 3, 3, 3, 2
    fe, fs = rng.uniform(1, 4, (by * r, bx * r)), rng.uniform(0, 0.05, (by * r, bx * r))
    dt = 0.9 / (C0 * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    m = rg.build_rom(bx, by, r, dx, dy, fe, fs, 0, 1e10, full=True)
    b = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    b.add_rom(m, i0, j0)
    pb, sb, _ = _run(b, 1500)
    g = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    g.add_subgrid(i0, j0, bx, by, r, fe, fs)
    pg, sg, _ = _run(g, 1500)
    assert np.abs(pb - pg).max() <= 1e-12 * np.abs(pg).max()
    for x, y in zip(sb[:3], sg[:3]):
        assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max()


def consistent_random_state(sim, model, i0, j0, rng):
    """Q26: random live fields, holes/PEC zero, interface y = L~^T E~ for a random ROM state."""
    nx, ny = sim.nx, sim.ny
    Ex = rng.standard_normal((ny + 1, nx))
    Ey = rng.standard_normal((ny, nx + 1))
    Hz = rng.standard_normal((ny, nx)) / 377.0
    Ex[0] = Ex[ny] = 0
    Ey[:, 0] = Ey[:, nx] = 0
    bx, by, q1, q2 = model["bx"], model["by"], model["q1"], model["q2"]
    Hz[j0:j0 + by, i0:i0 + bx] = 0
    Ex[j0 + 1:j0 + by, i0:i0 + bx] = 0
    Ey[j0:j0 + by, i0 + 1:i0 + bx] = 0
    xt = rng.standard_normal(q1 + q2)
    xt[q1:] /= 377.0
    y = model["L"].T @ xt[:q1]
    Ex[j0, i0:i0 + bx] = y[:bx]
    Ex[j0 + by, i0:i0 + bx] = y[bx:2 * bx]
    Ey[j0:j0 + by, i0] = y[2 * bx:2 * bx + by]
    Ey[j0:j0 + by, i0 + bx] = y[2 * bx + by:]
    sim.set_state(Ex, Ey, Hz, xt)


@pytest.mark.parametrize("reduced", [False, True])
def test_energy_conserved_lossless_and_monotone_lossy(reduced):
    """Storage function (R17): exactly conserved when sigma == 0, non-increasing when lossy (Sec. V)."""
    rng, nx, ny, dx, dy, eps, sig = _scene(4)
    r, i0, j0, bx, by = 3, 3, 3, 3, 2
    fe, fs = rng.uniform(1, 4, (by * r, bx * r)), rng.uniform(0, 0.05, (by * r, bx * r))
    dt = 0.9 / (C0 * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    for lossy in (False, True):
        f = 1.0 if lossy else 0.0
        m = rg.build_rom(bx, by, r, dx, dy, fe, f * fs, 24, 30e9, full=not reduced)
        s = O.OracleSim(nx, ny, dx, dy, dt, eps, f * sig)
        s.add_rom(m, i0, j0)
        consistent_random_state(s, m, i0, j0, rng)
        _, en = s.step(1500, probes=False)
        if lossy:
            assert np.diff(en).max() <= 1e-13 * en[0]
            assert en[-1] < 0.9 * en[0]
        else:
            assert np.abs(en - en[0]).max() <= 1e-12 * en[0]


def test_energy_plain_grid_lossless():
    nx, ny, dx, dy = 16, 12, 1e-3, 1e-3
    rng = np.random.default_rng(7)
    eps = rng.uniform(1, 5, (ny, nx))
    s = O.OracleSim(nx, ny, dx, dy, 0.99 * sc.cfl_limit(dx, dy), eps, 0.0)
    Ex = rng.standard_normal((ny + 1, nx))
    Ey = rng.standard_normal((ny, nx + 1))
    Ex[0] = Ex[-1] = 0
    Ey[:, 0] = Ey[:, -1] = 0
    s.set_state(Ex, Ey, rng.standard_normal((ny, nx)) / 377)
    _, en = s.step(3000, probes=False)
    assert np.abs(en - en[0]).max() <= 1e-12 * en[0]


def test_scheme_stability_and_cfl_extension():
    """Sec. V-D/E: rho <= 1 at 0.99 dt_f; an unclipped ROM is unstable at 1.9 dt_f;
    after extend_cfl to 2 dt_f the scheme is stable at 1.9 dt_f (lossless fills)."""
    rng = np.random.default_rng(8)
    nx, ny, dx, dy, r = 8, 8, 1e-3, 1e-3, 3
    i0, j0, bx, by = 3, 3, 2, 2
    fe = rng.uniform(1, 3, (by * r, bx * r))
    fs = np.zeros_like(fe)
    m = rg.build_rom(bx, by, r, dx, dy, fe, fs, 60, 60e9)
    dtf = m["fine_dt_limit"]
    assert m["natural_dt_limit"] < 1.9 * dtf  # high order: the natural limit sits near dt_f

    def radius(model, dt):
        s = O.OracleSim(nx, ny, dx, dy, dt, 1.0, 0.0)
        s.add_rom(model, i0, j0)
        return rho(one_step_matrix(s))

    assert radius(m, 0.99 * dtf) <= 1 + 1e-10
    assert radius(m, 1.9 * dtf) > 1 + 1e-3
    mc = rg.extend_cfl(m, 2 * dtf)
    assert mc["n_clipped"] > 0
    assert radius(mc, 1.9 * dtf) <= 1 + 1e-10


@pytest.mark.slow
def test_rom_converges_to_subgridding_as_q_grows():
    """SPRIM ROMs approach the full-order (direct subgridding) solution as q grows (SURVEY Appendix A:
    8.3e-2 / 1.9e-2 / 1.4e-4 at q = 24 / 48 / 96 for this setup).  Pins the construction quality of
    the emitted models; the paper's own accuracy figures (Figs. 5/7/9) remain unpinned (no data)."""
    from inputs import configs
    nx = ny = 40
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(4, 4, 5, 11, 1, 4, 0, 0.05)
    sysf = rg.fine_system(4, 4, 5, dx, dy, fe, fs)
    dt = 0.95 * rg.fine_cfl_limit(sysf)
    n = 6000
    g = sc.gaussian_samples(n, dt, 10e9, derivative=True)

    def run(add):
        s = O.OracleSim(nx, ny, dx, dy, dt, 1.0, 0.0)
        add(s)
        s.set_source(8, 8, g)
        s.set_probes([(30, 30)])
        return s.step(n, energy=False)[0][0]

    ref = run(lambda s: s.add_subgrid(18, 18, 4, 4, 5, fe, fs))
    errs = []
    for q in (24, 48, 96):
        m = rg.build_rom(4, 4, 5, dx, dy, fe, fs, q, 10e9)
        p = run(lambda s: s.add_rom(m, 18, 18))
        errs.append(np.linalg.norm(p - ref) / np.linalg.norm(ref))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-2, errs


# ----------------------------------------------------------------- paper-literal coupling (NEXT-1)
@pytest.mark.parametrize("r", [2, 3])
def test_literal_full_order_rom_equals_direct_subgridding(r):
    """The paper's own coupling (eq:sysform with T and 1/r, nP = r nY fine hanging variables) at
    full order reproduces the brute-force subgridded solution (1.2e-15)."""
    rng, nx, ny, dx, dy, eps, sig = _scene(3)
    i0, j0, bx, by = 3, 3, 3, 2
    fe, fs = rng.uniform(1, 4, (by * r, bx * r)), rng.uniform(0, 0.05, (by * r, bx * r))
    dt = 0.9 / (C0 * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    m = rg.build_rom(bx, by, r, dx, dy, fe, fs, 0, 1e10, full=True, literal=True)
    assert m["literal"] and m["L"].shape[1] == r * (2 * bx + 2 * by)
    b = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    b.add_rom(m, i0, j0)
    pb, sb, _ = _run(b, 1500)
    g = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    g.add_subgrid(i0, j0, bx, by, r, fe, fs)
    pg, sg, _ = _run(g, 1500)
    assert np.abs(pb - pg).max() <= 1e-12 * np.abs(pg).max()
    for x, y in zip(sb[:3], sg[:3]):
        assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max()


def test_literal_coupling_singular_below_port_count():
    """SURVEY finding 1 / DESIGN R9: the literal A1 is singular when the ROM's E basis does not span
    the nP port directions (q1 < nP); with the port directions in the basis it is regular."""
    r, bx, by = 3, 3, 3
    nY, nP = 2 * bx + 2 * by, 3 * (2 * bx + 2 * by)
    rng, nx, ny, dx, dy, eps, sig = _scene(5, nx=12, ny=12)
    fe, fs = rng.uniform(1, 4, (by * r, bx * r)), np.zeros((by * r, bx * r))
    dt = 0.9 / (C0 * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    lsys = rg.literal_system(rg.fine_system(bx, by, r, dx, dy, fe, fs))
    V1, V2 = rg.sprim_basis(lsys, 24, 30e9)
    bad = rg.reduce(lsys, V1, V2)                        # q1 = 12 < nP = 36
    assert bad["q1"] < nP and bad["literal"]
    o = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    with pytest.raises(ValueError):
        o.add_rom(bad, 4, 4)
    good = rg.build_rom(bx, by, r, dx, dy, fe, fs, 24, 30e9, literal=True)
    assert good["q1"] >= nP
    O.OracleSim(nx, ny, dx, dy, dt, eps, sig).add_rom(good, 4, 4)


def test_literal_reduced_rom_energy_conserved():
    """Lossless scene with a reduced literal ROM (q1 >= nP): the storage function is conserved."""
    rng, nx, ny, dx, dy, eps, sig = _scene(6)
    r, i0, j0, bx, by = 2, 3, 3, 3, 2
    fe = rng.uniform(1, 4, (by * r, bx * r))
    dt = 0.9 / (C0 * math.sqrt(1 / (dx / r) ** 2 + 1 / (dy / r) ** 2))
    m = rg.build_rom(bx, by, r, dx, dy, fe, 0 * fe, 48, 30e9, literal=True)
    s = O.OracleSim(nx, ny, dx, dy, dt, eps, 0 * sig)
    s.add_rom(m, i0, j0)
    Ex = rng.standard_normal((ny + 1, nx)); Ey = rng.standard_normal((ny, nx + 1))
    Hz = rng.standard_normal((ny, nx)) / 377.0
    Ex[0] = Ex[ny] = 0; Ey[:, 0] = Ey[:, nx] = 0
    Hz[j0:j0 + by, i0:i0 + bx] = 0                       # hole; interface y = 0 = L~^T 0 (R26)
    Ex[j0:j0 + by + 1, i0:i0 + bx] = 0
    Ey[j0:j0 + by, i0:i0 + bx + 1] = 0
    s.set_state(Ex, Ey, Hz, np.zeros(m["q1"] + m["q2"]))
    _, en = s.step(1500, probes=False)
    assert np.abs(en - en[0]).max() <= 1e-11 * en[0]


# ----------------------------------------------------------------- CPML and line source (NEXT-2)
def _channel(nx, pml, src_i, probe_i, n=1400, ny=8):
    """Parallel-plate channel (PEC top / bottom): a full-height Hz line source launches the TEM wave."""
    dx = dy = 1e-3
    dt = 0.99 / (C0 * math.sqrt(2) / dx)
    o = O.OracleSim(nx, ny, dx, dy, dt, np.ones((ny, nx)), np.zeros((ny, nx)))
    if pml:
        o.set_pml(pml, 3, 1e-8)
    k = np.arange(n)
    tau = 2e-11
    o.set_source_line(src_i, 0, ny, np.exp(-((k * dt - 4.5 * tau) / tau) ** 2))
    o.set_probes(np.array([[probe_i, ny // 2]], np.int32))
    p, e = o.step(n)
    return p[0], e


def test_cpml_absorbs_the_tem_wave():
    """CPML (kappa 1, alpha 0, m = 3, R0 = 1e-8) on both ends: the wave leaves a 200-cell channel
    with a reflection below 1e-4 of the incident peak (reference: the same run in a 4000-cell
    channel, whose far ends are out of reach), while a PEC termination reflects it fully; the
    field energy then decays by more than 1e6."""
    ref, _ = _channel(4000, 0, 2000, 2010)
    pml, e = _channel(200, 15, 100, 110)
    pec, _ = _channel(200, 0, 100, 110)
    scale = np.abs(ref).max()
    assert np.abs(pml - ref).max() <= 1e-4 * scale
    assert np.abs(pec - ref).max() >= 0.5 * scale
    assert e[-1] <= 1e-6 * e.max()


def test_line_source_is_superposition_of_cells():
    """A line source on cells (i, j0 .. j1-1) equals the sum of the single-cell sources (linearity)."""
    rng, nx, ny, dx, dy, eps, sig = _scene(8)
    dt = 0.9 / (C0 * math.sqrt(1 / dx ** 2 + 1 / dy ** 2))
    k = np.arange(300)
    w = np.sin(k * 0.3) * np.exp(-((k - 40) / 15.0) ** 2)
    a = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
    a.set_source_line(4, 2, 6, w)
    a.step(300, probes=False, energy=False)
    tot = 0
    for j in range(2, 6):
        b = O.OracleSim(nx, ny, dx, dy, dt, eps, sig)
        b.set_source(4, j, w)
        b.step(300, probes=False, energy=False)
        tot = tot + b.get_state()[2]
    assert np.abs(a.get_state()[2] - tot).max() <= 1e-12 * np.abs(tot).max()
