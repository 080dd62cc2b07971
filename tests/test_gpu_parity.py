"""CUDA path vs the fp64 oracle on identical seeded inputs (-m gpu).

Tolerances (BASELINE.json north_star): fp64 relative L2 <= 1e-10 on probe series
and final fields; fp32 relative L2 <= 1e-4 over the first 2000 steps, with the
energy never increasing by more than 1e-6 relative per step when source-free.
"""
import numpy as np
import pytest

from inputs import configs
from inputs import romgen as rg
from inputs import scene as sc

from helpers import consistent_random_state, gpu_from_scene, instance_pairs, oracle_from_scene, per_instance_errors, rel

pytestmark = pytest.mark.gpu


def _compare(scene, n, tol, energy=True, random_init=None, tuning=None, **kw):
    g = gpu_from_scene(scene, **kw)
    o = oracle_from_scene(scene)
    if tuning:
        g.set_tuning(*tuning)
    if random_init is not None:
        Ex, Ey, Hz, xs = consistent_random_state(scene, random_init)
        g.set_window(0, 0, Ex, Ey, Hz)
        o.set_state(Ex, Ey, Hz, xs if xs.size else None)
        if xs.size:
            g.set_rom_state(xs)
    g.record_energy(energy)
    g.step(n)
    pg, eg = g.probe(), g.energy()
    Exg, Eyg, Hzg = g.get_window()
    xg = g.get_rom_state()
    po, eo = o.step(n, energy=energy)
    Exo, Eyo, Hzo, xo = o.get_state()
    errs = dict(probe=rel(pg, po), Ex=rel(Exg, Exo), Ey=rel(Eyg, Eyo), Hz=rel(Hzg, Hzo))
    maxabs = {}
    if xo.size:
        errs["rom"] = rel(xg, xo)
        # per instance: x~ and the interface values y, each against its own norm (a global norm
        # would hide one bad instance among many); max-abs within 10x the L2 bar
        px, py = instance_pairs(scene, (Exg, Eyg, Hzg), (Exo, Eyo, Hzo), xg, xo)
        errs["rom_inst"], maxabs["rom_inst"] = per_instance_errors(px)
        errs["y_inst"], maxabs["y_inst"] = per_instance_errors(py)
    if energy:
        errs["energy"] = rel(eg, eo)
    g.close()
    print("errs", errs, "per-instance max-abs", maxabs)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    bad.update({k: v for k, v in maxabs.items() if not v <= 10 * tol})
    assert not bad, (errs, maxabs)
    return errs, (eg if energy else None)


@pytest.mark.parametrize("name", ["cfg1", "cfg1b", "cfg1c"])
def test_cfg1_full_fp64(name):
    """Config 1 in full (4000 steps, fp64): <= 1e-10 on probes, fields, ROM state and energy."""
    s = configs.make(name)
    _compare(s, s.steps, 1e-10)


def test_cfg1_random_init_fp64():
    s = configs.make("cfg1")
    _compare(s, 1500, 1e-10, random_init=11)


def _ragged_scene(nx, ny, precision, seed=3, rom=True):
    rng = np.random.default_rng(seed)
    eps = rng.uniform(1, 4, (ny, nx))
    sig = rng.uniform(0, 0.05, (ny, nx))
    dx, dy = 1e-3, 1.3e-3
    models, placements = [], None
    dt = 0.95 * sc.cfl_limit(dx, dy)
    if rom:
        fe, fs = sc.uniform_fill(3, 2, 3, seed + 1, 1, 4, 0, 0.05)
        m = rg.build_rom(3, 2, 3, dx, dy, fe, fs, 20, 30e9)
        fe2, fs2 = sc.uniform_fill(2, 2, 4, seed + 2, 1, 4, 0, 0.05)
        m2 = rg.build_rom(2, 2, 4, dx, dy, fe2, fs2, 16, 30e9)
        dt = 0.95 * min(m["fine_dt_limit"], m2["fine_dt_limit"])
        models = [m, m2]
        placements = np.array([[0, 4, 5], [1, nx - 8, ny - 7], [0, nx // 2, 3]], dtype=np.int32)
    steps = 600
    return sc.Scene(name="ragged", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=eps, sigma=sig, precision=precision,
                    steps=steps, source=(nx // 3, ny // 2), samples=sc.gaussian_samples(steps, dt, 30e9, True),
                    probes=np.array([[1, 1], [nx - 2, ny - 2], [nx // 2, ny // 2 + 1]], dtype=np.int32),
                    models=models, placements=placements)


@pytest.mark.parametrize("nx,ny", [(37, 29), (130, 61), (64, 64), (5, 7)])
def test_ragged_fp64(nx, ny):
    """Ragged widths (not multiples of the 16-byte vector or the warp strip), several tiles."""
    s = _ragged_scene(nx, ny, 64, rom=nx >= 30)
    _compare(s, s.steps, 1e-10, random_init=5)


@pytest.mark.parametrize("tuning", [(1, 1), (3, 2), (7, 8), (64, 4), (256, 4), (512, 2)])
def test_tuning_is_bitwise_invariant(tuning):
    """Chunk-start and warp-edge recomputation are bit-identical to the owner's values; chunks of >= 256
    rows take the four-row loop body of the fp32 K = 4 sweep (K1)."""
    s = _ragged_scene(301, 203, 32)
    base = gpu_from_scene(s)
    Ex, Ey, Hz, xs = consistent_random_state(s, 9)
    base.set_window(0, 0, Ex, Ey, Hz)
    base.set_rom_state(xs)
    base.step(50)
    ref = base.get_window()
    t = gpu_from_scene(s)
    t.set_tuning(*tuning)
    t.set_window(0, 0, Ex, Ey, Hz)
    t.set_rom_state(xs)
    t.step(50)
    got = t.get_window()
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    assert np.array_equal(t.get_rom_state(), base.get_rom_state())


def test_graph_and_eager_paths_agree():
    s = _ragged_scene(96, 80, 32)
    a = gpu_from_scene(s, use_graphs=True)
    b = gpu_from_scene(s, use_graphs=False)
    for sim in (a, b):
        sim.record_energy(True)
        sim.step(3)
        sim.step(120)
        sim.step(1)
    for x, y in zip(a.get_window(), b.get_window()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.probe(), b.probe())
    assert np.array_equal(a.energy(), b.energy())


@pytest.mark.parametrize("name,n", [("cfg2", 256), ("cfg3", 512), ("cfg4", 1024)])
def test_fp32_crops_2000_steps(name, n):
    """Seeded cropped sub-instances of configs 2, 3 and 4 (the headline config: 1024^2 with 4
    instances of its q = 128 model), fp32, first 2000 steps: <= 1e-4, per instance too."""
    s = configs.make(name, n=n)
    if name == "cfg4":
        assert len(s.placements) >= 4 and s.models[0]["q1"] + s.models[0]["q2"] == 128
    _compare(s, 2000, 1e-4, random_init=None if name == "cfg2" else 7)


@pytest.mark.parametrize("name,n", [("cfg3", 256), ("cfg4", 1024)])
def test_fp32_energy_non_increasing_source_free(name, n):
    """Q24: source-free, the fp32 GPU trace never rises by more than 1e-6 relative per step."""
    s = configs.make(name, n=n)
    g = gpu_from_scene(s, source=False)
    Ex, Ey, Hz, xs = consistent_random_state(s, 21)
    g.set_window(0, 0, Ex, Ey, Hz)
    g.set_rom_state(xs)
    g.record_energy(True)
    g.step(2000)
    e = g.energy()
    assert np.all(np.diff(e) <= 1e-6 * e[:-1]), np.max(np.diff(e) / e[:-1])
    assert e[-1] < e[0]


def test_fp32_lossless_energy_conserved():
    """sigma == 0 everywhere (coarse and fine): W^n is conserved up to fp32 roundoff."""
    nx = ny = 192
    dx = dy = 1e-3
    fe, fs = sc.inclusion_fill(6, 4, seed=2)
    m = rg.build_rom(6, 6, 4, dx, dy, fe, 0 * fs, 48, 10e9)
    dt = 1.9 * m["fine_dt_limit"]
    m = rg.extend_cfl(m, 2 * m["fine_dt_limit"])
    P = sc.place_blocks(nx, ny, [(6, 6)], 40, seed=3, nslabs=1)
    rng = np.random.default_rng(1)
    s = sc.Scene(name="lossless", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 3, (ny, nx)),
                 sigma=np.zeros((ny, nx)), precision=32, steps=0, source=(0, 0), samples=np.zeros(1),
                 probes=np.array([[5, 5]], dtype=np.int32), models=[m], placements=P)
    g = gpu_from_scene(s, source=False)
    Ex, Ey, Hz, xs = consistent_random_state(s, 4)
    g.set_window(0, 0, Ex, Ey, Hz)
    g.set_rom_state(xs)
    g.record_energy(True)
    g.step(2000)
    e = g.energy()
    assert np.max(np.abs(e - e[0])) <= 1e-5 * e[0]
    assert np.all(np.diff(e) <= 1e-6 * e[:-1])


@pytest.mark.parametrize("which", ["cfg1", "ragged", "cfg3crop", "lossless"])
def test_k_step_passes_bitwise_equal_one_step(which):
    """Temporal blocking (K = 2, 4 steps per pass + per-instance fix-up) reproduces the one-step
    path bit for bit: fields, ROM states and probes (energy up to summation order).  Step counts
    that are not multiples of K exercise the shallower remainder passes."""
    if which == "cfg1":
        s = configs.make("cfg1")
    elif which == "ragged":
        s = _ragged_scene(130, 61, 32)
        s.placements = s.placements[[0, 1]]  # keep the two that leave a 3-cell region inside the grid
    elif which == "cfg3crop":
        s = configs.make("cfg3", n=512)
    else:
        s = configs.make("cfg3", n=256)
        s.sigma = np.zeros((s.ny, s.nx))
    # deepest valid pass: fp64 vectors hold 2 columns (the ragged scene's instances sit 4-5 cells
    # from the walls: their fix-up regions reach beyond the walls, where they hold dead cells)
    kmax = 2 if s.precision == 64 else 4
    runs = []
    for spp in (1, 2, 4):
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        Ex, Ey, Hz, xs = consistent_random_state(s, 13)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.record_energy(True)
        for n in (1, 2, 3, 5, 8, 40, 1, 7):
            g.step(n)
        assert g.info().steps_per_pass == min(spp, kmax), (which, spp)
        runs.append((g.get_window(), g.get_rom_state(), g.probe(), g.energy()))
        g.close()
    w1, x1, p1, e1 = runs[0]
    for (w2, x2, p2, e2) in runs[1:]:
        for a, b in zip(w1, w2):
            assert np.array_equal(a, b), which
        assert np.array_equal(x1, x2)
        assert np.array_equal(p1, p2)
        np.testing.assert_allclose(e2, e1, rtol=1e-12 if s.precision == 64 else 2e-6)


def _cfg5_sub():
    return configs.make("cfg5", n=1024, max_fine=100, min_count=24)


def test_cfg5_subinstance_fp32_2000_steps():
    """Config 5 recipe (12 distinct ROM models, q 32..256, nY up to 64): <= 1e-4 over 2000 steps."""
    s = _cfg5_sub()
    assert len({(m["bx"], m["q1"]) for m in s.models}) >= 8
    _compare(s, 2000, 1e-4, random_init=17)


def test_cfg5_k_step_bitwise_and_energy():
    s = _cfg5_sub()
    out = []
    for spp in (1, 4):
        g = gpu_from_scene(s, source=False)
        g.set_time_blocking(spp)
        Ex, Ey, Hz, xs = consistent_random_state(s, 19)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.record_energy(True)
        g.step(301)
        assert g.info().steps_per_pass == spp
        out.append((g.get_window(), g.get_rom_state(), g.energy()))
        g.close()
    for a, b in zip(out[0][0], out[1][0]):
        assert np.array_equal(a, b)
    assert np.array_equal(out[0][1], out[1][1])
    e = out[1][2]
    assert np.all(np.diff(e) <= 1e-6 * e[:-1])


@pytest.mark.parametrize("precision", [64, 32])
def test_large_rom_order_unstaged_operators(precision):
    """q = 600 (q1 = q2 = 300): the shared operators no longer fit in shared memory and are read
    from L2; parity with the oracle and two-step bit-equality still hold."""
    nx = ny = 64
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(6, 6, 5, 31, 1, 4, 0, 0.05)
    m = rg.build_rom(6, 6, 5, dx, dy, fe, fs, 600, 30e9)
    assert m["q1"] == 300 and m["q2"] == 300
    dt = 0.95 * m["fine_dt_limit"]
    rng = np.random.default_rng(2)
    s = sc.Scene(name="bigq", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 3, (ny, nx)),
                 sigma=rng.uniform(0, 0.05, (ny, nx)), precision=precision, steps=800, source=(10, 10),
                 samples=sc.gaussian_samples(800, dt, 30e9, True), probes=np.array([[50, 50], [30, 12]], np.int32),
                 models=[m], placements=np.array([[0, 29, 30]], np.int32))
    _compare(s, 800, 1e-10 if precision == 64 else 1e-4, random_init=3)
    outs = []
    for spp in (1, 2, 4):
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        g.step(101)
        outs.append(g.get_window() + (g.get_rom_state(),))
        g.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


# ----------------------------------------------------------------- paper-literal coupling (NEXT-1)
def test_cfg1_literal_fp64():
    """Config 1 with the paper's own nP-port coupling (eq:sysform with T and 1/r; nP = 80, q1 = 92):
    the factored GPU update matches the oracle's LU of the literal A1 to 1e-10 over 4000 steps."""
    s = configs.make("cfg1lit")
    assert s.models[0]["literal"] and s.models[0]["L"].shape[1] == 80
    _compare(s, s.steps, 1e-10)


def _literal_scene(precision, n=128, seed=21):
    rng = np.random.default_rng(seed)
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(4, 4, 3, seed, 1, 4, 0, 0.05)
    m = rg.build_rom(4, 4, 3, dx, dy, fe, fs, 16, 30e9, literal=True)   # nP = 48, q1 = 56, q2 = 8
    dt = 0.95 * m["fine_dt_limit"]
    P = sc.place_blocks(n, n, [(4, 4)], 12, seed=seed, nslabs=1)
    return sc.Scene(name="literal", nx=n, ny=n, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 3, (n, n)),
                    sigma=rng.uniform(0, 0.05, (n, n)), precision=precision, steps=1000, source=(n // 2, n // 2),
                    samples=sc.gaussian_samples(1000, dt, 30e9, True),
                    probes=np.array([[5, 9], [n - 7, n - 12]], np.int32), models=[m], placements=P)


@pytest.mark.parametrize("precision", [64, 32])
def test_literal_rom_instances_parity(precision):
    """12 literal ROM instances in a lossy medium: <= 1e-10 (fp64) / 1e-4 (fp32) vs the oracle."""
    s = _literal_scene(precision)
    _compare(s, 1000, 1e-10 if precision == 64 else 1e-4, random_init=5)


def test_literal_rom_k_step_bitwise():
    """K = 1, 2, 4 steps per pass agree bit for bit with literal ROMs (fix-up with the literal update)."""
    s = _literal_scene(32)
    outs = []
    for spp in (1, 2, 4):
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        Ex, Ey, Hz, xs = consistent_random_state(s, 8)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.step(203)
        assert g.info().steps_per_pass == spp
        outs.append(g.get_window() + (g.get_rom_state(), g.probe()))
        g.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("src", [(55, 31), (56, 32), (111, 64), (112, 63)])
def test_source_and_probes_on_warp_and_chunk_seams(src):
    """K = 4 strips store 28 lanes x 2 columns (seams at columns 56 w) and chunks of 32 rows: a source
    and probes on / next to those seams are applied / recorded exactly once and match the one-step
    path bit for bit and the oracle to 1e-4."""
    n = 160
    rng = np.random.default_rng(9)
    dx = dy = 1e-3
    dt = 0.95 * sc.cfl_limit(dx, dy)
    probes = np.array([[src[0] + d, src[1] + e] for d in (-1, 0, 1) for e in (-1, 0, 1)] + [[56, 5], [55, 150]],
                      np.int32)
    s = sc.Scene(name="seams", nx=n, ny=n, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 4, (n, n)),
                 sigma=rng.uniform(0, 0.05, (n, n)), precision=32, steps=300, source=src,
                 samples=sc.gaussian_samples(300, dt, 30e9, True), probes=probes, models=[], placements=None)
    outs = []
    for spp, tuning in ((1, None), (4, None), (4, (256, 4))):  # (256, 4): the four-row sweep body
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        if tuning:
            g.set_tuning(*tuning)
        g.record_energy(True)
        g.step(300)
        assert g.info().steps_per_pass == spp
        outs.append((g.get_window(), g.probe(), g.energy()))
        g.close()
    for o in outs[1:]:
        for a, b in zip(outs[0][0], o[0]):
            assert np.array_equal(a, b)
        assert np.array_equal(outs[0][1], o[1])
        np.testing.assert_allclose(o[2], outs[0][2], rtol=1e-6)  # the same terms, summed in another order
    _compare(s, 300, 1e-4)


@pytest.mark.parametrize("precision", [64, 32])
def test_degenerate_roms(precision):
    """The method's smallest cases: a one-cell block (bx = by = 1, r = 2) and order q = 2
    (q1 = q2 = 1), next to full-order 1x1 blocks, in one lossy grid with a random start:
    fp64 <= 1e-10 / fp32 <= 1e-4 against the oracle."""
    rng = np.random.default_rng(21)
    nx, ny, dx = 40, 36, 1e-3
    eps, sig = rng.uniform(1, 3, (ny, nx)), rng.uniform(0, 0.03, (ny, nx))
    fe, fs = sc.uniform_fill(1, 1, 2, 5, 1, 4, 0, 0.05)
    m_q2 = rg.build_rom(1, 1, 2, dx, dx, fe, fs, 2, 30e9)
    m_full = rg.build_rom(1, 1, 3, dx, dx, *sc.uniform_fill(1, 1, 3, 6, 1, 4, 0, 0.05), 4, 30e9, full=True)
    assert (m_q2["q1"], m_q2["q2"]) == (1, 1)
    dt = 0.95 * min(m_q2["fine_dt_limit"], m_full["fine_dt_limit"], sc.cfl_limit(dx, dx))
    s = sc.Scene(name="degenerate", nx=nx, ny=ny, dx=dx, dy=dx, dt=dt, eps_r=eps, sigma=sig, precision=precision,
                 steps=500, source=(8, 9), samples=sc.gaussian_samples(500, dt, 30e9, True),
                 probes=np.array([[30, 30], [20, 18], [11, 25]], np.int32), models=[m_q2, m_full],
                 placements=np.array([[0, 18, 18], [0, 26, 12], [1, 12, 24]], np.int32))
    _compare(s, 500, 1e-10 if precision == 64 else 1e-4, random_init=7)


# ----------------------------------------------------------------- the large-model cooperative path
@pytest.fixture
def big_path(monkeypatch):
    """Route every model through bigrom_kernel (FDTD_BIG_Q = 1: the whole-GPU one-instance path)."""
    monkeypatch.setenv("FDTD_BIG_Q", "1")


@pytest.mark.parametrize("precision", [64, 32])
def test_big_rom_path_parity(big_path, precision):
    """Several instances of two models (a lossy inclusion and the literal coupling) on the cooperative
    large-model path: the oracle's LU route to 1e-10 (fp64) / 1e-4 (fp32), per instance too."""
    s = _ragged_scene(130, 61, precision)
    _compare(s, 600, 1e-10 if precision == 64 else 1e-4, random_init=5)


def test_big_rom_path_literal_fp64(big_path):
    s = _literal_scene(64)
    _compare(s, 400, 1e-10, random_init=5)


def test_big_rom_path_k_bitwise(big_path):
    """K = 1, 2, 4 steps per pass agree bit for bit on the large-model path too."""
    s = configs.make("cfg3", n=256)
    outs = []
    for spp in (1, 2, 4):
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        Ex, Ey, Hz, xs = consistent_random_state(s, 13)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.record_energy(True)
        for n in (1, 2, 3, 5, 8, 40, 1, 7):
            g.step(n)
        assert g.info().steps_per_pass == spp
        outs.append((g.get_window(), g.get_rom_state(), g.probe(), g.energy()))
        g.close()
    for (w, x, p, e) in outs[1:]:
        for a, b in zip(outs[0][0], w):
            assert np.array_equal(a, b)
        assert np.array_equal(outs[0][1], x)
        assert np.array_equal(outs[0][2], p)
        np.testing.assert_allclose(e, outs[0][3], rtol=2e-6)


# ----------------------------------------------------------------- clusters (no global pass-depth cliff)
def _dense_scene(precision, n=192, count=50, seed=5, nslabs=1):
    """SURVEY Q19's placement rule: footprint + one-cell ring inside the grid, rings pairwise disjoint
    -- instances 2 cells apart and next to the PEC walls, so four-step passes need fix-up clusters
    and wall-clipped regions."""
    rng = np.random.default_rng(seed)
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(6, 6, 3, seed, 1, 4, 0, 0.05)
    m = rg.build_rom(6, 6, 3, dx, dy, fe, fs, 24, 30e9)
    dt = 0.95 * m["fine_dt_limit"]
    P = sc.place_blocks(n, n, [(6, 6)], count, seed, nslabs=nslabs, margin=1, clear=1)
    probes = np.array([[1, 1], [n - 2, n - 2], [n // 2, 3]], np.int32)
    steps = 400
    return sc.Scene(name="dense", nx=n, ny=n, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 3, (n, n)),
                    sigma=rng.uniform(0, 0.05, (n, n)), precision=precision, steps=steps, source=(n // 3, n // 2 + 1),
                    samples=sc.gaussian_samples(steps, dt, 30e9, True), probes=probes, models=[m], placements=P)


def test_clusters_k4_bitwise_equal_k1():
    """Dense placement: the deepest pass stays 4 (clusters + wall-clipped regions instead of the
    round-1 global drop to one step per pass) and reproduces one-step passes bit for bit."""
    s = _dense_scene(32)
    outs = []
    for spp in (1, 2, 4):
        g = gpu_from_scene(s)
        g.set_time_blocking(spp)
        Ex, Ey, Hz, xs = consistent_random_state(s, 13)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.record_energy(True)
        for n in (1, 2, 3, 5, 8, 40, 1, 7):
            g.step(n)
        info = g.info()
        assert info.steps_per_pass == spp, (spp, info.steps_per_pass)
        if spp > 1:
            assert info.fixup_clusters >= (3 if spp == 4 else 1), (spp, info.fixup_clusters)
        outs.append((g.get_window(), g.get_rom_state(), g.probe(), g.energy()))
        g.close()
    for (w, x, p, e) in outs[1:]:
        for a, b in zip(outs[0][0], w):
            assert np.array_equal(a, b)
        assert np.array_equal(outs[0][1], x)
        assert np.array_equal(outs[0][2], p)
        np.testing.assert_allclose(e, outs[0][3], rtol=2e-6)


@pytest.mark.parametrize("precision", [64, 32])
def test_clusters_parity(precision):
    s = _dense_scene(precision)
    _compare(s, 400, 1e-10 if precision == 64 else 1e-4, random_init=5)


def test_clusters_energy_non_increasing():
    s = _dense_scene(32)
    g = gpu_from_scene(s, source=False)
    Ex, Ey, Hz, xs = consistent_random_state(s, 21)
    g.set_window(0, 0, Ex, Ey, Hz)
    g.set_rom_state(xs)
    g.record_energy(True)
    g.step(1000)
    e = g.energy()
    assert g.info().fixup_clusters >= 3
    assert np.all(np.diff(e) <= 1e-6 * e[:-1]), np.max(np.diff(e) / e[:-1])
