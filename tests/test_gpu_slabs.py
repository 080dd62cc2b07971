"""Row-slab decomposition on one device (-m gpu): N in-process slab contexts exchanging halo rows
with the same plan as the NCCL path must reproduce the single-context fields bit for bit."""
import numpy as np
import pytest

from inputs import romgen as rg
from inputs import scene as sc
from paper_1609_07114_b200 import slabs

from helpers import consistent_random_state, gpu_from_scene, ordered_instances

pytestmark = pytest.mark.gpu


def slab_scene(precision=32, literal=False):
    nx, ny = 203, 240
    rng = np.random.default_rng(12)
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(3, 2, 3, 1, 1, 4, 0, 0.05)
    m1 = rg.build_rom(3, 2, 3, dx, dy, fe, fs, 20, 30e9, literal=literal)
    fe, fs = sc.uniform_fill(2, 2, 4, 2, 1, 4, 0, 0.05)
    m2 = rg.build_rom(2, 2, 4, dx, dy, fe, fs, 16, 30e9)
    dt = 0.95 * min(m1["fine_dt_limit"], m2["fine_dt_limit"])
    src = (50, 119)
    probes = np.array([[50, 120], [50, 119], [10, 60], [150, 179], [100, 180], [5, 239]], dtype=np.int32)
    # slab-compatible for 2, 3 and 4 slabs: footprints + rings stay inside 20-row bands
    P = sc.place_blocks(nx, ny, [(3, 2), (2, 2)], 14, seed=5, nslabs=12,
                        forbid=[src] + [tuple(p) for p in probes])
    return sc.Scene(name="slabs", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 4, (ny, nx)),
                    sigma=rng.uniform(0, 0.05, (ny, nx)), precision=precision, steps=400, source=src,
                    samples=sc.gaussian_samples(400, dt, 30e9, True), probes=probes, models=[m1, m2],
                    placements=P)


def run_single(s, n, init):
    g = gpu_from_scene(s)
    Ex, Ey, Hz, xs = init
    g.set_window(0, 0, Ex, Ey, Hz)
    g.set_rom_state(xs)
    g.record_energy(True)
    g.step(n)
    out = g.get_window(), g.get_rom_state(), g.probe(), g.energy()
    g.close()
    return out


def run_group(s, n, init, nslab, spp=2, check_spp=True, tuning=None):
    import torch

    from paper_1609_07114_b200 import Simulation, step_group

    Ex, Ey, Hz, xs = init
    glob = ordered_instances(s)
    offs = np.cumsum([0] + [m["q1"] + m["q2"] for m, _, _ in glob])
    stream = torch.cuda.Stream()
    sims, local = [], []
    for k in range(nslab):
        rb, re = slabs.slab_rows(s.ny, nslab, k)
        m0, m1 = max(rb - 4, 0), min(re + 4, s.ny)
        sim = Simulation(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r[m0:m1], s.sigma[m0:m1], precision=s.precision,
                         stream=stream, rank=k, nranks=nslab, row_begin=rb, row_end=re, materials_row0=m0,
                         local_group=True)
        mine = []
        own = slabs.owned_placements(s.placements, s.models, rb, re)
        for mk, m in enumerate(s.models):
            sel = own[own[:, 0] == mk]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
                mine += [(m, int(i0), int(j0)) for _, i0, j0 in sel]
        if "pml" in s.meta:
            sim.set_pml(*s.meta["pml"])
        if "source_rows" in s.meta:
            sim.set_source_line(s.source[0], *s.meta["source_rows"], s.samples)
        else:
            sim.set_source(*s.source, s.samples)
        sim.set_probes(s.probes)
        sim.record_energy(True)
        sim.set_time_blocking(spp)
        if tuning:
            sim.set_tuning(*tuning)
        sim.set_window(0, 0, Ex, Ey, Hz)
        idx = [next(t for t, (mm, a, b) in enumerate(glob) if (a, b) == (i0, j0)) for _, i0, j0 in mine]
        if idx:
            sim.set_rom_state(np.concatenate([xs[offs[t]:offs[t + 1]] for t in idx]))
        sims.append(sim)
        local.append(idx)
    step_group(sims, n)
    if check_spp:
        assert all(sim.info().steps_per_pass == min(spp, 4 if s.precision == 32 else 2) for sim in sims)
    F = [np.zeros((s.ny + 1, s.nx)), np.zeros((s.ny, s.nx + 1)), np.zeros((s.ny, s.nx))]
    xs_out = np.zeros_like(xs)
    pr, en = 0, 0
    for sim, idx in zip(sims, local):
        w = sim.get_window()
        for a, b in zip(F, w):
            a += b  # each row is owned by exactly one slab (other rows come back as zeros)
        st = sim.get_rom_state()
        o = 0
        for t in idx:
            q = offs[t + 1] - offs[t]
            xs_out[offs[t]:offs[t + 1]] = st[o:o + q]
            o += q
        pr = pr + sim.probe()
        en = en + sim.energy()
        sim.close()
    return tuple(F), xs_out, pr, en


@pytest.mark.parametrize("spp", [1, 2, 4])
@pytest.mark.parametrize("nslab", [2, 3, 4])
@pytest.mark.parametrize("precision", [32, 64])
def test_slabs_bitwise_equal_single(nslab, precision, spp):
    """spp = K: K-step passes with K-row-deep halos (K = 4 falls back to 2 in fp64)."""
    s = slab_scene(precision)
    assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 3)
    (W1, x1, p1, e1) = run_single(s, 301, init)
    (W2, x2, p2, e2) = run_group(s, 301, init, nslab, spp)
    for a, b in zip(W1, W2):
        assert np.array_equal(a, b)
    assert np.array_equal(x1, x2)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(e2, e1, rtol=1e-12 if precision == 64 else 1e-6)


@pytest.mark.parametrize("spp", [1, 2, 4])
@pytest.mark.parametrize("nslab", [2, 3])
@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("rom", [False, True])
def test_cpml_slabs_bitwise_equal_single(nslab, precision, spp, rom):
    """NEXT-2 on row slabs: CPML layers + a line source across the slab edges; the psi rows of the
    ghost rows travel with the halo exchange.  Fields, ROM states and probes bit-identical to one
    context."""
    from test_gpu_pml import channel_scene

    s = channel_scene(precision, ny=60, rom=rom)
    if rom:
        s.placements = np.array([[0, 98, 11], [0, 120, 41]], np.int32)
        assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 5)
    (W1, x1, p1, e1) = run_single(s, 301, init)
    (W2, x2, p2, e2) = run_group(s, 301, init, nslab, spp, check_spp=not rom)  # 3 slabs: ROM regions cross a slab edge -> shallower passes
    for a, b in zip(W1, W2):
        assert np.array_equal(a, b)
    assert np.array_equal(x1, x2)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(e2, e1, rtol=1e-12 if precision == 64 else 1e-6)


@pytest.mark.parametrize("nslab", [2, 3])
def test_literal_models_on_slabs_bitwise(nslab):
    """NEXT-1 (paper-literal nP-port) models on row slabs: bit-identical to one context."""
    s = slab_scene(64, literal=True)
    assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 4)
    (W1, x1, p1, e1) = run_single(s, 201, init)
    (W2, x2, p2, e2) = run_group(s, 201, init, nslab, 2)
    for a, b in zip(W1, W2):
        assert np.array_equal(a, b)
    assert np.array_equal(x1, x2)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(e2, e1, rtol=1e-12)


@pytest.mark.parametrize("nslab", [2, 4])
def test_dense_clusters_slabs_bitwise_equal_single(nslab):
    """Clusters and wall-clipped regions on row slabs (SURVEY Q19's placement rule, rings inside the
    slabs): bit-identical to one context."""
    from test_gpu_parity import _dense_scene

    s = _dense_scene(32, nslabs=4)
    assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 3)
    (W1, x1, p1, e1) = run_single(s, 301, init)
    (W2, x2, p2, e2) = run_group(s, 301, init, nslab, 4, check_spp=False)
    for a, b in zip(W1, W2):
        assert np.array_equal(a, b)
    assert np.array_equal(x1, x2)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(e2, e1, rtol=1e-6)


@pytest.mark.parametrize("nslab", [2, 3])
@pytest.mark.parametrize("precision", [32, 64])
def test_slabs_match_oracle_directly(nslab, precision):
    """S8 against the oracle itself (not only against one context): the slabs' halo plan through the
    in-process transport, K-step passes (K = 4 fp32, 2 fp64), gathered fields, ROM states (global and
    per instance), probes and the energy vs the undivided fp64 oracle -- 1e-10 fp64, 1e-4 fp32
    (north_star tolerances)."""
    from helpers import instance_pairs, oracle_from_scene, per_instance_errors, rel

    s = slab_scene(precision)
    assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 7)
    n = 301
    (Wg, xg, pg, eg) = run_group(s, n, init, nslab, 4)
    o = oracle_from_scene(s)
    Ex, Ey, Hz, xs = init
    o.set_state(Ex, Ey, Hz, xs)
    po, eo = o.step(n, energy=True)
    Exo, Eyo, Hzo, xo = o.get_state()
    tol = 1e-10 if precision == 64 else 1e-4
    errs = dict(probe=rel(pg, po), Ex=rel(Wg[0], Exo), Ey=rel(Wg[1], Eyo), Hz=rel(Wg[2], Hzo), rom=rel(xg, xo),
                energy=rel(eg, eo))
    px, py = instance_pairs(s, Wg, (Exo, Eyo, Hzo), xg, xo)
    errs["rom_inst"], mx_rom = per_instance_errors(px)
    errs["y_inst"], mx_y = per_instance_errors(py)
    print("slabs", nslab, "fp%d" % precision, errs)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad and mx_rom <= 10 * tol and mx_y <= 10 * tol, (errs, mx_rom, mx_y)


@pytest.mark.parametrize("nslab", [2, 3])
def test_tall_slabs_with_long_chunks_bitwise(nslab):
    """Slabs of several 256-row chunks (the multi-GPU rule for 8,192-16,383-row slabs, four-row sweep
    body): the interior / slab-edge chunk split with K = 4 passes is bit-identical to one context."""
    nx, ny = 120, 1600
    rng = np.random.default_rng(21)
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(3, 2, 3, 1, 1, 4, 0, 0.05)
    m1 = rg.build_rom(3, 2, 3, dx, dy, fe, fs, 20, 30e9)
    dt = 0.95 * m1["fine_dt_limit"]
    src = (60, 799)
    probes = np.array([[60, 800], [10, 255], [100, 1023], [5, 1599]], dtype=np.int32)
    P = sc.place_blocks(nx, ny, [(3, 2)], 40, seed=6, nslabs=12, forbid=[src] + [tuple(p) for p in probes])
    # keep the fix-up regions (block + 7 cells for K = 4) clear of the 2- and 3-slab boundaries
    cuts = sorted({slabs.slab_rows(ny, n, k)[0] for n in (2, 3) for k in range(1, n)})
    P = P[[all(not (j0 - 8 <= c < j0 + 2 + 8) for c in cuts) for _, _, j0 in P]]
    s = sc.Scene(name="tall", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 4, (ny, nx)),
                 sigma=rng.uniform(0, 0.05, (ny, nx)), precision=32, steps=200, source=src,
                 samples=sc.gaussian_samples(200, dt, 30e9, True), probes=probes, models=[m1], placements=P)
    assert slabs.check_partition(s.placements, s.models, s.ny, nslab)
    init = consistent_random_state(s, 2)
    (W1, x1, p1, e1) = run_single(s, 101, init)
    (W2, x2, p2, e2) = run_group(s, 101, init, nslab, 4, tuning=(256, 4))
    for a, b in zip(W1, W2):
        assert np.array_equal(a, b)
    assert np.array_equal(x1, x2)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(e2, e1, rtol=1e-6)
