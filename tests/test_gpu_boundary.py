"""The C ABI's promises beyond parity (-m gpu): the non-finite sentinel (include/fdtdrom.h "Errors";
SPEC.md L379 / L419 "instability detected"), a new source window keeping the captured graph, and
the per-rank collective rules."""
import numpy as np
import pytest

from inputs import configs
from inputs import scene as sc

from helpers import consistent_random_state, gpu_from_scene

pytestmark = pytest.mark.gpu


def _cavity(precision, dt_factor, n=48):
    """Lossless vacuum PEC cavity at dt_factor x eq.(1) (the oracle pins the dichotomy: bounded at
    0.99 x, blown up at 1.01 x)."""
    dx = dy = 1e-3
    dt = dt_factor * sc.cfl_limit(dx, dy)
    return sc.Scene(name="cavity", nx=n, ny=n, dx=dx, dy=dy, dt=dt, eps_r=np.ones((n, n)), sigma=np.zeros((n, n)),
                    precision=precision, steps=2000, source=(5, 7), samples=np.zeros(1), probes=np.array([[20, 20]]),
                    models=[], placements=None)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("energy", [True, False])
def test_nonfinite_sentinel_at_105_eq1(precision, energy):
    """dt = 1.05 x eq.(1) with FDTD_ALLOW_DT_ABOVE_EQ1: the grid blows up (|lambda| ~ 1.9 per step)
    and the next synchronous call returns FDTD_E_UNSTABLE instead of NaN probes; the energy-off
    path is caught by the sampled Hz cells."""
    from paper_1609_07114_b200 import FDTDError
    s = _cavity(precision, 1.05)
    g = gpu_from_scene(s, allow_unstable=True)
    Ex, Ey, Hz, _ = consistent_random_state(s, 1)
    g.set_window(0, 0, Ex, Ey, Hz)
    g.record_energy(energy)
    g.step(2000)
    with pytest.raises(FDTDError) as e:
        g.probe()
    assert e.value.status == 4, e.value
    for call in (g.sync, g.get_window, g.energy):  # sticky
        with pytest.raises(FDTDError) as e:
            call()
        assert e.value.status == 4
    g.close()


@pytest.mark.parametrize("precision", [32, 64])
def test_sentinel_quiet_below_eq1(precision):
    s = _cavity(precision, 0.99)
    g = gpu_from_scene(s)
    Ex, Ey, Hz, _ = consistent_random_state(s, 1)
    g.set_window(0, 0, Ex, Ey, Hz)
    g.record_energy(True)
    g.step(2000)
    p, e = g.probe(), g.energy()
    assert np.all(np.isfinite(p)) and np.all(np.isfinite(e))
    assert abs(e[-1] / e[0] - 1) < 1e-4  # lossless: conserved
    g.close()


def test_create_refuses_dt_above_eq1():
    from paper_1609_07114_b200 import FDTDError
    s = _cavity(32, 1.001)
    with pytest.raises(FDTDError) as e:
        gpu_from_scene(s)
    assert e.value.status == 4


def test_source_window_keeps_graph():
    """The end-to-end pattern (per call: a new source window on the same cell, step(2K), read
    probes and energy) replays one captured graph and is bit-identical to one source upload."""
    s = configs.make("cfg3", n=256)
    n, chunk = 96, 8
    a = gpu_from_scene(s)
    a.record_energy(True)
    a.step(n)
    pa, ea, wa = a.probe(), a.energy(), a.get_window()
    b = gpu_from_scene(s)
    b.record_energy(True)
    pb, eb = [], []
    for k in range(0, n, chunk):
        b.set_source(*s.source, s.samples[k:k + chunk], step0=k)
        b.step(chunk)
        pb.append(b.probe())
        eb.append(b.energy())
    assert b.info().graph_builds == 1, b.info().graph_builds
    assert np.array_equal(np.concatenate(pb, axis=1), pa)
    assert np.array_equal(np.concatenate(eb), ea)
    for x, y in zip(b.get_window(), wa):
        assert np.array_equal(x, y)
    # a different source cell must re-capture
    b.set_source(s.source[0] + 1, s.source[1], s.samples[:chunk], step0=n)
    b.step(chunk)
    b.sync()
    assert b.info().graph_builds == 2
    a.close()
    b.close()


def _holes(s):
    """Masks of the ROM hole cells and of the interface edges (Ex rows / Ey columns on a block's rim)."""
    hz = np.zeros((s.ny, s.nx), bool)
    ex = np.zeros((s.ny + 1, s.nx), bool)
    ey = np.zeros((s.ny, s.nx + 1), bool)
    for k, i0, j0 in s.placements:
        bx, by = s.models[k]["bx"], s.models[k]["by"]
        hz[j0:j0 + by, i0:i0 + bx] = True
        ex[j0:j0 + by + 1, i0:i0 + bx] = True
        ey[j0:j0 + by, i0:i0 + bx + 1] = True
    return ex, ey, hz


@pytest.mark.parametrize("name,whole", [("cfg3", False), ("cfg1", False), ("cfg1", True)])
def test_random_fields_state_and_parity(name, whole):
    """fdtd_set_random_fields: every live cell and edge populated, holes / interface edges / PEC walls
    untouched (zero), and the state evolves like the oracle's from the same fields (fp32 1e-4 / fp64
    1e-10, energy non-increasing source-free) -- the pass path and the whole-grid path."""
    from helpers import oracle_from_scene, rel
    s = configs.make("cfg3", n=256) if name == "cfg3" else configs.make(name)
    g = gpu_from_scene(s, source=False, whole_grid=whole)
    g.set_random_fields(5, 1.0)
    Ex, Ey, Hz = g.get_window()
    mx, my, mh = _holes(s)
    assert not Hz[mh].any() and not Ex[mx].any() and not Ey[my].any()
    assert not Ex[0].any() and not Ex[-1].any() and not Ey[:, 0].any() and not Ey[:, -1].any()
    live = ~mh
    assert np.count_nonzero(Hz[live]) > 0.99 * live.sum()
    assert 0.5 < np.abs(Ex[1:-1][~mx[1:-1]]).max() <= 1.0
    assert np.abs(Hz).max() <= 1.0 / 376.0
    o = oracle_from_scene(s, source=False)
    o.set_state(Ex, Ey, Hz, None)
    g.record_energy(True)
    g.step(500)
    _, eo = o.step(500, energy=True)
    eg = g.energy()
    Exg, Eyg, Hzg = g.get_window()
    Exo, Eyo, Hzo, _ = o.get_state()
    errs = dict(Ex=rel(Exg, Exo), Ey=rel(Eyg, Eyo), Hz=rel(Hzg, Hzo), energy=rel(eg, eo))
    assert max(errs.values()) <= (1e-4 if s.precision == 32 else 1e-10), errs
    assert g.info().whole_grid == int(whole)
    assert np.all(np.diff(eg) <= 1e-6 * eg[:-1])
    g.close()


def test_random_fields_decomposition_independent():
    """The same seed gives the same state on one context and on 3 row slabs."""
    from paper_1609_07114_b200 import Simulation, slabs
    s = configs.make("cfg3", n=256)
    g = gpu_from_scene(s, source=False)
    g.set_random_fields(11, 2.0)
    ref = g.get_window()
    g.close()
    from helpers import np_materials
    eps, sig = np_materials(s)
    acc = [np.zeros_like(a) for a in ref]
    for k in range(3):
        rb, re = slabs.slab_rows(s.ny, 3, k)
        m0, m1 = max(rb - 4, 0), min(re + 4, s.ny)
        sim = Simulation(s.nx, s.ny, s.dx, s.dy, s.dt, eps[m0:m1], sig[m0:m1], precision=s.precision,
                         rank=k, nranks=3, row_begin=rb, row_end=re, materials_row0=m0, local_group=True)
        own = slabs.owned_placements(s.placements, s.models, rb, re)
        for mk, m in enumerate(s.models):
            sel = own[own[:, 0] == mk]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
        sim.set_random_fields(11, 2.0)
        for a, b in zip(acc, sim.get_window()):
            a += b
        sim.close()
    for a, b in zip(acc, ref):
        assert np.array_equal(a, b)
