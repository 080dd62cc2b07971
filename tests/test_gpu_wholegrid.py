"""The whole-grid path (K3c, -m gpu): small grids run every step of fdtd_step(n) in one
CTA (the grid plus a ring of dead wall cells and every ROM instance in shared memory, one launch per
call).  It must match the fp64 oracle like the pass path does (fp64 1e-10, fp32 1e-4, per instance)
and reproduce the sweep + fix-up passes bit for bit (fields, ROM states, probes; the energy up to
summation order), whatever the step counts per call."""
import numpy as np
import pytest

from inputs import configs
from inputs import romgen as rg
from inputs import scene as sc

from helpers import consistent_random_state, gpu_from_scene, oracle_from_scene, rel
from test_gpu_parity import _compare, _ragged_scene

pytestmark = pytest.mark.gpu


def _one_model(nx, ny, precision, seed=3):
    """_ragged_scene with one model: instances of model 0 only (the whole-grid path batches the
    instances of one model), plus one more of it near the top wall."""
    s = _ragged_scene(nx, ny, precision, seed=seed)
    s.models = s.models[:1]
    P = s.placements[s.placements[:, 0] == 0]
    s.placements = np.concatenate([P, np.array([[0, 2, ny - 4]], dtype=np.int32)])
    return s


def _dense_fp32(n=64, count=5, seed=11):
    """fp32 lossy medium with `count` instances of one 6 x 6 (r = 4) inclusion ROM placed with the
    one-cell-ring rule (instances next to each other and to the walls)."""
    rng = np.random.default_rng(seed)
    dx = dy = 1e-3
    fe, fs = sc.inclusion_fill(6, 4, seed=seed + 1)
    m0 = rg.build_rom(6, 6, 4, dx, dy, fe, fs, 40, 20e9)
    m = rg.extend_cfl(m0, 2 * m0["fine_dt_limit"])
    dt = min(1.9 * m0["fine_dt_limit"], 0.99 * sc.cfl_limit(dx, dy))
    P = sc.place_blocks(n, n, [(6, 6)], count, seed=seed + 2, nslabs=1, margin=1, clear=1)
    steps = 2000
    return sc.Scene(name="dense32", nx=n, ny=n, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 6, (n, n)),
                    sigma=rng.uniform(0, 0.05, (n, n)), precision=32, steps=steps, source=(n // 3, n // 2 + 1),
                    samples=sc.gaussian_samples(steps, dt, 20e9, True),
                    probes=np.array([[1, 1], [n - 2, n - 3], [n // 2, 5], [n // 3, n // 2 + 1]], dtype=np.int32),
                    models=[m], placements=P)


def test_cfg1_takes_the_whole_grid_path():
    s = configs.make("cfg1")
    g = gpu_from_scene(s, whole_grid=True)
    g.step(10)
    info = g.info()
    assert info.whole_grid == 1
    assert info.kernel_launches == 1  # one launch for the call
    g.step(7)
    assert g.info().kernel_launches == 2
    g.close()
    g = gpu_from_scene(s)  # helpers default: FDTD_NO_WHOLE (the pass path)
    g.step(10)
    assert g.info().whole_grid == 0
    g.close()


@pytest.mark.parametrize("name", ["cfg1", "cfg1b", "cfg1c", "cfg1lit"])
def test_whole_cfg1_vs_oracle_fp64(name):
    """Config 1 in full (4000 steps, fp64) through the whole-grid path: <= 1e-10."""
    s = configs.make(name)
    _compare(s, s.steps, 1e-10, whole_grid=True)


def test_whole_random_init_fp64():
    s = configs.make("cfg1")
    _compare(s, 1000, 1e-10, random_init=3, whole_grid=True)


@pytest.mark.parametrize("nx,ny", [(37, 29), (64, 48)])
def test_whole_ragged_fp64(nx, ny):
    """Ragged grids, instances next to the walls (the dead ring): <= 1e-10."""
    s = _one_model(nx, ny, 64)
    _compare(s, s.steps, 1e-10, random_init=5, whole_grid=True)


def test_whole_dense_fp32():
    """fp32, five instances on the one-cell-ring rule, 2000 steps: <= 1e-4 (per instance too)."""
    s = _dense_fp32()
    _compare(s, 2000, 1e-4, random_init=9, whole_grid=True)


def _run(s, whole, calls, spp=4, seed=13, energy=True, source=True):
    g = gpu_from_scene(s, whole_grid=whole, source=source)
    g.set_time_blocking(spp)
    Ex, Ey, Hz, xs = consistent_random_state(s, seed)
    g.set_window(0, 0, Ex, Ey, Hz)
    if xs.size:
        g.set_rom_state(xs)
    g.record_energy(energy)
    for n in calls:
        g.step(n)
    assert g.info().whole_grid == int(whole)
    out = (g.get_window(), g.get_rom_state(), g.probe(), g.energy() if energy else None)
    g.close()
    return out


@pytest.mark.parametrize("which", ["cfg1", "ragged64", "dense32"])
def test_whole_bitwise_equals_passes(which):
    """The whole-grid path and the sweep + fix-up passes (K = 2 fp64 / 4 fp32, remainder passes
    included) give the same fields, ROM states and probes bit for bit; the energy agrees to
    summation order.  Uneven step counts per call on the whole-grid side too."""
    s = {"cfg1": lambda: configs.make("cfg1"), "ragged64": lambda: _one_model(37, 29, 64),
         "dense32": _dense_fp32}[which]()
    calls = (1, 2, 3, 5, 8, 40, 1, 7)
    a = _run(s, False, calls)
    b = _run(s, True, (sum(calls),))
    c = _run(s, True, calls)
    for other in (b, c):
        for x, y in zip(a[0], other[0]):
            assert np.array_equal(x, y), which
        assert np.array_equal(a[1], other[1])
        assert np.array_equal(a[2], other[2])
        np.testing.assert_allclose(other[3], a[3], rtol=1e-12 if s.precision == 64 else 2e-6)


def test_whole_energy_non_increasing_source_free_fp32():
    s = _dense_fp32()
    _, _, _, e = _run(s, True, (2000,), source=False)
    assert np.all(np.diff(e) <= 1e-6 * e[:-1]), np.max(np.diff(e) / e[:-1])
    assert e[-1] < e[0]


def test_whole_nonfinite_sentinel():
    """A non-finite field value surfaces as FDTD_E_UNSTABLE at the next synchronous call."""
    from paper_1609_07114_b200 import FDTDError
    s = configs.make("cfg1")
    g = gpu_from_scene(s, whole_grid=True)
    Ex, Ey, Hz = g.get_window()
    Hz[20, 5] = np.nan
    g.set_window(0, 0, Ex, Ey, Hz)
    g.record_energy(False)
    g.step(50)
    assert g.info().whole_grid == 1
    with pytest.raises(FDTDError) as e:
        g.probe()
    assert e.value.status == 4, e.value
    g.close()


def test_whole_successive_calls_vs_oracle():
    """Successive calls (each one launch) continue the state and the record rings: probes read
    between calls and the final fields match the oracle."""
    s = configs.make("cfg1")
    o = oracle_from_scene(s)
    g = gpu_from_scene(s, whole_grid=True)
    g.step(123)
    po, _ = o.step(123)
    pg = g.probe()
    assert rel(pg, po) <= 1e-10
    g.step(77)
    po2, _ = o.step(77)
    assert rel(g.probe(), po2) <= 1e-10
    Exg, Eyg, Hzg = g.get_window()
    Exo, Eyo, Hzo, _ = o.get_state()
    assert max(rel(Exg, Exo), rel(Eyg, Eyo), rel(Hzg, Hzo)) <= 1e-10
    g.close()


def test_whole_line_source_and_probe_in_hole():
    """A line source across the grid (through an instance's row span) and a probe inside a ROM hole:
    the whole-grid path equals the passes bit for bit and the oracle to 1e-10."""
    s = _one_model(40, 36, 64)
    i0, j0 = int(s.placements[0, 1]), int(s.placements[0, 2])
    s.meta["source_rows"] = (2, s.ny - 2)
    s.source = (s.nx - 9, 0)
    s.probes = np.concatenate([s.probes, np.array([[i0 + 1, j0 + 1]], dtype=np.int32)])
    calls = (5, 17, 40)
    a = _run(s, False, calls, spp=2)
    b = _run(s, True, calls)
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    _compare(s, 300, 1e-10, whole_grid=True)
