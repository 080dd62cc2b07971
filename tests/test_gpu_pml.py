"""CPML layers and line sources (NEXT-2) on the GPU vs the fp64 oracle (-m gpu)."""
import numpy as np
import pytest

from inputs import romgen as rg
from inputs import scene as sc

from helpers import consistent_random_state, gpu_from_scene, oracle_from_scene, rel

pytestmark = pytest.mark.gpu


def channel_scene(precision, nx=200, ny=40, w=15, rom=False, seed=4):
    rng = np.random.default_rng(seed)
    dx = dy = 1e-3
    eps = rng.uniform(1, 3, (ny, nx))
    sig = rng.uniform(0, 0.02, (ny, nx))
    models, placements = [], None
    dt = 0.95 * sc.cfl_limit(dx, dy)
    if rom:
        fe, fs = sc.uniform_fill(4, 4, 3, seed, 1, 4, 0, 0.05)
        m = rg.build_rom(4, 4, 3, dx, dy, fe, fs, 24, 30e9)
        dt = 0.95 * min(m["fine_dt_limit"], sc.cfl_limit(dx, dy))
        models = [m]
        placements = np.array([[0, nx // 2 - 2, ny // 2 - 2], [0, nx // 2 + 20, 8]], np.int32)
    probes = np.array([[3, ny // 2], [w - 1, 5], [w + 2, ny - 3], [nx // 2 - 30, 7], [nx - 2, ny // 2],
                       [nx - w - 3, 11]], np.int32)
    return sc.Scene(name="channel", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=eps, sigma=sig, precision=precision,
                    steps=1500, source=(w + 12, 0), samples=sc.gaussian_samples(1500, dt, 30e9, True),
                    probes=probes, models=models, placements=placements,
                    meta=dict(pml=(w, 3, 1e-8), source_rows=(0, ny)))


def _compare(scene, n, tol, random_init=None):
    g = gpu_from_scene(scene)
    o = oracle_from_scene(scene)
    if random_init is not None:
        Ex, Ey, Hz, xs = consistent_random_state(scene, random_init)
        g.set_window(0, 0, Ex, Ey, Hz)
        o.set_state(Ex, Ey, Hz, xs if xs.size else None)
        if xs.size:
            g.set_rom_state(xs)
    g.record_energy(True)
    g.step(n)
    pg, eg = g.probe(), g.energy()
    Exg, Eyg, Hzg = g.get_window()
    po, eo = o.step(n)
    Exo, Eyo, Hzo, _ = o.get_state()
    errs = dict(probe=rel(pg, po), Ex=rel(Exg, Exo), Ey=rel(Eyg, Eyo), Hz=rel(Hzg, Hzo), energy=rel(eg, eo))
    g.close()
    assert max(errs.values()) <= tol, errs
    return errs


@pytest.mark.parametrize("precision", [64, 32])
def test_cpml_channel_parity(precision):
    """Line source in a CPML-terminated lossy channel: <= 1e-10 (fp64) / 1e-4 (fp32) vs the oracle."""
    s = channel_scene(precision)
    _compare(s, 1500, 1e-10 if precision == 64 else 1e-4)


def test_cpml_with_rom_instances_parity():
    s = channel_scene(64, rom=True)
    _compare(s, 1200, 1e-10, random_init=3)


def test_cpml_k_step_bitwise():
    """K = 1, 2, 4 steps per pass with CPML bands (band fix-up kernel) agree bit for bit, from a
    random state that fills the layers at once (301 steps: the K = 4 and K = 2 runs end with a
    shorter pass, whose band region must still cover the Kz-deep write-back columns)."""
    s = channel_scene(32, rom=True)
    Ex, Ey, Hz, xs = consistent_random_state(s, 8)
    outs = []
    for spp, tuning in ((1, None), (2, None), (4, None), (4, (256, 4))):  # (256, 4): four-row sweep body
        g = gpu_from_scene(s)
        if tuning:
            g.set_tuning(*tuning)
        g.set_window(0, 0, Ex, Ey, Hz)
        g.set_rom_state(xs)
        g.set_time_blocking(spp)
        g.step(301)
        assert g.info().steps_per_pass == spp
        outs.append(g.get_window() + (g.get_rom_state(), g.probe()))
        g.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_cpml_absorbs_on_gpu():
    """The GPU channel absorbs the wave: energy falls by > 1e6 once the pulse has left."""
    s = channel_scene(64, nx=160, ny=16)
    s.eps_r = np.ones_like(s.eps_r)  # homogeneous lossless channel (no trapped scattered energy)
    s.sigma = np.zeros_like(s.sigma)
    g = gpu_from_scene(s)
    g.record_energy(True)
    g.step(3000)
    e = g.energy()
    g.close()
    assert e[-1] <= 1e-6 * e.max()
