"""BASELINE.json configs as seeded synthetic scenes.

``make(name, n=None, device="cpu")`` builds config ``name`` at its full size or,
with ``n``, a seeded n x n sub-instance with the same recipe (same material
statistics and correlation length, ROM placements scaled with the area).  The
sub-instances are the "seeded cropped sub-instances" the oracle can finish.

  cfg1   40x40 fp64 vacuum PEC cavity, one 4x4 block r=5 (U[1,4], U[0,0.05]), q=24,
         dt = 0.95 eq.(1); ROM clipped at dt/0.95 (R22); Gaussian-derivative 30 GHz
         at (8,8); probe (30,30); 4000 steps.
  cfg1b  as cfg1 with dt = 0.95 dt_f (the MOR-only variant, R22).
  cfg1c  as cfg1 with q = 48, whose clip is active (4 singular values clipped).
  cfg2   8192^2 fp32, copula eps_r U[1,10], sigma U[0,0.1], l = 32; dt = 0.99 eq.(1);
         Gaussian 10 GHz at the centre; 64 seeded probes; 10000 steps.
  cfg3   cfg2 + 1024 placements of one model: 8x8 block, r=8, disc inclusion (R23),
         q=64; clip at 2 dt_f; dt = 1.9 dt_f; 10000 steps.
  cfg4   32768^2 fp32 medium as cfg2 + 4096 placements: 16x16 block, r=4, inclusion,
         q=128; clip at 2 dt_f; dt = 1.9 dt_f; 5000 steps.
  cfg4dense  cfg4 with SURVEY Q19's placement rule (one-cell rings disjoint, 1 cell from the walls).
  cfg5   49152^2 fp32, 32 models (b U{4..32}, r U{4..10}, q U{32,64,128,256}, fill
         eps_r U[1,12], sigma U[0,0.2]), 8192 placements; dt = 1.9 min dt_f; 2000 steps.
"""
from __future__ import annotations

import functools
import math

import numpy as np

from . import romgen as rg
from . import scene as sc

DX = DY = 1e-3  # R21


@functools.lru_cache(maxsize=64)
def _model(kind, b, r, q, fmax, seed, dt_target_factor, literal=False):
    if kind == "uniform14":
        fe, fs = sc.uniform_fill(b, b, r, seed, 1.0, 4.0, 0.0, 0.05)
    elif kind == "uniform112":
        fe, fs = sc.uniform_fill(b, b, r, seed, 1.0, 12.0, 0.0, 0.2)
    else:
        fe, fs = sc.inclusion_fill(b, r, seed)
    sysf = rg.fine_system(b, b, r, DX, DY, fe, fs)
    csys = rg.literal_system(sysf) if literal else rg.collapse(sysf)
    V1, V2 = rg.sprim_basis(csys, q, fmax)
    if literal:  # the E basis must hold the nP port directions (q1 >= nP)
        V1 = rg.with_port_directions(V1, csys["nY"])[:, : csys["nY"] + (q + 1) // 2]
    m = rg.reduce(csys, V1, V2)
    m["natural_dt_limit"] = rg.rom_cfl_limit(m)
    m["fine_dt_limit"] = rg.fine_cfl_limit(sysf)
    m["fine_eps_r"], m["fine_sigma"] = fe, fs
    return m


def model(kind, b, r, q, fmax, seed, dt_target=None, literal=False):
    """A cached ROM of the given fill kind (see _model), optionally clipped at dt_target.
    literal: the paper's own nP-port coupling (NEXT-1) instead of the collapsed ports (R9)."""
    m = dict(_model(kind, b, r, q, fmax, seed, None, literal))
    if dt_target is not None:
        m = rg.extend_cfl(m, dt_target)
    return m


def _cfg1(variant, n=None):
    """Config 1; variants b (dt = 0.95 dt_f), c (q = 48, active clip) and lit (the paper-literal
    coupling through the nP = 80 fine hanging variables, NEXT-1: q = 24 + 80 port directions)."""
    nx = ny = 40
    eps = np.ones((ny, nx))
    sig = np.zeros((ny, nx))
    q = 48 if variant == "c" else 24
    m = model("uniform14", 4, 5, q, 30e9, 11, literal=(variant == "lit"))
    dtc = sc.cfl_limit(DX, DY)
    if variant == "b":
        dt = 0.95 * m["fine_dt_limit"]
        m = rg.extend_cfl(m, dt / 0.95)
    else:
        dt = 0.95 * dtc
        m = rg.extend_cfl(m, dtc)  # dt_target = dt / 0.95 (R22)
    steps = 4000
    samples = sc.gaussian_samples(steps, dt, 30e9, derivative=True)
    return sc.Scene(name="cfg1" + ("" if variant == "a" else variant), nx=nx, ny=ny, dx=DX, dy=DY, dt=dt,
                    eps_r=eps, sigma=sig, precision=64, steps=steps, source=(8, 8), samples=samples,
                    probes=np.array([[30, 30]], dtype=np.int32), models=[m],
                    placements=np.array([[0, 18, 18]], dtype=np.int32),
                    meta=dict(n_clipped=[m["n_clipped"]]))


def _medium(n, seed, device, lo_e=1.0, hi_e=10.0, hi_s=0.1):
    eps = sc.smooth_field(n, n, 32, lo_e, hi_e, seed, device=device)
    sig = sc.smooth_field(n, n, 32, 0.0, hi_s, seed + 1, device=device)
    return eps, sig


def _grid_scene(name, N, n, device, steps, rom=None, count=0, seed=100, dense=False):
    n = N if n is None else int(n)
    eps, sig = _medium(n, seed, device)
    dtc = sc.cfl_limit(DX, DY, eps_r_min=1.0)  # c_max: eps_r >= 1 everywhere
    models, placements, dt = [], None, 0.99 * dtc
    src = (n // 2, n // 2)
    fmax = 10e9
    probes = sc.probes_random(n, n, 64 if n >= 64 else 4, seed + 7)
    if rom is not None:
        b, r, q = rom
        m0 = model("inclusion", b, r, q, fmax, seed + 3)
        dtf = m0["fine_dt_limit"]
        m = rg.extend_cfl(m0, 2.0 * dtf)
        dt = min(1.9 * dtf, 0.99 * dtc)
        cnt = max(1, int(round(count * (n / N) ** 2)))
        # dense: SURVEY Q19's own rule -- footprint + one-cell ring inside the grid and the slab, rings
        # pairwise disjoint (instances may sit 2 cells apart and next to the walls: the fix-up then
        # merges close instances into clusters); default: 7 / 4 cells
        placements = sc.place_blocks(n, n, [(b, b)], cnt, seed + 5, nslabs=8 if n % 8 == 0 else 1,
                                     forbid=[src] + [tuple(p) for p in probes],
                                     **(dict(margin=1, clear=1) if dense else {}))
        models = [m]
    samples = sc.gaussian_samples(steps, dt, fmax, derivative=False)
    return sc.Scene(name=name, nx=n, ny=n, dx=DX, dy=DY, dt=dt, eps_r=eps, sigma=sig, precision=32,
                    steps=steps, source=src, samples=samples, probes=probes, models=models,
                    placements=placements,
                    meta=dict(full_n=N, n_clipped=[m["n_clipped"] for m in models]))


CFG5_SEED = 500


def cfg5_specs(seed=CFG5_SEED):
    """The 32 (b, r, q) model specs of config 5 (b ~ U{4..32}, r ~ U{4..10}, q ~ U{32,64,128,256})."""
    rng = np.random.default_rng(seed)
    specs = []
    for _ in range(32):
        b = int(rng.integers(4, 33))
        r = int(rng.integers(4, 11))
        q = int(rng.choice([32, 64, 128, 256]))
        specs.append((b, r, q))
    return specs


def _cfg5(n, device, seed=CFG5_SEED, max_fine=None, min_count=0):
    """Config 5.  Sub-instances may restrict the models to fine grids of at most max_fine cells per
    side (fast to build) and place at least min_count instances."""
    N = 49152
    n = N if n is None else int(n)
    eps, sig = _medium(n, seed, device)
    specs = cfg5_specs(seed)
    cnt = max(min_count, int(round(8192 * (n / N) ** 2)))
    use = [k for k, (b, r, q) in enumerate(specs) if (max_fine is None or b * r <= max_fine) and b <= max(4, n // 16)]
    models = [model("uniform112", *specs[k], 10e9, seed + 10 + k) for k in use]
    dtf = min(m["fine_dt_limit"] for m in models)
    dt = min(1.9 * dtf, 0.99 * sc.cfl_limit(DX, DY))
    models = [rg.extend_cfl(m, dt / 0.95) for m in models]
    src = (n // 2, n // 2)
    probes = sc.probes_random(n, n, 64, seed + 7)
    placements = sc.place_blocks(n, n, [(m["bx"], m["by"]) for m in models], cnt, seed + 5,
                                 nslabs=8 if n % 8 == 0 else 1, forbid=[src] + [tuple(p) for p in probes])
    steps = 2000
    samples = sc.gaussian_samples(steps, dt, 10e9)
    return sc.Scene(name="cfg5", nx=n, ny=n, dx=DX, dy=DY, dt=dt, eps_r=eps, sigma=sig, precision=32,
                    steps=steps, source=src, samples=samples, probes=probes, models=models,
                    placements=placements, meta=dict(full_n=N, n_clipped=[m["n_clipped"] for m in models],
                                                     model_specs=[specs[k] for k in use]))


def make(name, n=None, device="cpu", **kw):
    if name in ("cfg1", "cfg1b", "cfg1c", "cfg1lit"):
        return _cfg1({"cfg1": "a", "cfg1b": "b", "cfg1c": "c", "cfg1lit": "lit"}[name])
    if name == "cfg2":
        return _grid_scene("cfg2", 8192, n, device, 10000)
    if name == "cfg3":
        return _grid_scene("cfg3", 8192, n, device, 10000, rom=(8, 8, 64), count=1024, seed=300)
    if name == "cfg4":
        return _grid_scene("cfg4", 32768, n, device, 5000, rom=(16, 4, 128), count=4096, seed=400)
    if name == "cfg4dense":  # cfg4 with SURVEY Q19's one-cell-ring placement rule
        return _grid_scene("cfg4dense", 32768, n, device, 5000, rom=(16, 4, 128), count=4096, seed=400, dense=True)
    if name == "cfg5":
        return _cfg5(n, device, **kw)
    raise KeyError(name)


def to_numpy(a):
    try:
        import torch

        if isinstance(a, torch.Tensor):
            return a.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a, dtype=np.float64)
