"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu).

The GPU runs the whole 8192^2 / 32768^2 grid (all ROM instances, default tuning, CUDA graphs);
the fp64 oracle recomputes sampled outputs one window at a time: each sample box is advanced in a
window that contains its backward dependency cone (helpers.cone_window), so the window's PEC edge
cannot reach the samples.  Initial state: random live fields inside the windows (holes and
interface edges zero, ROM states zero, R26), zero elsewhere; the source stays on.
"""
import numpy as np
import pytest

import oracle as O
from inputs import configs

from helpers import cone_window, instance_boxes, rel

pytestmark = pytest.mark.gpu
NSTEPS = 16


def _boxes(scene):
    n = scene.nx
    cx, cy = scene.source
    boxes = [(cx - 16, cy - 16, cx + 16, cy + 16),          # the source
             (0, 0, 24, 24),                                  # the south-west PEC corner
             (n - 24, n - 24, n, n),                          # the north-east corner (last warp strip)
             (n // 3, 2 * n // 3, n // 3 + 24, 2 * n // 3 + 24)]
    ib = instance_boxes(scene)
    if ib:  # a ROM instance far from the others, with some margin
        r = ib[len(ib) // 2]
        boxes.append((r[0] - 4, r[1] - 4, r[2] + 4, r[3] + 4))
    return boxes


def _random_window(rng, W, holes):
    a0, b0, a1, b1 = W
    w, h = a1 - a0, b1 - b0
    Ex = rng.standard_normal((h + 1, w))
    Ey = rng.standard_normal((h, w + 1))
    Hz = rng.standard_normal((h, w)) / 377.0
    return Ex, Ey, Hz


def _zero_rom_parts(scene, W, Ex, Ey, Hz, nx, ny):
    """Holes, interface edges and PEC walls inside window W set to zero (R26 with x~ = 0)."""
    a0, b0 = W[0], W[1]
    if a0 == 0:
        Ey[:, 0] = 0
    if W[2] == nx:
        Ey[:, -1] = 0
    if b0 == 0:
        Ex[0] = 0
    if W[3] == ny:
        Ex[-1] = 0
    for k, i0, j0 in (scene.placements if scene.placements is not None else []):
        m = scene.models[k]
        bx, by = m["bx"], m["by"]
        if not (i0 + bx >= a0 and i0 <= W[2] and j0 + by >= b0 and j0 <= W[3]):
            continue
        for jj in range(j0, j0 + by + 1):        # Ex edges of the block (interface rows included)
            for ii in range(i0, i0 + bx):
                if 0 <= jj - b0 < Ex.shape[0] and 0 <= ii - a0 < Ex.shape[1]:
                    Ex[jj - b0, ii - a0] = 0
        for jj in range(j0, j0 + by):
            for ii in range(i0, i0 + bx + 1):
                if 0 <= jj - b0 < Ey.shape[0] and 0 <= ii - a0 < Ey.shape[1]:
                    Ey[jj - b0, ii - a0] = 0
            for ii in range(i0, i0 + bx):
                if 0 <= jj - b0 < Hz.shape[0] and 0 <= ii - a0 < Hz.shape[1]:
                    Hz[jj - b0, ii - a0] = 0


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_full_size_sampled_parity(name):
    import torch

    from paper_1609_07114_b200 import Simulation

    scene = configs.make(name, device="cuda")
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, scene.eps_r, scene.sigma,
                     precision=scene.precision)
    if scene.placements is not None:
        for k, m in enumerate(scene.models):
            sel = scene.placements[scene.placements[:, 0] == k]
            sim.add_rom(m, sel[:, 1:3])
    sim.set_source(*scene.source, scene.samples)
    rng = np.random.default_rng(77)
    boxes = _boxes(scene)
    wins = [cone_window(scene, b, NSTEPS) for b in boxes]
    for i in range(len(wins)):
        for j in range(i + 1, len(wins)):
            a, b = wins[i], wins[j]
            assert not (a[0] < b[2] and b[0] < a[2] and a[1] < b[3] and b[1] < a[3]), "windows overlap"
    n_rom_windows = 0
    inits = []
    for W in wins:
        Ex, Ey, Hz = _random_window(rng, W, None)
        _zero_rom_parts(scene, W, Ex, Ey, Hz, scene.nx, scene.ny)
        sim.set_window(W[0], W[1], Ex, Ey, Hz)
        inits.append((Ex, Ey, Hz))
    sim.step(NSTEPS)
    for b, W, (Ex, Ey, Hz) in zip(boxes, wins, inits):
        a0, b0, a1, b1 = W
        eps = scene.eps_r[b0:b1, a0:a1].double().cpu().numpy()
        sig = scene.sigma[b0:b1, a0:a1].double().cpu().numpy()
        o = O.OracleSim(a1 - a0, b1 - b0, scene.dx, scene.dy, scene.dt, eps, sig)
        nrom = 0
        for k, m in enumerate(scene.models):
            for kk, i0, j0 in (scene.placements if scene.placements is not None else []):
                if kk == k and a0 <= i0 - 1 and i0 + m["bx"] + 1 <= a1 and b0 <= j0 - 1 and j0 + m["by"] + 1 <= b1:
                    o.add_rom(m, int(i0) - a0, int(j0) - b0)
                    nrom += 1
        n_rom_windows += nrom > 0
        sx, sy = scene.source
        if a0 <= sx < a1 and b0 <= sy < b1:
            o.set_source(sx - a0, sy - b0, scene.samples)
        o.set_state(Ex, Ey, Hz)
        o.step(NSTEPS, probes=False, energy=False)
        Exo, Eyo, Hzo, _ = o.get_state()
        i0, j0, i1, j1 = max(b[0], 0), max(b[1], 0), min(b[2], scene.nx), min(b[3], scene.ny)
        gEx, gEy, gHz = sim.get_window(i0, j0, i1 - i0, j1 - j0)
        sl = (slice(j0 - b0, j1 - b0), slice(i0 - a0, i1 - a0))
        e = [rel(gHz, Hzo[sl]),
             rel(gEx, Exo[j0 - b0:j1 - b0 + 1, i0 - a0:i1 - a0]),
             rel(gEy, Eyo[j0 - b0:j1 - b0, i0 - a0:i1 - a0 + 1])]
        print("%s box %s window %s roms %d rel-L2 Hz/Ex/Ey %s |Hz| %.3g" % (name, b, W, nrom, e, np.linalg.norm(Hzo[sl])))
        assert np.linalg.norm(Hzo[sl]) > 0
        assert max(e) <= 1e-4, (name, b, W, e)
    if scene.placements is not None:
        assert n_rom_windows >= 1
    sim.close()
    del scene
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["cfg3"])
def test_full_grid_first_200_steps(name):
    """Config 3 in full (8192^2, all 1024 ROM instances) for the first 200 steps from a random
    consistent state, every cell and every ROM state compared (config 2 is the same
    stencil without ROMs and is covered at full size by the sampled-window test)."""
    import torch

    from helpers import consistent_random_state, gpu_from_scene, oracle_from_scene

    scene = configs.make(name, device="cuda")
    scene.eps_r = scene.eps_r.double().cpu().numpy()
    scene.sigma = scene.sigma.double().cpu().numpy()
    O.set_threads(0)
    g = gpu_from_scene(scene)
    o = oracle_from_scene(scene)
    Ex, Ey, Hz, xs = consistent_random_state(scene, 23)
    g.set_window(0, 0, Ex, Ey, Hz)
    o.set_state(Ex, Ey, Hz, xs if xs.size else None)
    if xs.size:
        g.set_rom_state(xs)
    del Ex, Ey, Hz
    g.record_energy(True)
    g.step(200)
    po, eo = o.step(200)
    pg, eg = g.probe(), g.energy()
    Exg, Eyg, Hzg = g.get_window()
    Exo, Eyo, Hzo, xo = o.get_state()
    errs = dict(probe=rel(pg, po), Ex=rel(Exg, Exo), Ey=rel(Eyg, Eyo), Hz=rel(Hzg, Hzo), energy=rel(eg, eo))
    if xo.size:
        errs["rom"] = rel(g.get_rom_state(), xo)
    print(name, errs)
    assert max(errs.values()) <= 1e-4, errs
    g.close()
    o.close()
    torch.cuda.empty_cache()


def _clusters(scene, k=3, count=2):
    """Boxes (footprint + ring + 2) around clusters of k ROM instances: an instance and its k-1
    nearest neighbours, one cluster near the grid's centre and one near its south-west quarter."""
    P = np.asarray(scene.placements)
    byx = np.array([[scene.models[m]["bx"], scene.models[m]["by"]] for m in P[:, 0]])
    c = P[:, 1:3] + byx / 2.0
    out = []
    for tx, ty in [(0.5, 0.5), (0.25, 0.3)][:count]:
        a = int(np.argmin(np.hypot(c[:, 0] - tx * scene.nx, c[:, 1] - ty * scene.ny)))
        near = np.argsort(np.hypot(c[:, 0] - c[a, 0], c[:, 1] - c[a, 1]))[:k]
        x0 = min(P[t, 1] for t in near) - 3
        y0 = min(P[t, 2] for t in near) - 3
        x1 = max(P[t, 1] + byx[t, 0] for t in near) + 3
        y1 = max(P[t, 2] + byx[t, 1] for t in near) + 3
        out.append(((int(x0), int(y0), int(x1), int(y1)), [int(t) for t in near]))
    return out


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_first_200_steps_rom_clusters(name):
    """BASELINE configs 4 (32768^2, 4096 instances) and 5 (49152^2, 8192 instances of 32 models) at
    full size, in bench.py's launch configuration (K = 4 passes, CUDA graphs): the first 200 steps
    of two clusters of >= 3 ROM instances each, from random fields and random consistent ROM states
    (R26), against the fp64 oracle run on each cluster's 200-step dependency cone.  Fields in the
    clusters <= 1e-4; every instance's x~ and y <= 1e-4 (relative L2, own norm) and <= 1e-3
    (relative max-abs)."""
    import torch

    from helpers import instance_y, ordered_instances, per_instance_errors
    from paper_1609_07114_b200 import Simulation

    n_steps = 200
    scene = configs.make(name, device="cuda")
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, scene.eps_r, scene.sigma,
                     precision=scene.precision)
    for k, m in enumerate(scene.models):
        sel = scene.placements[scene.placements[:, 0] == k]
        if len(sel):
            sim.add_rom(m, sel[:, 1:3])
    sim.set_source(*scene.source, scene.samples)
    inst = ordered_instances(scene)  # the order of get_rom_state
    where = {(i0, j0): t for t, (_, i0, j0) in enumerate(inst)}
    qs = [m["q1"] + m["q2"] for m, _, _ in inst]
    offs = np.cumsum([0] + qs)
    xs_all = np.zeros(offs[-1])
    rng = np.random.default_rng(5)
    # cluster members as indices into `inst` (placement order differs from it with several models)
    cl = [(box, [where[(int(scene.placements[t, 1]), int(scene.placements[t, 2]))] for t in near])
          for box, near in _clusters(scene)]
    wins = [cone_window(scene, box, n_steps) for box, _ in cl]
    a, b = wins
    assert not (a[0] < b[2] and b[0] < a[2] and a[1] < b[3] and b[1] < a[3]), "windows overlap"
    runs = []
    for (box, near), W in zip(cl, wins):
        a0, b0, a1, b1 = W
        Ex, Ey, Hz = _random_window(rng, W, None)
        _zero_rom_parts(scene, W, Ex, Ey, Hz, scene.nx, scene.ny)
        inside = []  # instances whose footprint + ring lies in the window (the oracle embeds them)
        for m, i0, j0 in inst:
            if a0 <= i0 - 1 and i0 + m["bx"] + 1 <= a1 and b0 <= j0 - 1 and j0 + m["by"] + 1 <= b1:
                t = where[(i0, j0)]
                xt = rng.standard_normal(qs[t])
                xt[m["q1"]:] /= 377.0
                y = m["L"].T @ xt[:m["q1"]]
                bx, by = m["bx"], m["by"]
                u, v = i0 - a0, j0 - b0
                Ex[v, u:u + bx], Ex[v + by, u:u + bx] = y[:bx], y[bx:2 * bx]
                Ey[v:v + by, u], Ey[v:v + by, u + bx] = y[2 * bx:2 * bx + by], y[2 * bx + by:]
                xs_all[offs[t]:offs[t + 1]] = xt
                inside.append((m, i0, j0, t))
        assert all(any(t == x[3] for x in inside) for t in near)
        sim.set_window(a0, b0, Ex, Ey, Hz)
        runs.append((Ex, Ey, Hz, inside))
    sim.set_rom_state(xs_all)
    sim.step(n_steps)
    xg_all = sim.get_rom_state()
    for (box, near), W, (Ex, Ey, Hz, inside) in zip(cl, wins, runs):
        a0, b0, a1, b1 = W
        eps = scene.eps_r[b0:b1, a0:a1].double().cpu().numpy()
        sig = scene.sigma[b0:b1, a0:a1].double().cpu().numpy()
        o = O.OracleSim(a1 - a0, b1 - b0, scene.dx, scene.dy, scene.dt, eps, sig)
        for m, i0, j0, t in inside:
            o.add_rom(m, i0 - a0, j0 - b0)
        sx, sy = scene.source
        if a0 <= sx < a1 and b0 <= sy < b1:
            o.set_source(sx - a0, sy - b0, scene.samples)
        o.set_state(Ex, Ey, Hz, np.concatenate([xs_all[offs[t]:offs[t + 1]] for *_, t in inside]))
        o.step(n_steps, probes=False, energy=False)
        Exo, Eyo, Hzo, xo = o.get_state()
        i0, j0, i1, j1 = box
        gEx, gEy, gHz = sim.get_window(i0, j0, i1 - i0, j1 - j0)
        e = [rel(gHz, Hzo[j0 - b0:j1 - b0, i0 - a0:i1 - a0]),
             rel(gEx, Exo[j0 - b0:j1 - b0 + 1, i0 - a0:i1 - a0]),
             rel(gEy, Eyo[j0 - b0:j1 - b0, i0 - a0:i1 - a0 + 1])]
        xo_split, o_off = {}, 0
        for m, ii, jj, t in inside:
            xo_split[t] = xo[o_off:o_off + qs[t]]
            o_off += qs[t]
        px, py = [], []
        for t in near:
            m, ii, jj = inst[t]
            px.append((xg_all[offs[t]:offs[t + 1]], xo_split[t]))
            py.append((instance_y(m, ii, jj, gEx, gEy, i0, j0), instance_y(m, ii, jj, Exo, Eyo, a0, b0)))
        ex = per_instance_errors(px, floor_frac=0.0)
        ey = per_instance_errors(py, floor_frac=0.0)
        print("%s cluster %s window %s instances %d fields %s x~ %s y %s" % (name, box, W, len(inside), e, ex, ey))
        assert len(near) >= 3 and max(e) <= 1e-4, (name, box, e)
        assert ex[0] <= 1e-4 and ey[0] <= 1e-4 and ex[1] <= 1e-3 and ey[1] <= 1e-3, (name, box, ex, ey)
    sim.close()
    del scene
    torch.cuda.empty_cache()
