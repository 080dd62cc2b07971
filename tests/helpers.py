"""Shared test helpers: build the oracle and the CUDA path from the same seeded Scene."""
import numpy as np

import oracle as O
from inputs import configs


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def np_materials(scene):
    return configs.to_numpy(scene.eps_r), configs.to_numpy(scene.sigma)


def oracle_from_scene(scene, source=True, probes=True):
    eps, sig = np_materials(scene)
    s = O.OracleSim(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, eps, sig)
    if scene.placements is not None:
        # same instance order as the CUDA path (grouped by model, in placement order)
        for k, m in enumerate(scene.models):
            for kk, i0, j0 in scene.placements:
                if kk == k:
                    s.add_rom(m, int(i0), int(j0))
    if source:
        s.set_source(*scene.source, scene.samples)
    if probes:
        s.set_probes(scene.probes)
    return s


def gpu_from_scene(scene, source=True, probes=True, **kw):
    from paper_1609_07114_b200 import Simulation
    eps, sig = np_materials(scene)
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, eps, sig, precision=scene.precision, **kw)
    if scene.placements is not None:
        for k, m in enumerate(scene.models):
            sel = scene.placements[scene.placements[:, 0] == k]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
    if source:
        sim.set_source(*scene.source, scene.samples)
    if probes:
        sim.set_probes(scene.probes)
    return sim


def ordered_instances(scene):
    out = []
    if scene.placements is None:
        return out
    for k, m in enumerate(scene.models):
        for kk, i0, j0 in scene.placements:
            if kk == k:
                out.append((m, int(i0), int(j0)))
    return out


def consistent_random_state(scene, seed, lossless_scale=1.0):
    """DESIGN.md R26: random live fields; PEC and holes zero; interface y = L~^T E~ of a random ROM state."""
    rng = np.random.default_rng(seed)
    nx, ny = scene.nx, scene.ny
    Ex = rng.standard_normal((ny + 1, nx))
    Ey = rng.standard_normal((ny, nx + 1))
    Hz = rng.standard_normal((ny, nx)) / 377.0
    Ex[0] = Ex[ny] = 0
    Ey[:, 0] = Ey[:, nx] = 0
    xs = []
    for m, i0, j0 in ordered_instances(scene):
        bx, by, q1, q2 = m["bx"], m["by"], m["q1"], m["q2"]
        Hz[j0:j0 + by, i0:i0 + bx] = 0
        Ex[j0 + 1:j0 + by, i0:i0 + bx] = 0
        Ey[j0:j0 + by, i0 + 1:i0 + bx] = 0
        xt = rng.standard_normal(q1 + q2)
        xt[q1:] /= 377.0
        y = m["L"].T @ xt[:q1]
        Ex[j0, i0:i0 + bx] = y[:bx]
        Ex[j0 + by, i0:i0 + bx] = y[bx:2 * bx]
        Ey[j0:j0 + by, i0] = y[2 * bx:2 * bx + by]
        Ey[j0:j0 + by, i0 + bx] = y[2 * bx + by:]
        xs.append(xt)
    return Ex, Ey, Hz, (np.concatenate(xs) if xs else np.zeros(0))
