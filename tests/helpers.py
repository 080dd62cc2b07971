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
    if "pml" in scene.meta:
        s.set_pml(*scene.meta["pml"])
    if source:
        if "source_rows" in scene.meta:
            s.set_source_line(scene.source[0], *scene.meta["source_rows"], scene.samples)
        else:
            s.set_source(*scene.source, scene.samples)
    if probes:
        s.set_probes(scene.probes)
    return s


def gpu_from_scene(scene, source=True, probes=True, **kw):
    """The CUDA path for a scene.  whole_grid defaults to False here: the parity tests exercise the
    sweep + fix-up passes even on grids small enough for the whole-grid path (K3c), which
    tests/test_gpu_wholegrid.py covers (and compares with the passes bit for bit)."""
    from paper_1609_07114_b200 import Simulation
    kw.setdefault("whole_grid", False)
    eps, sig = np_materials(scene)
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, eps, sig, precision=scene.precision, **kw)
    if "pml" in scene.meta:
        sim.set_pml(*scene.meta["pml"])
    if scene.placements is not None:
        for k, m in enumerate(scene.models):
            sel = scene.placements[scene.placements[:, 0] == k]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
    if source:
        if "source_rows" in scene.meta:
            sim.set_source_line(scene.source[0], *scene.meta["source_rows"], scene.samples)
        else:
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
        if m.get("literal", False):  # T y = L~^T E~ would constrain E~; start the ROM at rest
            xt[:] = 0.0
        y = (m["L"].T @ xt[:q1])[: 2 * bx + 2 * by]
        Ex[j0, i0:i0 + bx] = y[:bx]
        Ex[j0 + by, i0:i0 + bx] = y[bx:2 * bx]
        Ey[j0:j0 + by, i0] = y[2 * bx:2 * bx + by]
        Ey[j0:j0 + by, i0 + bx] = y[2 * bx + by:]
        xs.append(xt)
    return Ex, Ey, Hz, (np.concatenate(xs) if xs else np.zeros(0))


# ------------------------------------------------------------------ light-cone windows
def instance_boxes(scene):
    """(i0-1, j0-1, i0+bx+1, j0+by+1) footprint + ring boxes (half-open), in placement order."""
    out = []
    if scene.placements is None:
        return out
    for k, i0, j0 in scene.placements:
        m = scene.models[k]
        out.append((int(i0) - 1, int(j0) - 1, int(i0) + m["bx"] + 1, int(j0) + m["by"] + 1))
    return out


def _inter(a, b):
    return a[0] < b[2] and b[0] < a[2] and a[1] < b[3] and b[1] < a[3]


def _union(a, b):
    return (min(a[0], b[0]), min(a[1], b[1]), max(a[2], b[2]), max(a[3], b[3]))


def cone_window(scene, box, nsteps, margin=3):
    """A window (half-open cell box) that contains the backward dependency cone of `box` over
    `nsteps` steps: one cell per half-step pair, plus a whole ROM footprint + ring whenever the
    cone touches it (a ROM couples all its ports within one step).  Instances touching the
    window are included whole."""
    inst = instance_boxes(scene)
    B = box
    for _ in range(nsteps + 1):
        B = (B[0] - 1, B[1] - 1, B[2] + 1, B[3] + 1)
        changed = True
        while changed:
            changed = False
            for r in inst:
                if _inter(B, r) and _union(B, r) != B:
                    B = _union(B, r)
                    changed = True
    W = (B[0] - margin, B[1] - margin, B[2] + margin, B[3] + margin)
    changed = True
    while changed:
        changed = False
        for r in inst:
            if _inter(W, r) and _union(W, r) != W:
                W = _union(W, r)
                changed = True
    return (max(W[0], 0), max(W[1], 0), min(W[2], scene.nx), min(W[3], scene.ny))


# ------------------------------------------------------------------ per-instance checks
def instance_y(m, i0, j0, Ex, Ey, a0=0, b0=0):
    """The nY interface values y (ports S, N, W, E) of an instance at (i0, j0), read from window
    arrays whose lower-left cell is (a0, b0)."""
    bx, by = m["bx"], m["by"]
    u, v = i0 - a0, j0 - b0
    return np.concatenate([Ex[v, u:u + bx], Ex[v + by, u:u + bx], Ey[v:v + by, u], Ey[v:v + by, u + bx]])


def per_instance_errors(pairs, floor_frac=1e-3):
    """pairs: list of (got, ref) vectors, one per instance.  Returns (max per-instance relative L2,
    max per-instance relative max-abs).  Each instance is normalised by its own reference norm,
    floored at floor_frac of the largest instance's (so that an instance still at rest is not
    divided by dust): one bad instance among thousands cannot hide in a global norm."""
    if not pairs:
        return 0.0, 0.0
    gl2 = max(np.linalg.norm(r) for _, r in pairs)
    gmx = max(np.abs(r).max() if r.size else 0.0 for _, r in pairs)
    l2 = mx = 0.0
    for g, r in pairs:
        if r.size == 0:
            continue
        d = np.asarray(g, np.float64) - np.asarray(r, np.float64)
        l2 = max(l2, np.linalg.norm(d) / max(np.linalg.norm(r), floor_frac * gl2, 1e-300))
        mx = max(mx, np.abs(d).max() / max(np.abs(r).max(), floor_frac * gmx, 1e-300))
    return float(l2), float(mx)


def split_states(scene, xs):
    """Split a concatenated ROM state vector into per-instance vectors (ordered_instances order)."""
    out, o = [], 0
    for m, _, _ in ordered_instances(scene):
        q = m["q1"] + m["q2"]
        out.append(np.asarray(xs[o:o + q]))
        o += q
    return out


def instance_pairs(scene, Wg, Wo, xg, xo):
    """Per-instance (got, ref) pairs of x~ and of y for whole-grid windows Wg, Wo = (Ex, Ey, Hz)."""
    px = list(zip(split_states(scene, xg), split_states(scene, xo)))
    py = [(instance_y(m, i0, j0, Wg[0], Wg[1]), instance_y(m, i0, j0, Wo[0], Wo[1]))
          for m, i0, j0 in ordered_instances(scene)]
    return px, py
