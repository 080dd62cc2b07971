"""The slab halo protocol on CPU (-m "not gpu"): the fp64 oracle split into 2 row slabs over a
world-size-2 gloo group, exchanging exactly the rows of DESIGN.md "Multi-GPU" before each step,
is bit-identical to the undivided oracle.  Uses the same partition helpers as bench.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _scene():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_slabs import slab_scene
    s = slab_scene(64)
    s.steps = 120
    return s


def _window(s, rb, re):
    """Oracle over rows [rb-1, re) (ghost row below when rb > 0); returns (sim, row0)."""
    import oracle as O
    from paper_1609_07114_b200 import slabs
    r0 = max(rb - 1, 0)
    w = O.OracleSim(s.nx, re - r0, s.dx, s.dy, s.dt, s.eps_r[r0:re], s.sigma[r0:re])
    own = slabs.owned_placements(s.placements, s.models, rb, re)
    for mk, m in enumerate(s.models):
        for k, i0, j0 in own:
            if k == mk:
                w.add_rom(m, int(i0), int(j0) - r0)
    if r0 <= s.source[1] < re:
        w.set_source(s.source[0], s.source[1] - r0, s.samples)
    return w, r0


def _worker(rank, world, port, q):
    import torch
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    from paper_1609_07114_b200 import slabs
    s = _scene()
    rb, re = slabs.slab_rows(s.ny, world, rank)
    w, r0 = _window(s, rb, re)
    lr = lambda g: g - r0  # global -> window row
    for _ in range(s.steps):
        Ex, Ey, Hz, xs = w.get_state()
        # plan: top owned row (Ex, Ey, Hz) -> rank+1's ghost row; bottom owned Ex row -> rank-1's top Ex row
        reqs = []
        if rank + 1 < world:
            for a in (Ex[lr(re - 1)], Ey[lr(re - 1)], Hz[lr(re - 1)]):
                dist.send(torch.from_numpy(np.ascontiguousarray(a)), rank + 1)
            t = torch.zeros(s.nx, dtype=torch.float64)
            dist.recv(t, rank + 1)
            Ex[lr(re)] = t.numpy()
        if rank - 1 >= 0:
            bufs = [torch.zeros(s.nx, dtype=torch.float64), torch.zeros(s.nx + 1, dtype=torch.float64),
                    torch.zeros(s.nx, dtype=torch.float64)]
            for t in bufs:
                dist.recv(t, rank - 1)
            Ex[0], Ey[0], Hz[0] = (t.numpy() for t in bufs)
            dist.send(torch.from_numpy(np.ascontiguousarray(Ex[lr(rb)])), rank - 1)
        w.set_state(Ex, Ey, Hz, xs if xs.size else None)
        w.step(1, probes=False, energy=False)
    Ex, Ey, Hz, _ = w.get_state()
    q.put((rank, rb, re, Ex[lr(rb):lr(re)], Ey[lr(rb):lr(re)], Hz[lr(rb):lr(re)]))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_oracle_slabs_over_gloo_equal_undivided():
    import oracle as O
    s = _scene()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.OracleSim(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r, s.sigma)
    for mk, m in enumerate(s.models):
        for k, i0, j0 in s.placements:
            if k == mk:
                full.add_rom(m, int(i0), int(j0))
    full.set_source(*s.source, s.samples)
    full.step(s.steps, probes=False, energy=False)
    Ex, Ey, Hz, _ = full.get_state()
    for rank, rb, re, ex, ey, hz in parts:
        assert np.array_equal(ex, Ex[rb:re]), rank
        assert np.array_equal(ey, Ey[rb:re]), rank
        assert np.array_equal(hz, Hz[rb:re]), rank


def _pml_scene():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_pml import channel_scene
    s = channel_scene(64, ny=40)
    s.steps = 150
    return s


def _pml_worker(rank, world, port, q):
    """NEXT-2 on slabs: as _worker, plus the CPML psi rows of the ghost row (psi_ey with Ey, psi_hz
    with Hz; the plan of fdtd_api.cpp halo_plan) and a line source spanning both slabs."""
    import torch
    import oracle as O
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    from paper_1609_07114_b200 import slabs
    s = _pml_scene()
    rb, re = slabs.slab_rows(s.ny, world, rank)
    r0 = max(rb - 1, 0)
    w = O.OracleSim(s.nx, re - r0, s.dx, s.dy, s.dt, s.eps_r[r0:re], s.sigma[r0:re])
    w.set_pml(*s.meta["pml"])
    w.set_source_line(s.source[0], 0, re - r0, s.samples)
    lr = lambda g: g - r0
    f64 = lambda n: torch.zeros(n, dtype=torch.float64)
    for _ in range(s.steps):
        Ex, Ey, Hz, _ = w.get_state()
        ph, pe = w.get_psi()
        if rank + 1 < world:
            for a in (Ex[lr(re - 1)], Ey[lr(re - 1)], pe[lr(re - 1)], Hz[lr(re - 1)], ph[lr(re - 1)]):
                dist.send(torch.from_numpy(np.ascontiguousarray(a)), rank + 1)
            t = f64(s.nx)
            dist.recv(t, rank + 1)
            Ex[lr(re)] = t.numpy()
        if rank - 1 >= 0:
            bufs = [f64(s.nx), f64(s.nx + 1), f64(s.nx + 1), f64(s.nx), f64(s.nx)]
            for t in bufs:
                dist.recv(t, rank - 1)
            Ex[0], Ey[0], pe[0], Hz[0], ph[0] = (t.numpy() for t in bufs)
            dist.send(torch.from_numpy(np.ascontiguousarray(Ex[lr(rb)])), rank - 1)
        w.set_state(Ex, Ey, Hz, None)
        w.set_psi(ph, pe)
        w.step(1, probes=False, energy=False)
    Ex, Ey, Hz, _ = w.get_state()
    ph, pe = w.get_psi()
    q.put((rank, rb, re, Ex[lr(rb):lr(re)], Ey[lr(rb):lr(re)], Hz[lr(rb):lr(re)], ph[lr(rb):lr(re)],
           pe[lr(rb):lr(re)]))
    dist.destroy_process_group()


def test_oracle_cpml_slabs_over_gloo_equal_undivided():
    """The psi rows are part of the halo: with them two CPML slabs reproduce the undivided oracle
    bit for bit (fields and psi)."""
    import oracle as O
    s = _pml_scene()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pml_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.OracleSim(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r, s.sigma)
    full.set_pml(*s.meta["pml"])
    full.set_source_line(s.source[0], *s.meta["source_rows"], s.samples)
    full.step(s.steps, probes=False, energy=False)
    Ex, Ey, Hz, _ = full.get_state()
    ph, pe = full.get_psi()
    assert np.abs(ph).max() > 0 and np.abs(pe).max() > 0
    for rank, rb, re, ex, ey, hz, qh, qe in parts:
        for a, b in ((ex, Ex), (ey, Ey), (hz, Hz), (qh, ph), (qe, pe)):
            assert np.array_equal(a, b[rb:re]), rank


# ---------------------------------------------------------------------------------------------
# The product's own K-deep halo plan (fdtd_halo_plan, the plan fdtd_step's NCCL exchange and
# fdtd_step_group's device copies follow) driven over gloo: each rank advances the fp64 oracle on
# its slab plus the ghost rows the plan fills (one more, never-received row on each side stands in
# for the device buffer's stale ghost rows), exchanging exactly the plan's rows before every
# K-step pass and nothing else.  The owned rows must equal the undivided oracle bit for bit; a
# plan one row too shallow (depth K-1 for K-step passes) must not.
def _plan_scene(pml=False):
    from inputs import romgen as rg
    from inputs import scene as sc
    rng = np.random.default_rng(31)
    nx, ny = 96, 120  # three slabs of 40 rows
    dx = dy = 1e-3
    fe, fs = sc.uniform_fill(3, 2, 3, 1, 1, 4, 0, 0.05)
    m1 = rg.build_rom(3, 2, 3, dx, dy, fe, fs, 20, 30e9)
    fe, fs = sc.uniform_fill(2, 2, 4, 2, 1, 4, 0, 0.05)
    m2 = rg.build_rom(2, 2, 4, dx, dy, fe, fs, 16, 30e9)
    dt = 0.95 * min(m1["fine_dt_limit"], m2["fine_dt_limit"])
    # footprints 7 rows inside their slab (the four-step rule of fdtd_add_rom / passes_valid)
    P = np.array([[0, 10, 15], [1, 50, 20], [0, 30 if not pml else 40, 55], [1, 70 if not pml else 52, 60],
                  [0, 20 if not pml else 30, 95], [1, 60, 100]], np.int32)
    steps = 48
    meta = {}
    if pml:
        meta = dict(pml=(8, 3, 1e-8), source_rows=(30, 90))
    return sc.Scene(name="plan", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 4, (ny, nx)),
                    sigma=rng.uniform(0, 0.05, (ny, nx)), precision=64, steps=steps, source=(48, 41),
                    samples=sc.gaussian_samples(steps, dt, 30e9, True), probes=np.zeros((0, 2), np.int32),
                    models=[m1, m2], placements=P, meta=meta)


def _plan_worker(rank, world, port, q, K, depth, pml):
    import torch
    import oracle as O
    from paper_1609_07114_b200 import halo_plan, slabs
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    s = _plan_scene(pml)
    rb, re = slabs.slab_rows(s.ny, world, rank)
    w0, w1 = max(rb - K - 1, 0), min(re + K, s.ny)
    w = O.OracleSim(s.nx, w1 - w0, s.dx, s.dy, s.dt, s.eps_r[w0:w1], s.sigma[w0:w1])
    if pml:
        w.set_pml(*s.meta["pml"])
    own = slabs.owned_placements(s.placements, s.models, rb, re)
    for mk, m in enumerate(s.models):
        for k, i0, j0 in own:
            if k == mk:
                w.add_rom(m, int(i0), int(j0) - w0)
    if pml:
        a, b = s.meta["source_rows"]
        a, b = max(a, w0), min(b, w1)
        if a < b:
            w.set_source_line(s.source[0], a - w0, b - w0, s.samples)
    elif w0 <= s.source[1] < w1:
        w.set_source(s.source[0], s.source[1] - w0, s.samples)
    plan = halo_plan(world, rank, rb, re, depth, pml)
    for _ in range(s.steps // K):
        Ex, Ey, Hz, _ = w.get_state()
        arrs = [Ex, Ey, Hz]
        if pml:
            ph, pe = w.get_psi()
            arrs += [pe, pe, ph, ph]  # psi_ey left / right, psi_hz left / right (whole rows)
        keep, works = [], []
        for d, a, g, peer in plan:
            if d == 0:
                t = torch.from_numpy(np.ascontiguousarray(arrs[a][g - w0]))
                keep.append(t)
                works.append(dist.isend(t, int(peer)))
        for d, a, g, peer in plan:
            if d == 1:
                t = torch.zeros(arrs[a].shape[1], dtype=torch.float64)
                dist.recv(t, int(peer))
                arrs[a][g - w0] = t.numpy()
        for x in works:
            x.wait()
        w.set_state(Ex, Ey, Hz, None)
        if pml:
            w.set_psi(ph, pe)
        w.step(K, probes=False, energy=False)
    Ex, Ey, Hz, xs = w.get_state()
    out = [Ex[rb - w0:re - w0], Ey[rb - w0:re - w0], Hz[rb - w0:re - w0]]
    if pml:
        ph, pe = w.get_psi()
        out += [ph[rb - w0:re - w0], pe[rb - w0:re - w0]]
    q.put((rank, rb, re, out, xs, [(int(i0), int(j0)) for _, i0, j0 in own]))
    dist.destroy_process_group()


def _run_plan(world, K, depth, pml=False):
    import oracle as O
    s = _plan_scene(pml)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q, K, depth, pml)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.OracleSim(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r, s.sigma)
    if pml:
        full.set_pml(*s.meta["pml"])
    order = []
    for mk, m in enumerate(s.models):
        for k, i0, j0 in s.placements:
            if k == mk:
                full.add_rom(m, int(i0), int(j0))
                order.append((int(i0), int(j0), m["q1"] + m["q2"]))
    if pml:
        full.set_source_line(s.source[0], *s.meta["source_rows"], s.samples)
    else:
        full.set_source(*s.source, s.samples)
    full.step(s.steps, probes=False, energy=False)
    Ex, Ey, Hz, xs = full.get_state()
    ref = [Ex, Ey, Hz]
    if pml:
        ph, pe = full.get_psi()
        ref += [ph, pe]
    offs = np.cumsum([0] + [o[2] for o in order])
    where = {(o[0], o[1]): (offs[t], offs[t + 1]) for t, o in enumerate(order)}
    equal = True
    for rank, rb, re, out, xs_r, own in parts:
        for a, b in zip(out, ref):
            equal &= np.array_equal(a, b[rb:re])
        got = []  # the rank's ROM states in its own order (grouped by model)
        for mk, m in enumerate(s.models):
            for k, i0, j0 in s.placements:
                if k == mk and (int(i0), int(j0)) in own:
                    a0, a1 = where[(int(i0), int(j0))]
                    got.append(xs[a0:a1])
        equal &= np.array_equal(xs_r, np.concatenate(got) if got else np.zeros(0))
    assert np.abs(Hz).max() > 0
    return equal


@pytest.mark.parametrize("K", [1, 2, 4])
def test_product_halo_plan_over_gloo_equals_undivided(K):
    """Three ranks (one with both neighbours), K-step passes on the product's K-deep plan."""
    assert _run_plan(3, K, K)


def test_product_halo_plan_cpml_over_gloo():
    """CPML layers: the plan's psi rows (with Ey and Hz) make four-step slab passes exact."""
    assert _run_plan(3, 4, 4, pml=True)


@pytest.mark.parametrize("K", [2, 4])
def test_shallower_plan_breaks_k_step_passes(K):
    """Negative control: the plan of depth K-1 does not carry enough rows for K-step passes."""
    assert not _run_plan(3, K, K - 1)


def test_halo_plan_shape():
    """Counts of the plan: per neighbour below 3K rows received; above, Ex of K rows and Ey/Hz of
    K-1 rows; PML adds two psi rows per Ey / Hz row; slabs shorter than 4 rows are refused."""
    from paper_1609_07114_b200 import FDTDError, halo_plan
    for K in (1, 2, 4):
        p = halo_plan(3, 1, 40, 80, K)
        recv = p[p[:, 0] == 1]
        send = p[p[:, 0] == 0]
        assert (recv[:, 3] == 0).sum() == 3 * K and (recv[:, 3] == 2).sum() == K + 2 * (K - 1)
        assert (send[:, 3] == 2).sum() == 3 * K and (send[:, 3] == 0).sum() == K + 2 * (K - 1)
        below = recv[recv[:, 3] == 0]
        assert set(below[:, 2]) == set(range(40 - K, 40))
        above = recv[recv[:, 3] == 2]
        assert set(above[above[:, 1] == 0][:, 2]) == set(range(80, 80 + K))
        pp = halo_plan(3, 1, 40, 80, K, pml=True)
        assert len(pp) == len(p) + 2 * (p[:, 1] != 0).sum()
    assert len(halo_plan(1, 0, 0, 100, 4)) == 0
    with pytest.raises(FDTDError):
        halo_plan(2, 0, 0, 3, 4)
