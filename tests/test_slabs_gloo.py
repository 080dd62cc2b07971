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
