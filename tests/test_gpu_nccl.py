"""The real NCCL row-slab transport (-m gpu, needs >= 2 visible GPUs; skipped otherwise): two
processes, one per GPU, each a rank of fdtd_create's NCCL communicator, run the K-step passes with
the K-row halo exchange of fdtd_halo_plan.  Gathered fields, ROM states, probes and energy must
match the fp64 oracle (fp64 1e-10, fp32 1e-4) and the one-GPU run bit for bit (energy: summation
order)."""
import os
import socket

import numpy as np
import pytest

from helpers import consistent_random_state, gpu_from_scene, oracle_from_scene, ordered_instances, rel

pytestmark = pytest.mark.gpu
N_STEPS = 301


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _rank(rank, world, port, precision, q):
    import torch
    import torch.distributed as dist

    from paper_1609_07114_b200 import Simulation, nccl_unique_id, slabs
    from test_gpu_slabs import slab_scene
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    s = slab_scene(precision)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone()
    dist.broadcast(t, 0)
    rb, re = slabs.slab_rows(s.ny, world, rank)
    m0, m1 = max(rb - 4, 0), min(re + 4, s.ny)
    sim = Simulation(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r[m0:m1], s.sigma[m0:m1], precision=precision,
                     device=rank, rank=rank, nranks=world, nccl_id=bytes(t.numpy().tobytes()), row_begin=rb,
                     row_end=re, materials_row0=m0)
    Ex, Ey, Hz, xs = consistent_random_state(s, 3)
    glob = ordered_instances(s)
    offs = np.cumsum([0] + [m["q1"] + m["q2"] for m, _, _ in glob])
    own = slabs.owned_placements(s.placements, s.models, rb, re)
    mine = []
    for mk, m in enumerate(s.models):  # collective: every rank adds every model
        sel = own[own[:, 0] == mk]
        sim.add_rom(m, sel[:, 1:3])
        mine += [next(k for k, (mm, a, b) in enumerate(glob) if (a, b) == (int(i0), int(j0))) for _, i0, j0 in sel]
    sim.set_source(*s.source, s.samples)
    sim.set_probes(s.probes)
    sim.record_energy(True)
    sim.set_window(0, 0, Ex, Ey, Hz)
    if mine:
        sim.set_rom_state(np.concatenate([xs[offs[k]:offs[k + 1]] for k in mine]))
    sim.step(N_STEPS)
    pr, en = sim.probe(), sim.energy()  # collective reads: summed over ranks
    W = sim.get_window()
    st = sim.get_rom_state()
    info = sim.info()
    q.put((rank, W, st, mine, pr, en, info.steps_per_pass))
    sim.close()
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs (NCCL refuses two ranks on one device)")
@pytest.mark.parametrize("precision", [32, 64])
def test_two_rank_nccl_matches_oracle_and_one_gpu(precision):
    import torch.multiprocessing as mp

    from test_gpu_slabs import run_single, slab_scene
    s = slab_scene(precision)
    init = consistent_random_state(s, 3)
    (W1, x1, p1, e1) = run_single(s, N_STEPS, init)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    env_path = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = env_path + os.pathsep + os.environ.get("PYTHONPATH", "")
    procs = [ctx.Process(target=_rank, args=(r, 2, port, precision, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    glob = ordered_instances(s)
    offs = np.cumsum([0] + [m["q1"] + m["q2"] for m, _, _ in glob])
    W = [np.zeros_like(a) for a in W1]
    xs = np.zeros_like(x1)
    for rank, w, st, mine, pr, en, spp in res:
        assert spp == (4 if precision == 32 else 2)
        for a, b in zip(W, w):
            a += b
        o = 0
        for k in mine:
            n = offs[k + 1] - offs[k]
            xs[offs[k]:offs[k + 1]] = st[o:o + n]
            o += n
        assert np.array_equal(pr, p1)  # every rank holds the rank-summed records
        np.testing.assert_allclose(en, e1, rtol=1e-12 if precision == 64 else 1e-6)
    for a, b in zip(W, W1):
        assert np.array_equal(a, b)
    assert np.array_equal(xs, x1)
    o = oracle_from_scene(s)
    Ex, Ey, Hz, xo = init
    o.set_state(Ex, Ey, Hz, xo)
    po, eo = o.step(N_STEPS)
    Exo, Eyo, Hzo, xso = o.get_state()
    tol = 1e-10 if precision == 64 else 1e-4
    errs = dict(Ex=rel(W[0], Exo), Ey=rel(W[1], Eyo), Hz=rel(W[2], Hzo), rom=rel(xs, xso), probe=rel(res[0][4], po),
                energy=rel(res[0][5], eo))
    assert max(errs.values()) <= tol, errs
