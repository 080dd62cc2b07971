"""Replay of the paper's Sec. VI-A stability experiment (Fig. 4) on the GPU.

1 m x 1 m PEC cavity, coarse 2 mm (500 x 500 cells), a central 20 mm x 20 mm block (10 x 10 coarse
cells, R14) refined r = 5 (N^ = 50, full order 7,600, L840) reduced to order 1,200
(q1 = q2 = 600) with SPRIM at f_max = 0.5 GHz, CFL limit extended 2x by the clip (L840), run at
1.98 x the fine-grid limit (L842 "1.98%" = 1.98x), empty (vacuum) cavity, Gaussian pulse of
0.5 GHz bandwidth at (0.089, 0.089) m, probe at (0.933, 0.933) m (read off the schematic TikZ,
L776-779), 10^6 steps in fp64.  Coupling: the collapsed reading R9, or with --literal the paper's own
eq:sysform through the nP = 200 fine hanging variables (T, 1/r; NEXT-1): the E basis holds the 200
port directions plus 500 SPRIM directions, q1 = 700, q2 = 500 (order 1,200 as in L840).

Reports: the fp64 parity of the first `--check` steps against the oracle, the boundedness of the
probe (max over the last 10 % vs the first 10 %, SPEC.md criterion 6), the storage-function drift
(lossless: conserved), and the device time.  Writes a JSON summary.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import romgen as rg  # noqa: E402
from inputs import scene as sc  # noqa: E402


def build(steps, literal=False):
    nx = ny = 500
    dx = dy = 2e-3
    b, r = 10, 5
    i0 = j0 = 245
    fe = np.ones((b * r, b * r))
    fs = np.zeros_like(fe)
    sysf = rg.fine_system(b, b, r, dx, dy, fe, fs)
    assert rg.full_order(sysf) == 7600
    if literal:
        cs = rg.literal_system(sysf)
        V1, V2 = rg.sprim_basis(cs, 1000, 0.5e9)
        V1 = rg.with_port_directions(V1, cs["nY"])[:, : cs["nY"] + 500]
    else:
        cs = rg.collapse(sysf)
        V1, V2 = rg.sprim_basis(cs, 1200, 0.5e9)
    m = rg.reduce(cs, V1, V2)
    dtf = rg.fine_cfl_limit(sysf)
    m["natural_dt_limit"] = rg.rom_cfl_limit(m)
    m = rg.extend_cfl(m, 2.0 * dtf)
    dt = 1.98 * dtf
    samples = sc.gaussian_samples(steps, dt, 0.5e9)
    scene = sc.Scene(name="cavity_VI_A", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=np.ones((ny, nx)),
                     sigma=np.zeros((ny, nx)), precision=64, steps=steps, source=(44, 44), samples=samples,
                     probes=np.array([[466, 466]], dtype=np.int32), models=[m],
                     placements=np.array([[0, i0, j0]], dtype=np.int32),
                     meta=dict(dt_f=dtf, q=(m["q1"], m["q2"]), n_clipped=m["n_clipped"],
                               natural_dt_limit=m["natural_dt_limit"]))
    return scene


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1_000_000)
    ap.add_argument("--check", type=int, default=2000)
    ap.add_argument("--literal", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.out is None:
        args.out = os.path.join(ROOT, "profiles", "r01_cavity_replay%s.json" % ("_literal" if args.literal else ""))
    import torch

    import oracle as O
    from paper_1609_07114_b200 import Simulation

    t0 = time.time()
    s = build(args.steps, args.literal)
    t_build = time.time() - t0
    m = s.models[0]
    sim = Simulation(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r, s.sigma, precision=64,
                     record_capacity=args.steps + 16)
    sim.add_rom(m, s.placements[:, 1:3])
    sim.set_source(*s.source, s.samples)
    sim.set_probes(s.probes)
    sim.record_energy(True)
    # fp64 parity of the first `check` steps against the oracle
    o = O.OracleSim(s.nx, s.ny, s.dx, s.dy, s.dt, s.eps_r, s.sigma)
    o.add_rom(m, 245, 245)
    o.set_source(*s.source, s.samples)
    o.set_probes(s.probes)
    po, eo = o.step(args.check)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(sim.stream)
    sim.step(args.check)
    ev1.record(sim.stream)
    pg = sim.probe()
    eg = sim.energy()
    Exg, Eyg, Hzg = sim.get_window()
    Exo, Eyo, Hzo, _ = o.get_state()
    rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    parity = dict(steps=args.check, probe=rel(pg, po), Hz=rel(Hzg, Hzo), Ex=rel(Exg, Exo), Ey=rel(Eyg, Eyo),
                  energy=rel(eg, eo))
    # the long run
    probe = [pg[0]]
    energy = [eg]
    rest = args.steps - args.check
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(sim.stream)
    done = 0
    while done < rest:
        k = min(100_000, rest - done)
        sim.step(k)
        probe.append(sim.probe()[0])
        energy.append(sim.energy())
        done += k
    e3.record(sim.stream)
    torch.cuda.synchronize()
    p = np.concatenate(probe)
    e = np.concatenate(energy)
    n10 = max(1, len(p) // 10)
    src_off = args.check + 2000  # energy after the source has switched off (t > t0 + 5 tau)
    tau = sc.pulse_tau(0.5e9)
    k_off = int(np.ceil((4.5 * tau + 6 * tau) / s.dt))
    e_after = e[k_off:] if k_off < len(e) else e[-1:]
    out = dict(
        experiment="PAPER.md Sec. VI-A cavity (Fig. 4), %s" % (
            "paper-literal coupling (eq:sysform with T, 1/r; nP = 200)" if args.literal else "collapsed coupling (R9)"),
        grid=[s.nx, s.ny], dx=s.dx, block=[245, 245, 10, 10], r=5, full_order=7600,
        reduced_order=int(m["q1"] + m["q2"]), q1q2=[int(m["q1"]), int(m["q2"])],
        dt=s.dt, dt_over_fine_limit=s.dt / s.meta["dt_f"], natural_rom_limit_over_fine=m["natural_dt_limit"] /
        s.meta["dt_f"], n_clipped=int(m["n_clipped"]), steps=int(len(p)),
        parity_first_steps=parity,
        probe_max_first_10pct=float(np.abs(p[:n10]).max()), probe_max_last_10pct=float(np.abs(p[-n10:]).max()),
        bounded=bool(np.abs(p[-n10:]).max() <= 2 * np.abs(p[:n10]).max() and np.all(np.isfinite(p))),
        energy_after_source_rel_drift=float((e_after.max() - e_after.min()) / e_after[0]),
        energy_max_step_increase_rel=float(np.max(np.diff(e_after) / e_after[:-1])) if len(e_after) > 1 else 0.0,
        device_ms_first=ev0.elapsed_time(ev1), device_ms_rest=e2.elapsed_time(e3),
        ms_per_step=(ev0.elapsed_time(ev1) + e2.elapsed_time(e3)) / len(p),
        rom_build_s=t_build, steps_per_pass=int(sim.info().steps_per_pass))
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    np.save(args.out.replace(".json", "_probe_decimated.npy"), p[::100])
    sim.close()


if __name__ == "__main__":
    main()
