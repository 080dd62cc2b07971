"""Row-slab decomposition cost on one GPU: config 4 advanced as N in-process slab
contexts (the halo plan executed as device copies, the first / last row chunks of every slab split
off as for NCCL) against one context, same GPU, same steps.  The N slabs run one after another on
one stream, so their summed time against the single context is the decomposition's own overhead
(ghost-row recomputation, split launches, halo copies, no CUDA graph) -- what an N-GPU run adds per
GPU before any communication cost.  Writes profiles/r01_slab_overhead.json.
Run under gpurun:  python tools/slab_overhead.py
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import configs  # noqa: E402
from paper_1609_07114_b200 import Simulation, slabs, step_group  # noqa: E402


def build(scene, n, stream):
    sims = []
    for k in range(n):
        rb, re = slabs.slab_rows(scene.ny, n, k)
        m0, m1 = max(rb - 4, 0), min(re + 4, scene.ny)
        sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, scene.eps_r[m0:m1].contiguous(),
                         scene.sigma[m0:m1].contiguous(), precision=scene.precision, stream=stream, rank=k,
                         nranks=n, row_begin=rb, row_end=re, materials_row0=m0, local_group=n > 1)
        P = slabs.owned_placements(scene.placements, scene.models, rb, re)
        for mk, m in enumerate(scene.models):
            sel = P[P[:, 0] == mk]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
        sim.set_source(*scene.source, scene.samples)
        sim.set_probes(scene.probes)
        sim.record_energy(True)
        sims.append(sim)
    return sims


def timed(sims, steps):
    adv = (lambda k: step_group(sims, k)) if len(sims) > 1 else (lambda k: sims[0].step(k))
    adv(16)
    for s in sims:
        s.sync()
    t0 = time.perf_counter()
    adv(steps)
    for s in sims:
        s.sync()
    dt = time.perf_counter() - t0
    for s in sims:
        s.energy()
        s.probe()
    return dt * 1e3 / steps


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=96)
    ap.add_argument("--slabs", default="1,2,4,8")
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--slab-chunk", type=int, default=0, help="rows per CTA on the slab contexts (0: default)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_slab_overhead.json"))
    a = ap.parse_args()
    scene = configs.make(a.workload, device="cuda")
    stream = torch.cuda.Stream()
    rows = []
    base = None
    for n in [int(x) for x in a.slabs.split(",")]:
        sims = build(scene, n, stream)
        if n > 1 and a.slab_chunk:
            for sim in sims:
                sim.set_tuning(a.slab_chunk, 0)
        ms = timed(sims, a.steps)
        for sm in sims:
            sm.profile(True)
        (lambda k: step_group(sims, k)) (16) if n > 1 else sims[0].step(16)
        prof = [sm.profile_read() for sm in sims]
        for sm in sims:
            sm.profile(False)
        sweep_ms = sum(p_[0] / max(p_[2], 1) for p_ in prof)  # per pass, summed over the slabs
        post_ms = sum(p_[1] / max(p_[2], 1) for p_ in prof)
        for s in sims:
            s.close()
        del sims
        torch.cuda.empty_cache()
        base = base or ms
        rows.append(dict(slabs=n, ms_per_step=ms, overhead=ms / base - 1.0,
                         cell_updates_per_s=scene.nx * scene.ny / ms * 1e3,
                         per_pass_sum_over_slabs_ms=dict(sweep=sweep_ms, fixup=post_ms)))
        print(json.dumps(rows[-1]), flush=True)
    out = dict(what="%s as N in-process row slabs on one B200 (sequential on one stream) vs one context" % a.workload,
               steps=a.steps, rows=rows)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
