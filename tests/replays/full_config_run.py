"""Full-length runs of the bench configurations on the GPU (north_star's energy criterion at full size).

Each config runs its own step count (`inputs/configs.py`: cfg2 10,000 steps, cfg3 10,000, cfg4
5,000, cfg5 2,000) with the storage function W^n (eq:R, R17) recorded every step and the
64 probes, read back every `--chunk` steps.  Reported per config: every value finite; after the last
source sample (|g| below 1e-6 of its peak) the largest relative step increase of W^n, which must stay
at fp32 roundoff (north_star: "the GPU energy trace never increasing beyond fp32 roundoff (1e-6
relative)" -- the configs' media are lossy, so W^n decays); and the device time per step.  The oracle
cannot run these grids; parity at full size is sampled by tests/test_gpu_fullsize.py.

    python tests/replays/full_config_run.py --out gpurun_out/full_config_run.json [--configs cfg4 ...]
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


def run(name, chunk):
    import torch

    from inputs import configs
    from paper_1609_07114_b200 import from_scene

    s = configs.make(name, device="cuda")
    sim = from_scene(s, device=0)
    sim.record_energy(True)
    steps = int(s.steps)
    W, P = [], []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        n = min(chunk, steps - done)
        sim.step(n)
        P.append(sim.probe())
        W.append(sim.energy())
        done += n
    wall = time.perf_counter() - t0
    W = np.concatenate(W)
    P = np.concatenate(P, axis=1)
    g = np.abs(np.asarray(s.samples, dtype=np.float64))
    src_end = int(np.nonzero(g > 1e-6 * g.max())[0].max()) + 1 if g.size else 0
    tail = W[src_end:]
    inc = np.diff(tail) / np.maximum(np.abs(tail[:-1]), 1e-300) if tail.size > 1 else np.zeros(0)
    info = sim.info()
    out = {
        "config": name, "nx": s.nx, "ny": s.ny, "steps": steps, "instances": int(info.n_instances),
        "steps_per_pass": int(info.steps_per_pass), "finite": bool(np.isfinite(W).all() and np.isfinite(P).all()),
        "source_end_step": src_end, "W_peak": float(W.max()), "W_at_source_end": float(W[min(src_end, steps - 1)]),
        "W_final": float(W[-1]), "max_rel_step_increase_after_source": float(inc.max()) if inc.size else 0.0,
        "energy_non_increasing_1e-6": bool(inc.size == 0 or inc.max() <= 1e-6),
        "probe_max_abs": float(np.abs(P).max()), "wall_s_incl_readback": wall,
        "ms_per_step_incl_readback": 1e3 * wall / steps,
    }
    sim.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--chunk", type=int, default=500)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for c in a.configs:
        r = run(c, a.chunk)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if a.out:
        json.dump({"tool": "tests/replays/full_config_run.py", "rows": rows}, open(a.out, "w"), indent=1)
    return 0 if all(r["finite"] and r["energy_non_increasing_1e-6"] for r in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
