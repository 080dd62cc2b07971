"""Config 1 (and other small scenes) through both hot paths: the K-step sweep + fix-up passes
(CUDA graphs of two passes) and the whole-grid kernel (K3c, one launch per call).

    python tools/wholegrid_bench.py [--out profiles/rNN_wholegrid.json]

Times fdtd_step(n) with CUDA events on the library stream after a warm-up (the same call
shape: one call of `steps` steps), energy and probes recorded every step."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    from inputs import configs
    from paper_1609_07114_b200 import from_scene

    rows = []
    for name in ("cfg1", "cfg1b", "cfg1lit"):
        s = configs.make(name)
        for whole in (False, True):
            sim = from_scene(s, device=0, whole_grid=whole, record_capacity=4 * s.steps + 16)
            sim.record_energy(True)
            sim.step(s.steps)  # warm-up (graph capture, first launch)
            sim.sync()
            sim.probe()
            sim.energy()
            ts = []
            for _ in range(a.reps):
                l0 = sim.info().kernel_launches
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(sim.stream)
                sim.step(s.steps)
                e1.record(sim.stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
                launches = sim.info().kernel_launches - l0
                sim.probe()
                sim.energy()
            info = sim.info()
            ms = sorted(ts)[len(ts) // 2]
            r = dict(scene=name, path="whole-grid" if info.whole_grid else "sweep + fix-up passes",
                     nx=s.nx, ny=s.ny, instances=int(info.n_instances), precision=s.precision, steps=s.steps,
                     ms_total=ms, us_per_step=1e3 * ms / s.steps, launches_per_call=int(launches),
                     cell_updates_per_s=s.nx * s.ny * s.steps / (ms * 1e-3), steps_per_pass=int(info.steps_per_pass))
            print(json.dumps(r))
            rows.append(r)
            sim.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(dict(tool="tools/wholegrid_bench.py", gpu=torch.cuda.get_device_name(0), rows=rows), f, indent=1)


if __name__ == "__main__":
    main()
