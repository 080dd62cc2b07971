"""Small hot-path runs for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize.py --case cfg1 --k 2

The library allocates with cudaMalloc here (no PyTorch caching allocator), so memcheck sees every
device buffer's true bounds -- including the 32 KB tails the sweep's lanes past the last column
load from.  Every kernel of a pass runs: the K-step sweep, the ROM fix-up (cp.async region loads),
the CPML band fix-up (--pml) and the finalize kernel (energy on: its done-counter / last-block
reduction)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="cfg1", choices=["cfg1", "cfg3crop", "pml"])
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--steps", type=int, default=12)
    a = ap.parse_args()
    import numpy as np

    from helpers import consistent_random_state, gpu_from_scene
    from inputs import configs

    if a.case == "cfg1":
        s = configs.make("cfg1")
    elif a.case == "cfg3crop":
        s = configs.make("cfg3", n=256)
    else:
        from test_gpu_pml import channel_scene
        s = channel_scene(32, nx=120, ny=40, rom=True)
    g = gpu_from_scene(s, torch_allocator=False)
    g.set_time_blocking(a.k)
    Ex, Ey, Hz, xs = consistent_random_state(s, 3)
    g.set_window(0, 0, Ex, Ey, Hz)
    if xs.size:
        g.set_rom_state(xs)
    g.record_energy(True)
    g.step(a.steps)
    p, e = g.probe(), g.energy()
    info = g.info()
    print("case %s K requested %d used %d steps %d launches %d finite %s" % (
        a.case, a.k, info.steps_per_pass, a.steps, info.kernel_launches,
        bool(np.all(np.isfinite(p)) and np.all(np.isfinite(e)))))
    g.close()


if __name__ == "__main__":
    main()
