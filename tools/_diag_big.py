import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from inputs import romgen as rg, scene as sc
from helpers import gpu_from_scene, consistent_random_state
nx = ny = 64; dx = dy = 1e-3
fe, fs = sc.uniform_fill(6, 6, 5, 31, 1, 4, 0, 0.05)
m = rg.build_rom(6, 6, 5, dx, dy, fe, fs, int(sys.argv[2]), 30e9)
dt = 0.95 * m["fine_dt_limit"]
rng = np.random.default_rng(2)
s = sc.Scene(name="bigq", nx=nx, ny=ny, dx=dx, dy=dy, dt=dt, eps_r=rng.uniform(1, 3, (ny, nx)),
             sigma=rng.uniform(0, 0.05, (ny, nx)), precision=int(sys.argv[1]), steps=800, source=(10, 10),
             samples=sc.gaussian_samples(800, dt, 30e9, True), probes=np.array([[50, 50], [30, 12]], np.int32),
             models=[m], placements=np.array([[0, 29, 30]], np.int32))
g = gpu_from_scene(s)
for k in (1, 2, 4):
    g.set_time_blocking(k)
    for e in (False, True):
        g.record_energy(e)
        g.step(3); g.sync()
        print("K", k, "energy", e, "ok", g.info().steps_per_pass, g.info().big_instances, flush=True)
