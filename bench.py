#!/usr/bin/env python
"""Benchmark of the hot path: coarse-grid cell-updates/s incl. ROMs (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg4]

A "step" is one time step of the whole hot path (S1..S8 of DESIGN.md) over the
workload.  Default workload: BASELINE config 4 (the metric's 1/2/4/8-GPU
config): 32768^2 fp32 coarse grid, smooth random lossy medium, 4096 instances of
one ROM (16x16 block, r = 4, q = 128), source, 64 probes and the energy trace
recorded every step.  N > 1: one rank per GPU (bench.py re-launches itself under
torch.distributed.run when it is not already a torchrun rank, and fails when fewer than N GPUs
are visible), row slabs of 32768/N rows with the K-row NCCL halo exchange per K-step pass
(strong scaling).
``--impl reference`` times the fp64 CPU oracle (the base contract's reference
arm for this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "coarse-grid cell-updates/s incl. ROMs"
UNIT = "cell-updates/s"
WORKLOADS = {
    "cfg4": "BASELINE config 4: 32768^2 fp32 coarse TEz grid, copula medium eps_r U[1,10] sigma U[0,0.1] l=32, "
            "4096 instances of one ROM (16x16 coarse block, r=4, disc inclusion, q=128, clipped at 2 dt_f), "
            "dt = 1.9 dt_f, Gaussian source, 64 probes, energy every step",
    "cfg4dense": "BASELINE config 4 with SURVEY Q19's placement rule (footprint + one-cell ring disjoint, 1 cell "
                 "from the walls and slab rows): close instances are fixed up as clusters",
    "cfg3": "BASELINE config 3: 8192^2 fp32, 1024 instances of one ROM (8x8 block, r=8, q=64), dt = 1.9 dt_f",
    "cfg2": "BASELINE config 2: 8192^2 fp32 plain grid, no ROMs, dt = 0.99 eq.(1)",
    "cfg5": "BASELINE config 5: 49152^2 fp32, copula medium, 32 distinct ROM models (b 4..32, r 4..10, "
            "q in {32,64,128,256}, uniform fills eps_r U[1,12] sigma U[0,0.2]), 8192 placements, dt = 1.9 min dt_f "
            "(the 8-GPU config, run here on the GPUs given)",
}
SAMPLE_N = 1024  # bounded CPU sample: a seeded 1024^2 sub-instance of the same recipe


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, lrank


def kernel_source_sha():
    """Hash of the sources that define the kernels and their build flags: the ncu traffic recorded
    in profiles/sweep_traffic.json is only valid for the build it was measured on."""
    import hashlib
    h = hashlib.sha256()
    for f in ("paper_1609_07114_b200/csrc/fdtd_kernels.cu", "paper_1609_07114_b200/csrc/fdtd_kernels.cuh",
              "paper_1609_07114_b200/build.py"):
        h.update(open(os.path.join(ROOT, f), "rb").read())
    return h.hexdigest()[:16]


def ensure_ranks(args):
    """--gpus N > 1 outside torchrun: re-launch this command as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; fail loudly when fewer than N GPUs are visible."""
    ws, _, _ = dist_env()
    if "WORLD_SIZE" in os.environ:
        if ws != args.gpus:
            sys.exit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, ws))
        return
    if args.gpus <= 1:
        return
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit("bench.py: --gpus %d but only %d CUDA device(s) visible" % (args.gpus, have))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------ CPU oracle timing
def oracle_rate(workload, steps, max_seconds=None, threads=0):
    """Time the fp64 oracle (as it stands) on the bounded sample; cell-updates/s.

    threads = 0: all host cores (OpenMP over rows); 1: the plain single-threaded oracle."""
    import oracle as O
    from inputs import configs

    O.set_threads(threads)
    nthreads = O.get_threads()

    s = configs.make(workload, n=SAMPLE_N)
    eps, sig = configs.to_numpy(s.eps_r), configs.to_numpy(s.sigma)
    o = O.OracleSim(s.nx, s.ny, s.dx, s.dy, s.dt, eps, sig)
    ninst = 0
    if s.placements is not None:
        for k, i0, j0 in s.placements:
            o.add_rom(s.models[k], int(i0), int(j0))
            ninst += 1
    o.set_source(*s.source, s.samples)
    o.set_probes(s.probes)
    o.step(1)
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        o.step(1)
        done += 1
        if max_seconds and time.perf_counter() - t0 > max_seconds:
            break
    dt = time.perf_counter() - t0
    sample = "%s sub-instance %dx%d with %d ROM instances, %d steps (fp64 oracle, %d host threads)" % (
        workload, s.nx, s.ny, ninst, done, nthreads)
    return s.nx * s.ny * done / dt, dt, done, sample, nthreads


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = args.workload
    # warm-up steps, then the timed steps of the bounded sample: at least K and at least ~10 s of
    # stepping (a 20-step run would time mostly start-up), at most 240 s
    oracle_rate(wl, max(args.warmup, 0), max_seconds=60)
    v0, dt0, done0, _, _ = oracle_rate(wl, max(args.steps, 8), max_seconds=30)
    want = max(args.steps, int(10.0 * done0 / max(dt0, 1e-9)))
    v, dt, done, sample, cores = oracle_rate(wl, want, max_seconds=240)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": done,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl + " (bounded CPU sample)", "description": WORKLOADS.get(wl, wl),
                       "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip().lower() == "active"})
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].strip() not in ("", "[N/A]"))}


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from inputs import configs
    from paper_1609_07114_b200 import Simulation, nccl_unique_id, slabs

    ws, rank, lrank = dist_env()
    if torch.cuda.device_count() < max(ws, lrank + 1):
        sys.exit("bench.py: rank %d needs CUDA device %d, %d visible" % (rank, lrank, torch.cuda.device_count()))
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    if ws > 1:
        # NCCL init lines (one per rank: "nranks N") go to stderr, keeping stdout to the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    t_setup = time.perf_counter()
    scene = configs.make(wl, device="cuda")
    ny = scene.ny
    rb, re = slabs.slab_rows(ny, ws, rank)
    nid = None
    if ws > 1:
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone().to(dev)
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().numpy().tobytes())
    m0, m1 = max(rb - 4, 0), min(re + 4, ny)  # materials of rows [rb-4, re+4): the 4-step halo
    eps = scene.eps_r[m0:m1].contiguous()
    sig = scene.sigma[m0:m1].contiguous()
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, eps, sig, precision=scene.precision,
                     device=lrank, rank=rank, nranks=ws, nccl_id=nid, row_begin=rb, row_end=re,
                     materials_row0=m0, record_capacity=max(4096, args.steps + args.warmup + 8))
    del eps, sig
    ninst = 0
    if scene.placements is not None:
        # fdtd_add_rom is collective with several ranks: every rank adds every model (count 0
        # where it owns none of its instances)
        P = slabs.owned_placements(scene.placements, scene.models, rb, re)
        for k, m in enumerate(scene.models):
            sel = P[P[:, 0] == k]
            sim.add_rom(m, sel[:, 1:3])
            ninst += len(sel)
    sim.set_source(*scene.source, scene.samples)
    sim.set_probes(scene.probes)
    sim.record_energy(not args.no_energy)
    if args.init == "random":  # every live cell and edge populated (the source pulse leaves most zero)
        sim.set_random_fields(20261020, 1.0)
    scene.eps_r = scene.sigma = None
    torch.cuda.empty_cache()
    setup_s = time.perf_counter() - t_setup
    cells_rank = scene.nx * (re - rb)
    cells_total = scene.nx * scene.ny
    stream = sim.stream

    def barrier():
        if ws > 1:
            dist.barrier()

    # ---- warm-up
    sim.step(args.warmup)
    sim.sync()
    sim.probe()
    sim.energy()
    # ---- timed region: K steps, per-kernel events (sweep / post) on the launching stream
    clk = Clocks(lrank)
    clk.start()
    l0 = sim.info().kernel_launches
    barrier()
    torch.cuda.synchronize()
    sim.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    sweep_ms, post_ms, nl = sim.profile_read()
    sim.profile(False)
    clocks = clk.stop()
    launches = sim.info().kernel_launches - l0
    ms_all = ms
    if ws > 1:
        t = torch.tensor([ms, sweep_ms, post_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_all, sweep_ms_max, post_ms_max = t.tolist()
    value = cells_total * args.steps / (ms_all / 1e3)
    pr = sim.probe()
    en = sim.energy()
    finite = bool(np.all(np.isfinite(pr)) and np.all(np.isfinite(en)))

    # ---- end-to-end through the public API with host buffers: every call advances E2E_CHUNK steps
    #      and copies exactly those steps' inputs in (source samples, host -> device) and their
    #      results out (probe samples + energy, device -> host); chunk = two K-step passes
    e2e = None
    if not args.no_e2e:
        samples = np.ascontiguousarray(scene.samples, dtype=np.float64)
        chunk = 2 * sim.info().steps_per_pass
        k_e2e = max(chunk, min(args.steps, args.e2e_steps) // chunk * chunk)
        start = sim.info().steps_taken
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(0, k_e2e, chunk):
            n = start + k
            sim.set_source(*scene.source, samples[n:n + chunk], step0=n)
            sim.step(chunk)
            p = sim.probe()
            e = sim.energy()
        torch.cuda.synchronize()
        barrier()
        dt_e2e = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt_e2e = t.item()
        es = 8 if scene.precision == 64 else 4
        e2e = {"value": cells_total * k_e2e / dt_e2e, "unit": UNIT, "h2d_bytes_per_step": 8,
               "d2h_bytes_per_step": len(scene.probes) * es + (0 if args.no_energy else 8),
               "steps": k_e2e, "steps_per_call": chunk,
               "api": "per call: fdtd_set_source(host samples) + fdtd_step(%d) + fdtd_probe + fdtd_energy (host)"
                      % chunk}
        finite = finite and bool(np.all(np.isfinite(p)))
    if rank != 0:
        sim.close()
        if ws > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (the fused sweep), rank 0's slab
    pk = peaks()
    es = 8 if scene.precision == 64 else 4
    info = sim.info()
    spp = info.steps_per_pass              # time steps advanced by one sweep pass (1, 2 or 4)
    sweep_avg_s = (sweep_ms / max(nl, 1)) / 1e3
    peak = pk.get("hbm_gbs", 6650.0)
    # Bytes one launch must move as implemented: Ex, Ey, Hz and the two per-cell material terms read
    # once, Ex, Ey, Hz written once per K-step pass (8 arrays x es per cell).  The DRAM traffic
    # ncu measured on this build (profiles/sweep_traffic.json, valid only while the kernel sources'
    # hash matches) replaces it when present: `frac` is then the fraction of the measured copy
    # bandwidth the kernel's actual DRAM traffic reaches.
    compulsory = 8 * es * cells_rank
    traffic, tsrc = None, None
    tpath = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if (tj.get("workload") == wl and int(tj.get("steps_per_pass", 1)) == spp and ws == 1
                    and tj.get("kernel_src_sha") == kernel_source_sha()):
                traffic = tj.get("bytes_per_launch_per_cell") * cells_rank
                tsrc = tj.get("source")
        except Exception:
            traffic = None
    moved = traffic if traffic else compulsory
    achieved = moved / sweep_avg_s / 1e9
    # SURVEY 8(d)'s algorithmic count (40 B per cell-step fp32 -- Ex, Ey, Hz read and written plus
    # the per-edge (ca, cb) pairs -- times the cell-steps of one launch): with K steps per HBM pass
    # this is an *effective* bandwidth, above the roof by up to K x 40/32
    alg_bytes = 10 * es * cells_rank * spp
    kname = "sweepk_kernel<%s, K=%d> (fused H+E, %d time step%s per HBM pass)" % (
        "float" if es == 4 else "double", spp, spp, "s" if spp > 1 else "")
    roof = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "bytes_per_launch": moved,
            "bytes_source": ("ncu dram__bytes_read.sum + dram__bytes_write.sum of this build (%s)" % tsrc) if traffic
            else "compulsory bytes as implemented (8 arrays x %d B per cell per pass; no ncu capture of this build)"
            % es,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in pk else "fallback",
            "kernel_src_sha": kernel_source_sha(),
            "algorithmic_bytes_per_launch": alg_bytes, "steps_per_launch": spp,
            "achieved_algorithmic_gbs": alg_bytes / sweep_avg_s / 1e9,
            "frac_algorithmic": alg_bytes / sweep_avg_s / 1e9 / peak,
            "implemented_bytes_per_cell_step": info.bytes_per_cell_step,
            "sweep_ms_per_launch": sweep_avg_s * 1e3,
            "post_ms_per_launch": post_ms / max(nl, 1), "sweep_share_of_step": sweep_ms / max(ms, 1e-9)}
    cpu = None
    if ws == 1 and not args.no_cpu:
        v, dt, done, sample, cores = oracle_rate(wl, 10 ** 6, max_seconds=args.cpu_seconds)
        v1, _, done1, sample1, _ = oracle_rate(wl, 10 ** 6, max_seconds=args.cpu_seconds / 3, threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "single_thread": {"value": v1, "cores": 1, "sample": sample1}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_all / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if scene.precision == 32 else "f64",
            "data": "synthetic",
            "config": {"workload": wl, "description": WORKLOADS.get(wl, wl), "nx": scene.nx, "ny": scene.ny,
                       "rom_instances": int(len(scene.placements)) if scene.placements is not None else 0,
                       "rom_instances_rank0": ninst, "steps_in_config": scene.steps,
                       "parallelism": "row-slab x%d" % ws, "l2": "inputs larger than L2 (%.1f GB/step)" %
                       (10 * es * cells_total / 1e9), "energy_recorded": not args.no_energy,
                       "init": "seeded random fields on every live cell and edge" if args.init == "random" else
                       "zero fields + the Gaussian source pulse (the config's own workload)",
                       "n_clipped": scene.meta.get("n_clipped"), "setup_s": setup_s, "finite": finite},
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks, "e2e": e2e, "gpu_launches": launches}
    print(json.dumps(line), flush=True)
    sim.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-energy", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--init", default="zero", choices=["zero", "random"],
                    help="initial fields: the config's (zero + source pulse) or seeded random live fields")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    ensure_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
