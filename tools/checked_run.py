"""Checked-build runs (the stand-in for compute-sanitizer, which is closed on the GPU pool).

    python tools/checked_run.py [--out gpurun_out/checked.json]

Loads paper_1609_07114_b200/libfdtdrom_check.so (built with -DFDTD_CHECK=1: every global access of
the sweep, the fix-up region loads / write-backs / scatters, the zone probes, the CPML band kernel's
loads and stores trap on a bounds violation, and write-backs must stay in the owned rows), then runs
small hot-path cases with cudaMalloc'd buffers (no caching allocator), K = 1, 2, 4:
  * parity with the fp64 oracle (fp64 1e-10 / fp32 1e-4);
  * the whole-grid path (cfg1whole, densewhole: K3c, one launch per call) the same way;
  * determinism: the same run twice, and with the fix-up at 128 / 256 / 512 threads per CTA, must be
    bit-identical -- a shared-memory race or a missing barrier would show as a difference
    (the racecheck / synccheck stand-in).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_1609_07114_b200", "libfdtdrom_check.so")


def run_case(case, k, threads, steps):
    """One case in a fresh process (FDTD_POST_THREADS is read at context creation)."""
    env = dict(os.environ, FDTD_LIB=CHECK_LIB, FDTD_POST_THREADS=str(threads))
    code = r'''
import sys, json, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
from helpers import consistent_random_state, gpu_from_scene, oracle_from_scene, rel
from inputs import configs
case, k, steps = %r, %d, %d
if case == "cfg1":
    s = configs.make("cfg1")
elif case in ("cfg3crop", "cfg3crop4row"):
    s = configs.make("cfg3", n=256)
elif case == "cfg5sub":
    s = configs.make("cfg5", n=512, max_fine=64, min_count=8)
elif case == "cfg1whole":
    s = configs.make("cfg1")
elif case == "densewhole":
    from test_gpu_wholegrid import _dense_fp32
    s = _dense_fp32()
elif case == "literal":
    from test_gpu_parity import _literal_scene
    s = _literal_scene(32, n=128)
else:
    from test_gpu_pml import channel_scene
    s = channel_scene(32, nx=120, ny=40, rom=True)
g = gpu_from_scene(s, torch_allocator=False, whole_grid=case.endswith("whole"))
g.set_time_blocking(k)
if case == "cfg3crop4row":
    g.set_tuning(256, 4)  # one 256-row chunk: the four-row sweep body
Ex, Ey, Hz, xs = consistent_random_state(s, 3)
g.set_window(0, 0, Ex, Ey, Hz)
if xs.size:
    g.set_rom_state(xs)
g.record_energy(True)
g.step(steps)
p, e = g.probe(), g.energy()
W = g.get_window()
x = g.get_rom_state()
o = oracle_from_scene(s)
o.set_state(Ex, Ey, Hz, xs if xs.size else None)
po, eo = o.step(steps)
Wo = o.get_state()
err = max(rel(p, po), rel(e, eo), *[rel(a, b) for a, b in zip(W, Wo[:3])], rel(x, Wo[3]) if x.size else 0.0)
import hashlib
h = hashlib.sha256()
for a in (*W, x, p):
    h.update(np.ascontiguousarray(a).tobytes())
print("RESULT " + json.dumps(dict(case=case, k=k, used=g.info().steps_per_pass, err=err, prec=s.precision,
                                  whole_grid=int(g.info().whole_grid),
                                  digest=h.hexdigest()[:16])))
''' % (ROOT, os.path.join(ROOT, "tests"), case, k, steps)
    try:
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    except subprocess.TimeoutExpired as e:
        return {"case": case, "k": k, "rc": -9, "threads": threads, "trap": False,
                "tail": "timeout: " + ((e.stdout or b"")[-300:].decode(errors="replace") if isinstance(e.stdout, bytes)
                                       else str(e.stdout)[-300:])}
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    out = json.loads(line[-1][7:]) if line else {"case": case, "k": k}
    out.update(rc=r.returncode, threads=threads, trap="FDTD_CHECK" in (r.stdout + r.stderr),
               tail=(r.stdout + r.stderr)[-600:] if r.returncode else "")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "checked.json"))
    ap.add_argument("--steps", type=int, default=64)
    a = ap.parse_args()
    if not os.path.exists(CHECK_LIB):
        sys.path.insert(0, ROOT)
        from paper_1609_07114_b200 import build
        build.build_checked()
    cases = [("cfg1", 1), ("cfg1", 2), ("cfg3crop", 1), ("cfg3crop", 2), ("cfg3crop", 4), ("cfg3crop4row", 4), ("pml", 4),
             ("literal", 4), ("cfg5sub", 4), ("cfg1whole", 2), ("densewhole", 4)]
    res = []
    ok = True
    for case, k in cases:
        runs = [run_case(case, k, t, a.steps) for t in (256, 256, 128, 512)]
        digests = {r.get("digest") for r in runs}
        tol = 1e-10 if runs[0].get("prec") == 64 else 1e-4
        good = all(r["rc"] == 0 and not r["trap"] and r.get("err", 1) <= tol for r in runs) and len(digests) == 1
        ok &= good
        res.append(dict(case=case, k=k, ok=good, runs=runs, bitwise_identical_across_runs_and_threads=len(digests) == 1))
        print("%-12s K=%d used=%s err=%s traps=%s identical=%s -> %s" % (
            case, k, runs[0].get("used"), max(r.get("err", float("nan")) for r in runs),
            any(r["trap"] for r in runs), len(digests) == 1, "ok" if good else "FAIL"), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(dict(lib="libfdtdrom_check.so (-DFDTD_CHECK=1)", steps=a.steps, ok=ok, cases=res), open(a.out, "w"),
              indent=1)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
