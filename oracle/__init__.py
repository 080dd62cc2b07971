"""Oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 CPU implementation of the hot path of arXiv 1609.07114
("A Stable FDTD Method with Embedded Reduced-Order Models"), written from the
paper (see ``fdtd_oracle.c`` for the per-function citations).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The CUDA product path
(``paper_1609_07114_b200``) never imports it and shares no code with it.

Parity status of each oracle function ("Oracle pins"):
  * coarse H/E half-steps      -- pinned (PEC-cavity spectrum, CFL threshold, hand values)
  * soft source, probes        -- pinned (superposition / hand values)
  * coupled ROM step (LU)      -- pinned (r=1 == uniform Yee; full order == direct subgridding)
  * direct subgridding         -- pinned (r=1 == uniform Yee)
  * storage function W^n       -- pinned (exact conservation when lossless, monotone when lossy)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fdtd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(force: bool = False) -> str:
    """Compile the plain-C oracle (gcc, -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.osim_create.restype = C.c_void_p
        L.osim_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.osim_destroy.argtypes = [C.c_void_p]
        L.osim_add_rom.restype = C.c_int
        L.osim_add_rom.argtypes = [C.c_void_p] + [C.c_int] * 6 + [_dp] * 5 + [C.c_int, C.c_int]
        L.osim_add_subgrid.restype = C.c_int
        L.osim_add_subgrid.argtypes = [C.c_void_p] + [C.c_int] * 5 + [_dp, _dp]
        L.osim_set_source.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int64, C.c_int64]
        L.osim_set_source_line.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, C.c_int64, C.c_int64]
        L.osim_set_pml.restype = C.c_int
        L.osim_set_pml.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double]
        for n in ("osim_get_psi", "osim_set_psi"):
            getattr(L, n).restype = C.c_int
            getattr(L, n).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.osim_set_probes.argtypes = [C.c_void_p, _ip, C.c_int]
        L.osim_step.argtypes = [C.c_void_p, C.c_int64, _dp, C.c_int64, _dp]
        L.osim_get_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.osim_set_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.osim_set_threads.argtypes = [C.c_int]
        L.osim_get_threads.restype = C.c_int
        L.osim_steps_taken.restype = C.c_int64
        L.osim_steps_taken.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n):
    """Host threads for the oracle's row loops (0: all cores).  Results do not depend on it."""
    lib().osim_set_threads(int(n))


def get_threads():
    return lib().osim_get_threads()


class OracleSim:
    """fp64 CPU reference simulation (coarse TEz Yee grid + embedded ROMs)."""

    def __init__(self, nx, ny, dx, dy, dt, eps_r, sigma):
        self.nx, self.ny, self.dx, self.dy, self.dt = int(nx), int(ny), float(dx), float(dy), float(dt)
        self._eps = _f64(np.broadcast_to(eps_r, (ny, nx)))
        self._sig = _f64(np.broadcast_to(sigma, (ny, nx)))
        self._h = lib().osim_create(self.nx, self.ny, self.dx, self.dy, self.dt, _p(self._eps), _p(self._sig))
        if not self._h:
            raise ValueError("osim_create rejected its arguments")
        self.rom_q = []
        self.nprobe = 0

    def close(self):
        if self._h:
            lib().osim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add_rom(self, model, i0, j0):
        """Embed one instance of a reduced model (dict with R11,R22,F11,K,L,bx,by[,r,literal]).

        literal models couple through the r nY fine hanging variables of the paper's eq:sysform
        (T, 1/r; L is q1 x r nY); the default is the collapsed reading (R9)."""
        R11, R22, F11, K, L = (_f64(model[k]) for k in ("R11", "R22", "F11", "K", "L"))
        q1, q2 = R11.shape[0], R22.shape[0]
        literal = bool(model.get("literal", False))
        rc = lib().osim_add_rom(self._h, int(i0), int(j0), int(model["bx"]), int(model["by"]), q1, q2,
                                _p(R11), _p(R22), _p(F11), _p(K), _p(L), int(model.get("r", 1)),
                                1 if literal else 0)
        if rc < 0:
            raise ValueError("osim_add_rom failed with code %d" % rc)
        self.rom_q.append(q1 + q2)
        return rc

    def add_subgrid(self, i0, j0, bx, by, r, fine_eps_r, fine_sigma):
        fe, fs = _f64(fine_eps_r), _f64(fine_sigma)
        assert fe.shape == (by * r, bx * r) and fs.shape == fe.shape
        rc = lib().osim_add_subgrid(self._h, int(i0), int(j0), int(bx), int(by), int(r), _p(fe), _p(fs))
        if rc < 0:
            raise ValueError("osim_add_subgrid failed with code %d" % rc)
        return rc

    def set_source(self, i, j, samples, t0=0):
        self._src = _f64(samples)
        lib().osim_set_source(self._h, int(i), int(j), _p(self._src), len(self._src), int(t0))

    def set_source_line(self, i, j0, j1, samples, t0=0):
        """Soft Hz source on the cells (i, j0 .. j1-1) (a line source, NEXT-2)."""
        a = _f64(samples)
        lib().osim_set_source_line(self._h, int(i), int(j0), int(j1), _p(a), a.size, int(t0))

    def set_pml(self, width, order=3, r0=1e-8):
        """CPML of `width` cells on both x-ends (NEXT-2)."""
        rc = lib().osim_set_pml(self._h, int(width), int(order), float(r0))
        if rc != 0:
            raise ValueError("osim_set_pml failed with code %d" % rc)

    def get_psi(self):
        """CPML auxiliary state (psi_hz [ny, nx], psi_ey [ny, nx + 1]); state only."""
        ph, pe = np.zeros((self.ny, self.nx)), np.zeros((self.ny, self.nx + 1))
        if lib().osim_get_psi(self._h, _p(ph), _p(pe)) != 0:
            raise ValueError("no CPML layers")
        return ph, pe

    def set_psi(self, psi_hz, psi_ey):
        ph, pe = _f64(psi_hz), _f64(psi_ey)
        assert ph.size == self.ny * self.nx and pe.size == self.ny * (self.nx + 1)
        if lib().osim_set_psi(self._h, _p(ph), _p(pe)) != 0:
            raise ValueError("no CPML layers")

    def set_probes(self, ij):
        a = np.ascontiguousarray(np.asarray(ij, dtype=np.int32).reshape(-1, 2))
        lib().osim_set_probes(self._h, a.ctypes.data_as(_ip), a.shape[0])
        self.nprobe = a.shape[0]

    def step(self, n, probes=True, energy=True):
        """Advance n steps; returns (probe [P, n], energy [n])."""
        pr = np.zeros((self.nprobe, n)) if probes and self.nprobe else None
        en = np.zeros(n) if energy else None
        lib().osim_step(self._h, int(n), _p(pr), int(n), _p(en))
        return pr, en

    def get_state(self):
        Ex = np.zeros((self.ny + 1, self.nx))
        Ey = np.zeros((self.ny, self.nx + 1))
        Hz = np.zeros((self.ny, self.nx))
        rs = np.zeros(max(1, sum(self.rom_q)))
        lib().osim_get_state(self._h, _p(Ex), _p(Ey), _p(Hz), _p(rs))
        return Ex, Ey, Hz, rs[: sum(self.rom_q)]

    def set_state(self, Ex=None, Ey=None, Hz=None, rom_state=None):
        args = []
        for a, shp in ((Ex, (self.ny + 1, self.nx)), (Ey, (self.ny, self.nx + 1)), (Hz, (self.ny, self.nx))):
            if a is None:
                args.append(None)
            else:
                a = _f64(a)
                assert a.shape == shp, (a.shape, shp)
                args.append(a)
        rs = None if rom_state is None else _f64(rom_state)
        self._keep = args + [rs]
        lib().osim_set_state(self._h, _p(args[0]), _p(args[1]), _p(args[2]), _p(rs))

    @property
    def steps_taken(self):
        return lib().osim_steps_taken(self._h)

    # ---- helpers for tests -------------------------------------------------
    def state_vector(self):
        Ex, Ey, Hz, rs = self.get_state()
        return np.concatenate([Ex.ravel(), Ey.ravel(), Hz.ravel(), rs])

    def set_state_vector(self, v):
        nx, ny = self.nx, self.ny
        a = nx * (ny + 1)
        b = a + (nx + 1) * ny
        c = b + nx * ny
        self.set_state(v[:a].reshape(ny + 1, nx), v[a:b].reshape(ny, nx + 1), v[b:c].reshape(ny, nx),
                       v[c:] if sum(self.rom_q) else None)


C0 = 299792458.0
MU0 = 4e-7 * np.pi
EPS0 = 1.0 / (MU0 * C0 * C0)
