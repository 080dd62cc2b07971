"""Thin ctypes binding of include/fdtdrom.h (argument marshalling only).

Every step of the hot path runs in libfdtdrom.so's CUDA kernels.  There is no CPU
fallback: if the library or a CUDA device is missing, the calls raise.
PyTorch is used for device memory (the caching allocator backs the library's
allocations), streams, and the process group that broadcasts the NCCL id.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FDTD_LIB: an alternative in-tree build of the same library (kernel tuning experiments)
LIB_PATH = os.environ.get("FDTD_LIB") or os.path.join(_HERE, "libfdtdrom.so")

FDTD_MATERIALS_ON_DEVICE = 0x1
FDTD_MATERIALS_F32 = 0x2
FDTD_ALLOW_DT_ABOVE_EQ1 = 0x4
FDTD_NO_GRAPH = 0x8
FDTD_LOCAL_GROUP = 0x10
FDTD_NO_WHOLE = 0x20

STATUS = {0: "FDTD_OK", 1: "FDTD_E_ARG", 2: "FDTD_E_STATE", 3: "FDTD_E_PASSIVITY", 4: "FDTD_E_UNSTABLE",
          5: "FDTD_E_CUDA", 6: "FDTD_E_NCCL", 7: "FDTD_E_NOMEM"}

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class GridDesc(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("dx", C.c_double), ("dy", C.c_double),
                ("dt", C.c_double), ("precision", C.c_int32), ("flags", C.c_uint32),
                ("eps_r", C.c_void_p), ("sigma", C.c_void_p), ("materials_row0", C.c_int64),
                ("device", C.c_int32), ("stream", C.c_void_p), ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_user", C.c_void_p), ("nranks", C.c_int32), ("rank", C.c_int32),
                ("nccl_id", C.c_void_p), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("record_capacity", C.c_int64)]


class RomModel(C.Structure):
    _fields_ = [("bx", C.c_int32), ("by", C.c_int32), ("r", C.c_int32), ("q1", C.c_int32), ("q2", C.c_int32),
                ("R11", C.c_void_p), ("R22", C.c_void_p), ("F11", C.c_void_p), ("K", C.c_void_p),
                ("L", C.c_void_p), ("literal", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("steps_taken", C.c_int64), ("n_instances", C.c_int64), ("kernel_launches", C.c_int64),
                ("pitch", C.c_int64), ("sweep_ctas", C.c_int64), ("graphs", C.c_int32),
                ("precision", C.c_int32), ("bytes_per_cell_step", C.c_double), ("steps_per_pass", C.c_int32),
                ("sweep_stream", C.c_void_p), ("graph_builds", C.c_int64), ("fixup_clusters", C.c_int32),
                ("big_instances", C.c_int32), ("whole_grid", C.c_int32)]


class RomSpec(C.Structure):  # fdtdrom_build.h
    _fields_ = [("bx", C.c_int32), ("by", C.c_int32), ("r", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
                ("eps_r", C.c_void_p), ("sigma", C.c_void_p), ("q", C.c_int32), ("fmax", C.c_double),
                ("dt_target", C.c_double), ("cg_tol", C.c_double), ("literal", C.c_int32)]


class RomBuilt(C.Structure):
    _fields_ = [("R11", C.c_void_p), ("R22", C.c_void_p), ("F11", C.c_void_p), ("K", C.c_void_p),
                ("L", C.c_void_p), ("q1", C.c_int32), ("q2", C.c_int32), ("nY", C.c_int32),
                ("n_clipped", C.c_int32), ("natural_dt_limit", C.c_double), ("krylov_vectors", C.c_int32),
                ("cg_iterations_max", C.c_int32), ("jacobi_sweeps_max", C.c_int32), ("ms_total", C.c_double),
                ("ms_solve", C.c_double), ("ms_orth", C.c_double), ("ms_svd", C.c_double)]


class FDTDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


_lib = None


def lib():
    """Load libfdtdrom.so (built in-tree by build.py); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libfdtdrom.so not built: run `python -m paper_1609_07114_b200.build` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_double)
        L.fdtd_create.argtypes = [C.POINTER(GridDesc), C.POINTER(vp)]
        L.fdtd_add_rom.argtypes = [vp, C.POINTER(RomModel), vp, i64, C.POINTER(i32)]
        L.fdtd_set_source.argtypes = [vp, i64, i64, vp, i64, i64]
        L.fdtd_set_source_line.argtypes = [vp, i64, i64, i64, vp, i64, i64]
        L.fdtd_set_pml.argtypes = [vp, i32, i32, C.c_double]
        L.fdtd_set_probes.argtypes = [vp, vp, i32]
        L.fdtd_record_energy.argtypes = [vp, i32]
        L.fdtd_step.argtypes = [vp, i64]
        L.fdtd_step_group.argtypes = [C.POINTER(vp), i32, i64]
        L.fdtd_probe.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.fdtd_energy.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.fdtd_get_window.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp]
        L.fdtd_set_window.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp]
        L.fdtd_set_random_fields.argtypes = [vp, C.c_uint64, C.c_double]
        L.fdtd_get_rom_state.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.fdtd_set_rom_state.argtypes = [vp, vp, i64]
        L.fdtd_sync.argtypes = [vp]
        L.fdtd_get_info.argtypes = [vp, C.POINTER(Info)]
        L.fdtd_set_tuning.argtypes = [vp, i32, i32]
        L.fdtd_profile.argtypes = [vp, i32]
        L.fdtd_set_time_blocking.argtypes = [vp, i32]
        L.fdtd_profile_read.argtypes = [vp, dp, dp, C.POINTER(i64)]
        L.fdtd_nccl_unique_id.argtypes = [vp]
        L.fdtd_halo_plan.argtypes = [i32, i32, i64, i64, i32, i32, vp, i32, C.POINTER(i32)]
        L.fdtd_pass_regions.argtypes = [vp, vp, i64, i32, vp, vp, C.POINTER(i64)]
        L.fdtd_last_error.argtypes = [vp]
        L.fdtd_last_error.restype = C.c_char_p
        L.fdtd_status_string.restype = C.c_char_p
        L.fdtd_destroy.argtypes = [vp]
        L.fdtd_destroy.restype = None
        L.fdtd_rom_build.argtypes = [C.POINTER(RomSpec), C.POINTER(RomBuilt)]
        L.fdtd_rom_build.restype = C.c_int
        L.fdtd_rom_build_last_error.argtypes = []
        L.fdtd_rom_build_last_error.restype = C.c_char_p
        if hasattr(L, "fdtd_debug_phases"):  # tuning builds (FDTD_PHASES)
            L.fdtd_debug_phases.argtypes = [vp, i32]
        for n in ("create", "add_rom", "set_source", "set_probes", "record_energy", "step", "probe", "energy",
                  "get_window", "set_window", "get_rom_state", "set_rom_state", "sync", "get_info", "set_tuning",
                  "nccl_unique_id", "profile", "profile_read", "step_group", "set_time_blocking",
                  "set_source_line", "set_pml", "halo_plan", "pass_regions"):
            getattr(L, "fdtd_" + n).restype = C.c_int
        _lib = L
    return _lib


def exported_symbols():
    """Names declared in include/fdtdrom.h (used by the ABI test)."""
    import re
    names = set()
    for h in ("fdtdrom.h", "fdtdrom_build.h"):
        hdr = open(os.path.join(os.path.dirname(_HERE), "include", h)).read()
        names |= set(re.findall(r"\b(fdtd_[a-z_0-9]+)\s*\(", hdr))
    return sorted(names)


def build_rom(bx, by, r, dx, dy, eps_r, sigma, q, fmax, dt_target=None, cg_tol=0.0, literal=False):
    """GPU-side ROM construction (fdtdrom_build.h, NEXT-3): fine assembly, collapse onto coarse-edge
    ports, SPRIM(q) with CG-solved shifts, congruence, optional CFL clip at dt_target.  Returns the
    model dict fdtd_add_rom consumes (R11, R22, F11, K, L, q1, q2, bx, by, r, n_clipped, literal,
    natural_dt_limit) plus the builder's diagnostics under "gpu_build"."""
    eps = _f64(eps_r).reshape(by * r, bx * r)
    sig = _f64(sigma).reshape(by * r, bx * r)
    nY = (2 * bx + 2 * by) * (r if literal else 1)
    q1w, q2w = (q + 1) // 2 + (nY if literal else 0), q // 2
    R11, F11 = np.zeros((q1w, q1w)), np.zeros((q1w, q1w))
    R22, K, L = np.zeros((q2w, q2w)), np.zeros((q1w, q2w)), np.zeros((q1w, nY))
    spec = RomSpec(int(bx), int(by), int(r), float(dx), float(dy), eps.ctypes.data, sig.ctypes.data, int(q),
                   float(fmax), float(dt_target or 0.0), float(cg_tol), int(bool(literal)))
    out = RomBuilt(R11.ctypes.data, R22.ctypes.data, F11.ctypes.data, K.ctypes.data, L.ctypes.data)
    st = lib().fdtd_rom_build(C.byref(spec), C.byref(out))
    if st:
        raise FDTDError(st, lib().fdtd_rom_build_last_error().decode())
    q1, q2 = out.q1, out.q2
    unpack = lambda a, m, n: np.ascontiguousarray(a.ravel()[: m * n].reshape(m, n))
    return dict(bx=int(bx), by=int(by), r=int(r), q1=q1, q2=q2, R11=unpack(R11, q1, q1), R22=unpack(R22, q2, q2),
                F11=unpack(F11, q1, q1), K=unpack(K, q1, q2), L=unpack(L, q1, nY), n_clipped=int(out.n_clipped),
                literal=bool(literal), natural_dt_limit=float(out.natural_dt_limit),
                gpu_build=dict(krylov_vectors=out.krylov_vectors, cg_iterations_max=out.cg_iterations_max,
                               jacobi_sweeps_max=out.jacobi_sweeps_max, ms_total=out.ms_total,
                               ms_solve=out.ms_solve, ms_orth=out.ms_orth, ms_svd=out.ms_svd))


def halo_plan(nranks, rank, row_begin, row_end, depth, pml=False):
    """fdtd_halo_plan: the rows exchanged before a `depth`-step pass, as an int64 array of
    (direction 0 send / 1 receive, array, global row, peer) rows, sends first (host only)."""
    n = C.c_int32(0)
    lib().fdtd_halo_plan(int(nranks), int(rank), int(row_begin), int(row_end), int(depth), int(bool(pml)), None, 0,
                         C.byref(n))
    out = np.zeros((max(n.value, 1), 4), dtype=np.int64)
    st = lib().fdtd_halo_plan(int(nranks), int(rank), int(row_begin), int(row_end), int(depth), int(bool(pml)),
                              _ptr(out), n.value, C.byref(n))
    if st:
        raise FDTDError(st, "fdtd_halo_plan rejected its arguments")
    return out[: n.value]


def pass_regions(rects, models, depth):
    """fdtd_pass_regions: (region index per instance, boxes [n_regions, 5] = i0, j0, w, h, mixed)."""
    r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
    m = np.ascontiguousarray(np.asarray(models, dtype=np.int32).reshape(-1))
    n = r.shape[0]
    reg = np.zeros(max(n, 1), np.int32)
    boxes = np.zeros((max(n, 1), 5), np.int32)
    nr = C.c_int64(0)
    st = lib().fdtd_pass_regions(_ptr(r), _ptr(m), n, int(depth), _ptr(reg), _ptr(boxes), C.byref(nr))
    if st:
        raise FDTDError(st, "fdtd_pass_regions rejected its arguments")
    return reg[:n], boxes[: nr.value]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().fdtd_nccl_unique_id(buf)
    if st:
        raise FDTDError(st, "ncclGetUniqueId failed")
    return buf.raw


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Simulation:
    """One coarse TEz grid (or row slab of it) with embedded ROMs, advanced on a CUDA device."""

    def __init__(self, nx, ny, dx, dy, dt, eps_r, sigma, precision=32, device=0, stream=None, rank=0,
                 nranks=1, nccl_id=None, row_begin=0, row_end=None, materials_row0=0, record_capacity=0,
                 allow_unstable=False, use_graphs=True, torch_allocator=True, local_group=False, whole_grid=True):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1609_07114_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        self.device = int(device)
        self.nx, self.ny, self.dx, self.dy, self.dt = int(nx), int(ny), float(dx), float(dy), float(dt)
        self.precision = int(precision)
        self.row_begin = int(row_begin)
        self.row_end = int(ny if row_end is None else row_end)
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        flags = 0
        if isinstance(eps_r, torch.Tensor):
            assert eps_r.is_cuda and sigma.is_cuda and eps_r.dtype == sigma.dtype
            # fdtd_create copies them on self.stream: order it after their producer (the current stream)
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            self._mat = (eps_r.contiguous(), sigma.contiguous())
            flags |= FDTD_MATERIALS_ON_DEVICE
            if eps_r.dtype == torch.float32:
                flags |= FDTD_MATERIALS_F32
            else:
                assert eps_r.dtype == torch.float64
            pe, ps = self._mat[0].data_ptr(), self._mat[1].data_ptr()
        else:
            self._mat = (_f64(eps_r), _f64(sigma))
            pe, ps = self._mat[0].ctypes.data, self._mat[1].ctypes.data
        if allow_unstable:
            flags |= FDTD_ALLOW_DT_ABOVE_EQ1
        if not use_graphs:
            flags |= FDTD_NO_GRAPH
        if local_group:
            flags |= FDTD_LOCAL_GROUP
        if not whole_grid:
            flags |= FDTD_NO_WHOLE
        d = GridDesc()
        d.nx, d.ny, d.dx, d.dy, d.dt = self.nx, self.ny, self.dx, self.dy, self.dt
        d.precision, d.flags = self.precision, flags
        d.eps_r, d.sigma, d.materials_row0 = pe, ps, int(materials_row0)
        d.device, d.stream = self.device, self.stream.cuda_stream
        if torch_allocator:
            dev, st = self.device, self.stream

            def _alloc(n, _u):
                return torch.cuda.caching_allocator_alloc(int(n), dev, st)

            def _free(p, _u):
                torch.cuda.caching_allocator_delete(p)

            self._cb = (ALLOC_FN(_alloc), FREE_FN(_free))
            d.alloc, d.free = self._cb
        d.nranks, d.rank = int(nranks), int(rank)
        self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        d.nccl_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None
        d.row_begin, d.row_end = self.row_begin, self.row_end
        d.record_capacity = int(record_capacity)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = lib().fdtd_create(C.byref(d), C.byref(h))
        if st:
            raise FDTDError(st, "fdtd_create failed")
        self._h = h
        self._mat = None  # copied by fdtd_create
        self.n_probe = 0
        self.rom_state_len = 0

    # ---------------------------------------------------------------- plumbing
    def _ck(self, st, what):
        if st:
            raise FDTDError(st, "%s: %s" % (what, lib().fdtd_last_error(self._h).decode()))

    def close(self):
        if getattr(self, "_h", None):
            with self._torch.cuda.device(self.device):
                lib().fdtd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------------- API
    def add_rom(self, model, anchors):
        R11, R22, F11, K, L = (_f64(model[k]) for k in ("R11", "R22", "F11", "K", "L"))
        m = RomModel(int(model["bx"]), int(model["by"]), int(model.get("r", 1)), R11.shape[0], R22.shape[0],
                     R11.ctypes.data, R22.ctypes.data, F11.ctypes.data, K.ctypes.data, L.ctypes.data,
                     1 if model.get("literal", False) else 0)
        a = np.ascontiguousarray(np.asarray(anchors, dtype=np.int32).reshape(-1, 2))
        mid = C.c_int32(-1)
        self._ck(lib().fdtd_add_rom(self._h, C.byref(m), _ptr(a), a.shape[0], C.byref(mid)), "fdtd_add_rom")
        self.rom_state_len += a.shape[0] * (R11.shape[0] + R22.shape[0])
        return mid.value

    def set_source(self, i, j, samples, step0=0):
        s = _f64(samples)
        self._ck(lib().fdtd_set_source(self._h, int(i), int(j), _ptr(s), s.size, int(step0)), "fdtd_set_source")

    def set_source_line(self, i, j0, j1, samples, step0=0):
        s = _f64(samples)
        self._ck(lib().fdtd_set_source_line(self._h, int(i), int(j0), int(j1), _ptr(s), s.size, int(step0)),
                 "fdtd_set_source_line")

    def set_pml(self, width, order=3, r0=1e-8):
        self._ck(lib().fdtd_set_pml(self._h, int(width), int(order), float(r0)), "fdtd_set_pml")

    def set_probes(self, ij):
        a = np.ascontiguousarray(np.asarray(ij, dtype=np.int64).reshape(-1, 2))
        self._ck(lib().fdtd_set_probes(self._h, _ptr(a), a.shape[0]), "fdtd_set_probes")
        self.n_probe = a.shape[0]

    def record_energy(self, on=True):
        self._ck(lib().fdtd_record_energy(self._h, 1 if on else 0), "fdtd_record_energy")

    def step(self, n=1):
        self._ck(lib().fdtd_step(self._h, int(n)), "fdtd_step")

    def probe(self, cap=None):
        cap = int(cap or self.info().steps_taken + 1)
        out = np.zeros((max(self.n_probe, 1), cap))
        n = C.c_int64(0)
        self._ck(lib().fdtd_probe(self._h, _ptr(out), cap, C.byref(n)), "fdtd_probe")
        return out[: self.n_probe, : n.value]

    def energy(self, cap=None):
        cap = int(cap or self.info().steps_taken + 1)
        out = np.zeros(cap)
        n = C.c_int64(0)
        self._ck(lib().fdtd_energy(self._h, _ptr(out), cap, C.byref(n)), "fdtd_energy")
        return out[: n.value]

    def get_window(self, i0=0, j0=0, w=None, h=None):
        w = self.nx - i0 if w is None else int(w)
        h = self.ny - j0 if h is None else int(h)
        Ex, Ey, Hz = np.zeros((h + 1, w)), np.zeros((h, w + 1)), np.zeros((h, w))
        self._ck(lib().fdtd_get_window(self._h, int(i0), int(j0), w, h, _ptr(Ex), _ptr(Ey), _ptr(Hz)),
                 "fdtd_get_window")
        return Ex, Ey, Hz

    def set_window(self, i0=0, j0=0, Ex=None, Ey=None, Hz=None, w=None, h=None):
        if Hz is not None:
            h, w = Hz.shape
        elif Ex is not None:
            h, w = Ex.shape[0] - 1, Ex.shape[1]
        elif Ey is not None:
            h, w = Ey.shape[0], Ey.shape[1] - 1
        arrs = [None if a is None else _f64(a) for a in (Ex, Ey, Hz)]
        self._ck(lib().fdtd_set_window(self._h, int(i0), int(j0), int(w), int(h), *[_ptr(a) for a in arrs]),
                 "fdtd_set_window")

    def set_random_fields(self, seed, amplitude=1.0):
        """Seeded random live fields on the device (fdtd_set_random_fields)."""
        self._ck(lib().fdtd_set_random_fields(self._h, C.c_uint64(int(seed)), C.c_double(float(amplitude))),
                 "fdtd_set_random_fields")

    def get_rom_state(self):
        out = np.zeros(max(self.rom_state_len, 1))
        n = C.c_int64(0)
        self._ck(lib().fdtd_get_rom_state(self._h, _ptr(out), out.size, C.byref(n)), "fdtd_get_rom_state")
        return out[: n.value]

    def set_rom_state(self, x):
        x = _f64(x)
        self._ck(lib().fdtd_set_rom_state(self._h, _ptr(x), x.size), "fdtd_set_rom_state")

    def sync(self):
        self._ck(lib().fdtd_sync(self._h), "fdtd_sync")

    def info(self):
        o = Info()
        self._ck(lib().fdtd_get_info(self._h, C.byref(o)), "fdtd_get_info")
        return o

    def set_time_blocking(self, steps_per_pass=4):
        self._ck(lib().fdtd_set_time_blocking(self._h, int(steps_per_pass)), "fdtd_set_time_blocking")

    def profile(self, on=True):
        self._ck(lib().fdtd_profile(self._h, 1 if on else 0), "fdtd_profile")

    def profile_read(self):
        a, b, n = C.c_double(0), C.c_double(0), C.c_int64(0)
        self._ck(lib().fdtd_profile_read(self._h, C.byref(a), C.byref(b), C.byref(n)), "fdtd_profile_read")
        return a.value, b.value, n.value

    def set_tuning(self, rows_per_cta=0, warps_per_cta=0):
        self._ck(lib().fdtd_set_tuning(self._h, int(rows_per_cta), int(warps_per_cta)), "fdtd_set_tuning")


def step_group(sims, n):
    """Advance an in-process slab group (contexts created with local_group=True on one stream)."""
    arr = (C.c_void_p * len(sims))(*[s._h.value for s in sims])
    st = lib().fdtd_step_group(arr, len(sims), int(n))
    if st:
        msgs = [lib().fdtd_last_error(s._h).decode() for s in sims]
        raise FDTDError(st, "fdtd_step_group: %s" % [m for m in msgs if m])


def from_scene(scene, device=0, torch_materials=None, **kw):
    """Build a Simulation from an inputs.scene.Scene (materials, ROMs, source, probes)."""
    eps, sig = scene.eps_r, scene.sigma
    if torch_materials is not None:
        eps, sig = torch_materials
    else:
        try:
            import torch

            if isinstance(eps, torch.Tensor) and not eps.is_cuda:
                eps, sig = eps.double().numpy(), sig.double().numpy()
        except ImportError:  # pragma: no cover
            pass
    sim = Simulation(scene.nx, scene.ny, scene.dx, scene.dy, scene.dt, eps, sig, precision=scene.precision,
                     device=device, **kw)
    if scene.placements is not None and len(scene.placements):
        for k, m in enumerate(scene.models):
            sel = scene.placements[scene.placements[:, 0] == k]
            if len(sel):
                sim.add_rom(m, sel[:, 1:3])
    sim.set_source(*scene.source, scene.samples)
    sim.set_probes(scene.probes)
    return sim
