"""Seeded synthetic scene generators shared by the oracle and the CUDA path.

Holds none of the time-marching arithmetic: it only produces inputs -- per-cell
materials, ROM placements, source waveform samples and probe locations -- with
the shapes and statistics of BASELINE.json's configs (recipe: DESIGN.md
"Input recipe").  The paper measures on no public dataset; every input is
synthetic and stands in for the paper's PEC-cavity-style tests (Sec. VI).

Material fields (R20): Gaussian copula -- white N(0,1) noise,
Gaussian filter with sigma_f = l/2 cells (applied in Fourier space, periodic),
normalised to unit variance, u = Phi(g), value = lo + (hi - lo) u.  Runs on any
torch device (the 32768^2 bench field is generated on the GPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

C0 = 299792458.0
MU0 = 4e-7 * math.pi
EPS0 = 1.0 / (MU0 * C0 * C0)


def cfl_limit(dx, dy, eps_r_min=1.0, mu_r_min=1.0):
    """eq.(1) with c_max = c0 / sqrt(min eps_r mu_r) (R13)."""
    c = C0 / math.sqrt(eps_r_min * mu_r_min)
    return 1.0 / (c * math.sqrt(1.0 / dx ** 2 + 1.0 / dy ** 2))


# ---------------------------------------------------------------- materials
def smooth_field(ny, nx, corr_len, lo, hi, seed, device="cpu", dtype=None):
    """Smooth random field in [lo, hi] with correlation length corr_len cells (torch tensor)."""
    import torch

    dtype = dtype or (torch.float64 if str(device) == "cpu" else torch.float32)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    w = torch.randn((ny, nx), generator=g, device=device, dtype=dtype)
    sf = corr_len / 2.0
    ky = torch.fft.fftfreq(ny, device=device, dtype=dtype)
    kx = torch.fft.rfftfreq(nx, device=device, dtype=dtype)
    W = torch.fft.rfft2(w)
    del w
    W *= torch.exp(-2.0 * math.pi ** 2 * sf ** 2 * ky[:, None] ** 2)
    W *= torch.exp(-2.0 * math.pi ** 2 * sf ** 2 * kx[None, :] ** 2)
    f = torch.fft.irfft2(W, s=(ny, nx))
    del W
    f /= f.std()
    f = 0.5 * (1.0 + torch.erf(f / math.sqrt(2.0)))
    return lo + (hi - lo) * f


# ---------------------------------------------------------------- waveforms
def pulse_tau(fmax):
    """tau with the spectrum at fmax at 10 % of DC (R15)."""
    return math.sqrt(2.0 * math.log(10.0)) / (2.0 * math.pi * fmax)


def gaussian_samples(n, dt, fmax, derivative=False, t0=None):
    """Soft Hz source samples g[k] at t = (k + 1/2) dt, amplitude 1 A/m (R15)."""
    tau = pulse_tau(fmax)
    t0 = 4.5 * tau if t0 is None else t0
    t = (np.arange(n) + 0.5) * dt
    a = (t - t0) / tau
    if derivative:
        return -a * np.exp(0.5 - 0.5 * a * a)
    return np.exp(-0.5 * a * a)


# ---------------------------------------------------------------- placements
def place_blocks(nx, ny, sizes, count, seed, nslabs=8, forbid=(), max_tries=2_000_000, margin=7, clear=4):
    """Seeded non-overlapping placements (R19).

    sizes: list of (bx, by) per model; the model of each placement is drawn uniformly.
    Every footprint stays ``margin`` cells away from the PEC walls and from the boundaries of
    ``nslabs`` equal row slabs, and the footprints expanded by ``clear`` cells are pairwise
    disjoint.  The defaults (7, 4) are what four-step passes need (K3: fix-up region =
    block + 2K-1 cells inside the slab, block + K rectangles disjoint); every placement also
    satisfies the one-cell-ring rule of fdtd_add_rom.  ``forbid``: cells (i, j) that must stay
    outside every footprint plus ring (source, probes).
    Returns int32 array (count, 3): (model, i0, j0).
    """
    assert margin >= 1 and clear >= 1
    rng = np.random.default_rng(seed)
    slab = ny // nslabs if nslabs > 1 and ny % nslabs == 0 else ny
    forbid = [(int(i), int(j)) for i, j in forbid]
    B = 64
    buckets = {}  # (bi, bj) -> list of occupied rects [x0, x1) x [y0, y1) (expanded footprints)
    out = []
    tries = 0
    while len(out) < count:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("placement failed after %d tries (%d placed)" % (tries, len(out)))
        m = int(rng.integers(len(sizes)))
        bx, by = sizes[m]
        if nx - bx - margin <= margin or ny - by - margin <= margin:
            raise RuntimeError("grid too small for a %dx%d block with margin %d" % (bx, by, margin))
        i0 = int(rng.integers(margin, nx - bx - margin + 1))
        j0 = int(rng.integers(margin, ny - by - margin + 1))
        if (j0 - margin) // slab != (j0 + by + margin - 1) // slab:  # inside one slab with its margin
            continue
        x0, x1, y0, y1 = i0 - clear, i0 + bx + clear, j0 - clear, j0 + by + clear
        keys = [(a, b) for a in range(x0 // B, (x1 - 1) // B + 1) for b in range(y0 // B, (y1 - 1) // B + 1)]
        hit = False
        for k in keys:
            for (u0, u1, v0, v1) in buckets.get(k, ()):
                if u0 < x1 and x0 < u1 and v0 < y1 and y0 < v1:
                    hit = True
                    break
            if hit:
                break
        if hit:
            continue
        if any(i0 - 1 <= fi <= i0 + bx and j0 - 1 <= fj <= j0 + by for fi, fj in forbid):
            continue
        rect = (x0, x1, y0, y1)
        for k in keys:
            buckets.setdefault(k, []).append(rect)
        out.append((m, i0, j0))
    return np.array(out, dtype=np.int32).reshape(-1, 3)


def inclusion_fill(b, r, seed, eps_lo=2.0, eps_hi=12.0, sig_lo=0.0, sig_hi=0.1, radius=0.35):
    """Centred lossy dielectric disc of radius 0.35 r b fine cells, vacuum outside (R23)."""
    rng = np.random.default_rng(seed)
    N = b * r
    c = (N - 1) / 2.0
    jj, ii = np.mgrid[0:N, 0:N]
    disc = (ii - c) ** 2 + (jj - c) ** 2 <= (radius * N) ** 2
    eps = np.where(disc, rng.uniform(eps_lo, eps_hi, (N, N)), 1.0)
    sig = np.where(disc, rng.uniform(sig_lo, sig_hi, (N, N)), 0.0)
    return eps, sig


def uniform_fill(bx, by, r, seed, eps_lo, eps_hi, sig_lo, sig_hi):
    rng = np.random.default_rng(seed)
    eps = rng.uniform(eps_lo, eps_hi, (by * r, bx * r))
    sig = rng.uniform(sig_lo, sig_hi, (by * r, bx * r))
    return eps, sig


def probes_random(nx, ny, count, seed, holes_mask=None):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        i, j = int(rng.integers(1, nx - 1)), int(rng.integers(1, ny - 1))
        if holes_mask is not None and holes_mask[j, i]:
            continue
        if (i, j) in out:
            continue
        out.append((i, j))
    return np.array(out, dtype=np.int32)


# ---------------------------------------------------------------- scenes
@dataclass
class Scene:
    name: str
    nx: int
    ny: int
    dx: float
    dy: float
    dt: float
    eps_r: object          # (ny, nx) numpy or torch tensor
    sigma: object
    precision: int         # 32 | 64
    steps: int
    source: tuple          # (i, j)
    samples: np.ndarray    # source samples per step
    probes: np.ndarray     # (P, 2) int32 (i, j)
    models: list = field(default_factory=list)      # romgen models
    placements: np.ndarray = None                    # (n, 3) (model, i0, j0)
    meta: dict = field(default_factory=dict)

    def holes_mask(self):
        m = np.zeros((self.ny, self.nx), dtype=bool)
        if self.placements is not None:
            for k, i0, j0 in self.placements:
                md = self.models[k]
                m[j0: j0 + md["by"], i0: i0 + md["bx"]] = True
        return m
