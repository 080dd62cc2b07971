"""ROM construction -- the one-time CPU input-generation step (north_star).

``BASELINE.json`` north_star: "The ROM construction (projection, CFL-extension
perturbation) is a one-time CPU input-generation step that emits the reduced
matrices both paths consume."  This module is that step.  Both the fp64 oracle
(``oracle/``) and the CUDA path (``paper_1609_07114_b200``) read the matrices
it emits; neither imports the other.  Everything here is fp64 NumPy/SciPy.

Pipeline (citations are PAPER.md lines):
  1. ``fine_system``  -- descriptor system of the fine region, eq:sys1a/b
     (L286-292) with R^, F^, B^, L^ of eq:R, eq:F_f, eq:B, eq:L, eq:F11, eq:K
     (L323-382); boundary rows with half lengths (eq:updateExS L217-222, L257).
  2. ``collapse``     -- exact projection onto coarse-edge ports (R9):
     the r fine boundary E nodes of one coarse edge are one degree of freedom
     under eq:equalE (L608-611); ports become the nY coarse interface edges.
  3. ``sprim``        -- SPRIM (L393): block Arnoldi on (G + s0 C)^{-1} C with
     starting block (G + s0 C)^{-1} B, basis split into E / H rows and each part
     orthonormalised in Krylov order, giving V = blkdiag(V1, V2) (eq:V L394-400;
     DESIGN.md R10).
  4. ``reduce``       -- congruence eq:R11_tilde ... eq:K_tilde (L431-447).
  5. ``extend_cfl``   -- clip the singular values of R11~^-1/2 K~ R22~^-1/2 at
     2/dt_target (eq:CFLgeneralized L741-745; R11/R12).

Emitted model (dict, fp64, C order): bx, by, r, q1, q2, R11 (q1 x q1), R22
(q2 x q2), F11 (q1 x q1), K (q1 x q2), L (q1 x nY) with nY = 2 bx + 2 by, ports
ordered S (bx), N (bx), W (by), E (by).  B~ = L~ S_c is implied, S_c =
diag(-dx, +dx, +dy, -dy) per side (eq:cond3rom L717 with eq:S L698-707,
collapsed).  literal=True (NEXT-1): L is q1 x nP with the nP = r nY fine ports in
the same side order, B~ = L~ diag(-dx/r, +dx/r, +dy/r, -dy/r per side) and the
coupling is the paper's own eq:sysform with T and 1/r (eq:equalE, eq:averH).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

C0 = 299792458.0
MU0 = 4e-7 * math.pi
EPS0 = 1.0 / (MU0 * C0 * C0)


# --------------------------------------------------------------------------
# 1. fine-region descriptor system
# --------------------------------------------------------------------------
def fine_system(bx, by, r, dx, dy, eps_r, sigma, mu_r=None):
    """Assemble the fine-region system of Sec. II for a bx x by coarse block refined r times.

    eps_r, sigma: per fine cell, shape (Ny, Nx) with Nx = bx r, Ny = by r.
    Returns dict with diagonal vectors r11, f11 (nE), r22 (nH), sparse K (nE x nH),
    B (nE x nP, E rows only), L (nE x nP selector), S (nP diag), plus sizes.
    State order: Ex row-major (j outer), then Ey, then Hz.
    """
    Nx, Ny = bx * r, by * r
    fdx, fdy = dx / r, dy / r
    eps_r = np.asarray(eps_r, dtype=np.float64).reshape(Ny, Nx)
    sigma = np.asarray(sigma, dtype=np.float64).reshape(Ny, Nx)
    mu = MU0 * (np.ones((Ny, Nx)) if mu_r is None else np.asarray(mu_r, dtype=np.float64).reshape(Ny, Nx))
    nEx, nEy, nH = Nx * (Ny + 1), (Nx + 1) * Ny, Nx * Ny
    nE = nEx + nEy

    def ex(i, j):
        return j * Nx + i

    def ey(i, j):
        return nEx + j * (Nx + 1) + i

    def hz(i, j):
        return j * Nx + i

    r11 = np.zeros(nE)
    f11 = np.zeros(nE)
    rows, cols, vals = [], [], []
    # Ex nodes: eq:updateEx (interior) / eq:updateExS (S, N boundary: half dual length fdy/2)
    for j in range(Ny + 1):
        for i in range(Nx):
            if j == 0:
                e, s, lp = eps_r[0, i], sigma[0, i], fdy / 2
            elif j == Ny:
                e, s, lp = eps_r[Ny - 1, i], sigma[Ny - 1, i], fdy / 2
            else:
                e = 0.5 * (eps_r[j - 1, i] + eps_r[j, i])
                s = 0.5 * (sigma[j - 1, i] + sigma[j, i])
                lp = fdy
            k = ex(i, j)
            r11[k] = fdx * lp * EPS0 * e       # D_lx D_l'y D_eps_x (eq:R11)
            f11[k] = fdx * lp * s / 2          # D_lx D_l'y D_sig_x / 2 (eq:F11)
            if j < Ny:                          # + dx^ H_above (eq:updateEx)
                rows.append(k); cols.append(hz(i, j)); vals.append(+fdx)
            if j > 0:                           # - dx^ H_below
                rows.append(k); cols.append(hz(i, j - 1)); vals.append(-fdx)
    # Ey nodes: Ey analogue (L223), sign of eq:updateEymat: - dy^ (H_right - H_left)
    for j in range(Ny):
        for i in range(Nx + 1):
            if i == 0:
                e, s, lp = eps_r[j, 0], sigma[j, 0], fdx / 2
            elif i == Nx:
                e, s, lp = eps_r[j, Nx - 1], sigma[j, Nx - 1], fdx / 2
            else:
                e = 0.5 * (eps_r[j, i - 1] + eps_r[j, i])
                s = 0.5 * (sigma[j, i - 1] + sigma[j, i])
                lp = fdx
            k = ey(i, j)
            r11[k] = fdy * lp * EPS0 * e
            f11[k] = fdy * lp * s / 2
            if i < Nx:
                rows.append(k); cols.append(hz(i, j)); vals.append(-fdy)
            if i > 0:
                rows.append(k); cols.append(hz(i - 1, j)); vals.append(+fdy)
    K = sp.csr_matrix((vals, (rows, cols)), shape=(nE, nH))
    r22 = fdx * fdy * mu.ravel()                  # D_A D_mu (R^22)
    # ports S, N, W, E (eq:B, eq:L, eq:S; signs DESIGN.md R4)
    port_node, port_sign, port_len = [], [], []
    for i in range(Nx):
        port_node.append(ex(i, 0)); port_sign.append(-1.0); port_len.append(fdx)
    for i in range(Nx):
        port_node.append(ex(i, Ny)); port_sign.append(+1.0); port_len.append(fdx)
    for j in range(Ny):
        port_node.append(ey(0, j)); port_sign.append(+1.0); port_len.append(fdy)
    for j in range(Ny):
        port_node.append(ey(Nx, j)); port_sign.append(-1.0); port_len.append(fdy)
    nP = len(port_node)
    pn = np.array(port_node)
    S = np.array(port_sign) * np.array(port_len)
    B = sp.csr_matrix((S, (pn, np.arange(nP))), shape=(nE, nP))
    L = sp.csr_matrix((np.ones(nP), (pn, np.arange(nP))), shape=(nE, nP))
    return dict(bx=bx, by=by, r=r, dx=dx, dy=dy, Nx=Nx, Ny=Ny, nE=nE, nH=nH, nP=nP,
                r11=r11, f11=f11, r22=r22, K=K, B=B, L=L, S=S, port_node=pn)


def full_order(sysf):
    """Total state count nE + nH (the paper's 'order', e.g. 7,600 at N^=50, L840)."""
    return sysf["nE"] + sysf["nH"]


def descriptor_matrices(sysf, dt):
    """Dense-free sparse R^, F^ of eq:R / eq:F_f (L323-338) at time step dt."""
    nE, nH, K = sysf["nE"], sysf["nH"], sysf["K"]
    R11 = sp.diags(sysf["r11"] / dt)
    R22 = sp.diags(sysf["r22"] / dt)
    R = sp.bmat([[R11, -0.5 * K], [-0.5 * K.T, R22]], format="csr")
    F = sp.bmat([[sp.diags(sysf["f11"]), -0.5 * K], [0.5 * K.T, sp.csr_matrix((nH, nH))]], format="csr")
    B = sp.vstack([sysf["B"], sp.csr_matrix((nH, sysf["nP"]))], format="csr")
    L = sp.vstack([sysf["L"], sp.csr_matrix((nH, sysf["nP"]))], format="csr")
    return R, F, B, L


def fine_cfl_limit(sysf):
    """dt_f = 2 / s_max(R^11^-1/2 K^ R^22^-1/2): the dt at which eq:cond1 fails (L708, R13)."""
    X = sp.diags(1 / np.sqrt(sysf["r11"])) @ sysf["K"] @ sp.diags(1 / np.sqrt(sysf["r22"]))
    smax = _smax(X)
    return 2.0 / smax


def _smax(X):
    n = min(X.shape)
    if n <= 400:
        A = X.toarray() if sp.issparse(X) else np.asarray(X)
        return float(np.linalg.svd(A, compute_uv=False)[0])
    v = spla.svds(X, k=1, return_singular_vectors=False, tol=1e-12)
    return float(v[0])


# --------------------------------------------------------------------------
# 2. collapse onto coarse-edge ports (R9)
# --------------------------------------------------------------------------
def collapse(sysf):
    """Merge the r fine boundary E nodes of every coarse interface edge into one node.

    Collapsed E ordering: the nY merged port nodes first (port order S,N,W,E), then the
    interior E nodes.  Returns the collapsed system: diagonal r11c, f11c (nEc), r22,
    Kc (nEc x nH), Sc (nY), plus the 0/1 map Pi (nE x nEc).
    B_c = Pi^T B^ T = [diag(Sc); 0], L_c = Pi^T L^ T / r = [I; 0].
    """
    r, nE, nP = sysf["r"], sysf["nE"], sysf["nP"]
    nY = nP // r
    col = np.full(nE, -1, dtype=np.int64)
    col[sysf["port_node"]] = np.arange(nP) // r          # fine port k -> coarse port k // r
    interior = np.flatnonzero(col < 0)
    col[interior] = nY + np.arange(interior.size)
    nEc = nY + interior.size
    Pi = sp.csr_matrix((np.ones(nE), (np.arange(nE), col)), shape=(nE, nEc))
    r11c = Pi.T @ sysf["r11"]
    f11c = Pi.T @ sysf["f11"]
    Kc = (Pi.T @ sysf["K"]).tocsr()
    Sc = np.array([sysf["S"][k * r: (k + 1) * r].sum() for k in range(nY)])  # = +-dx, +-dy
    return dict(bx=sysf["bx"], by=sysf["by"], r=r, dx=sysf["dx"], dy=sysf["dy"], nY=nY, nEc=nEc,
                nH=sysf["nH"], r11=r11c, f11=f11c, r22=sysf["r22"], K=Kc, Sc=Sc, Pi=Pi)


def full_order_model(csys):
    """V = I on the collapsed (or literal) system: the exact (unreduced) embedded model."""
    nEc, nY = csys["nEc"], csys["nY"]
    L = np.zeros((nEc, nY))
    L[np.arange(nY), np.arange(nY)] = 1.0
    return dict(bx=csys["bx"], by=csys["by"], r=csys["r"], q1=nEc, q2=csys["nH"],
                R11=np.diag(csys["r11"]), R22=np.diag(csys["r22"]), F11=np.diag(csys["f11"]),
                K=csys["K"].toarray(), L=L, n_clipped=0, literal=bool(csys.get("literal", False)))


# --------------------------------------------------------------------------
# 2b. the paper-literal port set (NEXT-1): nP fine boundary nodes, no collapse
# --------------------------------------------------------------------------
def literal_system(sysf):
    """The uncollapsed fine system with its E nodes reordered port nodes first (port order
    S, N, W, E; nP = r nY of them), in the dict layout `sprim_basis` / `reduce` consume: the
    ports are the nP fine hanging-variable nodes of eq:equalE / eq:averH (L608-616) and
    B^ = L^ S with S the signed fine lengths (eq:B, eq:S)."""
    nE, nP = sysf["nE"], sysf["nP"]
    perm = np.concatenate([sysf["port_node"], np.setdiff1d(np.arange(nE), sysf["port_node"])])
    Pm = sp.csr_matrix((np.ones(nE), (perm, np.arange(nE))), shape=(nE, nE))  # old -> new
    return dict(bx=sysf["bx"], by=sysf["by"], r=sysf["r"], dx=sysf["dx"], dy=sysf["dy"], nY=nP, nEc=nE,
                nH=sysf["nH"], r11=sysf["r11"][perm], f11=sysf["f11"][perm], r22=sysf["r22"],
                K=(Pm.T @ sysf["K"]).tocsr(), Sc=sysf["S"].copy(), Pi=Pm, literal=True)


def with_port_directions(V1, nP):
    """Make the E basis contain the nP port-node unit vectors (ports are the first nP rows):
    the literal coupling needs L~^T = V1[:nP] of full row rank (A1 regular, R9).
    The port directions come first, then V1's columns in order with the port rows projected out
    (ordered Gram-Schmidt, R10), so truncating keeps V1's leading directions."""
    P = np.zeros((V1.shape[0], nP))
    P[np.arange(nP), np.arange(nP)] = 1.0
    return _orth_ordered(np.hstack([P, V1]))


# --------------------------------------------------------------------------
# 3. SPRIM (R10)
# --------------------------------------------------------------------------
def sprim_basis(csys, q, fmax, defl_tol=1e-10):
    """SPRIM basis with q1 = ceil(q/2), q2 = floor(q/2) where the Krylov space allows it.

    The E and H parts of an m-vector Krylov basis can have rank < m, so m grows until both parts
    reach their share (or the space is exhausted); each part keeps its first directions in Krylov
    order (the span of the E / H rows of the leading Krylov vectors, so the moments they match and
    the port directions of the first block are never traded for later ones).
    """
    q1w, q2w = (q + 1) // 2, q // 2
    m = q1w
    for _ in range(8):
        V1, V2 = _sprim_basis_m(csys, m, fmax, defl_tol)
        if (V1.shape[1] >= q1w and V2.shape[1] >= q2w) or m >= csys["nEc"] + csys["nH"]:
            break
        m = int(m + max(q1w - V1.shape[1], q2w - V2.shape[1], 1) * 1.5)
    return V1[:, :q1w], V2[:, :q2w]


def _sprim_basis_m(csys, m, fmax, defl_tol=1e-10):
    """Structure-preserving block Arnoldi basis V1 (nEc x q1), V2 (nH x q2) from m Krylov vectors.

    Semi-discrete pencil of R(x'-x) + F(x'+x) = B u (eq:sys1a): C = blkdiag(R11, R22),
    G = [[2 F11, -K], [K^T, 0]].  Krylov space of (G + s0 C)^{-1} C from (G + s0 C)^{-1} B,
    real s0 = pi * fmax, C-inner product, Gram-Schmidt run twice, deflation defl_tol; the E and
    H rows of the m vectors are orthonormalised separately (directions ordered by singular value).
    """
    nEc, nH, nY = csys["nEc"], csys["nH"], csys["nY"]
    s0 = math.pi * fmax
    r11, f11, r22, K = csys["r11"], csys["f11"], csys["r22"], csys["K"]
    # (G + s0 C) x = b, eliminating H: x_H = (b_H - K^T x_E) / (s0 r22)
    schur = (sp.diags(2 * f11 + s0 * r11) + K @ sp.diags(1.0 / (s0 * r22)) @ K.T).tocsc()
    lu = spla.splu(schur)

    def solve(bE, bH):
        xE = lu.solve(bE + K @ (bH / (s0 * r22)[:, None]))
        xH = (bH - K.T @ xE) / (s0 * r22)[:, None]
        return np.vstack([xE, xH])

    cdiag = np.concatenate([r11, r22])

    def cdot(u, v):
        return float(np.dot(u * cdiag, v))

    B0 = np.zeros((nEc, nY))
    B0[np.arange(nY), np.arange(nY)] = csys["Sc"]
    X0 = solve(B0, np.zeros((nH, nY)))
    m = min(m, nEc + nH)
    Wmat = np.zeros((nEc + nH, m))
    W = []

    def add(v):
        """Classical Gram-Schmidt in the C-inner product, run twice (CGS2), with deflation."""
        n0 = math.sqrt(cdot(v, v))
        if n0 == 0.0:
            return False
        k = len(W)
        for _ in range(2):
            if k:
                v = v - Wmat[:, :k] @ (Wmat[:, :k].T @ (cdiag * v))
        n1 = math.sqrt(cdot(v, v))
        if n1 <= defl_tol * n0:
            return False
        Wmat[:, k] = v / n1
        W.append(Wmat[:, k])
        return True

    # block Arnoldi: the next block is M applied to the whole previous block (one multi-RHS
    # solve per block), then Gram-Schmidt column by column; the Krylov space is unchanged.
    block = [X0[:, c] for c in range(nY)]
    while len(W) < m and block:
        nxt = []
        for v in block:
            if len(W) >= m:
                break
            if add(v):
                nxt.append(W[-1])
        if len(W) >= m or not nxt:
            break
        Wb = np.array(nxt).T
        Y = solve(r11[:, None] * Wb[:nEc], r22[:, None] * Wb[nEc:])  # M w = (G+s0C)^-1 C w
        block = [Y[:, c] for c in range(Y.shape[1])]
    Wm = Wmat[:, :len(W)]
    V1 = _orth_ordered(Wm[:nEc])
    V2 = _orth_ordered(Wm[nEc:])
    return V1, V2


def _orth_ordered(A, tol=1e-10):
    """Orthonormal basis of span(A) built column by column in Krylov order (classical Gram-Schmidt
    run twice; a column is deflated when less than tol of its norm remains), so that the first k
    directions span the E (or H) rows of the first Krylov vectors and keep their moments, ports
    included (R10)."""
    Q = np.zeros_like(A)
    k = 0
    for j in range(A.shape[1]):
        v = A[:, j].copy()
        n0 = np.linalg.norm(v)
        if n0 == 0.0:
            continue
        for _ in range(2):
            if k:
                v = v - Q[:, :k] @ (Q[:, :k].T @ v)
        n1 = np.linalg.norm(v)
        if n1 <= tol * n0:
            continue
        Q[:, k] = v / n1
        k += 1
    return Q[:, :k]


def _orth(A, tol=1e-12):
    try:
        U, s, _ = np.linalg.svd(A, full_matrices=False)
    except np.linalg.LinAlgError:  # gesdd can fail to converge on ill-scaled bases; gesvd does not
        import scipy.linalg as sla
        U, s, _ = sla.svd(A, full_matrices=False, lapack_driver="gesvd")
    k = int(np.sum(s > tol * s[0])) if s.size and s[0] > 0 else 0
    return U[:, :k]


# --------------------------------------------------------------------------
# 4. congruence (eq:R11_tilde ... eq:K_tilde)
# --------------------------------------------------------------------------
def reduce(csys, V1, V2):
    R11 = V1.T @ (csys["r11"][:, None] * V1)
    R22 = V2.T @ (csys["r22"][:, None] * V2)
    F11 = V1.T @ (csys["f11"][:, None] * V1)
    K = V1.T @ (csys["K"] @ V2)
    L = V1[: csys["nY"], :].T.copy()           # V1^T L_c with L_c = [I; 0] (ports first)
    sym = lambda A: 0.5 * (A + A.T)            # exact symmetry of congruences
    return dict(bx=csys["bx"], by=csys["by"], r=csys["r"], q1=V1.shape[1], q2=V2.shape[1],
                R11=sym(R11), R22=sym(R22), F11=sym(F11), K=np.ascontiguousarray(K),
                L=np.ascontiguousarray(L), n_clipped=0, literal=bool(csys.get("literal", False)))


# --------------------------------------------------------------------------
# 5. CFL extension (eq:CFLgeneralized)
# --------------------------------------------------------------------------
def _sqrtm_spd(A):
    w, U = np.linalg.eigh(A)
    if w.min() <= 1e-14 * w.max():
        raise ValueError("matrix is not SPD (eigenvalue floor check)")
    return (U * np.sqrt(w)) @ U.T, (U / np.sqrt(w)) @ U.T


def generalized_singular_values(model):
    """s_k of R11~^-1/2 K~ R22~^-1/2 (eq:CFLgeneralized), descending."""
    _, i1 = _sqrtm_spd(model["R11"])
    _, i2 = _sqrtm_spd(model["R22"])
    return np.linalg.svd(i1 @ model["K"] @ i2, compute_uv=False)


def rom_cfl_limit(model):
    s = generalized_singular_values(model)
    return 2.0 / s[0] if s.size and s[0] > 0 else math.inf


def extend_cfl(model, dt_target, margin=1e-6):
    """Clip s_k at (2/dt_target)(1 - margin); only K~ changes (L740-745, R11)."""
    h1, i1 = _sqrtm_spd(model["R11"])
    h2, i2 = _sqrtm_spd(model["R22"])
    U, s, Wt = np.linalg.svd(i1 @ model["K"] @ i2, full_matrices=False)
    cap = (2.0 / dt_target) * (1.0 - margin)
    out = dict(model)
    nclip = int(np.sum(s > cap))
    out["n_clipped"] = nclip
    if nclip == 0:
        return out
    out["K"] = np.ascontiguousarray(h1 @ (U * np.minimum(s, cap)) @ Wt @ h2)
    return out


def check_passivity(model, dt, tol=1e-12):
    """eq:cond1rom-3rom (L713-719): returns (ok, min_eig_R, min_eig_FpFt)."""
    q1, q2 = model["q1"], model["q2"]
    Kt = model["K"]
    R = np.block([[model["R11"] / dt, -0.5 * Kt], [-0.5 * Kt.T, model["R22"] / dt]])
    F = np.block([[model["F11"], -0.5 * Kt], [0.5 * Kt.T, np.zeros((q2, q2))]])
    # scale-free test: symmetric scaling by diag(R)^-1/2
    d = 1 / np.sqrt(np.abs(np.diag(R)))
    lamR = np.linalg.eigvalsh((R * d[:, None]) * d[None, :]).min()
    FF = F + F.T
    lamF = np.linalg.eigvalsh(FF).min() if q1 + q2 else 0.0
    okF = lamF >= -tol * max(1e-300, np.abs(FF).max())
    return bool(lamR > 0 and okF), float(lamR), float(lamF)


# --------------------------------------------------------------------------
# one-call driver
# --------------------------------------------------------------------------
def build_rom(bx, by, r, dx, dy, eps_r, sigma, q, fmax, dt_target=None, full=False, literal=False):
    """Fine assembly -> collapse (or the literal nP-port set) -> SPRIM(q) -> reduce -> optional
    clip at dt_target.  literal: the paper's own port set (nP = r nY fine hanging variables,
    eq:equalE / eq:averH); the E basis then holds the nP port directions plus ceil(q/2) SPRIM
    directions (q1 = nP + ceil(q/2), q2 = floor(q/2))."""
    sysf = fine_system(bx, by, r, dx, dy, eps_r, sigma)
    csys = literal_system(sysf) if literal else collapse(sysf)
    if full:
        model = full_order_model(csys)
    else:
        V1, V2 = sprim_basis(csys, q, fmax)
        if literal:
            V1 = with_port_directions(V1, csys["nY"])[:, : csys["nY"] + (q + 1) // 2]
        model = reduce(csys, V1, V2)
    model["natural_dt_limit"] = rom_cfl_limit(model) if not full else None
    model["fine_dt_limit"] = fine_cfl_limit(sysf)
    if dt_target is not None:
        model = extend_cfl(model, dt_target)
    return model


def save_model(path, model):
    np.savez(path, **{k: np.asarray(v) for k, v in model.items() if v is not None})


def load_model(path):
    z = np.load(path)
    m = {k: z[k] for k in z.files}
    for k in ("bx", "by", "r", "q1", "q2", "n_clipped"):
        if k in m:
            m[k] = int(m[k])
    if "literal" in m:
        m["literal"] = bool(m["literal"])
    return m
