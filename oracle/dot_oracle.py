"""DOT hot-path oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain, slow, obviously-correct CPU implementation, in float64 / complex128, of
what the B200 path computes, written from PAPER.md (arXiv 1706.05586).  Each
function cites the passage it follows ("PAPER.md L<line>, <section/equation>").
Where the paper is silent the DESIGN.md reading (R<n>) is named.

Library primitives used as single steps: scipy.sparse (assembly container),
scipy.sparse.linalg.splu (sparse direct LU, the forward/adjoint solves),
numpy.linalg.svd / qr (the small SVDs of PAPER.md Sec. 3.2-3.3).  No blocking,
fusion or reordering beyond the paper's formulas.

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  operator      second-order manufactured solution (Dirichlet + Robin), symmetry,
                reciprocity C^T A^-1 B = (C^T A^-1 B)^T for coinciding src/det,
                dense-inverse solve on a tiny grid
  PaLS          Wendland closed forms, Heaviside closed forms, dmu/dp vs central FD
  misfit        W = V = I equals the dense-inverse full-data misfit; exhaustive
                Rademacher enumeration averages to it (Theorem 3.1)
  jacobian      central finite differences of the sketched residual
  optimize      Lemma 3.2 optimality certificates, dominance over random feasible
                candidates, angular brute force, Table 1 SVD sizes (golden)
  subspace      converges to the exact Theorem 3.6/3.7 direction; one step equals the
                brute-force best direction in span(P X0) (Rayleigh-Ritz); orthogonality
No function here is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "Grid", "make_grid", "assemble", "frequency_matrix", "wendland", "wendland_d",
    "heaviside", "heaviside_d", "pals_phi", "absorption", "dmu_dp", "jacobian_weights",
    "source_matrix", "detector_matrix", "Problem", "make_problem", "simulate_data",
    "measurements", "sketched_residual", "misfit", "jacobian", "jacobian_from_fields",
    "frob_objective", "remove_sources", "remove_detectors", "add_sources", "add_detectors",
    "optimize_directions", "complement_basis", "subspace_add_direction", "optimize_directions_subspace",
]


# --------------------------------------------------------------------------- grid
@dataclass
class Grid:
    """Interior FD nodes of [0,Lx]x[0,Ly]x[0,Lz] (Eq. (2.1)).

    Lateral faces x1 = 0, Lx and x2 = 0, Ly carry phi = 0 (Dirichlet, L136): the
    nodes x_i = (i+1) hx, i = 0..nx-1, hx = Lx/(nx+1), exclude them.  The faces
    x3 = 0 and x3 = c carry the Robin condition (L137): z_k = k hz,
    k = 0..nz-1, hz = Lz/(nz-1) include them (reading R1).
    theta = 1/2 on the Robin planes, 1 elsewhere (row scaling, reading R2).
    """
    n: tuple
    L: tuple
    hx: float
    hy: float
    hz: float
    X: np.ndarray
    Y: np.ndarray
    Z: np.ndarray
    theta: np.ndarray

    @property
    def N(self):
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def cell_volume(self):
        return self.hx * self.hy * self.hz


def make_grid(n, L) -> Grid:
    nx, ny, nz = n
    if min(nx, ny) < 1 or nz < 2:
        raise ValueError("need nx, ny >= 1 and nz >= 2")
    hx, hy, hz = L[0] / (nx + 1), L[1] / (ny + 1), L[2] / (nz - 1)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    X = ((i + 1) * hx).reshape(-1).astype(np.float64)
    Y = ((j + 1) * hy).reshape(-1).astype(np.float64)
    Z = (k * hz).reshape(-1).astype(np.float64)
    theta = np.where((k == 0) | (k == nz - 1), 0.5, 1.0).reshape(-1)
    return Grid(tuple(n), tuple(L), hx, hy, hz, X, Y, Z, theta)


# ----------------------------------------------------------------------- operator
def assemble(grid: Grid, D: float, mu: np.ndarray, omega: float, nu: float) -> sp.csr_matrix:
    """A(p, omega): FD discretisation of Eq. (2.1).

    -div(D grad phi) + mu phi + i omega/nu phi with constant D (L141 "D(x) is
    well-specified"; reading R4).  7-point stencil; Dirichlet lateral faces enter
    as zero neighbours; the Robin rows 0.25 phi + (D/2) dphi/dxi = 0 are handled
    by ghost-node elimination and the Robin-plane rows are scaled by 1/2 so that
    A is complex symmetric (reading R2/R3).  Row n:

      theta_n [ D/hx^2 (2u - u_W - u_E) + D/hy^2 (2u - u_S - u_N) + (mu_n + i omega/nu) u ]
      + D/hz^2 sum_{existing z-neighbours m} (u - u_m) + rho_n u,

    rho_n = 1/(2 hz) on the Robin planes (from the ghost node), 0 elsewhere.
    """
    nx, ny, nz = grid.n
    N = grid.N
    idx = np.arange(N).reshape(nz, ny, nx)
    th = grid.theta.reshape(nz, ny, nx)
    cx, cy, cz = D / grid.hx ** 2, D / grid.hy ** 2, D / grid.hz ** 2
    rows, cols, vals = [], [], []

    diag = th * (2 * cx + 2 * cy) + th * (mu.reshape(nz, ny, nx) + 1j * omega / nu)
    diag = diag.astype(np.complex128)
    # z couplings: each existing z-neighbour adds cz to the diagonal
    nzn = np.full((nz, ny, nx), 2.0)
    nzn[0] -= 1
    nzn[-1] -= 1
    diag = diag + cz * nzn
    robin = np.zeros((nz, ny, nx))
    robin[0] = robin[-1] = 1.0 / (2 * grid.hz)
    diag = diag + robin
    rows.append(idx.reshape(-1))
    cols.append(idx.reshape(-1))
    vals.append(diag.reshape(-1))

    def couple(a, b, w):
        rows.extend([a.reshape(-1), b.reshape(-1)])
        cols.extend([b.reshape(-1), a.reshape(-1)])
        vals.extend([-w.reshape(-1).astype(np.complex128)] * 2)

    couple(idx[:, :, :-1], idx[:, :, 1:], th[:, :, :-1] * cx)   # x neighbours
    couple(idx[:, :-1, :], idx[:, 1:, :], th[:, :-1, :] * cy)   # y neighbours
    couple(idx[:-1], idx[1:], np.full(idx[:-1].shape, cz))      # z neighbours
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(N, N))
    return A


def frequency_matrix(grid: Grid) -> sp.dia_matrix:
    """E: the frequency term's matrix, A(omega) = A(0) + i omega/nu E.

    Here E = diag(theta) (reading R2: the paper's E has zero Robin rows because
    its Robin rows are pure boundary-condition rows; ours keep half a cell)."""
    return sp.diags(grid.theta.astype(np.complex128))


# --------------------------------------------------------------------------- PaLS
def wendland(r):
    """Wendland C2 CSRBF psi(r) = (1-r)_+^4 (4r+1) ("compactly
    supported radial basis function"; reading R7)."""
    r = np.asarray(r, dtype=np.float64)
    return np.where(r < 1.0, (1.0 - r) ** 4 * (4.0 * r + 1.0), 0.0)


def wendland_d(r):
    """psi'(r) = -20 r (1-r)_+^3."""
    r = np.asarray(r, dtype=np.float64)
    return np.where(r < 1.0, -20.0 * r * (1.0 - r) ** 3, 0.0)


def heaviside(t, eps):
    """Approximate Heaviside H_eps (reading R8):
    0 for t < -eps, 1 for t > eps, (1 + t/eps + sin(pi t/eps)/pi)/2 between."""
    t = np.asarray(t, dtype=np.float64)
    mid = 0.5 * (1.0 + t / eps + np.sin(np.pi * t / eps) / np.pi)
    return np.where(t < -eps, 0.0, np.where(t > eps, 1.0, mid))


def heaviside_d(t, eps):
    """dH_eps/dt = (1 + cos(pi t/eps)) / (2 eps) on |t| <= eps, 0 outside."""
    t = np.asarray(t, dtype=np.float64)
    return np.where(np.abs(t) <= eps, (1.0 + np.cos(np.pi * t / eps)) / (2.0 * eps), 0.0)


def _rbf_geometry(p, grid, gamma):
    P = np.asarray(p, dtype=np.float64).reshape(-1, 5)
    out = []
    for a, b, cx, cy, cz in P:
        dx, dy, dz = grid.X - cx, grid.Y - cy, grid.Z - cz
        d2 = dx * dx + dy * dy + dz * dz
        r = np.sqrt(b * b * d2 + gamma * gamma)   # ||beta (x - chi)||^dagger
        out.append((a, b, dx, dy, dz, d2, r))
    return out


def pals_phi(p, grid: Grid, gamma: float) -> np.ndarray:
    """PaLS function phi(x, p) = sum_j alpha_j psi(||beta_j (x - chi_j)||^dagger)
    with ||x||^dagger = sqrt(||x||^2 + gamma^2) (Eq. (2.3))."""
    phi = np.zeros(grid.N)
    for a, b, dx, dy, dz, d2, r in _rbf_geometry(p, grid, gamma):
        phi += a * wendland(r)
    return phi


def absorption(p, grid: Grid, cfg) -> np.ndarray:
    """mu(x, p) = mu_in H(phi - c) + mu_out (1 - H(phi - c)) (Eq. (2.4))."""
    H = heaviside(pals_phi(p, grid, cfg.gamma) - cfg.cutoff, cfg.eps)
    return cfg.mua_anom * H + cfg.mua_bg * (1.0 - H)


def dmu_dp(p, grid: Grid, cfg) -> np.ndarray:
    """d mu / d p_k (N x n_p): chain rule through Eq. (2.4) and Eq. (2.3).

    d phi/d alpha_j = psi(r_j); d phi/d beta_j = alpha_j psi'(r_j) beta_j |x-chi_j|^2 / r_j;
    d phi/d chi_j,d = -alpha_j psi'(r_j) beta_j^2 (x_d - chi_j,d) / r_j,
    with r_j = ||beta_j (x - chi_j)||^dagger; parameter order (alpha, beta, cx, cy, cz) per basis.
    """
    geo = _rbf_geometry(p, grid, cfg.gamma)
    phi = np.zeros(grid.N)
    for a, b, dx, dy, dz, d2, r in geo:
        phi += a * wendland(r)
    s = (cfg.mua_anom - cfg.mua_bg) * heaviside_d(phi - cfg.cutoff, cfg.eps)
    cols = []
    for a, b, dx, dy, dz, d2, r in geo:
        dpsi = wendland_d(r)
        cols.append(s * wendland(r))
        cols.append(s * a * dpsi * b * d2 / r)
        for dd in (dx, dy, dz):
            cols.append(s * a * dpsi * (-b * b * dd) / r)
    return np.stack(cols, axis=1)


def jacobian_weights(p, grid: Grid, cfg) -> np.ndarray:
    """G(x, k): the diagonal of dA/dp_k ("a diagonal matrix if we only
    invert for absorption").  With our row scaling dA/dp_k = diag(theta dmu/dp_k)."""
    return grid.theta[:, None] * dmu_dp(p, grid, cfg)


# --------------------------------------------------------------- sources/detectors
def source_matrix(grid: Grid, nodes) -> sp.csc_matrix:
    """B = [b_1 .. b_ns]: unit point sources at grid nodes,
    b_s = theta_s e_s / (hx hy hz) (reading R6)."""
    nodes = np.asarray(nodes)
    vals = grid.theta[nodes] / grid.cell_volume
    return sp.csc_matrix((vals.astype(np.complex128), (nodes, np.arange(len(nodes)))),
                         shape=(grid.N, len(nodes)))


def detector_matrix(grid: Grid, nodes) -> sp.csc_matrix:
    """C: rows of C^T are the detectors; point detectors
    measure phi at a node, c_d = e_d (reading R6)."""
    nodes = np.asarray(nodes)
    return sp.csc_matrix((np.ones(len(nodes), np.complex128), (nodes, np.arange(len(nodes)))),
                         shape=(grid.N, len(nodes)))


# ------------------------------------------------------------------------ problem
@dataclass
class Problem:
    cfg: object
    grid: Grid
    src_nodes: np.ndarray
    det_nodes: np.ndarray
    B: sp.csc_matrix
    C: sp.csc_matrix
    omegas: np.ndarray
    data: np.ndarray | None = None       # (n_freq, n_d, n_s) complex
    solves: int = 0                      # PDE solves performed (Table 4 accounting)

    def operator(self, mu, f):
        return assemble(self.grid, self.cfg.D, mu, self.omegas[f], self.cfg.nu)

    def factor(self, p, f):
        mu = absorption(p, self.grid, self.cfg)
        return spla.splu(self.operator(mu, f).tocsc(), permc_spec="MMD_AT_PLUS_A")

    def solve(self, lu, rhs, trans="N"):
        rhs = np.asarray(rhs.todense() if sp.issparse(rhs) else rhs, dtype=np.complex128)
        self.solves += rhs.shape[1]
        return lu.solve(rhs, trans=trans)


def make_problem(cfg, src_nodes, det_nodes) -> Problem:
    grid = make_grid(cfg.n, cfg.L)
    return Problem(cfg, grid, np.asarray(src_nodes), np.asarray(det_nodes),
                   source_matrix(grid, src_nodes), detector_matrix(grid, det_nodes),
                   2.0 * np.pi * np.asarray(cfg.freqs_hz, dtype=np.float64))


def measurements(prob: Problem, p) -> np.ndarray:
    """M_f = C^T A(omega_f, p)^-1 B, (n_freq, n_d, n_s) (Eq. (2.5))."""
    out = []
    for f in range(len(prob.omegas)):
        lu = prob.factor(p, f)
        Z = prob.solve(lu, prob.B)
        out.append(np.asarray(prob.C.T @ Z))
    return np.stack(out)


def simulate_data(prob: Problem, p_true, xi, noise) -> np.ndarray:
    """Synthetic data d: measurements at the hidden level set plus relative
    Gaussian noise, d = m + noise |m| xi with xi complex standard normal drawn by
    synth (BASELINE.json configs[0] "1% Gaussian noise"; reading R10)."""
    M = measurements(prob, p_true)
    return M + noise * np.abs(M) * xi


def sketched_residual(prob: Problem, p, W, V, return_fields=False):
    """V^T R_f W = V^T C^T z_i - V^T D_f w_i with A z_i = B w_i
    (Eq. (EsTResidual)); (n_freq, ld, ls)."""
    out, fields = [], []
    for f in range(len(prob.omegas)):
        lu = prob.factor(p, f)
        Z = prob.solve(lu, prob.B @ W)
        out.append(V.T @ (prob.C.T @ Z) - V.T @ prob.data[f] @ W)
        fields.append((lu, Z))
    out = np.stack(out)
    return (out, fields) if return_fields else out


def misfit(prob: Problem, p, W, V) -> float:
    """||(W^T (x) V^T) r(p)||_2^2 = sum_f ||V^T R_f W||_F^2 (
    frequencies stacked per footnote L269)."""
    S = sketched_residual(prob, p, W, V)
    return float(np.sum(np.abs(S) ** 2))


def jacobian_from_fields(Z, Y, G) -> np.ndarray:
    """Entries y_j^T (dA/dp_k) z_i with the minus sign of Eq. (2.8), by a direct
    triple loop (Eq. (Jacobian kth column)).
    Z: (N, ls) forward fields, Y: (N, ld) adjoint fields, G: (N, n_p)
    diagonal of dA/dp_k.  Returns (ld, ls, n_p)."""
    ld, ls, n_p = Y.shape[1], Z.shape[1], G.shape[1]
    J = np.zeros((ld, ls, n_p), dtype=np.complex128)
    for j in range(ld):
        for i in range(ls):
            for k in range(n_p):
                J[j, i, k] = -np.sum(Y[:, j] * G[:, k] * Z[:, i])
    return J


def jacobian(prob: Problem, p, W, V, return_fields=False):
    """Sketched Jacobian (W^T (x) V^T) J, (n_freq, ld, ls, n_p) (PAPER.md L372-376,
    Eq. (3.12); L966-972): z_i = A^-1 B w_i, y_j = A^-T C v_j,
    J[f, j, i, k] = -y_j^T diag(G_k) z_i."""
    G = jacobian_weights(p, prob.grid, prob.cfg)
    out, fields = [], []
    for f in range(len(prob.omegas)):
        lu = prob.factor(p, f)
        Z = prob.solve(lu, prob.B @ W)
        Y = prob.solve(lu, prob.C @ V, trans="T")
        out.append(jacobian_from_fields(Z, Y, G))
        fields.append((Z, Y))
    out = np.stack(out)
    return (out, fields) if return_fields else out


# ----------------------------------------- simultaneous optimized sources/detectors
def _real_rows(Mc):
    """Stack real and imaginary parts as extra columns: the Frobenius norm of a
    complex block equals that of [Re, Im] (footnote L185 "split m_i in its real
    and imaginary parts")."""
    return np.concatenate([Mc.real, Mc.imag], axis=1)


def frob_objective(Jsk) -> float:
    """||(W^T (x) V^T) J||_F^2 over all frequencies (PAPER.md Eq. (maxprob))."""
    return float(np.sum(np.abs(Jsk) ** 2))


def complement_basis(M) -> np.ndarray:
    """Orthonormal V_c with [orth(M) V_c] orthogonal ("[V V_c] is orthogonal")."""
    n, l = M.shape
    Q, _ = np.linalg.qr(M, mode="complete")
    return Q[:, l:]


def remove_detectors(Jsk, s):
    """Theorem 3.4: SVD of V^T [J^_1 .. J^_ls] = Phi Omega Psi^T,
    Gamma = first ld - s left singular vectors.  Jsk = (W^T (x) V^T) J as
    (n_freq, ld, ls, n_p); its (ld x ls n_p n_freq) unfolding is V^T[J^_1..J^_ls]."""
    nf, ld, ls, n_p = Jsk.shape
    M = _real_rows(np.transpose(Jsk, (1, 0, 2, 3)).reshape(ld, -1))
    Phi, om, _ = np.linalg.svd(M, full_matrices=False)
    return Phi[:, :ld - s], om


def remove_sources(Jsk, s):
    """Theorem 3.5: SVD of W^T [J~_1 .. J~_ld], Gamma = first
    ls - s left singular vectors."""
    nf, ld, ls, n_p = Jsk.shape
    M = _real_rows(np.transpose(Jsk, (2, 0, 1, 3)).reshape(ls, -1))
    Phi, om, _ = np.linalg.svd(M, full_matrices=False)
    return Phi[:, :ls - s], om


def add_detectors(J_WI, V, s):
    """Theorem 3.6: J_WI = (W^T (x) I) J, (n_freq, n_d, ls, n_p);
    SVD of V_c^T [J^_1 .. J^_ls] = Phi Omega Psi^T; Q_s = V_c [phi_1..phi_s]."""
    nf, nd, ls, n_p = J_WI.shape
    M = _real_rows(np.transpose(J_WI, (1, 0, 2, 3)).reshape(nd, -1))
    Vc = complement_basis(V)
    Phi, om, _ = np.linalg.svd(Vc.T @ M, full_matrices=False)
    return Vc @ Phi[:, :s], om, (Vc.T @ M).shape


def add_sources(J_IV, W, s):
    """Theorem 3.7: J_IV = (I (x) V^T) J, (n_freq, ld, n_s, n_p);
    SVD of W_c^T [J~_1 .. J~_ld]; Q~_s = W_c [phi_1..phi_s]."""
    nf, ld, ns, n_p = J_IV.shape
    M = _real_rows(np.transpose(J_IV, (2, 0, 1, 3)).reshape(ns, -1))
    Wc = complement_basis(W)
    Phi, om, _ = np.linalg.svd(Wc.T @ M, full_matrices=False)
    return Wc @ Phi[:, :s], om, (Wc.T @ M).shape


def optimize_directions(prob: Problem, p, W, V, s, trace=None):
    """Replace s simultaneous random sources and s detectors by simultaneous
    optimized ones (Sec. 3.3.2): phase one alternately removes
    one source, then one detector (Theorems 3.5, 3.4); phase two alternately adds
    one source, then one detector (Theorems 3.7, 3.6).  The full Jacobian is
    computed once (n_s + n_d solves per frequency, L462-463); every step
    re-contracts it with the current W, V (reading R13).  New columns are scaled
    to length sqrt(n_s) / sqrt(n_d) (L475-477).  Returns (W_hat, V_hat).
    """
    ns, nd = W.shape[0], V.shape[0]
    G = jacobian_weights(p, prob.grid, prob.cfg)
    U_all, L_all = [], []
    for f in range(len(prob.omegas)):
        lu = prob.factor(p, f)
        U_all.append(prob.solve(lu, prob.B))
        L_all.append(prob.solve(lu, prob.C, trans="T"))

    def jac(Wm, Vm):
        return np.stack([jacobian_from_fields(U_all[f] @ Wm, L_all[f] @ Vm, G)
                         for f in range(len(prob.omegas))])

    W, V = np.array(W, dtype=np.float64), np.array(V, dtype=np.float64)
    for _ in range(s):                         # phase one: remove
        Gam, _ = remove_sources(jac(W, V), 1)
        W = W @ Gam
        Gam, _ = remove_detectors(jac(W, V), 1)
        V = V @ Gam
        if trace is not None:
            trace.append(("remove", W.shape[1], V.shape[1], frob_objective(jac(W, V))))
    for _ in range(s):                         # phase two: add
        q, _, shape = add_sources(jac(np.eye(ns), V), W, 1)
        W = np.concatenate([W, np.sqrt(ns) * q], axis=1)
        if trace is not None:
            trace.append(("add_source", shape))
        q, _, shape = add_detectors(jac(W, np.eye(nd)), V, 1)
        V = np.concatenate([V, np.sqrt(nd) * q], axis=1)
        if trace is not None:
            trace.append(("add_detector", shape, frob_objective(jac(W, V))))
    return W, V


# ------------------------ optimized directions by subspace iteration (reading R16)
def _orth(M):
    """Orthonormal basis of span(M) (reduced QR)."""
    Q, _ = np.linalg.qr(M)
    return Q


def _sign_fix(q):
    """Sign convention shared with the GPU path: the largest-magnitude entry is positive."""
    i = int(np.argmax(np.abs(q)))
    return q if q[i] >= 0 else -q


def subspace_add_direction(Xr, M, X0, iters):
    """Matrix-free form of Theorems 3.6 / 3.7 by subspace iteration
    (BASELINE.json configs[3] "5 subspace iterations maximizing ||V^T J W||_F";
    reading R16).  Xr: (n, m) real unfolding [Re, Im] of V^T-combined (or W-combined)
    Jacobian slices, M: (n, l) current directions, X0: (n, p) starting block (caller's
    random draws).  With P = I - Q_M Q_M^T and K = P Xr Xr^T P:
        Q_0 = orth(P X0);  Y_t = K Q_{t-1},  Q_t = orth(Y_t)  (t = 1 .. iters-1);
        Y_iters = K Q_{iters-1};  H = Q^T Y (Rayleigh-Ritz);  q = Q e_max(H).
    As iters grows, q -> V_c phi_1 of Theorem 3.6 (top left singular vector of
    V_c^T [J^_1 .. J^_ls]).  Returns the unit vector q (sign: largest entry > 0)."""
    n = Xr.shape[0]
    QM = _orth(M)
    P = np.eye(n) - QM @ QM.T
    K = P @ Xr @ Xr.T @ P
    Q = _orth(P @ X0)
    Y = K @ Q
    for _ in range(iters - 1):
        Q = _orth(Y)
        Y = K @ Q
    H = Q.T @ Y
    H = 0.5 * (H + H.T)
    w, E = np.linalg.eigh(H)
    q = Q @ E[:, np.argmax(w)]
    q = P @ q
    return _sign_fix(q / np.linalg.norm(q))


def optimize_directions_subspace(prob: Problem, p, W, V, s, iters, X0_src, X0_det):
    """Two-phase replacement of s directions where the add steps
    use subspace_add_direction instead of the exact SVD (reading R16); the remove
    steps are Theorems 3.5 / 3.4 as in optimize_directions.  X0_src (n_s, s*blk),
    X0_det (n_d, s*blk): add step t starts from columns t*blk .. (t+1)*blk - 1 (a block
    reused after its own Ritz vector was added would be rank deficient).  The oracle builds the
    explicit Jacobian slices from all-source / all-detector LU solves; the GPU path
    applies K matrix-free with 2 n_freq solves per block vector per iteration."""
    ns, nd = W.shape[0], V.shape[0]
    G = jacobian_weights(p, prob.grid, prob.cfg)
    U_all, L_all = [], []
    for f in range(len(prob.omegas)):
        lu = prob.factor(p, f)
        U_all.append(prob.solve(lu, prob.B))
        L_all.append(prob.solve(lu, prob.C, trans="T"))

    def jac(Wm, Vm):
        return np.stack([jacobian_from_fields(U_all[f] @ Wm, L_all[f] @ Vm, G)
                         for f in range(len(prob.omegas))])

    W, V = np.array(W, dtype=np.float64), np.array(V, dtype=np.float64)
    for _ in range(s):                         # phase one: remove (exact, Theorems 3.5, 3.4)
        Gam, _ = remove_sources(jac(W, V), 1)
        W = W @ Gam
        Gam, _ = remove_detectors(jac(W, V), 1)
        V = V @ Gam
    blk = X0_src.shape[1] // s
    for t in range(s):                         # phase two: add by subspace iteration
        J_IV = jac(np.eye(ns), V)               # (nf, ld, ns, n_p)
        Xr = _real_rows(np.transpose(J_IV, (2, 0, 1, 3)).reshape(ns, -1))
        q = subspace_add_direction(Xr, W, X0_src[:, t * blk:(t + 1) * blk], iters)
        W = np.concatenate([W, np.sqrt(ns) * q[:, None]], axis=1)
        J_WI = jac(W, np.eye(nd))               # (nf, nd, ls, n_p)
        Xr = _real_rows(np.transpose(J_WI, (1, 0, 2, 3)).reshape(nd, -1))
        q = subspace_add_direction(Xr, V, X0_det[:, t * blk:(t + 1) * blk], iters)
        V = np.concatenate([V, np.sqrt(nd) * q[:, None]], axis=1)
    return W, V
