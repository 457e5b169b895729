"""B200-native DOT hot path (arXiv 1706.05586): thin Python binding of libdot_b200.so.

Every numerical step runs in the library's sm_100a kernels; this module only
marshals arguments (numpy arrays -> DOT_HOST, CUDA torch tensors -> DOT_DEVICE)
and owns the device workspace as a torch tensor.  There is no CPU fallback: if
the shared library is missing, importing the problem class raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import DOT_DEVICE, DOT_HOST, DotError  # noqa: F401

__all__ = ["DOTProblem", "DotError", "contract", "sym_eig", "version", "lib"]


def lib():
    return _abi.load()


def version() -> str:
    return lib().dot_version().decode()


def _is_torch(x):
    return type(x).__module__.startswith("torch")


class _Args:
    """Collects the array arguments of one call and fixes their location."""

    def __init__(self, where):
        self.where = where
        self.keep = []

    def ptr(self, x, dtype):
        if x is None:
            return None
        if self.where == DOT_DEVICE:
            import torch
            tdt = {np.float64: torch.float64, np.complex128: torch.complex128, np.int32: torch.int32}[dtype]
            if not _is_torch(x):
                x = torch.as_tensor(np.asarray(x, dtype=dtype))
            x = x.to(device="cuda", dtype=tdt).contiguous()
            self.keep.append(x)
            return C.c_void_p(x.data_ptr())
        if _is_torch(x):
            x = x.detach().cpu().numpy()
        a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
        self.keep.append(a)
        return C.c_void_p(a.ctypes.data)

    def out(self, shape, dtype):
        if self.where == DOT_DEVICE:
            import torch
            tdt = {np.float64: torch.float64, np.complex128: torch.complex128}[dtype]
            t = torch.empty(shape, dtype=tdt, device="cuda")
            self.keep.append(t)
            return t, C.c_void_p(t.data_ptr())
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        if n >= (1 << 20):
            # large host results land in pinned memory (asynchronous DMA, no staging copy)
            import torch
            tdt = {np.float64: torch.float64, np.complex128: torch.complex128}[dtype]
            a = torch.empty(shape, dtype=tdt, pin_memory=torch.cuda.is_available()).numpy()
        else:
            a = np.empty(shape, dtype=dtype)
        self.keep.append(a)
        return a, C.c_void_p(a.ctypes.data)


def _where_of(*xs):
    for x in xs:
        if x is not None and _is_torch(x) and x.is_cuda:
            return DOT_DEVICE
    return DOT_HOST


class DOTProblem:
    """One DOT problem instance (grid, optics, frequencies, sources, detectors)
    on the current CUDA device.  Methods mirror include/dot_b200.h."""

    def __init__(self, n, L, D, mua_in, mua_out, nu, omegas, src_nodes, det_nodes, n_rbf,
                 gamma, eps, cutoff, tol=1e-17, max_iter=4000, workspace_bytes=None, max_rhs=None,
                 stream=None):
        import torch
        self._lib = lib()
        if not torch.cuda.is_available():
            raise RuntimeError("DOTProblem needs a CUDA device (B200); there is no CPU path")
        self.n = tuple(int(v) for v in n)
        self.N = self.n[0] * self.n[1] * self.n[2]
        self.tol = float(tol)
        self.omegas = np.ascontiguousarray(np.asarray(omegas, dtype=np.float64))
        self.src_nodes = np.ascontiguousarray(np.asarray(src_nodes, dtype=np.int64))
        self.det_nodes = np.ascontiguousarray(np.asarray(det_nodes, dtype=np.int64))
        self.n_freq, self.n_src, self.n_det = len(self.omegas), len(self.src_nodes), len(self.det_nodes)
        self.n_rbf, self.n_p = int(n_rbf), 5 * int(n_rbf)
        cfg = _abi.DotConfig(
            self.n[0], self.n[1], self.n[2], float(L[0]), float(L[1]), float(L[2]), float(D),
            float(mua_in), float(mua_out), float(nu), self.n_freq,
            self.omegas.ctypes.data_as(_abi.dp), self.n_src, self.src_nodes.ctypes.data_as(_abi.i64p),
            self.n_det, self.det_nodes.ctypes.data_as(_abi.i64p), self.n_rbf, float(gamma), float(eps),
            float(cutoff), float(tol), int(max_iter))
        h = C.c_void_p()
        _abi.check(self._lib.dot_create(C.byref(cfg), C.byref(h)), None)
        self._h = h
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        _abi.check(self._lib.dot_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)), self._h)
        if workspace_bytes is None:
            want = self._lib.dot_workspace_bytes(
                self._h, int(max_rhs if max_rhs else self.n_freq * (self.n_src + self.n_det)))
            free, _ = torch.cuda.mem_get_info()
            workspace_bytes = int(min(want, 0.85 * free))
        self._ws = torch.empty(int(workspace_bytes), dtype=torch.uint8, device="cuda")
        _abi.check(self._lib.dot_bind_workspace(self._h, C.c_void_p(self._ws.data_ptr()), self._ws.numel()),
                   self._h)

    @classmethod
    def from_config(cls, cfg, src_nodes, det_nodes, **kw):
        """Build from any object with the attributes of synth.DOTConfig."""
        return cls(cfg.n, cfg.L, cfg.D, cfg.mua_anom, cfg.mua_bg, cfg.nu,
                   2.0 * np.pi * np.asarray(cfg.freqs_hz, dtype=np.float64), src_nodes, det_nodes,
                   cfg.n_rbf, cfg.gamma, cfg.eps, cfg.cutoff, **kw)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dot_destroy(self._h)
            self._h = None
            self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code):
        _abi.check(code, self._h)

    # ---------------------------------------------------------------- state
    def set_data(self, data):
        a = _Args(_where_of(data))
        self._check(self._lib.dot_set_data(self._h, a.ptr(data, np.complex128), a.where))

    def set_params(self, p):
        if int(np.prod(p.shape)) != self.n_p:
            raise ValueError(f"p has {int(np.prod(p.shape))} entries, the problem has n_p = {self.n_p}")
        a = _Args(_where_of(p))
        self._check(self._lib.dot_set_params(self._h, a.ptr(p, np.float64), a.where))

    def enable_timing(self, on=True):
        self._check(self._lib.dot_enable_timing(self._h, 1 if on else 0))

    def stats(self) -> dict:
        s = _abi.DotStats()
        self._check(self._lib.dot_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        self._check(self._lib.dot_reset_stats(self._h))

    # ---------------------------------------------------------- paper calls
    def misfit(self, W=None, V=None, return_resid=False):
        """sum_f ||V^T R_f W||_F^2 (and V^T R_f W, [n_freq][ld][ls])."""
        ls = self.n_src if W is None else int(W.shape[1])
        ld = self.n_det if V is None else int(V.shape[1])
        a = _Args(_where_of(W, V))
        m = C.c_double()
        res, rp = a.out((self.n_freq, ld, ls), np.complex128) if return_resid else (None, None)
        self._check(self._lib.dot_misfit(self._h, a.ptr(W, np.float64), ls, a.ptr(V, np.float64), ld, a.where,
                                         C.byref(m), rp))
        return (m.value, res) if return_resid else m.value

    def prefetch_fields(self, W=None, V=None, ls=None, ld=None):
        """Solve the uncached forward fields of B W and adjoint fields of C V in one batch
        (ls / ld = 0 skips a side; W / V None = identity)."""
        ls = self.n_src if (W is None and ls is None) else (0 if ls == 0 else (ls if W is None else int(W.shape[1])))
        ld = self.n_det if (V is None and ld is None) else (0 if ld == 0 else (ld if V is None else int(V.shape[1])))
        a = _Args(_where_of(W, V))
        self._check(self._lib.dot_prefetch_fields(self._h, a.ptr(W, np.float64) if ls else None, ls,
                                                  a.ptr(V, np.float64) if ld else None, ld, a.where))

    def jacobian(self, W=None, V=None, where=None):
        """(W^T (x) V^T) J as [n_freq][ld][ls][n_p] complex."""
        ls = self.n_src if W is None else int(W.shape[1])
        ld = self.n_det if V is None else int(V.shape[1])
        a = _Args(where if where is not None else _where_of(W, V))
        J, jp = a.out((self.n_freq, ld, ls, self.n_p), np.complex128)
        self._check(self._lib.dot_jacobian(self._h, a.ptr(W, np.float64), ls, a.ptr(V, np.float64), ld, a.where, jp))
        return J

    def optimize_directions(self, k, W, V):
        """Replace k random simultaneous sources/detectors by optimized ones.
        Returns (W_hat, V_hat, objective)."""
        a = _Args(_where_of(W, V))
        Wo, wp = a.out(tuple(W.shape), np.float64)
        Vo, vp = a.out(tuple(V.shape), np.float64)
        obj = C.c_double()
        self._check(self._lib.dot_optimize_directions(self._h, int(k), a.ptr(W, np.float64), int(W.shape[1]),
                                                      a.ptr(V, np.float64), int(V.shape[1]), a.where, wp, vp,
                                                      C.byref(obj)))
        return Wo, Vo, obj.value

    def optimize_directions_subspace(self, k, W, V, X0_src, X0_det, iters=5):
        """Replace k random simultaneous sources/detectors by optimized ones found by
        `iters` subspace-iteration steps, matrix-free.  X0_src [n_src][k*block],
        X0_det [n_det][k*block]: add step t starts from block t.
        Returns (W_hat, V_hat, objective)."""
        a = _Args(_where_of(W, V))
        if k < 1 or X0_src.shape[1] % k or X0_det.shape[1] != X0_src.shape[1]:
            raise ValueError("X0_src, X0_det need k*block columns")
        blk = int(X0_src.shape[1]) // k
        Wo, wp = a.out(tuple(W.shape), np.float64)
        Vo, vp = a.out(tuple(V.shape), np.float64)
        obj = C.c_double()
        self._check(self._lib.dot_optimize_directions_subspace(
            self._h, int(k), int(iters), blk, a.ptr(W, np.float64), int(W.shape[1]), a.ptr(V, np.float64),
            int(V.shape[1]), a.ptr(X0_src, np.float64), a.ptr(X0_det, np.float64), a.where, wp, vp, C.byref(obj)))
        return Wo, Vo, obj.value

    # ------------------------------------------------------------ components
    def absorption(self):
        a = _Args(DOT_HOST)
        mu, mp = a.out((self.N,), np.float64)
        self._check(self._lib.dot_absorption(self._h, mp, DOT_HOST))
        return mu

    def support(self):
        K = C.c_int32()
        self._check(self._lib.dot_support(self._h, C.byref(K), None, None, DOT_HOST))
        nodes = np.empty(K.value, dtype=np.int64)
        G = np.empty((K.value, self.n_p), dtype=np.float64)
        if K.value:
            self._check(self._lib.dot_support(self._h, C.byref(K), C.c_void_p(nodes.ctypes.data),
                                              C.c_void_p(G.ctypes.data), DOT_HOST))
        return nodes, G

    def support_weights(self):
        """G on the support as a CUDA tensor [K][n_p] (device copy, no host trip)."""
        import torch
        K = C.c_int32()
        self._check(self._lib.dot_support(self._h, C.byref(K), None, None, DOT_DEVICE))
        G = torch.empty((K.value, self.n_p), dtype=torch.float64, device="cuda")
        if K.value:
            self._check(self._lib.dot_support(self._h, C.byref(K), None, C.c_void_p(G.data_ptr()), DOT_DEVICE))
        return G

    def fields_on_support(self, side, coeff=None, where=None):
        """Fields of B coeff (side 0) / C coeff (side 1) on the support S:
        [n_freq][ncols][K] complex (cached solves reused / combined)."""
        n_side = self.n_src if side == 0 else self.n_det
        ncols = n_side if coeff is None else int(coeff.shape[1])
        K = C.c_int32()
        self._check(self._lib.dot_support(self._h, C.byref(K), None, None, DOT_HOST))
        a = _Args(where if where is not None else _where_of(coeff))
        X, xp = a.out((self.n_freq, ncols, K.value), np.complex128)
        self._check(self._lib.dot_fields_on_support(self._h, int(side), a.ptr(coeff, np.float64), ncols, a.where,
                                                    xp))
        return X

    def contract(self, Lam, U, G=None):
        """J[f][j][i][k] = -sum_s Lam[f][j][s] U[f][i][s] G[s][k] with this problem's support
        weights G (block-sparse by basis), on its stream: Lam [n_freq][ld][K], U [n_freq][ls][K]
        CUDA complex128 tensors.  (G is accepted for interface symmetry and must be the
        problem's own support weights.)"""
        import torch
        Lam, U = Lam.contiguous(), U.contiguous()
        nf, ld, K = Lam.shape
        ls = U.shape[1]
        if nf != self.n_freq or U.shape[0] != nf or U.shape[2] != K:
            raise ValueError("panels must be [n_freq][cols][K] on this problem's support")
        J = torch.empty((nf, ld, ls, self.n_p), dtype=torch.complex128, device=Lam.device)
        self._check(self._lib.dot_contract_fields(self._h, int(ld), int(ls), C.c_void_p(Lam.data_ptr()),
                                                  C.c_void_p(U.data_ptr()), C.c_void_p(J.data_ptr())))
        return J

    def samples(self):
        n = C.c_int32()
        self._check(self._lib.dot_samples(self._h, C.byref(n), None, DOT_HOST))
        nodes = np.empty(n.value, dtype=np.int64)
        if n.value:
            self._check(self._lib.dot_samples(self._h, C.byref(n), C.c_void_p(nodes.ctypes.data), DOT_HOST))
        return nodes

    def apply(self, freq, u):
        u = u.reshape(-1, self.N)
        a = _Args(_where_of(u))
        out, op = a.out(tuple(u.shape), np.complex128)
        self._check(self._lib.dot_apply(self._h, int(freq), int(u.shape[0]), a.ptr(u, np.complex128), op, a.where))
        return out

    def solve(self, b, freq):
        """Dense right-hand sides b [nrhs][N]; freq [nrhs] frequency indices."""
        b = b.reshape(-1, self.N)
        nr = int(b.shape[0])
        freq = np.broadcast_to(np.asarray(freq, dtype=np.int32), (nr,))
        a = _Args(_where_of(b))
        x, xp = a.out((nr, self.N), np.complex128)
        iters = np.zeros(nr, dtype=np.int32)
        self._check(self._lib.dot_solve(self._h, nr, a.ptr(freq, np.int32), a.ptr(b, np.complex128), xp, a.where,
                                        iters.ctypes.data_as(_abi.i32p)))
        return x, iters

    def solve_sampled(self, side, coeff=None):
        """Sampled solutions [n_freq][ncols][n_samples] for side 0 (B coeff) / 1 (C coeff)."""
        n_side = self.n_src if side == 0 else self.n_det
        ncols = n_side if coeff is None else int(coeff.shape[1])
        a = _Args(_where_of(coeff))
        nP = len(self.samples())
        X, xp = a.out((self.n_freq, ncols, nP), np.complex128)
        self._check(self._lib.dot_solve_sampled(self._h, int(side), a.ptr(coeff, np.float64), ncols, a.where, xp))
        return X


def contract(Lam, U, G, stream=None):
    """Stateless DMMA contraction J[b][j][i][k] = -sum_s Lam[b][j][s] U[b][i][s] G[s][k]
    on CUDA torch tensors (complex128 Lam [nb][ld][K], U [nb][ls][K]; float64 G [K][n_p])."""
    import torch
    nb, ld, K = Lam.shape
    ls = U.shape[1]
    n_p = G.shape[1]
    Lam, U, G = Lam.contiguous(), U.contiguous(), G.contiguous()
    J = torch.empty((nb, ld, ls, n_p), dtype=torch.complex128, device=Lam.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _abi.check(lib().dot_contract(C.c_void_p(s.cuda_stream), nb, K, ld, ls, n_p, C.c_void_p(Lam.data_ptr()),
                                  C.c_void_p(U.data_ptr()), C.c_void_p(G.data_ptr()), C.c_void_p(J.data_ptr())))
    return J


def sym_eig(A):
    """Host symmetric eigensolver of the library (descending eigenvalues)."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    w = np.empty(n)
    Z = np.empty((n, n))
    code = lib().dot_sym_eig(n, A.ctypes.data_as(_abi.dp), w.ctypes.data_as(_abi.dp), Z.ctypes.data_as(_abi.dp))
    if code:
        raise DotError(code, "sym_eig failed")
    return w, Z
