"""Multi-GPU orchestration of the DOT step: RHS columns sharded across ranks
(one process per GPU, torch.distributed for the plumbing).

Partition: rank r owns a contiguous block of the point
sources and of the point detectors and solves only those (n_freq x (n_s + n_d)/N
RHS).  Exchange steps that the method really has:
  * misfit: sum over source blocks of ||R[:, block]||_F^2  -> all_reduce (scalar)
  * sketched fields U W = sum_blocks U_block W_block on the support S
    (and Lambda V likewise)                                   -> all_reduce (K x l x n_freq)
  * full Jacobian rows of a detector block need every source field on S
                                                              -> all_gather (K x n_s x n_freq)
  * Jacobian blocks of the detector shards                   -> gather to rank 0
Only fields restricted to the support S of dA/dp cross NVLink,
so the exchanged volume is tiny next to the solves.

`backend` is any object with the DOTProblem methods used below; the GPU path
passes a DOTProblem, the CPU gloo tests pass an oracle-backed stand-in.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ShardPlan:
    rank: int
    world: int
    n_s: int
    n_d: int

    @staticmethod
    def _block(n, world, r):
        """Balanced contiguous split: block sizes differ by at most one (a rank may own
        nothing when n < world)."""
        return r * n // world, (r + 1) * n // world

    @property
    def per_src(self):
        return (self.n_s + self.world - 1) // self.world

    @property
    def per_det(self):
        return (self.n_d + self.world - 1) // self.world

    def src_block(self, r=None):
        return self._block(self.n_s, self.world, self.rank if r is None else r)

    def det_block(self, r=None):
        return self._block(self.n_d, self.world, self.rank if r is None else r)


def selection(n, lo, hi):
    E = np.zeros((n, max(hi - lo, 0)))
    E[np.arange(lo, hi), np.arange(hi - lo)] = 1.0
    return E


def make_problem_for_rank(dot, cfg, wl, plan, **kw):
    """Every rank holds the full problem description (all sources/detectors);
    the shard decides which RHS it solves.  The workspace is sized for this rank's share of
    the systems (n_freq x (its source + detector columns)), leaving device memory for the
    gathered fields and Jacobian blocks."""
    if plan.world > 1 and "max_rhs" not in kw and "workspace_bytes" not in kw:
        kw["max_rhs"] = cfg.n_freq * (plan.per_src + plan.per_det)
    return dot.DOTProblem.from_config(cfg, wl.src_nodes, wl.det_nodes, **kw)


def _torch():
    import torch
    return torch


def _as_dev(x, like):
    torch = _torch()
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return x.to(like.device) if like is not None else x
    t = torch.as_tensor(np.asarray(x))
    return t.to(like.device) if like is not None else t


def sharded_step(backend, plan: ShardPlan, p, W, V, data=None, device=None, comm_device=None):
    """One step: set_params, all-source + all-detector solves, full-data misfit,
    full Jacobian and (when W or V is given) the sketched Jacobian (W, V).  Returns a
    dict with misfit, J_full (rank 0), J_sketch, d2h_bytes."""
    torch = _torch()
    host_io = not (isinstance(p, torch.Tensor) and p.is_cuda)
    sketch = W is not None or V is not None
    if data is not None:
        backend.set_data(data)
    backend.set_params(p)
    if plan.world == 1:
        where = 0 if host_io else 1
        J_full = backend.jacobian(None, None, where=where)          # all solves + full J (DMMA)
        m = backend.misfit(None, None)                                # cached forward fields
        J_sk = backend.jacobian(W, V) if sketch else None             # by combination of cached fields
        d2h = (J_full.nbytes + (J_sk.nbytes if sketch else 0) + 8) if host_io else 0
        return {"misfit": m, "J_full": J_full, "J_sketch": J_sk, "d2h_bytes": d2h}

    import torch.distributed as tdist
    # compute device: where the backend's fields live (CUDA for DOTProblem); comm device:
    # where the process group wants tensors (CUDA for NCCL, CPU for gloo)
    dev = device
    if dev is None:
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    cdev = comm_device if comm_device is not None else dev

    def T(x):                                   # backend output -> torch tensor on the compute device
        return x.to(dev) if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x), device=dev)

    def all_reduce_(t):
        tc = t if t.device == cdev else t.to(cdev)
        tdist.all_reduce(torch.view_as_real(tc) if tc.is_complex() else tc)
        if tc is not t:
            t.copy_(tc)

    slo, shi = plan.src_block()
    dlo, dhi = plan.det_block()
    Es = _as_dev(selection(plan.n_s, slo, shi), torch.empty(0, device=dev))
    Ed = _as_dev(selection(plan.n_d, dlo, dhi), torch.empty(0, device=dev))
    if sketch:
        Wn = np.eye(plan.n_s) if W is None else (W.detach().cpu().numpy() if isinstance(W, torch.Tensor)
                                                  else np.asarray(W))
        Vn = np.eye(plan.n_d) if V is None else (V.detach().cpu().numpy() if isinstance(V, torch.Tensor)
                                                  else np.asarray(V))
        Wm = np.zeros_like(Wn)
        Wm[slo:shi] = Wn[slo:shi]
        Vm = np.zeros_like(Vn)
        Vm[dlo:dhi] = Vn[dlo:dhi]
        Wm, Vm = _as_dev(Wm, Es), _as_dev(Vm, Es)

    # forward solves of my source block and adjoint solves of my detector block, one batch
    if hasattr(backend, "prefetch_fields"):
        backend.prefetch_fields(Es if shi > slo else None, Ed if dhi > dlo else None,
                                ls=None if shi > slo else 0, ld=None if dhi > dlo else 0)
    # misfit over my source block, all detectors
    m_part = backend.misfit(Es, None) if shi > slo else 0.0
    m = torch.tensor([m_part], dtype=torch.float64, device=dev)
    all_reduce_(m)
    # sampled fields of my blocks on S (cached from the solves); an empty block contributes
    # a zero-width panel
    G = T(backend.support_weights())
    K = G.shape[0]

    def fields(side, E, nonempty):
        if nonempty:
            return T(backend.fields_on_support(side, E))
        return torch.zeros((backend.n_freq, 0, K), dtype=torch.complex128, device=dev)
    U_blk = fields(0, Es, shi > slo)                  # [nf][ns_r][K]
    L_blk = fields(1, Ed, dhi > dlo)                  # [nf][nd_r][K]
    J_sk = None
    if sketch:
        # sketched fields: partial combinations of my blocks, summed over ranks
        UW = T(backend.fields_on_support(0, Wm))
        LV = T(backend.fields_on_support(1, Vm))
        for t in (UW, LV):
            all_reduce_(t)
        J_sk = T(backend.contract(LV, UW, G))
    # full Jacobian: every source field on S to every rank, rows of my detector block
    nf, K = U_blk.shape[0], U_blk.shape[2]
    pad = torch.zeros((nf, plan.per_src, K), dtype=U_blk.dtype, device=cdev)
    pad[:, : U_blk.shape[1]] = U_blk.to(cdev)
    parts = [torch.empty_like(pad) for _ in range(plan.world)]
    tdist.all_gather([torch.view_as_real(t) for t in parts], torch.view_as_real(pad))
    U_all = torch.cat([parts[r][:, : plan.src_block(r)[1] - plan.src_block(r)[0]] for r in range(plan.world)], 1)
    J_rows = T(backend.contract(L_blk, U_all.to(dev), G)) if dhi > dlo else None   # [nf][nd_r][ns][np]
    # J blocks to rank 0, one rank at a time into the final array (peak: J + one block)
    J_full = None
    n_p = G.shape[1]
    if plan.rank == 0:
        J_full = torch.empty((nf, plan.n_d, plan.n_s, n_p), dtype=torch.complex128, device=cdev)
        if J_rows is not None:
            J_full[:, dlo:dhi] = J_rows.to(cdev)
        tmp = torch.empty(nf * plan.per_det * plan.n_s * n_p, dtype=torch.complex128, device=cdev)
        for r in range(1, plan.world):
            lo, hi = plan.det_block(r)
            if hi <= lo:
                continue
            blk = tmp[: nf * (hi - lo) * plan.n_s * n_p].view(nf, hi - lo, plan.n_s, n_p)   # contiguous
            tdist.recv(torch.view_as_real(blk), src=r)
            J_full[:, lo:hi] = blk
        del tmp
    elif J_rows is not None:
        tdist.send(torch.view_as_real(J_rows.to(cdev).contiguous()), dst=0)
    d2h = 0
    if host_io:
        d2h += 8
        if J_sk is not None:
            J_sk = J_sk.cpu().numpy()
            d2h += J_sk.nbytes
        if J_full is not None:
            J_full = J_full.cpu().numpy()
            d2h += J_full.nbytes
    return {"misfit": float(m.item()), "J_full": J_full, "J_sketch": J_sk, "d2h_bytes": d2h}
