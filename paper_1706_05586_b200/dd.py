"""z-slab domain decomposition of the batched COCG solves (thin binding of the
dot_dd_* calls of include/dot_b200.h).

Two layouts, both running the same library code path:
  * LocalDD(problems): all ranks in this process (single-GPU emulation: the halo
    exchange and the all-reduce of the Krylov partial sums are device copies);
  * NcclDD(problem, rank, world): one rank per process/GPU, NCCL for the exchange;
    the NCCL id travels over the caller's torch.distributed group.
After `fields(W, V)` every rank's problem has the forward fields of B W and the
adjoint fields of C V cached, and misfit / jacobian run without further solves.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import DotError


class _DD:
    def __init__(self, problems, rank0, world, nccl_id=None):
        self._lib = _abi.load()
        self.problems = list(problems)
        arr = (C.c_void_p * len(self.problems))(*[p._h.value for p in self.problems])
        h = C.c_void_p()
        idp = None
        if nccl_id is not None:
            self._id = (C.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
            idp = C.cast(self._id, C.c_void_p)
        code = self._lib.dot_dd_create(arr, len(self.problems), int(rank0), int(world), idp, C.byref(h))
        if code:
            raise DotError(code, (self._lib.dot_dd_last_error(None) or b"").decode())
        self._h = h

    def fields(self, W=None, V=None, ls=None, ld=None):
        """Decomposed solve of B W (ls = 0 to skip) and C V (ld = 0 to skip); W/V None = identity."""
        p0 = self.problems[0]
        ls = p0.n_src if (W is None and ls is None) else (0 if ls == 0 else (ls if W is None else int(W.shape[1])))
        ld = p0.n_det if (V is None and ld is None) else (0 if ld == 0 else (ld if V is None else int(V.shape[1])))
        keep = []

        def ptr(M):
            if M is None:
                return None
            a = np.ascontiguousarray(np.asarray(M, dtype=np.float64))
            keep.append(a)
            return C.c_void_p(a.ctypes.data)
        code = self._lib.dot_dd_fields(self._h, ptr(W) if ls else None, ls, ptr(V) if ld else None, ld, 0)
        if code:
            raise DotError(code, (self._lib.dot_dd_last_error(self._h) or b"").decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dot_dd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalDD(_DD):
    """All `world` ranks in this process (problems[r] is rank r)."""

    def __init__(self, problems):
        super().__init__(problems, 0, len(problems))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    lib = _abi.load()
    code = lib.dot_nccl_unique_id(C.cast(buf, C.c_void_p))
    if code:
        raise DotError(code, (lib.dot_dd_last_error(None) or b"").decode())
    return bytes(buf)


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank receives it over torch.distributed."""
    import torch
    import torch.distributed as tdist
    obj = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class NcclDD(_DD):
    """One rank per process; `problem` is this rank's (same config and parameters on all)."""

    def __init__(self, problem, rank, world, group=None):
        super().__init__([problem], rank, world, nccl_id=broadcast_unique_id(rank, group))
