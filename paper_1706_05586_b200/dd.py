"""z-slab domain decomposition of the batched multi-shift CG solves (thin binding of the
dot_dd_* calls of include/dot_b200.h).

Three layouts, all running the same library code path:
  * LocalDD(problems): all ranks in this process (single-GPU emulation: the halo
    exchange and the sum of the Krylov partials are device copies);
  * NcclDD(problem, rank, world): one rank per process/GPU, NCCL for the exchange;
    the NCCL id travels over the caller's torch.distributed group;
  * TransportDD(problem, rank, world): one rank per process, the library's packed
    halo buffers and partial sums staged through host memory and exchanged by
    torch.distributed point-to-point / all_reduce on the caller's group (gloo).
After `fields(W, V)` every rank's problem has the forward fields of B W and the
adjoint fields of C V cached, and misfit / jacobian run without further solves.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import DotError


class _DD:
    def __init__(self, problems, rank0, world, nccl_id=None, transport=None):
        self._lib = _abi.load()
        self.problems = list(problems)
        if transport is not None:
            h = C.c_void_p()
            self._transport = transport
            code = self._lib.dot_dd_create_transport(self.problems[0]._h, int(rank0), int(world),
                                                     C.byref(transport.struct), C.byref(h))
            if code:
                raise DotError(code, (self._lib.dot_dd_last_error(None) or b"").decode())
            self._h = h
            return
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


class TorchTransport:
    """dot_transport callbacks over a torch.distributed group (CPU tensors: gloo).

    sendrecv(peer, send, recv): isend of the library's host send buffer and irecv into its
    receive buffer (both posted before waiting, so neighbour chains cannot deadlock);
    allreduce_sum(buf, n): in-place all_reduce of n doubles.  Argument marshalling only."""

    SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t)
    ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t)

    def __init__(self, group=None):
        self.group = group
        self.errors = []
        self._sr = self.SENDRECV(self._sendrecv)
        self._ar = self.ALLREDUCE(self._allreduce)
        self.struct = _abi.DotTransport(None, C.cast(self._sr, C.c_void_p), C.cast(self._ar, C.c_void_p))

    @staticmethod
    def _view(addr, nbytes, dtype):
        import torch
        return torch.frombuffer((C.c_char * nbytes).from_address(addr), dtype=dtype)

    def _sendrecv(self, ctx, peer, send, send_bytes, recv, recv_bytes):
        import torch
        import torch.distributed as tdist
        try:
            reqs = []
            if send_bytes:
                reqs.append(tdist.isend(self._view(send, send_bytes, torch.uint8), int(peer), group=self.group))
            if recv_bytes:
                reqs.append(tdist.irecv(self._view(recv, recv_bytes, torch.uint8), int(peer), group=self.group))
            for r in reqs:
                r.wait()
            return 0
        except Exception as e:          # reported to the library as a failed exchange
            self.errors.append(repr(e))
            return 1

    def _allreduce(self, ctx, buf, n):
        import torch
        import torch.distributed as tdist
        try:
            if n:
                tdist.all_reduce(self._view(buf, 8 * n, torch.float64), group=self.group)
            return 0
        except Exception as e:
            self.errors.append(repr(e))
            return 1


class TransportDD(_DD):
    """One rank per process, exchanged through torch.distributed (e.g. gloo) on `group`."""

    def __init__(self, problem, rank, world, group=None):
        super().__init__([problem], rank, world, transport=TorchTransport(group))


class NcclDD(_DD):
    """One rank per process; `problem` is this rank's (same config and parameters on all)."""

    def __init__(self, problem, rank, world, group=None):
        super().__init__([problem], rank, world, nccl_id=broadcast_unique_id(rank, group))
