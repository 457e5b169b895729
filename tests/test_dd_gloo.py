"""Host side of the multi-process z-slab decomposition on CPU (gloo, world 2): rank 0
creates the NCCL unique id through the library (dot_nccl_unique_id, NCCL loaded at
run time) and every rank receives the same 128 bytes over torch.distributed -- the
handshake NcclDD performs before ncclCommInitRank (which needs the GPUs)."""
import os
import socket

import torch
import torch.distributed as tdist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1706_05586_b200.dd import broadcast_unique_id
        nid = broadcast_unique_id(rank)
        out = [None] * world
        tdist.all_gather_object(out, nid)
        q.put(("ok", rank, out))
        tdist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put(("error", rank, repr(e)))


def test_nccl_unique_id_broadcast_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] == "ok" for r in res), res
    for _, _, ids in res:
        assert len(ids[0]) == 128 and ids[0] == ids[1]
    assert res[0][2][0] == res[1][2][0]


def _transport_worker(rank, world, port, q):
    """The TorchTransport callbacks as the library calls them (through the C function
    pointers of dot_transport, on library-owned host buffers)."""
    try:
        import ctypes as C

        import numpy as np
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1706_05586_b200.dd import TorchTransport
        t = TorchTransport()
        SR = TorchTransport.SENDRECV
        AR = TorchTransport.ALLREDUCE
        sr = C.cast(t.struct.sendrecv, SR)
        ar = C.cast(t.struct.allreduce_sum, AR)
        out = {}
        # halo chain as dd_solve issues it: lower neighbour first, then upper (sizes mirror)
        for peer in (rank - 1, rank + 1):
            if not 0 <= peer < world:
                continue
            n_send, n_recv = 3 + rank, 3 + peer
            send = (C.c_double * n_send)(*[100.0 * rank + i for i in range(n_send)])
            recv = (C.c_double * n_recv)()
            rc = sr(None, peer, C.addressof(send), 8 * n_send, C.addressof(recv), 8 * n_recv)
            out[peer] = (rc, list(recv))
        buf = (C.c_double * 5)(*[rank + 1.0 + i for i in range(5)])
        rc = ar(None, C.addressof(buf), 5)
        out["sum"] = (rc, list(buf))
        q.put(("ok", rank, out, t.errors))
        tdist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("error", rank, repr(e), []))


def test_torch_transport_callbacks_three_ranks():
    """dot_transport over gloo: every rank exchanges
    mirrored-size buffers with both neighbours and the all-reduce sums in place."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r[1]: r for r in [q.get(timeout=300) for _ in range(world)]}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        status, _, out, errors = res[rank]
        assert status == "ok" and not errors, res[rank]
        for peer in (rank - 1, rank + 1):
            if 0 <= peer < world:
                rc, got = out[peer]
                assert rc == 0
                assert got == [100.0 * peer + i for i in range(3 + peer)]
        rc, s = out["sum"]
        assert rc == 0 and s == [sum(r + 1.0 + i for r in range(world)) for i in range(5)]
