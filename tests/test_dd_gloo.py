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
