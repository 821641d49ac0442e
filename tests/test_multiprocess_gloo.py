"""N > 1 host logic on CPU: world_size-2/4 `gloo` process groups (one process per stage,
as `bench.py --gpus N` runs under torch.distributed.run).

Each rank walks ITS OWN static order from libtps (`tps_schedule_events`, host-only) and
performs the exchanges the GPU path performs with NCCL, as gloo isend / blocking recv (a blocking send would deadlock
exactly like a single-stream design: stage s's forward send and stage s+1's backward send
wait on each other; the GPU path avoids it with one stream + communicator per direction):
activations forward per forward group (s -> s+1) and activation-gradients backward once
per mini-batch (s+1 -> s).  Messages carry (mb, group, sender's version) so the test
checks that (1) the independently generated orders pair every send with the matching
receive in the same order, without deadlock, and (2) the per-stage versions and δ each
rank derives locally equal the oracle's closed forms.  It also
exercises the bench's rendezvous helpers: ncclUniqueId broadcast and max-over-ranks.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, g, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_23241_b200 import tps
        S, s = world, rank
        order = tps.schedule_events(S, s, m, g, M)
        version = 0
        pending = []          # sends are asynchronous, like the GPU's per-direction comm streams
        fwd_ver = {}
        deltas = {}
        for e in order:
            if e.kind == tps.TPS_EV_F:
                grp = e.micro // g
                if s > 0:
                    t = torch.zeros(3, dtype=torch.int64)
                    dist.recv(t, src=s - 1, tag=1)
                    assert (t[0].item(), t[1].item()) == (e.mb, grp), (s, t.tolist(), e.mb, grp)
                fwd_ver.setdefault(e.mb, version)
                if s < S - 1:
                    pending.append(dist.isend(torch.tensor([e.mb, grp, version]), dst=s + 1, tag=1))
            elif e.kind == tps.TPS_EV_B:
                if s < S - 1:
                    t = torch.zeros(2, dtype=torch.int64)
                    dist.recv(t, src=s + 1, tag=2)
                    assert t[0].item() == e.mb
                deltas[e.mb] = version - fwd_ver[e.mb]
                if s > 0:
                    pending.append(dist.isend(torch.tensor([e.mb, version]), dst=s - 1, tag=2))
            else:
                version += 1
        for r in pending:
            r.wait()
        # closed forms (pinned by tests/golden against the paper)
        for j in range(M):
            assert fwd_ver[j] == max(0, j - S + s + 1)
            assert deltas[j] == min(j, S - 1 - s)
        # bench rendezvous helpers
        obj = [b"".join(tps.nccl_unique_id() for _ in range(2 * (S - 1)))] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        assert len(obj[0]) == 128 * 2 * (S - 1)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,g,M", [(2, 4, 2, 7), (2, 1, 1, 3), (4, 2, 1, 9), (4, 8, 4, 6)])
def test_stage_processes_exchange_in_static_order(world, m, g, M):
    try:
        from paper_2509_23241_b200 import tps
        tps.nccl_unique_id()
    except Exception as ex:  # pragma: no cover
        pytest.skip(f"NCCL unique id unavailable here: {ex}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, g, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
