"""CPU, world_size 2 (gloo): the per-rank view of a multi-device plan.

Each rank takes only its own device's ExecutionPlan (what a one-process-per-GPU transport
holds) and the ranks cross-check over gloo collectives what such a transport relies on:
every send tag has a matching posted receive with the same byte count on the peer
(inc/simexec.hpp:263-327 pairs them by tag), each rank's bytes equal the planner's
CommVolume (inc/placement.hpp:180-243), every receive is waited on, and the per-rank FLOPs
add up to BlockGraph::total_flops (inc/blocks.hpp:191)."""
import os
import socket
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _messages(bundle, rank):
    dp = bundle.devices[rank]
    sizes = bundle.data_blocks["size_bytes"]
    sends, recvs, waits = {}, {}, set()
    for ins in dp.instructions():
        if ins["op"] == 3:
            blocks = dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]
            nbytes = int(sum(int(sizes[b["block"]]) for b in blocks))
            (sends if ins["send"] else recvs)[ins["tag"]] = (int(ins["peer"]), nbytes)
        elif ins["op"] == 4:
            waits.add(ins["tag"])
    return sends, recvs, waits


def _worker(rank, world, port, name, q):
    try:
        import torch.distributed as dist
        sys.path.insert(0, REPO)
        sys.path.insert(0, os.path.join(REPO, "tools"))
        from make_plans import load
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        bundle = load(name)
        assert bundle.R == world
        sends, recvs, waits = _messages(bundle, rank)
        # per-rank bytes == the planner's CommVolume for this device, bit-exact
        assert sum(b for _, b in sends.values()) == int(bundle.per_device_send[rank])
        assert sum(b for _, b in recvs.values()) == int(bundle.per_device_recv[rank])
        assert set(recvs) <= waits, "a posted receive is never waited on"
        everyone = [None] * world
        dist.all_gather_object(everyone, (sends, recvs))
        for tag, (peer, nbytes) in recvs.items():
            psends = everyone[peer][0]
            assert tag in psends and psends[tag] == (rank, nbytes), f"unmatched receive {tag}"
        for tag, (peer, nbytes) in sends.items():
            assert everyone[peer][1].get(tag) == (rank, nbytes), f"unmatched send {tag}"
        import torch
        flops = torch.tensor([int(bundle.dev_flops[rank])], dtype=torch.int64)
        dist.all_reduce(flops)
        assert int(flops.item()) == int(bundle.total_flops)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"{type(e).__name__}: {e}"))


@pytest.mark.parametrize("name", ["cfg1_R2", "cfg2_R2", "cfg3_R2"])
def test_per_rank_plans_exchange_consistently(name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {0: "ok", 1: "ok"}, results
