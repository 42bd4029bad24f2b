"""One rank of the per-rank (one process per GPU) executor, launched by torchrun from
tests/test_gpu_rank.py. Rank r executes plan device r of the MIXED_SPECS plan on GPU
r % device_count (several ranks may share a GPU: CUDA IPC works within one device too),
with the packed single-buffer I/O, for `--iters` load/forward/backward calls, and saves
the rows it wrote (O, LSE, dQ, dK, dV; float32) of the first and last call to --out."""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--placement", default="dcp")
    ap.add_argument("--host", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="executor option key=value")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from common import MIXED_SPECS, bundle_for, inputs
    from paper_2510_10620_b200.executor import DCPExecutor

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", init_method="env://")
    ordinal = rank % torch.cuda.device_count()
    torch.cuda.set_device(ordinal)
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=world, placement=args.placement)
    (q, k, v), _ = inputs(bundle, seed=21)
    g = torch.Generator().manual_seed(22)
    T = bundle.total_tokens
    d_o = torch.randn((T, 4, 128), generator=g).to(torch.bfloat16)
    dev = f"cuda:{ordinal}"
    q, k, v, d_o = (x.to(dev) for x in (q, k, v, d_o))
    ex = DCPExecutor(rank=rank, world=world, cuda_ordinal=ordinal)
    for kv in args.opt:
        key, val = kv.split("=")
        ex.set_option(key, int(val))
    ex.prepare(bundle)
    outs = []
    for it in range(args.iters):
        # the last call goes through the host I/O path (pinned buffers; this rank uploads and
        # downloads only the token rows of its plan device)
        host = args.host and it == args.iters - 1
        where = "cpu" if host else dev
        mk = (lambda x: torch.zeros(x.shape, dtype=x.dtype).pin_memory()) if host else torch.zeros_like
        o = mk(torch.empty((T, 4, 128), dtype=torch.bfloat16, device=where))
        lse = mk(torch.empty((4, T), device=where))
        dq, dk, dv = mk(q), mk(k), mk(v)
        src = [x.cpu().pin_memory() for x in (q, k, v, d_o)] if host else (q, k, v, d_o)
        ex.load_inputs(*src[:3])
        rep = ex.forward(o, lse, host=host)
        ex.backward(src[3], dq, dk, dv, host=host)
        ex.synchronize()
        outs.append((o, lse, dq, dk, dv, rep))
    for tag, (o, lse, dq, dk, dv, rep) in (("first", outs[0]), ("last", outs[-1])):
        np.savez(os.path.join(args.out, f"rank{rank}_{tag}.npz"), o=o.float().cpu().numpy(),
                 lse=lse.cpu().numpy(), dq=dq.float().cpu().numpy(), dk=dk.float().cpu().numpy(),
                 dv=dv.float().cpu().numpy(), total_bytes=rep["total_bytes"])
    dist.barrier()  # no rank unmaps / frees while a peer may still read its arenas
    ex.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
