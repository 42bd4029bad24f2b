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
    ex.prepare(bundle)
    outs = []
    for it in range(args.iters):
        o = torch.zeros((T, 4, 128), dtype=torch.bfloat16, device=dev)
        lse = torch.zeros((4, T), device=dev)
        dq, dk, dv = torch.zeros_like(q), torch.zeros_like(k), torch.zeros_like(v)
        ex.load_inputs(q, k, v)
        rep = ex.forward(o, lse)
        ex.backward(d_o, dq, dk, dv)
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
