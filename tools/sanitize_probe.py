"""Small forward + backward through the C ABI, for protocol checks of the kernels' barriers:
    python tools/sanitize_probe.py [--out outputs.npz]     (DCPX_LIB selects the build)
A 2-device DCP plan of mixed masks (both plan devices on cuda:0: transfers, merges, returns),
a block-128 plan with ragged tails and config 1 (16K tokens, 2 devices); every output is
checked against the FP64 oracle, and --out saves them so tests/test_gpu_jitter.py can compare
the race-detection build (random delays after every barrier wait, -DDCPX_JITTER) with the
product build bit for bit. (compute-sanitizer racecheck / synccheck were the first choice;
that tool is closed on the GPU pool: profiles/r2_race_checks.md.)"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    import numpy as np
    import torch

    import oracle as O
    from common import MIXED_SPECS, bundle_for, inputs, rel_err
    from paper_2510_10620_b200 import planner as PL
    from paper_2510_10620_b200.executor import DCPExecutor
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(REPO, "tools"))
    from make_plans import load
    cases = [bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=2),
             bundle_for([PL.SeqSpec(300), PL.SeqSpec(77, "lambda", sink=5, window=20)], H=2, G=1, block=128, R=2),
             load("cfg1_R2")]
    saved = {}
    for i, bundle in enumerate(cases):
        (q, k, v), (q64, k64, v64) = inputs(bundle, seed=3 + i)
        T, H, G = bundle.total_tokens, bundle.H, bundle.G
        g = torch.Generator().manual_seed(9)
        d_o = torch.randn((T, H, 128), generator=g).to(torch.bfloat16)
        with DCPExecutor([0] * bundle.R) as ex:
            ex.prepare(bundle)
            o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
            lse = torch.zeros((H, T), device="cuda")
            dq = torch.zeros_like(o)
            dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
            dv = torch.zeros_like(dk)
            for _ in range(2):
                ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
                ex.forward(o, lse)
                ex.backward(d_o.cuda(), dq, dk, dv)
            ex.synchronize()
        o_ref, _, _, st, msg = O.run(bundle, q64, k64, v64)
        rq, rk, rv = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
        errs = [rel_err(o.float().cpu().numpy(), o_ref), rel_err(dq.float().cpu().numpy(), rq),
                rel_err(dk.float().cpu().numpy(), rk), rel_err(dv.float().cpu().numpy(), rv)]
        print(f"case {i}: R={bundle.R} tokens={T} rel errs o/dq/dk/dv", " ".join(f"{e:.2e}" for e in errs))
        assert st == 0 and max(errs) <= 2e-2
        for name, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
            saved[f"{i}_{name}"] = t.float().cpu().numpy()
    if args.out:
        np.savez(args.out, **saved)
    print("SANITIZE PROBE OK")


if __name__ == "__main__":
    main()
