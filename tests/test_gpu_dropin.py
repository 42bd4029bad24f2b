"""GPU: the reference's executor tests run through the C++ drop-in dcp::gpu::run
(include/dcp_gpu.hpp) — same signature as dcp::run (simexec.hpp:207)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_dcp_gpu_run")


def test_dropin_reference_suite():
    assert os.path.exists(BIN), "drop-in test binary not built (tools/build.py)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr


def test_lookahead_pipeline_with_gpu_consumer():
    """dcp::gpu::pipeline_run (include/dcp_gpu_pipeline.hpp) vs the
    reference's pipeline_run (pipeline.hpp:105) on the same batches: identical reports,
    look-ahead protocol respected (tests/cpp/test_gpu_pipeline.cpp)."""
    binp = os.path.join(os.path.dirname(BIN), "test_gpu_pipeline")
    assert os.path.exists(binp), "pipeline test binary not built (tools/build.py)"
    r = subprocess.run([binp], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0 and "OK (0 failures)" in r.stdout, r.stdout + r.stderr


def test_plan_from_reference_json_files_on_gpu():
    """a plan read from the reference's own plan files (planio) runs on the
    GPU exactly like the same plan coming from the planner shim."""
    import os

    import numpy as np
    import torch

    from common import O_TOL, LSE_TOL, inputs, lse_err, rel_err
    import oracle as O
    from paper_2510_10620_b200 import planio
    from paper_2510_10620_b200.executor import DCPExecutor
    from paper_2510_10620_b200.plans import PlanBundle
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plan_json")
    jb = planio.load_reference_plan(gold)
    pb = PlanBundle.load(os.path.join(gold, "bundle.npz"))
    (q, k, v), (q64, k64, v64) = inputs(pb, seed=21)
    T = pb.total_tokens
    g = torch.Generator().manual_seed(4)
    d_o = torch.randn((T, pb.H, 128), generator=g).to(torch.bfloat16).cuda()
    outs = []
    for bundle in (pb, jb):
        ex = DCPExecutor([0] * bundle.R)
        ex.prepare(bundle)
        o = torch.zeros((T, bundle.H, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.zeros((bundle.H, T), device="cuda")
        dq = torch.zeros_like(o)
        dk = torch.zeros((T, bundle.G, 128), dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
        rep = ex.forward(o, lse)
        ex.backward(d_o, dq, dk, dv)
        ex.synchronize()
        outs.append((o.float().cpu(), lse.cpu(), dq.float().cpu(), dk.float().cpu(), dv.float().cpu(),
                     rep["total_bytes"]))
        ex.close()
    (o1, l1, dq1, dk1, dv1, b1), (o2, l2, dq2, dk2, dv2, b2) = outs
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for a, b in ((dq1, dq2), (dk1, dk2), (dv1, dv2)):
        assert rel_err(a.numpy(), b.numpy()) <= 4e-3
    assert b1 == b2 == int(pb.volume[0])
    o_ref, lse_ref, _, st, msg = O.run(jb, q64, k64, v64)
    assert st == 0, msg
    assert rel_err(o2.numpy(), o_ref) <= O_TOL
    assert lse_err(l2.numpy(), lse_ref) <= LSE_TOL
