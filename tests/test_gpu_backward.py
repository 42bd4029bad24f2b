"""GPU parity of the backward executor (K1b + fetch/return exchange) against the dense
FP64 backward restatement (oracle/dcp_oracle.c:orc_dense_backward) on the same bf16
inputs. Tolerance (north_star): max relative error <= 2e-2 on dQ, dK, dV."""
import numpy as np
import pytest

import oracle as O
from paper_2510_10620_b200 import planner as PL
from paper_2510_10620_b200.executor import DCPExecutor

from common import MIXED_SPECS, O_TOL, bundle_for, inputs, rel_err

pytestmark = pytest.mark.gpu


def _fwd_bwd(bundle, q, k, v, d_o):
    import torch
    ex = DCPExecutor([0] * bundle.R)
    ex.prepare(bundle)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((H, T), device="cuda")
    dq = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
    dv = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
    ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
    ex.forward(o, lse)
    rep = ex.backward(d_o.cuda(), dq, dk, dv)
    ex.synchronize()
    ex.close()
    return [t.float().cpu().numpy() for t in (o, dq, dk, dv)], rep


def _d_o(bundle, seed):
    import torch
    g = torch.Generator().manual_seed(1000 + seed)
    return torch.randn((bundle.total_tokens, bundle.H, 128), generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("R", [1, 2, 4])
def test_backward_mixed_masks_vs_dense(R):
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=R)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=R)
    d_o = _d_o(bundle, R)
    (o, dq, dk, dv), rep = _fwd_bwd(bundle, q, k, v, d_o)
    rq, rk, rv = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
    assert rel_err(dq, rq) <= O_TOL
    assert rel_err(dk, rk) <= O_TOL
    assert rel_err(dv, rv) <= O_TOL
    assert rep["total_flops"] == bundle.total_flops // 2 * 5
    send, recv = bundle.bwd_bytes()
    assert rep["per_device_send"] == [int(x) for x in send]
    assert rep["per_device_recv"] == [int(x) for x in recv]


@pytest.mark.parametrize("block", [128, 512])
def test_backward_ragged_and_gqa(block):
    specs = [PL.SeqSpec(1000), PL.SeqSpec(77, "lambda", sink=5, window=20), PL.SeqSpec(1),
             PL.SeqSpec(513, "shared_question", question_len=100, answer_lens=[200, 213])]
    bundle = bundle_for(specs, H=4, G=1, block=block, R=2)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=block)
    d_o = _d_o(bundle, block)
    (o, dq, dk, dv), _ = _fwd_bwd(bundle, q, k, v, d_o)
    rq, rk, rv = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
    assert rel_err(dq, rq) <= O_TOL
    assert rel_err(dk, rk) <= O_TOL
    assert rel_err(dv, rv) <= O_TOL


def test_backward_fuzz_random_batches():
    for seed in range(5):
        b = PL.Batch.random(100 + seed, max_seq_len=600, max_seqs=3, max_heads=2, head_dim=128)
        R = 1 + seed % 3
        try:
            bundle = PL.plan(b, R, 128, eps_intra=0.5, eps_data=0.6, eps_inter=0.5, seed=seed)
        except PL.PlannerError as e:
            if e.kind == "InfeasibleError":
                continue
            raise
        (q, k, v), (q64, k64, v64) = inputs(bundle, seed=seed)
        d_o = _d_o(bundle, seed)
        (o, dq, dk, dv), _ = _fwd_bwd(bundle, q, k, v, d_o)
        rq, rk, rv = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
        assert rel_err(dq, rq) <= O_TOL, seed
        assert rel_err(dk, rk) <= O_TOL, seed
        assert rel_err(dv, rv) <= O_TOL, seed


def test_async_host_io_double_buffered():
    """dcpx_load_inputs_host / dcpx_backward_host are asynchronous with two alternating
    staging slots: three back-to-back steps with different (pinned) inputs, synchronised
    once at the end, each equal the device-buffer path on the same inputs."""
    import torch

    from paper_2510_10620_b200.executor import DCPExecutor
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=2)
    T = bundle.total_tokens
    ex = DCPExecutor([0, 0])
    ex.prepare(bundle)
    steps = []
    for s in range(3):
        (q, k, v), _ = inputs(bundle, seed=40 + s)
        g = torch.Generator().manual_seed(50 + s)
        d_o = torch.randn((T, 4, 128), generator=g).to(torch.bfloat16)
        pin = lambda x: x.contiguous().pin_memory()  # noqa: E731
        host = dict(q=pin(q), k=pin(k), v=pin(v), d_o=pin(d_o),
                    dq=torch.zeros((T, 4, 128), dtype=torch.bfloat16).pin_memory(),
                    dk=torch.zeros((T, 2, 128), dtype=torch.bfloat16).pin_memory(),
                    dv=torch.zeros((T, 2, 128), dtype=torch.bfloat16).pin_memory())
        steps.append(host)
    o = torch.zeros((T, 4, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((4, T), device="cuda")
    ex.set_option("timing", 0)
    for h in steps:
        ex.load_inputs(h["q"], h["k"], h["v"])
        ex.forward(o, lse)
        ex.backward(h["d_o"], h["dq"], h["dk"], h["dv"], host=True)
    ex.synchronize()
    for h in steps:
        dq = torch.zeros((T, 4, 128), dtype=torch.bfloat16, device="cuda")
        dk = torch.zeros((T, 2, 128), dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        ex.load_inputs(h["q"].cuda(), h["k"].cuda(), h["v"].cuda())
        ex.forward(o, lse)
        ex.backward(h["d_o"].cuda(), dq, dk, dv)
        ex.synchronize()
        for a, b in ((h["dq"], dq), (h["dk"], dk), (h["dv"], dv)):
            assert rel_err(a.float().numpy(), b.float().cpu().numpy()) <= 4e-3
    ex.close()


@pytest.mark.parametrize("H,G,block", [(2, 2, 200), (3, 1, 96), (8, 8, 160)])
def test_forward_backward_unusual_shapes(H, G, block):
    """Plain multi-head (H = G) and multi-query (G = 1, odd H) attention, block sizes that are
    not multiples of the 128-row tiles (slots padded to 128 rows): forward and backward
    against the FP64 oracle, backward bytes equal to the builder's formula."""
    specs = [PL.SeqSpec(611), PL.SeqSpec(300, "lambda", sink=17, window=90),
             PL.SeqSpec(450, "causal_blockwise", block=50, window_blocks=2, sink_blocks=1, test_blocks=1)]
    bundle = bundle_for(specs, H=H, G=G, block=block, R=2)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=block)
    d_o = _d_o(bundle, block)
    (o, dq, dk, dv), rep = _fwd_bwd(bundle, q, k, v, d_o)
    o_ref, lse_ref, orep, st, msg = O.run(bundle, q64, k64, v64)
    assert st == 0, msg
    assert rel_err(o, o_ref) <= O_TOL
    rq, rk, rv = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
    assert rel_err(dq, rq) <= O_TOL
    assert rel_err(dk, rk) <= O_TOL
    assert rel_err(dv, rv) <= O_TOL
    send, recv = bundle.bwd_bytes()
    assert rep["per_device_send"] == [int(x) for x in send]
