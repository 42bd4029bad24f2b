"""GPU parity of the production backward unit path against the dense FP64 backward
(oracle/dcp_oracle.c:orc_dense_backward, the gradient of exec_attention, simexec.hpp:33-76).

Every BASELINE config runs K1b with q-windowed units that span all heads of a GQA group
(compile.cu, executor.h Options: bwd_window, bwd_order, bwd_merge_heads), switched on by
bwd_window_min_steps. The small plans here have short units, so the threshold is forced to
0 to reach that path, and each combination of window width (including windows that do not
divide the 16 q tiles of a 1024-row block, and single-tile windows), unit order and head
merging is compared with the oracle. The report's `windowed` count proves the path ran.
Tolerance (north_star): max |x - ref| / max |ref| <= 2e-2 on dQ, dK, dV."""
import numpy as np
import pytest

import oracle as O
from paper_2510_10620_b200 import planner as PL
from paper_2510_10620_b200.executor import DCPExecutor

from common import O_TOL, inputs, rel_err

pytestmark = pytest.mark.gpu

# one 1024-row block holds 16 backward q tiles of 64 rows; GQA 8 q / 2 kv heads (4 heads per
# group, as in the 8B config); causal, lambda (window edges inside a block) and
# shared-question (rows with no keys in some kv tiles); 2 plan devices (fetches + returns)
SPECS = [PL.SeqSpec(2600), PL.SeqSpec(2100, "lambda", sink=64, window=700),
         PL.SeqSpec(1900, "shared_question", question_len=500, answer_lens=[600, 800])]


@pytest.fixture(scope="module")
def case():
    import torch
    b = PL.Batch.from_specs(SPECS, 8, 2, 128)
    bundle = PL.plan(b, 2, 1024, eps_intra=0.05, eps_data=0.2)  # both devices send (fetches + returns)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=31)
    g = torch.Generator().manual_seed(32)
    d_o = torch.randn((bundle.total_tokens, bundle.H, 128), generator=g).to(torch.bfloat16)
    ref = O.dense_backward(bundle, q64, k64, v64, d_o.double().numpy())
    return bundle, (q, k, v, d_o), ref


def _grads(bundle, q, k, v, d_o, opts):
    import torch
    ex = DCPExecutor([0] * bundle.R)
    for key, val in opts.items():
        ex.set_option(key, val)
    ex.prepare(bundle)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((H, T), device="cuda")
    dq = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
    dv = torch.zeros_like(dk)
    ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
    ex.forward(o, lse)
    rep = ex.backward(d_o.cuda(), dq, dk, dv)
    ex.synchronize()
    ex.close()
    return [t.float().cpu().numpy() for t in (dq, dk, dv)], rep


@pytest.mark.parametrize("window", [1, 3, 12, 16])
@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("merge", [0, 1])
def test_windowed_units_vs_dense(case, window, order, merge):
    bundle, (q, k, v, d_o), (rq, rk, rv) = case
    opts = dict(bwd_window_min_steps=0, bwd_window=window, bwd_order=order, bwd_merge_heads=merge)
    (dq, dk, dv), rep = _grads(bundle, q, k, v, d_o, opts)
    assert rep["windowed"] > 0  # the windowed path ran
    assert rel_err(dq, rq) <= O_TOL, (window, order, merge)
    assert rel_err(dk, rk) <= O_TOL, (window, order, merge)
    assert rel_err(dv, rv) <= O_TOL, (window, order, merge)


def test_unit_count_follows_windows(case):
    """Narrower windows split units: window 1 gives more units than window 16, and whole-item
    units (threshold not reached) give the fewest; the gradients agree across all three."""
    bundle, (q, k, v, d_o), (rq, rk, rv) = case
    runs = {}
    for name, opts in {"w1": dict(bwd_window_min_steps=0, bwd_window=1),
                       "w16": dict(bwd_window_min_steps=0, bwd_window=16),
                       "whole": dict(bwd_window_min_steps=1 << 30)}.items():
        runs[name] = _grads(bundle, q, k, v, d_o, opts)
    assert runs["w1"][1]["units"] > runs["w16"][1]["units"] >= runs["whole"][1]["units"]
    assert runs["whole"][1]["windowed"] == 0
    for name, ((dq, dk, dv), _) in runs.items():
        assert rel_err(dq, rq) <= O_TOL, name
        assert rel_err(dk, rk) <= O_TOL, name
        assert rel_err(dv, rv) <= O_TOL, name


def test_backward_wire_bytes(case):
    """dcpx_report wire bytes: what the transfers actually move (fp32 sidecars and fp32
    gradient returns), equal to the formula in plans.PlanBundle.wire_bytes; planned bytes
    stay the builder's backward formula."""
    import torch
    bundle, (q, k, v, d_o), _ = case
    ex = DCPExecutor([0] * bundle.R)
    ex.prepare(bundle)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((H, T), device="cuda")
    ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
    rf = ex.forward(o, lse)
    dq = torch.zeros_like(o)
    dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
    rb = ex.backward(d_o.cuda(), dq, dk, torch.zeros_like(dk))
    ex.synchronize()
    ex.close()
    (fs, fr), (bs, br) = bundle.wire_bytes()
    assert rf["wire_per_device_send"] == [int(x) for x in fs]
    assert rf["wire_per_device_recv"] == [int(x) for x in fr]
    assert rb["wire_per_device_send"] == [int(x) for x in bs]
    assert rb["wire_per_device_recv"] == [int(x) for x in br]
    assert rf["wire_bytes"] == int(fs.sum()) > rf["total_bytes"] == int(bundle.volume[0])
    send, _ = bundle.bwd_bytes()
    assert rb["wire_bytes"] == int(bs.sum()) > rb["total_bytes"] == int(send.sum())
