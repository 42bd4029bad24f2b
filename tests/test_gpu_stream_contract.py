"""GPU: the stream contract of the C ABI (dcpx.h). Inputs produced on the
caller's stream right before the call (behind a long sleep kernel, so a call that did not
wait for that stream would read stale buffers), and outputs consumed on the same stream
right after it without any host synchronisation, give the same results as a fully
synchronised run -- on a non-default torch stream (passed through dcpx_set_streams) and on
the default stream."""
import numpy as np
import pytest

from paper_2510_10620_b200.executor import DCPExecutor

from common import MIXED_SPECS, bundle_for, inputs

pytestmark = pytest.mark.gpu


def _reference(bundle, q, k, v, d_o):
    import torch
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    with DCPExecutor([0] * bundle.R) as ex:
        ex.prepare(bundle)
        o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.zeros((H, T), device="cuda")
        dq = torch.zeros_like(o)
        dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        ex.load_inputs(q, k, v)
        ex.forward(o, lse)
        ex.backward(d_o, dq, dk, dv)
        ex.synchronize()
        torch.cuda.synchronize()
        return [t.float().cpu().numpy() for t in (o, lse, dq, dk, dv)]


@pytest.mark.parametrize("side_stream", [True, False])
def test_inputs_and_outputs_ordered_by_caller_stream(side_stream):
    import torch
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=2)
    (q0, k0, v0), _ = inputs(bundle, seed=61)
    g = torch.Generator().manual_seed(62)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    d_o0 = torch.randn((T, H, 128), generator=g).to(torch.bfloat16)
    src = [x.cuda() for x in (q0, k0, v0, d_o0)]
    want = _reference(bundle, *src)
    stream = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    with DCPExecutor([0] * bundle.R) as ex:
        ex.prepare(bundle)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            q, k, v, d_o = (torch.zeros_like(x) for x in src)
            o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
            lse = torch.zeros((H, T), device="cuda")
            dq = torch.zeros_like(o)
            dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
            dv = torch.zeros_like(dk)
            torch.cuda.synchronize()
            torch.cuda._sleep(200_000_000)  # ~0.1 s on the caller's stream, then the inputs
            for dst, s in zip((q, k, v, d_o), src):
                dst.copy_(s)
            ex.load_inputs(q, k, v)
            ex.forward(o, lse)
            ex.backward(d_o, dq, dk, dv)
            # consumers on the caller's stream, no host synchronisation in between
            got = [t.float().clone() for t in (o, lse, dq, dk, dv)]
            done = torch.cuda.Event()
            done.record(stream)
        done.synchronize()
    for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), got, want):
        a = a.cpu().numpy()
        if name in ("o", "lse"):
            assert np.array_equal(a, b), name
        else:
            assert np.abs(a - b).max() <= 4e-3 * max(1.0, np.abs(b).max()), name


def test_deferred_kernel_timing():
    """Option kernel_timing = 2: the attention launches of several calls are timed without
    blocking the host and read back once by dcpx_kernel_times (then reset); option 1 puts
    the same per-call numbers in the report."""
    import torch
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=2)
    (q, k, v), _ = inputs(bundle, seed=63)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    with DCPExecutor([0] * bundle.R) as ex:
        ex.prepare(bundle)
        o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.zeros((H, T), device="cuda")
        dq = torch.zeros_like(o)
        dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        d_o = torch.randn((T, H, 128), device="cuda").to(torch.bfloat16)
        ex.set_option("kernel_timing", 1)
        ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
        rf = ex.forward(o, lse)
        rb = ex.backward(d_o, dq, dk, dv)
        assert rf["attn_launches"] > 0 and rb["attn_launches"] > 0 and rf["attn_ms_sum"] > 0
        ex.set_option("kernel_timing", 2)
        for _ in range(3):
            ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
            r2 = ex.forward(o, lse)
            ex.backward(d_o, dq, dk, dv)
        assert r2["attn_launches"] == 0  # deferred: nothing in the per-call report
        kt = ex.kernel_times()
        assert kt["fwd_launches"] == 3 * rf["attn_launches"] and kt["bwd_launches"] == 3 * rb["attn_launches"]
        assert kt["fwd_ms_sum"] > 0 and kt["bwd_ms_sum"] > 0 and kt["bwd_ms_max"] <= kt["bwd_ms_sum"]
        again = ex.kernel_times()
        assert again["fwd_launches"] == 0 and again["bwd_ms_sum"] == 0
