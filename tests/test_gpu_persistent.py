"""GPU: the persistent cross-division forward (executor option "persistent", off by default;
DESIGN.md section 4.3). One launch per device runs every division's forward units, ordered on
the device by transfer / unit-completion counters instead of launch boundaries. Its (O, LSE)
must be bit-identical to the per-division launches (same units, same per-unit arithmetic),
and the option must actually engage (fewer kernel launches) on a plan it is eligible for.
Needs two or more GPUs: devices sharing a GPU keep per-division launches."""
import pytest

from paper_2510_10620_b200.executor import DCPExecutor

from common import MIXED_SPECS, bundle_for, inputs

pytestmark = pytest.mark.gpu


def _run(bundle, persistent, q, k, v, d_o, ngpu, iters=2, opts=None):
    import torch
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    with DCPExecutor([d % ngpu for d in range(bundle.R)]) as ex:
        ex.set_option("persistent", persistent)
        for key, val in (opts or {}).items():
            ex.set_option(key, val)
        ex.prepare(bundle)
        o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.zeros((H, T), device="cuda")
        dq = torch.zeros_like(o)
        dk = torch.zeros((T, G, 128), dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        for _ in range(iters):  # the second pass reuses the counters (epoch stamps, re-zeroing)
            ex.load_inputs(q, k, v)
            rf = ex.forward(o, lse)
            ex.backward(d_o, dq, dk, dv)
        ex.synchronize()
        torch.cuda.synchronize()
        return rf["kernel_launches"], [t.float().cpu() for t in (o, lse, dq, dk, dv)]


@pytest.mark.parametrize("placement", ["zigzag", "dcp"])
def test_persistent_forward_bit_identical(placement):
    import torch
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("the persistent forward needs one GPU per plan device")
    R = 4 if ngpu >= 4 else 2
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=R, placement=placement)
    (q0, k0, v0), _ = inputs(bundle, seed=71)
    g = torch.Generator().manual_seed(72)
    d_o0 = torch.randn((bundle.total_tokens, bundle.H, 128), generator=g).to(torch.bfloat16)
    q, k, v, d_o = (x.cuda() for x in (q0, k0, v0, d_o0))
    n0, base = _run(bundle, 0, q, k, v, d_o, ngpu)
    n1, pers = _run(bundle, 1, q, k, v, d_o, ngpu)
    bad = [name for name, a, b in zip(("o", "lse"), base, pers) if not torch.equal(a, b)]
    assert not bad, f"{placement}: {bad} differ with the persistent forward"
    # the gradients accumulate in fp32 with order-dependent atomics (not bit-reproducible run
    # to run, with or without this option): same values up to bf16 rounding of the sums
    for name, a, b in zip(("dq", "dk", "dv"), base[2:], pers[2:]):
        err = ((a - b).abs().max() / a.abs().max().clamp_min(1e-30)).item()
        assert err < 1e-2, f"{placement}: {name} max rel diff {err:.2e}"
    if placement == "zigzag":
        assert n1 < n0, f"persistent forward did not engage ({n1} vs {n0} launches)"
