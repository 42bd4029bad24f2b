"""GPU: LOCAL transfers on the DMA copy engines (option sm_transfers = 0, one
cudaMemcpyAsync per contiguous run) give the same results as the SM copy kernels: (O, LSE)
bit-identical, gradients equal up to the order of their fp32 atomic sums. Runs on one GPU
(plan devices emulated on it) or across the GPUs present, alone and with the persistent
forward."""
import pytest

from common import MIXED_SPECS, bundle_for, inputs
from test_gpu_persistent import _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("persistent", [0, 1])
def test_dma_transfers_match_copy_kernels(persistent):
    import torch
    ngpu = torch.cuda.device_count()
    R = 4 if ngpu >= 4 or ngpu == 1 else 2
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=R, placement="zigzag")
    (q0, k0, v0), _ = inputs(bundle, seed=81)
    g = torch.Generator().manual_seed(82)
    d_o0 = torch.randn((bundle.total_tokens, bundle.H, 128), generator=g).to(torch.bfloat16)
    q, k, v, d_o = (x.cuda() for x in (q0, k0, v0, d_o0))
    _, base = _run(bundle, 0, q, k, v, d_o, ngpu)
    _, dma = _run(bundle, persistent, q, k, v, d_o, ngpu, opts={"sm_transfers": 0})
    bad = [name for name, a, b in zip(("o", "lse"), base, dma) if not torch.equal(a, b)]
    assert not bad, f"{bad} differ with DMA transfers"
    for name, a, b in zip(("dq", "dk", "dv"), base[2:], dma[2:]):
        err = ((a - b).abs().max() / a.abs().max().clamp_min(1e-30)).item()
        assert err < 1e-2, f"{name} max rel diff {err:.2e}"
