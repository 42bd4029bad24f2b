"""GPU parity of the forward executor (K1 fused attention + K2 merge + transfers)
against the CPU oracle on the same bf16 inputs, through the C ABI."""
import numpy as np
import pytest

import oracle as O
from paper_2510_10620_b200 import planner as PL
from paper_2510_10620_b200.executor import DCPExecutor, DCPXError

from common import (LSE_TOL, MIXED_SPECS, O_TOL, bundle_for, dense_rows_forward, inputs, lse_err,
                    rel_err, sampled_rows)

pytestmark = pytest.mark.gpu


def _run_gpu(bundle, q, k, v, fuse=True, remap=True):
    import torch
    ex = DCPExecutor([0] * bundle.R)
    ex.set_option("fuse_reductions", int(fuse))
    ex.set_option("remap_copies", int(remap))
    ex.prepare(bundle)
    T, H = bundle.total_tokens, bundle.H
    o = torch.zeros((T, H, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((H, T), float("-inf"), device="cuda")
    ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
    rep = ex.forward(o, lse)
    ex.synchronize()
    ex.close()
    return o.float().cpu().numpy(), lse.cpu().numpy(), rep


@pytest.mark.parametrize("R", [1, 2, 4])
@pytest.mark.parametrize("fuse", [True, False])
def test_forward_mixed_masks_vs_oracle(R, fuse):
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=R)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=R)
    o, lse, rep = _run_gpu(bundle, q, k, v, fuse=fuse, remap=fuse)
    o_ref, lse_ref, orep, st, msg = O.run(bundle, q64, k64, v64)
    assert st == 0, msg
    assert rel_err(o, o_ref) <= O_TOL
    assert lse_err(lse, lse_ref) <= LSE_TOL
    # planned bytes are bit-exact with the reference's CommVolume (placement.hpp:180-243)
    assert rep["total_bytes"] == int(bundle.volume[0]) == orep.total_bytes
    assert rep["per_device_send"] == [int(x) for x in bundle.per_device_send]
    assert rep["per_device_recv"] == [int(x) for x in bundle.per_device_recv]
    assert rep["total_flops"] == orep.total_flops == bundle.total_flops


@pytest.mark.parametrize("block", [128, 512])
def test_forward_block_sizes_and_ragged_tails(block):
    specs = [PL.SeqSpec(1000), PL.SeqSpec(77, "lambda", sink=5, window=20), PL.SeqSpec(1),
             PL.SeqSpec(513, "shared_question", question_len=100, answer_lens=[200, 213])]
    bundle = bundle_for(specs, H=2, G=1, block=block, R=2)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=block)
    o, lse, rep = _run_gpu(bundle, q, k, v)
    o_ref, lse_ref, _, st, msg = O.run(bundle, q64, k64, v64)
    assert st == 0, msg
    assert rel_err(o, o_ref) <= O_TOL
    assert lse_err(lse, lse_ref) <= LSE_TOL


def test_forward_empty_rows_shared_question():
    # answer-2 rows vs answer-1 kv tiles are fully masked inside non-empty items
    specs = [PL.SeqSpec(1024, "shared_question", question_len=128, answer_lens=[300, 300, 296])]
    bundle = bundle_for(specs, H=2, G=2, block=256, R=4, eps_intra=0.6)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=5)
    o, lse, _ = _run_gpu(bundle, q, k, v)
    assert np.isfinite(o).all()
    o_ref, lse_ref, _, st, msg = O.run(bundle, q64, k64, v64)
    assert rel_err(o, o_ref) <= O_TOL
    assert lse_err(lse, lse_ref) <= LSE_TOL


def test_forward_fuzz_random_batches():
    for seed in range(6):
        b = PL.Batch.random(seed, max_seq_len=700, max_seqs=3, max_heads=2, head_dim=128)
        R = 1 + seed % 3
        try:
            bundle = PL.plan(b, R, 128, eps_intra=0.5, eps_data=0.6, eps_inter=0.5, seed=seed)
        except PL.PlannerError as e:
            if e.kind == "InfeasibleError":
                continue
            raise
        (q, k, v), (q64, k64, v64) = inputs(bundle, seed=seed)
        o, lse, rep = _run_gpu(bundle, q, k, v)
        o_ref, lse_ref, orep, st, msg = O.run(bundle, q64, k64, v64)
        assert st == 0, msg
        assert rel_err(o, o_ref) <= O_TOL, seed
        assert lse_err(lse, lse_ref) <= LSE_TOL, seed
        assert rep["total_bytes"] == orep.total_bytes


def test_forward_large_block_sampled_rows():
    # config-1 shape (16K tokens, 8/2 heads, block 1024, 2 devices), checked on sampled rows
    specs = [PL.SeqSpec(8192), PL.SeqSpec(4096), PL.SeqSpec(2048), PL.SeqSpec(2048)]
    bundle = bundle_for(specs, H=8, G=2, block=1024, R=2, eps_intra=0.1, eps_data=0.05)
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=11)
    o, lse, rep = _run_gpu(bundle, q, k, v)
    toks, heads = sampled_rows(bundle, 256, seed=1)
    o_ref, lse_ref = dense_rows_forward(bundle, q64, k64, v64, toks, heads)
    assert rel_err(o[toks, heads], o_ref) <= O_TOL
    assert lse_err(lse[heads, toks], lse_ref) <= LSE_TOL
    assert rep["total_bytes"] == 12582912  # SURVEY.md section 6 probe of config 1


def test_deadlock_missing_sender():
    # tests/test_simexec.cpp:251-270: deleting the sends is reported as a deadlock
    specs = [PL.SeqSpec(256)]
    b = PL.Batch.from_specs(specs, 1, 1, 128)
    gt, cq = b.graph_counts(128)
    bundle = PL.plan(b, 2, 128, placement="explicit", group_dev=gt, comp_dev=cq, divisions=2)
    dp = bundle.devices[0]
    keep = [i for i, r in enumerate(dp.instr) if not (r[0] == 3 and r[2] == 1)]
    dp.instr = dp.instr[keep]
    ex = DCPExecutor([0, 0])
    with pytest.raises(DCPXError) as ei:
        ex.prepare(bundle)
    assert ei.value.kind == "DeadlockError"


def test_reduction_with_many_partials():
    """ReductionInstr with more partials than a merge kernel would hold per thread (here 132,
    simexec.hpp:80-111 takes any number): 132 kv tiles of block 64, unfused merge path."""
    bundle = bundle_for([PL.SeqSpec(8448)], H=1, G=1, block=64, R=1, divisions=2)
    nsrc = max(int(r[5]) for r in bundle.devices[0].instr if r[0] == 1)
    assert nsrc > 64
    (q, k, v), (q64, k64, v64) = inputs(bundle, seed=13)
    o, lse, rep = _run_gpu(bundle, q, k, v, fuse=False, remap=False)
    o_ref, lse_ref, orep, st, msg = O.run(bundle, q64, k64, v64)
    assert st == 0, msg
    assert rel_err(o, o_ref) <= O_TOL
    assert lse_err(lse, lse_ref) <= LSE_TOL
