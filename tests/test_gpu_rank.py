"""GPU: the per-rank mode (dcpx_create_rank -- one process per plan device, peer arenas
mapped over CUDA IPC, cross-process ordering by device-side epoch flags). Each rank
writes only the rows its plan device owns; their union must equal the single-process
context's output on the same plan and inputs (O and LSE bit for bit, gradients to bf16
rounding: atomic accumulation order differs), on the first and on a repeated call (the
cross-call hazards: peers still pulling the previous call's resident blocks, zeroed
accumulators; with `host`, the last call through the host I/O path, where each rank
copies only its own token rows), and the planned bytes must be bit-exact. Ranks spread over the GPUs
present (several share a GPU on a 1-GPU box)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from common import MIXED_SPECS, bundle_for, inputs, rel_err

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _single_process(R, placement):
    import torch

    from paper_2510_10620_b200.executor import DCPExecutor
    bundle = bundle_for(MIXED_SPECS, H=4, G=2, block=256, R=R, placement=placement)
    (q, k, v), _ = inputs(bundle, seed=21)
    g = torch.Generator().manual_seed(22)
    T = bundle.total_tokens
    d_o = torch.randn((T, 4, 128), generator=g).to(torch.bfloat16).cuda()
    n = torch.cuda.device_count()
    with DCPExecutor([d % n for d in range(R)]) as ex:
        ex.prepare(bundle)
        o = torch.zeros((T, 4, 128), dtype=torch.bfloat16, device="cuda:0")
        lse = torch.zeros((4, T), device="cuda:0")
        dq = torch.zeros_like(o)
        dk = torch.zeros((T, 2, 128), dtype=torch.bfloat16, device="cuda:0")
        dv = torch.zeros_like(dk)
        ex.load_inputs(q.cuda(), k.cuda(), v.cuda())
        rep = ex.forward(o, lse)
        ex.backward(d_o, dq, dk, dv)
        ex.synchronize()
        return dict(o=o.float().cpu().numpy(), lse=lse.cpu().numpy(), dq=dq.float().cpu().numpy(),
                    dk=dk.float().cpu().numpy(), dv=dv.float().cpu().numpy()), rep, bundle


# the last case runs the persistent cross-division forward in every rank (engaged when each
# rank has its own GPU; per-division launches otherwise) against the default single process
@pytest.mark.parametrize("R,placement,host,opts", [(2, "dcp", False, ()), (4, "dcp", True, ()),
                                                   (4, "zigzag", False, ()), (8, "dcp", False, ()),
                                                   (4, "zigzag", False, ("persistent=1",))])
def test_rank_mode_matches_single_process(R, placement, host, opts, tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "rank_worker.py"), "--out", str(tmp_path), "--iters", "3",
           "--placement", placement] + (["--host"] if host else []) + [f"--opt={o}" for o in opts]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    want, rep, bundle = _single_process(R, placement)
    for tag in ("first", "last"):
        parts = [np.load(os.path.join(tmp_path, f"rank{d}_{tag}.npz")) for d in range(R)]
        for d in range(R):
            assert int(parts[d]["total_bytes"]) == rep["total_bytes"] == int(bundle.volume[0])
        for key in ("o", "lse", "dq", "dk", "dv"):
            got = sum(p[key].astype(np.float64) for p in parts)  # owned rows are disjoint
            if key in ("o", "lse"):
                assert np.array_equal(got, want[key].astype(np.float64)), (tag, key)
            else:
                assert rel_err(got, want[key]) <= 4e-3, (tag, key)
