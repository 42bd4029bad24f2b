"""GPU race detection with the jitter build (build/jitter/libdcpx.so, -DDCPX_JITTER): every
mbarrier wait, scheduler read and cross-process flag poll of the kernels returns after a
pseudo-random delay, so each warp role's timing against the others is perturbed. A missing or
misplaced barrier (a TMA overwrite of a stage still read, a TMEM slot reused early, a send
flag set before its data) then shows up as different numbers. compute-sanitizer racecheck /
synccheck, the first choice, is closed on the GPU pool (profiles/r2_race_checks.md).

The forward is deterministic (no atomics): O and LSE must be bit-identical to the product
build; the backward accumulates with fp32 atomics, so gradients are compared to 1e-3; both
builds are checked against the FP64 oracle by the probe itself."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
JITTER = os.path.join(REPO, "build", "jitter", "libdcpx.so")


def _probe(lib, out):
    env = dict(os.environ)
    if lib:
        env["DCPX_LIB"] = lib
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize_probe.py"), "--out", out],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0 and "SANITIZE PROBE OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


def test_jitter_build_matches_product_single_process(tmp_path):
    assert os.path.exists(JITTER), "jitter build missing (tools/build.py builds it)"
    a = _probe(None, str(tmp_path / "product.npz"))
    b = _probe(JITTER, str(tmp_path / "jitter.npz"))
    assert sorted(a.files) == sorted(b.files)
    for key in a.files:
        if key.endswith(("_o", "_lse")):
            assert np.array_equal(a[key], b[key]), key
        else:
            den = np.abs(a[key]).max() or 1.0
            assert np.abs(a[key] - b[key]).max() / den <= 1e-3, key


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("R", [2, 4])
def test_jitter_build_per_rank_flags(R, tmp_path):
    """The per-rank mode's cross-process epoch flags with late pollers: the ranks' union of
    owned rows equals the single-process product run (tests/test_gpu_rank.py's check)."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_rank import _single_process
    from common import rel_err
    env = dict(os.environ, DCPX_LIB=JITTER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(REPO, "tests", "rank_worker.py"), "--out", str(tmp_path), "--iters", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    want, rep, bundle = _single_process(R, "dcp")
    for tag in ("first", "last"):
        parts = [np.load(os.path.join(tmp_path, f"rank{d}_{tag}.npz")) for d in range(R)]
        for key in ("o", "lse", "dq", "dk", "dv"):
            got = sum(p[key].astype(np.float64) for p in parts)
            if key in ("o", "lse"):
                assert np.array_equal(got, want[key].astype(np.float64)), (tag, key)
            else:
                assert rel_err(got, want[key]) <= 4e-3, (tag, key)


def test_jitter_build_persistent_forward():
    """The persistent forward's device-side ordering (fetch counter, per-tile unit stamps,
    slot-free counters) under late pollers: tests/test_gpu_persistent.py run against the
    jitter build, i.e. (O, LSE) of the persistent launch bit-identical to the per-division
    launches with every wait perturbed. Needs one GPU per plan device."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("the persistent forward needs one GPU per plan device")
    assert os.path.exists(JITTER), "jitter build missing (tools/build.py builds it)"
    env = dict(os.environ, DCPX_LIB=JITTER)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu",
                        os.path.join(REPO, "tests", "test_gpu_persistent.py")],
                       capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
