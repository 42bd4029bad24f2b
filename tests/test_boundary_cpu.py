"""CPU: the C-ABI library loads and exports every symbol include/dcpx.h declares, the
product never imports the oracle, and the plan bundles / byte formulas are consistent
with the reference planner (no GPU needed)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2510_10620_b200 import executor as E
from paper_2510_10620_b200 import planner as PL
from paper_2510_10620_b200 import plans as P

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "dcpx.h")).read()
    return sorted(set(re.findall(r"\b(dcpx_[a-z_]+)\s*\(", src)))


def test_header_symbols_are_exported():
    syms = header_symbols()
    assert set(syms) == set(E.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", E.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dcpx_[a-z_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    lib = E.lib()
    assert lib.dcpx_version().startswith(b"dcpx")


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "-sass", E.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out  # TMA loads
    assert "LDTM" in out and "STTM" in out  # TMEM
    assert "HMMA" not in out.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2510_10620_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "dcp_oracle" not in text, f


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(E.DCPXError):
        E.DCPExecutor([0])


def test_bundle_roundtrip_and_bytes(tmp_path):
    b = PL.Batch.from_specs([PL.SeqSpec(300), PL.SeqSpec(200, "lambda", sink=8, window=50)], 4, 2, 128)
    bundle = PL.plan(b, 2, 128, eps_intra=0.4, eps_data=0.6)
    path = str(tmp_path / "b.npz")
    bundle.save(path)
    back = P.PlanBundle.load(path)
    assert back.R == bundle.R and back.total_flops == bundle.total_flops
    for a, c in zip(bundle.devices, back.devices):
        assert np.array_equal(a.instr, c.instr) and a.tags == c.tags
        assert np.array_equal(a.items, c.items)
    # plan send bytes == communication_volume (test_plan.cpp:94-119)
    sent = 0
    for dp in bundle.devices:
        for ins in dp.instructions():
            if ins["op"] == P.OP_COMM_LAUNCH and ins["send"]:
                blks = dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]
                sent += int(bundle.data_blocks["size_bytes"][blks["block"]].sum())
    assert sent == int(bundle.volume[0])
    send, recv = bundle.bwd_bytes()
    assert int(send.sum()) == int(recv.sum())


def test_plan_fuzz_bytes_equal_volume():  # test_plan.cpp:371-389 (placement via the planner)
    for seed in range(10):
        b = PL.Batch.random(seed, max_seq_len=32, max_seqs=3, max_heads=2, head_dim=4)
        try:
            bundle = PL.plan(b, 1 + seed % 4, 1 + seed % 6, eps_intra=0.5, eps_inter=0.5, eps_data=0.8)
        except PL.PlannerError as e:
            assert e.kind == "InfeasibleError"
            continue
        sent = 0
        for dp in bundle.devices:
            for ins in dp.instructions():
                if ins["op"] == P.OP_COMM_LAUNCH and ins["send"]:
                    blks = dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]
                    sent += int(bundle.data_blocks["size_bytes"][blks["block"]].sum())
        assert sent == int(bundle.volume[0])


def test_buffer_overflow_maps_to_status():  # test_plan.cpp:423-430
    b = PL.Batch.from_specs([PL.SeqSpec(64, "shared_question", question_len=8, answer_lens=[16, 12, 12, 16])], 1, 1, 8)
    with pytest.raises(PL.PlannerError) as ei:
        PL.plan(b, 4, 4, placement="ring", max_slots_per_kind=1)
    assert ei.value.kind == "BufferOverflowError"


def test_cached_configs_present():
    # the bench / GPU tests never plan at run time; configs 1-3 are cached in plans/
    for name in ("cfg1_R1", "cfg1_R2", "cfg2_R1", "cfg2_R2", "cfg2_R4", "cfg2_R8", "cfg3_R1", "cfg3_R8"):
        path = os.path.join(REPO, "plans", name + ".npz")
        assert os.path.exists(path), name
    b = P.PlanBundle.load(os.path.join(REPO, "plans", "cfg1_R2.npz"))
    assert int(b.volume[0]) == 12582912 and len(b.comp_blocks) == 416  # SURVEY.md section 6 probe


def test_check_plans_host_only():
    """dcpx_check_plans: verify_plans + the lockstep replay without a GPU. A planner bundle
    passes; deleting a device's sends is a deadlock (tests/test_simexec.cpp:251-270); a
    renamed receive tag is a tag mismatch; an out-of-range slot is a buffer overflow
    (plan.hpp:368-380)."""
    specs = [PL.SeqSpec(256)]
    b = PL.Batch.from_specs(specs, 1, 1, 128)
    gt, cq = b.graph_counts(128)

    def fresh():
        return PL.plan(b, 2, 128, placement="explicit", group_dev=gt, comp_dev=cq, divisions=2)

    E.check_plans(fresh())  # no exception
    bad = fresh()
    dp = bad.devices[0]
    dp.instr = dp.instr[[i for i, r in enumerate(dp.instr) if not (r[0] == 3 and r[2] == 1)]]
    with pytest.raises(E.DCPXError) as ei:
        E.check_plans(bad)
    assert ei.value.kind == "DeadlockError"

    bad = fresh()
    dp = bad.devices[1]
    waits = [i for i, r in enumerate(dp.instr) if r[0] == 4]
    assert waits
    dp.tags = list(dp.tags) + ["no-such-tag"]  # the wait names a tag no receive posted
    dp.instr = dp.instr.copy()
    dp.instr[waits[0], 7] = len(dp.tags) - 1
    with pytest.raises(E.DCPXError) as ei:
        E.check_plans(bad)
    assert ei.value.kind == "TagMismatchError"

    bad = fresh()
    dp = bad.devices[0]
    att = [i for i, r in enumerate(dp.instr) if r[0] == 0]
    dp.items = dp.items.copy()
    dp.items["out_slot"][int(dp.instr[att[0]][6])] = int(dp.capacity[2]) + 5
    with pytest.raises(E.DCPXError) as ei:
        E.check_plans(bad)
    assert ei.value.kind == "BufferOverflowError"


def test_check_plans_any_head_dim():
    """The host-only check executes nothing, so it accepts shapes the sm_100a kernels do not
    (head_dim 64): the cost-only drop-in path (include/dcp_gpu.hpp) relies on this."""
    b = PL.Batch.from_specs([PL.SeqSpec(300), PL.SeqSpec(100, "lambda", sink=4, window=20)], 2, 1, 64)
    bundle = PL.plan(b, 2, 128, eps_intra=0.5, eps_data=0.6)
    E.check_plans(bundle)


def test_dropin_cost_only_without_gpu():
    """include/dcp_gpu.hpp in cost-only mode (SimOptions::numeric = false) runs without a GPU
    and equals the reference's cost-mode run() report for D = 64, raising DeadlockError where
    the reference does (tests/cpp/test_dcp_gpu_cost.cpp)."""
    binp = os.path.join(REPO, "tests", "cpp", "_build", "test_dcp_gpu_cost")
    if not os.path.exists(binp):
        pytest.skip("drop-in test binaries are built where /root/reference exists (tools/build.py)")
    r = subprocess.run([binp], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "COST PASS" in r.stdout, r.stdout + r.stderr


def test_item_sample_bundle_and_reference_items():
    """bench.py's CPU-baseline check: PlanBundle.item_sample builds a valid one-device plan
    running sampled AttentionItems alone (host-only check), and oracle.ref_run_items (the
    reference exec_attention on given inputs) returns (out, m + ln l) equal to the C
    restatement on the same items."""
    import oracle as O
    if not O.ref_available():
        pytest.skip("reference shim not built")
    specs = [PL.SeqSpec(700), PL.SeqSpec(500, "lambda", sink=16, window=100),
             PL.SeqSpec(600, "shared_question", question_len=100, answer_lens=[250, 250])]
    b = PL.Batch.from_specs(specs, 4, 2, 128)
    bundle = PL.plan(b, 2, 256, eps_intra=0.4, eps_data=0.6)
    items = np.concatenate([dp.items for dp in bundle.devices])[::3]
    sb = bundle.item_sample(items)
    E.check_plans(sb)
    assert sb.devices[0].capacity[2] == len(items)
    rng = np.random.default_rng(0)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    q, k, v = (rng.standard_normal((T, n, 128)) for n in (H, G, G))
    work = []
    for it in items[:6]:
        s, h = int(it["seq"]), int(it["head"])
        off = int(bundle.seq_offsets[s])
        rows = O.item_rows(bundle, s, int(it["q_begin"]), int(it["q_end"]), int(it["kv_begin"]), int(it["kv_end"]))
        gq = h * G // H
        work.append(dict(rows=rows, q=q[off + int(it["q_begin"]):off + int(it["q_end"]), h],
                         k=k[off + int(it["kv_begin"]):off + int(it["kv_end"]), gq],
                         v=v[off + int(it["kv_begin"]):off + int(it["kv_end"]), gq]))
    outs, lses, sec = O.ref_run_items(work, 128, 2)
    for w, o, l in zip(work, outs, lses):
        o2, m2, l2 = O.exec_attention(w["q"], w["k"], w["v"], w["rows"])
        assert np.abs(o - o2).max() <= 1e-12
        fin = l2 > 0
        assert np.array_equal(np.isfinite(l), fin)
        assert np.abs(l[fin] - (m2[fin] + np.log(l2[fin]))).max() <= 1e-12


def test_package_import_sets_hardware_queue_count():
    """Importing the package before any CUDA call defaults CUDA_DEVICE_MAX_CONNECTIONS to 32
    (the compute and comm streams must not share a hardware work queue,
    profiles/r2_n4_scheduler_queues_persistent.md); a caller's own setting wins."""
    import subprocess
    import sys
    code = "import os, paper_2510_10620_b200; print(os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS'))"
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=REPO, capture_output=True, text=True)
    assert out.stdout.strip() == "32", out.stderr
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "16"
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=REPO, capture_output=True, text=True)
    assert out.stdout.strip() == "16", out.stderr
