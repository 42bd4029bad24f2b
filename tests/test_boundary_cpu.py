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
