"""Plan files in the reference's JSON formats, CPU.

tests/golden/plan_json/ was written by the reference's own writers (inc/io.hpp:72-350,
via tests/golden/make_plan_json.py); bundle.npz is the same plan flattened by the planner
shim. The JSON loader must give the same views, the reference's explicit item rows must
equal the rows derived from the mask (inc/plan.hpp:231-242), the byte tables recomputed
from the plans must be bit-exact with CommVolume, and writing the plans back must give
the reference's files (tests/test_plan.cpp:177-190 is the reference's own round trip)."""
import json
import os

import numpy as np

import oracle as O
from paper_2510_10620_b200 import planio
from paper_2510_10620_b200.plans import PlanBundle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plan_json")


def _load():
    return planio.load_reference_plan(GOLD), PlanBundle.load(os.path.join(GOLD, "bundle.npz"))


def test_json_plan_matches_planner_views():
    jb, pb = _load()
    assert (jb.R, jb.T, jb.H, jb.G, jb.D, jb.bpe) == (pb.R, pb.T, pb.H, pb.G, pb.D, pb.bpe)
    assert np.array_equal(jb.seq_lengths, pb.seq_lengths)
    assert np.array_equal(jb.block_sizes, pb.block_sizes)
    assert np.array_equal(jb.data_blocks, pb.data_blocks)
    assert np.array_equal(jb.comp_blocks, pb.comp_blocks)
    assert np.array_equal(jb.data_block_device, pb.data_block_device)
    assert np.array_equal(jb.comp_block_device, pb.comp_block_device)
    assert np.array_equal(jb.dev_flops, pb.dev_flops)
    # CommVolume (placement.hpp:180-243) recomputed from the plan files, bit-exact
    assert np.array_equal(jb.per_device_send, pb.per_device_send)
    assert np.array_equal(jb.per_device_recv, pb.per_device_recv)
    assert np.array_equal(jb.volume, pb.volume)
    for a, b in zip(jb.devices, pb.devices):
        assert np.array_equal(a.capacity, b.capacity)
        for f in ("resident_q", "resident_kv", "resident_o", "instr", "srcs", "copies", "blocks"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        assert a.tags == b.tags
        names = [n for n in a.items.dtype.names if n != "rows_offset"]
        assert np.array_equal(a.items[names], b.items[names])
        assert (a.items["rows_offset"] >= 0).all() and (b.items["rows_offset"] == -1).all()


def test_json_rows_equal_rows_derived_from_the_mask():
    jb, pb = _load()
    n = 0
    for dp in jb.devices:
        for it in dp.items:
            nq = int(it["q_end"] - it["q_begin"])
            mine = dp.rows[int(it["rows_offset"]): int(it["rows_offset"]) + nq]
            derived = O.item_rows(pb, int(it["seq"]), int(it["q_begin"]), int(it["q_end"]),
                                  int(it["kv_begin"]), int(it["kv_end"]))
            assert np.array_equal(mine, derived)
            n += 1
    assert n > 0


def test_dump_reproduces_reference_plan_files(tmp_path):
    jb, _ = _load()
    planio.dump_reference_plan(jb, str(tmp_path))
    for d in range(jb.R):
        with open(os.path.join(GOLD, f"plan_d{d}.json")) as f:
            ref = json.load(f)
        with open(os.path.join(tmp_path, f"plan_d{d}.json")) as f:
            mine = json.load(f)
        assert mine == ref


def test_json_plan_runs_in_the_oracle_like_the_planner_plan():
    """Same lockstep execution (bytes, FLOPs, outputs) from either source of the plan."""
    jb, pb = _load()
    rng = np.random.default_rng(3)
    T = int(pb.seq_offsets[-1])
    q = rng.standard_normal((T, pb.H, pb.D))
    k = rng.standard_normal((T, pb.G, pb.D))
    v = rng.standard_normal((T, pb.G, pb.D))
    o1, l1, r1, s1, m1 = O.run(pb, q, k, v)
    o2, l2, r2, s2, m2 = O.run(jb, q, k, v)
    assert s1 == s2 == 0, (m1, m2)
    assert r1.total_bytes == r2.total_bytes == int(pb.volume[0])
    assert np.array_equal(o1, o2) and np.array_equal(l1, l2)
