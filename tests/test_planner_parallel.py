"""CPU: the parallel DCP placement (planner/dcp_partition_parallel.hpp; SURVEY.md 8(f)3,
planner throughput) produces plans bit-identical to the reference's single-threaded
plan_batch (pipeline.hpp:29-38, partition_heuristic hypergraph.hpp:623-784): on the cached
BASELINE plans made by the reference planner in round 1 (plans/*.npz), and against a fresh
reference run on random batches (one and two machines, graphs small enough for fm_pass and
large enough for greedy passes, infeasible epsilons raising the same error)."""
import os
import sys

import numpy as np
import pytest

from paper_2510_10620_b200 import planner as PL

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools"))


def _same(a, b):
    if not (np.array_equal(a.comp_block_device, b.comp_block_device)
            and np.array_equal(a.data_block_device, b.data_block_device) and np.array_equal(a.volume, b.volume)
            and np.array_equal(a.per_device_send, b.per_device_send) and len(a.devices) == len(b.devices)):
        return False
    for x, y in zip(a.devices, b.devices):
        for f in ("capacity", "resident_q", "resident_kv", "resident_o", "instr", "items", "srcs", "copies",
                  "blocks", "rows"):
            if not np.array_equal(getattr(x, f), getattr(y, f)):
                return False
        if list(x.tags) != list(y.tags):
            return False
    return True


@pytest.mark.parametrize("name", ["cfg1_R2", "cfg2_R8", "cfg3_R4", "cfg3_R8", "cfg4_cb_B2048_R8",
                                  "cfg4_sq_B2048_R8"])
def test_parallel_plan_equals_cached_reference_plan(name):
    from make_plans import CONFIGS, load
    fn, R, block, kw = CONFIGS[name]
    cached = load(name)  # planned by the reference's plan_batch (round 1)
    assert _same(PL.plan(fn(), R, block, threads=0, **kw), cached), name


def test_parallel_plan_equals_reference_random():
    ran = 0
    for seed in range(12):
        b = PL.Batch.random(500 + seed, max_seq_len=2400 if seed % 3 else 300, max_seqs=4, max_heads=4)
        R = 2 + seed % 3
        machines = 2 if seed % 4 == 3 and R % 2 == 0 else 1
        kw = dict(eps_intra=0.2 + 0.1 * (seed % 3), eps_data=0.3, eps_inter=0.3, seed=seed, machines=machines)
        block = 128 if seed % 2 else 256
        outs = []
        for threads in (1, 0, 3):
            try:
                outs.append(PL.plan(b, R, block, threads=threads, **kw))
            except PL.PlannerError as e:
                outs.append((e.kind, str(e)))
        ref = outs[0]
        for o in outs[1:]:
            if isinstance(ref, tuple):
                assert o == ref, seed
            else:
                assert not isinstance(o, tuple) and _same(o, ref), seed
        ran += not isinstance(ref, tuple)
    assert ran >= 6
