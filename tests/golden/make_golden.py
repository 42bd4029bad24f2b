"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libdcpref.so, built
from /root/reference by oracle/Makefile). Run here (needs /root/reference); the fixtures are
committed so the CPU oracle can be pinned anywhere.

  golden_payload.npz : make_payload(seed 1, H 2, G 1, L 3, D 4)  (simexec.hpp:125-146)
  golden_runs.npz    : plan_batch + run outputs of the reference for small mixed-mask batches
                       on 1/2/4 devices (inputs = make_payload), with bytes / FLOP accounting
  golden_kat.npz     : exec_attention / exec_reduction known answers (test_simexec.cpp:36-162)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import oracle as O  # noqa: E402
from paper_2510_10620_b200 import planner as PL  # noqa: E402

RUN_CASES = [
    # (specs, H, G, D, R, block, eps(inter, intra, data), seed)
    ([PL.SeqSpec(40), PL.SeqSpec(23, "lambda", sink=3, window=5)], 2, 1, 8, 1, 8, (0.4, 0.1, 0.05), 1),
    ([PL.SeqSpec(30, "shared_question", question_len=6, answer_lens=[10, 14]),
      PL.SeqSpec(33, "causal_blockwise", block=4, window_blocks=2, sink_blocks=1, test_blocks=1)],
     4, 2, 16, 2, 8, (0.4, 0.5, 0.6), 2),
    ([PL.SeqSpec(48), PL.SeqSpec(17, "lambda", sink=2, window=4),
      PL.SeqSpec(25, "shared_question", question_len=5, answer_lens=[7, 6, 7])],
     4, 2, 16, 4, 4, (0.4, 0.5, 0.6), 3),
]


def main():
    q, k, v = O.ref_make_payload([PL.SeqSpec(3)], 2, 1, 4, 1)
    np.savez(os.path.join(HERE, "golden_payload.npz"), q=q, k=k, v=v)
    arrs = {}
    for i, (specs, H, G, D, R, block, eps, seed) in enumerate(RUN_CASES):
        q, k, v = O.ref_make_payload(specs, H, G, D, seed)
        o, stats, _ = O.ref_plan_run(specs, H, G, D, R, block, q, k, v, eps=eps)
        arrs[f"c{i}_q"], arrs[f"c{i}_k"], arrs[f"c{i}_v"], arrs[f"c{i}_o"] = q, k, v, o
        arrs[f"c{i}_stats"] = np.array([stats["total_bytes"], stats["total_flops"]] +
                                       list(stats["send"]) + list(stats["recv"]), np.uint64)
    np.savez_compressed(os.path.join(HERE, "golden_runs.npz"), **arrs)
    # known answers
    rng = np.random.default_rng(97)
    kat = {}
    q, k, v = (rng.standard_normal((9, 4)) for _ in range(3))
    rows = np.zeros((9, 4), np.int32)
    rows[:, 1] = 9
    kat["full_q"], kat["full_k"], kat["full_v"] = q, k, v
    kat["full_o"], kat["full_m"], kat["full_l"] = O.ref_exec_attention(q, k, v, rows)
    rows2 = np.zeros((9, 4), np.int32)
    rows2[0] = [0, 2, 0, 0]
    rows2[3] = [1, 3, 5, 8]
    kat["mask_rows"] = rows2
    kat["mask_o"], kat["mask_m"], kat["mask_l"] = O.ref_exec_attention(q, k, v, rows2)
    parts = [O.ref_exec_attention(q, k[:4], v[:4], np.tile([0, 4, 0, 0], (9, 1)).astype(np.int32)),
             O.ref_exec_attention(q, k[4:], v[4:], np.tile([0, 5, 0, 0], (9, 1)).astype(np.int32))]
    for j, (o_, m_, l_) in enumerate(parts):
        kat[f"part{j}_o"], kat[f"part{j}_m"], kat[f"part{j}_l"] = o_, m_, l_
    kat["red_o"], kat["red_m"], kat["red_l"] = O.ref_exec_reduction(parts)
    np.savez(os.path.join(HERE, "golden_kat.npz"), **kat)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
