"""Plans the BASELINE.json configurations once with the reference planner (unchanged,
via planner/_build/libdcpplanner.so) and caches them as plans/<name>.npz.

Planning is slow single-threaded reference code and is never
timed; bench.py and the GPU tests load these caches. Usage:
    python tools/make_plans.py [name ...]      # default: every config below
"""
from __future__ import annotations

import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2510_10620_b200 import planner as PL  # noqa: E402

PLAN_DIR = os.path.join(REPO, "plans")

# name -> (batch factory, R, block, planner kwargs)
CFG1 = [PL.SeqSpec(8192), PL.SeqSpec(4096), PL.SeqSpec(2048), PL.SeqSpec(2048)]


def cfg1_batch():
    return PL.Batch.from_specs(CFG1, 8, 2, 128)


# configs[4]: long-tail stress, one 512K causal sequence plus many short ones (48 sequences of
# 0.5K-4K tokens, 110,592 tokens): 634,880 tokens in one batch
CFG5 = [PL.SeqSpec(524288)] + [PL.SeqSpec(1024 * (1 + i % 4) - 256 * (i % 3)) for i in range(48)]


def cfg5_batch():
    return PL.Batch.from_specs(CFG5, 32, 8, 128)


def synth(mask, max_len, budget, index):
    def f():
        b, _ = PL.Batch.from_synth(mask, max_len, budget, index, 32, 8, seed=42)
        return b
    return f


CONFIGS = {
    # configs[0]: CPU-reference workload (4 varlen causal seqs, 16K tokens, H 8 / G 2, block 1024)
    "cfg1_R1": (cfg1_batch, 1, 1024, {}),
    "cfg1_R2": (cfg1_batch, 2, 1024, {}),
    # configs[1]: 8B-GPT layer (32/8 heads), causal, LongAlign-skewed 64K batch
    # (synth seed 42, make_batches budget 65536, batch index 2: 6 sequences, 63,855 tokens)
    "cfg2_R1": (synth("causal", 65536, 65536, 2), 1, 1024, {}),
    "cfg2_R2": (synth("causal", 65536, 65536, 2), 2, 1024, {}),
    "cfg2_R4": (synth("causal", 65536, 65536, 2), 4, 1024, {}),
    "cfg2_R8": (synth("causal", 65536, 65536, 2), 8, 1024, {}),
    # the paper's baseline placements of the same batch (inc/baselines.hpp:46-112)
    "cfg2_ring_R4": (synth("causal", 65536, 65536, 2), 4, 1024, {"placement": "ring"}),
    "cfg2_ring_R8": (synth("causal", 65536, 65536, 2), 8, 1024, {"placement": "ring"}),
    "cfg2_zigzag_R4": (synth("causal", 65536, 65536, 2), 4, 1024, {"placement": "zigzag"}),
    "cfg2_zigzag_R8": (synth("causal", 65536, 65536, 2), 8, 1024, {"placement": "zigzag"}),
    # configs[2]: 128K lambda (sink 64 + window 4096), 1/2/4/8 GPUs
    "cfg3_R1": (synth("lambda", 131072, 131072, 0), 1, 1024, {}),
    "cfg3_R2": (synth("lambda", 131072, 131072, 0), 2, 1024, {}),
    "cfg3_R4": (synth("lambda", 131072, 131072, 0), 4, 1024, {}),
    "cfg3_R8": (synth("lambda", 131072, 131072, 0), 8, 1024, {}),
    # configs[3]: shared-question / causal-blockwise at 128K, block sweep (R 8)
    "cfg4_sq_B2048_R8": (synth("shared_question", 131072, 131072, 0), 8, 2048, {}),
    "cfg4_cb_B512_R8": (synth("causal_blockwise", 131072, 131072, 0), 8, 512, {}),
    "cfg4_cb_B1024_R8": (synth("causal_blockwise", 131072, 131072, 0), 8, 1024, {}),
    "cfg4_cb_B2048_R8": (synth("causal_blockwise", 131072, 131072, 0), 8, 2048, {}),
    # the same block sweep on one device (bench.py --config cfg4_cb_B512 etc.)
    "cfg4_cb_B512_R1": (synth("causal_blockwise", 131072, 131072, 0), 1, 512, {}),
    "cfg4_cb_B1024_R1": (synth("causal_blockwise", 131072, 131072, 0), 1, 1024, {}),
    "cfg4_cb_B2048_R1": (synth("causal_blockwise", 131072, 131072, 0), 1, 2048, {}),
    "cfg4_sq_B2048_R1": (synth("shared_question", 131072, 131072, 0), 1, 2048, {}),
    # configs[4]: long-tail stress (512K + short tail), causal. With the reference's
    # single-threaded partitioner block 4096 did not finish within 20 min for 4 or 8 devices
    # (265,728 comp blocks), so block-8192 plans exist as well (68,096 comp blocks).
    "cfg5_R1": (cfg5_batch, 1, 4096, {}),
    # block 4096 on 4 / 8 devices (265,728 comp blocks): unplannable by the single-threaded
    # reference partitioner (> 20 min); the bit-identical parallel partitioner
    # (planner/dcp_partition_parallel.hpp, planner.plan threads=0) plans them in minutes
    "cfg5_R4": (cfg5_batch, 4, 4096, {}),
    "cfg5_R8": (cfg5_batch, 8, 4096, {}),
    "cfg5_B8192_R1": (cfg5_batch, 1, 8192, {}),
    "cfg5_B8192_R4": (cfg5_batch, 4, 8192, {}),
    "cfg5_B8192_R8": (cfg5_batch, 8, 8192, {}),
}


def make(name: str, force: bool = False):
    path = os.path.join(PLAN_DIR, name + ".npz")
    if os.path.exists(path) and not force:
        return path
    fn, R, block, kw = CONFIGS[name]
    t = time.time()
    bundle = PL.plan(fn(), R, block, **kw)
    bundle.meta["name"] = name
    bundle.meta["plan_seconds"] = f"{time.time() - t:.1f}"
    os.makedirs(PLAN_DIR, exist_ok=True)
    bundle.save(path)
    print(f"{name}: R={R} block={block} tokens={bundle.total_tokens} comp_blocks={len(bundle.comp_blocks)} "
          f"fwd_flops={bundle.total_flops / 1e12:.3f}T bytes={int(bundle.volume[0])} "
          f"plan={time.time() - t:.1f}s size={os.path.getsize(path) / 1e6:.2f}MB", flush=True)
    return path


def load(name: str):
    from paper_2510_10620_b200.plans import PlanBundle
    path = os.path.join(PLAN_DIR, name + ".npz")
    if not os.path.exists(path):
        make(name)
    return PlanBundle.load(path)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS)
    for n in names:
        try:
            make(n, force="--force" in os.environ.get("MAKE_PLANS_FLAGS", ""))
        except Exception as e:  # noqa: BLE001
            print(f"{n}: FAILED {e}", flush=True)
