"""Shared test helpers: plan bundles from the reference planner, seeded inputs,
tolerances (north_star: O/dQ/dK/dV max relative error <= 2e-2, LSE <= 1e-3)."""
from __future__ import annotations

import numpy as np

from paper_2510_10620_b200 import planner as PL
from paper_2510_10620_b200 import plans as P

O_TOL = 2e-2     # max |x - ref| / max |ref| on O, dQ, dK, dV
LSE_TOL = 1e-3   # max |lse - ref| / max |ref| on finite LSE entries

MIXED_SPECS = [
    PL.SeqSpec(700),
    PL.SeqSpec(900, "lambda", sink=64, window=300),
    PL.SeqSpec(700, "shared_question", question_len=200, answer_lens=[150, 250, 100]),
    PL.SeqSpec(600, "causal_blockwise", block=64, window_blocks=2, sink_blocks=1, test_blocks=1),
]


def bundle_for(specs, H=4, G=2, block=256, R=1, **kw) -> P.PlanBundle:
    b = PL.Batch.from_specs(specs, H, G, 128)
    kw.setdefault("eps_intra", 0.4)
    kw.setdefault("eps_data", 0.6)
    return PL.plan(b, R, block, **kw)


def inputs(bundle: P.PlanBundle, seed: int = 0, scale: float = 1.0):
    """Seeded N(0,1) q [T,H,D], k, v [T,G,D] rounded to bf16; returns torch bf16 (CPU)
    tensors and their exact float64 values (fed to the oracle)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    T, H, G, D = bundle.total_tokens, bundle.H, bundle.G, bundle.D
    q = (torch.randn((T, H, D), generator=g) * scale).to(torch.bfloat16)
    k = (torch.randn((T, G, D), generator=g) * scale).to(torch.bfloat16)
    v = torch.randn((T, G, D), generator=g).to(torch.bfloat16)
    return (q, k, v), tuple(x.double().numpy() for x in (q, k, v))


def rel_err(x, ref) -> float:
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    return float(np.abs(x - ref).max() / (den if den > 0 else 1.0))


def lse_err(lse, ref) -> float:
    lse = np.asarray(lse, np.float64)
    ref = np.asarray(ref, np.float64)
    fin = np.isfinite(ref)
    assert np.array_equal(fin, np.isfinite(lse)), "LSE -inf pattern differs"
    if not fin.any():
        return 0.0
    return float(np.abs(lse[fin] - ref[fin]).max() / max(1.0, np.abs(ref[fin]).max()))


def sampled_rows(bundle: P.PlanBundle, n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    T, H = bundle.total_tokens, bundle.H
    return rng.integers(0, T, n), rng.integers(0, H, n)


def dense_rows_forward(bundle: P.PlanBundle, q, k, v, toks, heads):
    """FP64 masked attention (tests/oracle.hpp:80-120 semantics) for selected (token,
    head) rows only; cheap enough for full-size configs."""
    D = bundle.D
    G, H = bundle.G, bundle.H
    seq_of = np.searchsorted(bundle.seq_offsets, toks, side="right") - 1
    outs, lses = [], []
    for t, h, s in zip(toks, heads, seq_of):
        off = int(bundle.seq_offsets[s])
        r = bundle.ranges[t]
        keys = np.concatenate([np.arange(r[0], r[1]), np.arange(r[2], r[3])]).astype(np.int64) + off
        grp = h * G // H
        if len(keys) == 0:
            outs.append(np.zeros(D)); lses.append(-np.inf); continue
        sc = k[keys, grp, :] @ q[t, h, :] / np.sqrt(D)
        m = sc.max()
        w = np.exp(sc - m)
        l = w.sum()
        outs.append((w / l) @ v[keys, grp, :])
        lses.append(m + np.log(l))
    return np.array(outs), np.array(lses)
