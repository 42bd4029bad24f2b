"""Host-side enqueue cost of one forward / backward call (executor option timing=0, so
the calls do not wait for the GPU).
    python tools/host_probe.py cfg3_R4 [ngpus]"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import torch  # noqa: E402

from make_plans import load  # noqa: E402
from paper_2510_10620_b200.executor import DCPExecutor  # noqa: E402


def main():
    name = sys.argv[1]
    b = load(name)
    ng = int(sys.argv[2]) if len(sys.argv) > 2 else min(b.R, torch.cuda.device_count())
    devs = [d % ng for d in range(b.R)]
    T, H, G = b.total_tokens, b.H, b.G
    rep = lambda x: [x.to(f"cuda:{d}") for d in devs]  # noqa: E731
    q = rep(torch.randn((T, H, 128), device="cuda").to(torch.bfloat16))
    k = rep(torch.randn((T, G, 128), device="cuda").to(torch.bfloat16))
    v = rep(torch.randn((T, G, 128), device="cuda").to(torch.bfloat16))
    o = [torch.empty_like(x) for x in q]
    lse = [torch.empty((H, T), device=f"cuda:{d}") for d in devs]
    dq, dk, dv = [torch.empty_like(x) for x in q], [torch.empty_like(x) for x in k], [torch.empty_like(x) for x in v]
    ex = DCPExecutor(devs)
    ex.prepare(b)
    ex.set_option("timing", 0)
    for _ in range(2):
        ex.load_inputs(q, k, v); ex.forward(o, lse); ex.backward(q, dq, dk, dv)
    ex.synchronize()
    tl, tf, tb = [], [], []
    for _ in range(5):
        t0 = time.perf_counter(); ex.load_inputs(q, k, v)
        t1 = time.perf_counter(); ex.forward(o, lse)
        t2 = time.perf_counter(); ex.backward(q, dq, dk, dv)
        t3 = time.perf_counter()
        ex.synchronize()
        tl.append(t1 - t0); tf.append(t2 - t1); tb.append(t3 - t2)
    print(f"{name} on {ng} GPUs host enqueue: load {min(tl) * 1e3:.3f} ms, fwd {min(tf) * 1e3:.3f} ms, "
          f"bwd {min(tb) * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
