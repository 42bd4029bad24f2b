"""Quick device-time probe of the executor on a cached plan (not the bench contract).
    python tools/perf_probe.py cfg2_R1 [iters]"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import torch  # noqa: E402

from make_plans import load  # noqa: E402
from paper_2510_10620_b200.executor import DCPExecutor  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_R1"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    b = load(name)
    T, H, G = b.total_tokens, b.H, b.G
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((T, H, 128), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((T, G, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((T, G, 128), device="cuda", generator=g).to(torch.bfloat16)
    ex = DCPExecutor([0] * b.R)
    ex.set_option("timing", 1)  # device_ms in the reports
    for opt in sys.argv[3:]:
        key, _, val = opt.partition("=")
        ex.set_option(key, int(val))
    ex.prepare(b)
    o = torch.empty((T, H, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((H, T), device="cuda")
    ex.load_inputs(q, k, v)
    for _ in range(3):
        rep = ex.forward(o, lse)
    times = []
    reload = os.environ.get("PROBE_RELOAD")  # scatter the inputs again before every forward
    for _ in range(iters):
        if reload:
            ex.load_inputs(q, k, v)
        rep = ex.forward(o, lse)
        times.append(rep["device_ms"])
    ms = min(times)
    print(f"{name}: fwd flops {b.total_flops / 1e12:.3f} T  device {ms:.3f} ms (median {sorted(times)[len(times)//2]:.3f})"
          f"  -> {b.total_flops / ms / 1e9:.1f} TFLOP/s  launches {rep['kernel_launches']}")
    d_o = torch.randn((T, H, 128), device="cuda", generator=g).to(torch.bfloat16)
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    bt = []
    for _ in range(3):
        ex.forward(o, lse)
        ex.backward(d_o, dq, dk, dv)
    for _ in range(iters):
        ex.forward(o, lse)
        rep = ex.backward(d_o, dq, dk, dv)
        bt.append(rep["device_ms"])
    bms = min(bt)
    print(f"{name}: bwd flops {rep['total_flops'] / 1e12:.3f} T  device {bms:.3f} ms -> {rep['total_flops'] / bms / 1e9:.1f} TFLOP/s;"
          f"  fwd+bwd {ms + bms:.3f} ms -> {3.5 * b.total_flops / (ms + bms) / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
