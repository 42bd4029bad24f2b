"""Per-device op timeline of one forward+backward (executor option "trace").
    python tools/trace_probe.py cfg2_R4 [ngpus]"""
import os
import sys

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
    T, H, G = b.total_tokens, b.H, b.G
    q = torch.randn((T, H, 128), device="cuda").to(torch.bfloat16)
    k = torch.randn((T, G, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((T, G, 128), device="cuda").to(torch.bfloat16)
    ex = DCPExecutor([d % ng for d in range(b.R)])
    ex.set_option("timing", 1)
    for kv in filter(None, os.environ.get("PROBE_OPTS", "").split(",")):  # e.g. persistent=0
        key, val = kv.split("=")
        ex.set_option(key, int(val))
    ex.prepare(b)
    o = torch.empty_like(q)
    lse = torch.empty((H, T), device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    if ng > 1:  # distributed layout, as bench.py: per-device packed buffers
        devs = [d % ng for d in range(b.R)]
        rep = lambda x, like=False: [torch.empty_like(x, device=f"cuda:{d}") if like else x.to(f"cuda:{d}")  # noqa: E731
                                     for d in devs]
        q, k, v = rep(q), rep(k), rep(v)
        o, lse, dq, dk, dv = rep(o, True), rep(lse, True), rep(dq, True), rep(dk, True), rep(dv, True)
    for _ in range(2):
        ex.load_inputs(q, k, v); ex.forward(o, lse); ex.backward(q, dq, dk, dv)
    ex.set_option("trace", 1)

    def sync():  # align the devices' time origins (each span is relative to its device's t0)
        for d in range(ng):
            torch.cuda.synchronize(d)
    ex.load_inputs(q, k, v)
    sync()
    rf = ex.forward(o, lse)
    tf = ex.trace()
    sync()
    rb = ex.backward(q, dq, dk, dv)
    tb = ex.trace()
    print(f"{name} on {ng} GPUs: fwd {rf['device_ms']:.3f} ms, bwd {rb['device_ms']:.3f} ms")
    for label, tr in (("fwd", tf), ("bwd", tb))[: 1 if os.environ.get("PROBE_FWD_ONLY") else 2]:
        for d in range(b.R):
            rows = [t for t in tr if t["dev"] == d]
            s = "  ".join(f"{t['kind']}{t['division']}[{t['start']:.2f}-{t['end']:.2f}]" if t['kind'] != 'launch'
                          else f"L{t['division']}@{t['start']:.2f}" for t in rows)
            print(f"{label} dev{d}: {s}")
    for d in range(b.R):
        print(f"dev{d} flops {int(b.dev_flops[d]) / 1e12:.3f} T")


if __name__ == "__main__":
    main()
