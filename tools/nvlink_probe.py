"""NVLink evidence for the block exchange (simexec.hpp:263-327 CommLaunch/CommWait): one
forward + backward of a cached multi-device plan in one process on N GPUs with the executor's
op trace on; every transfer span ("xfer": the copy kernel a CommWait runs on the receiver's
comm stream once its send / receive events resolved) is matched with the bytes that message
moves (PlanBundle.wire_bytes's per-message rule) -> achieved GB/s per transfer, per
direction and overall, next to a plain torch peer copy of 1 GiB as the link reference.
    python tools/nvlink_probe.py cfg3_R4 [ngpus]   -> JSON on stdout"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from make_plans import load  # noqa: E402
from paper_2510_10620_b200 import plans as P  # noqa: E402
from paper_2510_10620_b200.executor import DCPExecutor  # noqa: E402


def message_bytes(b):
    """(device, instr index of the CommWait) -> (src, fwd bytes, bwd bytes) for every message."""
    db = b.data_blocks
    out = {}
    for dp in b.devices:
        recv = {}
        for i, ins in enumerate(dp.instructions()):
            if ins["op"] == P.OP_COMM_LAUNCH and not ins["send"]:
                fwd = bwd = 0
                for blk in dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]["block"]:
                    kind, size = int(db["kind"][blk]), int(db["size_bytes"][blk])
                    rows = int(db["tok_end"][blk] - db["tok_begin"][blk])
                    fwd += size + (4 * rows if kind == P.KIND_O else 0)
                    bwd += (2 * size + 8 * rows) if kind == P.KIND_Q else size if kind == P.KIND_KV else 0
                recv[ins["tag"]] = (ins["peer"], fwd, bwd)
            elif ins["op"] == P.OP_COMM_WAIT:
                out[(dp.device, i)] = recv[ins["tag"]]
    return out


def peer_copy_gbs(src, dst, nbytes=1 << 30):
    a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src}")
    b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dst}")
    for _ in range(2):
        b.copy_(a)
    torch.cuda.synchronize(src); torch.cuda.synchronize(dst)
    with torch.cuda.device(dst):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            b.copy_(a)
        e1.record()
        e1.synchronize()
    return 5 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_R4"
    b = load(name)
    ng = int(sys.argv[2]) if len(sys.argv) > 2 else min(b.R, torch.cuda.device_count())
    devs = [d % ng for d in range(b.R)]
    T, H, G = b.total_tokens, b.H, b.G
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((T, n, 128), device="cuda", generator=g).to(torch.bfloat16) for n in (H, G, G))
    rep = lambda x, like=False: [torch.empty_like(x, device=f"cuda:{d}") if like else x.to(f"cuda:{d}")  # noqa: E731
                                 for d in devs]
    o, lse = torch.empty_like(q), torch.empty((H, T), device="cuda")
    qs, ks, vs, os_, ls = rep(q), rep(k), rep(v), rep(o, True), rep(lse, True)
    dqs, dks, dvs = rep(q, True), rep(k, True), rep(v, True)
    ex = DCPExecutor(devs)
    ex.prepare(b)
    for _ in range(2):
        ex.load_inputs(qs, ks, vs); ex.forward(os_, ls); ex.backward(qs, dqs, dks, dvs)
    ex.set_option("trace", 1)
    ex.set_option("timing", 1)
    msgs = message_bytes(b)
    spans = []
    for pass_ in ("fwd", "bwd"):
        ex.load_inputs(qs, ks, vs)
        for d in set(devs):
            torch.cuda.synchronize(d)
        r = ex.forward(os_, ls) if pass_ == "fwd" else ex.backward(qs, dqs, dks, dvs)
        for t in ex.trace():
            if t["kind"] != "xfer":
                continue
            src, fb, bb = msgs[(t["dev"], t["instr"])]
            nbytes = fb if pass_ == "fwd" else bb
            ms = t["end"] - t["start"]
            if nbytes and ms > 0:
                spans.append(dict(pass_=pass_, src=int(src), dst=t["dev"], division=t["division"], bytes=nbytes,
                                  ms=ms, gbs=nbytes / (ms * 1e-3) / 1e9))
        if pass_ == "fwd":
            fwd_ms = r["device_ms"]
        else:
            bwd_ms = r["device_ms"]
    ex.close()
    big = [s for s in spans if s["bytes"] >= 8 << 20]
    res = {"plan": name, "gpus": ng, "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "transfers": len(spans),
           "bytes": int(sum(s["bytes"] for s in spans)),
           "gbs_weighted": sum(s["bytes"] for s in spans) / (sum(s["ms"] for s in spans) * 1e-3) / 1e9,
           "gbs_median": float(np.median([s["gbs"] for s in spans])) if spans else None,
           "gbs_large_median": float(np.median([s["gbs"] for s in big])) if big else None,
           "large_transfers": len(big),
           "peer_copy_gbs_ref": peer_copy_gbs(0, 1) if ng > 1 else None,
           "spans": spans}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
