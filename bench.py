"""bench.py — DCP executor fwd+bwd throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): 8B-GPT attention layer, 32 query / 8 KV heads, d 128,
causal mask, LongAlign-like skewed lengths, 64K-token batch (synth seed 42, make_batches
budget 65536, batch index 2: 6 sequences, 63,855 tokens), block 1024, T = 4 divisions,
planned by the reference planner for R = N devices (plans/cfg2_R{N}.npz; planning is never
timed). One step = load packed bf16 Q/K/V into the slot arenas + forward + backward of the
whole plan. FLOPs count only attended pairs: F_fwd = 4 * D * pairs (blocks.hpp:191),
F_total = 3.5 * F_fwd.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dcpx|reference] [--config cfg2]

N > 1 (launched by torchrun, default --mode rank): one process per GPU, rank r executes
plan device r (dcpx_create_rank: peer arenas mapped over CUDA IPC, transfers are pulls
over NVLink ordered by device-side flags); timing is the max over ranks. --mode single:
rank 0's context owns all N devices and the other ranks join the barriers only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:  # noqa: BLE001
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """Samples nvidia-smi SM clocks and throttle reasons during the timed region."""

    def __init__(self, gpus):
        self.gpus = gpus
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                      "-i", ",".join(str(g) for g in self.gpus)],
                                     capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    f = [x.strip() for x in line.split(",")]
                    if len(f) >= 6:
                        self.samples.append(f)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons}


def load_bundle(name):
    from make_plans import load
    return load(name)


def cpu_baseline(bundle, seconds_target=15.0):
    """Reference exec_attention (simexec.hpp:33-76, the reference's CPU executor hot loop)
    on a deterministic sample of this plan's AttentionItems, all host threads."""
    import numpy as np

    import oracle as O
    if not O.ref_available():
        return None
    threads = os.cpu_count() or 1
    items = []
    for dp in bundle.devices:
        for ins in dp.instructions():
            if ins["op"] == 0:
                items.extend(dp.items[ins["offset"]: ins["offset"] + ins["count"]])
    # every k-th item, ~1.68 GFLOP/s/core for FP64 exec_attention
    per_item = float(np.mean([(it["q_end"] - it["q_begin"]) * (it["kv_end"] - it["kv_begin"]) for it in items]))
    budget_flops = seconds_target * threads * 1.5e9
    n = max(threads, min(len(items), int(budget_flops / (4 * 128 * per_item * 0.6))))
    stride = max(1, len(items) // n)
    sample = items[::stride][:n]
    nq, nk, offs, rows, flops = [], [], [], [], 0
    off = 0
    for it in sample:
        r = O.item_rows(bundle, int(it["seq"]), int(it["q_begin"]), int(it["q_end"]),
                        int(it["kv_begin"]), int(it["kv_end"]))
        nq.append(len(r)); nk.append(int(it["kv_end"] - it["kv_begin"])); offs.append(off)
        rows.append(r); off += len(r)
        flops += 4 * 128 * int(np.maximum(r[:, 1] - r[:, 0], 0).sum() + np.maximum(r[:, 3] - r[:, 2], 0).sum())
    sec = O.ref_time_items(nq, nk, offs, np.concatenate(rows), 128, threads)
    return {"value": flops / sec / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
            "sample": f"reference exec_attention (FP64, forward only: the reference has no backward) on "
                      f"{len(sample)} of {len(items)} AttentionItems (every {stride}th), {flops / 1e9:.1f} GFLOP "
                      f"in {sec:.2f}s on {threads} host threads",
            "seconds": sec, "flops": flops}


def covered_tokens(bundle, d, key):
    """Tokens of the packed layout covered by plan device d's resident blocks (`key`:
    resident_q / resident_kv / resident_o): the rows a rank's host I/O copies."""
    import numpy as np
    mask = np.zeros(bundle.total_tokens, bool)
    for r in getattr(bundle.devices[d], key):
        db = bundle.data_blocks[int(r["block"])]
        off = int(bundle.seq_offsets[int(db["seq"])])
        mask[off + int(db["tok_begin"]):off + int(db["tok_end"])] = True
    return int(mask.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dcpx", choices=["dcpx", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--transport", default="local", choices=["local", "nccl"],
                    help="block exchange: local = copy kernels over NVLink peer memory, nccl = send/recv")
    ap.add_argument("--opt", action="append", default=[],
                    help="executor option key=value (repeatable), e.g. bwd_window=8")
    ap.add_argument("--sm-reserve", type=int, default=-1,
                    help="SMs kept free of attention CTAs for transfer kernels (-1: executor default)")
    ap.add_argument("--placement", default="dcp", choices=["dcp", "ring", "zigzag"],
                    help="plan placement: DCP (default) or the paper's baselines (cfg2 only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="rank", choices=["rank", "single"],
                    help="N > 1 under torchrun: one process per GPU (rank) or one process owning all GPUs")

    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    N = args.gpus
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")

    def barrier():
        if dist is not None:
            dist.barrier()

    def reduce(x, op):
        """max / sum of a float over the ranks (identity without torch.distributed)."""
        if dist is None or not rank_mode:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
        return float(t.item())

    name = f"{args.config}_R{N}" if args.placement == "dcp" else f"{args.config}_{args.placement}_R{N}"
    metric = "masked attention fwd+bwd TFLOPS"
    workloads = {  # BASELINE.json configs[1..3] (synth seed 42 -> make_batches)
        "cfg2": ("causal, LongAlign-skewed 64K-token batch (6 seqs, 63,855 tokens)", 1024),
        "cfg3": ("lambda (sink 64 + window 4096), 128K-token batch (5 seqs, 130,968 tokens)", 1024),
        "cfg4_cb_B512": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 512),
        "cfg4_cb_B1024": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 1024),
        "cfg4_cb_B2048": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 2048),
        "cfg4_sq_B2048": ("shared-question (4 answers x 20 %), 128K-token batch", 2048),
        "cfg5": ("causal long-tail stress: one 512K-token sequence + 48 short seqs (634,880 tokens)", 4096),
        "cfg5_B8192": ("causal long-tail stress: one 512K-token sequence + 48 short seqs (634,880 tokens)", 8192),
    }
    desc, block = workloads.get(args.config, (args.config, None))
    config = {"workload": f"{args.config}: 8B-GPT attention layer (32 q / 8 kv heads, d 128), {desc}, "
                          f"block {block}, T 4, {args.placement.upper()} plan for {N} device(s)",
              "global_batch_tokens": None, "heads": "32/8", "block": block,
              "parallelism": f"{args.placement}{N}", "placement": args.placement,
              "l2": "inputs larger than L2"}

    if args.impl == "reference":
        if rank != 0:
            barrier()
            return
        bundle = load_bundle(name)
        config["global_batch_tokens"] = bundle.total_tokens
        vals = []
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(bundle, seconds_target=12.0 / max(1, (args.warmup + args.steps) / 4))
            if cb is None:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdcpref.so not built"}))
                barrier()
                return
            if i >= args.warmup:
                vals.append(cb)
        v = sum(c["value"] for c in vals) / len(vals)
        ms = 3.5 * bundle.total_flops / (v * 1e12) * 1e3
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "TFLOP/s", "n_gpus": N,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config,
                "cpu_baseline": {k: vals[-1][k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "TFLOP/s"},
                "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        barrier()
        return

    import torch

    rank_mode = world > 1 and args.mode == "rank"
    if world > 1 and not rank_mode and rank != 0:
        barrier()   # bundle ready
        barrier()   # timed region start
        barrier()   # timed region end
        return

    from paper_2510_10620_b200.executor import DCPExecutor

    bundle = load_bundle(name)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    config["global_batch_tokens"] = T
    F_fwd = bundle.total_flops
    F_total = 3.5 * F_fwd
    # (ranks beyond the GPUs present share them: a functional check of an N-rank plan on a
    # smaller box; such a run is not a valid measurement)
    ordinal = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count() if rank_mode else 0
    devs = [ordinal] if rank_mode else list(range(N))  # the GPUs this process drives
    torch.cuda.set_device(ordinal)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((T, H, 128), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((T, G, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((T, G, 128), device="cuda", generator=g).to(torch.bfloat16)
    d_o = torch.randn((T, H, 128), device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty((H, T), device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

    if rank_mode:
        if world != N:
            raise SystemExit("--mode rank needs --nproc-per-node == --gpus")
        ex = DCPExecutor(rank=rank, world=world, cuda_ordinal=ordinal)
        config["transport"] = "per-rank: CUDA IPC peer arenas, device-side flags"
    else:
        ex = DCPExecutor(list(range(N)), transport=args.transport)
        config["transport"] = args.transport
    config["processes"] = world if rank_mode else 1
    ex.set_option("kernel_timing", 1)
    if args.sm_reserve >= 0:
        ex.set_option("sm_reserve", args.sm_reserve)
    for kv in args.opt:
        key, _, val = kv.partition("=")
        ex.set_option(key, int(val))
    if args.opt:
        config["executor_options"] = ",".join(args.opt)
    ex.prepare(bundle)
    # N > 1: the distributed layout (dcpx_*_dev) -- every GPU holds the packed Q/K/V/dO of
    # the batch in its own HBM and receives the output rows it owns, as in a training step
    # where each GPU produced its own tokens; no input or output crosses NVLink.
    if N > 1 and not rank_mode:
        def per_dev(x, like=False):
            return [torch.empty_like(x, device=f"cuda:{d}") if like else x.to(f"cuda:{d}") for d in range(N)]
        io = dict(q=per_dev(q), k=per_dev(k), v=per_dev(v), d_o=per_dev(d_o), o=per_dev(o, True),
                  lse=per_dev(lse, True), dq=per_dev(dq, True), dk=per_dev(dk, True), dv=per_dev(dv, True))
    else:
        io = dict(q=q, k=k, v=v, d_o=d_o, o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    config["io_layout"] = ("per-rank packed buffers in each GPU's HBM" if rank_mode else
                           "per-device packed buffers (dcpx_*_dev)" if N > 1 else "packed buffers on cuda:0")
    barrier()

    def step():
        ex.load_inputs(io["q"], io["k"], io["v"])
        rf = ex.forward(io["o"], io["lse"])
        rb = ex.backward(io["d_o"], io["dq"], io["dk"], io["dv"])
        return rf, rb

    for _ in range(args.warmup):
        step()
    for d in devs:
        torch.cuda.synchronize(d)
    barrier()
    fwd_ms, bwd_ms, fwd_k, bwd_k, launches = [], [], [], [], 0
    with ClockSampler(list(range(min(N, torch.cuda.device_count()))) if rank == 0 else []) as clk:
        starts = {d: torch.cuda.Event(enable_timing=True) for d in devs}
        ends = {d: torch.cuda.Event(enable_timing=True) for d in devs}
        for d in devs:
            with torch.cuda.device(d):
                torch.cuda.synchronize(d)
                starts[d].record()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rf, rb = step()
            fwd_ms.append(rf["device_ms"]); bwd_ms.append(rb["device_ms"])
            fwd_k.append(rf["attn_ms_sum"]); bwd_k.append(rb["attn_ms_sum"])
            launches += rf["kernel_launches"] + rb["kernel_launches"] + 3 * len(devs)  # + q/k/v scatters
        for d in devs:
            with torch.cuda.device(d):
                ends[d].record()
                torch.cuda.synchronize(d)
        wall = time.perf_counter() - t0
        barrier()
    # executor events bracket each call on every device (max over devices); the torch events
    # on the default stream bracket the whole region per device; max over ranks
    total_ms = max(starts[d].elapsed_time(ends[d]) for d in devs)
    ms_step = reduce(max(total_ms / args.steps, (sum(fwd_ms) + sum(bwd_ms)) / args.steps), "max")
    wall = reduce(wall, "max")
    value = F_total / (ms_step * 1e-3) / 1e12
    if rank_mode:  # GPU-time in the kernels and launches summed over the ranks
        fwd_k = [reduce(sum(fwd_k) / len(fwd_k), "sum")]
        bwd_k = [reduce(sum(bwd_k) / len(bwd_k), "sum")]
        launches = int(reduce(launches, "sum"))

    # roofline of the dominant kernel (backward attention, K1b) and of the forward (K1):
    # algorithmic FLOPs of all launches / GPU-time summed over the devices' launches
    pk, src = peaks()
    peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    bwd_kernel_ms = sum(bwd_k) / len(bwd_k) or 1e-9
    fwd_kernel_ms = sum(fwd_k) / len(fwd_k) or 1e-9
    bwd_flops, fwd_flops = 2.5 * F_fwd, F_fwd
    dominant = "attn_bwd_kernel" if bwd_kernel_ms >= fwd_kernel_ms else "attn_fwd_kernel"
    if dominant == "attn_bwd_kernel":
        ach = bwd_flops / (bwd_kernel_ms * 1e-3) / 1e12
    else:
        ach = fwd_flops / (fwd_kernel_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{name}:{dominant}")
        except Exception:  # noqa: BLE001
            traffic = None
    roof = {"bound": "tensor", "kernel": dominant, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "traffic": traffic,
            "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)",
            "per_kernel": {"attn_fwd_kernel": {"gpu_ms": fwd_kernel_ms, "tflops": fwd_flops / (fwd_kernel_ms * 1e-3) / 1e12},
                           "attn_bwd_kernel": {"gpu_ms": bwd_kernel_ms, "tflops": bwd_flops / (bwd_kernel_ms * 1e-3) / 1e12}},
            "algorithmic": "F_fwd = 4*D*attended pairs per launch (blocks.hpp:191); bwd = 2.5*F_fwd"}
    if N > 1:
        # compute-or-NVLink roofline
        send_b, recv_b = bundle.bwd_bytes()
        B = [max(int(bundle.per_device_send[d]) + int(send_b[d]), int(bundle.per_device_recv[d]) + int(recv_b[d]))
             for d in range(N)]
        Fd = [3.5 * int(x) for x in bundle.dev_flops]
        t_roof = max(max(Fd) / (pk["bf16_tflops"] * 1e12), max(B) / 900e9)
        roof["plan_roofline_ms"] = t_roof * 1e3
        roof["plan_roofline_frac"] = t_roof * 1e3 / ms_step

    # end to end through the C ABI with host buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, d_o))
        hdq, hdk, hdv = (torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (q, k, v))
        def e2e_step():
            ex.load_inputs(hq, hk, hv)
            ex.forward(o, lse)
            ex.backward(hdo, hdq, hdk, hdv, host=True)
        # the host calls are asynchronous (double-buffered staging, uploads and downloads on
        # their own streams): with per-call timing off nothing blocks the host, so step
        # i+1's uploads and step i's downloads overlap step i's compute; wall clock around
        # the whole loop, synchronized at the end
        ex.set_option("timing", 0)
        ex.set_option("kernel_timing", 0)
        for _ in range(2):
            e2e_step()
        ex.synchronize()
        if rank_mode:
            barrier()
        t0 = time.perf_counter()
        ne = max(2, args.steps // 2)
        for _ in range(ne):
            e2e_step()
        ex.synchronize()
        e_ms = reduce((time.perf_counter() - t0) / ne * 1e3, "max")
        if rank_mode:  # each rank copies the token rows of its own plan device
            rows_q = sum(covered_tokens(bundle, d, "resident_q") for d in range(N))
            rows_kv = sum(covered_tokens(bundle, d, "resident_kv") for d in range(N))
        else:
            rows_q = rows_kv = T
        e2e = {"value": F_total / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": 2 * rows_q * H * 256 + 2 * rows_kv * G * 256,
               "d2h_bytes_per_step": rows_q * H * 256 + 2 * rows_kv * G * 256,
               "path": "dcpx_load_inputs_host + dcpx_forward + dcpx_backward_host (pinned host buffers, "
                       "asynchronous: uploads/downloads overlap compute across steps"
                       + ("; every rank copies only its plan device's token rows)" if rank_mode else ")")}

    cb = None
    if not args.no_cpu_baseline and N == 1:
        try:
            cb = cpu_baseline(bundle)
            if cb:
                cb = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # noqa: BLE001
            cb = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    line = {"metric": metric, "value": value, "unit": "TFLOP/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config, "roofline": roof, "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
            "detail": {"fwd_ms": sum(fwd_ms) / len(fwd_ms), "bwd_ms": sum(bwd_ms) / len(bwd_ms),
                       "F_fwd": F_fwd, "F_total": F_total, "wall_ms_per_step": wall / args.steps * 1e3,
                       "planned_fwd_bytes": int(bundle.volume[0])}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if rank_mode:
        barrier()  # no rank unmaps its arenas while a peer may still read them
    ex.close()


if __name__ == "__main__":
    main()
