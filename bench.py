"""bench.py — DCP executor fwd+bwd throughput on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[2], the config the metric is quoted on at 1/2/4/8
GPUs): 8B-GPT attention layer, 32 query / 8 KV heads, d 128, lambda mask (sink 64 + sliding
window 4096), LongAlign-like skewed 128K-token batch (synth seed 42, make_batches budget
131072, batch 0: 5 sequences, 130,968 tokens), block 1024, T = 4 divisions, planned by the
reference planner for R = N devices (plans/cfg3_R{N}.npz; planning is never timed). At
N = 1 the line also carries configs[1] (causal 64K batch, cfg2) under "secondary". One step =
load packed bf16 Q/K/V into the slot arenas + forward + backward of the whole plan. FLOPs
count only attended pairs: F_fwd = 4 * D * pairs (blocks.hpp:191), F_total = 3.5 * F_fwd.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dcpx|reference] [--config cfg3]

`value`: device time (CUDA events on the caller's stream, which every executor call joins
and releases -- dcpx.h stream contract) over K steps, max over ranks. `e2e`: the same steps
through the host-buffer calls (dcpx_load_inputs_host, dcpx_forward_host, dcpx_backward_host)
with pinned host buffers: Q/K/V/dO up and O/LSE/dQ/dK/dV down every step, wall clock.
N > 1 (launched by torchrun, default --mode rank): one process per GPU, rank r executes plan
device r (dcpx_create_rank: peer arenas mapped over CUDA IPC, transfers are pulls over
NVLink ordered by device-side flags). --mode single: rank 0's context owns all N devices.
"""
from __future__ import annotations

import argparse
import json
import os

# before torch creates a CUDA context (see paper_2510_10620_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import platform
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "masked attention fwd+bwd TFLOPS"
NVLINK_GBS = 900.0  # per direction per GPU (NVLink 5 / NVSwitch)

WORKLOADS = {  # BASELINE.json configs[1..4] (synth seed 42 -> make_batches)
    "cfg2": ("causal, LongAlign-skewed 64K-token batch (6 seqs, 63,855 tokens)", 1024),
    "cfg3": ("lambda (sink 64 + window 4096), LongAlign-skewed 128K-token batch (5 seqs, 130,968 tokens)", 1024),
    "cfg4_cb_B512": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 512),
    "cfg4_cb_B1024": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 1024),
    "cfg4_cb_B2048": ("causal-blockwise (256, 2, 1, 1), 128K-token batch", 2048),
    "cfg4_sq_B2048": ("shared-question (4 answers x 20 %), 128K-token batch", 2048),
    "cfg5": ("causal long-tail stress: one 512K-token sequence + 48 short seqs (634,880 tokens)", 4096),
    "cfg5_B8192": ("causal long-tail stress: one 512K-token sequence + 48 short seqs (634,880 tokens)", 8192),
}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return platform.processor() or "unknown"


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
        if self.gpus:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def load_bundle(name):
    from make_plans import load
    return load(name)


def config_of(name_cfg, placement, N, bundle=None):
    """The `config` object, identical in both arms (no implementation keys)."""
    desc, block = WORKLOADS.get(name_cfg, (name_cfg, None))
    return {"workload": f"{name_cfg}: 8B-GPT attention layer (32 q / 8 kv heads, d 128), {desc}, "
                        f"block {block}, T 4, {placement.upper()} plan for {N} device(s)",
            "global_batch_tokens": bundle.total_tokens if bundle is not None else None,
            "heads": "32/8", "head_dim": 128, "block": block, "parallelism": f"{placement}{N}",
            "placement": placement, "l2": "inputs larger than L2 (Q alone 0.5-1 GB per step)"}


def sample_items(bundle, seconds_target, threads):
    """Every k-th AttentionItem of the plan, sized for ~seconds_target of FP64 exec_attention
    on `threads` host threads (~1.6 GFLOP/s/core)."""
    import numpy as np
    items = []
    for dp in bundle.devices:
        for ins in dp.instructions():
            if ins["op"] == 0:
                items.append(dp.items[ins["offset"]: ins["offset"] + ins["count"]])
    items = np.concatenate(items)
    per_item = float(np.mean((items["q_end"] - items["q_begin"]) * (items["kv_end"] - items["kv_begin"])))
    budget_flops = seconds_target * threads * 1.5e9
    n = max(threads, min(len(items), int(budget_flops / (4 * 128 * per_item * 0.6))))
    stride = max(1, len(items) // n)
    return items[::stride][:n], len(items), stride


def cpu_baseline(bundle, q, k, v, seconds_target=15.0, check=True):
    """The reference executor's hot loop, exec_attention (simexec.hpp:33-76, FP64), on a
    deterministic sample of this plan's AttentionItems over all host threads, on the SAME
    bf16 inputs as the GPU run; each sampled item's (O, LSE = m + ln l) is compared with the
    GPU kernel's result for that item (PlanBundle.item_sample: the items executed one by one
    by K1 through the C ABI). Reported, not optimised."""
    import numpy as np
    import torch

    import oracle as O
    if not O.ref_available():
        return None
    threads = os.cpu_count() or 1
    sample, n_items, stride = sample_items(bundle, seconds_target, threads)
    G, H = bundle.G, bundle.H
    offs = bundle.seq_offsets
    work, flops = [], 0
    for it in sample:
        s, h = int(it["seq"]), int(it["head"])
        off = int(offs[s])
        rows = O.item_rows(bundle, s, int(it["q_begin"]), int(it["q_end"]), int(it["kv_begin"]), int(it["kv_end"]))
        grp = h * G // H
        qs = slice(off + int(it["q_begin"]), off + int(it["q_end"]))
        ks = slice(off + int(it["kv_begin"]), off + int(it["kv_end"]))
        work.append(dict(rows=rows, q=q[qs, h].double().cpu().numpy(), k=k[ks, grp].double().cpu().numpy(),
                         v=v[ks, grp].double().cpu().numpy()))
        flops += 4 * 128 * int(np.maximum(rows[:, 1] - rows[:, 0], 0).sum() + np.maximum(rows[:, 3] - rows[:, 2], 0).sum())
    outs, lses, sec = O.ref_run_items(work, 128, threads)
    res = {"value": flops / sec / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
           "cpu_model": cpu_model(), "nproc": os.cpu_count(),
           "sample": f"reference exec_attention (simexec.hpp:33-76, FP64; forward only: the reference has no "
                     f"backward) on {len(sample)} of {n_items} AttentionItems (every {stride}th), "
                     f"{flops / 1e9:.1f} GFLOP in {sec:.2f} s on {threads} host threads, same bf16 inputs as the GPU",
           "seconds": sec, "flops": flops}
    if check:
        from paper_2510_10620_b200.executor import DCPExecutor
        sb = bundle.item_sample(sample)
        with DCPExecutor([torch.cuda.current_device()]) as ex:
            ex.prepare(sb)
            ex.load_inputs(q, k, v)
            ex.forward()
            ex.synchronize()
            o_ar = ex.arena_view(0, 2, len(sample)).float()
            l_ar = ex.arena_view(0, 3, len(sample))
            num = den = lse_err = 0.0
            for i, (o_ref, l_ref) in enumerate(zip(outs, lses)):
                nq = o_ref.shape[0]
                og = o_ar[i, :nq].cpu().numpy()
                lg = l_ar[i, :nq].cpu().numpy()
                num = max(num, float(np.abs(og - o_ref).max()))
                den = max(den, float(np.abs(o_ref).max()))
                fin = np.isfinite(l_ref)
                assert np.array_equal(fin, np.isfinite(lg)), "LSE -inf pattern differs"
                if fin.any():
                    lse_err = max(lse_err, float(np.abs(lg[fin] - l_ref[fin]).max() / max(1.0, np.abs(l_ref[fin]).max())))
        o_err = num / (den or 1.0)
        res["check"] = {"items": len(sample), "o_max_rel_err": o_err, "lse_max_rel_err": lse_err,
                        "tolerance": {"o": 2e-2, "lse": 1e-3}, "ok": bool(o_err <= 2e-2 and lse_err <= 1e-3),
                        "gpu": "K1 attn_fwd_kernel on each sampled item alone (PlanBundle.item_sample)"}
    return res


def pcie_gbs(ordinal, nbytes=1 << 30):
    """Pinned host <-> device copy bandwidth of this GPU's link, both directions running
    concurrently (as in the e2e steps): (h2d GB/s, d2h GB/s)."""
    import torch
    hu = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    hd = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    du = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{ordinal}")
    dd = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{ordinal}")
    su, sd = torch.cuda.Stream(ordinal), torch.cuda.Stream(ordinal)
    res = []
    for _ in range(3):
        eu = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ed = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(su):
            eu[0].record(); du.copy_(hu, non_blocking=True); eu[1].record()
        with torch.cuda.stream(sd):
            ed[0].record(); hd.copy_(dd, non_blocking=True); ed[1].record()
        torch.cuda.synchronize(ordinal)
        res.append((nbytes / (eu[0].elapsed_time(eu[1]) * 1e-3) / 1e9, nbytes / (ed[0].elapsed_time(ed[1]) * 1e-3) / 1e9))
    return max(r[0] for r in res), max(r[1] for r in res)


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


def reference_arm(args, N, rank, barrier):
    """--impl reference: the reference's own CPU executor hot loop (exec_attention, FP64, all
    host threads) on bounded samples of the same workload; rank 0 only."""
    if rank != 0:
        barrier()
        return
    name = f"{args.config}_R{N}" if args.placement == "dcp" else f"{args.config}_{args.placement}_R{N}"
    bundle = load_bundle(name)
    import torch
    g = torch.Generator().manual_seed(0)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
    q = torch.randn((T, H, 128), generator=g).to(torch.bfloat16)
    k = torch.randn((T, G, 128), generator=g).to(torch.bfloat16)
    v = torch.randn((T, G, 128), generator=g).to(torch.bfloat16)
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(bundle, q, k, v, seconds_target=12.0 / max(1, (args.warmup + args.steps) / 4), check=False)
        if cb is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdcpref.so not built"}))
            barrier()
            return
        if i >= args.warmup:
            vals.append(cb)
    v_ = sum(c["value"] for c in vals) / len(vals)
    ms = 3.5 * bundle.total_flops / (v_ * 1e12) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v_, "unit": "TFLOP/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args.config, args.placement, N, bundle),
            "cpu_baseline": {k2: vals[-1][k2] for k2 in ("kind", "cores", "sample", "cpu_model", "nproc")}
            | {"value": v_, "unit": "TFLOP/s"},
            "e2e": {"value": v_, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "exec_attention throughput on sampled items; ms_per_step extrapolates it to the whole "
                    "step's F_total (the reference executes forward only)"}
    print(json.dumps(line), flush=True)
    barrier()


def measure(args, cfg_name, N, world, rank, rank_mode, barrier, reduce, steps, warmup, do_e2e, do_cpu,
            sample_clocks):
    import torch

    from paper_2510_10620_b200.executor import DCPExecutor
    name = f"{cfg_name}_R{N}" if args.placement == "dcp" else f"{cfg_name}_{args.placement}_R{N}"
    bundle = load_bundle(name)
    T, H, G = bundle.total_tokens, bundle.H, bundle.G
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
    run = {}
    if rank_mode:
        if world != N:
            raise SystemExit("--mode rank needs --nproc-per-node == --gpus")
        ex = DCPExecutor(rank=rank, world=world, cuda_ordinal=ordinal)
        run["transport"] = "per-rank: CUDA IPC peer arenas, device-side flags"
    else:
        ex = DCPExecutor(list(range(N)), transport=args.transport)
        run["transport"] = args.transport
    run["processes"] = world if rank_mode else 1
    if args.sm_reserve >= 0:
        ex.set_option("sm_reserve", args.sm_reserve)
    for kv in args.opt:
        key, _, val = kv.partition("=")
        ex.set_option(key, int(val))
    if args.opt:
        run["executor_options"] = ",".join(args.opt)
    ex.prepare(bundle)
    # N > 1 single-process: the distributed layout (dcpx_*_dev) -- every GPU holds the packed
    # inputs in its own HBM and receives the output rows it owns; no input or output crosses NVLink
    if N > 1 and not rank_mode:
        def per_dev(x, like=False):
            return [torch.empty_like(x, device=f"cuda:{d}") if like else x.to(f"cuda:{d}") for d in range(N)]
        io = dict(q=per_dev(q), k=per_dev(k), v=per_dev(v), d_o=per_dev(d_o), o=per_dev(o, True),
                  lse=per_dev(lse, True), dq=per_dev(dq, True), dk=per_dev(dk, True), dv=per_dev(dv, True))
    else:
        io = dict(q=q, k=k, v=v, d_o=d_o, o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    run["io_layout"] = ("per-rank packed buffers in each GPU's HBM" if rank_mode else
                        "per-device packed buffers (dcpx_*_dev)" if N > 1 else "packed buffers on cuda:0")
    barrier()

    def step():
        ex.load_inputs(io["q"], io["k"], io["v"])
        rf = ex.forward(io["o"], io["lse"])
        rb = ex.backward(io["d_o"], io["dq"], io["dk"], io["dv"])
        return rf, rb

    # kernel timing: CUDA events around every attention launch on its stream (executor option
    # kernel_timing = 2: accumulated without blocking the host, read after the timed region)
    ex.set_option("kernel_timing", args.kernel_timing)
    for _ in range(warmup):
        step()
    for d in devs:
        torch.cuda.synchronize(d)
    ex.kernel_times()  # drop the warm-up launches
    barrier()
    fwd_k, bwd_k, fwd_n, bwd_n, launches = [], [], [], [], 0
    with ClockSampler(list(range(min(N, torch.cuda.device_count()))) if (rank == 0 and sample_clocks) else []) as clk:
        starts = {d: torch.cuda.Event(enable_timing=True) for d in devs}
        ends = {d: torch.cuda.Event(enable_timing=True) for d in devs}
        for d in devs:
            with torch.cuda.device(d):
                torch.cuda.synchronize(d)
                starts[d].record()
        t0 = time.perf_counter()
        for _ in range(steps):
            rf, rb = step()
            if args.kernel_timing == 1:
                fwd_k.append(rf["attn_ms_sum"]); bwd_k.append(rb["attn_ms_sum"])
                fwd_n.append(rf["attn_launches"]); bwd_n.append(rb["attn_launches"])
            launches += rf["kernel_launches"] + rb["kernel_launches"] + 3 * len(devs)  # + q/k/v scatters
        for d in devs:
            with torch.cuda.device(d):
                ends[d].record()
                torch.cuda.synchronize(d)
        wall = time.perf_counter() - t0
        barrier()
    if args.kernel_timing == 2:
        kt = ex.kernel_times()
        fwd_k, bwd_k = [kt["fwd_ms_sum"] / steps], [kt["bwd_ms_sum"] / steps]
        fwd_n, bwd_n = [kt["fwd_launches"] / steps], [kt["bwd_launches"] / steps]
    ex.set_option("kernel_timing", 0)
    total_ms = max(starts[d].elapsed_time(ends[d]) for d in devs)
    ms_step = reduce(total_ms / steps, "max")
    wall = reduce(wall, "max")
    value = F_total / (ms_step * 1e-3) / 1e12
    if rank_mode:  # GPU-time in the kernels and launches summed over the ranks
        fwd_k = [reduce(sum(fwd_k) / len(fwd_k), "sum")]
        bwd_k = [reduce(sum(bwd_k) / len(bwd_k), "sum")]
        fwd_n = [reduce(sum(fwd_n) / len(fwd_n), "sum")]
        bwd_n = [reduce(sum(bwd_n) / len(bwd_n), "sum")]
        launches = int(reduce(launches, "sum"))

    # roofline of the dominant kernel: algorithmic FLOPs of its launches in one step
    # (F_fwd for K1, 2.5 F_fwd for K1b, summed over devices) / the GPU time of those launches
    pk, src = peaks()
    burst = pk["bf16_tflops"]
    sustained = pk.get("bf16_tflops_sustained", burst)
    bwd_kernel_ms = sum(bwd_k) / len(bwd_k) or 1e-9
    fwd_kernel_ms = sum(fwd_k) / len(fwd_k) or 1e-9
    # (kernel GPU time is summed over the N devices; its share is of N x the step time)
    per_kernel = {"attn_fwd_kernel": {"gpu_ms_per_step": fwd_kernel_ms, "launches_per_step": sum(fwd_n) / len(fwd_n),
                                      "tflops": F_fwd / (fwd_kernel_ms * 1e-3) / 1e12,
                                      "share_of_step": fwd_kernel_ms / (ms_step * N)},
                  "attn_bwd_kernel": {"gpu_ms_per_step": bwd_kernel_ms, "launches_per_step": sum(bwd_n) / len(bwd_n),
                                      "tflops": 2.5 * F_fwd / (bwd_kernel_ms * 1e-3) / 1e12,
                                      "share_of_step": bwd_kernel_ms / (ms_step * N)}}
    dominant = "attn_bwd_kernel" if bwd_kernel_ms >= fwd_kernel_ms else "attn_fwd_kernel"
    ach = per_kernel[dominant]["tflops"]
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(f"{name}:{dominant}")
            if t:
                traffic = t["bytes_per_launch"] if isinstance(t, dict) else t
        except Exception:  # noqa: BLE001
            traffic = None
    roof = {"bound": "tensor", "kernel": dominant, "achieved": ach, "peak": burst, "unit": "TFLOP/s",
            "frac": ach / burst, "frac_sustained": ach / sustained, "peak_sustained": sustained,
            "traffic": traffic,
            "peak_source": f"{src}: bf16_tflops (burst) and bf16_tflops_sustained",
            "per_kernel": per_kernel,
            "step_frac": value / burst / max(1, N),
            "algorithmic": "F_fwd = 4*D*attended pairs (blocks.hpp:191) per forward pass of K1; K1b = 2.5*F_fwd; "
                           "traffic = ncu dram bytes read+write per launch (profiles/traffic.json)"}
    if N > 1:
        # compute-or-NVLink roofline: planned bytes (CommVolume + the
        # backward formula) and the bytes the transfers actually move (wire)
        send_b, recv_b = bundle.bwd_bytes()
        (wfs, wfr), (wbs, wbr) = bundle.wire_bytes()
        B = [max(int(bundle.per_device_send[d]) + int(send_b[d]), int(bundle.per_device_recv[d]) + int(recv_b[d]))
             for d in range(N)]
        W = [max(int(wfs[d]) + int(wbs[d]), int(wfr[d]) + int(wbr[d])) for d in range(N)]
        Fd = [3.5 * int(x) for x in bundle.dev_flops]
        t_comp = max(Fd) / (burst * 1e12)
        t_roof = max(t_comp, max(B) / (NVLINK_GBS * 1e9))
        t_wire = max(t_comp, max(W) / (NVLINK_GBS * 1e9))
        roof["plan_roofline_ms"] = t_roof * 1e3
        roof["plan_roofline_frac"] = t_roof * 1e3 / ms_step
        roof["plan_roofline_wire_ms"] = t_wire * 1e3
        roof["plan_roofline_wire_frac"] = t_wire * 1e3 / ms_step
        roof["max_device_planned_bytes"] = max(B)
        roof["max_device_wire_bytes"] = max(W)

    # end to end through the C ABI with host buffers (pinned): H2D of Q/K/V/dO and D2H of
    # O/LSE/dQ/dK/dV inside the timed region, every step
    e2e = None
    if do_e2e:
        hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, d_o))
        ho, hdq = (torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (q, q))
        hdk, hdv = (torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (k, v))
        hlse = torch.empty((H, T), dtype=torch.float32).pin_memory()

        def e2e_step():
            ex.load_inputs(hq, hk, hv)
            ex.forward(ho, hlse, host=True)
            ex.backward(hdo, hdq, hdk, hdv, host=True)
        # the host calls are asynchronous (double-buffered device staging, uploads and
        # downloads on their own streams), so step i+1's uploads and step i's downloads
        # overlap step i's compute; wall clock around the loop, synchronized at the end
        for _ in range(2):
            e2e_step()
        ex.synchronize()
        if rank_mode:
            barrier()
        t0 = time.perf_counter()
        ne = max(2, steps // 2)
        for _ in range(ne):
            e2e_step()
        ex.synchronize()
        e_ms = reduce((time.perf_counter() - t0) / ne * 1e3, "max")
        if rank_mode:  # each rank copies the token rows of its own plan device
            rows_q = sum(covered_tokens(bundle, d, "resident_q") for d in range(N))
            rows_kv = sum(covered_tokens(bundle, d, "resident_kv") for d in range(N))
            rows_o = sum(covered_tokens(bundle, d, "resident_o") for d in range(N))
        else:
            rows_q = rows_kv = rows_o = T
        # PCIe roofline of the e2e step: the same byte counts at the pinned-copy bandwidth of
        # this box, measured here in both directions at once (the steps overlap them)
        h2d_b = 2 * rows_q * H * 256 + 2 * rows_kv * G * 256
        d2h_b = rows_o * H * (256 + 4) + rows_q * H * 256 + 2 * rows_kv * G * 256
        up_gbs, down_gbs = pcie_gbs(ordinal)
        pcie_ms = max(h2d_b / (up_gbs * 1e9), d2h_b / (down_gbs * 1e9)) * 1e3
        e2e = {"value": F_total / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
               "pcie_gbs_measured": {"h2d": up_gbs, "d2h": down_gbs, "how": "1 GiB pinned copies, both directions at once"},
               "pcie_bound_ms": pcie_ms, "pcie_frac": pcie_ms / e_ms,
               "h2d_bytes_per_step": h2d_b,   # Q, dO; K, V
               "d2h_bytes_per_step": d2h_b,   # O + LSE; dQ; dK, dV
               "path": "dcpx_load_inputs_host + dcpx_forward_host + dcpx_backward_host (pinned host buffers; "
                       "asynchronous: uploads/downloads overlap compute across steps"
                       + ("; every rank copies only its plan device's token rows)" if rank_mode else ")")}

    cb = None
    if do_cpu:
        try:
            cb = cpu_baseline(bundle, q, k, v)
            if cb:
                cb = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample", "cpu_model", "nproc", "check")
                      if k2 in cb}
        except Exception as e:  # noqa: BLE001
            cb = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e!r}"}
    res = dict(name=name, value=value, ms_step=ms_step, wall=wall, launches=launches, roof=roof, e2e=e2e, cb=cb,
               clocks=clk.summary(), run=run, bundle=bundle, F_fwd=F_fwd, F_total=F_total)
    if rank_mode:
        barrier()  # no rank unmaps its arenas while a peer may still read them
    ex.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dcpx", choices=["dcpx", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--secondary", default="cfg2",
                    help="second config measured at N = 1 and reported under 'secondary' ('' to skip)")
    ap.add_argument("--transport", default="local", choices=["local", "nccl"],
                    help="block exchange: local = copy kernels over NVLink peer memory, nccl = send/recv")
    ap.add_argument("--opt", action="append", default=[],
                    help="executor option key=value (repeatable), e.g. bwd_window=8")
    ap.add_argument("--sm-reserve", type=int, default=-1,
                    help="SMs kept free of attention CTAs for transfer kernels (-1: executor default)")
    ap.add_argument("--placement", default="dcp", choices=["dcp", "ring", "zigzag"],
                    help="plan placement: DCP (default) or the paper's baselines (cfg2 only)")
    ap.add_argument("--kernel-timing", type=int, default=2, choices=[1, 2],
                    help="attention-launch events: 2 = read after the timed region (default), "
                         "1 = read at the end of every call (blocks the host each step)")
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
    rank_mode = world > 1 and args.mode == "rank"

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

    if args.impl == "reference":
        reference_arm(args, N, rank, barrier)
        return
    if world > 1 and not rank_mode and rank != 0:
        barrier()   # bundle ready
        barrier()   # timed region start
        barrier()   # timed region end
        return

    r = measure(args, args.config, N, world, rank, rank_mode, barrier, reduce, args.steps, args.warmup,
                do_e2e=not args.no_e2e, do_cpu=(not args.no_cpu_baseline and N == 1), sample_clocks=True)
    secondary = None
    if args.secondary and N == 1 and args.secondary != args.config and args.placement == "dcp":
        s = measure(args, args.secondary, N, world, rank, rank_mode, barrier, reduce, max(3, args.steps // 2),
                    args.warmup, do_e2e=not args.no_e2e, do_cpu=False, sample_clocks=True)
        secondary = {args.secondary: {"value": s["value"], "unit": "TFLOP/s", "ms_per_step": s["ms_step"],
                                      "config": config_of(args.secondary, args.placement, N, s["bundle"]),
                                      "roofline": {k2: s["roof"][k2] for k2 in ("kernel", "achieved", "frac",
                                                                                "frac_sustained", "per_kernel")},
                                      "e2e": s["e2e"], "clocks": s["clocks"], "gpu_launches": s["launches"]}}
    line = {"metric": METRIC, "value": r["value"], "unit": "TFLOP/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) bf16 Q/K/V/dO)",
            "config": config_of(args.config, args.placement, N, r["bundle"]), "roofline": r["roof"],
            "cpu_baseline": r["cb"], "e2e": r["e2e"], "gpu_launches": r["launches"], "clocks": r["clocks"],
            "run": r["run"],
            "detail": {"F_fwd": r["F_fwd"], "F_total": r["F_total"], "wall_ms_per_step": r["wall"] / args.steps * 1e3,
                       "planned_fwd_bytes": int(r["bundle"].volume[0])},
            "secondary": secondary}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
