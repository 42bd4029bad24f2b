"""Python mirror of the DCP executor interface over the C ABI (include/dcpx.h).

The paper's user-facing API is ``DCPExecutor(group).prepare(plan)`` plus
``DCPAttn.apply(executor, q, kv)``; the reference's executor entry
point is ``dcp::run(plans, g, payload, topo, opts) -> SimResult`` (simexec.hpp:207-209).
This module exposes both shapes on top of ``libdcpx.so``:

* :class:`DCPExecutor` — ``prepare(bundle)``, ``load_inputs(q, k, v)``, ``forward()``,
  ``backward(d_o)`` on packed bf16 CUDA tensors (token-major ``[T, H, D]`` / ``[T, G, D]``).
* :func:`run` — the reference-shaped convenience call returning outputs + report.

There is no CPU fallback: importing works without a GPU, but every compute call goes
through the sm_100a library and raises if it is missing or fails.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

from . import plans as P

_HERE = os.path.dirname(os.path.abspath(__file__))
# DCPX_LIB: an experiment build (tools/build.py DCPX_VARIANT) instead of the product library
LIB_PATH = os.environ.get("DCPX_LIB") or os.path.join(_HERE, "libdcpx.so")

STATUS = {0: "OK", 1: "Error", 2: "DeadlockError", 3: "TagMismatchError", 4: "BufferOverflowError",
          5: "InfeasibleError", 6: "CudaError", 7: "Unsupported"}

# Every symbol include/dcpx.h declares (checked by tests/test_boundary_cpu.py).
EXPORTS = ["dcpx_create", "dcpx_create_rank", "dcpx_rank_export", "dcpx_rank_connect", "dcpx_prepare",
           "dcpx_load_inputs", "dcpx_load_inputs_host", "dcpx_forward", "dcpx_forward_host",
           "dcpx_backward", "dcpx_backward_host", "dcpx_load_inputs_dev", "dcpx_forward_dev",
           "dcpx_backward_dev", "dcpx_synchronize", "dcpx_set_streams", "dcpx_check_plans", "dcpx_kernel_times",
           "dcpx_debug_arena", "dcpx_set_option", "dcpx_trace", "dcpx_last_error", "dcpx_version",
           "dcpx_destroy"]


class DCPXError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libdcpx.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.dcpx_last_error.restype = C.c_char_p
        L.dcpx_version.restype = C.c_char_p
        for name in ("dcpx_create", "dcpx_create_rank", "dcpx_rank_export", "dcpx_rank_connect", "dcpx_prepare",
                     "dcpx_load_inputs", "dcpx_load_inputs_host", "dcpx_forward",
                     "dcpx_forward_host", "dcpx_backward", "dcpx_backward_host",
                     "dcpx_load_inputs_dev", "dcpx_forward_dev", "dcpx_backward_dev",
                     "dcpx_synchronize", "dcpx_debug_arena", "dcpx_set_option", "dcpx_set_streams",
                     "dcpx_check_plans", "dcpx_kernel_times"):
            getattr(L, name).restype = C.c_int
        L.dcpx_set_streams.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.dcpx_kernel_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_check_plans.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64]
        L.dcpx_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
        L.dcpx_create_rank.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.dcpx_rank_export.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.dcpx_rank_connect.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.dcpx_prepare.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_load_inputs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_load_inputs_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_forward_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        L.dcpx_backward_host.argtypes = L.dcpx_backward.argtypes
        L.dcpx_load_inputs_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_forward_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.dcpx_backward_dev.argtypes = L.dcpx_backward.argtypes
        L.dcpx_synchronize.argtypes = [C.c_void_p]
        L.dcpx_debug_arena.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_int64)]
        L.dcpx_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.dcpx_last_error.argtypes = [C.c_void_p]
        L.dcpx_destroy.argtypes = [C.c_void_p]
        L.dcpx_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.dcpx_trace.restype = C.c_int
        _lib = L
    return _lib


def _report_dict(r: P.c_report) -> dict:
    n = r.devices
    return dict(devices=n, stages=r.stages, total_bytes=int(r.total_bytes),
                total_flops=int(r.total_flops), per_device_send=[int(x) for x in r.per_device_send[:n]],
                per_device_recv=[int(x) for x in r.per_device_recv[:n]], wire_bytes=int(r.wire_bytes),
                makespan=r.makespan, device_ms=r.device_ms, kernel_launches=r.kernel_launches,
                attn_launches=r.attn_launches, attn_ms=r.attn_ms, attn_ms_sum=r.attn_ms_sum,
                wire_per_device_send=[int(x) for x in r.wire_per_device_send[:n]],
                wire_per_device_recv=[int(x) for x in r.wire_per_device_recv[:n]],
                units=int(r.units), windowed=int(r.windowed))


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _ptrs(ts):
    """void* array (one entry per plan device) for the dcpx_*_dev calls; None -> NULL."""
    if ts is None:
        return None
    return (C.c_void_p * len(ts))(*[None if t is None else t.data_ptr() for t in ts])


class DCPExecutor:
    """One context executing the plans of `bundle`.

    devices: CUDA ordinals, one per plan device (one process). Several plan devices may
    share one GPU (single-GPU emulation of an R-device plan). transport: "local" (copy
    kernels reading peer memory over NVLink) or "nccl" (NCCL send/recv per message, one
    GPU per plan device).
    ``rank``/``world``/``cuda_ordinal`` select the one-process-per-GPU mode
    (dcpx_create_rank): this process executes plan device ``rank``; ``prepare`` takes the
    whole bundle and exchanges arena handles with the other ranks through
    ``torch.distributed`` (initialised by the caller; any backend). Every rank must make
    the same sequence of calls. Usable as a context manager (``with DCPExecutor(...) as
    ex:``) to release device memory deterministically."""

    def __init__(self, devices: Optional[Sequence[int]] = None, rank: Optional[int] = None,
                 world: Optional[int] = None, cuda_ordinal: int = 0, transport: str = "local"):
        self._h = C.c_void_p()
        self.rank = rank
        if rank is not None:
            self._check(lib().dcpx_create_rank(rank, world, cuda_ordinal, C.byref(self._h)), create=True)
            self.ndev = world
            self.ordinals = [cuda_ordinal] * world
        else:
            devices = list(devices or [0])
            arr = (C.c_int * len(devices))(*devices)
            tr = {"local": 0, "p2p": 0, "nccl": 1}[transport]  # dcpx_transport
            self._check(lib().dcpx_create(len(devices), arr, tr, C.byref(self._h)), create=True)
            self.ndev = len(devices)
            self.ordinals = devices
        self.bundle: Optional[P.PlanBundle] = None
        self._keep = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().dcpx_destroy(self._h)
            self._h = C.c_void_p()

    def _check(self, rc: int, create: bool = False):
        if rc != 0:
            msg = lib().dcpx_last_error(None if create else self._h).decode()
            raise DCPXError(rc, msg)

    def set_option(self, key: str, value: int):
        self._check(lib().dcpx_set_option(self._h, key.encode(), int(value)))

    # -- DCPExecutor.prepare(execution_plan)
    def prepare(self, bundle: P.PlanBundle):
        keep, g, m, pv = bundle.c_views()
        self._check(lib().dcpx_prepare(self._h, len(pv), pv, C.byref(g), C.byref(m)))
        self.bundle = bundle
        self._keep = (keep, g, m, pv)
        if self.rank is not None:
            self._connect()

    def _connect(self):
        """All-gathers the arena handle blobs of the ranks and maps the peers' arenas."""
        import torch.distributed as dist
        size = C.c_int64()
        self._check(lib().dcpx_rank_export(self._h, None, 0, C.byref(size)))
        blob = C.create_string_buffer(size.value)
        self._check(lib().dcpx_rank_export(self._h, blob, size.value, C.byref(size)))
        blobs = [None] * self.ndev
        dist.all_gather_object(blobs, blob.raw)
        allb = C.create_string_buffer(b"".join(blobs), size.value * self.ndev)
        self._check(lib().dcpx_rank_connect(self._h, allb, size.value))
        dist.barrier()  # every rank mapped every arena before anyone runs

    def _streams(self):
        """Orders the next call after torch's current stream on every plan device's GPU and
        makes that stream wait for the call (dcpx.h stream contract)."""
        import torch
        cur = {o: torch.cuda.current_stream(o).cuda_stream for o in set(self.ordinals)}
        arr = (C.c_void_p * self.ndev)(*[cur[o] for o in self.ordinals])
        self._check(lib().dcpx_set_streams(self._h, self.ndev, arr))

    # Tensors, or lists with one tensor per plan device in that device's own memory
    # (the distributed layout: dcpx_*_dev; device d touches only the rows it owns).
    def load_inputs(self, q, k, v):
        self._streams()
        if isinstance(q, (list, tuple)):
            self._check(lib().dcpx_load_inputs_dev(self._h, _ptrs(q), _ptrs(k), _ptrs(v)))
        elif q.is_cuda:
            self._check(lib().dcpx_load_inputs(self._h, _ptr(q), _ptr(k), _ptr(v)))
        else:
            self._check(lib().dcpx_load_inputs_host(self._h, _ptr(q), _ptr(k), _ptr(v)))

    def forward(self, o=None, lse=None, host: bool = False) -> dict:
        self._streams()
        rep = P.c_report()
        if isinstance(o, (list, tuple)) or isinstance(lse, (list, tuple)):
            self._check(lib().dcpx_forward_dev(self._h, _ptrs(o), _ptrs(lse), C.byref(rep)))
            return _report_dict(rep)
        fn = lib().dcpx_forward_host if host else lib().dcpx_forward
        self._check(fn(self._h, _ptr(o), _ptr(lse), C.byref(rep)))
        return _report_dict(rep)

    def backward(self, d_o, dq, dk, dv, host: bool = False) -> dict:
        self._streams()
        rep = P.c_report()
        if isinstance(d_o, (list, tuple)):
            self._check(lib().dcpx_backward_dev(self._h, _ptrs(d_o), _ptrs(dq), _ptrs(dk), _ptrs(dv),
                                                C.byref(rep)))
            return _report_dict(rep)
        fn = lib().dcpx_backward_host if host else lib().dcpx_backward
        self._check(fn(self._h, _ptr(d_o), _ptr(dq), _ptr(dk), _ptr(dv), C.byref(rep)))
        return _report_dict(rep)

    def synchronize(self):
        self._check(lib().dcpx_synchronize(self._h))

    def kernel_times(self) -> dict:
        """Attention-kernel GPU time since the last read (option kernel_timing = 2):
        fwd/bwd ms summed over this context's devices and max over devices, launch counts."""
        ms = (C.c_double * 4)()
        n = (C.c_int32 * 2)()
        self._check(lib().dcpx_kernel_times(self._h, ms, n))
        return dict(fwd_ms_sum=ms[0], bwd_ms_sum=ms[1], fwd_ms_max=ms[2], bwd_ms_max=ms[3],
                    fwd_launches=n[0], bwd_launches=n[1])

    def trace(self):
        """Op spans of the last call when option "trace" is set: list of dicts."""
        import numpy as np
        n = lib().dcpx_trace(self._h, None, 0)
        buf = np.zeros((max(n, 1), 7))
        lib().dcpx_trace(self._h, buf.ctypes.data, n)
        kinds = ["attn", "merge", "copy", "launch", "wait", "nop", "xfer"]
        return [dict(dev=int(r[0]), instr=int(r[1]), kind=kinds[int(r[2])], division=int(r[3]),
                     pass_="bwd" if r[4] else "fwd", start=r[5], end=r[6]) for r in buf[:n]]

    def arena(self, dev: int, kind: int):
        ptr, rows = C.c_void_p(), C.c_int64()
        self._check(lib().dcpx_debug_arena(self._h, dev, kind, C.byref(ptr), C.byref(rows)))
        return ptr.value, rows.value

    def arena_view(self, dev: int, kind: int, slots: int):
        """torch view (no copy) of the first `slots` slots of an arena of plan device `dev`:
        kind 0 Q / 2 O -> bf16 [slots, slot_rows, 128]; 1 KV -> bf16 [slots, 2, slot_rows, 128];
        3 LSE -> fp32 [slots, slot_rows] (natural log). Introspection (dcpx_debug_arena)."""
        import torch
        ptr, rows = self.arena(dev, kind)
        shape = {0: (slots, rows, 128), 1: (slots, 2, rows, 128), 2: (slots, rows, 128), 3: (slots, rows)}[kind]

        class _CAI:
            __cuda_array_interface__ = {"shape": shape, "typestr": "<f4" if kind == 3 else "<i2",
                                        "data": (ptr, False), "version": 3}
        t = torch.as_tensor(_CAI(), device=f"cuda:{self.ordinals[dev]}")
        return t if kind == 3 else t.view(torch.bfloat16)


def check_plans(bundle: P.PlanBundle) -> None:
    """Host-only verification of a bundle's plans (dcpx_check_plans: verify_plans plus the
    lockstep deadlock / tag replay); raises DCPXError with the reference's exception kind.
    Needs no GPU."""
    keep, g, m, pv = bundle.c_views()
    err = C.create_string_buffer(4096)
    rc = lib().dcpx_check_plans(len(pv), pv, C.byref(g), C.byref(m), err, 4096)
    del keep
    if rc != 0:
        raise DCPXError(rc, err.value.decode())


def run(bundle: P.PlanBundle, q, k, v, devices: Optional[Sequence[int]] = None):
    """Reference-shaped call (simexec.hpp:207): executes all plans of `bundle` on the
    given CUDA devices and returns (o [T,H,D] bf16, lse [H,T] fp32, report)."""
    import torch
    ex = DCPExecutor(devices or [q.device.index or 0] * bundle.R)
    ex.prepare(bundle)
    ex.load_inputs(q, k, v)
    T, H, D = bundle.total_tokens, bundle.H, bundle.D
    o = torch.zeros((T, H, D), dtype=torch.bfloat16, device=q.device)
    lse = torch.full((H, T), float("-inf"), dtype=torch.float32, device=q.device)
    rep = ex.forward(o, lse)
    ex.synchronize()
    ex.close()
    return o, lse, rep
