"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracle.

``liboracle.so``  : plain-C FP64 restatement of the reference executor (dcp_oracle.c).
``libdcpref.so``  : the reference executor itself (oracle/_ref, built from /root/reference).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
leg may import this package; the product (paper_2510_10620_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(_HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libdcpref.so")

_orc = None
_ref = None


class OracleReport(C.Structure):
    _fields_ = [("total_bytes", C.c_uint64), ("total_flops", C.c_uint64),
                ("per_device_send", C.c_uint64 * 64), ("per_device_recv", C.c_uint64 * 64),
                ("comm_bytes", C.c_uint64 * (64 * 64 * 8)), ("comp_flops", C.c_uint64 * (8 * 64)),
                ("stages", C.c_int32), ("devices", C.c_int32)]


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"oracle not built: {ORACLE_LIB}")
        _orc = C.CDLL(ORACLE_LIB)
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise RuntimeError(f"reference shim not built: {REF_LIB}")
        _ref = C.CDLL(REF_LIB)
        _ref.dcpr_last_error.restype = C.c_char_p
    return _ref


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- restatement -------------------------------------------------------------------
def exec_attention(q, k, v, rows):
    """simexec.hpp:33-76 restated. rows int32 [n_q, 4] relative to the kv tile."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    rows = np.ascontiguousarray(rows, np.int32)
    nq, D = q.shape
    nk = k.shape[0]
    out = np.zeros((nq, D))
    m = np.zeros(nq)
    l = np.zeros(nq)
    rc = orc().orc_exec_attention(_p(q), _p(k), _p(v), nq, nk, D, _p(rows), _p(out), _p(m), _p(l))
    if rc:
        raise ValueError("exec_attention: range outside kv tile")
    return out, m, l


def exec_reduction(parts):
    """simexec.hpp:80-111 restated. parts = [(out, m, l), ...]."""
    n = len(parts)
    rows, D = parts[0][0].shape
    keep = [(_f64(o), _f64(m), _f64(l)) for o, m, l in parts]
    outs = (C.c_void_p * n)(*[o.ctypes.data for o, _, _ in keep])
    ms = (C.c_void_p * n)(*[m.ctypes.data for _, m, _ in keep])
    ls = (C.c_void_p * n)(*[l.ctypes.data for _, _, l in keep])
    out = np.zeros((rows, D))
    m = np.zeros(rows)
    l = np.zeros(rows)
    orc().orc_exec_reduction(n, outs, ms, ls, rows, D, _p(out), _p(m), _p(l))
    return out, m, l


def item_rows(bundle, seq, q_begin, q_end, kv_begin, kv_end):
    """plan.hpp:231-242 restated over the bundle's flattened masks."""
    keep, g, mview, _ = bundle.c_views([])
    out = np.zeros((q_end - q_begin, 4), np.int32)
    orc().orc_item_rows(C.byref(mview), C.c_int(seq), C.c_int64(q_begin), C.c_int64(q_end),
                        C.c_int64(kv_begin), C.c_int64(kv_end), _p(out))
    return out


def run(bundle, q, k, v, numeric=True, devices=None):
    """run (simexec.hpp:207-423) restated over the flat plans. Returns (o, lse, report,
    status, message); o [T][H][D], lse [H][T]."""
    keep, g, mview, pv = bundle.c_views(devices)
    T, H, D = bundle.total_tokens, bundle.H, bundle.D
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros((T, H, D))
    lse = np.zeros((H, T))
    rep = OracleReport()
    err = C.create_string_buffer(1024)
    st = orc().orc_run(len(pv), pv, C.byref(g), C.byref(mview), _p(q), _p(k), _p(v), _p(o),
                       _p(lse), C.byref(rep), 1 if numeric else 0, err, 1024)
    return o, lse, rep, st, err.value.decode()


def dense_forward(bundle, q, k, v):
    keep, g, mview, _ = bundle.c_views([])
    T, H, D = bundle.total_tokens, bundle.H, bundle.D
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros((T, H, D))
    lse = np.zeros((H, T))
    orc().orc_dense_forward(C.byref(g), C.byref(mview), _p(q), _p(k), _p(v), _p(o), _p(lse))
    return o, lse


def dense_backward(bundle, q, k, v, d_o):
    keep, g, mview, _ = bundle.c_views([])
    T, H, G, D = bundle.total_tokens, bundle.H, bundle.G, bundle.D
    q, k, v, d_o = _f64(q), _f64(k), _f64(v), _f64(d_o)
    dq = np.zeros((T, H, D))
    dk = np.zeros((T, G, D))
    dv = np.zeros((T, G, D))
    orc().orc_dense_backward(C.byref(g), C.byref(mview), _p(q), _p(k), _p(v), _p(d_o), _p(dq),
                             _p(dk), _p(dv))
    return dq, dk, dv


# ---- the reference itself -------------------------------------------------------------
def _specs_c(specs):
    from paper_2510_10620_b200.planner import SeqSpecC
    return (SeqSpecC * len(specs))(*[s.to_c() for s in specs])


def ref_plan_run(specs, H, G, D, devices, block_size, q, k, v, divisions=4, eps=(0.4, 0.1, 0.05),
                 seed=0):
    """plan_batch + run of the reference (FP64). Returns (o, stats dict, seconds)."""
    from paper_2510_10620_b200.planner import CfgC
    cfg = CfgC()
    cfg.machines, cfg.devices_per_machine, cfg.divisions = 1, devices, divisions
    cfg.block_size = block_size
    cfg.eps_inter, cfg.eps_intra, cfg.eps_data = eps
    cfg.seed = seed
    T = sum(s.length for s in specs)
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros((T, H, D))
    stats = np.zeros(2 + 2 * devices, np.uint64)
    sec, mk = C.c_double(), C.c_double()
    rc = ref().dcpr_plan_run(_specs_c(specs), len(specs), H, G, D, C.byref(cfg), _p(q), _p(k),
                             _p(v), _p(o), _p(stats), C.byref(sec), C.byref(mk))
    if rc:
        raise RuntimeError(f"reference run failed ({rc}): {ref().dcpr_last_error().decode()}")
    return o, dict(total_bytes=int(stats[0]), total_flops=int(stats[1]),
                   send=stats[2:2 + devices].copy(), recv=stats[2 + devices:].copy(),
                   makespan=mk.value), sec.value


def ref_make_payload(specs, H, G, D, seed):
    T = sum(s.length for s in specs)
    q = np.zeros((T, H, D))
    k = np.zeros((T, G, D))
    v = np.zeros((T, G, D))
    rc = ref().dcpr_make_payload(_specs_c(specs), len(specs), H, G, D, C.c_uint64(seed), _p(q),
                                 _p(k), _p(v))
    if rc:
        raise RuntimeError(ref().dcpr_last_error().decode())
    return q, k, v


def ref_exec_attention(q, k, v, rows):
    q, k, v = _f64(q), _f64(k), _f64(v)
    rows = np.ascontiguousarray(rows, np.int32)
    nq, D = q.shape
    out = np.zeros((nq, D))
    m = np.zeros(nq)
    l = np.zeros(nq)
    rc = ref().dcpr_exec_attention(_p(q), _p(k), _p(v), nq, k.shape[0], D, _p(rows), _p(out),
                                   _p(m), _p(l))
    if rc:
        raise ValueError(ref().dcpr_last_error().decode())
    return out, m, l


def ref_exec_reduction(parts):
    n = len(parts)
    rows, D = parts[0][0].shape
    keep = [(_f64(o), _f64(m), _f64(l)) for o, m, l in parts]
    outs = (C.c_void_p * n)(*[o.ctypes.data for o, _, _ in keep])
    ms = (C.c_void_p * n)(*[m.ctypes.data for _, m, _ in keep])
    ls = (C.c_void_p * n)(*[l.ctypes.data for _, _, l in keep])
    out = np.zeros((rows, D))
    m = np.zeros(rows)
    l = np.zeros(rows)
    ref().dcpr_exec_reduction(n, outs, ms, ls, rows, D, _p(out), _p(m), _p(l))
    return out, m, l


def ref_dense_attention(specs, H, G, D, q, k, v):
    T = sum(s.length for s in specs)
    q, k, v = _f64(q), _f64(k), _f64(v)
    o = np.zeros((T, H, D))
    rc = ref().dcpr_dense_attention(_specs_c(specs), len(specs), H, G, D, _p(q), _p(k), _p(v),
                                    _p(o))
    if rc:
        raise RuntimeError(ref().dcpr_last_error().decode())
    return o


def ref_time_tiles(count, nq, nk, D, rows, threads):
    """Reference exec_attention on `count` identical tiles over `threads` host threads."""
    rows = np.ascontiguousarray(rows, np.int32)
    sec = C.c_double()
    rc = ref().dcpr_time_tiles(count, nq, nk, D, _p(rows), threads, C.byref(sec))
    if rc:
        raise RuntimeError(ref().dcpr_last_error().decode())
    return sec.value


def ref_time_items(nq, nk, row_off, rows, D, threads):
    """Reference exec_attention over sampled items (CPU baseline). Returns seconds."""
    nq = np.ascontiguousarray(nq, np.int32)
    nk = np.ascontiguousarray(nk, np.int32)
    row_off = np.ascontiguousarray(row_off, np.int64)
    rows = np.ascontiguousarray(rows, np.int32)
    sec = C.c_double()
    rc = ref().dcpr_time_items(len(nq), _p(nq), _p(nk), _p(row_off), _p(rows), D, threads,
                               C.byref(sec))
    if rc:
        raise RuntimeError(ref().dcpr_last_error().decode())
    return sec.value


def ref_run_items(items, D, threads):
    """Reference exec_attention (simexec.hpp:33-76) on `items`, a list of dicts with
    nq, nk, rows [nq, 4] (kv-tile-relative) and q [nq, D], k, v [nk, D] float64 inputs, on
    `threads` host threads. Returns (outs list of [nq, D], lses list of [nq], seconds)."""
    n = len(items)
    nq = np.array([it["q"].shape[0] for it in items], np.int32)
    nk = np.array([it["k"].shape[0] for it in items], np.int32)
    row_off = np.concatenate([[0], np.cumsum(nq)[:-1]]).astype(np.int64)
    k_off = np.concatenate([[0], np.cumsum(nk)[:-1]]).astype(np.int64)
    rows = np.ascontiguousarray(np.concatenate([it["rows"] for it in items]), np.int32)
    qa = _f64(np.concatenate([it["q"] for it in items]))
    ka = _f64(np.concatenate([it["k"] for it in items]))
    va = _f64(np.concatenate([it["v"] for it in items]))
    out = np.zeros((int(nq.sum()), D))
    lse = np.zeros(int(nq.sum()))
    sec = C.c_double()
    rc = ref().dcpr_run_items(n, _p(nq), _p(nk), _p(row_off), _p(rows), D, _p(qa), _p(ka), _p(va),
                              _p(row_off), _p(k_off), _p(row_off), _p(out), _p(lse), threads, C.byref(sec))
    if rc:
        raise RuntimeError(ref().dcpr_last_error().decode())
    outs = [out[o:o + a] for o, a in zip(row_off, nq)]
    lses = [lse[o:o + a] for o, a in zip(row_off, nq)]
    return outs, lses, sec.value
