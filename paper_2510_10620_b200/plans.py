"""Flat plan bundles: the reference planner's artefacts as numpy arrays.

A ``PlanBundle`` holds exactly what ``dcp::run`` receives (simexec.hpp:207-209):
the per-device ``ExecutionPlan``s (plan.hpp:101-107) and the ``BlockGraph``
(blocks.hpp:53-85, including the per-sequence ``AttendRanges`` masks), plus the
placement and ``CommVolume`` (placement.hpp:164-243) needed to check bytes
bit-exactly. Arrays use the POD layouts of ``include/dcpx.h`` so they can be
handed to ``dcpx_prepare`` without conversion. Bundles are cached as ``.npz``
files so planning (slow, single-threaded reference code) is never timed.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

# --- numpy mirrors of include/dcpx.h --------------------------------------------------
DATA_BLOCK = np.dtype([("id", "<i4"), ("kind", "<i4"), ("seq", "<i4"), ("head", "<i4"),
                       ("tile", "<i4"), ("_pad", "<i4"), ("tok_begin", "<i8"),
                       ("tok_end", "<i8"), ("size_bytes", "<u8")])
COMP_BLOCK = np.dtype([("id", "<i4"), ("q_block", "<i4"), ("kv_block", "<i4"),
                       ("o_block", "<i4"), ("seq", "<i4"), ("head", "<i4"), ("q_tile", "<i4"),
                       ("kv_tile", "<i4"), ("attended_pairs", "<u8"), ("flops_weight", "<u8")])
ATT_ITEM = np.dtype([("comp_id", "<i4"), ("q_slot", "<i4"), ("kv_slot", "<i4"),
                     ("out_slot", "<i4"), ("seq", "<i4"), ("head", "<i4"), ("q_begin", "<i8"),
                     ("q_end", "<i8"), ("kv_begin", "<i8"), ("kv_end", "<i8"),
                     ("rows_offset", "<i8")])
BLOCK_SLOT = np.dtype([("block", "<i4"), ("slot", "<i4")])
COPY_ITEM = np.dtype([("src_slot", "<i4"), ("dst_slot", "<i4")])

OP_ATTENTION, OP_REDUCTION, OP_COPY, OP_COMM_LAUNCH, OP_COMM_WAIT = range(5)
KIND_Q, KIND_KV, KIND_O = range(3)

assert DATA_BLOCK.itemsize == 48 and COMP_BLOCK.itemsize == 48 and ATT_ITEM.itemsize == 64


class c_data_block(C.Structure):
    _fields_ = [("id", C.c_int32), ("kind", C.c_int32), ("seq", C.c_int32),
                ("head", C.c_int32), ("tile", C.c_int32), ("_pad", C.c_int32),
                ("tok_begin", C.c_int64), ("tok_end", C.c_int64), ("size_bytes", C.c_uint64)]


class c_graph_view(C.Structure):
    _fields_ = [("heads", C.c_int32), ("kv_groups", C.c_int32), ("head_dim", C.c_int32),
                ("bytes_per_element", C.c_int32), ("num_seqs", C.c_int32),
                ("num_data_blocks", C.c_int32), ("num_comp_blocks", C.c_int32),
                ("_pad", C.c_int32), ("seq_lengths", C.c_void_p), ("block_sizes", C.c_void_p),
                ("data_blocks", C.c_void_p), ("comp_blocks", C.c_void_p)]


class c_mask_view(C.Structure):
    _fields_ = [("seq_offsets", C.c_void_p), ("ranges", C.c_void_p)]


class c_instruction(C.Structure):
    _fields_ = [("op", C.c_int32), ("division", C.c_int32), ("send", C.c_int32),
                ("peer", C.c_int32), ("dst", C.c_int32), ("count", C.c_int32),
                ("offset", C.c_int64), ("tag", C.c_char_p)]


class c_plan_view(C.Structure):
    _fields_ = [("version", C.c_int32), ("device", C.c_int32), ("divisions", C.c_int32),
                ("_pad", C.c_int32), ("capacity", C.c_int32 * 3), ("n_resident_q", C.c_int32),
                ("n_resident_kv", C.c_int32), ("n_resident_o", C.c_int32),
                ("resident_q", C.c_void_p), ("resident_kv", C.c_void_p),
                ("resident_o", C.c_void_p), ("n_instructions", C.c_int32), ("_pad2", C.c_int32),
                ("instructions", C.c_void_p), ("items", C.c_void_p), ("srcs", C.c_void_p),
                ("copies", C.c_void_p), ("blocks", C.c_void_p), ("rows", C.c_void_p)]


class c_report(C.Structure):
    _fields_ = [("devices", C.c_int32), ("stages", C.c_int32), ("total_bytes", C.c_uint64),
                ("total_flops", C.c_uint64), ("per_device_send", C.c_uint64 * 64),
                ("per_device_recv", C.c_uint64 * 64), ("wire_bytes", C.c_uint64),
                ("makespan", C.c_double), ("device_ms", C.c_double),
                ("kernel_launches", C.c_int32), ("attn_launches", C.c_int32),
                ("attn_ms", C.c_double), ("attn_ms_sum", C.c_double),
                ("wire_per_device_send", C.c_uint64 * 64), ("wire_per_device_recv", C.c_uint64 * 64),
                ("units", C.c_int32), ("windowed", C.c_int32)]


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


@dataclass
class DevicePlan:
    device: int
    divisions: int
    capacity: np.ndarray            # int32[3]
    resident_q: np.ndarray          # BLOCK_SLOT
    resident_kv: np.ndarray
    resident_o: np.ndarray
    instr: np.ndarray               # int32[n, 8]: op, division, send, peer, dst, count, offset, tag
    items: np.ndarray               # ATT_ITEM
    srcs: np.ndarray                # int32
    copies: np.ndarray              # COPY_ITEM
    blocks: np.ndarray              # BLOCK_SLOT
    tags: List[str]
    rows: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int32))

    def instructions(self):
        for r in self.instr:
            yield dict(op=int(r[0]), division=int(r[1]), send=int(r[2]), peer=int(r[3]),
                       dst=int(r[4]), count=int(r[5]), offset=int(r[6]),
                       tag=self.tags[int(r[7])] if r[7] >= 0 else None)

    def copy(self) -> "DevicePlan":
        return DevicePlan(self.device, self.divisions, self.capacity.copy(),
                          self.resident_q.copy(), self.resident_kv.copy(),
                          self.resident_o.copy(), self.instr.copy(), self.items.copy(),
                          self.srcs.copy(), self.copies.copy(), self.blocks.copy(),
                          list(self.tags), self.rows.copy())


@dataclass
class PlanBundle:
    """Reference planner output for one batch (all devices)."""
    R: int
    T: int
    H: int
    G: int
    D: int
    bpe: int
    seq_lengths: np.ndarray
    block_sizes: np.ndarray
    seq_offsets: np.ndarray
    ranges: np.ndarray              # int32 [total_tokens, 4]
    data_blocks: np.ndarray         # DATA_BLOCK
    comp_blocks: np.ndarray         # COMP_BLOCK
    data_block_device: np.ndarray
    comp_block_device: np.ndarray
    dev_flops: np.ndarray           # uint64 [R]   PlacementResult.balance[d].flops
    per_device_send: np.ndarray     # uint64 [R]   CommVolume
    per_device_recv: np.ndarray
    volume: np.ndarray              # uint64 [5]: total, q_xfer, kv_xfer, o_xfer, inter_machine
    devices: List[DevicePlan]
    meta: Dict[str, str] = field(default_factory=dict)

    # ---- derived quantities ------------------------------------------------------
    @property
    def total_tokens(self) -> int:
        return int(self.seq_offsets[-1])

    @property
    def total_flops(self) -> int:
        """BlockGraph::total_flops (blocks.hpp:74-78) = 4 * D * attended pairs."""
        return int(self.comp_blocks["flops_weight"].sum(dtype=np.uint64))

    def bwd_bytes(self):
        """Backward planned bytes per device (builder-defined):
        per forward Q fetch 3x Q bytes (Q + dO out, dQ back), per KV fetch 2x KV bytes
        (KV out, dK/dV back). Returns (send[R], recv[R])."""
        send = np.zeros(self.R, np.uint64)
        recv = np.zeros(self.R, np.uint64)
        db = self.data_blocks
        for dp in self.devices:
            for ins in dp.instructions():
                if ins["op"] != OP_COMM_LAUNCH or ins["send"]:
                    continue
                blks = dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]
                for b in blks["block"]:
                    kind = int(db["kind"][b])
                    size = np.uint64(db["size_bytes"][b])
                    src, dst = ins["peer"], dp.device
                    if kind == KIND_Q:      # Q + dO forward, dQ back
                        send[src] += 2 * size; recv[dst] += 2 * size
                        send[dst] += size; recv[src] += size
                    elif kind == KIND_KV:   # KV forward, dK+dV back
                        send[src] += size; recv[dst] += size
                        send[dst] += size; recv[src] += size
        return send, recv

    def wire_bytes(self):
        """Bytes the executor's transfers actually move, per device (forward and backward):
        forward O blocks travel with their fp32 LSE (4 B/row); backward Q fetches move Q, dO
        and the fp32 LSE and Delta rows (8 B/row); gradient returns are fp32 (2x the planned
        block bytes). Returns ((fwd_send, fwd_recv), (bwd_send, bwd_recv)), uint64[R] each."""
        fs, fr, bs, br = (np.zeros(self.R, np.uint64) for _ in range(4))
        db = self.data_blocks
        for dp in self.devices:
            for ins in dp.instructions():
                if ins["op"] != OP_COMM_LAUNCH or ins["send"]:
                    continue
                src, dst = ins["peer"], dp.device
                for b in dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]["block"]:
                    kind = int(db["kind"][b])
                    size = int(db["size_bytes"][b])
                    rows = int(db["tok_end"][b] - db["tok_begin"][b])
                    fwd = size + (4 * rows if kind == KIND_O else 0)
                    fs[src] += fwd; fr[dst] += fwd
                    if kind == KIND_Q:
                        out = 2 * size + 8 * rows
                        bs[src] += out; br[dst] += out
                        bs[dst] += 2 * size; br[src] += 2 * size
                    elif kind == KIND_KV:
                        bs[src] += size; br[dst] += size
                        bs[dst] += 2 * size; br[src] += 2 * size
        return (fs, fr), (bs, br)

    def item_sample(self, items: np.ndarray) -> "PlanBundle":
        """A one-device bundle executing each of `items` (ATT_ITEM rows taken from any of this
        bundle's plans) on its own: their Q / KV blocks resident, one AttentionInstr, item i
        writing O slot i, no reductions. After a forward, O-arena slot i holds item i's
        normalised partial and the LSE arena its m + ln l -- exactly what exec_attention
        (simexec.hpp:33-76) returns for that item, so a sample of the plan's items can be
        compared one by one with the reference executor (bench.py's cpu_baseline leg)."""
        cb = self.comp_blocks
        qb = [int(cb["q_block"][int(c)]) for c in items["comp_id"]]
        kb = [int(cb["kv_block"][int(c)]) for c in items["comp_id"]]
        uq = {b: i for i, b in enumerate(dict.fromkeys(qb))}
        uk = {b: i for i, b in enumerate(dict.fromkeys(kb))}
        its = np.array(items, ATT_ITEM).copy()
        rows = []
        for i in range(len(its)):
            its["q_slot"][i], its["kv_slot"][i], its["out_slot"][i] = uq[qb[i]], uk[kb[i]], i
            if its["rows_offset"][i] >= 0:
                raise ValueError("item_sample: items with explicit rows are not supported")
        res_q = np.array([(b, s) for b, s in uq.items()], BLOCK_SLOT)
        res_kv = np.array([(b, s) for b, s in uk.items()], BLOCK_SLOT)
        dp = DevicePlan(device=0, divisions=1, capacity=np.array([len(uq), len(uk), len(its)], np.int32),
                        resident_q=res_q, resident_kv=res_kv, resident_o=np.zeros(0, BLOCK_SLOT),
                        instr=np.array([[OP_ATTENTION, 0, 0, 0, 0, len(its), 0, -1]], np.int32),
                        items=its, srcs=np.zeros(0, np.int32), copies=np.zeros(0, COPY_ITEM),
                        blocks=np.zeros(0, BLOCK_SLOT), tags=[])
        z = np.zeros(1, np.uint64)
        return PlanBundle(R=1, T=1, H=self.H, G=self.G, D=self.D, bpe=self.bpe,
                          seq_lengths=self.seq_lengths, block_sizes=self.block_sizes,
                          seq_offsets=self.seq_offsets, ranges=self.ranges, data_blocks=self.data_blocks,
                          comp_blocks=self.comp_blocks,
                          data_block_device=np.zeros(len(self.data_blocks), np.int32),
                          comp_block_device=np.zeros(len(self.comp_blocks), np.int32),
                          dev_flops=z, per_device_send=z, per_device_recv=z.copy(),
                          volume=np.zeros(5, np.uint64), devices=[dp], meta={"item_sample": str(len(its))})

    # ---- persistence -------------------------------------------------------------
    def save(self, path: str) -> None:
        arrs = dict(header=np.array([self.R, self.T, self.H, self.G, self.D, self.bpe], np.int64),
                    seq_lengths=self.seq_lengths, block_sizes=self.block_sizes,
                    seq_offsets=self.seq_offsets, ranges=self.ranges,
                    data_blocks=self.data_blocks, comp_blocks=self.comp_blocks,
                    data_block_device=self.data_block_device,
                    comp_block_device=self.comp_block_device, dev_flops=self.dev_flops,
                    per_device_send=self.per_device_send, per_device_recv=self.per_device_recv,
                    volume=self.volume,
                    meta=np.array([f"{k}={v}" for k, v in self.meta.items()]))
        for dp in self.devices:
            p = f"d{dp.device}_"
            arrs[p + "hdr"] = np.array([dp.device, dp.divisions], np.int64)
            arrs[p + "capacity"] = dp.capacity
            arrs[p + "resident_q"] = dp.resident_q
            arrs[p + "resident_kv"] = dp.resident_kv
            arrs[p + "resident_o"] = dp.resident_o
            arrs[p + "instr"] = dp.instr
            arrs[p + "items"] = dp.items
            arrs[p + "srcs"] = dp.srcs
            arrs[p + "copies"] = dp.copies
            arrs[p + "blocks"] = dp.blocks
            arrs[p + "tags"] = np.array(dp.tags if dp.tags else [""])
            arrs[p + "ntags"] = np.array([len(dp.tags)], np.int64)
        tmp = path + ".tmp.npz"
        np.savez_compressed(tmp, **arrs)
        os.replace(tmp, path)

    @staticmethod
    def load(path: str) -> "PlanBundle":
        z = np.load(path, allow_pickle=False)
        R, T, H, G, D, bpe = (int(x) for x in z["header"])
        devs = []
        for d in range(R):
            p = f"d{d}_"
            ntags = int(z[p + "ntags"][0])
            devs.append(DevicePlan(
                device=int(z[p + "hdr"][0]), divisions=int(z[p + "hdr"][1]),
                capacity=z[p + "capacity"].astype(np.int32), resident_q=z[p + "resident_q"],
                resident_kv=z[p + "resident_kv"], resident_o=z[p + "resident_o"],
                instr=z[p + "instr"], items=z[p + "items"], srcs=z[p + "srcs"],
                copies=z[p + "copies"], blocks=z[p + "blocks"],
                tags=[str(t) for t in z[p + "tags"][:ntags]]))
        meta = {}
        for m in z["meta"]:
            k, _, v = str(m).partition("=")
            if k:
                meta[k] = v
        return PlanBundle(R, T, H, G, D, bpe, z["seq_lengths"], z["block_sizes"],
                          z["seq_offsets"], z["ranges"], z["data_blocks"], z["comp_blocks"],
                          z["data_block_device"], z["comp_block_device"], z["dev_flops"],
                          z["per_device_send"], z["per_device_recv"], z["volume"], devs, meta)

    # ---- C views -------------------------------------------------------------------
    def c_views(self, device_ids=None):
        """Returns (keepalive, graph_view, mask_view, plan_view_array) for dcpx_prepare."""
        keep = []
        g = c_graph_view()
        g.heads, g.kv_groups, g.head_dim, g.bytes_per_element = self.H, self.G, self.D, self.bpe
        g.num_seqs = len(self.seq_lengths)
        g.num_data_blocks = len(self.data_blocks)
        g.num_comp_blocks = len(self.comp_blocks)
        arrs = [np.ascontiguousarray(self.seq_lengths, np.int64),
                np.ascontiguousarray(self.block_sizes, np.int64),
                np.ascontiguousarray(self.data_blocks), np.ascontiguousarray(self.comp_blocks),
                np.ascontiguousarray(self.seq_offsets, np.int64),
                np.ascontiguousarray(self.ranges, np.int32)]
        keep += arrs
        g.seq_lengths, g.block_sizes, g.data_blocks, g.comp_blocks = (_ptr(a) for a in arrs[:4])
        m = c_mask_view()
        m.seq_offsets, m.ranges = _ptr(arrs[4]), _ptr(arrs[5])
        ids = list(range(self.R)) if device_ids is None else list(device_ids)
        pv = (c_plan_view * len(ids))()
        for i, d in enumerate(ids):
            dp = self.devices[d]
            v = pv[i]
            v.version, v.device, v.divisions = 1, dp.device, dp.divisions
            for k in range(3):
                v.capacity[k] = int(dp.capacity[k])
            rq, rkv, ro = (np.ascontiguousarray(a) for a in (dp.resident_q, dp.resident_kv,
                                                             dp.resident_o))
            v.n_resident_q, v.n_resident_kv, v.n_resident_o = len(rq), len(rkv), len(ro)
            v.resident_q, v.resident_kv, v.resident_o = _ptr(rq), _ptr(rkv), _ptr(ro)
            tagbufs = [C.create_string_buffer(t.encode()) for t in dp.tags]
            ins = (c_instruction * max(1, len(dp.instr)))()
            for j, r in enumerate(dp.instr):
                x = ins[j]
                x.op, x.division, x.send, x.peer, x.dst, x.count = (int(r[k]) for k in range(6))
                x.offset = int(r[6])
                x.tag = C.cast(tagbufs[int(r[7])], C.c_char_p) if r[7] >= 0 else None
            v.n_instructions = len(dp.instr)
            v.instructions = C.addressof(ins)
            pools = [np.ascontiguousarray(dp.items), np.ascontiguousarray(dp.srcs, np.int32),
                     np.ascontiguousarray(dp.copies), np.ascontiguousarray(dp.blocks),
                     np.ascontiguousarray(dp.rows, np.int32)]
            v.items, v.srcs, v.copies, v.blocks, v.rows = (_ptr(a) for a in pools)
            keep += [rq, rkv, ro, tagbufs, ins, pools]
        return keep, g, m, pv
