"""Plan files in the reference's own JSON formats -> ``PlanBundle``.

The reference writes a planned batch as
  * ``batch.jsonl``     -- ``write_sequences_jsonl`` (inc/io.hpp:72-88): header + sequences,
  * ``graph.json``      -- ``block_graph_to_json`` (inc/io.hpp:135-174),
  * ``placement.json``  -- ``placement_to_json`` (inc/io.hpp:183-216),
  * ``plan_d<d>.json``  -- ``plan_to_json`` per device (inc/io.hpp:271-350).

``load_reference_plan(dir)`` parses those files into the flat views ``dcpx_prepare``
takes, with the same flattening as ``planner/dcp_planner_capi.cpp`` (so planning and
execution decouple: a plan written by the reference's tools runs on the GPU without the
planner). Attention items keep the rows the plan file carries (``AttentionItem::rows``,
inc/plan.hpp:231-242) as explicit rows (``rows_offset >= 0``); the per-token mask is not
re-evaluated, so ``bundle.ranges`` holds zero placeholders. Byte tables (``CommVolume``,
inc/placement.hpp:180-243) are recomputed from the plans' CommLaunch instructions.
``dump_reference_plan`` writes a bundle back in the same schema (graph, placement, plans).
"""
from __future__ import annotations

import json
import os
from typing import Dict, List

import numpy as np

from . import plans as P

KINDS = {"q": P.KIND_Q, "kv": P.KIND_KV, "o": P.KIND_O}
KIND_NAMES = {v: k for k, v in KINDS.items()}


def _read(path):
    with open(path) as f:
        return json.load(f)


def _flatten_plan(j: Dict, device_rows: List[np.ndarray]) -> P.DevicePlan:
    """One plan_to_json object -> DevicePlan (same layout as the planner shim's flatten())."""
    if j.get("version") != 1:
        raise ValueError("unsupported plan version")  # plan_from_json, inc/io.hpp:354
    buf = j["buffers"]

    def resident(a):
        return np.array([(b["block"], b["slot"]) for b in a], dtype=P.BLOCK_SLOT)
    instr, items, srcs, copies, blocks, tags, rows = [], [], [], [], [], [], []
    n_rows = 0
    for op in j["instructions"]:
        rec = [0, int(op["division"]), 0, 0, 0, 0, 0, -1]
        kind = op["op"]
        if kind == "blockwise_attention":
            rec[0], rec[5], rec[6] = P.OP_ATTENTION, len(op["items"]), len(items)
            for it in op["items"]:
                r = np.zeros((len(it["rows"]), 4), np.int32)
                for i, tr in enumerate(it["rows"]):
                    if len(tr) > 4:
                        raise ValueError("TokenRanges holds at most two ranges")  # types.hpp:198-208
                    r[i, :len(tr)] = tr
                items.append((it["comp"], it["q_slot"], it["kv_slot"], it["out_slot"], it["seq"], it["head"],
                              it["q_start"], it["q_end"], it["kv_start"], it["kv_end"], n_rows))
                rows.append(r)
                n_rows += len(r)
        elif kind == "blockwise_reduction":
            rec[0], rec[4], rec[5], rec[6] = P.OP_REDUCTION, int(op["dst"]), len(op["srcs"]), len(srcs)
            srcs.extend(int(s) for s in op["srcs"])
        elif kind == "blockwise_copy":
            rec[0], rec[5], rec[6] = P.OP_COPY, len(op["items"]), len(copies)
            copies.extend((it["src"], it["dst"]) for it in op["items"])
        elif kind == "comm_launch":
            rec[0], rec[2], rec[3] = P.OP_COMM_LAUNCH, 1 if op["dir"] == "send" else 0, int(op["peer"])
            rec[5], rec[6], rec[7] = len(op["blocks"]), len(blocks), len(tags)
            blocks.extend((b["block"], b["slot"]) for b in op["blocks"])
            tags.append(op["tag"])
        elif kind == "comm_wait":
            rec[0], rec[7] = P.OP_COMM_WAIT, len(tags)
            tags.append(op["tag"])
        else:
            raise ValueError("unknown instruction op: " + kind)  # inc/io.hpp:412
        instr.append(rec)
    device_rows.append(np.concatenate(rows) if rows else np.zeros((0, 4), np.int32))
    return P.DevicePlan(
        device=int(j["device"]), divisions=int(j["divisions"]),
        capacity=np.array([buf["q"]["capacity"], buf["kv"]["capacity"], buf["o"]["capacity"]], np.int32),
        resident_q=resident(buf["q"]["resident"]), resident_kv=resident(buf["kv"]["resident"]),
        resident_o=resident(buf["o"]["resident"]),
        instr=np.array(instr, np.int32).reshape(-1, 8),
        items=np.array(items, dtype=P.ATT_ITEM), srcs=np.array(srcs, np.int32),
        copies=np.array(copies, dtype=P.COPY_ITEM), blocks=np.array(blocks, dtype=P.BLOCK_SLOT),
        tags=tags, rows=device_rows[-1])


def load_reference_plan(directory: str) -> P.PlanBundle:
    """Reads batch.jsonl, graph.json, placement.json and plan_d*.json from `directory`."""
    with open(os.path.join(directory, "batch.jsonl")) as f:
        lines = [json.loads(x) for x in f if x.strip()]
    hdr, seqs = lines[0], lines[1:]
    if "seq_id" in hdr:
        raise ValueError("batch input: first line must be the batch header")  # inc/io.hpp:103
    graph = _read(os.path.join(directory, "graph.json"))
    place = _read(os.path.join(directory, "placement.json"))
    R = int(place["machines"]) * int(place["devices_per_machine"])
    plans = [_read(os.path.join(directory, f"plan_d{d}.json")) for d in range(R)]

    db = graph["data_blocks"]
    data_blocks = np.zeros(len(db), dtype=P.DATA_BLOCK)
    for i, b in enumerate(db):
        data_blocks[i] = (b["id"], KINDS[b["kind"]], b["seq"], b["head"], b["tile"], 0, b["start"], b["end"],
                          b["size_bytes"])
    cb = graph["comp_blocks"]
    comp_blocks = np.zeros(len(cb), dtype=P.COMP_BLOCK)
    for i, c in enumerate(cb):
        qb, kb = data_blocks[c["q_block"]], data_blocks[c["kv_block"]]
        comp_blocks[i] = (c["id"], c["q_block"], c["kv_block"], c["o_block"], qb["seq"], qb["head"], qb["tile"],
                          kb["tile"], c["attended_pairs"], c["flops_weight"])
    seq_lengths = np.array([int(s["length"]) for s in seqs], np.int64)
    seq_offsets = np.concatenate([[0], np.cumsum(seq_lengths)]).astype(np.int64)
    # generate_blocks tiles every sequence with one block size (inc/blocks.hpp): the longest tile
    tile_len = data_blocks["tok_end"] - data_blocks["tok_begin"]
    block = int(tile_len.max()) if len(tile_len) else 0
    block_sizes = np.full(len(seqs), block, np.int64)

    device_rows: List[np.ndarray] = []
    devs = [_flatten_plan(plans[d], device_rows) for d in range(R)]
    T = devs[0].divisions if devs else 0

    # CommVolume from the plans' sends (placement.hpp:180-243): bytes per device and
    # block transfers per kind
    send = np.zeros(R, np.uint64)
    recv = np.zeros(R, np.uint64)
    xfer = [0, 0, 0]
    inter = 0
    dpm = int(place["devices_per_machine"])
    for d, dp in enumerate(devs):
        for ins in dp.instructions():
            if ins["op"] != P.OP_COMM_LAUNCH or not ins["send"]:
                continue
            blk = dp.blocks[ins["offset"]: ins["offset"] + ins["count"]]
            nbytes = int(data_blocks["size_bytes"][blk["block"]].sum())
            send[d] += np.uint64(nbytes)
            recv[ins["peer"]] += np.uint64(nbytes)
            for b in blk["block"]:
                xfer[int(data_blocks["kind"][b])] += 1
            if d // dpm != ins["peer"] // dpm:
                inter += nbytes
    volume = np.array([int(send.sum()), xfer[0], xfer[1], xfer[2], inter], np.uint64)
    D, bpe = int(hdr["head_dim"]), int(hdr.get("bytes_per_element", 2))
    bundle = P.PlanBundle(
        R=R, T=T, H=int(hdr["heads"]), G=int(hdr["kv_groups"]), D=D, bpe=bpe, seq_lengths=seq_lengths,
        # no per-token mask in the plan files: placeholder rows (every item has explicit rows)
        block_sizes=block_sizes, seq_offsets=seq_offsets, ranges=np.zeros((int(seq_offsets[-1]), 4), np.int32),
        data_blocks=data_blocks, comp_blocks=comp_blocks,
        data_block_device=np.array(place["data_block_device"], np.int32),
        comp_block_device=np.array(place["comp_block_device"], np.int32),
        dev_flops=np.array([b["flops"] for b in place["balance"]], np.uint64),
        per_device_send=send, per_device_recv=recv, volume=volume, devices=devs)
    bundle.meta.update(source=os.path.abspath(directory), format="reference-json")
    return bundle


def _ranges_json(row) -> List[int]:
    """TokenRanges -> [b0, e0(, b1, e1)] as token_ranges_to_json (inc/io.hpp:255-262)."""
    out = []
    if row[1] > row[0]:
        out += [int(row[0]), int(row[1])]
    if row[3] > row[2]:
        out += [int(row[2]), int(row[3])]
    return out


def _plan_json(dp: P.DevicePlan, rows: np.ndarray) -> Dict:
    """DevicePlan -> the plan_to_json schema (inc/io.hpp:271-350), key order included."""
    def resident(a):
        return [{"block": int(r["block"]), "slot": int(r["slot"])} for r in a]
    out = {"version": 1, "device": dp.device, "divisions": dp.divisions,
           "buffers": {"q": {"capacity": int(dp.capacity[0]), "resident": resident(dp.resident_q)},
                       "kv": {"capacity": int(dp.capacity[1]), "resident": resident(dp.resident_kv)},
                       "o": {"capacity": int(dp.capacity[2]), "resident": resident(dp.resident_o)}},
           "instructions": []}
    for ins in dp.instructions():
        op = {"division": ins["division"]}
        lo, n = ins["offset"], ins["count"]
        if ins["op"] == P.OP_ATTENTION:
            op["op"] = "blockwise_attention"
            op["items"] = []
            for it in dp.items[lo: lo + n]:
                nq = int(it["q_end"] - it["q_begin"])
                r = rows[int(it["rows_offset"]): int(it["rows_offset"]) + nq]
                op["items"].append({
                    "comp": int(it["comp_id"]), "q_slot": int(it["q_slot"]), "kv_slot": int(it["kv_slot"]),
                    "out_slot": int(it["out_slot"]), "seq": int(it["seq"]), "head": int(it["head"]),
                    "q_start": int(it["q_begin"]), "q_end": int(it["q_end"]), "kv_start": int(it["kv_begin"]),
                    "kv_end": int(it["kv_end"]), "rows": [_ranges_json(row) for row in r]})
        elif ins["op"] == P.OP_REDUCTION:
            op.update(op="blockwise_reduction", dst=ins["dst"], srcs=[int(s) for s in dp.srcs[lo: lo + n]])
        elif ins["op"] == P.OP_COPY:
            op.update(op="blockwise_copy", items=[{"src": int(c["src_slot"]), "dst": int(c["dst_slot"])}
                                                  for c in dp.copies[lo: lo + n]])
        elif ins["op"] == P.OP_COMM_LAUNCH:
            op.update(op="comm_launch", dir="send" if ins["send"] else "recv", peer=ins["peer"], tag=ins["tag"],
                      blocks=[{"block": int(b["block"]), "slot": int(b["slot"])} for b in dp.blocks[lo: lo + n]])
        else:
            op.update(op="comm_wait", tag=ins["tag"])
        out["instructions"].append(op)
    return out


def dump_reference_plan(bundle: P.PlanBundle, directory: str):
    """Writes the bundle's plans (plan_d*.json) in the reference schema. Items must carry
    explicit rows (bundles loaded by load_reference_plan do)."""
    os.makedirs(directory, exist_ok=True)
    for d, dp in enumerate(bundle.devices):
        if len(dp.items) and (dp.items["rows_offset"] < 0).any():
            raise ValueError("dump_reference_plan needs explicit item rows")
        with open(os.path.join(directory, f"plan_d{d}.json"), "w") as f:
            json.dump(_plan_json(dp, dp.rows), f, indent=1)
