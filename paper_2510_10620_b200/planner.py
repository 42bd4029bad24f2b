"""ctypes binding of the caller-side planner shim (planner/dcp_planner_capi.cpp).

The planner itself is the reference's, unchanged (pipeline.hpp:29-38 ``plan_batch``);
this module only builds batches, calls it, and converts the flattened artefacts to a
:class:`~paper_2510_10620_b200.plans.PlanBundle`.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import plans as P

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_REPO, "planner", "_build", "libdcpplanner.so")

MASKS = {"causal": 0, "lambda": 1, "causal_blockwise": 2, "shared_question": 3}
ERRORS = {1: "Error", 2: "DeadlockError", 3: "TagMismatchError", 4: "BufferOverflowError",
          5: "InfeasibleError"}


class PlannerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class SeqSpecC(C.Structure):
    _fields_ = [("length", C.c_int64), ("kind", C.c_int32), ("window_blocks", C.c_int32),
                ("sink_blocks", C.c_int32), ("test_blocks", C.c_int32), ("sink", C.c_int64),
                ("window", C.c_int64), ("block", C.c_int64), ("question_len", C.c_int64),
                ("n_answers", C.c_int32), ("_pad", C.c_int32), ("answer_lens", C.c_int64 * 16)]


class CfgC(C.Structure):
    _fields_ = [("machines", C.c_int32), ("devices_per_machine", C.c_int32),
                ("divisions", C.c_int32), ("max_slots_per_kind", C.c_int32),
                ("block_size", C.c_int64), ("eps_inter", C.c_double), ("eps_intra", C.c_double),
                ("eps_data", C.c_double), ("seed", C.c_uint64), ("verify", C.c_int32),
                ("threads", C.c_int32)]


@dataclass
class SeqSpec:
    """SequenceSpec + MaskDescriptor (types.hpp:86-174)."""
    length: int
    mask: str = "causal"
    sink: int = 0
    window: int = 0
    block: int = 0
    window_blocks: int = 0
    sink_blocks: int = 0
    test_blocks: int = 0
    question_len: int = 0
    answer_lens: List[int] = field(default_factory=list)

    def to_c(self) -> SeqSpecC:
        s = SeqSpecC()
        s.length, s.kind = self.length, MASKS[self.mask]
        s.sink, s.window, s.block = self.sink, self.window, self.block
        s.window_blocks, s.sink_blocks, s.test_blocks = (self.window_blocks, self.sink_blocks,
                                                         self.test_blocks)
        s.question_len = self.question_len
        if len(self.answer_lens) > 16:
            raise ValueError("at most 16 answers supported by the shim")
        s.n_answers = len(self.answer_lens)
        for i, a in enumerate(self.answer_lens):
            s.answer_lens[i] = a
        return s

    @staticmethod
    def from_c(s: SeqSpecC) -> "SeqSpec":
        inv = {v: k for k, v in MASKS.items()}
        return SeqSpec(int(s.length), inv[int(s.kind)], int(s.sink), int(s.window), int(s.block),
                       int(s.window_blocks), int(s.sink_blocks), int(s.test_blocks),
                       int(s.question_len), [int(s.answer_lens[i]) for i in range(s.n_answers)])


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"planner shim not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.dcpp_last_error.restype = C.c_char_p
        L.dcpp_batch_sparsity.restype = C.c_double
        L.dcpp_batch_from_specs.argtypes = [C.POINTER(SeqSpecC), C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_int64, C.POINTER(C.c_void_p)]
        L.dcpp_batch_from_synth.argtypes = [C.c_int, C.c_double, C.c_int64, C.c_int64, C.c_int,
                                            C.c_int, C.c_uint64, C.c_int64, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_int)]
        L.dcpp_batch_random.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]
        L.dcpp_batch_num_seqs.argtypes = [C.c_void_p]
        L.dcpp_batch_seq.argtypes = [C.c_void_p, C.c_int, C.POINTER(SeqSpecC)]
        L.dcpp_batch_shape.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.dcpp_batch_sparsity.argtypes = [C.c_void_p]
        L.dcpp_batch_free.argtypes = [C.c_void_p]
        L.dcpp_plan.argtypes = [C.c_void_p, C.POINTER(CfgC), C.c_int, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_void_p)]
        L.dcpp_plan_free.argtypes = [C.c_void_p]
        L.dcpp_array.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_int64)]
        L.dcpp_graph_counts.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_int]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise PlannerError(rc, lib().dcpp_last_error().decode())


class Batch:
    """A reference ``dcp::Batch`` (types.hpp:245-274) owned by the shim."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib().dcpp_batch_free(self._h)
            self._h = None

    @staticmethod
    def from_specs(specs: Sequence[SeqSpec], heads: int, kv_groups: int, head_dim: int = 128,
                   bpe: int = 2, token_budget: int = 0) -> "Batch":
        arr = (SeqSpecC * len(specs))(*[s.to_c() for s in specs])
        h = C.c_void_p()
        _check(lib().dcpp_batch_from_specs(arr, len(specs), heads, kv_groups, head_dim, bpe,
                                           token_budget, C.byref(h)))
        return Batch(h)

    @staticmethod
    def from_synth(mask: str, max_len: int, token_budget: int, index: int, heads: int,
                   kv_groups: int, head_dim: int = 128, seed: int = 42, count: int = 64,
                   dist: int = 0, scale: float = 1.0, min_len: int = 0):
        """synth_sequences (synth.hpp:84-100) -> make_batches (pipeline.hpp:42-65)[index]."""
        h = C.c_void_p()
        n = C.c_int()
        _check(lib().dcpp_batch_from_synth(dist, scale, max_len, min_len, MASKS[mask], count, seed,
                                           token_budget, index, heads, kv_groups, head_dim, 2,
                                           C.byref(h), C.byref(n)))
        return Batch(h), n.value

    @staticmethod
    def random(seed: int, max_seq_len: int = 64, max_seqs: int = 3, max_heads: int = 2,
               head_dim: int = 128) -> "Batch":
        """fixtures::random_batch (tests/fixtures.hpp:172-189), head_dim overridden."""
        h = C.c_void_p()
        _check(lib().dcpp_batch_random(seed, max_seq_len, max_seqs, max_heads, head_dim,
                                       C.byref(h)))
        return Batch(h)

    @property
    def sequences(self) -> List[SeqSpec]:
        out = []
        for i in range(lib().dcpp_batch_num_seqs(self._h)):
            s = SeqSpecC()
            lib().dcpp_batch_seq(self._h, i, C.byref(s))
            out.append(SeqSpec.from_c(s))
        return out

    @property
    def shape(self):
        a = (C.c_int32 * 4)()
        lib().dcpp_batch_shape(self._h, a)
        return tuple(a)  # heads, kv_groups, head_dim, bpe

    @property
    def sparsity(self) -> float:
        return lib().dcpp_batch_sparsity(self._h)

    def graph_counts(self, block_size: int):
        g, c = C.c_int32(), C.c_int32()
        _check(lib().dcpp_graph_counts(self._h, block_size, C.byref(g), C.byref(c), None, None, 0))
        gt = np.zeros(g.value, np.int32)
        cq = np.zeros(c.value, np.int32)
        _check(lib().dcpp_graph_counts(self._h, block_size, C.byref(g), C.byref(c),
                                       gt.ctypes.data, cq.ctypes.data, max(g.value, c.value)))
        return gt, cq


def _arr(h, name: str, device: int, dtype) -> np.ndarray:
    ptr, nb = C.c_void_p(), C.c_int64()
    _check(lib().dcpp_array(h, name.encode(), device, C.byref(ptr), C.byref(nb)))
    dt = np.dtype(dtype)
    if nb.value == 0:
        return np.zeros(0, dt)
    buf = (C.c_char * nb.value).from_address(ptr.value)
    return np.frombuffer(bytes(buf), dtype=dt).copy()


def plan(batch: Batch, devices: int, block_size: int, divisions: int = 4,
         eps_inter: float = 0.4, eps_intra: float = 0.1, eps_data: float = 0.05, seed: int = 0,
         machines: int = 1, placement: str = "dcp", group_dev: Optional[np.ndarray] = None,
         comp_dev: Optional[np.ndarray] = None, verify: bool = True,
         max_slots_per_kind: int = 0, json_dir: Optional[str] = None, threads: int = 0) -> P.PlanBundle:
    """Runs the reference planner (plan_batch, pipeline.hpp:29-38) and flattens it.
    json_dir: also write the plan in the reference's file formats there (batch.jsonl,
    graph.json, placement.json, plan_d<d>.json, with the reference's own writers).
    threads: 1 = the reference's single-threaded plan_batch, unchanged; 0 (all host cores) or
    n > 1 = the same plan, bit for bit, with the partitioner's candidate evaluation and
    repair scans on host threads (planner/dcp_partition_parallel.hpp)."""
    cfg = CfgC()
    cfg.machines, cfg.devices_per_machine = machines, devices // machines
    cfg.divisions, cfg.max_slots_per_kind, cfg.block_size = divisions, max_slots_per_kind, block_size
    cfg.eps_inter, cfg.eps_intra, cfg.eps_data, cfg.seed = eps_inter, eps_intra, eps_data, seed
    cfg.verify = 1 if verify else 0
    cfg.threads = threads
    mode = {"dcp": 0, "ring": 1, "zigzag": 2, "explicit": 3}[placement]
    gd = np.ascontiguousarray(group_dev, np.int32) if group_dev is not None else None
    cd = np.ascontiguousarray(comp_dev, np.int32) if comp_dev is not None else None
    h = C.c_void_p()
    _check(lib().dcpp_plan(batch._h, C.byref(cfg), mode, gd.ctypes.data if gd is not None else None,
                           cd.ctypes.data if cd is not None else None, C.byref(h)))
    try:
        if json_dir is not None:
            _check(lib().dcpp_dump_json(h, batch._h, json_dir.encode()))
        hdr = _arr(h, "header", 0, np.int32)
        R, T, H, G, D, bpe = (int(x) for x in hdr[:6])
        devs = []
        for d in range(R):
            instr = _arr(h, "instr", d, np.int32).reshape(-1, 8)
            tags_blob = _arr(h, "tags", d, np.uint8).tobytes().decode()
            tags = tags_blob.split("\n")[:-1] if tags_blob else []
            devs.append(P.DevicePlan(
                device=d, divisions=T, capacity=_arr(h, "capacity", d, np.int32),
                resident_q=_arr(h, "resident_q", d, P.BLOCK_SLOT),
                resident_kv=_arr(h, "resident_kv", d, P.BLOCK_SLOT),
                resident_o=_arr(h, "resident_o", d, P.BLOCK_SLOT), instr=instr,
                items=_arr(h, "items", d, P.ATT_ITEM), srcs=_arr(h, "srcs", d, np.int32),
                copies=_arr(h, "copies", d, P.COPY_ITEM), blocks=_arr(h, "blocks", d, P.BLOCK_SLOT),
                tags=tags))
        bundle = P.PlanBundle(
            R=R, T=T, H=H, G=G, D=D, bpe=bpe, seq_lengths=_arr(h, "seq_lengths", 0, np.int64),
            block_sizes=_arr(h, "block_sizes", 0, np.int64),
            seq_offsets=_arr(h, "seq_offsets", 0, np.int64),
            ranges=_arr(h, "ranges", 0, np.int32).reshape(-1, 4),
            data_blocks=_arr(h, "data_blocks", 0, P.DATA_BLOCK),
            comp_blocks=_arr(h, "comp_blocks", 0, P.COMP_BLOCK),
            data_block_device=_arr(h, "data_block_device", 0, np.int32),
            comp_block_device=_arr(h, "comp_block_device", 0, np.int32),
            dev_flops=_arr(h, "dev_flops", 0, np.uint64),
            per_device_send=_arr(h, "per_device_send", 0, np.uint64),
            per_device_recv=_arr(h, "per_device_recv", 0, np.uint64),
            volume=_arr(h, "volume", 0, np.uint64), devices=devs)
        bundle.meta.update(block_size=str(block_size), divisions=str(divisions),
                           eps=f"{eps_inter},{eps_intra},{eps_data}", placement=placement,
                           seed=str(seed))
        return bundle
    finally:
        lib().dcpp_plan_free(h)
