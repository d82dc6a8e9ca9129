"""Multi-GPU plumbing of the fix-up prefill.

* Llama-3-8B-shaped work shards **requests**: one process per GPU, each with
  its own model copy, HBM chunk pool and host variant store; no collective on
  the data path (``shard_requests`` decides which rank serves a request).
* Llama-3-70B-shaped work shards **heads** (tensor parallel): rank r holds q
  heads [r*Hq/w, (r+1)*Hq/w), kv heads [r*Hkv/w, ...) (its slice of every
  pool block, so the K1 gather stays local), a column slice of Wq/Wk/Wv and
  of gate/up, a row slice of Wo and down.  The only exchange is the sum of
  the o_proj and down_proj partial outputs (NCCL all-reduce over NVLink),
  the two real reductions of the layer (model.py:417, :419).

``tp_slices`` is the single definition of the partition; the engine and the
CPU tests (oracle + gloo) both use it.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError


# ---------------------------------------------------------------------------
# request sharding (configs 2/3)
# ---------------------------------------------------------------------------


def request_owner(chunk_ids, world: int, policy: str = "affinity") -> int:
    """Rank that serves a request.  ``affinity`` hashes the request's first
    chunk id so requests that share a leading chunk meet the same pool
    (better hit rate under a Zipf trace); ``round_robin`` is used by callers
    that pass a request index instead."""
    if world <= 1:
        return 0
    if policy == "round_robin":
        return int(chunk_ids) % world
    key = str(chunk_ids[0]).encode()
    return int.from_bytes(hashlib.blake2b(key, digest_size=8).digest(), "little") % world


def shard_requests(records, rank: int, world: int, policy: str = "affinity") -> list:
    """The requests rank ``rank`` serves, in trace order (disjoint, complete)."""
    out = []
    for i, rec in enumerate(records):
        ids = getattr(rec, "chunk_ids", rec)
        owner = request_owner(i if policy == "round_robin" else ids, world, policy)
        if owner == rank:
            out.append(rec)
    return out


# ---------------------------------------------------------------------------
# tensor parallel partition (config 4)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TPSlices:
    rank: int
    world: int
    q_heads: tuple  # (first, count) of this rank's query heads
    kv_heads: tuple  # (first, count) of this rank's kv heads
    ff: tuple  # (first, count) of this rank's MLP columns

    def q_cols(self, dh: int) -> slice:
        return slice(self.q_heads[0] * dh, (self.q_heads[0] + self.q_heads[1]) * dh)

    def kv_cols(self, dh: int) -> slice:
        return slice(self.kv_heads[0] * dh, (self.kv_heads[0] + self.kv_heads[1]) * dh)

    def ff_cols(self) -> slice:
        return slice(self.ff[0], self.ff[0] + self.ff[1])


def tp_slices(n_heads: int, n_kv_heads: int, d_ff: int, rank: int, world: int) -> TPSlices:
    """Head/column partition of rank ``rank`` of ``world``.  GQA groups stay
    whole: a rank's q heads all read its own kv heads."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad tensor-parallel rank/world")
    if n_kv_heads % world or n_heads % world or d_ff % world:
        raise ConfigError(f"heads ({n_heads}/{n_kv_heads}) and d_ff ({d_ff}) must divide by world {world}")
    hq, hkv, ff = n_heads // world, n_kv_heads // world, d_ff // world
    return TPSlices(rank=rank, world=world, q_heads=(rank * hq, hq), kv_heads=(rank * hkv, hkv), ff=(rank * ff, ff))


def shard_layer_weights(lw: dict, cfg, sl: TPSlices) -> dict:
    """Slice one layer's [in, out] host weights (oracle/reference layout) for
    rank ``sl.rank``: column-parallel wq/wk/wv/gate/up, row-parallel wo/down."""
    dh = cfg.head_dim() if hasattr(cfg, "head_dim") else cfg.dh
    out = {
        "wq": lw["wq"][:, sl.q_cols(dh)],
        "wk": lw["wk"][:, sl.kv_cols(dh)],
        "wv": lw["wv"][:, sl.kv_cols(dh)],
        "wo": lw["wo"][sl.q_cols(dh), :],
        "w_up": lw["w_up"][:, sl.ff_cols()],
        "w_down": lw["w_down"][sl.ff_cols(), :],
    }
    if lw.get("w_gate") is not None:
        out["w_gate"] = lw["w_gate"][:, sl.ff_cols()]
    for k in ("attn_norm", "mlp_norm"):
        if k in lw:
            out[k] = lw[k]
    return out


def local_config(cfg, sl: TPSlices):
    """The per-rank model shape the kernels see (d_model stays full)."""
    from dataclasses import replace

    return replace(cfg, n_heads=sl.q_heads[1], n_kv_heads=sl.kv_heads[1], d_ff=sl.ff[1],
                   d_head=cfg.head_dim())


class _Peers(ctypes.Structure):
    """cc_tp_peers (include/cachecraft_b200.h)."""

    _fields_ = [("recv", ctypes.c_void_p * 8), ("flags", ctypes.c_void_p * 8), ("sum", ctypes.c_void_p * 8),
                ("done", ctypes.c_void_p * 8), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("slice", ctypes.c_int32), ("m_cap", ctypes.c_int32), ("epoch", ctypes.c_int32)]


class PeerComm:
    """One rank's view of the symmetric buffers of the fused TP reduction
    (csrc/tp_peer.cu): the o_proj / down_proj GEMM pushes each fp32 tile of
    its partial output into the column owner's ``recv`` slab over NVLink as it
    is produced (reduce-scatter fused into the epilogue); the owner sums the
    world's partials in rank order and stores the sum into every rank's
    ``sum`` (all-gather); each rank waits on its ``done`` counter and adds
    ``sum`` to its residual.  Replaces the NCCL all-reduce of those two
    reductions (model.py:417, :419) — NCCL stays for the small K8 masses."""

    def __init__(self, rank: int, world: int, d: int, m_cap: int, local: dict, ptrs: list):
        self.rank, self.world, self.d, self.m_cap = rank, world, d, m_cap
        self.slice = d // world
        self.local = local  # this rank's tensors (kept alive)
        self.ptrs = ptrs  # per rank: (recv, flags, sum, done) device pointers valid here
        self.epoch = 0
        self.done_target = 0

    @staticmethod
    def alloc(device, world: int, d: int, m_cap: int) -> dict:
        import torch

        slice_ = d // world
        n_m = -(-m_cap // 128)
        return {
            "recv": torch.zeros((world, m_cap, slice_), dtype=torch.float32, device=device),
            "flags": torch.full((world * n_m * (slice_ // 128) + 8,), -1, dtype=torch.int32, device=device),
            "sum": torch.zeros((m_cap, d), dtype=torch.float32, device=device),
            "done": torch.zeros((8,), dtype=torch.int32, device=device),
        }

    @classmethod
    def in_process(cls, world: int, d: int, m_cap: int, device) -> list:
        """All ranks' buffers in one process (tests; one GPU or P2P peers)."""
        if d % world or (d // world) % 128:
            raise ConfigError("peer TP needs d / world to be a multiple of 128")
        bufs = [cls.alloc(device, world, d, m_cap) for _ in range(world)]
        ptrs = [tuple(b[k].data_ptr() for k in ("recv", "flags", "sum", "done")) for b in bufs]
        return [cls(r, world, d, m_cap, bufs[r], ptrs) for r in range(world)]

    @classmethod
    def over_ipc(cls, rank: int, world: int, d: int, m_cap: int, device, group=None) -> "PeerComm":
        """One process per GPU: exchange CUDA-IPC handles of the symmetric
        buffers over torch.distributed and map every peer's buffers."""
        import torch.distributed as dist

        from . import _native as N

        if d % world or (d // world) % 128:
            raise ConfigError("peer TP needs d / world to be a multiple of 128")
        local = cls.alloc(device, world, d, m_cap)
        mine = []
        for k in ("recv", "flags", "sum", "done"):
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64()
            N.check(N.lib().cc_ipc_get_handle(ctypes.c_void_p(local[k].data_ptr()), h, ctypes.byref(off)),
                    "cc_ipc_get_handle")
            mine.append((h.raw, off.value))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        ptrs = []
        opened: dict = {}  # one mapping per peer allocation (buffers may share one)
        for r in range(world):
            if r == rank:
                ptrs.append(tuple(local[k].data_ptr() for k in ("recv", "flags", "sum", "done")))
                continue
            row = []
            for raw, off in allh[r]:
                if raw not in opened:
                    out = ctypes.c_void_p()
                    N.check(N.lib().cc_ipc_open_handle(ctypes.create_string_buffer(raw, 64), ctypes.byref(out)),
                            "cc_ipc_open_handle")
                    opened[raw] = out.value
                row.append(opened[raw] + off)
            ptrs.append(tuple(row))
        return cls(rank, world, d, m_cap, local, ptrs)

    def table(self) -> _Peers:
        t = _Peers()
        for r, (rv, fl, sm, dn) in enumerate(self.ptrs):
            t.recv[r], t.flags[r], t.sum[r], t.done[r] = rv, fl, sm, dn
        t.rank, t.world, t.slice, t.m_cap, t.epoch = self.rank, self.world, self.slice, self.m_cap, self.epoch
        return t


class TPContext:
    """What the engine needs to run one rank of a TP group: the slices and an
    all-reduce (sum, in place) over the group.  The default all-reduce is
    torch.distributed (NCCL on GPUs); tests inject their own.  With ``peer``
    (a PeerComm) the o_proj / down_proj reductions of bf16 runs use the
    fused push GEMM + peer reduction instead."""

    def __init__(self, slices: TPSlices, allreduce=None, group=None, peer: "PeerComm | None" = None):
        self.slices = slices
        self.group = group
        self._allreduce = allreduce
        self.peer = peer

    @property
    def world(self) -> int:
        return self.slices.world

    def allreduce_(self, t):
        if self.world == 1:
            return t
        if self._allreduce is not None:
            return self._allreduce(t)
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t


def split_rows(n: int, world: int, rank: int) -> slice:
    """Contiguous near-equal row range of ``rank`` (used for request lists)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return slice(lo, lo + base + (1 if rank < extra else 0))


def kv_slice_of(keys: np.ndarray, cfg, sl: TPSlices) -> np.ndarray:
    """A rank's kv-head columns of a reference-layout [n, Hkv*dh] K/V matrix."""
    return keys[:, sl.kv_cols(cfg.head_dim())]
