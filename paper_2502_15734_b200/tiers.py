"""Tiered chunk-cache pool and layer-wise preloading.

The reference models hierarchical placement and layer-wise preloading as a
discrete-event simulation (tiers.py:62-209).
Here the tiers are real memory:

* ``hbm``  — blocks of the model's paged HBM pool (``model.KVPool``); the K1
  gather reads them directly.
* ``host`` — one page-locked host tensor per variant, laid out
  ``[L][n_blocks][K|V][16][kv_width]`` so that a layer's slab of a variant
  is one contiguous range: one DMA per (variant, layer).
* ``disk`` — one raw file per variant (NVMe/SSD stand-in); promoted to the
  host tier by a background thread ("asynchronous preloading while the
  request is queued") and waited on at plan execution.

Layer-wise preloading (Algorithm 2) runs in
``engine.execute``: host-tier blocks of layer l are copied by the copy
engine on a side stream into a ring of ``L_p`` HBM layer slots while the
SMs compute earlier layers; layer l's K1 gather waits for its slot, and the
slot is released to layer l + L_p once that gather is done.  ``L_p`` is the
reference's ``preload_depth`` (tiers.py:62-71).

``Tier``, ``TierConfig``, ``preload_depth`` and ``place_and_migrate`` keep
the reference's names, fields, results and errors (checked against
reference fixtures).  The reference's discrete-event timeline simulator
(``simulate``, ``Timeline``, ``timeline_to_csv``) is out of scope: the tiers
here are real, and ``demote_slow_hits`` replaces its ``fallback_decision``
with a cost check on the measured host->HBM rate.
"""

from __future__ import annotations

import math
import os
import tempfile
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError, PlacementError, PlanError
from .model import BLOCK, ChunkCache, _Payload

HBM, HOST, DISK = "hbm", "host", "disk"


# ---------------------------------------------------------------------------
# placement policy and preload depth (reference tiers.py:27-71, :212-257)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Tier:
    """One storage level: ``bandwidth`` bytes/s, ``latency`` s per load,
    optional byte budget and the share of variants (by f_r rank) it targets."""

    name: str
    bandwidth: float
    latency: float = 0.0
    capacity_bytes: float | None = None
    placement_fraction: float | None = None


@dataclass(frozen=True)
class TierConfig:
    """Tiers ordered fastest first, plus the per-layer timing model."""

    tiers: tuple
    n_layers: int
    t_prefill_layer: float
    t_decode_step: float = 0.0
    t_compute_per_token: float = 0.0
    bytes_per_token_layer: float = 512.0

    def validate(self):
        if len(self.tiers) == 0:
            raise ArgumentError("need at least one tier")
        bad_bw = next((t for t in self.tiers if not t.bandwidth > 0), None)
        if bad_bw is not None:
            raise ArgumentError(f"tier {bad_bw.name} bandwidth must be positive")
        bad_lat = next((t for t in self.tiers if t.latency < 0), None)
        if bad_lat is not None:
            raise ArgumentError(f"tier {bad_lat.name} latency must be non-negative")
        if not (self.n_layers >= 1 and self.t_prefill_layer > 0):
            raise ArgumentError("layer count and per-layer prefill time must be positive")

    def tier(self, name: str) -> Tier:
        by_name = {t.name: t for t in reversed(self.tiers)}  # first definition wins
        if name not in by_name:
            raise ArgumentError(f"unknown tier {name!r}")
        return by_name[name]


def preload_depth(n_layers: int, t_prefill: float, t_load: float) -> int:
    """Layers to fetch ahead so compute never waits on a load (Algorithm 2,
    PAPER.md:758-776): L_p = ceil((L - 1)(1 - T_prefill/T_load) + 1), at least
    1 and at most L (the 1e-9 slack keeps exact integers from rounding up)."""
    if n_layers < 1:
        raise ArgumentError("layer count must be >= 1")
    if not (t_prefill > 0 and t_load > 0):
        raise ArgumentError("per-layer times must be positive")
    ahead = 1.0 + (n_layers - 1) * (1.0 - t_prefill / t_load)
    return int(np.clip(math.ceil(ahead - 1e-9), 1, n_layers))


def _band_sizes(n: int, tiers) -> list:
    """How many of the n ranked variants each tier's band targets: a tier's
    floor(fraction * n) (capped by what is left); the last tier, and any tier
    without a fraction, takes the remainder."""
    sizes, left = [], n
    for pos, t in enumerate(tiers):
        last = pos == len(tiers) - 1
        take = left if (last or t.placement_fraction is None) else min(left, math.floor(t.placement_fraction * n))
        sizes.append(int(take))
        left -= int(take)
    sizes[-1] += left
    return sizes


def place_and_migrate(variants, cfg: TierConfig) -> dict:
    """Assign every variant a tier: rank by reuse frequency (f_r desc, then
    older first, then lower id), cut the ranking into the tiers' bands, and
    let a variant whose band tier is out of budget spill to the next slower
    tier with room.  Returns {variant_id: tier name}; PlacementError if the
    fastest budget cannot hold the largest variant or nothing has room."""
    cfg.validate()
    ranked = sorted(variants, key=lambda v: (-v.f_r, v.created_at, v.variant_id))
    if not ranked:
        return {}
    sizes = [v.payload_bytes() for v in ranked]
    head = cfg.tiers[0]
    if head.capacity_bytes is not None and max(sizes) > head.capacity_bytes:
        raise PlacementError(
            f"fast tier budget {head.capacity_bytes} cannot hold the largest variant ({max(sizes)} bytes)")
    band = np.repeat(np.arange(len(cfg.tiers)), _band_sizes(len(ranked), cfg.tiers))
    room = [math.inf if t.capacity_bytes is None else float(t.capacity_bytes) for t in cfg.tiers]
    out = {}
    for v, nbytes, first in zip(ranked, sizes, band):
        fits = [k for k in range(int(first), len(cfg.tiers)) if nbytes <= room[k]]
        if not fits:
            raise PlacementError(f"no tier has room for variant {v.variant_id}")
        room[fits[0]] -= nbytes
        out[v.variant_id] = cfg.tiers[fits[0]].name
    return out


def demote_slow_hits(plan, model, disk_bytes_per_s: float = 3e9):
    """Real-tier counterpart of the reference's fallback_decision
    (tiers.py:260-299): a HIT whose payload sits in host memory or on disk is
    demoted to a MISS (fresh recompute) when streaming its K/V would take
    longer than recomputing the chunk.  With layer-wise preloading the load
    overlaps compute, so the test is load time vs the chunk's own share of
    the prefill: bytes / rate  >  tokens * L * (per-token-layer compute).
    HBM-resident hits are never demoted.  Returns a new InferencePlan."""
    from dataclasses import replace

    from .planner import HIT, MISS, InferencePlan

    cfg = model.kcfg
    d, q, kv, ff = cfg.d_model, cfg.q_width(), cfg.kv_width(), cfg.ff_dim()
    m = 3 if cfg.mlp == "swiglu" else 2
    # linear FLOPs per token per layer at the rate the engine's GEMMs sustain
    # (engine._estimate_layer_seconds uses the same figure)
    tok_layer_s = 2.0 * (d * (q + 2 * kv) + q * d + m * d * ff) / 1.0e15
    chunks = []
    for cp in plan.chunks:
        cache = getattr(cp, "cache", None)
        t = tier_of(cache) if (cp.status == HIT and cache is not None) else HBM
        if t in (HOST, DISK):
            nbytes = cache._payload.nbytes()
            rate = model.h2d_bytes_per_s if t == HOST else min(model.h2d_bytes_per_s, disk_bytes_per_s)
            if nbytes / rate > cp.n_tokens * cfg.n_layers * tok_layer_s:
                cp = replace(cp, status=MISS, variant_id=None, cfo=1.0, recompute=None, recompute_depth=None,
                             score=None, cache=None, n_slots=cp.n_tokens)
        chunks.append(cp)
    return InferencePlan(chunks=chunks, question=plan.question, alpha=plan.alpha, focus_window=plan.focus_window)


# ---------------------------------------------------------------------------
# payloads of the slower tiers
# ---------------------------------------------------------------------------


class HostPayload:
    """Page-locked host copy of one chunk cache: ``data`` [L][nb][2][16][kvw]
    (one contiguous slab per layer -> one DMA per layer)."""

    tier = HOST

    def __init__(self, data, n_slots: int, kvw: int, L: int):
        self.data = data  # torch pinned tensor
        self.n_slots = int(n_slots)
        self.kvw = kvw
        self.L = L

    @property
    def n_blocks(self) -> int:
        return self.data.shape[1]

    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    def all_rows(self, kv: int):
        """[L, n_slots, kvw] host tensor of K (kv=0) or V (kv=1)."""
        return self.data[:, :, kv].reshape(self.L, -1, self.kvw)[:, : self.n_slots]


class DiskPayload:
    """One raw file per variant (same byte layout as ``HostPayload``);
    ``prefetch`` starts the read into pinned memory on a background thread."""

    tier = DISK
    _pool = ThreadPoolExecutor(max_workers=4, thread_name_prefix="cc-disk")

    def __init__(self, path: str, shape, dtype, n_slots: int, kvw: int, L: int):
        self.path, self.shape, self.dtype = path, tuple(shape), dtype
        self.n_slots, self.kvw, self.L = int(n_slots), kvw, L
        self._future = None
        self._lock = threading.Lock()

    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * _elem_size(self.dtype)

    def _read(self) -> HostPayload:
        import torch

        data = torch.empty(self.shape, dtype=self.dtype, pin_memory=True)
        buf = data.view(torch.uint8).numpy().reshape(-1)
        with open(self.path, "rb", buffering=0) as fh:
            got = fh.readinto(memoryview(buf))
        if got != buf.size:
            raise PlanError(f"short read of disk-tier payload {self.path}")
        return HostPayload(data, self.n_slots, self.kvw, self.L)

    def prefetch(self):
        with self._lock:
            if self._future is None:
                self._future = self._pool.submit(self._read)
        return self._future

    def load(self) -> HostPayload:
        return self.prefetch().result()

    def drop(self):
        try:
            os.unlink(self.path)
        except OSError:
            pass


def _elem_size(dtype) -> int:
    import torch

    return torch.empty((), dtype=dtype).element_size()


def tier_of(cache: ChunkCache) -> str:
    p = cache._payload
    if p is None:
        return "none"
    return getattr(p, "tier", HBM)


# ---------------------------------------------------------------------------
# migration between tiers
# ---------------------------------------------------------------------------


class TieredPool:
    """Moves chunk-cache payloads between HBM, pinned host and disk for one
    model.  Payload objects are immutable once written, so a migration
    swaps the cache's payload (the old HBM blocks return to the pool when
    their last reference dies)."""

    def __init__(self, model, disk_dir: str | None = None):
        self.model = model
        self.disk_dir = disk_dir or tempfile.mkdtemp(prefix="cc_b200_tier_")
        self._seq = 0

    # -- HBM <-> host -------------------------------------------------------
    def to_host(self, cache: ChunkCache) -> HostPayload:
        import torch

        p = self._resolve(cache)
        if isinstance(p, HostPayload):
            return p
        pool = self.model.pool
        idx = torch.from_numpy(p.blocks.astype(np.int64)).to(pool.storage.device)
        dev = pool.storage[:, idx]  # [L, nb, 2, 16, kvw] (gathered copy)
        host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
        host.copy_(dev)
        hp = HostPayload(host, p.n_slots, pool.kvw, pool.L)
        cache._payload = hp
        cache._payload_from_host = False
        return hp

    def to_hbm(self, cache: ChunkCache) -> _Payload:
        import torch

        p = self._resolve(cache)
        if isinstance(p, _Payload):
            return p
        pool = self.model.pool
        blocks = pool.alloc(p.n_blocks)
        idx = torch.from_numpy(blocks.astype(np.int64)).to(pool.storage.device)
        pool.storage[:, idx] = p.data.to(pool.storage.device, non_blocking=False)
        dp = _Payload(pool, blocks, p.n_slots)
        cache._payload = dp
        cache._payload_from_host = False
        return dp

    # -- host <-> disk --------------------------------------------------------
    def to_disk(self, cache: ChunkCache) -> DiskPayload:
        p = cache._payload
        if isinstance(p, DiskPayload):
            return p
        hp = p if isinstance(p, HostPayload) else self.to_host(cache)
        self._seq += 1
        path = os.path.join(self.disk_dir, f"variant_{id(cache):x}_{self._seq}.kv")
        raw = hp.data.view(__import__("torch").uint8).numpy()
        with open(path, "wb") as fh:
            fh.write(memoryview(raw.reshape(-1)))
        dp = DiskPayload(path, tuple(hp.data.shape), hp.data.dtype, hp.n_slots, hp.kvw, hp.L)
        cache._payload = dp
        return dp

    def _resolve(self, cache: ChunkCache):
        """The cache's payload, uploading host arrays / reading disk first."""
        p = cache._payload
        if p is None:
            p = cache.device_payload(self.model)
        if isinstance(p, DiskPayload):
            hp = p.load()
            p.drop()
            cache._payload = hp
            p = hp
        return p

    def move(self, cache: ChunkCache, tier: str):
        if tier == HBM:
            return self.to_hbm(cache)
        if tier == HOST:
            return self.to_host(cache)
        if tier == DISK:
            return self.to_disk(cache)
        raise ArgumentError(f"unknown tier {tier!r}")

    def apply_placement(self, store, placement: dict):
        """Migrate every variant of ``store`` to the tier ``placement`` names
        for it (the output of ``place_and_migrate``)."""
        for vid, tier in placement.items():
            v = store.get(vid)
            self.move(v.cache, tier)

    @staticmethod
    def prefetch(plan) -> int:
        """Start disk -> host reads for every HIT variant of an inference
        plan that lives on disk (asynchronous preloading while queued).
        Returns the number of reads started."""
        n = 0
        for cp in plan.chunks:
            cache = getattr(cp, "cache", None)
            if cache is not None and isinstance(cache._payload, DiskPayload):
                cache._payload.prefetch()
                n += 1
        return n


def calibrate_h2d(model, nbytes: int = 256 << 20) -> float:
    """Measure the pinned-host -> HBM copy-engine rate on this box (bytes/s)
    and store it on the model for the preload depth."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=model.device)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    rate = 3 * nbytes / (a.elapsed_time(b) / 1e3)
    model.h2d_bytes_per_s = rate
    return rate


def host_slab_bytes(payloads) -> int:
    """Bytes of one layer's host-tier slabs of a request."""
    return sum(p.n_blocks * 2 * BLOCK * p.kvw * p.data.element_size() for p in payloads)
