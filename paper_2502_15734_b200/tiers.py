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
the reference's names, fields, arithmetic and errors (checked against
reference fixtures); the timeline simulator itself is out of scope.
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
# reference control logic (tiers.py:27-71, :209-261)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Tier:
    name: str
    bandwidth: float  # bytes/s
    latency: float = 0.0  # fixed seconds per load operation
    capacity_bytes: float | None = None
    placement_fraction: float | None = None  # share of variants targeted, by f_r rank


@dataclass(frozen=True)
class TierConfig:
    tiers: tuple  # ordered fast -> slow
    n_layers: int
    t_prefill_layer: float
    t_decode_step: float = 0.0
    t_compute_per_token: float = 0.0
    bytes_per_token_layer: float = 512.0

    def validate(self):
        if not self.tiers:
            raise ArgumentError("need at least one tier")
        for tier in self.tiers:
            if tier.bandwidth <= 0:
                raise ArgumentError(f"tier {tier.name} bandwidth must be positive")
            if tier.latency < 0:
                raise ArgumentError(f"tier {tier.name} latency must be non-negative")
        if self.n_layers < 1 or self.t_prefill_layer <= 0:
            raise ArgumentError("layer count and per-layer prefill time must be positive")

    def tier(self, name: str) -> Tier:
        for tier in self.tiers:
            if tier.name == name:
                return tier
        raise ArgumentError(f"unknown tier {name!r}")


def preload_depth(n_layers: int, t_prefill: float, t_load: float) -> int:
    """Smallest layer count to fetch ahead so computation never stalls:
    L_p = ceil((L - 1)(1 - T_prefill / T_load) + 1), clamped to [1, L]
    (tiers.py:62-71, PAPER.md eq. layerwise)."""
    if n_layers < 1:
        raise ArgumentError("layer count must be >= 1")
    if t_prefill <= 0 or t_load <= 0:
        raise ArgumentError("per-layer times must be positive")
    raw = (n_layers - 1) * (1.0 - t_prefill / t_load) + 1.0
    depth = max(1, math.ceil(raw - 1e-9))
    return min(depth, n_layers)


def place_and_migrate(variants, cfg: TierConfig) -> dict:
    """Partition variants into tiers by f_r rank bands, respecting byte
    budgets (spill to the next slower tier when a band is full)
    (tiers.py:209-261).  Returns {variant_id: tier name}."""
    cfg.validate()
    variants = sorted(variants, key=lambda v: (-v.f_r, v.created_at, v.variant_id))
    if not variants:
        return {}
    fast = cfg.tiers[0]
    largest = max(v.payload_bytes() for v in variants)
    if fast.capacity_bytes is not None and largest > fast.capacity_bytes:
        raise PlacementError(
            f"fast tier budget {fast.capacity_bytes} cannot hold the largest variant ({largest} bytes)")
    n = len(variants)
    targets = []
    assigned = 0
    for idx, tier in enumerate(cfg.tiers):
        if idx == len(cfg.tiers) - 1 or tier.placement_fraction is None:
            targets.append(n - assigned)
            assigned = n
        else:
            count = min(n - assigned, int(math.floor(tier.placement_fraction * n)))
            targets.append(count)
            assigned += count
    if assigned < n:
        targets[-1] += n - assigned
    placement = {}
    used = [0.0] * len(cfg.tiers)
    band_of = []
    for band, count in enumerate(targets):
        band_of.extend([band] * count)
    for variant, band in zip(variants, band_of):
        placed = False
        for idx in range(band, len(cfg.tiers)):
            tier = cfg.tiers[idx]
            size = variant.payload_bytes()
            if tier.capacity_bytes is None or used[idx] + size <= tier.capacity_bytes:
                placement[variant.variant_id] = tier.name
                used[idx] += size
                placed = True
                break
        if not placed:
            raise PlacementError(f"no tier has room for variant {variant.variant_id}")
    return placement


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
