"""Model, chunk-cache and request types of the fix-up prefill path, with the
weights and KV payloads resident in B200 HBM.

Mirrors the reference's engine types (cachecraft/model.py:36-492): the same
names, fields, validation and error behaviour; the tensor work behind
``prefill`` / ``Model.logits`` / ``extract_chunk_cache`` runs in the CUDA
library through ``engine.py``.  Host-side numpy views (``ChunkCache.keys``,
``PrefillResult.hidden``, ...) are materialised lazily from device memory.

Extensions over the reference ``ModelConfig`` (all defaulting to the
reference architecture): ``n_kv_heads`` (GQA), ``d_ff``, ``mlp``
("gelu_tanh" | "swiglu"), ``norm_weight``, ``rms_eps`` and ``dtype``
("fp64" | "fp32" parity modes, "bf16" performance mode).
"""

from __future__ import annotations

import math
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigError, PlanError, ShapeError
from .rpe import DEFAULT_BASE

FULL_DEPTH = -1  # model.py:32 sentinel: recompute through every layer
BLOCK = 16  # pool block rows (store.py:18)
_DTYPES = {"fp64": N.F64, "fp32": N.F32, "bf16": N.BF16}


# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ModelConfig:
    """Shape, seed and numeric mode of the model (model.py:36-67)."""

    n_layers: int = 4
    n_heads: int = 4
    d_model: int = 64
    d_head: int | None = None
    vocab_size: int = 256
    rpe_base: float = DEFAULT_BASE
    seed: int = 0
    n_kv_heads: int | None = None
    d_ff: int | None = None
    mlp: str = "gelu_tanh"
    norm_weight: bool = False
    rms_eps: float = 1e-6
    dtype: str = "fp64"

    def head_dim(self) -> int:
        return self.d_model // self.n_heads if self.d_head is None else self.d_head

    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    def ff_dim(self) -> int:
        return 4 * self.d_model if self.d_ff is None else self.d_ff

    def kv_width(self) -> int:
        return self.kv_heads() * self.head_dim()

    def q_width(self) -> int:
        return self.n_heads * self.head_dim()

    def validate(self):
        if self.n_layers < 1 or self.n_heads < 1 or self.d_model < 1:
            raise ConfigError("layer, head, and dimension counts must be positive")
        if self.vocab_size < 2:
            raise ConfigError("vocab_size must be at least 2")
        dh = self.head_dim()
        if dh % 2 != 0:
            raise ConfigError(f"d_head must be even for pairwise rotation, got {dh}")
        if self.d_head is None and self.d_model != self.n_heads * dh:
            raise ConfigError(f"d_model ({self.d_model}) != n_heads ({self.n_heads}) * d_head ({dh})")
        if self.d_head is not None and self.d_head * self.n_heads != self.d_model and self.n_kv_heads is None:
            raise ConfigError(f"d_model ({self.d_model}) != n_heads ({self.n_heads}) * d_head ({dh})")
        if self.rpe_base <= 0:
            raise ConfigError("rpe_base must be positive")
        if self.kv_heads() < 1 or self.n_heads % self.kv_heads() != 0:
            raise ConfigError("n_heads must be a multiple of n_kv_heads")
        if self.mlp not in ("gelu_tanh", "swiglu"):
            raise ConfigError(f"unknown mlp {self.mlp!r}")
        if self.mlp == "swiglu" and self.ff_dim() % 64 != 0:
            raise ConfigError("swiglu d_ff must be a multiple of 64 (gate|up column groups)")
        if self.dtype not in _DTYPES:
            raise ConfigError(f"dtype must be one of {sorted(_DTYPES)}")
        if self.dtype == "bf16":
            why = self.tensor_core_shape_error()
            if why:
                raise ConfigError(f"bf16 mode runs the tcgen05 kernels only (no fallback): {why}; "
                                  "use dtype='fp32' or 'fp64' for this shape")

    def tensor_core_shape_error(self) -> str | None:
        """Why the bf16 tcgen05 GEMM / attention kernels cannot run this
        shape (None if they can): d_head 64 or 128, a GQA group dividing
        128, d_model / q width / ff multiples of 128 and a QKV width
        multiple of 128 (the 128-row tiles and 64-deep k-blocks)."""
        dh, g = self.head_dim(), self.n_heads // self.kv_heads()
        if dh not in (64, 128):
            return f"d_head {dh} not in (64, 128)"
        if 128 % g:
            return f"GQA group {g} does not divide 128"
        for name, v in (("d_model", self.d_model), ("q width", self.q_width()), ("d_ff", self.ff_dim()),
                        ("QKV width", self.q_width() + 2 * self.kv_width())):
            if v % 128:
                return f"{name} {v} is not a multiple of 128"
        return None

    # Llama-3 shaped presets (random init; the reference has no such config)
    @classmethod
    def llama3_8b(cls, n_layers=32, dtype="bf16", seed=0):
        return cls(n_layers=n_layers, n_heads=32, d_model=4096, d_head=128, vocab_size=128256, rpe_base=500000.0,
                   seed=seed, n_kv_heads=8, d_ff=14336, mlp="swiglu", norm_weight=True, rms_eps=1e-5, dtype=dtype)

    @classmethod
    def llama3_70b(cls, n_layers=80, dtype="bf16", seed=0):
        return cls(n_layers=n_layers, n_heads=64, d_model=8192, d_head=128, vocab_size=128256, rpe_base=500000.0,
                   seed=seed, n_kv_heads=8, d_ff=28672, mlp="swiglu", norm_weight=True, rms_eps=1e-5, dtype=dtype)

    def n_params(self) -> int:
        d, q, kv, ff = self.d_model, self.q_width(), self.kv_width(), self.ff_dim()
        per = d * q + 2 * d * kv + q * d + (3 if self.mlp == "swiglu" else 2) * d * ff
        return 2 * self.vocab_size * d + self.n_layers * per


@dataclass(frozen=True)
class LayerWeights:
    """Host view of one layer's weights, [in, out] like the reference."""

    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray
    w_gate: np.ndarray | None = None


# ---------------------------------------------------------------------------
# device KV pool: position-free K/V in 16-row blocks, [L][block][K|V][16][kvw]
# ---------------------------------------------------------------------------


class KVPool:
    """Paged HBM pool holding every chunk-cache payload of one model.

    Blocks are reference-counted through ``_Payload`` finalizers; the pool
    grows by doubling (block ids stay valid, raw pointers do not — callers
    read ``storage`` at launch time)."""

    def __init__(self, model: "Model", n_blocks: int = 256):
        import torch

        cfg = model.kcfg
        self.L, self.kvw = cfg.n_layers, cfg.kv_width()
        self.torch_dtype = model.torch_dtype
        self.storage = torch.zeros((self.L, n_blocks, 2, BLOCK, self.kvw), dtype=self.torch_dtype, device=model.device)
        self._free = list(range(n_blocks - 1, -1, -1))

    @property
    def n_blocks(self) -> int:
        return self.storage.shape[1]

    @property
    def layer_stride(self) -> int:
        return self.storage.stride(0)

    @property
    def block_stride(self) -> int:
        return self.storage.stride(1)

    def blocks_in_use(self) -> int:
        return self.n_blocks - len(self._free)

    def reserve(self, n_blocks: int):
        """Grow capacity to at least ``n_blocks`` blocks."""
        import torch

        old = self.n_blocks
        if n_blocks <= old:
            return
        new = torch.zeros((self.L, n_blocks, 2, BLOCK, self.kvw), dtype=self.torch_dtype, device=self.storage.device)
        new[:, :old].copy_(self.storage)
        self.storage = new
        self._free = list(range(n_blocks - 1, old - 1, -1)) + self._free

    def alloc(self, count: int) -> np.ndarray:
        if count > len(self._free):
            self.reserve(max(2 * self.n_blocks, self.blocks_in_use() + count))
        ids = [self._free.pop() for _ in range(count)]
        return np.asarray(ids, dtype=np.int32)

    def free(self, ids):
        self._free.extend(int(i) for i in ids)


class _Payload:
    """Device-resident K/V of one chunk cache: pool blocks + slot count."""

    def __init__(self, pool: KVPool, blocks: np.ndarray, n_slots: int, base: "_Payload | None" = None):
        self.pool = pool
        self.blocks = blocks
        self.n_slots = n_slots
        self._base = base  # a view keeps its base (and the blocks) alive
        self._fin = None if base is not None else weakref.finalize(self, KVPool.free, pool, blocks.tolist())

    def layer_rows(self, layer: int, kv: int):
        """[n_slots, kvw] device view (copy) of K (kv=0) or V (kv=1) rows."""
        import torch

        idx = torch.from_numpy(self.blocks.astype(np.int64)).to(self.pool.storage.device)
        rows = self.pool.storage[layer, idx, kv]  # [nb, 16, kvw]
        return rows.reshape(-1, self.pool.kvw)[: self.n_slots]

    def all_rows(self, kv: int):
        import torch

        idx = torch.from_numpy(self.blocks.astype(np.int64)).to(self.pool.storage.device)
        rows = self.pool.storage[:, idx, kv]  # [L, nb, 16, kvw]
        return rows.reshape(self.pool.L, -1, self.pool.kvw)[:, : self.n_slots]


# ---------------------------------------------------------------------------
# model
# ---------------------------------------------------------------------------


class Model:
    """Weights resident on the GPU (K-major [out, in] layout) + the KV pool."""

    def copy_stream(self):
        """Side stream of the layer-wise host-tier preload (created once)."""
        import torch

        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        return self._copy_stream

    def __init__(self, config: ModelConfig, weights: dict, device, host_weights: dict | None = None, tp=None):
        import torch

        self.config = config
        self.tp = tp  # parallel.TPContext or None
        # host -> HBM copy-engine rate used for the preload depth (tiers.py);
        # tiers.calibrate_h2d measures it on this box
        self.h2d_bytes_per_s = 50e9
        self._copy_stream = None
        self.l2_prefetch = False  # o_proj weights -> L2 during attention: measured -1% (noise level), off
        # programmatic dependent launch for the prefill chain: each kernel's
        # prologue (barriers, TMEM, first weight tiles) overlaps its predecessor
        self.prefill_pdl = os.environ.get("CCB_PDL", "1") != "0"
        if tp is not None and tp.world > 1:
            from .parallel import local_config

            self.kcfg = local_config(config, tp.slices)  # rank-local head / MLP shape for the kernels
        else:
            self.kcfg = config
        self.device = device
        self.w = weights
        self.dtype_code = _DTYPES[config.dtype]
        self.torch_dtype = {"fp64": torch.float64, "fp32": torch.float32, "bf16": torch.bfloat16}[config.dtype]
        self.hidden_dtype = torch.float64 if config.dtype == "fp64" else torch.float32
        self._host = host_weights
        self._pool = None
        self._rope = None

    # -- pool / rope table ------------------------------------------------------
    @property
    def pool(self) -> KVPool:
        if self._pool is None:
            self._pool = KVPool(self)
        return self._pool

    def rope_table(self, max_pos: int):
        """Device (cos, sin) table for positions [0, max_pos), fp64 angles."""
        import torch

        from .rpe import inv_freq

        if self._rope is None or self._rope[0] < max_pos:
            cap = 1 << max(10, int(math.ceil(math.log2(max(max_pos, 2)))))
            half = self.config.head_dim() // 2
            f = torch.from_numpy(inv_freq(self.config.rpe_base, self.config.head_dim())).to(self.device)
            elem = torch.float64 if self.config.dtype == "fp64" else torch.float32
            tab = torch.empty((cap, half, 2), dtype=elem, device=self.device)
            N.call("cc_rope_table", N.ptr(tab), N.ptr(f), cap, half, self.dtype_code, N.stream_ptr())
            self._rope = (cap, tab)
        return self._rope[1]

    # -- reference API ------------------------------------------------------------
    def logits(self, hidden_rows) -> np.ndarray:
        """rmsnorm(h) @ unembed (model.py:94-95), computed on the GPU."""
        from .engine import logits_device

        return logits_device(self, hidden_rows)[0]

    @property
    def layers(self) -> tuple:
        return tuple(self._host_weights()["layers"])

    @property
    def embed(self) -> np.ndarray:
        return self._host_weights()["embed"]

    @property
    def unembed(self) -> np.ndarray:
        return self._host_weights()["unembed"]

    def weight_bytes(self) -> bytes:
        hw = self._host_weights()
        parts = [hw["embed"].tobytes(), hw["unembed"].tobytes()]
        for lw in hw["layers"]:
            for w in (lw.wq, lw.wk, lw.wv, lw.wo, lw.w_gate, lw.w_up, lw.w_down):
                if w is not None:
                    parts.append(w.tobytes())
        return b"".join(parts)

    def _host_weights(self) -> dict:
        """[in, out] host views recovered from the device layout."""
        if self._host is None:
            cfg = self.config
            q, kv, ff = cfg.q_width(), cfg.kv_width(), cfg.ff_dim()

            def h(t):
                return t.float().cpu().numpy().astype(np.float64) if cfg.dtype == "bf16" else t.cpu().numpy()

            layers = []
            for lw in self.w["layers"]:
                qkv = h(lw["w_qkv"]).T
                if cfg.mlp == "swiglu":
                    gu = h(lw["w_gu"]).reshape(ff // 64, 2, 64, cfg.d_model)
                    gate = gu[:, 0].reshape(ff, cfg.d_model).T
                    up = gu[:, 1].reshape(ff, cfg.d_model).T
                else:
                    gate, up = None, h(lw["w_up"]).T
                layers.append(LayerWeights(wq=qkv[:, :q], wk=qkv[:, q:q + kv], wv=qkv[:, q + kv:], wo=h(lw["w_o"]).T,
                                           w_up=up, w_down=h(lw["w_down"]).T, w_gate=gate))
            self._host = {"embed": h(self.w["embed"]), "unembed": h(self.w["unembed_t"]).T, "layers": layers}
        return self._host


def _draw_host(config: ModelConfig) -> dict:
    """Seeded numpy draw in the reference order (model.py:103-116); the
    extension adds w_gate before w_up for SwiGLU."""
    g = np.random.default_rng(config.seed)
    d, q, kv, ff = config.d_model, config.q_width(), config.kv_width(), config.ff_dim()

    def normal(r, c, fan=None):
        m = g.standard_normal((r, c))
        return m if fan is None else m / np.sqrt(fan)

    embed = normal(config.vocab_size, d)
    unembed = normal(d, config.vocab_size, d)
    layers = []
    for _ in range(config.n_layers):
        wq, wk, wv, wo = normal(d, q, d), normal(d, kv, d), normal(d, kv, d), normal(q, d, q)
        gate = normal(d, ff, d) if config.mlp == "swiglu" else None
        up, down = normal(d, ff, d), normal(ff, d, ff)
        layers.append(LayerWeights(wq=wq, wk=wk, wv=wv, wo=wo, w_up=up, w_down=down, w_gate=gate))
    return {"embed": embed, "unembed": unembed, "layers": layers}


def build_model(config: ModelConfig, device=None, host_draw: bool | None = None, tp=None) -> Model:
    """Fill all weights from a seeded stream (model.py:98-118) and place them
    on the GPU.  Small models use the reference's numpy stream exactly (so
    fp64 mode reproduces the reference weights bit for bit); large
    (Llama-shaped) models are drawn on the device with a seeded torch
    generator, N(0,1)/sqrt(fan_in), norms = 1.

    ``tp`` (a ``parallel.TPContext``) builds one tensor-parallel rank: its
    slice of the host-drawn weights (so ranks compose exactly into the full
    model), or for device-drawn (large) models its own seeded shard."""
    import torch

    config.validate()
    N.require_cuda()
    dev = torch.device("cuda") if device is None else torch.device(device)
    tdt = {"fp64": torch.float64, "fp32": torch.float32, "bf16": torch.bfloat16}[config.dtype]
    sl = tp.slices if (tp is not None and tp.world > 1) else None
    kc = config
    if sl is not None:
        from .parallel import local_config, shard_layer_weights

        kc = local_config(config, sl)
    d, q, kv, ff = kc.d_model, kc.q_width(), kc.kv_width(), kc.ff_dim()
    if host_draw is None:
        host_draw = config.n_params() <= 64_000_000
    host = _draw_host(config) if host_draw else None
    if host is not None and sl is not None:
        full = host
        host = {"embed": full["embed"], "unembed": full["unembed"], "layers": []}
        for hl in full["layers"]:
            sh = shard_layer_weights({"wq": hl.wq, "wk": hl.wk, "wv": hl.wv, "wo": hl.wo, "w_up": hl.w_up,
                                      "w_down": hl.w_down, "w_gate": hl.w_gate}, config, sl)
            host["layers"].append(LayerWeights(wq=sh["wq"], wk=sh["wk"], wv=sh["wv"], wo=sh["wo"], w_up=sh["w_up"],
                                               w_down=sh["w_down"], w_gate=sh.get("w_gate")))
    seed = config.seed if sl is None else config.seed * 1000003 + sl.rank
    gen = None if host_draw else torch.Generator(device=dev).manual_seed(seed)

    def dev_normal(r, c, fan):
        t = torch.randn((r, c), generator=gen, device=dev, dtype=torch.float32)
        if fan is not None:
            t.mul_(1.0 / math.sqrt(fan))
        return t

    def put(arr_in_out):  # [in, out] host -> [out, in] device
        return torch.from_numpy(np.ascontiguousarray(arr_in_out.T)).to(dev, tdt)

    w: dict = {"layers": []}
    if host_draw:
        w["embed"] = torch.from_numpy(host["embed"]).to(dev, tdt)
        w["unembed_t"] = put(host["unembed"])
    else:
        w["embed"] = dev_normal(config.vocab_size, d, None).to(tdt)
        w["unembed_t"] = dev_normal(d, config.vocab_size, d).t().contiguous().to(tdt)
    for li in range(config.n_layers):
        if host_draw:
            hl = host["layers"][li]
            wq, wk, wv, wo = put(hl.wq), put(hl.wk), put(hl.wv), put(hl.wo)
            gate = put(hl.w_gate) if hl.w_gate is not None else None
            up, down = put(hl.w_up), put(hl.w_down)
        else:
            wq = dev_normal(d, q, d).t().contiguous().to(tdt)
            wk = dev_normal(d, kv, d).t().contiguous().to(tdt)
            wv = dev_normal(d, kv, d).t().contiguous().to(tdt)
            wo = dev_normal(q, d, q).t().contiguous().to(tdt)
            gate = dev_normal(d, ff, d).t().contiguous().to(tdt) if config.mlp == "swiglu" else None
            up = dev_normal(d, ff, d).t().contiguous().to(tdt)
            down = dev_normal(ff, d, ff).t().contiguous().to(tdt)
        lw = {"w_qkv": torch.cat([wq, wk, wv], dim=0).contiguous(), "w_o": wo, "w_down": down}
        if config.mlp == "swiglu":
            lw["w_gu"] = torch.stack([gate.reshape(ff // 64, 64, d), up.reshape(ff // 64, 64, d)], dim=1).reshape(2 * ff, d).contiguous()
        else:
            lw["w_up"] = up
        if config.norm_weight:
            lw["attn_norm"] = torch.ones(d, dtype=torch.float32, device=dev)
            lw["mlp_norm"] = torch.ones(d, dtype=torch.float32, device=dev)
        w["layers"].append(lw)
        del wq, wk, wv, wo, gate, up, down
    if config.norm_weight:
        w["final_norm"] = torch.ones(d, dtype=torch.float32, device=dev)
    host_view = None
    if host is not None and config.dtype == "fp64" and sl is None:
        host_view = host
    return Model(config, w, dev, host_view, tp=tp)


# ---------------------------------------------------------------------------
# chunk caches, segments, requests
# ---------------------------------------------------------------------------


def _host_layers(t) -> list:
    """[L, rows, w] device tensor -> list of float64 numpy arrays."""
    import torch

    if t.dtype != torch.float64:
        t = t.double()
    return list(t.cpu().numpy())


class ChunkCache:
    """Per-layer position-free K/V rows of one chunk (model.py:130-156).

    Constructed either from host arrays (reference signature) — uploaded to
    the model's HBM pool on first use — or device-first by
    ``extract_chunk_cache`` / the store.  Pad rows trail the real rows."""

    def __init__(self, keys=None, values=None, n_tokens: int = 0, source_prefix: tuple = (), *, _payload=None):
        self._keys = list(keys) if keys is not None else None
        self._values = list(values) if values is not None else None
        self.n_tokens = int(n_tokens)
        self.source_prefix = tuple(source_prefix)
        self._payload = _payload
        self._payload_from_host = False
        if self._keys is None and _payload is None:
            raise ShapeError("ChunkCache needs keys/values or a device payload")

    # reference fields materialise lazily from HBM (or the host / disk tier)
    def _rows(self, kv: int):
        p = self._payload
        if getattr(p, "tier", None) == "disk":
            p = self._payload = p.load()
        return p.all_rows(kv)

    @property
    def keys(self) -> list:
        if self._keys is None:
            self._keys = _host_layers(self._rows(0))
        return self._keys

    @keys.setter
    def keys(self, v):
        self._keys = list(v)
        self._drop_host_payload()

    @property
    def values(self) -> list:
        if self._values is None:
            self._values = _host_layers(self._rows(1))
        return self._values

    @values.setter
    def values(self, v):
        self._values = list(v)
        self._drop_host_payload()

    def _drop_host_payload(self):
        if self._payload_from_host:
            self._payload = None

    @property
    def n_slots(self) -> int:
        if self._payload is not None:
            return self._payload.n_slots
        return self._keys[0].shape[0]

    @property
    def n_layers(self) -> int:
        if self._payload is not None:
            return self._payload.pool.L if hasattr(self._payload, "pool") else self._payload.L
        return len(self._keys)

    @property
    def width(self) -> int:
        if self._payload is not None:
            return self._payload.pool.kvw if hasattr(self._payload, "pool") else self._payload.kvw
        return self._keys[0].shape[1]

    def copy(self) -> "ChunkCache":
        """Deep copy.  Device payloads are immutable once written, so the copy
        shares them; host arrays are copied."""
        c = ChunkCache(
            keys=[k.copy() for k in self._keys] if self._keys is not None else None,
            values=[v.copy() for v in self._values] if self._values is not None else None,
            n_tokens=self.n_tokens,
            source_prefix=self.source_prefix,
            _payload=self._payload,
        )
        c._payload_from_host = self._payload_from_host
        return c

    def device_payload(self, model: Model) -> _Payload:
        """The cache's rows in ``model``'s pool, uploading host rows if needed."""
        import torch

        p = self._payload
        if p is not None and getattr(p, "pool", None) is model.pool:
            return p
        tier = getattr(p, "tier", None)
        if tier == "disk":  # asynchronous read started by tiers.TieredPool.prefetch (or now)
            p = self._payload = p.load()
            tier = "host"
        if tier == "host" and p.L == model.kcfg.n_layers and p.kvw == model.kcfg.kv_width():
            return p  # gathered layer by layer through the copy engine (engine.execute)
        keys, values = self.keys, self.values
        if model.tp is not None and model.tp.world > 1 and keys[0].shape[1] == model.config.kv_width():
            cols = model.tp.slices.kv_cols(model.config.head_dim())
            keys = [np.asarray(k)[:, cols] for k in keys]
            values = [np.asarray(v)[:, cols] for v in values]
        n = keys[0].shape[0]
        nb = max(1, -(-n // BLOCK))
        pool = model.pool
        blocks = pool.alloc(nb)
        L, kvw = pool.L, pool.kvw
        buf = torch.zeros((L, nb * BLOCK, 2, kvw), dtype=torch.float64)
        buf[:, :n, 0] = torch.from_numpy(np.stack([np.asarray(k, dtype=np.float64) for k in keys]))
        buf[:, :n, 1] = torch.from_numpy(np.stack([np.asarray(v, dtype=np.float64) for v in values]))
        dev = buf.to(pool.storage.device, pool.torch_dtype).reshape(L, nb, BLOCK, 2, kvw).permute(0, 1, 3, 2, 4)
        idx = torch.from_numpy(blocks.astype(np.int64)).to(pool.storage.device)
        pool.storage[:, idx] = dev
        self._payload = _Payload(pool, blocks, n)
        self._payload_from_host = True
        return self._payload


@dataclass
class Segment:
    """Fresh text, or an injected chunk-cache with optional recompute mask and
    per-token recompute depth (model.py:160-171)."""

    tokens: np.ndarray
    cache: ChunkCache | None = None
    recompute: np.ndarray | None = None
    recompute_depth: np.ndarray | None = None


def _segment_layout(seg: Segment, first_position: int):
    """Per-slot arrays of one segment: ids, positions, pad, mask, depth
    (model.py:199-238 semantics)."""
    toks = np.asarray(seg.tokens, dtype=np.int64).reshape(-1)
    nt = toks.size
    if nt == 0:
        raise PlanError("empty segment")
    if seg.cache is None:
        if seg.recompute is not None or seg.recompute_depth is not None:
            raise PlanError("fresh-text segments are always fully recomputed")
        return (toks, first_position + np.arange(nt), np.zeros(nt, bool), np.ones(nt, bool),
                np.full(nt, FULL_DEPTH, np.int64), nt)
    if seg.cache.n_tokens != nt:
        raise PlanError(f"injected cache holds {seg.cache.n_tokens} tokens, segment declares {nt}")
    ns = seg.cache.n_slots
    mask = np.zeros(ns, bool)
    if seg.recompute is not None:
        rc = np.asarray(seg.recompute, dtype=bool)
        if rc.shape != (nt,):
            raise PlanError("recompute mask length != segment token count")
        mask[:nt] = rc
    depth = np.zeros(ns, np.int64)
    if seg.recompute_depth is not None:
        dp = np.asarray(seg.recompute_depth, dtype=np.int64)
        if dp.shape != (nt,):
            raise PlanError("recompute depth length != segment token count")
        depth[:nt] = np.where(mask[:nt], dp, 0)
    else:
        depth[:nt] = np.where(mask[:nt], FULL_DEPTH, 0)
    ids = np.zeros(ns, np.int64)
    ids[:nt] = toks
    pos = np.full(ns, -1, np.int64)
    pos[:nt] = first_position + np.arange(nt)
    pad = np.arange(ns) >= nt
    return ids, pos, pad, mask, depth, ns


@dataclass
class PrefillRequest:
    """Resolved slot layout of one prefill call (model.py:175-270)."""

    segments: list
    question: np.ndarray
    token_ids: np.ndarray = field(init=False)
    positions: np.ndarray = field(init=False)
    is_pad: np.ndarray = field(init=False)
    recompute_mask: np.ndarray = field(init=False)
    recompute_depth: np.ndarray = field(init=False)
    question_span: tuple = field(init=False)
    segment_slots: list = field(init=False)

    def __post_init__(self):
        cols = ([], [], [], [], [])
        self.segment_slots = []
        slot, position = 0, 0
        for seg in self.segments:
            ids, pos, pad, mask, depth, ns = _segment_layout(seg, position)
            for acc, a in zip(cols, (ids, pos, pad, mask, depth)):
                acc.append(a)
            n_real = int(np.asarray(seg.tokens).size)
            self.segment_slots.append((slot, slot + n_real))
            slot += ns
            position += n_real
        q = np.asarray(self.question, dtype=np.int64).reshape(-1)
        self.question_span = (slot, slot + q.size)
        if q.size:
            for acc, a in zip(cols, (q, position + np.arange(q.size), np.zeros(q.size, bool), np.ones(q.size, bool),
                                     np.full(q.size, FULL_DEPTH, np.int64))):
                acc.append(a)
        if not cols[0]:
            raise PlanError("request has no tokens")
        self.token_ids, self.positions, self.is_pad, self.recompute_mask, self.recompute_depth = (
            np.concatenate(c) for c in cols)
        self.question = q

    @property
    def n_slots(self) -> int:
        return int(self.token_ids.size)

    @property
    def n_tokens(self) -> int:
        return int(np.count_nonzero(~self.is_pad))


def build_request(segments, question) -> PrefillRequest:
    return PrefillRequest(segments=list(segments), question=np.asarray(question))


def plain_request(*token_groups) -> PrefillRequest:
    """All-fresh request; the last group is the question span (model.py:277-282)."""
    groups = [np.asarray(g) for g in token_groups]
    if not groups:
        raise PlanError("need at least one token group")
    return build_request([Segment(tokens=g) for g in groups[:-1]], groups[-1])


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------


class KVCache:
    """Merged per-layer KV of a processed request, keys position-free
    (model.py:286-316).  Device-backed: ``keys``/``values`` materialise from
    the request's HBM buffers on first access."""

    def __init__(self, keys=None, values=None, positions=None, valid=None, *, _dev=None):
        self._keys = keys
        self._values = values
        self.positions = np.asarray(positions)
        self.valid = np.asarray(valid, dtype=bool)
        self._dev = _dev  # (kv_k, kv_v) torch [L, n, kvw]

    def _host(self, which):
        return _host_layers(self._dev[which])

    @property
    def keys(self) -> list:
        if self._keys is None:
            self._keys = self._host(0)
        return self._keys

    @keys.setter
    def keys(self, v):
        self._keys = v
        self._dev = None if self._values is not None else self._dev

    @property
    def values(self) -> list:
        if self._values is None:
            self._values = self._host(1)
        return self._values

    @values.setter
    def values(self, v):
        self._values = v

    @property
    def n_slots(self) -> int:
        return int(self.positions.size)

    def copy(self) -> "KVCache":
        return KVCache(keys=[k.copy() for k in self.keys], values=[v.copy() for v in self.values],
                       positions=self.positions.copy(), valid=self.valid.copy())

    def append_token(self, per_layer_kv, position: int):
        keys, values = self.keys, self.values
        for l, (k_row, v_row) in enumerate(per_layer_kv):
            keys[l] = np.vstack([keys[l], k_row])
            values[l] = np.vstack([values[l], v_row])
        self._dev = None
        self.positions = np.append(self.positions, position)
        self.valid = np.append(self.valid, True)

    def slice_rows(self, start: int, stop: int):
        return [k[start:stop].copy() for k in self.keys], [v[start:stop].copy() for v in self.values]


class AttentionRecord:
    """Per-layer, per-head softmax weights of the computed rows
    (model.py:320-335).  Engine records keep the device operands and
    materialise ``weights`` with the ``cc_attention_probs`` kernel on access."""

    def __init__(self, weights=None, query_slots=None, *, _lazy=None):
        self._weights = list(weights) if weights is not None else None
        self.query_slots = list(query_slots) if query_slots is not None else []
        self._lazy = _lazy  # engine.LazyAttention

    @property
    def weights(self) -> list:
        if self._weights is None:
            self._weights = self._lazy.materialize_all()
        return self._weights

    @property
    def n_layers(self) -> int:
        return len(self.query_slots)

    def head_mean(self, layer: int) -> np.ndarray:
        return self.weights[layer].mean(axis=0)

    def row_lookup(self, layer: int) -> dict:
        return {int(s): r for r, s in enumerate(self.query_slots[layer])}


class PrefillResult:
    """Output of :func:`prefill` (model.py:338-345) plus the device extras:
    ``first_token`` (greedy argmax of the question's last row, computed on
    the GPU when requested) and the per-chunk creation statistics."""

    def __init__(self, *, kv, attn, question_span, computed, active_per_layer, positions, hidden_fn, extras=None):
        self.kv = kv
        self.attn = attn
        self.question_span = question_span
        self.computed = computed
        self.active_per_layer = active_per_layer
        self.positions = positions
        self._hidden_fn = hidden_fn
        self._hidden = None
        self.extras = extras or {}

    @property
    def hidden(self) -> np.ndarray:
        if self._hidden is None:
            self._hidden = self._hidden_fn()
        return self._hidden

    @hidden.setter
    def hidden(self, v):
        self._hidden = v

    @property
    def first_token(self):
        """Greedy first token; read back from the device on first access (so a
        caller can plan the next request while this one computes)."""
        if "first_token" not in self.extras and "first_token_host" in self.extras:
            host_tok, ev = self.extras["first_token_host"]
            ev.synchronize()
            self.extras["first_token"] = int(host_tok[0])
        elif "first_token" not in self.extras and "first_token_dev" in self.extras:
            self.extras["first_token"] = int(self.extras["first_token_dev"].item())
        return self.extras.get("first_token")


def prefill(model: Model, request: PrefillRequest, record_values: bool = False, **options) -> PrefillResult:
    """Partial prefill with injected position-free chunk caches, on the GPU
    (model.py:348-442).  See ``engine.run_prefill`` for the options
    (``record_attention``, ``stats``, ``first_token``)."""
    from .engine import run_prefill

    return run_prefill(model, request, record_values=record_values, **options)


def decode(model: Model, kv: KVCache, last_hidden, max_steps: int) -> list:
    """Greedy decode extending ``kv`` by one row per layer per step
    (model.py:445-484), each step run by the device engine."""
    from .engine import run_decode

    return run_decode(model, kv, last_hidden, max_steps)


def extract_chunk_cache(result: PrefillResult, start: int, stop: int, source_prefix: tuple = ()) -> ChunkCache:
    """Cut one chunk's rows out of a prefill result into fresh pool blocks
    (model.py:487-492; kernel K10)."""
    from .engine import extract_rows

    return extract_rows(result, start, stop, source_prefix)
