"""SlideNetwork on the B200 (drop-in for reference network.py).

Shape: the reference's generic stack is restricted to what every BASELINE
config uses -- one ReLU hidden layer and the softmax output, LSH on the
output layer only (``widths=[H, N]``, ``lsh_layers`` absent or ``{1: ...}``).
Other shapes raise NotImplementedError instead of silently falling back.

State lives in device memory (torch tensors; every weight row padded to a
multiple of 128 floats, W1 stored transposed so a feature row is contiguous)
and every stage of the step is an sm_100a kernel behind the C ABI
(include/slide_b200.h).  Host views (``layer.w`` etc.) are copies that write
back on item assignment.

Schedules of ``train_batch``:

* ``"sequential"`` -- slot i sees the updates of slots < i; identical to the
  reference's ``train_batch(workers=1)``.  Default for ``workers=1``.
* ``"snapshot"`` -- all slots forward/backward on the pre-step weights, then
  every row applies its slots' Adam updates in slot order: the deterministic
  member of the reference's HOGWILD contract (network.py:9-13).
  Default for ``workers > 1`` and the throughput mode of ``bench.py``.
"""

from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hashing import HashFamilyConfig, SimHashFamily, new_hash_family
from .samplers import STRATEGY_CODE, SamplerConfig
from .sparse import SparseVector
from .tables import LshTables, RebuildSchedule

CHECKPOINT_MAGIC = b"SLDE"
CHECKPOINT_VERSION = 1
_KIND_CODES = {"relu": 0, "softmax": 1}
_KIND_NAMES = {v: k for k, v in _KIND_CODES.items()}


def check_positive_int(value, name: str) -> int:
    if not isinstance(value, (int, np.integer)) or isinstance(value, bool) or value < 1:
        raise ValueError(f"{name} must be a positive integer, got {value!r}")
    return int(value)


@dataclass(frozen=True)
class TrainConfig:
    """Optimizer and schedule hyperparameters (reference network.py:36-56)."""

    batch_size: int = 128
    learning_rate: float = 1e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    n0: int = 50
    decay: float = 0.0
    epochs: int = 1
    seed: int = 0

    def validate(self) -> "TrainConfig":
        check_positive_int(self.batch_size, "batch_size")
        check_positive_int(self.epochs, "epochs")
        check_positive_int(self.n0, "n0")
        if self.learning_rate <= 0:
            raise ValueError(f"learning_rate must be > 0, got {self.learning_rate}")
        return self


@dataclass(frozen=True)
class LshLayerConfig:
    """How one layer hashes and samples its neurons (reference network.py:59-71)."""

    family: str = "simhash"
    k: int = 6
    l: int = 25
    sampler: SamplerConfig = field(default_factory=SamplerConfig)
    capacity: int = 128
    policy: str = "fifo"
    simhash_sparsity: float = 1.0 / 3.0
    wta_bin_size: int = 8
    doph_top_k: int = 32


class _Mirror(np.ndarray):
    """Host copy of device state that writes back on item assignment."""

    def __new__(cls, arr, flush):
        obj = np.asarray(arr).view(cls)
        obj._flush = flush
        return obj

    def __array_finalize__(self, obj):
        self._flush = None  # slices / derived views do not write back

    def _push(self):
        if self._flush is not None:
            self._flush(np.asarray(self))

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._push()

    def __iadd__(self, o):
        np.ndarray.__iadd__(self, o)
        self._push()
        return self

    def __isub__(self, o):
        np.ndarray.__isub__(self, o)
        self._push()
        return self

    def __imul__(self, o):
        np.ndarray.__imul__(self, o)
        self._push()
        return self

    def __itruediv__(self, o):
        np.ndarray.__itruediv__(self, o)
        self._push()
        return self


class Layer:
    """View of one layer's device state (reference network.py:74-98)."""

    def __init__(self, net: "SlideNetwork", index: int, width: int, fan_in: int, kind: str):
        self._net = net
        self._i = index
        self.width = width
        self.fan_in = fan_in
        self.kind = kind
        self.lsh: LshTables | None = None
        self.sampler_cfg: SamplerConfig | None = None
        self.static_sample = None
        slots = net.cfg.batch_size
        small = width * slots <= 4_000_000
        # per-slot neuron arrays, maintained by the single-sample forward API
        self.active_flags = np.zeros((width, slots), dtype=bool) if small else None
        self.activations = np.zeros((width, slots)) if small else None
        self.gradients = np.zeros((width, slots)) if small else None

    # The device keeps the hidden units in a physical order of its own (the
    # live units adjacent, SlideNetwork._maybe_relabel); the views below are in
    # the caller's unit order: unit u sits at physical column unit_cols()[u].
    def _mat(self, name):
        t = getattr(self._net, name + ("1t" if self._i == 0 else "2"))
        H = self._net.hidden
        cols = self._net._unit_cols_dev()
        if cols is not None:
            t = t[:, cols]  # (a gathered copy; writes go through _mirror_mat's flush)
            return t.T if self._i == 0 else t
        return t[:, :H].T if self._i == 0 else t[:, :H]

    def _vec(self, name):
        t = getattr(self._net, name + ("1" if self._i == 0 else "2"))
        cols = self._net._unit_cols_dev() if self._i == 0 else None
        return t[cols] if cols is not None else t[: self.width]

    def _mirror_mat(self, name):
        dev = self._mat(name)
        net = self._net
        raw = getattr(net, name + ("1t" if self._i == 0 else "2"))
        first = self._i == 0
        H = net.hidden

        def flush(a):
            import torch

            # the unit order of the moment of the write (a mirror may outlive a renumbering)
            cols = net._unit_cols_dev()
            src = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(raw.device)
            if first:
                src = src.T
            if cols is None:
                raw[:, :H] = src
            else:
                raw[:, cols] = src

        return _Mirror(dev.double().cpu().numpy(), flush)

    def _mirror_vec(self, name, dtype=np.float64):
        dev = self._vec(name)
        net = self._net
        raw = getattr(net, name + ("1" if self._i == 0 else "2"))
        first = self._i == 0
        width = self.width
        np_dtype = dev.cpu().numpy().dtype

        def flush(a):
            import torch

            cols = net._unit_cols_dev() if first else None
            src = torch.from_numpy(np.ascontiguousarray(a).astype(np_dtype)).to(raw.device)
            if cols is None:
                raw[:width] = src
            else:
                raw[cols] = src

        return _Mirror(dev.cpu().numpy().astype(dtype), flush)

    w = property(lambda self: self._mirror_mat("w"), lambda self, a: self._mirror_mat("w").__setitem__(slice(None), a))
    adam_m = property(lambda self: self._mirror_mat("m"), lambda self, a: self._mirror_mat("m").__setitem__(slice(None), a))
    adam_v = property(lambda self: self._mirror_mat("v"), lambda self, a: self._mirror_mat("v").__setitem__(slice(None), a))
    b = property(lambda self: self._mirror_vec("b"), lambda self, a: self._mirror_vec("b").__setitem__(slice(None), a))
    adam_mb = property(lambda self: self._mirror_vec("mb"), lambda self, a: self._mirror_vec("mb").__setitem__(slice(None), a))
    adam_vb = property(lambda self: self._mirror_vec("vb"), lambda self, a: self._mirror_vec("vb").__setitem__(slice(None), a))
    steps = property(lambda self: self._mirror_vec("steps", np.int64),
                     lambda self, a: self._mirror_vec("steps", np.int64).__setitem__(slice(None), a))

    def neuron(self, idx: int) -> "Neuron":
        return Neuron(self, idx)


class Neuron:
    """View of one neuron (reference network.py:101-142)."""

    __slots__ = ("layer", "idx")

    def __init__(self, layer: Layer, idx: int):
        if not 0 <= idx < layer.width:
            raise IndexError(f"neuron {idx} out of range for width {layer.width}")
        self.layer = layer
        self.idx = idx

    weights = property(lambda s: s.layer.w[s.idx])
    bias = property(lambda s: float(s.layer.b[s.idx]))
    adam_m = property(lambda s: s.layer.adam_m[s.idx])
    adam_v = property(lambda s: s.layer.adam_v[s.idx])
    step_count = property(lambda s: int(s.layer.steps[s.idx]))
    active_flags = property(lambda s: s.layer.active_flags[s.idx])
    activations = property(lambda s: s.layer.activations[s.idx])
    gradients = property(lambda s: s.layer.gradients[s.idx])


@dataclass
class ForwardTrace:
    """Per-layer active ids and inputs for one slot plus the output softmax."""

    slot: int
    active: list
    inputs: list
    probs: np.ndarray

    def loss(self, labels) -> float:
        """Cross entropy against the uniform label distribution (network.py:154-158)."""
        ids = self.active[-1]
        pos = np.searchsorted(ids, np.fromiter(labels, dtype=np.int64))
        return float(-np.log(np.maximum(self.probs[pos], 1e-300)).mean())


@dataclass
class BatchStats:
    loss: float
    active_fraction: dict
    rebuilt: list


class TrainingDivergedError(RuntimeError):
    """Loss became non-finite; training state is unusable."""


_FAMILY_CODE = {"simhash": 1, "dwta": 2, "wta": 3}


def _family_desc(desc, family, capacity, policy, sampler=None):
    """Fill the family / table fields of a NetDesc; returns host arrays to keep alive."""
    keep = []
    name = type(family).__name__
    code = {"SimHashFamily": 1, "DwtaFamily": 2, "WtaFamily": 3}[name]
    desc.family = code
    desc.k = family.k
    desc.l = family.l
    desc.key_bits = family.key_bits
    desc.capacity = capacity
    desc.policy = 0 if policy == "fifo" else 1
    if sampler is not None:
        desc.strategy = STRATEGY_CODE[sampler.strategy]
        desc.beta = sampler.beta
        desc.min_freq = sampler.min_freq
    family._check_device_width()
    if code == 1:
        packed = np.ascontiguousarray(family.packed())
        desc.sh_c = family.entries_per_proj
        desc.sh_packed_host = packed.ctypes.data
        keep.append(packed)
    else:
        perms = np.ascontiguousarray(family.perms.astype(np.int16))
        donors = np.ascontiguousarray(family.donors())
        desc.bin_size = family.bin_size
        desc.bins_per_perm = family.bins_per_perm
        desc.n_perms = family.n_perms
        desc.bits = family.bits_per_code
        desc.dw_perms_host = perms.ctypes.data
        desc.dw_donors_host = donors.ctypes.data
        keep += [perms, donors]
    return keep


@dataclass
class HostCsr:
    """One batch as host CSR (int32 offsets/ids, float32 values)."""

    x_ptr: np.ndarray
    x_idx: np.ndarray
    x_val: np.ndarray
    y_ptr: np.ndarray
    y_idx: np.ndarray

    @property
    def batch(self) -> int:
        return len(self.x_ptr) - 1

    @staticmethod
    def from_corpus(corpus) -> "HostCsr":
        """A ``data.Corpus`` (int64 offsets) as one batch."""
        return HostCsr(corpus.x_ptr.astype(np.int32), corpus.x_idx, corpus.x_val, corpus.y_ptr.astype(np.int32),
                       corpus.y_idx)


def csr_from_batch(batch, input_dim: int, n_out: int) -> HostCsr:
    xp, yp = [0], [0]
    xi, xv, yi = [], [], []
    for x, labels in batch:
        if x.dim != input_dim:
            raise ValueError(f"input dim {x.dim} != network input dim {input_dim}")
        lab = np.unique(np.fromiter(labels, dtype=np.int64)) if len(labels) else np.empty(0, np.int64)
        if lab.size and (lab[0] < 0 or lab[-1] >= n_out):
            raise IndexError(f"label outside [0, {n_out})")
        xi.append(x.indices.astype(np.int32))
        xv.append(x.values.astype(np.float32))
        yi.append(lab.astype(np.int32))
        xp.append(xp[-1] + x.nnz)
        yp.append(yp[-1] + lab.size)
    cat = lambda p, dt: np.concatenate(p).astype(dt) if p else np.empty(0, dt)
    return HostCsr(np.asarray(xp, np.int32), cat(xi, np.int32), cat(xv, np.float32), np.asarray(yp, np.int32),
                   cat(yi, np.int32))


class SlideNetwork:
    """Input -> ReLU hidden (dense) -> LSH-sampled softmax output, on the device."""

    def __init__(self, input_dim: int, widths, cfg: TrainConfig, lsh_layers: dict | None = None,
                 static_layers: dict | None = None, *, shard: tuple | None = None, group=None):
        import torch

        from . import _device

        check_positive_int(input_dim, "input_dim")
        if not widths:
            raise ValueError("need at least one layer")
        cfg.validate()
        widths = [check_positive_int(w, "width") for w in widths]
        if len(widths) != 2:
            raise NotImplementedError("the B200 step supports exactly one hidden ReLU layer + softmax (widths=[H, N])")
        lsh_layers = dict(lsh_layers or {})
        if set(lsh_layers) - {1}:
            raise NotImplementedError("LSH sampling is supported on the output layer (index 1) only")
        if static_layers:
            raise NotImplementedError("static uniform sampling is outside the B200 hot path")
        self.cfg = cfg
        self.input_dim = input_dim
        self.hidden, self.n_out = widths
        self.access_log = None
        # output-layer column shard: rank g of G owns ids % G == g
        self.shard_rank, self.shard_count = shard if shard is not None else (0, 1)
        self.group = group
        dev = _device.device()
        H, N, D = self.hidden, self.n_out, input_dim
        g, G = self.shard_rank, self.shard_count
        n_local = (N - g + G - 1) // G
        self.n_local = n_local
        hp = _device.round_up(H, 128)
        self.hidden_pad = hp
        f32 = dict(dtype=torch.float32, device=dev)
        # -- parameters: the reference's draw order (network.py:79-89, 187-193)
        rng = np.random.default_rng(cfg.seed)
        # sharded: W1^T holds this rank's hidden units [u0, u0 + hg)
        if G > 1 and (H % G or (H // G) % 4 or H // G > 128):
            raise NotImplementedError("sharded hidden layer: hidden / shard_count must be a multiple of 4, <= 128")
        hg = H // G if G > 1 else hp
        u0 = g * hg if G > 1 else 0
        self.w1t = torch.zeros((D, hg), **f32)
        bound = 1.0 / np.sqrt(D)
        rows = max(1, (1 << 22) // D)
        for r0 in range(0, H, rows):
            r1 = min(H, r0 + rows)
            chunk = rng.uniform(-bound, bound, size=(r1 - r0, D)).astype(np.float32)
            a, b = max(r0, u0), min(r1, u0 + (H if G == 1 else hg))
            if a < b:
                self.w1t[:, a - u0 : b - u0] = torch.from_numpy(chunk[a - r0 : b - r0]).to(dev).T
        self.m1t = torch.zeros((D, hg), **f32)
        self.v1t = torch.zeros((D, hg), **f32)
        self.b1 = torch.zeros(hp, **f32)
        self.mb1 = torch.zeros(hp, **f32)
        self.vb1 = torch.zeros(hp, **f32)
        self.steps1 = torch.zeros(hp, dtype=torch.int64, device=dev)
        self.w2 = torch.zeros((n_local, hp), **f32)
        bound = 1.0 / np.sqrt(H)
        rows = max(G, ((1 << 22) // H) // G * G)
        for r0 in range(0, N, rows):  # the whole stream is drawn; a shard keeps its rows
            r1 = min(N, r0 + rows)
            chunk = rng.uniform(-bound, bound, size=(r1 - r0, H)).astype(np.float32)
            if G > 1:
                chunk = chunk[(g - r0) % G :: G]
            l0 = (r0 + G - 1 - g) // G if r0 > g else 0
            self.w2[l0 : l0 + chunk.shape[0], :H] = torch.from_numpy(np.ascontiguousarray(chunk)).to(dev)
        self.m2 = torch.zeros((n_local, hp), **f32)
        self.v2 = torch.zeros((n_local, hp), **f32)
        self.b2 = torch.zeros(n_local, **f32)
        self.mb2 = torch.zeros(n_local, **f32)
        self.vb2 = torch.zeros(n_local, **f32)
        self.steps2 = torch.zeros(n_local, dtype=torch.int64, device=dev)
        self.layers = [Layer(self, 0, H, D, "relu"), Layer(self, 1, N, H, "softmax")]
        # -- device context
        desc = _lib.NetDesc()
        desc.input_dim, desc.hidden, desc.hidden_pad, desc.n_out = D, H, hp, N
        desc.max_batch = cfg.batch_size
        desc.lr, desc.beta1, desc.beta2, desc.eps = cfg.learning_rate, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
        desc.seed = cfg.seed
        for name in ("w1t", "m1t", "v1t", "b1", "mb1", "vb1", "steps1", "w2", "m2", "v2", "b2", "mb2", "vb2",
                     "steps2"):
            setattr(desc, name, getattr(self, name).data_ptr())
        desc.shard_rank, desc.shard_count = g, G
        self._keep = []
        spec = lsh_layers.get(1)
        family = None
        if spec is not None:
            family = new_hash_family(HashFamilyConfig(
                family=spec.family, k_per_table=spec.k, num_tables=spec.l, dim=H,
                simhash_sparsity=spec.simhash_sparsity, wta_bin_size=spec.wta_bin_size,
                doph_top_k=spec.doph_top_k, seed=cfg.seed + 7919 * 2))
            sampler = spec.sampler.validate(spec.l)
            self._keep = _family_desc(desc, family, spec.capacity, spec.policy, sampler)
        self._desc = desc
        h = _lib.vp()
        _lib.call("slide_create", desc, _lib.vp(_device.stream_handle()), _lib.C.byref(h))
        self._ctx = h
        if spec is not None:
            layer = self.layers[1]
            layer.lsh = LshTables(family, policy=spec.policy, capacity=spec.capacity,
                                  schedule=RebuildSchedule(cfg.n0, cfg.decay), seed=cfg.seed + 104729 * 2,
                                  _ctx=self._ctx)
            layer.lsh._owner_rebuild = self._rebuild_tables
            layer.sampler_cfg = sampler
            self._rebuild_tables()  # network.py:221
        self._pinned = {}
        self._live = None
        # physical column of every hidden unit (identity until a relabel)
        self._pos = np.arange(hp, dtype=np.int64)
        self._pos_dev = None
        self.relabels = 0
        if spec is not None:
            self.layers[1].lsh._unit_cols = self.unit_cols
        if self.relabel_units and G == 1 and spec is not None:
            # an identity renumbering now: the first call's one-time costs (its
            # buffer, the kernels' first launch) stay out of the training steps
            ident = np.arange(H, dtype=np.int32)
            _lib.call("slide_relabel_units", self._ctx, ident.ctypes.data)

    #: keep the live hidden units physically adjacent (checked at every table rebuild)
    relabel_units = os.environ.get("SLIDE_NO_RELABEL") is None

    def unit_cols(self) -> np.ndarray:
        """Physical column (in w1t / w2 / h and their companions) of hidden
        unit u, for u in [0, hidden)."""
        return self._pos[: self.hidden]

    def _unit_cols_dev(self):
        """The same as a device index tensor; None while it is the identity."""
        if self.relabels == 0:
            return None
        if self._pos_dev is None:
            import torch

            self._pos_dev = torch.from_numpy(self._pos[: self.hidden].copy()).to(self.w2.device)
        return self._pos_dev

    def _maybe_relabel(self) -> bool:
        """Renumber the hidden units on the device so that the ones live in
        the last batch are adjacent (``slide_relabel_units``), when they are
        scattered over noticeably more 32-byte sectors than they need.  Called
        at the rebuild barrier, between steps."""
        if not self.relabel_units or self.shard_count > 1:
            return False
        H = self.hidden
        try:
            live = self._read_raw(13, 1 + self.hidden_pad, np.int32)
        except ValueError:
            return False  # no forward yet
        n = int(live[0])
        if n <= 0 or n >= H:
            return False
        units = live[1 : 1 + n].astype(np.int64)
        units = units[units < H]
        need = -(-units.size // 8)
        have = int(np.count_nonzero(np.bincount(units // 8)))  # (np.unique's first call costs ~50 ms of lazy imports)
        if have <= need + max(2, need // 2):
            return False
        is_live = np.zeros(H, dtype=bool)
        is_live[units] = True
        dead = np.flatnonzero(~is_live)
        self._relabel(np.concatenate([units, dead]))
        return True

    def _relabel(self, src):
        """New physical unit p takes the state of old physical unit src[p]."""
        H = self.hidden
        src = np.ascontiguousarray(np.asarray(src).astype(np.int32))
        if src.shape != (H,):
            raise ValueError(f"src must hold {H} units")
        _lib.call("slide_relabel_units", self._ctx, src.ctypes.data)
        inv = np.empty(H, dtype=np.int64)
        inv[src] = np.arange(H)
        self._pos[:H] = inv[self._pos[:H]]
        self._pos_dev = None
        self.relabels += 1

    def __del__(self):
        try:
            if getattr(self, "_ctx", None) is not None:
                _lib.lib().slide_destroy(self._ctx)
                self._ctx = None
        except Exception:
            pass

    # -- tables ---------------------------------------------------------------
    def _rebuild_tables(self):
        lsh = self.layers[1].lsh
        st = _lib.mt_state_from_random(lsh._rng)
        if self.shard_count > 1:
            from .sharded import GpuShardBackend, rebuild_sharded

            rebuild_sharded(GpuShardBackend(self), self.group)
        else:
            _lib.call("slide_rebuild_tables", self._ctx, st.ctypes.data)
        _lib.mt_state_to_random(st, lsh._rng)
        lsh.n_items = self.n_out
        lsh._views = None
        lsh._dirty = False
        lsh._last_keys = None
        lsh.cache_valid = isinstance(lsh.family, SimHashFamily)

    # -- batch upload ---------------------------------------------------------
    def _upload(self, csr: HostCsr, rng_states=None, forced=None):
        """Host CSR -> device tensors (+ the C Batch struct)."""
        import torch

        from . import _device

        dev = _device.device()
        self.h2d_bytes = 0
        # the pinned staging buffers are reused: the previous upload's
        # asynchronous copies must have read them before they are rewritten
        ev = getattr(self, "_pin_ev", None)
        if ev is not None:
            ev.synchronize()

        def up(a, dt):
            # stage through a pinned host buffer so the copy is a true async DMA
            a = np.ascontiguousarray(a, dtype=dt).reshape(-1)
            key = (len(self._pinned), a.dtype.str)
            key = next((k for k in self._pinned if k[1] == a.dtype.str and k not in used), key)
            buf = self._pinned.get(key)
            if buf is None or buf.numel() < a.size:
                buf = torch.empty(max(a.size, 1) * 2, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
                self._pinned[key] = buf
            used.add(key)
            view = buf[: a.size]
            view.numpy()[...] = a
            self.h2d_bytes += a.nbytes
            return view.to(dev, non_blocking=True)

        used = set()

        t = {
            "x_ptr": up(csr.x_ptr, np.int32), "x_idx": up(csr.x_idx if csr.x_idx.size else np.zeros(1), np.int32),
            "x_val": up(csr.x_val if csr.x_val.size else np.zeros(1), np.float32),
            "y_ptr": up(csr.y_ptr, np.int32), "y_idx": up(csr.y_idx if csr.y_idx.size else np.zeros(1), np.int32),
        }
        hx = np.ascontiguousarray(csr.x_ptr, dtype=np.int32)
        hy = np.ascontiguousarray(csr.y_ptr, dtype=np.int32)
        if rng_states is None and forced is None:
            self._pin_ev = torch.cuda.Event()
            self._pin_ev.record()
        bt = _lib.Batch()
        bt.batch = csr.batch
        bt.x_ptr, bt.x_idx, bt.x_val = t["x_ptr"].data_ptr(), t["x_idx"].data_ptr(), t["x_val"].data_ptr()
        bt.y_ptr, bt.y_idx = t["y_ptr"].data_ptr(), t["y_idx"].data_ptr()
        bt.x_ptr_host, bt.y_ptr_host = hx.ctypes.data, hy.ctypes.data
        keep = [t, hx, hy]
        if rng_states is not None:
            rs = up(rng_states.view(np.int64), np.int64)
            bt.rng_states = rs.data_ptr()
            t["rng"] = rs
        if forced is not None:
            fp, fi = forced
            hf = np.ascontiguousarray(fp, dtype=np.int32)
            t["fptr"] = up(hf, np.int32)
            t["fidx"] = up(fi if len(fi) else np.zeros(1), np.int32)
            bt.forced_ptr, bt.forced_idx, bt.forced_ptr_host = t["fptr"].data_ptr(), t["fidx"].data_ptr(), hf.ctypes.data
            keep.append(hf)
        if rng_states is not None or forced is not None:
            self._pin_ev = torch.cuda.Event()
            self._pin_ev.record()
        return bt, keep

    def _read_raw(self, what, n, dtype):
        out = np.empty(n, dtype=dtype)
        got = _lib.i64()
        _lib.call("slide_read", self._ctx, what, out.ctypes.data, out.nbytes, _lib.C.byref(got))
        return out[: got.value // out.itemsize]

    def _read(self, what, n, dtype):
        """A stage readout in the caller's unit order: hidden activations (0),
        hidden errors (8) and the live-unit list (13) are stored in the
        device's physical order."""
        out = self._read_raw(what, n, dtype)
        if self.relabels == 0 or what not in (0, 8, 13):
            return out
        hp, H = self.hidden_pad, self.hidden
        if what == 13:
            unit_of = np.arange(hp, dtype=np.int64)
            unit_of[self._pos[:H]] = np.arange(H)
            nl = int(out[0])
            res = out.copy()
            res[1 : 1 + hp] = unit_of[out[1 : 1 + hp]]
            res[1 : 1 + nl] = np.sort(res[1 : 1 + nl])
            return res
        rows = out[: out.size // hp * hp].reshape(-1, hp)
        return np.ascontiguousarray(rows[:, self._pos]).reshape(-1)

    # -- training -----------------------------------------------------------
    def train_batch(self, batch, iteration: int, workers: int = 1, executor=None, schedule: str | None = None) -> BatchStats:
        """Forward+backward every slot, then the rebuild barrier (network.py:340-379)."""
        if not batch:
            raise ValueError("batch is empty")
        if len(batch) > self.cfg.batch_size:
            raise ValueError(f"batch of {len(batch)} exceeds configured size {self.cfg.batch_size}")
        for _, labels in batch:
            if not len(labels):
                raise ValueError("backward needs at least one true label")
        csr = csr_from_batch(batch, self.input_dim, self.n_out)
        if schedule is None:
            schedule = "sequential" if workers <= 1 else "snapshot"
        return self.train_batch_csr(csr, iteration, schedule=schedule)

    def train_batch_csr(self, csr: HostCsr, iteration: int, schedule: str = "snapshot") -> BatchStats:
        """Batch given as host CSR (the e2e path: one upload, one step, the
        per-slot losses back)."""
        if schedule not in ("sequential", "snapshot"):
            raise ValueError(f"unknown schedule {schedule!r}")
        B = csr.batch
        if B < 1 or B > self.cfg.batch_size:
            raise ValueError(f"batch of {B} outside 1..{self.cfg.batch_size}")
        if self.shard_count > 1:
            if schedule != "snapshot":
                raise NotImplementedError("the sharded output layer runs the snapshot schedule")
            from .sharded import GpuShardBackend, sharded_step

            loss, active = sharded_step(GpuShardBackend(self), csr, iteration, self.group).host()
        else:
            loss, active = self._step(csr, iteration, 1 if schedule == "sequential" else B)
        return self._barrier(iteration, loss, active)

    def train_batches_csr(self, batches, first_iteration: int = 1, schedule: str = "snapshot") -> list:
        """``train_batch_csr`` over consecutive batches (iterations
        first_iteration, first_iteration + 1, ...), pipelined: step k+1 (its
        H2D copies, the graph, the D2H of its losses) is queued on the device
        behind step k before the host waits for step k's losses, and the
        host stages batch k+2 meanwhile.  The rebuild barrier that follows
        step k is enqueued on the context stream between the two (the
        schedule depends only on the iteration), so the results equal
        train_batch_csr per batch; only the losses arrive one step late (no
        divergence check between the two steps)."""
        batches = list(batches)
        if (schedule != "snapshot" or not self.use_graphs or self.shard_count > 1
                or any(c.batch != self.cfg.batch_size for c in batches)):
            return [self.train_batch_csr(c, first_iteration + k, schedule) for k, c in enumerate(batches)]
        out = []
        if not batches:
            return out
        B = self.cfg.batch_size
        loss = np.empty(B, dtype=np.float64)
        active = np.empty(B, dtype=np.int64)
        lsh = self.layers[1].lsh
        keeps = {}

        def launch(k):
            # pinned set k % 2 was step k-2's, whose results were taken
            bt, keep = self._pinned_batch(batches[k], k % 2)
            keeps[k % 2] = keep
            if lsh is not None:
                lsh.sync_to_device()
            _lib.call("slide_graph_step_async", self._ctx, _lib.C.byref(bt), first_iteration + k)
            return self.h2d_bytes

        h2d = launch(0)
        for k in range(len(batches)):
            it = first_iteration + k
            rebuilt = self._rebuild_after(it)  # stream-ordered after step k, before step k+1
            h2d_next = launch(k + 1) if k + 1 < len(batches) else 0
            _lib.call("slide_graph_step_wait", self._ctx, loss.ctypes.data, active.ctypes.data)
            out.append(self._stats(loss, active, rebuilt))
            self.h2d_bytes = h2d
            h2d = h2d_next
        self._live = keeps
        return out

    #: snapshot steps replay one captured CUDA graph per batch shape
    use_graphs = True

    def _pinned_batch(self, csr: HostCsr, buf_set: int = 0):
        """Batch struct over pinned host copies of the CSR (graph steps copy
        them into the context's own device buffers).  The pinned buffers and
        their numpy views are cached; each call is five plain copies."""
        import torch

        self.h2d_bytes = 0
        keep = []
        ptrs = []
        for name, a, dt in (("xp", csr.x_ptr, np.int32), ("xi", csr.x_idx, np.int32), ("xv", csr.x_val, np.float32),
                            ("yp", csr.y_ptr, np.int32), ("yi", csr.y_idx, np.int32)):
            n = len(a)
            ent = self._pinned.get(("g", name, buf_set))
            if ent is None or ent[1].size < max(n, 1):
                buf = torch.empty(max(n, 1) * 2, dtype=torch.from_numpy(np.empty(0, dt)).dtype, pin_memory=True)
                ent = (buf, buf.numpy(), buf.data_ptr())
                self._pinned[("g", name, buf_set)] = ent
            np.copyto(ent[1][:n], a, casting="unsafe")
            self.h2d_bytes += n * 4
            keep.append(ent[0])
            ptrs.append(ent[2])
        bt = _lib.Batch()
        bt.batch = csr.batch
        bt.x_ptr_host = bt.x_ptr = ptrs[0]
        bt.x_idx = ptrs[1]
        bt.x_val = ptrs[2]
        bt.y_ptr_host = bt.y_ptr = ptrs[3]
        bt.y_idx = ptrs[4]
        return bt, keep

    def _step(self, csr: HostCsr, iteration: int, sub_batch: int):
        if self.layers[1].lsh is not None:
            self.layers[1].lsh.sync_to_device()
        B = csr.batch
        loss = np.empty(B, dtype=np.float64)
        active = np.empty(B, dtype=np.int64)
        if sub_batch == B and self.use_graphs:
            bt, keep = self._pinned_batch(csr)
            _lib.call("slide_graph_step", self._ctx, _lib.C.byref(bt), iteration, loss.ctypes.data,
                      active.ctypes.data)
        else:
            bt, keep = self._upload(csr)
            _lib.call("slide_train_batch", self._ctx, _lib.C.byref(bt), iteration, sub_batch, loss.ctypes.data,
                      active.ctypes.data)
        del keep
        return loss, active

    def _barrier(self, iteration, loss, active) -> BatchStats:
        return self._stats(loss, active, self._rebuild_after(iteration))

    def _rebuild_after(self, iteration) -> list:
        """The rebuild barrier after a batch (network.py:368-373): the layers
        rebuilt (enqueued on the context stream)."""
        lsh = self.layers[1].lsh
        if lsh is None:
            return []
        lsh.mark_weights_changed()
        rebuilt = lsh.maybe_rebuild(iteration)
        # the live hidden units settle within the first few steps: look at
        # them after steps 4, 8, 16, ... and at every rebuild (one small
        # device read; the renumbering itself only runs when they are scattered)
        if rebuilt or (iteration >= 4 and iteration & (iteration - 1) == 0):
            self._maybe_relabel()
        return [1] if rebuilt else []

    def _stats(self, loss, active, rebuilt) -> BatchStats:
        fractions = {}
        if self.layers[1].lsh is not None:
            fractions[1] = float(np.mean(active / self.n_out))
        return BatchStats(float(np.mean(loss)), fractions, rebuilt)

    # -- single-sample API ---------------------------------------------------
    def forward(self, x: SparseVector, slot: int, labels=None, rng=None, forced_active=None) -> ForwardTrace:
        """One input through the net on the device (network.py:241-286)."""
        if x.dim != self.input_dim:
            raise ValueError(f"input dim {x.dim} != network input dim {self.input_dim}")
        if not 0 <= slot < self.cfg.batch_size:
            raise ValueError(f"slot {slot} out of range for batch size {self.cfg.batch_size}")
        if rng is None:
            rng = np.random.default_rng(0)
        forced = None
        if forced_active is not None:
            if forced_active[0] is not None and not np.array_equal(np.sort(np.asarray(forced_active[0])),
                                                                   np.arange(self.hidden)):
                raise NotImplementedError("the hidden layer is dense on the device path; forced hidden sets unsupported")
            if forced_active[-1] is not None:
                ids = np.unique(np.asarray(forced_active[-1], dtype=np.int64))
                forced = (np.array([0, ids.size]), ids.astype(np.int32))
        lab = list(labels) if labels is not None else []
        csr = csr_from_batch([(x, lab)], self.input_dim, self.n_out)
        lsh = self.layers[1].lsh
        use_rng = lsh is not None and forced is None
        if use_rng:
            lsh.sync_to_device()
        states = _lib.pcg64_state_from_generator(rng)[None, :].copy() if use_rng else None
        bt, keep = self._upload(csr, states, forced)
        n_pairs = _lib.i64()
        _lib.call("slide_forward", self._ctx, _lib.C.byref(bt), 0, slot, _lib.C.byref(n_pairs))
        P = n_pairs.value
        hp = self.hidden_pad
        h = self._read(0, hp, np.float32)[: self.hidden].astype(np.float64)
        ids = self._read(3, P, np.int32).astype(np.int64)
        probs = self._read(5, P, np.float32).astype(np.float64)
        if use_rng:
            _lib.pcg64_state_to_generator(self._read(10, 6, np.uint64), rng)
        self._live = keep
        nz = np.flatnonzero(h > 0)
        trace = ForwardTrace(slot, [np.arange(self.hidden, dtype=np.int64), ids],
                             [x, SparseVector(nz, h[nz], self.hidden)], probs)
        l0, l1 = self.layers
        if l0.activations is not None:
            l0.active_flags[:, slot] = True
            l0.activations[:, slot] = h
            l0.gradients[:, slot] = 0.0
        if l1.activations is not None:
            l1.active_flags[:, slot] = False
            l1.active_flags[ids, slot] = True
            l1.gradients[ids, slot] = 0.0
            l1.activations[ids, slot] = probs
        if self.access_log is not None:
            self.access_log.append((0, trace.active[0], x.indices))
            if nz.size:
                self.access_log.append((1, ids, nz))
        return trace

    def backward(self, trace: ForwardTrace, labels, slot: int, update: bool = True, capture=None):
        """Errors over the active subnetwork, then Adam (network.py:290-336).

        The device replays the trace (its active set, hidden activations and
        output probabilities) and runs the backward kernels on it."""
        if slot != trace.slot:
            raise ValueError(f"trace belongs to slot {trace.slot}, not {slot}")
        if not len(labels):
            raise ValueError("backward needs at least one true label")
        rows = trace.active[-1]
        label_arr = np.fromiter(labels, dtype=np.int64)
        pos = np.searchsorted(rows, label_arr)
        if np.any(pos >= rows.size) or np.any(rows[np.minimum(pos, rows.size - 1)] != label_arr):
            raise ValueError("a true label is missing from the output active set")
        x, hs = trace.inputs[0], trace.inputs[1]
        delta = trace.probs.copy()
        delta[pos] -= 1.0 / label_arr.size
        csr = csr_from_batch([(x, np.unique(label_arr))], self.input_dim, self.n_out)
        forced = (np.array([0, rows.size]), rows.astype(np.int32))
        bt, keep = self._upload(csr, None, forced)
        n_pairs = _lib.i64()
        _lib.call("slide_forward", self._ctx, _lib.C.byref(bt), 0, slot, _lib.C.byref(n_pairs))
        hdense = np.zeros(self.hidden_pad, dtype=np.float32)
        hdense[self._pos[hs.indices]] = hs.values
        _lib.call("slide_write", self._ctx, 0, hdense.ctypes.data, hdense.nbytes)
        d32 = delta.astype(np.float32)
        _lib.call("slide_write", self._ctx, 6, d32.ctypes.data, d32.nbytes)
        _lib.call("slide_backward", self._ctx, 1 if update else 0)
        dh_full = self._read(8, self.hidden_pad, np.float32).astype(np.float64)
        l0, l1 = self.layers
        if l1.gradients is not None:
            l1.gradients[rows, slot] = delta
        nz = hs.indices
        if self.access_log is not None:
            self.access_log.append((1, rows, nz))
            if nz.size:
                self.access_log.append((0, nz, x.indices))
        if capture is not None:
            if nz.size == 0:
                capture.append((1, rows, None, None, delta.copy()))
            else:
                capture.append((1, rows, nz, np.outer(delta, hs.values), delta.copy()))
                dh = dh_full[nz]
                if x.nnz == 0:
                    capture.append((0, nz, None, None, dh.copy()))
                else:
                    capture.append((0, nz, x.indices, np.outer(dh, x.values), dh.copy()))
        if l0.gradients is not None and nz.size:
            l0.gradients[nz, slot] = dh_full[nz]
        del keep

    def predict(self, x: SparseVector, rng=None, sampled: bool = True) -> np.ndarray:
        """Ranked label ids, best first (network.py:383-391)."""
        forced = [None, np.arange(self.n_out)] if not sampled else None
        trace = self.forward(x, 0, labels=None, rng=rng, forced_active=forced)
        order = np.argsort(-trace.probs, kind="stable")
        return trace.active[-1][order]

    def predict_batch(self, xs, topn: int = 5, rng=None, sampled: bool = True, fresh_seed=None) -> list:
        """Ranked label ids (best first, at most ``topn``) for many inputs,
        equal to ``[self.predict(x, rng=rng)[:topn] for x in xs]`` with one
        generator shared across the queries in order -- the evaluator's
        semantics (reference estimator.py:203-207) -- but ``batch_size``
        queries per device pass.

        The generator's draws depend on the data only through whether a
        query's sampled set is empty (then ``choice(N, beta)`` follows its
        probe ``permutation(L)``), and emptiness does not depend on the probe
        order.  So each chunk runs twice: a first pass yields the empty
        flags, the host advances the caller's generator through exactly the
        reference's draws recording each query's starting state, and the
        second pass replays every slot from its own state; the device then
        ranks each slot (``slide_topk``).

        ``fresh_seed``: every query starts from its own ``default_rng(fresh_seed)``
        instead -- the CLI evaluator's per-call generator (reference
        cli.py:167-178 calling estimator.py:203-207 once per example)."""
        check_positive_int(topn, "topn")
        xs = list(xs)
        for x in xs:
            if x.dim != self.input_dim:
                raise ValueError(f"input dim {x.dim} != network input dim {self.input_dim}")
        if rng is None:
            rng = np.random.default_rng(0)
        lsh = self.layers[1].lsh
        cfg = self.layers[1].sampler_cfg
        out = []
        B = self.cfg.batch_size
        for lo in range(0, len(xs), B):
            chunk = xs[lo : lo + B]
            nb = len(chunk)
            csr = csr_from_batch([(x, []) for x in chunk], self.input_dim, self.n_out)
            forced = None
            states = None
            if not sampled or lsh is None:
                forced = (np.arange(nb + 1, dtype=np.int64) * self.n_out,
                          np.tile(np.arange(self.n_out, dtype=np.int32), nb))
            else:
                lsh.sync_to_device()
                # any valid generator state will do for the emptiness pass (an
                # all-zero PCG64 state would never leave numpy's rejection loops)
                probe = np.tile(_lib.pcg64_state_from_generator(np.random.default_rng(0)), (nb, 1))
                bt, keep = self._upload(csr, probe, None)
                _lib.call("slide_forward", self._ctx, _lib.C.byref(bt), 0, 0, None)
                empty = self._read(9, nb, np.int32)
                states = np.empty((nb, 6), np.uint64)
                L = lsh.family.l
                if fresh_seed is not None:
                    states[:] = _lib.pcg64_state_from_generator(np.random.default_rng(fresh_seed))
                for i in range(nb if fresh_seed is None else 0):
                    states[i] = _lib.pcg64_state_from_generator(rng)
                    if cfg.strategy == "vanilla":
                        rng.permutation(L)
                    if empty[i]:
                        rng.choice(self.n_out, size=min(cfg.beta, self.n_out), replace=False)
            bt, keep = self._upload(csr, states, forced)
            _lib.call("slide_forward", self._ctx, _lib.C.byref(bt), 0, 0, None)
            ids = np.empty((nb, topn), np.int32)
            cnt = np.empty(nb, np.int32)
            _lib.call("slide_topk", self._ctx, topn, ids.ctypes.data, cnt.ctypes.data)
            out.extend(ids[i, : cnt[i]].astype(np.int64) for i in range(nb))
            self._live = keep
        return out


def train_network(net: SlideNetwork, dataset, *, workers: int = 1, on_batch=None, schedule: str | None = None) -> int:
    """Run the configured epochs over a dataset (reference network.py:398-425):
    batches in the seeded order ``data.batches(dataset, B, seed=(seed,
    epoch))``, the iteration counter running across epochs, a non-finite
    loss raising ``TrainingDivergedError``, ``on_batch(iteration, stats)``
    after every batch (raise from it to stop early).  ``dataset`` is a
    ``data.Dataset`` or a CSR ``data.Corpus`` (same order; batches go to the
    device without building SparseVectors).  Returns the iterations run."""
    from .data import Corpus, batches

    check_positive_int(workers, "workers")
    cfg = net.cfg
    if schedule is None:
        schedule = "sequential" if workers <= 1 else "snapshot"
    iteration = 0
    for epoch in range(cfg.epochs):
        for batch in batches(dataset, cfg.batch_size, seed=(cfg.seed, epoch)):
            iteration += 1
            if isinstance(dataset, Corpus):
                stats = net.train_batch_csr(HostCsr.from_corpus(batch), iteration, schedule=schedule)
            else:
                stats = net.train_batch(batch, iteration, workers=workers, schedule=schedule)
            if not np.isfinite(stats.loss):
                raise TrainingDivergedError(f"non-finite loss {stats.loss} at iteration {iteration}")
            if on_batch is not None:
                on_batch(iteration, stats)
    return iteration


# -- checkpoints (SLDE v1, reference network.py:478-548) ----------------------


def save_checkpoint(net: SlideNetwork, path, with_adam: bool = True):
    """Little-endian SLDE v1: per layer width, fan_in, kind, f32 w / b, adam
    flag and f32 moments + u64 steps (reference network.py:478-499).  The
    bytes equal the reference's for the same float32 state."""
    if net.shard_count > 1:
        raise NotImplementedError("save_checkpoint of a column-sharded network: gather the output layer first "
                                  "(sharded.gather_output_layer)")
    with open(path, "wb") as fh:
        fh.write(CHECKPOINT_MAGIC)
        fh.write(struct.pack("<II", CHECKPOINT_VERSION, len(net.layers)))
        for li, layer in enumerate(net.layers):
            fh.write(struct.pack("<IIB", layer.width, layer.fan_in, _KIND_CODES[layer.kind]))
            fh.write(layer._mat("w").contiguous().cpu().numpy().astype("<f4").tobytes())
            fh.write(layer._vec("b").cpu().numpy().astype("<f4").tobytes())
            fh.write(struct.pack("<B", 1 if with_adam else 0))
            if with_adam:
                fh.write(layer._mat("m").contiguous().cpu().numpy().astype("<f4").tobytes())
                fh.write(layer._mat("v").contiguous().cpu().numpy().astype("<f4").tobytes())
                fh.write(layer._vec("mb").cpu().numpy().astype("<f4").tobytes())
                fh.write(layer._vec("vb").cpu().numpy().astype("<f4").tobytes())
                fh.write(layer._vec("steps").cpu().numpy().astype("<u8").tobytes())


def load_checkpoint(path, cfg: TrainConfig | None = None) -> SlideNetwork:
    """Network (no tables) from an SLDE v1 file (reference network.py:502-548)."""
    import torch

    def read(fh, n):
        buf = fh.read(n)
        if len(buf) != n:
            raise ValueError("truncated checkpoint")
        return buf

    cfg = cfg or TrainConfig(batch_size=1)
    with open(path, "rb") as fh:
        if read(fh, 4) != CHECKPOINT_MAGIC:
            raise ValueError("not a SLDE checkpoint")
        version, n_layers = struct.unpack("<II", read(fh, 8))
        if version != CHECKPOINT_VERSION:
            raise ValueError(f"unsupported checkpoint version {version}")
        widths, payload, input_dim = [], [], None
        for _ in range(n_layers):
            width, fan_in, kind = struct.unpack("<IIB", read(fh, 9))
            input_dim = fan_in if input_dim is None else input_dim
            w = np.frombuffer(read(fh, 4 * width * fan_in), dtype="<f4").reshape(width, fan_in)
            b = np.frombuffer(read(fh, 4 * width), dtype="<f4")
            (has_adam,) = struct.unpack("<B", read(fh, 1))
            adam = None
            if has_adam:
                m = np.frombuffer(read(fh, 4 * width * fan_in), dtype="<f4").reshape(width, fan_in)
                v = np.frombuffer(read(fh, 4 * width * fan_in), dtype="<f4").reshape(width, fan_in)
                mb = np.frombuffer(read(fh, 4 * width), dtype="<f4")
                vb = np.frombuffer(read(fh, 4 * width), dtype="<f4")
                steps = np.frombuffer(read(fh, 8 * width), dtype="<u8")
                adam = (m, v, mb, vb, steps)
            widths.append(width)
            payload.append((w, b, _KIND_NAMES[kind], adam))
    net = SlideNetwork(input_dim, widths, cfg)
    for layer, (w, b, kind, adam) in zip(net.layers, payload):
        layer.kind = kind
        dev = net.w1t.device

        def put(dst, a):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(a)).to(dev))

        put(layer._mat("w"), w)
        put(layer._vec("b"), b)
        if adam is not None:
            put(layer._mat("m"), adam[0])
            put(layer._mat("v"), adam[1])
            put(layer._vec("mb"), adam[2])
            put(layer._vec("vb"), adam[3])
            put(layer._vec("steps"), adam[4].astype(np.int64))
    return net
