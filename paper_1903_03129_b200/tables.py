"""Per-layer (K, L) bucket index (drop-in for reference tables.py).

The buckets live on the device (``csrc/tables.cu``): one stable radix sort of
the N*L (table, key) inserts, FIFO tail / reservoir replay, and a directory
per table.  The host only keeps the rebuild schedule and the reservoir's
``random.Random`` stream (so it continues across rebuilds exactly like
tables.py:101).  ``tables`` is a host view, materialised on read; mutations of
the view (``clear()``, planting ``Bucket`` objects) are pushed back to the
device before the next query.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hashing import HashFamily, SimHashFamily
from .sparse import SparseVector


def _check_positive_int(value, name):
    if not isinstance(value, (int, np.integer)) or isinstance(value, bool) or value < 1:
        raise ValueError(f"{name} must be a positive integer, got {value!r}")
    return int(value)


class Bucket:
    """Fixed-capacity slot array plus the insert count (reference tables.py:26-41)."""

    __slots__ = ("slots", "head", "occupancy", "count")

    def __init__(self):
        self.slots = []
        self.head = 0
        self.occupancy = 0
        self.count = 0

    def ids(self) -> list:
        """Stored ids oldest first (FIFO ring order)."""
        if self.head:
            return self.slots[self.head :] + self.slots[: self.head]
        return self.slots


@dataclass
class RebuildSchedule:
    """Rebuild t at floor(sum_{i<=t} n0 e^{lam i} + 0.5) (reference tables.py:44-67)."""

    n0: int
    lam: float = 0.0
    t: int = field(default=0, init=False)
    next_at: int = field(init=False)
    _sum: float = field(init=False, repr=False)

    def __post_init__(self):
        _check_positive_int(self.n0, "n0")
        if self.lam < 0:
            raise ValueError(f"decay constant must be >= 0, got {self.lam}")
        self._sum = float(self.n0)
        self.next_at = math.floor(self._sum + 0.5)

    def due(self, iteration: int) -> bool:
        return iteration >= self.next_at

    def advance(self):
        self.t += 1
        self._sum += self.n0 * math.exp(self.lam * self.t)
        self.next_at = math.floor(self._sum + 0.5)


@dataclass
class RawCandidates:
    """Per-table bucket contents for one query (reference tables.py:70-75)."""

    per_table: list
    width: int


class _TableView(dict):
    """Host copy of one table; edits mark the owner dirty."""

    def __init__(self, owner, index, *a):
        super().__init__(*a)
        self._owner = owner
        self._index = index

    def clear(self):
        super().clear()
        self._owner._view_changed()

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._owner._view_changed()

    def __delitem__(self, key):
        super().__delitem__(key)
        self._owner._view_changed()


class LshTables:
    """L device hash tables for one layer plus rebuild state."""

    def __init__(self, family: HashFamily, *, policy: str = "fifo", capacity: int = 128,
                 schedule: RebuildSchedule | None = None, seed: int = 0, _ctx=None):
        if policy not in ("fifo", "reservoir"):
            raise ValueError(f"unknown insertion policy {policy!r}")
        _check_positive_int(capacity, "capacity")
        self.family = family
        self.policy = policy
        self.capacity = capacity
        self.schedule = schedule or RebuildSchedule(50)
        self.n_items = 0
        self.cached_dots = None
        self.cache_valid = False
        self._rng = random.Random(seed)
        self._ctx = _ctx
        self._owns_ctx = _ctx is None
        self._views = None
        self._dirty = False
        self._last_keys = None
        self._owner_rebuild = None  # set by SlideNetwork: rebuild from its device W2
        self._unit_cols = None  # set by SlideNetwork: physical column of every hidden unit

    # -- context ----------------------------------------------------------
    def _context(self):
        if self._ctx is None:
            from . import _device
            from .network import _family_desc

            desc = _lib.NetDesc()
            desc.input_dim = 1
            desc.hidden = self.family.dim
            desc.hidden_pad = _device.round_up(self.family.dim, 128)
            desc.n_out = 1
            desc.max_batch = 1
            keep = _family_desc(desc, self.family, self.capacity, self.policy)
            h = _lib.vp()
            _lib.call("slide_create", desc, _lib.vp(_device.stream_handle()), _lib.C.byref(h))
            self._ctx = h
            self._keep = keep
        return self._ctx

    def __del__(self):
        try:
            if self._owns_ctx and self._ctx is not None:
                _lib.lib().slide_destroy(self._ctx)
        except Exception:
            pass

    # -- construction -------------------------------------------------------
    def build(self, weights) -> None:
        """Hash every row and rebuild all L tables (reference tables.py:105-116)."""
        import torch

        from . import _device

        w = np.asarray(weights, dtype=np.float64)
        if w.ndim != 2 or w.shape[1] != self.family.dim:
            raise ValueError(f"expected weight matrix of shape (n, {self.family.dim}), got {w.shape}")
        self.family._check_device_width()
        ctx = self._context()
        x = _device.pad_rows(w, self.family.dim)
        keys = torch.empty((w.shape[0], self.family.l), dtype=torch.int32, device=x.device)
        self.family._keys_dev(x, w.shape[0], self.family.dim, keys)
        self._insert_dev(keys, w.shape[0])
        self.cache_valid = isinstance(self.family, SimHashFamily)

    def _insert_dev(self, keys_dev, n):
        ctx = self._context()
        st = _lib.mt_state_from_random(self._rng)
        _lib.call("slide_build_tables_from_keys", ctx, keys_dev.data_ptr(), n, st.ctypes.data)
        _lib.mt_state_to_random(st, self._rng)
        self.n_items = n
        self._last_keys = keys_dev
        self._views = None
        self._dirty = False

    def insert_codes(self, codes: np.ndarray) -> None:
        """Insert ids 0..n-1 with precomputed (n, L) keys into empty tables
        (reference tables.py:127-161)."""
        from . import _device

        codes = np.asarray(codes, dtype=np.int64)
        if codes.ndim != 2 or codes.shape[1] != self.family.l:
            raise ValueError(f"codes must have shape (n, {self.family.l})")
        if self._nonempty():
            raise NotImplementedError("device tables insert into cleared tables only (call build or clear first)")
        self._insert_dev(_device.to_dev(codes.astype(np.uint32).view(np.int32)), codes.shape[0])

    def _nonempty(self) -> bool:
        if self._views is not None:
            return any(len(v) for v in self._views)
        nb = _lib.i64()
        ns = _lib.i64()
        ni = _lib.i64()
        if self._ctx is None:
            return False
        _lib.call("slide_tables_info", self._ctx, _lib.C.byref(nb), _lib.C.byref(ns), _lib.C.byref(ni))
        return nb.value > 0

    def _clear(self):
        if self._ctx is not None:
            _lib.call("slide_clear_tables", self._ctx)
        self._views = None

    # -- host view ------------------------------------------------------------
    @property
    def tables(self):
        if self._views is None:
            self._views = self._export()
        return self._views

    @tables.setter
    def tables(self, value):
        self._views = [v if isinstance(v, _TableView) else _TableView(self, t, v) for t, v in enumerate(value)]
        self._dirty = True

    def _export(self):
        L = self.family.l
        views = [_TableView(self, t) for t in range(L)]
        if self._ctx is None:
            return views
        nb, ns, ni = _lib.i64(), _lib.i64(), _lib.i64()
        _lib.call("slide_tables_info", self._ctx, _lib.C.byref(nb), _lib.C.byref(ns), _lib.C.byref(ni))
        r = nb.value
        if r == 0:
            return views
        skeys = np.empty(r, np.uint32)
        counts = np.empty(r, np.int32)
        starts = np.empty(r, np.int32)
        lens = np.empty(r, np.int32)
        ids = np.empty(ns.value, np.int32)
        _lib.call("slide_tables_export", self._ctx, skeys.ctypes.data, counts.ctypes.data, starts.ctypes.data,
                  lens.ctypes.data, ids.ctypes.data)
        kb = self.family.key_bits
        cap = self.capacity
        for q in range(r):
            t = int(skeys[q]) >> kb
            key = int(skeys[q]) & ((1 << kb) - 1)
            b = Bucket()
            kept = ids[starts[q] : starts[q] + lens[q]].tolist()
            cnt = int(counts[q])
            b.count = cnt
            b.occupancy = len(kept)
            if self.policy == "fifo" and cnt > cap:
                # ring slot p % cap holds insert p of the kept tail
                slots = [0] * cap
                for j, nid in enumerate(kept):
                    slots[(cnt - cap + j) % cap] = nid
                b.slots = slots
                b.head = cnt % cap
            else:
                b.slots = kept
            dict.__setitem__(views[t], key, b)
        return views

    def _view_changed(self):
        self._dirty = True

    def sync_to_device(self):
        """Push host-view edits (cleared tables, planted buckets) to the device."""
        if not self._dirty or self._views is None:
            return
        kb = self.family.key_bits
        sk, cnt, st, ln, ids = [], [], [], [], []
        for t, view in enumerate(self._views):
            for key in sorted(view):
                b = view[key]
                sk.append((t << kb) | int(key))
                cnt.append(int(b.count))
                st.append(len(ids))
                ln.append(len(b.slots))
                ids.extend(int(s) for s in b.slots)
        sk = np.asarray(sk, np.uint32)
        cnt = np.asarray(cnt, np.int32)
        st = np.asarray(st, np.int32)
        ln = np.asarray(ln, np.int32)
        ids = np.asarray(ids, np.int32)
        _lib.call("slide_tables_load", self._context(), sk.ctypes.data, cnt.ctypes.data, st.ctypes.data,
                  ln.ctypes.data, len(sk), ids.ctypes.data, len(ids), self.n_items)
        self._dirty = False

    # -- queries --------------------------------------------------------------
    def query_union_batch(self, queries, *, return_device: bool = False):
        """Ascending union of every probed bucket for each dense query row --
        the sampler's ``hard_threshold(min_freq=1)`` over all L tables
        (reference samplers.py:109-112) -- for a whole batch on the device
        (``slide_query_union``: hash, probe, union).  Returns a list of int64
        arrays, or the device (counts, ids) pair with ``return_device``."""
        import torch

        from . import _device

        q = np.asarray(queries, dtype=np.float64)
        if q.ndim != 2 or q.shape[1] != self.family.dim:
            raise ValueError(f"expected query rows of shape (n, {self.family.dim}), got {q.shape}")
        n = q.shape[0]
        self.sync_to_device()
        if self._ctx is None or not self.n_items or n == 0:
            return [np.zeros(0, dtype=np.int64) for _ in range(n)]
        if self._unit_cols is not None:  # a network's tables hash in its physical unit order
            cols = np.asarray(self._unit_cols())
            qp = np.zeros_like(q)
            qp[:, cols] = q
            q = qp
        x = q if isinstance(queries, torch.Tensor) else _device.pad_rows(q, _device.round_up(self.family.dim, 128))
        return self._query_union_dev(x, n, return_device)

    def _query_union_dev(self, x_dev, n: int, return_device: bool = False):
        import torch

        stride = self.family.l * self.capacity
        cnt = torch.empty(n, dtype=torch.int32, device=x_dev.device)
        ids = torch.empty((n, stride), dtype=torch.int32, device=x_dev.device)
        _lib.call("slide_query_union", self._context(), x_dev.data_ptr(), n, self.n_items, stride, cnt.data_ptr(),
                  ids.data_ptr())
        if return_device:
            return cnt, ids
        c = cnt.cpu().numpy()
        got = ids.cpu().numpy()
        return [(got[i, : c[i]] & 0x7FFFFFFF).astype(np.int64) for i in range(n)]

    def query(self, v: SparseVector) -> RawCandidates:
        """Hash the query and probe each table once (reference tables.py:165-169)."""
        if v.dim != self.family.dim:
            raise ValueError(f"lsh query: vector dim {v.dim} does not match expected {self.family.dim}")
        return self.query_codes(self.family.hash(v))

    def query_codes(self, codes) -> RawCandidates:
        """Exactly L probes (reference tables.py:171-176): each probed bucket's
        kept ids come back from the device in the reference's physical slot
        order (a full FIFO bucket is a ring whose head is its insert count
        modulo the capacity, ref tables.py:130-145)."""
        self.sync_to_device()
        codes = np.asarray(codes, dtype=np.int64).reshape(1, -1)
        L = self.family.l
        if codes.shape[1] != L:
            raise ValueError(f"expected {L} codes, got {codes.shape[1]}")
        if self._ctx is None:
            return RawCandidates([[] for _ in range(L)], self.n_items)
        if self._views is not None:  # host-side edits already pushed; views equal the device
            return RawCandidates([list(v[int(codes[0, t])].slots) if int(codes[0, t]) in v else []
                                  for t, v in enumerate(self._views)], self.n_items)
        cap = self.capacity
        keys = np.ascontiguousarray(codes.astype(np.uint32))
        lens = np.empty(L, np.int32)
        counts = np.empty(L, np.int32)
        ids = np.empty(L * cap, np.int32)
        _lib.call("slide_tables_probe_ids", self._ctx, keys.ctypes.data, 1, lens.ctypes.data, counts.ctypes.data,
                  ids.ctypes.data)
        per = []
        for t in range(L):
            kept = ids[t * cap : t * cap + lens[t]].tolist()
            cnt = int(counts[t])
            if self.policy == "fifo" and cnt > cap:
                slots = [0] * cap
                for j, nid in enumerate(kept):
                    slots[(cnt - cap + j) % cap] = nid
                kept = slots
            per.append(kept)
        return RawCandidates(per, self.n_items)

    # -- maintenance ----------------------------------------------------------
    def maybe_rebuild(self, iteration: int, weights=None) -> bool:
        """Rebuild when the schedule is due (reference tables.py:180-196)."""
        if not self.schedule.due(iteration):
            return False
        if self.cache_valid and self._last_keys is not None:
            self._clear()
            self._insert_dev(self._last_keys, self.n_items)
        elif self._owner_rebuild is not None and weights is None:
            self._owner_rebuild()
        else:
            self.build(weights)
        self.schedule.advance()
        return True

    def mark_weights_changed(self):
        self.cache_valid = False

    def incremental_simhash_update(self, neuron_id: int, changed):
        if not isinstance(self.family, SimHashFamily):
            raise TypeError("incremental updates require a simhash family")
        if self.cached_dots is None or not (0 <= neuron_id < self.n_items):
            raise KeyError(f"no cached codes for neuron {neuron_id}; build() it first")
        raise NotImplementedError("incremental SimHash is off the training path (SURVEY.md section 2)")

    def occupancy_totals(self) -> list:
        return [sum(b.occupancy for b in tbl.values()) for tbl in self.tables]
