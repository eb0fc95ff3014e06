"""SLIDE hot-path CPU oracle -- TEST INFRASTRUCTURE ONLY.

Who may use this module: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``, and only as the
checker or the reported CPU baseline.  The product package
(``paper_1903_03129_b200``) never imports it; its CUDA path fails loudly when
the extension is missing instead of falling back here.

What it is: a numpy restatement of the reference's adaptive-sparsity training
step (reference = the pure-Python ``slide`` 0.1.0 package, read-only at
/root/reference/pkg/src/slide).  Every function cites the reference
file:line whose behaviour it restates.  The structure is deliberately
different (vectorised bucket builds, a transposed W1, functional helpers), the
semantics are the same:

* SimHash ``bit = dot > 0`` (sign(0) -> 0), hashing.py:168-178;
* DWTA winner = max value, ties to the lowest bin offset, donor-chain
  densification, hashing.py:219-259;
* FIFO buckets keep the ``cap`` highest ids, reservoir buckets replay
  ``random.Random`` draws in (table, id) order, tables.py:127-161;
* vanilla / topk / hard_threshold samplers, samplers.py:57-112;
* active set = sorted(sample U labels) with the beta-random fallback,
  network.py:225-239;
* sparse forward, softmax-CE, backward with pre-update weights and per-row
  step-counter Adam, network.py:241-336, 428-451;
* two batch schedules: ``sequential`` (= reference ``train_batch`` with
  workers=1, network.py:340-379) and ``snapshot`` (SURVEY.md section 8(c):
  every slot's forward/backward on the pre-step weights, then ``_adam_block``
  per captured entry in slot order).

Parity pin: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by importing the reference itself
(``tests/golden/make_golden.py``); see DESIGN.md "Oracle".

Random streams (numpy ``Generator``/PCG64 and Python ``random.Random``) are
the same third-party generators the reference calls, called with the same
seeds in the same order (reference call sites: network.py:83,187,231,353;
hashing.py:132-140,214-215; samplers.py:69; tables.py:101,149-161).
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# hashing (reference hashing.py)
# ---------------------------------------------------------------------------


def mix64(a: int, b: int, c: int) -> int:
    """splitmix-style 64-bit mix; restates hashing.py:31-38."""
    x = (a * 0x9E3779B97F4A7C15 + b * 0xBF58476D1CE4E5B9 + c * 0x94D049BB133111EB) & _M64
    for shift, mult in ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB)):
        x ^= x >> shift
        x = (x * mult) & _M64
    return x ^ (x >> 31)


def pack_keys(codes: np.ndarray, bits: int) -> np.ndarray:
    """Concatenate the last axis of sub-codes, code j at bit offset j*bits
    (hashing.py:41-48)."""
    codes = np.asarray(codes, dtype=np.int64)
    k = codes.shape[-1]
    weights = np.left_shift(np.int64(1), np.arange(k, dtype=np.int64) * bits)
    return (codes * weights).sum(axis=-1, dtype=np.int64)


@dataclass
class SimHashParams:
    """K*L sparse {+1,-1} projections (hashing.py:121-148)."""

    dim: int
    k: int
    l: int
    idx: np.ndarray  # (K*L, c) int64, each row sorted
    signs: np.ndarray  # (K*L, c) float64 in {-1, +1}

    @property
    def key_bits(self) -> int:
        return self.k

    def projection_matrix(self) -> np.ndarray:
        """Dense (dim, K*L) projection, zero off the stored entries."""
        p = np.zeros((self.dim, self.idx.shape[0]))
        cols = np.repeat(np.arange(self.idx.shape[0]), self.idx.shape[1])
        p[self.idx.ravel(), cols] = self.signs.ravel()
        return p


def simhash_params(dim: int, k: int, l: int, sparsity: float, seed: int) -> SimHashParams:
    """Projection draw order of hashing.py:132-140: one sorted
    ``choice(d, c, replace=False)`` per projection, then all signs at once."""
    rng = np.random.default_rng(seed)
    c = min(dim, max(1, int(round(dim * sparsity))))
    n_codes = k * l
    idx = np.stack([np.sort(rng.choice(dim, size=c, replace=False)) for _ in range(n_codes)])
    signs = rng.choice(np.array([-1.0, 1.0]), size=(n_codes, c))
    return SimHashParams(dim, k, l, idx.astype(np.int64), signs)


def simhash_keys(params: SimHashParams, dense: np.ndarray) -> np.ndarray:
    """(n, dim) -> (n, L) keys: bit = [projection . v > 0], key = sum bit_j 2^j
    (hashing.py:150-178, tables.py:118-121)."""
    dense = np.atleast_2d(np.asarray(dense, dtype=np.float64))
    dots = dense @ params.projection_matrix()
    bits = (dots > 0.0).reshape(dense.shape[0], params.l, params.k)
    return pack_keys(bits, 1)


@dataclass
class DwtaParams:
    """Permutation-bin family state (hashing.py:196-217)."""

    dim: int
    k: int
    l: int
    m: int
    bins_per_perm: int
    n_perms: int
    bits: int
    perms: np.ndarray  # (n_perms, dim)
    salt: int

    @property
    def key_bits(self) -> int:
        return self.bits * self.k

    @property
    def n_codes(self) -> int:
        return self.k * self.l

    def donor(self, g: int, attempt: int) -> int:
        return mix64(self.salt, g, attempt) % self.n_codes


def dwta_params(dim: int, k: int, l: int, m: int, seed: int) -> DwtaParams:
    """ceil(d/m) bins per permutation, ceil(KLm/d) permutations, ceil(log2 m)
    bits per code, salt = mix(seed, 0xD1F7, 0xA0B1) (hashing.py:207-217)."""
    bins_per_perm = -(-dim // m)
    n_perms = -(-(k * l * m) // dim)
    bits = max(1, math.ceil(math.log2(m))) if m > 1 else 1
    rng = np.random.default_rng(seed)
    perms = np.stack([rng.permutation(dim) for _ in range(n_perms)])
    salt = mix64(seed & _M64, 0xD1F7, 0xA0B1)
    return DwtaParams(dim, k, l, m, bins_per_perm, n_perms, bits, perms.astype(np.int64), salt)


def dwta_keys(params: DwtaParams, dense: np.ndarray) -> np.ndarray:
    """(n, dim) -> (n, L) keys.  Only nonzero entries take part (a sparse
    vector's stored entries, sparse.py:49-53).  Per global bin: winner = max
    value, ties to the lowest in-bin offset (hashing.py:236-259); empty bins
    borrow the code of the first occupied donor on their mix chain, else 0
    (hashing.py:219-231)."""
    dense = np.atleast_2d(np.asarray(dense, dtype=np.float64))
    n = dense.shape[0]
    p = params
    codes = np.zeros((n, p.n_codes), dtype=np.int64)
    occupied = np.zeros((n, p.n_codes), dtype=bool)
    for g in range(p.n_codes):
        q, b = divmod(g, p.bins_per_perm)
        lo = b * p.m
        hi = min(lo + p.m, p.dim)
        vals = dense[:, p.perms[q, lo:hi]]
        present = vals != 0.0
        masked = np.where(present, vals, -np.inf)
        codes[:, g] = np.argmax(masked, axis=1)  # first maximum = lowest offset
        occupied[:, g] = present.any(axis=1)
    codes[~occupied] = 0
    for row in np.nonzero(~occupied.all(axis=1))[0]:
        occ = occupied[row]
        orig = codes[row].copy()
        for g in np.nonzero(~occ)[0]:
            code = 0
            for attempt in range(1, 101):
                d = p.donor(int(g), attempt)
                if occ[d]:
                    code = orig[d]
                    break
            codes[row, g] = code
    return pack_keys(codes.reshape(n, p.l, p.k), p.bits)


def family_keys(params, dense) -> np.ndarray:
    if isinstance(params, SimHashParams):
        return simhash_keys(params, dense)
    return dwta_keys(params, dense)


# ---------------------------------------------------------------------------
# tables (reference tables.py)
# ---------------------------------------------------------------------------


@dataclass
class Schedule:
    """Rebuild t at floor(sum_{i<=t} n0 e^{lam i} + 0.5) (tables.py:44-67)."""

    n0: int
    lam: float = 0.0
    done: int = 0
    acc: float = field(init=False)
    next_at: int = field(init=False)

    def __post_init__(self):
        self.acc = float(self.n0)
        self.next_at = math.floor(self.acc + 0.5)

    def due(self, iteration: int) -> bool:
        return iteration >= self.next_at

    def advance(self):
        self.done += 1
        self.acc += self.n0 * math.exp(self.lam * self.done)
        self.next_at = math.floor(self.acc + 0.5)


def build_buckets(keys: np.ndarray, cap: int, policy: str, pyrand: random.Random | None):
    """Per table: dict key -> (physical slot array, insert count).

    Ids 0..n-1 enter each table in ascending order (tables.py:127-161).
    FIFO: a full bucket overwrites its ring, so it ends up holding the ``cap``
    highest ids; slot j holds the id at the last insert position p with
    p % cap == j.  Reservoir: the first ``cap`` ids fill the slots, every
    later insert n (1-based count) draws u1 and, when u1*n < cap, u2 picks the
    slot; draws are consumed across tables in (table, id) order.
    """
    keys = np.asarray(keys, dtype=np.int64)
    n, n_tables = keys.shape
    out = []
    for t in range(n_tables):
        col = keys[:, t]
        order = np.argsort(col, kind="stable")
        sk = col[order]
        starts = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]])
        ends = np.r_[starts[1:], n]
        table = {}
        overflow = []
        for s, e in zip(starts.tolist(), ends.tolist()):
            ids = order[s:e]
            cnt = e - s
            if cnt <= cap:
                table[int(sk[s])] = (ids.copy(), cnt)
            elif policy == "fifo":
                last = ids[cnt - cap :]
                pos = np.arange(cnt - cap, cnt) % cap
                slots = np.empty(cap, dtype=np.int64)
                slots[pos] = last
                table[int(sk[s])] = (slots, cnt)
            else:
                slots = ids[:cap].copy()
                table[int(sk[s])] = (slots, cnt)
                for j in range(cap, cnt):
                    overflow.append((int(ids[j]), j + 1, int(sk[s])))
        if overflow:
            rand = pyrand.random
            overflow.sort()
            for nid, count, key in overflow:
                if rand() * count < cap:
                    table[key][0][int(rand() * cap)] = nid
        out.append(table)
    return out


class BucketTable:
    """One table in array form: sorted distinct keys, insert counts and a CSR
    of physical slots -- the same content as a ``build_buckets`` dict (its
    ``get`` has the dict's result), built without a per-bucket Python loop so
    the oracle can hold full-size tables (205k - 4M rows x L)."""

    def __init__(self, keys, counts, ptr, slots):
        self.keys = np.asarray(keys, dtype=np.int64)
        self.counts = np.asarray(counts, dtype=np.int64)
        self.ptr = np.asarray(ptr, dtype=np.int64)
        self.slots = np.asarray(slots, dtype=np.int64)

    def __len__(self):
        return self.keys.size

    def get(self, key):
        i = int(np.searchsorted(self.keys, key))
        if i >= self.keys.size or self.keys[i] != key:
            return None
        return self.slots[self.ptr[i] : self.ptr[i + 1]], int(self.counts[i])

    def items(self):
        for i in range(self.keys.size):
            yield int(self.keys[i]), (self.slots[self.ptr[i] : self.ptr[i + 1]], int(self.counts[i]))


def build_bucket_arrays(keys: np.ndarray, cap: int, policy: str, pyrand: random.Random | None) -> list:
    """``build_buckets`` (tables.py:127-161) in array form: per table a stable
    sort by key gives every run of ids in ascending insert order; runs of at
    most ``cap`` ids are stored whole; an overflowing FIFO run keeps its last
    ``cap`` inserts at ring slots p % cap; an overflowing reservoir run keeps
    its first ``cap`` ids and then replays the draws (u1 * count < cap, slot
    int(u2 * cap)) in (table, id) order, continuing ``pyrand``."""
    keys = np.asarray(keys, dtype=np.int64)
    n, n_tables = keys.shape
    out = []
    for t in range(n_tables):
        col = keys[:, t]
        order = np.argsort(col, kind="stable")
        sk = col[order]
        starts = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]]) if n else np.zeros(0, np.int64)
        ends = np.r_[starts[1:], n].astype(np.int64)
        counts = ends - starts
        kept = np.minimum(counts, cap)
        ptr = np.zeros(starts.size + 1, dtype=np.int64)
        np.cumsum(kept, out=ptr[1:])
        # position of every kept slot inside its run: first `kept` inserts
        run = np.repeat(np.arange(starts.size), kept)
        j = np.arange(ptr[-1]) - ptr[run]
        slots = order[starts[run] + j]
        over = np.flatnonzero(counts > cap)
        if over.size and policy == "fifo":
            for r in over.tolist():
                cnt = int(counts[r])
                last = order[starts[r] + cnt - cap : starts[r] + cnt]
                pos = np.arange(cnt - cap, cnt) % cap
                seg = np.empty(cap, dtype=np.int64)
                seg[pos] = last
                slots[ptr[r] : ptr[r] + cap] = seg
        elif over.size:
            # (id, 1-based count, run) of every insert past the cap, id order
            ev = []
            for r in over.tolist():
                for q in range(cap, int(counts[r])):
                    ev.append((int(order[starts[r] + q]), q + 1, r))
            ev.sort()
            rand = pyrand.random
            for nid, count, r in ev:
                if rand() * count < cap:
                    slots[ptr[r] + int(rand() * cap)] = nid
        out.append(BucketTable(sk[starts], counts, ptr, slots))
    return out


def probe(buckets, keys_row) -> list:
    """Exactly L probes; missing keys give empty lists (tables.py:171-176)."""
    res = []
    for t, key in enumerate(np.asarray(keys_row).tolist()):
        hit = buckets[t].get(int(key))
        res.append(hit[0] if hit is not None else np.empty(0, dtype=np.int64))
    return res


# ---------------------------------------------------------------------------
# samplers (reference samplers.py)
# ---------------------------------------------------------------------------


def vanilla_ids(per_table, beta: int, order) -> np.ndarray:
    """Union of whole buckets over the first tau probes of ``order``, tau the
    first prefix whose union reaches beta distinct ids (checked after every
    probe, empty ones included), else all L (samplers.py:57-87)."""
    seen: set = set()
    for t in order:
        seen.update(np.asarray(per_table[t]).tolist())
        if len(seen) >= beta:
            break
    return np.array(sorted(seen), dtype=np.int64)


def _freq(per_table):
    allids = [np.asarray(b, dtype=np.int64) for b in per_table if len(b)]
    if not allids:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
    return np.unique(np.concatenate(allids), return_counts=True)


def topk_ids(per_table, beta: int) -> np.ndarray:
    """beta ids by (frequency desc, id asc) (samplers.py:97-106)."""
    ids, cnt = _freq(per_table)
    order = np.lexsort((ids, -cnt))
    return ids[order][:beta]


def threshold_ids(per_table, min_freq: int) -> np.ndarray:
    """ids with frequency >= min_freq, ascending (samplers.py:109-112)."""
    ids, cnt = _freq(per_table)
    return ids[cnt >= min_freq]


def sampled_ids(per_table, strategy: str, beta: int, min_freq: int, rng) -> np.ndarray:
    """Dispatch of samplers.py:115-120; vanilla consumes rng.permutation(L)."""
    if strategy == "vanilla":
        return vanilla_ids(per_table, beta, rng.permutation(len(per_table)))
    if strategy == "topk":
        return topk_ids(per_table, beta)
    return threshold_ids(per_table, min_freq)


# ---------------------------------------------------------------------------
# network (reference network.py), one hidden ReLU layer + softmax output
# ---------------------------------------------------------------------------


@dataclass
class AdamCfg:
    lr: float = 1e-3
    b1: float = 0.9
    b2: float = 0.999
    eps: float = 1e-8


@dataclass
class LshSpec:
    family: str = "simhash"
    k: int = 6
    l: int = 25
    cap: int = 128
    policy: str = "fifo"
    sparsity: float = 1.0 / 3.0
    bin_size: int = 8
    strategy: str = "vanilla"
    beta: int = 128
    min_freq: int = 1


class OutputLsh:
    """Hash params + buckets + schedule + reservoir stream of the output layer
    (network.py:199-221, tables.py:81-116)."""

    def __init__(self, spec: LshSpec, dim: int, seed: int, n0: int, lam: float, layer_index: int = 1):
        fam_seed = seed + 7919 * (layer_index + 1)
        if spec.family == "simhash":
            self.params = simhash_params(dim, spec.k, spec.l, spec.sparsity, fam_seed)
        elif spec.family == "dwta":
            self.params = dwta_params(dim, spec.k, spec.l, spec.bin_size, fam_seed)
        else:
            raise ValueError(f"oracle covers simhash/dwta only, got {spec.family!r}")
        self.spec = spec
        self.schedule = Schedule(n0, lam)
        self.pyrand = random.Random(seed + 104729 * (layer_index + 1))
        self.buckets = None

    def build(self, w2: np.ndarray):
        keys = family_keys(self.params, w2)
        self.buckets = build_bucket_arrays(keys, self.spec.cap, self.spec.policy, self.pyrand)
        return keys

    def query(self, h_dense: np.ndarray):
        keys = family_keys(self.params, h_dense[None, :])[0]
        return keys, probe(self.buckets, keys)


@dataclass
class NetState:
    """Parameters of a 1-hidden-layer SLIDE net, float64.

    ``w1t`` is W1 transposed, (D, H): the reference keeps (H, D)
    (network.py:83); the transpose changes no arithmetic."""

    w1t: np.ndarray
    b1: np.ndarray
    m1t: np.ndarray
    v1t: np.ndarray
    mb1: np.ndarray
    vb1: np.ndarray
    steps1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    m2: np.ndarray
    v2: np.ndarray
    mb2: np.ndarray
    vb2: np.ndarray
    steps2: np.ndarray

    def copy(self) -> "NetState":
        return NetState(**{k: v.copy() for k, v in self.__dict__.items()})


def init_state(input_dim: int, hidden: int, n_out: int, seed: int) -> NetState:
    """One default_rng(seed): W1 ~ U(+-1/sqrt(D)) (H, D) then W2 ~ U(+-1/sqrt(H))
    (N, H); biases and moments zero (network.py:79-89, 187-193)."""
    rng = np.random.default_rng(seed)
    b = 1.0 / np.sqrt(input_dim)
    w1 = rng.uniform(-b, b, size=(hidden, input_dim))
    b = 1.0 / np.sqrt(hidden)
    w2 = rng.uniform(-b, b, size=(n_out, hidden))
    z = np.zeros
    return NetState(
        np.ascontiguousarray(w1.T), z(hidden), z((input_dim, hidden)), z((input_dim, hidden)),
        z(hidden), z(hidden), z(hidden, dtype=np.int64),
        w2, z(n_out), z((n_out, hidden)), z((n_out, hidden)), z(n_out), z(n_out), z(n_out, dtype=np.int64),
    )


@dataclass
class SlotTrace:
    """What one slot's forward produced (network.py:145-158, 241-286)."""

    x_idx: np.ndarray
    x_val: np.ndarray
    h: np.ndarray  # dense hidden activation (H,), zeros where ReLU clamped
    keys: np.ndarray | None  # output-layer query keys (L,) or None
    sampled: np.ndarray | None  # sampler output before labels (sorted)
    fell_back: bool
    active: np.ndarray  # sorted output active ids
    logits: np.ndarray
    probs: np.ndarray
    loss: float


@dataclass
class SlotGrads:
    """Captured gradients of one slot (the ``capture`` list of network.py:317-327)."""

    active: np.ndarray
    delta: np.ndarray  # output error per active row
    h_idx: np.ndarray  # nz(h)
    h_val: np.ndarray
    dh: np.ndarray | None  # hidden error on nz(h), None if h empty
    x_idx: np.ndarray
    x_val: np.ndarray
    # |W2[A, nz(h)]|^T |delta|: the magnitude of the terms dh sums (dh cancels
    # because delta sums to ~0); parity tests scale the hidden layer's fp32
    # rounding floor by it
    dh_abs: np.ndarray | None = None


def slot_forward(st: NetState, lsh: OutputLsh | None, x_idx, x_val, labels, rng, n_out: int) -> SlotTrace:
    """Forward of one sample (network.py:241-286) with the output active set
    of network.py:225-239 and the loss of network.py:154-158."""
    x_idx = np.asarray(x_idx, dtype=np.int64)
    x_val = np.asarray(x_val, dtype=np.float64)
    if x_idx.size:
        z1 = x_val @ st.w1t[x_idx] + st.b1
    else:
        z1 = st.b1.copy()
    h = np.maximum(z1, 0.0)
    nz = np.flatnonzero(h > 0)
    keys = sampled = None
    fell_back = False
    if lsh is not None:
        keys, per_table = lsh.query(h)
        spec = lsh.spec
        sampled = sampled_ids(per_table, spec.strategy, spec.beta, spec.min_freq, rng)
        ids = sampled
        if ids.size == 0:
            fell_back = True
            ids = rng.choice(n_out, size=min(spec.beta, n_out), replace=False)
        if labels is not None and len(labels):
            active = np.union1d(ids, np.asarray(sorted(labels), dtype=np.int64)).astype(np.int64)
        else:
            active = np.sort(np.asarray(ids, dtype=np.int64))
    else:
        active = np.arange(n_out, dtype=np.int64)
    if nz.size:
        logits = st.w2[np.ix_(active, nz)] @ h[nz] + st.b2[active]
    else:
        logits = st.b2[active].copy()
    e = np.exp(logits - (logits.max() if logits.size else 0.0))
    probs = e / e.sum()
    loss = float("nan")
    if labels is not None and len(labels):
        pos = np.searchsorted(active, np.asarray(list(labels), dtype=np.int64))
        loss = float(-np.log(np.maximum(probs[pos], 1e-300)).mean())
    return SlotTrace(x_idx, x_val, h, keys, sampled, fell_back, active, logits, probs, loss)


def slot_backward(st: NetState, tr: SlotTrace, labels) -> SlotGrads:
    """Errors of one slot from the weights in ``st`` (network.py:290-336):
    delta = p - 1/|Y| on labels; dh = W2[A, nz(h)]^T delta (pre-update)."""
    lab = np.asarray(list(labels), dtype=np.int64)
    pos = np.searchsorted(tr.active, lab)
    if np.any(pos >= tr.active.size) or np.any(tr.active[np.minimum(pos, tr.active.size - 1)] != lab):
        raise ValueError("a true label is missing from the output active set")
    delta = tr.probs.copy()
    delta[pos] -= 1.0 / lab.size
    h_idx = np.flatnonzero(tr.h > 0)
    h_val = tr.h[h_idx]
    dh = dh_abs = None
    if h_idx.size:
        blk = st.w2[np.ix_(tr.active, h_idx)]
        dh = blk.T @ delta
        dh_abs = np.abs(blk).T @ np.abs(delta)
    return SlotGrads(tr.active, delta, h_idx, h_val, dh, tr.x_idx, tr.x_val, dh_abs)


def _adam_rows(w, m, v, b, mb, vb, steps, rows, cols, grad, bgrad, cfg: AdamCfg):
    """Per-row-counter Adam on the (rows x cols) block plus row biases
    (network.py:428-451).  ``w``/``m``/``v`` are indexed [row, col]."""
    t = steps[rows] + 1
    steps[rows] = t
    bc1 = 1.0 - cfg.b1 ** t
    bc2 = 1.0 - cfg.b2 ** t
    if cols is not None and len(cols):
        ix = np.ix_(rows, cols)
        mm = cfg.b1 * m[ix] + (1 - cfg.b1) * grad
        vv = cfg.b2 * v[ix] + (1 - cfg.b2) * grad * grad
        m[ix] = mm
        v[ix] = vv
        w[ix] -= cfg.lr * (mm / bc1[:, None]) / (np.sqrt(vv / bc2[:, None]) + cfg.eps)
    mbb = cfg.b1 * mb[rows] + (1 - cfg.b1) * bgrad
    vbb = cfg.b2 * vb[rows] + (1 - cfg.b2) * bgrad * bgrad
    mb[rows] = mbb
    vb[rows] = vbb
    b[rows] -= cfg.lr * (mbb / bc1) / (np.sqrt(vbb / bc2) + cfg.eps)


def apply_slot_update(st: NetState, g: SlotGrads, cfg: AdamCfg):
    """The two ``_adam_block`` calls one slot's backward makes
    (network.py:311-336): output rows first; if h is empty only the output
    biases move and the hidden layer is left alone; if x is empty the hidden
    layer is bias-only."""
    if g.h_idx.size == 0:
        _adam_rows(st.w2, st.m2, st.v2, st.b2, st.mb2, st.vb2, st.steps2, g.active, None, None, g.delta, cfg)
        return
    grad2 = np.outer(g.delta, g.h_val)
    _adam_rows(st.w2, st.m2, st.v2, st.b2, st.mb2, st.vb2, st.steps2, g.active, g.h_idx, grad2, g.delta, cfg)
    # hidden layer: rows = nz(h), cols = x.idx; state indexed [hidden, feature]
    w1, m1, v1 = st.w1t.T, st.m1t.T, st.v1t.T
    if g.x_idx.size == 0:
        _adam_rows(w1, m1, v1, st.b1, st.mb1, st.vb1, st.steps1, g.h_idx, None, None, g.dh, cfg)
    else:
        grad1 = np.outer(g.dh, g.x_val)
        _adam_rows(w1, m1, v1, st.b1, st.mb1, st.vb1, st.steps1, g.h_idx, g.x_idx, grad1, g.dh, cfg)


@dataclass
class StepResult:
    losses: list
    traces: list
    grads: list
    rebuilt: bool
    active_fraction: float


def train_step(st: NetState, lsh: OutputLsh | None, batch, iteration: int, seed: int,
               n_out: int, cfg: AdamCfg, mode: str = "sequential", slot_offset: int = 0) -> StepResult:
    """One batch.  ``sequential`` restates train_batch(workers=1)
    (network.py:340-379): slot i forwards with default_rng((seed, it, i)) on
    the weights already updated by slots < i.  ``snapshot``:
    all slots forward/backward on the pre-step weights, then the updates are
    applied per slot in slot order.  Both end with the rebuild barrier
    (network.py:368-373): a due rebuild is a full re-hash of the current W2.
    """
    if mode not in ("sequential", "snapshot"):
        raise ValueError(f"unknown mode {mode!r}")
    traces, grads, losses = [], [], []
    for i, (x_idx, x_val, labels) in enumerate(batch):
        rng = np.random.default_rng((seed, iteration, slot_offset + i))
        tr = slot_forward(st, lsh, x_idx, x_val, labels, rng, n_out)
        g = slot_backward(st, tr, labels)
        if mode == "sequential":
            apply_slot_update(st, g, cfg)
        traces.append(tr)
        grads.append(g)
        losses.append(tr.loss)
    if mode == "snapshot":
        for g in grads:
            apply_slot_update(st, g, cfg)
    rebuilt = False
    if lsh is not None and lsh.schedule.due(iteration):
        lsh.build(st.w2)
        lsh.schedule.advance()
        rebuilt = True
    frac = float(np.mean([tr.active.size / n_out for tr in traces]))
    return StepResult(losses, traces, grads, rebuilt, frac)


def predict_ranked(st: NetState, lsh: OutputLsh | None, x_idx, x_val, rng, n_out: int) -> np.ndarray:
    """Sampled inference ranking: active set without labels, stable argsort of
    -p (network.py:383-391)."""
    tr = slot_forward(st, lsh, x_idx, x_val, None, rng, n_out)
    return tr.active[np.argsort(-tr.probs, kind="stable")]


def precision_at_k(ranked, truth, k: int) -> float:
    """|top-k ∩ truth| / k (data.py:126-133)."""
    top = list(ranked[:k])
    if not top:
        return 0.0
    truth = set(truth)
    return sum(1 for r in top if r in truth) / k
