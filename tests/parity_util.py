"""Helpers that hand device state to the CPU oracle (test infrastructure).

Tolerance model (north_star: logits / loss 1e-5, weights and Adam state 1e-4
relative, fp32 device against the oracle's fp64 from the same fp32 state):

* every coordinate no update of the step touched must be bit-identical;
* a touched coordinate may differ by ``rtol * |want| + rtol * scale``, where
  ``scale`` is the magnitude of the terms the step summed into it -- for the
  moments the sum over the step's updates of (1 - beta) |g|, with |g| taken
  from term magnitudes (|W2|^T |delta| for the hidden error, which cancels
  because delta sums to ~0; |x| |W1| for a hidden activation) -- and for a
  weight the first-order propagation of those moment floors through
  ``lr * m_hat / (sqrt(v_hat) + eps)``.  That is "1e-4 relative" measured
  against the operands of each sum rather than its cancelled result.
"""

from __future__ import annotations

import ctypes as C
import random

import numpy as np

from oracle import slide_oracle as O


def oracle_state_from_net(net) -> O.NetState:
    """f64 copy of the device's f32 state: 'identical weights' for parity.
    Hidden units in the caller's order (the device keeps them in a physical
    order of its own after a relabel: SlideNetwork.unit_cols)."""
    H, N = net.hidden, net.n_out
    f = lambda t: t.cpu().numpy().astype(np.float64)  # noqa: E731
    cols = np.asarray(net.unit_cols())

    def _host(t, H):
        a = t.cpu().numpy()
        return a[:, cols].astype(np.float64) if a.ndim == 2 else a[cols]

    return O.NetState(
        _host(net.w1t, H), f(net.b1[cols]), _host(net.m1t, H), _host(net.v1t, H), f(net.mb1[cols]), f(net.vb1[cols]),
        net.steps1.cpu().numpy()[cols].astype(np.int64),
        _host(net.w2, H), f(net.b2[:N]), _host(net.m2, H), _host(net.v2, H), f(net.mb2[:N]), f(net.vb2[:N]),
        net.steps2[:N].cpu().numpy().astype(np.int64),
    )


def oracle_spec(spec) -> O.LshSpec:
    return O.LshSpec(spec.family, spec.k, spec.l, spec.capacity, spec.policy, spec.simhash_sparsity,
                     spec.wta_bin_size, spec.sampler.strategy, spec.sampler.beta, spec.sampler.min_freq)


def oracle_lsh_from_net(net, spec, st=None) -> O.OutputLsh:
    """Oracle tables built from the net's (f32) W2 with a fresh reservoir
    stream -- the same inserts and draws the device made at construction."""
    cfg = net.cfg
    lsh = O.OutputLsh(oracle_spec(spec), net.hidden, cfg.seed, cfg.n0, cfg.decay)
    lsh.build((st or oracle_state_from_net(net)).w2)
    return lsh


def device_table_arrays(lsh):
    """The device tables as (table, key, count, kept ids sorted) arrays."""
    from paper_1903_03129_b200 import _lib

    ctx = lsh._context()
    nb, ns, ni = _lib.i64(), _lib.i64(), _lib.i64()
    _lib.call("slide_tables_info", ctx, C.byref(nb), C.byref(ns), C.byref(ni))
    r = nb.value
    skeys = np.empty(max(r, 1), np.uint32)
    counts = np.empty(max(r, 1), np.int32)
    starts = np.empty(max(r, 1), np.int32)
    lens = np.empty(max(r, 1), np.int32)
    ids = np.empty(max(ns.value, 1), np.int32)
    if r:
        _lib.call("slide_tables_export", ctx, skeys.ctypes.data, counts.ctypes.data, starts.ctypes.data,
                  lens.ctypes.data, ids.ctypes.data)
    kb = lsh.family.key_bits
    sk = skeys[:r].astype(np.int64)
    return (sk >> kb, sk & ((1 << kb) - 1), counts[:r].astype(np.int64), starts[:r].astype(np.int64),
            lens[:r].astype(np.int64), ids[: ns.value].astype(np.int64))


def oracle_tables_from_device(lsh) -> list:
    """The device's current tables as oracle BucketTables (teacher forcing:
    the oracle queries exactly what the device queries).  Slot order inside
    a bucket never changes a result (every consumer re-sorts or counts)."""
    t, key, cnt, st, ln, ids = device_table_arrays(lsh)
    out = []
    for q in range(lsh.family.l):
        sel = np.flatnonzero(t == q)
        o = np.argsort(key[sel], kind="stable")
        sel = sel[o]
        ptr = np.zeros(sel.size + 1, np.int64)
        np.cumsum(ln[sel], out=ptr[1:])
        run = np.repeat(np.arange(sel.size), ln[sel])
        slots = ids[st[sel][run] + np.arange(ptr[-1]) - ptr[run]] if ptr[-1] else np.zeros(0, np.int64)
        out.append(O.BucketTable(key[sel], cnt[sel], ptr, slots))
    return out


def assert_tables_equal(lsh, oracle_tables, what=""):
    """Device tables == oracle tables: same (table, key) buckets, insert
    counts and kept id sets, vectorised (full-size tables)."""
    t, key, cnt, st, ln, ids = device_table_arrays(lsh)
    for q, ot in enumerate(oracle_tables):
        sel = np.flatnonzero(t == q)
        o = np.argsort(key[sel], kind="stable")
        sel = sel[o]
        np.testing.assert_array_equal(key[sel], ot.keys, err_msg=f"{what} table {q} keys")
        np.testing.assert_array_equal(cnt[sel], ot.counts, err_msg=f"{what} table {q} counts")
        np.testing.assert_array_equal(ln[sel], np.diff(ot.ptr), err_msg=f"{what} table {q} occupancy")
        run = np.repeat(np.arange(sel.size), ln[sel])
        dev_ids = ids[st[sel][run] + np.arange(run.size) - np.r_[0, np.cumsum(ln[sel])][run]]
        a = np.lexsort((dev_ids, run))
        b = np.lexsort((ot.slots, run))
        np.testing.assert_array_equal(dev_ids[a], ot.slots[b], err_msg=f"{what} table {q} ids")


def copy_random(r: random.Random) -> random.Random:
    c = random.Random()
    c.setstate(r.getstate())
    return c


def _substep(net, bt, s0: int, nb: int, iteration: int, update: bool = True):
    """slide_forward + slide_backward on slots s0..s0+nb of an uploaded batch
    (what slide_train_batch runs per sub-batch); each slot's active set,
    probabilities and loss."""
    from paper_1903_03129_b200 import _lib

    v = _lib.Batch()
    C.pointer(v)[0] = bt
    v.batch = nb
    v.x_ptr = bt.x_ptr + 4 * s0
    v.y_ptr = bt.y_ptr + 4 * s0
    v.x_ptr_host = bt.x_ptr_host + 4 * s0
    v.y_ptr_host = bt.y_ptr_host + 4 * s0
    n = _lib.i64()
    _lib.call("slide_forward", net._ctx, C.byref(v), iteration, s0, C.byref(n))
    offs = net._read(2, nb + 1, np.int32)
    rows = net._read(3, n.value, np.int32).astype(np.int64)
    probs = net._read(5, n.value, np.float32).astype(np.float64)
    loss = net._read(7, nb, np.float64)
    if update:
        _lib.call("slide_backward", net._ctx, 1)
    return [(rows[offs[i]:offs[i + 1]], probs[offs[i]:offs[i + 1]], float(loss[i])) for i in range(nb)]


def device_step_capture(net, csr, iteration: int, schedule: str):
    """One train step through the device stages (slide_forward + slide_backward,
    the kernels slide_train_batch runs), reading each slot's active set,
    probabilities and loss.  ``sequential``: one 1-sample sub-step per slot
    with slot offset i (the rng of slot i); ``snapshot``: one forward of the
    whole batch.  No rebuild barrier (the caller runs it)."""
    lsh = net.layers[1].lsh
    if lsh is not None:
        lsh.sync_to_device()
    bt, keep = net._upload(csr)
    B = csr.batch
    out = []
    subs = [(i, 1) for i in range(B)] if schedule == "sequential" else [(0, B)]
    for s0, nb in subs:
        out += _substep(net, bt, s0, nb, iteration)
    del keep
    return out


def assert_slots_match(got, want, what="", rtol=1e-5):
    """Per slot: active set exact, probabilities and loss 1e-5 relative."""
    assert len(got) == len(want.traces)
    for i, ((rows, probs, loss), tr) in enumerate(zip(got, want.traces)):
        np.testing.assert_array_equal(rows, tr.active, err_msg=f"{what} slot {i} active set")
        np.testing.assert_allclose(probs, tr.probs, rtol=rtol, atol=1e-12, err_msg=f"{what} slot {i} probs")
        assert abs(loss - tr.loss) <= rtol * abs(tr.loss) + 1e-12, (what, i, loss, tr.loss)


class _Scales:
    """Per-coordinate magnitude of the update terms of one step on the rows
    it touched (dense over the row's columns)."""

    def __init__(self, rows, width):
        self.rows = np.asarray(rows, dtype=np.int64)
        self.m = np.zeros((self.rows.size, width))
        self.v = np.zeros((self.rows.size, width))
        self.mb = np.zeros(self.rows.size)
        self.vb = np.zeros(self.rows.size)

    def idx(self, r):
        return np.searchsorted(self.rows, r)

    def add(self, rows, cols, row_scale, col_scale, cfg):
        ri = self.idx(rows)
        self.mb[ri] += (1 - cfg.b1) * row_scale
        self.vb[ri] += (1 - cfg.b2) * 2 * row_scale * row_scale
        if cols is not None and len(cols):
            g = np.outer(row_scale, col_scale)
            ix = np.ix_(ri, np.asarray(cols))
            self.m[ix] += (1 - cfg.b1) * g
            self.v[ix] += (1 - cfg.b2) * 2 * g * g


def step_scales(st_pre: O.NetState, want, cfg: O.AdamCfg):
    """Term magnitudes of one step's updates (see the module docstring)."""
    grads = want.grads
    H = st_pre.w2.shape[1]
    rows2 = np.unique(np.concatenate([g.active for g in grads]))
    s2 = _Scales(rows2, H)
    feats = [g.x_idx for g in grads if g.h_idx.size]
    hid = [g.h_idx for g in grads if g.h_idx.size]
    s1 = _Scales(np.unique(np.concatenate(feats)) if feats else np.zeros(0, np.int64), H)
    sh = _Scales(np.arange(H), 1)  # hidden units: biases / step counters
    for g, tr in zip(grads, want.traces):
        # delta_a = p_a - [a in Y]/|Y|: scale |delta| + p
        p_abs = np.abs(g.delta) + tr.probs
        if g.h_idx.size == 0:
            s2.add(g.active, None, p_abs, None, cfg)
            continue
        xa = np.abs(g.x_val)
        h_abs = xa @ np.abs(st_pre.w1t[np.ix_(g.x_idx, g.h_idx)]) + np.abs(st_pre.b1[g.h_idx]) if g.x_idx.size \
            else np.abs(st_pre.b1[g.h_idx])
        s2.add(g.active, g.h_idx, p_abs, np.maximum(h_abs, g.h_val), cfg)
        dha = g.dh_abs
        sh.mb[g.h_idx] += (1 - cfg.b1) * dha
        sh.vb[g.h_idx] += (1 - cfg.b2) * 2 * dha * dha
        if g.x_idx.size:
            ri = s1.idx(g.x_idx)
            gg = np.outer(xa, dha)
            ix = np.ix_(ri, g.h_idx)
            s1.m[ix] += (1 - cfg.b1) * gg
            s1.v[ix] += (1 - cfg.b2) * 2 * gg * gg
    return s1, s2, sh


def _check_block(name, got, want, pre, floor, rtol, what):
    """Untouched (floor == 0 and unchanged in the oracle): bit-identical;
    touched: rtol * |want| + rtol * floor."""
    fixed = (floor == 0) & (want == pre)
    bad = fixed & (got != want)
    assert not bad.any(), f"{what} {name}: {np.count_nonzero(bad)} untouched coordinates changed"
    tol = rtol * np.abs(want) + rtol * floor
    err = np.abs(got - want)
    ok = err <= tol
    assert ok.all(), (f"{what} {name}: {np.count_nonzero(~ok)} of {ok.size} off, worst err {err[~ok].max():.3g} "
                      f"tol {tol[~ok][np.argmax(err[~ok])]:.3g} want {want[~ok][np.argmax(err[~ok])]:.3g}")
    return float(np.max(err / np.maximum(tol, 1e-300))) if err.size else 0.0


def _weight_floor(m, v, t, mfl, vfl, dt, cfg):
    """First-order propagation of moment floors into the weight (per update
    the move is lr m_hat / (sqrt(v_hat) + eps)); dt updates this step."""
    bc1 = 1.0 - cfg.b1 ** np.maximum(t, 1)
    bc2 = 1.0 - cfg.b2 ** np.maximum(t, 1)
    sv = np.sqrt(np.maximum(v, 0) / bc2)
    den = sv + cfg.eps
    dm = mfl / bc1 / den
    dv = np.abs(m) / bc1 * (vfl / bc2) / (2 * np.maximum(sv, 1e-300) * den * den)
    dv = np.where(sv > 0, dv, 0.0)
    return cfg.lr * dt * (dm + dv)


def assert_step_state_close(net, st: O.NetState, st_pre: O.NetState, want, cfg: O.AdamCfg, rtol=1e-4, what=""):
    """Device state after one step == oracle state after the same step from
    the same f32 state (``st_pre``), under the module's tolerance model.
    Returns the worst err / tol ratio per tensor."""
    dev = oracle_state_from_net(net)
    s1, s2, sh = step_scales(st_pre, want, cfg)
    worst = {}
    np.testing.assert_array_equal(dev.steps1, st.steps1, err_msg=f"{what} steps1")
    np.testing.assert_array_equal(dev.steps2, st.steps2, err_msg=f"{what} steps2")
    # output layer: touched rows dense, everything else bit-identical
    for name, fl in (("m2", s2.m), ("v2", s2.v)):
        got, want, pre = getattr(dev, name), getattr(st, name), getattr(st_pre, name)
        mask = np.ones(got.shape[0], bool)
        mask[s2.rows] = False
        assert np.array_equal(got[mask], want[mask]), f"{what} {name}: untouched rows changed"
        worst[name] = _check_block(name, got[s2.rows], want[s2.rows], pre[s2.rows], fl, rtol, what)
    dt2 = (st.steps2 - st_pre.steps2)[s2.rows].astype(np.float64)
    wfl2 = _weight_floor(st.m2[s2.rows], st.v2[s2.rows], st.steps2[s2.rows][:, None], s2.m, s2.v, dt2[:, None], cfg)
    mask = np.ones(dev.w2.shape[0], bool)
    mask[s2.rows] = False
    assert np.array_equal(dev.w2[mask], st.w2[mask]), f"{what} w2: untouched rows changed"
    worst["w2"] = _check_block("w2", dev.w2[s2.rows], st.w2[s2.rows], st_pre.w2[s2.rows],
                               np.where(s2.m > 0, wfl2, 0.0), rtol, what)
    for name, fl in (("mb2", s2.mb), ("vb2", s2.vb)):
        got, want, pre = getattr(dev, name), getattr(st, name), getattr(st_pre, name)
        f = np.zeros(got.shape)
        f[s2.rows] = fl
        worst[name] = _check_block(name, got, want, pre, f, rtol, what)
    bfl = np.zeros(dev.b2.shape)
    bfl[s2.rows] = _weight_floor(st.mb2[s2.rows], st.vb2[s2.rows], st.steps2[s2.rows], s2.mb, s2.vb, dt2, cfg)
    worst["b2"] = _check_block("b2", dev.b2, st.b2, st_pre.b2, bfl, rtol, what)
    # hidden layer: W1^T rows = input features
    r1 = s1.rows
    for name, fl in (("m1t", s1.m), ("v1t", s1.v)):
        got, want, pre = getattr(dev, name), getattr(st, name), getattr(st_pre, name)
        mask = np.ones(got.shape[0], bool)
        mask[r1] = False
        assert np.array_equal(got[mask], want[mask]), f"{what} {name}: untouched rows changed"
        worst[name] = _check_block(name, got[r1], want[r1], pre[r1], fl, rtol, what)
    dt1 = (st.steps1 - st_pre.steps1).astype(np.float64)[None, :]
    wfl1 = _weight_floor(st.m1t[r1], st.v1t[r1], st.steps1[None, :], s1.m, s1.v, dt1, cfg)
    mask = np.ones(dev.w1t.shape[0], bool)
    mask[r1] = False
    assert np.array_equal(dev.w1t[mask], st.w1t[mask]), f"{what} w1t: untouched rows changed"
    worst["w1t"] = _check_block("w1t", dev.w1t[r1], st.w1t[r1], st_pre.w1t[r1], np.where(s1.m > 0, wfl1, 0.0),
                                rtol, what)
    for name, fl in (("mb1", sh.mb), ("vb1", sh.vb)):
        worst[name] = _check_block(name, getattr(dev, name), getattr(st, name), getattr(st_pre, name), fl, rtol, what)
    dth = (st.steps1 - st_pre.steps1).astype(np.float64)
    worst["b1"] = _check_block("b1", dev.b1, st.b1, st_pre.b1,
                               _weight_floor(st.mb1, st.vb1, st.steps1, sh.mb, sh.vb, dth, cfg), rtol, what)
    return worst


def csr_from_triples(trip):
    from paper_1903_03129_b200.network import HostCsr

    xp = np.r_[0, np.cumsum([len(t[0]) for t in trip])].astype(np.int32)
    yp = np.r_[0, np.cumsum([len(t[2]) for t in trip])].astype(np.int32)
    cat = lambda parts, dt: np.concatenate([np.asarray(p) for p in parts]).astype(dt) if len(parts) else np.zeros(0, dt)  # noqa: E731
    return HostCsr(xp, cat([t[0] for t in trip], np.int32), cat([t[1] for t in trip], np.float32), yp,
                   cat([sorted(t[2]) for t in trip], np.int32))


def forward_capture(net, csr, iteration: int):
    """Forward only (no update): each slot's active set, probabilities, loss."""
    from paper_1903_03129_b200 import _lib

    lsh = net.layers[1].lsh
    if lsh is not None:
        lsh.sync_to_device()
    bt, keep = net._upload(csr)
    n = _lib.i64()
    _lib.call("slide_forward", net._ctx, C.byref(bt), iteration, 0, C.byref(n))
    B = csr.batch
    offs = net._read(2, B + 1, np.int32)
    rows = net._read(3, n.value, np.int32).astype(np.int64)
    probs = net._read(5, n.value, np.float32).astype(np.float64)
    loss = net._read(7, B, np.float64)
    del keep
    return [(rows[offs[i]:offs[i + 1]], probs[offs[i]:offs[i + 1]], float(loss[i])) for i in range(B)]


def teacher_forced_step(net, trip, iteration: int, mode: str, lr: float, what="", rtol=1e-4, per_slot=False):
    """One step of the device from its current state against the oracle
    from the same (f32) state and the device's own tables:

    * active sets exact, probabilities and losses 1e-5 relative per slot;
    * every state tensor under the module's tolerance model;
    * when the rebuild barrier rebuilds, the device tables equal the oracle's
      build from the device's post-step W2 (same reservoir stream).

    ``snapshot`` captures the sets with a forward-only pass and then takes
    the production step (``train_batch_csr``, the CUDA-graph path);
    ``sequential`` drives the per-slot stages slide_train_batch runs; with
    ``per_slot`` every one of its B sub-steps is teacher-forced on its own
    (slot i's forward reads the weights slots < i updated, so from the
    second slot on a whole-step comparison also carries the earlier slots'
    fp32 rounding).
    Returns (oracle StepResult, device BatchStats, worst err/tol per tensor)."""
    cfg = net.cfg
    lsh = net.layers[1].lsh
    acfg = O.AdamCfg(lr=lr, b1=cfg.adam_beta1, b2=cfg.adam_beta2, eps=cfg.adam_eps)
    st_pre = oracle_state_from_net(net)
    st = st_pre.copy()
    olsh = None
    if lsh is not None:
        olsh = O.OutputLsh.__new__(O.OutputLsh)
        olsh.params = oracle_params(lsh.family)
        spec = lsh_spec_of(net)
        olsh.spec = spec
        olsh.schedule = O.Schedule(1 << 40)
        olsh.pyrand = copy_random(lsh._rng)
        olsh.buckets = oracle_tables_from_device(lsh)
    csr = csr_from_triples(trip)
    if per_slot and mode == "sequential":
        return _per_slot_sequential(net, olsh, trip, csr, iteration, acfg, what, rtol)
    want = O.train_step(st, olsh, trip, iteration, cfg.seed, net.n_out, acfg, mode=mode)
    if mode == "snapshot":
        got = forward_capture(net, csr, iteration)
        stats = net.train_batch_csr(csr, iteration, schedule="snapshot")
    else:
        got = device_step_capture(net, csr, iteration, "sequential")
        loss = np.array([g[2] for g in got])
        stats = net._barrier(iteration, loss, np.array([g[0].size for g in got], dtype=np.int64))
    assert_slots_match(got, want, what)
    assert stats.loss == float(np.mean([g[2] for g in got])) or mode == "snapshot"
    assert abs(stats.loss - float(np.mean(want.losses))) <= 1e-5 * abs(float(np.mean(want.losses)))
    worst = assert_step_state_close(net, st, st_pre, want, acfg, rtol=rtol, what=what)
    if stats.rebuilt:
        _check_rebuild(net, lsh, olsh, what)
    return want, stats, worst


def _check_rebuild(net, lsh, olsh, what):
    dev_w2 = oracle_state_from_net(net).w2
    keys = O.family_keys(olsh.params, dev_w2)
    tabs = O.build_bucket_arrays(keys, olsh.spec.cap, olsh.spec.policy, olsh.pyrand)
    assert_tables_equal(lsh, tabs, what=f"{what} rebuild")
    assert lsh._rng.getstate() == olsh.pyrand.getstate()


def _per_slot_sequential(net, olsh, trip, csr, iteration, acfg, what, rtol):
    cfg = net.cfg
    lsh = net.layers[1].lsh
    if lsh is not None:
        lsh.sync_to_device()
    bt, keep = net._upload(csr)
    got_all, traces, grads, losses, worst = [], [], [], [], {}
    for i in range(len(trip)):
        st_pre = oracle_state_from_net(net)
        st = st_pre.copy()
        want = O.train_step(st, olsh, [trip[i]], iteration, cfg.seed, net.n_out, acfg, mode="sequential",
                            slot_offset=i)
        got = _substep(net, bt, i, 1, iteration)
        assert_slots_match(got, want, f"{what} slot {i}")
        w = assert_step_state_close(net, st, st_pre, want, acfg, rtol=rtol, what=f"{what} slot {i}")
        for k, v in w.items():
            worst[k] = max(worst.get(k, 0.0), v)
        got_all += got
        traces += want.traces
        grads += want.grads
        losses += want.losses
    del keep
    loss = np.array([g[2] for g in got_all])
    stats = net._barrier(iteration, loss, np.array([g[0].size for g in got_all], dtype=np.int64))
    if stats.rebuilt:
        _check_rebuild(net, lsh, olsh, what)
    frac = float(np.mean([tr.active.size / net.n_out for tr in traces]))
    return O.StepResult(losses, traces, grads, bool(stats.rebuilt), frac), stats, worst


def oracle_params(family):
    """Oracle hash parameters equal to a device family's (same draws)."""
    from paper_1903_03129_b200.hashing import SimHashFamily

    if isinstance(family, SimHashFamily):
        return O.SimHashParams(family.dim, family.k, family.l, np.asarray(family.proj_indices, np.int64),
                               np.asarray(family.proj_signs, np.float64))
    return O.DwtaParams(family.dim, family.k, family.l, family.bin_size, family.bins_per_perm, family.n_perms,
                        family.bits_per_code, np.asarray(family.perms, np.int64), int(family._densify_salt))


def lsh_spec_of(net) -> O.LshSpec:
    lsh = net.layers[1].lsh
    fam = lsh.family
    sc = net.layers[1].sampler_cfg
    from paper_1903_03129_b200.hashing import SimHashFamily

    name = "simhash" if isinstance(fam, SimHashFamily) else "dwta"
    return O.LshSpec(name, fam.k, fam.l, lsh.capacity, lsh.policy, fam.config.simhash_sparsity,
                     getattr(fam, "bin_size", 8), sc.strategy, sc.beta, sc.min_freq)


def assert_state_close(net, st: O.NetState, rtol=1e-4, atol=1e-6, what="", adam_lr=None):
    """State after several Adam steps (no per-step term record): 1e-4
    relative with an absolute floor, every tensor including the hidden bias
    moments.  Single steps use ``assert_step_state_close``."""
    dev = oracle_state_from_net(net)
    for name in ("w1t", "b1", "m1t", "v1t", "mb1", "vb1", "w2", "b2", "m2", "v2", "mb2", "vb2"):
        got, want = getattr(dev, name), getattr(st, name)
        a = atol if not name.startswith("v") else max(atol * 1e-4, 1e-12)
        if adam_lr is not None and name[0] == "w":
            steps = st.steps1 if name == "w1t" else st.steps2
            moved = rtol * adam_lr * np.asarray(steps, dtype=np.float64)
            a = np.maximum(a, moved[None, :] if name == "w1t" else moved[:, None])
        np.testing.assert_allclose(got, want, rtol=rtol, atol=a, err_msg=f"{what} {name}")
    np.testing.assert_array_equal(dev.steps1, st.steps1, err_msg=f"{what} steps1")
    np.testing.assert_array_equal(dev.steps2, st.steps2, err_msg=f"{what} steps2")
