"""World-size-2 gloo test of the column-sharded step on CPU.

The orchestration that production runs on B200s (``sharded.sharded_step``
and ``sharded.all_gather_rows``: the all-reduces of the softmax max / sum,
the loss terms and the hidden gradient, the all-gather of the table keys) is
driven here with a numpy backend built from the CPU oracle, one process per
rank over gloo.  The sharded result must equal the single-process oracle
step: same losses, same W1 on every rank, and the ranks' W2 rows assembled
back into the single-process W2.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import slide_oracle as O
from paper_1903_03129_b200 import sharded
from paper_1903_03129_b200.network import HostCsr

D, H, N, B, SEED = 40, 16, 61, 6, 3
LR = 1e-2


def _spec(family):
    if family == "simhash":
        return O.LshSpec("simhash", 3, 5, 6, "fifo", strategy="vanilla", beta=9)
    if family == "simhash_ht":
        return O.LshSpec("simhash", 3, 5, 6, "fifo", strategy="hard_threshold", beta=9, min_freq=2)
    if family == "dwta_fifo":
        return O.LshSpec("dwta", 2, 5, 3, "fifo", bin_size=4, strategy="vanilla", beta=7)
    # reservoir: a capacity no bucket reaches over all ranks (the sharded proof)
    return O.LshSpec("dwta", 2, 5, 40, "reservoir", bin_size=4, strategy="vanilla", beta=7)


def _batches(n_steps):
    rng = np.random.default_rng(42)
    out = []
    for _ in range(n_steps):
        trip = []
        for i in range(B):
            idx = np.sort(rng.choice(D, size=int(rng.integers(1, 9)), replace=False))
            val = (np.abs(rng.standard_normal(idx.size)) + 0.1).astype(np.float32).astype(np.float64)
            lab = sorted(rng.choice(N, size=int(rng.integers(1, 4)), replace=False).tolist())
            if i == 2:
                idx, val = idx[:0], val[:0]  # an empty input
            trip.append((idx, val, lab))
        out.append(trip)
    return out


def _csr(trip):
    xp, yp = [0], [0]
    for xi, _, y in trip:
        xp.append(xp[-1] + len(xi))
        yp.append(yp[-1] + len(y))
    cat = lambda a, dt: np.concatenate(a).astype(dt) if a else np.empty(0, dt)
    return HostCsr(np.array(xp, np.int32), cat([t[0] for t in trip], np.int32), cat([t[1] for t in trip], np.float32),
                   np.array(yp, np.int32), cat([np.array(t[2]) for t in trip], np.int32))


class NumpyShardBackend:
    """Rank g's share of the step (SURVEY 8(e) partition), computed by the
    oracle's primitives: W2 rows id % G == g, W1 units [g H/G, (g+1) H/G),
    tables over the rank's own rows (global ids)."""

    def __init__(self, full: O.NetState, spec, g, G):
        self.g, self.G = g, G
        rows = np.arange(g, N, G)
        self.hg = H // G
        u = slice(g * self.hg, (g + 1) * self.hg)
        self.w1s, self.m1s, self.v1s = full.w1t[:, u].copy(), full.m1t[:, u].copy(), full.v1t[:, u].copy()
        self.st = O.NetState(
            None, full.b1.copy(), None, None, full.mb1.copy(), full.vb1.copy(),
            full.steps1.copy(), full.w2[rows].copy(), full.b2[rows].copy(), full.m2[rows].copy(),
            full.v2[rows].copy(), full.mb2[rows].copy(), full.vb2[rows].copy(), full.steps2[rows].copy())
        self.spec = spec
        self.lsh = O.OutputLsh(spec, H, SEED, n0=2, lam=0.0)
        self.capacity, self.policy, self.device = spec.cap, spec.policy, "cpu"
        self.exchanged = 0

    # -- tables over the rank's own rows (global ids r G + g)
    def build_local(self):
        keys = O.family_keys(self.lsh.params, self.st.w2)
        self.tabs = []
        mx = 0
        for t in range(keys.shape[1]):
            tab = {}
            for r in range(keys.shape[0]):  # ascending ids: the insert order
                tab.setdefault(int(keys[r, t]), []).append(r * self.G + self.g)
            out = {}
            for k, ids in tab.items():
                mx = max(mx, len(ids))
                out[k] = (len(ids), np.array(ids[-self.capacity:] if self.policy == "fifo" else ids[: self.capacity]))
            self.tabs.append(out)
        return mx

    def pack(self):
        kb = 30
        ent = sorted(((t << kb) | k, c, ids) for t, tab in enumerate(self.tabs) for k, (c, ids) in tab.items())
        R = len(ent)
        lens = [len(e[2]) for e in ent]
        starts = np.r_[0, np.cumsum(lens)[:-1]] if R else np.zeros(0, np.int64)
        ids = np.concatenate([e[2] for e in ent]) if R else np.zeros(0, np.int64)
        flat = np.r_[R, ids.size, [e[0] for e in ent], [e[1] for e in ent], starts, lens, ids].astype(np.int64)
        return torch.from_numpy(flat)

    def reconcile(self, gathered):
        self.exchanged += 1
        kb = 30
        other = []
        for q, row in enumerate(gathered.numpy()):
            R, S = int(row[0]), int(row[1])
            sk, cnt, st, ln = (row[2 + j * R : 2 + (j + 1) * R] for j in range(4))
            ids = row[2 + 4 * R : 2 + 4 * R + S]
            other.append({int(sk[r]): (int(cnt[r]), ids[st[r] : st[r] + ln[r]]) for r in range(R)})
        for t, tab in enumerate(self.tabs):
            for k, (c, ids) in list(tab.items()):
                got = [o[(t << kb) | k] for o in other if (t << kb) | k in o]
                total = sum(x[0] for x in got)
                if total > self.capacity:
                    top = np.sort(np.concatenate([x[1] for x in got]))[-self.capacity:]
                    ids = ids[ids >= top[0]]
                tab[k] = (total, ids)

    # -- step
    def hidden(self, csr):
        self.csr = csr
        part = np.zeros((csr.batch, self.hg))
        for i in range(csr.batch):
            a, b = csr.x_ptr[i], csr.x_ptr[i + 1]
            xi, xv = csr.x_idx[a:b].astype(np.int64), csr.x_val[a:b].astype(np.float64)
            if xi.size:
                part[i] = xv @ self.w1s[xi]
        return torch.from_numpy(part)

    def assemble(self, parts):
        z = parts.numpy().transpose(1, 0, 2).reshape(self.csr.batch, H)
        self.h = np.maximum(z + self.st.b1, 0.0)

    def select(self, it):
        L = self.lsh.spec.l
        self.slots = []
        hist = np.zeros((self.csr.batch, L + 1), dtype=np.int64)
        for i in range(self.csr.batch):
            rng = np.random.default_rng((SEED, it, i))
            vanilla = self.spec.strategy == "vanilla"
            order = rng.permutation(L) if vanilla else np.arange(L)
            keys = O.family_keys(self.lsh.params, self.h[i][None, :])[0]
            first, freq = {}, {}
            for p, t in enumerate(order.tolist()):
                hit = self.tabs[t].get(int(keys[t]))
                for r in (hit[1].tolist() if hit is not None else []):
                    first.setdefault(r, p)
                    freq[r] = freq.get(r, 0) + 1
            if vanilla:
                for p in first.values():
                    hist[i, p] += 1
                hist[i, L] = len(first)
            else:  # hard_threshold: an id's frequency is its owner rank's
                hist[i, L] = sum(f >= self.spec.min_freq for f in freq.values())
            self.slots.append(dict(rng=rng, first=first, freq=freq))
        return torch.from_numpy(hist)

    def forward(self, it, ghist):
        ghist = ghist.numpy()
        L = self.lsh.spec.l
        beta = self.lsh.spec.beta
        csr = self.csr
        mx = np.full(csr.batch, -np.inf)
        for i in range(csr.batch):
            s = self.slots[i]
            cum = np.cumsum(ghist[i, :L])
            hitp = np.flatnonzero(cum >= beta)
            tau = int(hitp[0]) + 1 if hitp.size else L
            if self.spec.strategy == "vanilla":
                ids = np.array(sorted(r for r, p in s["first"].items() if p < tau), dtype=np.int64)
            else:
                ids = np.array(sorted(r for r, f in s["freq"].items() if f >= self.spec.min_freq), dtype=np.int64)
            if ghist[i, L] == 0:
                ids = s["rng"].choice(N, size=min(beta, N), replace=False)
            a, b = csr.x_ptr[i], csr.x_ptr[i + 1]
            xi, xv = csr.x_idx[a:b].astype(np.int64), csr.x_val[a:b].astype(np.float64)
            y = csr.y_idx[csr.y_ptr[i]:csr.y_ptr[i + 1]].astype(np.int64)
            act = np.union1d(ids, y)
            own = act[act % self.G == self.g]
            loc = own // self.G
            h = self.h[i]
            nz = np.flatnonzero(h > 0)
            z = (self.st.w2[np.ix_(loc, nz)] @ h[nz] if nz.size else 0.0) + self.st.b2[loc]
            z = np.asarray(z, dtype=np.float64) * np.ones(loc.size)
            s.update(xi=xi, xv=xv, y=y, h=h, loc=loc, own=own, z=z)
            if z.size:
                mx[i] = z.max()
        return torch.from_numpy(mx)

    def softmax_sum(self, gmax):
        return torch.tensor([np.exp(s["z"] - gmax[i].item()).sum() for i, s in enumerate(self.slots)])

    def softmax_finish(self, gmax, gsum):
        out, cnt = [], []
        for i, s in enumerate(self.slots):
            m, se = gmax[i].item(), gsum[i].item()
            p = np.exp(s["z"] - m) / se
            is_lab = np.isin(s["own"], s["y"])
            s["delta"] = p - is_lab / s["y"].size
            zl = s["z"][is_lab] - m - np.log(se)
            out.append(float(np.minimum(-zl, 690.7755278982137).sum()))
            cnt.append(float(s["own"].size))
        return torch.tensor(out + cnt, dtype=torch.float64)

    def hidden_grad(self):
        dh = np.zeros((len(self.slots), H))
        for i, s in enumerate(self.slots):
            if s["loc"].size:
                dh[i] = s["delta"] @ self.st.w2[s["loc"]]
        return torch.from_numpy(dh)

    def update(self, dh):
        dh = dh.numpy()
        cfg = O.AdamCfg(lr=LR)
        st = self.st
        u0 = self.g * self.hg
        for i, s in enumerate(self.slots):
            nz = np.flatnonzero(s["h"] > 0)
            grad2 = np.outer(s["delta"], s["h"][nz]) if nz.size else None
            O._adam_rows(st.w2, st.m2, st.v2, st.b2, st.mb2, st.vb2, st.steps2, s["loc"], nz if nz.size else None,
                         grad2, s["delta"], cfg)
            if not nz.size:
                continue
            g = dh[i][nz]
            mine = (nz >= u0) & (nz < u0 + self.hg)
            if s["xi"].size and mine.any():  # this rank's units, at the step counts before the bias update
                _adam_cols(self.w1s, self.m1s, self.v1s, nz[mine] - u0, s["xi"], np.outer(g[mine], s["xv"]),
                           st.steps1[nz[mine]] + 1, cfg)
            O._adam_rows(np.zeros((H, 0)), np.zeros((H, 0)), np.zeros((H, 0)), st.b1, st.mb1, st.vb1, st.steps1,
                         nz, None, None, g, cfg)

    def active_counts(self):
        return np.array([s["own"].size for s in self.slots])


def _adam_cols(w1s, m1s, v1s, rows, cols, grad, t, cfg):
    """_adam_block on W1[rows, cols] with W1 stored transposed by shard
    columns (reference network.py:428-451)."""
    ix = np.ix_(cols, rows)
    bc1 = 1.0 - cfg.b1 ** t
    bc2 = 1.0 - cfg.b2 ** t
    mm = cfg.b1 * m1s[ix] + (1 - cfg.b1) * grad.T
    vv = cfg.b2 * v1s[ix] + (1 - cfg.b2) * grad.T * grad.T
    m1s[ix] = mm
    v1s[ix] = vv
    w1s[ix] -= cfg.lr * (mm / bc1[None, :]) / (np.sqrt(vv / bc2[None, :]) + cfg.eps)


def _worker(rank, world, port, family, n0, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = O.init_state(D, H, N, seed=SEED)
        be = NumpyShardBackend(full, _spec(family), rank, world)
        sharded.rebuild_sharded(be)
        sched = O.Schedule(n0)
        losses, active = [], None
        for it, trip in enumerate(_batches(3), start=1):
            loss, active = sharded.sharded_step(be, _csr(trip), it, None).host()
            losses.append(float(np.mean(loss)))
            if sched.due(it):  # the rebuild barrier (network.py:368-373)
                sharded.rebuild_sharded(be)
                sched.advance()
        w1t = sharded.all_gather_units(torch.from_numpy(be.w1s)).numpy()
        w2 = sharded.all_gather_rows(torch.from_numpy(be.st.w2), N).numpy()
        steps2 = sharded.all_gather_rows(torch.from_numpy(be.st.steps2[:, None]), N).numpy()[:, 0]
        tabs = [{k: (c, ids.tolist()) for k, (c, ids) in tab.items()} for tab in be.tabs]
        out_q.put((rank, losses, w1t, be.st.b1, be.st.steps1, w2, steps2, list(active), tabs, be.exchanged))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("family,world,n0", [("simhash", 2, 2), ("simhash", 4, 2), ("simhash_ht", 2, 1),
                                             ("dwta_fifo", 4, 1), ("dwta", 2, 2), ("dwta", 4, 1)])
def test_sharded_step_equals_single_process(family, world, n0):
    """World 2 and 4: losses, every rank's assembled W1 / W2 / step counters
    and the global active-set sizes equal the single-process oracle step;
    the union of the ranks' tables equals the single-process tables (FIFO
    reconciliation exercised: cap 6 with world 4)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, family, n0, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle, snapshot schedule
    st = O.init_state(D, H, N, seed=SEED)
    lsh = O.OutputLsh(_spec(family), H, SEED, n0=n0, lam=0.0)
    lsh.build(st.w2)
    want = []
    for it, trip in enumerate(_batches(3), start=1):
        r = O.train_step(st, lsh, trip, it, SEED, N, O.AdamCfg(lr=LR), mode="snapshot")
        want.append(float(np.mean(r.losses)))
        last_active = [tr.active.size for tr in r.traces]
    for rank, losses, w1t, b1, steps1, w2, steps2, active, tabs, exchanged in res:
        np.testing.assert_allclose(losses, want, rtol=1e-12)
        np.testing.assert_allclose(w1t, st.w1t, rtol=0, atol=1e-12)
        np.testing.assert_allclose(b1, st.b1, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(steps1, st.steps1)
        np.testing.assert_allclose(w2, st.w2, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(steps2, st.steps2)
        assert active == last_active
    # the ranks' buckets partition the single-process buckets (as sets)
    for t, want_t in enumerate(lsh.buckets):
        want_d = dict(want_t.items())
        keys = set(want_d) | set().union(*(set(r[8][t]) for r in res))
        for k in keys:
            got = sorted(i for r in res for i in r[8][t].get(k, (0, []))[1])
            exp = sorted(int(i) for i in want_d[k][0]) if k in want_d else []
            assert got == exp, (t, k, got, exp)
    if family in ("simhash", "dwta_fifo") and world == 4:
        assert all(r[9] > 0 for r in res)  # the FIFO exchange ran


def test_interleave_layout():
    parts = [torch.arange(4).reshape(4, 1) * 3, torch.arange(4).reshape(4, 1) * 3 + 1,
             torch.arange(4).reshape(4, 1) * 3 + 2]
    out = sharded.interleave(parts, 10)
    np.testing.assert_array_equal(out[:, 0].numpy(), np.arange(10))
