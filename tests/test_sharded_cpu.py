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

D, H, N, B, SEED = 40, 12, 61, 6, 3
LR = 1e-2


def _spec(family):
    if family == "simhash":
        return O.LshSpec("simhash", 3, 5, 6, "fifo", strategy="vanilla", beta=9)
    return O.LshSpec("dwta", 2, 5, 4, "reservoir", bin_size=4, strategy="vanilla", beta=7)


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
    """Rank g's share of the step, computed by the oracle's primitives."""

    def __init__(self, full: O.NetState, spec, g, G):
        self.g, self.G = g, G
        rows = np.arange(g, N, G)
        self.rows = rows
        self.st = O.NetState(
            full.w1t.copy(), full.b1.copy(), full.m1t.copy(), full.v1t.copy(), full.mb1.copy(), full.vb1.copy(),
            full.steps1.copy(), full.w2[rows].copy(), full.b2[rows].copy(), full.m2[rows].copy(),
            full.v2[rows].copy(), full.mb2[rows].copy(), full.vb2[rows].copy(), full.steps2[rows].copy())
        self.lsh = O.OutputLsh(spec, H, SEED, n0=2, lam=0.0)
        self.rebuild()

    def rebuild(self):
        local = torch.from_numpy(O.family_keys(self.lsh.params, self.st.w2).astype(np.int64))
        keys = sharded.all_gather_rows(local, N).numpy()
        self.lsh.buckets = O.build_buckets(keys, self.lsh.spec.cap, self.lsh.spec.policy, self.lsh.pyrand)

    def forward(self, csr, it):
        self.slots = []
        mx = np.full(csr.batch, -np.inf)
        for i in range(csr.batch):
            a, b = csr.x_ptr[i], csr.x_ptr[i + 1]
            xi, xv = csr.x_idx[a:b].astype(np.int64), csr.x_val[a:b].astype(np.float64)
            y = csr.y_idx[csr.y_ptr[i]:csr.y_ptr[i + 1]].astype(np.int64)
            rng = np.random.default_rng((SEED, it, i))
            h = np.maximum((xv @ self.st.w1t[xi] if xi.size else 0.0) + self.st.b1, 0.0)
            _, per_table = self.lsh.query(h)
            ids = O.sampled_ids(per_table, "vanilla", self.lsh.spec.beta, 1, rng)
            if ids.size == 0:
                ids = rng.choice(N, size=min(self.lsh.spec.beta, N), replace=False)
            act = np.union1d(ids, y)
            own = act[act % self.G == self.g]
            loc = own // self.G
            nz = np.flatnonzero(h > 0)
            z = (self.st.w2[np.ix_(loc, nz)] @ h[nz] if nz.size else 0.0) + self.st.b2[loc]
            z = np.asarray(z, dtype=np.float64) * np.ones(loc.size)
            self.slots.append(dict(xi=xi, xv=xv, y=y, h=h, act_n=act.size, loc=loc, own=own, z=z))
            if z.size:
                mx[i] = z.max()
        return torch.from_numpy(mx)

    def softmax_sum(self, gmax):
        return torch.tensor([np.exp(s["z"] - gmax[i].item()).sum() for i, s in enumerate(self.slots)])

    def softmax_finish(self, gmax, gsum):
        out = []
        for i, s in enumerate(self.slots):
            m, se = gmax[i].item(), gsum[i].item()
            p = np.exp(s["z"] - m) / se
            is_lab = np.isin(s["own"], s["y"])
            s["delta"] = p - is_lab / s["y"].size
            zl = s["z"][is_lab] - m - np.log(se)
            out.append(float(np.minimum(-zl, 690.7755278982137).sum()))
        return torch.tensor(out, dtype=torch.float64)

    def hidden_grad(self):
        dh = np.zeros((len(self.slots), H))
        for i, s in enumerate(self.slots):
            if s["loc"].size:
                dh[i] = s["delta"] @ self.st.w2[s["loc"]]
        return torch.from_numpy(dh)

    def update(self, dh):
        dh = dh.numpy()
        for i, s in enumerate(self.slots):
            nz = np.flatnonzero(s["h"] > 0)
            g = O.SlotGrads(s["loc"], s["delta"], nz, s["h"][nz], dh[i][nz] if nz.size else None, s["xi"], s["xv"])
            O.apply_slot_update(self.st, g, O.AdamCfg(lr=LR))

    def active_counts(self):
        return np.array([s["act_n"] for s in self.slots])


def _worker(rank, world, port, family, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = O.init_state(D, H, N, seed=SEED)
        be = NumpyShardBackend(full, _spec(family), rank, world)
        losses = []
        for it, trip in enumerate(_batches(3), start=1):
            loss, active = sharded.sharded_step(be, _csr(trip), it, None)
            losses.append(float(np.mean(loss)))
            if be.lsh.schedule.due(it):  # the rebuild barrier (network.py:368-373)
                be.rebuild()
                be.lsh.schedule.advance()
        w2 = sharded.all_gather_rows(torch.from_numpy(be.st.w2), N).numpy()
        steps2 = sharded.all_gather_rows(torch.from_numpy(be.st.steps2[:, None]), N).numpy()[:, 0]
        out_q.put((rank, losses, be.st.w1t, be.st.b1, be.st.steps1, w2, steps2, list(active)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("family", ["simhash", "dwta"])
def test_sharded_step_equals_single_process(family):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, family, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle, snapshot schedule
    st = O.init_state(D, H, N, seed=SEED)
    lsh = O.OutputLsh(_spec(family), H, SEED, n0=2, lam=0.0)
    lsh.build(st.w2)
    want = []
    for it, trip in enumerate(_batches(3), start=1):
        r = O.train_step(st, lsh, trip, it, SEED, N, O.AdamCfg(lr=LR), mode="snapshot")
        want.append(float(np.mean(r.losses)))
        last_active = [tr.active.size for tr in r.traces]
    for rank, losses, w1t, b1, steps1, w2, steps2, active in res:
        np.testing.assert_allclose(losses, want, rtol=1e-12)
        np.testing.assert_allclose(w1t, st.w1t, rtol=0, atol=1e-12)
        np.testing.assert_allclose(b1, st.b1, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(steps1, st.steps1)
        np.testing.assert_allclose(w2, st.w2, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(steps2, st.steps2)
        assert active == last_active


def test_interleave_layout():
    parts = [torch.arange(4).reshape(4, 1) * 3, torch.arange(4).reshape(4, 1) * 3 + 1,
             torch.arange(4).reshape(4, 1) * 3 + 2]
    out = sharded.interleave(parts, 10)
    np.testing.assert_array_equal(out[:, 0].numpy(), np.arange(10))
