"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by the reference package ``slide`` 0.1.0 itself
(or, for the random streams, by the numpy / CPython generators the reference
calls), so the oracle and the device path are pinned to the reference's own
outputs.  Fixtures are small .npz files; nothing at run time reads
/root/reference.
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import slide  # noqa: E402  (the reference)
from slide.hashing import HashFamilyConfig, new_hash_family  # noqa: E402
from slide.network import LshLayerConfig, SlideNetwork, TrainConfig, _adam_block  # noqa: E402
from slide.samplers import SamplerConfig, sample  # noqa: E402
from slide.sparse import SparseVector  # noqa: E402
from slide.tables import LshTables, RawCandidates  # noqa: E402

from paper_1903_03129_b200.configs import TINY  # noqa: E402
from paper_1903_03129_b200.data import synthetic_corpus  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sum(np.asarray(a).nbytes for a in arrays.values()), "bytes raw")


# ---------------------------------------------------------------- rng streams
def rng_streams():
    ents = [(0, 1, 0), (0, 1, 127), (0, 50, 3), (7, 123, 255), (123456789, 9, 1), (2**33 + 5, 2, 0)]
    perms = {}
    for L in (20, 50, 64):
        perms[L] = np.stack([np.random.default_rng(e).permutation(L) for e in ents])
    choices = []
    cases = [(5000, 250), (670091, 128), (30, 4), (12, 12), (20000, 401), (205443, 10272), (10001, 5000)]
    rows = []
    for e in ents[:3]:
        for pop, size in cases:
            for pre_perm in (0, 50):
                r = np.random.default_rng(e)
                if pre_perm:
                    r.permutation(pre_perm)
                c = r.choice(pop, size=size, replace=False)
                rows.append((e[0], e[1], e[2], pop, size, pre_perm))
                choices.append(c.astype(np.int64))
    lens = np.array([c.size for c in choices])
    save("rng_streams.npz", ents=np.array(ents, dtype=np.uint64), perm20=perms[20], perm50=perms[50],
         perm64=perms[64], choice_cases=np.array(rows, dtype=np.int64), choice_lens=lens,
         choice_vals=np.concatenate(choices))


# -------------------------------------------------------------- python random
def mt19937():
    seeds = [104729 * 2, 0, 5 + 104729 * 2, 2**40 + 3]
    states, draws = [], []
    for s in seeds:
        r = random.Random(s)
        st = r.getstate()[1]
        states.append(np.array(st, dtype=np.uint64))
        draws.append(np.array([r.random() for _ in range(2000)]))
    save("mt19937.npz", seeds=np.array(seeds, dtype=np.uint64), states=np.stack(states), draws=np.stack(draws))


# ------------------------------------------------------------------- hashing
def hashing():
    rng = np.random.default_rng(11)
    out = {}
    specs = {
        "sh_main": dict(family="simhash", k_per_table=9, num_tables=50, dim=128, seed=7919 * 2),
        "sh_small": dict(family="simhash", k_per_table=2, num_tables=4, dim=24, seed=5),
        "sh_full": dict(family="simhash", k_per_table=4, num_tables=2, dim=6, simhash_sparsity=1.0, seed=11),
        "dw_main": dict(family="dwta", k_per_table=8, num_tables=50, dim=128, wta_bin_size=8, seed=7919 * 2),
        "dw_small": dict(family="dwta", k_per_table=2, num_tables=1, dim=9, wta_bin_size=3, seed=5),
        "dw_ragged": dict(family="dwta", k_per_table=2, num_tables=3, dim=10, wta_bin_size=4, seed=1),
        "dw_scaled": dict(family="dwta", k_per_table=8, num_tables=64, dim=256, wta_bin_size=8, seed=7919 * 2),
    }
    for name, kw in specs.items():
        fam = new_hash_family(HashFamilyConfig(**kw))
        d = kw["dim"]
        # queries: relu-like sparse vectors (about half zeros), a zero vector,
        # a single-entry vector, f32-representable values
        q = rng.standard_normal((40, d)).astype(np.float32).astype(np.float64)
        q = np.maximum(q, 0.0)
        q[0] = 0.0
        q[1] = 0.0
        q[1, d // 2] = 1.5
        q[2] = np.abs(q[2]) + 0.25  # fully dense positive
        qk = np.stack([fam.hash(SparseVector.from_dense(v)) for v in q])
        # rows: dense f32-representable weights, some exact zeros
        w = (rng.standard_normal((64, d)) * 0.01).astype(np.float32).astype(np.float64)
        w[3, :5] = 0.0
        wk = fam.hash_batch(w)
        out[name + "_q"] = q
        out[name + "_qkeys"] = qk
        out[name + "_w"] = w
        out[name + "_wkeys"] = wk
        if kw["family"] == "simhash":
            out[name + "_idx"] = fam.proj_indices
            out[name + "_signs"] = fam.proj_signs
        else:
            out[name + "_perms"] = fam.perms
            out[name + "_salt"] = np.array([fam._densify_salt], dtype=np.uint64)
    save("hashing.npz", **out)


# -------------------------------------------------------------------- tables
def flatten_tables(tables):
    t_, k_, cnt_, ptr, slots = [], [], [], [0], []
    for t, tbl in enumerate(tables.tables):
        for key in sorted(tbl):
            b = tbl[key]
            t_.append(t)
            k_.append(key)
            cnt_.append(b.count)
            slots.extend(b.slots)
            ptr.append(len(slots))
    return dict(t=np.array(t_), key=np.array(k_, dtype=np.int64), count=np.array(cnt_),
                ptr=np.array(ptr), slots=np.array(slots, dtype=np.int64))


def tables():
    out = {}
    rng = np.random.default_rng(3)
    # heavy collisions: K=2 simhash, 300 rows, cap 16 -> overflow in every table
    for policy in ("fifo", "reservoir"):
        fam = new_hash_family(HashFamilyConfig("simhash", 2, 5, 24, seed=5))
        tbl = LshTables(fam, policy=policy, capacity=16, seed=104729 * 2)
        w = rng.standard_normal((300, 24)).astype(np.float32).astype(np.float64)
        tbl.build(w)
        first = flatten_tables(tbl)
        tbl.build(w[::-1].copy())  # second build continues the reservoir stream
        second = flatten_tables(tbl)
        out[policy + "_w"] = w
        for k, v in first.items():
            out[f"{policy}_b1_{k}"] = v
        for k, v in second.items():
            out[f"{policy}_b2_{k}"] = v
    # dwta reservoir without overflow
    fam = new_hash_family(HashFamilyConfig("dwta", 8, 10, 128, wta_bin_size=8, seed=9))
    tbl = LshTables(fam, policy="reservoir", capacity=128, seed=1)
    w = (rng.standard_normal((2000, 128)) * 0.01).astype(np.float32).astype(np.float64)
    tbl.build(w)
    out["dwta_w"] = w
    for k, v in flatten_tables(tbl).items():
        out["dwta_" + k] = v
    save("tables.npz", **out)


# ------------------------------------------------------------------ samplers
def samplers():
    rng = np.random.default_rng(21)
    cases = []
    res = []
    for case in range(60):
        L = int(rng.integers(1, 12))
        width = 200
        per_table = []
        for _ in range(L):
            n = int(rng.integers(0, 20)) if rng.random() > 0.2 else 0
            per_table.append(np.sort(rng.choice(width, size=n, replace=False)).tolist())
        strat = ["vanilla", "topk", "hard_threshold"][case % 3]
        beta = int(rng.integers(1, 60))
        mf = int(rng.integers(1, L + 1))
        cfg = SamplerConfig(strategy=strat, beta=beta, min_freq=mf)
        seed = (case, 1, 2)
        rep = sample(RawCandidates(per_table, width), cfg, np.random.default_rng(seed))
        cases.append((case % 3, beta, mf, L))
        res.append(np.sort(rep.active_ids))
        for t in range(L):
            out_key = f"c{case}_t{t}"
            SAMP[out_key] = np.array(per_table[t], dtype=np.int64)
    SAMP["cases"] = np.array(cases)
    SAMP["lens"] = np.array([r.size for r in res])
    SAMP["ids"] = np.concatenate(res).astype(np.int64)
    save("samplers.npz", **SAMP)


SAMP: dict = {}


# ------------------------------------------------------------------- network
def batch_from(rng, n, dim, n_labels, empty_x_slot=None):
    batch = []
    for i in range(n):
        nnz = int(rng.integers(1, min(dim, 12) + 1))
        idx = np.sort(rng.choice(dim, size=nnz, replace=False))
        vals = np.abs(rng.standard_normal(nnz)).astype(np.float32).astype(np.float64) + 0.125
        if i == empty_x_slot:
            idx, vals = idx[:0], vals[:0]
        labels = set(rng.choice(n_labels, size=int(rng.integers(1, 4)), replace=False).tolist())
        batch.append((SparseVector(idx, vals, dim), labels))
    return batch


def to_f32(net):
    for layer in net.layers:
        for name in ("w", "b", "adam_m", "adam_v", "adam_mb", "adam_vb"):
            setattr(layer, name, getattr(layer, name).astype(np.float32).astype(np.float64))


def dump_net(prefix, net, out):
    for li, layer in enumerate(net.layers):
        for name in ("w", "b", "adam_m", "adam_v", "adam_mb", "adam_vb", "steps"):
            out[f"{prefix}_l{li}_{name}"] = getattr(layer, name).copy()


def record_forward(net, log):
    orig = net.forward

    def fwd(x, slot, labels=None, rng=None, forced_active=None):
        tr = orig(x, slot, labels, rng, forced_active)
        log.append((slot, tr.active[-1].copy(), tr.probs.copy()))
        return tr

    net.forward = fwd


def snapshot_step(net, batch, it):
    """SURVEY 8(c) snapshot-HOGWILD oracle from reference functions."""
    caps = []
    losses = []
    for i, (x, labels) in enumerate(batch):
        rng = np.random.default_rng((net.cfg.seed, it, i))
        tr = net.forward(x, i, labels, rng)
        losses.append(tr.loss(labels))
        cap = []
        net.backward(tr, labels, i, update=False, capture=cap)
        caps.append(cap)
    for cap in caps:
        for li, rows, cols, grad, delta in cap:
            _adam_block(net.layers[li], rows, cols, grad, delta, net.cfg)
    for li, layer in enumerate(net.layers):
        if layer.lsh is not None:
            layer.lsh.mark_weights_changed()
            layer.lsh.maybe_rebuild(it, layer.w)
    return float(np.mean(losses))


def network():
    out = {}
    setups = {
        # D, H, N, lsh, B, n0
        "sh": (50, 16, 40, LshLayerConfig("simhash", k=3, l=6, capacity=8, sampler=SamplerConfig("vanilla", beta=10)), 6, 2),
        "shtopk": (50, 16, 40, LshLayerConfig("simhash", k=3, l=6, capacity=8, sampler=SamplerConfig("topk", beta=7)), 6, 2),
        "dw": (40, 12, 60, LshLayerConfig("dwta", k=2, l=5, capacity=4, policy="reservoir", wta_bin_size=4,
                                           sampler=SamplerConfig("vanilla", beta=6)), 5, 2),
        "dwth": (40, 12, 60, LshLayerConfig("dwta", k=2, l=5, capacity=4, policy="reservoir", wta_bin_size=4,
                                             sampler=SamplerConfig("hard_threshold", beta=6, min_freq=2)), 5, 2),
        "dense": (20, 8, 12, None, 4, 50),
    }
    for name, (D, H, N, lsh, B, n0) in setups.items():
        for mode in ("seq", "snap"):
            cfg = TrainConfig(batch_size=B, seed=3, learning_rate=1e-2, n0=n0)
            net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: lsh} if lsh else None)
            if mode == "seq":
                dump_net(f"{name}_init", net, out)
            rng = np.random.default_rng(99)
            for it in range(1, 4):
                batch = batch_from(rng, B, D, N, empty_x_slot=1 if it == 2 else None)
                log = []
                if mode == "seq":
                    orig = net.forward
                    record_forward(net, log)
                    stats = net.train_batch(batch, it)
                    net.forward = orig
                    loss = stats.loss
                else:
                    orig = net.forward
                    record_forward(net, log)
                    loss = snapshot_step(net, batch, it)
                    net.forward = orig
                out[f"{name}_{mode}_it{it}_loss"] = np.array([loss])
                for i, (x, labels) in enumerate(batch):
                    out[f"{name}_it{it}_x{i}_idx"] = x.indices
                    out[f"{name}_it{it}_x{i}_val"] = x.values
                    out[f"{name}_it{it}_y{i}"] = np.array(sorted(labels))
                for slot, act, probs in log:
                    out[f"{name}_{mode}_it{it}_active{slot}"] = act
                    out[f"{name}_{mode}_it{it}_probs{slot}"] = probs
                dump_net(f"{name}_{mode}_it{it}", net, out)
    save("network.npz", **out)


def tiny_config():
    """The BASELINE tiny config (configs[0]) on the SURVEY 8(d) corpus: two
    sequential reference steps; checksums + slices of the state."""
    w = TINY
    corpus = synthetic_corpus(w.corpus, 2 * w.batch, seed=0)
    cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr, n0=w.n0)
    lsh = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
    net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: lsh})
    out = {}
    out["init_w2_head"] = net.layers[1].w[:8].copy()
    out["init_w1_head"] = net.layers[0].w[:, :8].copy()
    for it in (1, 2):
        rows = np.arange((it - 1) * w.batch, it * w.batch)
        batch = [corpus.example(int(r)) for r in rows]
        log = []
        orig = net.forward
        record_forward(net, log)
        stats = net.train_batch(batch, it)
        net.forward = orig
        out[f"it{it}_loss"] = np.array([stats.loss])
        out[f"it{it}_frac"] = np.array([stats.active_fraction[1]])
        out[f"it{it}_active_sizes"] = np.array([a.size for _, a, _ in log])
        out[f"it{it}_active_sum"] = np.array([int(a.sum()) for _, a, _ in log])
        for li, layer in enumerate(net.layers):
            out[f"it{it}_l{li}_wsum"] = np.array([layer.w.sum(), np.abs(layer.w).sum()])
            out[f"it{it}_l{li}_msum"] = np.array([layer.adam_m.sum(), np.abs(layer.adam_m).sum()])
            out[f"it{it}_l{li}_bsum"] = np.array([layer.b.sum(), np.abs(layer.b).sum()])
            out[f"it{it}_l{li}_steps"] = layer.steps.copy()
    out["final_w2_head"] = net.layers[1].w[:64].copy()
    save("tiny_config.npz", **out)


def tiny_run():
    """The BASELINE tiny config (configs[0]) end to end: 200 steps of the
    reference's ``train_network`` (workers=1, the sequential schedule; epoch
    order ``default_rng((seed, 0))``) over 200 x 128 synthetic examples, per-step
    losses / active fractions / rebuild flags, then P@1 on a held-out stream
    from the same generator with the evaluator's shared ``default_rng(seed)``
    (reference estimator.py:203-223).  The same 200 batches are also run
    through the snapshot schedule built from reference functions
    (``snapshot_step``) for the snapshot-vs-sequential P@1 report."""
    from slide.data import Dataset, precision_at_k
    from slide.network import train_network

    w = TINY
    n_train, n_eval = 200 * w.batch, 4000
    corpus = synthetic_corpus(w.corpus, n_train, seed=0)
    held = synthetic_corpus(w.corpus, n_eval, seed=1)
    train = [corpus.example(i) for i in range(n_train)]
    evals = [held.example(i) for i in range(n_eval)]
    out = {"corpus_check": np.array([corpus.x_idx.astype(np.int64).sum(), corpus.y_idx.astype(np.int64).sum(),
                                     held.x_idx.astype(np.int64).sum(), held.y_idx.astype(np.int64).sum()]),
           "corpus_vsum": np.array([corpus.x_val.astype(np.float64).sum(), held.x_val.astype(np.float64).sum()])}

    def make():
        cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr, n0=w.n0, decay=w.decay)
        lsh = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
        return SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: lsh})

    def p_at_1(net):
        rng = np.random.default_rng(0)
        return float(np.mean([precision_at_k(net.predict(x, rng=rng)[:1], y, 1) for x, y in evals]))

    # sequential: the reference's own train_network
    net = make()
    log = []
    train_network(net, Dataset(train, w.input_dim, w.n_out),
                  on_batch=lambda it, st: log.append((st.loss, st.active_fraction[1], bool(st.rebuilt))))
    assert len(log) == 200
    out["seq_loss"] = np.array([r[0] for r in log])
    out["seq_frac"] = np.array([r[1] for r in log])
    out["seq_rebuilt"] = np.array([r[2] for r in log])
    out["seq_p1"] = np.array([p_at_1(net)])
    out["seq_final_w2_head"] = net.layers[1].w[:16].copy()
    print("sequential P@1", out["seq_p1"])
    # snapshot schedule over the same batches in the same order
    net = make()
    order = np.random.default_rng((0, 0)).permutation(n_train)
    losses = []
    for it in range(1, 201):
        batch = [train[i] for i in order[(it - 1) * w.batch : it * w.batch]]
        losses.append(snapshot_step(net, batch, it))
    out["snap_loss"] = np.array(losses)
    out["snap_p1"] = np.array([p_at_1(net)])
    print("snapshot P@1", out["snap_p1"])
    save("tiny_run.npz", **out)


def _round_f32(net):
    """The device's starting point: the reference's init rounded to fp32."""
    for layer in net.layers:
        for a in (layer.w, layer.b):
            a[...] = a.astype(np.float32).astype(np.float64)


def _p1_runs(corpus, evals, n_steps, rounded, noise=0.0, noise_seed=0):
    """Reference sequential (train_network, workers=1) and snapshot runs over
    the same batches; P@1 on ``evals`` with the evaluator's shared rng."""
    from slide.data import Dataset, precision_at_k
    from slide.network import train_network

    w = TINY
    n_train = n_steps * w.batch
    train = [corpus.example(i) for i in range(n_train)]

    def make():
        cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr, n0=w.n0, decay=w.decay)
        lsh = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
        net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: lsh})
        if rounded:
            _round_f32(net)
            net.layers[1].lsh.build(net.layers[1].w)
        return net

    def p_at_1(net):
        rng = np.random.default_rng(0)
        return float(np.mean([precision_at_k(net.predict(x, rng=rng)[:1], y, 1) for x, y in evals]))

    nrng = np.random.default_rng(noise_seed)

    def jitter(net):
        if noise:
            for layer in net.layers:
                layer.w *= 1 + noise * nrng.standard_normal(layer.w.shape)

    net = make()
    seq = []

    def on_seq(it, st):
        seq.append(st.loss)
        jitter(net)

    train_network(net, Dataset(train, w.input_dim, w.n_out), on_batch=on_seq)
    seq_p1 = p_at_1(net)
    net = make()
    order = np.random.default_rng((0, 0)).permutation(n_train)
    snap = []
    for it in range(1, n_steps + 1):
        snap.append(snapshot_step(net, [train[i] for i in order[(it - 1) * w.batch : it * w.batch]], it))
        jitter(net)
    return np.array(seq), seq_p1, np.array(snap), p_at_1(net)


def p1_runs():
    """P@1-after-N-steps evidence (north_star: within 1 point of the
    reference).  (1) The rounding spread on the BASELINE tiny corpus: the
    reference's own 200-step runs restarted from its fp32-rounded init, next
    to tiny_run.npz's f64-init runs -- the labels there are independent of
    the features, so P@1 moves by points under rounding alone.  (2) A
    learnable corpus (tests/learnable_corpus.py) at the tiny shape, where
    P@1 measures the training algorithm: reference sequential and snapshot
    runs from the f64 init and from the fp32-rounded one.  (3) Rounding-noise
    ensembles: the reference re-run with every weight multiplied by
    (1 + 3e-8 N(0,1)) after every step (fp32 half-ulp noise, four seeds) --
    the spread a correct fp32 implementation can land in."""
    from tests.learnable_corpus import learnable_corpus

    w = TINY
    out = {}
    corpus = synthetic_corpus(w.corpus, 200 * w.batch, seed=0)
    held = synthetic_corpus(w.corpus, 4000, seed=1)
    evals = [held.example(i) for i in range(len(held))]
    _, out["tiny_seq_p1_f32init"], _, out["tiny_snap_p1_f32init"] = _p1_runs(corpus, evals, 200, True)
    lc = learnable_corpus(w.input_dim, w.n_out, 200 * w.batch, seed=0)
    lh = learnable_corpus(w.input_dim, w.n_out, 4000, seed=1)
    levals = [lh.example(i) for i in range(len(lh))]
    for rounded in (False, True):
        tag = "_f32init" if rounded else ""
        sl, sp, nl, np1 = _p1_runs(lc, levals, 200, rounded)
        out["learn_seq_loss" + tag], out["learn_seq_p1" + tag] = sl, np.array([sp])
        out["learn_snap_loss" + tag], out["learn_snap_p1" + tag] = nl, np.array([np1])
    for tag, (cor, ev) in (("tiny", (corpus, evals)), ("learn", (lc, levals))):
        ens = [_p1_runs(cor, ev, 200, True, noise=3e-8, noise_seed=s) for s in range(4)]
        out[f"{tag}_seq_p1_noise"] = np.array([e[1] for e in ens])
        out[f"{tag}_snap_p1_noise"] = np.array([e[3] for e in ens])
    out["tiny_seq_p1_f32init"] = np.array([out["tiny_seq_p1_f32init"]])
    out["tiny_snap_p1_f32init"] = np.array([out["tiny_snap_p1_f32init"]])
    out["learn_check"] = np.array([lc.x_idx.astype(np.int64).sum(), lc.y_idx.astype(np.int64).sum(),
                                   lh.x_idx.astype(np.int64).sum(), lh.y_idx.astype(np.int64).sum()])
    print({k: v for k, v in out.items() if "p1" in k})
    save("p1_runs.npz", **out)


def p1_seeds():
    """The P@1 criterion as a distribution: on the learnable corpus (tiny
    shape, 200 steps) a single run's P@1 swings by tens of points between
    consecutive checkpoints (per-sample Adam at lr 1e-3), so the reference is
    run for seeds 0..3 in both schedules and P@1 (2,000 held-out examples,
    evaluator rng default_rng(0)) recorded after steps 150, 175 and 200."""
    from slide.data import Dataset, precision_at_k
    from slide.network import train_network

    from tests.learnable_corpus import learnable_corpus

    w = TINY
    n_train = 200 * w.batch
    lc = learnable_corpus(w.input_dim, w.n_out, n_train, seed=0)
    lh = learnable_corpus(w.input_dim, w.n_out, 2000, seed=1)
    train = [lc.example(i) for i in range(n_train)]
    evals = [lh.example(i) for i in range(len(lh))]
    marks = (150, 175, 200)

    def p_at_1(net):
        rng = np.random.default_rng(0)
        return float(np.mean([precision_at_k(net.predict(x, rng=rng)[:1], y, 1) for x, y in evals]))

    out = {"marks": np.array(marks)}
    for seed in range(4):
        def make():
            cfg = TrainConfig(batch_size=w.batch, seed=seed, learning_rate=w.lr, n0=w.n0, decay=w.decay)
            lsh = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap,
                                 sampler=SamplerConfig("vanilla", beta=w.beta))
            return SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: lsh})

        net = make()
        got = []
        train_network(net, Dataset(train, w.input_dim, w.n_out),
                      on_batch=lambda it, st: got.append(p_at_1(net)) if it in marks else None)
        out[f"seq_seed{seed}"] = np.array(got)
        net = make()
        order = np.random.default_rng((seed, 0)).permutation(n_train)
        got = []
        for it in range(1, 201):
            snapshot_step(net, [train[i] for i in order[(it - 1) * w.batch : it * w.batch]], it)
            if it in marks:
                got.append(p_at_1(net))
        out[f"snap_seed{seed}"] = np.array(got)
        print(seed, out[f"seq_seed{seed}"], out[f"snap_seed{seed}"], flush=True)
    save("p1_seeds.npz", **out)


from tests.golden.make_golden_data import XC_BAD, XC_GOOD  # noqa: E402


def data_io():
    """The reference's XC corpus parser on a file exercising CRLF, empty
    label lists, missing feature tails, explicit zeros and trailing blank
    lines, its writer on the result, and its error message for each
    malformed file (reference data.py:51-115)."""
    import tempfile

    from slide.data import DatasetFormatError, load_xc_file, save_xc_file

    out = {}
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "good.txt")
        with open(path, "w", newline="") as fh:
            fh.write(XC_GOOD)
        ds = load_xc_file(path)
        out["good_header"] = np.array([len(ds.examples), ds.num_features, ds.num_labels])
        for i, (x, labels) in enumerate(ds.examples):
            out[f"good_{i}_idx"] = x.indices
            out[f"good_{i}_val"] = x.values
            out[f"good_{i}_labels"] = np.array(sorted(labels), dtype=np.int64)
        save_xc_file(ds, os.path.join(d, "saved.txt"))
        out["saved_text"] = np.frombuffer(open(os.path.join(d, "saved.txt"), "rb").read(), dtype=np.uint8)
        for name, text in XC_BAD.items():
            bp = os.path.join(d, name + ".txt")
            with open(bp, "w", newline="") as fh:
                fh.write(text)
            try:
                load_xc_file(bp)
                msg = "<no error>"
            except DatasetFormatError as e:
                msg = str(e)
            out["bad_" + name] = np.array(msg)
    save("data_io.npz", **out)


def checkpoint():
    """SLDE v1 bytes written by the reference's save_checkpoint (with and
    without Adam state) for a small LSH net after two sequential steps whose
    state was rounded to float32 (reference network.py:478-499)."""
    import tempfile

    from slide.network import save_checkpoint

    cfg = TrainConfig(batch_size=6, seed=3, learning_rate=1e-2, n0=2)
    lsh = LshLayerConfig("simhash", k=3, l=6, capacity=8, sampler=SamplerConfig("vanilla", beta=10))
    net = SlideNetwork(50, [16, 40], cfg, lsh_layers={1: lsh})
    rng = np.random.default_rng(99)
    for it in (1, 2):
        net.train_batch(batch_from(rng, 6, 50, 40), it)
    to_f32(net)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for adam in (True, False):
            path = os.path.join(d, "ck.slde")
            save_checkpoint(net, path, with_adam=adam)
            out["adam" if adam else "plain"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    save("checkpoint.npz", **out)


def cli():
    """The reference CLI's config parsing and config hash (cli.py:99-123) on a
    TOML exercising every section, plus its rejection of unknown keys."""
    import tempfile

    from slide.cli import config_hash, load_config

    from tests.golden.make_golden_data import CLI_TOML

    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "run.toml")
        with open(path, "w") as fh:
            fh.write(CLI_TOML)
        cfg = load_config(path)
    import dataclasses

    from slide.cli import RunConfig

    save("cli.npz", hash=np.array([config_hash(cfg)]), hash_default=np.array([config_hash(RunConfig())]),
         beta=np.array([cfg.beta]), hidden=np.array(cfg.hidden),
         fields=np.array([f.name for f in dataclasses.fields(RunConfig)]))


if __name__ == "__main__":
    assert slide.__version__ == "0.1.0"
    which = sys.argv[1:] or ["rng_streams", "mt19937", "hashing", "tables", "samplers", "network", "tiny_config",
                             "tiny_run", "p1_runs", "p1_seeds", "data_io", "checkpoint", "cli"]
    for name in which:
        globals()[name]()
