"""Device parity: every stage of the CUDA path against the reference's golden
vectors and the CPU oracle on identical (float32) state.

Tolerances (north_star): hash keys, bucket contents and active sets
bit-exact; logits / probabilities / loss 1e-5 relative; weights and Adam
state after a step 1e-4 relative.
"""

import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import slide_oracle as O  # noqa: E402
from paper_1903_03129_b200 import (  # noqa: E402
    HashFamilyConfig,
    LshLayerConfig,
    LshTables,
    SamplerConfig,
    SlideNetwork,
    SparseVector,
    TrainConfig,
    new_hash_family,
)
from paper_1903_03129_b200.network import HostCsr, csr_from_batch  # noqa: E402
from tests.parity_util import (  # noqa: E402
    assert_step_state_close,
    oracle_lsh_from_net,
    oracle_state_from_net,
    teacher_forced_step,
)

HASH_SPECS = {
    "sh_main": dict(family="simhash", k_per_table=9, num_tables=50, dim=128, seed=7919 * 2),
    "sh_small": dict(family="simhash", k_per_table=2, num_tables=4, dim=24, seed=5),
    "sh_full": dict(family="simhash", k_per_table=4, num_tables=2, dim=6, simhash_sparsity=1.0, seed=11),
    "dw_main": dict(family="dwta", k_per_table=8, num_tables=50, dim=128, wta_bin_size=8, seed=7919 * 2),
    "dw_small": dict(family="dwta", k_per_table=2, num_tables=1, dim=9, wta_bin_size=3, seed=5),
    "dw_ragged": dict(family="dwta", k_per_table=2, num_tables=3, dim=10, wta_bin_size=4, seed=1),
    "dw_scaled": dict(family="dwta", k_per_table=8, num_tables=64, dim=256, wta_bin_size=8, seed=7919 * 2),
}


@pytest.mark.parametrize("name", sorted(HASH_SPECS))
def test_device_hash_keys_match_reference(golden, name):
    g = golden("hashing")
    fam = new_hash_family(HashFamilyConfig(**HASH_SPECS[name]))
    np.testing.assert_array_equal(fam.hash_batch(g[name + "_w"]), g[name + "_wkeys"])
    q = g[name + "_q"]
    np.testing.assert_array_equal(fam.hash_dense_rows(q), g[name + "_qkeys"])
    for row in (0, 1, 2, 5):
        np.testing.assert_array_equal(fam.hash(SparseVector.from_dense(q[row])), g[name + "_qkeys"][row])


def test_tensor_core_rebuild_hash_matches_oracle():
    """>= 148 x 128 rows take the tcgen05 path (bf16x3 split, fp32 TMEM
    accumulation, certified signs + exact fp64 fix-up): keys bit-exact against
    the oracle, including rows whose projections cancel exactly (sign(0) -> 0),
    all-zero rows and rows spanning a huge dynamic range."""
    spec = HASH_SPECS["sh_main"]
    fam = new_hash_family(HashFamilyConfig(**spec))
    rng = np.random.default_rng(17)
    n, d = 30000, spec["dim"]
    w = rng.standard_normal((n, d)).astype(np.float32)
    w[::97] = 0.0  # all-zero rows: every dot is exactly 0
    for r in range(1, n, 101):  # exact cancellations inside projections
        p = rng.integers(fam.n_codes)
        i = fam.proj_indices[p]
        w[r] = 0.0
        w[r, i[0]], w[r, i[1]] = 0.75, 0.75 * fam.proj_signs[p, 0] * fam.proj_signs[p, 1] * -1
    w[5::211] *= np.float32(1e18)
    w[7::223, :3] = np.float32(1e-30)
    w = w.astype(np.float64)
    params = O.SimHashParams(d, spec["k_per_table"], spec["num_tables"], fam.proj_indices, fam.proj_signs)
    np.testing.assert_array_equal(fam.hash_batch(w), O.simhash_keys(params, w))


def test_wta_dense_equals_dwta_on_dense_inputs():
    rng = np.random.default_rng(3)
    wta = new_hash_family(HashFamilyConfig("wta", 3, 2, 12, wta_bin_size=4, seed=13))
    dwta = new_hash_family(HashFamilyConfig("dwta", 3, 2, 12, wta_bin_size=4, seed=13))
    x = rng.standard_normal((20, 12)).astype(np.float32).astype(np.float64)
    x[x == 0] = 0.5
    np.testing.assert_array_equal(wta.hash_batch(x), dwta.hash_batch(x))


def _golden_tables(g, prefix):
    out = {}
    for i in range(len(g[prefix + "t"])):
        a, b = g[prefix + "ptr"][i], g[prefix + "ptr"][i + 1]
        out[(int(g[prefix + "t"][i]), int(g[prefix + "key"][i]))] = (g[prefix + "slots"][a:b].tolist(),
                                                                      int(g[prefix + "count"][i]))
    return out


def _device_tables(tbl):
    return {(t, k): (list(b.slots), b.count) for t, view in enumerate(tbl.tables) for k, b in view.items()}


@pytest.mark.parametrize("policy", ["fifo", "reservoir"])
def test_device_tables_match_reference(golden, policy):
    g = golden("tables")
    fam = new_hash_family(HashFamilyConfig("simhash", 2, 5, 24, seed=5))
    tbl = LshTables(fam, policy=policy, capacity=16, seed=104729 * 2)
    w = g[policy + "_w"]
    tbl.build(w)
    assert _device_tables(tbl) == _golden_tables(g, f"{policy}_b1_")
    tbl.build(w[::-1].copy())  # reservoir stream continues across builds
    assert _device_tables(tbl) == _golden_tables(g, f"{policy}_b2_")


def test_device_dwta_reservoir_tables(golden):
    g = golden("tables")
    fam = new_hash_family(HashFamilyConfig("dwta", 8, 10, 128, wta_bin_size=8, seed=9))
    tbl = LshTables(fam, policy="reservoir", capacity=128, seed=1)
    tbl.build(g["dwta_w"])
    assert _device_tables(tbl) == _golden_tables(g, "dwta_")


def test_query_self_collision_and_probe_count():
    rng = np.random.default_rng(3)
    fam = new_hash_family(HashFamilyConfig("simhash", 2, 6, 24, seed=5))
    tbl = LshTables(fam)
    w = rng.standard_normal((8, 24)).astype(np.float32)
    tbl.build(w)
    raw = tbl.query(SparseVector.from_dense(w[4]))
    assert len(raw.per_table) == 6
    assert all(4 in ids for ids in raw.per_table)


NET_SETUPS = {
    "sh": (50, 16, 40, LshLayerConfig("simhash", k=3, l=6, capacity=8, sampler=SamplerConfig("vanilla", beta=10)), 6, 2),
    "shtopk": (50, 16, 40, LshLayerConfig("simhash", k=3, l=6, capacity=8, sampler=SamplerConfig("topk", beta=7)), 6, 2),
    "dw": (40, 12, 60, LshLayerConfig("dwta", k=2, l=5, capacity=4, policy="reservoir", wta_bin_size=4,
                                       sampler=SamplerConfig("vanilla", beta=6)), 5, 2),
    "dwth": (40, 12, 60, LshLayerConfig("dwta", k=2, l=5, capacity=4, policy="reservoir", wta_bin_size=4,
                                         sampler=SamplerConfig("hard_threshold", beta=6, min_freq=2)), 5, 2),
    "dense": (20, 8, 12, None, 4, 50),
}


@pytest.mark.parametrize("family", ["simhash", "dwta"])
def test_full_union_vanilla_matches_oracle(family):
    """beta >= L*cap: every table is probed (the bitmap selection path)."""
    rng = np.random.default_rng(8)
    D, H, N, B = 60, 16, 300, 8
    spec = LshLayerConfig(family, k=2, l=6, capacity=8, wta_bin_size=4, policy="fifo",
                          sampler=SamplerConfig("vanilla", beta=100))
    cfg = TrainConfig(batch_size=B, seed=4, learning_rate=1e-2, n0=2)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec})
    for it in (1, 2, 3):
        batch = []
        for _ in range(B):
            idx = np.sort(rng.choice(D, size=int(rng.integers(1, 10)), replace=False))
            vals = (np.abs(rng.standard_normal(idx.size)) + 0.1).astype(np.float32).astype(np.float64)
            batch.append((SparseVector(idx, vals, D), set(rng.choice(N, size=2, replace=False).tolist())))
        trip = [(x.indices, x.values, sorted(y)) for x, y in batch]
        want, got, _ = teacher_forced_step(net, trip, it, "snapshot", 1e-2, what=f"full-union {family} it{it}")
        assert got.active_fraction[1] == pytest.approx(want.active_fraction, rel=1e-12)


@pytest.mark.parametrize("shape", ["sparse", "mixed", "dense"])
def test_dense_and_sparse_tiles_match_oracle(shape):
    """The logits pick a register-tiled dense path or the per-row path for
    each 64-row tile from its pair density; every mix must equal the
    oracle."""
    rng = np.random.default_rng(21)
    D, H = 80, 24
    N, B, beta, cap, l = {"sparse": (3000, 32, 4, 2, 3), "mixed": (700, 40, 60, 8, 8),
                          "dense": (150, 48, 150, 32, 8)}[shape]
    spec = LshLayerConfig("simhash", k=2, l=l, capacity=cap, sampler=SamplerConfig("vanilla", beta=beta))
    cfg = TrainConfig(batch_size=B, seed=6, learning_rate=1e-2, n0=2)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec})
    for it in (1, 2, 3):
        trip = []
        for _ in range(B):
            idx = np.sort(rng.choice(D, size=int(rng.integers(1, 12)), replace=False))
            vals = (np.abs(rng.standard_normal(idx.size)) + 0.1).astype(np.float32).astype(np.float64)
            # Zipf-ish labels: a few hot rows held by most samples, a long tail
            lab = sorted(set(int(v) % N for v in rng.zipf(1.3, size=3)))
            trip.append((idx, vals, lab))
        want, got, _ = teacher_forced_step(net, trip, it, "snapshot", 1e-2, what=f"{shape} it{it}")
        assert got.active_fraction[1] == pytest.approx(want.active_fraction, rel=1e-12)


def _golden_batch(g, name, it, B):
    return [(g[f"{name}_it{it}_x{i}_idx"], g[f"{name}_it{it}_x{i}_val"], g[f"{name}_it{it}_y{i}"].tolist())
            for i in range(B)]


@pytest.mark.parametrize("mode", ["sequential", "snapshot"])
@pytest.mark.parametrize("name", sorted(NET_SETUPS))
def test_train_steps_match_oracle(golden, name, mode):
    """Three steps (a rebuild after step 2, an empty input in step 2), each
    teacher-forced from the device's state: per-slot active sets exact,
    probabilities and loss 1e-5, every state tensor (hidden bias moments
    included) under the per-coordinate 1e-4 model, rebuilt tables exact."""
    g = golden("network")
    D, H, N, spec, B, n0 = NET_SETUPS[name]
    cfg = TrainConfig(batch_size=B, seed=3, learning_rate=1e-2, n0=n0)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec} if spec else None)
    st = oracle_state_from_net(net)
    # the f32 initial weights equal the reference's f64 draws rounded
    np.testing.assert_allclose(st.w2, g[f"{name}_init_l1_w"], rtol=1e-7, atol=0)
    for it in range(1, 4):
        trip = _golden_batch(g, name, it, B)
        want, stats, _ = teacher_forced_step(net, trip, it, mode, 1e-2, what=f"{name} {mode} it{it}")
        assert stats.rebuilt == ([1] if (spec and it % n0 == 0) else [])


@pytest.mark.parametrize("name", ["sh", "dw", "dense"])
def test_relabelled_units_keep_the_network(golden, name):
    """slide_relabel_units renumbers the hidden units on the device (live
    units adjacent); the caller's views, the hash keys / active sets and the
    training steps must not notice.  A random renumbering before step 1 and
    another after step 2: views unchanged bit for bit, every step still
    equal to the oracle, single-sample forward / backward in the caller's
    unit order."""
    g = golden("network")
    D, H, N, spec, B, n0 = NET_SETUPS[name]
    cfg = TrainConfig(batch_size=B, seed=3, learning_rate=1e-2, n0=n0)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec} if spec else None)
    net.relabel_units = False  # only the explicit renumberings below
    rng = np.random.default_rng(17)
    queries = rng.standard_normal((5, H))
    for it in range(1, 4):
        if it != 2:
            before = oracle_state_from_net(net)
            unions = net.layers[1].lsh.query_union_batch(queries) if spec else None
            net._relabel(rng.permutation(H))
            after = oracle_state_from_net(net)
            if spec:  # external queries (caller's unit order) probe the same buckets
                for a, b in zip(unions, net.layers[1].lsh.query_union_batch(queries)):
                    np.testing.assert_array_equal(a, b)
            for a, b in zip(vars(before).values(), vars(after).values()):
                np.testing.assert_array_equal(a, b)
            assert not np.array_equal(net.unit_cols(), np.arange(H))
            np.testing.assert_array_equal(net.layers[0].w, before.w1t.T)
            np.testing.assert_array_equal(net.layers[1].adam_m, before.m2)
            np.testing.assert_array_equal(net.layers[0].steps, before.steps1)
        trip = _golden_batch(g, name, it, B)
        teacher_forced_step(net, trip, it, "snapshot", 1e-2, what=f"relabelled {name} it{it}")
    # view writes land in the right physical columns -- also through a view
    # taken before a renumbering
    w = net.layers[1].w
    w[3, 5] = 0.25
    b = net.layers[0].b
    b[2] = -0.5
    w1 = net.layers[0].w
    net._relabel(rng.permutation(H))
    w1[1, 4] = 0.125
    st = oracle_state_from_net(net)
    assert st.w2[3, 5] == 0.25 and st.b1[2] == -0.5 and st.w1t[4, 1] == 0.125
    # single-sample API: activations and hidden errors in the caller's order
    xi, xv, y = _golden_batch(g, name, 1, B)[0]
    x = SparseVector(np.asarray(xi), np.asarray(xv), D)
    tr = net.forward(x, 0, labels=y, rng=np.random.default_rng(1))
    hh = np.maximum(np.asarray(xv) @ st.w1t[np.asarray(xi)] + st.b1, 0.0)
    np.testing.assert_allclose(tr.inputs[1].to_dense(), hh, rtol=1e-5, atol=1e-7)
    cap = []
    net.backward(tr, y, 0, update=False, capture=cap)
    delta = cap[0][4]
    dh = delta @ st.w2[tr.active[-1]]
    nz = tr.inputs[1].indices
    np.testing.assert_allclose(cap[1][4], dh[nz], rtol=1e-4, atol=1e-7)


@pytest.mark.parametrize("H", [128, 96, 256])
def test_hot_rows_in_sparse_set_steps(H):
    """Sparse-set regime (sets x 4 < N) with labels shared by most of the batch:
    rows held by more than 64 samples take the CTA-per-row W2 Adam
    (adam_rows_vlong_kernel: 16 segments with folded moment recurrences, two
    unit groups and the bias per walk) beside the persistent kernel.  Three
    teacher-forced steps from step 1, where every hidden unit is live (four
    unit groups at H = 128: two walks; eight at H = 256 through the
    wide-hidden kernels; a ragged last group at H = 96) down to the few-group
    regime."""
    rng = np.random.default_rng(31)
    D, N, B = 300, 20000, 128
    spec = LshLayerConfig("dwta", k=4, l=8, capacity=16, policy="fifo", wta_bin_size=4,
                          sampler=SamplerConfig("vanilla", beta=32))
    cfg = TrainConfig(batch_size=B, seed=9, learning_rate=1e-3, n0=1000)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec})
    held = []
    for it in (1, 2, 3):
        trip = []
        for i in range(B):
            idx = np.sort(rng.choice(D, size=int(rng.integers(3, 12)), replace=False))
            vals = (rng.random(idx.size) + 0.05).astype(np.float32).astype(np.float64)
            labels = {7, int(rng.integers(0, N))}  # row 7: every sample; row 11: ~2/3 of them
            if i % 3:
                labels.add(11)
            trip.append((idx.astype(np.int64), vals, sorted(labels)))
        want, got, _ = teacher_forced_step(net, trip, it, "snapshot", 1e-3, what=f"hot rows H{H} it{it}")
        held.append(sum(7 in t.active for t in want.traces))
    assert min(held) == B  # the hot row really was held by the whole batch


def test_two_pass_selection_mixed_samples():
    """Sparse buckets with one hot bucket per table: the selection runs its
    1,024-candidate pass first and the bound-sized pass (L x capacity + labels
    = 5,120 + candidates) only for the samples flagged by it.  Half of the W2
    rows are copies of one vector v and the hidden layer is rigged so that a
    sample's activations are either exactly v (it probes the copies' full
    bucket in all 40 tables: 5,120 candidates) or all zero (key 0 everywhere:
    a handful) -- both kinds in one batch, against the oracle."""
    rng = np.random.default_rng(5)
    D, H, N, B = 64, 32, 3000, 24
    spec = LshLayerConfig("simhash", k=10, l=40, capacity=128, sampler=SamplerConfig("vanilla", beta=64))
    cfg = TrainConfig(batch_size=B, seed=2, learning_rate=1e-3, n0=1000)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec})
    v = (np.abs(rng.standard_normal(H)) + 0.1).astype(np.float32).astype(np.float64)
    w1 = np.zeros((H, D))
    w1[:, 0] = -4.0 * v  # feature 0 (value 1) switches every unit off
    net.layers[0].w = w1
    net.layers[0].b = v
    w2 = np.asarray(net.layers[1].w).copy()
    w2[:1500] = v
    net.layers[1].w = w2
    net._rebuild_tables()
    sizes = set()
    for it in (1, 2):
        trip = []
        for i in range(B):
            idx = np.sort(rng.choice(np.arange(1, D), size=int(rng.integers(2, 6)), replace=False))
            if i % 3 == 0:
                idx = np.concatenate([[0], idx])
            vals = np.ones(idx.size)
            # (labels outside the copies: with both labels among them the hidden
            # error v * sum(delta) cancels to rounding noise, which Adam normalises)
            labels = sorted(rng.choice(np.arange(1500, N), size=2, replace=False).tolist())
            trip.append((idx.astype(np.int64), vals, labels))
        want, got, _ = teacher_forced_step(net, trip, it, "snapshot", 1e-3, what=f"two-pass select it{it}")
        sizes |= {len(t.active) for t in want.traces}
    # both kinds were in the batches: the copies' bucket (128 ids + labels) and beta-sized sets
    assert max(sizes) >= 128 and min(sizes) < 128


def _stage_forward(net, csr, iteration):
    from paper_1903_03129_b200 import _lib

    net.layers[1].lsh.sync_to_device()
    bt, keep = net._upload(csr)
    n = _lib.i64()
    _lib.call("slide_forward", net._ctx, _lib.C.byref(bt), iteration, 0, _lib.C.byref(n))
    B, hp, L = csr.batch, net.hidden_pad, net.layers[1].lsh.family.l
    out = {
        "h": net._read(0, B * hp, np.float32).reshape(B, hp)[:, : net.hidden],
        "keys": net._read(1, B * L, np.uint32).reshape(B, L).astype(np.int64),
        "offs": net._read(2, B + 1, np.int32),
        "rows": net._read(3, n.value, np.int32),
        "probs": net._read(5, n.value, np.float32),
        "logits": net._read(11, n.value, np.float32),
        "loss": net._read(7, B, np.float64),
    }
    return out, keep


def test_tiny_config_stage_by_stage():
    """BASELINE configs[0] shape: each stage of one snapshot step against the
    oracle fed the device's own upstream values."""
    from paper_1903_03129_b200 import _lib
    from paper_1903_03129_b200.configs import TINY as w
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(w.corpus, w.batch, seed=0)
    cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr, n0=w.n0)
    spec = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
    net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
    st = oracle_state_from_net(net)
    lsh = oracle_lsh_from_net(net, spec, st)
    csr = HostCsr(corpus.x_ptr.astype(np.int32), corpus.x_idx, corpus.x_val, corpus.y_ptr.astype(np.int32), corpus.y_idx)
    got, keep = _stage_forward(net, csr, 1)
    trip = corpus.triples()
    for i, (xi, xv, y) in enumerate(trip):
        rng = np.random.default_rng((0, 1, i))
        tr = O.slot_forward(st, lsh, xi, xv, y, rng, w.n_out)
        np.testing.assert_allclose(got["h"][i], tr.h, rtol=1e-5, atol=1e-6)
        hd = got["h"][i].astype(np.float64)  # the device's own h
        keys = O.simhash_keys(lsh.params, hd[None, :])[0]
        np.testing.assert_array_equal(got["keys"][i], keys)
        per_table = O.probe(lsh.buckets, keys)
        samp = O.sampled_ids(per_table, "vanilla", w.beta, 1, np.random.default_rng((0, 1, i)))
        active = np.union1d(samp, y) if samp.size else None
        a, b = got["offs"][i], got["offs"][i + 1]
        if active is not None:
            np.testing.assert_array_equal(got["rows"][a:b], active)
        np.testing.assert_array_equal(got["rows"][a:b], tr.active)
        np.testing.assert_allclose(got["probs"][a:b], tr.probs, rtol=1e-5, atol=1e-9)
        assert got["loss"][i] == pytest.approx(tr.loss, rel=1e-5)
    # full snapshot step
    _lib.call("slide_backward", net._ctx, 1)
    torch.cuda.synchronize()
    st_pre = st.copy()
    lsh.schedule = O.Schedule(1 << 40)
    want = O.train_step(st, lsh, trip, 1, 0, w.n_out, O.AdamCfg(lr=w.lr), mode="snapshot")
    assert_step_state_close(net, st, st_pre, want, O.AdamCfg(lr=w.lr), what="tiny snapshot")


def test_forward_emulates_the_callers_generator():
    cfg = TrainConfig(batch_size=2, seed=5)
    spec = LshLayerConfig(k=2, l=4, sampler=SamplerConfig(beta=4))
    net = SlideNetwork(6, [5, 30], cfg, lsh_layers={1: spec})
    x = SparseVector(np.array([0, 3]), np.array([1.0, 2.0]), 6)
    r_dev = np.random.default_rng(11)
    r_ref = np.random.default_rng(11)
    tr = net.forward(x, 1, labels={7}, rng=r_dev)
    st = oracle_state_from_net(net)
    lsh = oracle_lsh_from_net(net, spec, st)
    want = O.slot_forward(st, lsh, x.indices, x.values, [7], r_ref, 30)
    np.testing.assert_array_equal(tr.active[-1], want.active)
    assert r_dev.bit_generator.state == r_ref.bit_generator.state
    assert r_dev.random() == r_ref.random()


def test_empty_buckets_fall_back_to_random_plus_labels():
    cfg = TrainConfig(batch_size=3, seed=5)
    spec = LshLayerConfig(k=2, l=2, sampler=SamplerConfig(beta=4))
    net = SlideNetwork(4, [4, 30], cfg, lsh_layers={1: spec})
    for tbl in net.layers[1].lsh.tables:
        tbl.clear()
    x = SparseVector(np.array([0, 1]), np.array([1.0, 1.0]), 4)
    r1, r2 = np.random.default_rng(1), np.random.default_rng(1)
    tr = net.forward(x, 0, labels={7}, rng=r1)
    assert 7 in tr.active[-1]
    assert tr.active[-1].size >= 4
    r2.permutation(2)  # vanilla draws its probe order first (samplers.py:69)
    want = np.union1d(r2.choice(30, size=4, replace=False), [7])
    np.testing.assert_array_equal(tr.active[-1], want)
    assert r1.bit_generator.state == r2.bit_generator.state


@pytest.mark.parametrize("beta", [128, 3000])
def test_large_fallback_sets_match_numpy(beta):
    """Floyd (beta small) and tail-shuffle (beta > N/50, N > 10000) branches
    of numpy's choice(), replayed on the device."""
    cfg = TrainConfig(batch_size=4, seed=9)
    spec = LshLayerConfig("dwta", k=2, l=3, capacity=4, wta_bin_size=4, sampler=SamplerConfig(beta=beta))
    n_out = 20000
    net = SlideNetwork(8, [8, n_out], cfg, lsh_layers={1: spec})
    for tbl in net.layers[1].lsh.tables:
        tbl.clear()
    batch = [(SparseVector(np.array([i]), np.array([1.0]), 8), {i}) for i in range(4)]
    csr = csr_from_batch(batch, 8, n_out)
    got, keep = _stage_forward(net, csr, 3)
    from paper_1903_03129_b200 import _lib

    states = net._read(10, 4 * 6, np.uint64).reshape(4, 6)
    for i in range(4):
        r = np.random.default_rng((9, 3, i))
        r.permutation(3)
        want = np.union1d(r.choice(n_out, size=beta, replace=False), [i])
        np.testing.assert_array_equal(got["rows"][got["offs"][i]: got["offs"][i + 1]], want)
        # the slot's generator ends where numpy's does (the parallel draws
        # restore the state after exactly the values numpy consumed)
        np.testing.assert_array_equal(states[i], _lib.pcg64_state_from_generator(r))


def test_hand_computed_forward_and_views():
    net = SlideNetwork(2, [3, 2], TrainConfig(batch_size=1))
    w1 = np.array([[1.0, 2.0], [10.0, 10.0], [0.5, -1.0]])
    w2 = np.array([[1.0, 5.0, 2.0], [-1.0, 5.0, 1.0]])
    net.layers[0].w[:] = w1
    net.layers[0].b[:] = np.array([0.1, 0.0, 0.2])
    net.layers[1].w[:] = w2
    net.layers[1].b[:] = 0.0
    x = SparseVector.from_dense([1.0, 1.0])
    # hidden unit 1 forced off by a large negative bias instead of a forced set
    net.layers[0].b[1] = -1000.0
    trace = net.forward(x, 0)
    h0 = 1.0 * 1 + 2.0 * 1 + 0.1
    assert net.layers[0].activations[0, 0] == pytest.approx(h0, rel=1e-6)
    z = np.array([w2[0, 0] * h0, w2[1, 0] * h0])
    e = np.exp(z - z.max())
    np.testing.assert_allclose(trace.probs, e / e.sum(), rtol=1e-5)


def test_empty_input_and_dead_hidden_layer_match_oracle():
    cfg = TrainConfig(batch_size=3, seed=2, learning_rate=1e-2)
    spec = LshLayerConfig("simhash", k=2, l=3, capacity=4, sampler=SamplerConfig(beta=5))
    net = SlideNetwork(10, [6, 20], cfg, lsh_layers={1: spec})
    net.layers[0].b[:] = np.array([0.3, -5.0, 0.2, -5.0, 0.1, 0.4])
    batch = [(SparseVector(np.empty(0, np.int64), np.empty(0), 10), {1}),
             (SparseVector(np.array([2, 5]), np.array([1.0, 0.5]), 10), {3, 4}),
             (SparseVector(np.array([7]), np.array([0.25]), 10), {19})]
    trip = [(x.indices, x.values, sorted(y)) for x, y in batch]
    for it, mode in ((1, "snapshot"), (2, "sequential")):
        teacher_forced_step(net, trip, it, mode, 1e-2, what=f"edge {mode}")
    # all hidden units dead: only output biases move, hidden layer untouched
    net.layers[0].b[:] = -50.0
    w1 = np.array(net.layers[0].w)
    teacher_forced_step(net, trip, 3, "snapshot", 1e-2, what="dead hidden")
    np.testing.assert_array_equal(np.array(net.layers[0].w), w1)


def test_snapshot_step_is_deterministic():
    from paper_1903_03129_b200.configs import TINY as w
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(w.corpus, w.batch, seed=4)
    csr = HostCsr(corpus.x_ptr.astype(np.int32), corpus.x_idx, corpus.x_val, corpus.y_ptr.astype(np.int32), corpus.y_idx)
    outs = []
    for _ in range(2):
        cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr)
        spec = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
        net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
        for it in (1, 2, 3):
            net.train_batch_csr(csr, it, schedule="snapshot")
        outs.append((net.w2.cpu().numpy().copy(), net.w1t.cpu().numpy().copy(), net.m2.cpu().numpy().copy()))
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


def test_graph_steps_equal_eager_steps():
    """The captured-graph snapshot step (eager run, capture, replays, a
    re-capture on a larger batch) is bit-identical to eager snapshot steps."""
    from paper_1903_03129_b200.configs import TINY as w
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(w.corpus, 6 * 64, seed=5)

    def run(graphs):
        cfg = TrainConfig(batch_size=64, seed=0, learning_rate=w.lr, n0=3)
        spec = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
        net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
        net.use_graphs = graphs
        losses = []
        for it in range(1, 7):
            sub = corpus.subset(np.arange((it - 1) * 64, it * 64))
            if it == 5:  # heavier batch: grows the capacities -> re-capture
                sub = corpus.subset(np.concatenate([np.arange(0, 64)] * 1)[:64])
            csr = HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx)
            losses.append(net.train_batch_csr(csr, it, schedule="snapshot").loss)
        return losses, net.w2.cpu().numpy(), net.w1t.cpu().numpy(), net.v2.cpu().numpy()

    a, b = run(True), run(False)
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


def test_backward_capture_matches_finite_differences_shape():
    """backward(update=False, capture=...) returns the reference's capture
    tuples; gradients equal the oracle's on the same trace."""
    cfg = TrainConfig(batch_size=2, seed=4)
    net = SlideNetwork(6, [7, 9], cfg)
    rng = np.random.default_rng(0)
    x = SparseVector(np.arange(6), rng.standard_normal(6).astype(np.float32), 6)
    trace = net.forward(x, 0, labels={2, 5})
    cap = []
    net.backward(trace, {2, 5}, 0, update=False, capture=cap)
    st = oracle_state_from_net(net)
    tr = O.slot_forward(st, None, x.indices, x.values, [2, 5], np.random.default_rng(0), 9)
    g = O.slot_backward(st, tr, [2, 5])
    li, rows, cols, grad, delta = cap[0]
    assert li == 1
    np.testing.assert_allclose(delta, g.delta, rtol=1e-5, atol=1e-7)
    if g.dh is not None:
        assert cap[1][0] == 0
        np.testing.assert_allclose(cap[1][4], g.dh, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("strategy", ["vanilla", "topk"])
def test_batched_ranking_equals_sequential_predict(strategy):
    """predict_batch (the evaluator: one generator shared across queries,
    B queries per device pass, device top-k) equals query-by-query predict
    with the same generator -- including queries whose buckets are all empty
    (the fallback draw advances the shared generator) and empty inputs."""
    from paper_1903_03129_b200.data import precision_at_k, score_precision_at_k

    rng = np.random.default_rng(31)
    D, H, N, B = 60, 16, 300, 16
    spec = LshLayerConfig("simhash", k=3, l=4, capacity=8, sampler=SamplerConfig(strategy, beta=10))
    cfg = TrainConfig(batch_size=B, seed=2, learning_rate=1e-2, n0=5)
    net = SlideNetwork(D, [H, N], cfg, lsh_layers={1: spec})
    ex = []
    for _ in range(45):
        nnz = int(rng.integers(0, 8))
        idx = np.sort(rng.choice(D, size=nnz, replace=False))
        ex.append((SparseVector(idx, np.abs(rng.standard_normal(nnz)) + 0.1, D), sorted(rng.choice(N, 2, replace=False).tolist())))
    net.train_batch(ex[:B], 1)
    lsh = net.layers[1].lsh
    for view in lsh.tables:  # drop half of every table's buckets: some queries come back empty
        for key in list(view.keys())[::2]:
            del view[key]
    lsh.sync_to_device()
    xs = [x for x, _ in ex]
    n_empty = 0
    for x in xs:
        net.forward(x, 0, rng=np.random.default_rng(0))
        n_empty += int(net._read(9, 1, np.int32)[0])
    assert 0 < n_empty < len(xs)
    r1, r2 = np.random.default_rng(7), np.random.default_rng(7)
    want = [net.predict(x, rng=r1)[:5] for x in xs]
    got = net.predict_batch(xs, topn=5, rng=r2)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    assert r1.bit_generator.state == r2.bit_generator.state
    p1 = score_precision_at_k(net, ex, k=1, seed=3)
    r3 = np.random.default_rng(3)
    assert p1 == pytest.approx(float(np.mean([precision_at_k(net.predict(x, rng=r3)[:1], y, 1) for x, y in ex])))


@pytest.mark.parametrize("family", ["simhash", "dwta"])
def test_batched_query_union_equals_per_query_probes(family):
    """slide_query_union (hash + L probes + union for a batch) equals the
    union of each query's own L probes (reference tables.py:165-176,
    samplers.py:109-112 with min_freq=1)."""
    rng = np.random.default_rng(4)
    if family == "simhash":
        fam = new_hash_family(HashFamilyConfig("simhash", 4, 6, 32, seed=3))
    else:
        fam = new_hash_family(HashFamilyConfig("dwta", 3, 6, 32, wta_bin_size=4, seed=3))
    tbl = LshTables(fam, policy="fifo", capacity=8, seed=1)
    tbl.build(rng.standard_normal((500, 32)).astype(np.float32))
    q = rng.standard_normal((70, 32)).astype(np.float32).astype(np.float64)
    got = tbl.query_union_batch(q)
    for i in range(q.shape[0]):
        raw = tbl.query(SparseVector.from_dense(q[i]))
        want = np.unique(np.concatenate([np.asarray(p, dtype=np.int64) for p in raw.per_table] + [np.zeros(0, np.int64)]))
        np.testing.assert_array_equal(got[i], want)


REBUILD_SPECS = {
    "dw_main": HASH_SPECS["dw_main"],
    "dw_scaled": HASH_SPECS["dw_scaled"],
    # 4- and 16-wide bins, a ragged last bin (96 = 19 x 5 + 1)
    "dw_m4": dict(family="dwta", k_per_table=6, num_tables=20, dim=64, wta_bin_size=4, seed=3),
    "dw_m16": dict(family="dwta", k_per_table=4, num_tables=30, dim=128, wta_bin_size=16, seed=4),
    "dw_ragged96": dict(family="dwta", k_per_table=5, num_tables=12, dim=96, wta_bin_size=5, seed=6),
}


@pytest.mark.parametrize("name", list(REBUILD_SPECS))
def test_dwta_rebuild_path_matches_oracle(name):
    """> 148 x 8 rows take the tiled rebuild kernel (64 rows per tile, lanes =
    rows): keys equal the oracle's, including sparse rows whose empty bins
    borrow donor codes (the tile's densification pass), rows with ties, and a
    partial last tile."""
    spec = REBUILD_SPECS[name]
    fam = new_hash_family(HashFamilyConfig(**spec))
    rng = np.random.default_rng(12)
    n, d = 5000, spec["dim"]
    w = rng.standard_normal((n, d)).astype(np.float32)
    w[::3] *= rng.random((w[::3].shape[0], d)) < 0.05  # mostly-zero rows: empty bins, donors
    w[1::7] = np.round(w[1::7])  # many ties: lowest in-bin offset wins
    w = w.astype(np.float64)
    params = O.dwta_params(d, spec["k_per_table"], spec["num_tables"], spec["wta_bin_size"], spec["seed"])
    np.testing.assert_array_equal(fam.hash_batch(w), O.dwta_keys(params, w))


def test_wta_rebuild_path_equals_dwta_on_dense_rows():
    """The tiled kernel in WTA mode (zeros take part): on rows without zeros
    WTA and DWTA agree (hashing.py:262-274)."""
    rng = np.random.default_rng(5)
    w = rng.standard_normal((3000, 128)).astype(np.float32).astype(np.float64)
    w[w == 0] = 1.0
    wta = new_hash_family(HashFamilyConfig("wta", 8, 10, 128, wta_bin_size=8, seed=8))
    dwta = new_hash_family(HashFamilyConfig("dwta", 8, 10, 128, wta_bin_size=8, seed=8))
    np.testing.assert_array_equal(wta.hash_batch(w), dwta.hash_batch(w))


def test_pipelined_batches_equal_per_call_steps():
    """train_batches_csr (step k on the device while batch k+1 is staged,
    rebuild barrier between steps) equals train_batch_csr per batch bit for
    bit, across a table rebuild."""
    from paper_1903_03129_b200.configs import TINY as w
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(w.corpus, 7 * 64, seed=8)
    batches = []
    for it in range(7):
        sub = corpus.subset(np.arange(it * 64, (it + 1) * 64))
        batches.append(HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx))

    def make():
        cfg = TrainConfig(batch_size=64, seed=0, learning_rate=w.lr, n0=3)
        spec = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
        return SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})

    a = make()
    sa = [a.train_batch_csr(c, it) for it, c in enumerate(batches, start=1)]
    b = make()
    sb = b.train_batches_csr(batches, first_iteration=1)
    assert [s.loss for s in sa] == [s.loss for s in sb]
    assert [s.rebuilt for s in sa] == [s.rebuilt for s in sb]
    assert any(s.rebuilt for s in sb)
    np.testing.assert_array_equal(a.w2.cpu().numpy(), b.w2.cpu().numpy())
    np.testing.assert_array_equal(a.w1t.cpu().numpy(), b.w1t.cpu().numpy())


@pytest.mark.parametrize("alive", ["half", "36"])
def test_live_unit_permutation_tracks_the_batch(alive):
    """The hidden forward's live-unit list (the units nonzero in some sample,
    ascending, then the dead ones) equals h's nonzero columns after every
    step; with half the hidden units dead (bias -5) the row kernels walk only
    the live groups, and with 36 live units (bias +0.5, the rest -5) the W2
    Adam takes the 4 units past the first group in scan form; the trained
    state matches the oracle either way."""
    from paper_1903_03129_b200.configs import TINY as w
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(w.corpus, 3 * 64, seed=12)
    cfg = TrainConfig(batch_size=64, seed=0, learning_rate=w.lr, n0=50)
    spec = LshLayerConfig("simhash", k=w.k, l=w.l, capacity=w.cap, sampler=SamplerConfig("vanilla", beta=w.beta))
    net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
    b = np.array(net.layers[0].b)
    if alive == "half":
        b[::2] = -5.0  # even units dead for every input
    else:
        b[:] = -5.0
        b[np.random.default_rng(3).choice(w.hidden, 36, replace=False)] = 0.5
    net.layers[0].b[:] = b
    hp = net.hidden_pad
    for it in range(1, 4):
        sub = corpus.subset(np.arange((it - 1) * 64, it * 64))
        # teacher forcing: each step from the device's own state
        teacher_forced_step(net, sub.triples(), it, "snapshot", w.lr, what=f"live-unit step {it}")
        h = net._read(0, 64 * hp, np.float32).reshape(64, hp)
        live = net._read(13, 1 + hp, np.int32)
        on = np.flatnonzero((h > 0).any(0))
        n = int(live[0])
        assert 0 < n <= hp // 2 and n == on.size
        if alive != "half":
            assert n == 36
        np.testing.assert_array_equal(live[1:1 + n], on)
        np.testing.assert_array_equal(np.sort(live[1:]), np.arange(hp))
        assert np.all(np.diff(live[1 + n:]) > 0)
