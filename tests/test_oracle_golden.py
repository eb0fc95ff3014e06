"""Pin the CPU oracle to the reference: every check compares oracle output
with golden vectors produced by the reference itself (tests/golden/make_golden.py)."""

import random

import numpy as np
import pytest

from oracle import slide_oracle as O
from paper_1903_03129_b200.configs import TINY
from paper_1903_03129_b200.data import synthetic_corpus

HASH_SPECS = {
    "sh_main": ("simhash", 128, 9, 50, 1 / 3, 8, 7919 * 2),
    "sh_small": ("simhash", 24, 2, 4, 1 / 3, 8, 5),
    "sh_full": ("simhash", 6, 4, 2, 1.0, 8, 11),
    "dw_main": ("dwta", 128, 8, 50, 1 / 3, 8, 7919 * 2),
    "dw_small": ("dwta", 9, 2, 1, 1 / 3, 3, 5),
    "dw_ragged": ("dwta", 10, 2, 3, 1 / 3, 4, 1),
    "dw_scaled": ("dwta", 256, 8, 64, 1 / 3, 8, 7919 * 2),
}


def make_params(name):
    fam, d, k, l, sp, m, seed = HASH_SPECS[name]
    if fam == "simhash":
        return O.simhash_params(d, k, l, sp, seed)
    return O.dwta_params(d, k, l, m, seed)


@pytest.mark.parametrize("name", sorted(HASH_SPECS))
def test_hash_params_and_keys(golden, name):
    g = golden("hashing")
    p = make_params(name)
    if isinstance(p, O.SimHashParams):
        np.testing.assert_array_equal(p.idx, g[name + "_idx"])
        np.testing.assert_array_equal(p.signs, g[name + "_signs"])
    else:
        np.testing.assert_array_equal(p.perms, g[name + "_perms"])
        assert p.salt == int(g[name + "_salt"][0])
    np.testing.assert_array_equal(O.family_keys(p, g[name + "_q"]), g[name + "_qkeys"])
    np.testing.assert_array_equal(O.family_keys(p, g[name + "_w"]), g[name + "_wkeys"])


def test_dwta_salt_known_value():
    # seed 0 at layer 1 -> 0xf2163b224f9e990e
    assert O.mix64(7919 * 2, 0xD1F7, 0xA0B1) == 0xF2163B224F9E990E


def _tables_from_golden(g, prefix):
    out = {}
    for i in range(len(g[prefix + "t"])):
        t, key = int(g[prefix + "t"][i]), int(g[prefix + "key"][i])
        a, b = g[prefix + "ptr"][i], g[prefix + "ptr"][i + 1]
        out[(t, key)] = (g[prefix + "slots"][a:b].tolist(), int(g[prefix + "count"][i]))
    return out


def _tables_from_oracle(buckets):
    return {(t, k): (v[0].tolist(), v[1]) for t, tbl in enumerate(buckets) for k, v in tbl.items()}


@pytest.mark.parametrize("policy", ["fifo", "reservoir"])
def test_bucket_build_matches_reference(golden, policy):
    g = golden("tables")
    p = O.simhash_params(24, 2, 5, 1 / 3, 5)
    w = g[policy + "_w"]
    rnd = random.Random(104729 * 2)
    b1 = O.build_buckets(O.simhash_keys(p, w), 16, policy, rnd)
    assert _tables_from_oracle(b1) == _tables_from_golden(g, f"{policy}_b1_")
    b2 = O.build_buckets(O.simhash_keys(p, w[::-1].copy()), 16, policy, rnd)
    assert _tables_from_oracle(b2) == _tables_from_golden(g, f"{policy}_b2_")


def test_dwta_reservoir_build(golden):
    g = golden("tables")
    p = O.dwta_params(128, 8, 10, 8, 9)
    b = O.build_buckets(O.dwta_keys(p, g["dwta_w"]), 128, "reservoir", random.Random(1))
    assert _tables_from_oracle(b) == _tables_from_golden(g, "dwta_")


def _tables_from_arrays(tables):
    return {(t, k): (v[0].tolist(), v[1]) for t, tbl in enumerate(tables) for k, v in tbl.items()}


@pytest.mark.parametrize("policy", ["fifo", "reservoir"])
def test_array_bucket_build_equals_dict_build(golden, policy):
    """The array-form builder the oracle's OutputLsh uses (full-size tables)
    holds exactly the reference-pinned dict builder's buckets, physical slot
    order and reservoir draws included (golden overflow case, two builds on
    one stream, plus a random many-overflow case)."""
    g = golden("tables")
    p = O.simhash_params(24, 2, 5, 1 / 3, 5)
    w = g[policy + "_w"]
    ra, rd = random.Random(104729 * 2), random.Random(104729 * 2)
    for ws in (w, w[::-1].copy()):
        keys = O.simhash_keys(p, ws)
        a = O.build_bucket_arrays(keys, 16, policy, ra)
        assert _tables_from_arrays(a) == _tables_from_oracle(O.build_buckets(keys, 16, policy, rd))
    assert _tables_from_arrays(O.build_bucket_arrays(O.simhash_keys(p, w), 16, policy,
                                                     random.Random(104729 * 2))) == _tables_from_golden(g, f"{policy}_b1_")
    keys = np.random.default_rng(5).integers(0, 7, size=(500, 3))
    ra, rd = random.Random(9), random.Random(9)
    assert _tables_from_arrays(O.build_bucket_arrays(keys, 5, policy, ra)) == _tables_from_oracle(
        O.build_buckets(keys, 5, policy, rd))
    assert ra.random() == rd.random()
    empty = O.build_bucket_arrays(np.zeros((0, 2), np.int64), 4, policy, ra)
    assert [len(t) for t in empty] == [0, 0] and empty[0].get(3) is None


def test_samplers_match_reference(golden):
    g = golden("samplers")
    off = 0
    for case, (strat, beta, mf, L) in enumerate(g["cases"].tolist()):
        per_table = [g[f"c{case}_t{t}"] for t in range(L)]
        name = ["vanilla", "topk", "hard_threshold"][strat]
        got = np.sort(O.sampled_ids(per_table, name, beta, mf, np.random.default_rng((case, 1, 2))))
        n = g["lens"][case]
        np.testing.assert_array_equal(got, g["ids"][off : off + n], err_msg=f"case {case} {name}")
        off += n


NET_SETUPS = {
    "sh": (50, 16, 40, O.LshSpec("simhash", 3, 6, 8, "fifo", strategy="vanilla", beta=10), 6, 2),
    "shtopk": (50, 16, 40, O.LshSpec("simhash", 3, 6, 8, "fifo", strategy="topk", beta=7), 6, 2),
    "dw": (40, 12, 60, O.LshSpec("dwta", 2, 5, 4, "reservoir", bin_size=4, strategy="vanilla", beta=6), 5, 2),
    "dwth": (40, 12, 60, O.LshSpec("dwta", 2, 5, 4, "reservoir", bin_size=4, strategy="hard_threshold", beta=6, min_freq=2), 5, 2),
    "dense": (20, 8, 12, None, 4, 50),
}


def golden_batch(g, name, it, B):
    out = []
    for i in range(B):
        out.append((g[f"{name}_it{it}_x{i}_idx"], g[f"{name}_it{it}_x{i}_val"], g[f"{name}_it{it}_y{i}"].tolist()))
    return out


def check_state(st, g, prefix, tol=1e-10):
    pairs = [("w", st.w1t.T, st.w2), ("b", st.b1, st.b2), ("adam_m", st.m1t.T, st.m2),
             ("adam_v", st.v1t.T, st.v2), ("adam_mb", st.mb1, st.mb2), ("adam_vb", st.vb1, st.vb2)]
    for name, l0, l1 in pairs:
        np.testing.assert_allclose(l0, g[f"{prefix}_l0_{name}"], rtol=0, atol=tol, err_msg=f"{prefix} l0 {name}")
        np.testing.assert_allclose(l1, g[f"{prefix}_l1_{name}"], rtol=0, atol=tol, err_msg=f"{prefix} l1 {name}")
    np.testing.assert_array_equal(st.steps1, g[f"{prefix}_l0_steps"])
    np.testing.assert_array_equal(st.steps2, g[f"{prefix}_l1_steps"])


@pytest.mark.parametrize("mode", ["seq", "snap"])
@pytest.mark.parametrize("name", sorted(NET_SETUPS))
def test_train_steps_match_reference(golden, name, mode):
    g = golden("network")
    D, H, N, spec, B, n0 = NET_SETUPS[name]
    st = O.init_state(D, H, N, seed=3)
    check_state(st, g, f"{name}_init", tol=0)
    lsh = None
    if spec is not None:
        lsh = O.OutputLsh(spec, H, seed=3, n0=n0, lam=0.0)
        lsh.build(st.w2)
    cfg = O.AdamCfg(lr=1e-2)
    for it in range(1, 4):
        batch = golden_batch(g, name, it, B)
        res = O.train_step(st, lsh, batch, it, 3, N, cfg, mode="sequential" if mode == "seq" else "snapshot")
        assert np.mean(res.losses) == pytest.approx(float(g[f"{name}_{mode}_it{it}_loss"][0]), rel=1e-12)
        for i, tr in enumerate(res.traces):
            np.testing.assert_array_equal(tr.active, g[f"{name}_{mode}_it{it}_active{i}"])
            np.testing.assert_allclose(tr.probs, g[f"{name}_{mode}_it{it}_probs{i}"], rtol=1e-12, atol=1e-15)
        check_state(st, g, f"{name}_{mode}_it{it}")


def test_tiny_baseline_config_two_sequential_steps(golden):
    """BASELINE configs[0] shape (10k -> 128 -> 5k, SimHash K6 L20, vanilla
    beta 250) for two reference steps on the SURVEY 8(d) corpus."""
    g = golden("tiny_config")
    w = TINY
    corpus = synthetic_corpus(w.corpus, 2 * w.batch, seed=0)
    st = O.init_state(w.input_dim, w.hidden, w.n_out, seed=0)
    np.testing.assert_array_equal(st.w2[:8], g["init_w2_head"])
    np.testing.assert_array_equal(st.w1t[:8].T, g["init_w1_head"])
    spec = O.LshSpec("simhash", w.k, w.l, w.cap, w.policy, strategy="vanilla", beta=w.beta)
    lsh = O.OutputLsh(spec, w.hidden, seed=0, n0=w.n0, lam=0.0)
    lsh.build(st.w2)
    cfg = O.AdamCfg(lr=w.lr)
    trip = corpus.triples()
    for it in (1, 2):
        batch = trip[(it - 1) * w.batch : it * w.batch]
        res = O.train_step(st, lsh, batch, it, 0, w.n_out, cfg, mode="sequential")
        assert np.mean(res.losses) == pytest.approx(float(g[f"it{it}_loss"][0]), rel=1e-10)
        np.testing.assert_array_equal([tr.active.size for tr in res.traces], g[f"it{it}_active_sizes"])
        np.testing.assert_array_equal([int(tr.active.sum()) for tr in res.traces], g[f"it{it}_active_sum"])
        np.testing.assert_allclose([st.w2.sum(), np.abs(st.w2).sum()], g[f"it{it}_l1_wsum"], rtol=1e-10)
        np.testing.assert_allclose([st.w1t.sum(), np.abs(st.w1t).sum()], g[f"it{it}_l0_wsum"], rtol=1e-10)
        np.testing.assert_array_equal(st.steps2, g[f"it{it}_l1_steps"])
        np.testing.assert_array_equal(st.steps1, g[f"it{it}_l0_steps"])
    np.testing.assert_allclose(st.w2[:64], g["final_w2_head"], rtol=0, atol=1e-12)


def test_schedule_values():
    # reference tests/test_acceptance.py:275-290: lam=0.1 -> 50, 105, 166, 234
    s = O.Schedule(50, 0.1)
    got = []
    for _ in range(4):
        got.append(s.next_at)
        s.advance()
    assert got == [50, 105, 166, 234]
    s = O.Schedule(50, 0.0)
    assert [s.next_at, (s.advance(), s.next_at)[1]] == [50, 100]


def test_tiny_baseline_config_200_steps_and_precision_at_1(golden):
    """BASELINE configs[0] end to end: the reference's train_network
    (sequential, workers=1) for 200 steps -- four table rebuilds -- then P@1
    on a 4,000-example held-out stream with the evaluator's shared
    default_rng(seed).  The oracle reproduces every step's loss, the rebuild
    flags and the final P@1 exactly."""
    g = golden("tiny_run")
    w = TINY
    corpus = synthetic_corpus(w.corpus, 200 * w.batch, seed=0)
    held = synthetic_corpus(w.corpus, 4000, seed=1)
    np.testing.assert_array_equal(
        [corpus.x_idx.astype(np.int64).sum(), corpus.y_idx.astype(np.int64).sum(),
         held.x_idx.astype(np.int64).sum(), held.y_idx.astype(np.int64).sum()], g["corpus_check"])
    st = O.init_state(w.input_dim, w.hidden, w.n_out, seed=0)
    spec = O.LshSpec("simhash", w.k, w.l, w.cap, w.policy, strategy="vanilla", beta=w.beta)
    lsh = O.OutputLsh(spec, w.hidden, seed=0, n0=w.n0, lam=w.decay)
    lsh.build(st.w2)
    cfg = O.AdamCfg(lr=w.lr)
    trip = corpus.triples()
    order = np.random.default_rng((0, 0)).permutation(len(trip))  # reference data.py:118-123
    for it in range(1, 201):
        batch = [trip[i] for i in order[(it - 1) * w.batch : it * w.batch]]
        res = O.train_step(st, lsh, batch, it, 0, w.n_out, cfg, mode="sequential")
        assert np.mean(res.losses) == pytest.approx(float(g["seq_loss"][it - 1]), rel=1e-12, abs=0), it
        assert res.rebuilt == bool(g["seq_rebuilt"][it - 1])
        assert res.active_fraction == pytest.approx(float(g["seq_frac"][it - 1]), rel=1e-12)
    np.testing.assert_allclose(st.w2[:16], g["seq_final_w2_head"], rtol=0, atol=1e-12)
    rng = np.random.default_rng(0)
    p1 = np.mean([O.precision_at_k(O.predict_ranked(st, lsh, xi, xv, rng, w.n_out), y, 1)
                  for xi, xv, y in held.triples()])
    assert p1 == float(g["seq_p1"][0])
