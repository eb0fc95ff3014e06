"""Full-size (BASELINE wide-in) checks through size-independent properties.

At 205k output rows the CPU oracle cannot replay whole steps in test time, so
these pin the device path with properties that hold at any size: the
tensor-core rebuild hash equals the CUDA-core hash and the oracle's keys bit
for bit, the built FIFO tables hold exactly the last `cap` ids of every key,
graph-replayed steps are bit-identical to eager ones, and training lowers the
loss.
"""

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
    TrainConfig,
    new_hash_family,
)
from paper_1903_03129_b200.configs import WIDE_IN as W  # noqa: E402
from paper_1903_03129_b200.network import HostCsr  # noqa: E402


@pytest.fixture(scope="module")
def wide_rows():
    rng = np.random.default_rng(11)
    bound = 1.0 / np.sqrt(W.hidden)
    return rng.uniform(-bound, bound, size=(W.n_out, W.hidden)).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def wide_family():
    return new_hash_family(HashFamilyConfig("simhash", W.k, W.l, W.hidden, seed=7919))


def test_rebuild_keys_tensor_core_equal_cuda_core_and_oracle(wide_rows, wide_family):
    keys_tc = wide_family.hash_batch(wide_rows)  # >= 148 x 128 rows: the tcgen05 path
    keys_cc = np.concatenate([wide_family.hash_batch(wide_rows[i : i + 9000])  # CUDA-core path
                              for i in range(0, W.n_out, 9000)])
    np.testing.assert_array_equal(keys_tc, keys_cc)
    params = O.SimHashParams(W.hidden, W.k, W.l, wide_family.proj_indices, wide_family.proj_signs)
    sample = np.random.default_rng(3).choice(W.n_out, 20000, replace=False)
    np.testing.assert_array_equal(keys_tc[sample], O.simhash_keys(params, wide_rows[sample]))


def test_fifo_tables_hold_the_last_cap_ids_of_every_key(wide_rows, wide_family):
    tbl = LshTables(wide_family, policy="fifo", capacity=W.cap, seed=1)
    tbl.build(wide_rows)
    keys = wide_family.hash_batch(wide_rows)
    ids = np.arange(W.n_out)
    for t in (0, 17, W.l - 1):
        col = keys[:, t]
        order = np.argsort(col, kind="stable")  # ids ascending within each key
        uk, first, count = np.unique(col[order], return_index=True, return_counts=True)
        view = tbl.tables[t]
        assert set(view.keys()) == set(uk.tolist())
        for k, f, c in zip(uk, first, count):
            b = view[int(k)]
            assert b.count == c
            assert sorted(b.slots) == ids[order[f + max(0, c - W.cap) : f + c]].tolist()


def _batches(n_steps, seed=1000):
    from paper_1903_03129_b200.data import synthetic_corpus

    corpus = synthetic_corpus(W.corpus, n_steps * W.batch, seed=seed)
    out = []
    for s in range(n_steps):
        sub = corpus.subset(np.arange(s * W.batch, (s + 1) * W.batch))
        out.append(HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx))
    return out


def _net():
    cfg = TrainConfig(batch_size=W.batch, learning_rate=W.lr, n0=W.n0, decay=W.decay, seed=0)
    spec = LshLayerConfig(W.family, k=W.k, l=W.l, capacity=W.cap, policy=W.policy,
                          sampler=SamplerConfig(W.strategy, beta=W.beta))
    return SlideNetwork(W.input_dim, [W.hidden, W.n_out], cfg, lsh_layers={1: spec})


def test_full_size_graph_steps_equal_eager_steps():
    batches = _batches(3)

    def run(graphs):
        net = _net()
        net.use_graphs = graphs
        losses = [net.train_batch_csr(b, it, schedule="snapshot").loss for it, b in enumerate(batches, start=1)]
        out = (losses, net.w2.cpu().numpy(), net.w1t.cpu().numpy(), net.m2.cpu().numpy())
        del net
        torch.cuda.empty_cache()
        return out

    a, b = run(True), run(False)
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


def test_full_size_training_lowers_the_loss_and_keeps_sets_bounded():
    net = _net()
    losses, fracs = [], []
    for it, b in enumerate(_batches(30, seed=77), start=1):
        st = net.train_batch_csr(b, it, schedule="snapshot")
        assert np.isfinite(st.loss)
        losses.append(st.loss)
        fracs.append(st.active_fraction[1])
    assert np.mean(losses[-5:]) < np.mean(losses[:5])
    # full-union vanilla: |A_i| <= L * cap + |Y_i|
    assert max(fracs) * W.n_out <= W.l * W.cap + 400


def test_graph_steps_across_a_rebuild_that_moves_table_buffers():
    """Scaled-family shape (DWTA K8 L64, H=256, B=1024) at 1M rows with a
    rebuild after every other step: a rebuild can need more bucket runs than
    any earlier build, which moves the table buffers the captured step graph
    points into; the graph must be re-captured (it used to replay stale
    pointers: illegal address).  Graph steps stay bit-identical to eager."""
    import dataclasses

    from paper_1903_03129_b200.configs import SCALED
    from paper_1903_03129_b200.data import synthetic_corpus

    w = dataclasses.replace(SCALED, n_out=1_000_000, n0=2)
    corpus = synthetic_corpus(dataclasses.replace(w.corpus, num_labels=w.n_out), 4 * w.batch, seed=0)
    batches = []
    for s in range(4):
        sub = corpus.subset(np.arange(s * w.batch, (s + 1) * w.batch))
        batches.append(HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx))

    def run(graphs):
        cfg = TrainConfig(batch_size=w.batch, learning_rate=w.lr, n0=w.n0, seed=0)
        spec = LshLayerConfig(w.family, k=w.k, l=w.l, capacity=w.cap, policy=w.policy, wta_bin_size=w.bin_size,
                              sampler=SamplerConfig(w.strategy, beta=w.beta))
        net = SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
        net.use_graphs = graphs
        stats = [net.train_batch_csr(b, it, schedule="snapshot") for it, b in enumerate(batches, start=1)]
        out = ([s.loss for s in stats], [s.rebuilt for s in stats], net.w2.cpu().numpy(), net.v2.cpu().numpy())
        del net
        torch.cuda.empty_cache()
        return out

    a, b = run(True), run(False)
    assert a[0] == b[0] and a[1] == b[1]
    assert sum(bool(r) for r in a[1]) >= 2
    for x, y in zip(a[2:], b[2:]):
        np.testing.assert_array_equal(x, y)
