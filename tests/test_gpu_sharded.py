"""Column-sharded layer on the device (W2 rows, their tables
and W1 units split over the ranks): 2 and 4 ranks (processes) on one GPU
with host-mediated gloo collectives (no kernel waits on another rank),
checked against the unsharded device step from the same initial state --
identical active-set sizes, losses 1e-5, the assembled W1 / W2 1e-4; the
simhash case overflows its FIFO buckets, so the table exchange runs."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

D, H, N, B = 300, 128, 997, 16


def _shape(family):
    if family == "tiny":  # BASELINE configs[0]: 10,000 -> 128 -> 5,000, B = 128
        from paper_1903_03129_b200.configs import TINY

        return TINY.input_dim, TINY.hidden, TINY.n_out, TINY.batch
    return D, H, N, B


def _setup(family):
    from paper_1903_03129_b200 import LshLayerConfig, SamplerConfig, TrainConfig

    if family == "tiny":
        from paper_1903_03129_b200.configs import TINY as w

        cfg = TrainConfig(batch_size=w.batch, seed=0, learning_rate=w.lr, n0=2)
        return cfg, LshLayerConfig(w.family, k=w.k, l=w.l, capacity=w.cap, policy=w.policy,
                                   sampler=SamplerConfig(w.strategy, beta=w.beta))
    cfg = TrainConfig(batch_size=B, seed=5, learning_rate=1e-2, n0=2)
    if family == "simhash":
        spec = LshLayerConfig("simhash", k=4, l=8, capacity=16, sampler=SamplerConfig("vanilla", beta=40))
    else:
        spec = LshLayerConfig("dwta", k=3, l=6, capacity=32, policy="reservoir", wta_bin_size=8,
                              sampler=SamplerConfig("vanilla", beta=12))
    return cfg, spec


def _csrs(family="simhash"):
    from paper_1903_03129_b200.data import CorpusSpec, synthetic_corpus
    from paper_1903_03129_b200.network import HostCsr

    if family == "tiny":
        from paper_1903_03129_b200.configs import TINY

        bs = TINY.batch
        corpus = synthetic_corpus(TINY.corpus, 3 * bs, seed=9)
    else:
        bs = B
        corpus = synthetic_corpus(CorpusSpec(D, N, ("uniform", 3, 20), 1.1, ("uniform", 1, 4), 1.1, True), 3 * B, seed=9)
    out = []
    for s in range(3):
        sub = corpus.subset(np.arange(s * bs, (s + 1) * bs))
        out.append(HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx))
    return out


def _worker(rank, world, port, family, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_03129_b200 import SlideNetwork, sharded

        cfg, spec = _setup(family)
        d, h, n, _ = _shape(family)
        net = SlideNetwork(d, [h, n], cfg, lsh_layers={1: spec}, shard=(rank, world))
        losses, fracs = [], []
        for it, csr in enumerate(_csrs(family), start=1):
            st = net.train_batch_csr(csr, it, schedule="snapshot")
            losses.append(st.loss)
            fracs.append(st.active_fraction[1])
        w2 = sharded.all_gather_rows(net.w2.cpu(), n).numpy()
        v2 = sharded.all_gather_rows(net.v2.cpu(), n).numpy()
        w1 = sharded.all_gather_units(net.w1t.cpu()).numpy()
        q.put((rank, losses, fracs, w1, w2, v2))
    except BaseException as e:  # surface a rank's failure instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,world", [("simhash", 2), ("simhash", 4), ("dwta", 2), ("tiny", 2)])
def test_shards_match_one_gpu(family, world):
    from paper_1903_03129_b200 import SlideNetwork

    cfg, spec = _setup(family)
    d, h, n, _ = _shape(family)
    ref = SlideNetwork(d, [h, n], cfg, lsh_layers={1: spec})
    ref.use_graphs = False
    want_l, want_f = [], []
    for it, csr in enumerate(_csrs(family), start=1):
        st = ref.train_batch_csr(csr, it, schedule="snapshot")
        want_l.append(st.loss)
        want_f.append(st.active_fraction[1])
    cols = np.asarray(ref.unit_cols())  # the unsharded net may have renumbered its units
    w1_ref, w2_ref = ref.w1t.cpu().numpy()[:, cols], ref.w2.cpu().numpy()[:, cols]
    del ref
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, world, port, family, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    errs = [r for r in res if len(r) == 2]
    assert not errs, errs
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, losses, fracs, w1t, w2, v2 in res:
        np.testing.assert_allclose(losses, want_l, rtol=1e-5)
        np.testing.assert_allclose(fracs, want_f, rtol=0, atol=0)  # identical active sets
        np.testing.assert_allclose(w1t, w1_ref[:, :h], rtol=1e-4, atol=1e-6)
        np.testing.assert_allclose(w2[:, :h], w2_ref, rtol=1e-4, atol=1e-6)
