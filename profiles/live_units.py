"""Per-step hidden-layer statistics of a BASELINE workload on the device:
nonzero hidden units per sample, the batch live-unit count (checked against
the kernels' own live list, slide_read stage 13), pairs, unique rows and
the pairs-per-row distribution.  usage: python profiles/live_units.py
[workload] [steps] [corpus seed]"""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03129_b200.configs import WORKLOADS
from paper_1903_03129_b200.data import synthetic_corpus
import bench  # noqa: E402
wl = sys.argv[1] if len(sys.argv) > 1 else "wide_in"
w = WORKLOADS[wl]
torch.cuda.set_device(0)
net = bench.make_net(w, torch)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
corpus = synthetic_corpus(w.corpus, w.batch * n, seed=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
bs = bench.csr_batches(corpus, w.batch, n)
for it, b in enumerate(bs, 1):
    st = net.train_batch_csr(b, it, schedule="snapshot")
    if it in (1, 2, 5, 10, 20, 30, 40, 50, 60) or it % 10 == 0:
        h = net._read(0, w.batch * net.hidden_pad if hasattr(net, "hidden_pad") else w.batch * 128, np.float32).reshape(w.batch, -1)
        nz = h > 0
        C = nz.any(0).sum()
        offs = net._read(2, w.batch + 1, np.int32)
        rows = net._read(3, int(offs[-1]), np.int32)
        # pair-weighted on fraction
        per = nz.sum(1)
        pair_on = np.repeat(per, np.diff(offs)).mean() / h.shape[1]
        # per-row union of nz(h) columns
        slots = np.repeat(np.arange(w.batch), np.diff(offs))
        order = np.argsort(rows, kind="stable")
        r_s, s_s = rows[order], slots[order]
        starts = np.flatnonzero(np.r_[True, r_s[1:] != r_s[:-1]])
        uni = np.logical_or.reduceat(nz[s_s], starts, axis=0).sum(1)
        lens = np.diff(np.r_[starts, len(r_s)])
        lv = net._read(13, 1 + h.shape[1], np.int32)
        assert lv[0] == C and sorted(lv[1:1 + C]) == list(np.flatnonzero(nz.any(0))), (lv[:8], C)
        print(f"it {it} n_live {lv[0]} loss {st.loss:.3f} nnz(h) mean {per.mean():.1f} min {per.min()} max {per.max()} live cols {C} "
              f"pairs {len(rows)} rows {len(starts)} pair_on {pair_on:.3f} row-union mean {uni.mean():.1f} "
              f"len mean {lens.mean():.1f} p50 {np.median(lens):.0f} p99 {np.percentile(lens,99):.0f} max {lens.max()}", flush=True)
