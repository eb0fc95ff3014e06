"""A learnable synthetic corpus for the P@1-after-N-steps criterion (test
data, not product).

The BASELINE tiny corpus draws labels independently of the features, so its
P@1 only measures which frequent labels a trajectory happens to rank first:
fp32 rounding alone moves it by several points (tests/golden/p1_spread.npz).
Here every sample belongs to a class c (Zipf(1.1) over the label space); its
features are 8 of the class's 12 signature features (fixed per class) plus
background features (the tiny corpus's Zipf), and its labels are c plus 0-2
Zipf labels -- a signal the network learns, so P@1 is a stable function of
the training algorithm.  One default_rng(seed) stream, consumed per sample.
"""

from __future__ import annotations

import numpy as np

from paper_1903_03129_b200.data import Corpus, _Zipf


def learnable_corpus(num_features: int, num_labels: int, n: int, seed: int) -> Corpus:
    sig_rng = np.random.default_rng(4242)
    signatures = np.stack([sig_rng.choice(num_features, 12, replace=False) for _ in range(num_labels)])
    fz = _Zipf(num_features, 1.1, np.random.default_rng(101).permutation(num_features))
    lz = _Zipf(num_labels, 1.1, np.random.default_rng(102).permutation(num_labels))
    rng = np.random.default_rng(seed)
    x_ptr = np.zeros(n + 1, dtype=np.int64)
    y_ptr = np.zeros(n + 1, dtype=np.int64)
    xi, xv, yi = [], [], []
    for s in range(n):
        c = int(lz.distinct(rng, 1)[0])
        sig = rng.choice(signatures[c], 8, replace=False)
        bg = fz.distinct(rng, int(rng.integers(10, 31)))
        f = np.unique(np.concatenate([sig, bg]))
        v = 1.0 - rng.random(f.size)
        extra = lz.distinct(rng, int(rng.integers(0, 3)))
        lab = np.unique(np.concatenate([[c], extra]).astype(np.int64))
        xi.append(f.astype(np.int32))
        xv.append(v.astype(np.float32))
        yi.append(lab.astype(np.int32))
        x_ptr[s + 1] = x_ptr[s] + f.size
        y_ptr[s + 1] = y_ptr[s] + lab.size
    return Corpus(x_ptr, np.concatenate(xi), np.concatenate(xv), y_ptr, np.concatenate(yi), num_features, num_labels)
