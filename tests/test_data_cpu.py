"""Corpus ingestion and batching (SURVEY 8(f) F2, A16's batch order) against
the reference's own parser output, writer bytes and error messages
(tests/golden/data_io.npz, made by tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

from paper_1903_03129_b200 import Dataset, DatasetFormatError, SparseVector, batches, load_xc_file, save_xc_file
from paper_1903_03129_b200.data import batch_indices, corpus_from_examples, l2_normalize
from tests.golden.make_golden_data import XC_BAD, XC_GOOD


def _write(tmp_path, name, text):
    p = os.path.join(tmp_path, name)
    with open(p, "w", newline="") as fh:
        fh.write(text)
    return p


def test_xc_parse_matches_reference(golden, tmp_path):
    g = golden("data_io")
    ds = load_xc_file(_write(tmp_path, "good.txt", XC_GOOD))
    np.testing.assert_array_equal([len(ds.examples), ds.num_features, ds.num_labels], g["good_header"])
    for i, (x, labels) in enumerate(ds.examples):
        np.testing.assert_array_equal(x.indices, g[f"good_{i}_idx"])
        np.testing.assert_array_equal(x.values, g[f"good_{i}_val"])  # explicit zeros dropped
        assert sorted(labels) == g[f"good_{i}_labels"].tolist()
        assert isinstance(labels, frozenset)
    out = os.path.join(tmp_path, "saved.txt")
    save_xc_file(ds, out)
    assert open(out, "rb").read() == bytes(g["saved_text"])
    again = load_xc_file(out)
    assert len(again) == len(ds)
    for (x, y), (x2, y2) in zip(ds.examples, again.examples):
        np.testing.assert_array_equal(x.indices, x2.indices)
        np.testing.assert_array_equal(x.values, x2.values)
        assert y == y2


@pytest.mark.parametrize("name", sorted(XC_BAD))
def test_xc_errors_match_reference_messages(golden, tmp_path, name):
    g = golden("data_io")
    with pytest.raises(DatasetFormatError) as e:
        load_xc_file(_write(tmp_path, name + ".txt", XC_BAD[name]))
    assert str(e.value) == str(g["bad_" + name])
    assert isinstance(e.value, ValueError)


def _toy(n=11, dim=7, n_labels=5):
    rng = np.random.default_rng(4)
    ex = []
    for i in range(n):
        idx = np.sort(rng.choice(dim, size=3, replace=False))
        ex.append((SparseVector(idx, rng.random(3) + 0.5, dim), frozenset({i % n_labels})))
    return Dataset(ex, dim, n_labels)


def test_batches_follow_the_reference_epoch_shuffle():
    """batches(ds, B, seed) yields lists of the dataset's own examples in
    default_rng(seed).permutation(n) order, the last batch short
    (reference data.py:118-123); a CSR corpus yields the same rows."""
    ds = _toy()
    order = np.random.default_rng((0, 1)).permutation(11)
    got = list(batches(ds, 4, seed=(0, 1)))
    assert [len(b) for b in got] == [4, 4, 3]
    flat = [ex for b in got for ex in b]
    assert all(a is ds.examples[i] for a, i in zip(flat, order))
    np.testing.assert_array_equal(np.concatenate(list(batch_indices(11, 4, (0, 1)))), order)
    corpus = corpus_from_examples(ds.examples, 7, 5)
    subs = list(batches(corpus, 4, seed=(0, 1)))
    for sub, b in zip(subs, got):
        assert len(sub) == len(b)
        for j, (x, y) in enumerate(b):
            x2, y2 = sub.example(j)
            np.testing.assert_array_equal(x2.indices, x.indices)
            assert y2 == y
    with pytest.raises(ValueError):
        next(batches(ds, 0, seed=1))


def test_dataset_validate_and_normalize():
    ds = _toy()
    assert ds.validate() is ds
    with pytest.raises(ValueError, match="at least one"):
        Dataset([], 3, 3).validate()
    bad = Dataset([(SparseVector(np.array([1]), np.array([1.0]), 4), frozenset({9}))], 4, 5)
    with pytest.raises(ValueError, match="label"):
        bad.validate()
    nrm = l2_normalize(ds)
    for x, _ in nrm.examples:
        assert np.isclose(np.dot(x.values, x.values), 1.0)
