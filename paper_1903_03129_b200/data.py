"""Corpora, batches, the BASELINE synthetic corpora and P@k.

* ``Dataset`` / ``load_xc_file`` / ``save_xc_file`` are the reference's
  extreme-classification corpus carrier and text format (reference
  data.py:1-115): a header ``N d L`` then one ``l1,l2 i1:v1 i2:v2`` line per
  example; malformed content raises ``DatasetFormatError`` naming the line.
* ``batches`` restates the seeded epoch shuffle of the reference
  (reference data.py:118-123): ``default_rng(seed).permutation(n)`` cut into
  batches of examples, the last one possibly short; ``batch_indices`` is the
  same order as row indices (for CSR corpora).
* ``precision_at_k`` restates reference data.py:126-133.
* ``synthetic_corpus`` is the generator of SURVEY.md section 8(d) that stands
  in for Delicious-200K / Amazon-670K (not in the container): bounded Zipf
  feature and label ids mapped through fixed permutations, U(0,1] values,
  optional L2 normalisation.  One ``default_rng(seed)`` stream is consumed per
  sample in the order nnz count, features, values, label count, labels.

Corpora are held as CSR (``Corpus``) because that is what the device step
consumes; ``Corpus.example(i)`` gives the reference-style (SparseVector,
labels) pair.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import SparseVector


@dataclass
class Corpus:
    """CSR multi-label corpus.  Feature ids sorted per row, values float32
    (nonzero), labels sorted unique per row."""

    x_ptr: np.ndarray  # int64 (n+1,)
    x_idx: np.ndarray  # int32
    x_val: np.ndarray  # float32
    y_ptr: np.ndarray  # int64 (n+1,)
    y_idx: np.ndarray  # int32
    num_features: int
    num_labels: int

    def __len__(self) -> int:
        return len(self.x_ptr) - 1

    def example(self, i: int):
        a, b = self.x_ptr[i], self.x_ptr[i + 1]
        c, d = self.y_ptr[i], self.y_ptr[i + 1]
        x = SparseVector(self.x_idx[a:b].astype(np.int64), self.x_val[a:b].astype(np.float64), self.num_features)
        return x, frozenset(self.y_idx[c:d].tolist())

    def subset(self, rows) -> "Corpus":
        rows = np.asarray(rows, dtype=np.int64)
        xl = self.x_ptr[rows + 1] - self.x_ptr[rows]
        yl = self.y_ptr[rows + 1] - self.y_ptr[rows]
        x_ptr = np.zeros(rows.size + 1, dtype=np.int64)
        y_ptr = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(xl, out=x_ptr[1:])
        np.cumsum(yl, out=y_ptr[1:])
        xi = np.concatenate([np.arange(self.x_ptr[r], self.x_ptr[r + 1]) for r in rows]) if rows.size else np.empty(0, np.int64)
        yi = np.concatenate([np.arange(self.y_ptr[r], self.y_ptr[r + 1]) for r in rows]) if rows.size else np.empty(0, np.int64)
        return Corpus(x_ptr, self.x_idx[xi], self.x_val[xi], y_ptr, self.y_idx[yi], self.num_features, self.num_labels)

    def triples(self):
        """[(x_idx int64, x_val float64, labels sorted list)] for CPU checkers."""
        out = []
        for i in range(len(self)):
            a, b = self.x_ptr[i], self.x_ptr[i + 1]
            c, d = self.y_ptr[i], self.y_ptr[i + 1]
            out.append((self.x_idx[a:b].astype(np.int64), self.x_val[a:b].astype(np.float64),
                        self.y_idx[c:d].astype(np.int64).tolist()))
        return out


def corpus_from_examples(examples, num_features: int, num_labels: int) -> Corpus:
    """Pack (SparseVector, labels) pairs into CSR (values rounded to float32)."""
    x_ptr = [0]
    y_ptr = [0]
    xi, xv, yi = [], [], []
    for x, labels in examples:
        if x.dim != num_features:
            raise ValueError(f"input dim {x.dim} != {num_features}")
        xi.append(np.asarray(x.indices, dtype=np.int32))
        xv.append(np.asarray(x.values, dtype=np.float32))
        lab = np.array(sorted(set(int(l) for l in labels)), dtype=np.int32)
        if lab.size and (lab[0] < 0 or lab[-1] >= num_labels):
            raise ValueError(f"label outside [0, {num_labels})")
        yi.append(lab)
        x_ptr.append(x_ptr[-1] + len(x.indices))
        y_ptr.append(y_ptr[-1] + lab.size)
    cat = lambda parts, dt: np.concatenate(parts).astype(dt) if parts else np.empty(0, dt)
    return Corpus(np.asarray(x_ptr, np.int64), cat(xi, np.int32), cat(xv, np.float32),
                  np.asarray(y_ptr, np.int64), cat(yi, np.int32), num_features, num_labels)


class DatasetFormatError(ValueError):
    """Malformed corpus file; the message carries the offending line number
    (reference data.py:20-21)."""


@dataclass
class Dataset:
    """(SparseVector, frozenset labels) examples plus the feature and label
    dimensions (reference data.py:24-47)."""

    examples: list
    num_features: int
    num_labels: int

    def __len__(self) -> int:
        return len(self.examples)

    def validate(self) -> "Dataset":
        if not self.examples:
            raise ValueError("dataset must contain at least one example")
        for x, labels in self.examples:
            x.validate()
            if x.dim != self.num_features:
                raise ValueError("feature dim mismatch")
            if labels and (min(labels) < 0 or max(labels) >= self.num_labels):
                raise ValueError("label out of range")
        return self

    def to_corpus(self) -> "Corpus":
        """CSR form (float32 values) -- what the device step consumes."""
        return corpus_from_examples(self.examples, self.num_features, self.num_labels)


def _bad(line_no: int, msg: str):
    raise DatasetFormatError(f"line {line_no}: {msg}")


def _parse_labels(tok: str, line_no: int, n_labels: int) -> frozenset:
    if not tok:
        return frozenset()
    if ":" in tok:
        _bad(line_no, "feature token found where labels belong")
    out = set()
    for part in tok.split(","):
        try:
            lab = int(part)
        except ValueError:
            _bad(line_no, f"non-integer label {part!r}")
        if lab < 0 or lab >= n_labels:
            _bad(line_no, f"label {lab} outside [0, {n_labels})")
        out.add(lab)
    return frozenset(out)


def _parse_features(toks, line_no: int, dim: int) -> SparseVector:
    pairs = []
    for tok in toks:
        i_s, colon, v_s = tok.partition(":")
        if not colon:
            _bad(line_no, f"feature token {tok!r} is not 'index:value'")
        try:
            i, v = int(i_s), float(v_s)
        except ValueError:
            _bad(line_no, f"non-numeric feature token {tok!r}")
        if not np.isfinite(v):
            _bad(line_no, f"non-finite feature value {tok!r}")
        if i < 0 or i >= dim:
            _bad(line_no, f"feature index {i} outside [0, {dim})")
        if v != 0.0:  # explicit zeros are dropped on parse
            pairs.append((i, v))
    return SparseVector.from_pairs(pairs, dim)


def load_xc_file(path) -> Dataset:
    """Parse an extreme-classification corpus file (reference data.py:51-103):
    header ``N d L`` (positive integers), then exactly N example lines
    ``labels features`` -- labels comma-separated (may be empty), features
    ``index:value`` tokens (may be absent); trailing blank lines are allowed.
    Errors raise ``DatasetFormatError`` with the 1-based line number."""
    with open(path, "r", encoding="utf-8", newline=None) as fh:
        head = fh.readline()
        if not head.strip():
            _bad(1, "missing header 'N d L'")
        fields = head.split()
        if len(fields) != 3:
            _bad(1, f"header must be 'N d L', got {head.strip()!r}")
        try:
            n, dim, n_labels = (int(f) for f in fields)
        except ValueError:
            _bad(1, f"non-integer header field in {head.strip()!r}")
        if min(n, dim, n_labels) < 1:
            _bad(1, "header counts must be positive")
        examples = []
        line_no = 1
        for line_no, line in enumerate(fh, start=2):
            line = line.rstrip("\r\n")
            if len(examples) == n:
                if not line.strip():
                    continue
                _bad(line_no, f"more than the declared {n} examples")
            lab_tok, _, rest = line.partition(" ")
            labels = _parse_labels(lab_tok, line_no, n_labels)
            examples.append((_parse_features(rest.split(), line_no, dim), labels))
        if len(examples) != n:
            _bad(line_no if examples else 1, f"expected {n} examples, found {len(examples)}")
    return Dataset(examples, dim, n_labels)


def save_xc_file(ds: Dataset, path) -> None:
    """Write ``ds`` in the format ``load_xc_file`` reads (reference
    data.py:106-115); values are written with ``repr`` so a reload is equal."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"{len(ds.examples)} {ds.num_features} {ds.num_labels}\n")
        for x, labels in ds.examples:
            head = ",".join(str(v) for v in sorted(labels))
            feats = " ".join(f"{i}:{v!r}" for i, v in zip(x.indices.tolist(), x.values.tolist()))
            fh.write((f"{head} {feats}".rstrip() if feats else head) + "\n")


def l2_normalize(ds: Dataset) -> Dataset:
    """Every example's features scaled to unit L2 norm (reference data.py:136-141)."""
    return Dataset([(x.l2_normalized(), labels) for x, labels in ds.examples], ds.num_features, ds.num_labels)


def _check_batch_size(batch_size):
    if not isinstance(batch_size, (int, np.integer)) or isinstance(batch_size, bool) or batch_size < 1:
        raise ValueError(f"batch_size must be a positive integer, got {batch_size!r}")


def batch_indices(n_examples: int, batch_size: int, seed):
    """Row-index batches of one epoch in ``batches``' order (CSR corpora)."""
    _check_batch_size(batch_size)
    order = np.random.default_rng(seed).permutation(n_examples)
    for lo in range(0, len(order), batch_size):
        yield order[lo : lo + batch_size]


def batches(ds, batch_size: int, seed):
    """Seeded epoch shuffle cut into batches of examples, the last possibly
    short (reference data.py:118-123).  ``ds`` is a ``Dataset`` (lists of
    (SparseVector, labels) pairs, as the reference yields) or a CSR
    ``Corpus`` (batches are sub-corpora)."""
    if isinstance(ds, Corpus):
        for rows in batch_indices(len(ds), batch_size, seed):
            yield ds.subset(rows)
        return
    for rows in batch_indices(len(ds.examples), batch_size, seed):
        yield [ds.examples[i] for i in rows]


def score_precision_at_k(net, examples, k: int = 1, seed: int = 0) -> float:
    """Mean P@k over (x, labels) examples, ranked on the device with one
    ``default_rng(seed)`` shared across the queries in order -- the
    evaluator's semantics (reference estimator.py:203-223, ``score``; the
    facade's l2 normalisation of inputs is the caller's)."""
    rng = np.random.default_rng(seed)
    ranked = net.predict_batch([x for x, _ in examples], topn=k, rng=rng)
    return float(np.mean([precision_at_k(r, y, k) for r, (_, y) in zip(ranked, examples)])) if examples else 0.0


def precision_at_k(ranked, truth, k: int) -> float:
    """|top-k of ranked that are true| / k; an empty ranking scores 0
    (reference data.py:126-133)."""
    if not isinstance(k, (int, np.integer)) or k < 1:
        raise ValueError(f"k must be a positive integer, got {k!r}")
    top = list(ranked[:k])
    if not top:
        return 0.0
    truth = set(truth)
    return sum(1 for r in top if r in truth) / k


# ---------------------------------------------------------------------------
# SURVEY 8(d) synthetic generator
# ---------------------------------------------------------------------------


class _Zipf:
    """Bounded Zipf over ranks [0, n): P(r) ~ (r+1)^-a, inverse-CDF sampling,
    rank -> id through ``perm``."""

    def __init__(self, n: int, a: float, perm: np.ndarray):
        w = np.arange(1, n + 1, dtype=np.float64) ** (-a)
        self.cdf = np.cumsum(w) / w.sum()
        self.n = n
        self.perm = perm

    def distinct(self, rng, count: int) -> np.ndarray:
        count = min(count, self.n)
        got: list = []
        seen: set = set()
        while len(got) < count:
            u = rng.random(2 * (count - len(got)) + 8)
            r = np.minimum(np.searchsorted(self.cdf, u, side="right"), self.n - 1)
            for v in r.tolist():
                if v not in seen:
                    seen.add(v)
                    got.append(v)
        return self.perm[np.asarray(got[:count], dtype=np.int64)]


@dataclass(frozen=True)
class CorpusSpec:
    num_features: int
    num_labels: int
    nnz: tuple  # ("uniform", lo, hi) or ("poisson", mean)
    feat_zipf: float
    labels: tuple  # ("uniform", lo, hi) or ("poisson", mean)
    label_zipf: float
    l2_normalize: bool


def _count(rng, spec: tuple) -> int:
    if spec[0] == "uniform":
        return int(rng.integers(spec[1], spec[2] + 1))
    return max(1, int(rng.poisson(spec[1])))


def synthetic_corpus(spec: CorpusSpec, n: int, seed: int = 0) -> Corpus:
    """SURVEY.md 8(d) procedure, consuming one default_rng(seed) stream."""
    fz = _Zipf(spec.num_features, spec.feat_zipf, np.random.default_rng(101).permutation(spec.num_features))
    lz = _Zipf(spec.num_labels, spec.label_zipf, np.random.default_rng(102).permutation(spec.num_labels))
    rng = np.random.default_rng(seed)
    x_ptr = np.zeros(n + 1, dtype=np.int64)
    y_ptr = np.zeros(n + 1, dtype=np.int64)
    xi, xv, yi = [], [], []
    for s in range(n):
        c = _count(rng, spec.nnz)
        f = np.sort(fz.distinct(rng, c))
        v = 1.0 - rng.random(f.size)
        if spec.l2_normalize:
            v = v / np.sqrt(np.dot(v, v))
        cl = _count(rng, spec.labels)
        lab = np.sort(lz.distinct(rng, cl))
        xi.append(f.astype(np.int32))
        xv.append(v.astype(np.float32))
        yi.append(lab.astype(np.int32))
        x_ptr[s + 1] = x_ptr[s] + f.size
        y_ptr[s + 1] = y_ptr[s] + lab.size
    return Corpus(x_ptr, np.concatenate(xi), np.concatenate(xv), y_ptr, np.concatenate(yi),
                  spec.num_features, spec.num_labels)
