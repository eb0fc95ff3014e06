"""LSH hash families (drop-in for reference hashing.py).

Random state is drawn on the host with numpy exactly as the reference draws
it (SimHash hashing.py:132-140; permutations hashing.py:214-217), then
uploaded once; every code is computed by the sm_100a kernels in
``csrc/hashing.cu`` (queries and weight rows alike).  Inputs are taken as
float32: codes are bit-exact with the reference for float32-representable
inputs (the "identical weights" of the parity contract).

Supported on the device: simhash, dwta, wta with K*bits <= 32.  DOPH is out
of the hot-path scope and raises NotImplementedError.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sparse import SparseVector

_M64 = (1 << 64) - 1

HashCodes = np.ndarray


def _mix(a: int, b: int, c: int) -> int:
    """splitmix-style 64-bit mix of three integers (reference hashing.py:31-38)."""
    x = (a * 0x9E3779B97F4A7C15 + b * 0xBF58476D1CE4E5B9 + c * 0x94D049BB133111EB) & _M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _mix_many(a: int, b: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Vectorised _mix over uint64 arrays (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        x = (np.uint64(a * 0x9E3779B97F4A7C15 & _M64) + b.astype(np.uint64) * np.uint64(0xBF58476D1CE4E5B9)
             + c.astype(np.uint64) * np.uint64(0x94D049BB133111EB))
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def pack_subcodes(codes: np.ndarray, bits: int) -> np.ndarray:
    """Concatenate K sub-codes per row into one int64 key (hashing.py:41-48)."""
    codes = np.asarray(codes, dtype=np.int64)
    shifts = np.arange(codes.shape[-1], dtype=np.int64) * bits
    return (codes << shifts).sum(axis=-1, dtype=np.int64)


def _check_positive_int(value, name):
    if not isinstance(value, (int, np.integer)) or isinstance(value, bool) or value < 1:
        raise ValueError(f"{name} must be a positive integer, got {value!r}")
    return int(value)


@dataclass(frozen=True)
class HashFamilyConfig:
    """Same fields, defaults and validation as reference hashing.py:51-90."""

    family: str
    k_per_table: int
    num_tables: int
    dim: int
    simhash_sparsity: float = 1.0 / 3.0
    wta_bin_size: int = 8
    doph_top_k: int = 32
    seed: int = 0

    def validate(self) -> "HashFamilyConfig":
        if self.family not in ("simhash", "wta", "dwta", "doph"):
            raise ValueError(f"unknown hash family {self.family!r}")
        _check_positive_int(self.k_per_table, "k_per_table")
        _check_positive_int(self.num_tables, "num_tables")
        _check_positive_int(self.dim, "dim")
        if self.family == "simhash":
            s = float(self.simhash_sparsity)
            if not 0.0 < s <= 1.0:
                raise ValueError(f"simhash_sparsity must lie in (0, 1], got {self.simhash_sparsity!r}")
        if self.family in ("wta", "dwta"):
            _check_positive_int(self.wta_bin_size, "wta_bin_size")
            if self.wta_bin_size > self.dim:
                raise ValueError(f"wta_bin_size {self.wta_bin_size} exceeds dim {self.dim}")
        if self.family == "doph":
            _check_positive_int(self.doph_top_k, "doph_top_k")
        return self


class HashFamily:
    """Fixed random state from the seed; (K, L) keys computed on the device."""

    bits_per_code = 1

    def __init__(self, config: HashFamilyConfig):
        self.config = config.validate()
        self.dim = config.dim
        self.k = config.k_per_table
        self.l = config.num_tables
        self.n_codes = self.k * self.l
        self._dev = None

    def _check_key_width(self, bits_per_code: int):
        total = bits_per_code * self.k
        if total > 63:
            raise ValueError(
                f"key would need {total} bits ({self.k} sub-codes of {bits_per_code} bits); must fit in 63"
            )

    @property
    def key_bits(self) -> int:
        return self.bits_per_code * self.k

    # -- device ---------------------------------------------------------
    def _device_params(self):
        raise NotImplementedError

    def _keys_dev(self, x_dev, n: int, ld: int, keys_dev):
        raise NotImplementedError

    def _check_device_width(self):
        if self.key_bits > 32:
            raise NotImplementedError(f"device keys hold at most 32 bits, this family needs {self.key_bits}")

    def hash_dense_rows(self, w) -> np.ndarray:
        """(n, dim) dense rows (zeros = absent entries) -> (n, L) int64 keys."""
        import torch

        from . import _device

        self._check_device_width()
        w = np.asarray(w, dtype=np.float64)
        n = w.shape[0]
        if n == 0:
            return np.zeros((0, self.l), dtype=np.int64)
        x = _device.pad_rows(w, self.dim)
        keys = torch.empty((n, self.l), dtype=torch.int32, device=x.device)
        self._keys_dev(x, n, self.dim, keys)
        return keys.cpu().numpy().view(np.uint32).astype(np.int64)

    def hash(self, v: SparseVector) -> HashCodes:
        if v.dim != self.dim:
            raise ValueError(f"{type(self).__name__}: vector dim {v.dim} does not match expected {self.dim}")
        return self.hash_dense_rows(v.to_dense()[None, :])[0]

    def hash_batch(self, weights) -> np.ndarray:
        w = np.asarray(weights, dtype=np.float64)
        if w.ndim != 2 or w.shape[1] != self.dim:
            raise ValueError(f"expected weight matrix of shape (n, {self.dim}), got {w.shape}")
        return self.hash_dense_rows(w)


class SimHashFamily(HashFamily):
    """Sparse {+1, 0, -1} projections; bit = [projection . v > 0]
    (reference hashing.py:121-178)."""

    def __init__(self, config: HashFamilyConfig):
        super().__init__(config)
        self._check_key_width(1)
        rng = np.random.default_rng(config.seed)
        d = self.dim
        self.entries_per_proj = min(d, max(1, int(round(d * config.simhash_sparsity))))
        c = self.entries_per_proj
        idx = np.empty((self.n_codes, c), dtype=np.int64)
        for p in range(self.n_codes):
            idx[p] = np.sort(rng.choice(d, size=c, replace=False))
        self.proj_indices = idx
        self.proj_signs = rng.choice(np.array([-1.0, 1.0]), size=(self.n_codes, c))

    def packed(self) -> np.ndarray:
        if self.dim > 32767:
            raise NotImplementedError("device simhash supports dim <= 32767")
        return (self.proj_indices.astype(np.uint16) | ((self.proj_signs < 0).astype(np.uint16) << 15)).astype(np.uint16)

    def _device_params(self):
        if self._dev is None:
            from . import _device

            self._dev = _device.to_dev(self.packed().view(np.int16))
        return self._dev

    def _keys_dev(self, x_dev, n, ld, keys_dev):
        from . import _device

        p = self._device_params()
        _lib.call("slide_simhash_keys", x_dev.data_ptr(), n, ld, self.dim, self.k, self.l, self.entries_per_proj,
                  p.data_ptr(), keys_dev.data_ptr(), _device.stream_handle())

    def codes_from_dots(self, dots: np.ndarray) -> HashCodes:
        bits = (np.asarray(dots) > 0).astype(np.int64)  # sign(0) contributes bit 0
        return bits.reshape(self.l, self.k) @ (np.int64(1) << np.arange(self.k, dtype=np.int64))


class _PermutationBinFamily(HashFamily):
    """ceil(KLm/d) permutations cut into m-bins (reference hashing.py:196-217)."""

    dense_mode = 0

    def __init__(self, config: HashFamilyConfig):
        super().__init__(config)
        d, m = self.dim, config.wta_bin_size
        self.bin_size = m
        self.bins_per_perm = -(-d // m)
        self.n_perms = -(-(self.n_codes * m) // d)
        self.bits_per_code = max(1, math.ceil(math.log2(m))) if m > 1 else 1
        self._check_key_width(self.bits_per_code)
        rng = np.random.default_rng(config.seed)
        self._perms = np.stack([rng.permutation(d) for _ in range(self.n_perms)])
        self.inv_perms = np.argsort(self._perms, axis=1)
        self._densify_salt = _mix(config.seed & _M64, 0xD1F7, 0xA0B1)

    @property
    def perms(self):
        return self._perms

    @perms.setter
    def perms(self, value):
        self._perms = np.asarray(value)
        self._dev = None

    def donors(self) -> np.ndarray:
        """(K*L, 100): donor bin of attempt a+1 for empty bin g (hashing.py:225-226)."""
        g = np.repeat(np.arange(self.n_codes, dtype=np.uint64), 100)
        a = np.tile(np.arange(1, 101, dtype=np.uint64), self.n_codes)
        return (_mix_many(self._densify_salt, g, a) % np.uint64(self.n_codes)).astype(np.int16).reshape(self.n_codes, 100)

    def _device_params(self):
        if self._dev is None:
            from . import _device

            if self.dim > 32767 or self.bin_size > 256:
                raise NotImplementedError("device wta/dwta supports dim <= 32767 and bins <= 256")
            self._dev = (_device.to_dev(self._perms.astype(np.int16)), _device.to_dev(self.donors()))
        return self._dev

    def _keys_dev(self, x_dev, n, ld, keys_dev):
        from . import _device

        perms, donors = self._device_params()
        _lib.call("slide_dwta_keys", x_dev.data_ptr(), n, ld, self.dim, self.k, self.l, self.bin_size,
                  self.bins_per_perm, self.n_perms, self.bits_per_code, self.dense_mode, perms.data_ptr(),
                  donors.data_ptr(), keys_dev.data_ptr(), _device.stream_handle())


class WtaFamily(_PermutationBinFamily):
    """Winner-take-all over every dimension, zeros included (hashing.py:262-274)."""

    dense_mode = 1


class DwtaFamily(_PermutationBinFamily):
    """Densified WTA over the nonzeros (hashing.py:277-287)."""

    dense_mode = 0


_FAMILIES = {"simhash": SimHashFamily, "wta": WtaFamily, "dwta": DwtaFamily}


def new_hash_family(config: HashFamilyConfig) -> HashFamily:
    """Construct a family; equal configs give identical codes (hashing.py:353-356)."""
    config.validate()
    if config.family == "doph":
        raise NotImplementedError("doph is outside the B200 hot path (no BASELINE config uses it)")
    return _FAMILIES[config.family](config)


def _expect(family, cls, name):
    if not isinstance(family, cls):
        raise TypeError(f"{name} requires a {cls.__name__}, got {type(family).__name__}")
    return family


def simhash_codes(family: HashFamily, v: SparseVector) -> HashCodes:
    return _expect(family, SimHashFamily, "simhash_codes").hash(v)


def wta_codes(family: HashFamily, v: SparseVector) -> HashCodes:
    return _expect(family, WtaFamily, "wta_codes").hash(v)


def dwta_codes(family: HashFamily, v: SparseVector) -> HashCodes:
    return _expect(family, DwtaFamily, "dwta_codes").hash(v)
