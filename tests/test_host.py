"""CPU-only checks: the C-ABI library loads and exports its header, the host
random streams match the golden numpy / CPython streams, and the host-side
logic mirrors the reference's validation and schedule."""

import os
import random
import re

import numpy as np
import pytest

from paper_1903_03129_b200 import _lib
from paper_1903_03129_b200.hashing import HashFamilyConfig, _mix, _mix_many, pack_subcodes
from paper_1903_03129_b200.network import LshLayerConfig, TrainConfig
from paper_1903_03129_b200.samplers import SamplerConfig
from paper_1903_03129_b200.tables import RawCandidates, RebuildSchedule

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slide_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(slide_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)
    assert b"sm_100a" in L.slide_version()


def test_pcg64_seed_matches_numpy():
    for ent in [(0, 1, 0), (0, 5, 3), (7, 123456, 255), (2**33 + 5, 2, 0), (12345678901234,)]:
        st = _lib.pcg64_seed(ent)
        ref = _lib.pcg64_state_from_generator(np.random.default_rng(ent))
        np.testing.assert_array_equal(st, ref)


def test_pcg64_permutations_match_golden(golden):
    g = golden("rng_streams")
    for L in (20, 50, 64):
        for row, ent in enumerate(g["ents"].tolist()):
            st = _lib.pcg64_seed(ent)
            out = np.empty(L, dtype=np.int64)
            _lib.call("slide_pcg64_permutation", st.ctypes.data, L, out.ctypes.data)
            np.testing.assert_array_equal(out, g[f"perm{L}"][row])


def test_pcg64_choice_matches_golden(golden):
    g = golden("rng_streams")
    off = 0
    for case, (s0, s1, s2, pop, size, pre) in enumerate(g["choice_cases"].tolist()):
        st = _lib.pcg64_seed((s0, s1, s2))
        if pre:
            tmp = np.empty(pre, dtype=np.int64)
            _lib.call("slide_pcg64_permutation", st.ctypes.data, pre, tmp.ctypes.data)
        out = np.empty(size, dtype=np.int64)
        _lib.call("slide_pcg64_choice", st.ctypes.data, pop, size, out.ctypes.data)
        n = g["choice_lens"][case]
        np.testing.assert_array_equal(out, g["choice_vals"][off : off + n], err_msg=f"case {case} pop {pop} size {size}")
        off += n
        # the generator state after the call matches numpy's as well
        r = np.random.default_rng((s0, s1, s2))
        if pre:
            r.permutation(pre)
        r.choice(pop, size=size, replace=False)
        np.testing.assert_array_equal(st, _lib.pcg64_state_from_generator(r))


def test_pcg64_state_roundtrip_through_generator():
    r = np.random.default_rng(42)
    r.random(3)
    r.integers(0, 10, size=3)  # leaves a buffered uint32
    st = _lib.pcg64_state_from_generator(r)
    r2 = np.random.default_rng(0)
    _lib.pcg64_state_to_generator(st, r2)
    assert r.random() == r2.random()


def test_mt19937_matches_cpython(golden):
    g = golden("mt19937")
    for k in range(len(g["seeds"])):
        st = g["states"][k].astype(np.uint64).copy()
        out = np.empty(2000)
        _lib.call("slide_mt19937_random", st.ctypes.data, 2000, out.ctypes.data)
        np.testing.assert_array_equal(out, g["draws"][k])
        r = random.Random(int(g["seeds"][k]))
        for _ in range(2000):
            r.random()
        np.testing.assert_array_equal(st, np.asarray(r.getstate()[1], dtype=np.uint64))


def test_mix_and_packing():
    assert _mix(7919 * 2, 0xD1F7, 0xA0B1) == 0xF2163B224F9E990E
    g = np.arange(50, dtype=np.uint64)
    a = np.full(50, 3, dtype=np.uint64)
    np.testing.assert_array_equal(_mix_many(123, g, a), np.array([_mix(123, int(x), 3) for x in g], dtype=np.uint64))
    codes = np.array([[1, 2, 3], [7, 0, 5]])
    np.testing.assert_array_equal(pack_subcodes(codes, 3), [1 + (2 << 3) + (3 << 6), 7 + (5 << 6)])


def test_config_validation_messages():
    with pytest.raises(ValueError, match="63"):
        from paper_1903_03129_b200.hashing import SimHashFamily

        SimHashFamily(HashFamilyConfig("simhash", 64, 1, 128))
    with pytest.raises(ValueError):
        HashFamilyConfig("dwta", 2, 2, 8, wta_bin_size=9).validate()
    with pytest.raises(ValueError):
        HashFamilyConfig("bogus", 2, 2, 8).validate()
    with pytest.raises(ValueError):
        TrainConfig(learning_rate=0).validate()
    with pytest.raises(ValueError):
        SamplerConfig("vanilla", beta=0).validate()
    with pytest.raises(ValueError):
        SamplerConfig("hard_threshold", min_freq=5).validate(num_tables=3)
    assert LshLayerConfig().sampler == SamplerConfig()


def test_schedule_values():
    s = RebuildSchedule(50, 0.1)
    got = []
    for _ in range(4):
        got.append(s.next_at)
        s.advance()
    assert got == [50, 105, 166, 234]
    with pytest.raises(ValueError):
        RebuildSchedule(50, -1.0)


def test_reference_arm_parallel_step_equals_serial_snapshot():
    """bench.py --impl reference runs the reference path on every host core
    (slots' forward/backward in worker processes, the Adam updates
    partitioned by row); its state after two steps equals the serial
    snapshot oracle bit for bit."""
    import multiprocessing as mp

    import bench
    from oracle import slide_oracle as O
    from paper_1903_03129_b200.data import CorpusSpec, synthetic_corpus

    D, H, N = 300, 16, 120
    spec = CorpusSpec(D, N, ("uniform", 3, 12), 1.1, ("uniform", 1, 3), 1.1, True)
    trip = synthetic_corpus(spec, 24, seed=5).triples()
    lspec = O.LshSpec("simhash", 3, 6, 8, "fifo", strategy="vanilla", beta=20)
    cfg = O.AdamCfg(lr=1e-2)

    def fresh():
        st = O.init_state(D, H, N, seed=3)
        lsh = O.OutputLsh(lspec, H, 0, 50, 0.0)
        lsh.build(st.w2)
        return st, lsh

    want, lw = fresh()
    for it in (1, 2):
        O.train_step(want, lw, trip[(it - 1) * 12 : it * 12], it, 0, N, cfg, mode="snapshot")
    st, lsh = fresh()
    st = bench._shared_state(st)
    bench._REF.update(st=st, lsh=lsh, n_out=N)
    ctx = mp.get_context("fork")
    with ctx.Pool(3) as pool:
        for it in (1, 2):
            bench.reference_parallel_step(st, lsh, trip[(it - 1) * 12 : it * 12], it, cfg, 3, pool, ctx)
    for name in ("w1t", "m1t", "v1t", "b1", "mb1", "vb1", "steps1", "w2", "m2", "v2", "b2", "mb2", "vb2", "steps2"):
        np.testing.assert_array_equal(getattr(st, name), getattr(want, name), err_msg=name)
