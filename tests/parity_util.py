"""Helpers that hand device state to the CPU oracle (test infrastructure)."""

from __future__ import annotations

import numpy as np

from oracle import slide_oracle as O


def oracle_state_from_net(net) -> O.NetState:
    """f64 copy of the device's f32 state: 'identical weights' for parity."""
    l0, l1 = net.layers
    return O.NetState(
        np.ascontiguousarray(np.asarray(l0.w).T), np.asarray(l0.b).copy(),
        np.ascontiguousarray(np.asarray(l0.adam_m).T), np.ascontiguousarray(np.asarray(l0.adam_v).T),
        np.asarray(l0.adam_mb).copy(), np.asarray(l0.adam_vb).copy(), np.asarray(l0.steps).astype(np.int64),
        np.asarray(l1.w).copy(), np.asarray(l1.b).copy(), np.asarray(l1.adam_m).copy(), np.asarray(l1.adam_v).copy(),
        np.asarray(l1.adam_mb).copy(), np.asarray(l1.adam_vb).copy(), np.asarray(l1.steps).astype(np.int64),
    )


def oracle_spec(spec) -> O.LshSpec:
    return O.LshSpec(spec.family, spec.k, spec.l, spec.capacity, spec.policy, spec.simhash_sparsity,
                     spec.wta_bin_size, spec.sampler.strategy, spec.sampler.beta, spec.sampler.min_freq)


def oracle_lsh_from_net(net, spec, st=None) -> O.OutputLsh:
    """Oracle tables built from the net's (f32) W2 with a fresh reservoir
    stream -- the same inserts and draws the device made at construction."""
    cfg = net.cfg
    lsh = O.OutputLsh(oracle_spec(spec), net.hidden, cfg.seed, cfg.n0, cfg.decay)
    lsh.build((st or oracle_state_from_net(net)).w2)
    return lsh


def assert_state_close(net, st: O.NetState, rtol=1e-4, atol=1e-6, what=""):
    l0, l1 = net.layers
    pairs = [("w1", np.asarray(l0.w), st.w1t.T), ("b1", np.asarray(l0.b), st.b1),
             ("m1", np.asarray(l0.adam_m), st.m1t.T), ("v1", np.asarray(l0.adam_v), st.v1t.T),
             ("w2", np.asarray(l1.w), st.w2), ("b2", np.asarray(l1.b), st.b2),
             ("m2", np.asarray(l1.adam_m), st.m2), ("v2", np.asarray(l1.adam_v), st.v2),
             ("mb2", np.asarray(l1.adam_mb), st.mb2), ("vb2", np.asarray(l1.adam_vb), st.vb2)]
    for name, got, want in pairs:
        # v is ~g^2: compare relative to its own scale
        a = atol if not name.startswith("v") else max(atol * 1e-4, 1e-12)
        np.testing.assert_allclose(got, want, rtol=rtol, atol=a, err_msg=f"{what} {name}")
    np.testing.assert_array_equal(np.asarray(l0.steps), st.steps1, err_msg=f"{what} steps1")
    np.testing.assert_array_equal(np.asarray(l1.steps), st.steps2, err_msg=f"{what} steps2")
