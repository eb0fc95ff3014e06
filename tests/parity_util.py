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


def assert_state_close(net, st: O.NetState, rtol=1e-4, atol=1e-6, what="", adam_lr=None):
    """State after Adam steps, 1e-4 relative.  With ``adam_lr`` the weights'
    absolute floor is scaled by how far Adam can have moved them (each step
    moves a weight by at most ~lr): rtol * lr * steps of the row -- hot rows
    whose many +-lr moves cancel to a near-zero weight are compared against
    their movement, not their (tiny) value; the moments get an absolute floor of
    rtol times the array's largest moment."""
    l0, l1 = net.layers
    pairs = [("w1", np.asarray(l0.w), st.w1t.T, st.steps1), ("b1", np.asarray(l0.b), st.b1, st.steps1),
             ("m1", np.asarray(l0.adam_m), st.m1t.T, None), ("v1", np.asarray(l0.adam_v), st.v1t.T, None),
             ("w2", np.asarray(l1.w), st.w2, st.steps2), ("b2", np.asarray(l1.b), st.b2, st.steps2),
             ("m2", np.asarray(l1.adam_m), st.m2, None), ("v2", np.asarray(l1.adam_v), st.v2, None),
             ("mb2", np.asarray(l1.adam_mb), st.mb2, None), ("vb2", np.asarray(l1.adam_vb), st.vb2, None)]
    for name, got, want, steps in pairs:
        # v is ~g^2: compare relative to its own scale
        a = atol if not name.startswith("v") else max(atol * 1e-4, 1e-12)
        if adam_lr is not None and name[0] in "mv":
            # moments carry the gradients' cancellation error (the hidden
            # gradient sums delta over the active set, which sums to ~0):
            # floor at the array's scale
            a = max(a, rtol * float(np.max(np.abs(want), initial=0.0)))
        if adam_lr is not None and steps is not None:
            moved = rtol * adam_lr * np.asarray(steps, dtype=np.float64)
            a = np.maximum(a, moved.reshape((-1,) + (1,) * (np.ndim(want) - 1)))
            ok = np.abs(got - want) <= a + rtol * np.abs(want)
            assert ok.all(), f"{what} {name}: {np.count_nonzero(~ok)} off, max {np.abs(got - want)[~ok].max()}"
            continue
        np.testing.assert_allclose(got, want, rtol=rtol, atol=a, err_msg=f"{what} {name}")
    np.testing.assert_array_equal(np.asarray(l0.steps), st.steps1, err_msg=f"{what} steps1")
    np.testing.assert_array_equal(np.asarray(l1.steps), st.steps2, err_msg=f"{what} steps2")
