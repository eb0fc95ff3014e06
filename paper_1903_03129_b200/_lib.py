"""ctypes binding of the C ABI in include/slide_b200.h.

The library (``libslide_b200.so``, built in-tree for sm_100a by
``__graft_entry__.build()`` / ``make -C paper_1903_03129_b200/csrc``) is the
only compute path: there is no CPU fallback.  Importing the package works
without it; the first call that needs it raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

LIB_PATH = os.environ.get("SLIDE_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                             "libslide_b200.so")

i64 = C.c_int64
u64 = C.c_uint64
vp = C.c_void_p
dbl = C.c_double


class NetDesc(C.Structure):
    _fields_ = [
        ("input_dim", i64), ("hidden", i64), ("hidden_pad", i64), ("n_out", i64), ("max_batch", i64),
        ("family", i64), ("k", i64), ("l", i64), ("key_bits", i64), ("capacity", i64), ("policy", i64),
        ("strategy", i64), ("beta", i64), ("min_freq", i64),
        ("sh_c", i64), ("sh_packed_host", vp),
        ("bin_size", i64), ("bins_per_perm", i64), ("n_perms", i64), ("bits", i64),
        ("dw_perms_host", vp), ("dw_donors_host", vp),
        ("lr", dbl), ("beta1", dbl), ("beta2", dbl), ("eps", dbl), ("seed", u64),
        ("w1t", vp), ("m1t", vp), ("v1t", vp), ("b1", vp), ("mb1", vp), ("vb1", vp), ("steps1", vp),
        ("w2", vp), ("m2", vp), ("v2", vp), ("b2", vp), ("mb2", vp), ("vb2", vp), ("steps2", vp),
        ("shard_rank", i64), ("shard_count", i64),
    ]


class Batch(C.Structure):
    _fields_ = [
        ("batch", i64), ("x_ptr", vp), ("x_idx", vp), ("x_val", vp), ("y_ptr", vp), ("y_idx", vp),
        ("x_ptr_host", vp), ("y_ptr_host", vp), ("rng_states", vp),
        ("forced_ptr", vp), ("forced_idx", vp), ("forced_ptr_host", vp),
    ]


# name -> (argtypes); every function returns int status
_SIGS = {
    "slide_create": [C.POINTER(NetDesc), vp, C.POINTER(vp)],
    "slide_destroy": [vp],
    "slide_set_stream": [vp, vp],
    "slide_simhash_keys": [vp, i64, i64, i64, i64, i64, i64, vp, vp, vp],
    "slide_dwta_keys": [vp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp],
    "slide_rebuild_tables": [vp, vp],
    "slide_relabel_units": [vp, vp],
    "slide_build_tables_from_keys": [vp, vp, i64, vp],
    "slide_clear_tables": [vp],
    "slide_tables_info": [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)],
    "slide_tables_export": [vp, vp, vp, vp, vp, vp],
    "slide_tables_probe": [vp, vp, i64, vp, vp],
    "slide_tables_probe_ids": [vp, vp, i64, vp, vp, vp],
    "slide_tables_load": [vp, vp, vp, vp, vp, i64, vp, i64, i64],
    "slide_tables_mask": [vp, u64],
    "slide_forward": [vp, C.POINTER(Batch), i64, i64, C.POINTER(i64)],
    "slide_backward": [vp, i64],
    "slide_train_batch": [vp, C.POINTER(Batch), i64, i64, vp, vp],
    "slide_graph_step": [vp, C.POINTER(Batch), i64, vp, vp],
    "slide_graph_step_async": [vp, C.POINTER(Batch), i64],
    "slide_graph_step_wait": [vp, vp, vp],
    "slide_read": [vp, i64, vp, i64, C.POINTER(i64)],
    "slide_topk": [vp, i64, vp, vp],
    "slide_query_union": [vp, vp, i64, i64, i64, vp, vp],
    "slide_write": [vp, i64, vp, i64],
    "slide_profile": [vp, i64],
    "slide_profile_read": [vp, vp, vp],
    "slide_launch_count": [vp],
    "slide_shard_hash_rows": [vp, vp],
    "slide_shard_forward": [vp, C.POINTER(Batch), i64, vp, vp],
    "slide_shard_hidden": [vp, C.POINTER(Batch), vp],
    "slide_shard_assemble": [vp, i64, vp],
    "slide_shard_select": [vp, C.POINTER(Batch), i64, vp],
    "slide_shard_build_local": [vp, C.POINTER(i64)],
    "slide_shard_tables_pack_size": [vp, C.POINTER(i64)],
    "slide_shard_tables_pack": [vp, vp],
    "slide_shard_tables_reconcile": [vp, vp, i64],
    "slide_shard_softmax_sum": [vp, vp, vp],
    "slide_shard_softmax_finish": [vp, vp, vp, vp],
    "slide_shard_hidden_grad": [vp, vp],
    "slide_shard_update": [vp, vp],
    "slide_sample_lists": [vp, vp, i64, i64, i64, i64, i64, vp, vp, C.POINTER(i64), C.POINTER(i64), vp, vp],
    "slide_pcg64_seed": [vp, i64, vp],
    "slide_pcg64_permutation": [vp, i64, vp],
    "slide_pcg64_choice": [vp, i64, i64, vp],
    "slide_mt19937_random": [vp, i64, vp],
}

EXPORTED = tuple(_SIGS) + ("slide_version", "slide_last_error")

_ERRORS = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: NotImplementedError, 5: RuntimeError}

_lock = threading.Lock()
_lib = None


def lib():
    """Load the CUDA library once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA library {LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
                )
            L = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = C.c_int
            L.slide_version.restype = C.c_char_p
            L.slide_last_error.restype = C.c_char_p
            _lib = L
    return _lib


def check(status: int):
    if status != 0:
        msg = lib().slide_last_error().decode()
        raise _ERRORS.get(status, RuntimeError)(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Device/host address of a torch tensor or numpy array (None for None)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


# --------------------------------------------------------------- host rng
def pcg64_seed(entropy) -> np.ndarray:
    ent = np.asarray([int(e) for e in entropy], dtype=np.uint64)
    st = np.zeros(6, dtype=np.uint64)
    call("slide_pcg64_seed", ent.ctypes.data, len(ent), st.ctypes.data)
    return st


def pcg64_state_from_generator(rng: np.random.Generator) -> np.ndarray:
    """numpy Generator(PCG64) state -> the 6 words the kernels use."""
    s = rng.bit_generator.state
    if s.get("bit_generator") != "PCG64":
        raise ValueError("device sampling emulates numpy PCG64 generators only")
    st, inc = int(s["state"]["state"]), int(s["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([st >> 64, st & m, inc >> 64, inc & m, int(s["has_uint32"]), int(s["uinteger"])],
                    dtype=np.uint64)


def pcg64_state_to_generator(words, rng: np.random.Generator) -> None:
    w = [int(x) for x in words]
    rng.bit_generator.state = {
        "bit_generator": "PCG64",
        "state": {"state": (w[0] << 64) | w[1], "inc": (w[2] << 64) | w[3]},
        "has_uint32": w[4],
        "uinteger": w[5],
    }


def mt_state_from_random(r) -> np.ndarray:
    st = r.getstate()
    return np.asarray(st[1], dtype=np.uint64)


def mt_state_to_random(words, r) -> None:
    version, _, gauss = r.getstate()
    r.setstate((version, tuple(int(x) for x in words), gauss))
