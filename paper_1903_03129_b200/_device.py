"""Device plumbing: torch owns device memory and streams, the C ABI computes."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1903_03129_b200 computes on a CUDA device (B200); none is visible")
    _lib.lib()  # fail loudly if the extension is missing
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_dev(a, dtype=None) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


def pad_rows(w: np.ndarray, ld: int) -> torch.Tensor:
    """(n, d) float -> device (n, ld) float32, zero padded."""
    w = np.asarray(w)
    n, d = w.shape
    out = torch.zeros((n, ld), dtype=torch.float32, device=device())
    if n and d:
        out[:, :d] = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).to(out.device)
    return out


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m
