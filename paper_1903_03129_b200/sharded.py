"""Column-sharded output layer over a torch.distributed group.

Partition: output row ``id`` lives on rank ``id % G`` at local row
``id // G`` (round-robin spreads the hot Zipf labels and FIFO buckets across
ranks); W2, its Adam state and step counters are sharded, W1 is replicated.

Tables: every rank hashes its own rows; the keys are all-gathered and every
rank builds the complete L tables from them -- the exact single-GPU tables
(FIFO tails and the reservoir stream included), so no bucket reconciliation
is needed and the active sets are selected identically on every rank.  A
rank then keeps the (sample, row) pairs it owns.

Per step, over the group: all-reduce MAX of the per-sample logit max,
all-reduce SUM of the exponential sums, all-reduce SUM of the label loss
terms, all-reduce SUM of the hidden-layer gradient (B x hidden).  W1's Adam
then runs identically on every rank.  At a rebuild: one all-gather of the
row keys (N x L uint32).

The orchestration (``sharded_step``) is backend-agnostic: ``GpuShardBackend``
runs the sm_100a stages of the C ABI; the CPU tests drive the same function
with a numpy backend over gloo.
"""

from __future__ import annotations

import numpy as np


def interleave(parts, n_total: int):
    """parts[g] (n_local_g, L) -> (n_total, L), global row r = local * G + g."""
    import torch

    G = len(parts)
    out = torch.empty((n_total,) + tuple(parts[0].shape[1:]), dtype=parts[0].dtype, device=parts[0].device)
    for g, p in enumerate(parts):
        n_g = (n_total - g + G - 1) // G
        out[g::G] = p[:n_g]
    return out


def all_gather_rows(local, n_total: int, group=None):
    """All-gather every rank's local rows (padded to the largest shard)."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    n_max = (n_total + G - 1) // G
    pad = torch.zeros((n_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(G)]
    dist.all_gather(parts, pad, group=group)
    return interleave(parts, n_total)


def gather_row_keys(net, group=None):
    """Global (N, L) table keys from every rank's local W2 rows (device)."""
    import torch

    from . import _lib

    L = net.layers[1].lsh.family.l
    local = torch.empty((net.n_local, L), dtype=torch.int32, device=net.w2.device)
    _lib.call("slide_shard_hash_rows", net._ctx, local.data_ptr())
    return all_gather_rows(local, net.n_out, group).contiguous()


def sharded_step(backend, csr, iteration: int, group=None):
    """One snapshot step of a column-sharded layer; returns (per-slot loss,
    per-slot global active-set size) like the single-GPU step."""
    import torch.distributed as dist

    mx = backend.forward(csr, iteration)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    se = backend.softmax_sum(mx)
    dist.all_reduce(se, op=dist.ReduceOp.SUM, group=group)
    lp = backend.softmax_finish(mx, se)
    dist.all_reduce(lp, op=dist.ReduceOp.SUM, group=group)
    dh = backend.hidden_grad()
    dist.all_reduce(dh, op=dist.ReduceOp.SUM, group=group)
    backend.update(dh)
    ny = np.diff(np.asarray(csr.y_ptr, dtype=np.int64))
    lp = lp.double().cpu().numpy()
    with np.errstate(invalid="ignore", divide="ignore"):
        loss = np.where(ny > 0, lp / np.maximum(ny, 1), np.nan)
    return loss, backend.active_counts()


class GpuShardBackend:
    """The C-ABI stages of a sharded SlideNetwork (slide_shard_*)."""

    def __init__(self, net):
        self.net = net
        self.keep = None

    def forward(self, csr, iteration):
        import torch

        from . import _lib

        net = self.net
        if net.layers[1].lsh is not None:
            net.layers[1].lsh.sync_to_device()
        pre = getattr(csr, "dev", None)  # batch already resident on the device (bench)
        bt, keep = pre if pre is not None else net._upload(csr)
        self.keep = (bt, keep)
        self.B = csr.batch
        mx = torch.empty(csr.batch, dtype=torch.float32, device=net.w2.device)
        _lib.call("slide_shard_forward", net._ctx, _lib.C.byref(bt), iteration, mx.data_ptr())
        return mx

    def softmax_sum(self, gmax):
        import torch

        from . import _lib

        out = torch.empty_like(gmax)
        _lib.call("slide_shard_softmax_sum", self.net._ctx, gmax.data_ptr(), out.data_ptr())
        return out

    def softmax_finish(self, gmax, gsum):
        import torch

        from . import _lib

        out = torch.empty(self.B, dtype=torch.float64, device=gmax.device)
        _lib.call("slide_shard_softmax_finish", self.net._ctx, gmax.data_ptr(), gsum.data_ptr(), out.data_ptr())
        return out

    def hidden_grad(self):
        import torch

        from . import _lib

        out = torch.empty((self.B, self.net.hidden_pad), dtype=torch.float32, device=self.net.w2.device)
        _lib.call("slide_shard_hidden_grad", self.net._ctx, out.data_ptr())
        return out

    def update(self, dh):
        import torch

        from . import _lib

        _lib.call("slide_shard_update", self.net._ctx, dh.data_ptr())
        torch.cuda.current_stream().synchronize()
        self.keep = None

    def active_counts(self):
        return self.net._read(12, self.B, np.int32).astype(np.int64)
