"""Column-sharded SLIDE layer over a torch.distributed group.

Partition (rank g of G):

* output rows: row ``id`` lives on rank ``id % G`` at local row ``id // G``
  (round-robin spreads the hot Zipf labels and FIFO buckets); W2, its Adam
  state, its step counters and **its LSH tables** (built over the rank's own
  rows, buckets holding global ids) are sharded;
* hidden units: W1^T is split by units, rank g holding the H/G columns
  [g H/G, (g+1) H/G) and their Adam moments; the hidden biases, their
  moments and the per-unit step counters (H values) are replicated and
  updated identically on every rank.

Per step, over the group (reference network.py:241-336 for one shard):

1. ``all_gather`` of the ranks' hidden pre-activation slices (B x H/G), so
   every rank holds h = relu(. + b1) (the same bits as the unsharded layer);
2. ``all_reduce(SUM)`` of the per-sample sampler counts (B x (L+1) int32):
   a rank's buckets hold only its ids, and ids are disjoint across ranks, so
   vanilla's "distinct ids after p probes" and every emptiness test are sums
   of the ranks' counts (samplers.py:57-112, network.py:225-239);
3. ``all_reduce(MAX)`` of the per-sample logit max over owned pairs;
4. ``all_reduce(SUM)`` of the exponential sums;
5. ``all_reduce(SUM)`` of the label loss terms and owned set sizes;
6. ``all_reduce(SUM)`` of the hidden-layer gradient partials (B x H).

Each rank then updates its W2 rows, the replicated hidden biases and its W1
units.  At a rebuild (tables.py:105-161): every rank builds its tables from
its own rows; ``all_reduce(MAX)`` of the largest local bucket proves no
global bucket overflows (G * max <= cap), else the ranks all-gather their
packed runs and each keeps its members of every FIFO bucket's global last
``cap`` ids.  Reservoir tables must not overflow (checked).

``sharded_step`` / ``rebuild_sharded`` are backend-agnostic: ``GpuShardBackend``
runs the sm_100a stages of the C ABI; the CPU tests drive the same functions
with a numpy backend over gloo.  Only the topk sampler is unsupported
(its frequency cutoff is a global order statistic).
"""

from __future__ import annotations

import numpy as np


def interleave(parts, n_total: int):
    """parts[g] (n_local_g, ...) -> (n_total, ...), global row r = local * G + g."""
    import torch

    G = len(parts)
    out = torch.empty((n_total,) + tuple(parts[0].shape[1:]), dtype=parts[0].dtype, device=parts[0].device)
    for g, p in enumerate(parts):
        n_g = (n_total - g + G - 1) // G
        out[g::G] = p[:n_g]
    return out


def all_gather_stack(t, group=None):
    """(G, *t.shape): every rank's tensor of one shape, stacked in rank order."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((G,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    parts = [torch.empty_like(t) for _ in range(G)]
    dist.all_gather(parts, t, group=group)
    return torch.stack(parts)


def all_gather_rows(local, n_total: int, group=None):
    """All-gather every rank's local rows (padded to the largest shard) into
    the global row order."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    n_max = (n_total + G - 1) // G
    pad = torch.zeros((n_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    return interleave(list(all_gather_stack(pad, group)), n_total)


def all_gather_units(local, group=None):
    """(rows, H/G) unit slices of every rank -> (rows, H) in unit order."""
    st = all_gather_stack(local, group)  # (G, rows, hg)
    return st.permute(1, 0, 2).reshape(local.shape[0], -1)


def rebuild_sharded(backend, group=None) -> bool:
    """Rebuild this rank's tables (tables.py:105-161 restricted to its rows).
    Returns True when the FIFO exchange ran."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    m = torch.tensor([backend.build_local()], dtype=torch.int64, device=backend.device)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    if int(m.item()) * G <= backend.capacity:
        return False  # no bucket can hold more than cap ids over all ranks
    if backend.policy != "fifo":
        raise NotImplementedError("sharded reservoir tables need every bucket within capacity "
                                  f"(shard_count {G} x largest local bucket {int(m.item())} > cap {backend.capacity})")
    pack = backend.pack()
    n = torch.tensor([pack.numel()], dtype=torch.int64, device=backend.device)
    dist.all_reduce(n, op=dist.ReduceOp.MAX, group=group)
    padded = torch.zeros(int(n.item()), dtype=pack.dtype, device=pack.device)
    padded[: pack.numel()] = pack
    backend.reconcile(all_gather_stack(padded, group))
    return True


class StepResult:
    """Per-slot loss and global active-set size of a sharded step, read from
    the device lazily (the step itself never waits on the host)."""

    def __init__(self, lp, y_counts):
        self._lp = lp
        self._ny = np.asarray(y_counts, dtype=np.int64)

    def host(self):
        v = self._lp.double().cpu().numpy()
        B = self._ny.size
        with np.errstate(invalid="ignore", divide="ignore"):
            loss = np.where(self._ny > 0, v[:B] / np.maximum(self._ny, 1), np.nan)
        return loss, np.rint(v[B : 2 * B]).astype(np.int64)


def sharded_step(backend, csr, iteration: int, group=None) -> StepResult:
    """One snapshot step of the column-sharded layer (the 6 collectives of
    the module docstring); no host synchronisation inside."""
    import torch.distributed as dist

    SUM, MAX = dist.ReduceOp.SUM, dist.ReduceOp.MAX
    part = backend.hidden(csr)
    backend.assemble(all_gather_stack(part, group))
    hist = backend.select(iteration)
    dist.all_reduce(hist, op=SUM, group=group)
    mx = backend.forward(iteration, hist)
    dist.all_reduce(mx, op=MAX, group=group)
    se = backend.softmax_sum(mx)
    dist.all_reduce(se, op=SUM, group=group)
    lp = backend.softmax_finish(mx, se)
    dist.all_reduce(lp, op=SUM, group=group)
    dh = backend.hidden_grad()
    dist.all_reduce(dh, op=SUM, group=group)
    backend.update(dh)
    return StepResult(lp, np.diff(np.asarray(csr.y_ptr, dtype=np.int64)))


class GpuShardBackend:
    """The C-ABI stages of a sharded SlideNetwork (slide_shard_*)."""

    def __init__(self, net):
        self.net = net
        self.keep = None
        self.device = net.w2.device
        lsh = net.layers[1].lsh
        self.capacity = lsh.capacity if lsh is not None else 0
        self.policy = lsh.policy if lsh is not None else "fifo"

    def _call(self, name, *args):
        from . import _lib

        _lib.call(name, self.net._ctx, *args)

    # -- tables
    def build_local(self) -> int:
        from . import _lib

        m = _lib.i64()
        self._call("slide_shard_build_local", _lib.C.byref(m))
        return int(m.value)

    def pack(self):
        import torch

        from . import _lib

        n = _lib.i64()
        self._call("slide_shard_tables_pack_size", _lib.C.byref(n))
        out = torch.empty(max(int(n.value), 1), dtype=torch.int32, device=self.device)
        self._call("slide_shard_tables_pack", out.data_ptr())
        self._pack_keep = out
        return out[: int(n.value)]

    def reconcile(self, gathered):
        gathered = gathered.contiguous()
        self._call("slide_shard_tables_reconcile", gathered.data_ptr(), gathered.shape[1])
        self._gathered_keep = gathered

    # -- step
    def hidden(self, csr):
        import torch

        from . import _lib

        net = self.net
        if net.layers[1].lsh is not None:
            net.layers[1].lsh.sync_to_device()
        pre = getattr(csr, "dev", None)  # batch already resident on the device (bench)
        bt, keep = pre if pre is not None else net._upload(csr)
        self.bt, self.keep = bt, keep
        self.B = csr.batch
        part = torch.empty((csr.batch, net.hidden // net.shard_count), dtype=torch.float32, device=self.device)
        self._call("slide_shard_hidden", _lib.C.byref(bt), part.data_ptr())
        return part

    def assemble(self, parts):
        self._parts = parts.contiguous()
        self._call("slide_shard_assemble", self.B, self._parts.data_ptr())

    def select(self, iteration):
        import torch

        from . import _lib

        L = self.net.layers[1].lsh.family.l
        self._hist = torch.empty((self.B, L + 1), dtype=torch.int32, device=self.device)
        self._call("slide_shard_select", _lib.C.byref(self.bt), iteration, self._hist.data_ptr())
        return self._hist

    def forward(self, iteration, ghist):
        import torch

        from . import _lib

        self._ghist = ghist.contiguous()
        mx = torch.empty(self.B, dtype=torch.float32, device=self.device)
        self._call("slide_shard_forward", _lib.C.byref(self.bt), iteration, self._ghist.data_ptr(), mx.data_ptr())
        return mx

    def softmax_sum(self, gmax):
        import torch

        out = torch.empty_like(gmax)
        self._call("slide_shard_softmax_sum", gmax.data_ptr(), out.data_ptr())
        self._gmax = gmax
        return out

    def softmax_finish(self, gmax, gsum):
        import torch

        out = torch.empty(2 * self.B, dtype=torch.float64, device=gmax.device)
        self._call("slide_shard_softmax_finish", gmax.data_ptr(), gsum.data_ptr(), out.data_ptr())
        self._gsum = gsum
        return out

    def hidden_grad(self):
        import torch

        out = torch.empty((self.B, self.net.hidden_pad), dtype=torch.float32, device=self.device)
        self._call("slide_shard_hidden_grad", out.data_ptr())
        return out

    def update(self, dh):
        self._dh = dh
        self._call("slide_shard_update", dh.data_ptr())
