"""Kernel timeline of warm graph steps (CUPTI through torch.profiler).

usage: python profiles/timeline.py [workload] [steps]
Runs the bench workload's graph step (two in flight, as bench.py times it),
records every kernel's start / end / stream for `steps` steps after a
warm-up and prints, per step, each kernel's start offset and duration, its
stream and the step's span -- the critical path that the serialised ncu
launch list cannot show.  Not a bench number (profiler attached).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(workload="wide_in", steps=3):
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_1903_03129_b200 import _lib
    from paper_1903_03129_b200.data import synthetic_corpus

    from paper_1903_03129_b200.configs import WORKLOADS

    w = WORKLOADS[workload]
    W = 8
    n = W + steps
    corpus = synthetic_corpus(w.corpus, n * w.batch, seed=1000)
    batches = bench.csr_batches(corpus, w.batch, n)
    net = bench.make_net(w, torch)
    dev = [net._upload(b) for b in batches]
    loss = np.empty(w.batch, np.float64)
    act = np.empty(w.batch, np.int64)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def run(its):
        for k, it in enumerate(its):
            flush.zero_()
            _lib.call("slide_graph_step_async", net._ctx, _lib.C.byref(dev[it - 1][0]), it)
            net._rebuild_after(it)
            if k:
                _lib.call("slide_graph_step_wait", net._ctx, loss.ctypes.data, act.ctypes.data)
        _lib.call("slide_graph_step_wait", net._ctx, loss.ctypes.data, act.ctypes.data)
        torch.cuda.synchronize()

    run(range(1, W + 1))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run(range(W + 1, n + 1))
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = []
    for e in ev:
        name = e.name
        if "Memcpy" in name or "Memset" in name:
            kind = "copy"
        else:
            kind = "kernel"
        ks.append((e.time_range.start, e.time_range.end, name, kind))
    ks.sort()
    # steps are separated by the flush kernel (at::...FillFunctor / zero_)
    cuts = [i for i, k in enumerate(ks) if "FillFunctor" in k[2] or "fill" in k[2].lower()]
    cuts.append(len(ks))
    for s in range(len(cuts) - 1):
        seg = ks[cuts[s] + 1:cuts[s + 1]]
        if not seg:
            continue
        t0 = seg[0][0]
        span = max(k[1] for k in seg) - t0
        busy = sum(k[1] - k[0] for k in seg if k[3] == "kernel")
        print(f"--- step {s}: span {span:.1f} us, {len(seg)} ops, summed kernel time {busy:.1f} us")
        for a, b, name, kind in seg:
            nm = name.split("(")[0].replace("void ", "").replace("slide::", "")[:60]
            print(f"  {a - t0:8.1f} +{b - a:7.1f}  end {b - t0:8.1f}  {nm}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "wide_in", int(sys.argv[2]) if len(sys.argv) > 2 else 3)
