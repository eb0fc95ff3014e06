"""Benchmark: SLIDE LSH-sparse training step (fwd + bwd + Adam + rebuild).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload wide_in]
    python bench.py --impl reference ...   # the reference algorithm on the CPU

One JSON line on rank 0.  A "step" is one train_batch of B synthetic
samples (SURVEY.md 8(d) generator, standing in for Delicious-200K /
Amazon-670K) through the snapshot schedule, including the table rebuild
whenever the schedule makes it due (every ~50 steps) -- the timed steps are
chosen so that one rebuild falls inside them.

* value: samples/s with every batch already resident in HBM; each step is
  timed with CUDA events on the launching stream, L2 flushed (256 MiB write)
  between steps outside the events;
* e2e: same metric through the public API (SlideNetwork.train_batch_csr)
  from pinned host CSR, host->device copy and the per-slot loss readback
  inside the timed region;
* roofline: the dominant kernel's algorithmic bytes / its event-timed
  duration vs the measured HBM copy bandwidth (MEASURED_PEAKS.json);
* cpu_baseline: the CPU oracle (a numpy restatement of the reference path,
  kind "port") on a bounded sample of the same workload, 1 thread.

N>1 (torchrun): the layer is sharded over the N GPUs (SURVEY 8(e),
paper_1903_03129_b200/sharded.py): W2 rows, their Adam state and their LSH
tables by output id, W1 by hidden unit; the global batch is N x the
workload's batch (weak scaling: per-rank work stays ~constant), and the step
runs one all-gather (hidden slices) and five all-reduces (sampler counts,
softmax max / sum, loss terms, hidden gradient) over NCCL; max-over-ranks
device time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STAGES = ["hidden_fwd", "query_hash", "slot_rng", "select", "fallback", "compact", "logits", "softmax",
          "hidden_grad", "group_rows", "adam_w2", "hidden_counts", "group_features", "adam_w1", "hidden_bias",
          "rebuild_hash", "rebuild_build"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=53)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="wide_in")
    p.add_argument("--schedule", default="snapshot", choices=["snapshot", "sequential"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-flush", action="store_true", help="experiments only: keep L2 warm between steps")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-samples", type=int, default=128)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region (NVML,
    every 2 ms; the same fields as the recipe's nvidia-smi clocks line)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.err = None
        self._hnd = None
        try:  # NVML init here, in the caller's thread and outside any timed region
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._hnd = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._hnd, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report it rather than invent clocks
            self.err = repr(e)

    def _run(self):
        if self._hnd is None:
            return
        nv, hnd = self._nvml, self._hnd
        try:
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(hnd, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(hnd)
                self.rows.append((sm, self._max, rs))
                self._stop.wait(0.002)
        except Exception as e:
            self.err = repr(e)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"no samples ({self.err})"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


def config_of(w, args, world):
    """The workload's `config` object -- identical on both arms' lines."""
    return {"workload": w.name, "input_dim": w.input_dim, "hidden": w.hidden, "n_out": w.n_out,
            "batch": w.batch * world, "hash": f"{w.family} K={w.k} L={w.l} cap={w.cap} {w.policy}",
            "sampler": f"{w.strategy} beta={w.beta}", "lr": w.lr, "rebuild": f"n0={w.n0} decay={w.decay}",
            "schedule": args.schedule,
            "parallelism": f"output layer column-sharded x{world}" if world > 1 else "1 GPU",
            "rebuild_in_step": "amortised: measured table rebuild ms / n0 added to every step",
            "l2": "flushed between steps (256 MiB write, outside the events)"}


def make_net(w, torch, rank=0, world=1):
    from paper_1903_03129_b200 import LshLayerConfig, SamplerConfig, SlideNetwork, TrainConfig

    cfg = TrainConfig(batch_size=w.batch * world, learning_rate=w.lr, n0=w.n0, decay=w.decay, seed=0)
    spec = LshLayerConfig(w.family, k=w.k, l=w.l, capacity=w.cap, policy=w.policy, wta_bin_size=w.bin_size,
                          sampler=SamplerConfig(w.strategy, beta=w.beta))
    shard = (rank, world) if world > 1 else None
    return SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec}, shard=shard)


def csr_batches(corpus, B, n):
    from paper_1903_03129_b200.network import HostCsr

    out = []
    for s in range(n):
        sub = corpus.subset(np.arange(s * B, (s + 1) * B))
        out.append(HostCsr(sub.x_ptr.astype(np.int32), sub.x_idx, sub.x_val, sub.y_ptr.astype(np.int32), sub.y_idx))
    return out


def stage_bytes(w, ms, cnt, steps):
    """Algorithmic bytes per stage per step from the realised sets.

    Every touched row / coordinate counted once per step; fp32 state."""
    H = w.hidden
    per = lambda v: v / max(steps, 1)
    P, nnz, B = per(cnt[8]), per(cnt[9]), per(cnt[10])
    U2, U1 = per(cnt[2]), per(cnt[3])
    t2, t1 = per(cnt[0]), per(cnt[1])
    probed = per(cnt[4])
    rebuilds = per(cnt[11])
    b = {
        "hidden_fwd": U1 * 4 * H + nnz * 8 + B * 4 * H,
        "query_hash": B * 4 * H + B * w.l * 4,
        "select": B * w.l * 8 + probed * 4 + P * 4,
        "logits": U2 * (4 * H + 4) + P * 12 + B * 4 * H,
        "softmax": P * 13,
        "hidden_grad": U2 * 4 * H + P * 8 + B * 8 * H,
        "adam_w2": t2 * 24 + U2 * (24 + 16 + 12) + P * 12,
        "adam_w1": t1 * 24 + U1 * 12 + nnz * 12,
        "hidden_bias": B * 4 * H * 3,
        "rebuild_hash": rebuilds * (w.n_out * 4 * H + w.n_out * w.l * 4),
        "rebuild_build": rebuilds * (w.n_out * w.l * 4 * 4),
    }
    # whole step (SURVEY 8(d) formula): inputs + W1 rows + Adam W1 + probes + W2 rows + Adam W2 + rebuild
    step = (nnz * 8 + per(cnt[10]) * 0 + U1 * 4 * H + 20 * t1 + 24 * H + B * w.l * 8 + probed * 4
            + U2 * (4 * H + 24) + 20 * t2 + b["rebuild_hash"] + b["rebuild_build"])
    return b, step


def measure_rebuild(net, torch, flush, args, reps=3):
    """Median event time of `reps` full table rebuilds (hash every W2 row +
    build all L tables: the barrier's path, network._rebuild_tables), L2
    flushed before each."""
    out = []
    for _ in range(reps):
        if not args.no_flush:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        net._rebuild_tables()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


def recaptures(net):
    """Graph re-captures so far on the net's context (host_counts[5])."""
    from paper_1903_03129_b200 import _lib

    ms = np.zeros(32, np.float64)
    cnt = np.zeros(16, np.int64)
    _lib.call("slide_profile_read", net._ctx, ms.ctypes.data, cnt.ctypes.data)
    return int(cnt[8 + 5])


def run_ours(args, rank, world):
    import torch

    from paper_1903_03129_b200 import _lib
    from paper_1903_03129_b200.configs import WORKLOADS
    from paper_1903_03129_b200.data import synthetic_corpus

    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist

        # NCCL over NVLink on B200s; SLIDE_BENCH_DIST=gloo exercises the same
        # path with several ranks on one GPU (correctness only, not timing)
        dist.init_process_group(os.environ.get("SLIDE_BENCH_DIST", "nccl"))
    w = WORKLOADS[args.workload]
    K, W = args.steps, args.warmup
    n_batches = W + K
    # N > 1: weak scaling -- a global batch of N x the workload's batch, every
    # rank holds 1/N of the output rows (W2, its tables) and of the hidden
    # units (W1), so per-rank work stays ~constant
    B = w.batch * world
    corpus = synthetic_corpus(w.corpus, n_batches * B, seed=1000)
    batches = csr_batches(corpus, B, n_batches)
    net = make_net(w, torch, rank, world)
    sub = 1 if args.schedule == "sequential" else B
    # device-resident inputs for `value`
    dev_batches = []
    for b in batches:
        bt, keep = net._upload(b)
        dev_batches.append((bt, keep, b))
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    loss_buf = np.empty(B, np.float64)
    act_buf = np.empty(B, np.int64)

    def step_dev(it, barrier=True):
        bt, keep, hb = dev_batches[it - 1]
        if world > 1:  # column-sharded output layer: stages + all-reduces
            from paper_1903_03129_b200.sharded import GpuShardBackend, sharded_step

            hb.dev = (bt, keep)
            loss, act = sharded_step(GpuShardBackend(net), hb, it, None).host()
            return net._barrier(it, loss, act) if barrier else net._stats(loss, act, [])
        if sub == B and net.use_graphs:  # the captured-graph snapshot step
            _lib.call("slide_graph_step", net._ctx, _lib.C.byref(bt), it, loss_buf.ctypes.data, act_buf.ctypes.data)
        else:
            _lib.call("slide_train_batch", net._ctx, _lib.C.byref(bt), it, sub, loss_buf.ctypes.data,
                      act_buf.ctypes.data)
        return net._barrier(it, loss_buf, act_buf) if barrier else net._stats(loss_buf, act_buf, [])

    # one GPU, graph steps: two steps in flight (slide_graph_step_async), so
    # the host's launch work overlaps the device -- per step, on the context
    # stream: L2 flush, event, step, its rebuild barrier, event; the events
    # bracket exactly the step + barrier, the flush stays outside
    pipelined_dev = world == 1 and sub == B and net.use_graphs

    def run_pipelined(its, evs=None, losses=None):
        def wait_oldest():
            _lib.call("slide_graph_step_wait", net._ctx, loss_buf.ctypes.data, act_buf.ctypes.data)
            if losses is not None:
                losses.append(float(np.mean(loss_buf)))

        for k, it in enumerate(its):
            bt = dev_batches[it - 1][0]
            if not args.no_flush:
                flush.zero_()
            e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            _lib.call("slide_graph_step_async", net._ctx, _lib.C.byref(bt), it)
            em.record()
            rebuilt = net._rebuild_after(it)
            e1.record()
            if evs is not None:
                evs.append((e0, em, e1, bool(rebuilt)))
            if k > 0:
                wait_oldest()
        wait_oldest()
        torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device())  # NVML init before the warm-up
    if pipelined_dev:  # the warm-up also allocates both in-flight slots' staging
        run_pipelined(range(1, W + 1))
    else:
        for it in range(1, W + 1):
            step_dev(it)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    lc0 = np.zeros(1, np.uint64)
    _lib.call("slide_launch_count", lc0.ctypes.data)
    times = []
    losses = []
    with sampler as clk:
        # per step: the step (e0 -> em) and its rebuild barrier (em -> e1)
        if pipelined_dev:
            evs = []
            run_pipelined(range(W + 1, W + K + 1), evs, losses)
        else:
            evs = []
            for it in range(W + 1, W + K + 1):
                if not args.no_flush:
                    flush.zero_()
                e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                torch.cuda.synchronize()
                e0.record()
                st = step_dev(it, barrier=False)
                em.record()
                rebuilt = net._rebuild_after(it)
                e1.record()
                torch.cuda.synchronize()
                evs.append((e0, em, e1, bool(rebuilt)))
                losses.append(st.loss)
        times = [a.elapsed_time(m) for a, m, _, _ in evs]
        barrier_ms = [m.elapsed_time(b) for _, m, b, r in evs if r]
    lc1 = np.zeros(1, np.uint64)
    _lib.call("slide_launch_count", lc1.ctypes.data)
    if dist:
        dist.barrier()
    # the table rebuild of the barrier, amortised over its period: measured
    # live (event-timed forced rebuilds of this net, the barrier's own path)
    # unless the window itself held rebuilds
    rebuild_ms = float(np.median(barrier_ms)) if barrier_ms else measure_rebuild(net, torch, flush, args)
    amort_ms = rebuild_ms / w.n0
    total_ms = float(np.sum(times)) + K * amort_ms
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # N > 1: the ranks share one global batch per step (sharded output layer)
    value = K * B / (total_ms / 1e3)
    # -- e2e: public API from host CSR, fresh net state continues.
    # (1) pipelined SlideNetwork.train_batches_csr over the K batches, timed
    #     as one region (each step: H2D of its batch, the step, D2H of its
    #     losses; the next batch is staged while the device runs); L2 flushed
    #     once before -- the step's inputs include the 1.5 GB model state,
    #     far above the 126 MB L2;
    # (2) one synchronous train_batch_csr call per step, L2 flushed between
    #     steps outside the events (reported as e2e.sync_value).
    e2e = None
    if not args.no_e2e:
        it0 = W + K + 1
        order = [batches[(W + k) % n_batches] for k in range(K)]
        pipelined = world == 1 and args.schedule == "snapshot"
        p_passes, p_recap = [], []
        if pipelined:
            # untimed warm-up pass over W batches: both in-flight slots' pinned
            # staging exist before the timed passes
            net.train_batches_csr(order[:max(W, 2)], first_iteration=it0, schedule=args.schedule)
            it0 += max(W, 2)
            # three consecutive passes over the K batches (training continues);
            # the median pass is reported, every pass and its graph
            # re-captures (host_counts[5]) alongside
            for _ in range(3):
                rc0 = recaptures(net)
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                stats = net.train_batches_csr(order, first_iteration=it0, schedule=args.schedule)
                e1.record()
                torch.cuda.synchronize()
                # the pass's own rebuilds replaced by the amortised share
                n_rb = sum(bool(x.rebuilt) for x in stats)
                p_passes.append(e0.elapsed_time(e1) - n_rb * rebuild_ms + K * amort_ms)
                p_recap.append(recaptures(net) - rc0)
                it0 += K
            p_total = float(np.median(p_passes))
        e_times = []
        h2d = d2h = 0
        for k in range(K):
            it = it0 + k
            b = order[k]
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = net.train_batch_csr(b, it, schedule=args.schedule)
            e1.record()
            torch.cuda.synchronize()
            e_times.append(e0.elapsed_time(e1) - bool(st.rebuilt) * rebuild_ms + amort_ms)
            h2d += net.h2d_bytes
            d2h += B * 16 + (B + 1) * 4 * (B // sub)
        e_total = float(np.sum(e_times))
        if dist:
            t = torch.tensor([e_total], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_total = float(t.item())
        sync_value = K * B / (e_total / 1e3)
        e2e = {"value": K * B / (p_total / 1e3) if pipelined else sync_value, "unit": "samples/s",
               "h2d_bytes_per_step": int(h2d / K), "d2h_bytes_per_step": int(d2h / K),
               "api": ("SlideNetwork.train_batches_csr (pipelined: batch k+1 staged while step k runs), "
                       "L2 flushed once before the K steps" if pipelined else "SlideNetwork.train_batch_csr"),
               "sync_value": sync_value,
               "pipelined_passes": [K * B / (t / 1e3) for t in p_passes], "pipelined_recaptures": p_recap,
               "sync_api": "SlideNetwork.train_batch_csr per step, L2 flushed between steps outside the events"}
    # -- profiled pass: per-stage event times + realised sets
    # -- profiled pass: per-stage event times + realised sets
    _lib.call("slide_profile", net._ctx, 1)
    it0 = W + 3 * K + 1
    for k in range(K):
        step_dev_it = it0 + k
        bt, keep, hb = dev_batches[(W + k) % n_batches]
        if world > 1:
            from paper_1903_03129_b200.sharded import GpuShardBackend, sharded_step

            hb.dev = (bt, keep)
            loss, act = sharded_step(GpuShardBackend(net), hb, step_dev_it, None).host()
            net._barrier(step_dev_it, loss, act)
            continue
        _lib.call("slide_train_batch", net._ctx, _lib.C.byref(bt), step_dev_it, sub, loss_buf.ctypes.data,
                  act_buf.ctypes.data)
        net._barrier(step_dev_it, loss_buf, act_buf)
    ms = np.zeros(32)
    cnt = np.zeros(16, np.int64)
    _lib.call("slide_profile_read", net._ctx, ms.ctypes.data, cnt.ctypes.data)
    _lib.call("slide_profile", net._ctx, 0)
    stage_ms = {STAGES[i]: float(ms[i]) / K for i in range(len(STAGES))}
    sb, step_bytes = stage_bytes(w, ms, cnt, K)
    dom = max((k for k in sb if stage_ms.get(k, 0) > 0), key=lambda k: stage_ms[k])
    peak, peak_kind = peaks()
    achieved = sb[dom] / (stage_ms[dom] / 1e3) / 1e9
    traffic = None
    issue = None
    try:  # dram bytes per launch from the committed `ncu --set full` capture of that kernel
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(w.name, {}).get(dom)
        if tr:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            inst = tr.get("warp_instructions")
            if inst:
                # the kernel is issue-bound, not HBM-bound: its instruction
                # count (same capture) over its event time against 4 warp
                # instructions per SM cycle at the sampled clock
                sm_hz = (clk.summary().get("sm_mhz") or 1965) * 1e6
                peak_i = 148 * 4 * sm_hz / 1e9
                got_i = inst / (stage_ms[dom] / 1e3) / 1e9
                issue = {"bound": "issue", "warp_instructions_per_launch": inst, "achieved": got_i,
                         "peak": peak_i, "unit": "G warp-inst/s", "frac": got_i / peak_i,
                         "source": tr.get("source")}
    except Exception:
        traffic = None
    ms_per_step = total_ms / K
    out = {
        "metric": "train samples/sec (LSH-sparse fwd+bwd+Adam), % of HBM roofline, 1/2/4/8 GPU",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        # per-step spread (the steps whose barrier rebuilt the tables are the max)
        "ms_per_step_p50": float(np.median(times)), "ms_per_step_max": float(np.max(times)),
        # the step alone (no rebuild) and the rebuild it amortises
        "ms_step_only_mean": float(np.mean(times)), "rebuild_ms": rebuild_ms,
        "rebuild_amortised_ms_per_step": amort_ms, "rebuilds_in_window": len(barrier_ms),
        "value_without_rebuild": K * B / (float(np.sum(times)) / 1e3),
        "dtype": "f32", "data": "synthetic (SURVEY 8(d) Zipf generator; Delicious-200K shape)",
        "config": config_of(w, args, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind, "issue": issue,
                     "algorithmic_bytes_per_launch": sb[dom], "ms_per_launch": stage_ms[dom]},
        "step_roofline": {"bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms_per_step / 1e3) / 1e9,
                          "frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak},
        "stages_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
        "realised_per_step": {"pairs": cnt[8] / K, "unique_rows": cnt[2] / K, "unique_features": cnt[3] / K,
                              "touched_w2": cnt[0] / K, "touched_w1": cnt[1] / K, "input_nnz": cnt[9] / K,
                              "probed_slots": cnt[4] / K, "rebuilds_in_profile": int(cnt[11]),
                              # hidden-unit renumberings so far (live units kept adjacent)
                              "unit_relabels": int(getattr(net, "relabels", 0))},
        "gpu_launches": int(lc1[0] - lc0[0]),
        "clocks": clk.summary(),
        "loss_first_last": [losses[0], losses[-1]],
    }
    if e2e:
        out["e2e"] = e2e
    del dev_batches
    return out, net, w


def cpu_port_rate(w, n_samples, threads=1):
    """CPU oracle (numpy restatement of the reference, test infrastructure)
    on a bounded sample of the workload: sequential schedule = the
    reference's train_batch(workers=1)."""
    from threadpoolctl import threadpool_limits

    from oracle import slide_oracle as O
    from paper_1903_03129_b200.data import synthetic_corpus

    with threadpool_limits(threads):
        st = O.init_state(w.input_dim, w.hidden, w.n_out, seed=0)
        spec = O.LshSpec(w.family, w.k, w.l, w.cap, w.policy, bin_size=w.bin_size, strategy=w.strategy, beta=w.beta)
        lsh = O.OutputLsh(spec, w.hidden, 0, w.n0, w.decay)
        lsh.build(st.w2)
        corpus = synthetic_corpus(w.corpus, n_samples, seed=7)
        trip = corpus.triples()
        t0 = time.perf_counter()
        O.train_step(st, lsh, trip, 1, 0, w.n_out, O.AdamCfg(lr=w.lr), mode="sequential")
        dt = time.perf_counter() - t0
    return n_samples / dt, dt


_REF = {}


def _ref_slot(task):
    """One slot's forward + backward on the pre-step state (a forked worker;
    the state arrays are shared memory, so it sees the parent's updates;
    the slot's input comes with the task)."""
    from oracle import slide_oracle as O

    r = _REF
    i, it, (xi, xv, y) = task
    rng = np.random.default_rng((0, it, i))
    tr = O.slot_forward(r["st"], r["lsh"], xi, xv, y, rng, r["n_out"])
    return O.slot_backward(r["st"], tr, y), tr.loss


def _ref_update(p):
    """Worker p of P applies every slot's Adam updates (slot order) to its
    share of the rows: output rows with id % P == p, input features with
    id % P == p.  Rows are independent in the reference's update
    (network.py:428-451: per-row step counters, per-row moments), so the
    partition reproduces the serial result; the hidden units' step counters
    advance identically in every worker, and worker 0 alone writes the
    hidden biases and counters."""
    from oracle import slide_oracle as O

    r = _REF
    st, cfg, P = r["st"], r["cfg"], r["P"]
    w1, m1, v1 = st.w1t.T, st.m1t.T, st.v1t.T
    steps1 = r["steps1"].copy()  # pre-step hidden-unit counters (worker 0's are written back)
    b1 = st.b1 if p == 0 else st.b1.copy()
    mb1 = st.mb1 if p == 0 else st.mb1.copy()
    vb1 = st.vb1 if p == 0 else st.vb1.copy()
    for g in r["grads"]:
        sel = g.active % P == p
        rows, d = g.active[sel], g.delta[sel]
        if g.h_idx.size == 0:
            O._adam_rows(st.w2, st.m2, st.v2, st.b2, st.mb2, st.vb2, st.steps2, rows, None, None, d, cfg)
            continue
        O._adam_rows(st.w2, st.m2, st.v2, st.b2, st.mb2, st.vb2, st.steps2, rows, g.h_idx,
                     np.outer(d, g.h_val), d, cfg)
        fs = g.x_idx % P == p
        cols = g.x_idx[fs]
        O._adam_rows(w1, m1, v1, b1, mb1, vb1, steps1, g.h_idx, cols if cols.size else None,
                     np.outer(g.dh, g.x_val[fs]) if cols.size else None, g.dh, cfg)
    if p == 0:
        st.steps1[:] = steps1
    return p


def reference_parallel_step(st, lsh, batch, it, cfg, cores, pool, ctx):
    """One snapshot step of the reference path on `cores` processes: the
    slots' forward/backward in `pool` (forked with _REF["st"] / ["lsh"] /
    ["n_out"] set), the row-partitioned updates in fresh workers, then the
    rebuild barrier (True when the tables were rebuilt: re-fork `pool`)."""
    res = pool.map(_ref_slot, [(i, it, x) for i, x in enumerate(batch)], chunksize=1)
    # the hidden counters are snapshotted before any update worker runs: worker
    # 0 writes st.steps1 back when it finishes, possibly before another starts
    _REF.update(grads=[g for g, _ in res], cfg=cfg, P=cores, steps1=st.steps1.copy())
    with ctx.Pool(cores) as up:
        up.map(_ref_update, range(cores), chunksize=1)
    if lsh is not None and lsh.schedule.due(it):
        lsh.build(st.w2)
        lsh.schedule.advance()
        return True
    return False


def _shared_state(st):
    """The NetState's arrays moved into anonymous shared memory (fork-inherited)."""
    import dataclasses
    import mmap

    out = {}
    for f in dataclasses.fields(st):
        a = getattr(st, f.name)
        if isinstance(a, np.ndarray) and a.size:
            buf = mmap.mmap(-1, a.nbytes)
            b = np.frombuffer(buf, dtype=a.dtype).reshape(a.shape)
            b[...] = a
            out[f.name] = b
    return dataclasses.replace(st, **out)


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU path (oracle port), K
    bounded steps on rank 0 with every host core: the reference's HOGWILD
    batch (workers = cpu_count, network.py:340-379) in its deterministic
    snapshot member -- the slots' forward/backward run in parallel worker
    processes on the pre-step weights, the Adam updates are applied in slot
    order."""
    import multiprocessing as mp

    from threadpoolctl import threadpool_limits

    from oracle import slide_oracle as O
    from paper_1903_03129_b200.configs import WORKLOADS
    from paper_1903_03129_b200.data import synthetic_corpus

    w = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    per_step = w.batch * world  # the full (global) batch: the same config as the GPU arm
    with threadpool_limits(1):
        st = _shared_state(O.init_state(w.input_dim, w.hidden, w.n_out, seed=0))
        spec = O.LshSpec(w.family, w.k, w.l, w.cap, w.policy, bin_size=w.bin_size, strategy=w.strategy, beta=w.beta)
        lsh = O.OutputLsh(spec, w.hidden, 0, w.n0, w.decay)
        lsh.build(st.w2)
        corpus = synthetic_corpus(w.corpus, (args.warmup + args.steps) * per_step, seed=1000)
        trip = corpus.triples()
        _REF.update(st=st, lsh=lsh, n_out=w.n_out)
        cfg = O.AdamCfg(lr=w.lr)
        ctx = mp.get_context("fork")
        pool = None
        rebuilds = [0]

        rb_s = []

        def step(it):
            nonlocal pool
            batch = trip[(it - 1) * per_step : it * per_step]
            if pool is None:  # forked after the tables exist (rebuilds re-fork)
                pool = ctx.Pool(cores)
            t0 = time.perf_counter()
            if reference_parallel_step(st, lsh, batch, it, cfg, cores, pool, ctx):
                pool.close()
                pool = None
                if it > args.warmup:
                    rebuilds[0] += 1
                    rb_s.append(time.perf_counter() - t0)
            return time.perf_counter() - t0

        try:
            for it in range(1, args.warmup + 1):
                step(it)
            t0 = time.perf_counter()
            for it in range(args.warmup + 1, args.warmup + args.steps + 1):
                step(it)
            dt = time.perf_counter() - t0
        finally:
            if pool is not None:
                pool.close()
        # the rebuild amortised like the GPU arm's: one timed full build
        # (hash every W2 row + all L tables) / n0 per step, in place of the
        # window's own rebuilds (their whole step time is charged, an upper
        # bound on the build inside it)
        t0 = time.perf_counter()
        lsh.build(st.w2)
        build_s = time.perf_counter() - t0
    dt = dt - sum(rb_s) + args.steps * build_s / w.n0
    v = args.steps * per_step / dt
    pkg = run_reference_package(args, w, per_step, corpus, cores)
    sample = (f"{args.steps} steps x {per_step} samples (the full batch) of {w.name}, snapshot schedule on "
              f"{cores} processes (numpy), table build {build_s:.2f} s amortised over n0={w.n0} steps")
    return {
        "impl": "reference", "metric": "train samples/sec (LSH-sparse fwd+bwd+Adam), % of HBM roofline, 1/2/4/8 GPU",
        "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SURVEY 8(d) Zipf generator)",
        "config": config_of(w, args, world),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_package": pkg,
    }


def run_reference_package(args, w, per_step, corpus, cores):
    """The reference package itself (``slide`` 0.1.0, pip-installed into
    baseline/_ref when present -- git-ignored, it travels with the repo),
    timed beside the port on the same batches: ``SlideNetwork.train_batch``
    with ``workers = cpu_count`` threads (its HOGWILD path, network.py:340-379),
    a bounded number of steps after one warm-up step, the table build
    amortised over n0 like the other arms.  Reported, not the arm's value
    (this tier's reference arm is the oracle port)."""
    import importlib
    from concurrent.futures import ThreadPoolExecutor

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "slide")) or os.environ.get("SLIDE_SKIP_REF_PACKAGE"):
        return {"unavailable": "baseline/_ref holds no reference install"}
    sys.path.insert(0, ref_dir)
    try:
        net_mod = importlib.import_module("slide.network")
        smp = importlib.import_module("slide.samplers")
        sp = importlib.import_module("slide.sparse")
        cfg = net_mod.TrainConfig(batch_size=per_step, learning_rate=w.lr, n0=w.n0, decay=w.decay, seed=0)
        spec = net_mod.LshLayerConfig(w.family, k=w.k, l=w.l, capacity=w.cap, policy=w.policy,
                                      wta_bin_size=w.bin_size, sampler=smp.SamplerConfig(w.strategy, beta=w.beta))
        t0 = time.perf_counter()
        net = net_mod.SlideNetwork(w.input_dim, [w.hidden, w.n_out], cfg, lsh_layers={1: spec})
        init_s = time.perf_counter() - t0
        trip = corpus.triples()
        steps = max(1, min(args.steps, 3))

        def batch(it):
            rows = trip[(it - 1) * per_step : it * per_step]
            return [(sp.SparseVector(np.asarray(i, np.int64), np.asarray(v, np.float64), w.input_dim), list(y))
                    for i, v, y in rows]

        with ThreadPoolExecutor(max_workers=cores) as ex:
            net.train_batch(batch(1), 1, workers=cores, executor=ex)
            t0 = time.perf_counter()
            for it in range(2, steps + 2):
                net.train_batch(batch(it), it, workers=cores, executor=ex)
            dt = time.perf_counter() - t0
        layer = net.layers[1]
        t0 = time.perf_counter()
        layer.lsh.build(layer.w)
        build_s = time.perf_counter() - t0
        dt += steps * build_s / w.n0
        return {"value": steps * per_step / dt, "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": (f"{steps} steps x {per_step} samples of {w.name} after one warm-up step through "
                           f"slide.SlideNetwork.train_batch(workers={cores}) from baseline/_ref; table build "
                           f"{build_s:.2f} s amortised over n0={w.n0}; init {init_s:.1f} s")}
    except Exception as exc:  # the port stays the arm's value
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:300]}
    finally:
        sys.path.remove(ref_dir)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL log shows the ranks and transports used
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd, env=env))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args, rank, world)), flush=True)
        return
    out, net, w = run_ours(args, rank, world)
    if rank == 0:
        if not args.no_cpu and world == 1:
            rate, dt = cpu_port_rate(w, args.cpu_samples)
            out["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": 1, "kind": "port",
                                   "sample": f"{args.cpu_samples} samples of {w.name}, sequential schedule, "
                                             f"{dt:.1f} s, rebuild excluded"}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
