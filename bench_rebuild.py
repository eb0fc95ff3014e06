"""Rebuild microbenchmark (the "rebuild" config row).

670,091 W2 rows x 128 with N(0, 0.01) entries (0.01 read as the standard
deviation; SimHash codes are invariant to positive scaling and DWTA codes to
monotone transforms, so only fp magnitudes depend on it), for both families
of the BASELINE configs:

* DWTA K=8 L=50 m=8, reservoir buckets (wide-out's tables);
* SimHash K=9 L=50 s=1/3, FIFO buckets (wide-in's tables);

timing, with CUDA events on the device, the build split into the row hash
and the table build (sort + runs + directory, + the host MT19937 replay for
reservoir overflows), and separately the query + union of 4,096 dense N(0,1)
queries (hash, L probes, union = hard_threshold(min_freq=1)).  One JSON line
per family; `value` = hash + build ms per rebuild.  The CPU baseline is the
numpy oracle on a row subsample, extrapolated linearly and labelled so.

usage: python bench_rebuild.py [--rows N] [--queries Q] [--repeats R] [--cpu-rows M] [--no-cpu]
"""

import argparse
import json
import os
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

# per-build algorithmic bytes: W2 read + stored ids + directory
BYTES = {"dwta": 0.87e9, "simhash": 0.36e9}


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def events_ms(fn, repeats):
    import torch

    out = []
    for _ in range(repeats):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out)), out


def cpu_port(family_name, fam, rows, queries, cpu_rows):
    """Oracle (numpy, 1 thread) on cpu_rows rows and 256 queries, per-row /
    per-query rates extrapolated to the full sizes."""
    from threadpoolctl import threadpool_limits

    from oracle import slide_oracle as O

    with threadpool_limits(1):
        if family_name == "simhash":
            params = O.SimHashParams(fam.dim, fam.k, fam.l, fam.proj_indices, fam.proj_signs)
            keyfn = lambda w: O.simhash_keys(params, w)  # noqa: E731
            policy = "fifo"
        else:
            params = O.dwta_params(fam.dim, fam.k, fam.l, fam.bin_size, fam.config.seed)
            keyfn = lambda w: O.dwta_keys(params, w)  # noqa: E731
            policy = "reservoir"
        sub = rows[:cpu_rows]
        t0 = time.perf_counter()
        keys = keyfn(sub)
        t1 = time.perf_counter()
        import random

        O.build_buckets(keys, 128, policy, random.Random(1))
        t2 = time.perf_counter()
    scale = rows.shape[0] / cpu_rows
    return {"hash_s": (t1 - t0) * scale, "build_s": (t2 - t1) * scale,
            "sample": f"{cpu_rows} of {rows.shape[0]} rows, numpy oracle, 1 thread, extrapolated linearly"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=670_091)
    p.add_argument("--queries", type=int, default=4096)
    p.add_argument("--repeats", type=int, default=5)
    p.add_argument("--cpu-rows", type=int, default=20_000)
    p.add_argument("--no-cpu", action="store_true")
    args = p.parse_args()

    import torch

    from paper_1903_03129_b200 import HashFamilyConfig, LshTables, new_hash_family
    from paper_1903_03129_b200 import _device

    rng = np.random.default_rng(2024)
    rows_np = (0.01 * rng.standard_normal((args.rows, 128))).astype(np.float32)
    q_np = rng.standard_normal((args.queries, 128)).astype(np.float32)
    x = _device.pad_rows(rows_np, 128)
    q = _device.pad_rows(q_np, 128)
    for name, cfg, policy in (
        ("dwta", HashFamilyConfig("dwta", 8, 50, 128, wta_bin_size=8, seed=7919), "reservoir"),
        ("simhash", HashFamilyConfig("simhash", 9, 50, 128, seed=7919), "fifo"),
    ):
        fam = new_hash_family(cfg)
        tbl = LshTables(fam, policy=policy, capacity=128, seed=1)
        keys = torch.empty((args.rows, fam.l), dtype=torch.int32, device=x.device)
        tbl.build(rows_np[:1024])  # context + first allocations outside the timing
        fam._keys_dev(x, args.rows, 128, keys)
        tbl._insert_dev(keys, args.rows)
        hash_ms, _ = events_ms(lambda: fam._keys_dev(x, args.rows, 128, keys), args.repeats)
        build_ms, _ = events_ms(lambda: tbl._insert_dev(keys, args.rows), args.repeats)
        tbl._views = None
        query_ms, _ = events_ms(lambda: tbl._query_union_dev(q, args.queries, return_device=True), args.repeats)
        cnt, _ids = tbl._query_union_dev(q, args.queries, return_device=True)
        mean_union = float(cnt.double().mean().item())
        total = hash_ms + build_ms
        line = {
            "metric": "table rebuild, hash + build (ms per rebuild)", "value": total, "unit": "ms",
            "higher_is_better": False, "n_gpus": 1, "dtype": "f32", "data": "synthetic N(0, 0.01) rows",
            "config": {"workload": "rebuild", "family": name, "k": fam.k, "l": fam.l, "policy": policy,
                       "capacity": 128, "rows": args.rows, "queries": args.queries},
            "hash_ms": hash_ms, "build_ms": build_ms,
            "query_union_ms": query_ms, "queries_per_s": args.queries / (query_ms / 1e3),
            "mean_union_size": mean_union,
            "roofline": {"bound": "hbm", "achieved": BYTES[name] / (total / 1e3) / 1e9, "peak": peak_gbs(),
                         "unit": "GB/s", "frac": BYTES[name] / (total / 1e3) / 1e9 / peak_gbs(),
                         "traffic": None, "bytes_per_build": BYTES[name]},
        }
        if not args.no_cpu:
            cpu = cpu_port(name, fam, rows_np.astype(np.float64), q_np, min(args.cpu_rows, args.rows))
            line["cpu_baseline"] = {"value": (cpu["hash_s"] + cpu["build_s"]) * 1e3, "unit": "ms", "cores": 1,
                                    "kind": "port", "sample": cpu["sample"], "hash_ms": cpu["hash_s"] * 1e3,
                                    "build_ms": cpu["build_s"] * 1e3}
        print(json.dumps(line), flush=True)
        del tbl, keys
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
