"""Secondary bench configurations (bench.py --config 3|4|5): BASELINE.json
configs[2..4].  Same timing rules as bench.py (events on the launch stream,
barrier + synchronize both sides, max over ranks)."""

from __future__ import annotations

import statistics

import bench


def _time_steps(args, world, fn, local):
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        fn()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bench.barrier_sync(world)
    with bench.ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            fn()
        t1.record(stream)
        bench.barrier_sync(world)
    return bench.max_over_ranks(t0.elapsed_time(t1) * 1e-3, world), clk.summary()


def _base_line(args, world, value, elapsed, clk, config, launches):
    return {"metric": bench.METRIC, "value": value, "unit": "Gnumbers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32 Montgomery / u64 skip + f64 map", "data": "synthetic: derived stream params",
            "config": config, "clocks": clk, "gpu_launches": launches}


def run_other(args, world, rank, local):
    import torch
    import paper_1811_11629_b200 as R
    from paper_1811_11629_b200 import _device, _lib, vecgen
    from paper_1811_11629_b200.shard import shard_range
    dev = torch.device("cuda", local)
    peak = bench.probe_imad_peak(dev)

    if args.config == 3:
        total, mv, blocks = 1 << 16, 64, 1024
        first, n = shard_range(total, world, rank)
        t = R.derive_params_table(R.DEFAULT_MASTER_SEED, first, n, dev=dev)
        m1, m2, s = vecgen._init_lanes(t.inst, n, mv, 0, 1, dev)
        out = torch.empty((n, blocks * mv), dtype=torch.float64, device=dev)

        def fn():
            _lib.call("rsa_fill", t.inst.data_ptr(), n, mv, blocks, 9, _lib.RSA_FLAG_FAST,
                      m1.data_ptr(), m2.data_ptr(), s.data_ptr(), None, out.data_ptr(),
                      blocks * mv, _device.stream(dev))

        el, clk = _time_steps(args, world, fn, local)
        numbers = total * mv * blocks
        line = _base_line(args, world, numbers * args.steps / el / 1e9, el, clk,
                          {"workload": "config3: 65536 instances (ids 0..65535), e=9, Mv=64, 1024 blocks, "
                                       "2^16 f64 each, instance-major, sharded by contiguous id range",
                           "l2": "32 GiB output per step (> L2)"}, args.steps)
        per = el / args.steps
        line["roofline"] = {"bound": "imad", "achieved": bench.w_imad(9) * numbers / world / per / 1e12,
                            "peak": peak["ops_per_s"] / 1e12, "unit": "Tops/s",
                            "frac": bench.w_imad(9) * numbers / world / per / peak["ops_per_s"],
                            "traffic": bench.load_traffic("fill_c3")}
        line["_table"] = t  # for the rank-0 CPU baseline (bench.run_gpu)
        return line

    if args.config == 4:
        total, N = 1 << 20, 1 << 16
        first, n = shard_range(total, world, rank, align=2)
        t = R.derive_params_table(R.DEFAULT_MASTER_SEED, first, n, dev=dev)
        fc = R.FusedConsumer(t)
        box = {}

        def fn():
            res = fc.run(N)
            if world > 1:
                R.all_reduce_pooled(res)
            box["res"] = res

        el, clk = _time_steps(args, world, fn, local)
        numbers = total * N
        line = _base_line(args, world, numbers * args.steps / el / 1e9, el, clk,
                          {"workload": "config4 fused consumer: 2^20 instances x 2^16 draws, Mv=1, e=9; "
                                       "per-instance mean/var/lag-1/64-bin hist + pooled pair correlation; "
                                       "NCCL all-reduce of pooled stats", "l2": "no stream in HBM"},
                          args.steps * (3 + (2 if world > 1 else 0)))
        per = el / args.steps
        line["roofline"] = {"bound": "imad", "achieved": bench.w_imad(9) * numbers / world / per / 1e12,
                            "peak": peak["ops_per_s"] / 1e12, "unit": "Tops/s",
                            "frac": bench.w_imad(9) * numbers / world / per / peak["ops_per_s"],
                            "traffic": bench.load_traffic("fused")}
        line["pooled_correlation"] = box["res"].pooled_correlation(total // 2)
        line["_table"] = t  # for the rank-0 CPU baseline (bench.run_gpu)
        return line

    if args.config == 1:
        # config 1: one instance (stream 0), 2^20 draws at Mv = 1 (the scalar
        # stream), 64 (`rsarand gen` default) and 65536 (`rsarand bench` default)
        p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0), dev=dev)
        count = 1 << 20
        per_mv = {}
        stream = torch.cuda.current_stream()
        for mv in (1, 64, 65536):
            st = R.init_vector(p, m0=0, s0=1, mv=mv, device=dev)
            out = torch.empty(count, dtype=torch.float64, device=dev)
            for _ in range(args.warmup):
                R.take_floats(st, count, out=out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            bench.barrier_sync(world)
            a.record(stream)
            for _ in range(args.steps):
                R.take_floats(st, count, out=out)
            b.record(stream)
            b.synchronize()
            per_mv[str(mv)] = {"ms_per_2e20": a.elapsed_time(b) / args.steps,
                               "gnumbers_s": count * args.steps / (a.elapsed_time(b) * 1e-3) / 1e9}
        el = sum(v["ms_per_2e20"] for v in per_mv.values()) * 1e-3 * args.steps
        line = _base_line(args, world, 3 * count * args.steps / el / 1e9, el, {"sm_mhz": None},
                          {"workload": "config1: stream 0, e=9, 2^20 f64 per take_floats at Mv=1, 64, 65536 "
                                       "(Mv<2^17 lanes are split across threads: rsa_fill_segmented)"},
                          args.steps * 3 * 3)
        line["per_mv"] = per_mv
        line["reference_context"] = ("reference scalar rsacore.take_raws 2.35 us/draw (4.26e5/s) and "
                                     "vecgen bench_throughput 1.18e7/s at Mv=65536, one core (SURVEY §6)")
        return line

    if args.config == 6:
        # F1: the full chi-square battery (13 core tests + 10 low-bit reruns)
        # on 2 interleaved streams at the reference's DEFAULT_BUDGET (1e8 per test)
        import time
        from paper_1811_11629_b200 import bitsource, stats
        budget = 100_000_000
        plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2, dev=dev)

        def make(sel):
            return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16, device=dev)
                                        for p in plist], sel)

        stats.run_battery(make, budget=1 << 23)  # warm-up (allocator, cuFFT plans)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = stats.run_battery(make, budget=budget)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        variates = sum(r.samples for r in rep.reports)
        line = _base_line(args, world, variates / el / 1e9, el * args.steps, {"sm_mhz": None},
                          {"workload": "config6 (F1): stats.run_battery, 23 tests at budget 1e8 each, "
                                       "2 interleaved streams (9, 10), Mv=2^16"}, None)
        line["unit"] = "Gvariates/s"
        line["ms_per_step"] = el * 1e3
        line["battery"] = {"tests": len(rep.reports), "errors": rep.errors, "all_pass": rep.all_pass,
                           "n_outside_warn": rep.n_outside_warn,
                           "records": [r.record() for r in rep.reports]}
        line["reference_context"] = ("reference run_battery at budget 2^23 took 57.6 s on one CPU core here "
                                     "(tests/golden/battery.json): 3.35e6 variates/s")
        return line

    # config 5: safe-prime scan of [2^31, 2^32) + 2^20 instance tuples
    from paper_1811_11629_b200 import paramfactory
    lo_all, hi_all = 1 << 31, 1 << 32
    span = (hi_all - lo_all) // world
    lo = lo_all + rank * span
    hi = hi_all if rank == world - 1 else lo + span
    first, n = shard_range(1 << 20, world, rank)
    paramfactory.safe_prime_table(dev)  # the derivation table (built once, untimed)

    phase = {"scan": [], "setup": []}

    def fn():
        st = torch.cuda.current_stream()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        sp = paramfactory.safe_primes_u32(lo, hi, dev)
        if world > 1:  # all-gather the per-rank counts and lists -> the global table
            from paper_1811_11629_b200.shard import gather_sorted
            sp = gather_sorted(sp.view(torch.int32))
        e1.record(st)
        R.derive_params_table(R.DEFAULT_MASTER_SEED, first, n, dev=dev)
        e2.record(st)
        e2.synchronize()
        phase["scan"].append(e0.elapsed_time(e1))
        phase["setup"].append(e1.elapsed_time(e2))
        phase["count"] = int(sp.numel())

    el, clk = _time_steps(args, world, fn, local)
    cands = (hi_all - lo_all) // 2
    line = _base_line(args, world, cands * args.steps / el / 1e9, el, clk,
                      {"workload": "config5 setup: safe-prime scan (sieve to 8191, base-2 SPRP, spsp(2) table) of all 2^30 odd candidates in "
                                   "[2^31,2^32) + 2^20 instance tuples (ids 0..2^20-1)",
                       "unit_note": "value = odd candidates per second (scan + tuples in the step; at N>1 the scan phase includes the all-gather of the per-rank counts and lists)"},
                      args.steps * 5)
    line["unit"] = "Gcandidates/s"
    scan_ms = statistics.median(phase["scan"][-args.steps:])
    setup_ms = statistics.median(phase["setup"][-args.steps:])
    line["phases"] = {"scan_ms": scan_ms, "scan_gcandidates_s": cands / world / (scan_ms * 1e-3) / 1e9,
                      "safe_primes_found": phase["count"], "setup_ms": setup_ms,
                      "tuples_per_s": n / (setup_ms * 1e-3)}
    if world == 1:
        line["literal_mr"] = literal_mr_scan(args, lo, hi, dev, phase["count"])
    return line


def literal_mr_scan(args, lo, hi, dev, want_count):
    """The census exactly as BASELINE config 5 words it (MR 2, 7, 61 on every
    odd n and on (n-1)/2; rsa_safe_prime_scan_mr), timed beside the production
    scan.  Roofline: SURVEY §8(d)'s 55.5 Montgomery products per odd candidate
    against the in-run Montgomery-triple probe (products/s)."""
    import torch
    from bench import probe_imad_peak
    from paper_1811_11629_b200 import paramfactory
    st = torch.cuda.current_stream()
    paramfactory.safe_primes_u32(lo, hi, dev, literal_mr=True)  # warm-up
    times = []
    for _ in range(max(1, min(args.steps, 3))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        sp = paramfactory.safe_primes_u32(lo, hi, dev, literal_mr=True)
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    ms = statistics.median(times)
    cands = (hi - lo) // 2
    products = 55.5 * cands
    peak = probe_imad_peak(dev)["ops_per_s"] / 3.0  # Montgomery triples (products) per second
    return {"ms": ms, "gcandidates_s": cands / (ms * 1e-3) / 1e9, "safe_primes_found": int(sp.numel()),
            "equal_count": int(sp.numel()) == want_count,
            "roofline": {"bound": "imad", "kernel": "k_mr_base2 + k_mr_rest",
                         "achieved": products / (ms * 1e-3) / 1e12, "peak": peak / 1e12,
                         "unit": "T Montgomery products/s", "frac": products / (ms * 1e-3) / peak,
                         "algorithmic_products_per_candidate": 55.5},
            "note": "literal MR(2,7,61) census (no sieve, no pseudoprime table); the production scan "
                    "(phases.scan_ms) returns the same list"}


# ---------------------------------------------------------------------------
# CPU baselines per configuration (rank 0, N = 1, bounded samples): the
# reference's algorithm restated in oracle/ (test infrastructure), timed on
# the box's host cores the way each configuration's workload runs.

def _cpu_cfg1(args):
    """Scalar stream (Mv = 1): the rsacore per-draw path in Python ints."""
    import time
    from oracle import rsa_oracle as O
    P, count = args
    t = time.perf_counter()
    O.scalar_raws(P, count)
    return count, time.perf_counter() - t


def _cpu_cfg3(args):
    """One config-3 instance: the numpy lockstep port at Mv = 64, e = 9."""
    import time
    from oracle import rsa_oracle as O
    P, blocks = args
    st = O.init(P, m0=0, s0=1, mv=64)
    m1, m2, s = st.m1.copy(), st.m2.copy(), st.s.copy()
    t = time.perf_counter()
    for _ in range(blocks):
        raw, m1, m2, s = O.block_raw(m1, m2, s, P)
        O.floats_from_raw(raw, P)
    return blocks * 64, time.perf_counter() - t


def _cpu_cfg4(args):
    """Config-4 instances: the C restatement draws each Mv = 1 stream, the
    numpy restatement of the A13 statistics reduces them."""
    import time
    import numpy as np
    from oracle import coracle
    from oracle import rsa_oracle as O
    plist, N = args
    one = lambda v: np.array([v], dtype=np.uint64)
    t = time.perf_counter()
    rows = []
    for (p1, p2, a) in plist:
        _, f = coracle.fill(coracle.params(p1, p2, 9, a), one(0), one(0), one(1), N, raw=False)
        rows.append(f.reshape(-1))
    O.fused_reference(np.stack(rows))
    return len(plist) * N, time.perf_counter() - t


def _cpu_cfg5(args):
    """A window of the census: the C restatement of the segmented sieve."""
    import time
    from oracle import coracle
    lo, hi = args
    t = time.perf_counter()
    coracle.census(lo, hi)
    return (hi - lo) // 2, time.perf_counter() - t


def cpu_baseline_for(config: int, table=None) -> dict | None:
    """cpu_baseline object for bench.py --config N (N != 2; config 2 uses
    bench.cpu_port_rate).  `table`: the derived InstanceTable of the run."""
    import multiprocessing as mp
    import os
    from oracle import rsa_oracle as O
    procs = os.cpu_count() or 1
    with open(os.path.join(bench.ROOT, "tests", "golden", "regression.json")) as fh:
        import json
        P0 = O.from_fields(json.load(fh)["params"])
    if config == 1:
        n = 1 << 17
        draws, wall = _cpu_cfg1((P0, n))
        return {"value": draws / wall / 1e9, "unit": "Gnumbers/s", "cores": 1, "kind": "port",
                "sample": f"{n} scalar draws of stream 0 (oracle.scalar_raws: rsacore's per-draw path in "
                          f"Python ints, rsacore.py:236-258), one process"}
    if config == 3:
        plist = [table.params(j) for j in range(procs)]
        jobs = [(O.Params(p.p1, p.p2, 9, p.skip.a), 400) for p in plist]
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_cfg3, jobs)
        return {"value": sum(d for d, _ in res) / max(w for _, w in res) / 1e9, "unit": "Gnumbers/s",
                "cores": procs, "kind": "port",
                "sample": f"{procs} config-3 instances (ids 0..{procs - 1}), one per process, 400 blocks of "
                          f"Mv = 64 each (numpy lockstep port of vecgen, e = 9)"}
    if config == 4:
        per = 4
        plist = [(table.params(j).p1, table.params(j).p2, table.params(j).skip.a) for j in range(per * procs)]
        N = 1 << 16
        jobs = [(plist[per * k:per * k + per], N) for k in range(procs)]
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_cfg4, jobs)
        return {"value": sum(d for d, _ in res) / max(w for _, w in res) / 1e9, "unit": "Gnumbers/s",
                "cores": procs, "kind": "port",
                "sample": f"{per * procs} config-4 instances x {N} draws, {per} per process (C restatement "
                          f"draws + numpy A13 statistics)"}
    if config == 5:
        span = 1 << 27
        n5 = min(procs, (1 << 31) // span)  # disjoint windows inside [2^31, 2^32)
        jobs = [((1 << 31) + k * span, (1 << 31) + (k + 1) * span) for k in range(n5)]
        procs = n5
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_cfg5, jobs)
        return {"value": sum(d for d, _ in res) / max(w for _, w in res) / 1e9, "unit": "Gcandidates/s",
                "cores": procs, "kind": "port",
                "sample": f"safe-prime census of {procs} disjoint 2^27-wide windows from 2^31, one per "
                          f"process (C restatement of the reference's segmented sieve, "
                          f"paramfactory.py:85-130; faster than the reference's numpy sieve)"}
    return None
