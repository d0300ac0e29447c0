"""Bench workloads: one class per BASELINE.json configuration, shared by
bench.py (which times them) and the full-size parity tests (which check the
very launches the bench times: tests/test_gpu_fullsize.py).

    Config2  configs[1]  single-instance bulk fill, 4 x 2^30 f64 (e = 3, 5, 17, 65537)
    Config1  configs[0]  stream 0, 2^20 f64 per take at Mv = 1, 64, 65536
    Config3  configs[2]  65,536 instances x Mv 64 x 1024 blocks, e = 9 (strong scaling)
    Config4  configs[3]  2^20 instances x 2^16 draws fused, e = 9 (strong scaling + all-reduce)
    Config5  configs[4]  safe-prime census of [2^31, 2^32) + 2^20 instance tuples

Every workload builds its inputs once (untimed) and exposes `step()`, one
pass of the hot path over one batch, launched on torch's current stream.
Units: `numbers_per_step` is the WHOLE-JOB count (all ranks); each rank does
its shard.  The reference's own CPU timer for the path is `cli.bench_throughput`
(/root/reference/pkg/src/rsarand/cli.py:189-200); `cpu_baseline_for` times the
restated algorithm (oracle/, test infrastructure) on bounded samples of the
same workloads.
"""

from __future__ import annotations

import dataclasses
import json
import os
import statistics

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

EXPONENTS = (3, 5, 17, 65537)
M0_RNG_SEED = 181111629


def w_imad(e: int) -> int:
    """Algorithmic IMAD-class ops per draw, W(e) = 6 M(e) + 13."""
    m = e.bit_length() - 1 + bin(e).count("1") - 1
    return 6 * m + 13


def seeded_m0(n: int) -> int:
    return int(np.random.default_rng(M0_RNG_SEED).integers(0, n, dtype=np.uint64))


def _profiles_json(name: str) -> dict:
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def load_slots(key: str):
    return _profiles_json("slots.json").get(key)


def load_traffic(key: str):
    return _profiles_json("traffic.json").get(key)


def heavy_pipe(key: str, draws: int, seconds: float, peak: dict, clk: dict) -> dict | None:
    """The datapath that bounds the draw kernels: IMAD.WIDE/IMAD.HI (2 slots),
    IMAD and FP64 ops (1 slot) share 64 slots/clk/SM on B200
    (profiles/r01_probe_hybrid.txt).  Slots per draw are counted from the SASS
    (tools/slots_json.py -> profiles/slots.json); the measured peak is the
    in-run Montgomery-triple probe (3 instructions = 5 slots)."""
    spd = load_slots(key)
    if not spd:
        return None
    ach = spd * draws / seconds
    meas = peak["ops_per_s"] * 5.0 / 3.0
    out = {"slots_per_draw": spd, "achieved_tslots": ach / 1e12, "peak_tslots_measured": meas / 1e12,
           "frac_of_measured": ach / meas}
    if clk.get("sm_mhz"):
        nominal = 64.0 * peak["sms"] * clk["sm_mhz"] * 1e6
        out["peak_tslots_nominal_at_clock"] = nominal / 1e12
        out["frac_of_nominal"] = ach / nominal
    return out


def imad_roofline(e: int, draws: int, seconds: float, peak: dict, kernel: str, traffic_key: str | None,
                  slots_key: str | None, clk: dict, hbm_bytes_per_draw: int = 8) -> dict:
    """IMAD roofline of one draw kernel launch: W(e) IMAD-class ops per draw
     / launch time, against the in-run Montgomery-triple
    probe; plus the HBM write fraction and the heavy-datapath slot rate."""
    from bench import peaks
    ach = w_imad(e) * draws / seconds
    hbm_peak = peaks().get("hbm_gbs")
    hbm = hbm_bytes_per_draw * draws / seconds / 1e9
    return {"bound": "imad", "kernel": kernel, "achieved": ach / 1e12, "peak": peak["ops_per_s"] / 1e12,
            "unit": "Tops/s", "frac": ach / peak["ops_per_s"],
            "traffic": load_traffic(traffic_key) if traffic_key else None,
            "algorithmic_ops_per_draw": w_imad(e), "draws_per_launch": draws, "launch_ms": seconds * 1e3,
            "peak_source": "measured in-run: rsa_probe_imad Montgomery-triple stream (IMAD-class ops/s)",
            "hbm": {"achieved_gbs": hbm, "peak_gbs": hbm_peak,
                    "frac": hbm / hbm_peak if hbm_peak else None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"},
            "heavy_pipe": heavy_pipe(slots_key, draws, seconds, peak, clk) if slots_key else None}


# ---------------------------------------------------------------------------
# workloads

class Config2:
    """configs[1]: one instance per rank (stream id = rank, DEFAULT_MASTER_SEED),
    seeded uniform m0, Mv = 2^22; per exponent e in {3, 5, 17, 65537} one
    take_floats of 2^30 doubles (256 blocks) into HBM.  Weak scaling."""

    MV = 1 << 22
    BLOCKS = 256
    scaling = "weak"

    def __init__(self, dev, world: int, rank: int):
        import paper_1811_11629_b200 as R
        from paper_1811_11629_b200 import vecgen
        self.R = R
        base = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, rank), dev=dev)
        self.m0 = seeded_m0(base.n)
        params = {e: dataclasses.replace(base, e=e) for e in EXPONENTS}  # e=65537 bypasses validation
        st0 = R.init_vector(base, m0=self.m0, mv=self.MV, device=dev)
        self.states = {e: vecgen.VectorState(params=params[e], mv=self.MV, m1=st0.m1.clone(),
                                             m2=st0.m2.clone(), s=st0.s.clone()) for e in EXPONENTS}
        self.count = self.MV * self.BLOCKS
        import torch
        self.out = torch.empty(self.count, dtype=torch.float64, device=dev)
        self.numbers_per_step = world * len(EXPONENTS) * self.count
        self.launches_per_step = len(EXPONENTS)

    def step(self, events=None):
        import torch
        stream = torch.cuda.current_stream()
        for e in EXPONENTS:
            if events is not None:
                events[e][0].record(stream)
            self.R.take_floats(self.states[e], self.count, out=self.out)
            if events is not None:
                events[e][1].record(stream)


class Config1:
    """configs[0]: stream 0, e = 9, m0 = 0, s0 = 1; one step = a take_floats of
    2^20 doubles at each of Mv = 1 (the scalar stream), 64 (`rsarand gen`'s
    default) and 65536 (`rsarand bench`'s default).  Latency-bound at this
    size.  Every rank runs its own copy (weak)."""

    COUNT = 1 << 20
    MVS = (1, 64, 65536)
    scaling = "weak"

    def __init__(self, dev, world: int, rank: int):
        import torch
        import paper_1811_11629_b200 as R
        self.R = R
        p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0), dev=dev)
        self.states = {mv: R.init_vector(p, m0=0, s0=1, mv=mv, device=dev) for mv in self.MVS}
        self.outs = {mv: torch.empty(self.COUNT, dtype=torch.float64, device=dev) for mv in self.MVS}
        self.numbers_per_step = world * len(self.MVS) * self.COUNT

    def step(self, events=None):
        import torch
        stream = torch.cuda.current_stream()
        for mv in self.MVS:
            if events is not None:
                events[mv][0].record(stream)
            self.R.take_floats(self.states[mv], self.COUNT, out=self.outs[mv])
            if events is not None:
                events[mv][1].record(stream)


class Config3:
    """configs[2]: stream ids [0, 65536) of DEFAULT_MASTER_SEED, e = 9, m0 = 0,
    s0 = 1, Mv = 64, 1024 blocks: 2^16 doubles per instance,
    instance-major rows out[i, k*64 + g] (2^32 doubles = 32 GiB).  One step =
    ONE rsa_fill launch over this rank's contiguous id shard (strong scaling:
    the 2^32 total is fixed, no inter-GPU traffic)."""

    TOTAL, MV, BLOCKS, E = 1 << 16, 64, 1024, 9
    scaling = "strong"

    def __init__(self, dev, world: int = 1, rank: int = 0, first: int | None = None, n: int | None = None):
        import torch
        import paper_1811_11629_b200 as R
        from paper_1811_11629_b200 import vecgen
        from paper_1811_11629_b200.shard import shard_range
        sharded = first is None
        if sharded:
            first, n = shard_range(self.TOTAL, world, rank)
        self.first, self.n, self.dev = first, n, dev
        self.table = R.derive_params_table(R.DEFAULT_MASTER_SEED, first, n, dev=dev)
        self.m1, self.m2, self.s = vecgen._init_lanes(self.table.inst, n, self.MV, 0, 1, dev)
        self.out = torch.empty((n, self.BLOCKS * self.MV), dtype=torch.float64, device=dev)
        self.numbers_per_step = (self.TOTAL if sharded else n) * self.MV * self.BLOCKS
        self.local_numbers = n * self.MV * self.BLOCKS
        self.launches_per_step = 1

    def step(self):
        from paper_1811_11629_b200 import _device, _lib
        _lib.call("rsa_fill", self.table.inst.data_ptr(), self.n, self.MV, self.BLOCKS, self.E,
                  _lib.RSA_FLAG_FAST, self.m1.data_ptr(), self.m2.data_ptr(), self.s.data_ptr(), None,
                  self.out.data_ptr(), self.BLOCKS * self.MV, _device.stream(self.dev))


class Config4:
    """configs[3]: stream ids [0, 2^20), e = 9, Mv = 1, 2^16 draws per instance
    generated in registers and reduced in-kernel (A13 statistics); at N > 1
    the pooled sums are NCCL all-reduced.  Strong scaling over contiguous
    pair-aligned id shards."""

    TOTAL, DRAWS, E = 1 << 20, 1 << 16, 9
    scaling = "strong"

    def __init__(self, dev, world: int = 1, rank: int = 0, first: int | None = None, n: int | None = None):
        import paper_1811_11629_b200 as R
        from paper_1811_11629_b200.shard import shard_range
        sharded = first is None
        if sharded:
            first, n = shard_range(self.TOTAL, world, rank, align=2)
        self.R, self.world = R, world
        self.first, self.n = first, n
        self.table = R.derive_params_table(R.DEFAULT_MASTER_SEED, first, n, dev=dev)
        self.fc = R.FusedConsumer(self.table)
        self.numbers_per_step = (self.TOTAL if sharded else n) * self.DRAWS
        self.local_numbers = n * self.DRAWS
        self.launches_per_step = 3
        self.result = None

    def step(self):
        res = self.fc.run(self.DRAWS)
        if self.world > 1:
            self.R.all_reduce_pooled(res)
        self.result = res
        return res


class Config5:
    """configs[4]: the safe-prime census of every odd candidate in [2^31, 2^32)
    (production scan: sieve + base-2 SPRP + the spsp(2) table; the literal
    MR(2, 7, 61) census is timed beside it) + the 2^20 instance tuples of ids
    [0, 2^20).  At N > 1 each rank scans a contiguous sub-interval and the
    counts and lists are all-gathered."""

    scaling = "strong"

    def __init__(self, dev, world: int = 1, rank: int = 0):
        from paper_1811_11629_b200 import paramfactory
        from paper_1811_11629_b200.shard import shard_interval, shard_range
        self.dev, self.world = dev, world
        self.lo, self.hi = shard_interval(1 << 31, 1 << 32, world, rank)
        self.first, self.n = shard_range(1 << 20, world, rank)
        paramfactory.safe_prime_table(dev)  # the derivation table (built once, untimed)
        self.numbers_per_step = (1 << 30)  # odd candidates in [2^31, 2^32)
        self.launches_per_step = 8
        self.phase = {"scan": [], "setup": []}
        self.count = None

    def step(self):
        import torch
        import paper_1811_11629_b200 as R
        from paper_1811_11629_b200 import paramfactory
        st = torch.cuda.current_stream()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        sp = paramfactory.safe_primes_u32(self.lo, self.hi, self.dev)
        if self.world > 1:
            from paper_1811_11629_b200.shard import gather_sorted
            sp = gather_sorted(sp.view(torch.int32))
        e1.record(st)
        R.derive_params_table(R.DEFAULT_MASTER_SEED, self.first, self.n, dev=self.dev)
        e2.record(st)
        self._pending = (e0, e1, e2, sp)

    def collect(self):
        e0, e1, e2, sp = self._pending
        e2.synchronize()
        self.phase["scan"].append(e0.elapsed_time(e1))
        self.phase["setup"].append(e1.elapsed_time(e2))
        self.count = int(sp.numel())


def literal_mr_scan(steps: int, lo: int, hi: int, dev, want_count: int, peak: dict) -> dict:
    """The census exactly as BASELINE config 5 words it (MR 2, 7, 61 on every
    odd n and on (n-1)/2; rsa_safe_prime_scan_mr), timed beside the production
    scan.  Roofline: SURVEY §8(d)'s 55.5 Montgomery products per odd candidate
    against the in-run Montgomery-triple probe (products/s)."""
    import torch
    from paper_1811_11629_b200 import paramfactory
    st = torch.cuda.current_stream()
    paramfactory.safe_primes_u32(lo, hi, dev, literal_mr=True)  # warm-up
    times = []
    for _ in range(max(1, min(steps, 3))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        sp = paramfactory.safe_primes_u32(lo, hi, dev, literal_mr=True)
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    ms = statistics.median(times)
    cands = (hi - lo) // 2
    products = 55.5 * cands
    pk = peak["ops_per_s"] / 3.0  # Montgomery triples (products) per second
    return {"ms": ms, "gcandidates_s": cands / (ms * 1e-3) / 1e9, "safe_primes_found": int(sp.numel()),
            "equal_count": int(sp.numel()) == want_count,
            "roofline": {"bound": "imad", "kernel": "k_mr_base2 + k_mr_rest",
                         "achieved": products / (ms * 1e-3) / 1e12, "peak": pk / 1e12,
                         "unit": "T Montgomery products/s", "frac": products / (ms * 1e-3) / pk,
                         "algorithmic_products_per_candidate": 55.5},
            "note": "literal MR(2,7,61) census (no sieve, no pseudoprime table); the production scan "
                    "(phases.scan_ms) returns the same list"}


# ---------------------------------------------------------------------------
# CPU baselines per configuration (rank 0, N = 1, bounded samples): the
# reference's algorithm restated in oracle/ (test infrastructure), timed on
# the box's host cores the way each configuration's workload runs.

def _stream0():
    from oracle import rsa_oracle as O
    with open(os.path.join(ROOT, "tests", "golden", "regression.json")) as fh:
        return O.from_fields(json.load(fh)["params"])


_C2_SEEDS: np.ndarray | None = None


def _c2_lane_seeds(n_lanes: int) -> np.ndarray:
    """Skip seeds of the first n_lanes lanes of config 2's Mv = 2^22 vector
    (s0 = 1: lane g starts at a^(g * floor((q-1)/Mv)) mod q, skipgen.py:124-138),
    by one modular product per lane."""
    global _C2_SEEDS
    if _C2_SEEDS is None or len(_C2_SEEDS) < n_lanes:
        P = _stream0()
        A = pow(P.a, (P.q - 1) // Config2.MV, P.q)
        out, x = [], 1
        for _ in range(n_lanes):
            out.append(x)
            x = x * A % P.q
        _C2_SEEDS = np.array(out, dtype=np.uint64)
    return _C2_SEEDS[:n_lanes]


def config2_desc(world: int, m0: int) -> dict:
    """The `config` object of the config-2 line (both arms)."""
    return {"workload": "config2 bulk fill: 2^30 f64 per exponent e in {3,5,17,65537}, Mv=2^22, 256 blocks, "
                        "one instance per GPU",
            "global_numbers_per_step": world * len(EXPONENTS) * Config2.MV * Config2.BLOCKS,
            "mv": Config2.MV, "blocks": Config2.BLOCKS, "exponents": list(EXPONENTS), "m0": m0,
            "l2": "outputs 8 GiB per fill (> L2), no flush needed",
            "parallelism": f"independent instances x{world}"}


def _cpu_cfg2(args):
    """vecgen's lockstep path (numpy port) over lanes [lo, hi) of config 2's
    Mv = 2^22 vector (stream 0, seeded m0), for each bench exponent."""
    import time
    from oracle import rsa_oracle as O
    e_list, blocks, lo, hi = args
    P0 = _stream0()
    m0 = seeded_m0(P0.n)
    s0 = _c2_lane_seeds(hi)[lo:hi].copy()
    out = {}
    for e in e_list:
        P = dataclasses.replace(P0, e=e)
        m1 = np.full(hi - lo, m0 % P.p1, dtype=np.uint64)
        m2 = np.full(hi - lo, m0 % P.p2, dtype=np.uint64)
        s = s0.copy()
        O.block_raw(m1, m2, s, P)  # warm-up
        t0 = time.perf_counter()
        for _ in range(blocks):
            raw, m1, m2, s = O.block_raw(m1, m2, s, P)
            O.floats_from_raw(raw, P)
        out[e] = (blocks * (hi - lo), time.perf_counter() - t0)
    return out


def cpu_port_rate(procs: int | None = None, blocks: int = 4, lanes_per_proc: int = 65536) -> dict:
    """Aggregate numbers/s of the numpy port of vecgen's lockstep path on a
    bounded sample of config 2 itself: each process advances its own
    contiguous 65536-lane slice (the reference CLI bench's vector width,
    cli.py:26) of the Mv = 2^22 vector for `blocks` blocks at every bench
    exponent, all host cores; the step's exponent mix weighted equally per draw."""
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    _c2_lane_seeds(procs * lanes_per_proc)  # in the parent: the forked workers share it
    jobs = [(EXPONENTS, blocks, k * lanes_per_proc, (k + 1) * lanes_per_proc) for k in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cpu_cfg2, jobs)
    per_e = {}
    for e in EXPONENTS:
        draws = sum(r[e][0] for r in res)
        wall = max(r[e][1] for r in res)
        per_e[e] = draws / wall
    rate = len(EXPONENTS) / sum(1.0 / per_e[e] for e in EXPONENTS)  # equal draws per e
    draws = sum(r[e][0] for r in res for e in EXPONENTS)
    return {"value": rate / 1e9, "unit": "Gnumbers/s", "cores": procs, "kind": "port",
            "per_e": {str(e): per_e[e] / 1e9 for e in EXPONENTS},
            "sample": f"config 2 itself on a bounded sample: lanes [0, {procs * lanes_per_proc}) of the Mv=2^22 "
                      f"vector (stream 0, seeded m0), {blocks} blocks per e in {list(EXPONENTS)}, one "
                      f"{lanes_per_proc}-lane slice per process ({procs} processes, {draws} draws); numpy port "
                      f"of vecgen's lockstep path (oracle/rsa_oracle.py); {os.cpu_count()} host cores"}


def _cpu_cfg1(count):
    """Scalar stream (Mv = 1): the rsacore per-draw path in Python ints."""
    import time
    from oracle import rsa_oracle as O
    P = _stream0()
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
    """cpu_baseline object of configuration `config` (rank 0, N = 1), measured
    in a fresh Python process (`python bench_configs.py cpu N [instances]`):
    worker processes forked from the GPU process (CUDA context, gigabytes of
    pinned host memory) ran the same numpy work ~40 % slower than the same
    port in a clean process (profiles/r02_bench_default.json vs the reference
    arm).  `table`: the InstanceTable the GPU run derived (configs 3 and 4)."""
    import subprocess
    import sys
    insts = []
    if table is not None and config in (3, 4):
        n = (os.cpu_count() or 1) * (4 if config == 4 else 1)
        insts = [[p.p1, p.p2, p.skip.a] for p in (table.params(j) for j in range(n))]
    res = subprocess.run([sys.executable, os.path.abspath(__file__), "cpu", str(config), json.dumps(insts)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        return {"unavailable": res.stderr.strip().splitlines()[-1] if res.stderr.strip() else "failed"}
    return json.loads(res.stdout.strip().splitlines()[-1])


class _Inst:
    """The (p1, p2, a) of an instance, shaped like GeneratorParams for the ports."""

    def __init__(self, p1, p2, a):
        self.p1, self.p2 = p1, p2
        self.skip = type("S", (), {"a": a})()


class _Table:
    def __init__(self, insts):
        self.insts = [_Inst(*x) for x in insts]

    def params(self, j):
        return self.insts[j]


def _cpu_baseline_here(config: int, table=None) -> dict | None:
    import multiprocessing as mp
    from oracle import rsa_oracle as O
    procs = os.cpu_count() or 1
    if config == 2:
        # the box's vCPUs are noisy (+-40 % between back-to-back runs, tools/cpu_probe.py):
        # best of three, the reference's most favourable figure
        cb = max((cpu_port_rate() for _ in range(3)), key=lambda r: r["value"])
        cb["sample"] += " (best of 3 runs)"
        one = cpu_port_rate(procs=1)  # also the single-process figure
        cb["one_process"] = {"value": one["value"], "unit": one["unit"], "cores": 1}
        return cb
    if config == 1:
        n = 1 << 17
        draws, wall = _cpu_cfg1(n)
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
        recs = [table.params(j) for j in range(per * procs)]
        plist = [(p.p1, p.p2, p.skip.a) for p in recs]
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
        with mp.get_context("fork").Pool(n5) as pool:
            res = pool.map(_cpu_cfg5, jobs)
        return {"value": sum(d for d, _ in res) / max(w for _, w in res) / 1e9, "unit": "Gcandidates/s",
                "cores": n5, "kind": "port",
                "sample": f"safe-prime census of {n5} disjoint 2^27-wide windows from 2^31, one per "
                          f"process (C restatement of the reference's segmented sieve, "
                          f"paramfactory.py:85-130; faster than the reference's numpy sieve)"}
    return None


def run_battery_config(args, world, rank, local, dev) -> dict:
    """--config 6 (F1, builder runs): the full chi-square battery (13 core
    tests + 10 low-bit reruns, stats.run_battery, stats.py:548-581) on 2
    interleaved streams at the reference's DEFAULT_BUDGET (1e8 per test)."""
    import time
    import torch
    import paper_1811_11629_b200 as R
    from bench import METRIC, ClockSampler
    from paper_1811_11629_b200 import bitsource, stats
    budget = 100_000_000
    plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, 9, 2, dev=dev)

    def make(sel):
        return bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=1 << 16, device=dev) for p in plist], sel)

    for _ in range(max(1, args.warmup)):
        stats.run_battery(make, budget=budget)  # warm-up (allocator, cuFFT plans, pinned buffers)
    torch.cuda.synchronize()
    from bench import barrier_sync, launch_count, max_over_ranks
    walls = []
    with ClockSampler(local) as clk:
        for _ in range(max(1, min(args.steps, 5))):
            barrier_sync(world)
            c0 = launch_count()
            t0 = time.perf_counter()
            rep = stats.run_battery(make, budget=budget)
            torch.cuda.synchronize()
            walls.append(max_over_ranks(time.perf_counter() - t0, world))  # every rank runs its own battery
            launches = launch_count() - c0
    el = statistics.median(walls)
    variates = world * sum(r.samples for r in rep.reports)
    return {"metric": METRIC, "value": variates / el / 1e9, "unit": "Gvariates/s", "n_gpus": world,
            "steps": len(walls), "warmup": max(1, args.warmup), "ms_per_step": el * 1e3,
            "wall_ms_each": [w * 1e3 for w in walls], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 draws -> f64 / low bits", "data": "synthetic: derived stream params",
            "config": {"workload": "config6 (F1): stats.run_battery, 23 tests at budget 1e8 each, "
                                   "2 interleaved streams (9, 10), Mv=2^16; wall time per battery (median)"},
            "clocks": clk.summary(), "gpu_launches": launches,
            "battery": {"tests": len(rep.reports), "errors": rep.errors, "all_pass": rep.all_pass,
                        "n_outside_warn": rep.n_outside_warn, "records": [r.record() for r in rep.reports]},
            "reference_context": ("reference run_battery at budget 2^23 took 57.6 s on one CPU core here "
                                  "(tests/golden/battery.json): 3.35e6 variates/s")}


if __name__ == "__main__":
    import sys
    if len(sys.argv) >= 3 and sys.argv[1] == "cpu":
        sys.path.insert(0, ROOT)
        insts = json.loads(sys.argv[3]) if len(sys.argv) > 3 else []
        print(json.dumps(_cpu_baseline_here(int(sys.argv[2]), _Table(insts) if insts else None)))
