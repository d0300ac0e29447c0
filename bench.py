"""Benchmark harness (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..6] [--impl ours|reference]

`--gpus N` with N > 1 outside torchrun re-launches this script under
`torch.distributed.run --nproc-per-node N` (127.0.0.1); under torchrun the
world size must equal N.  One process per GPU, NCCL.

Default run: BASELINE.json configs[1] ("single instance bulk fill") is the
headline `value`; the other configurations are measured in the same run and
reported under `configs` (bench_configs.py holds the workloads):

  value    config 2: per rank one generator instance (stream id = rank), Mv =
           2^22, seeded m0; for each e in {3, 5, 17, 65537} a fill of 2^30
           float64 (256 blocks) into HBM.  One step = the four fills.  Weak
           scaling (independent instances, no data-path collective).  Outputs
           are 8 GiB per fill (> 126 MB L2): no flush needed.
  configs  "1" (stream 0, 2^20 draws at Mv 1/64/65536), "3" (65,536 instances,
           strong scaling), "4" (2^20 instances fused + all-reduce, strong),
           "5" (safe-prime census + 2^20 tuples): each with its own value,
           device-timed K-step blocks, clocks, roofline and (N = 1) cpu_baseline.

`e2e`      config 2 through the public API with the lane state resumed from
           pinned host memory and every output copied to pinned host memory.
`roofline` the dominant kernel of config 2 against the measured
           Montgomery-triple IMAD peak, plus its HBM fraction.
`cpu_baseline` the reference's algorithm (oracle/ port) on bounded samples,
           all host cores, rank 0 at N = 1 only.
`--impl reference` times that same CPU port as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bench_configs as C  # noqa: E402
from bench_configs import EXPONENTS, cpu_port_rate, seeded_m0, w_imad  # noqa: E402,F401

METRIC = "RSA-PRNG Gnumbers/s at 1/2/4/8 B200; % of IMAD/HBM roofline; vs CPU"
SUB_CONFIGS = (1, 3, 4, 5, 6)
MIN_REGION_S = 0.5  # short steps are timed in repeated K-step blocks until the sampler saw this much


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# clocks sampler (NVML every 5 ms during the timed region; nvidia-smi fallback)

_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


class ClockSampler:
    """SM clock and throttle reasons sampled while the timed region runs.

    NVML (pynvml) is polled from a thread every 5 ms, so even a 0.1 s region
    yields ~20 samples; without NVML, `nvidia-smi -lms 50` as the recipe's
    clocks line.  summary() -> {sm_mhz (median), sm_max_mhz, reasons, samples}.
    """
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")
    PERIOD_S = 0.005

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.rows: list[tuple] = []  # (sm_mhz, max_mhz, reason names)
        self._first = threading.Event()
        self._stop = threading.Event()
        self.source = "none"

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = self._nvml_handle(pynvml)
            self._bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.source = "nvml/5ms"
            self.thread = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={','.join(self.FIELDS)}",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.source = "nvidia-smi/50ms"
                self.thread = threading.Thread(target=self._read, daemon=True)
            except OSError:
                self.proc = None
                return self
        self.thread.start()
        self._first.wait(timeout=5.0)  # sampling has started before the timed region
        return self

    def _nvml_handle(self, pynvml):
        # the CUDA device this rank uses, matched by PCI bus id (CUDA_VISIBLE_DEVICES may remap)
        try:
            import torch
            props = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        pynvml = self.nvml
        while not self._stop.is_set():
            try:
                sm = float(pynvml.nvmlDeviceGetClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
                bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.rows.append((sm, self.max_mhz, tuple(n for n, b in zip(_REASONS, self._bits) if bits & b)))
            except Exception:
                pass
            self._first.set()
            self._stop.wait(self.PERIOD_S)
        self._first.set()

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) >= 6 and r[0].replace(".", "").isdigit():
                mx = float(r[1]) if r[1].replace(".", "").isdigit() else None
                self.rows.append((float(r[0]), mx, tuple(n for i, n in enumerate(_REASONS)
                                                         if r[2 + i].lower() == "active")))
            self._first.set()
        self._first.set()

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.nvml is not None:
            self.thread.join(timeout=1.0)

    def summary(self) -> dict:
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        mx = [r[1] for r in rows if r[1] is not None]
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted({n for r in rows for n in r[2]}), "samples": len(rows),
                "source": self.source}


# ---------------------------------------------------------------------------
# reference arm: the reference's algorithm (oracle/ port) on the host cores

def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_port_rate(blocks=2)
        if i >= args.warmup:
            steps.append(r)
            walls.append(time.perf_counter() - t0)
    value = statistics.median([s["value"] for s in steps])
    cb = dict(steps[-1])
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gnumbers/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32 Montgomery / u64 skip + f64 map",
            "data": "synthetic: derived stream params (DEFAULT_MASTER_SEED, stream id = rank), "
                    "seeded uniform m0 in [0, n)",
            "config": C.config2_desc(args.gpus, C.seeded_m0(C._stream0().n)),
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "Gnumbers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# process launch and distributed plumbing

def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args, argv) -> int:
    """`--gpus N` outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def dist_setup(args, cpu: bool = False):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N ranks with "
                         f"torchrun --nproc-per-node N, or run without torchrun and let bench.py spawn them)")
    # RSARAND_BENCH_BACKEND=gloo exercises the multi-rank path on fewer GPUs
    # than ranks (harness check only; ranks never wait on one another in a kernel)
    backend = "gloo" if cpu else os.environ.get("RSARAND_BENCH_BACKEND", "nccl")
    if not cpu:
        if backend == "gloo":
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier_sync(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def launch_check(args) -> int:
    """CPU-only harness check of the launcher: every rank joins a gloo group
    and rank 0 prints the world it saw (tests/test_multirank.py)."""
    import torch.distributed as dist
    world, rank, _ = dist_setup(args, cpu=True)
    ranks = [rank]
    if world > 1:
        got = [None] * world
        dist.all_gather_object(got, {"rank": rank, "pid": os.getpid()})
        ranks = [g["rank"] for g in got]
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks": ranks}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def probe_imad_peak(dev) -> dict:
    """Measured Montgomery-triple IMAD-class rate (ops/s) on this GPU."""
    import ctypes
    import torch
    from paper_1811_11629_b200 import _lib
    sink = torch.zeros(1, dtype=torch.int32, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid, iters = sms * 8, 8192
    ops = ctypes.c_double(0)
    st = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _lib.call("rsa_probe_imad", grid, iters, sink.data_ptr(), ctypes.byref(ops), st.cuda_stream)
        b.record(st)
        b.synchronize()
        best = max(best, ops.value / (a.elapsed_time(b) * 1e-3))
    return {"ops_per_s": best, "sms": sms}


def launch_count() -> int:
    """Kernels of this repo's library executed so far in this process (the C
    ABI's launch counter, corrected for CUDA-graph replays: vecgen.launch_count)."""
    from paper_1811_11629_b200 import vecgen
    return vecgen.launch_count()


# ---------------------------------------------------------------------------
# timing

def time_workload(w, args, world, local, events_keys=(), min_region_s=0.0):
    """W untimed warm-up steps, then K-step blocks bracketed by barrier +
    synchronize, CUDA events on the launch stream, max over ranks.  Short
    steps repeat the K-step block until the clock sampler has watched at
    least `min_region_s` of timed work; the block time reported is the median.
    Returns (seconds per K-step block, clock summary, per-key mean seconds of
    the first block's sub-events)."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        w.step()
    ev = None
    if events_keys:
        ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)] for k in events_keys}
    blocks = []
    launches = None
    barrier_sync(world)
    with ClockSampler(local) as clk:
        while True:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier_sync(world)
            c0 = launch_count()
            t0.record(stream)
            for k in range(args.steps):
                if ev is not None and not blocks:
                    w.step({key: ev[key][k] for key in events_keys})
                else:
                    w.step()
            t1.record(stream)
            if launches is None:
                launches = launch_count() - c0  # this library's kernels in the K timed steps
            barrier_sync(world)
            blocks.append(max_over_ranks(t0.elapsed_time(t1) * 1e-3, world))
            if sum(blocks) >= min_region_s or len(blocks) >= 200:
                break
    per_key = {}
    if ev is not None:
        per_key = {k: statistics.mean(a.elapsed_time(b) * 1e-3 for a, b in ev[k]) for k in events_keys}
    return statistics.median(blocks), clk.summary(), per_key, len(blocks), launches


# ---------------------------------------------------------------------------
# configurations

def run_config2(args, world, rank, local, dev, peak):
    import torch
    w = C.Config2(dev, world, rank)
    R = w.R
    count = w.count
    el, clk, per_e, nblocks, launches = time_workload(w, args, world, local, events_keys=EXPONENTS)
    value = w.numbers_per_step * args.steps / el / 1e9
    dom = max(EXPONENTS, key=lambda e: per_e[e])  # dominant kernel: largest share of the step
    roofline = C.imad_roofline(dom, count, per_e[dom], peak, f"k_fill_fast<{dom}, 2, 0, 1> (e={dom})",
                               f"fill_e{dom}", f"fill_e{dom}", clk)
    roofline["per_exponent"] = {
        str(e): {"ms": per_e[e] * 1e3, "gnumbers_s": count / per_e[e] / 1e9,
                 "imad_frac": w_imad(e) * count / per_e[e] / peak["ops_per_s"],
                 "hbm_frac": roofline["hbm"]["frac"] * per_e[dom] / per_e[e] if roofline["hbm"]["frac"] else None}
        for e in EXPONENTS}

    e2e = None
    if not args.no_e2e:
        # the public API end to end: lane state resumed from pinned host memory,
        # every output copied to pinned host memory (take_floats(out=host))
        host_out = torch.empty(count, dtype=torch.float64, pin_memory=True)
        host_state = {e: [t.cpu().pin_memory() for t in (w.states[e].m1, w.states[e].m2, w.states[e].s)]
                      for e in EXPONENTS}
        e2e_steps = max(1, min(args.steps, 2))
        R.take_floats(w.states[EXPONENTS[0]], count, out=host_out)  # first DMA touch of 8 GiB, untimed
        barrier_sync(world)
        t = time.perf_counter()
        for _ in range(e2e_steps):
            for e in EXPONENTS:
                hs, st = host_state[e], w.states[e]
                st.m1.copy_(hs[0], non_blocking=True)
                st.m2.copy_(hs[1], non_blocking=True)
                st.s.copy_(hs[2], non_blocking=True)
                R.take_floats(st, count, out=host_out)
        barrier_sync(world)
        e2e_t = max_over_ranks(time.perf_counter() - t, world)
        d2h = len(EXPONENTS) * 8 * count
        # the bound of this path: a plain pinned device->host copy of 1 GiB, best of 3
        st = torch.cuda.current_stream()
        copy_gbs = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            host_out[:1 << 27].copy_(w.out[:1 << 27], non_blocking=True)
            b.record(st)
            b.synchronize()
            copy_gbs = max(copy_gbs, 8 * (1 << 27) / (a.elapsed_time(b) * 1e-3) / 1e9)
        e2e = {"value": world * e2e_steps * len(EXPONENTS) * count / e2e_t / 1e9, "unit": "Gnumbers/s",
               "h2d_bytes_per_step": len(EXPONENTS) * 3 * 8 * w.MV,
               "d2h_bytes_per_step": d2h,
               "steps": e2e_steps, "path": "vecgen.take_floats(state, 2^30, out=pinned host)",
               "pcie": {"d2h_gbs": d2h * e2e_steps / e2e_t / 1e9, "copy_gbs_measured": copy_gbs,
                        "frac": d2h * e2e_steps / e2e_t / 1e9 / copy_gbs,
                        "note": "e2e is bound by the device->host link: 8 B per number leave the GPU; "
                                "copy_gbs_measured = a plain 1 GiB pinned D2H copy in this run"}}
        del host_out, host_state

    line = {"metric": METRIC, "value": value, "unit": "Gnumbers/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32 Montgomery / u64 skip + f64 map",
            "data": "synthetic: derived stream params (DEFAULT_MASTER_SEED, stream id = rank), "
                    "seeded uniform m0 in [0, n)",
            "config": C.config2_desc(world, w.m0),
            "roofline": roofline, "clocks": clk,
            "gpu_launches": launches,
            "gpu_launches_source": "librsarand_b200 launch counter (rsa_launch_count) over the K timed steps",
            "e2e": e2e, "imad_peak_tops": peak["ops_per_s"] / 1e12,
            "published_context": ("BASELINE.md: the paper's C/OpenMP generator on a 24-core Xeon E5-2680 v3 "
                                  "reached 1.25e8-1.72e8 numbers/s at e <= 17 (PAPER.md:420-421); a different "
                                  "implementation, hardware and exponent mix, so vs_baseline stays null")}
    del w
    return line, None


def _sub_line(args, world, value, unit, el, clk, nblocks, config, scaling, launches):
    return {"value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "timed_blocks": nblocks, "scaling": scaling,
            "higher_is_better": True, "config": config, "clocks": clk, "gpu_launches": launches}


def run_config1(args, world, rank, local, dev, peak):
    w = C.Config1(dev, world, rank)
    el, clk, per_mv, nblocks, launches = time_workload(w, args, world, local, events_keys=w.MVS,
                                                       min_region_s=MIN_REGION_S)
    line = _sub_line(args, world, w.numbers_per_step * args.steps / el / 1e9, "Gnumbers/s", el, clk, nblocks,
                     {"workload": "config1: stream 0, e=9, 2^20 f64 per take_floats at Mv=1, 64, 65536 "
                                  "(< 2^17 lanes: split across threads by K1p/K1s, graph-replayed)"},
                     "weak", launches)
    line["per_mv"] = {str(mv): {"ms_per_2e20": per_mv[mv] * 1e3, "gnumbers_s": w.COUNT / per_mv[mv] / 1e9}
                      for mv in w.MVS}
    dom = max(w.MVS, key=lambda mv: per_mv[mv])
    rf = C.imad_roofline(9, w.COUNT, per_mv[dom], peak, f"take_floats(2^20) at Mv={dom}", None, None, clk)
    rf["bound"] = "latency"
    rf["note"] = "2^20 draws per call: a few us of kernel work per launch; launch/latency-bound"
    line["roofline"] = rf
    line["reference_context"] = ("reference scalar rsacore.take_raws 2.35 us/draw (4.26e5/s) and "
                                 "vecgen bench_throughput 1.18e7/s at Mv=65536, one core (SURVEY §6)")
    return line, None


def run_config3(args, world, rank, local, dev, peak):
    w = C.Config3(dev, world, rank)
    el, clk, _, nblocks, launches = time_workload(w, args, world, local)
    per = el / args.steps
    line = _sub_line(args, world, w.numbers_per_step * args.steps / el / 1e9, "Gnumbers/s", el, clk, nblocks,
                     {"workload": "config3: 65536 instances (ids 0..65535), e=9, Mv=64, 1024 blocks, "
                                  "2^16 f64 each, instance-major, sharded by contiguous id range",
                      "shard": [w.first, w.n], "l2": "32 GiB output per step (> L2)"},
                     "strong", launches)
    line["roofline"] = C.imad_roofline(9, w.local_numbers, per, peak, "k_fill_fast<9, 2, 0, 1>", "fill_c3",
                                       "fill_e9", clk)
    table = w.table
    del w
    return line, table


def run_config4(args, world, rank, local, dev, peak):
    w = C.Config4(dev, world, rank)
    el, clk, _, nblocks, launches = time_workload(w, args, world, local)
    per = el / args.steps
    line = _sub_line(args, world, w.numbers_per_step * args.steps / el / 1e9, "Gnumbers/s", el, clk, nblocks,
                     {"workload": "config4 fused consumer: 2^20 instances x 2^16 draws, Mv=1, e=9; "
                                  "per-instance mean/var/lag-1/64-bin hist + pooled pair correlation; "
                                  "NCCL all-reduce of pooled stats at N>1", "shard": [w.first, w.n],
                      "l2": "no stream in HBM"},
                     "strong", launches)
    line["roofline"] = C.imad_roofline(9, w.local_numbers, per, peak, "k_fused<9>", "fused", "fused_e9", clk,
                                       hbm_bytes_per_draw=0)
    line["pooled_correlation"] = w.result.pooled_correlation(w.TOTAL // 2)
    table = w.table
    del w
    return line, table


def run_config5(args, world, rank, local, dev, peak):
    w = C.Config5(dev, world, rank)

    class Timed:  # the step plus its phase bookkeeping
        def step(self_inner):
            w.step()
            w.collect()

    el, clk, _, nblocks, launches = time_workload(Timed(), args, world, local, min_region_s=MIN_REGION_S)
    line = _sub_line(args, world, w.numbers_per_step * args.steps / el / 1e9, "Gcandidates/s", el, clk, nblocks,
                     {"workload": "config5 setup: safe-prime scan (sieve to 8191, base-2 SPRP, spsp(2) table) "
                                  "of all 2^30 odd candidates in [2^31,2^32) + 2^20 instance tuples "
                                  "(ids 0..2^20-1)",
                      "unit_note": "value = odd candidates per second (scan + tuples in the step; at N>1 the "
                                   "scan phase includes the all-gather of the per-rank counts and lists)"},
                     "strong", launches)
    scan_ms = statistics.median(w.phase["scan"])
    setup_ms = statistics.median(w.phase["setup"])
    line["phases"] = {"scan_ms": scan_ms, "scan_gcandidates_s": (w.hi - w.lo) // 2 / (scan_ms * 1e-3) / 1e9,
                      "safe_primes_found": w.count, "setup_ms": setup_ms,
                      "tuples_per_s": w.n / (setup_ms * 1e-3)}
    if world == 1:
        lm = C.literal_mr_scan(args.steps, w.lo, w.hi, dev, w.count, peak)
        line["literal_mr"] = lm
        line["roofline"] = dict(lm["roofline"], note="literal MR(2,7,61) census kernels; the production scan "
                                                     "is sieve/issue-bound (profiles/r01_ncu_scan.md)")
    return line, None


def run_config6(args, world, rank, local, dev, peak):
    """F1: the 23-test battery at budget 1e8 on 2 interleaved
    streams, consumers fed in registers (bench_configs.run_battery_config)."""
    line = C.run_battery_config(args, world, rank, local, dev)
    keep = ("value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "wall_ms_each", "higher_is_better",
            "scaling", "config", "clocks", "gpu_launches", "battery", "reference_context")
    return {k: line[k] for k in keep if k in line}, None


RUNNERS = {1: run_config1, 2: run_config2, 3: run_config3, 4: run_config4, 5: run_config5, 6: run_config6}


def run_gpu(args):
    import torch
    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", local)
    peak = probe_imad_peak(dev)
    if args.config == 6:
        line = C.run_battery_config(args, world, rank, local, dev)
        tables = {}
    else:
        main_cfg = args.config
        line, t0 = RUNNERS[main_cfg](args, world, rank, local, dev, peak)
        tables = {main_cfg: t0}
        if main_cfg != 2 and "metric" not in line:
            line = {"metric": METRIC, **line, "vs_baseline": None,
                    "dtype": "u32 Montgomery / u64 skip + f64 map", "data": "synthetic: derived stream params"}
        if main_cfg == 2 and not args.no_sub:
            line["configs"] = {}
            for c in [int(x) for x in args.sub.split(",") if x]:
                torch.cuda.empty_cache()
                sub, tables[c] = RUNNERS[c](args, world, rank, local, dev, peak)
                line["configs"][str(c)] = sub
    if rank == 0 and not args.no_cpu and world == 1:  # the CPU baseline is an N=1, rank-0 measurement
        line["cpu_baseline"] = C.cpu_baseline_for(args.config, tables.get(args.config))
        for c, sub in line.get("configs", {}).items():
            cb = C.cpu_baseline_for(int(c), tables.get(int(c)))
            if cb:
                sub["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=(1, 2, 3, 4, 5, 6))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="config 2 only (no configs{} sub-results)")
    ap.add_argument("--sub", default=",".join(map(str, SUB_CONFIGS)),
                    help="comma-separated sub-configurations measured beside config 2 (default: all)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args, argv)
    if args.launch_check:
        return launch_check(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
