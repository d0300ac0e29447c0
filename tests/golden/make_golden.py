"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Test infrastructure only.  This script imports the reference package
`rsarand` from /root/reference/pkg/src (read-only, present only in the build
container) and freezes its outputs as small fixtures, so the parity tests can
run on the GPU box where the reference does not exist.  Nothing in the product
path reads these files.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-derive-all]

Fixtures written (all small; big streams are pinned by sha256 + samples):
  regression.json  stream-0 params, first draws (reference rsacore.take_raws)
  streams.json     derive_stream_params tuples for a set of stream ids
  vectors.npz      raw/f64 outputs of vecgen/rsacore for the parity cases
  vectors.json     metadata + sha256 digests of the long streams
  census.json      safe-prime census of [2^31, 2^32) (count, sha256, samples)
  derive_all.json  sha256 of the packed tuples for ids [0, 2^20) (+ [0, 65536))
  snapshot.json    snapshot / params text of the reference for two streams
"""

from __future__ import annotations

import argparse
import dataclasses
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from rsarand import paramfactory as pf  # noqa: E402
from rsarand import rsacore, skipgen, vecgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = pf.DEFAULT_MASTER_SEED
M0_SEED = 181111629  # seeded-m0 convention from SURVEY.md §8(d)

# stream ids whose derivation exercises the ordinal-advance loop or repeats a
# pair, plus range ends
SPECIAL_IDS = [61644, 63194, 226495, 968244, 309449, 971806, 450672, 739451,
               589423, 690101, 868427, 658530, 953605, 65535, 65536,
               (1 << 20) - 1, 1000, 4095, 40000]


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def params_dict(p) -> dict:
    return dict(p1=p.p1, p2=p.p2, n=p.n, e=p.e, q=p.skip.q, a=p.skip.a,
                q1=p.skip.q1, q2=p.skip.q2, p2inv=p.p2inv, b=p.b,
                skip_mode=p.skip_mode, skip_const=p.skip_const,
                test_mode=p.test_mode, n_float_hex=p.n_float.hex())


def stream(sid, e=9, **kw):
    return pf.derive_stream_params(pf.StreamKey(SEED, sid), e=e, **kw)


def seeded_m0(n: int) -> int:
    return int(np.random.default_rng(M0_SEED).integers(0, n, dtype=np.uint64))


def lane_subset_state(params, m0, s0, mv, lanes):
    """SURVEY.md §8(c) lane-subset recipe: a VectorState holding only the
    lanes in `lanes` of an Mv-lane vector (no revalidation, so e=65537 works)."""
    stride = (params.skip.q - 1) // mv
    s = [s0 * skipgen.skip_power(params.skip, g * stride) % params.skip.q for g in lanes]
    k = len(lanes)
    return vecgen.VectorState(
        params=params, mv=k,
        m1=np.full(k, m0 % params.p1, dtype=np.uint64),
        m2=np.full(k, m0 % params.p2, dtype=np.uint64),
        s=np.array(s, dtype=np.uint64))


def gen_regression(out):
    p = stream(0)
    st = rsacore.init(p)
    raws = rsacore.take_raws(st, p, 16)
    st = rsacore.init(p)
    f64 = rsacore.take_floats(st, p, 16)
    out["regression.json"] = dict(
        source="rsarand.rsacore.take_raws/take_floats, stream 0 of DEFAULT_MASTER_SEED, e=9",
        params=params_dict(p), raw=raws, f64_hex=[x.hex() for x in f64],
        state_after_16=dict(m1=st.m1, m2=st.m2, s=st.s, draws=st.draws))


def gen_streams(out):
    ids = list(range(512)) + SPECIAL_IDS
    rows = {}
    for sid in ids:
        rows[str(sid)] = params_dict(stream(sid))
    # other exponents and a non-default master seed / multiplier override
    extra = {
        "e17_id7_seed7": params_dict(pf.derive_stream_params(pf.StreamKey(7, 8), e=17)),
        "seed_beef_id3": params_dict(pf.derive_stream_params(pf.StreamKey(0xBEEF, 3))),
        "mult5_seed1_id2": params_dict(pf.derive_stream_params(
            pf.StreamKey(1, 2), multiplier=skipgen.MULTIPLIER_TABLE[5])),
        "seed_big_id5": params_dict(pf.derive_stream_params(pf.StreamKey((1 << 64) - 3, 5))),
    }
    idx = {str(sid): list(pf.stream_indices(pf.StreamKey(SEED, sid))) for sid in ids}
    out["streams.json"] = dict(source="rsarand.paramfactory.derive_stream_params",
                               master_seed=SEED, streams=rows, extra=extra,
                               stream_indices=idx,
                               find_pair_anchor=list(pf.find_pair(3037000943)),
                               find_pair_first=list(pf.find_pair(2147483783)))


def gen_vectors(arrays, meta):
    p0 = stream(0)
    # config 1: stream 0, m0=0 / seeded, s0=1, Mv in {1,2,8,64}, 4096 draws
    for mv in (1, 2, 8, 64):
        st = vecgen.init_vector(p0, mv=mv)
        raw = vecgen.take_raw(st, 4096)
        arrays[f"c1_mv{mv}_raw"] = raw
        arrays[f"c1_mv{mv}_f64"] = vecgen.floats_from_raw(raw, p0)
    m0 = seeded_m0(p0.n)
    meta["seeded_m0"] = m0
    st = vecgen.init_vector(p0, m0=m0, mv=64)
    arrays["c1_seeded_mv64_raw"] = vecgen.take_raw(st, 4096)
    # Mv=65536 (cli bench default): two full blocks, pinned by digest + samples
    st = vecgen.init_vector(p0, mv=65536)
    raw = vecgen.take_raw(st, 2 * 65536)
    f64 = vecgen.floats_from_raw(raw, p0)
    meta["c1_mv65536"] = dict(blocks=2, raw_sha256=_sha(raw.astype("<u8")),
                              f64_sha256=_sha(f64.astype("<f8")))
    arrays["c1_mv65536_raw_head"] = raw[:1024]
    arrays["c1_mv65536_raw_tail"] = raw[-1024:]
    # scalar path: 2^16 draws, digest (full 2^20 pinned by the C oracle tests)
    st = rsacore.init(p0)
    raws = np.array(rsacore.take_raws(st, p0, 1 << 16), dtype=np.uint64)
    meta["c1_scalar_65536_raw_sha256"] = _sha(raws.astype("<u8"))
    arrays["c1_scalar_raw_head"] = raws[:4096]
    # take_raw partial-block semantics (reference test_vecgen TestTake)
    st = vecgen.init_vector(p0, mv=8)
    parts = [vecgen.take_raw(st, k) for k in (7, 1, 21, 0, 3)]
    arrays["take_parts_mv8"] = np.concatenate(parts)
    meta["take_parts_sizes"] = [7, 1, 21, 0, 3]

    # config 2: exponents, seeded m0, Mv=2^22 lane subset, 16 blocks
    mv = 1 << 22
    rng = np.random.default_rng(2718)
    lanes = sorted(set([0, 1, 2, 31, 32, mv // 2, mv - 2, mv - 1] +
                       rng.integers(0, mv, size=56).tolist()))
    arrays["c2_lanes"] = np.array(lanes, dtype=np.int64)
    meta["c2"] = dict(mv=mv, blocks=16, lanes=len(lanes))
    for e in (3, 5, 9, 17, 257, 65537):
        pe = dataclasses.replace(p0, e=e)
        st = lane_subset_state(pe, m0, 1, mv, lanes)
        blocks = np.stack([vecgen.next_block_raw(st) for _ in range(16)])  # [16, L]
        arrays[f"c2_e{e}_raw"] = blocks
        arrays[f"c2_e{e}_f64"] = vecgen.floats_from_raw(blocks.reshape(-1), pe).reshape(blocks.shape)
    # also a small full-vector case at e=65537 (Mv=256, 8 blocks)
    pe = dataclasses.replace(p0, e=65537)
    st = lane_subset_state(pe, m0, 1, 256, list(range(256)))
    arrays["c2_e65537_mv256_raw"] = np.stack([vecgen.next_block_raw(st) for _ in range(8)])

    # config 3: many instances, Mv=64, instance-major take_floats
    c3_ids = [0, 1, 2, 3, 1000, 4095, 40000, 65535]
    meta["c3_ids"] = c3_ids
    for sid in c3_ids:
        p = stream(sid)
        st = vecgen.init_vector(p, m0=0, s0=1, mv=64)
        f = vecgen.take_floats(st, 1 << 16)
        meta[f"c3_id{sid}_f64_sha256"] = _sha(f.astype("<f8"))
        arrays[f"c3_id{sid}_f64_head"] = f[:512]
        arrays[f"c3_id{sid}_f64_tail"] = f[-512:]

    # config 4: Mv=1 streams, 2^16 draws, digests of the raw streams
    c4_ids = [0, 1, 2, 3, 61644, 63194, (1 << 20) - 1]
    meta["c4_ids"] = c4_ids
    for sid in c4_ids:
        p = stream(sid)
        st = vecgen.init_vector(p, mv=1)
        raw = vecgen.take_raw(st, 1 << 16)
        meta[f"c4_id{sid}_raw_sha256"] = _sha(raw.astype("<u8"))
        arrays[f"c4_id{sid}_f64"] = vecgen.floats_from_raw(raw, p)

    # miniature (test_mode, q=13) full period, tiny unit-mode worked example
    skip13 = skipgen.SkipParams.create(2, q=13, allow_weak=True)
    mini = rsacore.make_params(11, 23, e=3, skip=skip13, test_mode=True)
    meta["miniature"] = params_dict(mini)
    st = rsacore.init(mini)
    arrays["mini_scalar_raw"] = np.array(rsacore.take_raws(st, mini, 3036 * 2), dtype=np.uint64)
    st = vecgen.init_vector(mini, mv=3)
    arrays["mini_mv3_raw"] = vecgen.take_raw(st, 3036 * 3)
    st = vecgen.init_vector(mini, mv=4)
    arrays["mini_mv4_seeds"] = st.s.copy()
    tiny = rsacore.make_params(7, 11, e=3, skip=skip13, skip_mode=rsacore.SKIP_UNIT, test_mode=True)
    meta["tiny"] = params_dict(tiny)
    st = rsacore.init(tiny)
    arrays["tiny_unit_raw"] = np.array(rsacore.take_raws(st, tiny, 200), dtype=np.uint64)

    # unit / const skip modes on production primes (reference TestCounterModes)
    unit9 = rsacore.make_params(p0.p1, p0.p2, 9, p0.skip, skip_mode=rsacore.SKIP_UNIT)
    for mv in (1, 3, 8):
        st = vecgen.init_vector(unit9, m0=5, mv=mv)
        arrays[f"unit_m05_mv{mv}_raw"] = vecgen.take_raw(st, 64)
    const9 = rsacore.make_params(p0.p1, p0.p2, 9, p0.skip, skip_mode=rsacore.SKIP_CONST,
                                 skip_const=1234567890123)
    meta["const_skip"] = 1234567890123
    st = vecgen.init_vector(const9, mv=7)
    arrays["const_mv7_raw"] = vecgen.take_raw(st, 50)
    # clamp cases: c = n-1 must map to MAX_BELOW_ONE
    raw = np.array([0, p0.n - 1, p0.n // 2, p0.n - 2, 1], dtype=np.uint64)
    arrays["clamp_raw"] = raw
    arrays["clamp_f64"] = vecgen.floats_from_raw(raw, p0)
    # lane seeds at production Mv=64 and the miniature worked example
    arrays["lane_seeds_mv64"] = np.array(skipgen.lane_offset_seeds(p0.skip, 1, 64), dtype=np.uint64)
    arrays["lane_seeds_mv64_s0_777"] = np.array(skipgen.lane_offset_seeds(p0.skip, 777, 64),
                                                dtype=np.uint64)


def gen_census(out):
    t = time.time()
    lo, hi = 1 << 31, 1 << 32
    seg = 1 << 24
    primes = 0
    parts = []
    for start in range(lo, hi, seg):
        end = min(start + seg, hi)
        _, mask = pf._odd_prime_mask(start, end)
        primes += int(mask.sum())
        parts.append(pf.safe_primes_in(start, end))
    sp = np.concatenate(parts).astype("<u4")
    p1win = sp[(sp >= pf.P1_WINDOW[0]) & (sp < pf.P1_WINDOW[1])]
    out["census.json"] = dict(
        source="rsarand.paramfactory._odd_prime_mask / safe_primes_in over [2^31, 2^32)",
        primes=primes, safe_primes=int(len(sp)), sha256_u32le=_sha(sp),
        p1_window=list(pf.P1_WINDOW), p1_window_count=int(len(p1win)),
        p1_window_sha256_u32le=_sha(p1win),
        head=sp[:64].tolist(), tail=sp[-64:].tolist(),
        every_10000=sp[::10000].tolist(), seconds=round(time.time() - t, 1))


TUPLE_DTYPE = np.dtype([("p1", "<u4"), ("p2", "<u4"), ("a", "<u4"), ("p2inv", "<u4"),
                        ("n", "<u8"), ("b", "<u8")])


def _derive_chunk(args):
    lo, hi = args
    rows = np.zeros(hi - lo, dtype=TUPLE_DTYPE)
    steps = {}
    for i, sid in enumerate(range(lo, hi)):
        p = stream(sid)
        rows[i] = (p.p1, p.p2, p.skip.a, p.p2inv, p.n, p.b)
        ordinal, _ = pf.stream_indices(pf.StreamKey(SEED, sid))
        if pf._P1_TABLE.nth(ordinal) != p.p1:
            k = 0
            while pf._P1_TABLE.nth((ordinal + k) % pf.K_P1) != p.p1:
                k += 1
            steps[sid] = k
    return lo, rows, steps


def gen_derive_all(out, n_ids=1 << 20, procs=None):
    t = time.time()
    procs = procs or os.cpu_count()
    chunk = 4096
    tasks = [(lo, min(lo + chunk, n_ids)) for lo in range(0, n_ids, chunk)]
    rows = np.zeros(n_ids, dtype=TUPLE_DTYPE)
    steps = {}
    with mp.get_context("fork").Pool(procs) as pool:
        for lo, r, s in pool.imap_unordered(_derive_chunk, tasks):
            rows[lo:lo + len(r)] = r
            steps.update(s)
    pairs = set(zip(rows["p1"].tolist(), rows["p2"].tolist()))
    out["derive_all.json"] = dict(
        source="rsarand.paramfactory.derive_stream_params(StreamKey(DEFAULT_MASTER_SEED, id), e=9)",
        layout="packed little-endian struct {u32 p1, u32 p2, u32 a, u32 p2inv, u64 n, u64 b}",
        ids=n_ids, sha256=_sha(rows), sha256_first_65536=_sha(rows[:65536]),
        distinct_pairs=len(pairs), advanced_ids={str(k): v for k, v in sorted(steps.items())},
        procs=procs, seconds=round(time.time() - t, 1))


def gen_streamio(out):
    """Byte digests of the reference CLI `gen` output (cli.py:131-151)."""
    import tempfile
    from rsarand import cli
    rows = {}
    with tempfile.TemporaryDirectory() as td:
        for fmt in ("raw64", "f64le", "text"):
            for count, lanes, chunkcase in ((5000, 64, "small"), ((1 << 22) + 777, 64, "multi_chunk")):
                if fmt == "text" and chunkcase == "multi_chunk":
                    continue
                path = os.path.join(td, f"{fmt}_{chunkcase}")
                cli.main(["gen", "--seed", str(SEED), "--stream", "3", "--count", str(count),
                          "--lanes", str(lanes), "--format", fmt, "--out", path])
                data = open(path, "rb").read()
                rows[f"{fmt}_{chunkcase}"] = dict(count=count, lanes=lanes, stream=3, bytes=len(data),
                                                  sha256=hashlib.sha256(data).hexdigest())
    out["streamio.json"] = dict(source="rsarand.cli gen --seed DEFAULT --stream 3", cases=rows)


def gen_bitsource(out, arrays):
    """rsarand.stats.BitSource over the interstream protocol of cli.cmd_test
    (cli.py:162-176): distinct pairs, common multiplier, m0=0, s0=1."""
    from rsarand import stats
    first = stream(5)
    plist = [first] + [stream(5 + j, multiplier=first.skip.a) for j in range(1, 3)]
    meta = {"streams": [5, 6, 7], "lanes": 16, "takes": [1000, 5000, 3, 333]}
    for sel in ("float_leading", "raw_low_bits", "raw_word"):
        for k in (1, 3):
            src = stats.BitSource([vecgen.init_vector(p, m0=0, s0=1, mv=16) for p in plist[:k]], sel)
            parts = [src.take(n) for n in meta["takes"]]
            arrays[f"bitsource_{sel}_{k}"] = np.concatenate(parts)
    out["bitsource.json"] = meta


def gen_battery(out):
    """rsarand.stats.run_battery on interstream sources at a small budget:
    every core test and low-bit rerun (statistic, dof, p, samples)."""
    from rsarand import stats
    first = stream(9)
    plist = [first] + [stream(9 + j, multiplier=first.skip.a) for j in range(1, 2)]
    budget = 1 << 23

    def make(sel):
        return stats.BitSource([vecgen.init_vector(p, m0=0, s0=1, mv=256) for p in plist], sel)

    t = time.time()
    rep = stats.run_battery(make, budget=budget)
    out["battery.json"] = dict(
        source="rsarand.stats.run_battery (2 interleaved streams 9,10, common multiplier, mv=256)",
        streams=[9, 10], lanes=256, budget=budget,
        reports=[r.record() for r in rep.reports], errors=rep.errors, seconds=round(time.time() - t, 1))


def gen_snapshot(out):
    """The reference's snapshot / params text for stream 0 after 1234 draws,
    and for a const-mode test stream (rsacore.py:292-417)."""
    p = pf.derive_stream_params(pf.StreamKey(SEED, 0))
    st = rsacore.init(p)
    rsacore.take_raws(st, p, 1234)
    cases = {"stream0_after_1234": (rsacore.snapshot(st, p).to_text(), rsacore.params_to_text(p))}
    pc = rsacore.make_params(p.p1, p.p2, 9, p.skip, skip_mode=rsacore.SKIP_CONST, skip_const=12345)
    sc = rsacore.init(pc)
    rsacore.take_raws(sc, pc, 7)
    cases["const_after_7"] = (rsacore.snapshot(sc, pc).to_text(), rsacore.params_to_text(pc))
    out["snapshot.json"] = {k: {"snapshot": a, "params": b} for k, (a, b) in cases.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-derive-all", action="store_true")
    ap.add_argument("--skip-census", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None
    out = {}
    if not only or "regression" in only:
        gen_regression(out)
    if not only or "streams" in only:
        gen_streams(out)
    if not only or "vectors" in only:
        arrays, meta = {}, {}
        gen_vectors(arrays, meta)
        np.savez_compressed(os.path.join(HERE, "vectors.npz"), **arrays)
        out["vectors.json"] = meta
    if not only or "battery" in only:
        gen_battery(out)
    if not only or "bitsource" in only:
        arr = {}
        gen_bitsource(out, arr)
        np.savez_compressed(os.path.join(HERE, "bitsource.npz"), **arr)
    if not only or "streamio" in only:
        gen_streamio(out)
    if not only or "snapshot" in only:
        gen_snapshot(out)
    if (not only or "census" in only) and not args.skip_census:
        gen_census(out)
    if (not only or "derive_all" in only) and not args.skip_derive_all:
        gen_derive_all(out)
    for name, obj in out.items():
        with open(os.path.join(HERE, name), "w") as fh:
            json.dump(obj, fh, indent=1, sort_keys=True)
            fh.write("\n")
        print("wrote", name)


if __name__ == "__main__":
    main()
