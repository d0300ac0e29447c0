// segfill.cu — K1s: one lane split across many threads.
//
// A lane is sequential in the draw index k, but only through two
// recurrences, and both can be cut into segments:
//   * the skip s_k = a^k s_0 mod q jumps ahead exactly: a segment starting at
//     draw j*L begins from s_0 * (a^L)^j mod q;
//   * the message m_k = m_0 + sum_{i<=k} s_i (mod p) is a prefix sum, so each
//     segment's contribution sum_{i in seg} s_i (mod p1, mod p2) can be formed
//     independently and combined by an exclusive scan over the segments.
// Three stages: k_seg_sums (per segment: jump, walk L skips, sum REDC(s) in
// the R^-1 domain), the exclusive scan of each lane's segment sums (k_seg_scan
// for a few segments per lane, else the chunked k_seg_chunk_tot/apply pair),
// k_seg_fill (per segment: jump again, start from m_0 + prefix, run the full
// draw and write the outputs).  The result is bit-identical to the sequential
// lane (same values, same stream order); the cost is one extra skip + 2 REDC
// per draw (~12 heavy slots), bought back many times over whenever the lane
// count alone cannot fill 148 SMs (the scalar stream, `rsarand gen`'s Mv=64).
#include "common.cuh"
#include "draw.cuh"

namespace rsa {

// s0 * a^(j*L) mod q63 given aL = a^L mod q63
RSA_DEV uint64_t seg_start(uint64_t s0, uint64_t aL, uint64_t j) {
    uint64_t r = s0, b = aL;
    while (j) {
        if (j & 1) r = mulmod_q63(r, b);
        j >>= 1;
        if (j) b = mulmod_q63(b, b);
    }
    return r;
}

RSA_DEV uint64_t pow_q63(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r = mulmod_q63(r, b);
        e >>= 1;
        if (e) b = mulmod_q63(b, b);
    }
    return r;
}

// Lane state snapshot taken by the first kernel: the fill kernel reads the
// starting state from here, so the segment that writes the final state back
// cannot race with segments still reading the initial one.
struct SegState {
    uint64_t m1, m2, s;
};

// thread t -> (segment j = t / lanes, lane g = t % lanes): lane-minor, so a warp
// covers consecutive lanes of one segment (coalesced when mv >= 32)
__global__ void __launch_bounds__(256)
k_seg_sums(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes, uint64_t blocks,
           uint64_t L, uint64_t nseg, const uint64_t* __restrict__ m1, const uint64_t* __restrict__ m2,
           const uint64_t* __restrict__ s, SegState* __restrict__ st0, uint32_t* __restrict__ sums) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= lanes * nseg) return;
    const uint64_t j = t / lanes, lane = t - j * lanes, i = lane / mv;
    if (j == 0) st0[lane] = SegState{m1[lane], m2[lane], s[lane]};
    const FastInst P = load_fast(inst + i);
    const uint64_t k0 = j * L, len = min(L, blocks - k0);
    uint64_t sk = seg_start(s[lane], pow_q63(P.a, L), j);
    uint32_t a1 = 0, a2 = 0;
    for (uint64_t k = 0; k < len; ++k) {
        sk = skip_q63(sk, P.a);
        a1 = add_mod(a1, mont_redc(sk, P.p1, P.p1_inv), P.p1);
        a2 = add_mod(a2, mont_redc(sk, P.p2, P.p2_inv), P.p2);
    }
    sums[2 * t] = a1;
    sums[2 * t + 1] = a2;
}

// inclusive warp scan of (v1, v2) mod (p1, p2)
RSA_DEV void warp_scan2(uint32_t& v1, uint32_t& v2, uint32_t p1, uint32_t p2, int wl) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o1 = __shfl_up_sync(0xffffffffu, v1, d), o2 = __shfl_up_sync(0xffffffffu, v2, d);
        if (wl >= d) { v1 = add_mod(v1, o1, p1); v2 = add_mod(v2, o2, p2); }
    }
}

// exclusive scan over the segments of each lane (in place), mod p1 / p2
__global__ void k_seg_scan(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes,
                           uint64_t nseg, uint32_t* __restrict__ sums) {
    const uint64_t lane = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    const rsa_instance* ip = inst + lane / mv;
    const uint32_t p1 = ip->p1, p2 = ip->p2;
    uint32_t r1 = 0, r2 = 0;
    for (uint64_t j = 0; j < nseg; ++j) {
        const uint64_t t = j * lanes + lane;
        const uint32_t v1 = sums[2 * t], v2 = sums[2 * t + 1];
        sums[2 * t] = r1;
        sums[2 * t + 1] = r2;
        r1 = add_mod(r1, v1, p1);
        r2 = add_mod(r2, v2, p2);
    }
}

// Chunked scan for many segments per lane: chunks of SEG_CHUNK segments of
// one lane per CTA.  Pass A: chunk totals.  Pass C: each CTA adds up the
// totals of its lane's earlier chunks (at most a few dozen), then a block
// scan of its own segments writes the exclusive prefixes in place.  Two
// fully parallel launches instead of one CTA walking every segment of a lane.
constexpr int SEG_SCAN_BLOCK = 256, SEG_PER_THREAD = 4;
constexpr uint64_t SEG_CHUNK = (uint64_t)SEG_SCAN_BLOCK * SEG_PER_THREAD;

// block-wide exclusive scan of (v1, v2) mod (p1, p2); returns the block totals
RSA_DEV void block_excl_scan2(uint32_t& v1, uint32_t& v2, uint32_t p1, uint32_t p2,
                              uint32_t* tot1, uint32_t* tot2) {
    __shared__ uint32_t w1[SEG_SCAN_BLOCK / 32], w2[SEG_SCAN_BLOCK / 32];
    const int wl = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t x1 = v1, x2 = v2;
    warp_scan2(v1, v2, p1, p2, wl);  // inclusive within the warp
    if (wl == 31) { w1[wid] = v1; w2[wid] = v2; }
    __syncthreads();
    uint32_t b1 = 0, b2 = 0, a1 = 0, a2 = 0;
#pragma unroll
    for (int k = 0; k < SEG_SCAN_BLOCK / 32; ++k) {
        if (k < wid) { b1 = add_mod(b1, w1[k], p1); b2 = add_mod(b2, w2[k], p2); }
        a1 = add_mod(a1, w1[k], p1);
        a2 = add_mod(a2, w2[k], p2);
    }
    v1 = add_mod(b1, sub_mod(v1, x1, p1), p1);
    v2 = add_mod(b2, sub_mod(v2, x2, p2), p2);
    *tot1 = a1;
    *tot2 = a2;
}

__global__ void __launch_bounds__(SEG_SCAN_BLOCK)
k_seg_chunk_tot(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes, uint64_t nseg,
                uint64_t nchunk, const uint32_t* __restrict__ sums, uint32_t* __restrict__ ctot) {
    const uint64_t lane = blockIdx.x / nchunk, c = blockIdx.x - lane * nchunk;
    const rsa_instance* ip = inst + lane / mv;
    const uint32_t p1 = ip->p1, p2 = ip->p2;
    uint32_t v1 = 0, v2 = 0;
#pragma unroll
    for (int i = 0; i < SEG_PER_THREAD; ++i) {
        const uint64_t j = c * SEG_CHUNK + (uint64_t)i * SEG_SCAN_BLOCK + threadIdx.x;
        if (j < nseg) {
            const uint64_t t = j * lanes + lane;
            v1 = add_mod(v1, sums[2 * t], p1);
            v2 = add_mod(v2, sums[2 * t + 1], p2);
        }
    }
    uint32_t a1, a2;
    block_excl_scan2(v1, v2, p1, p2, &a1, &a2);
    if (threadIdx.x == 0) { ctot[2 * blockIdx.x] = a1; ctot[2 * blockIdx.x + 1] = a2; }
}

__global__ void __launch_bounds__(SEG_SCAN_BLOCK)
k_seg_chunk_apply(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes, uint64_t nseg,
                  uint64_t nchunk, uint32_t* __restrict__ sums, const uint32_t* __restrict__ ctot) {
    const uint64_t lane = blockIdx.x / nchunk, c = blockIdx.x - lane * nchunk;
    const rsa_instance* ip = inst + lane / mv;
    const uint32_t p1 = ip->p1, p2 = ip->p2;
    // offset of this chunk: the lane's earlier chunk totals (warp 0 adds them up)
    __shared__ uint32_t off1, off2;
    if (threadIdx.x < 32) {
        uint32_t o1 = 0, o2 = 0;
        for (uint64_t k = threadIdx.x; k < c; k += 32) {
            o1 = add_mod(o1, ctot[2 * (lane * nchunk + k)], p1);
            o2 = add_mod(o2, ctot[2 * (lane * nchunk + k) + 1], p2);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            o1 = add_mod(o1, __shfl_xor_sync(0xffffffffu, o1, d), p1);
            o2 = add_mod(o2, __shfl_xor_sync(0xffffffffu, o2, d), p2);
        }
        if (threadIdx.x == 0) { off1 = o1; off2 = o2; }
    }
    // the SEG_PER_THREAD segments of a thread are strided by the block size;
    // scan them one stride-row at a time, carrying the row totals
    uint32_t c1 = 0, c2 = 0;
    __syncthreads();
    c1 = off1;
    c2 = off2;
#pragma unroll
    for (int i = 0; i < SEG_PER_THREAD; ++i) {
        const uint64_t j = c * SEG_CHUNK + (uint64_t)i * SEG_SCAN_BLOCK + threadIdx.x;
        const uint64_t t = j * lanes + lane;
        uint32_t v1 = 0, v2 = 0;
        if (j < nseg) { v1 = sums[2 * t]; v2 = sums[2 * t + 1]; }
        uint32_t a1, a2;
        block_excl_scan2(v1, v2, p1, p2, &a1, &a2);
        if (j < nseg) { sums[2 * t] = add_mod(c1, v1, p1); sums[2 * t + 1] = add_mod(c2, v2, p2); }
        c1 = add_mod(c1, a1, p1);
        c2 = add_mod(c2, a2, p2);
        __syncthreads();  // the block scan's shared words are reused by the next row
    }
}

template <uint32_t E, bool RAW, bool F64>
__global__ void __launch_bounds__(256)
k_seg_fill(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes, uint64_t blocks,
           uint64_t L, uint64_t nseg, uint64_t* __restrict__ m1, uint64_t* __restrict__ m2,
           uint64_t* __restrict__ s, const SegState* __restrict__ st0, const uint32_t* __restrict__ prefix,
           uint64_t* __restrict__ raw, double* __restrict__ f64, uint64_t inst_stride) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= lanes * nseg) return;
    const uint64_t j = t / lanes, lane = t - j * lanes, i = lane / mv;
    const uint32_t g = (uint32_t)(lane - i * mv);
    const FastInst P = load_fast(inst + i);
    const uint64_t k0 = j * L, len = min(L, blocks - k0);
    const SegState z = st0[lane];
    Lane Ln = lane_in(P, z.m1, z.m2, z.s);
    Ln.s = seg_start(Ln.s, pow_q63(P.a, L), j);
    Ln.x1 = add_mod(Ln.x1, prefix[2 * t], P.p1);
    Ln.x2 = add_mod(Ln.x2, prefix[2 * t + 1], P.p2);
    uint64_t off = i * inst_stride + k0 * mv + g;
    with_garner(P, [&](auto gf) {
        constexpr bool GF = decltype(gf)::value;
        for (uint64_t k = 0; k < len; ++k, off += mv) {
            const uint64_t c = draw_fast<E, GF>(P, Ln);
            if constexpr (RAW) __stcs(reinterpret_cast<unsigned long long*>(raw + off), (unsigned long long)c);
            if constexpr (F64) __stcs(f64 + off, to_unit(c, P.n_float, P.n_recip));
        }
    });
    if (j == nseg - 1) {  // the last segment owns the lane's final state
        m1[lane] = lane_m1(P, Ln);
        m2[lane] = lane_m2(P, Ln);
        s[lane] = Ln.s;
    }
}

// ---- K1p: few lanes, moderate draw counts, one thread per draw ---------------
//
// For take sizes where even 16-draw segments leave the lane chains latency
// bound (the scalar stream's 2^20 draws), the message recurrence is cut at
// every draw instead: pass 1 walks the skip in PD_SEG = 16-draw segments (one thread
// each, jump-started like K1s) and stores every draw's message increment
// REDC(s) mod p1, p2, the segments' in-CTA exclusive prefix and the CTA
// totals; pass 2 runs one thread per draw: a warp-wide inclusive scan of the
// increments within its segment, plus the segment and CTA prefixes, gives the
// draw's message, and the draw itself (chain, Garner, float map) is fully
// parallel.  Two launches instead of K1s's four; bit-identical results.
constexpr int PD_SEG = 16;     // draws per pass-1 segment (one thread each)
#ifndef RSA_PD_DPT
#define RSA_PD_DPT 8  // A/B on B200: 4 -> 8 draws per thread, 22.1 -> 21.1 us per 2^20 scalar draws (16: 22.7)
#endif
constexpr int PD_DPT = RSA_PD_DPT;  // consecutive draws per pass-2 thread
constexpr int PD_BLOCK = 256;  // threads per CTA in both passes
constexpr int PD_CTA2 = PD_BLOCK * PD_DPT;  // draws per pass-2 CTA
static_assert((PD_BLOCK * PD_SEG) % PD_CTA2 == 0 && (32 * PD_DPT) % PD_SEG == 0,
              "a pass-2 CTA lies inside one pass-1 CTA; a warp starts on a segment boundary");

struct PdLane {
    uint64_t m1, m2, s_end;  // initial residues (snapshot), skip after the last draw
};

// Segment starts: thread j needs s_0 a^(PD_SEG j) mod q.  The CTA's first
// PD_TBITS threads build T[k] = a^(PD_SEG 2^k) (4 + k squarings each, in
// parallel) and every thread multiplies the entries of its set bits: ~log2(j)/2
// products instead of a per-thread square-and-multiply over a^PD_SEG
// (k_pd_skips issued 3.9k instructions per 16-draw segment that way).
constexpr int PD_TBITS = 20;  // nseg <= RSA_PD_MAX / PD_SEG = 2^19
constexpr int PD_SEG_LOG = 4;
static_assert(PD_SEG == 1 << PD_SEG_LOG, "segment length is a power of two");
constexpr int PD_STAGE = PD_SEG + 1;  // staging row pitch (uint2): 2-way bank conflicts at most

// pass 1: CTA (lane, c) covers segments [c*PD_BLOCK, (c+1)*PD_BLOCK) of lane,
// i.e. draws [c*PD_BLOCK*PD_SEG, ...); increments are staged in shared memory
// and written back coalesced (one thread per 16 consecutive uint2 would touch
// 32 lines per warp store)
__global__ void __launch_bounds__(PD_BLOCK)
k_pd_skips(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t blocks, uint64_t nseg,
           uint32_t cta_per_lane, const uint64_t* __restrict__ m1, const uint64_t* __restrict__ m2,
           const uint64_t* __restrict__ s, uint2* __restrict__ inc, uint2* __restrict__ segpre,
           uint2* __restrict__ ctot, PdLane* __restrict__ snap) {
    __shared__ uint64_t T[PD_TBITS];
    __shared__ uint2 stage[PD_BLOCK * PD_STAGE];
    const uint32_t lane = blockIdx.x / cta_per_lane, c = blockIdx.x - lane * cta_per_lane;
    const uint64_t j = (uint64_t)c * PD_BLOCK + threadIdx.x;
    const FastInst P = load_fast(inst + lane / mv);
    const int nbits = 64 - __clzll(nseg > 1 ? nseg - 1 : 1);  // bits of the largest segment index
    if (threadIdx.x < nbits) {
        uint64_t x = P.a;
        for (uint32_t k = 0; k < PD_SEG_LOG + threadIdx.x; ++k) x = mulmod_q63(x, x);
        T[threadIdx.x] = x;
    }
    __syncthreads();
    uint32_t a1 = 0, a2 = 0;
    if (j < nseg) {
        const uint64_t k0 = j * PD_SEG, len = min((uint64_t)PD_SEG, blocks - k0);
        uint64_t sk = s[lane];
        for (int k = 0; k < nbits; ++k)
            if ((j >> k) & 1) sk = mulmod_q63(sk, T[k]);
        uint2* row = stage + threadIdx.x * PD_STAGE;
#pragma unroll
        for (int k = 0; k < PD_SEG; ++k) {
            if (k < len) {
                sk = skip_q63(sk, P.a);
                const uint32_t r1 = mont_redc(sk, P.p1, P.p1_inv), r2 = mont_redc(sk, P.p2, P.p2_inv);
                row[k] = make_uint2(r1, r2);
                a1 = add_mod(a1, r1, P.p1);
                a2 = add_mod(a2, r2, P.p2);
            }
        }
        if (j == nseg - 1) snap[lane] = PdLane{m1[lane], m2[lane], sk};
    }
    uint32_t t1, t2;
    block_excl_scan2(a1, a2, P.p1, P.p2, &t1, &t2);  // (its __syncthreads also orders the staging)
    if (j < nseg) segpre[(uint64_t)lane * nseg + j] = make_uint2(a1, a2);
    if (threadIdx.x == 0) ctot[blockIdx.x] = make_uint2(t1, t2);
    const uint64_t d0 = (uint64_t)c * PD_BLOCK * PD_SEG;
    const uint32_t n = (uint32_t)min((uint64_t)PD_BLOCK * PD_SEG, blocks - d0);
    uint2* out = inc + (uint64_t)lane * blocks + d0;
    for (uint32_t e = threadIdx.x; e < n; e += PD_BLOCK)
        out[e] = stage[(e >> PD_SEG_LOG) * PD_STAGE + (e & (PD_SEG - 1))];
}

// pass 2: CTA (lane, b) covers draws [b*PD_CTA2, (b+1)*PD_CTA2) of lane,
// PD_DPT consecutive draws per thread; warp w starts on pass-1 segment
// (b*PD_CTA2 + w*32*PD_DPT) / PD_SEG
template <uint32_t E, bool RAW, bool F64>
__global__ void __launch_bounds__(PD_BLOCK)
k_pd_draws(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t blocks, uint64_t nseg,
           uint32_t cta1_per_lane, uint32_t cta_per_lane, const uint2* __restrict__ inc,
           const uint2* __restrict__ segpre, const uint2* __restrict__ ctot, const PdLane* __restrict__ snap,
           uint64_t* __restrict__ m1, uint64_t* __restrict__ m2, uint64_t* __restrict__ s,
           uint64_t* __restrict__ raw, double* __restrict__ f64, uint64_t inst_stride) {
    static_assert(PD_DPT % 2 == 0, "16-byte increment loads");
    __shared__ uint32_t off1, off2;
    const uint32_t lane = blockIdx.x / cta_per_lane, b = blockIdx.x - lane * cta_per_lane;
    const uint32_t i = lane / mv;
    const uint32_t g = lane - i * mv;
    const FastInst P = load_fast(inst + i);
    const int wl = threadIdx.x & 31;
    const uint64_t d0 = (uint64_t)b * PD_CTA2 + (uint64_t)threadIdx.x * PD_DPT;  // this thread's first draw
    if (threadIdx.x < 32) {  // the lane's pass-1 CTA totals before this CTA's pass-1 CTA
        const uint32_t c1 = (uint32_t)(((uint64_t)b * PD_CTA2 / PD_SEG) / PD_BLOCK);
        const uint2* ct = ctot + (uint64_t)lane * cta1_per_lane;
        uint32_t o1 = 0, o2 = 0;
        for (uint32_t k0 = 0; k0 < c1; k0 += 8 * 32) {  // 8 loads in flight per thread
            uint2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t k = k0 + u * 32 + threadIdx.x;
                v[u] = k < c1 ? ct[k] : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                o1 = add_mod(o1, v[u].x, P.p1);
                o2 = add_mod(o2, v[u].y, P.p2);
            }
        }
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) {
            o1 = add_mod(o1, __shfl_xor_sync(0xffffffffu, o1, dd), P.p1);
            o2 = add_mod(o2, __shfl_xor_sync(0xffffffffu, o2, dd), P.p2);
        }
        if (threadIdx.x == 0) { off1 = o1; off2 = o2; }
    }
    // this thread's increments (past the end: zero) and their running sums
    uint2 v[PD_DPT];
    const uint2* src = inc + (uint64_t)lane * blocks + d0;
    if (d0 + PD_DPT <= blocks && ((uintptr_t)src & 15) == 0) {
#pragma unroll
        for (int k = 0; k < PD_DPT / 2; ++k) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(src) + k);
            v[2 * k] = make_uint2(w.x, w.y);
            v[2 * k + 1] = make_uint2(w.z, w.w);
        }
    } else {
#pragma unroll
        for (int k = 0; k < PD_DPT; ++k) v[k] = d0 + k < blocks ? src[k] : make_uint2(0u, 0u);
    }
    uint32_t q1[PD_DPT], q2[PD_DPT];
    uint32_t t1 = 0, t2 = 0;
#pragma unroll
    for (int k = 0; k < PD_DPT; ++k) {
        t1 = add_mod(t1, v[k].x, P.p1);
        t2 = add_mod(t2, v[k].y, P.p2);
        q1[k] = t1;
        q2[k] = t2;
    }
    uint32_t e1 = t1, e2 = t2;
    warp_scan2(e1, e2, P.p1, P.p2, wl);  // inclusive over the warp's threads
    e1 = sub_mod(e1, t1, P.p1);          // exclusive: the warp's draws before this thread
    e2 = sub_mod(e2, t2, P.p2);
    // loads that do not need warp 0's offsets are issued before the barrier
    const bool live = d0 < blocks;
    const PdLane z = live ? snap[lane] : PdLane{0, 0, 0};
    const uint2 sp = live ? segpre[(uint64_t)lane * nseg + (d0 - (uint64_t)wl * PD_DPT) / PD_SEG] : make_uint2(0u, 0u);
    __syncthreads();
    if (!live) return;
    // message before this thread's draws: x0 + pass-1 CTA offset + segment prefix + warp prefix
    const uint32_t b1 = add_mod(add_mod(add_mod(mont_redc(z.m1, P.p1, P.p1_inv), off1, P.p1), sp.x, P.p1), e1, P.p1);
    const uint32_t b2 = add_mod(add_mod(add_mod(mont_redc(z.m2, P.p2, P.p2_inv), off2, P.p2), sp.y, P.p2), e2, P.p2);
    const uint64_t o = (uint64_t)i * inst_stride + d0 * mv + g;
    with_garner(P, [&](auto gf) {
        constexpr bool GF = decltype(gf)::value;
#pragma unroll
        for (int k = 0; k < PD_DPT; ++k) {
            if (d0 + k >= blocks) break;
            Lane L;
            L.s = 0;  // the skip is folded into the increments by pass 1
            L.x1 = add_mod(b1, q1[k], P.p1);
            L.x2 = add_mod(b2, q2[k], P.p2);
            uint32_t h, c2;
            draw_tail<E, GF>(P, L, h, c2);
            const uint64_t c = (uint64_t)h * P.p2 + c2;
            if constexpr (RAW) raw[o + (uint64_t)k * mv] = c;
            if constexpr (F64) f64[o + (uint64_t)k * mv] = to_unit(c, P.n_float, P.n_recip);
            if (d0 + k == blocks - 1) {  // the lane's final state
                m1[lane] = lane_m1(P, L);
                m2[lane] = lane_m2(P, L);
                s[lane] = z.s_end;
            }
        }
    });
}

// ---- scalar look-ahead: the next `count` draws of one stream with every
// intermediate state (rsacore.next_raw / next_f64 serve from it) ------------
//
// One warp; lane j owns draws [j*L, (j+1)*L): it jumps its skip to the
// segment start, walks L skips (recording s), the warp scans the segments'
// message increments, and each lane then walks its draws again writing the
// raw value, the float and the state (m1, m2, s) after every draw.
template <uint32_t E>
__global__ void __launch_bounds__(32)
k_scalar_lookahead(const rsa_instance* __restrict__ inst, uint64_t m1_0, uint64_t m2_0, uint64_t s_0,
                   uint32_t L, uint64_t* __restrict__ raw, double* __restrict__ f64,
                   uint64_t* __restrict__ ts, uint32_t* __restrict__ tm1, uint32_t* __restrict__ tm2) {
    const FastInst P = load_fast(inst);
    const uint32_t j = threadIdx.x;
    const uint64_t k0 = (uint64_t)j * L;
    uint64_t sk = seg_start(s_0, pow_q63(P.a, L), j);
    uint32_t a1 = 0, a2 = 0;
    for (uint32_t k = 0; k < L; ++k) {
        sk = skip_q63(sk, P.a);
        ts[k0 + k] = sk;
        a1 = add_mod(a1, mont_redc(sk, P.p1, P.p1_inv), P.p1);
        a2 = add_mod(a2, mont_redc(sk, P.p2, P.p2_inv), P.p2);
    }
    uint32_t e1 = a1, e2 = a2;
    warp_scan2(e1, e2, P.p1, P.p2, j);
    Lane Ln;
    Ln.s = 0;
    Ln.x1 = add_mod(mont_redc(m1_0, P.p1, P.p1_inv), sub_mod(e1, a1, P.p1), P.p1);
    Ln.x2 = add_mod(mont_redc(m2_0, P.p2, P.p2_inv), sub_mod(e2, a2, P.p2), P.p2);
    __syncwarp();
    with_garner(P, [&](auto gf) {
        constexpr bool GF = decltype(gf)::value;
        for (uint32_t k = 0; k < L; ++k) {
            const uint64_t v = ts[k0 + k];
            Ln.x1 = add_mod(Ln.x1, mont_redc(v, P.p1, P.p1_inv), P.p1);
            Ln.x2 = add_mod(Ln.x2, mont_redc(v, P.p2, P.p2_inv), P.p2);
            uint32_t h, c2;
            draw_tail<E, GF>(P, Ln, h, c2);
            const uint64_t c = (uint64_t)h * P.p2 + c2;
            raw[k0 + k] = c;
            f64[k0 + k] = to_unit(c, P.n_float, P.n_recip);
            tm1[k0 + k] = (uint32_t)lane_m1(P, Ln);
            tm2[k0 + k] = (uint32_t)lane_m2(P, Ln);
        }
    });
}

}  // namespace rsa

using namespace rsa;

template <uint32_t E>
static void launch_seg_fill(unsigned grid, cudaStream_t st, const rsa_instance* inst, uint32_t mv,
                            uint64_t lanes, uint64_t blocks, uint64_t L, uint64_t nseg, uint64_t* m1,
                            uint64_t* m2, uint64_t* s, const SegState* st0, const uint32_t* pre,
                            uint64_t* raw, double* f64, uint64_t stride) {
    if (raw && f64)
        k_seg_fill<E, true, true><<<grid, 256, 0, st>>>(inst, mv, lanes, blocks, L, nseg, m1, m2, s, st0, pre, raw, f64, stride);
    else if (raw)
        k_seg_fill<E, true, false><<<grid, 256, 0, st>>>(inst, mv, lanes, blocks, L, nseg, m1, m2, s, st0, pre, raw, f64, stride);
    else
        k_seg_fill<E, false, true><<<grid, 256, 0, st>>>(inst, mv, lanes, blocks, L, nseg, m1, m2, s, st0, pre, raw, f64, stride);
}

#ifndef RSA_SEG_MIN
#define RSA_SEG_MIN 16  // shortest segment (draws); jump-ahead cost ~ 20 q63 products per segment
#endif
extern "C" uint64_t rsa_fill_segments(uint64_t lanes, uint64_t blocks) {
    // enough threads to fill the chip (~2^18), segments of >= RSA_SEG_MIN draws
    if (lanes == 0 || blocks < 2 * RSA_SEG_MIN) return 1;
    const uint64_t target = 1ull << 18;
    if (lanes >= target / 2) return 1;
    uint64_t nseg = target / lanes;
    uint64_t maxseg = blocks / RSA_SEG_MIN;
    if (nseg > maxseg) nseg = maxseg;
    return nseg < 1 ? 1 : nseg;
}

// K1p (one thread per draw) for lanes x blocks up to PD_MAX draws; its
// scratch holds 8 bytes per draw
#ifndef RSA_PD_MAX
#define RSA_PD_MAX (1ull << 23)
#endif
static_assert(RSA_PD_MAX / PD_SEG <= (1ull << PD_TBITS), "k_pd_skips' jump table covers every segment index");
static bool use_pd(uint64_t lanes, uint64_t blocks) {
    return blocks >= 4 * PD_SEG && lanes * blocks <= RSA_PD_MAX && rsa_fill_segments(lanes, blocks) > 1;
}

struct PdLayout {
    uint64_t nseg, cta1, cta2, inc, segpre, ctot, snap, bytes;  // offsets in bytes
};
static PdLayout pd_layout(uint64_t lanes, uint64_t blocks) {
    PdLayout Lo;
    Lo.nseg = (blocks + PD_SEG - 1) / PD_SEG;
    Lo.cta1 = (Lo.nseg + PD_BLOCK - 1) / PD_BLOCK;
    Lo.cta2 = (blocks + PD_CTA2 - 1) / PD_CTA2;
    Lo.inc = 0;
    Lo.segpre = Lo.inc + lanes * blocks * 8;
    Lo.ctot = Lo.segpre + lanes * Lo.nseg * 8;
    Lo.snap = Lo.ctot + lanes * Lo.cta1 * 8;
    Lo.bytes = Lo.snap + lanes * sizeof(PdLane);
    return Lo;
}

template <uint32_t E>
static void launch_pd(unsigned grid, cudaStream_t st, const rsa_instance* inst, uint32_t mv, uint64_t blocks,
                      const PdLayout& Lo, const char* sc, uint64_t* m1, uint64_t* m2, uint64_t* s,
                      uint64_t* raw, double* f64, uint64_t stride) {
    const uint2* inc = reinterpret_cast<const uint2*>(sc + Lo.inc);
    const uint2* pre = reinterpret_cast<const uint2*>(sc + Lo.segpre);
    const uint2* tot = reinterpret_cast<const uint2*>(sc + Lo.ctot);
    const PdLane* snap = reinterpret_cast<const PdLane*>(sc + Lo.snap);
#define RSA_PD(R, F) k_pd_draws<E, R, F><<<grid, PD_BLOCK, 0, st>>>(inst, mv, blocks, Lo.nseg, (uint32_t)Lo.cta1, (uint32_t)Lo.cta2, inc, pre, tot, snap, m1, m2, s, raw, f64, stride)
    if (raw && f64) RSA_PD(true, true);
    else if (raw) RSA_PD(true, false);
    else RSA_PD(false, true);
#undef RSA_PD
}

extern "C" uint64_t rsa_fill_segmented_scratch_bytes(uint64_t lanes, uint64_t blocks) {
    if (use_pd(lanes, blocks)) return pd_layout(lanes, blocks).bytes;
    const uint64_t nseg = rsa_fill_segments(lanes, blocks);
    const uint64_t nchunk = (nseg + SEG_CHUNK - 1) / SEG_CHUNK;
    return lanes * sizeof(SegState) + (nseg + nchunk) * lanes * 2 * sizeof(uint32_t);
}

extern "C" int rsa_fill_segmented(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
                                  uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
                                  uint64_t* raw_out, double* f64_out, uint64_t inst_stride,
                                  void* scratch, uint64_t scratch_bytes, void* stream) {
    if (!inst || !m1 || !m2 || !s || n_inst == 0 || mv == 0 || e == 0) return RSA_EINVAL;
    if (!(flags & RSA_FLAG_FAST)) return RSA_EPARAMS;  // q63 jump-ahead needs the fast layout
    const uint64_t lanes = (uint64_t)n_inst * mv;
    if (n_inst > 1 && (raw_out || f64_out) && inst_stride < blocks * (uint64_t)mv) return RSA_EINVAL;
    if (blocks == 0) return RSA_OK;
    if (!raw_out && !f64_out) return RSA_EINVAL;
    const uint64_t nseg = rsa_fill_segments(lanes, blocks);
    if (!scratch || scratch_bytes < rsa_fill_segmented_scratch_bytes(lanes, blocks)) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    int rc;
    if (use_pd(lanes, blocks)) {  // K1p: one thread per draw, two launches
        const PdLayout Lo = pd_layout(lanes, blocks);
        char* sc = static_cast<char*>(scratch);
        if (!grid_fits(lanes * Lo.cta1 * PD_BLOCK, PD_BLOCK) || !grid_fits(lanes * Lo.cta2 * PD_BLOCK, PD_BLOCK))
            return RSA_EINVAL;
        k_pd_skips<<<(unsigned)(lanes * Lo.cta1), PD_BLOCK, 0, st>>>(
            inst, mv, blocks, Lo.nseg, (uint32_t)Lo.cta1, m1, m2, s, reinterpret_cast<uint2*>(sc + Lo.inc),
            reinterpret_cast<uint2*>(sc + Lo.segpre), reinterpret_cast<uint2*>(sc + Lo.ctot),
            reinterpret_cast<PdLane*>(sc + Lo.snap));
        if ((rc = launch_status("rsa_fill_segmented(per-draw skips)"))) return rc;
        const unsigned g2 = (unsigned)(lanes * Lo.cta2);
        switch (e) {
            case 3: launch_pd<3>(g2, st, inst, mv, blocks, Lo, sc, m1, m2, s, raw_out, f64_out, inst_stride); break;
            case 5: launch_pd<5>(g2, st, inst, mv, blocks, Lo, sc, m1, m2, s, raw_out, f64_out, inst_stride); break;
            case 9: launch_pd<9>(g2, st, inst, mv, blocks, Lo, sc, m1, m2, s, raw_out, f64_out, inst_stride); break;
            case 17: launch_pd<17>(g2, st, inst, mv, blocks, Lo, sc, m1, m2, s, raw_out, f64_out, inst_stride); break;
            default: launch_pd<0>(g2, st, inst, mv, blocks, Lo, sc, m1, m2, s, raw_out, f64_out, inst_stride); break;
        }
        return launch_status("rsa_fill_segmented(per-draw fill)");
    }
    const uint64_t L = (blocks + nseg - 1) / nseg;
    const uint64_t nseg_eff = (blocks + L - 1) / L;
    SegState* st0 = static_cast<SegState*>(scratch);
    uint32_t* sums = reinterpret_cast<uint32_t*>(st0 + lanes);
    const uint64_t threads = lanes * nseg_eff;
    if (!grid_fits(threads, 256)) return RSA_EINVAL;
    k_seg_sums<<<grid_for(threads, 256), 256, 0, st>>>(inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums);
    if ((rc = launch_status("rsa_fill_segmented(sums)"))) return rc;
    if (nseg_eff >= 64) {  // long segment chains: chunked parallel scan
        const uint64_t nchunk = (nseg_eff + SEG_CHUNK - 1) / SEG_CHUNK;
        uint32_t* ctot = sums + 2 * nseg_eff * lanes;
        k_seg_chunk_tot<<<(unsigned)(lanes * nchunk), SEG_SCAN_BLOCK, 0, st>>>(inst, mv, lanes, nseg_eff, nchunk, sums, ctot);
        if ((rc = launch_status("rsa_fill_segmented(scan totals)"))) return rc;
        k_seg_chunk_apply<<<(unsigned)(lanes * nchunk), SEG_SCAN_BLOCK, 0, st>>>(inst, mv, lanes, nseg_eff, nchunk, sums, ctot);
    } else {
        k_seg_scan<<<grid_for(lanes, 128), 128, 0, st>>>(inst, mv, lanes, nseg_eff, sums);
    }
    if ((rc = launch_status("rsa_fill_segmented(scan)"))) return rc;
    const unsigned grid = grid_for(threads, 256);
    switch (e) {
        case 3: launch_seg_fill<3>(grid, st, inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums, raw_out, f64_out, inst_stride); break;
        case 5: launch_seg_fill<5>(grid, st, inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums, raw_out, f64_out, inst_stride); break;
        case 9: launch_seg_fill<9>(grid, st, inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums, raw_out, f64_out, inst_stride); break;
        case 17: launch_seg_fill<17>(grid, st, inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums, raw_out, f64_out, inst_stride); break;
        default: launch_seg_fill<0>(grid, st, inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums, raw_out, f64_out, inst_stride); break;
    }
    return launch_status("rsa_fill_segmented(fill)");
}

template <uint32_t E>
static void launch_lookahead(cudaStream_t st, const rsa_instance* inst, uint64_t m1, uint64_t m2, uint64_t s,
                             uint32_t L, char* out, uint32_t count) {
    uint64_t* raw = reinterpret_cast<uint64_t*>(out);
    double* f64 = reinterpret_cast<double*>(out + 8ull * count);
    uint64_t* ts = reinterpret_cast<uint64_t*>(out + 16ull * count);
    uint32_t* tm1 = reinterpret_cast<uint32_t*>(out + 24ull * count);
    uint32_t* tm2 = reinterpret_cast<uint32_t*>(out + 28ull * count);
    k_scalar_lookahead<E><<<1, 32, 0, st>>>(inst, m1, m2, s, L, raw, f64, ts, tm1, tm2);
}

extern "C" int rsa_scalar_lookahead(const rsa_instance* inst, uint64_t m1, uint64_t m2, uint64_t s,
                                    uint32_t e, uint32_t flags, uint32_t count, void* out, void* stream) {
    if (!inst || !out || e == 0 || count == 0 || count % 32 != 0 || count > 32u * 1024u) return RSA_EINVAL;
    if (!(flags & RSA_FLAG_FAST)) return RSA_EPARAMS;
    const uint32_t L = count / 32;
    cudaStream_t st = as_stream(stream);
    char* o = static_cast<char*>(out);
    switch (e) {
        case 3: launch_lookahead<3>(st, inst, m1, m2, s, L, o, count); break;
        case 5: launch_lookahead<5>(st, inst, m1, m2, s, L, o, count); break;
        case 9: launch_lookahead<9>(st, inst, m1, m2, s, L, o, count); break;
        case 17: launch_lookahead<17>(st, inst, m1, m2, s, L, o, count); break;
        default: launch_lookahead<0>(st, inst, m1, m2, s, L, o, count); break;
    }
    return launch_status("rsa_scalar_lookahead");
}
