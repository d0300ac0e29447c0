// segfill.cu — K1s: one lane split across many threads.
//
// A lane is sequential in the draw index k, but only through two
// recurrences, and both can be cut into segments:
//   * the skip s_k = a^k s_0 mod q jumps ahead exactly: a segment starting at
//     draw j*L begins from s_0 * (a^L)^j mod q;
//   * the message m_k = m_0 + sum_{i<=k} s_i (mod p) is a prefix sum, so each
//     segment's contribution sum_{i in seg} s_i (mod p1, mod p2) can be formed
//     independently and combined by an exclusive scan over the segments.
// Three launches: k_seg_sums (per segment: jump, walk L skips, sum REDC(s) in
// the R^-1 domain), k_seg_scan (per lane: exclusive scan of its segment sums),
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

// Exclusive scan over the segments of each lane (in place), mod p1 / p2:
// one CTA per lane, warp w owns a contiguous run of segments and walks it 32
// at a time (coalesced loads, a shuffle scan per step, a running carry); the
// warp totals are scanned once more and added on the way out.  Modular
// addition is associative, so the result equals the sequential scan.
RSA_DEV void warp_scan2(uint32_t& v1, uint32_t& v2, uint32_t p1, uint32_t p2, int wl) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o1 = __shfl_up_sync(0xffffffffu, v1, d), o2 = __shfl_up_sync(0xffffffffu, v2, d);
        if (wl >= d) { v1 = add_mod(v1, o1, p1); v2 = add_mod(v2, o2, p2); }
    }
}

__global__ void __launch_bounds__(1024)
k_seg_scan_block(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t lanes, uint64_t nseg,
                 uint32_t* __restrict__ sums) {
    __shared__ uint32_t w1[32], w2[32];
    const uint64_t lane = blockIdx.x;
    const rsa_instance* ip = inst + lane / mv;
    const uint32_t p1 = ip->p1, p2 = ip->p2;
    const int wl = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t per = (nseg + nw - 1) / nw;  // segments per warp
    const uint64_t j0 = (uint64_t)wid * per, j1 = min(nseg, j0 + per);
    // pass 1: warp totals
    uint32_t t1 = 0, t2 = 0;
    for (uint64_t j = j0 + wl; j < j1; j += 32) {
        const uint64_t t = j * lanes + lane;
        t1 = add_mod(t1, sums[2 * t], p1);
        t2 = add_mod(t2, sums[2 * t + 1], p2);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        t1 = add_mod(t1, __shfl_xor_sync(0xffffffffu, t1, d), p1);
        t2 = add_mod(t2, __shfl_xor_sync(0xffffffffu, t2, d), p2);
    }
    if (wl == 0) { w1[wid] = t1; w2[wid] = t2; }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the warp totals
        uint32_t x1 = wl < nw ? w1[wl] : 0, x2 = wl < nw ? w2[wl] : 0;
        uint32_t y1 = x1, y2 = x2;
        warp_scan2(y1, y2, p1, p2, wl);
        if (wl < nw) { w1[wl] = sub_mod(y1, x1, p1); w2[wl] = sub_mod(y2, x2, p2); }
    }
    __syncthreads();
    // pass 2: rewrite each run with its exclusive prefix, 32 segments per step
    uint32_t c1 = w1[wid], c2 = w2[wid];
    for (uint64_t base = j0; base < j1; base += 32) {
        const uint64_t j = base + wl;
        const bool in = j < j1;
        const uint64_t t = j * lanes + lane;
        const uint32_t v1 = in ? sums[2 * t] : 0, v2 = in ? sums[2 * t + 1] : 0;
        uint32_t i1 = v1, i2 = v2;
        warp_scan2(i1, i2, p1, p2, wl);
        if (in) {
            sums[2 * t] = add_mod(c1, sub_mod(i1, v1, p1), p1);
            sums[2 * t + 1] = add_mod(c2, sub_mod(i2, v2, p2), p2);
        }
        c1 = add_mod(c1, __shfl_sync(0xffffffffu, i1, 31), p1);
        c2 = add_mod(c2, __shfl_sync(0xffffffffu, i2, 31), p2);
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
            if constexpr (F64) __stcs(f64 + off, to_unit(c, P.n_float, P.n_recip, P.n_recip_lo));
        }
    });
    if (j == nseg - 1) {  // the last segment owns the lane's final state
        m1[lane] = lane_m1(P, Ln);
        m2[lane] = lane_m2(P, Ln);
        s[lane] = Ln.s;
    }
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

extern "C" uint64_t rsa_fill_segments(uint64_t lanes, uint64_t blocks) {
    // enough threads to fill the chip (~2^18), segments of >= 64 draws
    if (lanes == 0 || blocks < 128) return 1;
    const uint64_t target = 1ull << 18;
    if (lanes >= target / 2) return 1;
    uint64_t nseg = target / lanes;
    uint64_t maxseg = blocks / 64;
    if (nseg > maxseg) nseg = maxseg;
    return nseg < 1 ? 1 : nseg;
}

extern "C" uint64_t rsa_fill_segmented_scratch_bytes(uint64_t lanes, uint64_t blocks) {
    return lanes * sizeof(SegState) + rsa_fill_segments(lanes, blocks) * lanes * 2 * sizeof(uint32_t);
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
    const uint64_t L = (blocks + nseg - 1) / nseg;
    const uint64_t nseg_eff = (blocks + L - 1) / L;
    SegState* st0 = static_cast<SegState*>(scratch);
    uint32_t* sums = reinterpret_cast<uint32_t*>(st0 + lanes);
    cudaStream_t st = as_stream(stream);
    const uint64_t threads = lanes * nseg_eff;
    if (!grid_fits(threads, 256)) return RSA_EINVAL;
    k_seg_sums<<<grid_for(threads, 256), 256, 0, st>>>(inst, mv, lanes, blocks, L, nseg_eff, m1, m2, s, st0, sums);
    int rc = launch_status("rsa_fill_segmented(sums)");
    if (rc) return rc;
    if (nseg_eff >= 64) {  // long segment chains: one CTA per lane
        unsigned tb = 32;
        while (tb < 1024 && tb * 8 < nseg_eff) tb <<= 1;
        k_seg_scan_block<<<(unsigned)lanes, tb, 0, st>>>(inst, mv, lanes, nseg_eff, sums);
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
