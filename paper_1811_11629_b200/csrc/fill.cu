// fill.cu — K1 bulk fill, lane initialisation and the float map.
//
// Replaces vecgen.next_block_raw / next_block / floats_from_raw
// (vecgen.py:87-112), the block loop of take_raw (vecgen.py:115-139) for whole
// blocks, and vecgen.init_vector + skipgen.lane_offset_seeds (vecgen.py:44-69,
// skipgen.py:119-138).
//
// Layout: one thread owns LPT adjacent lanes of one instance and walks them
// through `blocks` draws (a lane is inherently sequential — SURVEY §5); a warp
// covers 32*LPT consecutive lanes, so each block's stores are contiguous
// 8*32*LPT-byte runs (128-bit streaming stores when LPT = 2).  State is read
// once and written once per launch; the stream itself never re-touches HBM.
#include "common.cuh"
#include "draw.cuh"

namespace rsa {

template <int LPT>
RSA_DEV void store_u64(uint64_t* p, const uint64_t (&v)[LPT]) {
    if constexpr (LPT == 2) __stcs(reinterpret_cast<ulonglong2*>(p), make_ulonglong2(v[0], v[1]));
    else __stcs(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v[0]);
}

template <int LPT>
RSA_DEV void store_f64(double* p, const double (&v)[LPT]) {
    if constexpr (LPT == 2) __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    else __stcs(p, v[0]);
}

// Fast path: E = compile-time exponent (0 = runtime e), LPT lanes per thread.
// On B200 IMAD.WIDE / IMAD.HI (2 slots) and FP64 ops (1 slot) share one
// 64-slot/clk/SM datapath (profiles/r01_probe_hybrid.txt): a Montgomery
// product costs 5 slots, a REDC 3, the skip 6, the float map 5.
#ifndef RSA_FILL_BLOCK
#define RSA_FILL_BLOCK 128
#endif
// F64: 0 = no float output, 1 = the float map, 2 = low 32 bits / 2^32
// (stats.BitSource's raw_low_bits selector, stats.py:118-136).  ilv != 0: the
// n_inst = ilv instances are interleaved round-robin, draw t of instance i at
// out[t*ilv + i] (LPT = 1 only).
template <uint32_t E, int LPT, bool RAW, int F64>
__global__ void __launch_bounds__(RSA_FILL_BLOCK)
k_fill_fast(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t total_lanes,
            uint64_t blocks, uint64_t* __restrict__ m1, uint64_t* __restrict__ m2,
            uint64_t* __restrict__ s, uint64_t* __restrict__ raw, double* __restrict__ f64,
            uint64_t inst_stride, uint32_t ilv) {
    uint64_t lane = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * LPT;
    if (lane >= total_lanes) return;
    uint64_t i;
    uint32_t g;
    if (LPT == 1 && ilv) {  // instance fastest across threads: a warp's stores are contiguous
        g = (uint32_t)(lane / ilv);
        i = lane - (uint64_t)g * ilv;
        lane = i * mv + g;
    } else {
        i = lane / mv;
        g = (uint32_t)(lane - i * mv);
    }
    const FastInst P = load_fast(inst + i);
    Lane L[LPT];
#pragma unroll
    for (int j = 0; j < LPT; ++j) L[j] = lane_in(P, m1[lane + j], m2[lane + j], s[lane + j]);
    uint64_t off = i * inst_stride + g, step = mv;
    if (LPT == 1 && ilv) {
        off = (uint64_t)g * ilv + i;
        step = (uint64_t)mv * ilv;
    }
    // per-exponent schedule choices measured on B200 (profiles/r02_ab_draw.txt):
    // the 4-op quotient at e = 3, a 2x-unrolled block loop at e = 5 and 9
    constexpr bool DD = E == 3;
    constexpr int UNROLL = (E == 5 || E == 9) ? 2 : 1;
    with_garner(P, [&](auto gf) {
        constexpr bool GF = decltype(gf)::value;
#pragma unroll UNROLL
        for (uint64_t k = 0; k < blocks; ++k, off += step) {
            uint64_t c[LPT];
#pragma unroll
            for (int j = 0; j < LPT; ++j) c[j] = draw_fast<E, GF>(P, L[j]);
            if constexpr (RAW) store_u64<LPT>(raw + off, c);
            if constexpr (F64 != 0) {
                double r[LPT];
#pragma unroll
                for (int j = 0; j < LPT; ++j)
                    r[j] = F64 == 1 ? (DD ? to_unit_dd(c[j], P.n_float, P.n_recip, P.n_recip_lo)
                                          : to_unit(c[j], P.n_float, P.n_recip))
                                    : __uint2double_rn((uint32_t)c[j]) * 0x1p-32;
                store_f64<LPT>(f64 + off, r);
            }
        }
    });
#pragma unroll
    for (int j = 0; j < LPT; ++j) {
        m1[lane + j] = lane_m1(P, L[j]);
        m2[lane + j] = lane_m2(P, L[j]);
        s[lane + j] = L[j].s;
    }
}

// General path: any odd prime sizes < 2^32, any prime q with a*a <= q, unit /
// const skips (test_mode instances, rsacore.py:166-181; vecgen.py:61-68).
__global__ void __launch_bounds__(256)
k_fill_general(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t total_lanes,
               uint64_t blocks, uint64_t* __restrict__ m1, uint64_t* __restrict__ m2,
               uint64_t* __restrict__ s, uint64_t* __restrict__ raw, double* __restrict__ f64,
               uint64_t inst_stride) {
    uint64_t lane = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= total_lanes) return;
    uint64_t i = lane / mv;
    uint32_t g = (uint32_t)(lane - i * mv);
    const GenInst G = load_gen(inst + i);
    Lane L;
    L.s = s[lane];
    L.x1 = mont_redc(m1[lane], G.p1, G.p1_inv);
    L.x2 = mont_redc(m2[lane], G.p2, G.p2_inv);
    uint64_t off = i * inst_stride + g;
    for (uint64_t k = 0; k < blocks; ++k, off += mv) {
        uint64_t c = draw_general(G, L);
        if (raw) raw[off] = c;
        if (f64) f64[off] = to_unit(c, G.n_float, G.n_recip);
    }
    m1[lane] = mont_mul(L.x1, G.r2_1, G.p1, G.p1_inv);
    m2[lane] = mont_mul(L.x2, G.r2_2, G.p2, G.p2_inv);
    s[lane] = L.s;
}

template <bool DD>
__global__ void k_floats_from_raw(const uint64_t* __restrict__ raw, uint64_t count, uint64_t n,
                                  double* __restrict__ out) {
    double nf = __ull2double_rn(n);
    double nr = __drcp_rn(nf);
    double nl = recip_lo(nf, nr);
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x)
        out[j] = DD ? to_unit_dd(raw[j], nf, nr, nl) : to_unit(raw[j], nf, nr);
}

// out[j] = a * s[j] mod q: skipgen.next_skip_array (skipgen.py:108-116), one
// step of the skip for a batch of registers (the q = 2^63-25 fold, or the
// exact 128-bit product for any other q).
__global__ void k_skip_array(const uint64_t* __restrict__ s, uint64_t count, uint64_t a, uint64_t q,
                             uint64_t* __restrict__ out) {
    const bool fold = q == Q63 && a < (1ull << 32);
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = s[j];
        out[j] = fold && v < (1ull << 63) ? skip_q63(v, (uint32_t)a) : mulmod64(a % q, v % q, q);
    }
}

// (hi*2^64 + lo) mod p for p < 2^32.
RSA_DEV uint32_t mod128_32(uint64_t lo, uint64_t hi, uint32_t p) {
    uint64_t r64 = (1ull << 32) % p;               // 2^32 mod p
    r64 = (r64 * r64) % p;                         // 2^64 mod p
    uint64_t h = hi % p;
    return (uint32_t)(((h * r64) % p + lo % p) % p);
}

__global__ void k_init_lanes(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t total_lanes,
                             uint64_t m0_lo, uint64_t m0_hi, uint64_t s0,
                             uint64_t* __restrict__ m1, uint64_t* __restrict__ m2,
                             uint64_t* __restrict__ s) {
    // a^stride (63-bit exponent) is shared by every lane of an instance: the
    // first thread computes it for the CTA's first instance
    __shared__ uint64_t A0, S0;  // a^stride; s0 * A0^(g of the CTA's first lane)
    __shared__ uint64_t i0;
    __shared__ uint32_t r1_0, r2_0;  // m0 mod p1, p2 of that instance
    const uint64_t lane0 = (uint64_t)blockIdx.x * blockDim.x;
    if (threadIdx.x == 0 && lane0 < total_lanes) {
        const uint64_t ii = lane0 / mv;
        const rsa_instance* ip0 = inst + ii;
        i0 = ii;
        r1_0 = mod128_32(m0_lo, m0_hi, ip0->p1);
        r2_0 = mod128_32(m0_lo, m0_hi, ip0->p2);
        A0 = 0;
        if (ip0->skip_mode == RSA_SKIP_LCG && ip0->q == Q63) {
            uint64_t A = 1, b = ip0->a, e = (ip0->q - 1) / mv;
            while (e) { if (e & 1) A = mulmod_q63(A, b); e >>= 1; if (e) b = mulmod_q63(b, b); }
            A0 = A;
            uint64_t t = 1;
            e = lane0 - ii * mv;  // the first lane's g
            b = A;
            while (e) { if (e & 1) t = mulmod_q63(t, b); e >>= 1; if (e) b = mulmod_q63(b, b); }
            S0 = mulmod_q63(s0 % Q63, t);
        }
    }
    __syncthreads();
    uint64_t lane = lane0 + threadIdx.x;
    if (lane >= total_lanes) return;
    uint64_t i = lane / mv;
    uint32_t g = (uint32_t)(lane - i * mv);
    const rsa_instance* ip = inst + i;
    uint32_t p1 = ip->p1, p2 = ip->p2;
    const uint32_t r1 = i == i0 ? r1_0 : mod128_32(m0_lo, m0_hi, p1);
    const uint32_t r2 = i == i0 ? r2_0 : mod128_32(m0_lo, m0_hi, p2);
    if (ip->skip_mode == RSA_SKIP_LCG) {
        // lane g: s0 * (a^stride)^g mod q (skipgen.py:124-138)
        uint64_t q = ip->q, stride = (q - 1) / mv;
        uint64_t A, sg;
        if (q == Q63) {
            uint64_t b, e;
            if (i == i0) {  // lane g = g0 + threadIdx.x: s0 A^g0 (shared) times A^threadIdx.x
                uint64_t t = 1;
                b = A0;
                e = threadIdx.x;
                while (e) { if (e & 1) t = mulmod_q63(t, b); e >>= 1; if (e) b = mulmod_q63(b, b); }
                sg = mulmod_q63(S0, t);
            } else {
                A = 1;
                b = ip->a;
                e = stride;
                while (e) { if (e & 1) A = mulmod_q63(A, b); e >>= 1; if (e) b = mulmod_q63(b, b); }
                uint64_t t = 1;
                b = A;
                e = g;
                while (e) { if (e & 1) t = mulmod_q63(t, b); e >>= 1; if (e) b = mulmod_q63(b, b); }
                sg = mulmod_q63(s0, t);
            }
        } else {
            A = powmod64(ip->a, stride, q);
            sg = mulmod64(s0, powmod64(A, g, q), q);
        }
        m1[lane] = r1;
        m2[lane] = r2;
        s[lane] = sg;
    } else {
        // lane g holds m0 + (g+1-mv)*v, steps by mv*v (vecgen.py:61-68)
        uint64_t v = ip->skip_mode == RSA_SKIP_UNIT ? 1ull : ip->skip_const;
        uint64_t n = ip->n;
        uint64_t back = (uint64_t)(mv - 1 - g);
        uint32_t b1 = (uint32_t)(((back % p1) * (v % p1)) % p1);
        uint32_t b2 = (uint32_t)(((back % p2) * (v % p2)) % p2);
        m1[lane] = r1 >= b1 ? r1 - b1 : r1 + (p1 - b1);
        m2[lane] = r2 >= b2 ? r2 - b2 : r2 + (p2 - b2);
        s[lane] = mulmod64(mv % n, v % n, n);
    }
}

}  // namespace rsa

using namespace rsa;

template <uint32_t E, int LPT>
static void launch_fast(unsigned grid, cudaStream_t st, const rsa_instance* inst, uint32_t mv,
                        uint64_t lanes, uint64_t blocks, uint64_t* m1, uint64_t* m2, uint64_t* s,
                        uint64_t* raw, double* f64, uint64_t stride, uint32_t ilv, bool low32) {
#define RSA_LAUNCH(R, F) k_fill_fast<E, LPT, R, F><<<grid, RSA_FILL_BLOCK, 0, st>>>(inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv)
    if constexpr (LPT == 1) {
        if (f64 && low32) {
            if (raw) RSA_LAUNCH(true, 2); else RSA_LAUNCH(false, 2);
            return;
        }
    }
    if (raw && f64) RSA_LAUNCH(true, 1);
    else if (raw) RSA_LAUNCH(true, 0);
    else if (f64) RSA_LAUNCH(false, 1);
    else RSA_LAUNCH(false, 0);
#undef RSA_LAUNCH
}

template <int LPT>
static void dispatch_e(uint32_t e, unsigned grid, cudaStream_t st, const rsa_instance* inst,
                       uint32_t mv, uint64_t lanes, uint64_t blocks, uint64_t* m1, uint64_t* m2,
                       uint64_t* s, uint64_t* raw, double* f64, uint64_t stride, uint32_t ilv, bool low32) {
    switch (e) {
        case 3: launch_fast<3, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
        case 5: launch_fast<5, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
        case 9: launch_fast<9, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
        case 17: launch_fast<17, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
        case 65537: launch_fast<65537, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
        default: launch_fast<0, LPT>(grid, st, inst, mv, lanes, blocks, m1, m2, s, raw, f64, stride, ilv, low32); break;
    }
}

extern "C" int rsa_fill(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
                        uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
                        uint64_t* raw_out, double* f64_out, uint64_t inst_stride, void* stream) {
    if (!inst || !m1 || !m2 || !s || n_inst == 0 || mv == 0 || e == 0) return RSA_EINVAL;
    uint64_t lanes = (uint64_t)n_inst * mv;
    const bool ilv = flags & RSA_FLAG_INTERLEAVE, low32 = flags & RSA_FLAG_LOW32;
    if (n_inst > 1 && !ilv && (raw_out || f64_out) && inst_stride < blocks * (uint64_t)mv) return RSA_EINVAL;
    if (blocks == 0) return RSA_OK;
    if (!grid_fits(lanes, RSA_FILL_BLOCK)) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    if ((flags & RSA_FLAG_FAST) && !(flags & RSA_FLAG_GENERAL_PATH)) {
        // two lanes per thread needs even mv and 16-byte aligned output rows
        bool pair = (mv % 2 == 0) && (n_inst == 1 || inst_stride % 2 == 0) &&
                    ((uintptr_t)raw_out % 16 == 0) && ((uintptr_t)f64_out % 16 == 0) &&
                    !(flags & RSA_FLAG_ONE_LANE) && !ilv && !low32;
        if (pair)
            dispatch_e<2>(e, grid_for(lanes / 2, RSA_FILL_BLOCK), st, inst, mv, lanes, blocks, m1, m2, s, raw_out,
                          f64_out, inst_stride, 0, false);
        else
            dispatch_e<1>(e, grid_for(lanes, RSA_FILL_BLOCK), st, inst, mv, lanes, blocks, m1, m2, s, raw_out,
                          f64_out, inst_stride, ilv ? n_inst : 0, low32);
        return launch_status("rsa_fill(fast)");
    }
    if (ilv || low32) return RSA_EPARAMS;  // layouts of the fast kernel only
    k_fill_general<<<grid_for(lanes, 256), 256, 0, st>>>(inst, mv, lanes, blocks, m1, m2, s, raw_out,
                                                        f64_out, inst_stride);
    return launch_status("rsa_fill(general)");
}

extern "C" int rsa_floats_from_raw(const uint64_t* raw, uint64_t count, uint64_t n, double* out,
                                   void* stream) {
    if ((!raw || !out) && count) return RSA_EINVAL;
    if (n == 0) return RSA_EINVAL;
    if (count == 0) return RSA_OK;
    unsigned grid = grid_for(count, 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_floats_from_raw<false><<<grid, 256, 0, as_stream(stream)>>>(raw, count, n, out);
    return launch_status("rsa_floats_from_raw");
}

extern "C" int rsa_floats_from_raw_dd(const uint64_t* raw, uint64_t count, uint64_t n, double* out,
                                      void* stream) {
    if ((!raw || !out) && count) return RSA_EINVAL;
    if (n == 0) return RSA_EINVAL;
    if (count == 0) return RSA_OK;
    unsigned grid = grid_for(count, 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_floats_from_raw<true><<<grid, 256, 0, as_stream(stream)>>>(raw, count, n, out);
    return launch_status("rsa_floats_from_raw_dd");
}

extern "C" int rsa_skip_array(const uint64_t* s, uint64_t count, uint64_t a, uint64_t q, uint64_t* out,
                              void* stream) {
    if ((!s || !out) && count) return RSA_EINVAL;
    if (q < 2) return RSA_EINVAL;
    if (count == 0) return RSA_OK;
    unsigned grid = grid_for(count, 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_skip_array<<<grid, 256, 0, as_stream(stream)>>>(s, count, a, q, out);
    return launch_status("rsa_skip_array");
}

extern "C" int rsa_init_lanes(const rsa_instance* inst, uint32_t n_inst, uint32_t mv,
                              uint64_t m0_lo, uint64_t m0_hi, uint64_t s0,
                              uint64_t* m1, uint64_t* m2, uint64_t* s, void* stream) {
    if (!inst || !m1 || !m2 || !s || n_inst == 0 || mv == 0) return RSA_EINVAL;
    uint64_t lanes = (uint64_t)n_inst * mv;
    if (!grid_fits(lanes, 128)) return RSA_EINVAL;
    k_init_lanes<<<grid_for(lanes, 128), 128, 0, as_stream(stream)>>>(inst, mv, lanes, m0_lo, m0_hi,
                                                                       s0, m1, m2, s);
    return launch_status("rsa_init_lanes");
}
