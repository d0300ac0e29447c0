// draw.cuh — one draw of one lane: skip step, message step, two modpows,
// Garner, (float map done by the caller).  Shared by the bulk-fill (K1) and
// fused-consumer (K2) kernels so both produce the identical stream.
//
// Reference per draw (vecgen.py:87-100 lockstep form; rsacore.py:213-226 scalar):
//   s  <- a*s mod q                       (skipgen.py:92-116)
//   m1 <- (m1+s) mod p1 ; m2 <- (m2+s) mod p2
//   c1 = m1^e mod p1 ; c2 = m2^e mod p2
//   c  = ((c1 + p1 - c2 mod p1) mod p1 * p2inv mod p1) * p2 + c2
#pragma once
#include "modarith.cuh"

namespace rsa {

// Register-resident constants of one instance on the fast path
// (q = 2^63-25, p1, p2 in (2^31, 2^32), lcg skip).
struct FastInst {
    uint32_t p1, p2, p1_inv, p2_inv, a, k1, k2, garner, r2_1, r2_2, e;
    uint32_t gA, gB;  // fused-Garner constants (draw_fast_hc<E, true>)
    double n_float, n_recip, n_recip_lo;  // n_recip_lo: recip_lo(n_float, n_recip), per thread
};

// Fused Garner (p1's k-correction folded into the Garner product): valid when
// 2 (p1-1)^2 < 2^64, i.e. p1 <= floor(sqrt(q)) — every derived stream
// (paramfactory.py:27-30 puts p1 in (2^31, floor(sqrt q)]).  Instances with a
// larger p1 (make_params with the primes given in the other order) take the
// two-product form.
#ifndef RSA_GARNER_FUSED
#define RSA_GARNER_FUSED 1
#endif
constexpr uint32_t GF_P1_MAX = 3037000499u;  // floor(sqrt(2^63 - 25))

template <bool B>
struct BoolC { static constexpr bool value = B; };

// f(BoolC<GF>) with GF = "this instance may use the fused Garner".  Branches
// once per thread, outside the draw loop, so each loop body is straight-line.
template <class F>
RSA_DEV void with_garner(const FastInst& P, F&& f) {
#if RSA_GARNER_FUSED
    if (P.p1 <= GF_P1_MAX) { f(BoolC<true>{}); return; }
#endif
    f(BoolC<false>{});
}

RSA_DEV FastInst load_fast(const rsa_instance* __restrict__ ip) {
    FastInst P;
    const uint4* v = reinterpret_cast<const uint4*>(ip);
    uint4 w0 = __ldg(v + 0), w1 = __ldg(v + 1), w2 = __ldg(v + 2);
    P.p1 = w0.x; P.p2 = w0.y; P.p1_inv = w0.z; P.p2_inv = w0.w;
    P.a = w1.x; P.e = w1.y; P.k1 = w1.z; P.k2 = w1.w;
    P.r2_1 = w2.x; P.r2_2 = w2.y; P.garner = w2.z;
    P.gA = mont_mul(P.k1, P.garner, P.p1, P.p1_inv);  // k1 * p2inv mod p1
    P.gB = P.p1 - P.garner;                            // -p2inv * R mod p1 (garner != 0)
    P.n_float = __ldg(&ip->n_float);
    P.n_recip = __ldg(&ip->n_recip);
    P.n_recip_lo = recip_lo(P.n_float, P.n_recip);
    return P;
}

// Lane state in registers: skip s (< q) and canonical scaled messages
// x = m R^-1 mod p.  (Lazy [0, 2^32) representatives and a word-level skip were
// measured 1-3 % slower on B200 — profiles/r01_ab_variants.txt.)
struct Lane {
    uint64_t s;
    uint32_t x1, x2;
};

RSA_DEV Lane lane_in(const FastInst& P, uint64_t m1, uint64_t m2, uint64_t s) {
    Lane L;
    L.s = s;
    L.x1 = mont_redc(m1, P.p1, P.p1_inv);  // m < p => REDC(m) = m R^-1
    L.x2 = mont_redc(m2, P.p2, P.p2_inv);
    return L;
}

RSA_DEV uint64_t lane_m1(const FastInst& P, const Lane& L) { return mont_mul(L.x1, P.r2_1, P.p1, P.p1_inv); }
RSA_DEV uint64_t lane_m2(const FastInst& P, const Lane& L) { return mont_mul(L.x2, P.r2_2, P.p2, P.p2_inv); }

// x + REDC(s) mod p (the message step in the R^-1 domain, vecgen.py:94-95),
// written as x - w with w = (u - s_hi) mod p = -REDC(s) mod p (u = hi(m p),
// m = s_lo p^-1 mod 2^32; s_hi = s >> 32 < 2^31 < p on the fast path): two
// modular subtractions, each ISETP + SEL + IADD3 on the ALU, where
// add_mod(x, REDC(s)) cost a negation and an add that ptxas placed on the
// IMAD pipe (profiles/r02_ab_draw.txt: +2-5 % per exponent).  Rejected
// alternatives: tools/variants/draw_variants.cuh.
RSA_DEV uint32_t msg_add(uint32_t x, uint64_t s, uint32_t p, uint32_t pinv) {
    const uint32_t m = (uint32_t)s * pinv;
    const uint32_t u = __umulhi(m, p);
    const uint32_t vh = (uint32_t)(s >> 32);
    uint32_t w = u - vh;
    w = u < vh ? w + p : w;
    const uint32_t r = x - w;
    return x < w ? r + p : r;
}

template <uint32_t E>
RSA_DEV uint32_t pow_e(uint32_t x, uint32_t e, uint32_t p, uint32_t pinv) {
    if constexpr (E != 0) return Chain<E>::pow(x, p, pinv);
    else return pow_runtime(x, e, p, pinv);
}

// One draw on the fast path: advances the lane and returns (h, c2) with the
// ciphertext c = h*p2 + c2, h = (c1 - c2)*p2inv mod p1 (Garner).
// GF: h = REDC(y1*A + c2r*B) with A = k1 p2inv, B = -p2inv R (mod p1), since
// y1 k1 R^-1 = c1: one REDC of a two-product sum (7 heavy slots) replaces the
// k1 product + Garner product (10 slots) and the sub_mod between them.  The
// sum is < 2 p1^2 < 2^64 and its REDC lies in (-p1, 2^32) < 2 p1, so one
// conditional add or subtract makes h canonical.
template <uint32_t E, bool GF = false>
RSA_DEV void draw_tail(const FastInst& P, const Lane& L, uint32_t& h, uint32_t& c2);

template <uint32_t E, bool GF = false>
RSA_DEV void draw_fast_hc(const FastInst& P, Lane& L, uint32_t& h, uint32_t& c2) {
    L.s = skip_q63(L.s, P.a);
    L.x1 = msg_add(L.x1, L.s, P.p1, P.p1_inv);
    L.x2 = msg_add(L.x2, L.s, P.p2, P.p2_inv);
    draw_tail<E, GF>(P, L, h, c2);
}

// The draw after its message step: two modpows, the p2 correction and Garner.
template <uint32_t E, bool GF>
RSA_DEV void draw_tail(const FastInst& P, const Lane& L, uint32_t& h, uint32_t& c2) {
    uint32_t y1 = pow_e<E>(L.x1, P.e, P.p1, P.p1_inv);   // m1^e R^-(2e-1)
    uint32_t y2 = pow_e<E>(L.x2, P.e, P.p2, P.p2_inv);
    c2 = mont_mul(y2, P.k2, P.p2, P.p2_inv);             // m2^e mod p2
    // c2 < 2^32 < 2 p1: the conditional subtract as an unsigned min (one
    // VIADDMNMX on the ALU; c2 - p1 wraps above c2 exactly when c2 < p1)
    uint32_t c2r = min(c2, c2 - P.p1);
    if constexpr (GF) {
        uint64_t t = (uint64_t)y1 * P.gA + (uint64_t)c2r * P.gB;  // < 2 p1^2 < 2^64
        uint32_t m = (uint32_t)t * P.p1_inv;
        uint32_t u = __umulhi(m, P.p1);
        uint32_t th = (uint32_t)(t >> 32);
        uint32_t r = th - u;
        r = th < u ? r + P.p1 : r;
        h = min(r, r - P.p1);  // r < 2 p1, as for c2r
    } else {
        uint32_t c1 = mont_mul(y1, P.k1, P.p1, P.p1_inv);  // m1^e mod p1
        uint32_t d = sub_mod(c1, c2r, P.p1);
        h = mont_mul(d, P.garner, P.p1, P.p1_inv);         // d * p2inv mod p1
    }
}

template <uint32_t E, bool GF = false>
RSA_DEV uint64_t draw_fast(const FastInst& P, Lane& L) {
    uint32_t h, c2;
    draw_fast_hc<E, GF>(P, L, h, c2);
    return (uint64_t)h * P.p2 + c2;
}

// One draw mapped to r = min(fl(c)/fl(n), 1-2^-53) (vecgen.py:103-107), the
// 4-op quotient (fused consumer).
template <uint32_t E, bool GF>
RSA_DEV double draw_unit(const FastInst& P, Lane& L) {
    return to_unit_dd(draw_fast<E, GF>(P, L), P.n_float, P.n_recip, P.n_recip_lo);
}

// ---- general path (test-mode sizes, any prime q, unit/const skip) -------------

struct GenInst {
    uint32_t p1, p2, p1_inv, p2_inv, a, e, k1, k2, r2_1, r2_2, garner, q1, q2, mode;
    uint64_t q, n;
    double n_float, n_recip;
};

RSA_DEV GenInst load_gen(const rsa_instance* __restrict__ ip) {
    GenInst G;
    G.p1 = ip->p1; G.p2 = ip->p2; G.p1_inv = ip->p1_inv; G.p2_inv = ip->p2_inv;
    G.a = ip->a; G.e = ip->e; G.k1 = ip->k1; G.k2 = ip->k2;
    G.r2_1 = ip->r2_1; G.r2_2 = ip->r2_2; G.garner = ip->garner;
    G.q1 = ip->q1; G.q2 = ip->q2; G.mode = ip->skip_mode;
    G.q = ip->q; G.n = ip->n; G.n_float = ip->n_float; G.n_recip = ip->n_recip;
    return G;
}

RSA_DEV uint64_t draw_general(const GenInst& G, Lane& L) {
    if (G.mode == RSA_SKIP_LCG) {
        if (G.q == Q63) L.s = skip_q63(L.s, G.a);
        else L.s = skip_schrage(L.s, G.a, G.q, G.q1, G.q2);
    }
    // s may exceed p*2^32 for small primes: reduce first, then scale.
    L.x1 = add_mod(L.x1, mont_redc(L.s % G.p1, G.p1, G.p1_inv), G.p1);
    L.x2 = add_mod(L.x2, mont_redc(L.s % G.p2, G.p2, G.p2_inv), G.p2);
    uint32_t c1 = mont_mul(pow_runtime(L.x1, G.e, G.p1, G.p1_inv), G.k1, G.p1, G.p1_inv);
    uint32_t c2 = mont_mul(pow_runtime(L.x2, G.e, G.p2, G.p2_inv), G.k2, G.p2, G.p2_inv);
    uint32_t d = sub_mod(c1, c2 % G.p1, G.p1);
    uint32_t h = mont_mul(d, G.garner, G.p1, G.p1_inv);
    return (uint64_t)h * G.p2 + c2;
}

}  // namespace rsa
