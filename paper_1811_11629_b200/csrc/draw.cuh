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
    double p2d, n_float, n_recip, n_recip_lo;
};

RSA_DEV FastInst load_fast(const rsa_instance* __restrict__ ip) {
    FastInst P;
    const uint4* v = reinterpret_cast<const uint4*>(ip);
    uint4 w0 = __ldg(v + 0), w1 = __ldg(v + 1), w2 = __ldg(v + 2);
    P.p1 = w0.x; P.p2 = w0.y; P.p1_inv = w0.z; P.p2_inv = w0.w;
    P.a = w1.x; P.e = w1.y; P.k1 = w1.z; P.k2 = w1.w;
    P.r2_1 = w2.x; P.r2_2 = w2.y; P.garner = w2.z;
    P.p2d = (double)P.p2;
    P.n_float = __ldg(&ip->n_float);
    P.n_recip = __ldg(&ip->n_recip);
    P.n_recip_lo = __ldg(&ip->n_recip_lo);
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

template <uint32_t E>
RSA_DEV uint32_t pow_e(uint32_t x, uint32_t e, uint32_t p, uint32_t pinv) {
    if constexpr (E != 0) return Chain<E>::pow(x, p, pinv);
    else return pow_runtime(x, e, p, pinv);
}

// One draw on the fast path: advances the lane and returns (h, c2) with the
// ciphertext c = h*p2 + c2, h = (c1 - c2)*p2inv mod p1 (Garner).
template <uint32_t E>
RSA_DEV void draw_fast_hc(const FastInst& P, Lane& L, uint32_t& h, uint32_t& c2) {
    L.s = skip_q63(L.s, P.a);
    L.x1 = add_mod(L.x1, mont_redc(L.s, P.p1, P.p1_inv), P.p1);
    L.x2 = add_mod(L.x2, mont_redc(L.s, P.p2, P.p2_inv), P.p2);
    uint32_t y1 = pow_e<E>(L.x1, P.e, P.p1, P.p1_inv);   // m1^e R^-(2e-1)
    uint32_t y2 = pow_e<E>(L.x2, P.e, P.p2, P.p2_inv);
    uint32_t c1 = mont_mul(y1, P.k1, P.p1, P.p1_inv);    // m1^e mod p1
    c2 = mont_mul(y2, P.k2, P.p2, P.p2_inv);             // m2^e mod p2
    uint32_t c2r = c2 >= P.p1 ? c2 - P.p1 : c2;          // c2 < 2^32 < 2 p1
    uint32_t d = sub_mod(c1, c2r, P.p1);
    h = mont_mul(d, P.garner, P.p1, P.p1_inv);           // d * p2inv mod p1
}

template <uint32_t E>
RSA_DEV uint64_t draw_fast(const FastInst& P, Lane& L) {
    uint32_t h, c2;
    draw_fast_hc<E>(P, L, h, c2);
    return (uint64_t)h * P.p2 + c2;
}

// ---- general path (test-mode sizes, any prime q, unit/const skip) -------------

struct GenInst {
    uint32_t p1, p2, p1_inv, p2_inv, a, e, k1, k2, r2_1, r2_2, garner, q1, q2, mode;
    uint64_t q, n;
    double n_float, n_recip, n_recip_lo;
};

RSA_DEV GenInst load_gen(const rsa_instance* __restrict__ ip) {
    GenInst G;
    G.p1 = ip->p1; G.p2 = ip->p2; G.p1_inv = ip->p1_inv; G.p2_inv = ip->p2_inv;
    G.a = ip->a; G.e = ip->e; G.k1 = ip->k1; G.k2 = ip->k2;
    G.r2_1 = ip->r2_1; G.r2_2 = ip->r2_2; G.garner = ip->garner;
    G.q1 = ip->q1; G.q2 = ip->q2; G.mode = ip->skip_mode;
    G.q = ip->q; G.n = ip->n; G.n_float = ip->n_float; G.n_recip = ip->n_recip;
    G.n_recip_lo = ip->n_recip_lo;
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
