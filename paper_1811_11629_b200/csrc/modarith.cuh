// modarith.cuh — exact modular arithmetic for the RSA-PRNG draw on sm_100a.
//
// Everything here is bit-exact integer (or correctly rounded IEEE) arithmetic;
// the reference restates the same operations with Python ints / numpy uint64:
//   skip      a*s mod q            skipgen.py:92-116   (Schrage; any exact a*s mod q)
//   message   m <- (m + s) mod p   vecgen.py:94-95, rsacore.py:221-222
//   modpow    m^e mod p            vecgen.py:72-84,  rsacore.py:223-224
//   Garner    CRT recombination    vecgen.py:98-100, rsacore.py:207-210
//   float     min(fl(c)/fl(n), .)  vecgen.py:103-107, rsacore.py:229-233
//
// Montgomery arithmetic with R = 2^32 over odd p < 2^32.  Messages are kept
// in the R^-1-scaled domain x = m*R^-1 mod p: adding the skip is then one REDC
// of the 63-bit s (no separate "s mod p"), a Montgomery product of two scaled
// values stays scaled (x = m^i R^-(2i-1) is preserved by any multiplication
// chain), and one product with k = R^(2e) mod p at the end returns m^e mod p.
#pragma once
#include <stdint.h>
#include "../../include/rsarand_b200.h"

#define RSA_DEV __device__ __forceinline__

namespace rsa {

// ---- 32-bit Montgomery -------------------------------------------------------

// x*y*R^-1 mod p for x, y < p (odd p < 2^32), pinv = p^-1 mod 2^32.
// T - m*p with m = T*pinv mod R is divisible by R and lies in (-pR, pR), so the
// high word difference is exact and one conditional +p makes it canonical.
// SASS: IMAD.WIDE.U32, IMAD, IMAD.HI.U32, ISETP, SEL, IADD3.
RSA_DEV uint32_t mont_mul(uint32_t x, uint32_t y, uint32_t p, uint32_t pinv) {
    uint64_t t = (uint64_t)x * y;
    uint32_t m = (uint32_t)t * pinv;
    uint32_t u = __umulhi(m, p);
    uint32_t th = (uint32_t)(t >> 32);
    uint32_t r = th - u;
    return th < u ? r + p : r;
}

// v*R^-1 mod p for any v < p*2^32 (in particular any 63-bit skip when p > 2^31).
RSA_DEV uint32_t mont_redc(uint64_t v, uint32_t p, uint32_t pinv) {
    uint32_t m = (uint32_t)v * pinv;
    uint32_t u = __umulhi(m, p);
    uint32_t vh = (uint32_t)(v >> 32);
    uint32_t r = vh - u;
    return vh < u ? r + p : r;
}

// (x + y) mod p, x, y < p < 2^32 (the sum may carry out of 32 bits).
RSA_DEV uint32_t add_mod(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t d = p - y;
    return x >= d ? x - d : x + y;
}

// (x - y) mod p, x, y < p.
RSA_DEV uint32_t sub_mod(uint32_t x, uint32_t y, uint32_t p) {
    uint32_t r = x - y;
    return x < y ? r + p : r;
}

// Compile-time exponent chain: left-to-right square-and-multiply, exactly
// floor(log2 E) squarings and popcount(E)-1 products (the M(e) of SURVEY §8).
__host__ __device__ constexpr int top_bit(uint32_t e) {
    int b = 31;
    while (b > 0 && !((e >> b) & 1u)) --b;
    return b;
}

template <uint32_t E>
struct Chain {
    static constexpr int TOP = top_bit(E);
    RSA_DEV static uint32_t pow(uint32_t x, uint32_t p, uint32_t pinv) {
        uint32_t r = x;
#pragma unroll
        for (int b = TOP - 1; b >= 0; --b) {
            r = mont_mul(r, r, p, pinv);
            if ((E >> b) & 1u) r = mont_mul(r, x, p, pinv);
        }
        return r;
    }
};

// Runtime exponent, same left-to-right chain.
RSA_DEV uint32_t pow_runtime(uint32_t x, uint32_t e, uint32_t p, uint32_t pinv) {
    uint32_t r = x;
    int b = 31 - __clz(e);
    for (--b; b >= 0; --b) {
        r = mont_mul(r, r, p, pinv);
        if ((e >> b) & 1u) r = mont_mul(r, x, p, pinv);
    }
    return r;
}

// ---- 63-bit skip modulus q = 2^63 - 25 ----------------------------------------

constexpr uint64_t Q63 = 0x7FFFFFFFFFFFFFE7ull;  // 2^63 - 25 (skipgen.py:20)

// a*s mod q for q = 2^63-25, a < 2^32, s < q.  a*s = H*2^63 + L with H < 2^32,
// and 2^63 == 25 (mod q), so a*s == L + 25H < 2q: one conditional subtract.
// Equal to the reference's Schrage update (skipgen.py:92-116), which the
// reference itself pins to exact a*s mod q (test_acceptance.py:99-119).
RSA_DEV uint64_t skip_q63(uint64_t s, uint32_t a) {
    uint64_t t0 = (uint64_t)a * (uint32_t)s;
    uint64_t t1 = (uint64_t)a * (uint32_t)(s >> 32) + (t0 >> 32);  // < 2^63
    uint32_t H = (uint32_t)(t1 >> 31);
    uint64_t L = ((t1 & 0x7FFFFFFFull) << 32) | (uint32_t)t0;
    uint64_t r = L + (uint64_t)H * 25u;
    uint64_t t = r + 25u;  // r >= q  <=>  r + 25 >= 2^63
    return (t >> 63) ? (t & 0x7FFFFFFFFFFFFFFFull) : r;
}

// floor(x / d) for d < 2^62 when the quotient is known to be < 2^50: an FP64
// estimate (x, d, 1/d and the product each rounded once: relative error
// < 2^-51, so the estimate is off by at most one) fixed up exactly in
// wrapping 64-bit arithmetic; *rem = x mod d.  Stands in for the software
// 64-bit division (~100 instructions) on the setup paths.
RSA_DEV uint64_t div_small_q(uint64_t x, uint64_t d, uint64_t* rem) {
    uint64_t q = __double2ull_rz(__dmul_rn(__ull2double_rn(x), __drcp_rn(__ull2double_rn(d))));
    int64_t r = (int64_t)(x - q * d);  // true remainder +- d: within int64 since d < 2^62
    if (r < 0) { r += (int64_t)d; --q; }
    else if (r >= (int64_t)d) { r -= (int64_t)d; ++q; }
    *rem = (uint64_t)r;
    return q;
}

RSA_DEV uint64_t mod_small_q(uint64_t x, uint64_t d) {
    uint64_t r;
    div_small_q(x, d, &r);
    return r;
}

// x*y mod n for x, y < n, 2^32 <= n < 2^64, without the software 128-bit
// modulo: the quotient is estimated in FP64 (five roundings on a quotient
// below 2^64: off by < 5*2^11 < 2^14), the residue
// P - Qe*n is formed exactly in 128-bit integers, one more FP64 rounding of
// residue/n brings it into (-n, n), and one conditional add finishes.
RSA_DEV uint64_t mulmod64_fp(uint64_t x, uint64_t y, uint64_t n) {
    const unsigned __int128 P = (unsigned __int128)x * y;
    const double ninv = __drcp_rn(__ull2double_rn(n));
    const double Pd = __fma_rn(__ull2double_rn((uint64_t)(P >> 64)), 0x1p64, __ull2double_rn((uint64_t)P));
    const double qd = __dmul_rn(Pd, ninv);
    const uint64_t qe = qd >= 0x1p64 ? ~0ull : __double2ull_rz(qd);
    __int128 R = (__int128)(P - (unsigned __int128)qe * n);  // exact: |R| < 2^14 n
    const double Rd = __fma_rn((double)(int64_t)(uint64_t)((unsigned __int128)R >> 64), 0x1p64,
                               __ull2double_rn((uint64_t)R));
    const int64_t q2 = __double2ll_rn(__dmul_rn(Rd, ninv));
    R -= (__int128)q2 * (__int128)n;  // now |R| < n
    if (R < 0) R += n;
    if (R >= (__int128)n) R -= n;
    return (uint64_t)R;
}

// Exact x*y mod m for 64-bit operands (setup paths only).
RSA_DEV uint64_t mulmod64(uint64_t x, uint64_t y, uint64_t m) {
    unsigned __int128 t = (unsigned __int128)x * y;
    return (uint64_t)(t % m);
}

RSA_DEV uint64_t powmod64(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod64(r, b, m);
        e >>= 1;
        if (e) b = mulmod64(b, b, m);
    }
    return r;
}

// x*y mod (2^63-25) for x, y < 2^63 by folds of 2^64 == 50 (mod q): x*y =
// hi 2^64 + lo == lo + 50 hi < 2^69; folding that once more leaves < 2^64 +
// 1600, a third fold (+50 on a carry) < 2^64 = 2q + 50, so at most two
// subtractions of q remain.  ~24 instructions where the 2^63 fold of the
// full 128-bit product took ~40 (jump-ahead and lane-seed paths).
RSA_DEV uint64_t mulmod_q63(uint64_t x, uint64_t y) {
    const uint64_t lo = x * y, hi = __umul64hi(x, y);          // hi < 2^62
    const unsigned __int128 v = (unsigned __int128)hi * 50u + lo;  // < 2^69
    const unsigned __int128 w = (unsigned __int128)(uint64_t)(v >> 64) * 50u + (uint64_t)v;  // < 2^64 + 1600
    uint64_t r = (uint64_t)w + ((w >> 64) ? 50u : 0u);
    if (r >= Q63) r -= Q63;
    if (r >= Q63) r -= Q63;
    return r;
}

// Generic skip update for any prime q with a*a <= q: the reference Schrage
// form itself (skipgen.py:92-105), used by the test-mode (miniature) path.
RSA_DEV uint64_t skip_schrage(uint64_t s, uint64_t a, uint64_t q, uint64_t q1, uint64_t q2) {
    uint64_t hi = s / q1, lo = s - hi * q1;
    uint64_t s1 = a * lo, s2 = q2 * hi;
    return s1 >= s2 ? s1 - s2 : s1 + (q - s2);
}

// ---- float map -----------------------------------------------------------------

constexpr double MAX_BELOW_ONE = 0x1.fffffffffffffp-1;  // rsacore.py:30

// RN(x / N) given y = RN(1/N), without the hardware divide sequence.
// q0 = RN(x*y) is within 1.5 ulp of x/N; one residual step r = x - q0*N (FMA),
// q1 = RN(q0 + r*y) makes it faithful (within 1 ulp); a second step is then
// Markstein's correctly rounded final iteration (y within 1/2 ulp of 1/N, q1
// faithful => RN(q1 + (x - q1 N) y) == RN(x/N)).  x >= 0, N > 0 normal; no
// underflow/overflow at our magnitudes (x, N < 2^64).  5 FP64-pipe slots
// against __ddiv_rn's ~16.  (A 4-op variant seeded with a double-double
// reciprocal is also correctly rounded, but scheduled 3.7 % slower in the
// e=65537 fill on B200 — profiles/r01_ab_v1_v3.txt.)  Checked bit-exact
// against IEEE division by tests/test_gpu_fill.py::test_clamp_and_float_map.
RSA_DEV double div_rn(double x, double N, double y) {
    double q = __dmul_rn(x, y);
    double r = __fma_rn(-q, N, x);
    q = __fma_rn(r, y, q);
    r = __fma_rn(-q, N, x);
    return __fma_rn(r, y, q);
}

// The same quotient in 4 FP64 ops from the double-double reciprocal y + y_lo,
// y_lo = RN((1 - N y) y) (1 - N y is exact for y = RN(1/N)): x (y + y_lo) is
// within ~2^-104 relative of x/N, so q0 = RN(x y + RN(x y_lo)) is faithful
// and one Markstein step rounds it correctly.  Faster where the FP64 slot is
// worth more than the extra register (fused consumer, e = 3 fill: +1.0-1.3 %,
// profiles/r02_ab_draw.txt); slower at e = 65537, which keeps div_rn.
RSA_DEV double div_rn_dd(double x, double N, double y, double y_lo) {
    double q = __fma_rn(x, y, __dmul_rn(x, y_lo));
    double r = __fma_rn(-q, N, x);
    return __fma_rn(r, y, q);
}

RSA_DEV double recip_lo(double N, double y) { return __dmul_rn(__fma_rn(-N, y, 1.0), y); }

// r = min(fl(c)/fl(n), MAX_BELOW_ONE)  (vecgen.py:103-107)
RSA_DEV double unit_from_fl(double x, double n_float, double n_recip) {
    double r = div_rn(x, n_float, n_recip);
    return r < 1.0 ? r : MAX_BELOW_ONE;
}

RSA_DEV double to_unit(uint64_t c, double n_float, double n_recip) {
    return unit_from_fl(__ull2double_rn(c), n_float, n_recip);
}

RSA_DEV double to_unit_dd(uint64_t c, double n_float, double n_recip, double n_recip_lo) {
    const double r = div_rn_dd(__ull2double_rn(c), n_float, n_recip, n_recip_lo);
    return r < 1.0 ? r : MAX_BELOW_ONE;
}

// ---- primality (setup kernels) --------------------------------------------------

// 32-bit Montgomery exponentiation in the Montgomery domain (x_m = x*R).
RSA_DEV uint32_t mont_pow_m(uint32_t xm, uint32_t e, uint32_t onem, uint32_t p, uint32_t pinv) {
    uint32_t r = onem;
    while (e) {
        if (e & 1u) r = mont_mul(r, xm, p, pinv);
        e >>= 1;
        if (e) xm = mont_mul(xm, xm, p, pinv);
    }
    return r;
}

// p^-1 mod 2^32 for odd p (Newton: each step doubles the correct low bits).
RSA_DEV uint32_t inv32(uint32_t p) {
    uint32_t x = p;  // correct to 3 bits (p*p == 1 mod 8)
#pragma unroll
    for (int i = 0; i < 4; ++i) x *= 2u - p * x;
    return x;
}

// Strong-probable-prime test of odd n > 3 to base g (numtheory.py:60-78 semantics).
RSA_DEV bool sprp32(uint32_t n, uint32_t g, uint32_t ninv, uint32_t onem, uint32_t r2) {
    uint32_t d = n - 1;
    int u = __ffs(d) - 1;
    d >>= u;
    uint32_t gm = mont_mul(g % n, r2, n, ninv);  // g*R mod n
    uint32_t x = mont_pow_m(gm, d, onem, n, ninv);
    uint32_t minus1 = n - onem;  // (n-1)*R mod n == n - R mod n
    if (x == onem || x == minus1) return true;
    for (int j = 1; j < u; ++j) {
        x = mont_mul(x, x, n, ninv);
        if (x == minus1) return true;
    }
    return false;
}

// Exact primality for n < 2^32: trial division by primes < 100, then MR with
// bases (2, 7, 61), deterministic below 4,759,123,141.
RSA_DEV bool is_prime32(uint32_t n) {
    const uint32_t small[25] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41,
                                43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89, 97};
    if (n < 2) return false;
#pragma unroll
    for (int i = 0; i < 25; ++i) {
        if (n == small[i]) return true;
        if (n % small[i] == 0) return false;
    }
    if (n < 10201u) return true;  // no factor below 101
    uint32_t ninv = inv32(n);
    uint32_t onem = (uint32_t)((1ull << 32) % n);        // R mod n
    uint32_t r2 = (uint32_t)(((uint64_t)onem * onem) % n);  // R^2 mod n
    return sprp32(n, 2, ninv, onem, r2) && sprp32(n, 7, ninv, onem, r2) &&
           sprp32(n, 61, ninv, onem, r2);
}

RSA_DEV bool is_safe_prime32(uint32_t p) {
    return p > 4 && is_prime32(p) && is_prime32((p - 1) >> 1);
}

}  // namespace rsa
