// primes.cu — K3 safe-prime scan, batched primality predicates, find_pair.
//
// Replaces paramfactory.safe_primes_in / _odd_prime_mask (paramfactory.py:85-130,
// a numpy segmented sieve), numtheory.is_prime64 / is_safe_prime
// (numtheory.py:81-98, trial division + Miller-Rabin) and paramfactory.find_pair
// (paramfactory.py:195-219, an outward scan of 11-mod-12 positions).
//
// Scan: every safe prime above 7 is 11 mod 12, so the candidate sequence is
// {5, 7} u {first + 12 j}.  Pass 1 decides 16384 consecutive candidates per
// CTA in three compacted stages (see the comment above SCAN_CHUNK_CTAS) into a
// bitmask (one u32 word per 32 candidates); pass 2 counts and scans; pass 3
// re-reads the bitmask and writes the primes in ascending order.  Only 1 bit
// per candidate touches memory, so the scan is bound by the base-2 SPRP IMAD
// work, not HBM.
#include "common.cuh"
#include "modarith.cuh"
#include "spsp2_table.inc"

namespace rsa {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITERS = 64;
constexpr uint64_t SCAN_PER_CTA = (uint64_t)SCAN_BLOCK * SCAN_ITERS;  // 16384 candidates
constexpr int WORDS_PER_CTA = (int)(SCAN_PER_CTA / 32);                  // 512

// n is divisible by odd l  <=>  n * l^-1 mod 2^32 <= floor((2^32-1)/l)
struct DivTest {
    uint32_t inv, lim;
};
constexpr uint32_t cinv32(uint32_t l) {
    uint32_t x = l;
    for (int i = 0; i < 5; ++i) x *= 2u - l * x;
    return x;
}
#define DT(l) DivTest{cinv32(l), 0xFFFFFFFFu / (l)}
__constant__ DivTest c_div[23] = {DT(5),  DT(7),  DT(11), DT(13), DT(17), DT(19), DT(23), DT(29),
                                  DT(31), DT(37), DT(41), DT(43), DT(47), DT(53), DT(59), DT(61),
                                  DT(67), DT(71), DT(73), DT(79), DT(83), DT(89), DT(97)};
#undef DT

// Shared-memory sieve primes 5..251 with 12^-1 and 6^-1 mod l: for the CTA's
// candidates p_u = P0 + 12u (q_u = Q0 + 6u), l | p_u <=> u == -P0 12^-1 (mod l).
constexpr int NSIEVE = 52;
struct SievePrime {
    uint16_t l, inv12, inv6;
};
__constant__ SievePrime c_sieve[NSIEVE] = {
    {5, 3, 1}, {7, 3, 6}, {11, 1, 2}, {13, 12, 11}, {17, 10, 3}, {19, 8, 16},
    {23, 2, 4}, {29, 17, 5}, {31, 13, 26}, {37, 34, 31}, {41, 24, 7}, {43, 18, 36},
    {47, 4, 8}, {53, 31, 9}, {59, 5, 10}, {61, 56, 51}, {67, 28, 56}, {71, 6, 12},
    {73, 67, 61}, {79, 33, 66}, {83, 7, 14}, {89, 52, 15}, {97, 89, 81}, {101, 59, 17},
    {103, 43, 86}, {107, 9, 18}, {109, 100, 91}, {113, 66, 19}, {127, 53, 106}, {131, 11, 22},
    {137, 80, 23}, {139, 58, 116}, {149, 87, 25}, {151, 63, 126}, {157, 144, 131}, {163, 68, 136},
    {167, 14, 28}, {173, 101, 29}, {179, 15, 30}, {181, 166, 151}, {191, 16, 32}, {193, 177, 161},
    {197, 115, 33}, {199, 83, 166}, {211, 88, 176}, {223, 93, 186}, {227, 19, 38}, {229, 210, 191},
    {233, 136, 39}, {239, 20, 40}, {241, 221, 201}, {251, 21, 42},
};

// Sieve primes 257 .. RSA_SIEVE_MAX, generated at compile time.  Too sparse
// for the cooperative loop (fewer marks per CTA than threads), so each thread
// takes whole (prime, p-or-q) entries.  Sieving p and q this far leaves ~0.44x
// the survivors of the 251 bound, and the base-2 SPRP stages after the sieve
// cost ~70x more per survivor than a mark.
#ifndef RSA_SIEVE_MAX
#define RSA_SIEVE_MAX 8192
#endif
constexpr bool cx_is_prime(uint32_t n) {
    if (n < 2) return false;
    for (uint32_t f = 2; f * f <= n; ++f)
        if (n % f == 0) return false;
    return true;
}
constexpr uint32_t cx_powmod(uint32_t b, uint32_t e, uint32_t m) {
    uint32_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = r * b % m;
        b = b * b % m;
        e >>= 1;
    }
    return r;
}
constexpr int cx_count_primes(uint32_t lo, uint32_t hi) {
    int c = 0;
    for (uint32_t n = lo; n < hi; ++n) c += cx_is_prime(n);
    return c;
}
constexpr int NBIG = cx_count_primes(257, RSA_SIEVE_MAX);
struct BigPrime {
    uint16_t l, inv12, inv6, r32;  // r32 = 2^32 mod l
    uint64_t M;                    // floor((2^64 - 1) / l) + 1: a mod l = mulhi64(M a, l) for 32-bit a
};
struct BigTable {
    BigPrime e[NBIG];
};
constexpr BigTable cx_big_table() {
    BigTable t{};
    int k = 0;
    for (uint32_t n = 257; n < RSA_SIEVE_MAX; ++n)
        if (cx_is_prime(n))
            t.e[k++] = BigPrime{(uint16_t)n, (uint16_t)cx_powmod(12, n - 2, n), (uint16_t)cx_powmod(6, n - 2, n),
                                (uint16_t)((1ull << 32) % n), ~0ull / n + 1};
    return t;
}
static_assert(RSA_SIEVE_MAX <= 65536 && RSA_SIEVE_MAX < 10201, "sieve primes must stay below the smallest sieved candidate");
__device__ const BigTable g_big = cx_big_table();

// branch-free: no early exit, so a warp never waits on its slowest lane here
RSA_DEV bool has_small_factor(uint32_t n) {
    bool f = false;
#pragma unroll
    for (int i = 0; i < 23; ++i) f |= n * c_div[i].inv <= c_div[i].lim;
    return f;
}

// 2^32 mod n for odd n in (2^29, 2^32): 2^32 - k n with k = floor(2^32 / n) <= 7
RSA_DEV uint32_t r_mod(uint32_t n) {
    uint32_t r = 0u - n;  // 2^32 - n
    while (r >= n) r -= n;
    return r;
}

// The 2314 base-2 strong pseudoprimes below 2^32 (tools/gen_spsp2.c, which
// decides compositeness with the deterministic bases 2, 7, 61).  An n < 2^32
// that is a base-2 SPRP is prime iff it is not in this table, so the scan's
// last stage is a lookup instead of two more exponentiations.  The table is
// bucketed at compile time by a multiplicative hash (4096 buckets, at most 4
// entries each): one load of the bucket bounds, then independent loads of
// its entries.
constexpr int SPSP_HASH_BITS = 12, SPSP_NB = 1 << SPSP_HASH_BITS, SPSP_MAXB = 4;
__host__ __device__ constexpr uint32_t spsp_hash(uint32_t n) { return (n * 0x9E3779B1u) >> (32 - SPSP_HASH_BITS); }
struct SpspHash {
    uint16_t start[SPSP_NB + 1];
    uint32_t v[RSA_SPSP2_COUNT];
};
constexpr SpspHash cx_spsp_hash() {
    const uint32_t tab[RSA_SPSP2_COUNT] = {RSA_SPSP2_TABLE};
    SpspHash h{};
    uint16_t fill[SPSP_NB] = {};
    for (uint32_t k = 0; k < RSA_SPSP2_COUNT; ++k) ++h.start[spsp_hash(tab[k]) + 1];
    for (int b = 0; b < SPSP_NB; ++b) h.start[b + 1] += h.start[b];
    for (uint32_t k = 0; k < RSA_SPSP2_COUNT; ++k) {
        const uint32_t b = spsp_hash(tab[k]);
        h.v[h.start[b] + fill[b]++] = tab[k];
    }
    return h;
}
constexpr int cx_spsp_max_bucket(const SpspHash& h) {
    int m = 0;
    for (int b = 0; b < SPSP_NB; ++b) m = h.start[b + 1] - h.start[b] > m ? h.start[b + 1] - h.start[b] : m;
    return m;
}
constexpr SpspHash kSpspHash = cx_spsp_hash();
static_assert(cx_spsp_max_bucket(kSpspHash) <= SPSP_MAXB, "spsp(2) hash bucket overflow");
__device__ const SpspHash g_spsp = kSpspHash;

RSA_DEV bool is_spsp2(uint32_t n) {
    const uint32_t b = spsp_hash(n);
    const uint32_t lo = __ldg(&g_spsp.start[b]), hi = __ldg(&g_spsp.start[b + 1]);
    bool hit = false;
#pragma unroll
    for (uint32_t k = 0; k < SPSP_MAXB; ++k)
        if (lo + k < hi) hit |= __ldg(&g_spsp.v[lo + k]) == n;
    return hit;
}

struct ScanRange {
    uint64_t first;   // first 11-mod-12 candidate
    uint64_t total;   // nspec + main candidates
    uint32_t spec[2];
    uint32_t nspec;
};

RSA_DEV uint32_t cand_at(const ScanRange& R, uint64_t j) {
    return j < R.nspec ? R.spec[j] : (uint32_t)(R.first + 12ull * (j - R.nspec));
}

// Pass 1 (per chunk of SCAN_CHUNK_CTAS x 16384 candidates), three kernels with
// global compaction between them so every stage runs dense, grid-balanced work:
//  (a) k_scan_sieve: a shared-memory sieve of p and (p-1)/2 by the primes
//      5..251 (candidates are already 11 mod 12) writes the CTA's 512 bitmask
//      words (zero, or the exact verdicts of small candidates) and appends the
//      survivors (~8 %) to a global list with one atomic per CTA;
//  (b) k_scan_sprp2: base-2 SPRP on p over that list, passers appended;
//  (c) k_scan_final: base-2 SPRP on (p-1)/2, then p and (p-1)/2 must both be
//      absent from the base-2 strong-pseudoprime table (c_spsp2); verdict bits
//      OR-ed into the bitmask.  Exact for n < 2^32 (the table is complete
//      there); the bitmask (hence the output) does not depend on the append
//      order.
#ifndef RSA_SCAN_CHUNK_CTAS
#define RSA_SCAN_CHUNK_CTAS 4096
#endif
constexpr uint32_t SCAN_CHUNK_CTAS = RSA_SCAN_CHUNK_CTAS;
// Capacity of the survivor lists per CTA.  Sieving by 5, 7, 11 and 13 alone
// leaves exactly 3*5*9*11 = 1485 of every 5*7*11*13 = 5005 consecutive
// 11-mod-12 candidates (p and (p-1)/2 each avoid one residue class per
// prime, CRT), so a CTA's 16384 candidates (< 4 periods) hold at most
// 4 * 1485 = 5940 <= 6144 survivors; the trial-division CTAs test the same
// primes.  The base-2 passers are a subset.
constexpr uint64_t LIST_PER_CTA = SCAN_PER_CTA * 3 / 8;
static_assert(4 * 1485 <= LIST_PER_CTA && SCAN_PER_CTA <= 4 * 5005, "survivor bound");

// Wheel for 5, 7, 11, 13.  With s = -P0 12^-1 (mod 5005), candidate u of a
// CTA has l | p_u iff u = s (mod l) and l | q_u iff u = s + 12^-1 (mod l), so
// the CTA's sieve starts as the 5005-periodic byte pattern
//   W[v] = [v = 0 or v = 12^-1 (mod l) for some l in {5, 7, 11, 13}]
// read from offset t0 = -s = P0 12^-1 (mod 5005): one funnel-shifted copy
// instead of ~16k byte marks per CTA.
constexpr uint32_t WHEEL = 5 * 7 * 11 * 13;
constexpr uint32_t cx_inv_mod(uint32_t a, uint32_t m) {
    for (uint32_t x = 1; x < m; ++x)
        if (a * x % m == 1) return x;
    return 0;
}
constexpr uint32_t WHEEL_INV12 = cx_inv_mod(12, WHEEL);
constexpr int WHEEL_WORDS = (int)((WHEEL + SCAN_PER_CTA + 3) / 4 + 1);
struct Wheel {
    uint32_t w[WHEEL_WORDS];
};
constexpr Wheel cx_wheel() {
    Wheel t{};
    const uint32_t ls[4] = {5, 7, 11, 13};
    for (uint32_t x = 0; x < 4u * WHEEL_WORDS; ++x) {
        const uint32_t v = x % WHEEL;
        bool m = false;
        for (uint32_t l : ls) m = m || v % l == 0 || v % l == WHEEL_INV12 % l;
        if (m) t.w[x / 4] |= 1u << (8 * (x % 4));
    }
    return t;
}
__device__ const Wheel g_wheel = cx_wheel();

#ifndef RSA_WHEEL2
#define RSA_WHEEL2 1
#endif
#if RSA_WHEEL2
// Second wheel for 17, 19, 23 (period 7429), OR-ed into the first.
constexpr uint32_t WHEEL2 = 17 * 19 * 23;
constexpr uint32_t WHEEL2_INV12 = cx_inv_mod(12, WHEEL2);
constexpr int WHEEL2_WORDS = (int)((WHEEL2 + SCAN_PER_CTA + 3) / 4 + 1);
struct Wheel2 {
    uint32_t w[WHEEL2_WORDS];
};
constexpr Wheel2 cx_wheel2() {
    Wheel2 t{};
    const uint32_t ls[3] = {17, 19, 23};
    for (uint32_t x = 0; x < 4u * WHEEL2_WORDS; ++x) {
        const uint32_t v = x % WHEEL2;
        bool m = false;
        for (uint32_t l : ls) m = m || v % l == 0 || v % l == WHEEL2_INV12 % l;
        if (m) t.w[x / 4] |= 1u << (8 * (x % 4));
    }
    return t;
}
__device__ const Wheel2 g_wheel2 = cx_wheel2();
#endif

// first u with l | p_u (q = false) or l | q_u (q = true), inv = 12^-1 or 6^-1 mod l
RSA_DEV uint32_t sieve_start(uint64_t P0, uint32_t l, uint32_t inv, bool q) {
    const uint64_t v = q ? (P0 - 1) >> 1 : P0;
    const uint32_t r = ((uint32_t)(v >> 32) * ((0u - l) % l) + (uint32_t)v % l) % l;
    return (l - r) % l * inv % l;
}

// sieve tiers over c_sieve: [0, 4) the wheel, [4, 16) CTA-cooperative marking,
// [16, NSIEVE) warp-cooperative, then g_big one entry per thread
constexpr int TIER_A0 = RSA_WHEEL2 ? 7 : 4, TIER_B0 = 16;
static_assert(2 * (TIER_B0 - TIER_A0) <= SCAN_BLOCK, "tier-A starts: one thread each");
static_assert(2 * (NSIEVE - TIER_B0) <= 32 * (SCAN_BLOCK / 32), "tier-B entries: <= 32 per warp");

// SIEVE = true: CTAs whose candidates are all 11 mod 12 and >= 10201 (no
// sieving prime divides p or q trivially, MR's bases are below n);
// SIEVE = false: the (at most one or two) leading CTAs of a range that starts
// low, decided by trial division with small candidates settled exactly.
// Split into two kernels so the hot sieve kernel stays register-lean.
template <bool SIEVE>
__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_sieve(ScanRange R, uint64_t cta0, uint32_t* __restrict__ words, uint32_t* __restrict__ surv,
             uint32_t* __restrict__ nsurv) {
    __shared__ uint32_t flags[SIEVE ? 1 : WORDS_PER_CTA];
    __shared__ __align__(16) uint8_t comp[SIEVE ? SCAN_PER_CTA : 4];
    __shared__ uint16_t start[SIEVE ? 2 * (TIER_B0 - TIER_A0) : 1];
    __shared__ uint16_t wcnt[SIEVE ? 1 : SCAN_ITERS][SCAN_BLOCK / 32];  // survivors per (iteration, warp)
    __shared__ uint32_t gbase;
    const uint64_t cta = cta0 + blockIdx.x;
    const uint64_t base = cta * SCAN_PER_CTA;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (!SIEVE)
        for (uint32_t w = threadIdx.x; w < WORDS_PER_CTA; w += SCAN_BLOCK) flags[w] = 0;
    if constexpr (SIEVE) {
        const uint64_t P0 = R.first + 12ull * (base - R.nspec);
        {   // wheel copy (5, 7, 11, 13; and 17, 19, 23)
            const uint32_t t0 = (uint32_t)(P0 % WHEEL) * WHEEL_INV12 % WHEEL;
            const uint32_t a0 = t0 >> 2, sh = (t0 & 3) * 8;
#if RSA_WHEEL2
            const uint32_t t1 = (uint32_t)(P0 % WHEEL2) * WHEEL2_INV12 % WHEEL2;
            const uint32_t b0 = t1 >> 2, sh2 = (t1 & 3) * 8;
#endif
            uint32_t* c32 = reinterpret_cast<uint32_t*>(comp);
            for (uint32_t x = threadIdx.x; x < SCAN_PER_CTA / 4; x += SCAN_BLOCK) {
                uint32_t w = __funnelshift_r(__ldg(&g_wheel.w[a0 + x]), __ldg(&g_wheel.w[a0 + x + 1]), sh);
#if RSA_WHEEL2
                w |= __funnelshift_r(__ldg(&g_wheel2.w[b0 + x]), __ldg(&g_wheel2.w[b0 + x + 1]), sh2);
#endif
                c32[x] = w;
            }
        }
        if (threadIdx.x < 2 * (TIER_B0 - TIER_A0)) {
            const uint32_t k = 2 * TIER_A0 + threadIdx.x;
            const SievePrime sp = c_sieve[k >> 1];
            start[threadIdx.x] = (uint16_t)sieve_start(P0, sp.l, (k & 1) ? sp.inv6 : sp.inv12, k & 1);
        }
        __syncthreads();  // wheel stored, tier-A starts ready
        // tier A: primes 17..61, the whole CTA strides through each entry
        for (int k = 0; k < 2 * (TIER_B0 - TIER_A0); ++k) {
            const uint32_t l = c_sieve[TIER_A0 + (k >> 1)].l;
            for (uint32_t u = start[k] + l * threadIdx.x; u < SCAN_PER_CTA; u += l * SCAN_BLOCK) comp[u] = 1;
        }
        {   // tier B: primes 67..251, entries dealt to warps, lanes stride each entry
            constexpr int NB_ENT = 2 * (NSIEVE - TIER_B0);
            constexpr int NWARP = SCAN_BLOCK / 32;
            const int e_l = warp + NWARP * lane;  // entry whose start this lane computes
            uint32_t st = 0;
            if (e_l < NB_ENT) {
                const uint32_t k = 2 * TIER_B0 + e_l;
                const SievePrime sp = c_sieve[k >> 1];
                st = sieve_start(P0, sp.l, (k & 1) ? sp.inv6 : sp.inv12, k & 1);
            }
            for (int i = 0; warp + NWARP * i < NB_ENT; ++i) {
                const uint32_t s0 = __shfl_sync(0xffffffffu, st, i);
                const uint32_t l = c_sieve[TIER_B0 + ((warp + NWARP * i) >> 1)].l;
                for (uint32_t u = s0 + l * lane; u < SCAN_PER_CTA; u += 32 * l) comp[u] = 1;
            }
        }
        {   // tier C: primes 257..RSA_SIEVE_MAX, one (prime, p-or-q) entry per thread at a time
            const uint64_t Q0 = (P0 - 1) >> 1;
            for (uint32_t k = threadIdx.x; k < 2u * NBIG; k += SCAN_BLOCK) {
                const BigPrime bp = g_big.e[k >> 1];
                const uint32_t l = bp.l;
                const uint64_t v = (k & 1) ? Q0 : P0;
                // Lemire's fastmod (a mod l = mulhi64(M a, l)) instead of two 32-bit divisions
                uint32_t r = (uint32_t)__umul64hi(bp.M * (uint32_t)v, l) + (uint32_t)(v >> 32) * bp.r32;
                r = r >= l ? r - l : r;
                const uint32_t inv = (k & 1) ? bp.inv6 : bp.inv12;
                const uint32_t neg = r ? l - r : 0;
                for (uint32_t u = (uint32_t)__umul64hi(bp.M * (neg * inv), l); u < SCAN_PER_CTA; u += l) comp[u] = 1;
            }
        }
    }
    __syncthreads();
    if constexpr (SIEVE) {
        // candidates past the end of the range count as sieved out
        const uint64_t valid = R.total > base ? (R.total - base < SCAN_PER_CTA ? R.total - base : SCAN_PER_CTA) : 0;
        for (uint64_t u = valid + threadIdx.x; u < SCAN_PER_CTA; u += SCAN_BLOCK) comp[u] = 1;
        __syncthreads();
        // thread t owns the 16-candidate groups g = i * SCAN_BLOCK + t (i < 4):
        // conflict-free 128-bit reads, survivors counted as zero bytes
        const uint4* c4 = reinterpret_cast<const uint4*>(comp);
        uint32_t w[16], cnt = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 v = c4[i * SCAN_BLOCK + threadIdx.x];
            w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) cnt += 4 - __popc(w[i]);
        // block exclusive scan of the counts -> one global reservation per CTA
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        __shared__ uint32_t wtot[SCAN_BLOCK / 32];
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (int k = 0; k < SCAN_BLOCK / 32; ++k) { const uint32_t c = wtot[k]; wtot[k] = run; run += c; }
            gbase = run ? atomicAdd(nsurv, run) : 0;
        }
        __syncthreads();
        uint32_t pos = gbase + wtot[warp] + inc - cnt;
        for (uint32_t x = threadIdx.x; x < WORDS_PER_CTA; x += SCAN_BLOCK) words[cta * WORDS_PER_CTA + x] = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t z = ~w[i] & 0x01010101u;
            const uint32_t u0 = 16u * ((i >> 2) * SCAN_BLOCK + threadIdx.x) + 4u * (i & 3);
            while (z) {
                surv[pos++] = (uint32_t)(base + u0 + ((__ffs(z) - 1) >> 3));
                z &= z - 1;
            }
        }
        return;
    } else {
    // verdict per candidate: trial-division survivor, small candidates decided
    // exactly (their bit set here, not listed)
    auto keep_at = [&](uint32_t off, bool decide) -> bool {
        const uint64_t j = base + off;
        if (j >= R.total) return false;
        const uint32_t c = cand_at(R, j);
        if (c < 10201u) {
            if (decide && is_safe_prime32(c)) atomicOr(&flags[off >> 5], 1u << (off & 31));
            return false;
        }
        return !has_small_factor(c) && !has_small_factor((c - 1) >> 1);
    };
    for (int it = 0; it < SCAN_ITERS; ++it) {
        const uint32_t bal = __ballot_sync(0xffffffffu, keep_at(it * SCAN_BLOCK + threadIdx.x, true));
        if (lane == 0) wcnt[it][warp] = (uint16_t)__popc(bal);
    }
    __syncthreads();
    // exclusive prefix over (iteration, warp) in row-major order, total -> global reservation
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int it = 0; it < SCAN_ITERS; ++it)
            for (int w = 0; w < SCAN_BLOCK / 32; ++w) { uint32_t c = wcnt[it][w]; wcnt[it][w] = (uint16_t)run; run += c; }
        gbase = run ? atomicAdd(nsurv, run) : 0;
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < WORDS_PER_CTA; w += SCAN_BLOCK) words[cta * WORDS_PER_CTA + w] = flags[w];
    for (int it = 0; it < SCAN_ITERS; ++it) {
        const uint32_t off = it * SCAN_BLOCK + threadIdx.x;
        const bool k = keep_at(off, false);
        const uint32_t bal = __ballot_sync(0xffffffffu, k);
        if (k) surv[gbase + wcnt[it][warp] + __popc(bal & ((1u << lane) - 1))] = (uint32_t)(base + off);
    }
    }
}

// K independent base-2 SPRP tests interleaved in one thread.  Each test is a
// chain of ~31 dependent Montgomery squarings; one chain per thread leaves the
// IMAD pipe mostly idle (64 warps x 1 chain cannot cover its latency), K
// chains per thread give the scheduler K-fold ILP.  Leading zero bits of a
// shorter exponent square the Montgomery one, which stays one, so all K run
// the same 32-bit-position loop.  Verdicts of the strong probable-prime test
// to base 2 (numtheory.py:60-78), with "multiply by 2" a modular doubling.
template <int K>
RSA_DEV void sprp2_multi(const uint32_t (&n)[K], bool (&ok)[K]) {
    uint32_t ninv[K], onem[K], d[K], x[K];
    int u[K];
    uint32_t dall = 0;
    int umax = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        ninv[k] = inv32(n[k]);
        onem[k] = r_mod(n[k]);
        d[k] = n[k] - 1;
        u[k] = __ffs(d[k]) - 1;
        d[k] >>= u[k];
        x[k] = onem[k];
        dall |= d[k];
        umax = max(umax, u[k]);
    }
    for (int b = 31 - __clz(dall); b >= 0; --b) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = mont_mul(x[k], x[k], n[k], ninv[k]);
            if ((d[k] >> b) & 1u) x[k] = add_mod(x[k], x[k], n[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) ok[k] = x[k] == onem[k] || x[k] == n[k] - onem[k];
    for (int j = 1; j < umax; ++j) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = mont_mul(x[k], x[k], n[k], ninv[k]);
            ok[k] = ok[k] || (j < u[k] && x[k] == n[k] - onem[k]);
        }
    }
}

#ifndef RSA_SPRP_ILP
#define RSA_SPRP_ILP 2
#endif
constexpr int SPRP_ILP = RSA_SPRP_ILP;
constexpr uint32_t SPRP_DUMMY = 4294967291u;  // a prime: padding lanes stay well-formed

// (b) base-2 SPRP on p over the sieve survivors, passers appended
__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_sprp2(ScanRange R, const uint32_t* __restrict__ in, const uint32_t* __restrict__ nin,
             uint32_t* __restrict__ out, uint32_t* __restrict__ nout) {
    const uint32_t n = *nin;
    const uint32_t tile = SPRP_ILP * SCAN_BLOCK, stride = gridDim.x * tile;
    for (uint32_t i0 = blockIdx.x * tile; i0 < n; i0 += stride) {  // warp-uniform trip count
        uint32_t j[SPRP_ILP], v[SPRP_ILP];
        bool ok[SPRP_ILP];
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            const uint32_t i = i0 + k * SCAN_BLOCK + threadIdx.x;
            j[k] = i < n ? in[i] : 0;
            v[k] = i < n ? cand_at(R, j[k]) : SPRP_DUMMY;
        }
        sprp2_multi<SPRP_ILP>(v, ok);
        // one reservation per warp for all SPRP_ILP groups
        const int lane = threadIdx.x & 31;
        uint32_t bal[SPRP_ILP], tot = 0;
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            ok[k] = ok[k] && i0 + k * SCAN_BLOCK + threadIdx.x < n;
            bal[k] = __ballot_sync(0xffffffffu, ok[k]);
            tot += __popc(bal[k]);
        }
        uint32_t pos = 0;
        if (lane == 0 && tot) pos = atomicAdd(nout, tot);
        pos = __shfl_sync(0xffffffffu, pos, 0);
        const uint32_t below = (1u << lane) - 1;
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            if (ok[k]) out[pos + __popc(bal[k] & below)] = j[k];
            pos += __popc(bal[k]);
        }
    }
}

// (c) base-2 SPRP on q = (p-1)/2, then both p and q looked up in the
// pseudoprime table; verdict bits OR-ed into the bitmask
__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_final(ScanRange R, const uint32_t* __restrict__ in, const uint32_t* __restrict__ nin,
             uint32_t* __restrict__ words) {
    const uint32_t n = *nin;
    const uint32_t tile = SPRP_ILP * SCAN_BLOCK, stride = gridDim.x * tile;
    for (uint32_t i0 = blockIdx.x * tile; i0 < n; i0 += stride) {
        uint32_t j[SPRP_ILP], q[SPRP_ILP];
        bool ok[SPRP_ILP];
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            const uint32_t i = i0 + k * SCAN_BLOCK + threadIdx.x;
            j[k] = i < n ? in[i] : 0;
            q[k] = i < n ? (cand_at(R, j[k]) - 1) >> 1 : SPRP_DUMMY;
        }
        sprp2_multi<SPRP_ILP>(q, ok);
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            if (ok[k] && i0 + k * SCAN_BLOCK + threadIdx.x < n && !is_spsp2(q[k]) && !is_spsp2(2 * q[k] + 1))
                atomicOr(&words[j[k] >> 5], 1u << (j[k] & 31));
        }
    }
}

// Tail of the scan: per-range (16384 candidates = 512 bitmask words) counts,
// their exclusive scan, and the ordered write.  128 threads x one uint4 cover
// a range; CTAs loop over ranges so the ~11k ranges of a full 2^31 scan run
// as one resident wave instead of 11k tiny CTAs.
constexpr int TAIL_BLOCK = WORDS_PER_CTA / 4;
static_assert(TAIL_BLOCK == 128, "one uint4 of the bitmask per thread");

RSA_DEV uint32_t block_excl_scan128(uint32_t c, uint32_t* total, uint32_t* smem4) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) smem4[warp] = incl;
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int k = 0; k < TAIL_BLOCK / 32; ++k) {
        const uint32_t t = smem4[k];
        before += k < warp ? t : 0;
        all += t;
    }
    __syncthreads();  // smem4 reusable by the next range
    *total = all;
    return before + incl - c;
}

__global__ void __launch_bounds__(TAIL_BLOCK)
k_scan_counts(const uint32_t* __restrict__ words, uint64_t ranges, uint32_t* __restrict__ counts) {
    __shared__ uint32_t wsum[TAIL_BLOCK / 32];
    for (uint64_t r = blockIdx.x; r < ranges; r += gridDim.x) {
        const uint4 v = reinterpret_cast<const uint4*>(words + r * WORDS_PER_CTA)[threadIdx.x];
        uint32_t tot;
        block_excl_scan128(__popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w), &tot, wsum);
        if (threadIdx.x == 0) counts[r] = tot;
    }
}

// Exclusive scan of the per-range counts (single CTA, deterministic).
__global__ void __launch_bounds__(1024)
k_scan_offsets(const uint32_t* __restrict__ counts, uint64_t n, uint64_t* __restrict__ offsets,
               uint64_t* __restrict__ total) {
    __shared__ uint64_t wsum[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t per = (n + 1023) / 1024;
    const uint64_t b = threadIdx.x * per, e = min(n, b + per);
    uint64_t sum = 0;
    for (uint64_t i = b; i < e; ++i) sum += counts[i];
    uint64_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t x = wsum[lane], xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, xi, d);
            if (lane >= d) xi += v;
        }
        wsum[lane] = xi - x;
        if (lane == 31) *total = xi;
    }
    __syncthreads();
    uint64_t run = wsum[warp] + incl - sum;
    for (uint64_t i = b; i < e; ++i) { offsets[i] = run; run += counts[i]; }
}

__global__ void __launch_bounds__(TAIL_BLOCK)
k_scan_write(ScanRange R, const uint32_t* __restrict__ words, uint64_t ranges,
             const uint64_t* __restrict__ offsets, uint32_t* __restrict__ out, uint64_t out_cap) {
    __shared__ uint32_t wsum[TAIL_BLOCK / 32];
    for (uint64_t r = blockIdx.x; r < ranges; r += gridDim.x) {
        const uint4 v = reinterpret_cast<const uint4*>(words + r * WORDS_PER_CTA)[threadIdx.x];
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
        uint32_t tot;
        const uint32_t ex = block_excl_scan128(__popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w), &tot, wsum);
        uint64_t pos = offsets[r] + ex;
        const uint64_t j0 = r * SCAN_PER_CTA + 128ull * threadIdx.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t bits = w4[k];
            while (bits) {
                const int bit = __ffs(bits) - 1;
                bits &= bits - 1;
                if (pos < out_cap) out[pos] = cand_at(R, j0 + 32 * k + bit);
                ++pos;
            }
        }
    }
}

// ---- literal scan: deterministic Miller-Rabin (2, 7, 61) on every odd n ----
//
// The BASELINE config-5 statement of the census: every odd n in [lo, hi) is
// tested with MR bases 2, 7, 61 (exact below 4,759,123,141) and so is
// (n-1)/2 when it is odd (numtheory.py:60-98 semantics; an even (n-1)/2 is
// rejected before MR).  No sieve and no pseudoprime table: this is the
// reference algorithm restated for the GPU, kept beside the production scan
// (rsa_safe_prime_scan) as its cross-check and as the IMAD-bound yardstick
// the sieve is measured against.  Two compacted stages per chunk so warps do
// not idle on their few prime lanes: (1) base 2 on every odd n, passers
// listed; (2) bases 7 and 61 on n, then 2, 7, 61 on (n-1)/2; verdicts go into
// the same candidate bitmask, whose count / offsets / ordered write are the
// production tail.

// g*R mod n for a small base g (binary method with modular doublings)
RSA_DEV uint32_t small_times_r(uint32_t g, uint32_t onem, uint32_t n) {
    uint32_t x = onem;
    for (int b = 30 - __clz(g); b >= 0; --b) {
        x = add_mod(x, x, n);
        if ((g >> b) & 1u) x = add_mod(x, onem, n);
    }
    return x;
}

// strong probable-prime test to the small base g of K odd n > g, interleaved
template <int K>
RSA_DEV void sprp_multi(const uint32_t (&n)[K], uint32_t g, bool (&ok)[K]) {
    uint32_t ninv[K], onem[K], gm[K], d[K], x[K];
    int u[K];
    uint32_t dall = 0;
    int umax = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        ninv[k] = inv32(n[k]);
        onem[k] = r_mod(n[k]);
        gm[k] = small_times_r(g, onem[k], n[k]);
        d[k] = n[k] - 1;
        u[k] = __ffs(d[k]) - 1;
        d[k] >>= u[k];
        x[k] = onem[k];
        dall |= d[k];
        umax = max(umax, u[k]);
    }
    for (int b = 31 - __clz(dall); b >= 0; --b) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = mont_mul(x[k], x[k], n[k], ninv[k]);
            if ((d[k] >> b) & 1u) x[k] = mont_mul(x[k], gm[k], n[k], ninv[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) ok[k] = x[k] == onem[k] || x[k] == n[k] - onem[k];
    for (int j = 1; j < umax; ++j) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = mont_mul(x[k], x[k], n[k], ninv[k]);
            ok[k] = ok[k] || (j < u[k] && x[k] == n[k] - onem[k]);
        }
    }
}

// bitmask index of n in the scan's candidate sequence ({5, 7} u first + 12 j), or ~0
RSA_DEV uint64_t cand_index(const ScanRange& R, uint32_t n) {
    for (uint32_t k = 0; k < R.nspec; ++k)
        if (R.spec[k] == n) return k;
    if (n < R.first || (n - R.first) % 12 != 0) return ~0ull;
    return R.nspec + (n - R.first) / 12;
}

constexpr uint32_t MR_SMALL = 10201u;  // below: trial division decides (no base reaches n)

// stage 1: odd n = lo_odd + 2 i, i in [i0, i1): base-2 SPRP, passers listed
__global__ void __launch_bounds__(SCAN_BLOCK)
k_mr_base2(ScanRange R, uint64_t lo_odd, uint64_t i0, uint64_t i1, uint32_t* __restrict__ list,
           uint32_t* __restrict__ nlist, uint32_t* __restrict__ words) {
    const uint64_t tile = (uint64_t)SPRP_ILP * SCAN_BLOCK, stride = (uint64_t)gridDim.x * tile;
    const int lane = threadIdx.x & 31;
    for (uint64_t b0 = i0 + blockIdx.x * tile; b0 < i1; b0 += stride) {
        uint32_t v[SPRP_ILP];
        bool ok[SPRP_ILP], in[SPRP_ILP];
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            const uint64_t i = b0 + k * SCAN_BLOCK + threadIdx.x;
            const uint64_t n = lo_odd + 2 * i;
            in[k] = i < i1;
            v[k] = in[k] && n >= MR_SMALL ? (uint32_t)n : SPRP_DUMMY;
            if (in[k] && n < MR_SMALL) {  // small n: exact by trial division
                in[k] = false;
                if (is_safe_prime32((uint32_t)n)) {
                    const uint64_t j = cand_index(R, (uint32_t)n);
                    if (j != ~0ull) atomicOr(&words[j >> 5], 1u << (j & 31));
                }
            }
        }
        sprp2_multi<SPRP_ILP>(v, ok);
        uint32_t bal[SPRP_ILP], tot = 0;
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            ok[k] = ok[k] && in[k];
            bal[k] = __ballot_sync(0xffffffffu, ok[k]);
            tot += __popc(bal[k]);
        }
        uint32_t pos = 0;
        if (lane == 0 && tot) pos = atomicAdd(nlist, tot);
        pos = __shfl_sync(0xffffffffu, pos, 0);
        const uint32_t below = (1u << lane) - 1;
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            if (ok[k]) list[pos + __popc(bal[k] & below)] = v[k];
            pos += __popc(bal[k]);
        }
    }
}

// stage 2: bases 7, 61 on n; then 2, 7, 61 on q = (n-1)/2 (odd q only)
__global__ void __launch_bounds__(SCAN_BLOCK)
k_mr_rest(ScanRange R, const uint32_t* __restrict__ list, const uint32_t* __restrict__ nlist,
          uint32_t* __restrict__ words) {
    const uint32_t n = *nlist;
    const uint32_t tile = SPRP_ILP * SCAN_BLOCK, stride = gridDim.x * tile;
    for (uint32_t b0 = blockIdx.x * tile; b0 < n; b0 += stride) {
        uint32_t v[SPRP_ILP], q[SPRP_ILP];
        bool ok[SPRP_ILP], t[SPRP_ILP];
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            const uint32_t i = b0 + k * SCAN_BLOCK + threadIdx.x;
            v[k] = i < n ? list[i] : SPRP_DUMMY;
        }
        sprp_multi<SPRP_ILP>(v, 7, ok);
        sprp_multi<SPRP_ILP>(v, 61, t);
#pragma unroll
        for (int k = 0; k < SPRP_ILP; ++k) {
            // p prime; (p-1)/2 even (p = 1 mod 4) is rejected before MR
            ok[k] = ok[k] && t[k] && (v[k] & 3u) == 3u && b0 + k * SCAN_BLOCK + threadIdx.x < n;
            q[k] = ok[k] ? v[k] >> 1 : SPRP_DUMMY;
        }
        // the warp runs the q tests only when one of its lanes needs them
        if (__any_sync(0xffffffffu, ok[0] || (SPRP_ILP > 1 && ok[SPRP_ILP - 1]))) {
            sprp2_multi<SPRP_ILP>(q, t);
#pragma unroll
            for (int k = 0; k < SPRP_ILP; ++k) ok[k] = ok[k] && t[k];
            sprp_multi<SPRP_ILP>(q, 7, t);
#pragma unroll
            for (int k = 0; k < SPRP_ILP; ++k) ok[k] = ok[k] && t[k];
            sprp_multi<SPRP_ILP>(q, 61, t);
#pragma unroll
            for (int k = 0; k < SPRP_ILP; ++k) {
                ok[k] = ok[k] && t[k];
                if (ok[k]) {
                    const uint64_t j = cand_index(R, v[k]);
                    if (j != ~0ull) atomicOr(&words[j >> 5], 1u << (j & 31));
                }
            }
        }
    }
}

__global__ void k_is_safe(const uint32_t* __restrict__ n, uint64_t count, uint8_t* __restrict__ is_p,
                          uint8_t* __restrict__ is_s) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = n[j];
        bool pr = is_prime32(v);
        if (is_p) is_p[j] = pr;
        if (is_s) is_s[j] = pr && v > 4 && is_prime32((v - 1) >> 1);
    }
}

}  // namespace rsa

using namespace rsa;

static bool make_range(uint64_t lo, uint64_t hi, ScanRange* R) {
    if (hi > (1ull << 32)) return false;
    if (lo < 2) lo = 2;
    R->nspec = 0;
    if (lo <= 5 && 5 < hi) R->spec[R->nspec++] = 5;
    if (lo <= 7 && 7 < hi) R->spec[R->nspec++] = 7;
    uint64_t body = lo > 11 ? lo : 11;
    uint64_t first = body + (11 + 12 - body % 12) % 12;
    R->first = first;
    uint64_t main = hi > first ? (hi - first + 11) / 12 : 0;
    R->total = R->nspec + main;
    return true;
}

static uint64_t scan_ctas(const ScanRange& R) { return (R.total + SCAN_PER_CTA - 1) / SCAN_PER_CTA; }

static uint64_t chunk_ctas(uint64_t ctas) { return ctas < SCAN_CHUNK_CTAS ? ctas : SCAN_CHUNK_CTAS; }

// scratch: words | counts | offsets | surv | surv2 | counters
extern "C" uint64_t rsa_safe_prime_scan_scratch_bytes(uint64_t lo, uint64_t hi) {
    ScanRange R;
    if (!make_range(lo, hi, &R)) return 0;
    uint64_t ctas = scan_ctas(R);
    if (ctas == 0) ctas = 1;
    uint64_t words = ctas * WORDS_PER_CTA * 4, counts = ((ctas * 4 + 15) / 16) * 16;
    uint64_t lists = 2 * chunk_ctas(ctas) * LIST_PER_CTA * 4;
    return words + counts + ctas * 8 + lists + 16;  // counters
}

extern "C" int rsa_safe_prime_scan(uint64_t lo, uint64_t hi, uint32_t* out, uint64_t out_cap,
                                   uint64_t* count, void* scratch, uint64_t scratch_bytes,
                                   void* stream) {
    ScanRange R;
    if (!count || !make_range(lo, hi, &R)) return RSA_EINVAL;
    if (scratch_bytes < rsa_safe_prime_scan_scratch_bytes(lo, hi) || !scratch) return RSA_EINVAL;
    if (out_cap && !out) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    uint64_t ctas = scan_ctas(R);
    if (ctas == 0) {
        cudaError_t err = cudaMemsetAsync(count, 0, sizeof(uint64_t), st);
        if (err != cudaSuccess) { set_last_error("rsa_safe_prime_scan", err); return RSA_ECUDA; }
        return RSA_OK;
    }
    const uint64_t cc = chunk_ctas(ctas);
    char* p = static_cast<char*>(scratch);
    uint32_t* words = reinterpret_cast<uint32_t*>(p);
    p += ctas * WORDS_PER_CTA * 4;
    uint32_t* counts = reinterpret_cast<uint32_t*>(p);
    p += ((ctas * 4 + 15) / 16) * 16;
    uint64_t* offsets = reinterpret_cast<uint64_t*>(p);
    p += ctas * 8;
    uint32_t* surv = reinterpret_cast<uint32_t*>(p);
    p += cc * LIST_PER_CTA * 4;
    uint32_t* surv2 = reinterpret_cast<uint32_t*>(p);
    p += cc * LIST_PER_CTA * 4;
    uint32_t* ctr = reinterpret_cast<uint32_t*>(p);  // sieve survivors, base-2(p) passers
    const unsigned mr_grid = 148 * (16 / SPRP_ILP);
    // CTAs [0, small_ctas) hold a special candidate or one below 10201
    uint64_t small_ctas = 0;
    while (small_ctas < ctas) {
        const uint64_t b = small_ctas * SCAN_PER_CTA;
        if (b >= R.nspec && R.first + 12ull * (b - R.nspec) >= 10201u) break;
        ++small_ctas;
    }
    int rc;
    for (uint64_t c0 = 0; c0 < ctas; c0 += cc) {
        const uint64_t n = ctas - c0 < cc ? ctas - c0 : cc;
        cudaError_t err = cudaMemsetAsync(ctr, 0, 2 * sizeof(uint32_t), st);
        if (err != cudaSuccess) { set_last_error("rsa_safe_prime_scan(memset)", err); return RSA_ECUDA; }
        // leading CTAs holding candidates below 10201 (or 5, 7) take the trial-division kernel
        const uint64_t nsmall = c0 < small_ctas ? (small_ctas - c0 < n ? small_ctas - c0 : n) : 0;
        if (nsmall) {
            k_scan_sieve<false><<<(unsigned)nsmall, SCAN_BLOCK, 0, st>>>(R, c0, words, surv, ctr);
            if ((rc = launch_status("rsa_safe_prime_scan(trial)"))) return rc;
        }
        if (n > nsmall) {
            k_scan_sieve<true><<<(unsigned)(n - nsmall), SCAN_BLOCK, 0, st>>>(R, c0 + nsmall, words, surv, ctr);
            if ((rc = launch_status("rsa_safe_prime_scan(sieve)"))) return rc;
        }
        k_scan_sprp2<<<mr_grid, SCAN_BLOCK, 0, st>>>(R, surv, ctr, surv2, ctr + 1);
        if ((rc = launch_status("rsa_safe_prime_scan(sprp2 p)"))) return rc;
        k_scan_final<<<mr_grid, SCAN_BLOCK, 0, st>>>(R, surv2, ctr + 1, words);
        if ((rc = launch_status("rsa_safe_prime_scan(sprp2 q + table)"))) return rc;
    }
    const unsigned tail_grid = (unsigned)(ctas < 148 * 16 ? ctas : 148 * 16);
    k_scan_counts<<<tail_grid, TAIL_BLOCK, 0, st>>>(words, ctas, counts);
    if ((rc = launch_status("rsa_safe_prime_scan(counts)"))) return rc;
    k_scan_offsets<<<1, 1024, 0, st>>>(counts, ctas, offsets, count);
    if ((rc = launch_status("rsa_safe_prime_scan(offsets)"))) return rc;
    k_scan_write<<<tail_grid, TAIL_BLOCK, 0, st>>>(R, words, ctas, offsets, out, out_cap);
    return launch_status("rsa_safe_prime_scan(write)");
}

// literal scan: chunks of MR_CHUNK odd candidates, list capacity bounded by
// the prime density among odd n >= 10201 (< 2 / ln 10201 < 1/4)
constexpr uint64_t MR_CHUNK = 1ull << 26;
constexpr uint64_t MR_LIST = MR_CHUNK / 4 + 4096;

static bool mr_range(uint64_t lo, uint64_t hi, uint64_t* lo_odd, uint64_t* n_odd) {
    if (hi > (1ull << 32)) return false;
    if (lo < 3) lo = 3;
    *lo_odd = lo | 1;
    *n_odd = hi > *lo_odd ? (hi - *lo_odd + 1) / 2 : 0;
    return true;
}

extern "C" uint64_t rsa_safe_prime_scan_mr_scratch_bytes(uint64_t lo, uint64_t hi) {
    ScanRange R;
    uint64_t a, b;
    if (!make_range(lo, hi, &R) || !mr_range(lo, hi, &a, &b)) return 0;
    uint64_t ctas = scan_ctas(R);
    if (ctas == 0) ctas = 1;
    uint64_t words = ctas * WORDS_PER_CTA * 4, counts = ((ctas * 4 + 15) / 16) * 16;
    return words + counts + ctas * 8 + MR_LIST * 4 + 16;
}

extern "C" int rsa_safe_prime_scan_mr(uint64_t lo, uint64_t hi, uint32_t* out, uint64_t out_cap,
                                      uint64_t* count, void* scratch, uint64_t scratch_bytes,
                                      void* stream) {
    ScanRange R;
    uint64_t lo_odd, n_odd;
    if (!count || !make_range(lo, hi, &R) || !mr_range(lo, hi, &lo_odd, &n_odd)) return RSA_EINVAL;
    if (scratch_bytes < rsa_safe_prime_scan_mr_scratch_bytes(lo, hi) || !scratch) return RSA_EINVAL;
    if (out_cap && !out) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    uint64_t ctas = scan_ctas(R);
    if (ctas == 0) {
        cudaError_t err = cudaMemsetAsync(count, 0, sizeof(uint64_t), st);
        if (err != cudaSuccess) { set_last_error("rsa_safe_prime_scan_mr", err); return RSA_ECUDA; }
        return RSA_OK;
    }
    char* p = static_cast<char*>(scratch);
    uint32_t* words = reinterpret_cast<uint32_t*>(p);
    p += ctas * WORDS_PER_CTA * 4;
    uint32_t* counts = reinterpret_cast<uint32_t*>(p);
    p += ((ctas * 4 + 15) / 16) * 16;
    uint64_t* offsets = reinterpret_cast<uint64_t*>(p);
    p += ctas * 8;
    uint32_t* list = reinterpret_cast<uint32_t*>(p);
    p += MR_LIST * 4;
    uint32_t* ctr = reinterpret_cast<uint32_t*>(p);
    cudaError_t err = cudaMemsetAsync(words, 0, ctas * WORDS_PER_CTA * 4, st);
    if (err != cudaSuccess) { set_last_error("rsa_safe_prime_scan_mr(memset)", err); return RSA_ECUDA; }
    const unsigned grid = 148 * (16 / SPRP_ILP);
    int rc;
    for (uint64_t c0 = 0; c0 < n_odd; c0 += MR_CHUNK) {
        const uint64_t c1 = n_odd - c0 < MR_CHUNK ? n_odd : c0 + MR_CHUNK;
        if ((err = cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st)) != cudaSuccess) {
            set_last_error("rsa_safe_prime_scan_mr(memset)", err);
            return RSA_ECUDA;
        }
        k_mr_base2<<<grid, SCAN_BLOCK, 0, st>>>(R, lo_odd, c0, c1, list, ctr, words);
        if ((rc = launch_status("rsa_safe_prime_scan_mr(base 2)"))) return rc;
        k_mr_rest<<<grid, SCAN_BLOCK, 0, st>>>(R, list, ctr, words);
        if ((rc = launch_status("rsa_safe_prime_scan_mr(bases 7, 61; q)"))) return rc;
    }
    const unsigned tail_grid = (unsigned)(ctas < 148 * 16 ? ctas : 148 * 16);
    k_scan_counts<<<tail_grid, TAIL_BLOCK, 0, st>>>(words, ctas, counts);
    if ((rc = launch_status("rsa_safe_prime_scan_mr(counts)"))) return rc;
    k_scan_offsets<<<1, 1024, 0, st>>>(counts, ctas, offsets, count);
    if ((rc = launch_status("rsa_safe_prime_scan_mr(offsets)"))) return rc;
    k_scan_write<<<tail_grid, TAIL_BLOCK, 0, st>>>(R, words, ctas, offsets, out, out_cap);
    return launch_status("rsa_safe_prime_scan_mr(write)");
}

extern "C" int rsa_is_safe_prime32(const uint32_t* n, uint64_t count, uint8_t* is_prime,
                                   uint8_t* is_safe, void* stream) {
    if (!n && count) return RSA_EINVAL;
    if (count == 0) return RSA_OK;
    unsigned grid = grid_for(count, 256);
    if (grid > 148 * 32) grid = 148 * 32;
    k_is_safe<<<grid, 256, 0, as_stream(stream)>>>(n, count, is_prime, is_safe);
    return launch_status("rsa_is_safe_prime32");
}
