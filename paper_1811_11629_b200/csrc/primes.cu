// primes.cu — K3 safe-prime scan, batched primality predicates, find_pair.
//
// Replaces paramfactory.safe_primes_in / _odd_prime_mask (paramfactory.py:85-130,
// a numpy segmented sieve), numtheory.is_prime64 / is_safe_prime
// (numtheory.py:81-98, trial division + Miller-Rabin) and paramfactory.find_pair
// (paramfactory.py:195-219, an outward scan of 11-mod-12 positions).
//
// Scan: every safe prime above 7 is 11 mod 12, so the candidate sequence is
// {5, 7} u {first + 12 j}.  Pass 1 decides 4096 consecutive candidates per CTA
// in three compacted stages (see k_scan_flags) into a bitmask (one u32 word
// per 32 candidates) plus a per-CTA count; pass 2 scans the counts; pass 3
// re-reads the bitmask and writes the primes in ascending order.  Only 1 bit
// per candidate touches memory, so the scan is bound by the Miller-Rabin IMAD
// work, not HBM.
#include "common.cuh"
#include "modarith.cuh"

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

// g R mod n for a small base g by a doubling chain on R mod n (ALU only)
RSA_DEV uint32_t small_base_m(uint32_t g, uint32_t onem, uint32_t n) {
    uint32_t x = onem;
    for (int b = 30 - __clz(g); b >= 0; --b) {
        x = add_mod(x, x, n);
        if ((g >> b) & 1u) x = add_mod(x, onem, n);
    }
    return x;
}

// strong probable prime to a small base g (numtheory.py:60-78), Montgomery domain
RSA_DEV bool sprp_small(uint32_t n, uint32_t g) {
    const uint32_t ninv = inv32(n), onem = r_mod(n);
    uint32_t d = n - 1;
    const int u = __ffs(d) - 1;
    d >>= u;
    const uint32_t x = mont_pow_m(small_base_m(g, onem, n), d, onem, n, ninv);
    const uint32_t minus1 = n - onem;
    if (x == onem || x == minus1) return true;
    uint32_t y = x;
    for (int j = 1; j < u; ++j) {
        y = mont_mul(y, y, n, ninv);
        if (y == minus1) return true;
    }
    return false;
}

// Strong probable prime to base 2 (numtheory.py:60-78): left-to-right powering
// in the Montgomery domain where "multiply by 2" is a modular doubling, so the
// 31-bit exponent costs only squarings.
RSA_DEV bool sprp2(uint32_t n) {
    const uint32_t ninv = inv32(n), onem = r_mod(n);
    uint32_t d = n - 1;
    const int u = __ffs(d) - 1;
    d >>= u;
    uint32_t x = onem;  // 1 in Montgomery form
    for (int b = 31 - __clz(d); b >= 0; --b) {
        x = mont_mul(x, x, n, ninv);
        if ((d >> b) & 1u) x = add_mod(x, x, n);
    }
    const uint32_t minus1 = n - onem;
    if (x == onem || x == minus1) return true;
    for (int j = 1; j < u; ++j) {
        x = mont_mul(x, x, n, ninv);
        if (x == minus1) return true;
    }
    return false;
}

RSA_DEV bool mr_7_61(uint32_t n) { return sprp_small(n, 7) && sprp_small(n, 61); }

// Safe-prime predicate for one scan candidate (5, 7, or p = 11 mod 12).
RSA_DEV bool candidate_is_safe(uint32_t p) {
    if (p < 10201u) return is_safe_prime32(p);  // small: exact generic path
    uint32_t q = (p - 1) >> 1;                   // odd, not divisible by 3
    if (has_small_factor(p) || has_small_factor(q)) return false;
    return sprp2(p) && sprp2(q) && mr_7_61(p) && mr_7_61(q);
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

// Pass 1 (per chunk of SCAN_CHUNK_CTAS x 16384 candidates), four kernels with
// global compaction between them so every stage runs dense, grid-balanced work:
//  (a) k_scan_sieve: a shared-memory sieve of p and (p-1)/2 by the primes
//      5..251 (candidates are already 11 mod 12) writes the CTA's 512 bitmask
//      words (zero, or the exact verdicts of small candidates) and appends the
//      survivors (~8 %) to a global list with one atomic per CTA;
//  (b) k_scan_sprp2<Q=0>: base-2 SPRP on p over that list, passers appended;
//  (c) k_scan_sprp2<Q=1>: base-2 SPRP on (p-1)/2, passers appended;
//  (d) k_scan_mr761: bases 7 and 61 on both, verdict bits OR-ed into the
//      bitmask.  Deterministic for n < 4,759,123,141; the bitmask (hence the
//      output) does not depend on the append order.
constexpr uint32_t SCAN_CHUNK_CTAS = 1024;

// SIEVE = true: CTAs whose candidates are all 11 mod 12 and >= 10201 (no
// sieving prime divides p or q trivially, MR's bases are below n);
// SIEVE = false: the (at most one or two) leading CTAs of a range that starts
// low, decided by trial division with small candidates settled exactly.
// Split into two kernels so the hot sieve kernel stays register-lean.
template <bool SIEVE>
__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_sieve(ScanRange R, uint64_t cta0, uint32_t* __restrict__ words, uint32_t* __restrict__ surv,
             uint32_t* __restrict__ nsurv) {
    __shared__ uint32_t flags[WORDS_PER_CTA];
    __shared__ uint8_t comp[SIEVE ? SCAN_PER_CTA : 4];
    __shared__ uint16_t start[2 * NSIEVE];
    __shared__ uint16_t wcnt[SCAN_ITERS][SCAN_BLOCK / 32];  // survivors per (iteration, warp)
    __shared__ uint32_t gbase;
    const uint64_t cta = cta0 + blockIdx.x;
    const uint64_t base = cta * SCAN_PER_CTA;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t w = threadIdx.x; w < WORDS_PER_CTA; w += SCAN_BLOCK) flags[w] = 0;
    if constexpr (SIEVE) {
        uint32_t* c32 = reinterpret_cast<uint32_t*>(comp);
        for (uint32_t u = threadIdx.x; u < SCAN_PER_CTA / 4; u += SCAN_BLOCK) c32[u] = 0;
        if (threadIdx.x < 2 * NSIEVE) {
            const SievePrime sp = c_sieve[threadIdx.x >> 1];
            const uint64_t P0 = R.first + 12ull * (base - R.nspec);
            const uint32_t l = sp.l;
            uint32_t r, inv;
            if (threadIdx.x & 1) { r = (uint32_t)(((P0 - 1) >> 1) % l); inv = sp.inv6; }
            else { r = (uint32_t)(P0 % l); inv = sp.inv12; }
            start[threadIdx.x] = (uint16_t)(((l - r) % l) * inv % l);
        }
        __syncthreads();
        for (int k = 0; k < 2 * NSIEVE; ++k) {
            const uint32_t l = c_sieve[k >> 1].l;
            for (uint32_t u = start[k] + l * threadIdx.x; u < SCAN_PER_CTA; u += l * SCAN_BLOCK) comp[u] = 1;
        }
    }
    __syncthreads();
    // verdict per candidate: sieve survivor, or trial-division survivor with
    // small candidates decided exactly (their bit set here, not listed)
    auto keep_at = [&](uint32_t off, bool decide) -> bool {
        const uint64_t j = base + off;
        if (j >= R.total) return false;
        if constexpr (SIEVE) {
            return !comp[off];
        } else {
            const uint32_t c = cand_at(R, j);
            if (c < 10201u) {
                if (decide && is_safe_prime32(c)) atomicOr(&flags[off >> 5], 1u << (off & 31));
                return false;
            }
            return !has_small_factor(c) && !has_small_factor((c - 1) >> 1);
        }
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

// Append the lanes with keep=true to out[] (one atomic per warp).
RSA_DEV void append_warp(bool keep, uint32_t v, uint32_t* out, uint32_t* n) {
    const int lane = threadIdx.x & 31;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    uint32_t pos = 0;
    if (lane == 0 && bal) pos = atomicAdd(n, __popc(bal));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (keep) out[pos + __popc(bal & ((1u << lane) - 1))] = v;
}

template <int Q>
__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_sprp2(ScanRange R, const uint32_t* __restrict__ in, const uint32_t* __restrict__ nin,
             uint32_t* __restrict__ out, uint32_t* __restrict__ nout) {
    const uint32_t n = *nin;
    const uint32_t stride = gridDim.x * SCAN_BLOCK;
    for (uint32_t i0 = blockIdx.x * SCAN_BLOCK; i0 < n; i0 += stride) {  // warp-uniform trip count
        const uint32_t i = i0 + threadIdx.x;
        uint32_t j = 0;
        bool keep = false;
        if (i < n) {
            j = in[i];
            const uint32_t p = cand_at(R, j);
            keep = sprp2(Q ? (p - 1) >> 1 : p);
        }
        append_warp(keep, j, out, nout);
    }
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan_mr761(ScanRange R, const uint32_t* __restrict__ in, const uint32_t* __restrict__ nin,
             uint32_t* __restrict__ words) {
    const uint32_t n = *nin;
    for (uint32_t i = blockIdx.x * SCAN_BLOCK + threadIdx.x; i < n; i += gridDim.x * SCAN_BLOCK) {
        const uint32_t j = in[i];
        const uint32_t p = cand_at(R, j);
        if (mr_7_61(p) && mr_7_61((p - 1) >> 1)) atomicOr(&words[j >> 5], 1u << (j & 31));
    }
}

// per-CTA-range population counts of the finished bitmask
__global__ void __launch_bounds__(WORDS_PER_CTA)
k_scan_counts(const uint32_t* __restrict__ words, uint32_t* __restrict__ counts) {
    __shared__ uint32_t tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    uint32_t c = __popc(words[(uint64_t)blockIdx.x * WORDS_PER_CTA + threadIdx.x]);
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, c);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// Exclusive scan of the per-CTA counts (single CTA, chunked, deterministic).
__global__ void __launch_bounds__(1024)
k_scan_offsets(const uint32_t* __restrict__ counts, uint64_t n, uint64_t* __restrict__ offsets,
               uint64_t* __restrict__ total) {
    __shared__ uint64_t part[1024];
    const uint64_t per = (n + 1023) / 1024;
    const uint64_t b = threadIdx.x * per, e = min(n, b + per);
    uint64_t sum = 0;
    for (uint64_t i = b; i < e; ++i) sum += counts[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (int t = 0; t < 1024; ++t) { uint64_t v = part[t]; part[t] = run; run += v; }
        *total = run;
    }
    __syncthreads();
    uint64_t run = part[threadIdx.x];
    for (uint64_t i = b; i < e; ++i) { offsets[i] = run; run += counts[i]; }
}

__global__ void __launch_bounds__(WORDS_PER_CTA)
k_scan_write(ScanRange R, const uint32_t* __restrict__ words, const uint64_t* __restrict__ offsets,
             uint32_t* __restrict__ out, uint64_t out_cap) {
    __shared__ uint32_t warp_tot[WORDS_PER_CTA / 32];
    const uint64_t w = (uint64_t)blockIdx.x * WORDS_PER_CTA + threadIdx.x;
    const uint32_t bits = words[w];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t c = __popc(bits), incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (int k = 0; k < warp; ++k) before += warp_tot[k];
    uint64_t pos = offsets[blockIdx.x] + before + incl - c;
    uint32_t b = bits;
    while (b) {
        int bit = __ffs(b) - 1;
        b &= b - 1;
        if (pos < out_cap) out[pos] = cand_at(R, w * 32 + bit);
        ++pos;
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

// scratch: words | counts | offsets | surv | surv2 | 3 counters
extern "C" uint64_t rsa_safe_prime_scan_scratch_bytes(uint64_t lo, uint64_t hi) {
    ScanRange R;
    if (!make_range(lo, hi, &R)) return 0;
    uint64_t ctas = scan_ctas(R);
    if (ctas == 0) ctas = 1;
    uint64_t words = ctas * WORDS_PER_CTA * 4, counts = ((ctas * 4 + 15) / 16) * 16;
    uint64_t lists = 2 * chunk_ctas(ctas) * SCAN_PER_CTA * 4;
    return words + counts + ctas * 8 + lists + 16;  // 3 counters
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
    p += cc * SCAN_PER_CTA * 4;
    uint32_t* surv2 = reinterpret_cast<uint32_t*>(p);
    p += cc * SCAN_PER_CTA * 4;
    uint32_t* ctr = reinterpret_cast<uint32_t*>(p);  // survivors, base-2(p) passers, base-2(q) passers
    const unsigned mr_grid = 148 * 8;
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
        cudaError_t err = cudaMemsetAsync(ctr, 0, 3 * sizeof(uint32_t), st);
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
        k_scan_sprp2<0><<<mr_grid, SCAN_BLOCK, 0, st>>>(R, surv, ctr, surv2, ctr + 1);
        if ((rc = launch_status("rsa_safe_prime_scan(sprp2 p)"))) return rc;
        k_scan_sprp2<1><<<mr_grid, SCAN_BLOCK, 0, st>>>(R, surv2, ctr + 1, surv, ctr + 2);
        if ((rc = launch_status("rsa_safe_prime_scan(sprp2 q)"))) return rc;
        k_scan_mr761<<<mr_grid, SCAN_BLOCK, 0, st>>>(R, surv, ctr + 2, words);
        if ((rc = launch_status("rsa_safe_prime_scan(mr 7,61)"))) return rc;
    }
    k_scan_counts<<<(unsigned)ctas, WORDS_PER_CTA, 0, st>>>(words, counts);
    if ((rc = launch_status("rsa_safe_prime_scan(counts)"))) return rc;
    k_scan_offsets<<<1, 1024, 0, st>>>(counts, ctas, offsets, count);
    if ((rc = launch_status("rsa_safe_prime_scan(offsets)"))) return rc;
    k_scan_write<<<(unsigned)ctas, WORDS_PER_CTA, 0, st>>>(R, words, offsets, out, out_cap);
    return launch_status("rsa_safe_prime_scan(write)");
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
