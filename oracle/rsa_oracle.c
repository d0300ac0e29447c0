/*
 * rsa_oracle.c — CPU ORACLE in plain C (test infrastructure only).
 *
 * A scalar C restatement of the reference algorithm
 * (/root/reference/pkg/src/rsarand) for the sizes the numpy oracle cannot
 * reach in seconds: long lane runs, the full safe-prime census of
 * [2^31, 2^32), and derive_stream_params over 2^20 stream ids.  Exact 128-bit
 * integer arithmetic (unsigned __int128) and IEEE double division; no
 * Montgomery, no tricks — deliberately unlike the CUDA kernels it checks.
 * Only tests/, smoke() and bench.py's CPU legs load it (via oracle/coracle.py);
 * it is pinned against the reference's own golden vectors by
 * tests/test_oracle_golden.py.
 *
 *   oracle_fill      vecgen.next_block_raw/floats_from_raw   vecgen.py:87-107
 *                    (many instances, lane-major state)      + rsacore.py:213-233
 *   oracle_census    paramfactory.safe_primes_in             paramfactory.py:85-130
 *   oracle_derive    paramfactory.derive_stream_params       paramfactory.py:195-278
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
    uint64_t p1, p2, e, a, q, p2inv;  /* p2inv = p2^-1 mod p1 */
    uint64_t mode;                    /* 0 lcg, 1 unit, 2 const */
    uint64_t n;
} oracle_params;

static uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = (uint64_t)((u128)r * b % m);
        b = (uint64_t)((u128)b * b % m);
        e >>= 1;
    }
    return r;
}

/* Advance `lanes` lanes of instance P by `blocks` steps (lane-major state),
 * writing raw[k*out_stride + g] / f64[...] (either may be NULL). */
void oracle_fill(const oracle_params* P, uint64_t lanes, uint64_t blocks, uint64_t* m1, uint64_t* m2,
                 uint64_t* s, uint64_t* raw, double* f64, uint64_t out_stride) {
    const double nf = (double)P->n;
    for (uint64_t g = 0; g < lanes; ++g) {
        uint64_t a1 = m1[g], a2 = m2[g], sk = s[g];
        for (uint64_t k = 0; k < blocks; ++k) {
            if (P->mode == 0) sk = (uint64_t)((u128)P->a * sk % P->q);
            a1 = (uint64_t)(((u128)a1 + sk) % P->p1);
            a2 = (uint64_t)(((u128)a2 + sk) % P->p2);
            uint64_t c1 = powmod(a1, P->e, P->p1), c2 = powmod(a2, P->e, P->p2);
            uint64_t d = (c1 + P->p1 - c2 % P->p1) % P->p1;
            uint64_t c = (uint64_t)((u128)d * P->p2inv % P->p1) * P->p2 + c2;
            if (raw) raw[k * out_stride + g] = c;
            if (f64) {
                double r = (double)c / nf;
                f64[k * out_stride + g] = r < 1.0 ? r : 0x1.fffffffffffffp-1;
            }
        }
        m1[g] = a1; m2[g] = a2; s[g] = sk;
    }
}

/* Segmented sieve: primality of odd numbers in [lo, hi) (hi <= 2^33), one
 * segment of SEG odd numbers at a time, bytes m[i] <-> lo_odd + 2i. */
#define SEG (1u << 21)

typedef struct {
    uint32_t* primes; /* odd base primes <= sqrt(hi) */
    uint64_t n;
} base_primes;

static base_primes make_base(uint64_t hi) {
    uint64_t lim = (uint64_t)sqrt((double)hi) + 2;
    uint8_t* c = (uint8_t*)calloc(lim + 1, 1);
    base_primes b;
    b.primes = (uint32_t*)malloc(sizeof(uint32_t) * (lim / 2 + 8));
    b.n = 0;
    for (uint64_t p = 3; p <= lim; p += 2) {
        if (c[p]) continue;
        b.primes[b.n++] = (uint32_t)p;
        for (uint64_t j = p * p; j <= lim; j += 2 * p) c[j] = 1;
    }
    free(c);
    return b;
}

static void sieve_segment(const base_primes* b, uint64_t seg_lo, uint64_t count, uint8_t* m) {
    /* seg_lo odd; marks m[i] = 1 iff seg_lo + 2i is prime */
    memset(m, 1, count);
    uint64_t seg_hi = seg_lo + 2 * count;
    for (uint64_t k = 0; k < b->n; ++k) {
        uint64_t p = b->primes[k];
        if (p * p >= seg_hi) break;
        uint64_t start = p * p;
        if (start < seg_lo) start = (seg_lo + p - 1) / p * p;
        if (!(start & 1)) start += p;
        for (uint64_t j = (start - seg_lo) / 2; j < count; j += p) m[j] = 0;
    }
    if (seg_lo == 1 && count) m[0] = 0;
}

/* Safe primes in [lo, hi) with 11 <= lo, hi <= 2^32, ascending into out.
 * Returns the count (writes at most cap).  *n_primes = primes in [lo, hi). */
uint64_t oracle_census(uint64_t lo, uint64_t hi, uint32_t* out, uint64_t cap, uint64_t* n_primes) {
    base_primes b = make_base(hi);
    uint8_t* pm = (uint8_t*)malloc(SEG);
    uint8_t* qm = (uint8_t*)malloc(SEG / 2 + 2);
    uint64_t np = 0, ns = 0;
    for (uint64_t base = lo | 1; base < hi; base += 2ull * SEG) {
        uint64_t cnt = (hi - base + 1) / 2;
        if (cnt > SEG) cnt = SEG;
        sieve_segment(&b, base, cnt, pm);
        /* q = (p-1)/2 for p in [base, base+2cnt): q in [(base-1)/2, ...), odd q only */
        uint64_t qlo = ((base - 1) / 2) | 1, qcnt = cnt / 2 + 2;
        sieve_segment(&b, qlo, qcnt, qm);
        for (uint64_t i = 0; i < cnt; ++i) {
            if (!pm[i]) continue;
            ++np;
            uint64_t p = base + 2 * i, q = (p - 1) / 2;
            if (!(q & 1)) continue;
            if (qm[(q - qlo) / 2]) {
                if (ns < cap) out[ns] = (uint32_t)p;
                ++ns;
            }
        }
    }
    free(pm);
    free(qm);
    free(b.primes);
    if (n_primes) *n_primes = np;
    return ns;
}

static int64_t find_pair_sorted(uint64_t p1, const uint32_t* sp, uint64_t n_sp, uint64_t q, uint64_t tol) {
    uint64_t target = q / p1, lo = 0, hi = n_sp;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (sp[mid] <= target) lo = mid + 1; else hi = mid;
    }
    int64_t L = (int64_t)lo - 1;
    uint64_t H = lo;
    for (;;) {
        int lo_ok = 0, hi_ok = 0;
        uint64_t cl = 0, ch = 0;
        if (L >= 0) {
            cl = sp[L];
            u128 pr = (u128)p1 * cl;
            u128 d = pr >= q ? pr - q : q - pr;
            lo_ok = cl > (1ull << 31) && d <= tol;
        }
        if (H < n_sp) {
            ch = sp[H];
            u128 pr = (u128)p1 * ch;
            u128 d = pr >= q ? pr - q : q - pr;
            hi_ok = ch > (1ull << 31) && d <= tol;
        }
        if (!lo_ok && !hi_ok) return -1;
        uint64_t c;
        if (lo_ok && (!hi_ok || target - cl <= ch - target)) { c = cl; --L; }
        else { c = ch; ++H; }
        if (c != p1) return (int64_t)c;
    }
}

/* Packed row written by oracle_derive (matches tests/golden derive_all layout). */
typedef struct {
    uint32_t p1, p2, a, p2inv;
    uint64_t n, b;
} oracle_tuple;

/* derive_stream_params(StreamKey(seed, first+j), e) for j < count; sp = sorted
 * safe primes of [2^31, 2^32), the p1 table is its first k_p1 entries.
 * steps[j] = ordinal advance, or 256 for DerivationExhausted. */
void oracle_derive(uint64_t seed_mod_S, uint64_t first, uint64_t count, const uint32_t* sp,
                   uint64_t n_sp, const uint32_t* mult, uint64_t n_a, uint64_t q, uint64_t tol,
                   oracle_tuple* out, uint32_t* steps) {
    const uint64_t K1 = 1291831, K2 = 1768937, SIG = 35705744587ull;
    const uint64_t S = K1 * K2 * n_a;
    for (uint64_t j = 0; j < count; ++j) {
        uint64_t id = first + j;
        uint64_t x = (uint64_t)(((u128)seed_mod_S + (u128)(id % S) * (SIG % S)) % S);
        uint64_t beta = powmod(x, 7, S);
        uint64_t ordinal = beta % K1;
        uint32_t a = mult[(beta / (K1 * K2)) % n_a];
        uint32_t st = 256;
        memset(&out[j], 0, sizeof(oracle_tuple));
        for (uint32_t step = 0; step < 256; ++step) {
            uint64_t p1 = sp[(ordinal + step) % K1];
            int64_t p2 = find_pair_sorted(p1, sp, n_sp, q, tol);
            if (p2 < 0) continue;
            uint64_t n = p1 * (uint64_t)p2;
            out[j].p1 = (uint32_t)p1;
            out[j].p2 = (uint32_t)p2;
            out[j].a = a;
            out[j].p2inv = (uint32_t)powmod((uint64_t)p2 % p1, p1 - 2, p1);
            out[j].n = n;
            out[j].b = (uint64_t)((u128)(q % n) * (((q - 1) / 2) % n) % n);
            st = step;
            break;
        }
        steps[j] = st;
    }
}
