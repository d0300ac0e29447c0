/*
 * rsarand_b200.h — C ABI of the B200 (sm_100a) RSA-exponentiation PRNG hot path.
 *
 * The reference (arXiv 1811.11629, package `rsarand`) has no FFI layer: its
 * drop-in surface is the Python API of vecgen / rsacore / paramfactory.  Each
 * entry point below replaces one reference function (or a fused group of
 * them); the citation names the reference file:line it stands in for, relative
 * to /root/reference/pkg/src/rsarand/.
 *
 * Conventions (all entry points):
 *   - Plain pointers to caller-owned DEVICE buffers; the library never
 *     allocates device memory and keeps no mutable global state.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     Every call is asynchronous on that stream; results are valid after the
 *     caller synchronises it.
 *   - Return value: 0 on success, a negative RSA_E* code otherwise.  Argument
 *     errors are detected before any launch, mirroring the reference, which
 *     raises before any arithmetic (rsacore.py:117-181, vecgen.py:47-51).
 *   - Functions are reentrant; distinct states may be advanced concurrently
 *     on distinct streams.  One state must not be advanced concurrently
 *     (SPEC.md:304, 421-423).
 */
#ifndef RSARAND_B200_H
#define RSARAND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSA_ABI_VERSION 4

/* status codes */
#define RSA_OK 0
#define RSA_EINVAL (-1)        /* bad argument (null pointer, zero size, ...) */
#define RSA_ECUDA (-2)         /* CUDA launch / runtime error                */
#define RSA_EPARAMS (-3)       /* instance table fails a kernel precondition */
#define RSA_ECAPACITY (-4)     /* output capacity too small                  */
#define RSA_EALIGN (-5)        /* buffer misaligned for the requested layout */

/* skip modes (rsacore.py:24-27) */
#define RSA_SKIP_LCG 0
#define RSA_SKIP_UNIT 1
#define RSA_SKIP_CONST 2

/* rsa_instance.flags */
#define RSA_FLAG_FAST 1u   /* q = 2^63-25, p1,p2 in (2^31,2^32), lcg mode: fast kernels */
#define RSA_FLAG_FIXED 2u  /* unit / const skip: per-lane skip register is constant     */
#define RSA_FLAG_GENERAL_PATH 4u /* rsa_fill hint: force the general kernel (cross-checks) */
#define RSA_FLAG_ONE_LANE 8u     /* rsa_fill hint: one lane per thread (tuning / A-B)       */
#define RSA_FLAG_INTERLEAVE 16u  /* rsa_fill: instances round-robin, draw t of i at out[t*n_inst+i] */
#define RSA_FLAG_LOW32 32u       /* rsa_fill: f64_out = (c mod 2^32) / 2^32 instead of the float map */

/*
 * Per-instance constants, 128 bytes, one per generator instance.  The first
 * block holds the reference GeneratorParams fields (rsacore.py:56-76; skip
 * constants skipgen.py:54-82); the rest are Montgomery / float constants the
 * kernels need.  R = 2^32.  Built on the host for single streams
 * (rsacore.make_params) or on the device by rsa_setup_instances.
 */
typedef struct rsa_instance {
    uint32_t p1, p2;          /*   0  safe primes                                */
    uint32_t p1_inv, p2_inv;  /*   8  p^-1 mod 2^32 (Montgomery)                 */
    uint32_t a, e;            /*  16  skip multiplier; exponent                  */
    uint32_t k1, k2;          /*  24  R^(2e) mod p: undoes the R^-1 message scale*/
    uint32_t r2_1, r2_2;      /*  32  R^2 mod p                                  */
    uint32_t garner, p2inv;   /*  40  p2inv*R mod p1 ; p2^-1 mod p1 (reference)  */
    uint32_t q1, q2;          /*  48  Schrage constants q/a, q mod a (skipgen.py:82) */
    uint32_t flags, skip_mode;/*  56  RSA_FLAG_* ; RSA_SKIP_*                    */
    uint64_t n;               /*  64  p1*p2                                      */
    uint64_t q;               /*  72  skip modulus                               */
    uint64_t b;               /*  80  q(q-1)/2 mod n (rsacore.py:102)            */
    double n_float;           /*  88  float(n) (rsacore.py:104)                  */
    double n_recip;           /*  96  RN(1/n_float)                              */
    uint64_t skip_const;      /* 104  const-mode skip value (rsacore.py:91)      */
    uint64_t reserved1;       /* 112  0                                          */
    uint64_t reserved2;       /* 120  0                                          */
} rsa_instance;

/* ---------------------------------------------------------------------------
 * K1: bulk fill.  Replaces vecgen.next_block_raw + floats_from_raw
 * (vecgen.py:87-107), and with n_inst > 1 a batch of init_vector'd streams.
 *
 * Lanes: instance i owns lanes [i*mv, (i+1)*mv); state arrays m1, m2, s hold
 * n_inst*mv entries (uint64, values < p1, < p2, < q — the reference layout,
 * vecgen.py:31-41).  Each call advances every lane `blocks` steps in place, so
 * chained calls equal one long call.  Block k lane g of instance i is written
 * to out[i*inst_stride + k*mv + g] (stream order block-major, lane-minor,
 * vecgen.py:115-139) for raw_out (uint64 ciphertexts c in [0,n)) and/or
 * f64_out (r = min(fl(c)/fl(n), 1-2^-53), vecgen.py:103-107).  Either output
 * pointer may be NULL; both NULL just advances the state.
 * `e` and `flags` are the exponent and RSA_FLAG_* bits common to all n_inst
 * instances (the caller built the table and promises homogeneity): with
 * RSA_FLAG_FAST an exponent-specialised kernel runs (e in {3,5,9,17,65537}
 * fully unrolled, any other e through the runtime chain); otherwise the
 * general kernel (test-mode sizes, any prime q, unit/const skips) runs.
 * RSA_FLAG_GENERAL_PATH forces the general kernel (independent cross-check);
 * RSA_FLAG_ONE_LANE forces one lane per thread.
 * RSA_FLAG_INTERLEAVE (fast path): the n_inst streams are written round-robin,
 * draw t = k*mv + g of instance i at out[t*n_inst + i] (inst_stride unused) —
 * the interleaved multi-stream source of stats.BitSource (stats.py:118-136).
 * RSA_FLAG_LOW32 (fast path): f64_out holds (c mod 2^32) * 2^-32, the
 * BitSource "raw_low_bits" view, instead of the float map.
 * The general path returns RSA_EPARAMS for either layout flag.
 * --------------------------------------------------------------------------- */
int rsa_fill(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
             uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
             uint64_t* raw_out, double* f64_out, uint64_t inst_stride,
             void* stream);

/* One skip step for a batch of registers: out[j] = a * s[j] mod q
 * (skipgen.next_skip_array, skipgen.py:108-116).  s may alias out. */
int rsa_skip_array(const uint64_t* s, uint64_t count, uint64_t a, uint64_t q, uint64_t* out,
                   void* stream);

/* K1s: the same fill with every lane split into segments of draws, for lane
 * counts too small to fill the GPU (the scalar stream, Mv = 64).  The skip is
 * jumped ahead exactly (s0 * (a^L)^j mod q) and the message prefix sums of the
 * segments are scanned, so results and final state are bit-identical to
 * rsa_fill.  Requires RSA_FLAG_FAST and at least one output.
 * rsa_fill_segments(lanes, blocks) = segments per lane it will use (1 = no
 * benefit: call rsa_fill); scratch >= rsa_fill_segmented_scratch_bytes. */
uint64_t rsa_fill_segments(uint64_t lanes, uint64_t blocks);
uint64_t rsa_fill_segmented_scratch_bytes(uint64_t lanes, uint64_t blocks);
int rsa_fill_segmented(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
                       uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
                       uint64_t* raw_out, double* f64_out, uint64_t inst_stride,
                       void* scratch, uint64_t scratch_bytes, void* stream);

/* Scalar look-ahead (rsacore.next_raw / next_f64, rsacore.py:213-233): the
 * next `count` draws (a multiple of 32, <= 32768) of the one-lane stream whose
 * state is (m1, m2, s), with the state after every draw, so the host can
 * serve single draws from a buffer and still expose the reference's state
 * fields after each one.  `out` (device) receives count * 32 bytes:
 * raw u64[count] | f64[count] | s u64[count] | m1 u32[count] | m2 u32[count].
 * The caller's state is not modified.  Requires RSA_FLAG_FAST. */
int rsa_scalar_lookahead(const rsa_instance* inst, uint64_t m1, uint64_t m2, uint64_t s,
                         uint32_t e, uint32_t flags, uint32_t count, void* out, void* stream);

/* floats_from_raw (vecgen.py:103-107): out[j] = min(fl(raw[j])/fl(n), 1-2^-53). */
int rsa_floats_from_raw(const uint64_t* raw, uint64_t count, uint64_t n, double* out,
                        void* stream);
/* The same map by the 4-op quotient the fused kernels use (double-double
 * reciprocal + one Markstein step): an independent cross-check of that path,
 * bit-identical to rsa_floats_from_raw. */
int rsa_floats_from_raw_dd(const uint64_t* raw, uint64_t count, uint64_t n, double* out,
                           void* stream);

/* Lane initialisation, vecgen.init_vector (vecgen.py:44-69) for every instance.
 * lcg mode: s[i*mv+g] = s0 * a^(g*floor((q-1)/mv)) mod q
 *           (skipgen.lane_offset_seeds, skipgen.py:124-138), m1 = m0 mod p1,
 *           m2 = m0 mod p2 for all lanes.  s0 must already be in [1, q).
 * unit/const mode (RSA_FLAG_FIXED): lane g holds message m0 + (g+1-mv)*v mod n
 *           and skip mv*v mod n, v = 1 (unit) or skip_const (vecgen.py:61-68).
 * m0 = m0_hi*2^64 + m0_lo (< 2^128; the caller reduces larger seeds mod n). */
int rsa_init_lanes(const rsa_instance* inst, uint32_t n_inst, uint32_t mv,
                   uint64_t m0_lo, uint64_t m0_hi, uint64_t s0,
                   uint64_t* m1, uint64_t* m2, uint64_t* s, void* stream);

/* ---------------------------------------------------------------------------
 * K2: fused consumer (no reference equivalent).
 * Each instance is one Mv=1 stream advanced `draws` steps in place; the
 * doubles r are reduced in registers, never written:
 *   stats[i] = {S1=sum r, S2=sum r^2, L=sum_{k<N-1} r_k r_{k+1}, r_first, r_last,
 *               XY=sum_k r_k^(i) r_k^(i^1)  (only meaningful for even i)}
 *   hist[i*64 + b] = #{k : floor(64 r_k) = b}
 * n_inst must be even (pairs (2j, 2j+1) for the inter-stream correlation) and
 * every instance must carry RSA_FLAG_FAST with exponent e.
 * --------------------------------------------------------------------------- */
typedef struct rsa_fused_stat {
    double s1, s2, lag, first, last, xy;
} rsa_fused_stat;

int rsa_fused_stats(const rsa_instance* inst, uint32_t n_inst, uint64_t draws, uint32_t e,
                    uint64_t* m1, uint64_t* m2, uint64_t* s,
                    rsa_fused_stat* stats, uint32_t* hist, void* stream);

/* Deterministic pooled reduction of rsa_fused_stats output:
 * pooled[0..6] = {sum S1, sum S2, sum XY (even i), sum S1 even, sum S1 odd,
 *                 sum S2 even, sum S2 odd}; pooled_hist[64] = sum of hist rows. */
int rsa_fused_pool(const rsa_fused_stat* stats, const uint32_t* hist, uint32_t n_inst,
                   double* pooled, uint64_t* pooled_hist, void* stream);

/* ---------------------------------------------------------------------------
 * K3: safe-prime scan.  Replaces paramfactory.safe_primes_in (paramfactory.py:105-130)
 * and numtheory.is_safe_prime (numtheory.py:96-98) for [lo, hi), hi <= 2^32:
 * writes the ascending safe primes to out[0..*count) (device count).  Primality of p
 * and (p-1)/2 is exact: a shared-memory sieve by the primes 5..8191, the base-2
 * strong-probable-prime test, then a lookup in the complete table of the 2314
 * base-2 strong pseudoprimes below 2^32.
 * scratch must hold rsa_safe_prime_scan_scratch_bytes(lo, hi) bytes.
 * Returns RSA_ECAPACITY (after writing *count) when out_cap is too small.
 * --------------------------------------------------------------------------- */
uint64_t rsa_safe_prime_scan_scratch_bytes(uint64_t lo, uint64_t hi);
int rsa_safe_prime_scan(uint64_t lo, uint64_t hi, uint32_t* out, uint64_t out_cap,
                        uint64_t* count, void* scratch, uint64_t scratch_bytes,
                        void* stream);

/* The same census by the reference algorithm as BASELINE config 5 states it:
 * deterministic Miller-Rabin with bases 2, 7, 61 (exact below 4,759,123,141)
 * on every odd n in [lo, hi) and on (n-1)/2 (numtheory.py:60-98,
 * paramfactory.py:105-130; n < 10201 by trial division).  No sieve, no
 * pseudoprime table: a cross-check of rsa_safe_prime_scan and the IMAD-bound
 * yardstick it is measured against.  Same output contract as
 * rsa_safe_prime_scan; scratch >= rsa_safe_prime_scan_mr_scratch_bytes. */
uint64_t rsa_safe_prime_scan_mr_scratch_bytes(uint64_t lo, uint64_t hi);
int rsa_safe_prime_scan_mr(uint64_t lo, uint64_t hi, uint32_t* out, uint64_t out_cap,
                           uint64_t* count, void* scratch, uint64_t scratch_bytes,
                           void* stream);

/* Batched is_prime / is_safe_prime predicates (numtheory.py:81-98) for 32-bit n. */
int rsa_is_safe_prime32(const uint32_t* n, uint64_t count, uint8_t* is_prime,
                        uint8_t* is_safe, void* stream);

/* Bucket index of a sorted u32 table: index[b] = number of entries
 * < b*2^RSA_SP_INDEX_SHIFT, b = 0..2^(32-RSA_SP_INDEX_SHIFT) (RSA_SP_INDEX_LEN
 * entries).  Lets rsa_find_pair / rsa_setup_instances start their search
 * inside one 2^12-wide bucket
 * (~3 safe primes) instead of the whole table. */
#define RSA_SP_INDEX_SHIFT 12u
#define RSA_SP_INDEX_LEN ((1u << (32u - RSA_SP_INDEX_SHIFT)) + 1u)
int rsa_safe_prime_index(const uint32_t* sp, uint64_t n_sp, uint32_t* index, void* stream);

/* find_pair (paramfactory.py:195-219) for a batch of p1 values against the
 * sorted safe-prime table sp[0..n_sp): p2 = nearest table entry to floor(q/p1),
 * ties to the smaller, p2 != p1, 2^31 < p2 < 2^32, |p1*p2 - q| <= tol.
 * sp_index = rsa_safe_prime_index of sp, or NULL (plain binary search).
 * status[j] = 0 found, 1 NotFound. */
int rsa_find_pair(const uint32_t* p1, uint64_t count, uint64_t q, uint64_t tol,
                  const uint32_t* sp, uint64_t n_sp, const uint32_t* sp_index,
                  uint32_t* p2, int32_t* status, void* stream);

/* ---------------------------------------------------------------------------
 * K4: instance setup.  Replaces paramfactory.derive_stream_params +
 * stream_indices + rsacore.make_params (paramfactory.py:242-278,
 * rsacore.py:89-107) for ids first_id .. first_id+count-1:
 *   beta = ((seed_mod_S + id*SIGMA) mod S)^EPSILON mod S, S = K_P1*K_P2*n_a
 *   ordinal = beta mod K_P1, a = mult[beta/(K_P1*K_P2) mod n_a] (or `multiplier`)
 *   p1 = p1tab[(ordinal+step) mod K_P1], step = 0..255, first with a find_pair partner.
 * seed_mod_S = master_seed mod S (reduced by the caller, exact for any seed size).
 * sp = sorted safe primes of [2^31, 2^32) (sp_index: its rsa_safe_prime_index, or
 * NULL); p1tab = its prefix inside the p1 window.
 * Steps start at cfg->start_step (0 for the reference order; a host caller
 * that rejects a pair for a host-only reason resumes after it).
 * status[j] = 0 ok, 2 DerivationExhausted; step_out[j] = ordinal advance (may be NULL).
 * --------------------------------------------------------------------------- */
typedef struct rsa_setup_config {
    uint64_t seed_mod_S;    /* master_seed mod S                         */
    uint64_t first_id;      /* stream id of instance 0                   */
    uint64_t sigma;         /* SIGMA (paramfactory.py:47)                */
    uint64_t k_p1, k_p2;    /* index radices (paramfactory.py:41-42)     */
    uint64_t q;             /* skip modulus                              */
    uint64_t tol;           /* floor(1e-6*q) (exact integer tolerance)   */
    uint32_t epsilon;       /* EPSILON (paramfactory.py:48)              */
    uint32_t e;             /* exponent (validated by the caller)        */
    uint32_t n_mult;        /* multiplier table size n_a                 */
    uint32_t multiplier;    /* 0 = table choice, else override           */
    uint32_t max_steps;     /* 256 (paramfactory.py:270)                 */
    uint32_t start_step;    /* first ordinal advance to try (0)          */
} rsa_setup_config;

int rsa_setup_instances(const rsa_setup_config* cfg, uint64_t count,
                        const uint32_t* mult_table, const uint32_t* sp, uint64_t n_sp,
                        const uint32_t* sp_index, const uint32_t* p1tab, uint64_t n_p1tab,
                        rsa_instance* out, int32_t* status, uint32_t* step_out,
                        void* stream);

/* ---------------------------------------------------------------------------
 * Battery counting (reference stats.py:233-466): integer
 * cell counts of one chi-square test over a device buffer of variates in
 * [0, 1) (a BitSource chunk), accumulated (+=) into counts.  The statistic is
 * formed by the caller from the counts exactly as the reference does.
 *   RSA_BT_HIST        n values, p1 = bins            (frequency)
 *   RSA_BT_SERIAL      n d-tuples, p1 = d, p2 = axis  (serial)
 *   RSA_BT_POKER       n 5-card hands                 (poker, counts[5])
 *   RSA_BT_MAX_OF_T    n t-tuples, p1 = t, p2 = bins  (max-of-t)
 *   RSA_BT_PERMUTATION n t-tuples, p1 = t <= 10; *flag = 1 on a tie
 *   RSA_BT_COLLISION   n trials of 2^14 balls (x20 variates when p1 = 1),
 *                      counts[collisions] += 1        (collision)
 * --------------------------------------------------------------------------- */
#define RSA_BT_HIST 1
#define RSA_BT_SERIAL 2
#define RSA_BT_POKER 3
#define RSA_BT_MAX_OF_T 4
#define RSA_BT_PERMUTATION 5
#define RSA_BT_COLLISION 6

int rsa_battery_count(int test, const double* v, uint64_t n, uint32_t p1, uint32_t p2,
                      unsigned long long* counts, int* flag, void* stream);

/* ---------------------------------------------------------------------------
 * Fused battery counting (consumers fed in registers like
 * K2).  The variates of a BitSource over n_inst interleaved streams
 * (stats.BitSource, stats.py:118-136: round-robin by draw, stream 0 first —
 * the RSA_FLAG_INTERLEAVE order) are generated for `blocks` whole blocks of
 * every stream and counted without ever being written: each CTA holds a tile
 * of RSA_BT_TILE consecutive positions in shared memory, counts the tuples
 * that lie inside it, and hands the variates of the (at most one) tuple
 * straddling each tile boundary to a slot; rsa_battery_stitch counts those.
 * Selector: RSA_FLAG_LOW32 ? low 32 bits / 2^32 (raw_low_bits) : the float
 * map (float_leading).  Lane state advances exactly as rsa_fill would.
 * Requires n_inst | 256 and (mv * n_inst) % RSA_BT_TILE == 0.
 *
 * spec->pos0 is the test-relative position of the first generated variate;
 * tuples start at test positions 0, d, 2d, ...  Tile t (t = 0 .. blocks *
 * mv * n_inst / RSA_BT_TILE - 1, in stream order) covers test positions
 * pos0 + t*RSA_BT_TILE ...; boundary b (b = 0 .. tiles) sits at pos0 +
 * b*RSA_BT_TILE and owns slots[(spec->seg0 + b) * d .. + d): the part of the
 * straddling tuple before the boundary at [0, phase), after it at [phase, d),
 * phase = position mod d.  The caller fills the parts of boundaries 0 and
 * `tiles` that lie outside the launch (materialised head / tail variates).
 *
 * RSA_BT_COLLISION (d = 1: urn = cell of one variate among 2^20; d = 20: urn
 * = the bits (u > 1/2) of 20 consecutive variates; stats.py collision_test):
 * ball b = test position / d belongs to trial b >> 14; each ball sets its
 * urn's bit in the trial's 2^20-bit bitmap (spec->aux, uint32[trials][2^15],
 * zeroed by the caller) and a ball whose bit was already set adds 1 to
 * counts[trial]; rsa_battery_collision_hist turns those into the test's
 * histogram.  Collision counts are order-independent.
 *
 * RSA_BT_GAPS: runs of (u > 1/2) / (u <= 1/2) (stats.py gaps_test): runs that
 * start and end inside one tile are counted (counts[min(len, 64) - 1]); every
 * tile writes records[spec->seg0 + t] for rsa_battery_gaps_stitch.
 * rsa_battery_gaps_array does the same over a device array of n variates
 * (tiles of RSA_BT_TILE, the last one short).
 * --------------------------------------------------------------------------- */
#define RSA_BT_GAPS 7
#define RSA_BT_TILE 256

typedef struct rsa_battery_spec {
    int32_t test;      /* RSA_BT_HIST / SERIAL / POKER / MAX_OF_T / PERMUTATION / GAPS */
    uint32_t d;        /* variates per tuple: 1 (HIST, GAPS), d, 5, t, t           */
    uint32_t p1, p2;   /* as rsa_battery_count (bins / axis / t)                   */
    uint64_t pos0;     /* test-relative position of the first variate              */
    uint64_t seg0;     /* first boundary slot / gap record of this launch          */
    uint64_t aux;      /* RSA_BT_COLLISION: device address of the trial bitmaps   */
} rsa_battery_spec;

typedef struct rsa_gap_record {
    uint32_t head;     /* values before the tile's first internal flip (or len)    */
    uint32_t tail;     /* values from its last internal flip to the end (or len)   */
    uint32_t len;      /* values in the tile                                        */
    uint32_t bits;     /* 1: has an internal flip, 2: first value > 1/2, 4: last   */
} rsa_gap_record;

int rsa_battery_fused(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
                      uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
                      const rsa_battery_spec* spec, unsigned long long* counts, int* flag,
                      double* slots, rsa_gap_record* records, void* stream);
int rsa_battery_gaps_array(const double* v, uint64_t n, const rsa_battery_spec* spec,
                           unsigned long long* counts, rsa_gap_record* records, void* stream);
/* Tuples of boundary slots [first, first + n) whose phase (position mod d,
 * position = pos0 + (b - seg0) * RSA_BT_TILE for slot b) is nonzero. */
int rsa_battery_stitch(const rsa_battery_spec* spec, const double* slots, uint64_t first, uint64_t n,
                       unsigned long long* counts, int* flag, void* stream);
/* RSA_BT_COLLISION over a device array of n variates holding whole balls
 * (spec->pos0 = test position of v[0], a multiple of spec->d). */
int rsa_battery_collision_array(const double* v, uint64_t n, const rsa_battery_spec* spec,
                                unsigned long long* trial_counts, void* stream);
/* counts[trial_counts[t]] += 1 for t < trials (the collision histogram). */
int rsa_battery_collision_hist(const unsigned long long* trial_counts, uint64_t trials,
                               unsigned long long* counts, void* stream);
/* Runs that cross tile boundaries, from n_rec records in stream order (the
 * test's open final run is not counted). */
int rsa_battery_gaps_stitch(const rsa_gap_record* records, uint64_t n_rec,
                            unsigned long long* counts, void* stream);
/* Fourier cells: the real and imaginary parts of n complex coefficients
 * (interleaved re, im doubles) binned against 63 sorted interior edges:
 * counts[cell] (real) and counts[64 + cell] (imag), cell = #edges < value
 * (numpy searchsorted side='left'). */
int rsa_battery_fourier_bin(const double* coeff, uint64_t n, const double* edges,
                            unsigned long long* counts, void* stream);
/* *out = sum over i < n of (counts[i] - e)^2, each term and every addition
 * rounded exactly as numpy's np.square(counts - e).sum() (pairwise summation,
 * blocks of 128 with eight accumulators): the equiprobable tests' statistic
 * without moving the count vector to the host.  Scratch: device memory of
 * rsa_battery_chi2_scratch_bytes(n) bytes (0 when n is out of range). */
uint64_t rsa_battery_chi2_scratch_bytes(uint64_t n);
int rsa_battery_chi2_sum(const long long* counts, uint64_t n, double e, double* out, void* scratch,
                         uint64_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Roofline probe: a dependency-free stream of Montgomery triples
 * (IMAD.WIDE.U32, IMAD, IMAD.WIDE.U32) over `grid` CTAs of 256 threads,
 * `iters` iterations; returns through *ops the IMAD-class instruction count
 * the launch issues (3 per triple).  Time it with events on `stream`.
 * --------------------------------------------------------------------------- */
int rsa_probe_imad(uint32_t grid, uint32_t iters, uint32_t* sink, double* ops, void* stream);

/* Library identity: ABI version, and the SM arch the cubin was built for (100). */
int rsa_abi_version(void);
int rsa_built_arch(void);
/* Last CUDA error string seen by this thread (static storage). */
const char* rsa_last_error(void);
/* Kernels this library has launched in this process (all entry points; a
 * launch recorded into a CUDA graph counts once, at capture). */
uint64_t rsa_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RSARAND_B200_H */
