// setup.cu — K4 instance setup and find_pair.
//
// Replaces paramfactory.stream_indices / derive_stream_params / find_pair
// (paramfactory.py:195-278) and rsacore.make_params (rsacore.py:89-107) for a
// contiguous range of stream ids: one thread per id.  The reference's lazily
// sieved p1 table (paramfactory.py:160-189) is the prefix of the device
// safe-prime list produced by K3, and find_pair's outward scan over 11-mod-12
// positions becomes a binary search plus an outward merge over that sorted
// list (same order: nearest to floor(q/p1), ties to the smaller, p1 skipped,
// stop when both sides leave the tolerance window).
#include "common.cuh"
#include "modarith.cuh"

namespace rsa {

// |p1*c - q| <= tol and 2^31 < c < 2^32 (paramfactory.py:209-210; rsacore.py:180
// compares against the float 1e-6*q, i.e. the integer floor of it).
RSA_DEV bool pair_ok(uint32_t p1, uint32_t c, uint64_t q, uint64_t tol) {
    if (c <= 0x80000000u) return false;
    uint64_t prod = (uint64_t)p1 * c;
    uint64_t d = prod >= q ? prod - q : q - prod;
    return d <= tol;
}

// 0 = found (*p2 set), 1 = NotFound.  idx (optional): rsa_safe_prime_index of
// sp, narrowing the search to the 2^RSA_SP_INDEX_SHIFT-wide bucket of the target.
RSA_DEV int find_partner(uint32_t p1, uint64_t q, uint64_t tol, const uint32_t* __restrict__ sp,
                         uint64_t n_sp, const uint32_t* __restrict__ idx, uint32_t* p2) {
    uint64_t rr, target = p1 > (1u << 14) ? div_small_q(q, p1, &rr) : q / p1;  // quotient < 2^50
    uint64_t lo = 0, hi = n_sp;  // first index with sp[idx] > target
    if (idx) {
        if (target >= 0xFFFFFFFFull) {
            lo = hi = n_sp;
        } else {  // entries with value >> SHIFT == b lie in [idx[b], idx[b+1])
            const uint32_t b = (uint32_t)(target >> RSA_SP_INDEX_SHIFT);
            lo = __ldg(idx + b);
            hi = __ldg(idx + b + 1);
        }
    }
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(sp + mid) <= target) lo = mid + 1;
        else hi = mid;
    }
    int64_t L = (int64_t)lo - 1;
    uint64_t H = lo;
    for (;;) {
        uint32_t cl = L >= 0 ? __ldg(sp + L) : 0u;
        uint32_t ch = H < n_sp ? __ldg(sp + H) : 0u;
        bool lo_ok = L >= 0 && pair_ok(p1, cl, q, tol);
        bool hi_ok = H < n_sp && pair_ok(p1, ch, q, tol);
        if (!lo_ok && !hi_ok) return 1;
        uint32_t c;
        if (lo_ok && (!hi_ok || target - cl <= (uint64_t)ch - target)) { c = cl; --L; }
        else { c = ch; ++H; }
        if (c != p1) { *p2 = c; return 0; }
    }
}

// Montgomery / float constants of one instance (the host twin is
// paper_1811_11629_b200/rsacore.py:_pack_instance).
RSA_DEV void build_instance(rsa_instance* o, uint32_t p1, uint32_t p2, uint32_t a, uint32_t e,
                            uint64_t q) {
    uint64_t n = (uint64_t)p1 * p2;
    uint32_t i1 = inv32(p1), i2 = inv32(p2);
    uint32_t R1 = (uint32_t)mod_small_q(1ull << 32, p1), R2 = (uint32_t)mod_small_q(1ull << 32, p2);
    uint32_t r21 = (uint32_t)mod_small_q((uint64_t)R1 * R1, p1), r22 = (uint32_t)mod_small_q((uint64_t)R2 * R2, p2);
    // R^(2e) mod p: r2 is R in Montgomery form; power it, then leave the domain
    uint32_t k1 = mont_redc(mont_pow_m(r21, 2 * e, R1, p1, i1), p1, i1);
    uint32_t k2 = mont_redc(mont_pow_m(r22, 2 * e, R2, p2, i2), p2, i2);
    // p2^-1 mod p1 by Fermat (p1 prime)
    uint32_t p2m = mont_mul((uint32_t)mod_small_q(p2, p1), r21, p1, i1);
    uint32_t p2inv = mont_redc(mont_pow_m(p2m, p1 - 2, R1, p1, i1), p1, i1);
    rsa_instance v;
    v.p1 = p1; v.p2 = p2; v.p1_inv = i1; v.p2_inv = i2;
    v.a = a; v.e = e; v.k1 = k1; v.k2 = k2; v.r2_1 = r21; v.r2_2 = r22;
    v.garner = mont_mul(p2inv, r21, p1, i1);
    v.p2inv = p2inv;
    uint64_t qr, qa = a > (1u << 14) ? div_small_q(q, a, &qr) : (qr = q % a, q / a);  // quotient < 2^50
    v.q1 = (uint32_t)qa;
    v.q2 = (uint32_t)qr;
    bool fast = q == Q63 && p1 > 0x80000000u && p2 > 0x80000000u;
    v.flags = fast ? RSA_FLAG_FAST : 0u;
    v.skip_mode = RSA_SKIP_LCG;
    v.n = n; v.q = q;
    // q(q-1)/2 mod n, q odd; n > 2^62 here, so both factors reduce by at most a subtraction
    const uint64_t h = (q - 1) >> 1;
    const uint64_t qm = q >= n ? (q - n >= n ? q % n : q - n) : q, hm = h >= n ? h % n : h;
    v.b = n >= (1ull << 32) ? mulmod64_fp(qm, hm, n) : mulmod64(qm, hm, n);
    v.n_float = __ull2double_rn(n);
    v.n_recip = __drcp_rn(v.n_float);
    v.skip_const = 0; v.reserved1 = 0; v.reserved2 = 0;
    *o = v;
}

// x*y mod m for x, y < m < 2^50: the quotient from an FP64 estimate is off by
// at most one (relative error <= 3 * 2^-53 on a quotient < 2^50), and the
// remainder is formed exactly in wrapping 64-bit arithmetic.
RSA_DEV uint64_t mulmod50(uint64_t x, uint64_t y, uint64_t m, double minv) {
    const uint64_t qd = (uint64_t)(__dmul_rn(__dmul_rn((double)x, (double)y), minv));
    int64_t r = (int64_t)(x * y - qd * m);
    if (r < 0) r += (int64_t)m;
    else if (r >= (int64_t)m) r -= (int64_t)m;
    return (uint64_t)r;
}

RSA_DEV uint64_t powmod50(uint64_t b, uint32_t e, uint64_t m, double minv) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r = mulmod50(r, b, m, minv);
        e >>= 1;
        if (e) b = mulmod50(b, b, m, minv);
    }
    return r;
}

__global__ void k_sp_index(const uint32_t* __restrict__ sp, uint64_t n_sp, uint32_t* __restrict__ index) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= RSA_SP_INDEX_LEN) return;
    const uint64_t key = (uint64_t)b << RSA_SP_INDEX_SHIFT;  // lower_bound(key)
    uint64_t lo = 0, hi = n_sp;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)sp[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    index[b] = (uint32_t)lo;
}

// One thread per stream id.  The 128-byte records are built in shared memory
// and written out by the whole CTA as contiguous 16-byte words (a thread
// storing its own record directly would scatter every warp store over 32
// lines).  The launch constants first_id, seed and sigma arrive reduced mod S
// (rsa_setup_instances does it once on the host side).
constexpr int SETUP_BLOCK = 128;

__global__ void __launch_bounds__(SETUP_BLOCK)
k_setup(rsa_setup_config cfg, uint64_t count, const uint32_t* __restrict__ mult,
        const uint32_t* __restrict__ sp, uint64_t n_sp, const uint32_t* __restrict__ sp_index,
        const uint32_t* __restrict__ p1tab, uint64_t n_p1tab,
        rsa_instance* __restrict__ out, int32_t* __restrict__ status,
        uint32_t* __restrict__ step_out) {
    __shared__ __align__(16) rsa_instance stage[SETUP_BLOCK];
    __shared__ uint8_t found[SETUP_BLOCK];
    const uint64_t j0 = (uint64_t)blockIdx.x * SETUP_BLOCK;
    const uint64_t j = j0 + threadIdx.x;
    found[threadIdx.x] = 0;
    if (j < count) {
        // beta = (t + id*SIGMA mod S)^EPSILON mod S   (paramfactory.py:242-250)
        const uint64_t S = cfg.k_p1 * cfg.k_p2 * cfg.n_mult;
        const bool small = S < (1ull << 50);  // the published radices: S = K_P1*K_P2*n_a ~ 2^45
        uint64_t beta;
        if (small) {
            const double Sinv = __drcp_rn((double)S);
            uint64_t id_mod = cfg.first_id + (j < S ? j : mod_small_q(j, S));
            id_mod = id_mod >= S ? id_mod - S : id_mod;
            uint64_t x = cfg.seed_mod_S + mulmod50(id_mod, cfg.sigma, S, Sinv);
            x = x >= S ? x - S : x;
            beta = powmod50(x, cfg.epsilon, S, Sinv);
        } else {
            uint64_t id_mod = (uint64_t)(((unsigned __int128)cfg.first_id + j) % S);
            uint64_t x = (uint64_t)(((unsigned __int128)cfg.seed_mod_S + mulmod64(id_mod, cfg.sigma, S)) % S);
            beta = powmod64(x, cfg.epsilon, S);
        }
        // every quotient below is small on the published radices (beta < S < 2^50)
        uint64_t ordinal = small ? mod_small_q(beta, cfg.k_p1) : beta % cfg.k_p1;
        uint64_t junk, hiq = small ? div_small_q(beta, cfg.k_p1 * cfg.k_p2, &junk) : beta / (cfg.k_p1 * cfg.k_p2);
        uint32_t a = cfg.multiplier ? cfg.multiplier : mult[small ? mod_small_q(hiq, cfg.n_mult) : hiq % cfg.n_mult];
        // bounded ordinal advance (paramfactory.py:270-278)
        uint32_t step = cfg.start_step;
        int32_t st = 2;
        for (; step < cfg.max_steps; ++step) {
            uint64_t k = ordinal + step;
            k = small ? mod_small_q(k, cfg.k_p1) : k % cfg.k_p1;
            if (k >= n_p1tab) break;
            uint32_t p1 = __ldg(p1tab + k), p2;
            if (find_partner(p1, cfg.q, cfg.tol, sp, n_sp, sp_index, &p2) == 0) {
                build_instance(&stage[threadIdx.x], p1, p2, a, cfg.e, cfg.q);
                found[threadIdx.x] = 1;
                st = 0;
                break;
            }
        }
        status[j] = st;
        if (step_out) step_out[j] = st == 0 ? step : cfg.max_steps;
    }
    __syncthreads();
    const uint64_t nrec = count - j0 < SETUP_BLOCK ? count - j0 : SETUP_BLOCK;
    const uint4* src = reinterpret_cast<const uint4*>(stage);
    uint4* dst = reinterpret_cast<uint4*>(out + j0);
    constexpr int W = sizeof(rsa_instance) / 16;
    for (uint32_t w = threadIdx.x; w < nrec * W; w += SETUP_BLOCK)
        if (found[w / W]) dst[w] = src[w];
}

__global__ void k_find_pair(const uint32_t* __restrict__ p1, uint64_t count, uint64_t q, uint64_t tol,
                            const uint32_t* __restrict__ sp, uint64_t n_sp, const uint32_t* __restrict__ sp_index,
                            uint32_t* __restrict__ p2, int32_t* __restrict__ status) {
    uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    uint32_t v = 0;
    status[j] = find_partner(p1[j], q, tol, sp, n_sp, sp_index, &v);
    p2[j] = v;
}

}  // namespace rsa

using namespace rsa;

extern "C" int rsa_safe_prime_index(const uint32_t* sp, uint64_t n_sp, uint32_t* index, void* stream) {
    if ((!sp && n_sp) || !index || n_sp >= (1ull << 32)) return RSA_EINVAL;
    k_sp_index<<<grid_for(RSA_SP_INDEX_LEN, 256), 256, 0, as_stream(stream)>>>(sp, n_sp, index);
    return launch_status("rsa_safe_prime_index");
}

extern "C" int rsa_setup_instances(const rsa_setup_config* cfg, uint64_t count,
                                   const uint32_t* mult_table, const uint32_t* sp, uint64_t n_sp,
                                   const uint32_t* sp_index, const uint32_t* p1tab, uint64_t n_p1tab,
                                   rsa_instance* out, int32_t* status, uint32_t* step_out, void* stream) {
    if (!cfg || !sp || !p1tab || !out || !status || count == 0) return RSA_EINVAL;
    if (cfg->k_p1 == 0 || cfg->k_p2 == 0 || cfg->n_mult == 0 || cfg->e == 0 || cfg->q < 3) return RSA_EINVAL;
    if (!cfg->multiplier && !mult_table) return RSA_EINVAL;
    if (!grid_fits(count, 128)) return RSA_EINVAL;
    rsa_setup_config c = *cfg;  // launch constants reduced mod S once, here
    const uint64_t S = c.k_p1 * c.k_p2 * c.n_mult;
    c.first_id %= S;
    c.seed_mod_S %= S;
    c.sigma %= S;
    k_setup<<<grid_for(count, SETUP_BLOCK), SETUP_BLOCK, 0, as_stream(stream)>>>(c, count, mult_table, sp, n_sp,
                                                                              sp_index, p1tab, n_p1tab, out,
                                                                              status, step_out);
    return launch_status("rsa_setup_instances");
}

extern "C" int rsa_find_pair(const uint32_t* p1, uint64_t count, uint64_t q, uint64_t tol,
                             const uint32_t* sp, uint64_t n_sp, const uint32_t* sp_index, uint32_t* p2,
                             int32_t* status, void* stream) {
    if (!p1 || !sp || !p2 || !status) return RSA_EINVAL;
    if (count == 0) return RSA_OK;
    if (!grid_fits(count, 128)) return RSA_EINVAL;
    k_find_pair<<<grid_for(count, 128), 128, 0, as_stream(stream)>>>(p1, count, q, tol, sp, n_sp, sp_index,
                                                                     p2, status);
    return launch_status("rsa_find_pair");
}
