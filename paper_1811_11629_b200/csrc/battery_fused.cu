// battery_fused.cu — F1: chi-square battery consumers fed in registers
// (reference tests stats.py:233-442 over the
// interleaved source stats.BitSource, stats.py:118-136).
//
// K5 `k_bat_fused<E, KIND>`: the draw kernel of K1 (draw.cuh) produces the
// BitSource's variates in registers — thread = (lane, stream) in the
// round-robin order of RSA_FLAG_INTERLEAVE, R lanes per thread — and the
// consumer counts them without writing a single variate to HBM:
//   HIST         one cell per variate (frequency), straight from registers
//   tuple tests  (serial d, poker, max-of-t, permutation) the CTA's tile of
//                RSA_BT_TILE consecutive positions is staged in shared
//                memory; tuples inside the tile are counted by the CTA, the
//                (at most one) tuple straddling each tile boundary is handed
//                to a boundary slot (d doubles) and counted by
//                rsa_battery_stitch
//   GAPS         run boundaries of the tile from a flip bitmask (warp
//                ballots); runs inside the tile are counted, each tile leaves
//                a 16-byte record and rsa_battery_gaps_stitch counts the runs
//                that cross tiles (a segmented scan over the records)
// Small cell sets (poker 5, max-of-t bins, gaps 64) are counted in shared
// memory and flushed once per CTA; large ones (2^20 cells) with RED.64.
//
// Cells are the reference's (stats._bin_uniform, stats.py:178-180, and the
// per-test rules), counted with integer atomics: order-independent, so the
// counts — and the host-side statistics formed from them — are bit-identical
// to the materialised path and to the reference for the same variates.
#include "common.cuh"
#include "draw.cuh"

namespace rsa {

constexpr int BT_TB = 256;                 // threads per CTA
constexpr int BT_R = RSA_BT_TILE / BT_TB;  // lanes per thread (1: a BitSource has ~2^17 lanes, keep them all in flight)
constexpr int BT_SMALL = 128;              // shared-memory cells (poker, max-of-t, gaps)

__device__ __forceinline__ uint32_t bt_bin(double u, uint32_t bins) {
    long long k = (long long)__dmul_rn(u, (double)bins);  // truncation, as astype(int64)
    return k < (long long)bins ? (uint32_t)k : bins - 1;
}

// Cell of one tuple x[0..d) (d <= 32); *tie for the permutation test.
template <int KIND>
__device__ __forceinline__ uint32_t bt_tuple_cell(const double* x, const rsa_battery_spec& sp, bool* tie) {
    const uint32_t d = sp.d;
    if constexpr (KIND == RSA_BT_SERIAL) {
        uint32_t idx = 0;
        for (uint32_t c = 0; c < d; ++c) idx = idx * sp.p2 + bt_bin(x[c], sp.p2);
        return idx;
    } else if constexpr (KIND == RSA_BT_POKER) {
        uint32_t mask = 0;
#pragma unroll
        for (int c = 0; c < 5; ++c) mask |= 1u << bt_bin(x[c], 16);
        return __popc(mask) - 1;
    } else if constexpr (KIND == RSA_BT_MAX_OF_T) {
        double m = x[0];
        for (uint32_t c = 1; c < d; ++c) m = fmax(m, x[c]);
        return bt_bin(pow(m, (double)d), sp.p2);
    } else if constexpr (KIND == RSA_BT_COLLISION) {  // msb_of_20: bit k = (x_k > 1/2)
        uint32_t urn = 0;
        for (uint32_t c = 0; c < d; ++c) urn |= (uint32_t)(x[c] > 0.5) << c;
        return urn;
    } else {  // RSA_BT_PERMUTATION: Lehmer rank
        uint32_t rank = 0;
        bool eq = false;
        for (uint32_t a = 0; a + 1 < d; ++a) {
            uint32_t less = 0;
            for (uint32_t b = a + 1; b < d; ++b) {
                less += x[b] < x[a];
                eq |= x[b] == x[a];
            }
            rank = rank * (d - a) + less;
        }
        *tie = eq;
        return rank;
    }
}

// Collision test: ball `ball` (trial ball >> 14) lands in `urn`; a ball whose
// urn bit was already set in its trial's 2^20-bit bitmap is a collision.
constexpr uint32_t BT_COLL_BALLS_LOG = 14, BT_COLL_WORDS = (1u << 20) / 32;
__device__ __forceinline__ void bt_collide(const rsa_battery_spec& sp, uint64_t ball, uint32_t urn,
                                           unsigned long long* trial_counts) {
    const uint64_t trial = ball >> BT_COLL_BALLS_LOG;
    uint32_t* bm = reinterpret_cast<uint32_t*>(sp.aux) + trial * BT_COLL_WORDS;
    const uint32_t bit = 1u << (urn & 31);
    if (atomicOr(&bm[urn >> 5], bit) & bit) atomicAdd(&trial_counts[trial], 1ull);
}

template <int KIND>
__host__ __device__ constexpr bool bt_small() { return KIND == RSA_BT_POKER || KIND == RSA_BT_MAX_OF_T || KIND == RSA_BT_GAPS; }

// Shared state of one CTA's consumer.
struct BtShared {
    double tile[RSA_BT_TILE];
    uint32_t flips[RSA_BT_TILE / 32];
    uint32_t small[BT_SMALL];
    int tie;
};

template <int KIND>
__device__ __forceinline__ void bt_count(BtShared& sh, unsigned long long* counts, uint32_t cell) {
    if constexpr (bt_small<KIND>()) atomicAdd(&sh.small[cell], 1u);
    else atomicAdd(&counts[cell], 1ull);
}

// Tuple consumer over sh.tile[0, len) at test position P (tiles are full
// except possibly the last tile of a materialised array, which ends on a
// tuple boundary).  Slots: boundary `b` (left) and `b + 1` (right).
template <int KIND>
__device__ void bt_consume_tuples(BtShared& sh, const rsa_battery_spec& sp, uint64_t P, uint32_t len,
                                  uint64_t b, unsigned long long* counts, double* slots) {
    const uint32_t d = sp.d;
    const uint32_t phase = (uint32_t)(P % d);
    const uint32_t psi = (d - phase) % d;  // first tuple start in the tile
    const uint32_t body = len > psi ? len - psi : 0;
    const uint32_t n_t = body / d;
    const uint32_t suf = body - n_t * d;
    if constexpr (KIND == RSA_BT_MAX_OF_T) {
        // long tuples (t = 32): one warp per tuple, lane c holds value c, shuffle max.
        // (A warp-per-tuple Lehmer rank measured 3.4x slower than one thread per
        // tuple for the permutation test: profiles/r02_battery_per_test.txt.)
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (uint32_t j = warp; j < n_t; j += BT_TB / 32) {
            double m = lane < (int)d ? sh.tile[psi + j * d + lane] : 0.0;  // values >= 0: 0 is neutral
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) bt_count<KIND>(sh, counts, bt_bin(pow(m, (double)d), sp.p2));
        }
    } else {
        for (uint32_t j = threadIdx.x; j < n_t; j += BT_TB) {
            bool tie = false;
            const uint32_t cell = bt_tuple_cell<KIND>(&sh.tile[psi + j * d], sp, &tie);
            if (KIND == RSA_BT_PERMUTATION && tie) sh.tie = 1;
            if constexpr (KIND == RSA_BT_COLLISION) bt_collide(sp, (P + psi + j * d) / d, cell, counts);
            else bt_count<KIND>(sh, counts, cell);
        }
    }
    const uint32_t pre = psi < len ? psi : len;
    if (threadIdx.x < pre) slots[b * d + phase + threadIdx.x] = sh.tile[threadIdx.x];
    if (threadIdx.x < suf) slots[(b + 1) * d + threadIdx.x] = sh.tile[len - suf + threadIdx.x];
}

// Gaps consumer: run boundaries inside the tile, record for the stitch.
__device__ void bt_consume_gaps(BtShared& sh, uint32_t len, rsa_gap_record* rec) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // flip bit at position p >= 1: side(p) != side(p - 1)
    for (uint32_t w = warp; w < RSA_BT_TILE / 32; w += BT_TB / 32) {
        const uint32_t p = w * 32 + lane;
        bool f = false;
        if (p >= 1 && p < len) f = (sh.tile[p] > 0.5) != (sh.tile[p - 1] > 0.5);
        const uint32_t m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) sh.flips[w] = m;
    }
    __syncthreads();
    const uint32_t nw = (len + 31) / 32;
    // each flip p closes the run that the previous flip q < p opened: count p - q
    for (uint32_t p = threadIdx.x; p < len; p += BT_TB) {
        if (!((sh.flips[p >> 5] >> (p & 31)) & 1u)) continue;
        uint32_t w = p >> 5;
        uint32_t below = sh.flips[w] & ((1u << (p & 31)) - 1u);
        int q = -1;
        if (below) q = (int)(w * 32 + 31 - __clz(below));
        else
            for (int v = (int)w - 1; v >= 0; --v)
                if (sh.flips[v]) { q = v * 32 + 31 - __clz(sh.flips[v]); break; }
        if (q >= 0) {
            const uint32_t L = (uint32_t)(p - q);
            atomicAdd(&sh.small[(L < 64 ? L : 64) - 1], 1u);
        }
    }
    if (threadIdx.x == 0) {
        int first = -1, last = -1;
        for (uint32_t v = 0; v < nw; ++v)
            if (sh.flips[v]) {
                if (first < 0) first = v * 32 + __ffs(sh.flips[v]) - 1;
                last = v * 32 + 31 - __clz(sh.flips[v]);
            }
        rsa_gap_record r;
        r.len = len;
        r.head = first < 0 ? len : (uint32_t)first;
        r.tail = last < 0 ? len : len - (uint32_t)last;
        r.bits = (first >= 0 ? 1u : 0u) | (sh.tile[0] > 0.5 ? 2u : 0u) | (sh.tile[len - 1] > 0.5 ? 4u : 0u);
        *rec = r;
    }
}

template <int KIND>
__device__ __forceinline__ void bt_init(BtShared& sh) {
    if constexpr (bt_small<KIND>())
        for (int c = threadIdx.x; c < BT_SMALL; c += BT_TB) sh.small[c] = 0;
    if (threadIdx.x == 0) sh.tie = 0;
}

template <int KIND>
__device__ __forceinline__ void bt_flush(BtShared& sh, const rsa_battery_spec& sp, unsigned long long* counts,
                                         int* flag) {
    __syncthreads();
    if constexpr (bt_small<KIND>()) {
        const uint32_t cells = KIND == RSA_BT_POKER ? 5 : KIND == RSA_BT_GAPS ? 64 : sp.p2;
        for (uint32_t c = threadIdx.x; c < cells; c += BT_TB)
            if (sh.small[c]) atomicAdd(&counts[c], (unsigned long long)sh.small[c]);
    }
    if (KIND == RSA_BT_PERMUTATION && threadIdx.x == 0 && sh.tie) atomicExch(flag, 1);
}

// ---- K5: generate + count ------------------------------------------------------

template <uint32_t E, int KIND, bool LOW32>
__global__ void __launch_bounds__(BT_TB)
k_bat_fused(const rsa_instance* __restrict__ inst, uint32_t S, uint32_t mv, uint64_t blocks,
            uint64_t* __restrict__ m1, uint64_t* __restrict__ m2, uint64_t* __restrict__ s,
            const rsa_battery_spec sp, unsigned long long* __restrict__ counts, int* __restrict__ flag,
            double* __restrict__ slots, rsa_gap_record* __restrict__ records) {
    __shared__ BtShared sh;
    bt_init<KIND>(sh);
    const uint32_t C = mv * S / RSA_BT_TILE;  // tiles per block
    const uint32_t c = blockIdx.x;            // this CTA's tile within every block
    const uint32_t stream = threadIdx.x % S;  // S | BT_TB: the same stream for all R lanes
    const FastInst P = load_fast(inst + stream);
    Lane L[BT_R];
    uint64_t li[BT_R];
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        const uint64_t q = (uint64_t)c * RSA_BT_TILE + r * BT_TB + threadIdx.x;  // position in the block
        li[r] = (uint64_t)stream * mv + q / S;
        L[r] = lane_in(P, m1[li[r]], m2[li[r]], s[li[r]]);
    }
    __syncthreads();
    with_garner(P, [&](auto gf) {
        constexpr bool GF = decltype(gf)::value;
        for (uint64_t k = 0; k < blocks; ++k) {
            double v[BT_R];
#pragma unroll
            for (int r = 0; r < BT_R; ++r) {
                const uint64_t cc = draw_fast<E, GF>(P, L[r]);
                v[r] = LOW32 ? __uint2double_rn((uint32_t)cc) * 0x1p-32
                             : to_unit_dd(cc, P.n_float, P.n_recip, P.n_recip_lo);
            }
            if constexpr (KIND == RSA_BT_HIST) {
#pragma unroll
                for (int r = 0; r < BT_R; ++r) atomicAdd(&counts[bt_bin(v[r], sp.p1)], 1ull);
            } else if (KIND == RSA_BT_COLLISION && sp.d == 1) {  // top20bits: one ball per variate
                const uint64_t base = sp.pos0 + (k * C + c) * RSA_BT_TILE;
#pragma unroll
                for (int r = 0; r < BT_R; ++r)
                    bt_collide(sp, base + r * BT_TB + threadIdx.x, bt_bin(v[r], 1u << 20), counts);
            } else {
#pragma unroll
                for (int r = 0; r < BT_R; ++r) sh.tile[r * BT_TB + threadIdx.x] = v[r];
                __syncthreads();
                const uint64_t t = k * C + c;  // tile index within the launch
                if constexpr (KIND == RSA_BT_GAPS)
                    bt_consume_gaps(sh, RSA_BT_TILE, records + sp.seg0 + t);
                else
                    bt_consume_tuples<KIND>(sh, sp, sp.pos0 + t * RSA_BT_TILE, RSA_BT_TILE, sp.seg0 + t,
                                            counts, slots);
                __syncthreads();
            }
        }
    });
#pragma unroll
    for (int r = 0; r < BT_R; ++r) {
        m1[li[r]] = lane_m1(P, L[r]);
        m2[li[r]] = lane_m2(P, L[r]);
        s[li[r]] = L[r].s;
    }
    bt_flush<KIND>(sh, sp, counts, flag);
}

// Gaps over a materialised array: one tile per CTA iteration.
__global__ void __launch_bounds__(BT_TB)
k_bat_gaps_array(const double* __restrict__ v, uint64_t n, const rsa_battery_spec sp,
                 unsigned long long* __restrict__ counts, rsa_gap_record* __restrict__ records) {
    __shared__ BtShared sh;
    bt_init<RSA_BT_GAPS>(sh);
    const uint64_t tiles = (n + RSA_BT_TILE - 1) / RSA_BT_TILE;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const uint64_t base = t * RSA_BT_TILE;
        const uint32_t len = (uint32_t)(n - base < RSA_BT_TILE ? n - base : RSA_BT_TILE);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < len; i += BT_TB) sh.tile[i] = v[base + i];
        __syncthreads();
        bt_consume_gaps(sh, len, records + sp.seg0 + t);
    }
    bt_flush<RSA_BT_GAPS>(sh, sp, counts, nullptr);
}

// Boundary tuples: slot b holds the d variates of the tuple straddling
// boundary b when its phase is nonzero.
template <int KIND>
__global__ void k_bat_stitch(const rsa_battery_spec sp, const double* __restrict__ slots, uint64_t first,
                             uint64_t n, unsigned long long* __restrict__ counts, int* __restrict__ flag) {
    __shared__ BtShared sh;
    bt_init<KIND>(sh);
    __syncthreads();
    for (uint64_t j = (uint64_t)blockIdx.x * BT_TB + threadIdx.x; j < n; j += (uint64_t)gridDim.x * BT_TB) {
        const uint64_t b = first + j;
        const uint64_t pos = sp.pos0 + (b - sp.seg0) * RSA_BT_TILE;
        if (pos % sp.d == 0) continue;
        double x[32];
        for (uint32_t i = 0; i < sp.d; ++i) x[i] = slots[b * sp.d + i];
        bool tie = false;
        const uint32_t cell = bt_tuple_cell<KIND>(x, sp, &tie);
        if (KIND == RSA_BT_PERMUTATION && tie) sh.tie = 1;
        if constexpr (KIND == RSA_BT_COLLISION) bt_collide(sp, (pos - pos % sp.d) / sp.d, cell, counts);
        else bt_count<KIND>(sh, counts, cell);
    }
    bt_flush<KIND>(sh, sp, counts, flag);
}

// Runs crossing tiles.  ext(j) = length of the run that ends at the end of
// tile j = tail(j) if tile j has an internal flip, else len(j) + ext(j-1)
// when the run continues from tile j-1 (same side), else len(j): a
// segmented scan, done by one CTA in thread-contiguous chunks.  Then every
// tile j counts (a) the run ending at its left boundary when the side
// changes there (ext(j-1)), (b) the run ending at its first internal flip
// (head(j) + ext(j-1) when the run continues into the tile).
__global__ void __launch_bounds__(1024)
k_bat_gaps_stitch(const rsa_gap_record* __restrict__ rec, uint64_t n, unsigned long long* __restrict__ counts) {
    __shared__ uint64_t agg_sum[1024];
    __shared__ uint32_t agg_reset[1024];
    __shared__ uint32_t small[64];
    const uint32_t t = threadIdx.x;
    if (t < 64) small[t] = 0;
    const uint64_t per = (n + 1023) / 1024;
    const uint64_t lo = t * per, hi = lo + per < n ? lo + per : n;
    // local segmented scan aggregate: (sum since the last reset, whether a reset occurred)
    uint64_t sum = 0;
    uint32_t reset = 0;
    for (uint64_t j = lo; j < hi; ++j) {
        const rsa_gap_record r = rec[j];
        const bool link = j > 0 && ((rec[j - 1].bits >> 2) & 1u) == ((r.bits >> 1) & 1u);
        if (r.bits & 1u) { sum = r.tail; reset = 1; }
        else if (link) sum += r.len;
        else { sum = r.len; reset = 1; }
    }
    agg_sum[t] = sum;
    agg_reset[t] = reset;
    __syncthreads();
    // exclusive carry into chunk t: compose the aggregates of chunks < t (sequential over
    // the chunk aggregates from the nearest reset; the chain is short for real data)
    uint64_t carry = 0;
    for (int u = (int)t - 1; u >= 0; --u) {
        carry += agg_sum[u];
        if (agg_reset[u]) break;
    }
    __syncthreads();
    uint64_t ext_prev = carry;  // ext(lo - 1) (0 before the first tile)
    for (uint64_t j = lo; j < hi; ++j) {
        const rsa_gap_record r = rec[j];
        const bool link = j > 0 && ((rec[j - 1].bits >> 2) & 1u) == ((r.bits >> 1) & 1u);
        if (j > 0 && !link) {  // (a) side change at the boundary closes the previous run
            const uint64_t L = ext_prev;
            atomicAdd(&small[(L < 64 ? L : 64) - 1], 1u);
        }
        if (r.bits & 1u) {  // (b) the run closed by the tile's first internal flip
            const uint64_t L = r.head + (link ? ext_prev : 0);
            atomicAdd(&small[(L < 64 ? L : 64) - 1], 1u);
        }
        uint64_t ext;
        if (r.bits & 1u) ext = r.tail;
        else ext = r.len + (link ? ext_prev : 0);
        ext_prev = ext;
    }
    __syncthreads();
    if (t < 64 && small[t]) atomicAdd(&counts[t], (unsigned long long)small[t]);
}

// Fourier cells: searchsorted(edges, value) for the real and imaginary parts.
__global__ void k_bat_fourier_bin(const double* __restrict__ z, uint64_t n, const double* __restrict__ edges,
                                  unsigned long long* __restrict__ counts) {
    __shared__ double e[63];
    __shared__ uint32_t cells[128];
    if (threadIdx.x < 63) e[threadIdx.x] = edges[threadIdx.x];
    if (threadIdx.x < 128) cells[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = z[i];
        uint32_t lo = 0, hi = 63;  // first edge >= x (side='left'): #edges < x
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (e[mid] < x) lo = mid + 1; else hi = mid;
        }
        atomicAdd(&cells[(i & 1) * 64 + lo], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 128 && cells[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)cells[threadIdx.x]);
}

}  // namespace rsa

using namespace rsa;

template <uint32_t E, int KIND>
static void launch_bat(unsigned grid, cudaStream_t st, bool low32, const rsa_instance* inst, uint32_t S,
                       uint32_t mv, uint64_t blocks, uint64_t* m1, uint64_t* m2, uint64_t* s,
                       const rsa_battery_spec& sp, unsigned long long* counts, int* flag, double* slots,
                       rsa_gap_record* rec) {
    if (low32)
        k_bat_fused<E, KIND, true><<<grid, BT_TB, 0, st>>>(inst, S, mv, blocks, m1, m2, s, sp, counts, flag, slots, rec);
    else
        k_bat_fused<E, KIND, false><<<grid, BT_TB, 0, st>>>(inst, S, mv, blocks, m1, m2, s, sp, counts, flag, slots, rec);
}

template <int KIND>
static void dispatch_bat_e(uint32_t e, unsigned grid, cudaStream_t st, bool low32, const rsa_instance* inst,
                           uint32_t S, uint32_t mv, uint64_t blocks, uint64_t* m1, uint64_t* m2, uint64_t* s,
                           const rsa_battery_spec& sp, unsigned long long* counts, int* flag, double* slots,
                           rsa_gap_record* rec) {
    switch (e) {
        case 3: launch_bat<3, KIND>(grid, st, low32, inst, S, mv, blocks, m1, m2, s, sp, counts, flag, slots, rec); break;
        case 9: launch_bat<9, KIND>(grid, st, low32, inst, S, mv, blocks, m1, m2, s, sp, counts, flag, slots, rec); break;
        default: launch_bat<0, KIND>(grid, st, low32, inst, S, mv, blocks, m1, m2, s, sp, counts, flag, slots, rec); break;
    }
}

static bool bat_tuple_ok(const rsa_battery_spec& sp) {
    switch (sp.test) {
        case RSA_BT_COLLISION: return (sp.d == 1 || sp.d == 20) && sp.aux != 0;
        case RSA_BT_SERIAL: return sp.d >= 2 && sp.d <= 6 && sp.p2 > 0;
        case RSA_BT_POKER: return sp.d == 5;
        case RSA_BT_MAX_OF_T: return sp.d >= 1 && sp.d <= 32 && sp.p2 > 0 && sp.p2 <= BT_SMALL;
        case RSA_BT_PERMUTATION: return sp.d >= 2 && sp.d <= 10;
        default: return false;
    }
}

extern "C" int rsa_battery_fused(const rsa_instance* inst, uint32_t n_inst, uint32_t mv, uint64_t blocks,
                                 uint32_t e, uint32_t flags, uint64_t* m1, uint64_t* m2, uint64_t* s,
                                 const rsa_battery_spec* spec, unsigned long long* counts, int* flag,
                                 double* slots, rsa_gap_record* records, void* stream) {
    if (!inst || !m1 || !m2 || !s || !spec || !counts || n_inst == 0 || mv == 0 || e == 0) return RSA_EINVAL;
    if (BT_TB % n_inst || ((uint64_t)mv * n_inst) % RSA_BT_TILE) return RSA_EINVAL;
    const rsa_battery_spec sp = *spec;
    const bool tuple = sp.test != RSA_BT_HIST && sp.test != RSA_BT_GAPS &&
                       !(sp.test == RSA_BT_COLLISION && sp.d == 1);
    if (sp.test == RSA_BT_COLLISION && !bat_tuple_ok(sp)) return RSA_EINVAL;
    if (sp.test == RSA_BT_HIST && (sp.p1 == 0 || sp.d != 1)) return RSA_EINVAL;
    if (sp.test == RSA_BT_GAPS && (sp.d != 1 || !records)) return RSA_EINVAL;
    if (tuple && (!bat_tuple_ok(sp) || !slots)) return RSA_EINVAL;
    if (sp.test == RSA_BT_PERMUTATION && !flag) return RSA_EINVAL;
    if (blocks == 0) return RSA_OK;
    const unsigned grid = (unsigned)((uint64_t)mv * n_inst / RSA_BT_TILE);
    cudaStream_t st = as_stream(stream);
    const bool low32 = flags & RSA_FLAG_LOW32;
#define RSA_BT_CASE(K) \
    case K: dispatch_bat_e<K>(e, grid, st, low32, inst, n_inst, mv, blocks, m1, m2, s, sp, counts, flag, slots, records); break;
    switch (sp.test) {
        RSA_BT_CASE(RSA_BT_HIST)
        RSA_BT_CASE(RSA_BT_SERIAL)
        RSA_BT_CASE(RSA_BT_POKER)
        RSA_BT_CASE(RSA_BT_MAX_OF_T)
        RSA_BT_CASE(RSA_BT_PERMUTATION)
        RSA_BT_CASE(RSA_BT_GAPS)
        RSA_BT_CASE(RSA_BT_COLLISION)
        default: return RSA_EINVAL;
    }
#undef RSA_BT_CASE
    return launch_status("rsa_battery_fused");
}

extern "C" int rsa_battery_gaps_array(const double* v, uint64_t n, const rsa_battery_spec* spec,
                                      unsigned long long* counts, rsa_gap_record* records, void* stream) {
    if ((!v && n) || !spec || !counts || !records) return RSA_EINVAL;
    if (n == 0) return RSA_OK;
    const uint64_t tiles = (n + RSA_BT_TILE - 1) / RSA_BT_TILE;
    const unsigned grid = (unsigned)(tiles < 148 * 8 ? tiles : 148 * 8);
    k_bat_gaps_array<<<grid, BT_TB, 0, as_stream(stream)>>>(v, n, *spec, counts, records);
    return launch_status("rsa_battery_gaps_array");
}

extern "C" int rsa_battery_stitch(const rsa_battery_spec* spec, const double* slots, uint64_t first, uint64_t n,
                                  unsigned long long* counts, int* flag, void* stream) {
    if (!spec || !counts || (!slots && n)) return RSA_EINVAL;
    const rsa_battery_spec sp = *spec;
    if (!bat_tuple_ok(sp) || first < sp.seg0) return RSA_EINVAL;
    if (sp.test == RSA_BT_PERMUTATION && !flag) return RSA_EINVAL;
    if (sp.test == RSA_BT_COLLISION && sp.d == 1) return RSA_EINVAL;  // single-variate balls never straddle
    if (n == 0) return RSA_OK;
    const unsigned grid = (unsigned)((n + BT_TB - 1) / BT_TB < 148 * 4 ? (n + BT_TB - 1) / BT_TB : 148 * 4);
    cudaStream_t st = as_stream(stream);
    switch (sp.test) {
        case RSA_BT_SERIAL: k_bat_stitch<RSA_BT_SERIAL><<<grid, BT_TB, 0, st>>>(sp, slots, first, n, counts, flag); break;
        case RSA_BT_POKER: k_bat_stitch<RSA_BT_POKER><<<grid, BT_TB, 0, st>>>(sp, slots, first, n, counts, flag); break;
        case RSA_BT_MAX_OF_T: k_bat_stitch<RSA_BT_MAX_OF_T><<<grid, BT_TB, 0, st>>>(sp, slots, first, n, counts, flag); break;
        case RSA_BT_COLLISION: k_bat_stitch<RSA_BT_COLLISION><<<grid, BT_TB, 0, st>>>(sp, slots, first, n, counts, flag); break;
        default: k_bat_stitch<RSA_BT_PERMUTATION><<<grid, BT_TB, 0, st>>>(sp, slots, first, n, counts, flag); break;
    }
    return launch_status("rsa_battery_stitch");
}

extern "C" int rsa_battery_gaps_stitch(const rsa_gap_record* records, uint64_t n_rec, unsigned long long* counts,
                                       void* stream) {
    if ((!records && n_rec) || !counts) return RSA_EINVAL;
    if (n_rec == 0) return RSA_OK;
    k_bat_gaps_stitch<<<1, 1024, 0, as_stream(stream)>>>(records, n_rec, counts);
    return launch_status("rsa_battery_gaps_stitch");
}

extern "C" int rsa_battery_fourier_bin(const double* coeff, uint64_t n, const double* edges,
                                       unsigned long long* counts, void* stream) {
    if ((!coeff && n) || !edges || !counts) return RSA_EINVAL;
    if (n == 0) return RSA_OK;
    unsigned grid = grid_for(2 * n, 256);
    if (grid > 148 * 8) grid = 148 * 8;
    k_bat_fourier_bin<<<grid, 256, 0, as_stream(stream)>>>(coeff, n, edges, counts);
    return launch_status("rsa_battery_fourier_bin");
}

// Collision balls from a materialised array of whole balls.
__global__ void k_bat_collision_array(const double* __restrict__ v, uint64_t balls, const rsa_battery_spec sp,
                                      unsigned long long* __restrict__ trial_counts) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < balls;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t urn;
        if (sp.d == 1) urn = bt_bin(v[j], 1u << 20);
        else {
            urn = 0;
            for (uint32_t c = 0; c < sp.d; ++c) urn |= (uint32_t)(v[j * sp.d + c] > 0.5) << c;
        }
        bt_collide(sp, sp.pos0 / sp.d + j, urn, trial_counts);
    }
}

__global__ void k_bat_collision_hist(const unsigned long long* __restrict__ trial_counts, uint64_t trials,
                                     unsigned long long* __restrict__ counts) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < trials;
         t += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[trial_counts[t]], 1ull);
}

// ---- chi-square sum in numpy's order -------------------------------------------
//
// The equiprobable tests' statistic is float(np.square(counts - e).sum() / e)
// (stats.py: _uniform_report).  numpy sums a contiguous float64 vector
// pairwise (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum): n < 8
// sequentially from 0.0; n <= 128 with eight strided accumulators combined
// as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential remainder;
// otherwise split at n2 = n/2 rounded down to a multiple of 8 and add the two
// halves.  Restated here exactly (tree built level by level, leaves in
// parallel, internal nodes bottom-up), so the device statistic is
// bit-identical to the host's and only one double leaves the GPU.

struct PwNode {
    uint64_t off;
    uint32_t size;
    uint32_t child;  // first child's node index; PW_LEAF for leaves
};
constexpr uint32_t PW_LEAF = 0xFFFFFFFFu;
constexpr int PW_MAX_LEVELS = 62;

__device__ __forceinline__ double pw_term(const long long* c, uint64_t i, double e) {
    const double d = __dsub_rn(__ll2double_rn(c[i]), e);
    return __dmul_rn(d, d);
}

__device__ double pw_leaf(const long long* c, uint32_t n, double e) {
    if (n < 8) {
        double r = 0.0;
        for (uint32_t i = 0; i < n; ++i) r = __dadd_rn(r, pw_term(c, i, e));
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = pw_term(c, j, e);
    uint32_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], pw_term(c, i + j, e));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, pw_term(c, i, e));
    return res;
}

// One CTA: the recursion tree level by level.  levels[0] = number of levels,
// levels[1 + L] = first node index of level L (levels[1 + nlev] = node count).
__global__ void __launch_bounds__(1024) k_pw_build(uint64_t n, PwNode* __restrict__ nodes, uint32_t* __restrict__ levels) {
    __shared__ uint32_t base[PW_MAX_LEVELS + 2];
    __shared__ uint32_t scan[1024];
    const uint32_t t = threadIdx.x;
    if (t == 0) {
        nodes[0].off = 0;
        nodes[0].size = (uint32_t)n;
        base[0] = 0;
        base[1] = 1;
    }
    int L = 0;
    for (;; ++L) {
        __syncthreads();
        const uint32_t b0 = base[L], b1 = base[L + 1];
        if (b1 == b0 || L >= PW_MAX_LEVELS) break;
        const uint32_t cnt = b1 - b0, per = (cnt + 1023) / 1024;
        const uint32_t lo = b0 + t * per < b1 ? b0 + t * per : b1;
        const uint32_t hi = lo + per < b1 ? lo + per : b1;
        uint32_t mine = 0;
        for (uint32_t i = lo; i < hi; ++i) mine += nodes[i].size > 128;
        scan[t] = mine;
        __syncthreads();
        for (uint32_t w = 1; w < 1024; w <<= 1) {  // inclusive Hillis-Steele scan
            const uint32_t v = t >= w ? scan[t - w] : 0;
            __syncthreads();
            scan[t] += v;
            __syncthreads();
        }
        uint32_t next = b1 + 2 * (scan[t] - mine);
        for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t sz = nodes[i].size;
            if (sz > 128) {
                uint32_t n2 = sz / 2;
                n2 -= n2 % 8;
                nodes[i].child = next;
                nodes[next].off = nodes[i].off;
                nodes[next].size = n2;
                nodes[next + 1].off = nodes[i].off + n2;
                nodes[next + 1].size = sz - n2;
                next += 2;
            } else {
                nodes[i].child = PW_LEAF;
            }
        }
        if (t == 1023) base[L + 2] = b1 + 2 * scan[1023];
    }
    __syncthreads();
    if (t == 0) levels[0] = (uint32_t)L;
    for (int l = t; l <= L; l += 1024) levels[1 + l] = base[l];
}

__global__ void k_pw_leaves(const long long* __restrict__ c, double e, const PwNode* __restrict__ nodes,
                            const uint32_t* __restrict__ levels, double* __restrict__ vals) {
    const uint32_t total = levels[1 + levels[0]];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const PwNode nd = nodes[i];
        if (nd.child == PW_LEAF) vals[i] = pw_leaf(c + nd.off, nd.size, e);
    }
}

__global__ void __launch_bounds__(1024) k_pw_combine(const PwNode* __restrict__ nodes, const uint32_t* __restrict__ levels,
                                                     double* __restrict__ vals, double* __restrict__ out) {
    const int nlev = (int)levels[0];
    for (int L = nlev - 1; L >= 0; --L) {
        const uint32_t b0 = levels[1 + L], b1 = levels[2 + L];
        for (uint32_t i = b0 + threadIdx.x; i < b1; i += 1024) {
            const uint32_t ch = nodes[i].child;
            if (ch != PW_LEAF) vals[i] = __dadd_rn(vals[ch], vals[ch + 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = vals[0];
}

extern "C" uint64_t rsa_battery_chi2_scratch_bytes(uint64_t n) {
    if (n == 0 || n > 0xFFFFFFFFull) return 0;
    const uint64_t nodes = 4 * (n / 64 + 1) + 64;  // leaves hold >= 64 values except a root below 128
    return nodes * (sizeof(PwNode) + sizeof(double)) + (PW_MAX_LEVELS + 2) * sizeof(uint32_t) + 64;
}

extern "C" int rsa_battery_chi2_sum(const long long* counts, uint64_t n, double e, double* out, void* scratch,
                                    uint64_t scratch_bytes, void* stream) {
    if (!counts || !out || !scratch || n == 0 || n > 0xFFFFFFFFull) return RSA_EINVAL;
    if (scratch_bytes < rsa_battery_chi2_scratch_bytes(n)) return RSA_ECAPACITY;
    const uint64_t max_nodes = 4 * (n / 64 + 1) + 64;
    char* p = static_cast<char*>(scratch);
    PwNode* nodes = reinterpret_cast<PwNode*>(p);
    double* vals = reinterpret_cast<double*>(p + max_nodes * sizeof(PwNode));
    uint32_t* levels = reinterpret_cast<uint32_t*>(p + max_nodes * (sizeof(PwNode) + sizeof(double)));
    cudaStream_t st = as_stream(stream);
    k_pw_build<<<1, 1024, 0, st>>>(n, nodes, levels);
    unsigned g = grid_for(max_nodes, 256);
    if (g > 148 * 4) g = 148 * 4;
    k_pw_leaves<<<g, 256, 0, st>>>(counts, e, nodes, levels, vals);
    k_pw_combine<<<1, 1024, 0, st>>>(nodes, levels, vals, out);
    return launch_status("rsa_battery_chi2_sum", 3);
}

extern "C" int rsa_battery_collision_array(const double* v, uint64_t n, const rsa_battery_spec* spec,
                                           unsigned long long* trial_counts, void* stream) {
    if ((!v && n) || !spec || !trial_counts) return RSA_EINVAL;
    const rsa_battery_spec sp = *spec;
    if (sp.test != RSA_BT_COLLISION || !bat_tuple_ok(sp) || n % sp.d || sp.pos0 % sp.d) return RSA_EINVAL;
    if (n == 0) return RSA_OK;
    const uint64_t balls = n / sp.d;
    unsigned grid = grid_for(balls, 256);
    if (grid > 148 * 8) grid = 148 * 8;
    k_bat_collision_array<<<grid, 256, 0, as_stream(stream)>>>(v, balls, sp, trial_counts);
    return launch_status("rsa_battery_collision_array");
}

extern "C" int rsa_battery_collision_hist(const unsigned long long* trial_counts, uint64_t trials,
                                          unsigned long long* counts, void* stream) {
    if ((!trial_counts && trials) || !counts) return RSA_EINVAL;
    if (trials == 0) return RSA_OK;
    unsigned grid = grid_for(trials, 256);
    if (grid > 148 * 8) grid = 148 * 8;
    k_bat_collision_hist<<<grid, 256, 0, as_stream(stream)>>>(trial_counts, trials, counts);
    return launch_status("rsa_battery_collision_hist");
}
