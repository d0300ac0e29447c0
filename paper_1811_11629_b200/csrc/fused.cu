// fused.cu — K2 fused consumer: generate in registers, reduce in registers /
// shared memory, never write the stream (no reference
// function — the conventions borrowed are stats._bin_uniform bin = floor(r*B)
// (stats.py:178-180) and the interstream pairing of stats.BitSource
// (stats.py:118-136)).
//
// One thread = one Mv=1 instance (rsacore.take_floats semantics,
// rsacore.py:261-264), drawn by draw.cuh's fast path (the fill kernels' draw).
// Per draw, beyond the fill path: 1 DADD + 3 DFMA for the
// moments/lag/pair sums, 2 SHFL for the partner stream (adjacent lanes hold
// instances 2j, 2j+1), 1 DFMA(rz) for the bin, and a u16 shared-memory counter
// bump (flushed to the u32 global row after every 2^15 draws so it cannot wrap).
#include "common.cuh"
#include "draw.cuh"

namespace rsa {

constexpr int FUSED_BLOCK = 128;
constexpr uint64_t FLUSH_MASK = (1u << 15) - 1;

// u16 counters (u32 shared-memory atomics measured +0.1 %, twice the smem:
// profiles/r01_ab_msg_fl.txt, tools/variants/draw_variants.cuh)
typedef uint16_t hist_t;
#define RSA_HIST_BUMP(p) (*(p) += 1)
RSA_DEV void flush_hist(hist_t* h, uint32_t* gh, bool active) {
#pragma unroll 8
    for (int b = 0; b < 64; ++b) {
        hist_t v = h[b * FUSED_BLOCK + threadIdx.x];
        if (v) {
            if (active) gh[b] += v;
            h[b * FUSED_BLOCK + threadIdx.x] = 0;
        }
    }
}

#ifndef RSA_FUSED_MINB
#define RSA_FUSED_MINB 8
#endif
template <uint32_t E>
__global__ void __launch_bounds__(FUSED_BLOCK, RSA_FUSED_MINB)
k_fused(const rsa_instance* __restrict__ inst, uint32_t n_inst, uint64_t draws,
        uint64_t* __restrict__ m1, uint64_t* __restrict__ m2, uint64_t* __restrict__ s,
        rsa_fused_stat* __restrict__ stats, uint32_t* __restrict__ hist) {
    __shared__ hist_t h[64 * FUSED_BLOCK];
    const uint32_t tid = threadIdx.x;
    const uint32_t i = blockIdx.x * FUSED_BLOCK + tid;
    const bool active = i < n_inst;
    const uint32_t ii = active ? i : n_inst - 1;  // idle lanes shadow a real one (shuffles)
    const FastInst P = load_fast(inst + ii);
    Lane L = lane_in(P, m1[ii], m2[ii], s[ii]);
    uint32_t* gh = hist + (uint64_t)ii * 64;
#pragma unroll 8
    for (int b = 0; b < 64; ++b) h[b * FUSED_BLOCK + tid] = 0;
    if (active)
        for (int b = 0; b < 64; ++b) gh[b] = 0;
    hist_t* hb = h + tid;

    double s1 = 0.0, s2 = 0.0, lag = 0.0, xy = 0.0, prev = 0.0, first = 0.0;
    // chunks of <= 2^15 draws: the u16 counters cannot wrap inside a chunk, and
    // the inner loop carries no flush test
    // the partner-stream shuffles need the whole warp on one loop body
    const bool gf = RSA_GARNER_FUSED && __all_sync(0xffffffffu, P.p1 <= GF_P1_MAX);
    auto run = [&](auto gfc) {
        constexpr bool GF = decltype(gfc)::value;
        for (uint64_t done = 0; done < draws;) {
            const uint64_t left = draws - done;
            const uint32_t len = (uint32_t)(left < FLUSH_MASK + 1 ? left : FLUSH_MASK + 1);
            uint32_t kk = 0;
            if (done == 0) {  // peeled first draw: r_0 is reported, no lag term yet
                double r = draw_unit<E, GF>(P, L);
                first = r;
                s1 = r;
                s2 = __dmul_rn(r, r);
                double o = __shfl_xor_sync(0xffffffffu, r, 1);
                xy = __dmul_rn(r, o);
                RSA_HIST_BUMP(&hb[(uint32_t)__double2loint(__fma_rz(r, 64.0, 0x1p52)) * FUSED_BLOCK]);
                prev = r;
                kk = 1;
            }
    #pragma unroll 2
            for (; kk < len; ++kk) {
                double r = draw_unit<E, GF>(P, L);
                s1 += r;
                s2 = __fma_rn(r, r, s2);
                lag = __fma_rn(prev, r, lag);
                prev = r;
                double o = __shfl_xor_sync(0xffffffffu, r, 1);
                xy = __fma_rn(r, o, xy);
                // floor(64 r) exactly: 2^52 + 64r rounded toward zero keeps the integer part
                uint32_t b = (uint32_t)__double2loint(__fma_rz(r, 64.0, 0x1p52));
                RSA_HIST_BUMP(&hb[b * FUSED_BLOCK]);
            }
            done += len;
            flush_hist(h, gh, active);
        }
    };
    if (gf) run(BoolC<true>{});
    else run(BoolC<false>{});
    if (active) {
        rsa_fused_stat st;
        st.s1 = s1; st.s2 = s2; st.lag = lag; st.first = first; st.last = prev; st.xy = xy;
        stats[i] = st;
        m1[i] = lane_m1(P, L);
        m2[i] = lane_m2(P, L);
        s[i] = L.s;
    }
}

// Deterministic pooled FP64 sums: thread t owns instances t, t+512, ... (all of
// one parity), fixed-order tree across threads.
__global__ void __launch_bounds__(512)
k_pool_stats(const rsa_fused_stat* __restrict__ stats, uint32_t n_inst, double* __restrict__ pooled) {
    __shared__ double red[7][512];
    const uint32_t t = threadIdx.x;
    double a[7] = {0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = t; i < n_inst; i += 512) {
        const rsa_fused_stat st = stats[i];
        a[0] += st.s1;
        a[1] += st.s2;
        if ((i & 1) == 0) { a[2] += st.xy; a[3] += st.s1; a[5] += st.s2; }
        else { a[4] += st.s1; a[6] += st.s2; }
    }
    for (int j = 0; j < 7; ++j) red[j][t] = a[j];
    __syncthreads();
    for (uint32_t w = 256; w > 0; w >>= 1) {
        if (t < w)
            for (int j = 0; j < 7; ++j) red[j][t] += red[j][t + w];
        __syncthreads();
    }
    if (t < 7) pooled[t] = red[t][0];
}

__global__ void k_pool_hist(const uint32_t* __restrict__ hist, uint32_t n_inst,
                            unsigned long long* __restrict__ pooled_hist) {
    __shared__ unsigned long long acc[64];
    if (threadIdx.x < 64) acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t b = threadIdx.x & 63;
    unsigned long long v = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 64) + threadIdx.x / 64; i < n_inst;
         i += (uint64_t)gridDim.x * (blockDim.x / 64))
        v += hist[i * 64 + b];
    atomicAdd(&acc[b], v);
    __syncthreads();
    if (threadIdx.x < 64) atomicAdd(&pooled_hist[threadIdx.x], acc[threadIdx.x]);
}

}  // namespace rsa

using namespace rsa;

template <uint32_t E>
static void launch_fused(cudaStream_t st, const rsa_instance* inst, uint32_t n, uint64_t draws,
                         uint64_t* m1, uint64_t* m2, uint64_t* s, rsa_fused_stat* stats,
                         uint32_t* hist) {
    k_fused<E><<<grid_for(n, FUSED_BLOCK), FUSED_BLOCK, 0, st>>>(inst, n, draws, m1, m2, s, stats, hist);
}

extern "C" int rsa_fused_stats(const rsa_instance* inst, uint32_t n_inst, uint64_t draws, uint32_t e,
                               uint64_t* m1, uint64_t* m2, uint64_t* s, rsa_fused_stat* stats,
                               uint32_t* hist, void* stream) {
    if (!inst || !m1 || !m2 || !s || !stats || !hist || n_inst == 0 || (n_inst & 1) || e == 0)
        return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    switch (e) {
        case 3: launch_fused<3>(st, inst, n_inst, draws, m1, m2, s, stats, hist); break;
        case 5: launch_fused<5>(st, inst, n_inst, draws, m1, m2, s, stats, hist); break;
        case 9: launch_fused<9>(st, inst, n_inst, draws, m1, m2, s, stats, hist); break;
        case 17: launch_fused<17>(st, inst, n_inst, draws, m1, m2, s, stats, hist); break;
        default: launch_fused<0>(st, inst, n_inst, draws, m1, m2, s, stats, hist); break;
    }
    return launch_status("rsa_fused_stats");
}

extern "C" int rsa_fused_pool(const rsa_fused_stat* stats, const uint32_t* hist, uint32_t n_inst,
                              double* pooled, uint64_t* pooled_hist, void* stream) {
    if (!stats || !hist || !pooled || !pooled_hist || n_inst == 0) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    cudaError_t err = cudaMemsetAsync(pooled_hist, 0, 64 * sizeof(uint64_t), st);
    if (err != cudaSuccess) { set_last_error("rsa_fused_pool(memset)", err); return RSA_ECUDA; }
    k_pool_stats<<<1, 512, 0, st>>>(stats, n_inst, pooled);
    int rc = launch_status("rsa_fused_pool(stats)");
    if (rc) return rc;
    unsigned grid = grid_for(n_inst, 4);
    if (grid > 592) grid = 592;
    k_pool_hist<<<grid, 256, 0, st>>>(hist, n_inst, reinterpret_cast<unsigned long long*>(pooled_hist));
    return launch_status("rsa_fused_pool(hist)");
}
