// battery.cu — device counting kernels of the chi-square battery
// (reference stats.py:233-466).  Each kernel turns a
// device buffer of variates (a BitSource chunk) into the integer cell counts
// the reference computes with numpy; the chi-square statistic and p-value are
// then formed on the host from those (small) count vectors exactly as the
// reference forms them.  Counts are order-independent (integer atomics), so
// they are bit-identical to the reference's for identical inputs.
//
// Binning convention (stats._bin_uniform, stats.py:178-180): cell =
// min(trunc(RN(u * B)), B - 1).
#include "common.cuh"

namespace rsa {

__device__ __forceinline__ uint32_t bin_of(double u, uint32_t bins) {
    long long k = (long long)__dmul_rn(u, (double)bins);  // truncation, as astype(int64)
    return k < (long long)bins ? (uint32_t)k : bins - 1;
}

// frequency (stats.py:236-245): one cell per variate
__global__ void k_hist(const double* __restrict__ v, uint64_t n, uint32_t bins,
                       unsigned long long* __restrict__ counts) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[bin_of(v[i], bins)], 1ull);
}

// serial (stats.py:251-273): non-overlapping d-tuples, row-major cell index
__global__ void k_serial(const double* __restrict__ v, uint64_t tuples, int d, uint32_t axis,
                         unsigned long long* __restrict__ counts) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tuples;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = 0;
        for (int c = 0; c < d; ++c) idx = idx * axis + bin_of(v[t * d + c], axis);
        atomicAdd(&counts[idx], 1ull);
    }
}

// poker (stats.py:291-305): 5 cards of 16 denominations, number of distinct ones
__global__ void k_poker(const double* __restrict__ v, uint64_t hands, unsigned long long* __restrict__ counts) {
    __shared__ unsigned long long c5[5];
    if (threadIdx.x < 5) c5[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t h = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; h < hands;
         h += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t mask = 0;
#pragma unroll
        for (int c = 0; c < 5; ++c) mask |= 1u << bin_of(v[h * 5 + c], 16);
        atomicAdd(&c5[__popc(mask) - 1], 1ull);
    }
    __syncthreads();
    if (threadIdx.x < 5) atomicAdd(&counts[threadIdx.x], c5[threadIdx.x]);
}

// max-of-t (stats.py:403-417): cell of (max of t values)^t
__global__ void k_max_of_t(const double* __restrict__ v, uint64_t tuples, int t, uint32_t bins,
                           unsigned long long* __restrict__ counts) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tuples;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double m = v[i * t];
        for (int c = 1; c < t; ++c) m = fmax(m, v[i * t + c]);
        atomicAdd(&counts[bin_of(pow(m, (double)t), bins)], 1ull);
    }
}

// permutation (stats.py:420-442): Lehmer rank of each t-tuple; *tie set on
// exactly equal values inside a tuple
__global__ void k_permutation(const double* __restrict__ v, uint64_t tuples, int t,
                              unsigned long long* __restrict__ counts, int* __restrict__ tie) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tuples;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x[10];
        for (int c = 0; c < t; ++c) x[c] = v[i * t + c];
        uint64_t rank = 0;
        bool eq = false;
        for (int a = 0; a < t - 1; ++a) {
            uint32_t less = 0;
            for (int b = a + 1; b < t; ++b) {
                less += x[b] < x[a];
                eq |= x[b] == x[a];
            }
            rank = rank * (t - a) + less;
        }
        if (eq) atomicExch(tie, 1);
        atomicAdd(&counts[rank], 1ull);
    }
}

// collision (stats.py:331-362): one CTA per trial, 2^20-urn bitmap in shared
// memory; a ball whose urn bit was already set is a collision.
// mode 0: urn = cell of one variate (top 20 bits); mode 1: urn = the bits
// (u > 1/2) of 20 sequential variates, variate k -> bit k.
constexpr uint32_t COLL_BALLS = 1u << 14;
constexpr uint32_t COLL_WORDS = (1u << 20) / 32;

__global__ void __launch_bounds__(1024)
k_collision(const double* __restrict__ v, uint32_t trials, int mode, unsigned long long* __restrict__ observed) {
    extern __shared__ uint32_t bm[];
    __shared__ uint32_t coll;
    const uint32_t per_ball = mode ? 20 : 1;
    for (uint32_t trial = blockIdx.x; trial < trials; trial += gridDim.x) {
        for (uint32_t w = threadIdx.x; w < COLL_WORDS; w += blockDim.x) bm[w] = 0;
        if (threadIdx.x == 0) coll = 0;
        __syncthreads();
        const double* tv = v + (uint64_t)trial * COLL_BALLS * per_ball;
        uint32_t mine = 0;
        for (uint32_t b = threadIdx.x; b < COLL_BALLS; b += blockDim.x) {
            uint32_t urn;
            if (mode == 0) {
                urn = bin_of(tv[b], 1u << 20);
            } else {
                urn = 0;
                for (int k = 0; k < 20; ++k) urn |= (uint32_t)(tv[(uint64_t)b * 20 + k] > 0.5) << k;
            }
            const uint32_t bit = 1u << (urn & 31);
            mine += (atomicOr(&bm[urn >> 5], bit) & bit) != 0;
        }
        atomicAdd(&coll, mine);
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(&observed[coll], 1ull);
        __syncthreads();
    }
}

}  // namespace rsa

using namespace rsa;

static unsigned grid_cap(uint64_t n, unsigned block) {
    uint64_t g = (n + block - 1) / block;
    return (unsigned)(g > 148 * 16 ? 148 * 16 : (g ? g : 1));
}

extern "C" int rsa_battery_count(int test, const double* v, uint64_t n, uint32_t p1, uint32_t p2,
                                 unsigned long long* counts, int* flag, void* stream) {
    if (!v || !counts) return RSA_EINVAL;
    cudaStream_t st = as_stream(stream);
    switch (test) {
        case RSA_BT_HIST:  // n values, p1 = bins
            if (!p1) return RSA_EINVAL;
            k_hist<<<grid_cap(n, 256), 256, 0, st>>>(v, n, p1, counts);
            break;
        case RSA_BT_SERIAL:  // n tuples, p1 = d, p2 = axis bins
            if (p1 < 2 || p1 > 6 || !p2) return RSA_EINVAL;
            k_serial<<<grid_cap(n, 256), 256, 0, st>>>(v, n, (int)p1, p2, counts);
            break;
        case RSA_BT_POKER:  // n hands
            k_poker<<<grid_cap(n, 256), 256, 0, st>>>(v, n, counts);
            break;
        case RSA_BT_MAX_OF_T:  // n tuples, p1 = t, p2 = bins
            if (!p1 || !p2) return RSA_EINVAL;
            k_max_of_t<<<grid_cap(n, 256), 256, 0, st>>>(v, n, (int)p1, p2, counts);
            break;
        case RSA_BT_PERMUTATION:  // n tuples, p1 = t (<= 10)
            if (p1 < 2 || p1 > 10 || !flag) return RSA_EINVAL;
            k_permutation<<<grid_cap(n, 256), 256, 0, st>>>(v, n, (int)p1, counts, flag);
            break;
        case RSA_BT_COLLISION: {  // n trials, p1 = 0 top20bits / 1 msb_of_20
            if (p1 > 1) return RSA_EINVAL;
            const size_t smem = COLL_WORDS * sizeof(uint32_t);
            cudaError_t err = cudaFuncSetAttribute(k_collision, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (err != cudaSuccess) { set_last_error("rsa_battery_count(collision smem)", err); return RSA_ECUDA; }
            unsigned g = n < 148 * 2 ? (unsigned)n : 148 * 2;
            k_collision<<<g ? g : 1, 1024, smem, st>>>(v, (uint32_t)n, (int)p1, counts);
            break;
        }
        default:
            return RSA_EINVAL;
    }
    return launch_status("rsa_battery_count");
}
