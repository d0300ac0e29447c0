// Schedule search for the bulk-fill draw loop (tools only, not product code).
//
// k_var<E, V> is k_fill_fast<E, 2, false, 1> (paper_1811_11629_b200/csrc/fill.cu)
// with the same arithmetic (draw.cuh) in different statement orders, chosen
// by the bits of V; V = 0 is the production order.  Every variant's output is
// checked bit-for-bit against V = 0, then timed at config-2 size (Mv = 2^22,
// 256 blocks).  Bits:
//   1  lanes one after another (draw, float map) instead of both draws first
//   2  p2's exponent chain before p1's
//   4  block loop unrolled 2x (production: e = 5, 9) vs 1x
//   8  4-op double-double quotient (production: e = 3)
//  16  the next block's skip hoisted to the top of the loop body
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1811_11629_b200/csrc/draw.cuh"
using namespace rsa;

template <uint32_t E, int V>
RSA_DEV void tail_v(const FastInst& P, const Lane& L, uint32_t& h, uint32_t& c2) {
    if constexpr (V & 2) {
        uint32_t y2 = pow_e<E>(L.x2, P.e, P.p2, P.p2_inv);
        uint32_t y1 = pow_e<E>(L.x1, P.e, P.p1, P.p1_inv);
        c2 = mont_mul(y2, P.k2, P.p2, P.p2_inv);
        uint32_t c2r = min(c2, c2 - P.p1);
        uint64_t t = (uint64_t)y1 * P.gA + (uint64_t)c2r * P.gB;
        uint32_t m = (uint32_t)t * P.p1_inv;
        uint32_t u = __umulhi(m, P.p1);
        uint32_t th = (uint32_t)(t >> 32);
        uint32_t r = th - u;
        r = th < u ? r + P.p1 : r;
        h = min(r, r - P.p1);
    } else {
        draw_tail<E, true>(P, L, h, c2);
    }
}

template <uint32_t E, int V>
RSA_DEV double unit_v(const FastInst& P, uint64_t c) {
    if constexpr (V & 8) return to_unit_dd(c, P.n_float, P.n_recip, P.n_recip_lo);
    else return to_unit(c, P.n_float, P.n_recip);
}

template <uint32_t E, int V>
__global__ void __launch_bounds__(128)
k_var(const rsa_instance* __restrict__ inst, uint32_t mv, uint64_t blocks, uint64_t* __restrict__ m1,
      uint64_t* __restrict__ m2, uint64_t* __restrict__ s, double* __restrict__ f64) {
    const uint64_t lane = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (lane >= mv) return;
    const FastInst P = load_fast(inst);
    Lane L[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) L[j] = lane_in(P, m1[lane + j], m2[lane + j], s[lane + j]);
    uint64_t off = lane;
    constexpr int UNROLL = (V & 4) ? 2 : 1;
#pragma unroll UNROLL
    for (uint64_t k = 0; k < blocks; ++k, off += mv) {
        double r[2];
        if constexpr (V & 16) {
#pragma unroll
            for (int j = 0; j < 2; ++j) L[j].s = skip_q63(L[j].s, P.a);
        }
        if constexpr (V & 1) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if constexpr (!(V & 16)) L[j].s = skip_q63(L[j].s, P.a);
                L[j].x1 = msg_add(L[j].x1, L[j].s, P.p1, P.p1_inv);
                L[j].x2 = msg_add(L[j].x2, L[j].s, P.p2, P.p2_inv);
                uint32_t h, c2;
                tail_v<E, V>(P, L[j], h, c2);
                r[j] = unit_v<E, V>(P, (uint64_t)h * P.p2 + c2);
            }
        } else {
            uint64_t c[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if constexpr (!(V & 16)) L[j].s = skip_q63(L[j].s, P.a);
                L[j].x1 = msg_add(L[j].x1, L[j].s, P.p1, P.p1_inv);
                L[j].x2 = msg_add(L[j].x2, L[j].s, P.p2, P.p2_inv);
                uint32_t h, c2;
                tail_v<E, V>(P, L[j], h, c2);
                c[j] = (uint64_t)h * P.p2 + c2;
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) r[j] = unit_v<E, V>(P, c[j]);
        }
        __stcs(reinterpret_cast<double2*>(f64 + off), make_double2(r[0], r[1]));
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        m1[lane + j] = lane_m1(P, L[j]);
        m2[lane + j] = lane_m2(P, L[j]);
        s[lane + j] = L[j].s;
    }
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

struct Buf { uint64_t *m1, *m2, *s; };

template <uint32_t E, int V>
double run(const rsa_instance* d_inst, uint32_t mv, uint64_t blocks, const std::vector<uint64_t>& h1,
           const std::vector<uint64_t>& h2, const std::vector<uint64_t>& hs, Buf b, double* out, int reps) {
    cudaEvent_t a, z; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&z));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemcpy(b.m1, h1.data(), 8ull * mv, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(b.m2, h2.data(), 8ull * mv, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(b.s, hs.data(), 8ull * mv, cudaMemcpyHostToDevice));
        CK(cudaEventRecord(a));
        k_var<E, V><<<mv / 256, 128>>>(d_inst, mv, blocks, b.m1, b.m2, b.s, out);
        CK(cudaEventRecord(z)); CK(cudaEventSynchronize(z));
        float ms; CK(cudaEventElapsedTime(&ms, a, z)); if (ms < best) best = ms;
    }
    return best;
}

template <uint32_t E, int V>
void one(const rsa_instance* d_inst, uint32_t mv, uint64_t blocks, const std::vector<uint64_t>& h1,
         const std::vector<uint64_t>& h2, const std::vector<uint64_t>& hs, Buf b, double* out, double* ref,
         size_t n) {
    double ms = run<E, V>(d_inst, mv, blocks, h1, h2, hs, b, out, 4);
    // bit-exact against V = 0 on a 2^20-element prefix and the final state sum
    std::vector<double> x(1 << 20), y(1 << 20);
    CK(cudaMemcpy(x.data(), out, 8 << 20, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y.data(), ref, 8 << 20, cudaMemcpyDeviceToHost));
    bool same = memcmp(x.data(), y.data(), 8 << 20) == 0;
    CK(cudaMemcpy(x.data(), out + n - (1 << 20), 8 << 20, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y.data(), ref + n - (1 << 20), 8 << 20, cudaMemcpyDeviceToHost));
    same = same && memcmp(x.data(), y.data(), 8 << 20) == 0;
    printf("e=%-6u V=%2d  %.3f ms  %.2f G/s  %s\n", E, V, ms, (double)n / ms / 1e6, same ? "same" : "DIFF");
    fflush(stdout);
}

template <uint32_t E, int... Vs>
void sweep(const rsa_instance* d_inst, uint32_t mv, uint64_t blocks, const std::vector<uint64_t>& h1,
           const std::vector<uint64_t>& h2, const std::vector<uint64_t>& hs, Buf b, double* out, double* ref,
           size_t n) {
    run<E, 0>(d_inst, mv, blocks, h1, h2, hs, b, ref, 1);  // reference output
    (one<E, Vs>(d_inst, mv, blocks, h1, h2, hs, b, out, ref, n), ...);
    (one<E, Vs>(d_inst, mv, blocks, h1, h2, hs, b, out, ref, n), ...);  // second pass: drift check
}

int main(int argc, char** argv) {
    // instance: 128 bytes written by tools/variants/dump_instance.py (stream 0 of DEFAULT_MASTER_SEED)
    FILE* f = fopen(argc > 1 ? argv[1] : "tools/variants/inst_stream0.bin", "rb");
    if (!f) { printf("no instance file\n"); return 1; }
    rsa_instance hi; if (fread(&hi, sizeof hi, 1, f) != 1) return 1; fclose(f);
    const uint32_t mv = 1u << 22; const uint64_t blocks = 256; const size_t n = (size_t)mv * blocks;
    std::vector<uint64_t> h1(mv), h2(mv), hs(mv);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (uint32_t g = 0; g < mv; ++g) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17; h1[g] = x % hi.p1;
        x ^= x << 13; x ^= x >> 7; x ^= x << 17; h2[g] = x % hi.p2;
        x ^= x << 13; x ^= x >> 7; x ^= x << 17; hs[g] = 1 + x % (hi.q - 1);
    }
    rsa_instance* d_inst; CK(cudaMalloc(&d_inst, sizeof hi)); CK(cudaMemcpy(d_inst, &hi, sizeof hi, cudaMemcpyHostToDevice));
    Buf b; CK(cudaMalloc(&b.m1, 8ull * mv)); CK(cudaMalloc(&b.m2, 8ull * mv)); CK(cudaMalloc(&b.s, 8ull * mv));
    double *out, *ref; CK(cudaMalloc(&out, 8 * n)); CK(cudaMalloc(&ref, 8 * n));
    sweep<3, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 24, 25, 26, 27>(d_inst, mv, blocks, h1, h2, hs, b, out, ref, n);
    sweep<9, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>(d_inst, mv, blocks, h1, h2, hs, b, out, ref, n);
    return 0;
}
