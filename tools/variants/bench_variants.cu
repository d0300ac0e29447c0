// A/B harness for draw-path micro-variants (tools only, not product code).
// Compile with -DADD=0/1 -DSKIP=0/1 -DFL=0/1 -DDIV=0/1 -DCLAMP=0/1 -DLPT=1/2.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1811_11629_b200/csrc/modarith.cuh"
using namespace rsa;
#ifndef ADD
#define ADD 0
#endif
#ifndef SKIP
#define SKIP 0
#endif
#ifndef FL
#define FL 0
#endif
#ifndef DIV
#define DIV 0
#endif
#ifndef CLAMP
#define CLAMP 0
#endif
#ifndef LPT
#define LPT 2
#endif
#ifndef MINB
#define MINB 1
#endif

struct C {
    uint32_t p1, p2, i1, i2, a, k1, k2, g;
    double p2d, nf, nr, nl;
};

RSA_DEV uint32_t addv(uint32_t x, uint32_t t, uint32_t p) {
#if ADD
    uint32_t r = x + t;
    return r < t ? r - p : r;
#else
    return add_mod(x, t, p);
#endif
}

RSA_DEV uint64_t skipv(uint64_t s, uint32_t a) {
#if SKIP
    uint64_t A = (uint64_t)a * (uint32_t)(s >> 32);
    uint64_t B = (uint64_t)a * (uint32_t)s;
    uint32_t w0 = (uint32_t)B, w1, w2;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(w1), "=r"(w2)
        : "r"((uint32_t)A), "r"((uint32_t)(B >> 32)), "r"((uint32_t)(A >> 32)));
    uint32_t H = __funnelshift_l(w1, w2, 1);
    uint64_t L = ((uint64_t)(w1 & 0x7FFFFFFFu) << 32) | w0;
    uint64_t r = L + (uint64_t)H * 25u;
    uint64_t t = r + 25u;
    return (t >> 63) ? (t & 0x7FFFFFFFFFFFFFFFull) : r;
#else
    return skip_q63(s, a);
#endif
}

RSA_DEV double divv(double x, const C& P) {
#if DIV
    double q = __fma_rn(x, P.nr, __dmul_rn(x, P.nl));
    double r = __fma_rn(-q, P.nf, x);
    return __fma_rn(r, P.nr, q);
#else
    double q = __dmul_rn(x, P.nr);
    double r = __fma_rn(-q, P.nf, x);
    q = __fma_rn(r, P.nr, q);
    r = __fma_rn(-q, P.nf, x);
    return __fma_rn(r, P.nr, q);
#endif
}

RSA_DEV double clampv(double q) {
#if CLAMP
    return __double2hiint(q) >= 0x3FF00000 ? MAX_BELOW_ONE : q;
#else
    return q < 1.0 ? q : MAX_BELOW_ONE;
#endif
}

template <uint32_t E>
RSA_DEV double draw(const C& P, uint64_t& s, uint32_t& x1, uint32_t& x2) {
    s = skipv(s, P.a);
    x1 = addv(x1, mont_redc(s, P.p1, P.i1), P.p1);
    x2 = addv(x2, mont_redc(s, P.p2, P.i2), P.p2);
    uint32_t y1 = Chain<E>::pow(x1, P.p1, P.i1), y2 = Chain<E>::pow(x2, P.p2, P.i2);
    uint32_t c1 = mont_mul(y1, P.k1, P.p1, P.i1), c2 = mont_mul(y2, P.k2, P.p2, P.i2);
    uint32_t c2r = c2 >= P.p1 ? c2 - P.p1 : c2;
    uint32_t h = mont_mul(sub_mod(c1, c2r, P.p1), P.g, P.p1, P.i1);
#if FL
    double x = __fma_rn((double)h, P.p2d, (double)c2);
#else
    double x = __ull2double_rn((uint64_t)h * P.p2 + c2);
#endif
    return clampv(divv(x, P));
}

template <uint32_t E>
__global__ void __launch_bounds__(256, MINB) k(C P, uint32_t mv, uint64_t blocks, uint64_t* s_, uint32_t* m1_,
                                         uint32_t* m2_, double* out) {
    uint64_t lane = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * LPT;
    uint64_t s[LPT];
    uint32_t x1[LPT], x2[LPT];
#pragma unroll
    for (int j = 0; j < LPT; ++j) { s[j] = s_[lane + j]; x1[j] = m1_[lane + j]; x2[j] = m2_[lane + j]; }
    uint64_t off = lane;
    for (uint64_t b = 0; b < blocks; ++b, off += mv) {
        double r[LPT];
#pragma unroll
        for (int j = 0; j < LPT; ++j) r[j] = draw<E>(P, s[j], x1[j], x2[j]);
        if constexpr (LPT == 2) __stcs(reinterpret_cast<double2*>(out + off), make_double2(r[0], r[1]));
        else if constexpr (LPT == 4) {
            __stcs(reinterpret_cast<double2*>(out + off), make_double2(r[0], r[1]));
            __stcs(reinterpret_cast<double2*>(out + off + 2), make_double2(r[2], r[3]));
        } else __stcs(out + off, r[0]);
    }
#pragma unroll
    for (int j = 0; j < LPT; ++j) { s_[lane + j] = s[j]; m1_[lane + j] = x1[j]; m2_[lane + j] = x2[j]; }
}

__global__ void kx(const uint64_t* o, uint64_t n, unsigned long long* acc) {
    uint64_t v = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v ^= o[i] * (i | 1);
    atomicXor(acc, (unsigned long long)v);
}

typedef unsigned __int128 u128;
static uint64_t pw(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m; b %= m;
    while (e) { if (e & 1) r = (u128)r * b % m; b = (u128)b * b % m; e >>= 1; }
    return r;
}
static uint32_t inv32h(uint32_t p) { uint32_t x = p; for (int i = 0; i < 5; ++i) x *= 2u - p * x; return x; }

int main() {
    const uint32_t p1 = 2663418827u, p2 = 3462982283u, a = 2983799827u;
    const uint64_t R = 1ull << 32;
    const uint32_t MV = 1 << 22;
    const uint64_t BLOCKS = 64;
    C P;
    P.p1 = p1; P.p2 = p2; P.i1 = inv32h(p1); P.i2 = inv32h(p2); P.a = a;
    uint64_t p2inv = pw(p2, p1 - 2, p1);
    P.g = (uint32_t)((u128)p2inv * R % p1);
    P.p2d = p2;
    uint64_t n = (uint64_t)p1 * p2;
    P.nf = (double)n; P.nr = 1.0 / P.nf;
    P.nl = (1.0 - P.nf * P.nr) * P.nr;  // host approximation (same formula as the device, fma-contracted or not)
    {
        // exact residual via fma
        P.nl = __builtin_fma(-P.nf, P.nr, 1.0) * P.nr;
    }
    uint64_t *s; uint32_t *m1, *m2; double* out; unsigned long long* acc;
    cudaMalloc(&s, MV * 8); cudaMalloc(&m1, MV * 4); cudaMalloc(&m2, MV * 4);
    cudaMalloc(&out, (size_t)MV * BLOCKS * 8); cudaMalloc(&acc, 8);
    uint64_t* hs = new uint64_t[MV];
    uint32_t* hz = new uint32_t[MV];
    for (uint32_t g = 0; g < MV; ++g) { hs[g] = 1 + (uint64_t)g * 2654435761ull % ((1ull << 63) - 26); hz[g] = g % 1000; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (uint32_t E : {3u, 65537u}) {
        P.k1 = (uint32_t)pw(R % p1, 2 * E, p1); P.k2 = (uint32_t)pw(R % p2, 2 * E, p2);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaMemcpy(s, hs, MV * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(m1, hz, MV * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(m2, hz, MV * 4, cudaMemcpyHostToDevice);
            cudaEventRecord(e0);
            if (E == 3) k<3><<<MV / LPT / 256, 256>>>(P, MV, BLOCKS, s, m1, m2, out);
            else k<65537><<<MV / LPT / 256, 256>>>(P, MV, BLOCKS, s, m1, m2, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        cudaMemset(acc, 0, 8);
        kx<<<1184, 256>>>((const uint64_t*)out, (uint64_t)MV * BLOCKS, acc);
        unsigned long long h; cudaMemcpy(&h, acc, 8, cudaMemcpyDeviceToHost);
        double clk = best * 1e-3 * 1.965e9 * 148 / ((double)MV * BLOCKS);
        printf("MINB=%d ADD=%d SKIP=%d FL=%d DIV=%d CLAMP=%d LPT=%d  e=%-6u %8.3f ms  %.3f SM-clk/draw  chk=%016llx\n",
               MINB, ADD, SKIP, FL, DIV, CLAMP, LPT, E, best, clk, h);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
