// Throughput probe for the integer / FP64 pipes the RSA-PRNG draw uses.
// Not product code: run once on a B200 to size the roofline denominators.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CH 8

__global__ void k_imad_lo(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = x[i] * a + b;
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_imad_wide(uint64_t* out, uint32_t a) {
  uint64_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = (uint64_t)(uint32_t)x[i] * a + x[i];
  }
  uint64_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_imad_hi(uint32_t* out, uint32_t a) {
  uint32_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i + 77;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __umulhi(x[i], a) + x[i];
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_iadd3(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = (x[i] ^ a) + b;  // LOP3 + IADD3 (or one LOP3/IADD3 pair)
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 0.12345) out[0] = s;
}

__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 0.12345f) out[0] = s;
}

// Montgomery product x*y*2^-32 mod p, p odd < 2^32, x,y < p; pinv = p^-1 mod 2^32.
__device__ __forceinline__ uint32_t mont(uint32_t x, uint32_t y, uint32_t p, uint32_t pinv) {
  uint64_t t = (uint64_t)x * y;
  uint32_t m = (uint32_t)t * pinv;
  uint32_t u = __umulhi(m, p);
  uint32_t th = (uint32_t)(t >> 32);
  uint32_t r = th - u;
  return th < u ? r + p : r;
}

__global__ void k_mont(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = (threadIdx.x * 7919u + i) % p;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = mont(x[i], x[i], p, pinv);
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

// Montgomery "triple" only (no conditional) - the SURVEY's peak stream.
__global__ void k_triple(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CH];
  for (int i = 0; i < CH; ++i) x[i] = (threadIdx.x * 7919u + i) % p;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      uint64_t t = (uint64_t)x[i] * x[i];
      uint32_t m = (uint32_t)t * pinv;
      uint64_t w = (uint64_t)m * p + t;  // IMAD.WIDE with 64-bit addend
      x[i] = (uint32_t)(w >> 32) ^ m;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_i2f_div(double* out, uint64_t base, double n) {
  double acc = 0;
  uint64_t c = base + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      acc += __ddiv_rn(__ull2double_rn(c + i * 12345u), n);
    }
    c += 0x9E3779B97F4A7C15ull;
  }
  if (acc == 0.12345) out[0] = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d clock(kHz) %d\n", prop.name, sms, prop.clockRate);
  void* buf; cudaMalloc(&buf, 64);
  for (int bpsm : {4, 8}) {
    int grid = sms * bpsm, block = 256;
    double ops = (double)grid * block * ITERS * CH;
    auto rep = [&](const char* name, float ms, double per) {
      double r = ops * per / (ms * 1e-3);
      printf("bpsm=%d %-12s %8.3f ms  %.3f Tops/s  %.1f /clk/SM@1.965GHz\n", bpsm, name, ms, r / 1e12,
             r / sms / 1.965e9);
    };
    rep("imad_lo", timeit([&] { k_imad_lo<<<grid, block>>>((uint32_t*)buf, 2654435761u, 12345u); }), 1);
    rep("imad_wide", timeit([&] { k_imad_wide<<<grid, block>>>((uint64_t*)buf, 2654435761u); }), 1);
    rep("imad_hi+add", timeit([&] { k_imad_hi<<<grid, block>>>((uint32_t*)buf, 2654435761u); }), 1);
    rep("lop+add", timeit([&] { k_iadd3<<<grid, block>>>((uint32_t*)buf, 0x5bd1e995u, 12345u); }), 1);
    rep("dfma", timeit([&] { k_dfma<<<grid, block>>>((double*)buf, 1.0000001, 1e-9); }), 1);
    rep("ffma", timeit([&] { k_ffma<<<grid, block>>>((float*)buf, 1.0000001f, 1e-9f); }), 1);
    rep("montmul", timeit([&] { k_mont<<<grid, block>>>((uint32_t*)buf, 3462982283u, 0u); }), 1);
    rep("mont_triple", timeit([&] { k_triple<<<grid, block>>>((uint32_t*)buf, 3462982283u, 0u); }), 1);
    rep("i2f+ddiv", timeit([&] { k_i2f_div<<<grid, block>>>((double*)buf, 123456789ull, 9.223372e18); }), 1);
  }
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
