// Pipe-sharing probe: a stream of Montgomery triples (IMAD.WIDE, IMAD,
// IMAD.HI: 5 heavy slots) with one extra select/add per product in different
// forms (SEL, FSEL, IADD3, VIADD imm, predicated add).  If the extra op runs
// on a pipe the triples do not use, the time stays at the triples' own.
// Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 1024
#define CH 8
template <int K>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CH], z[CH];
  for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 7919u + i * 104729u + blockIdx.x; z[i] = x[i] ^ 0x5555; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      uint64_t t = (uint64_t)x[i] * x[i];
      uint32_t m = (uint32_t)t * pinv;
      uint32_t u = __umulhi(m, p);
      uint32_t th = (uint32_t)(t >> 32);
      uint32_t r = th ^ u;                     // 1 LOP3 (ALU) in every variant
      bool c = th < u;                          // ISETP (ALU) in variants 1..5
      if (K == 1) r = c ? r : z[i];             // SEL
      if (K == 2) r = __float_as_uint(c ? __uint_as_float(r) : __uint_as_float(z[i]));  // FSEL?
      if (K == 3) r = r + z[i] + th;            // IADD3 (R+R+R)
      if (K == 4) r = r + 0x9E3779B9u;          // VIADD imm? (no ISETP use)
      if (K == 5) { if (c) r += 0x9E3779B9u; }  // predicated add
      x[i] = r;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 0x12345) out[0] = s;
}
template <int K> float run(uint32_t* o) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<K><<<148 * 8, 256>>>(o, 3462982283u, 3018205987u); cudaDeviceSynchronize();
  cudaEventRecord(a); k<K><<<148 * 8, 256>>>(o, 3462982283u, 3018205987u); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  uint32_t* o; cudaMalloc(&o, 4);
  const char* names[] = {"triple+lop3", "+isetp+SEL", "+isetp+FSEL", "+IADD3", "+VIADD imm", "+isetp+@p add"};
  float t[6] = {run<0>(o), run<1>(o), run<2>(o), run<3>(o), run<4>(o), run<5>(o)};
  double prods = 148.0 * 8 * 256 * ITERS * CH;
  for (int i = 0; i < 6; ++i) printf("%-16s %.3f ms  %.2f products/clk/SM  (%.1f heavy slots/clk/SM)\n", names[i], t[i],
                                     prods / (t[i] * 1e-3) / 148 / 1.965e9, 5 * prods / (t[i] * 1e-3) / 148 / 1.965e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
