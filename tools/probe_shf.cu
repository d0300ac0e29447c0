// Throughput probe: 64-bit funnel shift (SHF.R.U64), 32-bit funnel shift
// (SHF.L.W.U32.HI), signed / unsigned ISETP+SEL, LOP3 — which ALU forms are
// full rate on B200.  Not product code (profiles/r02s_stalls_by_opcode.txt).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
template <int K>
__global__ void k(uint32_t* out, uint32_t a) {
  uint32_t x[CH], y[CH];
  for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 77 + i; y[i] = threadIdx.x ^ (i * 31); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (K == 0) { uint64_t t = ((uint64_t)y[i] << 32) | x[i]; x[i] = (uint32_t)(t >> 31) ^ a; }       // SHF.R.U64
      if (K == 1) { x[i] = __funnelshift_l(x[i], y[i], 1) ^ a; }                                      // SHF.L.W
      if (K == 2) { x[i] = ((int32_t)x[i] >= 0 ? x[i] : y[i]) + a; }                                   // signed ISETP + SEL
      if (K == 3) { x[i] = (x[i] >= y[i] ? x[i] : y[i]) + a; }                                         // unsigned
      if (K == 4) { x[i] = (x[i] ^ y[i]) + a; }                                                        // LOP3 + VIADD
      if (K == 5) { x[i] = x[i] + y[i]; y[i] = y[i] + x[i]; }                                          // R + R adds
      if (K == 6) { x[i] = x[i] - y[i]; y[i] = y[i] - x[i]; }                                          // R - R
      if (K == 7) { x[i] = x[i] + y[i] + a * i; y[i] = y[i] - x[i] + 7; }                               // 3-input
      if (K == 8) { uint32_t r = x[i] - y[i]; x[i] = x[i] < y[i] ? r + a : r; y[i] ^= x[i]; }           // Montgomery-style fix
      if (K == 9) { x[i] = min(x[i], y[i]); y[i] = max(y[i] ^ a, x[i]); }                              // VIMNMX
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < CH; ++i) s ^= x[i] ^ y[i];
  if (s == 0x12345) out[0] = s;
}
template <int K> float run(uint32_t* o) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<K><<<148 * 8, 256>>>(o, 3); cudaDeviceSynchronize();
  cudaEventRecord(a); k<K><<<148 * 8, 256>>>(o, 3); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  uint32_t* o; cudaMalloc(&o, 4);
  const char* names[] = {"shf.r.u64+lop", "shf.l.w.u32+lop", "isetp.s32+sel+iadd", "isetp.u32+sel+iadd", "lop3+iadd3",
                         "add r+r (x2)", "sub r-r (x2)", "3-input adds (x2)", "mont fix + lop", "min/max(x2)"};
  float t[10] = {run<0>(o), run<1>(o), run<2>(o), run<3>(o), run<4>(o), run<5>(o), run<6>(o), run<7>(o), run<8>(o), run<9>(o)};
  double ops = 148.0 * 8 * 256 * ITERS * CH;
  for (int i = 0; i < 10; ++i) printf("%-22s %.3f ms  %.2f G elements/s  %.1f per clk per SM @1.965\n", names[i], t[i], ops / t[i] / 1e6, ops / (t[i] * 1e-3) / 148 / 1.965e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
