/* c_abi_stream0.c — the whole hot path through the C ABI alone (no Python):
 * safe-prime scan of [2^31, 2^32) (K3), bucket index, the derivation of
 * stream 0 of the default master seed (K4), lane seeding and four draws of the
 * scalar stream (K1).  Prints p1 p2 a and the four raw ciphertexts — the
 * reference's pinned regression vector (test_acceptance.py:22-29) — which
 * tests/test_gpu_integration.py checks.
 *
 *   gcc -O2 -Iinclude examples/c_abi_stream0.c -o /tmp/c_abi_stream0 \
 *       -Lpaper_1811_11629_b200 -lrsarand_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1811_11629_b200:/usr/local/cuda/lib64
 *
 * Constants are the reference's published ones (paramfactory.py:24-48,
 * skipgen.py:20-47). */
#include <cuda_runtime.h>
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>

#include "rsarand_b200.h"

#define CHECK(x)                                                              \
    do {                                                                      \
        int rc_ = (x);                                                        \
        if (rc_) {                                                            \
            fprintf(stderr, "%s -> %d (%s)\n", #x, rc_, rsa_last_error());    \
            return 1;                                                         \
        }                                                                     \
    } while (0)
#define CUDA(x)                                                               \
    do {                                                                      \
        cudaError_t e_ = (x);                                                 \
        if (e_ != cudaSuccess) {                                              \
            fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));        \
            return 1;                                                         \
        }                                                                     \
    } while (0)

static const uint32_t MULT[16] = {2358014131u, 3027930091u, 2663770345u, 2989232495u,
                                  2966714411u, 2517859571u, 2584241481u, 2831318399u,
                                  3001167565u, 2425226767u, 3003776879u, 2548386679u,
                                  2416530305u, 2983799827u, 2861425803u, 2203334683u};

int main(void) {
    const uint64_t lo = 1ull << 31, hi = 1ull << 32, cap = 3100000;
    const uint64_t Q = (1ull << 63) - 25, SEED = 0x243F6A8885A308D3ull;
    const uint64_t K_P1 = 1291831, K_P2 = 1768937, SIGMA = 35705744587ull;
    const uint64_t P1_HI = 3037000500ull;  /* p1 window (2^31, floor(sqrt(q))] */

    /* K3: every safe prime of [2^31, 2^32), then its bucket index */
    uint64_t nb = rsa_safe_prime_scan_scratch_bytes(lo, hi);
    void *scratch;
    uint32_t *sp, *idx;
    uint64_t *dcount, n_sp;
    CUDA(cudaMalloc(&scratch, nb));
    CUDA(cudaMalloc((void**)&sp, cap * 4));
    CUDA(cudaMalloc((void**)&dcount, 8));
    CUDA(cudaMalloc((void**)&idx, RSA_SP_INDEX_LEN * 4));
    CHECK(rsa_safe_prime_scan(lo, hi, sp, cap, dcount, scratch, nb, 0));
    CUDA(cudaMemcpy(&n_sp, dcount, 8, cudaMemcpyDeviceToHost));
    CHECK(rsa_safe_prime_index(sp, n_sp, idx, 0));
    uint32_t *hsp = (uint32_t*)malloc(n_sp * 4);
    CUDA(cudaMemcpy(hsp, sp, n_sp * 4, cudaMemcpyDeviceToHost));
    uint64_t n_p1 = 0;
    while (n_p1 < n_sp && hsp[n_p1] < P1_HI) ++n_p1;

    /* K4: stream 0 of the default master seed */
    uint32_t *dmult, *dstep;
    int32_t* dstatus;
    rsa_instance* dinst;
    CUDA(cudaMalloc((void**)&dmult, sizeof MULT));
    CUDA(cudaMemcpy(dmult, MULT, sizeof MULT, cudaMemcpyHostToDevice));
    CUDA(cudaMalloc((void**)&dinst, sizeof(rsa_instance)));
    CUDA(cudaMalloc((void**)&dstatus, 4));
    CUDA(cudaMalloc((void**)&dstep, 4));
    rsa_setup_config cfg = {0};
    const uint64_t S = K_P1 * K_P2 * 16;
    cfg.seed_mod_S = SEED % S;
    cfg.first_id = 0;
    cfg.sigma = SIGMA;
    cfg.k_p1 = K_P1;
    cfg.k_p2 = K_P2;
    cfg.q = Q;
    cfg.tol = 9223372036854ull; /* floor(1e-6 * q) */
    cfg.epsilon = 7;
    cfg.e = 9;
    cfg.n_mult = 16;
    cfg.multiplier = 0;
    cfg.max_steps = 256;
    cfg.start_step = 0;
    CHECK(rsa_setup_instances(&cfg, 1, dmult, sp, n_sp, idx, sp, n_p1, dinst, dstatus, dstep, 0));
    int32_t status;
    rsa_instance inst;
    CUDA(cudaMemcpy(&status, dstatus, 4, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(&inst, dinst, sizeof inst, cudaMemcpyDeviceToHost));
    if (status) { fprintf(stderr, "derivation failed: %d\n", status); return 1; }

    /* K1: seed the lane (m0 = 0, s0 = 1) and draw four ciphertexts */
    uint64_t *m1, *m2, *s, *raw, hraw[4];
    CUDA(cudaMalloc((void**)&m1, 8));
    CUDA(cudaMalloc((void**)&m2, 8));
    CUDA(cudaMalloc((void**)&s, 8));
    CUDA(cudaMalloc((void**)&raw, 4 * 8));
    CHECK(rsa_init_lanes(dinst, 1, 1, 0, 0, 1, m1, m2, s, 0));
    CHECK(rsa_fill(dinst, 1, 1, 4, inst.e, inst.flags, m1, m2, s, raw, NULL, 4, 0));
    CUDA(cudaMemcpy(hraw, raw, sizeof hraw, cudaMemcpyDeviceToHost));
    printf("%" PRIu64 " %u %u %u\n", n_sp, inst.p1, inst.p2, inst.a);
    for (int i = 0; i < 4; ++i) printf("%" PRIu64 "\n", hraw[i]);
    return 0;
}
