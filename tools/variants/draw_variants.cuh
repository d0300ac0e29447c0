// draw_variants.cuh — measured-and-rejected A/B variants of the draw path,
// kept for reproducibility (tools only; the product kernels include none of
// this).  Results: profiles/r01_ab_msg_fl.txt, r01_ab_v1_v3.txt.
//
//   msg_add_carry    carry-flag message add (was RSA_MSG_VARIANT=1 in draw.cuh):
//                    -5 heavy slots per 2 draws at e=3, measured 2 % slower
//   fl_from_hc       fl(c) = RN(h*p2 + c2) as one FMA of exact operands (was
//                    RSA_FL_FMA in draw.cuh / fill.cu): a second I2F per draw on
//                    the XU pipe, measured 1-3 % slower
//   div_rn_dd        4-op correctly rounded quotient from a double-double
//                    reciprocal y + y_lo (was rsa_instance.n_recip_lo): 3.7 %
//                    slower at e=65537
//   hist32 bump      u32 shared-memory atomics for the fused histogram (was
//                    RSA_FUSED_HIST32 in fused.cu): +0.1 %, twice the smem
#pragma once
#include "../../paper_1811_11629_b200/csrc/modarith.cuh"

namespace rsa_variants {
using namespace rsa;

RSA_DEV uint32_t msg_add_carry(uint32_t x, uint64_t s, uint32_t p, uint32_t pinv) {
    uint32_t y = mont_redc(s, p, pinv);
    uint32_t r, c;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(r), "=r"(c) : "r"(x), "r"(y));
    return (c | (uint32_t)(r >= p)) ? r - p : r;
}

RSA_DEV double fl_from_hc(uint32_t h, uint32_t c2, double p2d) {
    return __fma_rn((double)h, p2d, (double)c2);
}

// y_lo = RN(RN(1 - N*y) * y): 1/N ~ y + y_lo
RSA_DEV double div_rn_dd(double x, double N, double y, double y_lo) {
    double q = __dmul_rn(x, y);
    double r = __fma_rn(-q, N, x);
    q = __fma_rn(r, y, __fma_rn(x, y_lo, q));
    r = __fma_rn(-q, N, x);
    return __fma_rn(r, y, q);
}

RSA_DEV void hist32_bump(uint32_t* p) { atomicAdd(p, 1u); }

}  // namespace rsa_variants
