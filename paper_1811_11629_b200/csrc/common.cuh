// common.cuh — launch/error plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/rsarand_b200.h"

namespace rsa {

void set_last_error(const char* what, cudaError_t err);
void count_launches(uint64_t n);  // capi.cu: process-wide count of kernel launches (rsa_launch_count)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Report the launch status of the n kernels just issued (configuration errors
// and sticky faults from earlier work) and count them; never synchronises.
inline int launch_status(const char* what, uint64_t n = 1) {
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        set_last_error(what, err);
        return RSA_ECUDA;
    }
    count_launches(n);
    return RSA_OK;
}

inline unsigned grid_for(uint64_t threads, unsigned block) {
    return (unsigned)((threads + block - 1) / block);
}

// One-thread-per-item launches must fit the 2^31 - 1 grid.x limit.
inline bool grid_fits(uint64_t threads, unsigned block) {
    return (threads + block - 1) / block <= 0x7FFFFFFFull;
}

}  // namespace rsa
