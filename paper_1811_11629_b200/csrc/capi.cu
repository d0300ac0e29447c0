// capi.cu — library identity and error reporting for the C ABI.
#include <stdio.h>
#include <atomic>
#include "common.cuh"

namespace rsa {

static thread_local char g_last_error[256] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_last_error(const char* what, cudaError_t err) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%d)", what, cudaGetErrorString(err), (int)err);
}

}  // namespace rsa

extern "C" int rsa_abi_version(void) { return RSA_ABI_VERSION; }

extern "C" int rsa_built_arch(void) { return 100; }

extern "C" const char* rsa_last_error(void) { return rsa::g_last_error; }

extern "C" uint64_t rsa_launch_count(void) { return rsa::g_launches.load(std::memory_order_relaxed); }
