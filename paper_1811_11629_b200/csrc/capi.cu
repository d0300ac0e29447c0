// capi.cu — library identity and error reporting for the C ABI.
#include <stdio.h>
#include "common.cuh"

namespace rsa {

static thread_local char g_last_error[256] = "";

void set_last_error(const char* what, cudaError_t err) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%d)", what, cudaGetErrorString(err), (int)err);
}

}  // namespace rsa

extern "C" int rsa_abi_version(void) { return RSA_ABI_VERSION; }

extern "C" int rsa_built_arch(void) { return 100; }

extern "C" const char* rsa_last_error(void) { return rsa::g_last_error; }
