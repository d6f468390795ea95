// rsr_capi.cu -- library-level C ABI entry points (version, error reporting).
#include <string.h>

#include "rsr_common.cuh"

namespace rsr {
static thread_local char g_last_error[256] = "";

void set_cuda_error(cudaError_t e) {
    strncpy(g_last_error, cudaGetErrorString(e), sizeof(g_last_error) - 1);
    g_last_error[sizeof(g_last_error) - 1] = '\0';
}
}  // namespace rsr

extern "C" {

const char *rsr_version(void) { return "rsr_b200 0.1.0 sm_100a"; }

const char *rsr_last_cuda_error(void) { return rsr::g_last_error; }

int rsr_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return n;
}

}  // extern "C"
