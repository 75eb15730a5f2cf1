// api.cu — library-wide C ABI entry points (errors, version, device info).
#include "common.cuh"

namespace rfxc {
std::string& last_error()
{
    static thread_local std::string msg;
    return msg;
}
}  // namespace rfxc

extern "C" const char* rfxc_last_error(void) { return rfxc::last_error().c_str(); }

extern "C" int rfxc_version(void) { return 1; }

extern "C" int rfxc_device_info(int device, int* sm_count, int64_t* l2_bytes,
                                int64_t* smem_per_block_optin)
{
    int v = 0;
    cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return rfxc::fail(RFXC_ECUDA, "device_info: %s", cudaGetErrorString(e));
    if (sm_count) *sm_count = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
    if (l2_bytes) *l2_bytes = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (smem_per_block_optin) *smem_per_block_optin = v;
    return RFXC_OK;
}
