// Error plumbing and device queries of the C ABI (include/cachecraft_b200.h).
#include <mutex>
#include <string>

#include "common.cuh"

namespace ccb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace ccb

extern "C" {

int cc_abi_version(void) { return CC_ABI_VERSION; }

const char* cc_last_error(void) { return ccb::g_last_error.c_str(); }

int cc_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return ccb::fail(CC_E_CUDA, "cudaDeviceGetAttribute failed");
  return v;
}

}  // extern "C"
