// Error plumbing and device queries of the C ABI (include/cachecraft_b200.h).
#include <mutex>
#include <unordered_map>
#include <string>

#include "common.cuh"

namespace ccb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int g_pdl = 0;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

// Device scratch owned by the library, one buffer per (device, stream, tag):
// kernels on different streams (e.g. tensor-parallel ranks in one process)
// never share it.  Grows on demand; never freed (process lifetime).
void* stream_scratch(cudaStream_t st, int tag, size_t bytes) {
  static std::mutex mu;
  struct Buf { void* p = nullptr; size_t n = 0; };
  static std::unordered_map<uint64_t, Buf> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(st) * 1315423911ull) ^ ((uint64_t)dev << 56) ^ (uint64_t)tag;
  std::lock_guard<std::mutex> g(mu);
  Buf& b = bufs[key];
  if (b.n < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) { b.n = 0; return nullptr; }
    b.n = bytes;
  }
  return b.p;
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

int cc_set_pdl(int on) {
  const int prev = ccb::g_pdl;
  ccb::g_pdl = on ? 1 : 0;
  return prev;
}

const char* cc_last_error(void) { return ccb::g_last_error.c_str(); }

int cc_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return ccb::fail(CC_E_CUDA, "cudaDeviceGetAttribute failed");
  return v;
}

}  // extern "C"
