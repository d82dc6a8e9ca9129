// Error plumbing and device queries of the C ABI (include/cachecraft_b200.h).
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace ccb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int g_pdl = 0;
int g_stream_k = 1;

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
// never share it.  Grows on demand.  A grown-out buffer is retired, never
// freed: a captured CUDA graph (DecodeSession) may still reference it, and
// cudaFree would synchronise the device.
void* stream_scratch(cudaStream_t st, int tag, size_t bytes) {
  static std::mutex mu;
  struct Buf { void* p = nullptr; size_t n = 0; };
  static std::unordered_map<uint64_t, Buf> bufs;
  static std::vector<void*> retired;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(st) * 1315423911ull) ^ ((uint64_t)dev << 56) ^ (uint64_t)tag;
  std::lock_guard<std::mutex> g(mu);
  Buf& b = bufs[key];
  if (b.n < bytes) {
    if (b.p) retired.push_back(b.p);
    b.p = nullptr;
    // grow geometrically so a slowly growing request retires few buffers
    size_t want = std::max(bytes, b.n * 2);
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
      b.p = nullptr;
      if (cudaMalloc(&b.p, bytes) != cudaSuccess) { b.n = 0; return nullptr; }
      want = bytes;
    }
    b.n = want;
  }
  return b.p;
}

int set_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  // the attribute is an upper bound: only ever raised, so a kernel launched
  // with several shared-memory sizes keeps the largest one requested
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  int& cur = done[std::make_pair(dev, fn)];
  if (bytes <= cur) return 0;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  cur = bytes;
  return 0;
}

static std::atomic<long long> g_bf16_simt{0};
void note_simt(int dtype) {
  if (dtype == CC_BF16) g_bf16_simt.fetch_add(1, std::memory_order_relaxed);
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

int cc_set_stream_k(int on) {
  const int prev = ccb::g_stream_k;
  ccb::g_stream_k = on ? 1 : 0;
  return prev;
}

int cc_set_pdl(int on) {
  const int prev = ccb::g_pdl;
  ccb::g_pdl = on ? 1 : 0;
  return prev;
}

const char* cc_last_error(void) { return ccb::g_last_error.c_str(); }

long long cc_bf16_simt_launches(void) { return ccb::g_bf16_simt.load(); }

int cc_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return ccb::fail(CC_E_CUDA, "cudaDeviceGetAttribute failed");
  return v;
}

}  // extern "C"
