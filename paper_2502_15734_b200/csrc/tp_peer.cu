// Tensor-parallel reduction of the o_proj / down_proj partial outputs over
// peer memory (SURVEY §8e; model.py:417, :419), the B200-native alternative
// to an NCCL all-reduce after the GEMM:
//   1. cc_tp_push_gemm: the tcgen05 GEMM epilogue stores each fp32 tile into
//      its column owner's receive slab (P2P stores over NVLink) and stamps it
//      -> the reduce-scatter traffic overlaps the GEMM tile by tile;
//   2. tp_reduce_kernel (owner): per owned tile wait for all ranks' stamps,
//      sum the partials in rank order (deterministic; every rank ends with the
//      same bits), store the sum into every rank's `sum` buffer (all-gather)
//      and bump their `done` counters;
//   3. tp_wait_kernel: stream-ordered wait on this rank's `done` counter.
// The residual add (hidden += sum) is cc_add_f32 on the local stream.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "gemm.cuh"

namespace ccb {
namespace {

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) tp_reduce_kernel(const PeerTab tab, int M, int bn, int num_m) {
  const int per = tab.slice / bn;
  const int tile = blockIdx.x;  // local tile of my slice: (mt, lt)
  const int mt = tile / per, lt = tile % per;
  const int tiles_mine = num_m * per;
  if (threadIdx.x < tab.world) {  // one waiter per source rank
    const int* f = tab.flags[tab.rank] + (int64_t)threadIdx.x * tiles_mine + tile;
    while (ld_acquire_sys(f) != tab.epoch) __nanosleep(100);
  }
  __syncthreads();
  const float* recv = tab.recv[tab.rank];
  const int d = tab.slice * tab.world;
  const int q4 = bn / 4;
  for (int idx = threadIdx.x; idx < 128 * q4; idx += blockDim.x) {
    const int r = idx / q4, c = (idx % q4) * 4;
    const int row = mt * 128 + r;
    if (row >= M) continue;
    const int lc = lt * bn + c;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int src = 0; src < tab.world; ++src) {  // fixed rank order
      const float4 p = __ldcv(reinterpret_cast<const float4*>(recv + ((int64_t)src * tab.m_cap + row) * tab.slice + lc));
      s.x += p.x; s.y += p.y; s.z += p.z; s.w += p.w;
    }
    const int64_t off = (int64_t)row * d + tab.rank * tab.slice + lc;
    for (int dst = 0; dst < tab.world; ++dst) *reinterpret_cast<float4*>(tab.sum[dst] + off) = s;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < tab.world)
    asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(tab.done[threadIdx.x]) : "memory");
}

__global__ void tp_wait_kernel(const int* done, long long target) {
  while ((long long)ld_acquire_sys(done) < target) __nanosleep(200);
}

int tab_ok(const PeerTab* t) {
  if (!t || t->world < 1 || t->world > TP_MAX || t->rank < 0 || t->rank >= t->world || t->slice <= 0 || t->m_cap <= 0)
    return fail(CC_E_ARG, "tp: bad peer table");
  return 0;
}

}  // namespace
}  // namespace ccb

using namespace ccb;

extern "C" int cc_tp_push_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                               const cc_tp_peers* tab, void* stream) {
  if (int rc = tab_ok(tab)) return rc;
  CCB_REQUIRE(M >= 0 && M <= tab->m_cap, "tp_push_gemm: rows exceed the peer buffers");
  if (M == 0) return 0;
  return gemm_tc_peer_push(A, lda, B, ldb, M, N, K, *tab, as_stream(stream));
}

extern "C" int cc_tp_reduce(const cc_tp_peers* tab, int M, int N, void* stream) {
  if (int rc = tab_ok(tab)) return rc;
  CCB_REQUIRE(N == tab->slice * tab->world && M <= tab->m_cap, "tp_reduce: shape != peer table");
  if (M == 0) return 0;
  const int bn = tab->slice % 256 == 0 ? 256 : 128;
  const int num_m = (M + 127) / 128;
  tp_reduce_kernel<<<num_m * (tab->slice / bn), 256, 0, as_stream(stream)>>>(*tab, M, bn, num_m);
  return check_launch("tp_reduce");
}

extern "C" int cc_tp_wait(const cc_tp_peers* tab, int64_t target, void* stream) {
  if (int rc = tab_ok(tab)) return rc;
  tp_wait_kernel<<<1, 1, 0, as_stream(stream)>>>(tab->done[tab->rank], (long long)target);
  return check_launch("tp_wait");
}

// An IPC handle names the whole allocation a pointer lies in (a caching
// allocator hands out sub-ranges of larger cudaMalloc blocks): *offset gets
// the pointer's byte offset from that allocation's base, which the peer adds
// to the base cudaIpcOpenMemHandle returns.
extern "C" int cc_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset) {
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<RangeFn>(p);
  });
  if (!range) return fail(CC_E_CUDA, "ipc_get_handle: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(CC_E_CUDA, "ipc_get_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string("ipc_get_handle: ") + cudaGetErrorString(e));
  memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return 0;
}

extern "C" int cc_ipc_open_handle(const void* handle64, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string("ipc_open_handle: ") + cudaGetErrorString(e));
  return 0;
}
