// Shared device helpers for the cachecraft_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cachecraft_b200.h"

namespace ccb {

// ---- error plumbing (thread-local last message, see cc_last_error) --------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

#define CCB_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) return ::ccb::fail(CC_E_ARG, msg); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- scalar conversions --------------------------------------------------
template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ double to_f(double x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_f<double>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <typename T> __device__ __forceinline__ T from_d(double x);
template <> __device__ __forceinline__ float from_d<float>(double x) { return (float)x; }
template <> __device__ __forceinline__ double from_d<double>(double x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double x) { return __float2bfloat16_rn((float)x); }

// cos/sin pair type of the RoPE table: double2 in fp64 mode, float2 otherwise
template <typename T> struct CS { using type = float2; };
template <> struct CS<double> { using type = double2; };

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * x * (1.f + tanhf(k0 * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ double gelu_tanh(double x) {
  const double k0 = 0.7978845608028654;
  return 0.5 * x * (1.0 + tanh(k0 * (x + 0.044715 * x * x * x)));
}
// (fast reciprocal division: the IEEE x / y slow path dominated the GEMM epilogues)
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.f + __expf(-x)); }
__device__ __forceinline__ double silu(double x) { return x / (1.0 + exp(-x)); }

// RoPE rotation of one pair (x, y) by (cos, sin) in fp32 with a fixed FMA
// order, shared by every kernel that rotates fresh rows (rope_scatter, the
// fused QKV epilogue) so they produce the same bits
__device__ __forceinline__ void rope_pair(float a, float b, float c, float s, float& xr, float& yr) {
  xr = __fmaf_rn(a, c, -__fmul_rn(b, s));
  yr = __fmaf_rn(a, s, __fmul_rn(b, c));
}

// ---- dtype dispatch -------------------------------------------------------
#define CCB_DISPATCH_DTYPE(dtype, T, ...)                         \
  [&]() -> int {                                                  \
    switch (dtype) {                                              \
      case CC_F64: { using T = double; return __VA_ARGS__(); }    \
      case CC_F32: { using T = float; return __VA_ARGS__(); }     \
      case CC_BF16: { using T = __nv_bfloat16; return __VA_ARGS__(); } \
      default: return ::ccb::fail(CC_E_ARG, "unknown dtype");     \
    }                                                             \
  }()

inline size_t dtype_size(int dtype) { return dtype == CC_F64 ? 8 : (dtype == CC_F32 ? 4 : 2); }

int num_sms();
void note_simt(int dtype);  // counts bf16 SIMT launches (cc_bf16_simt_launches)
// scratch tags: one per kernel family, so no two families share a buffer
enum ScratchTag { SCR_LOGITS = 1, SCR_SEGMASS = 2, SCR_ATTN = 3, SCR_DECODE_ATTN = 4, SCR_PAIR_KSPLIT = 5 };
// zero-initialised buffers (decode.cu): tickets the kernels reset themselves
enum ZeroedTag { ZSCR_GEMV_SEAMS = 1, ZSCR_DECODE_TICKETS = 2, ZSCR_PAIR_TICKETS = 3 };
void* zeroed_scratch(cudaStream_t st, int tag, size_t bytes);
void* stream_scratch(cudaStream_t st, int tag, size_t bytes);

// Dynamic shared-memory opt-in, once per (device, kernel): thread-safe, and
// correct when one process drives several GPUs (a function attribute is
// per-device state).
int set_smem_attr(const void* fn, int bytes);
template <typename... KArgs>
inline int ensure_smem(void (*fn)(KArgs...), size_t bytes) {
  return set_smem_attr(reinterpret_cast<const void*>(fn), (int)bytes);
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels of the decode chain call pdl_trigger() first (the next kernel may be
// scheduled now) and pdl_wait() before reading anything a predecessor wrote;
// their independent prologue (weight streaming) overlaps the predecessor's
// tail.  Both are no-ops for a kernel launched without the PDL attribute.
extern int g_pdl;  // cc_set_pdl
extern int g_stream_k;  // cc_set_stream_k
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
int launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const char* what,
             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (g_pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return fail(CC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

}  // namespace ccb
