// Decode-side kernels (greedy continuation on the repaired KV, model.py:445-484):
//   * gemv_kernel       bandwidth-bound projections for M <= 4 rows (weight
//                       streaming: one warp per output row, 16-byte
//                       no-allocate loads, 4 in flight per lane), with the
//                       GEMM epilogues (store / residual add / SwiGLU / GELU)
//   * decode_attn_*     split-KV attention of ONE query row over all keys:
//                       128-key chunks per CTA (one GQA group), fixed-order
//                       combine -> deterministic
//   * rope_rows_kernel  rotate stored position-free keys at their positions
//                       (rpe.py:19-44), once per decode session
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include <type_traits>

#include <mutex>
#include <set>
#include <unordered_map>

#include "common.cuh"
#include "sm100.cuh"

namespace ccb {

namespace {

using namespace sm100;

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float dot8(const uint4& w, const uint4& x) {
  const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&w);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&x);
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 fa = __bfloat1622float2(a[e]), fb = __bfloat1622float2(b[e]);
    s = fmaf(fa.x, fb.x, s);
    s = fmaf(fa.y, fb.y, s);
  }
  return s;
}

// ---- debug timeline of the decode chain (cc_debug_decode_trace) ---------------
// When armed, thread 0 of every CTA of the GEMV / fused-attention kernels
// appends {start, wait released, end, tag << 48 | smid << 32 | block} in
// %globaltimer ns; off (one predicated load) otherwise.
__device__ unsigned long long* g_dtrace = nullptr;
__device__ unsigned g_dtrace_cap = 0;
__device__ unsigned g_dtrace_n = 0;
// streaming GEMV: griddepcontrol.launch_dependents after the activation
// prologue (1, default) or right after the ring fills (0); CCB_GS_TRIGGER
__device__ int g_trigger_late = 1;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// (records are 8 x u64: start, released, end, tag|smid|block, checkpoints c1..c4 as offsets from released)
__device__ __forceinline__ void dtrace(unsigned tag, unsigned long long t0, unsigned long long t1,
                                       unsigned long long c1 = 0, unsigned long long c2 = 0,
                                       unsigned long long c3 = 0, unsigned long long c4 = 0) {
  unsigned long long* buf = g_dtrace;
  if (buf == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t2 = gtime();
    const unsigned i = atomicAdd(&g_dtrace_n, 1u);
    if (i < g_dtrace_cap) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      const unsigned blk = blockIdx.x + blockIdx.y * gridDim.x;
      buf[8 * i] = t0;
      buf[8 * i + 1] = t1;
      buf[8 * i + 2] = t2;
      buf[8 * i + 3] = ((unsigned long long)tag << 48) | ((unsigned long long)smid << 32) | blk;
      buf[8 * i + 4] = c1 ? c1 - t1 : 0;
      buf[8 * i + 5] = c2 ? c2 - t1 : 0;
      buf[8 * i + 6] = c3 ? c3 - t1 : 0;
      buf[8 * i + 7] = c4 ? c4 - t1 : 0;
    }
  }
}

constexpr int GV_MAXM = 4;
constexpr int GV_WARPS = 8;

// C[M, N] (+)= epi(A[M, K] W[N, K]^T); SwiGLU: W rows in 64-row gate/up groups,
// output column o = silu(gate row) * up row (N/2 outputs)
// NORM: A is the f32 residual stream; the prologue applies the weighted
// RMSNorm (model.py:121-122) and stages bf16(x * rsqrt(mean(x^2) + eps) * w)
// -- the rmsnorm kernel fused away (decode: one launch less per projection)
template <int EPI, bool NORM, int MR>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_kernel(const void* __restrict__ A_, int64_t lda,
                                                             const __nv_bfloat16* __restrict__ W, int64_t ldw,
                                                             void* __restrict__ C, int64_t ldc, int M, int N, int K,
                                                             const float* __restrict__ norm_w, float eps) {
  extern __shared__ uint4 xs[];  // [M][K / 8] staged activations
  const int kv8 = K / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool GLU = EPI == CC_EPI_SWIGLU;
  constexpr int B = 4;  // 16-byte weight loads in flight per lane (x2 for SwiGLU)
  const int n_out = GLU ? N / 2 : N;
  auto wrows = [&](int o, const uint4*& wg, const uint4*& wu) {
    const int rg = GLU ? (o / 64) * 128 + (o % 64) : o;
    wg = reinterpret_cast<const uint4*>(W + (int64_t)rg * ldw);
    wu = reinterpret_cast<const uint4*>(W + (int64_t)(rg + 64) * ldw);
  };
  const unsigned long long t0 = gtime();
  pdl_trigger();
  pdl_wait();  // activations come from the predecessor
  const unsigned long long t1 = gtime();
  if constexpr (NORM) {
    __shared__ float red[GV_WARPS];
    __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(xs);
    for (int r = 0; r < M; ++r) {
      const float4* x4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(A_) + (int64_t)r * lda);
      float ss = 0.f;
      for (int i = threadIdx.x; i < K / 4; i += blockDim.x) {
        const float4 v = x4[i];
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
      __syncthreads();
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < GV_WARPS; ++w) tot += red[w];
      const float inv = rsqrtf(tot / (float)K + eps);
      for (int i = threadIdx.x; i < K / 4; i += blockDim.x) {
        const float4 v = x4[i];
        float4 g = norm_w != nullptr ? reinterpret_cast<const float4*>(norm_w)[i] : make_float4(1.f, 1.f, 1.f, 1.f);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * g.x, v.y * inv * g.y);
        __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * g.z, v.w * inv * g.w);
        *reinterpret_cast<uint2*>(xb + (int64_t)r * K + 4 * i) =
            make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
      }
      __syncthreads();
    }
  } else {
    const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(A_);
    for (int r = 0; r < M; ++r)
      for (int i = threadIdx.x; i < kv8; i += blockDim.x)
        xs[r * kv8 + i] = reinterpret_cast<const uint4*>(A + (int64_t)r * lda)[i];
    __syncthreads();
  }
  for (int o = blockIdx.x * GV_WARPS + warp; o < n_out; o += gridDim.x * GV_WARPS) {
    const uint4 *wg, *wu;
    wrows(o, wg, wu);
    float ag[MR], au[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) ag[r] = au[r] = 0.f;
    int i = lane;
    for (; i + 32 * (B - 1) < kv8; i += 32 * B) {  // B independent 16-byte weight loads per lane
      uint4 g4[B], u4[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        g4[j] = ld_stream16(wg + i + 32 * j);
        if (GLU) u4[j] = ld_stream16(wu + i + 32 * j);
      }
#pragma unroll
      for (int j = 0; j < B; ++j)
#pragma unroll
        for (int r = 0; r < MR; ++r)
          if (r < M) {
            const uint4 x = xs[r * kv8 + i + 32 * j];
            ag[r] += dot8(g4[j], x);
            if (GLU) au[r] += dot8(u4[j], x);
          }
    }
    for (; i < kv8; i += 32) {
      const uint4 g1 = ld_stream16(wg + i);
      uint4 u1;
      if (GLU) u1 = ld_stream16(wu + i);
#pragma unroll
      for (int r = 0; r < MR; ++r)
        if (r < M) {
          const uint4 x = xs[r * kv8 + i];
          ag[r] += dot8(g1, x);
          if (GLU) au[r] += dot8(u1, x);
        }
    }
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      if (r >= M) break;
      float g = ag[r], u = au[r];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        g += __shfl_xor_sync(0xffffffffu, g, off);
        if (GLU) u += __shfl_xor_sync(0xffffffffu, u, off);
      }
      if (lane == 0) {
        if constexpr (EPI == CC_EPI_RESID_ADD) {
          reinterpret_cast<float*>(C)[(int64_t)r * ldc + o] += g;
        } else {
          float y = g;
          if constexpr (EPI == CC_EPI_GELU) y = gelu_tanh(g);
          if constexpr (GLU) y = silu(g) * u;
          reinterpret_cast<__nv_bfloat16*>(C)[(int64_t)r * ldc + o] = __float2bfloat16_rn(y);
        }
      }
    }
  }
  dtrace(2, t0, t1);
}

// ---- weight-streaming GEMV for one row (decode) -------------------------------
// One CTA per SM, GS_CFG.nw warps.  The n_out x (K / pe) row pieces ("stages")
// are split evenly over all warps of the grid (to one stage); a row cut by a
// warp boundary (a "seam") is finished by whichever of its two warps comes
// second, lo + hi in that fixed order (deterministic).  Each warp streams its
// pieces through its own ring of 2 KiB shared-memory stages with 16-byte
// cp.async (L2 evict-first: weights are read once per token, the KV cache and
// activations stay).  The ring is filled BEFORE griddepcontrol.wait -- weights
// never depend on the predecessor -- so under programmatic dependent launch
// the first stages load while the previous kernel of the decode chain drains.
// A stage is one 1024-element piece of a row (SwiGLU: a 512-element piece of
// the gate row + the same piece of its up row); lane l copies and later reads
// the 16-byte words l, l + 32, ... of the piece (no cross-lane hand-off)
// against the staged activation row; the warp reduces once per output.
// Measured and dropped: 1D bulk copies through the TMA unit (2.2-3.3 TB/s at
// these shapes: not enough bytes in flight per SM for a pure stream), L2
// bulk prefetch ahead of the ring (cp.async.bulk.prefetch.L2, rolling or
// before the wait: 5-25% slower per token), the previous kernel prefetching
// the next projection's weights into L2 (3% slower).
// 28 warps x 2 stages x 2 KiB (measured best of {8..32} warps x {1, 2, 4} KiB
// stages x {1..6} stages at config 2: 3.30 ms/token vs 3.38 for 24 x 2 x 2 KiB,
// 3.42-3.56 with 4 stages, 4.1-4.2 with 1 KiB stages or 8 warps).
struct GsCfg { int nw, sb, ns, min_smem, maxr; };
constexpr GsCfg GS_CFG = {28, 2048, 2, 116 * 1024, 80};
// (Measured and dropped: alternating footprints -- the NORM projections at
// 24 warps / 104 KiB, the others at 22 warps / >= 116 KiB, <= 40 registers --
// so each projection's CTAs land next to the previous one's and stream while
// it drains: 3.41 vs 3.13 ms/token; the co-resident pair slows both.)
// Every launch requests > 114 KiB of shared memory, so at most ONE CTA of it
// is resident per SM: under programmatic dependent launch the CTAs are
// placed while the previous kernel still occupies the SMs, and a statically
// partitioned grid whose CTAs doubled up on some SMs (measured: 148 CTAs on
// 77 SMs) runs at half speed.  The 116 KiB still leave room for the fused
// attention step's CTAs (19 KiB) to land early next to the QKV projection.
constexpr int GS_MIN_SMEM = 116 * 1024;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld_f4_hint(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void cp_async16_plain(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int GS_EPI_LOGITS = 16;  // internal epilogue: K7 logits (f32 normed row, f32 out)
__device__ __forceinline__ float dot8f(const uint4& w, const float4& x0, const float4& x1) {
  const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&w);
  float2 f0 = __bfloat1622float2(a[0]), f1 = __bfloat1622float2(a[1]), f2 = __bfloat1622float2(a[2]),
         f3 = __bfloat1622float2(a[3]);
  float s = 0.f;
  s = fmaf(f0.x, x0.x, s);
  s = fmaf(f0.y, x0.y, s);
  s = fmaf(f1.x, x0.z, s);
  s = fmaf(f1.y, x0.w, s);
  s = fmaf(f2.x, x1.x, s);
  s = fmaf(f2.y, x1.y, s);
  s = fmaf(f3.x, x1.z, s);
  s = fmaf(f3.y, x1.w, s);
  return s;
}

// Register cap per configuration (MAXR): 80 (48 kept a 896-thread CTA small
// enough for an attention CTA to land next to the QKV projection, which only
// pays with the maximum shared-memory carveout -- measured: 48 / 64 / 80 / 128
// registers 3.23 / 3.11 / 3.10 / 3.10 ms per token with the driver's carveout).
template <int EPI, bool NORM, int GS_WARPS, int GS_STAGE, int GS_STAGES, int MAXR>
__global__ void __maxnreg__(MAXR) gemv_stream_kernel(const void* __restrict__ A_,
                                                                    const __nv_bfloat16* __restrict__ W, int64_t ldw,
                                                                    void* __restrict__ C, int N, int K,
                                                                    const float* __restrict__ norm_w, float eps,
                                                                    float4* __restrict__ seam, unsigned* seam_ticket) {
  extern __shared__ __align__(128) uint8_t gs_smem[];
  __shared__ float red[GS_WARPS];
  constexpr bool GLU = EPI == CC_EPI_SWIGLU;
  constexpr bool F32X = EPI == GS_EPI_LOGITS;  // f32 activations (unrounded normed row), f32 output
  constexpr int VPL = GLU ? GS_STAGE / 1024 : GS_STAGE / 512;  // 16-byte words per lane per stage (per row for SwiGLU)
  constexpr int GS_RING = GS_WARPS * GS_STAGES * GS_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_out = GLU ? N / 2 : N;
  const int pe = GLU ? min(K, GS_STAGE / 4) : min(K, GS_STAGE / 2);  // row elements per stage
  const int nv = pe / 256;                                             // words per lane actually used (<= VPL)
  const int np = K / pe;                              // stages per output
  // warps split the n_out * np stages evenly (to one stage); a row cut by a
  // range boundary ("seam") is finished by whichever of its two warps comes
  // second, as lo + hi (fixed order).  Every used warp covers >= 1 row, so a
  // row has at most one seam.
  const int gw = blockIdx.x * GS_WARPS + warp;
  const int used = min(gridDim.x * GS_WARPS, n_out);
  const int64_t tot = (int64_t)n_out * np;
  const int64_t s0 = gw < used ? tot * gw / used : 0, s1 = gw < used ? tot * (gw + 1) / used : 0;
  const int n_st = (int)(s1 - s0);
  uint8_t* ring = gs_smem + (size_t)warp * GS_STAGES * GS_STAGE;
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(gs_smem + GS_RING);
  float* xsf = reinterpret_cast<float*>(gs_smem + GS_RING);
  const unsigned long long t0 = gtime();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int st) {  // this lane's words of stage st (one commit group per stage, empty past the end)
    if (st < n_st) {
      const int o = (int)((s0 + st) / np), p = (int)((s0 + st) % np);
      uint4* dst = reinterpret_cast<uint4*>(ring + (size_t)(st % GS_STAGES) * GS_STAGE);
      const int64_t rg = GLU ? (int64_t)(o / 64) * 128 + (o % 64) : o;
      const uint4* src = reinterpret_cast<const uint4*>(W + rg * ldw + (int64_t)p * pe);
#pragma unroll
      for (int i = 0; i < VPL; ++i)
        if (i < nv) cp_async16(dst + lane + 32 * i, src + lane + 32 * i, pol);
      if constexpr (GLU) {
        const uint4* src_u = reinterpret_cast<const uint4*>(W + (rg + 64) * ldw + (int64_t)p * pe);
#pragma unroll
        for (int i = 0; i < VPL; ++i)
          if (i < nv) cp_async16(dst + GS_STAGE / 32 + lane + 32 * i, src_u + lane + 32 * i, pol);
      }
    }
    cp_async_commit();
  };
  // RMSNorm weights are weights: loaded before the ring fills and before the
  // wait (issued after the predecessor they would queue behind ~20 MB of
  // streaming loads: measured 3.3-5.5 us for the prologue)
  constexpr int TAILMAX = 256;  // words past one per thread, kept in shared memory (K / 4 <= threads + 256)
  __shared__ float4 xt[NORM ? TAILMAX : 1], gt[NORM ? TAILMAX : 1];
  float4 gr = make_float4(1.f, 1.f, 1.f, 1.f);
  if constexpr (NORM) {
    const float4* g4 = reinterpret_cast<const float4*>(norm_w);
    if (norm_w != nullptr) {  // L2 evict-last: 32 KiB per layer that every CTA reads, kept across tokens
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      if ((int)threadIdx.x < K / 4) gr = ld_f4_hint(g4 + threadIdx.x, keep);
      for (int j = threadIdx.x + blockDim.x; j < K / 4 && j - (int)blockDim.x < TAILMAX; j += blockDim.x)
        gt[j - blockDim.x] = ld_f4_hint(g4 + j, keep);
    } else {
      for (int j = threadIdx.x; j < TAILMAX; j += blockDim.x) gt[j] = make_float4(1.f, 1.f, 1.f, 1.f);
    }
  }
#pragma unroll
  for (int st = 0; st < GS_STAGES; ++st) issue(st);  // the ring fills before the wait
  if (!g_trigger_late) pdl_trigger();
  pdl_wait();  // the activation row comes from the predecessor
  const unsigned long long t1 = gtime();
  unsigned long long c_x = 0, c_r = 0;
  if constexpr (NORM) {  // weighted RMSNorm of the f32 residual row (same expression as gemv_kernel)
    const float4* x4 = reinterpret_cast<const float4*>(A_);
    const float4* g4 = reinterpret_cast<const float4*>(norm_w);
    // one round trip (L2: the predecessor just wrote the row)
    const int i0 = threadIdx.x;
    const float4 xr = i0 < K / 4 ? x4[i0] : make_float4(0.f, 0.f, 0.f, 0.f);
    float ss = fmaf(xr.x, xr.x, fmaf(xr.y, xr.y, fmaf(xr.z, xr.z, fmaf(xr.w, xr.w, 0.f))));
    for (int i = i0 + blockDim.x; i < K / 4; i += blockDim.x) {
      const float4 v = x4[i];
      ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
      if (i - (int)blockDim.x < TAILMAX) xt[i - blockDim.x] = v;
    }
    if (g_dtrace && threadIdx.x == 0 && ss != 12345.f) c_x = gtime();  // (timeline: the row has landed)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (g_dtrace && threadIdx.x == 0) c_r = gtime();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < GS_WARPS; ++w) tot += red[w];
    const float inv = rsqrtf(tot / (float)K + eps);
    auto put = [&](int i, const float4& v, const float4& g) {
      if constexpr (F32X) {
        *reinterpret_cast<float4*>(xsf + 4 * i) =
            make_float4(v.x * inv * g.x, v.y * inv * g.y, v.z * inv * g.z, v.w * inv * g.w);
        return;
      }
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * g.x, v.y * inv * g.y);
      __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * g.z, v.w * inv * g.w);
      *reinterpret_cast<uint2*>(xs + 4 * i) =
          make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    };
    if (i0 < K / 4) put(i0, xr, gr);
    for (int i = i0 + blockDim.x; i < K / 4; i += blockDim.x) {
      const int t = i - blockDim.x;  // (own words: no barrier needed)
      if (t < TAILMAX) put(i, xt[t], gt[t]);
      else put(i, x4[i], norm_w != nullptr ? g4[i] : make_float4(1.f, 1.f, 1.f, 1.f));
    }
  } else {
    const uint4* a8 = reinterpret_cast<const uint4*>(A_);
    for (int i = threadIdx.x; i < K / 8; i += blockDim.x) reinterpret_cast<uint4*>(xs)[i] = a8[i];
  }
  __syncthreads();
  // dependents (the attention step after QKV) land only now: their ~6k
  // per-SM pre-wait loads issued during this prologue queued its shared-memory
  // writes and barrier behind them (measured: the RMSNorm reduction 0.3 -> 3 us)
  if (g_trigger_late) pdl_trigger();
  const unsigned long long c1 = g_dtrace ? gtime() : 0;
  float ag = 0.f, au = 0.f;
  float c_pre = 0.f;  // residual: the row's old value, loaded when its first piece starts
  for (int st = 0; st < n_st; ++st) {
    cp_async_wait<GS_STAGES - 1>();  // this lane's words of stage st have landed
    const int p = (int)((s0 + st) % np);
    if constexpr (EPI == CC_EPI_RESID_ADD)
      if (lane == 0 && (p == 0 || st == 0)) c_pre = reinterpret_cast<const float*>(C)[(s0 + st) / np];
    const uint4* wv = reinterpret_cast<const uint4*>(ring + (size_t)(st % GS_STAGES) * GS_STAGE);
    const uint4* xv = reinterpret_cast<const uint4*>(xs + (size_t)p * pe);
    const float4* xf = reinterpret_cast<const float4*>(xsf + (size_t)p * pe);
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (i < nv) {
        if constexpr (F32X) {
          ag += dot8f(wv[lane + 32 * i], xf[2 * (lane + 32 * i)], xf[2 * (lane + 32 * i) + 1]);
        } else {
          const uint4 x = xv[lane + 32 * i];
          ag += dot8(wv[lane + 32 * i], x);
          if constexpr (GLU) au += dot8(wv[GS_STAGE / 32 + lane + 32 * i], x);
        }
      }
    issue(st + GS_STAGES);  // refill the slot just read (same lane, same words)
    if (p == np - 1 || st == n_st - 1) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        ag += __shfl_xor_sync(0xffffffffu, ag, off);
        if constexpr (GLU) au += __shfl_xor_sync(0xffffffffu, au, off);
      }
      const int o = (int)((s0 + st) / np);
      bool finish = true;
      if ((int64_t)o * np < s0 || (int64_t)(o + 1) * np > s1) {  // a seam row: lo (ends past s1) or hi part
        const bool hi = (int64_t)o * np < s0;
        const int sm = hi ? gw : gw + 1;
        if (lane == 0) {
          seam[2 * sm + (hi ? 1 : 0)] = make_float4(ag, au, 0.f, 0.f);
          unsigned prev;  // release our partial, acquire the other's
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&seam_ticket[sm]) : "memory");
          finish = prev == 1u;
          if (finish) {
            const float4 other = __ldcg(&seam[2 * sm + (hi ? 0 : 1)]);
            ag = hi ? other.x + ag : ag + other.x;
            au = hi ? other.y + au : au + other.y;
            seam_ticket[sm] = 0u;  // ready for the next launch on this stream
          }
        }
      }
      if (lane == 0 && finish) {
        if constexpr (EPI == CC_EPI_RESID_ADD) {
          reinterpret_cast<float*>(C)[o] = c_pre + ag;
        } else if constexpr (F32X) {
          reinterpret_cast<float*>(C)[o] = ag;
        } else {
          float y = ag;
          if constexpr (EPI == CC_EPI_GELU) y = gelu_tanh(ag);
          if constexpr (GLU) y = silu(ag) * au;
          reinterpret_cast<__nv_bfloat16*>(C)[o] = __float2bfloat16_rn(y);
        }
      }
      ag = au = 0.f;
    }
  }
  cp_async_wait<0>();
  dtrace(1, t0, t1, c1, g_dtrace ? gtime() : 0, c_x, c_r);
}

// ---- split-KV decode attention ------------------------------------------------
constexpr int DA_KEYS = 128;  // keys per CTA (one per thread); 64 measured slower (14.7 vs 13.5 us + a longer combine)
constexpr int DA_DH = 128;
constexpr int DA_MAXG = 8;
constexpr int DA_COMBINE_MAX = 4096;  // chunks of 128 keys: 512k keys

// grid (Hkv, n_chunks); thread t owns key j = chunk * 128 + t for the scores
// and output column t for P.V.  Partials: o [chunk][Hq][DH] (unnormalised),
// ml [chunk][Hq] = (max, sum) in the log2 domain.
template <int G>
__global__ void __launch_bounds__(DA_KEYS) decode_attn_partial(const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ K,
                                                               const __nv_bfloat16* __restrict__ V,
                                                               const uint8_t* __restrict__ key_pad,
                                                               float* __restrict__ part_o, float2* __restrict__ part_ml,
                                                               int n_keys, const int32_t* __restrict__ n_keys_dev,
                                                               int Hq, int Hkv, float scale_log2) {
  pdl_trigger();
  pdl_wait();
  if (n_keys_dev != nullptr) n_keys = *n_keys_dev;  // CUDA-graph replay: key count lives on the device
  if ((int)blockIdx.y * DA_KEYS >= n_keys) return;   // chunk beyond the live keys (grid sized for capacity)
  __shared__ __align__(16) float qs[G][DA_DH];
  __shared__ float ps[G][DA_KEYS];
  __shared__ float2 ml_s[G];
  const int g = blockIdx.x, c = blockIdx.y, t = threadIdx.x;
  const int kvw = Hkv * DA_DH;
  for (int i = t; i < G * DA_DH; i += DA_KEYS) qs[i / DA_DH][i % DA_DH] = __bfloat162float(q[(int64_t)g * G * DA_DH + i]);
  __syncthreads();
  // V rows of this thread's P.V role are loaded up front so their latency
  // overlaps the K loads and the score math (thread = 8 columns x 16 keys)
  constexpr int NKG = DA_KEYS / 16;  // key groups of the P.V role (16 keys each)
  const int cg = t & 15, kg = t >> 4;
  const int jn = min(DA_KEYS, n_keys - c * DA_KEYS);
  const __nv_bfloat16* vbase = V + (int64_t)c * DA_KEYS * kvw + g * DA_DH + cg * 8;
  uint4 vv[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int jj = kg + NKG * u;
    vv[u] = jj < jn ? *reinterpret_cast<const uint4*>(vbase + (int64_t)jj * kvw) : make_uint4(0, 0, 0, 0);
  }
  const int j = c * DA_KEYS + t;
  const bool valid = j < n_keys && (key_pad == nullptr || key_pad[j] == 0);
  float sc[G];
#pragma unroll
  for (int h = 0; h < G; ++h) sc[h] = 0.f;
  if (valid) {
    const uint4* kr = reinterpret_cast<const uint4*>(K + (int64_t)j * kvw + g * DA_DH);
    uint4 kv16[DA_DH / 8];
#pragma unroll
    for (int u = 0; u < DA_DH / 8; ++u) kv16[u] = kr[u];  // 16 independent 16-byte loads
#pragma unroll
    for (int u = 0; u < DA_DH / 8; ++u) {
      const uint4 kk = kv16[u];
      const __nv_bfloat162* kb = reinterpret_cast<const __nv_bfloat162*>(&kk);
      float kf[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(kb[e]);
        kf[2 * e] = f.x;
        kf[2 * e + 1] = f.y;
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        // q as two 16-byte shared loads per 8 products (same FMA order)
        const float4 qa = *reinterpret_cast<const float4*>(&qs[h][u * 8]);
        const float4 qb = *reinterpret_cast<const float4*>(&qs[h][u * 8 + 4]);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[h] = fmaf(kf[2 * e], qv[2 * e], fmaf(kf[2 * e + 1], qv[2 * e + 1], sc[h]));
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h) ps[h][t] = valid ? sc[h] * scale_log2 : -INFINITY;
  __syncthreads();
  // per head: max and exp-sum over the 128 keys (warp w handles heads w, w+4, ...)
  const int warp = t >> 5, lane = t & 31;
  for (int h = warp; h < G; h += DA_KEYS / 32) {
    float v[DA_KEYS / 32], m = -INFINITY;
#pragma unroll
    for (int e = 0; e < DA_KEYS / 32; ++e) {
      v[e] = ps[h][lane + 32 * e];
      m = fmaxf(m, v[e]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
#pragma unroll
    for (int e = 0; e < DA_KEYS / 32; ++e) {
      const float p = m == -INFINITY ? 0.f : exp2f(v[e] - m);
      ps[h][lane + 32 * e] = p;
      l += p;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0) ml_s[h] = make_float2(m, l);
  }
  __syncthreads();
  // P.V: thread t = (column group cg = t & 15: 8 columns, key group kg = t >> 4:
  // keys kg, kg + 8, ...) -> 16 independent 16-byte V loads per thread; the 8
  // key-group partials are folded through smem in a fixed order
  float o[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[h][e] = 0.f;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int jj = kg + NKG * u;
    const __nv_bfloat162* vb = reinterpret_cast<const __nv_bfloat162*>(&vv[u]);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float p = ps[h][jj];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 vf = __bfloat1622float2(vb[e]);
        o[h][2 * e] = fmaf(p, vf.x, o[h][2 * e]);
        o[h][2 * e + 1] = fmaf(p, vf.y, o[h][2 * e + 1]);
      }
    }
  }
  __syncthreads();  // ps no longer needed: reuse as [8 key groups][G][128] partials? (too small) -> red below
  __shared__ float red[NKG][G][DA_DH];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[kg][h][cg * 8 + e] = o[h][e];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int head = g * G + h;
    for (int col = t; col < DA_DH; col += DA_KEYS) {
      float acc = 0.f;
#pragma unroll
      for (int k2 = 0; k2 < NKG; ++k2) acc += red[k2][h][col];
      part_o[((int64_t)c * Hq + head) * DA_DH + col] = acc;
    }
    if (t == 0) part_ml[(int64_t)c * Hq + head] = ml_s[h];
  }
}

// ---- fused decode attention step (one launch per layer) -------------------------
// Same split-KV partial as decode_attn_partial, plus what the decode chain ran
// as separate kernels around it:
//   * RoPE of the new row's q heads of this group (rope_scatter's arithmetic:
//     rope_pair on the bf16 inputs, rounded to bf16);
//   * the append: the CTA whose chunk holds the new slot writes its kv head's
//     k (position-free), rotated k and v at the slot (rope_scatter's bits)
//     and uses them from shared memory for that key;
//   * the combine: each CTA bumps its group's ticket after writing its
//     partial; the last one folds the chunks (fixed chunk order: the result
//     does not depend on which CTA came last) and resets the ticket.
// grid (Hkv, chunks of the capacity); CTAs past the live keys exit at once.
constexpr int DF_MAXC = 1024;  // chunks the in-kernel combine folds (128k keys)

template <int G>
__global__ void __launch_bounds__(DA_KEYS) decode_attn_fused(
    const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ slot_p, const int32_t* __restrict__ pos_p,
    const float2* __restrict__ table, __nv_bfloat16* kv_k, __nv_bfloat16* kv_v, __nv_bfloat16* k_rot,
    const uint8_t* __restrict__ key_pad, float* part_o, float2* part_ml, unsigned* tickets,
    __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse, int n_keys, const int32_t* __restrict__ n_keys_dev,
    int Hq, int Hkv, float scale_log2) {
  const unsigned long long t0 = gtime();
  pdl_trigger();
  pdl_wait();
  const unsigned long long t1 = gtime();
  if (n_keys_dev != nullptr) n_keys = *n_keys_dev;
  const int n_chunks = (n_keys + DA_KEYS - 1) / DA_KEYS;
  const int g = blockIdx.x, c = blockIdx.y, t = threadIdx.x;
  if (c >= n_chunks) return;
  constexpr int NKG = DA_KEYS / 16;
  __shared__ __align__(16) float qs[G][DA_DH];
  __shared__ float ps[G][DA_KEYS];
  __shared__ float2 ml_s[G];
  __shared__ __align__(16) float red[NKG][G][DA_DH];
  __shared__ __align__(16) __nv_bfloat16 knew[DA_DH], vnew[DA_DH];
  __shared__ unsigned ticket_s;
  const int kvw = Hkv * DA_DH;
  const int slot = *slot_p;
  const int cg = t & 15, kg = t >> 4;
  const int jn = min(DA_KEYS, n_keys - c * DA_KEYS);
  // V rows of the P.V role first (their latency overlaps the rest)
  const __nv_bfloat16* vbase = kv_v + (int64_t)c * DA_KEYS * kvw + g * DA_DH + cg * 8;
  uint4 vv[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int jj = kg + NKG * u;
    vv[u] = jj < jn ? *reinterpret_cast<const uint4*>(vbase + (int64_t)jj * kvw) : make_uint4(0, 0, 0, 0);
  }
  const float2* cs = table + (int64_t)(*pos_p) * (DA_DH / 2);
  const __nv_bfloat16* qrow = qkv + (int64_t)g * G * DA_DH;
  for (int i = t; i < G * DA_DH / 2; i += DA_KEYS) {
    const int h = i / (DA_DH / 2), jj = i % (DA_DH / 2);
    const float a = __bfloat162float(qrow[h * DA_DH + jj]), b = __bfloat162float(qrow[h * DA_DH + jj + DA_DH / 2]);
    float xr, yr;
    rope_pair(a, b, cs[jj].x, cs[jj].y, xr, yr);
    qs[h][jj] = __bfloat162float(__float2bfloat16_rn(xr));
    qs[h][jj + DA_DH / 2] = __bfloat162float(__float2bfloat16_rn(yr));
  }
  const bool owner = slot / DA_KEYS == c;
  if (owner) {  // append this kv head's slice of the new row
    const int64_t off = (int64_t)slot * kvw + g * DA_DH;
    const __nv_bfloat16* krow = qkv + (int64_t)(Hq + g) * DA_DH;
    const __nv_bfloat16* vrow = qkv + (int64_t)(Hq + Hkv + g) * DA_DH;
    if (t < DA_DH / 2) {
      const __nv_bfloat16 x = krow[t], y = krow[t + DA_DH / 2];
      float xr, yr;
      rope_pair(__bfloat162float(x), __bfloat162float(y), cs[t].x, cs[t].y, xr, yr);
      const __nv_bfloat16 bx = __float2bfloat16_rn(xr), by = __float2bfloat16_rn(yr);
      kv_k[off + t] = x;
      kv_k[off + t + DA_DH / 2] = y;
      k_rot[off + t] = bx;
      k_rot[off + t + DA_DH / 2] = by;
      knew[t] = bx;
      knew[t + DA_DH / 2] = by;
    }
    const __nv_bfloat16 vx = vrow[t];
    kv_v[off + t] = vx;
    vnew[t] = vx;
  }
  __syncthreads();
  if (owner) {  // the new key's V words from shared memory (the global copy may be stale in this CTA)
    const int jn_new = slot - c * DA_KEYS;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (kg + NKG * u == jn_new) vv[u] = *reinterpret_cast<const uint4*>(&vnew[cg * 8]);
  }
  const int j = c * DA_KEYS + t;
  const bool valid = j < n_keys && (key_pad == nullptr || key_pad[j] == 0);
  float sc[G];
#pragma unroll
  for (int h = 0; h < G; ++h) sc[h] = 0.f;
  if (valid) {
    const uint4* kr = j == slot ? reinterpret_cast<const uint4*>(knew)
                                : reinterpret_cast<const uint4*>(k_rot + (int64_t)j * kvw + g * DA_DH);
    uint4 kv16[DA_DH / 8];
#pragma unroll
    for (int u = 0; u < DA_DH / 8; ++u) kv16[u] = kr[u];
#pragma unroll
    for (int u = 0; u < DA_DH / 8; ++u) {
      const uint4 kk = kv16[u];
      const __nv_bfloat162* kb = reinterpret_cast<const __nv_bfloat162*>(&kk);
      float kf[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(kb[e]);
        kf[2 * e] = f.x;
        kf[2 * e + 1] = f.y;
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float4 qa = *reinterpret_cast<const float4*>(&qs[h][u * 8]);
        const float4 qb = *reinterpret_cast<const float4*>(&qs[h][u * 8 + 4]);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[h] = fmaf(kf[2 * e], qv[2 * e], fmaf(kf[2 * e + 1], qv[2 * e + 1], sc[h]));
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h) ps[h][t] = valid ? sc[h] * scale_log2 : -INFINITY;
  __syncthreads();
  const int warp = t >> 5, lane = t & 31;
  for (int h = warp; h < G; h += DA_KEYS / 32) {
    float v[DA_KEYS / 32], m = -INFINITY;
#pragma unroll
    for (int e = 0; e < DA_KEYS / 32; ++e) {
      v[e] = ps[h][lane + 32 * e];
      m = fmaxf(m, v[e]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
#pragma unroll
    for (int e = 0; e < DA_KEYS / 32; ++e) {
      const float p = m == -INFINITY ? 0.f : exp2f(v[e] - m);
      ps[h][lane + 32 * e] = p;
      l += p;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0) ml_s[h] = make_float2(m, l);
  }
  __syncthreads();
  float o[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[h][e] = 0.f;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int jj = kg + NKG * u;
    const __nv_bfloat162* vb = reinterpret_cast<const __nv_bfloat162*>(&vv[u]);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float p = ps[h][jj];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 vf = __bfloat1622float2(vb[e]);
        o[h][2 * e] = fmaf(p, vf.x, o[h][2 * e]);
        o[h][2 * e + 1] = fmaf(p, vf.y, o[h][2 * e + 1]);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[kg][h][cg * 8 + e] = o[h][e];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int head = g * G + h;
    float acc = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < NKG; ++k2) acc += red[k2][h][t];
    part_o[((int64_t)c * Hq + head) * DA_DH + t] = acc;
    if (t == 0) part_ml[(int64_t)c * Hq + head] = ml_s[h];
  }
  // ---- last CTA of the group folds the chunks ----
  __threadfence();
  __syncthreads();
  if (t == 0) ticket_s = atomicAdd(&tickets[g], 1u);
  __syncthreads();
  if (ticket_s != (unsigned)(n_chunks - 1)) {
    dtrace(3, t0, t1);
    return;
  }
  if (t == 0) tickets[g] = 0u;  // ready for the next layer / step
  __threadfence();
  float* wsm = &red[0][0][0] + warp * DF_MAXC;  // chunk weights of this warp's head (red is free now)
  for (int h = warp; h < G; h += DA_KEYS / 32) {
    const int head = g * G + h;
    float m = -INFINITY;
    for (int cc = lane; cc < n_chunks; cc += 32) m = fmaxf(m, __ldcg(&part_ml[(int64_t)cc * Hq + head]).x);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
    for (int cc = lane; cc < n_chunks; cc += 32) {
      const float2 ml = __ldcg(&part_ml[(int64_t)cc * Hq + head]);
      const float w = (m == -INFINITY || ml.x == -INFINITY) ? 0.f : exp2f(ml.x - m);
      wsm[cc] = w;
      l = fmaf(ml.y, w, l);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    __syncwarp();
    // lane = 4 output columns; 16 chunk rows in flight
    const float4* po = reinterpret_cast<const float4*>(part_o) + (int64_t)head * (DA_DH / 4) + lane;
    const int64_t cstride = (int64_t)Hq * (DA_DH / 4);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int cc = 0;
    for (; cc + 15 < n_chunks; cc += 16) {
      float4 v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = __ldcg(po + (int64_t)(cc + k) * cstride);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float w = wsm[cc + k];
        acc.x = fmaf(v[k].x, w, acc.x);
        acc.y = fmaf(v[k].y, w, acc.y);
        acc.z = fmaf(v[k].z, w, acc.z);
        acc.w = fmaf(v[k].w, w, acc.w);
      }
    }
    for (; cc < n_chunks; ++cc) {
      const float4 v = __ldcg(po + (int64_t)cc * cstride);
      const float w = wsm[cc];
      acc.x = fmaf(v.x, w, acc.x);
      acc.y = fmaf(v.y, w, acc.y);
      acc.z = fmaf(v.z, w, acc.z);
      acc.w = fmaf(v.w, w, acc.w);
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(ctx + (int64_t)head * DA_DH + 4 * lane) =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    if (lane == 0 && lse != nullptr) lse[head] = l > 0.f ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
  }
  dtrace(4, t0, t1);  // the combining CTA
}

// ---- tensor-core decode attention step (default) ------------------------------
// Same contract as decode_attn_fused (RoPE of q / the new key, the append,
// split-KV partials, last-CTA combine) with the per-chunk math on mma.sync
// (m16n8k16 bf16 -> f32) in the swapped orientation: S^T = K Q^T (M = 16
// keys, N = 8 query heads of the group, zero-padded past G), O^T += V^T P^T
// (M = 16 head dims, N = heads, K = 16 keys).  Both operands are fed straight
// from 16-byte global loads by permuting the reduction index consistently on
// both sides (dims inside each 32-dim pair for S, keys per step for O) and the
// output rows (dims) -- no shared-memory staging; P^T comes from the S^T
// accumulator through movmatrix.trans.
// Each warp owns 32 keys (2 steps of 16) of the CTA's 128-key chunk; the K/V
// words of those keys are loaded BEFORE griddepcontrol.wait: rows other than
// the new slot were appended by this layer's attention step of an earlier
// decode token, and the decode chain keeps at most ~3 grids in flight (every
// GEMV grid holds > 114 KiB of shared memory per SM), so they are complete.
// The new key's words are patched in from shared memory after the append;
// V words of rows past the live keys (uninitialised capacity) are zeroed.
#ifndef CCB_DT_STEPS
#define CCB_DT_STEPS 6  // 384-key chunks: 4 steps 3.085, 6 steps 3.068, 8 steps 3.181 ms/token
#endif
constexpr int DT_WARPS = 4, DT_STEPS = CCB_DT_STEPS, DT_KC = DT_WARPS * DT_STEPS * 16;  // keys per CTA
constexpr int DT_SMEM = DT_WARPS * (DT_STEPS - 2) * 16 * 32 * 16;  // staged steps 2..: 32 KiB per step

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t u4w(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

template <int G>
__global__ void __launch_bounds__(DT_WARPS * 32, 2) decode_attn_tc(
    const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ slot_p, const int32_t* __restrict__ pos_p,
    const float2* __restrict__ table, __nv_bfloat16* kv_k, __nv_bfloat16* kv_v, __nv_bfloat16* k_rot,
    const uint8_t* __restrict__ key_pad, float* part_o, float2* part_ml, unsigned* tickets,
    __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse, int n_keys, const int32_t* __restrict__ n_keys_dev,
    int max_keys, int Hq, int Hkv, float scale_log2, int stage_pre) {
  static_assert(G <= 8, "one n-tile of query heads");
  extern __shared__ __align__(16) uint4 stg[];  // [warp][staged step][word][lane]
  const unsigned long long t0 = gtime();
  const int g = blockIdx.x, c = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, r = lane >> 2, q = lane & 3;
  const int kvw = Hkv * DA_DH;
  const int kbase = c * DT_KC + warp * (DT_STEPS * 16);
  // a step's 16 words per lane: K keys r, r + 8 (dims 32p + 8q .. + 7) then V
  // keys 2q, 2q+1, 2q+8, 2q+9 (dims 16r .. 16r + 15)
  auto word_src = [&](int s, int i) -> const __nv_bfloat16* {
    if (i < 8) {
      const int e = i >> 2, p = i & 3;
      const int key = min(kbase + s * 16 + r + 8 * e, max_keys - 1);
      return k_rot + (int64_t)key * kvw + g * DA_DH + 8 * q + 32 * p;
    }
    const int e = (i - 8) >> 1, h = (i - 8) & 1;
    const int key = min(kbase + s * 16 + 2 * q + (e & 1) + 8 * (e >> 1), max_keys - 1);
    return kv_v + (int64_t)key * kvw + g * DA_DH + 16 * r + 8 * h;
  };
  uint4 kf[2][2][4];  // register buffers of two steps
  uint4 vf[2][4][2];
  // ---- pre-wait: steps 0-1 into registers, steps 2.. into shared memory ----
  auto preload = [&]() {
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint4 w = ld_stream16(word_src(s, i));
        if (i < 8) kf[s][i >> 2][i & 3] = w;
        else vf[s][(i - 8) >> 1][(i - 8) & 1] = w;
      }
  };
  if (stage_pre & 2) preload();
  auto stage = [&]() {
#pragma unroll
    for (int s = 2; s < DT_STEPS; ++s)
#pragma unroll
      for (int i = 0; i < 16; ++i)
        cp_async16_plain(&stg[((warp * (DT_STEPS - 2) + (s - 2)) * 16 + i) * 32 + lane], word_src(s, i));
    cp_async_commit();
  };
  if (stage_pre & 1) stage();
  pdl_trigger();
  pdl_wait();
  if (!(stage_pre & 2)) preload();
  if (!(stage_pre & 1)) stage();
  const unsigned long long t1 = gtime();
  // one round trip: key count, slot, position and the raw q / k / v words of
  // this group (their addresses do not depend on the position)
  if (n_keys_dev != nullptr) n_keys = *n_keys_dev;
  const int slot = *slot_p, pos = *pos_p;
  constexpr int QP = (G * DA_DH / 2 + DT_WARPS * 32 - 1) / (DT_WARPS * 32);  // q rotation pairs per thread
  const __nv_bfloat16* qrow = qkv + (int64_t)g * G * DA_DH;
  __nv_bfloat16 qlo[QP], qhi[QP];
#pragma unroll
  for (int j = 0; j < QP; ++j) {
    const int i = tid + j * DT_WARPS * 32, h = i / (DA_DH / 2), jj = i % (DA_DH / 2);
    if (i < G * DA_DH / 2) {
      qlo[j] = qrow[h * DA_DH + jj];
      qhi[j] = qrow[h * DA_DH + jj + DA_DH / 2];
    }
  }
  const __nv_bfloat16* krow = qkv + (int64_t)(Hq + g) * DA_DH;
  const __nv_bfloat16 kx = krow[tid & (DA_DH / 2 - 1)], ky = krow[(tid & (DA_DH / 2 - 1)) + DA_DH / 2];
  const __nv_bfloat16 vx = qkv[(int64_t)(Hq + Hkv + g) * DA_DH + tid];
  const int n_chunks = (n_keys + DT_KC - 1) / DT_KC;
  if (c >= n_chunks) {
    cp_async_wait<0>();
    return;
  }
  __shared__ __align__(16) __nv_bfloat16 qb[8][DA_DH];
  __shared__ __align__(16) __nv_bfloat16 knew[DA_DH], vnew[DA_DH];
  __shared__ __align__(16) float wo[DT_WARPS][8][DA_DH];
  __shared__ float wm[DT_WARPS][8], wl[DT_WARPS][8];
  __shared__ unsigned ticket_s;
  const float2* cs = table + (int64_t)pos * (DA_DH / 2);
#pragma unroll
  for (int j = 0; j < QP; ++j) {
    const int i = tid + j * DT_WARPS * 32, h = i / (DA_DH / 2), jj = i % (DA_DH / 2);
    if (i < G * DA_DH / 2) {
      float xr, yr;
      rope_pair(__bfloat162float(qlo[j]), __bfloat162float(qhi[j]), cs[jj].x, cs[jj].y, xr, yr);
      qb[h][jj] = __float2bfloat16_rn(xr);
      qb[h][jj + DA_DH / 2] = __float2bfloat16_rn(yr);
    }
  }
  for (int i = G * DA_DH + tid; i < 8 * DA_DH; i += DT_WARPS * 32) (&qb[0][0])[i] = __float2bfloat16_rn(0.f);
  const bool owner = slot / DT_KC == c;
  if (owner) {  // append this kv head's slice of the new row (rope_scatter's bits)
    const int64_t off = (int64_t)slot * kvw + g * DA_DH;
    if (tid < DA_DH / 2) {
      float xr, yr;
      rope_pair(__bfloat162float(kx), __bfloat162float(ky), cs[tid].x, cs[tid].y, xr, yr);
      const __nv_bfloat16 bx = __float2bfloat16_rn(xr), by = __float2bfloat16_rn(yr);
      kv_k[off + tid] = kx;
      kv_k[off + tid + DA_DH / 2] = ky;
      k_rot[off + tid] = bx;
      k_rot[off + tid + DA_DH / 2] = by;
      knew[tid] = bx;
      knew[tid + DA_DH / 2] = by;
    }
    kv_v[off + tid] = vx;
    vnew[tid] = vx;
  }
  __syncthreads();
  // the new key's words from shared memory; V of rows past the live keys zeroed
  auto fix = [&](int s, uint4 (&kb)[2][4], uint4 (&vb)[4][2]) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int key = kbase + s * 16 + r + 8 * e;
      if (owner && key == slot)
#pragma unroll
        for (int p = 0; p < 4; ++p) kb[e][p] = *reinterpret_cast<const uint4*>(&knew[32 * p + 8 * q]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int key = kbase + s * 16 + 2 * q + (e & 1) + 8 * (e >> 1);
      if (owner && key == slot) {
        vb[e][0] = *reinterpret_cast<const uint4*>(&vnew[16 * r]);
        vb[e][1] = *reinterpret_cast<const uint4*>(&vnew[16 * r + 8]);
      }
      if (key >= n_keys) vb[e][0] = vb[e][1] = make_uint4(0, 0, 0, 0);
    }
  };
  fix(0, kf[0], vf[0]);
  fix(1, kf[1], vf[1]);
  const unsigned long long c1 = g_dtrace ? gtime() : 0;
  uint4 qf[4];  // B operand of S^T: head r, dims 32p + 8q .. + 7
#pragma unroll
  for (int p = 0; p < 4; ++p) qf[p] = *reinterpret_cast<const uint4*>(&qb[r][32 * p + 8 * q]);
  float M0 = -INFINITY, M1 = -INFINITY, L0 = 0.f, L1 = 0.f;  // heads 2q, 2q + 1
  float o[8][4];
#pragma unroll
  for (int t = 0; t < 8; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  // two steps per online-softmax round (steps 0-1 from registers, 2-3 staged)
#pragma unroll
  for (int pr = 0; pr < DT_STEPS / 2; ++pr) {
    if (pr >= 1) {  // staged steps: this lane's own words back from shared memory
      if (pr == 1) cp_async_wait<0>();
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint4 w = stg[((warp * (DT_STEPS - 2) + 2 * pr - 2 + b) * 16 + i) * 32 + lane];
          if (i < 8) kf[b][i >> 2][i & 3] = w;
          else vf[b][(i - 8) >> 1][(i - 8) & 1] = w;
        }
      fix(2 * pr, kf[0], vf[0]);
      fix(2 * pr + 1, kf[1], vf[1]);
    }
    float x[2][4];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int s = 2 * pr + b;
      float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};  // even / odd k-tile chains
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        mma16816(sc, kf[b][0][p].x, kf[b][1][p].x, kf[b][0][p].y, kf[b][1][p].y, qf[p].x, qf[p].y);
        mma16816(sd, kf[b][0][p].z, kf[b][1][p].z, kf[b][0][p].w, kf[b][1][p].w, qf[p].z, qf[p].w);
      }
      const int j0 = kbase + s * 16 + r, j1 = j0 + 8;
      const bool v0 = j0 < n_keys && (key_pad == nullptr || key_pad[j0] == 0);
      const bool v1 = j1 < n_keys && (key_pad == nullptr || key_pad[j1] == 0);
      x[b][0] = v0 ? (sc[0] + sd[0]) * scale_log2 : -INFINITY;
      x[b][1] = v0 ? (sc[1] + sd[1]) * scale_log2 : -INFINITY;
      x[b][2] = v1 ? (sc[2] + sd[2]) * scale_log2 : -INFINITY;
      x[b][3] = v1 ? (sc[3] + sd[3]) * scale_log2 : -INFINITY;
    }
    float m0 = fmaxf(fmaxf(x[0][0], x[0][2]), fmaxf(x[1][0], x[1][2]));
    float m1 = fmaxf(fmaxf(x[0][1], x[0][3]), fmaxf(x[1][1], x[1][3]));
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, off));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, off));
    }
    const float N0 = fmaxf(M0, m0), N1 = fmaxf(M1, m1);
    const float a0 = N0 == -INFINITY ? 1.f : exp2f(M0 - N0), a1 = N1 == -INFINITY ? 1.f : exp2f(M1 - N1);
    float pv[2][4];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      pv[b][0] = N0 == -INFINITY ? 0.f : exp2f(x[b][0] - N0);
      pv[b][2] = N0 == -INFINITY ? 0.f : exp2f(x[b][2] - N0);
      pv[b][1] = N1 == -INFINITY ? 0.f : exp2f(x[b][1] - N1);
      pv[b][3] = N1 == -INFINITY ? 0.f : exp2f(x[b][3] - N1);
    }
    M0 = N0;
    M1 = N1;
    L0 = fmaf(L0, a0, (pv[0][0] + pv[0][2]) + (pv[1][0] + pv[1][2]));
    L1 = fmaf(L1, a1, (pv[0][1] + pv[0][3]) + (pv[1][1] + pv[1][3]));
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      o[t][0] *= a0;
      o[t][1] *= a1;
      o[t][2] *= a0;
      o[t][3] *= a1;
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const uint32_t b0 = movtrans(pack_bf16(pv[b][0], pv[b][1])), b1 = movtrans(pack_bf16(pv[b][2], pv[b][3]));
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t wa = u4w(vf[b][0][t >> 2], t & 3), wb = u4w(vf[b][1][t >> 2], t & 3);
        const uint32_t wc = u4w(vf[b][2][t >> 2], t & 3), wd = u4w(vf[b][3][t >> 2], t & 3);
        mma16816(o[t], __byte_perm(wa, wb, 0x5410), __byte_perm(wa, wb, 0x7632), __byte_perm(wc, wd, 0x5410),
                 __byte_perm(wc, wd, 0x7632), b0, b1);
      }
    }
  }
  const unsigned long long c2 = g_dtrace ? gtime() : 0;
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    L0 += __shfl_xor_sync(0xffffffffu, L0, off);
    L1 += __shfl_xor_sync(0xffffffffu, L1, off);
  }
  // ---- CTA merge of the 4 warps (fixed order) ----
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    wo[warp][2 * q][16 * r + 2 * t] = o[t][0];
    wo[warp][2 * q + 1][16 * r + 2 * t] = o[t][1];
    wo[warp][2 * q][16 * r + 2 * t + 1] = o[t][2];
    wo[warp][2 * q + 1][16 * r + 2 * t + 1] = o[t][3];
  }
  if (r == 0) {
    wm[warp][2 * q] = M0;
    wm[warp][2 * q + 1] = M1;
    wl[warp][2 * q] = L0;
    wl[warp][2 * q + 1] = L1;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float mc = -INFINITY;
#pragma unroll
    for (int w = 0; w < DT_WARPS; ++w) mc = fmaxf(mc, wm[w][h]);
    float acc = 0.f, lc = 0.f;
#pragma unroll
    for (int w = 0; w < DT_WARPS; ++w) {
      const float a = (mc == -INFINITY || wm[w][h] == -INFINITY) ? 0.f : exp2f(wm[w][h] - mc);
      acc = fmaf(wo[w][h][tid], a, acc);
      lc = fmaf(wl[w][h], a, lc);
    }
    const int head = g * G + h;
    part_o[((int64_t)c * Hq + head) * DA_DH + tid] = acc;
    if (tid == 0) part_ml[(int64_t)c * Hq + head] = make_float2(mc, lc);
  }
  // ---- last CTA of the group folds the chunks ----
  __syncthreads();
  if (tid == 0) {  // release the CTA's partial (cumulative over the barrier), acquire the others'
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&tickets[g]) : "memory");
    ticket_s = prev;
  }
  __syncthreads();
  const unsigned long long c3 = g_dtrace ? gtime() : 0;
  if (ticket_s != (unsigned)(n_chunks - 1)) {
    dtrace(3, t0, t1, c1, c2, c3);
    return;
  }
  if (tid == 0) tickets[g] = 0u;  // (thread 0's acquire + the barrier order the loads below)
  float* wsm = &wo[0][0][0] + warp * DF_MAXC;  // chunk weights of this warp's head (wo is free now)
  constexpr int DF_BATCH = 24;  // chunk rows whose loads go out together with the (max, sum) loads
  for (int h = warp; h < G; h += DT_WARPS) {
    const int head = g * G + h;
    const float4* po = reinterpret_cast<const float4*>(part_o) + (int64_t)head * (DA_DH / 4) + lane;
    const int64_t cstride = (int64_t)Hq * (DA_DH / 4);
    float4 vb[DF_BATCH];
#pragma unroll
    for (int k = 0; k < DF_BATCH; ++k)
      vb[k] = k < n_chunks ? __ldcg(po + (int64_t)k * cstride) : make_float4(0.f, 0.f, 0.f, 0.f);
    float m = -INFINITY;
    for (int cc = lane; cc < n_chunks; cc += 32) m = fmaxf(m, __ldcg(&part_ml[(int64_t)cc * Hq + head]).x);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
    for (int cc = lane; cc < n_chunks; cc += 32) {
      const float2 ml = __ldcg(&part_ml[(int64_t)cc * Hq + head]);
      const float w = (m == -INFINITY || ml.x == -INFINITY) ? 0.f : exp2f(ml.x - m);
      wsm[cc] = w;
      l = fmaf(ml.y, w, l);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    __syncwarp();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < DF_BATCH; ++k) {
      const float w = k < n_chunks ? wsm[k] : 0.f;
      acc.x = fmaf(vb[k].x, w, acc.x);
      acc.y = fmaf(vb[k].y, w, acc.y);
      acc.z = fmaf(vb[k].z, w, acc.z);
      acc.w = fmaf(vb[k].w, w, acc.w);
    }
    int cc = DF_BATCH;
    for (; cc + 15 < n_chunks; cc += 16) {
      float4 v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = __ldcg(po + (int64_t)(cc + k) * cstride);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float w = wsm[cc + k];
        acc.x = fmaf(v[k].x, w, acc.x);
        acc.y = fmaf(v[k].y, w, acc.y);
        acc.z = fmaf(v[k].z, w, acc.z);
        acc.w = fmaf(v[k].w, w, acc.w);
      }
    }
    for (; cc < n_chunks; ++cc) {
      const float4 v = __ldcg(po + (int64_t)cc * cstride);
      const float w = wsm[cc];
      acc.x = fmaf(v.x, w, acc.x);
      acc.y = fmaf(v.y, w, acc.y);
      acc.z = fmaf(v.z, w, acc.z);
      acc.w = fmaf(v.w, w, acc.w);
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(ctx + (int64_t)head * DA_DH + 4 * lane) =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    if (lane == 0 && lse != nullptr) lse[head] = l > 0.f ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
  }
  dtrace(4, t0, t1, c1, c2, c3);
}

// grid Hq, 128 threads: fold the chunks in index order
// One warp per (head, 32 output columns): 4 x Hq CTAs instead of Hq, every
// chunk partial a coalesced 128-byte row load.  Same arithmetic order as the
// one-CTA-per-head form (weights and sum by lane-strided chunks + butterfly,
// output in 4 fixed chains).
__global__ void __launch_bounds__(32) decode_attn_combine(const float* __restrict__ part_o,
                                                          const float2* __restrict__ part_ml, int n_chunks, int Hq,
                                                          __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse,
                                                          const int32_t* __restrict__ n_keys_dev) {
  const int head = blockIdx.x, lane = threadIdx.x, col = blockIdx.y * 32 + lane;
  pdl_trigger();
  pdl_wait();
  if (n_keys_dev != nullptr) n_chunks = (*n_keys_dev + DA_KEYS - 1) / DA_KEYS;
  __shared__ float w_s[DA_COMBINE_MAX];
  // global max and the chunk weights 2^(m_c - m), sum l (fixed order)
  float m = -INFINITY;
  for (int c = lane; c < n_chunks; c += 32) m = fmaxf(m, part_ml[(int64_t)c * Hq + head].x);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float l = 0.f;
  for (int c = lane; c < n_chunks; c += 32) {
    const float2 ml = part_ml[(int64_t)c * Hq + head];
    const float w = (m == -INFINITY || ml.x == -INFINITY) ? 0.f : exp2f(ml.x - m);
    w_s[c] = w;
    l = fmaf(ml.y, w, l);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
  __syncwarp();
  float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;  // 4 independent chains
  int c = 0;
  for (; c + 15 < n_chunks; c += 16) {  // 16 loads in flight, then the same 4-chain order
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = part_o[((int64_t)(c + k) * Hq + head) * DA_DH + col];
#pragma unroll
    for (int k = 0; k < 16; k += 4) {
      o0 = fmaf(v[k], w_s[c + k], o0);
      o1 = fmaf(v[k + 1], w_s[c + k + 1], o1);
      o2 = fmaf(v[k + 2], w_s[c + k + 2], o2);
      o3 = fmaf(v[k + 3], w_s[c + k + 3], o3);
    }
  }
  for (; c + 3 < n_chunks; c += 4) {
    o0 = fmaf(part_o[((int64_t)c * Hq + head) * DA_DH + col], w_s[c], o0);
    o1 = fmaf(part_o[((int64_t)(c + 1) * Hq + head) * DA_DH + col], w_s[c + 1], o1);
    o2 = fmaf(part_o[((int64_t)(c + 2) * Hq + head) * DA_DH + col], w_s[c + 2], o2);
    o3 = fmaf(part_o[((int64_t)(c + 3) * Hq + head) * DA_DH + col], w_s[c + 3], o3);
  }
  for (; c < n_chunks; ++c) o0 = fmaf(part_o[((int64_t)c * Hq + head) * DA_DH + col], w_s[c], o0);
  const float o = (o0 + o1) + (o2 + o3);
  ctx[(int64_t)head * DA_DH + col] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
  if (blockIdx.y == 0 && lane == 0 && lse != nullptr)
    lse[head] = l > 0.f ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
}

// y[row] = RoPE(x[row], pos[row % n]) for rows of `width` = heads x d_head
template <typename T>
__global__ void __launch_bounds__(128) rope_rows_kernel(const T* __restrict__ x, T* __restrict__ y, int n, int width,
                                                        const int32_t* __restrict__ pos,
                                                        const typename CS<T>::type* __restrict__ table, int dh) {
  using A = typename Acc<T>::type;
  const int64_t row = blockIdx.x;
  const int half = dh / 2;
  const typename CS<T>::type* cs = table + (int64_t)pos[row % n] * half;
  const T* xr = x + row * width;
  T* yr = y + row * width;
  for (int u = threadIdx.x; u < width / 2; u += blockDim.x) {
    const int h = u / half, jj = u % half;
    const int64_t off = (int64_t)h * dh + jj;
    const A a = (A)to_f(xr[off]), b = (A)to_f(xr[off + half]);
    const A cc = (A)cs[jj].x, ss = (A)cs[jj].y;
    if constexpr (sizeof(A) == 8) {
      yr[off] = from_d<T>(a * cc - b * ss);
      yr[off + half] = from_d<T>(a * ss + b * cc);
    } else {
      yr[off] = from_f<T>(a * cc - b * ss);
      yr[off + half] = from_f<T>(a * ss + b * cc);
    }
  }
}

}  // namespace

bool gemv_eligible(int M, int N, int K, int epi, const void* A, int64_t lda, const void* W, int64_t ldw) {
  if (M < 1 || M > GV_MAXM || K % 8 || lda % 8 || ldw % 8) return false;
  if ((size_t)M * K * 2 > 96 * 1024) return false;
  if (epi == CC_EPI_SWIGLU && N % 128) return false;
  return ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15) == 0;
}

// Optionally (CCB_DECODE_CARVEOUT=1) the decode kernels request the whole
// 228 KiB shared-memory carveout, so a CTA of the next kernel always finds
// the carveout for co-residency; measured slower than the driver's choice.
template <typename... KArgs>
int max_carveout(void (*fn)(KArgs...)) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, reinterpret_cast<const void*>(fn)})) return 0;
  if (cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return fail(CC_E_CUDA, "cudaFuncSetAttribute(carveout) failed");
  done.insert({dev, reinterpret_cast<const void*>(fn)});
  return 0;
}

// Zero-initialised device buffers per (device, stream, tag) for tickets the
// kernels reset themselves after use (allocated and cleared once, outside any
// graph capture: the first eager call on a stream).
void* zeroed_scratch(cudaStream_t st, int tag, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::pair<void*, size_t>> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(st) << 8) ^ ((uint64_t)dev << 4) ^ (uint64_t)tag;
  std::lock_guard<std::mutex> g(mu);
  auto& b = bufs[key];
  if (b.second < bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, bytes);
    b = {p, bytes};  // a smaller predecessor is retired, never freed (a captured graph may use it)
  }
  return b.first;
}
constexpr int GS_MAX_SEAMS = 8192;
// attention: which K/V words load before the wait -- bit 0 the shared-memory
// staged steps, bit 1 the register steps (3 measured best: 3.20 vs 3.28 / 3.31 / 3.33)
const int g_dt_stage_pre = [] {
  const char* e = getenv("CCB_DT_STAGE_PRE");
  return e ? atoi(e) : 3;
}();
const int g_carveout = [] {  // maximum carveout: measured 1.5% slower per token (3.27 vs 3.23 ms), off
  const char* e = getenv("CCB_DECODE_CARVEOUT");
  return e ? atoi(e) : 0;
}();

// the streaming kernel (one row, weights through cp.async rings) takes the shape?
bool gemv_stream_ok(int M, int K, int epi) {
  static const int on = [] {
    const char* e = getenv("CCB_GEMV_STREAM");
    return e ? atoi(e) : 1;
  }();
  if (!on || M != 1) return false;
  const int pe = epi == CC_EPI_SWIGLU ? std::min(K, GS_CFG.sb / 4) : std::min(K, GS_CFG.sb / 2);
  return pe % 256 == 0 && K % pe == 0 && GS_CFG.nw * GS_CFG.ns * GS_CFG.sb + K * 2 <= 227 * 1024;
}

void set_trigger_mode() {
  static std::once_flag once;
  std::call_once(once, [] {
    if (const char* e = getenv("CCB_GS_TRIGGER")) {
      int v = atoi(e);
      cudaMemcpyToSymbol(g_trigger_late, &v, sizeof(v));
    }

  });
}

int gemv_stream_launch(const void* A, const void* W, int64_t ldw, void* C, int N, int K, int epi, const float* norm_w,
                       float eps, bool norm, cudaStream_t st) {
  constexpr GsCfg c = GS_CFG;
  set_trigger_mode();
  float4* seam = reinterpret_cast<float4*>(zeroed_scratch(st, 1, GS_MAX_SEAMS * (2 * sizeof(float4) + sizeof(unsigned))));
  if (!seam) return fail(CC_E_CUDA, "gemv_stream: seam buffer allocation failed");
  if (num_sms() * c.nw + 1 > GS_MAX_SEAMS) return fail(CC_E_UNSUP, "gemv_stream: too many warps");
  const size_t smem = std::max<size_t>((size_t)c.nw * c.ns * c.sb + (size_t)K * 2, (size_t)c.min_smem);
  auto go = [&](auto kern) -> int {
    if (int rc = ensure_smem(kern, smem)) return rc;
    if (g_carveout)
      if (int rc = max_carveout(kern)) return rc;
    return launch_k(kern, dim3(num_sms()), dim3(c.nw * 32), smem, st, "gemv_stream", A, (const __nv_bfloat16*)W, ldw,
                    C, N, K, norm_w, eps, seam, reinterpret_cast<unsigned*>(seam + 2 * GS_MAX_SEAMS));
  };
  auto by_norm = [&](auto e_tag) -> int {
    constexpr int E = decltype(e_tag)::value;
    return norm ? go(gemv_stream_kernel<E, true, c.nw, c.sb, c.ns, c.maxr>)
                : go(gemv_stream_kernel<E, false, c.nw, c.sb, c.ns, c.maxr>);
  };
  switch (epi) {
    case CC_EPI_STORE: return by_norm(std::integral_constant<int, CC_EPI_STORE>{});
    case CC_EPI_RESID_ADD: return by_norm(std::integral_constant<int, CC_EPI_RESID_ADD>{});
    case CC_EPI_SWIGLU: return by_norm(std::integral_constant<int, CC_EPI_SWIGLU>{});
    case CC_EPI_GELU: return by_norm(std::integral_constant<int, CC_EPI_GELU>{});
    default: return fail(CC_E_ARG, "gemv: unknown epilogue");
  }
}

// K7 logits of one row through the streaming kernel (RMSNorm prologue in f32,
// f32 logits); CC_E_UNSUP when the shape does not fit
int logits_stream_bf16(const float* hidden, const float* norm_w, float eps, const void* U, float* logits, int d,
                       int vocab, cudaStream_t st) {
  static const int on = [] {
    const char* e = getenv("CCB_LOGITS_STREAM");
    return e ? atoi(e) : 1;
  }();
  const int pe = std::min(d, GS_CFG.sb / 2);
  const size_t smem = std::max<size_t>((size_t)GS_CFG.nw * GS_CFG.ns * GS_CFG.sb + (size_t)d * 4, GS_MIN_SMEM);
  if (!on || pe % 256 || d % pe || smem > 227 * 1024 || (reinterpret_cast<uintptr_t>(hidden) & 15) ||
      (reinterpret_cast<uintptr_t>(norm_w) & 15) || (reinterpret_cast<uintptr_t>(U) & 15))
    return CC_E_UNSUP;
  float4* seam = reinterpret_cast<float4*>(zeroed_scratch(st, 1, GS_MAX_SEAMS * (2 * sizeof(float4) + sizeof(unsigned))));
  if (!seam) return fail(CC_E_CUDA, "logits: seam buffer allocation failed");
  auto kern = gemv_stream_kernel<GS_EPI_LOGITS, true, GS_CFG.nw, GS_CFG.sb, GS_CFG.ns, GS_CFG.maxr>;
  if (int rc = ensure_smem(kern, smem)) return rc;
  return launch_k(kern, dim3(num_sms()), dim3(GS_CFG.nw * 32), smem, st, "logits_stream", (const void*)hidden,
                  (const __nv_bfloat16*)U, (int64_t)d, (void*)logits, vocab, d, norm_w, eps, seam,
                  reinterpret_cast<unsigned*>(seam + 2 * GS_MAX_SEAMS));
}

int gemv_launch(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
                int epi, const float* norm_w, float eps, bool norm, cudaStream_t st) {
  if (gemv_stream_ok(M, K, epi)) return gemv_stream_launch(A, W, ldw, C, N, K, epi, norm_w, eps, norm, st);
  const int n_out = epi == CC_EPI_SWIGLU ? N / 2 : N;
  const size_t smem = (size_t)M * K * 2;
  int grid = (n_out + GV_WARPS - 1) / GV_WARPS;
  {
    int rc = 0;
    auto set = [&](auto k) { if (!rc) rc = ensure_smem(k, 96 * 1024); };
#define CCB_GV_SET(E) set(gemv_kernel<E, false, 1>); set(gemv_kernel<E, true, 1>); \
    set(gemv_kernel<E, false, GV_MAXM>); set(gemv_kernel<E, true, GV_MAXM>);
    CCB_GV_SET(CC_EPI_STORE) CCB_GV_SET(CC_EPI_RESID_ADD) CCB_GV_SET(CC_EPI_SWIGLU) CCB_GV_SET(CC_EPI_GELU)
#undef CCB_GV_SET
    if (rc) return rc;
  }
  auto go = [&](auto kern) {
    return launch_k(kern, dim3(grid), dim3(GV_WARPS * 32), smem, st, "gemv", A, lda, (const __nv_bfloat16*)W, ldw,
                    C, ldc, M, N, K, norm_w, eps);
  };
  auto by_rows = [&](auto e_tag, auto n_tag) -> int {
    constexpr int E = decltype(e_tag)::value;
    constexpr bool NM = decltype(n_tag)::value;
    return M == 1 ? go(gemv_kernel<E, NM, 1>) : go(gemv_kernel<E, NM, GV_MAXM>);
  };
  auto by_norm = [&](auto e_tag) -> int {
    return norm ? by_rows(e_tag, std::true_type{}) : by_rows(e_tag, std::false_type{});
  };
  switch (epi) {
    case CC_EPI_STORE: return by_norm(std::integral_constant<int, CC_EPI_STORE>{});
    case CC_EPI_RESID_ADD: return by_norm(std::integral_constant<int, CC_EPI_RESID_ADD>{});
    case CC_EPI_SWIGLU: return by_norm(std::integral_constant<int, CC_EPI_SWIGLU>{});
    case CC_EPI_GELU: return by_norm(std::integral_constant<int, CC_EPI_GELU>{});
    default: return fail(CC_E_ARG, "gemv: unknown epilogue");
  }
}

int gemv_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
              int epi, cudaStream_t st) {
  return gemv_launch(A, lda, W, ldw, C, ldc, M, N, K, epi, nullptr, 0.f, false, st);
}

}  // namespace ccb

using namespace ccb;

extern "C" int cc_gemv(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N,
                       int K, int epilogue, void* stream) {
  CCB_REQUIRE(M >= 0 && N > 0 && K > 0, "gemv: bad shape");
  if (M == 0) return 0;
  if (!gemv_eligible(M, N, K, epilogue, A, lda, W, ldw))
    return fail(CC_E_UNSUP, "gemv: needs 1..4 rows, K % 8 == 0, 16-byte aligned rows, M*K*2 <= 96 KiB");
  return gemv_bf16(A, lda, W, ldw, C, ldc, M, N, K, epilogue, as_stream(stream));
}

namespace ccb {
namespace {
int decode_attention_impl(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad, void* ctx,
                          float* lse, int n_keys, const int32_t* n_keys_dev, int n_heads, int n_kv_heads, int d_head,
                          cudaStream_t st) {
  CCB_REQUIRE(n_keys >= 1 && n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0, "decode_attention: bad shape");
  CCB_REQUIRE(n_keys <= DA_COMBINE_MAX * DA_KEYS, "decode_attention: more than 512k keys");
  if (d_head != DA_DH) return fail(CC_E_UNSUP, "decode_attention: d_head must be 128");
  const int G = n_heads / n_kv_heads;
  const int n_chunks = (n_keys + DA_KEYS - 1) / DA_KEYS;
  const size_t bytes = (size_t)n_chunks * n_heads * (DA_DH * sizeof(float) + sizeof(float2));
  uint8_t* scratch = (uint8_t*)stream_scratch(st, SCR_DECODE_ATTN, bytes);
  if (!scratch) return fail(CC_E_CUDA, "decode_attention: scratch allocation failed");
  float* part_o = reinterpret_cast<float*>(scratch);
  float2* part_ml = reinterpret_cast<float2*>(scratch + (size_t)n_chunks * n_heads * DA_DH * sizeof(float));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)d_head);
  dim3 grid(n_kv_heads, n_chunks);
  auto go = [&](auto kern) {
    return launch_k(kern, grid, dim3(DA_KEYS), 0, st, "decode_attention", (const __nv_bfloat16*)q,
                    (const __nv_bfloat16*)k_rot, (const __nv_bfloat16*)v, key_pad, part_o, part_ml, n_keys,
                    n_keys_dev, n_heads, n_kv_heads, scale_log2);
  };
  int rc;
  switch (G) {
    case 1: rc = go(decode_attn_partial<1>); break;
    case 2: rc = go(decode_attn_partial<2>); break;
    case 4: rc = go(decode_attn_partial<4>); break;
    case 8: rc = go(decode_attn_partial<8>); break;
    default: return fail(CC_E_UNSUP, "decode_attention: GQA group must be 1, 2, 4 or 8");
  }
  if (rc) return rc;
  return launch_k(decode_attn_combine, dim3(n_heads, DA_DH / 32), dim3(32), 0, st, "decode_attention_combine",
                  (const float*)part_o, (const float2*)part_ml, n_chunks, n_heads, (__nv_bfloat16*)ctx, lse,
                  n_keys_dev);
}

int decode_attention_qkv_impl(const void* qkv, const int32_t* slot, const int32_t* pos, const void* rope_table,
                              void* kv_k, void* kv_v, void* k_rot, const uint8_t* key_pad, void* ctx, float* lse,
                              int n_keys, const int32_t* n_keys_dev, int max_keys, int n_heads, int n_kv_heads,
                              int d_head, cudaStream_t st) {
  CCB_REQUIRE(max_keys >= 1 && n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0 && n_kv_heads <= 1024,
              "decode_attention_qkv: bad shape");
  CCB_REQUIRE(n_keys_dev != nullptr || (n_keys >= 1 && n_keys <= max_keys), "decode_attention_qkv: bad key count");
  if (d_head != DA_DH) return fail(CC_E_UNSUP, "decode_attention_qkv: d_head must be 128");
  static const int use_tc = [] {
    const char* e = getenv("CCB_DECODE_ATTN_TC");
    return e ? atoi(e) : 1;
  }();
  const int kc = use_tc ? DT_KC : DA_KEYS;
  const int n_chunks = (max_keys + kc - 1) / kc;
  if (n_chunks > DF_MAXC) return fail(CC_E_UNSUP, "decode_attention_qkv: too many keys");
  const size_t bytes = (size_t)n_chunks * n_heads * (DA_DH * sizeof(float) + sizeof(float2));
  uint8_t* scratch = (uint8_t*)stream_scratch(st, SCR_DECODE_ATTN, bytes);
  unsigned* tickets = reinterpret_cast<unsigned*>(zeroed_scratch(st, 2, 1024 * sizeof(unsigned)));
  if (!scratch || !tickets) return fail(CC_E_CUDA, "decode_attention_qkv: scratch allocation failed");
  float* part_o = reinterpret_cast<float*>(scratch);
  float2* part_ml = reinterpret_cast<float2*>(scratch + (size_t)n_chunks * n_heads * DA_DH * sizeof(float));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)d_head);
  if (use_tc) {
    auto go_tc = [&](auto kern) {
      if (int rc = ensure_smem(kern, DT_SMEM)) return rc;
      if (g_carveout)
        if (int rc = max_carveout(kern)) return rc;
      return launch_k(kern, dim3(n_kv_heads, n_chunks), dim3(DT_WARPS * 32), DT_SMEM, st, "decode_attention_qkv",
                      (const __nv_bfloat16*)qkv, slot, pos, (const float2*)rope_table, (__nv_bfloat16*)kv_k,
                      (__nv_bfloat16*)kv_v, (__nv_bfloat16*)k_rot, key_pad, part_o, part_ml, tickets,
                      (__nv_bfloat16*)ctx, lse, n_keys, n_keys_dev, max_keys, n_heads, n_kv_heads, scale_log2,
                      g_dt_stage_pre);
    };
    switch (n_heads / n_kv_heads) {
      case 1: return go_tc(decode_attn_tc<1>);
      case 2: return go_tc(decode_attn_tc<2>);
      case 4: return go_tc(decode_attn_tc<4>);
      case 8: return go_tc(decode_attn_tc<8>);
      default: return fail(CC_E_UNSUP, "decode_attention_qkv: GQA group must be 1, 2, 4 or 8");
    }
  }
  auto go = [&](auto kern) {
    return launch_k(kern, dim3(n_kv_heads, n_chunks), dim3(DA_KEYS), 0, st, "decode_attention_qkv",
                    (const __nv_bfloat16*)qkv, slot, pos, (const float2*)rope_table, (__nv_bfloat16*)kv_k,
                    (__nv_bfloat16*)kv_v, (__nv_bfloat16*)k_rot, key_pad, part_o, part_ml, tickets,
                    (__nv_bfloat16*)ctx, lse, n_keys, n_keys_dev, n_heads, n_kv_heads, scale_log2);
  };
  switch (n_heads / n_kv_heads) {
    case 1: return go(decode_attn_fused<1>);
    case 2: return go(decode_attn_fused<2>);
    case 4: return go(decode_attn_fused<4>);
    case 8: return go(decode_attn_fused<8>);
    default: return fail(CC_E_UNSUP, "decode_attention_qkv: GQA group must be 1, 2, 4 or 8");
  }
}

// one decode step's bookkeeping on the device (graph-replayable):
// tokens[state[0]] = *cur_tok; state[0]++ (count); state[1]++ (slot);
// state[2]++ (position); state[3]++ (live keys)
__global__ void decode_advance_kernel(int32_t* state, const int32_t* cur_tok, int32_t* tokens) {
  pdl_trigger();
  pdl_wait();
  tokens[state[0]] = *cur_tok;
  state[0] += 1;
  state[1] += 1;
  state[2] += 1;
  state[3] += 1;
}
}  // namespace
}  // namespace ccb

extern "C" int cc_gemv_rmsnorm(const float* hidden, int64_t ld_hidden, const float* norm_w, double eps,
                               const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K, int epilogue,
                               void* stream) {
  CCB_REQUIRE(M >= 0 && N > 0 && K > 0, "gemv_rmsnorm: bad shape");
  if (M == 0) return 0;
  if (!gemv_eligible(M, N, K, epilogue, W, ldw, W, ldw) || K % 4 || ld_hidden % 4 ||
      (reinterpret_cast<uintptr_t>(hidden) & 15) || (reinterpret_cast<uintptr_t>(norm_w) & 15))
    return fail(CC_E_UNSUP, "gemv_rmsnorm: needs 1..4 rows, K % 8 == 0, 16-byte aligned rows, M*K*2 <= 96 KiB");
  return gemv_launch(hidden, ld_hidden, W, ldw, C, ldc, M, N, K, epilogue, norm_w, (float)eps, true,
                     as_stream(stream));
}

extern "C" int cc_decode_attention(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad, void* ctx,
                                   float* lse, int n_keys, int n_heads, int n_kv_heads, int d_head, void* stream) {
  return decode_attention_impl(q, k_rot, v, key_pad, ctx, lse, n_keys, nullptr, n_heads, n_kv_heads, d_head,
                               as_stream(stream));
}

extern "C" int cc_decode_attention_dev(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad,
                                       void* ctx, float* lse, const int32_t* n_keys_dev, int max_keys, int n_heads,
                                       int n_kv_heads, int d_head, void* stream) {
  CCB_REQUIRE(n_keys_dev != nullptr, "decode_attention_dev: needs the device key count");
  return decode_attention_impl(q, k_rot, v, key_pad, ctx, lse, max_keys, n_keys_dev, n_heads, n_kv_heads, d_head,
                               as_stream(stream));
}

extern "C" int cc_decode_advance(int32_t* state, const int32_t* cur_token, int32_t* tokens, void* stream) {
  return launch_k(decode_advance_kernel, dim3(1), dim3(1), 0, as_stream(stream), "decode_advance", state,
                  cur_token, tokens);
}

extern "C" int cc_rope_rows(const void* x, void* y, int64_t n_rows, int n, int width, const int32_t* positions,
                            const void* rope_table, int d_head, int dtype, void* stream) {
  CCB_REQUIRE(n_rows >= 0 && n >= 1 && width % d_head == 0 && d_head % 2 == 0, "rope_rows: bad shape");
  if (n_rows == 0) return 0;
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    rope_rows_kernel<T><<<(unsigned)n_rows, 128, 0, as_stream(stream)>>>(
        (const T*)x, (T*)y, n, width, positions, (const typename CS<T>::type*)rope_table, d_head);
    return check_launch("rope_rows");
  });
}

extern "C" int cc_decode_attention_qkv(const void* qkv, const int32_t* slot, const int32_t* pos,
                                       const void* rope_table, void* kv_k, void* kv_v, void* k_rot,
                                       const uint8_t* key_pad, void* ctx, float* lse, int n_keys,
                                       const int32_t* n_keys_dev, int max_keys, int n_heads, int n_kv_heads,
                                       int d_head, void* stream) {
  return decode_attention_qkv_impl(qkv, slot, pos, rope_table, kv_k, kv_v, k_rot, key_pad, ctx, lse, n_keys,
                                   n_keys_dev, max_keys, n_heads, n_kv_heads, d_head, as_stream(stream));
}

// Arm (buf != NULL: capacity records of 4 x u64) or disarm the decode-chain timeline.
extern "C" __attribute__((visibility("default"))) int cc_debug_decode_trace(void* buf, int cap) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  unsigned c = buf ? (unsigned)cap : 0u, z = 0u;
  if (cudaMemcpyToSymbol(g_dtrace, &p, sizeof(p)) != cudaSuccess || cudaMemcpyToSymbol(g_dtrace_cap, &c, sizeof(c)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_dtrace_n, &z, sizeof(z)) != cudaSuccess)
    return fail(CC_E_CUDA, "decode_trace: cudaMemcpyToSymbol failed");
  return 0;
}
