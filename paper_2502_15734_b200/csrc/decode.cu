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

#include "common.cuh"

namespace ccb {

namespace {

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

constexpr int GV_MAXM = 4;
constexpr int GV_WARPS = 8;

// C[M, N] (+)= epi(A[M, K] W[N, K]^T); SwiGLU: W rows in 64-row gate/up groups,
// output column o = silu(gate row) * up row (N/2 outputs)
template <int EPI>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_kernel(const __nv_bfloat16* __restrict__ A, int64_t lda,
                                                             const __nv_bfloat16* __restrict__ W, int64_t ldw,
                                                             void* __restrict__ C, int64_t ldc, int M, int N, int K) {
  extern __shared__ uint4 xs[];  // [M][K / 8] staged activations
  const int kv8 = K / 8;
  for (int r = 0; r < M; ++r)
    for (int i = threadIdx.x; i < kv8; i += blockDim.x)
      xs[r * kv8 + i] = reinterpret_cast<const uint4*>(A + (int64_t)r * lda)[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool GLU = EPI == CC_EPI_SWIGLU;
  const int n_out = GLU ? N / 2 : N;
  for (int o = blockIdx.x * GV_WARPS + warp; o < n_out; o += gridDim.x * GV_WARPS) {
    const int rg = GLU ? (o / 64) * 128 + (o % 64) : o;
    const uint4* wg = reinterpret_cast<const uint4*>(W + (int64_t)rg * ldw);
    const uint4* wu = reinterpret_cast<const uint4*>(W + (int64_t)(rg + 64) * ldw);
    float ag[GV_MAXM] = {0.f, 0.f, 0.f, 0.f}, au[GV_MAXM] = {0.f, 0.f, 0.f, 0.f};
    int i = lane;
    for (; i + 96 < kv8; i += 128) {  // 4 independent 16-byte weight loads per lane (x2 for SwiGLU)
      uint4 g4[4], u4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        g4[j] = ld_stream16(wg + i + 32 * j);
        if (GLU) u4[j] = ld_stream16(wu + i + 32 * j);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < GV_MAXM; ++r)
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
      for (int r = 0; r < GV_MAXM; ++r)
        if (r < M) {
          const uint4 x = xs[r * kv8 + i];
          ag[r] += dot8(g1, x);
          if (GLU) au[r] += dot8(u1, x);
        }
    }
#pragma unroll
    for (int r = 0; r < GV_MAXM; ++r) {
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
}

// ---- split-KV decode attention ------------------------------------------------
constexpr int DA_KEYS = 128;  // keys per CTA (one per thread)
constexpr int DA_DH = 128;
constexpr int DA_MAXG = 8;

// grid (Hkv, n_chunks); thread t owns key j = chunk * 128 + t for the scores
// and output column t for P.V.  Partials: o [chunk][Hq][DH] (unnormalised),
// ml [chunk][Hq] = (max, sum) in the log2 domain.
template <int G>
__global__ void __launch_bounds__(DA_KEYS) decode_attn_partial(const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ K,
                                                               const __nv_bfloat16* __restrict__ V,
                                                               const uint8_t* __restrict__ key_pad,
                                                               float* __restrict__ part_o, float2* __restrict__ part_ml,
                                                               int n_keys, int Hq, int Hkv, float scale_log2) {
  __shared__ float qs[G][DA_DH];
  __shared__ float ps[G][DA_KEYS];
  __shared__ float2 ml_s[G];
  const int g = blockIdx.x, c = blockIdx.y, t = threadIdx.x;
  const int kvw = Hkv * DA_DH;
  for (int i = t; i < G * DA_DH; i += DA_KEYS) qs[i / DA_DH][i % DA_DH] = __bfloat162float(q[(int64_t)g * G * DA_DH + i]);
  __syncthreads();
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
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 kf = __bfloat1622float2(kb[e]);
#pragma unroll
        for (int h = 0; h < G; ++h) sc[h] = fmaf(kf.x, qs[h][u * 8 + 2 * e], fmaf(kf.y, qs[h][u * 8 + 2 * e + 1], sc[h]));
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h) ps[h][t] = valid ? sc[h] * scale_log2 : -INFINITY;
  __syncthreads();
  // per head: max and exp-sum over the 128 keys (warp w handles heads w, w+4, ...)
  const int warp = t >> 5, lane = t & 31;
  for (int h = warp; h < G; h += DA_KEYS / 32) {
    float v[4], m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = ps[h][lane + 32 * e];
      m = fmaxf(m, v[e]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float l = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
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
  const int cg = t & 15, kg = t >> 4;
  float o[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[h][e] = 0.f;
  const int jn = min(DA_KEYS, n_keys - c * DA_KEYS);
  const __nv_bfloat16* vbase = V + (int64_t)c * DA_KEYS * kvw + g * DA_DH + cg * 8;
  uint4 vv[DA_KEYS / 8];
#pragma unroll
  for (int u = 0; u < DA_KEYS / 8; ++u) {
    const int jj = kg + 8 * u;
    vv[u] = jj < jn ? *reinterpret_cast<const uint4*>(vbase + (int64_t)jj * kvw) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < DA_KEYS / 8; ++u) {
    const int jj = kg + 8 * u;
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
  __shared__ float red[8][G][DA_DH];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[kg][h][cg * 8 + e] = o[h][e];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float acc = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) acc += red[k2][h][t];
    const int head = g * G + h;
    part_o[((int64_t)c * Hq + head) * DA_DH + t] = acc;
    if (t == 0) part_ml[(int64_t)c * Hq + head] = ml_s[h];
  }
}

// grid Hq, 128 threads: fold the chunks in index order
__global__ void __launch_bounds__(DA_DH) decode_attn_combine(const float* __restrict__ part_o,
                                                             const float2* __restrict__ part_ml, int n_chunks, int Hq,
                                                             __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse) {
  const int head = blockIdx.x, t = threadIdx.x;
  float m = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) m = fmaxf(m, part_ml[(int64_t)c * Hq + head].x);
  float l = 0.f, o = 0.f;
  if (m != -INFINITY) {
    for (int c = 0; c < n_chunks; ++c) {
      const float2 ml = part_ml[(int64_t)c * Hq + head];
      if (ml.x == -INFINITY) continue;
      const float w = exp2f(ml.x - m);
      l = fmaf(ml.y, w, l);
      o = fmaf(part_o[((int64_t)c * Hq + head) * DA_DH + t], w, o);
    }
  }
  ctx[(int64_t)head * DA_DH + t] = __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
  if (t == 0 && lse != nullptr) lse[head] = l > 0.f ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
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

int gemv_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
              int epi, cudaStream_t st) {
  const int n_out = epi == CC_EPI_SWIGLU ? N / 2 : N;
  const size_t smem = (size_t)M * K * 2;
  int grid = (n_out + GV_WARPS - 1) / GV_WARPS;
  static bool attr = false;  // (the four instantiations share one function-pointer type)
  if (!attr) {
    cudaFuncSetAttribute(gemv_kernel<CC_EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(gemv_kernel<CC_EPI_RESID_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(gemv_kernel<CC_EPI_SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(gemv_kernel<CC_EPI_GELU>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  auto go = [&](auto kern) {
    kern<<<grid, GV_WARPS * 32, smem, st>>>((const __nv_bfloat16*)A, lda, (const __nv_bfloat16*)W, ldw, C, ldc, M, N,
                                            K);
    return check_launch("gemv");
  };
  switch (epi) {
    case CC_EPI_STORE: return go(gemv_kernel<CC_EPI_STORE>);
    case CC_EPI_RESID_ADD: return go(gemv_kernel<CC_EPI_RESID_ADD>);
    case CC_EPI_SWIGLU: return go(gemv_kernel<CC_EPI_SWIGLU>);
    case CC_EPI_GELU: return go(gemv_kernel<CC_EPI_GELU>);
    default: return fail(CC_E_ARG, "gemv: unknown epilogue");
  }
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

extern "C" int cc_decode_attention(const void* q, const void* k_rot, const void* v, const uint8_t* key_pad, void* ctx,
                                   float* lse, int n_keys, int n_heads, int n_kv_heads, int d_head, void* stream) {
  CCB_REQUIRE(n_keys >= 1 && n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0, "decode_attention: bad shape");
  if (d_head != DA_DH) return fail(CC_E_UNSUP, "decode_attention: d_head must be 128");
  const int G = n_heads / n_kv_heads;
  const int n_chunks = (n_keys + DA_KEYS - 1) / DA_KEYS;
  cudaStream_t st = as_stream(stream);
  const size_t bytes = (size_t)n_chunks * n_heads * (DA_DH * sizeof(float) + sizeof(float2));
  uint8_t* scratch = (uint8_t*)stream_scratch(st, 2, bytes);
  if (!scratch) return fail(CC_E_CUDA, "decode_attention: scratch allocation failed");
  float* part_o = reinterpret_cast<float*>(scratch);
  float2* part_ml = reinterpret_cast<float2*>(scratch + (size_t)n_chunks * n_heads * DA_DH * sizeof(float));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)d_head);
  dim3 grid(n_kv_heads, n_chunks);
  auto go = [&](auto kern) {
    kern<<<grid, DA_KEYS, 0, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k_rot, (const __nv_bfloat16*)v,
                                   key_pad, part_o, part_ml, n_keys, n_heads, n_kv_heads, scale_log2);
    return check_launch("decode_attention");
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
  decode_attn_combine<<<n_heads, DA_DH, 0, st>>>(part_o, part_ml, n_chunks, n_heads, (__nv_bfloat16*)ctx, lse);
  return check_launch("decode_attention_combine");
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
