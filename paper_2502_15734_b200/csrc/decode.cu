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

#include <type_traits>

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
  pdl_trigger();
  pdl_wait();  // activations come from the predecessor
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

int gemv_launch(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
                int epi, const float* norm_w, float eps, bool norm, cudaStream_t st) {
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
