// Attention over scattered query rows (model.py:406-416) — SIMT kernels for
// the f64/f32 parity modes, softmax materialisation for AttentionRecord
// (model.py:320-335), and the K8a segment-mass statistics (stats.py:68-106).
//
// Masking rule shared by every kernel: query row r (slot q_slot[r]) sees key
// j iff j <= q_slot[r] and key_pad[j] == 0.  Slots are laid out in position
// order with pads consuming no position (model.py:236-238), so this equals
// the reference's `pos_k <= pos_q & ~pad_k` (model.py:409).
#include <math.h>

#include "attention.cuh"
#include "common.cuh"

namespace ccb {

template <typename A>
__device__ __forceinline__ A blk_reduce(A v, A* red, bool is_max) {
  for (int o = 16; o > 0; o >>= 1) {
    A t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? (t > v ? t : v) : v + t;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  A r = red[0];
  for (int i = 1; i < nw; ++i) r = is_max ? (red[i] > r ? red[i] : r) : r + red[i];
  return r;
}

template <typename T>
__device__ __forceinline__ typename Acc<T>::type dot_row(const typename Acc<T>::type* qs, const T* k, int dh) {
  using A = typename Acc<T>::type;
  A s = 0;
  for (int d = 0; d < dh; ++d) s += qs[d] * (A)to_f(k[d]);
  return s;
}

// one CTA per (query row, head); 128 threads; keys in tiles of 128
template <typename T>
__global__ void __launch_bounds__(128) attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                        const T* __restrict__ v, const int32_t* __restrict__ q_slot,
                                                        const uint8_t* __restrict__ key_pad, T* __restrict__ ctx,
                                                        typename Acc<T>::type* __restrict__ lse, int Hq, int Hkv,
                                                        int dh) {
  using A = typename Acc<T>::type;
  __shared__ A qs[256];
  __shared__ A ps[128];
  __shared__ A red[4];
  const int r = blockIdx.x, h = blockIdx.y, g = h / (Hq / Hkv);
  const int tid = threadIdx.x;
  const A scale = (A)1 / sqrt((A)dh);
  for (int d = tid; d < dh; d += 128) qs[d] = (A)to_f(q[((int64_t)r * Hq + h) * dh + d]);
  __syncthreads();
  const int limit = q_slot[r];
  A m = -INFINITY, l = 0, acc0 = 0, acc1 = 0;
  for (int kt = 0; kt <= limit; kt += 128) {
    const int j = kt + tid;
    A s = -INFINITY;
    if (j <= limit && !(key_pad && key_pad[j])) s = dot_row<T>(qs, k + ((int64_t)j * Hkv + g) * dh, dh) * scale;
    A tmax = blk_reduce<A>(s, red, true);
    A m_new = tmax > m ? tmax : m;
    if (m_new == -INFINITY) { __syncthreads(); continue; }
    A p = (s == -INFINITY) ? (A)0 : exp(s - m_new);
    ps[tid] = p;
    A lt = blk_reduce<A>(p, red, false);
    A alpha = (m == -INFINITY) ? (A)0 : exp(m - m_new);
    l = l * alpha + lt;
    const int nk = min(128, limit - kt + 1);
    for (int d = tid, c = 0; d < dh; d += 128, ++c) {
      A a = 0;
      for (int t = 0; t < nk; ++t) a += ps[t] * (A)to_f(v[((int64_t)(kt + t) * Hkv + g) * dh + d]);
      if (c == 0) acc0 = acc0 * alpha + a; else acc1 = acc1 * alpha + a;
    }
    m = m_new;
    __syncthreads();
  }
  const A inv = l > 0 ? (A)1 / l : (A)0;
  for (int d = tid, c = 0; d < dh; d += 128, ++c) {
    A o = (c == 0 ? acc0 : acc1) * inv;
    if constexpr (sizeof(A) == 8) ctx[(int64_t)r * Hq * dh + h * dh + d] = from_d<T>(o);
    else ctx[(int64_t)r * Hq * dh + h * dh + d] = from_f<T>(o);
  }
  if (tid == 0) lse[(int64_t)r * Hq + h] = (l > 0) ? m + log(l) : (A)-INFINITY;
}

// probs[h][r][j] = exp(s - lse) or 0 where masked
template <typename T>
__global__ void __launch_bounds__(128) attn_probs_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                         const int32_t* __restrict__ q_slot,
                                                         const uint8_t* __restrict__ key_pad,
                                                         const typename Acc<T>::type* __restrict__ lse,
                                                         typename Acc<T>::type* __restrict__ probs, int n_q,
                                                         int n_keys, int Hq, int Hkv, int dh) {
  using A = typename Acc<T>::type;
  __shared__ A qs[256];
  const int r = blockIdx.x, h = blockIdx.y, g = h / (Hq / Hkv);
  const A scale = (A)1 / sqrt((A)dh);
  for (int d = threadIdx.x; d < dh; d += blockDim.x) qs[d] = (A)to_f(q[((int64_t)r * Hq + h) * dh + d]);
  __syncthreads();
  const int limit = q_slot[r];
  const A L = lse[(int64_t)r * Hq + h];
  A* out = probs + ((int64_t)h * n_q + r) * n_keys;
  for (int j = threadIdx.x; j < n_keys; j += blockDim.x) {
    A p = 0;
    if (j <= limit && !(key_pad && key_pad[j])) p = exp(dot_row<T>(qs, k + ((int64_t)j * Hkv + g) * dh, dh) * scale - L);
    out[j] = p;
  }
}

// K8a: one CTA per stats row; heads in order; per segment a fixed-shape
// block reduction -> deterministic.  mass[s][seg] and diag in mass[s][n_seg].
template <typename T>
__global__ void __launch_bounds__(256) segment_mass_kernel(
    const T* __restrict__ q, const T* __restrict__ k, const int32_t* __restrict__ q_slot,
    const uint8_t* __restrict__ key_pad, const typename Acc<T>::type* __restrict__ lse,
    const int32_t* __restrict__ seg_lo, const int32_t* __restrict__ seg_hi, int n_seg,
    const int32_t* __restrict__ rows, double* __restrict__ mass, int Hq, int Hkv, int dh) {
  using A = typename Acc<T>::type;
  __shared__ A qs[256];
  __shared__ double red[8];
  const int s_idx = blockIdx.x;
  const int r = rows[s_idx];
  const int limit = q_slot[r];
  const A scale = (A)1 / sqrt((A)dh);
  double* out = mass + (int64_t)s_idx * (n_seg + 1);
  double diag = 0;
  for (int sg = threadIdx.x; sg < n_seg; sg += blockDim.x) out[sg] = 0;
  __syncthreads();
  for (int h = 0; h < Hq; ++h) {
    const int g = h / (Hq / Hkv);
    __syncthreads();
    for (int d = threadIdx.x; d < dh; d += blockDim.x) qs[d] = (A)to_f(q[((int64_t)r * Hq + h) * dh + d]);
    __syncthreads();
    const A L = lse[(int64_t)r * Hq + h];
    for (int sg = 0; sg < n_seg; ++sg) {
      const int lo = seg_lo[sg], hi = min(seg_hi[sg], limit + 1);
      double part = 0;
      for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        if (key_pad && key_pad[j]) continue;
        double p = (double)exp(dot_row<T>(qs, k + ((int64_t)j * Hkv + g) * dh, dh) * scale - L);
        part += p;
        if (j == limit) diag += p;
      }
      double tot = blk_reduce<double>(part, red, false);
      if (threadIdx.x == 0) out[sg] += tot;
    }
  }
  double dtot = blk_reduce<double>(diag, red, false);
  __syncthreads();
  if (threadIdx.x == 0) out[n_seg] = dtot / Hq;
  for (int sg = threadIdx.x; sg < n_seg; sg += blockDim.x) out[sg] /= Hq;
}

int attention_simt(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                   void* ctx, void* lse, int n_q, int n_keys, int Hq, int Hkv, int dh, int dtype, cudaStream_t st) {
  CCB_REQUIRE(dh <= 256, "attention: d_head must be <= 256");
  note_simt(dtype);
  dim3 grid(n_q, Hq);
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    attn_simt_kernel<T><<<grid, 128, 0, st>>>((const T*)q, (const T*)k, (const T*)v, q_slot, key_pad, (T*)ctx,
                                              (typename Acc<T>::type*)lse, Hq, Hkv, dh);
    return check_launch("attention_simt");
  });
}

}  // namespace ccb

using namespace ccb;

extern "C" {

int cc_attention(const void* q, const void* k_rot, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                 void* ctx, void* lse, int n_q, int n_keys, int n_heads, int n_kv_heads, int d_head, int dtype,
                 int impl, void* stream) {
  CCB_REQUIRE(n_kv_heads > 0 && n_heads % n_kv_heads == 0, "attention: n_heads must be a multiple of n_kv_heads");
  CCB_REQUIRE(d_head > 0 && d_head <= 256, "attention: bad d_head");
  if (n_q == 0) return 0;
  cudaStream_t st = as_stream(stream);
  // impl: 0 product path (bf16: the tcgen05 kernel only -- an unsupported
  // shape is an error, never a silent slower kernel; fp32/fp64 parity modes:
  // SIMT), 1 tcgen05, 2 SIMT reference (tests)
  if (dtype == CC_BF16 && impl != 2)
    return attention_tc_bf16(q, k_rot, v, q_slot, key_pad, ctx, (float*)lse, n_q, n_keys, n_heads, n_kv_heads,
                             d_head, st);
  if (impl == 1) return fail(CC_E_UNSUP, "attention: tcgen05 kernel requires bf16");
  return attention_simt(q, k_rot, v, q_slot, key_pad, ctx, lse, n_q, n_keys, n_heads, n_kv_heads, d_head, dtype, st);
}

int cc_attention_probs(const void* q, const void* k_rot, const int32_t* q_slot, const uint8_t* key_pad,
                       const void* lse, void* probs, int n_q, int n_keys, int n_heads, int n_kv_heads, int d_head,
                       int dtype, void* stream) {
  if (n_q == 0) return 0;
  CCB_REQUIRE(d_head <= 256, "attention_probs: d_head must be <= 256");
  dim3 grid(n_q, n_heads);
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    using A = typename Acc<T>::type;
    attn_probs_kernel<T><<<grid, 128, 0, as_stream(stream)>>>((const T*)q, (const T*)k_rot, q_slot, key_pad,
                                                              (const A*)lse, (A*)probs, n_q, n_keys, n_heads,
                                                              n_kv_heads, d_head);
    return check_launch("attention_probs");
  });
}

int cc_segment_mass(const void* q, const void* k_rot, const int32_t* q_slot, const uint8_t* key_pad, const void* lse,
                    const int32_t* seg_lo, const int32_t* seg_hi, int n_seg, const int32_t* rows, int n_rows,
                    double* mass, int n_keys, int n_heads, int n_kv_heads, int d_head, int dtype, void* stream) {
  if (n_rows == 0) return 0;
  CCB_REQUIRE(d_head <= 256, "segment_mass: d_head must be <= 256");
  if (dtype == CC_BF16)  // tcgen05 only: no silent SIMT fallback in the product path
    return segment_mass_tc_bf16(q, k_rot, q_slot, key_pad, (const float*)lse, seg_lo, seg_hi, n_seg, rows, n_rows,
                                mass, n_keys, n_heads, n_kv_heads, d_head, as_stream(stream));
  note_simt(dtype);
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    using A = typename Acc<T>::type;
    segment_mass_kernel<T><<<n_rows, 256, 0, as_stream(stream)>>>((const T*)q, (const T*)k_rot, q_slot, key_pad,
                                                                  (const A*)lse, seg_lo, seg_hi, n_seg, rows, mass,
                                                                  n_heads, n_kv_heads, d_head);
    return check_launch("segment_mass");
  });
}

}  // extern "C"
