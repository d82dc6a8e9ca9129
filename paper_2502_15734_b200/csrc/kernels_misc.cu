// Memory-bound kernels of the fix-up prefill path:
//   K1  gather + RoPE of cached chunk K/V      (model.py:387-393, :404; rpe.py:34-44)
//   K3e RoPE + scatter of fresh Q/K/V rows       (model.py:399-404)
//   K2  RMSNorm                                  (model.py:121-122)
//   K7  logits + greedy argmax                   (model.py:94-95, :455)
//   K8b chunk statistics reduction               (harness.py:331-354, stats.py:68-106)
//   K9  per-chunk top-k selection                (planner.py:17-34)
//   K10 extract fresh chunk rows into pool blocks (model.py:487-492, store.py:30-53)
// plus the RoPE table, embedding rows and an L2 flush helper.
#include <float.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <type_traits>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace ccb {

template <typename T, int N>
struct alignas(sizeof(T) * N) Vec {
  T v[N];
};

// pick the widest vector (<=16 B) whose element count divides `n`
template <typename T>
inline int pick_vec(int n) {
  int v = 16 / (int)sizeof(T);
  while (v > 1 && (n % v) != 0) v /= 2;
  return v;
}

#define CCB_DISPATCH_VEC(vec, V, ...)                  \
  [&]() -> int {                                       \
    switch (vec) {                                     \
      case 8: { constexpr int V = 8; return __VA_ARGS__(); } \
      case 4: { constexpr int V = 4; return __VA_ARGS__(); } \
      case 2: { constexpr int V = 2; return __VA_ARGS__(); } \
      default: { constexpr int V = 1; return __VA_ARGS__(); } \
    }                                                  \
  }()

// ---------------------------------------------------------------------------
// RoPE table: (cos, sin) of pos * inv_freq[j], angles in fp64 (rpe.py:34-37)
// ---------------------------------------------------------------------------
template <typename C>
__global__ void rope_table_kernel(C* table, const double* inv_freq, int max_pos, int half) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)max_pos * half) return;
  int p = (int)(i / half), j = (int)(i % half);
  double ang = (double)p * inv_freq[j];
  double s, c;
  sincos(ang, &s, &c);
  C out;
  out.x = c;
  out.y = s;
  table[i] = out;
}

// apply_rpe / remove_rpe in float64 (rpe.py:19-44)
__global__ void rope_apply_f64_kernel(const double* __restrict__ x, double* __restrict__ y,
                                      const int64_t* __restrict__ pos, int n, int width, int dh,
                                      const double* __restrict__ inv_freq, double sign) {
  int half = dh / 2;
  int64_t total = (int64_t)n * (width / 2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(i / (width / 2));
    int rem = (int)(i % (width / 2));
    int h = rem / half, j = rem % half;
    double ang = sign * (double)pos[r] * inv_freq[j];
    double s, c;
    sincos(ang, &s, &c);
    const double* row = x + (int64_t)r * width + h * dh;
    double a = row[j], b = row[j + half];
    double* out = y + (int64_t)r * width + h * dh;
    out[j] = a * c - b * s;
    out[j + half] = a * s + b * c;
  }
}

// ---------------------------------------------------------------------------
// K1: gather + RoPE.  One CTA per (gather item, layer).  Each CTA moves one
// 16-row pool block: K rows -> kv_k (copy) and k_rot (rotated at the slot's
// position), V rows -> kv_v.  Vectorised 16-byte accesses; pairs (j, j+half)
// of a head are loaded together so the rotation needs no shuffles.
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) gather_rope_kernel(
    const T* __restrict__ pool, int64_t pool_layer_stride, int64_t pool_block_stride,
    const cc_gather_item* __restrict__ items, int l0, const int32_t* __restrict__ slot_pos,
    const int32_t* __restrict__ active_until, const typename CS<T>::type* __restrict__ table,
    T* __restrict__ kv_k, T* __restrict__ kv_v, T* __restrict__ k_rot, int64_t req_layer_stride,
    int kvw, int dh) {
  using A = typename Acc<T>::type;
  using VT = Vec<T, V>;
  pdl_trigger();
  pdl_wait();
  const cc_gather_item it = items[blockIdx.x];
  const int l = l0 + blockIdx.y;
  const int half = dh / 2;
  const int hv = half / V;           // vectors per half-head
  const int nh = kvw / dh;           // kv heads
  const T* src = pool + (int64_t)l * pool_layer_stride + (int64_t)it.src_block * pool_block_stride;
  const T* srcK = src;
  const T* srcV = src + 16 * (int64_t)kvw;
  const int64_t lofs = (int64_t)l * req_layer_stride;
  // K: rotate pairs
  const int k_units = it.n_rows * nh * hv;
  for (int u = threadIdx.x; u < k_units; u += blockDim.x) {
    int r = u / (nh * hv);
    int rem = u % (nh * hv);
    int h = rem / hv, jv = rem % hv;
    int slot = it.dst_slot + r;
    if (active_until[slot] > l) continue;
    int64_t off = (int64_t)r * kvw + h * dh + jv * V;
    VT x = *reinterpret_cast<const VT*>(srcK + off);
    VT y = *reinterpret_cast<const VT*>(srcK + off + half);
    int64_t doff = lofs + (int64_t)slot * kvw + h * dh + jv * V;
    *reinterpret_cast<VT*>(kv_k + doff) = x;
    *reinterpret_cast<VT*>(kv_k + doff + half) = y;
    const typename CS<T>::type* cs = table + (int64_t)slot_pos[slot] * half + jv * V;
    VT xr, yr;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      A c = (A)cs[e].x, s = (A)cs[e].y;
      A a = (A)to_f(x.v[e]), b = (A)to_f(y.v[e]);
      if constexpr (sizeof(A) == 8) {
        xr.v[e] = from_d<T>(a * c - b * s);
        yr.v[e] = from_d<T>(a * s + b * c);
      } else {
        xr.v[e] = from_f<T>(a * c - b * s);
        yr.v[e] = from_f<T>(a * s + b * c);
      }
    }
    *reinterpret_cast<VT*>(k_rot + doff) = xr;
    *reinterpret_cast<VT*>(k_rot + doff + half) = yr;
  }
  // V: copy
  const int vpr = kvw / V;
  const int v_units = it.n_rows * vpr;
  for (int u = threadIdx.x; u < v_units; u += blockDim.x) {
    int r = u / vpr, c = u % vpr;
    int slot = it.dst_slot + r;
    if (active_until[slot] > l) continue;
    VT x = *reinterpret_cast<const VT*>(srcV + (int64_t)r * kvw + c * V);
    *reinterpret_cast<VT*>(kv_v + lofs + (int64_t)slot * kvw + c * V) = x;
  }
}

// ---------------------------------------------------------------------------
// K1, TMA-staged (the default): one CTA per (gather item, column chunk,
// layer), three per SM.  Warp 0 stages the block's live K and V rows into
// shared memory with bulk copies (cp.async.bulk completing on one mbarrier)
// and sends them straight back out to kv_k / kv_v with bulk stores; a run of
// consecutive live rows is one contiguous segment on both sides when the
// chunk spans the full row (the block's rows land on consecutive request
// slots), so a fully live 16-row block is 2 loads + 2 stores -- the TMA unit
// costs ~50 ns per bulk operation whatever its size, per-row copies would be
// operation-bound.  While the copies are in flight every thread fetches the
// (cos, sin) coefficients of its rotation units; then the CTA rotates K out
// of shared memory into k_rot with 16-byte stores.  Rows recomputed at the
// layer (active_until[slot] > l) are neither loaded nor stored.  Same
// arithmetic as gather_rope_kernel (bit-identical output).
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256, 3) gather_rope_bulk_kernel(
    const T* __restrict__ pool, int64_t pool_layer_stride, int64_t pool_block_stride,
    const cc_gather_item* __restrict__ items, int l0, const int32_t* __restrict__ slot_pos,
    const int32_t* __restrict__ active_until, const typename CS<T>::type* __restrict__ table,
    T* __restrict__ kv_k, T* __restrict__ kv_v, T* __restrict__ k_rot, int64_t req_layer_stride,
    int kvw, int dh, int cols, int stg) {
  using namespace sm100;
  using A = typename Acc<T>::type;
  using VT = Vec<T, V>;
  using C2 = typename CS<T>::type;
  constexpr int UPT = 4;  // rotation units per thread per round (coefficients held in registers)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  T* sK = reinterpret_cast<T*>(smem_raw);
  T* sV = sK + 16 * cols;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + 16 * cols);
  __shared__ uint32_t s_mask;
  pdl_trigger();
  pdl_wait();
  const int nchunk = kvw / cols;
  const cc_gather_item it = items[blockIdx.x / nchunk];
  const int c0 = (blockIdx.x % nchunk) * cols;
  const int l = l0 + blockIdx.y;
  const int tid = threadIdx.x;
  const uint32_t row_bytes = (uint32_t)cols * sizeof(T);
  const int64_t lofs = (int64_t)l * req_layer_stride;
  int len = 0;  // warp 0: the run of live rows starting at row tid
  if (tid < 32) {
    const bool live = tid < it.n_rows && active_until[it.dst_slot + tid] <= l;
    const uint32_t m = __ballot_sync(0xffffffffu, live);
    if (live) len = cols < kvw ? 1 : (tid > 0 && ((m >> (tid - 1)) & 1u)) ? 0 : __ffs(~(m >> tid)) - 1;
    if (tid == 0) {
      s_mask = m;
      mbar_init(bar, 1);
      fence_proxy_async_smem();  // the init is visible to the async proxy
      if (m) mbar_expect_tx(bar, 2u * __popc(m) * row_bytes);
    }
    __syncwarp();
    if (len) {
      const T* src = pool + (int64_t)l * pool_layer_stride + (int64_t)it.src_block * pool_block_stride +
                     (int64_t)tid * kvw + c0;
      bulk_load_1d(sK + tid * cols, src, len * row_bytes, bar);
      bulk_load_1d(sV + tid * cols, src + 16 * (int64_t)kvw, len * row_bytes, bar);
    }
  }
  __syncthreads();
  const uint32_t m = s_mask;
  if (!m) return;
  const int half = dh / 2, hv = half / V, nh = cols / dh;
  const int units = 16 * nh * hv;
  // the staged rows have landed: K and V leave for kv_k / kv_v
  auto stage_out = [&]() {
    mbar_wait(bar, 0);
    if (stg) {  // (experiment) position-free K and V written by the threads
      const int vpr = cols / V;
      for (int w = tid; w < 16 * vpr; w += 256) {
        const int r = w / vpr, c = w % vpr;
        if (!((m >> r) & 1u)) continue;
        const int64_t doff = lofs + (int64_t)(it.dst_slot + r) * kvw + c0 + c * V;
        *reinterpret_cast<VT*>(kv_k + doff) = *reinterpret_cast<const VT*>(sK + r * cols + c * V);
        *reinterpret_cast<VT*>(kv_v + doff) = *reinterpret_cast<const VT*>(sV + r * cols + c * V);
      }
    } else if (len) {  // position-free K and V leave as loaded
      const int64_t doff = lofs + (int64_t)(it.dst_slot + tid) * kvw + c0;
      bulk_store_1d(kv_k + doff, sK + tid * cols, len * row_bytes);
      bulk_store_1d(kv_v + doff, sV + tid * cols, len * row_bytes);
      bulk_commit();
    }
  };
  bool staged = false;
  for (int base = tid; base < units; base += UPT * 256) {
    C2 cs[UPT][V];
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
      const int w = base + k * 256;
      const int r = w / (nh * hv), jv = (w % (nh * hv)) % hv;
      if (w < units && ((m >> r) & 1u)) {
        const C2* t = table + (int64_t)slot_pos[it.dst_slot + r] * half + jv * V;
#pragma unroll
        for (int e = 0; e < V; ++e) cs[k][e] = t[e];
      }
    }
    if (!staged) {
      stage_out();
      staged = true;
    }
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
      const int w = base + k * 256;
      const int r = w / (nh * hv), rem = w % (nh * hv);
      if (w >= units || !((m >> r) & 1u)) continue;
      const int h = rem / hv, jv = rem % hv;
      const int off = r * cols + h * dh + jv * V;
      const VT x = *reinterpret_cast<const VT*>(sK + off);
      const VT y = *reinterpret_cast<const VT*>(sK + off + half);
      VT xr, yr;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        A c = (A)cs[k][e].x, s = (A)cs[k][e].y;
        A a = (A)to_f(x.v[e]), b = (A)to_f(y.v[e]);
        if constexpr (sizeof(A) == 8) {
          xr.v[e] = from_d<T>(a * c - b * s);
          yr.v[e] = from_d<T>(a * s + b * c);
        } else {
          xr.v[e] = from_f<T>(a * c - b * s);
          yr.v[e] = from_f<T>(a * s + b * c);
        }
      }
      const int64_t doff = lofs + (int64_t)(it.dst_slot + r) * kvw + c0 + h * dh + jv * V;
      *reinterpret_cast<VT*>(k_rot + doff) = xr;
      *reinterpret_cast<VT*>(k_rot + doff + half) = yr;
    }
  }
  if (!staged) stage_out();  // (threads without rotation units)
  if (len && !stg) bulk_wait_read<0>();  // shared memory stays valid until the stores have read it
}

// ---------------------------------------------------------------------------
// Fresh rows after the QKV GEMM: rotate q and k, scatter k/v into the
// request KV (position-free k, rotated k for attention).  One CTA per row.
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(1024) rope_scatter_kernel(
    const T* __restrict__ qkv, int64_t ld, const int32_t* __restrict__ row_slot,
    const int32_t* __restrict__ row_pos, const typename CS<T>::type* __restrict__ table,
    T* __restrict__ q_rot, T* __restrict__ kv_k, T* __restrict__ kv_v, T* __restrict__ k_rot,
    int Hq, int Hkv, int dh) {
  pdl_trigger();
  pdl_wait();
  using A = typename Acc<T>::type;
  using VT = Vec<T, V>;
  const int r = blockIdx.x;
  const int half = dh / 2, hv = half / V;
  const int slot = row_slot[r];
  const typename CS<T>::type* cs_row = table + (int64_t)row_pos[r] * half;
  const T* row = qkv + (int64_t)r * ld;
  const int kvw = Hkv * dh;
  const int rot_units = (Hq + Hkv) * hv;
  // work units: a rotated pair of V-vectors of a q or k head, or a V-vector of v
  for (int u = threadIdx.x; u < rot_units + kvw / V; u += blockDim.x) {
    if (u >= rot_units) {
      const int c = u - rot_units;
      const T* vrow = row + (int64_t)(Hq + Hkv) * dh;
      *reinterpret_cast<VT*>(kv_v + (int64_t)slot * kvw + c * V) = *reinterpret_cast<const VT*>(vrow + c * V);
      continue;
    }
    int h = u / hv, jv = u % hv;
    bool is_q = h < Hq;
    int64_t off = (int64_t)h * dh + jv * V;  // q heads then k heads are contiguous in the row
    VT x = *reinterpret_cast<const VT*>(row + off);
    VT y = *reinterpret_cast<const VT*>(row + off + half);
    VT xr, yr;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      A c = (A)cs_row[jv * V + e].x, s = (A)cs_row[jv * V + e].y;
      A a = (A)to_f(x.v[e]), b = (A)to_f(y.v[e]);
      if constexpr (sizeof(A) == 8) {
        xr.v[e] = from_d<T>(a * c - b * s);
        yr.v[e] = from_d<T>(a * s + b * c);
      } else {
        float fx, fy;
        rope_pair(a, b, c, s, fx, fy);
        xr.v[e] = from_f<T>(fx);
        yr.v[e] = from_f<T>(fy);
      }
    }
    if (is_q) {
      T* dst = q_rot + (int64_t)r * Hq * dh + off;
      *reinterpret_cast<VT*>(dst) = xr;
      *reinterpret_cast<VT*>(dst + half) = yr;
    } else {
      int64_t koff = (int64_t)slot * kvw + (h - Hq) * dh + jv * V;
      *reinterpret_cast<VT*>(kv_k + koff) = x;
      *reinterpret_cast<VT*>(kv_k + koff + half) = y;
      *reinterpret_cast<VT*>(k_rot + koff) = xr;
      *reinterpret_cast<VT*>(k_rot + koff + half) = yr;
    }
  }
}

// ---------------------------------------------------------------------------
// embedding rows and RMSNorm
// ---------------------------------------------------------------------------
template <typename T>
__global__ void embed_kernel(const T* __restrict__ embed, const int32_t* __restrict__ tok,
                             typename Acc<T>::type* __restrict__ hidden, int d) {
  pdl_trigger();
  pdl_wait();
  using A = typename Acc<T>::type;
  const T* src = embed + (int64_t)tok[blockIdx.x] * d;
  A* dst = hidden + (int64_t)blockIdx.x * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = (A)to_f(src[i]);
}

template <typename A>
__device__ __forceinline__ A block_sum(A v, A* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  A t = 0;
  if (threadIdx.x < 32) {
    t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : (A)0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Register-resident RMSNorm: one 128-thread CTA per row, the row read once
// with 16-byte loads (d / 512 float4 per thread), one block reduction.
template <typename T, int NV>
__global__ void __launch_bounds__(128) rmsnorm_vec_kernel(const float* __restrict__ h, T* __restrict__ out,
                                                          const float* __restrict__ w, int d, float eps) {
  __shared__ float red[4];
  pdl_trigger();
  pdl_wait();
  const float4* x = reinterpret_cast<const float4*>(h + (int64_t)blockIdx.x * d);
  float4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = x[threadIdx.x + i * 128];
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  ss = (red[0] + red[1]) + (red[2] + red[3]);
  const float inv = 1.f / sqrtf(ss / (float)d + eps);
  T* y = out + (int64_t)blockIdx.x * d;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (threadIdx.x + i * 128) * 4;
    float4 wv = w ? *reinterpret_cast<const float4*>(w + c) : make_float4(1.f, 1.f, 1.f, 1.f);
    float a0 = v[i].x * inv * wv.x, a1 = v[i].y * inv * wv.y, a2 = v[i].z * inv * wv.z, a3 = v[i].w * inv * wv.w;
    if constexpr (sizeof(T) == 2) {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(a0, a1), p1 = __floats2bfloat162_rn(a2, a3);
      uint2 pk = make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
      *reinterpret_cast<uint2*>(y + c) = pk;
    } else {
      *reinterpret_cast<float4*>(y + c) = make_float4(a0, a1, a2, a3);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const typename Acc<T>::type* __restrict__ h,
                                                      T* __restrict__ out, const float* __restrict__ w,
                                                      int d, double eps) {
  using A = typename Acc<T>::type;
  __shared__ A red[32];
  const A* x = h + (int64_t)blockIdx.x * d;
  A ss = 0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += x[i] * x[i];
  ss = block_sum<A>(ss, red);
  A inv = (A)1 / sqrt(ss / (A)d + (A)eps);
  T* y = out + (int64_t)blockIdx.x * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    A v = x[i] * inv;
    if (w) v *= (A)w[i];
    if constexpr (sizeof(A) == 8) y[i] = from_d<T>(v); else y[i] = from_f<T>(v);
  }
}

// ---------------------------------------------------------------------------
// K7 logits (GEMV over the unembedding, bandwidth-bound) + argmax
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) logits_kernel(const typename Acc<T>::type* __restrict__ hrows,
                                                     const float* __restrict__ w, double eps,
                                                     const T* __restrict__ U, typename Acc<T>::type* __restrict__ logits,
                                                     int m, int d, int vocab) {
  pdl_trigger();
  pdl_wait();
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* xs = reinterpret_cast<A*>(smem_raw);  // [m][d] normed rows
  __shared__ A red[32];
  for (int r = 0; r < m; ++r) {
    const A* x = hrows + (int64_t)r * d;
    A ss = 0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss += x[i] * x[i];
    ss = block_sum<A>(ss, red);
    A inv = (A)1 / sqrt(ss / (A)d + (A)eps);
    for (int i = threadIdx.x; i < d; i += blockDim.x) xs[r * d + i] = x[i] * inv * (w ? (A)w[i] : (A)1);
  }
  __syncthreads();
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  // one warp per vocab row: the row is streamed ONCE (16-byte no-allocate
  // loads, 4 in flight per lane) and dotted with all m normed rows
  for (int v = blockIdx.x * warps + (threadIdx.x >> 5); v < vocab; v += gridDim.x * warps) {
    const T* u = U + (int64_t)v * d;
    A acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0;
    if constexpr (sizeof(T) == 2) {
      auto ld = [&](int i) {
        uint4 raw;
        asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
            : "l"(u + i));
        return raw;
      };
      auto dot = [&](const uint4& raw, int i) {
        const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < m) {
            const A* x = xs + r * d + i;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[r] += __bfloat162float(hb[e]) * x[e];
          }
        }
      };
      int i = lane * 8;
      for (; i + 3 * 256 < d; i += 4 * 256) {  // 4 independent 16-byte loads in flight
        uint4 raw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) raw[j] = ld(i + j * 256);
#pragma unroll
        for (int j = 0; j < 4; ++j) dot(raw[j], i + j * 256);
      }
      for (; i < d; i += 256) dot(ld(i), i);
    } else {
      for (int i = lane; i < d; i += 32) {
        const A uv = (A)to_f(u[i]);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < m) acc[r] += uv * xs[r * d + i];
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < m) {
        A a = acc[r];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) logits[(int64_t)r * vocab + v] = a;
      }
    }
  }
}

// two-stage first-max argmax: stage 1 (gridDim.y chunks per row) writes
// partial (value, index); stage 2 (one CTA per row) folds the partials
template <typename A>
__global__ void __launch_bounds__(1024) argmax_kernel(const A* __restrict__ logits, int32_t* __restrict__ out, int vocab,
                                                      A* __restrict__ part_v, int32_t* __restrict__ part_i, int n_part) {
  pdl_trigger();
  pdl_wait();
  __shared__ A bv[32];
  __shared__ int bi[32];
  A best = -INFINITY;
  int idx = 0x7fffffff;
  if (part_v == nullptr || n_part == 0) {
    const A* x = logits + (int64_t)blockIdx.x * vocab;
    const int chunk = (vocab + gridDim.y - 1) / gridDim.y;
    const int lo = blockIdx.y * chunk, hi = min(vocab, lo + chunk);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      A v = x[i];
      if (v > best || (v == best && i < idx)) { best = v; idx = i; }
    }
  } else {
    for (int i = threadIdx.x; i < n_part; i += blockDim.x) {
      A v = part_v[(int64_t)blockIdx.x * n_part + i];
      int j = part_i[(int64_t)blockIdx.x * n_part + i];
      if (v > best || (v == best && j < idx)) { best = v; idx = j; }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    A ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { bv[w] = best; bi[w] = idx; }
  __syncthreads();
  if (w == 0) {
    best = lane < (int)(blockDim.x >> 5) ? bv[lane] : (A)-INFINITY;
    idx = lane < (int)(blockDim.x >> 5) ? bi[lane] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      A ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
    }
    if (lane == 0) {
      if (part_v != nullptr && n_part == 0) {
        part_v[(int64_t)blockIdx.x * gridDim.y + blockIdx.y] = best;
        part_i[(int64_t)blockIdx.x * gridDim.y + blockIdx.y] = idx;
      } else {
        out[blockIdx.x] = idx;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K9 top-k: bitonic sort of (score desc, index asc) in shared memory, then an
// ordered compaction of the selected indices (ascending output).
// ---------------------------------------------------------------------------
constexpr int TOPK_SMEM_MAX = 8192;  // longest chunk the shared-memory bitonic sort holds

__device__ __forceinline__ bool precedes(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// Exclusive scan of one int per thread over a 1024-thread block; *total gets
// the block sum.  `tmp` is 33 ints of shared memory.
__device__ __forceinline__ int block_excl_scan(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) tmp[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? tmp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    tmp[lane] = t;  // inclusive per-warp totals
  }
  __syncthreads();
  const int ex = incl - v + (w > 0 ? tmp[w - 1] : 0);
  *total = tmp[(blockDim.x >> 5) - 1];
  __syncthreads();  // tmp is reused by the next call
  return ex;
}

// Order-preserving map of a finite double to uint64 (larger score -> larger
// key; -0.0 and +0.0 map to the same key, as numpy compares them equal).
__device__ __forceinline__ unsigned long long score_key(double s) {
  if (s == 0.0) s = 0.0;
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// K9 for chunks longer than the shared-memory sort holds (planner.py:17-34,
// same result): an 8-pass radix select finds the key T of the k-th best
// score; every score above T is selected, plus the first `need` scores equal
// to T in index order (ties go to the lower index); one ordered block-wide
// compaction writes the indices ascending.  One CTA per chunk.
__global__ void __launch_bounds__(1024) topk_radix_kernel(const double* __restrict__ scores,
                                                          const int32_t* __restrict__ off,
                                                          const int32_t* __restrict__ count,
                                                          const int32_t* __restrict__ off_out,
                                                          int32_t* __restrict__ out) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long prefix_s;
  __shared__ int need_s;
  __shared__ int scan_tmp[33];
  const int c = blockIdx.x;
  const int base = off[c], n = off[c + 1] - off[c], k = min(count[c], n);
  if (k <= 0) return;
  const double* s = scores + base;
  unsigned long long prefix = 0, mask = 0;
  int need = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key = score_key(s[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, b = 255;
      for (; b > 0; --b) {
        if (acc + (int)hist[b] >= need) break;
        acc += (int)hist[b];
      }
      prefix_s = prefix | ((unsigned long long)b << shift);
      need_s = need - acc;
    }
    __syncthreads();
    prefix = prefix_s;
    need = need_s;
    mask |= 0xffull << shift;
  }
  const unsigned long long T = prefix;
  int32_t* o = out + off_out[c];
  int written = 0, ties = 0;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int i = t0 + threadIdx.x;
    const unsigned long long key = i < n ? score_key(s[i]) : 0ull;
    const bool gt = i < n && key > T, eq = i < n && key == T;
    int n_eq;
    const int tie_rank = block_excl_scan(eq ? 1 : 0, scan_tmp, &n_eq);
    const bool sel = gt || (eq && ties + tie_rank < need);
    int n_sel;
    const int pos = block_excl_scan(sel ? 1 : 0, scan_tmp, &n_sel);
    if (sel) o[written + pos] = i;
    written += n_sel;
    ties += n_eq;
  }
}

__global__ void __launch_bounds__(1024) topk_kernel(const double* __restrict__ scores,
                                                    const int32_t* __restrict__ off,
                                                    const int32_t* __restrict__ count,
                                                    const int32_t* __restrict__ off_out,
                                                    int32_t* __restrict__ out, int P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ks = reinterpret_cast<double*>(smem_raw);
  int* ki = reinterpret_cast<int*>(ks + P);
  unsigned char* sel = reinterpret_cast<unsigned char*>(ki + P);
  __shared__ int warp_tot[32];
  const int c = blockIdx.x;
  const int base = off[c], n = off[c + 1] - off[c], k = count[c];
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    ks[i] = i < n ? scores[base + i] : -INFINITY;
    ki[i] = i < n ? i : 0x7fffffff;
    sel[i] = 0;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int j = i ^ stride;
        if (j > i) {
          bool up = (i & size) == 0;  // ascending in "precedes" order
          bool swap = up ? precedes(ks[j], ki[j], ks[i], ki[i]) : precedes(ks[i], ki[i], ks[j], ki[j]);
          if (swap) {
            double ts = ks[i]; ks[i] = ks[j]; ks[j] = ts;
            int ti = ki[i]; ki[i] = ki[j]; ki[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) sel[ki[i]] = 1;
  __syncthreads();
  // ordered compaction: each thread owns a contiguous range of indices
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(n, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += sel[i];
  // exclusive block scan of cnt
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    warp_tot[lane] = t;  // inclusive totals per warp
  }
  __syncthreads();
  int pos = incl - cnt + (w > 0 ? warp_tot[w - 1] : 0);
  int32_t* o = out + off_out[c];
  for (int i = lo; i < hi; ++i)
    if (sel[i]) o[pos++] = i;
}

// ---------------------------------------------------------------------------
// K8b chunk statistics from per-row segment masses (deterministic: each
// output element is summed by one thread in row order)
// ---------------------------------------------------------------------------
__global__ void chunk_stats_kernel(const double* __restrict__ mass, int L, int n_rows, int n_seg,
                                   const int32_t* __restrict__ row0, const int32_t* __restrict__ len,
                                   const int32_t* __restrict__ seg_of, const int32_t* __restrict__ token_off,
                                   double* __restrict__ inter, double* __restrict__ intra,
                                   double* __restrict__ token) {
  const int c = blockIdx.x;
  const int r0 = row0[c], nr = len[c], sg = seg_of[c];
  const int W = n_seg + 1;
  // inter [c][l][j]
  for (int t = threadIdx.x; t < L * n_seg; t += blockDim.x) {
    int l = t / n_seg, j = t % n_seg;
    double s = 0;
    if (j < sg)
      for (int r = 0; r < nr; ++r) s += mass[((int64_t)l * n_rows + r0 + r) * W + j];
    inter[((int64_t)c * L + l) * n_seg + j] = s;
  }
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    double s = 0;
    for (int r = 0; r < nr; ++r) {
      const double* m = mass + ((int64_t)l * n_rows + r0 + r) * W;
      s += m[sg] - m[n_seg];
    }
    intra[(int64_t)c * L + l] = s;
  }
  for (int t = threadIdx.x; t < nr; t += blockDim.x) {
    double s = 0;
    for (int l = 0; l < L; ++l) {
      const double* m = mass + ((int64_t)l * n_rows + r0 + t) * W;
      double sl = 0;
      for (int j = 0; j < sg; ++j) sl += m[j];
      s += sl;
    }
    token[token_off[c] + t] = s;
  }
}

// ---------------------------------------------------------------------------
// K10: request rows -> fresh pool blocks (zero-padded to 16 rows)
// ---------------------------------------------------------------------------
template <typename T, int V>
__global__ void __launch_bounds__(256) extract_kernel(const T* __restrict__ kv_k, const T* __restrict__ kv_v,
                                                      int64_t req_layer_stride, int start, int n_rows,
                                                      const int32_t* __restrict__ blocks, T* __restrict__ pool,
                                                      int64_t pool_layer_stride, int64_t pool_block_stride, int kvw) {
  using VT = Vec<T, V>;
  const int b = blockIdx.x, l = blockIdx.y;
  T* dst = pool + (int64_t)l * pool_layer_stride + (int64_t)blocks[b] * pool_block_stride;
  const int vpr = kvw / V;
  for (int u = threadIdx.x; u < 2 * 16 * vpr; u += blockDim.x) {
    int kv = u / (16 * vpr);
    int rem = u % (16 * vpr);
    int r = rem / vpr, cidx = rem % vpr;
    int row = b * 16 + r;
    VT x;
    if (row < n_rows) {
      const T* src = (kv ? kv_v : kv_k) + (int64_t)l * req_layer_stride + (int64_t)(start + row) * kvw + cidx * V;
      x = *reinterpret_cast<const VT*>(src);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) x.v[e] = from_f<T>(0.f);
    }
    *reinterpret_cast<VT*>(dst + (int64_t)kv * 16 * kvw + (int64_t)r * kvw + cidx * V) = x;
  }
}

__global__ void add_f32_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = dst[i], b = src[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    dst[i] = a;
  }
}

// pull a read-only range (the next GEMM's weights) into L2 while other work
// runs; 128-byte lines, evict_last so the streaming GEMM operands do not
// displace it first
__global__ void __launch_bounds__(256) prefetch_l2_kernel(const char* __restrict__ p, size_t bytes) {
  const size_t lines = (bytes + 127) / 128;
  for (size_t l = blockIdx.x * (size_t)blockDim.x + threadIdx.x; l < lines; l += (size_t)gridDim.x * blockDim.x)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + l * 128));
}

__global__ void flush_kernel(int4* p, size_t n, int seed) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4(seed, (int)i, seed, (int)i);
}

}  // namespace ccb

using namespace ccb;

extern "C" {

int cc_rope_table(void* table, const double* inv_freq, int max_pos, int half, int dtype, void* stream) {
  CCB_REQUIRE(table && inv_freq && max_pos > 0 && half > 0, "rope_table: bad arguments");
  int64_t total = (int64_t)max_pos * half;
  int grid = (int)((total + 255) / 256);
  if (dtype == CC_F64)
    rope_table_kernel<double2><<<grid, 256, 0, as_stream(stream)>>>((double2*)table, inv_freq, max_pos, half);
  else
    rope_table_kernel<float2><<<grid, 256, 0, as_stream(stream)>>>((float2*)table, inv_freq, max_pos, half);
  return check_launch("rope_table");
}

int cc_rope_apply_f64(const double* x, double* y, const int64_t* positions, int n, int width, int d_head,
                      const double* inv_freq, int sign, void* stream) {
  CCB_REQUIRE(d_head > 0 && d_head % 2 == 0 && width % d_head == 0, "rope_apply: bad head width");
  if (n == 0) return 0;
  int64_t total = (int64_t)n * (width / 2);
  int grid = (int)std::min<int64_t>((total + 255) / 256, 65535);
  rope_apply_f64_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, y, positions, n, width, d_head, inv_freq,
                                                             sign >= 0 ? 1.0 : -1.0);
  return check_launch("rope_apply_f64");
}

// K1 kernel choice for experiments and tests (< 0: the environment's)
static std::atomic<int> g_k1_ldg{-1}, g_k1_cols{-1};
extern "C" __attribute__((visibility("default"))) void cc_debug_k1(int ldg, int cols) {
  g_k1_ldg = ldg;
  g_k1_cols = cols;
}

int cc_gather_rope_kv(const void* pool, int64_t pool_layer_stride, int64_t pool_block_stride,
                      const cc_gather_item* items, int n_items, int l0, int l1, const int32_t* slot_pos,
                      const int32_t* active_until, const void* rope_table, void* kv_k, void* kv_v, void* k_rot,
                      int64_t req_layer_stride, int kv_width, int d_head, int dtype, void* stream) {
  CCB_REQUIRE(d_head > 0 && d_head % 2 == 0 && kv_width % d_head == 0, "gather_rope_kv: bad head width");
  CCB_REQUIRE(l1 >= l0 && l0 >= 0, "gather_rope_kv: bad layer range");
  if (n_items == 0 || l1 == l0) return 0;
  CCB_REQUIRE(n_items <= 0x7fffffff && (l1 - l0) <= 65535, "gather_rope_kv: grid too large");
  // CCB_K1_LDG=1: the register-path kernel (A/B experiments); CCB_K1_COLS:
  // column chunk of the TMA-staged kernel (default: the widest multiple of
  // d_head dividing kv_width with 16 rows x cols <= 32 KiB)
  // (cc_debug_k1 overrides both at run time)
  static const int env_ldg = getenv("CCB_K1_LDG") ? atoi(getenv("CCB_K1_LDG")) : 0;
  static const int env_cols = getenv("CCB_K1_COLS") ? atoi(getenv("CCB_K1_COLS")) : 0;
  const int gl = g_k1_ldg.load(), gc = g_k1_cols.load();
  const int k1_ldg = gl >= 0 ? gl : env_ldg, k1_cols = gc >= 0 ? gc : env_cols;
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    int vec = std::min(pick_vec<T>(d_head / 2), pick_vec<T>(kv_width));
    return CCB_DISPATCH_VEC(vec, V, [&] {
      if (k1_ldg != 1) {
        int cols = d_head;
        for (int c = kv_width; c >= d_head; c -= d_head)
          if (kv_width % c == 0 && (k1_cols > 0 ? c <= k1_cols : 16 * c * (int)sizeof(T) <= 32768)) {
            cols = c;
            break;
          }
        const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        // bulk copies need 16-byte aligned rows and buffers; other layouts (none
        // in the engine) take the register-path kernel below (the same bits)
        const bool bulk_ok = (cols * sizeof(T)) % 16 == 0 && (kv_width * sizeof(T)) % 16 == 0 &&
                             (pool_layer_stride * sizeof(T)) % 16 == 0 && (pool_block_stride * sizeof(T)) % 16 == 0 &&
                             (req_layer_stride * sizeof(T)) % 16 == 0 && al(pool) && al(kv_k) && al(kv_v) &&
                             al(k_rot) && 2 * 16 * (size_t)cols * sizeof(T) <= 200 * 1024;
        if (bulk_ok) {
          const size_t smem = 2 * 16 * (size_t)cols * sizeof(T) + 16;
          auto kern = gather_rope_bulk_kernel<T, V>;
          if (int e = ensure_smem(kern, smem)) return e;
          const int64_t nx = (int64_t)n_items * (kv_width / cols);
          CCB_REQUIRE(nx <= 0x7fffffff, "gather_rope_kv: grid too large");
          return launch_k(kern, dim3((unsigned)nx, l1 - l0), dim3(256), smem, as_stream(stream), "gather_rope_kv",
                          (const T*)pool, pool_layer_stride, pool_block_stride, items, l0, slot_pos, active_until,
                          (const typename CS<T>::type*)rope_table, (T*)kv_k, (T*)kv_v, (T*)k_rot, req_layer_stride,
                          kv_width, d_head, cols, k1_ldg == 2 ? 1 : 0);
        }
      }
      dim3 grid(n_items, l1 - l0);
      return launch_k(gather_rope_kernel<T, V>, grid, dim3(256), 0, as_stream(stream), "gather_rope_kv",
                      (const T*)pool, pool_layer_stride, pool_block_stride, items, l0, slot_pos, active_until,
                      (const typename CS<T>::type*)rope_table, (T*)kv_k, (T*)kv_v, (T*)k_rot, req_layer_stride,
                      kv_width, d_head);
    });
  });
}

int cc_rope_scatter_qkv(const void* qkv, int64_t ld_qkv, int n_rows, const int32_t* row_slot, const int32_t* row_pos,
                        const void* rope_table, void* q_rot, void* kv_k, void* kv_v, void* k_rot, int n_heads,
                        int n_kv_heads, int d_head, int dtype, void* stream) {
  CCB_REQUIRE(d_head > 0 && d_head % 2 == 0, "rope_scatter: bad head width");
  if (n_rows == 0) return 0;
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    int vec = std::min(pick_vec<T>(d_head / 2), pick_vec<T>((int)ld_qkv));
    return CCB_DISPATCH_VEC(vec, V, [&] {
      // 128 threads striding the row's work units: measured 7.9 us per launch
      // at config 2 vs 8.3 (256) and 8.8 (one unit per thread, 448)
      const int threads = 128;
      return launch_k(rope_scatter_kernel<T, V>, dim3(n_rows), dim3(threads), 0, as_stream(stream), "rope_scatter_qkv",
                      (const T*)qkv, ld_qkv, row_slot, row_pos, (const typename CS<T>::type*)rope_table, (T*)q_rot,
                      (T*)kv_k, (T*)kv_v, (T*)k_rot, n_heads, n_kv_heads, d_head);
    });
  });
}

int cc_embed_rows(const void* embed, const int32_t* tokens, void* hidden, int n_rows, int d, int dtype, void* stream) {
  if (n_rows == 0) return 0;
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    return launch_k(embed_kernel<T>, dim3(n_rows), dim3(256), 0, as_stream(stream), "embed_rows", (const T*)embed,
                    tokens, (typename Acc<T>::type*)hidden, d);
  });
}

int cc_rmsnorm(const void* hidden, void* out, const float* weight, int n_rows, int d, double eps, int dtype,
               void* stream) {
  if (n_rows == 0) return 0;
  if (dtype != CC_F64 && d % 512 == 0 && d <= 512 * 32 &&
      ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(weight)) & 15) == 0) {
    const int nv = d / 512;
    auto go = [&](auto tag) -> int {
      constexpr int NV = decltype(tag)::value;
      if (dtype == CC_BF16)
        return launch_k(rmsnorm_vec_kernel<__nv_bfloat16, NV>, dim3(n_rows), dim3(128), 0, as_stream(stream),
                        "rmsnorm_vec", (const float*)hidden, (__nv_bfloat16*)out, weight, d, (float)eps);
      return launch_k(rmsnorm_vec_kernel<float, NV>, dim3(n_rows), dim3(128), 0, as_stream(stream), "rmsnorm_vec",
                      (const float*)hidden, (float*)out, weight, d, (float)eps);
    };
    switch (nv) {
      case 1: return go(std::integral_constant<int, 1>{});
      case 2: return go(std::integral_constant<int, 2>{});
      case 4: return go(std::integral_constant<int, 4>{});
      case 8: return go(std::integral_constant<int, 8>{});
      case 16: return go(std::integral_constant<int, 16>{});
      case 32: return go(std::integral_constant<int, 32>{});
      default: break;
    }
  }
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    rmsnorm_kernel<T><<<n_rows, 256, 0, as_stream(stream)>>>((const typename Acc<T>::type*)hidden, (T*)out,
                                                            weight, d, eps);
    return check_launch("rmsnorm");
  });
}

int cc_logits_argmax(const void* hidden_rows, const float* norm_w, double eps, const void* unembed, void* logits,
                     int32_t* argmax, int m, int d, int vocab, int dtype, void* stream) {
  CCB_REQUIRE(m >= 1 && m <= 8, "logits_argmax: 1..8 rows");
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    using A = typename Acc<T>::type;
    size_t smem = (size_t)m * d * sizeof(A);
    CCB_REQUIRE(smem <= 200 * 1024, "logits_argmax: rows too wide");
    if (smem > 48 * 1024)
      if (int rc = ensure_smem(logits_kernel<T>, smem)) return rc;
    // 24 CTAs per SM (several waves of short CTAs): measured 198 us for the
    // 128256 x 4096 unembedding vs 217 (8 per SM), 207 (12), 208 (16), 204 (32)
    int grid = std::min((vocab + 7) / 8, num_sms() * 24);
    int rc = CC_E_UNSUP;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)  // one row: the weight-streaming GEMV (decode.cu)
      if (m == 1) rc = logits_stream_bf16((const float*)hidden_rows, norm_w, (float)eps, unembed, (float*)logits, d,
                                          vocab, as_stream(stream));
    if (rc == CC_E_UNSUP)
      rc = launch_k(logits_kernel<T>, dim3(grid), dim3(256), smem, as_stream(stream), "logits",
                    (const A*)hidden_rows, norm_w, eps, (const T*)unembed, (A*)logits, m, d, vocab);
    if (rc) return rc;
    if (argmax) {
      // partials live after the logits rows in a small static scratch
      constexpr int PARTS = 64;
      uint8_t* scratch = (uint8_t*)stream_scratch(as_stream(stream), SCR_LOGITS, (sizeof(A) + sizeof(int32_t)) * 8 * PARTS);
      if (!scratch) return fail(CC_E_CUDA, "logits_argmax: scratch allocation failed");
      A* part_v = reinterpret_cast<A*>(scratch);
      int32_t* part_i = reinterpret_cast<int32_t*>(scratch + sizeof(A) * 8 * PARTS);
      rc = launch_k(argmax_kernel<A>, dim3(m, PARTS), dim3(1024), 0, as_stream(stream), "argmax_partial",
                    (const A*)logits, argmax, vocab, part_v, part_i, 0);
      if (rc) return rc;
      return launch_k(argmax_kernel<A>, dim3(m), dim3(64), 0, as_stream(stream), "argmax", (const A*)logits, argmax,
                      vocab, part_v, part_i, PARTS);
    }
    return 0;
  });
}

int cc_topk_select(const double* scores, const int32_t* off, const int32_t* count, const int32_t* off_out,
                   int32_t* out, int n_chunks, int max_len, void* stream) {
  if (n_chunks == 0) return 0;
  if (max_len > TOPK_SMEM_MAX) {  // long chunks: radix select over global memory, any length
    topk_radix_kernel<<<n_chunks, 1024, 0, as_stream(stream)>>>(scores, off, count, off_out, out);
    return check_launch("topk_select_radix");
  }
  int P = 1;
  while (P < std::max(max_len, 1)) P <<= 1;
  size_t smem = (size_t)P * (sizeof(double) + sizeof(int) + 1);
  if (smem > 48 * 1024)
    if (int rc = ensure_smem(topk_kernel, smem)) return rc;
  topk_kernel<<<n_chunks, 1024, smem, as_stream(stream)>>>(scores, off, count, off_out, out, P);
  return check_launch("topk_select");
}

int cc_chunk_stats(const double* mass, int L, int n_rows, int n_seg, const int32_t* row0, const int32_t* len,
                   const int32_t* seg_of, const int32_t* token_off, int n_chunks, double* inter, double* intra,
                   double* token, void* stream) {
  if (n_chunks == 0) return 0;
  chunk_stats_kernel<<<n_chunks, 256, 0, as_stream(stream)>>>(mass, L, n_rows, n_seg, row0, len, seg_of,
                                                              token_off, inter, intra, token);
  return check_launch("chunk_stats");
}

int cc_extract_to_pool(const void* kv_k, const void* kv_v, int64_t req_layer_stride, int L, int start, int n_rows,
                       const int32_t* blocks, int n_blocks, void* pool, int64_t pool_layer_stride,
                       int64_t pool_block_stride, int kv_width, int dtype, void* stream) {
  CCB_REQUIRE(n_blocks * 16 >= n_rows, "extract_to_pool: not enough blocks");
  if (n_blocks == 0) return 0;
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    int vec = pick_vec<T>(kv_width);
    return CCB_DISPATCH_VEC(vec, V, [&] {
      dim3 grid(n_blocks, L);
      extract_kernel<T, V><<<grid, 256, 0, as_stream(stream)>>>((const T*)kv_k, (const T*)kv_v, req_layer_stride,
                                                               start, n_rows, blocks, (T*)pool, pool_layer_stride,
                                                               pool_block_stride, kv_width);
      return check_launch("extract_to_pool");
    });
  });
}

int cc_add_f32(float* dst, const float* src, int64_t n, void* stream) {
  CCB_REQUIRE(n % 4 == 0 && ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0,
              "add_f32: needs 16-byte aligned buffers of a multiple of 4 floats");
  if (n == 0) return 0;
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)num_sms() * 8);
  add_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>((float4*)dst, (const float4*)src, n4);
  return check_launch("add_f32");
}

int cc_prefetch_l2(const void* p, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  prefetch_l2_kernel<<<32, 256, 0, as_stream(stream)>>>(reinterpret_cast<const char*>(p), bytes);
  return check_launch("prefetch_l2");
}

int cc_flush_l2(void* scratch, size_t bytes, void* stream) {
  size_t n = bytes / sizeof(int4);
  flush_kernel<<<num_sms() * 4, 512, 0, as_stream(stream)>>>((int4*)scratch, n, 7);
  return check_launch("flush_l2");
}

}  // extern "C"
