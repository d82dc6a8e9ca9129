// tcgen05 / TMEM / TMA bf16 GEMM for the recompute rows (K3/K5/K6):
// C[M,N] = A[M,K] B[N,K]^T, fp32 accumulation in TMEM, fused epilogues
// (model.py:399-401 QKV, :417 o_proj + residual, :418-419 MLP).
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0     TMA producer (A and B tiles, 128B swizzle, 4-stage ring)
//   warp 1     MMA issuer (single thread, tcgen05.mma 128x256x16) + TMEM owner
//   warps 2-5  epilogue (tcgen05.ld 32 lanes x 32 cols -> registers -> global)
// Two TMEM accumulators (2 x 256 columns) let tile i's epilogue overlap tile
// i+1's MMAs.  Tiles are walked M-fastest so the CTAs of one wave share the
// weight tile through L2.  No split-K: a row's result is independent of M.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace ccb {

namespace {

constexpr int TC_BM = 128, TC_BK = 64;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;   // 16 KiB
constexpr int TC_THREADS = 192;

// per-BN configuration: B tile bytes, ring depth filling ~200 KiB, TMEM columns
template <int BN>
struct TcCfg {
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGES = (200 * 1024) / (TC_A_BYTES + B_BYTES) > 6 ? 6 : (200 * 1024) / (TC_A_BYTES + B_BYTES);
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t SMEM = 1024 + STAGES * (TC_A_BYTES + B_BYTES) + 256;
};

using namespace sm100;

// Work unit u in [0, num_tiles * splits): split s = u / num_tiles, tile
// t = u % num_tiles (split-major, so a unit only ever waits on a smaller unit
// index: with a persistent grid of co-resident CTAs this cannot deadlock).
// Split s covers k-blocks [kb_begin(s), kb_begin(s+1)).
__device__ __forceinline__ int kb_begin(int s, int splits, int num_kb) {
  const int q = num_kb / splits, r = num_kb % splits;
  return s * q + (s < r ? s : r);
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int EPI, int TC_BN, bool SPLIT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* C,
                   int64_t ldc, int M, int N, int K, int splits_arg, float* __restrict__ ws, int* __restrict__ flags,
                   int epoch) {
  const int splits = SPLIT ? splits_arg : 1;
  constexpr int TC_B_BYTES = TcCfg<TC_BN>::B_BYTES;
  constexpr int TC_STAGES = TcCfg<TC_BN>::STAGES;
  constexpr int TMEM_COLS = TcCfg<TC_BN>::TMEM_COLS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + TC_STAGES * TC_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + TC_STAGES * TC_B_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + TC_BM - 1) / TC_BM;
  const int num_tiles = num_m * (N / TC_BN);
  const int num_kb = K / TC_BK;
  const int num_units = num_tiles * splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int sp = u / num_tiles, tile = u % num_tiles;
        const int mt = tile % num_m, nt = tile / num_m;
        const int k0 = kb_begin(sp, splits, num_kb), k1 = kb_begin(sp + 1, splits, num_kb);
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], TC_A_BYTES + TC_B_BYTES);
          tma_load_2d(sA + stage * TC_A_BYTES, &tmA, &full[stage], kb * TC_BK, mt * TC_BM);
          tma_load_2d(sB + stage * TC_B_BYTES, &tmB, &full[stage], kb * TC_BK, nt * TC_BN);
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, TC_BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int sp = u / num_tiles;
        const int k0 = kb_begin(sp, splits, num_kb), k1 = kb_begin(sp + 1, splits, num_kb);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TC_BN;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = desc_sw128(sA + stage * TC_A_BYTES);
          const uint64_t bd = desc_sw128(sB + stage * TC_B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > k0 || k > 0) ? 1u : 0u);
          mma_commit(&empty[stage]);
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;  // 0..127 within the epilogue warps
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int sp = u / num_tiles, tile = u % num_tiles;
      const int mt = tile % num_m, nt = tile / num_m;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mt * TC_BM + q * 32 + lane;
      const uint32_t t0 = tmem_base + acc * TC_BN + ((uint32_t)(q * 32) << 16);
      const int n0 = nt * TC_BN;
      // split-K: partial sums are folded in split order (deterministic)
      constexpr bool split = SPLIT;
      const bool last = sp == splits - 1;
      if (SPLIT && sp > 0) {
        if (et == 0)
          while (ld_acquire(&flags[tile]) != epoch * 64 + sp) __nanosleep(64);
        epi_bar();
      }
      float* wrow = ws + (int64_t)row * N + n0;  // fp32 workspace row (non-residual splits)
      if constexpr (EPI == CC_EPI_SWIGLU && TC_BN == 256) {
        // tile columns: [gate 64 | up 64 | gate 64 | up 64] -> 128 outputs
#pragma unroll 1
        for (int g = 0; g < 4; ++g) {
          const int gc = (g >> 1) * 128 + (g & 1) * 32;
          uint32_t rg[32], ru[32];
          tmem_ld32(t0 + gc, rg);
          tmem_ld32(t0 + gc + 64, ru);
          tmem_ld_wait();
          if (row < M) {
            if (split) {
              float4* wg = reinterpret_cast<float4*>(wrow + gc);
              float4* wu = reinterpret_cast<float4*>(wrow + gc + 64);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 a = make_float4(__uint_as_float(rg[4 * i]), __uint_as_float(rg[4 * i + 1]),
                                       __uint_as_float(rg[4 * i + 2]), __uint_as_float(rg[4 * i + 3]));
                float4 b = make_float4(__uint_as_float(ru[4 * i]), __uint_as_float(ru[4 * i + 1]),
                                       __uint_as_float(ru[4 * i + 2]), __uint_as_float(ru[4 * i + 3]));
                if (sp > 0) {
                  float4 pa = __ldcg(wg + i), pb = __ldcg(wu + i);
                  a.x += pa.x; a.y += pa.y; a.z += pa.z; a.w += pa.w;
                  b.x += pb.x; b.y += pb.y; b.z += pb.z; b.w += pb.w;
                }
                if (!last) { __stcg(wg + i, a); __stcg(wu + i, b); }
                rg[4 * i] = __float_as_uint(a.x); rg[4 * i + 1] = __float_as_uint(a.y);
                rg[4 * i + 2] = __float_as_uint(a.z); rg[4 * i + 3] = __float_as_uint(a.w);
                ru[4 * i] = __float_as_uint(b.x); ru[4 * i + 1] = __float_as_uint(b.y);
                ru[4 * i + 2] = __float_as_uint(b.z); ru[4 * i + 3] = __float_as_uint(b.w);
              }
            }
            if (last) {
              __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)row * ldc + n0 / 2 + (g >> 1) * 64 + (g & 1) * 32;
              uint4 pk[4];
              uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                float a0 = __uint_as_float(rg[2 * i]), a1 = __uint_as_float(rg[2 * i + 1]);
                float u0 = __uint_as_float(ru[2 * i]), u1 = __uint_as_float(ru[2 * i + 1]);
                __nv_bfloat162 h = __floats2bfloat162_rn(silu(a0) * u0, silu(a1) * u1);
                pw[i] = *reinterpret_cast<uint32_t*>(&h);
              }
              uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
              for (int i = 0; i < 4; ++i) o4[i] = pk[i];
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(t0 + c * 32, r);
          tmem_ld_wait();
          if (row < M) {
            const int64_t o = (int64_t)row * ldc + n0 + c * 32;
            if constexpr (EPI == CC_EPI_RESID_ADD) {
              float4* h = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + o);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 v = split ? __ldcg(h + i) : h[i];
                v.x += __uint_as_float(r[4 * i]);
                v.y += __uint_as_float(r[4 * i + 1]);
                v.z += __uint_as_float(r[4 * i + 2]);
                v.w += __uint_as_float(r[4 * i + 3]);
                if (split) __stcg(h + i, v); else h[i] = v;
              }
            } else {
              if (split) {
                float4* w4 = reinterpret_cast<float4*>(wrow + c * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  float4 a = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                         __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
                  if (sp > 0) {
                    float4 p = __ldcg(w4 + i);
                    a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
                  }
                  if (!last) __stcg(w4 + i, a);
                  r[4 * i] = __float_as_uint(a.x); r[4 * i + 1] = __float_as_uint(a.y);
                  r[4 * i + 2] = __float_as_uint(a.z); r[4 * i + 3] = __float_as_uint(a.w);
                }
              }
              if (last) {
                uint4 pk[4];
                uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  float a0 = __uint_as_float(r[2 * i]), a1 = __uint_as_float(r[2 * i + 1]);
                  if constexpr (EPI == CC_EPI_GELU) { a0 = gelu_tanh(a0); a1 = gelu_tanh(a1); }
                  __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                  pw[i] = *reinterpret_cast<uint32_t*>(&h);
                }
                uint4* o4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(C) + o);
#pragma unroll
                for (int i = 0; i < 4; ++i) o4[i] = pk[i];
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (SPLIT && !last) {
        __threadfence();
        epi_bar();
        if (et == 0) st_release(&flags[tile], epoch * 64 + sp + 1);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ---- host: tensor maps ------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* p;
  int64_t rows, cols, ld;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.p);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull + (size_t)k.cols * 0xC2B2AE3D27D4EB4Full;
    h ^= (size_t)k.ld * 0x165667B19E3779F9ull + (size_t)k.box_rows;
    return h;
  }
};

// 2D bf16 row-major [rows][cols] (leading dim ld elements), box [box_rows][64], 128B swizzle
int make_map(CUtensorMap* out, const void* p, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{p, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return 0; }
  }
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(CC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CC_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *out);
  return 0;
}

struct SplitScratch {
  float* ws = nullptr;
  size_t ws_elems = 0;
  int* flags = nullptr;
  int flag_elems = 0;
  int epoch = 0;
};

// one split-K scratch per (device, stream): concurrent GEMMs on different
// streams (e.g. tensor-parallel ranks sharing a process) never share it
SplitScratch& scratch(cudaStream_t st) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, SplitScratch*> by_key;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(st) << 4) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> g(mu);
  auto it = by_key.find(key);
  if (it != by_key.end()) return *it->second;
  SplitScratch* sc = new SplitScratch();
  by_key.emplace(key, sc);
  return *sc;
}

template <int EPI, int BN>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t ldc, int M, int N, int K, int splits,
              cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TcCfg<BN>::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TcCfg<BN>::SMEM);
    attr_set = true;
  }
  const int tiles = ((M + TC_BM - 1) / TC_BM) * (N / BN);
  const int units = tiles * splits;
  const int grid = units < num_sms() ? units : num_sms();
  SplitScratch& sc = scratch(st);
  if (splits > 1) {
    if (sc.flag_elems < tiles) {
      if (sc.flags) cudaFree(sc.flags);
      sc.flag_elems = tiles < 4096 ? 4096 : tiles;
      if (cudaMalloc(&sc.flags, sizeof(int) * sc.flag_elems) != cudaSuccess) return fail(CC_E_CUDA, "gemm_tc: flags");
      cudaMemset(sc.flags, 0xff, sizeof(int) * sc.flag_elems);
    }
    const size_t need = EPI == CC_EPI_RESID_ADD ? 0 : (size_t)((M + TC_BM - 1) / TC_BM) * TC_BM * N;
    if (sc.ws_elems < need) {
      if (sc.ws) cudaFree(sc.ws);
      sc.ws_elems = need;
      if (cudaMalloc(&sc.ws, sizeof(float) * need) != cudaSuccess) return fail(CC_E_CUDA, "gemm_tc: workspace");
    }
    sc.epoch = (sc.epoch + 1) & 0x00ffffff;
  }
  if (splits > 1)
    gemm_tc_kernel<EPI, BN, true><<<grid, TC_THREADS, TcCfg<BN>::SMEM, st>>>(ma, mb, C, ldc, M, N, K, splits, sc.ws,
                                                                            sc.flags, sc.epoch);
  else
    gemm_tc_kernel<EPI, BN, false><<<grid, TC_THREADS, TcCfg<BN>::SMEM, st>>>(ma, mb, C, ldc, M, N, K, 1, nullptr,
                                                                             nullptr, 0);
  return check_launch("gemm_tc");
}

// (BN, split-K) minimising the modelled time: persistent rounds x k-blocks per
// unit x per-k-block cost of the tile width + a fixed-up epilogue per split
void pick_tiling(int M, int N, int K, int epi, bool allow_split, int* bn_out, int* splits_out) {
  const int m_tiles = (M + TC_BM - 1) / TC_BM;
  const int sms = num_sms();
  const int num_kb = K / TC_BK;
  const int cand[3] = {256, 192, 128};
  const double kb_cost[3] = {1.0, 0.75 / 0.97, 0.5 / 0.88};  // relative time of one k-block of a 128xBN tile
  double best = 1e30;
  *bn_out = 0;
  *splits_out = 1;
  for (int i = 0; i < 3; ++i) {
    const int bn = cand[i];
    if (N % bn) continue;
    if (epi == CC_EPI_SWIGLU && bn != 256) continue;
    const int tiles = m_tiles * (N / bn);
    // split-K only pays when most SMs would idle (small M: weight streaming);
    // the in-order fix-ups cost more than wave quantisation at larger M
    const int max_s = (allow_split && 2 * tiles <= sms) ? (num_kb < 16 ? num_kb : 16) : 1;
    for (int s = 1; s <= max_s; ++s) {
      if (s > 1 && num_kb / s < 4) break;  // keep >= 4 k-blocks per split unit
      const int rounds = (tiles * s + sms - 1) / sms;
      const double t = rounds * ((double)(num_kb + s - 1) / s) * kb_cost[i] + (s > 1 ? 6.0 * s : 0.0);
      if (t < best - 1e-9) { best = t; *bn_out = bn; *splits_out = s; }
    }
  }
}

// CCB_GEMM_FORCE="bn,splits" pins the tiling (experiments / tests)
bool forced_tiling(int N, int epi, int* bn, int* splits) {
  static int fb = -1, fs = -1;
  static bool init = false;
  if (!init) {
    init = true;
    if (const char* e = getenv("CCB_GEMM_FORCE")) sscanf(e, "%d,%d", &fb, &fs);
  }
  if (fb <= 0 || N % fb || (epi == CC_EPI_SWIGLU && fb != 256)) return false;
  *bn = fb;
  *splits = fs > 0 ? fs : 1;
  return true;
}

template <int EPI>
int launch_epi(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
               bool allow_split, cudaStream_t st) {
  int bn, splits;
  if (!forced_tiling(N, EPI, &bn, &splits)) pick_tiling(M, N, K, EPI, allow_split, &bn, &splits);
  if (splits > K / TC_BK) splits = K / TC_BK;
  if (bn == 0) return fail(CC_E_UNSUP, "gemm_tc: N must be a multiple of 128 (SwiGLU: 256)");
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, TC_BM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, bn);
  if (rc) return rc;
  if (bn == 256) return launch_tc<EPI, 256>(ma, mb, C, ldc, M, N, K, splits, st);
  if (bn == 192) return launch_tc<EPI, 192>(ma, mb, C, ldc, M, N, K, splits, st);
  return launch_tc<EPI, 128>(ma, mb, C, ldc, M, N, K, splits, st);
}

}  // namespace

int gemm_tc_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
                 int epi, bool allow_split, cudaStream_t st) {
  if (N % 128 != 0 || K % TC_BK != 0 || lda % 8 != 0 || ldb % 8 != 0 || ldc % 8 != 0)
    return fail(CC_E_UNSUP, "gemm_tc: needs N % 128 == 0, K % 64 == 0, 16-byte aligned rows");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return fail(CC_E_UNSUP, "gemm_tc: pointers must be 16-byte aligned");
  switch (epi) {
    case CC_EPI_STORE: return launch_epi<CC_EPI_STORE>(A, lda, B, ldb, C, ldc, M, N, K, allow_split, st);
    case CC_EPI_RESID_ADD: return launch_epi<CC_EPI_RESID_ADD>(A, lda, B, ldb, C, ldc, M, N, K, allow_split, st);
    case CC_EPI_SWIGLU: return launch_epi<CC_EPI_SWIGLU>(A, lda, B, ldb, C, ldc, M, N, K, allow_split, st);
    case CC_EPI_GELU: return launch_epi<CC_EPI_GELU>(A, lda, B, ldb, C, ldc, M, N, K, allow_split, st);
    default: return fail(CC_E_ARG, "gemm_tc: unknown epilogue");
  }
}

}  // namespace ccb
