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

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace ccb {

namespace {

constexpr int TC_BM = 128, TC_BN = 256, TC_BK = 64, TC_STAGES = 4;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;   // 16 KiB
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;   // 32 KiB
constexpr int TC_THREADS = 192;
constexpr size_t TC_SMEM = 1024 + TC_STAGES * (TC_A_BYTES + TC_B_BYTES) + 256;

using namespace sm100;

template <int EPI>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* C,
                   int64_t ldc, int M, int N, int K) {
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
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile % num_m, nt = tile / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
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
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TC_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = desc_sw128(sA + stage * TC_A_BYTES);
          const uint64_t bd = desc_sw128(sB + stage * TC_B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mt = tile % num_m, nt = tile / num_m;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mt * TC_BM + q * 32 + lane;
      const uint32_t t0 = tmem_base + acc * TC_BN + ((uint32_t)(q * 32) << 16);
      const int n0 = nt * TC_BN;
      if constexpr (EPI == CC_EPI_SWIGLU) {
        // tile columns: [gate 64 | up 64 | gate 64 | up 64] -> 128 outputs
#pragma unroll 1
        for (int g = 0; g < 4; ++g) {
          const int gc = (g >> 1) * 128 + (g & 1) * 32;
          uint32_t rg[32], ru[32];
          tmem_ld32(t0 + gc, rg);
          tmem_ld32(t0 + gc + 64, ru);
          tmem_ld_wait();
          if (row < M) {
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
                float4 v = h[i];
                v.x += __uint_as_float(r[4 * i]);
                v.y += __uint_as_float(r[4 * i + 1]);
                v.z += __uint_as_float(r[4 * i + 2]);
                v.w += __uint_as_float(r[4 * i + 3]);
                h[i] = v;
              }
            } else {
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
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
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

template <int EPI>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t ldc, int M, int N, int K,
              cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
    attr_set = true;
  }
  int tiles = ((M + TC_BM - 1) / TC_BM) * (N / TC_BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  gemm_tc_kernel<EPI><<<grid, TC_THREADS, TC_SMEM, st>>>(ma, mb, C, ldc, M, N, K);
  return check_launch("gemm_tc");
}

}  // namespace

int gemm_tc_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
                 int epi, cudaStream_t st) {
  if (N % TC_BN != 0 || K % TC_BK != 0 || lda % 8 != 0 || ldb % 8 != 0 || ldc % 8 != 0)
    return fail(CC_E_UNSUP, "gemm_tc: needs N % 256 == 0, K % 64 == 0, 16-byte aligned rows");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return fail(CC_E_UNSUP, "gemm_tc: pointers must be 16-byte aligned");
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, TC_BM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, TC_BN);
  if (rc) return rc;
  switch (epi) {
    case CC_EPI_STORE: return launch_tc<CC_EPI_STORE>(ma, mb, C, ldc, M, N, K, st);
    case CC_EPI_RESID_ADD: return launch_tc<CC_EPI_RESID_ADD>(ma, mb, C, ldc, M, N, K, st);
    case CC_EPI_SWIGLU: return launch_tc<CC_EPI_SWIGLU>(ma, mb, C, ldc, M, N, K, st);
    case CC_EPI_GELU: return launch_tc<CC_EPI_GELU>(ma, mb, C, ldc, M, N, K, st);
    default: return fail(CC_E_ARG, "gemm_tc: unknown epilogue");
  }
}

}  // namespace ccb
