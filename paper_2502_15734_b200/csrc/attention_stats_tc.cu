// K8a on the tensor cores: head-mean attention mass of selected query rows
// onto key segments (stats.py:68-106, harness.py:331-354) without
// materialising the softmax weights.  Given the row's log-sum-exp from the
// attention kernel, p = exp(s - lse) is recomputed tile by tile:
//   warp 0     TMA K tiles (128 keys, 2-stage ring)
//   warp 1     tcgen05.mma S = Q K^T into one of two TMEM buffers
//   warps 2-5  load the CTA's Q rows (gathered by index, written 128B-swizzled
//              into smem), then take the EVEN key tiles, warps 6-9 the ODD
//              ones (each warpgroup owns one of the two TMEM S buffers):
//              tcgen05.ld S, p = exp2(s*c - lse*log2e) masked by the causal
//              limit and pads, accumulated per key segment (a tile inside one
//              segment: one sum; a tile across boundaries: a warp-uniform walk
//              over the segments it overlaps) into the warpgroup's own
//              per-row accumulators.
// The two warpgroups' sums and the G heads of the CTA are folded in fixed
// order; a second kernel folds the kv groups in fixed order and divides by
// Hq.  No atomics: run-to-run bit-identical.  (One warpgroup for all tiles
// measured latency-bound: the K8 pass cost 16% of a fresh 8B prefill.)
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "attention.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "f32x2.cuh"

namespace ccb {

namespace {

using namespace sm100;

constexpr int ST_BN = 128;
constexpr int ST_MAXSTAGES = 4;
constexpr int ST_MAXSEG = 112;  // n_seg + 1 (diagonal) <= 112 (two warpgroups' accumulators in smem)

__host__ __device__ constexpr uint32_t idesc_s(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DH, int ST_STAGES>
struct StSmem {
  static constexpr int Q_BYTES = 128 * DH * 2;
  static constexpr int K_BYTES = ST_BN * DH * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_BYTES;
  static constexpr int SEG_OFF = K_OFF + ST_STAGES * K_BYTES;  // int seg_lo[ST_MAXSEG], seg_hi[ST_MAXSEG]
  static constexpr int BAR_OFF = SEG_OFF + 2 * ST_MAXSEG * 4;
  static constexpr int ACC_OFF = BAR_OFF + 256;  // float [2 warpgroups][128][stride], stride odd >= n_seg + 1
  static size_t total(int stride) { return 1024 + ACC_OFF + (size_t)2 * 128 * stride * 4; }
};

template <int DH, int ST_STAGES, int PF>
__global__ void __launch_bounds__(320, 1)
    attn_stats_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __nv_bfloat16* __restrict__ q,
                         const int32_t* __restrict__ rows, int n_rows, const int32_t* __restrict__ q_slot,
                         const uint8_t* __restrict__ key_pad, const float* __restrict__ lse,
                         const int32_t* __restrict__ seg_lo, const int32_t* __restrict__ seg_hi, int n_seg,
                         float* __restrict__ part, int n_keys, int Hq, int Hkv, int G, float scale_log2, int stride) {
  using SM = StSmem<DH, ST_STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base + SM::Q_OFF;
  uint8_t* sK = base + SM::K_OFF;
  float* acc = reinterpret_cast<float*>(base + SM::ACC_OFF);  // [2][128][stride]
  int* segmap = reinterpret_cast<int*>(base + SM::SEG_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + SM::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + ST_STAGES;
  uint64_t* s_full = k_empty + ST_STAGES;
  uint64_t* s_empty = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);
  __shared__ int s_kmax;
  __shared__ uint32_t padw[2][8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int R = 128 / G;
  // row blocks in reverse: with causal limits the last rows see the most key
  // tiles, so the longest CTAs start first instead of forming the tail wave
  const int r0 = (gridDim.y - 1 - blockIdx.y) * R;  // first stats row of this CTA
  const int W = n_seg + 1;

  if (threadIdx.x == 0) s_kmax = -1;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmK);
    mbar_init(q_full, 128);
    for (int s = 0; s < ST_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 128);  // the warpgroup that owns buffer b
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  __syncthreads();
  if (threadIdx.x < 128) {
    const int sr = r0 + threadIdx.x / G;
    if (sr < n_rows) atomicMax(&s_kmax, q_slot[rows[sr]]);
  }
  (void)SM::ACC_OFF;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kmax = s_kmax;
  const int n_tiles = kmax < 0 ? 0 : kmax / ST_BN + 1;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i % ST_STAGES;
        mbar_wait(&k_empty[st], ((i / ST_STAGES) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], SM::K_BYTES);
#pragma unroll
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sK + st * SM::K_BYTES + a * ST_BN * 128, &tmK, &k_full[st], g * DH + a * 64, i * ST_BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t id = idesc_s(128, ST_BN);
      mbar_wait(q_full, 0);
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i % ST_STAGES, b = i & 1;
        mbar_wait(&k_full[st], (i / ST_STAGES) & 1);
        mbar_wait(&s_empty[b], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const int a = kk >> 2, w = kk & 3;
          uint64_t ad = desc_sw128(sQ + a * 128 * 128) + 2 * w;
          uint64_t bd = desc_sw128(sK + st * SM::K_BYTES + a * ST_BN * 128) + 2 * w;
          mma_bf16(tmem + b * ST_BN, ad, bd, id, kk > 0);
        }
        mma_commit(&s_full[b]);
        mma_commit(&k_empty[st]);
      }
    }
  } else {
    const int wg = (warp - 2) >> 2;  // 0: even key tiles (S buffer 0), 1: odd tiles (buffer 1)
    const int q4 = warp & 3;
    const int m = q4 * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..255
    const int sr = r0 + m / G;
    const int head = g * G + m % G;
    const bool valid = sr < n_rows;
    const int qrow = valid ? rows[sr] : 0;
    const int lim = valid ? q_slot[qrow] : -1;
    const float base_l2 = valid ? lse[(int64_t)qrow * Hq + head] * 1.4426950408889634f : 0.f;
    if (wg == 0) {
      // gather this M-row's q (dh bf16) into the 128B-swizzled K-major tile
      const uint4* src = reinterpret_cast<const uint4*>(q + ((int64_t)qrow * Hq + head) * DH);
#pragma unroll
      for (int ch = 0; ch < DH / 8; ++ch) {
        uint4 v = valid ? src[ch] : make_uint4(0, 0, 0, 0);
        const int a = ch >> 3, c16 = ch & 7;
        *reinterpret_cast<uint4*>(sQ + a * 128 * 128 + m * 128 + ((c16 ^ (m & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(q_full);
    }
    float* my = acc + ((int64_t)wg * 128 + m) * stride;  // odd stride: no bank conflicts
    for (int sg = 0; sg < W; ++sg) my[sg] = 0.f;
    // segment bounds in shared memory (segments are sorted, disjoint slot ranges)
    int* s_lo = segmap;
    int* s_hi = segmap + ST_MAXSEG;
    for (int sg = et; sg < n_seg; sg += 256) {
      s_lo[sg] = seg_lo[sg];
      s_hi[sg] = seg_hi[sg];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    float diag = 0.f;
    for (int i = wg; i < n_tiles; i += 2) {
      const int b = wg;  // this warpgroup's S buffer
      const int j0 = i * ST_BN;
      uint32_t pw[4] = {0u, 0u, 0u, 0u};
      if (key_pad != nullptr) {
        // 128-bit pad mask of the tile, built by this warpgroup's 128 threads
        const int jm = j0 + m;  // word q4 of the mask covers keys [32*q4, 32*q4+32)
        const unsigned word = __ballot_sync(0xffffffffu, jm >= n_keys || key_pad[jm] != 0);
        if (lane == 0) padw[wg][((i >> 1) & 1) * 4 + q4] = word;
        asm volatile("bar.sync %0, 128;" ::"r"(2 + wg) : "memory");
#pragma unroll
        for (int w = 0; w < 4; ++w) pw[w] = padw[wg][((i >> 1) & 1) * 4 + w];
      }
      mbar_wait(&s_full[b], (i >> 1) & 1);
      tc_fence_after();
      float p[ST_BN];
      {
        uint32_t ra[32], rb[32], rc[32], rd[32];
        const uint32_t ta = tmem + b * ST_BN + ((uint32_t)(q4 * 32) << 16);
        tmem_ld32(ta, ra);
        tmem_ld32(ta + 32, rb);
        tmem_ld32(ta + 64, rc);
        tmem_ld32(ta + 96, rd);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          p[e] = __uint_as_float(ra[e]);
          p[32 + e] = __uint_as_float(rb[e]);
          p[64 + e] = __uint_as_float(rc[e]);
          p[96 + e] = __uint_as_float(rd[e]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_empty[b]);
      const int lim_rel = lim - j0;
      // fast path: every key of the tile visible to this row and the tile
      // inside one segment (the common case: segments are chunk spans) --
      // packed f32x2 arithmetic, a quarter of the exponentials on the FMA
      // pipe, summed straight into four packed accumulators
      int one_seg = -1;
      if (lim_rel >= ST_BN && (pw[0] | pw[1] | pw[2] | pw[3]) == 0)  // (the diagonal tile: general path)
        for (int sg = 0; sg < n_seg; ++sg)
          if (s_lo[sg] <= j0 && s_hi[sg] >= j0 + ST_BN) {
            one_seg = sg;
            break;
          }
      if (__all_sync(0xffffffffu, one_seg >= 0) && one_seg == __shfl_sync(0xffffffffu, one_seg, 0)) {
        const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nb2 = f2_pack(-base_l2, -base_l2);
        uint64_t a2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int c2 = 0; c2 < ST_BN / 2; ++c2) {
          const uint64_t x2 = ffma2(f2_pack(p[2 * c2], p[2 * c2 + 1]), sc2, nb2);
          uint64_t e2;
          if ((c2 & 7) >= 8 - PF) {
            e2 = ex2_poly2(x2);
          } else {
            float x0, x1;
            f2_unpack(x2, x0, x1);
            e2 = f2_pack(ex2f(x0), ex2f(x1));
          }
          a2[c2 & 3] = fadd2(a2[c2 & 3], e2);
        }
        const uint64_t t2 = fadd2(fadd2(a2[0], a2[1]), fadd2(a2[2], a2[3]));
        float t0, t1;
        f2_unpack(t2, t0, t1);
        my[one_seg] += t0 + t1;
        continue;
      }
      // all probabilities first (independent -> full ILP); masked keys give 0
#pragma unroll
      for (int c = 0; c < ST_BN; ++c) {
        const bool vis = (c <= lim_rel) && !((pw[c >> 5] >> (c & 31)) & 1u);
        p[c] = vis ? ex2f(fmaf(p[c], scale_log2, -base_l2)) : 0.f;
      }
      if (lim_rel >= 0 && lim_rel < ST_BN) {
#pragma unroll
        for (int c = 0; c < ST_BN; ++c) diag += (c == lim_rel) ? p[c] : 0.f;
      }
      // each segment overlapping the tile: a tile inside one segment is one
      // 8-way sum; otherwise a predicated sum per overlapping segment
      for (int sg = 0; sg < n_seg; ++sg) {
        const int lo = s_lo[sg] - j0, hi = s_hi[sg] - j0;  // warp-uniform
        if (hi <= 0 || lo >= ST_BN) continue;
        float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (lo <= 0 && hi >= ST_BN) {
#pragma unroll
          for (int c = 0; c < ST_BN; ++c) a8[c & 7] += p[c];
        } else {
#pragma unroll
          for (int c = 0; c < ST_BN; ++c) a8[c & 7] += (c >= lo && c < hi) ? p[c] : 0.f;
        }
        my[sg] += ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
      }
    }
    my[n_seg] = diag;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    // fold the two warpgroups and the G heads of each row in fixed order -> part[sr][g][W]
    for (int t = et; t < R * W; t += 256) {
      const int rr = t / W, sg = t % W;
      if (r0 + rr < n_rows) {
        float v = 0.f;
        for (int h = 0; h < G; ++h)
          v += acc[(int64_t)(rr * G + h) * stride + sg] + acc[((int64_t)128 + rr * G + h) * stride + sg];
        part[((int64_t)(r0 + rr) * Hkv + g) * W + sg] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

__global__ void seg_mass_fold_kernel(const float* __restrict__ part, double* __restrict__ mass, int n_rows, int Hkv,
                                     int W, int Hq) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_rows * W) return;
  const int r = (int)(t / W), sg = (int)(t % W);
  double v = 0.0;
  for (int g = 0; g < Hkv; ++g) v += (double)part[((int64_t)r * Hkv + g) * W + sg];
  mass[t] = v / Hq;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int DH>
int launch(const void* q, const void* k, const int32_t* q_slot, const uint8_t* key_pad, const float* lse,
           const int32_t* seg_lo, const int32_t* seg_hi, int n_seg, const int32_t* rows, int n_rows, double* mass,
           int n_keys, int Hq, int Hkv, cudaStream_t st) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return fail(CC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<EncodeTiledFn>(p);
  }
  CUtensorMap mk;
  cuuint64_t dims[2] = {(cuuint64_t)Hkv * DH, (cuuint64_t)n_keys};
  cuuint64_t strides[1] = {(cuuint64_t)Hkv * DH * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)ST_BN};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(k), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(CC_E_CUDA, "segment_mass_tc: tensor map encode failed");
  const int G = Hq / Hkv, R = 128 / G, W = n_seg + 1;
  float* part = (float*)stream_scratch(st, SCR_SEGMASS, sizeof(float) * (size_t)n_rows * Hkv * W);
  if (!part) return fail(CC_E_CUDA, "segment_mass_tc: scratch allocation failed");
  const int stride = W | 1;  // odd: the rows' accumulators fall in distinct banks
  dim3 grid(Hkv, (n_rows + R - 1) / R);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  static const int stages = [] {
    const char* e = getenv("CCB_K8_STAGES");
    return e ? atoi(e) : 4;
  }();
  static const int k8_pf = [] {  // exponential pairs (of 8) on the FMA pipe in the fast path
    const char* e = getenv("CCB_K8_PF");
    return e ? atoi(e) : 2;
  }();
  auto go = [&](auto tag) -> int {
    constexpr int S = decltype(tag)::value;
    const size_t smem = StSmem<DH, S>::total(stride);
    auto kern = k8_pf == 0 ? attn_stats_tc_kernel<DH, S, 0>
                : k8_pf == 3 ? attn_stats_tc_kernel<DH, S, 3>
                : k8_pf == 4 ? attn_stats_tc_kernel<DH, S, 4> : attn_stats_tc_kernel<DH, S, 2>;
    if (int rc = ensure_smem(kern, smem)) return rc;
    kern<<<grid, 320, smem, st>>>(mk, (const __nv_bfloat16*)q, rows, n_rows, q_slot, key_pad,
                                                          lse, seg_lo, seg_hi, n_seg, part, n_keys, Hq, Hkv, G,
                                                          scale_log2, stride);
    return check_launch("segment_mass_tc");
  };
  // a 4-deep K ring while the per-row segment accumulators leave room (<= ~60 segments)
  const bool deep = stages != 2 && StSmem<DH, 4>::total(stride) <= 227 * 1024;
  int rc = deep ? go(std::integral_constant<int, 4>{}) : go(std::integral_constant<int, 2>{});
  if (rc) return rc;
  const int64_t total = (int64_t)n_rows * W;
  seg_mass_fold_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(part, mass, n_rows, Hkv, W, Hq);
  return check_launch("segment_mass_fold");
}

}  // namespace

int segment_mass_tc_bf16(const void* q, const void* k, const int32_t* q_slot, const uint8_t* key_pad,
                         const float* lse, const int32_t* seg_lo, const int32_t* seg_hi, int n_seg,
                         const int32_t* rows, int n_rows, double* mass, int n_keys, int Hq, int Hkv, int dh,
                         cudaStream_t st) {
  const int G = Hq / Hkv;
  if (G < 1 || G > 128 || (128 % G) != 0) return fail(CC_E_UNSUP, "segment_mass_tc: GQA group must divide 128");
  if (n_seg + 1 > ST_MAXSEG) return fail(CC_E_UNSUP, "segment_mass_tc: too many segments");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15)
    return fail(CC_E_UNSUP, "segment_mass_tc: pointers must be 16-byte aligned");
  if (dh == 128)
    return launch<128>(q, k, q_slot, key_pad, lse, seg_lo, seg_hi, n_seg, rows, n_rows, mass, n_keys, Hq, Hkv, st);
  if (dh == 64)
    return launch<64>(q, k, q_slot, key_pad, lse, seg_lo, seg_hi, n_seg, rows, n_rows, mass, n_keys, Hq, Hkv, st);
  return fail(CC_E_UNSUP, "segment_mass_tc: d_head must be 64 or 128");
}

}  // namespace ccb
