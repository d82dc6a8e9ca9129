// tcgen05 / TMEM / TMA bf16 GEMM for the recompute rows (K3/K5/K6):
// C[M,N] = A[M,K] B[N,K]^T, fp32 accumulation in TMEM, fused epilogues
// (model.py:399-401 QKV, :417 o_proj + residual, :418-419 MLP).
//
// Two kernels, both persistent and warp-specialised (one CTA per SM):
//   gemm_tc_kernel    1-CTA 128 x BN tiles (data-parallel, stream-K tail, or
//                     swap-AB with the activation rows as the MMA N side)
//   gemm_pair_kernel  CTA pairs (cta_group::2), 256 weight rows x n activation
//                     rows per unit from a host-planned unit table, TMA-store /
//                     TMA-reduce-add epilogues; pick_tiling chooses per shape
//   warp 0     TMA producer (A and B tiles, 128B swizzle, 4-6 stage ring)
//   warp 1     MMA issuer (single thread, tcgen05.mma) + TMEM owner
//   warps 2-5  epilogue (tcgen05.ld 32 lanes x 32 cols -> registers -> global)
// Both launch with programmatic dependent launch when enabled (cc_set_pdl):
// barrier init, TMEM allocation and the first weight tiles are issued before
// griddepcontrol.wait.
// Two TMEM accumulators (2 x 256 columns) let tile i's epilogue overlap tile
// i+1's MMAs.  Tiles are walked M-fastest so the CTAs of one wave share the
// weight tile through L2.  Wave quantisation (M ~ 800 gives 112-224 tiles on
// 148 SMs) is removed by a stream-K tail with deterministic fixed-order folds;
// impl 4 (no split) keeps a row's result independent of M.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <queue>
#include <vector>
#include <algorithm>
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
  // as many stages as fit next to the barriers and the 16 KiB transpose slabs
  // (227 KiB per CTA): BN 256 -> 4, 208 / 192 / 160 -> 5, 128 -> 6
  static constexpr int RING = 232448 - 1024 - 256 - 4 * 4096;
  static constexpr int STAGES = RING / (TC_A_BYTES + B_BYTES) > 6 ? 6 : RING / (TC_A_BYTES + B_BYTES);
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int ACC_STRIDE = 2 * BN <= 256 ? BN : 256;  // TMEM column of accumulator 1
  // + 4 per-warp 4 KiB transpose slabs + 8 KiB gate/up exchange (swap SwiGLU)
  static constexpr size_t SMEM = 1024 + STAGES * (TC_A_BYTES + B_BYTES) + 256 + 4 * 4096;
};

using namespace sm100;

// Work schedule (persistent grid of G co-resident CTAs):
//   tiles [0, t_dp)      data-parallel: CTA c takes tiles c, c + G, ... whole
//   tiles [t_dp, tiles)  stream-K: their k-blocks, linearised tile-major, are
//                        cut into G equal contiguous ranges, one per CTA
// A stream-K tile is covered by CTAs c_lo..c_hi.  Every CTA but c_lo meets
// the tile at the START of its range (its only non-final fragment): it parks
// its fp32 partial in its own workspace slot and stamps flags[c].  c_lo meets
// the tile at the END of its range, waits for the stamps of c_lo+1..c_hi and
// folds their slots onto its accumulator in that fixed order (deterministic,
// and a CTA only ever waits on work other CTAs do first: no deadlock).
struct Unit {
  int tile, k0, k1, order, nfrag;
};

struct UnitIter {
  int nkb, t_dp, G, c, dp_next;
  long long W, g, g_end;
  __device__ UnitIter(int nkb_, int t_dp_, long long W_, int G_, int c_)
      : nkb(nkb_), t_dp(t_dp_), G(G_), c(c_), dp_next(c_), W(W_) {
    g = W > 0 ? (long long)c * W / G : 0;
    g_end = W > 0 ? (long long)(c + 1) * W / G : 0;
  }
  __device__ int cta_of(long long x) const { return (int)(((x + 1) * G - 1) / W); }
  __device__ bool next(Unit& u) {
    if (dp_next < t_dp) {
      u.tile = dp_next; u.k0 = 0; u.k1 = nkb; u.order = 0; u.nfrag = 1;
      dp_next += G;
      return true;
    }
    if (g >= g_end) return false;
    const int t = (int)(g / nkb);
    const long long tb = (long long)t * nkb, te = tb + nkb;
    const long long e = te < g_end ? te : g_end;
    u.tile = t_dp + t;
    u.k0 = (int)(g - tb);
    u.k1 = (int)(e - tb);
    const int c_lo = cta_of(tb), c_hi = cta_of(te - 1);
    u.order = c_hi - c;
    u.nfrag = c_hi - c_lo + 1;
    g = e;
    return true;
  }
};

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 32x32 fp32 transpose through a per-warp 4 KiB smem slab (16-byte units
// XOR-swizzled by row: conflict-free both ways).  In: r = this lane's row
// (32 columns).  Out: v[i] = row (lane >> 3) + 4 i, columns (lane & 7) * 4 .. +3.
__device__ __forceinline__ void transpose32(uint32_t stg, const uint32_t (&r)[32], int lane, float4 (&v)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + (lane * 8 + (j ^ (lane & 7))) * 16),
                 "r"(r[4 * j]), "r"(r[4 * j + 1]), "r"(r[4 * j + 2]), "r"(r[4 * j + 3])
                 : "memory");
  __syncwarp();
  const int c4 = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (lane >> 3) + 4 * i;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[i].x), "=f"(v[i].y), "=f"(v[i].z), "=f"(v[i].w)
                 : "r"(stg + (rr * 8 + (c4 ^ (rr & 7))) * 16)
                 : "memory");
  }
  __syncwarp();
}

// fp32 fold of v with a global slab (row stride ld_rows4 = 4 rows, in
// floats) through L2 (.cg: written by other CTAs).  All loads are issued
// before any store: __ldcg/__stcg are volatile asm and would otherwise
// serialise on the L2 round trip.
__device__ __forceinline__ void fold8(float* p, int64_t ld_rows4, const bool (&ok)[8], float4 (&v)[8], bool add,
                                      bool store) {
  if (add) {
    float4 w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (ok[i]) w[i] = __ldcg(reinterpret_cast<const float4*>(p + i * ld_rows4));
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (ok[i]) { v[i].x += w[i].x; v[i].y += w[i].y; v[i].z += w[i].z; v[i].w += w[i].w; }
  }
  if (store) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (ok[i]) __stcg(reinterpret_cast<float4*>(p + i * ld_rows4), v[i]);
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// named barrier of epilogue warps q and q ^ 2 (ids 2, 3)
__device__ __forceinline__ void pair_bar(int q) { asm volatile("bar.sync %0, 64;" ::"r"(2 + (q & 1)) : "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// SWAP (swap-AB, small M): the kernel computes C^T = W X^T — the A slot
// holds 128-row weight tiles (MMA M), the B slot TC_BN-row activation tiles
// (MMA N, any multiple of 16: M = 802 rows -> 4 tiles of 208, 3.7% padding
// instead of 7 x 128).  M / N below are then (output features, rows); the
// epilogue transposes back and writes C[row][feature].
template <int EPI, int TC_BN, bool SPLIT, bool SWAP = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* C,
                   int64_t ldc, int M, int N, int K, int t_dp, long long W, float* __restrict__ ws,
                   int* __restrict__ flags, int epoch, long long* __restrict__ trace, const PeerTab peer) {
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
  // per-epilogue-warp 4 KiB transpose slabs, after the barriers (1 KiB aligned)
  float4* stg_base = reinterpret_cast<float4*>(sB + TC_STAGES * TC_B_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + TC_BM - 1) / TC_BM;
  const int num_tiles = num_m * ((N + TC_BN - 1) / TC_BN);  // last N tile may be ragged (TMA zero-fills)
  const int num_kb = K / TC_BK;
  if (!SPLIT) { t_dp = num_tiles; W = 0; }

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
  pdl_trigger();
  if (warp != 0) pdl_wait();  // (the producer waits after issuing its first weight tiles)

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      UnitIter it(num_kb, t_dp, W, gridDim.x, blockIdx.x);
      Unit w;
      const int num_n = (N + TC_BN - 1) / TC_BN;
      // (swap: row tiles fastest so a wave's CTAs share each weight tile)
      auto tile_mn = [&](const Unit& x, int& mt, int& nt) {
        mt = SWAP ? x.tile / num_n : x.tile % num_m;
        nt = SWAP ? x.tile % num_n : x.tile / num_m;
      };
      bool have = it.next(w);
      // PDL: the weight tiles of the first ring fill do not depend on the
      // predecessor kernel -> issue them before griddepcontrol.wait
      int pre = 0;
      if (have) {
        int mt, nt;
        tile_mn(w, mt, nt);
        pre = min(TC_STAGES, w.k1 - w.k0);
        for (int i = 0; i < pre; ++i) {
          mbar_expect_tx(&full[i], TC_A_BYTES + TC_B_BYTES);
          if (SWAP) tma_load_2d(sA + i * TC_A_BYTES, &tmA, &full[i], (w.k0 + i) * TC_BK, mt * TC_BM);
          else tma_load_2d(sB + i * TC_B_BYTES, &tmB, &full[i], (w.k0 + i) * TC_BK, nt * TC_BN);
        }
      }
      pdl_wait();
      for (bool first = true; have; first = false, have = it.next(w)) {
        int mt, nt;
        tile_mn(w, mt, nt);
        for (int kb = w.k0; kb < w.k1; ++kb) {
          if (first && kb - w.k0 < pre) {  // weights already in flight: the activation tile only
            if (SWAP) tma_load_2d(sB + stage * TC_B_BYTES, &tmB, &full[stage], kb * TC_BK, nt * TC_BN);
            else tma_load_2d(sA + stage * TC_A_BYTES, &tmA, &full[stage], kb * TC_BK, mt * TC_BM);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], TC_A_BYTES + TC_B_BYTES);
            tma_load_2d(sA + stage * TC_A_BYTES, &tmA, &full[stage], kb * TC_BK, mt * TC_BM);
            tma_load_2d(sB + stage * TC_B_BYTES, &tmB, &full[stage], kb * TC_BK, nt * TC_BN);
          }
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
      UnitIter it(num_kb, t_dp, W, gridDim.x, blockIdx.x);
      Unit w;
      while (it.next(w)) {
        const int k0 = w.k0, k1 = w.k1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TcCfg<TC_BN>::ACC_STRIDE;
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
    const uint32_t stg = smem_u32(stg_base + (warp - 2) * 256);
    int acc = 0;
    uint32_t acc_phase = 0;
    UnitIter it(num_kb, t_dp, W, gridDim.x, blockIdx.x);
    Unit w;
    int ui = 0;
    while (it.next(w)) {
      const int tile = w.tile, sp = w.order;
      const int num_n = (N + TC_BN - 1) / TC_BN;
      const int mt = SWAP ? tile / num_n : tile % num_m, nt = SWAP ? tile % num_n : tile / num_m;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      long long* tr = (trace != nullptr && et == 0 && ui < 8) ? trace + ((int64_t)blockIdx.x * 8 + ui) * 8 : nullptr;
      if (tr) { tr[0] = tile; tr[1] = sp; tr[2] = w.nfrag; tr[3] = w.k1 - w.k0; tr[4] = globaltimer(); }
      const int row = mt * TC_BM + q * 32 + lane;
      const uint32_t t0 = tmem_base + acc * TcCfg<TC_BN>::ACC_STRIDE + ((uint32_t)(q * 32) << 16);
      const int n0 = nt * TC_BN;
      // stream-K: non-final fragments park partials; the final one folds them
      const bool split = SPLIT && w.nfrag > 1;
      const bool last = sp == w.nfrag - 1;  // c_lo: applies the epilogue
      const int c_hi = blockIdx.x + sp;
      if (split && last) {
        for (int j = et; j < c_hi - (int)blockIdx.x; j += 128)
          while (ld_acquire(&flags[blockIdx.x + 1 + j]) != epoch) __nanosleep(32);
        epi_bar();
      }
      if (tr) tr[5] = globaltimer();
      // this CTA's partial slot [128][TC_BN] fp32 (non-final) / slot of CTA j (final)
      auto slot = [&](int cta, int col) -> float* {
        return ws + (int64_t)cta * (TC_BM * TC_BN) + (int64_t)(q * 32 + (lane >> 3)) * TC_BN + col + (lane & 7) * 4;
      };
      auto fold_in = [&](float4 (&v)[8], int col, const bool (&okr)[8]) {
        for (int j = blockIdx.x + 1; j <= c_hi; ++j) fold8(slot(j, col), 4 * TC_BN, okr, v, true, false);
      };
      // Coalesced epilogue: each 32x32 fp32 chunk (thread = row after
      // tcgen05.ld) is transposed through a 4 KiB swizzled smem slab so that
      // a warp instruction covers 4 rows x 128 B; lane -> (row rb + 4 i,
      // cols c4*4 .. +3), i = 0..7.
      const int rb = mt * TC_BM + q * 32 + (lane >> 3);
      const int c4 = lane & 7;
      bool ok[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) ok[i] = rb + 4 * i < M;
      if constexpr (SWAP) {
        // TMEM lane = output feature mt*128 + q*32 + lane, TMEM column = row:
        // a tcgen05.ld chunk already gives each thread one feature for 32 rows,
        // so a warp store covers 32 consecutive features of one row (coalesced
        // without a transpose).
        const int feat = mt * TC_BM + q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < (TC_BN + 31) / 32; ++c) {
          if (n0 + c * 32 >= N) break;
          uint32_t r[32];
          tmem_ld32(t0 + c * 32, r);
          tmem_ld_wait();
          const int jmax = min(32, min(TC_BN - c * 32, N - n0 - c * 32));  // rows of this chunk in tile and matrix
          static_assert(EPI != CC_EPI_SWIGLU, "swap-AB has no SwiGLU epilogue (measured slower; see pick_tiling)");
          if constexpr (false) {
          } else if constexpr (EPI == CC_EPI_RESID_ADD) {
            float* h = reinterpret_cast<float*>(C) + (int64_t)(n0 + c * 32) * ldc + feat;
            float cv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < jmax) cv[j] = h[(int64_t)j * ldc];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < jmax) h[(int64_t)j * ldc] = cv[j] + __uint_as_float(r[j]);
          } else {
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)(n0 + c * 32) * ldc + feat;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (j >= jmax) continue;
              float x = __uint_as_float(r[j]);
              if constexpr (EPI == CC_EPI_GELU) x = gelu_tanh(x);
              out[(int64_t)j * ldc] = __float2bfloat16_rn(x);
            }
          }
        }
      } else
      if constexpr (EPI == CC_EPI_SWIGLU && TC_BN == 256) {
        // tile columns: [gate 64 | up 64 | gate 64 | up 64] -> 128 outputs
#pragma unroll 1
        for (int g = 0; g < 4; ++g) {
          const int gc = (g >> 1) * 128 + (g & 1) * 32;
          float4 vg[8], vu[8];
          {
            uint32_t r[32];
            tmem_ld32(t0 + gc, r);
            tmem_ld_wait();
            transpose32(stg, r, lane, vg);
            tmem_ld32(t0 + gc + 64, r);
            tmem_ld_wait();
            transpose32(stg, r, lane, vu);
          }
          if (split && !last) {
            fold8(slot(blockIdx.x, gc), 4 * TC_BN, ok, vg, false, true);
            fold8(slot(blockIdx.x, gc + 64), 4 * TC_BN, ok, vu, false, true);
          } else if (split) {
            fold_in(vg, gc, ok);
            fold_in(vu, gc + 64, ok);
          }
          if (last) {
            __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)rb * ldc + n0 / 2 + (g >> 1) * 64 +
                                 (g & 1) * 32 + c4 * 4;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (!ok[i]) continue;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(silu(vg[i].x) * vu[i].x, silu(vg[i].y) * vu[i].y);
              __nv_bfloat162 h1 = __floats2bfloat162_rn(silu(vg[i].z) * vu[i].z, silu(vg[i].w) * vu[i].w);
              *reinterpret_cast<uint2*>(out + (int64_t)4 * i * ldc) =
                  make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < TC_BN / 32; ++c) {
          if (n0 + c * 32 >= N) break;  // ragged last tile (N % 32 == 0)
          float4 v[8];
          {
            uint32_t r[32];
            tmem_ld32(t0 + c * 32, r);
            tmem_ld_wait();
            transpose32(stg, r, lane, v);
          }
          const int col = n0 + c * 32 + c4 * 4;
          if constexpr (EPI == CC_EPI_PEER_PUSH) {
            // reduce-scatter push: this rank's fp32 partial of the tile goes
            // straight into the owner's receive slab over NVLink (P2P stores),
            // tile by tile as the GEMM produces it
            const int owner = n0 / peer.slice;
            float* dst = peer.recv[owner] + ((int64_t)peer.rank * peer.m_cap + rb) * peer.slice + (col - owner * peer.slice);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (ok[i]) *reinterpret_cast<float4*>(dst + (int64_t)4 * i * peer.slice) = v[i];
          } else if constexpr (EPI == CC_EPI_RESID_ADD) {
            float* h = reinterpret_cast<float*>(C) + (int64_t)rb * ldc + col;
            if (split && !last) {
              fold8(slot(blockIdx.x, c * 32), 4 * TC_BN, ok, v, false, true);
            } else {
              if (split) fold_in(v, c * 32, ok);
              float4 cv[8];
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (ok[i]) cv[i] = *reinterpret_cast<const float4*>(h + (int64_t)4 * i * ldc);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (ok[i])
                  *reinterpret_cast<float4*>(h + (int64_t)4 * i * ldc) =
                      make_float4(cv[i].x + v[i].x, cv[i].y + v[i].y, cv[i].z + v[i].z, cv[i].w + v[i].w);
            }
          } else {
            if (split && !last) fold8(slot(blockIdx.x, c * 32), 4 * TC_BN, ok, v, false, true);
            else if (split) fold_in(v, c * 32, ok);
            if (last) {
              __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (int64_t)rb * ldc + col;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (!ok[i]) continue;
                float4 x = v[i];
                if constexpr (EPI == CC_EPI_GELU) {
                  x.x = gelu_tanh(x.x); x.y = gelu_tanh(x.y); x.z = gelu_tanh(x.z); x.w = gelu_tanh(x.w);
                }
                __nv_bfloat162 h0 = __floats2bfloat162_rn(x.x, x.y), h1 = __floats2bfloat162_rn(x.z, x.w);
                *reinterpret_cast<uint2*>(out + (int64_t)4 * i * ldc) =
                    make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if constexpr (EPI == CC_EPI_PEER_PUSH) {
        // all 128 epilogue threads' stores are visible system-wide before the
        // owner sees this tile's stamp
        __threadfence_system();
        epi_bar();
        if (et == 0) {
          const int owner = n0 / peer.slice;
          const int per = peer.slice / TC_BN;
          const int local = mt * per + (nt - owner * per);
          int* f = peer.flags[owner] + (int64_t)peer.rank * (((M + TC_BM - 1) / TC_BM) * per) + local;
          asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(peer.epoch) : "memory");
        }
      }
      if (split && !last) {
        __threadfence();
        epi_bar();
        if (et == 0) st_release(&flags[blockIdx.x], epoch);
      }
      if (tr) tr[6] = globaltimer();
      ++ui;
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

// ---- unit table (host-planned work list of the CTA-pair kernel) -----------
// With the activation rows as the MMA N dimension a unit may cover any
// multiple of 32 rows (<= 256) of one 256-feature weight tile.  The host cuts
// every weight tile's rows into chunks and assigns the units to the CTA pairs
// (plan_units), passed as a kernel parameter.  Every output element is still
// produced by one unit with the full K reduction in order (no split, no
// workspace).
constexpr int SW_MAXG = 80;    // CTA pairs (>= SM count / 2)
constexpr int SW_MAXU = 4096;  // units per launch (the table rides in the kernel parameters: <= 32 KiB)
struct SwTab {
  uint16_t start[SW_MAXG + 1];  // CTA c runs units [start[c], start[c+1])
  uint32_t unit[SW_MAXU];       // feature tile | (row0 / 16) << 14 | (rows / 16 - 1) << 25
  uint8_t ks[SW_MAXU];          // K split: slice s << 4 | (slices - 1); 0 = the whole K
};
// K-split units (small M: too few (tile, row chunk) units for the CTA pairs):
// slice s of S covers k-blocks [s * nkb / S, (s + 1) * nkb / S).  Each CTA
// parks its fp32 partial in ws[s][row][feature] (row stride F), bumps the
// (tile, chunk, CTA rank) ticket, and the CTA that draws the last ticket sums
// the S partials in slice order (its own from TMEM) before the normal
// epilogue -- deterministic whichever CTA finishes last.
struct KSplit {
  float* ws;         // [S_max][Mpad][F] fp32
  unsigned* ticket;  // [F / 128][Mpad / 32], zero between launches
  int Mpad, F;
};
__host__ __device__ constexpr uint32_t sw_pack(int ft, int r0, int n) {
  return (uint32_t)ft | ((uint32_t)(r0 >> 4) << 14) | ((uint32_t)((n >> 4) - 1) << 25);
}

// ---- CTA-pair (cta_group::2) swap-AB with a unit table ----------------------
// A 1-CTA 128 x 256 tile moves 48 KiB into shared memory per k-block (TMA)
// and the MMA reads the same 48 KiB back: ~768 cycles at the ~128 B/clk
// shared-memory port where the MMA needs 512, so the kernel above is
// operand-feed bound (measured ~430 ns per k-block).  A CTA pair computes a
// 256-feature x n-row tile with one tcgen05.mma.cta_group::2: each SM holds
// its 128 weight rows and HALF of the n activation rows (the pair's tensor
// cores exchange the halves), so for n = 256 an SM moves 32 KiB in and 32 KiB
// out per k-block — matched to the MMA's 512 cycles.  The leader CTA (rank 0) issues
// the MMAs; both CTAs load through TMA onto the leader's full barrier, the
// commits multicast to both CTAs' empty / accumulator-full barriers, and both
// CTAs' epilogue warps release the accumulator to the leader's barrier.
// Units (256-feature tile, row0, n rows; n % 32 == 0) come from the host LPT
// table, one list per pair.
constexpr int P2_STAGES = 6;                       // 6 x (16 + 16) KiB
constexpr int P2_B_BYTES = 128 * TC_BK * 2;        // <= 128 activation rows per CTA
// + 32 KiB epilogue staging: per epilogue warp two 4 KiB slabs (32 rows x 32
// features, fp32 or bf16) drained by TMA stores / reduce-adds
constexpr size_t P2_SMEM = 1024 + P2_STAGES * (TC_A_BYTES + P2_B_BYTES) + 256 + 8 * 4096;

// QKV projection with RoPE and the K/V scatter in the epilogue (K3,
// model.py:399-404): the 128 features of a CTA are one head (d_head 128) of
// [q heads | k heads | v heads]; warps q and q ^ 2 hold the RoPE partners
// (features i and i + 64) and swap their chunks through shared memory, so
// each warp rotates its own 32 features for all 32 rows of a chunk.  q ->
// q_rot[row] (32 x 32 TMA stores); k -> kv_k[slot] (as computed) and
// k_rot[slot] (rotated); v -> kv_v[slot] (64-byte row segments).  Each value is rounded to bf16
// before the rotation, so the results equal the unfused GEMM + rope_scatter.
constexpr int EPI_ROPE_QKV = 5;  // (internal epilogue id, not part of the ABI enum)
struct RopeQkv {
  const int32_t* row_slot;
  const int32_t* row_pos;
  const float2* table;  // [max_pos][64] (cos, sin)
  __nv_bfloat16* q_rot;
  __nv_bfloat16* kv_k;
  __nv_bfloat16* kv_v;
  __nv_bfloat16* k_rot;
  int Hq, Hkv;
};

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX128,
                     const __grid_constant__ CUtensorMap tmX64, const __grid_constant__ CUtensorMap tmX32,
                     const __grid_constant__ CUtensorMap tmX16, const __grid_constant__ CUtensorMap tmC, int M,
                     int K, int dbg, const __grid_constant__ SwTab tab, const RopeQkv rq, const KSplit ksp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + P2_STAGES * TC_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + P2_STAGES * P2_B_BYTES);
  uint64_t* empty = full + P2_STAGES;
  uint64_t* tfull = empty + P2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* stg_base = sB + P2_STAGES * P2_B_BYTES + 256;
  __shared__ bool ks_last_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int num_kb = K / TC_BK;
  const int pair = blockIdx.x >> 1;
  const int u_begin = tab.start[pair], u_end = tab.start[pair + 1];

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX128);
    for (int s = 0; s < P2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  if (warp != 0) pdl_wait();  // (the producer waits after issuing its first weight tiles)

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // PDL: the first ring fill's weight tiles do not depend on the predecessor
      int pre = 0;
      if (u_begin < u_end && !(dbg & 2)) {
        const uint32_t e = tab.unit[u_begin];
        const int fp = e & 0x3fff, n = (((e >> 25) & 0xf) + 1) * 16;
        const int ks = tab.ks[u_begin], kb0 = (ks >> 4) * num_kb / ((ks & 15) + 1);
        const int kb1 = ((ks >> 4) + 1) * num_kb / ((ks & 15) + 1);
        pre = min(P2_STAGES, kb1 - kb0);
        for (int i = 0; i < pre; ++i) {
          const uint32_t fb = mapa_shared(smem_u32(&full[i]), 0);
          if (rank == 0) mbar_expect_tx(&full[i], 2 * (TC_A_BYTES + (n / 2) * TC_BK * 2));
          tma_load_2d_pair(sA + i * TC_A_BYTES, &tmW, fb, (kb0 + i) * TC_BK, fp * 2 * TC_BM + (int)rank * TC_BM);
        }
      }
      pdl_wait();
      for (int u = u_begin; u < u_end; ++u) {
        const uint32_t e = tab.unit[u];
        const int fp = e & 0x3fff, r0 = ((e >> 14) & 0x7ff) * 16, n = (((e >> 25) & 0xf) + 1) * 16;
        const int h = n / 2;  // rows per CTA (multiple of 16)
        const int rows0 = r0 + (int)rank * h;
        const int ks = tab.ks[u], kb0 = (ks >> 4) * num_kb / ((ks & 15) + 1);
        const int kb1 = ((ks >> 4) + 1) * num_kb / ((ks & 15) + 1);
        for (int kb = kb0; kb < kb1; ++kb) {
          const bool prefetched = u == u_begin && kb - kb0 < pre;
          if (!prefetched) mbar_wait(&empty[stage], phase ^ 1);
          if ((dbg & 2) && (u > u_begin || kb - kb0 >= P2_STAGES)) {  // debug: MMA on stale tiles (no feed)
            if (rank == 0) mbar_arrive(&full[stage]);
            if (++stage == P2_STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (!prefetched) {
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * (TC_A_BYTES + h * TC_BK * 2));
            tma_load_2d_pair(sA + stage * TC_A_BYTES, &tmW, fb, kb * TC_BK, fp * 2 * TC_BM + (int)rank * TC_BM);
          }
          uint8_t* dst = sB + stage * P2_B_BYTES;
          int off = 0;
          if (h & 128) { tma_load_2d_pair(dst, &tmX128, fb, kb * TC_BK, rows0); off += 128; }
          if (h & 64) { tma_load_2d_pair(dst + off * 128, &tmX64, fb, kb * TC_BK, rows0 + off); off += 64; }
          if (h & 32) { tma_load_2d_pair(dst + off * 128, &tmX32, fb, kb * TC_BK, rows0 + off); off += 32; }
          if (h & 16) tma_load_2d_pair(dst + off * 128, &tmX16, fb, kb * TC_BK, rows0 + off);
          if (++stage == P2_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = u_begin; u < u_end; ++u) {
        const int n = (((tab.unit[u] >> 25) & 0xf) + 1) * 16;
        const uint32_t idesc = idesc_bf16_f32(2 * TC_BM, n);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        const int ks = tab.ks[u], kb0 = (ks >> 4) * num_kb / ((ks & 15) + 1);
        const int kb1 = ((ks >> 4) + 1) * num_kb / ((ks & 15) + 1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = desc_sw128(sA + stage * TC_A_BYTES);
          const uint64_t bd = desc_sw128(sB + stage * P2_B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            mma_bf16_pair(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == P2_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter = features q*32 .. +31 of this CTA's 128
    // staging: warp q owns two 4 KiB slabs at stg_base + q * 8 KiB (alternate
    // chunks, so a chunk's TMA store drains while the next one is written);
    // SwiGLU stages 16 x 32 bf16 per slab and swaps half chunks with warp q ^ 2
    // through bytes 2048.. of its first slab
    uint8_t* my_slab = stg_base + q * 8192;
    int acc = 0;
    uint32_t acc_phase = 0;
    int nst = 0;  // TMA stores issued by this warp (slab parity)
    for (int u = u_begin; u < u_end; ++u) {
      const uint32_t e = tab.unit[u];
      const int fp = e & 0x3fff, r0 = ((e >> 14) & 0x7ff) * 16, n = (((e >> 25) & 0xf) + 1) * 16;
      const int ft = fp * 2 + (int)rank;  // this CTA's 128-feature tile
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t0 = tmem_base + acc * 256 + ((uint32_t)(q * 32) << 16);
      const int ks = tab.ks[u], ns = (ks & 15) + 1, my_s = ks >> 4;
      const int feat = ft * TC_BM + q * 32 + lane;  // this thread's feature (TMEM lane)
      if (ns > 1 && !(dbg & 16)) {  // (debug 16: no partials / tickets, every slice stores)
        // park this slice's partial: ws[my_s][row][feat] for rows r0 .. r0 + n
        // (a warp's store per row = 32 consecutive features = one 128-byte line)
        float* dst = ksp.ws + ((int64_t)my_s * ksp.Mpad + r0) * ksp.F + feat;
#pragma unroll 1
        for (int c = 0; c * 32 < n; ++c) {
          uint32_t r[32];
          tmem_ld32(t0 + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(dst + (int64_t)(c * 32 + j) * ksp.F, __uint_as_float(r[j]));
        }
        __threadfence();
        epi_bar();
        unsigned* tk = ksp.ticket + (int64_t)ft * (ksp.Mpad / 32) + r0 / 32;
        if (threadIdx.x == 64) {  // (first epilogue thread) release the partials, acquire the others'
          unsigned prev;
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(tk) : "memory");
          ks_last_s = prev == (unsigned)(ns - 1);
          if (ks_last_s) *tk = 0u;  // ready for the next launch on this stream
        }
        epi_bar();
        if (!ks_last_s) {  // another slice's CTA finishes this unit
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
      }
      // r[j] (row r0 + 32 c + j of this thread's feature) = the slices summed in order
      auto fold = [&](int c, uint32_t (&r)[32]) {
        if (ns == 1 || (dbg & 48)) return;  // (debug 32: partials parked, no fold)
        float a[32];
#pragma unroll 1
        for (int s2 = 0; s2 < ns; ++s2) {
          if (s2 == my_s) {
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = s2 == 0 ? __uint_as_float(r[j]) : a[j] + __uint_as_float(r[j]);
          } else {
            const float* src = ksp.ws + ((int64_t)s2 * ksp.Mpad + r0 + c * 32) * ksp.F + feat;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __ldcg(src + (int64_t)j * ksp.F);
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = s2 == 0 ? v[j] : a[j] + v[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(a[j]);
      };
      if constexpr (EPI == EPI_ROPE_QKV) {
        // warp slab (8 KiB): [0, 4K) this warp's fp32 chunk for the partner,
        // [4K, 6K) / [6K, 8K) bf16 [32 rows][32 features] output staging.
        // (Loading the next chunk's cos/sin during the current one measured
        // slower: 61.1 vs 57.8 us at M = 802.)
        const int kvw = rq.Hkv * 128;
        const int kind = ft < rq.Hq ? 0 : ft < rq.Hq + rq.Hkv ? 1 : 2;  // q / k / v head
        const int i = (q & 1) * 32 + lane;  // RoPE pair index (features i, i + 64)
        const int nch = min((n + 31) / 32, (M - r0 + 31) / 32);
        const uint32_t xo = smem_u32(my_slab), xi = smem_u32(stg_base + (q ^ 2) * 8192);
        float2 cs[32];
        int slot_c;
        auto meta = [&](int c, float2 (&cc)[32], int& slot) {
          const int row = r0 + c * 32, jmax = min(32, M - row);
          slot = (kind > 0 && lane < jmax) ? rq.row_slot[row + lane] : 0;
          if (kind < 2) {
            const int pos = lane < jmax ? rq.row_pos[row + lane] : 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) cc[j] = rq.table[(int64_t)__shfl_sync(0xffffffffu, pos, j) * 64 + i];
          }
        };
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          const int row = r0 + c * 32, jmax = min(32, M - row);
          uint32_t r[32];
          tmem_ld32(t0 + c * 32, r);
          meta(c, cs, slot_c);
          tmem_ld_wait();
          fold(c, r);
          if (dbg & 1) continue;  // debug: no stores
          // q heads alternate the two staging slabs (a chunk's TMA store drains
          // while the next is written); k / v heads use both, read back here
          const uint32_t ob0 = xo + 4096 + (kind == 0 ? (nst & 1) * 2048 : 0), ob1 = xo + 6144;
          if (lane == 0) {
            if (kind == 0) bulk_wait_read<1>();  // the store that last read this slab is done reading
            else bulk_wait_read<0>();
          }
          __syncwarp();
          if (kind < 2) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(xo + (j * 32 + lane) * 4), "r"(r[j]) : "memory");
            pair_bar(q);
            const bool xw = q < 2;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float other;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xi + (j * 32 + lane) * 4) : "memory");
              const __nv_bfloat16 ob = __float2bfloat16_rn(__uint_as_float(r[j]));
              const float mine = __bfloat162float(ob), oth = __bfloat162float(__float2bfloat16_rn(other));
              const float2 csj = cs[j];
              float fx, fy;
              rope_pair(xw ? mine : oth, xw ? oth : mine, csj.x, csj.y, fx, fy);
              const __nv_bfloat16 rb = __float2bfloat16_rn(xw ? fx : fy);
              if (kind == 0) {
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(ob0 + j * 64 + lane * 2),
                             "h"(*reinterpret_cast<const uint16_t*>(&rb)) : "memory");
              } else {
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(ob0 + j * 64 + lane * 2),
                             "h"(*reinterpret_cast<const uint16_t*>(&ob)) : "memory");
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(ob1 + j * 64 + lane * 2),
                             "h"(*reinterpret_cast<const uint16_t*>(&rb)) : "memory");
              }
            }
            pair_bar(q);  // both warps have read the other's chunk
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const __nv_bfloat16 ob = __float2bfloat16_rn(__uint_as_float(r[j]));
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(ob0 + j * 64 + lane * 2),
                           "h"(*reinterpret_cast<const uint16_t*>(&ob)) : "memory");
            }
          }
          if (kind == 0) {  // q rows are contiguous: one TMA store of the 32 x 32 block
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, my_slab + 4096 + (nst & 1) * 2048, ft * TC_BM + q * 32, row);
              bulk_commit();
            }
            ++nst;
          } else {
            // k / v rows go to their slots: two 64-byte rows per warp store
            __syncwarp();
            const int half = lane >> 4, c4 = lane & 15;
            const int64_t col = (int64_t)(ft - rq.Hq - (kind == 2 ? rq.Hkv : 0)) * 128 + q * 32 + c4 * 2;
            const int my_slot = slot_c;
#pragma unroll 4
            for (int it = 0; it < 16; ++it) {
              const int rr = it * 2 + half;
              const int sl = __shfl_sync(0xffffffffu, my_slot, rr);
              if (rr >= jmax) continue;
              uint32_t v0, v1 = 0;
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v0) : "r"(ob0 + rr * 64 + c4 * 4) : "memory");
              if (kind == 1)
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v1) : "r"(ob1 + rr * 64 + c4 * 4) : "memory");
              const int64_t o = (int64_t)sl * kvw + col;
              if (kind == 1) {
                *reinterpret_cast<uint32_t*>(rq.kv_k + o) = v0;
                *reinterpret_cast<uint32_t*>(rq.k_rot + o) = v1;
              } else {
                *reinterpret_cast<uint32_t*>(rq.kv_v + o) = v0;
              }
            }
          }
        }
      } else
#pragma unroll 1
      for (int c = 0; c * 32 < n; ++c) {
        const int row = r0 + c * 32;
        if (row >= M) break;
        uint32_t r[32];
        tmem_ld32(t0 + c * 32, r);
        tmem_ld_wait();
        fold(c, r);
        if (dbg & 1) continue;  // debug: no stores
        uint8_t* slab = my_slab + (nst & 1) * 4096;
        // the TMA store that last read this slab (two stores ago) is done reading
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        if constexpr (EPI == CC_EPI_SWIGLU) {
          // warps q (gate features) and q ^ 2 (the matching up features) swap
          // half a chunk: the gate warp finishes rows 0-15, the up warp 16-31
          const bool gate = q < 2;
          const uint32_t out_x = smem_u32(my_slab) + 2048, in_x = smem_u32(stg_base + (q ^ 2) * 8192) + 2048;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(out_x + (j * 32 + lane) * 4), "r"(r[gate ? 16 + j : j])
                         : "memory");
          pair_bar(q);
          const uint32_t dst = smem_u32(slab) + lane * 2;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float other;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(in_x + (j * 32 + lane) * 4) : "memory");
            const float g = gate ? __uint_as_float(r[j]) : other, up = gate ? other : __uint_as_float(r[16 + j]);
            const __nv_bfloat16 hv = __float2bfloat16_rn(silu(g) * up);
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(dst + j * 64), "h"(*reinterpret_cast<const uint16_t*>(&hv))
                         : "memory");
          }
          pair_bar(q);  // exchange buffers reusable
        } else if constexpr (EPI == CC_EPI_RESID_ADD) {
          const uint32_t dst = smem_u32(slab) + lane * 4;
#pragma unroll
          for (int j = 0; j < 32; ++j) asm volatile("st.shared.b32 [%0], %1;" ::"r"(dst + j * 128), "r"(r[j]) : "memory");
        } else {
          const uint32_t dst = smem_u32(slab) + lane * 2;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float x = __uint_as_float(r[j]);
            if constexpr (EPI == CC_EPI_GELU) x = gelu_tanh(x);
            const __nv_bfloat16 hv = __float2bfloat16_rn(x);
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(dst + j * 64), "h"(*reinterpret_cast<const uint16_t*>(&hv))
                         : "memory");
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(dbg & 8)) {
          // rows >= M and columns past the matrix are clipped by the TMA unit
          if constexpr (EPI == CC_EPI_RESID_ADD) tma_reduce_add_2d(&tmC, slab, ft * TC_BM + q * 32, row);
          else if constexpr (EPI == CC_EPI_SWIGLU) tma_store_2d(&tmC, slab, ft * 64 + (q & 1) * 32, row + (q >> 1) * 16);
          else tma_store_2d(&tmC, slab, ft * TC_BM + q * 32, row);
          bulk_commit();
        }
        ++nst;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();  // the leader's last MMAs read this CTA's smem / write its TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
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
  int box_rows;  // < 0: output map, no swizzle: -1 bf16 32 x 32, -2 fp32 32 x 32, -3 bf16 32 cols x 16 rows
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
  const bool outmap = box_rows < 0, f32 = box_rows == -2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (f32 ? 4 : 2))};
  cuuint32_t box[2] = {(cuuint32_t)(outmap ? 32 : TC_BK), (cuuint32_t)(outmap ? (box_rows == -3 ? 16 : 32) : box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(p), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   outmap ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

long long* g_trace = nullptr;  // debug: per-CTA unit timeline (cc_gemm_set_trace)

inline int n_tiles_of(int N, int bn) { return (N + bn - 1) / bn; }

// Tiling plan: tile width, how many tiles run data-parallel, the stream-K
// k-block total and the persistent grid.
struct TabPlan;
struct Tiling {
  int bn = 0;
  bool swap = false;  // swap-AB: bn = activation-row tile width, A slot = 128-row weight tiles
  const TabPlan* tab = nullptr;  // CTA-pair swap-AB with a planned unit table (gemm_pair_kernel)
  int t_dp = 0;
  long long W = 0;  // stream-K k-blocks (0: pure data-parallel)
  int grid = 0;
};

template <int EPI, int BN>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, void* C, int64_t ldc, int M, int N, int K,
              const Tiling& tl, cudaStream_t st) {
  if (int rc = ensure_smem(gemm_tc_kernel<EPI, BN, false>, TcCfg<BN>::SMEM)) return rc;
  if (int rc = ensure_smem(gemm_tc_kernel<EPI, BN, true>, TcCfg<BN>::SMEM)) return rc;
  const int tiles = ((M + TC_BM - 1) / TC_BM) * n_tiles_of(N, BN);
  SplitScratch& sc = scratch(st);
  if (tl.W > 0) {
    if (sc.flag_elems < tl.grid) {
      if (sc.flags) cudaFree(sc.flags);
      sc.flag_elems = 1024;
      if (cudaMalloc(&sc.flags, sizeof(int) * sc.flag_elems) != cudaSuccess) return fail(CC_E_CUDA, "gemm_tc: flags");
      cudaMemset(sc.flags, 0xff, sizeof(int) * sc.flag_elems);
    }
    const size_t need = (size_t)tl.grid * TC_BM * BN;  // one partial slot per CTA
    if (sc.ws_elems < need) {
      if (sc.ws) cudaFree(sc.ws);
      sc.ws_elems = need;
      if (cudaMalloc(&sc.ws, sizeof(float) * need) != cudaSuccess) return fail(CC_E_CUDA, "gemm_tc: workspace");
    }
    sc.epoch = (sc.epoch + 1) & 0x3fffffff;
    return launch_k(gemm_tc_kernel<EPI, BN, true>, dim3(tl.grid), dim3(TC_THREADS), TcCfg<BN>::SMEM, st, "gemm_tc",
                    ma, mb, C, ldc, M, N, K, tl.t_dp, tl.W, sc.ws, sc.flags, sc.epoch, g_trace, PeerTab{});
  }
  return launch_k(gemm_tc_kernel<EPI, BN, false>, dim3(tl.grid), dim3(TC_THREADS), TcCfg<BN>::SMEM, st, "gemm_tc", ma,
                  mb, C, ldc, M, N, K, tiles, 0LL, (float*)nullptr, (int*)nullptr, 0, g_trace, PeerTab{});
}

// tile widths: any multiple of 32 <= 256 (ragged last N tile); a width that
// makes the tile count fit the SM count removes most of the wave
// quantisation of M ~ 800 GEMMs (N = 4096: 7 x 19 tiles of 224 = one wave)
constexpr int kBnCand[5] = {256, 224, 192, 160, 128};
// swap-AB launch: the kernel sees M' = N (output features, A slot) and
// N' = M (activation rows, B slot); C stays row-major [M][ldc]
template <int EPI, int BNR>
int launch_swap(const CUtensorMap& mw, const CUtensorMap& mx, void* C, int64_t ldc, int M, int N, int K,
                const Tiling& tl, cudaStream_t st) {
  if (int rc = ensure_smem(gemm_tc_kernel<EPI, BNR, false, true>, TcCfg<BNR>::SMEM)) return rc;
  const int tiles = ((N + TC_BM - 1) / TC_BM) * n_tiles_of(M, BNR);
  return launch_k(gemm_tc_kernel<EPI, BNR, false, true>, dim3(tl.grid), dim3(TC_THREADS), TcCfg<BNR>::SMEM, st,
                  "gemm_tc_swap", mw, mx, C, ldc, N, M, K, tiles, 0LL, (float*)nullptr, (int*)nullptr, 0, g_trace,
                  PeerTab{});
}

// relative time of one k-block of a 128xBN tile (measured efficiency per width)
inline double kb_cost(int bn) {
  const double eff = bn >= 256 ? 1.0 : bn >= 224 ? 0.985 : bn >= 208 ? 0.98 : bn >= 192 ? 0.97 : bn >= 176 ? 0.95
                   : bn >= 160 ? 0.93 : bn >= 144 ? 0.91 : 0.88;
  return bn / 256.0 / eff;
}
// swap-AB activation-row tile widths (MMA N, multiples of 16)
constexpr int kSwapCand[6] = {256, 224, 208, 176, 144, 128};

// exposed cost of a CTA's final stream-K fold (read the partials, in 128x256 k-blocks)
constexpr double kFoldCost = 4.0;

Tiling plan_dp(int M, int N, int bn) {
  Tiling t;
  const int tiles = ((M + TC_BM - 1) / TC_BM) * n_tiles_of(N, bn);
  t.bn = bn;
  t.t_dp = tiles;
  t.grid = tiles < num_sms() ? tiles : num_sms();
  return t;
}

// hybrid: whole waves data-parallel, the last [G, 2G) tiles (or all, when
// fewer) stream-K; >= 4 k-blocks per CTA and <= ~3 fragments per tile (the
// final fragment folds the others' slots one after another)
Tiling plan_sk(int M, int N, int K, int bn) {
  Tiling t;
  const int sms = num_sms(), nkb = K / TC_BK;
  const int tiles = ((M + TC_BM - 1) / TC_BM) * n_tiles_of(N, bn);
  const int full = tiles / sms;
  t.bn = bn;
  t.t_dp = full >= 2 ? (full - 1) * sms : 0;
  t.W = (long long)(tiles - t.t_dp) * nkb;
  long long g = t.W / 4;
  if (g > 3LL * (tiles - t.t_dp)) g = 3LL * (tiles - t.t_dp);
  t.grid = (int)(g < sms ? (g > 0 ? g : 1) : sms);
  if (t.t_dp > 0) t.grid = sms;  // (the stream-K part then has >= sms tiles)
  return t;
}

Tiling plan_swap(int M, int N, int bnr) {
  Tiling t;
  const int tiles = ((N + TC_BM - 1) / TC_BM) * n_tiles_of(M, bnr);
  t.bn = bnr;
  t.swap = true;
  t.t_dp = tiles;
  t.grid = tiles < num_sms() ? tiles : num_sms();
  return t;
}

double model_time(const Tiling& t, int M, int N, int K) {
  const int nkb = K / TC_BK;
  const double kc = kb_cost(t.bn);
  if (t.swap) {
    const int tiles = ((N + TC_BM - 1) / TC_BM) * n_tiles_of(M, t.bn);
    return (double)((tiles + t.grid - 1) / t.grid) * nkb * kc;
  }
  const int tiles = ((M + TC_BM - 1) / TC_BM) * n_tiles_of(N, t.bn);
  if (t.W == 0) return (double)((tiles + t.grid - 1) / t.grid) * nkb * kc;
  const double per = (double)((t.W + t.grid - 1) / t.grid);
  const bool splits = (t.W / t.grid) % nkb != 0 || t.W / t.grid < nkb;
  return ((double)(t.t_dp / t.grid) * nkb + per) * kc + (splits ? kFoldCost * t.bn / 256.0 : 0.0);
}

// ---- unit-table plans (gemm_pair_kernel) -----------------------------------
// Time model in SM cycles per k-block (64-deep slice).  A 1-CTA 128 x 256
// tile streams 48 KiB into shared memory and the MMA reads 48 KiB back: at
// the ~128 B/clk shared-memory port that is 768 cycles (matches the measured
// ~430 ns per k-block; the kb_cost() plans above are converted at that
// rate).  A pair unit of n rows: max(MMA 2n, operand feed 256 + n) per SM,
// times the measured kPairFactor.
constexpr double kKbCycles = 768.0;
constexpr double kUnitOverhead = 2000.0;  // accumulator hand-off, pipeline turn (cycles)
// measured: a pair k-block runs ~1.25x the ideal (the MMA's operand reads and
// the TMA writes share the port); calibrated on the M = 802 / 2048 projection
// shapes against the 1-CTA plans
constexpr double kPairFactor = 1.25;

struct TabPlan {
  SwTab tab;
  int grid = 0;     // CTAs (2 per unit list)
  double t = 1e30;  // modelled makespan, cycles
  int slices = 1;   // K split (1: none)
};
// K-split cost per unit on top of its k-blocks: park the n x 128 fp32 partial,
// the ticket round trip, and (amortised over the slices) the last CTA's reads
// of the other slices' partials, in cycles per row
constexpr double kSplitFixed = 2500.0, kSplitPerRow = 12.0;
// K splits considered for short activation matrices only (few units per pair)
constexpr int kSplitMaxM = 384;  // (at M = 552 the split down_proj measured slower: 10.98 vs 10.72 ms per step)
constexpr int kSplitCand[5] = {1, 2, 3, 4, 6};

inline double unit_cycles(int n, int nkb) {
  const double mma = 2.0 * n, feed = 256.0 + n;
  return ((mma > feed ? mma : feed) * nkb + kUnitOverhead) * kPairFactor;
}

// Cut each 256-feature weight tile's M rows into k chunks (j chunks of 256
// rows, the rest split evenly, 32-row granules), k from ceil(M/256) to +3,
// schedule the units onto the CTA pairs, keep the smallest makespan.  Cached
// per shape (evicted plans are leaked, not freed: a caller may still hold one).
const TabPlan* plan_units(int M, int F, int K, bool ksplit, int force_s = 0) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, TabPlan*> cache;
  const uint64_t key = ((uint64_t)M << 44) ^ ((uint64_t)F << 20) ^ (uint64_t)K ^ (ksplit ? 1ull << 63 : 0ull) ^ ((uint64_t)force_s << 58);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  constexpr int gran = 32, maxb = 256 / gran;
  const int ntile = F / (2 * TC_BM), nkb = K / TC_BK;
  int G = num_sms() / 2;
  if (G > SW_MAXG) G = SW_MAXG;
  const int nb = (M + gran - 1) / gran, kmin = (nb + maxb - 1) / maxb;
  TabPlan* best = new TabPlan();
  struct U {
    double cost;
    int ft, r0, n, ks;
  };
  std::vector<U> units;
  std::vector<std::vector<int>> lists(G);
  std::vector<int> best_ch;
  const int Mpad = nb * gran;
  for (int S : kSplitCand)
  for (int k = kmin; k <= kmin + 3 && (long)ntile * k * S <= SW_MAXU; ++k) {
    if (force_s > 0 ? S != force_s : S > 1 && (!ksplit || M > kSplitMaxM)) break;
    if (S > 1 && (nkb / S < 8 || (double)S * F * Mpad * 4.0 > 256.0 * (1 << 20))) break;
    for (int j = 0; j < k; ++j) {
      const int rem = nb - maxb * j, parts = k - j;
      if (rem < parts) break;
      if ((rem + parts - 1) / parts > maxb) continue;
      std::vector<int> ch(j, maxb);
      for (int i = 0; i < parts; ++i) ch.push_back(rem / parts + (i < rem % parts ? 1 : 0));
      units.clear();
      for (int ft = 0; ft < ntile; ++ft)
        for (int ci = 0, r0 = 0; ci < (int)ch.size(); r0 += ch[ci] * gran, ++ci)
          for (int sl = 0; sl < S; ++sl) {
            const int n = ch[ci] * gran, kbs = (sl + 1) * nkb / S - sl * nkb / S;
            const double c = unit_cycles(n, kbs) + (S > 1 ? kSplitFixed + kSplitPerRow * n : 0.0);
            units.push_back({c, ft, r0, n, S > 1 ? (sl << 4) | (S - 1) : 0});
          }
      // Units of one weight tile should run side by side (one HBM read of the
      // weights, the rest from L2): list-schedule them in (tile, chunk) order
      // onto the earliest-free CTA, except the last ~1.5 rounds of work, which
      // go longest-first (LPT) to even out the finish.
      double total = 0, maxc = 0;
      for (auto& x : units) { total += x.cost; maxc = maxc > x.cost ? maxc : x.cost; }
      size_t split = 0;
      for (double pre = 0; split < units.size() && pre + units[split].cost <= total - 1.5 * G * maxc; ++split)
        pre += units[split].cost;
      std::stable_sort(units.begin() + split, units.end(), [](const U& a, const U& b) { return a.cost > b.cost; });
      std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>, std::greater<>> heap;
      for (int c = 0; c < G; ++c) heap.push({0.0, c});
      for (auto& l : lists) l.clear();
      double makespan = 0;
      for (int i = 0; i < (int)units.size(); ++i) {
        auto [load, c] = heap.top();
        heap.pop();
        load += units[i].cost;
        if (load > makespan) makespan = load;
        lists[c].push_back(i);
        heap.push({load, c});
      }
      if (makespan < best->t - 1e-9) {
        best->t = makespan;
        best->slices = S;
        best_ch = ch;
        int nl = 0, pos = 0;
        for (int c = 0; c < G; ++c) {
          if (lists[c].empty()) continue;
          best->tab.start[nl++] = (uint16_t)pos;
          for (int i : lists[c]) {
            best->tab.ks[pos] = (uint8_t)units[i].ks;
            best->tab.unit[pos++] = sw_pack(units[i].ft, units[i].r0, units[i].n);
          }
        }
        best->tab.start[nl] = (uint16_t)pos;
        best->grid = 2 * nl;
      }
    }
  }
  if (getenv("CCB_SW_DEBUG")) {
    fprintf(stderr, "[gemm_pair] M=%d F=%d K=%d makespan=%.0f cyc (%.2f x 768-cycle tiles) grid=%d slices=%d chunks(x%d):",
            M, F, K, best->t, best->t / (kKbCycles * nkb), best->grid, best->slices, gran);
    for (int c : best_ch) fprintf(stderr, " %d", c);
    fprintf(stderr, "\n");
  }
  if (best->grid == 0) {
    delete best;
    best = nullptr;
  }
  if (cache.size() > 1024) cache.clear();  // (plans of evicted shapes leak: bounded, rare)
  cache.emplace(key, best);
  return best;
}

// CCB_PAIR_KSPLIT=0 keeps the planner off K-split unit plans (A/B).  The
// config-2 step replayed from a CUDA graph (tools/graph_step.py, ms, split
// vs unsplit): r = 0 (32 rows) 5.96 vs 6.38, r = 0.05 (292 rows) 8.21 vs
// 8.56; at r = 0.10 (552 rows) the split down_proj was slower (10.98 vs
// 10.72), hence kSplitMaxM.
inline bool ksplit_enabled() {
  static const bool on = [] {
    const char* e = getenv("CCB_PAIR_KSPLIT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// workspace + tickets of a K-split plan, per (device, stream)
int ksplit_buffers(const TabPlan* tp, int M, int F, cudaStream_t st, KSplit* out) {
  if (tp->slices <= 1) return 0;
  const int Mpad = (M + 31) / 32 * 32;
  out->Mpad = Mpad;
  out->F = F;
  out->ws = reinterpret_cast<float*>(stream_scratch(st, SCR_PAIR_KSPLIT, (size_t)tp->slices * F * Mpad * sizeof(float)));
  out->ticket = reinterpret_cast<unsigned*>(
      zeroed_scratch(st, ZSCR_PAIR_TICKETS, (size_t)(F / TC_BM) * (Mpad / 32) * sizeof(unsigned)));
  if (!out->ws || !out->ticket) return fail(CC_E_CUDA, "gemm_pair: K-split workspace allocation failed");
  return 0;
}

// CCB_GEMM_PAIR=0 disables the CTA-pair plans (A/B measurements)
inline bool pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("CCB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the tiling minimising the modelled time.  Stream-K is considered where it
// measured faster: small M (fewer than half a wave of tiles: weight
// streaming) and long K with several waves (M ~ 5k down_proj).  At M ~ 800
// the data-parallel schedule wins: stream-K's scattered k offsets defeat the
// L2 sharing of the weight tiles across a wave's M tiles.
Tiling pick_tiling(int M, int N, int K, int epi, bool allow_split) {
  const int sms = num_sms(), nkb = K / TC_BK;
  Tiling best;
  double best_t = 1e30;
  for (int i = 0; i < 5; ++i) {
    const int bn = kBnCand[i];
    if (epi == CC_EPI_SWIGLU && (bn != 256 || N % 256)) continue;  // gate|up 64-column groups pair up per tile
    Tiling dp = plan_dp(M, N, bn);
    double t = model_time(dp, M, N, K);
    if (t < best_t - 1e-9) { best_t = t; best = dp; }
    const int tiles = dp.t_dp;
    // stream-K: weight-streaming shapes (under half a wave of tiles) only
    // below 128 rows -- at M = 290 it measured 44.0 / 38.4 / 70.6 us for
    // QKV / o_proj / down against the CTA-pair plans' 26.6 / 26.5 / 67.9
    // (tools/smallm_force.sh) -- and long-K multi-wave shapes
    if (allow_split && ((2 * tiles <= sms && M < 128) || (tiles >= 2 * sms && nkb >= 128))) {
      Tiling sk = plan_sk(M, N, K, bn);
      double ts = model_time(sk, M, N, K);
      if (ts < 0.97 * best_t) { best_t = ts; best = sk; }
    }
  }
  // swap-AB for short activation matrices: rows become the MMA N dimension,
  // so the padding of M ~ 800 and the wave count can both be fitted.  Used for
  // the residual (f32) epilogue, where a warp store is a full 128-byte row
  // segment; the bf16 outputs (QKV, SwiGLU) measured faster unswapped
  // (o_proj 29.7 -> 27.4 us, down 92 -> 86.7 us; QKV 38.9 vs 40.4 swapped)
  if (epi == CC_EPI_RESID_ADD && M <= 2048 && N % TC_BM == 0) {
    for (int i = 0; i < 6; ++i) {
      Tiling sw = plan_swap(M, N, kSwapCand[i]);
      double ts = model_time(sw, M, N, K);
      if (ts < 0.98 * best_t) { best_t = ts; best = sw; }
    }
  }
  // CTA-pair unit table (any epilogue; SwiGLU: [gate 64 | up 64] per 128 rows)
  if (M >= (allow_split && ksplit_enabled() ? 32 : 64) && M <= 8192 && N % (2 * TC_BM) == 0 && pair_enabled()) {
    const TabPlan* tp = plan_units(M, N, K, allow_split && ksplit_enabled());
    // below 64 rows the 1-CTA stream-K tiles measured far slower than their
    // model (r = 0 step: o_proj 29 us for 33.5 MB, QKV 29 us for 50 MB, i.e.
    // 1.2-1.8 TB/s) while the K-split pair units stream at 3.7 TB/s (down):
    // take the pair plan there whenever one exists
    if (tp && ((M < 64 && tp->slices > 1) || tp->t < 0.97 * best_t * kKbCycles)) {
      best = Tiling{};
      best.bn = 256;
      best.tab = tp;
      best.grid = tp->grid;
    }
  }
  return best;
}

// CCB_GEMM_FORCE="bn,mode" pins the tiling (experiments / tests): mode 0
// data-parallel, 1 stream-K hybrid
bool forced_tiling(int M, int N, int K, int epi, Tiling* out) {
  static int fb = -1, fs = -1;
  static bool init = false;
  if (!init) {
    init = true;
    if (const char* e = getenv("CCB_GEMM_FORCE")) sscanf(e, "%d,%d", &fb, &fs);
  }
  if (fs == 4 || fs == 5) {  // CTA-pair unit table (5: with fb K slices)
    const TabPlan* tp = M <= 8192 && N % (2 * TC_BM) == 0 ? plan_units(M, N, K, false, fs == 5 ? fb : 0) : nullptr;
    if (!tp) return false;
    *out = Tiling{};
    out->bn = 256;
    out->tab = tp;
    out->grid = tp->grid;
    return true;
  }
  if (fs == 2) {  // swap-AB with row tile fb
    if (fb <= 0 || fb % 16 || fb > 256 || N % TC_BM || epi == CC_EPI_SWIGLU) return false;
    *out = plan_swap(M, N, fb);
    return true;
  }
  if (fb <= 0 || fb % 32 || fb > 256 || (epi == CC_EPI_SWIGLU && fb != 256)) return false;
  *out = fs == 1 ? plan_sk(M, N, K, fb) : plan_dp(M, N, fb);
  return true;
}

template <int EPI>
int launch_epi(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
               bool allow_split, cudaStream_t st) {
  Tiling tl;
  if (!forced_tiling(M, N, K, EPI, &tl)) tl = pick_tiling(M, N, K, EPI, allow_split && g_stream_k);
  if (tl.bn == 0) return fail(CC_E_UNSUP, "gemm_tc: N must be a multiple of 128 (SwiGLU: 256)");
  if (tl.tab) {
    CUtensorMap mw, mx[4];
    int rc = make_map(&mw, B, N, K, ldb, TC_BM);
    for (int i = 0; i < 4 && !rc; ++i) rc = make_map(&mx[i], A, M, K, lda, 128 >> i);
    if (rc) return rc;
    CUtensorMap mc;  // output: [M][N] (SwiGLU [M][N/2]) with leading dim ldc
    rc = make_map(&mc, C, M, EPI == CC_EPI_SWIGLU ? N / 2 : N, ldc,
                  EPI == CC_EPI_RESID_ADD ? -2 : EPI == CC_EPI_SWIGLU ? -3 : -1);
    if (rc) return rc;
    if (int rc2 = ensure_smem(gemm_pair_kernel<EPI>, P2_SMEM)) return rc2;
    KSplit ksp{};
    if (int rc2 = ksplit_buffers(tl.tab, M, N, st, &ksp)) return rc2;
    static const int dbg = getenv("CCB_PAIR_DBG") ? atoi(getenv("CCB_PAIR_DBG")) : 0;
    return launch_k(gemm_pair_kernel<EPI>, dim3(tl.grid), dim3(TC_THREADS), P2_SMEM, st, "gemm_pair", mw, mx[0], mx[1],
                    mx[2], mx[3], mc, M, K, dbg, tl.tab->tab, RopeQkv{}, ksp);
  }
  if constexpr (EPI != CC_EPI_SWIGLU) if (tl.swap) {
    // A slot <- weights B [N][K] (128-row boxes), B slot <- activations A [M][K]
    CUtensorMap mw, mx;
    int rc = make_map(&mw, B, N, K, ldb, TC_BM);
    if (rc) return rc;
    rc = make_map(&mx, A, M, K, lda, tl.bn);
    if (rc) return rc;
    switch (tl.bn) {
      case 256: return launch_swap<EPI, 256>(mw, mx, C, ldc, M, N, K, tl, st);
      case 224: return launch_swap<EPI, 224>(mw, mx, C, ldc, M, N, K, tl, st);
      case 208: return launch_swap<EPI, 208>(mw, mx, C, ldc, M, N, K, tl, st);
      case 176: return launch_swap<EPI, 176>(mw, mx, C, ldc, M, N, K, tl, st);
      case 144: return launch_swap<EPI, 144>(mw, mx, C, ldc, M, N, K, tl, st);
      case 128: return launch_swap<EPI, 128>(mw, mx, C, ldc, M, N, K, tl, st);
      default: return fail(CC_E_UNSUP, "gemm_tc: unsupported swap tile width");
    }
  }
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, TC_BM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, tl.bn);
  if (rc) return rc;
  switch (tl.bn) {
    case 256: return launch_tc<EPI, 256>(ma, mb, C, ldc, M, N, K, tl, st);
    case 224: return launch_tc<EPI, 224>(ma, mb, C, ldc, M, N, K, tl, st);
    case 192: return launch_tc<EPI, 192>(ma, mb, C, ldc, M, N, K, tl, st);
    case 160: return launch_tc<EPI, 160>(ma, mb, C, ldc, M, N, K, tl, st);
    case 128: return launch_tc<EPI, 128>(ma, mb, C, ldc, M, N, K, tl, st);
    default: return fail(CC_E_UNSUP, "gemm_tc: unsupported tile width");
  }
}

}  // namespace

void gemm_tc_set_trace(void* p) { g_trace = reinterpret_cast<long long*>(p); }

// QKV projection + RoPE + K/V scatter in one CTA-pair GEMM (see RopeQkv).
// CC_E_UNSUP for shapes the fused epilogue does not cover (d_head != 128,
// N not a multiple of 256, M > 8192): the caller then runs the GEMM and
// rope_scatter separately.
int gemm_qkv_rope_bf16(const void* X, int64_t ldx, const void* Wqkv, int64_t ldw, int M, int K, int Hq, int Hkv,
                       int d_head, const int32_t* row_slot, const int32_t* row_pos, const void* table, void* q_rot,
                       void* kv_k, void* kv_v, void* k_rot, cudaStream_t st) {
  const int N = (Hq + 2 * Hkv) * d_head;
  // The epilogue re-reads a row's cos/sin once per head (40x the table
  // traffic of rope_scatter at Llama-3-8B widths) and the last unit's
  // epilogue is exposed: measured (qkv_rope_ab.py, us, fused vs GEMM +
  // rope_scatter) M = 290: 37.4 vs 51.7, 802: 57.8 vs 48.4, 1570: 86.6 vs
  // 74.3, 5152: 208 vs 198 -- so the fused kernel runs for short activation
  // matrices only (M <= CCB_QKV_FUSE_MAX, default 512).
  static const int fuse_max = getenv("CCB_QKV_FUSE_MAX") ? atoi(getenv("CCB_QKV_FUSE_MAX")) : 512;
  if (d_head != 128 || N % (2 * TC_BM) || M < 64 || M > fuse_max || M > 8192 || K % TC_BK || ldx % 8 || ldw % 8 ||
      !pair_enabled())
    return fail(CC_E_UNSUP, "gemm_qkv_rope: shape not covered by the fused epilogue");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Wqkv)) & 15)
    return fail(CC_E_UNSUP, "gemm_qkv_rope: pointers must be 16-byte aligned");
  const TabPlan* tp = plan_units(M, N, K, false);  // (no K split: the same bits as impl 4 + rope_scatter)
  if (!tp) return fail(CC_E_UNSUP, "gemm_qkv_rope: no unit plan");
  KSplit ksp{};
  if (int rc = ksplit_buffers(tp, M, N, st, &ksp)) return rc;
  CUtensorMap mw, mx[4];
  int rc = make_map(&mw, Wqkv, N, K, ldw, TC_BM);
  for (int i = 0; i < 4 && !rc; ++i) rc = make_map(&mx[i], X, M, K, ldx, 128 >> i);
  if (rc) return rc;
  CUtensorMap mq;  // q_rot [M][Hq * 128] bf16, 32 x 32 store boxes
  rc = make_map(&mq, q_rot, M, (int64_t)Hq * 128, (int64_t)Hq * 128, -1);
  if (rc) return rc;
  if (int rc2 = ensure_smem(gemm_pair_kernel<EPI_ROPE_QKV>, P2_SMEM)) return rc2;
  RopeQkv rq{row_slot, row_pos, reinterpret_cast<const float2*>(table), (__nv_bfloat16*)q_rot, (__nv_bfloat16*)kv_k,
             (__nv_bfloat16*)kv_v, (__nv_bfloat16*)k_rot, Hq, Hkv};
  static const int dbg = getenv("CCB_PAIR_DBG") ? atoi(getenv("CCB_PAIR_DBG")) : 0;
  return launch_k(gemm_pair_kernel<EPI_ROPE_QKV>, dim3(tp->grid), dim3(TC_THREADS), P2_SMEM, st, "gemm_qkv_rope", mw,
                  mx[0], mx[1], mx[2], mx[3], mq, M, K, dbg, tp->tab, rq, ksp);
}

// o_proj / down_proj of a tensor-parallel rank with the reduce-scatter fused
// into the epilogue (data-parallel schedule; BN must divide the owner slice)
int gemm_tc_peer_push(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                      const PeerTab& tab, cudaStream_t st) {
  if (N % 128 != 0 || K % TC_BK != 0 || lda % 8 != 0 || ldb % 8 != 0 || tab.slice % 128 != 0 || N != tab.slice * tab.world)
    return fail(CC_E_UNSUP, "gemm_tc_peer_push: needs N = slice * world, slice % 128 == 0, K % 64 == 0");
  const int bn = tab.slice % 256 == 0 ? 256 : 128;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, TC_BM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, bn);
  if (rc) return rc;
  Tiling tl = plan_dp(M, N, bn);
  auto go = [&](auto kern, size_t smem) {
    if (int rc = ensure_smem(kern, smem)) return rc;
    kern<<<tl.grid, TC_THREADS, smem, st>>>(ma, mb, nullptr, 0, M, N, K, tl.t_dp, 0LL, nullptr, nullptr, 0, g_trace,
                                            tab);
    return check_launch("gemm_tc_peer_push");
  };
  if (bn == 256) return go(gemm_tc_kernel<CC_EPI_PEER_PUSH, 256, false>, TcCfg<256>::SMEM);
  return go(gemm_tc_kernel<CC_EPI_PEER_PUSH, 128, false>, TcCfg<128>::SMEM);
}

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

// debug hook (not part of the ABI): per-CTA epilogue timeline of the next GEMMs
extern "C" __attribute__((visibility("default"))) void cc_debug_gemm_trace(void* p) { ccb::gemm_tc_set_trace(p); }
