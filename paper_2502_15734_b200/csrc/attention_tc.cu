// K4 on the 5th-generation tensor cores: flash-style attention of the
// recomputed (scattered) query rows over all request keys (model.py:406-416)
// with S and O accumulators in TMEM.
//
// CTA = 128 "M-rows" = R query rows x G heads of one GQA group (G = Hq/Hkv,
// R = 128/G), so one K/V tile in shared memory serves the whole group.
//   warp 0     TMA: Q once (3-D map), K tiles of BN keys (ring, one tile
//              ahead of V), V tiles (2 slots tied to the P buffers)
//   warp 1     MMA issuer: S_i = Q K_i^T (M128 N128 K16 x dh/16) into one of
//              two TMEM S buffers, O += P_i V_i (A = P from TMEM, B = V
//              MN-major from smem) into the TMEM O accumulator; two commits
//              per tile (s_full, p_empty)
//   warps 2-9  two softmax warpgroups: thread = (M-row, key half).  Reads
//              its 64 S columns (tcgen05.ld), causal+pad mask (key j visible
//              iff j <= q_slot[row] and !pad[j]), row-max exchange with the
//              other half through smem, online softmax in fp32 (exp2, a
//              quarter on the FMA pipe), lazy O rescale in TMEM, P packed to
//              bf16 and stored to TMEM (tcgen05.st) for the PV MMA.
// The PV MMA of tile i overlaps the S MMA of tile i+1 and the softmax of
// tile i+1 (double-buffered S and P).
#include <math.h>
#include <stdio.h>
#include <algorithm>
#include <cmath>
#include <stdlib.h>

#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "f32x2.cuh"

namespace ccb {

namespace {

using namespace sm100;

constexpr int AT_BN = 128;      // keys per tile
// P (softmax output, bf16) lives in TMEM and feeds the PV MMA as its A
// operand (tcgen05.mma ... [a-tmem]): no smem P buffers, 64 KiB less smem
// traffic per tile, room for a third K stage.
constexpr int AT_KST = 3;  // K ring depth
constexpr int AT_VST = 2;  // V ring depth = P buffers: V slot i % 2 is released by PV_i's p_empty commit
constexpr int AT_THREADS = 320;  // TMA warp, MMA warp, 2 x 4 softmax warps
constexpr int AT_MAXT = 512;     // row tiles the in-kernel work plan handles (more: no key splits)
constexpr int AT_MAXP = 4;       // key-range parts per row tile, merged by the last part (8 measured slower at r = 0)
constexpr int AT_MAXP_EXT = 16;  // key parts with the separate merge kernel (ping-pong kernel, few items)
constexpr int kExtMaxItems = 16; // (group, block) items up to which the ping-pong kernel uses it

// MN-major operand (B = V: N = head dim contiguous, K = keys), 128B swizzle:
// 64-element atoms along N at `lbo` bytes, 8-key groups at 1024 B.
__device__ __forceinline__ uint64_t desc_sw128_mn(const void* smem_tile, uint32_t lbo_bytes) {
  uint64_t addr = smem_u32(smem_tile);
  return ((addr >> 4) & 0x3FFFull) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (x <= 0): round-to-nearest split x = n + f,
// f in [-1/2, 1/2], cubic Taylor for 2^f (rel. error < 5e-4, below the bf16
// rounding of P), n added to the exponent; x < -125 (masked) gives 0
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -125.f);
  const float t = xc + 12582912.f;  // 1.5 * 2^23: rounds xc to an integer in the low mantissa bits
  const float n = t - 12582912.f;
  const float f = xc - n;
  float p = fmaf(f, fmaf(f, fmaf(f, 0.05550410866f, 0.2402265070f), 0.6931471806f), 1.f);
  const int e = __float_as_int(t) << 23;  // n in the exponent field (two's complement wraps correctly)
  p = __int_as_float(__float_as_int(p) + e);
  return x < -125.f ? 0.f : p;
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mbarrier wait that adds its stall cycles to acc when tracing (debug)
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t parity, bool tracing, long long& acc) {
  if (tracing) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}

// Kernel shape: DH head dim, BN keys per tile, NWG softmax warpgroups (a
// softmax thread owns one M-row and BN / NWG keys of it).  P (bf16) is
// written over the first BN/2 columns of its own S buffer once S has been
// read (both key halves have, at the pair barrier), so TMEM holds
// S0/P0 | S1/P1 | O: 2 BN + DH columns.  BN = 64 with DH = 128 needs 256
// columns and ~106 KiB of shared memory: two CTAs share an SM, and each
// CTA's MMAs fill the other's softmax gaps on the tensor pipe.
template <int DH, int BN, int NWG, int KST_ = (BN == 64 ? 2 : 3), int VST_ = 2>
struct At {
  static constexpr int KST = KST_;  // K ring depth
  static constexpr int VST = VST_;  // V ring depth (>= 2: slot i % VST also names P buffer i % 2's release)
  static constexpr int THREADS = 64 + 128 * NWG;
  static constexpr int KPT = BN / NWG;           // keys per softmax thread
  static constexpr int OPT = DH / NWG;           // O columns per softmax thread
  static constexpr int TMEM_USED = 2 * BN + DH;
  static constexpr int TMEM_COLS = TMEM_USED <= 256 ? 256 : 512;
  static constexpr int ATOMS = DH / 64;              // 64-element (128 B) column atoms
  static constexpr int Q_BYTES = 128 * DH * 2;       // 128 M-rows
  static constexpr int KV_BYTES = BN * DH * 2;       // one K (or V) tile
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + Q_BYTES;
  static constexpr int V_OFF = K_OFF + KST * KV_BYTES;
  static constexpr int BAR_OFF = V_OFF + VST * KV_BYTES;
  static constexpr int X_OFF = BAR_OFF + 512;        // [2 parities][NWG][128 rows] f32 exchange
  static constexpr int PLAN_OFF = X_OFF + 2 * NWG * 128 * 4;  // work-item plan: [3][AT_MAXT] ints
  // no alignment slack: the kernel holds no static shared memory, so the
  // dynamic window starts 1 KiB aligned (checked at run time)
  static constexpr size_t TOTAL = PLAN_OFF + 3 * AT_MAXT * 4;
  static constexpr int CTAS_PER_SM = (TMEM_COLS <= 256 && 2 * (TOTAL + 1024) <= 232448) ? 2 : 1;
  static_assert(KPT % 32 == 0, "a softmax thread reads whole 32-column TMEM chunks");
};

template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tmem_st_cols<32>(uint32_t taddr, const uint32_t* r) {
  tmem_st32(taddr, *reinterpret_cast<const uint32_t(*)[32]>(r));
}
template <>
__device__ __forceinline__ void tmem_st_cols<16>(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
template <>
__device__ __forceinline__ void tmem_st_cols<64>(uint32_t taddr, const uint32_t* r) {
  tmem_st_cols<32>(taddr, r);
  tmem_st_cols<32>(taddr + 32, r + 32);
}

template <int DH, int BN, int NWG, int KST_, int VST_>
__global__ void __launch_bounds__(At<DH, BN, NWG, KST_, VST_>::THREADS, At<DH, BN, NWG, KST_, VST_>::CTAS_PER_SM)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const int32_t* __restrict__ q_slot,
                   const uint8_t* __restrict__ key_pad, __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse,
                   int n_q, int n_keys, int Hq, int G, float scale_log2, long long* __restrict__ trace,
                   int n_groups, int n_row_tiles, int target, int max_parts, float* __restrict__ ws_o,
                   float2* __restrict__ ws_ml, int* __restrict__ counters, int exp) {
  using SM = At<DH, BN, NWG, KST_, VST_>;
  constexpr int KST = SM::KST, VST = SM::VST, KPT = SM::KPT, OPT = SM::OPT, NT = SM::THREADS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw;
  if (smem_u32(smem_raw) & 1023) __trap();  // 128B-swizzled TMA / UMMA tiles need 1 KiB alignment
  uint8_t* sQ = base + SM::Q_OFF;
  uint8_t* sK = base + SM::K_OFF;
  uint8_t* sV = base + SM::V_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + SM::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;                 // [KST]
  uint64_t* k_empty = k_full + KST;            // [KST] arrived by the softmax once S_i landed
  uint64_t* v_full = k_empty + KST;            // [VST]
  uint64_t* v_empty = v_full + VST;            // [VST] committed by the MMA thread after PV_i
  uint64_t* s_full = v_empty + VST;            // [2]
  uint64_t* s_empty = s_full + 2;              // [2]
  uint64_t* p_full = s_empty + 2;              // [2]
  uint64_t* p_empty = p_full + 2;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_empty + 2);
  int& s_kmax = *reinterpret_cast<int*>(tmem_slot + 1);
  uint32_t* padw = tmem_slot + 2;                                  // [2 parities][4 words]
  float* xmax = reinterpret_cast<float*>(base + SM::X_OFF);       // row maxima / sums of the key halves

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = 128 / G;
  const int T = n_row_tiles;
  // ---- work item of this CTA ------------------------------------------------
  // An item = (kv group, row tile, part of the row tile's key range).  Row
  // tile t's causal key range is estimated from its last row (rows are in
  // slot order in the engine) and cut into ceil(len / target) parts; items
  // are ordered longest first (LPT), so blockIdx x walks that list and the
  // longest work is dispatched in the first wave.  CTAs past the last item
  // exit.  Every CTA derives the same plan (deterministic); the exact key
  // range of the tile is still taken over all its rows below.
  int* s_item = reinterpret_cast<int*>(tmem_slot + 10);  // group, tile, part, parts, est
  pdl_trigger();
  pdl_wait();  // (q_slot and, below, q/k/v: written before this kernel)
  if (max_parts > 1) {
    int* p_len = reinterpret_cast<int*>(base + SM::PLAN_OFF);
    int* p_parts = p_len + AT_MAXT;
    int* p_order = p_parts + AT_MAXT;
    for (int t = threadIdx.x; t < T; t += NT) {
      const int kq = q_slot[min((t + 1) * R, n_q) - 1];
      const int est = kq < 0 ? 0 : min(kq, n_keys - 1) / BN + 1;
      const int parts = max(1, min(max_parts, (est + target - 1) / target));
      p_parts[t] = parts;
      p_len[t] = (est + parts - 1) / parts;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += NT) {
      const int lt = p_len[t];
      int rank = 0;
      for (int u = 0; u < T; ++u) rank += (p_len[u] > lt || (p_len[u] == lt && u > t)) ? 1 : 0;
      p_order[rank] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int idx = blockIdx.x;
      s_item[0] = -1;
      for (int r = 0; r < T; ++r) {
        const int t = p_order[r], c = n_groups * p_parts[t];
        if (idx < c) {
          s_item[0] = idx % n_groups;
          s_item[1] = t;
          s_item[2] = idx / n_groups;
          s_item[3] = p_parts[t];
          s_item[4] = p_len[t] * p_parts[t];
          break;
        }
        idx -= c;
      }
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    // one item per (group, row tile); row tiles last-first (longest first)
    s_item[0] = blockIdx.x % n_groups;
    s_item[1] = T - 1 - (int)blockIdx.x / n_groups;
    s_item[2] = 0;
    s_item[3] = 1;
    s_item[4] = 0;
  }
  if (max_parts <= 1) __syncthreads();
  const int g = s_item[0];
  if (g < 0) return;  // past the last item (before any barrier or TMEM use)
  const int tile = s_item[1], part = s_item[2], parts = s_item[3], est = s_item[4];
  const int row0 = tile * R;

  if (threadIdx.x == 0) s_kmax = -1;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 128 * NWG);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&p_full[b], 128 * NWG);
      mbar_init(&p_empty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<SM::TMEM_COLS>(tmem_slot);
  __syncthreads();
  // per-CTA key range: max causal limit over valid rows
  if (threadIdx.x < 128) {
    int r = row0 + threadIdx.x / G;
    if (r < n_q) atomicMax(&s_kmax, q_slot[r]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kmax = s_kmax;
  const int n_total = kmax < 0 ? 0 : kmax / BN + 1;
  // this part's key tiles [t0, t0 + n_tiles): boundaries from the planned
  // estimate, the last part runs to the exact end (every tile covered once)
  const bool split = parts > 1;
  const int t0 = split ? min(part * est / parts, n_total) : 0;
  const int t1 = !split || part == parts - 1 ? n_total : min((part + 1) * est / parts, n_total);
  const int n_tiles = max(0, t1 - t0);
  // TMEM columns: S0/P0 | S1/P1 | O
  const uint32_t t_s0 = tmem, t_o = tmem + 2 * BN;
  const bool tracing = trace != nullptr;
  long long w0 = 0, w1 = 0, w2 = 0, w3 = 0;  // per-role stall cycles (trace only)
  long long t_s_issue = 0, t_s_commit = 0, t_p_issue = 0, t_p_commit = 0;
  long long t_begin = 0;
  if (trace != nullptr && threadIdx.x == 64) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_begin));

  if (warp == 0) {
    if (lane == 0 && n_tiles > 0) {
      mbar_expect_tx(q_full, SM::Q_BYTES);
#pragma unroll
      for (int a = 0; a < SM::ATOMS; ++a) tma_load_3d(sQ + a * 128 * 128, &tmQ, q_full, a * 64, g * G, row0);
      // K runs one tile ahead of V: K_{i+1}'s slot frees when S_{i-1} is done
      // (early), V_i's when PV_{i-2} is done, so neither S nor PV waits on a
      // load issued after the previous PV
      auto load_k = [&](int i) {
        const int st = i % KST;
        twait(&k_empty[st], ((i / KST) & 1) ^ 1, tracing, w0);
        mbar_expect_tx(&k_full[st], SM::KV_BYTES);
#pragma unroll
        for (int a = 0; a < SM::ATOMS; ++a)
          tma_load_2d(sK + st * SM::KV_BYTES + a * BN * 128, &tmK, &k_full[st], g * DH + a * 64, (t0 + i) * BN);
      };
      load_k(0);
      for (int i = 0; i < n_tiles; ++i) {
        if (i + 1 < n_tiles) load_k(i + 1);
        const int st = i % VST;  // free once PV_{i-VST} completed
        twait(&v_empty[st], ((i / VST) & 1) ^ 1, tracing, w1);
        mbar_expect_tx(&v_full[st], SM::KV_BYTES);
#pragma unroll
        for (int a = 0; a < SM::ATOMS; ++a)
          tma_load_2d(sV + st * SM::KV_BYTES + a * BN * 128, &tmV, &v_full[st], g * DH + a * 64, (t0 + i) * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t id_s = idesc_bf16(128, BN, false);
      constexpr uint32_t id_o = idesc_bf16(128, DH, true);
      mbar_wait(q_full, 0);
      // S_i = Q K_i^T into S buffer i & 1.  It overwrites P_{i-2} (aliased):
      // issued after PV_{i-2} in this thread's program order, and tcgen05
      // MMAs of one CTA execute in issue order
      auto issue_s = [&](int i) {
        const int st = i % KST, b = i & 1;
        twait(&k_full[st], (i / KST) & 1, tracing, w0);
        twait(&s_empty[b], ((i >> 1) & 1) ^ 1, tracing, w1);
        tc_fence_after();
        const long long ts0 = tracing ? clock64() : 0;
        if (exp != 3 && exp != 9) {  // (exp 3, timing experiment: no S MMA)
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const int a = kk >> 2, w = kk & 3;
            uint64_t bd = desc_sw128(sK + st * SM::KV_BYTES + a * BN * 128) + 2 * w;
            uint64_t ad = desc_sw128(sQ + a * 128 * 128) + 2 * w;
            mma_bf16(t_s0 + b * BN, ad, bd, id_s, kk > 0);
          }
        }
        const long long ts1 = tracing ? clock64() : 0;
        mma_commit(&s_full[b]);  // (K slot released by the softmax when it sees s_full)
        if (tracing) { t_s_issue += ts1 - ts0; t_s_commit += clock64() - ts1; }
      };
      issue_s(0);
      for (int i = 0; i < n_tiles; ++i) {
        if (i + 1 < n_tiles) issue_s(i + 1);
        const int st = i % VST, pb = i & 1;
        twait(&p_full[pb], (i >> 1) & 1, tracing, w2);
        twait(&v_full[st], (i / VST) & 1, tracing, w3);
        tc_fence_after();
        const long long tp0 = tracing ? clock64() : 0;
        if (exp == 1) {  // timing experiment: V read as a K-major operand (wrong result)
          constexpr uint32_t id_k = idesc_bf16(128, DH, false);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            uint64_t bd = desc_sw128(sV + st * SM::KV_BYTES + (kk >> 2) * DH * 128) + 2 * (kk & 3);
            mma_bf16_ts(t_o, t_s0 + pb * BN + kk * 8, bd, id_k, (i > 0 || kk > 0) ? 1u : 0u);
          }
        } else if (exp != 2 && exp != 9) {  // (exp 2, timing experiment: no PV MMA)
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            uint64_t bd = desc_sw128_mn(sV + st * SM::KV_BYTES + kk * 16 * 128, BN * 128);
            // A = P in TMEM: row = lane, 2 bf16 keys per 32-bit column, 16 keys = 8 columns
            mma_bf16_ts(t_o, t_s0 + pb * BN + kk * 8, bd, id_o, (i > 0 || kk > 0) ? 1u : 0u);
          }
        }
        const long long tp1 = tracing ? clock64() : 0;
        mma_commit(&p_empty[pb]);       // P buffer pb (and O current through PV_i)
        mma_commit(&v_empty[i % VST]);  // V slot of tile i
        if (tracing) { t_p_issue += tp1 - tp0; t_p_commit += clock64() - tp1; }
      }
    }
  } else {
    // ---- softmax / correction / epilogue --------------------------------------
    // NWG softmax warpgroups: thread = (M-row m, key part h); part h owns S
    // columns [KPT h, KPT (h+1)), P columns [KPT/2 h, ...) and O columns
    // [OPT h, OPT (h+1)).  With two parts the pair exchanges its row max
    // through smem per tile (one named barrier per TMEM lane quarter); the
    // running sums stay per part and are added once at the end.
    const int q4 = warp & 3;               // TMEM lane quarter
    const int h = (warp - 2) >> 2;         // key / output-column part
    const int m = q4 * 32 + lane;
    const int row = row0 + m / G;
    const int head = g * G + m % G;
    const int lim = row < n_q ? q_slot[row] : -1;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    constexpr float kRescaleLog2 = 8.f;  // lazy rescale: keep the stale max while p <= 2^8
    auto pair_bar = [&]() {
      if constexpr (NWG > 1) asm volatile("bar.sync %0, %1;" ::"r"(2 + q4), "r"(32 * NWG) : "memory");
    };
    for (int i = 0; i < n_tiles; ++i) {
      const int b = i & 1;
      twait(&s_full[b], (i >> 1) & 1, tracing, w0);
      tc_fence_after();
      if (warp == 2 && lane == 0) mbar_arrive(&k_empty[i % KST]);  // S_i done: K_i's slot is free
      float s[KPT];
      {
        const uint32_t ta = t_s0 + b * BN + h * KPT + lane_off;
        if (exp == 7) {  // timing experiment: no S read
#pragma unroll
          for (int c = 0; c < KPT; ++c) s[c] = 0.001f * c;
        } else {
#pragma unroll
          for (int c = 0; c < KPT / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(ta + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(r[e]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&s_empty[b]);
      if (exp == 8 || exp == 9) {  // timing experiment: no softmax at all (barriers only)
        mbar_arrive(&p_full[i & 1]);
        continue;
      }
      const int j0 = (t0 + i) * BN;
      // keys j0 + KPT h + c visible iff c <= lim_rel (causal + bounds) and not a pad
      const int lim_rel = min(lim, n_keys - 1) - j0 - KPT * h;
      if (key_pad != nullptr) {
        // BN-bit pad mask of this tile (BN/32 words), built by the first warpgroup
        if (h == 0 && q4 < BN / 32) {
          const int jm = j0 + m;
          const unsigned word = __ballot_sync(0xffffffffu, jm >= n_keys || key_pad[jm] != 0);
          if (lane == 0) padw[(i & 1) * 4 + q4] = word;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(128 * NWG) : "memory");
        const uint32_t* pw = padw + (i & 1) * 4 + (KPT / 32) * h;
#pragma unroll
        for (int c = 0; c < KPT; ++c)
          s[c] = (c <= lim_rel && !((pw[c >> 5] >> (c & 31)) & 1u)) ? s[c] : -INFINITY;
      } else if (lim_rel < KPT - 1) {
#pragma unroll
        for (int c = 0; c < KPT; ++c) s[c] = (c <= lim_rel) ? s[c] : -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) mx[e] = s[e];
#pragma unroll
      for (int c = 8; c < KPT; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
      float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      if (NWG > 1 && exp != 6) {  // (exp 6, timing experiment: no max exchange)
        xmax[((i & 1) * NWG + h) * 128 + m] = tmax;
        pair_bar();
#pragma unroll
        for (int o = 0; o < NWG; ++o)
          if (o != h) tmax = fmaxf(tmax, xmax[((i & 1) * NWG + o) * 128 + m]);
      }
      bool grow = false;
      float alpha = 1.f;
      if (i > 0) {
        grow = (m_run != -INFINITY) && ((tmax - m_run) * scale_log2 > kRescaleLog2);
        if (grow) {
          alpha = ex2_fast((m_run - tmax) * scale_log2);
          l_run *= alpha;
          m_run = tmax;
        }
      }
      const int pb = i & 1;
      if (m_run == -INFINITY) m_run = tmax;  // first visible keys: nothing accumulated yet
      const float base_l2 = (m_run == -INFINITY) ? 0.f : m_run * scale_log2;
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pt[KPT / 2];  // this part's keys of P, packed bf16x2 (TMEM P)
#pragma unroll
      for (int ch = 0; ch < KPT / 8; ++ch) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = ch * 8 + e * 2;
          // a quarter of the exponentials on the FMA pipe (the MUFU pipe
          // alone would take as long as the two MMAs of a tile)
          const bool poly = (ch & 3) == 3;
          const float x0 = fmaf(s[c], scale_log2, -base_l2), x1 = fmaf(s[c + 1], scale_log2, -base_l2);
          const float p0 = exp == 4 ? x0 : (poly ? ex2_poly(x0) : ex2_fast(x0));
          const float p1 = exp == 4 ? x1 : (poly ? ex2_poly(x1) : ex2_fast(x1));
          ps[(2 * e) & 7] += p0;
          ps[(2 * e + 1) & 7] += p1;
          __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
          pt[ch * 4 + e] = *reinterpret_cast<uint32_t*>(&hv);
        }
      }
      // P_i over S_i's first BN/2 columns: every part finished reading S_i
      // before the pair barrier above (one part: this thread read its own)
      if (exp != 5) tmem_st_cols<KPT / 2>(t_s0 + pb * BN + h * (KPT / 2) + lane_off, pt);  // (5: no P store)
      l_run += ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      // O *= alpha (this part's columns) for rows whose max grew past the lazy
      // threshold.  tcgen05.ld/st are warp-collective: the whole warp joins,
      // alpha = 1 for rows that keep their max.
      if (__any_sync(0xffffffffu, grow)) {
        twait(&p_empty[(i - 1) & 1], ((i - 1) >> 1) & 1, tracing, w2);  // PV_{i-1} done: O current
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < OPT / 32; ++c) {
          const uint32_t to = t_o + h * OPT + c * 32 + lane_off;
          uint32_t r[32];
          tmem_ld32(to, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          tmem_st32(to, r);
        }
        tmem_st_wait();
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[pb]);
    }
    // epilogue: total row sum = all parts
    // (slot parity n_tiles & 1 was last read before the previous pair barrier)
    float l_tot = l_run;
    if constexpr (NWG > 1) {
      xmax[((n_tiles & 1) * NWG + h) * 128 + m] = l_run;
      pair_bar();
#pragma unroll
      for (int o = 0; o < NWG; ++o)
        if (o != h) l_tot += xmax[((n_tiles & 1) * NWG + o) * 128 + m];
    }
    if (n_tiles > 0) {
      mbar_wait(&p_empty[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    __nv_bfloat16* out = ctx + ((int64_t)row * Hq + head) * DH + h * OPT;
    if (split) {
      // park this part's partial (unnormalised O, max in log2 units, sum) ...
      const int key = g * T + tile, slot = key * AT_MAXP + part;
      const bool any = n_tiles > 0 && m_run != -INFINITY;
      const float m_l2 = any ? m_run * scale_log2 : -INFINITY;
      float* my_o = ws_o + ((int64_t)slot * 128 + m) * DH + h * OPT;
#pragma unroll 1
      for (int c = 0; c < OPT / 32; ++c) {
        uint32_t r[32];
        if (n_tiles > 0) {
          tmem_ld32(t_o + h * OPT + c * 32 + lane_off, r);
          tmem_ld_wait();
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
          __stcg(reinterpret_cast<float4*>(my_o + c * 32) + e,
                 any ? make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                   __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f));
      }
      if (h == 0) __stcg(&ws_ml[(int64_t)slot * 128 + m], make_float2(m_l2, any ? l_tot : 0.f));
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(128 * NWG) : "memory");
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(&counters[key], 1);
        padw[0] = prev;  // (pad words are no longer needed)
        if (prev == parts - 1) counters[key] = 0;  // reset for the next launch
      }
      asm volatile("bar.sync 1, %0;" ::"r"(128 * NWG) : "memory");
      if ((int)padw[0] == parts - 1) {
        // ... and the last part to finish merges all of them, in part order
        __threadfence();
        float2 ml[AT_MAXP];
        float M = -INFINITY;
#pragma unroll
        for (int p = 0; p < AT_MAXP; ++p) {
          ml[p] = p < parts ? __ldcg(&ws_ml[((int64_t)key * AT_MAXP + p) * 128 + m]) : make_float2(-INFINITY, 0.f);
          M = fmaxf(M, ml[p].x);
        }
        float w[AT_MAXP];
        float lt = 0.f;
#pragma unroll
        for (int p = 0; p < AT_MAXP; ++p) {
          w[p] = ml[p].x == -INFINITY ? 0.f : exp2f(ml[p].x - M);
          lt = fmaf(ml[p].y, w[p], lt);
        }
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        if (row < n_q) {
#pragma unroll 1
          for (int c = 0; c < OPT / 8; ++c) {
            float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int p = 0; p < AT_MAXP; ++p) {
              if (p >= parts) break;
              const float* op = ws_o + (((int64_t)key * AT_MAXP + p) * 128 + m) * DH + h * OPT + c * 8;
              const float4 a0 = __ldcg(reinterpret_cast<const float4*>(op));
              const float4 a1 = __ldcg(reinterpret_cast<const float4*>(op) + 1);
              v[0] = fmaf(a0.x, w[p], v[0]); v[1] = fmaf(a0.y, w[p], v[1]);
              v[2] = fmaf(a0.z, w[p], v[2]); v[3] = fmaf(a0.w, w[p], v[3]);
              v[4] = fmaf(a1.x, w[p], v[4]); v[5] = fmaf(a1.y, w[p], v[5]);
              v[6] = fmaf(a1.z, w[p], v[6]); v[7] = fmaf(a1.w, w[p], v[7]);
            }
            uint4 pk;
            uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 hv = __floats2bfloat162_rn(v[2 * e] * inv, v[2 * e + 1] * inv);
              pw[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(out + c * 8) = pk;
          }
          if (h == 0)
            lse[(int64_t)row * Hq + head] = lt > 0.f ? (M + log2f(lt)) * 0.6931471805599453f : -INFINITY;
        }
      }
    } else {
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
#pragma unroll 1
      for (int c = 0; c < OPT / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(t_o + h * OPT + c * 32 + lane_off, r);
        tmem_ld_wait();
        if (row < n_q && n_tiles > 0) {
          uint4 pk[4];
          uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            __nv_bfloat162 hv = __floats2bfloat162_rn(__uint_as_float(r[2 * e]) * inv, __uint_as_float(r[2 * e + 1]) * inv);
            pw[e] = *reinterpret_cast<uint32_t*>(&hv);
          }
          uint4* o4 = reinterpret_cast<uint4*>(out + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) o4[e] = pk[e];
        }
      }
      if (row < n_q && h == 0)
        lse[(int64_t)row * Hq + head] = l_tot > 0.f ? (m_run * scale_log2 + log2f(l_tot)) * 0.6931471805599453f : -INFINITY;
    }
  }
  if (tracing) {
    long long* tr = trace + 16 * (int64_t)blockIdx.x;
    if (threadIdx.x == 64) {
      long long t_end;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_end));
      int smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      tr[0] = n_tiles; tr[1] = t_begin; tr[2] = t_end; tr[3] = smid;
      tr[4] = w0; tr[5] = w1; tr[6] = w2; tr[7] = w3;  // softmax: s_full, -, p_empty(grow)
    } else if (threadIdx.x == 32) {
      tr[8] = w0; tr[9] = w1; tr[10] = w2; tr[11] = w3;  // mma: k_full, s_empty, p_full, v_full
      tr[12] = t_s_issue; tr[13] = t_s_commit; tr[14] = t_p_issue; tr[15] = t_p_commit;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<SM::TMEM_COLS>(tmem);
  }
}

// 8 x 16-byte L2 loads at a 4 KiB stride issued back to back (one asm block:
// the compiler cannot interleave their uses between them)
__device__ __forceinline__ void ld8_f4_cg_4k(const float4* p, float (&a)[32]) {
  asm volatile(
      "ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%32];\n"
      "ld.global.cg.v4.f32 {%4, %5, %6, %7}, [%32+4096];\n"
      "ld.global.cg.v4.f32 {%8, %9, %10, %11}, [%32+8192];\n"
      "ld.global.cg.v4.f32 {%12, %13, %14, %15}, [%32+12288];\n"
      "ld.global.cg.v4.f32 {%16, %17, %18, %19}, [%32+16384];\n"
      "ld.global.cg.v4.f32 {%20, %21, %22, %23}, [%32+20480];\n"
      "ld.global.cg.v4.f32 {%24, %25, %26, %27}, [%32+24576];\n"
      "ld.global.cg.v4.f32 {%28, %29, %30, %31}, [%32+28672];\n"
      : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7]), "=f"(a[8]),
        "=f"(a[9]), "=f"(a[10]), "=f"(a[11]), "=f"(a[12]), "=f"(a[13]), "=f"(a[14]), "=f"(a[15]), "=f"(a[16]),
        "=f"(a[17]), "=f"(a[18]), "=f"(a[19]), "=f"(a[20]), "=f"(a[21]), "=f"(a[22]), "=f"(a[23]), "=f"(a[24]),
        "=f"(a[25]), "=f"(a[26]), "=f"(a[27]), "=f"(a[28]), "=f"(a[29]), "=f"(a[30]), "=f"(a[31])
      : "l"(p)
      : "memory");
}

// ---- ping-pong kernel: two Q tiles per CTA share every K/V tile ---------------
//
// CTA = one work item (GQA group g, block of 2R query rows, part of its causal
// key range) = 2 Q tiles of 128 M-rows.
//   warp 0      TMA: Q0 + Q1 once, K_j / V_j (2-deep rings; each 128-key tile
//               feeds both Q tiles, so a K/V byte from L2 serves 256 M-rows)
//   warp 1      MMA issuer, per key tile j and Q tile X in turn:
//                 O_X += P_X(j) V_j, then S_X(j+1) = Q_X K_{j+1}^T
//               so while softmax X works on tile j the tensor pipe runs the
//               other Q tile's PV and S (the two softmax warpgroups ping-pong
//               on one tensor pipe)
//   warps 4-7   softmax of Q tile 0, warps 8-11 of Q tile 1: thread = one
//               M-row, all 128 keys of it (no cross-thread max exchange);
//               fp32 online softmax with packed f32x2 math, exp2 on MUFU for
//               three quarters and as a polynomial on the FMA pipe for one
//               quarter, lazy O rescale in TMEM, P as bf16 over the first half
//               of its own S buffer (the PV MMA's A operand)
// TMEM: S0/P0 | S1/P1 | O0 | O1.  S_X(j+1) overwrites P_X(j) only after
// PV_X(j) (one MMA thread, in-order tensor pipe), and softmax X sees S_X(j+1)
// only once PV_X(j) completed, so O_X is current whenever it is rescaled.
// Items are dispatched longest first; when the (group, block) grid leaves SMs
// idle the long items' key ranges are cut into parts merged in fixed order.
template <int DH>
struct Pp {
  static constexpr int BN = 128;
  static constexpr int KST = 2, VST = 2;
  static constexpr int THREADS = 384;
  static constexpr int ATOMS = DH / 64;
  static constexpr int Q_BYTES = 128 * DH * 2;  // one Q tile (128 M-rows)
  static constexpr int KV_BYTES = BN * DH * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * Q_BYTES;
  static constexpr int V_OFF = K_OFF + KST * KV_BYTES;
  static constexpr int BAR_OFF = V_OFF + VST * KV_BYTES;
  static constexpr int PLAN_OFF = BAR_OFF + 1024;
  static constexpr size_t TOTAL = PLAN_OFF + 3 * AT_MAXT * 4;
  static constexpr int TMEM_COLS = 512;
  static_assert(2 * BN + 2 * DH <= TMEM_COLS, "TMEM budget");
};

// PF: exponentials per 8 key pairs computed as a polynomial on the FMA pipe
// (A/B at config 2 / full / 32k / 70B rank, us: PF 2 63.9 / 221 / 1153 / 150,
// PF 0 -- / 258 / 1585 / 181, PF 1 -- / 226 / 1280 / 154, PF 4 -- / 235 /
// 1350 / 162)
// RH: registers per softmax thread (setmaxnreg; the TMA/MMA warpgroup keeps
// 504 - 2 RH).  A/B (us, config 2 / full / 32k / 70B rank): RH 224 62.0 /
// 205.5 / 1101 / 154, RH 200 61.8 / 209.4 / 1254 / 158, RH 168 (no split)
// 64.1 / 214.6 / 1236 / 158.
template <int DH, int PF = 2, int RH = 224>
__global__ void __launch_bounds__(384, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const int32_t* __restrict__ q_slot,
                   const uint8_t* __restrict__ key_pad, __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse,
                   int n_q, int n_keys, int Hq, int G, float scale_log2, int n_groups, int n_blocks, int target,
                   int max_parts, float* __restrict__ ws_o, float2* __restrict__ ws_ml, int* __restrict__ counters,
                   int pstride, int ext, long long* __restrict__ trace) {
  using SM = Pp<DH>;
  constexpr int BN = SM::BN, KST = SM::KST, VST = SM::VST, NT = SM::THREADS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw;
  if (smem_u32(smem_raw) & 1023) __trap();
  uint8_t* sQ = base + SM::Q_OFF;
  uint8_t* sK = base + SM::K_OFF;
  uint8_t* sV = base + SM::V_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + SM::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;        // [KST]
  uint64_t* k_empty = k_full + KST;   // [KST] committed after both S MMAs of the tile
  uint64_t* v_full = k_empty + KST;   // [VST]
  uint64_t* v_empty = v_full + VST;   // [VST] committed after both PV MMAs of the tile
  uint64_t* s_full = v_empty + VST;   // [2] per Q tile
  uint64_t* p_full = s_full + 2;      // [2] per Q tile (128 softmax arrivals)
  uint64_t* o_done = p_full + 2;      // [2] per Q tile: last PV completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  int* s_kmax = reinterpret_cast<int*>(tmem_slot + 1);  // [2]
  int* s_item = s_kmax + 2;                             // group, block, part, parts, est
  int* s_flag = s_item + 5;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = 128 / G;  // query rows per Q tile
  const int RB = 2 * R;   // query rows per CTA block
  const int T = n_blocks;
  pdl_trigger();
  pdl_wait();
  if (max_parts > 1) {
    // items (group, block, key part), longest first -- see attn_tc_kernel
    int* p_len = reinterpret_cast<int*>(base + SM::PLAN_OFF);
    int* p_parts = p_len + AT_MAXT;
    int* p_order = p_parts + AT_MAXT;
    for (int t = threadIdx.x; t < T; t += NT) {
      const int kq = q_slot[min((t + 1) * RB, n_q) - 1];
      const int est = kq < 0 ? 0 : min(kq, n_keys - 1) / BN + 1;
      const int parts = max(1, min(max_parts, (est + target - 1) / target));
      p_parts[t] = parts;
      p_len[t] = (est + parts - 1) / parts;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += NT) {
      const int lt = p_len[t];
      int rank = 0;
      for (int u = 0; u < T; ++u) rank += (p_len[u] > lt || (p_len[u] == lt && u > t)) ? 1 : 0;
      p_order[rank] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int idx = blockIdx.x;
      s_item[0] = -1;
      for (int r = 0; r < T; ++r) {
        const int t = p_order[r], c = n_groups * p_parts[t];
        if (idx < c) {
          s_item[0] = idx % n_groups;
          s_item[1] = t;
          s_item[2] = idx / n_groups;
          s_item[3] = p_parts[t];
          s_item[4] = p_len[t] * p_parts[t];
          break;
        }
        idx -= c;
      }
    }
  } else if (threadIdx.x == 0) {
    s_item[0] = blockIdx.x % n_groups;
    s_item[1] = T - 1 - (int)blockIdx.x / n_groups;
    s_item[2] = 0;
    s_item[3] = 1;
    s_item[4] = 0;
  }
  __syncthreads();
  const int g = s_item[0];
  if (g < 0) return;
  const int blk = s_item[1], part = s_item[2], parts = s_item[3], est = s_item[4];
  const int row0 = blk * RB;

  if (threadIdx.x < 2) s_kmax[threadIdx.x] = -1;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 128);
      mbar_init(&o_done[x], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<SM::TMEM_COLS>(tmem_slot);
  __syncthreads();
  if (threadIdx.x < 256) {  // causal key range of each Q tile: max slot over its rows
    const int X = threadIdx.x >> 7, m = threadIdx.x & 127;
    const int r = row0 + X * R + m / G;
    if (r < n_q) atomicMax(&s_kmax[X], min(q_slot[r], n_keys - 1));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntot0 = s_kmax[0] < 0 ? 0 : s_kmax[0] / BN + 1;
  const int ntot1 = s_kmax[1] < 0 ? 0 : s_kmax[1] / BN + 1;
  const int ntot = max(ntot0, ntot1);
  const bool split = parts > 1;
  const int t0 = split ? min(part * est / parts, ntot) : 0;
  const int t1 = !split || part == parts - 1 ? ntot : min((part + 1) * est / parts, ntot);
  const int n0 = max(0, min(t1, ntot0) - t0), n1 = max(0, min(t1, ntot1) - t0);
  const int nmax = max(n0, n1);
  const bool tracing = trace != nullptr;
  long long tr_a = 0, tr_b = 0, tr_c = 0;
  long long t_begin = 0;
  if (tracing && threadIdx.x == 128) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_begin));

  // Each role ends on its own (no control-flow join after the per-role
  // register allocation below): trace, CTA barrier, TMEM release.
  auto finish = [&]() {
    if (tracing) {
      long long* tr = trace + 24 * (int64_t)blockIdx.x;
      if (threadIdx.x == 128 || threadIdx.x == 256) {  // softmax X = 0 / 1: s_full wait, busy, epilogue
        const int o = threadIdx.x == 128 ? 4 : 7;
        tr[o] = tr_a; tr[o + 1] = tr_b; tr[o + 2] = tr_c;
      }
      if (threadIdx.x == 32) { tr[10] = tr_a; tr[11] = tr_b; }  // mma: p_full, k/v/q waits
      if (threadIdx.x == 0) { tr[12] = tr_a; tr[13] = tr_b; }   // producer: k_empty, v_empty
    }
    tc_fence_before();
    asm volatile("bar.sync 15, 384;" ::: "memory");
    if (tracing && threadIdx.x == 128) {
      long long* tr = trace + 24 * (int64_t)blockIdx.x;
      long long t_end;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_end));
      int smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      tr[0] = nmax; tr[1] = t_begin; tr[2] = t_end; tr[3] = smid;
    }
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc<SM::TMEM_COLS>(tmem);
    }
  };
  // registers: the TMA / MMA warpgroup needs few, a softmax thread holds a
  // 128-key S row ((504 - 2 RH) + 2 RH per 128 threads = 3 x 168)
#define PP_REG_LO "setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(504 - 2 * RH)
  if (warp == 0) {
    asm volatile(PP_REG_LO : "memory");
    if (lane == 0 && nmax > 0) {
      mbar_expect_tx(q_full, 2 * SM::Q_BYTES);
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int a = 0; a < SM::ATOMS; ++a)
          tma_load_3d(sQ + x * SM::Q_BYTES + a * 128 * 128, &tmQ, q_full, a * 64, g * G, row0 + x * R);
      for (int j = 0; j < nmax; ++j) {
        const int ks = j % KST;
        twait(&k_empty[ks], ((j / KST) & 1) ^ 1, tracing, tr_a);
        mbar_expect_tx(&k_full[ks], SM::KV_BYTES);
#pragma unroll
        for (int a = 0; a < SM::ATOMS; ++a)
          tma_load_2d(sK + ks * SM::KV_BYTES + a * BN * 128, &tmK, &k_full[ks], g * DH + a * 64, (t0 + j) * BN);
        const int vs = j % VST;
        twait(&v_empty[vs], ((j / VST) & 1) ^ 1, tracing, tr_b);
        mbar_expect_tx(&v_full[vs], SM::KV_BYTES);
#pragma unroll
        for (int a = 0; a < SM::ATOMS; ++a)
          tma_load_2d(sV + vs * SM::KV_BYTES + a * BN * 128, &tmV, &v_full[vs], g * DH + a * 64, (t0 + j) * BN);
      }
    }
    finish();
    return;
  } else if (warp == 1) {
    asm volatile(PP_REG_LO : "memory");
    if (lane == 0 && nmax > 0) {
      constexpr uint32_t id_s = idesc_bf16(128, BN, false);
      constexpr uint32_t id_o = idesc_bf16(128, DH, true);
      const int nx[2] = {n0, n1};
      auto issue_s = [&](int x, int j) {
        const int ks = j % KST;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const int a = kk >> 2, w = kk & 3;
          const uint64_t bd = desc_sw128(sK + ks * SM::KV_BYTES + a * BN * 128) + 2 * w;
          const uint64_t ad = desc_sw128(sQ + x * SM::Q_BYTES + a * 128 * 128) + 2 * w;
          mma_bf16(tmem + x * BN, ad, bd, id_s, kk > 0);
        }
        mma_commit(&s_full[x]);
      };
      twait(q_full, 0, tracing, tr_b);
      twait(&k_full[0], 0, tracing, tr_b);
      tc_fence_after();
      if (n0 > 0) issue_s(0, 0);
      if (n1 > 0) issue_s(1, 0);
      mma_commit(&k_empty[0]);
      for (int j = 0; j < nmax; ++j) {
        const int vs = j % VST;
        bool v_ready = false, k_ready = false;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (j >= nx[x]) continue;
          twait(&p_full[x], j & 1, tracing, tr_a);
          if (!v_ready) {
            twait(&v_full[vs], (j / VST) & 1, tracing, tr_b);
            v_ready = true;
          }
          tc_fence_after();
          const uint32_t t_o = tmem + 2 * BN + x * DH, t_p = tmem + x * BN;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            const uint64_t bd = desc_sw128_mn(sV + vs * SM::KV_BYTES + kk * 16 * 128, BN * 128);
            mma_bf16_ts(t_o, t_p + kk * 8, bd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (j + 1 < nx[x]) {
            if (!k_ready) {
              twait(&k_full[(j + 1) % KST], ((j + 1) / KST) & 1, tracing, tr_b);
              tc_fence_after();
              k_ready = true;
            }
            issue_s(x, j + 1);
          } else {
            mma_commit(&o_done[x]);
          }
        }
        mma_commit(&v_empty[vs]);
        if (k_ready) mma_commit(&k_empty[(j + 1) % KST]);
      }
    }
    finish();
    return;
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RH) : "memory");
    // ---- softmax of Q tile X: thread = M-row m, all BN keys -------------------
    const int X = (warp - 4) >> 2;
    const int q4 = warp & 3;  // TMEM lane quarter
    const int m = q4 * 32 + lane;
    const int row = row0 + X * R + m / G;
    const int head = g * G + m % G;
    const int lim = row < n_q ? min(q_slot[row], n_keys - 1) : -1;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t t_s = tmem + X * BN + lane_off, t_o = tmem + 2 * BN + X * DH + lane_off;
    const int nX = X == 0 ? n0 : n1;
    const uint64_t sl2 = f2_pack(scale_log2, scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    constexpr float kRescaleLog2 = 8.f;
    for (int j = 0; j < nX; ++j) {
      twait(&s_full[X], j & 1, tracing, tr_a);
      const long long tb0 = tracing ? clock64() : 0;
      tc_fence_after();
      float s[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
      const int j0 = (t0 + j) * BN;
      const int lim_rel = lim - j0;
      if (key_pad != nullptr) {
#pragma unroll
        for (int u = 0; u < BN / 16; ++u) {
          uint4 w = make_uint4(0u, 0u, 0u, 0u);
          const int kb = j0 + u * 16;
          if (kb + 16 <= n_keys) {
            w = __ldg(reinterpret_cast<const uint4*>(key_pad + kb));
          } else {
            uint8_t* wb = reinterpret_cast<uint8_t*>(&w);
            for (int e = 0; e < 16; ++e) wb[e] = kb + e < n_keys ? key_pad[kb + e] : 1;
          }
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int c = u * 16 + e;
            const bool padded = ((ww[e >> 2] >> (8 * (e & 3))) & 0xffu) != 0u;
            s[c] = (c <= lim_rel && !padded) ? s[c] : -INFINITY;
          }
        }
      } else if (lim_rel < BN - 1) {
#pragma unroll
        for (int c = 0; c < BN; ++c) s[c] = (c <= lim_rel) ? s[c] : -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) mx[e] = fmax3(s[e], s[8 + 2 * e], s[9 + 2 * e]);
#pragma unroll
      for (int c = 24; c < BN; c += 16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = fmax3(mx[e], s[c + 2 * e], s[c + 2 * e + 1]);
      }
      const float tmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
      bool grow = false;
      float alpha = 1.f;
      if (m_run == -INFINITY) {
        m_run = tmax;
      } else if ((tmax - m_run) * scale_log2 > kRescaleLog2) {
        grow = true;
        alpha = ex2_fast((m_run - tmax) * scale_log2);
        l_run *= alpha;
        m_run = tmax;
      }
      const float nb = (m_run == -INFINITY) ? 0.f : -m_run * scale_log2;
      const uint64_t nb2 = f2_pack(nb, nb);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
      // P in two 64-key halves (32 packed columns each): fewer live registers
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pt[BN / 4];
#pragma unroll
        for (int e2 = 0; e2 < BN / 4; ++e2) {
          const int e = hh * (BN / 4) + e2;
          const uint64_t x2 = ffma2(f2_pack(s[2 * e], s[2 * e + 1]), sl2, nb2);
          uint64_t p2;
          if ((e & 7) >= 8 - PF) {  // PF / 8 of the exponentials on the FMA pipe
            p2 = ex2_poly2(x2);
          } else {
            float x0, x1;
            f2_unpack(x2, x0, x1);
            p2 = f2_pack(ex2_fast(x0), ex2_fast(x1));
          }
          acc[e & 3] = fadd2(acc[e & 3], p2);
          float p0, p1;
          f2_unpack(p2, p0, p1);
          __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
          pt[e2] = *reinterpret_cast<uint32_t*>(&hv);
        }
        tmem_st_cols<32>(t_s + hh * 32, pt);
      }
      if (__any_sync(0xffffffffu, grow)) {  // O_X *= alpha (PV_X(j-1) completed before S_X(j))
        const uint64_t a2 = f2_pack(alpha, alpha);
#pragma unroll 1
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(t_o + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float o0, o1;
            f2_unpack(fmul2(f2_pack(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), a2), o0, o1);
            r[2 * e] = __float_as_uint(o0);
            r[2 * e + 1] = __float_as_uint(o1);
          }
          tmem_st32(t_o + c * 32, r);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[X]);
      if (tracing) tr_b += clock64() - tb0;
      const uint64_t a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
      float sa, sb;
      f2_unpack(a01, sa, sb);
      l_run += sa + sb;
    }
    const long long te0 = tracing ? clock64() : 0;
    if (nX > 0) {
      mbar_wait(&o_done[X], 0);
      tc_fence_after();
    }
    __nv_bfloat16* out = ctx + ((int64_t)row * Hq + head) * DH;
    if (split) {
      // park this part's partial ([part][column / 4][256 M-rows][4] per key: a
      // warp's 16-byte stores cover 512 contiguous bytes); the last part of
      // the block to finish merges all of them in part order
      const int key = g * T + blk, mm = X * 128 + m;
      const bool any = nX > 0 && m_run != -INFINITY;
      float4* my_o = reinterpret_cast<float4*>(ws_o) + ((int64_t)key * pstride + part) * (DH / 4) * 256 + mm;
#pragma unroll 1
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t r[32];
        if (nX > 0) {
          tmem_ld32(t_o + c * 32, r);
          tmem_ld_wait();
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
          __stcg(my_o + (c * 8 + e) * 256,
                 any ? make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                   __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f));
      }
      __stcg(&ws_ml[((int64_t)key * pstride + part) * 256 + mm],
             make_float2(any ? m_run * scale_log2 : -INFINITY, any ? l_run : 0.f));
      if (!ext) {  // (ext: the merge kernel attn_pp_merge folds the parts)
      __threadfence();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (warp == 4 && lane == 0) {
        const int prev = atomicAdd(&counters[key], 1);
        *s_flag = prev;
        if (prev == parts - 1) counters[key] = 0;  // reset for the next launch
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (*s_flag == parts - 1) {
        __threadfence();
        float mp[AT_MAXP], w[AT_MAXP], lp[AT_MAXP];
        float M = -INFINITY;
#pragma unroll
        for (int p = 0; p < AT_MAXP; ++p) {
          const float2 ml = p < parts ? __ldcg(&ws_ml[((int64_t)key * pstride + p) * 256 + mm])
                                      : make_float2(-INFINITY, 0.f);
          mp[p] = ml.x;
          lp[p] = ml.y;
          M = fmaxf(M, ml.x);
        }
        float lt = 0.f;
#pragma unroll
        for (int p = 0; p < AT_MAXP; ++p) {
          w[p] = mp[p] == -INFINITY ? 0.f : exp2f(mp[p] - M);
          lt = fmaf(lp[p], w[p], lt);
        }
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        if (row < n_q) {
#pragma unroll 1
          for (int cg = 0; cg < DH / 32; ++cg) {
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0.f;
#pragma unroll
            for (int p = 0; p < AT_MAXP; ++p) {
              if (p < parts) {
                const float4* op =
                    reinterpret_cast<const float4*>(ws_o) + ((int64_t)key * pstride + p) * (DH / 4) * 256 + (cg * 8) * 256 + mm;
                float a[32];
                ld8_f4_cg_4k(op, a);
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = fmaf(a[e], w[p], v[e]);
              }
            }
            uint4 pk[4];
            uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              __nv_bfloat162 hv = __floats2bfloat162_rn(v[2 * e] * inv, v[2 * e + 1] * inv);
              pw[e] = *reinterpret_cast<uint32_t*>(&hv);
            }
            uint4* o4 = reinterpret_cast<uint4*>(out + cg * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e) o4[e] = pk[e];
          }
          lse[(int64_t)row * Hq + head] = lt > 0.f ? (M + log2f(lt)) * 0.6931471805599453f : -INFINITY;
        }
      }
      }
    } else {
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll 1
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t r[32];
        if (nX > 0) {
          tmem_ld32(t_o + c * 32, r);
          tmem_ld_wait();
        }
        if (row < n_q) {
          uint4 pk[4];
          uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float o0 = nX > 0 ? __uint_as_float(r[2 * e]) * inv : 0.f;
            const float o1 = nX > 0 ? __uint_as_float(r[2 * e + 1]) * inv : 0.f;
            __nv_bfloat162 hv = __floats2bfloat162_rn(o0, o1);
            pw[e] = *reinterpret_cast<uint32_t*>(&hv);
          }
          uint4* o4 = reinterpret_cast<uint4*>(out + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) o4[e] = pk[e];
        }
      }
      if (row < n_q)
        lse[(int64_t)row * Hq + head] =
            l_run > 0.f ? (m_run * scale_log2 + log2f(l_run)) * 0.6931471805599453f : -INFINITY;
    }
    if (tracing) tr_c += clock64() - te0;
    finish();
    return;
  }
  asm volatile(PP_REG_LO : "memory");
  finish();  // warps 2-3
}
#undef PP_REG_LO

long long* g_attn_trace = nullptr;  // debug: per-CTA (n_tiles, start, end, sm, stalls)

// zero-initialised pair counters of the split-KV merge, one array per stream
// (the merging CTA resets its counter, so they stay zero between launches)
int* split_counters(cudaStream_t st, int n) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::pair<int*, int>> by_stream;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = (reinterpret_cast<uint64_t>(st) << 4) ^ (uint64_t)dev;
  std::lock_guard<std::mutex> g(mu);
  auto& e = by_stream[key];
  if (e.second < n) {
    if (e.first) cudaFree(e.first);
    const int cap = n < 4096 ? 4096 : n;
    if (cudaMalloc(&e.first, sizeof(int) * cap) != cudaSuccess) { e = {nullptr, 0}; return nullptr; }
    cudaMemset(e.first, 0, sizeof(int) * cap);
    e.second = cap;
  }
  return e.first;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

int encode(CUtensorMap* m, int rank, const void* p, const cuuint64_t* dims, const cuuint64_t* strides,
           const cuuint32_t* box) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(CC_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CC_E_CUDA, "attention_tc: tensor map encode failed " + std::to_string((int)r));
  return CC_OK;
}

int g_attn_variant = -1;  // debug hook / CCB_ATTN_VARIANT: kernel shape (see pick below)

// CCB_ATTN_EXP (timing experiments only, wrong results): 1 = V as a K-major
// PV operand, 2 = no PV MMA, 3 = no S MMA, 4 = no softmax exponentials,
// 5 = no P store, 6 = no max exchange, 7 = no S read, 8 = no softmax work,
// 9 = 8 without the S and PV MMAs
int attn_exp() {
  const char* e = getenv("CCB_ATTN_EXP");
  return e ? atoi(e) : 0;
}

template <int DH, int BN, int NWG, int KST = (BN == 64 ? 2 : 3), int VST = 2>
int launch(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad, void* ctx,
           float* lse, int n_q, int n_keys, int Hq, int Hkv, cudaStream_t st) {
  using SM = At<DH, BN, NWG, KST, VST>;
  const int G = Hq / Hkv;
  const int R = 128 / G;
  CUtensorMap mq, mk, mv;
  {
    cuuint64_t dims[3] = {(cuuint64_t)DH, (cuuint64_t)Hq, (cuuint64_t)n_q};
    cuuint64_t strides[2] = {(cuuint64_t)DH * 2, (cuuint64_t)Hq * DH * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)R};
    int rc = encode(&mq, 3, q, dims, strides, box);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)Hkv * DH, (cuuint64_t)n_keys};
    cuuint64_t strides[1] = {(cuuint64_t)Hkv * DH * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)BN};
    int rc = encode(&mk, 2, k, dims, strides, box);
    if (rc) return rc;
    rc = encode(&mv, 2, v, dims, strides, box);
    if (rc) return rc;
  }
  if (int rc = ensure_smem(attn_tc_kernel<DH, BN, NWG, KST, VST>, SM::TOTAL)) return rc;
  const int row_tiles = (n_q + R - 1) / R;
  // Work items: when the grid of (group, row tile) CTAs leaves CTA slots idle,
  // the row tiles with long causal key ranges are cut into up to AT_MAXP key
  // parts (merged in part order by the last part to finish), all items
  // dispatched longest first.  With a full grid the extra CTAs' fixed costs
  // (prologue, pipeline fill, partial write + merge) outweigh the better
  // balance: measured at config 2 (208 CTAs) 65.9 us unsplit vs 94.7 us with
  // parts of half the per-SM share.
  const int slots = num_sms() * SM::CTAS_PER_SM;
  const int max_tiles = (n_keys + BN - 1) / BN;
  int target = max_tiles, max_parts = 1;
  if (row_tiles <= AT_MAXT && max_tiles > 0 && Hkv * row_tiles < slots) {
    // (rounded up: at r = 0.05, 80 items on 148 SMs, 2 parts measured 51.5 us vs 70 us unsplit)
    max_parts = std::max(1, std::min(AT_MAXP, (slots + Hkv * row_tiles - 1) / (Hkv * row_tiles)));
    target = std::max(8 * 128 / BN, (max_tiles + max_parts - 1) / max_parts);
    max_parts = std::min(max_parts, (max_tiles + target - 1) / target);
    if (max_parts < 1) max_parts = 1;
  }
  if (getenv("CCB_ATTN_NOSPLIT")) max_parts = 1;
  if (const char* e = getenv("CCB_ATTN_SPLIT")) {  // experiments: "target,max_parts"
    int a = 0, b = 0;
    if (sscanf(e, "%d,%d", &a, &b) == 2 && a > 0 && b >= 1 && b <= AT_MAXP && row_tiles <= AT_MAXT) {
      target = a;
      max_parts = b;
    }
  }
  float* ws_o = nullptr;
  float2* ws_ml = nullptr;
  int* counters = nullptr;
  if (max_parts > 1) {
    const size_t keys = (size_t)Hkv * row_tiles;
    const size_t bytes = keys * AT_MAXP * 128 * (DH * sizeof(float) + sizeof(float2));
    uint8_t* scratch = (uint8_t*)stream_scratch(st, SCR_ATTN, bytes);
    counters = split_counters(st, (int)keys);
    if (!scratch || !counters) return fail(CC_E_CUDA, "attention_tc: split workspace allocation failed");
    ws_o = reinterpret_cast<float*>(scratch);
    ws_ml = reinterpret_cast<float2*>(scratch + keys * AT_MAXP * 128 * DH * sizeof(float));
  }
  // (an upper bound: CTAs past the planned items exit at once)
  dim3 grid(Hkv * row_tiles * max_parts);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  return launch_k(attn_tc_kernel<DH, BN, NWG, KST, VST>, grid, dim3(SM::THREADS), SM::TOTAL, st, "attention_tc", mq, mk, mv,
                  q_slot, key_pad, (__nv_bfloat16*)ctx, lse, n_q, n_keys, Hq, G, scale_log2, g_attn_trace, Hkv,
                  row_tiles, target, max_parts, ws_o, ws_ml, counters, attn_exp());
}

// Key-split plan of the ping-pong kernel for grids smaller than the SM count:
// the (target tiles per part, max parts) pair that minimises the modelled
// makespan -- block t's key range modelled as a ramp (rows spread over the
// prompt, est_t = ceil(max_tiles (t+1) / T) tiles), parts of ceil(est / parts)
// tiles plus a fixed cost of 3 tiles per CTA and 2 more per merged item,
// scheduled longest-first onto the SMs (the kernel's own order).  Measured at
// the 70B rank shape: 102.8 us (16/3) vs 135.5 us for the old rule (65/2);
// config 2 (21/2) and r = 0.05 (11/4) keep their plans.  Cached per shape.
std::pair<int, int> pp_split_plan(int T, int groups, int max_tiles, int slots, int maxp_cap = AT_MAXP,
                                  double merge_cost = 2.0) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, std::pair<int, int>> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(T, groups, max_tiles, slots * 64 + maxp_cap);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  double best = 1e30;
  size_t best_n = 0;
  std::pair<int, int> plan{max_tiles, 1};
  std::vector<double> ctas;
  std::vector<double> load(slots);
  for (int maxp = 1; maxp <= maxp_cap; ++maxp)
    for (int target = std::max(1, std::min(8, max_tiles)); target <= max_tiles; ++target) {
      ctas.clear();
      for (int t = 0; t < T; ++t) {
        const int est = (int)(((int64_t)max_tiles * (t + 1) + T - 1) / T);
        const int parts = std::max(1, std::min(maxp, (est + target - 1) / target));
        const double c = (est + parts - 1) / parts + 3.0 + (parts > 1 ? merge_cost : 0.0);
        for (int k = 0; k < groups * parts; ++k) ctas.push_back(c);
      }
      std::sort(ctas.begin(), ctas.end(), std::greater<double>());
      std::priority_queue<double, std::vector<double>, std::greater<double>> h;
      for (int i = 0; i < slots; ++i) h.push(0.0);
      double mk = 0.0;
      for (double c : ctas) {
        const double x = h.top() + c;
        h.pop();
        h.push(x);
        mk = std::max(mk, x);
      }
      if (mk < best - 1e-9 || (mk < best + 1e-9 && ctas.size() < best_n)) {
        best = mk;
        best_n = ctas.size();
        plan = {target, maxp};
      }
    }
  cache[key] = plan;
  return plan;
}

// Key-part merge for the ping-pong kernel's "ext" mode (few (group, block)
// items, many key parts): the parts only park their partials; this kernel
// folds them, one CTA per (item, 16 output columns), one thread per M-row,
// in part order (the same arithmetic as the in-kernel merge).  Items whose
// block was not split were written by the attention kernel itself.
template <int DH>
__global__ void __launch_bounds__(256) attn_pp_merge(const float* __restrict__ ws_o, const float2* __restrict__ ws_ml,
                                                     const int32_t* __restrict__ q_slot, __nv_bfloat16* __restrict__ ctx,
                                                     float* __restrict__ lse, int n_q, int n_keys, int Hq, int G,
                                                     int n_blocks, int target, int max_parts, int pstride) {
  constexpr int BN = Pp<DH>::BN;
  pdl_trigger();
  pdl_wait();
  const int key = blockIdx.x, cg = blockIdx.y, mm = threadIdx.x;
  const int g = key / n_blocks, blk = key % n_blocks;
  const int RB = 2 * (128 / G);
  const int kq = q_slot[min((blk + 1) * RB, n_q) - 1];
  const int est = kq < 0 ? 0 : min(kq, n_keys - 1) / BN + 1;
  const int parts = max(1, min(max_parts, (est + target - 1) / target));
  if (parts <= 1) return;
  const int row = blk * RB + mm / G, head = g * G + mm % G;
  if (row >= n_q) return;
  // all (max, sum) pairs in one round trip, then this CTA's 16 columns of the
  // partial rows eight parts per round trip (the loads of a group go out together)
  float mp[AT_MAXP_EXT], lp[AT_MAXP_EXT];
  float M = -INFINITY;
#pragma unroll
  for (int p = 0; p < AT_MAXP_EXT; ++p) {
    const float2 ml = p < parts ? __ldcg(&ws_ml[((int64_t)key * pstride + p) * 256 + mm]) : make_float2(-INFINITY, 0.f);
    mp[p] = ml.x;
    lp[p] = ml.y;
  }
#pragma unroll
  for (int p = 0; p < AT_MAXP_EXT; ++p) M = fmaxf(M, mp[p]);
  float lt = 0.f;
  float v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = 0.f;
#pragma unroll
  for (int p0 = 0; p0 < AT_MAXP_EXT; p0 += 8) {
    if (p0 >= parts) break;
    float4 a[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (p0 + i < parts) {
        const float4* op = reinterpret_cast<const float4*>(ws_o) + ((int64_t)key * pstride + p0 + i) * (DH / 4) * 256 +
                           (cg * 4) * 256 + mm;
#pragma unroll
        for (int c = 0; c < 4; ++c) a[i][c] = __ldcg(op + c * 256);
      }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (p0 + i >= parts) break;
      const float w = mp[p0 + i] == -INFINITY ? 0.f : exp2f(mp[p0 + i] - M);
      lt = fmaf(lp[p0 + i], w, lt);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v[4 * c] = fmaf(a[i][c].x, w, v[4 * c]);
        v[4 * c + 1] = fmaf(a[i][c].y, w, v[4 * c + 1]);
        v[4 * c + 2] = fmaf(a[i][c].z, w, v[4 * c + 2]);
        v[4 * c + 3] = fmaf(a[i][c].w, w, v[4 * c + 3]);
      }
    }
  }
  const float inv = lt > 0.f ? 1.f / lt : 0.f;
  uint4 pk[2];
  uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    __nv_bfloat162 hv = __floats2bfloat162_rn(v[2 * e] * inv, v[2 * e + 1] * inv);
    pw[e] = *reinterpret_cast<uint32_t*>(&hv);
  }
  uint4* o4 = reinterpret_cast<uint4*>(ctx + ((int64_t)row * Hq + head) * DH + cg * 16);
#pragma unroll
  for (int e = 0; e < 2; ++e) o4[e] = pk[e];
  if (cg == 0) lse[(int64_t)row * Hq + head] = lt > 0.f ? (M + log2f(lt)) * 0.6931471805599453f : -INFINITY;
}

template <int DH, int PF = 2, int RH = 224>
int launch_pp(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad, void* ctx,
              float* lse, int n_q, int n_keys, int Hq, int Hkv, cudaStream_t st) {
  using SM = Pp<DH>;
  constexpr int BN = SM::BN;
  const int G = Hq / Hkv;
  const int R = 128 / G;
  if (key_pad != nullptr && (reinterpret_cast<uintptr_t>(key_pad) & 15))
    return fail(CC_E_UNSUP, "attention_tc: key_pad must be 16-byte aligned");
  CUtensorMap mq, mk, mv;
  {
    cuuint64_t dims[3] = {(cuuint64_t)DH, (cuuint64_t)Hq, (cuuint64_t)n_q};
    cuuint64_t strides[2] = {(cuuint64_t)DH * 2, (cuuint64_t)Hq * DH * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)R};
    int rc = encode(&mq, 3, q, dims, strides, box);
    if (rc) return rc;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)Hkv * DH, (cuuint64_t)n_keys};
    cuuint64_t strides[1] = {(cuuint64_t)Hkv * DH * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)BN};
    int rc = encode(&mk, 2, k, dims, strides, box);
    if (rc) return rc;
    rc = encode(&mv, 2, v, dims, strides, box);
    if (rc) return rc;
  }
  if (int rc = ensure_smem(attn_pp_kernel<DH, PF, RH>, SM::TOTAL)) return rc;
  const int blocks = (n_q + 2 * R - 1) / (2 * R);
  // key splits when the (group, block) grid leaves SMs idle (see launch<>)
  const int slots = num_sms();
  const int max_tiles = (n_keys + BN - 1) / BN;
  int target = max_tiles, max_parts = 1;
  // few (group, block) items: up to AT_MAXP_EXT key parts, merged by a
  // second kernel (attn_pp_merge) instead of the last part
  static const int ext_env = getenv("CCB_ATTN_EXT") ? atoi(getenv("CCB_ATTN_EXT")) : -1;
  const bool ext = ext_env >= 0 ? ext_env > 0 : Hkv * blocks <= kExtMaxItems;
  if (blocks <= AT_MAXT && max_tiles > 0 && Hkv * blocks < slots) {
    const std::pair<int, int> plan =
        ext ? pp_split_plan(blocks, Hkv, max_tiles, slots, AT_MAXP_EXT, 1.0) : pp_split_plan(blocks, Hkv, max_tiles, slots);
    target = plan.first;
    max_parts = std::min(plan.second, (max_tiles + target - 1) / target);
    if (max_parts < 1) max_parts = 1;
  }
  if (getenv("CCB_ATTN_NOSPLIT")) max_parts = 1;
  if (const char* e = getenv("CCB_ATTN_SPLIT")) {  // experiments: "target,max_parts"
    int a = 0, b = 0;
    if (sscanf(e, "%d,%d", &a, &b) == 2 && a > 0 && b >= 1 && b <= (ext ? AT_MAXP_EXT : AT_MAXP) &&
        blocks <= AT_MAXT) {
      target = a;
      max_parts = b;
    }
  }
  const int pstride = ext ? max_parts : AT_MAXP;
  float* ws_o = nullptr;
  float2* ws_ml = nullptr;
  int* counters = nullptr;
  if (max_parts > 1) {
    const size_t keys = (size_t)Hkv * blocks;
    const size_t bytes = keys * pstride * 256 * (DH * sizeof(float) + sizeof(float2));
    uint8_t* scratch = (uint8_t*)stream_scratch(st, SCR_ATTN, bytes);
    counters = split_counters(st, (int)keys);
    if (!scratch || !counters) return fail(CC_E_CUDA, "attention_tc: split workspace allocation failed");
    ws_o = reinterpret_cast<float*>(scratch);
    ws_ml = reinterpret_cast<float2*>(scratch + keys * pstride * 256 * DH * sizeof(float));
  }
  const bool ext_merge = ext && max_parts > 1;
  dim3 grid(Hkv * blocks * max_parts);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  int rc = launch_k(attn_pp_kernel<DH, PF, RH>, grid, dim3(SM::THREADS), SM::TOTAL, st, "attention_pp", mq, mk, mv,
                    q_slot, key_pad, (__nv_bfloat16*)ctx, lse, n_q, n_keys, Hq, G, scale_log2, Hkv, blocks, target,
                    max_parts, ws_o, ws_ml, counters, pstride, ext_merge ? 1 : 0, g_attn_trace);
  if (rc || !ext_merge) return rc;
  return launch_k(attn_pp_merge<DH>, dim3(Hkv * blocks, DH / 16), dim3(256), 0, st, "attention_pp_merge",
                  (const float*)ws_o, (const float2*)ws_ml, q_slot, (__nv_bfloat16*)ctx, lse, n_q, n_keys, Hq, G,
                  blocks, target, max_parts, pstride);
}

// Kernel shape per launch: 0 = 128-key tiles, two softmax warpgroups (one
// CTA per SM); 1 = 64-key tiles, one warpgroup; 2 = 64-key tiles, two
// warpgroups (both two CTAs per SM); 3 = 128-key tiles, one warpgroup.
template <int DH>
int launch_variant(int variant, const void* q, const void* k, const void* v, const int32_t* q_slot,
                   const uint8_t* key_pad, void* ctx, float* lse, int n_q, int n_keys, int Hq, int Hkv,
                   cudaStream_t st) {
  switch (variant) {
    case 1: return launch<DH, 64, 1>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
    case 2: return launch<DH, 64, 2>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
    case 3: return launch<DH, 128, 1>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
    case 4: return launch_pp<DH>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);



    default: return launch<DH, 128, 2>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
  }
}

}  // namespace

int attention_tc_bf16(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                      void* ctx, float* lse, int n_q, int n_keys, int Hq, int Hkv, int dh, cudaStream_t st) {
  const int G = Hq / Hkv;
  if (G < 1 || G > 128 || (128 % G) != 0) return fail(CC_E_UNSUP, "attention_tc: GQA group must divide 128");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return fail(CC_E_UNSUP, "attention_tc: pointers must be 16-byte aligned");
  int variant = g_attn_variant;
  if (variant < 0) {
    static const int env = getenv("CCB_ATTN_VARIANT") ? atoi(getenv("CCB_ATTN_VARIANT")) : -1;
    variant = env;
  }
  if (variant < 0) {
    // The ping-pong kernel (two Q tiles per CTA share each K/V tile) wins at
    // every measured shape (attn_ab.py, one box): config 2 r = 0.15 63.9 vs
    // 86.5 us (v0), r = 0.05 47.6 vs 57.9, full recompute 220 vs 281 (v1),
    // 32k prompt 1158 vs 1604 (v1), 70B TP rank 144 vs 193 (v1).
    variant = 4;
  }
  if (dh == 128) return launch_variant<128>(variant, q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
  if (dh == 64) return launch_variant<64>(variant, q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
  return fail(CC_E_UNSUP, "attention_tc: d_head must be 64 or 128");
}

}  // namespace ccb

// debug hook (not part of the ABI): per-CTA timeline of the next attention launches
extern "C" __attribute__((visibility("default"))) void cc_debug_attn_trace(void* p) {
  ccb::g_attn_trace = reinterpret_cast<long long*>(p);
}
// debug hook (not part of the ABI): attention kernel shape of the next launches (-1: default)
extern "C" __attribute__((visibility("default"))) void cc_debug_attn_variant(int v) { ccb::g_attn_variant = v; }
