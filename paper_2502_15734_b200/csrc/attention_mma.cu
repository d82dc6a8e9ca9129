// K4 bf16 attention for the recomputed (scattered) query rows, flash-style
// online softmax on warp-level tensor-core MMAs (m16n8k16, fp32 accumulate).
// Semantics: model.py:406-416 — query row r attends to keys j <= q_slot[r]
// that are not pads; all rows of a GQA group share the K/V tile.
//
// CTA = 4 warps = 64 "M-rows"; an M-row is a (query row, q head) pair of the
// CTA's kv head g: M-row m -> row row0 + m / G, head g*G + m % G (G = Hq/Hkv),
// so one K/V tile in shared memory serves every head of the group.
// K/V tiles of 64 keys are double-buffered with cp.async.
#include <math.h>

#include "attention.cuh"
#include "common.cuh"

namespace ccb {

namespace {

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s_u32(smem)), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

constexpr int ABN = 64;  // keys per tile

template <int DH>
__global__ void __launch_bounds__(128) attn_mma_kernel(const __nv_bfloat16* __restrict__ q,
                                                       const __nv_bfloat16* __restrict__ k,
                                                       const __nv_bfloat16* __restrict__ v,
                                                       const int32_t* __restrict__ q_slot,
                                                       const uint8_t* __restrict__ key_pad,
                                                       __nv_bfloat16* __restrict__ ctx, float* __restrict__ lse,
                                                       int n_q, int n_keys, int Hq, int Hkv, int G, float scale_log2) {
  constexpr int LDS = DH + 8;
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* Ks = Qs + 64 * LDS;
  __nv_bfloat16* Vs = Ks + 2 * ABN * LDS;
  __shared__ int lim_s[64];
  __shared__ int kmax_s, kmin_s;

  const int g = blockIdx.y;
  const int R = 64 / G;
  const int row0 = blockIdx.x * R;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) { kmax_s = -1; kmin_s = 0x7fffffff; }
  for (int c = tid; c < 64 * CH; c += 128) {
    int mr = c / CH, ch = c % CH;
    int r = row0 + mr / G, h = g * G + mr % G;
    bool ok = r < n_q;
    const __nv_bfloat16* src = ok ? q + ((int64_t)r * Hq + h) * DH + ch * 8 : q;
    cp_async16(Qs + mr * LDS + ch * 8, src, ok);
  }
  cp_commit();
  __syncthreads();
  if (tid < 64) {
    int r = row0 + tid / G;
    int lim = r < n_q ? q_slot[r] : -1;
    lim_s[tid] = lim;
    if (lim >= 0) { atomicMax(&kmax_s, lim); atomicMin(&kmin_s, lim); }
  }
  __syncthreads();
  const int kmax = kmax_s;
  const int n_tiles = kmax < 0 ? 0 : kmax / ABN + 1;

  auto load_kv = [&](int t, int stage) {
    __nv_bfloat16* ks = Ks + stage * ABN * LDS;
    __nv_bfloat16* vs = Vs + stage * ABN * LDS;
    for (int c = tid; c < ABN * CH; c += 128) {
      int rr = c / CH, ch = c % CH;
      int key = t * ABN + rr;
      bool ok = key < n_keys;
      int64_t off = ((int64_t)key * Hkv + g) * DH + ch * 8;
      cp_async16(ks + rr * LDS + ch * 8, ok ? k + off : k, ok);
      cp_async16(vs + rr * LDS + ch * 8, ok ? v + off : v, ok);
    }
  };
  if (n_tiles > 0) load_kv(0, 0);
  cp_commit();

  const int mr_a = warp * 16 + (lane >> 2), mr_b = mr_a + 8;
  const int lim_a = lim_s[mr_a], lim_b = lim_s[mr_b];
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;

  cp_wait<1>();  // Q landed
  __syncthreads();
  uint32_t qf[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    uint32_t addr = s_u32(Qs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
    ldsm_x4(addr, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
  }

  for (int t = 0; t < n_tiles; ++t) {
    const int stage = t & 1;
    if (t + 1 < n_tiles) load_kv(t + 1, stage ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* ks = Ks + stage * ABN * LDS;
    const __nv_bfloat16* vs = Vs + stage * ABN * LDS;
    float s[ABN / 8][4];
#pragma unroll
    for (int i = 0; i < ABN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int n2 = 0; n2 < ABN / 16; ++n2) {
        uint32_t b0, b1, b2, b3;
        int key = n2 * 16 + (lane & 7) + ((lane >> 4) << 3);
        int dim = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(s_u32(ks + key * LDS + dim), b0, b1, b2, b3);
        mma16816(s[2 * n2], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
        mma16816(s[2 * n2 + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
      }
    }
    // mask + online softmax (rows a = lane/4, b = lane/4 + 8 of this warp)
    float tmax_a = -INFINITY, tmax_b = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < ABN / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int j = t * ABN + nt * 8 + (lane & 3) * 2 + e;
        bool padj = (j >= n_keys) || (key_pad != nullptr && key_pad[j]);
        if (padj || j > lim_a) s[nt][e] = -INFINITY;
        if (padj || j > lim_b) s[nt][2 + e] = -INFINITY;
        tmax_a = fmaxf(tmax_a, s[nt][e]);
        tmax_b = fmaxf(tmax_b, s[nt][2 + e]);
      }
    }
#pragma unroll
    for (int o2 = 1; o2 <= 2; o2 <<= 1) {
      tmax_a = fmaxf(tmax_a, __shfl_xor_sync(0xffffffffu, tmax_a, o2));
      tmax_b = fmaxf(tmax_b, __shfl_xor_sync(0xffffffffu, tmax_b, o2));
    }
    const float mn_a = fmaxf(m_a, tmax_a), mn_b = fmaxf(m_b, tmax_b);
    const float alpha_a = (mn_a == -INFINITY || m_a == -INFINITY) ? (mn_a == -INFINITY ? 1.f : 0.f)
                                                                  : exp2f((m_a - mn_a) * scale_log2);
    const float alpha_b = (mn_b == -INFINITY || m_b == -INFINITY) ? (mn_b == -INFINITY ? 1.f : 0.f)
                                                                  : exp2f((m_b - mn_b) * scale_log2);
    const float base_a = mn_a == -INFINITY ? 0.f : mn_a * scale_log2;
    const float base_b = mn_b == -INFINITY ? 0.f : mn_b * scale_log2;
    float rs_a = 0.f, rs_b = 0.f;
#pragma unroll
    for (int nt = 0; nt < ABN / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float pa = s[nt][e] == -INFINITY ? 0.f : exp2f(s[nt][e] * scale_log2 - base_a);
        float pb = s[nt][2 + e] == -INFINITY ? 0.f : exp2f(s[nt][2 + e] * scale_log2 - base_b);
        s[nt][e] = pa;
        s[nt][2 + e] = pb;
        rs_a += pa;
        rs_b += pb;
      }
    }
    l_a = l_a * alpha_a + rs_a;
    l_b = l_b * alpha_b + rs_b;
    m_a = mn_a;
    m_b = mn_b;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= alpha_a; o[i][1] *= alpha_a;
      o[i][2] *= alpha_b; o[i][3] *= alpha_b;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < ABN / 16; ++kk) {
      uint32_t a0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      uint32_t a1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      uint32_t a2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      uint32_t a3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int d2 = 0; d2 < DH / 16; ++d2) {
        uint32_t b0, b1, b2, b3;
        int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int dim = d2 * 16 + (lane >> 4) * 8;
        ldsm_x4_t(s_u32(vs + key * LDS + dim), b0, b1, b2, b3);
        mma16816(o[2 * d2], a0, a1, a2, a3, b0, b1);
        mma16816(o[2 * d2 + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int o2 = 1; o2 <= 2; o2 <<= 1) {
    l_a += __shfl_xor_sync(0xffffffffu, l_a, o2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, o2);
  }
  const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f, inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
  const int ra = row0 + mr_a / G, ha = g * G + mr_a % G;
  const int rb = row0 + mr_b / G, hb = g * G + mr_b % G;
  const float ln2 = 0.6931471805599453f;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    int dim = i * 8 + (lane & 3) * 2;
    if (ra < n_q)
      *reinterpret_cast<uint32_t*>(ctx + ((int64_t)ra * Hq + ha) * DH + dim) = pack_bf16(o[i][0] * inv_a, o[i][1] * inv_a);
    if (rb < n_q)
      *reinterpret_cast<uint32_t*>(ctx + ((int64_t)rb * Hq + hb) * DH + dim) = pack_bf16(o[i][2] * inv_b, o[i][3] * inv_b);
  }
  if ((lane & 3) == 0) {
    if (ra < n_q) lse[(int64_t)ra * Hq + ha] = l_a > 0.f ? (m_a * scale_log2 + log2f(l_a)) * ln2 : -INFINITY;
    if (rb < n_q) lse[(int64_t)rb * Hq + hb] = l_b > 0.f ? (m_b * scale_log2 + log2f(l_b)) * ln2 : -INFINITY;
  }
}

template <int DH>
int launch_attn(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad, void* ctx,
                float* lse, int n_q, int n_keys, int Hq, int Hkv, cudaStream_t st) {
  const int G = Hq / Hkv;
  const int R = 64 / G;
  const size_t smem = (size_t)(64 + 4 * ABN) * (DH + 8) * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_mma_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((n_q + R - 1) / R, Hkv);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  attn_mma_kernel<DH><<<grid, 128, smem, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                (const __nv_bfloat16*)v, q_slot, key_pad, (__nv_bfloat16*)ctx, lse,
                                                n_q, n_keys, Hq, Hkv, G, scale_log2);
  return check_launch("attention_mma");
}

}  // namespace

int attention_mma_bf16(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                       void* ctx, float* lse, int n_q, int n_keys, int Hq, int Hkv, int dh, cudaStream_t st) {
  const int G = Hq / Hkv;
  if (G < 1 || G > 64 || (64 % G) != 0) return fail(CC_E_UNSUP, "attention_mma: GQA group must divide 64");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return fail(CC_E_UNSUP, "attention_mma: pointers must be 16-byte aligned");
  if (dh == 128) return launch_attn<128>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
  if (dh == 64) return launch_attn<64>(q, k, v, q_slot, key_pad, ctx, lse, n_q, n_keys, Hq, Hkv, st);
  return fail(CC_E_UNSUP, "attention_mma: d_head must be 64 or 128");
}

}  // namespace ccb
