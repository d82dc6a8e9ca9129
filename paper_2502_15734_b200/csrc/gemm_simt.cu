// SIMT reference GEMM C = A B^T with the fix-up epilogues, templated on the
// element type.  Used for the f64/f32 parity modes (model.py:399-419 run in
// the reference's own float64) and as the in-library cross-check of the
// tcgen05 bf16 kernel (gemm_tc.cu).  Fixed K order, no split-K: a row's
// result never depends on how many rows are active (M-invariance).
#include "common.cuh"
#include "gemm.cuh"

namespace ccb {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename T, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, int64_t lda,
                                                        const T* __restrict__ B, int64_t ldb, void* C,
                                                        int64_t ldc, int M, int N, int K) {
  using Acc_t = typename Acc<T>::type;
  constexpr bool GLU = EPI == CC_EPI_SWIGLU;
  __shared__ Acc_t As[SB_K][SB_M + 1];
  __shared__ Acc_t Bs[SB_K][SB_N + 1];
  __shared__ Acc_t Bu[GLU ? SB_K : 1][GLU ? SB_N + 1 : 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;  // n0: output column tile
  // in GLU mode output tile [n0, n0+64) reads gate rows 2*n0 + c and up rows 2*n0 + 64 + c
  const int gate_row0 = GLU ? 2 * n0 : n0;
  Acc_t acc[4][4] = {};
  Acc_t accu[GLU ? 4 : 1][GLU ? 4 : 1] = {};
  for (int k0 = 0; k0 < K; k0 += SB_K) {
    for (int i = threadIdx.x; i < SB_M * SB_K; i += 256) {
      int r = i / SB_K, c = i % SB_K;
      int gm = m0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? (Acc_t)to_f(A[(int64_t)gm * lda + gk]) : (Acc_t)0;
      int gn = gate_row0 + r;
      bool okn = GLU ? (n0 + r < N / 2) : (gn < N);
      Bs[c][r] = (okn && gk < K) ? (Acc_t)to_f(B[(int64_t)gn * ldb + gk]) : (Acc_t)0;
      if constexpr (GLU) Bu[c][r] = (okn && gk < K) ? (Acc_t)to_f(B[(int64_t)(gn + 64) * ldb + gk]) : (Acc_t)0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      Acc_t a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
      if constexpr (GLU) {
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bu[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) accu[i][j] += a[i] * b[j];
      }
    }
    __syncthreads();
  }
  const int n_out = GLU ? N / 2 : N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= n_out) continue;
      Acc_t v = acc[i][j];
      int64_t o = (int64_t)m * ldc + n;
      if constexpr (EPI == CC_EPI_RESID_ADD) {
        Acc_t* H = reinterpret_cast<Acc_t*>(C);
        H[o] += v;
      } else {
        if constexpr (EPI == CC_EPI_GELU) v = gelu_tanh(v);
        if constexpr (GLU) v = silu(v) * accu[i][j];
        T* Ct = reinterpret_cast<T*>(C);
        if constexpr (sizeof(Acc_t) == 8) Ct[o] = from_d<T>(v); else Ct[o] = from_f<T>(v);
      }
    }
  }
}

int gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
              int epi, int dtype, cudaStream_t st) {
  if (epi == CC_EPI_SWIGLU) CCB_REQUIRE(N % 128 == 0, "gemm: SWIGLU needs N % 128 == 0 (64-col gate|up groups)");
  note_simt(dtype);
  int n_out = epi == CC_EPI_SWIGLU ? N / 2 : N;
  dim3 grid((n_out + SB_N - 1) / SB_N, (M + SB_M - 1) / SB_M);
  CCB_REQUIRE(grid.y <= 65535, "gemm: M too large");
  return CCB_DISPATCH_DTYPE(dtype, T, [&] {
    switch (epi) {
      case CC_EPI_STORE: gemm_simt_kernel<T, CC_EPI_STORE><<<grid, 256, 0, st>>>((const T*)A, lda, (const T*)B, ldb, C, ldc, M, N, K); break;
      case CC_EPI_RESID_ADD: gemm_simt_kernel<T, CC_EPI_RESID_ADD><<<grid, 256, 0, st>>>((const T*)A, lda, (const T*)B, ldb, C, ldc, M, N, K); break;
      case CC_EPI_SWIGLU: gemm_simt_kernel<T, CC_EPI_SWIGLU><<<grid, 256, 0, st>>>((const T*)A, lda, (const T*)B, ldb, C, ldc, M, N, K); break;
      case CC_EPI_GELU: gemm_simt_kernel<T, CC_EPI_GELU><<<grid, 256, 0, st>>>((const T*)A, lda, (const T*)B, ldb, C, ldc, M, N, K); break;
      default: return fail(CC_E_ARG, "gemm: unknown epilogue");
    }
    return check_launch("gemm_simt");
  });
}

}  // namespace ccb

extern "C" int cc_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N,
                       int K, int epilogue, int dtype, int impl, void* stream) {
  using namespace ccb;
  CCB_REQUIRE(M >= 0 && N > 0 && K > 0, "gemm: bad shape");
  if (M == 0) return 0;
  cudaStream_t st = as_stream(stream);
  // impl: 0 product path (bf16: <= 4 rows -> weight-streaming GEMV, else the
  // tcgen05 kernel with stream-K allowed; an unsupported shape is an error,
  // never a silent SIMT fallback; fp32/fp64 parity modes: SIMT),
  // 1 tcgen05 with stream-K, 4 tcgen05 without split (batch/M-invariant),
  // 2 SIMT reference (tests)
  if (dtype == CC_BF16 && impl == 0 && gemv_eligible(M, N, K, epilogue, A, lda, B, ldb))
    return gemv_bf16(A, lda, B, ldb, C, ldc, M, N, K, epilogue, st);
  if (dtype == CC_BF16 && impl != 2) return gemm_tc_bf16(A, lda, B, ldb, C, ldc, M, N, K, epilogue, impl != 4, st);
  if (impl == 1 || impl == 4) return fail(CC_E_UNSUP, "gemm: tcgen05 kernel requires bf16");
  return gemm_simt(A, lda, B, ldb, C, ldc, M, N, K, epilogue, dtype, st);
}

extern "C" int cc_rope_scatter_qkv(const void* qkv, int64_t ld_qkv, int n_rows, const int32_t* row_slot,
                                   const int32_t* row_pos, const void* rope_table, void* q_rot, void* kv_k, void* kv_v,
                                   void* k_rot, int n_heads, int n_kv_heads, int d_head, int dtype, void* stream);

extern "C" int cc_gemm_qkv_rope(const void* x, int64_t ldx, const void* w_qkv, int64_t ldw, int n_rows, int d,
                                const int32_t* row_slot, const int32_t* row_pos, const void* rope_table, void* q_rot,
                                void* kv_k, void* kv_v, void* k_rot, void* qkv_scratch, int n_heads, int n_kv_heads,
                                int d_head, int dtype, void* stream) {
  using namespace ccb;
  CCB_REQUIRE(n_rows >= 0 && d > 0 && n_heads > 0 && n_kv_heads > 0 && d_head > 0, "gemm_qkv_rope: bad shape");
  if (n_rows == 0) return 0;
  const int N = (n_heads + 2 * n_kv_heads) * d_head;
  if (dtype == CC_BF16) {
    const int rc = gemm_qkv_rope_bf16(x, ldx, w_qkv, ldw, n_rows, d, n_heads, n_kv_heads, d_head, row_slot, row_pos,
                                      rope_table, q_rot, kv_k, kv_v, k_rot, as_stream(stream));
    if (rc != CC_E_UNSUP) return rc;
  }
  // composition: the same GEMM into the qkv rows, then the RoPE / scatter pass
  // (bit-identical to the fused epilogue in bf16)
  CCB_REQUIRE(qkv_scratch != nullptr, "gemm_qkv_rope: shape needs the qkv scratch rows");
  // (bf16, >= 64 rows: no K split, like the fused kernel -- a row's result
  // does not depend on which of the two runs)
  const int impl = dtype == CC_BF16 && n_rows >= 64 ? 4 : 0;
  int rc = cc_gemm(x, ldx, w_qkv, ldw, qkv_scratch, N, n_rows, N, d, CC_EPI_STORE, dtype, impl, stream);
  if (rc) return rc;
  return cc_rope_scatter_qkv(qkv_scratch, N, n_rows, row_slot, row_pos, rope_table, q_rot, kv_k, kv_v, k_rot, n_heads,
                             n_kv_heads, d_head, dtype, stream);
}
