#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ccb {
int gemm_tc_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
                 int epi, bool allow_split, cudaStream_t st);
int gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
              int epi, int dtype, cudaStream_t st);
bool gemv_eligible(int M, int N, int K, int epi, const void* A, int64_t lda, const void* W, int64_t ldw);
int gemv_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
              int epi, cudaStream_t st);
}  // namespace ccb
