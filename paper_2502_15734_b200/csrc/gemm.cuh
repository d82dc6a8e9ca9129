#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cachecraft_b200.h"

namespace ccb {

// Tensor-parallel peer tables (symmetric buffers of every rank, device
// pointers valid in this process: P2P / CUDA-IPC mapped) for the fused
// GEMM -> reduce-scatter push (CC_EPI_PEER_PUSH) and the tp_reduce kernels.
constexpr int CC_EPI_PEER_PUSH = 4;
constexpr int TP_MAX = 8;
using PeerTab = cc_tp_peers;  // include/cachecraft_b200.h
int gemm_tc_peer_push(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                      const PeerTab& tab, cudaStream_t st);
int gemm_tc_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
                 int epi, bool allow_split, cudaStream_t st);
int gemm_simt(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int M, int N, int K,
              int epi, int dtype, cudaStream_t st);
int gemm_qkv_rope_bf16(const void* X, int64_t ldx, const void* Wqkv, int64_t ldw, int M, int K, int Hq, int Hkv,
                       int d_head, const int32_t* row_slot, const int32_t* row_pos, const void* table, void* q_rot,
                       void* kv_k, void* kv_v, void* k_rot, cudaStream_t st);
int logits_stream_bf16(const float* hidden, const float* norm_w, float eps, const void* U, float* logits, int d,
                       int vocab, cudaStream_t st);
bool gemv_eligible(int M, int N, int K, int epi, const void* A, int64_t lda, const void* W, int64_t ldw);
int gemv_bf16(const void* A, int64_t lda, const void* W, int64_t ldw, void* C, int64_t ldc, int M, int N, int K,
              int epi, cudaStream_t st);
}  // namespace ccb
