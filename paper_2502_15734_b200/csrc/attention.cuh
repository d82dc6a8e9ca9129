#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ccb {
int attention_tc_bf16(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                      void* ctx, float* lse, int n_q, int n_keys, int Hq, int Hkv, int dh, cudaStream_t st);
int segment_mass_tc_bf16(const void* q, const void* k, const int32_t* q_slot, const uint8_t* key_pad,
                         const float* lse, const int32_t* seg_lo, const int32_t* seg_hi, int n_seg,
                         const int32_t* rows, int n_rows, double* mass, int n_keys, int Hq, int Hkv, int dh,
                         cudaStream_t st);
int attention_simt(const void* q, const void* k, const void* v, const int32_t* q_slot, const uint8_t* key_pad,
                   void* ctx, void* lse, int n_q, int n_keys, int Hq, int Hkv, int dh, int dtype, cudaStream_t st);
}  // namespace ccb
