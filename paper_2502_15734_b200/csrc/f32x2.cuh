// Packed f32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100) and 2^x for a
// pair on the FMA pipe: shared by the attention kernel (softmax) and the K8
// statistics kernel, where part of the exponentials are moved off the MUFU.
#pragma once
#include <stdint.h>

namespace ccb {

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// 2^x for a pair on the FMA pipe (x <= 0), same arithmetic as ex2_poly
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float x0, x1;
  f2_unpack(x2, x0, x1);
  const uint64_t xc = f2_pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t t = fadd2(xc, f2_pack(12582912.f, 12582912.f));                        // rounds to an integer
  const uint64_t nn = ffma2(t, f2_pack(-1.f, -1.f), f2_pack(12582912.f, 12582912.f));  // -n
  const uint64_t f = fadd2(xc, nn);                                                      // x - n
  uint64_t p = ffma2(f, f2_pack(0.05550410866f, 0.05550410866f), f2_pack(0.2402265070f, 0.2402265070f));
  p = ffma2(f, p, f2_pack(0.6931471806f, 0.6931471806f));
  p = ffma2(f, p, f2_pack(1.f, 1.f));
  float p0, p1, t0, t1;
  f2_unpack(p, p0, p1);
  f2_unpack(t, t0, t1);
  p0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
  return f2_pack(p0, p1);
}


}  // namespace ccb
