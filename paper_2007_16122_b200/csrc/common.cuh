// common.cuh — device helpers and internal types of libcold (sm_100a).
// Shares nothing with oracle/ (the CPU definition used by the tests).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define COLD_MAX_GROUPS 64
#define COLD_MAX_LAYERS 16

namespace cold {

// ---- scalar definitions used inside the kernels ----------------------------------------

// linear_log (Eq. eq:log; natural log, DESIGN.md AMB-4).
// logf (not __logf): the fp32 path is held to 1e-5 relative.
__device__ __forceinline__ float linear_log(float x) {
  if (x > 1.0f) return logf(x) + 1.0f;
  if (x < -1.0f) return -logf(-x) - 1.0f;
  return x;
}

// PReLU hidden activation: x for x > 0, slope a x otherwise (NaN stays NaN).
__device__ __forceinline__ float prelu(float x, float a) { return x > 0.0f ? x : a * x; }

// sigma, branch form that never overflows expf.
__device__ __forceinline__ float sigmoid(float z) {
  if (z >= 0.0f) return 1.0f / (1.0f + expf(-z));
  float e = expf(z);
  return e / (1.0f + e);
}

// 16-bit storage paths (2e-2 tolerance) use the MUFU intrinsics: __logf has <= 2^-21.4 absolute error on
// the arguments (> 1) it sees here, __expf a few ulp; the fp32 path keeps logf / expf (1e-5 tolerance).
template <bool FAST>
__device__ __forceinline__ float linear_log_t(float x) {
  // branchy on purpose: elements with |x| <= 1 (most single-row sums) skip the MUFU; a branch-free select
  // measured 1.4% slower on the gather (tools/ab_build.sh A/B, sweep s13)
  if constexpr (FAST) {
    const float ax = fabsf(x);
    const float l = __logf(ax) + 1.0f;
    return ax > 1.0f ? copysignf(l, x) : x;
  } else {
    return linear_log(x);
  }
}
template <bool FAST>
__device__ __forceinline__ float sigmoid_t(float z) {
  if constexpr (FAST) return __fdividef(1.0f, 1.0f + __expf(-z));
  else return sigmoid(z);
}

// MurmurHash3 fmix64 and the cross-feature row (DESIGN.md AMB-9):
// row = floor(fmix64(fmix64(x ^ salt_g) ^ y) * C / 2^64), salt_g = (g+1) * 0x9E3779B97F4A7C15.
__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
__device__ __forceinline__ uint64_t cross_salt(int g) { return (uint64_t)(g + 1) * 0x9E3779B97F4A7C15ULL; }
__device__ __forceinline__ int64_t cross_row_from_hx(uint64_t hx, uint64_t y, uint64_t card) {
  return (int64_t)__umul64hi(fmix64(hx ^ y), card);
}

// ---- storage types -------------------------------------------------------------------------
template <typename T> struct Store;
// add(acc, v) = acc + (float)v rounded to nearest: the widening is exact, so this is the fp32 sum the
// oracle's fp32-ordered mode defines; for 16-bit v it is one sm_100 mixed-precision add (FHADD),
// instead of a convert + FADD pair.
template <> struct Store<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
  static __device__ __forceinline__ float add(float acc, float v) { return acc + v; }
};
template <> struct Store<__half> {
  static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }  // RNE, non-saturating
  static __device__ __forceinline__ float add(float acc, __half v) {
    float r;
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(r) : "h"(__half_as_ushort(v)), "f"(acc));
    return r;
  }
};
template <> struct Store<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
  static __device__ __forceinline__ float add(float acc, __nv_bfloat16 v) {
    float r;
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(r) : "h"(__bfloat16_as_ushort(v)), "f"(acc));
    return r;
  }
};

// ---- per-ctx static group description (device resident) ------------------------------------
struct DevGroup {
  const void* table;     // [card][k] in storage dtype
  int64_t card;
  int32_t side;          // 0 user, 1 ad, 2 cross
  int32_t pooled;        // AD: bag
  int32_t user_ref, ad_ref;
  int32_t sel_slot;      // USER: column block in x_u; AD/CROSS: column block in X_ac; -1 = not selected
  int32_t sel_pos;       // position among all selected groups (debug outputs); -1 = not selected
};

// ---- per-call batch view (kernel parameter) -------------------------------------------------
// ids of group g for ad a: ids[a - id_shift] (single) or ids[offs[a - offs_shift] - val_shift + i] (bag).
struct BatchGroup {
  const int32_t* ids;
  const int32_t* offs;
  int64_t id_shift;
  int64_t offs_shift;
  int64_t val_shift;
};
struct BatchView {
  BatchGroup g[COLD_MAX_GROUPS];
};

}  // namespace cold
