// epi.cuh — the store-mode epilogue shared by the tcgen05 GEMM kernels (sm_100a).
//
// One epilogue warp drains its 32 accumulator rows (TMEM lanes of its quadrant) x 64 columns at a
// time: two tcgen05.ld 32x32b.x32 in flight, + bias or + u1[request] (fp32), ReLU, RNE pack, one
// 32-row x 64-col box written in the 128 B-swizzled layout (full 128 B lines per row), one TMA store.
// Versus 32-column boxes with 64 B rows this halves the TMEM waits, fences, warp syncs and TMA
// stores per output and gives the TMA unit whole lines (FC1's epilogue was the kernel's bottleneck:
// 95 us per 151,552-ad chunk with the MMAs disabled vs 65 us for the MMA main loop alone).
#pragma once
#include "ptx.cuh"

namespace cold {

constexpr int EPI_WIDE_COLS = 64;
constexpr int EPI_WIDE_BOX = 32 * EPI_WIDE_COLS * 2;   // 4 KB, single-buffered per warp

template <bool BF16>
__device__ __forceinline__ void epi_store_wide(uint32_t taddr, int c_begin, int c_end, const float* __restrict__ bias,
                                               uint32_t u1s, const float* __restrict__ u1g, int relu, uint8_t* buf,
                                               const CUtensorMap* tmC, int col_base, int row0, int lane,
                                               int dbg = 0, unsigned long long* tacc = nullptr) {
  const uint32_t sbuf = smem_u32(buf);
  // debug timing (tacc != null, lane 0): cycles in [0] TMEM load+wait, [1] math+pack, [2] wait for the
  // staging buffer, [3] smem writes + fence, [4] store issue
  long long tc0 = 0, tsum[5] = {0, 0, 0, 0, 0};
  auto tick = [&](int k) {
    if (tacc) { const long long t = clock64(); if (k >= 0) tsum[k] += t - tc0; tc0 = t; }
  };
  tick(-1);
  for (int c = c_begin; c < c_end; c += EPI_WIDE_COLS) {
    uint32_t v[64];
    if (dbg != 5) {
      TMEM_LD32(taddr + c, v);
      TMEM_LD32(taddr + c + 32, (v + 32));
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < 64; i++) v[i] = (uint32_t)(lane + i);
    }
    tick(0);
    const int col0 = col_base + c;
    float f[64];
#pragma unroll
    for (int i = 0; i < 64; i++) f[i] = __uint_as_float(v[i]);
    if (bias) {
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col0 + i));
        f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
      }
    }
    if (u1s) {
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 b = lds128f(u1s + (uint32_t)(c + i) * 4u);
        f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
      }
    } else if (u1g) {
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(u1g + c + i));
        f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
      }
    }
    uint32_t pk[32];
    if (relu) {
#pragma unroll
      for (int i = 0; i < 32; i++) pk[i] = Pack<BF16>::two_relu(f[2 * i], f[2 * i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; i++) pk[i] = Pack<BF16>::two(f[2 * i], f[2 * i + 1]);
    }
    if (dbg == 3) {                       // timing experiment: no smem staging / store
      uint32_t t = 0;
#pragma unroll
      for (int i = 0; i < 32; i++) t ^= pk[i];
      if (t == 0x12345678u) asm volatile("st.global.u32 [%0], %1;" ::"l"(bias), "r"(t));
      continue;
    }
    tick(1);
    if (lane == 0) bulk_wait_read<0>();   // the previous box of this warp has left shared memory
    __syncwarp();
    tick(2);
    const uint32_t rowp = sbuf + (uint32_t)lane * 128u;
#pragma unroll
    for (int j = 0; j < 8; j++)
      sts128(rowp + (uint32_t)((j ^ (lane & 7)) << 4), make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
    fence_async_smem();
    __syncwarp();
    tick(3);
    if (lane == 0 && dbg != 4) {
      tma_store_2d(tmC, buf, col0, row0);
      bulk_commit();
    }
    tick(4);
  }
  if (tacc && lane == 0)
    for (int k = 0; k < 5; k++) atomicAdd(tacc + k, (unsigned long long)tsum[k]);
}

}  // namespace cold
