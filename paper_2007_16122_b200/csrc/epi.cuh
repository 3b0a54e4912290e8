// epi.cuh — the store-mode epilogue shared by the tcgen05 GEMM kernels (sm_100a).
//
// Each epilogue warp drains its 32 accumulator rows (TMEM lanes of its quadrant q) x 64 columns at a
// time: two tcgen05.ld 32x32b.x32 in flight, + bias or + u1[request] (fp32), ReLU fused into the RNE
// pack, and its 32 rows written into a 128-row x 64-column box in the 128 B-swizzled layout (full
// 128 B lines). The four quadrant warps of a column half form a group (named barrier 1 + h): once all
// four have written, one elected thread issues ONE 16 KB TMA store for the group. Timing of the FC1
// epilogue (tools/probes/epi_instr.py) showed the warps waiting ~40% of their time for their own
// 4 KB stores to drain: the TMA unit, shared with the operand loads, was limited by store count.
#pragma once
#include "ptx.cuh"

namespace cold {

constexpr int EPI_WIDE_COLS = 64;
constexpr int EPI_WIDE_BOX = 32 * EPI_WIDE_COLS * 2;   // 4 KB: one warp's rows of the group box
constexpr int EPI_GROUP_BOX = 4 * EPI_WIDE_BOX;        // 16 KB: 128 rows x 64 columns, single-buffered

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// group_buf: the group's 16 KB box (128 rows x 128 B, SW128, 1024 B aligned); q: this warp's quadrant;
// h: the column half (group id); tile_row0: the tile's first row (the box origin).
template <bool BF16>
__device__ __forceinline__ void epi_store_wide(uint32_t taddr, int c_begin, int c_end, const float* __restrict__ bias,
                                               uint32_t u1s, const float* __restrict__ u1g, int relu,
                                               uint8_t* group_buf, const CUtensorMap* tmC, int col_base,
                                               int tile_row0, int q, int h, int lane, int dbg = 0,
                                               unsigned long long* tacc = nullptr, void* gout = nullptr,
                                               int ldo = 0, int M = 0, uint64_t store_policy = 0,
                                               const float* __restrict__ slope = nullptr,
                                               uint8_t* group_buf2 = nullptr, int* box_ctr = nullptr) {
  // group_buf2 / box_ctr (optional): a second staging box; consecutive 64-column chunks alternate between
  // the two so the math of chunk c + 1 overlaps the TMA store of chunk c (box_ctr: running chunk count of
  // the group, identical in its four warps)
  const bool elected = (q == 0) && (lane == 0);
  // debug timing (tacc != null, lane 0): cycles in [0] TMEM load+wait, [1] math+pack, [2] wait for the
  // staging buffer, [3] smem writes, [4] store issue, [5] proxy fence, [6] group barrier after the writes
  long long tc0 = 0, tsum[7] = {0, 0, 0, 0, 0, 0, 0};
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
    if (slope) {                          // PReLU (F2): per-column slope, then the plain RNE pack
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(slope + col0 + i));
        f[i] = prelu(f[i], a.x); f[i + 1] = prelu(f[i + 1], a.y);
        f[i + 2] = prelu(f[i + 2], a.z); f[i + 3] = prelu(f[i + 3], a.w);
      }
#pragma unroll
      for (int i = 0; i < 32; i++) pk[i] = Pack<BF16>::two(f[2 * i], f[2 * i + 1]);
    } else if (relu) {
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
    if (gout) {                           // direct mode: this lane's row, 128 B, four 256-bit stores
      const int row = tile_row0 + q * 32 + lane;
      if (row < M) {
        uint16_t* dst = reinterpret_cast<uint16_t*>(gout) + (int64_t)row * ldo + col0;
#pragma unroll
        for (int j = 0; j < 4; j++)
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 16 * j), "r"(pk[8 * j]),
                       "r"(pk[8 * j + 1]), "r"(pk[8 * j + 2]), "r"(pk[8 * j + 3]), "r"(pk[8 * j + 4]),
                       "r"(pk[8 * j + 5]), "r"(pk[8 * j + 6]), "r"(pk[8 * j + 7])
                       : "memory");
      }
      tick(4);
      continue;
    }
    uint8_t* gbuf = group_buf;
    if (group_buf2) {
      gbuf = (*box_ctr & 1) ? group_buf2 : group_buf;
      ++*box_ctr;
      if (elected) bulk_wait_read<1>();   // the store issued two chunks ago (same box) has left smem
    } else {
      if (elected) bulk_wait_read<0>();   // the group's previous box has left shared memory
    }
    named_bar_sync(1 + h, 128);
    tick(2);
    const uint32_t sbuf = smem_u32(gbuf) + (uint32_t)q * EPI_WIDE_BOX;
    const uint32_t rowp = sbuf + (uint32_t)lane * 128u;
#pragma unroll
    for (int j = 0; j < 8; j++)
      sts128(rowp + (uint32_t)((j ^ (lane & 7)) << 4), make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
    tick(3);
    fence_async_smem();
    tick(5);
    named_bar_sync(1 + h, 128);           // all 128 rows of the box written
    tick(6);
    if (elected && dbg != 4) {
      // dbg 6 (timing experiment): every box to the same L2-resident location (no DRAM write traffic)
      if (store_policy) tma_store_2d_hint(tmC, gbuf, col0, tile_row0, store_policy);
      else tma_store_2d(tmC, gbuf, dbg == 6 ? 0 : col0, dbg == 6 ? 0 : tile_row0);
      bulk_commit();
    }
    tick(4);
  }
  if (tacc && lane == 0)
    for (int k = 0; k < 7; k++) atomicAdd(tacc + k, (unsigned long long)tsum[k]);
}

}  // namespace cold
