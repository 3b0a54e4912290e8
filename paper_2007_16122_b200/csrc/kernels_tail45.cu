// kernels_tail45.cu — the last two hidden layers and the head of the COLD FC stack in one
// persistent tcgen05 kernel (... x 256 x 128 x 64 x 2; L163 sigma), fed by H3
// from the preceding (CTA-pair) FC3 GEMM:
//
//   H4 = ReLU(H3 W4^T + b4)   (K = 256, N4 = 128)   A = H3 tile (TMA ring), B = W4 resident in smem
//   H5 = ReLU(H4 W5^T + b5)   (K = 128, N5 = 64)    A = H4 in smem (written by the epilogue), B = W5 resident
//   p  = sigma(z1 - z0), z = W6 H5 + b6             epilogue threads, fp32 (DESIGN D-2)
//
// Why a separate kernel: the earlier FC3-FC5 fusion restreamed W3 (256 KB) from L2 for every
// 128-row tile (86 B/cycle/SM of operand traffic) and could not double-buffer FC3's 256-column
// accumulator next to FC4/FC5 in TMEM, so its tensor pipe idled while H3 drained (33% active).
// FC3 now runs as a CTA-pair GEMM at the FC2 rate; here both remaining weights (64 KB + 16 KB) stay
// resident, only H3 streams, and every accumulator is double-buffered (TMEM 2x128 + 2x64 columns):
//   MMA order: FC4(0) | FC4(1) FC5(0) | FC4(2) FC5(1) | ... | FC5(T-1)
// so the tensor pipe runs FC4(t+1) while the epilogue drains acc4(t) into the swizzled H4 tile and
// FC5(t) while it finishes the head of tile t-1.
#include <cuda.h>
#include "internal.h"
#include "ptx.cuh"

namespace cold {

constexpr int Q_EPI_WARPS = 8;
constexpr int Q_THREADS = 64 + 32 * Q_EPI_WARPS;
constexpr int Q_K4 = 256, Q_N4 = 128, Q_N5 = 64;
constexpr int Q_STAGES = 4;   // (5 measured neutral: profiles/r02/ab_t5_*.jsonl)
constexpr int Q_A_BYTES = BM * BK * 2;                  // 16 KB: 128 rows x 64 cols of H3
constexpr int Q_W4_ATOM = Q_N4 * 128;                   // 16 KB: 128 rows x 64 K
constexpr int Q_W4_BYTES = (Q_K4 / BK) * Q_W4_ATOM;     // 64 KB
constexpr int Q_W5_ATOM = Q_N5 * 128;                   // 8 KB: 64 rows x 64 K
constexpr int Q_W5_BYTES = (Q_N4 / BK) * Q_W5_ATOM;     // 16 KB
constexpr int Q_H4_ATOM = BM * 128;                     // 16 KB: 128 rows x 64 cols
constexpr int Q_H4_BYTES = (Q_N4 / BK) * Q_H4_ATOM;     // 32 KB per buffer
constexpr int Q_SMEM = Q_W4_BYTES + Q_W5_BYTES + Q_STAGES * Q_A_BYTES + 2 * Q_H4_BYTES + 1024 + 256;
static_assert(Q_SMEM <= 232448, "tail45 shared memory");

template <bool BF16, bool PRELU>
__global__ void __launch_bounds__(Q_THREADS, 1)
    tail45_kernel(const __grid_constant__ CUtensorMap tmA4, const __grid_constant__ CUtensorMap tmB4,
                  const __grid_constant__ CUtensorMap tmB5, int M, TailParams tp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW4 = smem;
  uint8_t* sW5 = sW4 + Q_W4_BYTES;
  uint8_t* sA = sW5 + Q_W5_BYTES;
  uint8_t* sH4 = sA + Q_STAGES * Q_A_BYTES;               // [2][Q_H4_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH4 + 2 * Q_H4_BYTES);
  uint64_t* full = bars;                       // [Q_STAGES]
  uint64_t* empty = full + Q_STAGES;           // [Q_STAGES]
  uint64_t* wres = empty + Q_STAGES;           // [1] W4 + W5 resident
  uint64_t* tfull4 = wres + 1;                 // [2] acc4 ready
  uint64_t* hready = tfull4 + 2;               // [2] acc4 drained + H4 written (8 warps)
  uint64_t* tfull5 = hready + 2;               // [2] acc5 ready (H4 buffer free again)
  uint64_t* tempty5 = tfull5 + 2;              // [2] acc5 drained (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty5 + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = (M + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Q_STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(wres, 1);
    for (int i = 0; i < 2; i++) {
      mbar_init(&tfull4[i], 1);
      mbar_init(&hready[i], Q_EPI_WARPS);
      mbar_init(&tfull5[i], 1);
      mbar_init(&tempty5[i], Q_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA4) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB4) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB5) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // TMEM columns: acc4[b] at 128 b, acc5[b] at 256 + 64 b
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      // weights do not depend on the previous kernel: load them before the grid dependency wait
      mbar_expect_tx(wres, Q_W4_BYTES + Q_W5_BYTES);
      for (int kb = 0; kb < Q_K4 / BK; kb++) tma_load_2d(sW4 + kb * Q_W4_ATOM, &tmB4, wres, kb * BK, 0, pol_b);
      for (int kb = 0; kb < Q_N4 / BK; kb++) tma_load_2d(sW5 + kb * Q_W5_ATOM, &tmB5, wres, kb * BK, 0, pol_b);
      pdl_wait();
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int tt = tp.reverse ? num_tiles - 1 - t : t;
        for (int kb = 0; kb < Q_K4 / BK; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], Q_A_BYTES);
          tma_load_2d(sA + s * Q_A_BYTES, &tmA4, &full[s], kb * BK, tt * BM, pol_a);
          if (++s == Q_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id4 = idesc_f16<Q_N4, BF16>();
      constexpr uint32_t id5 = idesc_f16<Q_N5, BF16>();
      mbar_wait(wres, 0);
      int s = 0;
      uint32_t ph = 0;
      auto fc5 = [&](int lt) {
        const int b = lt & 1;
        mbar_wait(&hready[b], (lt >> 1) & 1);              // H4(lt) written
        mbar_wait(&tempty5[b], ((lt >> 1) & 1) ^ 1);       // acc5[b] drained (tile lt-2)
        tc_fence_after();
        const uint32_t d = tmem_base + 256 + 64 * b;
        const uint8_t* h4 = sH4 + b * Q_H4_BYTES;
        for (int kb = 0; kb < Q_N4 / BK; kb++) {
          const uint64_t ad = sdesc_sw128(smem_u32(h4 + kb * Q_H4_ATOM));
          const uint64_t bd = sdesc_sw128(smem_u32(sW5 + kb * Q_W5_ATOM));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++)
            umma_f16(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), id5, (kb | kk) != 0);
        }
        umma_commit(&tfull5[b]);
      };
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
        const int b = lt & 1;
        mbar_wait(&hready[b], ((lt >> 1) & 1) ^ 1);        // acc4[b] drained (tile lt-2)
        tc_fence_after();
        const uint32_t d = tmem_base + 128 * b;
        for (int kb = 0; kb < Q_K4 / BK; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * Q_A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sW4 + kb * Q_W4_ATOM));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++)
            umma_f16(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), id4, (kb | kk) != 0);
          umma_commit(&empty[s]);
          if (++s == Q_STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(&tfull4[b]);
        if (lt > 0) fc5(lt - 1);
      }
      if (lt > 0) fc5(lt - 1);
    }
  } else {
    // ===== epilogue warps: quadrant q (TMEM lanes / tile rows), column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    auto epi4 = [&](int lt) {
      const int b = lt & 1;
      mbar_wait(&tfull4[b], (lt >> 1) & 1);
      tc_fence_after();
      // this warp: columns [64 h, 64 h + 64) = atom h of H4 buffer b
      uint32_t v0[32], v1[32];
      TMEM_LD32(lane_base + 128 * b + 64 * h, v0);
      TMEM_LD32(lane_base + 128 * b + 64 * h + 32, v1);
      tmem_wait_ld();
      tc_fence_before();
      uint8_t* atom = sH4 + b * Q_H4_BYTES + h * Q_H4_ATOM;
      const float* bias = tp.b4 + 64 * h;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const uint32_t* v = j < 4 ? v0 : v1;
        const int o = (j & 3) * 8;
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + 8 * j));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + 8 * j + 4));
        uint4 w;
        if constexpr (PRELU) {   // PReLU (F2)
          const float4 a0 = __ldg(reinterpret_cast<const float4*>(tp.s4 + 64 * h + 8 * j));
          const float4 a1 = __ldg(reinterpret_cast<const float4*>(tp.s4 + 64 * h + 8 * j + 4));
          w.x = Pack<BF16>::two(prelu(__uint_as_float(v[o + 0]) + b0.x, a0.x), prelu(__uint_as_float(v[o + 1]) + b0.y, a0.y));
          w.y = Pack<BF16>::two(prelu(__uint_as_float(v[o + 2]) + b0.z, a0.z), prelu(__uint_as_float(v[o + 3]) + b0.w, a0.w));
          w.z = Pack<BF16>::two(prelu(__uint_as_float(v[o + 4]) + b1.x, a1.x), prelu(__uint_as_float(v[o + 5]) + b1.y, a1.y));
          w.w = Pack<BF16>::two(prelu(__uint_as_float(v[o + 6]) + b1.z, a1.z), prelu(__uint_as_float(v[o + 7]) + b1.w, a1.w));
        } else {
          w.x = Pack<BF16>::two_relu(__uint_as_float(v[o + 0]) + b0.x, __uint_as_float(v[o + 1]) + b0.y);
          w.y = Pack<BF16>::two_relu(__uint_as_float(v[o + 2]) + b0.z, __uint_as_float(v[o + 3]) + b0.w);
          w.z = Pack<BF16>::two_relu(__uint_as_float(v[o + 4]) + b1.x, __uint_as_float(v[o + 5]) + b1.y);
          w.w = Pack<BF16>::two_relu(__uint_as_float(v[o + 6]) + b1.z, __uint_as_float(v[o + 7]) + b1.w);
        }
        sts128(smem_u32(atom) + sw128_offset(r, j), w);
      }
      fence_async_smem();      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&hready[b]);
    };
    auto epi5 = [&](int lt, int tile) {
      const int b = lt & 1;
      mbar_wait(&tfull5[b], (lt >> 1) & 1);
      tc_fence_after();
      if (h == 0) {                               // one warp per quadrant owns the row's head dot product
        uint32_t v0[32], v1[32];
        TMEM_LD32(lane_base + 256 + 64 * b, v0);
        TMEM_LD32(lane_base + 256 + 64 * b + 32, v1);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty5[b]);
        float z0 = 0.0f, z1 = 0.0f;
#pragma unroll
        for (int i = 0; i < 64; i++) {
          const float x5 = __uint_as_float(i < 32 ? v0[i] : v1[i - 32]) + __ldg(tp.b5 + i);
          float a;
          if constexpr (PRELU) a = prelu(x5, __ldg(tp.s5 + i));
          else a = fmaxf(x5, 0.0f);
          z0 = fmaf(__ldg(tp.head_w + i), a, z0);
          if (tp.head_n == 2) z1 = fmaf(__ldg(tp.head_w + Q_N5 + i), a, z1);
        }
        const int row = tile * BM + r;
        if (row < M) {
          const float z = (tp.head_n == 2) ? (z1 + tp.head_b[1]) - (z0 + tp.head_b[0]) : z0 + tp.head_b[0];
          tp.scores[row] = sigmoid(z);
        }
      } else {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty5[b]);
      }
    };
    int lt = 0, prev_tile = -1;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
      epi4(lt);
      if (lt > 0) epi5(lt - 1, prev_tile);
      prev_tile = tp.reverse ? num_tiles - 1 - t : t;
    }
    if (lt > 0) epi5(lt - 1, prev_tile);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

bool tail45_supported(int n4, int n5, int k4) { return n4 == Q_N4 && n5 == Q_N5 && k4 == Q_K4; }

cudaError_t launch_tail45(const CUtensorMap* tmA4, const CUtensorMap* tmB4, const CUtensorMap* tmB5, int M, int bf16,
                          const TailParams& tp, int num_sms, bool pdl, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const bool pr = tp.s4 != nullptr;
  auto kern = bf16 ? (pr ? tail45_kernel<true, true> : tail45_kernel<true, false>)
                   : (pr ? tail45_kernel<false, true> : tail45_kernel<false, false>);
  static DevOnce attr[4];
  if (attr[(bf16 ? 2 : 0) + (pr ? 1 : 0)].first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_SMEM);
  }
  const int tiles = (M + BM - 1) / BM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles < num_sms ? tiles : num_sms);
  cfg.blockDim = dim3(Q_THREADS);
  cfg.dynamicSmemBytes = Q_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, *tmA4, *tmB4, *tmB5, M, tp);
}

}  // namespace cold
