// kernels_tail.cu — the last three hidden layers and the head of the COLD FC stack in one
// persistent tcgen05 kernel (... x 256 x 128 x 64 x 2; L163 sigma):
//
//   H3 = ReLU(H2 W3^T + b3)   (K3 = 512, N3 = 256)   A = H2 tile from HBM/L2 (TMA), B = W3 (TMA)
//   H4 = ReLU(H3 W4^T + b4)   (N4 = 128)             A = H3 in TMEM,            B = W4 (TMA)
//   H5 = ReLU(H4 W5^T + b5)   (N5 = 64)              A = H4 in TMEM,            B = W5 (TMA)
//   p  = sigma(z1 - z0), z = W6 H5 + b6              in the epilogue threads, fp32
//
// Per 128-row tile only the fp32 score leaves the SM. Accumulators live in TMEM at columns [0,256) /
// [256,384) / [384,448); the epilogue writes H3 (16-bit, two per column) back over acc3's columns
// [0,128) and H4 over acc4's [256,320) once both warps of a lane quadrant have read them, and FC4 / FC5
// take their A operand from there (tcgen05.mma with A in tensor memory: tools/probes/umma_ts_probe.cu).
// Shared memory then holds only the stage ring (4 stages of 48 KB instead of 2 beside 96 KB of H3 / H4
// tiles). The single MMA thread
// interleaves two tiles so the tensor pipe works on FC3(t+1) while the epilogue drains FC4(t):
//   FC3(0) | FC4(0) FC3(1) | FC5(0) FC4(1) FC3(2) | FC5(1) ...
// (each FC4 / FC5 waits for the epilogue to have written its A operand; the producer fills the
// stage ring in exactly that order).
#include <cuda.h>
#include "internal.h"
#include "ptx.cuh"

namespace cold {

constexpr int T_EPI_WARPS = 8;
constexpr int T_THREADS = 64 + 32 * T_EPI_WARPS;
constexpr int T_N3 = 256, T_N4 = 128, T_N5 = 64;
constexpr int T_STAGES = 4;
constexpr int T_A_BYTES = BM * BK * 2;                  // 16 KB
constexpr int T_B_BYTES = T_N3 * BK * 2;                // 32 KB (largest B k-block)
constexpr int T_STAGE_BYTES = T_A_BYTES + T_B_BYTES;    // 48 KB
constexpr int T_SMEM = T_STAGES * T_STAGE_BYTES + 1024 + 256;

template <bool BF16>
__global__ void __launch_bounds__(T_THREADS, 1)
    tail_kernel(const __grid_constant__ CUtensorMap tmA3, const __grid_constant__ CUtensorMap tmB3,
                const __grid_constant__ CUtensorMap tmB4, const __grid_constant__ CUtensorMap tmB5, int M, int K3,
                TailParams tp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T_STAGES * T_STAGE_BYTES);
  uint64_t* full = bars;                 // [T_STAGES]
  uint64_t* empty = bars + T_STAGES;     // [T_STAGES]
  uint64_t* tfull = bars + 2 * T_STAGES; // [3]: FC3, FC4, FC5 accumulators ready
  uint64_t* hready = tfull + 3;          // [2]: H3, H4 written into TMEM (and acc3 / acc4 drained)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hready + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = (M + BM - 1) / BM;
  const int kb3 = K3 / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < T_STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 3; i++) mbar_init(&tfull[i], 1);
    for (int i = 0; i < 2; i++) mbar_init(&hready[i], T_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA3) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB3) : "memory");
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
  pdl_launch_dependents();
  if (warp != 0) pdl_wait();   // PDL (the producer first issues the weight loads that do not depend on it)

  // the per-CTA op sequence (producer and MMA walk it identically):
  //   t = 0: FC3(0) FC4(0);  t >= 1: FC3(t) FC5(t-1) FC4(t);  end: FC5(T-1)
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      auto next = [&]() { if (++s == T_STAGES) { s = 0; ph ^= 1; } };
      // the first tile's first T_STAGES W3 k-blocks before the dependency wait
      int pre = (int)blockIdx.x < num_tiles ? (kb3 < T_STAGES ? kb3 : T_STAGES) : 0;
      for (int kb = 0; kb < pre; kb++) {
        mbar_expect_tx(&full[kb], T_STAGE_BYTES);
        tma_load_2d(sStage + kb * T_STAGE_BYTES + T_A_BYTES, &tmB3, &full[kb], kb * BK, 0, pol_b);
      }
      pdl_wait();
      auto load_fc3 = [&](int mb) {
        for (int kb = 0; kb < kb3; kb++) {
          if (pre > 0) {   // W3 already in flight for this stage
            tma_load_2d(sStage + s * T_STAGE_BYTES, &tmA3, &full[s], kb * BK, mb * BM, pol_a);
            pre--;
            next();
            continue;
          }
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], T_STAGE_BYTES);
          tma_load_2d(sStage + s * T_STAGE_BYTES, &tmA3, &full[s], kb * BK, mb * BM, pol_a);
          tma_load_2d(sStage + s * T_STAGE_BYTES + T_A_BYTES, &tmB3, &full[s], kb * BK, 0, pol_b);
          next();
        }
      };
      auto load_b = [&](const CUtensorMap* map, int kbs, int rows) {
        for (int kb = 0; kb < kbs; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], (uint32_t)(rows * BK * 2));
          tma_load_2d(sStage + s * T_STAGE_BYTES + T_A_BYTES, map, &full[s], kb * BK, 0, pol_b);
          next();
        }
      };
      int prev = -1;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        load_fc3(t);
        if (prev >= 0) load_b(&tmB5, T_N4 / BK, T_N5);
        load_b(&tmB4, T_N3 / BK, T_N4);
        prev = t;
      }
      if (prev >= 0) load_b(&tmB5, T_N4 / BK, T_N5);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id3 = idesc_f16<T_N3, BF16>();
      constexpr uint32_t id4 = idesc_f16<T_N4, BF16>();
      constexpr uint32_t id5 = idesc_f16<T_N5, BF16>();
      const uint32_t acc3 = tmem_base, acc4 = tmem_base + T_N3, acc5 = tmem_base + T_N3 + T_N4;
      int s = 0;
      uint32_t ph = 0;
      auto next = [&]() { if (++s == T_STAGES) { s = 0; ph ^= 1; } };
      auto mma_fc3 = [&]() {
        for (int kb = 0; kb < kb3; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sStage + s * T_STAGE_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sStage + s * T_STAGE_BYTES + T_A_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++)
            umma_f16(acc3, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), id3, (kb | kk) != 0);
          umma_commit(&empty[s]);
          next();
        }
        umma_commit(&tfull[0]);
      };
      // A (H3 / H4) from TMEM column tA: 16 K elements = 8 columns per MMA
      auto mma_from_tmem = [&](uint32_t tA, int kbs, uint32_t acc, uint32_t idesc, uint64_t* done) {
        for (int kb = 0; kb < kbs; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t bd = sdesc_sw128(smem_u32(sStage + s * T_STAGE_BYTES + T_A_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++)
            umma_f16_ts(acc, tA + (uint32_t)((kb * BK + kk * UMMA_K) / 2), bd + (uint64_t)(kk * 2), idesc,
                        (kb | kk) != 0);
          umma_commit(&empty[s]);
          next();
        }
        umma_commit(done);
      };
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
        // acc3 free: epi3(lt-1) preceded hready[0](lt-1); and FC4(lt-1), which reads H3(lt-1) from acc3's
        // columns, has completed (no MMA overwrites a TMEM operand of an MMA still in flight)
        if (lt > 0) mbar_wait(&tfull[1], (lt - 1) & 1);
        mma_fc3();
        if (lt > 0) {
          mbar_wait(&hready[1], (lt - 1) & 1);               // H4(lt-1) written, acc4 drained
          tc_fence_after();
          mma_from_tmem(acc4, T_N4 / BK, acc5, id5, &tfull[2]);
          mbar_wait(&tfull[2], (lt - 1) & 1);                // FC5(lt-1) read H4 from acc4's columns
        }
        mbar_wait(&hready[0], lt & 1);                       // H3(lt) written, acc3 drained
        tc_fence_after();
        mma_from_tmem(acc3, T_N3 / BK, acc4, id4, &tfull[1]);
      }
      if (lt > 0) {
        mbar_wait(&hready[1], (lt - 1) & 1);
        tc_fence_after();
        mma_from_tmem(acc4, T_N4 / BK, acc5, id5, &tfull[2]);
      }
    }
  } else {
    // ===== epilogue warps: quadrant q (TMEM lanes / tile rows), column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const int r = q * 32 + lane;                 // row inside the tile
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    // acc columns [c0, c0 + 128 or 64) of this warp -> bias + ReLU + RNE cast, packed two per 32-bit column, then
    // written back over the first half of the same accumulator (the next layer's A operand) once the
    // quadrant's other warp has read its columns too
    auto drain_pack = [&](uint32_t acc, int ncol, const float* bias, int bar) {
      uint32_t pk[64];
      const int c0 = h * ncol;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        if (c * 64 >= ncol) break;
        uint32_t v[64];
        TMEM_LD32(lane_base + acc + c0 + 64 * c, v);
        TMEM_LD32(lane_base + acc + c0 + 64 * c + 32, (v + 32));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c0 + 64 * c + i));
          pk[32 * c + i / 2] = Pack<BF16>::two_relu(__uint_as_float(v[i]) + b.x, __uint_as_float(v[i + 1]) + b.y);
          pk[32 * c + i / 2 + 1] = Pack<BF16>::two_relu(__uint_as_float(v[i + 2]) + b.z, __uint_as_float(v[i + 3]) + b.w);
        }
      }
      asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
      TMEM_ST32(lane_base + acc + c0 / 2, pk);
      if (ncol > 64) TMEM_ST32(lane_base + acc + c0 / 2 + 32, (pk + 32));
      tmem_wait_st();
    };
    auto epi3 = [&](int lt) {
      mbar_wait(&tfull[0], lt & 1);
      tc_fence_after();
      drain_pack(0, T_N3 / 2, tp.b3, 1 + q);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hready[0]);
    };
    auto epi4 = [&](int lt) {
      mbar_wait(&tfull[1], lt & 1);
      tc_fence_after();
      drain_pack(T_N3, T_N4 / 2, tp.b4, 1 + q);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hready[1]);
    };
    auto epi5 = [&](int lt, int tile) {
      mbar_wait(&tfull[2], lt & 1);
      tc_fence_after();
      if (h != 0) return;                       // one warp per quadrant owns the row's head dot product
      float z0 = 0.0f, z1 = 0.0f;
#pragma unroll 1
      for (int c = 0; c < T_N5; c += 32) {
        uint32_t v[32];
        TMEM_LD32(lane_base + T_N3 + T_N4 + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i++) {
          const float a = fmaxf(__uint_as_float(v[i]) + __ldg(tp.b5 + c + i), 0.0f);
          z0 = fmaf(__ldg(tp.head_w + c + i), a, z0);
          if (tp.head_n == 2) z1 = fmaf(__ldg(tp.head_w + T_N5 + c + i), a, z1);
        }
      }
      const int row = tile * BM + r;
      if (row < M) {
        const float z = (tp.head_n == 2) ? (z1 + tp.head_b[1]) - (z0 + tp.head_b[0]) : z0 + tp.head_b[0];
        tp.scores[row] = sigmoid(z);
      }
    };
    int lt = 0, prev_tile = -1;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
      epi3(lt);
      if (lt > 0) epi5(lt - 1, prev_tile);
      epi4(lt);
      prev_tile = t;
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

bool tail_supported(int n3, int n4, int n5, int k3) {
  return n3 == T_N3 && n4 == T_N4 && n5 == T_N5 && k3 % BK == 0 && k3 >= BK;
}

cudaError_t launch_tail(const CUtensorMap* tmA3, const CUtensorMap* tmB3, const CUtensorMap* tmB4,
                        const CUtensorMap* tmB5, int M, int K3, int bf16, const TailParams& tp, int num_sms, bool pdl,
                        cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  auto kern = bf16 ? tail_kernel<true> : tail_kernel<false>;
  static DevOnce attr[2];
  if (attr[bf16 ? 1 : 0].first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T_SMEM);
  }
  const int tiles = (M + BM - 1) / BM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles < num_sms ? tiles : num_sms);
  cfg.blockDim = dim3(T_THREADS);
  cfg.dynamicSmemBytes = T_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, *tmA3, *tmB3, *tmB4, *tmB5, M, K3, tp);
}

}  // namespace cold
