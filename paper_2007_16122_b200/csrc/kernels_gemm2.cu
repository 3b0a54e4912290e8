// kernels_gemm2.cu — one FC layer on a CTA PAIR (tcgen05.mma.cta_group::2), sm_100a.
//
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )   (PAPER.md L328 FC stack; L517 "dense matrix
//   multiplication, which needs extreme optimization")
//
// The two CTAs of a cluster (same TPC) own a 256-row tile: each CTA loads its own 128 rows of A and
// HALF of the BN-row weight tile (BN/2 rows); the leader CTA issues one M=256 x N=BN MMA per 16-wide
// K step that reads A and B from both CTAs' shared memory and accumulates each CTA's 128 rows into
// that CTA's TMEM. Versus the 1-CTA kernel this halves the weight bytes every SM stages and reads
// (48 KB -> 32 KB per 64-deep K step for BN = 256), so 6 stages fit instead of 4 and L2 serves a
// third fewer bytes per FLOP (FC2 / FC1 were measured 30-40% starved for operands).
//
// Roles per CTA: warp 0 = TMA producer (both CTAs; completion bytes land on the leader's "full"
// barrier), warp 1 = TMEM allocator (both, cta_group::2) + MMA issuer (leader only), warps 2..9 =
// epilogue (both CTAs, their own 128 rows; they release the accumulator on the leader's "tempty").
#include <cuda.h>
#include "internal.h"
#include "ptx.cuh"
#include "epi.cuh"

namespace cold {

constexpr int P_EPI_WARPS = 8;
constexpr int P_THREADS = 64 + 32 * P_EPI_WARPS;
constexpr int P_EPI_COLS = 32;
constexpr int P_OUT_BOX = 32 * P_EPI_COLS * 2;     // 2 KB staging box (32 rows x 32 cols)
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;        // shared::cluster address of the leader's copy

template <int BN, bool U1> struct PairCfg {
  static constexpr int A_BYTES = BM * BK * 2;                 // own 128 rows
  static constexpr int B_BYTES = (BN / 2) * BK * 2;           // own half of the weight tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int OUT_BYTES = P_EPI_WARPS * 2 * P_OUT_BOX;
  static constexpr int U1_BYTES = U1 ? 2 * 2 * BN * 4 : 0;
  static constexpr int STAGES_FIT = (232448 - OUT_BYTES - U1_BYTES - 1024 - 512) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + OUT_BYTES + U1_BYTES + 1024 + 512;
};

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar) & PEER_MASK), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the same barrier offset in both CTAs of the pair once all prior MMAs completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on CTA `rank`'s copy of a barrier
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

template <int BN, bool BF16>
__device__ __forceinline__ constexpr uint32_t idesc_pair() {
  return (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(256 >> 4) << 24);
}

template <int BN, bool BF16, bool U1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, int M, int N, int K, EpiParams ep) {
  using Cfg = PairCfg<BN, U1>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* sOut = smem + Cfg::STAGES * Cfg::STAGE_BYTES;
  float* sU1 = reinterpret_cast<float*>(sOut + Cfg::OUT_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + Cfg::OUT_BYTES + Cfg::U1_BYTES);
  uint64_t* full = bars;                          // leader: A+B bytes of both CTAs
  uint64_t* empty = bars + Cfg::STAGES;           // both: released by the leader's pair commit
  uint64_t* tfull = bars + 2 * Cfg::STAGES;       // both: accumulator ready
  uint64_t* tempty = tfull + 2;                   // leader: both CTAs' epilogues drained
  uint64_t* u1full = tempty + 2;                  // local: u1 rows staged
  uint64_t* u1empty = u1full + 2;                 // local: this CTA's epilogue is done with u1 buffer
  int32_t* u1hdr = reinterpret_cast<int32_t*>(u1empty + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u1hdr + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = (int)cluster_id_x(), npairs = (int)num_clusters_x();
  const int num_pm = (M + 2 * BM - 1) / (2 * BM), num_n = N / BN;
  const int items = num_pm * num_n;
  const int kb_count = K / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * P_EPI_WARPS); }
    for (int s = 0; s < 2; s++) { mbar_init(&u1full[s], 1); mbar_init(&u1empty[s], P_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
    if (ep.out) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmC) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int it = pair; it < items; it += npairs, lt++) {
        const int pm = it / num_n, nb = it % num_n;
        const int mrow = pm * 2 * BM + (int)rank * BM;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          tma_load_2d_pair(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * BK, mrow, pol_a);
          tma_load_2d_pair(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * BK, nb * BN + (int)rank * (BN / 2), pol_b);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        if (U1) {
          // FC1: stage this CTA's u1 row slice(s) [nb*BN, +BN); <= 2 requests per 128 rows, else global
          const int acc = lt & 1;
          mbar_wait(&u1empty[acc], ((lt >> 1) & 1) ^ 1);   // this CTA's epilogue finished tile lt-2
          const int rlo = mrow, rhi = min(M, rlo + BM) - 1;
          const int r0 = rlo < M ? ep.req_of_ad[ep.a0 + rlo] : 0;
          const int r1 = rlo < M ? ep.req_of_ad[ep.a0 + rhi] : 0;
          float* dst = sU1 + acc * 2 * BN;
          if (rlo < M && r1 - r0 <= 1) {
            u1hdr[acc] = (r1 != r0) ? (int)(ep.ad_offsets[r1] - ep.a0 - rlo) : BM;
            mbar_expect_tx(&u1full[acc], (uint32_t)(BN * 4 * (1 + (r1 != r0))));
            bulk_load(dst, ep.u1 + (int64_t)r0 * ep.ld_u1 + nb * BN, BN * 4, &u1full[acc]);
            if (r1 != r0) bulk_load(dst + BN, ep.u1 + (int64_t)r1 * ep.ld_u1 + nb * BN, BN * 4, &u1full[acc]);
          } else {
            u1hdr[acc] = -1;
            mbar_arrive(&u1full[acc]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===== MMA issuer (leader only) =====
      constexpr uint32_t idesc = idesc_pair<BN, BF16>();
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int it = pair; it < items; it += npairs, lt++) {
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * Cfg::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + s * Cfg::B_BYTES));
          if (ep.dbg_mode != 2) {
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; kk++)
              umma_f16_pair(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          }
          umma_commit_pair(&empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue warps 2..9 (both CTAs): TMEM lane quadrant q, column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const bool head = ep.head_n != 0;
    constexpr bool WIDE = (BN / 2) % EPI_WIDE_COLS == 0;   // 64-column SW128 store boxes
    const int c_begin = head ? 0 : h * (BN / 2);
    const int c_end = head ? (h == 0 ? BN : 0) : (h + 1) * (BN / 2);
    uint8_t* my_out = sOut + ew * 2 * P_OUT_BOX;
    int ob = 0;
    int lt = 0;
    for (int it = pair; it < items; it += npairs, lt++) {
      const int pm = it / num_n, nb = it % num_n;
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int row0 = pm * 2 * BM + (int)rank * BM + q * 32;
      const int row = row0 + lane;
      const bool valid = row < M;
      uint32_t u1s = 0;                 // staged u1 row in shared memory (column nb*BN)
      const float* u1row = nullptr;
      if (ep.u1) {
        int bnd = -1;
        if (U1) {
          mbar_wait(&u1full[acc], (lt >> 1) & 1);
          bnd = u1hdr[acc];
        }
        if (bnd >= 0) {
          u1s = smem_u32(sU1 + acc * 2 * BN + ((q * 32 + lane) < bnd ? 0 : BN));
        } else {
          const int req = valid ? ep.req_of_ad[ep.a0 + row] : 0;
          u1row = ep.u1 + (int64_t)req * ep.ld_u1 + nb * BN;
        }
      }
      if (WIDE && !head) {
        const int c_stop = ep.dbg_mode == 1 ? c_begin : c_end;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
        epi_store_wide<BF16>(tbase, c_begin, c_stop, ep.bias, u1s, u1row, ep.relu,
                             sOut + ew * EPI_WIDE_BOX, &tmC, nb * BN, row0, lane, ep.dbg_mode);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_remote(&tempty[acc], 0);
          if (U1) mbar_arrive(&u1empty[acc]);
        }
        continue;
      }
      float z0 = 0.0f, z1 = 0.0f;
      const int c_stop = ep.dbg_mode == 1 ? c_begin : c_end;   // debug: drain nothing
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      uint32_t v[32];
      if (c_begin < c_stop) TMEM_LD32(taddr + c_begin, v);
      for (int c = c_begin; c < c_stop; c += P_EPI_COLS) {
        tmem_wait_ld();
        const int col0 = nb * BN + c;
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; i++) f[i] = __uint_as_float(v[i]);
        if (c + P_EPI_COLS < c_stop) TMEM_LD32(taddr + c + P_EPI_COLS, v);
        if (ep.bias) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
            f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
          }
        }
        if (u1s) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = lds128f(u1s + (uint32_t)(c + i) * 4u);
            f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
          }
        } else if (u1row) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(u1row + c + i));
            f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
          }
        }
        if (ep.relu) {
#pragma unroll
          for (int i = 0; i < 32; i++) f[i] = fmaxf(f[i], 0.0f);
        }
        if (head) {
#pragma unroll
          for (int i = 0; i < 32; i++) z0 = fmaf(__ldg(ep.head_w + col0 + i), f[i], z0);
          if (ep.head_n == 2) {
#pragma unroll
            for (int i = 0; i < 32; i++) z1 = fmaf(__ldg(ep.head_w + N + col0 + i), f[i], z1);
          }
        } else if (ep.dbg_mode == 3) {
          float t = 0.0f;
#pragma unroll
          for (int i = 0; i < 32; i++) t += f[i];
          if (t == 12345.678f) ep.scores[0] = t;   // keep the math alive
        } else {
          uint8_t* buf = my_out + ob * P_OUT_BOX;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; j++) {
            uint4 w;
            w.x = Pack<BF16>::two(f[8 * j + 0], f[8 * j + 1]);
            w.y = Pack<BF16>::two(f[8 * j + 2], f[8 * j + 3]);
            w.z = Pack<BF16>::two(f[8 * j + 4], f[8 * j + 5]);
            w.w = Pack<BF16>::two(f[8 * j + 6], f[8 * j + 7]);
            const int phys = j ^ ((lane >> 1) & 3);
            sts128(smem_u32(buf) + (uint32_t)(lane * 64 + phys * 16), w);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0 && ep.dbg_mode != 4) {
            tma_store_2d(&tmC, buf, col0, row0);
            bulk_commit();
          }
          ob ^= 1;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_remote(&tempty[acc], 0);
        if (U1) mbar_arrive(&u1empty[acc]);
      }
      if (head && h == 0 && valid) {
        float z;
        if (ep.head_n == 2) z = (z1 + ep.head_b[1]) - (z0 + ep.head_b[0]);
        else z = z0 + ep.head_b[0];
        ep.scores[row] = sigmoid(z);
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, bool BF16, bool U1>
static cudaError_t launch_pair_t(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M,
                                 int N, int K, const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s) {
  using Cfg = PairCfg<BN, U1>;
  auto kern = gemm_pair_kernel<BN, BF16, U1>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  const int items = ((M + 2 * BM - 1) / (2 * BM)) * (N / BN);
  const int pairs = items < num_sms / 2 ? items : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(P_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, *tmA, *tmB, *tmC, M, N, K, ep);
}

cudaError_t launch_gemm_pair(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N,
                             int K, int bn, int bf16, const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const bool u1 = ep.u1 != nullptr;
#define PAIR_CASE(BNV)                                                                                      \
  if (bn == BNV) {                                                                                          \
    if (bf16) return u1 ? launch_pair_t<BNV, true, true>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s)        \
                        : launch_pair_t<BNV, true, false>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);      \
    return u1 ? launch_pair_t<BNV, false, true>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s)                 \
              : launch_pair_t<BNV, false, false>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);               \
  }
  PAIR_CASE(256)
  PAIR_CASE(128)
  PAIR_CASE(64)
#undef PAIR_CASE
  return cudaErrorInvalidValue;
}

}  // namespace cold
