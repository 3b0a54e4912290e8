// kernels_latchain.cu — the whole FC stack of a SMALL call (one request of a few thousand ads, the
// latency path: §4.1 D_in x 1024 x 512 x 256 x 128 x 64 x 2, L163 sigma) in ONE launch
// of 8-CTA clusters, instead of three (FC1 pair GEMM, FC2 pair GEMM, FC3-FC5 tail kernel).
//
// A cluster = 4 CTA pairs (cta_group::2, peers rank ^ 1) owns a 256-row block at a time:
//   FC1: pair p computes n-tile p (256 of the 1024 columns; u1[request] added by the extra K = 16 MMA,
//        as in the chain kernel, D-4) and stores its H1 slice (TMA, L2);
//   FC2: once all four pairs' H1 slices are stored (a cluster-scope mbarrier every epilogue warp of the
//        cluster arrives on), pair p computes 128 of the 512 columns over the whole K = 1024 and stores
//        its H2 slice;
//   FC3 -> FC4 -> FC5 -> head: pair 0, once all H2 slices are stored, runs FC3 (N = 256, K = 512) and
//        then FC4 / FC5 IN TMEM as in the chain kernel's TAIL variant: the FC3 epilogue writes H3 back
//        into its accumulator buffer as FC4's A operand (tcgen05.mma with A from tensor memory), acc4 in
//        the upper 128 columns, H4 and acc5 likewise, the head and sigma in the FC5 epilogue.
// Measured (profiles/r03/lat_ab_r03n.jsonl, COLD_K_LAT_CHAIN): 81.5 vs 61-63 us p50 at 4000 ads for the
// three layer launches: at most 15 eight-CTA clusters are co-resident (ncu: 120 CTAs), so one of the 16
// blocks runs as a second wave, and a block's path through the four pairs takes ~27 us. Off by default.
// Per CTA the roles are the chain kernel's: warp 0 TMA producer, warp 1 MMA issuer (pair leader),
// warps 2..9 epilogue (two per TMEM lane quadrant). Cross-pair data goes through L2: the writer waits for
// its bulk stores, fences the async proxy and arrives with release.cluster semantics; the reader waits with
// acquire.cluster and fences before its TMA loads.
#include <cuda.h>

#include "internal.h"
#include "ptx.cuh"
#include "epi.cuh"
#include "pair.cuh"

namespace cold {

constexpr int LC_CL = 8;                                  // CTAs per cluster
constexpr int LC_NP = LC_CL / 2;                          // CTA pairs per cluster
constexpr int LC_BN = 256;
constexpr int LC_EPI_WARPS = 8;
constexpr int LC_GROUPS = LC_EPI_WARPS / 4;
constexpr int LC_THREADS = 64 + 32 * LC_EPI_WARPS;
constexpr int LC_A_BYTES = BM * BK * 2;                   // 16 KB: own 128 rows x 64 K
constexpr int LC_B_BYTES = (LC_BN / 2) * BK * 2;          // 16 KB: at most half of a 256-row weight tile
constexpr int LC_STAGE_BYTES = LC_A_BYTES + LC_B_BYTES;
constexpr int LC_OUT_BYTES = LC_GROUPS * EPI_GROUP_BOX;
constexpr int LC_UXA = BM * 32, LC_UXB = (LC_BN / 2) * 16 * 4, LC_UX_BUF = LC_UXA + LC_UXB;
constexpr int LC_BIASF = 1024;                            // FC2 + FC3 biases (512 + 256)
constexpr int LC_BIAS_BYTES = LC_BIASF * 4;
constexpr int LC_STAGES = (232448 - LC_OUT_BYTES - LC_UX_BUF - 1024 - 512 - LC_BIAS_BYTES) / LC_STAGE_BYTES;
constexpr int LC_SMEM = LC_STAGES * LC_STAGE_BYTES + LC_OUT_BYTES + LC_UX_BUF + 1024 + 512 + LC_BIAS_BYTES;
static_assert(LC_STAGES >= 4, "latency chain pipeline depth");

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// the pair's MMA completion, signalled on the same barrier offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair_at(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// pair TMA loads whose completion bytes land on the pair leader's barrier (leader_bar: shared::cluster
// address from mapa)
__device__ __forceinline__ void tma2_pair_at(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(leader_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma3_pair_at(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1,
                                             int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

template <bool BF16>
__global__ void __launch_bounds__(LC_THREADS, 1)
    latchain_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                    const __grid_constant__ CUtensorMap tmW2q, const __grid_constant__ CUtensorMap tmW3,
                    const __grid_constant__ CUtensorMap tmW4h, const __grid_constant__ CUtensorMap tmW5h,
                    const __grid_constant__ CUtensorMap tmH1in, const __grid_constant__ CUtensorMap tmH2in,
                    const __grid_constant__ CUtensorMap tmH1out, const __grid_constant__ CUtensorMap tmH2out,
                    const __grid_constant__ CUtensorMap tmOH, const __grid_constant__ CUtensorMap tmU1T, int M,
                    ChainParams cp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + LC_STAGES * LC_A_BYTES;
  uint8_t* sOut = smem + LC_STAGES * LC_STAGE_BYTES;
  uint8_t* sUX = sOut + LC_OUT_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sUX + LC_UX_BUF);
  uint64_t* full = bars;                          // pair leader: A+B bytes of both CTAs
  uint64_t* empty = full + LC_STAGES;             // both: released by the leader's pair commit
  uint64_t* tfull = empty + LC_STAGES;            // both: accumulator ready [2]
  uint64_t* tempty = tfull + 2;                   // pair leader: both CTAs' epilogues drained [2]
  uint64_t* uxfull = tempty + 2;                  // pair leader: u1 operand landed
  uint64_t* uxempty = uxfull + 1;                 // both: u1 MMA done
  uint64_t* h1done = uxempty + 1;                 // every CTA: all H1 slices of the block stored (cluster)
  uint64_t* h2done = h1done + 1;                  // every CTA: all H2 slices stored (cluster; pair 0 waits)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h2done + 1);
  float* sBias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);
  for (int i = threadIdx.x; i < cp.n2 + cp.n3; i += blockDim.x) sBias[i] = i < cp.n2 ? cp.b2[i] : cp.b3[i - cp.n2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t r1 = rank & 1u;                  // row half of the pair
  const uint32_t lead = rank & ~1u;               // the pair leader's cluster rank
  const bool leader = r1 == 0;
  const int p = (int)(rank >> 1);                 // pair within the cluster
  const uint16_t pmask = (uint16_t)(3u << lead);
  const int cl = (int)cluster_id_x(), ncl = (int)num_clusters_x();
  const int nblk = (M + 2 * BM - 1) / (2 * BM);
  // layers 0..4 = FC1 .. FC5; per layer: K blocks, tile N, weight map
  const int kbs[5] = {cp.k1 / BK, cp.n1 / BK, cp.n2 / BK, cp.n3 / BK, cp.n4 / BK};
  const int tn[5] = {LC_BN, cp.n2 / LC_NP, cp.n3, cp.n4, cp.n5};
  const CUtensorMap* tB[5] = {&tmW1, &tmW2q, &tmW3, &tmW4h, &tmW5h};

  // tasks of this CTA per block (all roles walk the list identically): FC1 n-tile p [buffer 0],
  // FC2 n-tile p [buffer 1], and on pair 0: FC3 [0], FC4 [0], FC5 [0]
  auto for_tasks = [&](auto&& f) {
    int jj = 0;
    for (int j = cl; j < nblk; j += ncl, jj++) {
      f(0, j, jj, p, 0);
      f(1, j, jj, p, 1);
      if (p == 0) {
        f(2, j, jj, 0, 0);
        f(3, j, jj, 0, 0);
        f(4, j, jj, 0, 0);
      }
    }
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < LC_STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * LC_EPI_WARPS); }
    mbar_init(uxfull, 1);
    mbar_init(uxempty, 1);
    mbar_init(h1done, LC_CL * LC_EPI_WARPS);
    mbar_init(h2done, LC_CL * LC_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const CUtensorMap* maps[12] = {&tmX, &tmW1, &tmW2q, &tmW3, &tmW4h, &tmW5h, &tmH1in, &tmH2in, &tmH1out, &tmH2out, &tmOH, &tmU1T};
    for (int i = 0; i < 12; i++) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)maps[i]) : "memory");
  }
  if (BF16 && warp == 2) {   // bf16: the 4th K chunk of the B_x buffer stays zero
    for (int i = lane; i < LC_BN / 2; i += 32)
      sts128(smem_u32(sUX + LC_UXA + 3 * (LC_BN / 2) * 16 + i * 16), make_uint4(0, 0, 0, 0));
    fence_async_smem();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * LC_BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  if (warp != 0) pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      constexpr int TERMS = BF16 ? 3 : 2;
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      const uint32_t full_l = mapa_u32(full, lead), uxfull_l = mapa_u32(uxfull, lead);
      pdl_wait();
      int s = 0, ux_t = 0;
      uint32_t ph = 0;
      for_tasks([&](int l, int j, int jj, int nb, int) {
        const int mrow = j * 2 * BM + (int)r1 * BM;
        if (l == 1 || l == 2) {   // the whole block's H1 (FC2) / H2 (FC3) from all four pairs
          mbar_wait_cluster(l == 1 ? h1done : h2done, (uint32_t)(jj & 1));
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const int bhalf = tn[l] / 2;
        for (int kb = 0; kb < kbs[l]; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t fb = full_l + (uint32_t)(s * 8);
          if (l >= 3) {   // FC4 / FC5: A is in TMEM, only the weight half streams
            if (leader) mbar_expect_tx(&full[s], 2 * (bhalf * BK * 2));
          } else {
            if (leader) mbar_expect_tx(&full[s], 2 * (LC_A_BYTES + bhalf * BK * 2));
            if (l == 0) {
              if (cp.x_slab) tma3_pair_at(sA + s * LC_A_BYTES, &tmX, fb, 0, mrow / 32, kb * 8, pol_a);
              else tma2_pair_at(sA + s * LC_A_BYTES, &tmX, fb, kb * BK, mrow, pol_a);
            } else {
              tma2_pair_at(sA + s * LC_A_BYTES, l == 1 ? &tmH1in : &tmH2in, fb, kb * BK, mrow, pol_a);
            }
          }
          tma2_pair_at(sB + s * LC_B_BYTES, tB[l], fb, kb * BK, nb * tn[l] + (int)r1 * bhalf, pol_b);
          if (++s == LC_STAGES) { s = 0; ph ^= 1; }
        }
        if (l == 0) {   // FC1: the tile's u1 operand (one-hot rows + u1-term columns)
          mbar_wait(uxempty, (uint32_t)(ux_t & 1) ^ 1);
          const int r_first = cp.req_of_ad[cp.a0 + j * 2 * BM] & ~7;
          if (leader) mbar_expect_tx(uxfull, 2 * (LC_UXA + TERMS * (LC_BN / 2) * 16));
          tma2_pair_at(sUX, &tmOH, uxfull_l, 0, mrow, pol_a);
          tma2_pair_at(sUX + BM * 16, &tmOH, uxfull_l, 8, mrow, pol_a);
          const int n0 = nb * LC_BN + (int)r1 * (LC_BN / 2);
#pragma unroll
          for (int t = 0; t < TERMS; t++)
            tma2_pair_at(sUX + LC_UXA + t * (LC_BN / 2) * 16, &tmU1T, uxfull_l, r_first, t * cp.n1 + n0, pol_b);
          ux_t++;
        }
      });
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===== MMA issuer (pair leader) =====
      const uint32_t idesc[5] = {idesc_pair<256, BF16>(), idesc_pair<128, BF16>(), idesc_pair<256, BF16>(),
                                 idesc_pair<128, BF16>(), idesc_pair<64, BF16>()};
      int s = 0, ux_t = 0, uses0 = 0, uses1 = 0;
      uint32_t ph = 0;
      for_tasks([&](int l, int, int, int, int acc) {
        mbar_wait(&tempty[acc], (uint32_t)((acc ? uses1++ : uses0++) & 1) ^ 1);
        tc_fence_after();
        const uint32_t bufc = tmem_base + acc * LC_BN;
        const uint32_t d = l == 3 ? bufc + 128 : (l == 4 ? bufc + 64 : bufc);
        for (int kb = 0; kb < kbs[l]; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * LC_A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + s * LC_B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++) {
            if (l >= 3) {   // A = 16 K elements of H3 / H4 = 8 TMEM columns of the same buffer
              umma_f16_pair_ts(d, bufc + (uint32_t)((kb * BK + kk * UMMA_K) / 2), bd + (uint64_t)(kk * 2), idesc[l],
                               (kb | kk) != 0);
              continue;
            }
            const uint64_t a_kk = (l == 0 && cp.x_slab) ? sdesc_k16_plain(smem_u32(sA + s * LC_A_BYTES) + kk * BM * 32)
                                                         : ad + (uint64_t)(kk * 2);
            umma_f16_pair(d, a_kk, bd + (uint64_t)(kk * 2), idesc[l], (kb | kk) != 0);
          }
          umma_commit_pair_at(&empty[s], pmask);
          if (++s == LC_STAGES) { s = 0; ph ^= 1; }
        }
        if (l == 0) {   // D += A_x B_x^T = u1[request(row)][n]
          mbar_wait(uxfull, (uint32_t)(ux_t & 1));
          tc_fence_after();
          const uint32_t ux = smem_u32(sUX);
          const uint64_t adx = sdesc_k16_plain(ux);
          umma_f16_pair(d, adx, sdesc_k16_plain(ux + LC_UXA), idesc[0], 1u);
          if (BF16) umma_f16_pair(d, adx, sdesc_k16_plain(ux + LC_UXA + 2 * (LC_BN / 2) * 16), idesc[0], 1u);
          umma_commit_pair_at(uxempty, pmask);
          ux_t++;
        }
        umma_commit_pair_at(&tfull[acc], pmask);
      });
    }
  } else {
    // ===== epilogue warps 2..9: TMEM lane quadrant q, column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const bool elected = (q == 0) && (lane == 0);
    int box_ctr = 0, uses0 = 0, uses1 = 0;
    for_tasks([&](int l, int j, int, int nb, int acc) {
      mbar_wait(&tfull[acc], (uint32_t)((acc ? uses1++ : uses0++) & 1));
      tc_fence_after();
      const int trow0 = j * 2 * BM + (int)r1 * BM;
      const int row = trow0 + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * LC_BN);
      if (l == 0 || l == 1) {
        const float* u1row = nullptr;   // FC1 fallback: the block spans more than U1_NSLOT requests
        uint32_t bias_s = 0u;
        if (l == 0) {
          const int t0 = j * 2 * BM;
          if (cp.req_of_ad[cp.a0 + min(t0 + 2 * BM, M) - 1] - (cp.req_of_ad[cp.a0 + t0] & ~7) >= U1_NSLOT) {
            const int req = row < M ? cp.req_of_ad[cp.a0 + row] : 0;
            u1row = cp.u1 + (int64_t)req * cp.ld_u1 + nb * LC_BN;
          }
        } else {
          bias_s = smem_u32(sBias) + (uint32_t)(nb * tn[1]) * 4u;
        }
        const int half = tn[l] / LC_GROUPS;
        epi_store_wide<BF16>(tbase, h * half, (h + 1) * half, nullptr, bias_s, u1row, 1, sOut + h * EPI_GROUP_BOX,
                             l == 0 ? &tmH1out : &tmH2out, nb * tn[l], trow0, q, h, lane, 0, nullptr, nullptr, 0, M,
                             0ull, nullptr, nullptr, &box_ctr);
      } else if (l == 2) {
        // FC3 -> H3 = ReLU(acc3 + b3), 16-bit, packed two per column into columns [64 h, 64 h + 64) (FC4's A
        // operand); the quadrant's other warp must have read its acc3 columns first
        const float* b3 = sBias + cp.n2;
        uint32_t pk[64];
#pragma unroll
        for (int c = 0; c < 2; c++) {
          uint32_t v[64];
          TMEM_LD32(tbase + 128 * h + 64 * c, v);
          TMEM_LD32(tbase + 128 * h + 64 * c + 32, (v + 32));
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 64; i += 4) {
            const float4 b = *reinterpret_cast<const float4*>(b3 + 128 * h + 64 * c + i);
            pk[32 * c + i / 2] = Pack<BF16>::two_relu(__uint_as_float(v[i]) + b.x, __uint_as_float(v[i + 1]) + b.y);
            pk[32 * c + i / 2 + 1] = Pack<BF16>::two_relu(__uint_as_float(v[i + 2]) + b.z, __uint_as_float(v[i + 3]) + b.w);
          }
        }
        named_bar_sync(3 + q, 64);
        TMEM_ST32(tbase + 64 * h, pk);
        TMEM_ST32(tbase + 64 * h + 32, (pk + 32));
        tmem_wait_st();
      } else if (l == 3) {
        // FC4 -> H4 = ReLU(acc4 + b4) into columns [32 h, 32 h + 32) (FC5's A operand; H3 is dead)
        uint32_t v[64], pk[32];
        TMEM_LD32(tbase + 128 + 64 * h, v);
        TMEM_LD32(tbase + 128 + 64 * h + 32, (v + 32));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(cp.b4 + 64 * h + i));
          pk[i / 2] = Pack<BF16>::two_relu(__uint_as_float(v[i]) + b.x, __uint_as_float(v[i + 1]) + b.y);
          pk[i / 2 + 1] = Pack<BF16>::two_relu(__uint_as_float(v[i + 2]) + b.z, __uint_as_float(v[i + 3]) + b.w);
        }
        TMEM_ST32(tbase + 32 * h, pk);
        tmem_wait_st();
      } else {
        // FC5 + head: h == 0 warps own their quadrant's rows: ReLU(acc5 + b5) . head_w + head_b -> sigma
        if (h == 0) {
          float z0 = 0.0f, z1 = 0.0f;
#pragma unroll
          for (int c = 0; c < 64; c += 32) {
            uint32_t v[32];
            TMEM_LD32(tbase + 64 + c, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++) {
              const float a = fmaxf(__uint_as_float(v[i]) + __ldg(cp.b5 + c + i), 0.0f);
              z0 = fmaf(__ldg(cp.head_w + c + i), a, z0);
              if (cp.head_n == 2) z1 = fmaf(__ldg(cp.head_w + 64 + c + i), a, z1);
            }
          }
          if (row < M) {
            const float z = cp.head_n == 2 ? (z1 + cp.head_b[1]) - (z0 + cp.head_b[0]) : z0 + cp.head_b[0];
            cp.scores[row] = sigmoid(z);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);
      if (l == 0 || l == 1) {
        // this group's slice of H1 / H2 is stored: every CTA of the cluster (FC2 loads all of H1) or the
        // two CTAs of pair 0 (FC3 loads all of H2) may read it once all 64 epilogue warps have arrived
        if (elected) {
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        named_bar_sync(1 + h, 128);
        if (lane == 0) {
          if (l == 0) {
            for (uint32_t r = 0; r < (uint32_t)LC_CL; r++) mbar_arrive_cluster(h1done, r);
          } else {
            mbar_arrive_cluster(h2done, 0);
            mbar_arrive_cluster(h2done, 1);
          }
        }
      }
    });
    if (elected) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * LC_BN) : "memory");
  }
}

// the paper's widths (n1 = 4 pairs x 256, n2 = 4 x 128, FC3 256 -> 128 -> 64 -> head) and FC1's K
bool latchain_supported(int n1, int n2, int n3, int n4, int n5, int k1) {
  return n1 == LC_NP * LC_BN && n2 == LC_NP * 128 && n3 == LC_BN && n4 == 128 && n5 == 64 && k1 % BK == 0 &&
         n2 + n3 <= LC_BIASF;
}

cudaError_t launch_latchain(const CUtensorMap* tm[12], int M, int bf16, const ChainParams& cp, bool pdl,
                            cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  auto kern = bf16 ? latchain_kernel<true> : latchain_kernel<false>;
  static DevOnce attr[2];
  static int max_clusters[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = LC_CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(LC_THREADS);
  cfg.dynamicSmemBytes = LC_SMEM;
  cfg.stream = s;
  cfg.attrs = attrs;
  if (attr[bf16 ? 1 : 0].first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LC_SMEM);
    cfg.gridDim = dim3(LC_CL);
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) { cudaGetLastError(); n = 0; }
    if (dev < 64) max_clusters[dev] = n;
  }
  const int mc = dev < 64 && max_clusters[dev] > 0 ? max_clusters[dev] : 8;
  const int nblk = (M + 2 * BM - 1) / (2 * BM);
  const int clusters = nblk < mc ? nblk : mc;
  cfg.gridDim = dim3(LC_CL * clusters);
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, *tm[0], *tm[1], *tm[2], *tm[3], *tm[4], *tm[5], *tm[6], *tm[7], *tm[8],
                            *tm[9], *tm[10], *tm[11], M, cp);
}

}  // namespace cold
