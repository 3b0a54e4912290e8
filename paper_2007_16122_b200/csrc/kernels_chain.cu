// kernels_chain.cu — FC1 -> FC2 -> FC3 of the COLD stack (§4.1: D_in x 1024 x 512 x 256 ..)
// in ONE persistent CTA-pair kernel that walks 256-row blocks, so the activations H1 / H2 of a block are
// consumed while they are still in L2 and are then discarded instead of being written back.
//
// Why: the layer-by-layer launches wrote 310 + 155 MB of H1 / H2 per 151,552-ad chunk and read them
// back, and B200's pure-write bandwidth is 3.9 TB/s (measured): those round trips, not the tensor
// cores, bounded FC1 (~110 us per chunk, epilogue-bound) and slowed the kernels after it.
//
// A pair owns row blocks rb = pair, pair + npairs, ... For its j-th block it runs, in this order,
//   step j: FC1(j) n-tiles 0..3 | FC3(j-1) | FC2(j) n-tiles 0..1
// FC2(j) needs all of H1(j) (K = 1024) and FC3(j-1) all of H2(j-1) (K = 512); every row of them was
// written by this CTA's own epilogue (A is M-split across the pair), so the dependency is local: the
// epilogue warps arrive on hready[0] / hready[1] once their TMA stores of the block's last tile of
// FC1 / FC2 have completed, and the producer waits there before loading the block as an A operand.
// FC3(j-1) sits between FC1(j) and FC2(j) so the tensor pipe has work while H1(j) drains.
// After FC2(j) (resp. FC3(j-1)) has consumed H1(j) (H2(j-1)), the epilogue issues
// discard.global.L2 on the CTA's rows of that block: the lines are dead, so L2 drops them without a
// write-back. H3 is written for the tail kernel (FC4 / FC5 / head), or, with TAIL, never leaves the SM:
// FC4 and FC5 run as CTA-pair MMAs whose A operand (H3, H4) the epilogue writes back into TMEM
// (tcgen05.st) and whose weights stream through the same stage ring (see for_tasks).
//
// Per tile the machinery is gemm_pair_kernel's: TMA producer (warp 0), leader MMA issuer (warp 1),
// 8 epilogue warps (2..9) with double-buffered TMEM accumulators and group TMA stores (epi.cuh), and
// FC1's u1[request(row)] added by one extra K = 16 MMA from the one-hot / u1-term operands (D-4).
#include <cuda.h>

#include "internal.h"
#include "ptx.cuh"
#include "epi.cuh"
#include "pair.cuh"

namespace cold {

constexpr int C_BN = 256;
#ifdef COLD_CHAIN_H1_BLOCK   // A/B: FC2 waits for the whole H1 block (round-1 behaviour)
constexpr bool H1_TILES = false;
#else
constexpr bool H1_TILES = true;
#endif
constexpr bool FC1_DIRECT = false;
constexpr bool FC3_MID = false;   // (FC3 between the FC1 halves: 277.4 vs 272.0 us per chunk, not adopted)   // (direct st.global H1 stores from registers: 294 vs 273 us, not adopted)
constexpr int C_EPI_WARPS = 8;                         // 2 per TMEM lane quadrant, 128 columns each
constexpr int C_GROUPS = C_EPI_WARPS / 4;              // 4-warp store groups (one 16 KB staging box each)
constexpr int C_THREADS = 64 + 32 * C_EPI_WARPS;
constexpr int C_A_BYTES = BM * BK * 2;                 // 16 KB: own 128 rows x 64 K
constexpr int C_B_BYTES = (C_BN / 2) * BK * 2;         // 16 KB: own half of the 256-row weight tile
constexpr int C_STAGE_BYTES = C_A_BYTES + C_B_BYTES;
#ifdef COLD_CHAIN_EPI_DB
constexpr int C_OUT_BOXES = 2 * C_GROUPS;   // A/B: two 16 KB boxes per group (one pipeline stage fewer): neutral
#else
constexpr int C_OUT_BOXES = C_GROUPS;   // one 16 KB staging box per 4-warp group
#endif
constexpr int C_OUT_BYTES = C_OUT_BOXES * EPI_GROUP_BOX;
constexpr int C_UXA = BM * 32, C_UXB = (C_BN / 2) * 16 * 4, C_UX_BUF = C_UXA + C_UXB, C_NUX = 2;
constexpr int C_BIASF = 1024;                          // FC2 + FC3 biases staged in smem (n2 + n3 <= 1024)
constexpr int C_BIAS_BYTES = C_BIASF * 4;
// FC1's first XRES_KB k-blocks of the block's X rows stay resident for its n-tiles (loaded once per block
// instead of once per n-tile: 10 instead of 16 X k-block loads per block); the ring gives up the stage this
// takes (4 stages measured as fast as 5). Chain 277.2 vs 278.3 us per chunk, whole step +1%
// (profiles/r03/ab_xr_*.jsonl). -DCOLD_CHAIN_XRES_KB=0 restores the re-load per n-tile.
#ifdef COLD_CHAIN_XRES_KB
constexpr int XRES_KB = COLD_CHAIN_XRES_KB;
#else
constexpr int XRES_KB = 2;
#endif
constexpr int C_X_BYTES = XRES_KB * C_A_BYTES;
constexpr int C_STAGES = (232448 - C_OUT_BYTES - C_NUX * C_UX_BUF - 1024 - 512 - C_BIAS_BYTES - C_X_BYTES) / C_STAGE_BYTES;
constexpr int C_SMEM = C_STAGES * C_STAGE_BYTES + C_OUT_BYTES + C_NUX * C_UX_BUF + 1024 + 512 + C_BIAS_BYTES + C_X_BYTES;
static_assert(C_STAGES >= 4, "chain kernel pipeline depth");

// debug: cycles a role spent blocked in a barrier wait (cp.instr != null)
__device__ __forceinline__ void cwait(uint64_t* bar, uint32_t parity, unsigned long long& acc, bool on) {
  if (!on) { mbar_wait(bar, parity); return; }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += (unsigned long long)(clock64() - t0);
}

__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <bool BF16, bool TAIL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C_THREADS, 1)
    chain_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                 const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmW3,
                 const __grid_constant__ CUtensorMap tmH1, const __grid_constant__ CUtensorMap tmH2,
                 const __grid_constant__ CUtensorMap tmH3, const __grid_constant__ CUtensorMap tmOH,
                 const __grid_constant__ CUtensorMap tmU1T, const __grid_constant__ CUtensorMap tmW4,
                 const __grid_constant__ CUtensorMap tmW5, const __grid_constant__ CUtensorMap tmH4, int M,
                 ChainParams cp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C_STAGES * C_A_BYTES;
  uint8_t* sOut = smem + C_STAGES * C_STAGE_BYTES;
  uint8_t* sUX = sOut + C_OUT_BYTES;
  uint8_t* sX = sUX + C_NUX * C_UX_BUF;           // XRES_KB resident X k-blocks of the block (FC1)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + C_X_BYTES);
  uint64_t* full = bars;                          // leader: A+B bytes of both CTAs
  uint64_t* empty = full + C_STAGES;              // both: released by the leader's pair commit
  uint64_t* tfull = empty + C_STAGES;             // both: accumulator ready [2]
  uint64_t* tempty = tfull + 2;                   // leader: both CTAs' epilogues drained [2]
  uint64_t* uxfull = tempty + 2;                  // leader: u1 operand landed [C_NUX]
  uint64_t* uxempty = uxfull + C_NUX;             // both: u1 MMA of the buffer's last FC1 tile done [C_NUX]
  uint64_t* hready = uxempty + C_NUX;             // local: [l] block of layer l's output stored (H1..H4)
  uint64_t* h1t = hready + 4;                     // local: [nb] FC1 n-tile nb of the block stored (H1_TILES)
  uint64_t* xfull = h1t + 4;                      // leader: both CTAs' resident X k-blocks landed
  uint64_t* xempty = xfull + 1;                   // both: the block's last FC1 MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + 1);
  // FC2 / FC3 biases in shared memory: the epilogue reads them with LDS instead of a global load that
  // stalled it (ncu r01h: 9% of the chain's stall samples on the bias add)
  float* sBias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512);
  const bool sbias = cp.n2 + cp.n3 <= C_BIASF;
  if (sbias)
    for (int i = threadIdx.x; i < cp.n2 + cp.n3; i += blockDim.x) sBias[i] = i < cp.n2 ? cp.b2[i] : cp.b3[i - cp.n2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = (int)cluster_id_x(), npairs = (int)num_clusters_x();
  const int num_pm = (M + 2 * BM - 1) / (2 * BM);
  const int nrb = pair < num_pm ? (num_pm - 1 - pair) / npairs + 1 : 0;   // this pair's row blocks
  // layers 0..2 = FC1..FC3 (N = 256 per tile), TAIL: 3 = FC4 (N = n4 = 128), 4 = FC5 (N = n5 = 64) + head
  const int kbs[5] = {cp.k1 / BK, cp.n1 / BK, cp.n2 / BK, cp.n3 / BK, cp.n4 / BK};
  const CUtensorMap* tA[3] = {&tmX, &tmH1, &tmH2};
  const CUtensorMap* tB[5] = {&tmW1, &tmW2, &tmW3, &tmW4, &tmW5};
  const CUtensorMap* tC[3] = {&tmH1, &tmH2, &tmH3};
  const int ntile[5] = {cp.n1 / C_BN, cp.n2 / C_BN, cp.n3 / C_BN, 1, 1};
  const int tn[5] = {C_BN, C_BN, C_BN, cp.n4, cp.n5};          // tile N per layer

  // the per-pair task order (all roles walk it identically): step s = 0..nrb:
  //   FC1(s) n-tiles | FC3(s-1) | FC2(s) n-tiles
  // (measured: interleaving FC1(j) with FC2(j-1) to spread the epilogue load doubles the L2 working set
  // of live activations and ran 14% slower)
  // (FC3_MID would put FC3(s-1) between the two halves of FC1(s)'s n-tiles to spread FC1's epilogue-heavy
  // tiles: measured slower, off)
  // Each task names its TMEM accumulator buffer (0 / 1, C_BN columns each); MMA issuer and epilogue count
  // the uses of each buffer for the barrier phases. Without TAIL the buffers alternate in task order.
  // TAIL (FC4 / FC5 / head in TMEM, no H3 round trip): step s =
  //   FC1(s) n-tiles (buffers alternate by n-tile) | FC3(s-1) [buffer 0] | FC2(s) tile 0 [buffer 1] |
  //   FC4(s-1) [buffer 0] | FC2(s) tiles 1.. [buffer 1] | FC5(s-1) [buffer 0]
  // FC3 -> FC4 -> FC5 of a block run IN PLACE in buffer 0: the FC3 epilogue writes H3 (16-bit, packed two
  // per column) into columns [0, 128) as FC4's A operand, acc4 lands in [128, 256), H4 goes to [0, 64) and
  // acc5 to [64, 128); the FC5 epilogue applies the head and the sigmoid.
  auto for_tasks = [&](auto&& f) {
    int t = 0;
    auto go = [&](int l, int j, int nb, int tbuf) { f(l, j, nb, TAIL ? tbuf : (t & 1)); t++; };
    for (int s = 0; s <= nrb; s++) {
      if (!TAIL) {
        const int fc1_split = (FC3_MID && s >= 1 && s <= nrb) ? ntile[0] / 2 : ntile[0];
        if (s < nrb) for (int nb = 0; nb < fc1_split; nb++) go(0, s, nb, 0);
        if (s >= 1) for (int nb = 0; nb < ntile[2]; nb++) go(2, s - 1, nb, 0);
        if (s < nrb) for (int nb = fc1_split; nb < ntile[0]; nb++) go(0, s, nb, 0);
        if (s < nrb) for (int nb = 0; nb < ntile[1]; nb++) go(1, s, nb, 0);
      } else {
        if (s < nrb) for (int nb = 0; nb < ntile[0]; nb++) go(0, s, nb, nb & 1);
        if (s >= 1) go(2, s - 1, 0, 0);
        if (s < nrb) go(1, s, 0, 1);
        if (s >= 1) go(3, s - 1, 0, 0);
        if (s < nrb) for (int nb = 1; nb < ntile[1]; nb++) go(1, s, nb, 1);
        if (s >= 1) go(4, s - 1, 0, 0);
      }
    }
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C_STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * C_EPI_WARPS); }
    for (int s = 0; s < C_NUX; s++) { mbar_init(&uxfull[s], 1); mbar_init(&uxempty[s], 1); }
    for (int i = 0; i < 4; i++) mbar_init(&hready[i], C_EPI_WARPS);
    for (int i = 0; i < 4; i++) mbar_init(&h1t[i], C_EPI_WARPS);
    mbar_init(xfull, 1);
    mbar_init(xempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const CUtensorMap* maps[12] = {&tmX, &tmW1, &tmW2, &tmW3, &tmH1, &tmH2, &tmH3, &tmOH, &tmU1T, &tmW4, &tmW5, &tmH4};
    for (int i = 0; i < (TAIL ? 12 : 9); i++) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)maps[i]) : "memory");
  }
  if (BF16 && warp == 2) {   // bf16: the 4th K chunk of every B_x buffer stays zero
    for (int b = 0; b < C_NUX; b++)
      for (int i = lane; i < C_BN / 2; i += 32)
        sts128(smem_u32(sUX + b * C_UX_BUF + C_UXA + 3 * (C_BN / 2) * 16 + i * 16), make_uint4(0, 0, 0, 0));
    fence_async_smem();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * C_BN)
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
      constexpr int TERMS = BF16 ? 3 : 2;
      const uint64_t pol_x = policy_evict_first();  // X: read once
      const uint64_t pol_a = policy_evict_last();   // H1 / H2: read while hot, then discarded
      const uint64_t pol_b = policy_evict_last();   // weights: re-read by every block
      int s = 0, fc1_t = 0, x_t = 0;
      uint32_t ph = 0;
      const bool ins = cp.instr != nullptr;
      unsigned long long w_empty = 0, w_hready = 0;
      for_tasks([&](int l, int j, int nb, int) {
        const int pm = pair + j * npairs;
        const int mrow = pm * 2 * BM + (int)rank * BM;
        if (l == 2 || (l == 1 && !H1_TILES)) {
          if (nb == 0) cwait(&hready[l - 1], (uint32_t)(j & 1), w_hready, ins);   // own rows of the input
        }
        const int bhalf = tn[l] / 2;                  // weight rows this CTA stages (half the tile N)
        const int xres = l == 0 ? min(XRES_KB, kbs[0]) : 0;
        if (xres > 0 && nb == 0) {   // the block's resident X k-blocks, once for its FC1 n-tiles
          cwait(xempty, (uint32_t)(x_t & 1) ^ 1, w_empty, ins);
          if (leader) mbar_expect_tx(xfull, 2 * xres * C_A_BYTES);
          for (int kb = 0; kb < xres; kb++)
            tma_load_a_pair(sX + kb * C_A_BYTES, tA[0], xfull, kb, mrow, pol_x, cp.x_slab);
          x_t++;
        }
        for (int kb = 0; kb < kbs[l]; kb++) {
          // FC2 reads H1 one FC1 n-tile (C_BN columns) at a time: wait for that tile's stores only, so FC2(j)
          // starts on the first tiles of H1(j) while the last FC1 tile is still draining
          if (H1_TILES && l == 1 && (kb * BK) % C_BN == 0)
            cwait(&h1t[(kb * BK) / C_BN], (uint32_t)(j & 1), w_hready, ins);
          cwait(&empty[s], ph ^ 1, w_empty, ins);
          if ((TAIL && l >= 3) || kb < xres) {   // FC4 / FC5: A in TMEM; FC1: A resident: only the weights
            if (leader) mbar_expect_tx(&full[s], 2 * (bhalf * BK * 2));
          } else {
#ifdef COLD_CHAIN_NO_A   // timing experiment (results wrong): layer COLD_CHAIN_NO_A's A operand is not loaded
            if (l == COLD_CHAIN_NO_A) {
              if (leader) mbar_expect_tx(&full[s], 2 * (bhalf * BK * 2));
            } else
#endif
            {
              if (leader) mbar_expect_tx(&full[s], 2 * (C_A_BYTES + bhalf * BK * 2));
              tma_load_a_pair(sA + s * C_A_BYTES, tA[l], &full[s], kb, mrow, l == 0 ? pol_x : pol_a, l == 0 && cp.x_slab);
            }
          }
          tma_load_2d_pair(sB + s * C_B_BYTES, tB[l], &full[s], kb * BK, nb * tn[l] + (int)rank * bhalf, pol_b);
          if (++s == C_STAGES) { s = 0; ph ^= 1; }
        }
        if (l == 0) {   // FC1: the tile's u1 operand (one-hot rows + u1-term columns)
          const int b = fc1_t % C_NUX;
          mbar_wait(&uxempty[b], ((fc1_t / C_NUX) & 1) ^ 1);
          const int r_first = cp.req_of_ad[cp.a0 + pm * 2 * BM] & ~7;
          uint8_t* ux = sUX + b * C_UX_BUF;
          if (leader) mbar_expect_tx(&uxfull[b], 2 * (C_UXA + TERMS * (C_BN / 2) * 16));
          tma_load_2d_pair(ux, &tmOH, &uxfull[b], 0, mrow, pol_x);
          tma_load_2d_pair(ux + BM * 16, &tmOH, &uxfull[b], 8, mrow, pol_x);
          const int n0 = nb * C_BN + (int)rank * (C_BN / 2);
#pragma unroll
          for (int t = 0; t < TERMS; t++)
            tma_load_2d_pair(ux + C_UXA + t * (C_BN / 2) * 16, &tmU1T, &uxfull[b], r_first, t * cp.n1 + n0, pol_b);
          fc1_t++;
        }
      });
      if (ins) { atomicAdd(cp.instr + 0, w_empty); atomicAdd(cp.instr + 1, w_hready); }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===== MMA issuer (leader only) =====
      constexpr uint32_t id256 = idesc_pair<C_BN, BF16>();
      const uint32_t id_tail[2] = {cp.n4 == 128 ? idesc_pair<128, BF16>() : idesc_pair<64, BF16>(),
                                   cp.n5 == 64 ? idesc_pair<64, BF16>() : idesc_pair<32, BF16>()};
      int s = 0, fc1_t = 0, uses0 = 0, uses1 = 0, x_t = 0;
      uint32_t ph = 0;
      const bool ins = cp.instr != nullptr;
      unsigned long long w_full = 0, w_tempty = 0, w_ux = 0, wl_full[3] = {0, 0, 0}, wl_te[3] = {0, 0, 0};
      const long long t_begin = clock64();
      for_tasks([&](int l, int j, int nb, int acc) {
        const uint32_t idesc = l < 3 ? id256 : id_tail[l - 3];
        const unsigned long long te0 = w_tempty, fu0 = w_full;
        cwait(&tempty[acc], (uint32_t)((acc ? uses1++ : uses0++) & 1) ^ 1, w_tempty, ins);
        tc_fence_after();
        const uint32_t bufc = tmem_base + acc * C_BN;
        // TAIL in place: acc4 at column 128, acc5 at 64; their A (H3 / H4) from column 0 of the same buffer
        const uint32_t d = (TAIL && l == 3) ? bufc + 128 : ((TAIL && l == 4) ? bufc + 64 : bufc);
        const int xres = l == 0 ? min(XRES_KB, kbs[0]) : 0;
        if (xres > 0 && nb == 0) {
          cwait(xfull, (uint32_t)(x_t & 1), w_full, ins);
          tc_fence_after();
        }
        for (int kb = 0; kb < kbs[l]; kb++) {
          cwait(&full[s], ph, w_full, ins);
          tc_fence_after();
          uint8_t* a_tile = kb < xres ? sX + kb * C_A_BYTES : sA + s * C_A_BYTES;
          const uint64_t ad = sdesc_sw128(smem_u32(a_tile));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + s * C_B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++) {
            if (TAIL && l >= 3) {   // A = 16 K elements of H3 / H4 = 8 TMEM columns
              umma_f16_pair_ts(d, bufc + (uint32_t)((kb * BK + kk * UMMA_K) / 2), bd + (uint64_t)(kk * 2), idesc,
                               (kb | kk) != 0);
              continue;
            }
            const uint64_t a_kk = (l == 0 && cp.x_slab) ? sdesc_k16_plain(smem_u32(a_tile) + kk * BM * 32)
                                                         : ad + (uint64_t)(kk * 2);
            umma_f16_pair(d, a_kk, bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          }
          umma_commit_pair(&empty[s]);
          if (++s == C_STAGES) { s = 0; ph ^= 1; }
        }
        if (l == 0) {   // D += A_x B_x^T = u1[request(row)][n]
          const int b = fc1_t % C_NUX;
          cwait(&uxfull[b], (fc1_t / C_NUX) & 1, w_ux, ins);
          tc_fence_after();
          const uint32_t ux = smem_u32(sUX + b * C_UX_BUF);
          const uint64_t adx = sdesc_k16_plain(ux);
          umma_f16_pair(d, adx, sdesc_k16_plain(ux + C_UXA), id256, 1u);
          if (BF16) umma_f16_pair(d, adx, sdesc_k16_plain(ux + C_UXA + 2 * (C_BN / 2) * 16), id256, 1u);
          umma_commit_pair(&uxempty[b]);
          fc1_t++;
          if (XRES_KB > 0 && nb == ntile[0] - 1) {   // the block's FC1 MMAs are issued: X buffer free once done
            umma_commit_pair(xempty);
            x_t++;
          }
        }
        umma_commit_pair(&tfull[acc]);
        if (ins && l < 3) { wl_full[l] += w_full - fu0; wl_te[l] += w_tempty - te0; }
      });
      if (ins) {
        atomicAdd(cp.instr + 2, w_full); atomicAdd(cp.instr + 3, w_tempty); atomicAdd(cp.instr + 4, w_ux);
        atomicAdd(cp.instr + 6, (unsigned long long)(clock64() - t_begin));
        for (int l = 0; l < 3; l++) { atomicAdd(cp.instr + 8 + l, wl_full[l]); atomicAdd(cp.instr + 11 + l, wl_te[l]); }
      }
    }
  } else {
    // ===== epilogue warps 2..9 (both CTAs): TMEM lane quadrant q, column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const bool elected = (q == 0) && (lane == 0);
    const bool ins = cp.instr != nullptr && lane == 0;
    unsigned long long w_tfull = 0;
    int box_ctr = 0, uses0 = 0, uses1 = 0;
    for_tasks([&](int l, int j, int nb, int acc) {
      const int pm = pair + j * npairs;
      cwait(&tfull[acc], (uint32_t)((acc ? uses1++ : uses0++) & 1), w_tfull, ins);
      tc_fence_after();
      const int trow0 = pm * 2 * BM + (int)rank * BM;   // this CTA's first row of the block
      const int row = trow0 + q * 32 + lane;
      const float* u1row = nullptr;   // FC1 fallback: the pair block spans more than U1_NSLOT requests
      if (l == 0) {
        const int t0 = pm * 2 * BM;
        if (cp.req_of_ad[cp.a0 + min(t0 + 2 * BM, M) - 1] - (cp.req_of_ad[cp.a0 + t0] & ~7) >= U1_NSLOT) {
          const int req = row < M ? cp.req_of_ad[cp.a0 + row] : 0;
          u1row = cp.u1 + (int64_t)req * cp.ld_u1 + nb * C_BN;
        }
      }
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C_BN);
      if (TAIL && l == 2) {
        // FC3 -> H3 = ReLU(acc3 + b3), 16-bit, packed two per column into columns [64 h, 64 h + 64) of this
        // buffer (FC4's A operand); the quadrant's other warp must have read its acc3 columns first
        const float* b3 = sbias ? sBias + cp.n2 : cp.b3;
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
      } else if (TAIL && l == 3) {
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
      } else if (TAIL && l == 4) {
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
      } else {
        const int half = tn[l] / C_GROUPS;      // this group's columns of the tile
        const float* bias = l == 1 ? cp.b2 : (l == 2 ? cp.b3 : nullptr);
        uint32_t bias_s = 0u;   // smem address of this tile's bias columns (added like a u1 row)
        if (sbias && (l == 1 || l == 2)) {
          bias_s = smem_u32(sBias) + (uint32_t)((l == 1 ? 0 : cp.n2) + nb * tn[l]) * 4u;
          bias = nullptr;
        }
        const float* slope = l == 0 ? cp.s1 : (l == 1 ? cp.s2 : cp.s3);
#ifdef COLD_CHAIN_EPI_DBG   // timing experiment (results wrong): epi.cuh debug mode for one layer's epilogue
        const int edbg = l == COLD_CHAIN_EPI_DBG_L ? COLD_CHAIN_EPI_DBG : 0;
#else
        constexpr int edbg = 0;
#endif
        epi_store_wide<BF16>(tbase, h * half, (h + 1) * half, bias, bias_s, u1row, 1, sOut + h * EPI_GROUP_BOX, tC[l],
                             nb * tn[l], trow0, q, h, lane, edbg, cp.instr ? cp.instr + 16 + 8 * l : nullptr,
                             (FC1_DIRECT && l == 0) ? const_cast<void*>(cp.h1) : nullptr, cp.n1, M, 0ull, slope, C_OUT_BOXES == 2 * C_GROUPS ? sOut + (C_GROUPS + h) * EPI_GROUP_BOX : nullptr,
                             &box_ctr);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
      const bool last_of_layer = nb == ntile[l] - 1;
      if (FC1_DIRECT && l == 0) {
        // direct stores: this tile's H1 rows are written once every lane's stores are ordered before the
        // async-proxy (TMA) reads of FC2
        asm volatile("fence.proxy.async.global;" ::: "memory");
        named_bar_sync(1 + h, 128);
        if (lane == 0) mbar_arrive(&h1t[nb]);
      } else if (H1_TILES && l == 0) {
        // per-tile H1 readiness: tile nb - 1's stores are complete once at most this tile's two group stores
        // are pending (lazy: no wait on the tile just issued); the block's last tile waits for everything
        if (nb > 0) {
          if (elected) {
            bulk_wait_group<2>();
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          named_bar_sync(1 + h, 128);
          if (lane == 0) mbar_arrive(&h1t[nb - 1]);
        }
        if (last_of_layer) {
          if (elected) {
            bulk_wait_all();
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          named_bar_sync(1 + h, 128);
          if (lane == 0) mbar_arrive(&h1t[nb]);
        }
      } else if (l < 2 && last_of_layer) {
        // the block's rows of this layer are stored once this group's bulk stores completed
        if (elected) {
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        named_bar_sync(1 + h, 128);
        if (lane == 0) mbar_arrive(&hready[l]);
      }
      if ((l == 1 || l == 2) && last_of_layer) {
        // the input of this layer for the block (H1 for FC2, H2 for FC3) has been consumed by the MMAs
        // (tfull of the last tile): drop this CTA's rows from L2 without write-back
        const void* in_buf[3] = {nullptr, cp.h1, cp.h2};
        const int in_w[3] = {0, cp.n1, cp.n2};
        const uint8_t* base = reinterpret_cast<const uint8_t*>(in_buf[l]);
        const int ld = in_w[l] * 2;                            // bytes per row
        const int lines = ld / 128;
        const int rows = min(BM, M - trow0);
        for (int i = (ew * 32 + lane); i < rows * lines; i += C_EPI_WARPS * 32)
          discard_l2(base + (int64_t)(trow0 + i / lines) * ld + (i % lines) * 128);
      }
    });
    if (elected) bulk_wait_all();
    if (ins) atomicAdd(cp.instr + 5, w_tfull);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * C_BN) : "memory");
  }
}

bool chain_supported(int n1, int n2, int n3, int k1) {
  return n1 % C_BN == 0 && n2 % C_BN == 0 && n3 % C_BN == 0 && k1 % BK == 0 && n1 / BK >= 1;
}
// FC4 / FC5 / head in TMEM (TAIL): the paper's 256 -> 128 -> 64 -> head, in place in one C_BN-column buffer
bool chain_tail_supported(int n4, int n5, int n3) { return n3 == C_BN && n4 == 128 && n5 == 64; }

cudaError_t launch_chain(const CUtensorMap* tm[12], int M, int bf16, const ChainParams& cp, int num_sms, bool pdl,
                         cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  auto kern = bf16 ? (cp.tail ? chain_kernel<true, true> : chain_kernel<true, false>)
                   : (cp.tail ? chain_kernel<false, true> : chain_kernel<false, false>);
  static DevOnce attr[4];
  const int ai = (bf16 ? 2 : 0) + (cp.tail ? 1 : 0);
  if (attr[ai].first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_SMEM);
  }
  const int num_pm = (M + 2 * BM - 1) / (2 * BM);
  const int pairs = num_pm < num_sms / 2 ? num_pm : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(C_THREADS);
  cfg.dynamicSmemBytes = C_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, *tm[0], *tm[1], *tm[2], *tm[3], *tm[4], *tm[5], *tm[6], *tm[7], *tm[8],
                            *tm[9], *tm[10], *tm[11], M, cp);
}

}  // namespace cold
