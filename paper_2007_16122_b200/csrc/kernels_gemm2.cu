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
//
// FC1 (U1): the per-request user block u1[request(row)] (fp32, hoisted, DESIGN A2) is added by the
// tensor core instead of the epilogue, as one extra K = 16 operand pair per tile:
//   A_x[row][k] = 1 if k % 8 is the slot of row's request in the 256-row pair tile, else 0
//   B_x[n][8 t + s] = t-th 16-bit term of u1[r_first + s][n]   (u1 = sum_t term_t to ~2^-22)
// with s = request - base, base = the pair tile's first request rounded down to 8 (TMA boxes must start
// 16 B aligned). D += A_x B_x^T = u1[request(row)][n]. A_x rows are written by the gather kernel (one-hot "column"),
// the terms by the user kernel ([t * H + n][r] layout, so 8 consecutive requests of one column are
// 16 contiguous bytes); both arrive by TMA like the other operands (box 8 x 128, no swizzle, K-major
// core matrices of 8 rows x 16 B: SBO = 128 B, LBO = 2 KB). f16 uses 2 terms (one MMA), bf16 3 terms
// (two MMAs, the 4th K chunk zero). The epilogue is then ReLU -> pack -> store only (the u1 loads and
// adds had made it the FC1 bottleneck). A pair tile whose requests do not fit in [base, base + 8) has
// all-zero A_x rows and its epilogue adds u1 from global memory instead.
#include <cuda.h>
#include "internal.h"
#include "ptx.cuh"
#include "epi.cuh"
#include "pair.cuh"

namespace cold {

constexpr int P_EPI_WARPS = 8;
constexpr int P_THREADS = 64 + 32 * P_EPI_WARPS;
constexpr int P_EPI_COLS = 32;
constexpr int P_OUT_BOX = 32 * P_EPI_COLS * 2;     // 2 KB staging box (32 rows x 32 cols)

// RES: the CTA pair owns one n-tile for the whole launch and keeps its weight half (BN/2 x K) resident in
// shared memory, so only A streams (FC1: K = 256, 64 KB per CTA). The GEMMs here are L2/TMA-bandwidth
// bound (FC1 moved ~30 B/cycle/SM with or without its epilogue); this halves FC1's operand traffic.
constexpr int P_RES_BYTES = 64 * 1024;

template <int BN, bool U1, bool RES = false> struct PairCfg {
  static constexpr int A_BYTES = BM * BK * 2;                 // own 128 rows
  static constexpr int B_BYTES = RES ? 0 : (BN / 2) * BK * 2; // own half of the weight tile (streamed)
  static constexpr int B_ATOM = (BN / 2) * BK * 2;            // one resident K block of the weight half
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RES_BYTES = RES ? P_RES_BYTES : 0;
  static constexpr int OUT_BYTES = P_EPI_WARPS * 2 * P_OUT_BOX;   // = P_EPI_WARPS * EPI_WIDE_BOX
  static constexpr int UXA_BYTES = BM * 32;                   // A_x: 128 rows x 16 halves (2 K chunks)
  static constexpr int UXB_BYTES = (BN / 2) * 16 * 4;         // B_x: own BN/2 columns x 4 K chunks of 8
  static constexpr int UX_BUF = UXA_BYTES + UXB_BYTES;
  static constexpr int NUX = 2;
  static constexpr int UX_BYTES = U1 ? NUX * UX_BUF : 0;
  static constexpr int STAGES_FIT = (232448 - RES_BYTES - OUT_BYTES - UX_BYTES - 1024 - 512) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int THREADS = P_THREADS;
  static constexpr int SMEM = RES_BYTES + STAGES * STAGE_BYTES + OUT_BYTES + UX_BYTES + 1024 + 512;
};

template <int BN, bool BF16, bool U1, bool RES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<BN, U1, RES>::THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmOH,
                     const __grid_constant__ CUtensorMap tmU1T, int M, int N, int K, EpiParams ep) {
  using Cfg = PairCfg<BN, U1, RES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRes = smem;                                        // RES: [K/64][BN/2 rows x 128 B]
  uint8_t* sA = smem + Cfg::RES_BYTES;
  uint8_t* sB = sA + Cfg::STAGES * Cfg::A_BYTES;
  uint8_t* sOut = sA + Cfg::STAGES * Cfg::STAGE_BYTES;
  uint8_t* sUX = sOut + Cfg::OUT_BYTES;                        // [NUX][A_x | B_x]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sUX + Cfg::UX_BYTES);
  uint64_t* full = bars;                          // leader: A+B bytes of both CTAs
  uint64_t* empty = bars + Cfg::STAGES;           // both: released by the leader's pair commit
  uint64_t* tfull = bars + 2 * Cfg::STAGES;       // both: accumulator ready
  uint64_t* tempty = tfull + 2;                   // leader: both CTAs' epilogues drained
  uint64_t* uxfull = tempty + 2;                  // leader: both CTAs' u1 operand bytes landed [NUX]
  uint64_t* uxempty = uxfull + Cfg::NUX;          // both: the u1 MMA of the buffer's last tile completed [NUX]
  uint64_t* bres = uxempty + Cfg::NUX;            // leader: resident weight halves of both CTAs landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = (int)cluster_id_x(), npairs = (int)num_clusters_x();
  const int num_pm = (M + 2 * BM - 1) / (2 * BM), num_n = N / BN;
  const int items = num_pm * num_n;
  const int kb_count = K / BK;
  // work list: streaming -> items (pm, nb) strided over all pairs; RES -> this pair's fixed n-tile,
  // m-tiles strided over the pairs sharing it (pairs beyond groups * num_n get no work)
  int w_first, w_step, w_count;
  if (RES) {
    const int groups = npairs / num_n;
    w_first = pair / num_n;
    w_step = groups > 0 ? groups : 1;
    w_count = (pair < groups * num_n) ? num_pm : 0;
  } else {
    w_first = pair;
    w_step = npairs;
    w_count = items;
  }
  auto tile_of = [&](int it, int& pm, int& nb) {
    if (RES) { pm = it; nb = pair % num_n; }
    else { pm = it / num_n; nb = it % num_n; }
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * P_EPI_WARPS); }
    for (int s = 0; s < Cfg::NUX; s++) { mbar_init(&uxfull[s], 1); mbar_init(&uxempty[s], 1); }
    mbar_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
    if (ep.out) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmC) : "memory");
    if (U1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmOH) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmU1T) : "memory");
    }
  }
  if (U1 && BF16 && warp == 2) {   // bf16: the 4th K chunk of every B_x buffer stays zero
    for (int b = 0; b < Cfg::NUX; b++)
      for (int i = lane; i < (BN / 2); i += 32)
        sts128(smem_u32(sUX + b * Cfg::UX_BUF + Cfg::UXA_BYTES + 3 * (BN / 2) * 16 + i * 16), make_uint4(0, 0, 0, 0));
    fence_async_smem();
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
  // PDL: everything that reads what earlier kernels wrote (A, the u1 operand, req_of_ad, biases in the
  // epilogue) waits for them; the producer first issues the weight loads, which do not depend on them
  if (warp != 0) pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      constexpr int TERMS = BF16 ? 3 : 2;
      auto pm_of = [&](int it) { int pm, nb; tile_of(it, pm, nb); return pm; };
      if (RES && w_count > 0) {   // this pair's weight half, once
        if (leader) mbar_expect_tx(bres, 2 * kb_count * Cfg::B_ATOM);
        for (int kb = 0; kb < kb_count; kb++)
          tma_load_2d_pair(sRes + kb * Cfg::B_ATOM, &tmB, bres, kb * BK, (pair % num_n) * BN + (int)rank * (BN / 2),
                           pol_b);
      }
      // streamed weights: the first tile's first STAGES weight k-blocks before the dependency wait
      int pre = 0;
      if (!RES && w_first < w_count) {
        int pm0, nb0;
        tile_of(w_first, pm0, nb0);
        pre = kb_count < Cfg::STAGES ? kb_count : Cfg::STAGES;
        for (int kb = 0; kb < pre; kb++) {
          if (leader) mbar_expect_tx(&full[kb], 2 * Cfg::STAGE_BYTES);
          tma_load_2d_pair(sB + kb * Cfg::B_BYTES, &tmB, &full[kb], kb * BK, nb0 * BN + (int)rank * (BN / 2), pol_b);
        }
      }
      pdl_wait();
      // the pair tile's first request rounded down to 8 (16 B-aligned TMA box start), prefetched
      int r_next = (U1 && w_first < w_count) ? (ep.req_of_ad[ep.a0 + pm_of(w_first) * 2 * BM] & ~7) : 0;
      for (int it = w_first; it < w_count; it += w_step, lt++) {
        int pm, nb;
        tile_of(it, pm, nb);
        const int mrow = pm * 2 * BM + (int)rank * BM;
        const int r_first = r_next;
        if (U1 && it + w_step < w_count) r_next = ep.req_of_ad[ep.a0 + pm_of(it + w_step) * 2 * BM] & ~7;
        for (int kb = 0; kb < kb_count; kb++) {
          if (pre > 0) {   // weights already in flight (stage kb of the first tile): only A
            tma_load_a_pair(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb, mrow, pol_a, ep.a_slab != 0);
            pre--;
            if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
            continue;
          }
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
          tma_load_a_pair(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb, mrow, pol_a, ep.a_slab != 0);
          if (!RES)
            tma_load_2d_pair(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * BK, nb * BN + (int)rank * (BN / 2), pol_b);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        if (U1) {   // the tile's u1 operand: A_x one-hot rows (2 boxes) + B_x term columns (TERMS boxes)
          const int b = lt % Cfg::NUX;
          mbar_wait(&uxempty[b], ((lt / Cfg::NUX) & 1) ^ 1);
          uint8_t* ux = sUX + b * Cfg::UX_BUF;
          if (leader) mbar_expect_tx(&uxfull[b], 2 * (Cfg::UXA_BYTES + TERMS * (BN / 2) * 16));
          tma_load_2d_pair(ux, &tmOH, &uxfull[b], 0, mrow, pol_a);
          tma_load_2d_pair(ux + BM * 16, &tmOH, &uxfull[b], 8, mrow, pol_a);
          const int n0 = nb * BN + (int)rank * (BN / 2);
#pragma unroll
          for (int t = 0; t < TERMS; t++)
            tma_load_2d_pair(ux + Cfg::UXA_BYTES + t * (BN / 2) * 16, &tmU1T, &uxfull[b], r_first, t * N + n0, pol_b);
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
      if (RES && w_count > 0) mbar_wait(bres, 0);
      for (int it = w_first; it < w_count; it += w_step, lt++) {
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * Cfg::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(RES ? sRes + kb * Cfg::B_ATOM : sB + s * Cfg::B_BYTES));
          if (ep.dbg_mode != 2) {
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; kk++) {
              const uint64_t a_kk = ep.a_slab ? sdesc_k16_plain(smem_u32(sA + s * Cfg::A_BYTES) + kk * BM * 32)
                                              : ad + (uint64_t)(kk * 2);
              umma_f16_pair(d, a_kk, bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
            }
          }
          umma_commit_pair(&empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        if (U1) {   // D += A_x B_x^T: the tile's u1[request(row)] block (K = 16 per term pair)
          const int b = lt % Cfg::NUX;
          mbar_wait(&uxfull[b], (lt / Cfg::NUX) & 1);
          tc_fence_after();
          const uint32_t ux = smem_u32(sUX + b * Cfg::UX_BUF);
          const uint64_t ad = sdesc_k16_plain(ux);
          umma_f16_pair(d, ad, sdesc_k16_plain(ux + Cfg::UXA_BYTES), idesc, 1u);                  // terms 0, 1
          if (BF16) umma_f16_pair(d, ad, sdesc_k16_plain(ux + Cfg::UXA_BYTES + 2 * (BN / 2) * 16), idesc, 1u);  // 2, 0
          umma_commit_pair(&uxempty[b]);
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 2 && warp < 2 + P_EPI_WARPS) {
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
    for (int it = w_first; it < w_count; it += w_step, lt++) {
      int pm, nb;
      tile_of(it, pm, nb);
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int row0 = pm * 2 * BM + (int)rank * BM + q * 32;
      const int row = row0 + lane;
      const bool valid = row < M;
      const uint32_t u1s = 0;
      const float* u1row = nullptr;     // fallback: u1 added here when the tile had too many requests
      if (ep.u1) {
        bool add_here = !U1;
        if (U1) {   // same rule as the gather's one-hot rows: more than U1_NSLOT requests in the pair tile
          const int t0 = pm * 2 * BM;
          add_here = ep.req_of_ad[ep.a0 + min(t0 + 2 * BM, M) - 1] - (ep.req_of_ad[ep.a0 + t0] & ~7) >= U1_NSLOT;
        }
        if (add_here) {
          const int req = valid ? ep.req_of_ad[ep.a0 + row] : 0;
          u1row = ep.u1 + (int64_t)req * ep.ld_u1 + nb * BN;
        }
      }
      if (WIDE && !head) {
        const int c_stop = ep.dbg_mode == 1 ? c_begin : c_end;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
        epi_store_wide<BF16>(tbase, c_begin, c_stop, ep.bias, u1s, u1row, ep.relu,
                             sOut + h * EPI_GROUP_BOX, &tmC, nb * BN, row0 - q * 32, q, h, lane, ep.dbg_mode,
                             ep.instr, nullptr, ep.ldo, M, 0ull, ep.slope);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
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
        if (ep.slope) {   // PReLU (F2)
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(ep.slope + col0 + i));
            f[i] = prelu(f[i], a.x); f[i + 1] = prelu(f[i + 1], a.y);
            f[i + 2] = prelu(f[i + 2], a.z); f[i + 3] = prelu(f[i + 3], a.w);
          }
        } else if (ep.relu) {
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
      if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
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

template <int BN, bool BF16, bool U1, bool RES>
static cudaError_t launch_pair_t(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC,
                                 const CUtensorMap* tmOH, const CUtensorMap* tmU1T, int M, int N, int K,
                                 const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s) {
  using Cfg = PairCfg<BN, U1, RES>;
  auto kern = gemm_pair_kernel<BN, BF16, U1, RES>;
  static DevOnce attr;
  if (attr.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
  }
  const int num_pm = (M + 2 * BM - 1) / (2 * BM), num_n = N / BN;
  const int items = num_pm * num_n;
  int pairs = items < num_sms / 2 ? items : num_sms / 2;
  if (RES) {   // whole groups of num_n pairs (one per n-tile), no more groups than m-tiles
    int groups = (num_sms / 2) / num_n;
    if (groups > num_pm) groups = num_pm;
    if (groups < 1) groups = 1;
    pairs = groups * num_n;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 1 : 0;
  // tmOH / tmU1T are only read by the U1 variant; the others get tmA as a placeholder
  return cudaLaunchKernelEx(&cfg, kern, *tmA, *tmB, *tmC, U1 ? *tmOH : *tmA, U1 ? *tmU1T : *tmA, M, N, K, ep);
}

bool gemm_pair_resident_ok(int bn, int K) { return (int64_t)(bn / 2) * K * 2 <= P_RES_BYTES; }

cudaError_t launch_gemm_pair(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N,
                             int K, int bn, int bf16, const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s,
                             const CUtensorMap* tmOH, const CUtensorMap* tmU1T, bool res) {
  if (M <= 0) return cudaSuccess;
  // U1 variant: u1[request(row)] added on the tensor core (needs the one-hot rows and the u1 terms)
  const bool u1 = ep.u1 != nullptr && tmOH != nullptr && tmU1T != nullptr;
  res = res && gemm_pair_resident_ok(bn, K);
#define PAIR_ARGS tmA, tmB, tmC, tmOH, tmU1T, M, N, K, ep, num_sms, pdl, s
#define PAIR_CASE(BNV)                                                                                 \
  if (bn == BNV) {                                                                                     \
    if (bf16) {                                                                                        \
      if (u1) return res ? launch_pair_t<BNV, true, true, true>(PAIR_ARGS)                             \
                         : launch_pair_t<BNV, true, true, false>(PAIR_ARGS);                           \
      return res ? launch_pair_t<BNV, true, false, true>(PAIR_ARGS)                                    \
                 : launch_pair_t<BNV, true, false, false>(PAIR_ARGS);                                  \
    }                                                                                                  \
    if (u1) return res ? launch_pair_t<BNV, false, true, true>(PAIR_ARGS)                              \
                       : launch_pair_t<BNV, false, true, false>(PAIR_ARGS);                            \
    return res ? launch_pair_t<BNV, false, false, true>(PAIR_ARGS)                                     \
               : launch_pair_t<BNV, false, false, false>(PAIR_ARGS);                                   \
  }
  PAIR_CASE(256)
  PAIR_CASE(128)
  PAIR_CASE(64)
#undef PAIR_CASE
#undef PAIR_ARGS
  return cudaErrorInvalidValue;
}

}  // namespace cold
