// kernels_gemm.cu — one FC layer of the COLD stack on the 5th-generation tensor cores (sm_100a).
//
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )        A = activations, B = nn.Linear weight
//
// PAPER.md L328 (§4.1): FCN D_in x 1024 x 512 x 256 x 128 x 64 x 2; L276 "fully-connected layers
// use Float16"; L517 (Doc C) "involves almost only dense matrix multiplication, which needs
// extreme optimization". The paper ran fp16 HMMA on a T4 through an in-house engine; here each
// layer is a persistent, warp-specialised tcgen05 kernel launched as clusters of CS CTAs:
//   warp 0      : TMA producer. A (own 128 rows) is loaded per CTA; the weight tile B is split in
//                 CS row slices, each CTA loads one slice and multicasts it to the whole cluster,
//                 so L2 serves every weight byte once per cluster instead of once per CTA (the
//                 1-CTA kernel was L2-bandwidth bound: 87 FLOP/B at K=1024).
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per op).
//                 Its tcgen05.commit arrives on the stage's "empty" barrier of every CTA of the
//                 cluster (a slice is only overwritten once all CTAs have consumed it).
//   warps 2..9  : epilogue, two warps per TMEM lane quadrant (each owns half the columns):
//                 tcgen05.ld (32x32b) -> +bias [+ u1[request]] -> ReLU -> RNE cast -> 64B-swizzled
//                 shared tile -> TMA store (coalesced lines, rows past M clipped by the TMA unit).
//                 For the penultimate layer the last (1- or 2-wide) layer and the sigmoid are fused
//                 here instead and only the fp32 score leaves the kernel.
// The fp32 accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue of tile t
// overlaps the mainloop of tile t+1.
#include <cuda.h>
#include "internal.h"
#include "ptx.cuh"
#include "epi.cuh"

namespace cold {

constexpr int EPI_WARPS = 8;
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_COLS = 32;   // columns per TMEM load / TMA store box
constexpr int STAGE_OUT_BYTES = 32 * EPI_COLS * 2;   // one 32-row x 32-col fp16 box (2 KB)
constexpr int SMEM_LIMIT = 232448;                   // 227 KB opt-in per CTA
constexpr int RES_B_BYTES = 128 * 1024;              // resident weight slice budget

// RESB = false: A and B stream through a ring of stages (B optionally multicast in a cluster).
// RESB = true : the CTA owns one n-tile for the whole launch; its K x BN weight slice (<= 128 KB)
//               is loaded into shared memory once and only A streams (FC1: K=256, BN=256).
template <int BN, bool RESB> struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = RESB ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr int RES_BYTES = RESB ? RES_B_BYTES : 0;
  static constexpr int OUT_BYTES = EPI_WARPS * 2 * STAGE_OUT_BYTES;          // double-buffered per warp
  // staged u1 rows of FC1 (resident-weight mode only; streaming mode reads u1 from global)
  static constexpr int U1_BYTES = RESB ? 2 /*acc buffers*/ * 2 /*requests*/ * BN * 4 : 0;
  static constexpr int STAGES_FIT = (SMEM_LIMIT - RES_BYTES - OUT_BYTES - U1_BYTES - 1024 - 512) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int TMEM_COLS = 2 * BN;  // power of two >= 32
  static constexpr int SMEM =
      RES_BYTES + STAGES * STAGE_BYTES + OUT_BYTES + U1_BYTES + 1024 /*align*/ + 512 /*barriers*/;
};

// debug instrumentation: cycles a role spent blocked in a barrier wait
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, unsigned long long& acc, bool on) {
  if (!on) { mbar_wait(bar, parity); return; }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += (unsigned long long)(clock64() - t0);
}

// ---------------------------------------------------------------------------------------------
template <int BN, bool BF16, int CS, bool RESB>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, int M, int N, int K, EpiParams ep) {
  using Cfg = GemmCfg<BN, RESB>;
  static_assert(!RESB || CS == 1, "resident-B mode runs without clusters");
  constexpr int B_SLICE_ROWS = BN / CS;
  constexpr int B_SLICE_BYTES = B_SLICE_ROWS * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRes = smem;                                   // resident B: [K/64][BN rows x 128 B]
  uint8_t* sA = smem + Cfg::RES_BYTES;
  uint8_t* sB = sA + Cfg::STAGES * Cfg::A_BYTES;          // streaming B (RESB = false)
  uint8_t* sOut = smem + Cfg::RES_BYTES + Cfg::STAGES * Cfg::STAGE_BYTES;
  float* sU1 = reinterpret_cast<float*>(sOut + Cfg::OUT_BYTES);              // [2 acc][2 req][BN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + Cfg::OUT_BYTES + Cfg::U1_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + Cfg::STAGES;
  uint64_t* tfull = bars + 2 * Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;
  uint64_t* u1full = bres + 1;                                              // [2]
  int32_t* u1hdr = reinterpret_cast<int32_t*>(u1full + 2);                  // [2]: row boundary or -1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u1hdr + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = N / BN;
  const int kb_count = K / BK;
  // work decomposition. streaming: items = (CS m-tiles) x n-tile, clusters walk the item list.
  // resident: CTA -> fixed n-tile (blockIdx % num_n), m-tiles strided by the CTAs sharing it.
  const uint32_t crank = (CS > 1) ? cluster_rank() : 0;
  int first, stride, count;
  if (RESB) {
    const int groups = gridDim.x / num_n;
    first = blockIdx.x / num_n;
    stride = groups;
    count = num_m;
  } else {
    first = (CS > 1) ? (int)cluster_id_x() : blockIdx.x;
    stride = (CS > 1) ? (int)num_clusters_x() : gridDim.x;
    count = ((num_m + CS - 1) / CS) * num_n;
  }
  auto tile_of = [&](int it, int& mb, int& nb) {
    if (RESB) { mb = it; nb = blockIdx.x % num_n; }
    else { mb = (it / num_n) * CS + (int)crank; nb = it % num_n; }
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], CS); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI_WARPS); }
    mbar_init(bres, 1);
    mbar_init(&u1full[0], 1);
    mbar_init(&u1full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
    if (ep.out) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmC) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  if (CS > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();   // everything below reads or writes memory shared with the previous kernels

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_a = policy_evict_first();   // activations: streamed
      const uint64_t pol_b = policy_evict_last();    // weights: reused by every M tile
      if (RESB) {
        int nb0, mb0;
        tile_of(first, mb0, nb0);
        mbar_expect_tx(bres, (uint32_t)(kb_count * Cfg::B_BYTES));
        for (int kb = 0; kb < kb_count; kb++)
          tma_load_2d(sRes + kb * Cfg::B_BYTES, &tmB, bres, kb * BK, nb0 * BN, pol_b);
      }
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      const bool ins = ep.instr != nullptr;
      unsigned long long w_empty = 0;
      const long long t_start = clock64();
      for (int it = first; it < count; it += stride, lt++) {
        int mb, nb;
        tile_of(it, mb, nb);
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait_t(&empty[s], ph ^ 1, w_empty, ins);
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          tma_load_a(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb, mb * BM, pol_a, ep.a_slab != 0);
          if (!RESB) {
            uint8_t* dstB = sB + s * Cfg::B_BYTES + crank * B_SLICE_BYTES;
            if (CS > 1)
              tma_load_2d_mc(dstB, &tmB, &full[s], kb * BK, nb * BN + (int)crank * B_SLICE_ROWS,
                             (uint16_t)((1u << CS) - 1u), pol_b);
            else
              tma_load_2d(dstB, &tmB, &full[s], kb * BK, nb * BN, pol_b);
          }
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        if (RESB && ep.u1) {
          // FC1: stage this tile's u1 row slice(s) [nb*BN, +BN) into smem (<= 2 requests per tile;
          // more -> epilogue falls back to global loads). Buffer `acc` is free once tempty[acc] flips.
          const int acc = lt & 1;
          mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
          const int rlo = mb * BM, rhi = min(M, rlo + BM) - 1;
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
      if (ins) {
        atomicAdd(ep.instr + 0, w_empty);
        atomicAdd(ep.instr + 7, (unsigned long long)(clock64() - t_start));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (one thread) =====
      constexpr uint32_t idesc = idesc_f16<BN, BF16>();
      const bool ins = ep.instr != nullptr;
      unsigned long long w_full = 0, w_tempty = 0, w_bres = 0;
      if (RESB) mbar_wait_t(bres, 0, w_bres, ins);
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int it = first; it < count; it += stride, lt++) {
        const int acc = lt & 1;
        mbar_wait_t(&tempty[acc], ((lt >> 1) & 1) ^ 1, w_tempty, ins);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait_t(&full[s], ph, w_full, ins);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * Cfg::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(RESB ? sRes + kb * Cfg::B_BYTES : sB + s * Cfg::B_BYTES));
          if (ep.dbg_mode != 2) {
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; kk++) {   // +32 B along K inside the swizzle atom (slab: +4 KB)
              const uint64_t a_kk = ep.a_slab ? sdesc_k16_plain(smem_u32(sA + s * Cfg::A_BYTES) + kk * BM * 32)
                                              : ad + (uint64_t)(kk * 2);
              umma_f16(d, a_kk, bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
            }
          }
          if (CS > 1) umma_commit_mc(&empty[s], (uint16_t)((1u << CS) - 1u));
          else umma_commit(&empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
      if (ins) {
        atomicAdd(ep.instr + 1, w_full);
        atomicAdd(ep.instr + 2, w_tempty);
        atomicAdd(ep.instr + 3, w_bres);
      }
    }
  } else {
    // ===== epilogue warps 2..9: TMEM lane quadrant q, column half h =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int h = ew >> 2;
    const bool head = ep.head_n != 0;
    constexpr bool WIDE = (BN / 2) % EPI_WIDE_COLS == 0;   // 64-column SW128 store boxes
    // with a fused head one warp per quadrant walks all columns (the row's dot product stays in-thread)
    const int c_begin = head ? 0 : h * (BN / 2);
    const int c_end = head ? (h == 0 ? BN : 0) : (h + 1) * (BN / 2);
    uint8_t* my_out = sOut + ew * 2 * STAGE_OUT_BYTES;
    int ob = 0;
    int lt = 0;
    const bool ins = ep.instr != nullptr && lane == 0;
    unsigned long long w_tfull = 0, w_u1 = 0;
    for (int it = first; it < count; it += stride, lt++) {
      int mb, nb;
      tile_of(it, mb, nb);
      const int acc = lt & 1;
      mbar_wait_t(&tfull[acc], (lt >> 1) & 1, w_tfull, ins);
      tc_fence_after();
      const int row0 = mb * BM + q * 32;
      const int row = row0 + lane;
      const bool valid = row < M;
      uint32_t u1s = 0;                 // staged u1 row in shared memory (column nb*BN)
      const float* u1row = nullptr;      // points at column nb*BN of this row's u1 (smem or global)
      if (ep.u1) {
        int bnd = -1;
        if (RESB) {
          mbar_wait_t(&u1full[acc], (lt >> 1) & 1, w_u1, ins);
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
                             sOut + h * EPI_GROUP_BOX, &tmC, nb * BN, row0 - q * 32, q, h, lane, ep.dbg_mode,
                             nullptr, nullptr, 0, 0, 0ull, ep.slope);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        continue;
      }
      float z0 = 0.0f, z1 = 0.0f;
      const int c_stop = ep.dbg_mode == 1 ? c_begin : c_end;   // debug: drain nothing
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      // software-pipelined TMEM drain: the load of columns c+32 is in flight while c is processed
      uint32_t v[32];
      if (c_begin < c_stop) TMEM_LD32(taddr + c_begin, v);
      for (int c = c_begin; c < c_stop; c += EPI_COLS) {
        tmem_wait_ld();
        const int col0 = nb * BN + c;
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; i++) f[i] = __uint_as_float(v[i]);
        if (c + EPI_COLS < c_stop) TMEM_LD32(taddr + c + EPI_COLS, v);
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
          // 32 x 32 box, 64 B rows, SWIZZLE_64B: 16 B chunk j of row r sits at j ^ ((r >> 1) & 3)
          uint8_t* buf = my_out + ob * STAGE_OUT_BYTES;
          if (lane == 0) bulk_wait_read<1>();   // the store issued from this buffer 2 boxes ago has read it
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
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (head && h == 0 && valid) {
        float z;
        if (ep.head_n == 2) z = (z1 + ep.head_b[1]) - (z0 + ep.head_b[0]);
        else z = z0 + ep.head_b[0];
        ep.scores[row] = sigmoid(z);
      }
    }
    if (lane == 0) bulk_wait_all();
    if (ins) {
      atomicAdd(ep.instr + 4, w_tfull);
      atomicAdd(ep.instr + 5, w_u1);
      atomicAdd(ep.instr + 6, 1ull);
    }
  }
  tc_fence_before();
  if (CS > 1) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, bool BF16, int CS, bool RESB>
static cudaError_t launch_t(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N,
                            int K, const EpiParams& ep, int num_sms, bool pdl, cudaStream_t s) {
  using Cfg = GemmCfg<BN, RESB>;
  static DevOnce attr;
  auto kern = gemm_kernel<BN, BF16, CS, RESB>;
  if (attr.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (CS > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  const int num_m = (M + BM - 1) / BM;
  const int num_n = N / BN;
  int grid;
  if (RESB) {
    int groups = num_sms / num_n;
    if (groups > num_m) groups = num_m;
    if (groups < 1) groups = 1;
    grid = groups * num_n;
  } else {
    const int items = ((num_m + CS - 1) / CS) * num_n;
    static int max_clusters_dev[64] = {0};   // per device ordinal (occupancy is a per-device property)
    int dev = 0;
    cudaGetDevice(&dev);
    int& max_clusters = max_clusters_dev[dev & 63];
    if (max_clusters == 0) {
      max_clusters = num_sms / CS;
      if (CS > 1) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(CS * max_clusters);
        q.blockDim = dim3(GEMM_THREADS);
        q.dynamicSmemBytes = Cfg::SMEM;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CS;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n > 0) max_clusters = n;
        cudaGetLastError();
      }
    }
    grid = CS * (items < max_clusters ? items : max_clusters);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (CS > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = CS;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    na++;
  }
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, *tmA, *tmB, *tmC, M, N, K, ep);
}

bool gemm_resident_ok(int bn, int K) { return (int64_t)bn * K * 2 <= RES_B_BYTES; }

template <int BN, bool BF16>
static cudaError_t launch_mode(int cs, bool resb, const CUtensorMap* tmA, const CUtensorMap* tmB,
                               const CUtensorMap* tmC, int M, int N, int K, const EpiParams& ep, int num_sms, bool pdl,
                               cudaStream_t s) {
  if (resb) return launch_t<BN, BF16, 1, true>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  if (cs == 4) return launch_t<BN, BF16, 4, false>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  if (cs == 2) return launch_t<BN, BF16, 2, false>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  return launch_t<BN, BF16, 1, false>(tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
}

cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const CUtensorMap* tmC, int M, int N, int K,
                        int bn, int bf16, int cs, bool resb, const EpiParams& ep, int num_sms, bool pdl,
                        cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (bf16) {
    if (bn == 256) return launch_mode<256, true>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
    if (bn == 128) return launch_mode<128, true>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
    return launch_mode<64, true>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  }
  if (bn == 256) return launch_mode<256, false>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  if (bn == 128) return launch_mode<128, false>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
  return launch_mode<64, false>(cs, resb, tmA, tmB, tmC, M, N, K, ep, num_sms, pdl, s);
}

}  // namespace cold
