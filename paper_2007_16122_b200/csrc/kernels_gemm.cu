// kernels_gemm.cu — one FC layer of the COLD stack on the 5th-generation tensor cores (sm_100a).
//
//   out[M, N] = epilogue( A[M, K] . B[N, K]^T )        A = activations, B = nn.Linear weight
//
// PAPER.md L328 (§4.1): FCN D_in x 1024 x 512 x 256 x 128 x 64 x 2; L276 "fully-connected layers
// use Float16"; L517 (Doc C) "involves almost only dense matrix multiplication, which needs
// extreme optimization". The paper ran fp16 HMMA on a T4 through an in-house engine; here each
// layer is a persistent, warp-specialised tcgen05 kernel:
//   warp 0      : TMA producer  (cp.async.bulk.tensor, 128 B swizzle, mbarrier complete_tx)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per op)
//   warps 2..5  : epilogue — tcgen05.ld (32x32b) -> +bias [+ u1[request]] -> ReLU -> RNE cast
//                 -> global; for the penultimate layer the last (1- or 2-wide) layer and the
//                 sigmoid are fused here and only the fp32 score leaves the kernel.
// The fp32 accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue of tile t
// overlaps the mainloop of tile t+1.
#include <cuda.h>
#include "internal.h"

namespace cold {

constexpr int BM = 128;        // UMMA M (cta_group::1)
constexpr int BK = 64;         // K per stage: 64 x 16-bit = 128 B rows = one SW128 atom
constexpr int UMMA_K = 16;
constexpr int GEMM_THREADS = 192;

template <int BN> struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // power of two >= 32
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// ---- PTX wrappers ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor, K-major, 128 B swizzle (tcgen05 "version 1" format):
// start>>4 [0,14) | LBO>>4 [16,30) (unused for swizzled K-major, 1) | SBO>>4 [32,46) = 1024 B
// (8 rows x 128 B) | version 1 [46,48) | base offset 0 | layout SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32 [4,6)=1, A/B format [7,10)/[10,13) (0 f16, 1 bf16),
// K-major A and B, N>>3 at [17,23), M>>4 at [24,29).
template <int BN, bool BF16>
__device__ __forceinline__ constexpr uint32_t idesc_f16() {
  return (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define TMEM_LD32(taddr, v)                                                                                  \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                             \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),           \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),           \
        "=r"(v[30]), "=r"(v[31])                                                                             \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <bool BF16> struct Pack;
template <> struct Pack<false> {
  static __device__ __forceinline__ uint32_t two(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <> struct Pack<true> {
  static __device__ __forceinline__ uint32_t two(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

// ---------------------------------------------------------------------------------------------
template <int BN, bool BF16>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                int K, EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + Cfg::STAGES;
  uint64_t* tfull = bars + 2 * Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int kb_count = K / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; s++) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_a = policy_evict_first();   // activations: streamed once per N tile
      const uint64_t pol_b = policy_evict_last();    // weights: reused by every M tile
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mb = t / num_n, nb = t % num_n;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * BK, mb * BM, pol_a);
          tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * BK, nb * BN, pol_b);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (one thread) =====
      constexpr uint32_t idesc = idesc_f16<BN, BF16>();
      int s = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_count; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sA + s * Cfg::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + s * Cfg::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; kk++)   // +32 B along K inside the swizzle atom
            umma_f16(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
          umma_commit(&empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue warps 2..5: TMEM lanes [32*(warp%4), +32) =====
    const int q = warp & 3;
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, lt++) {
      const int mb = t / num_n, nb = t % num_n;
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int row = mb * BM + q * 32 + lane;
      const bool valid = row < M;
      const float* u1row = nullptr;
      if (ep.u1) {
        const int req = valid ? ep.req_of_ad[ep.a0 + row] : 0;
        u1row = ep.u1 + (int64_t)req * ep.ld_u1;
      }
      float z0 = 0.0f, z1 = 0.0f;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        TMEM_LD32(taddr + c, v);
        tmem_wait_ld();
        const int col0 = nb * BN + c;
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; i++) f[i] = __uint_as_float(v[i]);
        if (ep.bias) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + i));
            f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
          }
        }
        if (u1row) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(u1row + col0 + i));
            f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
          }
        }
        if (ep.relu) {
#pragma unroll
          for (int i = 0; i < 32; i++) f[i] = fmaxf(f[i], 0.0f);
        }
        if (ep.head_n) {
#pragma unroll
          for (int i = 0; i < 32; i++) z0 = fmaf(__ldg(ep.head_w + col0 + i), f[i], z0);
          if (ep.head_n == 2) {
#pragma unroll
            for (int i = 0; i < 32; i++) z1 = fmaf(__ldg(ep.head_w + N + col0 + i), f[i], z1);
          }
        } else if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(ep.out) + (int64_t)row * ep.ldo + col0);
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 w;
            w.x = Pack<BF16>::two(f[i], f[i + 1]);
            w.y = Pack<BF16>::two(f[i + 2], f[i + 3]);
            w.z = Pack<BF16>::two(f[i + 4], f[i + 5]);
            w.w = Pack<BF16>::two(f[i + 6], f[i + 7]);
            dst[i / 8] = w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (ep.head_n && valid) {
        float z;
        if (ep.head_n == 2) z = (z1 + ep.head_b[1]) - (z0 + ep.head_b[0]);
        else z = z0 + ep.head_b[0];
        ep.scores[row] = sigmoid(z);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

int gemm_smem_bytes(int bn) {
  switch (bn) {
    case 256: return GemmCfg<256>::SMEM;
    case 128: return GemmCfg<128>::SMEM;
    default: return GemmCfg<64>::SMEM;
  }
}

template <int BN, bool BF16>
static void launch_t(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, const EpiParams& ep,
                     int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel<BN, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::SMEM);
    attr = true;
  }
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  gemm_kernel<BN, BF16><<<grid, GEMM_THREADS, GemmCfg<BN>::SMEM, s>>>(*tmA, *tmB, M, N, K, ep);
}

void launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, int bn, int bf16,
                 const EpiParams& ep, int num_sms, cudaStream_t s) {
  if (M <= 0) return;
  if (bf16) {
    if (bn == 256) launch_t<256, true>(tmA, tmB, M, N, K, ep, num_sms, s);
    else if (bn == 128) launch_t<128, true>(tmA, tmB, M, N, K, ep, num_sms, s);
    else launch_t<64, true>(tmA, tmB, M, N, K, ep, num_sms, s);
  } else {
    if (bn == 256) launch_t<256, false>(tmA, tmB, M, N, K, ep, num_sms, s);
    else if (bn == 128) launch_t<128, false>(tmA, tmB, M, N, K, ep, num_sms, s);
    else launch_t<64, false>(tmA, tmB, M, N, K, ep, num_sms, s);
  }
}

}  // namespace cold
