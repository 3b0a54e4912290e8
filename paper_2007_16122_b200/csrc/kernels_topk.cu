// kernels_topk.cu — segmented top-K (§2: pre-ranking "selects top N candidates
// by certain metrics, e.g. eCPM"; footnote / L332: eCPM = pCTR * bid).
//
// One CTA per request. Keys are mapped to order-preserving uint32 (NaN -> 0, the minimum).
// An 8-bit-digit MSB radix select (4 passes, shared-memory histograms, warp-aggregated
// atomics) finds the K-th largest key T. Keys > T are taken, keys == T are taken in position
// order (block-wide scan) until K — so ties resolve to ascending position (AMB-13) with no
// extra sort key. The K winners are then bitonic-sorted in shared memory on the 64-bit
// composite (key << 32 | ~position), descending.
#include "internal.h"

namespace cold {

constexpr int TOPK_THREADS = 1024;
constexpr int TOPK_MAX_K = 4096;
constexpr int TOPK_STAGE = 12288;   // keys of a segment staged in shared memory when n <= this (48 KB)

__device__ __forceinline__ uint32_t orderable(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0u;       // NaN ranks last
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float from_orderable(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(TOPK_THREADS) topk_kernel(TopkArgs a) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_need;
  __shared__ uint32_t s_gt_count, s_eq_base;
  __shared__ uint32_t warp_sums[TOPK_THREADS / 32];
  extern __shared__ unsigned long long cand[];            // [P] composites, P = pow2 >= K

  const int r = blockIdx.x;
  const bool merge = a.G > 0;
  const int64_t base = merge ? 0 : a.ad_offsets[r];
  const int n = merge ? a.G * a.Kl : (int)(a.ad_offsets[r + 1] - base);
  const int K = a.K;
  // merge mode: candidate i = (rank g, slot j) lives at [(g * R + r) * Kl + j]
  auto addr = [&](int i) -> int64_t {
    return merge ? ((int64_t)(i / a.Kl) * a.R + r) * a.Kl + (i % a.Kl) : base + i;
  };
  auto key_at = [&](int i) -> uint32_t {
    const int64_t ai = addr(i);
    float v = a.scores[ai];
    if (a.bids && !merge) v *= a.bids[ai];
    return orderable(v);
  };

  // keys read once from global into shared memory (the radix passes and the collect re-read them)
  int P = 1;
  while (P < K) P <<= 1;
  uint32_t* skey = reinterpret_cast<uint32_t*>(cand + P);
  const bool staged = n <= a.stage;
  if (staged) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) skey[i] = key_at(i);
    __syncthreads();
  }
  auto key = [&](int i) -> uint32_t { return staged ? skey[i] : key_at(i); };

  // ---- radix select: the K-th largest orderable key ----
  uint32_t prefix = 0, mask = 0, need = (uint32_t)K;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t u = key(i);
      if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp 0 finds the bin b (scanning from 255 down) where the running count reaches `need`: lane L
      // owns bins 255-8L .. 248-8L; an exclusive warp scan of the lane totals locates the lane, which
      // then walks its 8 bins (was: one thread walking up to 256 bins)
      const int L = threadIdx.x;
      uint32_t cnt[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) { cnt[i] = hist[255 - 8 * L - i]; tot += cnt[i]; }
      uint32_t incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if (L >= off) incl += v;
      }
      const uint32_t excl = incl - tot;
      const bool mine = excl < need && (incl >= need || L == 31);
      if (mine) {
        uint32_t cum = excl;
        int b = 255 - 8 * L;
        for (int i = 0; i < 8; i++, b--) {
          if (cum + cnt[i] >= need || b == 0) break;
          cum += cnt[i];
        }
        s_prefix = prefix | ((uint32_t)b << shift);
        s_need = need - cum;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t T = prefix;            // K-th largest key; `need` keys equal to T are taken

  // ---- collect: all keys > T (any order), then the first `need` keys == T by position ----
  if (threadIdx.x == 0) { s_gt_count = 0; s_eq_base = 0; }
  __syncthreads();
  const uint32_t n_gt = (uint32_t)K - need;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    uint32_t u = 0;
    bool gt = false, eq = false;
    if (i < n) { u = key(i); gt = u > T; eq = u == T; }
    if (gt) {
      const uint32_t slot = atomicAdd(&s_gt_count, 1u);
      cand[slot] = ((unsigned long long)u << 32) | (0xffffffffu - (uint32_t)i);
    }
    // ordered rank of eq among this tile
    const uint32_t bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_sums[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 32 warp counts by warp 0
      const uint32_t c = warp_sums[threadIdx.x];
      uint32_t incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        if ((int)threadIdx.x >= off) incl += v;
      }
      const uint32_t base = s_eq_base;
      __syncwarp();
      warp_sums[threadIdx.x] = base + incl - c;
      if (threadIdx.x == 31) s_eq_base = base + incl;
    }
    __syncthreads();
    if (eq) {
      const uint32_t rank = warp_sums[warp] + __popc(bal & ((1u << lane) - 1u));
      if (rank < need) cand[n_gt + rank] = ((unsigned long long)u << 32) | (0xffffffffu - (uint32_t)i);
    }
    __syncthreads();
  }
  for (int i = K + threadIdx.x; i < P; i += blockDim.x) cand[i] = 0ull;
  __syncthreads();
  // ---- bitonic sort, descending ----
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const unsigned long long x = cand[i], y = cand[j];
          if (desc ? (x < y) : (x > y)) { cand[i] = y; cand[j] = x; }
        }
      }
      __syncthreads();
    }
  }
  const int n_r = merge ? (int)(a.ad_offsets[r + 1] - a.ad_offsets[r]) : 0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const unsigned long long c = cand[i];
    const int w = (int)(0xffffffffu - (uint32_t)(c & 0xffffffffu));
    int32_t pos = w;
    if (merge) {   // slice-local position -> position within the request (split rule of cold_merge_topk)
      const int g = w / a.Kl;
      pos = a.cand_idx[addr(w)] + (int32_t)(((int64_t)g * n_r) / a.G);
    }
    a.idx[(int64_t)r * K + i] = pos;
    a.key[(int64_t)r * K + i] = from_orderable((uint32_t)(c >> 32));
  }
}

void launch_topk(const TopkArgs& a0, cudaStream_t s) {
  TopkArgs a = a0;
  int P = 1;
  while (P < a.K) P <<= 1;
  a.stage = (a.max_n > 0 && a.max_n <= TOPK_STAGE) ? a.max_n : 0;
  const size_t smem = (size_t)P * sizeof(unsigned long long) + (size_t)a.stage * sizeof(uint32_t);
  static DevOnce attr;
  if (attr.first()) {
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TOPK_MAX_K * (int)sizeof(unsigned long long) + TOPK_STAGE * (int)sizeof(uint32_t));
  }
  topk_kernel<<<a.R, TOPK_THREADS, smem, s>>>(a);
}

}  // namespace cold
