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
#ifdef COLD_TOPK_TIMING
#include <cstdio>
#endif

namespace cold {

constexpr int TOPK_THREADS = 1024;
constexpr int TOPK_MAX_K = 4096;
constexpr int TOPK_STAGE = 12288;   // keys of a segment staged in shared memory when n <= this (48 KB)

__device__ __forceinline__ uint32_t orderable(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0u;       // NaN ranks last
  if ((u & 0x7fffffffu) == 0u) u = 0u;                  // -0 == +0 (a tie, resolved by position)
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

// ---------------------------------------------------------------------------------------------
// Register-resident top-K for segments of <= 512 * KPT keys and K <= 512 (the latency path: one
// 4,000-ad request). The radix kernel above is issue-bound on its single SM there (~20 us: one CTA,
// 1024 threads; ncu r03d). Same result, bit for bit, in a fifth of the instructions:
//   * 512 threads; thread t owns positions t*KPT .. t*KPT+KPT-1 (blocked: thread order = position order);
//   * the nibbles all keys share are skipped (block AND / OR); then a radix select with 4-bit digits and
//     no atomics: each thread counts its keys per digit in 4-bit
//     fields of a 64-bit word (one shift-add per key, <= 8 keys per word), widens them to 16-bit
//     fields, a warp sums them with __reduce_add_sync, lane 0 publishes 8 words; after a barrier warp 0
//     sums the 16 warps' counts per bin (lane = bin), finds the digit with a 16-lane scan + ballot and
//     publishes it (second barrier; the per-round buffers alternate); stops as soon as the keys above the
//     prefix and all keys on it fit the sort (<= 512), which the sort then orders (3 rounds instead of 6
//     for a 4000-ad request's sigmoid keys);
//   * launched as a programmatic dependent of the scoring kernels (PDL): its launch overlaps their tail;
//   * collect: keys above the prefix in any order, keys equal to it by ascending position (one
//     block-wide exclusive scan of the packed (gt, eq) counts);
//   * bitonic sort of the <= 512 composites (key << 32 | ~position), descending, one per thread:
//     strides < 32 by warp shuffles, larger strides through shared memory (double-buffered).
constexpr int TOPK_SMALL_THREADS = 512;
constexpr int TOPK_SMALL_MAX_K = TOPK_SMALL_THREADS;

template <int KPT>
__global__ void __launch_bounds__(TOPK_SMALL_THREADS) topk_small_kernel(TopkArgs a) {
  constexpr int NW = TOPK_SMALL_THREADS / 32;
  constexpr int NC = (KPT + 7) / 8;                   // 64-bit nibble counters (<= 8 keys each: no carry)
  __shared__ __align__(16) uint32_t wcnt[2][NW][8];   // per-warp digit counts (bin b: word b/2, half b%2)
  __shared__ uint32_t wtot[NW];                       // per-warp packed (gt << 16 | eq) totals
  __shared__ uint4 sres[2];                           // per round: digit, its count, count above it
  __shared__ uint2 spre[NW];                          // per-warp AND / OR of the keys (common prefix)
  __shared__ unsigned long long sbuf[2][TOPK_SMALL_THREADS];
  const int r = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: the scores of the previous kernel
#ifdef COLD_TOPK_TIMING
  long long tm0 = clock64(), tm1 = 0, tm2 = 0, tm3 = 0, tm4 = 0;
  int nrounds = 0;
#endif
  const int64_t base = a.ad_offsets[r];
  const int n = (int)(a.ad_offsets[r + 1] - base);
  const int K = a.K;
  constexpr unsigned FULL = 0xffffffffu;

  uint32_t u[KPT];
  uint32_t valid = 0;
  {
    float v[KPT];
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      const int p = t * KPT + j;
      v[j] = p < n ? a.scores[base + p] : 0.0f;
    }
    if (a.bids) {
#pragma unroll
      for (int j = 0; j < KPT; j++) {
        const int p = t * KPT + j;
        if (p < n) v[j] *= a.bids[base + p];
      }
    }
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      u[j] = orderable(v[j]);
      if (t * KPT + j < n) valid |= 1u << j;
    }
  }

  // ---- radix select (4-bit digits, MSB first) ----
#ifdef COLD_TOPK_TIMING
  __syncthreads();
  tm1 = clock64();
#endif
  // the nibbles every valid key shares (sigmoid keys share their top bits) are resolved up front
  uint32_t kand = 0xffffffffu, kor = 0u;
#pragma unroll
  for (int j = 0; j < KPT; j++)
    if ((valid >> j) & 1u) { kand &= u[j]; kor |= u[j]; }
  kand = __reduce_and_sync(FULL, kand);
  kor = __reduce_or_sync(FULL, kor);
  if (lane == 0) spre[warp] = make_uint2(kand, kor);
  __syncthreads();
#pragma unroll
  for (int w = 0; w < NW; w++) { const uint2 v = spre[w]; kand &= v.x; kor |= v.y; }
  const uint32_t diff = kand ^ kor;
  const int shift0 = diff ? ((31 - __clz(diff)) & ~3) : -4;   // the highest nibble in which keys differ
  uint32_t mask = shift0 >= 28 ? 0u : (0xffffffffu << (shift0 + 4));
  uint32_t P = kand & mask, need = (uint32_t)K;
  uint32_t csel = (uint32_t)n;   // keys on the prefix (all of them until a digit is chosen)
  int round = 0;
  for (int shift = shift0; shift >= 0; shift -= 4, round++) {
    unsigned long long nib[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) nib[c] = 0ull;
#pragma unroll
    for (int j = 0; j < KPT; j++)
      if (((valid >> j) & 1u) && (u[j] & mask) == P) nib[j / 8] += 1ull << (((u[j] >> shift) & 15u) << 2);
    uint32_t pk[8];   // word w: bins 2w (low half) and 2w + 1 (high half)
#pragma unroll
    for (int w = 0; w < 8; w++) {
      uint32_t x = 0;
#pragma unroll
      for (int c = 0; c < NC; c++) {
        const uint32_t byte = (uint32_t)(nib[c] >> (8 * w)) & 0xffu;
        x += (byte & 15u) | ((byte >> 4) << 16);
      }
      pk[w] = __reduce_add_sync(FULL, x);
    }
    uint32_t (*buf)[8] = wcnt[round & 1];
    if (lane == 0) {
      reinterpret_cast<uint4*>(buf[warp])[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      reinterpret_cast<uint4*>(buf[warp])[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
    __syncthreads();
    if (warp == 0) {
      // lane l < 16 sums bin 15 - l over the warps; inclusive scan from the top bin; the first lane whose
      // running count reaches `need` holds the digit
      const int b = 15 - (lane & 15);
      uint32_t cb = 0;
      if (lane < 16) {
#pragma unroll
        for (int w = 0; w < NW; w++) cb += (buf[w][b >> 1] >> ((b & 1) << 4)) & 0xffffu;
      }
      uint32_t cum = cb;
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, cum, off);
        if ((lane & 15) >= off) cum += y;
      }
      const unsigned hit = __ballot_sync(FULL, lane < 16 && cum >= need);
      const int ls = __ffs(hit) - 1;
      if (lane == ls) sres[round & 1] = make_uint4((uint32_t)(15 - ls), cb, cum - cb, 0u);
    }
    __syncthreads();
    const uint4 res = sres[round & 1];
    csel = res.y;
    need -= res.z;
    P |= res.x << shift;
    mask |= 15u << shift;
    // the keys above the prefix and ALL keys on it fit the sort: stop resolving (the sort orders them)
    if ((uint32_t)K - need + csel <= (uint32_t)TOPK_SMALL_THREADS) break;
  }
  // take every key on the prefix (sorted below) when they fit, else the first `need` of them by position
  const bool take_all = (uint32_t)K - need + csel <= (uint32_t)TOPK_SMALL_THREADS;

  // ---- collect: keys above the prefix (any order), then the first `need` keys on it by position ----
#ifdef COLD_TOPK_TIMING
  tm2 = clock64();
  nrounds = round;
#endif
  const uint32_t n_gt = (uint32_t)K - need;
  uint32_t cnt = 0;   // packed (gt << 16) | eq for this thread
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    if ((valid >> j) & 1u) {
      const uint32_t m = u[j] & mask;
      cnt += m > P ? (1u << 16) : (m == P ? 1u : 0u);
    }
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  uint32_t wbase;
  {
    const uint32_t c = lane < NW ? wtot[lane] : 0u;
    uint32_t wi = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, wi, off);
      if (lane >= off) wi += y;
    }
    wbase = __shfl_sync(FULL, wi - c, warp);
  }
  const uint32_t excl = wbase + incl - cnt;
  uint32_t gslot = excl >> 16, erank = excl & 0xffffu;
  unsigned long long* cand = sbuf[0];
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    if ((valid >> j) & 1u) {
      const uint32_t m = u[j] & mask;
      const unsigned long long comp = ((unsigned long long)u[j] << 32) | (0xffffffffu - (uint32_t)(t * KPT + j));
      if (m > P) cand[gslot++] = comp;
      else if (m == P) {
        if (take_all || erank < need) cand[n_gt + erank] = comp;
        erank++;
      }
    }
  }
  __syncthreads();

  // ---- bitonic sort of the P2 = pow2 >= K composites, descending (threads >= P2 sort padding) ----
#ifdef COLD_TOPK_TIMING
  tm3 = clock64();
#endif
  const int S = take_all ? (int)(n_gt + csel) : K;   // candidates to sort (the first K are the result)
  int P2 = 1;
  while (P2 < S) P2 <<= 1;
  unsigned long long x = t < S ? cand[t] : 0ull;
  int cur = 1;   // sbuf[0] holds the candidates; the first exchange writes sbuf[1]
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      unsigned long long y;
      if (stride >= 32) {
        sbuf[cur][t] = x;
        __syncthreads();
        y = sbuf[cur][t ^ stride];
        cur ^= 1;
      } else {
        y = __shfl_xor_sync(FULL, x, stride);
      }
      // keep the larger of the pair where the lower index of a descending block (or the upper index
      // of an ascending one) sits
      const bool keep_hi = ((t & stride) == 0) == ((t & size) == 0);
      x = (keep_hi == (x > y)) ? x : y;
    }
  }
  if (t < K) {
    a.idx[(int64_t)r * K + t] = (int32_t)(0xffffffffu - (uint32_t)(x & 0xffffffffu));
    a.key[(int64_t)r * K + t] = from_orderable((uint32_t)(x >> 32));
  }
#ifdef COLD_TOPK_TIMING
  __syncthreads();
  tm4 = clock64();
  if (t == 0 && r == 0)
    printf("topk_small timing: load %lld select %lld (%d rounds) collect %lld sort+store %lld cycles\n", tm1 - tm0,
           tm2 - tm1, nrounds, tm3 - tm2, tm4 - tm3);
#endif
}

void launch_topk(const TopkArgs& a0, cudaStream_t s) {
  TopkArgs a = a0;
  if (a.G == 0 && a.K <= TOPK_SMALL_MAX_K && a.max_n > 0 && a.max_n <= 24 * TOPK_SMALL_THREADS) {
    auto kern = a.max_n <= 8 * TOPK_SMALL_THREADS    ? topk_small_kernel<8>
                : a.max_n <= 16 * TOPK_SMALL_THREADS ? topk_small_kernel<16>
                                                     : topk_small_kernel<24>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.R);
    cfg.blockDim = dim3(TOPK_SMALL_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
    return;
  }
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
