// kernels_gather.cu — feature side of the scoring pass (sm_100a).
//
//  user_kernel   : per request, the selected USER groups once (gather -> sum-pool -> linear_log
//                  -> SE -> x_u), then the hoisted FC1 user block u1 = b1 + W1_u x_u (fp32).
//                  SURVEY §8 A2; PAPER.md L248 ("duplicated computation related to user
//                  features" — removed here: one user gather per request, broadcast to all ads).
//  gather_kernel : column-wise ("column based computation"): grid.y = one selected
//                  AD/CROSS group, threads = consecutive ads. Cross rows are hashed from the user
//                  bag x the ad bag (AMB-9), rows gathered with 16 B vector loads, pooled in fp32
//                  in bag order, linear_log -> SE gate -> v -> RNE cast into X_ac (A3-A5).
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace cold {

// 256-bit global access (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256): a 32 B table row is one request
// and one L1 sector lookup instead of two 16 B ones (the gather was L1TEX-throughput bound).
__device__ __forceinline__ void ldg256(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

template <typename T, int K>
__device__ __forceinline__ void add_row(const T* __restrict__ table, int64_t row, float* e) {
  constexpr int BYTES = K * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {          // 16 B vector loads (k=16 fp16: one 32 B sector)
    const uint4* p = reinterpret_cast<const uint4*>(table + row * K);
    uint4 qv[BYTES / 16];
    if constexpr (BYTES % 32 == 0) {
#pragma unroll
      for (int v = 0; v < BYTES / 16; v += 2) ldg256(p + v, qv[v], qv[v + 1]);
    } else {
#pragma unroll
      for (int v = 0; v < BYTES / 16; v++) qv[v] = __ldg(p + v);
    }
#pragma unroll
    for (int v = 0; v < BYTES / 16; v++) {
      const T* t = reinterpret_cast<const T*>(&qv[v]);
#pragma unroll
      for (int i = 0; i < 16 / (int)sizeof(T); i++) e[v * (16 / sizeof(T)) + i] = Store<T>::add(e[v * (16 / sizeof(T)) + i], t[i]);
    }
  } else {                                   // tiny rows (k = 2, 4)
#pragma unroll
    for (int d = 0; d < K; d++) e[d] = Store<T>::add(e[d], table[row * K + d]);
  }
}

__device__ __forceinline__ int64_t checked(int64_t id, int64_t card, int validate, int* err) {
  if (id < 0 || id >= card) {
    if (validate) atomicOr(err, 1);
    id = id < 0 ? 0 : card - 1;
  }
  return id;
}

// ---------------------------------------------------------------------------------------------
// user side: grid = (R requests, S output slices), block = 256 threads. Every CTA of a request pools
// the request's user groups (cheap: ~84 rows); the CTA with blockIdx.y == 0 also writes x_u, the
// ad -> request map, statistics and debug outputs. The hoisted GEMV u1 = b1 + W1_u x_u is split over
// the S CTAs in 64-output passes (S > 1, up to 16, when few requests are in flight: the single-request
// latency path).
// Bag pooling: the warp loads up to 32 rows of a bag in parallel (one row per lane, 256-bit), stages
// them in shared memory and lane d sums dimension d sequentially in bag order (the fp32 order the
// oracle's fp32-ordered mode defines), instead of a dependent id -> row chain per bag element.
template <typename T, int K>
__global__ void __launch_bounds__(256) user_kernel(UserArgs a) {
  extern __shared__ float xs[];           // [n_user * K] then per-warp row stage [8][32][K]
  float* stage = xs + ((a.n_user * K + 3) & ~3);
  const int r = blockIdx.x;
  const bool main_cta = blockIdx.y == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d_u = a.n_user * K;
  float* wst = stage + warp * 32 * K;
  // one warp per selected user group; lane d < K owns dimension d
  for (int j = warp; j < a.n_user; j += blockDim.x / 32) {
    const int g = a.user_g[j];
    const DevGroup G = a.groups[g];
    const BatchGroup& B = a.bv.g[g];
    const int64_t o0 = (int64_t)B.offs[r - B.offs_shift] - B.val_shift;
    const int64_t o1 = (int64_t)B.offs[r + 1 - B.offs_shift] - B.val_shift;
    float e = 0.0f;
    const T* tab = reinterpret_cast<const T*>(G.table);
    for (int64_t c0 = o0; c0 < o1; c0 += 32) {
      const int cnt = (int)min((int64_t)32, o1 - c0);
      if (lane < cnt) {                      // lane i fetches bag element c0 + i
        const int64_t row = checked(B.ids[c0 + lane], G.card, a.validate, a.err);
#pragma unroll
        for (int d = 0; d < K; d++) wst[lane * K + d] = Store<T>::to_f(tab[row * K + d]);
      }
      __syncwarp();
      if (lane < K)
        for (int i = 0; i < cnt; i++) e += wst[i * K + lane];
      __syncwarp();
    }
    float pooled = e;
    if (a.linear_log) e = linear_log(e);
    if (a.dense) {                          // dense SE: the gate needs the ad's columns (se_dense_kernel)
      if (lane < K) {
        xs[j * K + lane] = e;
        if (main_cta) {
          a.xu[(int64_t)r * d_u + j * K + lane] = e;
          if (a.dbg_pooled)
            for (int64_t ad = a.ad_offsets[r]; ad < a.ad_offsets[r + 1]; ad++)
              a.dbg_pooled[(ad * a.n_sel + G.sel_pos) * K + lane] = pooled;
        }
      }
      continue;
    }
    float z = (lane < K) ? a.se_w[g * K + lane] * e : 0.0f;
#pragma unroll
    for (int off = 16; off; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    const float s = sigmoid(z + a.se_b[g]);
    if (a.stats) {                          // SE statistics: every ad of the request shares s_g
      if (lane == 0 && main_cta)
        atomicAdd(a.stats + g, (double)s * (double)(a.ad_offsets[r + 1] - a.ad_offsets[r]));
      continue;
    }
    if (lane < K) {
      float v = s * e;
      if (a.in_scale) {                     // folded input batch norm (fp32, F2)
        const int col = G.sel_pos * K + lane;
        v = fmaf(v, a.in_scale[col], a.in_shift[col]);
      }
      xs[j * K + lane] = v;
      if (main_cta) {
        a.xu[(int64_t)r * d_u + j * K + lane] = v;
        if (a.dbg_pooled || a.dbg_feat) {
          const int pos = G.sel_pos;
          for (int64_t ad = a.ad_offsets[r]; ad < a.ad_offsets[r + 1]; ad++) {
            if (a.dbg_pooled) a.dbg_pooled[(ad * a.n_sel + pos) * K + lane] = pooled;
            if (a.dbg_feat) a.dbg_feat[ad * a.d_in + pos * K + lane] = v;
          }
        }
      }
    }
  }
  __syncthreads();
  // u1[r][o] = b1[o] + sum_i W1u[o][i] x_u[i]   (W1u stored transposed: coalesced over o)
  // 64 outputs per pass, 4 threads per output: thread part q sums inputs [q*P, q*P + P) (up to 32 weight
  // loads in flight, one L2 round trip instead of d_u / 16 dependent ones); after one barrier the four
  // partial sums of each output are added in part order. The order is fixed, so u1 does not depend on the
  // slice count or on the other requests of the call.
  float* part = xs + a.part_off;   // [4][H] partial sums
  const int q = threadIdx.x >> 6, ol = threadIdx.x & 63;
  const int P = (d_u + 3) / 4;
  const int i0 = min(q * P, d_u), i1 = min(i0 + P, d_u);
  const int npass = (a.H + 63) / 64;
  if (!a.stats) {
    for (int pass = blockIdx.y; pass < npass; pass += gridDim.y) {
      const int o = pass * 64 + ol;
      float acc = 0.0f;
      if (!a.dense && o < a.H) {   // dense SE: W1's user columns run inside FC1 with the gated per-ad x (u1 = b1)
        int i = i0;
        for (; i + 32 <= i1; i += 32) {
          float w[32];
#pragma unroll
          for (int j = 0; j < 32; j++) w[j] = __ldg(a.w1u_t + (int64_t)(i + j) * a.H + o);
#pragma unroll
          for (int j = 0; j < 32; j++) acc = fmaf(w[j], xs[i + j], acc);
        }
        for (; i + 8 <= i1; i += 8) {
          float w[8];
#pragma unroll
          for (int j = 0; j < 8; j++) w[j] = __ldg(a.w1u_t + (int64_t)(i + j) * a.H + o);
#pragma unroll
          for (int j = 0; j < 8; j++) acc = fmaf(w[j], xs[i + j], acc);
        }
        for (; i < i1; i++) acc = fmaf(__ldg(a.w1u_t + (int64_t)i * a.H + o), xs[i], acc);
      }
      if (o < a.H) part[q * a.H + o] = acc;
    }
    __syncthreads();
    for (int pass = blockIdx.y; pass < npass; pass += gridDim.y) {
      if (q != 0) break;
      const int o = pass * 64 + ol;
      if (o >= a.H) continue;
      const float acc = a.b1[o] + part[o] + part[a.H + o] + part[2 * a.H + o] + part[3 * a.H + o];
      a.u1[(int64_t)r * a.H + o] = acc;
      if (a.u1t) {   // u1 = term_0 + term_1 (+ term_2), each RNE in 16 bits: the FC1 tensor-core operand
        float u = acc;
        for (int t = 0; t < a.u1_terms; t++) {
          uint16_t bits;
          if (a.bf16) {
            const __nv_bfloat16 qq = __float2bfloat16_rn(u);
            bits = __bfloat16_as_ushort(qq);
            u -= __bfloat162float(qq);
          } else {
            const __half qq = __float2half_rn(u);
            bits = __half_as_ushort(qq);
            u -= __half2float(qq);
          }
          a.u1t[((int64_t)t * a.H + o) * a.u1t_ld + r] = bits;
        }
      }
    }
  }
  if (main_cta) {   // bounds in registers: the stores may alias ad_offsets, which would reload it per step
    const int64_t e0 = a.ad_offsets[r], e1 = a.ad_offsets[r + 1];
    for (int64_t ad = e0 + threadIdx.x; ad < e1; ad += blockDim.x) a.req_of_ad[ad] = r;
  }
}

// ---------------------------------------------------------------------------------------------
// ad + cross side: grid = (ceil(n / (128 * APT)), n_ac), block = 128 threads. blockIdx.y is one
// selected AD/CROSS group (column-wise), walked heaviest-first; thread t of block b owns the
// APT ads b*128*APT + t + i*128 (i < APT), so every id / X access of a warp stays coalesced.
// The kernel is bound by memory-level parallelism (random 32 B rows; one row per thread in flight
// left DRAM at 28% and L2 at 47% busy), so rows are fetched as raw 16 B vectors into registers, up to
// RB rows per thread in flight, and only then summed — still sequentially in bag order (x-major for
// cross bags), which keeps the fp32 pooled sums bit-identical to the oracle's fp32-ordered mode.
// A cross group's user-side half of the hash, hx = fmix64(x ^ salt_g), depends only on the request:
// a block spanning <= 2 requests hashes their user bags once into shared memory (AMB-9).
constexpr int GATHER_APT_BIG = 4;   // ads per thread on large spans
constexpr int HX_HALF = 256;        // user-bag hashes cached per request slot

template <typename T, int K>
struct RawRow {
  static constexpr int NV = K * (int)sizeof(T) / 16;   // 16 B vectors per row (>= 1 on the fast path)
  uint4 q[NV > 0 ? NV : 1];
  __device__ __forceinline__ void load(const T* __restrict__ table, int64_t row) {
    const uint4* p = reinterpret_cast<const uint4*>(table + row * K);
    if constexpr (NV % 2 == 0) {
#pragma unroll
      for (int v = 0; v < NV; v += 2) ldg256(p + v, q[v], q[v + 1]);
    } else {
#pragma unroll
      for (int v = 0; v < NV; v++) q[v] = __ldg(p + v);
    }
  }
  __device__ __forceinline__ void add_to(float* e) const {
#pragma unroll
    for (int v = 0; v < NV; v++) {
      const T* t = reinterpret_cast<const T*>(&q[v]);
#pragma unroll
      for (int i = 0; i < 16 / (int)sizeof(T); i++) e[v * (16 / sizeof(T)) + i] = Store<T>::add(e[v * (16 / sizeof(T)) + i], t[i]);
    }
  }
};

// group descriptors of the gather: from the kernel parameters (constant bank, no dependent global
// load at CTA start) unless the A/B build asks for the device array
#ifdef COLD_GATHER_GLOBAL_GROUPS
#define GGROUP(a, g) ((a).groups[g])
#else
#define GGROUP(a, g) ((a).gp[g])
#endif

// pooled e -> [debug] -> linear_log -> SE gate -> v = s ê -> RNE cast -> X_ac[local][slot]
// sew / seb: the group's SE weights in global memory; jcol >= 0 with a.sew_in_params: read them from the
// kernel parameters instead (a.sew_c[jcol * K + d], a.seb_c[jcol]: uniform constant-bank loads, no LSU)
template <typename T, int K, bool FAST>
__device__ __forceinline__ void finish_ad(const GatherArgs& a, const DevGroup& G, int g, int64_t local, float* e,
                                          const float* sew, float seb, int jcol) {
  const int64_t ad = a.a0 + local;
  if (a.dbg_pooled) {
#pragma unroll
    for (int d = 0; d < K; d++) a.dbg_pooled[(ad * a.n_sel + G.sel_pos) * K + d] = e[d];
  }
  if (a.linear_log) {
#pragma unroll
    for (int d = 0; d < K; d++) e[d] = linear_log_t<FAST>(e[d]);
  }
  if (a.E) {                                // dense SE: store ê (fp32); the gate runs in se_dense_kernel
    float* dst = a.E + local * a.lde + G.sel_pos * K;
    if constexpr (K % 4 == 0) {
#pragma unroll
      for (int d = 0; d < K; d += 4) *reinterpret_cast<float4*>(dst + d) = make_float4(e[d], e[d + 1], e[d + 2], e[d + 3]);
    } else {
#pragma unroll
      for (int d = 0; d < K; d++) dst[d] = e[d];
    }
    return;
  }
  float z = 0.0f;
  if (a.sew_in_params && jcol >= 0) {
#pragma unroll
    for (int d = 0; d < K; d++) z = fmaf(a.sew_c[jcol * K + d], e[d], z);
    seb = a.seb_c[jcol];
  } else {
#pragma unroll
    for (int d = 0; d < K; d++) z = fmaf(__ldg(sew + d), e[d], z);
  }
  const float s = sigmoid_t<FAST>(z + seb);
  if (a.stats) {                            // SE statistics mode (cold_se_stats)
    atomicAdd(a.stats + g, (double)s);
    return;
  }
  alignas(16) T out[K];
  if (a.in_scale) {                         // folded input batch norm in fp32 before the cast (F2)
    const int col = G.sel_pos * K;
#pragma unroll
    for (int d = 0; d < K; d++) out[d] = Store<T>::from_f(fmaf(s * e[d], __ldg(a.in_scale + col + d), __ldg(a.in_shift + col + d)));
  } else {
#pragma unroll
    for (int d = 0; d < K; d++) out[d] = Store<T>::from_f(s * e[d]);
  }
  constexpr int BYTES = K * (int)sizeof(T);
  if constexpr (sizeof(T) == 2 && K % 8 == 0) {
    if (a.x_slab) {   // half-slab layout: 8 columns (16 B) per plane, consecutive ads contiguous in a plane, so a
      //               warp's stores are 512 B runs (4 full lines) instead of 32 scattered 32 B sectors
      T* xb = reinterpret_cast<T*>(a.X);
#pragma unroll
      for (int v = 0; v < K / 8; v++)
        reinterpret_cast<uint4*>(xb + ((int64_t)(G.sel_slot * (K / 8) + v) * a.x_rows + local) * 8)[0] =
            reinterpret_cast<const uint4*>(out)[v];
      if (a.dbg_feat) {
#pragma unroll
        for (int d = 0; d < K; d++) a.dbg_feat[ad * a.d_in + G.sel_pos * K + d] = Store<T>::to_f(out[d]);
      }
      return;
    }
  }
  T* dst = reinterpret_cast<T*>(a.X) + local * a.ldx + G.sel_slot * K;
  if constexpr (BYTES % 32 == 0) {
#pragma unroll
    for (int v = 0; v < BYTES / 16; v += 2)
      stg256(reinterpret_cast<uint4*>(dst) + v, reinterpret_cast<const uint4*>(out)[v],
             reinterpret_cast<const uint4*>(out)[v + 1]);
  } else if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int v = 0; v < BYTES / 16; v++)
      reinterpret_cast<uint4*>(dst)[v] = reinterpret_cast<const uint4*>(out)[v];
  } else {
#pragma unroll
    for (int d = 0; d < K; d++) dst[d] = out[d];
  }
  if (a.dbg_feat) {
#pragma unroll
    for (int d = 0; d < K; d++) a.dbg_feat[ad * a.d_in + G.sel_pos * K + d] = Store<T>::to_f(out[d]);
  }
}

// request of a call-global ad: the map written by user_kernel, or (search_req: the few-request latency
// path, where the user kernel runs concurrently on the ctx's side stream) a binary search of ad_offsets
__device__ __forceinline__ int req_at(const GatherArgs& a, int64_t ad) {
  if (!a.search_req) return a.req_of_ad[ad];
  int lo = 0, hi = a.R;   // ad_offsets[lo] <= ad < ad_offsets[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(a.adoff + mid) <= ad) lo = mid;
    else hi = mid;
  }
  return lo;
}

// FC1 u1 operand rows: for span-local row i, slot = request(i) - base, base = the first request of its
// 256-row CTA-pair tile rounded down to a multiple of 8 (tiles are 256-aligned inside each FC chunk);
// 1.0 at k = slot and k = 8 + slot; all zero when the tile's requests do not fit in [base, base + 8)
// (the FC1 epilogue then adds u1 itself).
__device__ __forceinline__ void write_ohot(const GatherArgs& a, int64_t i, uint16_t one) {
  const int64_t j = i / a.chunk, q = i - j * a.chunk;
  const int64_t c_end = min((j + 1) * (int64_t)a.chunk, a.n);
  const int64_t t0 = j * a.chunk + (q & ~(int64_t)255);
  const int64_t t1 = min(t0 + 256, c_end) - 1;
  const int r0 = req_at(a, a.a0 + t0) & ~7;   // 8-aligned: the u1-term TMA box starts 16 B aligned
  const int slot = req_at(a, a.a0 + i) - r0;
  const bool ok = req_at(a, a.a0 + t1) - r0 < a.nslot;
  uint32_t w[8];
#pragma unroll
  for (int c = 0; c < 8; c++) {
    const int k0 = (2 * c) & 7, k1 = (2 * c + 1) & 7;
    w[c] = (ok && k0 == slot ? one : 0u) | ((ok && k1 == slot ? (uint32_t)one : 0u) << 16);
  }
  uint4* dst = reinterpret_cast<uint4*>(a.ohot + i * 16);
  dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
  dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// ---- cp.async (LDGSTS) helpers: 16 B global -> shared copies that complete asynchronously, tracked
// per thread in commit groups (no registers held while a row is in flight)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Cross group of a user bag x a single-valued ad id (S-paper: clk_cate x cate, clk_shop x shop,
// clk_brand x brand: 48 of the 61 rows of an ad). The thread's APT ads x L bag rows form one row
// stream: a producer cursor issues row j + RING (two 16 B cp.async into ring slot (j + RING) % RING of
// this thread) while the consumer adds row j from its slot, so RING rows stay in flight continuously
// instead of bursts of RB register-held rows with a full round trip between bursts. The ring is
// [RING][128 threads][32 B] (a warp reads 1 KB contiguous per slot: no bank conflicts). Rows are
// still summed one at a time in bag order (x-major), so the fp32 sums are unchanged (D-3).
template <typename T, int K, bool FAST, int APT, int RING>
__device__ __forceinline__ void cross_bag_ring(const GatherArgs& a, const DevGroup& G, int g, const T* __restrict__ tab,
                                               uint64_t card, const uint64_t (*s_hx)[HX_HALF], const int64_t* ul,
                                               int rfirst, const BatchGroup& BA, const DevGroup& A,
                                               const float* sew, float seb, int j, const int64_t* loc,
                                               const bool* ok) {
  static_assert(K * (int)sizeof(T) == 32, "ring rows are 32 B");
  extern __shared__ __align__(16) uint8_t ring_smem[];
  const uint32_t my = smem_addr(ring_smem) + threadIdx.x * 32u;
  constexpr uint32_t SLOT = 128u * 32u;
  uint64_t y[APT];
  int sl[APT], len[APT];
#pragma unroll
  for (int i = 0; i < APT; i++) {
    y[i] = (uint64_t)checked(BA.ids[a.a0 + loc[i] - BA.id_shift], A.card, a.validate, a.err);
    sl[i] = (req_at(a, a.a0 + loc[i]) == rfirst) ? 0 : 1;
    len[i] = (int)ul[sl[i]];
  }
  // producer cursor (ad pi, bag element px) and the ring slot it fills next
  int pi = 0, px = 0, ps = 0;
  while (pi < APT && len[pi] == 0) pi++;
  auto issue = [&]() {
    if (pi < APT) {
      uint64_t yy = y[0];
      int ss = sl[0], ll = len[0];
#pragma unroll
      for (int i = 1; i < APT; i++)
        if (pi == i) { yy = y[i]; ss = sl[i]; ll = len[i]; }
      const uint4* src = reinterpret_cast<const uint4*>(tab + cross_row_from_hx(s_hx[ss][px], yy, card) * K);
      const uint32_t dst = my + (uint32_t)ps * SLOT;
      cp_async16(dst, src);
      cp_async16(dst + 16u, src + 1);
      if (++px == ll) {
        px = 0;
        do pi++; while (pi < APT && len[pi] == 0);
      }
    }
    cp_async_commit();   // (an empty group once the stream is exhausted keeps the wait count uniform)
    ps = ps + 1 == RING ? 0 : ps + 1;
  };
#pragma unroll
  for (int r = 0; r < RING; r++) issue();
  int cs = 0;
#pragma unroll
  for (int i = 0; i < APT; i++) {
    float e[K];
#pragma unroll
    for (int d = 0; d < K; d++) e[d] = 0.0f;
#pragma unroll 1
    for (int x = 0; x < len[i]; x++) {
      cp_async_wait<RING - 1>();   // the oldest group (this row) has landed
      const uint32_t src = my + (uint32_t)cs * SLOT;
      uint4 q0, q1;
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w) : "r"(src));
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w)
                   : "r"(src + 16u));
      cs = cs + 1 == RING ? 0 : cs + 1;
      issue();                     // refill: the slot just read is reused RING rows later
      const T* t0 = reinterpret_cast<const T*>(&q0);
      const T* t1 = reinterpret_cast<const T*>(&q1);
#pragma unroll
      for (int d = 0; d < 8; d++) e[d] = Store<T>::add(e[d], t0[d]);
#pragma unroll
      for (int d = 0; d < 8; d++) e[8 + d] = Store<T>::add(e[8 + d], t1[d]);
    }
    if (ok[i]) finish_ad<T, K, FAST>(a, G, g, loc[i], e, sew, seb, j);
  }
  cp_async_wait<0>();
}

// APT: ads per thread (4 for large spans; 1 for small batches, where per-thread serial work is the latency)
// RING == 0: every column kind (one launch per span). RING != 0: a build launched over the cross-bag
// columns only (no AD-group / single-row code in it, so the register allocation serves the bag loop):
// RING == -1 holds GATHER_RB rows per burst in registers, RING > 0 streams them through a RING-deep
// cp.async ring (dynamic smem RING * 4 KB)
template <typename T, int K, bool FAST, int MINB = 4, int GATHER_APT = 4, int RING = 0>
__global__ void __launch_bounds__(128, MINB) gather_kernel(GatherArgs a) {
  if ((int)blockIdx.y == a.n_ac) {          // FC1's one-hot u1 operand rows
    for (int i = 0; i < GATHER_APT; i++) {
      const int64_t l = (int64_t)blockIdx.x * (128 * GATHER_APT) + threadIdx.x + i * 128;
      if (l < a.n) write_ohot(a, l, a.bf16 ? 0x3F80u : 0x3C00u);
    }
    return;
  }
  constexpr bool VEC = (K * (int)sizeof(T)) % 16 == 0;
  constexpr int NV = K * (int)sizeof(T) / 16;
  // bag rows in flight per thread (<= 16 vectors of raw registers; halved when the register budget
  // is halved for twice the resident warps)
  // (MINB <= 2, the single-request latency build: a whole 16-row bag in flight per thread)
  constexpr int GATHER_RB = MINB <= 2 && NV <= 2 ? 16
                          : (NV <= 2 ? 8 : (NV == 4 ? 4 : 2)) / (MINB >= 12 ? 4 : (MINB >= 8 ? 2 : 1));
  __shared__ uint64_t s_hx[2][HX_HALF];
#ifdef COLD_GATHER_PAD_SMEM   // A/B: the static shared footprint of the round-1 build (5376 B)
  __shared__ uint8_t s_pad[1280];
  if (a.n < 0) s_pad[threadIdx.x] = 1;
#endif
  const int j = a.order[blockIdx.y];
  const int g = a.ac_g[j];
  const float* sew = a.se_w + g * K;
  const float seb = a.sew_in_params ? 0.0f : __ldg(a.se_b + g);
  const DevGroup G = GGROUP(a, g);
  const T* tab = reinterpret_cast<const T*>(G.table);
  const int64_t base = (int64_t)blockIdx.x * (128 * GATHER_APT);
  int64_t loc[GATHER_APT];
  bool ok[GATHER_APT];
#pragma unroll
  for (int i = 0; i < GATHER_APT; i++) {
    const int64_t l = base + threadIdx.x + i * 128;
    ok[i] = l < a.n;
    loc[i] = ok[i] ? l : a.n - 1;           // clamped: loads stay in range, results are dropped
  }

  // (the RING build is launched over cross-bag columns only: no AD-group code in it)
  if (RING == 0 && G.side == 1) {           // ---------------- AD group ----------------
    const BatchGroup& B = a.bv.g[g];
    if (!G.pooled && VEC) {
      int64_t row[GATHER_APT];
#pragma unroll
      for (int i = 0; i < GATHER_APT; i++) row[i] = checked(B.ids[a.a0 + loc[i] - B.id_shift], G.card, a.validate, a.err);
      RawRow<T, K> raw[GATHER_APT];
#pragma unroll
      for (int i = 0; i < GATHER_APT; i++) raw[i].load(tab, row[i]);
#pragma unroll
      for (int i = 0; i < GATHER_APT; i++) {
        float e[K];
#pragma unroll
        for (int d = 0; d < K; d++) e[d] = 0.0f;
        raw[i].add_to(e);
        if (ok[i]) finish_ad<T, K, FAST>(a, G, g, loc[i], e, sew, seb, j);
      }
    } else {
      for (int i = 0; i < GATHER_APT; i++) {
        const int64_t li = base + threadIdx.x + i * 128;   // (no register-array indexing in rolled loops)
        if (li >= a.n) break;
        const int64_t ad = a.a0 + li;
        float e[K];
#pragma unroll
        for (int d = 0; d < K; d++) e[d] = 0.0f;
        if (!G.pooled) {
          add_row<T, K>(tab, checked(B.ids[ad - B.id_shift], G.card, a.validate, a.err), e);
        } else {
          const int64_t o0 = (int64_t)B.offs[ad - B.offs_shift] - B.val_shift;
          const int64_t o1 = (int64_t)B.offs[ad + 1 - B.offs_shift] - B.val_shift;
          for (int64_t q = o0; q < o1; q++) add_row<T, K>(tab, checked(B.ids[q], G.card, a.validate, a.err), e);
        }
        finish_ad<T, K, FAST>(a, G, g, li, e, sew, seb, j);
      }
    }
    return;
  }

  // ---------------- CROSS group: rows = hash(user bag x ad bag), x-major ----------------
  const DevGroup U = GGROUP(a, G.user_ref);
  const DevGroup A = GGROUP(a, G.ad_ref);
  const BatchGroup& BU = a.bv.g[G.user_ref];
  const BatchGroup& BA = a.bv.g[G.ad_ref];
  const uint64_t salt = cross_salt(g);
  const uint64_t card = (uint64_t)G.card;
  // requests of the block's first and last ad; <= 2 requests -> user-bag hashes in shared memory
  const int64_t last = (base + 128 * GATHER_APT < a.n ? base + 128 * GATHER_APT : a.n) - 1;
  const int rfirst = req_at(a, a.a0 + base);
  const int rlast = req_at(a, a.a0 + last);
  int64_t ub[2], ul[2];
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int r = q == 0 ? rfirst : rlast;
    ub[q] = (int64_t)BU.offs[r - BU.offs_shift] - BU.val_shift;
    ul[q] = (int64_t)BU.offs[r + 1 - BU.offs_shift] - BU.val_shift - ub[q];
  }
  const bool shared_hx = (rlast - rfirst <= 1) && ul[0] <= HX_HALF && ul[1] <= HX_HALF;
  if (shared_hx) {
    for (int q = 0; q < 2; q++)
      for (int64_t i = threadIdx.x; i < ul[q]; i += blockDim.x)
        s_hx[q][i] = fmix64((uint64_t)checked(BU.ids[ub[q] + i], U.card, a.validate, a.err) ^ salt);
    __syncthreads();
  }
  if (RING == 0 && shared_hx && !A.pooled && VEC && ul[0] == 1 && ul[1] == 1) {
    // single-id user group x single-id ad group: one row per ad, all APT rows in flight
    int64_t row[GATHER_APT];
#pragma unroll
    for (int i = 0; i < GATHER_APT; i++) {
      const uint64_t y = (uint64_t)checked(BA.ids[a.a0 + loc[i] - BA.id_shift], A.card, a.validate, a.err);
      const int sl = (req_at(a, a.a0 + loc[i]) == rfirst) ? 0 : 1;
      row[i] = cross_row_from_hx(s_hx[sl][0], y, card);
    }
    RawRow<T, K> raw[GATHER_APT];
#pragma unroll
    for (int i = 0; i < GATHER_APT; i++) raw[i].load(tab, row[i]);
#pragma unroll
    for (int i = 0; i < GATHER_APT; i++) {
      float e[K];
#pragma unroll
      for (int d = 0; d < K; d++) e[d] = 0.0f;
      raw[i].add_to(e);
      if (ok[i]) finish_ad<T, K, FAST>(a, G, g, loc[i], e, sew, seb, j);
    }
    return;
  }

  if constexpr (RING > 0 && K * (int)sizeof(T) == 32) {
    if (shared_hx && !A.pooled) {
      cross_bag_ring<T, K, FAST, GATHER_APT, RING>(a, G, g, tab, card, s_hx, ul, rfirst, BA, A, sew, seb, j, loc, ok);
      return;
    }
  }
  for (int i = 0; i < GATHER_APT; i++) {
    const int64_t li = base + threadIdx.x + i * 128;
    if (li >= a.n) break;
    const int64_t ad = a.a0 + li;
    const int sl = (req_at(a, ad) == rfirst) ? 0 : 1;
    int64_t u0, L;
    if (shared_hx) {
      u0 = sl ? ub[1] : ub[0];
      L = sl ? ul[1] : ul[0];
    } else {
      const int r = req_at(a, ad);
      u0 = (int64_t)BU.offs[r - BU.offs_shift] - BU.val_shift;
      L = (int64_t)BU.offs[r + 1 - BU.offs_shift] - BU.val_shift - u0;
    }
    auto hx_at = [&](int64_t x) -> uint64_t {
      return shared_hx ? s_hx[sl][x]
                       : fmix64((uint64_t)checked(BU.ids[u0 + x], U.card, a.validate, a.err) ^ salt);
    };
    float e[K];
#pragma unroll
    for (int d = 0; d < K; d++) e[d] = 0.0f;
    if (!A.pooled) {
      const uint64_t y = (uint64_t)checked(BA.ids[ad - BA.id_shift], A.card, a.validate, a.err);
      int64_t x = 0;
      if constexpr (VEC) {
        for (; x + GATHER_RB <= L; x += GATHER_RB) {     // RB rows in flight, then summed in bag order
          RawRow<T, K> raw[GATHER_RB];
#pragma unroll
          for (int t = 0; t < GATHER_RB; t++) raw[t].load(tab, cross_row_from_hx(hx_at(x + t), y, card));
#pragma unroll
          for (int t = 0; t < GATHER_RB; t++) raw[t].add_to(e);
        }
      }
      for (; x < L; x++) add_row<T, K>(tab, cross_row_from_hx(hx_at(x), y, card), e);
    } else {
      const int64_t y0 = (int64_t)BA.offs[ad - BA.offs_shift] - BA.val_shift;
      const int64_t y1 = (int64_t)BA.offs[ad + 1 - BA.offs_shift] - BA.val_shift;
      for (int64_t x = 0; x < L; x++) {
        const uint64_t hx = hx_at(x);
        for (int64_t q = y0; q < y1; q++) {
          const uint64_t y = (uint64_t)checked(BA.ids[q], A.card, a.validate, a.err);
          add_row<T, K>(tab, cross_row_from_hx(hx, y, card), e);
        }
      }
    }
    finish_ad<T, K, FAST>(a, G, g, li, e, sew, seb, j);
  }
}

// debug: rows of one group per ad
__global__ void rows_kernel(RowsArgs a) {
  const int64_t ad = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ad >= a.n) return;
  const DevGroup G = a.groups[a.g];
  int64_t* out = a.rows + ad * a.max_rows;
  int cnt = 0;
  auto put = [&](int64_t v) { if (cnt < a.max_rows) out[cnt] = v; cnt++; };
  const int r = a.req_of_ad[ad];
  if (G.side == 0) {
    const BatchGroup& B = a.bv.g[a.g];
    for (int64_t i = B.offs[r - B.offs_shift] - B.val_shift; i < B.offs[r + 1 - B.offs_shift] - B.val_shift; i++)
      put(B.ids[i]);
  } else if (G.side == 1) {
    const BatchGroup& B = a.bv.g[a.g];
    if (!G.pooled) put(B.ids[ad - B.id_shift]);
    else
      for (int64_t i = B.offs[ad - B.offs_shift] - B.val_shift; i < B.offs[ad + 1 - B.offs_shift] - B.val_shift; i++)
        put(B.ids[i]);
  } else {
    const DevGroup A = a.groups[G.ad_ref];
    const BatchGroup& BU = a.bv.g[G.user_ref];
    const BatchGroup& BA = a.bv.g[G.ad_ref];
    int64_t y0, y1;
    if (!A.pooled) { y0 = ad - BA.id_shift; y1 = y0 + 1; }
    else { y0 = BA.offs[ad - BA.offs_shift] - BA.val_shift; y1 = BA.offs[ad + 1 - BA.offs_shift] - BA.val_shift; }
    const uint64_t salt = cross_salt(a.g);
    for (int64_t i = BU.offs[r - BU.offs_shift] - BU.val_shift; i < BU.offs[r + 1 - BU.offs_shift] - BU.val_shift; i++) {
      const uint64_t hx = fmix64((uint64_t)BU.ids[i] ^ salt);
      for (int64_t q = y0; q < y1; q++) put(cross_row_from_hx(hx, (uint64_t)BA.ids[q], (uint64_t)G.card));
    }
  }
  for (int i = cnt; i < a.max_rows; i++) out[i] = -1;
}

// ---------------------------------------------------------------------------------------------
template <typename T>
static void user_dispatch(const UserArgs& a, int R, cudaStream_t s) {
  UserArgs b = a;
  b.part_off = (int)((((size_t)a.n_user * a.k + 3) & ~(size_t)3) + (size_t)8 * 32 * a.k);   // after x_u and the row stage
  const size_t smem = ((size_t)b.part_off + (size_t)4 * a.H) * sizeof(float);
  // few requests (the latency path): the u1 GEMV's 64-output passes over up to 16 CTAs per request
  const int slices = R >= 64 ? 1 : std::min(16, std::max(1, (a.H + 63) / 64));
  const dim3 grid((unsigned)R, (unsigned)slices);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, s>>>(b);
  };
  switch (a.k) {
    case 2: go(user_kernel<T, 2>); break;
    case 4: go(user_kernel<T, 4>); break;
    case 8: go(user_kernel<T, 8>); break;
    case 16: go(user_kernel<T, 16>); break;
    case 32: go(user_kernel<T, 32>); break;
  }
}

void launch_user(const UserArgs& a, int R, int precision, cudaStream_t s) {
  if (precision == 0) user_dispatch<float>(a, R, s);
  else if (precision == 1) user_dispatch<__half>(a, R, s);
  else user_dispatch<__nv_bfloat16>(a, R, s);
}

template <typename T, bool FAST>
static void gather_dispatch(const GatherArgs& a, cudaStream_t s) {
  const unsigned gy = (unsigned)(a.n_ac + (a.ohot ? 1 : 0));
  auto grid_for = [&](int apt) { return dim3((unsigned)((a.n + 128 * apt - 1) / (128 * apt)), gy); };
  const dim3 grid = grid_for(GATHER_APT_BIG);
  switch (a.k) {
    case 2: gather_kernel<T, 2, FAST><<<grid, 128, 0, s>>>(a); break;
    case 4: gather_kernel<T, 4, FAST><<<grid, 128, 0, s>>>(a); break;
    case 8: gather_kernel<T, 8, FAST><<<grid, 128, 0, s>>>(a); break;
    case 16: {
      // 8 CTAs of 128 threads per SM at <= 64 registers (12-16 CTAs spill; 6-7 CTAs with 8 rows in flight
      // per thread measured slower: DESIGN.md §9)
      if (a.ring == -1) gather_kernel<T, 16, FAST, 8, 4, -1><<<grid, 128, 0, s>>>(a);
      else if (sizeof(T) == 2 && a.ring == 4) gather_kernel<T, 16, FAST, 8, 4, 4><<<grid, 128, 4 * 4096, s>>>(a);
      else if (sizeof(T) == 2 && a.ring == 5) gather_kernel<T, 16, FAST, 8, 4, 5><<<grid, 128, 5 * 4096, s>>>(a);
      else if (sizeof(T) == 2 && a.ring == 8) gather_kernel<T, 16, FAST, 6, 4, 8><<<grid, 128, 8 * 4096, s>>>(a);
      else if (a.n < 148 * 128 * 4) {   // latency path: one ad per thread
        // 8 bag rows in flight per thread at 4 CTAs per SM: p50 63.0 us at 4000 ads, vs 4 rows at 8 CTAs/SM
        // 67.9 and a whole 16-row bag at 2 CTAs/SM 64.8 (profiles/r03/lat_ab_r03g_*.jsonl)
#if defined(COLD_GATHER_LAT_RB4)   // A/B: 4 bag rows in flight per thread (round-2 latency build)
        gather_kernel<T, 16, FAST, 8, 1><<<grid_for(1), 128, 0, s>>>(a);
#elif defined(COLD_GATHER_LAT_RB16)   // A/B: 16 rows in flight, 2 CTAs per SM
        gather_kernel<T, 16, FAST, 2, 1><<<grid_for(1), 128, 0, s>>>(a);
#else
        gather_kernel<T, 16, FAST, 4, 1><<<grid_for(1), 128, 0, s>>>(a);
#endif
      }
      else gather_kernel<T, 16, FAST, 8><<<grid, 128, 0, s>>>(a);   // (8 ads per thread at 6 CTAs/SM: 14% slower)
      break;
    }
    case 32: gather_kernel<T, 32, FAST><<<grid, 128, 0, s>>>(a); break;
  }
}

void launch_gather(const GatherArgs& a, int precision, cudaStream_t s) {
  if (a.n <= 0 || (a.n_ac <= 0 && !a.ohot)) return;
  if (precision == 0) gather_dispatch<float, false>(a, s);
  else if (precision == 1) gather_dispatch<__half, true>(a, s);
  else gather_dispatch<__nv_bfloat16, true>(a, s);
}

void launch_rows(const RowsArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  rows_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a);
}

}  // namespace cold
