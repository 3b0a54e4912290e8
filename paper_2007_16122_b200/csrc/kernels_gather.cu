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
#include "internal.h"

namespace cold {

template <typename T, int K>
__device__ __forceinline__ void add_row(const T* __restrict__ table, int64_t row, float* e) {
  constexpr int BYTES = K * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {          // 16 B vector loads (k=16 fp16: one 32 B sector)
    const uint4* p = reinterpret_cast<const uint4*>(table + row * K);
#pragma unroll
    for (int v = 0; v < BYTES / 16; v++) {
      uint4 q = __ldg(p + v);
      const T* t = reinterpret_cast<const T*>(&q);
#pragma unroll
      for (int i = 0; i < 16 / (int)sizeof(T); i++) e[v * (16 / sizeof(T)) + i] += Store<T>::to_f(t[i]);
    }
  } else {                                   // tiny rows (k = 2, 4)
#pragma unroll
    for (int d = 0; d < K; d++) e[d] += Store<T>::to_f(table[row * K + d]);
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
// user side: grid = R requests, block = 256 threads
template <typename T, int K>
__global__ void __launch_bounds__(256) user_kernel(UserArgs a) {
  extern __shared__ float xs[];           // [n_user * K]
  const int r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d_u = a.n_user * K;
  // one warp per selected user group; lane d < K owns dimension d
  for (int j = warp; j < a.n_user; j += blockDim.x / 32) {
    const int g = a.user_g[j];
    const DevGroup G = a.groups[g];
    const BatchGroup& B = a.bv.g[g];
    const int64_t o0 = (int64_t)B.offs[r - B.offs_shift] - B.val_shift;
    const int64_t o1 = (int64_t)B.offs[r + 1 - B.offs_shift] - B.val_shift;
    float e = 0.0f;
    const T* tab = reinterpret_cast<const T*>(G.table);
    for (int64_t i = o0; i < o1; i++) {
      int64_t row = checked(B.ids[i], G.card, a.validate, a.err);
      if (lane < K) e += Store<T>::to_f(tab[row * K + lane]);
    }
    float pooled = e;
    if (a.linear_log) e = linear_log(e);
    float z = (lane < K) ? a.se_w[g * K + lane] * e : 0.0f;
#pragma unroll
    for (int off = 16; off; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    const float s = sigmoid(z + a.se_b[g]);
    if (lane < K) {
      const float v = s * e;
      xs[j * K + lane] = v;
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
  __syncthreads();
  // u1[r][o] = b1[o] + sum_i W1u[o][i] x_u[i]   (W1u stored transposed: coalesced over o)
  for (int o = threadIdx.x; o < a.H; o += blockDim.x) {
    float acc = a.b1[o];
    for (int i = 0; i < d_u; i++) acc = fmaf(a.w1u_t[(int64_t)i * a.H + o], xs[i], acc);
    a.u1[(int64_t)r * a.H + o] = acc;
  }
  for (int64_t ad = a.ad_offsets[r] + threadIdx.x; ad < a.ad_offsets[r + 1]; ad += blockDim.x)
    a.req_of_ad[ad] = r;
}

// ---------------------------------------------------------------------------------------------
// ad + cross side: grid = (ceil(n / 128), n_ac), block = 128 threads, one thread per (ad, group).
// blockIdx.y walks the selected AD/CROSS groups heaviest-first (cross groups over user bags carry
// 16 rows per ad) so the long blocks start first. A cross group's user-side half of the hash,
// hx = fmix64(x ^ salt_g), depends only on the request: a block whose 128 ads belong to one request
// computes it once into shared memory (AMB-9: row = hi64(fmix64(hx ^ y) * C)).
constexpr int HX_SMEM = 512;

template <typename T, int K, bool FAST>
__global__ void __launch_bounds__(128) gather_kernel(GatherArgs a) {
  __shared__ uint64_t s_hx[HX_SMEM];
  const int64_t local = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in_range = local < a.n;
  const int64_t ad = a.a0 + (in_range ? local : a.n - 1);
  const int j = a.order[blockIdx.y];
  const int g = a.ac_g[j];
  const DevGroup G = a.groups[g];
  const T* tab = reinterpret_cast<const T*>(G.table);
  float e[K];
#pragma unroll
  for (int d = 0; d < K; d++) e[d] = 0.0f;

  if (G.side == 1) {                      // AD group
    if (!in_range) return;
    const BatchGroup& B = a.bv.g[g];
    if (!G.pooled) {
      add_row<T, K>(tab, checked(B.ids[ad - B.id_shift], G.card, a.validate, a.err), e);
    } else {
      const int64_t o0 = (int64_t)B.offs[ad - B.offs_shift] - B.val_shift;
      const int64_t o1 = (int64_t)B.offs[ad + 1 - B.offs_shift] - B.val_shift;
      for (int64_t i = o0; i < o1; i++) add_row<T, K>(tab, checked(B.ids[i], G.card, a.validate, a.err), e);
    }
  } else {                                // CROSS group: rows = hash(user bag x ad bag), x-major
    const DevGroup U = a.groups[G.user_ref];
    const DevGroup A = a.groups[G.ad_ref];
    const BatchGroup& BU = a.bv.g[G.user_ref];
    const BatchGroup& BA = a.bv.g[G.ad_ref];
    const uint64_t salt = cross_salt(g);
    const uint64_t card = (uint64_t)G.card;
    // block-uniform request? then hash the user bag once into shared memory
    const int64_t blk0 = a.a0 + (int64_t)blockIdx.x * blockDim.x;
    const int64_t blk_end = (int64_t)(blockIdx.x + 1) * blockDim.x;
    const int64_t blk1 = a.a0 + (blk_end < a.n ? blk_end : a.n) - 1;
    const int rb = a.req_of_ad[blk0];
    const int64_t ub0 = (int64_t)BU.offs[rb - BU.offs_shift] - BU.val_shift;
    const int64_t ub1 = (int64_t)BU.offs[rb + 1 - BU.offs_shift] - BU.val_shift;
    const bool shared_hx = (a.req_of_ad[blk1] == rb) && (ub1 - ub0 <= HX_SMEM);
    if (shared_hx) {
      for (int64_t i = threadIdx.x; i < ub1 - ub0; i += blockDim.x)
        s_hx[i] = fmix64((uint64_t)checked(BU.ids[ub0 + i], U.card, a.validate, a.err) ^ salt);
      __syncthreads();
    }
    if (!in_range) return;
    const int r = shared_hx ? rb : a.req_of_ad[ad];
    const int64_t u0 = (int64_t)BU.offs[r - BU.offs_shift] - BU.val_shift;
    const int64_t u1 = (int64_t)BU.offs[r + 1 - BU.offs_shift] - BU.val_shift;
    const int L = (int)(u1 - u0);
    auto hx_at = [&](int i) -> uint64_t {
      return shared_hx ? s_hx[i] : fmix64((uint64_t)checked(BU.ids[u0 + i], U.card, a.validate, a.err) ^ salt);
    };
    if (!A.pooled) {
      const uint64_t y = (uint64_t)checked(BA.ids[ad - BA.id_shift], A.card, a.validate, a.err);
      int i = 0;
      constexpr int U4 = 4;               // 4 rows in flight per thread, then summed in bag order
      for (; i + U4 <= L; i += U4) {
        int64_t rows[U4];
#pragma unroll
        for (int t = 0; t < U4; t++) rows[t] = cross_row_from_hx(hx_at(i + t), y, card);
        float v[U4][K];
#pragma unroll
        for (int t = 0; t < U4; t++) {
#pragma unroll
          for (int d = 0; d < K; d++) v[t][d] = 0.0f;
          add_row<T, K>(tab, rows[t], v[t]);
        }
#pragma unroll
        for (int t = 0; t < U4; t++) {
#pragma unroll
          for (int d = 0; d < K; d++) e[d] += v[t][d];
        }
      }
      for (; i < L; i++) add_row<T, K>(tab, cross_row_from_hx(hx_at(i), y, card), e);
    } else {
      const int64_t y0 = (int64_t)BA.offs[ad - BA.offs_shift] - BA.val_shift;
      const int64_t y1 = (int64_t)BA.offs[ad + 1 - BA.offs_shift] - BA.val_shift;
      for (int i = 0; i < L; i++) {
        const uint64_t hx = hx_at(i);
        for (int64_t q = y0; q < y1; q++) {
          const uint64_t y = (uint64_t)checked(BA.ids[q], A.card, a.validate, a.err);
          add_row<T, K>(tab, cross_row_from_hx(hx, y, card), e);
        }
      }
    }
  }

  if (a.dbg_pooled) {
#pragma unroll
    for (int d = 0; d < K; d++) a.dbg_pooled[(ad * a.n_sel + G.sel_pos) * K + d] = e[d];
  }
  // linear_log -> SE gate s = sigma(w . ê + b) -> v = s ê (fp32), then RNE to storage
  if (a.linear_log) {
#pragma unroll
    for (int d = 0; d < K; d++) e[d] = linear_log_t<FAST>(e[d]);
  }
  float z = 0.0f;
#pragma unroll
  for (int d = 0; d < K; d++) z = fmaf(__ldg(a.se_w + g * K + d), e[d], z);
  const float s = sigmoid_t<FAST>(z + __ldg(a.se_b + g));
  alignas(16) T out[K];
#pragma unroll
  for (int d = 0; d < K; d++) out[d] = Store<T>::from_f(s * e[d]);
  T* dst = reinterpret_cast<T*>(a.X) + local * a.ldx + G.sel_slot * K;
  constexpr int BYTES = K * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
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
  size_t smem = (size_t)a.n_user * a.k * sizeof(float) + 16;
  switch (a.k) {
    case 2: user_kernel<T, 2><<<R, 256, smem, s>>>(a); break;
    case 4: user_kernel<T, 4><<<R, 256, smem, s>>>(a); break;
    case 8: user_kernel<T, 8><<<R, 256, smem, s>>>(a); break;
    case 16: user_kernel<T, 16><<<R, 256, smem, s>>>(a); break;
    case 32: user_kernel<T, 32><<<R, 256, smem, s>>>(a); break;
  }
}

void launch_user(const UserArgs& a, int R, int precision, cudaStream_t s) {
  if (precision == 0) user_dispatch<float>(a, R, s);
  else if (precision == 1) user_dispatch<__half>(a, R, s);
  else user_dispatch<__nv_bfloat16>(a, R, s);
}

template <typename T, bool FAST>
static void gather_dispatch(const GatherArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.n + 127) / 128), (unsigned)a.n_ac);
  switch (a.k) {
    case 2: gather_kernel<T, 2, FAST><<<grid, 128, 0, s>>>(a); break;
    case 4: gather_kernel<T, 4, FAST><<<grid, 128, 0, s>>>(a); break;
    case 8: gather_kernel<T, 8, FAST><<<grid, 128, 0, s>>>(a); break;
    case 16: gather_kernel<T, 16, FAST><<<grid, 128, 0, s>>>(a); break;
    case 32: gather_kernel<T, 32, FAST><<<grid, 128, 0, s>>>(a); break;
  }
}

void launch_gather(const GatherArgs& a, int precision, cudaStream_t s) {
  if (a.n <= 0 || a.n_ac <= 0) return;
  if (precision == 0) gather_dispatch<float, false>(a, s);
  else if (precision == 1) gather_dispatch<__half, true>(a, s);
  else gather_dispatch<__nv_bfloat16, true>(a, s);
}

void launch_rows(const RowsArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  rows_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a);
}

}  // namespace cold
