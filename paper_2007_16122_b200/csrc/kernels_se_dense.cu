// kernels_se_dense.cu — the dense SE gate (COLD_SE_DENSE, DESIGN.md AMB-1).
//
// PAPER.md L229-234 (§3.2, Doc B) writes the SE block as s = σ(W [e_1, .., e_M] + b) with s ∈ R^M:
// every group's gate reads the whole concat of pooled (linear_log'ed) embeddings. Under this
// reading s_g depends on the ad, so the user block cannot be hoisted into u1: FC1 runs over all D_in
// columns and this kernel writes the user columns of X per ad too.
//
// se_dense_kernel: one CTA per ADS ads. (1) ê of its ads -> shared memory, transposed (ad fastest):
// ad + cross columns from E (written by gather_kernel in this mode), user columns from xu[request]
// (user_kernel). (2) z[ad][j] = bd[j] + Σ_c Wd[j][c] ê[ad][c] in fp32 FFMA (AMB-14: the gate is fp32),
// a thread owns one output j for 4 ads (one 128-bit smem read of ê feeds 4 FMAs). (3) x = s_g ê_g,
// input normalisation (fp32), RNE cast -> X[ad][c] (schema order of the selected groups).
#include <algorithm>

#include "internal.h"

namespace cold {

size_t se_dense_smem(int d_in, int n_sel);

// One thread per ad: z[j] for a block of JB outputs is accumulated in registers while the ad's ê row
// streams from global memory (16 B loads; E rows are written by gather_kernel, user columns come from
// xu[request]) and Wd^T is read from shared memory as warp-wide broadcasts (LDS.128): ~1.3 issued
// instructions per multiply-add, with all 128 threads of a CTA busy.
template <int K>
__device__ __forceinline__ const float* col_src(const SeDenseArgs& a, const int* upos, int req, int64_t row, int p) {
  const int u = upos[p];
  return u >= 0 ? a.xu + (int64_t)req * a.ldu + u * K : a.E + row * a.lde + p * K;
}

template <typename T, int K, int JB, bool V4>
__global__ void __launch_bounds__(128) se_dense_kernel(SeDenseArgs a) {
  extern __shared__ float sm[];
  const int ldw = (a.n_sel + JB - 1) / JB * JB;     // row stride of Wd^T in smem (zero pad)
  float* ws = sm;                                   // [d_in][ldw]    Wd^T
  float* sg = ws + (size_t)a.d_in * ldw;            // [n_sel][128]   gates of the CTA's ads
  __shared__ int upos[COLD_MAX_GROUPS];             // selected position -> user group j, or -1
  __shared__ int reqs[128];                         // request of each of the CTA's ads
  const int t = threadIdx.x;
  for (int p = t; p < a.n_sel; p += blockDim.x) upos[p] = -1;
  for (int q = t; q < a.d_in * ldw; q += blockDim.x) {
    const int c = q / ldw, j = q % ldw;
    ws[q] = j < a.n_sel ? a.wdt[(size_t)c * a.n_sel + j] : 0.0f;
  }
  __syncthreads();
  for (int j = t; j < a.n_user; j += blockDim.x) upos[a.user_pos[j]] = j;
  __syncthreads();
  const int64_t li = (int64_t)blockIdx.x * blockDim.x + t;
  const bool live = li < a.n;
  const int64_t row = live ? li : a.n - 1;          // clamped: loads stay in range, results dropped
  const int req = a.req_of_ad[a.a0 + row];
  reqs[t] = req;
  // (2) gate, JB outputs per pass
  for (int j0 = 0; j0 < a.n_sel; j0 += JB) {
    float z[JB];
#pragma unroll
    for (int j = 0; j < JB; j++) z[j] = 0.0f;
    if constexpr (V4) {   // 16 columns per step, the next step's 4 x 16 B loads issued before the FMAs
      auto load16 = [&](int c0, float4* e) {
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int c = c0 + 4 * v;
          e[v] = *reinterpret_cast<const float4*>(col_src<K>(a, upos, req, row, c / K) + c % K);
        }
      };
      float4 cur[4], nxt[4];
      load16(0, cur);
      for (int c0 = 0; c0 < a.d_in; c0 += 16) {
        if (c0 + 16 < a.d_in) load16(c0 + 16, nxt);
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const float ev[4] = {cur[v].x, cur[v].y, cur[v].z, cur[v].w};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float* w = ws + (size_t)(c0 + 4 * v + q) * ldw + j0;
#pragma unroll
            for (int j = 0; j < JB; j += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(w + j);
              z[j] = fmaf(w4.x, ev[q], z[j]);
              z[j + 1] = fmaf(w4.y, ev[q], z[j + 1]);
              z[j + 2] = fmaf(w4.z, ev[q], z[j + 2]);
              z[j + 3] = fmaf(w4.w, ev[q], z[j + 3]);
            }
          }
        }
#pragma unroll
        for (int v = 0; v < 4; v++) cur[v] = nxt[v];
      }
    } else {
      for (int p = 0; p < a.n_sel; p++) {
        const float* src = col_src<K>(a, upos, req, row, p);
        for (int d = 0; d < K; d++) {
          const float ev = src[d];
          const float* w = ws + (size_t)(p * K + d) * ldw + j0;
#pragma unroll
          for (int j = 0; j < JB; j++) z[j] = fmaf(w[j], ev, z[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < JB; j++)
      if (j0 + j < a.n_sel) sg[(size_t)(j0 + j) * blockDim.x + t] = sigmoid(z[j] + __ldg(a.bd + j0 + j));
  }
  __syncthreads();
  // (3) x = s_g ê_g (+ input normalisation, fp32) -> RNE cast -> X[row][c] (schema order). The CTA's rows
  // are contiguous in E and X: walk them as one flat block, 4 columns per item (coalesced).
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x;
  const int rows = (int)min((int64_t)blockDim.x, a.n - r0);
  const int n4 = (a.d_in + 3) / 4;
  const int q128 = blockDim.x / n4, r128 = blockDim.x % n4;
  int rl = t / n4, c4 = t % n4;   // (row, column quad) of item f, advanced by blockDim.x per step
  for (int f = t; f < rows * n4; f += blockDim.x, rl += q128, c4 += r128) {
    if (c4 >= n4) { c4 -= n4; rl++; }
    const int c0 = c4 * 4;
    const int64_t r = r0 + rl;
    T* xrow = reinterpret_cast<T*>(a.X) + r * a.ldx;
    alignas(8) T out[4];
    float ev[4];
    if (V4) {
      const float4 e = *reinterpret_cast<const float4*>(col_src<K>(a, upos, reqs[rl], r, c0 / K) + c0 % K);
      ev[0] = e.x; ev[1] = e.y; ev[2] = e.z; ev[3] = e.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int c = c0 + q;
        ev[q] = c < a.d_in ? col_src<K>(a, upos, reqs[rl], r, c / K)[c % K] : 0.0f;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int c = c0 + q;
      if (c >= a.d_in) break;
      float v = sg[(size_t)(c / K) * blockDim.x + rl] * ev[q];
      if (a.in_scale) v = fmaf(v, __ldg(a.in_scale + c), __ldg(a.in_shift + c));
      out[q] = Store<T>::from_f(v);
      if (a.dbg_feat) a.dbg_feat[(a.a0 + r) * a.d_in + c] = Store<T>::to_f(out[q]);
    }
    if (V4) {
      if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2*>(xrow + c0) = *reinterpret_cast<const uint2*>(out);
      else *reinterpret_cast<float4*>(xrow + c0) = *reinterpret_cast<const float4*>(out);
    } else {
      for (int q = 0; q < 4 && c0 + q < a.d_in; q++) xrow[c0 + q] = out[q];
    }
  }
}

template <typename T, int K, int JB, bool V4>
static void se_dense_launch(const SeDenseArgs& a, cudaStream_t s) {
  const size_t smem = se_dense_smem(a.d_in, a.n_sel);
  static std::atomic<size_t> attr[64];   // opt in per device (static + dynamic > 48 KB needs it)
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > attr[dev & 63].load()) {
    cudaFuncSetAttribute(se_dense_kernel<T, K, JB, V4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dev & 63].store(smem);
  }
  se_dense_kernel<T, K, JB, V4><<<(unsigned)((a.n + 127) / 128), 128, smem, s>>>(a);
}

static int se_dense_jb(int n_sel) { return n_sel % 24 == 0 ? 24 : (n_sel % 16 == 0 ? 16 : 8); }

size_t se_dense_smem(int d_in, int n_sel) {
  const int jb = se_dense_jb(n_sel);
  return ((size_t)d_in * ((n_sel + jb - 1) / jb * jb) + (size_t)n_sel * 128) * sizeof(float);
}

template <typename T, int K>
static void se_dense_dispatch_k(const SeDenseArgs& a, cudaStream_t s) {
  const bool v4 = K % 4 == 0 && a.d_in % 16 == 0;
  if constexpr (K % 4 == 0) {
    if (v4) {
      if (a.n_sel % 24 == 0) se_dense_launch<T, K, 24, true>(a, s);
      else if (a.n_sel % 16 == 0) se_dense_launch<T, K, 16, true>(a, s);
      else se_dense_launch<T, K, 8, true>(a, s);
      return;
    }
  }
  if (a.n_sel % 24 == 0) se_dense_launch<T, K, 24, false>(a, s);
  else if (a.n_sel % 16 == 0) se_dense_launch<T, K, 16, false>(a, s);
  else se_dense_launch<T, K, 8, false>(a, s);
}

template <typename T>
static void se_dense_dispatch(const SeDenseArgs& a, cudaStream_t s) {
  switch (a.k) {
    case 2: se_dense_dispatch_k<T, 2>(a, s); break;
    case 4: se_dense_dispatch_k<T, 4>(a, s); break;
    case 8: se_dense_dispatch_k<T, 8>(a, s); break;
    case 16: se_dense_dispatch_k<T, 16>(a, s); break;
    case 32: se_dense_dispatch_k<T, 32>(a, s); break;
  }
}

void launch_se_dense(const SeDenseArgs& a, int precision, cudaStream_t s) {
  if (a.n <= 0) return;
  if (precision == 0) se_dense_dispatch<float>(a, s);
  else if (precision == 1) se_dense_dispatch<__half>(a, s);
  else se_dense_dispatch<__nv_bfloat16>(a, s);
}

}  // namespace cold
