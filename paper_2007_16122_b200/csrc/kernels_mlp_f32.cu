// kernels_mlp_f32.cu — the fp32 FC stack on CUDA cores (FFMA, no TF32): the 1e-5-relative
// parity mode (BASELINE configs[0]) and the "Float32" row of PAPER.md Table tab:qps_cuda (L444).
//
// One CTA owns TILE ads; activations live in shared memory, weights are read transposed
// ([in][out], coalesced over the output index). Layer 0 starts from the per-request user
// block u1[req] = b1 + W1_u x_u computed once per request by user_kernel.
#include "internal.h"

namespace cold {

constexpr int MLP_TILE = 16;
constexpr int MLP_THREADS = 256;

// Register tiling: each thread owns 4 outputs (stride 64, so the 64 threads of a row group read
// 4 x 64 consecutive weights) x 16 ads; per 4 inputs it loads 16 weights and 16 float4 activations
// for 256 FFMAs (the naive one-output-per-thread loop was load-bound at 1 FFMA per load).
// Accumulation order per (ad, output) is the input index order, as before.
__global__ void __launch_bounds__(MLP_THREADS) mlp_f32_kernel(MlpF32Args a) {
  extern __shared__ float sm[];
  float* buf0 = sm;                                  // [TILE][max_w]
  float* buf1 = sm + MLP_TILE * a.max_w;             // [TILE][max_w]
  __shared__ int reqs[MLP_TILE];
  const int64_t t0 = (int64_t)blockIdx.x * MLP_TILE;
  const int nt = (int)(a.n - t0 < MLP_TILE ? a.n - t0 : MLP_TILE);
  for (int i = threadIdx.x; i < MLP_TILE * a.max_w; i += blockDim.x) {
    const int t = i / a.max_w, c = i % a.max_w;
    buf0[i] = (t < nt && c < a.d_ac) ? a.X[(t0 + t) * a.ldx + c] : 0.0f;   // zero pad up to max_w
  }
  if (threadIdx.x < MLP_TILE) reqs[threadIdx.x] = (threadIdx.x < nt) ? a.req_of_ad[a.a0 + t0 + threadIdx.x] : 0;
  __syncthreads();
  float* h = buf0;
  float* o = buf1;
  int in = a.d_ac;
  for (int l = 0; l < a.L; l++) {
    const int out = a.width[l];
    const float* wt = a.wt[l];
    const bool last = (l == a.L - 1);
    for (int jb = 0; jb < out; jb += 4 * MLP_THREADS) {      // 1024 outputs per pass
      const int tx = threadIdx.x;
      int js[4];
      bool jv[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        // thread tx of warp-group g: outputs jb + 256 q + tx  (consecutive across threads: coalesced)
        js[q] = jb + q * MLP_THREADS + tx;
        jv[q] = js[q] < out;
      }
      if (!(jv[0] || jv[1] || jv[2] || jv[3])) continue;
      float acc[4][MLP_TILE];
#pragma unroll
      for (int q = 0; q < 4; q++) {
#pragma unroll
        for (int t = 0; t < MLP_TILE; t++)
          acc[q][t] = jv[q] ? ((l == 0) ? a.u1[(int64_t)reqs[t] * a.ld_u1 + js[q]] : a.b[l][js[q]]) : 0.0f;
      }
      int i = 0;
      for (; i + 4 <= in; i += 4) {
        float w[4][4];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int q = 0; q < 4; q++) w[u][q] = jv[q] ? __ldg(wt + (int64_t)(i + u) * out + js[q]) : 0.0f;
#pragma unroll
        for (int t = 0; t < MLP_TILE; t++) {
          const float4 hv = *reinterpret_cast<const float4*>(h + t * a.max_w + i);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            acc[q][t] = fmaf(w[0][q], hv.x, acc[q][t]);
            acc[q][t] = fmaf(w[1][q], hv.y, acc[q][t]);
            acc[q][t] = fmaf(w[2][q], hv.z, acc[q][t]);
            acc[q][t] = fmaf(w[3][q], hv.w, acc[q][t]);
          }
        }
      }
      for (; i < in; i++) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const float w = jv[q] ? __ldg(wt + (int64_t)i * out + js[q]) : 0.0f;
#pragma unroll
          for (int t = 0; t < MLP_TILE; t++) acc[q][t] = fmaf(w, h[t * a.max_w + i], acc[q][t]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (!jv[q]) continue;
#pragma unroll
        for (int t = 0; t < MLP_TILE; t++)
          o[t * a.max_w + js[q]] = last ? acc[q][t]
                                        : (a.slope[l] ? prelu(acc[q][t], __ldg(a.slope[l] + js[q])) : fmaxf(acc[q][t], 0.0f));
      }
    }
    __syncthreads();
    float* tmp = h; h = o; o = tmp;
    in = out;
  }
  if (threadIdx.x < nt) {
    const int t = threadIdx.x;
    const float z = (in == 2) ? h[t * a.max_w + 1] - h[t * a.max_w + 0] : h[t * a.max_w + 0];
    a.scores[t0 + t] = sigmoid(z);
  }
}

void launch_mlp_f32(const MlpF32Args& a, cudaStream_t s) {
  if (a.n <= 0) return;
  size_t smem = 2 * (size_t)MLP_TILE * a.max_w * sizeof(float);
  static DevOnce attr_set;
  if (attr_set.first()) {
    cudaFuncSetAttribute(mlp_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  mlp_f32_kernel<<<(unsigned)((a.n + MLP_TILE - 1) / MLP_TILE), MLP_THREADS, smem, s>>>(a);
}

}  // namespace cold
