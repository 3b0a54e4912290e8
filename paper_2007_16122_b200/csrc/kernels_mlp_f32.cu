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

__global__ void __launch_bounds__(MLP_THREADS) mlp_f32_kernel(MlpF32Args a) {
  extern __shared__ float sm[];
  float* buf0 = sm;                                  // [TILE][max_w]
  float* buf1 = sm + MLP_TILE * a.max_w;             // [TILE][max_w]
  __shared__ int reqs[MLP_TILE];
  const int64_t t0 = (int64_t)blockIdx.x * MLP_TILE;
  const int nt = (int)(a.n - t0 < MLP_TILE ? a.n - t0 : MLP_TILE);
  for (int i = threadIdx.x; i < MLP_TILE * a.d_ac; i += blockDim.x) {
    int t = i / a.d_ac, c = i % a.d_ac;
    buf0[t * a.max_w + c] = (t < nt) ? a.X[(t0 + t) * a.ldx + c] : 0.0f;
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
    for (int j = threadIdx.x; j < out; j += blockDim.x) {
      float acc[MLP_TILE];
#pragma unroll
      for (int t = 0; t < MLP_TILE; t++) acc[t] = (l == 0) ? a.u1[(int64_t)reqs[t] * a.ld_u1 + j] : a.b[l][j];
      for (int i = 0; i < in; i++) {
        const float w = __ldg(wt + (int64_t)i * out + j);
#pragma unroll
        for (int t = 0; t < MLP_TILE; t++) acc[t] = fmaf(w, h[t * a.max_w + i], acc[t]);
      }
#pragma unroll
      for (int t = 0; t < MLP_TILE; t++) o[t * a.max_w + j] = last ? acc[t] : fmaxf(acc[t], 0.0f);
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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(mlp_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  mlp_f32_kernel<<<(unsigned)((a.n + MLP_TILE - 1) / MLP_TILE), MLP_THREADS, smem, s>>>(a);
}

}  // namespace cold
