// kernels_vps.cu — the vector-product based pre-ranking model COLD is compared with (PAPER.md L160-166
// §2.2, Eq. p = sigma(v_u^T v_a); Table tab:sys L377-391), served the way the paper describes it:
// the ad tower's output v_a is precomputed per ad, the user tower's v_u once per request, and the
// online step is a gather of v_a for every candidate, a dot product with v_u and a sigmoid
// (SURVEY §8(f) F4). HBM-bound: d * elem bytes of v_a + 4 B id + 4 B score per ad.
//
// grid = (x tiles, R requests): a block stages v_u[r] (fp32) in shared memory and walks its request's
// candidates; each thread loads one ad's whole vector with 256-bit loads (d = 64 fp16: 4 x LDG.256),
// accumulates in fp32 in index order, and writes sigma(z) (accurate expf).
#include <algorithm>
#include <cstdint>

#include "internal.h"

namespace cold {

__device__ __forceinline__ void ldg256v(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

template <typename T, int D>
__global__ void __launch_bounds__(256) vps_kernel(VpsArgs a) {
  constexpr int BYTES = D * (int)sizeof(T);
  constexpr int NV = BYTES / 16;                 // 16 B vectors per row
  constexpr int APT = BYTES <= 128 ? 2 : 1;      // ads per thread in flight (row registers <= 64)
  __shared__ float su[D];
  const int r = blockIdx.y;
  for (int i = threadIdx.x; i < D; i += blockDim.x) su[i] = a.user_vecs[(int64_t)r * D + i];
  const int64_t a0 = a.ad_offsets[r], a1 = a.ad_offsets[r + 1];
  const T* tab = reinterpret_cast<const T*>(a.ad_vecs);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * APT;
  for (int64_t base = a0 + (int64_t)blockIdx.x * blockDim.x * APT + threadIdx.x; base < a1; base += stride) {
    int64_t id[APT];
#pragma unroll
    for (int j = 0; j < APT; j++) {
      const int64_t ad = base + (int64_t)j * blockDim.x;
      int64_t v = ad < a1 ? a.ad_ids[ad] : 0;
      if (v < 0 || v >= a.num_vecs) v = v < 0 ? 0 : a.num_vecs - 1;   // clamp (memory-safe)
      id[j] = v;
    }
    uint4 q[APT][NV];
#pragma unroll
    for (int j = 0; j < APT; j++) {
      const uint4* row = reinterpret_cast<const uint4*>(tab + id[j] * D);
#pragma unroll
      for (int v = 0; v < NV; v += 2) ldg256v(row + v, q[j][v], q[j][v + 1]);
    }
#pragma unroll
    for (int j = 0; j < APT; j++) {
      const int64_t ad = base + (int64_t)j * blockDim.x;
      float z = 0.0f;
#pragma unroll
      for (int v = 0; v < NV; v++) {
        const T* t = reinterpret_cast<const T*>(&q[j][v]);
#pragma unroll
        for (int i = 0; i < 16 / (int)sizeof(T); i++) z = fmaf(su[v * (16 / sizeof(T)) + i], Store<T>::to_f(t[i]), z);
      }
      if (ad < a1) a.scores[ad] = sigmoid(z);
    }
  }
}

template <typename T>
static cudaError_t vps_dispatch(const VpsArgs& a, int max_n, cudaStream_t s) {
  // a block covers up to 8 * 256 * APT candidates of one request (loop), keeping the grid small
  dim3 grid((unsigned)std::min(64, std::max(1, (max_n + 4095) / 4096)), (unsigned)a.R);
  switch (a.d) {
    case 16: vps_kernel<T, 16><<<grid, 256, 0, s>>>(a); break;
    case 32: vps_kernel<T, 32><<<grid, 256, 0, s>>>(a); break;
    case 64: vps_kernel<T, 64><<<grid, 256, 0, s>>>(a); break;
    case 128: vps_kernel<T, 128><<<grid, 256, 0, s>>>(a); break;
    case 256: vps_kernel<T, 256><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_vps(const VpsArgs& a, int precision, int max_n, cudaStream_t s) {
  if (precision == 0) return vps_dispatch<float>(a, max_n, s);
  if (precision == 1) return vps_dispatch<__half>(a, max_n, s);
  return vps_dispatch<__nv_bfloat16>(a, max_n, s);
}

}  // namespace cold
