// Probe: tcgen05.mma kind::f16, M=128 N=128 K=16, A/B K-major with SWIZZLE_NONE descriptors.
// Checks the core-matrix layout offset(row, kchunk) = (row/8)*SBO + kchunk*LBO + (row%8)*16 against a
// host reference for several (LBO, SBO) encodings. Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include "../../paper_2007_16122_b200/csrc/ptx.cuh"
using namespace cold;

__global__ void probe(const __half* A, const __half* B, float* D, int lbo, int sbo, int mode) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[128 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // layout: row r, 8-half chunk j at (r/8)*256 + j*128 + (r%8)*16 (written with the probe's own offsets)
  for (int i = t; i < 128 * 2; i += blockDim.x) {
    const int r = i >> 1, j = i & 1;
    const uint32_t off = (uint32_t)((r >> 3) * 256 + j * 128 + (r & 7) * 16);
    *reinterpret_cast<uint4*>(sa + off) = *reinterpret_cast<const uint4*>(A + r * 16 + j * 8);
    *reinterpret_cast<uint4*>(sb + off) = *reinterpret_cast<const uint4*>(B + r * 16 + j * 8);
  }
  fence_async_smem();
  if (t == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (t == 0) {
    auto desc = [&](uint32_t a) {
      uint64_t d = 0;
      d |= (uint64_t)((a & 0x3FFFFu) >> 4);
      d |= (uint64_t)(lbo >> 4) << 16;
      d |= (uint64_t)(sbo >> 4) << 32;
      d |= (uint64_t)1 << 46;
      if (mode == 1) d |= (uint64_t)1 << 52;
      return d;
    };
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    umma_f16(tm, desc(smem_u32(sa)), desc(smem_u32(sb)), idesc, 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < 128; c += 32) {
    TMEM_LD32(tm + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 32; i++) D[(warp * 32 + lane) * 128 + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128) : "memory");
}

int main() {
  __half hA[128 * 16], hB[128 * 16];
  float fa[128 * 16], fb[128 * 16];
  srand(1);
  for (int i = 0; i < 128 * 16; i++) {
    fa[i] = (float)(rand() % 7 - 3); fb[i] = (float)(rand() % 5 - 2);
    hA[i] = __float2half(fa[i]); hB[i] = __float2half(fb[i]);
  }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  static float D[128 * 128];
  const int combos[][3] = {{128, 256, 0}, {256, 128, 0}, {128, 256, 1}, {256, 128, 1}};
  for (auto& cb : combos) {
    cudaMemset(dD, 0, 128 * 128 * 4);
    probe<<<1, 128>>>(dA, dB, dD, cb[0], cb[1], cb[2]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; m++)
      for (int n = 0; n < 128; n++) {
        float ref = 0;
        for (int k = 0; k < 16; k++) ref += fa[m * 16 + k] * fb[n * 16 + k];
        if (D[m * 128 + n] != ref) bad++;
      }
    printf("LBO=%d SBO=%d lbo_mode=%d: %s, mismatches %d / %d\n", cb[0], cb[1], cb[2], cudaGetErrorString(e), bad, 128 * 128);
  }
  return 0;
}
