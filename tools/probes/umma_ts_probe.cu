// Probe: tcgen05.mma kind::f16 with the A operand in TENSOR MEMORY (".ts" form: [d], [a_tmem], b_desc),
// cta_group::1, M=128, N=64, K=16. A is written to TMEM by tcgen05.st.32x32b.x8 (lane = row, 32-bit
// column c = K elements 2c (low half) and 2c+1 (high half)); B is K-major SWIZZLE_NONE in shared memory
// (the layout umma_k16_probe.cu established). Checks D = A B^T against a host reference, and the same
// product accumulated over K = 64 (4 MMAs at TMEM column offsets of 8 per K = 16 step).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ts tools/probes/umma_ts_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include "../../paper_2007_16122_b200/csrc/ptx.cuh"
using namespace cold;

constexpr int NN = 64, KK = 64;

__global__ void probe(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) uint8_t sb[NN * KK * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B: per K = 16 step s, a [2][NN rows][8] no-swizzle tile (LBO = NN * 16 B between the two 8-col halves,
  // SBO = 128 B between 8-row groups)
  for (int i = t; i < NN * (KK / 8); i += blockDim.x) {
    const int r = i / (KK / 8), j = i % (KK / 8);   // row, 8-element chunk
    const int s = j / 2, h = j % 2;
    const uint32_t off = (uint32_t)(s * NN * 32 + h * NN * 16 + (r >> 3) * 128 + (r & 7) * 16);
    *reinterpret_cast<uint4*>(sb + off) = *reinterpret_cast<const uint4*>(B + r * KK + j * 8);
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
  const uint32_t ta = tm + 64;   // A at columns [64, 64 + KK/2)
  {
    // row = warp * 32 + lane: KK halves -> KK/2 32-bit columns
    const int row = warp * 32 + lane;
    uint32_t v[KK / 2];
    for (int c = 0; c < KK / 2; c++) {
      const __half lo = A[row * KK + 2 * c], hi = A[row * KK + 2 * c + 1];
      v[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    const uint32_t addr = ta + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                 "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                 "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                 "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int s = 0; s < KK / 16; s++) {
      uint64_t d = 0;
      const uint32_t a = smem_u32(sb) + s * NN * 32;
      d |= (uint64_t)((a & 0x3FFFFu) >> 4);
      d |= (uint64_t)((NN * 16) >> 4) << 16;
      d |= (uint64_t)(128 >> 4) << 32;
      d |= (uint64_t)1 << 46;
      const uint32_t acc = s > 0 ? 1u : 0u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                   "r"(ta + 8 * s), "l"(d), "r"(idesc), "r"(acc)
                   : "memory");
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < NN; c += 32) {
    TMEM_LD32(tm + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 32; i++) D[(warp * 32 + lane) * NN + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128) : "memory");
}

int main() {
  static __half hA[128 * KK], hB[NN * KK];
  static float fa[128 * KK], fb[NN * KK];
  srand(1);
  for (int i = 0; i < 128 * KK; i++) { fa[i] = (float)(rand() % 7 - 3); hA[i] = __float2half(fa[i]); }
  for (int i = 0; i < NN * KK; i++) { fb[i] = (float)(rand() % 5 - 2); hB[i] = __float2half(fb[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 128 * NN * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 128 * NN * 4);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  static float D[128 * NN];
  cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; m++)
    for (int n = 0; n < NN; n++) {
      float ref = 0;
      for (int k = 0; k < KK; k++) ref += fa[m * KK + k] * fb[n * KK + k];
      if (D[m * NN + n] != ref) bad++;
    }
  printf("{\"probe\": \"umma_ts\", \"err\": \"%s\", \"mismatches\": %d, \"of\": %d}\n", cudaGetErrorString(e), bad, 128 * NN);
  return 0;
}
