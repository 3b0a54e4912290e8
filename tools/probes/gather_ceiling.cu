// gather_ceiling.cu — what random row gathers can reach on this B200 (the practical ceiling the
// embedding gather's HBM roofline fraction should be read against).
//
// Each thread issues RB independent 256-bit (32 B = one sector) loads of uniformly random rows
// (counter hash, no dependent id loads), sums them and writes one word per thread so nothing is
// dead-code eliminated. Table sizes: 4 GiB (HBM-resident), 32 MiB (L2-resident), plus a sequential
// copy for the peak. Useful bytes = rows x row bytes. Reported with CUDA events after warm-up.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_ceiling gather_ceiling.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL; k ^= k >> 33;
  return k;
}

template <int RB, int ROWB>
__global__ void __launch_bounds__(256) gather_rand(const uint4* __restrict__ tab, uint64_t rows, int iters,
                                                   uint32_t* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
    uint4 v[RB][ROWB / 16];
#pragma unroll
    for (int r = 0; r < RB; r++) {
      const uint64_t row = __umul64hi(fmix64(tid * 1315423911ULL + (uint64_t)(it * RB + r)), rows);
      const uint4* p = tab + row * (ROWB / 16);
#pragma unroll
      for (int q = 0; q < ROWB / 16; q += 2)
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[r][q].x), "=r"(v[r][q].y), "=r"(v[r][q].z), "=r"(v[r][q].w), "=r"(v[r][q + 1].x),
                       "=r"(v[r][q + 1].y), "=r"(v[r][q + 1].z), "=r"(v[r][q + 1].w)
                     : "l"(p + q));
    }
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int q = 0; q < ROWB / 16; q++) acc += v[r][q].x ^ v[r][q].y ^ v[r][q].z ^ v[r][q].w;
  }
  out[tid] = acc;
}

__global__ void copy_seq(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int RB, int ROWB>
void run(const char* name, const uint4* tab, uint64_t tab_bytes, uint32_t* out, int blocks) {
  const uint64_t rows = tab_bytes / ROWB;
  const int iters = 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_rand<RB, ROWB><<<blocks, 256>>>(tab, rows, iters, out);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; i++) gather_rand<RB, ROWB><<<blocks, 256>>>(tab, rows, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)reps * blocks * 256.0 * iters * RB * ROWB;
  printf("{\"probe\": \"%s\", \"row_bytes\": %d, \"rows_in_flight_per_thread\": %d, \"ctas\": %d, "
         "\"table_mib\": %.0f, \"useful_gbs\": %.1f, \"grows_per_s\": %.2f}\n",
         name, ROWB, RB, blocks, tab_bytes / 1048576.0, bytes / (ms * 1e-3) / 1e9,
         bytes / ROWB / (ms * 1e-3) / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t big = 4ull << 30, small = 32ull << 20;
  uint4 *tab, *dst;
  uint32_t* out;
  cudaMalloc(&tab, big);
  cudaMalloc(&dst, big);
  cudaMemset(tab, 1, big);
  const int blocks = sms * 8;
  cudaMalloc(&out, (size_t)blocks * 256 * 4);
  {   // sequential copy peak (read + write)
    const uint64_t n = big / 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    copy_seq<<<sms * 8, 512>>>(tab, dst, n);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; i++) copy_seq<<<sms * 8, 512>>>(tab, dst, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\": \"copy_seq\", \"gbs\": %.1f}\n", 5.0 * 2 * big / (ms * 1e-3) / 1e9);
  }
  run<4, 32>("hbm_rand32", tab, big, out, blocks);
  run<8, 32>("hbm_rand32", tab, big, out, blocks);
  run<16, 32>("hbm_rand32", tab, big, out, sms * 4);
  run<4, 64>("hbm_rand64", tab, big, out, blocks);
  run<8, 64>("hbm_rand64", tab, big, out, sms * 4);
  run<4, 128>("hbm_rand128", tab, big, out, sms * 4);
  for (uint64_t mb : {128ull, 256ull, 512ull, 1024ull, 2048ull})   // TLB reach vs table span
    run<8, 32>("span_rand32", tab, mb << 20, out, blocks);
  for (int gran : {32, 64, 128}) {   // cudaLimitMaxL2FetchGranularity: DRAM fetch size behind a miss
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity\": %zu}\n", got);
    run<8, 32>("hbm_rand32_gran", tab, big, out, blocks);
    run<8, 32>("span_rand32_gran", tab, 256ull << 20, out, blocks);
  }
  run<4, 32>("l2_rand32", tab, small, out, blocks);
  run<8, 32>("l2_rand32", tab, small, out, blocks);
  run<16, 32>("l2_rand32", tab, small, out, sms * 4);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
