// gather4_probe.cu — random 32 B row gathers on B200: LSU (ld.global.nc.v8 per thread, 8 rows in flight)
// vs TMA tile::gather4 (4 rows per instruction into a shared-memory ring, mbarrier completion) vs 32 B
// cp.async.bulk per row. Rows from an L2-resident 32 MB table and a 320 MB table. Prints JSON lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); exit(1); } \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- LSU: each thread sums 8 rows in flight per iteration
__global__ void __launch_bounds__(128, 8) lsu_kernel(const uint4* __restrict__ tab, const int* __restrict__ ids,
                                                     long n, float* out) {
  float acc = 0.f;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n / 8; i += stride) {
    uint4 a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint4* p = tab + 2 * (long)__ldg(ids + i * 8 + j);
      asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(a[j].x), "=r"(a[j].y), "=r"(a[j].z), "=r"(a[j].w), "=r"(b[j].x), "=r"(b[j].y),
                     "=r"(b[j].z), "=r"(b[j].w)
                   : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < 8; j++) acc += __uint_as_float(a[j].x ^ b[j].w) * 1e-30f;
  }
  if (acc == 1.2345f) out[0] = acc;
}

// ---- TMA: warp 0 produces (each lane one gather4 or four bulk copies per stage), warps 1..4 consume
constexpr int STAGES = 8, ROWS = 128, STAGE_BYTES = ROWS * 32;

template <int MODE>   // 0: tile::gather4, 1: cp.async.bulk 32 B per row
__global__ void __launch_bounds__(160) tma_kernel(const __grid_constant__ CUtensorMap tm, const uint4* __restrict__ tab,
                                                  const int* __restrict__ ids, long n, float* out) {
  __shared__ __align__(1024) uint8_t ring[STAGES][STAGE_BYTES];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long tiles = n / ROWS;
  auto wait = [](uint64_t* bar, uint32_t ph) {
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(bar)),
        "r"(ph)
        : "memory");
  };
  if (warp == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int4 r = __ldg(reinterpret_cast<const int4*>(ids + t * ROWS) + lane);
      if (lane == 0) {
        wait(&empty[s], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE_BYTES)
                     : "memory");
      }
      __syncwarp();
      const uint32_t dst = sa(&ring[s][lane * 128]);
      if (MODE == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
            "l"((uint64_t)&tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(sa(&full[s]))
            : "memory");
      } else {
        const int rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 4; j++)
          asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];" ::"r"(
                           dst + 32 * j),
                       "l"(tab + 2 * (long)rr[j]), "r"(sa(&full[s]))
                       : "memory");
      }
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else {
    const int c = threadIdx.x - 32;
    float acc = 0.f;
    int s = 0;
    uint32_t ph = 0;
    for (long t = blockIdx.x; t < tiles; t += gridDim.x) {
      wait(&full[s], ph);
      uint4 q;
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                   : "r"(sa(&ring[s][c * 32])));
      acc += __uint_as_float(q.x) * 1e-30f;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (acc == 1.2345f) out[0] = acc;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  const long n = 64L << 20;   // lookups
  int* d_ids;
  CK(cudaMalloc(&d_ids, n * 4));
  float* d_out;
  CK(cudaMalloc(&d_out, 4));
  for (long card : {1L << 20, 10000000L}) {
    uint4* tab;
    CK(cudaMalloc(&tab, card * 32));
    CK(cudaMemset(tab, 1, card * 32));
    std::vector<int> h(n);
    uint64_t x = 88172645463325252ull;
    for (long i = 0; i < n; i++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[i] = (int)(x % (uint64_t)card);
    }
    CK(cudaMemcpy(d_ids, h.data(), n * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t dims[2] = {16, (cuuint64_t)card};
    cuuint64_t strides[1] = {32};
    cuuint32_t box[2] = {16, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("{\"encode_error\": %d}\n", (int)r);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 5; mode++) {
      // mode 0 LSU; 1 gather4 x4 CTAs/SM; 2 gather4 x8; 3 bulk32 x4; 4 bulk32 x8
      auto launch = [&]() {
        if (mode == 0) lsu_kernel<<<148 * 8, 128>>>(tab, d_ids, n, d_out);
        else if (mode <= 2) tma_kernel<0><<<148 * (mode == 1 ? 4 : 8), 160>>>(tm, tab, d_ids, n, d_out);
        else tma_kernel<1><<<148 * (mode == 3 ? 4 : 8), 160>>>(tm, tab, d_ids, n, d_out);
      };
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int it = 0; it < 5; it++) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* names[5] = {"lsu_v8_8inflight", "gather4_4cta", "gather4_8cta", "bulk32_4cta", "bulk32_8cta"};
      printf("{\"table_rows\": %ld, \"mode\": \"%s\", \"grows_per_s\": %.2f}\n", card, names[mode],
             5.0 * n / (ms / 1e3) / 1e9);
      fflush(stdout);
    }
    cudaFree(tab);
  }
  return 0;
}
