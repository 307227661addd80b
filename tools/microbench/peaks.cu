// Microbenchmarks for the roofline denominators this path needs that
// MEASURED_PEAKS.json does not carry: FP64 FMA rate, FP64 RED throughput to
// global memory (L2-resident and HBM-resident targets, spread and clustered),
// shared-memory FP64 atomics, and a plain FP64 read stream.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// each thread issues `per` reds to hashed addresses in [0, n)
__global__ void red_spread(double* a, uint32_t n, int per) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < per; ++i) {
    uint32_t idx = hash32(t * 977u + i) % n;
    atomicAdd(a + idx, 1.0);
  }
}

// clustered: a warp's lanes hit `distinct` addresses (mimics shared mesh nodes)
__global__ void red_cluster(double* a, uint32_t n, int per, int distinct) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t w = t >> 5, lane = t & 31;
  for (int i = 0; i < per; ++i) {
    uint32_t base = hash32(w * 131u + i) % (n - 64);
    atomicAdd(a + base + (lane % distinct), 1.0);
  }
}

__global__ void smem_atomic(double* out, int per) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0;
  __syncthreads();
  for (int i = 0; i < per; ++i) atomicAdd(&s[(threadIdx.x * 37 + i * 11) & 1023], 1.0);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

__global__ void read_stream(const double2* __restrict__ a, size_t n, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i); acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* d; CK(cudaMalloc(&d, (size_t)1 << 31));
  CK(cudaMemset(d, 0, (size_t)1 << 31));
  // DFMA
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"dfma_tflops\": %.2f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // RED spread, L2-resident (64 MB) and HBM (1 GB)
  uint32_t sizes[3] = {1u << 20, 8u << 20, 128u << 20};
  for (int s = 0; s < 3; ++s) for (int rep = 0; rep < 2; ++rep) {
    int blocks = p.multiProcessorCount * 16, threads = 256, per = 64;
    cudaEventRecord(e0); red_spread<<<blocks, threads>>>(d, sizes[s], per); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * per;
    printf("{\"red_spread_Gops\": %.1f, \"target_MB\": %.0f}\n", ops / ms / 1e6, sizes[s] * 8.0 / 1e6);
  }
  int distincts[4] = {32, 16, 8, 4};
  for (int s = 0; s < 4; ++s) {
    int blocks = p.multiProcessorCount * 16, threads = 256, per = 64;
    cudaEventRecord(e0); red_cluster<<<blocks, threads>>>(d, 8u << 20, per, distincts[s]); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * per;
    printf("{\"red_cluster_Gops\": %.1f, \"distinct_per_warp\": %d}\n", ops / ms / 1e6, distincts[s]);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = p.multiProcessorCount * 8, threads = 256, per = 256;
    cudaEventRecord(e0); smem_atomic<<<blocks, threads>>>(d, per); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * per;
    printf("{\"smem_f64_atomic_Gops\": %.1f}\n", ops / ms / 1e6);
  }
  size_t n2 = ((size_t)1 << 31) / 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); read_stream<<<p.multiProcessorCount * 8, 512>>>((const double2*)d, n2, d); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"read_GBs\": %.1f}\n", (double)n2 * 16 / ms / 1e6);
  }
  return 0;
}
