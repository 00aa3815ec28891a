// DRAM cost of random 4-byte gathers on B200: one lookup per thread into a
// 1 GiB array, each lookup in its own 1 KiB row (the table access pattern).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void gather_cg(const float* __restrict__ t, const uint8_t* __restrict__ v,
                          float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __ldcg(t + (size_t)i * 256 + v[i]);
}
__global__ void gather_ca(const float* __restrict__ t, const uint8_t* __restrict__ v,
                          float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __ldg(t + (size_t)i * 256 + v[i]);
}
// sequential 32 B record per thread (the sparse-record alternative)
__global__ void rec32(const uint4* __restrict__ r, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint4 a = __ldcs(r + 2 * (size_t)i), b = __ldcs(r + 2 * (size_t)i + 1);
    out[i] = (float)(a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w);
  }
}

int main(int argc, char** argv) {
  int gran = argc > 1 ? atoi(argv[1]) : -1;
  if (gran >= 0) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("granularity request %d -> rc %d, now %zu\n", gran, (int)e, got);
  }
  const int n = 1 << 20;  // 1M lookups, 1 GiB table
  float *t, *out;
  uint8_t* v;
  uint4* r;
  cudaMalloc(&t, (size_t)n * 256 * 4);
  cudaMalloc(&out, (size_t)n * 4);
  cudaMalloc(&v, n);
  cudaMalloc(&r, (size_t)n * 32);
  cudaMemset(t, 0, (size_t)n * 256 * 4);
  cudaMemset(r, 1, (size_t)n * 32);
  uint8_t* hv = (uint8_t*)malloc(n);
  for (int i = 0; i < n; ++i) hv[i] = (uint8_t)(rand() & 255);
  cudaMemcpy(v, hv, n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a);
    gather_cg<<<n / 256, 256>>>(t, v, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("gather_cg  %.1f us  %.2f Glookups/s\n", ms * 1e3, n / ms / 1e6);
    cudaEventRecord(a);
    gather_ca<<<n / 256, 256>>>(t, v, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("gather_ca  %.1f us  %.2f Glookups/s\n", ms * 1e3, n / ms / 1e6);
    cudaEventRecord(a);
    rec32<<<n / 256, 256>>>(r, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("rec32      %.1f us  %.2f Grec/s  %.0f GB/s\n", ms * 1e3, n / ms / 1e6, n * 32.0 / ms / 1e6);
  }
  return 0;
}
