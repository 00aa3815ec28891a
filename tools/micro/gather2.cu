// DRAM bytes per random 4-byte lookup for different load flavours (B200).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define K(name, body)                                                          \
  __global__ void name(const float* __restrict__ t,                           \
                       const uint8_t* __restrict__ v, float* out, int n) {    \
    int i = blockIdx.x * blockDim.x + threadIdx.x;                            \
    if (i >= n) return;                                                        \
    const float* a = t + (size_t)i * 256 + v[i];                               \
    float r;                                                                   \
    body;                                                                      \
    out[i] = r;                                                                \
  }

K(k_cv, asm volatile("ld.global.cv.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_lu, asm volatile("ld.global.lu.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_relaxed, asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_volatile, asm volatile("ld.volatile.global.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_nc_na, asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_ef, asm volatile("ld.global.L1::evict_first.f32 %0, [%1];" : "=f"(r) : "l"(a)))
K(k_atom, unsigned u = atomicAdd((unsigned*)a, 0u); r = __uint_as_float(u))
K(k_v4, { const float4* q = (const float4*)((uintptr_t)a & ~(uintptr_t)15);
          float4 x = __ldcg(q); r = x.x + x.y + x.z + x.w; })

// TMA-path bulk copy of the 16-B chunk holding the entry, per thread
__global__ void k_bulk(const float* __restrict__ t, const uint8_t* __restrict__ v,
                       float* out, int n) {
  __shared__ __align__(16) float buf[256 * 4];
  __shared__ __align__(8) unsigned long long bar;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sb), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb),
                 "r"(16 * blockDim.x));
  __syncthreads();
  const float* a = t + (size_t)i * 256 + (v[i] & ~3);
  unsigned dst = (unsigned)__cvta_generic_to_shared(buf + threadIdx.x * 4);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(dst),
      "l"(a), "r"(sb)
      : "memory");
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(sb));
  out[i] = buf[threadIdx.x * 4 + (v[i] & 3)];
}

int main() {
  const int n = 1 << 20;
  float *t, *out;
  uint8_t* v;
  cudaMalloc(&t, (size_t)n * 256 * 4);
  cudaMalloc(&out, (size_t)n * 4);
  cudaMalloc(&v, n);
  cudaMemset(t, 0, (size_t)n * 256 * 4);
  uint8_t* hv = (uint8_t*)malloc(n);
  for (int i = 0; i < n; ++i) hv[i] = (uint8_t)(rand() & 255);
  cudaMemcpy(v, hv, n, cudaMemcpyHostToDevice);
  typedef void (*F)(const float*, const uint8_t*, float*, int);
  F fs[] = {k_cv, k_lu, k_relaxed, k_volatile, k_nc_na, k_ef, k_atom, k_v4, k_bulk};
  const char* nm[] = {"cv", "lu", "relaxed", "volatile", "nc_noalloc", "evict_first", "atom", "v4", "bulk16"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep)
    for (int k = 0; k < 9; ++k) {
      float ms;
      cudaEventRecord(a);
      fs[k]<<<n / 256, 256>>>(t, v, out, n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%-12s %7.1f us  %6.2f Glookups/s  (%s)\n", nm[k], ms * 1e3,
                      n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
