// launch_floor.cu — back-to-back launch cost of empty kernels (not product code):
// the floor under which no per-call latency of pp_count can go.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k() {}
__global__ void smem_k() { extern __shared__ char s[]; if (threadIdx.x == 999) s[0] = 1; }
__global__ void atom_k(unsigned long long *c) { if (threadIdx.x < 8) atomicAdd(c + threadIdx.x, 1ull); }
int main() {
  unsigned long long *c; cudaMalloc(&c, 64 * 8);
  cudaFuncSetAttribute(smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024 + 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char *name, auto f) {
    for (int i = 0; i < 100; ++i) f();
    cudaDeviceSynchronize(); cudaEventRecord(a);
    for (int i = 0; i < 1000; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %.2f us/launch\n", name, ms);
  };
  run("empty <<<1,32>>>", [] { empty_k<<<1, 32>>>(); });
  run("empty <<<148,288>>>", [] { empty_k<<<148, 288>>>(); });
  run("smem96K <<<1,288>>>", [] { smem_k<<<1, 288, 96 * 1024 + 64>>>(); });
  run("smem96K <<<148,288>>>", [] { smem_k<<<148, 288, 96 * 1024 + 64>>>(); });
  run("atomics <<<148,288>>>", [&] { atom_k<<<148, 288>>>(c); });
  return 0;
}
