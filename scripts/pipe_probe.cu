// Throughput of mad.lo.u32 / mad.hi.u32 (FMA pipe) against lop3 (ALU pipe) and of the
// two pipes together on one SM's worth of warps: lane-ops per clock per SM.
#include <cstdint>
#include <cstdio>
template <int OP>
__global__ void __launch_bounds__(512) k(uint32_t *out, uint32_t m, uint32_t n, long long *clk) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i;
  const long long t0 = clock64();
  for (uint32_t it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(it));
      if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(it));
      if (OP == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(m), "r"(it));
      if (OP == 3) {  // one lop3 + one mad.lo
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(it));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(m), "r"(it));
      }
      if (OP == 4) {  // one lop3 + one mad.hi
        if (i & 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(m), "r"(it));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(m), "r"(it));
      }
    }
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char *name, uint32_t *out, long long *clk) {
  const uint32_t n = 20000;
  k<OP><<<148, 512>>>(out, 3u, n, clk);
  k<OP><<<148, 512>>>(out, 3u, n, clk);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("%-18s %.1f lane-ops/clk/SM\n", name, 512.0 * 8 * n / c);
}
int main() {
  uint32_t *out; long long *clk;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&clk, 148 * 8);
  run<0>("mad.lo.u32", out, clk);
  run<1>("mad.hi.u32", out, clk);
  run<2>("lop3", out, clk);
  run<3>("lop3+mad.lo", out, clk);
  run<4>("lop3+mad.hi", out, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
