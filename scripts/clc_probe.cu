// Probe of Blackwell cluster launch control (clusterlaunchcontrol.try_cancel): a grid of G one-warp CTAs
// whose resident CTAs cancel and take over the pending ones; prints ns per work unit (every unit taken once).
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(unsigned long long *out, unsigned int *hist) {
  __shared__ __align__(16) uint4 resp;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  uint32_t bx = blockIdx.x;
  unsigned long long n = 0;
  if (threadIdx.x == 0) {
    for (;;) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile(
          "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
              smem_u32(&resp)),
          "r"(smem_u32(&bar))
          : "memory");
      ++n;
      atomicAdd(&hist[bx], 1u);
      uint32_t done;
      do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(&bar)), "r"(phase)
            : "memory");
      } while (!done);
      phase ^= 1;
      unsigned long long lo, hi;
      asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(smem_u32(&resp)) : "memory");
      uint32_t ok, x = 0;
      asm volatile(
          "{\n\t.reg .b128 r;\n\t.reg .pred p;\n\tmov.b128 r, {%2, %3};\n\t"
          "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t"
          "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n\t}"
          : "=r"(ok), "+r"(x)
          : "l"(lo), "l"(hi));
      if (!ok) break;
      bx = x;
    }
    atomicAdd(out, n);
  }
}
int main() {
  unsigned long long *out; unsigned int *hist;
  const int G = 100000;
  cudaMalloc(&out, 8); cudaMemset(out, 0, 8);
  cudaMalloc(&hist, 4 * G); cudaMemset(hist, 0, 4 * G);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaMemset(out, 0, 8); cudaMemset(hist, 0, 4 * G);
    cudaEventRecord(a);
    k<<<G, 32>>>(out, hist);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    unsigned int *hh = new unsigned int[G]; cudaMemcpy(hh, hist, 4 * G, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < G; ++i) bad += hh[i] != 1;
    printf("err=%s total=%llu (want %d) bad=%d  %.3f ms -> %.1f ns per unit\n", cudaGetErrorString(e), h, G, bad, ms, ms * 1e6 / G);
  }
  return 0;
}
