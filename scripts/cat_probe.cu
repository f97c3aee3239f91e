// cat_probe.cu -- A/B probe for the categories producer at W = 64 / 32:
// which pipe should histogram u8 codes?  (profiles/r2_categories.md)
//   V1  shared-memory RED (atomicAdd, fire-and-forget) into lane-private
//       bins hist[bin][lane] (bank = lane: conflict-free whatever the codes)
//   V2  same bins, u16 lane-private, plain LDS/IADD/STS
//   V3  warp-private bins hist[warp][bin], RED (conflicts on equal codes)
// Codes: 2^30 u8, Zipf(1.1) over W categories via thresholds (like C3) or
// uniform.  Each variant is checked against a CPU histogram.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cat_probe cat_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int W, int THREADS>
__global__ void __launch_bounds__(THREADS) v1_red_lane(const uint4 *codes, unsigned long long nvec,
                                                      unsigned long long *out) {
  extern __shared__ uint32_t h[];  // [W + 1][THREADS]: bin W = "code >= W"
  for (int i = threadIdx.x; i < (W + 1) * THREADS; i += THREADS) h[i] = 0;
  __syncthreads();
  uint32_t *col = h + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * THREADS;
  unsigned long long k = blockIdx.x * (unsigned long long)THREADS + threadIdx.x;
  for (; k + stride < nvec; k += 2 * stride) {
    uint4 a = ldg_stream(codes + k), b = ldg_stream(codes + k + stride);
    const uint32_t w8[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t c = __byte_perm(w8[i], 0u, 0x4440u | j);
        c = min(c, (uint32_t)W);
        atomicAdd(col + c * THREADS, 1u);
      }
    }
  }
  for (; k < nvec; k += stride) {
    uint4 a = ldg_stream(codes + k);
    const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t c = min(__byte_perm(w4[i], 0u, 0x4440u | j), (uint32_t)W);
        atomicAdd(col + c * THREADS, 1u);
      }
  }
  __syncthreads();
  for (int b = threadIdx.x >> 3; b < W; b += THREADS / 8) {
    uint32_t s = 0;
    for (int j = threadIdx.x & 7; j < THREADS; j += 8) s += h[b * THREADS + j];
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if ((threadIdx.x & 7) == 0 && s) atomicAdd(out + b, (unsigned long long)s);
  }
}

template <int W, int THREADS>
__global__ void __launch_bounds__(THREADS) v3_red_warp(const uint4 *codes, unsigned long long nvec,
                                                      unsigned long long *out) {
  __shared__ uint32_t h[THREADS / 32][W + 1];
  for (int i = threadIdx.x; i < (THREADS / 32) * (W + 1); i += THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t *mine = h[threadIdx.x >> 5];
  const unsigned long long stride = (unsigned long long)gridDim.x * THREADS;
  for (unsigned long long k = blockIdx.x * (unsigned long long)THREADS + threadIdx.x; k < nvec;
       k += stride) {
    uint4 a = ldg_stream(codes + k);
    const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) atomicAdd(mine + min(__byte_perm(w4[i], 0u, 0x4440u | j), (uint32_t)W), 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < W; b += THREADS) {
    uint32_t s = 0;
    for (int w = 0; w < THREADS / 32; ++w) s += h[w][b];
    if (s) atomicAdd(out + b, (unsigned long long)s);
  }
}

int main(int argc, char **argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 64;
  const unsigned long long n = 1ull << 30;
  std::vector<uint8_t> host(n);
  // Zipf(1.1) over W categories via a splitmix stream (codes < W)
  std::vector<double> cdf(W);
  double z = 0;
  for (int i = 0; i < W; ++i) z += 1.0 / pow(i + 1.0, 1.1);
  double acc = 0;
  for (int i = 0; i < W; ++i) { acc += 1.0 / pow(i + 1.0, 1.1) / z; cdf[i] = acc; }
  uint64_t x = 0x1234;
  std::vector<unsigned long long> want(W + 1, 0);
  for (unsigned long long i = 0; i < n; ++i) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t t = x;
    t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
    t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
    t ^= t >> 31;
    const double u = (t >> 11) * (1.0 / 9007199254740992.0);
    int c = 0;
    while (c < W - 1 && u > cdf[c]) ++c;
    host[i] = (uint8_t)c;
    want[c]++;
  }
  uint8_t *d;
  unsigned long long *out;
  CK(cudaMalloc(&d, n));
  CK(cudaMalloc(&out, 8 * 65));
  CK(cudaMemcpy(d, host.data(), n, cudaMemcpyHostToDevice));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    CK(cudaMemset(out, 0, 8 * 65));
    const int reps = 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> got(65);
    CK(cudaMemcpy(got.data(), out, 8 * 65, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (int i = 0; i < W; ++i) ok &= got[i] == reps * want[i];
    printf("W=%d %-28s %8.1f GB/s of codes  %s\n", W, name, n * reps / (ms / 1e3) / 1e9,
           ok ? "exact" : "MISMATCH");
  };
  const unsigned long long nvec = n / 16;
#define V1(T, B)                                                                                  \
  {                                                                                               \
    const size_t sm = (size_t)(W + 1) * T * 4;                                                    \
    if (W == 64) CK(cudaFuncSetAttribute(v1_red_lane<64, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    else CK(cudaFuncSetAttribute(v1_red_lane<32, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));         \
    run("v1 RED lane-private T=" #T " B=" #B, [&] {                                               \
      if (W == 64) v1_red_lane<64, T><<<sms * B, T, sm>>>((const uint4 *)d, nvec, out);           \
      else v1_red_lane<32, T><<<sms * B, T, sm>>>((const uint4 *)d, nvec, out);                   \
    });                                                                                           \
  }
  V1(256, 2) V1(256, 3) V1(512, 1) V1(512, 2) V1(384, 2) V1(1024, 1)
  run("v3 RED warp-private T=512 B=2", [&] {
    if (W == 64) v3_red_warp<64, 512><<<sms * 2, 512>>>((const uint4 *)d, nvec, out);
    else v3_red_warp<32, 512><<<sms * 2, 512>>>((const uint4 *)d, nvec, out);
  });
  return 0;
}
