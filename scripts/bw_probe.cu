// bw_probe.cu — load-path design-space probe for the counting kernel (not product code).
//
// Measures, on a 1 GiB / 4 GiB device buffer, the read bandwidth of
//   * TMA bulk-copy pipelines (chunk bytes x stages x consumer warps x
//     copies-per-stage x grid-stride/contiguous), consumer = XOR or full count
//   * LDG.128 register-fed streams (unroll x threads x blocks/SM)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2412_16370_b200/csrc/pp_device.cuh"

using namespace pp;

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

template <int NCW, int STAGES, int VPT, int SPLIT, bool COUNT, bool CONTIG>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    tma_probe(const uint8_t *body, unsigned long long nbytes, unsigned long long *sink) {
  static_assert(VPT % 8 == 0 && VPT >= 8, "consumers eat groups of 8 vectors");
  constexpr int SV = NCW * 32 * VPT;
  constexpr unsigned CH = SV * 16u;
  extern __shared__ __align__(128) uint8_t smem[];
  uint4 *stages = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)STAGES * CH);
  uint64_t *empty = full + STAGES;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long nch = nbytes / CH;
  unsigned long long c0, c1, cs;
  if (CONTIG) {
    c0 = nch * blockIdx.x / gridDim.x;
    c1 = nch * (blockIdx.x + 1) / gridDim.x;
    cs = 1;
  } else {
    c0 = blockIdx.x;
    c1 = nch;
    cs = gridDim.x;
  }
  if (warp == NCW) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t st = 0, ph = 0;
      for (unsigned long long ch = c0; ch < c1; ch += cs) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], CH);
#pragma unroll
        for (int k = 0; k < SPLIT; ++k)
          bulk_g2s(reinterpret_cast<uint8_t *>(stages + st * SV) + k * (CH / SPLIT),
                   body + ch * CH + k * (CH / SPLIT), CH / SPLIT, &full[st], pol);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    const TC t = make_tc(lane);
    Counter c;
    c.init();
    uint32_t xs = 0, st = 0, ph = 0;
    for (unsigned long long ch = c0; ch < c1; ch += cs) {
      mbar_wait(&full[st], ph);
      const uint4 *sv = stages + st * SV;
#pragma unroll
      for (int g = 0; g < VPT / 8; ++g) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = sv[threadIdx.x + (g * 8 + i) * (NCW * 32)];
        if (g == VPT / 8 - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (COUNT) {
          c.eat8(v, t);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) xs ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
        }
      }
      if (++st == STAGES) {
        st = 0;
        ph ^= 1;
      }
    }
    if (COUNT) {
      c.finish(t);
      xs = (uint32_t)(c.ce ^ c.co);
    }
    xs = __reduce_xor_sync(FULL, xs);
    if (lane == 0) atomicXor(sink, (unsigned long long)xs);
  }
}

template <int UNROLL, bool COUNT>
__global__ void ldg_probe(const uint4 *p, unsigned long long nvec, unsigned long long *sink) {
  const TC t = make_tc(threadIdx.x & 31);
  Counter c;
  c.init();
  uint32_t xs = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long step = stride * UNROLL;
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       b + (UNROLL - 1) * stride < nvec; b += step) {
    uint4 v[UNROLL];
#pragma unroll
    for (int i = 0; i < UNROLL; ++i) v[i] = ldg_stream(p + b + i * stride);
    if (COUNT) {
#pragma unroll
      for (int g = 0; g < UNROLL / 8; ++g) {
        uint4 w8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w8[i] = v[g * 8 + i];
        c.eat8(w8, t);
      }
    } else {
#pragma unroll
      for (int i = 0; i < UNROLL; ++i) xs ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
    }
  }
  if (COUNT) {
    c.finish(t);
    xs = (uint32_t)(c.ce ^ c.co);
  }
  xs = __reduce_xor_sync(FULL, xs);
  if ((threadIdx.x & 31) == 0) atomicXor(sink, (unsigned long long)xs);
}

static int g_sms;
static const int REPS = 20;

template <typename F>
static double time_it(F launch, unsigned long long bytes) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < REPS; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return (double)bytes * REPS / (ms / 1e3) / 1e9;
}

template <int NCW, int STAGES, int VPT, int SPLIT, bool COUNT, bool CONTIG>
static void run_tma(const uint8_t *buf, unsigned long long n, unsigned long long *sink) {
  constexpr size_t CH = (size_t)NCW * 32 * VPT * 16;
  const size_t smem = STAGES * CH + 2 * STAGES * 8;
  auto k = tma_probe<NCW, STAGES, VPT, SPLIT, COUNT, CONTIG>;
  if (smem > 227 * 1024) return;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, (NCW + 1) * 32, smem));
  const unsigned long long used = n / CH * CH;
  for (int bps = 1; bps <= occ && bps <= 2; ++bps) {
    double gbs = time_it([&] { k<<<g_sms * bps, (NCW + 1) * 32, smem>>>(buf, used, sink); }, used);
    printf("tma  %-5s %-6s ncw=%2d stages=%d chunk=%3zuKB split=%d ctas/sm=%d : %8.1f GB/s\n",
           COUNT ? "count" : "read", CONTIG ? "contig" : "stride", NCW, STAGES, CH >> 10, SPLIT,
           bps, gbs);
  }
}

template <int UNROLL, bool COUNT>
static void run_ldg(const uint8_t *buf, unsigned long long n, unsigned long long *sink, int threads) {
  auto k = ldg_probe<UNROLL, COUNT>;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0));
  const unsigned long long nvec = n / 16;
  double gbs = time_it(
      [&] { k<<<g_sms * occ, threads, 0>>>(reinterpret_cast<const uint4 *>(buf), nvec, sink); }, n);
  printf("ldg  %-5s unroll=%2d threads=%4d ctas/sm=%d : %8.1f GB/s\n", COUNT ? "count" : "read",
         UNROLL, threads, occ, gbs);
}

int main(int argc, char **argv) {
  unsigned long long n = (argc > 1 ? strtoull(argv[1], 0, 10) : 1ull) << 30;
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *buf;
  unsigned long long *sink;
  CK(cudaMalloc(&buf, n));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 0x5A, n));
  setvbuf(stdout, nullptr, _IONBF, 0);
  printf("bytes=%llu sms=%d\n", n, g_sms);
  for (int round = 0; round < 3; ++round) {
    printf("round %d\n", round);
    run_tma<8, 6, 8, 1, true, false>(buf, n, sink);
    run_tma<8, 4, 8, 1, true, false>(buf, n, sink);
    run_tma<8, 3, 8, 1, true, false>(buf, n, sink);
    run_tma<8, 5, 8, 1, true, false>(buf, n, sink);
    run_tma<4, 4, 8, 1, true, false>(buf, n, sink);
    run_tma<4, 6, 8, 1, true, false>(buf, n, sink);
    run_tma<4, 8, 8, 1, true, false>(buf, n, sink);
    run_tma<4, 5, 8, 1, true, false>(buf, n, sink);
    run_tma<6, 4, 8, 1, true, false>(buf, n, sink);
    run_tma<6, 5, 8, 1, true, false>(buf, n, sink);
    run_tma<2, 8, 8, 1, true, false>(buf, n, sink);
    run_tma<2, 12, 8, 1, true, false>(buf, n, sink);
    run_tma<4, 3, 16, 1, true, false>(buf, n, sink);
    run_tma<8, 4, 8, 1, false, false>(buf, n, sink);
    run_tma<4, 6, 8, 1, false, false>(buf, n, sink);
    run_ldg<8, true>(buf, n, sink, 256);
    run_ldg<16, true>(buf, n, sink, 256);
    run_ldg<16, false>(buf, n, sink, 256);
  }
  return 0;
}
