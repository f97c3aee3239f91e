// pp_categories.cu — fused one-hot producer + positional count (SURVEY.md 8f
// item 3): GROUP BY COUNT over a low-cardinality categorical column.
//
// The paper's motivating use is the histogram of one-hot
// encoded categories: pospopcnt over words (1 << code).  Materialising those
// words costs w/8 bytes per row written and read; this kernel consumes the
// category codes directly and produces exactly
//     counters[j] += #{i : codes[i] == j},  j < w
//                 == pospopcnt(one_hot_w(codes), w)[j]
// where one_hot_w(c) = (c < w) ? 1 << c : 0 (codes >= w have no bit in a
// w-bit word and are not counted).
//
// Layout: each thread owns a u16 counter column in shared memory,
// cnt[bin][thread] (bin-major, so a warp's 32 columns sit in 16 consecutive
// words of every bin row: conflict-free whatever the codes).  Codes stream in
// with coalesced LDG.128 (grid-stride); each code is one LDS.U16/IADD/STS.U16
// on the thread's own column.  The host splits launches so no column exceeds
// 65535; a block reduction then adds the columns into u64 global counters.
#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

constexpr int kCatThreads = 512;
constexpr int kCatBins = 64;
constexpr size_t kCatSmem = (size_t)kCatBins * kCatThreads * sizeof(uint16_t);  // 64 KiB
constexpr unsigned long long kCatMaxPerThread = 65535;

__device__ __forceinline__ void cat_bump(uint16_t *col, uint32_t c, uint32_t ncat) {
  if (c < ncat) col[c * kCatThreads] += 1;
}

template <int CB>
__device__ __forceinline__ void cat_vec(uint16_t *col, const uint4 &v, uint32_t ncat) {
  const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (CB == 1) {
#pragma unroll
      for (int b = 0; b < 4; ++b) cat_bump(col, (w4[i] >> (8 * b)) & 0xFFu, ncat);
    } else if (CB == 2) {
      cat_bump(col, w4[i] & 0xFFFFu, ncat);
      cat_bump(col, w4[i] >> 16, ncat);
    } else {
      cat_bump(col, w4[i], ncat);
    }
  }
}

__device__ __forceinline__ uint32_t load_code(const uint8_t *p, int cb) {
  if (cb == 1) return __ldg(p);
  if (cb == 2) return __ldg(reinterpret_cast<const uint16_t *>(p));
  return __ldg(reinterpret_cast<const uint32_t *>(p));
}

// codes: [head (< 16 bytes, code-aligned)] [body: nvec aligned 16-byte vectors]
// [tail (< 16 bytes)].  CTA 0 also counts head and tail codes.
template <int CB>
__global__ void __launch_bounds__(kCatThreads, 2)
    pp_cat_kernel(const uint8_t *head, uint32_t head_bytes, const uint4 *body,
                  unsigned long long nvec, const uint8_t *tail, uint32_t tail_bytes,
                  uint32_t ncat, unsigned long long *counters) {
  extern __shared__ __align__(16) uint16_t cnt[];
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < kCatBins * kCatThreads / 8; i += kCatThreads)
    reinterpret_cast<uint4 *>(cnt)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  uint16_t *col = cnt + tid;
  const unsigned long long stride = (unsigned long long)gridDim.x * kCatThreads;
  unsigned long long k = blockIdx.x * (unsigned long long)kCatThreads + tid;
  for (; k + 3 * stride < nvec; k += 4 * stride) {  // 4 loads in flight per thread
    const uint4 a = ldg_stream(body + k), b = ldg_stream(body + k + stride),
                c = ldg_stream(body + k + 2 * stride), d = ldg_stream(body + k + 3 * stride);
    cat_vec<CB>(col, a, ncat);
    cat_vec<CB>(col, b, ncat);
    cat_vec<CB>(col, c, ncat);
    cat_vec<CB>(col, d, ncat);
  }
  for (; k < nvec; k += stride) cat_vec<CB>(col, ldg_stream(body + k), ncat);
  if (blockIdx.x == 0) {
    if (tid * CB < head_bytes) cat_bump(col, load_code(head + tid * CB, CB), ncat);
    if (tid * CB < tail_bytes) cat_bump(col, load_code(tail + tid * CB, CB), ncat);
  }
  __syncthreads();
  // 8 threads per bin, 64 columns each, then a shuffle reduction
  const uint32_t bin = tid >> 3, part = tid & 7;
  uint32_t s = 0;
  if (bin < ncat)
    for (uint32_t j = part; j < kCatThreads; j += 8) s += cnt[bin * kCatThreads + j];
  s += __shfl_xor_sync(FULL, s, 4);
  s += __shfl_xor_sync(FULL, s, 2);
  s += __shfl_xor_sync(FULL, s, 1);
  if (part == 0 && bin < ncat && s) atomicAdd(counters + bin, (unsigned long long)s);
}

static int g_cat_attr_done[64];

cudaError_t launch_categories(const uint8_t *codes, unsigned long long nbytes, int code_bytes,
                              int ncat, unsigned long long *counters, const DevInfo &di,
                              int dev, cudaStream_t st) {
  if (nbytes == 0) return cudaSuccess;
  cudaError_t e;
  if (dev >= 0 && dev < 64 && !g_cat_attr_done[dev]) {
    if ((e = cudaFuncSetAttribute(pp_cat_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kCatSmem)))
      return e;
    if ((e = cudaFuncSetAttribute(pp_cat_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kCatSmem)))
      return e;
    if ((e = cudaFuncSetAttribute(pp_cat_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kCatSmem)))
      return e;
    g_cat_attr_done[dev] = 1;
  }
  const unsigned long long grid_cap = 2ull * di.num_sms;
  // split so that no thread's u16 column can wrap: codes per thread <= 65535
  const unsigned long long codes_per_vec = 16ull / code_bytes;
  const unsigned long long max_vec =
      grid_cap * kCatThreads * (kCatMaxPerThread / codes_per_vec - 1);
  const uint8_t *p = codes;
  unsigned long long left = nbytes;
  while (left) {
    const unsigned long long mis = (16u - ((uintptr_t)p & 15u)) & 15u;
    const unsigned long long hb = mis < left ? mis : left;
    unsigned long long nvec = (left - hb) >> 4;
    if (nvec > max_vec) nvec = max_vec;
    const unsigned long long used = hb + (nvec << 4);
    const unsigned long long tb = (nvec == (left - hb) >> 4) ? left - used : 0;
    unsigned long long g = (nvec + kCatThreads - 1) / kCatThreads;
    if (g > grid_cap) g = grid_cap;
    if (g == 0) g = 1;
    const uint4 *body = reinterpret_cast<const uint4 *>(p + hb);
    if (code_bytes == 1)
      pp_cat_kernel<1><<<(unsigned)g, kCatThreads, kCatSmem, st>>>(
          p, (uint32_t)hb, body, nvec, p + used, (uint32_t)tb, (uint32_t)ncat, counters);
    else if (code_bytes == 2)
      pp_cat_kernel<2><<<(unsigned)g, kCatThreads, kCatSmem, st>>>(
          p, (uint32_t)hb, body, nvec, p + used, (uint32_t)tb, (uint32_t)ncat, counters);
    else
      pp_cat_kernel<4><<<(unsigned)g, kCatThreads, kCatSmem, st>>>(
          p, (uint32_t)hb, body, nvec, p + used, (uint32_t)tb, (uint32_t)ncat, counters);
    if ((e = cudaGetLastError())) return e;
    p += used + tb;
    left -= used + tb;
  }
  return cudaSuccess;
}

}  // namespace pp
