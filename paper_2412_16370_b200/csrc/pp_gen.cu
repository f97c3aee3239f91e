// pp_gen.cu — seeded synthetic inputs generated in place on the device.
//
// Benchmark / test infrastructure, not the hot path.  Definitions (SURVEY.md
// section 8d) with byte-identical CPU twins in oracle/pospopcnt_oracle.c:
//   mix64(z)       splitmix64 finaliser
//   uniform        u64 word g = mix64(seed + (g+1) * GOLDEN)
//   bernoulli(q)   u64 word g = AND/OR ladder over draws
//                  r_k = mix64(seed + (16 g + k + 1) * GOLDEN), k = 0..15,
//                  LSB of q first: x = q_k ? x | r_k : x & r_k  -> P(bit) = q/2^16
//                  (q = 65536 -> all ones)
//   blocks         bernoulli with q_b = mix64((seed ^ SALT) + (b+1) GOLDEN) mod 65537
//                  for block b = (8 g) / block_bytes
//   onehot32       u32 word g = 1 << #{k < 31 : thr[k] <= hi32(mix64(seed + (g+1) GOLDEN))}
//   codes8         u8 code g = that same bit position (one_hot(codes8) == onehot32)
#include "pp_internal.h"

namespace pp {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t BLOCK_SALT = 0x5EEDB10C5EEDB10Cull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Every generator lets a programmatic dependent launch start immediately
// (PDL trigger at entry), before a single output byte is written.  The
// counting kernels launched behind it must therefore honour the PDL
// contract -- griddepcontrol.wait before their first read -- and the
// generate-then-count tests check exactly that.
__device__ __forceinline__ void pdl_trigger_now() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t ladder(uint64_t seed, uint64_t g, uint32_t q) {
  if (q >= 65536u) return ~0ull;
  uint64_t x = 0;
  const uint64_t base = seed + (16ull * g + 1ull) * GOLDEN;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint64_t r = mix64(base + (uint64_t)k * GOLDEN);
    x = ((q >> k) & 1u) ? (x | r) : (x & r);
  }
  return x;
}

__global__ void gen_uniform_kernel(uint64_t *dst, unsigned long long n, uint64_t seed,
                                   uint64_t off) {
  pdl_trigger_now();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = mix64(seed + (off + i + 1ull) * GOLDEN);
}

__global__ void gen_bernoulli_kernel(uint64_t *dst, unsigned long long n, uint64_t seed,
                                     uint64_t off, uint32_t q) {
  pdl_trigger_now();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = ladder(seed, off + i, q);
}

__global__ void gen_blocks_kernel(uint64_t *dst, unsigned long long n, uint64_t seed,
                                  uint64_t off, uint64_t block_bytes) {
  pdl_trigger_now();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint64_t g = off + i;
    const uint64_t b = (g * 8ull) / block_bytes;
    const uint32_t q = (uint32_t)(mix64((seed ^ BLOCK_SALT) + (b + 1ull) * GOLDEN) % 65537ull);
    dst[i] = ladder(seed, g, q);
  }
}

struct Thr31 {
  uint32_t t[31];
};

__global__ void gen_onehot32_kernel(uint32_t *dst, unsigned long long n, uint64_t seed,
                                    uint64_t off, Thr31 thr) {
  pdl_trigger_now();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(mix64(seed + (off + i + 1ull) * GOLDEN) >> 32);
    uint32_t cat = 0;
#pragma unroll
    for (int k = 0; k < 31; ++k) cat += (thr.t[k] <= u) ? 1u : 0u;
    dst[i] = 1u << cat;
  }
}

// u8 category codes with the C3 distribution: code i = the bit position of
// onehot32 word i (same draws), so one_hot(codes8[i]) == onehot32[i].
__global__ void gen_codes8_kernel(uint8_t *dst, unsigned long long n, uint64_t seed,
                                  uint64_t off, Thr31 thr) {
  pdl_trigger_now();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(mix64(seed + (off + i + 1ull) * GOLDEN) >> 32);
    uint32_t cat = 0;
#pragma unroll
    for (int k = 0; k < 31; ++k) cat += (thr.t[k] <= u) ? 1u : 0u;
    dst[i] = (uint8_t)cat;
  }
}

// One resident wave (4 x 256 threads per SM) with the shared-memory carveout
// at its maximum, so a counting CTA (96+ KiB of shared memory) can join each
// SM while the generator still runs: with the PDL trigger at entry, a count
// launched behind a generator really overlaps it -- the hazard the
// generate-then-count test needs (an SM can only host CTAs of one carveout).
static unsigned gen_grid(unsigned long long n) {
  static bool carveout_set = false;
  if (!carveout_set) {
    const void *ks[] = {(const void *)gen_uniform_kernel, (const void *)gen_bernoulli_kernel,
                        (const void *)gen_blocks_kernel, (const void *)gen_onehot32_kernel,
                        (const void *)gen_codes8_kernel};
    for (const void *k : ks)
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
    cudaGetLastError();
    carveout_set = true;
  }
  unsigned long long g = (n + 255) / 256;
  const unsigned long long cap = 148ull * 4;
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

cudaError_t launch_gen_uniform(uint64_t *dst, unsigned long long n, uint64_t seed,
                               uint64_t off, cudaStream_t st) {
  if (!n) return cudaSuccess;
  gen_uniform_kernel<<<gen_grid(n), 256, 0, st>>>(dst, n, seed, off);
  return cudaGetLastError();
}
cudaError_t launch_gen_bernoulli(uint64_t *dst, unsigned long long n, uint64_t seed,
                                 uint64_t off, uint32_t q, cudaStream_t st) {
  if (!n) return cudaSuccess;
  gen_bernoulli_kernel<<<gen_grid(n), 256, 0, st>>>(dst, n, seed, off, q);
  return cudaGetLastError();
}
cudaError_t launch_gen_blocks(uint64_t *dst, unsigned long long n, uint64_t seed,
                              uint64_t off, uint64_t block_bytes, cudaStream_t st) {
  if (!n) return cudaSuccess;
  gen_blocks_kernel<<<gen_grid(n), 256, 0, st>>>(dst, n, seed, off, block_bytes);
  return cudaGetLastError();
}
cudaError_t launch_gen_onehot32(uint32_t *dst, unsigned long long n, uint64_t seed,
                                uint64_t off, const uint32_t *thr31, cudaStream_t st) {
  if (!n) return cudaSuccess;
  Thr31 t;
  for (int k = 0; k < 31; ++k) t.t[k] = thr31[k];
  gen_onehot32_kernel<<<gen_grid(n), 256, 0, st>>>(dst, n, seed, off, t);
  return cudaGetLastError();
}

cudaError_t launch_gen_codes8(uint8_t *dst, unsigned long long n, uint64_t seed, uint64_t off,
                              const uint32_t *thr31, cudaStream_t st) {
  if (!n) return cudaSuccess;
  Thr31 t;
  for (int k = 0; k < 31; ++k) t.t[k] = thr31[k];
  gen_codes8_kernel<<<gen_grid(n), 256, 0, st>>>(dst, n, seed, off, t);
  return cudaGetLastError();
}

}  // namespace pp
