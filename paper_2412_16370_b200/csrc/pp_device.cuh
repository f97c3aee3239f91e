// pp_device.cuh — device building blocks of the sm_100a positional popcount.
//
// The reference (pure Python, /root/reference/pkg) counts with the paper's
// Harley-Seal scheme over r-bit vectors: full adders (csa.py:16-23), a
// 16-input carry-save network that skims a weight-16 plane (csa.py:63-87),
// a split-and-fold of that plane into 16-bit counters (accumulate.py:70-75)
// and a final nibble transpose of the leftover 4-bit accumulators
// (accumulate.py:78-107).  On B200 the same arithmetic is re-expressed per
// thread over 32-bit lanes:
//   * full adder            -> two LOP3 (0x96 parity, 0xE8 majority)
//   * CSA16+4 per lane       -> 15 full adders per 16 words (same wiring)
//   * second CSA level       -> a 4-bit bit-sliced counter of a16 planes
//   * split-and-fold         -> a 32x32 warp bit-matrix transpose
//                               (SHFL + PRMT/SHF/LOP3) so lane j owns bit
//                               position j, then __popc
//   * 16-bit counter flushes -> exact u64 per-lane counters (no headroom rule)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pp {

constexpr unsigned FULL = 0xffffffffu;

// ---- checked builds (PP_CHECK_BOUNDS=1; build.build_checked()) -------------
// The reference's contract is that no byte outside the caller's buffer is
// read (edges.py:1-10, pkg/tests/test_kernels.py:83-91).  A checked build
// tests, before it happens, every global load and bulk-copy source range
// against the caller's range (CountArgs/SegArgs chk_lo/chk_hi, set by the
// host API from the caller's own pointer and length before any split), every
// shared-memory stage index, every chunk id a consumer sees (in range and,
// per CTA, strictly increasing) and, at the end of each counting grid, that
// the chunks consumed add up to exactly the chunks of the launch (a skipped
// or repeated mbarrier phase breaks that).  A failed check skips the access
// (nothing out of range is ever touched) and is recorded in this translation
// unit's ChkRec, read back by pp_check_status().  No __trap(): a recorded
// failure leaves the context usable.  Unchecked builds compile all of it out.
#ifndef PP_CHECK_BOUNDS
#define PP_CHECK_BOUNDS 0
#endif
struct ChkRec {
  unsigned int fails;       // failed checks since the last reset
  unsigned int first_line;  // source line of the first one
  unsigned long long first_addr, first_lo, first_hi;  // its address and allowed range
};
#if PP_CHECK_BOUNDS
static __device__ ChkRec pp_chk;  // one per translation unit (no -rdc)
static __device__ __noinline__ void chk_fail(int line, unsigned long long addr, unsigned long long lo,
                                      unsigned long long hi) {
  if (atomicAdd(&pp_chk.fails, 1u) == 0u) {
    pp_chk.first_line = (unsigned)line;
    pp_chk.first_addr = addr;
    pp_chk.first_lo = lo;
    pp_chk.first_hi = hi;
  }
}
#define PP_CHK_RANGE(p, n, lo, hi) \
  ::pp::chk_range(reinterpret_cast<uintptr_t>(p), (unsigned long long)(n), (lo), (hi), __LINE__)
#define PP_CHK(cond) ((cond) ? true : (::pp::chk_fail(__LINE__, 0ull, 0ull, 0ull), false))
static __device__ __forceinline__ bool chk_range(uintptr_t a, unsigned long long n, uintptr_t lo,
                                          uintptr_t hi, int line) {
  if (a >= lo && a + n >= a && a + n <= hi) return true;
  chk_fail(line, a, lo, hi);
  return false;
}
#else
#define PP_CHK_RANGE(p, n, lo, hi) true
#define PP_CHK(cond) true
#endif

__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Positionwise full adder: carry = majority, sum = parity (csa.py:16-23).
#define PP_FA(carry, sum, a, b, c)        \
  do {                                    \
    uint32_t _a = (a), _b = (b), _c = (c); \
    sum = xor3(_a, _b, _c);               \
    carry = maj3(_a, _b, _c);             \
  } while (0)

// Four bit planes forming a 4-bit counter per bit position (csa.py:26-32).
struct Planes {
  uint32_t p1, p2, p4, p8;
};

// 16 equal-weight words + the 4-bit accumulator -> (a16, accumulator').
// Wiring of csa.py:63-87 / _nbkern.py:101-115: exactly 15 full adders,
// 16*a16 + val(acc') == val(acc) + popcount(v) per position.
__device__ __forceinline__ uint32_t csa16_4(Planes &acc, const uint32_t (&v)[16]) {
  uint32_t c1, s1, c2, s2, c3, s3, c4, s4, c5, s5;
  PP_FA(c1, s1, v[0], v[1], v[2]);
  PP_FA(c2, s2, v[3], v[4], v[5]);
  PP_FA(c3, s3, v[6], v[7], v[8]);
  PP_FA(c4, s4, v[9], v[10], v[11]);
  PP_FA(c5, s5, v[12], v[13], v[14]);
  uint32_t d1, t1, d2, t2, d3, e1, u1, e2, u2, e3, u3, e4, f1, x1, f2, a16;
  PP_FA(d1, t1, s1, s2, s3);
  PP_FA(d2, t2, s4, s5, v[15]);
  PP_FA(d3, acc.p1, t1, t2, acc.p1);
  PP_FA(e1, u1, c1, c2, c3);
  PP_FA(e2, u2, c4, c5, d1);
  PP_FA(e3, u3, d2, d3, acc.p2);
  PP_FA(e4, acc.p2, u1, u2, u3);
  PP_FA(f1, x1, e1, e2, e3);
  PP_FA(f2, acc.p4, x1, e4, acc.p4);
  PP_FA(a16, acc.p8, f1, f2, acc.p8);
  return a16;
}

// Ripple-increment a 4-bit bit-sliced counter by the plane x (caller keeps
// the count <= 15, so no carry leaves p8).  Second Harley-Seal level.
__device__ __forceinline__ void inc4(Planes &b, uint32_t x) {
  uint32_t c1 = b.p1 & x;
  b.p1 ^= x;
  uint32_t c2 = b.p2 & c1;
  b.p2 ^= c1;
  uint32_t c3 = b.p4 & c2;
  b.p4 ^= c2;
  b.p8 ^= c3;
}

// Per-lane constants of the warp transpose (see wtranspose).
struct TC {
  uint32_t sel16, sel8;
  uint32_t keep4, keep2, keep1;
  uint32_t rot4, rot2, rot1;
};

__device__ __forceinline__ TC make_tc(uint32_t lane) {
  TC t;
  t.sel16 = (lane & 16) ? 0x3276u : 0x5410u;
  t.sel8 = (lane & 8) ? 0x3715u : 0x6240u;
  t.keep4 = (lane & 4) ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
  t.keep2 = (lane & 2) ? 0xCCCCCCCCu : 0x33333333u;
  t.keep1 = (lane & 1) ? 0xAAAAAAAAu : 0x55555555u;
  t.rot4 = (lane & 4) ? 4u : 28u;
  t.rot2 = (lane & 2) ? 2u : 30u;
  t.rot1 = (lane & 1) ? 1u : 31u;
  return t;
}

// 32x32 bit-matrix transpose across the warp: on return, bit i of lane L's
// word equals bit L of lane i's input word.  So __popc of the result is the
// number of lanes whose input has bit L set: the positional count of bit L
// over the warp.  5 SHFL + 2 PRMT + 3 SHF + 3 LOP3 per lane.
// (Plays the role of the reference's split-and-fold, accumulate.py:37-75.)
__device__ __forceinline__ uint32_t wtranspose(uint32_t x, const TC &t) {
  uint32_t y = __shfl_xor_sync(FULL, x, 16);
  x = __byte_perm(x, y, t.sel16);
  y = __shfl_xor_sync(FULL, x, 8);
  x = __byte_perm(x, y, t.sel8);
  y = __shfl_xor_sync(FULL, x, 4);
  y = __funnelshift_r(y, y, t.rot4);
  x = (x & t.keep4) | (y & ~t.keep4);
  y = __shfl_xor_sync(FULL, x, 2);
  y = __funnelshift_r(y, y, t.rot2);
  x = (x & t.keep2) | (y & ~t.keep2);
  y = __shfl_xor_sync(FULL, x, 1);
  y = __funnelshift_r(y, y, t.rot1);
  x = (x & t.keep1) | (y & ~t.keep1);
  return x;
}

__device__ __forceinline__ uint32_t wcount(uint32_t plane, const TC &t) {
  return __popc(wtranspose(plane, t));
}

// Lane L's positional count (over the warp) of a weighted 4-plane counter.
__device__ __forceinline__ uint32_t wcount_planes(const Planes &p, uint32_t shift,
                                                  const TC &t) {
  uint32_t s = wcount(p.p1, t) + (wcount(p.p2, t) << 1) + (wcount(p.p4, t) << 2) +
               (wcount(p.p8, t) << 3);
  return s << shift;
}

// Per-thread two-level Harley-Seal state for one 64-bit frame:
// "e" = frame bits 0..31 (u32 lanes at address = 0 mod 8),
// "o" = frame bits 32..63 (u32 lanes at address = 4 mod 8).
struct Counter {
  Planes l1e, l1o;  // weights 1,2,4,8
  Planes l2e, l2o;  // weights 16,32,64,128
  uint32_t l2n;     // a16 increments held in l2 (<= 15)
  unsigned long long ce, co;  // lane-owned exact counts: frame bit lane / 32+lane

  __device__ __forceinline__ void init() {
    l1e = l1o = l2e = l2o = Planes{0u, 0u, 0u, 0u};
    l2n = 0;
    ce = co = 0ull;
  }

  // Eat 8 16-byte vectors (all lanes of the warp call this in lockstep).
  __device__ __forceinline__ void eat8(const uint4 (&v)[8], const TC &t) {
    uint32_t ev[16], od[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      ev[2 * i] = v[i].x;
      ev[2 * i + 1] = v[i].z;
      od[2 * i] = v[i].y;
      od[2 * i + 1] = v[i].w;
    }
    uint32_t a16e = csa16_4(l1e, ev);
    uint32_t a16o = csa16_4(l1o, od);
    inc4(l2e, a16e);
    inc4(l2o, a16o);
    if (++l2n == 15) flush_l2(t);
  }

  // l2n is warp-uniform, so the plane skipping below never diverges.
  __device__ __forceinline__ void flush_l2(const TC &t) {
    if (l2n >= 8) {
      ce += wcount_planes(l2e, 4, t);
      co += wcount_planes(l2o, 4, t);
    } else {
      uint32_t se = wcount(l2e.p1, t), so = wcount(l2o.p1, t);
      if (l2n >= 2) {
        se += wcount(l2e.p2, t) << 1;
        so += wcount(l2o.p2, t) << 1;
      }
      if (l2n >= 4) {
        se += wcount(l2e.p4, t) << 2;
        so += wcount(l2o.p4, t) << 2;
      }
      ce += se << 4;
      co += so << 4;
    }
    l2e = l2o = Planes{0u, 0u, 0u, 0u};
    l2n = 0;
  }

  // Fold everything still held in planes into ce/co (warp-collective).
  __device__ __forceinline__ void finish(const TC &t) {
    ce += wcount_planes(l1e, 0, t);
    co += wcount_planes(l1o, 0, t);
    if (l2n) flush_l2(t);
    l1e = l1o = Planes{0u, 0u, 0u, 0u};
  }
};

// Chunk-batched counter of the fused one-hot producer.  One chunk of a
// thread (8 vectors of codes) expands into a STATIC number of eat8 groups
// (W / 8 for u8 codes), so the a16 planes of a whole chunk are known at
// compile time and are combined by a static Harley-Seal tree (M - 1 full
// adders into persistent planes of weight 16, 32, ...) before ONE ripple
// increment of the second-level counter -- instead of an increment per
// group (7 ops each) and a second-level count every 15 groups.  NT = 1:
// both u32 lanes of a frame word count the same W <= 32 positions (the fold
// sums frame[j] and frame[j + 32]), so every word goes through one tree;
// NT = 2 (W = 64): e = frame bits 0..31, o = 32..63, as Counter.
// (The paper's own scheme, csa.py:63-87, applied a second time.)
template <int NT, int M>
struct CatCounter {
  static_assert(NT == 1 || NT == 2, "trees");
  static_assert(M == 1 || M == 2 || M == 4 || M == 8 || M == 16, "a16 planes per chunk");
  static constexpr int kLog = M >= 16 ? 4 : M >= 8 ? 3 : M >= 4 ? 2 : M >= 2 ? 1 : 0;
  Planes l1[NT];           // weights 1, 2, 4, 8
  uint32_t h[NT][kLog > 0 ? kLog : 1];     // weights 16 << k
  uint32_t slot[NT][kLog > 0 ? kLog : 1];  // a plane waiting for its pair, level k
  Planes l2[NT];           // weights 16 M << (0..3)
  uint32_t l2n;            // chunks held in l2 (<= 15; warp-uniform)
  unsigned long long ce, co;

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      l1[r] = l2[r] = Planes{0u, 0u, 0u, 0u};
#pragma unroll
      for (int k = 0; k < (kLog > 0 ? kLog : 1); ++k) h[r][k] = 0u;
    }
    l2n = 0u;
    ce = co = 0ull;
  }
  // The idx-th a16 plane of the chunk (idx static): a binary counter over
  // idx with a full adder per trailing one, resolved at compile time, so at
  // most log2(M) planes wait at any time; the last one (idx = M - 1) leaves
  // the chunk's single carry of weight 16 M for the ripple increment.
  __device__ __forceinline__ void put(int r, int idx, uint32_t x) {
#pragma unroll
    for (int k = 0; k < kLog; ++k) {
      if (!((idx >> k) & 1)) {
        slot[r][k] = x;
        return;
      }
      PP_FA(x, h[r][k], h[r][k], slot[r][k], x);
    }
    inc4(l2[r], x);
  }
  // Group g of the chunk (static): 32 words, two csa16_4
  __device__ __forceinline__ void csa(const uint4 (&v)[8], int g) {
    uint32_t x[16], y[16];
    if (NT == 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[4 * i] = v[i].x;
        x[4 * i + 1] = v[i].y;
        x[4 * i + 2] = v[i].z;
        x[4 * i + 3] = v[i].w;
        y[4 * i] = v[4 + i].x;
        y[4 * i + 1] = v[4 + i].y;
        y[4 * i + 2] = v[4 + i].z;
        y[4 * i + 3] = v[4 + i].w;
      }
      put(0, 2 * g, csa16_4(l1[0], x));
      put(0, 2 * g + 1, csa16_4(l1[0], y));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[2 * i] = v[i].x;
        x[2 * i + 1] = v[i].z;
        y[2 * i] = v[i].y;
        y[2 * i + 1] = v[i].w;
      }
      put(0, g, csa16_4(l1[0], x));
      put(NT - 1, g, csa16_4(l1[NT - 1], y));
    }
  }
  // after the chunk's last group
  __device__ __forceinline__ void end_chunk(const TC &t) {
    if (++l2n == 15u) flush_l2(t);
  }
  __device__ __forceinline__ void flush_l2(const TC &t) {
    ce += (unsigned long long)wcount_planes(l2[0], 0, t) << (4 + kLog);
    if (NT == 2) co += (unsigned long long)wcount_planes(l2[NT - 1], 0, t) << (4 + kLog);
#pragma unroll
    for (int r = 0; r < NT; ++r) l2[r] = Planes{0u, 0u, 0u, 0u};
    l2n = 0u;
  }
  __device__ __forceinline__ void finish(const TC &t) {
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      unsigned long long s = wcount_planes(l1[r], 0, t);
#pragma unroll
      for (int k = 0; k < kLog; ++k) s += (unsigned long long)wcount(h[r][k], t) << (4 + k);
      if (r == 0) ce += s; else co += s;
      l1[r] = Planes{0u, 0u, 0u, 0u};
#pragma unroll
      for (int k = 0; k < (kLog > 0 ? kLog : 1); ++k) h[r][k] = 0u;
    }
    if (l2n) flush_l2(t);
  }
};

// Segment-parallel variant: G lanes share one segment, so a warp carries
// S = 32/G independent segments.  Each transpose stage swaps one bit of the
// lane index with the same bit of the bit index, and the stages commute, so
// running only the stages j < G transposes inside each G-lane group: lane r
// of a group then holds, in G-bit field f, the group's bits of position
// G*f + r, and one masked __popc per field gives its segment's count.
template <int G>
__device__ __forceinline__ uint32_t gtranspose(uint32_t x, const TC &t) {
  uint32_t y;
  if (G > 16) {
    y = __shfl_xor_sync(FULL, x, 16);
    x = __byte_perm(x, y, t.sel16);
  }
  if (G > 8) {
    y = __shfl_xor_sync(FULL, x, 8);
    x = __byte_perm(x, y, t.sel8);
  }
  if (G > 4) {
    y = __shfl_xor_sync(FULL, x, 4);
    y = __funnelshift_r(y, y, t.rot4);
    x = (x & t.keep4) | (y & ~t.keep4);
  }
  if (G > 2) {
    y = __shfl_xor_sync(FULL, x, 2);
    y = __funnelshift_r(y, y, t.rot2);
    x = (x & t.keep2) | (y & ~t.keep2);
  }
  y = __shfl_xor_sync(FULL, x, 1);
  y = __funnelshift_r(y, y, t.rot1);
  x = (x & t.keep1) | (y & ~t.keep1);
  return x;
}

// SMEM = true keeps the 2S exact u64 counts of each lane in shared memory
// (slot i of lane l at sc[i*32 + l], conflict-free): they are touched only
// when planes are flushed, and dropping them from registers lets 32 warps
// per SM stay resident (more loads in flight).
template <int G, bool SMEM = false>
struct GroupCounter {
  static_assert(G == 2 || G == 4 || G == 8 || G == 16 || G == 32, "lanes per segment");
  static constexpr int S = 32 / G;  // positions per lane per tree
  Planes l1e, l1o, l2e, l2o;
  uint32_t l2n;
  // lane r of a segment's group: frame bits G*f + r (e) and 32 + G*f + r (o)
  unsigned long long ce[SMEM ? 1 : S], co[SMEM ? 1 : S];
  unsigned long long *sc;  // SMEM: this lane's slot 0 (stride 32)

  __device__ __forceinline__ void init(unsigned long long *slots = nullptr) {
    l1e = l1o = l2e = l2o = Planes{0u, 0u, 0u, 0u};
    l2n = 0;
    sc = slots;
#pragma unroll
    for (int f = 0; f < S; ++f) {
      if (SMEM) {
        sc[f * 32] = 0ull;
        sc[(S + f) * 32] = 0ull;
      } else {
        ce[f] = co[f] = 0ull;
      }
    }
  }
  __device__ __forceinline__ unsigned long long e(int f) const { return SMEM ? sc[f * 32] : ce[f]; }
  __device__ __forceinline__ unsigned long long o(int f) const {
    return SMEM ? sc[(S + f) * 32] : co[f];
  }

  static __device__ __forceinline__ uint32_t field_popc(uint32_t x, int f) {
    if (G == 32) return __popc(x);
    return __popc(x & (((1u << G) - 1u) << (f * G)));
  }

  // Count the first np planes (weights 1,2,4,8 << shift) of both trees.
  __device__ __forceinline__ void count_planes(const Planes &pe, const Planes &po, int np,
                                               int shift, const TC &t) {
    uint32_t se[S], so[S];
#pragma unroll
    for (int f = 0; f < S; ++f) se[f] = so[f] = 0u;
    const uint32_t ve[4] = {pe.p1, pe.p2, pe.p4, pe.p8};
    const uint32_t vo[4] = {po.p1, po.p2, po.p4, po.p8};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < np) {  // np is warp-uniform
        const uint32_t te = gtranspose<G>(ve[k], t), to = gtranspose<G>(vo[k], t);
#pragma unroll
        for (int f = 0; f < S; ++f) {
          se[f] += field_popc(te, f) << k;
          so[f] += field_popc(to, f) << k;
        }
      }
    }
#pragma unroll
    for (int f = 0; f < S; ++f) {
      if (SMEM) {
        sc[f * 32] += (unsigned long long)se[f] << shift;
        sc[(S + f) * 32] += (unsigned long long)so[f] << shift;
      } else {
        ce[f] += (unsigned long long)se[f] << shift;
        co[f] += (unsigned long long)so[f] << shift;
      }
    }
  }

  __device__ __forceinline__ void eat8(const uint4 (&v)[8], const TC &t) {
    uint32_t ev[16], od[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      ev[2 * i] = v[i].x;
      ev[2 * i + 1] = v[i].z;
      od[2 * i] = v[i].y;
      od[2 * i + 1] = v[i].w;
    }
    inc4(l2e, csa16_4(l1e, ev));
    inc4(l2o, csa16_4(l1o, od));
    if (++l2n == 15) {
      count_planes(l2e, l2o, 4, 4, t);
      l2e = l2o = Planes{0u, 0u, 0u, 0u};
      l2n = 0;
    }
  }

  __device__ __forceinline__ void finish(const TC &t) {
    count_planes(l1e, l1o, 4, 0, t);
    if (l2n) count_planes(l2e, l2o, l2n >= 8 ? 4 : l2n >= 4 ? 3 : l2n >= 2 ? 2 : 1, 4, t);
  }
};

// Frame position (mod 64) of bit 0 of the byte at address a.
__device__ __forceinline__ uint32_t frame_shift(const void *a) {
  return 8u * (uint32_t)(reinterpret_cast<uintptr_t>(a) & 7u);
}

// Streaming 16-byte global load that bypasses L1 allocation.
// Streamed loads: no L1 allocation, and (PP_LDG_EVICT_FIRST) an L2
// evict-first cache policy, so bytes streamed once do not displace lines
// still in use (counter rows, offsets, neighbouring segments' edges): ragged
// 0-8 KiB CSR 209.9 -> 192.0 us per GiB, misaligned 1 KiB arrays 449 -> 437
// (profiles/r1_segmented_ablation.md).  The createpolicy is volatile and
// per load: a pure one let ptxas drop the hint (measured: no gain), the
// volatile asm alone without the hint gains nothing either.
#ifndef PP_LDG_EVICT_FIRST
#define PP_LDG_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
#if PP_LDG_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
#endif
  return r;
}

// ---- mbarrier / bulk-copy (TMA) primitives --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "PP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PP_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// One-dimensional bulk copy global -> shared (SASS: UBLKCP), completion
// counted in bytes on the stage's mbarrier.
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes,
                                         uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

}  // namespace pp
