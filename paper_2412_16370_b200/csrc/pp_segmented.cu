// pp_segmented.cu — many independent arrays in one launch:
// row s of the output = the reference's count of segment s alone
// (NumbaKernel.run on InputView(base, off[s], len_s), kernels.py:242-270).
//
//   pp_seg_kernel<G>      G = 8/16/32 lanes per segment, LDG-fed, warp
//                         transposes restricted to the G-lane group.
//   pp_segtma_kernel<G>   fixed-size segments through a CTA-wide TMA ring.
//   pp_seglane_kernel     one lane per tiny array, SWAR counts.
#include <cstdlib>
#include <cstring>

#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

constexpr int kSegThreads = 256;
// Groups of S = 32/G segments per scheduler ticket in pp_seg_kernel.  Every
// ticket is one atomic on the stream's single counter, and same-address
// atomics serialise at ~2-3 ns each: 262,144 tickets (1 GiB of 4 KiB
// segments at G = 32, one segment per ticket) took 592 instead of 200 us.
// Below ~50k tickets per launch the finest batches balance ragged lengths
// best (scripts/seg_shape_sweep.py, profiles/r1_segmented_ablation.md), so
// the batch is the smallest T that keeps the launch under kSegMaxTickets.
constexpr unsigned long long kSegMaxTickets = 49152;
constexpr unsigned kSegMaxBatchGroups = 63;
static unsigned seg_batch_groups(unsigned long long nseg, int G) {
  const unsigned long long groups = (nseg + (32 / G) - 1) / (32 / G);
  unsigned long long t = (groups + kSegMaxTickets - 1) / kSegMaxTickets;
  if (t < 1) t = 1;
  if (t > kSegMaxBatchGroups) t = kSegMaxBatchGroups;
  return (unsigned)t;
}
static unsigned long long seg_batches(unsigned long long nseg, int G, unsigned T) {
  const unsigned long long per = (unsigned long long)(32 / G) * T;
  return (nseg + per - 1) / per;
}
#ifndef PP_SEG_SMEM_COUNTS
#define PP_SEG_SMEM_COUNTS true
#endif
#ifndef PP_SEG_MIN_BLOCKS
#define PP_SEG_MIN_BLOCKS 3  // <= 85 registers: 24 warps/SM of loads in flight
#endif

// Bytes [max(va, lo), min(va + 16, hi)) of the aligned 16-byte block at va,
// zero elsewhere: the masked head / tail vector of a segment.  Exact-bounds
// byte loads, so nothing outside the segment is ever read.
__device__ __noinline__ uint4 load_partial(uintptr_t va, uintptr_t lo, uintptr_t hi,
                                           uintptr_t chk_lo = 0, uintptr_t chk_hi = 0) {
  uint32_t q[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const uintptr_t ad = va + b;
    if (ad >= lo && ad < hi && PP_CHK_RANGE(ad, 1, chk_lo, chk_hi))
      q[b >> 2] |= (uint32_t)__ldg(reinterpret_cast<const uint8_t *>(ad)) << (8 * (b & 3));
  }
  return make_uint4(q[0], q[1], q[2], q[3]);
}

// Geometry of segment s as "virtual vectors": the aligned 16-byte blocks
// covering [p0, e).  Only vector 0 (head) and vector nvv-1 (tail) can be
// partial; they are read with exact-bounds byte loads (load_partial).
struct SegGeom {
  uintptr_t p0, e, A;
  unsigned long long nvv;
  bool hp, tp;
};

__device__ __forceinline__ SegGeom seg_geom(const SegArgs &a, unsigned long long s) {
  unsigned long long s0 = 0, s1 = 0;
  uintptr_t origin = reinterpret_cast<uintptr_t>(a.base);
  if (s < a.nseg) {
    if (a.ptrs) {  // pointer mode: absolute address + length
      origin = 0;
      s0 = a.ptrs[s];
      s1 = s0 + a.lens[s];
    } else if (a.seg_off) {
      s0 = a.seg_off[s];
      s1 = a.seg_off[s + 1];
      if (s1 < s0) s1 = s0;
    } else {
      s0 = s * a.seg_bytes;
      s1 = s0 + a.seg_bytes;
    }
  }
  SegGeom g;
  g.p0 = origin + s0;
  g.e = g.p0 + (s1 - s0);
  g.A = g.p0 & ~(uintptr_t)15;
  g.nvv = (s1 > s0) ? (((g.e + 15) & ~(uintptr_t)15) - g.A) >> 4 : 0;
  g.hp = (g.p0 & 15) != 0;
  g.tp = (g.e & 15) != 0;
  return g;
}

__device__ __forceinline__ bool seg_partial(const SegGeom &g, unsigned long long k) {
  return (k == 0 && g.hp) || (k == g.nvv - 1 && g.tp);
}

// 0xFF in bytes [lo, hi) of a u32 holding bytes 4q..4q+3 of a vector
__device__ __forceinline__ uint32_t byte_range_mask(int q, int lo, int hi) {
  const int a = min(max(lo - 4 * q, 0), 4), b = min(max(4 * q + 4 - hi, 0), 4);
  uint32_t m1, m2;
  asm("shl.b32 %0, %1, %2;" : "=r"(m1) : "r"(0xFFFFFFFFu), "r"(8 * a));  // 32 -> 0
  asm("shr.b32 %0, %1, %2;" : "=r"(m2) : "r"(0xFFFFFFFFu), "r"(8 * b));
  return m1 & m2;
}

// A segment's partial head/tail vector: when the whole aligned 16 bytes lie
// inside the caller's view (they then belong to neighbouring segments),
// one vector load and a byte mask; else exact-bounds byte loads.
__device__ __noinline__ uint4 load_edge(uintptr_t va, uintptr_t p0, uintptr_t e,
                                           uintptr_t view_lo, uintptr_t view_hi,
                                           uintptr_t chk_lo = 0, uintptr_t chk_hi = 0) {
  if (va >= view_lo && va + 16 <= view_hi) {
    if (!PP_CHK_RANGE(va, 16, chk_lo, chk_hi)) return make_uint4(0u, 0u, 0u, 0u);
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(va));
    const int lo = va < p0 ? (int)(p0 - va) : 0;
    const int hi = va + 16 > e ? (int)(e - va) : 16;
    v.x &= byte_range_mask(0, lo, hi);
    v.y &= byte_range_mask(1, lo, hi);
    v.z &= byte_range_mask(2, lo, hi);
    v.w &= byte_range_mask(3, lo, hi);
    return v;
  }
  return load_partial(va, p0, e, chk_lo, chk_hi);
}

#ifndef PP_ROW_STREAM
#define PP_ROW_STREAM 1
#endif
#ifndef PP_ROW_STREAM_MAXG
#define PP_ROW_STREAM_MAXG 16
#endif
// *d = v (overwrite) or *d += v (accumulate).  STREAM: an evict-first
// store (st.global.cs) -- the rows are not read back by the kernel.  Used
// for G <= 16, where a store instruction carries pieces of several rows:
// C4 batch 177.1 -> 173.5 us, misaligned 1 KiB arrays 473 -> 449, ragged
// 0-8 KiB 221 -> 210, misaligned 8 KiB 191 -> 185; with one row per warp
// (G = 32, 16 KiB segments) it measured up to 5 % slower, so plain stores.
template <bool STREAM>
__device__ __forceinline__ void put_count(unsigned long long *d, unsigned long long v, bool ow) {
  if (ow) {
    if (STREAM)
      __stcs(d, v);
    else
      *d = v;
  } else {
    *d += v;
  }
}

// Row s of out <- the counts lane r of the segment's G-lane group holds
// (frame bits G*f + r and 32 + G*f + r), rotated by rot = 8*(p0 mod 8) and
// folded mod w exactly like flush_fw (accumulate.py:115-130).  All G lanes of
// the group call this together (they share s).
template <int G, bool SM>
__device__ __forceinline__ void write_row(const SegArgs &a, unsigned long long s,
                                          uintptr_t p0, const GroupCounter<G, SM> &c,
                                          uint32_t lane) {
  constexpr int S = 32 / G;
  constexpr bool kStream = PP_ROW_STREAM && G <= PP_ROW_STREAM_MAXG;
  const int w = a.width;
  const int r = (int)(lane % G);
  const int rot = (int)(8u * (uint32_t)(p0 & 7u));
  unsigned long long *row = a.out + s * (unsigned long long)w;
  const bool ow = a.overwrite != 0;
  if (w == 64) {
#pragma unroll
    for (int f = 0; f < S; ++f) {
      const int pe = G * f + r;
      unsigned long long *de = row + ((pe - rot) & 63), *dd = row + ((pe + 32 - rot) & 63);
      put_count<kStream>(de, c.e(f), ow);
      put_count<kStream>(dd, c.o(f), ow);
    }
  } else if (G <= w) {
    // lane r's positions G*f + r fall in w/G classes mod w; class of f is f % nc
    const int nc = w / G;
#pragma unroll
    for (int cc = 0; cc < S; ++cc) {
      if (cc < nc) {
        unsigned long long tot = 0ull;
#pragma unroll
        for (int f = cc; f < S; ++f)
          if (f % nc == cc) tot += c.e(f) + c.o(f);
        unsigned long long *d = row + ((G * cc + r - rot) & (w - 1));
        put_count<kStream>(d, tot, ow);
      }
    }
  } else {
    // G > w: all of lane r's positions are = r (mod w); lanes r, r^w, ... of
    // the group share a class.
    unsigned long long tot = 0ull;
#pragma unroll
    for (int f = 0; f < S; ++f) tot += c.e(f) + c.o(f);
    const unsigned gmask =
        (G == 32) ? FULL : (((1u << G) - 1u) << (lane & ~(uint32_t)(G - 1)));
    for (int m = w; m < G; m <<= 1) tot += __shfl_xor_sync(gmask, tot, m);
    if (r < w) {
      unsigned long long *d = row + ((r - rot) & (w - 1));
      put_count<kStream>(d, tot, ow);
    }
  }
}

// Segmented count fed by LDG, G lanes per segment (S = 32/G segments per
// warp), grid-stride over groups of S segments.  Lane r of a segment eats
// vectors r, r+G, ... in groups of 8 (G x 16 contiguous bytes per load
// instruction per segment).  A TMA-fed variant (per-warp bulk-copy rings) was
// 1.5x slower here: profiles/r1_segmented_ablation.md.
template <int G, bool HYBRID = false>
__global__ void __launch_bounds__(kSegThreads, PP_SEG_MIN_BLOCKS)
    pp_seg_kernel(SegArgs a) {
  constexpr int S = 32 / G;
  __shared__ unsigned long long slots[(kSegThreads / 32) * 2 * S * 32];
  const uint32_t lane = threadIdx.x & 31, r = lane % G, sl = lane / G;
  const unsigned long long gw = (blockIdx.x * (unsigned long long)kSegThreads + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)kSegThreads) >> 5;
  const TC t = make_tc(lane);
  // the caller's view (pointer mode: none -- every array is its own view)
  const uintptr_t base_u = reinterpret_cast<uintptr_t>(a.base);
  const uintptr_t view_lo = a.ptrs ? 0 : base_u + (a.seg_off ? a.seg_off[0] : 0ull);
  const uintptr_t view_hi =
      a.ptrs ? 0 : base_u + (a.seg_off ? a.seg_off[a.nseg] : a.nseg * a.seg_bytes);
  // checked builds: the caller's range (host-given for fixed segments,
  // else this view; pointer mode: per array, below)
  const uintptr_t chk_lo = a.chk_hi ? a.chk_lo : view_lo;
  const uintptr_t chk_hi = a.chk_hi ? a.chk_hi : view_hi;
  // group gw first, then (a.sched) tickets of the stream's scheduler slot,
  // one per group of S segments (group nw + ticket), else the grid stride:
  // ragged lengths no longer leave a few warps with most of the bytes
  // work comes in batches of T groups: batch gw first, then (a.sched) one
  // ticket of the stream's counter per batch (batch nw + ticket), else the
  // grid stride -- ragged lengths no longer leave a few warps with most of
  // the bytes.  T groups per ticket (seg_batch_groups: as few as keep the
  // single counter from serialising; one group whenever possible -- a batch
  // of 8 long segments on one warp starved the others: 1023 x 64 KiB took
  // 117 instead of 21 us)
  const unsigned T = a.batch_groups;
  for (unsigned long long batch = gw;;) {
    if (batch * T * S >= a.nseg) break;
    for (unsigned tg = 0; tg < T; ++tg) {
      const unsigned long long first = (batch * T + tg) * S;
      if (first >= a.nseg) break;
      const unsigned long long slot = first + sl;
      // the segment this slot counts (caller-given order, else the slot)
      const unsigned long long s = (a.order && slot < a.nseg) ? a.order[slot] : slot;
      SegGeom g = seg_geom(a, s);
      bool mine = slot < a.nseg && s < a.nseg;  // (an out-of-range order entry writes nothing)
      if (HYBRID) {  // short segments belong to the one-lane kernel
        mine = mine && g.e - g.p0 > a.short_max;
        if (!mine) g.nvv = 0;
        if (!__any_sync(FULL, mine)) continue;  // the whole group is short
      }
      GroupCounter<G, PP_SEG_SMEM_COUNTS> c;
      c.init(slots + (threadIdx.x >> 5) * (2 * S * 32) + lane);
      // full (aligned, in-range) vectors are [kf0, kf1)
      const unsigned long long kf0 = g.hp ? 1 : 0;
      const unsigned long long kf1 = (g.tp && g.nvv) ? g.nvv - 1 : g.nvv;
      const uint4 *vp = reinterpret_cast<const uint4 *>(g.A) + r;
      // checked builds: whole vectors must lie inside the segment itself,
      // edge vectors inside the caller's range
      const uintptr_t clo = a.ptrs ? g.p0 : chk_lo, chi = a.ptrs ? g.e : chk_hi;
      auto load_round = [&](unsigned long long k0, uint4 (&v)[8]) {
        if (k0 + r >= kf0 && k0 + r + 7 * G < kf1) {
          // fast path: 8 full vectors, base pointer + immediate offsets
#pragma unroll
          for (int j = 0; j < 8; ++j)
            v[j] = PP_CHK_RANGE(vp + k0 + j * G, 16, g.p0, g.e) &&
                           PP_CHK_RANGE(vp + k0 + j * G, 16, clo, chi)
                       ? ldg_stream(vp + k0 + j * G)
                       : make_uint4(0u, 0u, 0u, 0u);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const unsigned long long k = k0 + j * G + r;
            v[j] = make_uint4(0u, 0u, 0u, 0u);
            if (k < g.nvv) {
              const uintptr_t va = g.A + 16 * k;
              if (seg_partial(g, k))
                v[j] = load_edge(va, g.p0, g.e, view_lo, view_hi, clo, chi);
              else if (PP_CHK_RANGE(va, 16, g.p0, g.e) && PP_CHK_RANGE(va, 16, clo, chi))
                v[j] = ldg_stream(reinterpret_cast<const uint4 *>(va));
            }
          }
        }
      };
      // (a software-pipelined variant that keeps the next round in flight was
      // no faster: profiles/r1_segmented_ablation.md)
      for (unsigned long long k0 = 0; __any_sync(FULL, k0 < g.nvv); k0 += 8 * G) {
        uint4 v[8];
        load_round(k0, v);
        c.eat8(v, t);
      }
      c.finish(t);
      if (mine && PP_CHK(s < a.nseg)) write_row(a, s, g.p0, c, lane);
    }
    if (a.sched) {
      unsigned long long tk = 0;
      if (lane == 0) tk = (unsigned int)(atomicAdd(a.sched, 1u) - a.sched_base);
      batch = nw + __shfl_sync(FULL, tk, 0);
    } else {
      batch += nw;
    }
  }
}

// ---- one lane per segment (tiny arrays) ------------------------------------
// For arrays of a few words the G-lane kernels spend most of their time in
// the per-segment flush (warp transposes).  Here each lane owns one segment
// and counts it with SWAR adds, no cross-lane work at all: the aligned
// 16-byte vectors covering [p0, e) are masked to the segment, and for
// b = 0..3 the bits (x >> b) & 0x11111111 are added into nibble counters
// (nibble n of nl[b] = frame position 4n + b; nh: 32 + 4n + b).  Nibbles
// take <= 7 vectors (<= 14 per nibble), then spill into byte counters
// (bl[c] byte m = frame 8m + c), which take <= 18 nibble spills (<= 252),
// then spill into per-lane u32 counts in shared memory.  The final counts go
// to shared memory at their folded index i = (p - rot) & 63, so row j of
// the output is sum_m fr[j + m*w] (flush_fw, accumulate.py:115-130), and the
// warp writes its 32 consecutive rows with coalesced stores.
constexpr int kLaneWarps = 4;
constexpr int kLaneThreads = kLaneWarps * 32;
constexpr int kLaneStride = 33;  // fr[pos * 33 + lane]
#ifndef PP_LANE_UNROLL
#define PP_LANE_UNROLL 1  // 2 and 4 measured: no gain up to 64 words, -15 % at 1 word
#endif
constexpr int kLaneUnroll = PP_LANE_UNROLL;
// The one-lane kernel keeps L1-cached __ldg: a warp's 32 lanes read 32
// consecutive segments, strided by the segment size, so L1 sectors are
// shared between lanes; no-allocate + evict-first loads measured 1.03-1.7x
// slower (PP_LANE_LDG_STREAM=1, scripts/seg_lane_ab.py).
#ifndef PP_LANE_LDG_STREAM
#define PP_LANE_LDG_STREAM 0
#endif  // vectors loaded per step (<= 7)

template <bool FIXED, bool HYBRID = false, bool PTRS = false>
__global__ void __launch_bounds__(kLaneThreads)
    pp_seglane_kernel(SegArgs a) {
  __shared__ uint32_t frs[kLaneWarps][64 * kLaneStride];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *fr = frs[warp];
  const uintptr_t base = PTRS ? 0 : reinterpret_cast<uintptr_t>(a.base);
  // the caller's view: vectors entirely inside it are read whole, the
  // others byte by byte (nothing outside the view is ever read); in pointer
  // mode every array is its own view
  const uintptr_t view_lo = PTRS ? 0 : base + (FIXED ? 0ull : a.seg_off[0]);
  const uintptr_t view_hi =
      PTRS ? 0 : base + (FIXED ? a.nseg * a.seg_bytes : a.seg_off[a.nseg]);
  const uintptr_t chk_lo = a.chk_hi ? a.chk_lo : view_lo;  // checked builds
  const uintptr_t chk_hi = a.chk_hi ? a.chk_hi : view_hi;
  const unsigned long long nw = (unsigned long long)gridDim.x * kLaneWarps;
  for (unsigned long long s0 = ((unsigned long long)blockIdx.x * kLaneWarps + warp) * 32;
       s0 < a.nseg; s0 += nw * 32) {
    const unsigned long long s = s0 + lane;
    unsigned long long b0 = 0, b1 = 0;
    if (s < a.nseg) {
      if (PTRS) {
        b0 = a.ptrs[s];
        b1 = b0 + a.lens[s];
      } else if (FIXED) {
        b0 = s * a.seg_bytes;
        b1 = b0 + a.seg_bytes;
      } else {
        b0 = a.seg_off[s];
        b1 = a.seg_off[s + 1];
        if (b1 < b0) b1 = b0;
      }
    }
    // hybrid split: longer segments belong to the G-lane kernel (row
    // untouched).  A template parameter: the plain kernel must not carry this
    // test (it cost the per-vector loop ~40 % at 1 KiB segments)
    unsigned rows_mine = FULL;
    if (HYBRID) {
      const bool mine = s < a.nseg && b1 - b0 <= a.short_max;
      if (!mine) b1 = b0;
      rows_mine = __ballot_sync(FULL, mine);
    }
    const uintptr_t p0 = base + b0, e = base + b1;
    const int rot = 8 * (int)(p0 & 7u);
    uint32_t nl[4] = {0u, 0u, 0u, 0u}, nh[4] = {0u, 0u, 0u, 0u};
    uint32_t bl[8], bh[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) bl[c] = bh[c] = 0u;
    bool spilled = false;
    uint32_t nvec = 0, nnib = 0;
    auto nib_to_byte = [&]() {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        bl[b] += nl[b] & 0x0F0F0F0Fu;
        bl[b + 4] += (nl[b] >> 4) & 0x0F0F0F0Fu;
        bh[b] += nh[b] & 0x0F0F0F0Fu;
        bh[b + 4] += (nh[b] >> 4) & 0x0F0F0F0Fu;
        nl[b] = nh[b] = 0u;
      }
    };
    // counts of frame p = 8m + c (+32) -> fr at the folded index (p - rot) & 63
    auto byte_to_smem = [&](bool first) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int pl = 8 * m + c;
          uint32_t *dl = fr + ((pl - rot) & 63) * kLaneStride + lane;
          uint32_t *dh = fr + ((pl + 32 - rot) & 63) * kLaneStride + lane;
          const uint32_t vl = (bl[c] >> (8 * m)) & 0xFFu, vh = (bh[c] >> (8 * m)) & 0xFFu;
          *dl = first ? vl : *dl + vl;
          *dh = first ? vh : *dh + vh;
        }
        bl[c] = bh[c] = 0u;
      }
    };
    const uintptr_t vlo = PTRS ? p0 : view_lo, vhi = PTRS ? e : view_hi;
    const uintptr_t clo = PTRS ? p0 : chk_lo, chi = PTRS ? e : chk_hi;
    auto load_vec = [&](uintptr_t va) -> uint4 {
      uint4 v;
      if (va >= vlo && va + 16 <= vhi) {
        if (!PP_CHK_RANGE(va, 16, clo, chi)) return make_uint4(0u, 0u, 0u, 0u);
#if PP_LANE_LDG_STREAM
        v = ldg_stream(reinterpret_cast<const uint4 *>(va));
#else
        v = __ldg(reinterpret_cast<const uint4 *>(va));
#endif
        if (va < p0 || va + 16 > e) {  // mask to the segment
          const int lo = va < p0 ? (int)(p0 - va) : 0;
          const int hi = va + 16 > e ? (int)(e - va) : 16;
          v.x &= byte_range_mask(0, lo, hi);
          v.y &= byte_range_mask(1, lo, hi);
          v.z &= byte_range_mask(2, lo, hi);
          v.w &= byte_range_mask(3, lo, hi);
        }
      } else {
        v = load_partial(va, p0, e, clo, chi);
      }
      return v;
    };
    auto eat_vec = [&](const uint4 &v) {  // x, z: frame bits 0-31; y, w: 32-63
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        nl[b] += ((v.x >> b) & 0x11111111u) + ((v.z >> b) & 0x11111111u);
        nh[b] += ((v.y >> b) & 0x11111111u) + ((v.w >> b) & 0x11111111u);
      }
    };
    // a vector adds <= 2 to a nibble: at most 7 between nibble spills
    auto make_room = [&](uint32_t k) {
      if (nvec + k > 7) {
        nvec = 0;
        nib_to_byte();
        if (++nnib == 18) {
          nnib = 0;
          byte_to_smem(!spilled);
          spilled = true;
        }
      }
      nvec += k;
    };
    uintptr_t va = p0 & ~(uintptr_t)15;
    // kLaneUnroll vectors per step: their loads are in flight together
    for (; va + 16 * (kLaneUnroll - 1) < e; va += 16 * kLaneUnroll) {
      uint4 vv[kLaneUnroll];
#pragma unroll
      for (int u = 0; u < kLaneUnroll; ++u) vv[u] = load_vec(va + 16 * u);
      make_room(kLaneUnroll);
#pragma unroll
      for (int u = 0; u < kLaneUnroll; ++u) eat_vec(vv[u]);
    }
    for (; va < e; va += 16) {
      const uint4 v = load_vec(va);
      make_room(1);
      eat_vec(v);
    }
    nib_to_byte();
    byte_to_smem(!spilled);
    __syncwarp();
    // rows s0 .. s0 + nrows - 1 are contiguous in out: coalesced stores
    const int w = a.width;
    const uint32_t nrows = (uint32_t)min(32ull, a.nseg - s0);
    unsigned long long *dst = a.out + s0 * (unsigned long long)w;
    const int lw = __ffs(w) - 1;
    for (uint32_t idx = lane; idx < nrows * (uint32_t)w; idx += 32) {
      const uint32_t r = idx >> lw, j = idx & (uint32_t)(w - 1);
      if (!((rows_mine >> r) & 1u)) continue;
      unsigned long long val = 0ull;
      for (int i = (int)j; i < 64; i += w) val += fr[i * kLaneStride + r];
      dst[idx] = a.overwrite ? val : dst[idx] + val;
    }
    __syncwarp();
  }
}

// Fixed-size segments (pp_count_fixed) fed by a CTA-wide TMA ring.  A chunk
// is k whole "items" of S = 32/G consecutive segments (one warp's worth), so
// no segment straddles a stage.  The 8 consumer warps form two teams of 4;
// team q consumes this CTA's chunks j = q (mod 2), each warp taking items
// wi, wi + 4, ... of the chunk.  Chunk j uses stage j mod 2, so each stage
// belongs to one team and is consumed in order (an mbarrier parity wait is
// only sound when the waiter is at most one phase ahead).  Lanes
// read their segment's vectors from shared memory (a quarter/half/whole warp
// reads 128/256/512 contiguous bytes: conflict-free), count with the same
// G-lane carry-save counter as pp_seg_kernel and write the row.  Requires a
// 16-byte aligned base, seg_bytes % 16 == 0 and S * seg_bytes <= 16 KiB.
#ifndef PP_SEGTMA_EARLY_RELEASE
#define PP_SEGTMA_EARLY_RELEASE 1
#endif
#ifndef PP_SEGTMA_TEAMS  // A/B knobs (scripts/gpu_segtma.sh)
#define PP_SEGTMA_TEAMS 2
#define PP_SEGTMA_TEAM_WARPS 4
#define PP_SEGTMA_STAGES 2
#define PP_SEGTMA_STAGE_KIB 64
#endif
constexpr int kSegTmaTeams = PP_SEGTMA_TEAMS, kSegTmaTeamWarps = PP_SEGTMA_TEAM_WARPS;
constexpr int kSegTmaWarps = kSegTmaTeams * kSegTmaTeamWarps, kSegTmaStages = PP_SEGTMA_STAGES;
constexpr unsigned kSegTmaStageBytes = PP_SEGTMA_STAGE_KIB << 10;
static_assert(kSegTmaStages % kSegTmaTeams == 0, "each stage must belong to one team");
constexpr int kSegTmaThreads = (kSegTmaWarps + 1) * 32;
constexpr size_t kSegTmaSmem = kSegTmaStages * (size_t)kSegTmaStageBytes + 2 * kSegTmaStages * 8;

template <int G>
__global__ void __launch_bounds__(kSegTmaThreads, 1)
    pp_segtma_kernel(SegArgs a, unsigned items_per_chunk) {
  constexpr int S = 32 / G;
  extern __shared__ __align__(128) uint8_t smem[];
  uint4 *stages = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kSegTmaStages * kSegTmaStageBytes);
  uint64_t *empty = full + kSegTmaStages;
  __shared__ unsigned long long chunk_id[kSegTmaStages];  // written before the stage's arrival
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSegTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSegTmaTeamWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const unsigned long long seg_bytes = a.seg_bytes, nseg = a.nseg;
  const unsigned long long segs_per_chunk = (unsigned long long)items_per_chunk * S;
  const unsigned long long chunk_bytes = segs_per_chunk * seg_bytes;
  const unsigned long long total = nseg * seg_bytes;
  const unsigned long long nchunks = (nseg + segs_per_chunk - 1) / segs_per_chunk;
  constexpr uint32_t kStageVecs = kSegTmaStageBytes / 16;

  if (warp == kSegTmaWarps) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // chunk blockIdx.x first, then tickets of the stream's scheduler slot
      // (chunk gridDim.x + ticket) or the static grid stride; one stop
      // sentinel per team once the chunks are gone
      unsigned long long ch = blockIdx.x;
      int stops = 0;
      for (uint32_t j = 0;; ++j) {
        const uint32_t stage = j % kSegTmaStages;
        mbar_wait(&empty[stage], ((j / kSegTmaStages) & 1u) ^ 1u);
        if (ch >= nchunks) {
          chunk_id[stage] = kNoChunk;
          mbar_arrive(&full[stage]);
          if (++stops == kSegTmaTeams) break;
          continue;
        }
        chunk_id[stage] = ch;
        const unsigned long long off = ch * chunk_bytes;
        const unsigned long long rem = total - off;
        const uint32_t bytes = (uint32_t)(rem < chunk_bytes ? rem : chunk_bytes);
        if (PP_CHK(bytes <= kSegTmaStageBytes) &&
            PP_CHK_RANGE(a.base + off, bytes, a.chk_lo, a.chk_hi)) {
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(stages + stage * kStageVecs, a.base + off, bytes, &full[stage], pol);
        } else {  // checked build, failed check: no copy, the stage completes empty
          mbar_arrive(&full[stage]);
        }
        ch = a.sched ? gridDim.x + (unsigned long long)(atomicAdd(a.sched, 1u) - a.sched_base)
                     : ch + gridDim.x;
      }
    }
  } else {
  const uint32_t team = warp / kSegTmaTeamWarps, wi = warp % kSegTmaTeamWarps;
  const uint32_t r = lane % G, sl = lane / G;
  const uint32_t segv = (uint32_t)(seg_bytes >> 4);  // vectors per segment
  const TC t = make_tc(lane);
  for (uint32_t j = team;; j += kSegTmaTeams) {
    const uint32_t stage = j % kSegTmaStages;
    mbar_wait(&full[stage], (j / kSegTmaStages) & 1u);
    const unsigned long long ch = chunk_id[stage];
    if (ch == kNoChunk) break;
    PP_CHK(ch < nchunks);
    const uint4 *sv = stages + stage * kStageVecs;
    const unsigned long long seg0 = ch * segs_per_chunk;
    bool released = false;
    for (uint32_t it = wi; it < items_per_chunk; it += kSegTmaTeamWarps) {
      const unsigned long long s = seg0 + (unsigned long long)it * S + sl;
      if (seg0 + (unsigned long long)it * S >= nseg) break;  // warp-uniform
      const bool item_full = seg0 + (unsigned long long)(it + 1) * S <= nseg;
      const uint4 *sp = sv + (it * S + sl) * segv + r;
      PP_CHK((unsigned long long)(it * S + sl + 1) * segv <= kStageVecs);  // inside the stage
      GroupCounter<G, false> c;
      c.init();
      for (uint32_t k0 = 0; k0 < segv; k0 += 8 * G) {
        uint4 v[8];
        if (item_full && k0 + 8 * G <= segv) {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = sp[k0 + q * G];
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t k = k0 + q * G + r;
            v[q] = (k < segv && s < nseg) ? sp[k0 + q * G] : make_uint4(0u, 0u, 0u, 0u);
          }
        }
        c.eat8(v, t);
      }
      if (PP_SEGTMA_EARLY_RELEASE && it + kSegTmaTeamWarps >= items_per_chunk) {
        // this warp's last read of the stage is done: release it before the
        // flush and the row stores
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        released = true;
      }
      c.finish(t);
      if (s < nseg) write_row(a, s, reinterpret_cast<uintptr_t>(a.base) + s * seg_bytes, c, lane);
    }
    if (!released) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
  }
  }
}
// ------------------------------------------------------------------ host side
cudaError_t segmented_setup(DevInfo *d) {
  cudaError_t e;
  for (auto k : {pp_segtma_kernel<2>, pp_segtma_kernel<4>, pp_segtma_kernel<8>,
                 pp_segtma_kernel<16>, pp_segtma_kernel<32>})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSegTmaSmem)))
      return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d->seg_blocks_per_sm, pp_seg_kernel<8>,
                                                         kSegThreads, 0)))
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d->lane_blocks_per_sm,
                                                         pp_seglane_kernel<true>, kLaneThreads, 0)))
    return e;
  if (d->seg_blocks_per_sm < 1) d->seg_blocks_per_sm = 1;
  if (d->lane_blocks_per_sm < 1) d->lane_blocks_per_sm = 1;
  return cudaSuccess;
}

// Fixed segments take the TMA ring when they tile its 64 KiB stages into at
// least one item per team warp and there are enough chunks to fill the grid;
// PP_SEG_PATH=ldg forces pp_seg_kernel (A/B runs, tests).
static bool seg_use_tma(const SegArgs &a, const DevInfo &di, unsigned *items_per_chunk) {
  static const char *path = std::getenv("PP_SEG_PATH");
  if (path && std::strcmp(path, "ldg") == 0) return false;
  const bool force = path && std::strcmp(path, "tma") == 0;
  if (a.ptrs || a.seg_off || a.seg_bytes == 0 || (a.seg_bytes & 15) || ((uintptr_t)a.base & 15))
    return false;
  const unsigned long long item = (unsigned long long)(32 / a.lanes_per_segment) * a.seg_bytes;
  const unsigned long long k = kSegTmaStageBytes / item;
  if (k < (unsigned long long)kSegTmaTeamWarps) return false;
  // >= 32 vectors per lane per segment: below that the per-segment flush
  // dominates and the LDG kernel's 24 warps/SM hide it better
  // (scripts/seg_sweep.py, profiles/r1_segmented_ablation.md)
  if (!force && a.seg_bytes < 512ull * a.lanes_per_segment) return false;
  const unsigned long long chunks = (a.nseg * a.seg_bytes + k * item - 1) / (k * item);
  if (!force && chunks < 4ull * di.num_sms) return false;  // small batches: LDG latency wins
  *items_per_chunk = (unsigned)k;
  return true;
}

cudaError_t launch_segmented(const SegArgs &a0, const DevInfo &di, cudaStream_t st) {
  if (a0.nseg == 0) return cudaSuccess;
  SegArgs a = a0;
#if PP_CHECK_BOUNDS
  if (chk_corrupt_mode() == 3 && !a.ptrs && !a.short_max) a.base -= 16;  // pp_debug_corrupt
#endif
  unsigned ipc = 0;
  // G = 2 / 4 (1-2 KiB fixed segments: 32 vectors per lane) exist only on the
  // TMA ring; elsewhere their segments go one lane each (G = 2) or to G = 8
  if ((a.lanes_per_segment == 2 || a.lanes_per_segment == 4) && !seg_use_tma(a, di, &ipc)) {
    a.lanes_per_segment = a.lanes_per_segment == 2 ? 1 : 8;
    // G = 2 demoted to one lane per segment: that single pass counts every
    // segment, so the hybrid split must go -- else the one-lane kernel would
    // count only the short segments and no pass would take the long ones
    // (the hybrid's own one-lane pass below arrives here with G = 1 as asked
    // and keeps its short_max)
    if (a.lanes_per_segment == 1) a.short_max = 0;
  }
  const int G = a.lanes_per_segment;
  if (a.short_max && G != 1) {
    // hybrid: short segments one lane each, then the rest with G lanes
    SegArgs sh = a;
    sh.lanes_per_segment = 1;
    cudaError_t e = launch_segmented(sh, di, st);
    if (e != cudaSuccess) return e;
  }
  if (G == 1) {  // one lane per segment
    const unsigned long long need = (a.nseg + kLaneThreads - 1) / kLaneThreads;
    const unsigned g = grid_for(need, (unsigned long long)di.num_sms * di.lane_blocks_per_sm);
    if (a.ptrs)
      pp_seglane_kernel<false, false, true><<<g, kLaneThreads, 0, st>>>(a);
    else if (a.seg_off && a.short_max)
      pp_seglane_kernel<false, true><<<g, kLaneThreads, 0, st>>>(a);
    else if (a.seg_off)
      pp_seglane_kernel<false><<<g, kLaneThreads, 0, st>>>(a);
    else
      pp_seglane_kernel<true><<<g, kLaneThreads, 0, st>>>(a);
    return cudaGetLastError();
  }
  if (seg_use_tma(a, di, &ipc)) {
    const unsigned long long chunks =
        (a.nseg + (unsigned long long)ipc * (32 / G) - 1) / ((unsigned long long)ipc * (32 / G));
    const unsigned g = grid_for(chunks, (unsigned long long)di.num_sms);
    SegArgs b = a;  // dynamic chunk order once CTAs stream tens of chunks
    std::unique_lock<std::mutex> lk;  // base hand-out and launch: one critical section
    if (chunks >= 16ull * g) {
      lk = sched_lock();
      b.sched = sched_slot(di, st, chunks, &b.sched_base);
    }
    if (G == 2)
      pp_segtma_kernel<2><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(b, ipc);
    else if (G == 4)
      pp_segtma_kernel<4><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(b, ipc);
    else if (G == 8)
      pp_segtma_kernel<8><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(b, ipc);
    else if (G == 16)
      pp_segtma_kernel<16><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(b, ipc);
    else
      pp_segtma_kernel<32><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(b, ipc);
    const cudaError_t e = cudaGetLastError();
    if (b.sched) {
      if (e != cudaSuccess)
        sched_rollback(chunks);
      else
        sched_commit(st);
    }
    return e;
  }
  const unsigned long long segs_per_block = (kSegThreads / 32) * (32 / G);
  const unsigned long long need = (a.nseg + segs_per_block - 1) / segs_per_block;
  const unsigned g = grid_for(need, (unsigned long long)di.num_sms * di.seg_blocks_per_sm);
  SegArgs b = a;  // dynamic group order once warps see several groups each
  if (b.batch_groups == 0)
    b.batch_groups = seg_batch_groups(a.nseg, G);
  // work units = the kernel's batches (its tickets)
  const unsigned long long batches = seg_batches(a.nseg, G, b.batch_groups);
  std::unique_lock<std::mutex> lk;  // base hand-out and launch: one critical section
  if (need >= 4ull * g) {
    lk = sched_lock();
    b.sched = sched_slot(di, st, batches, &b.sched_base);
  }
  if (b.short_max) {
    if (G == 8)
      pp_seg_kernel<8, true><<<g, kSegThreads, 0, st>>>(b);
    else if (G == 16)
      pp_seg_kernel<16, true><<<g, kSegThreads, 0, st>>>(b);
    else
      pp_seg_kernel<32, true><<<g, kSegThreads, 0, st>>>(b);
  } else if (G == 8) {
    pp_seg_kernel<8><<<g, kSegThreads, 0, st>>>(b);
  } else if (G == 16) {
    pp_seg_kernel<16><<<g, kSegThreads, 0, st>>>(b);
  } else {
    pp_seg_kernel<32><<<g, kSegThreads, 0, st>>>(b);
  }
  const cudaError_t e = cudaGetLastError();
  if (b.sched) {
    if (e != cudaSuccess)
      sched_rollback(batches);
    else
      sched_commit(st);
  }
  return e;
}

cudaError_t chk_read_seg(ChkRecHost *out, bool reset) {
#if PP_CHECK_BOUNDS
  ChkRec r{};
  cudaError_t e = cudaMemcpyFromSymbol(&r, pp_chk, sizeof r);
  if (e != cudaSuccess) return e;
  *out = ChkRecHost{r.fails, r.first_line, r.first_addr, r.first_lo, r.first_hi};
  if (reset) {
    const ChkRec z{};
    return cudaMemcpyToSymbol(pp_chk, &z, sizeof z);
  }
#else
  (void)reset;
  *out = ChkRecHost{};
#endif
  return cudaSuccess;
}

}  // namespace pp
