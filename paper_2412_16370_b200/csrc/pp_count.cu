// pp_count.cu — sm_100a kernels of the positional population count.
//
// Hot path (replaces NumbaKernel.run + _nbkern.run_main, kernels.py:242-270,
// _nbkern.py:43-177):
//
//   pp_count_tma_kernel   persistent, one CTA per SM.  One elected producer
//                         thread streams 32 KiB chunks of the aligned body
//                         HBM -> shared memory with cp.async.bulk (UBLKCP),
//                         3-deep mbarrier ring; 8 consumer warps read
//                         the stage with conflict-free LDS.128 and run the
//                         two-level carry-save count (pp_device.cuh).
//   pp_count_ldg_kernel   same arithmetic fed by LDG.128 straight to
//                         registers (tuning alternative / A-B evidence).
//
// Both finish with a warp bit-transpose + __popc per bit position, a shared
// u64 frame[64] per CTA, and one u64 atomicAdd per (CTA, counter) after the
// rotate-and-fold of flush_fw (accumulate.py:115-130).
//
// Segmented mode: pp_seg_kernel<G>, G lanes per segment.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaStages = 3;  // 3 x 32 KiB: best of the scripts/bw_probe.cu sweep (profiles/)
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
constexpr int kTmaStageVecs = kTmaConsumerWarps * 32 * 8;  // 2048 x 16 B = 32 KiB
constexpr unsigned long long kTmaStageBytes = kTmaStageVecs * 16ull;
constexpr size_t kTmaSmemBytes = kTmaStages * kTmaStageBytes + 2 * kTmaStages * 8;

// Shape of the TMA pipeline for NCW consumer warps (8 vectors per thread per
// stage).  The counting kernel uses 8 warps; the fused one-hot producer does
// ~4x more ALU work per byte and uses more consumer warps.
template <int NCW>
struct TmaShape {
  static constexpr int kThreads = (NCW + 1) * 32;
  static constexpr int kStageVecs = NCW * 32 * 8;
  static constexpr unsigned long long kStageBytes = kStageVecs * 16ull;
  static constexpr size_t kSmem = kTmaStages * kStageBytes + 2 * kTmaStages * 8;
};
#ifndef PP_CAT_NCW
#define PP_CAT_NCW 16
#endif
using CatShape = TmaShape<PP_CAT_NCW>;

constexpr int kLdgWarps = 8;
constexpr int kLdgThreads = kLdgWarps * 32;
constexpr int kLdgChunkVecs = kLdgThreads * 8;
constexpr unsigned long long kLdgChunkBytes = kLdgChunkVecs * 16ull;

constexpr int kSegThreads = 256;
#ifndef PP_SEG_SMEM_COUNTS
#define PP_SEG_SMEM_COUNTS true
#endif
#ifndef PP_SEG_MIN_BLOCKS
#define PP_SEG_MIN_BLOCKS 3  // <= 85 registers: 24 warps/SM of loads in flight
#endif

// Head/tail bytes (< 16 each) as one extra weight-1 plane pair, counted by
// warp 0 of CTA 0.  Lane l < 16 takes head byte l, lane 16+l tail byte l.
__device__ __forceinline__ void count_edges(Counter &c, const uint8_t *head, uint32_t hb,
                                            const uint8_t *tail, uint32_t tb, uint32_t lane,
                                            const TC &t) {
  const uint8_t *p = nullptr;
  if (lane < 16) {
    if (lane < hb) p = head + lane;
  } else if (lane - 16 < tb) {
    p = tail + (lane - 16);
  }
  unsigned long long fw = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // input complete (PDL)
  if (p) fw = (unsigned long long)__ldg(p) << frame_shift(p);
  c.ce += wcount((uint32_t)fw, t);
  c.co += wcount((uint32_t)(fw >> 32), t);
}

// counters[j] += sum_{i = j mod w} frame[(i + rot) mod 64]   (flush_fw)
// With pp_count_multi the same sums also go to a.extra[] -- typically the
// other ranks' counters mapped over NVLink, so these atomics ARE the sharded
// job's allreduce, fused into the counting kernel (remote RED.ADD.64).
__device__ __forceinline__ void fold_frame_to_counters(const unsigned long long *frame,
                                                       const CountArgs &a) {
  const int j = threadIdx.x, width = a.width;
  if (j < width) {
    // under programmatic dependent launch the previous grid on the stream may
    // still be running: its counter updates complete before ours (no-op
    // without PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned long long s = 0;
    for (int i = j; i < 64; i += width) s += frame[(i + a.rot) & 63];
    if (s) {
      atomicAdd(a.counters + j, s);
      for (int k = 0; k < a.nextra; ++k) atomicAdd(a.extra[k] + j, s);
    }
  }
}

// ---- fused one-hot producer (pp_count_categories on u8 codes) -------------
// A code c < W becomes bit c of a one-hot word; words are packed so that the
// frame position of that bit is = c (mod W) and the epilogue is the plain
// fold with rot = 0:  W=8: four codes per word (byte k holds 1 << code_k),
// W=16: two codes per word (half k), W=32: one code per word, W=64: one code
// per (x|z = bits 0-31, y|w = bits 32-63) pair.  Codes >= W give no bit.

// 4 u8 codes -> 4 one-hot bytes.  PRMT against the table {1,2,4,...,128}
// turns nibble-packed codes into one-hot bytes in one instruction; bytes
// whose code is >= 8 are cleared only when such a byte is present.
__device__ __forceinline__ uint32_t onehot8x4(uint32_t x, bool any_big) {
  const uint32_t xl = x & 0x07070707u;
  const uint32_t tt = xl | (xl >> 4);
  const uint32_t sel = (tt & 0xFFu) | ((tt >> 8) & 0xFF00u);
  uint32_t oh = __byte_perm(0x08040201u, 0x80402010u, sel);
  if (any_big) {
    const uint32_t hi = x & 0xF8F8F8F8u;
    const uint32_t nz = (((hi & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | hi) & 0x80808080u;
    oh &= ~((nz >> 7) * 0xFFu);
  }
  return oh;
}
#ifndef PP_CAT_V2
#define PP_CAT_V2 1
#endif
// v2 of the same: 2 ops for the nibble-packed selector (the LOP3 select
// leaves junk only in the nibbles of codes >= 8, which the mask clears), and
// a 5-op mask: z = (x | 0x80..) - 0x08.. has a byte's msb set iff that byte
// is in [8, 0x80) (no borrow crosses a byte), x's msb covers [0x80, 0xFF];
// PRMT's sign-replicate mode (selector nibble 8|i) widens msb -> 0xFF.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t onehot8x4_v2(uint32_t x, bool any_big) {
  uint32_t tt;  // (x & 0x07070707) | ((x >> 4) & ~0x07070707): one LOP3
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(tt) : "r"(x), "r"(x >> 4), "r"(0x07070707u));
  const uint32_t sel = prmt(tt, 0u, 0x0020u);  // nibbles: code0..code3 (low 16 bits)
  uint32_t oh = prmt(0x08040201u, 0x80402010u, sel);  // junk nibbles: masked below
  if (any_big) {
    const uint32_t z = (x | 0x80808080u) - 0x08080808u;
    oh &= ~prmt(z | x, 0u, 0xBA98u);
  }
  return oh;
}
// (1 << c) as a (lo, hi) pair; c >= 64 gives 0 (shl.b64 clamps)
__device__ __forceinline__ void onehot64(uint32_t c, uint32_t &lo, uint32_t &hi) {
  asm("{\n\t.reg .b64 t;\n\tmov.b64 t, 1;\n\tshl.b64 t, t, %2;\n\tmov.b64 {%0, %1}, t;\n\t}"
      : "=r"(lo), "=r"(hi) : "r"(c));
}

// byte k of x, zero-extended: one PRMT
__device__ __forceinline__ uint32_t byte_of(uint32_t x, int k) {
  return __byte_perm(x, 0u, 0x4440u | (uint32_t)k);
}
// 2 u8 codes (bytes k, k+1 of x) -> one word with 16-bit one-hot halves
__device__ __forceinline__ uint32_t onehot16x2(uint32_t x, int k) {
  const uint32_t a = byte_of(x, k), b = byte_of(x, k + 1);
  uint32_t lo, hi;
  asm("shl.b32 %0, 1, %1;" : "=r"(lo) : "r"(a));        // >= 32 -> 0 (clamped)
  asm("shl.b32 %0, 65536, %1;" : "=r"(hi) : "r"(b));    // >= 16 -> 0
  return (lo & 0xFFFFu) | hi;
}
__device__ __forceinline__ uint32_t onehot32(uint32_t c) {
  uint32_t r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(c));  // c >= 32 -> 0
  return r;
}

// Expand and count 8 vectors (128 u8 codes) of one thread; vectors with
// valid bit i clear are absent (partial last chunk) and contribute nothing.
// FULL: every vector present (all but the last chunk) -- no per-word selects.
template <int W, bool FULL>
__device__ __forceinline__ void eat_codes(Counter &c, const uint4 (&v)[8], uint32_t valid,
                                          const TC &t) {
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  if (W == 8) {
    uint4 u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool big = ((v[i].x | v[i].y | v[i].z | v[i].w) & 0xF8F8F8F8u) != 0;
#if PP_CAT_V2
      u[i] = make_uint4(onehot8x4_v2(v[i].x, big), onehot8x4_v2(v[i].y, big),
                        onehot8x4_v2(v[i].z, big), onehot8x4_v2(v[i].w, big));
#else
      u[i] = make_uint4(onehot8x4(v[i].x, big), onehot8x4(v[i].y, big),
                        onehot8x4(v[i].z, big), onehot8x4(v[i].w, big));
#endif
      if (!FULL && !((valid >> i) & 1u)) u[i] = z4;
    }
    c.eat8(u, t);
  } else if (W == 16) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint4 u[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 x = v[4 * h + i];
        const bool ok = FULL || ((valid >> (4 * h + i)) & 1u);
        u[2 * i] = ok ? make_uint4(onehot16x2(x.x, 0), onehot16x2(x.x, 2), onehot16x2(x.y, 0),
                                   onehot16x2(x.y, 2))
                      : z4;
        u[2 * i + 1] = ok ? make_uint4(onehot16x2(x.z, 0), onehot16x2(x.z, 2),
                                       onehot16x2(x.w, 0), onehot16x2(x.w, 2))
                          : z4;
      }
      c.eat8(u, t);
    }
  } else if (W == 32) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint4 u[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint4 x = v[2 * h + i];
        const bool ok = FULL || ((valid >> (2 * h + i)) & 1u);
        const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t wd = w4[q];
          u[4 * i + q] = ok ? make_uint4(onehot32(wd & 0xFFu), onehot32(byte_of(wd, 1)),
                                         onehot32(byte_of(wd, 2)), onehot32(wd >> 24))
                            : z4;
        }
      }
      c.eat8(u, t);
    }
  } else {  // W == 64: code c -> (x|z, y|w) = (1 << c, 1 << (c - 32))
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const uint4 x = v[h];
      const bool ok = FULL || ((valid >> h) & 1u);
      const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint32_t c0 = byte_of(w4[q], 2 * k), c1 = byte_of(w4[q], 2 * k + 1);
#if PP_CAT_V2
          uint32_t l0, h0, l1, h1;
          onehot64(c0, l0, h0);
          onehot64(c1, l1, h1);
          u[2 * q + k] = ok ? make_uint4(l0, h0, l1, h1) : z4;
#else
          u[2 * q + k] = ok ? make_uint4(onehot32(c0), onehot32(c0 - 32u), onehot32(c1),
                                         onehot32(c1 - 32u))
                            : z4;
#endif
        }
      }
      c.eat8(u, t);
    }
  }
}

// Head/tail codes (< 16 each) of the fused producer: frame position = code.
__device__ __forceinline__ void count_code_edges(Counter &c, const uint8_t *head, uint32_t hb,
                                                 const uint8_t *tail, uint32_t tb, uint32_t lane,
                                                 int width, const TC &t) {
  uint32_t code = 0xFFu;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // input complete (PDL)
  if (lane < 16) {
    if (lane < hb) code = __ldg(head + lane);
  } else if (lane - 16 < tb) {
    code = __ldg(tail + (lane - 16));
  }
  const bool ok = code < (uint32_t)width;
  c.ce += wcount(ok ? onehot32(code) : 0u, t);
  c.co += wcount(ok ? onehot32(code - 32u) : 0u, t);
}

// MODE 0: read-only roofline (XOR of every word), MODE 1: positional count,
// MODE 8/16/32/64: fused one-hot producer over u8 codes at that width.
template <int MODE, int NCW = kTmaConsumerWarps>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    pp_tma_kernel(CountArgs a, unsigned long long *sink) {
  constexpr bool kCount = MODE != 0;
  using Sh = TmaShape<NCW>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint4 *stages = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kTmaStages * Sh::kStageBytes);
  uint64_t *empty = full + kTmaStages;
  __shared__ unsigned long long frame[64];

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < 64) frame[threadIdx.x] = 0;
  __syncthreads();

  const unsigned long long nchunks = a.nchunks;
  if (warp == NCW) {
    // ---------------- producer: one elected thread issues bulk copies
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // programmatic dependent launch: everything above overlapped the
      // previous grid's tail; its outputs (possibly our input) are complete
      // and visible only after this wait
      asm volatile("griddepcontrol.wait;" ::: "memory");
      uint32_t stage = 0, phase = 0;
      for (unsigned long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        mbar_wait(&empty[stage], phase ^ 1);
        const unsigned long long off = ch * Sh::kStageBytes;
        const unsigned long long rem = a.body_bytes - off;
        const uint32_t bytes = (uint32_t)(rem < Sh::kStageBytes ? rem : Sh::kStageBytes);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(stages + stage * Sh::kStageVecs, a.body + off, bytes, &full[stage], pol);
        if (++stage == kTmaStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      // every load of this CTA is in flight: the next launch on the stream
      // (programmatic dependent launch) may start filling its own ring
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
  } else {
    // ---------------- consumers
    const TC t = make_tc(lane);
    Counter c;
    c.init();
    uint32_t xs = 0;  // read-only roofline accumulator
    uint32_t stage = 0, phase = 0;
    const uint32_t tid = threadIdx.x;
    for (unsigned long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
      mbar_wait(&full[stage], phase);
      const uint4 *sv = stages + stage * Sh::kStageVecs;
      uint4 v[8];
      uint32_t valid = 0xFFu;  // vectors present in this (possibly partial) chunk
      const unsigned long long off = ch * Sh::kStageBytes;
      const unsigned long long rem = a.body_bytes - off;
      if (rem >= Sh::kStageBytes) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = sv[tid + i * (NCW * 32)];
      } else {
        const uint32_t nv = (uint32_t)(rem >> 4);
        valid = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t idx = tid + i * (NCW * 32);
          v[i] = idx < nv ? sv[idx] : make_uint4(0u, 0u, 0u, 0u);
          valid |= (idx < nv ? 1u : 0u) << i;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (MODE == 1) {
        c.eat8(v, t);
      } else if (MODE >= 8) {
        if (valid == 0xFFu)
          eat_codes<(MODE >= 8 ? MODE : 8), true>(c, v, valid, t);
        else
          eat_codes<(MODE >= 8 ? MODE : 8), false>(c, v, valid, t);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) xs ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
      }
      if (++stage == kTmaStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (kCount) {
      c.finish(t);
      if (blockIdx.x == 0 && warp == 0) {
        if (MODE == 1)
          count_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, t);
        else
          count_code_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, a.width, t);
      }
      atomicAdd(&frame[lane], c.ce);
      atomicAdd(&frame[32 + lane], c.co);
    } else {
      xs = __reduce_xor_sync(FULL, xs);
      if (lane == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        atomicXor(sink, (unsigned long long)xs);
      }
    }
  }
  __syncthreads();
  if (kCount) fold_frame_to_counters(frame, a);
}

__global__ void __launch_bounds__(kLdgThreads)
    pp_count_ldg_kernel(CountArgs a) {
  __shared__ unsigned long long frame[64];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) frame[threadIdx.x] = 0;
  __syncthreads();
  const TC t = make_tc(lane);
  Counter c;
  c.init();
  const uint4 *body = reinterpret_cast<const uint4 *>(a.body);
  const unsigned long long nvec = a.body_bytes >> 4;
  for (unsigned long long ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x) {
    const unsigned long long base = ch * kLdgChunkVecs + threadIdx.x;
    uint4 v[8];
    if ((ch + 1) * kLdgChunkVecs <= nvec) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ldg_stream(body + base + i * kLdgThreads);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const unsigned long long idx = base + i * kLdgThreads;
        v[i] = idx < nvec ? ldg_stream(body + idx) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    c.eat8(v, t);
  }
  c.finish(t);
  if (blockIdx.x == 0 && warp == 0)
    count_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, t);
  atomicAdd(&frame[lane], c.ce);
  atomicAdd(&frame[32 + lane], c.co);
  __syncthreads();
  fold_frame_to_counters(frame, a);
}

// Bytes [max(va, lo), min(va + 16, hi)) of the aligned 16-byte block at va,
// zero elsewhere: the masked head / tail vector of a segment.  Exact-bounds
// byte loads, so nothing outside the segment is ever read.
__device__ __noinline__ uint4 load_partial(uintptr_t va, uintptr_t lo, uintptr_t hi) {
  uint32_t q[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    const uintptr_t ad = va + b;
    if (ad >= lo && ad < hi)
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
  if (s < a.nseg) {
    if (a.seg_off) {
      s0 = a.seg_off[s];
      s1 = a.seg_off[s + 1];
      if (s1 < s0) s1 = s0;
    } else {
      s0 = s * a.seg_bytes;
      s1 = s0 + a.seg_bytes;
    }
  }
  SegGeom g;
  g.p0 = reinterpret_cast<uintptr_t>(a.base) + s0;
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

// Row s of out <- the counts lane r of the segment's G-lane group holds
// (frame bits G*f + r and 32 + G*f + r), rotated by rot = 8*(p0 mod 8) and
// folded mod w exactly like flush_fw (accumulate.py:115-130).  All G lanes of
// the group call this together (they share s).
template <int G, bool SM>
__device__ __forceinline__ void write_row(const SegArgs &a, unsigned long long s,
                                          uintptr_t p0, const GroupCounter<G, SM> &c,
                                          uint32_t lane) {
  constexpr int S = 32 / G;
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
      *de = ow ? c.e(f) : *de + c.e(f);
      *dd = ow ? c.o(f) : *dd + c.o(f);
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
        *d = ow ? tot : *d + tot;
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
      *d = ow ? tot : *d + tot;
    }
  }
}

// Segmented count fed by LDG, G lanes per segment (S = 32/G segments per
// warp), grid-stride over groups of S segments.  Lane r of a segment eats
// vectors r, r+G, ... in groups of 8 (G x 16 contiguous bytes per load
// instruction per segment).  A TMA-fed variant (per-warp bulk-copy rings) was
// 1.5x slower here: profiles/r1_segmented_ablation.md.
template <int G>
__global__ void __launch_bounds__(kSegThreads, PP_SEG_MIN_BLOCKS)
    pp_seg_kernel(SegArgs a) {
  constexpr int S = 32 / G;
  __shared__ unsigned long long slots[(kSegThreads / 32) * 2 * S * 32];
  const uint32_t lane = threadIdx.x & 31, r = lane % G, sl = lane / G;
  const unsigned long long gw = (blockIdx.x * (unsigned long long)kSegThreads + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)kSegThreads) >> 5;
  const TC t = make_tc(lane);
  for (unsigned long long first = gw * S; first < a.nseg; first += nw * S) {
    const unsigned long long s = first + sl;
    const SegGeom g = seg_geom(a, s);
    GroupCounter<G, PP_SEG_SMEM_COUNTS> c;
    c.init(slots + (threadIdx.x >> 5) * (2 * S * 32) + lane);
    // full (aligned, in-range) vectors are [kf0, kf1)
    const unsigned long long kf0 = g.hp ? 1 : 0;
    const unsigned long long kf1 = (g.tp && g.nvv) ? g.nvv - 1 : g.nvv;
    const uint4 *vp = reinterpret_cast<const uint4 *>(g.A) + r;
    auto load_round = [&](unsigned long long k0, uint4 (&v)[8]) {
      if (k0 + r >= kf0 && k0 + r + 7 * G < kf1) {
        // fast path: 8 full vectors, base pointer + immediate offsets
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = ldg_stream(vp + k0 + j * G);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const unsigned long long k = k0 + j * G + r;
          v[j] = make_uint4(0u, 0u, 0u, 0u);
          if (k < g.nvv) {
            const uintptr_t va = g.A + 16 * k;
            if (seg_partial(g, k))
              v[j] = load_partial(va, g.p0, g.e);
            else
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
    if (s < a.nseg) write_row(a, s, g.p0, c, lane);
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

// 0xFF in bytes [lo, hi) of a u32 holding bytes 4q..4q+3 of a vector
__device__ __forceinline__ uint32_t byte_range_mask(int q, int lo, int hi) {
  const int a = min(max(lo - 4 * q, 0), 4), b = min(max(4 * q + 4 - hi, 0), 4);
  uint32_t m1, m2;
  asm("shl.b32 %0, %1, %2;" : "=r"(m1) : "r"(0xFFFFFFFFu), "r"(8 * a));  // 32 -> 0
  asm("shr.b32 %0, %1, %2;" : "=r"(m2) : "r"(0xFFFFFFFFu), "r"(8 * b));
  return m1 & m2;
}

template <bool FIXED>
__global__ void __launch_bounds__(kLaneThreads)
    pp_seglane_kernel(SegArgs a) {
  __shared__ uint32_t frs[kLaneWarps][64 * kLaneStride];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *fr = frs[warp];
  const uintptr_t base = reinterpret_cast<uintptr_t>(a.base);
  // the caller's view: vectors entirely inside it are read whole, the
  // others byte by byte (nothing outside the view is ever read)
  const uintptr_t view_lo = base + (FIXED ? 0ull : a.seg_off[0]);
  const uintptr_t view_hi = base + (FIXED ? a.nseg * a.seg_bytes : a.seg_off[a.nseg]);
  const unsigned long long nw = (unsigned long long)gridDim.x * kLaneWarps;
  for (unsigned long long s0 = ((unsigned long long)blockIdx.x * kLaneWarps + warp) * 32;
       s0 < a.nseg; s0 += nw * 32) {
    const unsigned long long s = s0 + lane;
    unsigned long long b0 = 0, b1 = 0;
    if (s < a.nseg) {
      if (FIXED) {
        b0 = s * a.seg_bytes;
        b1 = b0 + a.seg_bytes;
      } else {
        b0 = a.seg_off[s];
        b1 = a.seg_off[s + 1];
        if (b1 < b0) b1 = b0;
      }
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
    for (uintptr_t va = p0 & ~(uintptr_t)15; va < e; va += 16) {
      uint4 v;
      if (va >= view_lo && va + 16 <= view_hi) {
        v = __ldg(reinterpret_cast<const uint4 *>(va));
        if (va < p0 || va + 16 > e) {  // mask to the segment
          const int lo = va < p0 ? (int)(p0 - va) : 0;
          const int hi = va + 16 > e ? (int)(e - va) : 16;
          v.x &= byte_range_mask(0, lo, hi);
          v.y &= byte_range_mask(1, lo, hi);
          v.z &= byte_range_mask(2, lo, hi);
          v.w &= byte_range_mask(3, lo, hi);
        }
      } else {
        v = load_partial(va, p0, e);
      }
      // x, z: frame bits 0-31; y, w: 32-63
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        nl[b] += ((v.x >> b) & 0x11111111u) + ((v.z >> b) & 0x11111111u);
        nh[b] += ((v.y >> b) & 0x11111111u) + ((v.w >> b) & 0x11111111u);
      }
      if (++nvec == 7) {
        nvec = 0;
        nib_to_byte();
        if (++nnib == 18) {
          nnib = 0;
          byte_to_smem(!spilled);
          spilled = true;
        }
      }
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
      uint32_t j = 0;
      for (unsigned long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++j) {
        const uint32_t stage = j % kSegTmaStages;
        mbar_wait(&empty[stage], ((j / kSegTmaStages) & 1u) ^ 1u);
        const unsigned long long off = ch * chunk_bytes;
        const unsigned long long rem = total - off;
        const uint32_t bytes = (uint32_t)(rem < chunk_bytes ? rem : chunk_bytes);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(stages + stage * kStageVecs, a.base + off, bytes, &full[stage], pol);
      }
    }
    return;
  }

  const uint32_t team = warp / kSegTmaTeamWarps, wi = warp % kSegTmaTeamWarps;
  const uint32_t r = lane % G, sl = lane / G;
  const uint32_t segv = (uint32_t)(seg_bytes >> 4);  // vectors per segment
  const TC t = make_tc(lane);
  uint32_t j = team;
  for (unsigned long long ch = blockIdx.x + (unsigned long long)team * gridDim.x; ch < nchunks;
       ch += (unsigned long long)kSegTmaTeams * gridDim.x, j += kSegTmaTeams) {
    const uint32_t stage = j % kSegTmaStages;
    mbar_wait(&full[stage], (j / kSegTmaStages) & 1u);
    const uint4 *sv = stages + stage * kStageVecs;
    const unsigned long long seg0 = ch * segs_per_chunk;
    bool released = false;
    for (uint32_t it = wi; it < items_per_chunk; it += kSegTmaTeamWarps) {
      const unsigned long long s = seg0 + (unsigned long long)it * S + sl;
      if (seg0 + (unsigned long long)it * S >= nseg) break;  // warp-uniform
      const bool item_full = seg0 + (unsigned long long)(it + 1) * S <= nseg;
      const uint4 *sp = sv + (it * S + sl) * segv + r;
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

// ------------------------------------------------------------------ host side
void split_range(const uint8_t *data, unsigned long long nbytes,
                 unsigned long long chunk_bytes, CountArgs *a) {
  const unsigned long long mis = (16u - ((uintptr_t)data & 15u)) & 15u;
  const unsigned long long hb = mis < nbytes ? mis : nbytes;
  const unsigned long long body = (nbytes - hb) & ~15ull;
  a->head = data;
  a->head_bytes = (uint32_t)hb;
  a->body = data + hb;
  a->body_bytes = body;
  a->nchunks = (body + chunk_bytes - 1) / chunk_bytes;
  a->tail = data + hb + body;
  a->tail_bytes = (uint32_t)(nbytes - hb - body);
  a->rot = (int)(8u * ((uintptr_t)data & 7u));
}

unsigned long long codes8_chunk_bytes() { return CatShape::kStageBytes; }

unsigned long long count_chunk_bytes(LoadPath path) {
  return path == LoadPath::kTma ? kTmaStageBytes : kLdgChunkBytes;
}

// Per-device launch facts, computed once per device (thread-safe: double-
// checked under a mutex; the kernel attributes are set with `dev` current).
static cudaError_t compute_device_info(int dev, DevInfo *out) {
  DevInfo d{};
  cudaError_t e;
  if ((e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  if ((e = cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev))) return e;
  if ((e = cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev))) return e;
  if ((e = cudaFuncSetAttribute(pp_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kTmaSmemBytes)))
    return e;
  if ((e = cudaFuncSetAttribute(pp_tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kTmaSmemBytes)))
    return e;
  for (auto k : {pp_tma_kernel<8, PP_CAT_NCW>, pp_tma_kernel<16, PP_CAT_NCW>,
                 pp_tma_kernel<32, PP_CAT_NCW>, pp_tma_kernel<64, PP_CAT_NCW>})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)CatShape::kSmem)))
      return e;
  for (auto k : {pp_segtma_kernel<8>, pp_segtma_kernel<16>, pp_segtma_kernel<32>})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSegTmaSmem)))
      return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.seg_blocks_per_sm, pp_seg_kernel<8>,
                                                         kSegThreads, 0)))
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.ldg_blocks_per_sm,
                                                         pp_count_ldg_kernel, kLdgThreads, 0)))
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.lane_blocks_per_sm,
                                                         pp_seglane_kernel<true>, kLaneThreads, 0)))
    return e;
  d.seg_blocks_per_sm = std::max(d.seg_blocks_per_sm, 1);
  d.ldg_blocks_per_sm = std::max(d.ldg_blocks_per_sm, 1);
  d.lane_blocks_per_sm = std::max(d.lane_blocks_per_sm, 1);
  {  // SMs left free for concurrent work (e.g. NCCL kernels of a sharded job)
    const char *r = std::getenv("PP_RESERVE_SMS");
    const int reserve = r ? std::atoi(r) : 0;
    d.count_sms = (reserve > 0 && reserve < d.num_sms) ? d.num_sms - reserve : d.num_sms;
  }
  d.ready = true;
  *out = d;
  return cudaSuccess;
}

cudaError_t device_info(int dev, DevInfo *out) {
  constexpr int kMaxDev = 64;
  static DevInfo cache[kMaxDev];
  static std::atomic<bool> ready[kMaxDev];
  static std::mutex m;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!ready[dev].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lk(m);
    if (!ready[dev].load(std::memory_order_relaxed)) {
      int cur = -1;
      cudaError_t e = cudaGetDevice(&cur);
      if (e != cudaSuccess) return e;
      if (cur != dev && (e = cudaSetDevice(dev)) != cudaSuccess) return e;
      DevInfo d;
      e = compute_device_info(dev, &d);
      if (cur != dev) cudaSetDevice(cur);
      if (e != cudaSuccess) return e;
      cache[dev] = d;
      ready[dev].store(true, std::memory_order_release);
    }
  }
  *out = cache[dev];
  return cudaSuccess;
}

static unsigned grid_for(unsigned long long nchunks, unsigned long long cap) {
  unsigned long long g = nchunks < cap ? nchunks : cap;
  return (unsigned)(g ? g : 1);
}

// Launch a TMA-ring kernel, with programmatic dependent launch when `pdl`:
// two CTAs of consecutive launches fit on one SM, so launch i+1 streams while
// launch i drains its tail.  Measured (scripts/pdl_sweep.py): 4.9 -> 3.8 us
// per 1 MiB call, 14.4 -> 10.8 us per 64 MiB, +7 % at 256 MiB, but -1 % at
// 1 GiB where the overlapping CTAs contend; hence the size cut below.
// PP_NO_PDL=1 disables it (A/B runs).
static unsigned long long pdl_max_body() {  // PP_PDL_MAX_MIB overrides (A/B runs)
  static const unsigned long long v = [] {
    const char *e = std::getenv("PP_PDL_MAX_MIB");
    return (e ? std::strtoull(e, nullptr, 10) : 512ull) << 20;
  }();
  return v;
}

template <typename Kern>
static cudaError_t launch_tma(Kern kernel, unsigned grid, unsigned block, size_t smem,
                              cudaStream_t st, const CountArgs &a, unsigned long long *sink,
                              bool want_pdl) {
  static const bool pdl_off = std::getenv("PP_NO_PDL") != nullptr;
  const bool pdl = want_pdl && !pdl_off;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, a, sink);
}

cudaError_t launch_count(const CountArgs &a, LoadPath path, const DevInfo &di,
                         cudaStream_t st) {
  if (path == LoadPath::kTma) {
    const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
    cudaError_t e = launch_tma(pp_tma_kernel<1>, g, kTmaThreads, kTmaSmemBytes, st, a, nullptr,
                               a.body_bytes < pdl_max_body());
    if (e != cudaSuccess) return e;
  } else {
    const unsigned g =
        grid_for(a.nchunks, (unsigned long long)di.num_sms * di.ldg_blocks_per_sm);
    pp_count_ldg_kernel<<<g, kLdgThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_count_codes8(const CountArgs &a, const DevInfo &di, cudaStream_t st) {
  const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
  switch (a.width) {
    case 8:
      return launch_tma(pp_tma_kernel<8, PP_CAT_NCW>, g, CatShape::kThreads, CatShape::kSmem, st,
                        a, nullptr, true);
    case 16:
      return launch_tma(pp_tma_kernel<16, PP_CAT_NCW>, g, CatShape::kThreads, CatShape::kSmem,
                        st, a, nullptr, true);
    case 32:
      return launch_tma(pp_tma_kernel<32, PP_CAT_NCW>, g, CatShape::kThreads, CatShape::kSmem,
                        st, a, nullptr, true);
    default:
      return launch_tma(pp_tma_kernel<64, PP_CAT_NCW>, g, CatShape::kThreads, CatShape::kSmem,
                        st, a, nullptr, true);
  }
  return cudaGetLastError();
}

cudaError_t launch_readonly(const CountArgs &a, unsigned long long *sink, const DevInfo &di,
                            cudaStream_t st) {
  const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
  return launch_tma(pp_tma_kernel<0>, g, kTmaThreads, kTmaSmemBytes, st, a, sink,
                    a.body_bytes < pdl_max_body());
}

// Fixed segments take the TMA ring when they tile its 64 KiB stages into at
// least one item per team warp and there are enough chunks to fill the grid;
// PP_SEG_PATH=ldg forces pp_seg_kernel (A/B runs, tests).
static bool seg_use_tma(const SegArgs &a, const DevInfo &di, unsigned *items_per_chunk) {
  static const char *path = std::getenv("PP_SEG_PATH");
  if (path && std::strcmp(path, "ldg") == 0) return false;
  const bool force = path && std::strcmp(path, "tma") == 0;
  if (a.seg_off || a.seg_bytes == 0 || (a.seg_bytes & 15) || ((uintptr_t)a.base & 15)) return false;
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

cudaError_t launch_segmented(const SegArgs &a, const DevInfo &di, cudaStream_t st) {
  if (a.nseg == 0) return cudaSuccess;
  const int G = a.lanes_per_segment;
  if (G == 1) {  // one lane per segment
    const unsigned long long need = (a.nseg + kLaneThreads - 1) / kLaneThreads;
    const unsigned g = grid_for(need, (unsigned long long)di.num_sms * di.lane_blocks_per_sm);
    if (a.seg_off)
      pp_seglane_kernel<false><<<g, kLaneThreads, 0, st>>>(a);
    else
      pp_seglane_kernel<true><<<g, kLaneThreads, 0, st>>>(a);
    return cudaGetLastError();
  }
  unsigned ipc = 0;
  if (seg_use_tma(a, di, &ipc)) {
    const unsigned long long chunks =
        (a.nseg + (unsigned long long)ipc * (32 / G) - 1) / ((unsigned long long)ipc * (32 / G));
    const unsigned g = grid_for(chunks, (unsigned long long)di.num_sms);
    if (G == 8)
      pp_segtma_kernel<8><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(a, ipc);
    else if (G == 16)
      pp_segtma_kernel<16><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(a, ipc);
    else
      pp_segtma_kernel<32><<<g, kSegTmaThreads, kSegTmaSmem, st>>>(a, ipc);
    return cudaGetLastError();
  }
  const unsigned long long segs_per_block = (kSegThreads / 32) * (32 / G);
  const unsigned long long need = (a.nseg + segs_per_block - 1) / segs_per_block;
  const unsigned g = grid_for(need, (unsigned long long)di.num_sms * di.seg_blocks_per_sm);
  if (G == 8)
    pp_seg_kernel<8><<<g, kSegThreads, 0, st>>>(a);
  else if (G == 16)
    pp_seg_kernel<16><<<g, kSegThreads, 0, st>>>(a);
  else
    pp_seg_kernel<32><<<g, kSegThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace pp
