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
// The fused one-hot producer (pp_count_categories on u8 codes) and the
// read-only roofline kernel are modes of the same TMA kernel.  Segmented
// (many-array) counting lives in pp_segmented.cu.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>

#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

#ifndef PP_TIMELINE
#define PP_TIMELINE 0
#endif
#ifndef PP_TMA_NCW
#define PP_TMA_NCW 8
#endif
constexpr int kTmaConsumerWarps = PP_TMA_NCW;
constexpr int kSchedSlotsAlloc = 256;  // = kSchedSlots (scheduler slots per device)
#ifndef PP_TMA_STAGES
#define PP_TMA_STAGES 3
#endif
constexpr int kTmaStages = PP_TMA_STAGES;  // 3 x 32 KiB: best of the scripts/bw_probe.cu sweep (profiles/)
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
constexpr int kTmaStageVecs = kTmaConsumerWarps * 32 * 8;  // 2048 x 16 B = 32 KiB
constexpr unsigned long long kTmaStageBytes = kTmaStageVecs * 16ull;
constexpr size_t kTmaSmemBytes = kTmaStages * kTmaStageBytes + 2 * kTmaStages * 8;

#ifndef PP_CAT_STAGES
#define PP_CAT_STAGES 3
#endif
// Shape of the TMA pipeline for NCW consumer warps (8 vectors per thread per
// stage).  The counting kernel uses 8 warps; the fused one-hot producer does
// ~4x more ALU work per byte and uses more consumer warps.
template <int NCW>
struct TmaShape {
  static constexpr int kThreads = (NCW + 1) * 32;
  static constexpr int kStageVecs = NCW * 32 * 8;
  static constexpr unsigned long long kStageBytes = kStageVecs * 16ull;
  // ring depth: the counting kernel's is tunable (A/B), the fused producer's
  // 64 KiB stages allow three
  static constexpr int kStages = NCW == kTmaConsumerWarps ? kTmaStages : PP_CAT_STAGES;
  static constexpr size_t kSmem = kStages * kStageBytes + 2 * kStages * 8;
};
#ifndef PP_CAT_NCW
#define PP_CAT_NCW 16
#endif
using CatShape = TmaShape<PP_CAT_NCW>;

// One-hot words from a shared-memory table (u8 codes at W = 32 / 64): for a
// static share of the codes of a chunk -- PP_CAT_TAB64 of every 16 at W = 64,
// PP_CAT_TAB32 of every 32 at W = 32; 0 = off -- the one-hot word (pair) is
// LOADED from a per-lane table -- entry c of lane l at (c * 32 + l) * E
// bytes, E = 8 / 4: every lane has its own banks, so the loads are
// conflict-free whatever the codes; entries c >= W are zero, so large codes
// and absent slots (0xFF) vanish -- at an address made by one IMAD, instead
// of being computed on the ALU pipe (two shifts / one BMSK).  The counter's
// LOP3s keep more of the ALU pipe and the LSU / FMA pipes, mostly idle
// otherwise, carry part of the one-hot step; the share balances the ALU
// pipe against the shared-memory data pipe (one wavefront per clock: the
// codes' LDS.U8 1, LDS.64 2, LDS.32 1 per 32 codes).  W = 64 (ALU 3.1 - 1.0 f
// vs LSU 1 + 2 f clocks per 32 codes per SM): 0 / 6 / 8 / 10 / 11 / 12 / 14 /
// 16 of 16 = 2806 / 3113 / 3196 / 3280 / 3291 / 3204 / 2992 / 2803 G codes/s
// (scripts/gpu_cat_tab.sh); its 64 KiB table takes the third stage's shared
// memory, so it runs a 2-stage ring (no loss at 3.3 TB/s).  W = 32: 0 / 5 /
// 7 / 9 / 11 / 13 of 32 = 5293 / 5370 / 5470 / 5570 / 5533 / 5494
// (scripts/gpu_cat_tab32.sh); the 32 KiB table fits beside the 3-stage ring
// once the epilogue's per-warp rows move into the ring (with a 2-stage ring
// the same table gained 1.3 % only: the ring depth costs 2 % at 5.3 TB/s).
// W = 16 (two codes per word, the same 32-bit table; PP_CAT_TAB16 of every
// 64 codes): 0 / 6 / 10 / 14 / 18 / 24 = 6207 / 6277 / 6318 / 6241 / 6112 /
// 5756 (scripts/gpu_cat_tab16.sh) -- a small gain, the kernel is within 15 %
// of the HBM roofline there.
#ifndef PP_CAT_TAB64
#define PP_CAT_TAB64 11
#endif
#ifndef PP_CAT_TAB32
#define PP_CAT_TAB32 9
#endif
#ifndef PP_CAT_TAB16
#define PP_CAT_TAB16 10
#endif
template <int MODE, int NCW, int CB>
struct KShape {
  using Sh = TmaShape<NCW>;
  static constexpr int kTabEntry = (CB == 1 && MODE == 64 && PP_CAT_TAB64 > 0)   ? 8
                                   : (CB == 1 && MODE == 32 && PP_CAT_TAB32 > 0) ? 4
                                   : (CB == 1 && MODE == 16 && PP_CAT_TAB16 > 0) ? 4
                                                                                 : 0;
  static constexpr int kTabBytes = 256 * 32 * kTabEntry;
  // the ring keeps its depth when the table fits beside it (W = 32: 192 + 32
  // KiB, the epilogue's per-warp rows then live in the ring's last stage),
  // else it gives up a stage (W = 64)
  static constexpr bool kFits =
      Sh::kStages * Sh::kStageBytes + 2 * Sh::kStages * 8 + 16 + kTabBytes + 1024 <= 227 * 1024;
  static constexpr int kStages = (kTabBytes && !kFits) ? Sh::kStages - 1 : Sh::kStages;
  // per-warp epilogue rows in the stage that carried the "no chunk" sentinel
  static constexpr bool kRowsInStage = kTabBytes != 0;
  static constexpr size_t kBarOff = kStages * Sh::kStageBytes;
  static constexpr size_t kTabOff = (kBarOff + 2 * kStages * 8 + 15) & ~(size_t)15;
  static constexpr size_t kSmem = kTabOff + kTabBytes;
};

constexpr int kLdgWarps = 8;
constexpr int kLdgThreads = kLdgWarps * 32;
constexpr int kLdgChunkVecs = kLdgThreads * 8;
constexpr unsigned long long kLdgChunkBytes = kLdgChunkVecs * 16ull;


// Head/tail bytes (< 16 each) as one extra weight-1 plane pair, counted by
// warp 0 of CTA 0.  Lane l < 16 takes head byte l, lane 16+l tail byte l.
__device__ __forceinline__ void count_edges(Counter &c, const uint8_t *head, uint32_t hb,
                                            const uint8_t *tail, uint32_t tb, uint32_t lane,
                                            const TC &t, uintptr_t chk_lo = 0,
                                            uintptr_t chk_hi = 0) {
  const uint8_t *p = nullptr;
  if (lane < 16) {
    if (lane < hb) p = head + lane;
  } else if (lane - 16 < tb) {
    p = tail + (lane - 16);
  }
  unsigned long long fw = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // input complete (PDL)
  if (p && PP_CHK_RANGE(p, 1, chk_lo, chk_hi)) fw = (unsigned long long)__ldg(p) << frame_shift(p);
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
      if (a.nextra == 0) {
        atomicAdd(a.counters + j, s);
      } else {
        // several GPUs add into the same arrays: system scope, so the adds of
        // different devices are atomic with respect to each other (PTX memory
        // model; device scope only orders this GPU's threads)
        atomicAdd_system(a.counters + j, s);
        for (int k = 0; k < a.nextra; ++k) atomicAdd_system(a.extra[k] + j, s);
      }
    }
  }
}

// The same fold over per-warp frame rows (the TMA kernel): thread j < w sums
// rows[k][(i + rot) mod 64] over i = j (mod w) and the NCW consumer warps.
// Replaces 2 x 32 u64 shared atomicAdd per warp -- compiled as CAS loops,
// with all 8 warps contending for the same 64 words -- by plain stores.
#ifndef PP_EPI_SLOTS
#define PP_EPI_SLOTS 1
#endif
template <int NCW>
__device__ __forceinline__ void fold_rows_to_counters(const unsigned long long (*rows)[64],
                                                      const CountArgs &a) {
  const int j = threadIdx.x, width = a.width;
  if (j < width) {
    unsigned long long s = 0;
    for (int i = j; i < 64; i += width) {
      const int p = (i + a.rot) & 63;
#pragma unroll
      for (int k = 0; k < NCW; ++k) s += rows[k][p];
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // see fold_frame_to_counters
    if (s) {
      if (a.nextra == 0) {
        atomicAdd(a.counters + j, s);
      } else {
        atomicAdd_system(a.counters + j, s);
        for (int k = 0; k < a.nextra; ++k) atomicAdd_system(a.extra[k] + j, s);
      }
    }
  }
}

// ---- fused one-hot producer (pp_count_categories on u8 codes) -------------
// A code c < W becomes bit c of a one-hot word; words are packed so that the
// frame position of that bit is = c (mod W) and the epilogue is the plain
// fold with rot = 0:  W=8: four codes per word (byte k holds 1 << code_k),
// W=16: two codes per word (half k), W=32: one code per word, W=64: one code
// per (x|z = bits 0-31, y|w = bits 32-63) pair.  Codes >= W give no bit.
// u8 codes at W >= 16 are read one byte per lane from shared memory
// (eat_lds8); W = 8 and 2-/4-byte codes go through vector loads.

// 4 u8 codes -> 4 one-hot bytes.  2 ops for the nibble-packed selector (the
// LOP3 select leaves junk only in the nibbles of codes >= 8, which the mask
// clears), one PRMT against the table {1,2,4,...,128}, and -- only when a
// byte >= 8 is present -- a 5-op mask: z = (x | 0x80..) - 0x08.. has a
// byte's msb set iff that byte is in [8, 0x80) (no borrow crosses a byte),
// x's msb covers [0x80, 0xFF]; PRMT's sign-replicate mode (selector nibble
// 8|i) widens msb -> 0xFF.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t onehot8x4(uint32_t x, bool any_big) {
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
__device__ __forceinline__ uint32_t onehot32(uint32_t c) {
  uint32_t r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(c));  // c >= 32 -> 0
  return r;
}

// Expand and count 8 vectors (128 u8 codes, W = 8) of one thread; vectors
// with valid bit i clear are absent (partial last chunk) and contribute
// nothing.  FULL: every vector present (all but the last chunk).
template <bool FULL, class Ctr>
__device__ __forceinline__ void eat_codes8(Ctr &c, const uint4 (&v)[8], uint32_t valid,
                                           const TC &t) {
  uint4 u[8];
  // Does any code of the warp's chunk need the >= 8 mask?  One warp-uniform
  // branch per chunk: a per-vector test compiled to predicated mask code
  // that was issued for every word whether needed or not (2.95 ALU lane-ops
  // per code with or without large codes); categories that all fit the
  // width -- the usual case -- now skip it.
  uint32_t any = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) any |= v[i].x | v[i].y | v[i].z | v[i].w;
  if (__any_sync(0xFFFFFFFFu, (any & 0xF8F8F8F8u) != 0)) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      u[i] = make_uint4(onehot8x4(v[i].x, true), onehot8x4(v[i].y, true),
                        onehot8x4(v[i].z, true), onehot8x4(v[i].w, true));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      u[i] = make_uint4(onehot8x4(v[i].x, false), onehot8x4(v[i].y, false),
                        onehot8x4(v[i].z, false), onehot8x4(v[i].w, false));
  }
  if (!FULL) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (!((valid >> i) & 1u)) u[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  c.csa(u, 0);
  c.end_chunk(t);
}

// eat8 groups per chunk of one thread (8 vectors of CB-byte codes): the
// one-hot words of 128 / CB codes, W / 32 words per code (W = 8: four codes
// per word, 16: two), 32 words per group
template <int W, int CB>
constexpr int groups_per_chunk() {
  return CB == 1 ? W / 8 : CB == 2 ? (W <= 16 ? 1 : W == 32 ? 2 : 4) : (W <= 32 ? 1 : 2);
}
// the fused producer's counter: one tree at W <= 32, two at W = 64
template <int W, int CB>
using CatCtr = CatCounter<W == 64 ? 2 : 1, (W == 64 ? 1 : 2) * groups_per_chunk<W, CB>()>;

// 2-byte codes at W = 64 (the one wide-code case that is ALU-bound), the
// same way: LDS.U16 puts each code alone in a register, `1 << c` is one
// 64-bit shift (amounts >= 64 give 0, so negative / large codes vanish).
// Warp w owns 4 KiB of the stage = 64 codes per lane; code slot j of a lane
// sits at code index 32 * j + lane.  !FULL: slots at or past `lim` (codes of
// this warp's slice that exist) are no code.
template <bool FULL, class Ctr>
__device__ __forceinline__ void eat_lds16_w64(Ctr &c, const uint16_t *sb, int lim, const TC &t) {
  auto code = [&](int j) -> uint32_t {
    if (FULL) return sb[32 * j];
    return (32 * j < lim) ? (uint32_t)sb[32 * j] : 0xFFFFu;
  };
#pragma unroll
  for (int g = 0; g < 4; ++g) {  // 4 groups of 16 codes (32 words)
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t l0, h0, l1, h1;
      onehot64(code(16 * g + 2 * q), l0, h0);
      onehot64(code(16 * g + 2 * q + 1), l1, h1);
      u[q] = make_uint4(l0, h0, l1, h1);
    }
    c.csa(u, g);
  }
  c.end_chunk(t);
}

// 2- / 4-byte codes (CB = code bytes): the same packed one-hot words, built
// from wider lanes.  shl clamps any shift amount >= the register width to a
// zero result, so codes >= W need no test however large they are; the
// byte/half masks drop the rest.  Words of absent vectors (partial chunk)
// must be zero, not "code 0".
__device__ __forceinline__ uint32_t shl32(uint32_t x, uint32_t n) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}
// codes c0..c3 -> byte k = one-hot8(c_k) (c_k < 8)
__device__ __forceinline__ uint32_t oh8quad(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  return (shl32(1u, c0) & 0xFFu) | (shl32(0x100u, c1) & 0xFF00u) |
         (shl32(0x10000u, c2) & 0xFF0000u) | shl32(0x1000000u, c3);
}
// codes c0, c1 -> half k = one-hot16(c_k) (c_k < 16)
__device__ __forceinline__ uint32_t oh16pair(uint32_t c0, uint32_t c1) {
  return (shl32(1u, c0) & 0xFFFFu) | shl32(0x10000u, c1);
}

// u8 codes read one byte per lane straight from the shared-memory stage
// (W = 16 / 32 / 64): LDS.U8 puts each code alone in a
// register, so `shl` (which clamps amounts >= 32 to a zero result) makes
// the one-hot word with no byte extraction and no range test, and no vote
// for a small-code path -- the extraction moves from the ALU/FMA pipes to
// the LSU.  Warp w owns bytes [w * 4096, (w + 1) * 4096) of the stage; its
// j-th load reads 32 consecutive bytes (conflict-free).  Code slot j of a
// lane sits at byte 32 * j + lane: any assignment works, the counts are a
// histogram.  !FULL: slots at or past `lim` (bytes of this warp's slice
// that hold codes) are no code.
// 1 << n, 0 for n >= 32: one BMSK (a 1-bit mask at position n, clamped),
// no register holding the constant 1 as `shl` needs
__device__ __forceinline__ uint32_t bit_at(uint32_t n) {
  uint32_t r;
  asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(r) : "r"(n));
  return r;
}
// table entry of code c for this lane (tab = shared address of the lane's
// column, mul = bytes per table row, a kernel argument so that the address
// is one IMAD on the FMA pipe and not shifts/adds on the ALU pipe)
__device__ __forceinline__ uint32_t tab_load32(uint32_t c, uint32_t mul, uint32_t tab) {
  uint32_t addr, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(c), "r"(mul), "r"(tab));
  asm("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void tab_load64(uint32_t c, uint32_t mul, uint32_t tab, uint32_t &lo,
                                           uint32_t &hi) {
  uint32_t addr;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(c), "r"(mul), "r"(tab));
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(addr));
}
// slot k of every n takes the table path when this is true: `share` of n, spread evenly
__host__ __device__ constexpr bool tab_slot(int k, int n, int share) {
  return ((k + 1) * share / n) != (k * share / n);
}
template <int W, bool FULL, class Ctr>
__device__ __forceinline__ void eat_lds8(Ctr &c, const uint8_t *sb, int lim, const TC &t,
                                         uint32_t tab, uint32_t mul) {
  auto code = [&](int j) -> uint32_t {
    const int pos = 32 * j;  // + lane (sb is this lane's base)
    if (FULL) return sb[pos];
    return (pos < lim) ? (uint32_t)sb[pos] : 0xFFu;
  };
  if (W == 32) {  // one word per code: 4 groups of 32
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = 32 * g + 4 * q;
        uint32_t wq[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          wq[e] = tab_slot(4 * q + e, 32, PP_CAT_TAB32) ? tab_load32(code(j + e), mul, tab)
                                                        : bit_at(code(j + e));
        u[q] = make_uint4(wq[0], wq[1], wq[2], wq[3]);
      }
      c.csa(u, g);
    }
  } else if (W == 64) {  // (lo, hi) per code: 8 groups of 16
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t l[2], h[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t ce = code(16 * g + 2 * q + e);
          if (tab_slot(2 * q + e, 16, PP_CAT_TAB64))
            tab_load64(ce, mul, tab, l[e], h[e]);
          else  // 1 << c as a 64-bit shift: two SHF (the clamp makes c >= 64 vanish)
            onehot64(ce, l[e], h[e]);
        }
        u[q] = make_uint4(l[0], h[0], l[1], h[1]);
      }
      c.csa(u, g);
    }
  } else {  // W == 16: two codes per word, 2 groups of 32 words
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t wq[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = 64 * g + 8 * q + 2 * e;
          // low halves of the two one-hot words (codes 16..31 fall in the
          // dropped high halves): one PRMT
          const uint32_t b0 = tab_slot(8 * q + 2 * e, 64, PP_CAT_TAB16)
                                  ? tab_load32(code(j), mul, tab) : bit_at(code(j));
          const uint32_t b1 = tab_slot(8 * q + 2 * e + 1, 64, PP_CAT_TAB16)
                                  ? tab_load32(code(j + 1), mul, tab) : bit_at(code(j + 1));
          wq[e] = prmt(b0, b1, 0x5410u);
        }
        u[q] = make_uint4(wq[0], wq[1], wq[2], wq[3]);
      }
      c.csa(u, g);
    }
  }
  c.end_chunk(t);
}

template <int W, bool FULL, int CB, class Ctr>
__device__ __forceinline__ void eat_wide_codes(Ctr &c, const uint4 (&v)[8], uint32_t valid,
                                               const TC &t) {
  static_assert(CB == 2 || CB == 4, "code bytes");
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  // this thread's K codes, in order: vector i holds 16 / CB of them
  constexpr int K = 8 * 16 / CB;
  auto code = [&](int k) -> uint32_t {
    const uint4 x = v[k / (16 / CB)];
    const int j = k % (16 / CB);
    const uint32_t wd = (CB == 4) ? (j == 0 ? x.x : j == 1 ? x.y : j == 2 ? x.z : x.w)
                                  : (j / 2 == 0 ? x.x : j / 2 == 1 ? x.y : j / 2 == 2 ? x.z : x.w);
    return CB == 4 ? wd : (j & 1 ? wd >> 16 : wd & 0xFFFFu);
  };
  auto present = [&](int k) -> bool { return FULL || ((valid >> (k / (16 / CB))) & 1u); };
  if (W == 32) {  // one word per code: K / 32 rounds
#pragma unroll
    for (int r = 0; r < K / 32; ++r) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = 32 * r + 4 * q;
        u[q] = present(k) ? make_uint4(shl32(1u, code(k)), shl32(1u, code(k + 1)),
                                       shl32(1u, code(k + 2)), shl32(1u, code(k + 3)))
                          : z4;
      }
      c.csa(u, r);
    }
  } else if (W == 64) {  // one (lo, hi) pair per code: K / 16 rounds
#pragma unroll
    for (int r = 0; r < K / 16; ++r) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = 16 * r + 2 * q;
        uint32_t l0, h0, l1, h1;
        onehot64(code(k), l0, h0);
        onehot64(code(k + 1), l1, h1);
        u[q] = present(k) ? make_uint4(l0, h0, l1, h1) : z4;
      }
      c.csa(u, r);
    }
  } else {  // W = 16: two codes per word, W = 8: four; one round, padded
    constexpr int PER = W == 16 ? 2 : 4;
    constexpr int NW = K / PER;  // packed words (<= 32)
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t wq[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int n = 4 * q + e;  // packed word index
        const int k = PER * n;
        if (n >= NW || !present(k)) {
          wq[e] = 0u;
        } else if (W == 16) {
          wq[e] = oh16pair(code(k), code(k + 1));
        } else {
          wq[e] = oh8quad(code(k), code(k + 1), code(k + 2), code(k + 3));
        }
      }
      u[q] = make_uint4(wq[0], wq[1], wq[2], wq[3]);
    }
    c.csa(u, 0);
  }
  c.end_chunk(t);
}

// The same split in two for the TMA kernel, whose warp 0 of CTA 0 loads its
// head/tail byte (or code) BEFORE streaming, so the ~1 us global-load
// latency is not added after the last chunk (C4, 64 MiB at offset 3:
// 10.7 -> 8 us per launch).  CB = 0: raw bytes (positional count), else
// CB-byte category codes (0xFFFFFFFF = no code).
template <int CB>
__device__ __forceinline__ uint64_t edge_load(const CountArgs &a, uint32_t lane) {
  const uint32_t unit = CB ? CB : 1;
  const uint8_t *p = nullptr;
  if (lane < 16) {
    if (lane < a.head_bytes / unit) p = a.head + unit * lane;
  } else if (lane - 16 < a.tail_bytes / unit) {
    p = a.tail + unit * (lane - 16);
  }
  if (!a.input_ready) asm volatile("griddepcontrol.wait;" ::: "memory");  // input complete (PDL)
  if (p && !PP_CHK_RANGE(p, unit, a.chk_lo, a.chk_hi)) p = nullptr;
  if (CB == 0) return p ? (uint64_t)__ldg(p) << frame_shift(p) : 0ull;
  if (!p) return 0xFFFFFFFFull;
  return CB == 1 ? __ldg(p)
                 : CB == 2 ? __ldg(reinterpret_cast<const uint16_t *>(p))
                           : __ldg(reinterpret_cast<const uint32_t *>(p));
}
template <int CB, class Ctr>
__device__ __forceinline__ void edge_count(Ctr &c, uint64_t v, int width, const TC &t) {
  if (CB == 0) {  // v = the byte, already placed at its frame position
    c.ce += wcount((uint32_t)v, t);
    c.co += wcount((uint32_t)(v >> 32), t);
  } else {  // v = a code: frame position = code
    const uint32_t code = (uint32_t)v;
    const bool ok = code < (uint32_t)width;
    c.ce += wcount(ok ? onehot32(code) : 0u, t);
    c.co += wcount(ok ? onehot32(code - 32u) : 0u, t);
  }
}

// PP_TIMELINE (diagnostic builds only, scripts/timeline.py): %globaltimer
// stamps per CTA of the counting kernel -- entry, first copy issued, first
// stage consumed, last copy issued, last chunk consumed, epilogue start, end.
#if PP_TIMELINE
__device__ unsigned long long pp_tl[1024][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PP_TL(k)                                                   \
  do {                                                             \
    if (MODE == 1 && blockIdx.x < 1024) pp_tl[blockIdx.x][k] = gtime(); \
  } while (0)
#else
#define PP_TL(k) \
  do {           \
  } while (0)
#endif

// MODE 0: read-only roofline (XOR of every word), MODE 1: positional count,
// MODE 8/16/32/64: fused one-hot producer over CB-byte codes at that width.
template <int MODE, int NCW = kTmaConsumerWarps, int CB = 1>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    pp_tma_kernel(CountArgs a, unsigned long long *sink) {
  constexpr bool kCount = MODE != 0;
  using Sh = TmaShape<NCW>;
  using KS = KShape<MODE, NCW, CB>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint4 *stages = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + KS::kBarOff);
  uint64_t *empty = full + KS::kStages;
  __shared__ unsigned long long frame[PP_EPI_SLOTS ? 1 : 64];
  // per-warp frame rows of the epilogue; kernels whose table leaves no room
  // keep them in the ring's stage that carried the sentinel instead (free by
  // then: every warp released it before the producer could reuse it, and no
  // copy is issued after the sentinel)
  __shared__ unsigned long long wframe[(PP_EPI_SLOTS && !KS::kRowsInStage) ? NCW : 1][64];
  unsigned long long (*rows)[64] = wframe;
  __shared__ unsigned long long chunk_id[KS::kStages];  // written before the stage's arrival

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    PP_TL(0);
    for (int s = 0; s < KS::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  if (!PP_EPI_SLOTS && threadIdx.x < 64) frame[threadIdx.x] = 0;
  if constexpr (KS::kTabBytes != 0) {  // per-lane one-hot tables (see KShape)
    for (uint32_t i = threadIdx.x; i < 256u * 32u; i += (NCW + 1) * 32) {
      // entry i / 32, lane i % 32
      if constexpr (KS::kTabEntry == 8) {
        uint32_t lo, hi;
        onehot64(i >> 5, lo, hi);
        reinterpret_cast<uint2 *>(smem + KS::kTabOff)[i] = make_uint2(lo, hi);
      } else {
        reinterpret_cast<uint32_t *>(smem + KS::kTabOff)[i] = onehot32(i >> 5);
      }
    }
  }
  __syncthreads();

  const unsigned long long nchunks = a.nchunks;
  if (warp == NCW) {
    // ---------------- producer: one elected thread issues bulk copies
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // programmatic dependent launch: everything above overlapped the
      // previous grid's tail; its outputs (possibly our input) are complete
      // and visible only after this wait.  With input_ready the caller
      // vouches that the previous grid does not write the input: the copies
      // start at once, and only the first ticket draw (the previous launch
      // on this stream may share the ticket counter) waits.
      bool waited = !a.input_ready;
      bool triggered = a.early_trigger != 0;
      if (triggered) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      if (waited) asm volatile("griddepcontrol.wait;" ::: "memory");
      PP_TL(1);
      uint32_t stage = 0, phase = 0;
      // chunk sequence: the static grid stride (blockIdx.x + j * gridDim.x),
      // for ticketed launches only the first a.lead chunks, then ticket t of
      // the stream's counter = chunk a.lead * gridDim.x + t, so every CTA
      // finishes within about one chunk of the others
      unsigned long long ch = blockIdx.x;
      uint32_t issued = 0;  // chunks this CTA has issued
      for (;;) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (ch >= nchunks) {  // tell the consumers to stop: no bytes, one arrival
          chunk_id[stage] = kNoChunk;
          mbar_arrive(&full[stage]);
          break;
        }
        chunk_id[stage] = ch;
        const unsigned long long off = ch * Sh::kStageBytes;
        const unsigned long long rem = a.body_bytes - off;
        const uint32_t bytes = (uint32_t)(rem < Sh::kStageBytes ? rem : Sh::kStageBytes);
        if (PP_CHK(stage < (uint32_t)KS::kStages) &&
            PP_CHK_RANGE(a.body + off, bytes, a.chk_lo, a.chk_hi)) {
          mbar_arrive_expect_tx(&full[stage], bytes);
          bulk_g2s(stages + stage * Sh::kStageVecs, a.body + off, bytes, &full[stage], pol);
        } else {  // checked build, failed check: no copy, the stage completes empty
          mbar_arrive(&full[stage]);
        }
        // the first a.lead chunks of every CTA are static (blockIdx.x +
        // j * gridDim.x): a whole ring's worth can be issued before the
        // first ticket, i.e. (with input_ready) while the previous launch on
        // the stream still drains; tickets number the chunks after those
        if (a.sched && ++issued >= a.lead) {
          if (!waited) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
          }
          ch = (unsigned long long)a.lead * gridDim.x +
               (unsigned long long)(atomicAdd(a.sched, 1u) - a.sched_base);
          // tickets are drawn in order across the grid: once they reach the
          // last trigger_tail chunks per CTA, let the next launch on the
          // stream become resident and fill its ring (A/B: PP_TRIGGER_TAIL)
          if (!triggered && ch + (unsigned long long)a.trigger_tail * gridDim.x >= nchunks) {
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            triggered = true;
          }
        } else {
          ch += gridDim.x;
        }
        if (++stage == KS::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      PP_TL(3);
      // every load of this CTA is in flight: the next launch on the stream
      // (programmatic dependent launch) may start filling its own ring
      if (!triggered) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
  } else {
    // ---------------- consumers
    const TC t = make_tc(lane);
    // the fused producer batches a chunk's a16 planes (CatCounter); the
    // positional count keeps one eat8 per chunk (Counter)
    using Ctr = typename std::conditional<(MODE >= 8), CatCtr<(MODE >= 8 ? MODE : 8), CB>,
                                          Counter>::type;
    Ctr c;
    c.init();
    uint32_t xs = 0;  // read-only roofline accumulator
    constexpr int kEdgeCB = MODE == 1 ? 0 : CB;
    uint64_t edge = 0;  // warp 0 of CTA 0: its head/tail byte or code, loaded up front
    if (kCount && blockIdx.x == 0 && warp == 0) edge = edge_load<kEdgeCB>(a, lane);
    uint32_t stage = 0, phase = 0;
    const uint32_t tid = threadIdx.x;
#if PP_CHECK_BOUNDS
    unsigned long long prev_ch = 0, seen = 0;
#endif
    for (bool first = true;; first = false) {
      mbar_wait(&full[stage], phase);
      const unsigned long long ch = chunk_id[stage];
      if (ch == kNoChunk) break;
#if PP_CHECK_BOUNDS
      // chunk ids: in range, strictly increasing per CTA (static stride and
      // scheduler tickets both increase); a skipped or repeated ring phase
      // shows up here or in the grid-wide total below
      PP_CHK(ch < nchunks && (first || ch > prev_ch));
      prev_ch = ch;
      ++seen;
#endif
      if (first && threadIdx.x == 0) PP_TL(2);
      const uint4 *sv = stages + stage * Sh::kStageVecs;
      if constexpr (CB == 2 && MODE == 64) {
        // 2-byte codes at W = 64: one code per lane from the stage
        constexpr int kSlice = (int)(Sh::kStageBytes / NCW);  // bytes per warp
        static_assert(kSlice == 2 * 32 * 64, "eat_lds16_w64 expects 64 codes per lane");
        const uint16_t *sb =
            reinterpret_cast<const uint16_t *>(reinterpret_cast<const uint8_t *>(sv) +
                                               warp * kSlice) + lane;
        const unsigned long long rem = a.body_bytes - ch * Sh::kStageBytes;
        if (rem >= Sh::kStageBytes) {
          eat_lds16_w64<true>(c, sb, 0, t);
        } else {
          const long long lim = ((long long)rem - (long long)warp * kSlice) / 2 - (long long)lane;
          eat_lds16_w64<false>(c, sb, (int)(lim < 0 ? 0 : lim > kSlice / 2 ? kSlice / 2 : lim), t);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == KS::kStages) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      if constexpr (CB == 1 && (MODE == 16 || MODE == 32 || MODE == 64)) {
        // u8 codes straight from the stage, one byte per lane (eat_lds8);
        // the stage is released after the chunk is counted
        constexpr int kSlice = (int)(Sh::kStageBytes / NCW);  // bytes per warp = 128 per lane
        static_assert(kSlice == 32 * 128, "eat_lds8 expects 128 codes per lane");
        const uint8_t *sb = reinterpret_cast<const uint8_t *>(sv) + warp * kSlice + lane;
        const unsigned long long rem = a.body_bytes - ch * Sh::kStageBytes;
        PP_CHK(stage < (uint32_t)KS::kStages);
        const uint32_t tab =
            (uint32_t)__cvta_generic_to_shared(smem + KS::kTabOff) + lane * KS::kTabEntry;
        if (rem >= Sh::kStageBytes) {
          eat_lds8<MODE, true>(c, sb, 0, t, tab, a.tab_mul);
        } else {
          const long long lim = (long long)rem - (long long)warp * kSlice - (long long)lane;
          eat_lds8<MODE, false>(c, sb, (int)(lim < 0 ? 0 : lim > kSlice ? kSlice : lim), t, tab,
                                a.tab_mul);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == KS::kStages) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      uint4 v[8];
      uint32_t valid = 0xFFu;  // vectors present in this (possibly partial) chunk
      const unsigned long long off = ch * Sh::kStageBytes;
      const unsigned long long rem = a.body_bytes - off;
      if (rem >= Sh::kStageBytes) {
        PP_CHK(stage < (uint32_t)KS::kStages && tid + 7 * (NCW * 32) < (uint32_t)Sh::kStageVecs);
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
      if constexpr (MODE == 1) {
        c.eat8(v, t);
      } else if constexpr (MODE == 8 && CB == 1) {
        if (valid == 0xFFu)
          eat_codes8<true>(c, v, valid, t);
        else
          eat_codes8<false>(c, v, valid, t);
      } else if constexpr (MODE >= 8 && CB > 1 && !(CB == 2 && MODE == 64)) {
        if (valid == 0xFFu)
          eat_wide_codes<MODE, true, CB>(c, v, valid, t);
        else
          eat_wide_codes<MODE, false, CB>(c, v, valid, t);
      } else if constexpr (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) xs ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
      }  // (u8 codes at W >= 16 took the eat_lds8 path above)
      if (++stage == KS::kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
#if PP_CHECK_BOUNDS
    if (threadIdx.x == 0 && a.chk_ctr) {  // this CTA's chunks, then the grid-wide total
      atomicAdd(a.chk_ctr, seen);
      __threadfence();
      if (atomicAdd(a.chk_ctr + 1, 1ull) == gridDim.x - 1ull) {
        const unsigned long long tot = atomicAdd(a.chk_ctr, 0ull);
        if (tot != nchunks) chk_fail(__LINE__, tot, nchunks, nchunks);
      }
    }
#endif
    if (kCount) {
      if (threadIdx.x == 0) PP_TL(4);
      c.finish(t);
      if (blockIdx.x == 0 && warp == 0) edge_count<kEdgeCB>(c, edge, a.width, t);
      if (KS::kRowsInStage)
        rows = reinterpret_cast<unsigned long long(*)[64]>(stages + stage * Sh::kStageVecs);
      if (PP_EPI_SLOTS) {  // one row per warp: plain stores, summed by the fold
        rows[warp][lane] = c.ce;
        rows[warp][32 + lane] = c.co;
      } else {  // u64 shared atomics (a CAS loop in SASS, 8 warps contending)
        atomicAdd(&frame[lane], c.ce);
        atomicAdd(&frame[32 + lane], c.co);
      }
    } else {
      xs = __reduce_xor_sync(FULL, xs);
      if (lane == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        atomicXor(sink, (unsigned long long)xs);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) PP_TL(5);
  if (kCount) {
    if (PP_EPI_SLOTS)
      fold_rows_to_counters<NCW>(rows, a);  // (threads < 64 are consumers: their `rows`)
    else
      fold_frame_to_counters(frame, a);
  }
  if (threadIdx.x == 0) PP_TL(6);
}

// One CTA's grid-stride pass over the body's chunks (chunk cta, cta + ncta, ...).
__device__ __forceinline__ void ldg_eat_chunks(Counter &c, const CountArgs &a, const TC &t,
                                               unsigned long long cta, unsigned long long ncta) {
  const uint4 *body = reinterpret_cast<const uint4 *>(a.body);
  const unsigned long long nvec = a.body_bytes >> 4;
  for (unsigned long long ch = cta; ch < a.nchunks; ch += ncta) {
    const unsigned long long base = ch * kLdgChunkVecs + threadIdx.x;
    uint4 v[8];
    if ((ch + 1) * kLdgChunkVecs <= nvec) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = PP_CHK_RANGE(body + base + i * kLdgThreads, 16, a.chk_lo, a.chk_hi)
                   ? ldg_stream(body + base + i * kLdgThreads)
                   : make_uint4(0u, 0u, 0u, 0u);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const unsigned long long idx = base + i * kLdgThreads;
        v[i] = idx < nvec && PP_CHK_RANGE(body + idx, 16, a.chk_lo, a.chk_hi)
                   ? ldg_stream(body + idx)
                   : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    c.eat8(v, t);
  }
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
  ldg_eat_chunks(c, a, t, blockIdx.x, gridDim.x);
  c.finish(t);
  if (blockIdx.x == 0 && warp == 0)
    count_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, t, a.chk_lo, a.chk_hi);
  atomicAdd(&frame[lane], c.ce);
  atomicAdd(&frame[32 + lane], c.co);
  __syncthreads();
  fold_frame_to_counters(frame, a);
}

// Small synchronous calls (pp_count_sync, small pp_count_host): ONE CTA counts
// the whole range -- device memory, or host memory it reads over the link
// through its mapped pinned address -- and publishes the result itself:
// out[j] = count of position j (plain stores into mapped pinned host memory,
// not accumulated), then *flag = seq.  The host polls the flag instead of
// queueing a counter memset, a D2H copy and a stream synchronisation.
__global__ void __launch_bounds__(kLdgThreads)
    pp_count_direct_kernel(CountArgs a, unsigned long long *out, unsigned int *flag,
                           unsigned int seq) {
  __shared__ unsigned long long frame[64];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) frame[threadIdx.x] = 0;
  __syncthreads();
  const TC t = make_tc(lane);
  Counter c;
  c.init();
  ldg_eat_chunks(c, a, t, 0, 1);
  c.finish(t);
  if (warp == 0)
    count_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, t, a.chk_lo, a.chk_hi);
  atomicAdd(&frame[lane], c.ce);
  atomicAdd(&frame[32 + lane], c.co);
  __syncthreads();
  const int j = threadIdx.x, width = a.width;
  if (j < width) {
    unsigned long long s = 0;
    for (int i = j; i < 64; i += width) s += frame[(i + a.rot) & 63];
    *reinterpret_cast<volatile unsigned long long *>(out + j) = s;
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // every out[] store is ordered before the flag
    __threadfence_system();
    *reinterpret_cast<volatile unsigned int *>(flag) = seq;
  }
}

// The same publish for ranges of several chunks: one CTA per 32 KiB chunk
// (grid-stride beyond the grid), every CTA adds its folded counts into the
// zeroed device scratch acc[0..63]; the CTA that draws the last ticket
// (acc[64]) moves the totals to out[], leaves the scratch zeroed for the
// next call and writes the flag.
__global__ void __launch_bounds__(kLdgThreads)
    pp_count_direct_multi_kernel(CountArgs a, unsigned long long *acc, unsigned long long *out,
                                 unsigned int *flag, unsigned int seq) {
  __shared__ unsigned long long frame[64];
  __shared__ int last;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) frame[threadIdx.x] = 0;
  __syncthreads();
  const TC t = make_tc(lane);
  Counter c;
  c.init();
  ldg_eat_chunks(c, a, t, blockIdx.x, gridDim.x);
  c.finish(t);
  if (blockIdx.x == 0 && warp == 0)
    count_edges(c, a.head, a.head_bytes, a.tail, a.tail_bytes, lane, t, a.chk_lo, a.chk_hi);
  atomicAdd(&frame[lane], c.ce);
  atomicAdd(&frame[32 + lane], c.co);
  __syncthreads();
  const int j = threadIdx.x, width = a.width;
  if (j < width) {
    unsigned long long s = 0;
    for (int i = j; i < 64; i += width) s += frame[(i + a.rot) & 63];
    if (s) atomicAdd(acc + j, s);
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(acc + 64, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (j < width) {
    const unsigned long long v = atomicExch(acc + j, 0ull);
    *reinterpret_cast<volatile unsigned long long *>(out + j) = v;
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    acc[64] = 0;  // the next launch on any stream of this thread starts from zero
    __threadfence_system();
    *reinterpret_cast<volatile unsigned int *>(flag) = seq;
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
  a->chk_lo = (uintptr_t)data;  // the caller's range, before any corruption (checked builds)
  a->chk_hi = (uintptr_t)data + nbytes;
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
#define PP_CAT_ATTR(W, CB)                                                              \
  if ((e = cudaFuncSetAttribute(pp_tma_kernel<W, PP_CAT_NCW, CB>,                        \
                                cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                (int)KShape<W, PP_CAT_NCW, CB>::kSmem)))                 \
    return e;
  PP_CAT_ATTR(8, 1) PP_CAT_ATTR(16, 1) PP_CAT_ATTR(32, 1) PP_CAT_ATTR(64, 1)
  PP_CAT_ATTR(8, 2) PP_CAT_ATTR(16, 2) PP_CAT_ATTR(32, 2) PP_CAT_ATTR(64, 2)
  PP_CAT_ATTR(8, 4) PP_CAT_ATTR(16, 4) PP_CAT_ATTR(32, 4) PP_CAT_ATTR(64, 4)
#undef PP_CAT_ATTR
  if ((e = segmented_setup(&d))) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.ldg_blocks_per_sm,
                                                         pp_count_ldg_kernel, kLdgThreads, 0)))
    return e;
  d.ldg_blocks_per_sm = std::max(d.ldg_blocks_per_sm, 1);
  {  // SMs left free for concurrent work (e.g. NCCL kernels of a sharded job)
    const char *r = std::getenv("PP_RESERVE_SMS");
    const int reserve = r ? std::atoi(r) : 0;
    d.count_sms = (reserve > 0 && reserve < d.num_sms) ? d.num_sms - reserve : d.num_sms;
  }
  {  // dynamic scheduler slots (sched_slot), zeroed once
    const size_t bytes = kSchedSlotsAlloc * sizeof(unsigned int);
    if ((e = cudaMalloc(&d.sched, bytes))) return e;
    if ((e = cudaMemset(d.sched, 0, bytes))) return e;
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

// Launch a TMA-ring kernel, with programmatic dependent launch when `pdl`:
// launch i+1's CTAs start, set up their rings and park in
// griddepcontrol.wait while launch i drains its tail, hiding the launch gap.
// Measured (scripts/pdl_sweep.py, profiles/r1_pdl_sweep.md): 4.9 -> 3.2 us
// per 4 MiB call, 14.4 -> 13.4 us per 64 MiB; at 1 GiB it cost 1-2 % with
// the static chunk order (CTAs finishing up to 8 us apart) and gains 1 % with
// the dynamic order (148.0 -> 146.4 us), so it is on at every size.
// PP_NO_PDL=1 disables it, PP_PDL_MAX_MIB caps it (A/B runs).
static unsigned long long pdl_max_body() {
  static const unsigned long long v = [] {
    const char *e = std::getenv("PP_PDL_MAX_MIB");
    return e ? std::strtoull(e, nullptr, 10) << 20 : ~0ull;
  }();
  return v;
}

// Dynamic chunk scheduling: every stream gets its own scheduler slot (keyed
// by the stream's unique id, so a recycled handle cannot alias a live
// stream); launches on one stream are ordered, so a slot is never shared by
// two running grids.  Captured launches (a graph may be replayed on several
// streams at once) use the static order; a stream beyond kSchedSlots takes
// over a slot whose last launch has completed (sched_commit), else static.
// PP_STATIC_SCHED=1 forces the static order (A/B runs).
constexpr int kSchedSlots = kSchedSlotsAlloc;
constexpr unsigned long long kDynMinChunks = 4096;  // 128 MiB of 32 KiB chunks
struct SchedSlot {
  int idx;
  unsigned int next;  // the counter's value once every launch so far is done
  // completion of the slot's last launch (recorded by sched_commit).  It is
  // created BEFORE the slot's first hand-out, so a slot some launch has used
  // always has one; nullptr = the slot was never handed out.
  cudaEvent_t done;
  // a completion record failed: the slot's in-flight state is unknown, so it
  // is never taken over by another stream (its own stream may keep it)
  bool pinned;
};
static SchedSlot *&last_slot() {  // guarded by sched_lock()
  static SchedSlot *p = nullptr;
  return p;
}
// pp_sched_stats: {slots handed to streams, takeovers, all-busy static
// launches, dynamic launches}, all devices (guarded by sched_lock())
static unsigned long long g_sched_stats[4];

std::unique_lock<std::mutex> sched_lock() {
  static std::mutex m;
  return std::unique_lock<std::mutex>(m);
}

unsigned int *sched_slot(const DevInfo &di, cudaStream_t st, unsigned long long units,
                         unsigned int *base) {
  static const bool off = std::getenv("PP_STATIC_SCHED") != nullptr;
  last_slot() = nullptr;
  if (off || !di.sched) return nullptr;
  // an error the caller left pending must survive this function: with one
  // pending, take the static order and touch no CUDA error state at all
  if (cudaPeekAtLastError() != cudaSuccess) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone ||
      cudaStreamGetId(st, &id) != cudaSuccess) {
    cudaGetLastError();  // ours (nothing was pending)
    return nullptr;
  }
  static std::map<std::pair<unsigned int *, unsigned long long>, SchedSlot> slots;
  static std::map<unsigned int *, int> used;
  const auto key = std::make_pair(di.sched, id);
  auto it = slots.find(key);
  if (it == slots.end()) {
    int &n = used[di.sched];
    if (n < kSchedSlots) {
      it = slots.emplace(key, SchedSlot{n++, 0u, nullptr, false}).first;
      ++g_sched_stats[0];
    } else {
      // every slot of this device is taken: reuse one whose stream has no
      // launch in flight any more (its last launch's event has completed),
      // so a service that keeps creating streams does not fall back to the
      // static order for good.  The slot's counter continues from `next`.
      for (auto j = slots.begin(); j != slots.end(); ++j) {
        if (j->first.first != di.sched || j->second.pinned) continue;
        const SchedSlot sl = j->second;
        if (sl.done) {
          const cudaError_t q = cudaEventQuery(sl.done);
          if (q != cudaSuccess) {
            cudaGetLastError();  // NotReady (still running) or a fault: not free
            continue;
          }
        }
        slots.erase(j);
        it = slots.emplace(key, sl).first;
        ++g_sched_stats[1];
        break;
      }
      if (it == slots.end()) {  // all busy: static order
        ++g_sched_stats[2];
        return nullptr;
      }
    }
  }
  SchedSlot &sl = it->second;
  if (!sl.done && cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
    // without a completion event the slot could be taken over while this
    // launch runs: static order for this launch, retry the event next time
    cudaGetLastError();
    sl.done = nullptr;
    return nullptr;
  }
  *base = sl.next;
  sl.next += (unsigned int)units;  // mod 2^32, as on the device
  last_slot() = &sl;
  ++g_sched_stats[3];
  return di.sched + sl.idx;
}

// A launch that failed to enqueue draws no tickets: give its units back
// (caller still holds sched_lock(), so this is the slot just handed out).
void sched_rollback(unsigned long long units) {
  if (last_slot()) {
    last_slot()->next -= (unsigned int)units;
    --g_sched_stats[3];
  }
}

// The launch using the slot just handed out was enqueued on `st`: record
// its completion event (what a later stream checks before taking the slot).
// The event exists (sched_slot created it before the hand-out); if the
// record fails the event still shows an older, completed launch, so the
// slot is pinned to its stream instead.
void sched_commit(cudaStream_t st) {
  SchedSlot *sl = last_slot();
  if (!sl) return;
  if (!sl->done || cudaEventRecord(sl->done, st) != cudaSuccess) {
    cudaGetLastError();  // the launch itself succeeded just before: this error is ours
    sl->pinned = true;
  }
}

template <typename Kern>
static cudaError_t launch_tma(Kern kernel, unsigned grid, unsigned block, size_t smem,
                              cudaStream_t st, const CountArgs &a0, unsigned long long *sink,
                              bool want_pdl, const DevInfo &di, unsigned stages) {
  static const bool pdl_off = std::getenv("PP_NO_PDL") != nullptr;
  static const int lead_env = [] {
    const char *e = std::getenv("PP_STATIC_LEAD");  // A/B: static chunks per CTA before tickets
    return e ? std::atoi(e) : 0;
  }();
  const bool pdl = want_pdl && !pdl_off;
  CountArgs a = a0;
  // static lead: at least a ring per CTA (so, with input_ready, a whole
  // ring is in flight before the first ticket waits for the previous
  // launch), up to 16 chunks when a CTA streams >= 128 of them (1 GiB:
  // 7450 -> 7490 GB/s, scripts/gpu_lead_ab.sh; lead 8..32 equal), leaving
  // >= 7/8 of the chunks to the tickets that even out the tail
  const unsigned long long per_cta = a.nchunks / (grid ? grid : 1);
  a.lead = lead_env > 0 ? (unsigned)lead_env
                        : (unsigned)std::max<unsigned long long>(
                              stages, std::min<unsigned long long>(16, per_cta / 8));
  // every CTA's first `lead` chunks are static; tickets cover the rest, plus
  // one failing draw per CTA: the launch consumes exactly `units` tickets
  const unsigned long long static_chunks = (unsigned long long)a.lead * grid;
  const unsigned long long units =
      a.nchunks > static_chunks ? a.nchunks - static_chunks + grid : 0;
  // the dynamic order pays off once a CTA streams tens of chunks (+6 % at
  // 256 MiB, +2 % at 1 GiB); below that the static order has no tail to
  // even out and saves the slot lookup (scripts/pdl_sweep.py).  The slot's
  // base and the launch are one critical section: launches on a stream must
  // reach it in the order their bases were handed out.
  std::unique_lock<std::mutex> lk;
  static const unsigned long long dyn_min = [] {  // A/B: PP_DYN_MIN_CHUNKS
    const char *e = std::getenv("PP_DYN_MIN_CHUNKS");
    return e ? std::strtoull(e, nullptr, 10) : kDynMinChunks;
  }();
  if (a.nchunks >= dyn_min && units > 0) {
    lk = sched_lock();
    a.sched = sched_slot(di, st, units, &a.sched_base);
  }
  // Static-order launches (< 128 MiB) trigger the dependent launch at kernel
  // start: this grid (<= one CTA per SM) is fully resident by then, the next
  // grid's CTAs take the second shared-memory slot of each SM and (with
  // INPUT_READY) stream their own input while this one drains -- back-to-
  // back counts of distinct inputs overlap completely (C4 64 MiB 5650 ->
  // 7125-7200 GB/s, C1 2 MiB 1222 -> 1387-1490); without INPUT_READY they
  // only wait there (griddepcontrol.wait).  Ticketed launches trigger after
  // each CTA's last load, as before: their successor cannot draw tickets
  // before they complete, and the early trigger measured 0.9 % slower at
  // 1 GiB (two interleaved streams).  scripts/gpu_trigger_ab.sh.  A/B:
  // PP_LATE_TRIGGER=1 never triggers early.
  static const int early = std::getenv("PP_LATE_TRIGGER") ? 0 : 1;
  a.early_trigger = early && a.sched == nullptr;
  // ticketed launches trigger their successor once the tickets reach the
  // last 4 chunks per CTA: it becomes resident and fills its ring (static
  // lead chunks, INPUT_READY) during this launch's last ~3 us instead of
  // after its last load (1 GiB: 7450 -> 7528 GB/s; tail 2 / 4 / 8 / 16 =
  // 7508-7519 / 7525-7530 / 7511-7517 / 7290, scripts/gpu_tail_ab.sh).
  // A/B: PP_TRIGGER_TAIL=n (0 = after the CTA's last load).
  static const unsigned tail = [] {
    const char *e = std::getenv("PP_TRIGGER_TAIL");
    return e ? (unsigned)std::atoi(e) : 4u;
  }();
  a.trigger_tail = tail;
#if PP_CHECK_BOUNDS
  // per-launch {chunks consumed, CTAs finished} (stream-ordered scratch)
  if (cudaMallocAsync(reinterpret_cast<void **>(&a.chk_ctr), 16, st) != cudaSuccess ||
      cudaMemsetAsync(a.chk_ctr, 0, 16, st) != cudaSuccess)
    return cudaGetLastError();
  switch (chk_corrupt_mode()) {  // pp_debug_corrupt: derived fields go wrong
    case 1: a.body += 32; break;                              // last bulk copy past the end
    case 2: a.head -= 1; a.head_bytes += 1; a.tail_bytes += 1; break;  // edge bytes outside
    default: break;
  }
#endif
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
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, a, sink);
#if PP_CHECK_BOUNDS
  cudaFreeAsync(a.chk_ctr, st);
#endif
  if (a.sched) {
    if (e != cudaSuccess)
      sched_rollback(units);
    else
      sched_commit(st);
  }
  return e;
}

cudaError_t launch_count(const CountArgs &a, LoadPath path, const DevInfo &di,
                         cudaStream_t st) {
  if (path == LoadPath::kTma) {
    const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
    cudaError_t e = launch_tma(pp_tma_kernel<1>, g, kTmaThreads, kTmaSmemBytes, st, a, nullptr,
                               a.body_bytes < pdl_max_body(), di, kTmaStages);
    if (e != cudaSuccess) return e;
  } else {
    const unsigned g =
        grid_for(a.nchunks, (unsigned long long)di.num_sms * di.ldg_blocks_per_sm);
    pp_count_ldg_kernel<<<g, kLdgThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

template <int W, int CB>
static cudaError_t launch_codes_w(const CountArgs &a0, unsigned g, const DevInfo &di,
                                  cudaStream_t st) {
  using KS = KShape<W, PP_CAT_NCW, CB>;
  CountArgs a = a0;
  a.tab_mul = 32u * KS::kTabEntry;  // bytes per table row (0: no table)
  return launch_tma(pp_tma_kernel<W, PP_CAT_NCW, CB>, g, CatShape::kThreads, KS::kSmem, st, a,
                    nullptr, true, di, KS::kStages);
}
template <int CB>
static cudaError_t launch_codes(const CountArgs &a, const DevInfo &di, cudaStream_t st) {
  const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
  switch (a.width) {
    case 8: return launch_codes_w<8, CB>(a, g, di, st);
    case 16: return launch_codes_w<16, CB>(a, g, di, st);
    case 32: return launch_codes_w<32, CB>(a, g, di, st);
    default: return launch_codes_w<64, CB>(a, g, di, st);
  }
}

cudaError_t launch_count_direct(const CountArgs &a, unsigned long long *acc,
                                unsigned long long *out, unsigned int *flag, unsigned int seq,
                                cudaStream_t st) {
  if (a.nchunks <= 1) {
    pp_count_direct_kernel<<<1, kLdgThreads, 0, st>>>(a, out, flag, seq);
  } else {
    const unsigned g = (unsigned)std::min<unsigned long long>(a.nchunks, 128);
    pp_count_direct_multi_kernel<<<g, kLdgThreads, 0, st>>>(a, acc, out, flag, seq);
  }
  return cudaGetLastError();
}

cudaError_t launch_count_codes(const CountArgs &a, int code_bytes, const DevInfo &di,
                               cudaStream_t st) {
  return code_bytes == 1   ? launch_codes<1>(a, di, st)
         : code_bytes == 2 ? launch_codes<2>(a, di, st)
                           : launch_codes<4>(a, di, st);
}

cudaError_t launch_readonly(const CountArgs &a, unsigned long long *sink, const DevInfo &di,
                            cudaStream_t st) {
  const unsigned g = grid_for(a.nchunks, (unsigned long long)di.count_sms);
  return launch_tma(pp_tma_kernel<0>, g, kTmaThreads, kTmaSmemBytes, st, a, sink,
                    a.body_bytes < pdl_max_body(), di, kTmaStages);
}

cudaError_t chk_read_count(ChkRecHost *out, bool reset) {
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

extern "C" __attribute__((visibility("default"))) int pp_sched_stats(unsigned long long *out4) {
  if (!out4) return 4;  // PP_EARG
  auto lk = pp::sched_lock();
  for (int i = 0; i < 4; ++i) out4[i] = pp::g_sched_stats[i];
  return 0;
}

#if PP_TIMELINE
extern "C" __attribute__((visibility("default"))) int pp_debug_timeline(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, pp::pp_tl, sizeof(pp::pp_tl));
}
#endif
