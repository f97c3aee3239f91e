/*
 * pospopcnt_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference's positional population count, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg.  Nothing in paper_2412_16370_b200/ links or calls this file.
 *
 * The reference (/root/reference/pkg/src/pospopcnt, pure Python + one numba
 * kernel) cannot travel to the GPU box, so this file restates it in C:
 *
 *   oracle_scalar     core.py:82-96 (scalar_pospopcnt, the naive oracle)
 *   oracle_hs512      kernels.py:242-270 (NumbaKernel.run, the reference's
 *                     fastest CPU path) with _nbkern.py:43-177 (run_main),
 *                     edges.py:32-46 (head_load), edges.py:59-102
 *                     (count_tail / count_short), accumulate.py:115-130
 *                     (flush_fw).  Same uint16 counter vectors, same flush
 *                     rule (FLUSH_LIMIT, _nbkern.py:29), same rot.
 *   oracle_hs512_mt   the same over contiguous 64-byte-aligned shards on
 *                     pthreads, counters summed (additivity).
 *   oracle_gen_*      byte-identical CPU twins of the device generators
 *                     (paper_2412_16370_b200/csrc/pp_gen.cu).
 *
 * Parity of this restatement is pinned against the reference itself by
 * tests/golden/make_golden.py (fixtures in tests/golden/) and
 * tests/test_oracle.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define W_MAX 64

/* ------------------------------------------------------------ core.py:82-96 */
int oracle_scalar(const uint8_t *data, size_t n, int w, uint64_t *counters) {
  if (w != 8 && w != 16 && w != 32 && w != 64) return 1;
  const size_t step = (size_t)w / 8;
  if (n % step) return 2;
  for (size_t k = 0; k < n; k += step) {
    uint64_t word = 0;
    for (size_t b = 0; b < step; ++b) word |= (uint64_t)data[k + b] << (8 * b);
    for (int j = 0; j < w; ++j) counters[j] += (word >> j) & 1u;
  }
  return 0;
}

/* ------------------------------------------------------ accumulate.py:115-130 */
static void flush_fw_u16(uint64_t *counters, const uint16_t *c, int w, int rot) {
  for (int j = 0; j < w; ++j) {
    uint64_t total = 0;
    for (int i = j; i < W_MAX; i += w) total += c[(i + rot) % W_MAX];
    counters[j] += total;
  }
}
static void flush_fw_u64(uint64_t *counters, const uint64_t *c, int w, int rot) {
  for (int j = 0; j < w; ++j) {
    uint64_t total = 0;
    for (int i = j; i < W_MAX; i += w) total += c[(i + rot) % W_MAX];
    counters[j] += total;
  }
}

/* -------------------------------------------------------------- edges.py:59-93
 * Byte counters per 64-bit group, flushed into the 16-bit c vector.  The
 * reference's numpy route (>= 24 bytes) and int route (< 24 bytes) compute the
 * same exact counts; the final partial group is zero padded. */
static void count_tail_u16(uint16_t *c, const uint8_t *tail, size_t n) {
  uint32_t t[W_MAX];
  memset(t, 0, sizeof t);
  for (size_t i = 0; i < n; ++i) {
    const uint8_t b = tail[i];
    const int base = 8 * (int)(i % 8);
    for (int k = 0; k < 8; ++k) t[base + k] += (b >> k) & 1u;
  }
  for (int i = 0; i < W_MAX; ++i) c[i] = (uint16_t)(c[i] + t[i]);
}

/* ----------------------------------------------------------- _nbkern.py:15-40 */
#define M1 0x5555555555555555ull
#define M2 0x3333333333333333ull
#define M4 0x0F0F0F0F0F0F0F0Full
#define MA 0xAAAAAAAAAAAAAAAAull
#define MC 0xCCCCCCCCCCCCCCCCull
#define FLUSH_LIMIT (0xFFFF - 30 * 8)

static inline void fa8(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t *carry,
                       uint64_t *s) {
  for (int k = 0; k < 8; ++k) {
    const uint64_t ak = a[k], bk = b[k], ck = c[k];
    const uint64_t s1 = ak ^ bk;
    carry[k] = (ak & bk) | (ck & s1);
    s[k] = s1 ^ ck;
  }
}

static inline void load8(uint64_t *dst, const uint8_t *src) { memcpy(dst, src, 64); }

/* _nbkern.py:43-177 (run_main): head block (CSA15), main loop (CSA16+4 + a16
 * split-and-fold into uint16 c, flush into c64), final nibble transpose.
 * words: the aligned vectors after the head slot, 14 + 16*nblocks vectors. */
static void run_main(const uint64_t *head, const uint8_t *words, size_t nblocks, uint16_t *c,
                     uint64_t *c64) {
  uint64_t v[16][8];
  uint64_t s1[8], s2[8], s3[8], s4[8], s5[8], k1[8], k2[8], k3[8], k4[8], k5[8];
  uint64_t d1[8], d2[8], d3[8], t1[8], t2[8], e1[8], e2[8], e3[8], e4[8];
  uint64_t u1[8], u2[8], u3[8], f1[8], f2[8], x1[8], a16[8];
  uint64_t a1[8], a2[8], a4[8], a8[8];

  /* initial 15-vector block: 11 full adders (_nbkern.py:84-95) */
  memcpy(v[0], head, 64);
  for (int i = 1; i < 15; ++i) load8(v[i], words + 64 * (i - 1));
  fa8(v[0], v[1], v[2], k1, s1);
  fa8(v[3], v[4], v[5], k2, s2);
  fa8(v[6], v[7], v[8], k3, s3);
  fa8(v[9], v[10], v[11], k4, s4);
  fa8(v[12], v[13], v[14], k5, s5);
  fa8(s1, s2, s3, d1, t1);
  fa8(t1, s4, s5, d2, a1);
  fa8(k1, k2, k3, e1, u1);
  fa8(k4, k5, d1, e2, u2);
  fa8(u1, u2, d2, e3, a2);
  fa8(e1, e2, e3, a8, a4);

  uint32_t h = 0;
  const uint8_t *p = words + 14 * 64;
  for (size_t blk = 0; blk < nblocks; ++blk, p += 1024) {
    for (int i = 0; i < 16; ++i) load8(v[i], p + 64 * i);
    /* 16+4 CSA network, 15 full adders (_nbkern.py:101-115) */
    fa8(v[0], v[1], v[2], k1, s1);
    fa8(v[3], v[4], v[5], k2, s2);
    fa8(v[6], v[7], v[8], k3, s3);
    fa8(v[9], v[10], v[11], k4, s4);
    fa8(v[12], v[13], v[14], k5, s5);
    fa8(s1, s2, s3, d1, t1);
    fa8(s4, s5, v[15], d2, t2);
    fa8(t1, t2, a1, d3, a1);
    fa8(k1, k2, k3, e1, u1);
    fa8(k4, k5, d1, e2, u2);
    fa8(d2, d3, a2, e3, u3);
    fa8(u1, u2, u3, e4, a2);
    fa8(e1, e2, e3, f1, x1);
    fa8(x1, e4, a4, f2, a4);
    fa8(f1, f2, a8, a16, a8);

    /* a16 split-and-fold to byte planes (_nbkern.py:118-137) */
    uint64_t ev[4], od[4];
    for (int k = 0; k < 4; ++k) {
      ev[k] = (a16[k] & M1) + (a16[k + 4] & M1);
      od[k] = ((a16[k] >> 1) & M1) + ((a16[k + 4] >> 1) & M1);
    }
    const uint64_t ee = (ev[0] & M2) + (ev[2] & M2);
    const uint64_t eo = ((ev[0] >> 2) & M2) + ((ev[2] >> 2) & M2);
    const uint64_t oe = (od[0] & M2) + (od[2] & M2);
    const uint64_t oo = ((od[0] >> 2) & M2) + ((od[2] >> 2) & M2);
    const uint64_t ee2 = (ev[1] & M2) + (ev[3] & M2);
    const uint64_t eo2 = ((ev[1] >> 2) & M2) + ((ev[3] >> 2) & M2);
    const uint64_t oe2 = (od[1] & M2) + (od[3] & M2);
    const uint64_t oo2 = ((od[1] >> 2) & M2) + ((od[3] >> 2) & M2);
    const uint64_t x0 = (ee & M4) + (ee2 & M4);
    const uint64_t x4 = ((ee >> 4) & M4) + ((ee2 >> 4) & M4);
    const uint64_t x2 = (eo & M4) + (eo2 & M4);
    const uint64_t x6 = ((eo >> 4) & M4) + ((eo2 >> 4) & M4);
    const uint64_t xs1 = (oe & M4) + (oe2 & M4);
    const uint64_t x5 = ((oe >> 4) & M4) + ((oe2 >> 4) & M4);
    const uint64_t x3 = (oo & M4) + (oo2 & M4);
    const uint64_t x7 = ((oo >> 4) & M4) + ((oo2 >> 4) & M4);
    /* 64 u16 adds (_nbkern.py:138-148) */
    for (int e = 0; e < 8; ++e) {
      const int sh = 8 * e, o = 8 * e;
      c[o + 0] = (uint16_t)(c[o + 0] + (((x0 >> sh) & 0xFF) << 4));
      c[o + 4] = (uint16_t)(c[o + 4] + (((x4 >> sh) & 0xFF) << 4));
      c[o + 2] = (uint16_t)(c[o + 2] + (((x2 >> sh) & 0xFF) << 4));
      c[o + 6] = (uint16_t)(c[o + 6] + (((x6 >> sh) & 0xFF) << 4));
      c[o + 1] = (uint16_t)(c[o + 1] + (((xs1 >> sh) & 0xFF) << 4));
      c[o + 5] = (uint16_t)(c[o + 5] + (((x5 >> sh) & 0xFF) << 4));
      c[o + 3] = (uint16_t)(c[o + 3] + (((x3 >> sh) & 0xFF) << 4));
      c[o + 7] = (uint16_t)(c[o + 7] + (((x7 >> sh) & 0xFF) << 4));
    }
    /* overflow discipline (_nbkern.py:150-155) */
    h += 128;
    if (h > FLUSH_LIMIT) {
      for (int i = 0; i < 64; ++i) {
        c64[i] += c[i];
        c[i] = 0;
      }
      h = 0;
    }
  }

  /* final accumulation: 4x4 transpose of (a8,a4,a2,a1) into nibbles
   * (_nbkern.py:157-177, accumulate.py:78-98) */
  for (int k = 0; k < 8; ++k) {
    const uint64_t b1 = a1[k], b2 = a2[k], b4 = a4[k], b8 = a8[k];
    const uint64_t l12 = (b1 & M1) | ((b2 << 1) & MA);
    const uint64_t h12 = (b2 & MA) | ((b1 >> 1) & M1);
    const uint64_t l48 = (b4 & M1) | ((b8 << 1) & MA);
    const uint64_t h48 = (b8 & MA) | ((b4 >> 1) & M1);
    const uint64_t aa = (l12 & M2) | ((l48 << 2) & MC);
    const uint64_t ab = (h12 & M2) | ((h48 << 2) & MC);
    const uint64_t ac = (l48 & MC) | ((l12 >> 2) & M2);
    const uint64_t ad = (h48 & MC) | ((h12 >> 2) & M2);
    for (int g = 0; g < 16; ++g) {
      const int sh = 4 * g, o = 4 * g;
      c[o + 0] = (uint16_t)(c[o + 0] + ((aa >> sh) & 0xF));
      c[o + 1] = (uint16_t)(c[o + 1] + ((ab >> sh) & 0xF));
      c[o + 2] = (uint16_t)(c[o + 2] + ((ac >> sh) & 0xF));
      c[o + 3] = (uint16_t)(c[o + 3] + ((ad >> sh) & 0xF));
    }
  }
}

/* kernels.py:242-270 (NumbaKernel.run) over the view (base, offset, n).
 * Alignment is base-relative, exactly like InputView (core.py:37-55). */
int oracle_hs512(const uint8_t *base, size_t offset, size_t n, int w, uint64_t *counters) {
  if (w != 8 && w != 16 && w != 32 && w != 64) return 1;
  if (n % ((size_t)w / 8)) return 2;
  const size_t rb = 64;
  if (n < 15 * rb) { /* count_short, edges.py:96-102 (rot 0: view-relative) */
    uint16_t c[W_MAX];
    memset(c, 0, sizeof c);
    /* count_short accumulates into a list of ints; < 960 bytes cannot wrap u16 */
    count_tail_u16(c, base + offset, n);
    flush_fw_u16(counters, c, w, 0);
    return 0;
  }
  /* head_load (edges.py:32-46) */
  const size_t a = offset % rb;
  const size_t astart = offset - a;
  uint64_t v0[8];
  uint8_t hb[64];
  memcpy(hb, base + astart, 64);
  memset(hb, 0, a);
  memcpy(v0, hb, 64);
  size_t pos = (rb - a) + 14 * rb;
  const size_t block = 16 * rb;
  const size_t nblocks = (n - pos) / block;
  uint16_t c[W_MAX];
  uint64_t c64[W_MAX];
  memset(c, 0, sizeof c);
  memset(c64, 0, sizeof c64);
  run_main(v0, base + astart + rb, nblocks, c, c64);
  pos += nblocks * block;
  const int rot = (int)(8 * (offset % 8));
  count_tail_u16(c, base + offset + pos, n - pos);
  flush_fw_u16(counters, c, w, rot);
  flush_fw_u64(counters, c64, w, rot);
  return 0;
}

/* ----------------------------------------------------- threaded shards */
typedef struct {
  const uint8_t *base;
  size_t offset, n;
  int w;
  uint64_t counters[W_MAX];
  int rc;
} shard_t;

static void *shard_main(void *arg) {
  shard_t *s = (shard_t *)arg;
  s->rc = oracle_hs512(s->base, s->offset, s->n, s->w, s->counters);
  return NULL;
}

int oracle_hs512_mt(const uint8_t *base, size_t offset, size_t n, int w, uint64_t *counters,
                    int nthreads) {
  if (w != 8 && w != 16 && w != 32 && w != 64) return 1;
  if (n % ((size_t)w / 8)) return 2;
  if (nthreads < 1) nthreads = 1;
  const size_t min_shard = 1 << 20;
  if ((size_t)nthreads > n / min_shard) nthreads = (int)(n / min_shard);
  if (nthreads <= 1) return oracle_hs512(base, offset, n, w, counters);
  shard_t *sh = (shard_t *)calloc((size_t)nthreads, sizeof(shard_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!sh || !th) {
    free(sh);
    free(th);
    return 3;
  }
  size_t start = 0;
  for (int t = 0; t < nthreads; ++t) {
    size_t end = (t == nthreads - 1) ? n : (n / (size_t)nthreads) * (size_t)(t + 1) / 64 * 64;
    if (end < start) end = start;
    sh[t].base = base;
    sh[t].offset = offset + start;
    sh[t].n = end - start;
    sh[t].w = w;
    start = end;
  }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, shard_main, &sh[t]);
  int rc = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (sh[t].rc) rc = sh[t].rc;
    for (int j = 0; j < w; ++j) counters[j] += sh[t].counters[j];
  }
  free(sh);
  free(th);
  return rc;
}

/* Many views of one buffer: out[s*w + j] += counts of bytes
 * [seg_off[s], seg_off[s+1]) (each a base-relative InputView), threaded. */
typedef struct {
  const uint8_t *base;
  const uint64_t *starts, *ends;
  size_t s0, s1;
  int w;
  uint64_t *out;
  int rc;
} segjob_t;

static void *seg_main(void *arg) {
  segjob_t *j = (segjob_t *)arg;
  for (size_t s = j->s0; s < j->s1; ++s) {
    const uint64_t a = j->starts[s], b = j->ends[s];
    int rc = oracle_hs512(j->base, a, b - a, j->w, j->out + s * (size_t)j->w);
    if (rc) j->rc = rc;
  }
  return NULL;
}

/* Arbitrary views [starts[s], ends[s]) of one buffer, threaded. */
int oracle_views(const uint8_t *base, const uint64_t *starts, const uint64_t *ends, size_t nseg,
                 int w, uint64_t *out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > nseg) nthreads = nseg ? (int)nseg : 1;
  segjob_t *jobs = (segjob_t *)calloc((size_t)nthreads, sizeof(segjob_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!jobs || !th) {
    free(jobs);
    free(th);
    return 3;
  }
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].base = base;
    jobs[t].starts = starts;
    jobs[t].ends = ends;
    jobs[t].s0 = nseg * (size_t)t / (size_t)nthreads;
    jobs[t].s1 = nseg * (size_t)(t + 1) / (size_t)nthreads;
    jobs[t].w = w;
    jobs[t].out = out;
    pthread_create(&th[t], NULL, seg_main, &jobs[t]);
  }
  int rc = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].rc) rc = jobs[t].rc;
  }
  free(jobs);
  free(th);
  return rc;
}

/* CSR partition: segment s = [seg_off[s], seg_off[s+1]). */
int oracle_segments(const uint8_t *base, const uint64_t *seg_off, size_t nseg, int w,
                    uint64_t *out, int nthreads) {
  return oracle_views(base, seg_off, seg_off + 1, nseg, w, out, nthreads);
}

/* ---------------------------------------------------------- generators
 * CPU twins of paper_2412_16370_b200/csrc/pp_gen.cu (see its header). */
#define GOLDEN 0x9E3779B97F4A7C15ull
#define BLOCK_SALT 0x5EEDB10C5EEDB10Cull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t ladder(uint64_t seed, uint64_t g, uint32_t q) {
  if (q >= 65536u) return ~0ull;
  uint64_t x = 0;
  const uint64_t b = seed + (16ull * g + 1ull) * GOLDEN;
  for (int k = 0; k < 16; ++k) {
    const uint64_t r = mix64(b + (uint64_t)k * GOLDEN);
    x = ((q >> k) & 1u) ? (x | r) : (x & r);
  }
  return x;
}

void oracle_gen_uniform(uint64_t *dst, size_t nwords, uint64_t seed, uint64_t off) {
  for (size_t i = 0; i < nwords; ++i) dst[i] = mix64(seed + (off + i + 1ull) * GOLDEN);
}

void oracle_gen_bernoulli(uint64_t *dst, size_t nwords, uint64_t seed, uint64_t off, uint32_t q) {
  for (size_t i = 0; i < nwords; ++i) dst[i] = ladder(seed, off + i, q);
}

void oracle_gen_blocks(uint64_t *dst, size_t nwords, uint64_t seed, uint64_t off,
                       uint64_t block_bytes) {
  for (size_t i = 0; i < nwords; ++i) {
    const uint64_t g = off + i;
    const uint64_t b = (g * 8ull) / block_bytes;
    const uint32_t q = (uint32_t)(mix64((seed ^ BLOCK_SALT) + (b + 1ull) * GOLDEN) % 65537ull);
    dst[i] = ladder(seed, g, q);
  }
}

void oracle_gen_onehot32(uint32_t *dst, size_t nwords, uint64_t seed, uint64_t off,
                         const uint32_t *thr31) {
  for (size_t i = 0; i < nwords; ++i) {
    const uint32_t u = (uint32_t)(mix64(seed + (off + i + 1ull) * GOLDEN) >> 32);
    uint32_t cat = 0;
    for (int k = 0; k < 31; ++k) cat += thr31[k] <= u;
    dst[i] = 1u << cat;
  }
}

void oracle_gen_codes8(uint8_t *dst, size_t n, uint64_t seed, uint64_t off,
                       const uint32_t *thr31) {
  for (size_t i = 0; i < n; ++i) {
    const uint32_t u = (uint32_t)(mix64(seed + (off + i + 1ull) * GOLDEN) >> 32);
    uint32_t cat = 0;
    for (int k = 0; k < 31; ++k) cat += thr31[k] <= u;
    dst[i] = (uint8_t)cat;
  }
}

/* per-block q values of oracle_gen_blocks (for closed-form expectations) */
uint32_t oracle_block_q(uint64_t seed, uint64_t b) {
  return (uint32_t)(mix64((seed ^ BLOCK_SALT) + (b + 1ull) * GOLDEN) % 65537ull);
}
