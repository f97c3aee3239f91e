/*
 * pospopcnt_b200.h — C ABI of the B200 (sm_100a) positional population count.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (/root/reference/pkg, pure Python) exposes the operation as a duck-typed
 * kernel object whose `run(view, w, counters)` mutates a list of w counters
 * (pkg/src/pospopcnt/kernels.py:242-270, NumbaKernel.run) behind the entry
 * point `pospopcnt(data, width, counters=None, kernel=None)`
 * (kernels.py:315-333).  The reference has no FFI of its own; the binding a
 * maintainer adds is a ctypes kernel object over these symbols (see
 * INTEGRATION.md).  Every entry point below replaces one reference interface,
 * cited per function.
 *
 * Conventions
 *  - plain C types only: pointers, sizes, ints; no torch/CUDA C++ types.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - device entry points are asynchronous on `stream`; they never synchronise
 *    except where stated.
 *  - counters are 64-bit unsigned integers, one per bit position, and are
 *    ACCUMULATED into, never cleared (core.py:82-87).
 *  - return 0 on success, otherwise a PP_E* code; pp_last_error() gives a
 *    thread-local message for the last failure on the calling thread.
 *  - word assembly is little-endian, bit position 0 = least significant bit
 *    of a word (core.py:3-6).
 *  - results do not depend on the alignment of `data` nor on bytes outside
 *    [data, data+nbytes) (pkg/tests/test_kernels.py:75-91); no byte outside
 *    that range is ever read.
 */
#ifndef POSPOPCNT_B200_H
#define POSPOPCNT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PP_API __attribute__((visibility("default")))
#else
#define PP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 1

/* error codes (mirroring the reference's exception classes, core.py:19-34) */
#define PP_OK        0
#define PP_EWIDTH    1  /* width not in {8,16,32,64}      -> ValueError (core.py:31-34)       */
#define PP_ELENGTH   2  /* nbytes not word-complete        -> InputLengthError (core.py:68-74) */
#define PP_ECUDA     3  /* CUDA runtime error              -> RuntimeError                     */
#define PP_EARG      4  /* bad pointer / argument          -> ValueError                       */
#define PP_ENODEV    5  /* no usable sm_100 device         -> KernelUnavailableError           */

/* flags for the segmented entry points */
#define PP_SEG_ACCUMULATE 0  /* out[s*w+j] += count (reference semantics)  */
#define PP_SEG_OVERWRITE  1  /* out[s*w+j]  = count (fresh counter rows)   */
/* optional launch-shape hint: lanes per segment (1, 2, 4, 8, 16 or 32) in bits 8-15;
 * 0 = automatic (fixed: 1 up to 512-byte segments, else from seg_bytes;
 * CSR / batch: 8).  1 = one lane per segment (SWAR counts, for arrays of a
 * few words; a long segment then runs on a single lane); 2 / 4 = the TMA
 * ring's shapes for 1-2 KiB fixed segments. */
#define PP_SEG_LANES(g)   ((g) << 8)
/* CSR only, opt-in: arrays of <= 512 bytes are counted one lane each and
 * the longer ones with the PP_SEG_LANES shape (two launches, each row written
 * once).  Pays for strongly bimodal lengths (profiles/r1_segmented_ablation.md). */
#define PP_SEG_HYBRID     (1 << 16)
/* optional tuning hint for the G-lane kernel: groups of 32/G segments per
 * dynamic-scheduler ticket, 1-63 in bits 20-25 (0 = automatic: the smallest
 * batch that keeps a launch under ~49k tickets). */
#define PP_SEG_BATCH(t)   ((t) << 20)

PP_API int         pp_abi_version(void);
PP_API const char *pp_strerror(int code);
PP_API const char *pp_last_error(void);

/* Number of SMs / sm major.minor of `device`; used for launch sizing. */
PP_API int pp_device_info(int device, int *num_sms, int *cc_major, int *cc_minor);

/*
 * pp_count — counters[j] += #{words k : bit j of word k is set}, j < width.
 *
 * data:     DEVICE pointer to nbytes bytes (any alignment).
 * counters: DEVICE pointer to `width` uint64 counters (8-byte aligned).
 * Replaces: NumbaKernel.run / Kernel.run(view, w, counters)
 *           (kernels.py:242-270; protocol kernels.py:93, 178, 242) and the
 *           dispatch body of pospopcnt() (kernels.py:315-333).
 * Errors:   PP_EWIDTH (check_width, core.py:31-34), PP_ELENGTH
 *           (InputView.check_complete, core.py:68-74), PP_EARG (host pointer).
 */
PP_API int pp_count(const void *data, size_t nbytes, int width,
             unsigned long long *counters, void *stream);

/*
 * pp_count_ex — pp_count with flags.  PP_COUNT_INPUT_READY: the caller
 * vouches that the input was complete before the previous kernel on
 * `stream` started (that kernel does not write it).  Every count launch
 * uses programmatic dependent launch; with this flag its bulk copies start
 * while the previous kernel drains instead of after it completes (back-to-
 * back counts of independent inputs: the next input's first loads overlap
 * the previous launch's tail).  Counter updates still wait for the previous
 * kernel.  Without the flag (pp_count) the loads wait, so a producer kernel
 * of the input that itself uses programmatic launch is always safe.
 * Replaces: as pp_count (kernels.py:242-270, 315-333).
 */
#define PP_COUNT_INPUT_READY 1u
PP_API int pp_count_ex(const void *data, size_t nbytes, int width,
                unsigned long long *counters, unsigned int flags, void *stream);

/*
 * pp_count_sync — pp_count over DEVICE bytes with the result added into HOST
 * counters: one call = zero a per-thread device scratch, count, copy the w
 * counters back, synchronise `stream`.  The reference's list-returning call
 * shape (kernels.py:315-333: pospopcnt(view, w) -> counters) for data that
 * already lives in HBM, without a caller-side D2H.  Up to 16 MiB the call is
 * ONE launch: one CTA per 32 KiB counts the range and the kernel itself
 * writes the w counts and a sequence flag into mapped pinned host memory,
 * which the calling thread polls (no memset, D2H copy or stream
 * synchronisation: 19.5 -> 14.4-15.5 us per call up to 4 MiB; the reference's
 * short arrays, edges.py:96-102 count_short).
 */
PP_API int pp_count_sync(const void *data, size_t nbytes, int width,
                         unsigned long long *host_counters, void *stream);

/*
 * pp_count_host — the same count over a HOST buffer (pinned or pageable):
 * pipelined host->device copies overlapped with counting, result added into
 * HOST counters.  Synchronous.  Replaces the bytes-like path of pospopcnt()
 * (kernels.py:315-333 with data = bytes/bytearray/memoryview; cli.py:82-94).
 * Resources, per calling host thread and device, allocated on first use and
 * kept: 3 x 64 MiB device buffers (inputs > 1 MiB), 3 x 16 MiB pinned staging
 * buffers (pageable inputs >= 2 MiB: copied there in <= 8 MiB pieces by a pool
 * of host threads with non-temporal stores, so the copy engine reads them from
 * DRAM and not out of the cores' caches), 1 MiB pinned + 1 MiB device for small
 * inputs.  Inputs up to 512 KiB are copied into that pinned buffer and
 * counted in place by CTAs reading it over the link (the direct path of
 * pp_count_sync: no H2D copy either; 8 B..4 KiB 23 -> 18.5 us, 32 KiB 33 ->
 * 20.5, 256 KiB 44.5 -> 34-37 us per call).
 */
PP_API int pp_count_host(const void *host_data, size_t nbytes, int width,
                  unsigned long long *host_counters);

/*
 * pp_count_host_multi — pp_count_host fanned out over several GPUs, so one
 * call over a host buffer uses one host link per device instead of one:
 * [host_data, +nbytes) is cut into ndevices contiguous ranges at multiples
 * of 64 bytes (word-complete for every width; counts add), range
 * k is copied to and counted on devices[k] through that device's own pinned
 * staging ring and copy stream, and the per-device counters are summed on
 * the host into host_counters.  Synchronous.  A device may be listed more
 * than once (each listing is its own range and staging context).  Fan-out
 * calls are serialised process-wide; ndevices <= PP_MAX_FANOUT.
 * Replaces: the bytes-like path of pospopcnt() (kernels.py:315-333,
 * cli.py:82-94), like pp_count_host.
 */
#define PP_MAX_FANOUT 16
PP_API int pp_count_host_multi(const void *host_data, size_t nbytes, int width,
                               unsigned long long *host_counters, const int *devices,
                               int ndevices);

/*
 * pp_count_segmented — many independent arrays in one launch.
 * Segment s is device bytes [base + seg_off[s], base + seg_off[s+1]);
 * out (DEVICE, nseg*width uint64, row-major) row s receives its counters.
 * seg_off is a DEVICE array of nseg+1 non-decreasing byte offsets; every
 * segment length must be a multiple of width/8 (caller-validated).
 * Replaces: nseg calls of Kernel.run (kernels.py:242) each with its own
 * counter list; the reference's short-array path is edges.py:96-102.
 */
PP_API int pp_count_segmented(const void *base, const unsigned long long *seg_off,
                       size_t nseg, int width, unsigned long long *out,
                       int flags, void *stream);

/*
 * pp_count_segmented_order — pp_count_segmented processing the segments in a
 * caller-given order: order (DEVICE, nseg uint32, a permutation of 0..nseg-1)
 * lists segment indices in the order the G-lane kernel takes them, in groups
 * of 32/G; rows still land at out[s].  With the segments of each group of
 * similar length (segmented.SegmentPlan sorts by length and alternates long
 * and short groups) no lane idles while a longer neighbour finishes.
 * Applies to the G-lane kernel (G = 8/16/32); the one-lane pass ignores it.
 */
PP_API int pp_count_segmented_order(const void *base, const unsigned long long *seg_off,
                                    const unsigned int *order, size_t nseg, int width,
                                    unsigned long long *out, int flags, void *stream);

/*
 * pp_count_batch — many independent arrays at arbitrary device addresses in
 * one launch: row i of out (DEVICE, n*width uint64, row-major) receives the
 * count of bytes [ptrs[i], ptrs[i] + lens[i]).  ptrs / lens are DEVICE
 * arrays of n u64 (absolute addresses, byte lengths; every length a multiple
 * of width/8, caller-validated).  flags as for pp_count_segmented (default
 * shape: 8 lanes per array; PP_SEG_LANES(1) one lane each for tiny arrays).
 * Replaces: n calls of Kernel.run (kernels.py:242), one per array.
 */
PP_API int pp_count_batch(const unsigned long long *ptrs, const unsigned long long *lens,
                          size_t n, int width, unsigned long long *out, int flags,
                          void *stream);

/* pp_count_fixed — as pp_count_segmented for nseg equal segments of seg_bytes each. */
PP_API int pp_count_fixed(const void *base, size_t seg_bytes, size_t nseg, int width,
                   unsigned long long *out, int flags, void *stream);

/*
 * pp_count_multi — pp_count whose result is added into EVERY target counter
 * array: the sharded job's allreduce fused into the counting kernel.  Each
 * CTA adds its folded counts into targets[0..ntargets-1] with u64 atomics;
 * targets may be peer-mapped device memory (other ranks' counters opened
 * with pp_ipc_open), i.e. remote atomics over NVLink.  When every rank has
 * run pp_count_multi over its shard with the same target set and the kernels
 * completed, every rank's counters hold the job total -- no NCCL call.
 * Replaces: the per-shard Kernel.run (kernels.py:242-270) + the combine of
 * the shard counters (additivity).  ntargets <= PP_MAX_TARGETS.
 */
#define PP_MAX_TARGETS 16
PP_API int pp_count_multi(const void *data, size_t nbytes, int width,
                          unsigned long long *const *targets, int ntargets, void *stream);
/* pp_count_multi with pp_count_ex's flags (PP_COUNT_INPUT_READY). */
PP_API int pp_count_multi_ex(const void *data, size_t nbytes, int width,
                      unsigned long long *const *targets, int ntargets, unsigned int flags,
                      void *stream);

/* CUDA IPC for the targets of pp_count_multi (one process per GPU): export
 * any device pointer (it may lie inside a larger allocation, e.g. a caching
 * allocator's block) as a 72-byte handle = the allocation's CUDA IPC handle
 * + the pointer's offset in it; open a peer's handle (peer access is enabled
 * lazily; the returned pointer includes the offset); close it again with
 * the pointer pp_ipc_open returned. */
#define PP_IPC_HANDLE_BYTES 72
PP_API int pp_ipc_handle(const void *dev_ptr, void *handle72);
PP_API int pp_ipc_open(const void *handle72, void **dev_ptr);
PP_API int pp_ipc_close(void *dev_ptr);

/*
 * pp_count_frame — one pass for every word width:
 * frame64[i] += #{set bits b of bytes at address A : 8*(A mod 8) + b == i}
 * over the device bytes [data, data+nbytes) (any length, any alignment).
 * Width w, for any w with nbytes % (w/8) == 0, is then the fold of
 * flush_fw (accumulate.py:115-130):
 *   C_w[j] = sum_{i = j mod w} frame64[(i + rot) mod 64],  rot = 8*(data mod 8)
 * which is the width-refinement identity of pkg/tests/test_core.py:66-72.
 */
PP_API int pp_count_frame(const void *data, size_t nbytes, unsigned long long *frame64,
                          void *stream);

/*
 * pp_count_categories — fused one-hot producer + count (
 * the paper's GROUP BY COUNT use case):
 *   counters[j] += #{i < ncodes : codes[i] == j},  j < width
 * i.e. exactly pospopcnt(one_hot_width(codes), width) without materialising
 * the one-hot words (codes >= width have no bit in a width-bit word).
 * codes: DEVICE array of ncodes unsigned integers of code_bytes (1, 2, 4),
 * aligned to code_bytes.  Replaces Kernel.run over one-hot words
 * (kernels.py:242-270) for categorical inputs.
 */
PP_API int pp_count_categories(const void *codes, size_t ncodes, int code_bytes, int width,
                               unsigned long long *counters, void *stream);
/* pp_count_categories with pp_count_ex's flags (PP_COUNT_INPUT_READY). */
PP_API int pp_count_categories_ex(const void *codes, size_t ncodes, int code_bytes, int width,
                           unsigned long long *counters, unsigned int flags, void *stream);

/*
 * pp_readonly_sum — the paper's "roofline" dummy kernel:
 * streams nbytes through exactly the load path of pp_count and XORs them into
 * *sink (DEVICE, 1 uint64).  Measurement only.
 */
PP_API int pp_readonly_sum(const void *data, size_t nbytes, unsigned long long *sink,
                    void *stream);
/* pp_readonly_sum with pp_count_ex's flags: the roofline kernel launched the
 * way the count it is compared with is launched. */
PP_API int pp_readonly_sum_ex(const void *data, size_t nbytes, unsigned long long *sink,
                       unsigned int flags, void *stream);

/*
 * pp_sched_stats — diagnostics of the dynamic chunk scheduler (per-stream
 * ticket counters of the persistent counting grids): out4 = {slots handed to
 * streams, slots taken over from streams whose last launch completed,
 * launches that found every slot busy and used the static order, launches
 * with a dynamic slot}, summed over devices, since process start.  No
 * reference counterpart (test/diagnostic only).
 */
PP_API int pp_sched_stats(unsigned long long *out4);

/*
 * pp_check_status — memory-safety evidence (no compute-sanitizer needed).
 * A checked build of this library (PP_CHECK_BOUNDS=1:
 * libpospopcnt_b200_checked.so, build.build_checked()) tests every global
 * load / bulk-copy source range against the caller's [data, data+nbytes)
 * before issuing it, every shared-memory stage index, every chunk id, and
 * per launch that the chunks consumed total exactly the chunks issued; a
 * failed check skips the access and is recorded.  out6 = {1 if this is a
 * checked build, failed checks, source line of the first, its address, its
 * allowed [lo, hi)}; reset != 0 clears the record.  Unchecked builds report
 * {0, 0, ...}.  Reference contract: edges.py:1-10, no byte outside the
 * buffer is read (pkg/tests/test_kernels.py:83-91).
 */
PP_API int pp_check_status(unsigned long long *out6, int reset);
/* pp_debug_corrupt — checked builds only: corrupt the launchers' derived
 * ranges (1: body shifted 32 bytes past the end, 2: head/tail edge bytes
 * outside, 3: fixed segmented base 16 bytes low) so a test can show the
 * checks fire; 0 restores normal launches.  PP_EARG in unchecked builds. */
PP_API int pp_debug_corrupt(int mode);

/* ---- seeded synthetic inputs, generated in place on the device ----------
 * Benchmark/test infrastructure.  Byte-identical twins
 * live in oracle/pospopcnt_oracle.c.  word_offset lets a shard generate its
 * slice of a larger logical array.  dst must be 8-byte aligned.           */

/* uniform bits: u64 word g = splitmix64(seed + (g+1)*golden) */
PP_API int pp_gen_uniform(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                   void *stream);
/* Bernoulli(q/65536) bits, q in [0, 65536], via a 16-draw AND/OR ladder */
PP_API int pp_gen_bernoulli(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                     uint32_t q, void *stream);
/* per-block Bernoulli: block b (block_bytes each) has q_b = mix(seed', b) mod 65537 */
PP_API int pp_gen_blocks(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                  uint64_t block_bytes, void *stream);
/* one-hot u32 words: bit = #{k < 31 : thresholds[k] <= u}, u uniform u32 */
/* u8 codes with the same draws: code i = bit position of one-hot word i    */
PP_API int pp_gen_codes8(void *dst, size_t n, uint64_t seed, uint64_t offset,
                         const uint32_t *thresholds31, void *stream);
PP_API int pp_gen_onehot32(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                    const uint32_t *thresholds31, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* POSPOPCNT_B200_H */
