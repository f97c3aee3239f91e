// pp_internal.h — launchers shared between the kernel and C-ABI translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>

namespace pp {

// Split of one contiguous device byte range into a 16-byte aligned body plus
// <16-byte head and tail (the reference's head_load / count_tail split,
// edges.py:32-93, with "aligned" meaning the device address).
struct CountArgs {
  const uint8_t *body;
  unsigned long long body_bytes;  // multiple of 16
  unsigned long long nchunks;     // ceil(body_bytes / chunk bytes)
  const uint8_t *head;
  const uint8_t *tail;
  uint32_t head_bytes;  // < 16
  uint32_t tail_bytes;  // < 16
  unsigned long long *counters;
  int width;
  int rot;  // 8 * (address of first byte mod 8), flush_fw's rot (accumulate.py:115-130)
  // pp_count_multi: further counter arrays (often peer-mapped over NVLink)
  // that receive the same counts as `counters`
  int nextra;
  unsigned long long *extra[15];
  // dynamic chunk scheduler: the stream's ticket counter and its value at
  // this launch's start (tickets are drawn as sched_base, sched_base + 1, ...
  // mod 2^32), or nullptr for the static grid-stride order (graph capture,
  // slots exhausted)
  unsigned int *sched;
  unsigned int sched_base;
  // PP_COUNT_INPUT_READY: the input is complete before the previous kernel on
  // the stream starts (that kernel does not write it), so under programmatic
  // dependent launch the loads need not wait for it; the ticket draws and the
  // counter atomics still do
  int input_ready;
  // static chunks per CTA before its first ticket (launch_tma: the ring depth)
  unsigned int lead;
  // trigger the dependent launch at kernel start (default; PP_LATE_TRIGGER=1:
  // after the CTA's last load)
  int early_trigger;
  // ticketed launches: trigger once tickets reach the last trigger_tail
  // chunks per CTA (0: after the CTA's last load)
  unsigned int trigger_tail;
  // fused one-hot producer: bytes per row of the shared-memory one-hot table
  // (pp_count.cu KShape; a kernel argument so the address is one IMAD)
  unsigned int tab_mul;
  // checked builds (PP_CHECK_BOUNDS): the caller's byte range as the API
  // received it, and a per-launch {chunks consumed, CTAs finished} pair
  uintptr_t chk_lo, chk_hi;
  unsigned long long *chk_ctr;
};

struct SegArgs {
  const uint8_t *base;
  const unsigned long long *seg_off;  // nullptr => fixed segments
  unsigned long long seg_bytes;       // fixed mode only
  unsigned long long nseg;
  unsigned long long *out;
  int width;
  int overwrite;
  int lanes_per_segment;  // G in {1, 8, 16, 32}
  // pp_seg_kernel: groups of 32/G segments per scheduler ticket (>= 1; 0 =
  // automatic, resolved by launch_segmented)
  unsigned int batch_groups;
  unsigned int *sched;    // dynamic scheduler ticket counter, or nullptr
  unsigned int sched_base;  // its value when this launch starts
  // hybrid split (0 = off): segments of <= short_max bytes are counted one
  // lane each (pp_seglane_kernel), the longer ones by the G-lane kernel
  unsigned long long short_max;
  // pointer mode (pp_count_batch): segment s = [ptrs[s], ptrs[s] + lens[s]),
  // device arrays of absolute addresses and byte lengths; base/seg_off unused
  const unsigned long long *ptrs;
  const unsigned long long *lens;
  // processing order of the G-lane kernel (pp_count_segmented_order): slot k
  // counts segment order[k]; nullptr = slot k is segment k
  const unsigned int *order;
  // checked builds: the caller's byte range (fixed segments: [base, base +
  // nseg * seg_bytes)); 0/0 = derived in the kernel (CSR: [base + seg_off[0],
  // base + seg_off[nseg]); pointer mode: each array's own range)
  uintptr_t chk_lo, chk_hi;
};

// checked builds: this translation unit's failure record (read / reset)
struct ChkRecHost {
  unsigned int fails, first_line;
  unsigned long long first_addr, first_lo, first_hi;
};
cudaError_t chk_read_count(ChkRecHost *out, bool reset);
cudaError_t chk_read_seg(ChkRecHost *out, bool reset);
// checked builds: deliberate argument corruption (pp_debug_corrupt), applied
// by the launchers after the caller's range was recorded; 0 = none
int chk_corrupt_mode();

enum class LoadPath : int { kTma = 0, kLdg = 1 };

struct DevInfo {
  int num_sms;
  int cc_major, cc_minor;
  int seg_blocks_per_sm;
  int ldg_blocks_per_sm;
  int lane_blocks_per_sm;
  int count_sms;  // SMs the persistent counting grid uses (num_sms - PP_RESERVE_SMS)
  unsigned int *sched;  // kSchedSlots ticket counters, zeroed (device memory)
  bool ready;
};

cudaError_t device_info(int dev, DevInfo *out);
// segmented kernels' attributes and occupancy into *d (pp_segmented.cu)
cudaError_t segmented_setup(DevInfo *d);

// "no chunk": the TMA producers' stop sentinel in a stage's chunk-id slot
constexpr unsigned long long kNoChunk = ~0ull;
// The stream's dynamic-scheduler ticket counter on di's device, or nullptr
// (graph capture, slots exhausted, PP_STATIC_SCHED).  *base receives the
// counter's value at the start of this launch; the launch must draw exactly
// `units` tickets (one per work unit: every unit is a CTA's or warp's first
// or the reward of one successful draw, and each CTA/warp draws once more
// to learn it is done), so the next launch's base is base + units.
// Caller holds sched_lock() from sched_slot() until the launch is enqueued.
unsigned int *sched_slot(const DevInfo &di, cudaStream_t st, unsigned long long units,
                         unsigned int *base);
std::unique_lock<std::mutex> sched_lock();
// undo the last sched_slot() hand-out (its launch failed to enqueue)
void sched_rollback(unsigned long long units);
// the launch of the last sched_slot() hand-out is enqueued on st: record its
// completion (a slot is reused by another stream only once that completed)
void sched_commit(cudaStream_t st);

inline unsigned grid_for(unsigned long long nchunks, unsigned long long cap) {
  const unsigned long long g = nchunks < cap ? nchunks : cap;
  return (unsigned)(g ? g : 1);
}

// Fills head/body/tail fields of a (given data pointer, nbytes, chunk size).
void split_range(const uint8_t *data, unsigned long long nbytes,
                 unsigned long long chunk_bytes, CountArgs *a);

unsigned long long count_chunk_bytes(LoadPath path);
unsigned long long codes8_chunk_bytes();
cudaError_t launch_count(const CountArgs &a, LoadPath path, const DevInfo &di,
                         cudaStream_t st);
// the range (split with the LDG chunk size) counted by one CTA per chunk,
// the result published by the kernel itself: out[j] (j < a.width, not
// accumulated) then *flag = seq, both in mapped pinned host memory.  acc:
// 65 zeroed u64 of device scratch (left zeroed), used when the range has
// more than one chunk.  a.counters is unused.
cudaError_t launch_count_direct(const CountArgs &a, unsigned long long *acc,
                                unsigned long long *out, unsigned int *flag, unsigned int seq,
                                cudaStream_t st);
cudaError_t launch_segmented(const SegArgs &a, const DevInfo &di, cudaStream_t st);
// fused one-hot producer over 1/2/4-byte codes (a.width = W, a.rot ignored)
cudaError_t launch_count_codes(const CountArgs &a, int code_bytes, const DevInfo &di,
                               cudaStream_t st);
cudaError_t launch_readonly(const CountArgs &a, unsigned long long *sink,
                            const DevInfo &di, cudaStream_t st);

cudaError_t launch_categories(const uint8_t *codes, unsigned long long nbytes, int code_bytes,
                              int ncat, unsigned long long *counters, const DevInfo &di,
                              int dev, cudaStream_t st);

cudaError_t launch_gen_codes8(uint8_t *dst, unsigned long long n, uint64_t seed,
                              uint64_t offset, const uint32_t *thr31, cudaStream_t st);
cudaError_t launch_gen_uniform(uint64_t *dst, unsigned long long nwords, uint64_t seed,
                               uint64_t word_offset, cudaStream_t st);
cudaError_t launch_gen_bernoulli(uint64_t *dst, unsigned long long nwords, uint64_t seed,
                                 uint64_t word_offset, uint32_t q, cudaStream_t st);
cudaError_t launch_gen_blocks(uint64_t *dst, unsigned long long nwords, uint64_t seed,
                              uint64_t word_offset, uint64_t block_bytes,
                              cudaStream_t st);
cudaError_t launch_gen_onehot32(uint32_t *dst, unsigned long long nwords, uint64_t seed,
                                uint64_t word_offset, const uint32_t *thr31,
                                cudaStream_t st);

}  // namespace pp
