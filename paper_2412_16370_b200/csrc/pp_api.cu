// pp_api.cu — the C ABI (include/pospopcnt_b200.h): validation, launch
// sizing, error mapping and the pipelined host-buffer path.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#define PP_HAVE_SSE2 1
#else
#define PP_HAVE_SSE2 0
#endif
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pospopcnt_b200.h"
#include "pp_internal.h"

namespace {

thread_local std::string g_err;
std::atomic<int> g_corrupt{0};  // pp_debug_corrupt (checked builds only)

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char *where) {
  return fail(PP_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

bool width_ok(int w) { return w == 8 || w == 16 || w == 32 || w == 64; }

// Which load path feeds the counting kernel.  TMA bulk copies are the
// default; PP_LOAD_PATH=ldg selects the register-fed variant for A/B runs.
pp::LoadPath load_path() {
  static pp::LoadPath path = [] {
    const char *s = std::getenv("PP_LOAD_PATH");
    return (s && std::strcmp(s, "ldg") == 0) ? pp::LoadPath::kLdg : pp::LoadPath::kTma;
  }();
  return path;
}

int current_devinfo(pp::DevInfo *di) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    // the reference's KernelUnavailableError (core.py:23-28), not a CUDA fault
    return fail(PP_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  e = pp::device_info(dev, di);
  if (e != cudaSuccess) return cuda_fail(e, "device_info");
  if (di->cc_major != 10)
    return fail(PP_ENODEV, "device %d is sm_%d%d; this build targets sm_100a", dev,
                di->cc_major, di->cc_minor);
  return PP_OK;
}

// Device memory (or managed) check; a host pointer handed to a kernel would
// fault the GPU, so it is rejected here.
int check_device_ptr(const void *p, const char *what) {
  if (!p) return fail(PP_EARG, "%s is NULL", what);
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PP_EARG, "%s: not a CUDA pointer (%s)", what, cudaGetErrorString(e));
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(PP_EARG, "%s must be device memory", what);
  return PP_OK;
}

// Base address of the device allocation containing p (driver API
// cuMemGetAddressRange, reached through the runtime's entry-point query so
// the library needs no link-time libcuda).
int alloc_base(const void *p, unsigned long long *base) {
  using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
  static GetRange fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRange>(f);
  }();
  if (!fn) return fail(PP_ECUDA, "cuMemGetAddressRange entry point unavailable");
  size_t size = 0;
  const int r = fn(base, &size, reinterpret_cast<uintptr_t>(p));
  if (r != 0) return fail(PP_EARG, "cuMemGetAddressRange failed (CUresult %d)", r);
  return PP_OK;
}

// pointers returned by pp_ipc_open -> the mapping base to close
std::mutex g_ipc_m;
std::map<void *, void *> g_ipc_base;

int count_device(const void *data, size_t nbytes, int width, unsigned long long *counters,
                 cudaStream_t st, const pp::DevInfo &di, bool raw_frame = false,
                 unsigned int flags = 0) {
  pp::CountArgs a{};
  const pp::LoadPath path = load_path();
  pp::split_range(static_cast<const uint8_t *>(data), nbytes, pp::count_chunk_bytes(path), &a);
  a.counters = counters;
  a.width = width;
  a.input_ready = (flags & PP_COUNT_INPUT_READY) ? 1 : 0;
  if (raw_frame) a.rot = 0;  // frame[i] as is: bit i mod 8 of bytes at address = i/8 mod 8
  cudaError_t e = pp::launch_count(a, path, di, st);
  if (e != cudaSuccess) return cuda_fail(e, "pp_count launch");
  return PP_OK;
}

}  // namespace

namespace pp {
int chk_corrupt_mode() { return g_corrupt.load(std::memory_order_relaxed); }
}  // namespace pp

extern "C" {

int pp_abi_version(void) { return PP_ABI_VERSION; }

int pp_check_status(unsigned long long *out6, int reset) {
  if (!out6) return fail(PP_EARG, "out6 is NULL");
  std::memset(out6, 0, 6 * sizeof *out6);
#if PP_CHECK_BOUNDS
  out6[0] = 1;
  pp::ChkRecHost r[2];
  cudaError_t e;
  if ((e = pp::chk_read_count(&r[0], reset != 0))) return cuda_fail(e, "pp_check_status");
  if ((e = pp::chk_read_seg(&r[1], reset != 0))) return cuda_fail(e, "pp_check_status");
  for (const auto &x : r) {
    if (x.fails && !out6[1]) {
      out6[2] = x.first_line;
      out6[3] = x.first_addr;
      out6[4] = x.first_lo;
      out6[5] = x.first_hi;
    }
    out6[1] += x.fails;
  }
#else
  (void)reset;
#endif
  return PP_OK;
}

int pp_debug_corrupt(int mode) {
#if PP_CHECK_BOUNDS
  if (mode < 0 || mode > 3) return fail(PP_EARG, "corruption mode %d not in 0..3", mode);
  g_corrupt.store(mode);
  return PP_OK;
#else
  (void)mode;
  return fail(PP_EARG, "pp_debug_corrupt exists in checked builds only (PP_CHECK_BOUNDS=1)");
#endif
}

const char *pp_strerror(int code) {
  switch (code) {
    case PP_OK: return "ok";
    case PP_EWIDTH: return "word width must be one of (8, 16, 32, 64)";
    case PP_ELENGTH: return "input length is not a multiple of the word size";
    case PP_ECUDA: return "CUDA error";
    case PP_EARG: return "invalid argument";
    case PP_ENODEV: return "no usable sm_100 device";
    default: return "unknown error";
  }
}

const char *pp_last_error(void) { return g_err.c_str(); }

int pp_device_info(int device, int *num_sms, int *cc_major, int *cc_minor) {
  pp::DevInfo di;
  cudaError_t e = pp::device_info(device, &di);
  if (e != cudaSuccess) return cuda_fail(e, "pp_device_info");
  if (num_sms) *num_sms = di.num_sms;
  if (cc_major) *cc_major = di.cc_major;
  if (cc_minor) *cc_minor = di.cc_minor;
  return PP_OK;
}

int pp_count(const void *data, size_t nbytes, int width, unsigned long long *counters,
             void *stream) {
  return pp_count_ex(data, nbytes, width, counters, 0u, stream);
}

int pp_count_ex(const void *data, size_t nbytes, int width, unsigned long long *counters,
                unsigned int flags, void *stream) {
  if (flags & ~PP_COUNT_INPUT_READY) return fail(PP_EARG, "unknown pp_count_ex flags 0x%x", flags);
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (nbytes % (size_t)(width / 8))
    return fail(PP_ELENGTH, "%zu bytes is not a multiple of the %d-byte word size", nbytes,
                width / 8);
  int rc;
  if ((rc = check_device_ptr(counters, "counters"))) return rc;
  if (nbytes == 0) return PP_OK;  // counters unchanged (core.py:82-96 on empty input)
  if ((rc = check_device_ptr(data, "data"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  return count_device(data, nbytes, width, counters, static_cast<cudaStream_t>(stream), di, false,
                      flags);
}

int pp_count_frame(const void *data, size_t nbytes, unsigned long long *frame64,
                   void *stream) {
  int rc;
  if ((rc = check_device_ptr(frame64, "frame64"))) return rc;
  if (nbytes == 0) return PP_OK;
  if ((rc = check_device_ptr(data, "data"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  return count_device(data, nbytes, 64, frame64, static_cast<cudaStream_t>(stream), di, true);
}

int pp_count_multi(const void *data, size_t nbytes, int width,
                   unsigned long long *const *targets, int ntargets, void *stream) {
  return pp_count_multi_ex(data, nbytes, width, targets, ntargets, 0u, stream);
}

int pp_count_multi_ex(const void *data, size_t nbytes, int width,
                      unsigned long long *const *targets, int ntargets, unsigned int flags,
                      void *stream) {
  if (flags & ~PP_COUNT_INPUT_READY) return fail(PP_EARG, "unknown flags 0x%x", flags);
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (nbytes % (size_t)(width / 8))
    return fail(PP_ELENGTH, "%zu bytes is not a multiple of the %d-byte word size", nbytes,
                width / 8);
  if (!targets || ntargets < 1 || ntargets > PP_MAX_TARGETS)
    return fail(PP_EARG, "need 1..%d target counter arrays, got %d", PP_MAX_TARGETS, ntargets);
  int rc;
  for (int k = 0; k < ntargets; ++k)
    if ((rc = check_device_ptr(targets[k], "targets[k]"))) return rc;
  if (nbytes == 0) return PP_OK;
  if ((rc = check_device_ptr(data, "data"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  pp::CountArgs a{};
  const pp::LoadPath path = load_path();
  pp::split_range(static_cast<const uint8_t *>(data), nbytes, pp::count_chunk_bytes(path), &a);
  a.counters = targets[0];
  a.width = width;
  a.nextra = ntargets - 1;
  for (int k = 1; k < ntargets; ++k) a.extra[k - 1] = targets[k];
  a.input_ready = (flags & PP_COUNT_INPUT_READY) ? 1 : 0;
  cudaError_t e = pp::launch_count(a, path, di, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_multi launch");
  return PP_OK;
}

int pp_ipc_handle(const void *dev_ptr, void *handle72) {
  if (!dev_ptr || !handle72) return fail(PP_EARG, "NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) + 8 == PP_IPC_HANDLE_BYTES, "IPC handle size");
  int rc;
  if ((rc = check_device_ptr(dev_ptr, "dev_ptr"))) return rc;
  // the IPC handle names the whole allocation; the offset travels with it
  unsigned long long base = 0;
  if ((rc = alloc_base(dev_ptr, &base))) return rc;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  const unsigned long long off = reinterpret_cast<uintptr_t>(dev_ptr) - base;
  std::memcpy(handle72, &h, sizeof h);
  std::memcpy(static_cast<char *>(handle72) + sizeof h, &off, 8);
  return PP_OK;
}

int pp_ipc_open(const void *handle72, void **dev_ptr) {
  if (!handle72 || !dev_ptr) return fail(PP_EARG, "NULL argument");
  cudaIpcMemHandle_t h;
  unsigned long long off = 0;
  std::memcpy(&h, handle72, sizeof h);
  std::memcpy(&off, static_cast<const char *>(handle72) + sizeof h, 8);
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<char *>(base) + off;
  std::lock_guard<std::mutex> lk(g_ipc_m);
  g_ipc_base[*dev_ptr] = base;
  return PP_OK;
}

int pp_ipc_close(void *dev_ptr) {
  void *base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_m);
    auto it = g_ipc_base.find(dev_ptr);
    if (it == g_ipc_base.end()) return fail(PP_EARG, "pointer was not returned by pp_ipc_open");
    base = it->second;
    g_ipc_base.erase(it);
  }
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return PP_OK;
}

int pp_count_categories(const void *codes, size_t ncodes, int code_bytes, int width,
                        unsigned long long *counters, void *stream) {
  return pp_count_categories_ex(codes, ncodes, code_bytes, width, counters, 0u, stream);
}

int pp_count_categories_ex(const void *codes, size_t ncodes, int code_bytes, int width,
                           unsigned long long *counters, unsigned int flags, void *stream) {
  if (flags & ~PP_COUNT_INPUT_READY) return fail(PP_EARG, "unknown flags 0x%x", flags);
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4)
    return fail(PP_EARG, "code_bytes must be 1, 2 or 4, got %d", code_bytes);
  int rc;
  if ((rc = check_device_ptr(counters, "counters"))) return rc;
  if (ncodes == 0) return PP_OK;
  if ((rc = check_device_ptr(codes, "codes"))) return rc;
  if ((uintptr_t)codes % (uintptr_t)code_bytes)
    return fail(PP_EARG, "codes must be %d-byte aligned", code_bytes);
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  // One-hot expansion on the TMA pipeline at every code width (faster than
  // the shared-memory histogram everywhere: profiles/r1_categories_ablation.md).
  // PP_CAT_PATH=smem|onehot forces a path (A/B runs).
  const char *force = std::getenv("PP_CAT_PATH");
  const bool onehot = force ? std::strcmp(force, "onehot") == 0 : true;
  if (onehot) {
    // expand to packed one-hot words in registers and run the carry-save
    // counter on the TMA pipeline (frame position = code mod w)
    pp::CountArgs a{};
    pp::split_range(static_cast<const uint8_t *>(codes), (unsigned long long)ncodes * code_bytes,
                    pp::codes8_chunk_bytes(), &a);
    a.counters = counters;
    a.width = width;
    a.rot = 0;
    a.input_ready = (flags & PP_COUNT_INPUT_READY) ? 1 : 0;
    e = pp::launch_count_codes(a, code_bytes, di, static_cast<cudaStream_t>(stream));
  } else {
    // the A/B alternative: per-thread shared-memory histogram columns
    e = pp::launch_categories(static_cast<const uint8_t *>(codes),
                              (unsigned long long)ncodes * code_bytes, code_bytes, width,
                              counters, di, dev, static_cast<cudaStream_t>(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_categories launch");
  return PP_OK;
}

// Lanes per segment: explicit hint in flags bits 8-15, else from the
// (average) segment size: one warp per segment from 16 KiB up, 8 lanes
// (4 segments per warp, 4x fewer transposes per segment) below 8 KiB.
// Lanes per segment: the hint (1, 2, 4, 8, 16 or 32), else from the segment
// length: one lane each for tiny segments (SWAR kernel), else G-lane groups.
// Crossover (scripts/seg_smallG.py): the one-lane kernel wins up to 512 B;
// at 1 KiB G = 8 is 1.75x faster on aligned segments and even on misaligned
// ones (whose partial edge vectors are single loads + masks inside the view).
static constexpr unsigned long long kLaneAutoMaxBytes = 512;
static constexpr unsigned long long kLaneAutoMaxAligned = 512;
// the length seg_lanes assumes when the caller's lengths are unknown (G = 8)
static constexpr unsigned long long kUnknownLengthBytes = 4096;

static int seg_lanes(int flags, unsigned long long avg_bytes, bool vec_aligned = false) {
  const int hint = (flags >> 8) & 0xFF;
  if (hint == 1 || hint == 2 || hint == 4 || hint == 8 || hint == 16 || hint == 32) return hint;
  if (avg_bytes <= (vec_aligned ? kLaneAutoMaxAligned : kLaneAutoMaxBytes)) return 1;
  if (avg_bytes >= 16384) return 32;
  if (avg_bytes >= 8192) return 16;
  return 8;
}

// PP_SEG_BATCH hint (0 = automatic)
static unsigned seg_batch_hint(int flags) { return (unsigned)((flags >> 20) & 0x3F); }

static int seg_common(const pp::SegArgs &a, void *stream) {
  if (!width_ok(a.width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", a.width);
  if (a.nseg == 0) return PP_OK;
  int rc;
  if ((rc = check_device_ptr(a.out, "out"))) return rc;
  if ((rc = check_device_ptr(a.base, "base"))) return rc;
  if (a.seg_off && (rc = check_device_ptr(a.seg_off, "seg_off"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  cudaError_t e = pp::launch_segmented(a, di, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_segmented launch");
  return PP_OK;
}

int pp_count_segmented(const void *base, const unsigned long long *seg_off, size_t nseg,
                       int width, unsigned long long *out, int flags, void *stream) {
  if (!seg_off && nseg) return fail(PP_EARG, "seg_off is NULL");
  pp::SegArgs a{};
  a.base = static_cast<const uint8_t *>(base);
  a.seg_off = seg_off;
  a.nseg = nseg;
  a.out = out;
  a.width = width;
  a.overwrite = (flags & PP_SEG_OVERWRITE) ? 1 : 0;
  a.batch_groups = seg_batch_hint(flags);
  // unknown lengths: G = 8 -- within 10 % of G = 32 on long segments and
  // 15-25 % faster on short or skewed ones (scripts/seg_ragged.py)
  a.lanes_per_segment = seg_lanes(flags, kUnknownLengthBytes);
  // opt-in: tiny arrays one lane each, the rest with G lanes (two passes)
  if ((flags & PP_SEG_HYBRID) && a.lanes_per_segment != 1) a.short_max = kLaneAutoMaxBytes;
  return seg_common(a, stream);
}

int pp_count_segmented_order(const void *base, const unsigned long long *seg_off,
                             const unsigned int *order, size_t nseg, int width,
                             unsigned long long *out, int flags, void *stream) {
  if (!seg_off && nseg) return fail(PP_EARG, "seg_off is NULL");
  if (!order && nseg) return fail(PP_EARG, "order is NULL");
  if (nseg > 0xFFFFFFFFull) return fail(PP_EARG, "order holds 32-bit indices: nseg < 2^32");
  int rc;
  if (nseg && (rc = check_device_ptr(order, "order"))) return rc;
  pp::SegArgs a{};
  a.base = static_cast<const uint8_t *>(base);
  a.seg_off = seg_off;
  a.order = order;
  a.nseg = nseg;
  a.out = out;
  a.width = width;
  a.overwrite = (flags & PP_SEG_OVERWRITE) ? 1 : 0;
  a.batch_groups = seg_batch_hint(flags);
  a.lanes_per_segment = seg_lanes(flags, kUnknownLengthBytes);
  if ((flags & PP_SEG_HYBRID) && a.lanes_per_segment != 1) a.short_max = kLaneAutoMaxBytes;
  return seg_common(a, stream);
}

int pp_count_batch(const unsigned long long *ptrs, const unsigned long long *lens, size_t n,
                   int width, unsigned long long *out, int flags, void *stream) {
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (n == 0) return PP_OK;
  if (!ptrs || !lens) return fail(PP_EARG, "ptrs / lens is NULL");
  int rc;
  if ((rc = check_device_ptr(ptrs, "ptrs"))) return rc;
  if ((rc = check_device_ptr(lens, "lens"))) return rc;
  if ((rc = check_device_ptr(out, "out"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  pp::SegArgs a{};
  a.ptrs = ptrs;
  a.lens = lens;
  a.nseg = n;
  a.out = out;
  a.width = width;
  a.overwrite = (flags & PP_SEG_OVERWRITE) ? 1 : 0;
  a.batch_groups = seg_batch_hint(flags);
  const int g = seg_lanes(flags, kUnknownLengthBytes);  // as for CSR offsets
  a.lanes_per_segment = (g == 2) ? 1 : (g == 4) ? 8 : g;  // no TMA ring for scattered arrays
  cudaError_t e = pp::launch_segmented(a, di, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_batch launch");
  return PP_OK;
}

int pp_count_fixed(const void *base, size_t seg_bytes, size_t nseg, int width,
                   unsigned long long *out, int flags, void *stream) {
  if (width_ok(width) && seg_bytes % (size_t)(width / 8))
    return fail(PP_ELENGTH, "%zu bytes is not a multiple of the %d-byte word size", seg_bytes,
                width / 8);
  pp::SegArgs a{};
  a.base = static_cast<const uint8_t *>(base);
  a.seg_off = nullptr;
  a.seg_bytes = seg_bytes;
  a.nseg = nseg;
  a.out = out;
  a.width = width;
  a.overwrite = (flags & PP_SEG_OVERWRITE) ? 1 : 0;
  a.batch_groups = seg_batch_hint(flags);
  a.lanes_per_segment =
      seg_lanes(flags, seg_bytes, ((uintptr_t)base % 16 == 0) && (seg_bytes % 16 == 0));
  a.chk_lo = (uintptr_t)base;  // the caller's range (checked builds)
  a.chk_hi = (uintptr_t)base + (uintptr_t)(seg_bytes * nseg);
  return seg_common(a, stream);
}

int pp_readonly_sum(const void *data, size_t nbytes, unsigned long long *sink, void *stream) {
  return pp_readonly_sum_ex(data, nbytes, sink, 0u, stream);
}

int pp_readonly_sum_ex(const void *data, size_t nbytes, unsigned long long *sink,
                       unsigned int flags, void *stream) {
  if (flags & ~PP_COUNT_INPUT_READY) return fail(PP_EARG, "unknown flags 0x%x", flags);
  int rc;
  if ((rc = check_device_ptr(sink, "sink"))) return rc;
  if (nbytes == 0) return PP_OK;
  if ((rc = check_device_ptr(data, "data"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  pp::CountArgs a{};
  pp::split_range(static_cast<const uint8_t *>(data), nbytes,
                  pp::count_chunk_bytes(pp::LoadPath::kTma), &a);
  a.input_ready = (flags & PP_COUNT_INPUT_READY) ? 1 : 0;
  cudaError_t e = pp::launch_readonly(a, sink, di, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pp_readonly_sum launch");
  return PP_OK;
}

// ---------------------------------------------------------------- host path
// Host-buffer path.  Per-thread staging context: NBUF device buffers, a copy
// stream and a count stream.  Chunk i is copied H2D into device buffer
// i % NBUF on the copy stream while chunk i-1 is counted on the count stream;
// chunks are word-complete (CHUNK is a multiple of 64), so their counts simply
// add.  Pinned sources are DMA'd directly.  Pageable sources
// (bytes / bytearray / numpy: the reference's own inputs) would be staged by
// the driver on one thread at ~15 GB/s, so they go through NBUF pinned
// buffers filled by a persistent copy pool, overlapped with the DMA of the
// previous chunk and the count of the one before.
namespace {
constexpr int kNbuf = 3;
#ifndef PP_HOST_CHUNK_MIB
#define PP_HOST_CHUNK_MIB 64  // H2D pieces: 32 MiB 55.0, 64 MiB 55.2, 128 MiB 55.3 GB/s (link max 55.4; scripts/e2e_ab.py)
#endif
constexpr size_t kChunk = (size_t)PP_HOST_CHUNK_MIB << 20;

// Parallel memcpy on a persistent pool; the calling thread works too.
// memcpy into a pinned staging buffer with non-temporal stores (PP_HOST_NT=0:
// plain memcpy).  The bytes are read next by the GPU's copy engine, not by
// this CPU: left dirty in the cores' caches they make the DMA snoop every
// line (the last chunk of a call, which nothing evicts, took 1.5 ms for
// 8 MiB); streamed past the caches they are in DRAM when the DMA starts.
inline void stage_copy(void *dst, const void *src, size_t n) {
#if !PP_HAVE_SSE2
  std::memcpy(dst, src, n);  // (no streaming stores written for this host ISA)
#else
  static const bool nt = [] {
    const char *e = std::getenv("PP_HOST_NT");
    return !e || std::atoi(e) != 0;
  }();
  uint8_t *d = static_cast<uint8_t *>(dst);
  const uint8_t *s = static_cast<const uint8_t *>(src);
  if (!nt || ((uintptr_t)d & 15u) || n < 256) {
    std::memcpy(d, s, n);
    return;
  }
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i *>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 48), e);
  }
  if (i < n) std::memcpy(d + i, s + i, n - i);
  _mm_sfence();
#endif
}

class CopyPool {
 public:
  static CopyPool &get() {
    static CopyPool *pool = new CopyPool();  // intentionally leaked (process lifetime)
    return *pool;
  }
  void copy(void *dst, const void *src, size_t n) {
    static const size_t pool_min = [] {  // PP_HOST_POOL_MIN: A/B of the threshold
      const char *env = std::getenv("PP_HOST_POOL_MIN");
      return env ? (size_t)std::strtoull(env, nullptr, 10) : (size_t)(1u << 20);
    }();
    if (workers_.empty() || n < pool_min) {
      stage_copy(dst, src, n);
      return;
    }
    std::lock_guard<std::mutex> one_job(job_m_);
    uint64_t my_gen;
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = static_cast<uint8_t *>(dst);
      src_ = static_cast<const uint8_t *>(src);
      n_ = n;
      const size_t parts = workers_.size() + 1;
      piece_ = ((n + parts - 1) / parts + 4095) & ~(size_t)4095;
      npieces_ = (n + piece_ - 1) / piece_;
      remaining_ = npieces_;
      next_.store(0);
      my_gen = ++gen_;
    }
    cv_.notify_all();
    work(my_gen);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return remaining_ == 0; });
  }

 private:
  CopyPool() {
    const char *env = std::getenv("PP_HOST_COPY_THREADS");
    unsigned hw = std::thread::hardware_concurrency();
    // 3/4 of the host threads, at most 12 (scripts/host_stage_sweep.py)
    long want = env ? std::strtol(env, nullptr, 10) : (long)std::min(12u, std::max(1u, hw * 3 / 4));
    for (long i = 1; i < want; ++i) workers_.emplace_back([this] { loop(); });
    for (auto &t : workers_) t.detach();
  }
  void work(uint64_t gen) {
    for (;;) {
      size_t i;
      uint8_t *d;
      const uint8_t *s;
      size_t len;
      {
        std::lock_guard<std::mutex> lk(m_);
        if (gen != gen_) return;
        i = next_.fetch_add(1);
        if (i >= npieces_) return;
        const size_t off = i * piece_;
        d = dst_ + off;
        s = src_ + off;
        len = std::min(piece_, n_ - off);
      }
      stage_copy(d, s, len);
      std::lock_guard<std::mutex> lk(m_);
      if (--remaining_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      uint64_t g;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        g = seen = gen_;
      }
      work(g);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, job_m_;
  std::condition_variable cv_, done_cv_;
  uint8_t *dst_ = nullptr;
  const uint8_t *src_ = nullptr;
  size_t n_ = 0, piece_ = 0, npieces_ = 0, remaining_ = 0;
  std::atomic<size_t> next_{0};
  uint64_t gen_ = 0;
};

constexpr size_t kStageMax = 16u << 20;  // pinned staging buffers (pageable inputs), each
struct HostCtx {
  int dev = -1;
  cudaStream_t copy = nullptr, count = nullptr;
  void *buf[kNbuf] = {};
  void *pinned[kNbuf] = {};  // staging for pageable sources (allocated on first use)
  cudaEvent_t copied[kNbuf] = {}, freed[kNbuf] = {};
  unsigned long long *dcnt = nullptr;
  unsigned long long *hcnt = nullptr;  // pinned
  // no destructor: the context lives until process exit (tearing CUDA
  // objects down from thread_local destructors races the runtime's own exit).
  void release() {
    if (dev < 0) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    for (int i = 0; i < kNbuf; ++i) {
      if (buf[i]) cudaFree(buf[i]);
      if (pinned[i]) cudaFreeHost(pinned[i]);
      if (copied[i]) cudaEventDestroy(copied[i]);
      if (freed[i]) cudaEventDestroy(freed[i]);
      buf[i] = pinned[i] = nullptr;
      copied[i] = freed[i] = nullptr;
    }
    if (dcnt) cudaFree(dcnt);
    if (hcnt) cudaFreeHost(hcnt);
    if (copy) cudaStreamDestroy(copy);
    if (count) cudaStreamDestroy(count);
    dcnt = nullptr;
    hcnt = nullptr;
    copy = count = nullptr;
    dev = -1;
    cudaSetDevice(cur);
  }
  cudaError_t ensure(int d) {  // the slot of device d (host_ctx): set up once
    if (dev == d) return cudaSuccess;
    release();  // a half-built slot after a failed setup
    cudaError_t e;
    dev = d;
    if ((e = cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking))) return e;
    if ((e = cudaStreamCreateWithFlags(&count, cudaStreamNonBlocking))) return e;
    for (int i = 0; i < kNbuf; ++i) {
      if ((e = cudaMalloc(&buf[i], kChunk))) return e;
      if ((e = cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming))) return e;
      if ((e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming))) return e;
    }
    if ((e = cudaMalloc(&dcnt, 64 * sizeof(unsigned long long)))) return e;
    if ((e = cudaMallocHost(&hcnt, 64 * sizeof(unsigned long long)))) return e;
    return cudaSuccess;
  }
  cudaError_t ensure_pinned() {
    cudaError_t e;
    for (int i = 0; i < kNbuf; ++i)
      if (!pinned[i] && (e = cudaMallocHost(&pinned[i], kStageMax))) return e;
    return cudaSuccess;
  }
};
// Per host thread, one context per device (a thread that alternates devices
// keeps each device's buffers instead of rebuilding or leaking them).
constexpr int kCtxDevs = 64;
thread_local HostCtx g_host[kCtxDevs];

bool host_is_pinned(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
bool is_device_memory(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice;
}
// Per-thread small-call context: device scratch + pinned result counters
// (pp_count_sync), and for small host inputs a 1 MiB pinned staging buffer,
// a 1 MiB device buffer and a stream, so a small pp_count_host is one
// memcpy + five stream operations + one synchronisation.
constexpr size_t kSmallHost = 1u << 20;
// Small and mid-size synchronous calls take the direct path
// (pp_count_direct_kernel / pp_count_direct_multi_kernel): one CTA per 32 KiB
// chunk reads the bytes where they are -- device memory, or the pinned
// small-call buffer over the link -- and the kernel itself writes the counts
// and a sequence flag into mapped pinned memory that the host polls: one
// launch per call instead of memset + launch + D2H copy + stream
// synchronisation (and, for host bytes, the H2D copy).  A/B: PP_NO_DIRECT=1,
// PP_DIRECT_HOST_MAX / PP_DIRECT_DEVICE_MAX (scripts/gpu_direct_ab.sh).
// C-ABI call time, queued -> direct: device bytes -> host counters 19-20 ->
// 14.4-15.5 us up to 4 MiB, 16 MiB 25.4-26.4 -> 17.7-18.7 (above that the
// TMA kernel's stream rate matters more than the saved operations); host
// bytes 8 B..4 KiB 23-27 -> 18.5-20.5 us, 16-32 KiB 33-38 -> 20-21, 128 KiB
// 39 -> 26-27.5, 256 KiB 44.5 -> 34-37, 512 KiB 57.8 -> 47-52 (1 MiB: 77-79
// vs 75-83, a wash, so host bytes stop at 512 KiB).
constexpr size_t kDirectHost = 512u << 10;
constexpr size_t kDirectDevice = 16u << 20;
struct SyncCtx {
  int dev = -1;
  unsigned long long *dcnt = nullptr, *hcnt = nullptr;
  unsigned long long *acc = nullptr;       // direct path: 64 sums + a ticket, zero between calls
  unsigned long long *hcnt_dev = nullptr;  // hcnt / flag as the device addresses them
  unsigned int *flag = nullptr, *flag_dev = nullptr;
  unsigned int seq = 0;
  void *pin = nullptr, *pin_dev = nullptr, *dbuf = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t ensure(int d) {  // the slot of device d (sync_ctx): set up once
    if (dev == d) return cudaSuccess;
    cudaError_t e;
    if (!dcnt && (e = cudaMalloc(&dcnt, 64 * sizeof(unsigned long long)))) return e;
    if (!acc) {
      if ((e = cudaMalloc(&acc, 65 * sizeof(unsigned long long)))) return e;
      if ((e = cudaMemset(acc, 0, 65 * sizeof(unsigned long long)))) return e;
    }
    if (!hcnt) {  // 64 counters + the flag word, mapped
      if ((e = cudaHostAlloc(&hcnt, 65 * sizeof(unsigned long long), cudaHostAllocMapped)))
        return e;
      flag = reinterpret_cast<unsigned int *>(hcnt + 64);
      *flag = 0;
      void *dp = nullptr;
      if ((e = cudaHostGetDevicePointer(&dp, hcnt, 0))) return e;
      hcnt_dev = static_cast<unsigned long long *>(dp);
      flag_dev = reinterpret_cast<unsigned int *>(hcnt_dev + 64);
    }
    dev = d;
    return cudaSuccess;
  }
  cudaError_t ensure_small_host() {
    cudaError_t e;
    if (!pin) {
      if ((e = cudaHostAlloc(&pin, kSmallHost, cudaHostAllocMapped))) return e;
      if ((e = cudaHostGetDevicePointer(&pin_dev, pin, 0))) return e;
    }
    if (!dbuf && (e = cudaMalloc(&dbuf, kSmallHost))) return e;
    if (!st && (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking))) return e;
    return cudaSuccess;
  }
};
thread_local SyncCtx g_sync[kCtxDevs];

// this thread's contexts of device `dev` (nullptr: device index out of range)
HostCtx *host_ctx(int dev) { return dev >= 0 && dev < kCtxDevs ? &g_host[dev] : nullptr; }
SyncCtx *sync_ctx(int dev) { return dev >= 0 && dev < kCtxDevs ? &g_sync[dev] : nullptr; }

bool direct_enabled() {
  static const bool on = std::getenv("PP_NO_DIRECT") == nullptr;
  return on;
}
size_t direct_max(const char *env, size_t dflt) {  // A/B of the size cut-offs
  const char *e = std::getenv(env);
  return e ? (size_t)std::strtoull(e, nullptr, 10) : dflt;
}

// The direct path: one launch of pp_count_direct_kernel over [data, data +
// nbytes) (device-addressable) on st, then poll the flag it writes after the
// counts.  The stream is queried now and then so a failed launch, a faulting
// kernel or an earlier error on the stream ends the wait.
int count_direct(SyncCtx &c, const void *data, size_t nbytes, int width, unsigned long long *out,
                 cudaStream_t st) {
  pp::CountArgs a{};
  pp::split_range(static_cast<const uint8_t *>(data), nbytes,
                  pp::count_chunk_bytes(pp::LoadPath::kLdg), &a);
  a.width = width;
  const unsigned int seq = ++c.seq ? c.seq : ++c.seq;  // never 0 (the initial flag)
  cudaError_t e = pp::launch_count_direct(a, c.acc, c.hcnt_dev, c.flag_dev, seq, st);
  if (e != cudaSuccess) return cuda_fail(e, "pp_count launch");
  volatile unsigned int *f = c.flag;
  for (unsigned spins = 1; *f != seq; ++spins) {
    if (spins == (1u << 16)) {
      // a few milliseconds without a result (the stream or the GPU is busy
      // with other work): stop burning the core, wait the stream's way
      if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "direct count");
      if (*f == seq) break;
      return fail(PP_ECUDA, "direct count finished without publishing its result");
    }
    if ((spins & 0x3FFu) == 0) {
      e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (*f == seq) break;
        return fail(PP_ECUDA, "direct count finished without publishing its result");
      }
      if (e != cudaErrorNotReady) return cuda_fail(e, "direct count");
    }
#if PP_HAVE_SSE2
    _mm_pause();
#endif
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  for (int j = 0; j < width; ++j) out[j] += c.hcnt[j];
  return PP_OK;
}

// Count nbytes (<= kSmallHost) of host memory through the small-call buffers.
int count_small_host(SyncCtx &c, const void *host, size_t nbytes, int width,
                     unsigned long long *out, const pp::DevInfo &di) {
  cudaError_t e;
  if ((e = c.ensure_small_host())) return cuda_fail(e, "pp_count_host setup");
  static const size_t direct_host = direct_max("PP_DIRECT_HOST_MAX", kDirectHost);
  if (nbytes <= direct_host && direct_enabled()) {
    // the CTA reads the pinned copy over the link (its address mod 16 does not
    // matter: counts of a word-complete range do not depend on it)
    stage_copy(c.pin, host, nbytes);
    return count_direct(c, c.pin_dev, nbytes, width, out, c.st);
  }
  if (nbytes >= (256u << 10))
    CopyPool::get().copy(c.pin, host, nbytes);
  else
    stage_copy(c.pin, host, nbytes);
  // same byte alignment on the device as on the host is not needed: counts
  // of a word-complete range do not depend on its address
  if ((e = cudaMemcpyAsync(c.dbuf, c.pin, nbytes, cudaMemcpyHostToDevice, c.st)))
    return cuda_fail(e, "cudaMemcpyAsync");
  if ((e = cudaMemsetAsync(c.dcnt, 0, (size_t)width * 8, c.st))) return cuda_fail(e, "memset");
  int rc;
  if ((rc = count_device(c.dbuf, nbytes, width, c.dcnt, c.st, di))) return rc;
  if ((e = cudaMemcpyAsync(c.hcnt, c.dcnt, (size_t)width * 8, cudaMemcpyDeviceToHost, c.st)))
    return cuda_fail(e, "cudaMemcpyAsync");
  if ((e = cudaStreamSynchronize(c.st))) return cuda_fail(e, "cudaStreamSynchronize");
  for (int j = 0; j < width; ++j) out[j] += c.hcnt[j];
  return PP_OK;
}
}  // namespace

int pp_count_sync(const void *data, size_t nbytes, int width, unsigned long long *host_counters,
                  void *stream) {
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (nbytes % (size_t)(width / 8))
    return fail(PP_ELENGTH, "%zu bytes is not a multiple of the %d-byte word size", nbytes,
                width / 8);
  if (!host_counters) return fail(PP_EARG, "host_counters is NULL");
  if (nbytes == 0) return PP_OK;
  int rc;
  if ((rc = check_device_ptr(data, "data"))) return rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  SyncCtx *c = sync_ctx(dev);
  if (!c) return fail(PP_EARG, "device %d: at most %d devices per process", dev, kCtxDevs);
  cudaError_t e = c->ensure(dev);
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_sync setup");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  static const size_t direct_dev = direct_max("PP_DIRECT_DEVICE_MAX", kDirectDevice);
  if (nbytes <= direct_dev && direct_enabled())
    return count_direct(*c, data, nbytes, width, host_counters, st);
  if ((e = cudaMemsetAsync(c->dcnt, 0, (size_t)width * 8, st)))
    return cuda_fail(e, "cudaMemsetAsync");
  if ((rc = count_device(data, nbytes, width, c->dcnt, st, di))) return rc;
  if ((e = cudaMemcpyAsync(c->hcnt, c->dcnt, (size_t)width * 8, cudaMemcpyDeviceToHost, st)))
    return cuda_fail(e, "cudaMemcpyAsync");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "cudaStreamSynchronize");
  for (int j = 0; j < width; ++j) host_counters[j] += c->hcnt[j];
  return PP_OK;
}

namespace {
// pp_count_host on the CURRENT device (validated arguments, nbytes > 0).
int count_host_current(const void *host_data, size_t nbytes, int width,
                       unsigned long long *host_counters) {
  int rc;
  pp::DevInfo di;
  if ((rc = current_devinfo(&di))) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  SyncCtx *sc = sync_ctx(dev);
  HostCtx *hc = host_ctx(dev);
  if (!sc || !hc) return fail(PP_EARG, "device %d: at most %d devices per process", dev, kCtxDevs);
  if (nbytes <= kSmallHost) {
    if ((e = sc->ensure(dev))) return cuda_fail(e, "pp_count_host setup");
    return count_small_host(*sc, host_data, nbytes, width, host_counters, di);
  }
  e = hc->ensure(dev);
  if (e != cudaSuccess) return cuda_fail(e, "pp_count_host setup");
  HostCtx &h = *hc;
  // pageable sources of >= 2 MiB go through our pinned ring + parallel copy
  // pool (non-temporal stores, stage_copy): 2 / 4 / 8 / 16 / 32 / 256 MiB =
  // 20 / 25 / 35 / 39 / 42 / 49 GB/s against 14 / 15 / 16 / 17 / 13 / 39 for
  // the driver's own pageable path below 32 MiB and cached stores above
  // (scripts/host_fixed_probe.py)
  static const size_t stage_min = [] {  // PP_HOST_STAGE_MIN: A/B of the threshold
    const char *env = std::getenv("PP_HOST_STAGE_MIN");
    return env ? (size_t)std::strtoull(env, nullptr, 10) : (size_t)(2u << 20);
  }();
  const bool staged = nbytes >= stage_min && !host_is_pinned(host_data);
  // staged chunks are smaller so the pool copy of chunk i+1 overlaps the DMA
  // of chunk i even for inputs of a few chunks
  static const size_t stage_chunk = [] {
    const char *env = std::getenv("PP_HOST_STAGE_CHUNK");
    size_t c = env ? (size_t)std::strtoull(env, nullptr, 10) : (size_t)(8u << 20);
    c &= ~(size_t)63;
    return (c < (1u << 20) || c > kStageMax) ? (size_t)(8u << 20) : c;
  }();
  // a few chunks even for mid-size inputs, so the pool copy of chunk i + 1
  // overlaps the DMA of chunk i
  const size_t chunk =
      !staged ? kChunk
              : std::min(stage_chunk, std::max<size_t>(kSmallHost, (nbytes / 4 + 63) & ~(size_t)63));
  if (staged && (e = h.ensure_pinned())) return cuda_fail(e, "pp_count_host staging");
  if ((e = cudaMemsetAsync(h.dcnt, 0, 64 * sizeof(unsigned long long), h.count)))
    return cuda_fail(e, "cudaMemsetAsync");
  const uint8_t *src = static_cast<const uint8_t *>(host_data);
  size_t off = 0;
  for (size_t i = 0; off < nbytes; ++i) {
    const int b = (int)(i % kNbuf);
    const size_t len = (nbytes - off) < chunk ? (nbytes - off) : chunk;
    const void *from = src + off;
    if (staged) {
      // pinned[b] is free once the H2D copy of chunk i - NBUF has completed
      if ((e = cudaEventSynchronize(h.copied[b]))) return cuda_fail(e, "staging wait");
      CopyPool::get().copy(h.pinned[b], src + off, len);
      from = h.pinned[b];
    }
    if ((e = cudaStreamWaitEvent(h.copy, h.freed[b], 0))) return cuda_fail(e, "wait freed");
    if ((e = cudaMemcpyAsync(h.buf[b], from, len, cudaMemcpyHostToDevice, h.copy)))
      return cuda_fail(e, "cudaMemcpyAsync H2D");
    if ((e = cudaEventRecord(h.copied[b], h.copy))) return cuda_fail(e, "record copied");
    if ((e = cudaStreamWaitEvent(h.count, h.copied[b], 0))) return cuda_fail(e, "wait copied");
    if ((rc = count_device(h.buf[b], len, width, h.dcnt, h.count, di))) return rc;
    if ((e = cudaEventRecord(h.freed[b], h.count))) return cuda_fail(e, "record freed");
    off += len;
  }
  if ((e = cudaMemcpyAsync(h.hcnt, h.dcnt, (size_t)width * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, h.count)))
    return cuda_fail(e, "cudaMemcpyAsync D2H");
  if ((e = cudaStreamSynchronize(h.count))) return cuda_fail(e, "cudaStreamSynchronize");
  for (int j = 0; j < width; ++j) host_counters[j] += h.hcnt[j];
  return PP_OK;
}

int host_args_check(const void *host_data, size_t nbytes, int width,
                    const unsigned long long *host_counters) {
  if (!width_ok(width)) return fail(PP_EWIDTH, "word width must be one of (8, 16, 32, 64), got %d", width);
  if (nbytes % (size_t)(width / 8))
    return fail(PP_ELENGTH, "%zu bytes is not a multiple of the %d-byte word size", nbytes,
                width / 8);
  if (!host_counters) return fail(PP_EARG, "host_counters is NULL");
  if (nbytes == 0) return PP_OK;
  if (!host_data) return fail(PP_EARG, "host_data is NULL");
  if (is_device_memory(host_data) || is_device_memory(host_counters))
    return fail(PP_EARG, "pp_count_host takes host buffers (device memory: use pp_count)");
  return PP_OK;
}

// Persistent workers of pp_count_host_multi: worker k runs its range on its
// device with its own (thread-local) staging context, kept across calls.
// One fan-out call at a time (g_fan_call); a worker serves one job at a time.
struct FanJob {
  int dev = 0;
  const void *src = nullptr;
  size_t n = 0;
  int width = 8;
  unsigned long long out[64] = {};
  int rc = PP_OK;
  std::string err;
};
class FanWorker {
 public:
  FanWorker() : th_([this] { loop(); }) { th_.detach(); }
  void post(FanJob *j) {
    std::lock_guard<std::mutex> lk(m_);
    job_ = j;
    done_ = false;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return done_; });
  }

 private:
  void loop() {
    for (;;) {
      FanJob *j;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return job_ != nullptr; });
        j = job_;
      }
      cudaError_t e = cudaSetDevice(j->dev);
      if (e != cudaSuccess) {
        j->rc = cuda_fail(e, "cudaSetDevice");
      } else {
        std::memset(j->out, 0, sizeof j->out);
        j->rc = count_host_current(j->src, j->n, j->width, j->out);
      }
      if (j->rc) j->err = g_err;
      std::lock_guard<std::mutex> lk(m_);
      job_ = nullptr;
      done_ = true;
      done_cv_.notify_all();
    }
  }
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  FanJob *job_ = nullptr;
  bool done_ = true;
  std::thread th_;
};
std::mutex g_fan_call;
FanWorker &fan_worker(int k) {
  static FanWorker *w[PP_MAX_FANOUT] = {};
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  if (!w[k]) w[k] = new FanWorker();  // intentionally leaked (process lifetime)
  return *w[k];
}
}  // namespace

int pp_count_host(const void *host_data, size_t nbytes, int width,
                  unsigned long long *host_counters) {
  int rc;
  if ((rc = host_args_check(host_data, nbytes, width, host_counters)) || nbytes == 0) return rc;
  return count_host_current(host_data, nbytes, width, host_counters);
}

int pp_count_host_multi(const void *host_data, size_t nbytes, int width,
                        unsigned long long *host_counters, const int *devices, int ndevices) {
  int rc;
  if ((rc = host_args_check(host_data, nbytes, width, host_counters))) return rc;
  if (!devices || ndevices < 1 || ndevices > PP_MAX_FANOUT)
    return fail(PP_EARG, "need 1..%d devices, got %d", PP_MAX_FANOUT, ndevices);
  int ndev_visible = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev_visible);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    return fail(PP_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  for (int k = 0; k < ndevices; ++k)
    if (devices[k] < 0 || devices[k] >= ndev_visible)
      return fail(PP_EARG, "devices[%d] = %d: %d devices visible", k, devices[k], ndev_visible);
  if (nbytes == 0) return PP_OK;
  // contiguous ranges cut at multiples of 64 bytes (word-complete for every
  // width): their counts add; tiny inputs use fewer devices
  const size_t units = nbytes / 64;
  int n = ndevices;
  if ((size_t)n > units) n = units ? (int)units : 1;
  std::lock_guard<std::mutex> one_call(g_fan_call);
  FanJob jobs[PP_MAX_FANOUT];
  const uint8_t *src = static_cast<const uint8_t *>(host_data);
  for (int k = 0; k < n; ++k) {
    const size_t lo = units * k / n * 64;
    const size_t hi = (k == n - 1) ? nbytes : units * (k + 1) / n * 64;
    jobs[k].dev = devices[k];
    jobs[k].src = src + lo;
    jobs[k].n = hi - lo;
    jobs[k].width = width;
    fan_worker(k).post(&jobs[k]);
  }
  for (int k = 0; k < n; ++k) fan_worker(k).wait();
  for (int k = 0; k < n; ++k)
    if (jobs[k].rc) {
      g_err = "device " + std::to_string(jobs[k].dev) + ": " + jobs[k].err;
      return jobs[k].rc;
    }
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < width; ++j) host_counters[j] += jobs[k].out[j];
  return PP_OK;
}

// ------------------------------------------------------------ generators
static int gen_check(void *dst, size_t nbytes, size_t unit) {
  if (nbytes % unit) return fail(PP_ELENGTH, "generator length %zu not a multiple of %zu", nbytes, unit);
  if (nbytes == 0) return PP_OK;
  if (((uintptr_t)dst) % unit) return fail(PP_EARG, "generator dst must be %zu-byte aligned", unit);
  return check_device_ptr(dst, "dst");
}

int pp_gen_uniform(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset, void *stream) {
  int rc;
  if ((rc = gen_check(dst, nbytes, 8)) || !nbytes) return rc;
  cudaError_t e = pp::launch_gen_uniform(static_cast<uint64_t *>(dst), nbytes / 8, seed,
                                         word_offset, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_gen_uniform");
}

int pp_gen_bernoulli(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset, uint32_t q,
                     void *stream) {
  int rc;
  if (q > 65536u) return fail(PP_EARG, "q must be in [0, 65536]");
  if ((rc = gen_check(dst, nbytes, 8)) || !nbytes) return rc;
  cudaError_t e = pp::launch_gen_bernoulli(static_cast<uint64_t *>(dst), nbytes / 8, seed,
                                           word_offset, q, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_gen_bernoulli");
}

int pp_gen_blocks(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                  uint64_t block_bytes, void *stream) {
  int rc;
  if (block_bytes == 0 || block_bytes % 8) return fail(PP_EARG, "block_bytes must be a positive multiple of 8");
  if ((rc = gen_check(dst, nbytes, 8)) || !nbytes) return rc;
  cudaError_t e = pp::launch_gen_blocks(static_cast<uint64_t *>(dst), nbytes / 8, seed,
                                        word_offset, block_bytes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_gen_blocks");
}

int pp_gen_codes8(void *dst, size_t n, uint64_t seed, uint64_t offset,
                  const uint32_t *thresholds31, void *stream) {
  int rc;
  if (!thresholds31) return fail(PP_EARG, "thresholds31 is NULL");
  if (n == 0) return PP_OK;
  if ((rc = check_device_ptr(dst, "dst"))) return rc;
  cudaError_t e = pp::launch_gen_codes8(static_cast<uint8_t *>(dst), n, seed, offset,
                                        thresholds31, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_gen_codes8");
}

int pp_gen_onehot32(void *dst, size_t nbytes, uint64_t seed, uint64_t word_offset,
                    const uint32_t *thresholds31, void *stream) {
  int rc;
  if (!thresholds31) return fail(PP_EARG, "thresholds31 is NULL");
  if ((rc = gen_check(dst, nbytes, 4)) || !nbytes) return rc;
  cudaError_t e = pp::launch_gen_onehot32(static_cast<uint32_t *>(dst), nbytes / 4, seed,
                                          word_offset, thresholds31,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_gen_onehot32");
}

}  // extern "C"
