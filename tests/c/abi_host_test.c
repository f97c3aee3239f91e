/*
 * abi_host_test.c — the C ABI driven from plain C, the way a non-Python
 * binding (cgo, JNI, N-API, a C++ service) would drive it: no CUDA headers,
 * no torch, only include/pospopcnt_b200.h and libpospopcnt_b200.so.
 *
 * Checks pp_count_host (host buffers in, host counters out) against the CPU
 * oracle (oracle/liboracle.so — test infrastructure, the checker only) over
 * lengths, host alignments and every width; the error codes of the
 * reference's validation order (kernels.py:315-333); accumulation into the
 * caller's counters; and concurrent calls from several threads with distinct
 * counter arrays (the reference's threading contract).
 *
 *   abi_host_test          full run (needs an sm_100 GPU); exit 0 = pass
 *   abi_host_test --nodev  no-GPU run: every compute call must fail with
 *                          PP_ENODEV (no CPU fallback); validation still works
 */
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pospopcnt_b200.h"

/* oracle/pospopcnt_oracle.c */
int oracle_hs512(const uint8_t *base, size_t offset, size_t n, int w, uint64_t *counters);
void oracle_gen_uniform(uint64_t *dst, size_t nwords, uint64_t seed, uint64_t off);

static int failures = 0;
#define CHECK(cond, ...)                          \
  do {                                            \
    if (!(cond)) {                                \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);               \
      fprintf(stderr, "\n");                      \
      ++failures;                                 \
    }                                             \
  } while (0)

static uint8_t *make_data(size_t n, uint64_t seed) {
  size_t words = n / 8 + 2;
  uint64_t *p = (uint64_t *)malloc(words * 8);
  oracle_gen_uniform(p, words, seed, 0);
  return (uint8_t *)p;
}

static int compare(const uint8_t *data, size_t n, int w, const char *what) {
  unsigned long long got[64];
  uint64_t want[64];
  memset(got, 0, sizeof got);
  memset(want, 0, sizeof want);
  int rc = pp_count_host(data, n, w, got);
  CHECK(rc == PP_OK, "%s: pp_count_host rc=%d (%s)", what, rc, pp_last_error());
  if (rc != PP_OK) return 1;
  oracle_hs512(data, 0, n, w, want);
  for (int j = 0; j < w; ++j)
    if (got[j] != want[j]) {
      CHECK(0, "%s: n=%zu w=%d counter %d: got %llu want %llu", what, n, w, j, got[j],
            (unsigned long long)want[j]);
      return 1;
    }
  return 0;
}

static void test_errors(int have_gpu) {
  unsigned long long c[64] = {0};
  uint8_t b[16] = {0x01, 0x80};
  CHECK(pp_abi_version() == 1, "abi version %d", pp_abi_version());
  CHECK(pp_count_host(b, 2, 12, c) == PP_EWIDTH, "bad width");
  CHECK(pp_count_host(b, 3, 16, c) == PP_ELENGTH, "length not word-complete");
  CHECK(pp_count_host(b, 2, 16, NULL) == PP_EARG, "NULL counters");
  CHECK(pp_count_host(b, 0, 16, c) == PP_OK, "empty input is a no-op");
  for (int k = 0; k <= PP_ENODEV; ++k) CHECK(pp_strerror(k) != NULL, "strerror %d", k);
  int rc = pp_count_host(b, 2, 16, c);
  if (have_gpu) {
    /* the package docstring example (__init__.py:3-5): C[0] = C[15] = 1 */
    CHECK(rc == PP_OK && c[0] == 1 && c[15] == 1 && c[1] == 0, "01 80 at w=16 (rc=%d)", rc);
  } else {
    CHECK(rc == PP_ENODEV, "no GPU must be PP_ENODEV, got %d (%s)", rc, pp_last_error());
    int sms = 0, ma = 0, mi = 0;
    CHECK(pp_device_info(0, &sms, &ma, &mi) != PP_OK, "device info without a GPU");
  }
}

static void test_sweep(void) {
  const size_t sizes[] = {1, 7, 8, 15, 16, 17, 64, 1000, 4096 + 24, 65536 + 8,
                          (1u << 20) + 40, (33u << 20) + 8, (80u << 20) + 16};
  uint8_t *data = make_data((80u << 20) + 64, 0xABCDEF);
  char what[64];
  for (size_t i = 0; i < sizeof sizes / sizeof sizes[0]; ++i)
    for (int off = 0; off < 8; off += (sizes[i] > (1u << 20) ? 3 : 1))
      for (int w = 8; w <= 64; w *= 2) {
        size_t n = sizes[i] - sizes[i] % (size_t)(w / 8);
        snprintf(what, sizeof what, "sweep off=%d", off);
        compare(data + off, n, w, what);
      }
  /* accumulation: counters are added into, not overwritten */
  unsigned long long c[64];
  uint64_t want[64] = {0};
  for (int j = 0; j < 64; ++j) c[j] = 1000;
  CHECK(pp_count_host(data + 5, 4096, 32, c) == PP_OK, "accumulate");
  oracle_hs512(data + 5, 0, 4096, 32, want);
  for (int j = 0; j < 32; ++j) CHECK(c[j] == want[j] + 1000, "accumulate counter %d", j);
  for (int j = 32; j < 64; ++j) CHECK(c[j] == 1000, "counters past w untouched (%d)", j);
  free(data);
}

struct job {
  const uint8_t *data;
  size_t n;
  int w, bad;
};

static void *worker(void *arg) {
  struct job *j = (struct job *)arg;
  for (int it = 0; it < 4; ++it) j->bad += compare(j->data, j->n, j->w, "thread");
  return NULL;
}

static void test_threads(void) {
  enum { T = 4 };
  pthread_t th[T];
  struct job jobs[T];
  uint8_t *bufs[T];
  for (int t = 0; t < T; ++t) {
    size_t n = ((size_t)(t + 1) << 22) + 8 * t;
    bufs[t] = make_data(n, 100 + t);
    jobs[t] = (struct job){bufs[t] + t, n, 8 << (t % 4), 0};
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < T; ++t) {
    pthread_join(th[t], NULL);
    CHECK(jobs[t].bad == 0, "thread %d mismatches", t);
    free(bufs[t]);
  }
}

int main(int argc, char **argv) {
  const int nodev = argc > 1 && strcmp(argv[1], "--nodev") == 0;
  test_errors(!nodev);
  if (!nodev) {
    test_sweep();
    test_threads();
  }
  if (failures) {
    fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  printf("ok\n");
  return 0;
}
