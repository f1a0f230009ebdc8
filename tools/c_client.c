/* c_client.c -- the drop-in boundary from plain C: no Python, no torch.
 * Boots a session on device 0, runs round-robin empty round trips, a
 * zero-copy int32 vector add on four workers (host-mapped buffers), checks
 * the sums, exercises an error path, and disposes.  Exit status 0 = pass.
 *
 *   gcc -O2 -std=c11 -I include tools/c_client.c \
 *       -L paper_2310_01212_b200 -llk -Wl,-rpath,$PWD/paper_2310_01212_b200 -o tools/c_client
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "lk.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    int rc_ = (call);                                                                \
    if (rc_ != LK_OK) {                                                              \
      fprintf(stderr, "%s -> %s: %s\n", #call, lk_strerror(rc_), lk_last_error()); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

int main(void) {
  lk_config cfg;
  memset(&cfg, 0, sizeof cfg);   /* zeros select the defaults: one worker per SM, DIRECT polling */
  cfg.device = 0;
  lk_session* s = NULL;
  uint64_t ns = 0;
  CHECK(lk_create(&cfg, &s, &ns));
  uint32_t nw = 0;
  CHECK(lk_num_workers(s, &nw));
  const uint32_t nwords = (nw + 63) / 64;
  uint64_t mask[4] = {0, 0, 0, 0};

  /* slot 0: the empty task; slot 1: a zero-copy vector add */
  lk_desc empty;
  memset(&empty, 0, sizeof empty);
  empty.kind = LK_KIND_EMPTY;
  CHECK(lk_register_desc(s, 0, &empty, NULL, 0));
  uint64_t total_ns = 0;
  for (uint32_t k = 0; k < 20000; ++k) {
    memset(mask, 0, sizeof mask);
    const uint32_t w = k % nw;
    mask[w / 64] = 1ull << (w % 64);
    uint64_t t = 0, d = 0;
    CHECK(lk_trigger(s, mask, nwords, 0, NULL, &t));
    CHECK(lk_wait(s, mask, nwords, &d));
    total_ns += d;
  }

  const uint64_t n = 100003;
  void *ha = NULL, *hb = NULL, *ho = NULL;
  CHECK(lk_host_alloc(0, 4 * n, &ha));
  CHECK(lk_host_alloc(0, 4 * n, &hb));
  CHECK(lk_host_alloc(0, 4 * n, &ho));
  int32_t *a = (int32_t*)ha, *b = (int32_t*)hb, *o = (int32_t*)ho;
  lk_desc add;
  memset(&add, 0, sizeof add);
  add.kind = LK_KIND_VECTOR_ADD_I32;
  add.n = n;
  add.in0 = (uint64_t)(uintptr_t)ha;
  add.in1 = (uint64_t)(uintptr_t)hb;
  add.out = (uint64_t)(uintptr_t)ho;
  memset(mask, 0, sizeof mask);
  mask[0] = 0xF;   /* four workers shard the payload */
  for (int rep = 0; rep < 50; ++rep) {
    for (uint64_t i = 0; i < n; ++i) {
      a[i] = (int32_t)(i * 2654435761u + (uint32_t)rep);
      b[i] = (int32_t)(~i * 40503u - (uint32_t)rep);
    }
    CHECK(lk_trigger(s, mask, nwords, 1, rep == 0 ? &add : NULL, &ns));
    CHECK(lk_wait(s, mask, nwords, &ns));
    for (uint64_t i = 0; i < n; ++i)
      if (o[i] != (int32_t)((uint32_t)a[i] + (uint32_t)b[i])) {
        fprintf(stderr, "vector add mismatch at rep %d index %llu\n", rep, (unsigned long long)i);
        return 1;
      }
  }

  /* the reference's error behaviour: re-triggering a busy worker is refused */
  memset(mask, 0, sizeof mask);
  mask[0] = 1;
  lk_desc busy;
  memset(&busy, 0, sizeof busy);
  busy.kind = LK_KIND_BUSY_LOOP;
  busy.iterations = 200000;
  CHECK(lk_trigger(s, mask, nwords, 2, &busy, &ns));
  const int rc = lk_trigger(s, mask, nwords, 3, &empty, &ns);
  if (rc != LK_E_BUSY) {
    fprintf(stderr, "expected LK_E_BUSY, got %d\n", rc);
    return 1;
  }
  CHECK(lk_wait(s, mask, nwords, &ns));

  CHECK(lk_dispose(s, &ns));
  CHECK(lk_destroy(s));
  lk_host_free(ha);
  lk_host_free(hb);
  lk_host_free(ho);
  printf("c_client ok: %u workers, 20000 round trips (mean trigger->done %.2f us), 50 checked zero-copy adds\n",
         nw, total_ns / 20000.0 / 1e3);
  return 0;
}
