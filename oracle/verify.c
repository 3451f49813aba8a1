/* Multi-threaded drivers of the C oracle for full-scale parity runs
 * (TEST INFRASTRUCTURE ONLY; scripts/verify_full.py).
 *
 *   ov_cells            scan_gather's grouping (sigstore.cpp:228-286) of every
 *                       (band, bucket) cell over all bands and buckets at once:
 *                       a counting sort by cell, rows ascending inside a cell.
 *   ov_compare_cells    compare_bucket (compare.cpp:24-67) over every cell with
 *                       the reference oracle's exact early exit (oracle.cpp:81-92:
 *                       once mismatches exceed H - min_matches the pair is
 *                       rejected), then the full count for survivors; cells are
 *                       dealt to threads dynamically.  Output: accepted (lo, hi,
 *                       match) row triples, unsorted, with repeats across cells.
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* cell = band * K + bucket; offsets[cells + 1], rows[n * bands] */
int ov_cells(const uint32_t* band, uint64_t n, uint32_t bands, uint32_t K, uint64_t* offsets,
             uint32_t* rows) {
  const uint64_t cells = (uint64_t)bands * K;
  uint64_t i, j;
  memset(offsets, 0, sizeof(uint64_t) * (cells + 1));
  for (i = 0; i < n; ++i)
    for (j = 0; j < bands; ++j) {
      uint32_t b = band[i * bands + j];
      if (b >= K) return -1;
      ++offsets[j * K + b + 1];
    }
  for (i = 0; i < cells; ++i) offsets[i + 1] += offsets[i];
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (cells ? cells : 1));
  if (!cur) return -2;
  memcpy(cur, offsets, sizeof(uint64_t) * cells);
  for (i = 0; i < n; ++i)
    for (j = 0; j < bands; ++j) rows[cur[j * K + band[i * bands + j]]++] = (uint32_t)i;
  free(cur);
  return 0;
}

typedef struct {
  uint32_t *lo, *hi, *m;
  uint64_t n, cap;
} ov_out;

static int ov_push(ov_out* o, uint32_t lo, uint32_t hi, uint32_t m) {
  if (o->n == o->cap) {
    uint64_t c = o->cap ? 2 * o->cap : 4096;
    uint32_t* a = (uint32_t*)realloc(o->lo, c * 4);
    uint32_t* b = (uint32_t*)realloc(o->hi, c * 4);
    uint32_t* d = (uint32_t*)realloc(o->m, c * 4);
    if (!a || !b || !d) return -1;
    o->lo = a;
    o->hi = b;
    o->m = d;
    o->cap = c;
  }
  o->lo[o->n] = lo;
  o->hi[o->n] = hi;
  o->m[o->n] = m;
  ++o->n;
  return 0;
}

typedef struct {
  const uint32_t* sig;
  uint32_t H;
  const uint64_t* offsets;
  const uint32_t* rows;
  uint64_t ncells;
  uint64_t num, den;
  uint32_t min_match;
  _Atomic uint64_t next;
  _Atomic uint64_t candidates;
  ov_out* outs;
  int err;
} ov_job;

static void* ov_worker(void* arg) {
  void** a = (void**)arg;
  ov_job* job = (ov_job*)a[0];
  ov_out* out = (ov_out*)a[1];
  const uint32_t H = job->H;
  const uint32_t allowed = H - job->min_match;
  uint64_t cand = 0;
  for (;;) {
    uint64_t c = atomic_fetch_add(&job->next, 1);
    if (c >= job->ncells) break;
    const uint64_t s = job->offsets[c], n = job->offsets[c + 1] - s;
    const uint32_t* rows = job->rows + s;
    cand += n * (n > 0 ? n - 1 : 0) / 2;
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t* x = job->sig + (uint64_t)rows[i] * H;
      for (uint64_t j = i + 1; j < n; ++j) {
        const uint32_t* y = job->sig + (uint64_t)rows[j] * H;
        /* the first min(H, 32) positions without branches (vectorised), then
           position by position with the early exit */
        const uint32_t head = H < 32 ? H : 32;
        uint32_t miss = 0, h = 0;
        for (; h < head; ++h) miss += x[h] != y[h];
        if (miss > allowed) continue;
        for (; h < H; ++h) {
          miss += x[h] != y[h];
          if (miss > allowed) break;
        }
        if (miss > allowed) continue;
        const uint32_t m = H - miss;
        if (or_accepts(m, H, job->num, job->den) && ov_push(out, rows[i], rows[j], m) != 0) {
          job->err = -1;
          return NULL;
        }
      }
    }
  }
  atomic_fetch_add(&job->candidates, cand);
  return NULL;
}

/* Returns the number of accepted triples (malloc'd arrays in *lo, *hi, *m, to
 * be released with free); *candidates = sum n(n-1)/2. */
int64_t ov_compare_cells(const uint32_t* sig, uint32_t H, const uint64_t* offsets,
                         const uint32_t* rows, uint64_t ncells, uint64_t num, uint64_t den,
                         int threads, uint32_t** lo, uint32_t** hi, uint32_t** m,
                         uint64_t* candidates) {
  ov_job job;
  memset(&job, 0, sizeof job);
  job.sig = sig;
  job.H = H;
  job.offsets = offsets;
  job.rows = rows;
  job.ncells = ncells;
  job.num = num;
  job.den = den;
  job.min_match = or_min_matches(H, num, den);
  if (job.min_match > H) job.min_match = H + 1;
  if (job.min_match > H) { /* threshold 1 with strict acceptance: nothing passes */
    *lo = *hi = *m = NULL;
    *candidates = 0;
    return 0;
  }
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  ov_out* outs = (ov_out*)calloc((size_t)threads, sizeof(ov_out));
  void** args = (void**)calloc((size_t)threads * 2, sizeof(void*));
  for (int t = 0; t < threads; ++t) {
    args[2 * t] = &job;
    args[2 * t + 1] = &outs[t];
    pthread_create(&th[t], NULL, ov_worker, &args[2 * t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) total += outs[t].n;
  *lo = (uint32_t*)malloc((total ? total : 1) * 4);
  *hi = (uint32_t*)malloc((total ? total : 1) * 4);
  *m = (uint32_t*)malloc((total ? total : 1) * 4);
  uint64_t o = 0;
  for (int t = 0; t < threads; ++t) {
    if (outs[t].n) {
      memcpy(*lo + o, outs[t].lo, outs[t].n * 4);
      memcpy(*hi + o, outs[t].hi, outs[t].n * 4);
      memcpy(*m + o, outs[t].m, outs[t].n * 4);
    }
    o += outs[t].n;
    free(outs[t].lo);
    free(outs[t].hi);
    free(outs[t].m);
  }
  free(th);
  free(outs);
  free(args);
  *candidates = atomic_load(&job.candidates);
  return job.err ? -1 : (int64_t)total;
}

void ov_free(void* p) { free(p); }
