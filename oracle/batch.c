/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Runs independent scenarios on a pool of host threads, one scenario per task
 * ("Parallelism is only across independent simulations").
 * Used for the CPU baseline that bench.py reports beside the GPU number.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#include "oracle.h"

typedef struct {
  const orc_inputs *in;
  const uint64_t *sids;
  uint64_t n;
  orc_result *res;
  uint64_t next;
  int err;
} pool;

static void *worker(void *arg) {
  pool *p = (pool *)arg;
  for (;;) {
    uint64_t i = __atomic_fetch_add(&p->next, 1, __ATOMIC_RELAXED);
    if (i >= p->n) break;
    if (orc_run_scenario(p->in, p->sids[i], &p->res[i], NULL)) __atomic_store_n(&p->err, 1, __ATOMIC_RELAXED);
  }
  return NULL;
}

int orc_run_batch(const orc_inputs *in, const uint64_t *sids, uint64_t n, orc_result *res, int nthreads) {
  pool p = {in, sids, n, res, 0, 0};
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  if (!th) return -1;
  int started = 0;
  for (int t = 0; t < nthreads; ++t)
    if (pthread_create(&th[started], NULL, worker, &p) == 0) started++; /* handles stay compact */
  if (started == 0) worker(&p);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
  free(th);
  return p.err ? -1 : 0;
}
