/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Counter-based random numbers and the integer exponential recipe.
 *
 *  - Philox4x32-10: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 *    easy as 1, 2, 3", SC'11 (the Random123 generator).  The paper only asks for
 *    "a synthetic trace using the Poisson process, where inter-arrival times
 *    follow an exponential distribution"; SPEC wants one named substream
 *    per concern.  Reading R32: a draw is indexed by (candidate j, tag),
 *    never by event order.  Pinned by the three Random123 known-answer vectors.
 *
 *  - -ln(U) in Q32 without libm on the sampling path (reading R33): U =
 *    (2u+1)/2^33, log2 via a 4097-entry table T[i] = round(2^32 log2(1+i/4096))
 *    with linear interpolation on the 20 bits below the table index.  Pinned
 *    against libm -log() (relative error < 2e-8) and T against a 50-digit
 *    Decimal evaluation.
 */
#include <math.h>
#include <stdint.h>

#include "oracle.h"

/* Philox4x32 round constants (SC'11 Table 2 / Random123 philox.h). */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: bump before rounds 2..10 */
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* T[i] = round(2^32 * log2(1 + i/4096)), evaluated in long double. */
uint64_t orc_log2_table(uint32_t i) {
  long double x = 1.0L + (long double)i / 4096.0L;
  long double v = log2l(x) * 4294967296.0L;
  return (uint64_t)floorl(v + 0.5L);
}

static uint64_t g_tab[4097];
static int g_tab_ready = 0;

static void ensure_table(void) {
  if (g_tab_ready) return;
  for (uint32_t i = 0; i <= 4096; ++i) g_tab[i] = orc_log2_table(i);
  __atomic_store_n(&g_tab_ready, 1, __ATOMIC_RELEASE);
}

/* ln 2 in Q32, round(0.6931471805599453 * 2^32). */
#define LN2_Q32 2977044472ull

uint64_t orc_neglog_q32(uint32_t u) {
  ensure_table();
  /* U = v / 2^33 with v = 2u + 1 odd in [1, 2^33). */
  uint64_t v = 2ull * (uint64_t)u + 1ull;
  /* e = floor(log2 v): the position of the leading one. */
  uint32_t e = 0;
  while ((v >> (e + 1)) != 0) e++;
  /* the bits below the leading one, as a 32-bit binary fraction */
  uint64_t frac = v - (1ull << e);
  uint32_t x = (uint32_t)(frac << (32 - e)); /* e <= 32 */
  uint32_t i = x >> 20;                      /* 12-bit table index */
  uint64_t f = x & 0xFFFFFu;                 /* 20-bit interpolation weight */
  uint64_t log2v = ((uint64_t)e << 32) + g_tab[i] + (((g_tab[i + 1] - g_tab[i]) * f) >> 20);
  /* -log2 U = 33 - log2 v ; -ln U = -log2 U * ln 2 */
  uint64_t neglog2 = (33ull << 32) - log2v;
  unsigned __int128 prod = (unsigned __int128)neglog2 * LN2_Q32;
  return (uint64_t)(prod >> 32);
}
