/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * a2: arrival + natural-length generation; a3: per-request model draws.
 *
 * Poisson arrivals with exponential inter-arrival times over a piecewise-linear
 * rate trace ("synthetic trace using the Poisson process, where
 * inter-arrival times follow an exponential distribution ... distinct phases
 * when the request arrivals ramp up, stay put, and ramp down").  Ramps are
 * sampled by thinning at the phase's maximum rate.  Readings R17, R32,
 * R33: per-segment lambda_max; a candidate crossing the segment end is
 * discarded (its index consumed) and the next segment restarts at its start;
 * one global candidate index j; accept with probability lambda(tau)/lambda_max
 * decided exactly in integers.
 *
 * Attributes: L = Ltab[u2>>20], input = Itab[u3>>20] (S:84 workload profile);
 * per request, a second Philox block (tag 1) gives Fvar, predictor noise and the
 * compliance factor (readings R14, R39).
 */
#include <stdint.h>
#include <stdlib.h>

#include "oracle.h"

#define SEED_HI 0xB311A000u

/* Draw the Philox block of candidate j, tag t, for scenario sid. */
static void block(const orc_inputs *in, uint64_t sid, uint32_t j, uint32_t tag, uint32_t out[4]) {
  uint64_t wid = in->sc_wid[sid];
  uint32_t ctr[4] = {j, tag, (uint32_t)wid, (uint32_t)(wid >> 32)};
  orc_philox(in->sc_seed[sid], SEED_HI, ctr, out);
}

/* per-request model draws (a3) of request index j from its tag-1 block */
static void draws(const orc_inputs *in, uint64_t sid, uint32_t j, orc_request *r) {
  uint32_t v[4];
  block(in, sid, j, 1, v);
  int64_t fvar = in->tab_fvar[v[0] >> 20];
  int64_t noise = in->tab_noise[v[1] >> 20];
  int64_t fcomp = in->tab_fcomp[v[2] >> 20];
  int64_t U = ((int64_t)r->L * fvar + 32768) / 65536; /* U = max(1, round(L Fvar)) (R14) */
  r->U = (uint32_t)(U < 1 ? 1 : U);
  int64_t P = (int64_t)r->L + noise; /* P = max(1, L + Laplace noise) */
  r->P = (uint32_t)(P < 1 ? 1 : P);
  r->fcomp_q16 = (int32_t)fcomp;
  r->qnoise = in->tab_qnoise[v[3] >> 20]; /* similarity noise (NEXT-2) */
}

int64_t orc_arrivals(const orc_inputs *in, uint64_t sid, orc_request *out, uint64_t cap_out) {
  uint32_t tr = in->sc_trace[sid];
  if (in->trace_kind[tr] == 1) { /* NEXT-4 replay: the list as given, j = index */
    uint32_t off = in->trace_knot_off[tr], n = in->trace_n_knots[tr], cap = in->trace_cap[tr];
    if (cap && cap < n) n = cap;
    if (!out) return n;
    if (n > cap_out) return -1;
    for (uint32_t k = 0; k < n; ++k) {
      orc_request *r = &out[k];
      r->a_us = (uint64_t)in->arr_a[off + k];
      r->j = k;
      r->L = in->arr_L[off + k];
      r->input = in->arr_input[off + k];
      r->cls = in->arr_cls[off + k];
      draws(in, sid, k, r);
    }
    return n;
  }
  uint32_t off = in->trace_knot_off[tr], nk = in->trace_n_knots[tr];
  uint32_t cap = in->trace_cap[tr];
  const int64_t *kt = in->knot_t + off;
  const uint32_t *kl = in->knot_lam + off;
  int64_t count = 0;
  uint32_t j = 0;
  for (uint32_t s = 0; s + 1 < nk; ++s) {
    uint64_t ta = (uint64_t)kt[s], tb = (uint64_t)kt[s + 1];
    uint64_t la = kl[s], lb = kl[s + 1];
    uint64_t lmax = la > lb ? la : lb;
    if (lmax == 0 || tb <= ta) continue; /* no candidates from a zero-rate phase */
    /* mean inter-arrival at lambda_max = 1e9 / lmax µs; M = floor(2^32 * 1e9 / lmax) */
    uint64_t M = (uint64_t)(((unsigned __int128)1000000000ull << 32) / lmax);
    uint64_t tau = ta;
    for (;;) {
      uint32_t u[4];
      block(in, sid, j, 0, u);
      uint32_t jj = j++;
      uint64_t nl = orc_neglog_q32(u[0]);
      uint64_t delta = (uint64_t)(((unsigned __int128)nl * M) >> 64);
      tau += delta;
      if (tau >= tb) break; /* crosses the phase end: discarded, restart at tb */
      /* thinning: accept iff u1/2^32 < lambda(tau)/lambda_max, with
       * lambda(tau) = (la (tb - tau) + lb (tau - ta)) / (tb - ta) exactly */
      unsigned __int128 lhs = (unsigned __int128)((uint64_t)u[1] * lmax) * (tb - ta);
      unsigned __int128 rhs = ((unsigned __int128)la * (tb - tau) + (unsigned __int128)lb * (tau - ta)) << 32;
      if (!(lhs < rhs)) continue;
      if (out) {
        if ((uint64_t)count >= cap_out) return -1;
        orc_request *r = &out[count];
        r->a_us = tau;
        r->j = jj;
        r->L = (uint32_t)in->tab_L[u[2] >> 20];
        r->input = (uint32_t)in->tab_I[u[3] >> 20];
        /* class from the 20 low bits of the word whose top 12 bits drew L (NEXT-3) */
        r->cls = 3;
        for (uint32_t c = 0; c < 4; ++c)
          if ((u[2] & 0xFFFFFu) < in->class_cum[c]) { r->cls = c; break; }
        draws(in, sid, jj, r);
      }
      count++;
      if (cap && (uint64_t)count >= cap) return count; /* arrival cap (R28) */
    }
  }
  return count;
}
