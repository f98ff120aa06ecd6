/* select_oracle.c — TEST ORACLE ONLY (never linked into the product).
 *
 * Scalar C restatement of OpTable.select (configurator.py:239-300) with OpTable.scores
 * (219-227) and OpTable._argmin (229-237), looped over a batch of invocations so that
 * full-size (2^20 x 4096) parity checks finish in seconds.  Arithmetic follows the numpy
 * evaluation order exactly; compile with -ffp-contract=off so no FMA is formed.
 * Tables are concatenated: table t owns entries [tab_off[t], tab_off[t+1]).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

static int better_tie(int64_t i, int64_t j, const double* cost, const double* res,
                      const int64_t* id_rank) {
  /* configurator.py:236  min(ties, key=lambda i: (cost[i], res[i], id_rank[i])) */
  if (cost[i] != cost[j]) return cost[i] < cost[j];
  if (res[i] != res[j]) return res[i] < res[j];
  return id_rank[i] < id_rank[j];
}

/* masked argmin with exact-equality ties (configurator.py:229-237) over [a, b) */
static int64_t argmin(int64_t a, int64_t b, const double* score, const double* cost,
                      const double* res, const int64_t* id_rank, const unsigned char* mask) {
  double best = INFINITY;
  for (int64_t j = a; j < b; ++j) {
    double m = mask[j - a] ? score[j - a] : INFINITY;
    if (m < best) best = m;
  }
  int64_t pick = -1;
  for (int64_t j = a; j < b; ++j) {
    double m = mask[j - a] ? score[j - a] : INFINITY;
    if (m == best) {
      if (pick < 0 || better_tie(j - a, pick - a, cost, res + a, id_rank + a)) pick = j;
    }
  }
  return pick;
}

int oracle_select_batch(const int64_t* tab_off, const double* lat, const double* res,
                        const int64_t* batch, const double* pool, const double* price,
                        const int64_t* gkind, const int64_t* id_rank, int K, double alpha,
                        int64_t N, const int32_t* op, const double* slack, const int32_t* avail,
                        const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                        int32_t* out_code, int32_t* out_idx, int32_t* out_fill, double* out_obj,
                        double* out_slack, double* out_wait, uint8_t* out_feas, int64_t max_m) {
  int rc = 0;
#pragma omp parallel
  {
    double* score = (double*)__builtin_alloca(sizeof(double) * (size_t)max_m);
    double* cost = (double*)__builtin_alloca(sizeof(double) * (size_t)max_m);
    unsigned char* mask = (unsigned char*)__builtin_alloca((size_t)max_m);
    unsigned char* mask2 = (unsigned char*)__builtin_alloca((size_t)max_m);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
      const int t = op ? op[i] : 0;
      const int64_t a = tab_off[t], b = tab_off[t + 1], M = b - a;
      const double* s = slack + i * K;
      const uint32_t fl = flags[i];
      const int av = avail[i], mb = min_batch[i];
      int any = 0;
      for (int64_t j = 0; j < M; ++j) {
        int64_t e = a + j;
        unsigned char m = 1;
        if ((fl >> (8 + gkind[e])) & 1u) m = 0;          /* excluded_kinds (259-263) */
        if (mb > 1 && batch[e] < mb) m = 0;               /* min_batch (264-265) */
        mask[j] = m;
        any |= m;
        double c = ((res[e] * lat[e]) * price[e]) / (double)batch[e];
        double pen = alpha * ((lat[e] * res[e]) / ((double)batch[e] * pool[e]));
        cost[j] = c;
        score[j] = c + ((lat[e] < s[gkind[e]]) ? 0.0 : pen);
      }
      out_wait[i] = 0.0;
      if (!any) {
        out_code[i] = 0; out_idx[i] = -1; out_fill[i] = 0; out_obj[i] = 0.0;
        out_slack[i] = 0.0; out_feas[i] = 0;
        continue;
      }
      int64_t e = argmin(a, b, score, cost, res, id_rank, mask);
      int64_t B = batch[e];
      double sk = s[gkind[e]];
      if ((fl & 1u) && B > av && (int64_t)supply[i] >= B - av) {
        double wait = sk - lat[e];
        if (wait > 0.0) {
          out_code[i] = 2; out_idx[i] = (int32_t)(e - a); out_fill[i] = av;
          out_obj[i] = score[e - a]; out_slack[i] = sk; out_wait[i] = wait;
          out_feas[i] = lat[e] < sk;
          continue;
        }
      }
      if (B > av) {
        int any2 = 0;
        for (int64_t j = 0; j < M; ++j) {
          mask2[j] = mask[j] && batch[a + j] <= av;
          any2 |= mask2[j];
        }
        if (any2) e = argmin(a, b, score, cost, res, id_rank, mask2);
      }
      B = batch[e];
      sk = s[gkind[e]];
      out_code[i] = 1; out_idx[i] = (int32_t)(e - a); out_fill[i] = (int32_t)(B < av ? B : av);
      out_obj[i] = score[e - a]; out_slack[i] = sk; out_feas[i] = lat[e] < sk;
    }
  }
  return rc;
}
