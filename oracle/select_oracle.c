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

/* ---- Alg. 1 slack over an explicit path list ---------------------------------------------
 * Literal restatement of Configurator._suffixes (configurator.py:415-417), _path_ratios
 * (493-509) and slack_by_kind (526-543): for every op column v, every path containing v
 * contributes own / (left-to-right sum of the suffix from v); per kind the slack is the
 * first-minimum of ratio * ((target - now) - Q[k]).  Paths are lists of ref columns
 * (path p = path_nodes[path_off[p] .. path_off[p+1])).  out_slack is I x V x K; columns on
 * no path are written as NaN (the reference raises for them, configurator.py:418-420). */
int oracle_slack_paths(int64_t I, int V, int K, const double* ref, const double* target,
                       const double* now, const double* Q, int n_paths, const int32_t* path_off,
                       const int32_t* path_nodes, double* out_slack) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < I; ++i) {
    const double* r = ref + i * V;
    for (int v = 0; v < V; ++v) {
      double ratios[256];
      int nr = 0;
      for (int p = 0; p < n_paths; ++p) {
        int at = -1;
        for (int q = path_off[p]; q < path_off[p + 1]; ++q)
          if (path_nodes[q] == v) { at = q; break; }
        if (at < 0) continue;
        double total = 0.0;
        for (int q = at; q < path_off[p + 1]; ++q) total += r[path_nodes[q]];
        if (nr < 256) ratios[nr++] = r[v] / total;
      }
      for (int k = 0; k < K; ++k) {
        double budget = (target[i] - now[i]) - Q[i * K + k];
        double s = NAN;
        for (int q = 0; q < nr; ++q) {
          double x = ratios[q] * budget;
          if (q == 0 || x < s) s = x;
        }
        out_slack[(i * V + v) * K + k] = s;
      }
    }
  }
  return 0;
}

/* ---- Alg. 1 slack on a DAG by the forward left-to-right DP --------------------------------
 * The restatement SURVEY.md §8(c) validated against compute_slack (0 / 128,045) and
 * oracle/slack.py dp_ratios / dp_slack restate: vertices in topological order (order[s] is
 * the ref column of position s), predecessors as a CSR over positions, terminal flags per
 * position.  hi[src] = lo[src] = 0.0 + ref[src]; hi[v] = max_p hi[p] + ref[v],
 * lo[v] = min_p lo[p] + ref[v]; Tmax / Tmin over reachable terminals; slack =
 * (budget >= 0 ? own/Tmax : own/Tmin) * budget.  out_slack[i][order[s]][k] (I x V x K);
 * out_ratio (optional) [i][order[s]][{lo, hi}]. */
int oracle_slack_dp(int64_t I, int V, int K, const double* ref, const double* target,
                    const double* now, const double* Q, const int32_t* order,
                    const int32_t* pred_off, const int32_t* pred_idx, const uint8_t* terminal,
                    double* out_slack, double* out_ratio) {
#pragma omp parallel
  {
    double hi[1024], lo[1024], rv[1024];
    unsigned char seen[1024];
#pragma omp for schedule(static)
    for (int64_t i = 0; i < I; ++i) {
      for (int s = 0; s < V; ++s) rv[s] = ref[i * V + order[s]];
      for (int src = 0; src < V; ++src) {
        for (int s = 0; s < V; ++s) seen[s] = 0;
        hi[src] = lo[src] = 0.0 + rv[src];
        seen[src] = 1;
        for (int v = src + 1; v < V; ++v) {
          int any = 0;
          double h = 0.0, l = 0.0;
          for (int q = pred_off[v]; q < pred_off[v + 1]; ++q) {
            int p = pred_idx[q];
            if (!seen[p]) continue;
            if (!any || hi[p] > h) h = hi[p];
            if (!any || lo[p] < l) l = lo[p];
            any = 1;
          }
          if (!any) continue;
          seen[v] = 1;
          hi[v] = h + rv[v];
          lo[v] = l + rv[v];
        }
        int anyt = 0;
        double tmax = 0.0, tmin = 0.0;
        for (int v = src; v < V; ++v) {
          if (!seen[v] || !terminal[v]) continue;
          if (!anyt || hi[v] > tmax) tmax = hi[v];
          if (!anyt || lo[v] < tmin) tmin = lo[v];
          anyt = 1;
        }
        double own = rv[src];
        double rlo = own / tmax, rhi = own / tmin;
        int col = order[src];
        if (out_ratio) {
          out_ratio[(i * V + col) * 2 + 0] = rlo;
          out_ratio[(i * V + col) * 2 + 1] = rhi;
        }
        for (int k = 0; k < K; ++k) {
          double b = (target[i] - now[i]) - Q[i * K + k];
          out_slack[(i * V + col) * K + k] = (b >= 0 ? rlo : rhi) * b;
        }
      }
    }
  }
  return 0;
}

/* ---- feedback fold ------------------------------------------------------------------------
 * Sequential restatement of PipelineRun._apply_feedback (manager.py:436-457): per
 * observation in completion order, completed_ref / obs_count bookkeeping, the EWMA
 * apply_feedback (manager.py:45-47: beta*obs + (1-beta)*old), and the gate lift
 * (Configurator.recalibrate_unobserved, configurator.py:470-491) when the reference entry's
 * completion count reaches dfp_count.  One table; state arrays are updated in place. */
int oracle_fold(int64_t M, double* lat, const double* lat_init, int64_t ref_index,
                int64_t* completed_ref, int64_t* obs_count, int64_t n, const int32_t* idx,
                const double* obs, double beta, int64_t dfp_count) {
  for (int64_t j = 0; j < n; ++j) {
    int64_t e = idx[j];
    if (e < 0 || e >= M) return -1;
    if (e == ref_index) *completed_ref += 1;
    obs_count[e] += 1;
    lat[e] = beta * obs[j] + (1.0 - beta) * lat[e];
    if (e == ref_index && *completed_ref == dfp_count && ref_index >= 0) {
      double init_ref = lat_init[ref_index];
      if (init_ref > 0.0) {
        double ratio = lat[ref_index] / init_ref;
        for (int64_t i = 0; i < M; ++i) {
          if (i == ref_index || obs_count[i] > 0) continue;
          lat[i] = lat_init[i] * ratio;
        }
      }
    }
  }
  return 0;
}
