// sp_des_host.h — host-side construction of the run engine's image and per-run arena layout
// (plain C++, shared by sp_des.cu and the CPU test harness tests/des_host.cpp).
//
// build_image validates an sp_des_spec and derives what the reference derives in
// PipelineRun.__init__ (manager.py:262-271: in-degrees, ancestors, the deep-first op order) and
// PipelineDag.depths (pipeline.py:328-337); plan_run sizes one replica's arena from the traces of
// a call (item-buffer bounds per op from the branch predicates and fan-outs of every frame).
#pragma once

#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "slackpipe_b200.h"
#include "sp_des.cuh"

namespace spdes {

struct HostImage {
  Image im;
  std::vector<double> dcols;   // lat0, lat_init, res, batch, pool, price, base, per_item
  std::vector<int32_t> icols;  // batch, kind, rank, cfg, then the path suffixes
  std::vector<int32_t> preds_of;  // scratch: per op sorted predecessors (CSR)
  std::vector<int32_t> pred_off;
  double cap_scale = 1.25;
};

SPD_HD Entries entries_view(const double* d, const int32_t* i, int n) {
  Entries e;
  e.lat0 = d;
  e.lat_init = d + n;
  e.res = d + 2 * (size_t)n;
  e.batch = d + 3 * (size_t)n;
  e.pool = d + 4 * (size_t)n;
  e.price = d + 5 * (size_t)n;
  e.base = d + 6 * (size_t)n;
  e.per_item = d + 7 * (size_t)n;
  e.bint = i;
  e.kind = i + n;
  e.rank = i + 2 * (size_t)n;
  e.cfg = i + 3 * (size_t)n;
  e.suf = i + 4 * (size_t)n;
  return e;
}

inline bool build_image(const sp_des_spec& s, HostImage& h, std::string& err) {
  Image& im = h.im;
  std::memset(&im, 0, sizeof(im));
  const int V = s.n_ops, K = s.n_kinds, N = s.n_entries;
  if (V < 1 || V > kMaxOps) return err = "run engine: 1..64 operations", false;
  if (K < 1 || K > kMaxKinds) return err = "run engine: 1..16 backend kinds", false;
  if (N < 1 || s.n_attrs < 0 || s.n_cfg_ids < 1) return err = "run engine: bad sizes", false;
  if (!s.entry_off || !s.lat || !s.lat_init || !s.res || !s.batch || !s.kind || !s.id_rank ||
      !s.cfg_id || !s.truth_base || !s.truth_per_item || !s.ref_index || !s.ref_latency ||
      !s.succ_off || !s.fanout_attr || !s.suffix_off || !s.suffix_ops || !s.instances ||
      !s.inst_resources || !s.price || !s.cq_capacity)
    return err = "run engine: missing spec array", false;
  const int n_edges = s.succ_off[V];
  if (n_edges < 0 || n_edges > kMaxEdges) return err = "run engine: at most 512 edges", false;
  if (n_edges > 0 && (!s.succ || !s.pred_attr || !s.pred_cmp || !s.pred_value))
    return err = "run engine: missing edge arrays", false;
  if (s.entry_off[0] != 0 || s.entry_off[V] != N) return err = "run engine: bad entry_off", false;
  im.n_ops = V;
  im.n_kinds = K;
  im.n_entries = N;
  im.n_attrs = s.n_attrs;
  im.n_cfg = s.n_cfg_ids;
  im.abl = s.ablations;
  im.dfp_count = s.dfp_count;
  im.draws = s.draws;
  im.alpha = s.alpha;
  im.beta = s.beta;
  im.timeout_factor = s.timeout_factor;
  im.dispatch = s.dispatch_overhead;
  im.straggle_factor = s.straggle_factor;
  for (int o = 0; o <= V; ++o) im.entry_off[o] = s.entry_off[o];
  for (int o = 0; o < V; ++o) {
    const int M = s.entry_off[o + 1] - s.entry_off[o];
    if (M < 1 || M > 32767) return err = "run engine: 1..32767 entries per operation", false;
    if (s.ref_index[o] < -1 || s.ref_index[o] >= M) return err = "run engine: bad ref_index", false;
    im.ref_index[o] = s.ref_index[o];
    im.ref_lat0[o] = s.ref_latency[o];
    im.fanout_attr[o] = s.fanout_attr[o];
    if (s.fanout_attr[o] >= s.n_attrs) return err = "run engine: bad fan-out attribute", false;
  }
  // edges, in-degrees, predecessor lists
  std::vector<std::vector<int>> preds(V);
  for (int o = 0; o <= V; ++o) im.succ_off[o] = s.succ_off[o];
  for (int o = 0; o < V; ++o)
    for (int q = s.succ_off[o]; q < s.succ_off[o + 1]; ++q) {
      const int d = s.succ[q];
      if (d < 0 || d >= V || d == o) return err = "run engine: bad successor", false;
      if (q > s.succ_off[o] && s.succ[q - 1] >= d) return err = "run engine: successors must be sorted", false;
      im.succ[q] = d;
      im.pred_attr[q] = s.pred_attr[q];
      im.pred_cmp[q] = s.pred_cmp[q];
      im.pred_val[q] = s.pred_value[q];
      if (s.pred_attr[q] >= s.n_attrs || s.pred_cmp[q] < 0 || s.pred_cmp[q] > 5)
        return err = "run engine: bad branch predicate", false;
      preds[d].push_back(o);
    }
  for (int o = 0; o < V; ++o) im.indeg[o] = (int)preds[o].size();
  // topological order (Kahn) -> depths (pipeline.py:328-337); cycles rejected
  std::vector<int> indeg(V), order;
  for (int o = 0; o < V; ++o) indeg[o] = im.indeg[o];
  for (int o = 0; o < V; ++o)
    if (!indeg[o]) order.push_back(o);
  for (size_t i = 0; i < order.size(); ++i)
    for (int q = s.succ_off[order[i]]; q < s.succ_off[order[i] + 1]; ++q)
      if (--indeg[s.succ[q]] == 0) order.push_back(s.succ[q]);
  if ((int)order.size() != V) return err = "pipeline contains a cycle", false;
  for (int o = 0; o < V; ++o) im.depth[o] = 0;
  for (int v : order)
    for (int q = s.succ_off[v]; q < s.succ_off[v + 1]; ++q)
      im.depth[s.succ[q]] = std::max(im.depth[s.succ[q]], im.depth[v] + 1);
  // ancestors (pipeline.py:339-347) as bit masks, in topological order
  for (int v : order) {
    uint64_t m = 0;
    for (int p : preds[v]) m |= (1ull << p) | im.anc_mask[p];
    im.anc_mask[v] = m;
  }
  // deep-first op order (manager.py:271): (-depth, name); ops are in name order
  std::vector<int> df(V);
  for (int o = 0; o < V; ++o) df[o] = o;
  std::stable_sort(df.begin(), df.end(), [&](int a, int b) { return im.depth[a] > im.depth[b]; });
  for (int o = 0; o < V; ++o) im.deep_first[o] = df[o];
  im.n_inputs = 0;
  for (int o = 0; o < V; ++o)
    if (im.indeg[o] == 0) im.inputs[im.n_inputs++] = o;
  // join staging: each join vertex gets indeg slots per frame; join_pos = the source's slot
  int st = 0;
  for (int o = 0; o < V; ++o) {
    im.join_base[o] = -1;
    if (im.indeg[o] > 1) {
      im.join_base[o] = st;
      st += im.indeg[o];
    }
  }
  im.staging_per_frame = st;
  for (int o = 0; o < V; ++o)
    for (int q = s.succ_off[o]; q < s.succ_off[o + 1]; ++q) {
      const int d = s.succ[q];
      im.join_pos[q] = 0;
      if (im.indeg[d] > 1) {
        for (int j = 0; j < im.indeg[d]; ++j)
          if (preds[d][j] == o) im.join_pos[q] = j;
      }
    }
  // suffixes (configurator.py:413-420)
  const int nsuf = s.suffix_off[V];
  if (nsuf > kMaxSuffixInts) return err = "run engine: path suffixes exceed 4M ints", false;
  for (int o = 0; o <= V; ++o) im.suf_off[o] = s.suffix_off[o];
  for (int o = 0; o < V; ++o) {
    int cnt = 0;
    for (int p = s.suffix_off[o]; p < s.suffix_off[o + 1];) {
      const int len = s.suffix_ops[p];
      if (len < 1 || p + 1 + len > s.suffix_off[o + 1]) return err = "run engine: bad suffix list", false;
      for (int j = 0; j < len; ++j)
        if (s.suffix_ops[p + 1 + j] < 0 || s.suffix_ops[p + 1 + j] >= V)
          return err = "run engine: bad suffix op", false;
      p += 1 + len;
      ++cnt;
    }
    if (cnt < 1) return err = "operation does not appear on any path", false;
    if (cnt > 32) return err = "run engine: at most 32 path suffixes per operation", false;
  }
  // fleet
  int inst = 0;
  std::vector<int> wcap(K, 0);
  for (int k = 0; k < K; ++k) {
    if (s.instances[k] < 1 || s.inst_resources[k] < 1 || s.cq_capacity[k] < 1)
      return err = "run engine: bad backend", false;
    im.inst_off[k] = inst;
    inst += s.instances[k];
    im.inst_res[k] = s.inst_resources[k];
    im.pool_res[k] = (double)((int64_t)s.instances[k] * s.inst_resources[k]);
    im.price[k] = s.price[k];
    im.cap[k] = s.cq_capacity[k];
  }
  im.inst_off[K] = inst;
  // entry columns
  h.dcols.assign(8 * (size_t)N, 0.0);
  h.icols.assign(4 * (size_t)N + nsuf, 0);
  for (int i = 0; i < nsuf; ++i) h.icols[4 * (size_t)N + i] = s.suffix_ops[i];
  for (int g = 0; g < N; ++g) {
    const int k = s.kind[g];
    if (k < 0 || k >= K) return err = "run engine: bad entry kind", false;
    if (s.batch[g] < 1 || s.res[g] < 1.0 || s.res[g] > s.inst_resources[k])
      return err = "run engine: entry does not fit its backend", false;
    if (s.cfg_id[g] < 0 || s.cfg_id[g] >= s.n_cfg_ids) return err = "run engine: bad cfg id", false;
    h.dcols[g] = s.lat[g];
    h.dcols[N + g] = s.lat_init[g];
    h.dcols[2 * (size_t)N + g] = s.res[g];
    h.dcols[3 * (size_t)N + g] = (double)s.batch[g];
    h.dcols[4 * (size_t)N + g] = im.pool_res[k];
    h.dcols[5 * (size_t)N + g] = s.price[k];
    h.dcols[6 * (size_t)N + g] = s.truth_base[g];
    h.dcols[7 * (size_t)N + g] = s.truth_per_item[g];
    h.icols[g] = s.batch[g];
    h.icols[N + g] = k;
    h.icols[2 * (size_t)N + g] = s.id_rank[g];
    h.icols[3 * (size_t)N + g] = s.cfg_id[g];
    wcap[k] += 1;
  }
  im.w_off[0] = 0;
  for (int k = 0; k < K; ++k) im.w_off[k + 1] = im.w_off[k] + wcap[k];
  return true;
}

static inline int64_t align16(int64_t x) { return (x + 15) & ~(int64_t)15; }

// Size one replica's arena for this call: item bounds per op = max over replicas of the items
// the trace can push into the op's buffer (every predicate-passing edge, fan-out counts summed
// over a join's in-edges), invocations <= items * cap_scale.
inline bool plan_run(HostImage& h, int T, const int32_t* frame_off, const int32_t* attrs,
                     int draw_cap, int log_cap, std::string& err, int ev_cap = 0) {
  Image& im = h.im;
  const int V = im.n_ops;
  std::vector<int64_t> cap(V, 0), tot(V), mult(V);
  int frames_cap = 0;
  std::vector<int> order;
  {  // topological order again (inputs first)
    std::vector<int> indeg(V);
    for (int o = 0; o < V; ++o) indeg[o] = im.indeg[o];
    for (int o = 0; o < V; ++o)
      if (!indeg[o]) order.push_back(o);
    for (size_t i = 0; i < order.size(); ++i)
      for (int q = im.succ_off[order[i]]; q < im.succ_off[order[i] + 1]; ++q)
        if (--indeg[im.succ[q]] == 0) order.push_back(im.succ[q]);
  }
  for (int r = 0; r < T; ++r) {  // per trace
    const int f0 = frame_off[r], f1 = frame_off[r + 1];
    if (f1 < f0) return err = "run engine: bad frame_off", false;
    frames_cap = std::max(frames_cap, f1 - f0);
    std::fill(tot.begin(), tot.end(), 0);
    for (int f = f0; f < f1; ++f) {
      const int32_t* at = attrs + (int64_t)f * im.n_attrs;
      std::fill(mult.begin(), mult.end(), 0);
      for (int v : order) {
        if (im.indeg[v] == 0) mult[v] = 1;
        tot[v] += mult[v];
        for (int q = im.succ_off[v]; q < im.succ_off[v + 1]; ++q) {
          const int d = im.succ[q];
          if (im.pred_attr[q] >= 0 && !pred_eval(im.pred_cmp[q], at[im.pred_attr[q]], im.pred_val[q]))
            continue;
          const int64_t n = im.fanout_attr[d] >= 0 ? at[im.fanout_attr[d]] : 1;
          if (n > 0) mult[d] += mult[v] * n;
        }
      }
    }
    for (int o = 0; o < V; ++o) cap[o] = std::max(cap[o], tot[o]);
  }
  int64_t items = 0, off = 0;
  for (int o = 0; o < V; ++o) {
    im.buf_off[o] = (int32_t)off;
    off += cap[o];
    items += cap[o];
  }
  if (off > (int64_t)1 << 30) return err = "run engine: trace too large", false;
  im.buf_off[V] = (int32_t)off;
  // invocation slots are recycled (sp_des.cuh maybe_free): the live set is a fraction of the
  // invocations a run forms (AMBER: <= 1k live of ~8k formed, 17.5k items); a replica that still
  // runs out reports a capacity status and the host re-runs it with cap_scale doubled
  const int64_t inv_cap = std::min<int64_t>((int64_t)((double)items * h.cap_scale) + 256,
                                            (int64_t)((double)items * h.cap_scale / 4) + 1024);
  if (inv_cap > (int64_t)1 << 30) return err = "run engine: trace too large", false;
  im.inv_cap = (int32_t)inv_cap;
  im.seg_cap = (int32_t)(2 * inv_cap);
  int64_t res_total = 0;
  for (int k = 0; k < im.n_kinds; ++k)
    res_total += (int64_t)(im.inst_off[k + 1] - im.inst_off[k]) * im.inst_res[k];
  (void)res_total;
  im.heap_cap = (int32_t)(2 * inv_cap + V + 64);  // completions + straggler wakes + hold wakes
  im.event_cap = 64 * (int64_t)((double)items * h.cap_scale + 256) + 4096;  // runaway guard
  im.frames_cap = frames_cap;
  im.draw_cap = draw_cap;
  im.log_cap = log_cap;
  im.ev_cap = ev_cap;
  const int K = im.n_kinds, N = im.n_entries;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = align16(o + bytes);
    return at;
  };
  // the small per-run state every event touches first (one contiguous block: a few cache lines
  // and one page), then the large arrays
  im.o_opi = take(4 * (int64_t)V * kOpiN);
  im.o_scver = take(4 * (int64_t)V);
  im.o_scval = take(8 * (int64_t)V * K);
  im.o_holddl = take(8 * (int64_t)V * 4);  // hold deadlines, r_min, r_max, ratio versions
  im.o_wkey = take(4 * 2 * (int64_t)std::max(im.w_off[K], 1));
  im.o_wcnt = take(4 * 2 * (int64_t)std::max(im.w_off[K], 1));
  im.o_cfg = take(4 * (int64_t)((im.n_cfg + 31) / 32));
  im.o_lat = take(24 * (int64_t)N);  // lat / cost / costpen (host harness, lane-group forms)
  im.o_obs = take(N);
  im.o_free = take(4 * (int64_t)std::max(im.inst_off[K], 1));
  im.o_heap = take((int64_t)sizeof(HeapEnt) * im.heap_cap);
  im.o_inv = take((int64_t)sizeof(Inv) * (inv_cap + 1));
  im.o_next = take(4 * (inv_cap + 1));
  im.o_live = take(4 * (inv_cap + 1));
  im.o_list = take((int64_t)sizeof(List) * (inv_cap + 1));
  im.o_free_slot = take(4 * (inv_cap + 1));
  im.o_seg = take((int64_t)sizeof(Seg) * im.seg_cap);
  im.o_free_seg = take(4 * (int64_t)im.seg_cap);
  im.o_buf = take(4 * std::max<int64_t>(off, 1));
  im.o_staging = take(4 * std::max<int64_t>((int64_t)frames_cap * im.staging_per_frame, 1));
  im.arena_bytes = align16(o);
  return true;
}

}  // namespace spdes
