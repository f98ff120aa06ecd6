// sp_des.cuh — the replica-parallel run engine: one tuned pipeline
// run of the reference (manager.py PipelineRun + backend.py BackendSim + the Configurator's
// queues, configurator.py:368-772) as a sequential event loop that one GPU thread executes per
// replica.  Every replica owns a fixed-stride arena in HBM (its mutable tables, invocations,
// item buffers, event heap, queue weights); the static run image (tables, DAG, fleet) is shared.
//
// The code is plain C++ on purpose (no CUDA intrinsics, no FMA: the library is built with
// --fmad=false and every product / sum is written in the reference's association order) so the
// same source is compiled for the device (k_des_run in sp_des.cu) and, by the CPU test suite
// only, for the host (tests/des_host.cpp), where it is checked against oracle/engine.py and the
// reference engine on machines without a GPU.  The product path is the device kernel.
//
// Exactness notes (cited per function below):
//   * the event heap orders by (time, code, seq) like heapq over backend.py:210-213's tuples;
//   * slack_by_kind is cached per op keyed by the weight version only (configurator.py:526-543):
//     a cached value may carry an earlier clock, so it is called exactly where the reference calls it;
//   * Eq. 2 sums the SQ weights then the CQ weights of a kind in dict insertion order
//     (configurator.py:511-524, _weights_add 553-561: an existing key keeps its place);
//   * selection is the reference's literal masked argmin over the op's entries with ties broken
//     by (cost, res, id_rank) (configurator.py:219-300), in numpy's operation order.
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define SPD_HD __host__ __device__ __forceinline__
#define SPD_HDN __host__ __device__ __noinline__
#else
#define SPD_HD inline
#define SPD_HDN
#endif

namespace spdes {

constexpr int kMaxOps = 64;
constexpr int kMaxKinds = 16;
constexpr int kMaxEdges = 512;
constexpr int kMaxSuffixInts = 1 << 22;  // path-suffix ints (kept with the entry columns)

// ablation bits (configurator.py:23)
constexpr int kAblFb = 1, kAblDfp = 2, kAblSdb = 4, kAblEslc = 8, kAblPbc = 16;
// draw bits: which of the reference's per-start RNG draws the scenario makes (backend.py:52-57,
// 186): the host supplies them per start in the reference's stream order
constexpr int kDrawNoise = 1, kDrawStraggle = 2, kDrawFail = 4;

// replica status codes
constexpr int kOk = 0, kErrInvCap = 1, kErrHeapCap = 2, kErrSegCap = 3, kErrLivelock = 4,
              kErrNoConfig = 5, kErrNonFinite = 6, kErrDrawCap = 7, kErrWeightCap = 8,
              kErrBufCap = 9, kErrEventCap = 10, kErrNoTruth = 11;

// invocation states (manager.py:33-42)
constexpr uint8_t kPending = 0, kSpeculated = 1, kCommitted = 3, kRunning = 4, kCompleted = 5,
                  kFailed = 6, kDuplicated = 7;
constexpr uint8_t kBitForced = 1, kBitDupSpawned = 2, kBitWillFail = 4, kBitResolved = 8,
                  kBitWakePending = 16;

struct alignas(16) Image {  // static run description, shared by every replica (built by sp_des_create)
  int32_t n_ops, n_kinds, n_entries, n_attrs, n_cfg;
  int32_t abl, dfp_count, draws;
  double alpha, beta, timeout_factor, dispatch, straggle_factor;
  int32_t n_inputs;
  int32_t inputs[kMaxOps];
  int32_t entry_off[kMaxOps + 1];
  int32_t ref_index[kMaxOps];
  double ref_lat0[kMaxOps];
  int32_t depth[kMaxOps], deep_first[kMaxOps], indeg[kMaxOps];
  uint64_t anc_mask[kMaxOps];
  int32_t succ_off[kMaxOps + 1];
  int32_t succ[kMaxEdges];
  int32_t pred_attr[kMaxEdges], pred_cmp[kMaxEdges], pred_val[kMaxEdges];  // per succ slot
  int32_t join_pos[kMaxEdges];  // position of the source among the join's predecessors
  int32_t join_base[kMaxOps];   // staging base of a join vertex (units of frames), -1 otherwise
  int32_t fanout_attr[kMaxOps];
  int32_t suf_off[kMaxOps + 1];
  double pool_res[kMaxKinds], price[kMaxKinds];
  int32_t inst_res[kMaxKinds], inst_off[kMaxKinds + 1], cap[kMaxKinds];
  int32_t w_off[kMaxKinds + 1];  // weight-list capacity per kind (prefix)
  // per-replica arena layout (filled per run by sp_des_run)
  int32_t inv_cap, seg_cap, heap_cap, log_cap, draw_cap, frames_cap, staging_per_frame, ev_cap, pad0;
  int64_t event_cap;
  int32_t buf_off[kMaxOps + 1];  // item buffer of each op (ints)
  int64_t o_lat, o_obs, o_inv, o_next, o_live, o_list, o_seg, o_buf, o_heap, o_wkey, o_wcnt,
      o_scver, o_scval, o_holddl, o_free, o_staging, o_cfg, o_opi, o_free_slot, o_free_seg,
      arena_bytes;
};

struct Entries {  // static per-entry columns (table order: ops sorted by name, entries in spec order)
  const double *lat0, *lat_init, *res, *batch, *pool, *price, *base, *per_item;
  const int32_t *bint, *kind, *rank, *cfg;
  const int32_t* suf;  // per op: [len, ops...] per path suffix containing it (Image::suf_off)
};

struct Inv {  // 72 B (manager.py:49-80 Invocation, backend.py:86-99 RunningInvocation)
  double spec_slack, spec_obj, com_slack, started_at, threshold, actual;
  int32_t unit;  // slot of the unit's first invocation (it holds the unit's items and counters)
  int32_t iid;   // invocation id (manager.py:303-305)
  int16_t spec_e, com_e;
  int32_t instance;
  uint8_t op, state, bits, pad;
};

struct Seg {
  int32_t pos, n, next;
};
struct List {
  int32_t count, first, last;
};
struct HeapEnt {
  double t;
  uint32_t key;  // code << 31 | seq (backend.py:207-213: (time, code, seq))
  int32_t payload;  // complete: iid; wake: iid (timeout) or -(op + 1) (hold)
};

struct EvRec {  // one BackendSim.trace row (backend.py:207, 243): start / complete / fail
  double t;
  int32_t iid;
  int32_t meta;  // event (0 start, 1 complete, 2 fail) | kind << 2 | instance << 8
};

struct LogRec {  // one decision_log row (configurator.py:608-618, 746-749)
  double t, slack, obj;
  int32_t iid;
  int32_t meta;  // op | entry << 8 | commit << 31
};

// per-op integer state block (o_opi): buffer head/tail, sq head/tail/len, unspawned,
// completed_ref, hold flag
constexpr int kOpiBufHead = 0, kOpiBufTail = 1, kOpiSqHead = 2, kOpiSqTail = 3, kOpiSqLen = 4,
              kOpiUnspawned = 5, kOpiCompletedRef = 6, kOpiHold = 7, kOpiN = 8;

struct Out {  // per-replica result
  double latency, cost, now;
  int32_t peak_slots, peak_heap;
  int32_t status, met, completed, failures, dups, invocations, terminal, n_spec, n_commit,
      configs_used, log_len, events, ev_len, pad;
};

struct Sel {
  int code;  // 0 none, 1 assign, 2 delay
  int e, fill;
  double obj, slack, wait;
};

SPD_HD bool pred_eval(int cmp, int a, int b) {  // pipeline.py:21-28
  switch (cmp) {
    case 0: return a < b;
    case 1: return a <= b;
    case 2: return a > b;
    case 3: return a >= b;
    case 4: return a == b;
    default: return a != b;
  }
}

struct Run {
  const Image& im;
  const Entries& E;
  // replica inputs
  const int32_t* attrs;  // [n_frames][n_attrs]
  int32_t n_frames;
  double target;
  const double* draw_factor;  // [draw_cap] exp(N(0, sigma)) per start, or null
  const uint8_t* draw_bits;   // [draw_cap] bit0 straggled, bit1 will_fail, or null
  LogRec* log;
  EvRec* evlog = nullptr;  // optional event trace (im.ev_cap rows)
  // mutable entry columns lat / cost / cost + penalty: entry g of column c at tab[(c*N + g) * ts]
  // (device: the 32 replicas of a warp interleaved, ts = 32, so converged scans coalesce)
  double* tab;
  int32_t ts;
  // arena views
  uint8_t* observed;
  Inv* inv;
  int32_t *next, *live;
  List* lists;
  Seg* segs;
  int32_t* items;
  HeapEnt* heap;
  int32_t *wkey, *wcnt;
  int32_t* scver;
  double *scval, *holddl, *rmin, *rmax;
  int32_t* rver;
  int32_t *freeres, *staging;
  uint32_t* cfg_used;
  int32_t* opi;
  // scalars
  double now = 0.0;
  int32_t version = 0, seq = 0, next_id = 0, running = 0, n_seg = 0, heap_n = 0, n_starts = 0;
  // invocation slots and item-list segments are recycled (free stacks) once nothing refers to them
  int32_t n_slot = 0, n_free_slot = 0, n_free_seg = 0, live_slots = 0, peak_slots = 0, peak_heap = 0;
  int32_t *free_slot, *free_seg;
  int32_t wn[2][kMaxKinds];
  // Eq. 2 per kind, cached until the kind's weight list or a latency of one of its entries
  // changes (a pure function of both, so the cache never changes a value)
  double qv[kMaxKinds];
  int32_t qver[kMaxKinds], kver[kMaxKinds];
  int32_t ref_version = 0;
  int32_t cq_head[kMaxKinds], cq_tail[kMaxKinds], cq_len[kMaxKinds];
  double total_cost = 0.0, last_accept = 0.0;
  int32_t failures = 0, dups = 0, completed = 0, met = 0, terminal = 0, n_spec = 0, n_commit = 0,
          log_len = 0, ev_len = 0, status = kOk;
  int64_t events = 0;
  int32_t lane = 0, nl = 1;  // lanes per run: this lane's index among the run's nl lanes
  uint32_t lmask = 0xffffffffu;  // the run's lanes within the warp

  SPD_HD Run(const Image& im_, const Entries& e_, char* arena, double* tab_, int32_t ts_,
             const int32_t* attrs_, int32_t nf, double tgt, const double* dfac, const uint8_t* dbits,
             LogRec* log_)
      : im(im_), E(e_), attrs(attrs_), n_frames(nf), target(tgt), draw_factor(dfac),
        draw_bits(dbits), log(log_), tab(tab_), ts(ts_) {
    observed = (uint8_t*)(arena + im.o_obs);
    inv = (Inv*)(arena + im.o_inv);
    next = (int32_t*)(arena + im.o_next);
    live = (int32_t*)(arena + im.o_live);
    lists = (List*)(arena + im.o_list);
    segs = (Seg*)(arena + im.o_seg);
    items = (int32_t*)(arena + im.o_buf);
    heap = (HeapEnt*)(arena + im.o_heap);
    wkey = (int32_t*)(arena + im.o_wkey);
    wcnt = (int32_t*)(arena + im.o_wcnt);
    scver = (int32_t*)(arena + im.o_scver);
    scval = (double*)(arena + im.o_scval);
    holddl = (double*)(arena + im.o_holddl);
    rmin = holddl + im.n_ops;
    rmax = holddl + 2 * im.n_ops;
    rver = (int32_t*)(holddl + 3 * im.n_ops);
    freeres = (int32_t*)(arena + im.o_free);
    staging = (int32_t*)(arena + im.o_staging);
    cfg_used = (uint32_t*)(arena + im.o_cfg);
    opi = (int32_t*)(arena + im.o_opi);
    free_slot = (int32_t*)(arena + im.o_free_slot);
    free_seg = (int32_t*)(arena + im.o_free_seg);
  }

  SPD_HD int32_t& OP(int op, int f) { return opi[op * kOpiN + f]; }
  SPD_HD double lat(int g) const { return tab[(size_t)g * ts]; }
  SPD_HD double cost(int g) const { return tab[(size_t)(im.n_entries + g) * ts]; }
  SPD_HD double costpen(int g) const { return tab[(size_t)(2 * im.n_entries + g) * ts]; }
  // OpTable.set_latency (configurator.py:211-213) + the Eq. 1 terms of the entry in numpy's order
  // (configurator.py:224-225): score = lat < slack ? cost + 0.0 : cost + penalty
  SPD_HDN void set_lat(int g, double L) {
    const double R = E.res[g], B = E.batch[g];
    const double c = ((R * L) * E.price[g]) / B;
    const double pen = im.alpha * ((L * R) / (B * E.pool[g]));
    ++kver[E.kind[g]];
    tab[(size_t)g * ts] = L;
    tab[(size_t)(im.n_entries + g) * ts] = c;
    tab[(size_t)(2 * im.n_entries + g) * ts] = c + pen;
  }
  SPD_HD void error(int code) {
    if (status == kOk) status = code;
  }

  // ---- initial state (manager.py:210-300, configurator.py:375-438) --------------------------
  SPD_HDN void init() {
    #pragma unroll 1
    for (int k = 0; k < kMaxKinds; ++k) {
      kver[k] = 0;
      qver[k] = -1;
    }
    #pragma unroll 1
    for (int i = 0; i < im.n_entries; ++i) {
      set_lat(i, E.lat0[i]);
      observed[i] = 0;
    }
    #pragma unroll 1
    for (int o = 0; o < im.n_ops; ++o) {
      #pragma unroll 1
      for (int f = 0; f < kOpiN; ++f) OP(o, f) = 0;
      OP(o, kOpiSqHead) = OP(o, kOpiSqTail) = -1;
      scver[o] = -1;
      rver[o] = -1;
    }
    #pragma unroll 1
    for (int k = 0; k < im.n_kinds; ++k) {
      wn[0][k] = wn[1][k] = 0;
      cq_head[k] = cq_tail[k] = -1;
      cq_len[k] = 0;
      #pragma unroll 1
      for (int i = im.inst_off[k]; i < im.inst_off[k + 1]; ++i) freeres[i] = im.inst_res[k];
    }
    #pragma unroll 1
    for (int64_t i = 0; i < (int64_t)n_frames * im.staging_per_frame; ++i) staging[i] = 0;
    #pragma unroll 1
    for (int i = 0; i < (im.n_cfg + 31) / 32; ++i) cfg_used[i] = 0;
  }

  // ---- event heap: heapq over (time, code, seq) (backend.py:207-233) -----------------------
  SPD_HD bool less(const HeapEnt& a, const HeapEnt& b) const {
    return a.t < b.t || (a.t == b.t && a.key < b.key);
  }
  SPD_HDN void push(double t, int code, int32_t payload) {
    if (heap_n >= im.heap_cap) {
      error(kErrHeapCap);
      return;
    }
    ++seq;
    HeapEnt x{t, ((uint32_t)code << 31) | (uint32_t)seq, payload};
    int i = heap_n++;
    if (heap_n > peak_heap) peak_heap = heap_n;
    #pragma unroll 1
    while (i > 0) {
      const int p = (i - 1) >> 1;
      if (!less(x, heap[p])) break;
      heap[i] = heap[p];
      i = p;
    }
    heap[i] = x;
  }
  SPD_HDN HeapEnt pop() {
    HeapEnt top = heap[0];
    const HeapEnt x = heap[--heap_n];
    int i = 0;
    #pragma unroll 1
    for (;;) {
      int c = 2 * i + 1;
      if (c >= heap_n) break;
      if (c + 1 < heap_n && less(heap[c + 1], heap[c])) ++c;
      if (!less(heap[c], x)) break;
      heap[i] = heap[c];
      i = c;
    }
    if (heap_n > 0) heap[i] = x;
    return top;
  }
  SPD_HD void wake(double t, int32_t payload) {  // schedule_wake (backend.py:215-217)
    push(t > now ? t : now, 1, payload);
  }

  // ---- Eq. 2 weights (configurator.py:553-561) ---------------------------------------------
  SPD_HDN void weights(int q, int k, int op, int e, int d) {
    const int base = im.w_off[k];
    const int cap = im.w_off[k + 1] - base;
    int32_t* key = wkey + q * im.w_off[im.n_kinds] + base;
    int32_t* cnt = wcnt + q * im.w_off[im.n_kinds] + base;
    const int32_t kk = (op << 16) | e;
    int n = wn[q][k], i = 0;
    #pragma unroll 1
    while (i < n && key[i] != kk) ++i;
    if (i < n) {
      const int32_t nv = cnt[i] + d;
      if (nv) {
        cnt[i] = nv;
      } else {  // m.pop(key): later keys keep their order
        #pragma unroll 1
        for (int j = i + 1; j < n; ++j) {
          key[j - 1] = key[j];
          cnt[j - 1] = cnt[j];
        }
        wn[q][k] = n - 1;
      }
    } else if (d) {
      if (n >= cap) {
        error(kErrWeightCap);
      } else {
        key[n] = kk;
        cnt[n] = d;
        wn[q][k] = n + 1;
      }
    }
    ++kver[k];
    ++version;  // self.bump()
  }

  // ---- slack_by_kind (configurator.py:493-543) --------------------------------------------
  SPD_HDN const double* slacks(int op) {
    double* out = scval + op * im.n_kinds;
    if (scver[op] == version) return out;
    const int K = im.n_kinds;
    // _path_ratios (configurator.py:493-509): own / (left-to-right suffix total) per suffix
    // containing op, recomputed when a reference latency changed.  min_r fl(r * budget) is
    // fl(r_min * budget) for budget >= 0 and fl(r_max * budget) below (rounding is monotone), so
    // only the two extremes are kept; NaN or non-positive ratios keep the literal loop.
    if (rver[op] != ref_version) {
      const double own = ref_lat(op);
      double lo = 0.0, hi = 0.0;
      bool plain = true;
      int nr = 0;
      #pragma unroll 1
      for (int p = im.suf_off[op]; p < im.suf_off[op + 1]; ++nr) {
        const int len = E.suf[p++];
        double tot = 0.0;
        #pragma unroll 1
        for (int j = 0; j < len; ++j) tot = tot + ref_lat(E.suf[p + j]);
        p += len;
        const double r = own / tot;
        if (!(r > 0.0) || r == INFINITY) plain = false;
        if (nr == 0 || r < lo) lo = r;
        if (nr == 0 || r > hi) hi = r;
      }
      rmin[op] = lo;
      rmax[op] = plain ? hi : NAN;
      rver[op] = ref_version;
    }
    const int wtot = im.w_off[K];
    #pragma unroll 1
    for (int k = 0; k < K; ++k) {
      if (qver[k] != kver[k]) {  // queueing_by_kind (configurator.py:511-524)
        double tot = 0.0;
        #pragma unroll 1
        for (int q = 0; q < 2; ++q) {
          const int32_t* key = wkey + q * wtot + im.w_off[k];
          const int32_t* cnt = wcnt + q * wtot + im.w_off[k];
          #pragma unroll 1
          for (int i = 0; i < wn[q][k]; ++i) {
            const int o = key[i] >> 16, e = key[i] & 0xffff;
            const int g = im.entry_off[o] + e;
            tot = tot + (double)cnt[i] * (lat(g) * E.res[g]);
          }
        }
        qv[k] = tot / im.pool_res[k];
        qver[k] = kver[k];
      }
      const double budget = (target - now) - qv[k];
      if (rmax[op] == rmax[op]) {
        out[k] = (budget >= 0.0 ? rmin[op] : rmax[op]) * budget;
      } else {  // literal min over the ratios in suffix order (configurator.py:536-541)
        const double own = ref_lat(op);
        double sl = 0.0;
        int j = 0;
        #pragma unroll 1
        for (int p = im.suf_off[op]; p < im.suf_off[op + 1]; ++j) {
          const int len = E.suf[p++];
          double tot = 0.0;
          #pragma unroll 1
          for (int i = 0; i < len; ++i) tot = tot + ref_lat(E.suf[p + i]);
          p += len;
          const double v = (own / tot) * budget;
          if (j == 0 || v < sl) sl = v;
        }
        out[k] = sl;
      }
    }
    scver[op] = version;
    return out;
  }
  SPD_HD double ref_lat(int op) const {  // _ref_latency (configurator.py:409, 463-468)
    const int ri = im.ref_index[op];
    return ri >= 0 ? lat(im.entry_off[op] + ri) : im.ref_lat0[op];
  }

  // ---- OpTable.select / affinity (configurator.py:219-318) ---------------------------------
  SPD_HD void score_of(int g, const double* sl, double& score, double& c) {
    c = cost(g);
    score = lat(g) < sl[E.kind[g]] ? c + 0.0 : costpen(g);
  }
  SPD_HD bool key_less(double s1, double c1, int g1, double s2, double c2, int g2) const {
    if (s1 != s2) return s1 < s2;
    if (c1 != c2) return c1 < c2;
    if (E.res[g1] != E.res[g2]) return E.res[g1] < E.res[g2];
    return E.rank[g1] < E.rank[g2];
  }
  // warp-per-run mode (nl = 32): every lane runs the same serial engine (identical state,
  // identical stores), only the entry scans are split across the lanes and reduced
  SPD_HD void reduce_best(int& best, double& bs, double& bc) const {
#ifdef __CUDA_ARCH__
    if (nl > 1) {
      for (int o = nl >> 1; o > 0; o >>= 1) {
        const int ob = __shfl_xor_sync(lmask, best, o);
        const double os = __shfl_xor_sync(lmask, bs, o);
        const double oc = __shfl_xor_sync(lmask, bc, o);
        if (ob >= 0 && (best < 0 || key_less(os, oc, ob, bs, bc, best))) {
          best = ob;
          bs = os;
          bc = oc;
        }
      }
    }
#endif
  }
  SPD_HD bool any_lane(bool v) const {
#ifdef __CUDA_ARCH__
    if (nl > 1) return __any_sync(lmask, v);
#endif
    return v;
  }
  SPD_HD double min_lanes(double v) const {
#ifdef __CUDA_ARCH__
    if (nl > 1)
      for (int o = nl >> 1; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(lmask, v, o);
        v = w < v ? w : v;
      }
#endif
    return v;
  }
  SPD_HDN Sel select(int op, const double* sl, int avail, bool allow_delay, int supply,
                     uint32_t excl, int min_batch) {
    Sel r{0, -1, 0, 0.0, 0.0, 0.0};
    const int b0 = im.entry_off[op], b1 = im.entry_off[op + 1];
    int best = -1, best2 = -1;
    double bs = 0, bc = 0, bs2 = 0, bc2 = 0;
    bool bad = false;
    #pragma unroll 1
    for (int g = b0 + lane; g < b1; g += nl) {
      if ((excl >> E.kind[g]) & 1u) continue;
      if (min_batch > 1 && E.bint[g] < min_batch) continue;
      double s, c;
      score_of(g, sl, s, c);
      if (!(s == s) || s == INFINITY) {
        bad = true;
        continue;
      }
      if (best < 0 || key_less(s, c, g, bs, bc, best)) {
        best = g;
        bs = s;
        bc = c;
      }
      if (E.bint[g] <= avail && (best2 < 0 || key_less(s, c, g, bs2, bc2, best2))) {
        best2 = g;
        bs2 = s;
        bc2 = c;
      }
    }
    if (any_lane(bad)) {
      error(kErrNonFinite);
      return r;
    }
    reduce_best(best, bs, bc);
    reduce_best(best2, bs2, bc2);
    if (best < 0) return r;  // no entry survives the mask: None (configurator.py:266-267)
    const int B = E.bint[best];
    if (allow_delay && B > avail && supply >= B - avail) {
      const double wait = sl[E.kind[best]] - lat(best);
      if (wait > 0.0) {
        r.code = 2;
        r.e = best - b0;
        r.fill = avail;
        r.obj = bs;
        r.slack = sl[E.kind[best]];
        r.wait = wait;
        return r;
      }
    }
    if (B > avail && best2 >= 0) {
      best = best2;
      bs = bs2;
    }
    r.code = 1;
    r.e = best - b0;
    r.fill = E.bint[best] < avail ? E.bint[best] : avail;
    r.obj = bs;
    r.slack = sl[E.kind[best]];
    return r;
  }
  // returns false for None; `out` = min score off the kind / min score on it (inf if only on it)
  SPD_HDN bool affinity(int op, int kind, const double* sl, double& out) {
    const int b0 = im.entry_off[op], b1 = im.entry_off[op + 1];
    double mon = INFINITY, moff = INFINITY;
    bool any_on = false, any_off = false, bad = false;
    #pragma unroll 1
    for (int g = b0 + lane; g < b1; g += nl) {
      double s, c;
      score_of(g, sl, s, c);
      if (!(s == s)) bad = true;
      if (E.kind[g] == kind) {
        any_on = true;
        if (s < mon) mon = s;
      } else {
        any_off = true;
        if (s < moff) moff = s;
      }
    }
    if (any_lane(bad)) error(kErrNonFinite);
    any_on = any_lane(any_on);
    any_off = any_lane(any_off);
    mon = min_lanes(mon);
    moff = min_lanes(moff);
    if (!any_on) return false;
    out = any_off ? moff / mon : INFINITY;
    return true;
  }


  // ---- invocations and item lists (manager.py:303-329) --------------------------------------
  SPD_HDN int new_inv(int op, int unit) {
    int id;
    if (n_free_slot > 0) {
      id = free_slot[--n_free_slot];
    } else if (n_slot < im.inv_cap) {
      id = ++n_slot;  // slots 1..inv_cap (a wake payload > 0 is a slot)
    } else {
      error(kErrInvCap);
      return -1;
    }
    if (++live_slots > peak_slots) peak_slots = live_slots;
    Inv& v = inv[id];
    v.iid = ++next_id;
    v.spec_slack = v.spec_obj = v.com_slack = v.actual = v.threshold = 0.0;
    v.started_at = -1.0;
    v.unit = unit < 0 ? id : unit;
    v.spec_e = v.com_e = -1;
    v.instance = -1;
    v.op = (uint8_t)op;
    v.state = kPending;
    v.bits = 0;
    next[id] = -1;
    if (unit < 0) {
      live[id] = 1;
      lists[id] = List{0, -1, -1};
    } else {
      live[unit] += 1;
    }
    return id;
  }
  SPD_HDN void take_items(int unit, int op, int n) {  // buffer.popleft() x n onto the list
    if (n <= 0) return;
    int s;
    if (n_free_seg > 0) {
      s = free_seg[--n_free_seg];
    } else if (n_seg < im.seg_cap) {
      s = n_seg++;
    } else {
      error(kErrSegCap);
      return;
    }
    segs[s] = Seg{OP(op, kOpiBufHead), n, -1};
    OP(op, kOpiBufHead) += n;
    List& L = lists[unit];
    if (L.last >= 0)
      segs[L.last].next = s;
    else
      L.first = s;
    L.last = s;
    L.count += n;
  }
  SPD_HD int buf_len(int op) { return OP(op, kOpiBufTail) - OP(op, kOpiBufHead); }
  SPD_HD int fill_of(int id) { return lists[inv[id].unit].count; }
  // A finished invocation's slot is recycled once its straggler wake has popped; a unit's first
  // slot (items, resolved flag, live count) only when the unit is resolved and none of its
  // duplicates / retries is still live.  Called when one of those conditions may have changed.
  SPD_HDN void maybe_free(int id) {
    const Inv& v = inv[id];
    if (v.state < kCompleted || (v.bits & kBitWakePending)) return;
    if (v.unit == id) {
      if (!(v.bits & kBitResolved) || live[id] != 0) return;
      #pragma unroll 1
      for (int sg = lists[id].first; sg >= 0; sg = segs[sg].next) free_seg[n_free_seg++] = sg;
    }
    inv[id].state = kPending;  // poisoned: never finished again until reused
    free_slot[n_free_slot++] = id;
    --live_slots;
  }

  // ---- backend pools (backend.py:155-201, manager.py:331-341) -------------------------------
  SPD_HDN void submit(int id) {
    const int g = im.entry_off[inv[id].op] + inv[id].com_e;
    const int k = E.kind[g];
    next[id] = -1;
    if (cq_tail[k] >= 0)
      next[cq_tail[k]] = id;
    else
      cq_head[k] = id;
    cq_tail[k] = id;
    ++cq_len[k];
    try_start(k);
  }
  SPD_HDN void try_start(int k) {
    #pragma unroll 1
    while (cq_head[k] >= 0 && status == kOk) {
      const int id = cq_head[k];
      const int g = im.entry_off[inv[id].op] + inv[id].com_e;
      const int need = (int)E.res[g];
      int inst = -1;
      #pragma unroll 1
      for (int i = im.inst_off[k]; i < im.inst_off[k + 1]; ++i)
        if (freeres[i] >= need) {
          inst = i;
          break;
        }
      if (inst < 0) return;  // the FIFO head blocks; no backfill (backend.py:171-173)
      cq_head[k] = next[id];
      if (cq_head[k] < 0) cq_tail[k] = -1;
      --cq_len[k];
      start(k, id, inst, need, g);
    }
  }
  SPD_HDN void start(int k, int id, int inst, int need, int g) {  // backend.py:179-201
    freeres[inst] -= need;
    Inv& v = inv[id];
    if (!(E.base[g] == E.base[g])) {  // no ground truth for (op, kind): KeyError (scenario.py:97-101)
      error(kErrNoTruth);
      return;
    }
    double L = E.base[g] + E.per_item[g] * (double)fill_of(id);  // backend.py:51
    if (im.draws) {
      if (n_starts >= im.draw_cap) {
        error(kErrDrawCap);
        return;
      }
      if (im.draws & kDrawNoise) L = L * draw_factor[n_starts];
      const uint8_t b = (im.draws & (kDrawStraggle | kDrawFail)) ? draw_bits[n_starts] : 0;
      if ((im.draws & kDrawStraggle) && (b & 1)) L = L * im.straggle_factor;
      if ((im.draws & kDrawFail) && (b & 2)) v.bits |= kBitWillFail;
    }
    ++n_starts;
    v.actual = L;
    v.instance = inst;
    ++running;
    push((now + im.dispatch) + L, 0, id);
    ev_row(now, id, 0, k, inst);
    // on_start -> _handle_start (manager.py:331-341)
    v.state = kRunning;
    v.started_at = now;
    const int c = E.cfg[g];
    cfg_used[c >> 5] |= 1u << (c & 31);
    weights(1, k, v.op, v.com_e, -1);  // notify_started (configurator.py:758-763)
    const double thr = im.timeout_factor * lat(g);
    v.threshold = thr;
    const double at = now + thr;
    v.bits |= kBitWakePending;
    wake(at + 1e-9 * (1.0 + fabs(at)), id);
  }

  // ---- speculation (configurator.py:563-637) ------------------------------------------------
  SPD_HDN void ev_row(double t, int id, int what, int k, int inst) {
    if (evlog && ev_len < im.ev_cap)
      evlog[ev_len] = EvRec{t, inv[id].iid, what | (k << 2) | ((inst - im.inst_off[k]) << 8)};
    ++ev_len;
  }
  SPD_HDN void log_row(int id, int op, int e, bool commit, double slack, double obj) {
    if (log) {
      if (log_len < im.log_cap)
        log[log_len] = LogRec{now, slack, obj, inv[id].iid, op | (e << 8) | (commit ? (1 << 30) : 0)};
    }
    ++log_len;
  }
  SPD_HDN void enqueue_spec(int id, int e, double slack, double obj) {  // 639-655
    Inv& v = inv[id];
    const int op = v.op;
    v.state = kSpeculated;
    v.spec_e = (int16_t)e;
    v.spec_slack = slack;
    v.spec_obj = obj;
    next[id] = -1;
    if (OP(op, kOpiSqTail) >= 0)
      next[OP(op, kOpiSqTail)] = id;
    else
      OP(op, kOpiSqHead) = id;
    OP(op, kOpiSqTail) = id;
    OP(op, kOpiSqLen) += 1;
    weights(0, E.kind[im.entry_off[op] + e], op, e, +1);
    log_row(id, op, e, false, slack, obj);
  }
  SPD_HDN int speculate_buffer(int op) {
    int formed = 0;
    const int ri = im.ref_index[op];
    #pragma unroll 1
    while (buf_len(op) > 0 && status == kOk) {
      const bool forced = !(im.abl & kAblDfp) && ri >= 0 && OP(op, kOpiCompletedRef) < im.dfp_count;
      const double* sl = slacks(op);
      int e, fill;
      double slack, obj;
      if (forced) {
        e = ri;
        fill = 1;
        obj = NAN;
        slack = sl[E.kind[im.entry_off[op] + ri]];
      } else {
        const bool hold = OP(op, kOpiHold) != 0;
        bool allow = !(im.abl & kAblSdb);
        if (hold && now >= holddl[op]) allow = false;
        const Sel d = select(op, sl, buf_len(op), allow, supply(op), 0u, 1);
        if (status != kOk) return formed;
        if (d.code == 2) {
          if (!hold) {
            const double dl = now + d.wait;
            OP(op, kOpiHold) = 1;
            holddl[op] = dl;
            if (dl != INFINITY) wake(dl, -(op + 1));
          }
          ++n_spec;
          break;
        }
        e = d.e;
        fill = d.fill;
        slack = d.slack;
        obj = d.obj;
      }
      OP(op, kOpiHold) = 0;
      const int id = new_inv(op, -1);
      if (id < 0) return formed;
      if (forced) inv[id].bits |= kBitForced;
      take_items(id, op, fill);
      enqueue_spec(id, e, slack, obj);
      ++n_spec;
      ++formed;
    }
    return formed;
  }
  SPD_HDN void speculate_fixed(int id) {
    const int op = inv[id].op;
    const int fill = fill_of(id);
    const Sel d = select(op, slacks(op), fill, false, 0, 0u, fill);
    if (status != kOk) return;
    if (d.code == 0) {
      error(kErrNoConfig);  // RuntimeError (configurator.py:633-636)
      return;
    }
    enqueue_spec(id, d.e, d.slack, d.obj);
    ++n_spec;
  }
  SPD_HDN int supply(int op) {  // manager.py:301-305
    int s = 0;
    const uint64_t m = im.anc_mask[op];
    #pragma unroll 1
    for (int a = 0; a < im.n_ops; ++a)
      if ((m >> a) & 1u) s += OP(a, kOpiUnspawned);
    return s;
  }

  // ---- commits (configurator.py:641-756) ----------------------------------------------------
  struct Key {
    int cls;
    double a, b;
    int iid;
  };
  SPD_HD bool key_lt(const Key& x, const Key& y) const {
    if (x.cls != y.cls) return x.cls < y.cls;
    if (x.a != y.a) return x.a < y.a;
    if (x.b != y.b) return x.b < y.b;
    return x.iid < y.iid;
  }
  SPD_HDN int pump_commits() {
    int committed = 0;
    const bool fifo = im.abl & kAblPbc;
    const bool eslc = im.abl & kAblEslc;
    #pragma unroll 1
    while (status == kOk) {
      uint32_t full = 0;
      #pragma unroll 1
      for (int k = 0; k < im.n_kinds; ++k)
        if (cq_len[k] >= im.cap[k]) full |= 1u << k;
      int bop = -1, be = -1, bfill = 0;
      double bslack = 0.0, bobj = 0.0;
      Key bkey{0, 0.0, 0.0, 0};
      #pragma unroll 1
      for (int op = 0; op < im.n_ops; ++op) {
        const int head = OP(op, kOpiSqHead);
        if (head < 0) continue;
        const Inv& h = inv[head];
        const int b0 = im.entry_off[op];
        const int hf = fill_of(head);
        int e, fill;
        double slack, obj;
        if (h.bits & kBitForced) {
          const int ri = im.ref_index[op];
          const int k = E.kind[b0 + ri];
          if ((full >> k) & 1u) continue;
          e = ri;
          fill = hf;
          slack = slacks(op)[k];
          obj = NAN;
        } else if (eslc) {
          if ((full >> E.kind[b0 + h.spec_e]) & 1u) continue;
          e = h.spec_e;
          fill = hf;
          slack = h.spec_slack;
          obj = h.spec_obj;
        } else {
          const Sel d = select(op, slacks(op), hf + buf_len(op), false, 0, full, hf);
          if (status != kOk) return committed;
          if (d.code == 0) continue;
          e = d.e;
          fill = d.fill > hf ? d.fill : hf;
          slack = d.slack;
          obj = d.obj;
        }
        Key key;
        if (fifo) {
          key = Key{0, 0.0, 0.0, h.iid};
        } else if (h.bits & kBitForced) {
          key = Key{0, -(double)im.depth[op], 0.0, h.iid};
        } else {
          double aff = 0.0;
          if (!affinity(op, E.kind[b0 + e], slacks(op), aff)) aff = 0.0;
          key = Key{1, -aff, slack, h.iid};
        }
        if (bop < 0 || key_lt(key, bkey)) {
          bkey = key;
          bop = op;
          be = e;
          bfill = fill;
          bslack = slack;
          bobj = obj;
        }
      }
      if (bop < 0) return committed;
      const int id = OP(bop, kOpiSqHead);
      Inv& v = inv[id];
      const int b0 = im.entry_off[bop];
      OP(bop, kOpiSqHead) = next[id];
      if (next[id] < 0) OP(bop, kOpiSqTail) = -1;
      OP(bop, kOpiSqLen) -= 1;
      weights(0, E.kind[b0 + v.spec_e], bop, v.spec_e, -1);
      const int hf = fill_of(id);
      if (bfill > hf) {  // _topup (manager.py:346-352)
        const int bl = buf_len(bop);
        const int n = bfill - hf < bl ? bfill - hf : bl;
        take_items(v.unit, bop, n);
        if (buf_len(bop) == 0) OP(bop, kOpiHold) = 0;
      }
      v.state = kCommitted;
      v.com_e = (int16_t)be;
      v.com_slack = bslack;
      weights(1, E.kind[b0 + be], bop, be, +1);
      log_row(id, bop, be, true, bslack, bobj);
      ++n_commit;
      ++committed;
      submit(id);
    }
    return committed;
  }

  // ---- run engine (manager.py:356-575) -------------------------------------------------------
  SPD_HDN void pump() {
    #pragma unroll 1
    while (status == kOk) {
      int formed = 0;
      #pragma unroll 1
      for (int j = 0; j < im.n_ops; ++j) {
        const int op = im.deep_first[j];
        if (buf_len(op) > 0) {
          formed += speculate_buffer(op);
          if (buf_len(op) == 0) OP(op, kOpiHold) = 0;
        }
      }
      const int committed = pump_commits();
      if (formed == 0 && committed == 0) return;
    }
  }
  SPD_HDN void append_items(int dst, int frame, int n) {
    int& tail = OP(dst, kOpiBufTail);
    const int cap = im.buf_off[dst + 1] - im.buf_off[dst];
    if (tail + n > cap) {
      error(kErrBufCap);
      return;
    }
    int32_t* b = items + im.buf_off[dst];
    #pragma unroll 1
    for (int i = 0; i < n; ++i) b[tail + i] = frame;
    tail += n;
    OP(dst, kOpiUnspawned) += n;
  }
  SPD_HDN void spawn(int id) {  // manager.py:392-434
    const int op = inv[id].op;
    const List L = lists[inv[id].unit];
    if (im.succ_off[op] == im.succ_off[op + 1]) {
      terminal += L.count;
      OP(op, kOpiUnspawned) -= L.count;
      return;
    }
    const int32_t* src = items + im.buf_off[op];
    #pragma unroll 1
    for (int s = L.first; s >= 0; s = segs[s].next) {
      #pragma unroll 1
      for (int j = 0; j < segs[s].n; ++j) {
        const int fr = src[segs[s].pos + j];
        const int32_t* at = attrs + (int64_t)fr * im.n_attrs;
        #pragma unroll 1
        for (int q = im.succ_off[op]; q < im.succ_off[op + 1]; ++q) {
          const int dst = im.succ[q];
          if (im.pred_attr[q] >= 0 && !pred_eval(im.pred_cmp[q], at[im.pred_attr[q]], im.pred_val[q]))
            continue;
          const int n = im.fanout_attr[dst] >= 0 ? at[im.fanout_attr[dst]] : 1;
          if (n <= 0) continue;
          if (im.indeg[dst] > 1) {  // _deliver_join (manager.py:416-434)
            int32_t* st = staging + ((int64_t)fr * im.staging_per_frame + im.join_base[dst]);
            st[im.join_pos[q]] += n;
            int m = st[0];
            #pragma unroll 1
            for (int p = 1; p < im.indeg[dst]; ++p) m = st[p] < m ? st[p] : m;
            if (m > 0) {
              #pragma unroll 1
              for (int p = 0; p < im.indeg[dst]; ++p) st[p] -= m;
              append_items(dst, fr, m);
            }
          } else {
            append_items(dst, fr, n);
          }
        }
      }
    }
    OP(op, kOpiUnspawned) -= L.count;
  }
  SPD_HDN void feedback(int id, double obs) {  // manager.py:436-457
    Inv& v = inv[id];
    const int op = v.op, e = v.com_e, g = im.entry_off[op] + e;
    const int ri = im.ref_index[op];
    if (e == ri) OP(op, kOpiCompletedRef) += 1;
    observed[g] = 1;
    if (im.abl & kAblFb) return;
    set_lat(g, im.beta * obs + (1.0 - im.beta) * lat(g));
    ++version;  // bump_profiles (configurator.py:463-468); _ref_latency reads lat[ref] live
    if (e == ri) ++ref_version;
    if (e == ri && OP(op, kOpiCompletedRef) == im.dfp_count && !(im.abl & kAblDfp)) {
      const double init = E.lat_init[g];  // recalibrate_unobserved (configurator.py:470-491)
      if (init > 0.0) {
        const double ratio = lat(g) / init;
        #pragma unroll 1
        for (int j = im.entry_off[op]; j < im.entry_off[op + 1]; ++j)
          if (j != g && !observed[j]) set_lat(j, E.lat_init[j] * ratio);
        ++version;
      }
    }
  }
  SPD_HDN void finish(int id, double t) {  // advance + _on_complete / _on_fail (manager.py:459-497)
    Inv& v = inv[id];
    const int g = im.entry_off[v.op] + v.com_e;
    const int k = E.kind[g];
    freeres[v.instance] += (int)E.res[g];
    --running;
    ev_row(t, id, (v.bits & kBitWillFail) ? 2 : 1, k, v.instance);
    try_start(k);  // FIFO successors start before the engine sees the event (backend.py:231)
    const double cost = (E.res[g] * v.actual) * im.price[k];  // invocation_cost (backend.py:61-63)
    total_cost = total_cost + cost;
    const int u = v.unit;
    live[u] -= 1;
    if (v.bits & kBitWillFail) {
      ++failures;
      v.state = kFailed;
      if (!(inv[u].bits & kBitResolved) && live[u] == 0) {
        const int r = new_inv(v.op, u);
        if (r >= 0) speculate_fixed(r);
      }
    } else {
      feedback(id, v.actual);
      if (inv[u].bits & kBitResolved) {
        v.state = kDuplicated;
      } else {
        inv[u].bits |= kBitResolved;
        v.state = kCompleted;
        if (v.actual <= v.com_slack) ++met;
        ++completed;
        last_accept = t;
        spawn(id);
      }
    }
    maybe_free(id);
    if (u != id) maybe_free(u);
  }
  SPD_HDN void straggler(int id) {  // manager.py:499-511
    Inv& v = inv[id];
    if (v.state != kRunning || (v.bits & kBitDupSpawned)) return;
    if (inv[v.unit].bits & kBitResolved) return;
    if (now - v.started_at > v.threshold) {
      v.bits |= kBitDupSpawned;
      ++dups;
      const int r = new_inv(v.op, v.unit);
      if (r >= 0) speculate_fixed(r);
    }
  }
  SPD_HDN bool work_remains() {  // manager.py:526-533
    #pragma unroll 1
    for (int o = 0; o < im.n_ops; ++o)
      if (buf_len(o) > 0 || OP(o, kOpiSqLen) > 0) return true;
    #pragma unroll 1
    for (int k = 0; k < im.n_kinds; ++k)
      if (cq_len[k] > 0) return true;
    return running > 0;
  }
  SPD_HDN void run() {  // start_run + run_to_completion (manager.py:535-575)
    init();
    #pragma unroll 1
    for (int j = 0; j < im.n_inputs; ++j) {
      const int v = im.inputs[j];
      #pragma unroll 1
      for (int f = 0; f < n_frames; ++f) items[im.buf_off[v] + f] = f;
      OP(v, kOpiBufTail) = n_frames;
      OP(v, kOpiUnspawned) += n_frames;
    }
    pump();
    bool flushed = false;
    #pragma unroll 1
    while (status == kOk) {
      if (heap_n == 0) {
        if (!work_remains()) break;
        bool any_hold = false;
        #pragma unroll 1
        for (int o = 0; o < im.n_ops; ++o) any_hold |= OP(o, kOpiHold) != 0;
        if (!flushed && any_hold) {
          flushed = true;
          #pragma unroll 1
          for (int o = 0; o < im.n_ops; ++o)
            if (OP(o, kOpiHold)) holddl[o] = now;
          pump();
          continue;
        }
        error(kErrLivelock);  // RuntimeError (manager.py:563)
        break;
      }
      if (++events > im.event_cap) {
        error(kErrEventCap);
        break;
      }
      flushed = false;
#ifdef __CUDA_ARCH__
      if (nl > 1) __syncwarp(lmask);  // lanes per run: their redundant stores stay in lockstep
#endif
      const HeapEnt ev = pop();
      now = ev.t;
      if (ev.key >> 31) {
        if (ev.payload > 0) {
          inv[ev.payload].bits &= (uint8_t)~kBitWakePending;
          straggler(ev.payload);
          maybe_free(ev.payload);
        }
      } else {
        finish(ev.payload, ev.t);
      }
      pump();
    }
  }

  SPD_HDN void write_out(Out& o) {
    o.latency = last_accept;
    o.cost = total_cost;
    o.now = now;
    o.peak_slots = peak_slots;
    o.peak_heap = peak_heap;
    o.status = status;
    o.met = met;
    o.completed = completed;
    o.failures = failures;
    o.dups = dups;
    o.invocations = next_id;
    o.terminal = terminal;
    o.n_spec = n_spec;
    o.n_commit = n_commit;
    int used = 0;
    #pragma unroll 1
    for (int i = 0; i < (im.n_cfg + 31) / 32; ++i) {
      uint32_t w = cfg_used[i];
      #pragma unroll 1
      while (w) {
        used += w & 1u;
        w >>= 1;
      }
    }
    o.configs_used = used;
    o.log_len = log_len;
    o.ev_len = ev_len;
    o.events = (int32_t)events;
  }
};

}  // namespace spdes
