// sp_spec.cuh — Configurator.speculate_from_buffer on the device (
// included by sp_select.cu after sp_k2b.cuh).
//
// One thread runs one call's sequential loop (configurator.py:563-620):
//   slack  — the entry value the caller passes (slack_by_kind is cached by weight version only,
//            configurator.py:526-529), then after every formed invocation Eq. 2 recomputed from
//            the weights (queueing_by_kind, 511-524: SQ then CQ weights in dict order,
//            total += count * (lat * res), / pool) and budget = (target - now) - Q,
//            slack = (budget >= 0 ? rmin : rmax) * budget (526-543);
//   decide — forced warm-up: the reference entry, fill 1, objective NaN (571-589); otherwise
//            OpTable.select(slack, alpha, buffered, allow_delay, supply) on the op's staircase
//            plan (K2b's decide_plan), allow_delay cleared on the first iteration when the
//            batching hold has expired (597-599); a delay decision ends the loop (606-612);
//   update — buffered -= fill; _weights_add(SQ, kind, op, entry, +1) (553-561): an existing key
//            is incremented in place, a new key appended after the kind's list.
// The input weight lists are read-only; the call's increments of input SQ keys live in a
// global array indexed like the weights (winc, zeroed per launch) and its new keys in a global
// list indexed like its output slots (a call forms at most as many invocations — and so new
// keys — as it has slots), so there is no per-call key limit and no per-thread key array.  The
// Eq. 2 order is: input SQ entries (count + increment), then the call's new keys of the kind in
// append order, then the CQ entries.

constexpr int kMaxSpecTables = 64;

struct SpecTabs {
  const double* lat[kMaxSpecTables];
  const double* res[kMaxSpecTables];
  const int32_t* kind[kMaxSpecTables];
  const uint8_t* plan[kMaxSpecTables];
  int32_t ref_index[kMaxSpecTables];
  double pool[kMaxKinds];
};

struct SpecIO {
  const int32_t* op;
  const int32_t* n_buf;
  const int32_t* supply;
  const double* now;
  const double* target;
  const double* rmin;
  const double* rmax;
  const double* slack0;  // R x K
  const uint32_t* flags;
  const int32_t* w_ptr;  // R * 2K + 1: (r, queue, kind) lists
  const int32_t* w_tab;
  const int32_t* w_eidx;
  const int32_t* w_count;
  const int32_t* out_off;  // R + 1
  int32_t* out_idx;
  int32_t* out_fill;
  double* out_slack;
  double* out_obj;
  int32_t* out_n;
  int32_t* out_delay_idx;
  double* out_delay_wait;
  int32_t* winc;     // per input weight: this call's increments (zeroed)
  int32_t* nkey_id;  // per output slot: a new key (tab << 20 | kind << 16 | eidx)
  int32_t* nkey_cnt;
  int R;
  int K;
};

__device__ __forceinline__ int32_t key_id(int tab, int kind, int eidx) {
  return (tab << 20) | (kind << 16) | eidx;
}

template <int KT>
__global__ void __launch_bounds__(128) k_speculate(SpecTabs tb, double alpha, SpecIO io,
                                                   SelectIO sel) {
  // Persistent threads: each thread runs calls r, r + stride, ... one loop ITERATION per pass of
  // the outer loop, taking its next call the moment the current one ends — the calls' loops
  // have different lengths, so lanes stay converged on the iteration body instead of idling
  // behind the longest call of the warp.
  const int stride = gridDim.x * blockDim.x;
  const int K = io.K;
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  int op = 0, n = 0, supply = 0, nk = 0, o0 = 0, nd = 0;
  double span = 0.0, rmin = 0.0, rmax = 0.0;
  uint32_t fl = 0;
  bool first = true, overflow = false;
  const int32_t* wp = io.w_ptr;
  View<KT> v;
  In<KT> x;
  int last_id = -1, last_w = -1, last_q = -1;  // the previous formed invocation's key
  auto start = [&](int rr) {  // load call rr's state
    op = io.op[rr];
    n = io.n_buf[rr];
    supply = io.supply[rr];
    span = __dsub_rn(io.target[rr], io.now[rr]);  // target - now
    rmin = io.rmin[rr];
    rmax = io.rmax[rr];
    fl = io.flags[rr];
    wp = io.w_ptr + (size_t)rr * 2 * K;
    make_view<KT>(v, tb.plan[op], *reinterpret_cast<const PlanHdr*>(tb.plan[op]), K);
    nk = 0;
    o0 = io.out_off[rr];
    nd = 0;
    first = true;
    overflow = false;
    last_id = last_w = last_q = -1;
    io.out_delay_idx[rr] = -1;
    io.out_delay_wait[rr] = 0.0;
  };
  if (r < io.R) start(r);
  while (r < io.R) {
    bool done = n <= 0;
    if (!done) {
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        if (k >= K) {
          x.s[k] = 0.0;
          continue;
        }
        if (first) {
          x.s[k] = io.slack0[(size_t)r * K + k];
          continue;
        }
        double total = 0.0;  // configurator.py:516-522
        for (int w = wp[k]; w < wp[k + 1]; ++w) {  // SQ, in dict order
          const int c = io.w_count[w] + io.winc[w];
          const int t = io.w_tab[w], e = io.w_eidx[w];
          total = __dadd_rn(total, __dmul_rn((double)c, __dmul_rn(tb.lat[t][e], tb.res[t][e])));
        }
        for (int q = 0; q < nk; ++q) {  // keys this call appended to the kind's SQ dict
          const int id = io.nkey_id[o0 + q];
          if (((id >> 16) & 15) != k) continue;
          const int t = id >> 20, e = id & 0xFFFF;
          total = __dadd_rn(total, __dmul_rn((double)io.nkey_cnt[o0 + q],
                                             __dmul_rn(tb.lat[t][e], tb.res[t][e])));
        }
        for (int w = wp[K + k]; w < wp[K + k + 1]; ++w) {  // CQ
          const int t = io.w_tab[w], e = io.w_eidx[w];
          total = __dadd_rn(total,
                            __dmul_rn((double)io.w_count[w], __dmul_rn(tb.lat[t][e], tb.res[t][e])));
        }
        const double budget = __dsub_rn(span, __ddiv_rn(total, tb.pool[k]));  // 535
        x.s[k] = __dmul_rn(budget >= 0.0 ? rmin : rmax, budget);             // 536-540
      }
      int idx = -1, fill = 0, kd = 0;
      double s_k = 0.0, obj = 0.0;
      if (fl & SP_SPEC_FORCED) {  // configurator.py:571-589
        idx = tb.ref_index[op];
        fill = 1;
        kd = tb.kind[op][idx];
        s_k = pick_kind<KT>(x.s, kd);
        obj = NAN;
      } else {
        const bool allow = (fl & SP_SPEC_SDB) && !(first && (fl & SP_SPEC_HOLD_EXPIRED));
        x.av = n;
        x.sup = supply;
        x.mb = 1;
        x.fl = allow ? SP_FLAG_ALLOW_DELAY : 0u;
        x.t = op;
        decide_plan<KT, false>(v, sel, r, x);
        const int code = sel.out_code[r];
        idx = sel.out_idx[r];
        if ((code & 3) == SP_DEC_DELAY) {  // configurator.py:606-612
          io.out_delay_idx[r] = idx;
          io.out_delay_wait[r] = sel.out_wait[r];
          done = true;
        } else if ((code & 3) != SP_DEC_ASSIGN) {  // cannot happen without exclusions (605)
          overflow = true;
          done = true;
        } else {
          fill = sel.out_fill[r];
          s_k = sel.out_slack[r];
          obj = sel.out_obj[r];
          kd = tb.kind[op][idx];
        }
      }
      if (!done) {
        first = false;
        n -= fill;
        // _weights_add(self._sq_weight, kind, op, idx, +1): an input key (increment), else a
        // key this call appended (count), else a new key at the end of the kind's dict
        const int id = key_id(op, kd, idx);
        if (id == last_id) {
          if (last_w >= 0) io.winc[last_w] += 1; else io.nkey_cnt[o0 + last_q] += 1;
        } else {
          int w_hit = -1;
          for (int w = wp[kd]; w < wp[kd + 1]; ++w)
            if (io.w_tab[w] == op && io.w_eidx[w] == idx) w_hit = w;
          int q_hit = -1;
          if (w_hit < 0)
            for (int q = 0; q < nk; ++q)
              if (io.nkey_id[o0 + q] == id) q_hit = q;
          if (w_hit >= 0) {
            io.winc[w_hit] += 1;
          } else if (q_hit >= 0) {
            io.nkey_cnt[o0 + q_hit] += 1;
          } else {
            q_hit = nk++;
            io.nkey_id[o0 + q_hit] = id;
            io.nkey_cnt[o0 + q_hit] = 1;
          }
          last_id = id;
          last_w = w_hit;
          last_q = q_hit;
        }
        {
          io.out_idx[o0 + nd] = idx;
          io.out_fill[o0 + nd] = fill;
          io.out_slack[o0 + nd] = s_k;
          io.out_obj[o0 + nd] = obj;
          ++nd;
          done = n <= 0;
        }
      }
    }
    if (done) {
      io.out_n[r] = overflow ? -1 : nd;
      r += stride;
      if (r < io.R) start(r);
    }
  }
}

}  // namespace

int speculate_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, double alpha, int K,
                     const double* pool, int R, const int32_t* op, const int32_t* n_buf,
                     const int32_t* supply, const double* now, const double* target,
                     const double* rmin, const double* rmax, const double* slack0,
                     const uint32_t* flags, const int32_t* w_ptr, const int32_t* w_tab,
                     const int32_t* w_eidx, const int32_t* w_count, const int32_t* out_off,
                     int32_t* out_idx, int32_t* out_fill, double* out_slack, double* out_obj,
                     int32_t* out_n, int32_t* out_delay_idx, double* out_delay_wait,
                     int n_weights, int n_slots) {
  if (n_tables > kMaxSpecTables) return fail(SP_E_UNSUPPORTED, "speculate: more than 64 tables");
  if (K > 8) return fail(SP_E_UNSUPPORTED, "speculate: more than 8 kinds");
  SpecTabs tb;
  memset(&tb, 0, sizeof(tb));
  for (int t = 0; t < n_tables; ++t) {
    if (!tables[t]->plan_ok || !tables[t]->finite_safe() || !isfinite(alpha))
      return fail(SP_E_UNSUPPORTED, "speculate: table without a plan (batch sizes, entries, "
                                    "kinds or non-finite latencies)");
    int rc;
    Plan* p = plan_get(ctx, tables[t], alpha, &rc);
    if (!p) return rc;
    tb.lat[t] = tables[t]->lat;
    tb.res[t] = tables[t]->res;
    tb.kind[t] = tables[t]->kind;
    tb.plan[t] = p->image;
    tb.ref_index[t] = tables[t]->ref_index;
  }
  for (int k = 0; k < K; ++k) tb.pool[k] = pool[k];
  // per-call decide_plan outputs (read back by the same thread)
  int rc = SP_OK;
  const size_t al = ((size_t)R * 8 + 255) & ~(size_t)255;
  uint8_t* s = static_cast<uint8_t*>(ctx_tmp(ctx, 6 * al, &rc));
  if (!s) return rc;
  SelectIO sel;
  memset(&sel, 0, sizeof(sel));
  sel.out_idx = reinterpret_cast<int32_t*>(s);
  sel.out_code = reinterpret_cast<int32_t*>(s + al);
  sel.out_fill = reinterpret_cast<int32_t*>(s + 2 * al);
  sel.out_obj = reinterpret_cast<double*>(s + 3 * al);
  sel.out_slack = reinterpret_cast<double*>(s + 4 * al);
  sel.out_wait = reinterpret_cast<double*>(s + 5 * al);
  sel.N = R;
  sel.K = K;
  SpecIO io{op, n_buf, supply, now, target, rmin, rmax, slack0, flags, w_ptr, w_tab, w_eidx,
            w_count, out_off, out_idx, out_fill, out_slack, out_obj, out_n, out_delay_idx,
            out_delay_wait, nullptr, nullptr, nullptr, R, K};
  {  // per-weight increments (zeroed) and per-slot new keys, after the select outputs
    int32_t nw = n_weights, nslots = n_slots;
    if (nw < 0 || nslots < 0) {  // device-resident arguments: read the two totals
      SP_CUDA(cudaMemcpyAsync(&nw, w_ptr + (size_t)2 * K * R, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, ctx->stream));
      SP_CUDA(cudaMemcpyAsync(&nslots, out_off + R, sizeof(int32_t), cudaMemcpyDeviceToHost,
                              ctx->stream));
      SP_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    const size_t a1 = ((size_t)std::max(nw, 1) * 4 + 255) & ~(size_t)255;
    const size_t a2 = ((size_t)std::max(nslots, 1) * 4 + 255) & ~(size_t)255;
    uint8_t* k = static_cast<uint8_t*>(ctx_tmp(ctx, 6 * al + a1 + 2 * a2, &rc));
    if (!k) return rc;
    if (k != s) {  // the scratch moved: re-point the select outputs
      s = k;
      sel.out_idx = reinterpret_cast<int32_t*>(s);
      sel.out_code = reinterpret_cast<int32_t*>(s + al);
      sel.out_fill = reinterpret_cast<int32_t*>(s + 2 * al);
      sel.out_obj = reinterpret_cast<double*>(s + 3 * al);
      sel.out_slack = reinterpret_cast<double*>(s + 4 * al);
      sel.out_wait = reinterpret_cast<double*>(s + 5 * al);
    }
    io.winc = reinterpret_cast<int32_t*>(s + 6 * al);
    io.nkey_id = reinterpret_cast<int32_t*>(s + 6 * al + a1);
    io.nkey_cnt = reinterpret_cast<int32_t*>(s + 6 * al + a1 + a2);
    SP_CUDA(cudaMemsetAsync(io.winc, 0, (size_t)std::max(nw, 1) * 4, ctx->stream));
  }
  // persistent grid: resident CTAs only (calls are taken by grid stride)
  int per_sm = 0;
  if (K <= 2)
    SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_speculate<2>, 128, 0));
  else if (K <= 4)
    SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_speculate<4>, 128, 0));
  else
    SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_speculate<8>, 128, 0));
  const int blocks = std::max(1, std::min((R + 127) / 128, ctx->num_sms * std::max(per_sm, 1)));
  if (K <= 2)
    k_speculate<2><<<blocks, 128, 0, ctx->stream>>>(tb, alpha, io, sel);
  else if (K <= 4)
    k_speculate<4><<<blocks, 128, 0, ctx->stream>>>(tb, alpha, io, sel);
  else
    k_speculate<8><<<blocks, 128, 0, ctx->stream>>>(tb, alpha, io, sel);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

namespace {
