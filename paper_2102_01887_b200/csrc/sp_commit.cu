// sp_commit.cu — batched commit step: Configurator.pump_commits rounds on the device
// (configurator.py:657-756).
//
// One round, for every operation whose speculative queue has a head:
//   _commit_candidate (657-691)
//     forced head (warm-up):  the reference entry, unless its kind's commit queue is full
//     eslc ablation:          the speculated entry, unless its kind is full
//     otherwise:              OpTable.select(slack_by_kind(op), alpha, head.fill + buffered,
//                             allow_delay=False, excluded_kinds=full, min_batch=head.fill)
//                             -> (entry, max(decision.fill, head.fill), slack, objective)
//   priority key (713-728)
//     pbc ablation:  (invocation_id,)
//     forced:        (0, -depth[op], invocation_id)
//     otherwise:     (1, -affinity(entry.kind), slack, invocation_id), affinity = Eq. 3
//                    OpTable.affinity (302-318) at the op's slack
//   winner = the minimum key (ids are unique, so the order is total).
// Device plan: k_commit_prep builds the K2 inputs of every (round, op), the K2 kernel
// (sp_select.cu, multi-table, with per-kind unmasked minima) re-selects all heads at once,
// k_commit_round forms candidates and keys and reduces each round with one warp.
#include <math.h>
#include <string.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kMaxCommitOps = 64;

struct CommitTabs {
  const int32_t* kind[kMaxCommitOps];  // global kind of every entry, per op table
  int32_t ref_index[kMaxCommitOps];
};

__global__ void k_commit_prep(int total, int n_ops, const int32_t* __restrict__ fill,
                              const int32_t* __restrict__ buffered,
                              const uint32_t* __restrict__ full_mask, int32_t* op,
                              int32_t* avail, int32_t* supply, int32_t* min_batch,
                              uint32_t* flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int r = i / n_ops;
  op[i] = i - r * n_ops;
  // configurator.py:679-686: available = head.fill + buffered, min_batch = head.fill,
  // allow_delay = False, excluded_kinds = kinds whose commit queue is saturated
  avail[i] = fill[i] + buffered[i];
  supply[i] = 0;
  min_batch[i] = fill[i];
  flags[i] = full_mask[r] << SP_FLAG_EXCL_SHIFT;
}

struct Key {
  int cls;     // 0 forced, 1 regular (pbc: 0 for all)
  double k1;   // -depth | -affinity
  double k2;   // 0 | slack
  long long id;
  int op;      // -1: no candidate
};

// Python tuple order of the reference keys; an absent candidate orders last
__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
  if (a.op < 0) return false;
  if (b.op < 0) return true;
  if (a.cls != b.cls) return a.cls < b.cls;
  if (a.k1 != b.k1) return a.k1 < b.k1;
  if (a.k2 != b.k2) return a.k2 < b.k2;
  return a.id < b.id;
}

__device__ __forceinline__ Key shfl_key(const Key& k, int src) {
  Key o;
  o.cls = __shfl_sync(0xffffffffu, k.cls, src);
  o.k1 = __shfl_sync(0xffffffffu, k.k1, src);
  o.k2 = __shfl_sync(0xffffffffu, k.k2, src);
  o.id = __shfl_sync(0xffffffffu, k.id, src);
  o.op = __shfl_sync(0xffffffffu, k.op, src);
  return o;
}

// LPR lanes per round (a power of two >= min(n_ops, 32)), 32 / LPR rounds per warp; lane l of a
// round's group handles ops l, l + LPR, ...
__global__ void k_commit_round(int R, int n_ops, int K, int lpr_log2, CommitTabs tb,
                               const double* __restrict__ slack,
                               const int32_t* __restrict__ fill,
                               const long long* __restrict__ head_id,
                               const int32_t* __restrict__ depth,
                               const uint32_t* __restrict__ hflags,
                               const int32_t* __restrict__ spec_idx,
                               const double* __restrict__ spec_slack,
                               const double* __restrict__ spec_obj,
                               const uint32_t* __restrict__ full_mask, int policy,
                               const int32_t* __restrict__ sel_idx,
                               const int32_t* __restrict__ sel_fill,
                               const double* __restrict__ sel_obj,
                               const double* __restrict__ sel_slack,
                               const double* __restrict__ kmin, int32_t* out_idx,
                               int32_t* out_fill, double* out_slack, double* out_obj,
                               double* out_aff, int32_t* out_best) {
  const int LPR = 1 << lpr_log2;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int warp = gid >> lpr_log2;  // the round this lane works on
  const int lane = gid & (LPR - 1);
  if (((gid >> 5) << 5) >= R * LPR) return;  // whole warp past the last round
  const bool live = warp < R;
  const bool fifo = policy & SP_COMMIT_FIFO;
  const bool eslc = policy & SP_COMMIT_ESLC;
  const uint32_t full = live ? full_mask[warp] : 0u;
  Key best;
  best.op = -1;
  best.cls = 0; best.k1 = 0.0; best.k2 = 0.0; best.id = 0;
  for (int j = lane; live && j < n_ops; j += LPR) {
    const int i = warp * n_ops + j;
    const uint32_t hf = hflags[i];
    int idx = -1, ft = 0;
    double sl = 0.0, ob = 0.0, aff = NAN;
    if (hf & SP_HEAD_PRESENT) {
      if (hf & SP_HEAD_FORCED) {  // configurator.py:670-675
        const int r = tb.ref_index[j];
        if (r >= 0) {
          const int kd = tb.kind[j][r];
          if (!((full >> kd) & 1u)) {
            idx = r; ft = fill[i]; sl = slack[(size_t)i * K + kd]; ob = NAN;
          }
        }
      } else if (eslc) {  // configurator.py:676-680
        const int e = spec_idx[i];
        const int kd = tb.kind[j][e];
        if (!((full >> kd) & 1u)) {
          idx = e; ft = fill[i]; sl = spec_slack[i]; ob = spec_obj[i];
        }
      } else if (sel_idx[i] >= 0) {  // configurator.py:681-691
        idx = sel_idx[i];
        ft = max(sel_fill[i], fill[i]);
        sl = sel_slack[i];
        ob = sel_obj[i];
      }
    }
    Key k;
    k.op = idx >= 0 ? j : -1;
    k.id = head_id[i];
    if (fifo) {  // configurator.py:716-717
      k.cls = 0; k.k1 = 0.0; k.k2 = 0.0;
    } else if (hf & SP_HEAD_FORCED) {  // 718-719
      k.cls = 0; k.k1 = -(double)depth[j]; k.k2 = 0.0;
    } else {  // 720-725: Eq. 3 of the candidate's kind at the op's slack
      k.cls = 1;
      if (idx >= 0) {
        const int c = tb.kind[j][idx];
        double other = INFINITY;
        for (int q = 0; q < K; ++q) {
          const double v = kmin[(size_t)i * K + q];
          if (q != c && v < other) other = v;
        }
        aff = __ddiv_rn(other, kmin[(size_t)i * K + c]);  // score[~on].min() / score[on].min()
      }
      k.k1 = idx >= 0 ? -aff : 0.0;
      k.k2 = sl;
    }
    out_idx[i] = idx;
    out_fill[i] = ft;
    out_slack[i] = sl;
    out_obj[i] = ob;
    out_aff[i] = aff;
    if (key_less(k, best)) best = k;
  }
  // reduction inside each LPR-lane group (xor partners stay inside the group)
  const int wl = threadIdx.x & 31;
  for (int off = LPR >> 1; off > 0; off >>= 1) {
    const Key o = shfl_key(best, wl ^ off);
    if (key_less(o, best)) best = o;
  }
  if (live && lane == 0) out_best[warp] = best.op;
}

}  // namespace

int commit_launch(sp_ctx* ctx, int R, int n_ops, sp_table* const* tables, double alpha,
                  const double* slack, const int32_t* fill, const int32_t* buffered,
                  const long long* head_id, const int32_t* depth, const uint32_t* hflags,
                  const int32_t* spec_idx, const double* spec_slack, const double* spec_obj,
                  const uint32_t* full_mask, int policy, void* scratch, int32_t* out_idx,
                  int32_t* out_fill, double* out_slack, double* out_obj, double* out_aff,
                  int32_t* out_best) {
  const int K = tables[0]->K;
  const int N = R * n_ops;
  CommitTabs tb;
  memset(&tb, 0, sizeof(tb));
  for (int j = 0; j < n_ops; ++j) {
    tb.kind[j] = tables[j]->kind;
    tb.ref_index[j] = tables[j]->ref_index;
  }
  // scratch layout: op, avail, supply, min_batch, flags (i32 x N each), then the select
  // outputs idx, code, fill (i32), obj, slack, wait (f64), kind_min (f64 x N*K)
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  uint8_t* s = static_cast<uint8_t*>(scratch);
  int32_t* d_op = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  int32_t* d_av = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  int32_t* d_sup = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  int32_t* d_mb = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  uint32_t* d_fl = reinterpret_cast<uint32_t*>(s); s += al(4u * N);
  int32_t* d_idx = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  int32_t* d_code = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  int32_t* d_fill = reinterpret_cast<int32_t*>(s); s += al(4u * N);
  double* d_obj = reinterpret_cast<double*>(s); s += al(8u * N);
  double* d_sl = reinterpret_cast<double*>(s); s += al(8u * N);
  double* d_wait = reinterpret_cast<double*>(s); s += al(8u * N);
  double* d_kmin = reinterpret_cast<double*>(s);
  k_commit_prep<<<(N + 255) / 256, 256, 0, ctx->stream>>>(N, n_ops, fill, buffered, full_mask,
                                                         d_op, d_av, d_sup, d_mb, d_fl);
  SP_CHECK_LAUNCH(ctx);
  int rc = select_launch(ctx, n_ops, tables, alpha, N, d_op, slack, d_av, d_sup, d_mb, d_fl, d_idx,
                         d_code, d_fill, d_obj, d_sl, d_wait, d_kmin, SP_MODE_AUTO);
  if (rc != SP_OK) return rc;
  const int threads = 256;
  int lg = 0;
  while ((1 << lg) < n_ops && lg < 5) ++lg;  // lanes per round: next power of two, <= 32
  k_commit_round<<<(int)(((size_t)R * (1 << lg) + threads - 1) / threads), threads, 0, ctx->stream>>>(
      R, n_ops, K, lg, tb, slack, fill, head_id, depth, hflags, spec_idx, spec_slack, spec_obj,
      full_mask, policy, d_idx, d_fill, d_obj, d_sl, d_kmin, out_idx, out_fill, out_slack,
      out_obj, out_aff, out_best);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

size_t commit_scratch_bytes(int R, int n_ops, int K) {
  const size_t N = (size_t)R * n_ops;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return 8 * al(4 * N) + 3 * al(8 * N) + al(8 * N * K);
}

}  // namespace sp
