// sp_slack.cu — K1: Alg. 1 slack allotment (configurator.py:493-543, compute_slack 76-106)
// and the Eq. 2 ordered queueing sum (configurator.py:109-119, 511-524).
//
// Reference: for operation `op`, every decomposed path containing it contributes the
// ratio ref[op] / total, where total is accumulated LEFT TO RIGHT from 0.0 along the
// path suffix starting at op; slack_k = min over suffixes of ratio * budget_k with
// budget_k = (target - now) - Q_k.
//
// Restatement (exact): IEEE addition is monotone in each operand, so the
// largest / smallest left-to-right suffix total is obtained by a forward DP from op over
// its descendants in topological order,
//     H[v] = fl(max_{p in preds(v)} H[p] + ref[v]),  L[v] = fl(min_p L[p] + ref[v]),
// seeded with H[op] = L[op] = 0.0 + ref[op], and Tmax / Tmin taken over path ends.  Because
// x -> fl(own / x) is monotone decreasing and r -> fl(r * b) is monotone in r with the sign
// of b, min_r fl(r*b) = fl(fl(own/Tmax) * b) for b >= 0 and fl(fl(own/Tmin) * b) for b < 0.
// (A backward DP would sum right-to-left and is NOT bit-exact — SURVEY.md finding 3.)
//
// Layout: one warp = (source vertex s, 32 consecutive pipeline instances).  Every lane runs
// the same per-source vertex program (descendants of s in topological order with their
// predecessor slots), so the warp never diverges; the DP values live in shared memory as
// [slot][lane] doubles (conflict-free 256-byte rows).
#include <math.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kWarpsPerBlock = 2;

// prog entry: x = value index, y = terminal flag, z = pred begin, w = pred end (into preds)
__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_slack(
    const int4* __restrict__ prog, const int32_t* __restrict__ prog_ptr,
    const uint16_t* __restrict__ preds, int slots_max, int I,
    const double* __restrict__ ref, int ref_stride, const double* __restrict__ target,
    const double* __restrict__ now, int K, const double* __restrict__ Q, int n_src,
    double* __restrict__ out_slack, double* __restrict__ out_ratio) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.y;
  const int i = (blockIdx.x * kWarpsPerBlock + warp) * 32 + lane;
  const bool live = i < I;
  const int ii = live ? i : 0;
  double* H = sm + (size_t)warp * slots_max * 64;
  double* L = H + (size_t)slots_max * 32;
  const double* r = ref + (size_t)ii * ref_stride;

  const int pb = prog_ptr[s], pe = prog_ptr[s + 1];
  const int4 head = prog[pb];
  const double own = __dadd_rn(0.0, __ldg(r + head.x));  // total = 0.0; total += ref[op]
  H[lane] = own;
  L[lane] = own;
  double tmax = head.y ? own : -INFINITY;
  double tmin = head.y ? own : INFINITY;
  for (int e = pb + 1; e < pe; ++e) {
    const int4 pr = prog[e];
    const double rv = __ldg(r + pr.x);
    double hm = -INFINITY, lm = INFINITY;
    int q = pr.z;
    for (; q + 1 < pr.w; q += 2) {  // two independent predecessor loads in flight
      const int a = preds[q], b = preds[q + 1];
      const double ha = H[a * 32 + lane], hb = H[b * 32 + lane];
      const double la = L[a * 32 + lane], lb = L[b * 32 + lane];
      const double hx = ha > hb ? ha : hb;
      const double lx = la < lb ? la : lb;
      hm = hx > hm ? hx : hm;
      lm = lx < lm ? lx : lm;
    }
    if (q < pr.w) {
      const int a = preds[q];
      const double ha = H[a * 32 + lane], la = L[a * 32 + lane];
      hm = ha > hm ? ha : hm;
      lm = la < lm ? la : lm;
    }
    const int slot = e - pb;
    const double h = __dadd_rn(hm, rv), l = __dadd_rn(lm, rv);
    H[slot * 32 + lane] = h;
    L[slot * 32 + lane] = l;
    if (pr.y) {
      tmax = h > tmax ? h : tmax;
      tmin = l < tmin ? l : tmin;
    }
  }
  if (!live) return;
  const double ratio_lo = __ddiv_rn(own, tmax);  // min over suffixes of own/total
  const double ratio_hi = __ddiv_rn(own, tmin);  // max over suffixes of own/total
  const size_t o = (size_t)i * n_src + s;
  if (out_ratio) {
    out_ratio[2 * o] = ratio_lo;
    out_ratio[2 * o + 1] = ratio_hi;
  }
  if (out_slack) {
    // configurator.py:535  budget = self.target_s - now - queueing[k]
    const double base = __dsub_rn(__ldg(target + i), __ldg(now + i));
    for (int k = 0; k < K; ++k) {
      const double b = __dsub_rn(base, __ldg(Q + (size_t)i * K + k));
      out_slack[o * K + k] = __dmul_rn(b >= 0.0 ? ratio_lo : ratio_hi, b);
    }
  }
}

// Eq. 2 ordered sum, one thread per kind (configurator.py:516-523 / 116-119).
__global__ void k_queueing(int K, const int32_t* __restrict__ ptr, const double* __restrict__ lat,
                           const double* __restrict__ res, const int32_t* __restrict__ cnt,
                           const double* __restrict__ pool, double* __restrict__ out) {
  int k = threadIdx.x;
  if (k >= K) return;
  double total = 0.0;
  const double P = pool[k];
  for (int j = ptr[k]; j < ptr[k + 1]; ++j) {
    if (cnt) {
      // total += count * (t.lat[eidx] * t.res[eidx])
      total = __dadd_rn(total, __dmul_rn((double)cnt[j], __dmul_rn(lat[j], res[j])));
    } else {
      // total += e.latency_s * e.resource_request / pool_resources
      total = __dadd_rn(total, __ddiv_rn(__dmul_rn(lat[j], res[j]), P));
    }
  }
  out[k] = cnt ? __ddiv_rn(total, P) : total;
}

}  // namespace

int slack_launch(sp_ctx* ctx, sp_dag* g, int I, const double* ref, int ref_stride,
                 const double* target, const double* now, int K, const double* Q,
                 double* out_slack, double* out_ratio) {
  if (I == 0) return SP_OK;
  const size_t smem = (size_t)kWarpsPerBlock * g->max_span * 64 * sizeof(double);
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    SP_CUDA(cudaFuncSetAttribute(k_slack, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_set = smem;
  }
  if (smem > 227 * 1024) return fail(SP_E_UNSUPPORTED, "slack: DAG too wide for shared memory");
  dim3 grid((I + 32 * kWarpsPerBlock - 1) / (32 * kWarpsPerBlock), g->n_src);
  k_slack<<<grid, 32 * kWarpsPerBlock, smem, ctx->stream>>>(
      g->prog, g->prog_ptr, g->preds, g->max_span, I, ref, ref_stride, target,
      now, K, Q, g->n_src, out_slack, out_ratio);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

int queueing_launch(sp_ctx* ctx, int K, const int32_t* ptr, const double* lat,
                    const double* res, const int32_t* cnt, const double* pool, double* out) {
  k_queueing<<<1, 32, 0, ctx->stream>>>(K, ptr, lat, res, cnt, pool, out);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace sp
