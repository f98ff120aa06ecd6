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
// Layout: one block = one source vertex s and 32 * kSlackWarps consecutive pipeline
// instances (one lane each).  The source's vertex program (descendants in topological
// order, predecessor slots as byte offsets in pairs) is staged once into shared memory, so
// every lane of every warp runs the same program without divergence and every program read
// is a shared-memory broadcast.  The DP values live in shared memory as [slot][lane]
// double2 {H, L}: one conflict-free 16-byte load per predecessor.  Slots are reused once a
// value's last reader has run (sp_dag_create), and the per-vertex ref loads from global
// memory run four vertices ahead in a register shift ring, so the per-vertex dependency
// chain is program broadcast -> DP loads -> compare tree -> add -> store.
#include <math.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kSlackWarps = 4;

__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }

// prog entry: x = value index, y = out slot | terminal << 16, z = pred offset (entries,
// relative to the source's pred block, even), w = pred pairs
__global__ void __launch_bounds__(32 * kSlackWarps) k_slack(
    const int4* __restrict__ prog, const int32_t* __restrict__ prog_ptr,
    const uint32_t* __restrict__ preds, const int32_t* __restrict__ pred_ptr, int nslots,
    int max_span, int I, const double* __restrict__ ref, int ref_stride,
    const double* __restrict__ target, const double* __restrict__ now, int K,
    const double* __restrict__ Q, int n_src, double* __restrict__ out_slack,
    double* __restrict__ out_ratio) {
  extern __shared__ __align__(16) double2 smd[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.y;
  int4* P = reinterpret_cast<int4*>(smd + (size_t)kSlackWarps * nslots * 32);
  uint32_t* G = reinterpret_cast<uint32_t*>(P + max_span);
  const int pb = prog_ptr[s], n = prog_ptr[s + 1] - pb;
  const int qb = pred_ptr[s], nq = pred_ptr[s + 1] - qb;
  for (int t = threadIdx.x; t < n; t += blockDim.x) P[t] = prog[pb + t];
  // predecessor slots -> byte offsets of the slot's [lane 0] element
  for (int t = threadIdx.x; t < nq; t += blockDim.x) G[t] = preds[qb + t] * (32 * sizeof(double2));
  __syncthreads();
  const int i0 = (blockIdx.x * kSlackWarps + warp) * 32;
  if (i0 >= I) return;
  const int i = i0 + lane;
  const bool live = i < I;
  double2* D = smd + (size_t)warp * nslots * 32 + lane;
  const char* Db = reinterpret_cast<const char*>(D);
  const double* r = ref + (size_t)(live ? i : i0) * ref_stride;

  // ref values of the next four program entries, loaded ahead of use
  double r0 = __ldg(r + P[0].x);
  double r1 = n > 1 ? __ldg(r + P[1].x) : 0.0;
  double r2 = n > 2 ? __ldg(r + P[2].x) : 0.0;
  double r3 = n > 3 ? __ldg(r + P[3].x) : 0.0;
  const int4 head = P[0];
  const double own = __dadd_rn(0.0, r0);  // total = 0.0; total += ref[op]
  D[(head.y & 0xffff) * 32] = make_double2(own, own);
  double tmax = (head.y >> 16) ? own : -INFINITY;
  double tmin = (head.y >> 16) ? own : INFINITY;
  for (int e = 1; e < n; ++e) {
    r0 = r1;
    r1 = r2;
    r2 = r3;
    r3 = e + 3 < n ? __ldg(r + P[e + 3].x) : 0.0;
    const int4 pr = P[e];
    const uint2* g = reinterpret_cast<const uint2*>(G + pr.z);
    double hm = -INFINITY, lm = INFINITY;
    int t = 0;
    for (; t + 2 <= pr.w; t += 2) {  // four independent predecessor loads in flight
      const uint2 w0 = g[t], w1 = g[t + 1];
      const double2 a = *reinterpret_cast<const double2*>(Db + w0.x);
      const double2 b = *reinterpret_cast<const double2*>(Db + w0.y);
      const double2 c = *reinterpret_cast<const double2*>(Db + w1.x);
      const double2 d = *reinterpret_cast<const double2*>(Db + w1.y);
      hm = dmax(hm, dmax(dmax(a.x, b.x), dmax(c.x, d.x)));
      lm = dmin(lm, dmin(dmin(a.y, b.y), dmin(c.y, d.y)));
    }
    if (t < pr.w) {
      const uint2 w0 = g[t];
      const double2 a = *reinterpret_cast<const double2*>(Db + w0.x);
      const double2 b = *reinterpret_cast<const double2*>(Db + w0.y);
      hm = dmax(hm, dmax(a.x, b.x));
      lm = dmin(lm, dmin(a.y, b.y));
    }
    const double h = __dadd_rn(hm, r0), l = __dadd_rn(lm, r0);
    D[(pr.y & 0xffff) * 32] = make_double2(h, l);
    if (pr.y >> 16) {
      tmax = dmax(h, tmax);
      tmin = dmin(l, tmin);
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
  const size_t smem = (size_t)kSlackWarps * g->max_slots * 32 * sizeof(double2) +
                      (size_t)g->max_span * sizeof(int4) +
                      (size_t)g->max_preds * sizeof(uint32_t);
  if (smem > 227 * 1024) return fail(SP_E_UNSUPPORTED, "slack: DAG too wide for shared memory");
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    SP_CUDA(cudaFuncSetAttribute(k_slack, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_set = smem;
  }
  dim3 grid((I + 32 * kSlackWarps - 1) / (32 * kSlackWarps), g->n_src);
  k_slack<<<grid, 32 * kSlackWarps, smem, ctx->stream>>>(
      g->prog, g->prog_ptr, g->preds, g->pred_ptr, g->max_slots, g->max_span, I, ref,
      ref_stride, target, now, K, Q, g->n_src, out_slack, out_ratio);
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
