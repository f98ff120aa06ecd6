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
#include <stdlib.h>
#include <string.h>

#include <cmath>

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

__device__ __forceinline__ void store_slack(int i, int s, int n_src, double own, double tmax,
                                            double tmin, double base, int K,
                                            const double* __restrict__ Q,
                                            double* __restrict__ out_slack,
                                            double* __restrict__ out_ratio) {
  const double ratio_lo = __ddiv_rn(own, tmax);  // min over suffixes of own/total
  const double ratio_hi = __ddiv_rn(own, tmin);  // max over suffixes of own/total
  const size_t o = (size_t)i * n_src + s;
  if (out_ratio) {
    out_ratio[2 * o] = ratio_lo;
    out_ratio[2 * o + 1] = ratio_hi;
  }
  if (out_slack) {
    for (int k = 0; k < K; ++k) {
      const double b = __dsub_rn(base, __ldg(Q + (size_t)i * K + k));
      out_slack[o * K + k] = __dmul_rn(b >= 0.0 ? ratio_lo : ratio_hi, b);
    }
  }
}

// store_slack with the K budgets b_k = (target - now) - Q[k] computed once per instance
// (K <= 4: the per-source loop then reads no Q)
__device__ __forceinline__ void store_slack4(int i, int s, int n_src, double own, double tmax,
                                             double tmin, int K, const double (&bq)[4],
                                             double* __restrict__ out_slack,
                                             double* __restrict__ out_ratio) {
  const double ratio_lo = __ddiv_rn(own, tmax);
  const double ratio_hi = __ddiv_rn(own, tmin);
  const size_t o = (size_t)i * n_src + s;
  if (out_ratio) {
    out_ratio[2 * o] = ratio_lo;
    out_ratio[2 * o + 1] = ratio_hi;
  }
  if (out_slack) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < K) out_slack[o * K + k] = __dmul_rn(bq[k] >= 0.0 ? ratio_lo : ratio_hi, bq[k]);
  }
}

// ---- K1c: certified backward pass -------------------------------------------------------
// The forward DP above relaxes every edge of every source's descendant set (19,227 edge
// relaxations per instance on config 3's 64-op DAG).  K1c finds each source's extremal path
// with ONE backward pass over the graph (845 edges) and then proves, per source, that the
// path it found is the one the reference's left-to-right sums make extremal:
//   backward:  Hb[v] = fl(ref[v] + max(end_v ? 0 : -inf, max_u Hb[u]))   (u: successors)
//              argmax[v] = the option taken, gap[v] = its value minus the runner-up option's,
//              rounded down to float (+inf without a runner-up), G[v] = min(gap[v],
//              G[argmax[v]]) the smallest margin along the path;  min side alike.
//   Monotone rounding makes Hb[v] = max over paths of the right-nested rounded path sums R, so
//   following argmax from s gives a path p^ with R(p^) = Hb[s]; the walk recomputes its forward
//   sum  Tmax = ((0 + r_s) + r_1) + ...  exactly as configurator.py:500-506 does.
//   Certificate: any other path p leaves p^ at some node v_j through a runner-up option, whose
//   best continuation has R <= Y_j - gap_j (Y_j = the chosen option's value, R of p^'s tail).
//   With recursive-summation bounds for non-negative terms (|fl - exact| <= g * exact,
//   g = V u / (1 - V u), u = 2^-53) on the forward sums of p and p^ and on R, p's forward sum
//   cannot exceed Tmax once gap_j >= 2g A_j + 4.01g Y_j, which min_j gap_j >= theta * Tmax
//   (theta = 5g + 8u), i.e. G[s] >= theta * Tmax, implies.  So Tmax IS the reference's maximum; the min side mirrors it
//   (max orientation on negated values, the same gap test against Tmin).
// Sources whose certificate fails (near-ties within ~1e-13 relative, exact ties, refs that are
// negative / non-finite / > 1e300) fall back to the exact forward DP of that source, so the
// output is bit-identical to k_slack in every case.
// Layout: TWO lanes per instance — the even lane runs the max side, the odd lane the min side
// (in max orientation on negated values, so both run the same code) — which halves the shared
// memory per lane and doubles the resident warps; the walks are then shared out by source
// parity, two sources per lane in flight.  Per instance and node 26 bytes of shared memory:
// {Hb, -Lb} (later the walk record {ref, G_max | G_min}), the two float margins, the two args.
constexpr uint32_t kArgNone = 0xFE, kArgEnd = 0xFF;
constexpr int kCertWarps = 2;  // 32 instances per block (4 warps per block measured the same)

// one walk step along an extremal path: add the node's ref to the forward sum, follow the arg
struct Walk {
  uint32_t v;  // current node; kArgEnd / kArgNone once the path has ended
  double acc;  // forward sum ((0 + r_s) + r_1) + ... along the path
};

template <bool MAX, int ROW = 16>
__device__ __forceinline__ void walk_step(Walk& c, const double2* __restrict__ W,
                                          const uint16_t* __restrict__ R) {
  // branch-free: a finished chain re-reads node 0 and keeps its state
  const bool on = c.v < kArgNone;
  const uint32_t v = on ? c.v : 0u;
  const double rv = W[v * ROW].x;
  const uint32_t rr = R[v * ROW];
  const double acc = __dadd_rn(c.acc, rv);
  c.acc = on ? acc : c.acc;
  c.v = on ? (MAX ? (rr & 0xFFu) : (rr >> 8)) : c.v;
}

__global__ void __launch_bounds__(32 * kCertWarps) k_slack_cert(
    const uint8_t* __restrict__ cert, int cert_bytes, int V, int n_src, int off_vidx,
    int off_term, int off_src, int off_succ, const int4* __restrict__ prog,
    const int32_t* __restrict__ prog_ptr, const uint32_t* __restrict__ preds,
    const int32_t* __restrict__ pred_ptr, int I, const double* __restrict__ ref, int ref_stride,
    const double* __restrict__ target, const double* __restrict__ now, int K,
    const double* __restrict__ Q, double theta, double* __restrict__ out_slack,
    double* __restrict__ out_ratio) {
  extern __shared__ __align__(16) uint8_t smc[];
  for (int t = threadIdx.x; t < cert_bytes / 16; t += blockDim.x)
    reinterpret_cast<uint4*>(smc)[t] = __ldg(reinterpret_cast<const uint4*>(cert) + t);
  __syncthreads();
  const uint16_t* SP = reinterpret_cast<const uint16_t*>(smc);
  const uint16_t* VI = reinterpret_cast<const uint16_t*>(smc + off_vidx);
  const uint8_t* TE = smc + off_term;
  const uint8_t* SRC = smc + off_src;
  const uint16_t* SU = reinterpret_cast<const uint16_t*>(smc + off_succ);  // groups of 4 offsets
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = lane >> 1, side = lane & 1;  // instance in the warp, 0 = max / 1 = min side
  const int nfw = (n_src + 31) >> 5;
  const size_t arow = (size_t)(V + 1) * 256;  // A has a sentinel row V (-inf on both sides)
  uint8_t* wb = smc + cert_bytes + (size_t)warp * (arow + (size_t)V * 160 + (size_t)nfw * 128);
  // element (v, k, side) of each [V][16][2] array sits at v * 32 + 2k + side
  double* A = reinterpret_cast<double*>(wb) + 2 * k;
  float* Cf = reinterpret_cast<float*>(wb + arow) + 2 * k;
  uint8_t* Rb = wb + arow + (size_t)V * 128 + 2 * k;
  uint32_t* Fw = reinterpret_cast<uint32_t*>(wb + arow + (size_t)V * 160) + lane;
  const char* As = reinterpret_cast<const char*>(A + side);  // + node * 256: this lane's value
  const double2* W = reinterpret_cast<const double2*>(A);  // walk record (v, k) at v * 16
  const uint16_t* R = reinterpret_cast<const uint16_t*>(Rb);
  const int i0 = (blockIdx.x * kCertWarps + warp) * 16;
  if (i0 >= I) return;
  const int i = i0 + k;
  const bool live = i < I;
  const double* r = ref + (size_t)(live ? i : i0) * ref_stride;

  // ---- backward pass in max orientation (the min side negates), reverse topological order ----
  A[V * 32 + side] = -INFINITY;
  bool bad = false;
  double rn = __ldg(r + VI[V - 1]);
  for (int v = V - 1; v >= 0; --v) {
    const double rv = rn;
    if (v > 0) rn = __ldg(r + VI[v - 1]);
    bad |= !(rv >= 0.0 && rv <= 1e300);
    const bool te = TE[v] != 0;
    double h1 = te ? 0.0 : -INFINITY, h2 = -INFINITY;
    uint32_t a1 = te ? (kArgEnd << 8) : (kArgNone << 8);  // chosen option as a byte offset
    for (int q = SP[v]; q < SP[v + 1]; ++q) {
      const uint2 w = *reinterpret_cast<const uint2*>(SU + 4 * q);
      const uint32_t u0 = w.x & 0xFFFFu, u1 = w.x >> 16, u2 = w.y & 0xFFFFu, u3 = w.y >> 16;
      const double x0 = *reinterpret_cast<const double*>(As + u0);
      const double x1 = *reinterpret_cast<const double*>(As + u1);
      const double x2 = *reinterpret_cast<const double*>(As + u2);
      const double x3 = *reinterpret_cast<const double*>(As + u3);
      // top two of the four (and the arg of the best), merged into the running pair; an exact
      // tie leaves the runner-up equal to the best, which fails the certificate as it must
      const bool g01 = x1 > x0, g23 = x3 > x2;
      const double m01 = g01 ? x1 : x0, s01 = g01 ? x0 : x1;
      const double m23 = g23 ? x3 : x2, s23 = g23 ? x2 : x3;
      const uint32_t i01 = g01 ? u1 : u0, i23 = g23 ? u3 : u2;
      const bool gq = m23 > m01;
      const double M = gq ? m23 : m01;
      const double lo = gq ? m01 : m23;
      const double sm = s01 > s23 ? s01 : s23;
      const double S = lo > sm ? lo : sm;
      const uint32_t iq = gq ? i23 : i01;
      const bool gt = M > h1;
      const double l2 = gt ? h1 : M;
      const double s2 = S > h2 ? S : h2;
      h2 = l2 > s2 ? l2 : s2;
      h1 = gt ? M : h1;
      a1 = gt ? iq : a1;
    }
    a1 >>= 8;  // node id, or kArgEnd / kArgNone
    A[v * 32 + side] = __dadd_rn(side ? -rv : rv, h1);
    // smallest margin along the extremal path from v: this node's chosen option over its
    // runner-up, then the successor's path (-inf when no path: the certificate fails)
    float gm = __double2float_rd(__dsub_rd(h1, h2));
    if (a1 < kArgNone) {
      const float gn = Cf[a1 * 32 + side];
      gm = gn < gm ? gn : gm;
    } else if (a1 == kArgNone) {
      gm = -INFINITY;
    }
    Cf[v * 32 + side] = gm;
    Rb[v * 32 + side] = (uint8_t)a1;
  }
  bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
  __syncwarp();
  // walk records {ref, G_max | G_min}: the even lane brings the ref, the odd lane the margins
#pragma unroll 8
  for (int v = 0; v < V; ++v)
    A[v * 32 + side] = side ? *reinterpret_cast<const double*>(Cf + v * 32) : __ldg(r + VI[v]);
  for (int w = 0; w < nfw; ++w) Fw[w * 32] = 0u;
  __syncwarp();

  // configurator.py:535  budget = self.target_s - now - queueing[k]
  const double base = live ? __dsub_rn(__ldg(target + i), __ldg(now + i)) : 0.0;
  // configurator.py:535 per kind, once per instance (K <= 4; larger K reads Q per source)
  double bq[4] = {0.0, 0.0, 0.0, 0.0};
  if (live && K <= 4)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      if (kk < K) bq[kk] = __dsub_rn(base, __ldg(Q + (size_t)i * K + kk));
  // ---- per source: walk both extremal paths, certify, emit (sources by parity, 2 at once) ----
  for (int g = side; g < n_src; g += 4) {
    const int sa = g, sb = g + 2 < n_src ? g + 2 : -1;
    const uint32_t va = SRC[sa], vb = sb >= 0 ? SRC[sb] : 0u;
    Walk ha{va, 0.0}, la{va, 0.0};
    Walk hb{sb >= 0 ? vb : kArgEnd, 0.0}, lb{sb >= 0 ? vb : kArgEnd, 0.0};
    while (ha.v < kArgNone || la.v < kArgNone || hb.v < kArgNone || lb.v < kArgNone) {
      walk_step<true>(ha, W, R);
      walk_step<false>(la, W, R);
      walk_step<true>(hb, W, R);
      walk_step<false>(lb, W, R);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int si = q ? sb : sa;
      if (si < 0) continue;
      const Walk& h = q ? hb : ha;
      const Walk& l = q ? lb : la;
      const double2 ws = W[SRC[si] * 16];
      const float gh = __int_as_float(__double2loint(ws.y));
      const float gl = __int_as_float(__double2hiint(ws.y));
      const bool ok = !bad && (double)gh >= __dmul_ru(theta, h.acc) &&
                      (double)gl >= __dmul_ru(theta, l.acc);
      if (ok) {
        if (live) {
          const double own = __dadd_rn(0.0, ws.x);
          if (K <= 4)
            store_slack4(i, si, n_src, own, h.acc, l.acc, K, bq, out_slack, out_ratio);
          else
            store_slack(i, si, n_src, own, h.acc, l.acc, base, K, Q, out_slack, out_ratio);
        }
      } else {
        Fw[(si >> 5) * 32] |= 1u << (si & 31);
      }
    }
  }
  __syncwarp();

  // ---- uncertified sources: the exact forward DP (k_slack's program, read from global), one
  // side at a time, slots in the instance's [V] x 16-byte column ----
  double2* D = reinterpret_cast<double2*>(A);
  for (int sd = 0; sd < 2; ++sd) {
    if (side == sd) {
      for (int w = 0; w < nfw; ++w) {
        uint32_t bits = Fw[w * 32];
        while (bits) {
          const int si = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          const int4* Ps = prog + prog_ptr[si];
          const int n = prog_ptr[si + 1] - prog_ptr[si];
          const uint32_t* Gs = preds + pred_ptr[si];
          const int4 head = Ps[0];
          const double own = __dadd_rn(0.0, __ldg(r + head.x));
          D[(head.y & 0xffff) * 16] = make_double2(own, own);
          double tmax = (head.y >> 16) ? own : -INFINITY;
          double tmin = (head.y >> 16) ? own : INFINITY;
          for (int e = 1; e < n; ++e) {
            const int4 pr = Ps[e];
            const double rv = __ldg(r + pr.x);
            double hm = -INFINITY, lm = INFINITY;
            for (int t = 0; t < 2 * pr.w; ++t) {
              const double2 a = D[Gs[pr.z + t] * 16];
              hm = hm > a.x ? hm : a.x;
              lm = lm < a.y ? lm : a.y;
            }
            const double h = __dadd_rn(hm, rv), l = __dadd_rn(lm, rv);
            D[(pr.y & 0xffff) * 16] = make_double2(h, l);
            if (pr.y >> 16) {
              tmax = h > tmax ? h : tmax;
              tmin = l < tmin ? l : tmin;
            }
          }
          if (live) store_slack(i, si, n_src, own, tmax, tmin, base, K, Q, out_slack, out_ratio);
        }
      }
    }
    __syncwarp();
  }
}

// K1c, four lanes per instance: lanes (instance k, side, sub) — 8 instances per warp, half the
// shared memory per warp of k_slack_cert, so twice the resident warps.  The two sub-lanes of a
// side split every node's successor groups (even / odd groups; the terminal option in sub 0)
// and merge their (best, runner-up, arg) by one shuffle — the merged best and runner-up are the
// sequential scan's (an exact tie leaves the runner-up equal to the best, failing the
// certificate exactly as there); the four lanes split the per-source walks (sources L, L + 4,
// L + 8, ... for L = 2 side + sub).  Everything else — the certificate, the forward sums, the
// fallback forward DP — is k_slack_cert's, so the results are identical.
__global__ void __launch_bounds__(32 * kCertWarps) k_slack_cert4(
    const uint8_t* __restrict__ cert, int cert_bytes, int V, int n_src, int off_vidx,
    int off_term, int off_src, int off_succ, const int4* __restrict__ prog,
    const int32_t* __restrict__ prog_ptr, const uint32_t* __restrict__ preds,
    const int32_t* __restrict__ pred_ptr, int I, const double* __restrict__ ref, int ref_stride,
    const double* __restrict__ target, const double* __restrict__ now, int K,
    const double* __restrict__ Q, double theta, double* __restrict__ out_slack,
    double* __restrict__ out_ratio) {
  extern __shared__ __align__(16) uint8_t smc[];
  for (int t = threadIdx.x; t < cert_bytes / 16; t += blockDim.x)
    reinterpret_cast<uint4*>(smc)[t] = __ldg(reinterpret_cast<const uint4*>(cert) + t);
  __syncthreads();
  const uint16_t* SP = reinterpret_cast<const uint16_t*>(smc);
  const uint16_t* VI = reinterpret_cast<const uint16_t*>(smc + off_vidx);
  const uint8_t* TE = smc + off_term;
  const uint8_t* SRC = smc + off_src;
  const uint16_t* SU = reinterpret_cast<const uint16_t*>(smc + off_succ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = lane >> 2, side = (lane >> 1) & 1, sub = lane & 1, L = lane & 3;
  const int nfw = (n_src + 31) >> 5;
  const size_t arow = (size_t)(V + 1) * 128;  // [V+1][8][2] doubles (sentinel row V)
  uint8_t* wb = smc + cert_bytes + (size_t)warp * (arow + (size_t)V * 80 + (size_t)nfw * 128);
  // element (v, k, side) of each [V][8][2] array sits at v * 16 + 2k + side
  double* A = reinterpret_cast<double*>(wb) + 2 * k;
  float* Cf = reinterpret_cast<float*>(wb + arow) + 2 * k;
  uint8_t* Rb = wb + arow + (size_t)V * 64 + 2 * k;
  uint32_t* Fw = reinterpret_cast<uint32_t*>(wb + arow + (size_t)V * 80) + lane;
  const char* As = reinterpret_cast<const char*>(A + side);  // + node * 128
  const double2* W = reinterpret_cast<const double2*>(A);   // walk record (v, k) at v * 8
  const uint16_t* R = reinterpret_cast<const uint16_t*>(Rb);
  const int i0 = (blockIdx.x * kCertWarps + warp) * 8;
  if (i0 >= I) return;
  const int i = i0 + k;
  const bool live = i < I;
  const double* r = ref + (size_t)(live ? i : i0) * ref_stride;

  if (sub == 0) A[V * 16 + side] = -INFINITY;
  __syncwarp();
  bool bad = false;
  double rn = __ldg(r + VI[V - 1]);
  for (int v = V - 1; v >= 0; --v) {
    const double rv = rn;
    if (v > 0) rn = __ldg(r + VI[v - 1]);
    bad |= !(rv >= 0.0 && rv <= 1e300);
    const bool te = TE[v] != 0 && sub == 0;  // the terminal option is sub 0's
    double h1 = te ? 0.0 : -INFINITY, h2 = -INFINITY;
    uint32_t a1 = te ? (kArgEnd << 8) : (kArgNone << 8);
    for (int q = SP[v] + sub; q < SP[v + 1]; q += 2) {
      const uint2 w = *reinterpret_cast<const uint2*>(SU + 4 * q);
      const uint32_t u0 = w.x & 0xFFFFu, u1 = w.x >> 16, u2 = w.y & 0xFFFFu, u3 = w.y >> 16;
      const double x0 = *reinterpret_cast<const double*>(As + (u0 >> 1));
      const double x1 = *reinterpret_cast<const double*>(As + (u1 >> 1));
      const double x2 = *reinterpret_cast<const double*>(As + (u2 >> 1));
      const double x3 = *reinterpret_cast<const double*>(As + (u3 >> 1));
      const bool g01 = x1 > x0, g23 = x3 > x2;
      const double m01 = g01 ? x1 : x0, s01 = g01 ? x0 : x1;
      const double m23 = g23 ? x3 : x2, s23 = g23 ? x2 : x3;
      const uint32_t i01 = g01 ? u1 : u0, i23 = g23 ? u3 : u2;
      const bool gq = m23 > m01;
      const double M = gq ? m23 : m01;
      const double lo = gq ? m01 : m23;
      const double sm = s01 > s23 ? s01 : s23;
      const double S = lo > sm ? lo : sm;
      const uint32_t iq = gq ? i23 : i01;
      const bool gt = M > h1;
      const double l2 = gt ? h1 : M;
      const double s2 = S > h2 ? S : h2;
      h2 = l2 > s2 ? l2 : s2;
      h1 = gt ? M : h1;
      a1 = gt ? iq : a1;
    }
    {  // merge the two halves: best, runner-up (a tie makes them equal), the best's arg
      const double ph1 = __shfl_xor_sync(0xffffffffu, h1, 1);
      const double ph2 = __shfl_xor_sync(0xffffffffu, h2, 1);
      const uint32_t pa1 = __shfl_xor_sync(0xffffffffu, a1, 1);
      const double H1 = h1 > ph1 ? h1 : ph1;
      const double lo = h1 > ph1 ? ph1 : h1;
      const double sm = h2 > ph2 ? h2 : ph2;
      h2 = lo > sm ? lo : sm;
      const uint32_t a0 = sub ? pa1 : a1, a1b = sub ? a1 : pa1;  // sub 0's, sub 1's
      const double h0 = sub ? ph1 : h1, h1b = sub ? h1 : ph1;
      a1 = h1b > h0 ? a1b : a0;
      h1 = H1;
    }
    a1 >>= 8;
    float gm = __double2float_rd(__dsub_rd(h1, h2));
    if (a1 < kArgNone) {
      const float gn = Cf[a1 * 16 + side];
      gm = gn < gm ? gn : gm;
    } else if (a1 == kArgNone) {
      gm = -INFINITY;
    }
    if (sub == 0) {  // both sub-lanes hold the merged values; one writes
      A[v * 16 + side] = __dadd_rn(side ? -rv : rv, h1);
      Cf[v * 16 + side] = gm;
      Rb[v * 16 + side] = (uint8_t)a1;
    }
    __syncwarp();
  }
  bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
  bad |= __shfl_xor_sync(0xffffffffu, bad, 2);
  __syncwarp();
  // walk records {ref, G_max | G_min}: side 0 brings the ref, side 1 the margins, sub-lanes split v
#pragma unroll 4
  for (int v = sub; v < V; v += 2)
    A[v * 16 + side] = side ? *reinterpret_cast<const double*>(Cf + v * 16) : __ldg(r + VI[v]);
  for (int w = 0; w < nfw; ++w) Fw[w * 32] = 0u;
  __syncwarp();

  const double base = live ? __dsub_rn(__ldg(target + i), __ldg(now + i)) : 0.0;
  double bq[4] = {0.0, 0.0, 0.0, 0.0};
  if (live && K <= 4)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      if (kk < K) bq[kk] = __dsub_rn(base, __ldg(Q + (size_t)i * K + kk));
  // ---- per source (sources L, L + 4, ... in pairs): walk both extremal paths, certify, emit ----
  for (int g = L; g < n_src; g += 8) {
    const int sa = g, sb = g + 4 < n_src ? g + 4 : -1;
    const uint32_t va = SRC[sa], vb = sb >= 0 ? SRC[sb] : 0u;
    Walk ha{va, 0.0}, la{va, 0.0};
    Walk hb{sb >= 0 ? vb : kArgEnd, 0.0}, lb{sb >= 0 ? vb : kArgEnd, 0.0};
    while (ha.v < kArgNone || la.v < kArgNone || hb.v < kArgNone || lb.v < kArgNone) {
      walk_step<true, 8>(ha, W, R);
      walk_step<false, 8>(la, W, R);
      walk_step<true, 8>(hb, W, R);
      walk_step<false, 8>(lb, W, R);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int si = q ? sb : sa;
      if (si < 0) continue;
      const Walk& h = q ? hb : ha;
      const Walk& l = q ? lb : la;
      const double2 ws = W[SRC[si] * 8];
      const float gh = __int_as_float(__double2loint(ws.y));
      const float gl = __int_as_float(__double2hiint(ws.y));
      const bool ok = !bad && (double)gh >= __dmul_ru(theta, h.acc) &&
                      (double)gl >= __dmul_ru(theta, l.acc);
      if (ok) {
        if (live) {
          const double own = __dadd_rn(0.0, ws.x);
          if (K <= 4)
            store_slack4(i, si, n_src, own, h.acc, l.acc, K, bq, out_slack, out_ratio);
          else
            store_slack(i, si, n_src, own, h.acc, l.acc, base, K, Q, out_slack, out_ratio);
        }
      } else {
        Fw[(si >> 5) * 32] |= 1u << (si & 31);
      }
    }
  }
  __syncwarp();

  // ---- uncertified sources: the exact forward DP, one lane of the instance at a time ----
  double2* D = reinterpret_cast<double2*>(A);
  for (int sd = 0; sd < 4; ++sd) {
    if (L == sd) {
      for (int w = 0; w < nfw; ++w) {
        uint32_t bits = Fw[w * 32];
        while (bits) {
          const int si = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          const int4* Ps = prog + prog_ptr[si];
          const int n = prog_ptr[si + 1] - prog_ptr[si];
          const uint32_t* Gs = preds + pred_ptr[si];
          const int4 head = Ps[0];
          const double own = __dadd_rn(0.0, __ldg(r + head.x));
          D[(head.y & 0xffff) * 8] = make_double2(own, own);
          double tmax = (head.y >> 16) ? own : -INFINITY;
          double tmin = (head.y >> 16) ? own : INFINITY;
          for (int e = 1; e < n; ++e) {
            const int4 pr = Ps[e];
            const double rv = __ldg(r + pr.x);
            double hm = -INFINITY, lm = INFINITY;
            for (int t = 0; t < 2 * pr.w; ++t) {
              const double2 a = D[Gs[pr.z + t] * 8];
              hm = hm > a.x ? hm : a.x;
              lm = lm < a.y ? lm : a.y;
            }
            const double h = __dadd_rn(hm, rv), l = __dadd_rn(lm, rv);
            D[(pr.y & 0xffff) * 8] = make_double2(h, l);
            if (pr.y >> 16) {
              tmax = h > tmax ? h : tmax;
              tmin = l < tmin ? l : tmin;
            }
          }
          if (live) store_slack(i, si, n_src, own, tmax, tmin, base, K, Q, out_slack, out_ratio);
        }
      }
    }
    __syncwarp();
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
  if (g->cert && ctx->opt.k1_cert != 1 && ctx->opt.k1c_lanes == 4) {
    const int nfw = (g->n_src + 31) / 32;
    const size_t smem = (size_t)g->cert_bytes +
                        (size_t)kCertWarps * ((size_t)(g->V + 1) * 128 + (size_t)g->V * 80 +
                                              (size_t)nfw * 128);
    if (smem <= 227 * 1024) {
      static size_t cert4_attr_dev[64] = {};
      size_t& cert_attr = cert4_attr_dev[cur_device()];
      if (smem > 48 * 1024 && smem > cert_attr) {
        SP_CUDA(cudaFuncSetAttribute(k_slack_cert4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        cert_attr = smem;
      }
      const double u = std::ldexp(1.0, -53);
      const double gam = g->V * u / (1.0 - g->V * u);
      const int per_block = 8 * kCertWarps;
      k_slack_cert4<<<(I + per_block - 1) / per_block, 32 * kCertWarps, smem, ctx->stream>>>(
          g->cert, g->cert_bytes, g->V, g->n_src, g->off_vidx, g->off_term, g->off_src,
          g->off_succ, g->prog, g->prog_ptr, g->preds, g->pred_ptr, I, ref, ref_stride, target,
          now, K, Q, 5.0 * gam + 8.0 * u, out_slack, out_ratio);
      SP_CHECK_LAUNCH(ctx);
      return SP_OK;
    }
  }
  if (g->cert && ctx->opt.k1_cert != 1) {
    const int nfw = (g->n_src + 31) / 32;
    const size_t smem = (size_t)g->cert_bytes +
                        (size_t)kCertWarps * ((size_t)(g->V + 1) * 256 + (size_t)g->V * 160 +
                                              (size_t)nfw * 128);
    if (smem <= 227 * 1024) {
      static size_t cert_attr_dev[64] = {};
      size_t& cert_attr = cert_attr_dev[cur_device()];
      if (smem > 48 * 1024 && smem > cert_attr) {
        SP_CUDA(cudaFuncSetAttribute(k_slack_cert, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        cert_attr = smem;
      }
      const double u = std::ldexp(1.0, -53);
      const double gam = g->V * u / (1.0 - g->V * u);
      const int per_block = 16 * kCertWarps;
      k_slack_cert<<<(I + per_block - 1) / per_block, 32 * kCertWarps, smem, ctx->stream>>>(
          g->cert, g->cert_bytes, g->V, g->n_src, g->off_vidx, g->off_term, g->off_src,
          g->off_succ, g->prog, g->prog_ptr, g->preds, g->pred_ptr, I, ref, ref_stride, target,
          now, K, Q, 5.0 * gam + 8.0 * u, out_slack, out_ratio);
      SP_CHECK_LAUNCH(ctx);
      return SP_OK;
    }
  }
  const size_t smem = (size_t)kSlackWarps * g->max_slots * 32 * sizeof(double2) +
                      (size_t)g->max_span * sizeof(int4) +
                      (size_t)g->max_preds * sizeof(uint32_t);
  if (smem > 227 * 1024) return fail(SP_E_UNSUPPORTED, "slack: DAG too wide for shared memory");
  static size_t attr_set_dev[64] = {};
  size_t& attr_set = attr_set_dev[cur_device()];
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
