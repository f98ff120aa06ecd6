// sp_select.cu — K2: batched OpTable.select (configurator.py:239-300) on sm_100a.
//
// Two kernels, bit-identical to each other and to the reference:
//   k_select_plan  (K2b, the product path)  persistent CTAs stage the per-table staircase
//                  plans into shared memory with one TMA bulk copy (cp.async.bulk +
//                  mbarrier), then every thread decides one invocation per iteration
//                  (inputs for the next iteration prefetched into registers):
//                    per kind: a radix-accelerated threshold search (order-key bucket,
//                    then a short binary search inside the bucket) and one 32/64-byte
//                    staircase row;  rows of all admitted kinds are min-reduced with SIMD
//                    half-word minima, batch lanes outside [min_batch, available] are
//                    masked once at the end (min(a|m, b|m) = min(a, b)|m per lane);
//                    the best feasible and best infeasible candidates are compared on
//                    (score, r1) and only the winner's payload is loaded.
//   k_select_scan  (K2a, literal restatement)  every thread scans all M entries of its
//                  table (staged in shared memory, broadcast reads) and keeps the
//                  lexicographic (score, cost, res, id_rank) minima — exactly the
//                  masked-argmin-with-ties of configurator.py:229-237.  General (any
//                  number of batch sizes), O(M) per decision.
// Both then apply the safe-delayed-batching rule and the downgrade argmin
// (configurator.py:271-300).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kMaxPlanTables = 64;
constexpr int kMaxScanTables = 16;

struct PlanPtrs {
  const uint8_t* p[kMaxPlanTables];
  int n;
  int hv;     // h holds table 0's plan header (single-table launches): read via the constant bank
  PlanHdr h;
};

struct ScanTab {
  const double *lat, *cost, *costpen, *res;
  const int32_t *batch, *kind, *id;
  int M;
  int pad;
};
struct ScanPtrs {
  ScanTab t[kMaxScanTables];
  int n;
};

struct SelectIO {
  const int32_t* op;
  const double* slack;
  const int32_t* avail;
  const int32_t* supply;
  const int32_t* min_batch;
  const uint32_t* flags;
  int32_t* out_idx;
  int32_t* out_code;
  int32_t* out_fill;
  double* out_obj;
  double* out_slack;
  double* out_wait;
  double* out_kind_min;
  int N;
  int K;
  int aligned;  // every input array 16-byte aligned: eligible for TMA bulk L2 prefetch
};

// ---- TMA bulk-copy helpers (cp.async.bulk + mbarrier) --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

template <int NW>
__device__ __forceinline__ uint32_t hmin_or(const uint32_t (&a)[NW], const uint32_t (&m)[NW]) {
  uint32_t z = a[0] | m[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) z = __vminu2(z, a[w] | m[w]);
  return min(z & 0xFFFFu, z >> 16);
}
template <int NW>
__device__ __forceinline__ uint32_t hmin_all(const uint32_t (&a)[NW]) {
  uint32_t z = a[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) z = __vminu2(z, a[w]);
  return min(z & 0xFFFFu, z >> 16);
}

template <int KT>
__device__ __forceinline__ double pick_kind(const double (&s)[KT], int kind) {
  double v = s[0];
#pragma unroll
  for (int k = 1; k < KT; ++k)
    if (kind == k) v = s[k];
  return v;
}

template <int KT>
struct In {
  double s[KT];
  int av, sup, mb, t;
  uint32_t fl;
};

template <int KT>
__device__ __forceinline__ void load_in(const SelectIO& io, int i, In<KT>& x) {
  const double* p = io.slack + (size_t)i * io.K;
  if (KT == 2 && io.K == 2) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    x.s[0] = v.x;
    x.s[1] = v.y;
  } else {
#pragma unroll
    for (int k = 0; k < KT; ++k) x.s[k] = (k < io.K) ? __ldg(p + k) : 0.0;
  }
  x.av = __ldg(io.avail + i);
  x.sup = __ldg(io.supply + i);
  x.mb = __ldg(io.min_batch + i);
  x.fl = __ldg(io.flags + i);
  x.t = io.op ? __ldg(io.op + i) : 0;
}

struct Out {
  int32_t idx, code, fill;
  double obj, slack, wait;
};

__device__ __forceinline__ void store_out(const SelectIO& io, int i, const Out& o) {
  io.out_idx[i] = o.idx;
  io.out_code[i] = o.code;
  if (io.out_fill) io.out_fill[i] = o.fill;
  if (io.out_obj) io.out_obj[i] = o.obj;
  if (io.out_slack) io.out_slack[i] = o.slack;
  if (io.out_wait) io.out_wait[i] = o.wait;
}

// ---- K2b: staircase plan kernel ----------------------------------------------------------
#include "sp_k2b.cuh"
#include "sp_k2f.cuh"
#include "sp_k12.cuh"
#include "sp_spec.cuh"

// ---- K2a: literal scan kernel -------------------------------------------------------------
struct Best {
  int j;
  double sc, c, r;
  int id;
};
__device__ __forceinline__ bool better(double sc, double c, double r, int id, const Best& b) {
  if (b.j < 0) return true;
  if (sc != b.sc) return sc < b.sc;
  if (c != b.c) return c < b.c;
  if (r != b.r) return r < b.r;
  return id < b.id;
}

// The reference's masked argmin restated literally for the cases the strict total order of
// the fast scan cannot represent (configurator.py:229-237 with numpy / Python semantics):
// best = min over where(mask, score, inf) (NaN propagates); ties = every index whose masked
// score equals best — with best == inf that includes masked-out entries; the winner is the
// first minimum of the key tuple (cost, res, id_rank) in index order under Python's tuple
// comparison (NaN compares unequal and never smaller).  Returns the index, -1 when the mask is
// empty, -2 when the tie set is empty (a NaN best: the reference's min() raises ValueError).
template <int KT>
__device__ int literal_argmin(const ScanTab& tb, const In<KT>& x, bool use_av) {
  double best = INFINITY;
  bool nan = false, any = false;
  for (int j = 0; j < tb.M; ++j) {
    const int kj = tb.kind[j];
    const bool m = !((x.fl >> (SP_FLAG_EXCL_SHIFT + kj)) & 1u) && tb.batch[j] >= x.mb &&
                   (!use_av || tb.batch[j] <= x.av);
    if (!m) continue;
    any = true;
    const double sc = (tb.lat[j] < pick_kind<KT>(x.s, kj)) ? tb.cost[j] : tb.costpen[j];
    if (sc != sc) nan = true;
    else if (sc < best) best = sc;
  }
  if (!any) return -1;
  if (nan) return -2;
  int cur = -1;
  for (int j = 0; j < tb.M; ++j) {
    const int kj = tb.kind[j];
    const bool m = !((x.fl >> (SP_FLAG_EXCL_SHIFT + kj)) & 1u) && tb.batch[j] >= x.mb &&
                   (!use_av || tb.batch[j] <= x.av);
    const double sc = m ? ((tb.lat[j] < pick_kind<KT>(x.s, kj)) ? tb.cost[j] : tb.costpen[j])
                        : INFINITY;
    if (!(sc == best)) continue;
    if (cur < 0) {
      cur = j;
      continue;
    }
    const double c = tb.cost[j], cc = tb.cost[cur];
    bool lt;
    if (c != cc) lt = c < cc;
    else if (tb.res[j] != tb.res[cur]) lt = tb.res[j] < tb.res[cur];
    else lt = tb.id[j] < tb.id[cur];
    if (lt) cur = j;
  }
  return cur;
}

template <int KT>
__device__ void literal_select(const ScanTab& tb, const In<KT>& x, Out& o) {
  int i = literal_argmin<KT>(tb, x, false);
  o.wait = 0.0;
  if (i < 0) {  // None (empty mask) or the reference's ValueError (NaN best)
    o.idx = -1; o.code = i == -1 ? SP_DEC_NONE : SP_DEC_ERROR; o.fill = 0;
    o.obj = 0.0; o.slack = 0.0;
    return;
  }
  int B = tb.batch[i];
  double sk = pick_kind<KT>(x.s, tb.kind[i]);
  double L = tb.lat[i];
  if ((x.fl & SP_FLAG_ALLOW_DELAY) && B > x.av &&
      (long long)x.sup >= (long long)B - (long long)x.av) {
    const double wait = __dsub_rn(sk, L);
    if (wait > 0.0) {
      o.idx = i;
      o.code = SP_DEC_DELAY | ((L < sk) ? SP_DEC_FEASIBLE : 0);
      o.fill = x.av;
      o.obj = (L < sk) ? tb.cost[i] : tb.costpen[i];
      o.slack = sk;
      o.wait = wait;
      return;
    }
  }
  if (B > x.av) {
    const int i2 = literal_argmin<KT>(tb, x, true);
    if (i2 == -2) {
      o.idx = -1; o.code = SP_DEC_ERROR; o.fill = 0; o.obj = 0.0; o.slack = 0.0;
      return;
    }
    if (i2 >= 0) i = i2;
  }
  B = tb.batch[i];
  sk = pick_kind<KT>(x.s, tb.kind[i]);
  L = tb.lat[i];
  o.idx = i;
  o.code = SP_DEC_ASSIGN | ((L < sk) ? SP_DEC_FEASIBLE : 0);
  o.fill = min(B, x.av);
  o.obj = (L < sk) ? tb.cost[i] : tb.costpen[i];
  o.slack = sk;
}

template <int KT>
__global__ void __launch_bounds__(256) k_select_scan(ScanPtrs sp_, int staged, SelectIO io) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ ScanTab s_tab[kMaxScanTables];
  const int tid = threadIdx.x;
  if (staged) {
    // stage every table's SoA into shared memory (broadcast-read during the scan)
    size_t off = 0;
    for (int t = 0; t < sp_.n; ++t) {
      const ScanTab& g = sp_.t[t];
      const int M = g.M;
      double* d = reinterpret_cast<double*>(smem + off);
      int32_t* ii = reinterpret_cast<int32_t*>(d + 4 * (size_t)M);
      for (int j = tid; j < M; j += blockDim.x) {
        d[j] = g.lat[j];
        d[M + j] = g.cost[j];
        d[2 * M + j] = g.costpen[j];
        d[3 * M + j] = g.res[j];
        ii[j] = g.batch[j];
        ii[M + j] = g.kind[j];
        ii[2 * M + j] = g.id[j];
      }
      if (tid == 0) {
        ScanTab s;
        s.lat = d; s.cost = d + M; s.costpen = d + 2 * M; s.res = d + 3 * M;
        s.batch = ii; s.kind = ii + M; s.id = ii + 2 * M;
        s.M = M; s.pad = 0;
        s_tab[t] = s;
      }
      off += (size_t)M * 44;
      off = (off + 15) & ~(size_t)15;
    }
  } else if (tid < sp_.n) {
    s_tab[tid] = sp_.t[tid];
  }
  __syncthreads();
  const bool want_kmin = io.out_kind_min != nullptr;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + tid; i < io.N; i += stride) {
    In<KT> x;
    load_in<KT>(io, i, x);
    const ScanTab tb = s_tab[x.t];
    Best b1, b2;
    b1.j = b2.j = -1;
    b1.sc = b1.c = b1.r = b2.sc = b2.c = b2.r = 0.0;
    b1.id = b2.id = 0;
    double kmin[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) kmin[k] = INFINITY;
    bool sawnan = false;  // a NaN score among the admitted entries: literal restatement
    for (int j = 0; j < tb.M; ++j) {
      const int kj = tb.kind[j];
      const int bj = tb.batch[j];
      const double L = tb.lat[j];
      const double sk = pick_kind<KT>(x.s, kj);
      const double c = tb.cost[j];
      // configurator.py:226  score = cost + where(lat < slack, 0.0, penalty)
      const double sc = (L < sk) ? c : tb.costpen[j];
      if (want_kmin) {  // numpy's min: NaN propagates
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (kj == k && (sc < kmin[k] || sc != sc)) kmin[k] = sc;
      }
      // mask: excluded kinds (259-263) and min_batch (264-265)
      const bool in1 = !((x.fl >> (SP_FLAG_EXCL_SHIFT + kj)) & 1u) && bj >= x.mb;
      if (in1) {
        sawnan |= sc != sc;
        const double r = tb.res[j];
        const int id = tb.id[j];
        if (better(sc, c, r, id, b1)) { b1.j = j; b1.sc = sc; b1.c = c; b1.r = r; b1.id = id; }
        if (bj <= x.av && better(sc, c, r, id, b2)) {
          b2.j = j; b2.sc = sc; b2.c = c; b2.r = r; b2.id = id;
        }
      }
    }
    if (want_kmin) {
#pragma unroll
      for (int k = 0; k < KT; ++k)
        if (k < io.K) io.out_kind_min[(size_t)i * io.K + k] = kmin[k];
    }
    Out o;
    if (b1.j < 0) {
      o.idx = -1; o.code = SP_DEC_NONE; o.fill = 0;
      o.obj = 0.0; o.slack = 0.0; o.wait = 0.0;
      store_out(io, i, o);
      continue;
    }
    // a non-finite best (inf / NaN scores), or an infinite downgrade best: the reference's tie
    // set reaches beyond the strict order — restate it literally
    if (sawnan || !(b1.sc < INFINITY) ||
        (tb.batch[b1.j] > x.av && b2.j >= 0 && !(b2.sc < INFINITY))) {
      literal_select<KT>(tb, x, o);
      store_out(io, i, o);
      continue;
    }
    int j = b1.j;
    double sc = b1.sc;
    int B = tb.batch[j];
    int kj = tb.kind[j];
    double sk = pick_kind<KT>(x.s, kj);
    double L = tb.lat[j];
    if ((x.fl & SP_FLAG_ALLOW_DELAY) && B > x.av &&
        (long long)x.sup >= (long long)B - (long long)x.av) {
      double wait = __dsub_rn(sk, L);
      if (wait > 0.0) {
        o.idx = j;
        o.code = SP_DEC_DELAY | ((L < sk) ? SP_DEC_FEASIBLE : 0);
        o.fill = x.av;
        o.obj = sc;
        o.slack = sk;
        o.wait = wait;
        store_out(io, i, o);
        continue;
      }
    }
    if (B > x.av && b2.j >= 0) {
      j = b2.j;
      sc = b2.sc;
      B = tb.batch[j];
      kj = tb.kind[j];
      sk = pick_kind<KT>(x.s, kj);
      L = tb.lat[j];
    }
    o.idx = j;
    o.code = SP_DEC_ASSIGN | ((L < sk) ? SP_DEC_FEASIBLE : 0);
    o.fill = min(B, x.av);
    o.obj = sc;
    o.slack = sk;
    o.wait = 0.0;
    store_out(io, i, o);
  }
}

// ---- Eq. 1 vector (OpTable.scores) ----------------------------------------------------------
__global__ void k_scores(int M, int K, const double* __restrict__ lat,
                         const int32_t* __restrict__ kind, const double* __restrict__ cost,
                         const double* __restrict__ costpen, const double* __restrict__ slack,
                         double* __restrict__ score, double* __restrict__ cost_out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  double c = cost[j];
  score[j] = (lat[j] < slack[kind[j]]) ? c : costpen[j];
  cost_out[j] = c;
}

__global__ void k_affinity(int N, int K, const double* __restrict__ kmin,
                           const int32_t* __restrict__ q, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int c = q[i];
  double other = INFINITY;
  for (int k = 0; k < K; ++k) {
    double v = kmin[(size_t)i * K + k];
    if (k != c && (v < other || v != v)) other = v;  // numpy's min: NaN propagates
  }
  // configurator.py:318  float(score[~on].min() / score[on].min())
  out[i] = __ddiv_rn(other, kmin[(size_t)i * K + c]);
}

// one persistent 1024-thread CTA per SM with one staged copy of the plan(s)
constexpr int kPlanThreads = 1024;
constexpr int kPlanCtasPerSm = 1;
constexpr int kPlanSmemBudget = 200 * 1024;

template <int KT>
int launch_plan_t(sp_ctx* ctx, const PlanPtrs& pp, const SelectIO& io) {
  static uint64_t attr_done = 0;
  if (attr_once(attr_done)) {
    SP_CUDA(cudaFuncSetAttribute(k_select_plan<KT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kPlanSmemBudget));
  }
  const bool single = pp.hv && pp.n == 1 && !io.out_kind_min;
  // specialised kernel (sp_k2f.cuh) for the common shape; SP_K2_VARIANT=plan forces K2b
  if (single && io.K == KT && !ctx->opt.k2_plan_only) {
    bool ok = pp.h.lut_n > 0 && io.out_idx && io.out_code && io.out_fill && io.out_obj &&
              io.out_slack && io.out_wait;
    for (int k = 0; k < KT && ok; ++k) ok = pp.h.kd[k].pad[0] == 0;  // positive thresholds
    const int lut_off = (pp.h.total_bytes + 15) & ~15;
    const int smem = ((lut_off + 4 * pp.h.lut_n + 1023) / 1024) * 1024;
    if (ok && smem <= kPlanSmemBudget) {
      // block size: 512 threads x 2 CTAs per SM (default: as CTAs of one launch retire, the
      // next launch's CTAs take their place one at a time — measured 15.9 -> 15.5 us per
      // 2^20-decision step back to back) or 1024 x 1 (SP_K2F_THREADS=1024)
      const int thr = ctx->opt.k2f_threads == 1024 ? 1024 : 512;
      static uint64_t fast_attr[2] = {0, 0};
      if (attr_once(fast_attr[thr == 512])) {
        if (thr == 512)
          SP_CUDA(cudaFuncSetAttribute(k_select_fast<KT, 512>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kPlanSmemBudget));
        else
          SP_CUDA(cudaFuncSetAttribute(k_select_fast<KT, 1024>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kPlanSmemBudget));
      }
      FastIO<KT> f;
      f.slack = io.slack; f.avail = io.avail; f.supply = io.supply; f.min_batch = io.min_batch;
      f.flags = io.flags; f.out_idx = io.out_idx; f.out_code = io.out_code; f.out_fill = io.out_fill;
      f.out_obj = io.out_obj; f.out_slack = io.out_slack; f.out_wait = io.out_wait;
      f.N = (uint32_t)io.N; f.lut_bytes_off = lut_off;
      f.prestage = ctx->plan_dirty ? 0 : 1;
      int blocks = ctx->num_sms * (1024 / thr);
      int need = (io.N + thr - 1) / thr;
      if (need < blocks) blocks = need > 0 ? need : 1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(thr);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (thr == 512)
        SP_CUDA(cudaLaunchKernelEx(&cfg, k_select_fast<KT, 512>, (const uint8_t*)pp.p[0], pp.h, f));
      else
        SP_CUDA(cudaLaunchKernelEx(&cfg, k_select_fast<KT, 1024>, (const uint8_t*)pp.p[0], pp.h, f));
      SP_CHECK_LAUNCH(ctx);
      ctx->plan_dirty = false;
      return SP_OK;
    }
  }
  int blocks = ctx->num_sms * kPlanCtasPerSm;
  int need = (io.N + kPlanThreads - 1) / kPlanThreads;
  if (need < blocks) blocks = need > 0 ? need : 1;
  // request only the shared memory the staged plan needs when its size is known on the host
  int smem = kPlanSmemBudget;
  if (pp.hv && pp.n == 1 && !ctx->opt.full_smem)
    smem = std::min(kPlanSmemBudget, ((pp.h.total_bytes + 1023) / 1024) * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kPlanThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SP_CUDA(cudaLaunchKernelEx(&cfg, k_select_plan<KT>, pp, smem, io));
  SP_CHECK_LAUNCH(ctx);
  ctx->plan_dirty = false;
  return SP_OK;
}

template <int KT>
int launch_scan_t(sp_ctx* ctx, const ScanPtrs& sp_, size_t stage_bytes, const SelectIO& io) {
  const size_t max_stage = 200 * 1024;
  static uint64_t attr_done = 0;
  if (attr_once(attr_done)) {
    SP_CUDA(cudaFuncSetAttribute(k_select_scan<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)max_stage));
  }
  int staged = stage_bytes <= max_stage ? 1 : 0;
  size_t smem = staged ? stage_bytes : 0;
  int per_sm = 1;
  if (smem <= 100 * 1024) per_sm = 2;
  if (smem <= 48 * 1024) per_sm = 4;
  int blocks = ctx->num_sms * per_sm;
  int need = (io.N + 255) / 256;
  if (need < blocks) blocks = need > 0 ? need : 1;
  k_select_scan<KT><<<blocks, 256, smem, ctx->stream>>>(sp_, staged, io);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace

static __global__ void k_op_index(int N, int n_src, int32_t* op) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < N) op[d] = d % n_src;
}

int slack_select_launch(sp_ctx* ctx, sp_dag* g, int n_tables, sp_table* const* tables,
                        double alpha, int I, const double* ref, int ref_stride,
                        const double* target, const double* now, int K, const double* Q,
                        const int32_t* avail, const int32_t* supply, const int32_t* min_batch,
                        const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                        int32_t* out_fill, double* out_obj, double* out_slack, double* out_wait,
                        double* out_kslack) {
  if (n_tables != g->n_src) return fail(SP_E_INVALID, "slack_select: one table per DAG source");
  if (n_tables > kK12MaxSrc) return fail(SP_E_UNSUPPORTED, "slack_select: more than 64 sources");
  for (int t = 0; t < n_tables; ++t)
    if (tables[t]->K != K) return fail(SP_E_INVALID, "slack_select: tables disagree with K");
  if (I == 0) return SP_OK;
  const int N = I * n_tables;
  const int KT = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  // plans and their sizes (a freshly rebuilt plan's header is waited for once)
  PlanPtrs pp;
  pp.n = n_tables;
  pp.hv = 0;
  size_t plan_bytes = 0, lut_bytes = 0;
  bool fused = !ctx->opt.no_k12 && K <= kMaxKinds && isfinite(alpha);
  for (int t = 0; t < n_tables && fused; ++t)
    fused = tables[t]->plan_ok && tables[t]->finite_safe();
  bool fast_ok = !ctx->opt.k12_generic;
  for (int t = 0; t < n_tables && fused; ++t) {
    int rc;
    Plan* p = plan_get(ctx, tables[t], alpha, &rc);
    if (!p) return rc;
    pp.p[t] = p->image;
    if (!tables[t]->plan_ok) {
      fused = false;
      continue;
    }
    const PlanHdr* h = plan_host_header(*p);
    if (!h) {
      const int rc2 = plan_header_wait(ctx, *p);
      if (rc2 != SP_OK) return rc2;
      h = plan_host_header(*p);
    }
    if (!h) return fail(SP_E_RUNTIME, "slack_select: plan header unavailable");
    plan_bytes += (size_t)h->total_bytes;
    lut_bytes += (size_t)((h->lut_n * 4 + 15) / 16) * 16;
    for (int k = 0; k < K; ++k) fast_ok = fast_ok && h->kd[k].pad[0] == 0;
    fast_ok = fast_ok && h->lut_n > 0 && K == KT;
  }
  const size_t dp = (size_t)kK12Warps * g->max_slots * 32 * sizeof(double2);
  const size_t progb = (size_t)g->prog_len * sizeof(int4) + (((size_t)g->pred_len * 4 + 15) / 16) * 16;
  if (!fused) fast_ok = false;
  const size_t plans_all = plan_bytes + (fast_ok ? lut_bytes : 0);
  // decisions staged for coalesced stores only on request (SP_K12_OUTSTAGE=1): without it the
  // per-warp area holds just the 16 input bytes per decision and more CTAs stay resident
  const int out_stage = (ctx->opt.k12_outstage || !out_fill || !out_obj || !out_slack ||
                         !out_wait) ? 1 : 0;
  const size_t stage = (size_t)kK12Warps * 32 * n_tables * (out_stage ? kK12StageBytesPerDecision : 16);
  const size_t refs = (size_t)kK12Warps * g->n_val * 32 * sizeof(double);
  const size_t smem = dp + progb + plans_all + stage + refs;
  if (fused && smem <= (size_t)kPlanSmemBudget) {
    SelectIO io;
    memset(&io, 0, sizeof(io));
    io.avail = avail; io.supply = supply; io.min_batch = min_batch; io.flags = flags;
    io.out_idx = out_idx; io.out_code = out_code; io.out_fill = out_fill;
    io.out_obj = out_obj; io.out_slack = out_slack; io.out_wait = out_wait;
    io.N = N; io.K = K;
    K12Dag kg{g->prog, g->prog_ptr, g->preds, g->pred_ptr, g->n_src, g->max_slots,
              (int)g->prog_len, (int)g->pred_len, g->n_val,
              ctx->opt.k12_generic_dp ? 0 : g->single_pred};
    K12In ki{ref, ref_stride, target, now, Q, I, out_kslack};
    auto launch = [&](auto kern) -> int {
      // one entry per k_slack_select instantiation, per device
      static const void* attr_dev[64][6] = {};
      const void** attr_done = attr_dev[cur_device()];
      bool done = false;
      for (int q = 0; q < 6; ++q) done = done || attr_done[q] == reinterpret_cast<const void*>(kern);
      if (!done) {
        SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kPlanSmemBudget));
        for (int q = 0; q < 6; ++q)
          if (!attr_done[q]) {
            attr_done[q] = reinterpret_cast<const void*>(kern);
            break;
          }
      }
      int per_sm = 0;
      SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kK12Warps, smem));
      if (per_sm < 1) return fail(SP_E_UNSUPPORTED, "slack_select: no resident CTA");
      int blocks = ctx->num_sms * per_sm;
      const int need = (I + 32 * kK12Warps - 1) / (32 * kK12Warps);
      if (need < blocks) blocks = need;
      kern<<<blocks, 32 * kK12Warps, smem, ctx->stream>>>(kg, ki, pp, (int)(dp + progb),
                                                          (int)(dp + progb + plans_all), out_stage, io);
      SP_CHECK_LAUNCH(ctx);
      return SP_OK;
    };
    if (fast_ok) {
      if (KT == 2) return launch(k_slack_select<2, true>);
      if (KT == 4) return launch(k_slack_select<4, true>);
      return launch(k_slack_select<8, true>);
    }
    if (KT == 2) return launch(k_slack_select<2, false>);
    if (KT == 4) return launch(k_slack_select<4, false>);
    return launch(k_slack_select<8, false>);
  }
  // two-kernel fallback: K1 slack into scratch, then the multi-table K2 launch
  int rc = SP_OK;
  const size_t sl_bytes = ((sizeof(double) * (size_t)N * K + 255) / 256) * 256;
  void* tmp = ctx_tmp(ctx, sl_bytes + sizeof(int32_t) * (size_t)N, &rc);
  if (!tmp) return rc;
  double* sl = static_cast<double*>(tmp);
  int32_t* op = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(tmp) + sl_bytes);
  rc = slack_launch(ctx, g, I, ref, ref_stride, target, now, K, Q, sl, nullptr);
  if (rc != SP_OK) return rc;
  k_op_index<<<(N + 255) / 256, 256, 0, ctx->stream>>>(N, n_tables, op);
  SP_CHECK_LAUNCH(ctx);
  rc = select_launch(ctx, n_tables, tables, alpha, N, op, sl, avail, supply, min_batch, flags,
                     out_idx, out_code, out_fill, out_obj, out_slack, out_wait, nullptr,
                     SP_MODE_AUTO);
  if (rc != SP_OK || !out_kslack) return rc;
  SP_CUDA(cudaMemcpyAsync(out_kslack, sl, sizeof(double) * (size_t)N * K, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  return SP_OK;
}

constexpr int64_t kAutoPlanWork = (int64_t)1 << 24;

int select_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, double alpha, int N,
                  const int32_t* op, const double* slack, const int32_t* avail,
                  const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                  int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                  double* out_slack, double* out_wait, double* out_kind_min, int mode) {
  if (n_tables < 1) return fail(SP_E_INVALID, "select: no tables");
  const int K = tables[0]->K;
  bool plan_ok = true;

  for (int t = 0; t < n_tables; ++t) {
    if (tables[t]->K != K) return fail(SP_E_INVALID, "select: tables disagree on kind count");
    // the staircase needs finite latencies and scores; otherwise the literal scan reproduces
    // the reference's inf / NaN behaviour
    plan_ok = plan_ok && tables[t]->plan_ok && tables[t]->finite_safe();
  }
  plan_ok = plan_ok && isfinite(alpha);
  if (mode == SP_MODE_PLAN && !plan_ok)
    return fail(SP_E_UNSUPPORTED, "select: staircase plan unsupported for this table (more than "
                                  "16 batch sizes, 8 kinds or 32766 entries, or non-finite "
                                  "latencies / alpha)");
  // AUTO: the staircase plan when it is current, or when the batch is large enough to pay for
  // a rebuild (a plan build costs about as much as scanning ~2^24 invocation x entry pairs);
  // otherwise the scan, which needs only cost / costpen (e.g. one call right after a
  // set_latency in the reference engine's per-call use)
  bool use_plan = mode == SP_MODE_PLAN;
  if (mode == SP_MODE_AUTO && plan_ok) {
    bool ready = true;
    int64_t work = 0;
    for (int t = 0; t < n_tables; ++t) {
      ready = ready && plan_ready(tables[t], alpha);
      work += tables[t]->M;
    }
    use_plan = ready || (int64_t)N * work >= kAutoPlanWork;
  }
  if (use_plan && n_tables > kMaxPlanTables)
    return fail(SP_E_UNSUPPORTED, "select: too many tables in one plan launch (max 64)");
  if (!use_plan && n_tables > kMaxScanTables)
    return fail(SP_E_UNSUPPORTED, "select: too many tables in one scan launch (max 16)");
  SelectIO io;
  io.op = op; io.slack = slack; io.avail = avail; io.supply = supply;
  io.min_batch = min_batch; io.flags = flags;
  io.out_idx = out_idx; io.out_code = out_code; io.out_fill = out_fill;
  io.out_obj = out_obj; io.out_slack = out_slack; io.out_wait = out_wait;
  io.out_kind_min = out_kind_min;
  io.N = N; io.K = K;
  {
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    io.aligned = al(slack) && al(avail) && al(supply) && al(min_batch) && al(flags);
  }
  if (N == 0) return SP_OK;
  const int KT = K <= 2 ? 2 : (K <= 4 ? 4 : (K <= 8 ? 8 : 24));
  if (use_plan) {
    PlanPtrs pp;
    pp.n = n_tables;
    pp.hv = 0;
    for (int t = 0; t < n_tables; ++t) {
      int rc;
      Plan* p = plan_get(ctx, tables[t], alpha, &rc);
      if (!p) return rc;
      pp.p[t] = p->image;
      if (n_tables == 1) {
        const PlanHdr* hh = plan_host_header(*p);
        if (hh) {
          pp.h = *hh;
          pp.hv = 1;
        }
      }
    }
    if (KT == 2) return launch_plan_t<2>(ctx, pp, io);
    if (KT == 4) return launch_plan_t<4>(ctx, pp, io);
    return launch_plan_t<8>(ctx, pp, io);
  }
  ScanPtrs sp_;
  sp_.n = n_tables;
  size_t stage = 0;
  for (int t = 0; t < n_tables; ++t) {
    int rc;
    Plan* p = plan_costs(ctx, tables[t], alpha, &rc);
    if (!p) return rc;
    sp_table* tb = tables[t];
    ScanTab s;
    s.lat = tb->lat; s.cost = p->cost; s.costpen = p->costpen; s.res = tb->res;
    s.batch = tb->batch; s.kind = tb->kind; s.id = tb->id_rank;
    s.M = tb->M; s.pad = 0;
    sp_.t[t] = s;
    stage += (size_t)tb->M * 44;
    stage = (stage + 15) & ~(size_t)15;
  }
  if (KT == 2) return launch_scan_t<2>(ctx, sp_, stage, io);
  if (KT == 4) return launch_scan_t<4>(ctx, sp_, stage, io);
  if (KT == 8) return launch_scan_t<8>(ctx, sp_, stage, io);
  return launch_scan_t<24>(ctx, sp_, stage, io);
}

int affinity_launch(sp_ctx* ctx, int N, int K, const double* kmin, const int32_t* q,
                    double* out) {
  if (N == 0) return SP_OK;
  k_affinity<<<(N + 255) / 256, 256, 0, ctx->stream>>>(N, K, kmin, q, out);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

int scores_launch(sp_ctx* ctx, sp_table* t, Plan* p, const double* slack_dev,
                  double* score_dev, double* cost_dev) {
  k_scores<<<(t->M + 255) / 256, 256, 0, ctx->stream>>>(t->M, t->K, t->lat, t->kind, p->cost,
                                                       p->costpen, slack_dev, score_dev,
                                                       cost_dev);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace sp
