// sp_select.cu — K2: batched OpTable.select (configurator.py:239-300) on sm_100a.
//
// Two kernels, bit-identical to each other and to the reference:
//   k_select_plan  (K2b, the product path)  persistent CTAs stage the per-table staircase
//                  plans into shared memory with one TMA bulk copy (cp.async.bulk +
//                  mbarrier), then every thread decides one invocation per iteration:
//                  per kind one branchless binary search over the staircase thresholds,
//                  one 32/64-byte row load, half-word SIMD minima over the admitted
//                  batch lanes, and at most four candidate-record loads.
//   k_select_scan  (K2a, literal restatement)  every thread scans all M entries of its
//                  table (staged in shared memory, broadcast reads) and keeps the
//                  lexicographic (score, cost, res, id_rank) minima — exactly the
//                  masked-argmin-with-ties of configurator.py:229-237.  General (any
//                  number of batch sizes), O(M) per decision.
// Both then apply the safe-delayed-batching rule and the downgrade argmin
// (configurator.py:271-300).
#include <math.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kMaxPlanTables = 64;
constexpr int kMaxScanTables = 16;

struct PlanPtrs {
  const uint8_t* p[kMaxPlanTables];
  int n;
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

__device__ __forceinline__ uint32_t hmin4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  uint32_t z = __vminu2(__vminu2(a, b), __vminu2(c, d));
  return min(z & 0xFFFFu, z >> 16);
}
__device__ __forceinline__ uint32_t hmin_words(const uint32_t* w, int n) {
  uint32_t z = w[0];
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (i < n) z = __vminu2(z, w[i]);
  return min(z & 0xFFFFu, z >> 16);
}

__device__ __forceinline__ void ld_rec(const CandRec* p, CandRec& r) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = q[0], b = q[1];
  r.score = __hiloint2double((int)a.y, (int)a.x);
  r.lat = __hiloint2double((int)a.w, (int)a.z);
  r.r1 = b.x;
  r.idx = (int32_t)b.y;
  r.batch = (int32_t)b.z;
  r.kind = (int32_t)b.w;
}

// (score, r1) lexicographic resolution between the best feasible (CP) and best infeasible
// (CS) candidate: r1 carries the reference's (cost, res, id_rank) tie order.
__device__ __forceinline__ bool resolve(const uint8_t* base, const PlanHdr* h, uint32_t f,
                                        uint32_t g, CandRec& out) {
  const CandRec* CP = reinterpret_cast<const CandRec*>(base + h->cp_off);
  const CandRec* CS = reinterpret_cast<const CandRec*>(base + h->cs_off);
  if (f == kNone16) {
    ld_rec(CS + g, out);
    return false;
  }
  if (g == kNone16) {
    ld_rec(CP + f, out);
    return true;
  }
  CandRec a, b;
  ld_rec(CP + f, a);
  ld_rec(CS + g, b);
  if (a.score < b.score || (a.score == b.score && a.r1 < b.r1)) {
    out = a;
    return true;
  }
  out = b;
  return false;
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
__device__ __forceinline__ void load_slack(const SelectIO& io, int i, double (&s)[KT]) {
  const double* p = io.slack + (size_t)i * io.K;
  if (KT == 2 && io.K == 2) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    s[0] = v.x;
    s[1] = v.y;
    return;
  }
#pragma unroll
  for (int k = 0; k < KT; ++k) s[k] = (k < io.K) ? __ldg(p + k) : 0.0;
}

// Writes the decision for invocation i given the resolved overall argmin (rec, feas) and
// the downgrade candidate supplier.
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
template <int KT, int WW>
__device__ __forceinline__ void decide_plan(const uint8_t* base, const SelectIO& io, int i,
                                            bool want_kmin) {
  constexpr int NW = WW / 2;  // 32-bit words per half-row
  const PlanHdr* h = reinterpret_cast<const PlanHdr*>(base);
  double s[KT];
  load_slack<KT>(io, i, s);
  const int av = __ldg(io.avail + i);
  const int sup = __ldg(io.supply + i);
  const int mb = __ldg(io.min_batch + i);
  const uint32_t fl = __ldg(io.flags + i);

  // batch lanes admitted by min_batch (configurator.py:264-265) and available (288)
  uint32_t lo = 0, cntle = 0;
#pragma unroll
  for (int b = 0; b < WW; ++b) {
    int bv = h->batch_vals[b];
    lo += (bv < mb);
    cntle += (bv <= av);
  }
  const uint32_t out1 = (1u << lo) - 1u;                // lanes below min_batch
  const uint32_t out2 = out1 | ~((1u << cntle) - 1u);   // ... or above available
  uint32_t m1[NW], m2[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    m1[w] = (((out1 >> (2 * w)) & 1u) ? 0xFFFFu : 0u) |
            (((out1 >> (2 * w + 1)) & 1u) ? 0xFFFF0000u : 0u);
    m2[w] = (((out2 >> (2 * w)) & 1u) ? 0xFFFFu : 0u) |
            (((out2 >> (2 * w + 1)) & 1u) ? 0xFFFF0000u : 0u);
  }
  uint32_t aF1[NW], aG1[NW], aF2[NW], aG2[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) aF1[w] = aG1[w] = aF2[w] = aG2[w] = 0xFFFFFFFFu;

#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k >= io.K) break;
    const int R = h->sec_rows[k];
    const bool ex = (fl >> (SP_FLAG_EXCL_SHIFT + k)) & 1u;
    double kmin = INFINITY;
    if (R > 0 && (!ex || want_kmin)) {
      const double* thr = reinterpret_cast<const double*>(base + h->sec_off[k]);
      const double sk = s[k];
      int r = 0, n = R;
      while (n > 1) {
        int half = n >> 1;
        r = (thr[r + half] < sk) ? r + half : r;
        n -= half;
      }
      const uint4* row =
          reinterpret_cast<const uint4*>(base + h->sec_rows_off[k] + (size_t)r * (4 * WW));
      uint32_t P[NW], S[NW];
#pragma unroll
      for (int q = 0; q < NW / 4; ++q) {
        uint4 a = row[q];
        uint4 b = row[NW / 4 + q];
        P[4 * q + 0] = a.x; P[4 * q + 1] = a.y; P[4 * q + 2] = a.z; P[4 * q + 3] = a.w;
        S[4 * q + 0] = b.x; S[4 * q + 1] = b.y; S[4 * q + 2] = b.z; S[4 * q + 3] = b.w;
      }
      if (!ex) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          aF1[w] = __vminu2(aF1[w], P[w] | m1[w]);
          aG1[w] = __vminu2(aG1[w], S[w] | m1[w]);
          aF2[w] = __vminu2(aF2[w], P[w] | m2[w]);
          aG2[w] = __vminu2(aG2[w], S[w] | m2[w]);
        }
      }
      if (want_kmin) {
        uint32_t fk = hmin_words(P, NW), gk = hmin_words(S, NW);
        if (fk != kNone16 || gk != kNone16) {
          CandRec c;
          resolve(base, h, fk, gk, c);
          kmin = c.score;
        }
      }
    }
    if (want_kmin) io.out_kind_min[(size_t)i * io.K + k] = kmin;
  }

  const uint32_t f1 = hmin_words(aF1, NW), g1 = hmin_words(aG1, NW);
  Out o;
  if (f1 == kNone16 && g1 == kNone16) {  // configurator.py:266-267
    o.idx = -1; o.code = SP_DEC_NONE; o.fill = 0;
    o.obj = 0.0; o.slack = 0.0; o.wait = 0.0;
    store_out(io, i, o);
    return;
  }
  CandRec rec;
  bool feas = resolve(base, h, f1, g1, rec);
  double sk = pick_kind<KT>(s, rec.kind);
  // safe delayed batching (configurator.py:271-286)
  if ((fl & SP_FLAG_ALLOW_DELAY) && rec.batch > av &&
      (long long)sup >= (long long)rec.batch - (long long)av) {
    double wait = __dsub_rn(sk, rec.lat);
    if (wait > 0.0) {
      o.idx = rec.idx;
      o.code = SP_DEC_DELAY | (feas ? SP_DEC_FEASIBLE : 0);
      o.fill = av;
      o.obj = rec.score;
      o.slack = sk;
      o.wait = wait;
      store_out(io, i, o);
      return;
    }
  }
  // downgrade to a batch size that fits what is available (configurator.py:287-291)
  if (rec.batch > av) {
    const uint32_t f2 = hmin_words(aF2, NW), g2 = hmin_words(aG2, NW);
    if (f2 != kNone16 || g2 != kNone16) {
      feas = resolve(base, h, f2, g2, rec);
      sk = pick_kind<KT>(s, rec.kind);
    }
  }
  o.idx = rec.idx;
  o.code = SP_DEC_ASSIGN | (feas ? SP_DEC_FEASIBLE : 0);
  o.fill = min(rec.batch, av);
  o.obj = rec.score;
  o.slack = sk;
  o.wait = 0.0;
  store_out(io, i, o);
}

template <int KT, int WW>
__global__ void __launch_bounds__(512, 2) k_select_plan(PlanPtrs pp, int smem_budget, SelectIO io) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ const uint8_t* s_base[kMaxPlanTables];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_fit;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int off = 0;
    int fit = 1;
    for (int t = 0; t < pp.n; ++t) {
      int bytes = reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes;
      if (off + bytes > smem_budget) fit = 0;
      off += bytes;
    }
    s_fit = fit;
    if (fit) {
      mbar_init(&s_bar, 1);
      mbar_expect_tx(&s_bar, (uint32_t)off);
      off = 0;
      for (int t = 0; t < pp.n; ++t) {
        int bytes = reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes;
        bulk_g2s(smem + off, pp.p[t], (uint32_t)bytes, &s_bar);
        s_base[t] = smem + off;
        off += bytes;
      }
    } else {
      for (int t = 0; t < pp.n; ++t) s_base[t] = pp.p[t];
    }
  }
  __syncthreads();
  if (s_fit) mbar_wait(&s_bar, 0);
  const bool want_kmin = io.out_kind_min != nullptr;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + tid; i < io.N; i += stride) {
    int t = io.op ? __ldg(io.op + i) : 0;
    decide_plan<KT, WW>(s_base[t], io, i, want_kmin);
  }
}

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
    const int t = io.op ? __ldg(io.op + i) : 0;
    const ScanTab tb = s_tab[t];
    double s[KT];
    load_slack<KT>(io, i, s);
    const int av = __ldg(io.avail + i);
    const int sup = __ldg(io.supply + i);
    const int mb = __ldg(io.min_batch + i);
    const uint32_t fl = __ldg(io.flags + i);
    Best b1, b2;
    b1.j = b2.j = -1;
    b1.sc = b1.c = b1.r = b2.sc = b2.c = b2.r = 0.0;
    b1.id = b2.id = 0;
    double kmin[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) kmin[k] = INFINITY;
    for (int j = 0; j < tb.M; ++j) {
      const int kj = tb.kind[j];
      const int bj = tb.batch[j];
      const double L = tb.lat[j];
      const double sk = pick_kind<KT>(s, kj);
      const double c = tb.cost[j];
      // configurator.py:226  score = cost + where(lat < slack, 0.0, penalty)
      const double sc = (L < sk) ? c : tb.costpen[j];
      if (want_kmin) {
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (kj == k && sc < kmin[k]) kmin[k] = sc;
      }
      // mask: excluded kinds (259-263) and min_batch (264-265)
      const bool in1 = !((fl >> (SP_FLAG_EXCL_SHIFT + kj)) & 1u) && bj >= mb;
      if (in1) {
        const double r = tb.res[j];
        const int id = tb.id[j];
        if (better(sc, c, r, id, b1)) { b1.j = j; b1.sc = sc; b1.c = c; b1.r = r; b1.id = id; }
        if (bj <= av && better(sc, c, r, id, b2)) {
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
    int j = b1.j;
    double sc = b1.sc;
    int B = tb.batch[j];
    int kj = tb.kind[j];
    double sk = pick_kind<KT>(s, kj);
    double L = tb.lat[j];
    if ((fl & SP_FLAG_ALLOW_DELAY) && B > av && (long long)sup >= (long long)B - (long long)av) {
      double wait = __dsub_rn(sk, L);
      if (wait > 0.0) {
        o.idx = j;
        o.code = SP_DEC_DELAY | ((L < sk) ? SP_DEC_FEASIBLE : 0);
        o.fill = av;
        o.obj = sc;
        o.slack = sk;
        o.wait = wait;
        store_out(io, i, o);
        continue;
      }
    }
    if (B > av && b2.j >= 0) {
      j = b2.j;
      sc = b2.sc;
      B = tb.batch[j];
      kj = tb.kind[j];
      sk = pick_kind<KT>(s, kj);
      L = tb.lat[j];
    }
    o.idx = j;
    o.code = SP_DEC_ASSIGN | ((L < sk) ? SP_DEC_FEASIBLE : 0);
    o.fill = min(B, av);
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
    if (k != c && v < other) other = v;
  }
  // configurator.py:318  float(score[~on].min() / score[on].min())
  out[i] = __ddiv_rn(other, kmin[(size_t)i * K + c]);
}

template <int KT, int WW>
int launch_plan_t(sp_ctx* ctx, const PlanPtrs& pp, const SelectIO& io) {
  static bool attr_done[2] = {false, false};
  const int budget = 96 * 1024;
  int dev_slot = 0;
  if (!attr_done[dev_slot]) {
    SP_CUDA(cudaFuncSetAttribute(k_select_plan<KT, WW>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, budget));
    attr_done[dev_slot] = true;
  }
  int blocks = ctx->num_sms * 2;
  int need = (io.N + 511) / 512;
  if (need < blocks) blocks = need > 0 ? need : 1;
  k_select_plan<KT, WW><<<blocks, 512, budget, ctx->stream>>>(pp, budget, io);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

template <int KT>
int launch_scan_t(sp_ctx* ctx, const ScanPtrs& sp_, size_t stage_bytes, const SelectIO& io) {
  const size_t max_stage = 200 * 1024;
  static bool attr_done = false;
  if (!attr_done) {
    SP_CUDA(cudaFuncSetAttribute(k_select_scan<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)max_stage));
    attr_done = true;
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

int select_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, double alpha, int N,
                  const int32_t* op, const double* slack, const int32_t* avail,
                  const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                  int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                  double* out_slack, double* out_wait, double* out_kind_min, int mode) {
  if (n_tables < 1) return fail(SP_E_INVALID, "select: no tables");
  const int K = tables[0]->K;
  bool plan_ok = true;
  int Wmax = 8;
  for (int t = 0; t < n_tables; ++t) {
    if (tables[t]->K != K) return fail(SP_E_INVALID, "select: tables disagree on kind count");
    plan_ok = plan_ok && tables[t]->plan_ok;
    if (tables[t]->nB > 8) Wmax = 16;
  }
  if (mode == SP_MODE_PLAN && !plan_ok)
    return fail(SP_E_UNSUPPORTED, "select: staircase plan unsupported for this table");
  bool use_plan = (mode == SP_MODE_PLAN) || (mode == SP_MODE_AUTO && plan_ok);
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
  if (N == 0) return SP_OK;
  const int KT = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  if (use_plan) {
    PlanPtrs pp;
    pp.n = n_tables;
    int maxW = 8;
    for (int t = 0; t < n_tables; ++t) {
      int rc;
      Plan* p = plan_get(ctx, tables[t], alpha, &rc);
      if (!p) return rc;
      pp.p[t] = p->image;
      if (tables[t]->nB > 8) maxW = 16;
    }
    (void)Wmax;
    if (maxW == 16) {
      // all plans of one launch must share the row width: rebuild narrower ones wide
      for (int t = 0; t < n_tables; ++t)
        if (tables[t]->nB <= 8)
          return fail(SP_E_UNSUPPORTED,
                      "select: mixing tables with <=8 and >8 batch sizes in one launch");
      if (KT == 2) return launch_plan_t<2, 16>(ctx, pp, io);
      if (KT == 4) return launch_plan_t<4, 16>(ctx, pp, io);
      return launch_plan_t<8, 16>(ctx, pp, io);
    }
    if (KT == 2) return launch_plan_t<2, 8>(ctx, pp, io);
    if (KT == 4) return launch_plan_t<4, 8>(ctx, pp, io);
    return launch_plan_t<8, 8>(ctx, pp, io);
  }
  ScanPtrs sp_;
  sp_.n = n_tables;
  size_t stage = 0;
  for (int t = 0; t < n_tables; ++t) {
    int rc;
    Plan* p = plan_get(ctx, tables[t], alpha, &rc);
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
  return launch_scan_t<8>(ctx, sp_, stage, io);
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
