// sp_k2f.cuh — K2f, the specialised single-table staircase decision kernel (included by
// sp_select.cu after sp_k2b.cuh).
//
// Same plan image, same decision sequence and bit-identical results as k_select_plan
// (sp_k2b.cuh), restricted to the shape every batched OpTable.select call over one table
// has: exactly K kinds (compile time), the plan header as a kernel parameter, all six
// decision outputs requested, a batch-value lookup table and positive staircase thresholds.
// What the specialisation buys (ncu, config 2): a branch-free decision body with
//   * one u32 lookup per batch bound: a CTA-private table built while the plan's TMA bulk
//     copy is in flight maps v -> (#batch < v) | (#batch <= v) << 8 | tri_base(#batch < v) << 16,
//     so both staircase-row lane offsets (full admitted range for the argmin and the
//     [min_batch, available] range for the downgrade, configurator.py:264-265, 288) are one add;
//   * the downgrade row minima loaded together with the argmin row minima (same rows,
//     second lane), so the decision has two dependent candidate-record rounds, not three;
//   * 32-bit shared-memory addressing from one uniform base and no per-kind descriptor loads;
//   * no null-output or table-index checks in the loop.
// The per-invocation decision is the reference's OpTable.select (configurator.py:239-300):
// masked tie-broken argmin -> safe delayed batching (271-286) -> downgrade (287-291) -> fill.

template <int K>
struct FastIO {
  const double* slack;  // N x K
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
  uint32_t N;
  int lut_bytes_off;  // byte offset of the CTA lookup table in dynamic shared memory
  int prestage;       // 1: the plan was completed by a kernel an earlier select launch waited
                      // on, so it may be staged before griddepcontrol.wait
};

template <int K>
struct InF {
  double s[K];
  int av, sup, mb;
  uint32_t fl;
};

template <int K>
__device__ __forceinline__ void load_fast(const FastIO<K>& io, uint32_t i, InF<K>& x) {
  if (K == 2) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(io.slack) + i);
    x.s[0] = v.x;
    x.s[1] = v.y;
  } else if (K % 2 == 0) {
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(io.slack + (size_t)i * K) + k / 2);
      x.s[k] = v.x;
      x.s[k + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) x.s[k] = __ldg(io.slack + (size_t)i * K + k);
  }
  x.av = __ldg(io.avail + i);
  x.sup = __ldg(io.supply + i);
  x.mb = __ldg(io.min_batch + i);
  x.fl = __ldg(io.flags + i);
}

// shared-memory reads at a 32-bit shared-window address (non-volatile asm: free to schedule;
// every address derives from `sb`, which is produced after the plan's mbarrier wait)
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

// staircase row of kind k for slack s (positive thresholds): bucket on the IEEE high word,
// two predicated bisection steps (exact for buckets of <= 3 thresholds), rare loop tail
__device__ __forceinline__ int fast_row(uint32_t sm, const KindDesc& d, double s) {
  const int dd = __double2hiint(s) - (int)d.kmin_hi;
  uint32_t b = dd < 0 ? 0u : ((uint32_t)dd >> (d.nb1_shift >> 16));
  b = min(b, d.nb1_shift & 0xFFFFu);
  const uint32_t e = lds_u32(sm + (uint32_t)d.bkt_off + 4u * b);
  const bool pos = s > 0.0;  // s <= 0 or NaN: below every (positive) threshold -> row 0
  int r = pos ? (int)(e & 0xFFFFu) : 0;
  int n = pos ? (int)(e >> 16) : 0;
  const uint32_t thr = (uint32_t)d.thr_off;
#pragma unroll
  for (int step = 0; step < 2; ++step) {
    const int hh = n >> 1;
    const int at = n > 0 ? r + hh + 1 : 0;
    const double t = lds_f64(sm + thr + 8u * (uint32_t)at);
    const bool lt = n > 0 && t < s;
    r = lt ? r + hh + 1 : r;
    n = n > 0 ? (lt ? n - hh - 1 : hh) : 0;
  }
  while (n > 0) {
    const int hh = n >> 1;
    const double t = lds_f64(sm + thr + 8u * (uint32_t)(r + hh + 1));
    const bool lt = t < s;
    r = lt ? r + hh + 1 : r;
    n = lt ? n - hh - 1 : hh;
  }
  return r;
}

// the decision of one invocation: the final candidate id (kNone16 for None), its record, the
// SP_DEC_* code, the fill, objective, slack and wait budget
struct FastDec {
  uint32_t u, meta;
  int code, fill;
  double score, sk, wait;
};

template <int K>
__device__ __forceinline__ FastDec decide_fast_core(const PlanHdr& h, uint32_t sm, uint32_t lut,
                                                    const InF<K>& x) {
  const int nB = h.nB;
  const int lmax = h.lut_n - 1;
  // batch lanes admitted by min_batch (configurator.py:264-265) and by available (288)
  const uint32_t A = lds_u32(sm + lut + 4u * (uint32_t)min(max(x.mb, 0), lmax));
  const uint32_t B = lds_u32(sm + lut + 4u * (uint32_t)min(max(x.av, 0), lmax));
  const int lo = (int)(A & 0xFFu);
  const int le = (int)((B >> 8) & 0xFFu);
  const int tb = (int)(A >> 16);          // tri_base(lo) - lo: lane [lo, hi] at tb + hi
  const bool any1 = lo < nB;              // some batch size >= min_batch
  const bool any2 = lo < le;              // some admitted batch size <= available
  const uint32_t o1 = 2u * (uint32_t)(any1 ? tb + nB - 1 : 0);
  const uint32_t o2 = 2u * (uint32_t)(any2 ? tb + le - 1 : 0);

  uint32_t u = kNone16, u2 = kNone16;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const KindDesc& d = h.kd[k];
    if (d.R == 0) continue;  // kind absent from this table (uniform)
    const int r = fast_row(sm, d, x.s[k]);
    const uint32_t row = (uint32_t)d.rows_off + (uint32_t)(r * h.row_stride);
    const uint32_t m1 = lds_u16(sm + row + o1);
    const uint32_t m2 = lds_u16(sm + row + o2);
    const bool ex = (x.fl >> (SP_FLAG_EXCL_SHIFT + k)) & 1u;  // configurator.py:259-263
    u = ex ? u : min(u, m1);
    u2 = ex ? u2 : min(u2, m2);
  }
  u = any1 ? u : kNone16;  // configurator.py:266-267: empty mask -> None
  u2 = any2 ? u2 : kNone16;

  const bool some = u != kNone16;
  const uint32_t uu = some ? u : 0u;
  const uint32_t recb = (uint32_t)h.recb_off;
  const uint32_t rsc = (uint32_t)h.score_off;
  const uint2 cb = lds_v2(sm + recb + 8u * uu);  // {idx | feas << 16 | kind << 17, batch}
  const double lat_u = lds_f64(sm + (uint32_t)h.lat_off + 8u * uu);
  double score = lds_f64(sm + rsc + 8u * uu);
  const int bat = (int)cb.y;
  double sk = pick_kind<K>(x.s, (int)(cb.x >> 17));
  // safe delayed batching (configurator.py:271-286)
  const bool big = bat > x.av;
  const double wait = __dsub_rn(sk, lat_u);
  const bool delay = (x.fl & SP_FLAG_ALLOW_DELAY) && big &&
                     (long long)x.sup >= (long long)bat - (long long)x.av && wait > 0.0;
  // downgrade to a batch size that fits what is available (configurator.py:287-291)
  const bool down = !delay && big && u2 != kNone16;
  uint32_t meta = cb.x;
  int fb = bat;
  if (down) {
    const uint2 c2 = lds_v2(sm + recb + 8u * u2);
    score = lds_f64(sm + rsc + 8u * u2);
    meta = c2.x;
    fb = (int)c2.y;
    sk = pick_kind<K>(x.s, (int)(c2.x >> 17));
  }
  FastDec r;
  r.u = some ? (down ? u2 : u) : kNone16;
  r.meta = meta;
  r.code = some ? ((delay ? SP_DEC_DELAY : SP_DEC_ASSIGN) |
                   (((meta >> 16) & 1u) ? SP_DEC_FEASIBLE : 0))
                : SP_DEC_NONE;
  r.fill = some ? (delay ? x.av : min(fb, x.av)) : 0;
  r.score = some ? score : 0.0;
  r.sk = some ? sk : 0.0;
  r.wait = (some && delay) ? wait : 0.0;
  return r;
}

template <int K>
__device__ __forceinline__ void decide_fast(const PlanHdr& h, uint32_t sm, uint32_t lut,
                                            const FastIO<K>& io, uint32_t i, const InF<K>& x) {
  const FastDec r = decide_fast_core<K>(h, sm, lut, x);
  io.out_idx[i] = r.code != SP_DEC_NONE ? (int)(r.meta & 0xFFFFu) : -1;
  io.out_code[i] = r.code;
  io.out_fill[i] = r.fill;
  io.out_obj[i] = r.score;
  io.out_slack[i] = r.sk;
  io.out_wait[i] = r.wait;
}

// CTA lookup table v -> (#batch < v) | (#batch <= v) << 8 | (tri_base(lo) - lo) << 16
__device__ __forceinline__ void build_lane_lut(const PlanHdr& h, uint32_t* lut) {
  const int nB = h.nB;
  for (int v = threadIdx.x; v < h.lut_n; v += blockDim.x) {
    int lo = 0, le = 0;
    for (int b = 0; b < nB; ++b) {
      lo += h.batch_vals[b] < v;
      le += h.batch_vals[b] <= v;
    }
    const int tb = lo * nB - ((lo * (lo - 1)) >> 1) - lo;
    lut[v] = (uint32_t)lo | ((uint32_t)le << 8) | ((uint32_t)tb << 16);
  }
}

constexpr int kK2fDepth = 3;

template <int K, int THREADS = 1024>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS) k_select_fast(
    const uint8_t* __restrict__ plan, PlanHdr h, FastIO<K> io) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  const int bytes = h.total_bytes;
  // Programmatic dependent launch: everything above griddepcontrol.wait touches only
  // parameters, this CTA's shared memory and (when io.prestage) a plan image that an earlier
  // select launch has already waited on, so it overlaps the previous kernel's tail; the
  // invocation stream is neither read nor written before the predecessor grid has completed.
  const bool pre = io.prestage != 0;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    if (pre) {  // TMA bulk copies of the plan image, completion on one mbarrier
      mbar_expect_tx(&s_bar, (uint32_t)bytes);
      for (int c = 0; c < bytes; c += kStageChunk)
        bulk_g2s(smem + c, plan + c, (uint32_t)min(kStageChunk, bytes - c), &s_bar);
    }
  }
  build_lane_lut(h, reinterpret_cast<uint32_t*>(smem + io.lut_bytes_off));
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the next launch in the stream may start its prologue as this grid's CTAs retire
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0 && !pre) {
    mbar_expect_tx(&s_bar, (uint32_t)bytes);
    for (int c = 0; c < bytes; c += kStageChunk)
      bulk_g2s(smem + c, plan + c, (uint32_t)min(kStageChunk, bytes - c), &s_bar);
  }
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t i = blockIdx.x * blockDim.x + tid;
  // kK2fDepth register buffers: the next kK2fDepth - 1 invocations of this thread are in
  // flight while one is decided
  InF<K> buf[kK2fDepth];
#pragma unroll
  for (int q = 0; q < kK2fDepth; ++q)
    if (i + q * stride < io.N) load_fast<K>(io, i + q * stride, buf[q]);
  __syncthreads();
  mbar_wait(&s_bar, 0);
  uint32_t sb;  // shared-window base of the staged plan, ordered after the wait
  asm volatile("mov.u32 %0, %1;" : "=r"(sb) : "r"(smem_u32(smem)) : "memory");
  for (; i < io.N; i += kK2fDepth * stride) {
#pragma unroll
    for (int q = 0; q < kK2fDepth; ++q) {
      const uint32_t j = i + q * stride;
      if (j >= io.N) break;
      decide_fast<K>(h, sb, (uint32_t)io.lut_bytes_off, io, j, buf[q]);
      if (j + kK2fDepth * stride < io.N) load_fast<K>(io, j + kK2fDepth * stride, buf[q]);
    }
  }
}
