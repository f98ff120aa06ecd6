// sp_k2b.cuh — K2b, the staircase decision kernel (included by sp_select.cu).
//
// Per invocation (one thread), against one staged plan image:
//   lo = #batch sizes < min_batch, le = #batch sizes <= available      (one u16 LUT load each)
//   for every kind k:  r_k = stair_row(slack_k)                         (bucket + short search)
//                      u  = min(u, rows_k[r_k][lo .. nB-1])             (one u16 load)
//   u is the reference's masked argmin (unified ids are ordered by (score, cost, res,
//   id_rank)); only when the winner's batch exceeds `available` and no delay is taken is
//   the downgrade argmin   min_k rows_k[r_k][lo .. le-1]   loaded (one more u16 per kind).
// One 1024-thread CTA per SM stages the plan(s) with TMA bulk copies while its threads
// already fetch their first two invocations; shared-memory plan addresses are formed from
// the extern array so every plan access is an LDS.  For single-table launches the plan
// header travels as a kernel parameter, so every descriptor field is a constant-bank
// (uniform-register) operand instead of a per-invocation load.

constexpr int kStageChunk = 8192;  // bytes per TMA bulk copy when staging a plan image

// Decoded plan header: field offsets and per-kind descriptors.
template <int KT>
struct View {
  const uint8_t* base;
  int nB, stride, score_off, recb_off, lat_off, lut_off, lut_n;
  uint4 q0[KT];  // {kmin_hi, nb1 | shift << 16, thr_off, rows_off}
  uint4 q1[KT];  // {bkt_off, R, nonpos, -}
};

template <int KT>
__device__ __forceinline__ void make_view(View<KT>& v, const uint8_t* base, const PlanHdr& h, int K) {
  v.base = base;
  v.nB = h.nB;
  v.stride = h.row_stride;
  v.score_off = h.score_off;
  v.recb_off = h.recb_off;
  v.lat_off = h.lat_off;
  v.lut_off = h.lut_off;
  v.lut_n = h.lut_n;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k < K) {
      v.q0[k] = *reinterpret_cast<const uint4*>(&h.kd[k]);
      v.q1[k] = *(reinterpret_cast<const uint4*>(&h.kd[k]) + 1);
    } else {
      v.q0[k] = make_uint4(0, 0, 0, 0);
      v.q1[k] = make_uint4(0, 0, 0, 0);
    }
  }
}

// Row of the threshold staircase for slack s: #{j in [1, R) : thr[j] < s}.
__device__ __forceinline__ int stair_row(const uint8_t* base, const uint4& q0, const uint4& q1,
                                         double s) {
  const double* thr = reinterpret_cast<const double*>(base + (int)q0.z);
  const bool nonpos = q1.z != 0;
  int r = 0, n = nonpos ? (int)q1.y - 1 : 0;  // generic: search every real threshold
  if (!nonpos && s > 0.0) {
    // positive thresholds: bucket on the high word of the IEEE encoding
    const uint32_t* bkt = reinterpret_cast<const uint32_t*>(base + (int)q1.x);
    const int d = __double2hiint(s) - (int)q0.x;
    const uint32_t nb1 = q0.y & 0xFFFFu;
    uint32_t b = d < 0 ? 0u : ((uint32_t)d >> (q0.y >> 16));
    b = b < nb1 ? b : nb1;
    const uint32_t e = bkt[b];
    r = (int)(e & 0xFFFFu);
    n = (int)(e >> 16);
  }  // else (s <= 0 or NaN, all thresholds positive): r = 0
  while (n > 0) {  // candidate thresholds thr[r+1 .. r+n], ascending
    const int hh = n >> 1;
    const bool lt = thr[r + hh + 1] < s;
    r = lt ? r + hh + 1 : r;
    n = lt ? n - hh - 1 : hh;
  }
  return r;
}

// index of the lane interval [lo, hi] inside a row
__device__ __forceinline__ int tri_index(int lo, int hi, int nB) {
  return lo * nB - ((lo * (lo - 1)) >> 1) + (hi - lo);
}

template <int KT, bool KMIN>
__device__ __forceinline__ void decide_plan(const View<KT>& v, const SelectIO& io, int i,
                                            const In<KT>& x) {
  const uint8_t* base = v.base;
  const int nB = v.nB;
  const double* rscore = reinterpret_cast<const double*>(base + v.score_off);
  const CandB* recb = reinterpret_cast<const CandB*>(base + v.recb_off);

  // batch lanes admitted by min_batch (configurator.py:264-265) and available (288)
  int lo, le;
  if (v.lut_n > 0) {  // lut[0] = (0, 0); lut[lut_n - 1] saturates at (nB, nB)
    const uint16_t* lut = reinterpret_cast<const uint16_t*>(base + v.lut_off);
    lo = (int)(lut[min(max(x.mb, 0), v.lut_n - 1)] & 0xFFu);
    le = (int)(lut[min(max(x.av, 0), v.lut_n - 1)] >> 8);
  } else {
    const PlanHdr* h = reinterpret_cast<const PlanHdr*>(base);
    lo = le = 0;
    for (int b = 0; b < nB; ++b) {
      const int bv = h->batch_vals[b];
      lo += (bv < x.mb);
      le += (bv <= x.av);
    }
  }
  const bool any1 = lo < nB;
  const int idx1 = any1 ? tri_index(lo, nB - 1, nB) : 0;

  uint32_t u = kNone16;
  int rowoff[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    rowoff[k] = -1;
    if (k >= io.K) break;
    const bool ex = (x.fl >> (SP_FLAG_EXCL_SHIFT + k)) & 1u;
    if (v.q1[k].y == 0 || (!KMIN && ex)) {
      if (KMIN) io.out_kind_min[(size_t)i * io.K + k] = INFINITY;
      continue;
    }
    const int r = stair_row(base, v.q0[k], v.q1[k], x.s[k]);
    const int ro = (int)v.q0[k].w + r * v.stride;
    const uint16_t* row = reinterpret_cast<const uint16_t*>(base + ro);
    if (!ex) {
      rowoff[k] = ro;
      if (any1) u = min(u, (uint32_t)row[idx1]);
    }
    if (KMIN) {  // Eq. 3 operand: unmasked min score of the kind = interval [0, nB-1]
      const uint32_t m = row[nB - 1];
      io.out_kind_min[(size_t)i * io.K + k] = (m != kNone16) ? rscore[m] : INFINITY;
    }
  }

  Out o;
  o.idx = -1; o.code = SP_DEC_NONE; o.fill = 0;
  o.obj = 0.0; o.slack = 0.0; o.wait = 0.0;
  if (u != kNone16) {  // else: configurator.py:266-267
    CandB cb = recb[u];
    double score = rscore[u];
    double sk = pick_kind<KT>(x.s, (int)(cb.meta >> 17));
    // safe delayed batching (configurator.py:271-286)
    const bool big = cb.batch > x.av;
    bool delay = false;
    double wait = 0.0;
    if ((x.fl & SP_FLAG_ALLOW_DELAY) && big &&
        (long long)x.sup >= (long long)cb.batch - (long long)x.av) {
      const double* rlat = reinterpret_cast<const double*>(base + v.lat_off);
      wait = __dsub_rn(sk, rlat[u]);
      delay = wait > 0.0;
    }
    // downgrade to a batch size that fits what is available (configurator.py:287-291)
    if (!delay && big && lo < le) {
      const int idx2 = tri_index(lo, le - 1, nB);
      uint32_t u2 = kNone16;
#pragma unroll
      for (int k = 0; k < KT; ++k)
        if (rowoff[k] >= 0)
          u2 = min(u2, (uint32_t)reinterpret_cast<const uint16_t*>(base + rowoff[k])[idx2]);
      if (u2 != kNone16) {
        cb = recb[u2];
        score = rscore[u2];
        sk = pick_kind<KT>(x.s, (int)(cb.meta >> 17));
      }
    }
    const int feas = (cb.meta >> 16) & 1u;
    o.idx = (int)(cb.meta & 0xFFFFu);
    o.code = (delay ? SP_DEC_DELAY : SP_DEC_ASSIGN) | (feas ? SP_DEC_FEASIBLE : 0);
    o.fill = delay ? x.av : min(cb.batch, x.av);
    o.obj = score;
    o.slack = sk;
    o.wait = delay ? wait : 0.0;
  }
  store_out(io, i, o);
}

// Single-table hot loop: the view is built once from the parameter-space header.
// Ping-pong over two register buffers (unrolled by two so no buffer is ever copied): while
// invocation i is decided from buffer A, invocation i + stride is already in flight into B.
// (Measured alternatives that were slower on B200: a 3-stage TMA input ring in shared
// memory, and cp.async.bulk.prefetch.L2 of the tiles 3-4 iterations ahead.)
template <int KT>
__device__ __forceinline__ void plan_loop_single(const View<KT>& v, const SelectIO& io, int i,
                                                 In<KT>& a, In<KT>& b) {
  const int stride = gridDim.x * blockDim.x;
  for (; i < io.N; i += 2 * stride) {
    decide_plan<KT, false>(v, io, i, a);
    const int j = i + stride;
    if (j >= io.N) break;
    if (j + stride < io.N) load_in<KT>(io, j + stride, a);
    decide_plan<KT, false>(v, io, j, b);
    if (j + 2 * stride < io.N) load_in<KT>(io, j + 2 * stride, b);
  }
}

// Generic loop: per-invocation table, header read from the (staged or global) image.
template <int KT, bool STAGED, bool KMIN>
__device__ __forceinline__ void plan_loop_multi(const uint8_t* smem, const PlanPtrs& pp,
                                                const int* s_off, const SelectIO& io, int i) {
  const int stride = gridDim.x * blockDim.x;
  for (; i < io.N; i += stride) {
    In<KT> x;
    load_in<KT>(io, i, x);
    const uint8_t* base = STAGED ? smem + s_off[x.t] : pp.p[x.t];
    View<KT> v;
    make_view<KT>(v, base, *reinterpret_cast<const PlanHdr*>(base), io.K);
    decide_plan<KT, KMIN>(v, io, i, x);
  }
}

template <int KT>
__global__ void __launch_bounds__(1024, 1) k_select_plan(PlanPtrs pp, int smem_budget, SelectIO io) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int s_off[kMaxPlanTables + 1];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_fit;
  const int tid = threadIdx.x;
  // programmatic dependent launch: nothing of the predecessor's output (the plan image, the
  // invocation stream) is touched before it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) {
    int off = 0;
    for (int t = 0; t < pp.n; ++t) {
      s_off[t] = off;
      off += pp.hv ? pp.h.total_bytes : reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes;
    }
    s_off[pp.n] = off;
    s_fit = off <= smem_budget;
    if (s_fit) {  // one TMA bulk copy per plan image, completion on one mbarrier
      mbar_init(&s_bar, 1);
      mbar_expect_tx(&s_bar, (uint32_t)off);
      for (int t = 0; t < pp.n; ++t)
        for (int c = s_off[t]; c < s_off[t + 1]; c += kStageChunk)  // several copies in flight
          bulk_g2s(smem + c, pp.p[t] + (c - s_off[t]),
                   (uint32_t)min(kStageChunk, s_off[t + 1] - c), &s_bar);
    }
  }
  // the first two invocations are fetched while the plan copy is in flight
  const int stride = gridDim.x * blockDim.x;
  const int i = blockIdx.x * blockDim.x + tid;
  const bool kmin = io.out_kind_min != nullptr;
  // one table without kind minima: the single-table loop, with the header from the kernel
  // parameter or (a plan rebuilt after the host last saw it) from the staged image
  const bool single = pp.n == 1 && !kmin;
  In<KT> cur, nxt;
  if (single) {
    if (i < io.N) load_in<KT>(io, i, cur);
    if (i + stride < io.N) load_in<KT>(io, i + stride, nxt);
  }
  __syncthreads();
  if (s_fit) {
    mbar_wait(&s_bar, 0);
    if (single) {
      View<KT> v;
      if (pp.hv) make_view<KT>(v, smem, pp.h, io.K);
      else make_view<KT>(v, smem, *reinterpret_cast<const PlanHdr*>(smem), io.K);
      plan_loop_single<KT>(v, io, i, cur, nxt);
    } else if (kmin) {
      plan_loop_multi<KT, true, true>(smem, pp, s_off, io, i);
    } else {
      plan_loop_multi<KT, true, false>(smem, pp, s_off, io, i);
    }
  } else {
    if (kmin) plan_loop_multi<KT, false, true>(smem, pp, s_off, io, i);
    else plan_loop_multi<KT, false, false>(smem, pp, s_off, io, i);
  }
}
