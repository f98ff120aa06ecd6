// sp_k2b.cuh — K2b, the staircase decision kernel (included by sp_select.cu).
//
// Per invocation (one thread), against one staged plan image:
//   for every admitted kind k:  r = stair_row(slack_k)  -> row = W u16 unified candidate
//                               ids; acc = vmin(acc, row) (two u16 lanes per instruction)
//   lanes outside [min_batch, available] are masked once (min(a|m, b|m) = min(a, b)|m);
//   the overall argmin is the smallest unified id (ids are ordered by the reference's
//   argmin key (score, cost, res, id_rank)); its records give the decision.
// One 1024-thread CTA per SM stages the plan(s) with TMA bulk copies while its threads
// already fetch their first two invocations; shared-memory plan addresses are formed from
// the extern array so every plan access is an LDS (plans over the budget are read from
// global memory by a second instantiation of the loop).

template <bool STAGED>
__device__ __forceinline__ const uint8_t* plan_base(const uint8_t* smem, const uint8_t* const* gptr,
                                                    const int* s_off, int t) {
  if (STAGED) return smem + s_off[t];
  return gptr[t];
}

// Row of the threshold staircase for slack s: #{j in [1, R) : thr[j] < s}.
//   q0 = {kmin_hi, nb1 | shift << 16, thr_off, rows_off},  q1 = {bkt_off, R, nonpos, -}
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

template <int KT, int WW, bool KMIN>
__device__ __forceinline__ void decide_plan(const uint8_t* base, const SelectIO& io, int i,
                                            const In<KT>& x, const uint32_t* s_mlo,
                                            const uint32_t* s_mhi) {
  constexpr int NW = WW / 2;  // 32-bit words per row
  const PlanHdr* h = reinterpret_cast<const PlanHdr*>(base);
  const int pw = h->W;        // this plan's row width (8 or 16 lanes)
  const CandA* reca = reinterpret_cast<const CandA*>(base + h->rec_off);
  const CandB* recb = reinterpret_cast<const CandB*>(base + h->recb_off);

  uint32_t acc[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) acc[w] = 0xFFFFFFFFu;

#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k >= io.K) break;
    const uint4* kd = reinterpret_cast<const uint4*>(&h->kd[k]);
    const uint4 q1 = kd[1];
    const int R = (int)q1.y;
    const uint32_t exm = ((x.fl >> (SP_FLAG_EXCL_SHIFT + k)) & 1u) ? 0xFFFFFFFFu : 0u;
    if (R == 0 || (!KMIN && exm)) {
      if (KMIN) io.out_kind_min[(size_t)i * io.K + k] = INFINITY;
      continue;
    }
    const uint4 q0 = kd[0];
    const int r = stair_row(base, q0, q1, x.s[k]);
    const uint4* row = reinterpret_cast<const uint4*>(base + (int)q0.w + r * (2 * pw));
    uint32_t U[NW];
    if (WW == 16 && pw == 8) {  // narrow plan in a wide launch
      const uint4 a = row[0];
      U[0] = a.x; U[1] = a.y; U[2] = a.z; U[3] = a.w;
#pragma unroll
      for (int w = 4; w < NW; ++w) U[w] = 0xFFFFFFFFu;
    } else {
#pragma unroll
      for (int q = 0; q < NW / 4; ++q) {
        const uint4 a = row[q];
        U[4 * q + 0] = a.x; U[4 * q + 1] = a.y; U[4 * q + 2] = a.z; U[4 * q + 3] = a.w;
      }
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) acc[w] = __vminu2(acc[w], U[w] | exm);
    if (KMIN) {  // Eq. 3 operand: unmasked min score of the kind
      const uint32_t u = hmin_all<NW>(U);
      io.out_kind_min[(size_t)i * io.K + k] = (u != kNone16) ? reca[u].score : INFINITY;
    }
  }

  // batch lanes admitted by min_batch (configurator.py:264-265) and available (288)
  int lo, le;
  const int lut_n = h->lut_n;
  if (lut_n > 0) {  // lut[0] = (0, 0); lut[lut_n - 1] saturates at (nB, nB)
    const uint16_t* lut = reinterpret_cast<const uint16_t*>(base + h->lut_off);
    const uint32_t a = lut[min(max(x.mb, 0), lut_n - 1)];
    const uint32_t b = lut[min(max(x.av, 0), lut_n - 1)];
    lo = (int)(a & 0xFFu);
    le = (int)(b >> 8);
  } else {
    lo = le = 0;
#pragma unroll
    for (int b = 0; b < WW; ++b) {
      const int bv = h->batch_vals[b];
      lo += (bv < x.mb);
      le += (bv <= x.av);
    }
  }
  uint32_t m1[NW];
  {
    const uint4* q = reinterpret_cast<const uint4*>(s_mlo + lo * NW);
#pragma unroll
    for (int u = 0; u < NW / 4; ++u) {
      const uint4 v = q[u];
      m1[4 * u] = v.x; m1[4 * u + 1] = v.y; m1[4 * u + 2] = v.z; m1[4 * u + 3] = v.w;
    }
  }
  Out o;
  o.idx = -1; o.code = SP_DEC_NONE; o.fill = 0;
  o.obj = 0.0; o.slack = 0.0; o.wait = 0.0;
  const uint32_t u = hmin_or<NW>(acc, m1);
  if (u != kNone16) {
    CandA ca = reca[u];
    CandB cb = recb[u];
    double sk = pick_kind<KT>(x.s, (int)(cb.meta >> 17));
    // safe delayed batching (configurator.py:271-286)
    const bool big = cb.batch > x.av;
    const double wait = __dsub_rn(sk, ca.lat);
    const bool delay = (x.fl & SP_FLAG_ALLOW_DELAY) && big &&
                       (long long)x.sup >= (long long)cb.batch - (long long)x.av && wait > 0.0;
    // downgrade to a batch size that fits what is available (configurator.py:287-291)
    if (!delay && big) {
      uint32_t m2[NW];
      const uint4* q = reinterpret_cast<const uint4*>(s_mhi + le * NW);
#pragma unroll
      for (int v4 = 0; v4 < NW / 4; ++v4) {
        const uint4 v = q[v4];
        m2[4 * v4] = m1[4 * v4] | v.x; m2[4 * v4 + 1] = m1[4 * v4 + 1] | v.y;
        m2[4 * v4 + 2] = m1[4 * v4 + 2] | v.z; m2[4 * v4 + 3] = m1[4 * v4 + 3] | v.w;
      }
      const uint32_t u2 = hmin_or<NW>(acc, m2);
      if (u2 != kNone16) {
        ca = reca[u2];
        cb = recb[u2];
        sk = pick_kind<KT>(x.s, (int)(cb.meta >> 17));
      }
    }
    const int feas = (cb.meta >> 16) & 1u;
    o.idx = (int)(cb.meta & 0xFFFFu);
    o.code = (delay ? SP_DEC_DELAY : SP_DEC_ASSIGN) | (feas ? SP_DEC_FEASIBLE : 0);
    o.fill = delay ? x.av : min(cb.batch, x.av);
    o.obj = ca.score;
    o.slack = sk;
    o.wait = delay ? wait : 0.0;
  }
  store_out(io, i, o);
}

template <int KT, int WW, bool STAGED, bool KMIN>
__device__ __forceinline__ void plan_loop(const uint8_t* smem, const PlanPtrs& pp, const int* s_off,
                                          const SelectIO& io, const uint32_t* s_mlo,
                                          const uint32_t* s_mhi, int i, In<KT>& cur,
                                          In<KT>& nxt) {
  const int stride = gridDim.x * blockDim.x;
  for (; i < io.N; i += stride) {
    const int j = i + 2 * stride;
    In<KT> nn;
    if (j < io.N) load_in<KT>(io, j, nn);  // prefetch two invocations ahead
    decide_plan<KT, WW, KMIN>(plan_base<STAGED>(smem, pp.p, s_off, cur.t), io, i, cur, s_mlo,
                              s_mhi);
    cur = nxt;
    nxt = nn;
  }
}

template <int KT, int WW>
__global__ void __launch_bounds__(1024, 1) k_select_plan(PlanPtrs pp, int smem_budget, SelectIO io) {
  constexpr int NW = WW / 2;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int s_off[kMaxPlanTables];
  __shared__ __align__(16) uint32_t s_mlo[(WW + 1) * NW];  // lanes b <  lo masked
  __shared__ __align__(16) uint32_t s_mhi[(WW + 1) * NW];  // lanes b >= c  masked
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_fit;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int off = 0;
    for (int t = 0; t < pp.n; ++t) {
      s_off[t] = off;
      off += reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes;
    }
    s_fit = off <= smem_budget;
    if (s_fit) {  // one TMA bulk copy per plan image, completion on one mbarrier
      mbar_init(&s_bar, 1);
      mbar_expect_tx(&s_bar, (uint32_t)off);
      for (int t = 0; t < pp.n; ++t) {
        const int bytes = reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes;
        bulk_g2s(smem + s_off[t], pp.p[t], (uint32_t)bytes, &s_bar);
      }
    }
  }
  // the first two invocations are fetched while the plan copy is in flight
  const int stride = gridDim.x * blockDim.x;
  const int i = blockIdx.x * blockDim.x + tid;
  In<KT> cur, nxt;
  if (i < io.N) load_in<KT>(io, i, cur);
  if (i + stride < io.N) load_in<KT>(io, i + stride, nxt);
  for (int u = tid; u < (WW + 1) * NW; u += blockDim.x) {
    const int row = u / NW, w = u % NW;
    const int b0 = 2 * w, b1 = 2 * w + 1;
    s_mlo[u] = (b0 < row ? 0xFFFFu : 0u) | (b1 < row ? 0xFFFF0000u : 0u);
    s_mhi[u] = (b0 >= row ? 0xFFFFu : 0u) | (b1 >= row ? 0xFFFF0000u : 0u);
  }
  __syncthreads();
  const bool kmin = io.out_kind_min != nullptr;
  if (s_fit) {
    mbar_wait(&s_bar, 0);
    if (kmin) plan_loop<KT, WW, true, true>(smem, pp, s_off, io, s_mlo, s_mhi, i, cur, nxt);
    else plan_loop<KT, WW, true, false>(smem, pp, s_off, io, s_mlo, s_mhi, i, cur, nxt);
  } else {
    if (kmin) plan_loop<KT, WW, false, true>(smem, pp, s_off, io, s_mlo, s_mhi, i, cur, nxt);
    else plan_loop<KT, WW, false, false>(smem, pp, s_off, io, s_mlo, s_mhi, i, cur, nxt);
  }
}
