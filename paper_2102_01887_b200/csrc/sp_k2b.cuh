// sp_k2b.cuh — K2b, the staircase decision kernel (included by sp_select.cu).
//
// Per invocation (one thread), against one staged plan image:
//   for every admitted kind k:  r = stair_row(slack_k)  -> row = W u16 unified candidate
//                               ids; acc = vmin(acc, row) (two u16 lanes per instruction)
//   lanes outside [min_batch, available] are masked once (min(a|m, b|m) = min(a, b)|m);
//   the overall argmin is the smallest unified id (ids are ordered by the reference's
//   argmin key (score, cost, res, id_rank)); its 32-byte record gives the decision.
// Shared-memory plan addresses are formed from the extern array so that every plan access
// compiles to LDS (STAGED); plans too big for the budget are read from global memory.

template <bool STAGED>
__device__ __forceinline__ const uint8_t* plan_base(const uint8_t* smem, const uint8_t* const* gptr,
                                                    const int* s_off, int t) {
  if (STAGED) return smem + s_off[t];
  return gptr[t];
}

// Row of the threshold staircase for slack s: #{j in [1, R) : thr[j] < s}.
__device__ __forceinline__ int stair_row(const uint8_t* base, const uint4& q0, const uint4& q1,
                                         double s) {
  if (s != s) return 0;  // NaN: nothing is feasible (lat < NaN is false)
  const double* thr = reinterpret_cast<const double*>(base + (int)q0.z);
  const uint32_t* bkt = reinterpret_cast<const uint32_t*>(base + (int)q1.x);
  const uint64_t kmin = ((uint64_t)q0.y << 32) | q0.x;
  const uint32_t nb1 = q1.y & 0xFFFFu, shift = q1.y >> 16;
  const uint64_t key = order_key((uint64_t)__double_as_longlong(s));
  uint64_t b = key < kmin ? 0ull : ((key - kmin) >> shift);
  b = b < nb1 ? b : nb1;
  const uint32_t e = bkt[b];
  int r = (int)(e & 0xFFFFu);
  int n = (int)(e >> 16);
  while (n > 0) {  // thresholds of this bucket: thr[r+1 .. r+n], ascending
    const int hh = n >> 1;
    if (thr[r + hh + 1] < s) {
      r += hh + 1;
      n -= hh + 1;
    } else {
      n = hh;
    }
  }
  return r;
}

template <int KT, int WW>
__device__ __forceinline__ void decide_plan(const uint8_t* base, const SelectIO& io, int i,
                                            const In<KT>& x, const uint32_t* s_mlo,
                                            const uint32_t* s_mhi, bool want_kmin) {
  constexpr int NW = WW / 2;  // 32-bit words per row
  const PlanHdr* h = reinterpret_cast<const PlanHdr*>(base);
  const int pw = h->W;        // this plan's row width (8 or 16 lanes)
  const CandRec* rec = reinterpret_cast<const CandRec*>(base + h->rec_off);

  uint32_t acc[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) acc[w] = 0xFFFFFFFFu;

#pragma unroll
  for (int k = 0; k < KT; ++k) {
    if (k >= io.K) break;
    const uint4* kd = reinterpret_cast<const uint4*>(&h->kd[k]);
    const uint4 q1 = kd[1];
    const int R = (int)q1.z;
    const bool ex = (x.fl >> (SP_FLAG_EXCL_SHIFT + k)) & 1u;
    if (R == 0 || (ex && !want_kmin)) {
      if (want_kmin) io.out_kind_min[(size_t)i * io.K + k] = INFINITY;
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
    if (!ex) {
#pragma unroll
      for (int w = 0; w < NW; ++w) acc[w] = __vminu2(acc[w], U[w]);
    }
    if (want_kmin) {  // Eq. 3 operand: unmasked min score of the kind
      const uint32_t u = hmin_all<NW>(U);
      io.out_kind_min[(size_t)i * io.K + k] = (u != kNone16) ? rec[u].score : INFINITY;
    }
  }

  // batch lanes admitted by min_batch (configurator.py:264-265) and available (288)
  int lo, le;
  const int lut_n = h->lut_n;
  if (lut_n > 0) {
    const uint16_t* lut = reinterpret_cast<const uint16_t*>(base + h->lut_off);
    const int nB = h->nB;
    lo = x.mb <= 0 ? 0 : (x.mb >= lut_n ? nB : (int)(lut[x.mb] & 0xFFu));
    le = x.av <= 0 ? 0 : (x.av >= lut_n ? nB : (int)(lut[x.av] >> 8));
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
  uint32_t u = hmin_or<NW>(acc, m1);
  if (u == kNone16) {  // configurator.py:266-267
    o.idx = -1; o.code = SP_DEC_NONE; o.fill = 0;
    o.obj = 0.0; o.slack = 0.0; o.wait = 0.0;
    store_out(io, i, o);
    return;
  }
  uint4 a = *reinterpret_cast<const uint4*>(rec + u);
  uint4 b = *(reinterpret_cast<const uint4*>(rec + u) + 1);
  double sk = pick_kind<KT>(x.s, (int)b.w);
  int B = (int)b.z;
  // safe delayed batching (configurator.py:271-286)
  if ((x.fl & SP_FLAG_ALLOW_DELAY) && B > x.av &&
      (long long)x.sup >= (long long)B - (long long)x.av) {
    const double wait = __dsub_rn(sk, __hiloint2double((int)b.y, (int)b.x));
    if (wait > 0.0) {
      o.idx = (int)a.z;
      o.code = SP_DEC_DELAY | (a.w ? SP_DEC_FEASIBLE : 0);
      o.fill = x.av;
      o.obj = __hiloint2double((int)a.y, (int)a.x);
      o.slack = sk;
      o.wait = wait;
      store_out(io, i, o);
      return;
    }
  }
  // downgrade to a batch size that fits what is available (configurator.py:287-291)
  if (B > x.av) {
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
      u = u2;
      a = *reinterpret_cast<const uint4*>(rec + u);
      b = *(reinterpret_cast<const uint4*>(rec + u) + 1);
      sk = pick_kind<KT>(x.s, (int)b.w);
      B = (int)b.z;
    }
  }
  o.idx = (int)a.z;
  o.code = SP_DEC_ASSIGN | (a.w ? SP_DEC_FEASIBLE : 0);
  o.fill = min(B, x.av);
  o.obj = __hiloint2double((int)a.y, (int)a.x);
  o.slack = sk;
  o.wait = 0.0;
  store_out(io, i, o);
}

template <int KT, int WW, bool STAGED>
__device__ __forceinline__ void plan_loop(const uint8_t* smem, const PlanPtrs& pp, const int* s_off,
                                          const SelectIO& io, const uint32_t* s_mlo,
                                          const uint32_t* s_mhi) {
  const bool want_kmin = io.out_kind_min != nullptr;
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  In<KT> cur, nxt;
  if (i < io.N) load_in<KT>(io, i, cur);
  for (; i < io.N; i += stride) {
    const int j = i + stride;
    if (j < io.N) load_in<KT>(io, j, nxt);  // prefetch the next invocation
    decide_plan<KT, WW>(plan_base<STAGED>(smem, pp.p, s_off, cur.t), io, i, cur, s_mlo, s_mhi,
                        want_kmin);
    cur = nxt;
  }
}

template <int KT, int WW>
__global__ void __launch_bounds__(512, 2) k_select_plan(PlanPtrs pp, int smem_budget, SelectIO io) {
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
  for (int u = tid; u < (WW + 1) * NW; u += blockDim.x) {
    const int row = u / NW, w = u % NW;
    const int b0 = 2 * w, b1 = 2 * w + 1;
    s_mlo[u] = (b0 < row ? 0xFFFFu : 0u) | (b1 < row ? 0xFFFF0000u : 0u);
    s_mhi[u] = (b0 >= row ? 0xFFFFu : 0u) | (b1 >= row ? 0xFFFF0000u : 0u);
  }
  __syncthreads();
  if (s_fit) {
    mbar_wait(&s_bar, 0);
    plan_loop<KT, WW, true>(smem, pp, s_off, io, s_mlo, s_mhi);
  } else {
    plan_loop<KT, WW, false>(smem, pp, s_off, io, s_mlo, s_mhi);
  }
}
