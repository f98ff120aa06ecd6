// sp_k12.cuh — K1 -> K2 fused: Alg. 1 slack straight into the staircase decision
// (included by sp_select.cu after sp_k2b.cuh).
//
// The snapshot workloads (BASELINE config 4: target sweep x replicas) decide one invocation of
// every operation per pipeline instance right after computing that instance's slack.  Run as
// two kernels, K1 writes slack[I][n_src][K] to HBM and K2 reads it back (2 x 8*n_src*K bytes
// per instance, 448 B for AMBER).  Here one thread owns one instance end to end: for every
// source operation s it runs the forward DP of K1 (sp_slack.cu; same program, same shared-
// memory DP slots, same bit-exact arithmetic), forms slack_k = (b_k >= 0 ? own/Tmax :
// own/Tmin) * b_k with b_k = (target - now) - Q_k (configurator.py:526-543), and decides
// invocation (i, s) against operation s's staircase plan (configurator.py:239-300) — the
// slack never leaves registers.  Persistent grid; every CTA stages all vertex programs and all
// plans once.

constexpr int kK12Warps = 4;
// per-warp staging of the group's 32 * n_src decisions: 4 input words + 36 output bytes each,
// so every global access of the per-decision streams is a coalesced, contiguous warp access
constexpr int kK12StageBytesPerDecision = 16 + 36;
constexpr int kK12MaxSrc = kMaxPlanTables;

struct K12Dag {
  const int4* prog;
  const int32_t* prog_ptr;   // n_src + 1
  const uint32_t* preds;
  const int32_t* pred_ptr;   // n_src + 1
  int n_src, nslots, prog_len, pred_len, n_val;
  int single_pred;  // every entry after the source has one predecessor: H = L along chains
};

struct K12In {
  const double* ref;
  int ref_stride;
  const double* target;
  const double* now;
  const double* Q;  // I x K
  int I;
  double* out_kslack;  // optional I x n_src x K
};

// FAST: every table has exactly KT kinds, positive thresholds and a batch lookup table, so the
// decision is K2f's decide_fast (per-table lane lookup table built next to each staged plan);
// otherwise the generic K2b decide_plan.
template <int KT, bool FAST>
__global__ void __launch_bounds__(32 * kK12Warps) k_slack_select(K12Dag g, K12In in, PlanPtrs pp,
                                                                 int plan_off, int stage_off,
                                                                 int out_stage, SelectIO io) {
  extern __shared__ __align__(16) uint8_t sm12[];
  __shared__ int s_pb[kK12MaxSrc + 1], s_qb[kK12MaxSrc + 1], s_off[kK12MaxSrc + 1];
  __shared__ int s_lut[kK12MaxSrc];  // lane lookup table of plan t, relative to its image
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double2* Dall = reinterpret_cast<double2*>(sm12);
  int4* P = reinterpret_cast<int4*>(Dall + (size_t)kK12Warps * g.nslots * 32);
  uint32_t* G = reinterpret_cast<uint32_t*>(P + g.prog_len);
  uint8_t* plans = sm12 + plan_off;
  // ---- stage programs, predecessor byte offsets and every plan image ----
  if (tid <= g.n_src) {
    s_pb[tid] = g.prog_ptr[tid];
    s_qb[tid] = g.pred_ptr[tid];
  }
  if (tid == 0) {
    int off = 0;
    for (int t = 0; t < pp.n; ++t) {
      const PlanHdr* hg = reinterpret_cast<const PlanHdr*>(pp.p[t]);
      s_off[t] = off;
      off += hg->total_bytes;
      if (FAST) {
        s_lut[t] = hg->total_bytes;  // images are multiples of 16 bytes
        off += ((hg->lut_n * 4 + 15) / 16) * 16;
      }
    }
    s_off[pp.n] = off;
  }
  for (int t = tid; t < g.prog_len; t += blockDim.x) P[t] = g.prog[t];
  for (int t = tid; t < g.pred_len; t += blockDim.x) G[t] = g.preds[t] * (32 * sizeof(double2));
  __syncthreads();
  for (int t = 0; t < pp.n; ++t) {
    const uint4* src = reinterpret_cast<const uint4*>(pp.p[t]);
    uint4* dst = reinterpret_cast<uint4*>(plans + s_off[t]);
    const int n16 = reinterpret_cast<const PlanHdr*>(pp.p[t])->total_bytes / 16;
    for (int c = tid; c < n16; c += blockDim.x) dst[c] = src[c];
  }
  __syncthreads();
  if (FAST) {
    for (int t = 0; t < pp.n; ++t)
      build_lane_lut(*reinterpret_cast<const PlanHdr*>(plans + s_off[t]),
                     reinterpret_cast<uint32_t*>(plans + s_off[t] + s_lut[t]));
    __syncthreads();
  }
  const uint32_t plans_sb = smem_u32(plans);
  // this warp's staging area: inputs avail, supply, min_batch, flags; with out_stage also the
  // outputs idx, code, fill, obj, slack, wait — decisions d0 + c of the current group at index c
  // (without it the decisions are stored straight to global memory and L2 merges the strided
  // partial-sector writes)
  const int Dw = 32 * g.n_src;
  const int bpd = out_stage ? kK12StageBytesPerDecision : 16;
  uint8_t* wst = sm12 + stage_off + (size_t)warp * Dw * bpd;
  // this lane's reference latencies, staged once per instance: [value][lane]
  double* Rs = reinterpret_cast<double*>(sm12 + stage_off + (size_t)kK12Warps * Dw * bpd) +
               (size_t)warp * g.n_val * 32 + lane;
  int32_t* s_av = reinterpret_cast<int32_t*>(wst);
  int32_t* s_sup = s_av + Dw;
  int32_t* s_mb = s_sup + Dw;
  uint32_t* s_fl = reinterpret_cast<uint32_t*>(s_mb + Dw);
  int32_t* o_idx = reinterpret_cast<int32_t*>(s_fl + Dw);
  int32_t* o_code = o_idx + Dw;
  int32_t* o_fill = o_code + Dw;
  double* o_obj = reinterpret_cast<double*>(o_fill + Dw);  // 28 * Dw bytes in: 8-aligned
  double* o_sl = o_obj + Dw;
  double* o_wait = o_sl + Dw;
  SelectIO sio = io;  // decisions land in the staging area
  sio.out_idx = o_idx; sio.out_code = o_code; sio.out_fill = o_fill;
  sio.out_obj = o_obj; sio.out_slack = o_sl; sio.out_wait = o_wait;
  FastIO<KT> fio;
  if (FAST) {
    fio.slack = nullptr; fio.avail = nullptr; fio.supply = nullptr;
    fio.min_batch = nullptr; fio.flags = nullptr; fio.out_idx = o_idx;
    fio.out_code = o_code; fio.out_fill = o_fill; fio.out_obj = o_obj;
    fio.out_slack = o_sl; fio.out_wait = o_wait; fio.N = (uint32_t)io.N;
    fio.lut_bytes_off = 0; fio.prestage = 0;
  }
  double2* D = Dall + (size_t)warp * g.nslots * 32 + lane;
  const char* Db = reinterpret_cast<const char*>(D);
  const int K = io.K;
  // ---- one instance per thread, grid-stride over warps of instances ----
  const int nwarps_total = gridDim.x * kK12Warps;
  for (int i0 = (blockIdx.x * kK12Warps + warp) * 32; i0 < in.I; i0 += nwarps_total * 32) {
    const int d0 = i0 * g.n_src;
    const int nd = min(Dw, io.N - d0);
    if (!out_stage) {
      sio.out_idx = io.out_idx + d0; sio.out_code = io.out_code + d0;
      sio.out_fill = io.out_fill ? io.out_fill + d0 : nullptr;
      sio.out_obj = io.out_obj ? io.out_obj + d0 : nullptr;
      sio.out_slack = io.out_slack ? io.out_slack + d0 : nullptr;
      sio.out_wait = io.out_wait ? io.out_wait + d0 : nullptr;
      fio.out_idx = sio.out_idx; fio.out_code = sio.out_code; fio.out_fill = sio.out_fill;
      fio.out_obj = sio.out_obj; fio.out_slack = sio.out_slack; fio.out_wait = sio.out_wait;
    }
    __syncwarp();
    for (int c = lane; c < nd; c += 32) {  // coalesced loads of the group's decision inputs
      s_av[c] = __ldg(io.avail + d0 + c);
      s_sup[c] = __ldg(io.supply + d0 + c);
      s_mb[c] = __ldg(io.min_batch + d0 + c);
      s_fl[c] = __ldg(io.flags + d0 + c);
    }
    __syncwarp();
    const int i = i0 + lane;
    const bool live = i < in.I;
    const int ii = live ? i : i0;
    const double* r = in.ref + (size_t)ii * in.ref_stride;
    for (int v = 0; v < g.n_val; ++v) Rs[v * 32] = __ldg(r + v);  // all loads in flight at once
    // configurator.py:535  budget = self.target_s - now - queueing[k]
    const double base = __dsub_rn(__ldg(in.target + ii), __ldg(in.now + ii));
    double bud[KT];
    bool need_lo = false, need_hi = false;  // which of own/Tmax, own/Tmin the kinds use
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      bud[k] = k < K ? __dsub_rn(base, __ldg(in.Q + (size_t)ii * K + k)) : 0.0;
      if (k < K) {
        need_lo |= bud[k] >= 0.0;
        need_hi |= !(bud[k] >= 0.0);
      }
    }
    for (int s = 0; s < g.n_src; ++s) {
      // K1: forward DP over the source's descendants (sp_slack.cu)
      const int4* Ps = P + s_pb[s];
      const int n = s_pb[s + 1] - s_pb[s];
      const uint32_t* Gs = G + s_qb[s];
      const int4 head = Ps[0];
      const double own = __dadd_rn(0.0, Rs[head.x * 32]);  // total = 0.0; total += ref[op]
      D[(head.y & 0xffff) * 32] = make_double2(own, own);
      double tmax = (head.y >> 16) ? own : -INFINITY;
      double tmin = (head.y >> 16) ? own : INFINITY;
      if (g.single_pred) {
        // trie programs (path lists): one predecessor each, so H and L stay equal along every
        // chain — the DP is one add per entry (the generic loop's max / min over the padded
        // predecessor pair would return the same value)
#pragma unroll 1
        for (int e = 1; e < n; ++e) {
          const int4 pr = Ps[e];
          const double h = __dadd_rn(reinterpret_cast<const double2*>(Db + Gs[pr.z])->x,
                                     Rs[pr.x * 32]);
          D[(pr.y & 0xffff) * 32] = make_double2(h, h);
          if (pr.y >> 16) {
            tmax = h > tmax ? h : tmax;
            tmin = h < tmin ? h : tmin;
          }
        }
      } else {
        for (int e = 1; e < n; ++e) {
          const int4 pr = Ps[e];
          const double rv = Rs[pr.x * 32];
          const uint2* gp = reinterpret_cast<const uint2*>(Gs + pr.z);
          double hm = -INFINITY, lm = INFINITY;
          for (int t = 0; t < pr.w; ++t) {
            const uint2 w0 = gp[t];
            const double2 a = *reinterpret_cast<const double2*>(Db + w0.x);
            const double2 b = *reinterpret_cast<const double2*>(Db + w0.y);
            hm = hm > a.x ? hm : a.x;
            hm = hm > b.x ? hm : b.x;
            lm = lm < a.y ? lm : a.y;
            lm = lm < b.y ? lm : b.y;
          }
          const double h = __dadd_rn(hm, rv), l = __dadd_rn(lm, rv);
          D[(pr.y & 0xffff) * 32] = make_double2(h, l);
          if (pr.y >> 16) {
            tmax = h > tmax ? h : tmax;
            tmin = l < tmin ? l : tmin;
          }
        }
      }
      // min / max over suffixes of own/total, each divided out only if some kind uses it
      const double lo = need_lo ? __ddiv_rn(own, tmax) : 0.0;
      const double hi = need_hi ? __ddiv_rn(own, tmin) : 0.0;
      if (!live) continue;
      // K2: decide invocation (i, s) against operation s's plan
      const int d = i * g.n_src + s;
      In<KT> x;
#pragma unroll
      for (int k = 0; k < KT; ++k) x.s[k] = k < K ? __dmul_rn(bud[k] >= 0.0 ? lo : hi, bud[k]) : 0.0;
      if (in.out_kslack) {
#pragma unroll
        for (int k = 0; k < KT; ++k)
          if (k < K) in.out_kslack[(size_t)d * K + k] = x.s[k];
      }
      const int dl = lane * g.n_src + s;  // index inside the group's staging area
      x.av = s_av[dl];
      x.sup = s_sup[dl];
      x.mb = s_mb[dl];
      x.fl = s_fl[dl];
      x.t = s;
      const uint8_t* bp = plans + s_off[s];
      if (FAST) {
        InF<KT> xf;
#pragma unroll
        for (int k = 0; k < KT; ++k) xf.s[k] = x.s[k];
        xf.av = x.av; xf.sup = x.sup; xf.mb = x.mb; xf.fl = x.fl;
        if (!out_stage) {
          // compact decision into the 16 input bytes it has just consumed: {candidate | code,
          // fill, slack}; the group's flush below expands it with coalesced stores
          const FastDec r = decide_fast_core<KT>(*reinterpret_cast<const PlanHdr*>(bp),
                                                 plans_sb + (uint32_t)s_off[s],
                                                 (uint32_t)s_lut[s], xf);
          s_av[dl] = (int32_t)(r.u | ((uint32_t)r.code << 16));
          s_sup[dl] = r.fill;
          s_mb[dl] = __double2loint(r.sk);
          s_fl[dl] = (uint32_t)__double2hiint(r.sk);
        } else {
          decide_fast<KT>(*reinterpret_cast<const PlanHdr*>(bp), plans_sb + (uint32_t)s_off[s],
                          (uint32_t)s_lut[s], fio, (uint32_t)dl, xf);
        }
      } else {
        View<KT> v;
        make_view<KT>(v, bp, *reinterpret_cast<const PlanHdr*>(bp), K);
        decide_plan<KT, false>(v, sio, dl, x);
      }
    }
    if (FAST && !out_stage) {
      // expand the compact decisions: one decision per lane, contiguous global stores (full
      // sectors); objective, index and wait budget come from the decision's plan records
      __syncwarp();
      int s = lane % g.n_src;
      const int r32 = 32 % g.n_src;
      for (int c = lane; c < nd; c += 32) {
        const uint32_t w0 = (uint32_t)s_av[c];
        const uint32_t u = w0 & 0xFFFFu;
        const int code = (int)(w0 >> 16);
        const double sk = __hiloint2double((int)s_fl[c], s_mb[c]);
        const uint8_t* bp = plans + s_off[s];
        const PlanHdr* hp = reinterpret_cast<const PlanHdr*>(bp);
        int idx = -1;
        double obj = 0.0, wait = 0.0;
        if (code != SP_DEC_NONE) {
          idx = (int)(reinterpret_cast<const CandB*>(bp + hp->recb_off)[u].meta & 0xFFFFu);
          obj = reinterpret_cast<const double*>(bp + hp->score_off)[u];
          if ((code & 3) == SP_DEC_DELAY)  // configurator.py:275-278: slack - latency
            wait = __dsub_rn(sk, reinterpret_cast<const double*>(bp + hp->lat_off)[u]);
        }
        const int d = d0 + c;
        io.out_idx[d] = idx;
        io.out_code[d] = code;
        io.out_fill[d] = s_sup[c];
        io.out_obj[d] = obj;
        io.out_slack[d] = sk;
        io.out_wait[d] = wait;
        s += r32;
        if (s >= g.n_src) s -= g.n_src;
      }
      continue;
    }
    if (!out_stage) continue;
    __syncwarp();
    for (int c = lane; c < nd; c += 32) {  // coalesced stores of the group's decisions
      io.out_idx[d0 + c] = o_idx[c];
      io.out_code[d0 + c] = o_code[c];
      if (io.out_fill) io.out_fill[d0 + c] = o_fill[c];
      if (io.out_obj) io.out_obj[d0 + c] = o_obj[c];
      if (io.out_slack) io.out_slack[d0 + c] = o_sl[c];
      if (io.out_wait) io.out_wait[d0 + c] = o_wait[c];
    }
  }
}
