// sp_plan_cluster.cu — the staircase decision plan built by ONE thread-block-cluster kernel.
//
// Same image, byte for byte, as the multi-kernel builder in sp_plan.cu (checked section by
// section against it and against the CPU restatement oracle/plan.py), but ~20 kernels become
// one launch of an 8-CTA cluster and no global sort over all M entries is needed:
//
//   The image only depends on the per-(kind, batch lane) staircases.  Within one lane, with the
//   entries in (latency, index) order, the feasible-side best entry for "lat < slack" changes
//   only at P-records (entries whose argmin key (cost, res, id_rank), configurator.py:229-237,
//   is strictly below every earlier entry's) and the penalized-side best only at S-records
//   (key (costpen, cost, res, id_rank) strictly below every later entry's).  A kind's rows are
//   therefore exactly row 0 (slack <= every latency) plus one row per distinct latency of a
//   record of any of its lanes; a row's lane value is the last P-record at or below the row's
//   latency and the first S-record above it.  Candidates are the records that some row uses.
//
//   phase 1  (CTA per segment = (kind, lane)): bitonic sort of the segment by (lat, index) in
//            shared memory, cost / costpen (configurator.py:224-225), exclusive prefix-argmin
//            scan (P-records) and suffix-argmin scan (S-records), record lists -> global scratch
//   cluster barrier
//   phase 2  CTA 0: the unified candidate order (score, cost, res, id_rank, side) by a bitonic
//            sort -> candidate ids; kind CTAs: the distinct record latencies of their kind,
//            sorted -> row thresholds and row counts
//   cluster barrier
//   phase 3  every CTA derives the image layout from the row / candidate counts; CTA 0 writes
//            header, batch lookup table and candidate records; kind CTAs write thresholds,
//            bucket tables and the rows (per row and lane two binary searches in the lane's
//            record lists, then the interval minima).
//
// Exactness conventions mirror sp_plan.cu's builder: latency and cost orders use the monotone
// u64 key of the double (so -0.0 sorts before +0.0), res and scores compare numerically, a
// latency group is a run of numerically equal latencies and its threshold is the latency of its
// last entry in (key, index) order.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "sp_internal.cuh"

namespace sp {

namespace {

constexpr int kPcThreads = 1024;
constexpr int kPcCluster = 8;
constexpr int kPcMaxSeg = 2048;       // entries of one (kind, lane) segment
constexpr int kPcMaxKind = 8192;      // entries of one kind (its records are sorted in smem)
constexpr int kPcCandSmem = 4096;     // candidates sorted in shared memory (else global)
constexpr uint32_t kFlagBit = 0x80000000u;
constexpr uint32_t kInfPc = 0xFFFFFFFFu;
constexpr int kPcRowChunk = 16384;  // lane values staged per row chunk (64 KB)

__device__ __forceinline__ uint64_t okey(double x) {
  return order_key(static_cast<uint64_t>(__double_as_longlong(x)));
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int pow2ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Bitonic sort of an index array (length N2, a power of two; -1 pads sort last) with a strict
// order on real indices; one __syncthreads per stage.
template <class Less>
__device__ void bitonic_idx(int32_t* ix, int N2, Less less) {
  const int half = N2 >> 1;
  for (int k = 2; k <= N2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < half; i += blockDim.x) {
        const int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
        const bool up = (lo & k) == 0;
        const int a = ix[lo], b = ix[hi];
        const bool b_lt_a = a < 0 ? b >= 0 : (b >= 0 && less(b, a));
        const bool a_lt_b = b < 0 ? a >= 0 : (a >= 0 && less(a, b));
        if (up ? b_lt_a : a_lt_b) {
          ix[lo] = b;
          ix[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Bitonic sort of u64 keys in place (pads = ~0).
__device__ void bitonic_u64(uint64_t* a, int N2) {
  const int half = N2 >> 1;
  for (int k = 2; k <= N2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < half; i += blockDim.x) {
        const int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
        const bool up = (lo & k) == 0;
        const uint64_t x = a[lo], y = a[hi];
        if (up ? (y < x) : (x < y)) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

// Block-wide exclusive sum (blockDim.x == kPcThreads); *total = sum over the block.
__device__ int pc_excl_sum(int v, int* s_w, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int y = s_w[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y += z;
    }
    s_w[lane] = y;
  }
  __syncthreads();
  const int r = (w ? s_w[w - 1] : 0) + x - v;
  *total = s_w[31];
  __syncthreads();
  return r;
}

// Exclusive argmin scan over positions in thread-chunk order: each thread passes its chunk's
// best position (or -1); returns the best position of all earlier chunks (or -1).  `better`
// picks the preferred of two positions (either may be -1).  `rev` numbers the chunks from the
// block's end (suffix scans).
template <class Better>
__device__ int pc_excl_best(int v, bool rev, int* s_w, Better better) {
  const int r = rev ? (int)(blockDim.x - 1 - threadIdx.x) : (int)threadIdx.x;
  const int lane = r & 31, w = r >> 5;
  // warp inclusive scan in rank order (rank r's lane order is reversed when rev)
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = rev ? __shfl_down_sync(0xffffffffu, x, off) : __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x = better(y, x);
  }
  const int ex_in = rev ? __shfl_down_sync(0xffffffffu, x, 1) : __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int y = s_w[threadIdx.x];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, off);
      if ((int)threadIdx.x >= off) y = better(z, y);
    }
    s_w[32 + threadIdx.x] = y;  // inclusive over warps in rank order
  }
  __syncthreads();
  int ex = lane == 0 ? -1 : ex_in;
  if (w > 0) ex = better(s_w[32 + w - 1], ex);
  __syncthreads();
  return ex;
}

// Bitonic sort of N2 (key, val) pairs (power of two, N2 <= E * blockDim.x) held E per thread in
// registers, element i = threadIdx.x + q * blockDim.x, ascending by (key, val); pads carry
// (~0, ~0).  Stages with partner distance < 32 exchange through warp shuffles, distances that
// cross warps through shared memory (sk / sv, E * blockDim.x entries), distances >= blockDim.x
// inside the thread.  Only the first N2 elements take part.
template <int E>
__device__ void reg_bitonic(uint64_t (&key)[E], uint32_t (&val)[E], int N2, uint64_t* sk,
                            uint32_t* sv) {
  const int T = blockDim.x, t = threadIdx.x;
  for (int k = 2; k <= N2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= T) {
        const int qj = j / T;
#pragma unroll
        for (int m = 1; m < E; m <<= 1) {  // static register indices: m == qj
          if (m != qj) continue;
#pragma unroll
          for (int q = 0; q < E; ++q) {
            if (q & m) continue;
            const int q2 = q | m;
            const int i = t + q * T;
            if (i >= N2) continue;
            const bool up = (i & k) == 0;
            const bool gt = key[q] > key[q2] || (key[q] == key[q2] && val[q] > val[q2]);
            if (gt == up) {
              const uint64_t tk = key[q];
              key[q] = key[q2];
              key[q2] = tk;
              const uint32_t tv = val[q];
              val[q] = val[q2];
              val[q2] = tv;
            }
          }
        }
      } else if (j >= 32) {
#pragma unroll
        for (int q = 0; q < E; ++q) {
          sk[t + q * T] = key[q];
          sv[t + q * T] = val[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int i = t + q * T;
          if (i < N2) {
            const int p = i ^ j;
            const uint64_t pk = sk[p];
            const uint32_t pv = sv[p];
            const bool want_min = ((i & j) == 0) == ((i & k) == 0);
            const bool pless = pk < key[q] || (pk == key[q] && pv < val[q]);
            if (pless == want_min) {
              key[q] = pk;
              val[q] = pv;
            }
          }
        }
        __syncthreads();
      } else {
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int i = t + q * T;
          const uint64_t pk = __shfl_xor_sync(0xffffffffu, key[q], j);
          const uint32_t pv = __shfl_xor_sync(0xffffffffu, val[q], j);
          const bool want_min = ((i & j) == 0) == ((i & k) == 0);
          const bool pless = pk < key[q] || (pk == key[q] && pv < val[q]);
          if (i < N2 && pless == want_min) {
            key[q] = pk;
            val[q] = pv;
          }
        }
      }
    }
  }
}

// Block scan in rank order (rank = threadIdx.x, or its mirror when rev) of "best position":
// returns the best of all earlier ranks (-1: none); *total = best of the whole block.
template <class Better>
__device__ int blk_best(int v, bool rev, int* s_w, int* total, Better better) {
  const int r = rev ? (int)(blockDim.x - 1 - threadIdx.x) : (int)threadIdx.x;
  const int lane = r & 31, w = r >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = rev ? __shfl_down_sync(0xffffffffu, x, off) : __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x = better(y, x);
  }
  const int ex_in = rev ? __shfl_down_sync(0xffffffffu, x, 1) : __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    int y = s_w[threadIdx.x];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, off);
      if ((int)threadIdx.x >= off) y = better(z, y);
    }
    s_w[32 + threadIdx.x] = y;
  }
  __syncthreads();
  int ex = lane == 0 ? -1 : ex_in;
  if (w > 0) ex = better(s_w[32 + w - 1], ex);
  *total = s_w[63];
  __syncthreads();
  return ex;
}

struct PcSegDev {
  int32_t off, n, kind, lane;
};
constexpr int kPcMaxSegs = 128;
// per-CTA shared copies of the static segment table and of the phase-1 counts
struct PcShared {
  PcSegDev seg[kPcMaxSegs];
  int32_t cnt[kPcMaxSegs * 4];
};

struct PcArgs {
  int M, K, nB, W, nseg;
  const PcSegDev* seg;
  int32_t* ord;                 // M: per segment slice, its entries in (lat, index) order
  const double *lat, *res, *pool, *price;
  const int32_t *batch, *kind, *id_rank;
  double alpha;
  double *cost, *costpen;
  uint8_t* image;
  int64_t image_cap;
  int32_t* status;
  // global scratch (carved by the host); per segment slices at seg.off
  double *rp_lat, *rs_lat;      // P / S record latencies (position order)
  uint32_t *rp_uid, *rs_uid;    // candidate id of a record (kInfPc: not a candidate)
  // candidates (P: final P-records, S: first S-records), compact per segment slice
  uint64_t *cp_key, *cs_key;    // order key of the score (cost / costpen)
  uint64_t *cp_ck, *cs_ck;      // order key of the cost
  double *cp_res, *cs_res;
  double *cp_lat, *cs_lat;
  int32_t *cp_idr, *cs_idr;
  int32_t *cp_er, *cs_er;       // entry | record index << 16
  int32_t* seg_cnt;             // nseg x 4: np, ns, ncp, ncs
  double* thr;                  // M + K: per kind thresholds at base_k + k
  int32_t* kinfo;               // [2k] rows, [2k+1] has +0.0 latency; [16], [17] ncp, ncs
  double* crec;                 // 2M x 3 (score, lat, meta|batch): candidate records by id
  double* gkey;                 // candidate keys when sorted outside shared memory
  int32_t* gix;
  int32_t base[kMaxKinds], count[kMaxKinds];
  int32_t seg_lo[kMaxKinds + 1];  // segments of kind k: [seg_lo[k], seg_lo[k+1])
  PlanHdr hdr;                    // magic, M, nB, W, K, batch_vals
  int debug;
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double key_double(uint64_t u) {  // inverse of okey
  const uint64_t b = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)b);
}

// layout of the image from the row / candidate counts (every CTA computes the same)
__device__ void pc_layout(const PcArgs& a, const int32_t* rows, const double* thr2, int ncp,
                          int ncs, PlanHdr& hdr) {
  hdr = a.hdr;
  hdr.row_stride = ((a.nB * (a.nB + 1) + 3) / 4) * 4;
  int off = (int)sizeof(PlanHdr);
  int maxB = 0;
  for (int b = 0; b < a.nB; ++b) maxB = max(maxB, hdr.batch_vals[b]);
  hdr.lut_n = (maxB + 2 <= kMaxLut) ? maxB + 2 : 0;
  hdr.lut_off = off;
  off += ((hdr.lut_n * 2 + 15) / 16) * 16;
  for (int k = 0; k < kMaxKinds; ++k) {
    KindDesc d;
    memset(&d, 0, sizeof(d));
    const int R = k < a.K ? rows[k] : 0;
    d.R = R;
    if (R > 0) {
      int nbk = 1, shift = 0;
      uint32_t kmin = 0;
      if (R >= 2) {
        const double t1 = thr2[2 * k];
        kmin = (uint32_t)__double2hiint(t1);
        const uint32_t kmax = (uint32_t)__double2hiint(thr2[2 * k + 1]);
        while (nbk < 2 * (R - 1) && nbk < kMaxBuckets) nbk <<= 1;
        while (((kmax - kmin) >> shift) >= (uint32_t)nbk) ++shift;
        d.pad[0] = !(t1 > 0.0);
      }
      d.kmin_hi = kmin;
      d.nb1_shift = (uint32_t)(nbk - 1) | ((uint32_t)shift << 16);
      d.thr_off = off;
      off += ((R * 8 + 15) / 16) * 16;
      d.rows_off = off;
      off += ((R * hdr.row_stride + 15) / 16) * 16;
      d.bkt_off = off;
      off += ((nbk * 4 + 15) / 16) * 16;
    }
    hdr.kd[k] = d;
  }
  hdr.ncp = ncp;
  hdr.ncs = ncs;
  hdr.score_off = off;
  off += (ncp + ncs) * 8;
  hdr.lat_off = off;
  off += (ncp + ncs) * 8;
  hdr.recb_off = off;
  off += (((ncp + ncs) * (int)sizeof(CandB) + 15) / 16) * 16;
  hdr.total_bytes = off;
  const bool ok = off <= a.image_cap && ncp + ncs < (int)kNone16;
  if (!ok) hdr.magic = 0;
}

// ---- phase 1: one (kind, lane) segment -----------------------------------------------------
template <int E>
__device__ void pc_segment(const PcArgs& a, const PcShared& S, int s, uint8_t* smem, int* s_w) {
  const PcSegDev sg = S.seg[s];
  const int n = sg.n, off = sg.off, N2 = pow2ceil(max(n, 2));
  const int T = blockDim.x, t = threadIdx.x;
  const int NE = E * T;
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);    // NE  (sort exchange)
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + NE);  // NE
  // position-order arrays (p < n)
  uint64_t* pck = reinterpret_cast<uint64_t*>(sv + NE);
  uint64_t* pcpk = pck + NE;
  double* pres = reinterpret_cast<double*>(pcpk + NE);
  double* plat = pres + NE;
  int32_t* pe = reinterpret_cast<int32_t*>(plat + NE);
  int32_t* pidr = pe + NE;
  int32_t* lP = pidr + NE;  // record positions
  int32_t* lS = lP + NE;
  // 1. the cached (lat, index) order of the previous build; re-sorted only if it no longer
  //    holds (a latency changed)
  uint64_t key[E];
  uint32_t val[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int i = t + q * T;
    if (i < n) {
      val[q] = (uint32_t)a.ord[off + i];
      key[q] = okey(a.lat[val[q]]);
    } else {
      val[q] = 0xFFFFFFFFu;
      key[q] = ~0ull;
    }
    sk[i] = key[q];
    sv[i] = val[q];
  }
  __syncthreads();
  bool bad = false;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int i = t + q * T;
    if (i + 1 < n) bad |= sk[i] > sk[i + 1] || (sk[i] == sk[i + 1] && sv[i] > sv[i + 1]);
  }
  if (__syncthreads_or(bad)) {
    reg_bitonic<E>(key, val, N2, sk, sv);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int i = t + q * T;
      if (i < n) a.ord[off + i] = (int32_t)val[q];
    }
  }
  // 2. per position: cost / costpen (configurator.py:224-225, numpy order, no FMA), keys
  bool pos_zero = false;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int p = t + q * T;
    if (p < n) {
      const int e = (int)val[q];
      const double L = a.lat[e], R = a.res[e], B = (double)a.batch[e], P = a.pool[e],
                   pr = a.price[e];
      const double c = __ddiv_rn(__dmul_rn(__dmul_rn(R, L), pr), B);
      const double pen = __dmul_rn(a.alpha, __ddiv_rn(__dmul_rn(L, R), __dmul_rn(B, P)));
      const double cp = __dadd_rn(c, pen);
      a.cost[e] = c;
      a.costpen[e] = cp;
      pe[p] = e;
      plat[p] = L;
      pck[p] = okey(c);
      pcpk[p] = okey(cp);
      pres[p] = R;
      pidr[p] = a.id_rank[e];
      pos_zero |= __double_as_longlong(L) == 0;
    }
  }
  if (__syncthreads_or(pos_zero) && t == 0) atomicOr(&a.kinfo[2 * sg.kind + 1], 1);
  // Key1 (the r1 order: cost key, res, id_rank) and Key2 (costpen key, then Key1)
  auto less1 = [&](int x, int y) {
    if (pck[x] != pck[y]) return pck[x] < pck[y];
    if (pres[x] != pres[y]) return pres[x] < pres[y];
    return pidr[x] < pidr[y];
  };
  auto less2 = [&](int x, int y) {
    if (pcpk[x] != pcpk[y]) return pcpk[x] < pcpk[y];
    return less1(x, y);
  };
  auto best1 = [&](int x, int y) { return x < 0 ? y : (y < 0 ? x : (less1(y, x) ? y : x)); };
  auto best2 = [&](int x, int y) { return x < 0 ? y : (y < 0 ? x : (less2(y, x) ? y : x)); };
  // 3. P-records (strictly below every earlier position's Key1), S-records (strictly below
  //    every later position's Key2); positions t + q*T, chunks in q order
  bool fP[E], fS[E];
  {
    int carry = -1;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int p = t + q * T;
      int tot;
      int ex = blk_best(p < n ? p : -1, false, s_w, &tot, best1);
      ex = best1(carry, ex);
      fP[q] = p < n && (ex < 0 || less1(p, ex));
      carry = best1(carry, tot);
    }
    carry = -1;
#pragma unroll
    for (int q = E - 1; q >= 0; --q) {
      const int p = t + q * T;
      int tot;
      int ex = blk_best(p < n ? p : -1, true, s_w, &tot, best2);
      ex = best2(carry, ex);
      fS[q] = p < n && (ex < 0 || less2(p, ex));
      carry = best2(carry, tot);
    }
  }
  // 4. record lists in position order
  int nP = 0, nS = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    int tp, ts;
    const int op = pc_excl_sum(fP[q] ? 1 : 0, s_w, &tp);
    const int os = pc_excl_sum(fS[q] ? 1 : 0, s_w, &ts);
    if (fP[q]) lP[nP + op] = t + q * T;
    if (fS[q]) lS[nS + os] = t + q * T;
    nP += tp;
    nS += ts;
  }
  __syncthreads();
  // 5. a P-record is a candidate iff no later P-record has the same latency (it is its own
  //    row's lane value); an S-record iff no earlier S-record has the same latency.  Records
  //    and candidates (with their full argmin keys) go to global scratch.
  int ncp = 0, ncs = 0;
  for (int j0 = 0; j0 < max(nP, nS); j0 += T) {
    const int j = j0 + t;
    const bool fin = j < nP && (j + 1 == nP || plat[lP[j + 1]] != plat[lP[j]]);
    const bool fst = j < nS && (j == 0 || plat[lS[j - 1]] != plat[lS[j]]);
    int tp, ts;
    const int op = pc_excl_sum(fin ? 1 : 0, s_w, &tp);
    const int os = pc_excl_sum(fst ? 1 : 0, s_w, &ts);
    if (j < nP) {
      const int p = lP[j];
      a.rp_lat[off + j] = plat[p];
      a.rp_uid[off + j] = kInfPc;
      if (fin) {
        const int c = off + ncp + op;
        a.cp_key[c] = pck[p];
        a.cp_ck[c] = pck[p];
        a.cp_res[c] = pres[p];
        a.cp_lat[c] = plat[p];
        a.cp_idr[c] = pidr[p];
        a.cp_er[c] = pe[p] | (j << 16);
      }
    }
    if (j < nS) {
      const int p = lS[j];
      a.rs_lat[off + j] = plat[p];
      a.rs_uid[off + j] = kInfPc;
      if (fst) {
        const int c = off + ncs + os;
        a.cs_key[c] = pcpk[p];
        a.cs_ck[c] = pck[p];
        a.cs_res[c] = pres[p];
        a.cs_lat[c] = plat[p];
        a.cs_idr[c] = pidr[p];
        a.cs_er[c] = pe[p] | (j << 16);
      }
    }
    ncp += tp;
    ncs += ts;
  }
  if (t == 0) {
    a.seg_cnt[4 * s + 0] = nP;
    a.seg_cnt[4 * s + 1] = nS;
    a.seg_cnt[4 * s + 2] = ncp;
    a.seg_cnt[4 * s + 3] = ncs;
  }
  __syncthreads();
}

// ---- phase 2a: unified candidate ids (CTA 0) -------------------------------------------------
// order (score, cost key, res, id_rank, side): the reference argmin key with the feasible side
// first on exact ties (sp_plan.cu k_fin_merge).  Sorted by (score key, candidate) in registers,
// then each run of numerically equal scores re-ordered by the rest of the key.  Outputs: the
// candidate id of every candidate record (rp_uid / rs_uid) and the candidate records by id
// (crec: score, latency, meta | batch).
struct CandRef {
  int seg, slot;
  bool sideP;
};
__device__ __forceinline__ CandRef cand_ref(const PcArgs& a, const PcShared& S, const int* s_off, int ncp, int c) {
  CandRef r;
  r.sideP = c < ncp;
  const int cc = r.sideP ? c : c - ncp;
  const int* so = r.sideP ? s_off : s_off + 129;
  int lo = 0, hi = a.nseg;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (so[mid] <= cc) lo = mid + 1; else hi = mid;
  }
  r.seg = lo - 1;
  r.slot = S.seg[r.seg].off + (cc - so[r.seg]);
  return r;
}

__device__ __forceinline__ void cand_out(const PcArgs& a, const PcShared& S, const CandRef& r, int u) {
  const PcSegDev sg = S.seg[r.seg];
  const int er = r.sideP ? a.cp_er[r.slot] : a.cs_er[r.slot];
  const int e = er & 0xFFFF, rec = er >> 16;
  (r.sideP ? a.rp_uid : a.rs_uid)[sg.off + rec] = (uint32_t)u;
  const double sc = key_double(r.sideP ? a.cp_key[r.slot] : a.cs_key[r.slot]);
  const double lt = r.sideP ? a.cp_lat[r.slot] : a.cs_lat[r.slot];
  CandB b;
  b.meta = (uint32_t)e | ((r.sideP ? 1u : 0u) << 16) | ((uint32_t)sg.kind << 17);
  b.batch = a.hdr.batch_vals[sg.lane];
  a.crec[3 * u + 0] = sc;
  a.crec[3 * u + 1] = lt;
  a.crec[3 * u + 2] = __longlong_as_double(*reinterpret_cast<const long long*>(&b));
}

template <int E>
__device__ void pc_cand_sort(const PcArgs& a, const PcShared& S, int ncp, int nc, const int* s_off, uint8_t* smem) {
  const int T = blockDim.x, t = threadIdx.x, NE = E * T;
  const int N2 = pow2ceil(max(nc, 2));
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + NE);
  uint64_t* sck = reinterpret_cast<uint64_t*>(sv + NE);  // by candidate: cost key, res, id_rank
  double* sres = reinterpret_cast<double*>(sck + NE);
  int32_t* sidr = reinterpret_cast<int32_t*>(sres + NE);
  uint64_t key[E];
  uint32_t val[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int c = t + q * T;
    key[q] = ~0ull;
    val[q] = 0xFFFFFFFFu;
    if (c < nc) {
      const CandRef r = cand_ref(a, S, s_off, ncp, c);
      key[q] = r.sideP ? a.cp_key[r.slot] : a.cs_key[r.slot];
      sck[c] = r.sideP ? a.cp_ck[r.slot] : a.cs_ck[r.slot];
      sres[c] = r.sideP ? a.cp_res[r.slot] : a.cs_res[r.slot];
      sidr[c] = r.sideP ? a.cp_idr[r.slot] : a.cs_idr[r.slot];
      val[q] = (uint32_t)c;
    }
  }
  reg_bitonic<E>(key, val, N2, sk, sv);
#pragma unroll
  for (int q = 0; q < E; ++q) {
    sk[t + q * T] = key[q];
    sv[t + q * T] = val[q];
  }
  __syncthreads();
  // runs of numerically equal scores: insertion sort by (cost key, res, id_rank, side)
  auto lessc = [&](uint32_t x, uint32_t y) {
    if (sck[x] != sck[y]) return sck[x] < sck[y];
    if (sres[x] != sres[y]) return sres[x] < sres[y];
    if (sidr[x] != sidr[y]) return sidr[x] < sidr[y];
    return (int)x < ncp && (int)y >= ncp;
  };
  for (int u = t; u < nc; u += T) {
    const double su = key_double(sk[u]);
    if (u > 0 && key_double(sk[u - 1]) == su) continue;
    if (u + 1 >= nc || key_double(sk[u + 1]) != su) continue;
    int end = u + 1;
    while (end < nc && key_double(sk[end]) == su) ++end;
    for (int i = u + 1; i < end; ++i) {
      const uint32_t x = sv[i];
      int j = i - 1;
      while (j >= u && lessc(x, sv[j])) {
        sv[j + 1] = sv[j];
        --j;
      }
      sv[j + 1] = x;
    }
  }
  __syncthreads();
  for (int u = t; u < nc; u += T) cand_out(a, S, cand_ref(a, S, s_off, ncp, (int)sv[u]), u);
  __syncthreads();
}

__device__ void pc_candidates(const PcArgs& a, const PcShared& S, uint8_t* smem, int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  __shared__ int s_off[2 * 129];
  if (t == 0) {
    int op = 0, os = 0;
    for (int s = 0; s < a.nseg; ++s) {
      s_off[s] = op;
      s_off[129 + s] = os;
      op += S.cnt[4 * s + 2];
      os += S.cnt[4 * s + 3];
    }
    s_off[a.nseg] = op;
    s_off[129 + a.nseg] = os;
    a.kinfo[16] = op;
    a.kinfo[17] = os;
  }
  __syncthreads();
  const int ncp = s_off[a.nseg], nc = ncp + s_off[129 + a.nseg];
  if (nc <= T) {
    pc_cand_sort<1>(a, S, ncp, nc, s_off, smem);
    return;
  }
  if (nc <= 2 * T) {
    pc_cand_sort<2>(a, S, ncp, nc, s_off, smem);
    return;
  }
  // large candidate counts: bitonic sort of candidate indices over global scratch
  const int N2 = pow2ceil(nc);
  int32_t* ix = a.gix;
  uint64_t* ks = reinterpret_cast<uint64_t*>(a.gkey);
  uint64_t* kc = reinterpret_cast<uint64_t*>(a.gkey + N2);
  double* kr = a.gkey + 2 * N2;
  int32_t* ki = reinterpret_cast<int32_t*>(a.gkey + 3 * N2);
  for (int c = t; c < N2; c += T) {
    ix[c] = -1;
    if (c < nc) {
      const CandRef r = cand_ref(a, S, s_off, ncp, c);
      ks[c] = r.sideP ? a.cp_key[r.slot] : a.cs_key[r.slot];
      kc[c] = r.sideP ? a.cp_ck[r.slot] : a.cs_ck[r.slot];
      kr[c] = r.sideP ? a.cp_res[r.slot] : a.cs_res[r.slot];
      ki[c] = r.sideP ? a.cp_idr[r.slot] : a.cs_idr[r.slot];
      ix[c] = c;
    }
  }
  __syncthreads();
  bitonic_idx(ix, N2, [&](int x, int y) {
    const double sx = key_double(ks[x]), sy = key_double(ks[y]);
    if (sx != sy) return sx < sy;
    if (kc[x] != kc[y]) return kc[x] < kc[y];
    if (kr[x] != kr[y]) return kr[x] < kr[y];
    if (ki[x] != ki[y]) return ki[x] < ki[y];
    return x < ncp && y >= ncp;
  });
  for (int u = t; u < nc; u += T) cand_out(a, S, cand_ref(a, S, s_off, ncp, ix[u]), u);
  __syncthreads();
}

// ---- phase 2b: a kind's thresholds and its record lists -----------------------------------
// Every CTA working on kind k stages the kind's records (per lane: the P list, then the S list,
// latencies in position order) in shared memory and sorts their latencies: row 0 is -inf, row
// r the r-th distinct latency (a group's threshold is its last entry's latency in key order: for
// the zero group +0.0 whenever the kind has a +0.0 latency, -0.0 otherwise).  Slot 0 publishes
// the row count and the thresholds (global) for every CTA's layout.
struct KindStage {
  int nr, R;          // records, rows
  int lane[kMaxB][4];  // per lane: P start, P count, S start, S count (record index space)
  bool staged;        // records and thresholds are in shared memory
};
constexpr int kPcStageMax = 4096;  // records staged in shared memory per kind

template <int E>
__device__ int pc_thr_sort(int nr, const double* L, double* thr, bool has_pz, uint8_t* scratch,
                           int* s_w) {
  const int T = blockDim.x, t = threadIdx.x, NE = E * T;
  const int N2 = pow2ceil(max(nr, 2));
  uint64_t* sk = reinterpret_cast<uint64_t*>(scratch);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + NE);
  uint64_t key[E];
  uint32_t val[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int j = t + q * T;
    key[q] = j < nr ? okey(L[j]) : ~0ull;
    val[q] = (uint32_t)j;
  }
  reg_bitonic<E>(key, val, N2, sk, sv);
#pragma unroll
  for (int q = 0; q < E; ++q) sk[t + q * T] = key[q];
  __syncthreads();
  int o = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int j = t + q * T;
    const bool st = j < nr && (j == 0 || key_double(sk[j]) != key_double(sk[j - 1]));
    int tot;
    const int ex = pc_excl_sum(st ? 1 : 0, s_w, &tot);
    if (st) {
      double v = key_double(sk[j]);
      if (v == 0.0) v = has_pz ? 0.0 : -0.0;
      thr[1 + o + ex] = v;
    }
    o += tot;
  }
  if (t == 0) thr[0] = -INFINITY;
  __syncthreads();
  return o + 1;
}

__device__ void pc_kind_stage(const PcArgs& a, const PcShared& S, int k, bool publish, KindStage& ks,
                              uint8_t* smem, int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const int ext = a.base[k] + k;
  const int s0 = a.seg_lo[k], s1 = a.seg_lo[k + 1];
  if (t == 0) {
    int acc = 0;
    for (int b = 0; b < kMaxB; ++b) ks.lane[b][0] = ks.lane[b][1] = ks.lane[b][2] = ks.lane[b][3] = 0;
    for (int s = s0; s < s1; ++s) {
      const int b = S.seg[s].lane;
      ks.lane[b][0] = acc;
      ks.lane[b][1] = S.cnt[4 * s + 0];
      acc += ks.lane[b][1];
      ks.lane[b][2] = acc;
      ks.lane[b][3] = S.cnt[4 * s + 1];
      acc += ks.lane[b][3];
    }
    ks.nr = acc;
    ks.staged = acc <= kPcStageMax;
  }
  __syncthreads();
  const int nr = ks.nr;
  if (a.count[k] == 0) {
    if (t == 0) ks.R = 0;
    if (publish && t == 0) a.kinfo[2 * k] = 0;
    __syncthreads();
    return;
  }
  const bool has_pz = a.kinfo[2 * k + 1] != 0;
  if (ks.staged) {
    // smem: L[nr] record latencies, U[nr] candidate ids (phase 3), thr[nr + 1], sort scratch
    double* L = reinterpret_cast<double*>(smem);
    double* thr = L + kPcStageMax;
    uint8_t* scratch = reinterpret_cast<uint8_t*>(thr + kPcStageMax + 1) + 8;
    for (int s = s0; s < s1; ++s) {
      const int b = S.seg[s].lane, off = S.seg[s].off;
      for (int j = t; j < ks.lane[b][1]; j += T) L[ks.lane[b][0] + j] = a.rp_lat[off + j];
      for (int j = t; j < ks.lane[b][3]; j += T) L[ks.lane[b][2] + j] = a.rs_lat[off + j];
    }
    __syncthreads();
    const int R = nr <= T ? pc_thr_sort<1>(nr, L, thr, has_pz, scratch, s_w)
                          : pc_thr_sort<4>(nr, L, thr, has_pz, scratch, s_w);
    if (t == 0) ks.R = R;
    if (publish) {
      for (int r = t; r < R; r += T) a.thr[ext + r] = thr[r];
      if (t == 0) a.kinfo[2 * k] = R;
    }
    __syncthreads();
    return;
  }
  // large record sets: shared-memory bitonic sort of the keys, thresholds through global
  const int N2 = pow2ceil(nr);
  uint64_t* key = reinterpret_cast<uint64_t*>(smem);
  for (int j = t; j < N2; j += T) {
    uint64_t v = ~0ull;
    if (j < nr) {
      int b = 0;
      while (b + 1 < kMaxB && !(j >= ks.lane[b][0] && j < ks.lane[b][2] + ks.lane[b][3])) ++b;
      int s = s0;
      while (S.seg[s].lane != b) ++s;
      v = okey(j < ks.lane[b][2] ? a.rp_lat[S.seg[s].off + j - ks.lane[b][0]]
                                 : a.rs_lat[S.seg[s].off + j - ks.lane[b][2]]);
    }
    key[j] = v;
  }
  __syncthreads();
  bitonic_u64(key, N2);
  const int P = (nr + T - 1) / T;
  const int j0 = min(t * P, nr), j1 = min(j0 + P, nr);
  int cnt = 0;
  for (int j = j0; j < j1; ++j) cnt += j == 0 || key_double(key[j]) != key_double(key[j - 1]);
  int nd = 0;
  int o = pc_excl_sum(cnt, s_w, &nd);
  if (publish) {
    for (int j = j0; j < j1; ++j) {
      if (j == 0 || key_double(key[j]) != key_double(key[j - 1])) {
        double v = key_double(key[j]);
        if (v == 0.0) v = has_pz ? 0.0 : -0.0;
        a.thr[ext + 1 + o++] = v;
      }
    }
    if (t == 0) {
      a.thr[ext] = -INFINITY;
      a.kinfo[2 * k] = 1 + nd;
    }
  }
  if (t == 0) ks.R = 1 + nd;
  __syncthreads();
}

// ---- phase 3 ---------------------------------------------------------------------------------
__device__ void pc_write_common(const PcArgs& a, const PlanHdr& H) {
  const int T = blockDim.x, t = threadIdx.x;
  if (t < (int)(sizeof(PlanHdr) / 4))
    reinterpret_cast<uint32_t*>(a.image)[t] = reinterpret_cast<const uint32_t*>(&H)[t];
  if (H.magic != kPlanMagic) return;
  uint16_t* lut = reinterpret_cast<uint16_t*>(a.image + H.lut_off);
  for (int v = t; v < H.lut_n; v += T) {
    int lo = 0, le = 0;
    for (int b = 0; b < H.nB; ++b) {
      lo += H.batch_vals[b] < v;
      le += H.batch_vals[b] <= v;
    }
    lut[v] = (uint16_t)(lo | (le << 8));
  }
  double* rscore = reinterpret_cast<double*>(a.image + H.score_off);
  double* rlat = reinterpret_cast<double*>(a.image + H.lat_off);
  double* recb = reinterpret_cast<double*>(a.image + H.recb_off);  // CandB (8 B) as a double
  const int nc = H.ncp + H.ncs;
  for (int u = t; u < nc; u += T) {
    rscore[u] = a.crec[3 * u + 0];
    rlat[u] = a.crec[3 * u + 1];
    recb[u] = a.crec[3 * u + 2];
  }
}

// rows [r0, r1) of kind k; `first` also writes the bucket table.  Lane b of row r = min(the
// candidate id of the last P-record of lane b with lat <= thr[r], of the first S-record with
// lat > thr[r]); stored as the minimum over every lane interval [lo, hi] at tri(lo) + hi - lo.
__device__ void pc_write_kind(const PcArgs& a, const PcShared& S, const PlanHdr& H, int k, int r0,
                              int r1, bool first, const KindStage& ks, uint8_t* smem, int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const KindDesc d = H.kd[k];
  const int R = d.R;
  if (R == 0 || H.magic != kPlanMagic) return;
  const int ext = a.base[k] + k;
  const int s0 = a.seg_lo[k], s1 = a.seg_lo[k + 1];
  const bool staged = ks.staged;
  double* L = reinterpret_cast<double*>(smem);
  const double* thr = staged ? L + kPcStageMax : a.thr + ext;
  uint32_t* U = reinterpret_cast<uint32_t*>(const_cast<double*>(L + 2 * kPcStageMax + 1) + 1);
  uint8_t* work = reinterpret_cast<uint8_t*>(U + kPcStageMax);
  double* ithr = reinterpret_cast<double*>(a.image + d.thr_off);
  for (int r = r0 + t; r < r1; r += T) ithr[r] = thr[r];
  if (first) {  // bucket table: histogram + block scan (as sp_plan.cu k_fin_buckets)
    uint32_t* s_h = reinterpret_cast<uint32_t*>(work);
    uint32_t* bkt = reinterpret_cast<uint32_t*>(a.image + d.bkt_off);
    const int nbk = (int)(d.nb1_shift & 0xFFFFu) + 1, shift = (int)(d.nb1_shift >> 16);
    for (int b = t; b < nbk; b += T) s_h[b] = 0u;
    __syncthreads();
    for (int j = 1 + t; j < R; j += T) {
      const uint32_t kk = (uint32_t)__double2hiint(thr[j]);
      atomicAdd(&s_h[min((kk - d.kmin_hi) >> shift, (uint32_t)(nbk - 1))], 1u);
    }
    __syncthreads();
    const int per = (nbk + T - 1) / T;
    const int b0 = min(t * per, nbk), b1 = min(b0 + per, nbk);
    int loc = 0;
    for (int b = b0; b < b1; ++b) loc += (int)s_h[b];
    int tot = 0;
    int below = pc_excl_sum(loc, s_w, &tot);
    for (int b = b0; b < b1; ++b) {
      const uint32_t c = s_h[b];
      bkt[b] = (uint32_t)below | (c << 16);
      below += (int)c;
    }
    __syncthreads();
  }
  if (r1 <= r0) return;
  const int nB = H.nB;
  if (staged) {  // the candidate ids of the staged records (written by CTA 0 in phase 2)
    for (int s = s0; s < s1; ++s) {
      const int b = S.seg[s].lane, off = S.seg[s].off;
      for (int j = t; j < ks.lane[b][1]; j += T) U[ks.lane[b][0] + j] = a.rp_uid[off + j];
      for (int j = t; j < ks.lane[b][3]; j += T) U[ks.lane[b][2] + j] = a.rs_uid[off + j];
    }
    __syncthreads();
  }
  __shared__ int s_seg_of[kMaxB];
  if (t < kMaxB) s_seg_of[t] = -1;
  __syncthreads();
  if (t < s1 - s0) s_seg_of[S.seg[s0 + t].lane] = s0 + t;
  __syncthreads();
  uint32_t* lv = reinterpret_cast<uint32_t*>(work);  // rows x nB lane values, by chunks
  const int rows = r1 - r0;
  const int rc = max(1, kPcRowChunk / 2 / nB);
  for (int c0 = 0; c0 < rows; c0 += rc) {
    const int nr = min(rc, rows - c0);
    for (int j = t; j < nr * nB; j += T) {
      const int rl = j / nB, b = j - rl * nB;
      const double x = thr[r0 + c0 + rl];  // row 0: -inf, the whole lane penalized
      uint32_t v = kInfPc;
      const int np = ks.lane[b][1], ns = ks.lane[b][3];
      if (staged) {
        const double* LP = L + ks.lane[b][0];
        const double* LS = L + ks.lane[b][2];
        int lo = 0, hi = np;  // #P-records with lat <= x
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (LP[mid] <= x) lo = mid + 1; else hi = mid;
        }
        if (lo > 0) v = U[ks.lane[b][0] + lo - 1];
        lo = 0;
        hi = ns;  // first S-record with lat > x
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (LS[mid] <= x) lo = mid + 1; else hi = mid;
        }
        if (lo < ns) v = min(v, U[ks.lane[b][2] + lo]);
      } else if (s_seg_of[b] >= 0) {
        const int off = S.seg[s_seg_of[b]].off;
        int lo = 0, hi = np;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (a.rp_lat[off + mid] <= x) lo = mid + 1; else hi = mid;
        }
        if (lo > 0) v = a.rp_uid[off + lo - 1];
        lo = 0;
        hi = ns;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (a.rs_lat[off + mid] <= x) lo = mid + 1; else hi = mid;
        }
        if (lo < ns) v = min(v, a.rs_uid[off + lo]);
      }
      lv[j] = v;
    }
    __syncthreads();
    // interval minima: one thread per (row, lo) runs hi = lo .. nB-1
    for (int j = t; j < nr * nB; j += T) {
      const int rl = j / nB, lo = j - rl * nB;
      uint16_t* out = reinterpret_cast<uint16_t*>(a.image + d.rows_off +
                                                  (size_t)(r0 + c0 + rl) * H.row_stride);
      const int base = lo * nB - ((lo * (lo - 1)) >> 1);
      uint32_t m = kInfPc;
      for (int hi = lo; hi < nB; ++hi) {
        m = min(m, lv[rl * nB + hi]);
        out[base + hi - lo] = m == kInfPc ? kNone16 : (uint16_t)m;
      }
    }
    __syncthreads();
  }
}

template <int ES>
__global__ void __launch_bounds__(kPcThreads, 1) k_plan_cluster(const __grid_constant__ PcArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_w[64];
  __shared__ PlanHdr s_hdr;
  __shared__ KindStage s_ks;
  __shared__ PcShared S;
  const int C = (int)gridDim.x;  // one cluster
  const int c = (int)cluster_rank();
  uint64_t tm[6];
  tm[0] = gtimer();
  const long long ck0 = clock64();
  if (threadIdx.x < 2 * kMaxKinds && c == 0) a.kinfo[threadIdx.x] = 0;
  if (threadIdx.x < a.nseg) S.seg[threadIdx.x] = a.seg[threadIdx.x];
  cluster_barrier();
  tm[1] = gtimer();
  for (int s = c; s < a.nseg; s += C) pc_segment<ES>(a, S, s, smem, s_w);
  tm[2] = gtimer();
  cluster_barrier();
  tm[3] = gtimer();
  for (int i = threadIdx.x; i < 4 * a.nseg; i += blockDim.x) S.cnt[i] = a.seg_cnt[i];
  __syncthreads();
  // CTA 0: the candidate order.  CTAs 1..C-1 are dealt round-robin to the kinds (w % K); every
  // CTA of a kind stages the kind's records and thresholds, the kind's first publishes them.
  // With fewer workers than kinds a worker handles several kinds, without staging.
  const int nw = C > 1 ? C - 1 : 1, w = C > 1 ? c - 1 : 0;
  const bool one_kind = nw >= a.K;
  if (c == 0) pc_candidates(a, S, smem, s_w);
  const uint64_t tmc = gtimer();
  if (C == 1 || c > 0) {
    if (one_kind) {
      if (w < nw) pc_kind_stage(a, S, w % a.K, w < a.K, s_ks, smem, s_w);
    } else {
      for (int k = w; k < a.K; k += nw) {
        pc_kind_stage(a, S, k, true, s_ks, smem, s_w);
        if (threadIdx.x == 0) s_ks.staged = false;  // phase 3 reads this kind from global
        __syncthreads();
      }
    }
  }
  const uint64_t tmk = gtimer();
  cluster_barrier();
  tm[4] = gtimer();
  {  // the layout inputs loaded in parallel (rows per kind, two thresholds per kind, counts)
    __shared__ int32_t s_rows[kMaxKinds], s_nc[2];
    __shared__ double s_thr[kMaxKinds + 1][2];
    const int k = threadIdx.x;
    if (k < kMaxKinds) s_rows[k] = k < a.K ? a.kinfo[2 * k] : 0;
    if (k < 2) s_nc[k] = a.kinfo[16 + k];
    __syncthreads();
    if (k < a.K && s_rows[k] >= 2) {
      const int ext = a.base[k] + k;
      s_thr[k][0] = a.thr[ext + 1];
      s_thr[k][1] = a.thr[ext + s_rows[k] - 1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pc_layout(a, s_rows, &s_thr[0][0], s_nc[0], s_nc[1], s_hdr);
      if (c == 0) *a.status = s_hdr.magic == kPlanMagic ? 0 : -1;
    }
    __syncthreads();
  }
  const PlanHdr& H = s_hdr;
  if (c == 0) pc_write_common(a, H);
  if (C == 1 || c > 0) {
    for (int k = 0; k < a.K; ++k) {
      int slot = -1, cnt = 1;
      if (one_kind) {
        cnt = nw / a.K + (k < nw % a.K ? 1 : 0);
        if (w % a.K == k) slot = w / a.K;
      } else if (k % nw == w) {
        slot = 0;
      }
      if (slot < 0) continue;
      if (!one_kind) {  // the stage of this kind is gone: read its records from global
        if (threadIdx.x == 0) {
          s_ks.staged = false;
          const int s0 = a.seg_lo[k], s1 = a.seg_lo[k + 1];
          int acc = 0;
          for (int b = 0; b < kMaxB; ++b)
            s_ks.lane[b][0] = s_ks.lane[b][1] = s_ks.lane[b][2] = s_ks.lane[b][3] = 0;
          for (int s = s0; s < s1; ++s) {
            const int b = S.seg[s].lane;
            s_ks.lane[b][0] = acc;
            s_ks.lane[b][1] = S.cnt[4 * s + 0];
            acc += s_ks.lane[b][1];
            s_ks.lane[b][2] = acc;
            s_ks.lane[b][3] = S.cnt[4 * s + 1];
            acc += s_ks.lane[b][3];
          }
        }
        __syncthreads();
      }
      const int R = H.kd[k].R;
      const int r0 = (int)((int64_t)R * slot / cnt), r1 = (int)((int64_t)R * (slot + 1) / cnt);
      pc_write_kind(a, S, H, k, r0, r1, slot == 0, s_ks, smem, s_w);
    }
  }
  tm[5] = gtimer();
  const long long ck1 = clock64();
  if (a.debug && threadIdx.x == 0 && c == 0)
    printf("pc clock %.0f MHz\n", 1e3 * (double)(ck1 - ck0) / (double)(tm[5] - tm[0]));
  if (a.debug && threadIdx.x == 0)
    printf("pc cta %d: p2 cand %llu kind %llu | init %llu seg %llu bar1 %llu p2 %llu p3 %llu ns\n", c,
           (unsigned long long)(tmc - tm[3]), (unsigned long long)(tmk - tmc),
           (unsigned long long)(tm[1] - tm[0]), (unsigned long long)(tm[2] - tm[1]),
           (unsigned long long)(tm[3] - tm[2]), (unsigned long long)(tm[4] - tm[3]),
           (unsigned long long)(tm[5] - tm[4]));
}

}  // namespace

int plan_cluster_supported(const sp_table* t) { return t->pc_ok ? 1 : 0; }

// Per-table static segment lists (entries grouped by (kind, batch lane), index order) and the
// scratch of the cluster builder; called once when the table is created.
int plan_cluster_prepare(sp_table* t, const int32_t* kind, const int32_t* bidx) {
  t->pc_ok = false;
  if (!t->plan_ok || t->K > kMaxKinds) return SP_OK;
  const int M = t->M, K = t->K, nB = t->nB;
  std::vector<std::vector<int32_t>> bucket((size_t)K * nB);
  for (int j = 0; j < M; ++j) bucket[(size_t)kind[j] * nB + bidx[j]].push_back(j);
  std::vector<PcSegDev> segs;
  std::vector<int32_t> ent;
  int max_seg = 0;
  for (int k = 0; k < K; ++k) {
    t->pc_seg_lo[k] = (int)segs.size();
    if (t->kind_count[k] > kPcMaxKind) return SP_OK;
    for (int b = 0; b < nB; ++b) {
      auto& v = bucket[(size_t)k * nB + b];
      if (v.empty()) continue;
      segs.push_back(PcSegDev{(int32_t)ent.size(), (int32_t)v.size(), k, b});
      ent.insert(ent.end(), v.begin(), v.end());
      max_seg = std::max(max_seg, (int)v.size());
    }
  }
  t->pc_seg_lo[K] = (int)segs.size();
  if (max_seg > kPcMaxSeg || (int)segs.size() > 128) return SP_OK;
  t->pc_nseg = (int)segs.size();
  t->pc_max_seg = max_seg;
  SP_CUDA(cudaMalloc(&t->pc_seg, sizeof(PcSegDev) * segs.size()));
  SP_CUDA(cudaMemcpy(t->pc_seg, segs.data(), sizeof(PcSegDev) * segs.size(), cudaMemcpyHostToDevice));
  SP_CUDA(cudaMalloc(&t->pc_seg_ent, sizeof(int32_t) * M));
  SP_CUDA(cudaMemcpy(t->pc_seg_ent, ent.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice));
  int n2 = 1;
  while (n2 < 2 * M) n2 <<= 1;
  const size_t bytes = (size_t)M * (2 * 8 + 2 * 4 + 2 * (8 * 4 + 4 * 2)) + 16u * segs.size() + 128 +
                       48u * M + 4 * sizeof(double) * n2 + sizeof(int32_t) * n2 + 64 * 16;
  SP_CUDA(cudaMalloc(&t->pc_scratch, bytes));
  t->pc_ok = true;
  return SP_OK;
}

int plan_cluster_launch(sp_ctx* ctx, sp_table* t, Plan& p, int W, const PlanHdr& hdr,
                        int32_t* status) {
  const int M = t->M;
  int n2 = 1;
  while (n2 < 2 * M) n2 <<= 1;
  PcArgs a;
  a.M = M;
  a.K = t->K;
  a.nB = t->nB;
  a.W = W;
  a.nseg = t->pc_nseg;
  a.seg = reinterpret_cast<const PcSegDev*>(t->pc_seg);
  a.ord = t->pc_seg_ent;  // cached per-segment latency order (index order before the first build)
  a.lat = t->lat;
  a.res = t->res;
  a.pool = t->pool;
  a.price = t->price;
  a.batch = t->batch;
  a.kind = t->kind;
  a.id_rank = t->id_rank;
  a.alpha = p.alpha;
  a.cost = p.cost;
  a.costpen = p.costpen;
  a.image = p.image;
  a.image_cap = p.image_cap;
  a.status = status;
  uint8_t* q = reinterpret_cast<uint8_t*>(t->pc_scratch);
  auto take = [&](size_t b) {
    uint8_t* r = q;
    q += (b + 15) & ~(size_t)15;
    return r;
  };
  a.rp_lat = reinterpret_cast<double*>(take(sizeof(double) * M));
  a.rs_lat = reinterpret_cast<double*>(take(sizeof(double) * M));
  a.rp_uid = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rs_uid = reinterpret_cast<uint32_t*>(take(4u * M));
  a.cp_key = reinterpret_cast<uint64_t*>(take(8u * M));
  a.cs_key = reinterpret_cast<uint64_t*>(take(8u * M));
  a.cp_ck = reinterpret_cast<uint64_t*>(take(8u * M));
  a.cs_ck = reinterpret_cast<uint64_t*>(take(8u * M));
  a.cp_res = reinterpret_cast<double*>(take(8u * M));
  a.cs_res = reinterpret_cast<double*>(take(8u * M));
  a.cp_lat = reinterpret_cast<double*>(take(8u * M));
  a.cs_lat = reinterpret_cast<double*>(take(8u * M));
  a.cp_idr = reinterpret_cast<int32_t*>(take(4u * M));
  a.cs_idr = reinterpret_cast<int32_t*>(take(4u * M));
  a.cp_er = reinterpret_cast<int32_t*>(take(4u * M));
  a.cs_er = reinterpret_cast<int32_t*>(take(4u * M));
  a.seg_cnt = reinterpret_cast<int32_t*>(take(16u * t->pc_nseg));
  a.kinfo = reinterpret_cast<int32_t*>(take(4u * 32));
  a.crec = reinterpret_cast<double*>(take(3 * 8u * 2 * M));
  a.gkey = reinterpret_cast<double*>(take(4 * sizeof(double) * n2));
  a.gix = reinterpret_cast<int32_t*>(take(4u * n2));
  a.thr = t->thrscratch;
  for (int k = 0; k < kMaxKinds; ++k) {
    a.base[k] = k < t->K ? t->kind_base[k] : 0;
    a.count[k] = k < t->K ? t->kind_count[k] : 0;
  }
  for (int k = 0; k <= kMaxKinds; ++k) a.seg_lo[k] = k <= t->K ? t->pc_seg_lo[k] : t->pc_nseg;
  a.hdr = hdr;
  a.debug = getenv("SP_PC_DEBUG") != nullptr;
  // shared memory: the largest phase (segment: 60 B per slot; candidates 16 B; thresholds 8 B
  // per record in the shared-memory fallback; rows 64 KB)
  const int es = t->pc_max_seg > kPcThreads ? 2 : 1;
  const size_t smem =
      std::max(std::max((size_t)es * kPcThreads * 60, (size_t)2 * kPcThreads * 36),
               std::max((size_t)2 * kPcMaxKind * 8,
                        (size_t)kPcStageMax * (8 + 8 + 4) + 64 + (size_t)kPcRowChunk * 2));
  auto kern = es == 1 ? k_plan_cluster<1> : k_plan_cluster<2>;
  static uint64_t attr[2] = {0, 0};
  static int csize[64] = {};
  const int dev = cur_device();
  if (attr_once(attr[es - 1])) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  if (csize[dev] == 0) {  // 16-CTA clusters when the device can place one, else 8
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(16);
    q.blockDim = dim3(kPcThreads);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 16;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &q) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 0;
    }
    csize[dev] = n >= 1 ? 16 : kPcCluster;
  }
  const int C = csize[dev];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kPcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SP_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace sp
