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

constexpr uint64_t kKeyNegZero = 0x7FFFFFFFFFFFFFFFull;  // okey(-0.0)
constexpr uint64_t kKeyPosZero = 0x8000000000000000ull;  // okey(+0.0)
// numeric order with -0.0 == +0.0: the order key of +0.0 for both zeros
__device__ __forceinline__ uint64_t canon(uint64_t k) { return k == kKeyNegZero ? kKeyPosZero : k; }

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
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
  const int nw = blockDim.x >> 5;
  if (w == 0) {
    int y = lane < nw ? s_w[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int z = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y += z;
    }
    s_w[lane] = y;
  }
  __syncthreads();
  const int r = (w ? s_w[w - 1] : 0) + x - v;
  *total = s_w[nw - 1];
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
    int y = (int)threadIdx.x < (int)(blockDim.x >> 5) ? s_w[threadIdx.x] : -1;
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
  const int nw = blockDim.x >> 5;
  if (threadIdx.x < 32) {
    int y = (int)threadIdx.x < nw ? s_w[threadIdx.x] : -1;
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
  *total = s_w[32 + nw - 1];
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
  uint8_t* dirty;               // M: latency changed since ord was sorted (cleared here)
  int32_t* order_stale;         // nonzero: ord is stale as a whole (cleared here)
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
  uint32_t *rp_rank, *rs_rank;  // fast path: #records of the kind with a smaller latency
  uint32_t *rp_nrep, *rs_nrep;  // fast path: the latency also occurs earlier in the kind's lists
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
  PlanHdr* host_hdr;              // mapped pinned copy of the header for the host
  uint32_t* host_seq;             // written after host_hdr (system fence): the build's seq
  uint32_t seq;
  int debug;
  // several plans of one table built by one launch (one cluster per plan, k_plan_cluster_multi):
  // no cluster writes the table's cached order / dirty flags / stale word, which the others are
  // still reading; the first plan's cluster writes the new order to ord_out and a follow-up
  // kernel (k_pc_commit_order) installs it
  int multi;
  int32_t* ord_out;
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define PC_STAMP(i)                                                \
  do {                                                             \
    if (threadIdx.x == 0) pc_stamps()[(i)] = gtimer();             \
  } while (0)
__device__ __forceinline__ uint64_t* pc_stamps() {
  __shared__ uint64_t st[32];
  return st;
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


// Full sort of a short segment (n <= 256 entries held one per thread in sk / sv, the rest of the
// block idle) by rank: G = blockDim / pow2(n) threads per entry each count a share of the
// entries ordered before it ((key, val) distinct), the lane group adds the counts, the entry
// goes to its rank.  ~8 comparisons per thread instead of the bitonic network's 36 stages.
__device__ __forceinline__ void rank_sort_small(uint64_t& key, uint32_t& val, int n, int N2,
                                                uint64_t* sk, uint32_t* sv, uint64_t* ok,
                                                uint32_t* ov) {
  const int t = threadIdx.x;
  const int G = min(32, (int)blockDim.x / N2);
  const int r = t / G, q = t % G;
  int cnt = 0;
  uint64_t k0 = 0;
  uint32_t v0 = 0;
  if (r < n) {
    k0 = sk[r];
    v0 = sv[r];
    for (int j = q; j < n; j += G) cnt += (sk[j] < k0 || (sk[j] == k0 && sv[j] < v0)) ? 1 : 0;
  }
  for (int o = 1; o < G; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (r < n && q == 0) {
    ok[cnt] = k0;
    ov[cnt] = v0;
  }
  __syncthreads();
  if (t < n) {
    key = ok[t];
    val = ov[t];
  } else {
    key = ~0ull;
    val = 0xFFFFFFFFu;
  }
  __syncthreads();
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
  bool pos_zero = false;
  if constexpr (E == 1) {
    // 1. (one entry per thread) the entry at this cached position with all its attributes,
    //    its cost / costpen (configurator.py:224-225, numpy order, no FMA) staged by cached
    //    position; then the position order: the cached (lat, index) order of the previous build
    //    with the entries whose latency changed since (dirty) taken out, sorted among themselves
    //    and merged back — the clean entries keep their relative order, so this equals a full
    //    sort; a stale order or many dirty entries take the full bitonic sort.  Sort values
    //    carry entry << 11 | cached position, so (key, value) orders exactly as (lat, index).
    const bool stale = *a.order_stale != 0;
    uint8_t* stg = smem + 65536;  // staged attributes by cached position (40 B each)
    uint64_t* A_ck = reinterpret_cast<uint64_t*>(stg);
    uint64_t* A_cpk = A_ck + 1024;
    double* A_res = reinterpret_cast<double*>(A_cpk + 1024);
    double* A_lat = A_res + 1024;
    int32_t* A_idr = reinterpret_cast<int32_t*>(A_lat + 1024);
    uint64_t key[1];
    uint32_t val[1];
    bool dq = false;
    if (t < n) {
      const int e = a.ord[off + t];
      const double L = a.lat[e], R = a.res[e], B = (double)a.batch[e], P = a.pool[e],
                   pr = a.price[e];
      const int idr = a.id_rank[e];
      dq = stale || a.dirty[e] != 0;
      const double c = __ddiv_rn(__dmul_rn(__dmul_rn(R, L), pr), B);
      const double pen = __dmul_rn(a.alpha, __ddiv_rn(__dmul_rn(L, R), __dmul_rn(B, P)));
      const double cp = __dadd_rn(c, pen);
      a.cost[e] = c;
      a.costpen[e] = cp;
      A_ck[t] = okey(c);
      A_cpk[t] = okey(cp);
      A_res[t] = R;
      A_lat[t] = L;
      A_idr[t] = idr;
      key[0] = okey(L);
      val[0] = (uint32_t)e << 11 | (uint32_t)t;
    } else {
      key[0] = ~0ull;
      val[0] = 0xFFFFFFFFu;
    }
    sk[t] = key[0];
    sv[t] = val[0];
    const int nd = __syncthreads_count(dq);
    PC_STAMP(1);
    constexpr int kIncMax = 256;  // dirty entries merged incrementally
    bool moved = nd > 0;
    if (nd == 0) {
      const bool bad = t + 1 < n && (sk[t] > sk[t + 1] || (sk[t] == sk[t + 1] && sv[t] > sv[t + 1]));
      moved = __syncthreads_or(bad);
      if (moved) {
        if (N2 <= 256) rank_sort_small(key[0], val[0], n, N2, sk, sv, (uint64_t*)(sv + NE), (uint32_t*)((uint64_t*)(sv + NE) + 256));
        else reg_bitonic<1>(key, val, N2, sk, sv);
      }
    } else if (stale || nd > kIncMax) {
      if (N2 <= 256) rank_sort_small(key[0], val[0], n, N2, sk, sv, (uint64_t*)(sv + NE), (uint32_t*)((uint64_t*)(sv + NE) + 256));
      else reg_bitonic<1>(key, val, N2, sk, sv);
    } else {
      // clean entries -> uk/uv (still sorted), dirty -> dk/dv (the position arrays' space)
      uint64_t* uk = reinterpret_cast<uint64_t*>(sv + NE);
      uint64_t* dk = uk + NE;
      uint32_t* uv = reinterpret_cast<uint32_t*>(dk + NE);
      uint32_t* dv = uv + NE;
      uint64_t* dk2 = reinterpret_cast<uint64_t*>(dv + NE);
      uint32_t* dv2 = reinterpret_cast<uint32_t*>(dk2 + kIncMax);
      int tot;
      const int od = pc_excl_sum(dq ? 1 : 0, s_w, &tot);
      const int nc = n - tot;
      if (t < n) {
        if (dq) {
          dk[od] = key[0];
          dv[od] = val[0];
        } else {
          uk[t - od] = key[0];
          uv[t - od] = val[0];
        }
      }
      __syncthreads();
      {  // rank of each dirty entry among the dirty ones: G threads per entry (a lane group)
        int p2 = 1;
        while (p2 < tot) p2 <<= 1;
        const int G = min(32, T / p2);
        const int r = t / G, q = t % G;
        int cntr = 0;
        uint64_t k0 = 0;
        uint32_t v0 = 0;
        if (r < tot) {
          k0 = dk[r];
          v0 = dv[r];
          for (int j = q; j < tot; j += G) cntr += (dk[j] < k0 || (dk[j] == k0 && dv[j] < v0)) ? 1 : 0;
        }
        for (int o = 1; o < G; o <<= 1) cntr += __shfl_xor_sync(0xffffffffu, cntr, o);
        if (r < tot && q == 0) {
          dk2[cntr] = k0;
          dv2[cntr] = v0;
        }
      }
      __syncthreads();
      // merge: final position = index in its own list + elements of the other list before it
      if (t < nc) {
        const uint64_t k0 = uk[t];
        const uint32_t v0 = uv[t];
        int lo = 0, hi = tot;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (dk2[mid] < k0 || (dk2[mid] == k0 && dv2[mid] < v0)) lo = mid + 1; else hi = mid;
        }
        sk[t + lo] = k0;
        sv[t + lo] = v0;
      } else if (t < n) {
        const int r = t - nc;
        const uint64_t k0 = dk2[r];
        const uint32_t v0 = dv2[r];
        int lo = 0, hi = nc;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (uk[mid] < k0 || (uk[mid] == k0 && uv[mid] < v0)) lo = mid + 1; else hi = mid;
        }
        sk[r + lo] = k0;
        sv[r + lo] = v0;
      }
      __syncthreads();
      key[0] = sk[t];
      val[0] = sv[t];
    }
    PC_STAMP(2);
    // 2. position arrays from the staged attributes; the cached order and the dirty flags
    if (t < n) {
      const int src = (int)(val[0] & 2047u), e = (int)(val[0] >> 11);
      if (a.multi) {
        if (a.ord_out) a.ord_out[off + t] = e;
      } else if (moved) {
        a.ord[off + t] = e;
        a.dirty[e] = 0;
      }
      pe[t] = e;
      const double L = A_lat[src];
      plat[t] = L;
      pck[t] = A_ck[src];
      pcpk[t] = A_cpk[src];
      pres[t] = A_res[src];
      pidr[t] = A_idr[src];
      pos_zero = __double_as_longlong(L) == 0;
    }
    if (__syncthreads_or(pos_zero) && t == 0) atomicOr(&a.kinfo[2 * sg.kind + 1], 1);
  } else {
  // 1. the cached (lat, index) order of the previous build; re-sorted when it no longer holds
  //    or a latency changed (E > 1: segments of more than 1024 entries)
  const bool stale = *a.order_stale != 0;
  uint64_t key[E];
  uint32_t val[E];
  int nd_local = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int i = t + q * T;
    if (i < n) {
      val[q] = (uint32_t)a.ord[off + i];
      key[q] = okey(a.lat[val[q]]);
      nd_local += (stale || a.dirty[val[q]] != 0) ? 1 : 0;
    } else {
      val[q] = 0xFFFFFFFFu;
      key[q] = ~0ull;
    }
    sk[i] = key[q];
    sv[i] = val[q];
  }
  __syncthreads();
  PC_STAMP(1);
  bool bad = nd_local > 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int i = t + q * T;
    if (i + 1 < n) bad |= sk[i] > sk[i + 1] || (sk[i] == sk[i + 1] && sv[i] > sv[i + 1]);
  }
  if (__syncthreads_or(bad)) {
    reg_bitonic<E>(key, val, N2, sk, sv);
    if (!a.multi) {
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int i = t + q * T;
        if (i < n) {
          a.ord[off + i] = (int32_t)val[q];
          a.dirty[val[q]] = 0;
        }
      }
    }
  }
  if (a.multi && a.ord_out) {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int i = t + q * T;
      if (i < n) a.ord_out[off + i] = (int32_t)val[q];
    }
  }
  PC_STAMP(2);
  // 2. per position: cost / costpen (configurator.py:224-225, numpy order, no FMA), keys
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
  }
  PC_STAMP(3);
  // Key1 (the r1 order: cost key, res, id_rank) and Key2 (costpen key, then Key1)
  // comparators capture the shared-memory pointers by value (a by-reference closure can leave
  // them in local memory)
  auto less1 = [=](int x, int y) {
    if (pck[x] != pck[y]) return pck[x] < pck[y];
    if (pres[x] != pres[y]) return pres[x] < pres[y];
    return pidr[x] < pidr[y];
  };
  auto less2 = [=](int x, int y) {
    if (pcpk[x] != pcpk[y]) return pcpk[x] < pcpk[y];
    return less1(x, y);
  };
  auto best1 = [=](int x, int y) { return x < 0 ? y : (y < 0 ? x : (less1(y, x) ? y : x)); };
  auto best2 = [=](int x, int y) { return x < 0 ? y : (y < 0 ? x : (less2(y, x) ? y : x)); };
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
  PC_STAMP(4);
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
  PC_STAMP(6);
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
      a.rp_uid[off + j] = fin ? 0u : kInfPc;
      a.rp_rank[off + j] = 0u;
      a.rp_nrep[off + j] = j > 0 && canon(okey(plat[lP[j - 1]])) == canon(okey(plat[p]));
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
      a.rs_uid[off + j] = fst ? 0u : kInfPc;
      a.rs_rank[off + j] = 0u;
      a.rs_nrep[off + j] = j > 0 && canon(okey(plat[lS[j - 1]])) == canon(okey(plat[p]));
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
  PC_STAMP(13);
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
  PC_STAMP(14);
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

// ---- phase 2, merge form ---------------------------------------------------------------------
// Every list phase 1 produced is already sorted: a segment's P-candidates (strictly falling
// Key1 along the latency order, score = cost) descend in the unified order, its S-candidates
// (strictly rising Key2, score = costpen) ascend, and every lane's P / S record lists ascend in
// latency.  So no sort is needed: a candidate's id is the number of candidates that precede it
// (binary searches in the other lists, spread over every CTA of the cluster), and a kind's row
// thresholds are the distinct record latencies placed by their count of smaller latencies.

constexpr int kPcCandMerge = 4096;   // candidates kept in shared memory by every CTA
constexpr int kPcStageMax = 4096;    // records of one kind staged in shared memory
// shared-memory map of phases 2 and 3 (bytes)
constexpr int kSmCandKey = 0;                                  // u64[kPcCandMerge]
constexpr int kSmCandEnt = kSmCandKey + 8 * kPcCandMerge;       // u32[kPcCandMerge]
constexpr int kSmL = kSmCandEnt + 4 * kPcCandMerge;             // f64[kPcStageMax] record lats
constexpr int kSmThr = kSmL + 8 * kPcStageMax;                  // f64[kPcStageMax + 2]
constexpr int kSmU = kSmThr + 8 * (kPcStageMax + 2);            // u32[kPcStageMax] record ids
constexpr int kSmWork = kSmU + 4 * kPcStageMax;                 // scratch (64 KB)
constexpr int kSmEnd = kSmWork + 16 * kPcStageMax;

struct KindStage {
  int nr, R;           // records, rows
  int lane[kMaxB][4];  // per lane: P start, P count, S start, S count (record index space)
  bool staged;         // records and thresholds are in shared memory
};

struct CandLists {
  int nl, nc;
  int off[2 * kPcMaxSegs + 1];  // list i = 2s (P of segment s, descending), 2s+1 (S, ascending)
};

// equal scores (rare): the rest of the argmin key from global memory — kept out of line so that
// the compiler never hoists these loads into the common comparison path
__device__ __noinline__ bool cand_tie_less(const PcArgs& a, int eu, int ev, uint32_t su, uint32_t sv) {
  const uint64_t cu = okey(a.cost[eu]), cv = okey(a.cost[ev]);
  if (cu != cv) return cu < cv;
  if (a.res[eu] != a.res[ev]) return a.res[eu] < a.res[ev];
  if (a.id_rank[eu] != a.id_rank[ev]) return a.id_rank[eu] < a.id_rank[ev];
  return !su && sv;
}

__device__ __forceinline__ int list_of(const CandLists& cl, int u) {
  int lo = 0, hi = cl.nl;  // last i with off[i] <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cl.off[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

// Pairwise merge tree of `nr` ascending runs (offsets off[0..nr], shared; rewritten) of n items:
// at every level an item of run r moves to (start of the merged pair) + (its index in r) +
// (the items of the partner run that precede it: strictly smaller ones for the left run,
// smaller-or-equal ones for the right run — equal items keep left-run-first order).  Returns the
// buffer (src or dst) that holds the merged items.
template <class T, class Less>
__device__ T* merge_runs(T* src, T* dst, int* off, int* s_nr, int n, Less less) {
  while (*s_nr > 1) {
    const int nr = *s_nr;
    for (int g = threadIdx.x; g < n; g += blockDim.x) {
      int lo = 0, hi = nr;  // run of g: last r with off[r] <= g (and a non-empty run)
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= g) lo = mid; else hi = mid;
      }
      int r = lo;
      while (r + 1 < nr && off[r + 1] <= g) ++r;
      const T x = src[g];
      const int pr = r ^ 1;
      const int base = off[r & ~1];
      if (pr >= nr) {
        dst[g] = x;
        continue;
      }
      const int pb = off[pr], pn = off[pr + 1] - pb;
      int a = 0, b = pn;
      if (r & 1) {
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (!less(x, src[pb + mid])) a = mid + 1; else b = mid;
        }
      } else {
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (less(src[pb + mid], x)) a = mid + 1; else b = mid;
        }
      }
      dst[base + (g - off[r]) + a] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = 0;
      for (int i = 0; i < nr; i += 2) off[m++] = off[i];
      off[m] = n;
      *s_nr = m;
    }
    __syncthreads();
    T* tsw = src;
    src = dst;
    dst = tsw;
  }
  return src;
}

// phase 2a: candidate ids; every CTA ranks its share of the candidates.  Returns false when
// the merge form does not apply (too many candidates, or a -0.0 penalized score whose order
// key would misplace it) — CTA 0 then sorts with the general path.
__device__ bool pc_cand_merge(const PcArgs& a, const PcShared& S, CandLists& cl, uint8_t* smem,
                              int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const int c = (int)cluster_rank();
  if (c != 0) return true;  // CTA 0 orders the candidates
  {
    const int i = t;
    const int len = i < 2 * a.nseg ? S.cnt[4 * (i >> 1) + 2 + (i & 1)] : 0;
    int tot;
    const int o = pc_excl_sum(len, s_w, &tot);
    if (i <= 2 * a.nseg) cl.off[i] = o;
    if (t == 0) {
      cl.nl = 2 * a.nseg;
      cl.nc = tot;
    }
    __syncthreads();
  }
  const int nc = cl.nc;
  if (nc > kPcCandMerge) return false;
  uint64_t* K = reinterpret_cast<uint64_t*>(smem + kSmCandKey);
  uint32_t* Ent = reinterpret_cast<uint32_t*>(smem + kSmCandEnt);
  bool negzero = false;
  for (int u = t; u < nc; u += T) {
    const int i = list_of(cl, u);
    const int sl = S.seg[i >> 1].off + (u - cl.off[i]);
    const uint64_t k = (i & 1) ? a.cs_key[sl] : a.cp_key[sl];
    negzero |= (i & 1) && k == kKeyNegZero;
    K[u] = canon(k);
    Ent[u] = (uint32_t)(((i & 1) ? a.cs_er[sl] : a.cp_er[sl]) & 0xFFFF);
  }
  if (__syncthreads_or(negzero)) return false;
  PC_STAMP(13);
  // u precedes v in (score, cost key, res, id_rank, side); items are candidate | S-side << 31
  auto prec = [&](uint32_t x, uint32_t y) {
    const int u = (int)(x & 0x7FFFFFFFu), v = (int)(y & 0x7FFFFFFFu);
    const uint64_t ku = K[u], kv = K[v];
    if (ku != kv) return ku < kv;
    return cand_tie_less(a, (int)Ent[u], (int)Ent[v], x >> 31, y >> 31);
  };
  if (c == 0) {
    // runs ascending: P lists are read backwards
    uint32_t* A = reinterpret_cast<uint32_t*>(smem + kSmWork);
    uint32_t* B = A + kPcCandMerge;
    __shared__ int s_off2[2 * kPcMaxSegs + 1];
    __shared__ int s_nr2;
    for (int u = t; u < nc; u += T) {
      const int i = list_of(cl, u);
      const int b = cl.off[i], n_i = cl.off[i + 1] - b, j = u - b;
      A[(i & 1) ? u : b + n_i - 1 - j] = (uint32_t)u | ((i & 1) ? 0x80000000u : 0u);
    }
    if (t <= cl.nl) s_off2[t] = cl.off[t];
    if (t == 0) s_nr2 = cl.nl;
    __syncthreads();
    PC_STAMP(15);
    uint32_t* R = merge_runs(A, B, s_off2, &s_nr2, nc, prec);
    PC_STAMP(14);
    for (int r = t; r < nc; r += T) {
      const uint32_t x = R[r];
      const int u = (int)(x & 0x7FFFFFFFu);
      const int i = list_of(cl, u);
      const bool su = (i & 1) != 0;
      const int j = u - cl.off[i];
      const int sg = i >> 1, sl = S.seg[sg].off + j;
      const int er = su ? a.cs_er[sl] : a.cp_er[sl];
      const int e = er & 0xFFFF, rec = er >> 16;
      (su ? a.rs_uid : a.rp_uid)[S.seg[sg].off + rec] = (uint32_t)r;
      CandB cb;
      cb.meta = (uint32_t)e | ((su ? 0u : 1u) << 16) | ((uint32_t)S.seg[sg].kind << 17);
      cb.batch = a.hdr.batch_vals[S.seg[sg].lane];
      a.crec[3 * r + 0] = key_double(su ? a.cs_key[sl] : a.cp_key[sl]);
      a.crec[3 * r + 1] = su ? a.cs_lat[sl] : a.cp_lat[sl];
      a.crec[3 * r + 2] = __longlong_as_double(*reinterpret_cast<const long long*>(&cb));
    }
  }
  if (c == 0 && t == 0) {
    int ncp = 0;
    for (int s = 0; s < a.nseg; ++s) ncp += S.cnt[4 * s + 2];
    a.kinfo[16] = ncp;
    a.kinfo[17] = nc - ncp;
  }
  __syncthreads();
  return true;
}

// phase 2b: the kind's records staged (latency, by lane: P list then S list) and its row
// thresholds: row 0 is -inf, row r the r-th distinct record latency (the zero group's
// threshold is +0.0 whenever the kind has a +0.0 latency, -0.0 otherwise).  `publish`: write
// the row count and thresholds for every CTA's layout.
__device__ void pc_kind_stage(const PcArgs& a, const PcShared& S, int k, bool publish, KindStage& ks,
                              uint8_t* smem, int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const int ext = a.base[k] + k;
  const int s0 = a.seg_lo[k], s1 = a.seg_lo[k + 1];
  __shared__ int s_loff[2 * kMaxB + 1];  // record-list offsets (list 2q: P of the q-th segment)
  if (t == 0) {
    int acc = 0;
    for (int b = 0; b < kMaxB; ++b) ks.lane[b][0] = ks.lane[b][1] = ks.lane[b][2] = ks.lane[b][3] = 0;
    for (int s = s0; s < s1; ++s) {
      const int b = S.seg[s].lane, q = s - s0;
      s_loff[2 * q] = acc;
      ks.lane[b][0] = acc;
      ks.lane[b][1] = S.cnt[4 * s + 0];
      acc += ks.lane[b][1];
      s_loff[2 * q + 1] = acc;
      ks.lane[b][2] = acc;
      ks.lane[b][3] = S.cnt[4 * s + 1];
      acc += ks.lane[b][3];
    }
    s_loff[2 * (s1 - s0)] = acc;
    ks.nr = acc;
    ks.staged = acc <= kPcStageMax;
    ks.R = 0;
  }
  __syncthreads();
  PC_STAMP(8);
  const int nr = ks.nr, nl = 2 * (s1 - s0);
  if (a.count[k] == 0) {
    if (publish && t == 0) a.kinfo[2 * k] = 0;
    __syncthreads();
    return;
  }
  const bool has_pz = a.kinfo[2 * k + 1] != 0;
  if (ks.staged) {
    double* L = reinterpret_cast<double*>(smem + kSmL);
    double* thr = reinterpret_cast<double*>(smem + kSmThr);
    uint64_t* tmp = reinterpret_cast<uint64_t*>(smem + kSmWork);  // 2 x kPcStageMax
    for (int g = t; g < nr; g += T) {
      int q = 0;
      while (q + 1 < nl && s_loff[q + 1] <= g) ++q;
      const int off = S.seg[s0 + (q >> 1)].off, j = g - s_loff[q];
      L[g] = (q & 1) ? a.rs_lat[off + j] : a.rp_lat[off + j];
    }
    __syncthreads();
    PC_STAMP(9);
    // the kind's record lists (each ascending) merged by canonical latency key, then the
    // distinct keys in order
    uint64_t* A = tmp;
    uint64_t* B = tmp + kPcStageMax;
    __shared__ int s_off3[2 * kMaxB + 1];
    __shared__ int s_nr3;
    for (int g = t; g < nr; g += T) A[g] = canon(okey(L[g]));
    if (t <= nl) s_off3[t] = s_loff[t];
    if (t == 0) s_nr3 = nl;
    __syncthreads();
    const uint64_t* Mg = merge_runs(A, B, s_off3, &s_nr3, nr, [](uint64_t x, uint64_t y) { return x < y; });
    int R = 1;
    for (int g0 = 0; g0 < nr; g0 += T) {
      const int g = g0 + t;
      const bool o = g < nr && (g == 0 || Mg[g] != Mg[g - 1]);
      int tot;
      const int ex = pc_excl_sum(o ? 1 : 0, s_w, &tot);
      if (o) {
        double v = key_double(Mg[g]);
        if (v == 0.0) v = has_pz ? 0.0 : -0.0;
        thr[R + ex] = v;
      }
      R += tot;
    }
    if (t == 0) {
      thr[0] = -INFINITY;
      ks.R = R;
    }
    __syncthreads();
    PC_STAMP(10);
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
  for (int g = t; g < N2; g += T) {
    uint64_t v = ~0ull;
    if (g < nr) {
      int q = 0;
      while (q + 1 < nl && s_loff[q + 1] <= g) ++q;
      const int off = S.seg[s0 + (q >> 1)].off, j = g - s_loff[q];
      v = okey((q & 1) ? a.rs_lat[off + j] : a.rp_lat[off + j]);
    }
    key[g] = v;
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

// ---- phases 2 and 3, distributed form (the common case) ---------------------------------------
// Every CTA stages every candidate key and every record latency (all kinds) in shared memory and
// takes an equal slice of the (item, list) pairs: a candidate's id is the number of candidates
// preceding it summed over all candidate lists, a record's slot among the kind's latencies the
// number of smaller record latencies summed over the kind's lists — binary searches in the sorted
// lists, the per-list counts added with global atomics into the record's uid / rank word.  A
// record "represents" its latency unless an earlier list of its kind (or its own predecessor)
// holds the same one.  After the cluster barrier every CTA reduces the representatives per kind
// (rows, first / last threshold) for the layout; each kind's CTAs compact the thresholds by slot.
constexpr int kFastCand = 2048, kFastRec = 4096;
constexpr int kFKc = 0;                          // u64[kFastCand] candidate keys (canonical)
constexpr int kFRc = kFKc + 8 * kFastCand;       // u32[kFastCand] record slot | S << 31
constexpr int kFCs = kFRc + 4 * kFastCand;       // u32[kFastCand] candidate slot (cp_ / cs_)
constexpr int kFKr = kFCs + 4 * kFastCand;       // u64[kFastRec] record keys (canonical)
constexpr int kFRr = kFKr + 8 * kFastRec;        // u32[kFastRec] record slot | S << 31
constexpr int kFThr = kFRr + 4 * kFastRec;       // f64[kFastRec + 2] thresholds
constexpr int kFTmp = kFThr + 8 * (kFastRec + 2);  // u64[kFastRec] keys by slot
constexpr int kFOcc = kFTmp + 8 * kFastRec;      // u8[kFastRec]
constexpr int kFWork = kFOcc + kFastRec;         // 32 KB: bucket histogram / lane values
constexpr int kFEnd = kFWork + 32768;

struct FastLists {
  int nseg, nc, nrec;
  int coff[2 * kPcMaxSegs + 1];  // candidate lists: 2s = P of segment s (descending), 2s+1 = S
  int roff[2 * kPcMaxSegs + 1];  // record lists: 2s = P records of segment s, 2s+1 = S (ascending)
  int klo[kMaxKinds + 1];        // kind k: record lists [2 seg_lo[k], 2 seg_lo[k+1])
  int64_t wc, wr[kMaxKinds + 1];  // pair counts: candidates, records of kinds < k
  bool ok;
};

__device__ __forceinline__ int last_le(const int* off, int n, int g) {  // last i: off[i] <= g
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= g) lo = mid; else hi = mid;
  }
  while (lo + 1 < n && off[lo + 1] <= g) ++lo;
  return lo;
}

// phase 2 (every CTA); returns false when the shapes exceed the staging capacity or a -0.0
// penalized score breaks the lists' order — the caller then takes the sorting path
__device__ bool pc_fast_phase2(const PcArgs& a, const PcShared& S, FastLists& fl, uint8_t* smem,
                               int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const int C = (int)cluster_size(), c = (int)cluster_rank();
  const int nl = 2 * a.nseg;
  {
    const int lc = t < nl ? S.cnt[4 * (t >> 1) + 2 + (t & 1)] : 0;
    const int lr = t < nl ? S.cnt[4 * (t >> 1) + (t & 1)] : 0;
    int tc, tr;
    const int oc = pc_excl_sum(lc, s_w, &tc);
    const int orr = pc_excl_sum(lr, s_w, &tr);
    if (t <= nl) {
      fl.coff[t] = oc;
      fl.roff[t] = orr;
    }
    if (t == 0) {
      fl.nseg = a.nseg;
      fl.nc = tc;
      fl.nrec = tr;
      fl.ok = tc <= kFastCand && tr <= kFastRec;
    }
    __syncthreads();
    if (t == 0) {
      fl.wc = (int64_t)fl.nc * nl;
      fl.wr[0] = 0;
      for (int k = 0; k < a.K; ++k) {
        fl.klo[k] = 2 * a.seg_lo[k];
        const int n_r = fl.roff[2 * a.seg_lo[k + 1]] - fl.roff[2 * a.seg_lo[k]];
        fl.wr[k + 1] = fl.wr[k] + (int64_t)n_r * (2 * (a.seg_lo[k + 1] - a.seg_lo[k]));
      }
      fl.klo[a.K] = nl;
    }
    __syncthreads();
  }
  if (!fl.ok) return false;
  PC_STAMP(20);
  uint64_t* Kc = reinterpret_cast<uint64_t*>(smem + kFKc);
  uint32_t* Rc = reinterpret_cast<uint32_t*>(smem + kFRc);
  uint32_t* Cs = reinterpret_cast<uint32_t*>(smem + kFCs);
  uint64_t* Kr = reinterpret_cast<uint64_t*>(smem + kFKr);
  uint32_t* Rr = reinterpret_cast<uint32_t*>(smem + kFRr);
  bool negzero = false;
  for (int u = t; u < fl.nc; u += T) {
    const int i = last_le(fl.coff, nl, u);
    const bool sS = i & 1;
    const int sl = S.seg[i >> 1].off + (u - fl.coff[i]);
    const uint64_t k = sS ? a.cs_key[sl] : a.cp_key[sl];
    const int er = sS ? a.cs_er[sl] : a.cp_er[sl];
    negzero |= sS && k == kKeyNegZero;
    Kc[u] = canon(k);
    Cs[u] = (uint32_t)sl;
    Rc[u] = (uint32_t)(S.seg[i >> 1].off + (er >> 16)) | (sS ? 0x80000000u : 0u);
  }
  uint8_t* own_list = smem + kFOcc;  // list of each record (phase 2 only)
  for (int g = t; g < fl.nrec; g += T) {
    const int i = last_le(fl.roff, nl, g);
    const bool sS = i & 1;
    const int sl = S.seg[i >> 1].off + (g - fl.roff[i]);
    Kr[g] = canon(okey(sS ? a.rs_lat[sl] : a.rp_lat[sl]));
    Rr[g] = (uint32_t)sl | (sS ? 0x80000000u : 0u);
    own_list[g] = (uint8_t)i;
  }
  if (__syncthreads_or(negzero)) {
    if (t == 0) fl.ok = false;
    __syncthreads();
    return false;
  }
  PC_STAMP(21);
  // candidate entries for the rare equal-score comparisons
  const PcArgs* ap = &a;
  auto cent = [=](int u) {
    const uint32_t sl = Cs[u];
    return (int)(((Rc[u] >> 31) ? ap->cs_er[sl] : ap->cp_er[sl]) & 0xFFFF);
  };
  auto prec = [=](int x, int y) {  // candidate x precedes candidate y in the unified order
    const uint64_t kx = Kc[x], ky = Kc[y];
    if (kx != ky) return kx < ky;
    return cand_tie_less(*ap, cent(x), cent(y), Rc[x] >> 31, Rc[y] >> 31);
  };
  // per-CTA partial counts in shared memory (the threshold area is free until phase 3), added
  // to the global words once per touched item
  uint32_t* accC = reinterpret_cast<uint32_t*>(smem + kFThr);
  uint32_t* accR = accC + kFastCand;
  for (int i = t; i < kFastCand + kFastRec; i += T) accC[i] = 0u;
  __syncthreads();
  // pair counts stay far below 2^31 for the staged sizes (2048 x 256 + 4096 x 32)
  const int wc = (int)fl.wc, W = (int)(fl.wc + fl.wr[a.K]);
  const int i0 = (int)((int64_t)W * c / C), i1 = (int)((int64_t)W * (c + 1) / C);
  for (int it = i0 + t; it < i1; it += T) {
    if (it < wc) {  // candidate u against candidate list m
      const int u = it / nl, m = it - u * nl;
      const int b = fl.coff[m], n = fl.coff[m + 1] - b;
      if (n == 0) continue;
      const uint64_t ku = Kc[u];
      int lo = 0, hi = n;
      if (u >= b && u < b + n) {  // its own list: the elements before it (ascending) / after it
        lo = (m & 1) ? u - b : b + n - 1 - u;
      } else if (m & 1) {  // ascending: the preceding elements are a prefix
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const uint64_t km = Kc[b + mid];
          if (km != ku ? km < ku : prec(b + mid, u)) lo = mid + 1; else hi = mid;
        }
      } else {      // descending: a suffix
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const uint64_t km = Kc[b + mid];
          if (!(km != ku ? km < ku : prec(b + mid, u))) lo = mid + 1; else hi = mid;
        }
        lo = n - lo;
      }
      if (lo) atomicAdd(&accC[u], (uint32_t)lo);
    } else {           // record g against a list m of its kind
      const int j = it - wc;
      int k = 0;
      while ((int)fl.wr[k + 1] <= j) ++k;
      const int nlk = fl.klo[k + 1] - fl.klo[k];
      const int jj = j - (int)fl.wr[k];
      const int q = jj / nlk;
      const int g = fl.roff[fl.klo[k]] + q, m = fl.klo[k] + (jj - q * nlk);
      const int b = fl.roff[m], n = fl.roff[m + 1] - b;
      if (n == 0) continue;
      const uint64_t x = Kr[g];
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (Kr[b + mid] < x) lo = mid + 1; else hi = mid;
      }
      if (lo) atomicAdd(&accR[g], (uint32_t)lo);
      if (m < own_list[g] && lo < n && Kr[b + lo] == x) {
        const uint32_t r = Rr[g];
        ((r >> 31) ? a.rs_nrep : a.rp_nrep)[r & 0x7FFFFFFFu] = 1u;
      }
    }
  }
  __syncthreads();
  for (int u = t; u < fl.nc; u += T)
    if (accC[u]) {
      const uint32_t r = Rc[u];
      atomicAdd(((r >> 31) ? a.rs_uid : a.rp_uid) + (r & 0x7FFFFFFFu), accC[u]);
    }
  for (int g = t; g < fl.nrec; g += T)
    if (accR[g]) {
      const uint32_t r = Rr[g];
      atomicAdd(((r >> 31) ? a.rs_rank : a.rp_rank) + (r & 0x7FFFFFFFu), accR[g]);
    }
  __syncthreads();
  PC_STAMP(22);
  return true;
}

// after the barrier, every CTA: per kind the representative count and the extreme latencies
__device__ void pc_fast_layout_inputs(const PcArgs& a, const FastLists& fl, int32_t* rows,
                                      double* thr2, uint8_t* smem) {
  const int T = blockDim.x, t = threadIdx.x;
  const uint64_t* Kr = reinterpret_cast<const uint64_t*>(smem + kFKr);
  const uint32_t* Rr = reinterpret_cast<const uint32_t*>(smem + kFRr);
  uint8_t* occ = smem + kFOcc;  // representative flag by record
  __shared__ int s_cnt[kMaxKinds];
  __shared__ unsigned long long s_min[kMaxKinds], s_max[kMaxKinds];
  if (t < kMaxKinds) {
    s_cnt[t] = 0;
    s_min[t] = ~0ull;
    s_max[t] = 0ull;
  }
  __syncthreads();
  for (int g = t; g < fl.nrec; g += T) {
    const uint32_t r = Rr[g];
    const bool rep = ((r >> 31) ? a.rs_nrep : a.rp_nrep)[r & 0x7FFFFFFFu] == 0u;
    occ[g] = rep;
    if (rep) {
      int k = 0;
      while (fl.roff[fl.klo[k + 1]] <= g) ++k;
      atomicAdd(&s_cnt[k], 1);
      atomicMin(&s_min[k], (unsigned long long)Kr[g]);
      atomicMax(&s_max[k], (unsigned long long)Kr[g]);
    }
  }
  __syncthreads();
  if (t < kMaxKinds) {
    rows[t] = t < a.K && a.count[t] > 0 ? 1 + s_cnt[t] : 0;
    const bool has_pz = t < a.K && a.kinfo[2 * t + 1] != 0;
    double lo = key_double(s_min[t]), hi = key_double(s_max[t]);
    if (lo == 0.0) lo = has_pz ? 0.0 : -0.0;
    if (hi == 0.0) hi = has_pz ? 0.0 : -0.0;
    thr2[2 * t] = lo;
    thr2[2 * t + 1] = hi;
  }
  __syncthreads();
}

// CTA 0: header, lookup table, candidate records at their ids
__device__ void pc_fast_common(const PcArgs& a, const PcShared& S, const FastLists& fl,
                               const PlanHdr& H, uint8_t* smem) {
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
  const uint32_t* Rc = reinterpret_cast<const uint32_t*>(smem + kFRc);
  const uint32_t* Cs = reinterpret_cast<const uint32_t*>(smem + kFCs);
  double* rscore = reinterpret_cast<double*>(a.image + H.score_off);
  double* rlat = reinterpret_cast<double*>(a.image + H.lat_off);
  CandB* recb = reinterpret_cast<CandB*>(a.image + H.recb_off);
  const int nl = 2 * a.nseg;
  for (int u = t; u < fl.nc; u += T) {
    const uint32_t r = Rc[u], sl = Cs[u];
    const bool sS = r >> 31;
    const uint32_t id = (sS ? a.rs_uid : a.rp_uid)[r & 0x7FFFFFFFu];
    const int i = last_le(fl.coff, nl, u);
    const PcSegDev sg = S.seg[i >> 1];
    const int e = (sS ? a.cs_er[sl] : a.cp_er[sl]) & 0xFFFF;
    rscore[id] = key_double(sS ? a.cs_key[sl] : a.cp_key[sl]);
    rlat[id] = sS ? a.cs_lat[sl] : a.cp_lat[sl];
    CandB b;
    b.meta = (uint32_t)e | ((sS ? 0u : 1u) << 16) | ((uint32_t)sg.kind << 17);
    b.batch = H.batch_vals[sg.lane];
    recb[id] = b;
  }
}

// rows [r0, r1) of kind k (`first`: also the bucket table); thresholds compacted by slot
__device__ void pc_fast_kind(const PcArgs& a, const PcShared& S, const FastLists& fl,
                             const PlanHdr& H, int k, int r0, int r1, bool first, uint8_t* smem,
                             int* s_w) {
  const int T = blockDim.x, t = threadIdx.x;
  const KindDesc d = H.kd[k];
  const int R = d.R;
  if (R == 0 || H.magic != kPlanMagic) return;
  const uint64_t* Kr = reinterpret_cast<const uint64_t*>(smem + kFKr);
  const uint32_t* Rr = reinterpret_cast<const uint32_t*>(smem + kFRr);
  double* thr = reinterpret_cast<double*>(smem + kFThr);
  uint64_t* tmp = reinterpret_cast<uint64_t*>(smem + kFTmp);
  uint8_t* occ = smem + kFOcc;  // representatives (pc_fast_layout_inputs)
  uint8_t* work = smem + kFWork;
  const int g0 = fl.roff[fl.klo[k]], g1 = fl.roff[fl.klo[k + 1]], nr = g1 - g0;
  uint8_t* slot = work;  // slot occupancy (nr bytes)
  for (int j = t; j < nr; j += T) slot[j] = 0;
  __syncthreads();
  for (int g = g0 + t; g < g1; g += T) {
    if (!occ[g]) continue;
    const uint32_t r = Rr[g];
    const uint32_t q = ((r >> 31) ? a.rs_rank : a.rp_rank)[r & 0x7FFFFFFFu];
    tmp[q] = Kr[g];
    slot[q] = 1;
  }
  __syncthreads();
  const bool has_pz = a.kinfo[2 * k + 1] != 0;
  {
    int o = 1;
    for (int j0 = 0; j0 < nr; j0 += T) {
      const int j = j0 + t;
      const bool f = j < nr && slot[j];
      int tot;
      const int ex = pc_excl_sum(f ? 1 : 0, s_w, &tot);
      if (f) {
        double v = key_double(tmp[j]);
        if (v == 0.0) v = has_pz ? 0.0 : -0.0;
        thr[o + ex] = v;
      }
      o += tot;
    }
    if (t == 0) thr[0] = -INFINITY;
    __syncthreads();
  }
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
      const uint32_t cc = s_h[b];
      bkt[b] = (uint32_t)below | (cc << 16);
      below += (int)cc;
    }
    __syncthreads();
  }
  if (r1 <= r0) return;
  // lane lists of the kind in the staged record keys: lane b = list pair of its segment
  __shared__ int s_pl[kMaxB][4];
  if (t < kMaxB) s_pl[t][0] = s_pl[t][1] = s_pl[t][2] = s_pl[t][3] = 0;
  __syncthreads();
  if (t < a.seg_lo[k + 1] - a.seg_lo[k]) {
    const int sgi = a.seg_lo[k] + t;
    const int b = S.seg[sgi].lane;
    s_pl[b][0] = fl.roff[2 * sgi];
    s_pl[b][1] = fl.roff[2 * sgi + 1] - fl.roff[2 * sgi];
    s_pl[b][2] = fl.roff[2 * sgi + 1];
    s_pl[b][3] = fl.roff[2 * sgi + 2] - fl.roff[2 * sgi + 1];
  }
  __syncthreads();
  const int nB = H.nB;
  uint32_t* lv = reinterpret_cast<uint32_t*>(work);  // rows x nB lane values, by chunks
  const int rows = r1 - r0;
  const int rc = max(1, 8192 / nB);
  for (int c0 = 0; c0 < rows; c0 += rc) {
    const int nrw = min(rc, rows - c0);
    for (int j = t; j < nrw * nB; j += T) {
      const int rl = j / nB, b = j - rl * nB;
      const int r = r0 + c0 + rl;
      // x: canonical key of the row threshold (row 0: below every latency)
      const uint64_t x = r == 0 ? 0ull : canon(okey(thr[r]));
      uint32_t v = kInfPc;
      const int pb = s_pl[b][0], np = s_pl[b][1], sb = s_pl[b][2], ns = s_pl[b][3];
      int lo = 0, hi = np;  // #P-records with lat <= x
      if (r > 0)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (Kr[pb + mid] <= x) lo = mid + 1; else hi = mid;
        }
      if (lo > 0) {
        const uint32_t rr = Rr[pb + lo - 1];
        v = a.rp_uid[rr & 0x7FFFFFFFu];
      }
      lo = 0;
      hi = ns;  // first S-record with lat > x
      if (r > 0)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (Kr[sb + mid] <= x) lo = mid + 1; else hi = mid;
        }
      if (lo < ns) {
        const uint32_t rr = Rr[sb + lo];
        v = min(v, a.rs_uid[rr & 0x7FFFFFFFu]);
      }
      lv[j] = v;
    }
    __syncthreads();
    for (int j = t; j < nrw * nB; j += T) {
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
  double* L = reinterpret_cast<double*>(smem + kSmL);
  const double* thr = staged ? reinterpret_cast<const double*>(smem + kSmThr) : a.thr + ext;
  uint32_t* U = reinterpret_cast<uint32_t*>(smem + kSmU);
  uint8_t* work = smem + kSmWork;
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
  if (staged) {  // the candidate ids of the staged records (written in phase 2)
    for (int g = t; g < ks.nr; g += T) {
      int b = 0;  // record g: lane b's P list or S list
      while (!(g >= ks.lane[b][0] && g < ks.lane[b][2] + ks.lane[b][3]) ||
             ks.lane[b][1] + ks.lane[b][3] == 0)
        ++b;
      int s = s0;
      while (S.seg[s].lane != b) ++s;
      const int off = S.seg[s].off;
      U[g] = g < ks.lane[b][2] ? a.rp_uid[off + g - ks.lane[b][0]] : a.rs_uid[off + g - ks.lane[b][2]];
    }
    __syncthreads();
  }
  PC_STAMP(17);
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
__device__ __forceinline__ void pc_build(const PcArgs& a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_w[64];
  __shared__ PlanHdr s_hdr;
  __shared__ KindStage s_ks;
  __shared__ PcShared S;
  const int C = (int)cluster_size();
  const int c = (int)cluster_rank();
  uint64_t tm[6];
  tm[0] = gtimer();
  const long long ck0 = clock64();
  if (threadIdx.x < 32) pc_stamps()[threadIdx.x] = tm[0];
  if (threadIdx.x < a.nseg) S.seg[threadIdx.x] = a.seg[threadIdx.x];  // static per table
  // programmatic dependent launch: the latencies (the fold's output) are read and the plan
  // image (the previous select's input) is written only after the predecessor has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x < 2 * kMaxKinds && c == 0) a.kinfo[threadIdx.x] = 0;
  cluster_barrier();
  tm[1] = gtimer();
  for (int s = c; s < a.nseg; s += C) pc_segment<ES>(a, S, s, smem, s_w);
  tm[2] = gtimer();
  cluster_barrier();
  if (c == 0 && threadIdx.x == 0 && !a.multi) *a.order_stale = 0;  // every CTA has read it
  tm[3] = gtimer();
  for (int i = threadIdx.x; i < 4 * a.nseg; i += blockDim.x) S.cnt[i] = a.seg_cnt[i];
  __syncthreads();
  // phase 2: every CTA ranks a share of the candidates (merge form; CTA 0 falls back to a sort
  // when it does not apply); CTAs 1..C-1 are dealt round-robin to the kinds (w % K), every CTA
  // of a kind stages the kind's records and thresholds, the kind's first publishes them.  With
  // fewer workers than kinds a worker handles several kinds, without staging.
  const int nw = C > 1 ? C - 1 : 1, w = C > 1 ? c - 1 : 0;
  const bool one_kind = nw >= a.K;
  __shared__ CandLists s_cl;
  __shared__ FastLists s_fl;
  const bool fast = pc_fast_phase2(a, S, s_fl, smem, s_w);
  if (!fast) {
    if (!pc_cand_merge(a, S, s_cl, smem, s_w) && c == 0) pc_candidates(a, S, smem, s_w);
  }
  const uint64_t tmc = gtimer();
  if (!fast && (C == 1 || c > 0)) {
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
  {  // layout inputs: rows per kind, first / last threshold per kind, candidate counts
    __shared__ int32_t s_rows[kMaxKinds], s_nc[2];
    __shared__ double s_thr[kMaxKinds + 1][2];
    if (fast) {
      pc_fast_layout_inputs(a, s_fl, s_rows, &s_thr[0][0], smem);
      if (threadIdx.x == 0) {
        int ncp = 0;
        for (int sgi = 0; sgi < a.nseg; ++sgi) ncp += S.cnt[4 * sgi + 2];
        s_nc[0] = ncp;
        s_nc[1] = s_fl.nc - ncp;
      }
    } else {
      const int k = threadIdx.x;
      if (k < kMaxKinds) s_rows[k] = k < a.K ? a.kinfo[2 * k] : 0;
      if (k < 2) s_nc[k] = a.kinfo[16 + k];
      __syncthreads();
      if (k < a.K && s_rows[k] >= 2) {
        const int ext = a.base[k] + k;
        s_thr[k][0] = a.thr[ext + 1];
        s_thr[k][1] = a.thr[ext + s_rows[k] - 1];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pc_layout(a, s_rows, &s_thr[0][0], s_nc[0], s_nc[1], s_hdr);
      if (c == 0) *a.status = s_hdr.magic == kPlanMagic ? 0 : -1;
    }
    __syncthreads();
    if (c == 0 && a.host_hdr) {  // the header for the host's next kernel parameter
      if (threadIdx.x < (int)(sizeof(PlanHdr) / 4))
        reinterpret_cast<volatile uint32_t*>(a.host_hdr)[threadIdx.x] =
            reinterpret_cast<const uint32_t*>(&s_hdr)[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(a.host_seq) = a.seq;
      }
    }
  }
  const PlanHdr& H = s_hdr;
  if (fast) {
    if (c == 0) pc_fast_common(a, S, s_fl, H, smem);
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
        const int R = H.kd[k].R;
        const int r0 = (int)((int64_t)R * slot / cnt), r1 = (int)((int64_t)R * (slot + 1) / cnt);
        pc_fast_kind(a, S, s_fl, H, k, r0, r1, slot == 0, smem, s_w);
      }
    }
  } else {
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
  }
  tm[5] = gtimer();
  const long long ck1 = clock64();
  if (a.debug && threadIdx.x == 0 && c == 0)
    printf("pc clock %.0f MHz\n", 1e3 * (double)(ck1 - ck0) / (double)(tm[5] - tm[0]));
  if (a.debug && threadIdx.x == 0 && c < 3) {
    uint64_t* st = pc_stamps();
    printf("pc cta %d stamps: s1 %lld s2 %lld s3 %lld s4 %lld s6 %lld | k8 %lld k9 %lld k10 %lld | c13 %lld c14 %lld | w17 %lld\n", c,
           (long long)(st[1] - tm[0]), (long long)(st[2] - tm[0]), (long long)(st[3] - tm[0]),
           (long long)(st[4] - tm[0]), (long long)(st[6] - tm[0]), (long long)(st[8] - tm[0]),
           (long long)(st[9] - tm[0]), (long long)(st[10] - tm[0]), (long long)(st[13] - tm[0]),
           (long long)(st[14] - tm[0]), (long long)(st[17] - tm[0]));
    printf("pc cta %d c15 %lld f20 %lld f21 %lld f22 %lld\n", c, (long long)(st[15] - tm[0]),
           (long long)(st[20] - tm[0]), (long long)(st[21] - tm[0]), (long long)(st[22] - tm[0]));
  }
  if (a.debug && threadIdx.x == 0)
    printf("pc cta %d: p2 cand %llu kind %llu | init %llu seg %llu bar1 %llu p2 %llu p3 %llu ns\n", c,
           (unsigned long long)(tmc - tm[3]), (unsigned long long)(tmk - tmc),
           (unsigned long long)(tm[1] - tm[0]), (unsigned long long)(tm[2] - tm[1]),
           (unsigned long long)(tm[3] - tm[2]), (unsigned long long)(tm[4] - tm[3]),
           (unsigned long long)(tm[5] - tm[4]));
}

template <int ES>
__global__ void __launch_bounds__(kPcThreads, 1) k_plan_cluster(const __grid_constant__ PcArgs a) {
  pc_build<ES>(a);
}

constexpr int kPcMaxMulti = 4;
struct PcMulti {
  PcArgs a[kPcMaxMulti];
};

// one cluster per plan: cluster q builds plan q (same table, its own alpha, scratch and image)
template <int ES>
__global__ void __launch_bounds__(kPcThreads, 1) k_plan_cluster_multi(const __grid_constant__ PcMulti m) {
  pc_build<ES>(m.a[blockIdx.x / cluster_size()]);
}

// after a multi-plan build: the new cached order, no entry dirty, the order no longer stale
__global__ void k_pc_commit_order(int M, const int32_t* __restrict__ ord_new, int32_t* __restrict__ ord,
                                  uint8_t* __restrict__ dirty, int32_t* __restrict__ order_stale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) {
    ord[i] = ord_new[i];
    dirty[i] = 0;
  }
  if (i == 0) *order_stale = 0;
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
  const size_t bytes = (size_t)M * (2 * 8 + 6 * 4 + 2 * (8 * 4 + 4 * 2)) + 16u * segs.size() + 128 +
                       48u * M + 4 * sizeof(double) * n2 + sizeof(int32_t) * n2 + 64 * 16;
  SP_CUDA(cudaMalloc(&t->pc_scratch, bytes));
  t->pc_scratch_bytes = bytes;
  t->pc_ok = true;
  return SP_OK;
}

// The cluster builder's arguments for plan p of table t; `scratch` / `thr` are the plan's
// private scratch (the table's own for a single build).
static void pc_fill_args(sp_ctx* ctx, sp_table* t, Plan& p, int W, const PlanHdr& hdr,
                         int32_t* status, PlanHdr* host_hdr, uint32_t* host_seq, uint32_t seq,
                         void* scratch, double* thr, PcArgs& a) {
  const int M = t->M;
  int n2 = 1;
  while (n2 < 2 * M) n2 <<= 1;
  a.M = M;
  a.K = t->K;
  a.nB = t->nB;
  a.W = W;
  a.nseg = t->pc_nseg;
  a.seg = reinterpret_cast<const PcSegDev*>(t->pc_seg);
  a.ord = t->pc_seg_ent;  // cached per-segment latency order (index order before the first build)
  a.dirty = t->dirty;
  a.order_stale = t->dev_counters + 4;
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
  uint8_t* q = reinterpret_cast<uint8_t*>(scratch);
  auto take = [&](size_t b) {
    uint8_t* r = q;
    q += (b + 15) & ~(size_t)15;
    return r;
  };
  a.rp_lat = reinterpret_cast<double*>(take(sizeof(double) * M));
  a.rs_lat = reinterpret_cast<double*>(take(sizeof(double) * M));
  a.rp_uid = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rs_uid = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rp_rank = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rs_rank = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rp_nrep = reinterpret_cast<uint32_t*>(take(4u * M));
  a.rs_nrep = reinterpret_cast<uint32_t*>(take(4u * M));
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
  a.thr = thr;
  for (int k = 0; k < kMaxKinds; ++k) {
    a.base[k] = k < t->K ? t->kind_base[k] : 0;
    a.count[k] = k < t->K ? t->kind_count[k] : 0;
  }
  for (int k = 0; k <= kMaxKinds; ++k) a.seg_lo[k] = k <= t->K ? t->pc_seg_lo[k] : t->pc_nseg;
  a.hdr = hdr;
  a.host_hdr = host_hdr;
  a.host_seq = host_seq;
  a.seq = seq;
  a.debug = ctx->opt.pc_debug;
  a.multi = 0;
  a.ord_out = nullptr;
}

static size_t pc_smem_bytes(const sp_table* t) {
  // shared memory: the largest phase (segment: 60 B per slot; candidates 16 B; thresholds 8 B
  // per record in the shared-memory fallback; rows 64 KB)
  const int es = t->pc_max_seg > 2 * kPcThreads ? 4 : (t->pc_max_seg > kPcThreads ? 2 : 1);
  return std::max(std::max((size_t)es * kPcThreads * 60, (size_t)2 * kPcThreads * 36),
                  std::max(std::max((size_t)2 * kPcMaxKind * 8, (size_t)kSmEnd), (size_t)kFEnd));
}

int plan_cluster_launch(sp_ctx* ctx, sp_table* t, Plan& p, int W, const PlanHdr& hdr,
                        int32_t* status, PlanHdr* host_hdr, uint32_t* host_seq, uint32_t seq) {
  PcArgs a;
  pc_fill_args(ctx, t, p, W, hdr, status, host_hdr, host_seq, seq, t->pc_scratch, t->thrscratch, a);
  const int es = t->pc_max_seg > 2 * kPcThreads ? 4 : (t->pc_max_seg > kPcThreads ? 2 : 1);
  const size_t smem = pc_smem_bytes(t);
  auto kern = es == 1 ? k_plan_cluster<1> : (es == 2 ? k_plan_cluster<2> : k_plan_cluster<4>);
  static uint64_t attr[3] = {0, 0, 0};
  static int csize[64] = {};
  const int dev = cur_device();
  if (attr_once(attr[es == 4 ? 2 : es - 1])) {
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
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  SP_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace sp

namespace sp {

// Several plans of one table (e.g. the alphas a workload sweeps) in ONE launch: one cluster per
// plan, each with its own scratch, threshold area, image and host header; the table's cached
// order is read by every cluster and replaced afterwards by k_pc_commit_order.  Every image is
// byte-identical to the plan's single build (tests/test_gpu_plan.py).
int plan_cluster_launch_multi(sp_ctx* ctx, sp_table* t, Plan* const* ps, int n, int W,
                              const PlanHdr& hdr, int32_t* status, void* const* scratch,
                              double* const* thr, int32_t* ord_new) {
  if (n < 1 || n > kPcMaxMulti) return fail(SP_E_INVALID, "plan multi: 1..4 plans");
  PcMulti m;
  for (int q = 0; q < n; ++q) {
    Plan& p = *ps[q];
    void* dh = nullptr;
    SP_CUDA(cudaHostGetDevicePointer(&dh, p.host_hdr, 0));
    ++p.seq;
    pc_fill_args(ctx, t, p, W, hdr, status + q, static_cast<PlanHdr*>(dh),
                 reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(dh) + sizeof(PlanHdr)), p.seq,
                 scratch[q], thr[q], m.a[q]);
    m.a[q].multi = 1;
    m.a[q].ord_out = q == 0 ? ord_new : nullptr;
  }
  for (int q = n; q < kPcMaxMulti; ++q) m.a[q] = m.a[0];
  const int es = t->pc_max_seg > 2 * kPcThreads ? 4 : (t->pc_max_seg > kPcThreads ? 2 : 1);
  const size_t smem = pc_smem_bytes(t);
  auto kern = es == 1 ? k_plan_cluster_multi<1>
                      : (es == 2 ? k_plan_cluster_multi<2> : k_plan_cluster_multi<4>);
  static uint64_t attr[3] = {0, 0, 0};
  static int csize[64] = {};
  const int dev = cur_device();
  if (attr_once(attr[es == 4 ? 2 : es - 1])) {
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  if (csize[dev] == 0) {  // 16-CTA clusters when n of them fit at once, else 8
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(16 * n);
    q.blockDim = dim3(kPcThreads);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 16;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, (const void*)kern, &q) != cudaSuccess || c < 1) {
      cudaGetLastError();
      c = 0;
    }
    csize[dev] = c >= kPcMaxMulti ? 16 : kPcCluster;
  }
  const int C = csize[dev];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * n);
  cfg.blockDim = dim3(kPcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  SP_CUDA(cudaLaunchKernelEx(&cfg, kern, m));
  SP_CHECK_LAUNCH(ctx);
  k_pc_commit_order<<<(t->M + 255) / 256, 256, 0, ctx->stream>>>(t->M, ord_new, t->pc_seg_ent,
                                                                  t->dirty, t->dev_counters + 4);
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace sp
