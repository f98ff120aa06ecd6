// sp_plan.cu — per-(table, alpha) decision plan, built on the device.
//
// What the reference does per call (configurator.py:219-237): for every entry j
//     cost_j    = ((res_j * lat_j) * price_j) / batch_j
//     pen_j     = alpha * ((lat_j * res_j) / (batch_j * pool_j))
//     score_j   = cost_j + (lat_j < slack[kind_j] ? 0 : pen_j)
// then a masked argmin with exact-equality ties broken by (cost, res, id_rank).
//
// What we precompute once per (profile version, alpha) so that each decision is
// O(K) shared-memory lookups instead of O(M) (SURVEY.md §8(d) "K2b"):
//   * cost_j, costpen_j = cost_j + pen_j                        (k_cost; bitwise equal to
//     cost + where(lat<slack, 0, pen) because cost + 0.0 == cost for cost > 0)
//   * r1_j = rank of j under (cost, res, id_rank)   -> tie order of feasible entries
//     r2_j = rank of j under (costpen, cost, res, id_rank) -> order of penalized entries
//   * per kind, entries sorted by latency; for every threshold position p the per-batch-
//     size prefix-min of r1 over positions < p (feasible: lat < slack) and suffix-min of r2
//     over positions >= p (penalized).  Consecutive identical rows are merged, leaving a
//     staircase of R_k rows keyed by the latency just below each step.
//   * every surviving candidate (entry, side) gets a unified id in (score, r1) order — the
//     reference's argmin key — so a row lane stores min(id of best feasible, id of best
//     penalized) and the whole decision reduces to a u16 minimum over admitted lanes.
//   * per kind, an order-key bucket table over the thresholds (radix-accelerated search)
//     and a batch-value lookup table for min_batch / available.
// See DESIGN.md §K2 for the proof of bit-exactness.
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>

#include <cub/cub.cuh>

#include "sp_internal.cuh"

namespace sp {

namespace {

constexpr uint32_t kInf32 = 0xFFFFFFFFu;

struct KindInfo {
  int32_t base[kMaxKinds];
  int32_t count[kMaxKinds];
};

__global__ void k_cost(int M, const double* __restrict__ lat, const double* __restrict__ res,
                       const int32_t* __restrict__ batch, const double* __restrict__ pool,
                       const double* __restrict__ price, double alpha,
                       double* __restrict__ cost, double* __restrict__ costpen) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  double L = lat[j], R = res[j], B = (double)batch[j], P = pool[j], pr = price[j];
  // configurator.py:224  cost = (self.res * self.lat) * self.price / self.batch
  double c = __ddiv_rn(__dmul_rn(__dmul_rn(R, L), pr), B);
  // configurator.py:225  penalty = alpha * ((self.lat * self.res) / (self.batch * self.pool))
  double pen = __dmul_rn(alpha, __ddiv_rn(__dmul_rn(L, R), __dmul_rn(B, P)));
  cost[j] = c;
  costpen[j] = __dadd_rn(c, pen);
}

// ---- the plan's three entry orders ---------------------------------------------------------
//   r1     rank under (cost, res, id_rank)            -> tie order of feasible entries
//   r2     rank under (costpen, cost, res, id_rank)   =  (costpen, r1)
//   order  entries by (kind, lat, index)              -> latency order inside each kind
// Each is a sort of M unique (u64 key, u32 tag) items: CTA tiles of 2048 items are sorted with
// a block merge sort (k_tile_sort), then every item's final position is its rank inside its
// tile plus, per other tile, the number of smaller items there (k_merge_pairs: one CTA per
// (tile, other tile) pair, the other tile staged in shared memory, binary searches there).
// r1 sorts by (cost, index) and then resolves exact-equality cost ties by (res, id_rank)
// inside each (short) tie run (k_rank_r1).

__device__ __forceinline__ uint64_t dkey(double x) {
  return order_key(static_cast<uint64_t>(__double_as_longlong(x)));
}

struct __align__(16) SItem {
  uint64_t k;
  uint32_t t;
  uint32_t pad;
};
constexpr int kSortThreads = 256, kSortIpt = 2, kSortTile = kSortThreads * kSortIpt;
constexpr int kSortR1 = 0, kSortR2 = 1, kSortOrder = 2;

template <int KIND>
struct SLess {
  __device__ __forceinline__ bool operator()(const SItem& a, const SItem& b) const {
    if (KIND == kSortOrder) {  // (kind, lat, index): kind in the tag's top byte
      const uint32_t ka = a.t >> 24, kb = b.t >> 24;
      if (ka != kb) return ka < kb;
      if (a.k != b.k) return a.k < b.k;
      return (a.t & 0xFFFFFFu) < (b.t & 0xFFFFFFu);
    }
    return a.k < b.k || (a.k == b.k && a.t < b.t);
  }
};

__device__ __forceinline__ SItem sentinel() {
  SItem x;
  x.k = ~0ull;
  x.t = 0xFFFFFFFFu;
  x.pad = 0;
  return x;
}

// item of entry / position j for sort KIND (j >= M: sentinel)
template <int KIND>
__device__ __forceinline__ SItem make_item(int j, int M, const double* __restrict__ a,
                                           const int32_t* __restrict__ b) {
  if (j >= M) return sentinel();
  SItem x;
  x.pad = 0;
  if (KIND == kSortR1) {        // a = cost
    x.k = dkey(a[j]);
    x.t = (uint32_t)j;
  } else if (KIND == kSortR2) {  // position j of the r1 order: a = costpen, b = ent_r1
    x.k = dkey(a[b[j]]);
    x.t = (uint32_t)j;           // r1 rank
  } else {                       // a = lat, b = kind
    x.k = dkey(a[j]);
    x.t = ((uint32_t)b[j] << 24) | (uint32_t)j;
  }
  return x;
}

template <int KIND>
__device__ void tile_sort(int M, int tile, const double* a, const int32_t* b, SItem* out,
                          int32_t* rank, void* temp) {
  using Sort = cub::BlockMergeSort<SItem, kSortThreads, kSortIpt>;
  SItem it[kSortIpt];
  const int base = tile * kSortTile + threadIdx.x * kSortIpt;
#pragma unroll
  for (int q = 0; q < kSortIpt; ++q) it[q] = make_item<KIND>(base + q, M, a, b);
  Sort(*reinterpret_cast<typename Sort::TempStorage*>(temp)).Sort(it, SLess<KIND>());
#pragma unroll
  for (int q = 0; q < kSortIpt; ++q) {
    out[base + q] = it[q];
    rank[base + q] = threadIdx.x * kSortIpt + q;  // rank inside the tile; k_merge_pairs adds
  }
}

// blockIdx.x < ntiles: sort A (KA) tile; otherwise sort B (KB) tile (B may be absent)
template <int KA, int KB>
__global__ void __launch_bounds__(kSortThreads) k_tile_sort(int M, int ntiles, const double* aA,
                                                            const int32_t* bA, SItem* outA,
                                                            int32_t* rkA, const double* aB,
                                                            const int32_t* bB, SItem* outB,
                                                            int32_t* rkB) {
  __shared__ typename cub::BlockMergeSort<SItem, kSortThreads, kSortIpt>::TempStorage temp;
  if ((int)blockIdx.x < ntiles)
    tile_sort<KA>(M, blockIdx.x, aA, bA, outA, rkA, &temp);
  else
    tile_sort<KB>(M, blockIdx.x - ntiles, aB, bB, outB, rkB, &temp);
}

// CTA (x, y): items of tile a (x < ntiles: sort A, else sort B, tile x - ntiles) against tile
// b = y of the same sort, staged in shared memory; every item adds the number of smaller items
// of tile b to its rank (items are unique, so the ranks form a permutation).
template <int KIND>
__device__ __forceinline__ void merge_pair(const SItem* __restrict__ tiles, int32_t* rank, int a,
                                           int b, SItem* sb) {
  for (int c = threadIdx.x; c < kSortTile; c += blockDim.x) sb[c] = tiles[(size_t)b * kSortTile + c];
  __syncthreads();
  SLess<KIND> less;
  for (int e = threadIdx.x; e < kSortTile; e += blockDim.x) {
    const SItem x = tiles[(size_t)a * kSortTile + e];
    int lo = 0, hi = kSortTile;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (less(sb[mid], x)) lo = mid + 1; else hi = mid;
    }
    if (lo) atomicAdd(&rank[(size_t)a * kSortTile + e], lo);
  }
}

template <int KA, int KB>
__global__ void __launch_bounds__(256) k_merge_pairs(int ntiles, const SItem* __restrict__ tA,
                                                     int32_t* rkA, const SItem* __restrict__ tB,
                                                     int32_t* rkB) {
  __shared__ SItem sb[kSortTile];
  const int x = blockIdx.x, b = blockIdx.y;
  if (x < ntiles) {
    if (x != b) merge_pair<KA>(tA, rkA, x, b, sb);
  } else if (x - ntiles != b) {
    merge_pair<KB>(tB, rkB, x - ntiles, b, sb);
  }
}

// final positions of both sorts' items; only real items (rank < M) are written
__global__ void k_scatter_items(int M, int n, const SItem* __restrict__ tA,
                                const int32_t* __restrict__ rkA, SItem* outA,
                                const SItem* __restrict__ tB, const int32_t* __restrict__ rkB,
                                SItem* outB) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const int r = rkA[p];
    if (r < M) outA[r] = tA[p];
  } else if (tB && p < 2 * n) {
    p -= n;
    const int r = rkB[p];
    if (r < M) outB[r] = tB[p];
  }
}

// position p of the (cost, index) order -> r1 (ties by (res, id_rank), configurator.py:235-237)
__global__ void k_rank_r1(int M, const SItem* __restrict__ srt, const double* __restrict__ res,
                          const int32_t* __restrict__ id_rank, uint32_t* r1, int32_t* ent_r1) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M) return;
  const uint64_t k = srt[p].k;
  const int e = (int)srt[p].t;
  int r = p;
  const bool tl = p > 0 && srt[p - 1].k == k, tr = p + 1 < M && srt[p + 1].k == k;
  if (tl || tr) {
    int a = p, b = p + 1;
    while (a > 0 && srt[a - 1].k == k) --a;
    while (b < M && srt[b].k == k) ++b;
    const double re = res[e];
    const int ie = id_rank[e];
    int c = 0;
    for (int q = a; q < b; ++q) {
      const int f = (int)srt[q].t;
      const double rf = res[f];
      c += (rf < re) || (rf == re && id_rank[f] < ie);
    }
    r = a + c;
  }
  r1[e] = (uint32_t)r;
  ent_r1[r] = e;
}

// sorted (costpen, r1) items -> ent_r2 / r2;  sorted (kind, lat, index) items -> order
__global__ void k_orders_out(int M, const SItem* __restrict__ s2, const int32_t* __restrict__ ent_r1,
                             int32_t* ent_r2, uint32_t* r2, const SItem* __restrict__ s3,
                             int32_t* order) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= M) return;
  if (s2) {
    const int e = ent_r1[s2[q].t];
    ent_r2[q] = e;
    r2[e] = (uint32_t)q;
  }
  if (s3) order[q] = (int32_t)(s3[q].t & 0xFFFFFFu);
}

__device__ __forceinline__ uint32_t warp_incl_min(uint32_t v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v = min(v, t);
  }
  return v;
}

// Block-wide exclusive scans over blockDim.x == 1024 (32 warps).
__device__ int block_excl_sum(int v, int* s_warp, int* total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += t;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    int y = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y += t;
    }
    s_warp[lane] = y;  // inclusive per warp
  }
  __syncthreads();
  int base = w ? s_warp[w - 1] : 0;
  *total = s_warp[(blockDim.x >> 5) - 1];
  int r = base + x - v;
  __syncthreads();
  return r;
}

__device__ int block_excl_max(int v, int* s_warp) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x = max(x, t);
  }
  int ex = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) ex = INT32_MIN;
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    int y = lane < nw ? s_warp[lane] : INT32_MIN;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y = max(y, t);
    }
    s_warp[lane] = y;
  }
  __syncthreads();
  int base = w ? s_warp[w - 1] : INT32_MIN;
  int r = max(base, ex);
  __syncthreads();
  return r;
}

// One CTA (1024 threads) per kind.  Phase A: per batch lane b the prefix-min of r1 (feasible
// side, positions < p) and the suffix-min of r2 (penalized side, positions >= p) over the
// kind's latency order — every thread owns a contiguous chunk of positions, the per-chunk
// lane minima are scanned across chunks in shared memory (one warp per lane and direction),
// then each thread writes its chunk with the carried minima.  Phase B: rows at latency
// boundaries, merged when identical to the previous boundary's row.
constexpr int kStairMaxW = 16;
__global__ void __launch_bounds__(1024) k_stair(int M, int K, int W, KindInfo ki,
                                                const int32_t* __restrict__ order,
                                                const int32_t* __restrict__ bidx,
                                                const double* __restrict__ lat,
                                                const uint32_t* __restrict__ r1,
                                                const uint32_t* __restrict__ r2, uint32_t* pf,
                                                uint32_t* sf, double* thrscratch,
                                                uint32_t* rowscratch, int32_t* rows_per_kind,
                                                uint32_t* candf, uint32_t* cands) {
  extern __shared__ uint32_t s_lane[];  // [2][W][blockDim.x]: chunk minima -> carries
  __shared__ int s_warp[32];
  __shared__ int s_carry_b, s_carry_rows, s_lastb;
  const int k = blockIdx.x;
  const int Mk = ki.count[k];
  const int base = ki.base[k];
  const int ext = base + k;  // extended positions 0..Mk of this kind
  const int stride = M + K;
  if (Mk == 0) {
    if (threadIdx.x == 0) rows_per_kind[k] = 0;
    return;
  }
  const int T = blockDim.x, t = threadIdx.x;
  uint32_t* A = s_lane;          // prefix side
  uint32_t* B = s_lane + W * T;  // suffix side
  const int P = (Mk + T - 1) / T;
  const int q0 = min(t * P, Mk), q1 = min(q0 + P, Mk);
  for (int b = 0; b < W; ++b) {
    A[b * T + t] = kInf32;
    B[b * T + t] = kInf32;
  }
  for (int q = q0; q < q1; ++q) {
    const int e = order[base + q];
    const int b = bidx[e];
    A[b * T + t] = min(A[b * T + t], r1[e]);
    B[b * T + t] = min(B[b * T + t], r2[e]);
  }
  __syncthreads();
  {  // warp w: lane b = w % W, direction w / W; exclusive scan over the T chunk minima
    const int w = t >> 5, l = t & 31;
    if (w < 2 * W) {
      const bool suf = w >= W;
      uint32_t* v = (suf ? B : A) + (w % W) * T;
      const int per = T / 32;
      uint32_t m = kInf32;
      for (int c = 0; c < per; ++c) {
        const int idx = suf ? T - 1 - (l * per + c) : l * per + c;
        m = min(m, v[idx]);
      }
      uint32_t incl = warp_incl_min(m, l);
      uint32_t carry = __shfl_up_sync(0xffffffffu, incl, 1);
      if (l == 0) carry = kInf32;
      for (int c = 0; c < per; ++c) {
        const int idx = suf ? T - 1 - (l * per + c) : l * per + c;
        const uint32_t x = v[idx];
        v[idx] = carry;  // minimum over the chunks before (prefix) / after (suffix) this one
        carry = min(carry, x);
      }
    }
  }
  __syncthreads();
  {
    uint32_t run[kStairMaxW];
#pragma unroll
    for (int b = 0; b < kStairMaxW; ++b) run[b] = b < W ? A[b * T + t] : kInf32;
    for (int q = q0; q < q1; ++q) {  // pf[b][ext + q] = min r1 over positions < q
#pragma unroll
      for (int b = 0; b < kStairMaxW; ++b)
        if (b < W) pf[(size_t)b * stride + ext + q] = run[b];
      const int e = order[base + q];
      const int bq = bidx[e];
      const uint32_t v = r1[e];
#pragma unroll
      for (int b = 0; b < kStairMaxW; ++b) run[b] = (b == bq) ? min(run[b], v) : run[b];
    }
    if (q1 == Mk && q0 < q1) {
#pragma unroll
      for (int b = 0; b < kStairMaxW; ++b)
        if (b < W) pf[(size_t)b * stride + ext + Mk] = run[b];
    }
#pragma unroll
    for (int b = 0; b < kStairMaxW; ++b) run[b] = b < W ? B[b * T + t] : kInf32;
    for (int q = q1 - 1; q >= q0; --q) {  // sf[b][ext + q] = min r2 over positions >= q
      const int e = order[base + q];
      const int bq = bidx[e];
      const uint32_t v = r2[e];
#pragma unroll
      for (int b = 0; b < kStairMaxW; ++b) {
        run[b] = (b == bq) ? min(run[b], v) : run[b];
        if (b < W) sf[(size_t)b * stride + ext + q] = run[b];
      }
    }
    if (t == 0) {
      for (int b = 0; b < W; ++b) sf[(size_t)b * stride + ext + Mk] = kInf32;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_carry_b = INT32_MIN;
    s_carry_rows = 0;
  }
  __syncthreads();
  const uint32_t* pfk = pf + ext;
  const uint32_t* sfk = sf + ext;
  for (int c0 = 0; c0 <= Mk; c0 += blockDim.x) {
    int p = c0 + threadIdx.x;
    bool valid = p <= Mk;
    bool isb = false;
    if (valid) {
      if (p == 0 || p == Mk) {
        isb = true;
      } else {
        isb = lat[order[base + p]] != lat[order[base + p - 1]];
      }
    }
    int carry_b = s_carry_b;
    int pex = block_excl_max(isb ? p : INT32_MIN, s_warp);
    int pp = max(pex, carry_b);
    bool changed = false;
    if (isb) {
      if (p == 0) {
        changed = true;
      } else {
        for (int b = 0; b < W && !changed; ++b) {
          changed = (pfk[(size_t)b * stride + p] != pfk[(size_t)b * stride + pp]) ||
                    (sfk[(size_t)b * stride + p] != sfk[(size_t)b * stride + pp]);
        }
      }
    }
    int total = 0;
    int row = block_excl_sum(changed ? 1 : 0, s_warp, &total);
    row += s_carry_rows;
    if (changed) {
      thrscratch[ext + row] = (p == 0) ? -INFINITY : lat[order[base + p - 1]];
      uint32_t* rr = rowscratch + (size_t)(ext + row) * (2 * W);
      for (int b = 0; b < W; ++b) {
        uint32_t a = pfk[(size_t)b * stride + p];
        uint32_t s = sfk[(size_t)b * stride + p];
        rr[b] = a;
        rr[W + b] = s;
        if (a != kInf32) candf[a] = 1u;
        if (s != kInf32) cands[s] = 1u;
      }
    }
    if (threadIdx.x == blockDim.x - 1) s_lastb = max(pp, isb ? p : INT32_MIN);
    __syncthreads();
    if (threadIdx.x == 0) {
      s_carry_b = max(s_carry_b, s_lastb);
      s_carry_rows += total;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) rows_per_kind[k] = s_carry_rows;
}

// Shared-memory variant of k_stair for kinds of at most kStairSmemMax entries (same output).
// The kind's positions are staged once — lane, r1, r2 and the latency-boundary flag, all loads
// in flight together — so the sequential scans run on shared memory instead of chains of
// dependent global loads:
//   phase A  warp w < 2W: lane b = w % W, direction w / W; each of its 32 threads owns a
//            contiguous run of positions (local minimum, warp exclusive scan, rewrite with the
//            carry), writing pf / sf for every position;
//   phase B  every thread owns a contiguous run of positions p in [0, Mk]: previous boundary
//            (block max-scan carry), "row changed" test against it, row numbers (block sum-scan
//            carry), row / threshold / candidate-flag writes.
constexpr int kStairSmemMax = 16384;
// Per-position arrays are laid out in 32 runs of S positions (S a power of two >= 128, one run
// per thread of a scanning warp) with one pad word after every run, so the 32 threads of a
// warp — each walking its own run — hit 32 different banks for 32-, 16- and 8-bit arrays.
__device__ __forceinline__ int i32(int q, int sh) { return q + (q >> sh); }
__device__ __forceinline__ int i16(int q, int sh) { return q + ((q >> sh) << 1); }
__device__ __forceinline__ int i8(int q, int sh) { return q + ((q >> sh) << 2); }
constexpr int kStairCap = kStairSmemMax + 160;  // positions 0..Mk plus the run pads
constexpr int kStairSmemBytes = 2 * kStairCap * 4 + kStairCap * 2 + 3 * kStairCap;
// Consecutive latency boundaries pp < p carry different rows iff some position of the group
// [pp, p) strictly improves its lane's running prefix minimum of r1 (scanning forward) or its
// running suffix minimum of r2 (scanning backward).  So: scan once to flag those positions,
// number the changed boundaries (= rows) with block scans, then scan again and write each
// lane's running minimum only where a row starts — no per-position pf / sf arrays.
__global__ void __launch_bounds__(1024) k_stair_smem(int M, int K, int W, KindInfo ki,
                                                     const int32_t* __restrict__ order,
                                                     const int32_t* __restrict__ bidx,
                                                     const double* __restrict__ lat,
                                                     const uint32_t* __restrict__ r1,
                                                     const uint32_t* __restrict__ r2,
                                                     double* thrscratch, uint32_t* rowscratch,
                                                     int32_t* rows_per_kind, uint32_t* candf,
                                                     uint32_t* cands) {
  extern __shared__ __align__(16) uint8_t s_st[];
  __shared__ int s_warp[32];
  const int k = blockIdx.x;
  const int Mk = ki.count[k];
  const int base = ki.base[k];
  const int ext = base + k;
  if (Mk == 0) {
    if (threadIdx.x == 0) rows_per_kind[k] = 0;
    return;
  }
  const int T = blockDim.x, t = threadIdx.x;
  int sh = 7;  // runs of S = 2^sh >= 128 positions, 32 runs cover Mk
  while ((32 << sh) < Mk + 1) ++sh;
  // rank | lane << 16 (ranks < 2^15 for plan tables)
  uint32_t* sr1 = reinterpret_cast<uint32_t*>(s_st);
  uint32_t* sr2 = sr1 + kStairCap;
  uint16_t* scnt = reinterpret_cast<uint16_t*>(sr2 + kStairCap);  // #flags before p
  uint16_t* srow = scnt;  // then: row starting at boundary p, or 0xFFFF
  uint8_t* sisb = reinterpret_cast<uint8_t*>(scnt + kStairCap);  // lat[q] != lat[q - 1]
  uint8_t* simpP = sisb + kStairCap;   // q improves its lane's prefix min of r1
  uint8_t* simpS = simpP + kStairCap;  // q improves its lane's suffix min of r2
  // ---- stage (several independent loads per thread in flight) ----
  for (int q0 = t; q0 < Mk; q0 += 4 * T) {
    int e[4], e1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * T;
      e[u] = q < Mk ? order[base + q] : 0;
      e1[u] = (q < Mk && q > 0) ? order[base + q - 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * T;
      if (q < Mk) {
        const uint32_t ln = (uint32_t)bidx[e[u]] << 16;
        sr1[i32(q, sh)] = r1[e[u]] | ln;
        sr2[i32(q, sh)] = r2[e[u]] | ln;
        sisb[i8(q, sh)] = q > 0 && lat[e[u]] != lat[e1[u]];
      }
    }
  }
  __syncthreads();
  const int w = t >> 5, l = t & 31;
  const int a0 = min(l << sh, Mk), a1 = min(a0 + (1 << sh), Mk);
  // inside a run, position q sits at q + l (32-bit), q + 2l (16-bit), q + 4l (8-bit)
  // lane carries of warp w < 2W (lane b = w % W, forward for w < W, backward otherwise)
  uint32_t carry = kInf32;
  // ---- phase A: flag improving positions ----
  if (w < 2 * W) {
    const uint32_t b = (uint32_t)(w % W);
    const bool suf = w >= W;
    const uint32_t* v = suf ? sr2 : sr1;
    uint32_t m = kInf32;
    for (int q = a0; q < a1; ++q) {
      const uint32_t x = v[q + l];
      m = ((x >> 16) == b) ? min(m, x & 0xFFFFu) : m;
    }
    if (!suf) {
      const uint32_t incl = warp_incl_min(m, l);
      carry = __shfl_up_sync(0xffffffffu, incl, 1);
      if (l == 0) carry = kInf32;
      uint32_t run = carry;
      for (int q = a0; q < a1; ++q) {
        const uint32_t x = v[q + l];
        if ((x >> 16) == b) {
          const uint32_t r = x & 0xFFFFu;
          simpP[q + 4 * l] = r < run;
          run = min(run, r);
        }
      }
    } else {
      uint32_t x = m;  // exclusive over the lanes after l
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, x, off);
        if (l + off < 32) x = min(x, y);
      }
      carry = __shfl_down_sync(0xffffffffu, x, 1);
      if (l == 31) carry = kInf32;
      uint32_t run = carry;
      for (int q = a1 - 1; q >= a0; --q) {
        const uint32_t y = v[q + l];
        if ((y >> 16) == b) {
          const uint32_t r = y & 0xFFFFu;
          simpS[q + 4 * l] = r < run;
          run = min(run, r);
        }
      }
    }
  }
  __syncthreads();
  // ---- phase B: boundaries p in [0, Mk] (each thread a contiguous run) -> rows ----
  const int n = Mk + 1;
  const int P = (n + T - 1) / T;
  const int p0 = min(t * P, n), p1 = min(p0 + P, n);
  int lastb = INT32_MIN, nf = 0;
  for (int p = p0; p < p1; ++p) {
    if (p == 0 || p == Mk || sisb[i8(p, sh)]) lastb = p;
    if (p < Mk) nf += (simpP[i8(p, sh)] | simpS[i8(p, sh)]) != 0;
  }
  int tot_f = 0;
  int cf = block_excl_sum(nf, s_warp, &tot_f);
  const int prevb = block_excl_max(lastb, s_warp);  // last boundary before this run
  for (int p = p0; p < p1; ++p) {
    scnt[i16(p, sh)] = (uint16_t)cf;
    if (p < Mk) cf += (simpP[i8(p, sh)] | simpS[i8(p, sh)]) != 0;
  }
  __syncthreads();
  uint32_t chmask = 0;  // changed boundaries of this run (P <= 17 for Mk <= 16384)
  int cnt = 0;
  {
    int pp = prevb;
    for (int p = p0; p < p1; ++p) {
      if (!(p == 0 || p == Mk || sisb[i8(p, sh)])) continue;
      if ((p == 0) || scnt[i16(p, sh)] > scnt[i16(pp, sh)]) {
        chmask |= 1u << (p - p0);
        ++cnt;
      }
      pp = p;
    }
  }
  int total = 0;
  int row = block_excl_sum(cnt, s_warp, &total);
  for (int p = p0; p < p1; ++p) {
    const bool ch = (chmask >> (p - p0)) & 1u;
    srow[i16(p, sh)] = ch ? (uint16_t)row : (uint16_t)0xFFFFu;
    if (ch) {
      thrscratch[ext + row] = (p == 0) ? -INFINITY : lat[order[base + p - 1]];
      ++row;
    }
  }
  __syncthreads();
  // ---- phase A again: each lane's running minimum where a row starts ----
  if (w < 2 * W) {
    const uint32_t b = (uint32_t)(w % W);
    const bool suf = w >= W;
    const uint32_t* v = suf ? sr2 : sr1;
    uint32_t run = carry;
    if (!suf) {
      for (int q = a0; q < a1; ++q) {  // row at boundary q: min r1 over positions < q
        const uint32_t rw = srow[q + 2 * l];
        if (rw != 0xFFFFu) {
          rowscratch[(size_t)(ext + rw) * (2 * W) + b] = run;
          if (run != kInf32) candf[run] = 1u;
        }
        const uint32_t x = v[q + l];
        run = ((x >> 16) == b) ? min(run, x & 0xFFFFu) : run;
      }
      if (a1 == Mk && a0 < a1) {  // boundary Mk: the whole-kind minimum
        const uint32_t rw = srow[i16(Mk, sh)];
        if (rw != 0xFFFFu) {
          rowscratch[(size_t)(ext + rw) * (2 * W) + b] = run;
          if (run != kInf32) candf[run] = 1u;
        }
      }
    } else {
      for (int q = a1 - 1; q >= a0; --q) {  // row at boundary q: min r2 over positions >= q
        const uint32_t y = v[q + l];
        run = ((y >> 16) == b) ? min(run, y & 0xFFFFu) : run;
        const uint32_t rw = srow[q + 2 * l];
        if (rw != 0xFFFFu) {
          rowscratch[(size_t)(ext + rw) * (2 * W) + W + b] = run;
          if (run != kInf32) cands[run] = 1u;
        }
      }
      if (l == 0) {
        const uint32_t rw = srow[i16(Mk, sh)];
        if (rw != 0xFFFFu) rowscratch[(size_t)(ext + rw) * (2 * W) + W + b] = kInf32;
      }
    }
  }
  if (t == 0) rows_per_kind[k] = total;
}

// ---- k_stair_lanes: the staircase by per-lane segmented scans (kinds of <= 8192 entries) ---
// Same output as k_stair.  The kind's positions are bucketed by batch lane (a stable counting
// sort inside the CTA), so each lane's prefix minimum of r1 and suffix minimum of r2 is a
// segmented scan over that lane's own positions only — one block-wide scan per direction for
// all lanes together instead of one scan of every position per lane.  "Improving" positions
// (strictly below their lane's running minimum) flag the latency groups whose boundary starts
// a new row (see k_stair_smem); a row's lane values are read from the scanned lane lists at
// (#lane positions before the boundary).
constexpr int kStairLanesMax = 8192;
constexpr int kFinChunk = 256;  // entries per compaction chunk (<= 1024 chunks: M <= 262,144)
constexpr int kStairLanesPer = (kStairLanesMax + 1 + 1023) / 1024;  // boundaries per thread

// exclusive block scan of NW packed u32 words (two 16-bit counters each)
template <int NW>
__device__ __forceinline__ void block_excl_sum_vec(uint32_t (&v)[NW], uint32_t (&tot)[NW],
                                                   uint32_t* s_w /* 32 * NW */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    x[q] = v[q];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x[q], off);
      if (lane >= off) x[q] += y;
    }
    if (lane == 31) s_w[w * NW + q] = x[q];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      uint32_t y = lane < nw ? s_w[lane * NW + q] : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, off);
        if (lane >= off) y += z;
      }
      s_w[lane * NW + q] = y;  // inclusive over warps
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const uint32_t base = w ? s_w[(w - 1) * NW + q] : 0u;
    tot[q] = s_w[(nw - 1) * NW + q];
    v[q] = base + x[q] - v[q];
  }
  __syncthreads();
}

// segmented scan operator on (segment, value): the running minimum restarts at a new segment
struct SegMin {
  uint32_t seg, val;
};
__device__ __forceinline__ SegMin seg_combine(SegMin a, SegMin b) {
  SegMin r;
  r.seg = b.seg;
  r.val = a.seg == b.seg ? min(a.val, b.val) : b.val;
  return r;
}
// exclusive block scan with SegMin; threads in order of `rank` (0..T-1)
__device__ __forceinline__ SegMin block_excl_segmin(SegMin v, int rank, uint32_t* s_seg,
                                                    uint32_t* s_val) {
  const int lane = rank & 31, w = rank >> 5, nw = blockDim.x >> 5;
  // warp shuffles follow the hardware lane order; `rank` is threadIdx.x or its mirror, so
  // warp membership is preserved and the lane order inside a warp is either kept or reversed
  const bool mirror = rank != (int)threadIdx.x;
  SegMin x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    SegMin y;
    y.seg = mirror ? __shfl_down_sync(0xffffffffu, x.seg, off) : __shfl_up_sync(0xffffffffu, x.seg, off);
    y.val = mirror ? __shfl_down_sync(0xffffffffu, x.val, off) : __shfl_up_sync(0xffffffffu, x.val, off);
    if (lane >= off) x = seg_combine(y, x);
  }
  if (lane == 31) {
    s_seg[w] = x.seg;
    s_val[w] = x.val;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    SegMin y;
    y.seg = l < nw ? s_seg[l] : 0xFFFFFFFFu;
    y.val = l < nw ? s_val[l] : kInf32;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      SegMin z;
      z.seg = __shfl_up_sync(0xffffffffu, y.seg, off);
      z.val = __shfl_up_sync(0xffffffffu, y.val, off);
      if (l >= off) y = seg_combine(z, y);
    }
    __syncwarp();
    s_seg[32 + l] = y.seg;  // inclusive over warps (in rank order)
    s_val[32 + l] = y.val;
  }
  __syncthreads();
  // exclusive: the inclusive value of the previous rank
  SegMin prev;
  SegMin xin;
  xin.seg = mirror ? __shfl_down_sync(0xffffffffu, x.seg, 1) : __shfl_up_sync(0xffffffffu, x.seg, 1);
  xin.val = mirror ? __shfl_down_sync(0xffffffffu, x.val, 1) : __shfl_up_sync(0xffffffffu, x.val, 1);
  if (lane == 0) {
    if (w == 0) {
      prev.seg = 0xFFFFFFFFu;
      prev.val = kInf32;
    } else {
      prev.seg = s_seg[32 + w - 1];
      prev.val = s_val[32 + w - 1];
    }
  } else {
    prev = xin;
    if (w > 0) {
      SegMin carry;
      carry.seg = s_seg[32 + w - 1];
      carry.val = s_val[32 + w - 1];
      prev = seg_combine(carry, prev);
    }
  }
  __syncthreads();
  return prev;
}

// Per position q of the kind-major latency order (entry e = order[q]): {r1[e], r2[e]},
// lane | (latency differs from the previous position of the kind) << 7, and lat[e] — the
// gathers of k_stair_lanes' staging spread over every SM instead of one CTA per kind.
__global__ void k_stair_stage(int M, int K, const __grid_constant__ KindInfo ki,
                              const int32_t* __restrict__ order, const int32_t* __restrict__ bidx,
                              const double* __restrict__ lat, const uint32_t* __restrict__ r1,
                              const uint32_t* __restrict__ r2, uint2* pos_r12, uint8_t* pos_meta,
                              double* pos_lat) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= M) return;
  bool first = false;
  for (int k = 0; k < K; ++k) first |= q == ki.base[k];
  const int e = order[q];
  const double l = lat[e];
  const bool sisb = !first && q > 0 && l != lat[order[q - 1]];
  pos_r12[q] = make_uint2(r1[e], r2[e]);
  pos_meta[q] = (uint8_t)(bidx[e] | (sisb ? 0x80 : 0));
  pos_lat[q] = l;
}

template <int NWW>  // NWW = W / 2 packed words (W = 8 -> 4, W = 16 -> 8)
__global__ void __launch_bounds__(1024) k_stair_lanes(int M, int K, int W, KindInfo ki,
                                                      const int32_t* __restrict__ order,
                                                      const int32_t* __restrict__ bidx,
                                                      const double* __restrict__ lat,
                                                      const uint32_t* __restrict__ r1,
                                                      const uint32_t* __restrict__ r2,
                                                      double* thrscratch, uint32_t* rowscratch,
                                                      int32_t* rows_per_kind, uint32_t* candf,
                                                      uint32_t* cands,
                                                      const uint2* __restrict__ pos_r12,
                                                      const uint8_t* __restrict__ pos_meta,
                                                      const double* __restrict__ pos_lat) {
  constexpr int WM = 2 * NWW;  // lanes held in registers
  extern __shared__ __align__(16) uint8_t s_l[];
  __shared__ int s_warp[32];
  __shared__ uint32_t s_w[32 * NWW], s_seg[64], s_val[64];
  __shared__ int s_start[WM + 1];
  const int k = blockIdx.x;
  const int Mk = ki.count[k];
  const int base = ki.base[k];
  const int ext = base + k;
  if (Mk == 0) {
    if (threadIdx.x == 0) rows_per_kind[k] = 0;
    return;
  }
  const int T = blockDim.x, t = threadIdx.x;
  constexpr int C = kStairLanesMax;
  uint32_t* pr1 = reinterpret_cast<uint32_t*>(s_l);  // position order (reused as scnt later)
  uint32_t* pr2 = pr1 + C;
  uint32_t* L1 = pr2 + C;       // lane order: r1, then the inclusive prefix minimum
  uint32_t* L2 = L1 + C;        // lane order: r2, then the inclusive suffix minimum
  uint16_t* Lpos = reinterpret_cast<uint16_t*>(L2 + C);
  uint8_t* plane = reinterpret_cast<uint8_t*>(Lpos + C);
  uint8_t* Llane = plane + C;
  uint8_t* sisb = Llane + C;    // lat[q] != lat[q - 1]
  uint8_t* impP = sisb + C;
  uint8_t* impS = impP + C;
  uint16_t* scnt = reinterpret_cast<uint16_t*>(pr1);  // #flags before p (after the scatter)
  // ---- 1. stage (coalesced: k_stair_stage gathered the per-position records) ----
  for (int q0 = t; q0 < Mk; q0 += 4 * T) {
    uint2 rr[4];
    uint32_t mm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * T;
      rr[u] = q < Mk ? pos_r12[base + q] : make_uint2(0u, 0u);
      mm[u] = q < Mk ? pos_meta[base + q] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * T;
      if (q < Mk) {
        plane[q] = (uint8_t)(mm[u] & 0x7Fu);
        pr1[q] = rr[u].x;
        pr2[q] = rr[u].y;
        sisb[q] = (uint8_t)(mm[u] >> 7);
      }
    }
  }
  __syncthreads();
  // ---- 2. per-thread chunk lane counts, block scan -> lane list offsets ----
  const int n = Mk + 1;  // boundaries 0..Mk; positions 0..Mk-1
  const int P = (n + T - 1) / T;
  const int p0 = min(t * P, n), p1 = min(p0 + P, n);
  uint32_t cw[NWW], tw[NWW];
#pragma unroll
  for (int q = 0; q < NWW; ++q) cw[q] = 0u;
  for (int p = p0; p < min(p1, Mk); ++p) {
    const int l = plane[p];
#pragma unroll
    for (int q = 0; q < NWW; ++q) cw[q] += (l == 2 * q ? 1u : 0u) | (l == 2 * q + 1 ? 0x10000u : 0u);
  }
  block_excl_sum_vec<NWW>(cw, tw, s_w);
  if (t == 0) {
    int acc = 0;
    for (int b = 0; b < WM; ++b) {
      s_start[b] = acc;
      acc += (int)((tw[b >> 1] >> (16 * (b & 1))) & 0xFFFFu);
    }
    s_start[WM] = acc;
  }
  __syncthreads();
  uint32_t before[WM];  // #lane-b positions before this thread's chunk
#pragma unroll
  for (int b = 0; b < WM; ++b) before[b] = (cw[b >> 1] >> (16 * (b & 1))) & 0xFFFFu;
  {  // ---- 3. stable scatter into lane order ----
    uint32_t run[WM];
#pragma unroll
    for (int b = 0; b < WM; ++b) run[b] = before[b];
    for (int p = p0; p < min(p1, Mk); ++p) {
      const int l = plane[p];
      uint32_t at = 0;
#pragma unroll
      for (int b = 0; b < WM; ++b) {
        at = (l == b) ? (uint32_t)s_start[b] + run[b] : at;
        run[b] += (l == b);
      }
      L1[at] = pr1[p];
      L2[at] = pr2[p];
      Lpos[at] = (uint16_t)p;
      Llane[at] = (uint8_t)l;
    }
  }
  __syncthreads();
  // ---- 4. segmented prefix minimum of r1 (forward) and suffix minimum of r2 (backward) ----
  const int E = (Mk + T - 1) / T;  // list elements per thread
  const int j0 = min(t * E, Mk), j1 = min(j0 + E, Mk);
  // a full chunk of 8 is moved with vector shared-memory accesses (one LDS.64 / LDS.128 per
  // array instead of eight 4-byte loads at an 8-word stride, which conflict 8 ways)
  const bool vec = E == 8 && j1 - j0 == 8;
  uint32_t vl[8], v1[8], v2[8], vp[8];
  if (vec) {
    const uint2 ll = *reinterpret_cast<const uint2*>(Llane + j0);
    const uint4 a0 = *reinterpret_cast<const uint4*>(L1 + j0);
    const uint4 a1 = *reinterpret_cast<const uint4*>(L1 + j0 + 4);
    const uint4 b0 = *reinterpret_cast<const uint4*>(L2 + j0);
    const uint4 b1 = *reinterpret_cast<const uint4*>(L2 + j0 + 4);
    const uint4 pp = *reinterpret_cast<const uint4*>(Lpos + j0);
#pragma unroll
    for (int u = 0; u < 8; ++u) vl[u] = ((u < 4 ? ll.x : ll.y) >> (8 * (u & 3))) & 0xFFu;
    v1[0] = a0.x; v1[1] = a0.y; v1[2] = a0.z; v1[3] = a0.w;
    v1[4] = a1.x; v1[5] = a1.y; v1[6] = a1.z; v1[7] = a1.w;
    v2[0] = b0.x; v2[1] = b0.y; v2[2] = b0.z; v2[3] = b0.w;
    v2[4] = b1.x; v2[5] = b1.y; v2[6] = b1.z; v2[7] = b1.w;
    const uint32_t pw[4] = {pp.x, pp.y, pp.z, pp.w};
#pragma unroll
    for (int u = 0; u < 8; ++u) vp[u] = (pw[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
  }
  {
    SegMin a;
    a.seg = 0xFFFFFFFFu;
    a.val = kInf32;
    if (vec) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        SegMin x;
        x.seg = vl[u];
        x.val = v1[u];
        a = (a.seg == 0xFFFFFFFFu) ? x : seg_combine(a, x);
      }
    } else {
      for (int j = j0; j < j1; ++j) {
        SegMin x;
        x.seg = Llane[j];
        x.val = L1[j];
        a = (a.seg == 0xFFFFFFFFu) ? x : seg_combine(a, x);
      }
    }
    if (j0 >= j1) a.seg = 0xFFFFFFFEu;  // empty chunk: passes nothing on
    SegMin c = block_excl_segmin(a, t, s_seg, s_val);
    uint32_t rn = kInf32;
    uint32_t sg = 0xFFFFFFFFu;
    if (j0 < j1 && c.seg == (vec ? vl[0] : (uint32_t)Llane[j0])) rn = c.val;
    if (vec) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (vl[u] != sg && u != 0) rn = kInf32;
        sg = vl[u];
        impP[vp[u]] = v1[u] < rn;
        rn = min(rn, v1[u]);
        v1[u] = rn;  // inclusive prefix minimum inside the lane
      }
      *reinterpret_cast<uint4*>(L1 + j0) = make_uint4(v1[0], v1[1], v1[2], v1[3]);
      *reinterpret_cast<uint4*>(L1 + j0 + 4) = make_uint4(v1[4], v1[5], v1[6], v1[7]);
    } else {
      for (int j = j0; j < j1; ++j) {
        const uint32_t l = Llane[j];
        if (l != sg && j != j0) rn = kInf32;
        sg = l;
        const uint32_t v = L1[j];
        impP[Lpos[j]] = v < rn;
        rn = min(rn, v);
        L1[j] = rn;  // inclusive prefix minimum inside the lane
      }
    }
  }
  {
    const int tm = T - 1 - t;  // mirrored rank: the scan runs from the end of the list
    const int k0 = j0, k1 = j1;  // same chunk, processed backwards: k1 - 1, ..., k0
    SegMin a;
    a.seg = 0xFFFFFFFFu;
    a.val = kInf32;
    if (vec) {
#pragma unroll
      for (int u = 7; u >= 0; --u) {
        SegMin x;
        x.seg = vl[u];
        x.val = v2[u];
        a = (a.seg == 0xFFFFFFFFu) ? x : seg_combine(a, x);
      }
    } else {
      for (int j = k1 - 1; j >= k0; --j) {
        SegMin x;
        x.seg = Llane[j];
        x.val = L2[j];
        a = (a.seg == 0xFFFFFFFFu) ? x : seg_combine(a, x);
      }
    }
    if (k0 >= k1) a.seg = 0xFFFFFFFEu;
    SegMin c = block_excl_segmin(a, tm, s_seg, s_val);
    uint32_t rn = kInf32;
    uint32_t sg = 0xFFFFFFFFu;
    if (k0 < k1 && c.seg == (vec ? vl[7] : (uint32_t)Llane[k1 - 1])) rn = c.val;
    if (vec) {
#pragma unroll
      for (int u = 7; u >= 0; --u) {
        if (vl[u] != sg && u != 7) rn = kInf32;
        sg = vl[u];
        impS[vp[u]] = v2[u] < rn;
        rn = min(rn, v2[u]);
        v2[u] = rn;  // inclusive suffix minimum inside the lane
      }
      *reinterpret_cast<uint4*>(L2 + j0) = make_uint4(v2[0], v2[1], v2[2], v2[3]);
      *reinterpret_cast<uint4*>(L2 + j0 + 4) = make_uint4(v2[4], v2[5], v2[6], v2[7]);
    } else {
      for (int j = k1 - 1; j >= k0; --j) {
        const uint32_t l = Llane[j];
        if (l != sg && j != k1 - 1) rn = kInf32;
        sg = l;
        const uint32_t v = L2[j];
        impS[Lpos[j]] = v < rn;
        rn = min(rn, v);
        L2[j] = rn;  // inclusive suffix minimum inside the lane
      }
    }
  }
  __syncthreads();
  // ---- 5. boundaries -> rows ----
  int lastb = INT32_MIN, nf = 0;
  for (int p = p0; p < p1; ++p) {
    if (p == 0 || p == Mk || sisb[p]) lastb = p;
    if (p < Mk) nf += (impP[p] | impS[p]) != 0;
  }
  int tot_f = 0;
  int cf = block_excl_sum(nf, s_warp, &tot_f);
  const int prevb = block_excl_max(lastb, s_warp);
  for (int p = p0; p < p1; ++p) {
    scnt[p] = (uint16_t)cf;
    if (p < Mk) cf += (impP[p] | impS[p]) != 0;
  }
  __syncthreads();
  uint32_t chmask = 0;
  int cnt = 0;
  {
    int pp = prevb;
    for (int p = p0; p < p1; ++p) {
      if (!(p == 0 || p == Mk || sisb[p])) continue;
      if ((p == 0) || scnt[p] > scnt[pp]) {
        chmask |= 1u << (p - p0);
        ++cnt;
      }
      pp = p;
    }
  }
  int total = 0;
  int row = block_excl_sum(cnt, s_warp, &total);
  // Rows are written cooperatively: each boundary position goes to rowp[row] (pr2 is dead since
  // the scatter), then the block writes the rows word by word — consecutive threads on
  // consecutive words, so the row stores are coalesced and the candidate flags spread over the
  // whole CTA; a word's lane count before the boundary is a lower bound in the lane's
  // ascending position list.
  uint16_t* rowp = reinterpret_cast<uint16_t*>(pr2);
#pragma unroll
  for (int u = 0; u < kStairLanesPer; ++u) {
    const int p = p0 + u;
    if (p >= p1) break;
    if ((chmask >> u) & 1u) rowp[row++] = (uint16_t)p;
  }
  __syncthreads();
  const int W2 = 2 * W;
  for (int j = t; j < total * W2; j += T) {
    const int rw = j / W2, b2 = j - rw * W2;
    const int p = rowp[rw];
    if (b2 == 0) thrscratch[ext + rw] = p > 0 ? pos_lat[base + p - 1] : -INFINITY;
    const int b = b2 < W ? b2 : b2 - W;
    const int st = s_start[b], nb = s_start[b + 1] - st;
    int lo = 0, hi = nb;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)Lpos[st + mid] < p) lo = mid + 1; else hi = mid;
    }
    uint32_t v;
    if (b2 < W) {  // best feasible entry of lane b among positions before the boundary
      v = lo > 0 ? L1[st + lo - 1] : kInf32;
      if (v != kInf32) candf[v] = 1u;
    } else {       // best penalized entry of lane b among positions from the boundary on
      v = lo < nb ? L2[st + lo] : kInf32;
      if (v != kInf32) cands[v] = 1u;
    }
    rowscratch[(size_t)(ext + rw) * W2 + b2] = v;
  }
  if (t == 0) rows_per_kind[k] = total;
}
constexpr int kStairLanesSmem = kStairLanesMax * (4 * 4 + 2 + 5);

// (score, r1) strict order of unified candidates
__device__ __forceinline__ bool key_lt(double sa, uint32_t ra, double sb, uint32_t rb) {
  return sa < sb || (sa == sb && ra < rb);
}

// Plan finalisation, four kernels (multi-CTA where the work is parallel):
//   k_fin_head   one CTA: order-preserving compaction of the two candidate sets (cidf / cids),
//                then the header (section offsets, per-kind bucket geometry) written to the
//                image — or an invalid magic when the image would not fit
//   k_fin_keys   per candidate its (score, r1) key: CP[c] (feasible side) in r1 order, CS[c]
//                (penalized side) in r2 order; both lists ascend in (score, r1)
//   k_fin_merge  unified ids: own position + #keys of the other list before it
//   k_fin_fill   lane lookup table, thresholds, staircase rows, buckets, candidate records
// candidate counts of every 256-entry chunk (the compaction of the two candidate sets runs over
// many CTAs: counts here, one scan of the chunk counts in k_fin_head, the in-chunk scan and the
// ids in k_fin_keys)
__global__ void __launch_bounds__(kFinChunk) k_fin_count(int M, const uint32_t* __restrict__ candf,
                                                        const uint32_t* __restrict__ cands,
                                                        int2* chunk_cnt) {
  const int r = blockIdx.x * kFinChunk + threadIdx.x;
  const int nf = __syncthreads_count(r < M && candf[r] != 0);
  const int ns = __syncthreads_count(r < M && cands[r] != 0);
  if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = make_int2(nf, ns);
}

__global__ void __launch_bounds__(1024) k_fin_head(
    int M, int K, int nB, KindInfo ki, const int32_t* __restrict__ rows_per_kind,
    const double* __restrict__ thrscratch, int nchunks, const int2* __restrict__ chunk_cnt,
    int2* chunk_base, PlanHdr hdr_in, uint8_t* image, int64_t image_cap, int32_t* status) {
  __shared__ int s_warp[32];
  __shared__ PlanHdr hdr;
  __shared__ int s_ncp, s_ncs;
  {  // exclusive scan of the per-chunk counts (nchunks <= blockDim.x)
    const int2 c = (int)threadIdx.x < nchunks ? chunk_cnt[threadIdx.x] : make_int2(0, 0);
    int tf = 0, ts = 0;
    const int bf = block_excl_sum(c.x, s_warp, &tf);
    const int bs = block_excl_sum(c.y, s_warp, &ts);
    if ((int)threadIdx.x < nchunks) chunk_base[threadIdx.x] = make_int2(bf, bs);
    if (threadIdx.x == 0) {
      s_ncp = tf;
      s_ncs = ts;
    }
    __syncthreads();
  }
  const int ncp = s_ncp, ncs = s_ncs;
  // per-kind bucket geometry in parallel (one thread per kind), offsets by thread 0
  __shared__ KindDesc s_kd[kMaxKinds];
  if (threadIdx.x < kMaxKinds) {
    const int k = threadIdx.x;
    KindDesc d;
    memset(&d, 0, sizeof(d));
    const int R = k < K ? rows_per_kind[k] : 0;
    d.R = R;
    if (R > 0) {
      const int ext = ki.base[k] + k;
      int nbk = 1, shift = 0;
      uint32_t kmin = 0;
      if (R >= 2) {
        // positive thresholds: the high word of the encoding is monotone
        const double t1 = thrscratch[ext + 1];
        kmin = (uint32_t)__double2hiint(t1);
        const uint32_t kmax = (uint32_t)__double2hiint(thrscratch[ext + R - 1]);
        while (nbk < 2 * (R - 1) && nbk < kMaxBuckets) nbk <<= 1;
        while (((kmax - kmin) >> shift) >= (uint32_t)nbk) ++shift;
        d.pad[0] = !(t1 > 0.0);  // non-positive latency: generic search
      }
      d.kmin_hi = kmin;
      d.nb1_shift = (uint32_t)(nbk - 1) | ((uint32_t)shift << 16);
    }
    s_kd[k] = d;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    hdr = hdr_in;
    hdr.row_stride = ((nB * (nB + 1) + 3) / 4) * 4;  // nB(nB+1)/2 u16, 4-byte aligned
    int off = (int)sizeof(PlanHdr);
    int maxB = 0;
    for (int b = 0; b < nB; ++b) maxB = max(maxB, hdr.batch_vals[b]);
    // entries 0..maxB plus one saturating entry for every value above maxB
    hdr.lut_n = (maxB + 2 <= kMaxLut) ? maxB + 2 : 0;
    hdr.lut_off = off;
    off += ((hdr.lut_n * 2 + 15) / 16) * 16;
    for (int k = 0; k < kMaxKinds; ++k) {
      KindDesc d = s_kd[k];
      const int R = d.R;
      if (R > 0) {
        d.thr_off = off;
        off += ((R * 8 + 15) / 16) * 16;
        d.rows_off = off;
        off += ((R * hdr.row_stride + 15) / 16) * 16;
        d.bkt_off = off;
        off += (((int)(d.nb1_shift & 0xFFFFu) + 1) * 4 + 15) / 16 * 16;
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
    const bool ok = off <= image_cap && ncp + ncs < (int)kNone16;
    *status = ok ? 0 : -1;
    if (!ok) hdr.magic = 0;  // invalid image: every later stage and every reader stops
  }
  __syncthreads();
  if (threadIdx.x < (int)(sizeof(PlanHdr) / 4))
    reinterpret_cast<uint32_t*>(image)[threadIdx.x] =
        reinterpret_cast<const uint32_t*>(&hdr)[threadIdx.x];
}

__global__ void __launch_bounds__(kFinChunk) k_fin_keys(
    int M, const uint8_t* __restrict__ image, const uint32_t* __restrict__ candf,
    const uint32_t* __restrict__ cands, const int2* __restrict__ chunk_base, uint32_t* cidf,
    uint32_t* cids, const int32_t* __restrict__ ent_r1, const int32_t* __restrict__ ent_r2,
    const uint32_t* __restrict__ r1, const double* __restrict__ cost,
    const double* __restrict__ costpen, double* ukey, uint32_t* ukr, int32_t* uent) {
  const PlanHdr* H = reinterpret_cast<const PlanHdr*>(image);
  if (H->magic != kPlanMagic) return;
  const int ncp = H->ncp;
  const int r = blockIdx.x * kFinChunk + threadIdx.x;
  // compaction ids: chunk base + exclusive count inside the chunk (order-preserving)
  __shared__ int s_wf[kFinChunk / 32], s_ws[kFinChunk / 32];
  const bool f = r < M && candf[r] != 0, sflag = r < M && cands[r] != 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bf = __ballot_sync(0xffffffffu, f), bs = __ballot_sync(0xffffffffu, sflag);
  const uint32_t below = (1u << lane) - 1u;
  if (lane == 0) {
    s_wf[w] = __popc(bf);
    s_ws[w] = __popc(bs);
  }
  __syncthreads();
  int of = __popc(bf & below), os = __popc(bs & below);
  for (int q = 0; q < w; ++q) {
    of += s_wf[q];
    os += s_ws[q];
  }
  const int2 base = chunk_base[blockIdx.x];
  if (r >= M) return;
  cidf[r] = (uint32_t)(base.x + of);
  cids[r] = (uint32_t)(base.y + os);
  if (f) {
    const int c = base.x + of, e = ent_r1[r];
    ukey[c] = cost[e];
    ukr[c] = (uint32_t)r;
    uent[c] = e;
  }
  if (sflag) {
    const int c = ncp + base.y + os, e = ent_r2[r];
    ukey[c] = costpen[e];
    ukr[c] = r1[e];
    uent[c] = e;
  }
}

// ties (which only occur for the two sides of one entry when the penalty is 0) put CP first
__global__ void k_fin_merge(const uint8_t* __restrict__ image, const double* __restrict__ ukey,
                            const uint32_t* __restrict__ ukr, uint32_t* umap) {
  const PlanHdr* H = reinterpret_cast<const PlanHdr*>(image);
  if (H->magic != kPlanMagic) return;
  const int ncp = H->ncp, ncs = H->ncs;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncp + ncs) return;
  const bool is_cp = c < ncp;
  const double s = ukey[c];
  const uint32_t rr = ukr[c];
  int lo = is_cp ? ncp : 0, hi = is_cp ? ncp + ncs : ncp;
  const int base = lo;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool before = is_cp ? key_lt(ukey[mid], ukr[mid], s, rr)
                              : !key_lt(s, rr, ukey[mid], ukr[mid]);
    if (before) lo = mid + 1; else hi = mid;
  }
  umap[c] = (uint32_t)((is_cp ? c : c - ncp) + (lo - base));
}

// bucket tables, one CTA per kind (runs beside the row / record fill)
__global__ void __launch_bounds__(1024) k_fin_buckets(KindInfo ki, const double* __restrict__ thrscratch,
                                                      uint8_t* image) {
  const PlanHdr* H = reinterpret_cast<const PlanHdr*>(image);
  if (H->magic != kPlanMagic) return;
  // bucket b holds thresholds j in [1, R) with (key_j - kmin) >> shift == b:
  // entry = (#thresholds in lower buckets) | (#thresholds in b) << 16 — CTA k builds kind k's
  // table from a shared-memory histogram and one block scan (no per-bucket searches)
  {
    __shared__ uint32_t s_h[kMaxBuckets];
    __shared__ int s_warp[32];
    const int k = blockIdx.x;
    const KindDesc d = H->kd[k];
    const int R = d.R;
    if (R > 0) {
      const int ext = ki.base[k] + k;
      uint32_t* bkt = reinterpret_cast<uint32_t*>(image + d.bkt_off);
      const int nbk = (int)(d.nb1_shift & 0xFFFFu) + 1, shift = (int)(d.nb1_shift >> 16);
      const uint32_t kmin = d.kmin_hi;
      for (int b = threadIdx.x; b < nbk; b += blockDim.x) s_h[b] = 0u;
      __syncthreads();
      for (int j0 = 1 + (int)threadIdx.x; j0 < R; j0 += 8 * blockDim.x) {
        double tv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + u * blockDim.x;
          tv[u] = j < R ? thrscratch[ext + j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (j0 + u * (int)blockDim.x >= R) break;
          const uint32_t kk = (uint32_t)__double2hiint(tv[u]);
          atomicAdd(&s_h[min((kk - kmin) >> shift, (uint32_t)(nbk - 1))], 1u);
        }
      }
      __syncthreads();
      const int per = (nbk + blockDim.x - 1) / blockDim.x;
      const int b0 = min((int)threadIdx.x * per, nbk), b1 = min(b0 + per, nbk);
      int loc = 0;
      for (int b = b0; b < b1; ++b) loc += (int)s_h[b];
      int tot = 0;
      int below = block_excl_sum(loc, s_warp, &tot);
      for (int b = b0; b < b1; ++b) {
        const uint32_t c = s_h[b];
        bkt[b] = (uint32_t)below | (c << 16);
        below += (int)c;
      }
    }
  }
}

__global__ void k_fin_fill(int K, int W, const __grid_constant__ KindInfo ki,
                           const double* __restrict__ thrscratch,
                           const uint32_t* __restrict__ rowscratch,
                           const uint32_t* __restrict__ cidf, const uint32_t* __restrict__ cids,
                           const double* __restrict__ ukey, const int32_t* __restrict__ uent,
                           const uint32_t* __restrict__ umap, const double* __restrict__ lat,
                           const int32_t* __restrict__ batch, const int32_t* __restrict__ kind,
                           uint8_t* image) {
  const PlanHdr* H = reinterpret_cast<const PlanHdr*>(image);
  if (H->magic != kPlanMagic) return;
  const int g = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int nB = H->nB, ncp = H->ncp, ncand = H->ncp + H->ncs;
  {  // batch lookup table of the generic kernels
    uint16_t* lut = reinterpret_cast<uint16_t*>(image + H->lut_off);
    for (int v = g; v < H->lut_n; v += gs) {
      int lo = 0, le = 0;
      for (int b = 0; b < nB; ++b) {
        lo += H->batch_vals[b] < v;
        le += H->batch_vals[b] <= v;
      }
      lut[v] = (uint16_t)(lo | (le << 8));
    }
  }
  for (int k = 0; k < K; ++k) {
    const KindDesc d = H->kd[k];
    const int R = d.R;
    if (R == 0) continue;
    const int ext = ki.base[k] + k;
    double* thr = reinterpret_cast<double*>(image + d.thr_off);
    for (int r = g; r < R; r += gs) thr[r] = thrscratch[ext + r];
    // row r: lane b = min(unified id of the best feasible, of the best penalized entry with
    // batch size batch_vals[b]); stored as the minimum over every lane interval [lo, hi] at
    // tri(lo) + hi - lo.  One warp per row: lane b resolves batch lane b (three independent
    // loads), every lane then folds one or more intervals from the shuffled lane values and the
    // row's nB(nB+1)/2 u16 are stored contiguously (thread-per-row stores were one sector per
    // lane and queued for ~20 us on the few SMs holding the rows)
    const int wg = g >> 5, nwg = gs >> 5, ln = threadIdx.x & 31;
    const int nq = nB * (nB + 1) / 2;
    for (int r = wg; r < R; r += nwg) {
      const uint32_t* rw = rowscratch + (size_t)(ext + r) * (2 * W);
      uint32_t v = kInf32;
      if (ln < nB) {
        const uint32_t a = rw[ln], c = rw[W + ln];
        const uint32_t ua = a != kInf32 ? umap[cidf[a]] : kInf32;
        const uint32_t us = c != kInf32 ? umap[ncp + cids[c]] : kInf32;
        v = min(ua, us);
      }
      uint16_t* out = reinterpret_cast<uint16_t*>(image + d.rows_off + (size_t)r * H->row_stride);
      for (int q0 = 0; q0 < nq; q0 += 32) {
        const int q = q0 + ln;
        int lo = 0, hi = -1;
        if (q < nq) {  // decode q -> (lo, hi)
          int rem = q;
          while (rem >= nB - lo) {
            rem -= nB - lo;
            ++lo;
          }
          hi = lo + rem;
        }
        uint32_t m = kInf32;
        for (int bb = 0; bb < nB; ++bb) {
          const uint32_t vb = __shfl_sync(0xffffffffu, v, bb);
          if (bb >= lo && bb <= hi) m = min(m, vb);
        }
        if (q < nq) out[q] = m == kInf32 ? kNone16 : (uint16_t)m;
      }
    }
  }
  double* rscore = reinterpret_cast<double*>(image + H->score_off);
  double* rlat = reinterpret_cast<double*>(image + H->lat_off);
  CandB* recb = reinterpret_cast<CandB*>(image + H->recb_off);
  for (int c = g; c < ncand; c += gs) {
    const int e = uent[c];
    const uint32_t u = umap[c];
    rscore[u] = ukey[c];
    rlat[u] = lat[e];
    CandB b;
    b.meta = (uint32_t)e | ((c < ncp ? 1u : 0u) << 16) | ((uint32_t)kind[e] << 17);
    b.batch = batch[e];
    recb[u] = b;
  }
}

int64_t plan_image_capacity(const sp_table* t, int W) {
  int64_t cap = sizeof(PlanHdr) + ((kMaxLut * 2 + 15) / 16) * 16;
  for (int k = 0; k < t->K; ++k) {
    int64_t R = t->kind_count[k] + 1;
    const int64_t stride = ((t->nB * (t->nB + 1) + 3) / 4) * 4;
    cap += ((R * 8 + 15) / 16) * 16 + ((R * stride + 15) / 16) * 16 + kMaxBuckets * 4;
  }
  cap += 2 * (int64_t)t->M * (int64_t)sizeof(CandRec);
  return (cap + 15) / 16 * 16;
}

int plan_width(const sp_table* t) { return t->nB <= 8 ? 8 : 16; }

}  // namespace

int plan_scratch_alloc(sp_table* t) {
  const int M = t->M, K = t->K;
  const int W = plan_width(t);
  size_t ext = (size_t)(M + K);
  SP_CUDA(cudaMalloc(&t->r1, sizeof(uint32_t) * M));
  SP_CUDA(cudaMalloc(&t->r2, sizeof(uint32_t) * M));
  SP_CUDA(cudaMalloc(&t->ent_r1, sizeof(int32_t) * M));
  SP_CUDA(cudaMalloc(&t->ent_r2, sizeof(int32_t) * M));
  SP_CUDA(cudaMalloc(&t->order, sizeof(int32_t) * M));
  {  // sort scratch: two tile buffers + two merged buffers of SItem
    const size_t n = (size_t)((M + kSortTile - 1) / kSortTile) * kSortTile;
    t->sort_tmp_bytes = 4 * n * sizeof(SItem) + 2 * n * sizeof(int32_t);
    SP_CUDA(cudaMalloc(&t->sort_tmp, t->sort_tmp_bytes));
  }
  if (t->plan_ok) {
    SP_CUDA(cudaMalloc(&t->pf, sizeof(uint32_t) * W * ext));
    SP_CUDA(cudaMalloc(&t->sf, sizeof(uint32_t) * W * ext));
    SP_CUDA(cudaMalloc(&t->rowscratch, sizeof(uint32_t) * 2 * W * ext));
    SP_CUDA(cudaMalloc(&t->thrscratch, sizeof(double) * ext));
    SP_CUDA(cudaMalloc(&t->rows_per_kind, sizeof(int32_t) * (kMaxKinds + 1)));
    SP_CUDA(cudaMalloc(&t->candf, sizeof(uint32_t) * M));
    SP_CUDA(cudaMalloc(&t->cands, sizeof(uint32_t) * M));
    SP_CUDA(cudaMalloc(&t->cidf, sizeof(uint32_t) * M));
    SP_CUDA(cudaMalloc(&t->cids, sizeof(uint32_t) * M));
    SP_CUDA(cudaMalloc(&t->fin_chunk, sizeof(int2) * 2 * ((M + kFinChunk - 1) / kFinChunk)));
    SP_CUDA(cudaMalloc(&t->pos_r12, sizeof(uint2) * M));
    SP_CUDA(cudaMalloc(&t->pos_meta, M));
    SP_CUDA(cudaMalloc(&t->pos_lat, sizeof(double) * M));
    SP_CUDA(cudaMalloc(&t->ukey, sizeof(double) * 2 * M));
    SP_CUDA(cudaMalloc(&t->ukr, sizeof(uint32_t) * 2 * M));
    SP_CUDA(cudaMalloc(&t->uent, sizeof(int32_t) * 2 * M));
    SP_CUDA(cudaMalloc(&t->umap, sizeof(uint32_t) * 2 * M));
  }
  return SP_OK;
}

static int plan_finish(sp_ctx* ctx, Plan& p, sp_table* t);

// pinned, mapped host copy of the header (+ the build sequence word after it)
static cudaError_t plan_host_alloc(Plan& p) {
  if (p.host_hdr) return cudaSuccess;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p.host_hdr), sizeof(PlanHdr) + 64,
                                cudaHostAllocMapped);
  if (e != cudaSuccess) return e;
  p.host_seq = reinterpret_cast<volatile uint32_t*>(reinterpret_cast<uint8_t*>(p.host_hdr) +
                                                    sizeof(PlanHdr));
  *p.host_seq = 0;
  if (!p.hdr_ready) e = cudaEventCreateWithFlags(&p.hdr_ready, cudaEventDisableTiming);
  return e;
}

static int plan_enqueue(sp_ctx* ctx, sp_table* t, Plan& p) {
  const int M = t->M, K = t->K;
  cudaStream_t st = ctx->stream;
  if (!p.cost) {
    SP_CUDA(cudaMalloc(&p.cost, sizeof(double) * M));
    SP_CUDA(cudaMalloc(&p.costpen, sizeof(double) * M));
  }
  const bool cluster = t->plan_ok && t->pc_ok && !ctx->opt.plan_legacy;
  if (!cluster) {
    k_cost<<<(M + 255) / 256, 256, 0, st>>>(M, t->lat, t->res, t->batch, t->pool, t->price,
                                            p.alpha, p.cost, p.costpen);
    SP_CHECK_LAUNCH(ctx);
  }
  if (!t->plan_ok) {
    p.valid = true;
    p.version = t->version;
    return SP_OK;
  }
  const int W = plan_width(t);
  if (!p.image) {
    p.image_cap = plan_image_capacity(t, W);
    SP_CUDA(cudaMalloc(&p.image, (size_t)p.image_cap));
  }
  if (cluster) {  // one cluster kernel writes cost / costpen, the whole image and the host header
    PlanHdr h;
    memset(&h, 0, sizeof(h));
    h.magic = kPlanMagic;
    h.M = M;
    h.nB = t->nB;
    h.W = W;
    h.K = K;
    for (int b = 0; b < kMaxB; ++b) h.batch_vals[b] = b < t->nB ? t->batch_vals[b] : INT32_MAX;
    SP_CUDA(plan_host_alloc(p));
    void* dh = nullptr;
    SP_CUDA(cudaHostGetDevicePointer(&dh, p.host_hdr, 0));
    ++p.seq;
    const int rc = plan_cluster_launch(ctx, t, p, W, h, t->rows_per_kind + kMaxKinds,
                                       static_cast<PlanHdr*>(dh),
                                       reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(dh) +
                                                                   sizeof(PlanHdr)),
                                       p.seq);
    if (rc != SP_OK) return rc;
    ctx->plan_dirty = true;
    p.hdr_mapped = true;
    p.hdr_pending = true;
    p.hdr_valid = false;
    p.valid = true;
    p.version = t->version;
    return SP_OK;
  }
  KindInfo ki;
  for (int k = 0; k < kMaxKinds; ++k) {
    ki.base[k] = k < K ? t->kind_base[k] : 0;
    ki.count[k] = k < K ? t->kind_count[k] : 0;
  }
  SP_CUDA(cudaMemsetAsync(t->candf, 0, sizeof(uint32_t) * M, st));
  SP_CUDA(cudaMemsetAsync(t->cands, 0, sizeof(uint32_t) * M, st));
  const int nb = (M + 255) / 256;
  const int ntiles = (M + kSortTile - 1) / kSortTile;
  const int nall = ntiles * kSortTile;
  SItem* tA = reinterpret_cast<SItem*>(t->sort_tmp);           // tiles of sort A
  SItem* tB = tA + (size_t)nall;                                // tiles of sort B
  SItem* oA = tB + (size_t)nall;                                // merged A
  SItem* oB = oA + (size_t)nall;                                // merged B
  int32_t* rkA = reinterpret_cast<int32_t*>(oB + (size_t)nall);  // ranks A / B
  int32_t* rkB = rkA + nall;
  // (cost, index) and (kind, lat, index) tile sorts + pairwise merges
  k_tile_sort<kSortR1, kSortOrder><<<2 * ntiles, kSortThreads, 0, st>>>(
      M, ntiles, p.cost, nullptr, tA, rkA, t->lat, t->kind, tB, rkB);
  SP_CHECK_LAUNCH(ctx);
  if (ntiles > 1) {
    k_merge_pairs<kSortR1, kSortOrder><<<dim3(2 * ntiles, ntiles), 256, 0, st>>>(ntiles, tA, rkA,
                                                                             tB, rkB);
    SP_CHECK_LAUNCH(ctx);
  }
  k_scatter_items<<<(2 * nall + 255) / 256, 256, 0, st>>>(M, nall, tA, rkA, oA, tB, rkB, oB);
  SP_CHECK_LAUNCH(ctx);
  k_rank_r1<<<nb, 256, 0, st>>>(M, oA, t->res, t->id_rank, t->r1, t->ent_r1);
  SP_CHECK_LAUNCH(ctx);
  // (costpen, r1): items at r1 positions
  k_tile_sort<kSortR2, kSortR2><<<ntiles, kSortThreads, 0, st>>>(
      M, ntiles, p.costpen, t->ent_r1, tA, rkA, nullptr, nullptr, nullptr, nullptr);
  SP_CHECK_LAUNCH(ctx);
  if (ntiles > 1) {
    k_merge_pairs<kSortR2, kSortR2><<<dim3(ntiles, ntiles), 256, 0, st>>>(ntiles, tA, rkA,
                                                                         nullptr, nullptr);
    SP_CHECK_LAUNCH(ctx);
  }
  k_scatter_items<<<(nall + 255) / 256, 256, 0, st>>>(M, nall, tA, rkA, oA, nullptr, nullptr,
                                                       nullptr);
  SP_CHECK_LAUNCH(ctx);
  k_orders_out<<<nb, 256, 0, st>>>(M, oA, t->ent_r1, t->ent_r2, t->r2, oB, t->order);
  SP_CHECK_LAUNCH(ctx);
  static uint64_t stair_attr = 0;
  if (attr_once(stair_attr)) {
    SP_CUDA(cudaFuncSetAttribute(k_stair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kStairMaxW * 1024 * (int)sizeof(uint32_t)));
    SP_CUDA(cudaFuncSetAttribute(k_stair_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kStairSmemBytes));
  }
  int max_mk = 0;
  for (int k = 0; k < K; ++k) max_mk = std::max(max_mk, t->kind_count[k]);
  static uint64_t lanes_attr = 0;
  if (attr_once(lanes_attr)) {
    SP_CUDA(cudaFuncSetAttribute(k_stair_lanes<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kStairLanesSmem));
    SP_CUDA(cudaFuncSetAttribute(k_stair_lanes<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kStairLanesSmem));
  }
  if (max_mk <= kStairLanesMax && !ctx->opt.stair_smem && !ctx->opt.stair_global) {
    k_stair_stage<<<(M + 255) / 256, 256, 0, st>>>(M, K, ki, t->order, t->bidx, t->lat, t->r1,
                                                   t->r2, t->pos_r12, t->pos_meta, t->pos_lat);
    SP_CHECK_LAUNCH(ctx);
    if (W <= 8)
      k_stair_lanes<4><<<K, 1024, kStairLanesSmem, st>>>(M, K, W, ki, t->order, t->bidx, t->lat,
                                                         t->r1, t->r2, t->thrscratch,
                                                         t->rowscratch, t->rows_per_kind,
                                                         t->candf, t->cands, t->pos_r12,
                                                         t->pos_meta, t->pos_lat);
    else
      k_stair_lanes<8><<<K, 1024, kStairLanesSmem, st>>>(M, K, W, ki, t->order, t->bidx, t->lat,
                                                         t->r1, t->r2, t->thrscratch,
                                                         t->rowscratch, t->rows_per_kind,
                                                         t->candf, t->cands, t->pos_r12,
                                                         t->pos_meta, t->pos_lat);
  } else if (max_mk <= kStairSmemMax && !ctx->opt.stair_global)
    k_stair_smem<<<K, 1024, kStairSmemBytes, st>>>(M, K, W, ki, t->order, t->bidx, t->lat, t->r1,
                                                   t->r2, t->thrscratch, t->rowscratch,
                                                   t->rows_per_kind, t->candf, t->cands);
  else
  k_stair<<<K, 1024, 2 * W * 1024 * sizeof(uint32_t), st>>>(M, K, W, ki, t->order, t->bidx, t->lat, t->r1, t->r2, t->pf,
                              t->sf, t->thrscratch, t->rowscratch, t->rows_per_kind, t->candf,
                              t->cands);
  SP_CHECK_LAUNCH(ctx);
  PlanHdr h;
  memset(&h, 0, sizeof(h));
  h.magic = kPlanMagic;
  h.M = M;
  h.nB = t->nB;
  h.W = W;
  h.K = K;
  for (int b = 0; b < kMaxB; ++b) h.batch_vals[b] = b < t->nB ? t->batch_vals[b] : INT32_MAX;
  int32_t* status = t->rows_per_kind + kMaxKinds;
  const int nfc = (M + kFinChunk - 1) / kFinChunk;
  int2* chunk_cnt = t->fin_chunk;
  int2* chunk_base = t->fin_chunk + nfc;
  k_fin_count<<<nfc, kFinChunk, 0, st>>>(M, t->candf, t->cands, chunk_cnt);
  SP_CHECK_LAUNCH(ctx);
  k_fin_head<<<1, 1024, 0, st>>>(M, K, t->nB, ki, t->rows_per_kind, t->thrscratch, nfc, chunk_cnt,
                                 chunk_base, h, p.image, p.image_cap, status);
  SP_CHECK_LAUNCH(ctx);
  k_fin_keys<<<nfc, kFinChunk, 0, st>>>(M, p.image, t->candf, t->cands, chunk_base, t->cidf,
                                        t->cids, t->ent_r1, t->ent_r2, t->r1, p.cost, p.costpen,
                                        t->ukey, t->ukr, t->uent);
  SP_CHECK_LAUNCH(ctx);
  k_fin_merge<<<(2 * M + 255) / 256, 256, 0, st>>>(p.image, t->ukey, t->ukr, t->umap);
  SP_CHECK_LAUNCH(ctx);
  k_fin_buckets<<<K, 1024, 0, st>>>(ki, t->thrscratch, p.image);
  SP_CHECK_LAUNCH(ctx);
  k_fin_fill<<<std::max(K, std::min(ctx->num_sms * 4, std::max(1, (2 * M + 255) / 256))), 256, 0,
               st>>>(
      K, W, ki, t->thrscratch, t->rowscratch, t->cidf, t->cids, t->ukey, t->uent, t->umap, t->lat,
      t->batch, t->kind, p.image);
  SP_CHECK_LAUNCH(ctx);
  return plan_finish(ctx, p, t);
}

static int plan_finish(sp_ctx* ctx, Plan& p, sp_table* t) {
  cudaStream_t st = ctx->stream;
  ctx->plan_dirty = true;
  p.hdr_mapped = false;
  // fetch the header back without blocking; it becomes a kernel parameter once it lands
  SP_CUDA(plan_host_alloc(p));
  SP_CUDA(cudaMemcpyAsync(p.host_hdr, p.image, sizeof(PlanHdr), cudaMemcpyDeviceToHost, st));
  // (the header-ready event is recorded by plan_build, outside any graph capture)
  p.hdr_pending = true;
  p.hdr_valid = false;
  p.valid = true;
  p.version = t->version;
  return SP_OK;
}

int plan_build(sp_ctx* ctx, sp_table* t, Plan& p) {
  // the cluster builder is one kernel: launched directly (programmatic dependent launch on
  // both sides), no graph and no header event
  if (t->plan_ok && t->pc_ok && !ctx->opt.plan_legacy) return plan_enqueue(ctx, t, p);
  if (p.graph && !ctx->opt.no_plan_graph) {
    SP_CUDA(cudaGraphLaunch(p.graph, ctx->stream));
    if (t->plan_ok) SP_CUDA(cudaEventRecord(p.hdr_ready, ctx->stream));
    ctx->launches += p.graph_kernels;
    ctx->plan_dirty = true;
    p.hdr_pending = t->plan_ok;
    p.hdr_valid = false;
    p.valid = true;
    p.version = t->version;
    return SP_OK;
  }
  if (p.builds == 0 || ctx->opt.no_plan_graph) {  // first build: allocations happen here
    ++p.builds;
    const int rc = plan_enqueue(ctx, t, p);
    if (rc == SP_OK && t->plan_ok) SP_CUDA(cudaEventRecord(p.hdr_ready, ctx->stream));
    return rc;
  }
  // second build: capture the whole build once on a private stream, then replay it
  if (!ctx->capture) SP_CUDA(cudaStreamCreateWithFlags(&ctx->capture, cudaStreamNonBlocking));
  cudaStream_t user = ctx->stream;
  const int64_t l0 = ctx->launches;
  ctx->stream = ctx->capture;
  cudaError_t e = cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal);
  int rc = e == cudaSuccess ? plan_enqueue(ctx, t, p) : cuda_fail(e, "cudaStreamBeginCapture");
  cudaGraph_t g = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(ctx->capture, &g);
  ctx->stream = user;
  const int64_t nk = ctx->launches - l0;
  ctx->launches = l0;
  if (rc != SP_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&p.graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    p.graph = nullptr;
    return cuda_fail(e, "cudaGraphInstantiate(plan)");
  }
  p.graph_kernels = nk;
  ++p.builds;
  return plan_build(ctx, t, p);  // replay
}

const PlanHdr* plan_host_header(Plan& p) {
  if (p.hdr_pending) {
    if (p.hdr_mapped) {
      if (*p.host_seq == p.seq) {  // written by the build kernel after the header (system fence)
        p.hdr_pending = false;
        p.hdr_valid = reinterpret_cast<volatile PlanHdr*>(p.host_hdr)->magic == kPlanMagic;
      }
    } else if (cudaEventQuery(p.hdr_ready) == cudaSuccess) {
      p.hdr_pending = false;
      p.hdr_valid = p.host_hdr->magic == kPlanMagic;
    }
  }
  return p.hdr_valid ? p.host_hdr : nullptr;
}

int plan_header_wait(sp_ctx* ctx, Plan& p) {
  if (p.hdr_pending) {
    if (p.hdr_mapped) SP_CUDA(cudaStreamSynchronize(ctx->stream));
    else SP_CUDA(cudaEventSynchronize(p.hdr_ready));
  }
  return SP_OK;
}

void plan_release(Plan& p) {
  if (p.graph) cudaGraphExecDestroy(p.graph);
  cudaFree(p.cost);
  cudaFree(p.costpen);
  cudaFree(p.image);
  if (p.host_hdr) cudaFreeHost(p.host_hdr);
  if (p.hdr_ready) cudaEventDestroy(p.hdr_ready);
  p = Plan();
}

// the table's plan slot for alpha (created empty when missing; at most 16 per table)
static Plan* plan_entry(sp_ctx* ctx, sp_table* t, double alpha) {
  for (auto& p : t->plans)
    if (p.alpha == alpha || (p.alpha != p.alpha && alpha != alpha)) return &p;
  if (t->plans.size() >= 16) {
    // evict the oldest entry's buffers (keep memory bounded)
    cudaStreamSynchronize(ctx->stream);
    plan_release(t->plans.front());
    t->plans.erase(t->plans.begin());
  }
  t->plans.emplace_back();
  Plan* hit = &t->plans.back();
  hit->alpha = alpha;
  return hit;
}

Plan* plan_get(sp_ctx* ctx, sp_table* t, double alpha, int* rc) {
  *rc = SP_OK;
  Plan* hit = plan_entry(ctx, t, alpha);
  if (!hit->valid || hit->version != t->version) {
    *rc = plan_build(ctx, t, *hit);
    if (*rc != SP_OK) return nullptr;
    hit->cost_version = t->version;
  }
  return hit;
}

// Every listed alpha's plan current for the table version; stale staircase plans of the
// cluster builder are rebuilt together, up to four per launch (one cluster each).
int plan_prepare_many(sp_ctx* ctx, sp_table* t, int n, const double* alphas) {
  const bool cluster = t->plan_ok && t->pc_ok && !ctx->opt.plan_legacy && t->finite_safe();
  std::vector<Plan*> todo;
  for (int i = 0; i < n; ++i) {
    const double al = alphas[i];
    int rc = SP_OK;
    if (!cluster || !isfinite(al)) {
      Plan* p = t->plan_ok && t->finite_safe() && isfinite(al) ? plan_get(ctx, t, al, &rc)
                                                               : plan_costs(ctx, t, al, &rc);
      if (!p) return rc;
      continue;
    }
    plan_entry(ctx, t, al);  // creates the slot (may grow t->plans)
  }
  if (cluster) {  // pointers into t->plans only once it no longer grows
    for (int i = 0; i < n; ++i) {
      if (!isfinite(alphas[i])) continue;
      Plan* p = plan_entry(ctx, t, alphas[i]);
      if (p->valid && p->version == t->version) continue;
      bool dup = false;
      for (Plan* q : todo) dup |= q == p;
      if (!dup) todo.push_back(p);
    }
  }
  if (todo.size() == 1) {
    int rc = SP_OK;
    return plan_get(ctx, t, todo[0]->alpha, &rc) ? SP_OK : rc;
  }
  if (todo.empty()) return SP_OK;
  const int M = t->M, K = t->K, W = plan_width(t);
  if (!t->pc_multi_status) SP_CUDA(cudaMalloc(&t->pc_multi_status, sizeof(int32_t) * 8));
  if (!t->pc_multi_ord) SP_CUDA(cudaMalloc(&t->pc_multi_ord, sizeof(int32_t) * M));
  PlanHdr h;
  memset(&h, 0, sizeof(h));
  h.magic = kPlanMagic;
  h.M = M;
  h.nB = t->nB;
  h.W = W;
  h.K = K;
  for (int b = 0; b < kMaxB; ++b) h.batch_vals[b] = b < t->nB ? t->batch_vals[b] : INT32_MAX;
  for (size_t c0 = 0; c0 < todo.size(); c0 += 4) {
    const int nq = (int)std::min<size_t>(4, todo.size() - c0);
    void* scratch[4];
    double* thr[4];
    for (int q = 0; q < nq; ++q) {
      Plan& p = *todo[c0 + q];
      if (!p.cost) {
        SP_CUDA(cudaMalloc(&p.cost, sizeof(double) * M));
        SP_CUDA(cudaMalloc(&p.costpen, sizeof(double) * M));
      }
      if (!p.image) {
        p.image_cap = plan_image_capacity(t, W);
        SP_CUDA(cudaMalloc(&p.image, (size_t)p.image_cap));
      }
      SP_CUDA(plan_host_alloc(p));
      if (q == 0) {
        scratch[q] = t->pc_scratch;
        thr[q] = t->thrscratch;
      } else {
        if (!t->pc_multi_scratch[q - 1]) {
          SP_CUDA(cudaMalloc(&t->pc_multi_scratch[q - 1], t->pc_scratch_bytes));
          SP_CUDA(cudaMalloc(&t->pc_multi_thr[q - 1], sizeof(double) * (M + K)));
        }
        scratch[q] = t->pc_multi_scratch[q - 1];
        thr[q] = t->pc_multi_thr[q - 1];
      }
    }
    const int rc = plan_cluster_launch_multi(ctx, t, todo.data() + c0, nq, W, h, t->pc_multi_status,
                                             scratch, thr, t->pc_multi_ord);
    if (rc != SP_OK) return rc;
    for (int q = 0; q < nq; ++q) {
      Plan& p = *todo[c0 + q];
      p.hdr_mapped = true;
      p.hdr_pending = true;
      p.hdr_valid = false;
      p.valid = true;
      p.version = t->version;
      p.cost_version = t->version;
    }
    ctx->plan_dirty = true;
  }
  return SP_OK;
}

bool plan_ready(sp_table* t, double alpha) {
  for (auto& p : t->plans)
    if (p.alpha == alpha || (p.alpha != p.alpha && alpha != alpha))
      return p.valid && p.version == t->version;
  return false;
}

// cost / costpen of the current table version only (the scan kernels' inputs): one k_cost
// launch when stale, no staircase build
Plan* plan_costs(sp_ctx* ctx, sp_table* t, double alpha, int* rc) {
  *rc = SP_OK;
  Plan* p = plan_entry(ctx, t, alpha);
  if (p->cost_version == t->version && p->cost) return p;
  const int M = t->M;
  if (!p->cost) {
    cudaError_t e = cudaMalloc(&p->cost, sizeof(double) * M);
    if (e == cudaSuccess) e = cudaMalloc(&p->costpen, sizeof(double) * M);
    if (e != cudaSuccess) {
      *rc = cuda_fail(e, "cudaMalloc(cost)");
      return nullptr;
    }
  }
  k_cost<<<(M + 255) / 256, 256, 0, ctx->stream>>>(M, t->lat, t->res, t->batch, t->pool, t->price,
                                                    p->alpha, p->cost, p->costpen);
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *rc = cuda_fail(e, "k_cost");
    return nullptr;
  }
  p->cost_version = t->version;
  return p;
}

}  // namespace sp
