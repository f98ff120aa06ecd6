// sp_fold.cu — K3: profile feedback fold (manager.py:436-457, 45-47; configurator.py:463-491).
//
// Reference, per completed invocation in completion order:
//     if eidx == ref_index: completed_ref += 1                         (manager.py:440-441)
//     observations[(op, config_id)] += 1                               (442)
//     if fb frozen: stop                                               (443-444)
//     lat[eidx] = beta*obs + (1-beta)*lat[eidx]                         (445-447, 45-47)
//     if eidx == ref_index and completed_ref == dfp_count and dfp on:  (449-457)
//         ratio = lat[ref] / lat_init[ref]
//         every entry never observed so far (except the reference):
//             lat[i] = lat_init[i] * ratio                             (configurator.py:486-490)
//
// Device restatement (bit-exact): the EWMA recurrence is order-dependent, so it is NOT
// tree-reduced; instead the observation batch is stably sorted by (table, entry) with a CUB
// radix sort (positions ascending inside each key = completion order), and each entry's
// segment is folded in completion order.  The gate lift is located inside the reference
// entry's own segment (the k-th reference observation, k = dfp_count - completed_ref_before);
// an entry is rescaled iff it had no observation before the batch and its first observation
// in the batch comes after the gate position — exactly the set recalibrate_unobserved sees.
//
// Long segments (a hot configuration can receive most of a batch) use a coalescing window
// instead of a sequential chain tens of thousands of steps long.  One step
// x -> fl(fl(beta*o) + fl((1-beta)*x)) is monotone non-decreasing in x (beta in (0, 1]), so the
// fold of a window is a monotone function of the window's input.  Every chain value lies in
// [lo, hi] (the range of the start value and the segment's observations, widened by a
// rounding margin, see fold_bounds); if the chains started at lo and at hi over the last W
// observations end on the same bits, every input in [lo, hi] — the true one included — gives
// exactly that value.  Otherwise the segment is folded sequentially.  W is sized so that a
// gap of 2^80 ulps decays below one ulp (80 / -log2(1 - beta) steps).
#include <algorithm>
#include <math.h>
#include <stdlib.h>

#include <cub/cub.cuh>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kMaxFoldTables = 64;

struct FoldTab {
  double* lat;
  const double* lat_init;
  int32_t* obs_count;
  int32_t* counters;  // [0] completed_ref
  uint8_t* dirty;     // latency written (the plan builder's cached order, sp_plan_cluster.cu)
  int32_t M;
  int32_t ref_index;
  int32_t gbase;  // global key base
  int32_t pad;
};
struct FoldTabs {
  FoldTab t[kMaxFoldTables];
  int n;
  int total;  // entries over all tables; the sort key of a skipped observation (idx < 0)
};
// per-table gate state produced by k_fold_ref, consumed by the other two kernels
struct Gate {
  int32_t lifted;   // gate lifts inside this batch
  int32_t gate_pos; // stream position of the lifting reference observation
  double ratio;
};

// Sort keys, and per table the number of keys below and equal to its reference entry's key
// (refcnt[2t], refcnt[2t+1]; zeroed by the caller) — the reference segment's bounds in the
// sorted order, so k_fold_ref needs no search.
__global__ void k_fold_keys(int n, FoldTabs ft, const int32_t* __restrict__ op,
                            const int32_t* __restrict__ idx, uint32_t* keys, uint32_t* pos,
                            int* refcnt) {
  __shared__ int s_c[2 * kMaxFoldTables];
  for (int i = threadIdx.x; i < 2 * ft.n; i += blockDim.x) s_c[i] = 0;
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    const int t = op ? op[j] : 0;
    const uint32_t key = idx[j] < 0 ? (uint32_t)ft.total : (uint32_t)(ft.t[t].gbase + idx[j]);
    keys[j] = key;
    pos[j] = (uint32_t)j;
    for (int u = 0; u < ft.n; ++u) {
      if (ft.t[u].ref_index < 0) continue;
      const uint32_t rk = (uint32_t)(ft.t[u].gbase + ft.t[u].ref_index);
      if (key < rk) atomicAdd(&s_c[2 * u], 1);
      else if (key == rk) atomicAdd(&s_c[2 * u + 1], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * ft.n; i += blockDim.x)
    if (s_c[i]) atomicAdd(&refcnt[i], s_c[i]);
}

__device__ __forceinline__ double ewma(double beta, double obs, double old) {
  // manager.py:47  beta * observed_s + (1.0 - beta) * old_estimate_s
  return __dadd_rn(__dmul_rn(beta, obs), __dmul_rn(__dsub_rn(1.0, beta), old));
}

__device__ int lower_bound_u32(const uint32_t* a, int n, uint32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Observations in sorted (entry, completion) order: a parallel gather, so the sequential
// recurrence below streams contiguous memory instead of chasing spos[] per step.
__global__ void k_fold_gather(int n, const uint32_t* __restrict__ spos,
                              const double* __restrict__ obs, double* __restrict__ sobs) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) sobs[q] = obs[spos[q]];
}

// Sequential EWMA over sobs[q, end): loads are issued eight ahead of the dependent chain.
__device__ __forceinline__ double fold_run(double L, const double* __restrict__ sobs, int q, int end,
                                           double beta) {
  const double ob = beta, ol = __dsub_rn(1.0, beta);
  int u = q;
  for (; u + 8 <= end; u += 8) {
    double o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __ldg(sobs + u + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) L = __dadd_rn(__dmul_rn(ob, o[j]), __dmul_rn(ol, L));
  }
  for (; u < end; ++u) L = __dadd_rn(__dmul_rn(ob, __ldg(sobs + u)), __dmul_rn(ol, L));
  return L;
}

// The chains from lo and from hi over sobs[w0, end), interleaved (two independent chains).
__device__ __forceinline__ bool fold_window(const double* __restrict__ sobs, int w0, int end,
                                            double beta, double lo, double hi, double* out) {
  const double ob = beta, ol = __dsub_rn(1.0, beta);
  double a = lo, b = hi;
  int u = w0;
  for (; u + 4 <= end; u += 4) {
    double o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = __ldg(sobs + u + j);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double t = __dmul_rn(ob, o[j]);
      a = __dadd_rn(t, __dmul_rn(ol, a));
      b = __dadd_rn(t, __dmul_rn(ol, b));
    }
  }
  for (; u < end; ++u) {
    const double t = __dmul_rn(ob, __ldg(sobs + u));
    a = __dadd_rn(t, __dmul_rn(ol, a));
    b = __dadd_rn(t, __dmul_rn(ol, b));
  }
  *out = a;
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// Exact fold of sobs[q, end) from L; bounds (lo, hi) must hold every chain value.
__device__ __forceinline__ double fold_exact(double L, const double* __restrict__ sobs, int q,
                                             int end, double beta, int win, bool bounded,
                                             double lo, double hi) {
  if (bounded && end - q > win) {
    double v;
    if (fold_window(sobs, end - win, end, beta, lo, hi, &v)) return v;
  }
  return fold_run(L, sobs, q, end, beta);
}

// Block-wide bounds of every chain value of a fold of sobs[q, end) started at L.  With
// ob = beta, ol = fl(1 - beta) >= 0, ob + ol <= 1 + u, a step from values in [m, M] stays in
// [m (1 - u)^4, M (1 + u)^4] (u = 2^-53) up to subnormal absolute error; over fewer than 2^31
// steps the relative drift is below 2^-20, so [m - |m| 2^-20 - 2^-1000, M + |M| 2^-20 +
// 2^-1000] holds the whole chain.  Non-finite values disable the window.  Result in
// bnd[0..1], finite flag in *ok (valid after the trailing barrier).
__device__ void fold_bounds(const double* __restrict__ sobs, int q, int end, double L,
                            double* bnd, int* ok) {
  __shared__ double smin[32], smax[32];
  __shared__ int sbad[32];
  double m = L, M = L;
  int bad = isfinite(L) ? 0 : 1;
  // eight independent loads in flight per thread (the segment is read once, latency-bound)
  const int step = blockDim.x;
  int u = q + threadIdx.x;
  for (; u + 7 * step < end; u += 8 * step) {
    double o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = __ldg(sobs + u + k * step);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      bad |= isfinite(o[k]) ? 0 : 1;
      m = o[k] < m ? o[k] : m;
      M = o[k] > M ? o[k] : M;
    }
  }
  for (; u < end; u += step) {
    const double o = __ldg(sobs + u);
    bad |= isfinite(o) ? 0 : 1;
    m = o < m ? o : m;
    M = o > M ? o : M;
  }
  for (int d = 16; d; d >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, m, d), oM = __shfl_xor_sync(0xffffffffu, M, d);
    m = om < m ? om : m;
    M = oM > M ? oM : M;
    bad |= __shfl_xor_sync(0xffffffffu, bad, d);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smin[w] = m;
    smax[w] = M;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < nw; ++j) {
      m = smin[j] < m ? smin[j] : m;
      M = smax[j] > M ? smax[j] : M;
      bad |= sbad[j];
    }
    bnd[0] = m - fabs(m) * 0x1p-20 - 0x1p-1000;
    bnd[1] = M + fabs(M) * 0x1p-20 + 0x1p-1000;
    *ok = !bad;
  }
  __syncthreads();
}

// One block per table: fold the reference entry's segment, locate the gate lift.  Block 0
// also resets the long-segment queue filled by k_fold_seg.
__global__ void k_fold_ref(int n, FoldTabs ft, const uint32_t* __restrict__ skeys,
                           const uint32_t* __restrict__ spos, const double* __restrict__ sobs,
                           double beta, int win, int dfp_count, int dfp_on, int fb_frozen,
                           Gate* gates, int* long_count, const int* __restrict__ refcnt) {
  __shared__ double bnd[2];
  __shared__ int bnd_ok;
  const int t = blockIdx.x;
  if (t == 0 && threadIdx.x == 0) *long_count = 0;
  FoldTab tb = ft.t[t];
  if (tb.ref_index < 0) {
    if (threadIdx.x == 0) gates[t] = Gate{0, -1, 1.0};
    return;
  }
  // the reference entry's segment of the sorted keys: [#keys below it, + #keys equal)
  const int q = refcnt[2 * t], cnt = refcnt[2 * t + 1], end = q + cnt;
  const double L0 = tb.lat[tb.ref_index];
  const bool bounded = !fb_frozen && cnt > win;
  if (bounded) fold_bounds(sobs, q, end, L0, bnd, &bnd_ok);
  if (threadIdx.x != 0) return;
  Gate g{0, -1, 1.0};
  const int before = tb.counters[0];
  if (cnt) {
    if (!fb_frozen) {
      const bool bd = bounded && bnd_ok;
      const double lo = bounded ? bnd[0] : 0.0, hi = bounded ? bnd[1] : 0.0;
      double L = L0;
      // the k-th reference completion of this batch makes completed_ref == dfp_count
      const int k = dfp_count - before;  // 1-based position inside the segment
      if (dfp_on && k >= 1 && k <= cnt && tb.lat_init[tb.ref_index] > 0.0) {
        L = fold_exact(L, sobs, q, q + k, beta, win, bd, lo, hi);
        g.lifted = 1;
        g.gate_pos = (int)spos[q + k - 1];
        g.ratio = __ddiv_rn(L, tb.lat_init[tb.ref_index]);  // configurator.py:486
        L = fold_exact(L, sobs, q + k, end, beta, win, bd, lo, hi);
      } else {
        L = fold_exact(L, sobs, q, end, beta, win, bd, lo, hi);
      }
      tb.lat[tb.ref_index] = L;
    }
    tb.counters[0] = before + cnt;
    tb.obs_count[tb.ref_index] += cnt;
  }
  gates[t] = g;
}

__device__ __forceinline__ int table_of_key(const FoldTabs& ft, uint32_t key) {
  int t = 0;
  for (int u = 1; u < ft.n; ++u)
    if ((int)key >= ft.t[u].gbase) t = u;
  return t;
}

struct LongSeg {
  int32_t q, end;
  double* dst;
  double L0;
  int64_t pad;
};

// One thread per segment head (non-reference entries); segments longer than long_min are
// queued for k_fold_long.
__global__ void k_fold_seg(int n, FoldTabs ft, const uint32_t* __restrict__ skeys,
                           const uint32_t* __restrict__ spos, const double* __restrict__ sobs,
                           double beta, int fb_frozen, const Gate* __restrict__ gates,
                           int long_min, LongSeg* long_q, int* long_count) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t key = skeys[q];
  if (q > 0 && skeys[q - 1] == key) return;
  if ((int)key >= ft.total) return;  // skipped observations (idx < 0) sort last
  const int t = table_of_key(ft, key);
  const FoldTab& tb = ft.t[t];
  const int e = (int)key - tb.gbase;
  if (e == tb.ref_index) return;  // folded by k_fold_ref
  // a segment longer than long_min is known from one probe; only those search for their end
  const bool is_long = q + long_min < n && skeys[q + long_min] == key;
  int end;
  if (is_long) {
    end = lower_bound_u32(skeys, n, key + 1);
  } else {  // the end lies within the next long_min positions: a short search there
    const int lim = min(n, q + long_min + 1);
    end = q + 1 + lower_bound_u32(skeys + q + 1, lim - q - 1, key + 1);
  }
  const int cnt = end - q;
  const int before = tb.obs_count[e];
  if (!fb_frozen) {
    const Gate g = gates[t];
    double L = tb.lat[e];
    // never observed before the batch and first observed after the gate lift: it was
    // rescaled by recalibrate_unobserved before its first fold
    if (g.lifted && before == 0 && (int)spos[q] > g.gate_pos)
      L = __dmul_rn(tb.lat_init[e], g.ratio);
    if (is_long) {
      const int j = atomicAdd(long_count, 1);
      long_q[j] = LongSeg{q, end, tb.lat + e, L, 0};
    } else {
      tb.lat[e] = fold_run(L, sobs, q, end, beta);
    }
  }
  tb.obs_count[e] = before + cnt;
}

// One block per queued long segment: bounds, then the coalescing window (or the chain).
__global__ void k_fold_long(const double* __restrict__ sobs, double beta, int win,
                            const LongSeg* __restrict__ long_q, const int* __restrict__ long_count) {
  __shared__ double bnd[2];
  __shared__ int bnd_ok;
  const int nl = *long_count;
  for (int j = blockIdx.x; j < nl; j += gridDim.x) {
    const LongSeg sg = long_q[j];
    fold_bounds(sobs, sg.q, sg.end, sg.L0, bnd, &bnd_ok);
    if (threadIdx.x == 0)
      *sg.dst = fold_exact(sg.L0, sobs, sg.q, sg.end, beta, win, bnd_ok, bnd[0], bnd[1]);
    __syncthreads();
  }
}

// Entries of gated tables that were never observed at all: plain rescale.
__global__ void k_fold_rescale(FoldTabs ft, const Gate* __restrict__ gates) {
  const int t = blockIdx.y;
  const FoldTab tb = ft.t[t];
  const Gate g = gates[t];
  if (!g.lifted) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tb.M; e += gridDim.x * blockDim.x) {
    if (e == tb.ref_index || tb.obs_count[e] != 0) continue;
    tb.lat[e] = __dmul_rn(tb.lat_init[e], g.ratio);  // configurator.py:490
  }
}

}  // namespace

static int fold_launch_legacy(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n,
                              const int32_t* op, const int32_t* idx, const double* obs,
                              double beta, int dfp_count, int dfp_on, int fb_frozen) {
  if (n_tables > kMaxFoldTables) return fail(SP_E_UNSUPPORTED, "fold: at most 64 tables");
  FoldTabs ft;
  ft.n = n_tables;
  int64_t gb = 0;
  int maxM = 0;
  for (int t = 0; t < n_tables; ++t) {
    sp_table* tb = tables[t];
    FoldTab f;
    f.lat = tb->lat;
    f.lat_init = tb->lat_init;
    f.obs_count = tb->obs_count;
    f.counters = tb->dev_counters;
    f.dirty = tb->dirty;
    f.M = tb->M;
    f.ref_index = tb->ref_index;
    f.gbase = (int32_t)gb;
    f.pad = 0;
    ft.t[t] = f;
    gb += tb->M;
    if (tb->M > maxM) maxM = tb->M;
  }
  if (gb >= (1ll << 31) - 1) return fail(SP_E_UNSUPPORTED, "fold: too many entries");
  ft.total = (int)gb;
  int end_bit = 1;
  while ((1ll << end_bit) <= gb) ++end_bit;
  cudaStream_t st = ctx->stream;
  // scratch: keys, pos, sorted keys, sorted pos, gates, cub temp
  size_t cub_bytes = 0;
  if (n > 0)
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, n, 0, end_bit, st);
  // coalescing window: ol^win * 2^80 < 1 ulp  (ol = 1 - beta); disabled when it would be long
  const double ol = 1.0 - beta;
  int win = 8;
  if (ol > 0.0) {
    const double w = ceil(80.0 / -log2(ol));
    win = w > 4096.0 ? (1 << 30) : (w < 8.0 ? 8 : (int)w);
  }
  // segments longer than two windows take the block-parallel window path (measured on config 5:
  // 2 * win = 160 beats 512 — a 512-step sequential chain in one thread is the longer pole)
  int long_min = win >= (1 << 30) ? (1 << 30) : std::max(2 * win, 128);
  if (ctx->opt.fold_long_min > 0) long_min = std::max(2 * win, ctx->opt.fold_long_min);
  const int long_cap = n / (long_min + 1) + 1;
  size_t a = ((size_t)n * 4 + 255) & ~(size_t)255;
  size_t gates_bytes = ((size_t)n_tables * sizeof(Gate) + 255) & ~(size_t)255;
  size_t long_bytes = ((size_t)long_cap * sizeof(LongSeg) + 256 + 255) & ~(size_t)255;
  size_t total = 4 * a + gates_bytes + long_bytes + cub_bytes + 256 +
                 (((size_t)n * 8 + 255) & ~(size_t)255) + 256 * 2;
  int rc = SP_OK;
  uint8_t* base = (uint8_t*)ctx_tmp(ctx, total, &rc);
  if (!base) return rc;
  uint32_t* keys = (uint32_t*)base;
  uint32_t* pos = (uint32_t*)(base + a);
  uint32_t* skeys = (uint32_t*)(base + 2 * a);
  uint32_t* spos = (uint32_t*)(base + 3 * a);
  Gate* gates = (Gate*)(base + 4 * a);
  int* long_count = (int*)(base + 4 * a + gates_bytes);
  LongSeg* long_q = (LongSeg*)(base + 4 * a + gates_bytes + 256);
  void* cub_tmp = base + 4 * a + gates_bytes + long_bytes;
  double* sobs = (double*)(base + 4 * a + gates_bytes + long_bytes +
                           ((cub_bytes + 255) & ~(size_t)255));
  int* refcnt = (int*)((uint8_t*)sobs + (((size_t)n * 8 + 255) & ~(size_t)255));
  SP_CUDA(cudaMemsetAsync(refcnt, 0, sizeof(int) * 2 * kMaxFoldTables, st));
  if (n > 0) {
    k_fold_keys<<<(n + 255) / 256, 256, 0, st>>>(n, ft, op, idx, keys, pos, refcnt);
    SP_CHECK_LAUNCH(ctx);
    SP_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, skeys, pos, spos, n, 0,
                                            end_bit, st));
    ctx->launches += 2;  // upsweep/downsweep passes (at least)
    k_fold_gather<<<(n + 255) / 256, 256, 0, st>>>(n, spos, obs, sobs);
    SP_CHECK_LAUNCH(ctx);
  }
  k_fold_ref<<<n_tables, 256, 0, st>>>(n, ft, skeys, spos, sobs, beta, win, dfp_count, dfp_on,
                                       fb_frozen, gates, long_count, refcnt);
  SP_CHECK_LAUNCH(ctx);
  if (n > 0) {
    k_fold_seg<<<(n + 255) / 256, 256, 0, st>>>(n, ft, skeys, spos, sobs, beta, fb_frozen,
                                                gates, long_min, long_q, long_count);
    SP_CHECK_LAUNCH(ctx);
    if (!fb_frozen && long_min < n) {
      k_fold_long<<<std::min(long_cap, 2 * ctx->num_sms), 256, 0, st>>>(sobs, beta, win, long_q,
                                                                        long_count);
      SP_CHECK_LAUNCH(ctx);
    }
  }
  if (!fb_frozen && dfp_on) {
    dim3 grid((maxM + 255) / 256, n_tables);
    k_fold_rescale<<<grid, 256, 0, st>>>(ft, gates);
    SP_CHECK_LAUNCH(ctx);
  }
  for (int t = 0; t < n_tables; ++t) {
    tables[t]->version++;
    // this path does not track written entries: the builder's cached order is re-sorted whole
    SP_CUDA(cudaMemsetAsync(tables[t]->dev_counters + 4, 1, 1, st));
  }
  return SP_OK;
}


// ---- one-kernel fold (default) ----------------------------------------------------------------
//
// The multi-kernel path above sorts the whole batch with a device-wide radix sort (several
// passes sized for millions of keys) and then folds in five more launches.  A config-5 batch is
// 65,536 records over a few hundred distinct entries, so the fold is latency-bound, not
// bandwidth-bound.  k_fold_coop does the whole batch in ONE cooperative launch (every CTA
// resident, grid barriers between phases), per chunk of up to 64 tiles x 1024 records:
//
//   phase A (CTA per tile): a block radix sort of the tile's keys (stable: positions ascend
//     inside a key), the sorted observations written out; every run (one entry's records inside
//     the tile) publishes (start, length) in the entry's per-tile slot, sets the tile's bit in
//     the entry's 64-bit tile mask (the first setter appends the entry to the touched list),
//     and folds its min / max into the entry's bounds (warp-segmented scan, one atomic pair per
//     run and warp); reference runs add to the table's reference count.
//   grid barrier (one returning atomic per CTA); every warp evaluates, per table, whether the
//     gate lifts in this chunk (k = dfp_count - completed_ref_before in [1, reference count]),
//     and issues its first entry's loads in the same round trip.
//   phase B (only when a gate lifts): one warp per lifting table folds the reference entry up to
//     its k-th observation (ratio = lat / lat_init, configurator.py:486) and on; grid barrier.
//   phase C (warp per touched entry): the entry's runs in tile order from the mask and slots;
//     the rescale rule of the multi-kernel path (never observed before the batch, first
//     observation after the gate); the EWMA fold in completion order — the coalescing window
//     over the last `win` observations when the bounds allow it, else sequentially — staged
//     through a per-warp shared-memory buffer; counts; the entry's mask / bounds reset.
//   grid barrier; phase D: completed_ref, the per-chunk counters reset, and (when a gate lifted)
//     the rescale of every entry still unobserved (configurator.py:486-490).  In the last chunk
//     with no gate lift there is no barrier: the last CTA to finish phase C does phase D.
// Touched entries are dealt CTA-major so the hottest (first-touched, longest chains) run on
// different SMs; observations are gathered by cp.async, beta * o precomputed by the lanes.
//
// Splitting a batch into consecutive chunks folds exactly as one batch does (the multi-kernel
// path's chunked tests rely on the same property).
namespace {

constexpr int kCoopThreads = 1024;
constexpr int kCoopTile = kCoopThreads;        // records per tile (one per thread)
constexpr int kCoopTiles = 64;                 // tiles per chunk (one mask bit each)
constexpr int kCoopChunk = kCoopTile * kCoopTiles;
constexpr int kCoopWarpBuf = 256;              // observations staged per warp
constexpr int kCoopWarps = kCoopThreads / 32;

struct CoopState {  // persistent per context; zero (lo: ~0) outside a launch
  uint32_t bar[2];      // grid barrier: arrival word (top bit flips per barrier); CTAs done
  int32_t touched_n[2];  // per chunk parity
  int32_t refcnt[2][kMaxFoldTables];
};

struct CoopArgs {
  FoldTabs ft;
  int n;
  const int32_t* op;
  const int32_t* idx;
  const double* obs;
  double beta;
  int win;
  int dfp_count, dfp_on, fb_frozen;
  int end_bit;
  uint32_t* skey;   // chunk: per tile sorted keys
  uint32_t* spos;   // chunk: global stream positions in sorted order
  double* sobs;     // chunk: observations in sorted order
  uint64_t* mask;   // per key: tiles of the chunk holding the key
  uint64_t* lo;     // per key: order-key minimum of the chunk's observations
  uint64_t* hi;     // per key: order-key maximum
  uint32_t* slot;   // per key x kCoopTiles: run start | length << 16
  int32_t* touched; // chunk: keys with at least one observation
  Gate* gates;      // per table
  CoopState* st;
  int debug;        // SP_PC_DEBUG: per-phase timestamps of CTA 0 (printf)
  // simulated backend fused into the load (sp_simulate_and_fold): record j is decision j —
  // an assignment runs and yields (base[idx] + per_item[idx] * fill) * noise (backend.py:52-54),
  // anything else yields no observation; the records are also written to rec_idx / rec_obs
  const int32_t *d_code, *d_idx, *d_fill;
  const double *t_base, *t_per_item, *t_noise;
  int32_t* rec_idx;
  double* rec_obs;
};

__device__ __forceinline__ int coop_entry(const CoopArgs& a, int j) {
  if (!a.d_code) return a.idx[j];
  return (a.d_code[j] & 3) == SP_DEC_ASSIGN ? a.d_idx[j] : -1;
}
__device__ __forceinline__ double coop_obs(const CoopArgs& a, int j) {
  if (!a.d_code) return a.obs[j];
  const int e = a.d_idx[j];  // only called for records that run
  double lat = a.t_base[e];
  if (a.t_per_item) lat = __dadd_rn(lat, __dmul_rn(a.t_per_item[e], (double)a.d_fill[j]));
  return __dmul_rn(lat, a.t_noise[j]);
}

__device__ __forceinline__ unsigned coop_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t coop_timer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


// Stable grouping of one 1024-record tile by key (one record per thread): the records of a key
// become one contiguous run, in thread order inside the run; runs are laid out in the order the
// keys were first inserted (the fold only needs each key's records together and in order).
//   1. keys go into a shared-memory hash table (linear probing, 2048 slots); the inserting
//      thread gives the key a dense id;
//   2. per warp, __match_any_sync groups equal keys: rank inside the warp, and the group's count
//      in cnt[id][warp] (bytes);
//   3. per id the run length (sum over warps) and, by a block scan, the run start;
//   4. every record scatters to run start + records of its key in earlier warps + rank.
// On return thread i holds the record at position i and `len` = its run's length when it is the
// run's first record (0 otherwise).  Shared memory: kTileGroupSmem bytes at `sm` (16-B aligned).
constexpr int kTileHash = 2048;
constexpr int kTileGroupSmem = kCoopTile * 32 + kTileHash * 4 + kTileHash * 2 + kCoopTile * 4 * 4 +
                               kCoopTile * 8;
// `pay` (the record's observation) travels with the record.
__device__ __forceinline__ void tile_group(uint32_t& key, uint32_t& val, uint32_t& len, double& pay,
                                           uint8_t* sm) {
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm);                 // [1024 ids][32 warps] bytes
  uint32_t* htab = cnt + kCoopTile * 8;                            // kTileHash keys
  uint16_t* hid = reinterpret_cast<uint16_t*>(htab + kTileHash);   // kTileHash ids
  uint32_t* start = reinterpret_cast<uint32_t*>(hid + kTileHash);  // per id: run start
  uint32_t* sk = start + kCoopTile;
  uint32_t* sv = sk + kCoopTile;
  uint32_t* sl = sv + kCoopTile;
  double* so = reinterpret_cast<double*>(sl + kCoopTile);  // 16-B aligned: offsets are multiples of 4 KB
  __shared__ uint32_t s_n, s_ws[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
  for (int u = 0; u < 8; ++u) cnt[t + u * kCoopTile] = 0;
  htab[t] = 0xFFFFFFFFu;
  htab[t + kCoopTile] = 0xFFFFFFFFu;
  if (t == 0) s_n = 0;
  __syncthreads();
  uint32_t h = (key * 2654435761u) >> 21;  // 11 bits
  for (;;) {
    const uint32_t old = atomicCAS(&htab[h], 0xFFFFFFFFu, key);
    if (old == 0xFFFFFFFFu) {
      hid[h] = (uint16_t)atomicAdd(&s_n, 1u);
      break;
    }
    if (old == key) break;
    h = (h + 1) & (kTileHash - 1);
  }
  __syncthreads();
  const uint32_t id = hid[h];
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
  uint8_t* cb = reinterpret_cast<uint8_t*>(cnt);
  if (rank == 0) cb[id * 32 + w] = (uint8_t)__popc(peers);
  __syncthreads();
  // run lengths, exclusive scan over ids (ids < s_n)
  const uint32_t nid = s_n;
  uint32_t tot = 0;
  if ((uint32_t)t < nid) {
#pragma unroll
    for (int u = 0; u < 8; ++u) tot = __dp4a(cnt[t * 8 + u], 0x01010101u, tot);
  }
  uint32_t x = tot;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) s_ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t y = s_ws[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t z = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) y += z;
    }
    s_ws[lane] = y;
  }
  __syncthreads();
  if ((uint32_t)t < nid) start[t] = x - tot + (w ? s_ws[w - 1] : 0u);
  __syncthreads();
  // records of this key in earlier warps: bytes [0, w) of the id's row
  uint32_t before = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t word = cnt[id * 8 + u];
    const int lo = 4 * u;
    const uint32_t m = w >= lo + 4 ? 0xFFFFFFFFu : (w <= lo ? 0u : (0xFFFFFFFFu >> (8 * (lo + 4 - w))));
    before = __dp4a(word & m, 0x01010101u, before);
  }
  const uint32_t pos = start[id] + before + rank;
  sk[pos] = key;
  sv[pos] = val;
  so[pos] = pay;
  uint32_t mylen = 0;
  if (before == 0 && rank == 0) {  // first record of the key
#pragma unroll
    for (int u = 0; u < 8; ++u) mylen = __dp4a(cnt[id * 8 + u], 0x01010101u, mylen);
  }
  sl[pos] = mylen;
  __syncthreads();
  key = sk[t];
  val = sv[t];
  len = sl[t];
  pay = so[t];
  __syncthreads();
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier (all CTAs are co-resident: cooperative launch).  One returning atomic per
// CTA on the arrival word: CTA 0 adds 2^31 - (G - 1), every other CTA adds 1, so the G arrivals
// add exactly 2^31 and flip the word's top bit whatever it held before (no reset, any grid size
// from launch to launch); a CTA leaves when the top bit differs from the one it saw on arrival.
__device__ __forceinline__ void coop_sync(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t add = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
    uint32_t old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(add) : "memory");
    while (((ld_acquire_u32(bar) ^ old) & 0x80000000u) == 0u) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint64_t fold_okey(double x) {
  return order_key(static_cast<uint64_t>(__double_as_longlong(x)));
}
__device__ __forceinline__ double fold_unkey(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

// The runs of one key in tile order, staged in shared memory by a warp: rstart[r] = index of
// the run's first record in the chunk arrays, rcum[r] = records before run r (rcum[nr] = cnt).
struct WarpRuns {
  int32_t rstart[kCoopTiles];
  int32_t rcum[kCoopTiles + 1];
  int32_t nr;
};

// An entry's fold inputs, loaded in one round trip (the 64 run slots unconditionally: the mask
// says which are live).  L2 loads (__ldcg): the chunk arrays are rewritten by other CTAs.
// (spread over the warp to save registers: lane 0 the tile mask, 1 / 2 the order-key bounds, 3
// obs_count, 4 the latency bits; every lane two run slots)
struct EntryPre {
  uint64_t w;
  uint32_t sv0, sv1;  // slots of tiles lane, lane + 32
  __device__ __forceinline__ uint64_t get(int l) const { return __shfl_sync(0xffffffffu, w, l); }
  __device__ __forceinline__ uint64_t mask() const { return get(0); }
  __device__ __forceinline__ uint64_t lo() const { return get(1); }
  __device__ __forceinline__ uint64_t hi() const { return get(2); }
  __device__ __forceinline__ int before() const { return (int)get(3); }
  __device__ __forceinline__ double L() const { return __longlong_as_double((long long)get(4)); }
};
__device__ __forceinline__ EntryPre entry_load(const CoopArgs& a, uint32_t key, const FoldTab& tb,
                                               int e) {
  const int lane = threadIdx.x & 31;
  EntryPre p;
  const uint64_t* src = reinterpret_cast<const uint64_t*>(lane == 1 ? a.lo : lane == 2 ? a.hi : a.mask) + key;
  if (lane == 4) src = reinterpret_cast<const uint64_t*>(tb.lat) + e;
  p.w = lane == 3 ? (uint64_t)(uint32_t)__ldcg(tb.obs_count + e)
                  : __ldcg(reinterpret_cast<const unsigned long long*>(src));
  p.sv0 = __ldcg(a.slot + (size_t)key * kCoopTiles + lane);
  p.sv1 = __ldcg(a.slot + (size_t)key * kCoopTiles + lane + 32);
  return p;
}

__device__ __forceinline__ int runs_load(const EntryPre& p, WarpRuns& R) {
  const int lane = threadIdx.x & 31;
  const uint64_t m = p.mask();
  int cnt = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int tl = lane + 32 * h;
    const bool has = (m >> tl) & 1ull;
    const uint32_t sv = h ? p.sv1 : p.sv0;
    const int len = has ? (int)(sv >> 16) : 0;
    // rank of this run among the key's runs, and records before it
    const uint64_t below = tl ? (m & ((1ull << tl) - 1ull)) : 0ull;
    const int r = __popcll(below);
    int pre = len;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, off);
      if (lane >= off) pre += y;
    }
    pre -= len;  // exclusive within this half
    if (has) {
      R.rstart[r] = tl * kCoopTile + (int)(sv & 0xFFFFu);
      R.rcum[r] = cnt + pre;
    }
    cnt += __shfl_sync(0xffffffffu, pre + len, 31);
  }
  if (lane == 0) {
    R.nr = __popcll(m);
    R.rcum[__popcll(m)] = cnt;
  }
  __syncwarp();
  return cnt;
}

// chunk-array index of the entry's ordinal-th observation
__device__ __forceinline__ int runs_at(const WarpRuns& R, int ordinal) {
  int lo = 0, hi = R.nr - 1;  // last run with rcum <= ordinal
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (R.rcum[mid] <= ordinal) lo = mid; else hi = mid - 1;
  }
  return R.rstart[lo] + (ordinal - R.rcum[lo]);
}

// buf[0, count) = the entry's observations [base, base + count), count <= kCoopWarpBuf: every
// lane's loads issued before any store (one memory round trip, not one per 32 observations)
// Elements from `scaled` on are stored as fl(beta * o), the chain's independent half, so the
// serial chains below carry one dependent DMUL + DADD per step.
__device__ __forceinline__ void gather_obs(const CoopArgs& a, const WarpRuns& R, double* buf,
                                           int base, int count, int scaled) {
  // cp.async: the copies need no registers while in flight (the grid barrier's acquire has
  // invalidated L1, so .ca sees the phase-A writes of other CTAs)
  for (int u = (threadIdx.x & 31); u < count; u += 32) {
    const double* src = a.sobs + runs_at(R, base + u);
    const unsigned dst = (unsigned)__cvta_generic_to_shared(buf + u);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  for (int u = scaled + (threadIdx.x & 31) - (scaled & 31); u < count; u += 32)  // own copies
    if (u >= scaled) buf[u] = __dmul_rn(a.beta, buf[u]);
  __syncwarp();
}

// Warp-cooperative exact fold of the entry's observations [o0, o1) from L (result valid in
// every lane).  With `bounded` (lo..hi holds every chain value) a window of the last `win`
// observations is tried first; it returns the exact value whenever the two bound chains meet.
__device__ double coop_fold(const CoopArgs& a, const WarpRuns& R, double* buf, double L, int o0,
                            int o1, bool bounded, double lo, double hi) {
  const int lane = threadIdx.x & 31;
  const double ob = a.beta, ol = __dsub_rn(1.0, a.beta);
  // Narrowed window (beta >= 1/2, positive normal-range values): the chain value 24 steps
  // before the end is bounded by interval arithmetic over the 64 observations before it —
  // every step y -> fl(fl(b o) + fl(a y)) lies in [(1-u)^2 (b o + a y), (1+u)^2 (b o + a y)]
  // (u = 2^-53) and is monotone in y, so from y in [lo, hi] 64 steps earlier
  //   y >= sum_j c_lo^(64-j) a^(63-j) b o_j + (c_lo a)^64 lo   (c_lo = 1 - 2^-52 <= (1-u)^2)
  //   y <= the same with c_hi = 1 + 2^-51 >= (1+u)^2 and hi,
  // evaluated by the warp with directed rounding (round-down / round-up); the exact chains then
  // run from the narrowed bounds over the last 24 observations only.  Bit-exact whenever the
  // two chains meet (else the full window below).
  constexpr int kNk = 64, kNw = 24;
  if (bounded && ol <= 0.5 && ob >= 0x1p-60 && ol >= 0x1p-60 && lo > 0x1p-900 && hi < 0x1p900 &&
      o1 - o0 >= kNk + kNw) {
    gather_obs(a, R, buf, o1 - kNw - kNk, kNk + kNw, kNk);
    const double cl = 1.0 - 0x1p-52, ch = 1.0 + 0x1p-51;
    const double ql = __dmul_rd(cl, ol), qh = __dmul_ru(ch, ol);
    const double bl = __dmul_rd(cl, ob), bh = __dmul_ru(ch, ob);
    double zl = 0.0, zh = 0.0, tl = 0.0, th = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h, m = kNk - 1 - j;
      double pl = 1.0, ph = 1.0, gl = ql, gh = qh;
#pragma unroll
      for (int bit = 0; bit < 6; ++bit) {
        if ((m >> bit) & 1) {
          pl = __dmul_rd(pl, gl);
          ph = __dmul_ru(ph, gh);
        }
        gl = __dmul_rd(gl, gl);
        gh = __dmul_ru(gh, gh);
      }
      tl = gl;  // (c_lo a)^64, (c_hi a)^64
      th = gh;
      const double o = buf[j];
      zl = __dadd_rd(zl, __dmul_rd(__dmul_rd(pl, bl), o));
      zh = __dadd_ru(zh, __dmul_ru(__dmul_ru(ph, bh), o));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      zl = __dadd_rd(zl, __shfl_xor_sync(0xffffffffu, zl, off));
      zh = __dadd_ru(zh, __shfl_xor_sync(0xffffffffu, zh, off));
    }
    zl = __dadd_rd(zl, __dmul_rd(tl, lo));
    zh = __dadd_ru(zh, __dmul_ru(th, hi));
    int same = 0;
    double v = 0.0;
    if (lane == 0) {
      double x = zl > lo ? zl : lo, y = zh < hi ? zh : hi;
#pragma unroll
      for (int u = kNk; u < kNk + kNw; ++u) {
        const double t = buf[u];  // fl(beta o)
        x = __dadd_rn(t, __dmul_rn(ol, x));
        y = __dadd_rn(t, __dmul_rn(ol, y));
      }
      v = x;
      same = __double_as_longlong(x) == __double_as_longlong(y);
    }
    same = __shfl_sync(0xffffffffu, same, 0);
    v = __shfl_sync(0xffffffffu, v, 0);
    __syncwarp();
    if (same) return v;
  }
  if (bounded && o1 - o0 > a.win && a.win <= kCoopWarpBuf) {
    gather_obs(a, R, buf, o1 - a.win, a.win, 0);
    int same = 0;
    double v = 0.0;
    if (lane == 0) {
      double x = lo, y = hi;
#pragma unroll 8
      for (int u = 0; u < a.win; ++u) {
        const double t = buf[u];  // fl(beta o)
        x = __dadd_rn(t, __dmul_rn(ol, x));
        y = __dadd_rn(t, __dmul_rn(ol, y));
      }
      v = x;
      same = __double_as_longlong(x) == __double_as_longlong(y);
    }
    same = __shfl_sync(0xffffffffu, same, 0);
    v = __shfl_sync(0xffffffffu, v, 0);
    __syncwarp();
    if (same) return v;
  }
  for (int p0 = o0; p0 < o1; p0 += kCoopWarpBuf) {
    const int p1 = min(o1, p0 + kCoopWarpBuf);
    gather_obs(a, R, buf, p0, p1 - p0, 0);
    if (lane == 0) {
#pragma unroll 8
      for (int u = 0; u < p1 - p0; ++u) L = __dadd_rn(buf[u], __dmul_rn(ol, L));  // buf: fl(beta o)
    }
    __syncwarp();
  }
  return __shfl_sync(0xffffffffu, L, 0);
}

// bounds of every chain value from the chunk's observation range of `key` and the start L
__device__ __forceinline__ bool coop_bounds(uint64_t klo, uint64_t khi, double L, double* lo,
                                            double* hi) {
  double m = fold_unkey(klo), M = fold_unkey(khi);
  if (!(isfinite(m) && isfinite(M) && isfinite(L))) return false;
  m = L < m ? L : m;
  M = L > M ? L : M;
  *lo = m - fabs(m) * 0x1p-20 - 0x1p-1000;
  *hi = M + fabs(M) * 0x1p-20 + 0x1p-1000;
  return true;
}

__global__ void __launch_bounds__(kCoopThreads, 1) k_fold_coop(const __grid_constant__ CoopArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_key[kCoopTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpRuns& R = reinterpret_cast<WarpRuns*>(smem)[warp];
  double* buf = reinterpret_cast<double*>(smem + sizeof(WarpRuns) * kCoopWarps) + warp * kCoopWarpBuf;
  const uint32_t sent = (uint32_t)a.ft.total;
  CoopState* st = a.st;
  __shared__ uint64_t tm[8];  // SP_PC_DEBUG phase timestamps (thread 0)
  const bool dbg = a.debug && threadIdx.x == 0;
  if (dbg) tm[0] = coop_timer();
  // programmatic dependent launch: the observation stream and the tables are the predecessors'
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  for (int c0 = 0, chunk = 0; c0 < a.n; c0 += kCoopChunk, ++chunk) {
    const int par = chunk & 1;
    const int nrec = min(kCoopChunk, a.n - c0);
    const int ntiles = (nrec + kCoopTile - 1) / kCoopTile;
    // ---- phase A (records grouped by key, not sorted: the runs only need to be contiguous) ----
    for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      const int j = c0 + tl * kCoopTile + (int)threadIdx.x;
      uint32_t key[1] = {sent}, val[1] = {(uint32_t)j};
      double o = 0.0;  // loaded before the grouping, carried through it
      if (j < a.n) {
        const int e = coop_entry(a, j);
        if (e >= 0) {
          key[0] = (uint32_t)(a.ft.t[a.op ? a.op[j] : 0].gbase + e);
          o = coop_obs(a, j);
        }
        if (a.rec_idx) {
          a.rec_idx[j] = e;
          a.rec_obs[j] = o;
        }
      }
      __syncthreads();  // tmp / s_key reuse across tiles
      if (dbg && chunk == 0) tm[1] = coop_timer();
      uint32_t run_len;
      tile_group(key[0], val[0], run_len, o, smem);
      if (dbg && chunk == 0) tm[2] = coop_timer();
      const uint32_t k = key[0];
      s_key[threadIdx.x] = k;
      const int q = tl * kCoopTile + (int)threadIdx.x;  // chunk-array index
      a.skey[q] = k;
      a.spos[q] = val[0];
      a.sobs[q] = o;
      __syncthreads();
      // warp-segmented min / max of the run inside this warp (keys are sorted)
      uint64_t mn = fold_okey(o), mx = mn;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t ko = __shfl_up_sync(0xffffffffu, k, off);
        const uint64_t a0 = __shfl_up_sync(0xffffffffu, mn, off);
        const uint64_t a1 = __shfl_up_sync(0xffffffffu, mx, off);
        if (lane >= off && ko == k) {
          mn = a0 < mn ? a0 : mn;
          mx = a1 > mx ? a1 : mx;
        }
      }
      const bool last_in_warp = lane == 31 || s_key[threadIdx.x + 1] != k;
      if (k != sent) {
        if (last_in_warp) {
          atomicMin(reinterpret_cast<unsigned long long*>(a.lo + k), (unsigned long long)mn);
          atomicMax(reinterpret_cast<unsigned long long*>(a.hi + k), (unsigned long long)mx);
        }
        if (run_len) {  // run head
          const int len = (int)run_len;
          a.slot[(size_t)k * kCoopTiles + tl] = threadIdx.x | (uint32_t)len << 16;
          const unsigned long long old =
              atomicOr(reinterpret_cast<unsigned long long*>(a.mask + k), 1ull << tl);
          if (old == 0ull) a.touched[atomicAdd(&st->touched_n[par], 1)] = (int32_t)k;
          const int t = table_of_key(a.ft, k);
          if ((int)k - a.ft.t[t].gbase == a.ft.t[t].ref_index) atomicAdd(&st->refcnt[par][t], len);
        }
      }
    }
    if (a.debug > 1) __syncthreads();
    if (dbg && chunk == 0) tm[3] = coop_timer();
    coop_sync(st->bar);
    if (dbg && chunk == 0) tm[4] = coop_timer();
    // ---- gates of this chunk: every warp evaluates them itself (lane t: tables t, t + 32; the
    // same value in every warp), with the first touched entry's loads in the same round trip ----
    const int nt = (int)__ldcg(&st->touched_n[par]);
    // touched entries dealt CTA-major (entry u -> CTA u mod G): the first-touched (hottest) entries
    // land on different SMs instead of contending for one SM's FP64 pipe with their serial chains
    const int u0 = warp * gridDim.x + blockIdx.x, ustride = gridDim.x * kCoopWarps;
    // speculative until nt is known: clamped into the key space, used only when u0 < nt
    const uint32_t key0 = min(__ldcg(reinterpret_cast<const uint32_t*>(a.touched) + u0), sent - 1u);
    const int t0 = table_of_key(a.ft, key0);
    EntryPre pre0 = entry_load(a, key0, a.ft.t[t0], (int)key0 - a.ft.t[t0].gbase);
    uint64_t lift = 0;
    {
      bool g[2] = {false, false};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        if (t < a.ft.n) {
          const FoldTab& tb = a.ft.t[t];
          const int rc = __ldcg(&st->refcnt[par][t]);
          const int done = __ldcg(tb.counters);
          const double li = __ldcg(tb.lat_init + (tb.ref_index > 0 ? tb.ref_index : 0));
          const int k = a.dfp_count - done;
          g[h] = !a.fb_frozen && a.dfp_on && tb.ref_index >= 0 && rc > 0 && k >= 1 && k <= rc && li > 0.0;
        }
      }
      lift = (uint64_t)__ballot_sync(0xffffffffu, g[0]) | (uint64_t)__ballot_sync(0xffffffffu, g[1]) << 32;
    }
    // last chunk, no gate lift: nothing after this point reads the counters phase D resets, and
    // nothing after phase C reads another CTA's phase-C writes in this launch — so no barrier
    // after phase C: every CTA checks in here (its warps have read touched_n and the gates) and
    // the last one to check in does phase D while the others fold
    const bool early_d = !lift && c0 + kCoopChunk >= a.n;
    if (early_d) {
      __syncthreads();
      if (warp == 0) {
        uint32_t old = 0;
        if (lane == 0)
          asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(st->bar + 1) : "memory");
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == gridDim.x - 1u) {
          for (int t = lane; t < a.ft.n; t += 32) {
            a.ft.t[t].counters[0] += st->refcnt[par][t];
            st->refcnt[par][t] = 0;
          }
          if (lane == 0) {
            st->touched_n[par] = 0;
            st->bar[1] = 0u;
          }
        }
      }
    }
    if (lift) {  // ---- phase B: the reference entries of the lifting tables ----
      const int gw = blockIdx.x * kCoopWarps + warp;
      for (int t = gw; t < a.ft.n; t += gridDim.x * kCoopWarps) {
        if (!((lift >> t) & 1ull)) continue;
        const FoldTab& tb = a.ft.t[t];
        const uint32_t rk = (uint32_t)(tb.gbase + tb.ref_index);
        const EntryPre pre = entry_load(a, rk, tb, tb.ref_index);
        const int cnt = runs_load(pre, R);
        const int k = a.dfp_count - __ldcg(tb.counters);
        double L = pre.L(), lo = 0.0, hi = 0.0;
        const bool bd = cnt > a.win && coop_bounds(pre.lo(), pre.hi(), L, &lo, &hi);
        L = coop_fold(a, R, buf, L, 0, k, bd, lo, hi);
        const double ratio = __ddiv_rn(L, tb.lat_init[tb.ref_index]);  // configurator.py:486
        const int gpos = (int)a.spos[runs_at(R, k - 1)];
        L = coop_fold(a, R, buf, L, k, cnt, bd, lo, hi);
        if (lane == 0) {
          tb.lat[tb.ref_index] = L;
          tb.dirty[tb.ref_index] = 1;
          tb.obs_count[tb.ref_index] += cnt;
          a.gates[t] = Gate{1, gpos, ratio};
          a.mask[rk] = 0ull;
          a.lo[rk] = ~0ull;
          a.hi[rk] = 0ull;
        }
        __syncwarp();
      }
      coop_sync(st->bar);
      pre0 = entry_load(a, key0, a.ft.t[t0], (int)key0 - a.ft.t[t0].gbase);  // not kept live across B
    }
    // ---- phase C: every touched entry (warp each) ----
    {
      uint32_t key = key0;
      EntryPre pre = pre0;
      for (int u = u0; u < nt;) {
        const int t = table_of_key(a.ft, key);
        const FoldTab& tb = a.ft.t[t];
        const int e = (int)key - tb.gbase;
        const bool skip = ((lift >> t) & 1ull) && e == tb.ref_index;  // folded in phase B
        if (skip) {
          u += ustride;
          if (u < nt) {
            key = __ldcg(reinterpret_cast<const uint32_t*>(a.touched) + u);
            const int tn = table_of_key(a.ft, key);
            pre = entry_load(a, key, a.ft.t[tn], (int)key - a.ft.t[tn].gbase);
          }
          continue;
        }
        const int before = pre.before();
        double L = pre.L();
        const uint64_t klo = pre.lo(), khi = pre.hi();
        const int cnt = runs_load(pre, R);
        if (!a.fb_frozen) {
          if ((lift >> t) & 1ull) {
            const Gate g = a.gates[t];
            if (before == 0 && (int)a.spos[R.rstart[0]] > g.gate_pos)
              L = __dmul_rn(tb.lat_init[e], g.ratio);
          }
          double lo = 0.0, hi = 0.0;
          const bool bd = cnt > a.win && coop_bounds(klo, khi, L, &lo, &hi);
          L = coop_fold(a, R, buf, L, 0, cnt, bd, lo, hi);
          if (lane == 0) {
            tb.lat[e] = L;
            tb.dirty[e] = 1;
          }
        }
        if (lane == 0) {
          tb.obs_count[e] = before + cnt;
          a.mask[key] = 0ull;
          a.lo[key] = ~0ull;
          a.hi[key] = 0ull;
        }
        __syncwarp();
        u += ustride;
        if (u < nt) {
          key = __ldcg(reinterpret_cast<const uint32_t*>(a.touched) + u);
          const int tn = table_of_key(a.ft, key);
          pre = entry_load(a, key, a.ft.t[tn], (int)key - a.ft.t[tn].gbase);
        }
      }
    }
    if (a.debug > 1) __syncthreads();
    if (dbg && chunk == 0) tm[5] = coop_timer();
    if (early_d) {  // phase D is done (above)
      if (dbg && chunk == 0) tm[6] = coop_timer();
      break;
    }
    coop_sync(st->bar);
    if (dbg && chunk == 0) tm[6] = coop_timer();
    // ---- phase D ----
    if (blockIdx.x == 0 && threadIdx.x < a.ft.n) {
      const int t = threadIdx.x;
      a.ft.t[t].counters[0] += st->refcnt[par][t];
      st->refcnt[par][t] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->touched_n[par] = 0;
    if (lift) {
      for (int t = 0; t < a.ft.n; ++t) {
        if (!((lift >> t) & 1ull)) continue;
        const FoldTab& tb = a.ft.t[t];
        const double ratio = a.gates[t].ratio;
        for (int e = blockIdx.x * kCoopThreads + threadIdx.x; e < tb.M; e += gridDim.x * kCoopThreads)
          if (e != tb.ref_index && tb.obs_count[e] == 0) {
            tb.lat[e] = __dmul_rn(tb.lat_init[e], ratio);  // configurator.py:490
            tb.dirty[e] = 1;
          }
      }
    }
    // the next chunk's phase C reads counters / latencies written here: its phase-A barrier
    // orders them
  }
  if (a.debug > 1 && threadIdx.x == 0) {
    tm[7] = coop_timer();
    printf("fold abs cta %d smid %u: t0 %llu A_end %llu barA_out %llu C_end %llu end %llu\n", blockIdx.x,
           coop_smid(), (unsigned long long)tm[0] % 100000000ull, (unsigned long long)tm[3] % 100000000ull,
           (unsigned long long)tm[4] % 100000000ull, (unsigned long long)tm[5] % 100000000ull,
           (unsigned long long)tm[7] % 100000000ull);
  }
  if (a.debug && threadIdx.x == 0 && blockIdx.x < 2) {
    tm[7] = coop_timer();
    printf("fold cta %d: start->sort %llu sort %llu runs %llu barA %llu C %llu barC %llu D %llu ns\n",
           blockIdx.x, (unsigned long long)(tm[1] - tm[0]), (unsigned long long)(tm[2] - tm[1]),
           (unsigned long long)(tm[3] - tm[2]), (unsigned long long)(tm[4] - tm[3]),
           (unsigned long long)(tm[5] - tm[4]), (unsigned long long)(tm[6] - tm[5]),
           (unsigned long long)(tm[7] - tm[6]));
  }
}

// Persistent state of the one-kernel fold: per-key masks / bounds / slots (sized for the
// largest key space seen), chunk arrays, the barrier and counters.
struct CoopBuffers {
  int64_t keys = 0;
  uint8_t* base = nullptr;
};

static int coop_buffers(sp_ctx* ctx, int64_t keys, CoopArgs& a) {
  // per context: two contexts of one device may fold concurrently on their own streams
  if (!ctx->coop) ctx->coop = new CoopBuffers();
  CoopBuffers& b = *static_cast<CoopBuffers*>(ctx->coop);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t chunk = al(4u * kCoopChunk) * 2 + al(8u * kCoopChunk) + al(4u * kCoopChunk);
  const size_t gates = al(sizeof(Gate) * kMaxFoldTables), stb = al(sizeof(CoopState));
  if (keys > b.keys) {
    int64_t cap = std::max<int64_t>(keys, 1 << 14);
    if (b.base) {
      SP_CUDA(cudaStreamSynchronize(ctx->stream));
      SP_CUDA(cudaFree(b.base));
      b.base = nullptr;
      b.keys = 0;
    }
    const size_t per = al(8u * cap) * 3 + al(4u * kCoopTiles * cap);
    SP_CUDA(cudaMalloc(&b.base, per + chunk + gates + stb));
    uint8_t* q = b.base;
    // stream-ordered before the fold kernel (the context stream is non-blocking: a legacy
    // cudaMemset on the NULL stream would race with it)
    SP_CUDA(cudaMemsetAsync(q, 0, al(8u * cap), ctx->stream));                    // mask
    SP_CUDA(cudaMemsetAsync(q + al(8u * cap), 0xFF, al(8u * cap), ctx->stream));  // lo
    SP_CUDA(cudaMemsetAsync(q + 2 * al(8u * cap), 0, al(8u * cap), ctx->stream)); // hi
    SP_CUDA(cudaMemsetAsync(q + per + chunk + gates, 0, stb, ctx->stream));       // barrier / counters
    // run slots and the touched list: read speculatively (ignored unless live), kept defined
    SP_CUDA(cudaMemsetAsync(q + 3 * al(8u * cap), 0, al(4u * kCoopTiles * cap), ctx->stream));
    SP_CUDA(cudaMemsetAsync(q + per, 0, chunk, ctx->stream));
    b.keys = cap;
  }
  const int64_t cap = b.keys;
  uint8_t* q = b.base;
  a.mask = reinterpret_cast<uint64_t*>(q);
  a.lo = reinterpret_cast<uint64_t*>(q + al(8u * cap));
  a.hi = reinterpret_cast<uint64_t*>(q + 2 * al(8u * cap));
  a.slot = reinterpret_cast<uint32_t*>(q + 3 * al(8u * cap));
  q += al(8u * cap) * 3 + al(4u * kCoopTiles * cap);
  a.skey = reinterpret_cast<uint32_t*>(q);
  a.spos = reinterpret_cast<uint32_t*>(q + al(4u * kCoopChunk));
  a.sobs = reinterpret_cast<double*>(q + 2 * al(4u * kCoopChunk));
  a.touched = reinterpret_cast<int32_t*>(q + 2 * al(4u * kCoopChunk) + al(8u * kCoopChunk));
  q += chunk;
  a.gates = reinterpret_cast<Gate*>(q);
  a.st = reinterpret_cast<CoopState*>(q + gates);
  return SP_OK;
}

static int fold_launch_coop(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n,
                            const int32_t* op, const int32_t* idx, const double* obs, double beta,
                            int dfp_count, int dfp_on, int fb_frozen, const CoopArgs* sim = nullptr) {
  CoopArgs a;
  a.d_code = sim ? sim->d_code : nullptr;
  a.d_idx = sim ? sim->d_idx : nullptr;
  a.d_fill = sim ? sim->d_fill : nullptr;
  a.t_base = sim ? sim->t_base : nullptr;
  a.t_per_item = sim ? sim->t_per_item : nullptr;
  a.t_noise = sim ? sim->t_noise : nullptr;
  a.rec_idx = sim ? sim->rec_idx : nullptr;
  a.rec_obs = sim ? sim->rec_obs : nullptr;
  a.ft.n = n_tables;
  int64_t gb = 0;
  for (int t = 0; t < n_tables; ++t) {
    sp_table* tb = tables[t];
    a.ft.t[t] = FoldTab{tb->lat, tb->lat_init, tb->obs_count, tb->dev_counters, tb->dirty, tb->M,
                        tb->ref_index, (int32_t)gb, 0};
    gb += tb->M;
  }
  if (gb >= (1ll << 31) - 1) return fail(SP_E_UNSUPPORTED, "fold: too many entries");
  a.ft.total = (int)gb;
  int end_bit = 1;
  while ((1ll << end_bit) <= gb) ++end_bit;
  a.end_bit = end_bit;
  a.n = n;
  a.op = op;
  a.idx = idx;
  a.obs = obs;
  a.beta = beta;
  const double ol = 1.0 - beta;
  int win = 8;
  if (ol > 0.0) {
    const double w = ceil(80.0 / -log2(ol));
    win = w > 4096.0 ? (1 << 30) : (w < 8.0 ? 8 : (int)w);
  }
  a.win = win;
  a.dfp_count = dfp_count;
  a.dfp_on = dfp_on;
  a.fb_frozen = fb_frozen;
  a.debug = ctx->opt.pc_debug;
  int rc = coop_buffers(ctx, gb + 1, a);
  if (rc != SP_OK) return rc;
  const size_t smem = std::max((size_t)kTileGroupSmem,
                               sizeof(WarpRuns) * kCoopWarps + 8u * kCoopWarpBuf * kCoopWarps);
  static uint64_t attr = 0;
  static int max_blocks[64] = {};
  const int dev = cur_device();
  if (attr_once(attr)) {
    SP_CUDA(cudaFuncSetAttribute(k_fold_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int per_sm = 0;
    SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fold_coop, kCoopThreads, smem));
    max_blocks[dev] = per_sm * ctx->num_sms;
  }
  if (max_blocks[dev] < 1) return fail(SP_E_RUNTIME, "fold: cooperative kernel cannot be resident");
  const int tiles = (std::min(n, kCoopChunk) + kCoopTile - 1) / kCoopTile;
  int grid = std::min(max_blocks[dev], std::max(tiles, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kCoopThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute la[2];
  la[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers
  la[0].val.cooperative = 1;
  la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[1].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
  cfg.attrs = la;
  cfg.numAttrs = 2;
  SP_CUDA(cudaLaunchKernelEx(&cfg, k_fold_coop, a));
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

}  // namespace

int fold_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n, const int32_t* op,
                const int32_t* idx, const double* obs, double beta, int dfp_count, int dfp_on,
                int fb_frozen) {
  if (n_tables > kMaxFoldTables) return fail(SP_E_UNSUPPORTED, "fold: at most 64 tables");
  if (ctx->opt.fold_legacy || n == 0)
    return fold_launch_legacy(ctx, n_tables, tables, n, op, idx, obs, beta, dfp_count, dfp_on,
                              fb_frozen);
  int rc = fold_launch_coop(ctx, n_tables, tables, n, op, idx, obs, beta, dfp_count, dfp_on,
                            fb_frozen);
  if (rc == SP_OK)
    for (int t = 0; t < n_tables; ++t) tables[t]->version++;
  return rc;
}

int simulate_and_fold(sp_ctx* ctx, sp_table* t, int n, const int32_t* code, const int32_t* idx,
                      const int32_t* fill, const double* base, const double* per_item,
                      const double* noise, double beta, int dfp_count, int dfp_on, int fb_frozen,
                      int32_t* rec_idx, double* rec_obs) {
  if (ctx->opt.fold_legacy || n == 0 || !rec_idx) {  // the two-kernel form
    if (!rec_idx) return fail(SP_E_INVALID, "simulate_and_fold: record buffers required");
    const int rc = sp_simulate_observations(ctx, n, code, idx, fill, base, per_item, noise, rec_idx,
                                            rec_obs);
    if (rc != SP_OK) return rc;
    return fold_launch(ctx, 1, &t, n, nullptr, rec_idx, rec_obs, beta, dfp_count, dfp_on, fb_frozen);
  }
  CoopArgs sim;
  sim.d_code = code;
  sim.d_idx = idx;
  sim.d_fill = fill;
  sim.t_base = base;
  sim.t_per_item = per_item;
  sim.t_noise = noise;
  sim.rec_idx = rec_idx;
  sim.rec_obs = rec_obs;
  const int rc = fold_launch_coop(ctx, 1, &t, n, nullptr, nullptr, nullptr, beta, dfp_count, dfp_on,
                                  fb_frozen, &sim);
  if (rc == SP_OK) t->version++;
  return rc;
}

}  // namespace sp

namespace sp {
void coop_release(sp_ctx* ctx) {
  if (!ctx->coop) return;
  CoopBuffers* b = static_cast<CoopBuffers*>(ctx->coop);
  cudaFree(b->base);
  delete b;
  ctx->coop = nullptr;
}
}  // namespace sp
