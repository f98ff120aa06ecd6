// sp_quantile.cu — K3 extension: per-entry latency percentiles of an observation batch.
//
// BASELINE.json's north star asks for a "profile-update / percentile-estimate" kernel.  The
// reference folds observations only through the EWMA (manager.py:45-47, reproduced bit-exactly
// by sp_fold.cu) and has no percentile anywhere, so this output is an
// extension whose parity is pinned to numpy, not to the reference:
//   out[e] = np.quantile(obs of entry e in the batch, q, method="inverted_cdf")
//          = the ceil(q * n_e)-th smallest observation (the smallest for q = 0), NaN if n_e = 0
//   count[e] = n_e
// optionally smoothed across batches (out_smooth[e] = beta*out[e] + (1-beta)*out_smooth[e]
// where n_e > 0, the EWMA of manager.py:45-47 applied to the batch percentile).
// Device plan: two stable CUB radix sorts — observations by value, then by (table, entry) —
// give every entry's observations as one ascending run; a histogram + exclusive scan of the
// entry counts locates each run, and one thread per entry reads its order statistic.
#include <math.h>

#include <cub/cub.cuh>

#include "sp_internal.cuh"

namespace sp {
namespace {

__device__ __forceinline__ uint64_t obs_key(double x) {  // monotone u64 key of a double
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct QTab {
  int32_t gbase[64];
  int n;
  int total;
};

__global__ void k_q_keys(int n, QTab qt, const int32_t* __restrict__ op,
                         const int32_t* __restrict__ idx, const double* __restrict__ obs,
                         uint64_t* vkey, uint32_t* ent) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int t = op ? op[j] : 0;
  vkey[j] = obs_key(obs[j]);
  ent[j] = idx[j] < 0 ? (uint32_t)qt.total : (uint32_t)(qt.gbase[t] + idx[j]);
}

__global__ void k_q_value_of(int n, const uint64_t* __restrict__ vkey_sorted, uint32_t* key2,
                             const uint32_t* __restrict__ ent_sorted, double* vals) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint64_t k = vkey_sorted[j];
  const uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  vals[j] = __longlong_as_double(static_cast<long long>(u));
  key2[j] = ent_sorted[j];
}

__global__ void k_q_count(int n, int total, const uint32_t* __restrict__ ent, int32_t* cnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t e = ent[j];
  if ((int)e < total) atomicAdd(&cnt[e], 1);
}

__global__ void k_q_pick(int total, double q, const int32_t* __restrict__ cnt,
                         const int32_t* __restrict__ start, const double* __restrict__ vals,
                         double beta, double* out, int32_t* out_count, double* out_smooth) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int c = cnt[e];
  double v = NAN;
  if (c > 0) {
    // numpy inverted_cdf: the smallest x with F(x) >= q  ->  rank ceil(q * n), 1-based
    int r = (int)ceil(__dmul_rn(q, (double)c));
    r = r < 1 ? 1 : (r > c ? c : r);
    v = vals[start[e] + r - 1];
    if (out_smooth) {
      const double old = out_smooth[e];
      out_smooth[e] = old == old ? __dadd_rn(__dmul_rn(beta, v), __dmul_rn(__dsub_rn(1.0, beta), old))
                                 : v;  // first batch with an observation: start at the value
    }
  }
  if (out) out[e] = v;
  if (out_count) out_count[e] = c;
}

}  // namespace

int quantile_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n, const int32_t* op,
                    const int32_t* idx, const double* obs, double q, double beta, double* out,
                    int32_t* out_count, double* out_smooth) {
  if (n_tables > 64) return fail(SP_E_UNSUPPORTED, "quantiles: at most 64 tables");
  QTab qt;
  int64_t gb = 0;
  for (int t = 0; t < n_tables; ++t) {
    qt.gbase[t] = (int32_t)gb;
    gb += tables[t]->M;
  }
  if (gb >= (1ll << 31) - 1) return fail(SP_E_UNSUPPORTED, "quantiles: too many entries");
  qt.n = n_tables;
  qt.total = (int)gb;
  const int total = (int)gb;
  int end_bit = 1;
  while ((1ll << end_bit) <= gb) ++end_bit;
  cudaStream_t st = ctx->stream;
  size_t b1 = 0, b2 = 0, b3 = 0;
  const int nn = n > 0 ? n : 1;
  SP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                          (const uint32_t*)nullptr, (uint32_t*)nullptr, nn, 0, 64, st));
  SP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                          (const double*)nullptr, (double*)nullptr, nn, 0, end_bit, st));
  SP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b3, (const int32_t*)nullptr, (int32_t*)nullptr,
                                        total > 0 ? total : 1, st));
  const size_t cb = std::max(b1, std::max(b2, b3));
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t need = 2 * al(8 * (size_t)nn) + 2 * al(4 * (size_t)nn) + al(8 * (size_t)nn) +
                      al(4 * (size_t)nn) + al(8 * (size_t)nn) + 2 * al(4 * (size_t)(total + 1)) +
                      al(cb);
  int rc = SP_OK;
  uint8_t* s = static_cast<uint8_t*>(ctx_tmp(ctx, need, &rc));
  if (!s) return rc;
  uint64_t* vk = reinterpret_cast<uint64_t*>(s); s += al(8 * (size_t)nn);
  uint64_t* vk2 = reinterpret_cast<uint64_t*>(s); s += al(8 * (size_t)nn);
  uint32_t* en = reinterpret_cast<uint32_t*>(s); s += al(4 * (size_t)nn);
  uint32_t* en2 = reinterpret_cast<uint32_t*>(s); s += al(4 * (size_t)nn);
  double* v1 = reinterpret_cast<double*>(s); s += al(8 * (size_t)nn);
  uint32_t* k2 = reinterpret_cast<uint32_t*>(s); s += al(4 * (size_t)nn);
  double* v2 = reinterpret_cast<double*>(s); s += al(8 * (size_t)nn);
  int32_t* cnt = reinterpret_cast<int32_t*>(s); s += al(4 * (size_t)(total + 1));
  int32_t* start = reinterpret_cast<int32_t*>(s); s += al(4 * (size_t)(total + 1));
  void* ctmp = s;
  SP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)total, st));
  if (n > 0) {
    k_q_keys<<<(n + 255) / 256, 256, 0, st>>>(n, qt, op, idx, obs, vk, en);
    SP_CHECK_LAUNCH(ctx);
    size_t t1 = cb;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(ctmp, t1, vk, vk2, en, en2, n, 0, 64, st));
    k_q_value_of<<<(n + 255) / 256, 256, 0, st>>>(n, vk2, k2, en2, v1);
    SP_CHECK_LAUNCH(ctx);
    // stable by entry: observations of each entry end up contiguous and still ascending
    size_t t2 = cb;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(ctmp, t2, k2, en, v1, v2, n, 0, end_bit, st));
    k_q_count<<<(n + 255) / 256, 256, 0, st>>>(n, total, en, cnt);
    SP_CHECK_LAUNCH(ctx);
    ctx->launches += 4;  // CUB passes (at least)
  }
  if (total > 0) {
    size_t t3 = cb;
    SP_CUDA(cub::DeviceScan::ExclusiveSum(ctmp, t3, cnt, start, total, st));
    k_q_pick<<<(total + 255) / 256, 256, 0, st>>>(total, q, cnt, start, v2, beta, out, out_count,
                                                  out_smooth);
    SP_CHECK_LAUNCH(ctx);
  }
  return SP_OK;
}

}  // namespace sp
