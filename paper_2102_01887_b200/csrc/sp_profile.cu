// sp_profile.cu — profile generation on the device (generation half).
//
// The reference profiles an operation by enumerating its knob template's cross product
// (pipeline.py:454-475, enumerate_configs: kinds sorted, then resource options, batch sizes
// ascending, then the knob values in template order, last knob fastest) and, for every
// assignment, averaging `samples` draws of the ground-truth latency law (profiler.py:35-85 ->
// backend.py:36-58 -> scenario.py:68-77):
//
//     lat  = base_seconds
//     lat *= (R / ref_resource) ** -resource_exponent        (only when the exponent is nonzero)
//     lat *= B ** batch_exponent
//     lat *= knob_multipliers[knob][str(value)]  per knob     (1.0 when absent)
//     draw = lat + per_item_seconds * B                       (item_count = B)
//     draw *= exp(N(0, sigma))   [noise]    draw *= straggle_factor   [straggle]
//     latency = sum(draws) / samples          (CPython's float sum: Neumaier-compensated)
//
// One thread per assignment decodes its (kind, resource, batch, knob values) from the
// enumeration index and evaluates the law in the reference's operation order.  The noise and
// straggle factors are the reference's RNG stream (numpy PCG64 normals through CPython's
// math.exp, Bernoulli straggles) drawn on the host in the reference's order and passed in; the
// device evaluates everything else.
//
// `**` is CPython's float pow = the C library's pow.  The kernel computes the CORRECTLY
// ROUNDED x ** y: log and exp in double-double arithmetic (~2^-94 relative), then one rounding.
// glibc's pow is accurate to 0.52 ulp, so the two agree except where glibc itself misrounds
// (measured: 0 of the 101 (x, y) pairs the synthetic and AMBER scenarios use, ~0.08 % of
// random arguments).
#include <math.h>

#include "sp_internal.cuh"

namespace sp {
namespace {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = __dadd_rn(p.lo, __dmul_rn(a.lo, b));
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b) {  // b a small exact integer
  const double q1 = __ddiv_rn(a.hi, b);
  const dd p = two_prod(q1, b);
  const double r = __dadd_rn(__dsub_rn(__dsub_rn(a.hi, p.hi), p.lo), a.lo);
  return quick_two_sum(q1, __ddiv_rn(r, b));
}

// ln 2 = L0 + L1 + L2 (each term 53 bits)
constexpr double kLn2Hi = 0x1.62e42fefa39efp-1;
constexpr double kLn2Mid = 0x1.abc9e3b39803fp-56;
constexpr double kLn2Lo = 0x1.7b57a079a1934p-111;

// e^x for a double-double x with |x| < 709: x = n ln2 + r, e^(r / 2^10) by its Taylor series
// (degree 9, Horner with exact small-integer divisions), squared ten times, scaled by 2^n
__device__ dd dd_exp(dd x) {
  const double n = rint(__dmul_rn(x.hi, 1.4426950408889634));
  // r = x - n ln2 with n ln2 as an (almost) exact triple-word product
  dd r = x;
  const dd a = two_prod(n, kLn2Hi), b = two_prod(n, kLn2Mid);
  r = dd_add(r, dd{-a.hi, -a.lo});
  r = dd_add(r, dd{-b.hi, -b.lo});
  r = dd_add(r, dd{-__dmul_rn(n, kLn2Lo), 0.0});
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  dd s{1.0, 0.0};
  for (int k = 9; k >= 1; --k) {  // 1 + r/1 (1 + r/2 (1 + ... (1 + r/9)))
    s = dd_div_d(dd_mul(s, r), (double)k);
    s = dd_add(s, dd{1.0, 0.0});
  }
  for (int k = 0; k < 10; ++k) s = dd_mul(s, s);
  const int ni = (int)n;
  return {ldexp(s.hi, ni), ldexp(s.lo, ni)};
}

// log x for a positive normal double: y0 = log x, one Newton step y0 + (x e^-y0 - 1) - u^2/2
__device__ dd dd_log(double x) {
  const double y0 = log(x);
  if (y0 == 0.0) return {0.0, 0.0};
  const dd t = dd_exp(dd{-y0, 0.0});
  dd u = dd_mul_d(t, x);
  u = dd_add(u, dd{-1.0, 0.0});
  const dd u2 = dd_mul(u, u);
  dd y = dd_add(dd{y0, 0.0}, u);
  return dd_add(y, dd{-0.5 * u2.hi, -0.5 * u2.lo});
}

}  // namespace

// Correctly rounded x ** y for x > 0 finite (the cases CPython's float pow reaches for the
// latency law); other arguments take CUDA's pow.
__device__ double cr_pow(double x, double y) {
  if (y == 0.0 || x == 1.0) return 1.0;
  if (y == 1.0) return x;
  if (!(x > 0.0) || !isfinite(x) || !isfinite(y) || x < 0x1p-1000 || x > 0x1p1000) return pow(x, y);
  const dd l = dd_log(x);
  const dd z = dd_mul_d(l, y);
  if (z.hi > 709.0 || z.hi < -708.0) return pow(x, y);  // overflow / subnormal range
  const dd e = dd_exp(z);
  return __dadd_rn(e.hi, e.lo);
}

namespace {

struct ProfArgs {
  int K;                      // kinds (sorted order)
  const int64_t* koff;        // K + 1: first assignment of each kind
  const int32_t* roff;        // K + 1: resource options of kind k at ropt[roff[k] ..]
  const int32_t* ropt;        // resource option values
  const double* base;         // per kind: base_seconds
  const double* ref_res;      // per kind: ref_resource (as double)
  const double* rexp;         // per kind: resource_exponent
  const double* bexp;         // per kind: batch_exponent
  const double* per_item;     // per kind: per_item_seconds
  int nb;                     // batch sizes (ascending)
  const int32_t* batches;
  int nk;                     // knobs (template order)
  const int32_t* kcnt;        // per knob: number of values
  const int32_t* moff;        // per knob: offset of its values in a kind's multiplier row
  int mrow;                   // multipliers per kind (sum of kcnt)
  const double* mult;         // K x mrow: multiplier of (kind, knob, value), 1.0 when absent
  int64_t combos;             // product of kcnt
  int S;                      // samples per configuration
  const double* noise;        // N x S factors exp(N(0, sigma)), or null
  const double* strag;        // N x S factors (straggle_factor or 1.0), or null
  int64_t N;
  double* out_lat;
  int32_t* out_kind;
  int32_t* out_res;
  int32_t* out_batch;
};

__global__ void k_profile(const __grid_constant__ ProfArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  int k = 0;
  while (k + 1 < a.K && a.koff[k + 1] <= i) ++k;
  const int64_t rem = i - a.koff[k];
  const int64_t per_res = (int64_t)a.nb * a.combos;
  const int ri = (int)(rem / per_res);
  const int64_t rem2 = rem - (int64_t)ri * per_res;
  const int bi = (int)(rem2 / a.combos);
  int64_t c = rem2 - (int64_t)bi * a.combos;
  const int R = a.ropt[a.roff[k] + ri], B = a.batches[bi];
  // scenario.py:68-77 OpKindTruth.base_latency, in its operation order
  double lat = a.base[k];
  if (a.rexp[k] != 0.0) lat = __dmul_rn(lat, cr_pow(__ddiv_rn((double)R, a.ref_res[k]), -a.rexp[k]));
  lat = __dmul_rn(lat, cr_pow((double)B, a.bexp[k]));
  int vi[16];
  for (int j = a.nk - 1; j >= 0; --j) {  // itertools.product: the last knob varies fastest
    vi[j] = (int)(c % a.kcnt[j]);
    c /= a.kcnt[j];
  }
  for (int j = 0; j < a.nk; ++j) lat = __dmul_rn(lat, a.mult[(size_t)k * a.mrow + a.moff[j] + vi[j]]);
  // backend.py:52-58 per sample; profiler.py:64-68 the mean (sum from int 0, then / samples)
  const double draw0 = __dadd_rn(lat, __dmul_rn(a.per_item[k], (double)B));
  // CPython's sum() of floats (3.12+, Objects/bltinmodule.c builtin_sum_impl): the int start 0
  // plus the first draw, then Neumaier-compensated additions, the compensation added at the end
  // when it is nonzero and finite
  double f = 0.0, comp = 0.0;
  for (int s = 0; s < a.S; ++s) {
    double d = draw0;
    if (a.noise) d = __dmul_rn(d, a.noise[i * a.S + s]);
    if (a.strag) d = __dmul_rn(d, a.strag[i * a.S + s]);
    if (s == 0) {
      f = __dadd_rn(0.0, d);
      continue;
    }
    const double t = __dadd_rn(f, d);
    if (fabs(f) >= fabs(d)) comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(f, t), d));
    else comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(d, t), f));
    f = t;
  }
  if (comp != 0.0 && isfinite(comp)) f = __dadd_rn(f, comp);
  a.out_lat[i] = __ddiv_rn(f, (double)a.S);
  if (a.out_kind) a.out_kind[i] = k;
  if (a.out_res) a.out_res[i] = R;
  if (a.out_batch) a.out_batch[i] = B;
}

__global__ void k_pow(int n, const double* __restrict__ x, const double* __restrict__ y,
                      double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = cr_pow(x[i], y[i]);
}

template <class T>
int upload(T** dst, const T* src, size_t n, std::vector<void*>& owned) {
  if (n == 0) {
    *dst = nullptr;
    return SP_OK;
  }
  SP_CUDA(cudaMalloc(dst, sizeof(T) * n));
  owned.push_back(*dst);
  SP_CUDA(cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return SP_OK;
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" int sp_profile_configs(sp_ctx* ctx, int32_t K, const int32_t* n_res,
                                  const int32_t* res_opts, const double* base_seconds,
                                  const int32_t* ref_resource, const double* resource_exponent,
                                  const double* batch_exponent, const double* per_item_seconds,
                                  int32_t n_batch, const int32_t* batch_sizes, int32_t n_knobs,
                                  const int32_t* knob_counts, const double* multipliers,
                                  int32_t samples, const double* noise, const double* straggle,
                                  int64_t n_out, double* out_lat, int32_t* out_kind,
                                  int32_t* out_res, int32_t* out_batch) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || K < 1 || !n_res || !base_seconds || !ref_resource || !resource_exponent ||
      !batch_exponent || !per_item_seconds || n_batch < 1 || !batch_sizes || n_knobs < 0 ||
      n_knobs > 16 || (n_knobs > 0 && (!knob_counts || !multipliers)) || samples < 1 || !out_lat)
    return fail(SP_E_INVALID, "profile_configs: bad argument");
  std::vector<int64_t> koff(K + 1, 0);
  std::vector<int32_t> roff(K + 1, 0), moff(n_knobs > 0 ? n_knobs : 1, 0);
  int64_t combos = 1;
  int mrow = 0;
  for (int j = 0; j < n_knobs; ++j) {
    if (knob_counts[j] < 1) return fail(SP_E_INVALID, "profile_configs: a knob without values");
    moff[j] = mrow;
    mrow += knob_counts[j];
    combos *= knob_counts[j];
  }
  for (int k = 0; k < K; ++k) {
    if (n_res[k] < 1) return fail(SP_E_INVALID, "profile_configs: a kind without resource options");
    roff[k + 1] = roff[k] + n_res[k];
    koff[k + 1] = koff[k] + (int64_t)n_res[k] * n_batch * combos;
  }
  const int64_t N = koff[K];
  if (n_out != N) return fail(SP_E_INVALID, "profile_configs: n_out must equal the cross product size");
  std::vector<double> refd(K);
  for (int k = 0; k < K; ++k) refd[k] = (double)ref_resource[k];
  std::vector<void*> owned;
  auto cleanup = [&]() {
    for (void* p : owned) cudaFree(p);
  };
  ProfArgs a;
  int rc = SP_OK;
  double* d_out = nullptr;
  int32_t *d_kind = nullptr, *d_res = nullptr, *d_batch = nullptr;
  do {
    int64_t* dko;
    int32_t *dro, *dropt, *dbat, *dkc = nullptr, *dmo = nullptr;
    double *dbase, *dref, *drexp, *dbexp, *dpi, *dmult = nullptr, *dnoise = nullptr, *dstrag = nullptr;
    if ((rc = upload(&dko, koff.data(), koff.size(), owned)) != SP_OK) break;
    if ((rc = upload(&dro, roff.data(), roff.size(), owned)) != SP_OK) break;
    if ((rc = upload(&dropt, res_opts, (size_t)roff[K], owned)) != SP_OK) break;
    if ((rc = upload(&dbase, base_seconds, (size_t)K, owned)) != SP_OK) break;
    if ((rc = upload(&dref, refd.data(), (size_t)K, owned)) != SP_OK) break;
    if ((rc = upload(&drexp, resource_exponent, (size_t)K, owned)) != SP_OK) break;
    if ((rc = upload(&dbexp, batch_exponent, (size_t)K, owned)) != SP_OK) break;
    if ((rc = upload(&dpi, per_item_seconds, (size_t)K, owned)) != SP_OK) break;
    if ((rc = upload(&dbat, batch_sizes, (size_t)n_batch, owned)) != SP_OK) break;
    if (n_knobs > 0) {
      if ((rc = upload(&dkc, knob_counts, (size_t)n_knobs, owned)) != SP_OK) break;
      if ((rc = upload(&dmo, moff.data(), (size_t)n_knobs, owned)) != SP_OK) break;
      if ((rc = upload(&dmult, multipliers, (size_t)K * mrow, owned)) != SP_OK) break;
    }
    if (noise && (rc = upload(&dnoise, noise, (size_t)N * samples, owned)) != SP_OK) break;
    if (straggle && (rc = upload(&dstrag, straggle, (size_t)N * samples, owned)) != SP_OK) break;
    cudaError_t e = cudaMalloc(&d_out, sizeof(double) * N);
    if (e == cudaSuccess) owned.push_back(d_out);
    if (e == cudaSuccess && out_kind && (e = cudaMalloc(&d_kind, 4 * N)) == cudaSuccess) owned.push_back(d_kind);
    if (e == cudaSuccess && out_res && (e = cudaMalloc(&d_res, 4 * N)) == cudaSuccess) owned.push_back(d_res);
    if (e == cudaSuccess && out_batch && (e = cudaMalloc(&d_batch, 4 * N)) == cudaSuccess) owned.push_back(d_batch);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "cudaMalloc(profile)");
      break;
    }
    a = ProfArgs{K, dko, dro, dropt, dbase, dref, drexp, dbexp, dpi, n_batch, dbat, n_knobs, dkc,
                 dmo, mrow, dmult, combos, samples, dnoise, dstrag, N, d_out, d_kind, d_res,
                 d_batch};
    k_profile<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(a);
    ctx->launches++;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_lat, d_out, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && out_kind) e = cudaMemcpyAsync(out_kind, d_kind, 4 * N, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && out_res) e = cudaMemcpyAsync(out_res, d_res, 4 * N, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && out_batch) e = cudaMemcpyAsync(out_batch, d_batch, 4 * N, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "profile_configs");
  } while (false);
  cleanup();
  return rc;
}

extern "C" int sp_pow_correctly_rounded(sp_ctx* ctx, int32_t n, const double* x, const double* y,
                                        double* out) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || n < 0 || (n > 0 && (!x || !y || !out))) return fail(SP_E_INVALID, "pow: bad argument");
  if (n == 0) return SP_OK;
  std::vector<void*> owned;
  double *dx, *dy, *dz;
  int rc = upload(&dx, x, (size_t)n, owned);
  if (rc == SP_OK) rc = upload(&dy, y, (size_t)n, owned);
  if (rc == SP_OK) {
    cudaError_t e = cudaMalloc(&dz, sizeof(double) * n);
    if (e == cudaSuccess) {
      owned.push_back(dz);
      k_pow<<<(n + 255) / 256, 256, 0, ctx->stream>>>(n, dx, dy, dz);
      ctx->launches++;
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaMemcpyAsync(out, dz, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "pow");
  }
  for (void* p : owned) cudaFree(p);
  return rc;
}
