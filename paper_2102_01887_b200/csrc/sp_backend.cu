// sp_backend.cu — the simulated backend's observation law on the device.
//
// The reference simulator (backend.py:36-58, draw_actual_latency) turns an executed
// configuration into an observed latency: truth.base_latency(assignment) +
// truth.per_item_seconds * items, multiplied by exp(N(0, sigma)).  For replica-parallel
// simulation and the online-mode workload (config 5) the decisions of
// a batch are already on the device; one kernel turns them into the observation records the
// feedback fold consumes: decision i executes iff it is an assignment (delayed and None
// decisions run nothing this batch, manager.py:379-390), with base / per-item truth per table
// entry and the caller's multiplicative noise (the exp of the normal draws, generated on the
// host in the reference's RNG order).  Products and sums in the reference's order, no FMA.
#include "sp_internal.cuh"

namespace sp {
namespace {

__global__ void k_observe(int n, const int32_t* __restrict__ code, const int32_t* __restrict__ idx,
                          const int32_t* __restrict__ fill, const double* __restrict__ base,
                          const double* __restrict__ per_item, const double* __restrict__ noise,
                          int32_t* __restrict__ obs_idx, double* __restrict__ obs) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the decisions are the predecessor's
  asm volatile("griddepcontrol.launch_dependents;");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool run = (code[i] & 3) == SP_DEC_ASSIGN;
  const int e = run ? idx[i] : -1;
  obs_idx[i] = e;
  double v = 0.0;
  if (run) {
    // backend.py:52  truth.base_latency(a) + truth.per_item_seconds * item_count
    double lat = base[e];
    if (per_item) lat = __dadd_rn(lat, __dmul_rn(per_item[e], (double)fill[i]));
    v = __dmul_rn(lat, noise[i]);  // backend.py:54  latency *= exp(N(0, sigma))
  }
  obs[i] = v;
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" int sp_simulate_observations(sp_ctx* ctx, int32_t N, const int32_t* code,
                                        const int32_t* idx, const int32_t* fill,
                                        const double* truth_base, const double* truth_per_item,
                                        const double* noise, int32_t* obs_idx, double* obs) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || N < 0 || (N > 0 && (!code || !idx || !truth_base || !noise || !obs_idx || !obs)))
    return fail(SP_E_INVALID, "simulate_observations: bad argument");
  if (truth_per_item && !fill)
    return fail(SP_E_INVALID, "simulate_observations: fill is required with per-item truth");
  if (N == 0) return SP_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((N + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->opt.no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SP_CUDA(cudaLaunchKernelEx(&cfg, k_observe, N, code, idx, fill, truth_base, truth_per_item,
                             noise, obs_idx, obs));
  SP_CHECK_LAUNCH(ctx);
  return SP_OK;
}

extern "C" int sp_simulate_and_fold(sp_ctx* ctx, sp_table* t, int32_t N, const int32_t* code,
                                    const int32_t* idx, const int32_t* fill,
                                    const double* truth_base, const double* truth_per_item,
                                    const double* noise, double beta, int32_t dfp_count,
                                    int32_t dfp_on, int32_t fb_frozen, int32_t* rec_idx,
                                    double* rec_obs) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || N < 0 || (N > 0 && (!code || !idx || !truth_base || !noise || !rec_idx || !rec_obs)))
    return fail(SP_E_INVALID, "simulate_and_fold: bad argument");
  if (truth_per_item && !fill)
    return fail(SP_E_INVALID, "simulate_and_fold: fill is required with per-item truth");
  if (!(beta > 0.0 && beta <= 1.0)) return fail(SP_E_INVALID, "smoothing_beta must be in (0, 1]");
  return simulate_and_fold(ctx, t, N, code, idx, fill, truth_base, truth_per_item, noise, beta,
                           dfp_count, dfp_on, fb_frozen, rec_idx, rec_obs);
}
