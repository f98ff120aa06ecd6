// sp_des.cu — replica-parallel run engine on the device.
//
// k_des_run: one thread per replica executes the whole tuned run of the reference
// (PipelineRun.run_to_completion, manager.py:535-575) — the event heap, backend pools, the
// Configurator's speculation / commit / feedback decisions — over its own arena in HBM
// (sp_des.cuh).  The run image (a few KB: DAG, fleet, parameters) and, when they fit, the
// static entry columns are staged into shared memory once per CTA; everything a replica mutates
// (its latency tables, invocations, queues, heap) lives in its arena.  Replicas are independent
// (no inter-thread communication), so the grid is simply ceil(R / 64) CTAs of 64 threads.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "sp_des_host.h"
#include "sp_internal.cuh"

struct sp_des {
  spdes::HostImage h;
  double* d_dcols = nullptr;
  int32_t* d_icols = nullptr;
  spdes::Image* d_image = nullptr;
  char* arena = nullptr;
  size_t arena_cap = 0;
  void* tabs = nullptr;  // lat / cost / costpen, the 32 replicas of a warp interleaved
  size_t tabs_cap = 0;
  int32_t prepared_R = 0;
  int32_t mode = 0;  // 0: by run count, 1: one thread per run, 2: `lanes` lanes per run
  int32_t lanes = 32;
  // staged host I/O
  void* io = nullptr;
  size_t io_cap = 0;
};

namespace {

using namespace spdes;

constexpr int kMaxThreads = 128;
constexpr size_t kSmemEntriesMax = 64 * 1024;

__global__ void __launch_bounds__(kMaxThreads)
k_des_run(const Image* __restrict__ g_im, const double* __restrict__ g_d,
          const int32_t* __restrict__ g_i, char* __restrict__ arena, double* __restrict__ tabs, int R,
          const int32_t* __restrict__ frame_off, const int32_t* __restrict__ attrs,
          const int32_t* __restrict__ trace_of,
          const double* __restrict__ targets, const double* __restrict__ dfac,
          const uint8_t* __restrict__ dbits, LogRec* __restrict__ log,
          double* __restrict__ lat_out, Out* __restrict__ out, int entries_in_smem,
          EvRec* __restrict__ ev) {
  static_assert(sizeof(Image) % 16 == 0, "Image is copied in 16-byte words");
  extern __shared__ __align__(16) unsigned char smem[];
  Image& im = *reinterpret_cast<Image*>(smem);
  {
    const int4* src = reinterpret_cast<const int4*>(g_im);
    int4* dst = reinterpret_cast<int4*>(smem);
    for (int i = threadIdx.x; i < (int)(sizeof(Image) / 16); i += blockDim.x) dst[i] = src[i];
  }
  const int N = g_im->n_entries;
  const double* dcol = g_d;
  const int32_t* icol = g_i;
  if (entries_in_smem) {
    double* sd = reinterpret_cast<double*>(smem + sizeof(Image));
    int32_t* si = reinterpret_cast<int32_t*>(sd + 8 * (size_t)N);
    for (int i = threadIdx.x; i < 8 * N; i += blockDim.x) sd[i] = g_d[i];
    const int ni = 4 * N + g_im->suf_off[g_im->n_ops];
    for (int i = threadIdx.x; i < ni; i += blockDim.x) si[i] = g_i[i];
    dcol = sd;
    icol = si;
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const Entries E = entries_view(dcol, icol, N);
  const int tr = trace_of ? trace_of[r] : r;
  const int f0 = frame_off[tr];
  Run run(im, E, arena + (size_t)r * im.arena_bytes, tabs + (size_t)(r >> 5) * (96 * (size_t)N) + (r & 31),
          32, attrs + (int64_t)f0 * im.n_attrs,
          frame_off[tr + 1] - f0, targets[r], dfac ? dfac + (size_t)r * im.draw_cap : nullptr,
          dbits ? dbits + (size_t)r * im.draw_cap : nullptr,
          log ? log + (size_t)r * im.log_cap : nullptr);
  if (ev) run.evlog = ev + (size_t)r * im.ev_cap;
  run.run();
  run.write_out(out[r]);
  if (lat_out)
    for (int i = 0; i < N; ++i) lat_out[(size_t)r * N + i] = run.lat(i);
}

// Warp-per-run form: the 32 lanes of a warp execute one run together — identical serial state in
// every lane, the entry scans of OpTable.select / affinity split across the lanes and reduced by
// shuffles — so the warp never diverges on the engine's control flow; the run's mutable entry
// columns are contiguous in its own arena (the lanes of a scan read consecutive entries).
__global__ void __launch_bounds__(kMaxThreads)
k_des_run_warp(const Image* __restrict__ g_im, const double* __restrict__ g_d,
               const int32_t* __restrict__ g_i, char* __restrict__ arena, int R,
               const int32_t* __restrict__ frame_off, const int32_t* __restrict__ attrs,
               const int32_t* __restrict__ trace_of, const double* __restrict__ targets,
               const double* __restrict__ dfac, const uint8_t* __restrict__ dbits,
               LogRec* __restrict__ log, double* __restrict__ lat_out, Out* __restrict__ out,
               int entries_in_smem, int nl, EvRec* __restrict__ ev) {
  extern __shared__ __align__(16) unsigned char smem[];
  Image& im = *reinterpret_cast<Image*>(smem);
  {
    const int4* src = reinterpret_cast<const int4*>(g_im);
    int4* dst = reinterpret_cast<int4*>(smem);
    for (int i = threadIdx.x; i < (int)(sizeof(Image) / 16); i += blockDim.x) dst[i] = src[i];
  }
  const int N = g_im->n_entries;
  const double* dcol = g_d;
  const int32_t* icol = g_i;
  if (entries_in_smem) {
    double* sd = reinterpret_cast<double*>(smem + sizeof(Image));
    int32_t* si = reinterpret_cast<int32_t*>(sd + 8 * (size_t)N);
    for (int i = threadIdx.x; i < 8 * N; i += blockDim.x) sd[i] = g_d[i];
    const int ni = 4 * N + g_im->suf_off[g_im->n_ops];
    for (int i = threadIdx.x; i < ni; i += blockDim.x) si[i] = g_i[i];
    dcol = sd;
    icol = si;
  }
  __syncthreads();
  const int lb = __ffs(nl) - 1;  // nl: lanes per run (1..32, a power of two)
  const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> lb);
  const int lane = threadIdx.x & (nl - 1);
  if (r >= R) return;  // whole lane groups
  const Entries E = entries_view(dcol, icol, N);
  const int tr = trace_of ? trace_of[r] : r;
  const int f0 = frame_off[tr];
  char* ar = arena + (size_t)r * im.arena_bytes;
  Run run(im, E, ar, reinterpret_cast<double*>(ar + im.o_lat), 1, attrs + (int64_t)f0 * im.n_attrs,
          frame_off[tr + 1] - f0, targets[r], dfac ? dfac + (size_t)r * im.draw_cap : nullptr,
          dbits ? dbits + (size_t)r * im.draw_cap : nullptr,
          log ? log + (size_t)r * im.log_cap : nullptr);
  run.lane = lane;
  run.nl = nl;
  if (ev) run.evlog = ev + (size_t)r * im.ev_cap;
  run.lmask = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u) << ((threadIdx.x & 31) & ~(nl - 1));
  run.run();
  __syncwarp(run.lmask);
  if (lane == 0) run.write_out(out[r]);
  if (lat_out)
    for (int i = lane; i < N; i += nl) lat_out[(size_t)r * N + i] = run.lat(i);
}

template <class T>
int upload_vec(T** dptr, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dptr, sizeof(T) * (v.empty() ? 1 : v.size()));
  if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
  return e == cudaSuccess ? SP_OK : sp::cuda_fail(e, "run engine upload");
}

int grow(void** p, size_t* cap, size_t bytes) {
  if (bytes <= *cap) return SP_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return sp::cuda_fail(e, "run engine arena");
  *cap = bytes;
  return SP_OK;
}

int prepare(sp_ctx* ctx, sp_des* d, int32_t R, int32_t T, const int32_t* frame_off,
            const int32_t* attrs, int32_t draw_cap, int32_t log_cap, int32_t ev_cap = 0) {
  std::string err;
  if (!plan_run(d->h, T, frame_off, attrs, draw_cap, log_cap, err, ev_cap))
    return sp::fail(SP_E_INVALID, err);
  const size_t need = (size_t)d->h.im.arena_bytes * (size_t)R;
  void* a = d->arena;
  int rc = grow(&a, &d->arena_cap, need);
  d->arena = (char*)a;
  if (rc != SP_OK) return rc;
  rc = grow(&d->tabs, &d->tabs_cap, sizeof(double) * 96 * (size_t)d->h.im.n_entries * (size_t)((R + 31) / 32));
  if (rc != SP_OK) return rc;
  cudaError_t e = cudaMemcpyAsync(d->d_image, &d->h.im, sizeof(Image), cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return sp::cuda_fail(e, "run engine image");
  d->prepared_R = R;
  return SP_OK;
}

int launch(sp_ctx* ctx, sp_des* d, int32_t R, const int32_t* frame_off, const int32_t* attrs,
           const int32_t* trace_of, const double* targets, const double* dfac, const uint8_t* dbits, LogRec* log,
           double* lat_out, Out* out, EvRec* ev) {
  const int N = d->h.im.n_entries;
  const size_t ebytes = (size_t)N * (8 * sizeof(double) + 4 * sizeof(int32_t)) +
                        sizeof(int32_t) * (size_t)d->h.im.suf_off[d->h.im.n_ops];
  const int in_smem = ebytes <= kSmemEntriesMax;
  const size_t smem = sizeof(Image) + (in_smem ? ebytes : 0);
  // default lanes per run by the number of runs (measured on AMBER, runs/s at 16k / 65k runs;
  // one run per thread: 1.3k / 4.0k; 2 lanes: 2.8k / 5.3k; 4 lanes: 3.2k / 4.7k; 8 lanes:
  // 3.7k / 3.9k; 16 lanes: 3.1k / 3.4k; 32 lanes: 0.42 s per run, 2.5-2.8k runs/s from 4k runs)
  const int nl = d->mode >= 2 ? d->lanes
                              : (d->mode == 1 ? 0 : (R < 2048 ? 32 : (R < 32768 ? 8 : 2)));
  if (nl) {
    cudaError_t e = cudaFuncSetAttribute(k_des_run_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return sp::cuda_fail(e, "run engine smem");
    if (R > 0) {
      const int per_cta = kMaxThreads / nl;
      k_des_run_warp<<<(R + per_cta - 1) / per_cta, kMaxThreads, smem, ctx->stream>>>(
          d->d_image, d->d_dcols, d->d_icols, d->arena, R, frame_off, attrs, trace_of, targets, dfac,
          dbits, log, lat_out, out, in_smem, nl, ev);
      ctx->launches++;
      e = cudaGetLastError();
      if (e != cudaSuccess) return sp::cuda_fail(e, "k_des_run_warp launch");
    }
    return SP_OK;
  }
  cudaError_t e = cudaFuncSetAttribute(k_des_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return sp::cuda_fail(e, "run engine smem");
  if (R > 0) {
    // one replica per thread; CTAs as wide as the replica count allows while every SM gets work
    const int threads = R >= 128 * ctx->num_sms ? 128 : (R >= 64 * ctx->num_sms ? 64 : 32);
    k_des_run<<<(R + threads - 1) / threads, threads, smem, ctx->stream>>>(
        d->d_image, d->d_dcols, d->d_icols, d->arena, (double*)d->tabs, R, frame_off, attrs, trace_of, targets, dfac, dbits,
        log, lat_out, out, in_smem, ev);
    ctx->launches++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return sp::cuda_fail(e, "k_des_run launch");
  }
  return SP_OK;
}

}  // namespace

extern "C" int sp_des_create(sp_ctx* ctx, const sp_des_spec* spec, sp_des** out) {
  sp::DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !spec || !out) return sp::fail(SP_E_INVALID, "des_create: bad argument");
  *out = nullptr;
  sp_des* d = new sp_des();
  std::string err;
  if (!build_image(*spec, d->h, err)) {
    delete d;
    return sp::fail(SP_E_INVALID, err);
  }
  int rc = upload_vec(&d->d_dcols, d->h.dcols);
  if (rc == SP_OK) rc = upload_vec(&d->d_icols, d->h.icols);
  if (rc == SP_OK) {
    cudaError_t e = cudaMalloc(&d->d_image, sizeof(Image));
    if (e != cudaSuccess) rc = sp::cuda_fail(e, "des_create");
  }
  if (rc != SP_OK) {
    cudaFree(d->d_dcols);
    cudaFree(d->d_icols);
    delete d;
    return rc;
  }
  *out = d;
  return SP_OK;
}

extern "C" int sp_des_destroy(sp_ctx* ctx, sp_des* d) {
  sp::DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!d) return SP_OK;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  cudaFree(d->d_dcols);
  cudaFree(d->d_icols);
  cudaFree(d->d_image);
  cudaFree(d->arena);
  cudaFree(d->tabs);
  cudaFree(d->io);
  delete d;
  return SP_OK;
}

extern "C" int64_t sp_des_arena_bytes(sp_des* d) { return d ? d->h.im.arena_bytes : -1; }

extern "C" int sp_des_prepare(sp_ctx* ctx, sp_des* d, int32_t R, int32_t n_traces,
                              const int32_t* frame_off, const int32_t* attrs, int32_t draw_cap,
                              int32_t log_cap) {
  sp::DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !d || R < 0 || n_traces < 0 || !frame_off ||
      (n_traces > 0 && !attrs && d->h.im.n_attrs > 0) || draw_cap < 0 || log_cap < 0)
    return sp::fail(SP_E_INVALID, "des_prepare: bad argument");
  return prepare(ctx, d, R, n_traces, frame_off, attrs, draw_cap, log_cap);
}

extern "C" int sp_des_set_mode(sp_des* d, int32_t lanes) {
  // 0 default, 1 one thread per run, 2 / 4 / 8 / 16 / 32 lanes per run
  if (!d || !(lanes == 0 || lanes == 1 || lanes == 2 || lanes == 4 || lanes == 8 || lanes == 16 ||
              lanes == 32))
    return sp::fail(SP_E_INVALID, "des_set_mode: 0 (default), 1 (thread per run), 2..32 lanes per run");
  d->mode = lanes <= 1 ? lanes : 2;
  d->lanes = lanes <= 1 ? 32 : lanes;
  return SP_OK;
}

extern "C" int sp_des_set_capacity(sp_des* d, double invocations_per_item) {
  if (!d || !(invocations_per_item >= 1.0) || invocations_per_item > 64.0)
    return sp::fail(SP_E_INVALID, "des_set_capacity: 1 <= invocations_per_item <= 64");
  d->h.cap_scale = invocations_per_item;
  return SP_OK;
}

extern "C" int sp_des_run(sp_ctx* ctx, sp_des* d, int32_t R, int32_t n_traces,
                          const int32_t* frame_off, const int32_t* attrs, const int32_t* trace_of,
                          const double* target_s, int32_t draw_cap,
                          const double* draw_factor, const uint8_t* draw_bits, int32_t log_cap,
                          sp_des_log* log, double* lat_out, sp_des_out* out, int32_t event_cap,
                          sp_des_event* events, int32_t mem) {
  sp::DeviceScope _dev_scope(ctx ? ctx->device : -1);
  static_assert(sizeof(sp_des_out) == sizeof(Out), "sp_des_out layout");
  static_assert(sizeof(sp_des_log) == sizeof(LogRec), "sp_des_log layout");
  static_assert(sizeof(sp_des_event) == sizeof(EvRec), "sp_des_event layout");
  if (event_cap < 0 || (event_cap > 0 && !events)) return sp::fail(SP_E_INVALID, "des_run: bad event buffer");
  if (!ctx || !d || R < 0 || n_traces < 1 || !frame_off || !target_s || !out || draw_cap < 0 ||
      log_cap < 0 || (!trace_of && n_traces != R) ||
      (mem != SP_MEM_HOST && mem != SP_MEM_DEVICE))
    return sp::fail(SP_E_INVALID, "des_run: bad argument");
  const Image& im = d->h.im;
  if (im.draws && (!draw_factor && (im.draws & kDrawNoise)))
    return sp::fail(SP_E_INVALID, "des_run: the scenario draws noise; draw_factor required");
  if (im.draws && !draw_bits && (im.draws & (kDrawStraggle | kDrawFail)))
    return sp::fail(SP_E_INVALID, "des_run: the scenario draws straggles / failures; draw_bits required");
  if (R == 0) return SP_OK;
  if (mem == SP_MEM_DEVICE) {
    if (d->prepared_R < R || im.draw_cap != draw_cap || im.log_cap != log_cap || im.ev_cap != event_cap)
      return sp::fail(SP_E_INVALID, "des_run: device buffers need sp_des_prepare with the same R / caps");
    int rc = launch(ctx, d, R, frame_off, attrs, trace_of, target_s, draw_factor, draw_bits,
                    reinterpret_cast<LogRec*>(log), lat_out, reinterpret_cast<Out*>(out),
                    reinterpret_cast<EvRec*>(events));
    return rc;
  }
  if (trace_of)
    for (int r = 0; r < R; ++r)
      if (trace_of[r] < 0 || trace_of[r] >= n_traces) return sp::fail(SP_E_INVALID, "des_run: bad trace_of");
  int rc = prepare(ctx, d, R, n_traces, frame_off, attrs, draw_cap, log_cap, event_cap);
  if (rc != SP_OK) return rc;
  const int64_t F = frame_off[n_traces];
  const int N = im.n_entries;
  // staged inputs / outputs in one device block
  size_t off = 0;
  auto slot = [&](size_t bytes) {
    const size_t at = off;
    off = (off + bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t s_off = slot(4 * (size_t)(n_traces + 1));
  const size_t s_trace = trace_of ? slot(4 * (size_t)R) : 0;
  const size_t s_attr = slot(4 * (size_t)std::max<int64_t>(F * im.n_attrs, 1));
  const size_t s_tgt = slot(8 * (size_t)R);
  const size_t s_fac = draw_factor ? slot(8 * (size_t)R * draw_cap) : 0;
  const size_t s_bits = draw_bits ? slot((size_t)R * draw_cap) : 0;
  const size_t s_log = log ? slot(sizeof(LogRec) * (size_t)R * log_cap) : 0;
  const size_t s_lat = lat_out ? slot(8 * (size_t)R * N) : 0;
  const size_t s_ev = events ? slot(sizeof(EvRec) * (size_t)R * event_cap) : 0;
  const size_t s_out = slot(sizeof(Out) * (size_t)R);
  rc = grow(&d->io, &d->io_cap, off);
  if (rc != SP_OK) return rc;
  char* io = (char*)d->io;
  cudaStream_t st = ctx->stream;
  cudaError_t e = cudaMemcpyAsync(io + s_off, frame_off, 4 * (size_t)(n_traces + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && trace_of)
    e = cudaMemcpyAsync(io + s_trace, trace_of, 4 * (size_t)R, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && F * im.n_attrs > 0)
    e = cudaMemcpyAsync(io + s_attr, attrs, 4 * (size_t)(F * im.n_attrs), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(io + s_tgt, target_s, 8 * (size_t)R, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && draw_factor)
    e = cudaMemcpyAsync(io + s_fac, draw_factor, 8 * (size_t)R * draw_cap, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && draw_bits)
    e = cudaMemcpyAsync(io + s_bits, draw_bits, (size_t)R * draw_cap, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return sp::cuda_fail(e, "des_run inputs");
  rc = launch(ctx, d, R, (const int32_t*)(io + s_off), (const int32_t*)(io + s_attr),
              trace_of ? (const int32_t*)(io + s_trace) : nullptr, (const double*)(io + s_tgt), draw_factor ? (const double*)(io + s_fac) : nullptr,
              draw_bits ? (const uint8_t*)(io + s_bits) : nullptr,
              log ? (LogRec*)(io + s_log) : nullptr, lat_out ? (double*)(io + s_lat) : nullptr,
              (Out*)(io + s_out), events ? (EvRec*)(io + s_ev) : nullptr);
  if (rc != SP_OK) return rc;
  e = cudaMemcpyAsync(out, io + s_out, sizeof(Out) * (size_t)R, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && log)
    e = cudaMemcpyAsync(log, io + s_log, sizeof(LogRec) * (size_t)R * log_cap, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && lat_out)
    e = cudaMemcpyAsync(lat_out, io + s_lat, 8 * (size_t)R * N, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && events)
    e = cudaMemcpyAsync(events, io + s_ev, sizeof(EvRec) * (size_t)R * event_cap, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return sp::cuda_fail(e, "des_run");
  return SP_OK;
}
