// sp_api.cu — C-ABI of libslackpipe_b200.so (declared in include/slackpipe_b200.h).
//
// Host-side responsibilities only: validation (mirroring the reference's ValueErrors),
// device allocation, host<->device staging for SP_MEM_HOST calls, and launching the
// kernels of sp_plan.cu / sp_select.cu / sp_slack.cu / sp_fold.cu.  No decision, score or
// slack is ever computed on the host.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "sp_internal.cuh"

namespace sp {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return SP_E_CUDA;
}

void* ctx_tmp(sp_ctx* ctx, size_t bytes, int* rc) {
  if (bytes <= ctx->tmp_cap) return ctx->tmp_dev;
  if (ctx->tmp_dev) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->tmp_dev);
    ctx->tmp_dev = nullptr;
    ctx->tmp_cap = 0;
  }
  size_t cap = std::max(bytes, (size_t)1 << 20);
  cudaError_t e = cudaMalloc(&ctx->tmp_dev, cap);
  if (e != cudaSuccess) {
    if (rc) *rc = cuda_fail(e, "cudaMalloc(tmp)");
    ctx->tmp_dev = nullptr;
    return nullptr;
  }
  ctx->tmp_cap = cap;
  return ctx->tmp_dev;
}

static void* ctx_io(sp_ctx* ctx, size_t bytes, int* rc) {
  if (bytes <= ctx->io_cap) return ctx->io_dev;
  if (ctx->io_dev) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->io_dev);
    ctx->io_dev = nullptr;
    ctx->io_cap = 0;
  }
  size_t cap = std::max(bytes, (size_t)4 << 20);
  cudaError_t e = cudaMalloc(&ctx->io_dev, cap);
  if (e != cudaSuccess) {
    *rc = cuda_fail(e, "cudaMalloc(io)");
    return nullptr;
  }
  ctx->io_cap = cap;
  return ctx->io_dev;
}

static void* ctx_pin(sp_ctx* ctx, size_t bytes, void** dev, int* rc) {
  if (bytes > ctx->pin_cap) {
    if (ctx->pin_host) {
      cudaStreamSynchronize(ctx->stream);
      cudaFreeHost(ctx->pin_host);
      ctx->pin_host = ctx->pin_dev = nullptr;
      ctx->pin_cap = 0;
    }
    size_t cap = std::max(bytes, (size_t)64 << 10);
    cudaError_t e = cudaHostAlloc(&ctx->pin_host, cap, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ctx->pin_dev, ctx->pin_host, 0);
    if (e != cudaSuccess) {
      *rc = cuda_fail(e, "cudaHostAlloc(staging)");
      ctx->pin_host = ctx->pin_dev = nullptr;
      return nullptr;
    }
    ctx->pin_cap = cap;
  }
  *dev = ctx->pin_dev;
  return ctx->pin_host;
}

// Simple bump allocator over the I/O arena.
struct Bump {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base + off);
    off += (n * sizeof(T) + 255) & ~(size_t)255;
    return p;
  }
};
template <typename T>
static size_t rsz(size_t n) {
  return (n * sizeof(T) + 255) & ~(size_t)255;
}

// Device address of a pinned, mapped host range [h, h + bytes), or false (pageable memory,
// or a range that leaves the registered allocation).
static bool mapped_host(const void* h, size_t bytes, void** dev) {
  if (!h || bytes == 0) return false;
  cudaPointerAttributes a0, a1;
  if (cudaPointerGetAttributes(&a0, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const void* last = static_cast<const uint8_t*>(h) + bytes - 1;
  if (cudaPointerGetAttributes(&a1, last) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a0.type != cudaMemoryTypeHost || a1.type != cudaMemoryTypeHost || !a0.devicePointer ||
      !a1.devicePointer)
    return false;
  if (static_cast<uint8_t*>(a1.devicePointer) - static_cast<uint8_t*>(a0.devicePointer) !=
      (ptrdiff_t)(bytes - 1))
    return false;
  *dev = a0.devicePointer;
  return true;
}

__global__ void k_scatter(int m, const int32_t* __restrict__ idx, const double* __restrict__ val,
                          double* __restrict__ dst, uint8_t* __restrict__ dirty) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) {
    dst[idx[i]] = val[i];
    dirty[idx[i]] = 1;
  }
}

static void free_table(sp_table* t) {
  double* dd[] = {t->lat, t->lat_init, t->res, t->pool, t->price, t->thrscratch};
  for (double* p : dd) cudaFree(p);
  int32_t* ii[] = {t->batch, t->bidx, t->kind, t->id_rank, t->obs_count, t->kind_slot,
                   t->ent_r1, t->ent_r2, t->order, t->rows_per_kind, t->dev_counters};
  for (int32_t* p : ii) cudaFree(p);
  cudaFree(t->ukey);
  cudaFree(t->uent);
  uint32_t* uu[] = {t->ukr, t->umap, t->r1, t->r2, t->pf, t->sf, t->rowscratch,
                    t->candf, t->cands, t->cidf, t->cids};
  for (uint32_t* p : uu) cudaFree(p);
  cudaFree(t->sort_tmp);
  cudaFree(t->fin_chunk);
  cudaFree(t->pos_r12);
  cudaFree(t->pos_meta);
  cudaFree(t->pos_lat);
  cudaFree(t->pc_seg);
  cudaFree(t->pc_seg_ent);
  cudaFree(t->pc_scratch);
  for (int q = 0; q < 3; ++q) {
    cudaFree(t->pc_multi_scratch[q]);
    cudaFree(t->pc_multi_thr[q]);
  }
  cudaFree(t->pc_multi_status);
  cudaFree(t->pc_multi_ord);
  cudaFree(t->dirty);
  for (auto& p : t->plans) plan_release(p);
  delete t;
}

static int env_int(const char* name, int def) {
  const char* e = getenv(name);
  return e ? atoi(e) : def;
}

void options_from_env(Options& o) {
  o.zero_copy = env_int("SP_ZERO_COPY", 1);
  o.pipe_chunks = env_int("SP_PIPE_CHUNKS", 0);
  if (const char* e = getenv("SP_K1_CERT")) o.k1_cert = !strcmp(e, "force") ? 2 : (!strcmp(e, "0") ? 1 : 0);
  o.fold_long_min = env_int("SP_FOLD_LONG_MIN", 0);
  o.k1c_lanes = env_int("SP_K1C_LANES", 4) == 2 ? 2 : 4;
  o.fold_legacy = getenv("SP_FOLD_LEGACY") != nullptr;
  o.stair_smem = getenv("SP_STAIR_SMEM") != nullptr;
  o.stair_global = getenv("SP_STAIR_GLOBAL") != nullptr;
  o.no_plan_graph = getenv("SP_NO_PLAN_GRAPH") != nullptr;
  o.plan_legacy = getenv("SP_PLAN_LEGACY") != nullptr;
  o.pc_debug = getenv("SP_PC_DEBUG") ? std::max(1, env_int("SP_PC_DEBUG", 1)) : 0;
  if (const char* e = getenv("SP_K2_VARIANT")) o.k2_plan_only = strcmp(e, "fast") != 0;
  o.k2f_threads = env_int("SP_K2F_THREADS", 512) == 1024 ? 1024 : 512;
  o.no_pdl = getenv("SP_NO_PDL") != nullptr;
  o.full_smem = getenv("SP_FULL_SMEM") != nullptr;
  o.no_k12 = getenv("SP_NO_K12") != nullptr;
  o.k12_generic = getenv("SP_K12_GENERIC") != nullptr;
  o.k12_outstage = getenv("SP_K12_OUTSTAGE") != nullptr;
  o.k12_generic_dp = getenv("SP_K12_GENERIC_DP") != nullptr;
}

int options_set(Options& o, const char* name, long long v) {
  struct {
    const char* n;
    int* f;
  } tab[] = {{"SP_ZERO_COPY", &o.zero_copy},     {"SP_PIPE_CHUNKS", &o.pipe_chunks},
             {"SP_K1_CERT", &o.k1_cert},         {"SP_K1C_LANES", &o.k1c_lanes},         {"SP_FOLD_LONG_MIN", &o.fold_long_min},
             {"SP_FOLD_LEGACY", &o.fold_legacy},
             {"SP_STAIR_SMEM", &o.stair_smem},   {"SP_STAIR_GLOBAL", &o.stair_global},
             {"SP_NO_PLAN_GRAPH", &o.no_plan_graph}, {"SP_PLAN_LEGACY", &o.plan_legacy},
             {"SP_PC_DEBUG", &o.pc_debug},       {"SP_K2_VARIANT", &o.k2_plan_only},
             {"SP_K2F_THREADS", &o.k2f_threads}, {"SP_NO_PDL", &o.no_pdl},
             {"SP_FULL_SMEM", &o.full_smem},     {"SP_NO_K12", &o.no_k12},
             {"SP_K12_GENERIC", &o.k12_generic}, {"SP_K12_OUTSTAGE", &o.k12_outstage},
             {"SP_K12_GENERIC_DP", &o.k12_generic_dp}};
  for (auto& x : tab)
    if (!strcmp(x.n, name)) {
      *x.f = (int)v;
      return SP_OK;
    }
  return fail(SP_E_INVALID, std::string("set_option: unknown option ") + name);
}

}  // namespace sp

using namespace sp;

extern "C" {

int sp_version(void) { return 10000; }

const char* sp_last_error(const sp_ctx*) { return g_last_error.c_str(); }

int sp_ctx_create(int device, sp_ctx** out) {
  if (!out) return fail(SP_E_INVALID, "ctx_create: null out");
  int n = 0;
  SP_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(SP_E_INVALID, "ctx_create: bad device ordinal");
  DeviceScope _dev_scope(device);
  cudaDeviceProp prop;
  SP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(SP_E_UNSUPPORTED, "ctx_create: this library is built for sm_100a (B200) only");
  sp_ctx* c = new (std::nothrow) sp_ctx();
  if (!c) return fail(SP_E_NOMEM, "ctx_create: host allocation");
  c->device = device;
  options_from_env(c->opt);
  c->num_sms = prop.multiProcessorCount;
  c->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  c->own_stream = true;
  *out = c;
  return SP_OK;
}

int sp_ctx_destroy(sp_ctx* ctx) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (ctx && ctx->capture) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->capture);
    ctx->capture = nullptr;
  }
  if (!ctx) return SP_OK;
  cudaStreamSynchronize(ctx->stream);
  coop_release(ctx);
  cudaFree(ctx->io_dev);
  cudaFree(ctx->ptr_dev);
  cudaFree(ctx->tmp_dev);
  if (ctx->pin_host) cudaFreeHost(ctx->pin_host);
  if (ctx->h2d) {
    cudaStreamSynchronize(ctx->h2d);
    cudaStreamSynchronize(ctx->d2h);
    cudaStreamDestroy(ctx->h2d);
    cudaStreamDestroy(ctx->d2h);
    for (int c = 0; c < sp_ctx::kPipeChunks; ++c) {
      cudaEventDestroy(ctx->ev_in[c]);
      cudaEventDestroy(ctx->ev_comp[c]);
      cudaEventDestroy(ctx->ev_out[c]);
    }
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return SP_OK;
}

int sp_ctx_set_stream(sp_ctx* ctx, void* stream) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx) return fail(SP_E_INVALID, "null ctx");
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = (cudaStream_t)stream;
  ctx->plan_dirty = true;
  ctx->own_stream = false;
  return SP_OK;
}

int sp_ctx_set_option(sp_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return fail(SP_E_INVALID, "set_option: null argument");
  return options_set(ctx->opt, name, (long long)value);
}

int sp_ctx_synchronize(sp_ctx* ctx) {
  if (!ctx) return fail(SP_E_INVALID, "null ctx");
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  return SP_OK;
}

int64_t sp_ctx_launch_count(const sp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sp_table_create(sp_ctx* ctx, int32_t M, const double* lat, const double* lat_init,
                    const double* res, const int32_t* batch, const double* pool,
                    const double* price, const int32_t* kind, const int32_t* id_rank,
                    int32_t K, int32_t ref_index, sp_table** out) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !out) return fail(SP_E_INVALID, "table_create: null argument");
  // configurator.py:178-179
  if (M < 1) return fail(SP_E_INVALID, "operation has no schedulable configuration");
  if (K < 1 || K > kMaxTableKinds)
    return fail(SP_E_UNSUPPORTED, "table_create: 1..24 backend kinds supported");
  if (ref_index < -1 || ref_index >= M) return fail(SP_E_INVALID, "table_create: bad ref_index");
  std::vector<int32_t> bv;
  for (int j = 0; j < M; ++j) {
    if (kind[j] < 0 || kind[j] >= K) return fail(SP_E_INVALID, "table_create: kind out of range");
    if (batch[j] < 1) return fail(SP_E_INVALID, "table_create: batch size must be >= 1");
    bv.push_back(batch[j]);
  }
  std::sort(bv.begin(), bv.end());
  bv.erase(std::unique(bv.begin(), bv.end()), bv.end());
  sp_table* t = new (std::nothrow) sp_table();
  if (!t) return fail(SP_E_NOMEM, "table_create: host allocation");
  t->M = M;
  t->K = K;
  t->ref_index = ref_index;
  t->nB = (int)bv.size();
  t->nonfinite_entry.assign(M, 0);
  for (int j = 0; j < M; ++j) {
    t->nonfinite_entry[j] = !isfinite(lat[j]);
    t->nonfinite += t->nonfinite_entry[j];
  }
  // unified candidate ids are u16: at most 2M - 1 < 65535 candidates; the plan header describes
  // at most 8 kinds
  t->plan_ok = t->nB <= kMaxB && M < 32767 && K <= kMaxKinds;
  for (int b = 0; b < kMaxB; ++b) t->batch_vals[b] = b < t->nB ? bv[b] : INT32_MAX;
  std::vector<int32_t> bidx(M), kslot(M);
  for (int j = 0; j < M; ++j)
    bidx[j] = (int32_t)(std::lower_bound(bv.begin(), bv.end(), batch[j]) - bv.begin());
  int cnt[kMaxTableKinds] = {0};
  for (int j = 0; j < M; ++j) kslot[j] = cnt[kind[j]]++;
  int base = 0;
  for (int k = 0; k < kMaxTableKinds; ++k) {
    t->kind_count[k] = k < K ? cnt[k] : 0;
    t->kind_base[k] = base;
    if (k < K) base += cnt[k];
  }
  cudaStream_t st = ctx->stream;
  int rc = SP_OK;
#define ALLOC_COPY(field, src, T)                                                  \
  do {                                                                             \
    cudaError_t _e = cudaMalloc(&t->field, sizeof(T) * M);                         \
    if (_e == cudaSuccess && (src))                                                \
      _e = cudaMemcpyAsync(t->field, (src), sizeof(T) * M, cudaMemcpyHostToDevice, st); \
    if (_e != cudaSuccess) {                                                       \
      rc = cuda_fail(_e, "table_create(" #field ")");                              \
      free_table(t);                                                               \
      return rc;                                                                   \
    }                                                                              \
  } while (0)
  ALLOC_COPY(lat, lat, double);
  ALLOC_COPY(lat_init, lat_init ? lat_init : lat, double);
  ALLOC_COPY(res, res, double);
  ALLOC_COPY(pool, pool, double);
  ALLOC_COPY(price, price, double);
  ALLOC_COPY(batch, batch, int32_t);
  ALLOC_COPY(bidx, bidx.data(), int32_t);
  ALLOC_COPY(kind, kind, int32_t);
  ALLOC_COPY(id_rank, id_rank, int32_t);
  ALLOC_COPY(kind_slot, kslot.data(), int32_t);
  ALLOC_COPY(obs_count, (const int32_t*)nullptr, int32_t);
#undef ALLOC_COPY
  cudaError_t e = cudaMemsetAsync(t->obs_count, 0, sizeof(int32_t) * M, st);
  if (e == cudaSuccess) e = cudaMalloc(&t->dev_counters, sizeof(int32_t) * 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->dev_counters, 0, sizeof(int32_t) * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->dev_counters + 4, 1, 1, st);  // order stale
  if (e == cudaSuccess) e = cudaMalloc(&t->dirty, (size_t)M);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->dirty, 0, (size_t)M, st);
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "table_create(counters)");
    free_table(t);
    return rc;
  }
  rc = plan_scratch_alloc(t);
  if (rc == SP_OK) rc = plan_cluster_prepare(t, kind, bidx.data());
  if (rc != SP_OK) {
    free_table(t);
    return rc;
  }
  // host arrays may be released by the caller once we return
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "table_create(sync)");
    free_table(t);
    return rc;
  }
  *out = t;
  return SP_OK;
}

int sp_table_destroy(sp_ctx* ctx, sp_table* t) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!t) return SP_OK;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  free_table(t);
  return SP_OK;
}

int sp_table_set_latency(sp_ctx* ctx, sp_table* t, int32_t n, const int32_t* idx,
                         const double* val) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || n < 0 || (n > 0 && (!idx || !val)))
    return fail(SP_E_INVALID, "set_latency: bad argument");
  // Repeated OpTable.set_latency calls: the last write to an index wins.
  std::map<int32_t, double> last;
  for (int i = 0; i < n; ++i) {
    if (idx[i] < 0 || idx[i] >= t->M) return fail(SP_E_INVALID, "set_latency: index out of range");
    last[idx[i]] = val[i];  // any float, as configurator.py:211-213
  }
  for (auto& kv : last) {  // non-finite entries switch decisions to the literal scan
    const uint8_t nf = !isfinite(kv.second);
    t->nonfinite += (int)nf - (int)t->nonfinite_entry[kv.first];
    t->nonfinite_entry[kv.first] = nf;
  }
  if (last.empty()) return SP_OK;
  std::vector<int32_t> ui;
  std::vector<double> uv;
  for (auto& kv : last) {
    ui.push_back(kv.first);
    uv.push_back(kv.second);
  }
  const int m = (int)ui.size();
  int rc = SP_OK;
  // the updates travel in the pinned staging block (read by the scatter kernel over PCIe)
  void* dbase = nullptr;
  uint8_t* hb = static_cast<uint8_t*>(ctx_pin(ctx, rsz<int32_t>(m) + rsz<double>(m), &dbase, &rc));
  if (!hb) return rc;
  memcpy(hb, ui.data(), sizeof(int32_t) * m);
  memcpy(hb + rsz<int32_t>(m), uv.data(), sizeof(double) * m);
  const int32_t* d_i = reinterpret_cast<const int32_t*>(dbase);
  const double* d_v = reinterpret_cast<const double*>(static_cast<uint8_t*>(dbase) + rsz<int32_t>(m));
  k_scatter<<<(m + 255) / 256, 256, 0, ctx->stream>>>(m, d_i, d_v, t->lat, t->dirty);
  SP_CHECK_LAUNCH(ctx);
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  t->version++;
  return SP_OK;
}

int sp_table_get_latency(sp_ctx* ctx, sp_table* t, double* out_lat) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || !out_lat) return fail(SP_E_INVALID, "get_latency: null argument");
  SP_CUDA(cudaMemcpyAsync(out_lat, t->lat, sizeof(double) * t->M, cudaMemcpyDeviceToHost,
                          ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  return SP_OK;
}

int sp_table_invalidate(sp_ctx* ctx, sp_table* t) {
  if (!ctx || !t) return fail(SP_E_INVALID, "invalidate: null argument");
  DeviceScope _dev_scope(ctx->device);
  t->version++;  // every plan of the table is rebuilt by its next use
  // the latencies may have been written behind the library's back: full re-sort
  SP_CUDA(cudaMemsetAsync(t->dev_counters + 4, 1, 1, ctx->stream));
  return SP_OK;
}

int sp_table_prepare(sp_ctx* ctx, sp_table* t, double alpha) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t) return fail(SP_E_INVALID, "prepare: null argument");
  int rc;
  // the staircase only where it applies; otherwise the scan's cost / costpen
  Plan* p = t->plan_ok && t->finite_safe() && isfinite(alpha) ? plan_get(ctx, t, alpha, &rc)
                                                              : plan_costs(ctx, t, alpha, &rc);
  return p ? SP_OK : rc;
}

int sp_table_prepare_many(sp_ctx* ctx, sp_table* t, int32_t n, const double* alphas) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || n < 0 || (n > 0 && !alphas)) return fail(SP_E_INVALID, "prepare_many: bad argument");
  return plan_prepare_many(ctx, t, n, alphas);
}

int sp_table_plan_supported(const sp_table* t) { return t && t->plan_ok ? 1 : 0; }

int sp_table_plan_bytes(sp_ctx* ctx, sp_table* t, double alpha, int64_t* out_bytes) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || !out_bytes) return fail(SP_E_INVALID, "plan_bytes: null argument");
  int rc;
  Plan* p = plan_get(ctx, t, alpha, &rc);
  if (!p) return rc;
  if (!t->plan_ok) {
    *out_bytes = 0;
    return SP_OK;
  }
  PlanHdr h;
  SP_CUDA(cudaMemcpyAsync(&h, p->image, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h.magic != kPlanMagic) return fail(SP_E_RUNTIME, "plan_bytes: plan image corrupt");
  if (h.total_bytes > p->image_cap) return fail(SP_E_RUNTIME, "plan_bytes: plan overflow");
  *out_bytes = h.total_bytes;
  return SP_OK;
}

int sp_table_plan_image(sp_ctx* ctx, sp_table* t, double alpha, int32_t builder, void* out,
                        int64_t cap, int64_t* out_bytes) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || !out_bytes || builder < 0 || builder > 3)
    return fail(SP_E_INVALID, "plan_image: bad argument");
  if (!t->plan_ok) return fail(SP_E_UNSUPPORTED, "plan_image: the table has no staircase plan");
  if (builder == 2 && !t->pc_ok)
    return fail(SP_E_UNSUPPORTED, "plan_image: the table's shape is outside the cluster builder");
  const int saved = ctx->opt.plan_legacy;
  if (builder == 1 || builder == 2) ctx->opt.plan_legacy = builder == 1;
  if (builder != 3)  // force a fresh build with the requested builder (3: the current plan)
    for (auto& p : t->plans)
      if (p.alpha == alpha || (p.alpha != p.alpha && alpha != alpha)) p.valid = false;
  int rc = SP_OK;
  Plan* p = nullptr;
  for (auto& q : t->plans)
    if (q.alpha == alpha || (q.alpha != q.alpha && alpha != alpha)) p = &q;
  if (p && p->graph && builder != 3) {  // a captured graph replays one builder only
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
    p->builds = 0;
  }
  p = plan_get(ctx, t, alpha, &rc);
  ctx->opt.plan_legacy = saved;
  if (!p) return rc;
  PlanHdr h;
  SP_CUDA(cudaMemcpyAsync(&h, p->image, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h.magic != kPlanMagic) return fail(SP_E_RUNTIME, "plan_image: plan image invalid");
  *out_bytes = h.total_bytes;
  if (out && cap >= h.total_bytes) {
    SP_CUDA(cudaMemcpyAsync(out, p->image, h.total_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  // the next select rebuilds with the context's own builder
  p->valid = false;
  if (p->graph) {
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
    p->builds = 0;
  }
  return SP_OK;
}

int sp_scores(sp_ctx* ctx, sp_table* t, const double* slack_by_kind, double alpha,
              double* out_score, double* out_cost) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t || !slack_by_kind || !out_score || !out_cost)
    return fail(SP_E_INVALID, "scores: null argument");
  int rc;
  Plan* p = plan_costs(ctx, t, alpha, &rc);
  if (!p) return rc;
  size_t need = rsz<double>(t->K) + 2 * rsz<double>(t->M);
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  double* d_slack = b.take<double>(t->K);
  double* d_score = b.take<double>(t->M);
  double* d_cost = b.take<double>(t->M);
  SP_CUDA(cudaMemcpyAsync(d_slack, slack_by_kind, sizeof(double) * t->K, cudaMemcpyHostToDevice,
                          ctx->stream));
  rc = scores_launch(ctx, t, p, d_slack, d_score, d_cost);
  if (rc != SP_OK) return rc;
  SP_CUDA(cudaMemcpyAsync(out_score, d_score, sizeof(double) * t->M, cudaMemcpyDeviceToHost,
                          ctx->stream));
  SP_CUDA(cudaMemcpyAsync(out_cost, d_cost, sizeof(double) * t->M, cudaMemcpyDeviceToHost,
                          ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  return SP_OK;
}

}  // extern "C"

namespace sp {
constexpr int kSmallHostN = 256;  // host calls up to this size go through the pinned staging block
// sp_select_batch without the final synchronisation when sync == false (host I/O is then
// complete only after select_host_wait): lets sp_group_select_batch run every member
// device's shard concurrently from one host thread.
int select_batch_impl(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                      int32_t N, const int32_t* op, const double* slack, const int32_t* avail,
                      const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                      int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                      double* out_slack, double* out_wait, double* out_kind_min, int32_t mode,
                      int32_t mem, bool sync) {
  if (!ctx || !tables || n_tables < 1) return fail(SP_E_INVALID, "select: null argument");
  if (N < 0) return fail(SP_E_INVALID, "select: negative N");
  if (N > 0 && (!slack || !avail || !supply || !min_batch || !flags || !out_idx || !out_code))
    return fail(SP_E_INVALID, "select: required array is null");
  if (!(alpha >= 0.0)) return fail(SP_E_INVALID, "alpha must be >= 0");  // configurator.py:37
  for (int t = 0; t < n_tables; ++t)
    if (!tables[t]) return fail(SP_E_INVALID, "select: null table");
  const int K = tables[0]->K;
  if (mem == SP_MEM_DEVICE) {
    return select_launch(ctx, n_tables, tables, alpha, N, op, slack, avail, supply, min_batch,
                         flags, out_idx, out_code, out_fill, out_obj, out_slack, out_wait,
                         out_kind_min, mode);
  }
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "select: bad mem flag");
  if (op) {
    for (int i = 0; i < N; ++i)
      if (op[i] < 0 || op[i] >= n_tables) return fail(SP_E_INVALID, "select: op out of range");
  }
  // Zero-copy: when every caller buffer is pinned, mapped host memory, the decision kernel
  // reads its inputs and writes its outputs over PCIe itself — one launch, both link
  // directions busy at once, no copy-engine operations.
  {
    const bool want = ctx->opt.zero_copy != 0;
    struct Buf {
      const void* h;
      size_t bytes;
      void* d;
    } bufs[] = {{slack, sizeof(double) * N * K, nullptr},  {avail, 4u * N, nullptr},
                {supply, 4u * N, nullptr},                  {min_batch, 4u * N, nullptr},
                {flags, 4u * N, nullptr},                   {op, 4u * N, nullptr},
                {out_idx, 4u * N, nullptr},                 {out_code, 4u * N, nullptr},
                {out_fill, 4u * N, nullptr},                {out_obj, 8u * N, nullptr},
                {out_slack, 8u * N, nullptr},               {out_wait, 8u * N, nullptr},
                {out_kind_min, sizeof(double) * N * K, nullptr}};
    bool ok = want && N > 0;
    for (auto& bf : bufs) {
      if (!ok) break;
      if (!bf.h) continue;
      ok = mapped_host(bf.h, bf.bytes, &bf.d);
    }
    if (ok) {
      int rc = select_launch(ctx, n_tables, tables, alpha, N, (const int32_t*)bufs[5].d,
                             (const double*)bufs[0].d, (const int32_t*)bufs[1].d,
                             (const int32_t*)bufs[2].d, (const int32_t*)bufs[3].d,
                             (const uint32_t*)bufs[4].d, (int32_t*)bufs[6].d, (int32_t*)bufs[7].d,
                             (int32_t*)bufs[8].d, (double*)bufs[9].d, (double*)bufs[10].d,
                             (double*)bufs[11].d, (double*)bufs[12].d, mode);
      if (rc != SP_OK) return rc;
      if (sync) SP_CUDA(cudaStreamSynchronize(ctx->stream));
      return SP_OK;
    }
  }
  size_t need = rsz<double>((size_t)N * K) + 4 * rsz<int32_t>(N) + (op ? rsz<int32_t>(N) : 0) +
                3 * rsz<int32_t>(N) + 3 * rsz<double>(N) +
                (out_kind_min ? rsz<double>((size_t)N * K) : 0);
  int rc = SP_OK;
  if (N <= kSmallHostN) {
    // small calls (the reference engine's one-invocation OpTable.select): inputs copied into a
    // pinned mapped staging block, one launch reads and writes it over PCIe, one sync
    void* dbase = nullptr;
    uint8_t* hb = static_cast<uint8_t*>(ctx_pin(ctx, need, &dbase, &rc));
    if (!hb) return rc;
    uint8_t* db = static_cast<uint8_t*>(dbase);
    size_t o = 0;
    auto put = [&](const void* src, size_t bytes) -> size_t {
      const size_t at = o;
      if (src) memcpy(hb + at, src, bytes);
      o += (bytes + 255) & ~(size_t)255;
      return at;
    };
    const size_t o_sl = put(slack, sizeof(double) * N * K), o_av = put(avail, 4u * N),
                 o_su = put(supply, 4u * N), o_mb = put(min_batch, 4u * N), o_fl = put(flags, 4u * N),
                 o_op = op ? put(op, 4u * N) : 0, o_ix = put(nullptr, 4u * N), o_cd = put(nullptr, 4u * N),
                 o_fi = put(nullptr, 4u * N), o_ob = put(nullptr, 8u * N), o_sk = put(nullptr, 8u * N),
                 o_wt = put(nullptr, 8u * N), o_km = out_kind_min ? put(nullptr, sizeof(double) * N * K) : 0;
    rc = select_launch(ctx, n_tables, tables, alpha, N, op ? (const int32_t*)(db + o_op) : nullptr,
                       (const double*)(db + o_sl), (const int32_t*)(db + o_av),
                       (const int32_t*)(db + o_su), (const int32_t*)(db + o_mb),
                       (const uint32_t*)(db + o_fl), (int32_t*)(db + o_ix), (int32_t*)(db + o_cd),
                       (int32_t*)(db + o_fi), (double*)(db + o_ob), (double*)(db + o_sk),
                       (double*)(db + o_wt), out_kind_min ? (double*)(db + o_km) : nullptr, mode);
    if (rc != SP_OK) return rc;
    SP_CUDA(cudaStreamSynchronize(ctx->stream));
    memcpy(out_idx, hb + o_ix, 4u * N);
    memcpy(out_code, hb + o_cd, 4u * N);
    if (out_fill) memcpy(out_fill, hb + o_fi, 4u * N);
    if (out_obj) memcpy(out_obj, hb + o_ob, 8u * N);
    if (out_slack) memcpy(out_slack, hb + o_sk, 8u * N);
    if (out_wait) memcpy(out_wait, hb + o_wt, 8u * N);
    if (out_kind_min) memcpy(out_kind_min, hb + o_km, sizeof(double) * N * K);
    return SP_OK;
  }
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  double* d_slack = b.take<double>((size_t)N * K);
  int32_t* d_avail = b.take<int32_t>(N);
  int32_t* d_supply = b.take<int32_t>(N);
  int32_t* d_minb = b.take<int32_t>(N);
  uint32_t* d_flags = b.take<uint32_t>(N);
  int32_t* d_op = op ? b.take<int32_t>(N) : nullptr;
  int32_t* d_idx = b.take<int32_t>(N);
  int32_t* d_code = b.take<int32_t>(N);
  int32_t* d_fill = b.take<int32_t>(N);
  double* d_obj = b.take<double>(N);
  double* d_sl = b.take<double>(N);
  double* d_wait = b.take<double>(N);
  double* d_kmin = out_kind_min ? b.take<double>((size_t)N * K) : nullptr;
  // Pipeline over chunks: H2D of chunk c+1 and D2H of chunk c-1 (separate copy streams, both
  // PCIe directions at once) overlap the decision kernel of chunk c.
  constexpr int kChunkMin = 1 << 18;  // 4 chunks for 2^20 invocations (measured best on B200)
  int nchunk = N >= 2 * kChunkMin
                   ? std::min(sp_ctx::kPipeChunks, (N + kChunkMin - 1) / kChunkMin)
                   : 1;
  if (ctx->opt.pipe_chunks > 0) nchunk = std::min(sp_ctx::kPipeChunks, ctx->opt.pipe_chunks);
  if (nchunk > 1 && !ctx->h2d) {
    SP_CUDA(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    for (int c = 0; c < sp_ctx::kPipeChunks; ++c) {
      SP_CUDA(cudaEventCreateWithFlags(&ctx->ev_in[c], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&ctx->ev_comp[c], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&ctx->ev_out[c], cudaEventDisableTiming));
    }
  }
  cudaStream_t sin = nchunk > 1 ? ctx->h2d : st;
  cudaStream_t sout = nchunk > 1 ? ctx->d2h : st;
  if (nchunk > 1) {  // copy streams must not overtake earlier work on the compute stream
    SP_CUDA(cudaEventRecord(ctx->ev_out[0], st));
    SP_CUDA(cudaStreamWaitEvent(sin, ctx->ev_out[0], 0));
    SP_CUDA(cudaStreamWaitEvent(sout, ctx->ev_out[0], 0));
  }
  const auto h2d = cudaMemcpyHostToDevice;
  const auto d2h = cudaMemcpyDeviceToHost;
  for (int c = 0; c < nchunk; ++c) {
    const size_t a = (size_t)N * c / nchunk, n = (size_t)N * (c + 1) / nchunk - a;
    if (n == 0) continue;
    SP_CUDA(cudaMemcpyAsync(d_slack + a * K, slack + a * K, sizeof(double) * n * K, h2d, sin));
    SP_CUDA(cudaMemcpyAsync(d_avail + a, avail + a, sizeof(int32_t) * n, h2d, sin));
    SP_CUDA(cudaMemcpyAsync(d_supply + a, supply + a, sizeof(int32_t) * n, h2d, sin));
    SP_CUDA(cudaMemcpyAsync(d_minb + a, min_batch + a, sizeof(int32_t) * n, h2d, sin));
    SP_CUDA(cudaMemcpyAsync(d_flags + a, flags + a, sizeof(uint32_t) * n, h2d, sin));
    if (op) SP_CUDA(cudaMemcpyAsync(d_op + a, op + a, sizeof(int32_t) * n, h2d, sin));
    if (nchunk > 1) {
      SP_CUDA(cudaEventRecord(ctx->ev_in[c], sin));
      SP_CUDA(cudaStreamWaitEvent(st, ctx->ev_in[c], 0));
    }
    rc = select_launch(ctx, n_tables, tables, alpha, (int)n, d_op ? d_op + a : nullptr,
                       d_slack + a * K, d_avail + a, d_supply + a, d_minb + a, d_flags + a,
                       d_idx + a, d_code + a, d_fill + a, d_obj + a, d_sl + a, d_wait + a,
                       d_kmin ? d_kmin + a * K : nullptr, mode);
    if (rc != SP_OK) return rc;
    if (nchunk > 1) {
      SP_CUDA(cudaEventRecord(ctx->ev_comp[c], st));
      SP_CUDA(cudaStreamWaitEvent(sout, ctx->ev_comp[c], 0));
    }
    SP_CUDA(cudaMemcpyAsync(out_idx + a, d_idx + a, sizeof(int32_t) * n, d2h, sout));
    SP_CUDA(cudaMemcpyAsync(out_code + a, d_code + a, sizeof(int32_t) * n, d2h, sout));
    if (out_fill) SP_CUDA(cudaMemcpyAsync(out_fill + a, d_fill + a, sizeof(int32_t) * n, d2h, sout));
    if (out_obj) SP_CUDA(cudaMemcpyAsync(out_obj + a, d_obj + a, sizeof(double) * n, d2h, sout));
    if (out_slack) SP_CUDA(cudaMemcpyAsync(out_slack + a, d_sl + a, sizeof(double) * n, d2h, sout));
    if (out_wait) SP_CUDA(cudaMemcpyAsync(out_wait + a, d_wait + a, sizeof(double) * n, d2h, sout));
    if (out_kind_min)
      SP_CUDA(cudaMemcpyAsync(out_kind_min + a * K, d_kmin + a * K, sizeof(double) * n * K, d2h, sout));
  }
  if (nchunk > 1) {  // the compute stream's later work must see the completed outputs
    SP_CUDA(cudaEventRecord(ctx->ev_out[0], sout));
    SP_CUDA(cudaStreamWaitEvent(st, ctx->ev_out[0], 0));
  }
  if (sync) {
    SP_CUDA(cudaStreamSynchronize(sout));
    SP_CUDA(cudaStreamSynchronize(st));
  }
  return SP_OK;
}

int select_host_wait(sp_ctx* ctx) {
  if (ctx->d2h) SP_CUDA(cudaStreamSynchronize(ctx->d2h));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  return SP_OK;
}
}  // namespace sp

extern "C" {

int sp_select_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                    int32_t N, const int32_t* op, const double* slack, const int32_t* avail,
                    const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                    int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                    double* out_slack, double* out_wait, double* out_kind_min, int32_t mode,
                    int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  return select_batch_impl(ctx, n_tables, tables, alpha, N, op, slack, avail, supply, min_batch,
                           flags, out_idx, out_code, out_fill, out_obj, out_slack, out_wait,
                           out_kind_min, mode, mem, true);
}

int sp_affinity_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                      int32_t N, const int32_t* op, const double* slack, const int32_t* query_kind,
                      double* out, int32_t mode) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !tables || n_tables < 1 || N < 0 || (N > 0 && (!slack || !query_kind || !out)))
    return fail(SP_E_INVALID, "affinity_batch: bad argument");
  if (!(alpha >= 0.0)) return fail(SP_E_INVALID, "alpha must be >= 0");  // configurator.py:37
  const int K = tables[0]->K;
  for (int i = 0; i < N; ++i) {
    if (query_kind[i] < 0 || query_kind[i] >= K) return fail(SP_E_INVALID, "affinity: kind out of range");
    if (op && (op[i] < 0 || op[i] >= n_tables)) return fail(SP_E_INVALID, "affinity: op out of range");
  }
  if (N == 0) return SP_OK;
  // one staging block: the unmasked select inputs (every kind admitted, min_batch 1), the
  // per-kind minima and the ratios; one sync
  int rc = SP_OK;
  const size_t need = rsz<double>((size_t)N * K) * 2 + rsz<int32_t>(N) * 8 + rsz<double>(N);
  void* dbase = nullptr;
  uint8_t* hb = static_cast<uint8_t*>(ctx_pin(ctx, need, &dbase, &rc));
  if (!hb) return rc;
  uint8_t* db = static_cast<uint8_t*>(dbase);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t o_sl = take(sizeof(double) * N * K), o_km = take(sizeof(double) * N * K),
               o_av = take(4u * N), o_su = take(4u * N), o_mb = take(4u * N), o_fl = take(4u * N),
               o_op = take(4u * N), o_q = take(4u * N), o_ix = take(4u * N), o_cd = take(4u * N),
               o_out = take(8u * N);
  memcpy(hb + o_sl, slack, sizeof(double) * N * K);
  memcpy(hb + o_q, query_kind, 4u * N);
  if (op) memcpy(hb + o_op, op, 4u * N);
  int32_t* av = (int32_t*)(hb + o_av);
  int32_t* su = (int32_t*)(hb + o_su);
  int32_t* mb = (int32_t*)(hb + o_mb);
  uint32_t* fl = (uint32_t*)(hb + o_fl);
  for (int i = 0; i < N; ++i) {
    av[i] = 1;
    su[i] = 0;
    mb[i] = 1;
    fl[i] = 0u;
  }
  rc = select_launch(ctx, n_tables, tables, alpha, N, op ? (const int32_t*)(db + o_op) : nullptr,
                     (const double*)(db + o_sl), (const int32_t*)(db + o_av),
                     (const int32_t*)(db + o_su), (const int32_t*)(db + o_mb),
                     (const uint32_t*)(db + o_fl), (int32_t*)(db + o_ix), (int32_t*)(db + o_cd),
                     nullptr, nullptr, nullptr, nullptr, (double*)(db + o_km), mode);
  if (rc != SP_OK) return rc;
  rc = affinity_launch(ctx, N, K, (const double*)(db + o_km), (const int32_t*)(db + o_q),
                       (double*)(db + o_out));
  if (rc != SP_OK) return rc;
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  memcpy(out, hb + o_out, 8u * N);
  return SP_OK;
}

int sp_affinity_from_minima(sp_ctx* ctx, int32_t N, int32_t K, const double* kind_min,
                            const int32_t* query_kind, double* out, void* reserved,
                            int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || N < 0 || K < 1 || K > kMaxTableKinds || reserved)
    return fail(SP_E_INVALID, "affinity: bad argument");
  if (N > 0 && (!kind_min || !query_kind || !out)) return fail(SP_E_INVALID, "affinity: null array");
  if (mem == SP_MEM_DEVICE) return affinity_launch(ctx, N, K, kind_min, query_kind, out);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "affinity: bad mem flag");
  for (int i = 0; i < N; ++i)
    if (query_kind[i] < 0 || query_kind[i] >= K) return fail(SP_E_INVALID, "affinity: kind out of range");
  int rc = SP_OK;
  void* io = ctx_io(ctx, rsz<double>((size_t)N * K) + rsz<int32_t>(N) + rsz<double>(N), &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  double* d_k = b.take<double>((size_t)N * K);
  int32_t* d_q = b.take<int32_t>(N);
  double* d_o = b.take<double>(N);
  cudaStream_t st = ctx->stream;
  if (N > 0) {
    SP_CUDA(cudaMemcpyAsync(d_k, kind_min, sizeof(double) * N * K, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_q, query_kind, sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
  }
  rc = affinity_launch(ctx, N, K, d_k, d_q, d_o);
  if (rc != SP_OK) return rc;
  if (N > 0) SP_CUDA(cudaMemcpyAsync(out, d_o, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

// ---- K1 graph ----------------------------------------------------------------------------
int sp_dag_create(sp_ctx* ctx, int32_t V, const int32_t* pred_ptr, const int32_t* pred_idx,
                  const int32_t* val_idx, const uint8_t* terminal, int32_t n_src,
                  const int32_t* sources, sp_dag** out) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !out || V < 1 || !pred_ptr || !val_idx || !terminal || n_src < 1 || !sources)
    return fail(SP_E_INVALID, "dag_create: bad argument");
  if (pred_ptr[0] != 0) return fail(SP_E_INVALID, "dag_create: pred_ptr[0] must be 0");
  for (int v = 0; v < V; ++v) {
    if (pred_ptr[v + 1] < pred_ptr[v]) return fail(SP_E_INVALID, "dag_create: bad pred_ptr");
    for (int q = pred_ptr[v]; q < pred_ptr[v + 1]; ++q)
      if (pred_idx[q] < 0 || pred_idx[q] >= v)
        return fail(SP_E_INVALID, "dag_create: vertices must be in topological order");
    if (val_idx[v] < 0) return fail(SP_E_INVALID, "dag_create: bad val_idx");
  }
  // successor lists to compute descendant sets
  std::vector<std::vector<int>> succ(V);
  for (int v = 0; v < V; ++v)
    for (int q = pred_ptr[v]; q < pred_ptr[v + 1]; ++q) succ[pred_idx[q]].push_back(v);
  std::vector<int4> prog;
  std::vector<int32_t> pptr(1, 0), qptr(1, 0);
  std::vector<uint32_t> preds;
  int max_span = 0, max_slots = 0, max_preds = 0, n_val = 0;
  bool single_pred = true;  // every descendant has exactly one reachable predecessor (a trie)
  for (int v = 0; v < V; ++v) n_val = std::max(n_val, val_idx[v] + 1);
  std::vector<int> slot(V, -1), last(V, -1);
  std::vector<int> free_slots;
  for (int s = 0; s < n_src; ++s) {
    int src = sources[s];
    if (src < 0 || src >= V) return fail(SP_E_INVALID, "dag_create: source out of range");
    std::fill(slot.begin(), slot.end(), -1);
    std::vector<char> reach(V, 0);
    reach[src] = 1;
    for (int v = src; v < V; ++v)
      if (reach[v])
        for (int w : succ[v]) reach[w] = 1;
    // last reader of each reachable value (vertices are in topological order, so the
    // largest reachable successor id); a value without readers dies where it is made
    for (int v = src; v < V; ++v) {
      if (!reach[v]) continue;
      last[v] = v;
      for (int w : succ[v]) last[v] = std::max(last[v], w);
    }
    free_slots.clear();
    int nslot = 0, nprog = 0;
    const int qbase = (int)preds.size();
    for (int v = src; v < V; ++v) {
      if (!reach[v]) continue;
      ++nprog;
      const int pb = (int)preds.size() - qbase;
      if (v != src) {
        for (int q = pred_ptr[v]; q < pred_ptr[v + 1]; ++q) {
          int p = pred_idx[q];
          if (reach[p]) preds.push_back((uint32_t)slot[p]);
        }
        if ((int)preds.size() - qbase - pb != 1) single_pred = false;
        if (((int)preds.size() - qbase - pb) & 1) preds.push_back(preds.back());
        // predecessors read for the last time here release their slots; the kernel reads
        // every predecessor before it writes the new value, so v may take one of them
        for (int q = pred_ptr[v]; q < pred_ptr[v + 1]; ++q) {
          int p = pred_idx[q];
          if (reach[p] && last[p] == v && slot[p] >= 0) {
            free_slots.push_back(slot[p]);
            slot[p] = -2;  // released (a predecessor may be listed twice)
          }
        }
      }
      int sl;
      if (!free_slots.empty()) {
        sl = free_slots.back();
        free_slots.pop_back();
      } else {
        sl = nslot++;
      }
      if (last[v] == v) {
        free_slots.push_back(sl);  // only the terminal fold reads it
        slot[v] = -2;
      } else {
        slot[v] = sl;
      }
      const int npairs = ((int)preds.size() - qbase - pb) >> 1;
      prog.push_back(make_int4(val_idx[v], sl | (terminal[v] ? 1 << 16 : 0), pb, npairs));
    }
    if (nslot > 65535 || (int)preds.size() - qbase > (1 << 24))
      return fail(SP_E_UNSUPPORTED, "dag_create: too many descendants");
    max_span = std::max(max_span, nprog);
    max_slots = std::max(max_slots, nslot);
    max_preds = std::max(max_preds, (int)preds.size() - qbase);
    pptr.push_back((int32_t)prog.size());
    qptr.push_back((int32_t)preds.size());
  }
  sp_dag* g = new (std::nothrow) sp_dag();
  if (!g) return fail(SP_E_NOMEM, "dag_create: host allocation");
  g->V = V;
  g->n_src = n_src;
  g->n_val = n_val;
  g->max_span = max_span;
  g->max_slots = max_slots;
  g->max_preds = max_preds;
  g->single_pred = single_pred ? 1 : 0;
  g->prog_len = (int64_t)prog.size();
  g->pred_len = (int64_t)preds.size();
  cudaError_t e = cudaMalloc(&g->prog, sizeof(int4) * prog.size());
  if (e == cudaSuccess) e = cudaMalloc(&g->prog_ptr, sizeof(int32_t) * pptr.size());
  if (e == cudaSuccess) e = cudaMalloc(&g->pred_ptr, sizeof(int32_t) * qptr.size());
  if (e == cudaSuccess) e = cudaMalloc(&g->preds, sizeof(uint32_t) * std::max<size_t>(4, preds.size()));
  if (e == cudaSuccess)
    e = cudaMemcpy(g->prog, prog.data(), sizeof(int4) * prog.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(g->prog_ptr, pptr.data(), sizeof(int32_t) * pptr.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(g->pred_ptr, qptr.data(), sizeof(int32_t) * qptr.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !preds.empty())
    e = cudaMemcpy(g->preds, preds.data(), sizeof(uint32_t) * preds.size(), cudaMemcpyHostToDevice);
  // certified backward form (k_slack_cert): worth it when the per-source forward programs
  // relax many more edges than one backward pass over the graph does
  // (SP_K1_CERT=force builds it for every eligible graph — the parity tests use that)
  int E = pred_ptr[V];
  const bool force = ctx->opt.k1_cert == 2;
  const bool off = ctx->opt.k1_cert == 1;
  if (e == cudaSuccess && !off && V <= kCertMaxV && n_val < 65536 &&
      (force || (int64_t)preds.size() >= 4 * (int64_t)(E + V))) {
    auto a16 = [](int x) { return (x + 15) & ~15; };
    // successor lists as u16 byte offsets (node * 256, the stride of a node's row in the
    // kernel's [node][lane] arrays), padded to groups of four with the sentinel row V
    int groups = 0;
    for (int v = 0; v < V; ++v) groups += ((int)succ[v].size() + 3) / 4;
    g->E = E;
    g->off_vidx = a16(2 * (V + 1));
    g->off_term = g->off_vidx + a16(2 * V);
    g->off_src = g->off_term + a16(V);
    g->off_succ = g->off_src + a16(n_src);
    g->cert_bytes = g->off_succ + a16(8 * std::max(groups, 1));
    std::vector<uint8_t> img(g->cert_bytes, 0);
    uint16_t* sp = reinterpret_cast<uint16_t*>(img.data());  // group index of each node's list
    uint16_t* vi = reinterpret_cast<uint16_t*>(img.data() + g->off_vidx);
    uint16_t* so = reinterpret_cast<uint16_t*>(img.data() + g->off_succ);
    int q = 0;
    for (int v = 0; v < V; ++v) {
      sp[v] = (uint16_t)q;
      const int n = (int)succ[v].size(), ng = (n + 3) / 4;
      for (int j = 0; j < 4 * ng; ++j) so[4 * q + j] = (uint16_t)((j < n ? succ[v][j] : V) * 256);
      q += ng;
      vi[v] = (uint16_t)val_idx[v];
      img[g->off_term + v] = terminal[v] ? 1 : 0;
    }
    sp[V] = (uint16_t)q;
    for (int s = 0; s < n_src; ++s) img[g->off_src + s] = (uint8_t)sources[s];
    e = cudaMalloc(&g->cert, img.size());
    if (e == cudaSuccess) e = cudaMemcpy(g->cert, img.data(), img.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(g->prog);
    cudaFree(g->prog_ptr);
    cudaFree(g->pred_ptr);
    cudaFree(g->preds);
    cudaFree(g->cert);
    delete g;
    return cuda_fail(e, "dag_create");
  }
  *out = g;
  return SP_OK;
}

int sp_dag_destroy(sp_ctx* ctx, sp_dag* g) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!g) return SP_OK;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  cudaFree(g->prog);
  cudaFree(g->prog_ptr);
  cudaFree(g->pred_ptr);
  cudaFree(g->preds);
  cudaFree(g->cert);
  delete g;
  return SP_OK;
}

int sp_slack_batch(sp_ctx* ctx, sp_dag* g, int32_t I, const double* ref_lat,
                   int32_t ref_stride, const double* target, const double* now, int32_t K,
                   const double* Q, double* out_slack, double* out_ratio, int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !g || I < 0 || !ref_lat || !target || !now || K < 0 || (K > 0 && !Q))
    return fail(SP_E_INVALID, "slack_batch: bad argument");
  if (ref_stride != 0 && ref_stride < g->n_val)
    return fail(SP_E_INVALID, "slack_batch: ref_stride smaller than the value count");
  if (mem == SP_MEM_DEVICE)
    return slack_launch(ctx, g, I, ref_lat, ref_stride, target, now, K, Q, out_slack,
                        out_ratio);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "slack_batch: bad mem flag");
  const size_t nref = ref_stride ? (size_t)I * ref_stride : (size_t)g->n_val;
  const size_t nout = (size_t)I * g->n_src;
  size_t need = rsz<double>(nref) + 2 * rsz<double>(I) + rsz<double>((size_t)I * K) +
                (out_slack ? rsz<double>(nout * K) : 0) + (out_ratio ? rsz<double>(nout * 2) : 0);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  double* d_ref = b.take<double>(nref);
  double* d_t = b.take<double>(I);
  double* d_n = b.take<double>(I);
  double* d_q = b.take<double>((size_t)I * K);
  double* d_out = out_slack ? b.take<double>(nout * K) : nullptr;
  double* d_rat = out_ratio ? b.take<double>(nout * 2) : nullptr;
  SP_CUDA(cudaMemcpyAsync(d_ref, ref_lat, sizeof(double) * nref, cudaMemcpyHostToDevice, st));
  if (I > 0) {
    SP_CUDA(cudaMemcpyAsync(d_t, target, sizeof(double) * I, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_n, now, sizeof(double) * I, cudaMemcpyHostToDevice, st));
    if (K > 0)
      SP_CUDA(cudaMemcpyAsync(d_q, Q, sizeof(double) * I * K, cudaMemcpyHostToDevice, st));
  }
  rc = slack_launch(ctx, g, I, d_ref, ref_stride, d_t, d_n, K, d_q, d_out, d_rat);
  if (rc != SP_OK) return rc;
  if (I > 0 && out_slack)
    SP_CUDA(cudaMemcpyAsync(out_slack, d_out, sizeof(double) * nout * K, cudaMemcpyDeviceToHost, st));
  if (I > 0 && out_ratio)
    SP_CUDA(cudaMemcpyAsync(out_ratio, d_rat, sizeof(double) * nout * 2, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_queueing(sp_ctx* ctx, int32_t K, const int32_t* ptr, const double* lat,
                const double* res, const int32_t* cnt, const double* pool, double* out) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || K < 1 || K > 32 || !ptr || !pool || !out)
    return fail(SP_E_INVALID, "queueing: bad argument");
  const int n = ptr[K];
  if (n < 0) return fail(SP_E_INVALID, "queueing: bad ptr");
  size_t need = rsz<int32_t>(K + 1) + 2 * rsz<double>(n) + rsz<int32_t>(n) + 2 * rsz<double>(K);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  int32_t* d_ptr = b.take<int32_t>(K + 1);
  double* d_lat = b.take<double>(n);
  double* d_res = b.take<double>(n);
  int32_t* d_cnt = cnt ? b.take<int32_t>(n) : nullptr;
  double* d_pool = b.take<double>(K);
  double* d_out = b.take<double>(K);
  SP_CUDA(cudaMemcpyAsync(d_ptr, ptr, sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, st));
  if (n > 0) {
    SP_CUDA(cudaMemcpyAsync(d_lat, lat, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_res, res, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    if (cnt) SP_CUDA(cudaMemcpyAsync(d_cnt, cnt, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  }
  SP_CUDA(cudaMemcpyAsync(d_pool, pool, sizeof(double) * K, cudaMemcpyHostToDevice, st));
  rc = queueing_launch(ctx, K, d_ptr, d_lat, d_res, d_cnt, d_pool, d_out);
  if (rc != SP_OK) return rc;
  SP_CUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_feedback_fold(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, int32_t n,
                     const int32_t* op, const int32_t* idx, const double* obs, double beta,
                     int32_t dfp_count, int32_t dfp_on, int32_t fb_frozen, int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !tables || n_tables < 1 || n < 0 || (n > 0 && (!idx || !obs)))
    return fail(SP_E_INVALID, "feedback_fold: bad argument");
  if (!(beta > 0.0 && beta <= 1.0)) return fail(SP_E_INVALID, "smoothing_beta must be in (0, 1]");
  if (mem == SP_MEM_DEVICE)
    return fold_launch(ctx, n_tables, tables, n, op, idx, obs, beta, dfp_count, dfp_on,
                       fb_frozen);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "feedback_fold: bad mem flag");
  for (int j = 0; j < n; ++j) {
    int t = op ? op[j] : 0;
    if (t < 0 || t >= n_tables) return fail(SP_E_INVALID, "feedback_fold: op out of range");
    if (idx[j] >= tables[t]->M)  // idx < 0: no observation (skipped)
      return fail(SP_E_INVALID, "feedback_fold: entry index out of range");
    // a non-finite observation (or a fold into a table already holding non-finite latencies,
    // which the gate lift can spread) leaves non-finite latencies behind: from now on the
    // table's decisions take the literal scan
    if (idx[j] >= 0 && !fb_frozen && (!isfinite(obs[j]) || tables[t]->nonfinite))
      tables[t]->tainted = true;
  }
  size_t need = 2 * rsz<int32_t>(n) + rsz<double>(n);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  int32_t* d_op = op ? b.take<int32_t>(n) : nullptr;
  int32_t* d_idx = b.take<int32_t>(n);
  double* d_obs = b.take<double>(n);
  if (n > 0) {
    if (op) SP_CUDA(cudaMemcpyAsync(d_op, op, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_idx, idx, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_obs, obs, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  }
  rc = fold_launch(ctx, n_tables, tables, n, d_op, d_idx, d_obs, beta, dfp_count, dfp_on,
                   fb_frozen);
  if (rc != SP_OK) return rc;
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_table_get_counters(sp_ctx* ctx, sp_table* t, int32_t* completed_ref,
                          int32_t* out_obs_count) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t) return fail(SP_E_INVALID, "get_counters: null argument");
  int32_t c[4];
  SP_CUDA(cudaMemcpyAsync(c, t->dev_counters, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  if (out_obs_count)
    SP_CUDA(cudaMemcpyAsync(out_obs_count, t->obs_count, sizeof(int32_t) * t->M,
                            cudaMemcpyDeviceToHost, ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (completed_ref) *completed_ref = c[0];
  return SP_OK;
}

int sp_table_set_counters(sp_ctx* ctx, sp_table* t, int32_t completed_ref,
                          const int32_t* obs_count) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !t) return fail(SP_E_INVALID, "set_counters: null argument");
  int32_t c[4] = {completed_ref, 0, 0, 0};
  SP_CUDA(cudaMemcpyAsync(t->dev_counters, c, sizeof(c), cudaMemcpyHostToDevice, ctx->stream));
  if (obs_count)
    SP_CUDA(cudaMemcpyAsync(t->obs_count, obs_count, sizeof(int32_t) * t->M,
                            cudaMemcpyHostToDevice, ctx->stream));
  SP_CUDA(cudaStreamSynchronize(ctx->stream));
  return SP_OK;
}

}  // extern "C"

// ---- batched commit step (configurator.py:657-756) ----------------------------------------
extern "C" int sp_speculate_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables,
                                  double alpha, int32_t K, const double* pool, int32_t R,
                                  const int32_t* op, const int32_t* n_buf, const int32_t* supply,
                                  const double* now, const double* target, const double* rmin,
                                  const double* rmax, const double* slack0,
                                  const uint32_t* flags, const int32_t* w_ptr,
                                  const int32_t* w_tab, const int32_t* w_eidx,
                                  const int32_t* w_count, const int32_t* out_off,
                                  int32_t* out_idx, int32_t* out_fill, double* out_slack,
                                  double* out_obj, int32_t* out_n, int32_t* out_delay_idx,
                                  double* out_delay_wait, int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !tables || !pool) return fail(SP_E_INVALID, "speculate: null argument");
  if (n_tables < 1 || n_tables > 64) return fail(SP_E_INVALID, "speculate: n_tables must be in [1, 64]");
  if (!(alpha >= 0.0)) return fail(SP_E_INVALID, "alpha must be >= 0");  // configurator.py:37
  if (R < 0) return fail(SP_E_INVALID, "speculate: negative call count");
  for (int t = 0; t < n_tables; ++t) {
    if (!tables[t]) return fail(SP_E_INVALID, "speculate: null table");
    if (tables[t]->K != K) return fail(SP_E_INVALID, "speculate: tables disagree with K");
  }
  if (R == 0) return SP_OK;
  if (!op || !n_buf || !supply || !now || !target || !rmin || !rmax || !slack0 || !flags ||
      !w_ptr || !w_tab || !w_eidx || !w_count || !out_off || !out_idx || !out_fill ||
      !out_slack || !out_obj || !out_n || !out_delay_idx || !out_delay_wait)
    return fail(SP_E_INVALID, "speculate: required array is null");
  if (mem == SP_MEM_DEVICE)
    return speculate_launch(ctx, n_tables, tables, alpha, K, pool, R, op, n_buf, supply, now,
                            target, rmin, rmax, slack0, flags, w_ptr, w_tab, w_eidx, w_count,
                            out_off, out_idx, out_fill, out_slack, out_obj, out_n,
                            out_delay_idx, out_delay_wait, -1, -1);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "speculate: bad mem flag");
  // host-side validation of everything the kernel indexes
  const size_t nw = (size_t)2 * K * R;
  if (w_ptr[0] != 0) return fail(SP_E_INVALID, "speculate: w_ptr[0] must be 0");
  for (size_t q = 0; q < nw; ++q)
    if (w_ptr[q + 1] < w_ptr[q]) return fail(SP_E_INVALID, "speculate: w_ptr not ascending");
  const int W = w_ptr[nw];
  for (int w = 0; w < W; ++w)
    if (w_tab[w] < 0 || w_tab[w] >= n_tables || w_eidx[w] < 0 || w_eidx[w] >= tables[w_tab[w]]->M)
      return fail(SP_E_INVALID, "speculate: weight key out of range");
  if (out_off[0] != 0) return fail(SP_E_INVALID, "speculate: out_off[0] must be 0");
  for (int r = 0; r < R; ++r) {
    if (op[r] < 0 || op[r] >= n_tables) return fail(SP_E_INVALID, "speculate: op out of range");
    if (n_buf[r] < 0) return fail(SP_E_INVALID, "speculate: negative buffer");
    if (out_off[r + 1] - out_off[r] < n_buf[r])
      return fail(SP_E_INVALID, "speculate: output slots smaller than the buffer");
    if ((flags[r] & SP_SPEC_FORCED) && tables[op[r]]->ref_index < 0)
      return fail(SP_E_INVALID, "speculate: forced call on a table without a reference entry");
  }
  const int O = out_off[R];
  const size_t need = 3 * rsz<int32_t>(R) + 4 * rsz<double>(R) + rsz<double>((size_t)R * K) +
                      rsz<uint32_t>(R) + rsz<int32_t>(nw + 1) + 3 * rsz<int32_t>(std::max(W, 1)) +
                      rsz<int32_t>(R + 1) + 2 * rsz<int32_t>(std::max(O, 1)) +
                      2 * rsz<double>(std::max(O, 1)) + 2 * rsz<int32_t>(R) + rsz<double>(R);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  auto up = [&](auto* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
  };
  int32_t* d_op = b.take<int32_t>(R);
  int32_t* d_n = b.take<int32_t>(R);
  int32_t* d_sup = b.take<int32_t>(R);
  double* d_now = b.take<double>(R);
  double* d_tgt = b.take<double>(R);
  double* d_rmin = b.take<double>(R);
  double* d_rmax = b.take<double>(R);
  double* d_s0 = b.take<double>((size_t)R * K);
  uint32_t* d_fl = b.take<uint32_t>(R);
  int32_t* d_wp = b.take<int32_t>(nw + 1);
  int32_t* d_wt = b.take<int32_t>(std::max(W, 1));
  int32_t* d_we = b.take<int32_t>(std::max(W, 1));
  int32_t* d_wc = b.take<int32_t>(std::max(W, 1));
  int32_t* d_off = b.take<int32_t>(R + 1);
  int32_t* o_idx = b.take<int32_t>(std::max(O, 1));
  int32_t* o_fill = b.take<int32_t>(std::max(O, 1));
  double* o_sl = b.take<double>(std::max(O, 1));
  double* o_ob = b.take<double>(std::max(O, 1));
  int32_t* o_n = b.take<int32_t>(R);
  int32_t* o_di = b.take<int32_t>(R);
  double* o_dw = b.take<double>(R);
  SP_CUDA(up(d_op, op, 4 * (size_t)R));
  SP_CUDA(up(d_n, n_buf, 4 * (size_t)R));
  SP_CUDA(up(d_sup, supply, 4 * (size_t)R));
  SP_CUDA(up(d_now, now, 8 * (size_t)R));
  SP_CUDA(up(d_tgt, target, 8 * (size_t)R));
  SP_CUDA(up(d_rmin, rmin, 8 * (size_t)R));
  SP_CUDA(up(d_rmax, rmax, 8 * (size_t)R));
  SP_CUDA(up(d_s0, slack0, 8 * (size_t)R * K));
  SP_CUDA(up(d_fl, flags, 4 * (size_t)R));
  SP_CUDA(up(d_wp, w_ptr, 4 * (nw + 1)));
  SP_CUDA(up(d_wt, w_tab, 4 * (size_t)W));
  SP_CUDA(up(d_we, w_eidx, 4 * (size_t)W));
  SP_CUDA(up(d_wc, w_count, 4 * (size_t)W));
  SP_CUDA(up(d_off, out_off, 4 * (size_t)(R + 1)));
  rc = speculate_launch(ctx, n_tables, tables, alpha, K, pool, R, d_op, d_n, d_sup, d_now, d_tgt,
                        d_rmin, d_rmax, d_s0, d_fl, d_wp, d_wt, d_we, d_wc, d_off, o_idx, o_fill,
                        o_sl, o_ob, o_n, o_di, o_dw, W, O);
  if (rc != SP_OK) return rc;
  auto down = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
  };
  SP_CUDA(down(out_idx, o_idx, 4 * (size_t)O));
  SP_CUDA(down(out_fill, o_fill, 4 * (size_t)O));
  SP_CUDA(down(out_slack, o_sl, 8 * (size_t)O));
  SP_CUDA(down(out_obj, o_ob, 8 * (size_t)O));
  SP_CUDA(down(out_n, o_n, 4 * (size_t)R));
  SP_CUDA(down(out_delay_idx, o_di, 4 * (size_t)R));
  SP_CUDA(down(out_delay_wait, o_dw, 8 * (size_t)R));
  SP_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < R; ++r)
    if (out_n[r] < 0)  // a select with no admissible entry inside the loop (configurator.py:605)
      return fail(SP_E_RUNTIME, "speculate: select returned None inside the speculation loop");
  return SP_OK;
}

extern "C" int sp_commit_round(sp_ctx* ctx, int32_t R, int32_t n_ops, sp_table* const* tables,
                               double alpha, const double* slack, const int32_t* head_fill,
                               const int32_t* buffered, const int64_t* head_id,
                               const int32_t* depth, const uint32_t* head_flags,
                               const int32_t* spec_idx, const double* spec_slack,
                               const double* spec_obj, const uint32_t* full_mask, int32_t policy,
                               int32_t* out_idx, int32_t* out_fill, double* out_slack,
                               double* out_obj, double* out_aff, int32_t* out_best,
                               int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !tables) return fail(SP_E_INVALID, "commit: null argument");
  if (n_ops < 1 || n_ops > 64) return fail(SP_E_INVALID, "commit: n_ops must be in [1, 64]");
  if (R < 0) return fail(SP_E_INVALID, "commit: negative round count");
  if (!(alpha >= 0.0)) return fail(SP_E_INVALID, "alpha must be >= 0");  // configurator.py:37
  for (int j = 0; j < n_ops; ++j)
    if (!tables[j]) return fail(SP_E_INVALID, "commit: null table");
  const int K = tables[0]->K;
  for (int j = 0; j < n_ops; ++j)
    if (tables[j]->K != K) return fail(SP_E_INVALID, "commit: tables disagree on kind count");
  if (R == 0) return SP_OK;
  if (!slack || !head_fill || !buffered || !head_id || !depth || !head_flags || !spec_idx ||
      !spec_slack || !spec_obj || !full_mask || !out_idx || !out_fill || !out_slack || !out_obj ||
      !out_aff || !out_best)
    return fail(SP_E_INVALID, "commit: required array is null");
  const size_t N = (size_t)R * n_ops;
  int rc = SP_OK;
  void* scratch = ctx_tmp(ctx, commit_scratch_bytes(R, n_ops, K), &rc);
  if (!scratch) return rc;
  if (mem == SP_MEM_DEVICE)
    return commit_launch(ctx, R, n_ops, tables, alpha, slack, head_fill, buffered,
                         reinterpret_cast<const long long*>(head_id), depth, head_flags, spec_idx,
                         spec_slack, spec_obj, full_mask, policy, scratch, out_idx, out_fill,
                         out_slack, out_obj, out_aff, out_best);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "commit: bad mem flag");
  for (size_t i = 0; i < N; ++i) {  // host-side validation of what the kernel will index
    const int j = (int)(i % n_ops);
    if ((head_flags[i] & SP_HEAD_PRESENT) && !(head_flags[i] & SP_HEAD_FORCED) &&
        (policy & SP_COMMIT_ESLC) && (spec_idx[i] < 0 || spec_idx[i] >= tables[j]->M))
      return fail(SP_E_INVALID, "commit: speculated entry index out of range");
    if (head_fill[i] < 0 || buffered[i] < 0) return fail(SP_E_INVALID, "commit: negative fill");
  }
  const size_t need = rsz<double>(N * K) + 5 * rsz<int32_t>(N) + rsz<int64_t>(N) +
                      rsz<int32_t>(n_ops) + 2 * rsz<double>(N) + rsz<uint32_t>(R) +
                      2 * rsz<int32_t>(N) + 3 * rsz<double>(N) + rsz<int32_t>(R);
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  auto up = [&](auto* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  double* d_slack = b.take<double>(N * K);
  int32_t* d_fill = b.take<int32_t>(N);
  int32_t* d_buf = b.take<int32_t>(N);
  long long* d_id = b.take<long long>(N);
  int32_t* d_depth = b.take<int32_t>(n_ops);
  uint32_t* d_hf = b.take<uint32_t>(N);
  int32_t* d_sidx = b.take<int32_t>(N);
  double* d_ssl = b.take<double>(N);
  double* d_sob = b.take<double>(N);
  uint32_t* d_full = b.take<uint32_t>(R);
  int32_t* o_idx = b.take<int32_t>(N);
  int32_t* o_fill = b.take<int32_t>(N);
  double* o_sl = b.take<double>(N);
  double* o_ob = b.take<double>(N);
  double* o_aff = b.take<double>(N);
  int32_t* o_best = b.take<int32_t>(R);
  SP_CUDA(up(d_slack, slack, sizeof(double) * N * K));
  SP_CUDA(up(d_fill, head_fill, 4 * N));
  SP_CUDA(up(d_buf, buffered, 4 * N));
  SP_CUDA(up(d_id, head_id, 8 * N));
  SP_CUDA(up(d_depth, depth, 4 * (size_t)n_ops));
  SP_CUDA(up(d_hf, head_flags, 4 * N));
  SP_CUDA(up(d_sidx, spec_idx, 4 * N));
  SP_CUDA(up(d_ssl, spec_slack, 8 * N));
  SP_CUDA(up(d_sob, spec_obj, 8 * N));
  SP_CUDA(up(d_full, full_mask, 4 * (size_t)R));
  rc = commit_launch(ctx, R, n_ops, tables, alpha, d_slack, d_fill, d_buf, d_id, d_depth, d_hf,
                     d_sidx, d_ssl, d_sob, d_full, policy, scratch, o_idx, o_fill, o_sl, o_ob,
                     o_aff, o_best);
  if (rc != SP_OK) return rc;
  auto down = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
  };
  SP_CUDA(down(out_idx, o_idx, 4 * N));
  SP_CUDA(down(out_fill, o_fill, 4 * N));
  SP_CUDA(down(out_slack, o_sl, 8 * N));
  SP_CUDA(down(out_obj, o_ob, 8 * N));
  SP_CUDA(down(out_aff, o_aff, 8 * N));
  SP_CUDA(down(out_best, o_best, 4 * (size_t)R));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

// ---- K1 -> K2 fused (sp_k12.cuh) ------------------------------------------------------------
extern "C" int sp_slack_select_batch(sp_ctx* ctx, sp_dag* g, int32_t n_tables,
                                     sp_table* const* tables, double alpha, int32_t I,
                                     const double* ref_lat, int32_t ref_stride,
                                     const double* target, const double* now, int32_t K,
                                     const double* Q, const int32_t* avail,
                                     const int32_t* supply, const int32_t* min_batch,
                                     const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                                     int32_t* out_fill, double* out_obj, double* out_slack,
                                     double* out_wait, double* out_kslack, int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !g || !tables || I < 0 || K < 1 || K > SP_MAX_KINDS)
    return fail(SP_E_INVALID, "slack_select: bad argument");
  for (int t = 0; t < n_tables; ++t)
    if (!tables[t]) return fail(SP_E_INVALID, "slack_select: null table");
  if (!(alpha >= 0.0)) return fail(SP_E_INVALID, "alpha must be >= 0");  // configurator.py:37
  if (ref_stride != 0 && ref_stride < g->n_val)
    return fail(SP_E_INVALID, "slack_select: ref_stride smaller than the value count");
  if (I > 0 && (!ref_lat || !target || !now || !Q || !avail || !supply || !min_batch || !flags ||
                !out_idx || !out_code))
    return fail(SP_E_INVALID, "slack_select: required array is null");
  if (mem == SP_MEM_DEVICE)
    return slack_select_launch(ctx, g, n_tables, tables, alpha, I, ref_lat, ref_stride, target,
                               now, K, Q, avail, supply, min_batch, flags, out_idx, out_code,
                               out_fill, out_obj, out_slack, out_wait, out_kslack);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "slack_select: bad mem flag");
  if (I == 0) return SP_OK;
  const size_t N = (size_t)I * n_tables;
  const size_t nref = ref_stride ? (size_t)I * ref_stride : (size_t)g->n_val;
  const size_t need = rsz<double>(nref) + 2 * rsz<double>(I) + rsz<double>((size_t)I * K) +
                      4 * rsz<int32_t>(N) + 3 * rsz<int32_t>(N) + 3 * rsz<double>(N) +
                      (out_kslack ? rsz<double>(N * K) : 0);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  double* d_ref = b.take<double>(nref);
  double* d_t = b.take<double>(I);
  double* d_n = b.take<double>(I);
  double* d_q = b.take<double>((size_t)I * K);
  int32_t* d_av = b.take<int32_t>(N);
  int32_t* d_sup = b.take<int32_t>(N);
  int32_t* d_mb = b.take<int32_t>(N);
  uint32_t* d_fl = b.take<uint32_t>(N);
  int32_t* o_idx = b.take<int32_t>(N);
  int32_t* o_code = b.take<int32_t>(N);
  int32_t* o_fill = b.take<int32_t>(N);
  double* o_obj = b.take<double>(N);
  double* o_sl = b.take<double>(N);
  double* o_wait = b.take<double>(N);
  double* o_ks = out_kslack ? b.take<double>(N * K) : nullptr;
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  };
  SP_CUDA(up(d_ref, ref_lat, sizeof(double) * nref));
  SP_CUDA(up(d_t, target, sizeof(double) * I));
  SP_CUDA(up(d_n, now, sizeof(double) * I));
  SP_CUDA(up(d_q, Q, sizeof(double) * I * K));
  SP_CUDA(up(d_av, avail, 4 * N));
  SP_CUDA(up(d_sup, supply, 4 * N));
  SP_CUDA(up(d_mb, min_batch, 4 * N));
  SP_CUDA(up(d_fl, flags, 4 * N));
  rc = slack_select_launch(ctx, g, n_tables, tables, alpha, I, d_ref, ref_stride, d_t, d_n, K,
                           d_q, d_av, d_sup, d_mb, d_fl, o_idx, o_code, o_fill, o_obj, o_sl,
                           o_wait, o_ks);
  if (rc != SP_OK) return rc;
  auto down = [&](void* dst, const void* src, size_t bytes) {
    return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
  };
  SP_CUDA(down(out_idx, o_idx, 4 * N));
  SP_CUDA(down(out_code, o_code, 4 * N));
  SP_CUDA(down(out_fill, o_fill, 4 * N));
  SP_CUDA(down(out_obj, o_obj, 8 * N));
  SP_CUDA(down(out_slack, o_sl, 8 * N));
  SP_CUDA(down(out_wait, o_wait, 8 * N));
  if (out_kslack) SP_CUDA(down(out_kslack, o_ks, 8 * N * K));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}

// ---- percentile estimate of an observation batch (sp_quantile.cu) ---------------------------
extern "C" int sp_observation_quantiles(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables,
                                        int32_t n, const int32_t* op, const int32_t* idx,
                                        const double* obs, double q, double beta, double* out,
                                        int32_t* out_count, double* out_smooth, int32_t mem) {
  DeviceScope _dev_scope(ctx ? ctx->device : -1);
  if (!ctx || !tables || n_tables < 1 || n < 0) return fail(SP_E_INVALID, "quantiles: bad argument");
  if (!(q >= 0.0 && q <= 1.0)) return fail(SP_E_INVALID, "quantiles: q must be in [0, 1]");
  if (out_smooth && !(beta >= 0.0 && beta <= 1.0))
    return fail(SP_E_INVALID, "quantiles: beta must be in [0, 1]");
  if (n > 0 && (!idx || !obs)) return fail(SP_E_INVALID, "quantiles: required array is null");
  size_t total = 0;
  for (int t = 0; t < n_tables; ++t) {
    if (!tables[t]) return fail(SP_E_INVALID, "quantiles: null table");
    total += (size_t)tables[t]->M;
  }
  if (mem == SP_MEM_DEVICE)
    return quantile_launch(ctx, n_tables, tables, n, op, idx, obs, q, beta, out, out_count,
                           out_smooth);
  if (mem != SP_MEM_HOST) return fail(SP_E_INVALID, "quantiles: bad mem flag");
  for (int j = 0; j < n; ++j) {
    const int t = op ? op[j] : 0;
    if (t < 0 || t >= n_tables) return fail(SP_E_INVALID, "quantiles: op out of range");
    if (idx[j] >= tables[t]->M) return fail(SP_E_INVALID, "quantiles: entry index out of range");
  }
  const size_t need = rsz<int32_t>(n) * 2 + rsz<double>(n) + rsz<double>(total) * 2 +
                      rsz<int32_t>(total);
  int rc = SP_OK;
  void* io = ctx_io(ctx, need, &rc);
  if (!io) return rc;
  Bump b{(uint8_t*)io};
  cudaStream_t st = ctx->stream;
  int32_t* d_op = op ? b.take<int32_t>(n) : nullptr;
  int32_t* d_idx = b.take<int32_t>(n);
  double* d_obs = b.take<double>(n);
  double* d_out = b.take<double>(total);
  int32_t* d_cnt = b.take<int32_t>(total);
  double* d_sm = out_smooth ? b.take<double>(total) : nullptr;
  if (n > 0) {
    if (op) SP_CUDA(cudaMemcpyAsync(d_op, op, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_idx, idx, 4 * (size_t)n, cudaMemcpyHostToDevice, st));
    SP_CUDA(cudaMemcpyAsync(d_obs, obs, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
  }
  if (out_smooth)
    SP_CUDA(cudaMemcpyAsync(d_sm, out_smooth, 8 * total, cudaMemcpyHostToDevice, st));
  rc = quantile_launch(ctx, n_tables, tables, n, d_op, d_idx, d_obs, q, beta, d_out, d_cnt, d_sm);
  if (rc != SP_OK) return rc;
  if (out) SP_CUDA(cudaMemcpyAsync(out, d_out, 8 * total, cudaMemcpyDeviceToHost, st));
  if (out_count) SP_CUDA(cudaMemcpyAsync(out_count, d_cnt, 4 * total, cudaMemcpyDeviceToHost, st));
  if (out_smooth) SP_CUDA(cudaMemcpyAsync(out_smooth, d_sm, 8 * total, cudaMemcpyDeviceToHost, st));
  SP_CUDA(cudaStreamSynchronize(st));
  return SP_OK;
}
