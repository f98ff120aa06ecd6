// sp_group.cu — single-process multi-GPU fan-out (SURVEY.md §8(b) Threading, §8(e)).
//
// The reference engine is one single-threaded Python process (configurator.py:368-373), so a
// drop-in that wants the eight GPUs of a box must fan out inside the library.  A group holds
// one context (device + non-blocking stream) per member; a group table is one replica of the
// OpTable per member, kept bit-identical because every mutation (set_latency, feedback fold)
// is applied to every replica in the same order.  sp_group_select_batch splits the N
// invocations into contiguous shards — member g owns [g*N/G, (g+1)*N/G) — and every member
// reads its shard of the caller's host buffers and writes its decisions straight into the
// caller's output arrays at the shard's offset (zero-copy when the buffers are pinned and
// mapped, else the chunked staging pipeline), all members in flight at once, then waits for
// all of them.  No collective is needed: decisions land in host memory in global invocation
// order, which is what sp_select_batch returns on one device.
#include <algorithm>
#include <vector>

#include "sp_internal.cuh"

struct sp_group {
  std::vector<sp_ctx*> ctx;
  std::vector<int32_t> device;
};

struct sp_group_table {
  std::vector<sp_table*> rep;  // one replica per member
  int32_t M = 0, K = 0;
};

namespace {

// Restores the caller's current device when a group call returns.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int member_device(sp_group* g, int i) {
  cudaError_t e = cudaSetDevice(g->device[i]);
  return e == cudaSuccess ? SP_OK : sp::cuda_fail(e, "cudaSetDevice(group member)");
}

}  // namespace

using namespace sp;

extern "C" {

int sp_group_create(int32_t n, const int32_t* devices, sp_group** out) {
  if (!out || n < 1 || !devices) return fail(SP_E_INVALID, "group_create: bad argument");
  DeviceGuard guard;
  sp_group* g = new (std::nothrow) sp_group();
  if (!g) return fail(SP_E_NOMEM, "group_create: host allocation");
  for (int i = 0; i < n; ++i) {
    sp_ctx* c = nullptr;
    int rc = sp_ctx_create(devices[i], &c);
    if (rc != SP_OK) {
      for (sp_ctx* x : g->ctx) sp_ctx_destroy(x);
      delete g;
      return rc;
    }
    g->ctx.push_back(c);
    g->device.push_back(devices[i]);
  }
  *out = g;
  return SP_OK;
}

int sp_group_destroy(sp_group* g) {
  if (!g) return SP_OK;
  DeviceGuard guard;
  for (sp_ctx* c : g->ctx) sp_ctx_destroy(c);
  delete g;
  return SP_OK;
}

int32_t sp_group_size(const sp_group* g) { return g ? (int32_t)g->ctx.size() : 0; }

int sp_group_member(sp_group* g, int32_t i, sp_ctx** ctx_out, int32_t* device_out) {
  if (!g || i < 0 || i >= (int)g->ctx.size()) return fail(SP_E_INVALID, "group_member: bad index");
  if (ctx_out) *ctx_out = g->ctx[i];
  if (device_out) *device_out = g->device[i];
  return SP_OK;
}

int64_t sp_group_launch_count(const sp_group* g) {
  int64_t n = 0;
  if (g)
    for (sp_ctx* c : g->ctx) n += sp_ctx_launch_count(c);
  return n;
}

int sp_group_table_create(sp_group* g, int32_t M, const double* lat, const double* lat_init,
                          const double* res, const int32_t* batch, const double* pool,
                          const double* price, const int32_t* kind, const int32_t* id_rank,
                          int32_t K, int32_t ref_index, sp_group_table** out) {
  if (!g || !out) return fail(SP_E_INVALID, "group_table_create: null argument");
  DeviceGuard guard;
  sp_group_table* t = new (std::nothrow) sp_group_table();
  if (!t) return fail(SP_E_NOMEM, "group_table_create: host allocation");
  t->M = M;
  t->K = K;
  for (size_t i = 0; i < g->ctx.size(); ++i) {
    int rc = member_device(g, (int)i);
    sp_table* r = nullptr;
    if (rc == SP_OK)
      rc = sp_table_create(g->ctx[i], M, lat, lat_init, res, batch, pool, price, kind, id_rank, K,
                           ref_index, &r);
    if (rc != SP_OK) {
      for (size_t j = 0; j < t->rep.size(); ++j) {
        cudaSetDevice(g->device[j]);
        sp_table_destroy(g->ctx[j], t->rep[j]);
      }
      delete t;
      return rc;
    }
    t->rep.push_back(r);
  }
  *out = t;
  return SP_OK;
}

int sp_group_table_destroy(sp_group* g, sp_group_table* t) {
  if (!g || !t) return SP_OK;
  DeviceGuard guard;
  for (size_t i = 0; i < t->rep.size(); ++i) {
    cudaSetDevice(g->device[i]);
    sp_table_destroy(g->ctx[i], t->rep[i]);
  }
  delete t;
  return SP_OK;
}

int sp_group_table_replica(sp_group_table* t, int32_t i, sp_table** out) {
  if (!t || !out || i < 0 || i >= (int)t->rep.size())
    return fail(SP_E_INVALID, "group_table_replica: bad index");
  *out = t->rep[i];
  return SP_OK;
}

int sp_group_table_set_latency(sp_group* g, sp_group_table* t, int32_t n, const int32_t* idx,
                               const double* val) {
  if (!g || !t) return fail(SP_E_INVALID, "group_set_latency: null argument");
  DeviceGuard guard;
  for (size_t i = 0; i < t->rep.size(); ++i) {
    int rc = member_device(g, (int)i);
    if (rc == SP_OK) rc = sp_table_set_latency(g->ctx[i], t->rep[i], n, idx, val);
    if (rc != SP_OK) return rc;
  }
  return SP_OK;
}

int sp_group_table_get_latency(sp_group* g, sp_group_table* t, int32_t member, double* out_lat) {
  if (!g || !t || member < 0 || member >= (int)t->rep.size())
    return fail(SP_E_INVALID, "group_get_latency: bad argument");
  DeviceGuard guard;
  int rc = member_device(g, member);
  if (rc != SP_OK) return rc;
  return sp_table_get_latency(g->ctx[member], t->rep[member], out_lat);
}

int sp_group_select_batch(sp_group* g, int32_t n_tables, sp_group_table* const* tables,
                          double alpha, int32_t N, const int32_t* op, const double* slack,
                          const int32_t* avail, const int32_t* supply, const int32_t* min_batch,
                          const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                          int32_t* out_fill, double* out_obj, double* out_slack,
                          double* out_wait, double* out_kind_min, int32_t mode) {
  if (!g || !tables || n_tables < 1 || N < 0) return fail(SP_E_INVALID, "group_select: bad argument");
  for (int t = 0; t < n_tables; ++t)
    if (!tables[t]) return fail(SP_E_INVALID, "group_select: null table");
  const int G = (int)g->ctx.size();
  const int K = tables[0]->K;
  DeviceGuard guard;
  std::vector<sp_table*> rep((size_t)n_tables);
  int rc = SP_OK, first_err = SP_OK;
  std::vector<bool> started((size_t)G, false);
  for (int m = 0; m < G && first_err == SP_OK; ++m) {
    const int64_t a = (int64_t)N * m / G, b = (int64_t)N * (m + 1) / G;
    const int n = (int)(b - a);
    if (n == 0) continue;
    for (int t = 0; t < n_tables; ++t) rep[t] = tables[t]->rep[m];
    rc = member_device(g, m);
    if (rc == SP_OK)
      rc = select_batch_impl(
          g->ctx[m], n_tables, rep.data(), alpha, n, op ? op + a : nullptr, slack + a * K,
          avail + a, supply + a, min_batch + a, flags + a, out_idx + a, out_code + a,
          out_fill ? out_fill + a : nullptr, out_obj ? out_obj + a : nullptr,
          out_slack ? out_slack + a : nullptr, out_wait ? out_wait + a : nullptr,
          out_kind_min ? out_kind_min + a * K : nullptr, mode, SP_MEM_HOST, false);
    if (rc != SP_OK) first_err = rc;
    started[m] = true;
  }
  // wait for every member that was started, even after an error, so that no kernel still
  // writes into the caller's buffers when this call returns
  for (int m = 0; m < G; ++m) {
    if (!started[m]) continue;
    cudaSetDevice(g->device[m]);
    rc = select_host_wait(g->ctx[m]);
    if (rc != SP_OK && first_err == SP_OK) first_err = rc;
  }
  return first_err;
}

int sp_group_feedback_fold(sp_group* g, int32_t n_tables, sp_group_table* const* tables,
                           int32_t n, const int32_t* op, const int32_t* idx, const double* obs,
                           double beta, int32_t dfp_count, int32_t dfp_on, int32_t fb_frozen) {
  if (!g || !tables || n_tables < 1) return fail(SP_E_INVALID, "group_fold: bad argument");
  DeviceGuard guard;
  std::vector<sp_table*> rep((size_t)n_tables);
  for (size_t m = 0; m < g->ctx.size(); ++m) {
    for (int t = 0; t < n_tables; ++t) {
      if (!tables[t]) return fail(SP_E_INVALID, "group_fold: null table");
      rep[t] = tables[t]->rep[m];
    }
    int rc = member_device(g, (int)m);
    if (rc == SP_OK)
      rc = sp_feedback_fold(g->ctx[m], n_tables, rep.data(), n, op, idx, obs, beta, dfp_count,
                            dfp_on, fb_frozen, SP_MEM_HOST);
    if (rc != SP_OK) return rc;
  }
  return SP_OK;
}

}  // extern "C"
