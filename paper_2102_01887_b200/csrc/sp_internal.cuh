// sp_internal.cuh — shared definitions of the slackpipe_b200 CUDA library (sm_100a).
//
// Numerics: every product/quotient/sum that the reference evaluates with numpy float64
// ufuncs is written with the explicit round-to-nearest intrinsics (__dmul_rn, __ddiv_rn,
// __dadd_rn, __dsub_rn) so that nvcc can never contract them into FMAs.
// The library is additionally compiled with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "slackpipe_b200.h"

namespace sp {

constexpr uint32_t kPlanMagic = 0x53504c4eu;  // "SPLN"
constexpr uint16_t kNone16 = 0xFFFFu;
constexpr int kMaxKinds = SP_MAX_PLAN_KINDS;    // plan / fused-kernel kind limit
constexpr int kMaxTableKinds = SP_MAX_KINDS;    // table kind limit (literal scan beyond 8)
constexpr int kMaxB = SP_MAX_BATCH_VALUES;

// One candidate record of the staircase plan (32 B).  Candidates live in ONE id space
// ordered by the reference's argmin key (score, cost, res, id_rank) = (score, r1): the
// feasible side of an entry carries score = cost, the infeasible side cost + penalty
// (configurator.py:224-237).  The first 16 B hold what the decision always needs, the
// second 16 B the winner's payload.
struct __align__(16) CandRec {
  double score;
  int32_t idx;
  int32_t feas;   // 1: feasible side (lat < slack), 0: penalized side
  double lat;
  int32_t batch;
  int32_t kind;
};
static_assert(sizeof(CandRec) == 32, "CandRec must be 32 bytes");
// In the plan image candidates are stored as three arrays indexed by unified id:
//   score[] (f64), lat[] (f64) and CandB (8 B) {idx | feas << 16 | kind << 17, batch}
struct __align__(8) CandB {
  uint32_t meta;   // entry index (15 bits) | feasible (bit 16) | kind (bits 17..19)
  int32_t batch;
};

constexpr int kMaxBuckets = 4096;   // per-kind threshold buckets
constexpr int kMaxLut = 4097;       // batch-lane lookup covers values 0..4096

// Per-kind section descriptor (32 B; the decision kernel reads the first 16 B + one word).
// Thresholds are positive latencies, so for a positive slack the high 32 bits of the IEEE
// encoding are a monotone key; buckets are (hi(s) - kmin_hi) >> shift, clamped.
struct __align__(16) KindDesc {
  uint32_t kmin_hi;    // high word of the smallest real threshold
  uint32_t nb1_shift;  // (buckets - 1) | shift << 16
  int32_t thr_off;     // byte offset of the threshold array (R doubles, thr[0] = -inf)
  int32_t rows_off;    // byte offset of the staircase rows (R x row_stride bytes)
  int32_t bkt_off;     // byte offset of the bucket table (u32: lo | cnt << 16)
  int32_t R;           // rows (0: kind absent from the table)
  int32_t pad[2];
};
static_assert(sizeof(KindDesc) == 32, "KindDesc must be 32 bytes");

// Plan header (512 B).  A plan is one contiguous, 16-B aligned byte image so that the
// decision kernel can stage it into shared memory with one bulk copy.
struct __align__(16) PlanHdr {
  uint32_t magic;
  int32_t total_bytes;  // whole image, multiple of 16
  int32_t M;
  int32_t nB;           // distinct batch sizes
  int32_t W;            // u16 lanes per row (8 or 16)
  int32_t K;            // global kind count
  int32_t ncp;          // feasible-side candidates
  int32_t ncs;          // penalized-side candidates
  int32_t score_off;    // byte offset of score[ncp + ncs] (f64)
  int32_t lat_off;      // byte offset of lat[ncp + ncs] (f64)
  int32_t recb_off;     // byte offset of CandB[ncp + ncs]
  int32_t row_stride;   // bytes per staircase row: u16 range minima for every batch-lane
                        // interval [lo, hi], at tri(lo) + hi - lo, tri(lo) = lo*nB - lo(lo-1)/2
  int32_t lut_off;      // u16 lut[v] = (#batch < v) | (#batch <= v) << 8, v in [0, lut_n)
  int32_t lut_n;        // max batch + 2, or 0 when the lookup table is not built
  int32_t pad0[2];
  int32_t batch_vals[kMaxB];  // ascending; unused = INT32_MAX
  KindDesc kd[kMaxKinds];
  int32_t pad1[32];
};
static_assert(sizeof(PlanHdr) == 512, "PlanHdr must be 512 bytes");

// Monotone u64 order key of a non-NaN double (x < y  <=>  key(x) < key(y), except that
// -0.0 orders below +0.0; thresholds are positive latencies so this never matters).
__host__ __device__ __forceinline__ uint64_t order_key(uint64_t u) {
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct Plan {
  double alpha = 0.0;
  uint64_t version = ~0ull;  // table version the plan was built for
  uint64_t cost_version = ~0ull;  // table version cost / costpen were computed for
  bool valid = false;
  // device buffers
  double* cost = nullptr;     // M
  double* costpen = nullptr;  // M
  uint8_t* image = nullptr;   // plan image (capacity image_cap)
  int64_t image_cap = 0;
  // host copy of the header, fetched asynchronously after each build (pinned + event);
  // single-table launches pass it as a kernel parameter once it has landed
  PlanHdr* host_hdr = nullptr;
  cudaEvent_t hdr_ready = nullptr;
  bool hdr_pending = false;
  bool hdr_valid = false;
  // cluster builds write the header (and then the build's sequence number) straight into
  // mapped pinned memory: no copy or event between the build and the next kernel, so the
  // programmatic-dependent-launch chain build -> select stays intact
  volatile uint32_t* host_seq = nullptr;
  uint32_t seq = 0;
  bool hdr_mapped = false;
  // rebuilds after the first are replayed from a CUDA graph of the whole build (one launch
  // instead of ~12 kernel launches + 3 memory operations)
  int builds = 0;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
};

}  // namespace sp

namespace sp {
// Dispatch options of a context: read once from the environment when the context is created
// (variable names as below), changeable per context with sp_ctx_set_option.  Variants exist for
// the tests and the measurement tools; the defaults are the product path.
struct Options {
  int zero_copy = 1;         // SP_ZERO_COPY: pinned mapped host buffers read by the kernel
  int pipe_chunks = 0;       // SP_PIPE_CHUNKS: pageable staging chunks (0 = by size)
  int k1_cert = 0;           // SP_K1_CERT: 0 auto, 1 off ("0"), 2 force ("force")
  int k1c_lanes = 4;         // SP_K1C_LANES: lanes per instance of the certified pass (4 or 2)
  int fold_long_min = 0;     // SP_FOLD_LONG_MIN: long-segment threshold of the fold (0 = default)
  int fold_legacy = 0;       // SP_FOLD_LEGACY: multi-kernel fold (radix sort + 5 kernels)
  int stair_smem = 0;        // SP_STAIR_SMEM: multi-kernel builder, shared-memory staircase
  int stair_global = 0;      // SP_STAIR_GLOBAL: multi-kernel builder, global staircase
  int no_plan_graph = 0;     // SP_NO_PLAN_GRAPH: no CUDA-graph replay of plan builds
  int plan_legacy = 0;       // SP_PLAN_LEGACY: multi-kernel plan builder
  int pc_debug = 0;          // SP_PC_DEBUG: per-phase timestamps of the cluster builder
  int k2_plan_only = 0;      // SP_K2_VARIANT (any value but "fast"): generic K2b only
  int k2f_threads = 512;     // SP_K2F_THREADS: K2f block size (512 or 1024)
  int no_pdl = 0;            // SP_NO_PDL: no programmatic dependent launch (K2f, K2b, the
                             // cluster plan build, the fold, the observation kernel)
  int full_smem = 0;         // SP_FULL_SMEM: K2b requests the whole shared-memory budget
  int no_k12 = 0;            // SP_NO_K12: K1 then K2 instead of the fused kernel
  int k12_generic = 0;       // SP_K12_GENERIC: fused kernel without the K2f decision core
  int k12_outstage = 0;      // SP_K12_OUTSTAGE: staged decision stores in K12
  int k12_generic_dp = 0;    // SP_K12_GENERIC_DP: generic DP in K12 for path-list graphs
};
void options_from_env(Options& o);
int options_set(Options& o, const char* name, long long value);
}  // namespace sp

struct sp_ctx {
  int device = 0;
  sp::Options opt;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 0;
  int max_smem_optin = 0;
  int64_t launches = 0;
  // a plan image was (re)written by a kernel that no select launch has waited on yet: the
  // next K2f launch must not read any plan before its griddepcontrol.wait
  bool plan_dirty = true;

  // grow-only device arena for staged host I/O
  void* io_dev = nullptr;
  size_t io_cap = 0;
  // small device scratch for pointer tables
  void* ptr_dev = nullptr;
  size_t ptr_cap = 0;
  // pinned, mapped host staging for small host-buffer calls (one launch reads / writes it over
  // PCIe, no copy-engine operations)
  void* pin_host = nullptr;
  void* pin_dev = nullptr;
  size_t pin_cap = 0;
  // generic device scratch (sort temp etc.)
  void* tmp_dev = nullptr;
  size_t tmp_cap = 0;
  // host-buffer pipeline: H2D and D2H copy streams (full-duplex PCIe) + per-chunk events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  static constexpr int kPipeChunks = 8;
  cudaEvent_t ev_in[kPipeChunks] = {}, ev_comp[kPipeChunks] = {}, ev_out[kPipeChunks] = {};
  cudaStream_t capture = nullptr;  // private stream for CUDA-graph captures
  void* coop = nullptr;            // the cooperative fold's persistent buffers (sp_fold.cu)
};

struct sp_table {
  int32_t M = 0, K = 0, nB = 0, ref_index = -1;
  int32_t batch_vals[sp::kMaxB];
  int32_t kind_count[sp::kMaxTableKinds];
  int32_t kind_base[sp::kMaxTableKinds];  // entries sorted by kind: base offset per kind
  // entries whose latency is not finite (host mirror, per entry): the staircase plan and the
  // fused kernels need finite latencies; with any non-finite entry decisions take the literal
  // scan, which reproduces the reference's inf / NaN behaviour
  std::vector<uint8_t> nonfinite_entry;
  int32_t nonfinite = 0;
  bool tainted = false;  // a host fold may have produced non-finite latencies
  bool finite_safe() const { return nonfinite == 0 && !tainted; }
  bool plan_ok = false;
  uint64_t version = 0;
  int32_t completed_ref = 0;
  // device arrays (length M)
  double *lat = nullptr, *lat_init = nullptr, *res = nullptr, *pool = nullptr,
         *price = nullptr;
  int32_t *batch = nullptr, *bidx = nullptr, *kind = nullptr, *id_rank = nullptr,
          *obs_count = nullptr;
  int32_t* kind_slot = nullptr;  // position of the entry inside its kind block (static order by kind, idx)
  // plan scratch (device)
  uint32_t *r1 = nullptr, *r2 = nullptr;
  // scratch of the plan's three entry-order sorts (tile + merged item buffers)
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  int32_t *ent_r1 = nullptr, *ent_r2 = nullptr, *order = nullptr;
  uint32_t *pf = nullptr, *sf = nullptr;      // W*(M+K) each
  uint32_t* rowscratch = nullptr;             // (M+K) * 2W
  double* thrscratch = nullptr;               // M+K
  int32_t* rows_per_kind = nullptr;           // K (+1 status word)
  int32_t* dev_counters = nullptr;            // [0] = completed_ref (device copy); [4] = the
                                              // cached latency order is stale as a whole
  // per entry: the latency changed since the cluster plan builder last sorted its cached
  // per-segment latency order (set by every device writer of lat, cleared by the builder)
  uint8_t* dirty = nullptr;
  uint32_t *candf = nullptr, *cands = nullptr;  // M flags each
  uint32_t *cidf = nullptr, *cids = nullptr;    // M maps each
  int2* fin_chunk = nullptr;  // 2 x ceil(M / 256): per-chunk candidate counts, then bases
  // per position of the kind-major latency order: {r1, r2}, lane | new-latency << 7, latency
  // (gathered by a wide kernel so the one-CTA-per-kind staircase reads them coalesced)
  uint2* pos_r12 = nullptr;
  uint8_t* pos_meta = nullptr;
  double* pos_lat = nullptr;
  double* ukey = nullptr;                       // 2M: unified candidate scores (CP then CS)
  uint32_t* ukr = nullptr;                      // 2M: unified candidate r1 ranks
  int32_t* uent = nullptr;                      // 2M: unified candidate entry index
  uint32_t* umap = nullptr;                     // 2M: candidate -> unified id
  // one-kernel cluster builder (sp_plan_cluster.cu): static (kind, lane) segments + scratch
  bool pc_ok = false;
  int32_t pc_nseg = 0, pc_max_seg = 0;
  int32_t pc_seg_lo[sp::kMaxKinds + 1] = {};
  void* pc_seg = nullptr;
  int32_t* pc_seg_ent = nullptr;
  void* pc_scratch = nullptr;
  size_t pc_scratch_bytes = 0;
  // multi-plan builds (plan_prepare_many): private scratch / thresholds of plans 1..3, the
  // per-plan status words and the new cached order
  void* pc_multi_scratch[3] = {};
  double* pc_multi_thr[3] = {};
  int32_t* pc_multi_status = nullptr;
  int32_t* pc_multi_ord = nullptr;
  std::vector<sp::Plan> plans;
};

struct sp_dag {
  int32_t V = 0, n_src = 0, n_val = 0;
  // Per-source vertex programs: prog[prog_ptr[s] .. prog_ptr[s+1]) lists
  // source s and then its descendants in topological order as int4
  //   {value index, out slot | terminal << 16, pred offset, pred groups}.
  // Slots are DP registers reused once every reader of a value has run (liveness), so a
  // lane needs max_slots of them.  preds[pred_ptr[s] ..] holds the source's predecessor
  // slots, each vertex's list padded to an even length by repeating its last entry
  // (max / min are idempotent); the pred offset is relative to pred_ptr[s].  The kernel
  // turns slots into shared-memory byte offsets when it stages the program.
  int4* prog = nullptr;         // device
  int32_t* prog_ptr = nullptr;  // device, n_src + 1
  uint32_t* preds = nullptr;    // device
  int32_t* pred_ptr = nullptr;  // device, n_src + 1
  int32_t max_span = 0;         // max program length
  int32_t max_slots = 0;        // max live DP values per lane
  int32_t max_preds = 0;        // max padded pred entries of one source
  int64_t prog_len = 0, pred_len = 0;
  // every program entry after a source has exactly one predecessor (path-list tries): the DP
  // is a chain of sums (K12 takes a lean loop)
  int32_t single_pred = 0;
  // Certified backward form (sp_slack.cu, k_slack_cert): one byte image, staged whole into
  // shared memory — group_ptr u16[V+1] | vidx u16[V] | term u8[V] | src u8[n_src] |
  // succ u16[4 * groups] (successor byte offsets node * 256, each list padded to a multiple of
  // four with the sentinel node V), 16-byte aligned sections.  Present when V <= kCertMaxV and the per-source programs are
  // long enough (Σ_s |E(desc s)|) for the backward pass to pay.
  uint8_t* cert = nullptr;  // device
  int32_t cert_bytes = 0, E = 0;
  int32_t off_vidx = 0, off_term = 0, off_src = 0, off_succ = 0;
};
constexpr int kCertMaxV = 253;  // node ids 0..252; 0xFE = no option, 0xFF = path ends here

// ---- error plumbing ------------------------------------------------------------------
namespace sp {
// Kernel attributes (cudaFuncSetAttribute) belong to the current device's context: a
// once-per-process flag would leave the other devices of a multi-GPU group unconfigured.
// attr_once(mask) is true the first time it is called on each device.
inline bool attr_once(uint64_t& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}
// Every ctx entry point runs on the context's device and restores the caller's current
// device on return (several contexts / a DeviceGroup may live in one process).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (dev < 0) return;
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & 63;
}
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
}  // namespace sp

#define SP_CUDA(call)                                              \
  do {                                                             \
    cudaError_t _e = (call);                                       \
    if (_e != cudaSuccess) return sp::cuda_fail(_e, #call);        \
  } while (0)

#define SP_STR2(x) #x
#define SP_STR(x) SP_STR2(x)
#define SP_CHECK_LAUNCH(ctx)                                                              \
  do {                                                                                    \
    (ctx)->launches++;                                                                    \
    cudaError_t _e = cudaGetLastError();                                                  \
    if (_e != cudaSuccess)                                                                \
      return sp::cuda_fail(_e, "kernel launch (" __FILE__ ":" SP_STR(__LINE__) ")");     \
  } while (0)

// ---- internal entry points implemented in the .cu files --------------------------------
namespace sp {
int plan_build(sp_ctx* ctx, sp_table* t, Plan& p);
int plan_scratch_alloc(sp_table* t);
int plan_cluster_prepare(sp_table* t, const int32_t* kind, const int32_t* bidx);
int plan_cluster_launch_multi(sp_ctx* ctx, sp_table* t, Plan* const* ps, int n, int W,
                              const PlanHdr& hdr, int32_t* status, void* const* scratch,
                              double* const* thr, int32_t* ord_new);
int plan_prepare_many(sp_ctx* ctx, sp_table* t, int n, const double* alphas);
void coop_release(sp_ctx* ctx);
int simulate_and_fold(sp_ctx* ctx, sp_table* t, int n, const int32_t* code, const int32_t* idx,
                      const int32_t* fill, const double* base, const double* per_item,
                      const double* noise, double beta, int dfp_count, int dfp_on, int fb_frozen,
                      int32_t* rec_idx, double* rec_obs);
int plan_cluster_launch(sp_ctx* ctx, sp_table* t, Plan& p, int W, const PlanHdr& hdr,
                        int32_t* status, PlanHdr* host_hdr, uint32_t* host_seq, uint32_t seq);
Plan* plan_get(sp_ctx* ctx, sp_table* t, double alpha, int* rc);
Plan* plan_costs(sp_ctx* ctx, sp_table* t, double alpha, int* rc);
bool plan_ready(sp_table* t, double alpha);
const PlanHdr* plan_host_header(Plan& p);  // nullptr until the async copy has landed
int plan_header_wait(sp_ctx* ctx, Plan& p);  // block until the header has landed
void plan_release(Plan& p);
int select_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, double alpha, int N,
                  const int32_t* op, const double* slack, const int32_t* avail,
                  const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                  int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                  double* out_slack, double* out_wait, double* out_kind_min, int mode);
int affinity_launch(sp_ctx* ctx, int N, int K, const double* kmin, const int32_t* q,
                    double* out);
int slack_select_launch(sp_ctx* ctx, sp_dag* g, int n_tables, sp_table* const* tables,
                        double alpha, int I, const double* ref, int ref_stride,
                        const double* target, const double* now, int K, const double* Q,
                        const int32_t* avail, const int32_t* supply, const int32_t* min_batch,
                        const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                        int32_t* out_fill, double* out_obj, double* out_slack, double* out_wait,
                        double* out_kslack);
int commit_launch(sp_ctx* ctx, int R, int n_ops, sp_table* const* tables, double alpha,
                  const double* slack, const int32_t* fill, const int32_t* buffered,
                  const long long* head_id, const int32_t* depth, const uint32_t* hflags,
                  const int32_t* spec_idx, const double* spec_slack, const double* spec_obj,
                  const uint32_t* full_mask, int policy, void* scratch, int32_t* out_idx,
                  int32_t* out_fill, double* out_slack, double* out_obj, double* out_aff,
                  int32_t* out_best);
size_t commit_scratch_bytes(int R, int n_ops, int K);
int quantile_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n, const int32_t* op,
                    const int32_t* idx, const double* obs, double q, double beta, double* out,
                    int32_t* out_count, double* out_smooth);
int scores_launch(sp_ctx* ctx, sp_table* t, Plan* p, const double* slack_dev,
                  double* score_dev, double* cost_dev);
int speculate_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, double alpha, int K,
                     const double* pool, int R, const int32_t* op, const int32_t* n_buf,
                     const int32_t* supply, const double* now, const double* target,
                     const double* rmin, const double* rmax, const double* slack0,
                     const uint32_t* flags, const int32_t* w_ptr, const int32_t* w_tab,
                     const int32_t* w_eidx, const int32_t* w_count, const int32_t* out_off,
                     int32_t* out_idx, int32_t* out_fill, double* out_slack, double* out_obj,
                     int32_t* out_n, int32_t* out_delay_idx, double* out_delay_wait,
                     int n_weights = -1, int n_slots = -1);
int slack_launch(sp_ctx* ctx, sp_dag* g, int I, const double* ref, int ref_stride,
                 const double* target, const double* now, int K, const double* Q,
                 double* out_slack, double* out_ratio);
int queueing_launch(sp_ctx* ctx, int K, const int32_t* ptr, const double* lat,
                    const double* res, const int32_t* cnt, const double* pool, double* out);
int fold_launch(sp_ctx* ctx, int n_tables, sp_table* const* tables, int n, const int32_t* op,
                const int32_t* idx, const double* obs, double beta, int dfp_count, int dfp_on,
                int fb_frozen);
void* ctx_tmp(sp_ctx* ctx, size_t bytes, int* rc);
int select_batch_impl(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                      int32_t N, const int32_t* op, const double* slack, const int32_t* avail,
                      const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                      int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                      double* out_slack, double* out_wait, double* out_kind_min, int32_t mode,
                      int32_t mem, bool sync);
int select_host_wait(sp_ctx* ctx);
}  // namespace sp
