/*
 * slackpipe_b200.h — C-ABI of the B200-native configuration-optimizer hot path.
 *
 * The reference (`slackpipe`, arXiv 2102.01887 "Llama") has no FFI: its hot path is
 * in-process Python + numpy in /root/reference/pkg/src/slackpipe/configurator.py and
 * manager.py.  Every entry point below replaces one reference interface (cited per
 * function).  The Python host mirror (paper_2102_01887_b200/configurator.py) binds these
 * through ctypes with the same class/function names as the reference; INTEGRATION.md shows
 * the binding a maintainer of the reference would add.
 *
 * Conventions
 *   - Every function returns SP_OK (0) or a negative SP_E* code; the message is available
 *     from sp_last_error().  No C++ exception crosses this boundary.
 *   - All floating point is IEEE binary64 evaluated in exactly the reference's numpy order,
 *     with no FMA contraction (SURVEY.md §8 rules P1-P3), so results are bit-identical.
 *   - `mem` arguments say where the caller's I/O buffers live:
 *       SP_MEM_HOST   host pointers (pinned or pageable).  The library copies them to the
 *                     device, launches, copies results back and synchronises before it
 *                     returns (the reference-facing path; bench.py's `e2e`).
 *       SP_MEM_DEVICE device pointers (e.g. torch CUDA tensors' data_ptr()).  Work is
 *                     stream-ordered on the context stream and the call returns without
 *                     synchronising (bench.py's device-resident `value`).
 *   - A context is bound to one device and one stream and is not re-entrant.
 */
#ifndef SLACKPIPE_B200_H
#define SLACKPIPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_OK 0
#define SP_E_INVALID (-1)   /* maps to Python ValueError   */
#define SP_E_CUDA (-2)      /* CUDA runtime / launch error  */
#define SP_E_NOMEM (-3)     /* device or host allocation    */
#define SP_E_UNSUPPORTED (-4)
#define SP_E_RUNTIME (-5)   /* maps to Python RuntimeError */

#define SP_MEM_HOST 0
#define SP_MEM_DEVICE 1

/* decision codes (out_code bits 0-1) — OpTable.select return shapes (configurator.py:239-300) */
#define SP_DEC_NONE 0      /* select returned None (configurator.py:266-267) */
#define SP_DEC_ASSIGN 1    /* Decision(kind="assign") (configurator.py:293-300) */
#define SP_DEC_DELAY 2     /* Decision(kind="delay")  (configurator.py:278-286) */
#define SP_DEC_FEASIBLE 4  /* bit 2: decision-time SLO flag L(x*) < slack[kind(x*)] (configurator.py:226) */
#define SP_DEC_ERROR 3     /* the reference raises here: a NaN score leaves _argmin's tie set empty
                              (configurator.py:233-236, min() of an empty sequence -> ValueError) */

/* per-invocation flags word (in_flags) */
#define SP_FLAG_ALLOW_DELAY 1u       /* bit 0: allow_delay (configurator.py:245) */
#define SP_FLAG_EXCL_SHIFT 8         /* bits 8..31: excluded_kinds as a mask over the K kinds */

/* select modes */
#define SP_MODE_AUTO 0   /* staircase kernel when the table's plan allows it, else scan */
#define SP_MODE_PLAN 1   /* K2b: staircase (sorted prefix-min) decision kernel */
#define SP_MODE_SCAN 2   /* K2a: brute-force fused scan over every entry */

#define SP_MAX_KINDS 24        /* backend kinds of a table (the reference has no limit; the
                                  excluded-kind mask of the flags word holds 24) */
#define SP_MAX_PLAN_KINDS 8    /* the staircase plan's limit; tables with more kinds are decided
                                  by the literal scan */
#define SP_MAX_BATCH_VALUES 16

typedef struct sp_ctx sp_ctx;
typedef struct sp_table sp_table;
typedef struct sp_dag sp_dag;

/* ---- context ---------------------------------------------------------------------- */
int sp_version(void);
/* device: CUDA ordinal.  The context owns a non-blocking stream unless sp_ctx_set_stream
 * installs a caller stream (cudaStream_t passed as void*). */
int sp_ctx_create(int device, sp_ctx** out);
int sp_ctx_destroy(sp_ctx* ctx);
int sp_ctx_set_stream(sp_ctx* ctx, void* stream);
int sp_ctx_synchronize(sp_ctx* ctx);
/* Dispatch variants of this context (read once from the environment at creation; names are the
 * variables: SP_ZERO_COPY, SP_PIPE_CHUNKS, SP_K1_CERT (0 auto / 1 off / 2 force), SP_K1C_LANES
 * (lanes per instance of the certified slack pass: 4 default / 2), SP_FOLD_LEGACY, SP_NO_PDL,
 * SP_PLAN_LEGACY, SP_K2_VARIANT, ... — see sp_internal.cuh Options).  For tests and tools. */
int sp_ctx_set_option(sp_ctx* ctx, const char* name, int64_t value);
/* Last error message of this thread (ctx may be NULL). */
const char* sp_last_error(const sp_ctx* ctx);
/* Kernels launched through this context since creation (evidence for bench gpu_launches). */
int64_t sp_ctx_launch_count(const sp_ctx* ctx);

/* ---- profile tables: OpTable (configurator.py:159-213) ------------------------------ */
/* Replaces OpTable.__init__ (configurator.py:166-209).  Arrays are the OpTable SoA after
 * filtering (host, length M): lat = latency_s, lat_init = latency_initial_s,
 * res = resource_request, batch = batch_size, pool/price = backend pool_resources /
 * price_rate, kind = index of backend_kind in the caller's global kind list (0..K-1),
 * id_rank = rank of config_id in Python str order (configurator.py:195-198).
 * ref_index = OpTable.ref_index (-1 when the reference is unschedulable). */
int sp_table_create(sp_ctx* ctx, int32_t M, const double* lat, const double* lat_init,
                    const double* res, const int32_t* batch, const double* pool,
                    const double* price, const int32_t* kind, const int32_t* id_rank,
                    int32_t K, int32_t ref_index, sp_table** out);
int sp_table_destroy(sp_ctx* ctx, sp_table* t);
/* OpTable.set_latency (configurator.py:211-213), batched: lat[idx[i]] = val[i] in order. */
int sp_table_set_latency(sp_ctx* ctx, sp_table* t, int32_t n, const int32_t* idx,
                         const double* val);
/* Copy the live device latency vector (length M) to host memory (OpTable.lat). */
int sp_table_get_latency(sp_ctx* ctx, sp_table* t, double* out_lat);
/* Build (or reuse) the per-alpha decision plan: cost/costpen precompute + staircase
 * index.  Called implicitly by the select entry points. */
int sp_table_prepare(sp_ctx* ctx, sp_table* t, double alpha);
/* Mark every plan of the table stale (as a latency change does) without touching the table:
 * the next select / prepare rebuilds its plan (bench: plan-inclusive timing). */
int sp_table_invalidate(sp_ctx* ctx, sp_table* t);
/* 1 when the table's staircase plan is available (<= 16 distinct batch sizes, M < 32767). */
/* Make the plans of n alphas current for the table's version (OpTable.scores' alpha,
 * configurator.py:219-227): stale staircase plans are rebuilt together, up to four per launch
 * (one thread-block cluster each) — e.g. the alphas a sweep decides with after one table change. */
int sp_table_prepare_many(sp_ctx* ctx, sp_table* t, int32_t n, const double* alphas);
int sp_table_plan_supported(const sp_table* t);
/* Plan byte size for alpha after sp_table_prepare (synchronises); for DESIGN/bench. */
int sp_table_plan_bytes(sp_ctx* ctx, sp_table* t, double alpha, int64_t* out_bytes);

/* Diagnostic: (re)build the plan for alpha with builder 0 = the context's default, 1 = the
 * multi-kernel builder, 2 = the one-kernel cluster builder (3 = no rebuild: the current plan, e.g.
 * one sp_table_prepare_many built), and copy its byte image (total
 * bytes in *out_bytes; copied when cap is large enough).  Tests compare the builders and the
 * CPU restatement oracle/plan.py section by section. */
int sp_table_plan_image(sp_ctx* ctx, sp_table* t, double alpha, int32_t builder, void* out,
                        int64_t cap, int64_t* out_bytes);

/* ---- Eq. 1 vector: OpTable.scores (configurator.py:219-227) -------------------------- */
/* slack_by_kind: K doubles (host).  Outputs length M (host, synchronous). */
int sp_scores(sp_ctx* ctx, sp_table* t, const double* slack_by_kind, double alpha,
              double* out_score, double* out_cost);

/* ---- K2: batched OpTable.select (configurator.py:239-300) --------------------------- */
/* For every invocation i (0..N-1) against table tables[op[i]] (op may be NULL: table 0):
 *   slack[i*K + k]  slack_by_kind for global kind k
 *   avail[i]        `available`       supply[i]   `upstream_supply`
 *   min_batch[i]    `min_batch`       flags[i]    SP_FLAG_* (allow_delay, excluded mask)
 * Outputs per invocation:
 *   out_idx   Decision.entry_index (-1 for None)      out_code SP_DEC_* | SP_DEC_FEASIBLE
 *   out_fill  Decision.fill                           out_obj  Decision.objective_value
 *   out_slack Decision.slack_s                        out_wait Decision.wait_budget_s
 *   out_kind_min (optional, N*K): per-kind unmasked min score, +inf for kinds absent from
 *             the table — the Eq. 3 operands of OpTable.affinity (configurator.py:302-318).
 * Any output pointer may be NULL except out_idx and out_code. */
int sp_select_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                    int32_t N, const int32_t* op, const double* slack, const int32_t* avail,
                    const int32_t* supply, const int32_t* min_batch, const uint32_t* flags,
                    int32_t* out_idx, int32_t* out_code, int32_t* out_fill, double* out_obj,
                    double* out_slack, double* out_wait, double* out_kind_min, int32_t mode,
                    int32_t mem);

/* OpTable.affinity (configurator.py:302-318) for N queries with HOST buffers in one call: the
 * unmasked per-kind minima of invocation i (table tables[op[i]], slack row i) and out[i] =
 * min_{k != q} minimum[k] / minimum[q], q = query_kind[i].  Queries whose kind is absent from
 * the table must be mapped to None by the caller (configurator.py:310-315).  Synchronous. */
int sp_affinity_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                      int32_t N, const int32_t* op, const double* slack, const int32_t* query_kind,
                      double* out, int32_t mode);

/* Eq. 3 epilogue of OpTable.affinity (configurator.py:302-318) on the device: for invocation i
 * and query kind q = query_kind[i], out[i] = min_{k != q} kind_min[i*K+k] / kind_min[i*K+q]
 * (kind_min as produced by sp_select_batch; +inf marks kinds absent from the table, so an
 * operation that runs only on q yields +inf exactly like the reference).  reserved must be
 * NULL.  The caller maps "q absent from the table" to None before calling. */
int sp_affinity_from_minima(sp_ctx* ctx, int32_t N, int32_t K, const double* kind_min,
                            const int32_t* query_kind, double* out, void* reserved,
                            int32_t mem);

/* ---- K1: Alg. 1 slack over a DAG (configurator.py:493-543, compute_slack 76-106) ----- */
/* A slack graph: V vertices in topological order (every pred index < vertex index),
 * predecessor CSR (pred_ptr V+1, pred_idx), val_idx[v] = which per-instance reference
 * latency the vertex carries, terminal[v] = 1 where a decomposed path may end (DAG sinks,
 * or suffix ends for an explicit path list).  sources[s] = vertex whose slack is wanted
 * (the operation itself, first element of its suffixes). */
int sp_dag_create(sp_ctx* ctx, int32_t V, const int32_t* pred_ptr, const int32_t* pred_idx,
                  const int32_t* val_idx, const uint8_t* terminal, int32_t n_src,
                  const int32_t* sources, sp_dag** out);
int sp_dag_destroy(sp_ctx* ctx, sp_dag* g);
/* For instance i: ref = ref_lat + i*ref_stride (ref_stride 0 = shared by all instances),
 * budget_k = (target[i] - now[i]) - Q[i*K+k]; out_slack[(i*n_src + s)*K + k] =
 * min over suffixes of (ref[own]/suffix_total) * budget_k, bit-identical to
 * Configurator.slack_by_kind / compute_slack.  out_ratio (optional, I*n_src*2) receives
 * (own/Tmax, own/Tmin). */
int sp_slack_batch(sp_ctx* ctx, sp_dag* g, int32_t I, const double* ref_lat,
                   int32_t ref_stride, const double* target, const double* now, int32_t K,
                   const double* Q, double* out_slack, double* out_ratio, int32_t mem);

/* ---- K1 -> K2 fused: slack of every source operation straight into its decision ----- */
/* For pipeline instance i and source s of g (tables[s] = that operation's table, n_tables =
 * n_src): the slack of sp_slack_batch (slack_k = (b_k >= 0 ? own/Tmax : own/Tmin) * b_k,
 * b_k = (target[i] - now[i]) - Q[i*K + k], configurator.py:526-543) is used as the
 * slack_by_kind of invocation d = i*n_src + s, decided exactly as sp_select_batch does with
 * avail[d], supply[d], min_batch[d], flags[d] (configurator.py:239-300).  Outputs per d as
 * in sp_select_batch; out_kslack (optional, N*K) receives the slack values.  One kernel when
 * every plan fits in shared memory with the vertex programs, else K1 then K2. */
int sp_slack_select_batch(sp_ctx* ctx, sp_dag* g, int32_t n_tables, sp_table* const* tables,
                          double alpha, int32_t I, const double* ref_lat, int32_t ref_stride,
                          const double* target, const double* now, int32_t K, const double* Q,
                          const int32_t* avail, const int32_t* supply, const int32_t* min_batch,
                          const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                          int32_t* out_fill, double* out_obj, double* out_slack,
                          double* out_wait, double* out_kslack, int32_t mem);

/* ---- Eq. 2: queueing_by_kind / estimate_queueing (configurator.py:109-119, 511-524) --- */
/* Ordered sequential sum per kind: out[k] = (sum_{j in [ptr[k],ptr[k+1])} cnt[j]*(lat[j]*res[j]))
 * / pool[k] when cnt != NULL (queueing_by_kind order), else sum of lat[j]*res[j]/pool[k]
 * (estimate_queueing order).  Host arrays, synchronous. */
int sp_queueing(sp_ctx* ctx, int32_t K, const int32_t* ptr, const double* lat,
                const double* res, const int32_t* cnt, const double* pool, double* out);

/* ---- K3: feedback fold (manager.py:436-457, configurator.py:463-491) ---------------- */
/* Folds n observations (in completion order) into the tables: for observation j on table
 * tables[op[j]], entry idx[j], value obs[j] (idx[j] < 0 marks "no observation" and is skipped,
 * so a decision batch's out_idx can be passed straight through):
 *   completed_ref += (idx == ref_index);  obs_count[idx] += 1;
 *   unless fb_frozen: lat[idx] = beta*obs + (1-beta)*lat[idx]            (manager.py:45-47)
 *   if idx == ref_index && completed_ref == dfp_count && dfp_on:        (manager.py:449-457)
 *       every entry never observed so far (obs_count == 0), except the reference, gets
 *       lat = lat_init * (lat[ref] / lat_init[ref])                   (configurator.py:470-491)
 * Bit-identical to the sequential reference loop.  out_ref_lat (optional, n_tables) gets the
 * final reference latency (Configurator._ref_latency refresh, configurator.py:466-468). */
int sp_feedback_fold(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, int32_t n,
                     const int32_t* op, const int32_t* idx, const double* obs, double beta,
                     int32_t dfp_count, int32_t dfp_on, int32_t fb_frozen, int32_t mem);
/* Percentile estimate of an observation batch (extension: the reference has no percentile,
 * SURVEY.md §8(c); pinned to numpy).  Entries are numbered across the tables (table t's entry e
 * is tables[0..t-1] sizes + e).  out[e] = np.quantile(observations of e, q,
 * method="inverted_cdf") (NaN when e has none), out_count[e] = #observations; out_smooth
 * (optional, in/out) <- beta * out[e] + (1 - beta) * out_smooth[e] for observed entries
 * (initialised to out[e] where it holds NaN).  idx[j] < 0 = no observation.  0 <= q <= 1. */
int sp_observation_quantiles(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, int32_t n,
                             const int32_t* op, const int32_t* idx, const double* obs, double q,
                             double beta, double* out, int32_t* out_count, double* out_smooth,
                             int32_t mem);
/* Per-table counters maintained by sp_feedback_fold (host out). */
int sp_table_get_counters(sp_ctx* ctx, sp_table* t, int32_t* completed_ref,
                          int32_t* out_obs_count /* M, may be NULL */);
int sp_table_set_counters(sp_ctx* ctx, sp_table* t, int32_t completed_ref,
                          const int32_t* obs_count /* M, may be NULL */);

/* ---- batched commit step: Configurator.pump_commits rounds (configurator.py:657-756) ---- */
/* head_flags bits and policy bits */
#define SP_HEAD_PRESENT 1u  /* the op's speculative queue has a head (configurator.py:708-711) */
#define SP_HEAD_FORCED 2u   /* the head is a warm-up (DFP) invocation: head.forced            */
#define SP_COMMIT_FIFO 1    /* "pbc" ablation: key = (invocation_id,)   (configurator.py:716)  */
#define SP_COMMIT_ESLC 2    /* "eslc" ablation: commit the speculated entry (676-680)          */
/* R independent rounds over the same n_ops operations (tables[j] = op j, n_ops <= 64, the
 * reference's `for op in self.tables` order).  Per (round r, op j), i = r*n_ops + j:
 *   slack[i*K + k]  Configurator.slack_by_kind(op)[kind k]     head_fill[i]  head.fill
 *   buffered[i]     buffered_count(op)                          head_id[i]    invocation_id
 *   head_flags[i]   SP_HEAD_*                                   spec_idx/spec_slack/spec_obj[i]
 *                   head.spec_eidx / spec_slack_s / spec_objective (read under SP_COMMIT_ESLC)
 * depth[j] = PipelineDag.depths()[op]; full_mask[r] = kinds whose commit queue is saturated.
 * Outputs per (r, j): the _commit_candidate result (configurator.py:657-691) — out_idx entry
 * (-1 = None), out_fill fill target, out_slack, out_obj (NaN for forced heads) — and
 * out_aff the Eq. 3 affinity of the candidate's kind (NaN when not part of the key); per
 * round out_best[r] = index j of the op whose head the round commits (the minimum priority
 * key, configurator.py:713-728), or -1 when no op has a candidate. */
int sp_commit_round(sp_ctx* ctx, int32_t R, int32_t n_ops, sp_table* const* tables, double alpha,
                    const double* slack, const int32_t* head_fill, const int32_t* buffered,
                    const int64_t* head_id, const int32_t* depth, const uint32_t* head_flags,
                    const int32_t* spec_idx, const double* spec_slack, const double* spec_obj,
                    const uint32_t* full_mask, int32_t policy, int32_t* out_idx,
                    int32_t* out_fill, double* out_slack, double* out_obj, double* out_aff,
                    int32_t* out_best, int32_t mem);

/* ---- speculation loop ------------------------------------------- */
#define SP_SPEC_SDB 1           /* safe delayed batching on ("sdb" not ablated, 594)            */
#define SP_SPEC_FORCED 2        /* dfp warm-up: every decision is the reference entry (571-589)  */
#define SP_SPEC_HOLD_EXPIRED 4  /* a batching hold exists and its deadline has passed (597-599)  */

/* Replaces Configurator.speculate_from_buffer (configurator.py:563-620) for R independent
 * calls (one call = one operation's buffer).  Call r speculates operation op[r] (index into
 * `tables`, the run's OpTables) holding n_buf[r] buffered items:
 *   supply[r] = self._supply(op), now[r] = self._clock(), target[r] = self.target_s,
 *   rmin/rmax[r] = min/max of self._path_ratios(op) (Alg. 1),
 *   slack0[r*K + k] = self.slack_by_kind(op)[k] at entry (cached by weight version only, 526-529),
 *   flags[r] = SP_SPEC_*, pool[k] = self._pool[kind k];
 *   weights: the SQ (queue 0) and CQ (queue 1) dicts of every kind in their iteration order,
 *   entries w_ptr[(r*2 + q)*K + k] .. w_ptr[(r*2 + q)*K + k + 1] of (w_tab, w_eidx, w_count)
 *   = ((op, entry) key, count) — w_ptr has 2*K*R + 1 offsets.
 * Every later iteration recomputes Eq. 2 (511-524) and Alg. 1's slack (526-543) on the device
 * from the weights the call itself has updated (_weights_add, 553-561).  Outputs: the
 * invocations formed, in order, at out_off[r] .. out_off[r] + out_n[r] (the caller reserves
 * out_off[r+1] - out_off[r] >= n_buf[r] slots): out_idx entry, out_fill items, out_slack
 * Decision.slack_s, out_obj objective (NaN when forced); out_delay_idx[r] / out_delay_wait[r]
 * the delay decision that stopped the loop (-1 when the buffer emptied).  A call may touch any
 * number of weight keys. */
int sp_speculate_batch(sp_ctx* ctx, int32_t n_tables, sp_table* const* tables, double alpha,
                       int32_t K, const double* pool, int32_t R, const int32_t* op,
                       const int32_t* n_buf, const int32_t* supply, const double* now,
                       const double* target, const double* rmin, const double* rmax,
                       const double* slack0, const uint32_t* flags, const int32_t* w_ptr,
                       const int32_t* w_tab, const int32_t* w_eidx, const int32_t* w_count,
                       const int32_t* out_off, int32_t* out_idx, int32_t* out_fill,
                       double* out_slack, double* out_obj, int32_t* out_n, int32_t* out_delay_idx,
                       double* out_delay_wait, int32_t mem);

/* ---- simulated backend: observation records of a decision batch (backend.py:36-58) ------ */
/* Device buffers, stream-ordered.  For decision i: when (code[i] & 3) == SP_DEC_ASSIGN the
 * configuration runs and obs_idx[i] = idx[i], obs[i] = (truth_base[idx] +
 * truth_per_item[idx] * fill[i]) * noise[i] (draw_actual_latency with the caller's
 * multiplicative noise exp(N(0, sigma))); otherwise obs_idx[i] = -1 (nothing runs this batch).
 * truth_per_item may be NULL (no per-item term).  The records feed sp_feedback_fold directly. */
int sp_simulate_observations(sp_ctx* ctx, int32_t N, const int32_t* code, const int32_t* idx,
                             const int32_t* fill, const double* truth_base,
                             const double* truth_per_item, const double* noise, int32_t* obs_idx,
                             double* obs);
/* sp_simulate_observations + sp_feedback_fold of one table in ONE cooperative kernel (device
 * buffers, stream-ordered): the fold's load phase evaluates each decision's observation itself
 * (same law, same bits) and also writes the records to rec_idx / rec_obs. */
int sp_simulate_and_fold(sp_ctx* ctx, sp_table* t, int32_t N, const int32_t* code,
                         const int32_t* idx, const int32_t* fill, const double* truth_base,
                         const double* truth_per_item, const double* noise, double beta,
                         int32_t dfp_count, int32_t dfp_on, int32_t fb_frozen, int32_t* rec_idx,
                         double* rec_obs);

/* ---- profile generation (replaces profiler.py:35-85
 *      profile_operation's latency loop over pipeline.py:454-475 enumerate_configs) --------- */
/* Host buffers, synchronous.  The knob template's cross product in the reference's
 * enumeration order (kinds in the given (sorted) order; per kind its n_res[k] resource options
 * from res_opts (concatenated); the n_batch ascending batch sizes; the knob values in template
 * order, last knob fastest) — n_out = sum_k n_res[k] * n_batch * prod(knob_counts) entries.
 * Per entry the ground-truth law of scenario.py:68-77 / backend.py:52-58 per kind k:
 *   lat = base_seconds[k] * (R / ref_resource[k]) ** -resource_exponent[k] (when nonzero)
 *         * B ** batch_exponent[k] * multipliers[k][knob j][value] (row of sum(knob_counts),
 *         1.0 when the scenario has none) ;  draw = lat + per_item_seconds[k] * B
 *   out_lat = (sum over samples of draw * noise[i*S+s] * straggle[i*S+s]) / samples
 * with noise / straggle the reference's RNG factors (exp(N(0, sigma)), straggle_factor or 1.0)
 * or NULL (factor 1).  `**` is the correctly rounded power (see sp_profile.cu).  out_kind /
 * out_res / out_batch (optional) receive each entry's kind index, resource and batch size. */
int sp_profile_configs(sp_ctx* ctx, int32_t K, const int32_t* n_res, const int32_t* res_opts,
                       const double* base_seconds, const int32_t* ref_resource,
                       const double* resource_exponent, const double* batch_exponent,
                       const double* per_item_seconds, int32_t n_batch, const int32_t* batch_sizes,
                       int32_t n_knobs, const int32_t* knob_counts, const double* multipliers,
                       int32_t samples, const double* noise, const double* straggle, int64_t n_out,
                       double* out_lat, int32_t* out_kind, int32_t* out_res, int32_t* out_batch);
/* Correctly rounded x[i] ** y[i] on the device (host buffers; the power of the profile law). */
int sp_pow_correctly_rounded(sp_ctx* ctx, int32_t n, const double* x, const double* y, double* out);

/* ---- single-process multi-GPU fan-out (SURVEY.md §8(b) Threading, §8(e)) ------------------ */
/* The reference engine is one single-threaded process (configurator.py:368-373); a drop-in
 * that uses the GPUs of a box fans out inside the library.  A group owns one context (device
 * + non-blocking stream) per member; devices may repeat (independent contexts on one GPU).
 * A group table is one OpTable replica per member, kept bit-identical because every mutation
 * (set_latency, feedback fold) is applied to every replica in the same order. */
typedef struct sp_group sp_group;
typedef struct sp_group_table sp_group_table;
int sp_group_create(int32_t n, const int32_t* devices, sp_group** out);
int sp_group_destroy(sp_group* g);
int32_t sp_group_size(const sp_group* g);
/* Member i's context and device (the context stays owned by the group). */
int sp_group_member(sp_group* g, int32_t i, sp_ctx** ctx_out, int32_t* device_out);
/* Kernels launched by every member context (bench evidence). */
int64_t sp_group_launch_count(const sp_group* g);
/* OpTable.__init__ (configurator.py:166-209) replicated on every member: same arguments as
 * sp_table_create. */
int sp_group_table_create(sp_group* g, int32_t M, const double* lat, const double* lat_init,
                          const double* res, const int32_t* batch, const double* pool,
                          const double* price, const int32_t* kind, const int32_t* id_rank,
                          int32_t K, int32_t ref_index, sp_group_table** out);
int sp_group_table_destroy(sp_group* g, sp_group_table* t);
/* Member i's replica (owned by the group table). */
int sp_group_table_replica(sp_group_table* t, int32_t i, sp_table** out);
/* OpTable.set_latency (configurator.py:211-213) on every replica, in member order. */
int sp_group_table_set_latency(sp_group* g, sp_group_table* t, int32_t n, const int32_t* idx,
                               const double* val);
/* Member `member`'s live latency vector (host out, synchronous). */
int sp_group_table_get_latency(sp_group* g, sp_group_table* t, int32_t member, double* out_lat);
/* Batched OpTable.select (configurator.py:239-300) over N invocations with HOST buffers, laid
 * out exactly as sp_select_batch's: member g decides the contiguous shard [g*N/G, (g+1)*N/G)
 * on its device and writes straight into the caller's outputs at that offset (zero-copy when
 * every buffer is pinned and mapped; else the staging pipeline); every member is in flight at
 * once and the call returns when all have finished.  Results equal sp_select_batch's bit for
 * bit. */
int sp_group_select_batch(sp_group* g, int32_t n_tables, sp_group_table* const* tables,
                          double alpha, int32_t N, const int32_t* op, const double* slack,
                          const int32_t* avail, const int32_t* supply, const int32_t* min_batch,
                          const uint32_t* flags, int32_t* out_idx, int32_t* out_code,
                          int32_t* out_fill, double* out_obj, double* out_slack,
                          double* out_wait, double* out_kind_min, int32_t mode);
/* sp_feedback_fold (manager.py:436-457) of one host observation stream into every replica. */
int sp_group_feedback_fold(sp_group* g, int32_t n_tables, sp_group_table* const* tables,
                           int32_t n, const int32_t* op, const int32_t* idx, const double* obs,
                           double beta, int32_t dfp_count, int32_t dfp_on, int32_t fb_frozen);

/* ---- replica-parallel run engine --------------------------------- */
/* One tuned pipeline run of the reference — PipelineRun.run_to_completion (manager.py:535-630)
 * over BackendSim (backend.py:125-269) and the Configurator's queues, speculation, commits and
 * feedback (configurator.py:368-772) — executed as a sequential discrete-event loop by one GPU
 * thread per replica.  Replicas share the run description (tables, DAG, fleet, parameters) and
 * differ in their trace (frames), latency target and RNG draws.  Every decision, the report and
 * the final latency tables equal the reference's run on the same inputs bit for bit. */
typedef struct sp_des sp_des;

/* Run description (built by the Python host from PipelineRun's constructor arguments). Ops are
 * in sorted-name order (the reference's table order, manager.py:259-261); kinds in the
 * scenario's backend order (Scenario.backend_kinds, scenario.py:139-140). */
typedef struct {
  int32_t n_ops, n_kinds, n_entries, n_attrs, n_cfg_ids;
  const int32_t* entry_off;      /* [n_ops+1] the op's OpTable entries (configurator.py:166-209) */
  const double* lat;             /* [n_entries] profiled latency (profile-scaled, manager.py:187-208) */
  const double* lat_init;        /* [n_entries] latency_initial_s (scaled) */
  const double* res;             /* [n_entries] resource request */
  const int32_t* batch;          /* [n_entries] batch size */
  const int32_t* kind;           /* [n_entries] kind index */
  const int32_t* id_rank;        /* [n_entries] rank of config_id within the op (configurator.py:195-198) */
  const int32_t* cfg_id;         /* [n_entries] index of the config_id string (configs_used counts strings) */
  const double* truth_base;      /* [n_entries] OpKindTruth.base_latency of the entry (scenario.py:68-77) */
  const double* truth_per_item;  /* [n_entries] per_item_seconds of the entry's (op, kind) */
  const int32_t* ref_index;      /* [n_ops] OpTable.ref_index (-1: reference unschedulable) */
  const double* ref_latency;     /* [n_ops] reference entry latency (the anchor when ref_index = -1) */
  const int32_t* succ_off;       /* [n_ops+1] CSR of sorted successors (pipeline.py:314-315) */
  const int32_t* succ;           /* [n_edges] */
  const int32_t* pred_attr;      /* [n_edges] branch predicate attribute (-1: none) (pipeline.py:283-295) */
  const int32_t* pred_cmp;       /* [n_edges] 0 <, 1 <=, 2 >, 3 >=, 4 ==, 5 != */
  const int32_t* pred_value;     /* [n_edges] */
  const int32_t* fanout_attr;    /* [n_ops] fan-out attribute of the destination (-1: one item) */
  const int32_t* suffix_off;     /* [n_ops+1] path suffixes containing the op (configurator.py:413-420) */
  const int32_t* suffix_ops;     /* per suffix: length, then the op indices */
  const int32_t* instances;      /* [n_kinds] instance_count */
  const int32_t* inst_resources; /* [n_kinds] resources_per_instance */
  const double* price;           /* [n_kinds] price_rate */
  const int32_t* cq_capacity;    /* [n_kinds] Configurator.cq_capacity (configurator.py:443-458) */
  double alpha, beta, timeout_factor, dispatch_overhead, straggle_factor;
  int32_t dfp_count;
  int32_t ablations;             /* bits: 1 fb, 2 dfp, 4 sdb, 8 eslc, 16 pbc (configurator.py:23) */
  int32_t draws;                 /* RNG draws made per start: 1 noise, 2 straggle, 4 failure (backend.py:52-57, 186) */
} sp_des_spec;

/* Per-replica result row (manager.py:577-630 RunReport inputs). status: 0 ok, 1-3 capacity,
 * 4 livelock (RuntimeError, manager.py:563), 5 speculate_fixed found no configuration
 * (RuntimeError, configurator.py:633-636), 6 non-finite score, 7 draw capacity, 8 weight
 * capacity, 9 buffer capacity, 10 event cap, 11 an execution of an entry without ground truth
 * (truth_base NaN: KeyError, scenario.py:97-101). */
typedef struct {
  double latency, cost, now;
  int32_t peak_slots, peak_heap;  /* most invocation slots / heap entries the replica held at once */
  int32_t status, met, completed, failures, duplicates, invocations, terminal_items, n_speculate,
      n_commit, configs_used, log_len, events, event_len, pad;
} sp_des_out;

/* One BackendSim.trace row (backend.py:207, 243): meta = event (0 start, 1 complete, 2 fail) |
 * backend kind << 2 | instance << 8. */
typedef struct {
  double t;
  int32_t iid, meta;
} sp_des_event;

/* One decision_log row (configurator.py:650-654, 746-749): meta = op | entry << 8 | commit << 30. */
typedef struct {
  double t, slack, obj;
  int32_t iid, meta;
} sp_des_log;

int sp_des_create(sp_ctx* ctx, const sp_des_spec* spec, sp_des** out);
int sp_des_destroy(sp_ctx* ctx, sp_des* des);
/* Run R replicas over n_traces traces: trace t is frames [frame_off[t], frame_off[t+1]) of
 * `attrs` (n_attrs ints per frame, 0 where the frame lacks the attribute); replica r runs trace
 * trace_of[r] (NULL: trace r, n_traces == R) with target target_s[r].
 * draw_factor / draw_bits (R x draw_cap, or NULL when spec.draws == 0): per start, in start order,
 * exp(N(0, sigma)) and bit0 straggled / bit1 will_fail from the replica's numpy stream.  log
 * (R x log_cap rows, optional), lat_out (R x n_entries final latencies, optional), out (R rows),
 * events (R x event_cap rows of the backend's event trace, optional).
 * mem: SP_MEM_HOST (copies in, launch, copies out, synchronises) or SP_MEM_DEVICE. */
int sp_des_run(sp_ctx* ctx, sp_des* des, int32_t R, int32_t n_traces, const int32_t* frame_off,
               const int32_t* attrs, const int32_t* trace_of, const double* target_s, int32_t draw_cap, const double* draw_factor,
               const uint8_t* draw_bits, int32_t log_cap, sp_des_log* log, double* lat_out,
               sp_des_out* out, int32_t event_cap, sp_des_event* events, int32_t mem);
/* Size the per-replica arenas for R replicas of these traces (host frame_off / attrs) and the
 * given draw / log capacities; sp_des_run with SP_MEM_DEVICE buffers requires it (the host-buffer
 * form calls it itself). */
int sp_des_prepare(sp_ctx* ctx, sp_des* des, int32_t R, int32_t n_traces, const int32_t* frame_off,
                   const int32_t* attrs, int32_t draw_cap, int32_t log_cap);
/* Invocation capacity per buffered item (default 1.25; retries and straggler duplicates add
 * invocations beyond one per item — a replica that runs out reports status 1). */
int sp_des_set_capacity(sp_des* des, double invocations_per_item);
/* Execution form: lanes = 1: one GPU thread per replica (the replicas of a warp diverge);
 * 2 / 4 / 8 / 16 / 32: that many lanes per replica (all lanes run the replica's serial engine, the
 * entry scans split across them; 32 = one warp per replica, ~17x lower latency per run than one
 * thread); 0 = default (32 lanes below 2,048 replicas, 8 below 32,768, else 2).  Results are
 * identical in every form. */
int sp_des_set_mode(sp_des* des, int32_t lanes);
/* The reference's per-start RNG draws of R runs (host, no GPU needed): replica r's numpy PCG64
 * state (state hi, lo, inc hi, lo in pcg_state[4r..4r+3], as default_rng(seed) sets it) and, per
 * start k < cap, in the reference's order (backend.py:52-57, 186): factor[r*cap+k] =
 * math.exp(rng.normal(0, noise_sigma)) (1 when noise_sigma is 0), bits[r*cap+k] bit 0 = straggled,
 * bit 1 = will fail.  Same bits as numpy + CPython. */
int sp_des_draws(int32_t R, const uint64_t* pcg_state, int32_t cap, double noise_sigma,
                 double straggle_rate, double failure_rate, double* factor, uint8_t* bits);
/* Bytes of one replica's arena as last prepared. */
int64_t sp_des_arena_bytes(sp_des* des);

#ifdef __cplusplus
}
#endif
#endif /* SLACKPIPE_B200_H */
