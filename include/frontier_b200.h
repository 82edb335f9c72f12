/*
 * frontier_b200.h -- C ABI of the B200-native batched Frontier simulation engine.
 *
 * One call simulates N independent instances (config x trace-seed points of a
 * design-space sweep) and returns one metric row per instance. The entry points
 * replace the reference's per-instance Python call chain:
 *
 *   run_one(config)                         pkg/src/frontier_sim/cli.py:82-102
 *     make_simulation(mode, deployment, requests, policy, af, routing, seed, ...)
 *                                            pkg/src/frontier_sim/orchestrator/__init__.py:43-50
 *     ServingSimulation.run() -> EventTrace  pkg/src/frontier_sim/orchestrator/base.py:220-229
 *     compute_metrics(trace, deployment)     pkg/src/frontier_sim/metrics.py:81-178
 *   _sweep_point / cmd_sweep                 pkg/src/frontier_sim/cli.py:197-275
 *
 * and the pure cost-model functions on the path:
 *
 *   CostModel.predict_attention (analytic)   pkg/src/frontier_sim/costmodel/model.py:313-321,
 *                                            costmodel/analytic.py:32-53
 *   route_tokens(policy="uniform")           pkg/src/frontier_sim/costmodel/routing.py:65-113
 *   moe_layer_latency                        pkg/src/frontier_sim/costmodel/moe.py:69-128
 *
 * Conventions
 *   - Plain pointers and sizes only; all structs are POD with explicit padding.
 *   - Calls are synchronous unless the name ends in _async. Host-buffer calls copy
 *     inputs to HBM, run, and copy results back (the drop-in path). _dev calls take
 *     device pointers (inputs already resident in HBM).
 *   - Return value: FS_OK or a call-level error; fs_last_error() has the text.
 *     Per-instance failures are reported in fs_metric_row.status, mirroring the
 *     exceptions the reference raises (the sweep's "failed: Type: msg" rows,
 *     cli.py:229-233).
 *   - An engine handle is bound to one CUDA device and is not re-entrant.
 */
#ifndef FRONTIER_B200_H
#define FRONTIER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 2

/* Limits of the device engine (checked by the host lowering; violations are
 * reported as FS_ERR_CAPACITY rather than silently truncated). */
#define FS_MAX_PREFIX_BYTES 192   /* "{seed}:{cluster_id}/{idx}:" router-seed prefix   */
#define FS_MAX_EXPERTS 1024       /* experts per MoE layer                              */
#define FS_MAX_TOPK 16            /* top_k of the register top-(k+1) lists; larger     
                                     top_k sorts whole rows (no limit below E)          */
#define FS_MAX_MICRO_BATCHES 64   /* AF micro-batches per step                         */
#define FS_MAX_REPLICAS 65536     /* replicas per instance (state spills to HBM)       */

enum fs_mode { FS_MODE_COLOCATED = 0, FS_MODE_PD = 1, FS_MODE_AF = 2 };

enum fs_role {               /* topology.py:33 CLUSTER_ROLES */
  FS_ROLE_COLOCATED = 0,
  FS_ROLE_PREFILL = 1,
  FS_ROLE_DECODE = 2,
  FS_ROLE_ATTENTION = 3,
  FS_ROLE_FFN = 4
};

enum fs_admission {          /* cluster.py:98 SchedulerPolicy.admission */
  FS_ADMIT_FCFS = 0,
  FS_ADMIT_FCFS_SKIP = 1,
  FS_ADMIT_PRIORITY = 2
};

enum fs_priority_key { FS_PRIO_PROMPT = 0, FS_PRIO_ARRIVAL = 1 };

enum fs_routing { FS_ROUTE_UNIFORM = 0, FS_ROUTE_DIRICHLET = 1, FS_ROUTE_TRACE = 2 };

/* Per-instance status. Names follow the exception the reference raises. */
enum fs_status {
  FS_OK = 0,
  FS_ERR_REQUEST_CANNOT_FIT = 1,   /* orchestrator/base.py:82 RequestCannotFit            */
  FS_ERR_SIMULATION = 2,           /* base.py:223-228 SimulationError (unfinished)        */
  FS_ERR_EVENT_BUDGET = 3,         /* core.py:66 EventBudgetExceeded                      */
  FS_ERR_SCHEDULING_IN_PAST = 4,   /* core.py:58 SchedulingInPast                         */
  FS_ERR_ROUTING = 5,              /* costmodel/routing.py:25 RoutingError                */
  FS_ERR_TOPOLOGY_MISMATCH = 6,    /* costmodel/moe.py:19 TopologyMismatch                */
  FS_ERR_EMPTY_BATCH = 7,          /* costmodel/features.py:17 EmptyBatch                 */
  FS_ERR_INVALID_TOPK = 8,         /* costmodel/routing.py:21 InvalidTopK                 */
  FS_ERR_ROUTING_TIE = 9,          /* exact key tie at the top-k boundary: which tied
                                      expert np.argpartition keeps depends on numpy's SIMD
                                      dispatch on the host CPU (AVX2+ and baseline kernels
                                      differ, tests/test_known_answers.py), so the engine
                                      flags it rather than guess one host's answer
                                      (probability ~E^2 2^-54 per row)               */
  FS_ERR_UNSUPPORTED = 10,         /* reserved: no current device path returns it          */
  FS_ERR_CAPACITY = 11,            /* engine limit (FS_MAX_*) exceeded                     */
  FS_ERR_INTERNAL = 12,            /* invariant violated inside the engine                 */
  FS_ERR_VALUE = 13,               /* ValueError raised by a cost-model argument check     */
  FS_ERR_SCHEMA = 14               /* costmodel/model.py:118-123, 315-320 SchemaMismatch:
                                      the model's schema is wrong for its slot; raised at
                                      the first prediction, like the reference             */
};

/* Hardware profile + the parallel degrees one OperatorCosts instance uses
 * (cluster.py:225-250; topology.py:134-145). */
typedef struct {
  double peak_flops;          /* FLOP/s per GPU */
  double mem_bw;              /* bytes/s per GPU */
  double kernel_overhead_us;
  int32_t tp, ep, moe_tp, pp;
} fs_cost_ctx;                /* 40 bytes */

/* Router-seed prefix (base.py:63-65): the text "{master_seed}:{scope}:" for a
 * replica scope or "{master_seed}:{replica_key}:mb" for an AF micro-batch scope
 * (af.py:317), len bytes long, mid_blocks = len / 64.
 *  - len <= FS_MAX_PREFIX_BYTES: bytes[] holds the whole text; the engine computes
 *    the SHA-256 state after its first mid_blocks complete 64-byte blocks.
 *  - longer (no limit): bytes[] holds only the last len - 64 * mid_blocks (< 64)
 *    bytes and mid[] the SHA-256 state after the first mid_blocks blocks, computed
 *    by the caller.
 * Either way the device hashes only the tail and the step/layer digits. */
typedef struct {
  uint8_t bytes[FS_MAX_PREFIX_BYTES];
  int32_t len;
  int32_t mid_blocks;
  uint32_t mid[8];
} fs_seed_prefix;             /* 232 bytes */

typedef struct {
  int32_t role;               /* enum fs_role */
  int32_t key_rank;           /* rank of "{cluster_id}/{index}" among this instance's
                                 replicas in Python str order (pd.py:40-48 tie-breaks) */
  int64_t kv_pool_tokens;     /* topology.py:289-302, derived on the host */
  fs_cost_ctx cost;           /* operator-cost context of this replica */
  int32_t prefix;             /* index into the prefix table: replica scope */
  int32_t prefix_mb;          /* AF attention replica: micro-batch scope prefix, else -1 */
} fs_replica_desc;            /* 64 bytes */

typedef struct {
  int32_t mode;               /* enum fs_mode */
  int32_t n_requests;
  int64_t req_offset;         /* first request of this instance in the request SoA */
  int32_t n_replicas;
  int32_t replica_offset;     /* first replica in the replica table */
  /* model (topology.py:70-104) */
  int32_t num_layers, d_model, d_ff, num_query_heads, num_kv_heads, head_dim, dtype_bytes;
  int32_t has_moe, num_experts, top_k, expert_d_ff, ffn_matrices;
  /* scheduler policy (cluster.py:96-118) */
  int32_t admission, priority_key, max_num_seqs, max_batch_tokens;
  int32_t paged, block_tokens;
  /* routing (base.py:43-49) */
  int32_t routing_policy, n_trace_counts;
  int64_t trace_offset;       /* into the trace-count table */
  double routing_alpha;
  /* AF (af.py:261-319, 378-424) */
  int32_t af_micro_batches, af_attn_dp;
  fs_cost_ctx af_attn;        /* attention-side step costs: tp=attn_tp, ep=1, moe_tp=1 */
  fs_cost_ctx af_ffn;         /* ffn-side step costs: tp=moe_tp, ep=moe_ep, moe_tp=moe_tp */
  /* network (topology.py:147-166) */
  double intra_latency_s, intra_bandwidth_bps;
  double inter_latency_s, inter_bandwidth_bps;
  int64_t kv_bytes_per_token; /* topology.py:241-243 */
  int64_t max_events;         /* core.py:142 (default 50,000,000) */
  int32_t total_gpus;         /* Deployment.total_gpus */
  int32_t attn_forest;        /* learned attention model: index into the forest set, -1 =
                                 analytic, -2 = model with a wrong schema (FS_ERR_SCHEMA at
                                 the first prediction); CostModel.predict_attention,
                                 costmodel/model.py:313-321 */
  int32_t gg_forest;          /* learned grouped-GEMM model, same encoding
                                 (CostModel.predict_grouped_gemm, model.py:323-327); on
                                 the device path for dense FFNs (cluster.py:286-296) */
  int32_t pad0;
  int64_t est_cost;           /* host estimate used to order the device work queue */
} fs_instance_desc;

/* Learned operator models (BaggedForest, costmodel/forest.py:46-242): trees as
 * flat node arrays, children addressed by global node index. */
typedef struct {
  int32_t n_trees;
  int32_t n_features;         /* 17 for attention_v1, 12 for grouped_gemm_v1 */
  int64_t tree_offset;        /* first entry of this forest in tree_root[] */
} fs_forest_desc;

typedef struct {
  const fs_forest_desc* forests;
  int32_t n_forests;
  int32_t pad0;
  const int64_t* tree_root;   /* global node index of each tree's root */
  int64_t n_trees;
  const int32_t* feature;     /* split feature, -1 marks a leaf */
  const double* threshold;    /* go left when x[feature] <= threshold */
  const int32_t* left;
  const int32_t* right;
  const double* value;        /* leaf prediction (us) */
  int64_t n_nodes;
} fs_forest_set;

typedef struct {
  const int64_t* arrival_ns;    /* request_order (stable sort by arrival), workload.py:219 */
  const int32_t* prompt_tokens;
  const int32_t* output_tokens;
  const int32_t* id_rank;       /* rank of the request id in Python str order (cluster.py:160) */
} fs_request_soa;

/* One metric row per instance: compute_metrics (metrics.py:81-178) reduced on device. */
typedef struct {
  int32_t status;             /* enum fs_status */
  int32_t status_detail;      /* e.g. local index of the request that cannot fit */
  int64_t iterations;         /* BATCH_COMPLETE events (prefill + decode + AF steps) */
  int64_t events;             /* processed events, no-op kinds included (core.py:187) */
  int64_t total_tokens;
  int64_t makespan_ns;
  int64_t prefill_batches, decode_batches, af_steps;
  int32_t n_requests, n_tpot;
  double makespan_s;
  double throughput_tokens_per_s_per_gpu;
  double ttft[4];             /* mean, p50, p90, p99 (seconds) */
  double tpot[4];             /* NaN when no request has > 1 output token */
  double e2e[4];
  double bubble_fraction;     /* NaN when the run had no AF step */
  double avg_input_tokens, avg_output_tokens;
  int64_t af_busy_ns[4];      /* attn_exec, a2f_link, ffn_exec, f2a_link (af.py:38) */
  double af_busy_fraction[4];
  int64_t moe_layer_samples;  /* number of moe_imbalance entries (base.py:247-252) */
  int64_t routing_calls;
  int64_t routing_draws;      /* router keys drawn: T x E per call with random keys */
} fs_metric_row;

typedef struct {
  int64_t busy_ns;
  double busy_fraction;       /* min(1, busy_ns / makespan_ns), metrics.py:143-145 */
  int64_t steps_executed;
} fs_replica_out;

/* Synthetic workload of one instance (workload.py:131-216 WorkloadSpec):
 * arrivals and lengths drawn from numpy's Philox streams
 * Generator(Philox(key=SeedSequence([seed, stream]).generate_state(2))) with
 * stream 0 arrival, 1 prompt, 2 output (workload.py:36,188-190). */
enum fs_arrival_kind { FS_ARRIVAL_POISSON = 0, FS_ARRIVAL_FIXED = 1, FS_ARRIVAL_AT_ZERO = 2 };
enum fs_length_kind { FS_LEN_FIXED = 0, FS_LEN_UNIFORM = 1, FS_LEN_LOGNORMAL = 2 };
typedef struct {
  int32_t kind;               /* enum fs_length_kind */
  int32_t pad;
  int64_t value, lo, hi;      /* fixed value; clamp / uniform bounds (inclusive) */
  double mu, sigma;           /* lognormal parameters */
} fs_length_dist;             /* 48 bytes */
typedef struct {
  uint64_t seed;              /* WorkloadSpec.seed */
  int32_t n_requests;
  int32_t arrival_kind;       /* enum fs_arrival_kind */
  double rate_rps;            /* poisson */
  int64_t gap_ns;             /* fixed_interval */
  int64_t out_offset;         /* first slot of this instance in the output arrays */
  fs_length_dist prompt, output;
} fs_workload_desc;           /* 136 bytes */

/* Optional per-request outputs (indexed like the request SoA). */
typedef struct {
  int64_t* first_token_ns;    /* first TOKEN_EMITTED */
  int64_t* done_ns;           /* REQUEST_COMPLETE */
  int32_t* completion_rank;   /* order of REQUEST_COMPLETE within the instance */
} fs_request_out;

/* Optional batch / routing log for parity checks. Offsets and capacities are
 * per instance; the engine appends and sets *_count; overflow sets truncated. */
typedef struct {
  int32_t replica;            /* local replica index */
  int32_t phase;              /* 0 prefill, 1 decode, 2 af_decode */
  int64_t t_complete;         /* BATCH_COMPLETE timestamp */
  int64_t duration_ns;
  int32_t n_members;
  int32_t member_offset;      /* into members[] (instance-relative) */
  int32_t moe_offset;         /* into moe_ratio[] (instance-relative), -1 if none */
  int32_t n_moe;
  int64_t seq;                /* sequence number of the BATCH_COMPLETE event (core.py:160) */
  int64_t pool_used;          /* replica.pool.snapshot()["used_tokens"] when the batch
                                 started (base.py:239-246; af.py:494-505) */
  int64_t af_step;            /* AF step id (af.py:477), -1 otherwise */
} fs_batch_rec;               /* 64 bytes; recorded when the batch starts, so records are
                                 in start order: sort by (t_complete, seq) for completion
                                 order */

/* Event-trace record: one per scheduled event, stored at index `seq` of the
 * instance's event array (every scheduled event is dispatched, so a complete
 * run fills 0..event_count-1). The trace the reference returns from
 * ServingSimulation.run() (core.py:85-129) is these records in (t, seq) order,
 * rendered as `t,seq,KIND,canonical_json(payload)` (paper_2508_03148_b200/trace.py).
 * Fields by kind (request / replica are instance-local indices):
 *   REQUEST_ARRIVAL          a = request
 *   BATCH_START              replica
 *   BATCH_COMPLETE           replica, a = index of its fs_batch_rec
 *   PREFILL_COMPLETE         replica, a = request
 *   MEMORY_AVAILABLE         replica, a = request, b = freed tokens, x = headroom after
 *   KV_CACHE_TRANSFER_START  replica = decode dst, a = request, b = reserved tokens,
 *                            c = prefill src, x = decode pool used after the reservation
 *                            (pd.py:161-175)
 *   KV_CACHE_TRANSFER_DONE   replica = decode dst, a = request, c = prefill src
 *   *_DONE (AF nodes)        a = micro-batch i, b = layer k (both 1-based), c = step,
 *                            x = node start ns (af.py:177-194)
 *   TOKEN_EMITTED            replica (request_ids = the batch completing on it at t)
 *   REQUEST_COMPLETE         replica, a = request                                     */
enum fs_event_kind {          /* core.py:38-51 EventKind, declaration order */
  FS_EV_REQUEST_ARRIVAL = 0, FS_EV_BATCH_START = 1, FS_EV_BATCH_COMPLETE = 2,
  FS_EV_PREFILL_COMPLETE = 3, FS_EV_MEMORY_AVAILABLE = 4, FS_EV_KV_TRANSFER_START = 5,
  FS_EV_KV_TRANSFER_DONE = 6, FS_EV_ATTN_DONE = 7, FS_EV_A2F_DONE = 8, FS_EV_FFN_DONE = 9,
  FS_EV_F2A_DONE = 10, FS_EV_TOKEN_EMITTED = 11, FS_EV_REQUEST_COMPLETE = 12
};
typedef struct {
  int64_t t;
  int64_t seq;
  int64_t x;
  int32_t a, b, c;
  int16_t replica;
  uint8_t kind;               /* enum fs_event_kind */
  uint8_t pad;
} fs_event_rec;               /* 40 bytes */

typedef struct {
  int32_t replica;            /* local replica index */
  int32_t micro_batch;        /* 0 for replica scope, i >= 1 for AF micro-batch scope */
  int64_t step;
  int32_t layer;
  int32_t tokens;
  int32_t counts_offset;      /* into counts[] (instance-relative) */
  int32_t n_experts;
} fs_route_rec;               /* 32 bytes */

typedef struct {
  /* per-instance capacities and bases (arrays of n_instances). Instance i writes
     at most `cap` records from base[i]; each host array must hold
     max_i(base[i] + cap) records (that many are copied back). */
  const int64_t* batch_base;  int32_t batch_cap;
  const int64_t* member_base; int32_t member_cap;
  const int64_t* moe_base;    int32_t moe_cap;
  const int64_t* route_base;  int32_t route_cap;
  const int64_t* counts_base; int32_t counts_cap;
  fs_batch_rec* batches;
  int32_t* members;           /* local request indices */
  double* moe_ratio;          /* expert_us / mean(per_rank_us), unrounded (host rounds to 6) */
  fs_route_rec* routes;
  int32_t* counts;
  int32_t* batch_count;       /* per instance */
  int32_t* route_count;
  int32_t* truncated;
  /* event trace (optional): records indexed by seq; event_count = events scheduled */
  const int64_t* event_base;  int32_t event_cap; int32_t pad0;
  fs_event_rec* events;
  int64_t* event_count;       /* per instance */
} fs_log;

/* ---- engine lifecycle ---------------------------------------------------- */
typedef struct fs_engine fs_engine;

int fs_abi_version(void);
/* sizeof of the ABI structs in declaration order (binding self-check); returns count */
int fs_struct_sizes(int64_t* out, int n);
int fs_create(int device, fs_engine** out);
void fs_destroy(fs_engine* e);
const char* fs_last_error(const fs_engine* e);

/* ---- batched simulation (the hot path) ------------------------------------ */

/* Drop-in path: host buffers in, host metric rows out (H2D + kernels + D2H). */
int fs_run_batch(fs_engine* e,
                 const fs_instance_desc* descs, int32_t n_instances,
                 const fs_replica_desc* replicas, int32_t n_replicas,
                 const fs_seed_prefix* prefixes, int32_t n_prefixes,
                 const int64_t* trace_counts, int64_t n_trace_counts,
                 fs_request_soa requests, int64_t n_requests,
                 fs_metric_row* rows_out,
                 fs_replica_out* replica_out,      /* nullable */
                 fs_request_out per_request,       /* members nullable */
                 fs_log* log);                     /* nullable */

/* Stage learned models (kept on the device until replaced); instances refer
 * to them by index (fs_instance_desc.attn_forest). */
int fs_set_forests(fs_engine* e, fs_forest_set forests);

/* Resident path: stage inputs once, then launch repeatedly on device data. */
int fs_stage(fs_engine* e,
             const fs_instance_desc* descs, int32_t n_instances,
             const fs_replica_desc* replicas, int32_t n_replicas,
             const fs_seed_prefix* prefixes, int32_t n_prefixes,
             const int64_t* trace_counts, int64_t n_trace_counts,
             fs_request_soa requests, int64_t n_requests);
/* Launch the simulation + metrics kernels on `stream` (a cudaStream_t, may be 0).
 * Fails (and launches nothing) when the staged batch uses learned models and
 * fs_set_forests replaced them after fs_stage. */
int fs_launch_async(fs_engine* e, void* stream);
/* Copy results of the last launch to host buffers: waits for that launch only (on
 * whichever stream it ran), so another engine's batch keeps running meanwhile. */
int fs_fetch(fs_engine* e, fs_metric_row* rows_out, fs_replica_out* replica_out,
             fs_request_out per_request);
/* Kernel launches issued by the last fs_launch_async. */
int fs_last_launch_count(const fs_engine* e);

/* ---- cost-model kernels ----------------------------------------------------- */

typedef struct {
  int32_t num_query_heads, num_kv_heads, head_dim, dtype_bytes;
  double peak_flops, mem_bw, kernel_overhead_us;
} fs_attn_params;

/* analytic.attention_us over CSR batches; device pointers, async on stream.
 * q_lens/kv_lens: int32 per request; offsets: int64 [n_batches+1];
 * is_decode: uint8 per batch; out_us: double per batch; status: int32 per batch
 * (0 ok, FS_ERR_EMPTY_BATCH / FS_ERR_VALUE for the AttentionFeatures checks). */
int fs_attention_cost_dev(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                          const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                          fs_attn_params params, double* out_us, int32_t* status,
                          void* stream);
/* Same, host buffers (synchronous). */
int fs_attention_cost(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                      const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                      fs_attn_params params, double* out_us, int32_t* status);
/* 17-dim attention_v1 feature vectors (features.py:101-115), numpy-exact std. */
int fs_attention_features_dev(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                              const int64_t* offsets, const uint8_t* is_decode,
                              int64_t n_batches, fs_attn_params params, double* out17,
                              void* stream);

/* Same, host buffers (synchronous); out17 is n_batches x 17. */
int fs_attention_features(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                          const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                          fs_attn_params params, double* out17);

/* LearnedOperatorModel.predict_us(AttentionFeatures(...).vector()) over CSR
 * batches with staged forest `forest` (costmodel/model.py:126-136,
 * forest.py:234-239): 17 features, tree walks, sorted-leaf numpy mean,
 * max(., 1e-6). A batch that fails AttentionFeatures' checks (empty, q < 1,
 * decode q != 1, prefill kv < q, kv < 1; features.py:44-66) yields NaN.
 * Device pointers, async on stream. */
int fs_attention_forest_dev(fs_engine* e, int32_t forest, const int32_t* q_lens,
                            const int32_t* kv_lens, const int64_t* offsets,
                            const uint8_t* is_decode, int64_t n_batches, fs_attn_params params,
                            double* out_us, void* stream);
/* Same, host buffers (synchronous). */
int fs_attention_forest(fs_engine* e, int32_t forest, const int32_t* q_lens,
                        const int32_t* kv_lens, const int64_t* offsets, const uint8_t* is_decode,
                        int64_t n_batches, fs_attn_params params, double* out_us);

/* route_tokens(T, E, k, "uniform", seed) for a list of calls (host buffers).
 * counts_out: n_calls x num_experts int32. status: per call. */
int fs_route_uniform(fs_engine* e, const int64_t* tokens, const uint64_t* seeds, int32_t n_calls,
                     int32_t num_experts, int32_t top_k, int32_t* counts_out, int32_t* status);

/* route_tokens(T, E, k, policy, seed, alpha) for a list of calls (host buffers):
 * policy FS_ROUTE_UNIFORM or FS_ROUTE_DIRICHLET (routing.py:65-113; the trace
 * policy needs no device). counts_out: n_calls x num_experts int32. status: per call. */
int fs_route_tokens(fs_engine* e, const int64_t* tokens, const uint64_t* seeds, int32_t n_calls,
                    int32_t num_experts, int32_t top_k, int32_t policy, double alpha,
                    int32_t* counts_out, int32_t* status);

/* generate(spec) for n instances on the device (workload.py:193-216): requests in
 * generation order, which is arrival order for every synthetic arrival kind
 * (cumulative gaps are non-decreasing), so the arrays are the request SoA of
 * fs_run_batch as they stand; id_rank = rank of "r{i}" in Python str order.
 * Host buffers indexed by out_offset + i. status per instance (FS_ERR_VALUE for
 * an unknown kind). */
int fs_generate_workload(fs_engine* e, const fs_workload_desc* w, int32_t n,
                         int64_t* arrival_ns, int32_t* prompt_tokens, int32_t* output_tokens,
                         int32_t* id_rank, int32_t* status);

/* derive_router_seed for (prefix, step, layer[, micro_batch]) tuples (host buffers). */
int fs_router_seeds(fs_engine* e, const fs_seed_prefix* prefixes, const int32_t* prefix_idx,
                    const int32_t* micro_batch, const int64_t* steps, const int32_t* layers,
                    int32_t n, uint32_t* seeds_out);

/* ---- diagnostics: the pure functions the simulator composes ----------------
 * fs_eval evaluates one of them elementwise on the device through the same
 * device functions sim_kernel calls, for parity tests against the reference's
 * golden vectors (tests/test_eval.py). Records of `in_stride` doubles in,
 * `out_stride` doubles out; integers as exact doubles; status per record.
 * Replaces nothing in the reference (its pure functions are Python calls):
 *   FS_EVAL_EXP/LOG/LOG1P   [x] -> [y]        libm as numpy's distributions.c
 *   FS_EVAL_POW             [x, y] -> [z]     calls it (glibc 2.39, fs_glibm.h)
 *   FS_EVAL_LINEAR          [m, n, k, peak_flops, mem_bw, overhead_us, dtype]
 *                           -> [us]          analytic.py:23-29
 *   FS_EVAL_GROUPED_GEMM    [routed, active, d_model, d_ff, n_matrices, peak_flops,
 *                            mem_bw, overhead_us, dtype] -> [us]   analytic.py:56-71
 *   FS_EVAL_COLLECTIVE_INT  [kind (0 all_to_all, 1 all_reduce, 2 all_gather),
 *   FS_EVAL_COLLECTIVE_FLT   bytes_per_rank, n_ranks, latency_s, bandwidth_bps]
 *                           -> [s]  topology.py:367-394 (int or float bytes)
 *   FS_EVAL_TRANSFER        [bytes, latency_s, bandwidth_bps] -> [s]  topology.py:241-243
 *   FS_EVAL_MOE_LAYER       [E, top_k, ep, moe_tp, n_matrices, T, d_model,
 *                            expert_d_ff, dtype, latency_s, bandwidth_bps,
 *                            peak_flops, mem_bw, overhead_us, counts[E]]
 *                           -> [total_us, expert_us / mean(per_rank_us)]  moe.py:69-128
 *   FS_EVAL_CUDA_*          CUDA's own libm for the same four functions (the
 *                           simulator never calls it; tests use it to show where
 *                           it would have diverged from the host) */
enum fs_eval_fn {
  FS_EVAL_EXP = 1, FS_EVAL_LOG = 2, FS_EVAL_LOG1P = 3, FS_EVAL_POW = 4,
  FS_EVAL_LINEAR = 5, FS_EVAL_GROUPED_GEMM = 6, FS_EVAL_COLLECTIVE_INT = 7,
  FS_EVAL_COLLECTIVE_FLT = 8, FS_EVAL_TRANSFER = 9, FS_EVAL_MOE_LAYER = 10,
  FS_EVAL_CUDA_EXP = 11, FS_EVAL_CUDA_LOG = 12, FS_EVAL_CUDA_LOG1P = 13, FS_EVAL_CUDA_POW = 14
};
int fs_eval(fs_engine* e, int32_t fn, const double* in, int32_t in_stride, int64_t n,
            double* out, int32_t out_stride, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif /* FRONTIER_B200_H */
