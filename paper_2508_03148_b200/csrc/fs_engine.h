// fs_engine.h -- internal types shared by the kernels and the C-ABI host code.
#pragma once
#include <cstdint>

#include "../../include/frontier_b200.h"
#include "fs_forest.cuh"

namespace fs {

// One stored event (state-changing kinds only).
struct HEv {
  int64_t t;
  int64_t seq;
  int32_t kind;
  int32_t a;   // replica (local index)
  int64_t b;   // duration (BATCH_COMPLETE) or request (KV done)
};

// Mutable per-replica state (global replica index).
struct RepState {
  int64_t used;          // KV pool used tokens
  int64_t outstanding;   // sum of prompt tokens in the queue (pd.py:40-45)
  int64_t steps;         // steps_executed
  int64_t busy_ns;       // sum of BATCH_COMPLETE durations
  int64_t sum_ctx;       // sum of (prompt + emitted) over the running list
  int64_t inflight_dur;
  int32_t qlen, rlen, ilen;
  int32_t busy, start_pending;
  int32_t dstep;         // decode iterations completed
  int32_t min_finish;    // earliest finish step among running requests
  int32_t inflight_phase;
  int32_t inflight_moe;  // a moe-ratio log slot was written for the in-flight batch
  int32_t pad;
};

constexpr int kJobLayers = 32;  // layers routed per job
// dirichlet_skew router scratch per warp (fs_dirichlet.cuh): popularity[E] + a key ring
// keys of up to 32 completed-but-untallied rows + one unfinished row + one window
// (rows are tallied 32 at a time, one per lane): 32 x 1024 + 1023 + 128 < 2^16
constexpr int kDirRing = 65536;
// per-warp scratch (doubles): popularity[E] | ring | sort buffer for top_k > FS_MAX_TOPK
// (FS_MAX_EXPERTS keys + FS_MAX_EXPERTS indices, fs_route.cuh select_sorted)
constexpr int kSortOffset = FS_MAX_EXPERTS + kDirRing;
constexpr int kDirScratch = kSortOffset + 2 * FS_MAX_EXPERTS;

// A routing job: the uniform router calls of up to kJobLayers layers of one
// batch (routing.py:65-113, one call per layer), split into chunks of rows
// that any idle warp on the GPU may claim (see fs_engine.cu, "job board").
struct RouteJob {
  unsigned long long ctr;  // epoch (24 bits) | n_chunks (20 bits) | next chunk (20 bits)
  int32_t done;            // chunks finished
  int32_t tie;             // status: 0, FS_ERR_ROUTING_TIE or another routing error
  int64_t T;               // tokens (rows per layer)
  int32_t E, k, nl, nseg, passes_per_chunk;
  int32_t kind;            // 0: uniform, chunks of rows; 1: dirichlet_skew, one chunk per layer
  double alpha;            // dirichlet_skew concentration
  uint64_t keys[kJobLayers][2];
};

struct EngineParams {
  // inputs
  const fs_instance_desc* descs;
  int32_t n_inst;
  const fs_replica_desc* reps;
  const fs_seed_prefix* prefixes;
  const uint32_t* midstate;      // 8 words per prefix (device-computed)
  const int64_t* trace_counts;
  const int64_t* arrival;
  const int32_t* prompt;
  const int32_t* output;
  const int32_t* id_rank;
  const int32_t* order;          // processing order (longest estimated first)
  // workspace
  int64_t* first_ns;
  int64_t* done_ns;
  int32_t* done_rank;
  int32_t* finish_at;
  int32_t* home;                 // prefill home (PD)
  int32_t* lists;
  const int64_t* list_base;      // per instance
  HEv* heap;
  const int64_t* heap_base;      // per instance
  int32_t* xfer;                 // transfer FIFO ring, indexed like requests
  RepState* rstate;
  int64_t* af_ffn;
  const int64_t* af_base;        // per instance (-1 when not AF)
  // outputs
  fs_metric_row* rows;
  fs_replica_out* rep_out;
  // optional log (device pointers)
  fs_log log;
  int32_t log_enabled;
  int32_t* work_counter;
  int64_t* inst_cycles;          // SM cycles each instance took (profiling aid)
  // routing job board (one slot per resident warp of the simulation grid)
  RouteJob* jobs;
  int32_t* job_counts;           // [n_slots][kJobLayers * job_max_e]
  int32_t n_slots;
  int32_t job_max_e;
  int32_t* inst_done;            // instances finished (helpers stop at n_inst)
  int32_t* open_jobs;            // published jobs with unclaimed chunks
  double* dir_scratch;           // [n_slots][kDirScratch]: dirichlet_skew popularity + key ring
  int32_t chunk_blocks;          // Philox blocks per lane per chunk (FS_CHUNK_BLOCKS)
  ForestView fv;                 // learned operator models (fs_set_forests)
};

// host-side launchers (fs_engine.cu / fs_metrics.cu / fs_costs.cu)
void launch_midstate(const fs_seed_prefix* prefixes, uint32_t* mid, int n, void* stream);
// simulation kernel variants (fs_sim.cuh compiled twice)
namespace analytic {
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers);
int launch(const EngineParams& p, void* stream);
}  // namespace analytic
namespace learned {
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers);
int launch(const EngineParams& p, void* stream);
}  // namespace learned
namespace longrow {
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers);
int launch(const EngineParams& p, void* stream);
}  // namespace longrow
namespace comoe {
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers);
int launch(const EngineParams& p, void* stream);
}  // namespace comoe
namespace dense {
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers);
int launch(const EngineParams& p, void* stream);
}  // namespace dense
// simulation kernel variants: analytic (the sweep kernel), learned (learned models,
// dirichlet routing), longrow (analytic, MoE rows of >= 64 experts), dense (no MoE)
enum SimVariant { kSimAnalytic = 0, kSimLearned = 1, kSimLongRow = 2, kSimDense = 3,
                  kSimCoMoe = 4 };
// ctas_per_sm <= 0: as many simulation CTAs per SM as fit
int simulation_slots(int n_sms, int n_inst, int variant, int ctas_per_sm, bool helpers);
int launch_simulation(const EngineParams& p, int variant, void* stream);
int launch_metrics(const EngineParams& p, void* stream);
int launch_attention_cost(const int32_t* q, const int32_t* kv, const int64_t* off,
                          const uint8_t* dec, int64_t nb, fs_attn_params prm, double* out,
                          int32_t* status, int n_sms, void* stream);
int launch_attention_features(const int32_t* q, const int32_t* kv, const int64_t* off,
                              const uint8_t* dec, int64_t nb, fs_attn_params prm, double* out17,
                              void* stream);
int launch_attention_forest(const ForestView& fv, int forest, const int32_t* q, const int32_t* kv,
                            const int64_t* off, const uint8_t* dec, int64_t nb, fs_attn_params prm,
                            double* out, int n_sms, void* stream);
int launch_route_tokens(const int64_t* tokens, const uint64_t* seeds, int n, int E, int k,
                        int policy, double alpha, double* scratch, int32_t* counts,
                        int32_t* status, void* stream);
int route_scratch_warps(int n);  // warps (scratch slots) launch_route_tokens uses for n calls
int launch_workload(const fs_workload_desc* w, int n, int64_t* arrival, int32_t* prompt,
                    int32_t* output, int32_t* rank, int32_t* status, void* stream);
int launch_eval(int fn, const double* in, int in_stride, int64_t n, double* out, int out_stride,
                int32_t* status, int n_sms, void* stream);
int launch_router_seeds(const fs_seed_prefix* pf, const uint32_t* mid, const int32_t* pidx,
                        const int32_t* mb, const int64_t* steps, const int32_t* layers, int n,
                        uint32_t* out, void* stream);

}  // namespace fs
