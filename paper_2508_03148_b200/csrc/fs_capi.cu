// fs_capi.cu -- the C ABI (include/frontier_b200.h): engine lifecycle, staging of
// instance descriptors into HBM, kernel launches, result readback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "fs_engine.h"

using fs::EngineParams;
using fs::HEv;
using fs::RepState;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

}  // namespace

struct fs_engine {
  int device = 0;
  int n_sms = 148;
  std::string err;
  cudaStream_t stream = nullptr;
  cudaEvent_t launched = nullptr;  // recorded after a batch's last kernel (fs_fetch waits on it)
  cudaEvent_t staged_ev = nullptr; // recorded after fs_stage's uploads + midstate kernel
  // inputs
  DevBuf descs, reps, prefixes, mid, trace, arrival, prompt, output, id_rank, order;
  // workspace
  DevBuf first, done, rank, finish, home, lists, list_base, heap, heap_base, xfer, rstate, af_ffn,
      af_base, work, cycles, jobs, job_counts, inst_done, dir_scratch;
  // outputs
  DevBuf rows, rep_out;
  // log mirrors
  DevBuf lg_batch_base, lg_member_base, lg_moe_base, lg_route_base, lg_counts_base, lg_batches,
      lg_members, lg_moe, lg_routes, lg_counts, lg_bcount, lg_rcount, lg_trunc, lg_event_base,
      lg_events, lg_ecount;
  // cost-model scratch
  DevBuf c_q, c_kv, c_off, c_dec, c_out, c_status, c_tok, c_seed, c_counts, c_pidx, c_mb, c_steps,
      c_layers, c_seeds, c_pf, c_mid, c_scratch, c_ein, c_eout;
  // workload generation
  DevBuf g_desc, g_arr, g_pr, g_out, g_rank, g_st;
  // learned models (persist across stages)
  DevBuf f_descs, f_roots, f_right, f_value, f_leaf;  // f_value: packed NodeP array
  fs::ForestView fv{};
  int64_t forest_gen = 0;         // bumped by every fs_set_forests
  int64_t staged_forest_gen = -1; // forest_gen the staged batch's indices refer to
  bool staged_uses_forests = false;
  bool learned = false;  // staged batch has instances for the learned simulation variant
  int variant = 0;       // fs::SimVariant of the first wave (single-wave batches: the batch)
  int n_moe = 0;         // MoE instances of the staged batch (first in the order)
  // waves: instances bucketed by kernel variant, consecutive in the order array
  struct Wave { int variant, start, count, slots; };
  Wave waves[5];
  int n_waves = 0;
  int split_families = 1;  // FS_SPLIT_FAMILIES: MoE and dense instances in separate waves
  int dense_variant = 1;   // FS_DENSE_VARIANT: dense instances on the MoE-free kernel
  int comoe_variant = 1;   // FS_COMOE_VARIANT: co-located MoE instances on their own kernel
  // routing job geometry (environment knobs read at fs_create)
  int sim_ctas = 0;          // FS_SIM_CTAS_PER_SM (0 = as many as fit)
  int chunk_blocks = 96;     // FS_CHUNK_BLOCKS: Philox blocks per lane per job chunk
  int32_t n_inst = 0, n_reps = 0, n_prefixes = 0;
  int64_t n_req = 0;
  int staged = 0;
  int last_launches = 0;
  EngineParams params{};
};

#define FS_CHECK(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      e->err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
      return (int)e_ ? (int)e_ : 1;                                           \
    }                                                                         \
  } while (0)

template <typename T>
static cudaError_t upload(DevBuf& b, const T* src, size_t n, cudaStream_t s) {
  cudaError_t r = b.ensure(n * sizeof(T));
  if (r != cudaSuccess) return r;
  if (n && src) return cudaMemcpyAsync(b.p, src, n * sizeof(T), cudaMemcpyHostToDevice, s);
  return cudaSuccess;
}

extern "C" {

int fs_abi_version(void) { return FS_ABI_VERSION; }

// sizes of the ABI structs, checked by the Python binding at load time
int fs_struct_sizes(int64_t* out, int n) {
  const int64_t s[] = {(int64_t)sizeof(fs_cost_ctx),     (int64_t)sizeof(fs_seed_prefix),
                       (int64_t)sizeof(fs_replica_desc), (int64_t)sizeof(fs_instance_desc),
                       (int64_t)sizeof(fs_metric_row),   (int64_t)sizeof(fs_replica_out),
                       (int64_t)sizeof(fs_batch_rec),    (int64_t)sizeof(fs_route_rec),
                       (int64_t)sizeof(fs_attn_params),  (int64_t)sizeof(fs_forest_desc),
                       (int64_t)sizeof(fs_workload_desc), (int64_t)sizeof(fs_event_rec),
                       (int64_t)sizeof(fs_log)};
  const int k = (int)(sizeof(s) / sizeof(s[0]));
  for (int i = 0; i < n && i < k; i++) out[i] = s[i];
  return k;
}

int fs_create(int device, fs_engine** out) {
  if (!out) return 1;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return 2;
  if (device < 0 || device >= count) return 3;
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  fs_engine* e = new fs_engine();
  e->device = device;
  cudaDeviceGetAttribute(&e->n_sms, cudaDevAttrMultiProcessorCount, device);
  auto env_int = [](const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
  };
  e->sim_ctas = env_int("FS_SIM_CTAS_PER_SM", 0);
  e->split_families = env_int("FS_SPLIT_FAMILIES", 1);
  e->dense_variant = env_int("FS_DENSE_VARIANT", 1);
  e->comoe_variant = env_int("FS_COMOE_VARIANT", 1);
  e->chunk_blocks = env_int("FS_CHUNK_BLOCKS", 96);
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->launched, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->staged_ev, cudaEventDisableTiming) != cudaSuccess) {
    if (e->launched) cudaEventDestroy(e->launched);
    if (e->launched) cudaEventDestroy(e->launched);
  if (e->staged_ev) cudaEventDestroy(e->staged_ev);
  if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
    return 5;
  }
  *out = e;
  return 0;
}

void fs_destroy(fs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamDestroy(e->stream);

  delete e;
}

const char* fs_last_error(const fs_engine* e) { return e ? e->err.c_str() : "null engine"; }

int fs_last_launch_count(const fs_engine* e) { return e ? e->last_launches : 0; }

// SM cycles each instance of the last launch took (profiling aid)
int fs_instance_cycles(fs_engine* e, int64_t* out) {
  if (!e || !e->staged) return 1;
  FS_CHECK(cudaDeviceSynchronize());
  FS_CHECK(cudaMemcpy(out, e->cycles.p, 8 * (size_t)e->n_inst, cudaMemcpyDeviceToHost));
  return 0;
}

int fs_stage(fs_engine* e, const fs_instance_desc* descs, int32_t n_instances,
             const fs_replica_desc* replicas, int32_t n_replicas, const fs_seed_prefix* prefixes,
             int32_t n_prefixes, const int64_t* trace_counts, int64_t n_trace_counts,
             fs_request_soa rq, int64_t n_requests) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  e->err.clear();
  cudaStream_t s = e->stream;
  // host-side workspace layout
  std::vector<int64_t> list_base(n_instances), heap_base(n_instances), af_base(n_instances);
  int64_t lb = 0, hb = 0, ab = 0;
  for (int i = 0; i < n_instances; i++) {
    const fs_instance_desc& d = descs[i];
    if (d.n_requests < 0 || d.n_replicas < 1 || d.req_offset < 0 ||
        d.req_offset + d.n_requests > n_requests || d.replica_offset < 0 ||
        d.replica_offset + d.n_replicas > n_replicas) {
      e->err = "instance " + std::to_string(i) + ": offsets out of range";
      return 10;
    }
    for (int r = 0; r < d.n_replicas; r++) {
      const fs_replica_desc& rd = replicas[d.replica_offset + r];
      if (rd.prefix < 0 || rd.prefix >= n_prefixes || rd.prefix_mb >= n_prefixes) {
        e->err = "instance " + std::to_string(i) + ": prefix index out of range";
        return 11;
      }
    }
    list_base[i] = lb;
    lb += 3LL * d.n_replicas * std::max(d.n_requests, 1);
    heap_base[i] = hb;
    hb += (int64_t)d.n_replicas + d.n_requests + 8;
    if (d.mode == FS_MODE_AF) {
      af_base[i] = ab;
      ab += (int64_t)std::min(std::max(d.af_micro_batches, 1), FS_MAX_MICRO_BATCHES) *
            std::max(d.num_layers, 1);
    } else {
      af_base[i] = -1;
    }
  }
  // Kernel variant per instance: learned models / dirichlet_skew need the extended
  // kernel, long MoE rows (>= 64 experts) the long-row one, other MoE instances the
  // sweep kernel, dense ones the MoE-free kernel. Each variant's instances form one
  // wave (fs_launch_async), so one learned or DeepSeek-V3 instance no longer moves
  // the whole batch onto a slower kernel; within a wave, longest estimated cost first
  // (the work queue is consumed in this order).
  const bool no_longrow = getenv("FS_NO_LONGROW") != nullptr;
  const bool split = e->split_families != 0;
  std::vector<int> cls(n_instances);
  for (int i = 0; i < n_instances; i++) {
    const fs_instance_desc& d = descs[i];
    // the extended (learned) kernel also carries dirichlet_skew routing and the
    // full-row sort for top_k > FS_MAX_TOPK
    const bool lrn = d.attn_forest != -1 || d.gg_forest != -1 ||
                     (d.has_moe && d.routing_policy == FS_ROUTE_DIRICHLET) ||
                     (d.has_moe && d.top_k > FS_MAX_TOPK && d.top_k < d.num_experts);
    int c;
    if (lrn) c = fs::kSimLearned;
    else if (d.has_moe && d.num_experts >= 64 && !no_longrow) c = fs::kSimLongRow;
    else if (d.has_moe && d.mode == FS_MODE_COLOCATED && d.top_k <= 3 && e->comoe_variant)
      c = fs::kSimCoMoe;
    else if (d.has_moe || !e->dense_variant) c = fs::kSimAnalytic;
    else c = fs::kSimDense;
    cls[i] = c;
  }
  if (!split) {  // FS_SPLIT_FAMILIES=0: one wave on the most general variant present
    int v = fs::kSimDense;
    for (int i = 0; i < n_instances; i++) {
      if (cls[i] == fs::kSimLearned) v = fs::kSimLearned;
      else if (cls[i] == fs::kSimLongRow && v != fs::kSimLearned) v = fs::kSimLongRow;
      else if ((cls[i] == fs::kSimAnalytic || cls[i] == fs::kSimCoMoe) && v == fs::kSimDense)
        v = fs::kSimAnalytic;
    }
    for (int i = 0; i < n_instances; i++) cls[i] = v;
  }
  static const int kWaveOrder[5] = {fs::kSimLearned, fs::kSimLongRow, fs::kSimAnalytic,
                                    fs::kSimCoMoe, fs::kSimDense};
  auto rank_of = [&](int c) { for (int k = 0; k < 5; k++) if (kWaveOrder[k] == c) return k; return 5; };
  std::vector<int32_t> order(n_instances);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (cls[a] != cls[b]) return rank_of(cls[a]) < rank_of(cls[b]);
    return descs[a].est_cost > descs[b].est_cost;
  });
  e->n_waves = 0;
  for (int k = 0; k < n_instances;) {
    int j = k;
    while (j < n_instances && cls[order[j]] == cls[order[k]]) j++;
    e->waves[e->n_waves++] = {cls[order[k]], k, j - k, 0};
    k = j;
  }
  e->n_moe = 0;
  for (int i = 0; i < n_instances; i++) e->n_moe += descs[i].has_moe ? 1 : 0;

  FS_CHECK(upload(e->descs, descs, n_instances, s));
  FS_CHECK(upload(e->reps, replicas, n_replicas, s));
  FS_CHECK(upload(e->prefixes, prefixes, n_prefixes, s));
  FS_CHECK(e->mid.ensure((size_t)std::max(n_prefixes, 1) * 8 * sizeof(uint32_t)));
  FS_CHECK(upload(e->trace, trace_counts, (size_t)n_trace_counts, s));
  FS_CHECK(upload(e->arrival, rq.arrival_ns, (size_t)n_requests, s));
  FS_CHECK(upload(e->prompt, rq.prompt_tokens, (size_t)n_requests, s));
  FS_CHECK(upload(e->output, rq.output_tokens, (size_t)n_requests, s));
  FS_CHECK(upload(e->id_rank, rq.id_rank, (size_t)n_requests, s));
  FS_CHECK(upload(e->order, order.data(), order.size(), s));
  FS_CHECK(upload(e->list_base, list_base.data(), list_base.size(), s));
  FS_CHECK(upload(e->heap_base, heap_base.data(), heap_base.size(), s));
  FS_CHECK(upload(e->af_base, af_base.data(), af_base.size(), s));
  // The caller's arrays may be pinned (truly asynchronous copies): wait for the
  // uploads, but not for the memsets and the midstate kernel below -- another engine's
  // resident wave can hold every SM they could run on (api.simulate stages its second
  // batch then); fs_launch_async orders itself after staged_ev instead.
  FS_CHECK(cudaEventRecord(e->staged_ev, s));
  FS_CHECK(cudaEventSynchronize(e->staged_ev));
  const size_t nr = (size_t)std::max<int64_t>(n_requests, 1);
  FS_CHECK(e->first.ensure(nr * 8));
  FS_CHECK(e->done.ensure(nr * 8));
  FS_CHECK(e->rank.ensure(nr * 4));
  FS_CHECK(e->finish.ensure(nr * 4));
  FS_CHECK(e->home.ensure(nr * 4));
  FS_CHECK(e->xfer.ensure(nr * 4));
  FS_CHECK(e->lists.ensure((size_t)std::max<int64_t>(lb, 1) * 4));
  FS_CHECK(e->heap.ensure((size_t)std::max<int64_t>(hb, 1) * sizeof(HEv)));
  FS_CHECK(e->rstate.ensure((size_t)std::max(n_replicas, 1) * sizeof(RepState)));
  FS_CHECK(e->af_ffn.ensure((size_t)std::max<int64_t>(ab, 1) * 8));
  FS_CHECK(e->work.ensure(sizeof(int32_t)));
  FS_CHECK(e->cycles.ensure((size_t)std::max(n_instances, 1) * 8));
  FS_CHECK(e->rows.ensure((size_t)std::max(n_instances, 1) * sizeof(fs_metric_row)));
  FS_CHECK(e->rep_out.ensure((size_t)std::max(n_replicas, 1) * sizeof(fs_replica_out)));
  // done_ns / first_ns start at -1 so a request the engine never reached is visible
  FS_CHECK(cudaMemsetAsync(e->first.p, 0xff, nr * 8, s));
  FS_CHECK(cudaMemsetAsync(e->done.p, 0xff, nr * 8, s));
  FS_CHECK(cudaMemsetAsync(e->rank.p, 0xff, nr * 4, s));

  EngineParams& P = e->params;
  memset(&P, 0, sizeof P);
  P.descs = e->descs.as<fs_instance_desc>();
  P.n_inst = n_instances;
  P.reps = e->reps.as<fs_replica_desc>();
  P.prefixes = e->prefixes.as<fs_seed_prefix>();
  P.midstate = e->mid.as<uint32_t>();
  P.trace_counts = e->trace.as<int64_t>();
  P.arrival = e->arrival.as<int64_t>();
  P.prompt = e->prompt.as<int32_t>();
  P.output = e->output.as<int32_t>();
  P.id_rank = e->id_rank.as<int32_t>();
  P.order = e->order.as<int32_t>();
  P.first_ns = e->first.as<int64_t>();
  P.done_ns = e->done.as<int64_t>();
  P.done_rank = e->rank.as<int32_t>();
  P.finish_at = e->finish.as<int32_t>();
  P.home = e->home.as<int32_t>();
  P.lists = e->lists.as<int32_t>();
  P.list_base = e->list_base.as<int64_t>();
  P.heap = e->heap.as<HEv>();
  P.heap_base = e->heap_base.as<int64_t>();
  P.xfer = e->xfer.as<int32_t>();
  P.rstate = e->rstate.as<RepState>();
  P.af_ffn = e->af_ffn.as<int64_t>();
  P.af_base = e->af_base.as<int64_t>();
  P.rows = e->rows.as<fs_metric_row>();
  P.rep_out = e->rep_out.as<fs_replica_out>();
  P.work_counter = e->work.as<int32_t>();
  P.inst_cycles = e->cycles.as<int64_t>();
  P.log_enabled = 0;
  // routing job board: one slot per resident warp of the persistent grid
  e->learned = false;
  e->staged_uses_forests = false;
  e->staged_forest_gen = e->forest_gen;
  for (int i = 0; i < n_instances; i++) {
    const int32_t fsel[2] = {descs[i].attn_forest, descs[i].gg_forest};
    for (int32_t f : fsel) {
      if (f >= e->fv.n_forests || f < -2) {
        e->err = "instance " + std::to_string(i) + ": forest index not staged (fs_set_forests)";
        return 13;
      }
      if (f != -1) e->learned = true;
      if (f >= 0) e->staged_uses_forests = true;
    }
    // dirichlet_skew routing is compiled into the extended (learned) kernel variant only
    if (descs[i].has_moe && descs[i].routing_policy == FS_ROUTE_DIRICHLET) e->learned = true;
  }
  int max_e = 0;
  for (int i = 0; i < n_instances; i++)
    if (descs[i].has_moe) max_e = std::max(max_e, descs[i].num_experts);
  e->variant = e->n_waves ? e->waves[0].variant : fs::kSimAnalytic;
  // per-wave resident grid; waves with MoE instances launch the full wave so warps
  // without an instance help route. Job-board slots cover the largest wave.
  P.n_slots = 0;
  for (int w = 0; w < e->n_waves; w++) {
    bool moe = false;
    for (int k = e->waves[w].start; k < e->waves[w].start + e->waves[w].count; k++)
      moe |= descs[order[k]].has_moe != 0;
    e->waves[w].slots = fs::simulation_slots(e->n_sms, e->waves[w].count, e->waves[w].variant,
                                             e->sim_ctas, moe);
    P.n_slots = std::max(P.n_slots, e->waves[w].slots);
  }
  if (P.n_slots == 0) P.n_slots = 32;
  P.chunk_blocks = e->chunk_blocks;
  P.job_max_e = std::min(max_e, FS_MAX_EXPERTS);
  FS_CHECK(e->inst_done.ensure(2 * sizeof(int32_t)));
  P.inst_done = e->inst_done.as<int32_t>();
  P.open_jobs = e->inst_done.as<int32_t>() + 1;
  P.fv = e->fv;
  if (max_e > 0) {
    FS_CHECK(e->jobs.ensure((size_t)P.n_slots * sizeof(fs::RouteJob)));
    FS_CHECK(e->job_counts.ensure((size_t)P.n_slots * fs::kJobLayers * P.job_max_e * 4));
    P.jobs = e->jobs.as<fs::RouteJob>();
    P.job_counts = e->job_counts.as<int32_t>();
  } else {
    P.jobs = nullptr;
    P.job_counts = nullptr;
  }
  bool dirichlet = false;
  for (int i = 0; i < n_instances; i++)
    dirichlet |= descs[i].has_moe && (descs[i].routing_policy == FS_ROUTE_DIRICHLET ||
                                      descs[i].gg_forest != -1 ||  // learned MoE: entropy
                                      descs[i].top_k > FS_MAX_TOPK);  // row sort buffer
  if (dirichlet) {
    FS_CHECK(e->dir_scratch.ensure((size_t)P.n_slots * fs::kDirScratch * sizeof(double)));
    P.dir_scratch = e->dir_scratch.as<double>();
  } else {
    P.dir_scratch = nullptr;
  }
  e->n_inst = n_instances;
  e->n_reps = n_replicas;
  e->n_prefixes = n_prefixes;
  e->n_req = n_requests;
  fs::launch_midstate(P.prefixes, e->mid.as<uint32_t>(), n_prefixes, s);
  FS_CHECK(cudaGetLastError());
  FS_CHECK(cudaEventRecord(e->staged_ev, s));
  e->staged = 1;
  return 0;
}

int fs_launch_async(fs_engine* e, void* stream) {
  if (!e || !e->staged) return 1;
  if (e->staged_uses_forests && e->staged_forest_gen != e->forest_gen) {
    // the staged instances' forest indices refer to a forest set that has been
    // replaced since fs_stage: running them would silently use other models
    e->err = "fs_set_forests was called after fs_stage; stage the batch again";
    return 14;
  }
  cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
  FS_CHECK(cudaStreamWaitEvent(s, e->staged_ev, 0));
  FS_CHECK(cudaMemsetAsync(e->work.p, 0, sizeof(int32_t), s));
  FS_CHECK(cudaMemsetAsync(e->inst_done.p, 0, 2 * sizeof(int32_t), s));
  if (e->params.jobs)
    FS_CHECK(cudaMemsetAsync(e->jobs.p, 0, (size_t)e->params.n_slots * sizeof(fs::RouteJob), s));
  e->last_launches = 0;
  // One wave per kernel variant, back to back on the stream: different variants on
  // the same SMs fight over instruction fetch (the C5 sweep took 280 ms with its MoE
  // and dense instances mixed, 184 + 71 ms as separate waves).
  // an event trace is recorded by the extended variant only (fs_sim.cuh tracing())
  const bool traced = e->params.log_enabled && e->params.log.events != nullptr;
  for (int w = 0; w < e->n_waves; w++) {
    fs::EngineParams p = e->params;
    p.n_inst = e->waves[w].count;
    p.order = e->params.order + e->waves[w].start;
    p.n_slots = e->waves[w].slots;
    int variant = e->waves[w].variant;
    if (traced && variant != fs::kSimLearned) {
      variant = fs::kSimLearned;
      p.n_slots = std::min(p.n_slots, fs::simulation_slots(e->n_sms, p.n_inst, variant,
                                                           e->sim_ctas, p.jobs != nullptr));
    }
    if (w > 0) {
      FS_CHECK(cudaMemsetAsync(e->work.p, 0, sizeof(int32_t), s));
      FS_CHECK(cudaMemsetAsync(e->inst_done.p, 0, 2 * sizeof(int32_t), s));
    }
    e->last_launches += fs::launch_simulation(p, variant, s);
  }
  e->last_launches += fs::launch_metrics(e->params, s);
  FS_CHECK(cudaGetLastError());
  FS_CHECK(cudaEventRecord(e->launched, s));
  return 0;
}

int fs_fetch(fs_engine* e, fs_metric_row* rows_out, fs_replica_out* replica_out,
             fs_request_out pr) {
  if (!e || !e->staged) return 1;
  cudaStream_t s = e->stream;
  // wait for this engine's batch only (the launch may have been on the caller's
  // stream): another engine's batch on the same device keeps running meanwhile
  FS_CHECK(cudaStreamWaitEvent(s, e->launched, 0));
  if (rows_out)
    FS_CHECK(cudaMemcpyAsync(rows_out, e->rows.p, sizeof(fs_metric_row) * e->n_inst,
                             cudaMemcpyDeviceToHost, s));
  if (replica_out)
    FS_CHECK(cudaMemcpyAsync(replica_out, e->rep_out.p, sizeof(fs_replica_out) * e->n_reps,
                             cudaMemcpyDeviceToHost, s));
  if (pr.first_token_ns)
    FS_CHECK(cudaMemcpyAsync(pr.first_token_ns, e->first.p, 8 * e->n_req, cudaMemcpyDeviceToHost, s));
  if (pr.done_ns)
    FS_CHECK(cudaMemcpyAsync(pr.done_ns, e->done.p, 8 * e->n_req, cudaMemcpyDeviceToHost, s));
  if (pr.completion_rank)
    FS_CHECK(cudaMemcpyAsync(pr.completion_rank, e->rank.p, 4 * e->n_req, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

static int64_t log_total(const int64_t* base, int n, int32_t cap) {
  int64_t t = 0;
  for (int i = 0; i < n; i++) t = std::max(t, base[i] + cap);
  return t;
}

int fs_run_batch(fs_engine* e, const fs_instance_desc* descs, int32_t n_instances,
                 const fs_replica_desc* replicas, int32_t n_replicas,
                 const fs_seed_prefix* prefixes, int32_t n_prefixes, const int64_t* trace_counts,
                 int64_t n_trace_counts, fs_request_soa requests, int64_t n_requests,
                 fs_metric_row* rows_out, fs_replica_out* replica_out, fs_request_out pr,
                 fs_log* log) {
  int rc = fs_stage(e, descs, n_instances, replicas, n_replicas, prefixes, n_prefixes,
                    trace_counts, n_trace_counts, requests, n_requests);
  if (rc) return rc;
  cudaStream_t s = e->stream;
  int64_t nb = 0, nm = 0, ne = 0, nro = 0, nc = 0, nev = 0;
  if (log) {
    // device mirror of the caller's log buffers
    nb = log->batches ? log_total(log->batch_base, n_instances, log->batch_cap) : 0;
    nm = log->members ? log_total(log->member_base, n_instances, log->member_cap) : 0;
    ne = log->moe_ratio ? log_total(log->moe_base, n_instances, log->moe_cap) : 0;
    nro = log->routes ? log_total(log->route_base, n_instances, log->route_cap) : 0;
    nc = log->counts ? log_total(log->counts_base, n_instances, log->counts_cap) : 0;
    nev = log->events ? log_total(log->event_base, n_instances, log->event_cap) : 0;
    fs_log& dl = e->params.log;
    memset(&dl, 0, sizeof dl);
    dl.batch_cap = log->batch_cap; dl.member_cap = log->member_cap; dl.moe_cap = log->moe_cap;
    dl.route_cap = log->route_cap; dl.counts_cap = log->counts_cap;
    dl.event_cap = log->event_cap;
    const int64_t zero = 0;
    (void)zero;
    std::vector<int64_t> zeros(n_instances, 0);
    FS_CHECK(upload(e->lg_batch_base, log->batch_base ? log->batch_base : zeros.data(), n_instances, s));
    FS_CHECK(upload(e->lg_member_base, log->member_base ? log->member_base : zeros.data(), n_instances, s));
    FS_CHECK(upload(e->lg_moe_base, log->moe_base ? log->moe_base : zeros.data(), n_instances, s));
    FS_CHECK(upload(e->lg_route_base, log->route_base ? log->route_base : zeros.data(), n_instances, s));
    FS_CHECK(upload(e->lg_counts_base, log->counts_base ? log->counts_base : zeros.data(), n_instances, s));
    FS_CHECK(upload(e->lg_event_base, log->event_base ? log->event_base : zeros.data(), n_instances, s));
    dl.batch_base = e->lg_batch_base.as<int64_t>();
    dl.member_base = e->lg_member_base.as<int64_t>();
    dl.moe_base = e->lg_moe_base.as<int64_t>();
    dl.route_base = e->lg_route_base.as<int64_t>();
    dl.counts_base = e->lg_counts_base.as<int64_t>();
    dl.event_base = e->lg_event_base.as<int64_t>();
    if (nb) { FS_CHECK(e->lg_batches.ensure(nb * sizeof(fs_batch_rec))); dl.batches = e->lg_batches.as<fs_batch_rec>(); }
    if (nm) { FS_CHECK(e->lg_members.ensure(nm * 4)); dl.members = e->lg_members.as<int32_t>(); }
    if (ne) { FS_CHECK(e->lg_moe.ensure(ne * 8)); dl.moe_ratio = e->lg_moe.as<double>(); }
    if (nro) { FS_CHECK(e->lg_routes.ensure(nro * sizeof(fs_route_rec))); dl.routes = e->lg_routes.as<fs_route_rec>(); }
    if (nc) { FS_CHECK(e->lg_counts.ensure(nc * 4)); dl.counts = e->lg_counts.as<int32_t>(); }
    if (nev) {
      FS_CHECK(e->lg_events.ensure(nev * sizeof(fs_event_rec)));
      dl.events = e->lg_events.as<fs_event_rec>();
    }
    FS_CHECK(e->lg_ecount.ensure(8 * (size_t)std::max(n_instances, 1)));
    FS_CHECK(cudaMemsetAsync(e->lg_ecount.p, 0, 8 * (size_t)n_instances, s));
    dl.event_count = e->lg_ecount.as<int64_t>();
    FS_CHECK(e->lg_bcount.ensure(4 * (size_t)std::max(n_instances, 1)));
    FS_CHECK(e->lg_rcount.ensure(4 * (size_t)std::max(n_instances, 1)));
    FS_CHECK(e->lg_trunc.ensure(4 * (size_t)std::max(n_instances, 1)));
    FS_CHECK(cudaMemsetAsync(e->lg_bcount.p, 0, 4 * (size_t)n_instances, s));
    FS_CHECK(cudaMemsetAsync(e->lg_rcount.p, 0, 4 * (size_t)n_instances, s));
    FS_CHECK(cudaMemsetAsync(e->lg_trunc.p, 0, 4 * (size_t)n_instances, s));
    dl.batch_count = e->lg_bcount.as<int32_t>();
    dl.route_count = e->lg_rcount.as<int32_t>();
    dl.truncated = e->lg_trunc.as<int32_t>();
    e->params.log_enabled = 1;
  }
  rc = fs_launch_async(e, s);
  if (rc) { e->params.log_enabled = 0; return rc; }
  rc = fs_fetch(e, rows_out, replica_out, pr);
  if (!rc && log) {
    if (nb) FS_CHECK(cudaMemcpy(log->batches, e->lg_batches.p, nb * sizeof(fs_batch_rec), cudaMemcpyDeviceToHost));
    if (nm) FS_CHECK(cudaMemcpy(log->members, e->lg_members.p, nm * 4, cudaMemcpyDeviceToHost));
    if (ne) FS_CHECK(cudaMemcpy(log->moe_ratio, e->lg_moe.p, ne * 8, cudaMemcpyDeviceToHost));
    if (nro) FS_CHECK(cudaMemcpy(log->routes, e->lg_routes.p, nro * sizeof(fs_route_rec), cudaMemcpyDeviceToHost));
    if (nc) FS_CHECK(cudaMemcpy(log->counts, e->lg_counts.p, nc * 4, cudaMemcpyDeviceToHost));
    if (log->batch_count) FS_CHECK(cudaMemcpy(log->batch_count, e->lg_bcount.p, 4 * (size_t)n_instances, cudaMemcpyDeviceToHost));
    if (log->route_count) FS_CHECK(cudaMemcpy(log->route_count, e->lg_rcount.p, 4 * (size_t)n_instances, cudaMemcpyDeviceToHost));
    if (log->truncated) FS_CHECK(cudaMemcpy(log->truncated, e->lg_trunc.p, 4 * (size_t)n_instances, cudaMemcpyDeviceToHost));
    if (nev) FS_CHECK(cudaMemcpy(log->events, e->lg_events.p, nev * sizeof(fs_event_rec), cudaMemcpyDeviceToHost));
    if (log->event_count) FS_CHECK(cudaMemcpy(log->event_count, e->lg_ecount.p, 8 * (size_t)n_instances, cudaMemcpyDeviceToHost));
  }
  e->params.log_enabled = 0;
  memset(&e->params.log, 0, sizeof e->params.log);
  return rc;
}

int fs_attention_cost_dev(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                          const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                          fs_attn_params params, double* out_us, int32_t* status, void* stream) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
  e->last_launches = fs::launch_attention_cost(q_lens, kv_lens, offsets, is_decode, n_batches,
                                               params, out_us, status, e->n_sms, s);
  FS_CHECK(cudaGetLastError());
  return 0;
}

int fs_attention_cost(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                      const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                      fs_attn_params params, double* out_us, int32_t* status) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  const int64_t n_el = n_batches > 0 ? offsets[n_batches] : 0;
  FS_CHECK(upload(e->c_q, q_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_kv, kv_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_off, offsets, (size_t)n_batches + 1, s));
  FS_CHECK(upload(e->c_dec, is_decode, (size_t)n_batches, s));
  FS_CHECK(e->c_out.ensure((size_t)std::max<int64_t>(n_batches, 1) * 8));
  FS_CHECK(e->c_status.ensure((size_t)std::max<int64_t>(n_batches, 1) * 4));
  int rc = fs_attention_cost_dev(e, e->c_q.as<int32_t>(), e->c_kv.as<int32_t>(),
                                 e->c_off.as<int64_t>(), e->c_dec.as<uint8_t>(), n_batches, params,
                                 e->c_out.as<double>(), e->c_status.as<int32_t>(), s);
  if (rc) return rc;
  FS_CHECK(cudaMemcpyAsync(out_us, e->c_out.p, 8 * n_batches, cudaMemcpyDeviceToHost, s));
  if (status) FS_CHECK(cudaMemcpyAsync(status, e->c_status.p, 4 * n_batches, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_attention_features_dev(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                              const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                              fs_attn_params params, double* out17, void* stream) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
  e->last_launches = fs::launch_attention_features(q_lens, kv_lens, offsets, is_decode, n_batches,
                                                   params, out17, s);
  FS_CHECK(cudaGetLastError());
  return 0;
}

// host-buffer variant of the features kernel (used by parity tests)
int fs_attention_features(fs_engine* e, const int32_t* q_lens, const int32_t* kv_lens,
                          const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                          fs_attn_params params, double* out17) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  const int64_t n_el = n_batches > 0 ? offsets[n_batches] : 0;
  FS_CHECK(upload(e->c_q, q_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_kv, kv_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_off, offsets, (size_t)n_batches + 1, s));
  FS_CHECK(upload(e->c_dec, is_decode, (size_t)n_batches, s));
  FS_CHECK(e->c_out.ensure((size_t)std::max<int64_t>(n_batches, 1) * 17 * 8));
  int rc = fs_attention_features_dev(e, e->c_q.as<int32_t>(), e->c_kv.as<int32_t>(),
                                     e->c_off.as<int64_t>(), e->c_dec.as<uint8_t>(), n_batches,
                                     params, e->c_out.as<double>(), s);
  if (rc) return rc;
  FS_CHECK(cudaMemcpyAsync(out17, e->c_out.p, 17 * 8 * n_batches, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_generate_workload(fs_engine* e, const fs_workload_desc* w, int32_t n,
                         int64_t* arrival_ns, int32_t* prompt_tokens, int32_t* output_tokens,
                         int32_t* id_rank, int32_t* status) {
  if (!e) return 1;
  if (n < 0 || (n > 0 && !w)) { e->err = "fs_generate_workload: bad arguments"; return 13; }
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  int64_t total = 0;
  for (int i = 0; i < n; i++) {
    if (w[i].n_requests < 0 || w[i].out_offset < 0) {
      e->err = "fs_generate_workload: negative size or offset";
      return 13;
    }
    total = std::max(total, w[i].out_offset + w[i].n_requests);
  }
  FS_CHECK(upload(e->g_desc, w, (size_t)n, s));
  FS_CHECK(e->g_arr.ensure((size_t)std::max<int64_t>(total, 1) * 8));
  FS_CHECK(e->g_pr.ensure((size_t)std::max<int64_t>(total, 1) * 4));
  FS_CHECK(e->g_out.ensure((size_t)std::max<int64_t>(total, 1) * 4));
  FS_CHECK(e->g_rank.ensure((size_t)std::max<int64_t>(total, 1) * 4));
  FS_CHECK(e->g_st.ensure((size_t)std::max(n, 1) * 4));
  FS_CHECK(cudaMemsetAsync(e->g_st.p, 0, (size_t)std::max(n, 1) * 4, s));
  e->last_launches = fs::launch_workload(e->g_desc.as<fs_workload_desc>(), n,
                                         e->g_arr.as<int64_t>(), e->g_pr.as<int32_t>(),
                                         e->g_out.as<int32_t>(), e->g_rank.as<int32_t>(),
                                         e->g_st.as<int32_t>(), s);
  FS_CHECK(cudaGetLastError());
  if (total > 0) {
    FS_CHECK(cudaMemcpyAsync(arrival_ns, e->g_arr.p, (size_t)total * 8, cudaMemcpyDeviceToHost, s));
    FS_CHECK(cudaMemcpyAsync(prompt_tokens, e->g_pr.p, (size_t)total * 4, cudaMemcpyDeviceToHost, s));
    FS_CHECK(cudaMemcpyAsync(output_tokens, e->g_out.p, (size_t)total * 4, cudaMemcpyDeviceToHost, s));
    FS_CHECK(cudaMemcpyAsync(id_rank, e->g_rank.p, (size_t)total * 4, cudaMemcpyDeviceToHost, s));
  }
  if (n > 0) FS_CHECK(cudaMemcpyAsync(status, e->g_st.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_route_tokens(fs_engine* e, const int64_t* tokens, const uint64_t* seeds, int32_t n_calls,
                    int32_t num_experts, int32_t top_k, int32_t policy, double alpha,
                    int32_t* counts_out, int32_t* status) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  FS_CHECK(upload(e->c_tok, tokens, (size_t)n_calls, s));
  FS_CHECK(upload(e->c_seed, seeds, (size_t)n_calls, s));
  const size_t nc = (size_t)std::max(n_calls, 1) * std::max(num_experts, 1);
  FS_CHECK(e->c_counts.ensure(nc * 4));
  FS_CHECK(e->c_status.ensure((size_t)std::max(n_calls, 1) * 4));
  double* scratch = nullptr;
  if (policy == FS_ROUTE_DIRICHLET || (top_k > FS_MAX_TOPK && top_k < num_experts)) {
    FS_CHECK(e->c_scratch.ensure((size_t)fs::route_scratch_warps(n_calls) * fs::kDirScratch * 8));
    scratch = e->c_scratch.as<double>();
  }
  e->last_launches = fs::launch_route_tokens(e->c_tok.as<int64_t>(), e->c_seed.as<uint64_t>(),
                                             n_calls, num_experts, top_k, policy, alpha, scratch,
                                             e->c_counts.as<int32_t>(), e->c_status.as<int32_t>(),
                                             s);
  FS_CHECK(cudaGetLastError());
  FS_CHECK(cudaMemcpyAsync(counts_out, e->c_counts.p, 4 * (size_t)n_calls * num_experts,
                           cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaMemcpyAsync(status, e->c_status.p, 4 * (size_t)n_calls, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_eval(fs_engine* e, int32_t fn, const double* in, int32_t in_stride, int64_t n,
            double* out, int32_t out_stride, int32_t* status) {
  if (!e) return 1;
  if (n < 0 || in_stride < 1 || out_stride < 1) { e->err = "fs_eval: bad sizes"; return 1; }
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  FS_CHECK(upload(e->c_ein, in, (size_t)n * in_stride, s));
  FS_CHECK(e->c_eout.ensure((size_t)std::max<int64_t>(n, 1) * out_stride * 8));
  FS_CHECK(e->c_status.ensure((size_t)std::max<int64_t>(n, 1) * 4));
  FS_CHECK(cudaMemsetAsync(e->c_eout.p, 0, (size_t)std::max<int64_t>(n, 1) * out_stride * 8, s));
  e->last_launches = fs::launch_eval(fn, e->c_ein.as<double>(), in_stride, n,
                                     e->c_eout.as<double>(), out_stride,
                                     e->c_status.as<int32_t>(), e->n_sms, s);
  FS_CHECK(cudaGetLastError());
  if (n > 0) {
    FS_CHECK(cudaMemcpyAsync(out, e->c_eout.p, (size_t)n * out_stride * 8, cudaMemcpyDeviceToHost, s));
    FS_CHECK(cudaMemcpyAsync(status, e->c_status.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  }
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_route_uniform(fs_engine* e, const int64_t* tokens, const uint64_t* seeds, int32_t n_calls,
                     int32_t num_experts, int32_t top_k, int32_t* counts_out, int32_t* status) {
  return fs_route_tokens(e, tokens, seeds, n_calls, num_experts, top_k, FS_ROUTE_UNIFORM, 0.3,
                         counts_out, status);
}

int fs_set_forests(fs_engine* e, fs_forest_set f) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  for (int i = 0; i < f.n_forests; i++) {
    const fs_forest_desc& d = f.forests[i];
    if (d.n_trees < 1 || d.n_trees > fs::kMaxForestTrees || d.tree_offset < 0 ||
        d.tree_offset + d.n_trees > f.n_trees) {
      e->err = "forest " + std::to_string(i) + ": bad tree range (1 <= n_trees <= 256)";
      return 12;
    }
  }
  // pack (threshold | leaf value, feature, left) into 16-byte nodes
  std::vector<fs::NodeP> packed((size_t)f.n_nodes);
  int consecutive = 1;
  for (int64_t i = 0; i < f.n_nodes; i++) {
    const bool leaf = f.feature[i] < 0;
    packed[i].v = leaf ? f.value[i] : f.threshold[i];
    packed[i].feature = f.feature[i];
    packed[i].left = f.left[i];
    if (!leaf) {
      if (f.feature[i] >= 17 || f.left[i] < 0 || f.left[i] >= f.n_nodes || f.right[i] < 0 ||
          f.right[i] >= f.n_nodes) {
        e->err = "forest node " + std::to_string(i) + ": feature or child index out of range";
        return 12;
      }
      if (f.right[i] != f.left[i] + 1) consecutive = 0;
    }
  }
  // leaf value ranks: the device sorts 32-bit ranks instead of fp64 values
  std::vector<double> leafv;
  for (int64_t i = 0; i < f.n_nodes; i++)
    if (f.feature[i] < 0) leafv.push_back(f.value[i]);
  std::sort(leafv.begin(), leafv.end());
  for (int64_t i = 0; i < f.n_nodes; i++)
    if (f.feature[i] < 0) {
      if (!(f.value[i] == f.value[i])) {
        e->err = "forest node " + std::to_string(i) + ": NaN leaf value";
        return 12;
      }
      packed[i].left =
          (int32_t)(std::lower_bound(leafv.begin(), leafv.end(), f.value[i]) - leafv.begin());
    }
  for (int64_t t = 0; t < f.n_trees; t++)
    if (f.tree_root[t] < 0 || f.tree_root[t] >= f.n_nodes) {
      e->err = "forest tree " + std::to_string(t) + ": root out of range";
      return 12;
    }
  FS_CHECK(upload(e->f_descs, f.forests, (size_t)f.n_forests, s));
  FS_CHECK(upload(e->f_roots, f.tree_root, (size_t)f.n_trees, s));
  FS_CHECK(upload(e->f_value, packed.data(), packed.size(), s));
  FS_CHECK(upload(e->f_right, f.right, (size_t)f.n_nodes, s));
  FS_CHECK(upload(e->f_leaf, leafv.data(), leafv.size(), s));
  FS_CHECK(cudaStreamSynchronize(s));
  e->fv.forests = e->f_descs.as<fs_forest_desc>();
  e->fv.n_forests = f.n_forests;
  e->fv.consecutive = consecutive;
  e->fv.tree_root = e->f_roots.as<int64_t>();
  e->fv.nodes = e->f_value.as<fs::NodeP>();
  e->fv.right = e->f_right.as<int32_t>();
  e->fv.leaf_by_rank = e->f_leaf.as<double>();
  e->params.fv = e->fv;
  e->forest_gen++;
  return 0;
}

int fs_attention_forest_dev(fs_engine* e, int32_t forest, const int32_t* q_lens,
                            const int32_t* kv_lens, const int64_t* offsets,
                            const uint8_t* is_decode, int64_t n_batches, fs_attn_params params,
                            double* out_us, void* stream) {
  if (!e) return 1;
  if (forest < 0 || forest >= e->fv.n_forests) {
    e->err = "forest index out of range (stage models with fs_set_forests)";
    return 13;
  }
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
  e->last_launches = fs::launch_attention_forest(e->fv, forest, q_lens, kv_lens, offsets, is_decode,
                                                 n_batches, params, out_us, e->n_sms, s);
  FS_CHECK(cudaGetLastError());
  return 0;
}

int fs_attention_forest(fs_engine* e, int32_t forest, const int32_t* q_lens, const int32_t* kv_lens,
                        const int64_t* offsets, const uint8_t* is_decode, int64_t n_batches,
                        fs_attn_params params, double* out_us) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  const int64_t n_el = n_batches > 0 ? offsets[n_batches] : 0;
  FS_CHECK(upload(e->c_q, q_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_kv, kv_lens, (size_t)n_el, s));
  FS_CHECK(upload(e->c_off, offsets, (size_t)n_batches + 1, s));
  FS_CHECK(upload(e->c_dec, is_decode, (size_t)n_batches, s));
  FS_CHECK(e->c_out.ensure((size_t)std::max<int64_t>(n_batches, 1) * 8));
  int rc = fs_attention_forest_dev(e, forest, e->c_q.as<int32_t>(), e->c_kv.as<int32_t>(),
                                   e->c_off.as<int64_t>(), e->c_dec.as<uint8_t>(), n_batches,
                                   params, e->c_out.as<double>(), s);
  if (rc) return rc;
  FS_CHECK(cudaMemcpyAsync(out_us, e->c_out.p, 8 * n_batches, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

int fs_router_seeds(fs_engine* e, const fs_seed_prefix* prefixes, const int32_t* prefix_idx,
                    const int32_t* micro_batch, const int64_t* steps, const int32_t* layers,
                    int32_t n, uint32_t* seeds_out) {
  if (!e) return 1;
  FS_CHECK(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  int np = 0;
  for (int i = 0; i < n; i++) np = std::max(np, prefix_idx[i] + 1);
  FS_CHECK(upload(e->c_pf, prefixes, (size_t)np, s));
  FS_CHECK(e->c_mid.ensure((size_t)std::max(np, 1) * 32));
  fs::launch_midstate(e->c_pf.as<fs_seed_prefix>(), e->c_mid.as<uint32_t>(), np, s);
  FS_CHECK(upload(e->c_pidx, prefix_idx, (size_t)n, s));
  FS_CHECK(upload(e->c_mb, micro_batch, (size_t)n, s));
  FS_CHECK(upload(e->c_steps, steps, (size_t)n, s));
  FS_CHECK(upload(e->c_layers, layers, (size_t)n, s));
  FS_CHECK(e->c_seeds.ensure((size_t)std::max(n, 1) * 4));
  e->last_launches = 1 + fs::launch_router_seeds(e->c_pf.as<fs_seed_prefix>(), e->c_mid.as<uint32_t>(),
                                                 e->c_pidx.as<int32_t>(), e->c_mb.as<int32_t>(),
                                                 e->c_steps.as<int64_t>(), e->c_layers.as<int32_t>(),
                                                 n, e->c_seeds.as<uint32_t>(), s);
  FS_CHECK(cudaGetLastError());
  FS_CHECK(cudaMemcpyAsync(seeds_out, e->c_seeds.p, 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
  FS_CHECK(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
