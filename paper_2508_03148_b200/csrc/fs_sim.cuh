// fs_sim.cuh -- batched discrete-event simulation of independent Frontier
// instances: one warp per instance, state as struct-of-arrays in HBM.
//
// Reference behaviour restated here (pkg/src/frontier_sim/...):
//   core.py:135-211           (timestamp, seq) event order, event budget
//   orchestrator/base.py      kick / start_batch / complete_request / run
//   orchestrator/colocated.py round-robin, prefill-first, continuous batching
//   orchestrator/pd.py        least-outstanding prefill routing, FIFO KV transfer
//                             queue with decode-memory backpressure
//   orchestrator/af.py        AF step graph under 4 exclusive resources
//   cluster.py                KvPool, admission (fcfs / fcfs_skip / priority),
//                             OperatorCosts, execute_batch
//   metrics.py:81-178         compute_metrics (separate kernel, fs_metrics.cu)
//
// Design (B200-first, not a translation of the reference's object graph):
//  * Only state-changing events live in a per-instance binary heap (BATCH_START,
//    BATCH_COMPLETE, KV_CACHE_TRANSFER_DONE); arrivals are a sorted cursor that
//    wins timestamp ties (they hold seq 0..N-1, base.py:167-177). The no-op
//    event kinds are counted, not stored -- skipping their sequence numbers
//    preserves the relative order of every stored event.
//  * A running request's completion step is known when it starts decoding, so
//    a decode iteration is O(1): batch size and context sum are maintained
//    incrementally and the running list is scanned only when the earliest
//    finish step is reached.
//  * Admission is a warp prefix-scan over the queue with a ballot for the
//    first request that does not fit (fcfs / priority) or an iterative ballot
//    (fcfs_skip).
//  * The AF step graph (af.py:100-229) is list-scheduled in closed form per
//    step; only its completion becomes an event.
//  * MoE routing is warp-cooperative Philox (fs_route.cuh); per-layer router
//    seeds (SHA-256 + two SeedSequence hashes) are derived one layer per lane.
//
// Per-warp scalar state is held redundantly in every lane's registers; global
// scalar writes are issued by lane 0 and ordered with __syncwarp().
#pragma once
// Compiled twice (fs_engine.cu, fs_engine_learned.cu): FS_LEARNED selects the
// learned attention model call sites, FS_SIM_NS the namespace of the variant.
#include <cuda_runtime.h>

#include "fs_device.cuh"
#include "fs_engine.h"
#include "fs_route.cuh"
#include "fs_dirichlet.cuh"

// compile-time knobs (scripts/variants.py builds and times alternatives)
#ifndef FS_PHILOX_ILP  // Philox blocks per lane in flight in the routing pass (1 measured best)
#define FS_PHILOX_ILP 1
#endif
#ifndef FS_DIR_IN_ANALYTIC
#define FS_DIR_IN_ANALYTIC 0
#endif
#ifndef FS_MODES  // serving modes compiled in: 1 colocated | 2 pd | 4 af
#define FS_MODES 7
#endif
#define FS_HAS_PD ((FS_MODES & 2) != 0)
#define FS_HAS_AF ((FS_MODES & 4) != 0)
#ifndef FS_DENSE_ONLY  // the MoE paths compiled out (the dense wave's kernel variant)
#define FS_DENSE_ONLY 0
#endif
#ifndef FS_TOPK_BRANCHFREE  // insert every key (no threshold test): in a warp some lane
#define FS_TOPK_BRANCHFREE 0  // almost always inserts, so the test only adds instructions
#endif
#ifndef FS_KCAP_MAX  // largest top-(k+1) list compiled in (4: k <= 3 only -- a variant for
#define FS_KCAP_MAX 17  // small-k MoE batches, whose routing then needs fewer registers)
#endif
#ifndef FS_LONG_ROW_UNROLL  // unrolled Philox rounds for long row segments (>= 64 draws):
#define FS_LONG_ROW_UNROLL 0  // C4 EP 430 -> 373 ms, but the C5 sweep 272 -> ~300 ms (code size)
#endif

namespace fs {
namespace FS_SIM_NS {

enum { K_BATCH_START = 1, K_BATCH_COMPLETE = 2, K_KV_DONE = 3 };
enum { PH_PREFILL = 0, PH_DECODE = 1, PH_AF = 2 };

constexpr int kWarpsPerCta = 4;
constexpr int kLayerChunk = 32;
constexpr int kSlabBytes = 12 * 1024;  // per-warp shared-memory slab for hot instance state
constexpr int32_t kNoFinish = 0x7fffffff;

#ifndef FS_TERM_MEMO  // memo of the batch terms that depend on n alone (analytic variants):
#define FS_TERM_MEMO (!FS_LEARNED)  // C5 dense wave 40.9 -> 30 ms, MoE wave -5 ms
#endif
constexpr int kMemoSlots = 32;  // direct-mapped on n_tokens (a decode batch's n <= 32 maps 1:1)
// One memo line: the n-only terms of execute_batch (qkv, out, ffn, tp all-reduce,
// pp transfers) for one (n, cost context); the context is compared bit for bit.
struct TermMemo {
  double qkv, out, ffn, coll, pp;
  double peak, bw, ovh;
  int64_t n;
  int32_t tp, ppd;
};

struct __align__(16) WarpSmem {
  uint64_t keys[kLayerChunk][2];
  int64_t af_attn[FS_MAX_MICRO_BATCHES];
  int64_t af_xfer[FS_MAX_MICRO_BATCHES];
  int32_t af_size[FS_MAX_MICRO_BATCHES];
  int32_t af_stage[FS_MAX_MICRO_BATCHES];
#if FS_TERM_MEMO && FS_DENSE_ONLY
  union {  // the dense variant never routes, so the tally space holds the memo
    int counts[FS_MAX_EXPERTS];
    TermMemo memo[kMemoSlots];
  };
#else
  int counts[FS_MAX_EXPERTS];
#if FS_TERM_MEMO
  TermMemo memo[kMemoSlots];
#endif
#endif
#if FS_LEARNED
  double fx[17];                   // learned attention model: feature vector
  double fvals[kMaxForestTrees];   // ... and per-tree leaf values
#endif
};

struct Inst {
  const fs_instance_desc* d;
  int idx, N, R, mode, lane, slot;
  int64_t ro;      // request offset (global index of local request 0)
  int rb;          // global index of local replica 0
  int32_t* lists;  // 3*N ints per replica: queue, running, inflight members
  HEv* heap;
  RepState* rs;    // replica states (shared-memory slab or HBM)
  int32_t* fin;    // per-request finish step, local index (slab or HBM)
  int hn;
  int64_t now, seq, events, max_events;
  int rr, n_done, cursor;
  int status, detail;
  int xh, xt;  // PD transfer FIFO (ring of N slots at xfer + ro)
  int64_t af_counter;
  int64_t af_busy[4];
  double bubble_weighted;
  int64_t bubble_total;
  int64_t prefill_batches, decode_batches, af_steps, moe_samples, routing_calls, routing_draws;
  int32_t log_batches, log_moff, log_eoff, log_routes;
};

__device__ __forceinline__ int32_t* qlist(const Inst& I, int r) { return I.lists + (int64_t)r * 3 * I.N; }
__device__ __forceinline__ int32_t* rlist(const Inst& I, int r) { return qlist(I, r) + I.N; }
__device__ __forceinline__ int32_t* ilist(const Inst& I, int r) { return qlist(I, r) + 2 * I.N; }
__device__ __forceinline__ int64_t gi(const Inst& I, int i) { return I.ro + i; }

__device__ __forceinline__ void fail(Inst& I, int st, int detail) {
  if (I.status == FS_OK) { I.status = st; I.detail = detail; }
}

// ---- replica state: every lane loads the same struct; lane 0 stores -------------
// Every write of a replica state is store_rep (lane 0, then __syncwarp) or the
// initialisation loop (followed by __syncwarp), so a load needs no barrier of
// its own; store_rep's leading barrier orders the other lanes' loads before the
// overwrite.
#ifndef FS_LOADREP_SYNC
#define FS_LOADREP_SYNC 0
#endif
__device__ __forceinline__ RepState load_rep(const EngineParams& P, const Inst& I, int r) {
  if (FS_LOADREP_SYNC) __syncwarp();
  return I.rs[r];
}
__device__ __forceinline__ void store_rep(const EngineParams& P, const Inst& I, int r,
                                          const RepState& s) {
  __syncwarp();
  if (I.lane == 0) I.rs[r] = s;
  __syncwarp();
}

// ---- event heap (lane 0 mutates, the popped event is broadcast) ----------------
// Only lane 0 ever reads or writes heap memory, so no warp barrier guards it; the
// other lanes track the size (I.hn) and the sequence counter in their registers
// and receive the popped event by shuffle.
__device__ __forceinline__ bool hev_less(const HEv& a, const HEv& b) {
  return a.t < b.t || (a.t == b.t && a.seq < b.seq);
}
__device__ void heap_push(Inst& I, int64_t t, int kind, int a, int64_t b) {
  if (t < I.now) { fail(I, FS_ERR_SCHEDULING_IN_PAST, kind); return; }
  if (I.lane == 0) {
    HEv e;
    e.t = t; e.seq = I.seq; e.kind = kind; e.a = a; e.b = b;
    int i = I.hn;
    while (i > 0) {
      int p = (i - 1) >> 1;
      HEv pe = I.heap[p];
      if (!hev_less(e, pe)) break;
      I.heap[i] = pe;
      i = p;
    }
    I.heap[i] = e;
  }
  I.hn++;
  I.seq++;
}
__device__ HEv heap_pop(Inst& I) {
  HEv top;
  top.t = 0; top.seq = 0; top.kind = 0; top.a = 0; top.b = 0;
  if (I.lane == 0) {
    top = I.heap[0];
    const int n = I.hn - 1;
    const HEv last = I.heap[n];
    int i = 0;
    for (;;) {
      int l = 2 * i + 1, r = l + 1, m = -1;
      HEv cur = last;
      if (l < n) { HEv le = I.heap[l]; if (hev_less(le, cur)) { m = l; cur = le; } }
      if (r < n) { HEv re = I.heap[r]; if (hev_less(re, cur)) { m = r; cur = re; } }
      if (m < 0) break;
      I.heap[i] = cur;
      i = m;
    }
    if (n > 0) I.heap[i] = last;
  }
  I.hn--;
  top.t = __shfl_sync(FS_FULL, top.t, 0);
  top.kind = __shfl_sync(FS_FULL, top.kind, 0);
  top.a = __shfl_sync(FS_FULL, top.a, 0);
  top.b = __shfl_sync(FS_FULL, top.b, 0);
  return top;
}
__device__ __forceinline__ int64_t heap_top_t(const Inst& I) {
  int64_t t = 0;
  if (I.lane == 0) t = I.heap[0].t;
  return __shfl_sync(FS_FULL, t, 0);
}

// ---- KvPool (cluster.py:36-93): every reservation here is a request's first in
// its pool, so the charge is rounded(tokens) and release returns the same ----------
__device__ __forceinline__ int64_t pool_rounded(const fs_instance_desc* d, int64_t tokens) {
  if (!d->paged) return tokens;
  const int64_t b = d->block_tokens;
  return (tokens + b - 1) / b * b;
}

// ---- OperatorCosts (cluster.py:252-314) ----------------------------------------------
__device__ __forceinline__ void heads_of(const fs_instance_desc* d, int tp, int& hq, int& hkv) {
  hq = d->num_query_heads / tp; if (hq < 1) hq = 1;
  hkv = d->num_kv_heads / tp; if (hkv < 1) hkv = 1;
}
__device__ __forceinline__ double qkv_us(const fs_instance_desc* d, const fs_cost_ctx& c, int64_t n) {
  int hq, hkv;
  heads_of(d, c.tp, hq, hkv);
  return linear_us(n, (int64_t)(hq + 2 * hkv) * d->head_dim, d->d_model, c, d->dtype_bytes);
}
__device__ __forceinline__ double out_us(const fs_instance_desc* d, const fs_cost_ctx& c, int64_t n) {
  int hq, hkv;
  heads_of(d, c.tp, hq, hkv);
  return linear_us(n, d->d_model, (int64_t)hq * d->head_dim, c, d->dtype_bytes);
}
__device__ __forceinline__ double tpcoll_us(const fs_instance_desc* d, const fs_cost_ctx& c, int64_t n) {
  const int64_t b = n * (int64_t)d->d_model * d->dtype_bytes;
  return collective_int(true, b, c.tp, d->intra_latency_s, d->intra_bandwidth_bps) * 1e6;
}
__device__ __forceinline__ double dense_ffn_us(const fs_instance_desc* d, const fs_cost_ctx& c, int64_t n) {
  int64_t dff = d->d_ff / c.tp;
  if (dff < 1) dff = 1;
  return grouped_gemm_us(n, 1, d->d_model, dff, d->ffn_matrices, c, d->dtype_bytes);
}
__device__ __forceinline__ double attn_cost_us(const fs_instance_desc* d, const fs_cost_ctx& c,
                                               double flops, int64_t sum_q, int64_t sum_kv) {
  int hq, hkv;
  heads_of(d, c.tp, hq, hkv);
  return attention_us_from(flops, sum_q, sum_kv, hq, hkv, d->head_dim, c, d->dtype_bytes);
}

// ---- router seeds for 32 layers at a time, one layer per lane --------------------------
__device__ void derive_layer_keys(const EngineParams& P, const Inst& I, int prefix, int mb,
                                  int64_t step, int l0, int L, WarpSmem* sm) {
  __syncwarp();
  const int layer = l0 + I.lane;
  if (layer < L) {
    const fs_seed_prefix* pf = &P.prefixes[prefix];
    int64_t ints[3];
    int n = 0;
    if (mb > 0) ints[n++] = mb;
    ints[n++] = step;
    ints[n++] = layer;
    int tl;
    const uint8_t* tail = prefix_tail(pf, tl);
    const uint32_t seed = sha256_tail_first_word(P.midstate + (int64_t)prefix * 8, pf->mid_blocks,
                                                 tail, tl, ints, n);
    uint64_t key[2];
    routing_key((uint64_t)seed, key);
    sm->keys[I.lane][0] = key[0];
    sm->keys[I.lane][1] = key[1];
  }
  __syncwarp();
}


// keys a router call draws (T x E; none for the trace policy and the RNG-free shortcuts)
__device__ __forceinline__ int64_t draws_of(const fs_instance_desc* d, int policy, int64_t T) {
  return (policy != FS_ROUTE_TRACE && T > 0 && d->top_k < d->num_experts)
             ? T * (int64_t)d->num_experts : 0;
}

// ---- one router call (routing.py:65-113) ------------------------------------------------
__device__ int route_layer(const EngineParams& P, const Inst& I, int policy, int64_t T,
                           uint64_t k0, uint64_t k1, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  const int E = d->num_experts, k = d->top_k;
  if (!(1 <= k && k <= E)) return FS_ERR_INVALID_TOPK;
  if (E > FS_MAX_EXPERTS) return FS_ERR_CAPACITY;
  if (T < 0) return FS_ERR_ROUTING;
  if (policy == FS_ROUTE_TRACE) {
    if (d->n_trace_counts != E) return FS_ERR_ROUTING;
    int64_t s = 0;
    int neg = 0;
    __syncwarp();
    for (int e = I.lane; e < E; e += 32) {
      const int64_t c = P.trace_counts[d->trace_offset + e];
      neg |= c < 0;
      s += c;
      sm->counts[e] = (int)c;
    }
    __syncwarp();
    s = warp_sum_i64(s);
    neg = __any_sync(FS_FULL, neg);
    if (neg || s != T * k) return FS_ERR_ROUTING;
    return FS_OK;
  }
  if (T == 0 || k == E || policy == FS_ROUTE_UNIFORM) {
    if (T > 0 && k < E && k > FS_MAX_TOPK) {
#if FS_LEARNED  // rows sorted whole; instances with such a top_k run in this variant
      if (!P.dir_scratch) return FS_ERR_INTERNAL;
      __syncwarp();
      return route_uniform_sorted(I.lane, T, E, k, k0, k1,
                                  P.dir_scratch + (int64_t)I.slot * kDirScratch, sm->counts);
#else
      return FS_ERR_INTERNAL;  // host dispatch error: top_k > FS_MAX_TOPK runs in `learned`
#endif
    }
    __syncwarp();
    return route_uniform_warp(I.lane, T, E, k, k0, k1, sm->counts);
  }
#if FS_LEARNED || FS_DIR_IN_ANALYTIC
  // dirichlet_skew instances run in the extended (learned) variant of this kernel:
  // the call would cost the analytic variant's register allocation
  if (policy == FS_ROUTE_DIRICHLET)
    return route_dirichlet_warp(I.lane, T, E, k, d->routing_alpha, k0, k1,
                                P.dir_scratch + (int64_t)I.slot * kDirScratch, sm->counts);
#endif
  return policy == FS_ROUTE_DIRICHLET ? FS_ERR_INTERNAL : FS_ERR_ROUTING;
}

__device__ void log_route(const EngineParams& P, Inst& I, int r, int mb, int64_t step, int layer,
                          int64_t T, const WarpSmem* sm) {
  if (!P.log_enabled || !P.log.routes) return;
  const int E = I.d->num_experts;
  const int32_t c = I.log_routes;
  const int64_t cb = (int64_t)c * E;
  if (c < P.log.route_cap && cb + E <= P.log.counts_cap) {
    if (I.lane == 0) {
      fs_route_rec rec;
      rec.replica = r; rec.micro_batch = mb; rec.step = step; rec.layer = layer;
      rec.tokens = (int32_t)T; rec.counts_offset = (int32_t)cb; rec.n_experts = E;
      P.log.routes[P.log.route_base[I.idx] + c] = rec;
    }
    for (int e = I.lane; e < E; e += 32) P.log.counts[P.log.counts_base[I.idx] + cb + e] = sm->counts[e];
    I.log_routes = c + 1;
  } else if (I.lane == 0) {
    P.log.truncated[I.idx] = 1;
  }
  __syncwarp();
}

// ---- routing job board -----------------------------------------------------------------------
// One batch's uniform router calls (up to kJobLayers layers x T tokens x E
// experts of Philox draws) dwarf everything else an MoE instance does, and a
// sweep's MoE instances are its longest. So the owning warp publishes the
// calls as a job of row chunks on a GPU-wide board; it works on its own job,
// and every warp whose share of the instance queue is exhausted scans the
// board and claims chunks of other warps' jobs. A claimed chunk pins its job
// (the job cannot complete, hence cannot be replaced, until the chunk's
// completion is counted), so chunk parameters are stable for the claimant.
// Counts land in the job's global tally with warp-aggregated atomics; the owner
// waits for every chunk, fences, and reads the tally through L2.
constexpr unsigned kChunkBits = 20;
constexpr unsigned long long kChunkMask = (1ull << kChunkBits) - 1;
constexpr int kMaxChunks = 1 << 18;
#ifndef FS_CHUNK_BLOCKS  // Philox blocks per lane per claimed chunk (96: 267 ms, 48: 276, 16: 350)
#define FS_CHUNK_BLOCKS 96
#endif
constexpr int kChunkBlocks = FS_CHUNK_BLOCKS;
#ifndef FS_ROWS_PATH  // whole-row, whole-block routing passes for top_k 1-3 and 8 (process_rows)
#define FS_ROWS_PATH 1
#endif
#ifndef FS_NSEG_ROWS  // rows are split into lane segments while rows * nseg stays below this
#define FS_NSEG_ROWS 64  // 64: C5 224-226 ms; 256: 225-228; 2048 (round 1): ~228; 4096: 232-236
#endif

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ int ld_volatile_i32(const int32_t* p) {
  return *reinterpret_cast<const volatile int32_t*>(p);
}

// acquire / release atomics (cheaper than a full __threadfence per chunk)
__device__ __forceinline__ unsigned long long atom_add_acquire_u64(unsigned long long* p,
                                                                   unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acquire.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_i32(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_i32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// returns a claimed chunk index or -1 (same on all lanes). The claim is an
// acquire (the job parameters were written before the job was published with a
// release), passed on to the other lanes by __syncwarp; the claimant of the
// last chunk closes the job.
__device__ int claim_chunk(const EngineParams& P, RouteJob* job, int lane) {
  long long c = -1;
  if (lane == 0) {
    const unsigned long long v = ld_volatile_u64(&job->ctr);
    if ((v & kChunkMask) < ((v >> kChunkBits) & kChunkMask)) {
      const unsigned long long old = atom_add_acquire_u64(&job->ctr, 1ull);
      const unsigned long long n = (old >> kChunkBits) & kChunkMask;
      if ((old & kChunkMask) < n) {
        c = (long long)(old & kChunkMask);
        if ((unsigned long long)c + 1 == n) atomicSub(P.open_jobs, 1);
      }
    }
  }
  __syncwarp();
  c = __shfl_sync(FS_FULL, c, 0);
  return (int)c;
}

// One pass: lane (row r of `layer`, segment seg) keeps the kc smallest keys of
// its draws. Fast path: 32-bit surrogate keys (the top 32 bits of each draw,
// whose order agrees with the 53-bit key except on a tie of those bits) with
// the expert index in the low `eb` bits; the set is exact unless the k-th and
// (k+1)-th surrogates tie above the index bits, in which case the pass is
// redone with the exact 64-bit keys (which also detects a true tie).
template <int KCAP>
__device__ __forceinline__ void pass_fast(uint32_t (&top)[KCAP], int kc, bool active, uint64_t rb,
                                          int e0, int e1, uint32_t emask, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int j = 0; j < KCAP; j++) top[j] = 0xFFFFFFFFu;
  uint32_t thr = 0xFFFFFFFFu;
  if (!active || e0 >= e1) return;
  const uint64_t n0 = rb + e0, n1 = rb + e1;
  auto consume = [&](const U4& blk, uint64_t b) {
    const uint64_t base = 4 * b;
    const int jlo = n0 > base ? (int)(n0 - base) : 0;
    const int jhi = (n1 - base) < 4 ? (int)(n1 - base) : 4;
    const uint32_t eb0 = (uint32_t)(base - rb);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j >= jlo && j < jhi) {
        uint32_t x = ((uint32_t)(blk.v[j] >> 32) & ~emask) | (eb0 + (uint32_t)j);
        if (KCAP <= 4 || FS_TOPK_BRANCHFREE || x < thr) {
#pragma unroll
          for (int q = 0; q < KCAP; q++) {
            const uint32_t lo = min(top[q], x);
            x = max(top[q], x);
            top[q] = lo;
          }
          if (KCAP > 4 && !FS_TOPK_BRANCHFREE) {
#pragma unroll
            for (int q = 0; q < KCAP; q++)
              if (q == kc - 1) thr = top[q];
          }
        }
      }
    }
  };
#if FS_PHILOX_ILP >= 2
  // two blocks per step (a trailing odd block is generated and ignored)
  const uint64_t blast = (n1 - 1) >> 2;
  for (uint64_t b = n0 >> 2; b <= blast; b += 2) {
    U4 A, B;
    philox4x64_10_x2(b + 1, b + 2, k0, k1, A, B);
    consume(A, b);
    if (b + 1 <= blast) consume(B, b + 1);
  }
#else
  if (FS_LONG_ROW_UNROLL && n1 - n0 >= 64) {
    // long rows (E >= 64 per segment): the unrolled rounds, see philox4x64_10_unrolled
    for (uint64_t b = n0 >> 2; b <= (n1 - 1) >> 2; b++)
      consume(philox4x64_10_unrolled(b + 1, k0, k1), b);
  } else {
    for (uint64_t b = n0 >> 2; b <= (n1 - 1) >> 2; b++) consume(philox4x64_10(b + 1, k0, k1), b);
  }
#endif
}


template <int KCAP>
__device__ void process_chunk_k(const EngineParams& P, RouteJob* job, int32_t* counts, int c,
                                int lane, int* tally) {
  const int64_t T = __ldcg(&job->T);
  const int E = __ldcg(&job->E), k = __ldcg(&job->k), nl = __ldcg(&job->nl);
  const int nseg = __ldcg(&job->nseg), ppc = __ldcg(&job->passes_per_chunk);
  const int rpp = 32 / nseg;
  const int seg_len = (E + nseg - 1) / nseg;
  const int64_t total_rows = (int64_t)nl * T;
  const int kc = k + 1;
  const int seg = lane & (nseg - 1);
  const int e0 = seg * seg_len, e1 = min(E, e0 + seg_len);
  int eb = 0;
  while ((1 << eb) < E) eb++;
  const uint32_t emask = (1u << eb) - 1u;
  int tie = 0;
  // this lane's first row; later passes advance it incrementally (no division)
  const int64_t row0 = (int64_t)c * ppc * rpp;
  int64_t row_j = row0 + lane / nseg;
  int layer = (int)(row_j / T);
  int64_t r = row_j - (int64_t)layer * T;
  int key_layer = -1;
  uint64_t k0 = 0, k1 = 0;
  // the chunk's tally goes to the warp's shared-memory histogram when the
  // layers it spans fit (flushed once at the end), else straight to global
  const int64_t row_end = min(total_rows, row0 + (int64_t)ppc * rpp);
  const int l_first = (int)(row0 / T);
  const int span = row_end > row0 ? (int)((row_end - 1) / T) - l_first + 1 : 0;
  const bool local = span * E <= FS_MAX_EXPERTS;
  if (local) {
    for (int i = lane; i < span * E; i += 32) tally[i] = 0;
    __syncwarp();
  }
  for (int p = 0; p < ppc; p++) {
    if (row0 + (int64_t)p * rpp >= total_rows) break;
    const bool active = row_j < total_rows;
    if (active && layer != key_layer) {
      k0 = __ldcg(&job->keys[layer][0]);
      k1 = __ldcg(&job->keys[layer][1]);
      key_layer = layer;
    }
    const uint64_t rb = (uint64_t)r * (uint64_t)E;
    uint32_t top[KCAP];
    pass_fast<KCAP>(top, kc, active, rb, e0, e1, emask, k0, k1);
    for (int s = 1; s < nseg; s <<= 1) {
      uint32_t other[KCAP];
#pragma unroll
      for (int j = 0; j < KCAP; j++) other[j] = __shfl_xor_sync(FS_FULL, top[j], s);
#pragma unroll
      for (int j = 0; j < KCAP; j++) {
        uint32_t x = other[j];
#pragma unroll
        for (int q = 0; q < KCAP; q++) {
          const uint32_t lo = min(top[q], x);
          x = max(top[q], x);
          top[q] = lo;
        }
      }
    }
    const bool leader = active && seg == 0;
    bool unsure = false;
#pragma unroll
    for (int j = 1; j < KCAP; j++)
      if (j == k && leader && (top[j] >> eb) == (top[j - 1] >> eb)) unsure = true;
    int ids[KCAP];
#pragma unroll
    for (int j = 0; j < KCAP; j++) ids[j] = (int)(top[j] & emask);
    if (__any_sync(FS_FULL, unsure)) {
      // exact 64-bit redo of this pass
      uint64_t t64[KCAP];
#pragma unroll
      for (int j = 0; j < KCAP; j++) t64[j] = ~0ull;
      uint64_t thr = ~0ull;
      if (active && e0 < e1) topk_scan<KCAP>(t64, kc, thr, rb + e0, rb + e1, rb, k0, k1);
      for (int s = 1; s < nseg; s <<= 1) {
        uint64_t other[KCAP];
#pragma unroll
        for (int j = 0; j < KCAP; j++) other[j] = __shfl_xor_sync(FS_FULL, t64[j], s);
#pragma unroll
        for (int j = 0; j < KCAP; j++)
          if (j < kc) topk_insert<KCAP>(t64, kc, other[j], thr);
      }
#pragma unroll
      for (int j = 0; j < KCAP; j++) {
        ids[j] = (int)(t64[j] & 0x7FF);
        if (j == k && leader && ((t64[j] >> 11) == (t64[j > 0 ? j - 1 : 0] >> 11))) tie = 1;
      }
    }
    if (local) {
      if (leader) {
#pragma unroll
        for (int j = 0; j < KCAP; j++)
          if (j < k) atomicAdd(&tally[(layer - l_first) * E + ids[j]], 1);
      }
    } else {
#pragma unroll
      for (int j = 0; j < KCAP; j++) {
        if (j < k) {
          const int key = leader ? layer * E + ids[j] : -1;
          const unsigned grp = __match_any_sync(FS_FULL, key);
          if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(&counts[key], __popc(grp));
        }
      }
    }
    r += rpp;
    row_j += rpp;
    while (r >= T) { r -= T; layer++; }
  }
  if (local) {
    __syncwarp();
    for (int i = lane; i < span * E; i += 32) {
      const int v = tally[i];
      if (v) atomicAdd(&counts[l_first * E + i], v);
    }
    __syncwarp();
  }
  if (__any_sync(FS_FULL, tie) && lane == 0) atomicExch(&job->tie, FS_ERR_ROUTING_TIE);
}

// Whole rows per lane (nseg == 1) of whole Philox blocks (E % 4 == 0, so a row's draws
// start block-aligned): the row's E/4 blocks with no per-draw range predicates, 32-bit
// expert indices and a sorted list of exactly k+1 surrogate keys (k+1 min/max pairs
// per draw). Same selection, tie test and exact redo as process_chunk_k; this is
// every decode-batch call of the C5 Mixtral family (k = 2) and of DeepSeek-V3 (k = 8).
template <int KC>
__device__ void process_rows(const EngineParams& P, RouteJob* job, int32_t* counts, int c,
                             int lane, int* tally) {
  constexpr int k = KC - 1;
  const int64_t T = __ldcg(&job->T);
  const int E = __ldcg(&job->E), nl = __ldcg(&job->nl);
  const int ppc = __ldcg(&job->passes_per_chunk);
  const int64_t total_rows = (int64_t)nl * T;
  int eb = 0;
  while ((1 << eb) < E) eb++;
  const uint32_t keep = ~((1u << eb) - 1u);
  const int nblk = E >> 2;
  int tie = 0;
  const int64_t row0 = (int64_t)c * ppc * 32;
  const int64_t row_end = min(total_rows, row0 + (int64_t)ppc * 32);
  int64_t row_j = row0 + lane;
  int layer = (int)(row_j / T);
  int64_t r = row_j - (int64_t)layer * T;
  int key_layer = -1;
  uint64_t k0 = 0, k1 = 0;
  const int l_first = (int)(row0 / T);
  const int span = row_end > row0 ? (int)((row_end - 1) / T) - l_first + 1 : 0;
  const bool local = span * E <= FS_MAX_EXPERTS;
  if (local) {
    for (int i = lane; i < span * E; i += 32) tally[i] = 0;
    __syncwarp();
  }
  for (int64_t pass0 = row0; pass0 < row_end; pass0 += 32) {
    const bool active = row_j < row_end;
    uint32_t top[KC];
#pragma unroll
    for (int j = 0; j < KC; j++) top[j] = 0xFFFFFFFFu;
    if (active) {
      if (layer != key_layer) {
        k0 = __ldcg(&job->keys[layer][0]);
        k1 = __ldcg(&job->keys[layer][1]);
        key_layer = layer;
      }
      const uint64_t b0 = (uint64_t)r * (uint64_t)nblk + 1;  // numpy pre-increments
#pragma unroll 1
      for (int q = 0; q < nblk; q++) {
#if FS_LONG_ROW_UNROLL
        const U4 blk = philox4x64_10_unrolled(b0 + q, k0, k1);  // long rows: see pass_fast
#else
        const U4 blk = philox4x64_10(b0 + q, k0, k1);
#endif
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint32_t x = ((uint32_t)(blk.v[j] >> 32) & keep) | (uint32_t)(4 * q + j);
#pragma unroll
          for (int t = 0; t < KC; t++) {
            const uint32_t lo = min(top[t], x);
            x = max(top[t], x);
            top[t] = lo;
          }
        }
      }
    }
    const bool unsure = active && (top[k] >> eb) == (top[k - 1] >> eb);
    int ids[k];
#pragma unroll
    for (int j = 0; j < k; j++) ids[j] = (int)(top[j] & ~keep);
    if (__any_sync(FS_FULL, unsure)) {
      // exact 64-bit redo of this pass (as process_chunk_k)
      uint64_t t64[KC];
#pragma unroll
      for (int j = 0; j < KC; j++) t64[j] = ~0ull;
      uint64_t thr = ~0ull;
      const uint64_t rb = (uint64_t)r * (uint64_t)E;
      if (active) topk_scan<KC>(t64, KC, thr, rb, rb + E, rb, k0, k1);
#pragma unroll
      for (int j = 0; j < k; j++) ids[j] = (int)(t64[j] & 0x7FF);
      if (active && (t64[k] >> 11) == (t64[k - 1] >> 11)) tie = 1;
    }
    if (local) {
      if (active) {
#pragma unroll
        for (int j = 0; j < k; j++) atomicAdd(&tally[(layer - l_first) * E + ids[j]], 1);
      }
    } else {
#pragma unroll
      for (int j = 0; j < k; j++) {
        const int key = active ? layer * E + ids[j] : -1;
        const unsigned grp = __match_any_sync(FS_FULL, key);
        if (key >= 0 && lane == __ffs(grp) - 1) atomicAdd(&counts[key], __popc(grp));
      }
    }
    r += 32;
    row_j += 32;
    while (r >= T) { r -= T; layer++; }
  }
  if (local) {
    __syncwarp();
    for (int i = lane; i < span * E; i += 32) {
      const int v = tally[i];
      if (v) atomicAdd(&counts[l_first * E + i], v);
    }
    __syncwarp();
  }
  if (__any_sync(FS_FULL, tie) && lane == 0) atomicExch(&job->tie, FS_ERR_ROUTING_TIE);
}

#if FS_LEARNED
// dirichlet_skew: chunk c is the whole router call of layer c (its exponentials are
// one stream with data-dependent word consumption); the claimant draws it with its
// own scratch and stores the layer's tally.
__device__ void dirichlet_chunk(const EngineParams& P, RouteJob* job, int32_t* counts, int c,
                                int lane, int* tally, int my_slot) {
  const int64_t T = __ldcg(&job->T);
  const int E = __ldcg(&job->E), k = __ldcg(&job->k);
  const double alpha = __ldcg(&job->alpha);
  const uint64_t k0 = __ldcg(&job->keys[c][0]), k1 = __ldcg(&job->keys[c][1]);
  const int st = route_dirichlet_warp(lane, T, E, k, alpha, k0, k1,
                                      P.dir_scratch + (int64_t)my_slot * kDirScratch, tally);
  __syncwarp();
  for (int e = lane; e < E; e += 32) counts[(int64_t)c * E + e] = tally[e];
  if (st != FS_OK && lane == 0) atomicExch(&job->tie, st);
}
#endif

// publish: completion is a release by lane 0 after __syncwarp (orders every
// lane's tally atomics before it); private jobs (run by their owner alone)
// skip it
__device__ void process_chunk(const EngineParams& P, RouteJob* job, int32_t* counts, int c,
                              int lane, int* tally, bool publish, int my_slot) {
  const int k = __ldcg(&job->k);
#if FS_LEARNED
  if (__ldcg(&job->kind) == 1) {
    dirichlet_chunk(P, job, counts, c, lane, tally, my_slot);
    __syncwarp();
    if (publish && lane == 0) red_add_release_i32(&job->done, 1);
    return;
  }
#endif
#if FS_ROWS_PATH
  const bool rows = __ldcg(&job->nseg) == 1 && (__ldcg(&job->E) & 3) == 0;
  if (rows && k == 2) process_rows<3>(P, job, counts, c, lane, tally);
  else if (rows && k == 1) process_rows<2>(P, job, counts, c, lane, tally);
  else if (rows && k == 3) process_rows<4>(P, job, counts, c, lane, tally);
#if FS_KCAP_MAX > 4
  else if (rows && k == 8) process_rows<9>(P, job, counts, c, lane, tally);  // DeepSeek-V3
#endif
  else
#endif
  if (k + 1 <= 4) process_chunk_k<4>(P, job, counts, c, lane, tally);
#if FS_KCAP_MAX > 4
  else if (k + 1 <= 9) process_chunk_k<9>(P, job, counts, c, lane, tally);
#endif
#if FS_KCAP_MAX > 9
  else process_chunk_k<FS_MAX_TOPK + 1>(P, job, counts, c, lane, tally);
#endif
  __syncwarp();
  if (publish && lane == 0) red_add_release_i32(&job->done, 1);
}

// Chunk loops. With FS_JOB_NOINLINE they are out-of-line calls: the caller's
// instance state is saved once per job around the call, and the routing loop
// inside gets the register file to itself (one copy of the code for owners and
// helpers alike).
#ifndef FS_JOB_NOINLINE  // round 1: 0 best (313 vs 340 ms); round 2, after the event-trace
#define FS_JOB_NOINLINE 1  // call sites: 1 best (227-234 vs 238-239 ms for the C5 sweep)
#endif
#if FS_JOB_NOINLINE
#define FS_JOB_FN __device__ __noinline__
#else
#define FS_JOB_FN __device__ __forceinline__
#endif
FS_JOB_FN void drain_job(const EngineParams& P, RouteJob* job, int32_t* counts, int lane,
                         int* tally, int my_slot) {
  for (int c; (c = claim_chunk(P, job, lane)) >= 0;)
    process_chunk(P, job, counts, c, lane, tally, true, my_slot);
}
FS_JOB_FN void run_chunks(const EngineParams& P, RouteJob* job, int32_t* counts, int n, int lane,
                          int* tally, int my_slot) {
  for (int c = 0; c < n; c++) process_chunk(P, job, counts, c, lane, tally, false, my_slot);
}

__device__ __forceinline__ int32_t* job_counts_of(const EngineParams& P, int slot) {
  return P.job_counts + (int64_t)slot * kJobLayers * P.job_max_e;
}

// Route layers [l0, l0+nl) of one batch; the tally of layer l0+j ends up at
// job_counts_of(slot)[j*E ...]. Returns FS_OK or a routing status (e.g.
// FS_ERR_ROUTING_TIE). kind 1: dirichlet_skew, one chunk per layer.
__device__ int run_route_job(const EngineParams& P, Inst& I, int prefix, int mb, int64_t step,
                             int l0, int nl, int64_t T, int* tally, int kind = 0) {
  const fs_instance_desc* d = I.d;
  RouteJob* job = &P.jobs[I.slot];
  int32_t* counts = job_counts_of(P, I.slot);
  const int E = d->num_experts, k = d->top_k;
  // router seeds + Philox keys, one layer per lane (base.py:63-65, routing.py:59-62)
  const int layer = l0 + I.lane;
  if (I.lane < nl) {
    const fs_seed_prefix* pf = &P.prefixes[prefix];
    int64_t ints[3];
    int n = 0;
    if (mb > 0) ints[n++] = mb;
    ints[n++] = step;
    ints[n++] = layer;
    int tl;
    const uint8_t* tail = prefix_tail(pf, tl);
    const uint32_t seed = sha256_tail_first_word(P.midstate + (int64_t)prefix * 8, pf->mid_blocks,
                                                 tail, tl, ints, n);
    uint64_t key[2];
    routing_key((uint64_t)seed, key);
    job->keys[I.lane][0] = key[0];
    job->keys[I.lane][1] = key[1];
  }
  for (int i = I.lane; i < nl * E; i += 32) counts[i] = 0;
  // geometry: split rows into segments while there are few of them; a chunk
  // carries >= ~16 Philox blocks per lane so claims and fences stay cheap
  const int64_t rows = (int64_t)nl * T;
  int nseg = 1;
  while (nseg < 32 && (nseg * 2) * 4 <= E && rows * nseg < FS_NSEG_ROWS) nseg *= 2;
  const int rpp = 32 / nseg;
  const int64_t passes = (rows + rpp - 1) / rpp;
  const int blocks_per_pass = ((E + nseg - 1) / nseg + 3) / 4 + 1;
  int ppc = (P.chunk_blocks > 0 ? P.chunk_blocks : kChunkBlocks) / blocks_per_pass;
  if (ppc < 1) ppc = 1;
  int64_t n_chunks = (passes + ppc - 1) / ppc;
  if (n_chunks > kMaxChunks) {
    ppc = (int)((passes + kMaxChunks - 1) / kMaxChunks);
    n_chunks = (passes + ppc - 1) / ppc;
  }
  if (kind == 1) n_chunks = nl;  // dirichlet_skew: a layer's stream is one chunk
  if (I.lane == 0) {
    job->T = T; job->E = E; job->k = k; job->nl = nl; job->nseg = nseg;
    job->passes_per_chunk = ppc; job->done = 0; job->tie = 0;
    job->kind = kind; job->alpha = d->routing_alpha;
  }
  __syncwarp();
  __threadfence();
  // small jobs are not worth publishing; a dirichlet layer always is
  const bool shared = kind == 1 ? n_chunks >= 2 : n_chunks >= 4;
  if (I.lane == 0) {
    const unsigned long long epoch =
        ((ld_volatile_u64(&job->ctr) >> (2 * kChunkBits)) + 1) & 0xFFFFFFull;
    const unsigned long long v = (epoch << (2 * kChunkBits)) |
                                 ((unsigned long long)n_chunks << kChunkBits);
    // a private job is published fully claimed, so helpers never see it
    atomicExch(&job->ctr, shared ? v : (v | (unsigned long long)n_chunks));
    if (shared) atomicAdd(P.open_jobs, 1);
  }
  __syncwarp();
  if (shared) {
    drain_job(P, job, counts, I.lane, tally, I.slot);
    while (ld_acquire_i32(&job->done) < n_chunks) __nanosleep(64);
  } else {
    run_chunks(P, job, counts, (int)n_chunks, I.lane, tally, I.slot);
  }
  __threadfence();
  __syncwarp();
  return ld_volatile_i32(&job->tie);
}

// uniform routing with real draws goes through the job board; the trace policy
// and the RNG-free shortcuts (T == 0, top_k == E) stay on the owning warp
__device__ __forceinline__ bool use_job_board(const fs_instance_desc* d, int policy, int64_t T) {
#if FS_LEARNED
  if (d->gg_forest != -1) return false;  // learned MoE layers cost per layer from sm->counts
#endif
  return policy == FS_ROUTE_UNIFORM && T > 0 && d->top_k < d->num_experts &&
         d->top_k >= 1 && d->top_k <= FS_MAX_TOPK && d->num_experts <= FS_MAX_EXPERTS;
}

// copy one layer's tally from the job (through L2) to the warp's counts
__device__ void load_job_layer(const EngineParams& P, const Inst& I, int j, WarpSmem* sm) {
  const int E = I.d->num_experts;
  const int32_t* counts = job_counts_of(P, I.slot) + (int64_t)j * E;
  __syncwarp();
  for (int e = I.lane; e < E; e += 32) sm->counts[e] = __ldcg(counts + e);
  __syncwarp();
}

// warps with no instance left help route other warps' jobs until every
// instance has finished; they sleep (exponential backoff) while no job is open
__device__ void help_route_jobs(const EngineParams& P, int lane, int my_slot, int* tally) {
  const int ns = P.n_slots;
  const int start = (int)(((unsigned)my_slot * 37u) % (unsigned)ns);
  unsigned backoff = 32;
  while (ld_volatile_i32(P.inst_done) < P.n_inst) {
    if (ld_volatile_i32(P.open_jobs) <= 0) {
      __nanosleep(backoff);
      backoff = backoff < 4096 ? backoff * 2 : 4096;
      continue;
    }
    backoff = 32;
    for (int base = 0; base < ns; base += 32) {
      int s = start + base + lane;
      if (s >= ns) s -= ns;
      bool avail = false;
      if (base + lane < ns) {
        const unsigned long long v = ld_volatile_u64(&P.jobs[s].ctr);
        avail = (v & kChunkMask) < ((v >> kChunkBits) & kChunkMask);
      }
      unsigned m = __ballot_sync(FS_FULL, avail);
      while (m) {
        const int pick = __ffs(m) - 1;
        m &= m - 1;
        const int sp = __shfl_sync(FS_FULL, s, pick);
        RouteJob* job = &P.jobs[sp];
        drain_job(P, job, job_counts_of(P, sp), lane, tally, my_slot);
      }
    }
  }
}

// ---- execute_batch (cluster.py:317-346) ---------------------------------------------------
struct BatchShape {
  int64_t n_tokens, sum_q, sum_kv;
  double attn_flops;
#if FS_LEARNED
  double learned_attn;  // learned-model attention us, NaN = analytic
#endif
};

#if FS_LEARNED
// CostModel.predict_attention with a learned model (model.py:313-321): the
// attention_v1 features of the batch members (prefill: q = kv = prompt;
// decode: q = 1, kv = prompt + emitted), then the forest. Out of line: only
// the learned simulation variant has these call sites.
__device__ __noinline__ double learned_attention_us(const EngineParams& P, Inst& I,
                                                    bool decode, const int32_t* members, int n,
                                                    int dstep, int tp, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  if (d->attn_forest < 0) {  // wrong schema for the attention slot (model.py:315-320)
    fail(I, FS_ERR_SCHEMA, 0);
    return 0.0;
  }
  int hq, hkv;
  heads_of(d, tp, hq, hkv);
  auto fq = [&](int64_t i) -> int64_t {
    return decode ? 1 : (int64_t)P.prompt[gi(I, members[i])];
  };
  auto fk = [&](int64_t i) -> int64_t {
    const int req = members[i];
    if (!decode) return P.prompt[gi(I, req)];
    return (int64_t)P.prompt[gi(I, req)] + P.output[gi(I, req)] + dstep - I.fin[req];
  };
  double x[17];
  attention_features_w(decode, n, fq, fk, hq, hkv, d->head_dim, I.lane, x);
  __syncwarp();
  if (I.lane < 17) {
#pragma unroll
    for (int j = 0; j < 17; j++)
      if (j == I.lane) sm->fx[j] = x[j];
  }
  __syncwarp();
  const double v = forest_predict_w(P.fv, d->attn_forest, sm->fx, sm->fvals, I.lane);
  __syncwarp();
  return v;
}

// Dense FFN with a learned grouped-GEMM model (cluster.py:286-296): one local
// expert holding all n tokens, so GroupedGemmFeatures.vector() is closed form
// (features.py:166-209: ratio 1, max/mean 1, cv 0, entropy 1, std 0).
__device__ __noinline__ double learned_dense_ffn_us(const EngineParams& P, Inst& I,
                                                    const fs_cost_ctx& c, int64_t n, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  if (d->gg_forest < 0) {  // check_schema("grouped_gemm_v1") (model.py:325)
    fail(I, FS_ERR_SCHEMA, 0);
    return 0.0;
  }
  if (n < 1) {
    fail(I, FS_ERR_EMPTY_BATCH, 2);
    return 0.0;
  }
  int64_t dff = d->d_ff / c.tp;
  if (dff < 1) dff = 1;
  __syncwarp();
  if (I.lane == 0) {
    double* x = sm->fx;
    x[0] = (double)n; x[1] = 1.0; x[2] = (double)d->d_model; x[3] = (double)dff;
    x[4] = 1.0; x[5] = 1.0; x[6] = 1.0; x[7] = 0.0; x[8] = 1.0;
    x[9] = (double)n; x[10] = (double)n; x[11] = 0.0;
  }
  __syncwarp();
  const double v = forest_predict_w(P.fv, d->gg_forest, sm->fx, sm->fvals, I.lane);
  __syncwarp();
  return v;
}
#define FFN_DENSE_US(c, n) \
  (d->gg_forest != -1 ? learned_dense_ffn_us(P, I, (c), (n), sm) : dense_ffn_us(d, (c), (n)))

// moe_layer_latency (moe.py:69-128) with a learned grouped-GEMM model: per EP
// rank with tokens, GroupedGemmFeatures(local, counts, d_model, d_ff_shard,
// top_k, "local").vector() (features.py:166-209) then the forest
// (model.py:323-326). Counts are the layer's tally in sm->counts. Sums of the
// integer loads are exact in any order; the std and the entropy sum follow
// numpy's pairwise order (the entropy terms p * log(p) of the active experts are
// compacted into the warp's global scratch first). Same outputs as
// moe_layer_warp; status uniform across lanes.
__device__ __noinline__ int learned_moe_layer_warp(const EngineParams& P, Inst& I, WarpSmem* sm,
                                                   int64_t T, int ep, int moe_tp,
                                                   const fs_cost_ctx& c, double* total,
                                                   double* ratio) {
  const fs_instance_desc* d = I.d;
  const int E = d->num_experts, lane = I.lane;
  if (ep < 1 || moe_tp < 1 || E % ep != 0 || d->expert_d_ff % moe_tp != 0)
    return FS_ERR_TOPOLOGY_MISMATCH;
  if (T < 1) return FS_ERR_EMPTY_BATCH;
  if (d->gg_forest < 0) return FS_ERR_SCHEMA;  // check_schema("grouped_gemm_v1")
  const double gate = linear_us(T, E, d->d_model, c, d->dtype_bytes);
  const int64_t routed_bytes = T * (int64_t)d->top_k * d->d_model * d->dtype_bytes;
  const double dispatch = collective_flt(false, i2d(routed_bytes) / (double)ep, ep,
                                         d->intra_latency_s, d->intra_bandwidth_bps) * 1e6;
  const int per = E / ep;
  const int64_t dffs = d->expert_d_ff / moe_tp;
  double* plogp = P.dir_scratch + (int64_t)I.slot * kDirScratch;
  double best = -1.0;
  PySum ps;
  ps.init();
  for (int r = 0; r < ep; r++) {
    const int* cr = sm->counts + r * per;
    int64_t loc = 0, mx = INT64_MIN, nact = 0;
    for (int e = lane; e < per; e += 32) {
      const int64_t v = cr[e];
      loc += v;
      mx = v > mx ? v : mx;
      nact += v > 0;
    }
    loc = warp_sum_i64(loc);
    mx = warp_max_i64(mx);
    nact = warp_sum_i64(nact);
    double v = 0.0;
    if (loc != 0) {
      if (dffs < 1 || d->top_k < 1) return FS_ERR_VALUE;
      const double sum = i2d(loc);
      const double mean = sum / (double)per;
      auto dev2 = [&](int64_t i) { const double dv = (double)cr[i] - mean; return dv * dv; };
      const double stdv = sqrt(np_pairwise_w(0, per, dev2, lane) / (double)per);
      const double amean = sum / (double)nact;  // active.mean(): exact integer sum
      double ent;
      if (per == 1) {
        ent = 1.0;
      } else {
        __syncwarp();
        int base = 0;  // active experts before this chunk (compaction keeps index order)
        for (int e0 = 0; e0 < per; e0 += 32) {
          const int e = e0 + lane;
          const bool act = e < per && cr[e] > 0;
          const unsigned m = __ballot_sync(FS_FULL, act);
          if (act) {
            const double pr = (double)cr[e] / sum;
            plogp[base + __popc(m & ((1u << lane) - 1u))] = pr * glm_log(pr);
          }
          base += __popc(m);
        }
        __syncwarp();
        auto term = [&](int64_t i) { return plogp[i]; };
        ent = -np_pairwise_w(0, nact, term, lane) / glm_log((double)per);
      }
      __syncwarp();
      if (lane == 0) {
        double* x = sm->fx;
        x[0] = sum; x[1] = (double)per; x[2] = (double)d->d_model; x[3] = (double)dffs;
        x[4] = (double)d->top_k; x[5] = (double)nact / (double)per;
        x[6] = (double)mx / amean; x[7] = mean > 0 ? stdv / mean : 0.0; x[8] = ent;
        x[9] = (double)mx; x[10] = mean; x[11] = stdv;
      }
      __syncwarp();
      v = forest_predict_w(P.fv, d->gg_forest, sm->fx, sm->fvals, lane);
      __syncwarp();
    }
    if (v > best) best = v;  // max(per_rank): first maximum
    ps.add(v);
  }
  double t = gate + dispatch;
  t = t + best;
  t = t + dispatch;
  *total = t;
  if (ratio) {
    const double sp = ps.result();
    *ratio = sp > 0 ? best / (sp / (double)ep) : 1.0;
  }
  return FS_OK;
}
#else
#define FFN_DENSE_US(c, n) dense_ffn_us(d, (c), (n))
#endif

// The per-batch operator costs that do not vary by layer, one per lane, then
// broadcast: lane 0 qkv_proj_us, 1 attention_us, 2 out_proj_us, 3 the dense ffn
// (grouped GEMM of one local expert), 4 tp_collective_us, 5 the (pp - 1) stage
// transfers. Each lane runs the same fp64 operations, in the same order, as the
// serial helpers above (qkv_us, attn_cost_us, ...), so every value is bit-identical;
// the warp pays for one roofline's two divisions instead of six.
struct BatchTerms {
  double qkv, att, out, ffn, coll, pp;
};
__device__ __forceinline__ BatchTerms batch_terms(const fs_instance_desc* d, const fs_cost_ctx& c,
                                                  const BatchShape& b, int lane) {
  int hq, hkv;
  heads_of(d, c.tp, hq, hkv);
  const int64_t n = b.n_tokens, dt = d->dtype_bytes, hd = d->head_dim, dm = d->d_model;
  const int j = lane < 6 ? lane : 5;
  // numerators / denominators of the lane's two divisions
  double num1, den1, num2, den2;
  if (j == 0 || j == 2 || j == 3) {  // linear_us / grouped_gemm_us rooflines
    int64_t a, bb, cc, e;
    int64_t nbytes;
    if (j == 3) {  // dense FFN: routed n, one active expert, d_ff / tp (>= 1)
      int64_t dff = d->d_ff / c.tp;
      if (dff < 1) dff = 1;
      const int64_t nm = d->ffn_matrices;
      a = nm; bb = n; cc = dm; e = dff;
      nbytes = 1 * nm * dm * dff * dt + n * nm * (dm + dff) * dt;
    } else {       // linear(m = n, nn, k)
      const int64_t nn = j == 0 ? (int64_t)(hq + 2 * hkv) * hd : dm;
      const int64_t k = j == 0 ? dm : (int64_t)hq * hd;
      a = n; bb = nn; cc = k; e = 1;
      nbytes = dt * (n * nn + nn * k + n * k);
    }
    double f = 2.0 * i2d(a);
    f = f * i2d(bb);
    f = f * i2d(cc);
    if (j == 3) f = f * i2d(e);
    num1 = f; den1 = c.peak_flops;
    num2 = i2d(nbytes); den2 = c.mem_bw;
  } else if (j == 1) {  // attention_us_from
    double kvb = 2.0 * i2d(b.sum_kv);
    kvb = kvb * (double)hkv;
    kvb = kvb * (double)hd;
    kvb = kvb * (double)dt;
    double qob = 2.0 * i2d(b.sum_q);
    qob = qob * (double)hq;
    qob = qob * (double)hd;
    qob = qob * (double)dt;
    num1 = b.attn_flops; den1 = c.peak_flops;
    num2 = kvb + qob; den2 = c.mem_bw;
  } else if (j == 4) {  // tpcoll_us: collective_int(all_reduce, n d_model dt, tp)
    num1 = i2d(n * dm * dt * (int64_t)(c.tp - 1)); den1 = (double)c.tp;
    num2 = 0.0; den2 = 1.0;
  } else {  // pp transfer: intra latency + n d_model dt / bandwidth
    num1 = 0.0; den1 = 1.0;
    num2 = i2d(n * dm * dt); den2 = d->intra_bandwidth_bps;
  }
  const double q1 = num1 / den1, q2 = num2 / den2;
  double v;
  if (j <= 3) {
    v = c.kernel_overhead_us + py_max(q1, q2) * 1e6;
  } else if (j == 4) {
    if (c.tp == 1) {
      v = 0.0;
    } else {
      const double wire = q1 / d->intra_bandwidth_bps;
      v = (2.0 * d->intra_latency_s + 2.0 * wire) * 1e6;
    }
  } else {
    const double tt = d->intra_latency_s + q2;
    v = (double)(c.pp - 1) * (tt * 1e6);
  }
  BatchTerms t;
  t.qkv = __shfl_sync(FS_FULL, v, 0);
  t.att = __shfl_sync(FS_FULL, v, 1);
  t.out = __shfl_sync(FS_FULL, v, 2);
  t.ffn = __shfl_sync(FS_FULL, v, 3);
  t.coll = __shfl_sync(FS_FULL, v, 4);
  t.pp = __shfl_sync(FS_FULL, v, 5);
  return t;
}

// attention_us_from(attn_flops, sum_q, sum_kv) alone (batch_terms' lane 1 term)
__device__ __forceinline__ double attention_term(const fs_instance_desc* d, const fs_cost_ctx& c,
                                                 const BatchShape& b) {
  int hq, hkv;
  heads_of(d, c.tp, hq, hkv);
  return attention_us_from(b.attn_flops, b.sum_q, b.sum_kv, hq, hkv, d->head_dim, c,
                           d->dtype_bytes);
}

#if FS_TERM_MEMO
// batch_terms with the n-only terms memoised per instance (the attention term
// depends on the batch's context sums and is always evaluated); bit-identical
// values, since a hit returns exactly what batch_terms computed for that n and
// context.
__device__ __forceinline__ BatchTerms batch_terms_memo(const fs_instance_desc* d,
                                                       const fs_cost_ctx& c, const BatchShape& b,
                                                       int lane, WarpSmem* sm) {
  TermMemo& m = sm->memo[b.n_tokens & (kMemoSlots - 1)];
  if (m.n == b.n_tokens && m.tp == c.tp && m.ppd == c.pp &&
      __double_as_longlong(m.peak) == __double_as_longlong(c.peak_flops) &&
      __double_as_longlong(m.bw) == __double_as_longlong(c.mem_bw) &&
      __double_as_longlong(m.ovh) == __double_as_longlong(c.kernel_overhead_us)) {
    BatchTerms t;
    t.qkv = m.qkv; t.out = m.out; t.ffn = m.ffn; t.coll = m.coll; t.pp = m.pp;
    t.att = attention_term(d, c, b);
    return t;
  }
  const BatchTerms t = batch_terms(d, c, b, lane);
  __syncwarp();
  if (lane == 0) {
    m.qkv = t.qkv; m.out = t.out; m.ffn = t.ffn; m.coll = t.coll; m.pp = t.pp;
    m.peak = c.peak_flops; m.bw = c.mem_bw; m.ovh = c.kernel_overhead_us;
    m.n = b.n_tokens; m.tp = c.tp; m.ppd = c.pp;
  }
  __syncwarp();
  return t;
}
#endif

// Duration in us (same on all lanes). moe_out (global) receives the per-layer
// moe_imbalance values round(expert / mean(per_rank), 6) when non-null.
__device__ double execute_batch(const EngineParams& P, Inst& I, int r, const fs_replica_desc& rd,
                                const BatchShape& b, int64_t step, WarpSmem* sm,
                                double* moe_out) {
  const fs_instance_desc* d = I.d;
  const fs_cost_ctx c = rd.cost;
  const int L = d->num_layers;
  const int64_t n = b.n_tokens;
#if FS_TERM_MEMO
  const BatchTerms bt = batch_terms_memo(d, c, b, I.lane, sm);
#else
  const BatchTerms bt = batch_terms(d, c, b, I.lane);
#endif
  const double qkv = bt.qkv, out = bt.out, coll = bt.coll;
#if FS_LEARNED
  const double att = isnan(b.learned_attn) ? bt.att : b.learned_attn;
#else
  const double att = bt.att;
#endif
  PySum ls;
  ls.init();
  if (FS_DENSE_ONLY || !d->has_moe) {
#if FS_LEARNED
    const double ffn = d->gg_forest != -1 ? learned_dense_ffn_us(P, I, c, n, sm) : bt.ffn;
#else
    const double ffn = bt.ffn;
#endif
    double tot = qkv + att;
    tot = tot + out;
    tot = tot + coll;
    tot = tot + ffn;
    tot = tot + coll;
    // sum(layer.total_us for L identical layers) (cluster.py:345): CPython's
    // Neumaier sum of L copies of tot is exactly fl(L * tot) -- every step's error
    // is caught exactly in the compensation, a multiple of ulp(tot) below 2^53 ulp
    // for L < 2^26 -- so one rounded product replaces the L-step chain
    // (tests/test_known_answers.py pins it against Python's sum()).
    return __dmul_rn((double)L, tot) + bt.pp;
  } else {
    const bool board = use_job_board(I.d, d->routing_policy, n);
#if FS_LEARNED
    // dirichlet_skew: the layers' router calls are independent streams, one chunk
    // each, so idle warps take whole layers (the analytic costs then read the tally)
    const bool dboard = d->routing_policy == FS_ROUTE_DIRICHLET && d->gg_forest == -1 && n > 0 &&
                        d->top_k < d->num_experts && d->top_k >= 1 &&
                        d->num_experts <= FS_MAX_EXPERTS && d->routing_alpha > 0;
#else
    const bool dboard = false;
#endif
    const bool log_routes = P.log_enabled && P.log.routes;
    for (int l0 = 0; l0 < L; l0 += kLayerChunk) {
      const int lend = min(L, l0 + kLayerChunk);
      double lane_ffn = 0.0, lane_ratio = 1.0;
      if (board || dboard) {
        int st = run_route_job(P, I, rd.prefix, 0, step, l0, lend - l0, n, sm->counts,
                               dboard ? 1 : 0);
        if (st == FS_OK)
          st = moe_layers_lanes(I.lane, job_counts_of(P, I.slot), lend - l0, n, d->num_experts,
                                d->top_k, d->d_model, d->expert_d_ff, d->ffn_matrices,
                                d->dtype_bytes, c.ep, c.moe_tp, d->intra_latency_s,
                                d->intra_bandwidth_bps, c, &lane_ffn,
                                moe_out ? &lane_ratio : nullptr);
        if (st != FS_OK) { fail(I, st, l0); return 0.0; }
      } else {
        derive_layer_keys(P, I, rd.prefix, 0, step, l0, L, sm);
      }
      for (int l = l0; l < lend; l++) {
        double ffn, ratio = 1.0;
        if (board || dboard) {
          ffn = __shfl_sync(FS_FULL, lane_ffn, l - l0);
          ratio = __shfl_sync(FS_FULL, lane_ratio, l - l0);
          I.routing_calls++;
          I.routing_draws += draws_of(d, d->routing_policy, n);
          if (log_routes) {
            load_job_layer(P, I, l - l0, sm);
            log_route(P, I, r, 0, step, l, n, sm);
          }
        } else {
          int st = route_layer(P, I, d->routing_policy, n, sm->keys[l - l0][0], sm->keys[l - l0][1], sm);
          if (st != FS_OK) { fail(I, st, l); return 0.0; }
          I.routing_calls++;
          I.routing_draws += draws_of(d, d->routing_policy, n);
          log_route(P, I, r, 0, step, l, n, sm);
#if FS_LEARNED
          if (d->gg_forest != -1)
            st = learned_moe_layer_warp(P, I, sm, n, c.ep, c.moe_tp, c, &ffn,
                                        moe_out ? &ratio : nullptr);
          else
#endif
          st = moe_layer_warp(I.lane, sm->counts, n, d->num_experts, d->top_k, d->d_model,
                              d->expert_d_ff, d->ffn_matrices, d->dtype_bytes, c.ep, c.moe_tp,
                              d->intra_latency_s, d->intra_bandwidth_bps, c, &ffn,
                              moe_out ? &ratio : nullptr);
          if (st != FS_OK) { fail(I, st, l); return 0.0; }
        }
        __syncwarp();
        if (moe_out && I.lane == 0) moe_out[l] = py_round6(ratio);
        double tot = qkv + att;
        tot = tot + out;
        tot = tot + coll;
        tot = tot + ffn;
        tot = tot + coll;
        ls.add(tot);
      }
    }
  }
  return ls.result() + bt.pp;
}

// ---- optional event trace (fs_event_rec at index seq; one lane writes) ------------------
// Event traces (run_one / make_simulation().run()) are recorded by the extended
// variant only (fs_launch_async runs a traced batch there): in the sweep kernels the
// trace call sites compile away instead of costing instruction fetch.
__device__ __forceinline__ bool tracing(const EngineParams& P) {
#if FS_LEARNED
  return P.log_enabled && P.log.events != nullptr;
#else
  return false;
#endif
}
__device__ void trace_put(const EngineParams& P, const Inst& I, int64_t seq, int64_t t, int kind,
                          int replica, int32_t a, int32_t b, int32_t c, int64_t x) {
  if (seq >= P.log.event_cap) { P.log.truncated[I.idx] = 1; return; }
  fs_event_rec r;
  r.t = t; r.seq = seq; r.x = x; r.a = a; r.b = b; r.c = c;
  r.replica = (int16_t)replica; r.kind = (uint8_t)kind; r.pad = 0;
  P.log.events[P.log.event_base[I.idx] + seq] = r;
}

// ---- optional batch log -------------------------------------------------------------------
// A batch is recorded when it starts (members, duration, pool snapshot, the seq of
// its BATCH_COMPLETE); its moe-ratio slot is reserved then too. Records are in
// start order; the host sorts by (t_complete, seq) for completion order.
// log_moe_reserve returns offset + 1 (0 = not logged).
__device__ int32_t log_moe_reserve(const EngineParams& P, Inst& I) {
  if (!P.log_enabled || !P.log.batches || !I.d->has_moe) return 0;
  if (I.log_eoff + I.d->num_layers > P.log.moe_cap) return 0;
  const int32_t off = I.log_eoff;
  I.log_eoff += I.d->num_layers;
  return off + 1;
}
__device__ int32_t log_batch(const EngineParams& P, Inst& I, int r, int phase, int64_t dur,
                             const int32_t* members, int nm, int32_t moe_off1, int64_t pool_used,
                             int64_t af_step) {
  if (!P.log_enabled || !P.log.batches) return -1;
  const int n_moe = moe_off1 ? I.d->num_layers : 0;
  const bool need_moe = I.d->has_moe && phase != PH_AF;
  const int32_t c = I.log_batches;
  if (c < P.log.batch_cap && I.log_moff + nm <= P.log.member_cap && (!need_moe || moe_off1)) {
    if (I.lane == 0) {
      fs_batch_rec rec;
      rec.replica = r; rec.phase = phase; rec.t_complete = I.now + dur; rec.duration_ns = dur;
      rec.n_members = nm; rec.member_offset = I.log_moff;
      rec.moe_offset = n_moe ? moe_off1 - 1 : -1;
      rec.n_moe = n_moe;
      rec.seq = I.seq;  // the BATCH_COMPLETE about to be scheduled
      rec.pool_used = pool_used;
      rec.af_step = af_step;
      P.log.batches[P.log.batch_base[I.idx] + c] = rec;
    }
    const int64_t mb = P.log.member_base[I.idx] + I.log_moff;
    for (int i = I.lane; i < nm; i += 32) P.log.members[mb + i] = members[i];
    I.log_moff += nm;
    I.log_batches = c + 1;
    __syncwarp();
    return c;
  }
  if (I.lane == 0) P.log.truncated[I.idx] = 1;
  __syncwarp();
  return -1;
}

// BATCH_COMPLETE at now + dur: batch record + trace record, then the heap event
__device__ void schedule_batch_complete(const EngineParams& P, Inst& I, int r, int phase,
                                        int64_t dur, const int32_t* members, int nm,
                                        int32_t moe_off1, int64_t pool_used, int64_t af_step) {
  const int32_t bi = log_batch(P, I, r, phase, dur, members, nm, moe_off1, pool_used, af_step);
  if (tracing(P) && I.lane == 0)
    trace_put(P, I, I.seq, I.now + dur, FS_EV_BATCH_COMPLETE, r, bi, 0, 0, 0);
}

// ---- list helpers ---------------------------------------------------------------------------
// remove the first m entries (stable shift)
__device__ void list_drop_front(int32_t* a, int len, int m, int lane) {
  if (m == 0) return;
  for (int base = 0; base < len - m; base += 32) {
    const int i = base + lane;
    const int v = (i < len - m) ? a[i + m] : 0;
    __syncwarp();
    if (i < len - m) a[i] = v;
    __syncwarp();
  }
}
// insert v at position pos (shifting the tail right)
__device__ void list_insert(int32_t* a, int len, int pos, int v, int lane) {
  for (int top = len; top > pos; top -= 32) {
    const int i = top - 1 - lane;  // source index, descending
    const bool act = i >= pos;
    const int x = act ? a[i] : 0;
    __syncwarp();
    if (act) a[i + 1] = x;
    __syncwarp();
  }
  if (lane == 0) a[pos] = v;
  __syncwarp();
}

// priority key (cluster.py:153-157): (prompt, arrival, id) or (arrival, id)
__device__ __forceinline__ bool prio_less(const EngineParams& P, const Inst& I, int a, int b) {
  if (I.d->priority_key == FS_PRIO_PROMPT) {
    const int pa = P.prompt[gi(I, a)], pb = P.prompt[gi(I, b)];
    if (pa != pb) return pa < pb;
  }
  const int64_t ta = P.arrival[gi(I, a)], tb = P.arrival[gi(I, b)];
  if (ta != tb) return ta < tb;
  return P.id_rank[gi(I, a)] < P.id_rank[gi(I, b)];
}

// enqueue a waiting request; priority admission keeps the queue in key order
__device__ void enqueue(const EngineParams& P, Inst& I, int r, RepState& s, int req) {
  int32_t* q = qlist(I, r);
  if (I.d->admission == FS_ADMIT_PRIORITY) {
    int pos = 0;
    for (int base = 0; base < s.qlen; base += 32) {
      const int i = base + I.lane;
      const bool less = i < s.qlen && prio_less(P, I, q[i], req);
      pos += __popc(__ballot_sync(FS_FULL, less));
    }
    list_insert(q, s.qlen, pos, req, I.lane);
  } else {
    __syncwarp();
    if (I.lane == 0) q[s.qlen] = req;
    __syncwarp();
  }
  s.qlen++;
}

// FIFO head of a queue (the queue in priority mode is key-ordered; the FIFO
// head is the earliest-arrived request, i.e. the smallest local index)
__device__ int queue_head(const Inst& I, int r, const RepState& s) {
  const int32_t* q = qlist(I, r);
  if (I.d->admission != FS_ADMIT_PRIORITY) return q[0];
  int64_t m = 0x7fffffff;
  for (int i = I.lane; i < s.qlen; i += 32) m = min(m, (int64_t)q[i]);
  return (int)warp_min_i64(m);
}

// ---- build_prefill_batch (cluster.py:145-183) ------------------------------------------------
struct Admit {
  int m;
  int64_t sum_p, sum_p2, max_p, charge;
};

// Admitted members (candidate order) go to the inflight list and leave the queue.
__device__ Admit admit_prefill(const EngineParams& P, Inst& I, int r, RepState& s, bool full,
                               int running_count, int64_t capacity) {
  const fs_instance_desc* d = I.d;
  int32_t* q = qlist(I, r);
  int32_t* il = ilist(I, r);
  const int64_t seats = (int64_t)d->max_num_seqs - running_count;
  const int64_t mbt = d->max_batch_tokens;
  const int64_t headroom = capacity - s.used;
  const unsigned lt = (1u << I.lane) - 1u;
  Admit A;
  A.m = 0; A.sum_p = 0; A.sum_p2 = 0; A.max_p = 0; A.charge = 0;
  int64_t tokens = 0;
  __syncwarp();
  if (d->admission != FS_ADMIT_FCFS_SKIP) {
    // strict order: the admitted set is the longest fitting prefix
    for (int base = 0; base < s.qlen; base += 32) {
      const int i = base + I.lane;
      const bool valid = i < s.qlen;
      const int req = valid ? q[i] : 0;
      const int64_t p = valid ? P.prompt[gi(I, req)] : 0;
      const int64_t fp = valid ? pool_rounded(d, full ? p + P.output[gi(I, req)] : p) : 0;
      const int64_t cp = warp_incl_scan_i64(p, I.lane);
      const int64_t cf = warp_incl_scan_i64(fp, I.lane);
      const bool ok = valid && (A.m + I.lane < seats) && (tokens + cp <= mbt) &&
                      (A.charge + cf <= headroom);
      const unsigned vm = __ballot_sync(FS_FULL, valid);
      const unsigned bad = vm & ~__ballot_sync(FS_FULL, ok);
      const int nadm = bad ? __ffs(bad) - 1 : __popc(vm);
      const bool adm = I.lane < nadm;
      if (adm) il[A.m + I.lane] = req;
      const int64_t ap = adm ? p : 0;
      A.sum_p += warp_sum_i64(ap);
      A.sum_p2 += warp_sum_i64(ap * ap);
      A.max_p = max(A.max_p, warp_max_i64(ap));
      A.charge += warp_sum_i64(adm ? fp : 0);
      tokens = A.sum_p;
      A.m += nadm;
      if (bad) break;
    }
    __syncwarp();
    list_drop_front(q, s.qlen, A.m, I.lane);
    s.qlen -= A.m;
  } else {
    // fcfs_skip: greedy in queue order; a request that does not fit is skipped
    // (totals only grow, so it can never fit later in the same scan)
    int w = 0;
    for (int base = 0; base < s.qlen; base += 32) {
      const int i = base + I.lane;
      const bool valid = i < s.qlen;
      const int req = valid ? q[i] : 0;
      const int64_t p = valid ? P.prompt[gi(I, req)] : 0;
      const int64_t fp = valid ? pool_rounded(d, full ? p + P.output[gi(I, req)] : p) : 0;
      unsigned admitted = 0;
      int last = -1;
      for (;;) {
        const bool fits = valid && I.lane > last && (A.m < seats) && (tokens + p <= mbt) &&
                          (A.charge + fp <= headroom);
        const unsigned fm = __ballot_sync(FS_FULL, fits);
        if (!fm) break;
        const int f = __ffs(fm) - 1;
        admitted |= 1u << f;
        const int64_t pv = __shfl_sync(FS_FULL, p, f);
        const int64_t fpv = __shfl_sync(FS_FULL, fp, f);
        if (I.lane == f) il[A.m] = req;
        A.m++;
        tokens += pv;
        A.charge += fpv;
        A.sum_p += pv;
        A.sum_p2 += pv * pv;
        A.max_p = max(A.max_p, pv);
        last = f;
      }
      const unsigned keep = __ballot_sync(FS_FULL, valid) & ~admitted;
      __syncwarp();
      if (keep & (1u << I.lane)) q[w + __popc(keep & lt)] = req;
      w += __popc(keep);
      __syncwarp();
    }
    s.qlen = w;
  }
  __syncwarp();
  return A;
}

// ---- batch launch helpers ----------------------------------------------------------------------
__device__ void launch_batch(const EngineParams& P, Inst& I, int r, RepState& s,
                             const fs_replica_desc& rd, const BatchShape& b, int phase,
                             WarpSmem* sm) {
  const int32_t moe_off1 = log_moe_reserve(P, I);
  double* moe_slot = moe_off1 ? P.log.moe_ratio + P.log.moe_base[I.idx] + (moe_off1 - 1) : nullptr;
  const double us = execute_batch(P, I, r, rd, b, s.steps, sm, moe_slot);
  if (I.status) return;
  const int64_t dur = py_round(us * 1000.0);
  s.busy = 1;
  s.steps++;
  s.inflight_phase = phase;
  s.inflight_dur = dur;
  s.inflight_moe = moe_off1;
  if (P.log_enabled)
    schedule_batch_complete(P, I, r, phase, dur, phase == PH_PREFILL ? ilist(I, r) : rlist(I, r),
                            phase == PH_PREFILL ? s.ilen : s.rlen, moe_off1, s.used, -1);
  heap_push(I, I.now + dur, K_BATCH_COMPLETE, r, dur);
}

__device__ void start_prefill(const EngineParams& P, Inst& I, int r, RepState& s,
                              const fs_replica_desc& rd, const Admit& A, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  BatchShape b;
  b.n_tokens = A.sum_p;
  b.sum_q = A.sum_p;
  b.sum_kv = A.sum_p;
  int hq, hkv;
  heads_of(d, rd.cost.tp, hq, hkv);
  const int64_t hd = (int64_t)hq * d->head_dim;
  // Each member contributes the exact integer 2*l*l*hd (c == l); while every
  // term and partial sum stays below 2^53 the sequential fp64 sum is exact in
  // any order, so the integer sum is bit-identical.
  const double lim = 9007199254740992.0;
  if (4.0 * (double)A.max_p * (double)A.max_p * (double)hd < lim &&
      2.0 * (double)hd * (double)A.sum_p2 < lim) {
    b.attn_flops = i2d(2 * hd * A.sum_p2);
  } else {
    double total = 0.0;
    if (I.lane == 0) {
      const int32_t* il = ilist(I, r);
      for (int i = 0; i < A.m; i++) {
        const int64_t p = P.prompt[gi(I, il[i])];
        total = total + attention_prefill_term(p, p, hd);
      }
    }
    b.attn_flops = __shfl_sync(FS_FULL, total, 0);
  }
#if FS_LEARNED
  b.learned_attn = d->attn_forest != -1
                       ? learned_attention_us(P, I, false, ilist(I, r), A.m, 0, rd.cost.tp, sm)
                       : __longlong_as_double(0x7ff8000000000000LL);
#endif
  s.ilen = A.m;
  launch_batch(P, I, r, s, rd, b, PH_PREFILL, sm);
}

__device__ void start_decode(const EngineParams& P, Inst& I, int r, RepState& s,
                             const fs_replica_desc& rd, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  BatchShape b;
  b.n_tokens = s.rlen;  // running <= max_num_seqs in every mode, so the batch is all of it
  b.sum_q = s.rlen;
  b.sum_kv = s.sum_ctx;
  int hq, hkv;
  heads_of(d, rd.cost.tp, hq, hkv);
  b.attn_flops = attention_decode_flops(s.sum_ctx, (int64_t)hq * d->head_dim);
#if FS_LEARNED
  b.learned_attn = d->attn_forest != -1
                       ? learned_attention_us(P, I, true, rlist(I, r), s.rlen, s.dstep, rd.cost.tp, sm)
                       : __longlong_as_double(0x7ff8000000000000LL);
#endif
  launch_batch(P, I, r, s, rd, b, PH_DECODE, sm);
}

__device__ void kick(const EngineParams& P, Inst& I, int r, RepState& s) {
  if (s.busy || s.start_pending) return;
  if (s.qlen == 0 && s.rlen == 0) return;
  s.start_pending = 1;
  if (tracing(P) && I.lane == 0) trace_put(P, I, I.seq, I.now, FS_EV_BATCH_START, r, 0, 0, 0, 0);
  heap_push(I, I.now, K_BATCH_START, r, 0);
}

// append requests (cooperatively: lane i holds req if has) to the running list
__device__ void running_append(const EngineParams& P, Inst& I, int r, RepState& s, bool has,
                               int req, int emitted) {
  const unsigned lt = (1u << I.lane) - 1u;
  const unsigned hm = __ballot_sync(FS_FULL, has);
  int32_t* rl = rlist(I, r);
  int64_t ctx = 0, fin = kNoFinish;
  if (has) {
    const int out = P.output[gi(I, req)];
    const int32_t f = s.dstep + (out - emitted);
    rl[s.rlen + __popc(hm & lt)] = req;
    I.fin[req] = f;
    ctx = (int64_t)P.prompt[gi(I, req)] + emitted;
    fin = f;
  }
  s.rlen += __popc(hm);
  s.sum_ctx += warp_sum_i64(ctx);
  s.min_finish = (int32_t)min((int64_t)s.min_finish, warp_min_i64(fin));
  __syncwarp();
}

// prefill completion (colocated.py:70-91, pd.py:98-112, af.py:514-535).
// to_running: co-located / AF; otherwise PD (unfinished go to the transfer FIFO).
__device__ void prefill_complete(const EngineParams& P, Inst& I, int r, RepState& s,
                                 bool to_running) {
  const fs_instance_desc* d = I.d;
  const int32_t* il = ilist(I, r);
  const int nm = s.ilen;
  const unsigned lt = (1u << I.lane) - 1u;
  I.events += nm + 1;  // PREFILL_COMPLETE per member + one TOKEN_EMITTED
  // sequence numbers (colocated.py:75-91): PREFILL_COMPLETE per member, TOKEN_EMITTED,
  // then REQUEST_COMPLETE + MEMORY_AVAILABLE per finished member, in member order
  const int64_t seq0 = I.seq;
  const bool tr = tracing(P);
  int nf = 0;
  if (tr && I.lane == 0)
    trace_put(P, I, seq0 + nm, I.now, FS_EV_TOKEN_EMITTED, r, 0, 0, 0, 0);
  for (int base = 0; base < nm; base += 32) {
    const int i = base + I.lane;
    const bool valid = i < nm;
    const int req = valid ? il[i] : 0;
    const int out = valid ? P.output[gi(I, req)] : 0;
    if (valid) P.first_ns[gi(I, req)] = I.now;
    const bool fin = valid && out == 1;
    const unsigned fm = __ballot_sync(FS_FULL, fin);
    // completions and appends interleave in member order; they touch disjoint state
    const int64_t fp = fin ? (to_running ? (int64_t)P.prompt[gi(I, req)] + out
                                         : (int64_t)P.prompt[gi(I, req)]) : 0;
    const int64_t freed = fin ? pool_rounded(d, fp) : 0;
    if (tr) {
      const int64_t used_after = s.used - warp_incl_scan_i64(freed, I.lane);
      if (valid) trace_put(P, I, seq0 + i, I.now, FS_EV_PREFILL_COMPLETE, r, req, 0, 0, 0);
      if (fin) {
        const int64_t sq = seq0 + nm + 1 + 2 * (nf + __popc(fm & lt));
        trace_put(P, I, sq, I.now, FS_EV_REQUEST_COMPLETE, r, req, 0, 0, 0);
        trace_put(P, I, sq + 1, I.now, FS_EV_MEMORY_AVAILABLE, r, req, (int32_t)freed, 0,
                  P.reps[I.rb + r].kv_pool_tokens - used_after);
      }
    }
    s.used -= warp_sum_i64(freed);
    if (fin) {
      P.done_ns[gi(I, req)] = I.now;
      P.done_rank[gi(I, req)] = I.n_done + __popc(fm & lt);
    }
    I.n_done += __popc(fm);
    nf += __popc(fm);
    I.events += 2 * __popc(fm);
    const bool keep = valid && !fin;
    if (to_running) {
      running_append(P, I, r, s, keep, req, 1);
    } else {
      const unsigned km = __ballot_sync(FS_FULL, keep);
      if (keep) P.xfer[I.ro + (I.xt + __popc(km & lt)) % I.N] = req;
      I.xt += __popc(km);
    }
    __syncwarp();
  }
  I.seq = seq0 + nm + 1 + 2 * nf;
}

// decode / AF completion: every member emitted one token; finished requests leave
// the running list in order (colocated.py:92-107, pd.py:113-127, af.py:536-551).
// Returns the number finished. pool charge per finished request = rounded(prompt+output).
__device__ int decode_complete(const EngineParams& P, Inst& I, int r, RepState& s) {
  const fs_instance_desc* d = I.d;
  I.events += 1;  // TOKEN_EMITTED
  // sequence numbers (colocated.py:92-107): TOKEN_EMITTED, then REQUEST_COMPLETE +
  // MEMORY_AVAILABLE per finished member in running order
  const int64_t seq0 = I.seq;
  const bool tr = tracing(P);
  if (tr && I.lane == 0) trace_put(P, I, seq0, I.now, FS_EV_TOKEN_EMITTED, r, 0, 0, 0, 0);
  I.seq = seq0 + 1;
  s.dstep++;
  s.sum_ctx += s.rlen;
  if (s.min_finish != s.dstep) return 0;
  int32_t* rl = rlist(I, r);
  const unsigned lt = (1u << I.lane) - 1u;
  int w = 0, nf = 0;
  int64_t freed_ctx = 0, freed_pool = 0, new_min = kNoFinish;
  int64_t freed_run = 0;  // pool tokens released by earlier chunks (tracing only)
  for (int base = 0; base < s.rlen; base += 32) {
    const int i = base + I.lane;
    const bool valid = i < s.rlen;
    const int req = valid ? rl[i] : 0;
    const int32_t f = valid ? I.fin[req] : kNoFinish;
    const bool fin = valid && f == s.dstep;
    const unsigned fm = __ballot_sync(FS_FULL, fin);
    const unsigned km = __ballot_sync(FS_FULL, valid && !fin);
    if (tr) {
      const int64_t fr = fin ? pool_rounded(d, (int64_t)P.prompt[gi(I, req)] + P.output[gi(I, req)]) : 0;
      const int64_t incl = warp_incl_scan_i64(fr, I.lane);
      if (fin) {
        const int64_t sq = seq0 + 1 + 2 * (nf + __popc(fm & lt));
        trace_put(P, I, sq, I.now, FS_EV_REQUEST_COMPLETE, r, req, 0, 0, 0);
        trace_put(P, I, sq + 1, I.now, FS_EV_MEMORY_AVAILABLE, r, req, (int32_t)fr, 0,
                  P.reps[I.rb + r].kv_pool_tokens - (s.used - freed_run - incl));
      }
      freed_run += warp_sum_i64(fr);
    }
    if (fin) {
      const int64_t fp = (int64_t)P.prompt[gi(I, req)] + P.output[gi(I, req)];
      freed_ctx += fp;
      freed_pool += pool_rounded(d, fp);
      P.done_ns[gi(I, req)] = I.now;
      P.done_rank[gi(I, req)] = I.n_done + __popc(fm & lt);
    } else if (valid) {
      new_min = min(new_min, (int64_t)f);
    }
    I.n_done += __popc(fm);
    nf += __popc(fm);
    __syncwarp();
    if (valid && !fin) rl[w + __popc(km & lt)] = req;
    w += __popc(km);
    __syncwarp();
  }
  s.rlen = w;
  s.sum_ctx -= warp_sum_i64(freed_ctx);
  s.used -= warp_sum_i64(freed_pool);
  s.min_finish = (int32_t)warp_min_i64(new_min);
  I.events += 2 * nf;
  I.seq = seq0 + 1 + 2 * nf;
  return nf;
}

// ---- co-located (colocated.py) ------------------------------------------------------------------
__device__ void co_arrival(const EngineParams& P, Inst& I, int req) {
  const int r = I.rr % I.R;
  I.rr++;
  RepState s = load_rep(P, I, r);
  enqueue(P, I, r, s, req);
  kick(P, I, r, s);
  store_rep(P, I, r, s);
}

__device__ void af_start_step(const EngineParams& P, Inst& I, RepState& s, const fs_replica_desc& rd,
                              WarpSmem* sm);

__device__ void co_batch_start(const EngineParams& P, Inst& I, int r, WarpSmem* sm) {
  RepState s = load_rep(P, I, r);
  s.start_pending = 0;
  if (!s.busy) {
    const fs_replica_desc rd = P.reps[I.rb + r];
    const Admit A = admit_prefill(P, I, r, s, true, s.rlen, rd.kv_pool_tokens);
    if (A.m) {
      s.used += A.charge;
      start_prefill(P, I, r, s, rd, A, sm);
    } else if (s.rlen) {
      if (FS_HAS_AF && I.mode == FS_MODE_AF) af_start_step(P, I, s, rd, sm);
      else start_decode(P, I, r, s, rd, sm);
    } else if (s.qlen) {
      fail(I, FS_ERR_REQUEST_CANNOT_FIT, queue_head(I, r, s));
    }
  }
  store_rep(P, I, r, s);
}

__device__ void co_batch_complete(const EngineParams& P, Inst& I, int r, int64_t dur) {
  RepState s = load_rep(P, I, r);
  s.busy = 0;
  s.busy_ns += dur;
  if (s.inflight_phase == PH_PREFILL) {
    I.prefill_batches++;
    prefill_complete(P, I, r, s, true);
  } else {
    if (s.inflight_phase == PH_AF) I.af_steps++; else I.decode_batches++;
    decode_complete(P, I, r, s);
  }
  kick(P, I, r, s);
  store_rep(P, I, r, s);
}

// ---- PD (pd.py) ---------------------------------------------------------------------------------
// argmin over replicas of `role` by (key value, key_rank); value from rstate
__device__ int pd_pick(const EngineParams& P, const Inst& I, int role, bool by_used) {
  int64_t best_v = INT64_MAX;
  int best_rank = 0x7fffffff, best_r = -1;
  for (int r = I.lane; r < I.R; r += 32) {
    const fs_replica_desc& rd = P.reps[I.rb + r];
    if (rd.role != role) continue;
    const RepState& st = I.rs[r];
    const int64_t v = by_used ? st.used : st.outstanding;
    if (v < best_v || (v == best_v && rd.key_rank < best_rank)) {
      best_v = v; best_rank = rd.key_rank; best_r = r;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(FS_FULL, best_v, o);
    const int ok = __shfl_xor_sync(FS_FULL, best_rank, o);
    const int orr = __shfl_xor_sync(FS_FULL, best_r, o);
    if (ov < best_v || (ov == best_v && ok < best_rank)) { best_v = ov; best_rank = ok; best_r = orr; }
  }
  return best_r;
}

__device__ void pd_arrival(const EngineParams& P, Inst& I, int req) {
  __syncwarp();
  const int r = pd_pick(P, I, FS_ROLE_PREFILL, false);
  RepState s = load_rep(P, I, r);
  if (I.lane == 0) P.home[gi(I, req)] = r;
  enqueue(P, I, r, s, req);
  s.outstanding += P.prompt[gi(I, req)];
  kick(P, I, r, s);
  store_rep(P, I, r, s);
}

// _pump_transfers (pd.py:141-192): strict FIFO, decode replica by (used, key)
__device__ void pd_pump(const EngineParams& P, Inst& I) {
  const fs_instance_desc* d = I.d;
  while (I.xt > I.xh && I.status == FS_OK) {
    const int req = P.xfer[I.ro + I.xh % I.N];
    const int r = pd_pick(P, I, FS_ROLE_DECODE, true);
    RepState s = load_rep(P, I, r);
    const int64_t cap = P.reps[I.rb + r].kv_pool_tokens;
    const int64_t prompt = P.prompt[gi(I, req)];
    const int64_t fp = pool_rounded(d, prompt + P.output[gi(I, req)]);
    if (fp > cap) { fail(I, FS_ERR_REQUEST_CANNOT_FIT, req); return; }
    if (fp > cap - s.used) return;  // Backpressure: wait for decode memory
    s.used += fp;
    store_rep(P, I, r, s);
    I.xh++;
    I.events += 1;  // KV_CACHE_TRANSFER_START
    const int64_t nbytes = d->kv_bytes_per_token * prompt;
    const double sec = transfer_s(nbytes, d->inter_latency_s, d->inter_bandwidth_bps);
    const int64_t t_done = I.now + py_round(sec * 1e9);
    if (tracing(P) && I.lane == 0) {
      const int32_t src = P.home[gi(I, req)];
      trace_put(P, I, I.seq, I.now, FS_EV_KV_TRANSFER_START, r, req, (int32_t)fp, src, s.used);
      trace_put(P, I, I.seq + 1, t_done, FS_EV_KV_TRANSFER_DONE, r, req, 0, src, 0);
    }
    I.seq++;
    heap_push(I, t_done, K_KV_DONE, r, req);
  }
}

__device__ void pd_batch_start(const EngineParams& P, Inst& I, int r, WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  RepState s = load_rep(P, I, r);
  s.start_pending = 0;
  if (!s.busy) {
    const fs_replica_desc rd = P.reps[I.rb + r];
    if (rd.role == FS_ROLE_PREFILL) {
      const Admit A = admit_prefill(P, I, r, s, false, 0, rd.kv_pool_tokens);
      if (A.m == 0) {
        if (s.qlen && s.used == 0) fail(I, FS_ERR_REQUEST_CANNOT_FIT, queue_head(I, r, s));
      } else {
        s.used += A.charge;
        s.outstanding -= A.sum_p;
        start_prefill(P, I, r, s, rd, A, sm);
      }
    } else {
      // queue -> running up to max_num_seqs (pd.py:89-96)
      const int take = min(s.qlen, max(0, d->max_num_seqs - s.rlen));
      int32_t* q = qlist(I, r);
      for (int base = 0; base < take; base += 32) {
        const int i = base + I.lane;
        const bool has = i < take;
        running_append(P, I, r, s, has, has ? q[i] : 0, 1);
      }
      list_drop_front(q, s.qlen, take, I.lane);
      s.qlen -= take;
      if (s.rlen) start_decode(P, I, r, s, rd, sm);
    }
  }
  store_rep(P, I, r, s);
}

__device__ void pd_batch_complete(const EngineParams& P, Inst& I, int r, int64_t dur) {
  RepState s = load_rep(P, I, r);
  s.busy = 0;
  s.busy_ns += dur;
  if (s.inflight_phase == PH_PREFILL) {
    I.prefill_batches++;
    prefill_complete(P, I, r, s, false);
    store_rep(P, I, r, s);
    pd_pump(P, I);
  } else {
    I.decode_batches++;
    const int nf = decode_complete(P, I, r, s);
    store_rep(P, I, r, s);
    if (nf) pd_pump(P, I);
  }
  s = load_rep(P, I, r);
  kick(P, I, r, s);
  store_rep(P, I, r, s);
}

__device__ void pd_transfer_done(const EngineParams& P, Inst& I, int dr, int req) {
  const fs_instance_desc* d = I.d;
  I.events += 1;  // MEMORY_AVAILABLE
  __syncwarp();
  const int ph = P.home[gi(I, req)];
  RepState sp = load_rep(P, I, ph);
  const int64_t freed = pool_rounded(d, P.prompt[gi(I, req)]);
  sp.used -= freed;
  if (tracing(P) && I.lane == 0)
    trace_put(P, I, I.seq, I.now, FS_EV_MEMORY_AVAILABLE, ph, req, (int32_t)freed, 0,
              P.reps[I.rb + ph].kv_pool_tokens - sp.used);
  I.seq++;
  store_rep(P, I, ph, sp);
  RepState sd = load_rep(P, I, dr);
  __syncwarp();
  if (I.lane == 0) qlist(I, dr)[sd.qlen] = req;
  sd.qlen++;
  store_rep(P, I, dr, sd);
  sp = load_rep(P, I, ph);
  kick(P, I, ph, sp);
  store_rep(P, I, ph, sp);
  sd = load_rep(P, I, dr);
  kick(P, I, dr, sd);
  store_rep(P, I, dr, sd);
}

// ---- AF step (af.py:244-319, 468-507) ------------------------------------------------------------
__device__ void af_start_step(const EngineParams& P, Inst& I, RepState& s, const fs_replica_desc& rd,
                              WarpSmem* sm) {
  const fs_instance_desc* d = I.d;
  const int L = d->num_layers;
  const int B = s.rlen;
  const int m = min(d->af_micro_batches, B);
  if (m > FS_MAX_MICRO_BATCHES) { fail(I, FS_ERR_CAPACITY, m); return; }
  const int64_t step = I.af_counter++;
  const int32_t* rl = rlist(I, 0);
  const fs_cost_ctx ca = d->af_attn, cf = d->af_ffn;
  int hq, hkv;
  heads_of(d, ca.tp, hq, hkv);
  const int64_t hd = (int64_t)hq * d->head_dim;
  const int base = B / m, rem = B % m;
  int64_t* ffn = P.af_ffn + P.af_base[I.idx];
  int off = 0;
  for (int i = 0; i < m; i++) {
    const int sz = base + (i < rem ? 1 : 0);
    // attention: largest attn_dp group = first ceil(sz / min(dp, sz)) members
    const int g = min(d->af_attn_dp, sz);
    const int w = sz / g + (sz % g ? 1 : 0);
    int64_t ctx = 0;
    for (int j = I.lane; j < w; j += 32) {
      const int req = rl[off + j];
      ctx += (int64_t)P.prompt[gi(I, req)] + P.output[gi(I, req)] + s.dstep - I.fin[req];
    }
    ctx = warp_sum_i64(ctx);
#if FS_LEARNED
    const double att =
        d->attn_forest != -1
            ? learned_attention_us(P, I, true, rl + off, w, s.dstep, ca.tp, sm)
            : attn_cost_us(d, ca, attention_decode_flops(ctx, hd), w, ctx);
#else
    const double att = attn_cost_us(d, ca, attention_decode_flops(ctx, hd), w, ctx);
#endif
    double us = qkv_us(d, ca, w) + att;
    us = us + out_us(d, ca, w);
    us = us + tpcoll_us(d, ca, w);
    const int64_t attn_ns = py_round(us * 1000.0);
    const int64_t nb = (int64_t)sz * d->d_model * d->dtype_bytes;
    const double sec = d->inter_latency_s + i2d(nb) / d->inter_bandwidth_bps;
    const int64_t xfer_ns = py_round(sec * 1e9);
    if (I.lane == 0) {
      sm->af_attn[i] = attn_ns;
      sm->af_xfer[i] = xfer_ns;
      sm->af_size[i] = sz;
    }
    // FFN durations per layer (af.py:289-301): MoE routes with the uniform policy
    if (FS_DENSE_ONLY || !d->has_moe) {
      double f = FFN_DENSE_US(cf, sz);
      f = f + tpcoll_us(d, cf, sz);
      const int64_t fns = py_round(f * 1000.0);
      for (int k = I.lane; k < L; k += 32) ffn[(int64_t)i * L + k] = fns;
    } else {
      const bool board = use_job_board(d, FS_ROUTE_UNIFORM, sz);
      for (int l0 = 0; l0 < L; l0 += kLayerChunk) {
        const int lend = min(L, l0 + kLayerChunk);
        if (board) {
          int st = run_route_job(P, I, rd.prefix_mb, i + 1, step, l0, lend - l0, sz, sm->counts);
          double lane_f = 0.0;
          if (st == FS_OK)
            st = moe_layers_lanes(I.lane, job_counts_of(P, I.slot), lend - l0, sz, d->num_experts,
                                  d->top_k, d->d_model, d->expert_d_ff, d->ffn_matrices,
                                  d->dtype_bytes, cf.ep, cf.moe_tp, d->intra_latency_s,
                                  d->intra_bandwidth_bps, cf, &lane_f, nullptr);
          if (st != FS_OK) { fail(I, st, l0); return; }
          if (I.lane < lend - l0) ffn[(int64_t)i * L + l0 + I.lane] = py_round(lane_f * 1000.0);
          I.routing_calls += lend - l0;
          I.routing_draws += (lend - l0) * draws_of(d, FS_ROUTE_UNIFORM, sz);
          if (P.log_enabled && P.log.routes) {
            for (int l = l0; l < lend; l++) {
              load_job_layer(P, I, l - l0, sm);
              log_route(P, I, 0, i + 1, step, l, sz, sm);
            }
          }
          __syncwarp();
          continue;
        }
        derive_layer_keys(P, I, rd.prefix_mb, i + 1, step, l0, L, sm);
        for (int l = l0; l < lend; l++) {
          int st = route_layer(P, I, FS_ROUTE_UNIFORM, sz, sm->keys[l - l0][0], sm->keys[l - l0][1], sm);
          if (st != FS_OK) { fail(I, st, l); return; }
          I.routing_calls++;
          I.routing_draws += draws_of(d, FS_ROUTE_UNIFORM, sz);
          log_route(P, I, 0, i + 1, step, l, sz, sm);
          double f;
#if FS_LEARNED
          if (d->gg_forest != -1)
            st = learned_moe_layer_warp(P, I, sm, sz, cf.ep, cf.moe_tp, cf, &f, nullptr);
          else
#endif
          st = moe_layer_warp(I.lane, sm->counts, sz, d->num_experts, d->top_k, d->d_model,
                              d->expert_d_ff, d->ffn_matrices, d->dtype_bytes, cf.ep, cf.moe_tp,
                              d->intra_latency_s, d->intra_bandwidth_bps, cf, &f, nullptr);
          if (st != FS_OK) { fail(I, st, l); return; }
          __syncwarp();
          if (I.lane == 0) ffn[(int64_t)i * L + l] = py_round(f * 1000.0);
        }
      }
    }
    off += sz;
  }
  __syncwarp();
  // list scheduling over 4 exclusive resources; lowest micro-batch claims first;
  // all completions at an instant are retired before dispatch (af.py:141-229)
  int64_t final_ts = 0, attn_busy = 0, busy4[4] = {0, 0, 0, 0};
  const bool tr = tracing(P);
  if (I.lane == 0) {
    int64_t nseq = I.seq;  // X_DONE events take seqs in dispatch order (af.py:177-201)
    for (int i = 0; i < m; i++) sm->af_stage[i] = 0;
    unsigned long long ready[4] = {0, 0, 0, 0};
    ready[0] = (m == 64) ? ~0ull : ((1ull << m) - 1ull);
    int busy_mb[4] = {-1, -1, -1, -1};
    int64_t endt[4] = {0, 0, 0, 0};
    int64_t t = 0;
    for (;;) {
      for (int res = 0; res < 4; res++) {
        if (busy_mb[res] < 0 && ready[res]) {
          const int i = __ffsll((long long)ready[res]) - 1;
          ready[res] &= ready[res] - 1;
          const int stg = sm->af_stage[i];
          const int k = stg >> 2;
          int64_t dur;
          if (res == 0) dur = sm->af_attn[i];
          else if (res == 2) dur = ffn[(int64_t)i * L + k];
          else dur = sm->af_xfer[i];
          busy_mb[res] = i;
          endt[res] = t + dur;
          busy4[res] += dur;
          if (tr)
            trace_put(P, I, nseq, I.now + t + dur, FS_EV_ATTN_DONE + res, 0, i + 1, k + 1,
                      (int32_t)step, I.now + t);
          nseq++;
        }
      }
      bool any = false;
      int64_t tmin = INT64_MAX;
      for (int res = 0; res < 4; res++)
        if (busy_mb[res] >= 0) { any = true; tmin = min(tmin, endt[res]); }
      if (!any) break;
      t = tmin;
      for (int res = 0; res < 4; res++) {
        if (busy_mb[res] >= 0 && endt[res] == t) {
          const int i = busy_mb[res];
          busy_mb[res] = -1;
          const int stg = sm->af_stage[i];
          const int k = stg >> 2;
          if (res == 2 && k == L - 1) {
            sm->af_stage[i] = -1;
            if (i == m - 1) final_ts = t;
          } else {
            const int nxt = stg + 1;
            sm->af_stage[i] = nxt;
            ready[nxt & 3] |= 1ull << i;
          }
        }
      }
    }
    attn_busy = busy4[0];
  }
  final_ts = __shfl_sync(FS_FULL, final_ts, 0);
  attn_busy = __shfl_sync(FS_FULL, attn_busy, 0);
  for (int res = 0; res < 4; res++) I.af_busy[res] += __shfl_sync(FS_FULL, busy4[res], 0);
  const int64_t dur = final_ts;
  if (dur > 0) {
    const int64_t idle = max((int64_t)0, dur - attn_busy);
    I.bubble_weighted = I.bubble_weighted + (double)idle;
    I.bubble_total += dur;
  }
  I.events += 4LL * m * L - m;  // node-completion events
  I.seq += 4LL * m * L - m;
  s.busy = 1;
  s.steps++;
  s.inflight_phase = PH_AF;
  s.inflight_dur = dur;
  s.inflight_moe = 0;
  if (P.log_enabled) schedule_batch_complete(P, I, 0, PH_AF, dur, rl, B, 0, s.used, step);
  heap_push(I, I.now + dur, K_BATCH_COMPLETE, 0, dur);
}

// ---- the per-instance event loop -------------------------------------------------------------------
// Bytes of per-instance hot state (replica states, event heap, queue / running /
// inflight lists, finish steps); kept in the warp's shared-memory slab when it
// fits, in HBM otherwise (generic pointers make both paths the same code).
__device__ __forceinline__ int64_t slab_need(int R, int N) {
  const int64_t rs = (int64_t)R * sizeof(RepState);
  const int64_t heap = ((int64_t)R + N + 8) * sizeof(HEv);
  const int64_t lists = 3LL * R * (N > 0 ? N : 1) * 4;
  const int64_t fin = ((int64_t)N * 4 + 15) / 16 * 16;
  return rs + heap + lists + fin;
}

__device__ void simulate_instance(const EngineParams& P, int idx, int lane, int slot, WarpSmem* sm,
                                  char* slab) {
  const long long t_start = clock64();
  Inst I;
  const fs_instance_desc* d = &P.descs[idx];
  I.d = d;
  I.idx = idx;
  I.lane = lane;
  I.slot = slot;
  I.N = d->n_requests;
  I.R = d->n_replicas;
  I.mode = d->mode;
  I.ro = d->req_offset;
  I.rb = d->replica_offset;
  if (slab && slab_need(I.R, I.N) <= kSlabBytes) {
    char* p = slab;
    I.rs = reinterpret_cast<RepState*>(p);
    p += (int64_t)I.R * sizeof(RepState);
    I.heap = reinterpret_cast<HEv*>(p);
    p += ((int64_t)I.R + I.N + 8) * sizeof(HEv);
    I.fin = reinterpret_cast<int32_t*>(p);
    p += ((int64_t)I.N * 4 + 15) / 16 * 16;
    I.lists = reinterpret_cast<int32_t*>(p);
  } else {
    I.rs = P.rstate + I.rb;
    I.heap = P.heap + P.heap_base[idx];
    I.fin = P.finish_at + I.ro;
    I.lists = P.lists + P.list_base[idx];
  }
  I.hn = 0;
  I.now = 0;
  I.seq = I.N;  // arrivals hold seq 0..N-1 (base.py:167-177)
  I.events = 0;
  I.max_events = d->max_events;
  I.rr = 0; I.n_done = 0; I.cursor = 0;
  I.status = FS_OK; I.detail = 0;
  I.xh = 0; I.xt = 0;
  I.af_counter = 0;
  for (int k = 0; k < 4; k++) I.af_busy[k] = 0;
  I.bubble_weighted = 0.0;
  I.bubble_total = 0;
  I.prefill_batches = I.decode_batches = I.af_steps = I.moe_samples = I.routing_calls = 0;
  I.routing_draws = 0;
  I.log_batches = I.log_moff = I.log_eoff = I.log_routes = 0;

  if (I.R > FS_MAX_REPLICAS || (d->has_moe && d->num_experts > FS_MAX_EXPERTS)) fail(I, FS_ERR_CAPACITY, 0);
  if (FS_DENSE_ONLY && d->has_moe) fail(I, FS_ERR_INTERNAL, 9);  // host dispatch error
  if ((I.mode == FS_MODE_PD && !FS_HAS_PD) || (I.mode == FS_MODE_AF && !FS_HAS_AF))
    fail(I, FS_ERR_INTERNAL, 10);  // host dispatch error: mode not compiled into this variant
  if (FS_KCAP_MAX <= 4 && d->has_moe && d->top_k + 1 > 4 && d->top_k < d->num_experts)
    fail(I, FS_ERR_INTERNAL, 11);  // host dispatch error: top_k beyond this variant's lists
#if FS_LEARNED
  {
    const int fsel[2] = {d->attn_forest, d->gg_forest};
    for (int k = 0; k < 2; k++) {
      if (fsel[k] >= P.fv.n_forests || fsel[k] < -2) fail(I, FS_ERR_INTERNAL, 7);
      if (fsel[k] >= 0 && fsel[k] < P.fv.n_forests) {
        const int nt = P.fv.forests[fsel[k]].n_trees;
        if (nt < 1 || nt > kMaxForestTrees) fail(I, FS_ERR_CAPACITY, nt);
      }
    }
  }
#else
  // the host picks the learned variant for any instance with a model
  if (d->attn_forest != -1 || d->gg_forest != -1) fail(I, FS_ERR_INTERNAL, 8);
#endif
#if FS_TERM_MEMO
  // the memo holds the previous instance's model: invalidate
  for (int i = lane; i < kMemoSlots; i += 32) sm->memo[i].n = -1;
#endif
  for (int r = lane; r < I.R; r += 32) {
    RepState s;
    s.used = 0; s.outstanding = 0; s.steps = 0; s.busy_ns = 0; s.sum_ctx = 0; s.inflight_dur = 0;
    s.qlen = 0; s.rlen = 0; s.ilen = 0; s.busy = 0; s.start_pending = 0; s.dstep = 0;
    s.min_finish = kNoFinish; s.inflight_phase = 0; s.inflight_moe = 0; s.pad = 0;
    I.rs[r] = s;
  }
  __syncwarp();

  while (I.status == FS_OK) {
    const bool have_arr = I.cursor < I.N;
    const bool have_ev = I.hn > 0;
    if (!have_arr && !have_ev) break;
    const int64_t ta = have_arr ? P.arrival[I.ro + I.cursor] : INT64_MAX;
    const int64_t te = have_ev ? heap_top_t(I) : INT64_MAX;
    I.events++;
    if (I.events > I.max_events) { fail(I, FS_ERR_EVENT_BUDGET, 0); break; }
    if (have_arr && ta <= te) {
      I.now = ta;
      const int req = I.cursor++;
      if (tracing(P) && lane == 0)
        trace_put(P, I, req, ta, FS_EV_REQUEST_ARRIVAL, -1, req, 0, 0, 0);
      if (FS_HAS_PD && I.mode == FS_MODE_PD) pd_arrival(P, I, req);
      else co_arrival(P, I, req);
    } else {
      const HEv e = heap_pop(I);
      I.now = e.t;
      if (e.kind == K_BATCH_START) {
        if (FS_HAS_PD && I.mode == FS_MODE_PD) pd_batch_start(P, I, e.a, sm);
        else co_batch_start(P, I, e.a, sm);
      } else if (e.kind == K_BATCH_COMPLETE) {
        if (FS_HAS_PD && I.mode == FS_MODE_PD) pd_batch_complete(P, I, e.a, e.b);
        else co_batch_complete(P, I, e.a, e.b);
      } else if (FS_HAS_PD && e.kind == K_KV_DONE) {
        pd_transfer_done(P, I, e.a, (int)e.b);
      }
    }
  }
  if (I.status == FS_OK && I.events > I.max_events) fail(I, FS_ERR_EVENT_BUDGET, 0);
  if (I.status == FS_OK && I.n_done != I.N) fail(I, FS_ERR_SIMULATION, I.N - I.n_done);

  __syncwarp();
  if (lane == 0) {
    fs_metric_row& row = P.rows[idx];
    row.status = I.status;
    row.status_detail = I.detail;
    row.events = I.events;
    row.prefill_batches = I.prefill_batches;
    row.decode_batches = I.decode_batches;
    row.af_steps = I.af_steps;
    row.iterations = I.prefill_batches + I.decode_batches + I.af_steps;
    row.routing_calls = I.routing_calls;
    row.routing_draws = I.routing_draws;
    row.moe_layer_samples = d->has_moe ? (I.prefill_batches + I.decode_batches) * (int64_t)d->num_layers : 0;
    row.n_requests = I.N;
    for (int k = 0; k < 4; k++) row.af_busy_ns[k] = I.af_busy[k];
    row.bubble_fraction = (I.mode == FS_MODE_AF && I.af_steps > 0)
                              ? (I.bubble_total ? I.bubble_weighted / (double)I.bubble_total : 0.0)
                              : __longlong_as_double(0x7ff8000000000000LL);
    if (P.log_enabled) {
      if (P.log.batch_count) P.log.batch_count[idx] = I.log_batches;
      if (P.log.route_count) P.log.route_count[idx] = I.log_routes;
      if (P.log.event_count) P.log.event_count[idx] = I.seq;
    }
    if (P.inst_cycles) P.inst_cycles[idx] = clock64() - t_start;
  }
  for (int r = lane; r < I.R; r += 32) {
    const RepState s = I.rs[r];
    fs_replica_out o;
    o.busy_ns = s.busy_ns;
    o.busy_fraction = 0.0;
    o.steps_executed = s.steps;
    P.rep_out[I.rb + r] = o;
  }
  __syncwarp();
  if (lane == 0 && P.inst_done) atomicAdd(P.inst_done, 1);
}

#ifndef FS_SIM_MIN_BLOCKS
#define FS_SIM_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(32 * kWarpsPerCta, FS_SIM_MIN_BLOCKS) sim_kernel(EngineParams P) {
  __shared__ WarpSmem smem[kWarpsPerCta];
  extern __shared__ __align__(16) char slabs[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem* sm = &smem[w];
  char* slab = slabs + (int64_t)w * kSlabBytes;
  for (;;) {
    int k = 0;
    if (lane == 0) k = atomicAdd(P.work_counter, 1);
    k = __shfl_sync(FS_FULL, k, 0);
    if (k >= P.n_inst) break;
    simulate_instance(P, P.order[k], lane, blockIdx.x * kWarpsPerCta + w, sm, slab);
  }
  if (P.jobs && !FS_DENSE_ONLY) help_route_jobs(P, lane, blockIdx.x * kWarpsPerCta + w, sm->counts);
}

// Persistent grid: every CTA resident at once (the job board relies on warps
// that run out of instances turning into helpers; correctness does not).
static size_t sim_dyn_smem() {
  static bool configured = false;
  const size_t bytes = (size_t)kWarpsPerCta * kSlabBytes;
  if (!configured) {
    cudaFuncSetAttribute(sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    configured = true;
  }
  return bytes;
}

// Grid: one resident wave. Without routing jobs a batch smaller than the wave
// gets one warp per instance; with them (MoE instances) the whole wave runs, so
// the warps beyond the instance count start as job-board helpers -- a batch of
// 148 DeepSeek-V3 instances otherwise has one warp per SM for 39 G router keys.
int slots(int n_sms, int n_inst, int ctas_per_sm, bool helpers) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sim_kernel, 32 * kWarpsPerCta,
                                                sim_dyn_smem());
  if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
  if (per_sm < 1) per_sm = 1;
  const int need = (n_inst + kWarpsPerCta - 1) / kWarpsPerCta;
  int grid = n_sms * per_sm;
  if (grid > need && !helpers) grid = need;
  if (grid < 1) grid = 1;
  return grid * kWarpsPerCta;
}

int launch(const EngineParams& p, void* stream) {
  if (p.n_inst <= 0) return 0;
  const int grid = p.n_slots / kWarpsPerCta;
  sim_kernel<<<grid, 32 * kWarpsPerCta, sim_dyn_smem(), (cudaStream_t)stream>>>(p);
  return 1;
}

}  // namespace FS_SIM_NS
}  // namespace fs
