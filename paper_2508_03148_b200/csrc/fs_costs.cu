// fs_costs.cu -- bulk cost-model kernels on the path.
//
//  attention_cost_kernel   CostModel.predict_attention, analytic mode
//                          (costmodel/model.py:313-321 -> analytic.py:32-53)
//                          over CSR batches of per-request (query, kv) lengths:
//                          a segmented reduction, one warp per batch, 128-bit
//                          loads of the length arrays (HBM-bound).
//  attention_features_kernel  AttentionFeatures.vector() (features.py:101-115), the
//                          17-dim input of the learned attention model, with
//                          numpy's pairwise summation order for the std.
//  route_kernel            route_tokens(T, E, k, "uniform", seed) per call.
//  seeds_kernel            derive_router_seed (orchestrator/base.py:63-65).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fs_device.cuh"
#include "fs_engine.h"
#include "fs_route.cuh"
#include "fs_dirichlet.cuh"

namespace fs {

constexpr double kTwo53 = 9007199254740992.0;

struct AttnAcc {
  int64_t sq, skv, s_eq, s_ne, max_term_q, bad_q, bad_dec, bad_pre, bad_kv;
  double max_term;  // 4*l*c*hd upper estimate (exactness guard)
};

__device__ __forceinline__ void attn_acc(AttnAcc& a, int64_t l, int64_t c, bool dec, double hd) {
  a.sq += l;
  a.skv += c;
  a.bad_q |= (l < 1);
  a.bad_dec |= (dec && l != 1);
  a.bad_pre |= (!dec && c < l);
  a.bad_kv |= (c < 1);
  if (c == l) a.s_eq += l * c; else a.s_ne += l * c;
  double t = 4.0 * (double)l * (double)c * hd;
  a.max_term = a.max_term > t ? a.max_term : t;
}

// kU batches in flight per warp: the offsets of kU batches, then every lane's
// 128-bit loads of all kU batches are issued before any reduction, so a warp
// keeps 2*kU independent 16-byte loads outstanding. Decode batches reduce only
// sum(kv) (q == 1 is validated by ballot); prefill batches reduce sum(q),
// sum(kv) and the c == l / c != l products. Lane u then finishes batch u's
// roofline, so the fp64 tail runs once for all kU batches. Batches that are
// unaligned or longer than 128 requests take a generic strided loop.
constexpr int kU = 4;

struct Lanes4 {
  int4 q, kv;
  int n;
};

__device__ __forceinline__ void acc4(int64_t& sq, int64_t& skv, int64_t& seq, int64_t& sne,
                                     int64_t& mlc, int& bad, const Lanes4& x, bool dec) {
  const int qa[4] = {x.q.x, x.q.y, x.q.z, x.q.w};
  const int ka[4] = {x.kv.x, x.kv.y, x.kv.z, x.kv.w};
#pragma unroll
  for (int j = 0; j < 4; j++) {
    if (j < x.n) {
      const int64_t l = qa[j], c = ka[j];
      skv += c;
      bad |= (l < 1) | (c < 1) | (dec ? (l != 1) : (c < l));
      if (!dec) {
        sq += l;
        const int64_t lc = l * c;
        if (c == l) seq += lc; else sne += lc;
        mlc = max(mlc, lc);
      }
    }
  }
}

__global__ void __launch_bounds__(256) attention_cost_kernel_u(
    const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t hd = (int64_t)prm.num_query_heads * prm.head_dim;
  fs_cost_ctx h;
  h.peak_flops = prm.peak_flops; h.mem_bw = prm.mem_bw; h.kernel_overhead_us = prm.kernel_overhead_us;
  h.tp = h.ep = h.moe_tp = h.pp = 1;
  for (int64_t g = warp * kU; g < nb; g += nwarps * kU) {
    int64_t o0[kU], o1[kU];
    bool dv[kU], fast[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int64_t b = g + u;
      const bool valid = b < nb;
      o0[u] = valid ? __ldg(off + b) : 0;
      o1[u] = valid ? __ldg(off + b + 1) : 0;
      dv[u] = valid ? __ldg(dec + b) != 0 : false;
      fast[u] = (o0[u] & 3) == 0 && o1[u] - o0[u] <= 128;
    }
    Lanes4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int64_t i = o0[u] + 4 * lane;
      x[u].n = 0;
      x[u].q = make_int4(0, 0, 0, 0);
      x[u].kv = make_int4(0, 0, 0, 0);
      if (fast[u] && i < o1[u]) {
        x[u].n = (int)min((int64_t)4, o1[u] - i);
        if (x[u].n == 4) {
          x[u].q = __ldg(reinterpret_cast<const int4*>(q + i));
          x[u].kv = __ldg(reinterpret_cast<const int4*>(kv + i));
        } else {
          x[u].q.x = __ldg(q + i); x[u].kv.x = __ldg(kv + i);
          if (x[u].n > 1) { x[u].q.y = __ldg(q + i + 1); x[u].kv.y = __ldg(kv + i + 1); }
          if (x[u].n > 2) { x[u].q.z = __ldg(q + i + 2); x[u].kv.z = __ldg(kv + i + 2); }
        }
      }
    }
    int64_t r_sq[kU], r_skv[kU], r_n[kU];
    double r_fl[kU];
    int r_st[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      int64_t sq = 0, skv = 0, seq = 0, sne = 0, mlc = 0;
      int bad = 0;
      if (fast[u]) {
        acc4(sq, skv, seq, sne, mlc, bad, x[u], dv[u]);
      } else {
        for (int64_t i0 = o0[u] + 4 * lane; i0 < o1[u]; i0 += 128) {
          Lanes4 y;
          y.n = (int)min((int64_t)4, o1[u] - i0);
          int qa[4] = {0, 0, 0, 0}, ka[4] = {0, 0, 0, 0};
          for (int j = 0; j < y.n; j++) { qa[j] = __ldg(q + i0 + j); ka[j] = __ldg(kv + i0 + j); }
          y.q = make_int4(qa[0], qa[1], qa[2], qa[3]);
          y.kv = make_int4(ka[0], ka[1], ka[2], ka[3]);
          acc4(sq, skv, seq, sne, mlc, bad, y, dv[u]);
        }
      }
      skv = warp_sum_i64(skv);
      bad = __any_sync(FS_FULL, bad);
      double flops;
      if (dv[u]) {
        sq = o1[u] - o0[u];  // every q is 1 unless `bad`
        flops = attention_decode_flops(skv, hd);
      } else {
        sq = warp_sum_i64(sq);
        seq = warp_sum_i64(seq);
        sne = warp_sum_i64(sne);
        mlc = warp_max_i64(mlc);
        // each term 4*l*c*hd and the total are exact integers below 2^53: the
        // sequential fp64 sum equals the integer sum in any order
        const double est = 4.0 * (double)hd * ((double)sne + 0.5 * (double)seq);
        if (4.0 * (double)mlc * (double)hd < kTwo53 * 0.5 && est < kTwo53 * 0.5) {
          flops = i2d(4 * hd * sne + 2 * hd * seq);
        } else {
          double tot = 0.0;  // sequential, member order (analytic.py:37-43)
          if (lane == 0)
            for (int64_t i = o0[u]; i < o1[u]; i++) tot = tot + attention_prefill_term(q[i], kv[i], hd);
          flops = __shfl_sync(FS_FULL, tot, 0);
        }
      }
      r_sq[u] = sq;
      r_skv[u] = skv;
      r_n[u] = o1[u] - o0[u];
      r_fl[u] = flops;
      r_st[u] = bad ? FS_ERR_VALUE : FS_OK;
    }
    // lane u finishes batch u
    int64_t msq = 0, mskv = 0, mn = 0;
    double mfl = 0.0;
    int mst = 0;
#pragma unroll
    for (int u = 0; u < kU; u++)
      if (lane == u) { msq = r_sq[u]; mskv = r_skv[u]; mn = r_n[u]; mfl = r_fl[u]; mst = r_st[u]; }
    const int64_t b = g + lane;
    if (lane < kU && b < nb) {
      if (mn <= 0) mst = FS_ERR_EMPTY_BATCH;
      const double us = attention_us_from(mfl, msq, mskv, prm.num_query_heads, prm.num_kv_heads,
                                          prm.head_dim, h, prm.dtype_bytes);
      out[b] = mst == FS_OK ? us : __longlong_as_double(0x7ff8000000000000LL);
      if (status) status[b] = mst;
    }
  }
}

// A batch's roofline from its integer reductions (analytic.py:32-53): decode
// flops from sum(kv); prefill flops as the exact integer sum while every partial
// sum stays below 2^53 (equal to Python's sequential fp64 sum), else the
// sequential fp64 loop in member order. NaN + status for invalid batches.
__device__ __forceinline__ void c2_finish(int64_t b, bool d, int64_t sq, int64_t skv, int64_t seq,
                                          int64_t sne, int64_t mlc, int bad, int64_t o0,
                                          int64_t o1, const int32_t* __restrict__ q,
                                          const int32_t* __restrict__ kv,
                                          const fs_attn_params& prm, const fs_cost_ctx& h,
                                          double* __restrict__ out, int32_t* __restrict__ status) {
  const int64_t hd = (int64_t)prm.num_query_heads * prm.head_dim;
  const int st = o1 <= o0 ? FS_ERR_EMPTY_BATCH : (bad ? FS_ERR_VALUE : FS_OK);
  double flops;
  if (d) {
    sq = o1 - o0;  // every q is 1 unless `bad`
    flops = attention_decode_flops(skv, hd);
  } else {
    const double est = 4.0 * (double)hd * ((double)sne + 0.5 * (double)seq);
    if (4.0 * (double)mlc * (double)hd < kTwo53 * 0.5 && est < kTwo53 * 0.5) {
      flops = i2d(4 * hd * sne + 2 * hd * seq);  // exact integer sum == sequential fp64 sum
    } else {
      flops = 0.0;  // sequential, member order (analytic.py:37-43)
      for (int64_t j = o0; j < o1; j++) flops = flops + attention_prefill_term(q[j], kv[j], hd);
    }
  }
  const double us = attention_us_from(flops, sq, skv, prm.num_query_heads, prm.num_kv_heads,
                                      prm.head_dim, h, prm.dtype_bytes);
  out[b] = st == FS_OK ? us : __longlong_as_double(0x7ff8000000000000LL);
  if (status) status[b] = st;
}

// Thread per batch: each thread streams its own batch's (q, kv) lengths with
// 128-bit loads (scalar head/tail to the 16-byte boundary) and accumulates in
// registers -- no cross-lane reduction at all, so a 72-request batch costs a
// few dozen instructions per warp-batch-slot. Offsets, phases and outputs are
// coalesced across the warp; the per-thread length streams are uncoalesced
// but every 32-byte sector is fully used through L1/L2, so DRAM traffic stays
// at the algorithmic bytes.
__global__ void __launch_bounds__(256) attention_cost_kernel_tpb(
    const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out, int32_t* __restrict__ status) {
  const int64_t hd = (int64_t)prm.num_query_heads * prm.head_dim;
  fs_cost_ctx h;
  h.peak_flops = prm.peak_flops; h.mem_bw = prm.mem_bw; h.kernel_overhead_us = prm.kernel_overhead_us;
  h.tp = h.ep = h.moe_tp = h.pp = 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
    const int64_t o0 = __ldg(off + b), o1 = __ldg(off + b + 1);
    const bool d = __ldg(dec + b) != 0;
    int64_t sq = 0, skv = 0, seq = 0, sne = 0, mlc = 0;
    int bad = 0;
    int64_t i = o0;
    const int64_t head_end = min(o1, (o0 + 3) & ~(int64_t)3);
    for (; i < head_end; i++) {
      Lanes4 x;
      x.q = make_int4(__ldg(q + i), 0, 0, 0);
      x.kv = make_int4(__ldg(kv + i), 0, 0, 0);
      x.n = 1;
      acc4(sq, skv, seq, sne, mlc, bad, x, d);
    }
    for (; i + 4 <= o1; i += 4) {
      Lanes4 x;
      x.q = __ldg(reinterpret_cast<const int4*>(q + i));
      x.kv = __ldg(reinterpret_cast<const int4*>(kv + i));
      x.n = 4;
      acc4(sq, skv, seq, sne, mlc, bad, x, d);
    }
    for (; i < o1; i++) {
      Lanes4 x;
      x.q = make_int4(__ldg(q + i), 0, 0, 0);
      x.kv = make_int4(__ldg(kv + i), 0, 0, 0);
      x.n = 1;
      acc4(sq, skv, seq, sne, mlc, bad, x, d);
    }
    c2_finish(b, d, sq, skv, seq, sne, mlc, bad, o0, o1, q, kv, prm, h, out, status);
  }
}

// ---- TMA-staged variant ----------------------------------------------------------------------
// The CSR length arrays are one contiguous stream per tile, so the whole tile
// (kC2TileBatches batches: their q and kv ranges, widened to 16-byte bounds) is
// moved into shared memory by two cp.async.bulk copies that complete on an
// mbarrier -- no per-thread address streams, no L1 thrash, DRAM reads at the
// algorithmic bytes. A kC2Stages-deep ring keeps that many tiles in flight per
// CTA. Four threads reduce one batch with 128-bit shared-memory loads (thread j
// of a group takes the int4 groups j, j+4, ...; scalar when the batch does not
// start on a 16-byte boundary), partial sums meet by shuffle, and the group
// leader runs the fp64 tail. A tile that does not fit a stage (long batches) or
// whose widened range would read past the arrays runs from global memory.
#ifndef FS_C2_STAGES  // ring depth: 2 stages = 41 KB per CTA, 5 CTAs (20 warps) per SM
#define FS_C2_STAGES 2
#endif
constexpr int kC2TileBatches = 32;   // 4 warps x 8 batches
constexpr int kC2Threads = 128;      // 4 threads per batch
constexpr int kC2Stages = FS_C2_STAGES;
constexpr int kC2StageElems = 2560;  // per array: 32 x 72 members + alignment slack

struct C2Smem {
  int32_t q[kC2Stages][kC2StageElems];
  int32_t kv[kC2Stages][kC2StageElems];
  unsigned long long full[kC2Stages];
  int64_t base[kC2Stages];   // element index of q[stage][0], or -1: read from global
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// producer: thread 0 stages tile `t` into `st` (or marks it for the global path)
__device__ __forceinline__ void c2_issue(C2Smem& S, int st, int64_t t, int64_t nb,
                                         const int32_t* q, const int32_t* kv, const int64_t* off,
                                         bool aligned) {
  const int64_t b0 = t * kC2TileBatches;
  const int64_t b1 = min(nb, b0 + kC2TileBatches);
  const int64_t e0 = __ldg(off + b0), e1 = __ldg(off + b1), eN = __ldg(off + nb);
  const int64_t a0 = e0 & ~(int64_t)3, a1 = (e1 + 3) & ~(int64_t)3;
  const uint32_t bar = smem_u32(&S.full[st]);
  if (!aligned || a1 - a0 > kC2StageElems || a1 > eN || a1 <= a0) {
    S.base[st] = -1;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    return;
  }
  S.base[st] = a0;
  const uint32_t bytes = (uint32_t)((a1 - a0) * 4);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(&S.q[st][0])), "l"(q + a0), "r"(bytes), "r"(bar)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(&S.kv[st][0])), "l"(kv + a0), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void c2_wait(C2Smem& S, int st, uint32_t parity) {
  const uint32_t bar = smem_u32(&S.full[st]);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "C2_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra C2_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kC2Threads) attention_cost_kernel_tma(
    const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out, int32_t* __restrict__ status) {
  extern __shared__ __align__(128) unsigned char c2_raw[];
  C2Smem& S = *reinterpret_cast<C2Smem*>(c2_raw);
  fs_cost_ctx h;
  h.peak_flops = prm.peak_flops; h.mem_bw = prm.mem_bw; h.kernel_overhead_us = prm.kernel_overhead_us;
  h.tp = h.ep = h.moe_tp = h.pp = 1;
  const int tid = threadIdx.x, grp = tid >> 2, j = tid & 3;
  const int64_t n_tiles = (nb + kC2TileBatches - 1) / kC2TileBatches;
  const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv)) & 15) == 0;
  if (tid == 0) {
    for (int s = 0; s < kC2Stages; s++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kC2Stages; s++) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < n_tiles) c2_issue(S, s, t, nb, q, kv, off, aligned);
    }
  }
  __syncthreads();
  int it = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, it++) {
    const int st = it % kC2Stages;
    c2_wait(S, st, (uint32_t)((it / kC2Stages) & 1));
    const int64_t base = S.base[st];
    // phase-sorted assignment inside the tile: decode batches to the first
    // groups, prefill batches to the rest, so a warp's eight batches mostly share
    // a phase and the decode-only / prefill-only work does not diverge
    const int64_t tb0 = t * kC2TileBatches;
    const int ntile = (int)min((int64_t)kC2TileBatches, nb - tb0);
    const int lane = tid & 31;
    const bool ldec = lane < ntile && __ldg(dec + tb0 + lane) != 0;
    const unsigned dmask = __ballot_sync(FS_FULL, ldec);
    const unsigned valid = ntile >= 32 ? 0xFFFFFFFFu : ((1u << ntile) - 1u);
    const int nd = __popc(dmask);
    int pos = ntile;  // groups beyond the tile do nothing
    if (grp < nd) pos = (int)__fns(dmask, 0, grp + 1);
    else if (grp < ntile) pos = (int)__fns(~dmask & valid, 0, grp - nd + 1);
    const int64_t b = pos < ntile ? tb0 + pos : nb;
    int64_t sq = 0, skv = 0, sall = 0, seq = 0, o0 = 0, o1 = 0;
    int bad = 0, ml = 0, mc = 0;
    bool d = false;
    auto member = [&](int l, int c) {
      skv += c;
      bad |= (l < 1) | (c < 1) | (d ? (l != 1) : (c < l));
      if (!d) {
        sq += l;
        const int64_t lc = (int64_t)l * c;
        sall += lc;
        seq += (c == l) ? lc : 0;
        ml = max(ml, l);
        mc = max(mc, c);
      }
    };
    if (b < nb) {
      o0 = __ldg(off + b);
      o1 = __ldg(off + b + 1);
      d = __ldg(dec + b) != 0;
      if (base >= 0 && ((o0 - base) & 3) == 0) {
        const int4* qv = reinterpret_cast<const int4*>(&S.q[st][o0 - base]);
        const int4* kvv = reinterpret_cast<const int4*>(&S.kv[st][o0 - base]);
        const int n4 = (int)((o1 - o0) >> 2);
        for (int i = j; i < n4; i += 4) {
          const int4 a = qv[i], c = kvv[i];
          member(a.x, c.x); member(a.y, c.y); member(a.z, c.z); member(a.w, c.w);
        }
        const int64_t tail = o0 + 4 * (int64_t)n4 + j;
        if (tail < o1) member(S.q[st][tail - base], S.kv[st][tail - base]);
      } else {
        const int32_t* sqp = base >= 0 ? &S.q[st][0] - base : q;
        const int32_t* skp = base >= 0 ? &S.kv[st][0] - base : kv;
        for (int64_t i = o0 + j; i < o1; i += 4) member(sqp[i], skp[i]);
      }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      sq += __shfl_xor_sync(FS_FULL, sq, o);
      skv += __shfl_xor_sync(FS_FULL, skv, o);
      sall += __shfl_xor_sync(FS_FULL, sall, o);
      seq += __shfl_xor_sync(FS_FULL, seq, o);
      ml = max(ml, __shfl_xor_sync(FS_FULL, ml, o));
      mc = max(mc, __shfl_xor_sync(FS_FULL, mc, o));
      bad |= __shfl_xor_sync(FS_FULL, bad, o);
    }
    // max(l) * max(c) bounds every l * c: a conservative exactness guard
    const int64_t mlc = (int64_t)ml * mc, sne = sall - seq;
    if (b < nb && j == 0)
      c2_finish(b, d, sq, skv, seq, sne, mlc, bad, o0, o1, q, kv, prm, h, out, status);
    __syncthreads();  // every thread is done with this stage
    if (tid == 0) {
      const int64_t tn = t + (int64_t)kC2Stages * gridDim.x;
      if (tn < n_tiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads -> TMA writes
        c2_issue(S, st, tn, nb, q, kv, off, aligned);
      }
    }
  }
}

// ---- four threads per batch, asynchronous copies ("g4a", the default) ------------------------
// A group of four threads reduces four consecutive batches one after another,
// the four threads taking interleaved 16-byte pieces of each batch (thread j
// the int4s j, j+4, ...), so every 64 contiguous bytes are read by one load
// instruction's four lanes and only ~57 K batches are partly consumed at any
// time (the thread-per-batch kernel: ~227 K, about the L2, and ~30% of its
// bytes re-read from DRAM). Per member: sums of l, c, l*c and of l*c where
// c == l, and min/max trackers instead of per-member flag logic; the
// validation flags are formed once per batch from them (the same predicates as
// acc4). Thread j then runs batch j's fp64 tail, so the tail uses every lane.
struct G4Acc {
  int64_t sq, skv, sall, seq;
  int minl, maxl, mincl, maxcl;  // min / max of l and of c - l
};
__device__ __forceinline__ void g4_init(G4Acc& a) {
  a.sq = a.skv = a.sall = a.seq = 0;
  a.minl = a.mincl = 0x7fffffff;
  a.maxl = a.maxcl = (int)0x80000000;
}
// products and the c == l split; min/max of l and c - l (validity: l >= 1 and
// c >= l, plus l == 1 for decode -- then c >= 1 follows)
__device__ __forceinline__ void g4_track(G4Acc& a, int l, int c) {
  const int64_t lc = (int64_t)l * c;
  a.sall += lc;
  if (c == l) a.seq += lc;
  const int d = c - l;  // wraps only for c < 0 (then min(d, c) < 0 flags it anyway)
  a.minl = min(a.minl, l);
  a.maxl = max(a.maxl, l);
  a.mincl = min(a.mincl, min(d, c));
  a.maxcl = max(a.maxcl, d);
}
__device__ __forceinline__ void g4_member(G4Acc& a, int l, int c) {
  a.sq += l;
  a.skv += c;
  g4_track(a, l, c);
}
// four members: the sums of l and of c in two 32-bit pair sums (exact for
// valid members, each in [1, 2^31); an invalid batch's sums are never used)
__device__ __forceinline__ void g4_piece(G4Acc& a, const int4& x, const int4& y) {
  a.sq += (int64_t)(uint64_t)((uint32_t)x.x + (uint32_t)x.y) +
          (int64_t)(uint64_t)((uint32_t)x.z + (uint32_t)x.w);
  a.skv += (int64_t)(uint64_t)((uint32_t)y.x + (uint32_t)y.y) +
           (int64_t)(uint64_t)((uint32_t)y.z + (uint32_t)y.w);
  g4_track(a, x.x, y.x); g4_track(a, x.y, y.y);
  g4_track(a, x.z, y.z); g4_track(a, x.w, y.w);
}
__device__ __forceinline__ void g4_reduce(G4Acc& a) {
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    a.sq += __shfl_xor_sync(FS_FULL, a.sq, o);
    a.skv += __shfl_xor_sync(FS_FULL, a.skv, o);
    a.sall += __shfl_xor_sync(FS_FULL, a.sall, o);
    a.seq += __shfl_xor_sync(FS_FULL, a.seq, o);
    a.minl = min(a.minl, __shfl_xor_sync(FS_FULL, a.minl, o));
    a.maxl = max(a.maxl, __shfl_xor_sync(FS_FULL, a.maxl, o));
    a.mincl = min(a.mincl, __shfl_xor_sync(FS_FULL, a.mincl, o));
    a.maxcl = max(a.maxcl, __shfl_xor_sync(FS_FULL, a.maxcl, o));
  }
}
// the batch's flags and the exactness guard's bound: every l*c <= max l * max c
// and max c <= max(c - l) + max l
__device__ __forceinline__ bool g4_bad(const G4Acc& a, bool d, bool empty) {
  return !empty && (a.minl < 1 || a.mincl < 0 || (d && a.maxl != 1));
}
__device__ __forceinline__ int64_t g4_bound(const G4Acc& a) {
  return (int64_t)max(a.maxl, 0) * max((int64_t)a.maxcl + a.maxl, (int64_t)0);
}

// Each thread's 16-byte pieces of the NEXT batch are copied global -> shared
// memory with cp.async (LDGSTS) while the current batch is reduced from shared
// memory: the bytes in flight cost no registers, so an SM keeps about a batch
// per thread in the air. A thread reads back only what it copied itself
// (cp.async.wait_group), so no barrier is needed. Slots hold kG4aSlots pieces
// per array per thread (an 80-member batch); longer batches read the rest from
// global memory. Needs 16-byte aligned length arrays (else: tpb).
#ifndef FS_C2_G4A_THREADS
#define FS_C2_G4A_THREADS 128
#endif
#ifndef FS_C2_G4A_SLOTS
#define FS_C2_G4A_SLOTS 5
#endif
constexpr int kG4aThreads = FS_C2_G4A_THREADS;
constexpr int kG4aSlots = FS_C2_G4A_SLOTS;

__device__ __forceinline__ void g4a_copy16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}

__global__ void __launch_bounds__(kG4aThreads) attention_cost_kernel_g4a(
    const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) int4 g4a_smem[];  // [stage][array][slot][thread]
  fs_cost_ctx h;
  h.peak_flops = prm.peak_flops; h.mem_bw = prm.mem_bw; h.kernel_overhead_us = prm.kernel_overhead_us;
  h.tp = h.ep = h.moe_tp = h.pp = 1;
  const int tid = threadIdx.x, j = tid & 3;
  const int64_t grp = ((int64_t)blockIdx.x * kG4aThreads + tid) >> 2;
  const int64_t ngrp = ((int64_t)gridDim.x * kG4aThreads) >> 2;
  auto slot = [&](int st, int arr, int i) -> int4* {
    return g4a_smem + (((st * 2 + arr) * kG4aSlots + i) * kG4aThreads + tid);
  };
  // the n-th batch this group handles: groups of four consecutive batches, grid-strided
  auto bidx = [&](int64_t n) { return (grp + (n >> 2) * ngrp) * 4 + (n & 3); };
  auto body = [&](int64_t o0, int64_t o1, int64_t& a0, int64_t& n4) {
    a0 = min(o1, (o0 + 3) & ~(int64_t)3);
    n4 = (o1 - a0) >> 2;
  };
  auto issue = [&](int st, int64_t o0, int64_t o1) {
    int64_t a0, n4;
    body(o0, o1, a0, n4);
#pragma unroll
    for (int i = 0; i < kG4aSlots; i++) {
      const int64_t pi = j + 4 * i;
      if (pi < n4) {
        g4a_copy16(slot(st, 0, i), q + a0 + 4 * pi);
        g4a_copy16(slot(st, 1, i), kv + a0 + 4 * pi);
      }
    }
  };
  struct Off { int64_t o0, o1; bool d, valid; };
  auto load_off = [&](int64_t n, Off& r) {
    const int64_t b = bidx(n);
    r.valid = b < nb;
    r.o0 = r.valid ? __ldg(off + b) : 0;
    r.o1 = r.valid ? __ldg(off + b + 1) : 0;
    r.d = r.valid && __ldg(dec + b) != 0;
  };
  Off A, B, C;
  load_off(0, A);
  load_off(1, B);
  if (A.valid) issue(0, A.o0, A.o1);
  asm volatile("cp.async.commit_group;" ::: "memory");
  int64_t m_sq = 0, m_skv = 0, m_seq = 0, m_sall = 0, m_o0 = 0, m_o1 = 0;
  int64_t m_mlc = 0;
  int m_bad = 0;
  bool m_d = false;
  for (int64_t n = 0;; n++) {
    const int64_t b = bidx(n);
    if ((b & ~(int64_t)3) >= nb) break;  // this group's four batches are past the end
    const int k = (int)(n & 3);
    if (B.valid) issue((int)((n + 1) & 1), B.o0, B.o1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    load_off(n + 2, C);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    if (A.valid) {
      const int st = (int)(n & 1);
      const int64_t o0 = A.o0, o1 = A.o1;
      const bool d = A.d;
      G4Acc a;
      g4_init(a);
      int64_t a0, n4;
      body(o0, o1, a0, n4);
      if (o0 + j < a0) g4_member(a, __ldg(q + o0 + j), __ldg(kv + o0 + j));
      const int4* sb = g4a_smem + st * 2 * kG4aSlots * kG4aThreads + tid;
#pragma unroll
      for (int i = 0; i < kG4aSlots; i++) {
        if (j + 4 * i < n4) g4_piece(a, sb[i * kG4aThreads], sb[(kG4aSlots + i) * kG4aThreads]);
      }
      const int4* q4 = reinterpret_cast<const int4*>(q + a0);
      const int4* k4 = reinterpret_cast<const int4*>(kv + a0);
#pragma unroll 1
      for (int64_t i = j + 4 * kG4aSlots; i < n4; i += 4) {  // beyond the slots
        const int4 x = __ldg(q4 + i), y = __ldg(k4 + i);
        g4_piece(a, x, y);
      }
      const int64_t t = a0 + 4 * n4 + j;
      if (t < o1) g4_member(a, __ldg(q + t), __ldg(kv + t));
      g4_reduce(a);
      if (j == k) {
        m_bad = g4_bad(a, d, o1 <= o0);
        m_sq = a.sq; m_skv = a.skv; m_seq = a.seq; m_sall = a.sall;
        m_mlc = g4_bound(a); m_o0 = o0; m_o1 = o1; m_d = d;
      }
    }
    if (k == 3) {
      const int64_t bj = (b & ~(int64_t)3) + j;
      if (bj < nb)
        c2_finish(bj, m_d, m_sq, m_skv, m_seq, m_sall - m_seq, m_mlc, m_bad, m_o0,
                  m_o1, q, kv, prm, h, out, status);
    }
    A = B;
    B = C;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---- synthetic workload generation (workload.py:131-216) --------------------------------------
// One thread per (instance, stream): numpy's streams are sequential (variable
// word consumption: ziggurat slow paths, Lemire rejections), so each stream is
// one lane's loop; a sweep supplies thousands of instances x 3 streams.
struct NpStream32 {
  NpStream g;
  int has32;
  uint32_t u32;
  __device__ uint32_t next_u32() {  // numpy Philox next_uint32: low half first
    if (has32) { has32 = 0; return u32; }
    const uint64_t v = g.next_u64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
};

// Generator.integers(lo, hi + 1, dtype=int64): Lemire's bounded draw
__device__ int64_t np_integer_dev(NpStream32& s, int64_t lo, int64_t hi) {
  const uint64_t rng = (uint64_t)(hi - lo);
  if (rng == 0) return lo;
  if (rng <= 0xFFFFFFFFull) {
    if (rng == 0xFFFFFFFFull) return lo + (int64_t)s.next_u32();
    const uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)s.next_u32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % excl;
      while (left < thr) { m = (uint64_t)s.next_u32() * excl; left = (uint32_t)m; }
    }
    return lo + (int64_t)(m >> 32);
  }
  if (rng == ~0ull) return lo + (int64_t)s.g.next_u64();
  const uint64_t excl = rng + 1;
  uint64_t x = s.g.next_u64();
  uint64_t left = x * excl;
  if (left < excl) {
    const uint64_t thr = (~0ull - rng) % excl;
    while (left < thr) { x = s.g.next_u64(); left = x * excl; }
  }
  return lo + (int64_t)__umul64hi(x, excl);
}

// key = SeedSequence([seed, stream]).generate_state(2, uint64) (workload.py:188-190)
__device__ void workload_key_dev(uint64_t seed, uint32_t stream, uint64_t& k0, uint64_t& k1) {
  uint32_t ent[4];
  int n = int_words(seed, ent);
  n += int_words(stream, ent + n);
  uint64_t key[2];
  seedseq_u64x2(ent, n, key);
  k0 = key[0];
  k1 = key[1];
}

__global__ void workload_kernel(const fs_workload_desc* __restrict__ w, int n,
                                int64_t* __restrict__ arrival, int32_t* __restrict__ prompt,
                                int32_t* __restrict__ output, int32_t* __restrict__ status) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * n) return;
  const int k = t / 3, which = t % 3;
  const fs_workload_desc d = w[k];
  const int64_t o = d.out_offset;
  const int nr = d.n_requests;
  NpStream32 s;
  s.has32 = 0;
  s.u32 = 0;
  s.g.n = 0;
  s.g.w0 = s.g.w1 = s.g.w2 = s.g.w3 = 0;
  workload_key_dev(d.seed, (uint32_t)which, s.g.k0, s.g.k1);
  if (which == 0) {
    if (d.arrival_kind == FS_ARRIVAL_POISSON) {
      const double scale = 1.0 / d.rate_rps;
      double acc = 0.0;
      for (int i = 0; i < nr; i++) {
        acc = acc + scale * np_std_exponential(s.g);  // np.cumsum(exponential(scale, n))
        arrival[o + i] = (int64_t)rint(acc * 1e9);
      }
    } else if (d.arrival_kind == FS_ARRIVAL_FIXED) {
      for (int i = 0; i < nr; i++) arrival[o + i] = (int64_t)i * d.gap_ns;
    } else if (d.arrival_kind == FS_ARRIVAL_AT_ZERO) {
      for (int i = 0; i < nr; i++) arrival[o + i] = 0;
    } else {
      atomicExch(&status[k], FS_ERR_VALUE);
    }
    return;
  }
  const fs_length_dist L = which == 1 ? d.prompt : d.output;
  int32_t* dst = (which == 1 ? prompt : output) + o;
  for (int i = 0; i < nr; i++) {
    int64_t v;
    if (L.kind == FS_LEN_FIXED) {
      v = L.value;
    } else if (L.kind == FS_LEN_UNIFORM) {
      v = np_integer_dev(s, L.lo, L.hi);
    } else if (L.kind == FS_LEN_LOGNORMAL) {
      // random_lognormal = exp(random_normal(mu, sigma)) with glibc's exp (fs_glibm.h)
      double x = rint(glm_exp(L.mu + L.sigma * np_std_normal(s.g)));
      x = x < (double)L.lo ? (double)L.lo : x;
      x = x > (double)L.hi ? (double)L.hi : x;
      v = (int64_t)x;
    } else {
      atomicExch(&status[k], FS_ERR_VALUE);
      return;
    }
    dst[i] = (int32_t)v;
  }
}

// rank of "r{i}" among "r0" .. "r{n-1}" in Python str order, counted per digit
// length in O(digits^2) (no sort)
__device__ int32_t id_str_rank_dev(int64_t i, int64_t n) {
  int dig[20];
  int m = 0;
  {
    int64_t v = i;
    int tmp[20];
    do { tmp[m++] = (int)(v % 10); v /= 10; } while (v);
    for (int q = 0; q < m; q++) dig[q] = tmp[m - 1 - q];
  }
  int64_t rank = 0, lo = 0, hi = 10;
  for (int d = 1; d <= 19 && lo < n; d++) {
    const int64_t end = hi < n ? hi : n;
    if (d <= m) {
      int64_t pre = 0;
      for (int q = 0; q < d; q++) pre = pre * 10 + dig[q];
      int64_t c = pre - lo;
      c = c < 0 ? 0 : (c > end - lo ? end - lo : c);
      rank += c;
      if (d < m && pre >= lo && pre < end) rank += 1;  // a proper prefix sorts first
    } else {
      int64_t tv = 0, scale = 1;
      for (int q = 0; q < m; q++) tv = tv * 10 + dig[q];
      for (int q = 0; q < d - m; q++) scale *= 10;
      int64_t c = tv * scale - lo;
      c = c < 0 ? 0 : (c > end - lo ? end - lo : c);
      rank += c;
    }
    lo = hi;
    hi = hi > INT64_MAX / 10 ? INT64_MAX : hi * 10;
  }
  return (int32_t)rank;
}

__global__ void id_rank_kernel(const fs_workload_desc* __restrict__ w, int n,
                               int32_t* __restrict__ rank) {
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int64_t o = w[k].out_offset;
    const int nr = w[k].n_requests;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) rank[o + i] = id_str_rank_dev(i, nr);
  }
}

int launch_workload(const fs_workload_desc* w, int n, int64_t* arrival, int32_t* prompt,
                    int32_t* output, int32_t* rank, int32_t* status, void* stream) {
  if (n <= 0) return 0;
  const int threads = 128;
  workload_kernel<<<(3 * n + threads - 1) / threads, threads, 0, (cudaStream_t)stream>>>(
      w, n, arrival, prompt, output, status);
  id_rank_kernel<<<n < 148 * 8 ? n : 148 * 8, 64, 0, (cudaStream_t)stream>>>(w, n, rank);
  return 2;
}

int launch_attention_cost(const int32_t* q, const int32_t* kv, const int64_t* off,
                          const uint8_t* dec, int64_t nb, fs_attn_params prm, double* out,
                          int32_t* status, int n_sms, void* stream) {
  if (nb <= 0) return 0;
  const int threads = 256;
  // "g4a" (default: 127 us for 2^20 x 72-request batches, DRAM reads = the algorithmic
  // bytes), "tpb" (167 us, +30% DRAM re-reads), "tma" (181 us), "warp"
  const char* mode = getenv("FS_C2");
  if (mode != nullptr && strcmp(mode, "tma") == 0) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(attention_cost_kernel_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(C2Smem));
      configured = true;
    }
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attention_cost_kernel_tma, kC2Threads,
                                                  sizeof(C2Smem));
    if (per < 1) per = 1;
    const int64_t tiles = (nb + kC2TileBatches - 1) / kC2TileBatches;
    int64_t blocks = (int64_t)n_sms * per;
    if (blocks > tiles) blocks = tiles;
    attention_cost_kernel_tma<<<(int)blocks, kC2Threads, sizeof(C2Smem), (cudaStream_t)stream>>>(
        q, kv, off, dec, nb, prm, out, status);
    return 1;
  }
  const bool al16 = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv)) & 15) == 0;
  if ((mode == nullptr || strcmp(mode, "g4a") == 0) && al16) {
    const int bytes = 2 * 2 * kG4aSlots * kG4aThreads * 16;
    static bool g4a_configured = false;
    if (!g4a_configured) {
      cudaFuncSetAttribute(attention_cost_kernel_g4a, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bytes);
      g4a_configured = true;
    }
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attention_cost_kernel_g4a, kG4aThreads,
                                                  bytes);
    if (per < 1) per = 1;
    int64_t blocks = (nb + kG4aThreads - 1) / kG4aThreads;
    const int64_t cap = (int64_t)n_sms * per;
    if (blocks > cap) blocks = cap;
    attention_cost_kernel_g4a<<<(int)blocks, kG4aThreads, bytes, (cudaStream_t)stream>>>(
        q, kv, off, dec, nb, prm, out, status);
    return 1;
  }
  if (mode == nullptr || strcmp(mode, "warp") != 0) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attention_cost_kernel_tpb, threads, 0);
    if (per < 1) per = 1;
    int64_t blocks = (nb + threads - 1) / threads;
    const int64_t cap = (int64_t)n_sms * per;
    if (blocks > cap) blocks = cap;
    attention_cost_kernel_tpb<<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(q, kv, off, dec, nb,
                                                                                prm, out, status);
    return 1;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attention_cost_kernel_u, threads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (nb + (threads / 32) * kU - 1) / ((threads / 32) * kU);
  const int64_t cap = (int64_t)n_sms * per_sm;  // one resident wave, grid-stride beyond
  if (blocks > cap) blocks = cap;
  attention_cost_kernel_u<<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(q, kv, off, dec, nb,
                                                                            prm, out, status);
  return 1;
}

// ---- features (features.py:23-32, 101-115) ----------------------------------------------
// numpy pairwise_sum for n <= 128 over a[i] = f(i): 8 strided accumulators, tree
// combine, then the tail in order. Computed by lanes 0..7, result on all lanes.
template <typename F>
__device__ double np_pairwise_small(int n, F f, int lane) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res = res + f(i);
    return res;
  }
  double r = 0.0;
  const int full = n - (n % 8);
  if (lane < 8) {
    r = f(lane);
    for (int i = 8; i < full; i += 8) r = r + f(i + lane);
  }
  const double r0 = __shfl_sync(FS_FULL, r, 0), r1 = __shfl_sync(FS_FULL, r, 1);
  const double r2 = __shfl_sync(FS_FULL, r, 2), r3 = __shfl_sync(FS_FULL, r, 3);
  const double r4 = __shfl_sync(FS_FULL, r, 4), r5 = __shfl_sync(FS_FULL, r, 5);
  const double r6 = __shfl_sync(FS_FULL, r, 6), r7 = __shfl_sync(FS_FULL, r, 7);
  double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (int i = full; i < n; i++) res = res + f(i);
  return res;
}
// general n: recursive halving (n2 = n/2 rounded down to a multiple of 8)
template <typename F>
__device__ double np_pairwise(int64_t o, int n, F f, int lane, int depth = 0) {
  if (n <= 128 || depth > 24) return np_pairwise_small(n, [&](int i) { return f(o + i); }, lane);
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double a = np_pairwise(o, n2, f, lane, depth + 1);
  const double b = np_pairwise(o + n2, n - n2, f, lane, depth + 1);
  return a + b;
}

__global__ void attention_features_kernel(const int32_t* q, const int32_t* kv, const int64_t* off,
                                          const uint8_t* dec, int64_t nb, fs_attn_params prm,
                                          double* out17) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nb; b += nwarps) {
    const int64_t o0 = off[b], o1 = off[b + 1];
    const int n = (int)(o1 - o0);
    double feat[17];
    feat[0] = dec[b] ? 1.0 : 0.0;
    feat[1] = (double)n;
    for (int which = 0; which < 2; which++) {
      const int32_t* a = which ? kv : q;
      int64_t s = 0, s2 = 0, mx = INT64_MIN, mn = INT64_MAX;
      for (int64_t i = o0 + lane; i < o1; i += 32) {
        const int64_t v = a[i];
        s += v; s2 += v * v; mx = max(mx, v); mn = min(mn, v);
      }
      s = warp_sum_i64(s);
      s2 = warp_sum_i64(s2);
      mx = warp_max_i64(mx);
      mn = warp_min_i64(mn);
      // integer-valued sums below 2^53 are exact in any summation order
      const double sum = i2d(s);
      const double sum_sq = i2d(s2);
      const double mean = sum / (double)n;
      const double var_sum = np_pairwise(
          o0, n, [&](int64_t i) { const double x = (double)a[i] - mean; return x * x; }, lane);
      const double stdv = sqrt(var_sum / (double)n);
      double* f = feat + 2 + 6 * which;
      f[0] = sum; f[1] = sum_sq; f[2] = (double)mx; f[3] = (double)mn; f[4] = mean; f[5] = stdv;
    }
    feat[14] = (double)prm.num_query_heads;
    feat[15] = (double)prm.num_kv_heads;
    feat[16] = (double)prm.head_dim;
    if (lane < 17) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < 17; j++)
        if (j == lane) v = feat[j];
      out17[b * 17 + lane] = v;
    }
  }
}

int launch_attention_features(const int32_t* q, const int32_t* kv, const int64_t* off,
                              const uint8_t* dec, int64_t nb, fs_attn_params prm, double* out17,
                              void* stream) {
  if (nb <= 0) return 0;
  const int threads = 256;
  int64_t blocks = (nb * 32 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  attention_features_kernel<<<(int)blocks, threads, 0, (cudaStream_t)stream>>>(q, kv, off, dec, nb,
                                                                              prm, out17);
  return 1;
}

// ---- routing / seeds (for parity tests and the routing benchmark) -----------------------------
constexpr int kRouteWarpsPerCta = 4;
constexpr int kRouteMaxCtas = 148 * 8;

__global__ void route_kernel(const int64_t* tokens, const uint64_t* seeds, int n, int E, int k,
                             int policy, double alpha, double* scratch, int32_t* counts,
                             int32_t* status) {
  __shared__ int sm_counts[kRouteWarpsPerCta][FS_MAX_EXPERTS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * kRouteWarpsPerCta + w;
  for (int c = gw; c < n; c += gridDim.x * kRouteWarpsPerCta) {
    int st;
    const int64_t T = tokens[c];
    if (!(1 <= k && k <= E)) st = FS_ERR_INVALID_TOPK;
    else if (E > FS_MAX_EXPERTS) st = FS_ERR_CAPACITY;
    else if (T < 0) st = FS_ERR_ROUTING;
    else if (policy != FS_ROUTE_UNIFORM && policy != FS_ROUTE_DIRICHLET) st = FS_ERR_ROUTING;
    else {
      uint64_t key[2] = {0, 0};
      routing_key(seeds[c], key);
      if (policy == FS_ROUTE_DIRICHLET && T > 0 && k < E)
        st = route_dirichlet_warp(lane, T, E, k, alpha, key[0], key[1],
                                  scratch + (int64_t)gw * kDirScratch, sm_counts[w]);
      else if (T > 0 && k < E && k > FS_MAX_TOPK)
        st = route_uniform_sorted(lane, T, E, k, key[0], key[1],
                                  scratch + (int64_t)gw * kDirScratch, sm_counts[w]);
      else
        st = route_uniform_warp(lane, T, E, k, key[0], key[1], sm_counts[w]);
    }
    __syncwarp();
    for (int e = lane; e < E; e += 32)
      counts[(int64_t)c * E + e] = (st == FS_OK || st == FS_ERR_ROUTING_TIE) ? sm_counts[w][e] : 0;
    if (lane == 0) status[c] = st;
    __syncwarp();
  }
}

int route_scratch_warps(int n) {
  int blocks = (n + kRouteWarpsPerCta - 1) / kRouteWarpsPerCta;
  if (blocks > kRouteMaxCtas) blocks = kRouteMaxCtas;
  return (blocks < 1 ? 1 : blocks) * kRouteWarpsPerCta;
}

int launch_route_tokens(const int64_t* tokens, const uint64_t* seeds, int n, int E, int k,
                        int policy, double alpha, double* scratch, int32_t* counts,
                        int32_t* status, void* stream) {
  if (n <= 0) return 0;
  const int blocks = route_scratch_warps(n) / kRouteWarpsPerCta;
  route_kernel<<<blocks, 32 * kRouteWarpsPerCta, 0, (cudaStream_t)stream>>>(
      tokens, seeds, n, E, k, policy, alpha, scratch, counts, status);
  return 1;
}

__global__ void seeds_kernel(const fs_seed_prefix* pf, const uint32_t* mid, const int32_t* pidx,
                             const int32_t* mb, const int64_t* steps, const int32_t* layers, int n,
                             uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const fs_seed_prefix* p = &pf[pidx[i]];
  int64_t ints[3];
  int k = 0;
  if (mb[i] > 0) ints[k++] = mb[i];
  ints[k++] = steps[i];
  ints[k++] = layers[i];
  int tl;
  const uint8_t* tail = prefix_tail(p, tl);
  out[i] = sha256_tail_first_word(mid + (int64_t)pidx[i] * 8, p->mid_blocks, tail, tl, ints, k);
}

// fs_eval (diagnostics): the pure functions the simulator composes, one record
// per warp, through the same device functions sim_kernel calls. Integers arrive
// as exact doubles. Layouts: include/frontier_b200.h, enum fs_eval_fn.
__device__ __forceinline__ int64_t evi(double x) { return (int64_t)x; }
__global__ void eval_kernel(int fn, const double* __restrict__ in, int in_stride, int64_t n,
                            double* __restrict__ out, int out_stride, int32_t* __restrict__ status) {
  __shared__ int counts[4][FS_MAX_EXPERTS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = (int64_t)blockIdx.x * 4 + w, nw = (int64_t)gridDim.x * 4;
  for (int64_t i = warp; i < n; i += nw) {
    const double* a = in + i * in_stride;
    double* o = out + i * out_stride;
    int st = FS_OK;
    if (fn == FS_EVAL_MOE_LAYER) {
      // [E, k, ep, moe_tp, n_matrices, T, d_model, expert_d_ff, dtype, latency_s,
      //  bandwidth_bps, peak_flops, mem_bw, overhead_us, counts[E]] -> [total_us, ratio]
      const int E = (int)a[0];
      if (E < 1 || E > FS_MAX_EXPERTS) {
        st = FS_ERR_CAPACITY;
      } else {
        for (int e = lane; e < E; e += 32) counts[w][e] = (int)a[14 + e];
        __syncwarp();
        fs_cost_ctx c;
        c.peak_flops = a[11]; c.mem_bw = a[12]; c.kernel_overhead_us = a[13];
        c.tp = 1; c.ep = (int)a[2]; c.moe_tp = (int)a[3]; c.pp = 1;
        double total = 0.0, ratio = 0.0;
        st = moe_layer_warp(lane, counts[w], evi(a[5]), E, (int)a[1], (int)a[6], (int)a[7],
                            (int)a[4], (int)a[8], (int)a[2], (int)a[3], a[9], a[10], c, &total,
                            &ratio);
        if (lane == 0) { o[0] = total; o[1] = ratio; }
        __syncwarp();
      }
    } else if (lane == 0) {
      switch (fn) {
        case FS_EVAL_EXP: o[0] = glm_exp(a[0]); break;
        case FS_EVAL_LOG: o[0] = glm_log(a[0]); break;
        case FS_EVAL_LOG1P: o[0] = glm_log1p(a[0]); break;
        case FS_EVAL_POW: o[0] = glm_pow(a[0], a[1]); break;
        case FS_EVAL_CUDA_EXP: o[0] = exp(a[0]); break;  // CUDA libm, for comparison only
        case FS_EVAL_CUDA_LOG: o[0] = log(a[0]); break;
        case FS_EVAL_CUDA_LOG1P: o[0] = log1p(a[0]); break;
        case FS_EVAL_CUDA_POW: o[0] = pow(a[0], a[1]); break;
        case FS_EVAL_LINEAR: {  // [m, n, k, peak_flops, mem_bw, overhead_us, dtype]
          fs_cost_ctx c;
          c.peak_flops = a[3]; c.mem_bw = a[4]; c.kernel_overhead_us = a[5];
          o[0] = linear_us(evi(a[0]), evi(a[1]), evi(a[2]), c, (int)a[6]);
          break;
        }
        case FS_EVAL_GROUPED_GEMM: {  // [routed, active, d_model, d_ff, n_matrices, peak, bw, ovh, dtype]
          fs_cost_ctx c;
          c.peak_flops = a[5]; c.mem_bw = a[6]; c.kernel_overhead_us = a[7];
          o[0] = grouped_gemm_us(evi(a[0]), evi(a[1]), evi(a[2]), evi(a[3]), (int)a[4], c,
                                 (int)a[8]);
          break;
        }
        case FS_EVAL_COLLECTIVE_INT:  // [kind, bytes_per_rank, n_ranks, latency_s, bandwidth_bps]
          o[0] = collective_int((int)a[0] == 1, evi(a[1]), (int)a[2], a[3], a[4]);
          break;
        case FS_EVAL_COLLECTIVE_FLT:
          o[0] = collective_flt((int)a[0] == 1, a[1], (int)a[2], a[3], a[4]);
          break;
        case FS_EVAL_TRANSFER:  // [bytes, latency_s, bandwidth_bps]
          o[0] = transfer_s(evi(a[0]), a[1], a[2]);
          break;
        default: st = FS_ERR_VALUE;
      }
    }
    if (lane == 0) status[i] = st;
  }
}

int launch_eval(int fn, const double* in, int in_stride, int64_t n, double* out, int out_stride,
                int32_t* status, int n_sms, void* stream) {
  if (n <= 0) return 0;
  int64_t blocks = (n + 3) / 4;
  if (blocks > 8 * n_sms) blocks = 8 * n_sms;
  eval_kernel<<<(int)blocks, 128, 0, (cudaStream_t)stream>>>(fn, in, in_stride, n, out,
                                                             out_stride, status);
  return 1;
}

int launch_router_seeds(const fs_seed_prefix* pf, const uint32_t* mid, const int32_t* pidx,
                        const int32_t* mb, const int64_t* steps, const int32_t* layers, int n,
                        uint32_t* out, void* stream) {
  if (n <= 0) return 0;
  seeds_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(pf, mid, pidx, mb, steps, layers,
                                                                   n, out);
  return 1;
}

}  // namespace fs

namespace fs {

// C2 in learned mode: LearnedOperatorModel.predict_us(AttentionFeatures(...).vector())
// per CSR batch, one warp per batch (features by lanes, one tree per lane).
constexpr int kForestWarps = 4;

__global__ void __launch_bounds__(32 * kForestWarps) attention_forest_kernel(
    ForestView fv, int forest, const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out) {
  __shared__ double sx[kForestWarps][17];
  __shared__ double svals[kForestWarps][kMaxForestTrees];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = (int64_t)blockIdx.x * kForestWarps + w;
  const int64_t nwarps = (int64_t)gridDim.x * kForestWarps;
  for (int64_t b = warp; b < nb; b += nwarps) {
    const int64_t o0 = off[b], n = off[b + 1] - o0;
    const bool d = dec[b] != 0;
    auto fq = [&](int64_t i) -> int64_t { return q[o0 + i]; };
    auto fk = [&](int64_t i) -> int64_t { return kv[o0 + i]; };
    double x[17];
    int bad;
    attention_features_w(d, n, fq, fk, prm.num_query_heads, prm.num_kv_heads, prm.head_dim, lane,
                         x, &bad);
    if (bad != FS_OK) {  // EmptyBatch / ValueError in AttentionFeatures.__post_init__
      if (lane == 0) out[b] = __longlong_as_double(0x7ff8000000000000LL);
      continue;
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 17; j++) sx[w][j] = x[j];
    }
    __syncwarp();
    const double v = forest_predict_w(fv, forest, sx[w], svals[w], lane);
    if (lane == 0) out[b] = v;
    __syncwarp();
  }
}

int launch_attention_forest(const ForestView& fv, int forest, const int32_t* q, const int32_t* kv,
                            const int64_t* off, const uint8_t* dec, int64_t nb, fs_attn_params prm,
                            double* out, int n_sms, void* stream) {
  if (nb <= 0) return 0;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attention_forest_kernel, 32 * kForestWarps, 0);
  if (per < 1) per = 1;
  int64_t blocks = (nb + kForestWarps - 1) / kForestWarps;
  const int64_t cap = (int64_t)n_sms * per;
  if (blocks > cap) blocks = cap;
  attention_forest_kernel<<<(int)blocks, 32 * kForestWarps, 0, (cudaStream_t)stream>>>(
      fv, forest, q, kv, off, dec, nb, prm, out);
  return 1;
}

}  // namespace fs
