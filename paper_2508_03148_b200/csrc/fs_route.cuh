// fs_route.cuh -- warp-cooperative uniform MoE routing + MoE layer cost.
//
// route_tokens(T, E, k, "uniform", seed)  costmodel/routing.py:65-113
// moe_layer_latency                        costmodel/moe.py:69-128
//
// Layout: row r of the T x E key matrix is split into `nseg` contiguous
// segments; lane (r mod rows_per_pass) * nseg + s generates segment s of row r
// from its own Philox blocks, keeps the (k+1) smallest 53-bit keys packed with
// the expert index ((u >> 11) << 11 | e) in registers, and the nseg lanes of a
// row merge their lists with butterfly shuffles. The k smallest are tallied
// into a per-warp shared-memory histogram; the (k+1)-th is kept only to detect
// an exact tie at the selection boundary (argpartition would pick arbitrarily).
#pragma once
#include "fs_device.cuh"

namespace fs {

// Insert x into the ascending list top[0..kc). Small lists insert branch-free
// (a compare-exchange chain); larger ones skip the chain when x cannot enter.
template <int KCAP>
__device__ __forceinline__ void topk_insert(uint64_t (&top)[KCAP], int kc, uint64_t x,
                                            uint64_t& thr) {
  if (KCAP > 4 && x >= thr) return;
#pragma unroll
  for (int j = 0; j < KCAP; j++) {
    if (j < kc) {
      const uint64_t lo = top[j] < x ? top[j] : x;
      x = top[j] < x ? x : top[j];
      top[j] = lo;
    }
  }
  if (KCAP > 4) {
#pragma unroll
    for (int j = 0; j < KCAP; j++)
      if (j == kc - 1) thr = top[j];
  }
}

// Keys of draws [n0, n1) of a fresh Philox stream (numpy pre-increments the
// counter: draw n is word n % 4 of block n / 4 + 1) inserted into `top`.
// Each block's four words are consumed by an unrolled, predicated loop so the
// block stays in registers; `ebase` maps a draw index to its expert index.
template <int KCAP>
__device__ __forceinline__ void topk_scan(uint64_t (&top)[KCAP], int kc, uint64_t& thr,
                                          uint64_t n0, uint64_t n1, uint64_t ebase, uint64_t k0,
                                          uint64_t k1) {
  for (uint64_t b = n0 >> 2; b <= (n1 - 1) >> 2; b++) {
    const U4 blk = philox4x64_10(b + 1, k0, k1);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint64_t n = 4 * b + j;
      if (n >= n0 && n < n1) {
        const uint64_t packed = ((blk.v[j] >> 11) << 11) | (n - ebase);
        topk_insert<KCAP>(top, kc, packed, thr);
      }
    }
  }
}

// Returns FS_OK or FS_ERR_ROUTING_TIE. counts[] (shared, >= E ints) receives the tally.
template <int KCAP>
__device__ int route_uniform_warp_k(int lane, int64_t T, int E, int k, uint64_t k0, uint64_t k1,
                                    int* counts) {
  for (int e = lane; e < E; e += 32) counts[e] = 0;
  __syncwarp();
  if (T == 0) return FS_OK;
  if (k == E) {
    for (int e = lane; e < E; e += 32) counts[e] = (int)T;
    __syncwarp();
    return FS_OK;
  }
  const int kc = k + 1;  // keep one extra to detect boundary ties
  int nseg = 1;
  if (T < 16) {
    int cap = (int)(32 / T);
    while (nseg * 2 <= cap && nseg * 2 <= E) nseg *= 2;
  }
  const int rows_per_pass = 32 / nseg;
  const int seg_len = (E + nseg - 1) / nseg;
  const int my_row_in_pass = lane / nseg, my_seg = lane % nseg;
  int tie = 0;
  for (int64_t r0 = 0; r0 < T; r0 += rows_per_pass) {
    const int64_t row = r0 + my_row_in_pass;
    const bool active = my_row_in_pass < rows_per_pass && row < T;
    uint64_t top[KCAP];
#pragma unroll
    for (int j = 0; j < KCAP; j++) top[j] = ~0ull;
    uint64_t thr = ~0ull;
    if (active) {
      const int e0 = my_seg * seg_len;
      const int e1 = min(E, e0 + seg_len);
      const uint64_t rb = (uint64_t)row * (uint64_t)E;
      if (e0 < e1) topk_scan<KCAP>(top, kc, thr, rb + e0, rb + e1, rb, k0, k1);
    }
    // merge the nseg partial lists of each row (all lanes participate in shuffles)
    for (int s = 1; s < nseg; s <<= 1) {
      uint64_t other[KCAP];
#pragma unroll
      for (int j = 0; j < KCAP; j++) other[j] = __shfl_xor_sync(FS_FULL, top[j], s);
#pragma unroll
      for (int j = 0; j < KCAP; j++)
        if (j < kc) topk_insert<KCAP>(top, kc, other[j], thr);
    }
    if (active && my_seg == 0) {
      uint64_t kth = 0, next = 0;
#pragma unroll
      for (int j = 0; j < KCAP; j++) {
        if (j < k) atomicAdd(&counts[(int)(top[j] & 0x7FF)], 1);
        if (j == k - 1) kth = top[j];
        if (j == k) next = top[j];
      }
      if ((kth >> 11) == (next >> 11)) tie = 1;
    }
  }
  __syncwarp();
  tie = __any_sync(FS_FULL, tie);
  return tie ? FS_ERR_ROUTING_TIE : FS_OK;
}

// ---- top_k > FS_MAX_TOPK: a full sort of the row ------------------------------------
// Rows too wide for the register top-(k+1) lists are sorted whole: n (key, expert)
// pairs in this warp's global scratch (L1/L2 resident), a warp bitonic network over
// the next power of two, then the k smallest are tallied. Keys are order-preserving
// u64s (the 53-bit draw; or a positive double's IEEE bits). Equal keys at positions
// k-1 and k are an exact boundary tie. Returns 1 on a tie.
__device__ inline int select_sorted(int lane, uint64_t* key, uint64_t* idx, int n, int k,
                                    int* counts) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + lane; i < m; i += 32) { key[i] = ~0ull; idx[i] = 0; }
  __syncwarp();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < m / 2; t += 32) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = key[lo], b = key[hi];
        if ((a > b) == up) {
          key[lo] = b; key[hi] = a;
          const uint64_t x = idx[lo];
          idx[lo] = idx[hi]; idx[hi] = x;
        }
      }
      __syncwarp();
    }
  }
  for (int j = lane; j < k; j += 32) atomicAdd(&counts[(int)idx[j]], 1);
  __syncwarp();
  return key[k - 1] == key[k] ? 1 : 0;
}

// route_tokens uniform for top_k > FS_MAX_TOPK: row by row, the row's E draws in
// Philox blocks spread over the lanes, then select_sorted.
__device__ inline int route_uniform_sorted(int lane, int64_t T, int E, int k, uint64_t k0,
                                           uint64_t k1, double* scratch, int* counts) {
  uint64_t* key = reinterpret_cast<uint64_t*>(scratch + kSortOffset);
  uint64_t* idx = key + FS_MAX_EXPERTS;
  for (int e = lane; e < E; e += 32) counts[e] = 0;
  __syncwarp();
  int tie = 0;
  for (int64_t r = 0; r < T; r++) {
    const uint64_t n0 = (uint64_t)r * E, n1 = n0 + E;
    for (uint64_t b = (n0 >> 2) + lane; b <= (n1 - 1) >> 2; b += 32) {
      const U4 blk = philox4x64_10(b + 1, k0, k1);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint64_t n = 4 * b + j;
        if (n >= n0 && n < n1) {
          key[n - n0] = blk.v[j] >> 11;
          idx[n - n0] = n - n0;
        }
      }
    }
    __syncwarp();
    tie |= select_sorted(lane, key, idx, E, k, counts);
  }
  return tie ? FS_ERR_ROUTING_TIE : FS_OK;
}

__device__ inline int route_uniform_warp(int lane, int64_t T, int E, int k, uint64_t k0,
                                         uint64_t k1, int* counts) {
  if (k + 1 <= 4) return route_uniform_warp_k<4>(lane, T, E, k, k0, k1, counts);
#if !defined(FS_KCAP_MAX) || FS_KCAP_MAX > 4
  if (k + 1 <= 9) return route_uniform_warp_k<9>(lane, T, E, k, k0, k1, counts);
#endif
#if !defined(FS_KCAP_MAX) || FS_KCAP_MAX > 9
  return route_uniform_warp_k<FS_MAX_TOPK + 1>(lane, T, E, k, k0, k1, counts);
#endif
  return FS_ERR_INTERNAL;
}

// moe_layer_latency from a tally in shared memory. All lanes return the same
// total; *ratio (if non-null) gets expert / mean(per_rank) (base.py:247-252).
// Returns FS_OK or a status.
__device__ inline int moe_layer_warp(int lane, const int* counts, int64_t T, int E, int top_k,
                                     int d_model, int expert_d_ff, int nm, int dt, int ep,
                                     int moe_tp, double lat, double bw, const fs_cost_ctx& c,
                                     double* total, double* ratio) {
  if (ep < 1 || moe_tp < 1 || E % ep != 0 || expert_d_ff % moe_tp != 0)
    return FS_ERR_TOPOLOGY_MISMATCH;
  if (T < 1) return FS_ERR_EMPTY_BATCH;
  double gate = linear_us(T, E, d_model, c, dt);
  int64_t routed_bytes = T * (int64_t)top_k * d_model * dt;
  double bpr = i2d(routed_bytes) / (double)ep;
  double dispatch = collective_flt(false, bpr, ep, lat, bw) * 1e6;
  const int per = E / ep;
  const int64_t dffs = expert_d_ff / moe_tp;
  // lane-local max over its ranks (ranks visited in increasing order)
  double best = -1.0;
  int best_r = 0x7fffffff;
  for (int r = lane; r < ep; r += 32) {
    int64_t routed = 0, active = 0;
    for (int j = 0; j < per; j++) {
      int cnt = counts[r * per + j];
      routed += cnt;
      active += cnt > 0;
    }
    double v = routed ? grouped_gemm_us(routed, active, d_model, dffs, nm, c, dt) : 0.0;
    if (v > best) { best = v; best_r = r; }
  }
  // warp arg-max, first index wins ties (per_rank.index(max), moe.py:115-116)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ob = __shfl_xor_sync(FS_FULL, best, o);
    int orr = __shfl_xor_sync(FS_FULL, best_r, o);
    if (ob > best || (ob == best && orr < best_r)) { best = ob; best_r = orr; }
  }
  double expert = best;
  double t = gate + dispatch;
  t = t + expert;
  t = t + dispatch;
  *total = t;
  if (ratio) {
    // sum(per_rank_us) in rank order (Neumaier) -- recomputed serially by every lane
    PySum ps;
    ps.init();
    for (int r = 0; r < ep; r++) {
      int64_t routed = 0, active = 0;
      for (int j = 0; j < per; j++) {
        int cnt = counts[r * per + j];
        routed += cnt;
        active += cnt > 0;
      }
      ps.add(routed ? grouped_gemm_us(routed, active, d_model, dffs, nm, c, dt) : 0.0);
    }
    double s = ps.result();
    *ratio = s > 0 ? expert / (s / (double)ep) : 1.0;
  }
  return FS_OK;
}

// moe_layer_latency for nl layers at once, one layer per lane: lane j < nl reads
// layer j's tally counts[j*E ...] (global, through L2) and returns that layer's
// total in *total (and expert / mean(per_rank) in *ratio when non-null). The
// status is uniform across lanes.
__device__ inline int moe_layers_lanes(int lane, const int32_t* counts, int nl, int64_t T, int E,
                                       int top_k, int d_model, int expert_d_ff, int nm, int dt,
                                       int ep, int moe_tp, double lat, double bw,
                                       const fs_cost_ctx& c, double* total, double* ratio) {
  if (ep < 1 || moe_tp < 1 || E % ep != 0 || expert_d_ff % moe_tp != 0)
    return FS_ERR_TOPOLOGY_MISMATCH;
  if (T < 1) return FS_ERR_EMPTY_BATCH;
  const double gate = linear_us(T, E, d_model, c, dt);
  const int64_t routed_bytes = T * (int64_t)top_k * d_model * dt;
  const double dispatch = collective_flt(false, i2d(routed_bytes) / (double)ep, ep, lat, bw) * 1e6;
  const int per = E / ep;
  const int64_t dffs = expert_d_ff / moe_tp;
  *total = 0.0;
  if (ratio) *ratio = 1.0;
  if (lane < nl) {
    const int32_t* cl = counts + (int64_t)lane * E;
    double expert = 0.0;
    PySum ps;
    ps.init();
    for (int r = 0; r < ep; r++) {
      int64_t routed = 0, active = 0;
      for (int j = 0; j < per; j++) {
        const int cnt = __ldcg(cl + r * per + j);
        routed += cnt;
        active += cnt > 0;
      }
      const double v = routed ? grouped_gemm_us(routed, active, d_model, dffs, nm, c, dt) : 0.0;
      if (r == 0 || v > expert) expert = v;  // max(): first maximum
      if (ratio) ps.add(v);
    }
    double t = gate + dispatch;
    t = t + expert;
    t = t + dispatch;
    *total = t;
    if (ratio) {
      const double s = ps.result();
      *ratio = s > 0 ? expert / (s / (double)ep) : 1.0;
    }
  }
  return FS_OK;
}

}  // namespace fs
