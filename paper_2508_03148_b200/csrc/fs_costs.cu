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

#include "fs_device.cuh"
#include "fs_engine.h"
#include "fs_route.cuh"

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

__global__ void attention_cost_kernel(const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
                                      const int64_t* __restrict__ off,
                                      const uint8_t* __restrict__ dec, int64_t nb,
                                      fs_attn_params prm, double* __restrict__ out,
                                      int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t hd = (int64_t)prm.num_query_heads * prm.head_dim;
  const double hdd = (double)hd;
  fs_cost_ctx h;
  h.peak_flops = prm.peak_flops; h.mem_bw = prm.mem_bw; h.kernel_overhead_us = prm.kernel_overhead_us;
  h.tp = h.ep = h.moe_tp = h.pp = 1;
  for (int64_t b = warp; b < nb; b += nwarps) {
    const int64_t o0 = __ldg(off + b), o1 = __ldg(off + b + 1);
    const bool is_dec = __ldg(dec + b) != 0;
    AttnAcc a = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0};
    if ((o0 & 3) == 0) {
      // 128-bit path: lane j covers elements o0 + 4*j .. +3 of each 128-element window
      for (int64_t base = o0; base < o1; base += 128) {
        const int64_t i = base + 4 * lane;
        if (i + 3 < o1) {
          const int4 qv = __ldg(reinterpret_cast<const int4*>(q + i));
          const int4 kvv = __ldg(reinterpret_cast<const int4*>(kv + i));
          attn_acc(a, qv.x, kvv.x, is_dec, hdd);
          attn_acc(a, qv.y, kvv.y, is_dec, hdd);
          attn_acc(a, qv.z, kvv.z, is_dec, hdd);
          attn_acc(a, qv.w, kvv.w, is_dec, hdd);
        } else {
          for (int64_t j = i; j < o1 && j < i + 4; j++) attn_acc(a, __ldg(q + j), __ldg(kv + j), is_dec, hdd);
        }
      }
    } else {
      for (int64_t i = o0 + lane; i < o1; i += 32) attn_acc(a, __ldg(q + i), __ldg(kv + i), is_dec, hdd);
    }
    const int64_t sq = warp_sum_i64(a.sq), skv = warp_sum_i64(a.skv);
    const int64_t s_eq = warp_sum_i64(a.s_eq), s_ne = warp_sum_i64(a.s_ne);
    const int bad_q = __any_sync(FS_FULL, a.bad_q), bad_dec = __any_sync(FS_FULL, a.bad_dec);
    const int bad_pre = __any_sync(FS_FULL, a.bad_pre), bad_kv = __any_sync(FS_FULL, a.bad_kv);
    double mt = a.max_term;
#pragma unroll
    for (int o = 16; o; o >>= 1) mt = fmax(mt, __shfl_xor_sync(FS_FULL, mt, o));
    // AttentionFeatures.__post_init__ checks (features.py:79-95)
    int st = FS_OK;
    if (o1 <= o0) st = FS_ERR_EMPTY_BATCH;
    else if (bad_q || (is_dec && bad_dec) || (!is_dec && bad_pre) || bad_kv) st = FS_ERR_VALUE;
    double flops;
    if (is_dec) {
      flops = attention_decode_flops(skv, hd);
    } else {
      const double total_est = 4.0 * hdd * (double)s_ne + 2.0 * hdd * (double)s_eq;
      if (mt < kTwo53 * 0.5 && total_est < kTwo53 * 0.5) {
        flops = i2d(4 * hd * s_ne + 2 * hd * s_eq);  // exact integer sum == sequential fp64 sum
      } else {
        double tot = 0.0;  // sequential, member order (analytic.py:37-43)
        if (lane == 0)
          for (int64_t i = o0; i < o1; i++) tot = tot + attention_prefill_term(q[i], kv[i], hd);
        flops = __shfl_sync(FS_FULL, tot, 0);
      }
    }
    const double us = attention_us_from(flops, sq, skv, prm.num_query_heads, prm.num_kv_heads,
                                        prm.head_dim, h, prm.dtype_bytes);
    if (lane == 0) {
      out[b] = st == FS_OK ? us : __longlong_as_double(0x7ff8000000000000LL);
      if (status) status[b] = st;
    }
  }
}

// Same reduction with kU batches in flight per warp: the offsets of kU batches,
// then every lane's 128-bit loads of all kU batches are issued before any
// reduction, so a warp keeps 2*kU independent 16-byte loads outstanding.
// Batches that are unaligned or longer than 128 requests take the generic loop.
constexpr int kU = 4;

__device__ __forceinline__ void acc_from_int4(AttnAcc& a, int4 qv, int4 kvv, int n, bool dec,
                                              double hd) {
  if (n > 0) attn_acc(a, qv.x, kvv.x, dec, hd);
  if (n > 1) attn_acc(a, qv.y, kvv.y, dec, hd);
  if (n > 2) attn_acc(a, qv.z, kvv.z, dec, hd);
  if (n > 3) attn_acc(a, qv.w, kvv.w, dec, hd);
}

__global__ void __launch_bounds__(256) attention_cost_kernel_u(
    const int32_t* __restrict__ q, const int32_t* __restrict__ kv,
    const int64_t* __restrict__ off, const uint8_t* __restrict__ dec, int64_t nb,
    fs_attn_params prm, double* __restrict__ out, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t hd = (int64_t)prm.num_query_heads * prm.head_dim;
  const double hdd = (double)hd;
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
    int4 qv[kU], kvv[kU];
    int nh[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int64_t i = o0[u] + 4 * lane;
      nh[u] = 0;
      qv[u] = make_int4(0, 0, 0, 0);
      kvv[u] = make_int4(0, 0, 0, 0);
      if (fast[u] && i < o1[u]) {
        nh[u] = (int)min((int64_t)4, o1[u] - i);
        if (nh[u] == 4) {
          qv[u] = __ldg(reinterpret_cast<const int4*>(q + i));
          kvv[u] = __ldg(reinterpret_cast<const int4*>(kv + i));
        } else {
          qv[u].x = __ldg(q + i); kvv[u].x = __ldg(kv + i);
          if (nh[u] > 1) { qv[u].y = __ldg(q + i + 1); kvv[u].y = __ldg(kv + i + 1); }
          if (nh[u] > 2) { qv[u].z = __ldg(q + i + 2); kvv[u].z = __ldg(kv + i + 2); }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const int64_t b = g + u;
      if (b >= nb) break;  // uniform across the warp
      AttnAcc a = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0};
      if (fast[u]) {
        acc_from_int4(a, qv[u], kvv[u], nh[u], dv[u], hdd);
      } else {
        for (int64_t i = o0[u] + lane; i < o1[u]; i += 32)
          attn_acc(a, __ldg(q + i), __ldg(kv + i), dv[u], hdd);
      }
      const int64_t sq = warp_sum_i64(a.sq), skv = warp_sum_i64(a.skv);
      const int bad = __any_sync(FS_FULL, a.bad_q | a.bad_kv | (dv[u] ? a.bad_dec : a.bad_pre));
      int st = FS_OK;
      if (o1[u] <= o0[u]) st = FS_ERR_EMPTY_BATCH;
      else if (bad) st = FS_ERR_VALUE;
      double flops;
      if (dv[u]) {
        flops = attention_decode_flops(skv, hd);
      } else {
        const int64_t s_eq = warp_sum_i64(a.s_eq), s_ne = warp_sum_i64(a.s_ne);
        double mt = a.max_term;
#pragma unroll
        for (int o = 16; o; o >>= 1) mt = fmax(mt, __shfl_xor_sync(FS_FULL, mt, o));
        const double total_est = 4.0 * hdd * (double)s_ne + 2.0 * hdd * (double)s_eq;
        if (mt < kTwo53 * 0.5 && total_est < kTwo53 * 0.5) {
          flops = i2d(4 * hd * s_ne + 2 * hd * s_eq);  // exact integer sum == sequential fp64 sum
        } else {
          double tot = 0.0;  // sequential, member order (analytic.py:37-43)
          if (lane == 0)
            for (int64_t i = o0[u]; i < o1[u]; i++) tot = tot + attention_prefill_term(q[i], kv[i], hd);
          flops = __shfl_sync(FS_FULL, tot, 0);
        }
      }
      if (lane == u) {
        const double us = attention_us_from(flops, sq, skv, prm.num_query_heads,
                                            prm.num_kv_heads, prm.head_dim, h, prm.dtype_bytes);
        out[b] = st == FS_OK ? us : __longlong_as_double(0x7ff8000000000000LL);
        if (status) status[b] = st;
      }
    }
  }
}

int launch_attention_cost(const int32_t* q, const int32_t* kv, const int64_t* off,
                          const uint8_t* dec, int64_t nb, fs_attn_params prm, double* out,
                          int32_t* status, int n_sms, void* stream) {
  if (nb <= 0) return 0;
  const int threads = 256;
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
__global__ void route_kernel(const int64_t* tokens, const uint64_t* seeds, int n, int E, int k,
                             int32_t* counts, int32_t* status) {
  __shared__ int sm_counts[4][FS_MAX_EXPERTS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = blockIdx.x * 4 + w; c < n; c += gridDim.x * 4) {
    int st;
    const int64_t T = tokens[c];
    if (!(1 <= k && k <= E)) st = FS_ERR_INVALID_TOPK;
    else if (E > FS_MAX_EXPERTS || (k < E && k > FS_MAX_TOPK)) st = FS_ERR_CAPACITY;
    else if (T < 0) st = FS_ERR_ROUTING;
    else {
      uint64_t key[2] = {0, 0};
      routing_key(seeds[c], key);
      st = route_uniform_warp(lane, T, E, k, key[0], key[1], sm_counts[w]);
    }
    __syncwarp();
    for (int e = lane; e < E; e += 32)
      counts[(int64_t)c * E + e] = (st == FS_OK || st == FS_ERR_ROUTING_TIE) ? sm_counts[w][e] : 0;
    if (lane == 0) status[c] = st;
    __syncwarp();
  }
}

int launch_route_uniform(const int64_t* tokens, const uint64_t* seeds, int n, int E, int k,
                         int32_t* counts, int32_t* status, void* stream) {
  if (n <= 0) return 0;
  int blocks = (n + 3) / 4;
  if (blocks > 148 * 8) blocks = 148 * 8;
  route_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(tokens, seeds, n, E, k, counts, status);
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
  out[i] = sha256_tail_first_word(mid + (int64_t)pidx[i] * 8, p->len / 64, p->bytes, p->len, ints, k);
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
