// fs_metrics.cu -- compute_metrics (pkg/src/frontier_sim/metrics.py:81-178) on device.
//
// One warp per instance reads the per-request SoA the simulation kernel left in
// HBM (arrival, first-token and completion ns, output tokens) and reduces it to
// the instance's metric row:
//   * means: CPython sum() (Neumaier) over the values in request order -- the
//     compensation makes the sum order-dependent, so it runs serially per warp
//     over register-staged chunks of 32 values;
//   * nearest-rank percentiles (metrics.py:25-29): an MSB-first radix select
//     (8 passes of 8-bit digits) on 64-bit keys -- integer ns for TTFT/E2E
//     (x/1e9 is monotone in x), the IEEE bit pattern of the positive fp64 TPOT
//     -- with a 256-bin shared-memory histogram per pass;
//   * makespan, throughput, busy fractions, workload averages.
#include <cuda_runtime.h>

#include "fs_device.cuh"
#include "fs_engine.h"

namespace fs {

constexpr int kMetricWarps = 4;

struct MReq {
  int64_t arr, first, done;
  int32_t out;
};

__device__ __forceinline__ MReq mload(const EngineParams& P, int64_t g) {
  MReq r;
  r.arr = P.arrival[g];
  r.first = P.first_ns[g];
  r.done = P.done_ns[g];
  r.out = P.output[g];
  return r;
}

// key of metric `m` for a request; valid=false when the metric is absent (TPOT of 1-token)
__device__ __forceinline__ uint64_t mkey(const MReq& q, int m, bool& valid) {
  valid = true;
  if (m == 0) return (uint64_t)(q.first - q.arr);
  if (m == 1) return (uint64_t)(q.done - q.arr);
  if (q.out <= 1) { valid = false; return 0; }
  const double ttft = i2d(q.first - q.arr) / 1e9;
  const double e2e = i2d(q.done - q.arr) / 1e9;
  const double tpot = (e2e - ttft) / (double)(q.out - 1);
  return (uint64_t)__double_as_longlong(tpot);
}

// k-th smallest (0-based) key of metric m among the instance's requests
__device__ uint64_t radix_select(const EngineParams& P, int64_t ro, int N, int m, int64_t k,
                                 int lane, int* hist) {
  uint64_t prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int i = lane; i < N; i += 32) {
      bool v;
      const uint64_t key = mkey(mload(P, ro + i), m, v);
      if (v && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncwarp();
    int c[8];
    int64_t mine = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) { c[j] = hist[lane * 8 + j]; mine += c[j]; }
    const int64_t incl = warp_incl_scan_i64(mine, lane);
    const int64_t excl = incl - mine;
    const bool here = excl <= k && k < incl;
    const unsigned hm = __ballot_sync(FS_FULL, here);
    const int owner = __ffs(hm) - 1;
    int bucket = 0;
    int64_t before = 0;
    if (lane == owner) {
      int64_t run = excl;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (k < run + c[j]) { bucket = lane * 8 + j; before = run; break; }
        run += c[j];
      }
    }
    bucket = __shfl_sync(FS_FULL, bucket, owner);
    before = __shfl_sync(FS_FULL, before, owner);
    prefix |= (uint64_t)bucket << shift;
    mask |= 0xFFull << shift;
    k -= before;
    __syncwarp();
  }
  return prefix;
}

__device__ __forceinline__ int64_t nearest_rank_idx(int pct, int64_t n) {
  const int64_t idx = (int64_t)ceil((double)pct / 100.0 * (double)n) - 1;
  return idx < 0 ? 0 : idx;
}

__global__ void __launch_bounds__(32 * kMetricWarps) metrics_kernel(EngineParams P) {
  __shared__ int hist_all[kMetricWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int* hist = hist_all[w];
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int idx = blockIdx.x * kMetricWarps + w; idx < P.n_inst; idx += gridDim.x * kMetricWarps) {
    const fs_instance_desc* d = &P.descs[idx];
    fs_metric_row* row = &P.rows[idx];
    const int N = d->n_requests;
    const int64_t ro = d->req_offset;
    const int status = row->status;
    if (status != FS_OK || N == 0) {
      if (lane == 0) {
        for (int j = 0; j < 4; j++) { row->ttft[j] = nan; row->tpot[j] = nan; row->e2e[j] = nan; }
        row->makespan_ns = 0; row->makespan_s = nan; row->throughput_tokens_per_s_per_gpu = nan;
        row->total_tokens = 0; row->n_tpot = 0;
        row->avg_input_tokens = nan; row->avg_output_tokens = nan;
        for (int j = 0; j < 4; j++) row->af_busy_fraction[j] = nan;
      }
      for (int r = lane; r < d->n_replicas; r += 32)
        P.rep_out[d->replica_offset + r].busy_fraction = nan;
      continue;
    }
    // pass 1: extents, token totals, serial Neumaier means in request order
    int64_t maxdone = INT64_MIN, minarr = INT64_MAX, sum_p = 0, sum_o = 0, ntp = 0;
    PySum s_ttft, s_e2e, s_tpot;
    s_ttft.init(); s_e2e.init(); s_tpot.init();
    for (int base = 0; base < N; base += 32) {
      const int i = base + lane;
      const bool valid = i < N;
      double ttft = 0, e2e = 0, tpot = 0;
      bool has_tpot = false;
      if (valid) {
        const MReq q = mload(P, ro + i);
        maxdone = max(maxdone, q.done);
        minarr = min(minarr, q.arr);
        sum_p += P.prompt[ro + i];
        sum_o += q.out;
        ttft = i2d(q.first - q.arr) / 1e9;
        e2e = i2d(q.done - q.arr) / 1e9;
        if (q.out > 1) { tpot = (e2e - ttft) / (double)(q.out - 1); has_tpot = true; }
      }
      const unsigned tm = __ballot_sync(FS_FULL, has_tpot);
      const int nvalid = min(32, N - base);
      for (int j = 0; j < nvalid; j++) {
        s_ttft.add(__shfl_sync(FS_FULL, ttft, j));
        s_e2e.add(__shfl_sync(FS_FULL, e2e, j));
        const double tp = __shfl_sync(FS_FULL, tpot, j);
        if (tm & (1u << j)) s_tpot.add(tp);
      }
      ntp += __popc(tm);
    }
    maxdone = warp_max_i64(maxdone);
    minarr = warp_min_i64(minarr);
    sum_p = warp_sum_i64(sum_p);
    sum_o = warp_sum_i64(sum_o);
    int64_t mk = maxdone - minarr;
    if (mk < 1) mk = 1;
    const double mks = i2d(mk) / 1e9;

    double agg[3][4];
    const int64_t counts[3] = {N, N, ntp};
    const double means[3] = {s_ttft.result() / (double)N, s_e2e.result() / (double)N,
                             ntp ? s_tpot.result() / (double)ntp : nan};
    const int pcts[3] = {50, 90, 99};
    for (int m = 0; m < 3; m++) {
      agg[m][0] = means[m];
      for (int p = 0; p < 3; p++) {
        if (counts[m] == 0) { agg[m][p + 1] = nan; continue; }
        const uint64_t key = radix_select(P, ro, N, m, nearest_rank_idx(pcts[p], counts[m]), lane, hist);
        agg[m][p + 1] = (m == 2) ? __longlong_as_double((long long)key) : i2d((int64_t)key) / 1e9;
      }
    }
    if (lane == 0) {
      row->makespan_ns = mk;
      row->makespan_s = mks;
      row->total_tokens = sum_o;
      row->throughput_tokens_per_s_per_gpu = i2d(sum_o) / mks / (double)d->total_gpus;
      row->n_tpot = (int32_t)ntp;
      for (int j = 0; j < 4; j++) {
        row->ttft[j] = agg[0][j];
        row->e2e[j] = agg[1][j];
        row->tpot[j] = agg[2][j];
      }
      row->avg_input_tokens = i2d(sum_p) / (double)N;
      row->avg_output_tokens = i2d(sum_o) / (double)N;
      for (int j = 0; j < 4; j++)
        row->af_busy_fraction[j] = py_min(1.0, i2d(row->af_busy_ns[j]) / i2d(mk));
    }
    for (int r = lane; r < d->n_replicas; r += 32) {
      fs_replica_out& o = P.rep_out[d->replica_offset + r];
      o.busy_fraction = py_min(1.0, i2d(o.busy_ns) / i2d(mk));
    }
    __syncwarp();
  }
}

int launch_metrics(const EngineParams& p, void* stream) {
  if (p.n_inst <= 0) return 0;
  int grid = (p.n_inst + kMetricWarps - 1) / kMetricWarps;
  if (grid > 148 * 16) grid = 148 * 16;
  metrics_kernel<<<grid, 32 * kMetricWarps, 0, (cudaStream_t)stream>>>(p);
  return 1;
}

}  // namespace fs
