// fs_forest.cuh -- learned attention model on device (warp-cooperative).
//
//   AttentionFeatures.vector()            costmodel/features.py:23-32, 101-115
//   RegressionTree.predict / BaggedForest  costmodel/forest.py:67-78, 234-239
//   LearnedOperatorModel.predict_matrix    costmodel/model.py:126-133
//
// Features: sums of integer lengths are exact, so any reduction order gives
// numpy's value; the std needs numpy's pairwise summation order over
// (x - mean)^2 (8 strided accumulators for n <= 128, recursive halving above).
// Prediction: one tree per lane, leaf values sorted ascending in shared memory
// (bitonic), numpy's pairwise mean of the sorted values, max(., 1e-6).
#pragma once
#include "fs_device.cuh"

namespace fs {

constexpr int kMaxForestTrees = 256;

struct ForestView {
  const fs_forest_desc* forests;
  int32_t n_forests;
  const int64_t* tree_root;
  const int32_t* feature;
  const double* threshold;
  const int32_t* left;
  const int32_t* right;
  const double* value;
};

// numpy DOUBLE_pairwise_sum over a[i] = f(o + i), i < n, for n <= 128 (all lanes
// get the result; lanes 0..7 hold the strided accumulators)
template <typename F>
__device__ double np_pairwise_small_w(int64_t o, int n, F f, int lane) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res = res + f(o + i);
    return res;
  }
  double r = 0.0;
  const int full = n - (n % 8);
  if (lane < 8) {
    r = f(o + lane);
    for (int i = 8; i < full; i += 8) r = r + f(o + i + lane);
  }
  const double r0 = __shfl_sync(FS_FULL, r, 0), r1 = __shfl_sync(FS_FULL, r, 1);
  const double r2 = __shfl_sync(FS_FULL, r, 2), r3 = __shfl_sync(FS_FULL, r, 3);
  const double r4 = __shfl_sync(FS_FULL, r, 4), r5 = __shfl_sync(FS_FULL, r, 5);
  const double r6 = __shfl_sync(FS_FULL, r, 6), r7 = __shfl_sync(FS_FULL, r, 7);
  double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (int i = full; i < n; i++) res = res + f(o + i);
  return res;
}

// general n: numpy's recursion (n2 = n/2 rounded down to a multiple of 8)
template <typename F>
__device__ double np_pairwise_w(int64_t o, int64_t n, F& f, int lane) {
  if (n <= 128) return np_pairwise_small_w(o, (int)n, f, lane);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double a = np_pairwise_w(o, n2, f, lane);
  const double b = np_pairwise_w(o + n2, n - n2, f, lane);
  return a + b;
}

// _stats(values) for values v(i) = f(i), i < n: sum, sum_sq, max, min, mean, std.
template <typename F>
__device__ void np_stats_w(int64_t n, F f, int lane, double out[6]) {
  int64_t s = 0, s2 = 0, mx = INT64_MIN, mn = INT64_MAX;
  for (int64_t i = lane; i < n; i += 32) {
    const int64_t v = f(i);
    s += v; s2 += v * v;
    mx = v > mx ? v : mx;
    mn = v < mn ? v : mn;
  }
  s = warp_sum_i64(s);
  s2 = warp_sum_i64(s2);
  mx = warp_max_i64(mx);
  mn = warp_min_i64(mn);
  const double sum = i2d(s);        // exact: integer partial sums < 2^53
  const double mean = sum / (double)n;
  auto sq = [&](int64_t i) { const double x = (double)f(i) - mean; return x * x; };
  const double var = np_pairwise_w(0, n, sq, lane);
  out[0] = sum;
  out[1] = i2d(s2);
  out[2] = (double)mx;
  out[3] = (double)mn;
  out[4] = mean;
  out[5] = sqrt(var / (double)n);
}

// AttentionFeatures(phase, q, kv, hq, hkv, hd).vector() into x[17] (all lanes)
template <typename FQ, typename FK>
__device__ void attention_features_w(bool decode, int64_t n, FQ fq, FK fk, int hq, int hkv,
                                     int hdim, int lane, double x[17]) {
  x[0] = decode ? 1.0 : 0.0;
  x[1] = (double)n;
  np_stats_w(n, fq, lane, x + 2);
  np_stats_w(n, fk, lane, x + 8);
  x[14] = (double)hq;
  x[15] = (double)hkv;
  x[16] = (double)hdim;
}

// np.maximum(BaggedForest.predict(x), 1e-6); x and vals in shared memory
// (vals: kMaxForestTrees doubles). Returns the prediction on all lanes.
__device__ inline double forest_predict_w(const ForestView& fv, int forest, const double* x,
                                          double* vals, int lane) {
  const fs_forest_desc fd = fv.forests[forest];
  const int nt = fd.n_trees;
  int np2 = 1;
  while (np2 < nt) np2 <<= 1;
  for (int t = lane; t < np2; t += 32) {
    double v = __longlong_as_double(0x7ff0000000000000LL);  // +inf pad
    if (t < nt) {
      int64_t node = fv.tree_root[fd.tree_offset + t];
      int f;
      while ((f = fv.feature[node]) >= 0) node = (x[f] <= fv.threshold[node]) ? fv.left[node] : fv.right[node];
      v = fv.value[node];
    }
    vals[t] = v;
  }
  __syncwarp();
  // bitonic sort ascending (np.sort; leaf values are finite)
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < np2; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double a = vals[i], b = vals[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { vals[i] = b; vals[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
  auto leaf = [&](int64_t i) { return vals[i]; };
  const double sum = np_pairwise_w(0, nt, leaf, lane);
  const double mean = sum / (double)nt;
  __syncwarp();
  return mean < 1e-6 ? 1e-6 : mean;
}

}  // namespace fs
