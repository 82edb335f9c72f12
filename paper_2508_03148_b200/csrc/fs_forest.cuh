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

// One tree node in a single 16-byte load: split threshold (or the leaf value
// when feature < 0), split feature, and the left child -- or, for a leaf, the
// rank of its value among all staged leaf values. Fitted trees lay children
// out consecutively (forest.py:194: right = left + 1); files that do not are
// walked through the separate right[] array.
struct __align__(16) NodeP {
  double v;
  int32_t feature;
  int32_t left;  // leaf: value rank (equal values share a rank)
};

struct ForestView {
  const fs_forest_desc* forests;
  int32_t n_forests;
  int32_t consecutive;  // every internal node has right == left + 1
  const int64_t* tree_root;
  const NodeP* nodes;
  const int32_t* right;
  const double* leaf_by_rank;  // leaf value of each rank (ascending)
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

// general n: numpy's recursion (n2 = n/2 rounded down to a multiple of 8),
// unrolled onto an explicit stack -- a recursive device function would leave
// the simulation kernel's stack size statically unknown (the runtime then
// caps it at cudaLimitStackSize, below the kernel's own frame).
template <typename F>
__device__ double np_pairwise_w(int64_t o, int64_t n, F& f, int lane) {
  constexpr int kDepth = 48;  // n < 2^53 needs < 47 levels
  int64_t so[kDepth], sn[kDepth];
  double sl[kDepth];
  bool right[kDepth];
  int top = -1;
  int64_t co = o, cn = n;
  for (;;) {
    while (cn > 128) {  // descend to the leftmost leaf of this call
      int64_t n2 = cn / 2;
      n2 -= n2 % 8;
      ++top;
      so[top] = co; sn[top] = cn; right[top] = false;
      cn = n2;
    }
    double val = np_pairwise_small_w(co, (int)cn, f, lane);
    for (;;) {  // return `val` to the pending calls
      if (top < 0) return val;
      int64_t n2 = sn[top] / 2;
      n2 -= n2 % 8;
      if (!right[top]) {
        sl[top] = val;
        right[top] = true;
        co = so[top] + n2;
        cn = sn[top] - n2;
        break;
      }
      val = sl[top] + val;
      --top;
    }
  }
}

// AttentionFeatures(phase, q, kv, hq, hkv, hd).vector() into x[17] (all lanes).
// One fused pass over (q, kv) gives the integer sums / extremes, the
// __post_init__ checks (features.py:44-66; returned in `bad`, 0 = valid) and
// whether q == kv elementwise; the pairwise std pass then runs only for the
// arrays that need it (decode q is all ones: std 0; q == kv: shared).
template <typename FQ, typename FK>
__device__ void attention_features_w(bool decode, int64_t n, FQ fq, FK fk, int hq, int hkv,
                                     int hdim, int lane, double x[17], int* bad = nullptr) {
  int64_t sq = 0, sq2 = 0, mxq = INT64_MIN, mnq = INT64_MAX;
  int64_t sk = 0, sk2 = 0, mxk = INT64_MIN, mnk = INT64_MAX;
  int b = 0, same = 1;
  for (int64_t i = lane; i < n; i += 32) {
    const int64_t l = fq(i), c = fk(i);
    sq += l; sq2 += l * l;
    mxq = l > mxq ? l : mxq;
    mnq = l < mnq ? l : mnq;
    sk += c; sk2 += c * c;
    mxk = c > mxk ? c : mxk;
    mnk = c < mnk ? c : mnk;
    b |= (l < 1) | (c < 1) | (decode ? (l != 1) : (c < l));
    same &= (l == c);
  }
  sq = warp_sum_i64(sq);
  sq2 = warp_sum_i64(sq2);
  mxq = warp_max_i64(mxq);
  mnq = warp_min_i64(mnq);
  sk = warp_sum_i64(sk);
  sk2 = warp_sum_i64(sk2);
  mxk = warp_max_i64(mxk);
  mnk = warp_min_i64(mnk);
  b = __any_sync(FS_FULL, b);
  same = __all_sync(FS_FULL, same);
  if (bad) *bad = n < 1 ? FS_ERR_EMPTY_BATCH : (b ? FS_ERR_VALUE : FS_OK);
  x[0] = decode ? 1.0 : 0.0;
  x[1] = (double)n;
  // exact: integer partial sums < 2^53
  const double sumq = i2d(sq), meanq = sumq / (double)n;
  const double sumk = i2d(sk), meank = sumk / (double)n;
  double varq;
  if (decode && !b) {
    varq = 0.0;  // every (1 - 1.0)^2 is 0.0
  } else {
    auto dq = [&](int64_t i) { const double d = (double)fq(i) - meanq; return d * d; };
    varq = np_pairwise_w(0, n, dq, lane);
  }
  double vark;
  if (same) {
    vark = varq;
  } else {
    auto dk = [&](int64_t i) { const double d = (double)fk(i) - meank; return d * d; };
    vark = np_pairwise_w(0, n, dk, lane);
  }
  x[2] = sumq; x[3] = i2d(sq2); x[4] = (double)mxq; x[5] = (double)mnq;
  x[6] = meanq; x[7] = sqrt(varq / (double)n);
  x[8] = sumk; x[9] = i2d(sk2); x[10] = (double)mxk; x[11] = (double)mnk;
  x[12] = meank; x[13] = sqrt(vark / (double)n);
  x[14] = (double)hq;
  x[15] = (double)hkv;
  x[16] = (double)hdim;
}

// Ascending bitonic sort of R*32 keys held as k[r] on lane l = element
// r*32 + l: partners 32 apart or more are in the same lane's registers,
// nearer ones are a shuffle away. No shared memory, no divergence.
template <int R>
__device__ __forceinline__ void bitonic_regs(uint32_t (&v)[kMaxForestTrees / 32], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int rp = r ^ (j >> 5);
          if (rp > r) {
            const bool up = (((r << 5) | lane) & k) == 0;
            const uint32_t a = v[r], b = v[rp];
            v[r] = up ? min(a, b) : max(a, b);
            v[rp] = up ? max(a, b) : min(a, b);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const uint32_t a = v[r];
          const uint32_t b = __shfl_xor_sync(FS_FULL, a, j);
          const bool up = (((r << 5) | lane) & k) == 0;
          const bool lower = (lane & j) == 0;
          v[r] = (lower == up) ? min(a, b) : max(a, b);
        }
      }
    }
  }
}

// np.maximum(BaggedForest.predict(x), 1e-6); x and vals in shared memory
// (vals: kMaxForestTrees doubles). Returns the prediction on all lanes.
// Lane l walks trees l, l+32, ... together, so one level of every tree it owns
// is one batch of independent 16-byte loads (the walk is L2-latency bound).
// np.sort of the per-tree values is a register bitonic sort of their 32-bit
// value ranks (host-computed at staging: same order, ties are equal values);
// the sorted values are then summed in numpy's pairwise order.
__device__ inline double forest_predict_w(const ForestView& fv, int forest, const double* x,
                                          double* vals, int lane) {
  constexpr int kPerLane = kMaxForestTrees / 32;
  const fs_forest_desc fd = fv.forests[forest];
  const int nt = fd.n_trees;
  int64_t node[kPerLane];
  uint32_t key[kPerLane];
  unsigned active = 0;
#pragma unroll
  for (int j = 0; j < kPerLane; j++) {
    const int t = lane + 32 * j;
    node[j] = 0;
    key[j] = 0xffffffffu;  // pad sorts last
    if (t < nt) {
      node[j] = __ldg(fv.tree_root + fd.tree_offset + t);
      active |= 1u << j;
    }
  }
  while (active) {
    NodeP nd[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; j++)
      if (active >> j & 1) nd[j] = fv.nodes[node[j]];
#pragma unroll
    for (int j = 0; j < kPerLane; j++) {
      if (!(active >> j & 1)) continue;
      if (nd[j].feature < 0) {
        key[j] = (uint32_t)nd[j].left;
        active &= ~(1u << j);
      } else {
        const bool go_left = x[nd[j].feature] <= nd[j].v;
        node[j] = fv.consecutive ? (int64_t)nd[j].left + (go_left ? 0 : 1)
                                 : (go_left ? (int64_t)nd[j].left : (int64_t)fv.right[node[j]]);
      }
    }
  }
  if (nt <= 32) bitonic_regs<1>(key, lane);
  else if (nt <= 64) bitonic_regs<2>(key, lane);
  else if (nt <= 128) bitonic_regs<4>(key, lane);
  else bitonic_regs<8>(key, lane);
#pragma unroll
  for (int j = 0; j < kPerLane; j++)
    if (lane + 32 * j < nt) vals[lane + 32 * j] = __ldg(fv.leaf_by_rank + key[j]);
  __syncwarp();
  auto leaf = [&](int64_t i) { return vals[i]; };
  const double sum = np_pairwise_w(0, nt, leaf, lane);
  const double mean = sum / (double)nt;
  __syncwarp();
  return mean < 1e-6 ? 1e-6 : mean;
}

}  // namespace fs
