// fs_dirichlet.cuh -- dirichlet_skew MoE routing on the device.
//
// route_tokens(T, E, k, "dirichlet_skew", seed, alpha)   costmodel/routing.py:99-113
//   popularity = max(rng.dirichlet(full(E, alpha)), 1e-12)
//   keys       = rng.exponential(1.0, (T, E)) / popularity
//   counts     = bincount(argpartition(keys, k-1)[:, :k])
//
// The stream is numpy's Generator(Philox(SeedSequence(...))) (routing.py:59-62),
// restated from numpy 2.3.5 (distributions.c, _generator.pyx): the popularity
// vector is E gamma variates (Marsaglia-Tsang / the alpha < 1 rejection loop; a
// beta stick-breaking for alpha < 0.1) drawn by one lane -- E <= 1024 draws with
// data-dependent word consumption. The T*E exponentials are the bulk and are
// drawn warp-parallel:
//
//   * a window is 32 Philox blocks (lane l computes block B+l: words 4(B+l)+j);
//   * numpy's ziggurat (random_standard_exponential) consumes one word per
//     attempt on the fast path (98.9%) and two on the slow path, where the
//     second word is a uniform for the wedge / tail test and a failed wedge test
//     restarts the variate. Which words start an attempt therefore depends on
//     every earlier slow word; the window's slow bits are gathered by ballot into
//     a 128-bit mask and the attempt starts are resolved by jumping from slow
//     word to slow word (about 1.4 per window);
//   * accepted attempts get their variate index from a warp prefix count, are
//     divided by popularity[e] and land in a per-warp ring of keys; completed
//     rows are reduced to their k smallest (k+1 kept to detect an exact
//     boundary tie, like the uniform router) and tallied.
//
// fp64 notes: pow / log / exp / log1p are glibc's own algorithms as numpy's
// distributions.c gets them from libm (fs_glibm.h: the x86-64 FMA variants,
// tables read from the installed libm), so every accept/reject comparison --
// and with it the number of words each variate consumes -- is decided exactly
// as on the host. Everything else is IEEE add/mul/div/sqrt in numpy's order
// (-fmad=false).
#pragma once
#include "fs_device.cuh"
#include "fs_engine.h"
#include "fs_ziggurat.h"

namespace fs {

__device__ __forceinline__ double zig(const uint64_t* t, int i) {
  return __longlong_as_double((long long)__ldg((const unsigned long long*)t + i));
}
__device__ __forceinline__ uint64_t zigu(const uint64_t* t, int i) {
  return (uint64_t)__ldg((const unsigned long long*)t + i);
}

// numpy's buffered Philox stream, one lane (the popularity phase)
struct NpStream {
  uint64_t k0, k1, n;
  uint64_t w0, w1, w2, w3;
  __device__ uint64_t next_u64() {
    if ((n & 3) == 0) {
      const U4 b = philox4x64_10(n / 4 + 1, k0, k1);
      w0 = b.v[0]; w1 = b.v[1]; w2 = b.v[2]; w3 = b.v[3];
    }
    const int j = (int)(n++ & 3);
    return j == 0 ? w0 : j == 1 ? w1 : j == 2 ? w2 : w3;
  }
  __device__ double next_double() { return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
};

static __device__ __noinline__ double np_std_exponential(NpStream& g) {
  for (;;) {
    uint64_t ri = g.next_u64() >> 3;
    const int idx = (int)(ri & 0xFF);
    ri >>= 8;
    const double x = (double)ri * zig(fs_zig_we, idx);
    if (ri < zigu(fs_zig_ke, idx)) return x;
    if (idx == 0) return FS_ZIG_EXP_R - glm_log1p(-g.next_double());
    if ((zig(fs_zig_fe, idx - 1) - zig(fs_zig_fe, idx)) * g.next_double() + zig(fs_zig_fe, idx) <
        glm_exp(-x))
      return x;
  }
}

static __device__ __noinline__ double np_std_normal(NpStream& g) {
  for (;;) {
    uint64_t r = g.next_u64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * zig(fs_zig_wi, idx);
    if (sign & 0x1) x = -x;
    if (rabs < zigu(fs_zig_ki, idx)) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -FS_ZIG_NOR_INV_R * glm_log1p(-g.next_double());
        const double yy = -glm_log1p(-g.next_double());
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 0x1) ? -(FS_ZIG_NOR_R + xx) : FS_ZIG_NOR_R + xx;
      }
    } else {
      if (((zig(fs_zig_fi, idx - 1) - zig(fs_zig_fi, idx)) * g.next_double() +
           zig(fs_zig_fi, idx)) < glm_exp(-0.5 * x * x))
        return x;
    }
  }
}

static __device__ __noinline__ double np_std_gamma(NpStream& g, double shape) {
  if (shape == 1.0) return np_std_exponential(g);
  if (shape == 0.0) return 0.0;
  if (shape < 1.0) {
    for (;;) {
      const double U = g.next_double();
      const double V = np_std_exponential(g);
      if (U <= 1.0 - shape) {
        const double X = glm_pow(U, 1. / shape);
        if (X <= V) return X;
      } else {
        const double Y = -glm_log((1 - U) / shape);
        const double X = glm_pow(1.0 - shape + shape * Y, 1. / shape);
        if (X <= (V + Y)) return X;
      }
    }
  }
  const double b = shape - 1. / 3.;
  const double c = 1. / sqrt(9 * b);
  for (;;) {
    double X, V;
    do {
      X = np_std_normal(g);
      V = 1.0 + c * X;
    } while (V <= 0.0);
    V = V * V * V;
    const double U = g.next_double();
    if (U < 1.0 - 0.0331 * (X * X) * (X * X)) return b * V;
    if (glm_log(U) < 0.5 * X * X + b * (1. - V + glm_log(V))) return b * V;
  }
}

static __device__ __noinline__ double np_beta(NpStream& g, double a, double b) {
  if (a <= 1.0 && b <= 1.0) {
    for (;;) {  // Johnk
      const double U = g.next_double(), V = g.next_double();
      const double X = glm_pow(U, 1.0 / a), Y = glm_pow(V, 1.0 / b);
      const double XpY = X + Y;
      if (XpY <= 1.0 && U + V > 0.0) {
        if (XpY > 0) return X / XpY;
        double logX = glm_log(U) / a, logY = glm_log(V) / b;
        const double logM = logX > logY ? logX : logY;
        logX -= logM;
        logY -= logM;
        return glm_exp(logX - glm_log(glm_exp(logX) + glm_exp(logY)));
      }
    }
  }
  const double Ga = np_std_gamma(g, a), Gb = np_std_gamma(g, b);
  return Ga / (Ga + Gb);
}

// Generator.dirichlet(np.full(E, alpha)) then np.maximum(., 1e-12) into pop[];
// returns the number of stream words consumed. One lane.
static __device__ __noinline__ uint64_t np_dirichlet_sym(uint64_t k0, uint64_t k1, int E, double alpha,
                                                  double* pop) {
  NpStream g;
  g.k0 = k0; g.k1 = k1; g.n = 0;
  g.w0 = g.w1 = g.w2 = g.w3 = 0;
  if (alpha < 0.1) {  // stick-breaking with beta variates
    double cs = 0.0;    // alpha_csum, accumulated right to left like numpy; pop[] holds it
    for (int q = E - 1; q >= 0; q--) { cs += alpha; pop[q] = cs; }
    double acc = 1.0;
    int j;
    for (j = 0; j < E - 1; j++) {
      const double c1 = pop[j + 1];
      const double v = np_beta(g, alpha, c1);
      pop[j] = acc * v;
      acc *= (1. - v);
      if (c1 == 0) { j++; break; }
    }
    for (; j < E - 1; j++) pop[j] = 0.0;
    pop[E - 1] = acc;
  } else {
    double acc = 0.;
    for (int j = 0; j < E; j++) {
      pop[j] = np_std_gamma(g, alpha);
      acc = acc + pop[j];
    }
    const double invacc = 1. / acc;
    for (int j = 0; j < E; j++) pop[j] = pop[j] * invacc;
  }
  for (int j = 0; j < E; j++) pop[j] = pop[j] > 1e-12 ? pop[j] : 1e-12;
  return g.n;
}

// spread the 32 bits of x to bit positions 4*i + j of a 128-bit mask (m[0..3])
__device__ __forceinline__ void spread4(uint32_t x, int j, uint32_t (&m)[4]) {
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t v = (x >> (8 * q)) & 0xFFu;  // lanes 8q..8q+7 -> word q of the mask
    v = (v | (v << 12)) & 0x000F000Fu;
    v = (v | (v << 6)) & 0x03030303u;
    v = (v | (v << 3)) & 0x11111111u;
    m[q] |= v << j;
  }
}
__device__ __forceinline__ bool bit128(const uint32_t (&m)[4], int i) {
  const uint32_t w = i < 32 ? m[0] : i < 64 ? m[1] : i < 96 ? m[2] : m[3];
  return (w >> (i & 31)) & 1u;
}
// first set bit >= i in the 128-bit mask, or 128
__device__ __forceinline__ int next_bit128(const uint32_t (&m)[4], int i) {
  for (int q = i >> 5; q < 4; q++) {
    uint32_t w = m[q];
    if (q == (i >> 5)) w &= ~0u << (i & 31);
    if (w) return 32 * q + __ffs(w) - 1;
  }
  return 128;
}

// ascending (key, expert) list of the kc smallest (keys: IEEE bits of positive doubles)
template <int KCAP>
__device__ __forceinline__ void dtop_insert(uint64_t (&key)[KCAP], int (&ex)[KCAP], int kc,
                                            uint64_t x, int e) {
  if (x >= key[kc - 1]) return;
#pragma unroll
  for (int q = 0; q < KCAP; q++) {
    if (q < kc && x < key[q]) {
      const uint64_t tk = key[q];
      const int te = ex[q];
      key[q] = x; ex[q] = e;
      x = tk; e = te;
    }
  }
}

// Tally the k smallest keys of rows [r0, r1) (keys in ring[(r*E + e) % kDirRing]);
// returns 1 on an exact tie between the k-th and (k+1)-th key of a row.
// E <= 32: one lane per row. Larger E: lanes split each row, lists merge by butterfly.
template <int KCAP>
static __device__ __noinline__ int dir_rows_topk(int lane, const double* ring, int64_t r0, int64_t r1,
                                          int E, int k, int* counts) {
  const int kc = k + 1;
  int tie = 0;
  if (E <= 32 || r1 - r0 >= 32) {  // one lane per row (the caller batches rows)
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      uint64_t key[KCAP];
      int ex[KCAP];
#pragma unroll
      for (int q = 0; q < KCAP; q++) { key[q] = ~0ull; ex[q] = 0; }
      const int64_t base = r * (int64_t)E;
      for (int e = 0; e < E; e++)
        dtop_insert<KCAP>(key, ex, kc,
                          (uint64_t)__double_as_longlong(ring[(base + e) & (kDirRing - 1)]), e);
#pragma unroll
      for (int q = 0; q < KCAP; q++) {
        if (q < k) atomicAdd(&counts[ex[q]], 1);
        if (q == k && key[q] == key[q - 1]) tie = 1;
      }
    }
    return tie;
  }
  for (int64_t r = r0; r < r1; r++) {
    uint64_t key[KCAP];
    int ex[KCAP];
#pragma unroll
    for (int q = 0; q < KCAP; q++) { key[q] = ~0ull; ex[q] = 0; }
    const int64_t base = r * (int64_t)E;
    for (int e = lane; e < E; e += 32)
      dtop_insert<KCAP>(key, ex, kc,
                        (uint64_t)__double_as_longlong(ring[(base + e) & (kDirRing - 1)]), e);
    for (int s = 1; s < 32; s <<= 1) {
      uint64_t ok[KCAP];
      int oe[KCAP];
#pragma unroll
      for (int q = 0; q < KCAP; q++) {
        ok[q] = __shfl_xor_sync(FS_FULL, key[q], s);
        oe[q] = __shfl_xor_sync(FS_FULL, ex[q], s);
      }
#pragma unroll
      for (int q = 0; q < KCAP; q++)
        if (q < kc && ok[q] != ~0ull) dtop_insert<KCAP>(key, ex, kc, ok[q], oe[q]);
    }
    // the partner lists are disjoint (each (row, e) key is inserted once), so
    // equal keys at the boundary are a true tie
#pragma unroll
    for (int q = 0; q < KCAP; q++) {
      if (q < k && lane == 0) atomicAdd(&counts[ex[q]], 1);
      if (q == k && key[q] == key[q - 1]) tie = 1;
    }
  }
  return tie;
}

// top_k > FS_MAX_TOPK: each completed row sorted whole (fs_route.cuh select_sorted)
static __device__ __noinline__ int dir_rows_sorted(int lane, const double* ring, int64_t r0,
                                                   int64_t r1, int E, int k, int* counts,
                                                   double* sortbuf) {
  uint64_t* key = reinterpret_cast<uint64_t*>(sortbuf);
  uint64_t* idx = key + FS_MAX_EXPERTS;
  int tie = 0;
  for (int64_t r = r0; r < r1; r++) {
    const int64_t base = r * (int64_t)E;
    for (int e = lane; e < E; e += 32) {
      key[e] = (uint64_t)__double_as_longlong(ring[(base + e) & (kDirRing - 1)]);
      idx[e] = e;
    }
    __syncwarp();
    tie |= select_sorted(lane, key, idx, E, k, counts);
  }
  return tie;
}

__device__ __forceinline__ int dir_rows(int lane, const double* ring, int64_t r0, int64_t r1,
                                        int E, int k, int* counts) {
  if (r0 >= r1) return 0;
  if (k > FS_MAX_TOPK)  // the ring sits at scratch + FS_MAX_EXPERTS (route_dirichlet_warp)
    return dir_rows_sorted(lane, ring, r0, r1, E, k, counts,
                           const_cast<double*>(ring) - FS_MAX_EXPERTS + kSortOffset);
  if (k + 1 <= 4) return dir_rows_topk<4>(lane, ring, r0, r1, E, k, counts);
  if (k + 1 <= 9) return dir_rows_topk<9>(lane, ring, r0, r1, E, k, counts);
  return dir_rows_topk<FS_MAX_TOPK + 1>(lane, ring, r0, r1, E, k, counts);
}

// route_tokens(T, E, k, "dirichlet_skew", seed, alpha) for T > 0, 1 <= k < E.
// scratch: kDirScratch doubles private to this warp (global). counts: shared.
// Returns FS_OK, FS_ERR_ROUTING (alpha <= 0) or FS_ERR_ROUTING_TIE.
static __device__ __noinline__ int route_dirichlet_warp(int lane, int64_t T, int E, int k, double alpha,
                                                 uint64_t k0, uint64_t k1, double* scratch,
                                                 int* counts) {
  if (!(alpha > 0)) return FS_ERR_ROUTING;
  if (E > FS_MAX_EXPERTS) return FS_ERR_CAPACITY;
  for (int e = lane; e < E; e += 32) counts[e] = 0;
  double* pop = scratch;
  double* ring = scratch + FS_MAX_EXPERTS;
  uint64_t pos = 0;
  if (lane == 0) pos = np_dirichlet_sym(k0, k1, E, alpha, pop);
  pos = __shfl_sync(FS_FULL, pos, 0);
  __syncwarp();
  const int64_t total = T * (int64_t)E;
  int64_t v = 0, next_row = 0;
  int tie = 0;
  while (v < total) {
    const uint64_t B = pos >> 2;
    const int skip = (int)(pos & 3);  // words of block B already consumed
    const U4 blk = philox4x64_10(B + lane + 1, k0, k1);
    // slow-path words (ziggurat fast test fails)
    uint32_t slow_m[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint64_t ri = (blk.v[j] >> 3) >> 8;
      const int idx = (int)((blk.v[j] >> 3) & 0xFF);
      const bool slow = !(ri < zigu(fs_zig_ke, idx));
      spread4(__ballot_sync(FS_FULL, slow), j, slow_m);
    }
    // attempt starts: every word from `skip` on, except the word after a slow start
    uint32_t start_m[4];
#pragma unroll
    for (int q = 0; q < 4; q++) start_m[q] = 0xFFFFFFFFu;
    start_m[0] &= ~0u << skip;
    int p = skip, carry = 0;
    for (;;) {
      const int s = next_bit128(slow_m, p);
      if (s >= 128) break;
      if (s + 1 < 128) {
        start_m[(s + 1) >> 5] &= ~(1u << ((s + 1) & 31));
        p = s + 2;
        // a word consumed as a uniform is not a start, and its own slow bit is moot
        if (p >= 128) break;
        // (the loop resumes at s + 2, the next attempt start)
      } else {
        carry = 1;  // the last word's attempt consumes word 0 of the next window
        break;
      }
    }
    // the next word of each slow start: same lane, or lane+1's word 0, or the
    // first word of the next window (lane 31, j == 3)
    const uint64_t nxt0 = __shfl_down_sync(FS_FULL, blk.v[0], 1);
    uint64_t lastw = nxt0;
    if (lane == 31 && carry) lastw = philox4x64_10(B + 32 + 1, k0, k1).v[0];
    double val[4];
    uint32_t acc_bits = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int i = 4 * lane + j;
      if (!bit128(start_m, i)) continue;
      uint64_t ri = blk.v[j] >> 3;
      const int idx = (int)(ri & 0xFF);
      ri >>= 8;
      const double x = (double)ri * zig(fs_zig_we, idx);
      if (ri < zigu(fs_zig_ke, idx)) { val[j] = x; acc_bits |= 1u << j; continue; }
      const uint64_t nw = j < 3 ? blk.v[j + 1] : lastw;
      const double U = (double)(nw >> 11) * (1.0 / 9007199254740992.0);
      if (idx == 0) {
        val[j] = FS_ZIG_EXP_R - glm_log1p(-U);
        acc_bits |= 1u << j;
      } else if ((zig(fs_zig_fe, idx - 1) - zig(fs_zig_fe, idx)) * U + zig(fs_zig_fe, idx) <
                 glm_exp(-x)) {
        val[j] = x;
        acc_bits |= 1u << j;
      }
    }
    // variate indices: warp exclusive prefix of accepted counts
    const int cnt = __popc(acc_bits);
    const unsigned lt = (1u << lane) - 1u;
    const int pre = __popc(__ballot_sync(FS_FULL, cnt & 1) & lt) +
                    2 * __popc(__ballot_sync(FS_FULL, cnt & 2) & lt) +
                    4 * __popc(__ballot_sync(FS_FULL, cnt & 4) & lt);
    int64_t vi = v + pre;
    int e = (int)(vi - (vi / E) * E);  // one division per lane per window, then a counter
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (!((acc_bits >> j) & 1u)) continue;
      if (vi < total) ring[vi & (kDirRing - 1)] = val[j] / pop[e];
      vi++;
      if (++e == E) e = 0;
    }
    int win = cnt;
#pragma unroll
    for (int o = 16; o; o >>= 1) win += __shfl_xor_sync(FS_FULL, win, o);
    v += win;
    pos = 4 * (B + 32) + (uint64_t)carry;
    __syncwarp();
    // completed rows, tallied 32 at a time (one lane each) once that many are
    // buffered in the ring, or at the end of the call
    const int64_t done_rows = (v < total ? v : total) / E;
    if (done_rows - next_row >= 32 || v >= total || E <= 32) {
      tie |= dir_rows(lane, ring, next_row, done_rows, E, k, counts);
      next_row = done_rows;
    }
    __syncwarp();
  }
  __syncwarp();
  return __any_sync(FS_FULL, tie) ? FS_ERR_ROUTING_TIE : FS_OK;
}

}  // namespace fs
