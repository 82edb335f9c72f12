// fs_device.cuh -- device primitives shared by the simulation and cost kernels.
//
// Bit-exactness contract: every fp64 expression below follows the reference's
// left-to-right Python evaluation order (file:line cited per function) and the
// library is compiled with -fmad=false, so no multiply-add is contracted.
#pragma once
#include <cstdint>

#include "../../include/frontier_b200.h"
#include "fs_glibm.h"  // glibc exp/log/log1p/pow, bit for bit

#define FS_FULL 0xffffffffu

namespace fs {

// ---------------------------------------------------------------------------
// Python float semantics
// ---------------------------------------------------------------------------
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }
// round(x) -> int, half to even (core.py:25-35)
__device__ __forceinline__ int64_t py_round(double x) { return __double2ll_rn(x); }
// Python's round(x, 6) (floatobject.c double_round: correctly rounded to 6
// decimals, ties to even on the exact binary value), for 0 <= x*1e6 < 2^52 --
// the moe_imbalance report format (base.py:247-252; ratios are >= 1). The exact
// product x*1e6 = hi + lo (FMA residual) decides the integer n; n / 1e6 is then
// the double nearest n * 10^-6, which is what strtod of the rounded decimal gives.
__device__ __forceinline__ double py_round6(double x) {
  const double hi = __dmul_rn(x, 1e6);
  const double lo = __fma_rn(x, 1e6, -hi);
  double n = rint(hi);
  const double f = __dsub_rn(hi, n);  // exact, |f| <= 0.5
  const double up = __dadd_rn(__dsub_rn(f, 0.5), lo), dn = __dadd_rn(__dadd_rn(f, 0.5), lo);
  const bool odd = fmod(n, 2.0) != 0.0;
  if (up > 0.0 || (up == 0.0 && odd)) n = __dadd_rn(n, 1.0);
  else if (dn < 0.0 || (dn == 0.0 && odd)) n = __dsub_rn(n, 1.0);
  return __ddiv_rn(n, 1e6);
}
__device__ __forceinline__ double i2d(int64_t v) { return __ll2double_rn(v); }

// CPython 3.12 builtin sum() of floats from int 0: first item exact, the rest
// Neumaier-compensated, compensation added at the end when finite and nonzero.
struct PySum {
  double f, c;
  int n;
  __device__ __forceinline__ void init() { f = 0.0; c = 0.0; n = 0; }
  __device__ __forceinline__ void add(double x) {
    if (n++ == 0) { f = x; return; }
    double t = f + x;
    if (fabs(f) >= fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  __device__ __forceinline__ double result() const {
    if (n == 0) return 0.0;
    double r = f;
    if (c != 0.0 && isfinite(c)) r += c;
    return r;
  }
};

// ---------------------------------------------------------------------------
// Analytic cost model (costmodel/analytic.py:18-71, topology.py:360-394)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double roofline_us(double flops, double nbytes, const fs_cost_ctx& h) {
  double sec = py_max(flops / h.peak_flops, nbytes / h.mem_bw);
  return h.kernel_overhead_us + sec * 1e6;
}

// analytic.py:23-29 linear_us(m, n, k)
__device__ __forceinline__ double linear_us(int64_t m, int64_t n, int64_t k, const fs_cost_ctx& h,
                                            int dt) {
  double flops = 2.0 * i2d(m);
  flops = flops * i2d(n);
  flops = flops * i2d(k);
  int64_t nbytes = (int64_t)dt * (m * n + n * k + m * k);
  return roofline_us(flops, i2d(nbytes), h);
}

// topology.py:367-394, integer bytes_per_rank (int*int, then int/int true division)
__device__ __forceinline__ double collective_int(bool all_reduce, int64_t bpr, int n, double lat,
                                                 double bw) {
  if (n == 1) return 0.0;
  double wire = i2d(bpr * (int64_t)(n - 1)) / (double)n;
  wire = wire / bw;
  if (all_reduce) return 2.0 * lat + 2.0 * wire;
  return lat + wire;
}
// float bytes_per_rank (moe.py:81-85)
__device__ __forceinline__ double collective_flt(bool all_reduce, double bpr, int n, double lat,
                                                 double bw) {
  if (n == 1) return 0.0;
  double wire = bpr * (double)(n - 1);
  wire = wire / (double)n;
  wire = wire / bw;
  if (all_reduce) return 2.0 * lat + 2.0 * wire;
  return lat + wire;
}

// topology.py:241-243 transfer_time(bytes, link) = alpha + bytes / beta (seconds);
// integer bytes (exact below 2^53)
__device__ __forceinline__ double transfer_s(int64_t nbytes, double lat, double bw) {
  return lat + i2d(nbytes) / bw;
}

// analytic.py:56-71 over one rank's (routed, active) summary
__device__ __forceinline__ double grouped_gemm_us(int64_t routed, int64_t active, int64_t d_model,
                                                  int64_t d_ff, int nm, const fs_cost_ctx& h,
                                                  int dt) {
  double flops = 2.0 * (double)nm;
  flops = flops * i2d(routed);
  flops = flops * i2d(d_model);
  flops = flops * i2d(d_ff);
  int64_t wb = active * nm * d_model * d_ff * dt;
  int64_t ab = routed * nm * (d_model + d_ff) * dt;
  return roofline_us(flops, i2d(wb + ab), h);
}

// analytic.py:46-53 given the batch sums; `flops` precomputed by the caller
__device__ __forceinline__ double attention_us_from(double flops, int64_t sum_q, int64_t sum_kv,
                                                    int hq, int hkv, int hdim,
                                                    const fs_cost_ctx& h, int dt) {
  double kvb = 2.0 * i2d(sum_kv);
  kvb = kvb * (double)hkv;
  kvb = kvb * (double)hdim;
  kvb = kvb * (double)dt;
  double qob = 2.0 * i2d(sum_q);
  qob = qob * (double)hq;
  qob = qob * (double)hdim;
  qob = qob * (double)dt;
  return roofline_us(flops, kvb + qob, h);
}
// analytic.py:35-36 decode flops
__device__ __forceinline__ double attention_decode_flops(int64_t sum_kv, int64_t hd) {
  double f = 4.0 * i2d(sum_kv);
  return f * i2d(hd);
}
// analytic.py:38-42 one prefill member's flops
__device__ __forceinline__ double attention_prefill_term(int64_t l, int64_t c, int64_t hd) {
  double per = 4.0 * i2d(l);
  per = per * i2d(c);
  per = per * i2d(hd);
  if (c == l) per = per / 2.0;
  return per;
}

// ---------------------------------------------------------------------------
// SHA-256 (FIPS 180-4) -- derive_router_seed (orchestrator/base.py:63-65)
// ---------------------------------------------------------------------------
__constant__ uint32_t kSha256K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ inline void sha256_compress(uint32_t h[8], const uint32_t wblk[16]) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; i++) w[i] = wblk[i];
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
  for (int i = 0; i < 64; i++) {
    uint32_t wi;
    if (i < 16) {
      wi = w[i];
    } else {
      uint32_t w15 = w[(i + 1) & 15], w2 = w[(i + 14) & 15];
      uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
      uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
      wi = w[i & 15] + s0 + w[(i + 9) & 15] + s1;
      w[i & 15] = wi;
    }
    uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
    uint32_t ch = (e & f) ^ (~e & g);
    uint32_t t1 = hh + S1 + ch + kSha256K[i] + wi;
    uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
    uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + (S0 + mj);
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// A prefix's bytes after its first mid_blocks full 64-byte blocks (include/
// frontier_b200.h: a long prefix stores only those, its midstate comes from the host).
__device__ __forceinline__ const uint8_t* prefix_tail(const fs_seed_prefix* pf, int& tail_len) {
  const int skip = pf->mid_blocks * 64;
  tail_len = pf->len - skip;
  return pf->len > FS_MAX_PREFIX_BYTES ? pf->bytes : pf->bytes + skip;
}

// Message = prefix ++ ascii(ints joined by ':'), hashed from the midstate `mid`
// (state after the first mid_blocks full blocks of the prefix); `tail` holds the
// prefix's remaining tail_len bytes. Returns int.from_bytes(sha256(msg)[:4], "big").
__device__ inline uint32_t sha256_tail_first_word(const uint32_t mid[8], int mid_blocks,
                                                  const uint8_t* tail, int tail_len,
                                                  const int64_t* ints, int nints) {
  uint32_t wbuf[32];  // up to two 64-byte blocks
#pragma unroll
  for (int i = 0; i < 32; i++) wbuf[i] = 0;
  int pos = 0;
  for (int i = 0; i < tail_len; i++, pos++)
    wbuf[pos >> 2] |= (uint32_t)tail[i] << (24 - 8 * (pos & 3));
  for (int j = 0; j < nints; j++) {
    if (j) { wbuf[pos >> 2] |= (uint32_t)':' << (24 - 8 * (pos & 3)); pos++; }
    int64_t v = ints[j];
    if (v < 0) { wbuf[pos >> 2] |= (uint32_t)'-' << (24 - 8 * (pos & 3)); pos++; v = -v; }
    char digits[20];
    int nd = 0;
    do { digits[nd++] = (char)('0' + (int)(v % 10)); v /= 10; } while (v);
    while (nd) {
      wbuf[pos >> 2] |= (uint32_t)(uint8_t)digits[--nd] << (24 - 8 * (pos & 3));
      pos++;
    }
  }
  uint64_t total_bits = (uint64_t)(mid_blocks * 64 + pos) * 8u;
  wbuf[pos >> 2] |= 0x80u << (24 - 8 * (pos & 3));
  int nblk = (pos + 9 <= 64) ? 1 : 2;
  wbuf[nblk * 16 - 2] = (uint32_t)(total_bits >> 32);
  wbuf[nblk * 16 - 1] = (uint32_t)total_bits;
  uint32_t h[8];
#pragma unroll
  for (int i = 0; i < 8; i++) h[i] = mid[i];
  sha256_compress(h, wbuf);
  if (nblk == 2) sha256_compress(h, wbuf + 16);
  return h[0];
}

// SHA-256 state after the first `nblocks` complete 64-byte blocks of `msg`.
__device__ inline void sha256_midstate(const uint8_t* msg, int nblocks, uint32_t h[8]) {
  h[0] = 0x6a09e667; h[1] = 0xbb67ae85; h[2] = 0x3c6ef372; h[3] = 0xa54ff53a;
  h[4] = 0x510e527f; h[5] = 0x9b05688c; h[6] = 0x1f83d9ab; h[7] = 0x5be0cd19;
  for (int b = 0; b < nblocks; b++) {
    uint32_t w[16];
    for (int i = 0; i < 16; i++) {
      const uint8_t* p = msg + 64 * b + 4 * i;
      w[i] = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
    }
    sha256_compress(h, w);
  }
}

// ---------------------------------------------------------------------------
// numpy SeedSequence (bit_generator.pyx) and Philox4x64-10 (_philox.pyx)
// as used by route_tokens' _rng (costmodel/routing.py:59-62)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  return r ^ (r >> 16);
}
// SeedSequence(entropy).generate_state(2, uint64), pool size 4, n_ent <= 8
__device__ inline void seedseq_u64x2(const uint32_t* ent, int n_ent, uint64_t out[2]) {
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
#pragma unroll
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n_ent ? ent[i] : 0u, hc);
#pragma unroll
  for (int s = 0; s < 4; s++)
#pragma unroll
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < n_ent; s++)
#pragma unroll
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
  uint32_t hb = 0x8b51f9ddu, st[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t v = pool[i] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    st[i] = v ^ (v >> 16);
  }
  out[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  out[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}
// _int_to_uint32_array (little-endian words; [0] for zero)
__device__ __forceinline__ int int_words(uint64_t v, uint32_t* w) {
  w[0] = (uint32_t)v;
  if ((v >> 32) == 0) return 1;
  w[1] = (uint32_t)(v >> 32);
  return 2;
}
// Philox key of np.random.Philox(SeedSequence([seed, 0xE0]).generate_state(2, u64)):
// the state array is passed as `seed`, so it goes through a second SeedSequence.
__device__ inline void routing_key(uint64_t seed, uint64_t key[2]) {
  uint32_t ent[8];
  int n = int_words(seed, ent);
  n += int_words(0xE0u, ent + n);
  uint64_t s[2];
  seedseq_u64x2(ent, n, s);
  n = int_words(s[0], ent);
  n += int_words(s[1], ent + n);
  seedseq_u64x2(ent, n, key);
}

struct U4 {
  uint64_t v[4];
};
// Philox4x64-10 block for counter (c0, 0, 0, 0); numpy pre-increments the
// counter, so draw n of a fresh generator is block(n / 4 + 1)[n % 4].
#ifndef FS_PHILOX_UNROLL  // rounds unrolled per loop trip: 1 measured best (275 vs 315 ms
#define FS_PHILOX_UNROLL 1  // for the C5 sweep; the kernel is instruction-fetch bound)
#endif
constexpr int kPhiloxUnroll = FS_PHILOX_UNROLL;
__device__ __forceinline__ U4 philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll kPhiloxUnroll
  for (int r = 0; r < 10; r++) {
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    uint64_t lo0 = m0 * c0, hi0 = __umul64hi(m0, c0);
    uint64_t lo1 = m1 * c2, hi1 = __umul64hi(m1, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull;  // next round's key
  }
  U4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// The same block with all ten rounds unrolled: no loop-carried register moves,
// ~30% fewer instructions, ten times the code. Used where a lane draws long
// rows (large expert counts), whose warps then run little else.
__device__ __forceinline__ U4 philox4x64_10_unrolled(uint64_t c0, uint64_t k0, uint64_t k1) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    uint64_t lo0 = m0 * c0, hi0 = __umul64hi(m0, c0);
    uint64_t lo1 = m1 * c2, hi1 = __umul64hi(m1, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull;
  }
  U4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// Two independent blocks (counters ca, cb) with their rounds interleaved, so a
// lane has two multiply chains in flight (Philox rounds are serially dependent).
__device__ __forceinline__ void philox4x64_10_x2(uint64_t ca, uint64_t cb, uint64_t k0,
                                                 uint64_t k1, U4& A, U4& B) {
  uint64_t a0 = ca, a1 = 0, a2 = 0, a3 = 0, b0 = cb, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll kPhiloxUnroll
  for (int r = 0; r < 10; r++) {
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    const uint64_t alo0 = m0 * a0, ahi0 = __umul64hi(m0, a0);
    const uint64_t blo0 = m0 * b0, bhi0 = __umul64hi(m0, b0);
    const uint64_t alo1 = m1 * a2, ahi1 = __umul64hi(m1, a2);
    const uint64_t blo1 = m1 * b2, bhi1 = __umul64hi(m1, b2);
    const uint64_t an0 = ahi1 ^ a1 ^ k0, an2 = ahi0 ^ a3 ^ k1;
    const uint64_t bn0 = bhi1 ^ b1 ^ k0, bn2 = bhi0 ^ b3 ^ k1;
    a0 = an0; a1 = alo1; a2 = an2; a3 = alo0;
    b0 = bn0; b1 = blo1; b2 = bn2; b3 = blo0;
    k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull;
  }
  A.v[0] = a0; A.v[1] = a1; A.v[2] = a2; A.v[3] = a3;
  B.v[0] = b0; B.v[1] = b1; B.v[2] = b2; B.v[3] = b3;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FS_FULL, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    int64_t u = __shfl_xor_sync(FS_FULL, v, o);
    v = u > v ? u : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    int64_t u = __shfl_xor_sync(FS_FULL, v, o);
    v = u < v ? u : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_incl_scan_i64(int64_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t u = __shfl_up_sync(FS_FULL, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

}  // namespace fs
