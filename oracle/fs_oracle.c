/*
 * fs_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's per-instance simulation
 * (Frontier, arXiv 2508.03148; reference at /root/reference/pkg/src/frontier_sim).
 * It is the checker for the CUDA engine and the CPU baseline ("port") of
 * bench.py; it is never linked into the product. Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's reference/cpu_baseline legs may
 * load it.
 *
 * Structure deliberately mirrors the reference, not the GPU engine: a binary
 * heap of (timestamp, seq) events where every scheduled event -- the no-op
 * kinds included -- takes a sequence number, exactly as core.py:160-197 does,
 * and the handlers of orchestrator/{colocated,pd,af}.py are restated one by
 * one. The GPU engine instead keeps only the state-changing events.
 *
 * Parity is pinned against golden vectors produced by running the reference
 * itself in the build container (tests/golden/make_golden.py); see
 * tests/test_oracle_golden.py.
 *
 * Floating point: every cost expression follows the reference's left-to-right
 * Python evaluation order in IEEE binary64 (compile with -ffp-contract=off);
 * Python's built-in sum() over floats is CPython 3.12's Neumaier-compensated
 * sum (py_fsum_* below).
 */
#include <math.h>
#include <setjmp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/frontier_b200.h"

/* ------------------------------------------------------------------------ */
/* SHA-256 (FIPS 180-4), used by derive_router_seed (base.py:63-65)          */
/* ------------------------------------------------------------------------ */
static const uint32_t K256[64] = {
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

#define ROTR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void sha256_block(uint32_t h[8], const uint8_t* p) {
  uint32_t w[64];
  for (int i = 0; i < 16; i++)
    w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) |
           ((uint32_t)p[4 * i + 2] << 8) | (uint32_t)p[4 * i + 3];
  for (int i = 16; i < 64; i++) {
    uint32_t s0 = ROTR(w[i - 15], 7) ^ ROTR(w[i - 15], 18) ^ (w[i - 15] >> 3);
    uint32_t s1 = ROTR(w[i - 2], 17) ^ ROTR(w[i - 2], 19) ^ (w[i - 2] >> 10);
    w[i] = w[i - 16] + s0 + w[i - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
  for (int i = 0; i < 64; i++) {
    uint32_t S1 = ROTR(e, 6) ^ ROTR(e, 11) ^ ROTR(e, 25);
    uint32_t ch = (e & f) ^ (~e & g);
    uint32_t t1 = hh + S1 + ch + K256[i] + w[i];
    uint32_t S0 = ROTR(a, 2) ^ ROTR(a, 13) ^ ROTR(a, 22);
    uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    uint32_t t2 = S0 + mj;
    hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

/* First 4 digest bytes, big-endian, of sha256(prior ++ msg) where h0 is the state
 * after the prior_bytes (a multiple of 64) of prior: int.from_bytes(digest[:4], "big"). */
static uint32_t sha256_first_word_from(const uint32_t h0[8], uint64_t prior_bytes,
                                       const uint8_t* msg, size_t len) {
  uint32_t h[8];
  memcpy(h, h0, sizeof h);
  size_t off = 0;
  while (len - off >= 64) { sha256_block(h, msg + off); off += 64; }
  uint8_t blk[128];
  size_t rem = len - off;
  memset(blk, 0, sizeof blk);
  memcpy(blk, msg + off, rem);
  blk[rem] = 0x80;
  size_t nblk = (rem + 9 <= 64) ? 1 : 2;
  uint64_t bits = (prior_bytes + (uint64_t)len) * 8u;
  for (int i = 0; i < 8; i++) blk[nblk * 64 - 1 - i] = (uint8_t)(bits >> (8 * i));
  for (size_t b = 0; b < nblk; b++) sha256_block(h, blk + 64 * b);
  return h[0];
}
static const uint32_t SHA256_IV[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                      0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
static uint32_t sha256_first_word(const uint8_t* msg, size_t len) {
  return sha256_first_word_from(SHA256_IV, 0, msg, len);
}

/* derive_router_seed(master, scope, step, layer): prefix holds "{master}:{scope}:"
 * (or "{master}:{key}:mb" with the micro-batch index as the first tail integer). */
static uint32_t router_seed(const fs_seed_prefix* pf, int mb, int64_t step, int32_t layer) {
  char buf[FS_MAX_PREFIX_BYTES + 64];
  /* a prefix longer than bytes[] arrives as its tail plus the SHA-256 state of
   * its leading 64-byte blocks (include/frontier_b200.h, fs_seed_prefix) */
  const int lng = pf->len > FS_MAX_PREFIX_BYTES;
  const int n0 = lng ? pf->len - 64 * pf->mid_blocks : pf->len;
  memcpy(buf, pf->bytes, (size_t)n0);
  int n = n0;
  if (mb > 0) n += sprintf(buf + n, "%d:", mb);
  n += sprintf(buf + n, "%lld:%d", (long long)step, (int)layer);
  if (lng) return sha256_first_word_from(pf->mid, 64u * (uint64_t)pf->mid_blocks,
                                         (const uint8_t*)buf, (size_t)n);
  return sha256_first_word((const uint8_t*)buf, (size_t)n);
}

/* ------------------------------------------------------------------------ */
/* numpy SeedSequence + Philox4x64-10 (numpy.random, bit_generator.pyx and   */
/* _philox.pyx, numpy 2.3.5), as called by routing.py:59-62                  */
/* ------------------------------------------------------------------------ */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}
/* SeedSequence(entropy words).generate_state(n32 words) with pool_size 4. */
static void seedseq_state(const uint32_t* ent, int n_ent, uint32_t* out, int n_out) {
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n_ent ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < n_ent; s++)
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < n_out; i++) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    out[i] = v;
  }
}
/* _int_to_uint32_array: little-endian 32-bit words, [0] for zero. */
static int int_words(uint64_t v, uint32_t* w) {
  if (v == 0) { w[0] = 0; return 1; }
  int n = 0;
  while (v) { w[n++] = (uint32_t)v; v >>= 32; }
  return n;
}
/* Philox key for route_tokens' _rng(seed): the SeedSequence state is passed
 * positionally, so Philox hashes it through a second SeedSequence. */
static void routing_key(uint64_t seed, uint64_t key[2]) {
  uint32_t ent[8], st[4];
  int n = int_words(seed, ent);
  n += int_words(0xE0u, ent + n);
  seedseq_state(ent, n, st, 4);
  uint64_t s0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  uint64_t s1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  n = int_words(s0, ent);
  n += int_words(s1, ent + n);
  seedseq_state(ent, n, st, 4);
  key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

static void philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * c0;
    unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------ */
/* numpy Generator distributions used by dirichlet_skew routing             */
/* (routing.py:99-106): rng.dirichlet(np.full(E, alpha)) then               */
/* rng.exponential(1.0, (T, E)). Restated from numpy 2.3.5                  */
/* (random/src/distributions/distributions.c: random_standard_exponential,  */
/* random_standard_normal, random_standard_gamma, random_beta; and          */
/* _generator.pyx Generator.dirichlet). The ziggurat tables are numpy's own  */
/* (fs_ziggurat.h, extracted from libnpyrandom.a); pow/log/exp/log1p are     */
/* glibc's, as in numpy's build, so the oracle is bit-exact by construction. */
/* ------------------------------------------------------------------------ */
#include "../paper_2508_03148_b200/csrc/fs_ziggurat.h"

typedef struct { uint64_t key[2]; uint64_t n; uint64_t blk[4]; } np_philox;

static uint64_t np_next_u64(np_philox* g) {
  if ((g->n & 3) == 0) {
    uint64_t ctr[4] = {g->n / 4 + 1, 0, 0, 0};
    philox4x64_10(ctr, g->key, g->blk);
  }
  return g->blk[g->n++ & 3];
}
static double np_next_double(np_philox* g) {
  return (double)(np_next_u64(g) >> 11) * (1.0 / 9007199254740992.0);
}
static double zig_d(uint64_t bits) { double d; memcpy(&d, &bits, 8); return d; }

static double np_std_exponential(np_philox* g) {
  for (;;) {
    uint64_t ri = np_next_u64(g) >> 3;
    uint8_t idx = (uint8_t)(ri & 0xFF);
    ri >>= 8;
    double x = (double)ri * zig_d(fs_zig_we[idx]);
    if (ri < fs_zig_ke[idx]) return x;
    if (idx == 0) return FS_ZIG_EXP_R - log1p(-np_next_double(g));
    if ((zig_d(fs_zig_fe[idx - 1]) - zig_d(fs_zig_fe[idx])) * np_next_double(g) +
            zig_d(fs_zig_fe[idx]) < exp(-x))
      return x;
  }
}
static double np_std_normal(np_philox* g) {
  for (;;) {
    uint64_t r = np_next_u64(g);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * zig_d(fs_zig_wi[idx]);
    if (sign & 0x1) x = -x;
    if (rabs < fs_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -FS_ZIG_NOR_INV_R * log1p(-np_next_double(g));
        double yy = -log1p(-np_next_double(g));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 0x1) ? -(FS_ZIG_NOR_R + xx) : FS_ZIG_NOR_R + xx;
      }
    } else {
      if (((zig_d(fs_zig_fi[idx - 1]) - zig_d(fs_zig_fi[idx])) * np_next_double(g) +
           zig_d(fs_zig_fi[idx])) < exp(-0.5 * x * x))
        return x;
    }
  }
}
static double np_std_gamma(np_philox* g, double shape) {
  if (shape == 1.0) return np_std_exponential(g);
  if (shape == 0.0) return 0.0;
  if (shape < 1.0) {
    for (;;) {
      double U = np_next_double(g);
      double V = np_std_exponential(g);
      if (U <= 1.0 - shape) {
        double X = pow(U, 1. / shape);
        if (X <= V) return X;
      } else {
        double Y = -log((1 - U) / shape);
        double X = pow(1.0 - shape + shape * Y, 1. / shape);
        if (X <= (V + Y)) return X;
      }
    }
  }
  double b = shape - 1. / 3.;
  double c = 1. / sqrt(9 * b);
  for (;;) {
    double X, V;
    do {
      X = np_std_normal(g);
      V = 1.0 + c * X;
    } while (V <= 0.0);
    V = V * V * V;
    double U = np_next_double(g);
    if (U < 1.0 - 0.0331 * (X * X) * (X * X)) return b * V;
    if (log(U) < 0.5 * X * X + b * (1. - V + log(V))) return b * V;
  }
}
static double np_beta(np_philox* g, double a, double b) {
  if (a <= 1.0 && b <= 1.0) {
    for (;;) { /* Johnk */
      double U = np_next_double(g), V = np_next_double(g);
      double X = pow(U, 1.0 / a), Y = pow(V, 1.0 / b);
      double XpY = X + Y;
      if (XpY <= 1.0 && U + V > 0.0) {
        if (XpY > 0) return X / XpY;
        double logX = log(U) / a, logY = log(V) / b;
        double logM = logX > logY ? logX : logY;
        logX -= logM;
        logY -= logM;
        return exp(logX - log(exp(logX) + exp(logY)));
      }
    }
  }
  double Ga = np_std_gamma(g, a), Gb = np_std_gamma(g, b);
  return Ga / (Ga + Gb);
}
/* Generator.dirichlet(np.full(E, alpha)) followed by np.maximum(., 1e-12). */
static void np_dirichlet_sym(np_philox* g, int E, double alpha, double* p) {
  if (alpha < 0.1) { /* stick-breaking with beta variates */
    double* csum = (double*)malloc(sizeof(double) * (size_t)E);
    double cs = 0.0;
    for (int j = E - 1; j >= 0; j--) { cs += alpha; csum[j] = cs; }
    double acc = 1.0;
    int j;
    for (j = 0; j < E; j++) p[j] = 0.0;
    for (j = 0; j < E - 1; j++) {
      double v = np_beta(g, alpha, csum[j + 1]);
      p[j] = acc * v;
      acc *= (1. - v);
      if (csum[j + 1] == 0) break;
    }
    p[E - 1] = acc;
    free(csum);
  } else {
    double acc = 0.;
    for (int j = 0; j < E; j++) { p[j] = np_std_gamma(g, alpha); acc = acc + p[j]; }
    double invacc = 1. / acc;
    for (int j = 0; j < E; j++) p[j] = p[j] * invacc;
  }
  for (int j = 0; j < E; j++) p[j] = p[j] > 1e-12 ? p[j] : 1e-12;
}

/* ------------------------------------------------------------------------ */
/* Python float helpers                                                     */
/* ------------------------------------------------------------------------ */
/* CPython 3.12 builtin sum() over a list of floats starting from int 0:
 * the first float is taken as-is (0 + x), the rest are Neumaier-compensated
 * (Python/bltinmodule.c builtin_sum_impl). */
typedef struct { double f, c; int n; } pysum_t;
static void pysum_init(pysum_t* s) { s->f = 0.0; s->c = 0.0; s->n = 0; }
static void pysum_add(pysum_t* s, double x) {
  if (s->n++ == 0) { s->f = x; return; }
  double t = s->f + x;
  if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
  else s->c += (x - t) + s->f;
  s->f = t;
}
static double pysum_result(const pysum_t* s) {
  if (s->n == 0) return 0.0; /* int 0: callers never divide an empty sum */
  double f = s->f;
  if (s->c != 0.0 && isfinite(s->c)) f += s->c;
  return f;
}
/* round(x) for a float: half-to-even, core.py:25-35 */
static int64_t py_round(double x) { return (int64_t)llrint(x); }
/* Python round(x, 6) for 0 <= x*1e6 < 2^52 (floatobject.c double_round): the exact
 * product x*1e6 = hi + lo decides the integer, ties to even; n / 1e6 is the double
 * nearest n * 10^-6. */
static double py_round6(double x) {
  double hi = x * 1e6;
  double lo = fma(x, 1e6, -hi);
  double n = rint(hi);
  double f = hi - n;
  double up = (f - 0.5) + lo, dn = (f + 0.5) + lo;
  int odd = fmod(n, 2.0) != 0.0;
  if (up > 0.0 || (up == 0.0 && odd)) n += 1.0;
  else if (dn < 0.0 || (dn == 0.0 && odd)) n -= 1.0;
  return n / 1e6;
}
double fso_round6(double x) { return py_round6(x); }
static double py_max(double a, double b) { return (b > a) ? b : a; }
static double py_min(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------------ */
/* Instance state                                                           */
/* ------------------------------------------------------------------------ */
enum {
  EV_ARRIVAL = 0, EV_BATCH_START, EV_BATCH_COMPLETE, EV_PREFILL_COMPLETE,
  EV_MEMORY_AVAILABLE, EV_KV_START, EV_KV_DONE, EV_ATTN_DONE, EV_A2F_DONE,
  EV_FFN_DONE, EV_F2A_DONE, EV_TOKEN_EMITTED, EV_REQUEST_COMPLETE
};

typedef struct { int64_t t, seq; int32_t kind, a; int64_t b; } Ev;

typedef struct { int32_t* v; int n, cap; } IVec;
static void iv_push(IVec* q, int32_t x) {
  if (q->n == q->cap) {
    q->cap = q->cap ? 2 * q->cap : 16;
    q->v = (int32_t*)realloc(q->v, sizeof(int32_t) * (size_t)q->cap);
  }
  q->v[q->n++] = x;
}
static void iv_free(IVec* q) { free(q->v); q->v = NULL; q->n = q->cap = 0; }

typedef struct {
  int64_t cap, used;
  int block;                 /* 0 = exact */
  int64_t* raw;              /* per request */
  int64_t* charged;
  uint8_t* has;
} Pool;

typedef struct {
  const fs_replica_desc* d;
  Pool pool;
  IVec queue, running;
  int busy, start_pending;
  int64_t steps;
  int64_t busy_ns;
} Rep;

typedef struct {
  int phase;                 /* 0 prefill, 1 decode, 2 af */
  int rep;
  IVec ids;
  int64_t duration_ns;
  int64_t pool_used;         /* pool.snapshot() at start (base.py:245) */
  int64_t af_step;
  double* moe;               /* per-layer raw ratios or NULL */
  int n_moe;
} Batch;

typedef struct Sim {
  const fs_instance_desc* d;
  const fs_seed_prefix* prefixes;
  const int64_t* trace_counts;
  const fs_forest_set* forests;
  int N, R;
  const int64_t* arrival;
  const int32_t* prompt;
  const int32_t* output;
  const int32_t* id_rank;
  /* event engine */
  Ev* heap; int hn, hcap;
  int64_t now, next_seq, processed;
  /* requests */
  int32_t* emitted;
  int64_t* first_ns;
  int64_t* done_ns;
  int32_t* done_rank;
  int32_t* prefill_home;
  int32_t* decode_home;
  int n_done;
  /* replicas */
  Rep* rep;
  int rr_next;
  IVec transfer_queue;
  /* batches */
  Batch* batches; int nb, bcap;
  /* af */
  int64_t af_counter;
  struct AfEngine* af;
  int64_t af_busy[4];
  int64_t* af_step_start; int64_t* af_step_dur; int64_t* af_step_attn; int n_af, af_cap;
  /* routing log */
  fs_log* log; int inst;
  int64_t routing_calls;
  int64_t routing_draws;
  int32_t log_moff, log_eoff;
  /* errors */
  jmp_buf jb;
  int status, detail;
} Sim;

static void fail(Sim* s, int status, int detail) {
  s->status = status;
  s->detail = detail;
  longjmp(s->jb, 1);
}

/* ---- heap (core.py:160-197) ---- */
static int ev_less(const Ev* a, const Ev* b) {
  return a->t < b->t || (a->t == b->t && a->seq < b->seq);
}
/* event-trace record of a scheduled event, stored at index seq (fs_event_rec) */
static void otrace(Sim* s, int64_t seq, int64_t t, int kind, int replica, int32_t a, int32_t b,
                   int32_t c, int64_t x) {
  fs_log* L = s->log;
  if (!L || !L->events) return;
  if (seq >= L->event_cap) { L->truncated[s->inst] = 1; return; }
  fs_event_rec* r = &L->events[L->event_base[s->inst] + seq];
  r->t = t; r->seq = seq; r->x = x; r->a = a; r->b = b; r->c = c;
  r->replica = (int16_t)replica; r->kind = (uint8_t)kind; r->pad = 0;
}
static int64_t schedule(Sim* s, int64_t t, int kind, int32_t a, int64_t b) {
  if (t < s->now) fail(s, FS_ERR_SCHEDULING_IN_PAST, kind);
  if (s->hn == s->hcap) {
    s->hcap = s->hcap ? 2 * s->hcap : 64;
    s->heap = (Ev*)realloc(s->heap, sizeof(Ev) * (size_t)s->hcap);
  }
  Ev e = {t, s->next_seq++, kind, a, b};
  int i = s->hn++;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!ev_less(&e, &s->heap[p])) break;
    s->heap[i] = s->heap[p];
    i = p;
  }
  s->heap[i] = e;
  return e.seq;
}
static Ev heap_pop(Sim* s) {
  Ev top = s->heap[0];
  Ev last = s->heap[--s->hn];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    const Ev* cur = (m == i) ? &last : &s->heap[m];
    if (l < s->hn && ev_less(&s->heap[l], cur)) { m = l; cur = &s->heap[l]; }
    if (r < s->hn && ev_less(&s->heap[r], cur)) { m = r; }
    if (m == i) break;
    s->heap[i] = s->heap[m];
    i = m;
  }
  if (s->hn > 0) s->heap[i] = last;
  return top;
}

/* ---- KvPool (cluster.py:36-93) ---- */
static int64_t pool_rounded(const Pool* p, int64_t tokens) {
  if (!p->block) return tokens;
  return (int64_t)ceil((double)tokens / (double)p->block) * p->block;
}
/* returns 0 on success, 1 on Backpressure */
static int pool_reserve(Pool* p, int r, int64_t tokens) {
  if (tokens == 0) return 0;
  int64_t raw = (p->has[r] ? p->raw[r] : 0) + tokens;
  int64_t charge = pool_rounded(p, raw) - (p->has[r] ? p->charged[r] : 0);
  if (charge > p->cap - p->used) return 1;
  p->raw[r] = raw;
  p->charged[r] = (p->has[r] ? p->charged[r] : 0) + charge;
  p->has[r] = 1;
  p->used += charge;
  return 0;
}
static int64_t pool_release(Sim* s, Pool* p, int r) {
  if (!p->has[r]) fail(s, FS_ERR_INTERNAL, r); /* UnknownAllocation */
  int64_t freed = p->charged[r];
  p->has[r] = 0;
  p->used -= freed;
  return freed;
}

/* ------------------------------------------------------------------------ */
/* Cost model (costmodel/analytic.py, topology.py:360-394, cluster.py)       */
/* ------------------------------------------------------------------------ */
static double roofline_us(double flops, double nbytes, const fs_cost_ctx* h) {
  double sec = py_max(flops / h->peak_flops, nbytes / h->mem_bw);
  return h->kernel_overhead_us + sec * 1e6;
}
static double linear_us(int64_t m, int64_t n, int64_t k, const fs_cost_ctx* h, int dt) {
  double flops = 2.0 * (double)m;
  flops = flops * (double)n;
  flops = flops * (double)k;
  int64_t nbytes = (int64_t)dt * (m * n + n * k + m * k);
  return roofline_us(flops, (double)nbytes, h);
}
/* collective_time with an integer bytes_per_rank (int*int then int/int true div) */
static double collective_int(int kind, int64_t bpr, int n, double lat, double bw) {
  if (n == 1) return 0.0;
  double wire = (double)(bpr * (int64_t)(n - 1)) / (double)n;
  wire = wire / bw;
  if (kind == 1) return 2.0 * lat + 2.0 * wire; /* all_reduce */
  return lat + wire;                             /* all_to_all, all_gather */
}
/* collective_time with a float bytes_per_rank */
static double collective_flt(int kind, double bpr, int n, double lat, double bw) {
  if (n == 1) return 0.0;
  double wire = bpr * (double)(n - 1);
  wire = wire / (double)n;
  wire = wire / bw;
  if (kind == 1) return 2.0 * lat + 2.0 * wire;
  return lat + wire;
}
/* analytic.attention_us over one batch */
static double attention_us_analytic(int decode, const int64_t* q, const int64_t* kv, int B,
                                    int hq, int hkv, int hdim, const fs_cost_ctx* h, int dt) {
  int64_t hd = (int64_t)hq * hdim;
  int64_t skv = 0, sq = 0;
  for (int i = 0; i < B; i++) { skv += kv[i]; sq += q[i]; }
  double flops;
  if (decode) {
    flops = 4.0 * (double)skv;
    flops = flops * (double)hd;
  } else {
    double total = 0.0;
    for (int i = 0; i < B; i++) {
      double per = 4.0 * (double)q[i];
      per = per * (double)kv[i];
      per = per * (double)hd;
      if (kv[i] == q[i]) per = per / 2.0;
      total = total + per;
    }
    flops = total;
  }
  double kvb = 2.0 * (double)skv;
  kvb = kvb * (double)hkv;
  kvb = kvb * (double)hdim;
  kvb = kvb * (double)dt;
  double qob = 2.0 * (double)sq;
  qob = qob * (double)hq;
  qob = qob * (double)hdim;
  qob = qob * (double)dt;
  return roofline_us(flops, kvb + qob, h);
}
/* analytic.grouped_gemm_us; counts of one rank */
static double grouped_gemm_us(Sim* s, const int64_t* counts, int n, int64_t d_model, int64_t d_ff,
                              int nm, const fs_cost_ctx* h, int dt) {
  int64_t routed = 0, active = 0;
  for (int i = 0; i < n; i++) { routed += counts[i]; active += counts[i] > 0; }
  if (routed < 1) fail(s, FS_ERR_EMPTY_BATCH, 0);
  double flops = 2.0 * (double)nm;
  flops = flops * (double)routed;
  flops = flops * (double)d_model;
  flops = flops * (double)d_ff;
  int64_t wb = active * nm * d_model * d_ff * dt;
  int64_t ab = routed * nm * (d_model + d_ff) * dt;
  return roofline_us(flops, (double)(wb + ab), h);
}

/* ---- learned attention model (features.py:23-32,101-115; forest.py:67-78,234-239;
 *      model.py:126-133) ---- */
/* numpy's pairwise summation of a contiguous float64 array (DOUBLE_pairwise_sum):
 * plain loop below 8 elements, 8 accumulators up to 128, recursive halving above */
static double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}
/* _stats(values): sum, sum_sq, max, min, mean, std (ddof 0) */
static void np_stats(const int64_t* v, int n, double out[6]) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n);
  double* sq = (double*)malloc(sizeof(double) * (size_t)n);
  double mx = (double)v[0], mn = (double)v[0];
  for (int i = 0; i < n; i++) {
    a[i] = (double)v[i];
    sq[i] = a[i] * a[i];
    if (a[i] > mx) mx = a[i];
    if (a[i] < mn) mn = a[i];
  }
  double sum = np_pairwise(a, n);
  double mean = sum / (double)n;
  for (int i = 0; i < n; i++) { double x = a[i] - mean; sq[i] = x * x; }
  double var = np_pairwise(sq, n) / (double)n;
  for (int i = 0; i < n; i++) sq[i] = a[i] * a[i];
  out[0] = sum;
  out[1] = np_pairwise(sq, n);
  out[2] = mx;
  out[3] = mn;
  out[4] = mean;
  out[5] = sqrt(var);
  free(a);
  free(sq);
}
/* AttentionFeatures.vector() */
static void attention_features(int decode, const int64_t* q, const int64_t* kv, int B, int hq,
                               int hkv, int hdim, double x[17]) {
  x[0] = decode ? 1.0 : 0.0;
  x[1] = (double)B;
  np_stats(q, B, x + 2);
  np_stats(kv, B, x + 8);
  x[14] = (double)hq;
  x[15] = (double)hkv;
  x[16] = (double)hdim;
}
static int cmp_dbl(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
/* np.maximum(np.sort(per_tree).mean(), 1e-6) */
static double forest_predict(const fs_forest_set* fs, int forest, const double* x) {
  const fs_forest_desc* f = &fs->forests[forest];
  double* vals = (double*)malloc(sizeof(double) * (size_t)f->n_trees);
  for (int t = 0; t < f->n_trees; t++) {
    int64_t node = fs->tree_root[f->tree_offset + t];
    while (fs->feature[node] >= 0)
      node = (x[fs->feature[node]] <= fs->threshold[node]) ? fs->left[node] : fs->right[node];
    vals[t] = fs->value[node];
  }
  qsort(vals, (size_t)f->n_trees, sizeof(double), cmp_dbl);
  double mean = np_pairwise(vals, f->n_trees) / (double)f->n_trees;
  free(vals);
  return mean < 1e-6 ? 1e-6 : mean;
}

/* The random part of route_tokens (routing.py:96-113) for T > 0, k < E:
 * keys per row from rng.random (uniform) or Exp(1)/popularity (dirichlet_skew),
 * the k smallest per row (np.argpartition(keys, k-1)[:, :k]) and their tally.
 * An exact key tie at the selection boundary makes argpartition's pick
 * implementation-defined: reported as FS_ERR_ROUTING_TIE. Returns a status. */
static int route_core(int64_t T, int E, int k, int policy, double alpha, uint64_t seed,
                      int64_t* counts) {
  if (policy == FS_ROUTE_DIRICHLET && !(alpha > 0)) return FS_ERR_ROUTING;
  if (policy != FS_ROUTE_UNIFORM && policy != FS_ROUTE_DIRICHLET) return FS_ERR_ROUTING;
  np_philox g;
  memset(&g, 0, sizeof g);
  routing_key(seed, g.key);
  double* pop = NULL;
  if (policy == FS_ROUTE_DIRICHLET) {
    pop = (double*)malloc(sizeof(double) * (size_t)E);
    np_dirichlet_sym(&g, E, alpha, pop);
  }
  /* keys as order-preserving u64: rng.random() keys are (u >> 11) (the common
   * 2^-53 scale does not change the order); dirichlet keys are positive
   * doubles, ordered like their IEEE bit patterns */
  uint64_t* row = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)E);
  int st = 0;
  for (int64_t t = 0; t < T && !st; t++) {
    for (int e = 0; e < E; e++) {
      if (pop) {
        double key = np_std_exponential(&g) / pop[e];
        memcpy(&row[e], &key, 8);
      } else {
        row[e] = np_next_u64(&g) >> 11;
      }
    }
    for (int j = 0; j < k; j++) {
      int best = -1;
      for (int e = 0; e < E; e++)
        if (row[e] != UINT64_MAX && (best < 0 || row[e] < row[best])) best = e;
      if (j == k - 1) {
        for (int e = 0; e < E; e++)
          if (e != best && row[e] == row[best]) st = FS_ERR_ROUTING_TIE;
      }
      counts[best]++;
      row[best] = UINT64_MAX;
    }
  }
  free(row);
  free(pop);
  return st;
}

/* ---- route_tokens (routing.py:65-113) ---- */
static int64_t* route(Sim* s, int64_t T, uint32_t seed, int policy_uniform_forced,
                      int rep, int mb, int64_t step, int layer) {
  const fs_instance_desc* d = s->d;
  int E = d->num_experts, k = d->top_k;
  int64_t* counts = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  int policy = policy_uniform_forced ? FS_ROUTE_UNIFORM : d->routing_policy;
  if (!(1 <= k && k <= E)) { free(counts); fail(s, FS_ERR_INVALID_TOPK, 0); }
  if (T < 0) { free(counts); fail(s, FS_ERR_ROUTING, 0); }
  if (policy == FS_ROUTE_TRACE) {
    if (d->n_trace_counts == 0 || d->n_trace_counts != E) { free(counts); fail(s, FS_ERR_ROUTING, 1); }
    int64_t sum = 0;
    for (int e = 0; e < E; e++) {
      int64_t c = s->trace_counts[d->trace_offset + e];
      if (c < 0) { free(counts); fail(s, FS_ERR_ROUTING, 2); }
      counts[e] = c;
      sum += c;
    }
    if (sum != T * k) { free(counts); fail(s, FS_ERR_ROUTING, 3); }
  } else if (T == 0) {
    /* zeros */
  } else if (k == E) {
    for (int e = 0; e < E; e++) counts[e] = T;
  } else {
    int st = route_core(T, E, k, policy, d->routing_alpha, (uint64_t)seed, counts);
    if (st) { free(counts); fail(s, st, 0); }
    s->routing_draws += T * E;
  }
  s->routing_calls++;
  fs_log* lg = s->log;
  if (lg && lg->routes) {
    int32_t c = lg->route_count[s->inst];
    int64_t cbase = (int64_t)c * E;
    if (c < lg->route_cap && cbase + E <= lg->counts_cap) {
      fs_route_rec* r = &lg->routes[lg->route_base[s->inst] + c];
      r->replica = rep; r->micro_batch = mb; r->step = step; r->layer = layer;
      r->tokens = (int32_t)T; r->counts_offset = (int32_t)cbase; r->n_experts = E;
      for (int e = 0; e < E; e++) lg->counts[lg->counts_base[s->inst] + cbase + e] = (int32_t)counts[e];
      lg->route_count[s->inst] = c + 1;
    } else {
      lg->truncated[s->inst] = 1;
    }
  }
  return counts;
}

/* GroupedGemmFeatures(total, counts, d_model, d_ff, top_k, "local").vector()
 * (features.py:126-209) for one EP rank's expert loads: numpy mean / std
 * (pairwise sums, _var's (x - mean)^2), active-expert mean, normalised entropy
 * -(p * log p).sum() / log(n). log is glibc's here; numpy's np.log may use its
 * own SIMD kernel (SVML on AVX-512 hosts), which can differ in the last bit --
 * the features only feed `x[f] <= threshold` comparisons. */
static void gg_local_features(const int64_t* counts, int n, int64_t d_model, int64_t d_ff,
                              int top_k, double x[12]) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t total = 0, nact = 0, mx = counts[0];
  for (int i = 0; i < n; i++) {
    a[i] = (double)counts[i];
    total += counts[i];
    nact += counts[i] > 0;
    if (counts[i] > mx) mx = counts[i];
  }
  const double sum = np_pairwise(a, n);           /* exact: integer values */
  const double mean = sum / (double)n;
  for (int i = 0; i < n; i++) { double dv = a[i] - mean; w[i] = dv * dv; }
  const double std = sqrt(np_pairwise(w, n) / (double)n);
  const double sel = (double)nact / (double)n;
  double mom = 0.0;
  if (nact) {
    int j = 0;
    for (int i = 0; i < n; i++) if (counts[i] > 0) w[j++] = a[i];
    const double amean = np_pairwise(w, nact) / (double)nact;
    mom = (double)mx / amean;
  }
  const double cv = mean > 0 ? std / mean : 0.0;
  double ent;
  if (n == 1) {
    ent = 1.0;
  } else if (sum > 0) {
    int j = 0;
    for (int i = 0; i < n; i++) {
      if (counts[i] > 0) { double pr = a[i] / sum; w[j++] = pr * log(pr); }
    }
    ent = -np_pairwise(w, nact) / log((double)n);
  } else {
    ent = 0.0;
  }
  x[0] = (double)total; x[1] = (double)n; x[2] = (double)d_model; x[3] = (double)d_ff;
  x[4] = (double)top_k; x[5] = sel; x[6] = mom; x[7] = cv; x[8] = ent;
  x[9] = (double)mx; x[10] = mean; x[11] = std;
  free(a);
  free(w);
}

/* moe_layer_latency (moe.py:69-128); returns total; *ratio gets the
 * moe_imbalance raw value (base.py:247-252) */
static double moe_layer(Sim* s, const int64_t* counts, int64_t T, const fs_cost_ctx* c,
                        int ep, int moe_tp, double* ratio) {
  const fs_instance_desc* d = s->d;
  int E = d->num_experts;
  if (ep < 1 || moe_tp < 1) fail(s, FS_ERR_TOPOLOGY_MISMATCH, 0);
  if (E % ep != 0) fail(s, FS_ERR_TOPOLOGY_MISMATCH, 1);
  if (d->expert_d_ff % moe_tp != 0) fail(s, FS_ERR_TOPOLOGY_MISMATCH, 2);
  if (T < 1) fail(s, FS_ERR_EMPTY_BATCH, 0);
  double gate = linear_us(T, E, d->d_model, c, d->dtype_bytes);
  int64_t routed_bytes = T * d->top_k * (int64_t)d->d_model * d->dtype_bytes;
  double bpr = (double)routed_bytes / (double)ep;
  double dispatch = collective_flt(0, bpr, ep, d->intra_latency_s, d->intra_bandwidth_bps) * 1e6;
  double combine = dispatch;
  int per = E / ep;
  int64_t dffs = d->expert_d_ff / moe_tp;
  double expert = 0.0;
  pysum_t ps;
  pysum_init(&ps);
  for (int r = 0; r < ep; r++) {
    int64_t local = 0;
    for (int e = 0; e < per; e++) local += counts[r * per + e];
    double v = 0.0;
    if (local != 0) {
      if (d->gg_forest != -1) {
        /* CostModel.predict_grouped_gemm with a learned model (model.py:323-326) */
        if (d->gg_forest < 0) fail(s, FS_ERR_SCHEMA, 0);
        if (!s->forests || d->gg_forest >= s->forests->n_forests) fail(s, FS_ERR_INTERNAL, 7);
        if (dffs < 1 || d->top_k < 1) fail(s, FS_ERR_VALUE, 3);
        double x[12];
        gg_local_features(counts + r * per, per, d->d_model, dffs, d->top_k, x);
        v = forest_predict(s->forests, d->gg_forest, x);
      } else {
        v = grouped_gemm_us(s, counts + r * per, per, d->d_model, dffs, d->ffn_matrices, c, d->dtype_bytes);
      }
    }
    if (r == 0 || v > expert) expert = v; /* max(): first maximum */
    pysum_add(&ps, v);
  }
  double total = gate + dispatch;
  total = total + expert;
  total = total + combine;
  double sum_pr = pysum_result(&ps);
  if (sum_pr > 0) *ratio = expert / (sum_pr / (double)ep);
  else *ratio = 1.0;
  return total;
}

typedef struct {
  int phase;             /* 0 prefill 1 decode */
  int n;
  const int32_t* ids;    /* request indices */
} Plan;

/* context length of a member */
static void plan_lengths(Sim* s, const Plan* p, int64_t* q, int64_t* kv) {
  for (int i = 0; i < p->n; i++) {
    int r = p->ids[i];
    if (p->phase == 0) { q[i] = s->prompt[r]; kv[i] = s->prompt[r]; }
    else { q[i] = 1; kv[i] = (int64_t)s->prompt[r] + s->emitted[r]; }
  }
}

static void heads(const fs_instance_desc* d, int tp, int* hq, int* hkv) {
  *hq = d->num_query_heads / tp; if (*hq < 1) *hq = 1;
  *hkv = d->num_kv_heads / tp; if (*hkv < 1) *hkv = 1;
}
static double qkv_us(const fs_instance_desc* d, const fs_cost_ctx* c, int64_t n) {
  int hq, hkv; heads(d, c->tp, &hq, &hkv);
  return linear_us(n, (int64_t)(hq + 2 * hkv) * d->head_dim, d->d_model, c, d->dtype_bytes);
}
static double out_us(const fs_instance_desc* d, const fs_cost_ctx* c, int64_t n) {
  int hq, hkv; heads(d, c->tp, &hq, &hkv);
  return linear_us(n, d->d_model, (int64_t)hq * d->head_dim, c, d->dtype_bytes);
}
static double tpcoll_us(const fs_instance_desc* d, const fs_cost_ctx* c, int64_t n) {
  int64_t b = n * d->d_model * (int64_t)d->dtype_bytes;
  return collective_int(1, b, c->tp, d->intra_latency_s, d->intra_bandwidth_bps) * 1e6;
}
static double attn_us(Sim* s, const fs_cost_ctx* c, const Plan* p) {
  const fs_instance_desc* d = s->d;
  int hq, hkv; heads(d, c->tp, &hq, &hkv);
  int64_t* q = (int64_t*)malloc(sizeof(int64_t) * (size_t)p->n * 2);
  int64_t* kv = q + p->n;
  plan_lengths(s, p, q, kv);
  double v;
  if (d->attn_forest != -1) {
    /* CostModel.predict_attention raises SchemaMismatch for a non-attention_v1
     * model at its first prediction (costmodel/model.py:313-320) */
    if (d->attn_forest < 0) { free(q); fail(s, FS_ERR_SCHEMA, 0); }
    if (!s->forests || d->attn_forest >= s->forests->n_forests) { free(q); fail(s, FS_ERR_INTERNAL, 7); }
    double x[17];
    attention_features(p->phase == 1, q, kv, p->n, hq, hkv, d->head_dim, x);
    v = forest_predict(s->forests, d->attn_forest, x);
  } else {
    v = attention_us_analytic(p->phase == 1, q, kv, p->n, hq, hkv, d->head_dim, c, d->dtype_bytes);
  }
  free(q);
  return v;
}
static double dense_ffn_us(Sim* s, const fs_cost_ctx* c, int64_t n) {
  const fs_instance_desc* d = s->d;
  int64_t dff = d->d_ff / c->tp; if (dff < 1) dff = 1;
  if (d->gg_forest != -1) {
    /* OperatorCosts.ffn_us for a dense model (cluster.py:286-296) with a learned
     * grouped-GEMM model: GroupedGemmFeatures(n, (n,), d_model, dff, 1, "local")
     * .vector() (features.py:166-209) -- one expert holding every token */
    if (d->gg_forest < 0) fail(s, FS_ERR_SCHEMA, 0);  /* check_schema, model.py:325 */
    if (!s->forests || d->gg_forest >= s->forests->n_forests) fail(s, FS_ERR_INTERNAL, 7);
    if (n < 1) fail(s, FS_ERR_EMPTY_BATCH, 2);
    const double cn = (double)n;
    const double active_mean = cn / 1.0, mean = cn / 1.0;
    const double dev = cn - mean;
    const double std = sqrt((dev * dev) / 1.0);
    double x[12] = {cn, 1.0, (double)d->d_model, (double)dff, 1.0,
                    1.0 / 1.0,            /* expert_selection_ratio */
                    cn / active_mean,     /* load_max_over_mean */
                    std / mean,           /* load_cv (mean > 0) */
                    1.0,                  /* load_entropy: single expert */
                    cn, mean, std};
    return forest_predict(s->forests, d->gg_forest, x);
  }
  int64_t counts[1] = {n};
  return grouped_gemm_us(s, counts, 1, d->d_model, dff, d->ffn_matrices, c, d->dtype_bytes);
}

/* execute_batch (cluster.py:317-346) for a replica-scope router; returns the
 * duration in us and fills the per-layer moe ratios (when MoE). */
static double execute_batch(Sim* s, int ri, const Plan* p, double* moe_ratio) {
  const fs_instance_desc* d = s->d;
  Rep* R = &s->rep[ri];
  const fs_cost_ctx* c = &R->d->cost;
  int64_t n = 0;
  for (int i = 0; i < p->n; i++) n += (p->phase == 0) ? s->prompt[p->ids[i]] : 1;
  pysum_t ls;
  pysum_init(&ls);
  for (int layer = 0; layer < d->num_layers; layer++) {
    double ffn;
    if (!d->has_moe) {
      ffn = dense_ffn_us(s, c, n);
    } else {
      uint32_t seed = router_seed(&s->prefixes[R->d->prefix], 0, R->steps, layer);
      int64_t* counts = route(s, n, seed, 0, ri, 0, R->steps, layer);
      double ratio;
      ffn = moe_layer(s, counts, n, c, c->ep, c->moe_tp, &ratio);
      free(counts);
      moe_ratio[layer] = ratio;
    }
    double qkv = qkv_us(d, c, n);
    double att = attn_us(s, c, p);
    double out = out_us(d, c, n);
    double coll = tpcoll_us(d, c, n);
    double coll2 = tpcoll_us(d, c, n);
    double tot = qkv + att;
    tot = tot + out;
    tot = tot + coll;
    tot = tot + ffn;
    tot = tot + coll2;
    pysum_add(&ls, tot);
  }
  double pp_tr = 0.0;
  {
    int64_t b = n * d->d_model * (int64_t)d->dtype_bytes;
    double tt = d->intra_latency_s + (double)b / d->intra_bandwidth_bps;
    pp_tr = (double)(c->pp - 1) * (tt * 1e6);
  }
  return pysum_result(&ls) + pp_tr;
}

/* ------------------------------------------------------------------------ */
/* Serving workflows                                                        */
/* ------------------------------------------------------------------------ */
static int batch_new(Sim* s, int phase, int rep, const int32_t* ids, int n) {
  if (s->nb == s->bcap) {
    s->bcap = s->bcap ? 2 * s->bcap : 256;
    s->batches = (Batch*)realloc(s->batches, sizeof(Batch) * (size_t)s->bcap);
  }
  Batch* b = &s->batches[s->nb];
  memset(b, 0, sizeof *b);
  b->phase = phase;
  b->rep = rep;
  for (int i = 0; i < n; i++) iv_push(&b->ids, ids[i]);
  return s->nb++;
}

static void kick(Sim* s, int ri) {
  Rep* R = &s->rep[ri];
  if (R->busy || R->start_pending) return;
  if (R->queue.n == 0 && R->running.n == 0) return;
  R->start_pending = 1;
  int64_t sq = schedule(s, s->now, EV_BATCH_START, ri, 0);
  otrace(s, sq, s->now, EV_BATCH_START, ri, 0, 0, 0, 0);
}

/* batch record (fs_batch_rec) written when the batch's BATCH_COMPLETE is scheduled */
static void olog_batch(Sim* s, int bi, int64_t t_complete, int64_t seq, int64_t af_step) {
  fs_log* log = s->log;
  Batch* b = &s->batches[bi];
  if (log && log->events) otrace(s, seq, t_complete, EV_BATCH_COMPLETE, b->rep, bi, 0, 0, 0);
  if (!log || !log->batches) return;
  int inst = s->inst;
  int32_t c = log->batch_count[inst];
  if (c < log->batch_cap && s->log_moff + b->ids.n <= log->member_cap &&
      s->log_eoff + b->n_moe <= log->moe_cap) {
    fs_batch_rec* br = &log->batches[log->batch_base[inst] + c];
    br->replica = b->rep; br->phase = b->phase; br->t_complete = t_complete;
    br->duration_ns = b->duration_ns; br->n_members = b->ids.n;
    br->member_offset = s->log_moff;
    br->seq = seq; br->pool_used = b->pool_used; br->af_step = af_step;
    for (int q = 0; q < b->ids.n; q++)
      log->members[log->member_base[inst] + s->log_moff + q] = b->ids.v[q];
    s->log_moff += b->ids.n;
    if (b->n_moe) {
      br->moe_offset = s->log_eoff; br->n_moe = b->n_moe;
      for (int q = 0; q < b->n_moe; q++)
        log->moe_ratio[log->moe_base[inst] + s->log_eoff + q] = py_round6(b->moe[q]);
      s->log_eoff += b->n_moe;
    } else { br->moe_offset = -1; br->n_moe = 0; }
    log->batch_count[inst] = c + 1;
  } else log->truncated[inst] = 1;
}

static void start_batch(Sim* s, int ri, int phase, const int32_t* ids, int n) {
  Rep* R = &s->rep[ri];
  const fs_instance_desc* d = s->d;
  Plan p = {phase, n, ids};
  double* moe = d->has_moe ? (double*)malloc(sizeof(double) * (size_t)d->num_layers) : NULL;
  double us = execute_batch(s, ri, &p, moe);
  int64_t dur = py_round(us * 1000.0);
  R->busy = 1;
  R->steps++;
  int bi = batch_new(s, phase, ri, ids, n);
  s->batches[bi].duration_ns = dur;
  s->batches[bi].moe = moe;
  s->batches[bi].n_moe = moe ? d->num_layers : 0;
  s->batches[bi].pool_used = R->pool.used;
  int64_t sq = schedule(s, s->now + dur, EV_BATCH_COMPLETE, ri, bi);
  olog_batch(s, bi, s->now + dur, sq, -1);
}

static void complete_request(Sim* s, int ri, int r) {
  s->done_ns[r] = s->now;
  s->done_rank[r] = s->n_done++;
  int64_t sq = schedule(s, s->now, EV_REQUEST_COMPLETE, ri, r);
  otrace(s, sq, s->now, EV_REQUEST_COMPLETE, ri, r, 0, 0, 0);
  Pool* pl = &s->rep[ri].pool;
  int64_t freed = pool_release(s, pl, r);
  sq = schedule(s, s->now, EV_MEMORY_AVAILABLE, ri, r);
  otrace(s, sq, s->now, EV_MEMORY_AVAILABLE, ri, r, (int32_t)freed, 0, pl->cap - pl->used);
}

/* build_prefill_batch (cluster.py:145-183); out ids in candidate order */
static int cand_less(Sim* s, int a, int b) {
  const fs_instance_desc* d = s->d;
  if (d->priority_key == FS_PRIO_PROMPT) {
    if (s->prompt[a] != s->prompt[b]) return s->prompt[a] < s->prompt[b];
  }
  if (s->arrival[a] != s->arrival[b]) return s->arrival[a] < s->arrival[b];
  return s->id_rank[a] < s->id_rank[b];
}
static int build_prefill(Sim* s, int ri, int running_count, int full, int32_t* out) {
  const fs_instance_desc* d = s->d;
  Rep* R = &s->rep[ri];
  int n = R->queue.n;
  int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  memcpy(cand, R->queue.v, sizeof(int32_t) * (size_t)n);
  if (d->admission == FS_ADMIT_PRIORITY) { /* stable insertion sort */
    for (int i = 1; i < n; i++) {
      int32_t x = cand[i];
      int j = i - 1;
      while (j >= 0 && cand_less(s, x, cand[j])) { cand[j + 1] = cand[j]; j--; }
      cand[j + 1] = x;
    }
  }
  int m = 0;
  int64_t seats = (int64_t)d->max_num_seqs - running_count;
  int64_t tokens = 0;
  int64_t headroom = R->pool.cap - R->pool.used;
  for (int i = 0; i < n; i++) {
    int r = cand[i];
    int64_t fp = full ? (int64_t)s->prompt[r] + s->output[r] : s->prompt[r];
    int fits = m < seats && tokens + s->prompt[r] <= d->max_batch_tokens &&
               pool_rounded(&R->pool, fp) <= headroom;
    if (fits) {
      out[m++] = r;
      tokens += s->prompt[r];
      headroom -= pool_rounded(&R->pool, fp);
    } else if (d->admission != FS_ADMIT_FCFS_SKIP) {
      break;
    }
  }
  free(cand);
  return m;
}
static void queue_remove_set(IVec* q, const int32_t* ids, int n) {
  int w = 0;
  for (int i = 0; i < q->n; i++) {
    int keep = 1;
    for (int j = 0; j < n; j++) if (ids[j] == q->v[i]) { keep = 0; break; }
    if (keep) q->v[w++] = q->v[i];
  }
  q->n = w;
}
static void running_remove(IVec* q, int r) {
  for (int i = 0; i < q->n; i++)
    if (q->v[i] == r) {
      memmove(q->v + i, q->v + i + 1, sizeof(int32_t) * (size_t)(q->n - i - 1));
      q->n--;
      return;
    }
}

/* ---- co-located + AF prefill: admission with full footprint ---- */
static int admit_full(Sim* s, int ri) {
  Rep* R = &s->rep[ri];
  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R->queue.n ? R->queue.n : 1));
  int m = build_prefill(s, ri, R->running.n, 1, ids);
  if (m) {
    for (int i = 0; i < m; i++) {
      int r = ids[i];
      if (pool_reserve(&R->pool, r, (int64_t)s->prompt[r] + s->output[r])) fail(s, FS_ERR_INTERNAL, 1);
    }
    queue_remove_set(&R->queue, ids, m);
    start_batch(s, ri, 0, ids, m);
  }
  free(ids);
  return m;
}

static void prefill_complete(Sim* s, int ri, const Batch* b, int to_running) {
  Rep* R = &s->rep[ri];
  for (int i = 0; i < b->ids.n; i++) {
    int r = b->ids.v[i];
    s->emitted[r] += 1;
    int64_t sq = schedule(s, s->now, EV_PREFILL_COMPLETE, ri, r);
    otrace(s, sq, s->now, EV_PREFILL_COMPLETE, ri, r, 0, 0, 0);
  }
  if (b->ids.n) {
    int64_t sq = schedule(s, s->now, EV_TOKEN_EMITTED, ri, -1);
    otrace(s, sq, s->now, EV_TOKEN_EMITTED, ri, 0, 0, 0, 0);
    for (int i = 0; i < b->ids.n; i++)
      if (s->first_ns[b->ids.v[i]] < 0) s->first_ns[b->ids.v[i]] = s->now;
  }
  for (int i = 0; i < b->ids.n; i++) {
    int r = b->ids.v[i];
    if (s->emitted[r] == s->output[r]) complete_request(s, ri, r);
    else if (to_running) iv_push(&R->running, r);
    else iv_push(&s->transfer_queue, r);
  }
}
static int decode_complete(Sim* s, int ri, const Batch* b) {
  Rep* R = &s->rep[ri];
  int64_t sq = schedule(s, s->now, EV_TOKEN_EMITTED, ri, -1);
  otrace(s, sq, s->now, EV_TOKEN_EMITTED, ri, 0, 0, 0, 0);
  for (int i = 0; i < b->ids.n; i++)
    if (s->first_ns[b->ids.v[i]] < 0) s->first_ns[b->ids.v[i]] = s->now;
  int nf = 0;
  int32_t* fin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(b->ids.n > 0 ? b->ids.n : 1) + 4);
  for (int i = 0; i < b->ids.n; i++) {
    int r = b->ids.v[i];
    s->emitted[r] += 1;
    if (s->emitted[r] > s->output[r]) fail(s, FS_ERR_INTERNAL, 2);
    if (s->emitted[r] == s->output[r]) fin[nf++] = r;
  }
  for (int i = 0; i < nf; i++) {
    running_remove(&R->running, fin[i]);
    complete_request(s, ri, fin[i]);
  }
  free(fin);
  return nf;
}

/* ---- colocated.py ---- */
static void co_on_arrival(Sim* s, int r) {
  int ri = s->rr_next % s->R;
  s->rr_next++;
  iv_push(&s->rep[ri].queue, r);
  kick(s, ri);
}
static void co_on_batch_start(Sim* s, int ri) {
  Rep* R = &s->rep[ri];
  R->start_pending = 0;
  if (R->busy) return;
  if (admit_full(s, ri)) return;
  if (R->running.n) {
    int n = R->running.n < s->d->max_num_seqs ? R->running.n : s->d->max_num_seqs;
    start_batch(s, ri, 1, R->running.v, n);
    return;
  }
  if (R->queue.n) fail(s, FS_ERR_REQUEST_CANNOT_FIT, R->queue.v[0]);
}
static void co_on_batch_complete(Sim* s, int ri, int bi) {
  Rep* R = &s->rep[ri];
  R->busy = 0;
  Batch* b = &s->batches[bi];
  if (b->phase == 0) prefill_complete(s, ri, b, 1);
  else decode_complete(s, ri, b);
  kick(s, ri);
}

/* ---- pd.py ---- */
static void pd_pump(Sim* s);
static void pd_on_arrival(Sim* s, int r) {
  int best = -1;
  int64_t best_out = 0;
  for (int ri = 0; ri < s->R; ri++) {
    Rep* R = &s->rep[ri];
    if (R->d->role != FS_ROLE_PREFILL) continue;
    int64_t out = 0;
    for (int i = 0; i < R->queue.n; i++) out += s->prompt[R->queue.v[i]];
    if (best < 0 || out < best_out || (out == best_out && R->d->key_rank < s->rep[best].d->key_rank)) {
      best = ri;
      best_out = out;
    }
  }
  s->prefill_home[r] = best;
  iv_push(&s->rep[best].queue, r);
  kick(s, best);
}
static void pd_on_batch_start(Sim* s, int ri) {
  Rep* R = &s->rep[ri];
  R->start_pending = 0;
  if (R->busy) return;
  if (R->d->role == FS_ROLE_PREFILL) {
    int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R->queue.n ? R->queue.n : 1));
    int m = build_prefill(s, ri, 0, 0, ids);
    if (m == 0) {
      if (R->queue.n && R->pool.used == 0) { int h = R->queue.v[0]; free(ids); fail(s, FS_ERR_REQUEST_CANNOT_FIT, h); }
      free(ids);
      return;
    }
    for (int i = 0; i < m; i++)
      if (pool_reserve(&R->pool, ids[i], s->prompt[ids[i]])) fail(s, FS_ERR_INTERNAL, 3);
    queue_remove_set(&R->queue, ids, m);
    start_batch(s, ri, 0, ids, m);
    free(ids);
  } else {
    while (R->queue.n && R->running.n < s->d->max_num_seqs) {
      int r = R->queue.v[0];
      memmove(R->queue.v, R->queue.v + 1, sizeof(int32_t) * (size_t)(R->queue.n - 1));
      R->queue.n--;
      iv_push(&R->running, r);
    }
    if (!R->running.n) return;
    int n = R->running.n < s->d->max_num_seqs ? R->running.n : s->d->max_num_seqs;
    start_batch(s, ri, 1, R->running.v, n);
  }
}
static void pd_on_batch_complete(Sim* s, int ri, int bi) {
  Rep* R = &s->rep[ri];
  R->busy = 0;
  Batch* b = &s->batches[bi];
  if (b->phase == 0) {
    prefill_complete(s, ri, b, 0);
    pd_pump(s);
  } else {
    if (decode_complete(s, ri, b)) pd_pump(s);
  }
  kick(s, ri);
}
static void pd_pump(Sim* s) {
  const fs_instance_desc* d = s->d;
  while (s->transfer_queue.n) {
    int r = s->transfer_queue.v[0];
    int best = -1;
    for (int ri = 0; ri < s->R; ri++) {
      Rep* R = &s->rep[ri];
      if (R->d->role != FS_ROLE_DECODE) continue;
      if (best < 0 || R->pool.used < s->rep[best].pool.used ||
          (R->pool.used == s->rep[best].pool.used && R->d->key_rank < s->rep[best].d->key_rank))
        best = ri;
    }
    Rep* D = &s->rep[best];
    int64_t fp = (int64_t)s->prompt[r] + s->output[r];
    if (pool_rounded(&D->pool, fp) > D->pool.cap) fail(s, FS_ERR_REQUEST_CANNOT_FIT, r);
    if (pool_reserve(&D->pool, r, fp)) return; /* Backpressure */
    memmove(s->transfer_queue.v, s->transfer_queue.v + 1,
            sizeof(int32_t) * (size_t)(s->transfer_queue.n - 1));
    s->transfer_queue.n--;
    s->decode_home[r] = best;
    int64_t nbytes = d->kv_bytes_per_token * s->prompt[r];
    int64_t sq = schedule(s, s->now, EV_KV_START, best, r);
    otrace(s, sq, s->now, EV_KV_START, best, r, (int32_t)D->pool.charged[r], s->prefill_home[r],
           D->pool.used);
    double sec = d->inter_latency_s + (double)nbytes / d->inter_bandwidth_bps;
    int64_t dur = py_round(sec * 1e9);
    sq = schedule(s, s->now + dur, EV_KV_DONE, best, r);
    otrace(s, sq, s->now + dur, EV_KV_DONE, best, r, 0, s->prefill_home[r], 0);
  }
}
static void pd_on_transfer_done(Sim* s, int r) {
  int ph = s->prefill_home[r];
  Pool* pl = &s->rep[ph].pool;
  int64_t freed = pool_release(s, pl, r);
  int64_t sq = schedule(s, s->now, EV_MEMORY_AVAILABLE, ph, r);
  otrace(s, sq, s->now, EV_MEMORY_AVAILABLE, ph, r, (int32_t)freed, 0, pl->cap - pl->used);
  int dh = s->decode_home[r];
  iv_push(&s->rep[dh].queue, r);
  kick(s, ph);
  kick(s, dh);
}

/* ---- af.py ---- */
typedef struct AfEngine {
  int m, L;
  int64_t step_id, start_ts;
  int64_t* dur;          /* [m][L][4] node durations */
  int* stage;            /* per micro-batch: next node index in chain (0..4L-2) */
  uint64_t ready[4];     /* bitmask of micro-batches ready per resource */
  int busy[4];           /* micro-batch + 1 running on resource, 0 if free */
  int64_t* pend_t; int* pend_n; int n_pend; /* pending_at */
  int64_t done_count, node_count, final_ts;
  int n_members;
  int32_t* ids;
  int* mb_size;
} AfEngine;

static int64_t af_transfer_ns(Sim* s, int64_t n) {
  const fs_instance_desc* d = s->d;
  int64_t nb = n * d->d_model * (int64_t)d->dtype_bytes;
  double sec = d->inter_latency_s + (double)nb / d->inter_bandwidth_bps;
  return py_round(sec * 1e9);
}
/* AfStepCosts._attn_duration_ns (af.py:276-287) */
static int64_t af_attn_ns(Sim* s, const int32_t* ids, int n) {
  const fs_instance_desc* d = s->d;
  int g = d->af_attn_dp < n ? d->af_attn_dp : n;
  int worst = n / g + (n % g ? 1 : 0);   /* partition_micro_batches(...)[0] */
  Plan p = {1, worst, ids};
  const fs_cost_ctx* c = &d->af_attn;
  double us = qkv_us(d, c, worst) + attn_us(s, c, &p);
  us = us + out_us(d, c, worst);
  us = us + tpcoll_us(d, c, worst);
  return py_round(us * 1000.0);
}
/* AfStepCosts._ffn_duration_ns (af.py:289-301) */
static int64_t af_ffn_ns(Sim* s, int ri, int mb, int64_t n, int layer, int64_t step) {
  const fs_instance_desc* d = s->d;
  const fs_cost_ctx* c = &d->af_ffn;
  double us;
  if (d->has_moe) {
    const fs_seed_prefix* pf = &s->prefixes[s->rep[ri].d->prefix_mb];
    uint32_t seed = router_seed(pf, mb, step, layer);
    int64_t* counts = route(s, n, seed, 1, ri, mb, step, layer);
    double ratio;
    us = moe_layer(s, counts, n, c, c->ep, c->moe_tp, &ratio);
    free(counts);
  } else {
    us = dense_ffn_us(s, c, n);
    us = us + tpcoll_us(d, c, n);
  }
  return py_round(us * 1000.0);
}

static void af_start_node(Sim* s, AfEngine* g, int res) {
  /* lowest micro-batch index among ready nodes of this resource */
  int i = __builtin_ctzll(g->ready[res]);
  g->ready[res] &= g->ready[res] - 1;
  g->busy[res] = i + 1;
  int st = g->stage[i];
  int k = st / 4, kind = st % 4;
  int64_t dur = g->dur[((int64_t)i * g->L + k) * 4 + kind];
  int64_t end = s->now + dur;
  int found = 0;
  for (int j = 0; j < g->n_pend; j++)
    if (g->pend_t[j] == end) { g->pend_n[j]++; found = 1; break; }
  if (!found) { g->pend_t[g->n_pend] = end; g->pend_n[g->n_pend] = 1; g->n_pend++; }
  s->af_busy[res] += dur;
  if (kind == 0) s->af_step_attn[s->n_af - 1] += dur;
  int64_t sq = schedule(s, end, EV_ATTN_DONE + kind, i, dur);
  otrace(s, sq, end, EV_ATTN_DONE + kind, 0, i + 1, k + 1, (int32_t)g->step_id, s->now);
}
static void af_dispatch_all(Sim* s, AfEngine* g) {
  for (int res = 0; res < 4; res++)
    if (!g->busy[res] && g->ready[res]) af_start_node(s, g, res);
}
static void af_on_batch_complete_schedule(Sim* s, AfEngine* g);
static void af_on_node_done(Sim* s, int kind, int i) {
  AfEngine* g = s->af;
  if (!g) fail(s, FS_ERR_INTERNAL, 4);
  g->busy[kind] = 0;
  g->done_count++;
  int st = g->stage[i];
  int k = st / 4;
  if (kind == 2 && i == g->m - 1 && k == g->L - 1) g->final_ts = s->now;
  /* successor: next node in the micro-batch chain (F2A omitted at k = L) */
  int next = st + 1;
  if (kind == 2 && k == g->L - 1) next = -1;
  g->stage[i] = next;
  if (next >= 0) g->ready[next % 4] |= 1ull << i;
  int j;
  for (j = 0; j < g->n_pend; j++) if (g->pend_t[j] == s->now) break;
  if (j == g->n_pend) fail(s, FS_ERR_INTERNAL, 5);
  if (--g->pend_n[j] == 0) {
    g->pend_t[j] = g->pend_t[g->n_pend - 1];
    g->pend_n[j] = g->pend_n[g->n_pend - 1];
    g->n_pend--;
    if (g->done_count == g->node_count) af_on_batch_complete_schedule(s, g);
    else af_dispatch_all(s, g);
  }
}
static void af_start_step(Sim* s, int ri) {
  const fs_instance_desc* d = s->d;
  Rep* R = &s->rep[ri];
  int n = R->running.n < d->max_num_seqs ? R->running.n : d->max_num_seqs;
  int m = d->af_micro_batches < n ? d->af_micro_batches : n;
  if (m > FS_MAX_MICRO_BATCHES) fail(s, FS_ERR_CAPACITY, m);
  AfEngine* g = (AfEngine*)calloc(1, sizeof(AfEngine));
  g->m = m;
  g->L = d->num_layers;
  g->n_members = n;
  g->ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  memcpy(g->ids, R->running.v, sizeof(int32_t) * (size_t)n);
  g->mb_size = (int*)malloc(sizeof(int) * (size_t)m);
  g->stage = (int*)calloc((size_t)m, sizeof(int));
  g->dur = (int64_t*)calloc((size_t)m * g->L * 4, sizeof(int64_t));
  g->pend_t = (int64_t*)malloc(sizeof(int64_t) * 8);
  g->pend_n = (int*)malloc(sizeof(int) * 8);
  int64_t step = s->af_counter++;
  g->step_id = step;
  s->af = g;
  /* build_af_graph evaluates every node duration eagerly, in (i, k) order */
  int base = n / m, rem = n % m, off = 0;
  for (int i = 0; i < m; i++) {
    int sz = base + (i < rem ? 1 : 0);
    g->mb_size[i] = sz;
    const int32_t* mids = g->ids + off;
    int64_t tr = -1;
    for (int k = 0; k < g->L; k++) {
      int64_t* nd = &g->dur[((int64_t)i * g->L + k) * 4];
      nd[0] = af_attn_ns(s, mids, sz);
      if (tr < 0) tr = af_transfer_ns(s, sz);
      nd[1] = tr;
      nd[2] = af_ffn_ns(s, ri, i + 1, sz, k, step);
      if (k < g->L - 1) nd[3] = tr;
    }
    off += sz;
  }
  g->node_count = 4LL * m * g->L - m;
  R->busy = 1;
  R->steps++;
  g->start_ts = s->now;
  if (s->n_af == s->af_cap) {
    s->af_cap = s->af_cap ? 2 * s->af_cap : 256;
    s->af_step_start = (int64_t*)realloc(s->af_step_start, sizeof(int64_t) * (size_t)s->af_cap);
    s->af_step_dur = (int64_t*)realloc(s->af_step_dur, sizeof(int64_t) * (size_t)s->af_cap);
    s->af_step_attn = (int64_t*)realloc(s->af_step_attn, sizeof(int64_t) * (size_t)s->af_cap);
  }
  s->af_step_start[s->n_af] = s->now;
  s->af_step_dur[s->n_af] = 0;
  s->af_step_attn[s->n_af] = 0;
  s->n_af++;
  for (int i = 0; i < m; i++) g->ready[0] |= 1ull << i;
  af_dispatch_all(s, g);
}
static void af_on_batch_complete_schedule(Sim* s, AfEngine* g) {
  int bi = batch_new(s, 2, 0, g->ids, g->n_members);
  s->batches[bi].duration_ns = g->final_ts - g->start_ts;
  s->batches[bi].af_step = g->step_id;
  s->af_step_dur[s->n_af - 1] = g->final_ts - g->start_ts;
  s->batches[bi].pool_used = s->rep[0].pool.used;
  int64_t sq = schedule(s, g->final_ts, EV_BATCH_COMPLETE, 0, bi);
  olog_batch(s, bi, g->final_ts, sq, g->step_id);
  free(g->ids); free(g->mb_size); free(g->stage); free(g->dur); free(g->pend_t); free(g->pend_n);
  free(g);
  s->af = NULL;
}
static void af_on_arrival(Sim* s, int r) {
  iv_push(&s->rep[0].queue, r);
  kick(s, 0);
}
static void af_on_batch_start(Sim* s, int ri) {
  Rep* R = &s->rep[ri];
  R->start_pending = 0;
  if (R->busy) return;
  if (admit_full(s, ri)) return;
  if (R->running.n) { af_start_step(s, ri); return; }
  if (R->queue.n) fail(s, FS_ERR_REQUEST_CANNOT_FIT, R->queue.v[0]);
}

/* ------------------------------------------------------------------------ */
/* Run + compute_metrics                                                    */
/* ------------------------------------------------------------------------ */
static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}
static int cmp_f64(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
static double nearest_rank(const double* sorted, int n, double pct) {
  long idx = (long)ceil(pct / 100.0 * (double)n) - 1;
  if (idx < 0) idx = 0;
  return sorted[idx];
}
static void aggregate(double* vals, int n, double out[4]) {
  if (n == 0) { out[0] = out[1] = out[2] = out[3] = NAN; return; }
  pysum_t ps;
  pysum_init(&ps);
  for (int i = 0; i < n; i++) pysum_add(&ps, vals[i]);
  out[0] = pysum_result(&ps) / (double)n;
  qsort(vals, (size_t)n, sizeof(double), cmp_f64);
  out[1] = nearest_rank(vals, n, 50);
  out[2] = nearest_rank(vals, n, 90);
  out[3] = nearest_rank(vals, n, 99);
}

/* Runs one instance. Exported for tests; all pointers are instance-local. */
int fso_run_instance(const fs_instance_desc* d, const fs_replica_desc* reps,
                     const fs_seed_prefix* prefixes, const int64_t* trace_counts,
                     const int64_t* arrival, const int32_t* prompt, const int32_t* output,
                     const int32_t* id_rank, fs_metric_row* row, fs_replica_out* rep_out,
                     int64_t* first_ns, int64_t* done_ns, int32_t* done_rank,
                     fs_log* log, int inst, const fs_forest_set* forests) {
  Sim S;
  Sim* s = &S;
  memset(s, 0, sizeof S);
  s->d = d;
  s->prefixes = prefixes;
  s->trace_counts = trace_counts;
  s->N = d->n_requests;
  s->R = d->n_replicas;
  s->arrival = arrival; s->prompt = prompt; s->output = output; s->id_rank = id_rank;
  s->log = log; s->inst = inst;
  s->forests = forests;
  int N = s->N, R = s->R;
  s->emitted = (int32_t*)calloc((size_t)N + 1, sizeof(int32_t));
  s->first_ns = first_ns; s->done_ns = done_ns; s->done_rank = done_rank;
  for (int i = 0; i < N; i++) { first_ns[i] = -1; done_ns[i] = -1; done_rank[i] = -1; }
  s->prefill_home = (int32_t*)calloc((size_t)N + 1, sizeof(int32_t));
  s->decode_home = (int32_t*)calloc((size_t)N + 1, sizeof(int32_t));
  s->rep = (Rep*)calloc((size_t)R, sizeof(Rep));
  for (int ri = 0; ri < R; ri++) {
    Rep* P = &s->rep[ri];
    P->d = &reps[ri];
    P->pool.cap = reps[ri].kv_pool_tokens;
    P->pool.block = d->paged ? d->block_tokens : 0;
    P->pool.raw = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
    P->pool.charged = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
    P->pool.has = (uint8_t*)calloc((size_t)N + 1, 1);
  }
  memset(row, 0, sizeof *row);
  if (log && log->batch_count) { log->batch_count[inst] = 0; log->route_count[inst] = 0; log->truncated[inst] = 0; }

  if (setjmp(s->jb) == 0) {
    /* learned grouped GEMM on MoE layers needs numpy's np.log (entropy): next */
    /* schedule_arrivals (base.py:167-177): seq 0..N-1 */
    for (int i = 0; i < N; i++) {
      int64_t sq = schedule(s, arrival[i], EV_ARRIVAL, -1, i);
      otrace(s, sq, arrival[i], EV_ARRIVAL, -1, i, 0, 0, 0);
    }
    while (s->hn) {
      Ev e = heap_pop(s);
      s->processed++;
      if (s->processed > d->max_events) fail(s, FS_ERR_EVENT_BUDGET, 0);
      s->now = e.t;
      switch (e.kind) {
        case EV_ARRIVAL:
          if (d->mode == FS_MODE_COLOCATED) co_on_arrival(s, (int)e.b);
          else if (d->mode == FS_MODE_PD) pd_on_arrival(s, (int)e.b);
          else af_on_arrival(s, (int)e.b);
          break;
        case EV_BATCH_START:
          if (d->mode == FS_MODE_COLOCATED) co_on_batch_start(s, e.a);
          else if (d->mode == FS_MODE_PD) pd_on_batch_start(s, e.a);
          else af_on_batch_start(s, e.a);
          break;
        case EV_BATCH_COMPLETE: {
          Batch* b = &s->batches[e.b];
          s->rep[e.a].busy_ns += b->duration_ns;
          if (b->phase == 0) row->prefill_batches++;
          else if (b->phase == 1) row->decode_batches++;
          else row->af_steps++;
          if (b->moe) row->moe_layer_samples += b->n_moe;
          if (d->mode == FS_MODE_COLOCATED) co_on_batch_complete(s, e.a, (int)e.b);
          else if (d->mode == FS_MODE_PD) pd_on_batch_complete(s, e.a, (int)e.b);
          else {
            Rep* A = &s->rep[0];
            A->busy = 0;
            if (b->phase == 0) prefill_complete(s, 0, b, 1);
            else decode_complete(s, 0, b);
            kick(s, 0);
          }
          break;
        }
        case EV_KV_DONE: pd_on_transfer_done(s, (int)e.b); break;
        case EV_ATTN_DONE: case EV_A2F_DONE: case EV_FFN_DONE: case EV_F2A_DONE:
          af_on_node_done(s, e.kind - EV_ATTN_DONE, e.a);
          break;
        default: break; /* no-op kinds */
      }
    }
    for (int i = 0; i < N; i++)
      if (s->emitted[i] != output[i]) fail(s, FS_ERR_SIMULATION, i);
  }

  if (log && log->event_count) log->event_count[inst] = s->next_seq;
  row->status = s->status;
  row->status_detail = s->detail;
  row->events = s->processed;
  row->iterations = row->prefill_batches + row->decode_batches + row->af_steps;
  row->n_requests = N;
  row->routing_calls = s->routing_calls;
  row->routing_draws = s->routing_draws;
  if (s->status == FS_OK && N > 0) {
    /* compute_metrics (metrics.py:81-178) */
    double* tt = (double*)malloc(sizeof(double) * (size_t)N * 3);
    double* tp = tt + N;
    double* ee = tp + N;
    int ntp = 0;
    int64_t maxdone = 0, minarr = arrival[0];
    int64_t sum_p = 0, sum_o = 0, tokens = 0;
    for (int i = 0; i < N; i++) {
      double ttft = (double)(first_ns[i] - arrival[i]) / 1e9;
      double e2e = (double)(done_ns[i] - arrival[i]) / 1e9;
      tt[i] = ttft;
      ee[i] = e2e;
      if (output[i] > 1) tp[ntp++] = (e2e - ttft) / (double)(output[i] - 1);
      if (i == 0 || done_ns[i] > maxdone) maxdone = done_ns[i];
      if (arrival[i] < minarr) minarr = arrival[i];
      sum_p += prompt[i];
      sum_o += output[i];
      tokens += output[i];
    }
    int64_t mk = maxdone - minarr;
    if (mk < 1) mk = 1;
    row->makespan_ns = mk;
    row->makespan_s = (double)mk / 1e9;
    row->total_tokens = tokens;
    row->throughput_tokens_per_s_per_gpu = (double)tokens / row->makespan_s / (double)d->total_gpus;
    row->n_tpot = ntp;
    aggregate(tt, N, row->ttft);
    aggregate(tp, ntp, row->tpot);
    aggregate(ee, N, row->e2e);
    row->avg_input_tokens = (double)sum_p / (double)N;
    row->avg_output_tokens = (double)sum_o / (double)N;
    for (int q = 0; q < 4; q++) {
      row->af_busy_ns[q] = s->af_busy[q];
      row->af_busy_fraction[q] = py_min(1.0, (double)s->af_busy[q] / (double)mk);
    }
    if (s->n_af) {
      double weighted = 0.0;
      int64_t total = 0;
      for (int q = 0; q < s->n_af; q++) {
        int64_t dur = s->af_step_dur[q];
        if (dur <= 0) continue;
        int64_t idle = dur - s->af_step_attn[q];
        if (idle < 0) idle = 0;
        weighted = weighted + (double)idle;
        total += dur;
      }
      row->bubble_fraction = total ? weighted / (double)total : 0.0;
    } else {
      row->bubble_fraction = NAN;
    }
    for (int ri = 0; ri < R; ri++) {
      rep_out[ri].busy_ns = s->rep[ri].busy_ns;
      rep_out[ri].busy_fraction = py_min(1.0, (double)s->rep[ri].busy_ns / (double)mk);
      rep_out[ri].steps_executed = s->rep[ri].steps;
    }
    free(tt);
  } else {
    for (int ri = 0; ri < R; ri++) {
      rep_out[ri].busy_ns = s->rep[ri].busy_ns;
      rep_out[ri].busy_fraction = NAN;
      rep_out[ri].steps_executed = s->rep[ri].steps;
    }
  }

  for (int i = 0; i < s->nb; i++) { iv_free(&s->batches[i].ids); free(s->batches[i].moe); }
  free(s->batches);
  for (int ri = 0; ri < R; ri++) {
    iv_free(&s->rep[ri].queue);
    iv_free(&s->rep[ri].running);
    free(s->rep[ri].pool.raw); free(s->rep[ri].pool.charged); free(s->rep[ri].pool.has);
  }
  if (s->af) {
    free(s->af->ids); free(s->af->mb_size); free(s->af->stage); free(s->af->dur);
    free(s->af->pend_t); free(s->af->pend_n); free(s->af);
  }
  free(s->rep); free(s->emitted); free(s->prefill_home); free(s->decode_home);
  iv_free(&s->transfer_queue);
  free(s->heap);
  free(s->af_step_start); free(s->af_step_dur); free(s->af_step_attn);
  return row->status;
}

/* Batch driver with the engine's calling convention; instances run on
 * `threads` POSIX threads (the CPU baseline uses every host core). */
#include <pthread.h>
typedef struct {
  const fs_instance_desc* descs; const fs_replica_desc* reps; const fs_seed_prefix* pf;
  const int64_t* tc; fs_request_soa rq; fs_metric_row* rows; fs_replica_out* ro;
  fs_request_out pr; fs_log* log; const fs_forest_set* forests; int n; int next; pthread_mutex_t mu;
} Job;
static void* worker(void* arg) {
  Job* j = (Job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->n) break;
    const fs_instance_desc* d = &j->descs[i];
    int64_t o = d->req_offset;
    int N = d->n_requests;
    int64_t* fn = j->pr.first_token_ns ? j->pr.first_token_ns + o : (int64_t*)malloc(8 * (size_t)(N + 1));
    int64_t* dn = j->pr.done_ns ? j->pr.done_ns + o : (int64_t*)malloc(8 * (size_t)(N + 1));
    int32_t* dr = j->pr.completion_rank ? j->pr.completion_rank + o : (int32_t*)malloc(4 * (size_t)(N + 1));
    fs_replica_out* tmp = j->ro ? NULL : (fs_replica_out*)malloc(sizeof(fs_replica_out) *
                                                                  (size_t)(d->n_replicas + 1));
    fs_replica_out* ro = j->ro ? j->ro + d->replica_offset : tmp;
    fso_run_instance(d, j->reps + d->replica_offset, j->pf, j->tc, j->rq.arrival_ns + o,
                     j->rq.prompt_tokens + o, j->rq.output_tokens + o, j->rq.id_rank + o,
                     &j->rows[i], ro, fn, dn, dr, j->log, i, j->forests);
    if (!j->pr.first_token_ns) free(fn);
    if (!j->pr.done_ns) free(dn);
    if (!j->pr.completion_rank) free(dr);
    free(tmp);
  }
  return NULL;
}

int fso_run_batch(const fs_instance_desc* descs, int32_t n_instances,
                  const fs_replica_desc* replicas, const fs_seed_prefix* prefixes,
                  const int64_t* trace_counts, fs_request_soa requests,
                  fs_metric_row* rows_out, fs_replica_out* replica_out,
                  fs_request_out per_request, fs_log* log, int threads,
                  const fs_forest_set* forests) {
  Job j;
  memset(&j, 0, sizeof j);
  j.descs = descs; j.reps = replicas; j.pf = prefixes; j.tc = trace_counts; j.rq = requests;
  j.rows = rows_out; j.ro = replica_out; j.pr = per_request; j.log = log; j.n = n_instances;
  j.forests = forests;
  pthread_mutex_init(&j.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  pthread_t th[512];
  for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker, &j);
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&j.mu);
  return 0;
}

/* ---- pure-function entry points for golden-vector tests ---- */
uint32_t fso_router_seed(const fs_seed_prefix* pf, int mb, int64_t step, int32_t layer) {
  return router_seed(pf, mb, step, layer);
}
uint32_t fso_sha256_first_word(const uint8_t* msg, int64_t len) {
  return sha256_first_word(msg, (size_t)len);
}
void fso_routing_key(uint64_t seed, uint64_t key[2]) { routing_key(seed, key); }
/* route_tokens(T, E, k, policy, seed, alpha).counts (routing.py:65-113) for
 * the uniform / dirichlet_skew policies; returns a status */
int fso_route(int64_t T, int32_t E, int32_t k, int32_t policy, double alpha, uint64_t seed,
              int32_t* counts_out) {
  if (!(1 <= k && k <= E)) return FS_ERR_INVALID_TOPK;
  if (T < 0) return FS_ERR_ROUTING;
  int64_t* counts = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  int st = 0;
  if (T == 0) {
  } else if (k == E) {
    for (int e = 0; e < E; e++) counts[e] = T;
  } else {
    st = route_core(T, E, k, policy, alpha, seed, counts);
  }
  for (int e = 0; e < E; e++) counts_out[e] = (int32_t)counts[e];
  free(counts);
  return st;
}
int fso_route_uniform(int64_t T, int32_t E, int32_t k, uint64_t seed, int32_t* counts_out) {
  return fso_route(T, E, k, FS_ROUTE_UNIFORM, 0.3, seed, counts_out);
}
/* ---- synthetic workload (workload.py:131-216) ---- */
/* numpy Philox next_uint32: low half of a 64-bit draw first, then the high half */
typedef struct { np_philox g; int has32; uint32_t u32; } np_stream32;
static uint32_t np_next_u32(np_stream32* s) {
  if (s->has32) { s->has32 = 0; return s->u32; }
  uint64_t v = np_next_u64(&s->g);
  s->has32 = 1;
  s->u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}
/* Generator.integers(lo, hi + 1, dtype=int64): random_bounded_uint64_fill, Lemire */
static int64_t np_integer(np_stream32* s, int64_t lo, int64_t hi) {
  uint64_t rng = (uint64_t)(hi - lo);
  if (rng == 0) return lo;
  if (rng <= 0xFFFFFFFFull) {
    if (rng == 0xFFFFFFFFull) return lo + (int64_t)np_next_u32(s);
    const uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)np_next_u32(s) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)(UINT32_MAX - (uint32_t)rng) % excl;
      while (left < thr) { m = (uint64_t)np_next_u32(s) * excl; left = (uint32_t)m; }
    }
    return lo + (int64_t)(m >> 32);
  }
  if (rng == UINT64_MAX) return lo + (int64_t)np_next_u64(&s->g);
  const uint64_t excl = rng + 1;
  unsigned __int128 m = (unsigned __int128)np_next_u64(&s->g) * excl;
  uint64_t left = (uint64_t)m;
  if (left < excl) {
    const uint64_t thr = (UINT64_MAX - rng) % excl;
    while (left < thr) { m = (unsigned __int128)np_next_u64(&s->g) * excl; left = (uint64_t)m; }
  }
  return lo + (int64_t)(m >> 64);
}
/* key = SeedSequence([seed, stream]).generate_state(2, uint64) (workload.py:188-190) */
static void workload_key(uint64_t seed, uint32_t stream, uint64_t key[2]) {
  uint32_t ent[4], st[4];
  int n = int_words(seed, ent);
  n += int_words(stream, ent + n);
  seedseq_state(ent, n, st, 4);
  key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}
static int sample_lengths(const fs_length_dist* L, uint64_t seed, uint32_t stream, int n,
                          int32_t* out) {
  np_stream32 s;
  memset(&s, 0, sizeof s);
  workload_key(seed, stream, s.g.key);
  for (int i = 0; i < n; i++) {
    int64_t v;
    if (L->kind == FS_LEN_FIXED) {
      v = L->value;
    } else if (L->kind == FS_LEN_UNIFORM) {
      v = np_integer(&s, L->lo, L->hi);
    } else if (L->kind == FS_LEN_LOGNORMAL) {
      double x = rint(exp(L->mu + L->sigma * np_std_normal(&s.g)));  /* random_lognormal */
      if (x < (double)L->lo) x = (double)L->lo;
      if (x > (double)L->hi) x = (double)L->hi;
      v = (int64_t)x;
    } else {
      return FS_ERR_VALUE;
    }
    out[i] = (int32_t)v;
  }
  return FS_OK;
}
/* Python str order rank of "r{i}" among "r0".."r{n-1}" */
static int32_t id_str_rank(int64_t i, int64_t n) {
  char t[24];
  int m = sprintf(t, "%lld", (long long)i);
  int64_t rank = 0, lo = 0, p10 = 1;
  for (int d = 1; d <= 19 && lo < n; d++) {
    const int64_t hi = (p10 > INT64_MAX / 10) ? INT64_MAX : p10 * 10;  /* [lo, hi) has d digits */
    const int64_t end = hi < n ? hi : n;
    if (d <= m) {
      int64_t pre = 0;
      for (int q = 0; q < d; q++) pre = pre * 10 + (t[q] - '0');
      int64_t c = pre - lo; if (c < 0) c = 0; if (c > end - lo) c = end - lo;
      rank += c;
      if (d < m && pre >= lo && pre < end) rank += 1;   /* proper prefix sorts first */
    } else {
      int64_t scale = 1;
      for (int q = 0; q < d - m; q++) scale *= 10;
      int64_t tv = 0;
      for (int q = 0; q < m; q++) tv = tv * 10 + (t[q] - '0');
      /* d-digit j with floor(j / scale) < tv */
      int64_t bound = tv * scale;               /* j < bound */
      int64_t c = bound - lo; if (c < 0) c = 0; if (c > end - lo) c = end - lo;
      rank += c;
    }
    lo = hi;
    p10 = hi;
    if (d == 1) lo = 10;
  }
  return (int32_t)rank;
}
int fso_generate_workload(const fs_workload_desc* w, int32_t n, int64_t* arrival_ns,
                          int32_t* prompt, int32_t* output, int32_t* id_rank, int32_t* status) {
  for (int k = 0; k < n; k++) {
    const fs_workload_desc* d = &w[k];
    const int64_t o = d->out_offset;
    const int nr = d->n_requests;
    int st = FS_OK;
    if (d->arrival_kind == FS_ARRIVAL_POISSON) {
      np_philox g;
      memset(&g, 0, sizeof g);
      workload_key(d->seed, 0, g.key);
      const double scale = 1.0 / d->rate_rps;
      double acc = 0.0;
      for (int i = 0; i < nr; i++) {
        acc = acc + scale * np_std_exponential(&g);   /* cumsum of exponential(scale) */
        arrival_ns[o + i] = (int64_t)rint(acc * 1e9);
      }
    } else if (d->arrival_kind == FS_ARRIVAL_FIXED) {
      for (int i = 0; i < nr; i++) arrival_ns[o + i] = (int64_t)i * d->gap_ns;
    } else if (d->arrival_kind == FS_ARRIVAL_AT_ZERO) {
      for (int i = 0; i < nr; i++) arrival_ns[o + i] = 0;
    } else {
      st = FS_ERR_VALUE;
    }
    if (!st) st = sample_lengths(&d->prompt, d->seed, 1, nr, prompt + o);
    if (!st) st = sample_lengths(&d->output, d->seed, 2, nr, output + o);
    for (int i = 0; i < nr; i++) id_rank[o + i] = id_str_rank(i, nr);
    status[k] = st;
  }
  return 0;
}

/* GroupedGemmFeatures(..., mode="local").vector() and, with a forest set, the
 * learned prediction (features.py:166-209, model.py:323-326) */
double fso_gg_features(const fs_forest_set* fs, int forest, const int64_t* counts, int n,
                       int64_t d_model, int64_t d_ff, int top_k, double* x12) {
  gg_local_features(counts, n, d_model, d_ff, top_k, x12);
  return fs ? forest_predict(fs, forest, x12) : 0.0;
}
/* debugging aid for the dirichlet stream: popularity[E] and the first row of keys */
void fso_dirichlet_row(int32_t E, double alpha, uint64_t seed, double* pop, double* keys) {
  np_philox g;
  memset(&g, 0, sizeof g);
  routing_key(seed, g.key);
  np_dirichlet_sym(&g, E, alpha, pop);
  for (int e = 0; e < E; e++) keys[e] = np_std_exponential(&g) / pop[e];
}
double fso_attention_us(int decode, const int64_t* q, const int64_t* kv, int B, int hq, int hkv,
                        int hdim, double peak, double bw, double ovh, int dt) {
  fs_cost_ctx c = {peak, bw, ovh, 1, 1, 1, 1};
  return attention_us_analytic(decode, q, kv, B, hq, hkv, hdim, &c, dt);
}
/* topology.collective_time(kind, bytes_per_rank, n, link) (topology.py:370-394);
 * kind 0 all_to_all, 1 all_reduce, 2 all_gather */
double fso_collective(int kind, double bytes_per_rank, int n, double lat, double bw) {
  return collective_flt(kind, bytes_per_rank, n, lat, bw);
}
double fso_linear_us(int64_t m, int64_t n, int64_t k, double peak, double bw, double ovh, int dt) {
  fs_cost_ctx c = {peak, bw, ovh, 1, 1, 1, 1};
  return linear_us(m, n, k, &c, dt);
}
/* LearnedOperatorModel.predict_us on one attention batch (for golden tests) */
double fso_attention_forest(const fs_forest_set* fs, int forest, int decode, const int64_t* q,
                            const int64_t* kv, int B, int hq, int hkv, int hdim, double* x17) {
  attention_features(decode, q, kv, B, hq, hkv, hdim, x17);
  return forest_predict(fs, forest, x17);
}
double fso_pysum(const double* x, int n) {
  pysum_t s;
  pysum_init(&s);
  for (int i = 0; i < n; i++) pysum_add(&s, x[i]);
  return pysum_result(&s);
}

/* The system libm's exp / log / log1p / pow (the functions numpy's distributions.c
 * calls) over arrays: fn 1 exp, 2 log, 3 log1p, 4 pow(x[i], y[i]). The device's
 * restatement (fs_glibm.h) is tested against these. */
void fso_libm(int fn, const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    switch (fn) {
      case 1: out[i] = exp(x[i]); break;
      case 2: out[i] = log(x[i]); break;
      case 3: out[i] = log1p(x[i]); break;
      case 4: out[i] = pow(x[i], y[i]); break;
      default: out[i] = 0.0;
    }
  }
}

int fso_struct_sizes(int64_t* out, int n) {
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
