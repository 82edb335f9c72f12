/*
 * abi_client.c -- a non-Python caller of include/frontier_b200.h (plain C, no
 * torch, linked against libfrontier_b200.so). It is what a maintainer binding
 * the engine from C/C++/cgo would write; tests/test_c_abi.py builds and runs it.
 *
 *   abi_client DIR
 *
 * DIR/batch.bin holds a lowered batch written by the test (counts, then the
 * descriptor / replica / prefix / trace-count arrays and the request SoA, all
 * in the ABI's own struct layouts). The client:
 *   1. checks fs_abi_version and the struct sizes it was compiled with,
 *   2. runs fs_run_batch on the batch and writes the metric rows and the
 *      per-request first-token / completion times to DIR/rows.bin, DIR/req.bin,
 *   3. generates one C1-shaped synthetic workload with fs_generate_workload and
 *      routes a few calls with fs_route_tokens, printing both for the test.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "frontier_b200.h"

static void* read_exact(FILE* f, size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (bytes && fread(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "short read\n");
    exit(3);
  }
  return p;
}

static int check(fs_engine* e, int rc, const char* what) {
  if (rc) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, e ? fs_last_error(e) : "");
    exit(4);
  }
  return rc;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: abi_client DIR\n");
    return 2;
  }
  if (fs_abi_version() != FS_ABI_VERSION) return 5;
  int64_t sizes[16];
  const int ns = fs_struct_sizes(sizes, 16);
  const int64_t mine[] = {sizeof(fs_cost_ctx),    sizeof(fs_seed_prefix), sizeof(fs_replica_desc),
                          sizeof(fs_instance_desc), sizeof(fs_metric_row), sizeof(fs_replica_out),
                          sizeof(fs_batch_rec),   sizeof(fs_route_rec),   sizeof(fs_attn_params),
                          sizeof(fs_forest_desc), sizeof(fs_workload_desc)};
  for (int i = 0; i < ns && i < (int)(sizeof(mine) / sizeof(mine[0])); i++)
    if (sizes[i] != mine[i]) { fprintf(stderr, "struct %d size mismatch\n", i); return 6; }

  fs_engine* e = NULL;
  if (fs_create(0, &e)) { fprintf(stderr, "fs_create failed\n"); return 7; }

  /* ---- 1. the batched simulation through fs_run_batch ---- */
  char path[4096];
  snprintf(path, sizeof path, "%s/batch.bin", argv[1]);
  FILE* f = fopen(path, "rb");
  if (!f) { perror(path); return 8; }
  int64_t hdr[5];  /* n_instances, n_replicas, n_prefixes, n_trace_counts, n_requests */
  if (fread(hdr, sizeof hdr, 1, f) != 1) return 9;
  const int32_t ni = (int32_t)hdr[0], nr = (int32_t)hdr[1], np = (int32_t)hdr[2];
  const int64_t nt = hdr[3], nq = hdr[4];
  fs_instance_desc* descs = read_exact(f, sizeof(fs_instance_desc) * (size_t)ni);
  fs_replica_desc* reps = read_exact(f, sizeof(fs_replica_desc) * (size_t)nr);
  fs_seed_prefix* pfx = read_exact(f, sizeof(fs_seed_prefix) * (size_t)np);
  int64_t* trace = read_exact(f, sizeof(int64_t) * (size_t)nt);
  fs_request_soa soa;
  soa.arrival_ns = read_exact(f, sizeof(int64_t) * (size_t)nq);
  soa.prompt_tokens = read_exact(f, sizeof(int32_t) * (size_t)nq);
  soa.output_tokens = read_exact(f, sizeof(int32_t) * (size_t)nq);
  soa.id_rank = read_exact(f, sizeof(int32_t) * (size_t)nq);
  fclose(f);

  fs_metric_row* rows = calloc((size_t)ni, sizeof(fs_metric_row));
  fs_request_out req;
  req.first_token_ns = calloc((size_t)nq, sizeof(int64_t));
  req.done_ns = calloc((size_t)nq, sizeof(int64_t));
  req.completion_rank = calloc((size_t)nq, sizeof(int32_t));
  check(e, fs_run_batch(e, descs, ni, reps, nr, pfx, np, trace, nt, soa, nq, rows, NULL, req, NULL),
        "fs_run_batch");
  snprintf(path, sizeof path, "%s/rows.bin", argv[1]);
  f = fopen(path, "wb");
  fwrite(rows, sizeof(fs_metric_row), (size_t)ni, f);
  fclose(f);
  snprintf(path, sizeof path, "%s/req.bin", argv[1]);
  f = fopen(path, "wb");
  fwrite(req.first_token_ns, sizeof(int64_t), (size_t)nq, f);
  fwrite(req.done_ns, sizeof(int64_t), (size_t)nq, f);
  fclose(f);
  int64_t its = 0;
  for (int i = 0; i < ni; i++) its += rows[i].iterations;
  printf("run_batch instances=%d iterations=%lld launches=%d\n", ni, (long long)its,
         fs_last_launch_count(e));

  /* ---- 2. one synthetic workload (C1 shape: Poisson 20 rps, lognormal lengths) ---- */
  fs_workload_desc w;
  memset(&w, 0, sizeof w);
  w.seed = 1;
  w.n_requests = 8;
  w.arrival_kind = FS_ARRIVAL_POISSON;
  w.rate_rps = 20.0;
  w.prompt.kind = FS_LEN_LOGNORMAL; w.prompt.mu = 6.0; w.prompt.sigma = 1.0;
  w.prompt.lo = 8; w.prompt.hi = 4096;
  w.output.kind = FS_LEN_LOGNORMAL; w.output.mu = 5.0; w.output.sigma = 0.8;
  w.output.lo = 1; w.output.hi = 1024;
  int64_t arr[8];
  int32_t pr[8], out[8], rk[8], st = -1;
  check(e, fs_generate_workload(e, &w, 1, arr, pr, out, rk, &st), "fs_generate_workload");
  printf("workload status=%d", st);
  for (int i = 0; i < 8; i++) printf(" %lld:%d:%d", (long long)arr[i], pr[i], out[i]);
  printf("\n");

  /* ---- 3. route_tokens(T, 8, 2, "uniform", seed) ---- */
  const int64_t tokens[3] = {17, 1, 300};
  const uint64_t seeds[3] = {3, 4, 3735928559ull};
  int32_t counts[3 * 8], rst[3];
  check(e, fs_route_tokens(e, tokens, seeds, 3, 8, 2, FS_ROUTE_UNIFORM, 0.3, counts, rst),
        "fs_route_tokens");
  for (int c = 0; c < 3; c++) {
    printf("route status=%d counts", rst[c]);
    for (int j = 0; j < 8; j++) printf(" %d", counts[c * 8 + j]);
    printf("\n");
  }
  fs_destroy(e);
  return 0;
}
