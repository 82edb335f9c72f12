// Throughput of the integer multiply forms Philox4x64-10 can be built from, on
// this GPU: IMAD (32-bit low), IMAD.HI (32-bit high), IMAD.WIDE (32x32 -> 64),
// the 64-bit low product and __umul64hi. 8 independent chains per thread so the
// pipe, not latency, bounds each loop; ops per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_rates imad_rates.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t a[8];
  uint64_t w[8];
#pragma unroll
  for (int j = 0; j < 8; j++) { a[j] = seed + threadIdx.x * 8 + j; w[j] = a[j] * 0x9E3779B97F4A7C15ull; }
  const uint32_t m = 0xD2E7470Eu;
  const uint64_t M = 0xD2E7470EE14C6C93ull;
  for (int i = 0; i < kIters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (OP == 0) a[j] = a[j] * m + 0x1234567u;                      // IMAD
      if (OP == 1) a[j] = __umulhi(a[j], m) ^ (uint32_t)j;              // IMAD.HI
      if (OP == 2) w[j] = (uint64_t)(uint32_t)w[j] * m + (w[j] >> 32);  // IMAD.WIDE
      if (OP == 3) w[j] = w[j] * M + 1;                                 // 64-bit low
      if (OP == 4) w[j] = __umul64hi(w[j], M) ^ j;                      // 64-bit high
    }
  }
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) acc ^= a[j] ^ w[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)acc ^ (uint32_t)(acc >> 32);
}

template <int OP>
void run(const char* name, int nsm, uint32_t* d) {
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  const int blocks = nsm * 8, threads = 256;
  k<OP><<<blocks, threads>>>(d, 1);
  cudaEventRecord(s);
  k<OP><<<blocks, threads>>>(d, 2);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  const double ops = (double)blocks * threads * kIters * 8;
  const double per_sm_clk = ops / (ms * 1e-3) / nsm / (clk * 1e3);
  printf("{\"op\": \"%s\", \"ms\": %.3f, \"ops_per_clk_per_sm\": %.1f}\n", name, ms, per_sm_clk);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d;
  cudaMalloc(&d, (size_t)nsm * 8 * 256 * 4);
  run<0>("imad_lo32", nsm, d);
  run<1>("imad_hi32", nsm, d);
  run<2>("imad_wide32", nsm, d);
  run<3>("mul_lo64", nsm, d);
  run<4>("umul64hi", nsm, d);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
