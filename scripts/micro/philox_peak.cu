// Measured peak of the routing core on B200: Philox4x64-10 blocks -> 32-bit
// surrogate keys -> top-(k+1) of each E-draw row -> expert tally. This is the
// denominator of the MoE routing roofline (router keys/s against what the
// SMs' integer pipes sustain for exactly this instruction mix), measured at
// several occupancies and ILP settings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o philox_peak philox_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct U4 { uint64_t v[4]; };

template <int UNROLL>
__device__ __forceinline__ U4 philox(uint64_t c0, uint64_t k0, uint64_t k1) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll UNROLL
  for (int r = 0; r < 10; r++) {
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    uint64_t lo0 = m0 * c0, hi0 = __umul64hi(m0, c0);
    uint64_t lo1 = m1 * c2, hi1 = __umul64hi(m1, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull;
  }
  U4 o; o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3; return o;
}

// two blocks, rounds interleaved
template <int UNROLL>
__device__ __forceinline__ void philox2(uint64_t ca, uint64_t cb, uint64_t k0, uint64_t k1, U4& A, U4& B) {
  uint64_t a0 = ca, a1 = 0, a2 = 0, a3 = 0, b0 = cb, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll UNROLL
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

__device__ __forceinline__ void ins3(uint32_t (&t)[3], uint32_t x) {
#pragma unroll
  for (int q = 0; q < 3; q++) { const uint32_t lo = min(t[q], x); x = max(t[q], x); t[q] = lo; }
}

// E = 8 experts, k = 2: a row is two Philox blocks; lane = row.
template <int UNROLL, int ILP>
__global__ void route_rows(int64_t rows, uint64_t k0, uint64_t k1, int* counts) {
  __shared__ int hist[8];
  if (threadIdx.x < 8) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += stride) {
    uint32_t t[3] = {~0u, ~0u, ~0u};
    U4 A, B;
    if (ILP == 2) {
      philox2<UNROLL>(2 * r + 1, 2 * r + 2, k0, k1, A, B);
    } else {
      A = philox<UNROLL>(2 * r + 1, k0, k1);
      B = philox<UNROLL>(2 * r + 2, k0, k1);
    }
#pragma unroll
    for (int j = 0; j < 4; j++) ins3(t, ((uint32_t)(A.v[j] >> 32) & ~7u) | j);
#pragma unroll
    for (int j = 0; j < 4; j++) ins3(t, ((uint32_t)(B.v[j] >> 32) & ~7u) | (4 + j));
    atomicAdd(&hist[t[0] & 7], 1);
    atomicAdd(&hist[t[1] & 7], 1);
  }
  __syncthreads();
  if (threadIdx.x < 8) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

template <int UNROLL, int ILP>
void run(const char* name, int threads, int ctas_per_sm, int nsm, int64_t rows, int* d_counts) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = nsm * ctas_per_sm;
  int maxc = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxc, route_rows<UNROLL, ILP>, threads, 0);
  route_rows<UNROLL, ILP><<<grid, threads>>>(rows / 16, 1, 2, d_counts);  // warm-up
  cudaEventRecord(a);
  route_rows<UNROLL, ILP><<<grid, threads>>>(rows, 0x1234, 0x5678, d_counts);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double keys = rows * 8.0;
  printf("{\"kernel\": \"%s\", \"warps_per_sm\": %d, \"occ_ctas\": %d, \"ms\": %.3f, "
         "\"G_keys_per_s\": %.1f, \"G_blocks_per_s\": %.1f}\n",
         name, threads / 32 * ctas_per_sm, maxc, ms, keys / ms / 1e6, keys / 4 / ms / 1e6);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* d;
  cudaMalloc(&d, 8 * sizeof(int));
  const int64_t rows = 1ll << 29;  // 4.3 G keys
  for (int w : {8, 16, 32, 48, 64}) {
    run<1, 1>("rolled", 128, w / 4, nsm, rows, d);
    run<10, 1>("unrolled", 128, w / 4, nsm, rows, d);
    run<1, 2>("rolled_ilp2", 128, w / 4, nsm, rows, d);
    run<10, 2>("unrolled_ilp2", 128, w / 4, nsm, rows, d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
