// fs_engine.cu -- the analytic-cost simulation kernel (the sweep's path), the
// SHA-256 midstate kernel, and the host dispatch between the two compiled
// variants of fs_sim.cuh. Instances that use a learned attention model run in
// the variant compiled in fs_engine_learned.cu, so the analytic kernel keeps
// its register allocation (the learned call sites cost it spills otherwise).
#define FS_LEARNED 0
#define FS_SIM_NS analytic
#include "fs_sim.cuh"

namespace fs {

__global__ void midstate_kernel(const fs_seed_prefix* pf, uint32_t* mid, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t h[8];
  if (pf[i].len > FS_MAX_PREFIX_BYTES) {  // long prefix: the host hashed its leading blocks
    for (int k = 0; k < 8; k++) h[k] = pf[i].mid[k];
  } else {
    sha256_midstate(pf[i].bytes, pf[i].mid_blocks, h);
  }
  for (int k = 0; k < 8; k++) mid[(int64_t)i * 8 + k] = h[k];
}

void launch_midstate(const fs_seed_prefix* prefixes, uint32_t* mid, int n, void* stream) {
  if (n <= 0) return;
  midstate_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(prefixes, mid, n);
}

int simulation_slots(int n_sms, int n_inst, int variant, int ctas_per_sm, bool helpers) {
  if (variant == kSimLearned) return learned::slots(n_sms, n_inst, ctas_per_sm, helpers);
  if (variant == kSimLongRow) return longrow::slots(n_sms, n_inst, ctas_per_sm, helpers);
  if (variant == kSimDense) return dense::slots(n_sms, n_inst, ctas_per_sm, helpers);
  if (variant == kSimCoMoe) return comoe::slots(n_sms, n_inst, ctas_per_sm, helpers);
  return analytic::slots(n_sms, n_inst, ctas_per_sm, helpers);
}

int launch_simulation(const EngineParams& p, int variant, void* stream) {
  if (variant == kSimLearned) return learned::launch(p, stream);
  if (variant == kSimLongRow) return longrow::launch(p, stream);
  if (variant == kSimDense) return dense::launch(p, stream);
  if (variant == kSimCoMoe) return comoe::launch(p, stream);
  return analytic::launch(p, stream);
}

}  // namespace fs
