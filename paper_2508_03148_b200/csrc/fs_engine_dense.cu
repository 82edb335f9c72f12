// fs_engine_dense.cu -- the analytic simulation kernel with the MoE paths compiled
// out, for dense instances (a batch without MoE, or the dense wave of a mixed
// one): no routing code in the instruction stream (fs_sim.cuh FS_DENSE_ONLY).
#define FS_LEARNED 0
#define FS_SIM_NS dense
#define FS_DENSE_ONLY 1
#define FS_SIM_MIN_BLOCKS 3  // 176 -> <= 168 registers: three CTAs (12 warps) per SM
#include "fs_sim.cuh"
