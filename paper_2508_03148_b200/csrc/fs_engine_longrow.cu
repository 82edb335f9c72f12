// fs_engine_longrow.cu -- the analytic simulation kernel for batches whose MoE
// rows are long (>= 64 experts per lane segment, e.g. DeepSeek-V3's 256): the
// Philox rounds run unrolled there (fs_sim.cuh FS_LONG_ROW_UNROLL). A separate
// variant because the extra code costs the small-expert sweep kernel ~10%.
#define FS_LEARNED 0
#define FS_SIM_NS longrow
#define FS_LONG_ROW_UNROLL 1
#define FS_TOPK_BRANCHFREE 1
#define FS_JOB_NOINLINE 0  // inline chunk loops: C4 EP 323 vs 350 ms, AF 437 vs 468 ms
#include "fs_sim.cuh"
