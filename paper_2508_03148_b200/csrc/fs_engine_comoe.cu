// fs_engine_comoe.cu -- the sweep kernel for co-located MoE instances only: the PD
// and AF handlers compiled out (fs_sim.cuh FS_MODES), which leaves the routing
// loop and the co-located DES step 251 registers with no spills (255 with spills
// for all modes): the C5 sweep's MoE wave, 221-224 -> 216-219 ms per step.
#define FS_LEARNED 0
#define FS_SIM_NS comoe
#define FS_MODES 1
#include "fs_sim.cuh"
