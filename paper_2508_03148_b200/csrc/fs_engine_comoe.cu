// fs_engine_comoe.cu -- the sweep kernel for co-located MoE instances with top_k <= 3
// (C5's Mixtral family): the PD and AF handlers compiled out (fs_sim.cuh FS_MODES),
// which leaves 251 registers and no spills (255 with spills for all modes), only the
// top-(k+1) <= 4 routing templates (FS_KCAP_MAX: 239 registers), and Philox rounds
// unrolled by two. C5 step: 218-223 (all-modes kernel) -> 212-215 (co-located)
// -> 207-209 ms.
#define FS_LEARNED 0
#define FS_SIM_NS comoe
#define FS_MODES 1
#define FS_KCAP_MAX 4
#ifndef FS_PHILOX_UNROLL
#define FS_PHILOX_UNROLL 2
#endif
#include "fs_sim.cuh"
