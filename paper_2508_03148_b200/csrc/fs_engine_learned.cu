// fs_engine_learned.cu -- the simulation kernel variant with the learned
// attention model call sites (costmodel/model.py:313-321); see fs_engine.cu.
#define FS_LEARNED 1
#define FS_SIM_NS learned
#include "fs_sim.cuh"
