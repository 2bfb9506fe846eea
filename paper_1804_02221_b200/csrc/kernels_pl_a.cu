// kernels_pl_a.cu — P-part line stage kernel for N+1 in [2, 8] (see stage_pl.cuh)
#define PL_N1_LO 2
#define PL_N1_HI 8
#define PL_UPLOAD pl_upload_ops_a
#define PL_LAUNCH launch_pl_stage_a
#include "kernels_pl.cuh"
