// kernels_pl_c.cu — P-part line stage kernel for N+1 in [13, 16] (see stage_pl.cuh)
#define PL_N1_LO 13
#define PL_N1_HI 16
#define PL_UPLOAD pl_upload_ops_c
#define PL_LAUNCH launch_pl_stage_c
#include "kernels_pl.cuh"
