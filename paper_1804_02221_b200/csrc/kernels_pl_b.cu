// kernels_pl_b.cu — P-part line stage kernel for N+1 in [9, 12] (see stage_pl.cuh)
#define PL_N1_LO 9
#define PL_N1_HI 12
#define PL_UPLOAD pl_upload_ops_b
#define PL_LAUNCH launch_pl_stage_b
#include "kernels_pl.cuh"
