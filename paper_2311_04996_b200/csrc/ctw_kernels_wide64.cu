// ctw_kernels_wide64.cu -- the wide frame kernel (1024-thread CTAs, 16 per
// lane) compiled for ONE resident CTA per SM, i.e. with 64 registers per
// thread instead of 32 (the 32-register build spills ~260 B per thread).
// Launches of up to one CTA per SM (n * 16 <= SMs: a streaming step's
// handful of lanes) take it; ctw_launch_decode dispatches.
#define CTW_BS 1024
#define CTW_WIDE 1
#define CTW_MINB 1
#define CTW_WIDE_FN ctw_launch_decode_wide64
#include "ctw_kernels.cu"
