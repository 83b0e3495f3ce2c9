// ctw_kernels_wide.cu -- the frame kernel again, with 1024-thread CTAs (16 per
// lane): the launch shape for batches too small to fill the GPU, where
// per-lane frame latency is the metric (streaming steps). Same source as
// ctw_kernels.cu; only ctw_launch_decode_wide is exported from here and
// ctw_launch_decode dispatches to it.
#define CTW_BS 1024
#define CTW_WIDE 1
#include "ctw_kernels.cu"
