// spmv_tiled_a.cu — tiled Heisenberg SpMV, L = 11..16.
#include "spmv_tiled.cuh"

SK_TILED_RANGE(launch_tiled_a, SK_TILED_CASE(11) SK_TILED_CASE(12) SK_TILED_CASE(13) SK_TILED_CASE(14) SK_TILED_CASE(15) SK_TILED_CASE(16))
