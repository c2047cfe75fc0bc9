// spmv_tiled_b.cu — tiled Heisenberg SpMV, L = 17..22.
#include "spmv_tiled.cuh"

SK_TILED_RANGE(launch_tiled_b, SK_TILED_CASE(17) SK_TILED_CASE(18) SK_TILED_CASE(19) SK_TILED_CASE(20) SK_TILED_CASE(21) SK_TILED_CASE(22))
