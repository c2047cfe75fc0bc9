// spmv_tiled_d.cu — tiled Heisenberg SpMV, L = 29..34.
#include "spmv_tiled.cuh"

SK_TILED_RANGE(launch_tiled_d, SK_TILED_CASE(29) SK_TILED_CASE(30) SK_TILED_CASE(31) SK_TILED_CASE(32) SK_TILED_CASE(33) SK_TILED_CASE(34))
