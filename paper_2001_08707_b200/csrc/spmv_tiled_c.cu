// spmv_tiled_c.cu — tiled Heisenberg SpMV, L = 23..28.
#include "spmv_tiled.cuh"

SK_TILED_RANGE(launch_tiled_c, SK_TILED_CASE(23) SK_TILED_CASE(24) SK_TILED_CASE(25) SK_TILED_CASE(26) SK_TILED_CASE(27) SK_TILED_CASE(28))
