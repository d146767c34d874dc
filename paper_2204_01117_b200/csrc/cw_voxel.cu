// Voxelizer (grid.py:233-325) -- placeholder until the device voxelizer lands.
#include "../../include/citywind_b200.h"

extern "C" int cw_voxelize(cw_ctx*, const cw_object*, int, const double*, const int*, int,
                           const signed char*, signed char*, double*, double*, int*, void*) {
  return CW_ERR_INVALID;
}
