// The flex kernels for the compact voxel-record format (kernels.h): the same
// source compiled with GD_TU_COMPACT=1, launchers suffixed _cp.
#define GD_TU_COMPACT 1
#include "flex.cu"
