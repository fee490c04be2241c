// fused multi-species kernels for 4 species (see dgb_msflux_impl.cuh)
#define DGB_NSPEC 4
#include "dgb_msflux_impl.cuh"
