// fused multi-species kernels for 3 species (see dgb_msflux_impl.cuh)
#define DGB_NSPEC 3
#include "dgb_msflux_impl.cuh"
