// fused multi-species kernels for 2 species (see dgb_msflux_impl.cuh)
#define DGB_NSPEC 2
#include "dgb_msflux_impl.cuh"
