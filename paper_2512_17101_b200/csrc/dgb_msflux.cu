// Public entry points of the fused multi-species operator: dispatch on the species count (mixture[0]) to the
// translation unit that instantiates the kernel templates for it (dgb_msflux2.cu, dgb_msflux3.cu, dgb_msflux4.cu).
#include "dgb_internal.h"

#define DGB_MS_COUNTS(X) X(2) X(3) X(4)

extern "C" {

#define X(K)                                                                                                              \
  DGB_HIDDEN int dgb_ms_flux_range_ns##K(const dgb_disc*, const double*, const double*, double*, const double*, const double*, \
                                         const double*, int64_t, int64_t, void*);                                         \
  DGB_HIDDEN int dgb_ms_div_range_ns##K(const dgb_disc*, const double*, const double*, const double*, const double*, double*, \
                                        const double*, const double*, const double*, int64_t, int64_t, void*);            \
  DGB_HIDDEN int dgb_ms_div_rk_ns##K(const dgb_disc*, const double*, const double*, const double*, const double*,        \
                                     const double*, double*, const double*, double*, const double*, const double*,        \
                                     const double*, const double*, void*);
DGB_MS_COUNTS(X)
#undef X

static int no_count(const double* mixture) {
  if (!mixture) return dgb_fail(DGB_ERR_INVALID, "qfar, transport and mixture are required");
  return dgb_fail(DGB_ERR_INVALID, "the fused multi-species kernels are built for 2, 3 and 4 species");
}

int dgb_ms_flux_range(const dgb_disc* d, const double* q, const double* ghost, double* T, const double* qfar,
                      const double* transport, const double* mixture, int64_t ebegin, int64_t eend, void* stream) {
#define X(K) if (mixture && (int)mixture[0] == K) return dgb_ms_flux_range_ns##K(d, q, ghost, T, qfar, transport, mixture, ebegin, eend, stream);
  DGB_MS_COUNTS(X)
#undef X
  return no_count(mixture);
}

int dgb_ms_div_range(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                     double* rhs, const double* qfar, const double* transport, const double* mixture,
                     int64_t ebegin, int64_t eend, void* stream) {
#define X(K) if (mixture && (int)mixture[0] == K) return dgb_ms_div_range_ns##K(d, q, T, ghost, Tghost, rhs, qfar, transport, mixture, ebegin, eend, stream);
  DGB_MS_COUNTS(X)
#undef X
  return no_count(mixture);
}

int dgb_ms_div_rk(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                  const double* x1, double* out1, const double* x2, double* out2, const double* rk,
                  const double* qfar, const double* transport, const double* mixture, void* stream) {
#define X(K) if (mixture && (int)mixture[0] == K) return dgb_ms_div_rk_ns##K(d, q, T, ghost, Tghost, x1, out1, x2, out2, rk, qfar, transport, mixture, stream);
  DGB_MS_COUNTS(X)
#undef X
  return no_count(mixture);
}

}  // extern "C"
