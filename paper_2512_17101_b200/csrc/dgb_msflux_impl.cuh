// Multi-species reactive Navier-Stokes (BASELINE configs[4], multispecies.py: dg_ms_flux / dg_ms_div) on the fused
// kernels of the flux arrangement.  Included by dgb_msflux2.cu / dgb_msflux3.cu / dgb_msflux4.cu, each of which compiles
// the SAME templates (k_nsflux3, k_nsdiv8, k_nsdiv3) once more with DGB_NSPEC extra species fields -- C = dim + 2 +
// DGB_NSPEC conserved fields, the mixture physics of dgb_kernels.cuh, the temperature gradient by the chain rule, the
// Arrhenius source in the store epilogue of pass 2.  The namespace of the templates is renamed per count so that the
// instantiation sets cannot collide in libdgb200.so; the plain structs the handle carries (DiscDev, Phys, Epilogue)
// do not depend on the field count.  dgb_msflux.cu holds the public entry points and dispatches on the count.
#ifndef DGB_NSPEC
#error "define DGB_NSPEC before including dgb_msflux_impl.cuh"
#endif
#define DGB_MS_CAT_(a, b) a##b
#define DGB_MS_CAT(a, b) DGB_MS_CAT_(a, b)
#define dgb DGB_MS_CAT(dgbms, DGB_NSPEC)
#define DGB_MS_FN(name) DGB_MS_CAT(name##_ns, DGB_NSPEC)
#include "dgb_flux_launch.cuh"

namespace {

constexpr int kNS = DGB_NSPEC;

// mixture = [ns, R[ns], cv[ns], h0[ns], A, Ta, reactant, product]; transport = [mu, kappa, D]
int make_ms_phys(dgb::Phys& ph, int dim, const double* qfar, const double* transport, const double* mixture) {
  if (!qfar || !transport || !mixture) return dgb_fail(DGB_ERR_INVALID, "qfar, transport and mixture are required");
  if ((int)mixture[0] != kNS) return dgb_fail(DGB_ERR_INVALID, "species count does not match this instantiation");
  ph = dgb::Phys{};
  ph.mu = transport[0]; ph.kappa = transport[1]; ph.dspec = transport[2];
  for (int c = 0; c < dim + 2 + kNS; ++c) ph.qfar[c] = qfar[c];
  for (int k = 0; k < kNS; ++k) { ph.mR[k] = mixture[1 + k]; ph.mcv[k] = mixture[1 + kNS + k]; ph.mh0[k] = mixture[1 + 2 * kNS + k]; }
  ph.arr_A = mixture[1 + 3 * kNS]; ph.arr_Ta = mixture[2 + 3 * kNS];
  ph.ra = (int)mixture[3 + 3 * kNS]; ph.rb = (int)mixture[4 + 3 * kNS];
  if (ph.ra < 0 || ph.ra >= kNS || ph.rb < 0 || ph.rb >= kNS) return dgb_fail(DGB_ERR_INVALID, "reaction species out of range");
  return DGB_OK;
}

int check_range(const dgb_disc* d, int64_t ebegin, int64_t eend) {
  if (ebegin < 0 || eend > d->dev.E || ebegin > eend) return dgb_fail(DGB_ERR_INVALID, "element range outside [0, E]");
  return DGB_OK;
}

}  // namespace

extern "C" {

DGB_HIDDEN int DGB_MS_FN(dgb_ms_flux_range)(const dgb_disc* d, const double* q, const double* ghost, double* T, const double* qfar,
                      const double* transport, const double* mixture, int64_t ebegin, int64_t eend, void* stream) {
  int rc = check_flux_args(d, ghost, q, T); if (rc) return rc;
  if (eend < 0) eend = d->dev.E;
  if ((rc = check_range(d, ebegin, eend))) return rc;
  dgb::Phys ph; if ((rc = make_ms_phys(ph, d->dim, qfar, transport, mixture))) return rc;
#define X(DIM, P) if (d->dim == DIM && d->order == P) return launch_flux<DIM, P>(d, q, ghost, T, ph, ebegin, eend, (cudaStream_t)stream);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return dgb_fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

static int ms_div_impl(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                       const dgb::Epilogue& ep, const double* qfar, const double* transport, const double* mixture,
                       int64_t ebegin, int64_t eend, void* stream) {
  int rc = check_flux_args(d, ghost, q, T); if (rc) return rc;
  if (eend < 0) eend = d->dev.E;
  if ((rc = check_range(d, ebegin, eend))) return rc;
  if (d->dev.G > 0 && !Tghost) return dgb_fail(DGB_ERR_INVALID, "ghost elements need the ghost flux planes");
  dgb::Phys ph; if ((rc = make_ms_phys(ph, d->dim, qfar, transport, mixture))) return rc;
#define X(DIM, P) if (d->dim == DIM && d->order == P)                                                         \
    return launch_div_any<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebegin, eend, (cudaStream_t)stream, div_kernel());
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return dgb_fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

DGB_HIDDEN int DGB_MS_FN(dgb_ms_div_range)(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                     double* rhs, const double* qfar, const double* transport, const double* mixture,
                     int64_t ebegin, int64_t eend, void* stream) {
  if (!rhs) return dgb_fail(DGB_ERR_INVALID, "null output");
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return ms_div_impl(d, q, T, ghost, Tghost, ep, qfar, transport, mixture, ebegin, eend, stream);
}

// pass 2 with the RK stage update fused into the store: out1 = rk[0]*x1 + rk[1]*rhs, out2 = rk[2]*x2 + rk[3]*rhs
DGB_HIDDEN int DGB_MS_FN(dgb_ms_div_rk)(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                  const double* x1, double* out1, const double* x2, double* out2, const double* rk,
                  const double* qfar, const double* transport, const double* mixture, void* stream) {
  if (!out1 || !rk) return dgb_fail(DGB_ERR_INVALID, "out1 and rk are required");
  if (out1 == q || (out2 && out2 == q) || (x2 && out1 == x2))
    return dgb_fail(DGB_ERR_INVALID, "RK outputs must not alias the stage input q (neighbours still read it)");
  if (out2 && !x2) return dgb_fail(DGB_ERR_INVALID, "out2 needs x2");
  if ((((uintptr_t)x1) | ((uintptr_t)out1) | ((uintptr_t)x2) | ((uintptr_t)out2)) & 15)
    return dgb_fail(DGB_ERR_INVALID, "RK operands and outputs must be 16-byte aligned");
  dgb::Epilogue ep{x1, out1, x2, out2, rk[0], rk[1], rk[2], rk[3]};
  return ms_div_impl(d, q, T, ghost, Tghost, ep, qfar, transport, mixture, 0, -1, stream);
}

}  // extern "C"
