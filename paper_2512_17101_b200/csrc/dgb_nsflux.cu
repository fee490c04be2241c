// C ABI of the Navier-Stokes flux arrangement (dg_ns_flux + dg_ns_div, operators.py) and its
// launch configuration.  Kernels: dgb_kernels_flux.cuh.
#include "dgb_internal.h"
#include "dgb_kernels_flux.cuh"
#include "dgb_kernels_div7.cuh"

#include <cstdlib>
#include <string>

namespace {

// Measured on B200 (profiles/r01_flux_variants.md): pass 1 is fastest with 12 warps (164 registers, four
// face nodes per lane in flight), pass 2 with 8 warps (235 registers, no spills, NB = 2).
#ifndef DGB_DIV_KERNEL_DEFAULT
#define DGB_DIV_KERNEL_DEFAULT 3
#endif
#ifndef DGB_FLUX_WARPS
#define DGB_FLUX_WARPS 12
#endif
#ifndef DGB_DIV_WARPS
#define DGB_DIV_WARPS 8
#endif
constexpr int kSmemBudget = 232448 - 1024;   // 227 KB usable per CTA minus the 1 KB system reserve
constexpr int fit_warps(size_t fixed, size_t per_warp, int cap) {
  int n = (int)((kSmemBudget - fixed) / per_warp);
  return n < 1 ? 1 : (n > cap ? cap : n);
}

template <int DIM, int P> struct CfgF {
  static constexpr int KW = DIM == 3 ? 3 : 4;
  static constexpr size_t flux_per = sizeof(dgb::Flux3Warp<DIM, P, KW>);
  static constexpr size_t flux_fixed = sizeof(dgb::Flux3Smem<DIM, P, KW, 1>) - flux_per;
  static constexpr int NWF = fit_warps(flux_fixed, flux_per, DGB_FLUX_WARPS);
  static constexpr size_t div_per = sizeof(dgb::Div3Warp<DIM, P, KW>);
  static constexpr size_t div_fixed = sizeof(dgb::Div3Smem<DIM, P, KW, 1>) - div_per;
  static constexpr int NWD = fit_warps(div_fixed, div_per, DGB_DIV_WARPS);
};

int env_int(const char* name, int dflt) { const char* e = getenv(name); return e ? atoi(e) : dflt; }

template <int DIM, int P>
int launch_flux(const dgb_disc* d, const double* q, const double* ghost, double* T, const dgb::Phys& ph,
                long long ebeg, long long eend, cudaStream_t st) {
  using C = CfgF<DIM, P>;
  // GH = false: no ghost elements (single partition): the ghost/owned selects vanish from the gathers
  auto kern = d->dev.G > 0 ? dgb::k_nsflux3<DIM, P, C::KW, C::NWF, true> : dgb::k_nsflux3<DIM, P, C::KW, C::NWF, false>;
  const size_t smem = sizeof(dgb::Flux3Smem<DIM, P, C::KW, C::NWF>);
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured[2];
  if (!configured[d->dev.G > 0]()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured[d->dev.G > 0]() = true; }
  const long long need = (nwb + C::NWF - 1) / C::NWF;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters, 0, sizeof(unsigned long long), st));
  kern<<<grid, C::NWF * 32, smem, st>>>(d->dev, q, ghost, T, ph, ebeg, eend, nwb, d->counters);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

template <int DIM, int P>
int launch_div(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
               const dgb::Epilogue& ep, const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st) {
  using C = CfgF<DIM, P>;
  auto kern = d->dev.G > 0 ? dgb::k_nsdiv3<DIM, P, C::KW, C::NWD, true> : dgb::k_nsdiv3<DIM, P, C::KW, C::NWD, false>;
  const size_t smem = sizeof(dgb::Div3Smem<DIM, P, C::KW, C::NWD>);
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured[2];
  if (!configured[d->dev.G > 0]()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured[d->dev.G > 0]() = true; }
  const long long need = (nwb + C::NWD - 1) / C::NWD;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters + 1, 0, sizeof(unsigned long long), st));
  kern<<<grid, C::NWD * 32, smem, st>>>(d->dev, q, T, ghost, Tghost, ep, ph, ebeg, eend, nwb, d->counters + 1);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}


// ---- role-split pass 2 (k_nsdiv7, dgb_kernels_div7.cuh): 4 consumer warps + NPROD producer warps ----
#ifndef DGB_DIV7_PRODUCERS
#define DGB_DIV7_PRODUCERS 8
#endif
#ifndef DGB_DIV7_NB
#define DGB_DIV7_NB 1
#endif
#ifndef DGB_DIV7_WREGS
#define DGB_DIV7_WREGS 76          // doubles of W fragments a consumer lane may keep in registers
#endif
template <int DIM, int P> struct Cfg7 {
  using EL = dgb::ElemT<DIM, P>;
  static constexpr int KW = DIM == 3 ? 3 : 4;
  static constexpr int per_tile = EL::KV / 4 + EL::KF / 4;
  static constexpr int NIR = DGB_DIV7_WREGS / per_tile < EL::NI ? DGB_DIV7_WREGS / per_tile : EL::NI;
  static constexpr size_t per = sizeof(dgb::Div7Prod<DIM, P, KW>);
  static constexpr size_t fixed = sizeof(dgb::Div7Smem<DIM, P, KW, 1, NIR>) - per;
  static constexpr int NPROD = fit_warps(fixed, per, DGB_DIV7_PRODUCERS);
};

template <int DIM, int P>
int launch_div7(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                const dgb::Epilogue& ep, const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st) {
  using C = Cfg7<DIM, P>;
  auto kern = d->dev.G > 0 ? dgb::k_nsdiv7<DIM, P, C::KW, C::NPROD, C::NIR, DGB_DIV7_NB, true>
                           : dgb::k_nsdiv7<DIM, P, C::KW, C::NPROD, C::NIR, DGB_DIV7_NB, false>;
  const size_t smem = sizeof(dgb::Div7Smem<DIM, P, C::KW, C::NPROD, C::NIR>);
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured[2];
  if (!configured[d->dev.G > 0]()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured[d->dev.G > 0]() = true; }
  const long long need = (nwb + C::NPROD - 1) / C::NPROD;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters + 1, 0, sizeof(unsigned long long), st));
  kern<<<grid, 128 + 128 * ((C::NPROD + 3) / 4), smem, st>>>(d->dev, q, T, ghost, Tghost, ep, ph, ebeg, eend, nwb, d->counters + 1);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

// DGB_DIV_KERNEL selects the pass-2 kernel at run time: 7 = role-split k_nsdiv7, 3 = warp-autonomous k_nsdiv3
int div_kernel() { return env_int("DGB_DIV_KERNEL", DGB_DIV_KERNEL_DEFAULT); }   // read per launch: tests toggle it

#ifdef DGB_ONLY_3D_P3   // fast kernel-tuning builds (scripts/ab_variants.py)
#define DGB_FOR_EACH_ELEMENT(X) X(3, 3)
#else
#define DGB_FOR_EACH_ELEMENT(X) X(2, 1) X(2, 2) X(2, 3) X(2, 4) X(3, 1) X(3, 2) X(3, 3) X(3, 4)
#endif

void make_phys(dgb::Phys& ph, int C, const double* qfar, const double* phys) {
  ph.gamma = phys ? phys[0] : 1.4; ph.mu = phys ? phys[1] : 0.0; ph.kappa = phys ? phys[2] : 0.0;
  ph.rgas = phys ? phys[3] : 1.0;
  for (int c = 0; c < 5; ++c) ph.qfar[c] = (qfar && c < C) ? qfar[c] : 0.0;
}

__global__ void k_face_jacobians(const double* __restrict__ fscale, const double* __restrict__ jac, long long E,
                                 int Nf, double* __restrict__ sj, double* __restrict__ rj) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= E * Nf) return;
  const long long e = n / Nf;
  sj[n] = fscale[n] * jac[e];
  if (n == e * Nf) rj[e] = 1.0 / jac[e];
}

int check_flux_args(const dgb_disc* d, const void* ghost, const void* a, const void* b) {
  if (!d) return dgb_fail(DGB_ERR_INVALID, "null handle");
  if (!d->dev.jac) return dgb_fail(DGB_ERR_INVALID, "dgb_disc_set_jacobian has not been called on this handle");
  if (d->dev.G > 0 && !ghost) return dgb_fail(DGB_ERR_INVALID, "discretisation has ghost elements but no ghost array was given");
  if ((((uintptr_t)a) | ((uintptr_t)b)) & 15) return dgb_fail(DGB_ERR_INVALID, "device arrays must be 16-byte aligned");
  return DGB_OK;
}

}  // namespace

#ifndef DGB_EULER_WARPS
#define DGB_EULER_WARPS 12
#endif
namespace {
template <int DIM, int P> struct CfgE {
  static constexpr int KW = DIM == 3 ? 3 : 4;
  static constexpr size_t per = sizeof(dgb::Euler4Warp<DIM, P, KW>);
  static constexpr size_t fixed = sizeof(dgb::Euler4Smem<DIM, P, KW, 1>) - per;
  static constexpr int NW = fit_warps(fixed, per, DGB_EULER_WARPS);
};

template <int DIM, int P>
int launch_euler4(const dgb_disc* d, const double* q, const double* ghost, const dgb::Epilogue& ep, const dgb::Phys& ph,
                  long long ebeg, long long eend, cudaStream_t st) {
  using C = CfgE<DIM, P>;
  auto kern = d->dev.G > 0 ? dgb::k_euler4<DIM, P, C::KW, C::NW, true> : dgb::k_euler4<DIM, P, C::KW, C::NW, false>;
  const size_t smem = sizeof(dgb::Euler4Smem<DIM, P, C::KW, C::NW>);
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured[2];
  if (!configured[d->dev.G > 0]()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured[d->dev.G > 0]() = true; }
  const long long need = (nwb + C::NW - 1) / C::NW;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters + 1, 0, sizeof(unsigned long long), st));
  kern<<<grid, C::NW * 32, smem, st>>>(d->dev, q, ghost, ep, ph, ebeg, eend, nwb, d->counters + 1);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}
}  // namespace

int dgb_launch_euler4(const dgb_disc* d, const double* q, const double* ghost, const dgb::Epilogue& ep,
                      const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st) {
  if (eend < 0) eend = d->dev.E;
  if ((((uintptr_t)q) | ((uintptr_t)ep.out1)) & 15) return dgb_fail(DGB_ERR_INVALID, "device arrays must be 16-byte aligned");
#define X(DIM, P) if (d->dim == DIM && d->order == P) return launch_euler4<DIM, P>(d, q, ghost, ep, ph, ebeg, eend, st);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return dgb_fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

int dgb_disc_free_jacobian(dgb_disc* d) {
  if (d) { cudaFree(d->sj); cudaFree(d->rj); d->sj = d->rj = nullptr; }
  return DGB_OK;
}

extern "C" {

int dgb_disc_set_jacobian(dgb_disc* d, const double* jac_dev, void* stream) {
  if (!d || !jac_dev) return dgb_fail(DGB_ERR_INVALID, "null handle or Jacobian array");
  dgb_disc_free_jacobian(d);
  const long long E = d->dev.E, n = E * d->Nf;
  DGB_CUDA(cudaMalloc((void**)&d->sj, sizeof(double) * (size_t)(n ? n : 1)));
  DGB_CUDA(cudaMalloc((void**)&d->rj, sizeof(double) * (size_t)(E ? E : 1)));
  if (n) {
    k_face_jacobians<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d->dev.fscale, jac_dev, E, d->Nf,
                                                                                    d->sj, d->rj);
    DGB_CUDA(cudaGetLastError());
  }
  d->dev.jac = jac_dev; d->dev.sj = d->sj; d->dev.rj = d->rj;
  return DGB_OK;
}

static int check_range(const dgb_disc* d, int64_t ebegin, int64_t eend) {
  if (ebegin < 0 || eend > d->dev.E || ebegin > eend) return dgb_fail(DGB_ERR_INVALID, "element range outside [0, E]");
  return DGB_OK;
}

int dgb_ns_flux_range(const dgb_disc* d, const double* q, const double* ghost, double* T, const double* qfar,
                      const double* phys, int64_t ebegin, int64_t eend, void* stream) {
  int rc = check_flux_args(d, ghost, q, T); if (rc) return rc;
  if ((rc = check_range(d, ebegin, eend))) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
#define X(DIM, P) if (d->dim == DIM && d->order == P) return launch_flux<DIM, P>(d, q, ghost, T, ph, ebegin, eend, (cudaStream_t)stream);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return dgb_fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

int dgb_ns_flux(const dgb_disc* d, const double* q, const double* ghost, double* T, const double* qfar,
                const double* phys, void* stream) {
  if (!d) return dgb_fail(DGB_ERR_INVALID, "null handle");
  return dgb_ns_flux_range(d, q, ghost, T, qfar, phys, 0, d->dev.E, stream);
}

static int ns_div_impl(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                       const dgb::Epilogue& ep, const double* qfar, const double* phys, void* stream,
                       int64_t ebegin = 0, int64_t eend = -1) {
  int rc = check_flux_args(d, ghost, q, T); if (rc) return rc;
  if (eend < 0) eend = d->dev.E;
  if ((rc = check_range(d, ebegin, eend))) return rc;
  if (d->dev.G > 0 && !Tghost) return dgb_fail(DGB_ERR_INVALID, "ghost elements need the ghost flux planes");
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
#define X(DIM, P) if (d->dim == DIM && d->order == P)                                                         \
    return div_kernel() == 7 ? launch_div7<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebegin, eend, (cudaStream_t)stream) \
                             : launch_div<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebegin, eend, (cudaStream_t)stream);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return dgb_fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

int dgb_ns_div(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
               double* rhs, const double* qfar, const double* phys, void* stream) {
  if (!rhs) return dgb_fail(DGB_ERR_INVALID, "null output");
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return ns_div_impl(d, q, T, ghost, Tghost, ep, qfar, phys, stream);
}

int dgb_ns_div_range(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                     double* rhs, const double* qfar, const double* phys, int64_t ebegin, int64_t eend, void* stream) {
  if (!rhs) return dgb_fail(DGB_ERR_INVALID, "null output");
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return ns_div_impl(d, q, T, ghost, Tghost, ep, qfar, phys, stream, ebegin, eend);
}

int dgb_ns_div_rk(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                  const double* x1, double* out1, const double* x2, double* out2, const double* rk,
                  const double* qfar, const double* phys, void* stream) {
  if (!out1 || !rk) return dgb_fail(DGB_ERR_INVALID, "out1 and rk are required");
  if (out1 == q || (out2 && out2 == q) || (x2 && out1 == x2))
    return dgb_fail(DGB_ERR_INVALID, "RK outputs must not alias the stage input q (neighbours still read it)");
  if (out2 && !x2) return dgb_fail(DGB_ERR_INVALID, "out2 needs x2");
  if ((((uintptr_t)x1) | ((uintptr_t)out1) | ((uintptr_t)x2) | ((uintptr_t)out2)) & 15)
    return dgb_fail(DGB_ERR_INVALID, "RK operands and outputs must be 16-byte aligned");
  dgb::Epilogue ep{x1, out1, x2, out2, rk[0], rk[1], rk[2], rk[3]};
  return ns_div_impl(d, q, T, ghost, Tghost, ep, qfar, phys, stream);
}

}  // extern "C"
