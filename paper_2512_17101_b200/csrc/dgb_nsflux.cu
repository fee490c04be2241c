// C ABI of the Navier-Stokes flux arrangement (dg_ns_flux + dg_ns_div, operators.py), the single-pass Euler
// kernel and the face Jacobians.  Kernels: dgb_kernels_flux.cuh, dgb_kernels_tma.cuh; launch configuration:
// dgb_flux_launch.cuh.
#include "dgb_flux_launch.cuh"

namespace {
__global__ void k_face_jacobians(const double* __restrict__ fscale, const double* __restrict__ jac, long long E,
                                 int Nf, double* __restrict__ sj, double* __restrict__ rj) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= E * Nf) return;
  const long long e = n / Nf;
  sj[n] = fscale[n] * jac[e];
  if (n == e * Nf) rj[e] = 1.0 / jac[e];
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
    return launch_div_any<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebegin, eend, (cudaStream_t)stream, div_kernel());
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

int dgb_ns_div_rk_range(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                        const double* x1, double* out1, const double* x2, double* out2, const double* rk,
                        const double* qfar, const double* phys, int64_t ebegin, int64_t eend, void* stream) {
  if (!out1 || !rk) return dgb_fail(DGB_ERR_INVALID, "out1 and rk are required");
  if (out1 == q || (out2 && out2 == q) || (x2 && out1 == x2))
    return dgb_fail(DGB_ERR_INVALID, "RK outputs must not alias the stage input q (neighbours still read it)");
  if (out2 && !x2) return dgb_fail(DGB_ERR_INVALID, "out2 needs x2");
  if ((((uintptr_t)x1) | ((uintptr_t)out1) | ((uintptr_t)x2) | ((uintptr_t)out2)) & 15)
    return dgb_fail(DGB_ERR_INVALID, "RK operands and outputs must be 16-byte aligned");
  dgb::Epilogue ep{x1, out1, x2, out2, rk[0], rk[1], rk[2], rk[3]};
  return ns_div_impl(d, q, T, ghost, Tghost, ep, qfar, phys, stream, ebegin, eend);
}

int dgb_ns_div_rk(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                  const double* x1, double* out1, const double* x2, double* out2, const double* rk,
                  const double* qfar, const double* phys, void* stream) {
  return dgb_ns_div_rk_range(d, q, T, ghost, Tghost, x1, out1, x2, out2, rk, qfar, phys, 0, -1, stream);
}

}  // extern "C"
