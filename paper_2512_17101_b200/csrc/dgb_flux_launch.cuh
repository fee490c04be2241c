// Launch configuration of the flux-arrangement kernels (k_nsflux3 + k_nsdiv8 / k_nsdiv3), shared by the
// translation units that instantiate them: dgb_nsflux.cu (single-species, DGB_NSPEC = 0) and dgb_msflux{2,3,4}.cu (the
// multi-species operator: the same templates compiled once more per species count, DGB_NSPEC = 2, 3, 4).
#pragma once
#include "dgb_internal.h"
#include "dgb_kernels_flux.cuh"
#include "dgb_kernels_tma.cuh"

#include <cstdlib>
#include <string>

namespace {

// Measured on B200 (profiles/r01_flux_variants.md): pass 1 is fastest with 12 warps (164 registers, four
// face nodes per lane in flight), pass 2 with 8 warps (235 registers, no spills, NB = 2).
#ifndef DGB_DIV_KERNEL_DEFAULT
#define DGB_DIV_KERNEL_DEFAULT 8          // TMA-staged pass 2 (profiles/r02_pass2_tma.md)
#endif
#ifndef DGB_FLUX_WARPS
#define DGB_FLUX_WARPS 12
#endif
#ifndef DGB_FLUX_WARPS_MS          // mixtures: the pointwise phase is heavier; 12 warps (168 registers) spill
#define DGB_FLUX_WARPS_MS 8
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
  // registers are allocated per SM sub-partition: 9-11 warps get the 168 registers of 12 without being 12, so a
  // configuration that shared memory limits below 12 warps runs 8 (255 registers) rather than 9-11 with spills
  static constexpr int NWF_fit = fit_warps(flux_fixed, flux_per, DGB_NSPEC > 0 ? DGB_FLUX_WARPS_MS : DGB_FLUX_WARPS);
  static constexpr int NWF = (NWF_fit >= 12 || NWF_fit <= 8) ? NWF_fit : 8;
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


// ---- TMA-staged pass 2 (k_nsdiv8, dgb_kernels_tma.cuh) ----------------------------------------------------
#ifndef DGB_DIV8_WARPS
#define DGB_DIV8_WARPS 8          // measured (3D p3, n=94, profiles/r02_pass2_tma.md): 8 warps with all 4 rounds in flight 6.69 ms,
                                  // 8 warps NB 2 7.86 ms, 10 warps NB 1 8.34 ms, 12 warps NB 1 8.56 ms
#endif
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// 2-D tensor (x = element*Np + node, y = plane) over `nplanes` planes of `width` doubles, `stride` doubles apart;
// box = boxw x boxh doubles, no swizzle (the box lands as [plane][x]), out-of-range reads give zeros
bool make_plane_map(CUtensorMap* m, const double* base, long long width, int nplanes, long long stride, int boxw, int boxh) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || (((uintptr_t)base) & 15) || (stride * 8) % 16 != 0 || boxw > 256 || boxh > 256 || width <= 0) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)width, (cuuint64_t)nplanes};
  cuuint64_t gstr[1] = {(cuuint64_t)stride * 8};
  cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)boxh};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DIM, int P> struct Cfg8 {
  static constexpr int KW = DIM == 3 ? 3 : 4;
  static constexpr size_t per = sizeof(dgb::Div8Warp<DIM, P, KW>);
  static constexpr size_t fixed = sizeof(dgb::Div8Smem<DIM, P, KW, 1>) - per;
  static constexpr int NW = fit_warps(fixed, per, DGB_DIV8_WARPS);
};

// returns 1 when the arrays cannot be described to the TMA unit (alignment): the caller falls back to k_nsdiv3
template <int DIM, int P>
int launch_div8(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                const dgb::Epilogue& ep, const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st, bool* ok) {
  using C = Cfg8<DIM, P>;
  using EL = dgb::ElemT<DIM, P>;
  using BX = dgb::TmaBox<DIM, P, C::KW>;
  *ok = false;
  const long long E = d->dev.E, width = E * EL::NP;
  if (width >= (1LL << 31) || !d->dev.gidx) return DGB_OK;
  CUtensorMap mq, mt, ml;
  if (!make_plane_map(&mq, q, width, EL::C, width, BX::BOXW, EL::C)) return DGB_OK;
  if (!make_plane_map(&mt, T, width, BX::NPL_T, width, BX::BOXW, BX::NPL_T)) return DGB_OK;
  if (!make_plane_map(&ml, T + (long long)dgb::FluxT<DIM, P>::LAMPL * width, width, 1, width, BX::BOXW, 1)) return DGB_OK;
  *ok = true;
  auto kern = d->dev.G > 0 ? dgb::k_nsdiv8<DIM, P, C::KW, C::NW, true> : dgb::k_nsdiv8<DIM, P, C::KW, C::NW, false>;
  const size_t smem = sizeof(dgb::Div8Smem<DIM, P, C::KW, C::NW>);
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured[2];
  if (!configured[d->dev.G > 0]()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured[d->dev.G > 0]() = true; }
  const long long need = (nwb + C::NW - 1) / C::NW;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters + 1, 0, sizeof(unsigned long long), st));
  dgb::GatherPlanes<EL::C> gp;
  for (int c = 0; c < EL::C; ++c) { gp.q[c] = q + c * width; gp.t[c] = T + c * width; }
  gp.lam = T + (long long)dgb::FluxT<DIM, P>::LAMPL * width;
  kern<<<grid, C::NW * 32, smem, st>>>(d->dev, mq, mt, ml, q, T, ghost, Tghost, ep, ph, ebeg, eend, nwb, d->counters + 1, gp);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

template <int DIM, int P>
int launch_div_any(const dgb_disc* d, const double* q, const double* T, const double* ghost, const double* Tghost,
                   const dgb::Epilogue& ep, const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st, int which) {
  if (which == 8) {
    bool ok = false;
    const int rc = launch_div8<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebeg, eend, st, &ok);
    if (rc != DGB_OK || ok) return rc;
  }
  return launch_div<DIM, P>(d, q, T, ghost, Tghost, ep, ph, ebeg, eend, st);
}

// DGB_DIV_KERNEL selects the pass-2 kernel at run time: 8 = TMA-staged k_nsdiv8 (falls back to 3 when the arrays
// cannot be described to the TMA unit), 3 = k_nsdiv3 (cp.async staging).  The role-split k_nsdiv7 of round 2
// (measured slower, profiles/r02_pass2_experiments.md) was retired with the sum planes.
int div_kernel() { return env_int("DGB_DIV_KERNEL", DGB_DIV_KERNEL_DEFAULT); }   // read per launch: tests toggle it

#ifdef DGB_ONLY_3D_P3   // fast kernel-tuning builds (scripts/ab_variants.py)
#define DGB_FOR_EACH_ELEMENT(X) X(3, 3)
#else
#define DGB_FOR_EACH_ELEMENT(X) X(2, 1) X(2, 2) X(2, 3) X(2, 4) X(3, 1) X(3, 2) X(3, 3) X(3, 4)
#endif

void make_phys(dgb::Phys& ph, int C, const double* qfar, const double* phys) {
  ph = dgb::Phys{};
  ph.gamma = phys ? phys[0] : 1.4; ph.mu = phys ? phys[1] : 0.0; ph.kappa = phys ? phys[2] : 0.0;
  ph.rgas = phys ? phys[3] : 1.0;
  for (int c = 0; c < dgb::DIM_MAX_FIELDS; ++c) ph.qfar[c] = (qfar && c < C) ? qfar[c] : 0.0;
}

int check_flux_args(const dgb_disc* d, const void* ghost, const void* a, const void* b) {
  if (!d) return dgb_fail(DGB_ERR_INVALID, "null handle");
  if (!d->dev.jac) return dgb_fail(DGB_ERR_INVALID, "dgb_disc_set_jacobian has not been called on this handle");
  if (d->dev.G > 0 && !ghost) return dgb_fail(DGB_ERR_INVALID, "discretisation has ghost elements but no ghost array was given");
  if ((((uintptr_t)a) | ((uintptr_t)b)) & 15) return dgb_fail(DGB_ERR_INVALID, "device arrays must be 16-byte aligned");
  return DGB_OK;
}

}  // namespace
