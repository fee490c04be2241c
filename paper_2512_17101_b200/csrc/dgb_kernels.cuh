// Building blocks of the fused sm_100a kernels of the DG right-hand side (hot path, SURVEY.md §8a
// rows a1-a4): element constants, the packed connectivity word, the pointwise physics (mirrors
// operators.py line by line), the FP64 tensor-core contraction (mma.sync.m8n8k4.f64 -> DMMA.8x8x4;
// M = (field, element) columns, N = output node, K = (reference direction, node) / face node;
// replaces the Einsum nodes, adfg.py:563-608) and the (optionally RK-fused) store epilogue.
// DMMA was chosen over register-blocked DFMA on measured numbers (profiles/r01_fp64_peak.txt:
// 29.7 vs 22.6 TFLOP/s useful for this contraction shape).  The kernels themselves are in
// dgb_kernels_flux.cuh (default Navier-Stokes arrangement + Euler) and dgb_kernels_warp.cuh
// (gradient arrangement).  The first-generation CTA-phased kernels (round 1, variants 0-4) were
// retired in round 2; their measurements stay in profiles/r01_variants.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef DGB_STREAMING_STORES
#define DGB_STREAMING_STORES 0
#endif
// Number of species fields carried next to [rho, rho E, rho u]: 0 = single-species Euler / Navier-Stokes
// (libdgb200's default translation units); dgb_msflux{2,3,4}.cu compile the SAME kernel templates once more with
// DGB_NSPEC = 2, 3, 4 (and the namespace renamed per count) for the multi-species reactive operator (multispecies.py).
#ifndef DGB_NSPEC
#define DGB_NSPEC 0
#endif
#define DGB_MAX_SPECIES 4

namespace dgb {

constexpr int ceil_to(int x, int m) { return (x + m - 1) / m * m; }
// row stride (in doubles) that makes the 8x4 DMMA fragment loads bank-conflict free:
// stride mod 16 in {4, 12}
constexpr int ldpad(int k) { return (ceil_to(k, 4) % 8 == 4) ? ceil_to(k, 4) : ceil_to(k, 4) + 4; }

template <int DIM, int P>
struct ElemT {
  static constexpr int C = DIM + 2 + DGB_NSPEC;  // conserved fields
  static constexpr int CG = C;                   // fields whose BR1 gradient pass 1 needs (the temperature gradient of mixtures follows by the chain rule)
  static constexpr int NF = DIM + 1;
  static constexpr int NP = DIM == 2 ? (P + 1) * (P + 2) / 2 : (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NFP = DIM == 2 ? (P + 1) : (P + 1) * (P + 2) / 2;
  static constexpr int NFT = NF * NFP;
  static constexpr int NPERM = DIM == 2 ? 2 : 6;
  static constexpr int NPK = ceil_to(NP, 4);     // K extent of one reference direction
  static constexpr int NI = ceil_to(NP, 8) / 8;  // 8-wide output-node tiles
  static constexpr int NPR = NI * 8;             // padded output rows of every W
  static constexpr int KV = DIM * NPK;           // volume contraction length
  static constexpr int LDV = ldpad(KV);
  static constexpr int KF = ceil_to(NFT, 4);     // lift contraction length
  static constexpr int LDF = ldpad(KF);
  static constexpr int LDQ = ldpad(NPK);         // gradient pass: q rows / Sw_r blocks
  static constexpr int NFPK = ceil_to(NFP, 4);   // gradient pass: per-face K extent
  static constexpr int LDL = ldpad(NFPK);        // lift_f blocks
  static constexpr int LDS = ldpad(NF * NFPK);   // gradient pass: q* rows
  static constexpr int NS = DIM + NF;            // partial products per column in the gradient pass
};

#ifdef DGB_PHASE_TIMING
#define DGB_TICK(k) do { if (tid == 0) { long long t_ = clock64(); d.timing[blockIdx.x * 8 + (k)] += t_ - tlast; tlast = t_; } } while (0)
#else
#define DGB_TICK(k) do { } while (0)
#endif

constexpr int DIM_MAX_FIELDS = 3 + 2 + DGB_MAX_SPECIES;

struct DiscDev {
  long long* timing;     // [grid][8] per-phase cycle counters (debug builds only)
  long long E, G;
  const double* Wv;      // [NPR][LDV]
  const double* Wl;      // [NPR][LDF]
  const double* Wq;      // [DIM][NPR][LDQ]
  const double* Wf;      // [NF][NPR][LDL]
  const double* drdx;    // [DIM][DIM][E]
  const double* normals; // [DIM][E][NF]
  const double* fscale;  // [E][NF]
  const long long* conn; // [E][NF] packed
  const int* tables;     // face_nodes [NF][NFP] then face_perms [NPERM][NFP]
  const unsigned* gidx;  // [E][NF*NFP] gather map: node index (nb*NP + jp) of the matching neighbour node in the
                         // (owned | ghost) node space = the int64 map vmap_p of the API narrowed to 32 bits;
                         // null when (E+G)*NP does not fit
  // flux arrangement (dgb_kernels_flux.cuh), bound by dgb_disc_set_jacobian
  const double* jac;     // [E] volume Jacobian
  const double* sj;      // [E][NF] face Jacobian = fscale * jac
  const double* rj;      // [E] 1 / jac
  const double* Wv2;     // [NPR][LDV] volume matrix minus half the lifted own-side face term
};

struct Phys {
  double gamma, mu, kappa, rgas;
  double qfar[DIM_MAX_FIELDS];
  // mixture (multispecies.py: Mixture): species gas constants, heat capacities, formation enthalpies, Fick
  // diffusivity, one Arrhenius step species ra -> species rb
  double dspec, mR[DGB_MAX_SPECIES], mcv[DGB_MAX_SPECIES], mh0[DGB_MAX_SPECIES], arr_A, arr_Ta;
  int ra, rb;
};

struct Epilogue {   // out1 = a1*x1 + b1*rhs ; out2 = a2*x2 + b2*rhs
  const double* x1; double* out1; const double* x2; double* out2;
  double a1, b1, a2, b2;
};

// conn packing
__host__ __device__ inline long long conn_pack(long long nb, int nf, int perm, int bc) {
  return (nb & 0xffffffffLL) | ((long long)nf << 32) | ((long long)perm << 35) | ((long long)bc << 38);
}
#define DGB_CONN_NB(c) ((long long)((c) & 0xffffffffLL))
#define DGB_CONN_NF(c) ((int)(((c) >> 32) & 7))
#define DGB_CONN_PERM(c) ((int)(((c) >> 35) & 7))
#define DGB_CONN_BC(c) ((int)(((c) >> 38) & 3))

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// {{{ pointwise physics -- mirrors operators.py line by line

template <int DIM>
struct Prim { double rho, E, m[DIM], u[DIM], p, inv_rho; };

template <int DIM>
__device__ __forceinline__ void make_prim(const double (&q)[DIM + 2], double gamma, Prim<DIM>& s) {
  s.rho = q[0]; s.E = q[1];
  s.inv_rho = 1.0 / s.rho;
  double ke = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) { s.m[i] = q[2 + i]; s.u[i] = s.m[i] * s.inv_rho; ke += s.m[i] * s.u[i]; }
  s.p = (gamma - 1.0) * (s.E - 0.5 * ke);
}

template <int DIM>
__device__ __forceinline__ void inviscid_flux(const Prim<DIM>& s, double (&F)[DIM][DIM + 2]) {
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    F[x][0] = s.m[x];
    F[x][1] = s.u[x] * (s.E + s.p);
#pragma unroll
    for (int i = 0; i < DIM; ++i) F[x][2 + i] = s.m[i] * s.u[x] + (i == x ? s.p : 0.0);
  }
}

template <int DIM>
__device__ __forceinline__ void inviscid_normal_flux(const Prim<DIM>& s, const double (&n)[DIM],
                                                      double (&Fn)[DIM + 2]) {
  double mn = 0.0, un = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) { mn += s.m[i] * n[i]; un += s.u[i] * n[i]; }
  Fn[0] = mn;
  Fn[1] = un * (s.E + s.p);
#pragma unroll
  for (int i = 0; i < DIM; ++i) Fn[2 + i] = s.m[i] * un + s.p * n[i];
}

template <int DIM>
__device__ __forceinline__ double wavespeed(const Prim<DIM>& s, double gamma) {
  double v2 = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) v2 += s.u[i] * s.u[i];
  return sqrt(v2) + sqrt(gamma * s.p * s.inv_rho);
}

// g[x][c] = d q_c / d x_x ; Fv[x][c] (Fv[x][0] == 0)
template <int DIM>
__device__ __forceinline__ void viscous_flux(const Prim<DIM>& s, const double (&g)[DIM][DIM + 2],
                                             const Phys& ph, double (&Fv)[DIM][DIM + 2]) {
  double du[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int x = 0; x < DIM; ++x) du[i][x] = (g[x][2 + i] - s.u[i] * g[x][0]) * s.inv_rho;
  double div = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) div += du[i][i];
  const double etot = s.E * s.inv_rho;
  const double tfac = (ph.gamma - 1.0) / ph.rgas;
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    double de = (g[x][1] - etot * g[x][0]) * s.inv_rho;
#pragma unroll
    for (int i = 0; i < DIM; ++i) de -= s.u[i] * du[i][x];
    double work = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double t = ph.mu * (du[i][x] + du[x][i]);
      if (i == x) t -= (2.0 / 3.0) * ph.mu * div;
      Fv[x][2 + i] = t;
      work += s.u[i] * t;
    }
    Fv[x][0] = 0.0;
    Fv[x][1] = work + ph.kappa * (tfac * de);
  }
}

// (Fv . n)[c] directly, without forming the 3x5 tensor: ~65 FP64 ops instead of ~135
template <int DIM>
__device__ __forceinline__ void viscous_normal_flux(const Prim<DIM>& s, const double (&g)[DIM][DIM + 2],
                                                    const double (&n)[DIM], const Phys& ph,
                                                    double (&Fn)[DIM + 2]) {
  double gn[DIM + 2];                       // normal derivative of every conserved field
#pragma unroll
  for (int c = 0; c < DIM + 2; ++c) {
    gn[c] = g[0][c] * n[0];
#pragma unroll
    for (int x = 1; x < DIM; ++x) gn[c] += g[x][c] * n[x];
  }
  double un = 0.0, div = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) { un += s.u[i] * n[i]; div += g[i][2 + i] - s.u[i] * g[i][0]; }
  div *= s.inv_rho;
  double work = 0.0, udun = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    const double dun = (gn[2 + i] - s.u[i] * gn[0]) * s.inv_rho;        // sum_x du_i/dx_x n_x
    double dnu = -un * g[i][0];                                         // sum_x du_x/dx_i n_x
#pragma unroll
    for (int x = 0; x < DIM; ++x) dnu += n[x] * g[i][2 + x];
    dnu *= s.inv_rho;
    const double t = ph.mu * (dun + dnu) - (2.0 / 3.0) * ph.mu * div * n[i];
    Fn[2 + i] = t;
    work += s.u[i] * t;
    udun += s.u[i] * dun;
  }
  const double etot = s.E * s.inv_rho;
  const double den = (gn[1] - etot * gn[0]) * s.inv_rho - udun;
  Fn[0] = 0.0;
  Fn[1] = work + ph.kappa * (((ph.gamma - 1.0) / ph.rgas) * den);
}

// exterior state for boundary faces (operators.py:_bc_state)
template <int DIM, bool NOSLIP>
__device__ __forceinline__ void bc_state(int bc, const double (&qm)[DIM + 2], const double (&n)[DIM],
                                         const Phys& ph, double (&qp)[DIM + 2]) {
  if (bc == 1) {
#pragma unroll
    for (int c = 0; c < DIM + 2; ++c) qp[c] = ph.qfar[c];
  } else if (bc == 2) {
    qp[0] = qm[0]; qp[1] = qm[1];
    if (NOSLIP) {
#pragma unroll
      for (int i = 0; i < DIM; ++i) qp[2 + i] = -qm[2 + i];
    } else {
      double mn = 0.0;
#pragma unroll
      for (int i = 0; i < DIM; ++i) mn += qm[2 + i] * n[i];
#pragma unroll
      for (int i = 0; i < DIM; ++i) qp[2 + i] = qm[2 + i] - 2.0 * mn * n[i];
    }
  }
}

// }}}

// {{{ mixture physics (DGB_NSPEC > 0) -- mirrors multispecies.py line by line

#if DGB_NSPEC > 0
template <int DIM>
struct MsPrim { double rho, inv_rho, E, u[DIM], Y[DGB_NSPEC], T, p, R, cv; };

// multispecies.py: _thermo
template <int DIM>
__device__ __forceinline__ void ms_thermo(const double (&q)[DIM + 2 + DGB_NSPEC], const Phys& ph, MsPrim<DIM>& s) {
  s.rho = q[0]; s.E = q[1];
  s.inv_rho = 1.0 / s.rho;
  double ke = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) { s.u[i] = q[2 + i] * s.inv_rho; ke = i == 0 ? s.u[i] * s.u[i] : ke + s.u[i] * s.u[i]; }
  double R = 0.0, cv = 0.0, hf = 0.0;
#pragma unroll
  for (int k = 0; k < DGB_NSPEC; ++k) {
    s.Y[k] = q[2 + DIM + k] * s.inv_rho;
    R = k == 0 ? ph.mR[0] * s.Y[0] : R + ph.mR[k] * s.Y[k];
    cv = k == 0 ? ph.mcv[0] * s.Y[0] : cv + ph.mcv[k] * s.Y[k];
    hf = k == 0 ? ph.mh0[0] * s.Y[0] : hf + ph.mh0[k] * s.Y[k];
  }
  s.R = R; s.cv = cv;
  s.T = (s.E * s.inv_rho - 0.5 * ke - hf) / cv;
  s.p = s.rho * R * s.T;
}

// multispecies.py: _inviscid
template <int DIM>
__device__ __forceinline__ void ms_inviscid_flux(const double (&q)[DIM + 2 + DGB_NSPEC], const MsPrim<DIM>& s,
                                                 double (&F)[DIM][DIM + 2 + DGB_NSPEC]) {
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    F[x][0] = q[2 + x];
    F[x][1] = s.u[x] * (q[1] + s.p);
#pragma unroll
    for (int i = 0; i < DIM; ++i) F[x][2 + i] = q[2 + i] * s.u[x] + (i == x ? s.p : 0.0);
#pragma unroll
    for (int k = 0; k < DGB_NSPEC; ++k) F[x][2 + DIM + k] = q[2 + DIM + k] * s.u[x];
  }
}

template <int DIM>
__device__ __forceinline__ double ms_wavespeed(const MsPrim<DIM>& s) {
  double v2 = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) v2 += s.u[i] * s.u[i];
  return sqrt(v2) + sqrt((1.0 + s.R / s.cv) * s.p / s.rho);
}

// multispecies.py: _viscous; g[x][c] = d q_c / d x_x; velocity, mass-fraction and temperature gradients by the chain rule
template <int DIM>
__device__ __forceinline__ void ms_viscous_flux(const MsPrim<DIM>& s, const double (&g)[DIM][DIM + 2 + DGB_NSPEC],
                                                const Phys& ph, double (&Fv)[DIM][DIM + 2 + DGB_NSPEC]) {
  double du[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int x = 0; x < DIM; ++x) du[i][x] = (g[x][2 + i] - s.u[i] * g[x][0]) * s.inv_rho;
  double div = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i) div += du[i][i];
#pragma unroll
  for (int x = 0; x < DIM; ++x) {
    double work = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double t = ph.mu * (du[i][x] + du[x][i]);
      if (i == x) t -= (2.0 / 3.0) * ph.mu * div;
      Fv[x][2 + i] = t;
      work += s.u[i] * t;
    }
    double dY[DGB_NSPEC];
    double de = (g[x][1] - (s.E * s.inv_rho) * g[x][0]) * s.inv_rho;
#pragma unroll
    for (int i = 0; i < DIM; ++i) de -= s.u[i] * du[i][x];
#pragma unroll
    for (int k = 0; k < DGB_NSPEC; ++k) {
      dY[k] = (g[x][2 + DIM + k] - s.Y[k] * g[x][0]) * s.inv_rho;
      de -= (ph.mh0[k] + ph.mcv[k] * s.T) * dY[k];
    }
    double heat = ph.kappa * (de / s.cv);
#pragma unroll
    for (int k = 0; k < DGB_NSPEC; ++k) {
      const double jk = (s.rho * ph.dspec) * dY[k];              // = -J_k
      const double hk = ph.mh0[k] + (ph.mcv[k] + ph.mR[k]) * s.T;
      heat += hk * jk;
      Fv[x][2 + DIM + k] = jk;
    }
    Fv[x][0] = 0.0;
    Fv[x][1] = work + heat;
  }
}
#endif

// }}}

// {{{ what the flux-arrangement kernels call: single-species or mixture physics behind one interface

// total flux F = F_inv - F_visc at a node and the local wave speed
template <int DIM>
__device__ __forceinline__ void pw_total_flux(const double (&qq)[DIM + 2 + DGB_NSPEC],
                                              const double (&g)[DIM][DIM + 2 + DGB_NSPEC],
                                              const Phys& ph, double (&F)[DIM][DIM + 2 + DGB_NSPEC], double& lam) {
  constexpr int C = DIM + 2 + DGB_NSPEC;
  double Fv[DIM][C];
#if DGB_NSPEC > 0
  MsPrim<DIM> s;
  ms_thermo<DIM>(qq, ph, s);
  ms_inviscid_flux<DIM>(qq, s, F);
  ms_viscous_flux<DIM>(s, g, ph, Fv);
  lam = ms_wavespeed<DIM>(s);
#else
  Prim<DIM> s;
  make_prim<DIM>(qq, ph.gamma, s);
  inviscid_flux<DIM>(s, F);
  viscous_flux<DIM>(s, g, ph, Fv);
  lam = wavespeed<DIM>(s, ph.gamma);
#endif
#pragma unroll
  for (int x = 0; x < DIM; ++x)
#pragma unroll
    for (int c = 1; c < C; ++c) F[x][c] -= Fv[x][c];
}

#if DGB_NSPEC > 0
template <int DIM>
__device__ __forceinline__ double pw_temperature(const double (&q)[DIM + 2 + DGB_NSPEC], const Phys& ph) {
  MsPrim<DIM> s;
  ms_thermo<DIM>(q, ph, s);
  return s.T;
}
// Arrhenius rate of the one reaction step (multispecies.py: _ms_pass2)
template <int DIM>
__device__ __forceinline__ double pw_arrhenius(const double (&q)[DIM + 2 + DGB_NSPEC], const Phys& ph) {
  return ph.arr_A * q[2 + DIM + ph.ra] * exp((-ph.arr_Ta) / pw_temperature<DIM>(q, ph));
}
#endif

// exterior state of a boundary face for the BR1 gradient (pass 1): qp is overwritten
template <int DIM>
__device__ __forceinline__ void pw_exterior_state(int bc, const double (&qm)[DIM + 2 + DGB_NSPEC], const double (&n)[DIM],
                                                  const Phys& ph, double (&qp)[DIM + 2 + DGB_NSPEC]) {
#if DGB_NSPEC > 0
#pragma unroll
  for (int c = 0; c < DIM + 2 + DGB_NSPEC; ++c) qp[c] = ph.qfar[c];       // far-field is the only boundary kind
#else
  bc_state<DIM, true>(bc, qm, n, ph, qp);
#endif
}

// }}}

// {{{ tensor-core contraction: acc[mt][ni] += X[col tile mt][k] * W[node tile ni][k]

template <int NI, int MT>
__device__ __forceinline__ void mma_block(double (&acc)[MT][NI][2], const double* __restrict__ Xs, int ldx,
                                          const double* __restrict__ Ws, int ldw, int ksteps, int lane) {
  const int r = lane >> 2, kq = lane & 3;
  const double* xp = Xs + r * ldx + kq;
  const double* wp = Ws + r * ldw + kq;
#pragma unroll 5
  for (int ks = 0; ks < ksteps; ++ks) {
    double a[MT], b[NI];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) a[mt] = xp[mt * 8 * ldx + ks * 4];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) b[ni] = wp[ni * 8 * ldw + ks * 4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) dmma884(acc[mt][ni][0], acc[mt][ni][1], a[mt], b[ni]);
  }
}

// }}}

// shared epilogue store of one accumulator fragment pair
template <int NP>
__device__ __forceinline__ void store_pair(const Epilogue& ep, long long idx, int i, double v0, double v1) {
  // idx = flat index of node i of this column; i even
  if ((NP % 2 == 0)) {
    if (i < NP) {
      double2 o;
      if (ep.x1) { double2 x = *reinterpret_cast<const double2*>(ep.x1 + idx); o.x = ep.a1 * x.x + ep.b1 * v0; o.y = ep.a1 * x.y + ep.b1 * v1; }
      else { o.x = ep.b1 * v0; o.y = ep.b1 * v1; }
#if DGB_STREAMING_STORES
      __stcs(reinterpret_cast<double2*>(ep.out1 + idx), o);      // written once, not re-read by this kernel: keep L2 for the gathers
#else
      *reinterpret_cast<double2*>(ep.out1 + idx) = o;
#endif
      if (ep.out2) {
        double2 x = *reinterpret_cast<const double2*>(ep.x2 + idx);
        double2 o2; o2.x = ep.a2 * x.x + ep.b2 * v0; o2.y = ep.a2 * x.y + ep.b2 * v1;
#if DGB_STREAMING_STORES
        __stcs(reinterpret_cast<double2*>(ep.out2 + idx), o2);
#else
        *reinterpret_cast<double2*>(ep.out2 + idx) = o2;
#endif
      }
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (i + h < NP) {
        double v = h ? v1 : v0;
        double o = ep.x1 ? ep.a1 * ep.x1[idx + h] + ep.b1 * v : ep.b1 * v;
        ep.out1[idx + h] = o;
        if (ep.out2) ep.out2[idx + h] = ep.a2 * ep.x2[idx + h] + ep.b2 * v;
      }
    }
  }
}

// Store epilogue of a warp's block: v[mt][ni] = the two values of node pair (ni*8 + 2*(lane&3)) of column mt*8 + lane/4.
// RK-fused stores with even Np: ALL operands x1 / x2 of the lane are loaded first and the results stored afterwards
// -- written as load, store, load, store ... the compiler must keep that order (out1 / out2 may alias x1 / x2: the
// accumulator of the scheme is updated in place) and every pair waits for its own round trip to L2
// (DeviceRK4 at 31 M DOFs: 24.5 -> 21.7 ms per step).
template <int NP, int KW, int NCOL, int NTILE, int NI>
__device__ __forceinline__ void store_block(const Epilogue& ep, const double (&v)[NTILE][NI][2], long long E,
                                            long long e0, int nel, int lane) {
  const bool rk_batch = (NP % 2 == 0) && ep.x1 != nullptr;
  if (rk_batch) {
    double2 xa[NTILE][NI], xb[NTILE][NI];
#pragma unroll
    for (int mt = 0; mt < NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      const bool ok = col < NCOL && e < nel;
      const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const int i = ni * 8 + 2 * (lane & 3);
        xa[mt][ni] = make_double2(0.0, 0.0); xb[mt][ni] = make_double2(0.0, 0.0);
        if (ok && i < NP) {
          xa[mt][ni] = *reinterpret_cast<const double2*>(ep.x1 + rowbase + i);
          if (ep.out2) xb[mt][ni] = *reinterpret_cast<const double2*>(ep.x2 + rowbase + i);
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < NCOL && e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int i = ni * 8 + 2 * (lane & 3);
          if (i < NP) {
            *reinterpret_cast<double2*>(ep.out1 + rowbase + i) =
                make_double2(ep.a1 * xa[mt][ni].x + ep.b1 * v[mt][ni][0], ep.a1 * xa[mt][ni].y + ep.b1 * v[mt][ni][1]);
            if (ep.out2)
              *reinterpret_cast<double2*>(ep.out2 + rowbase + i) =
                  make_double2(ep.a2 * xb[mt][ni].x + ep.b2 * v[mt][ni][0], ep.a2 * xb[mt][ni].y + ep.b2 * v[mt][ni][1]);
          }
        }
      }
    }
    return;
  }
#pragma unroll
  for (int mt = 0; mt < NTILE; ++mt) {
    const int col = mt * 8 + (lane >> 2);
    const int c = col / KW, e = col - c * KW;
    if (col < NCOL && e < nel) {
      const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const int i = ni * 8 + 2 * (lane & 3);
        store_pair<NP>(ep, rowbase + i, i, v[mt][ni][0], v[mt][ni][1]);
      }
    }
  }
}

}  // namespace dgb
