// Fused sm_100a kernels of the DG right-hand side (hot path).
//
// One persistent CTA processes blocks of K elements.  Per block:
//   phase 0  stage per-element geometry + compressed connectivity in shared memory
//   phase 1  pointwise volume flux at every node, contracted with the affine metric
//            -> Gs[col][r*NPK + j]           (replaces IndexLambda chains, frontend.py:374-410)
//   phase 2  face gather through the compressed index maps + boundary states + Rusanov /
//            central numerical flux -> Fs[col][f*NFP + m]   (replaces Indexing, adfg.py:502-560)
//   phase 3  out[col][i] = sum_k Wv[i][k] Gs[col][k] + sum_k Wl[i][k] Fs[col][k]
//            with FP64 tensor-core tiles (mma.sync.m8n8k4.f64 -> DMMA.8x8x4), M = (field,
//            element) columns, N = output node, K = (ref. direction, node) / face node;
//            replaces the Einsum nodes (adfg.py:563-608, reduction lowering scalar_ir.py:294-312)
//            and is followed directly by the (optionally RK-fused) store.
// col = c*K + e_local, so a column's row in shared memory has the same [field][element][node]
// order as global memory.  DMMA was chosen over register-blocked DFMA on measured numbers
// (profiles/r01_fp64_peak.txt: 29.7 vs 22.6 TFLOP/s useful for this contraction shape).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef DGB_STREAMING_STORES
#define DGB_STREAMING_STORES 0
#endif

namespace dgb {

constexpr int ceil_to(int x, int m) { return (x + m - 1) / m * m; }
// row stride (in doubles) that makes the 8x4 DMMA fragment loads bank-conflict free:
// stride mod 16 in {4, 12}
constexpr int ldpad(int k) { return (ceil_to(k, 4) % 8 == 4) ? ceil_to(k, 4) : ceil_to(k, 4) + 4; }

template <int DIM, int P>
struct ElemT {
  static constexpr int C = DIM + 2;
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
  // flux arrangement (dgb_kernels_flux.cuh), bound by dgb_disc_set_jacobian
  const double* jac;     // [E] volume Jacobian
  const double* sj;      // [E][NF] face Jacobian = fscale * jac
  const double* rj;      // [E] 1 / jac
  const double* Wv2;     // [NPR][LDV] volume matrix minus half the lifted own-side face term
};

struct Phys { double gamma, mu, kappa, rgas; double qfar[5]; };

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

// {{{ compute-warp barrier and the L2 prefetch helper warp

template <int NT>
__device__ __forceinline__ void compute_sync() {   // named barrier over the NT compute threads only
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Software prefetch into L2, issued by the compute threads themselves (non-blocking):
//  * at the top of iteration b: the own rows + geometry of block b+1 (addresses are arithmetic);
//  * the packed connectivity of block b+2 is loaded into a register at the top of iteration b and
//    used after phase 1 to prefetch that block's face-neighbour rows, so the load never stalls.
// The compute phases then see L2-hit latency instead of HBM latency.
template <int DIM, int P, int K, int NPLANES>
__device__ __forceinline__ void prefetch_own(const DiscDev& d, const double* p0, const double* p1,
                                             long long e0, int nel, int tid, int nthreads) {
  using EL = ElemT<DIM, P>;
  constexpr int NP = EL::NP, NF = EL::NF;
  const long long E = d.E;
  const int nlines = (nel * NP * 8 + 127) / 128 + 1;
  for (int n = tid; n < NPLANES * nlines; n += nthreads) {
    const int pl = n / nlines, ln = n - pl * nlines;
    const double* base = pl < EL::C ? p0 : p1;
    const int plane = pl < EL::C ? pl : pl - EL::C;
    prefetch_l2(reinterpret_cast<const char*>(base + ((long long)plane * E + e0) * NP) + ln * 128);
  }
  if (tid < DIM * DIM) prefetch_l2(d.drdx + (long long)tid * E + e0);
  if (tid < DIM) {
    prefetch_l2(d.normals + ((long long)tid * E + e0) * NF);
    prefetch_l2(reinterpret_cast<const char*>(d.normals + ((long long)tid * E + e0) * NF) + 128);
  }
  if (tid == DIM) { prefetch_l2(d.fscale + e0 * NF); prefetch_l2(d.conn + e0 * NF); }
}

template <int DIM, int P, int NPLANES>
__device__ __forceinline__ void prefetch_nbr(const DiscDev& d, const double* p0, const double* p1,
                                             long long cn, long long e0, int nel) {
  using EL = ElemT<DIM, P>;
  constexpr int NP = EL::NP;
  const long long E = d.E;
  const long long nb = DGB_CONN_NB(cn);
  if (DGB_CONN_BC(cn) != 0 || nb >= E || (nb >= e0 && nb < e0 + nel)) return;
#pragma unroll 4
  for (int pl = 0; pl < NPLANES; ++pl) {
    const double* base = pl < EL::C ? p0 : p1;
    const int plane = pl < EL::C ? pl : pl - EL::C;
    const char* a = reinterpret_cast<const char*>(base + ((long long)plane * E + nb) * NP);
    prefetch_l2(a);
    prefetch_l2(a + NP * 8 - 8);
  }
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

template <int DIM, int P, int K>
struct GeoSmem {
  using EL = ElemT<DIM, P>;
  double drdx[DIM * DIM][K];
  double nrm[DIM][K][EL::NF];
  double fsc[K][EL::NF];
  long long conn[K][EL::NF];
};

template <int DIM, int P, int K>
__device__ __forceinline__ void stage_geo(GeoSmem<DIM, P, K>& g, const DiscDev& d, long long e0, int nel,
                                          int tid, int nthreads) {
  using EL = ElemT<DIM, P>;
  for (int n = tid; n < DIM * DIM * K; n += nthreads) {
    int rx = n / K, e = n % K;
    g.drdx[rx][e] = e < nel ? d.drdx[(long long)rx * d.E + e0 + e] : 0.0;
  }
  for (int n = tid; n < DIM * K * EL::NF; n += nthreads) {
    int x = n / (K * EL::NF), ef = n % (K * EL::NF);
    int e = ef / EL::NF;
    g.nrm[x][0][ef] = e < nel ? d.normals[((long long)x * d.E + e0) * EL::NF + ef] : 0.0;
  }
  for (int n = tid; n < K * EL::NF; n += nthreads) {
    int e = n / EL::NF;
    g.fsc[0][n] = e < nel ? d.fscale[e0 * EL::NF + n] : 0.0;
    g.conn[0][n] = e < nel ? d.conn[e0 * EL::NF + n] : 0LL;
  }
}

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

// ------------------------------------------------------------------------------------------
// Euler (VISCOUS=false) and Navier-Stokes second pass (VISCOUS=true) right-hand side
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int K, int NW, int MT, bool VISCOUS>
struct RhsSmem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  double Gs[EL::C * K * EL::LDV];
  double Fs[EL::C * K * EL::LDF];
  double Lam[K * EL::NP];
  GeoSmem<DIM, P, K> geo;
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int K, int NW, int MT, bool VISCOUS, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
k_rhs(DiscDev d, const double* __restrict__ q, const double* __restrict__ gq,
      const double* __restrict__ ghost, const double* __restrict__ gghost,
      Epilogue ep, Phys ph, int nblocks) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NW * 32;
  static_assert((C * K) % 8 == 0, "columns per block must be a multiple of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<RhsSmem<DIM, P, K, NW, MT, VISCOUS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < C * K * EL::LDV; n += NT) S.Gs[n] = 0.0;
  for (int n = tid; n < C * K * EL::LDF; n += NT) S.Fs[n] = 0.0;
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  compute_sync<NT>();   // the zero fill above must not race with the first block's staging writes

#ifdef DGB_PHASE_TIMING
  long long tlast = clock64();
#endif
  for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    stage_geo<DIM, P, K>(S.geo, d, e0, nel, tid, NT);
    compute_sync<NT>();
    DGB_TICK(0);

    // ---- phase 1: volume flux ------------------------------------------------------------
    for (int n = tid; n < nel * NP; n += NT) {
      const int e = n / NP, j = n - e * NP;
      double qq[C];
#pragma unroll
      for (int c = 0; c < C; ++c) qq[c] = q[((long long)c * E + e0 + e) * NP + j];
      Prim<DIM> s;
      make_prim<DIM>(qq, ph.gamma, s);
      double F[DIM][C];
      inviscid_flux<DIM>(s, F);
      if (VISCOUS) {
        double g[DIM][C], Fv[DIM][C];
#pragma unroll
        for (int x = 0; x < DIM; ++x)
#pragma unroll
          for (int c = 0; c < C; ++c) g[x][c] = gq[((long long)(x * C + c) * E + e0 + e) * NP + j];
        viscous_flux<DIM>(s, g, ph, Fv);
#pragma unroll
        for (int x = 0; x < DIM; ++x)
#pragma unroll
          for (int c = 1; c < C; ++c) F[x][c] -= Fv[x][c];
      }
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        double m[DIM];
#pragma unroll
        for (int x = 0; x < DIM; ++x) m[x] = S.geo.drdx[r * DIM + x][e];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int x = 0; x < DIM; ++x) acc += m[x] * F[x][c];
          S.Gs[(c * K + e) * EL::LDV + r * EL::NPK + j] = acc;
        }
      }
      S.Lam[n] = wavespeed<DIM>(s, ph.gamma);
    }
    compute_sync<NT>();
    DGB_TICK(1);

    // ---- phase 2: face gather + numerical flux --------------------------------------------
    // Own side: the scaled normal flux fscale*(F.n)^- needs no recomputation.  On an affine simplex
    // with face f opposite vertex f and r_k = 2*lambda_k - 1,
    //     fscale_f * n_f . F = (f == 0) ? sum_r G_r : -G_{f-1},     G_r = sum_x drdx[r][x] F_x,
    // and G_r at the face node is already in shared memory from phase 1 (as is the wave speed).
    // Only the neighbour side is evaluated pointwise.
    for (int n = tid; n < nel * NFT; n += NT) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const long long cn = S.geo.conn[e][f];
      const long long nb = DGB_CONN_NB(cn);
      const int nf = DGB_CONN_NF(cn), pid = DGB_CONN_PERM(cn), bc = DGB_CONN_BC(cn);
      const int jm = S.fn[f * NFP + m];
      const int jp = S.fn[nf * NFP + S.perm[pid * NFP + m]];
      double nrm[DIM];
#pragma unroll
      for (int x = 0; x < DIM; ++x) nrm[x] = S.geo.nrm[x][e][f];
      const double fs = S.geo.fsc[e][f];
      double qm[C], qp[C];
      const bool in_ghost = nb >= E;
      const double* pbase = in_ghost ? ghost : q;
      const long long pE = in_ghost ? G : E;
      const long long pe = in_ghost ? nb - E : nb;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qm[c] = q[((long long)c * E + e0 + e) * NP + jm];
        qp[c] = pbase[((long long)c * pE + pe) * NP + jp];
      }
      double gp[DIM][C];
      if (VISCOUS) {
        const double* gbase = in_ghost ? gghost : gq;
#pragma unroll
        for (int x = 0; x < DIM; ++x)
#pragma unroll
          for (int c = 0; c < C; ++c) gp[x][c] = gbase[((long long)(x * C + c) * pE + pe) * NP + jp];
      }
      bc_state<DIM, VISCOUS>(bc, qm, nrm, ph, qp);
      Prim<DIM> sp_;
      make_prim<DIM>(qp, ph.gamma, sp_);
      double fnp[C];
      inviscid_normal_flux<DIM>(sp_, nrm, fnp);
      const double lam = fmax(S.Lam[e * NP + jm], wavespeed<DIM>(sp_, ph.gamma));
      if (VISCOUS) {
        double fvn[C];
        // boundary faces: the viscous flux is the interior one, Fv(q-, grad q-) (operators.py)
        if (bc != 0) make_prim<DIM>(qm, ph.gamma, sp_);
        viscous_normal_flux<DIM>(sp_, gp, nrm, ph, fvn);
#pragma unroll
        for (int c = 1; c < C; ++c) fnp[c] -= fvn[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double* grow = S.Gs + (c * K + e) * EL::LDV + jm;
        double own;                       // fscale * (F^- . n), inviscid minus viscous
        if (f == 0) {
          own = grow[0];
#pragma unroll
          for (int r = 1; r < DIM; ++r) own += grow[r * EL::NPK];
        } else {
          own = -grow[(f - 1) * EL::NPK];
        }
        S.Fs[(c * K + e) * EL::LDF + fm] = -0.5 * (own + fs * (fnp[c] + lam * (qm[c] - qp[c])));
      }
    }
    compute_sync<NT>();
    DGB_TICK(2);

    // ---- phase 3: tensor-core contraction + (RK-fused) store -------------------------------
    constexpr int NTILES = C * K / 8;
    for (int t0 = warp * MT; t0 < NTILES; t0 += NW * MT) {
      __syncwarp();
      double acc[MT][EL::NI][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
      // tiles beyond NTILES (when NTILES % MT != 0) alias the last tile; their stores are masked
      const int tbase = (t0 + MT <= NTILES) ? t0 : NTILES - MT;
      mma_block<EL::NI, MT>(acc, S.Gs + tbase * 8 * EL::LDV, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
      mma_block<EL::NI, MT>(acc, S.Fs + tbase * 8 * EL::LDF, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int tile = tbase + mt;
        if (tile < t0) continue;          // aliased duplicate
        const int col = tile * 8 + (lane >> 2);
        const int c = col / K, e = col - c * K;
        if (e >= nel) continue;
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) {
          const int i = ni * 8 + 2 * (lane & 3);
          store_pair<NP>(ep, rowbase + i, i, acc[mt][ni][0], acc[mt][ni][1]);
        }
      }
    }
    compute_sync<NT>();
    DGB_TICK(3);
  }
}

// ------------------------------------------------------------------------------------------
// Navier-Stokes first pass: BR1 gradient of the conserved variables
//   grad[x][c] = -sum_r drdx[r][x] (Sw_r q_c) + sum_f fscale_f n_{x,f} (lift_f q*_f)
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int K>
struct GradSmem {
  using EL = ElemT<DIM, P>;
  double Wq[DIM * EL::NPR * EL::LDQ];
  double Wf[EL::NF * EL::NPR * EL::LDL];
  double Qs[EL::C * K * EL::LDQ];
  double Ss[EL::C * K * EL::LDS];
  double coef[K][DIM][EL::NS];
  GeoSmem<DIM, P, K> geo;
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int K, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
k_grad(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
       double* __restrict__ grad, Phys ph, int nblocks) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NI = EL::NI;
  constexpr int NT = NW * 32;
  static_assert((C * K) % 8 == 0, "columns per block must be a multiple of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<GradSmem<DIM, P, K>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < DIM * EL::NPR * EL::LDQ; n += NT) S.Wq[n] = d.Wq[n];
  for (int n = tid; n < NF * EL::NPR * EL::LDL; n += NT) S.Wf[n] = d.Wf[n];
  for (int n = tid; n < C * K * EL::LDQ; n += NT) S.Qs[n] = 0.0;
  for (int n = tid; n < C * K * EL::LDS; n += NT) S.Ss[n] = 0.0;
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  compute_sync<NT>();   // the zero fill above must not race with the first block's staging writes

#ifdef DGB_PHASE_TIMING
  long long tlast = clock64();
#endif
  for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    stage_geo<DIM, P, K>(S.geo, d, e0, nel, tid, NT);
    // stage q rows (coalesced) for the volume part
    for (int n = tid; n < C * nel * NP; n += NT) {
      const int c = n / (nel * NP), ej = n - c * (nel * NP);
      const int e = ej / NP, j = ej - e * NP;
      S.Qs[(c * K + e) * EL::LDQ + j] = q[((long long)c * E + e0) * NP + ej];
    }
    compute_sync<NT>();
    DGB_TICK(4);

    // combination coefficients per element
    for (int n = tid; n < nel * DIM * EL::NS; n += NT) {
      const int e = n / (DIM * EL::NS), xs = n - e * (DIM * EL::NS);
      const int x = xs / EL::NS, s = xs - x * EL::NS;
      S.coef[e][x][s] = s < DIM ? -S.geo.drdx[s * DIM + x][e]
                                : S.geo.fsc[e][s - DIM] * S.geo.nrm[x][e][s - DIM];
    }
    // face averages q* = (q- + q+)/2 with boundary states
    for (int n = tid; n < nel * NFT; n += NT) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const long long cn = S.geo.conn[e][f];
      const long long nb = DGB_CONN_NB(cn);
      const int nf = DGB_CONN_NF(cn), pid = DGB_CONN_PERM(cn), bc = DGB_CONN_BC(cn);
      const int jm = S.fn[f * NFP + m];
      const int jp = S.fn[nf * NFP + S.perm[pid * NFP + m]];
      double nrm[DIM];
#pragma unroll
      for (int x = 0; x < DIM; ++x) nrm[x] = S.geo.nrm[x][e][f];
      const bool in_ghost = nb >= E;
      const double* pbase = in_ghost ? ghost : q;
      const long long pE = in_ghost ? G : E;
      const long long pe = in_ghost ? nb - E : nb;
      double qm[C], qp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qm[c] = S.Qs[(c * K + e) * EL::LDQ + jm];
        qp[c] = pbase[((long long)c * pE + pe) * NP + jp];
      }
      bc_state<DIM, true>(bc, qm, nrm, ph, qp);
#pragma unroll
      for (int c = 0; c < C; ++c) S.Ss[(c * K + e) * EL::LDS + f * EL::NFPK + m] = 0.5 * (qm[c] + qp[c]);
    }
    compute_sync<NT>();
    DGB_TICK(5);

    constexpr int NTILES = C * K / 8;
    for (int tile = warp; tile < NTILES; tile += NW) {
      __syncwarp();
      double accT[DIM][1][NI][2], accU[NF][1][NI][2];
#pragma unroll
      for (int s = 0; s < DIM; ++s)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { accT[s][0][ni][0] = 0.0; accT[s][0][ni][1] = 0.0; }
#pragma unroll
      for (int s = 0; s < NF; ++s)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { accU[s][0][ni][0] = 0.0; accU[s][0][ni][1] = 0.0; }
#pragma unroll
      for (int r = 0; r < DIM; ++r)
        mma_block<NI, 1>(accT[r], S.Qs + tile * 8 * EL::LDQ, EL::LDQ, S.Wq + r * EL::NPR * EL::LDQ, EL::LDQ,
                         EL::NPK / 4, lane);
#pragma unroll
      for (int f = 0; f < NF; ++f)
        mma_block<NI, 1>(accU[f], S.Ss + tile * 8 * EL::LDS + f * EL::NFPK, EL::LDS,
                         S.Wf + f * EL::NPR * EL::LDL, EL::LDL, EL::NFPK / 4, lane);
      const int col = tile * 8 + (lane >> 2);
      const int c = col / K, e = col - c * K;
      if (e >= nel) continue;
#pragma unroll
      for (int x = 0; x < DIM; ++x) {
        double cf[EL::NS];
#pragma unroll
        for (int s = 0; s < EL::NS; ++s) cf[s] = S.coef[e][x][s];
        const long long rowbase = ((long long)(x * C + c) * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          double v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int s = 0; s < DIM; ++s) { v0 += cf[s] * accT[s][0][ni][0]; v1 += cf[s] * accT[s][0][ni][1]; }
#pragma unroll
          for (int s = 0; s < NF; ++s) { v0 += cf[DIM + s] * accU[s][0][ni][0]; v1 += cf[DIM + s] * accU[s][0][ni][1]; }
          const int i = ni * 8 + 2 * (lane & 3);
          if (NP % 2 == 0) {
            if (i < NP) *reinterpret_cast<double2*>(grad + rowbase + i) = make_double2(v0, v1);
          } else {
            if (i < NP) grad[rowbase + i] = v0;
            if (i + 1 < NP) grad[rowbase + i + 1] = v1;
          }
        }
      }
    }
    compute_sync<NT>();
    DGB_TICK(6);
  }
}

}  // namespace dgb
