// Navier-Stokes right-hand side in the FLUX arrangement (operators.py: dg_ns_flux + dg_ns_div).
//
// The gradient arrangement (dgb_kernels_warp.cuh) evaluates the total flux three times per node and
// RHS: at the node (volume term), at the node again as the own side of a face, and once more by the
// neighbour for its plus side; ncu showed pass 2 spending as much of the FP64 datapath on that
// pointwise work (22.9 %) as on the DMMA contraction (28.9 %).  Here every node's flux is evaluated
// ONCE, by its owner, at the end of pass 1 while the BR1 gradient is still on chip:
//
//   k_nsflux3  (pass 1)  rows -> face averages -> DMMA (Sw_r q, lift_f q*) -> grad q into shared
//                        memory -> pointwise F = F_inv - F_visc -> T[r][c] = sum_x (J dr/dx)[r][x] F[x][c]
//                        and lam = |u| + c  ->  HBM  (dim*C + 1 planes instead of dim*C)
//   k_nsdiv3   (pass 2)  T rows arrive by cp.async straight into the DMMA operand layout (no
//                        pointwise volume work at all); per face node the kernel gathers the
//                        neighbour's q, lam and T rows: sJ F+.n = -(face 0 ? sum_r T+[r] : -T+[nf-1]),
//                        own side the same signed sum of its own rows -> Rusanov -> DMMA -> 1/J -> store.
//
// Algorithmic HBM bytes per DOF (3D): pass 1 reads 40, writes 128; pass 2 reads 168, writes 40.
#pragma once
#include "dgb_kernels.cuh"
#include "dgb_kernels_async.cuh"
#include "dgb_kernels_warp.cuh"

namespace dgb {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

template <int DIM, int P>
struct FluxT {
  using EL = ElemT<DIM, P>;
  static constexpr int NPL = DIM * EL::C + 1;                    // planes of T: contravariant flux + wave speed
  // q* rows of the gradient pass; a tile's 8 rows are reused for its 8 columns x DIM directions of grad q
  static constexpr int LDSX = ldpad((EL::NF * EL::NFPK > DIM * EL::NP) ? EL::NF * EL::NFPK : DIM * EL::NP);
};

// ------------------------------------------------------------------------------------------
// pass 1: BR1 gradient -> total flux -> contravariant planes
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct FluxGeo {
  using EL = ElemT<DIM, P>;
  double drdx[DIM * DIM][KW];
  double nrm[DIM][KW][EL::NF];
  double fsc[KW][EL::NF];
  long long conn[KW][EL::NF];
  double jac[KW];
};

template <int DIM, int P, int KW>
struct alignas(16) Flux3Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  static constexpr int NCOLP = NTILE * 8;
  double Qs[2][NCOLP * EL::LDQ];
  double Ss[NCOLP * FluxT<DIM, P>::LDSX];
  double coef[KW][DIM][EL::NS];
  FluxGeo<DIM, P, KW> geo[2];
};

template <int DIM, int P, int KW, int NWARPS>
struct Flux3Smem {
  using EL = ElemT<DIM, P>;
  double Wq[DIM * EL::NPR * EL::LDQ];
  double Wf[EL::NF * EL::NPR * EL::LDL];
  Flux3Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void flux_stage_async(double* Qs, FluxGeo<DIM, P, KW>& g, const DiscDev& d, const double* q,
                                                 long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const long long E = d.E;
  if (NP % 2 == 0) {
    constexpr int H = NP / 2;
    for (int n = lane; n < C * nel * H; n += 32) {
      const int c = n / (nel * H), ej = n - c * (nel * H);
      const int e = ej / H, j = 2 * (ej - e * H);
      cp_async16(Qs + (c * KW + e) * EL::LDQ + j, q + ((long long)c * E + e0 + e) * NP + j);
    }
  } else {
    for (int n = lane; n < C * nel * NP; n += 32) {
      const int c = n / (nel * NP), ej = n - c * (nel * NP);
      const int e = ej / NP, j = ej - e * NP;
      cp_async8(Qs + (c * KW + e) * EL::LDQ + j, q + ((long long)c * E + e0) * NP + ej);
    }
  }
  for (int n = lane; n < DIM * DIM * KW; n += 32) {
    const int rx = n / KW, e = n - rx * KW;
    if (e < nel) cp_async8(&g.drdx[rx][e], d.drdx + (long long)rx * E + e0 + e);
  }
  for (int n = lane; n < DIM * KW * NF; n += 32) {
    const int x = n / (KW * NF), ef = n - x * (KW * NF);
    if (ef < nel * NF) cp_async8(&g.nrm[x][0][ef], d.normals + ((long long)x * E + e0) * NF + ef);
  }
  for (int n = lane; n < nel * NF; n += 32) {
    cp_async8(&g.fsc[0][n], d.fscale + e0 * NF + n);
    cp_async8(&g.conn[0][n], d.conn + e0 * NF + n);
  }
  if (lane < nel) cp_async8(&g.jac[lane], d.jac + e0 + lane);
}

template <int DIM, int P, int KW, int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsflux3(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
          double* __restrict__ T, Phys ph, long long nwblocks, unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Flux3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NI = EL::NI;
  constexpr int LDSX = FluxT<DIM, P>::LDSX;
  constexpr int NT = NWARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Flux3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < DIM * EL::NPR * EL::LDQ; n += NT) S.Wq[n] = d.Wq[n];
  for (int n = tid; n < NF * EL::NPR * EL::LDL; n += NT) S.Wf[n] = d.Wf[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  for (int n = lane; n < 2 * WS::NCOLP * EL::LDQ; n += 32) W.Qs[0][n] = 0.0;
  for (int n = lane; n < WS::NCOLP * LDSX; n += 32) W.Ss[n] = 0.0;
  __syncthreads();

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  int buf = 0;
  if (wb < nwblocks) {
    const long long e0 = wb * KW;
    flux_stage_async<DIM, P, KW>(W.Qs[0], W.geo[0], d, q, e0, (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW), lane);
  }
  cp_async_commit();

  while (wb < nwblocks) {
    const long long e0 = wb * KW;
    const int nel = (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW);
    cp_async_wait<0>();
    __syncwarp();
    const double* Qs = W.Qs[buf];
    const FluxGeo<DIM, P, KW>& geo = W.geo[buf];
    const long long wb_next = next_block(counter, wstride, lane);
    if (wb_next < nwblocks) {
      const long long e1 = wb_next * KW;
      flux_stage_async<DIM, P, KW>(W.Qs[buf ^ 1], W.geo[buf ^ 1], d, q, e1,
                                   (int)((E - e1) < (long long)KW ? (E - e1) : (long long)KW), lane);
    }
    cp_async_commit();

    // ---- face averages q* (central flux, boundary states) -> Ss; metric coefficients ---------
    for (int n = lane; n < nel * DIM * EL::NS; n += 32) {
      const int e = n / (DIM * EL::NS), xs = n - e * (DIM * EL::NS);
      const int x = xs / EL::NS, s = xs - x * EL::NS;
      W.coef[e][x][s] = s < DIM ? -geo.drdx[s * DIM + x][e] : geo.fsc[e][s - DIM] * geo.nrm[x][e][s - DIM];
    }
    // the previous block left grad q in the q* rows: the K-padding columns must be zero again
    if (EL::NFPK != NFP) {
      for (int n = lane; n < WS::NCOLP * NF * (EL::NFPK - NFP); n += 32) {
        const int col = n / (NF * (EL::NFPK - NFP)), r = n - col * (NF * (EL::NFPK - NFP));
        const int f = r / (EL::NFPK - NFP), m = NFP + (r - f * (EL::NFPK - NFP));
        W.Ss[col * LDSX + f * EL::NFPK + m] = 0.0;
      }
    }
    for (int n = lane; n < nel * NFT; n += 32) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const long long cn = geo.conn[e][f];
      const long long nb = DGB_CONN_NB(cn);
      const int nf = DGB_CONN_NF(cn), pid = DGB_CONN_PERM(cn), bc = DGB_CONN_BC(cn);
      const int jm = S.fn[f * NFP + m];
      const int jp = S.fn[nf * NFP + S.perm[pid * NFP + m]];
      const bool in_ghost = nb >= E;
      const long long pE = in_ghost ? G : E;
      const double* pbase = (in_ghost ? ghost : q) + (in_ghost ? nb - E : nb) * NP + jp;
      double qm[C], qp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qp[c] = pbase[(long long)c * pE * NP];
        qm[c] = Qs[(c * KW + e) * EL::LDQ + jm];
      }
      if (bc != 0) {
        double nrm[DIM];
#pragma unroll
        for (int x = 0; x < DIM; ++x) nrm[x] = geo.nrm[x][e][f];
        bc_state<DIM, true>(bc, qm, nrm, ph, qp);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) W.Ss[(c * KW + e) * LDSX + f * EL::NFPK + m] = 0.5 * (qm[c] + qp[c]);
    }
    __syncwarp();

    // ---- tensor-core contractions, one 8-column tile at a time; grad q of the tile -> its Ss rows ----
#pragma unroll 1
    for (int tile = 0; tile < WS::NTILE; ++tile) {
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
        mma_block<NI, 1>(accT[r], Qs + tile * 8 * EL::LDQ, EL::LDQ, S.Wq + r * EL::NPR * EL::LDQ, EL::LDQ,
                         EL::NPK / 4, lane);
#pragma unroll
      for (int f = 0; f < NF; ++f)
        mma_block<NI, 1>(accU[f], W.Ss + tile * 8 * LDSX + f * EL::NFPK, LDSX,
                         S.Wf + f * EL::NPR * EL::LDL, EL::LDL, EL::NFPK / 4, lane);
      __syncwarp();                       // every lane has read this tile's q* rows: they may be overwritten
      const int k8 = lane >> 2;
      const int col = tile * 8 + k8;
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
        double* sg = W.Ss + tile * 8 * LDSX;
#pragma unroll
        for (int x = 0; x < DIM; ++x) {
          double cf[EL::NS];
#pragma unroll
          for (int s = 0; s < EL::NS; ++s) cf[s] = W.coef[e][x][s];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll
            for (int s = 0; s < DIM; ++s) { v0 += cf[s] * accT[s][0][ni][0]; v1 += cf[s] * accT[s][0][ni][1]; }
#pragma unroll
            for (int s = 0; s < NF; ++s) { v0 += cf[DIM + s] * accU[s][0][ni][0]; v1 += cf[DIM + s] * accU[s][0][ni][1]; }
            const int i = ni * 8 + 2 * (lane & 3);
            if (i < NP) sg[(x * 8 + k8) * NP + i] = v0;
            if (i + 1 < NP) sg[(x * 8 + k8) * NP + i + 1] = v1;
          }
        }
      }
    }
    __syncwarp();

    // ---- pointwise: total flux at every node, contravariant + Jacobian-scaled, and the wave speed ----
    for (int n = lane; n < nel * NP; n += 32) {
      const int e = n / NP, j = n - e * NP;
      double qq[C], g[DIM][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int col = c * KW + e;
        qq[c] = Qs[col * EL::LDQ + j];
        const double* sg = W.Ss + (col >> 3) * 8 * LDSX + (col & 7) * NP + j;
#pragma unroll
        for (int x = 0; x < DIM; ++x) g[x][c] = sg[x * 8 * NP];
      }
      Prim<DIM> s;
      make_prim<DIM>(qq, ph.gamma, s);
      double F[DIM][C], Fv[DIM][C];
      inviscid_flux<DIM>(s, F);
      viscous_flux<DIM>(s, g, ph, Fv);
#pragma unroll
      for (int x = 0; x < DIM; ++x)
#pragma unroll
        for (int c = 1; c < C; ++c) F[x][c] -= Fv[x][c];
      const double J = geo.jac[e];
      double* out = T + e0 * NP + n;
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        double m[DIM];
#pragma unroll
        for (int x = 0; x < DIM; ++x) m[x] = J * geo.drdx[r * DIM + x][e];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double acc = m[0] * F[0][c];
#pragma unroll
          for (int x = 1; x < DIM; ++x) acc += m[x] * F[x][c];
          out[(long long)(r * C + c) * E * NP] = acc;
        }
      }
      out[(long long)(DIM * C) * E * NP] = wavespeed<DIM>(s, ph.gamma);
    }
    __syncwarp();
    wb = wb_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------
// pass 2: divergence of the stored flux + face terms
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct alignas(16) Div3Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  // operand rows of the real columns only: the fragment loads of a padding column (at most one:
  // C*KW = 15 or 16) read the rows that follow it inside this struct; its accumulators are never
  // stored and DMMA rows do not mix
  double Ts[NCOL * EL::LDV];
  double Fs[NCOL * EL::LDF];
  double Qs[NCOL * EL::NP];
  double Lam[KW * EL::NP];
  double sj[KW][EL::NF];
  long long conn[KW][EL::NF];
  double rj[KW];
};

template <int DIM, int P, int KW, int NWARPS>
struct Div3Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Div3Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void div_stage_async(Div3Warp<DIM, P, KW>& W, const DiscDev& d, const double* q,
                                                const double* T, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const long long E = d.E;
  if (NP % 2 == 0) {
    constexpr int H = NP / 2;
    const int per = nel * H;                       // 16-byte chunks per plane
    for (int n = lane; n < DIM * C * per; n += 32) {
      const int pl = n / per, ej = n - pl * per;
      const int r = pl / C, c = pl - r * C;
      const int e = ej / H, j = 2 * (ej - e * H);
      cp_async16(W.Ts + (c * KW + e) * EL::LDV + r * EL::NPK + j, T + ((long long)pl * E + e0 + e) * NP + j);
    }
    for (int n = lane; n < C * per; n += 32) {
      const int c = n / per, ej = n - c * per;
      const int e = ej / H, j = 2 * (ej - e * H);
      cp_async16(W.Qs + (c * KW + e) * NP + j, q + ((long long)c * E + e0 + e) * NP + j);
    }
    for (int n = lane; n < per; n += 32)
      cp_async16(W.Lam + 2 * n, T + ((long long)(DIM * C) * E + e0) * NP + 2 * n);
  } else {
    const int per = nel * NP;
    for (int n = lane; n < DIM * C * per; n += 32) {
      const int pl = n / per, ej = n - pl * per;
      const int r = pl / C, c = pl - r * C;
      const int e = ej / NP, j = ej - e * NP;
      cp_async8(W.Ts + (c * KW + e) * EL::LDV + r * EL::NPK + j, T + ((long long)pl * E + e0) * NP + ej);
    }
    for (int n = lane; n < C * per; n += 32) {
      const int c = n / per, ej = n - c * per;
      const int e = ej / NP, j = ej - e * NP;
      cp_async8(W.Qs + (c * KW + e) * NP + j, q + ((long long)c * E + e0) * NP + ej);
    }
    for (int n = lane; n < per; n += 32) cp_async8(W.Lam + n, T + ((long long)(DIM * C) * E + e0) * NP + n);
  }
  for (int n = lane; n < nel * NF; n += 32) {
    cp_async8(&W.sj[0][n], d.sj + e0 * NF + n);
    cp_async8(&W.conn[0][n], d.conn + e0 * NF + n);
  }
  if (lane < nel) cp_async8(&W.rj[lane], d.rj + e0 + lane);
}

template <int DIM> struct VecC { double v[DIM + 2]; };

// Boundary face node (rare): inviscid flux of the exterior state, viscous flux of the interior
// state.  Returns sJ F*.n per field (operators.py: f_bnd).
template <int DIM>
__device__ __noinline__ VecC<DIM> boundary_flux(int bc, VecC<DIM> qm_, VecC<DIM> own_, double lam_m, double sj,
                                               const double* __restrict__ normals, long long nstride, Phys ph) {
  constexpr int C = DIM + 2;
  double nrm[DIM], qm[C], qb[C];
#pragma unroll
  for (int x = 0; x < DIM; ++x) nrm[x] = normals[x * nstride];
#pragma unroll
  for (int c = 0; c < C; ++c) { qm[c] = qm_.v[c]; qb[c] = qm_.v[c]; }
  bc_state<DIM, true>(bc, qm, nrm, ph, qb);
  Prim<DIM> sb, sm;
  make_prim<DIM>(qb, ph.gamma, sb);
  make_prim<DIM>(qm, ph.gamma, sm);
  double fnb[C], fni[C];
  inviscid_normal_flux<DIM>(sb, nrm, fnb);
  inviscid_normal_flux<DIM>(sm, nrm, fni);
  const double lam = fmax(lam_m, wavespeed<DIM>(sb, ph.gamma));
  VecC<DIM> out;
#pragma unroll
  for (int c = 0; c < C; ++c)
    out.v[c] = own_.v[c] + 0.5 * sj * (fnb[c] - fni[c]) + 0.5 * sj * lam * (qm[c] - qb[c]);
  return out;
}

template <int DIM, int P, int KW, int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsdiv3(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long nwblocks, unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Div3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NWARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  {
    double* z = reinterpret_cast<double*>(&W);
    for (int n = lane; n < (int)(sizeof(WS) / 8); n += 32) z[n] = 0.0;
  }
  __syncthreads();

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  if (wb < nwblocks) {
    const long long e0 = wb * KW;
    div_stage_async<DIM, P, KW>(W, d, q, T, e0, (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW), lane);
  }
  cp_async_commit();

  while (wb < nwblocks) {
    const long long e0 = wb * KW;
    const int nel = (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW);
    cp_async_wait<0>();
    __syncwarp();

    // ---- face gather + Rusanov: Fs = -(sJ F*.n) ----------------------------------------------
#pragma unroll 2
    for (int n = lane; n < nel * NFT; n += 32) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const long long cn = W.conn[e][f];
      const long long nb = DGB_CONN_NB(cn);
      const int nf = DGB_CONN_NF(cn), pid = DGB_CONN_PERM(cn), bc = DGB_CONN_BC(cn);
      const int jm = S.fn[f * NFP + m];
      const int jp = S.fn[nf * NFP + S.perm[pid * NFP + m]];
      const bool in_ghost = nb >= E;
      const long long pstride = (in_ghost ? G : E) * NP;
      const long long off = (in_ghost ? nb - E : nb) * NP + jp;
      const double* qbase = (in_ghost ? ghost : q) + off;
      const double* tbase = (in_ghost ? Tghost : T) + off;
      const int r0 = nf == 0 ? 0 : nf - 1;
      double qp[C], nbr[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qp[c] = qbase[c * pstride];
        nbr[c] = tbase[(r0 * C + c) * pstride];
      }
      const double lam_p = tbase[(DIM * C) * pstride];
      if (nf == 0) {
#pragma unroll
        for (int r = 1; r < DIM; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c) nbr[c] += tbase[(r * C + c) * pstride];
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) nbr[c] = -nbr[c];
      }
      const double sj = W.sj[e][f];
      const double lam_m = W.Lam[e * NP + jm];
      double qm[C], own[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qm[c] = W.Qs[(c * KW + e) * NP + jm];
        const double* trow = W.Ts + (c * KW + e) * EL::LDV + jm;
        if (f == 0) {
          own[c] = trow[0];
#pragma unroll
          for (int r = 1; r < DIM; ++r) own[c] += trow[r * EL::NPK];
        } else {
          own[c] = -trow[(f - 1) * EL::NPK];
        }
      }
      if (bc == 0) {
        const double pen = sj * fmax(lam_m, lam_p);
#pragma unroll
        for (int c = 0; c < C; ++c)
          W.Fs[(c * KW + e) * EL::LDF + fm] = -0.5 * ((own[c] - nbr[c]) + pen * (qm[c] - qp[c]));
      } else {
        VecC<DIM> a, b;
#pragma unroll
        for (int c = 0; c < C; ++c) { a.v[c] = qm[c]; b.v[c] = own[c]; }
        const VecC<DIM> fb = boundary_flux<DIM>(bc, a, b, lam_m, sj, d.normals + (e0 + e) * NF + f, E * NF, ph);
#pragma unroll
        for (int c = 0; c < C; ++c) W.Fs[(c * KW + e) * EL::LDF + fm] = -fb.v[c];
      }
    }
    __syncwarp();

    // ---- tensor-core contraction -------------------------------------------------------------
    double acc[WS::NTILE][EL::NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
    mma_block<EL::NI, WS::NTILE>(acc, W.Ts, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
    mma_block<EL::NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
    double rj[WS::NTILE];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int e = col % KW;
      rj[mt] = W.rj[e];
    }
    __syncwarp();                        // all operand rows consumed: the next block may land on them

    const long long wb_next = next_block(counter, wstride, lane);
    if (wb_next < nwblocks) {
      const long long e1 = wb_next * KW;
      div_stage_async<DIM, P, KW>(W, d, q, T, e1, (int)((E - e1) < (long long)KW ? (E - e1) : (long long)KW), lane);
    }
    cp_async_commit();

    // ---- 1/J and the (RK-fused) store --------------------------------------------------------
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) {
          const int i = ni * 8 + 2 * (lane & 3);
          store_pair<NP>(ep, rowbase + i, i, rj[mt] * acc[mt][ni][0], rj[mt] * acc[mt][ni][1]);
        }
      }
    }
    wb = wb_next;
  }
  cp_async_wait<0>();
}

}  // namespace dgb
