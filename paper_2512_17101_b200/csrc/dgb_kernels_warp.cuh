// Warp-autonomous versions of the fused DG kernels (default path).
//
// ncu on the CTA-phased kernels (dgb_kernels.cuh / dgb_kernels_async.cuh) showed 22-34% of all stall
// samples at __syncthreads and 19-41% on global-load scoreboards: every phase change idles the whole
// CTA and only 2-3 CTAs fit on an SM.  Here a WARP is the unit of work: each warp of a persistent CTA
// owns KW consecutive elements from load to store and keeps its operand rows in a private slice of
// shared memory; the only synchronisation is __syncwarp between its own phases.  The 14-16 warps of
// an SM drift apart, so at any moment some are waiting on HBM, some evaluate fluxes on the FP64 pipe
// and some issue DMMA tiles -- the overlap the phased kernels could not get.  The reference matrices
// W live once per SM in shared memory and are shared by all warps.
//
// Column layout inside a warp: col = c*KW + e (field-major), padded to a multiple of 8 columns; a
// padded column's operand row stays zero and its results are never stored.
#pragma once
#include "dgb_kernels.cuh"
#include "dgb_kernels_async.cuh"

namespace dgb {

// Dynamic work distribution: a warp takes its next block of elements from a global counter, so the set
// of blocks in flight is always the ~1800 most recent ones no matter how far individual warps drift
// apart.  (With a static grid-stride assignment the drift spread the in-flight window over hundreds of
// MB and the face-neighbour gathers missed L2: 35.9 GB of DRAM reads for 17 GB of compulsory traffic
// in pass 2 at 100M DOFs.)  The counter is zeroed by the host before every launch.
__device__ __forceinline__ long long next_block(unsigned long long* counter, long long first_dynamic, int lane) {
  unsigned long long v = 0;
  if (lane == 0) v = atomicAdd(counter, 1ULL);
  v = __shfl_sync(0xffffffffu, v, 0);
  return first_dynamic + (long long)v;
}

template <int DIM, int P, int KW>
struct WarpGeo {
  using EL = ElemT<DIM, P>;
  double drdx[DIM * DIM][KW];
  double nrm[DIM][KW][EL::NF];
  double fsc[KW][EL::NF];
  long long conn[KW][EL::NF];
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void warp_stage_geo(WarpGeo<DIM, P, KW>& g, const DiscDev& d, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  for (int n = lane; n < DIM * DIM * KW; n += 32) {
    const int rx = n / KW, e = n - rx * KW;
    if (e < nel) g.drdx[rx][e] = d.drdx[(long long)rx * d.E + e0 + e];
  }
  for (int n = lane; n < DIM * KW * EL::NF; n += 32) {
    const int x = n / (KW * EL::NF), ef = n - x * (KW * EL::NF);
    if (ef < nel * EL::NF) g.nrm[x][0][ef] = d.normals[((long long)x * d.E + e0) * EL::NF + ef];
  }
  for (int n = lane; n < nel * EL::NF; n += 32) {
    g.fsc[0][n] = d.fscale[e0 * EL::NF + n];
    g.conn[0][n] = d.conn[e0 * EL::NF + n];
  }
}

// ------------------------------------------------------------------------------------------
// right-hand side (Euler / Navier-Stokes second pass)
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct Rhs3Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  static constexpr int NCOLP = NTILE * 8;
  double Gs[NCOLP * EL::LDV];
  double Fs[NCOLP * EL::LDF];
  double Lam[KW * EL::NP];
  WarpGeo<DIM, P, KW> geo;
};

template <int DIM, int P, int KW, int NWARPS>
struct Rhs3Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Rhs3Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int KW, int NWARPS, bool VISCOUS>
// register budget note: ptxas sizes the per-thread cap from the warp count rounded up to a multiple
// of 4 (8 warps -> 255, 12 -> 168, 16 -> 128), so only those warp counts make sense
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_rhs3(DiscDev d, const double* __restrict__ q, const double* __restrict__ gq,
       const double* __restrict__ ghost, const double* __restrict__ gghost,
       Epilogue ep, Phys ph, long long nwblocks, unsigned long long* __restrict__ counter,
       long long ebeg, long long eend) {
  using EL = ElemT<DIM, P>;
  using WS = Rhs3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NWARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Rhs3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  for (int n = lane; n < WS::NCOLP * EL::LDV; n += 32) W.Gs[n] = 0.0;
  for (int n = lane; n < WS::NCOLP * EL::LDF; n += 32) W.Fs[n] = 0.0;
  __syncthreads();      // the only CTA-wide barrier: W and the tables are visible to every warp

  constexpr int NPL = VISCOUS ? (DIM + 1) * C : C;
  constexpr int NGEO = (int)(sizeof(WarpGeo<DIM, P, KW>) / 8);
  constexpr int GPL = (NGEO + 31) / 32;          // geometry words per lane
  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  // prologue: this lane's first-round node inputs and its share of the geometry, in registers
  double pre[NPL];
  double pgeo[GPL];
  auto prefetch = [&](long long wbn) {
    const long long e1 = ebeg + wbn * KW;
    const int nel1 = (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW);
    if (lane < nel1 * NP) {
#pragma unroll
      for (int c = 0; c < C; ++c) pre[c] = q[((long long)c * E + e1) * NP + lane];
      if (VISCOUS) {
#pragma unroll
        for (int pl = 0; pl < NPL - C; ++pl) pre[C + pl] = gq[((long long)pl * E + e1) * NP + lane];
      }
    }
    // geometry words in WarpGeo order: drdx[DIM*DIM][KW], nrm[DIM][KW][NF], fsc[KW][NF], conn[KW][NF]
#pragma unroll
    for (int k = 0; k < GPL; ++k) {
      const int n = lane + 32 * k;
      double v = 0.0;
      if (n < DIM * DIM * KW) {
        const int rx = n / KW, e = n - rx * KW;
        if (e < nel1) v = d.drdx[(long long)rx * E + e1 + e];
      } else if (n < DIM * DIM * KW + DIM * KW * NF) {
        const int m = n - DIM * DIM * KW;
        const int x = m / (KW * NF), ef = m - x * (KW * NF);
        if (ef < nel1 * NF) v = d.normals[((long long)x * E + e1) * NF + ef];
      } else if (n < DIM * DIM * KW + DIM * KW * NF + KW * NF) {
        const int ef = n - (DIM * DIM * KW + DIM * KW * NF);
        if (ef < nel1 * NF) v = d.fscale[e1 * NF + ef];
      } else if (n < NGEO) {
        const int ef = n - (DIM * DIM * KW + DIM * KW * NF + KW * NF);
        if (ef < nel1 * NF) v = __longlong_as_double(d.conn[e1 * NF + ef]);
      }
      pgeo[k] = v;
    }
  };
  if (wb < nwblocks) prefetch(wb);

  while (wb < nwblocks) {
    long long wb_next = nwblocks;
    const long long e0 = ebeg + wb * KW;
    const int nel = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
    {
      double* gw = reinterpret_cast<double*>(&W.geo);
#pragma unroll
      for (int k = 0; k < GPL; ++k) if (lane + 32 * k < NGEO) gw[lane + 32 * k] = pgeo[k];
    }
    __syncwarp();

    // ---- phase 1: volume flux (first round from the register prefetch) ----------------------
    for (int n = lane; n < nel * NP; n += 32) {
      const int e = n / NP, j = n - e * NP;
      double qq[C], g[DIM][C];
      if (n == lane) {
#pragma unroll
        for (int c = 0; c < C; ++c) qq[c] = pre[c];
        if (VISCOUS) {
#pragma unroll
          for (int x = 0; x < DIM; ++x)
#pragma unroll
            for (int c = 0; c < C; ++c) g[x][c] = pre[C + x * C + c];
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) qq[c] = q[((long long)c * E + e0) * NP + n];
        if (VISCOUS) {
#pragma unroll
          for (int x = 0; x < DIM; ++x)
#pragma unroll
            for (int c = 0; c < C; ++c) g[x][c] = gq[((long long)(x * C + c) * E + e0) * NP + n];
        }
      }
      Prim<DIM> s;
      make_prim<DIM>(qq, ph.gamma, s);
      double F[DIM][C];
      inviscid_flux<DIM>(s, F);
      if (VISCOUS) {
        double Fv[DIM][C];
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
        for (int x = 0; x < DIM; ++x) m[x] = W.geo.drdx[r * DIM + x][e];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int x = 0; x < DIM; ++x) acc += m[x] * F[x][c];
          W.Gs[(c * KW + e) * EL::LDV + r * EL::NPK + j] = acc;
        }
      }
      W.Lam[n] = wavespeed<DIM>(s, ph.gamma);
    }
    __syncwarp();

    // ---- phase 2: face gather + numerical flux (own side from Gs, see dgb_kernels.cuh) ------
    // (a two-register-set software pipeline over the rounds was measured and lost: it needs ~230
    //  registers, i.e. 8 warps per SM instead of 12 -- 4.56 ms vs 3.95 ms on the n=64 case.)
    for (int n = lane; n < nel * NFT; n += 32) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const long long cn = W.geo.conn[e][f];
      const long long nb = DGB_CONN_NB(cn);
      const int nf = DGB_CONN_NF(cn), pid = DGB_CONN_PERM(cn), bc = DGB_CONN_BC(cn);
      const int jm = S.fn[f * NFP + m];
      const int jp = S.fn[nf * NFP + S.perm[pid * NFP + m]];
      const bool in_ghost = nb >= E;
      const long long pstride = (in_ghost ? G : E) * NP;
      const long long off = (in_ghost ? nb - E : nb) * NP + jp;
      const double* pbase = (in_ghost ? ghost : q) + off;
      double qm[C], qp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qp[c] = pbase[c * pstride];
        qm[c] = q[((long long)c * E + e0 + e) * NP + jm];
      }
      double gp[DIM][C];
      if (VISCOUS) {
        const double* gbase = (in_ghost ? gghost : gq) + off;
#pragma unroll
        for (int x = 0; x < DIM; ++x)
#pragma unroll
          for (int c = 0; c < C; ++c) gp[x][c] = gbase[(x * C + c) * pstride];
      }
      double nrm[DIM];
#pragma unroll
      for (int x = 0; x < DIM; ++x) nrm[x] = W.geo.nrm[x][e][f];
      const double fs = W.geo.fsc[e][f];
      if (bc != 0) bc_state<DIM, VISCOUS>(bc, qm, nrm, ph, qp);
      Prim<DIM> sp_;
      make_prim<DIM>(qp, ph.gamma, sp_);
      double fnp[C];
      inviscid_normal_flux<DIM>(sp_, nrm, fnp);
      const double lam = fmax(W.Lam[e * NP + jm], wavespeed<DIM>(sp_, ph.gamma));
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
        const double* grow = W.Gs + (c * KW + e) * EL::LDV + jm;
        double own;                       // fscale * (F^- . n): (f == 0) ? sum_r G_r : -G_{f-1}
        if (f == 0) {
          own = grow[0];
#pragma unroll
          for (int r = 1; r < DIM; ++r) own += grow[r * EL::NPK];
        } else {
          own = -grow[(f - 1) * EL::NPK];
        }
        W.Fs[(c * KW + e) * EL::LDF + fm] = -0.5 * (own + fs * (fnp[c] + lam * (qm[c] - qp[c])));
      }
    }
    __syncwarp();

    // take the next block now: its inputs start their trip from HBM and land while the tensor cores work
    wb_next = next_block(counter, wstride, lane);
    if (wb_next < nwblocks) prefetch(wb_next);

    // ---- phase 3: tensor-core contraction + (RK-fused) store ---------------------------------
    {
      double acc[WS::NTILE][EL::NI][2];
#pragma unroll
      for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
      mma_block<EL::NI, WS::NTILE>(acc, W.Gs, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
      mma_block<EL::NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
#pragma unroll
      for (int mt = 0; mt < WS::NTILE; ++mt) {
        const int col = mt * 8 + (lane >> 2);
        const int c = col / KW, e = col - c * KW;
        if (col < WS::NCOL && e < nel) {
          const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
          for (int ni = 0; ni < EL::NI; ++ni) {
            const int i = ni * 8 + 2 * (lane & 3);
            store_pair<NP>(ep, rowbase + i, i, acc[mt][ni][0], acc[mt][ni][1]);
          }
        }
      }
    }
    __syncwarp();
    wb = wb_next;
  }
}

// ------------------------------------------------------------------------------------------
// Navier-Stokes first pass (BR1 gradient)
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct Grad3Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  static constexpr int NCOLP = NTILE * 8;
  double Qs[2][NCOLP * EL::LDQ];     // own rows, double-buffered: the next block arrives by cp.async
  double Ss[NCOLP * EL::LDS];
  double coef[KW][DIM][EL::NS];
  WarpGeo<DIM, P, KW> geo[2];
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void warp_stage_async(double* Qs, WarpGeo<DIM, P, KW>& g, const DiscDev& d, const double* q,
                                                 long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const long long E = d.E;
  for (int n = lane; n < C * nel * NP; n += 32) {
    const int c = n / (nel * NP), ej = n - c * (nel * NP);
    const int e = ej / NP, j = ej - e * NP;
    cp_async8(Qs + (c * KW + e) * EL::LDQ + j, q + ((long long)c * E + e0) * NP + ej);
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
}

template <int DIM, int P, int KW, int NWARPS>
struct Grad3Smem {
  using EL = ElemT<DIM, P>;
  double Wq[DIM * EL::NPR * EL::LDQ];
  double Wf[EL::NF * EL::NPR * EL::LDL];
  Grad3Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int KW, int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_grad3(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
        double* __restrict__ grad, Phys ph, long long nwblocks, unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Grad3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NI = EL::NI;
  constexpr int NT = NWARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Grad3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < DIM * EL::NPR * EL::LDQ; n += NT) S.Wq[n] = d.Wq[n];
  for (int n = tid; n < NF * EL::NPR * EL::LDL; n += NT) S.Wf[n] = d.Wf[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  for (int n = lane; n < 2 * WS::NCOLP * EL::LDQ; n += 32) W.Qs[0][n] = 0.0;
  for (int n = lane; n < WS::NCOLP * EL::LDS; n += 32) W.Ss[n] = 0.0;
  __syncthreads();

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  int buf = 0;
  if (wb < nwblocks) {
    const long long e0 = wb * KW;
    warp_stage_async<DIM, P, KW>(W.Qs[0], W.geo[0], d, q, e0, (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW), lane);
  }
  cp_async_commit();

  while (wb < nwblocks) {
    const long long e0 = wb * KW;
    const int nel = (int)((E - e0) < (long long)KW ? (E - e0) : (long long)KW);
    cp_async_wait<0>();
    __syncwarp();                        // this block's rows + geometry have landed (all lanes' copies)
    const double* Qs = W.Qs[buf];
    const WarpGeo<DIM, P, KW>& geo = W.geo[buf];
    // take the next block and start its copies; they land while this block computes
    const long long wb_next = next_block(counter, wstride, lane);
    if (wb_next < nwblocks) {
      const long long e1 = wb_next * KW;
      warp_stage_async<DIM, P, KW>(W.Qs[buf ^ 1], W.geo[buf ^ 1], d, q, e1,
                                   (int)((E - e1) < (long long)KW ? (E - e1) : (long long)KW), lane);
    }
    cp_async_commit();

    for (int n = lane; n < nel * DIM * EL::NS; n += 32) {
      const int e = n / (DIM * EL::NS), xs = n - e * (DIM * EL::NS);
      const int x = xs / EL::NS, s = xs - x * EL::NS;
      W.coef[e][x][s] = s < DIM ? -geo.drdx[s * DIM + x][e] : geo.fsc[e][s - DIM] * geo.nrm[x][e][s - DIM];
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
      for (int c = 0; c < C; ++c) W.Ss[(c * KW + e) * EL::LDS + f * EL::NFPK + m] = 0.5 * (qm[c] + qp[c]);
    }
    __syncwarp();

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
        mma_block<NI, 1>(accU[f], W.Ss + tile * 8 * EL::LDS + f * EL::NFPK, EL::LDS,
                         S.Wf + f * EL::NPR * EL::LDL, EL::LDL, EL::NFPK / 4, lane);
      const int col = tile * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
#pragma unroll
        for (int x = 0; x < DIM; ++x) {
          double cf[EL::NS];
#pragma unroll
          for (int s = 0; s < EL::NS; ++s) cf[s] = W.coef[e][x][s];
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
      __syncwarp();
    }
    wb = wb_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace dgb
