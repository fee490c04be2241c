// Asynchronous-pipeline versions of the fused DG kernels (the default path).
//
// Same math and shared-memory operand layouts as dgb_kernels.cuh, but no compute phase ever waits
// on HBM/L2 latency (ncu of the first version: 34-41% of stall samples long_scoreboard, 22-31%
// barrier; per-phase cycle counters: staging phases were 16% / 42% of wall time):
//   * per-block geometry + connectivity arrive by cp.async into a double buffer one block ahead;
//   * the face-neighbour values are gathered by cp.async (LDGSTS) into a shared staging area at the
//     top of the block and only consumed after the volume work has covered their latency;
//   * k_rhs2: the block's own nodal inputs for the NEXT block are loaded into registers right after
//     phase 2 and ride through the tensor-core phase;  k_grad2: the own rows of the next block
//     arrive by cp.async into a second Qs buffer while the current block computes.
#pragma once
#include "dgb_kernels.cuh"

namespace dgb {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int DIM, int P, int K>
__device__ __forceinline__ void stage_geo_async(GeoSmem<DIM, P, K>& g, const DiscDev& d, long long e0, int nel,
                                                int tid, int nthreads) {
  using EL = ElemT<DIM, P>;
  for (int n = tid; n < DIM * DIM * K; n += nthreads) {
    const int rx = n / K, e = n - rx * K;
    if (e < nel) cp_async8(&g.drdx[rx][e], d.drdx + (long long)rx * d.E + e0 + e);
  }
  for (int n = tid; n < DIM * K * EL::NF; n += nthreads) {
    const int x = n / (K * EL::NF), ef = n - x * (K * EL::NF);
    if (ef < nel * EL::NF) cp_async8(&g.nrm[x][0][ef], d.normals + ((long long)x * d.E + e0) * EL::NF + ef);
  }
  for (int n = tid; n < nel * EL::NF; n += nthreads) {
    cp_async8(&g.fsc[0][n], d.fscale + e0 * EL::NF + n);
    cp_async8(&g.conn[0][n], d.conn + e0 * EL::NF + n);
  }
}

// issue the cp.async gathers of the plus-side values of every face node of the block:
//   NB[(pl*K + e)*NFT + fm] = plane_pl[neighbour element][neighbour node]
template <int DIM, int P, int K, int NPL>
__device__ __forceinline__ void gather_async(double* NB, const GeoSmem<DIM, P, K>& geo, const int* fn, const int* perm,
                                             const double* p0, const double* g0, const double* p0_ghost,
                                             const double* g0_ghost, long long E, long long G, int nel, int tid,
                                             int nthreads) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NFP = EL::NFP, NFT = EL::NFT;
  for (int n = tid; n < nel * NFT; n += nthreads) {
    const int e = n / NFT, fm = n - e * NFT;
    const int f = fm / NFP, m = fm - f * NFP;
    const long long cn = geo.conn[e][f];
    const long long nb = DGB_CONN_NB(cn);
    const int jp = fn[DGB_CONN_NF(cn) * NFP + perm[DGB_CONN_PERM(cn) * NFP + m]];
    const bool in_ghost = nb >= E;
    const long long pE = in_ghost ? G : E;
    const long long off = (in_ghost ? nb - E : nb) * NP + jp;
    const long long pstride = pE * NP;
    const double* src = (in_ghost ? p0_ghost : p0) + off;
    double* dst = NB + e * NFT + fm;
#pragma unroll
    for (int pl = 0; pl < C; ++pl) cp_async8(dst + pl * (K * NFT), src + pl * pstride);
    if (NPL > C) {
      const double* gsrc = (in_ghost ? g0_ghost : g0) + off;
#pragma unroll
      for (int pl = 0; pl < NPL - C; ++pl) cp_async8(dst + (C + pl) * (K * NFT), gsrc + pl * pstride);
    }
  }
}

// ------------------------------------------------------------------------------------------
// right-hand side (Euler / Navier-Stokes second pass)
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int K, bool VISCOUS>
struct Rhs2Smem {
  using EL = ElemT<DIM, P>;
  static constexpr int NPL = VISCOUS ? (DIM + 1) * EL::C : EL::C;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  double Gs[EL::C * K * EL::LDV];
  double Fs[EL::C * K * EL::LDF];
  double Lam[K * EL::NP];
  double NB[NPL * K * EL::NFT];
  GeoSmem<DIM, P, K> geo[2];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int K, int NW, bool VISCOUS, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
k_rhs2(DiscDev d, const double* __restrict__ q, const double* __restrict__ gq,
       const double* __restrict__ ghost, const double* __restrict__ gghost,
       Epilogue ep, Phys ph, int nblocks) {
  using EL = ElemT<DIM, P>;
  using SM = Rhs2Smem<DIM, P, K, VISCOUS>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NPL = SM::NPL;
  constexpr int NT = NW * 32;
  constexpr int NTILES = C * K / 8;
  static_assert((C * K) % 8 == 0, "columns per block must be a multiple of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < C * K * EL::LDV; n += NT) S.Gs[n] = 0.0;
  for (int n = tid; n < C * K * EL::LDF; n += NT) S.Fs[n] = 0.0;
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];

  // prologue: geometry of the first block, and this thread's first node inputs in registers
  int blk = blockIdx.x;
  int buf = 0;
  double pre[NPL];
  if (blk < nblocks) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    stage_geo_async<DIM, P, K>(S.geo[0], d, e0, nel, tid, NT);
    if (tid < nel * NP) {
#pragma unroll
      for (int c = 0; c < C; ++c) pre[c] = q[((long long)c * E + e0) * NP + tid];
      if (VISCOUS) {
#pragma unroll
        for (int pl = 0; pl < NPL - C; ++pl) pre[C + pl] = gq[((long long)pl * E + e0) * NP + tid];
      }
    }
  }
  cp_async_commit();

  for (; blk < nblocks; blk += gridDim.x, buf ^= 1) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    const GeoSmem<DIM, P, K>& geo = S.geo[buf];
    cp_async_wait<0>();
    __syncthreads();            // geo[buf] landed; previous block's Gs/Fs/NB fully consumed

    // ---- issue the neighbour gathers of this block (consumed in phase 2) ---------------------
    gather_async<DIM, P, K, NPL>(S.NB, geo, S.fn, S.perm, q, gq, ghost, gghost, E, G, nel, tid, NT);
    cp_async_commit();

    // ---- phase 1: volume flux (first round from the register prefetch) ------------------------
    for (int n = tid; n < nel * NP; n += NT) {
      const int e = n / NP, j = n - e * NP;
      double qq[C], g[DIM][C];
      if (n == tid) {
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
        for (int x = 0; x < DIM; ++x) m[x] = geo.drdx[r * DIM + x][e];
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
    cp_async_wait<0>();
    __syncthreads();            // Gs/Lam complete, gathers landed

    // ---- phase 2: numerical flux from staged neighbour values ---------------------------------
    for (int n = tid; n < nel * NFT; n += NT) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const int bc = DGB_CONN_BC(geo.conn[e][f]);
      const int jm = S.fn[f * NFP + m];
      double qm[C];
#pragma unroll
      for (int c = 0; c < C; ++c) qm[c] = q[((long long)c * E + e0 + e) * NP + jm];   // used last (jump term)
      double nrm[DIM];
#pragma unroll
      for (int x = 0; x < DIM; ++x) nrm[x] = geo.nrm[x][e][f];
      const double fs = geo.fsc[e][f];
      const double* nbp = S.NB + e * NFT + fm;
      double qp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) qp[c] = nbp[c * (K * NFT)];
      if (bc != 0) bc_state<DIM, VISCOUS>(bc, qm, nrm, ph, qp);
      Prim<DIM> sp_;
      make_prim<DIM>(qp, ph.gamma, sp_);
      double fnp[C];
      inviscid_normal_flux<DIM>(sp_, nrm, fnp);
      const double lam = fmax(S.Lam[e * NP + jm], wavespeed<DIM>(sp_, ph.gamma));
      if (VISCOUS) {
        double gp[DIM][C], fvn[C];
#pragma unroll
        for (int x = 0; x < DIM; ++x)
#pragma unroll
          for (int c = 0; c < C; ++c) gp[x][c] = nbp[(C + x * C + c) * (K * NFT)];
        // boundary faces: the viscous flux is the interior one, Fv(q-, grad q-) (operators.py)
        if (bc != 0) make_prim<DIM>(qm, ph.gamma, sp_);
        viscous_normal_flux<DIM>(sp_, gp, nrm, ph, fvn);
#pragma unroll
        for (int c = 1; c < C; ++c) fnp[c] -= fvn[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double* grow = S.Gs + (c * K + e) * EL::LDV + jm;
        double own;                       // fscale * (F^- . n): (f == 0) ? sum_r G_r : -G_{f-1}
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

    // ---- prefetch for the next block: geometry (cp.async) and node inputs (registers) ----------
    {
      const int nblk = blk + gridDim.x;
      if (nblk < nblocks) {
        const long long e1 = (long long)nblk * K;
        const int nel1 = (int)((E - e1) < (long long)K ? (E - e1) : (long long)K);
        stage_geo_async<DIM, P, K>(S.geo[buf ^ 1], d, e1, nel1, tid, NT);
        if (tid < nel1 * NP) {
#pragma unroll
          for (int c = 0; c < C; ++c) pre[c] = q[((long long)c * E + e1) * NP + tid];
          if (VISCOUS) {
#pragma unroll
            for (int pl = 0; pl < NPL - C; ++pl) pre[C + pl] = gq[((long long)pl * E + e1) * NP + tid];
          }
        }
      }
      cp_async_commit();
    }
    __syncthreads();            // Fs complete

    // ---- phase 3: tensor-core contraction + (RK-fused) store -----------------------------------
    for (int tile = warp; tile < NTILES; tile += NW) {
      __syncwarp();
      double acc[1][EL::NI][2];
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[0][ni][0] = 0.0; acc[0][ni][1] = 0.0; }
      mma_block<EL::NI, 1>(acc, S.Gs + tile * 8 * EL::LDV, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
      mma_block<EL::NI, 1>(acc, S.Fs + tile * 8 * EL::LDF, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
      const int col = tile * 8 + (lane >> 2);
      const int c = col / K, e = col - c * K;
      if (e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) {
          const int i = ni * 8 + 2 * (lane & 3);
          store_pair<NP>(ep, rowbase + i, i, acc[0][ni][0], acc[0][ni][1]);
        }
      }
    }
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------
// Navier-Stokes first pass (BR1 gradient)
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int K>
struct Grad2Smem {
  using EL = ElemT<DIM, P>;
  double Wq[DIM * EL::NPR * EL::LDQ];
  double Wf[EL::NF * EL::NPR * EL::LDL];
  double Qs[2][EL::C * K * EL::LDQ];
  double Ss[EL::C * K * EL::LDS];
  double NB[EL::C * K * EL::NFT];
  double coef[K][DIM][EL::NS];
  GeoSmem<DIM, P, K> geo[2];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
};

template <int DIM, int P, int K>
__device__ __forceinline__ void stage_rows_async(double* Qs, const double* q, long long E, long long e0, int nel,
                                                 int tid, int nthreads) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP;
  for (int n = tid; n < C * nel * NP; n += nthreads) {
    const int c = n / (nel * NP), ej = n - c * (nel * NP);
    const int e = ej / NP, j = ej - e * NP;
    cp_async8(Qs + (c * K + e) * EL::LDQ + j, q + ((long long)c * E + e0) * NP + ej);
  }
}

template <int DIM, int P, int K, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
k_grad2(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
        double* __restrict__ grad, Phys ph, int nblocks) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NI = EL::NI;
  constexpr int NT = NW * 32;
  constexpr int NTILES = C * K / 8;
  constexpr int TPW = (NTILES + NW - 1) / NW;      // tiles per warp (register-resident accumulators)
  static_assert((C * K) % 8 == 0, "columns per block must be a multiple of 8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Grad2Smem<DIM, P, K>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < DIM * EL::NPR * EL::LDQ; n += NT) S.Wq[n] = d.Wq[n];
  for (int n = tid; n < NF * EL::NPR * EL::LDL; n += NT) S.Wf[n] = d.Wf[n];
  for (int n = tid; n < 2 * C * K * EL::LDQ; n += NT) S.Qs[0][n] = 0.0;
  for (int n = tid; n < C * K * EL::LDS; n += NT) S.Ss[n] = 0.0;
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  __syncthreads();              // zero fill before any cp.async lands in Qs

  int blk = blockIdx.x;
  int buf = 0;
  if (blk < nblocks) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    stage_geo_async<DIM, P, K>(S.geo[0], d, e0, nel, tid, NT);
    stage_rows_async<DIM, P, K>(S.Qs[0], q, E, e0, nel, tid, NT);
  }
  cp_async_commit();

  for (; blk < nblocks; blk += gridDim.x, buf ^= 1) {
    const long long e0 = (long long)blk * K;
    const int nel = (int)((E - e0) < (long long)K ? (E - e0) : (long long)K);
    const GeoSmem<DIM, P, K>& geo = S.geo[buf];
    const double* Qs = S.Qs[buf];
    cp_async_wait<0>();
    __syncthreads();            // Qs[buf], geo[buf] landed; previous block fully consumed

    // gathers of this block, then the next block's rows + geometry
    gather_async<DIM, P, K, C>(S.NB, geo, S.fn, S.perm, q, q, ghost, ghost, E, G, nel, tid, NT);
    cp_async_commit();
    {
      const int nblk = blk + gridDim.x;
      if (nblk < nblocks) {
        const long long e1 = (long long)nblk * K;
        const int nel1 = (int)((E - e1) < (long long)K ? (E - e1) : (long long)K);
        stage_geo_async<DIM, P, K>(S.geo[buf ^ 1], d, e1, nel1, tid, NT);
        stage_rows_async<DIM, P, K>(S.Qs[buf ^ 1], q, E, e1, nel1, tid, NT);
      }
      cp_async_commit();
    }
    for (int n = tid; n < nel * DIM * EL::NS; n += NT) {
      const int e = n / (DIM * EL::NS), xs = n - e * (DIM * EL::NS);
      const int x = xs / EL::NS, s = xs - x * EL::NS;
      S.coef[e][x][s] = s < DIM ? -geo.drdx[s * DIM + x][e] : geo.fsc[e][s - DIM] * geo.nrm[x][e][s - DIM];
    }

    // ---- volume part on the tensor cores while the gathers are in flight ----------------------
    double accT[TPW][DIM][1][NI][2];
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + t * NW;
#pragma unroll
      for (int r = 0; r < DIM; ++r)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { accT[t][r][0][ni][0] = 0.0; accT[t][r][0][ni][1] = 0.0; }
      if (tile < NTILES) {
#pragma unroll
        for (int r = 0; r < DIM; ++r)
          mma_block<NI, 1>(accT[t][r], Qs + tile * 8 * EL::LDQ, EL::LDQ, S.Wq + r * EL::NPR * EL::LDQ, EL::LDQ,
                           EL::NPK / 4, lane);
      }
    }
    cp_async_wait<1>();         // this block's gathers (the next block's rows may still be in flight)
    __syncthreads();

    // ---- face averages q* = (q- + q+)/2 with boundary states -----------------------------------
    for (int n = tid; n < nel * NFT; n += NT) {
      const int e = n / NFT, fm = n - e * NFT;
      const int f = fm / NFP, m = fm - f * NFP;
      const int bc = DGB_CONN_BC(geo.conn[e][f]);
      const int jm = S.fn[f * NFP + m];
      double qm[C], qp[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        qm[c] = Qs[(c * K + e) * EL::LDQ + jm];
        qp[c] = S.NB[(c * K + e) * NFT + fm];
      }
      if (bc != 0) {
        double nrm[DIM];
#pragma unroll
        for (int x = 0; x < DIM; ++x) nrm[x] = geo.nrm[x][e][f];
        bc_state<DIM, true>(bc, qm, nrm, ph, qp);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) S.Ss[(c * K + e) * EL::LDS + f * EL::NFPK + m] = 0.5 * (qm[c] + qp[c]);
    }
    __syncthreads();

    // ---- lift part, metric combination, store ---------------------------------------------------
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + t * NW;
      if (tile >= NTILES) continue;
      double accU[NF][1][NI][2];
#pragma unroll
      for (int s = 0; s < NF; ++s)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { accU[s][0][ni][0] = 0.0; accU[s][0][ni][1] = 0.0; }
#pragma unroll
      for (int f = 0; f < NF; ++f)
        mma_block<NI, 1>(accU[f], S.Ss + tile * 8 * EL::LDS + f * EL::NFPK, EL::LDS,
                         S.Wf + f * EL::NPR * EL::LDL, EL::LDL, EL::NFPK / 4, lane);
      const int col = tile * 8 + (lane >> 2);
      const int c = col / K, e = col - c * K;
      if (e < nel) {
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
            for (int s = 0; s < DIM; ++s) { v0 += cf[s] * accT[t][s][0][ni][0]; v1 += cf[s] * accT[t][s][0][ni][1]; }
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
    }
  }
  cp_async_wait<0>();
}

}  // namespace dgb
