// TMA-staged kernels of the flux arrangement (round 2).
//
// ncu on k_nsdiv3 (profiles/r02_ncu_pass2_occupancy.md): the L1/LSU pipe is what saturates first
// (62 % of its wavefront peak with 8 warps; at 12 warps the warps stall on `mio_throttle` and the
// kernel gets SLOWER).  A quarter of those wavefronts and ~10 % of the warp instructions are the
// LDGSTS copies that stage a block's own rows (28 per lane and block for 3D p3, 70 for p4 where the
// odd row length forces 8-byte copies).  Here a block's rows arrive by the Tensor Memory
// Accelerator instead: the state and the flux planes are described ONCE per launch as 2-D tensors
// (plane, element*Np + node) and a block's rows of ALL planes are one box
// [planes] x [KW*Np doubles] -- one `cp.async.bulk.tensor.2d` (SASS UTMALDG) issued by one lane,
// completion on an mbarrier, no registers, no LSU wavefronts, no address arithmetic.  The box lands
// as [plane][element][node], which IS a DMMA operand layout: column (field c, element e) of
// reference direction r starts at ((r*C + c)*BOXW + e*Np), K runs over the nodes.
//
// k_nsdiv8 = pass 2 (operators.py: dg_ns_div), same arithmetic in the same order as k_nsdiv3
// (bitwise identical results).
#pragma once
#include "dgb_kernels_flux.cuh"

// The schedule "gathers -> volume half of the contraction -> Rusanov -> lift half" was measured in round 2 (slower:
// pass 2 6.57 vs 6.37 ms at n=94, profiles/r02_pass2_tma.md section 8) and removed.
// 1: the gathers of the next block are issued before the store epilogue of the current one (every round in flight)
#ifndef DGB_DIV8_EARLY
#define DGB_DIV8_EARLY 1
#endif
// face phase as a rolled loop over batches of 3 rounds (no early gathers): -1 automatic (order 4: 64 -> 44 KB of SASS,
// pass 2 -3.6 %; order 3 keeps the unrolled loop with every round in flight: rolled it is 15 % slower), 0 / 1 off / on
// single-domain gathers addressed from opaque plane base pointers (GatherPlanes): pass 2 -0.1 ... -0.9 %
#ifndef DGB_DIV8_PLANEBASE
#define DGB_DIV8_PLANEBASE 1
#endif
#ifndef DGB_DIV8_ROLLED
#define DGB_DIV8_ROLLED -1
#endif
#ifndef DGB_DIV8_NB
#define DGB_DIV8_NB 0              // 0: every round of a block in flight together (8 warps) / one round (more warps)
#endif

#include <cuda.h>

namespace dgb {

__device__ __forceinline__ unsigned smem_addr_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init_(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test_(unsigned long long* bar, int parity) {
  unsigned ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_addr_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_(unsigned long long* bar, int parity) {
  while (!mbar_test_(bar, parity)) { }
}
// one box of a 2-D tensor (x = element*Np + node, y = plane) -> shared memory
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(smem_addr_u32(smem)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_addr_u32(bar)),
                 "r"(x), "r"(y) : "memory");
}
// contiguous bytes (multiple of 16, both sides 16-byte aligned) -> shared memory
__device__ __forceinline__ void bulk_load_1d(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_addr_u32(bar)) : "memory");
}

// operand fragments from per-lane column offsets (the box layout is not a single row stride when
// the box width is padded)
template <int NI, int MT>
__device__ __forceinline__ void mma_block_off(double (&acc)[MT][NI][2], const double* __restrict__ Xs,
                                              const int (&aoff)[MT], const double* __restrict__ Ws, int ldw,
                                              int ksteps, int lane) {
  const int r = lane >> 2, kq = lane & 3;
  const double* wp = Ws + r * ldw + kq;
#pragma unroll 5
  for (int ks = 0; ks < ksteps; ++ks) {
    double a[MT], b[NI];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) a[mt] = Xs[aoff[mt] + kq + ks * 4];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) b[ni] = wp[ni * 8 * ldw + ks * 4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) dmma884(acc[mt][ni][0], acc[mt][ni][1], a[mt], b[ni]);
  }
}

template <int DIM, int P, int KW>
struct TmaBox {
  using EL = ElemT<DIM, P>;
  // Box width in doubles, a multiple of 16 bytes.  The global address of a box must be 16-byte aligned as well:
  // with an odd Np a block that starts at an odd element is fetched from one double earlier and read at offset 1
  // (box_shift), so the box holds one double more than the block.
  static constexpr int BOXW = (KW * EL::NP + (EL::NP % 2) + 1) / 2 * 2;
  __device__ static __forceinline__ int box_shift(long long e0) { return (EL::NP % 2) ? (int)((e0 * EL::NP) & 1) : 0; }
  static constexpr int NPL_T = DIM * EL::C;                  // flux planes in the T box (the wave speed travels apart)
};

// small per-block inputs, double-buffered, by cp.async as before (a few instructions): face Jacobians,
// connectivity words, 1/J and the block's slice of the gather map (DiscDev::gidx)
template <int DIM, int P, int KW>
struct alignas(16) Div8Geo {
  using EL = ElemT<DIM, P>;
  alignas(16) unsigned gi[KW * EL::NFT];
  double sj[KW][EL::NF];
  long long conn[KW][EL::NF];
  double rj[KW];
};

// Everything a lane needs to know about its face node of round k, packed once per kernel from the
// face-lane code (face_lane_code): bits 0-7 e*NFT + fm (gather-map slot), 8-11 e*NF + f (face slot),
// 12-19 e*NP + jm (own volume node in the box rows), 20-27 e*LDF + fm (operand entry), 28-29 e; < 0: idle lane.
template <int DIM, int P, int KW>
__device__ __forceinline__ int lean_round_word(int flk) {
  using EL = ElemT<DIM, P>;
  if (flk < 0) return -1;
  const int e = flk & 3, f = (flk >> 2) & 3, jm = (flk >> 8) & 255, fm = (flk >> 16) & 255;
  static_assert(KW * EL::NFT <= 256 && KW * EL::NP <= 256 && KW * EL::LDF <= 256 && KW * EL::NF <= 16, "packing");
  return (e * EL::NFT + fm) | ((e * EL::NF + f) << 8) | ((e * EL::NP + jm) << 12) | ((e * EL::LDF + fm) << 20) | (e << 28);
}

// Plane base pointers of the gathered arrays as kernel parameters (constant bank): written q + c*stride, the compiler
// chains the 64-bit addresses from plane to plane (2 dependent instructions per value); opaque bases make every
// address one independent multiply-add on the lane's offset.
template <int C>
struct GatherPlanes {
  const double* q[C];
  const double* t[C];
  const double* lam;
};

// Lean face phase (pass 2): the neighbour's node comes from the precomputed gather map instead of being decoded
// from the connectivity word through the face-node / permutation tables, every lane carries its per-round
// constants in one register, and a face selects ONE plane group of T.  Same arithmetic as div_face_phase.
// the two halves of the lean face phase for rounds [k0, k0 + NB): issue the gathers / turn them into operand rows
template <int DIM, int P, int KW, int NB, bool GH>
__device__ __forceinline__ void face_lean_issue(int k0, const int (&rw)[face_rounds<DIM, P, KW>()], const Div8Geo<DIM, P, KW>& g,
                                                const DiscDev& d, const double* __restrict__ q, const double* __restrict__ T,
                                                const double* __restrict__ ghost, const double* __restrict__ Tghost,
                                                long long e0, int nel, double (&qp)[NB][ElemT<DIM, P>::C],
                                                double (&nbr)[NB][ElemT<DIM, P>::C], double (&lam_p)[NB], int (&hi)[NB],
                                                const GatherPlanes<ElemT<DIM, P>::C>& gp) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int LAMPL = FluxT<DIM, P>::LAMPL;
  const long long ps_own = d.E * NP;
  const unsigned enp = (unsigned)ps_own;
  const long long* connf = &g.conn[0][0];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    hi[b] = -1;                      // upper half of the connectivity word (neighbour face, bc kind); < 0: nothing to do
    if (k0 + b < NR) {
      const int w = rw[k0 + b];
      if (w >= 0 && ((w >> 28) & 3) < nel) {
#ifdef DGB_EXP_LOCALGATHER
        const unsigned gi = (unsigned)(e0 * NP) + ((w >> 12) & 255);      // timing experiment: own node
#else
        const unsigned gi = g.gi[w & 255];
#endif
        hi[b] = (int)(connf[(w >> 8) & 15] >> 32);
        const int nf = hi[b] & 7;
        const int grp = nf == 0 ? DIM : nf - 1;
#if DGB_DIV8_PLANEBASE
        if (!GH) {
          // single domain: every address is (plane base, uniform across the warp) + one per-lane offset -- no
          // serial chain of 64-bit address updates from plane to plane
          const long long goff = (long long)(grp * C) * ps_own + gi;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            qp[b][c] = __ldg(gp.q[c] + gi);          // q and T are read-only in this kernel (the C ABI rejects
            nbr[b][c] = __ldg(gp.t[c] + goff);        // RK outputs that alias q)
          }
          lam_p[b] = __ldg(gp.lam + gi);
          continue;
        }
#endif
        const bool in_ghost = GH && gi >= enp;
        const long long ps = in_ghost ? d.G * NP : ps_own;
        const double* qb = in_ghost ? ghost + (gi - enp) : q + gi;
        const double* tb = in_ghost ? Tghost + (gi - enp) : T + gi;
        const double* tg = tb + (long long)(grp * C) * ps;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          qp[b][c] = DGB_GLD(qb + c * ps);
          nbr[b][c] = DGB_GLD(tg + c * ps);
        }
        lam_p[b] = DGB_GLD(tb + LAMPL * ps);
      }
    }
  }
}

template <int DIM, int P, int KW, int NB>
__device__ __forceinline__ void face_lean_consume(int k0, const int (&rw)[face_rounds<DIM, P, KW>()], const Div8Geo<DIM, P, KW>& g,
                                                  const double* __restrict__ Qb, const double* __restrict__ Lam,
                                                  double* __restrict__ Fs, const DiscDev& d, const double* __restrict__ T,
                                                  const Phys& ph, long long e0, const double (&qp)[NB][ElemT<DIM, P>::C],
                                                  const double (&nbr)[NB][ElemT<DIM, P>::C], const double (&lam_p)[NB],
                                                  const int (&hi)[NB]) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int BOXW = TmaBox<DIM, P, KW>::BOXW;
  const long long ps_own = d.E * NP;
  const double* sjf = &g.sj[0][0];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (k0 + b < NR && hi[b] >= 0) {
      const int w = rw[k0 + b];
      const int cofs = (w >> 8) & 15, qofs = (w >> 12) & 255, fofs = (w >> 20) & 255;
      const int nf = hi[b] & 7, bc = (hi[b] >> 6) & 3;
      const double sj = sjf[cofs];
      const double lam_m = Lam[qofs];
      double qm[C];
#pragma unroll
      for (int c = 0; c < C; ++c) qm[c] = Qb[c * BOXW + qofs];
      double* fs = Fs + fofs;
      if (bc == 0) {
        const double hs = nf == 0 ? 0.5 : -0.5;
        const double pen = 0.5 * (sj * fmax(lam_m, lam_p[b]));
#pragma unroll
        for (int c = 0; c < C; ++c) fs[c * (KW * EL::LDF)] = hs * nbr[b][c] - pen * (qm[c] - qp[b][c]);
      } else {
        const int e = (w >> 28) & 3, f = cofs - e * NF, jm = qofs - e * NP;
        VecC<DIM> a_;
#pragma unroll
        for (int c = 0; c < C; ++c) a_.v[c] = qm[c];
        const VecC<DIM> fb = boundary_operand<DIM>(bc, f, a_, T + (e0 + e) * NP + jm, ps_own, lam_m, sj,
                                                   d.normals + (e0 + e) * NF + f, d.E * NF, ph);
#pragma unroll
        for (int c = 0; c < C; ++c) fs[c * (KW * EL::LDF)] = fb.v[c];
      }
    }
  }
}

template <int DIM, int P, int KW, int NB, bool GH>
__device__ __forceinline__ void div_face_lean(const int (&rw)[face_rounds<DIM, P, KW>()], const Div8Geo<DIM, P, KW>& g,
                                              const double* __restrict__ Qb, const double* __restrict__ Lam,
                                              double* __restrict__ Fs, const DiscDev& d,
                                              const double* __restrict__ q, const double* __restrict__ T,
                                              const double* __restrict__ ghost, const double* __restrict__ Tghost,
                                              const Phys& ph, long long e0, int nel,
                                              const GatherPlanes<ElemT<DIM, P>::C>& gp) {
  constexpr int C = ElemT<DIM, P>::C;
  constexpr int NR = face_rounds<DIM, P, KW>();
#pragma unroll
  for (int k0 = 0; k0 < NR; k0 += NB) {          // unrolled: rw[] stays in registers
    double qp[NB][C], nbr[NB][C], lam_p[NB];
    int hi[NB];
    face_lean_issue<DIM, P, KW, NB, GH>(k0, rw, g, d, q, T, ghost, Tghost, e0, nel, qp, nbr, lam_p, hi, gp);
    face_lean_consume<DIM, P, KW, NB>(k0, rw, g, Qb, Lam, Fs, d, T, ph, e0, qp, nbr, lam_p, hi);
  }
}

// The same with a ROLLED loop over the batches (the per-round words come from shared memory instead of registers):
// a third of the code for order 4, where the kernel is twice the size of the L1.5 instruction cache
template <int DIM, int P, int KW, int NB, bool GH>
__device__ __forceinline__ void div_face_lean_rolled(const int* __restrict__ flc, int lane, const Div8Geo<DIM, P, KW>& g,
                                                     const double* __restrict__ Qb, const double* __restrict__ Lam,
                                                     double* __restrict__ Fs, const DiscDev& d,
                                                     const double* __restrict__ q, const double* __restrict__ T,
                                                     const double* __restrict__ ghost, const double* __restrict__ Tghost,
                                                     const Phys& ph, long long e0, int nel,
                                                     const GatherPlanes<ElemT<DIM, P>::C>& gp) {
  constexpr int C = ElemT<DIM, P>::C;
  constexpr int NR = face_rounds<DIM, P, KW>();
#pragma unroll 1
  for (int k0 = 0; k0 < NR; k0 += NB) {
    int rwb[NR];
#pragma unroll
    for (int b = 0; b < NR; ++b) rwb[b] = (b < NB && k0 + b < NR) ? lean_round_word<DIM, P, KW>(flc[(k0 + b) * 32 + lane]) : -1;
    double qp[NB][C], nbr[NB][C], lam_p[NB];
    int hi[NB];
    face_lean_issue<DIM, P, KW, NB, GH>(0, rwb, g, d, q, T, ghost, Tghost, e0, nel, qp, nbr, lam_p, hi, gp);
    face_lean_consume<DIM, P, KW, NB>(0, rwb, g, Qb, Lam, Fs, d, T, ph, e0, qp, nbr, lam_p, hi);
  }
}

template <int DIM, int P, int KW>
struct alignas(128) Div8Warp {
  using EL = ElemT<DIM, P>;
  using BX = TmaBox<DIM, P, KW>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  alignas(128) double Tb[BX::NPL_T * BX::BOXW + 8];     // [plane r*C + c][element][node]  (+8: K padding of the last column)
  alignas(128) double Qb[EL::C * BX::BOXW];             // [field][element][node]
  alignas(128) double Lam[BX::BOXW];                    // wave speed rows of the block
  double Fs[NCOL * EL::LDF];
  // mixtures: Arrhenius rate at the block's nodes; it lives in the block's gather-map slice (dead once the gathers
  // are issued) when that is large enough -- the 480 bytes decide between 7 and 8 warps for 3D p3
  static constexpr bool OM_ALIAS = 2 * EL::NP <= EL::NFT;
  double Om[(DGB_NSPEC > 0 && !OM_ALIAS) ? KW * EL::NP : 1];
  Div8Geo<DIM, P, KW> geo[2];
  unsigned long long bar_q, bar_t;
};

template <int DIM, int P, int KW, int NWARPS>
struct Div8Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Div8Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

template <int DIM, int P, int KW, int NWARPS, bool GH>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsdiv8(DiscDev d, const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_t,
         const __grid_constant__ CUtensorMap map_l, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter, const GatherPlanes<ElemT<DIM, P>::C> gp) {
  using EL = ElemT<DIM, P>;
  using WS = Div8Warp<DIM, P, KW>;
  using BX = TmaBox<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();
  // face nodes per lane with their gathers in flight together: all NR rounds of a block at 8 warps (11 values per
  // node: 88 registers for 3D p3), one round at 9-12 warps (168 registers)
  constexpr bool ROLLED = DGB_DIV8_ROLLED >= 0 ? DGB_DIV8_ROLLED != 0 : (NP > 20 && DGB_NSPEC == 0);
  constexpr int NB = DGB_DIV8_NB > 0 ? DGB_DIV8_NB : (ROLLED ? (C <= 5 ? 3 : 2) : (NWARPS > 8 ? 1 : (C <= 5 ? NR : 2)));     // 2 C + 1 values per node
  constexpr int BOXW = BX::BOXW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div8Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv2[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  {
    double* z = reinterpret_cast<double*>(&W);
    for (int n = lane; n < (int)(sizeof(WS) / 8); n += 32) z[n] = 0.0;
  }
  __syncwarp();
  if (lane == 0) { mbar_init_(&W.bar_q, 1); mbar_init_(&W.bar_t, 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");     // the zero fill above precedes the TMA writes
  __syncthreads();
  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  __syncthreads();

  // per-lane operand column offsets inside a box group of C planes (constant for the whole kernel)
  int aoff[WS::NTILE];
#pragma unroll
  for (int mt = 0; mt < WS::NTILE; ++mt) {
    int col = mt * 8 + (lane >> 2);
    if (col >= WS::NCOL) col = WS::NCOL - 1;        // padding column: any finite rows, its accumulators are dropped
    const int c = col / KW, e = col - c * KW;
    aoff[mt] = c * BOXW + e * NP;
  }
  int foff[WS::NTILE];
#pragma unroll
  for (int mt = 0; mt < WS::NTILE; ++mt) {
    int col = mt * 8 + (lane >> 2);
    if (col >= WS::NCOL) col = WS::NCOL - 1;
    foff[mt] = col * EL::LDF;
  }

  int rw[NR];                        // per-round constants of this lane (div_face_lean)
#pragma unroll
  for (int k = 0; k < NR; ++k) rw[k] = lean_round_word<DIM, P, KW>(S.flc[k * 32 + lane]);

  auto nel_of = [&](long long wbx) -> int {
    if (wbx >= nwblocks) return 0;
    const long long e = ebeg + wbx * KW;
    return (int)((eend - e) < (long long)KW ? (eend - e) : (long long)KW);
  };
  auto issue_q = [&](long long e0) {                  // state box + wave-speed rows -> bar_q   (lane 0)
    mbar_expect_tx(&W.bar_q, (unsigned)((C + 1) * BOXW * 8));
    const int x = (int)(e0 * NP) - BX::box_shift(e0);
    tma_load_2d(W.Qb, &map_q, x, 0, &W.bar_q);
    tma_load_2d(W.Lam, &map_l, x, 0, &W.bar_q);
  };
  auto issue_t = [&](long long e0) {                  // flux-plane box -> bar_t   (lane 0)
    mbar_expect_tx(&W.bar_t, (unsigned)(BX::NPL_T * BOXW * 8));
    tma_load_2d(W.Tb, &map_t, (int)(e0 * NP) - BX::box_shift(e0), 0, &W.bar_t);
  };
  auto stage_geo = [&](Div8Geo<DIM, P, KW>& g, long long e0, int nelx) {
    if (lane < nelx * NF) {
      cp_async8(&g.sj[0][lane], d.sj + e0 * NF + lane);
      cp_async8(&g.conn[0][lane], d.conn + e0 * NF + lane);
    }
    if (lane < nelx) cp_async8(&g.rj[lane], d.rj + e0 + lane);
    stage_gather_map<DIM, EL::NFT, EL::NFP>(g.gi, d.gidx, e0, nelx, lane);
  };

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  if (wb >= nwblocks) return;
  // EARLY: the gathers of block b+1 are issued right after the contraction of block b, before its store epilogue,
  // and consumed at the top of the next iteration -- their L2 round trip (ncu: 17 % of the stall samples sit on the
  // first use of a gathered value) runs under the epilogue, the ticket, the staging and the mbarrier waits.
  constexpr bool EARLY = (DGB_DIV8_EARLY != 0) && NB >= NR && !ROLLED;
  constexpr int NG = EARLY ? NB : 1;
  double gqp[NG][C], gnb[NG][C], glam[NG];
  int ghi[NG];
  {
    const long long e0 = ebeg + wb * KW;
    if (lane == 0) { issue_q(e0); issue_t(e0); }
    stage_geo(W.geo[0], e0, nel_of(wb));
    cp_async_commit();
    if (EARLY) {
      cp_async_wait<0>();
      __syncwarp();
      face_lean_issue<DIM, P, KW, NG, GH>(0, rw, W.geo[0], d, q, T, ghost, Tghost, e0, nel_of(wb), gqp, gnb, glam, ghi, gp);
    }
  }
  TicketStream tks;
  tickets_init(tks, wb, ticket_counter(counter, S.fn, lane), lane);

  for (int it = 0;; ++it) {
    const int buf = it & 1, par = it & 1;
    const long long e0 = ebeg + wb * KW;
    const int nel = nel_of(wb);
    const long long wb_next = tickets_next(tks, wstride, ticket_counter(counter, S.fn, lane), lane);
    const int nel1 = nel_of(wb_next);
    const long long e1 = ebeg + wb_next * KW;
    if (nel1 > 0) stage_geo(W.geo[buf ^ 1], e1, nel1);
    cp_async_commit();
    if (!EARLY) {
      cp_async_wait<1>();                // gather map, connectivity, face Jacobians of this block
      __syncwarp();
    }
    const int sh = BX::box_shift(e0);
    mbar_wait_(&W.bar_q, par);           // state + wave speed of this block
#ifndef DGB_EXP_NOFACE              // timing experiments only (results invalid)
    if (EARLY)
      face_lean_consume<DIM, P, KW, NG>(0, rw, W.geo[buf], W.Qb + sh, W.Lam + sh, W.Fs, d, T, ph, e0, gqp, gnb, glam, ghi);
    else if (ROLLED)
      div_face_lean_rolled<DIM, P, KW, NB, GH>(S.flc, lane, W.geo[buf], W.Qb + sh, W.Lam + sh, W.Fs, d, q, T, ghost, Tghost, ph, e0, nel, gp);
    else
      div_face_lean<DIM, P, KW, NB, GH>(rw, W.geo[buf], W.Qb + sh, W.Lam + sh, W.Fs, d, q, T, ghost, Tghost, ph, e0, nel, gp);
#endif
    double rj[WS::NTILE];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) rj[mt] = W.geo[buf].rj[(mt * 8 + (lane >> 2)) % KW];
#if DGB_NSPEC > 0
    // chemistry: the Arrhenius rate at every node of the block, from the state box while it is still here
    double* om = WS::OM_ALIAS ? reinterpret_cast<double*>(W.geo[buf].gi) : W.Om;
    __syncwarp();                        // (aliased: every lane has read its gather-map words)
    for (int n = lane; n < KW * NP; n += 32) {
      const int e = n / NP;
      if (e < nel) {
        double qq[C];
#pragma unroll
        for (int c = 0; c < C; ++c) qq[c] = W.Qb[c * BOXW + n + sh];
        om[n] = pw_arrhenius<DIM>(qq, ph);
      }
    }
#endif
    __syncwarp();                        // every lane has read the state box: the next one may land on it
    if (nel1 > 0 && lane == 0) issue_q(e1);
    mbar_wait_(&W.bar_t, par);           // flux planes of this block

    // ---- tensor-core contraction: volume rows straight from the box, then the face operand rows ----
    double acc[WS::NTILE][EL::NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
#ifndef DGB_EXP_NOMMA
#pragma unroll
    for (int r = 0; r < DIM; ++r)
      mma_block_off<EL::NI, WS::NTILE>(acc, W.Tb + r * (C * BOXW) + sh, aoff, S.Wv + r * EL::NPK, EL::LDV, EL::NPK / 4, lane);
    mma_block_off<EL::NI, WS::NTILE>(acc, W.Fs, foff, S.Wl, EL::LDF, EL::KF / 4, lane);
#else
    acc[0][0][0] = W.Tb[aoff[0] + sh + lane] + W.Fs[foff[0] + lane];
#endif
    __syncwarp();                        // operand rows consumed
    if (nel1 > 0 && lane == 0) issue_t(e1);
    if (EARLY && nel1 > 0) {
      cp_async_wait<0>();                // gather map + connectivity of the next block (staged at the top of this one)
      __syncwarp();
#ifndef DGB_EXP_NOFACE
      face_lean_issue<DIM, P, KW, NG, GH>(0, rw, W.geo[buf ^ 1], d, q, T, ghost, Tghost, e1, nel1, gqp, gnb, glam, ghi, gp);
#endif
    }

    // ---- 1/J (+ chemistry) and the (RK-fused) store ----
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
#if DGB_NSPEC > 0
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col < WS::NCOL ? col - c * KW : 0;
      const double sgn = c == 2 + DIM + ph.ra ? -1.0 : (c == 2 + DIM + ph.rb ? 1.0 : 0.0);     // species a -> species b
#endif
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) {
        acc[mt][ni][0] *= rj[mt]; acc[mt][ni][1] *= rj[mt];
#if DGB_NSPEC > 0
        const int i = ni * 8 + 2 * (lane & 3);
        if (sgn != 0.0 && e < nel) {
          if (i < NP) acc[mt][ni][0] += sgn * om[e * NP + i];
          if (i + 1 < NP) acc[mt][ni][1] += sgn * om[e * NP + i + 1];
        }
#endif
      }
    }
    store_block<NP, KW, WS::NCOL, WS::NTILE, EL::NI>(ep, acc, E, e0, nel, lane);
    if (nel1 == 0) break;
    wb = wb_next;
  }
  cp_async_wait<0>();
}

}  // namespace dgb
