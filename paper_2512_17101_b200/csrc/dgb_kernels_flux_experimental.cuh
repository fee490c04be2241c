// Experimental variants of pass 2 of the flux arrangement (k_nsdiv4 / k_nsdiv5 / k_nsdiv6).
//
// All three are correct (each passed the full GPU test suite when it was measured) and all three are
// SLOWER than k_nsdiv3 on B200; they are kept as the record of what was tried
// (profiles/r01_flux_variants.md) and are compiled only with -DDGB_EXPERIMENTAL=1
// (scripts/ab_variants.py), then selected at run time with DGB_DIV_KERNEL=4|5|6.
//   k_nsdiv4  producer/consumer warp pairs, mbarrier hand-off           3.15-4.0 ms vs 2.62 ms (n=64)
//   k_nsdiv5  gathers of block i+1 issued before the DMMA of block i    3.49 ms
//   k_nsdiv6  TMA bulk copies (cp.async.bulk, UBLKCP) for all staging   2.77 ms
#pragma once
#include "dgb_kernels_flux.cuh"
#if DGB_T_RECORD
#error "the experimental pass-2 kernels address the flux planes plane-major only"
#endif

namespace dgb {

// ------------------------------------------------------------------------------------------
// pass 2, producer/consumer version.
//
// ncu on k_nsdiv3 (8 warps, 235 registers): 2.0 warps per scheduler, 0.34 eligible, 6.8 cycles between
// two issues of a warp -- each warp alternates between a latency-bound gather phase and a DMMA phase
// and there are too few warps to cover one with the other.  Here a block is handled by a PAIR of
// warps: the producer stages q/lam/connectivity, gathers the neighbour values and writes the face
// operand rows Fs (double-buffered); the consumer streams the T rows, runs the DMMA contraction and
// stores.  Neither holds the other's registers (gather values vs. accumulators), so 16 warps fit
// where 8 did, and the two phases of consecutive blocks overlap by construction.  Hand-off: two
// mbarriers per buffer (full / empty) in shared memory; block ids travel through a 4-slot mailbox.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}"
      ::"r"(a), "r"(parity) : "memory");
}

template <int DIM, int P, int KW>
struct alignas(16) Div4Pair {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  double Ts[NCOL * EL::LDV];
  double Fs[2][NCOL * EL::LDF];
  Div3Small<DIM, P, KW> sm[2];          // producer-private
  unsigned long long full[2], empty[2];
  long long blk[4];                     // block id of block i at slot i & 3
};

template <int DIM, int P, int KW, int NPAIR>
struct Div4Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Div4Pair<DIM, P, KW> w[NPAIR];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

template <int DIM, int P, int KW, int NPAIR>
__global__ void __launch_bounds__(NPAIR * 64, 1)
k_nsdiv4(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Div4Pair<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NPAIR * 64;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int NB = DGB_DIV_NB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div4Smem<DIM, P, KW, NPAIR>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp >= NPAIR;
  const int pair = producer ? warp - NPAIR : warp;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv2[n];
  for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  for (int n = tid; n < NPAIR * (int)(sizeof(WS) / 8); n += NT) reinterpret_cast<double*>(&S.w[0])[n] = 0.0;
  __syncthreads();
  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  WS& W = S.w[pair];
  const long long wstride = (long long)gridDim.x * NPAIR;
  const long long wb0 = (long long)blockIdx.x * NPAIR + pair;
  if (!producer && lane == 0) {
    mbar_init(&W.full[0], 32); mbar_init(&W.full[1], 32);
    mbar_init(&W.empty[0], 32); mbar_init(&W.empty[1], 32);
    W.blk[0] = wb0;
  }
  __syncthreads();
  if (wb0 >= nwblocks) return;

  if (producer) {
    // ================================ producer warp ================================
    long long wb = wb0;
    {
      const long long e0 = ebeg + wb * KW;
      div_stage_small<DIM, P, KW>(W.sm[0], d, q, T, e0, (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW), lane);
      cp_async_commit();
    }
    unsigned long long ticket = draw_ticket(counter, lane);
    for (int i = 0;; ++i) {
      const int buf = i & 1;
      const long long e0 = ebeg + wb * KW;
      const int nel = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
      const long long wb_next = ticket_block(ticket, wstride);
      if (lane == 0) W.blk[(i + 1) & 3] = wb_next;          // published by this block's full-arrive
      const long long e1 = ebeg + wb_next * KW;
      const int nel1 = wb_next < nwblocks ? (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW) : 0;
      if (nel1 > 0) div_stage_small<DIM, P, KW>(W.sm[buf ^ 1], d, q, T, e1, nel1, lane);
      cp_async_commit();
      ticket = draw_ticket(counter, lane);
      cp_async_wait<1>();                 // this block's q / lam / connectivity have landed
      __syncwarp();
      if (i >= 2) mbar_wait(&W.empty[buf], ((i >> 1) - 1) & 1);   // the consumer is done with Fs[buf] of block i-2
      const Div3Small<DIM, P, KW>& M = W.sm[buf];
      double* Fs = W.Fs[buf];
      div_face_phase<DIM, P, KW, DGB_DIV4_NB, (DGB_DIV4_LAZY_EX != 0)>(S.flc, S.fn, S.perm, M, Fs, d, q, T, ghost, Tghost, ph, e0, nel, lane);
      mbar_arrive(&W.full[buf]);          // all 32 lanes arrive: Fs[buf] and blk[(i+1)&3] are published
      if (wb_next >= nwblocks) break;
      wb = wb_next;
    }
    cp_async_wait<0>();
  } else {
    // ================================ consumer warp ================================
    long long wb = wb0;
    {
      const long long e0 = ebeg + wb * KW;
      div_stage_rows<DIM, P, KW>(W.Ts, d, T, e0, (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW), lane);
      cp_async_commit();
    }
    for (int i = 0;; ++i) {
      const int buf = i & 1;
      const long long e0 = ebeg + wb * KW;
      const int nel = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
      double rj[WS::NTILE];
#pragma unroll
      for (int mt = 0; mt < WS::NTILE; ++mt) {
        const int e = (mt * 8 + (lane >> 2)) % KW;
        rj[mt] = e < nel ? d.rj[e0 + e] : 0.0;
      }
      double acc[WS::NTILE][EL::NI][2];
#pragma unroll
      for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
      cp_async_wait<0>();                 // this block's T rows have landed
      __syncwarp();
      mma_block<EL::NI, WS::NTILE>(acc, W.Ts, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
      __syncwarp();                       // T rows consumed
      mbar_wait(&W.full[buf], (i >> 1) & 1);
      const long long wb_next = W.blk[(i + 1) & 3];
      if (wb_next < nwblocks) {           // next block's rows start their trip while the face part is contracted
        const long long e1 = ebeg + wb_next * KW;
        div_stage_rows<DIM, P, KW>(W.Ts, d, T, e1, (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW), lane);
      }
      cp_async_commit();
      mma_block<EL::NI, WS::NTILE>(acc, W.Fs[buf], EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
      mbar_arrive(&W.empty[buf]);         // Fs[buf] may be refilled (block i + 2)
#pragma unroll
      for (int mt = 0; mt < WS::NTILE; ++mt) {
        const int col = mt * 8 + (lane >> 2);
        const int c = col / KW, e = col - c * KW;
        if (col < WS::NCOL && e < nel) {
          const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
          for (int ni = 0; ni < EL::NI; ++ni) {
            const int i2 = ni * 8 + 2 * (lane & 3);
            store_pair<NP>(ep, rowbase + i2, i2, rj[mt] * acc[mt][ni][0], rj[mt] * acc[mt][ni][1]);
          }
        }
      }
      if (wb_next >= nwblocks) break;
      wb = wb_next;
    }
    cp_async_wait<0>();
  }
}

// ------------------------------------------------------------------------------------------
// pass 2, cross-block software pipeline (k_nsdiv5).
//
// Same data flow as k_nsdiv3, but the neighbour gathers of block i+1 are ISSUED (into registers)
// just before the DMMA contraction of block i and CONSUMED after its store, so their L2/HBM latency
// hides behind ~3 us of tensor-core work instead of stalling the warp twice per block.  The small
// per-block inputs (q, lam, connectivity) are therefore needed one block earlier: triple-buffered,
// staged two blocks ahead.  Register budget: NR*(2C+1) gather values live across the MMA phase
// (44 doubles for tets p3) next to the 24 accumulator registers -- 8 warps x 255 registers.
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct alignas(16) Div5Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  double Ts[NCOL * EL::LDV];
  double Fs[NCOL * EL::LDF];
  Div3Small<DIM, P, KW> sm[3];
};

template <int DIM, int P, int KW, int NWARPS>
struct Div5Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Div5Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

template <int DIM, int P, int KW, int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsdiv5(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Div5Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div5Smem<DIM, P, KW, NWARPS>*>(smem_raw);
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
  __syncthreads();
  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  __syncthreads();

  auto nel_of = [&](long long wbx) -> int {
    if (wbx >= nwblocks) return 0;
    const long long e = ebeg + wbx * KW;
    return (int)((eend - e) < (long long)KW ? (eend - e) : (long long)KW);
  };
  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;           // block i
  if (wb >= nwblocks) return;
  // prologue: S(0), T(0), S(1); gathers of block 0 in flight
  div_stage_small<DIM, P, KW>(W.sm[0], d, q, T, ebeg + wb * KW, nel_of(wb), lane);
  cp_async_commit();
  div_stage_rows<DIM, P, KW>(W.Ts, d, T, ebeg + wb * KW, nel_of(wb), lane);
  cp_async_commit();
  unsigned long long ticket = draw_ticket(counter, lane);
  long long wb1 = ticket_block(ticket, wstride);                  // block i+1
  ticket = draw_ticket(counter, lane);
  if (nel_of(wb1) > 0) div_stage_small<DIM, P, KW>(W.sm[1], d, q, T, ebeg + wb1 * KW, nel_of(wb1), lane);
  cp_async_commit();
  cp_async_wait<2>();                                             // S(0)
  __syncwarp();
  FaceRegs<DIM, P, KW> R;
  face_issue<DIM, P, KW>(R, S.flc, S.fn, S.perm, W.sm[0], d, q, T, ghost, Tghost, nel_of(wb), lane);

  for (int i = 0;; ++i) {
    const int b0 = i % 3, b1 = (i + 1) % 3, b2 = (i + 2) % 3;
    const long long e0 = ebeg + wb * KW;
    const int nel = nel_of(wb);
    const long long wb2 = ticket_block(ticket, wstride);          // block i+2: its small inputs start now
    ticket = draw_ticket(counter, lane);
    if (nel_of(wb2) > 0) div_stage_small<DIM, P, KW>(W.sm[b2], d, q, T, ebeg + wb2 * KW, nel_of(wb2), lane);
    cp_async_commit();                                            // S(i+2)
    // face phase of block i from the gathers issued one block ago
    face_finish<DIM, P, KW>(R, S.flc, S.fn, S.perm, W.sm[b0], W.Fs, d, T, Tghost, ph, e0, nel, lane);
    cp_async_wait<1>();                                           // S(i+1) and T(i) have landed
    __syncwarp();
    // gathers of block i+1 fly during the contraction of block i
    face_issue<DIM, P, KW>(R, S.flc, S.fn, S.perm, W.sm[b1], d, q, T, ghost, Tghost, nel_of(wb1), lane);

    double acc[WS::NTILE][EL::NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
    mma_block<EL::NI, WS::NTILE>(acc, W.Ts, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
    mma_block<EL::NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
    double rj[WS::NTILE];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) rj[mt] = W.sm[b0].rj[(mt * 8 + (lane >> 2)) % KW];
    __syncwarp();                                                 // operand rows consumed
    if (nel_of(wb1) > 0) div_stage_rows<DIM, P, KW>(W.Ts, d, T, ebeg + wb1 * KW, nel_of(wb1), lane);
    cp_async_commit();                                            // T(i+1)
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) {
          const int i2 = ni * 8 + 2 * (lane & 3);
          store_pair<NP>(ep, rowbase + i2, i2, rj[mt] * acc[mt][ni][0], rj[mt] * acc[mt][ni][1]);
        }
      }
    }
    if (wb1 >= nwblocks) break;
    wb = wb1;
    wb1 = wb2;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------
// pass 2 with TMA bulk copies (k_nsdiv6, even Np only).
//
// Per-phase timing of k_nsdiv3 (scripts/phase_timing_flux.py): a warp spends a third of its time
// issuing and waiting for its own staging -- 23 cp.async per LANE and block, each with its address
// arithmetic and its L1/LSU wavefronts.  A block's rows of one plane are KW*Np consecutive doubles
// in HBM; with the operand rows laid out [field][ref. direction][element][node] they are consecutive
// in shared memory too, so one `cp.async.bulk` (TMA, UBLKCP in SASS) per plane moves them: 21 copies
// per block, ONE instruction per lane, no LSU wavefronts, completion on an mbarrier.
// The DMMA A-fragment addressing follows the new layout (column base c*CS + e*Np, reference
// direction r at +r*KW*Np); CS is padded so that the 8 rows of a fragment fall on distinct banks.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes),
                 "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int DIM, int P, int KW>
struct Div6T {
  using EL = ElemT<DIM, P>;
  static constexpr int PL = KW * EL::NP;                     // doubles of one plane of a block
  static constexpr int CS0 = DIM * PL + 4;                   // room for the K padding of the last row
  static constexpr int CS = CS0 + ((12 - CS0 % 16) + 16) % 16;   // field stride = 12 (mod 16): conflict-free fragments for Np = 4 (mod 16)
};

template <int DIM, int P, int KW>
struct alignas(16) Div6Small {
  using EL = ElemT<DIM, P>;
  double Qs[EL::C * KW * EL::NP];
  double Lam[KW * EL::NP];
  double sj[KW][EL::NF];
  long long conn[KW][EL::NF];
};

template <int DIM, int P, int KW>
struct alignas(16) Div6Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  double Ts[EL::C * Div6T<DIM, P, KW>::CS + 16];
  double Fs[NCOL * EL::LDF];
  Div6Small<DIM, P, KW> sm[2];
  unsigned long long barS[2], barT;
};

template <int DIM, int P, int KW, int NWARPS>
struct Div6Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Div6Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

// one lane = one bulk copy; lane 0 posts the byte count first
template <int DIM, int P, int KW>
__device__ __forceinline__ void div6_stage_small(Div6Small<DIM, P, KW>& M, unsigned long long* bar, const DiscDev& d,
                                                 const double* q, const double* T, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const unsigned rowb = (unsigned)(nel * NP * 8), geob = (unsigned)(nel * NF * 8);
  if (lane == 0) mbar_expect_tx(bar, (C + 1) * rowb + 2 * geob);
  __syncwarp();
  const long long pstride = d.E * NP;
  if (lane < C) bulk_g2s(M.Qs + lane * (KW * NP), q + lane * pstride + e0 * NP, rowb, bar);
  else if (lane == C) bulk_g2s(M.Lam, T + (long long)(DIM * C) * pstride + e0 * NP, rowb, bar);
  else if (lane == C + 1) bulk_g2s(&M.sj[0][0], d.sj + e0 * NF, geob, bar);
  else if (lane == C + 2) bulk_g2s(&M.conn[0][0], d.conn + e0 * NF, geob, bar);
}

template <int DIM, int P, int KW>
__device__ __forceinline__ void div6_stage_rows(double* Ts, unsigned long long* bar, const DiscDev& d, const double* T,
                                                long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  using TT = Div6T<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP;
  const unsigned rowb = (unsigned)(nel * NP * 8);
  if (lane == 0) mbar_expect_tx(bar, DIM * C * rowb);
  __syncwarp();
  const long long pstride = d.E * NP;
  for (int pl = lane; pl < DIM * C; pl += 32) {
    const int r = pl / C, c = pl - r * C;
    bulk_g2s(Ts + c * TT::CS + r * TT::PL, T + (long long)pl * pstride + e0 * NP, rowb, bar);
  }
}

template <int DIM, int P, int KW, int NWARPS>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsdiv6(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Div6Warp<DIM, P, KW>;
  using TT = Div6T<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NI = EL::NI;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int NB = DGB_DIV_NB;
  static_assert(NP % 2 == 0, "bulk copies need rows that are multiples of 16 bytes");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div6Smem<DIM, P, KW, NWARPS>*>(smem_raw);
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
  __syncthreads();
  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  if (lane == 0) { mbar_init(&W.barS[0], 1); mbar_init(&W.barS[1], 1); mbar_init(&W.barT, 1); }
  fence_proxy_async();                 // zero fill + barrier init visible to the async proxy
  __syncthreads();

  auto nel_of = [&](long long wbx) -> int {
    if (wbx >= nwblocks) return 0;
    const long long e = ebeg + wbx * KW;
    return (int)((eend - e) < (long long)KW ? (eend - e) : (long long)KW);
  };
  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  if (wb >= nwblocks) return;
  div6_stage_small<DIM, P, KW>(W.sm[0], &W.barS[0], d, q, T, ebeg + wb * KW, nel_of(wb), lane);
  div6_stage_rows<DIM, P, KW>(W.Ts, &W.barT, d, T, ebeg + wb * KW, nel_of(wb), lane);
  unsigned long long ticket = draw_ticket(counter, lane);

  // per-lane fragment addressing of the T operand: column base of this lane's row in each tile
  int colbase[WS::NTILE];
#pragma unroll
  for (int mt = 0; mt < WS::NTILE; ++mt) {
    const int col = mt * 8 + (lane >> 2);
    const int c = col / KW, e = col - c * KW;
    colbase[mt] = (col < WS::NCOL ? c * TT::CS + e * NP : 0) + (lane & 3);
  }
  const double* wv = S.Wv + (lane >> 2) * EL::LDV + (lane & 3);

  for (int i = 0;; ++i) {
    const int buf = i & 1;
    const long long e0 = ebeg + wb * KW;
    const int nel = nel_of(wb);
    const long long wb_next = ticket_block(ticket, wstride);
    const int nel1 = nel_of(wb_next);
    // sm[buf ^ 1] was last read by the face phase of block i-1 (generic proxy): order before the async write
    fence_proxy_async();
    if (nel1 > 0) div6_stage_small<DIM, P, KW>(W.sm[buf ^ 1], &W.barS[buf ^ 1], d, q, T, ebeg + wb_next * KW, nel1, lane);
    ticket = draw_ticket(counter, lane);
    mbar_wait(&W.barS[buf], (i >> 1) & 1);
    const Div6Small<DIM, P, KW>& M = W.sm[buf];
    double rj[WS::NTILE];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int e = (mt * 8 + (lane >> 2)) % KW;
      rj[mt] = e < nel ? d.rj[e0 + e] : 0.0;
    }

    div_face_phase<DIM, P, KW, NB, (DGB_DIV_LAZY_EX != 0)>(S.flc, S.fn, S.perm,
        *reinterpret_cast<const Div3Small<DIM, P, KW>*>(&M), W.Fs, d, q, T, ghost, Tghost, ph, e0, nel, lane);
    __syncwarp();
    mbar_wait(&W.barT, i & 1);

    double acc[WS::NTILE][NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
#pragma unroll
    for (int r = 0; r < DIM; ++r) {
#pragma unroll
      for (int kk = 0; kk < EL::NPK / 4; ++kk) {
        double a[WS::NTILE], b[NI];
#pragma unroll
        for (int mt = 0; mt < WS::NTILE; ++mt) a[mt] = W.Ts[colbase[mt] + r * TT::PL + kk * 4];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) b[ni] = wv[ni * 8 * EL::LDV + r * EL::NPK + kk * 4];
#pragma unroll
        for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma884(acc[mt][ni][0], acc[mt][ni][1], a[mt], b[ni]);
      }
    }
    mma_block<NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
    __syncwarp();                        // operand rows consumed (generic proxy) ...
    fence_proxy_async();                 // ... before the async proxy overwrites them
    if (nel1 > 0) div6_stage_rows<DIM, P, KW>(W.Ts, &W.barT, d, T, ebeg + wb_next * KW, nel1, lane);

#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int i2 = ni * 8 + 2 * (lane & 3);
          store_pair<NP>(ep, rowbase + i2, i2, rj[mt] * acc[mt][ni][0], rj[mt] * acc[mt][ni][1]);
        }
      }
    }
    if (nel1 == 0) break;
    wb = wb_next;
  }
}

}  // namespace dgb
