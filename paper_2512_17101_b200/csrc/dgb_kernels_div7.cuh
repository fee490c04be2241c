// Pass 2 of the Navier-Stokes flux arrangement, role-split version (k_nsdiv7).
//
// ncu on k_nsdiv3 (round 1, profiles/r01_ncu_full_flux_n94.md): DMMA pipe 43.6 %, two resident warps per
// scheduler, every warp alternating between a latency-bound gather phase and the contraction; and the
// L1/LSU data pipe 58 % busy -- a third of its shared-memory wavefronts are the W fragment loads of
// the contraction (5 LDS.64 per 6 DMMA).  Both are attacked here:
//
//   * CONSUMER warps (warpgroup 0: one warp per SM sub-partition) do nothing but the contraction.
//     They hold the B fragments of the constant matrix [Wv2 | Wl] in REGISTERS for the whole kernel
//     (p3 tets: 3 node tiles x 25 k-steps = 75 doubles = 150 registers; `setmaxnreg` raises the
//     warpgroup to 232 registers), so a k-step is MT operand loads for MT*NI DMMAs
//     (0.33 LDS per DMMA instead of 0.83) and a single warp keeps its sub-partition's DMMA pipe fed.
//   * PRODUCER warps (warpgroups 1..NPG, `setmaxnreg`-shrunk) own one operand stage each: they stage the
//     block's small inputs, stream its T rows with cp.async straight into the operand layout, run the
//     face phase (gathers + Rusanov, identical code to k_nsdiv3), hand the stage to their consumer
//     through an mbarrier, and when the consumer hands it back with the contraction result in place
//     they apply 1/J and the (RK-fused) epilogue with fully coalesced 16-byte stores.
//
// A producer is served by the consumer of its own sub-partition (warp index mod 4); a consumer polls the
// `full` barriers of its NPG producers round-robin and takes whichever stage is ready.  Results are
// bitwise identical to k_nsdiv3 (same k order in every accumulator).
//
// Node tiles whose fragments do not fit in registers (orders with Np > 24) are taken from shared memory
// as before: NIR = number of register-resident node tiles.
#pragma once
#include "dgb_kernels_flux.cuh"

#ifndef DGB_DIV7_LAZY_EX
#define DGB_DIV7_LAZY_EX 0
#endif
#ifdef DGB_PHASE_TIMING
// consumer warp 0 and producer warp 4 of every CTA accumulate the cycles they spend per phase
#define DGB_T7(k) do { if (lane == 0 && (warp == 0 || warp == 4)) { long long t_ = clock64(); d.timing[blockIdx.x * 8 + (k)] += t_ - t7last; t7last = t_; } } while (0)
#define DGB_T7_INIT long long t7last = clock64();
#else
#define DGB_T7(k) do { } while (0)
#define DGB_T7_INIT
#endif

namespace dgb {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, int parity) {
  unsigned ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int parity) {
  while (!mbar_test(bar, parity)) { }
}

template <int DIM, int P, int KW>
struct alignas(16) Div7Stage {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  // operand rows of the real columns only: the fragment loads of a padding column (at most one) read
  // the rows that follow it in this struct; its accumulators are never stored and DMMA rows do not mix
  double Ts[NCOL * EL::LDV];          // T rows; the consumer leaves the contraction result in [col][0..NPR)
  double Fs[NCOL * EL::LDF];
  unsigned long long full, done;      // mbarriers: producer -> consumer, consumer -> producer
  long long more;                     // 0 = the producer has no further blocks (published with `full`)
  long long pad_;
};

// A producer owns two operand stages (it runs the face phase of block b+1 while its consumer contracts
// block b) and one private buffer of small inputs.
template <int DIM, int P, int KW>
struct alignas(16) Div7Prod {
  Div7Stage<DIM, P, KW> st[2];
  Div3Small<DIM, P, KW> sm;
};

template <int DIM, int P, int KW, int NPROD, int NIR>
struct Div7Smem {
  using EL = ElemT<DIM, P>;
  static constexpr bool WSM = NIR < EL::NI;             // some node tiles come from shared memory
  double Wv[WSM ? EL::NPR * EL::LDV : 2];
  double Wl[WSM ? EL::NPR * EL::LDF : 2];
  Div7Prod<DIM, P, KW> pr[NPROD];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

// consumer / producer register budgets (setmaxnreg; multiples of 8) for a CTA of 4 + 4*NPG warps whose
// launch-time allocation is REG0 per thread
template <int NPG> struct Div7Regs;
template <> struct Div7Regs<1> { static constexpr int REG0 = 255, CONS = 0, PROD = 0; };       // 256 threads: no split needed
template <> struct Div7Regs<2> { static constexpr int REG0 = 168, CONS = 232, PROD = 136; };   // 384 threads
template <> struct Div7Regs<3> { static constexpr int REG0 = 128, CONS = 232, PROD = 88; };    // 512 threads

template <int DIM, int P, int KW, int NPROD, int NIR, int NB, bool GH>
__global__ void __launch_bounds__(128 + 128 * ((NPROD + 3) / 4), 1)
k_nsdiv7(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using ST = Div7Stage<DIM, P, KW>;
  constexpr int NPG = (NPROD + 3) / 4;                 // producer warpgroups (warps beyond NPROD retire at once)
  using SM = Div7Smem<DIM, P, KW, NPROD, NIR>;
  using RG = Div7Regs<NPG>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NI = EL::NI;
  constexpr int NT = 128 + 128 * NPG;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int KSV = EL::KV / 4, KSF = EL::KF / 4, MT = ST::NTILE;
  static_assert(NIR >= 0 && NIR <= NI, "NIR out of range");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E;

  if (SM::WSM) {
    for (int n = tid; n < EL::NPR * EL::LDV; n += NT) S.Wv[n] = d.Wv2[n];
    for (int n = tid; n < EL::NPR * EL::LDF; n += NT) S.Wl[n] = d.Wl[n];
  }
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  for (int n = tid; n < NPROD * (int)(sizeof(Div7Prod<DIM, P, KW>) / 8); n += NT) reinterpret_cast<double*>(&S.pr[0])[n] = 0.0;
  __syncthreads();
  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  if (tid < 2 * NPROD) { mbar_init(&S.pr[tid >> 1].st[tid & 1].full, 1); mbar_init(&S.pr[tid >> 1].st[tid & 1].done, 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  if (warp < 4) {
    // ======================================= consumer =======================================
    if (RG::CONS > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(RG::CONS > 0 ? RG::CONS : 24));
    const int r = lane >> 2, kq = lane & 3;
    // B fragments of [Wv2 | Wl] for the register-resident node tiles
    double wv[NIR > 0 ? NIR : 1][KSV], wl[NIR > 0 ? NIR : 1][KSF];
#pragma unroll
    for (int ni = 0; ni < NIR; ++ni) {
#pragma unroll
      for (int ks = 0; ks < KSV; ++ks) wv[ni][ks] = d.Wv2[(ni * 8 + r) * EL::LDV + ks * 4 + kq];
#pragma unroll
      for (int ks = 0; ks < KSF; ++ks) wl[ni][ks] = d.Wl[(ni * 8 + r) * EL::LDF + ks * 4 + kq];
    }
    const double* wvs = S.Wv + r * EL::LDV + kq;     // shared-memory tiles NIR..NI-1
    const double* wls = S.Wl + r * EL::LDF + kq;
    // per-producer bit masks: finished / stage the producer fills next / expected parity of `full` per stage
    unsigned fin = 0, cur = 0, par = 0;
    const int ng = (NPROD - warp + 3) / 4;           // this consumer's producers: stages warp, warp + 4, ...
    int alive = ng, g = 0;
    DGB_T7_INIT
    while (alive > 0) {
      ST* st;
      for (;;) {
        const int sidx = (cur >> g) & 1;
        st = &S.pr[g * 4 + warp].st[sidx];
        if (!((fin >> g) & 1) && mbar_test(&st->full, (par >> (2 * g + sidx)) & 1)) break;
        g = g + 1 >= ng ? 0 : g + 1;
      }
      if (st->more == 0) { fin |= 1u << g; --alive; continue; }
      DGB_T7(0);
      double acc[MT][NI][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
      {
        const double* xp = st->Ts + r * EL::LDV + kq;
#pragma unroll
        for (int ks = 0; ks < KSV; ++ks) {
          double a[MT], b[NI];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) a[mt] = xp[mt * 8 * EL::LDV + ks * 4];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) b[ni] = ni < NIR ? wv[ni < NIR ? ni : 0][ks] : wvs[ni * 8 * EL::LDV + ks * 4];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma884(acc[mt][ni][0], acc[mt][ni][1], a[mt], b[ni]);
        }
      }
      {
        const double* xp = st->Fs + r * EL::LDF + kq;
#pragma unroll
        for (int ks = 0; ks < KSF; ++ks) {
          double a[MT], b[NI];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) a[mt] = xp[mt * 8 * EL::LDF + ks * 4];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) b[ni] = ni < NIR ? wl[ni < NIR ? ni : 0][ks] : wls[ni * 8 * EL::LDF + ks * 4];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma884(acc[mt][ni][0], acc[mt][ni][1], a[mt], b[ni]);
        }
      }
      __syncwarp();                      // every lane has read its operand rows: results may land on them
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int col = mt * 8 + r;
        if (col < ST::NCOL) {
          double* row = st->Ts + col * EL::LDV + 2 * kq;
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
            *reinterpret_cast<double2*>(row + ni * 8) = make_double2(acc[mt][ni][0], acc[mt][ni][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&st->done);
      DGB_T7(1);
      par ^= 1u << (2 * g + ((cur >> g) & 1));
      cur ^= 1u << g;
      g = g + 1 >= ng ? 0 : g + 1;
    }
  } else {
    // ======================================= producer =======================================
    if (RG::PROD > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(RG::PROD > 0 ? RG::PROD : 24));
    const int p = warp - 4;                          // producer index; its consumer is warp p & 3
    if (p >= NPROD) return;
    Div7Prod<DIM, P, KW>& W = S.pr[p];
    const long long wstride = (long long)gridDim.x * NPROD;
    long long wb = (long long)blockIdx.x * NPROD + p;
    auto nel_of = [&](long long wbx) -> int {
      if (wbx >= nwblocks) return 0;
      const long long e = ebeg + wbx * KW;
      return (int)((eend - e) < (long long)KW ? (eend - e) : (long long)KW);
    };
    DGB_T7_INIT
    // 1/J and the (RK-fused) store of a finished block, straight from its result rows: KW*Np consecutive
    // doubles per field in global memory, so every store instruction is fully coalesced
    auto retire = [&](ST& st, int parity, long long e0, int nelx, const double (&rj)[KW]) {
      mbar_wait(&st.done, parity);
      DGB_T7(5);
      constexpr int CH = (NP % 2 == 0) ? 2 : 1, NPC = NP / CH;
#pragma unroll
      for (int t0 = 0; t0 < KW * NPC; t0 += 32) {
        const int t = t0 + lane;
        const int e = t / NPC, j = CH * (t - e * NPC);
        if (t < KW * NPC && e < nelx) {
          double s = rj[0];
#pragma unroll
          for (int k = 1; k < KW; ++k) s = e == k ? rj[k] : s;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const long long idx = ((long long)c * E + e0 + e) * NP + j;
            if (CH == 2) {
              const double2 v = *reinterpret_cast<const double2*>(st.Ts + (c * KW + e) * EL::LDV + j);
              store_pair<NP>(ep, idx, j, s * v.x, s * v.y);
            } else {
              const double v = s * st.Ts[(c * KW + e) * EL::LDV + j];
              ep.out1[idx] = ep.x1 ? ep.a1 * ep.x1[idx] + ep.b1 * v : ep.b1 * v;
              if (ep.out2) ep.out2[idx] = ep.a2 * ep.x2[idx] + ep.b2 * v;
            }
          }
        }
      }
      __syncwarp();                                  // result rows consumed: this stage may be refilled
      DGB_T7(6);
    };
    int nel = nel_of(wb);
    if (nel > 0) div_stage_small<DIM, P, KW>(W.sm, d, q, T, ebeg + wb * KW, nel, lane);
    cp_async_commit();                               // S(b)
    TicketStream tks;
    tickets_init(tks, wb, counter, lane);
    int it = 0;
    long long e0_prev = 0;
    int nel_prev = 0;
    double rj_prev[KW];
#pragma unroll
    for (int e = 0; e < KW; ++e) rj_prev[e] = 0.0;
    // cp.async groups retire in order: S(b), T(b), S(b+1), T(b+1), ...
    while (nel > 0) {
      ST& st = W.st[it & 1];                         // free: the block that used it two iterations ago has been retired
      const long long e0 = ebeg + wb * KW;
      div_stage_rows<DIM, P, KW>(st.Ts, d, T, e0, nel, lane);
      cp_async_commit();                             // T(b)
      const long long wb_next = tickets_next(tks, wstride, counter, lane);
      const int nel1 = nel_of(wb_next);
      cp_async_wait<1>();                            // S(b) has landed; T(b) may still be in flight
      __syncwarp();
      DGB_T7(2);
      div_face_phase<DIM, P, KW, NB, (DGB_DIV7_LAZY_EX != 0), 0, GH, (DGB_DIV_INBLOCK != 0), 0>(S.flc, S.fn, S.perm, W.sm, st.Fs, d, q, T, ghost, Tghost, ph, e0, nel, lane, st.Ts);
      DGB_T7(3);
      double rj[KW];
#pragma unroll
      for (int e = 0; e < KW; ++e) rj[e] = W.sm.rj[e];
      __syncwarp();                                  // the small inputs are consumed: the next block's may land
      if (nel1 > 0) div_stage_small<DIM, P, KW>(W.sm, d, q, T, ebeg + wb_next * KW, nel1, lane);
      cp_async_commit();                             // S(b+1)
      cp_async_wait<1>();                            // T(b) has landed
      if (lane == 0) st.more = 1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&st.full);
      DGB_T7(4);
      // the previous block went to the consumer a whole face phase ago: retire it now
      if (it > 0) retire(W.st[(it - 1) & 1], ((it - 1) >> 1) & 1, e0_prev, nel_prev, rj_prev);
      e0_prev = e0; nel_prev = nel;
#pragma unroll
      for (int e = 0; e < KW; ++e) rj_prev[e] = rj[e];
      wb = wb_next;
      nel = nel1;
      ++it;
    }
    cp_async_wait<0>();
    if (it > 0) retire(W.st[(it - 1) & 1], ((it - 1) >> 1) & 1, e0_prev, nel_prev, rj_prev);
    {
      ST& st = W.st[it & 1];                         // end marker on the stage the consumer looks at next
      if (lane == 0) st.more = 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(&st.full);
    }
  }
}

}  // namespace dgb
