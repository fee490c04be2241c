// Navier-Stokes right-hand side in the FLUX arrangement (operators.py: dg_ns_flux + dg_ns_div).
//
// The gradient arrangement (dgb_kernels_warp.cuh) evaluates the total flux three times per node and
// RHS: at the node (volume term), at the node again as the own side of a face, and once more by the
// neighbour for its plus side; ncu showed pass 2 spending as much of the FP64 datapath on that
// pointwise work (22.9 %) as on the DMMA contraction (28.9 %).  Here every node's flux is evaluated
// ONCE, by its owner, at the end of pass 1 while the BR1 gradient is still on chip:
//
//   k_nsflux3  (pass 1)  rows -> face averages -> DMMA (Sw_r q, lift_f q*) -> grad q into shared
//                        memory -> pointwise F = F_inv - F_visc -> T[r][c] = sum_x (J dr/dx)[r][x] F[x][c],
//                        their sum over r (plane group dim) and lam = |u| + c  ->  HBM  ((dim+1)*C + 1 planes)
//   k_nsdiv3/8 (pass 2)  T rows arrive by cp.async / TMA straight into the DMMA operand layout (no
//                        pointwise volume work at all); per face node the kernel gathers the
//                        neighbour's q, lam and ONE plane group: sJ F+.n+ = (face 0 ? T+[dim] : -T+[nf-1]),
//                        own side folded into the volume matrix -> Rusanov -> DMMA -> 1/J -> store.
//
// HBM bytes per DOF (3D): pass 1 reads 40, writes 168; pass 2 streams 168, gathers q/lam/one group, writes 40.
#pragma once
#include "dgb_kernels.cuh"
#include "dgb_kernels_async.cuh"
#include "dgb_kernels_warp.cuh"

#ifndef DGB_DIV_NB
#define DGB_DIV_NB 2
#endif
#ifndef DGB_TICKET_BLOCKS
#define DGB_TICKET_BLOCKS 1
#endif
#ifndef DGB_TICKET_DEPTH
#define DGB_TICKET_DEPTH 2
#endif
#ifndef DGB_L2_PREFETCH_BLOCKS
#define DGB_L2_PREFETCH_BLOCKS 0
#endif
// pass 1 with ONE buffer for a block's state rows where shared memory limits the number of warps (order 4: 6 -> 8
// warps; mixtures: 7 -> 8): the next block's rows are staged right after the tensor-core phase and the pointwise phase
// reads the state from global memory (the rows were staged a moment ago: L2 hits) instead of the buffer.
// -1: automatic (Np > 20 or mixtures), 0 / 1: off / on
// pass 1 tensor-core phase: one column tile at a time (0), all column tiles of a block in one sweep (1), or all tiles
// with U_0 first and the Z_r chains started from -U_0 (2: 24 accumulator registers fewer per tile).  Sharing the W
// fragments across tiles takes the operand LDS from 1.33 to 0.83 per DMMA.  Measured (profiles/r02_pass2_tma.md, section 12):
// -1 % / -3 % of pass 1 where the launch has 8 warps and 255 registers (order 4, mixtures); at 3D p3 (12 warps, 168
// registers, 20 B of spills) equal over 10 timed steps and +0.8 % GDOF/s over 20 / 50 / 100 steps (fewer shared-memory
// reads: the step runs at the board power cap).  -1: automatic (2 up to 10 accumulator tiles per set -- beyond that it
// spills --, else 0)
#ifndef DGB_FLUX_MT
#define DGB_FLUX_MT -1
#endif
// pass 1: unroll factor of the pointwise node loop (2 lane rounds at order 3, 4 at order 4; ~10 KB of SASS per copy).
// Not unrolled, the kernel is 33 instead of 40 KB at order 3 (57 / 76 at order 4; the L1.5 instruction cache holds 32 KB):
// pass 1 -0.5 % at order 3, -1.9 % at order 4 (profiles/r02_pass2_tma.md section 13)
#ifndef DGB_FLUX_PW_UNROLL
#define DGB_FLUX_PW_UNROLL 1
#endif
#ifndef DGB_EULER_PW_UNROLL
#define DGB_EULER_PW_UNROLL 1
#endif
// pass 1: the flux planes are written once and not read again by this kernel: streaming stores (st.global.cs) keep
// L2 for the neighbour gathers
#ifndef DGB_FLUX_T_STCS
#define DGB_FLUX_T_STCS 0
#endif
#ifndef DGB_FLUX_SINGLEQ
#define DGB_FLUX_SINGLEQ -1
#endif
// cp.async pass 2 (k_nsdiv3): one buffer for a block's small inputs (q, lam, face Jacobians, connectivity) instead of
// two: the next block's are staged as soon as the face phase has read these and land during the contraction + store
// (15.6 instead of 18.7 KB of shared memory per warp at 3D p3; measured no faster: off)
#ifndef DGB_DIV_SINGLE_SMALL
#define DGB_DIV_SINGLE_SMALL 0
#endif

#ifdef DGB_PHASE_TIMING
// warp 0 of every CTA accumulates the cycles it spends in each phase (scripts/phase_timing_flux.py)
#define DGB_WTICK(k) do { if (warp == 0 && lane == 0) { long long t_ = clock64(); d.timing[blockIdx.x * 8 + (k)] += t_ - wtlast; wtlast = t_; } } while (0)
#define DGB_WTICK_INIT long long wtlast = clock64();
#else
#define DGB_WTICK(k) do { } while (0)
#define DGB_WTICK_INIT
#endif

// how the neighbour gathers of pass 2 go through the cache hierarchy: 0 = default (allocate in L1),
// 1 = ld.global.cg (L2 only: no L1 line per in-flight sector), 2 = ld.global.nc
#ifndef DGB_GATHER_LD
#define DGB_GATHER_LD 0
#endif
#if DGB_GATHER_LD == 1
#define DGB_GLD(p) __ldcg(p)
#elif DGB_GATHER_LD == 2
#define DGB_GLD(p) __ldg(p)
#else
#define DGB_GLD(p) (*(p))
#endif

namespace dgb {

// The flux planes T are the ((dim+1)*C + 1, E, Np) array of the operator program as it is (plane-major).  A
// record-major layout (all planes of an element contiguous) was measured in round 1: +3 %, not adopted.
template <int NPL, int NP>
__host__ __device__ __forceinline__ long long t_elem_stride() { return (long long)NP; }
template <int NPL, int NP>
__host__ __device__ __forceinline__ long long t_plane_stride(long long nelem) { return nelem * NP; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

// Split-phase dynamic work distribution: the ticket is drawn (atomicAdd on lane 0) one block ahead of
// its use, so the atomic's round trip to L2 overlaps a whole block of work instead of stalling the warp.
__device__ __forceinline__ unsigned long long draw_ticket(unsigned long long* counter, int lane) {
  // predicated atom inside the asm block: no select on the result, so nothing waits for it until
  // ticket_block() shuffles lane 0's value out (a C++ `if (lane == 0) v = atomicAdd()` merges the
  // result into `v` right away and stalled every warp for the full L2 round trip: 13 % of samples)
  unsigned long long v;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, 0;\n\t@p atom.global.add.u64 %0, [%1], 1;\n\t}"
               : "=l"(v) : "l"(counter), "r"(lane) : "memory");
  return v;
}
__device__ __forceinline__ long long ticket_block(unsigned long long v, long long first_dynamic) {
  return first_dynamic + (long long)__shfl_sync(0xffffffffu, v, 0);
}

// ptxas turns a predicated atomic on a warp-uniform address into a warp-aggregated one: leader election, ATOMG,
// and a SHFL of the result RIGHT AFTER it -- which makes the warp wait for the L2 round trip at the draw and defeats
// the split-phase scheme (ncu: 2.7 % of pass 1's stall samples sit on that SHFL).  An address ptxas cannot prove
// uniform keeps the atomic a plain single-lane ATOMG: the offset below comes from shared memory and is always 0.
#ifndef DGB_TICKET_NOAGG
#define DGB_TICKET_NOAGG 1
#endif
__device__ __forceinline__ unsigned long long* ticket_counter(unsigned long long* counter, const int* table, int lane) {
#if DGB_TICKET_NOAGG
  return counter + (table[lane & 1] >> 24);           // face-node indices are < 256
#else
  return counter;
#endif
}

// Tickets in batches of DGB_TICKET_BLOCKS consecutive blocks: one atomic on the (single, hot) work counter
// per batch instead of per block.  With ~1200 warps drawing a ticket every ~6 us the counter's L2 slice
// serialises ~200 same-address atomics per microsecond and a ticket drawn a whole block earlier was
// still not back when it was needed (19 % of a pass-2 warp's time sat in the shuffle that reads it).
struct TicketStream {
  unsigned long long pending;   // raw result of the oldest outstanding draw (valid on lane 0)
#if DGB_TICKET_DEPTH > 1
  unsigned long long pending2;  // second outstanding draw: every ticket gets two block times to come back
#endif
  long long cur;                // block most recently handed out
  int left;                     // blocks left in the current batch
};
__device__ __forceinline__ unsigned long long draw_tickets(unsigned long long* counter, int lane, int count) {
  unsigned long long v;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, 0;\n\t@p atom.global.add.u64 %0, [%1], %3;\n\t}"
               : "=l"(v) : "l"(counter), "r"(lane), "l"((unsigned long long)count) : "memory");
  return v;
}
__device__ __forceinline__ void tickets_init(TicketStream& ts, long long first_block, unsigned long long* counter, int lane) {
  ts.cur = first_block; ts.left = 0;
  ts.pending = draw_tickets(counter, lane, DGB_TICKET_BLOCKS);
#if DGB_TICKET_DEPTH > 1
  ts.pending2 = draw_tickets(counter, lane, DGB_TICKET_BLOCKS);
#endif
}
__device__ __forceinline__ long long tickets_next(TicketStream& ts, long long first_dynamic, unsigned long long* counter, int lane) {
  if (ts.left > 0) { --ts.left; return ++ts.cur; }
  ts.cur = ticket_block(ts.pending, first_dynamic);
  ts.left = DGB_TICKET_BLOCKS - 1;
#if DGB_TICKET_DEPTH > 1
  ts.pending = ts.pending2;
  ts.pending2 = draw_tickets(counter, lane, DGB_TICKET_BLOCKS);
#else
  ts.pending = draw_tickets(counter, lane, DGB_TICKET_BLOCKS);     // the next batch, a whole batch of blocks early
#endif
  return ts.cur;
}

// Face nodes of a warp's block are visited in rounds of WHOLE faces: round k, lane l handles node
// l % NFP of face k*FPR + l / NFP (FPR = 32 / NFP faces per round; the last 32 - FPR*NFP lanes idle).
// A face's nodes lie in one 8*Np-byte row of the neighbour, so one gather instruction then touches
// each of its sectors once; with plain n = lane + 32*k a quarter of the faces straddled two rounds
// and their sectors were requested twice.  Code: bits 0-1 element, 2-3 face, 4-7 node within the
// face, 8-15 own volume node, 16-23 f*NFP + m; negative = idle lane.
template <int DIM, int P, int KW>
__host__ __device__ constexpr int face_rounds() {
  using EL = ElemT<DIM, P>;
  return (KW * EL::NF + (32 / EL::NFP) - 1) / (32 / EL::NFP);
}

template <int DIM, int P, int KW>
__device__ __forceinline__ int face_lane_code(const int* fn, int n) {
  using EL = ElemT<DIM, P>;
  constexpr int FPR = 32 / EL::NFP;
  const int k = n >> 5, l = n & 31;
  const int g = k * FPR + l / EL::NFP, m = l % EL::NFP;
  if (l >= FPR * EL::NFP || g >= KW * EL::NF) return -1;
  const int e = g / EL::NF, f = g - e * EL::NF;
  const int fm = f * EL::NFP + m;
  return e | (f << 2) | (m << 4) | (fn[fm] << 8) | (fm << 16);
}

// L2 prefetch of the rows a block far ahead in ticket order will stream (TMA bulk prefetch: one
// instruction per plane).  The neighbour gathers of the blocks in flight mostly reach a few hundred
// elements ahead (Morton order: 92 % of forward neighbours within 1000 elements), i.e. rows nobody
// has streamed yet: without the prefetch those gathers are first-touch DRAM misses with their full
// latency exposed; with it the first touch happens here, asynchronously, DGB_L2_PREFETCH_BLOCKS
// blocks early, and both the gathers and the later cp.async staging hit L2.
__device__ __forceinline__ void l2_prefetch_bulk(const void* gmem, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}

__device__ __forceinline__ void l2_prefetch_line(const void* gmem) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(gmem) : "memory");
}

template <int NP, int KW>
__device__ __forceinline__ void prefetch_block_rows(const double* __restrict__ a, int nplanes_a, long long stride_a,
                                                    const double* __restrict__ b, int nplanes_b, long long stride_b,
                                                    long long e0, int nel, int lane) {
  if (NP % 2 != 0 || nel <= 0) return;              // bulk prefetch: 16-byte multiples only
  const unsigned bytes = (unsigned)(nel * NP * 8);
  for (int pl = lane; pl < nplanes_a + nplanes_b; pl += 32) {
    const double* p = pl < nplanes_a ? a + pl * stride_a + e0 * NP : b + (pl - nplanes_a) * stride_b + e0 * NP;
    l2_prefetch_bulk(p, bytes);
  }
}

template <int DIM, int P>
struct FluxT {
  using EL = ElemT<DIM, P>;
  static constexpr int NG = DIM + 1;                             // plane groups: T[0..dim-1] and their sum
  static constexpr int LAMPL = NG * EL::C;                       // plane of the wave speed
  static constexpr int NPL = NG * EL::C + 1;                     // planes of T
  // q* rows of the gradient pass; a tile's 8 rows are reused for its 8 columns x DIM directions of grad q
  static constexpr int LDSX = ldpad((EL::NF * EL::NFPK > DIM * EL::NP) ? EL::NF * EL::NFPK : DIM * EL::NP);
};

// ------------------------------------------------------------------------------------------
// pass 1: BR1 gradient -> total flux -> contravariant planes
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void DGB_T_STORE(double* p, double v) {
#if DGB_FLUX_T_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}

template <int DIM, int P, int KW>
struct FluxGeo {
  using EL = ElemT<DIM, P>;
  double drdx[DIM * DIM][KW];
  double nrm[DIM][KW][EL::NF];
  double fsc[KW][EL::NF];
  long long conn[KW][EL::NF];
  double jac[KW];
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}

// a block's slice of the 32-bit gather map -> shared memory
template <int DIM, int NFT, int NFP>
__device__ __forceinline__ void stage_gather_map(unsigned* dst, const unsigned* __restrict__ gidx, long long e0, int nel, int lane) {
  if (gidx == nullptr) return;
  if (DIM == 3) {                    // NFT = 4 NFP words per element: 16-byte chunks, always aligned
    for (int t = lane; t < nel * NFP; t += 32) cp_async16(dst + 4 * t, gidx + e0 * NFT + 4 * t);
  } else {
    for (int t = lane; t < nel * NFT; t += 32) cp_async4(dst + t, gidx + e0 * NFT + t);
  }
}

template <int NP>
__host__ __device__ constexpr int grad_row_swizzle(int k) {
  return (NP % 8 == 4) ? ((k & 4) | ((k & 1) << 1) | ((k >> 1) & 1)) : k;      // NP*8 bytes = 32 (mod 64): p3 tets (Np = 20)
}

template <int DIM, int P, int KW>
struct alignas(16) Flux3Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::CG * KW;     // columns of the BR1 gradient: (field, element)
  static constexpr int NTILE = (NCOL + 7) / 8;
  static constexpr int NCOLP = NTILE * 8;
  static constexpr bool SINGLEQ = DGB_FLUX_SINGLEQ < 0 ? (EL::NP > 20 || DGB_NSPEC > 0) : (DGB_FLUX_SINGLEQ != 0);
  static constexpr int NQB = SINGLEQ ? 1 : 2;
  double Qs[NQB][NCOLP * EL::LDQ];
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
  int flc[face_rounds<DIM, P, KW>() * 32];      // face_lane_code of every face node of a block
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void flux_stage_rows(double* Qs, const DiscDev& d, const double* q, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP;
  const long long E = d.E;
  // a block's rows are KW*NP consecutive doubles of every plane; lane t copies chunk t of each plane
  constexpr int CH = (NP % 2 == 0) ? 2 : 1, NPC = NP / CH;
#pragma unroll
  for (int t0 = 0; t0 < KW * NPC; t0 += 32) {
    const int t = t0 + lane;
    const int e = t / NPC, j = CH * (t - e * NPC);
    if (t < KW * NPC && e < nel) {
      double* dst = Qs + e * EL::LDQ + j;
      const double* src = q + (e0 + e) * NP + j;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (CH == 2) cp_async16(dst + c * (KW * EL::LDQ), src + (long long)c * E * NP);
        else cp_async8(dst + c * (KW * EL::LDQ), src + (long long)c * E * NP);
      }
    }
  }
}

template <int DIM, int P, int KW>
__device__ __forceinline__ void flux_stage_geo(FluxGeo<DIM, P, KW>& g, const DiscDev& d, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int NF = EL::NF;
  const long long E = d.E;
  {
    const int e = lane % KW, rx = lane / KW;        // drdx[rx][e]
    if (KW * DIM * DIM <= 32) {
      if (rx < DIM * DIM && e < nel) cp_async8(&g.drdx[rx][e], d.drdx + (long long)rx * E + e0 + e);
    } else {
      for (int n = lane; n < DIM * DIM * KW; n += 32) {
        const int rx2 = n / KW, e2 = n - rx2 * KW;
        if (e2 < nel) cp_async8(&g.drdx[rx2][e2], d.drdx + (long long)rx2 * E + e0 + e2);
      }
    }
  }
  if (lane < nel * NF) {
#pragma unroll
    for (int x = 0; x < DIM; ++x) cp_async8(&g.nrm[x][0][lane], d.normals + ((long long)x * E + e0) * NF + lane);
    cp_async8(&g.fsc[0][lane], d.fscale + e0 * NF + lane);
    cp_async8(&g.conn[0][lane], d.conn + e0 * NF + lane);
  }
  if (lane < nel) cp_async8(&g.jac[lane], d.jac + e0 + lane);
}

template <int DIM, int P, int KW>
__device__ __forceinline__ void flux_stage_async(double* Qs, FluxGeo<DIM, P, KW>& g, const DiscDev& d, const double* q,
                                                 long long e0, int nel, int lane) {
  flux_stage_rows<DIM, P, KW>(Qs, d, q, e0, nel, lane);
  flux_stage_geo<DIM, P, KW>(g, d, e0, nel, lane);
}

template <int DIM, int P, int KW, int NWARPS, bool GH>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsflux3(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
          double* __restrict__ T, Phys ph, long long ebeg, long long eend, long long nwblocks,
          unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Flux3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT, NI = EL::NI;
  constexpr int LDSX = FluxT<DIM, P>::LDSX;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();        // face-node rounds per block
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Flux3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

  for (int n = tid; n < DIM * EL::NPR * EL::LDQ; n += NT) S.Wq[n] = d.Wq[n];
  for (int n = tid; n < NF * EL::NPR * EL::LDL; n += NT) S.Wf[n] = d.Wf[n];
  for (int n = tid; n < NF * NFP; n += NT) S.fn[n] = d.tables[n];
  for (int n = tid; n < EL::NPERM * NFP; n += NT) S.perm[n] = d.tables[NF * NFP + n];
  WS& W = S.w[warp];
  for (int n = lane; n < WS::NQB * WS::NCOLP * EL::LDQ; n += 32) W.Qs[0][n] = 0.0;
  for (int n = lane; n < WS::NCOLP * LDSX; n += 32) W.Ss[n] = 0.0;
  __syncthreads();

  for (int n = tid; n < NR * 32; n += NT) S.flc[n] = face_lane_code<DIM, P, KW>(S.fn, n);
  __syncthreads();

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  int buf = 0;
  if (wb < nwblocks) {
    const long long e0 = ebeg + wb * KW;
    flux_stage_async<DIM, P, KW>(W.Qs[0], W.geo[0], d, q, e0, (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW), lane);
  }
  cp_async_commit();
  TicketStream tks;
  tickets_init(tks, wb, ticket_counter(counter, S.fn, lane), lane);
  DGB_WTICK_INIT
  // Neighbour states of ALL face nodes of a block, issued one phase early (during the pointwise flux
  // phase of the previous block, which is FP64 work and leaves the L1/LSU pipe to the gathers) and
  // consumed at the top of the block's own iteration.
  double qpE[NR][C];
  long long cnkE[NR];
  auto issue_gathers = [&](const FluxGeo<DIM, P, KW>& g, int nelx) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      cnkE[k] = -1;
      const int flk = S.flc[k * 32 + lane];
      const int e = flk & 3, f = (flk >> 2) & 3, m = (flk >> 4) & 15;
      if (flk >= 0 && e < nelx) {
        const long long cn = g.conn[e][f];
        cnkE[k] = cn;
        const long long nb = DGB_CONN_NB(cn);
        const int jp = S.fn[DGB_CONN_NF(cn) * NFP + S.perm[DGB_CONN_PERM(cn) * NFP + m]];
        const bool in_ghost = GH && nb >= E;
        const long long pstride = (in_ghost ? G : E) * NP;
        const double* pbase = (in_ghost ? ghost : q) + (in_ghost ? nb - E : nb) * NP + jp;
#pragma unroll
        for (int c = 0; c < C; ++c) qpE[k][c] = pbase[c * pstride];
      }
    }
  };
  if (wb < nwblocks) {
    cp_async_wait<0>();
    __syncwarp();
    const long long e0 = ebeg + wb * KW;
    issue_gathers(W.geo[0], (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW));
  }

  while (wb < nwblocks) {
    const long long e0 = ebeg + wb * KW;
    const int nel = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
    // the next block (its ticket was drawn one block ago) starts its trip from HBM now
    const long long wb_next = tickets_next(tks, wstride, ticket_counter(counter, S.fn, lane), lane);
    cp_async_wait<0>();
    __syncwarp();
    constexpr bool SQ = WS::SINGLEQ;
    const int qb = SQ ? 0 : buf;
    const double* Qs = W.Qs[qb];
    const FluxGeo<DIM, P, KW>& geo = W.geo[buf];
    if (wb_next < nwblocks) {
      const long long e1 = ebeg + wb_next * KW;
      const int nel1 = (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW);
      if (SQ) flux_stage_geo<DIM, P, KW>(W.geo[buf ^ 1], d, e1, nel1, lane);       // the rows follow after the tensor-core phase
      else flux_stage_async<DIM, P, KW>(W.Qs[buf ^ 1], W.geo[buf ^ 1], d, q, e1, nel1, lane);
    }
    cp_async_commit();
    if (DGB_L2_PREFETCH_BLOCKS > 0) {
      const long long wbp = wb_next + DGB_L2_PREFETCH_BLOCKS;
      if (wbp < nwblocks) {
        const long long ep = ebeg + wbp * KW;
        prefetch_block_rows<NP, KW>(q, C, E * NP, q, 0, 0, ep,
                                    (int)((eend - ep) < (long long)KW ? (eend - ep) : (long long)KW), lane);
      }
    }
    DGB_WTICK(0);

    // ---- face averages q* (central flux, boundary states) -> Ss; metric coefficients ---------
    // the previous block left grad q in the q* rows: the K-padding columns must be zero again
    if (EL::NFPK != NFP) {
      for (int n = lane; n < WS::NCOLP * NF * (EL::NFPK - NFP); n += 32) {
        const int col = n / (NF * (EL::NFPK - NFP)), r = n - col * (NF * (EL::NFPK - NFP));
        const int f = r / (EL::NFPK - NFP), m = NFP + (r - f * (EL::NFPK - NFP));
        W.Ss[col * LDSX + f * EL::NFPK + m] = 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      if (cnkE[k] >= 0) {
        const int flk = S.flc[k * 32 + lane];
        const int e = flk & 3, f = (flk >> 2) & 3, m = (flk >> 4) & 15, jm = (flk >> 8) & 255;
        const int bc = DGB_CONN_BC(cnkE[k]);
        double qm[C];
#pragma unroll
        for (int c = 0; c < C; ++c) qm[c] = Qs[(c * KW + e) * EL::LDQ + jm];
        if (bc != 0) {
          double nrm[DIM];
#pragma unroll
          for (int x = 0; x < DIM; ++x) nrm[x] = geo.nrm[x][e][f];
          pw_exterior_state<DIM>(bc, qm, nrm, ph, qpE[k]);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) W.Ss[(c * KW + e) * LDSX + f * EL::NFPK + m] = 0.5 * (qm[c] + qpE[k][c]);
      }
    }
    __syncwarp();
    DGB_WTICK(1);

    // ---- tensor-core contractions; grad q of a column tile -> its Ss rows ----
    // On a simplex  fscale n_x (face f) = sum_r a[f][r] dr/dx[r][x]  with a[0][r] = 1, a[r+1][r] = -1, so
    //   grad_x q = sum_f fscale n_x lift_f q*_f - sum_r dr/dx[r][x] Sw_r q
    //            = -sum_r dr/dx[r][x] (Z_r - U_0),   Z_r = Sw_r q + lift_{r+1} q*_{r+1},  U_0 = lift_0 q*_0:
    // DIM+1 accumulator sets instead of DIM+NF (Z_r simply continues its k-loop over the face-(r+1)
    // operand rows) and DIM*DIM + DIM FP64 operations per value in the combination instead of
    // DIM*(DIM+NF).
    // MTF column tiles share every W fragment load (DGB_FLUX_MT)
    constexpr int MTMODE = DGB_FLUX_MT >= 0 ? DGB_FLUX_MT : (WS::NTILE * NI <= 10 ? 2 : 0);
    constexpr int MTF = MTMODE ? WS::NTILE : 1;
#pragma unroll 1
    for (int tile0 = 0; tile0 < WS::NTILE; tile0 += MTF) {
      double accZ[DIM][MTF][NI][2];
      constexpr bool UFIRST = MTMODE == 2;     // Z_r - U_0 accumulated in place: the chain of Z_r starts from -U_0
      {
        double accU[MTF][NI][2];
#pragma unroll
        for (int mt = 0; mt < MTF; ++mt)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) { accU[mt][ni][0] = 0.0; accU[mt][ni][1] = 0.0; }
        if (UFIRST) mma_block<NI, MTF>(accU, W.Ss + tile0 * 8 * LDSX, LDSX, S.Wf, EL::LDL, EL::NFPK / 4, lane);
#pragma unroll
        for (int mt = 0; mt < MTF; ++mt)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int s = 0; s < DIM; ++s) {
              accZ[s][mt][ni][0] = UFIRST ? -accU[mt][ni][0] : 0.0;
              accZ[s][mt][ni][1] = UFIRST ? -accU[mt][ni][1] : 0.0;
            }
      }
#pragma unroll
      for (int r = 0; r < DIM; ++r) {
        mma_block<NI, MTF>(accZ[r], Qs + tile0 * 8 * EL::LDQ, EL::LDQ, S.Wq + r * EL::NPR * EL::LDQ, EL::LDQ,
                           EL::NPK / 4, lane);
        mma_block<NI, MTF>(accZ[r], W.Ss + tile0 * 8 * LDSX + (r + 1) * EL::NFPK, LDSX,
                           S.Wf + (r + 1) * EL::NPR * EL::LDL, EL::LDL, EL::NFPK / 4, lane);
      }
      double accU[MTF][NI][2];
#pragma unroll
      for (int mt = 0; mt < MTF; ++mt)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) { accU[mt][ni][0] = 0.0; accU[mt][ni][1] = 0.0; }
      if (!UFIRST) mma_block<NI, MTF>(accU, W.Ss + tile0 * 8 * LDSX, LDSX, S.Wf, EL::LDL, EL::NFPK / 4, lane);
      __syncwarp();                       // every lane has read these tiles' q* rows: they may be overwritten
      const int k8 = lane >> 2;
      // rows of grad q are NP doubles apart: for even NP consecutive columns of a quarter warp would overlap in
      // half their banks (2-way conflicts on every 16-byte store, ncu: 7.5 wavefronts instead of 4); swapping
      // bits 0 and 1 of the column puts them 2 rows = 64 bytes (mod 128) apart
      const int k8s = grad_row_swizzle<NP>(k8);
#pragma unroll
      for (int mt = 0; mt < MTF; ++mt) {
        const int tile = tile0 + mt;
        const int col = tile * 8 + k8;
        const int c = col / KW, e = col - c * KW;
        if (col < WS::NCOL && e < nel) {
          double* sg = W.Ss + tile * 8 * LDSX;
          double m[DIM][DIM];               // m[r][x] = -dr/dx[r][x]
#pragma unroll
          for (int r = 0; r < DIM; ++r)
#pragma unroll
            for (int x = 0; x < DIM; ++x) m[r][x] = -geo.drdx[r * DIM + x][e];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            double z0[DIM], z1[DIM];
#pragma unroll
            for (int r = 0; r < DIM; ++r) { z0[r] = accZ[r][mt][ni][0] - accU[mt][ni][0]; z1[r] = accZ[r][mt][ni][1] - accU[mt][ni][1]; }
            const int i = ni * 8 + 2 * (lane & 3);
#pragma unroll
            for (int x = 0; x < DIM; ++x) {
              double v0 = m[0][x] * z0[0], v1 = m[0][x] * z1[0];
#pragma unroll
              for (int r = 1; r < DIM; ++r) { v0 += m[r][x] * z0[r]; v1 += m[r][x] * z1[r]; }
              if (NP % 2 == 0) {
                if (i < NP) *reinterpret_cast<double2*>(sg + (x * 8 + k8s) * NP + i) = make_double2(v0, v1);
              } else {
                if (i < NP) sg[(x * 8 + k8s) * NP + i] = v0;
                if (i + 1 < NP) sg[(x * 8 + k8s) * NP + i + 1] = v1;
              }
            }
          }
        }
      }
    }
    __syncwarp();
    DGB_WTICK(2);
    if (SQ) {                             // every reader of the state rows but the pointwise phase is done: restage them
      if (wb_next < nwblocks) {
        const long long e1 = ebeg + wb_next * KW;
        flux_stage_rows<DIM, P, KW>(W.Qs[0], d, q, e1, (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW), lane);
      }
      cp_async_commit();
    }
    if (wb_next < nwblocks) {             // connectivity (and, double-buffered, the rows) of the next block have landed by now
      if (SQ) cp_async_wait<1>(); else cp_async_wait<0>();
      __syncwarp();
      const long long e1 = ebeg + wb_next * KW;
      issue_gathers(W.geo[buf ^ 1], (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW));
    }

    // ---- pointwise: total flux at every node, contravariant + Jacobian-scaled, and the wave speed ----
    constexpr int PWU = DGB_FLUX_PW_UNROLL;
#pragma unroll PWU
    for (int n0 = 0; n0 < KW * NP; n0 += 32) {
      const int n = n0 + lane;
      const int e = n / NP, j = n - e * NP;
      if (n < KW * NP && e < nel) {
        double qq[C], g[DIM][EL::CG];
#pragma unroll
        for (int c = 0; c < EL::CG; ++c) {
          const int col = c * KW + e;
          if (c < C) qq[c] = SQ ? q[((long long)c * E + e0 + e) * NP + j] : Qs[col * EL::LDQ + j];
          const double* sg = W.Ss + (col >> 3) * 8 * LDSX + grad_row_swizzle<NP>(col & 7) * NP + j;
#pragma unroll
          for (int x = 0; x < DIM; ++x) g[x][c] = sg[x * 8 * NP];
        }
        double F[DIM][C], lam;
        pw_total_flux<DIM>(qq, g, ph, F, lam);
        const double J = geo.jac[e];
        constexpr int NPLT = FluxT<DIM, P>::NPL;
        const long long t_ps = t_plane_stride<NPLT, NP>(E);
        double* out = T + (e0 + e) * t_elem_stride<NPLT, NP>() + j;
        constexpr int LAMPL_ = FluxT<DIM, P>::LAMPL;
        double tsum[C];
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
            DGB_T_STORE(out + (r * C + c) * t_ps, acc);
            tsum[c] = r == 0 ? acc : tsum[c] + acc;      // (T0 + T1) + T2, the order of the operator program
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) DGB_T_STORE(out + (DIM * C + c) * t_ps, tsum[c]);
        DGB_T_STORE(out + LAMPL_ * t_ps, lam);
      }
    }
    __syncwarp();
    DGB_WTICK(3);
    wb = wb_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------
// pass 2: divergence of the stored flux + face terms
// ------------------------------------------------------------------------------------------
// Per-block inputs of the face phase: small, double-buffered, prefetched one block ahead.
template <int DIM, int P, int KW>
struct alignas(16) Div3Small {
  using EL = ElemT<DIM, P>;
  double Qs[EL::C * KW * EL::NP];
  double Lam[KW * EL::NP];
  double sj[KW][EL::NF];
  long long conn[KW][EL::NF];
  double rj[KW];
  __device__ __forceinline__ double qv(int c, int e, int j) const { return Qs[(c * KW + e) * EL::NP + j]; }
  __device__ __forceinline__ double lamv(int e, int j) const { return Lam[e * EL::NP + j]; }
};

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
  Div3Small<DIM, P, KW> sm[DGB_DIV_SINGLE_SMALL ? 1 : 2];
};

template <int DIM, int P, int KW, int NWARPS>
struct Div3Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];      // volume matrix with the own-side face term folded in (Wv2)
  double Wl[EL::NPR * EL::LDF];
  Div3Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];      // face_lane_code of every face node of a block
};

// chunk t of every plane of a block: CH doubles at element e, node j
template <int DIM, int P, int KW>
__device__ __forceinline__ void div_stage_small(Div3Small<DIM, P, KW>& M, const DiscDev& d, const double* q,
                                                const double* T, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const long long pstride = d.E * NP;
  constexpr int CH = (NP % 2 == 0) ? 2 : 1, NPC = NP / CH;
#pragma unroll
  for (int t0 = 0; t0 < KW * NPC; t0 += 32) {
    const int t = t0 + lane;
    const int e = t / NPC, j = CH * (t - e * NPC);
    if (t < KW * NPC && e < nel) {
      const long long g0 = (e0 + e) * NP + j;
      double* qs = M.Qs + e * NP + j;
      const double* qg = q + g0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (CH == 2) cp_async16(qs + c * (KW * NP), qg + c * pstride);
        else cp_async8(qs + c * (KW * NP), qg + c * pstride);
      }
      const double* lg = T + (e0 + e) * NP + j + FluxT<DIM, P>::LAMPL * pstride;
      if (CH == 2) cp_async16(M.Lam + e * NP + j, lg);
      else cp_async8(M.Lam + e * NP + j, lg);
    }
  }
  if (lane < nel * NF) {
    cp_async8(&M.sj[0][lane], d.sj + e0 * NF + lane);
    cp_async8(&M.conn[0][lane], d.conn + e0 * NF + lane);
  }
  if (lane < nel) cp_async8(&M.rj[lane], d.rj + e0 + lane);
}

template <int DIM, int P, int KW>
__device__ __forceinline__ void div_stage_rows(double* Ts, const DiscDev& d, const double* T, long long e0, int nel,
                                               int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP;
  const long long pstride = d.E * NP;
  constexpr int CH = (NP % 2 == 0) ? 2 : 1, NPC = NP / CH;
#pragma unroll
  for (int t0 = 0; t0 < KW * NPC; t0 += 32) {
    const int t = t0 + lane;
    const int e = t / NPC, j = CH * (t - e * NPC);
    if (t < KW * NPC && e < nel) {
      double* ts = Ts + e * EL::LDV + j;
      const double* tg = T + (e0 + e) * NP + j;
#pragma unroll 1
      for (int r = 0; r < DIM; ++r) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (CH == 2) cp_async16(ts + c * (KW * EL::LDV), tg + c * pstride);
          else cp_async8(ts + c * (KW * EL::LDV), tg + c * pstride);
        }
        ts += EL::NPK;
        tg += C * pstride;
      }
    }
  }
}

template <int DIM> struct VecC { double v[DIM + 2 + DGB_NSPEC]; };

// Boundary face node (rare): inviscid flux of the exterior state, viscous flux of the interior
// state (operators.py: f_bnd = own + B).  The own-side term is read from HBM here (the block's
// rows may still be in flight), and half of it is already in the folded volume matrix, so this
// returns the operand entry  -(own/2 + B).
template <int DIM>
__device__ __noinline__ VecC<DIM> boundary_operand(int bc, int f, VecC<DIM> qm_, const double* __restrict__ Tnode,
                                                   long long pstride, double lam_m, double sj,
                                                   const double* __restrict__ normals, long long nstride, Phys ph) {
  constexpr int C = DIM + 2 + DGB_NSPEC;
  double nrm[DIM], qm[C], qb[C], own[C];
#pragma unroll
  for (int x = 0; x < DIM; ++x) nrm[x] = normals[x * nstride];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    qm[c] = qm_.v[c]; qb[c] = qm_.v[c];
    own[c] = f == 0 ? Tnode[(DIM * C + c) * pstride] : -Tnode[((f - 1) * C + c) * pstride];
  }
  double fnb[C], fni[C];
#if DGB_NSPEC > 0
  // multispecies.py: _ms_pass2 -- far-field exterior state, fnb - fni = n . (F_inv(far) - F_inv(q-))
  pw_exterior_state<DIM>(bc, qm, nrm, ph, qb);
  MsPrim<DIM> sb, sm;
  ms_thermo<DIM>(qb, ph, sb);
  ms_thermo<DIM>(qm, ph, sm);
  double Fb[DIM][C], Fm[DIM][C];
  ms_inviscid_flux<DIM>(qb, sb, Fb);
  ms_inviscid_flux<DIM>(qm, sm, Fm);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double d = nrm[0] * (Fb[0][c] - Fm[0][c]);
#pragma unroll
    for (int x = 1; x < DIM; ++x) d += nrm[x] * (Fb[x][c] - Fm[x][c]);
    fnb[c] = d; fni[c] = 0.0;
  }
  const double lam = fmax(lam_m, ms_wavespeed<DIM>(sb));
#else
  bc_state<DIM, true>(bc, qm, nrm, ph, qb);
  Prim<DIM> sb, sm;
  make_prim<DIM>(qb, ph.gamma, sb);
  make_prim<DIM>(qm, ph.gamma, sm);
  inviscid_normal_flux<DIM>(sb, nrm, fnb);
  inviscid_normal_flux<DIM>(sm, nrm, fni);
  const double lam = fmax(lam_m, wavespeed<DIM>(sb, ph.gamma));
#endif
  VecC<DIM> out;
#pragma unroll
  for (int c = 0; c < C; ++c)
    out.v[c] = -(0.5 * own[c] + 0.5 * sj * (fnb[c] - fni[c]) + 0.5 * sj * lam * (qm[c] - qb[c]));
  return out;
}

// Face phase of pass 2 for one block: gather the neighbour's q, lam and the plane group of T its face selects
// (group dim = sum of the others for its face 0, minus group nf-1 otherwise), Rusanov penalty, operand rows
//   Fs = (nbr - sJ max(lam-, lam+) (q- - q+)) / 2,   nbr = sJ F+.n+
// (the own-side half lives in the folded volume matrix Wv2).  NB face nodes per lane have their gathers in
// flight together.  `M` gives the block's own q / lam rows, face Jacobians and connectivity.
template <int DIM, int P, int KW, int NB, bool GH = true, class SMV>
__device__ __forceinline__ void div_face_phase(const int* flc, const int* fn, const int* perm,
                                               const SMV& M, double* Fs, const DiscDev& d,
                                               const double* __restrict__ q, const double* __restrict__ T,
                                               const double* __restrict__ ghost, const double* __restrict__ Tghost,
                                               const Phys& ph, long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP;
  constexpr int NR = face_rounds<DIM, P, KW>();
  constexpr int LAMPL = FluxT<DIM, P>::LAMPL;
  const long long E = d.E, G = d.G;
#pragma unroll 1
  for (int k0 = 0; k0 < NR; k0 += NB) {
    double qp[NB][C], nbr[NB][C], lam_p[NB];
    long long cnk[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = k0 + b;
      cnk[b] = -1;
      if (k < NR) {
        const int flk = flc[k * 32 + lane];
        const int e = flk & 3, f = (flk >> 2) & 3, m = (flk >> 4) & 15;
        if (flk >= 0 && e < nel) {
          const long long cn = M.conn[e][f];
          cnk[b] = cn;
#ifdef DGB_EXP_LOCALGATHER      // timing experiment only (results invalid): every neighbour is the element itself
          const long long nb = e0 + e;
#else
          const long long nb = DGB_CONN_NB(cn);
#endif
          const int nf = DGB_CONN_NF(cn);
          const int jp = fn[nf * NFP + perm[DGB_CONN_PERM(cn) * NFP + m]];
          const bool in_ghost = GH && nb >= E;
          const long long nbl = in_ghost ? nb - E : nb;
          const long long pstride = (in_ghost ? G : E) * NP;
          const double* qbase = (in_ghost ? ghost : q) + nbl * NP + jp;
          const double* tbase = (in_ghost ? Tghost : T) + nbl * NP + jp;
          const int grp = nf == 0 ? DIM : nf - 1;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            qp[b][c] = DGB_GLD(qbase + c * pstride);
            nbr[b][c] = DGB_GLD(tbase + (grp * C + c) * pstride);
          }
          lam_p[b] = DGB_GLD(tbase + LAMPL * pstride);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int k = k0 + b;
      if (k < NR && cnk[b] >= 0) {
        const int flk = flc[k * 32 + lane];
        const int e = flk & 3, f = (flk >> 2) & 3, jm = (flk >> 8) & 255, fm = (flk >> 16) & 255;
        const int nf = DGB_CONN_NF(cnk[b]), bc = DGB_CONN_BC(cnk[b]);
        const double sj = M.sj[e][f];
        const double lam_m = M.lamv(e, jm);
        double qm[C];
#pragma unroll
        for (int c = 0; c < C; ++c) qm[c] = M.qv(c, e, jm);
        double* fs = Fs + e * EL::LDF + fm;
        if (bc == 0) {
          const double hs = nf == 0 ? 0.5 : -0.5;
          const double pen = 0.5 * (sj * fmax(lam_m, lam_p[b]));
#pragma unroll
          for (int c = 0; c < C; ++c) fs[c * (KW * EL::LDF)] = hs * nbr[b][c] - pen * (qm[c] - qp[b][c]);
        } else {
          VecC<DIM> a_;
#pragma unroll
          for (int c = 0; c < C; ++c) a_.v[c] = qm[c];
          const VecC<DIM> fb = boundary_operand<DIM>(bc, f, a_, T + (e0 + e) * NP + jm, E * NP, lam_m, sj,
                                                     d.normals + (e0 + e) * NF + f, E * NF, ph);
#pragma unroll
          for (int c = 0; c < C; ++c) fs[c * (KW * EL::LDF)] = fb.v[c];
        }
      }
    }
  }
}

template <int DIM, int P, int KW, int NWARPS, bool GH>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_nsdiv3(DiscDev d, const double* __restrict__ q, const double* __restrict__ T,
         const double* __restrict__ ghost, const double* __restrict__ Tghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Div3Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP, NFT = EL::NFT;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();        // face-node rounds per block
  constexpr int NB = DGB_DIV_NB;                  // face nodes per lane whose gathers are in flight together
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Div3Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

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

  const long long wstride = (long long)gridDim.x * NWARPS;
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  int buf = 0;
  if (wb < nwblocks) {
    const long long e0 = ebeg + wb * KW;
    const int nel0 = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
    div_stage_small<DIM, P, KW>(W.sm[0], d, q, T, e0, nel0, lane);
    cp_async_commit();
    div_stage_rows<DIM, P, KW>(W.Ts, d, T, e0, nel0, lane);
    cp_async_commit();
  } else {
    cp_async_commit();
    cp_async_commit();
  }
  TicketStream tks;
  tickets_init(tks, wb, ticket_counter(counter, S.fn, lane), lane);

  // cp.async groups retire in order: S(b), T(b), S(b+1), T(b+1), ...
  constexpr bool SS = DGB_DIV_SINGLE_SMALL != 0;
  static_assert(!(SS && DGB_NSPEC > 0), "the mixture source term reads the block's state rows in the epilogue");
  DGB_WTICK_INIT
  while (wb < nwblocks) {
    const long long e0 = ebeg + wb * KW;
    const int nel = (int)((eend - e0) < (long long)KW ? (eend - e0) : (long long)KW);
    const long long wb_next = tickets_next(tks, wstride, ticket_counter(counter, S.fn, lane), lane);
    const long long e1 = ebeg + wb_next * KW;
    const int nel1 = wb_next < nwblocks ? (int)((eend - e1) < (long long)KW ? (eend - e1) : (long long)KW) : 0;
    if (!SS) {
      if (nel1 > 0) div_stage_small<DIM, P, KW>(W.sm[buf ^ 1], d, q, T, e1, nel1, lane);
      cp_async_commit();                 // S(b+1)
    }
    if (DGB_L2_PREFETCH_BLOCKS > 0) {
      const long long wbp = wb_next + DGB_L2_PREFETCH_BLOCKS;
      if (wbp < nwblocks) {
        const long long ep = ebeg + wbp * KW;
        prefetch_block_rows<NP, KW>(q, C, E * NP, T, DIM * C, E * NP, ep,
                                    (int)((eend - ep) < (long long)KW ? (eend - ep) : (long long)KW), lane);
      }
    }
    DGB_WTICK(5);
    if (SS) cp_async_wait<1>();          // S(b) has landed; T(b) may still be in flight
    else cp_async_wait<2>();             // S(b) has landed; T(b) and S(b+1) may still be in flight
    __syncwarp();
    const Div3Small<DIM, P, KW>& M = W.sm[SS ? 0 : buf];
    DGB_WTICK(0);

    // ---- face gather + Rusanov.  The own-side flux is linear in the block's own T rows with
    //      constant coefficients and lives in the folded volume matrix, so this phase needs only
    //      q, lam and the connectivity of the block -- not its T rows, which are still landing.
    //      Fs = (nbr - sJ max(lam-, lam+) (q- - q+)) / 2,  nbr = sJ F+.n+ gathered from the neighbour.
    div_face_phase<DIM, P, KW, NB, GH>(S.flc, S.fn, S.perm, M, W.Fs, d, q, T, ghost, Tghost, ph, e0, nel, lane);
    DGB_WTICK(1);
    double rj[WS::NTILE];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) rj[mt] = M.rj[(mt * 8 + (lane >> 2)) % KW];
    if (SS) {
      __syncwarp();                      // every lane has read the block's small inputs
      if (nel1 > 0) div_stage_small<DIM, P, KW>(W.sm[0], d, q, T, e1, nel1, lane);
      cp_async_commit();                 // S(b+1): lands during the contraction and the store
    }
    cp_async_wait<1>();                  // T(b) has landed
    __syncwarp();
    DGB_WTICK(2);

    // ---- tensor-core contraction -------------------------------------------------------------
    double acc[WS::NTILE][EL::NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
    mma_block<EL::NI, WS::NTILE>(acc, W.Ts, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
    mma_block<EL::NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
    __syncwarp();                        // all operand rows consumed: the next block may land on them
    DGB_WTICK(3);
    if (nel1 > 0) div_stage_rows<DIM, P, KW>(W.Ts, d, T, e1, nel1, lane);
    cp_async_commit();                   // T(b+1)

    // ---- 1/J and the (RK-fused) store --------------------------------------------------------
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt) {
      const int col = mt * 8 + (lane >> 2);
      const int c = col / KW, e = col - c * KW;
      if (col < WS::NCOL && e < nel) {
        const long long rowbase = ((long long)c * E + e0 + e) * NP;
#if DGB_NSPEC > 0
        const double sgn = c == 2 + DIM + ph.ra ? -1.0 : (c == 2 + DIM + ph.rb ? 1.0 : 0.0);     // species a -> species b
#endif
#pragma unroll
        for (int ni = 0; ni < EL::NI; ++ni) {
          const int i = ni * 8 + 2 * (lane & 3);
#if DGB_NSPEC > 0
          // chemistry (fallback kernel: the rate is evaluated per output pair from the block's own state rows, which
          // stay valid in the double-buffered small inputs until the next block's land)
          double w0 = 0.0, w1 = 0.0;
          if (sgn != 0.0 && !SS) {
            double qq[C];
            if (i < NP) {
#pragma unroll
              for (int cc = 0; cc < C; ++cc) qq[cc] = M.qv(cc, e, i);
              w0 = sgn * pw_arrhenius<DIM>(qq, ph);
            }
            if (i + 1 < NP) {
#pragma unroll
              for (int cc = 0; cc < C; ++cc) qq[cc] = M.qv(cc, e, i + 1);
              w1 = sgn * pw_arrhenius<DIM>(qq, ph);
            }
          }
          store_pair<NP>(ep, rowbase + i, i, rj[mt] * acc[mt][ni][0] + w0, rj[mt] * acc[mt][ni][1] + w1);
          continue;
#endif
          store_pair<NP>(ep, rowbase + i, i, rj[mt] * acc[mt][ni][0], rj[mt] * acc[mt][ni][1]);
        }
      }
    }
    DGB_WTICK(4);
    wb = wb_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------
// Euler right-hand side in one pass, built like k_nsdiv3 (k_euler4).
//
// rows + geometry by cp.async (double-buffered, one block ahead) -> the neighbour gathers of ALL face
// nodes of the block are issued first and fly while the volume flux is evaluated -> T[r][c] =
// sum_x dr/dx[r][x] F[x][c] into the DMMA operand rows -> face phase from the gathered q+:
// Fs = -(fscale F(q+).n + fscale max(lam-, lam+)(q- - q+)) / 2, the own-side half of the numerical flux
// being linear in the T rows and folded into the volume matrix (Wv2, as in pass 2 of Navier-Stokes)
// -> one DMMA contraction -> (RK-fused) store.  Boundary faces need no special path: the exterior
// state replaces q+.
// ------------------------------------------------------------------------------------------
template <int DIM, int P, int KW>
struct alignas(16) Euler4Geo {
  using EL = ElemT<DIM, P>;
  double drdx[DIM * DIM][KW];
  double nrm[DIM][KW][EL::NF];
  double fsc[KW][EL::NF];
  long long conn[KW][EL::NF];
};

template <int DIM, int P, int KW>
struct alignas(16) Euler4Warp {
  using EL = ElemT<DIM, P>;
  static constexpr int NCOL = EL::C * KW;
  static constexpr int NTILE = (NCOL + 7) / 8;
  double Ts[NCOL * EL::LDV];
  double Fs[NCOL * EL::LDF];
  double Lam[KW * EL::NP];
  double Qs[EL::C * KW * EL::NP];        // single buffer: the next block's rows are staged once the face phase has read these
  Euler4Geo<DIM, P, KW> geo[2];
};

template <int DIM, int P, int KW, int NWARPS>
struct Euler4Smem {
  using EL = ElemT<DIM, P>;
  double Wv[EL::NPR * EL::LDV];
  double Wl[EL::NPR * EL::LDF];
  Euler4Warp<DIM, P, KW> w[NWARPS];
  int fn[EL::NF * EL::NFP];
  int perm[EL::NPERM * EL::NFP];
  int flc[face_rounds<DIM, P, KW>() * 32];
};

template <int DIM, int P, int KW>
__device__ __forceinline__ void euler4_stage(double* Qs, Euler4Geo<DIM, P, KW>& M, const DiscDev& d, const double* q,
                                             long long e0, int nel, int lane) {
  using EL = ElemT<DIM, P>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF;
  const long long E = d.E;
  constexpr int CH = (NP % 2 == 0) ? 2 : 1, NPC = NP / CH;
#pragma unroll
  for (int t0 = 0; t0 < KW * NPC; t0 += 32) {
    const int t = t0 + lane;
    const int e = t / NPC, j = CH * (t - e * NPC);
    if (t < KW * NPC && e < nel) {
      double* qs = Qs + e * NP + j;
      const double* qg = q + (e0 + e) * NP + j;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (CH == 2) cp_async16(qs + c * (KW * NP), qg + c * E * NP);
        else cp_async8(qs + c * (KW * NP), qg + c * E * NP);
      }
    }
  }
  for (int n = lane; n < DIM * DIM * KW; n += 32) {
    const int rx = n / KW, e = n - rx * KW;
    if (e < nel) cp_async8(&M.drdx[rx][e], d.drdx + (long long)rx * E + e0 + e);
  }
  if (lane < nel * NF) {
#pragma unroll
    for (int x = 0; x < DIM; ++x) cp_async8(&M.nrm[x][0][lane], d.normals + ((long long)x * E + e0) * NF + lane);
    cp_async8(&M.fsc[0][lane], d.fscale + e0 * NF + lane);
    cp_async8(&M.conn[0][lane], d.conn + e0 * NF + lane);
  }
}

template <int DIM, int P, int KW, int NWARPS, bool GH>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_euler4(DiscDev d, const double* __restrict__ q, const double* __restrict__ ghost,
         Epilogue ep, Phys ph, long long ebeg, long long eend, long long nwblocks,
         unsigned long long* __restrict__ counter) {
  using EL = ElemT<DIM, P>;
  using WS = Euler4Warp<DIM, P, KW>;
  constexpr int C = EL::C, NP = EL::NP, NF = EL::NF, NFP = EL::NFP;
  constexpr int NT = NWARPS * 32;
  constexpr int NR = face_rounds<DIM, P, KW>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& S = *reinterpret_cast<Euler4Smem<DIM, P, KW, NWARPS>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = d.E, G = d.G;

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
  long long wb = (long long)blockIdx.x * NWARPS + warp;
  if (wb >= nwblocks) return;
  euler4_stage<DIM, P, KW>(W.Qs, W.geo[0], d, q, ebeg + wb * KW, nel_of(wb), lane);
  cp_async_commit();
  TicketStream tks;
  tickets_init(tks, wb, ticket_counter(counter, S.fn, lane), lane);

  for (int i = 0;; ++i) {
    const int buf = i & 1;
    const long long e0 = ebeg + wb * KW;
    const int nel = nel_of(wb);
    const long long wb_next = tickets_next(tks, wstride, ticket_counter(counter, S.fn, lane), lane);
    const int nel1 = nel_of(wb_next);
    cp_async_wait<0>();                  // this block's rows + geometry have landed (staged during the previous contraction)
    __syncwarp();
    const Euler4Geo<DIM, P, KW>& M = W.geo[buf];

    // ---- neighbour states of every face node: in flight during the volume phase --------------
    double qp[NR][C];
    long long cnk[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      cnk[k] = -1;
      const int flk = S.flc[k * 32 + lane];
      const int e = flk & 3, f = (flk >> 2) & 3, m = (flk >> 4) & 15;
      if (flk >= 0 && e < nel) {
        const long long cn = M.conn[e][f];
        cnk[k] = cn;
        const long long nb = DGB_CONN_NB(cn);
        const int jp = S.fn[DGB_CONN_NF(cn) * NFP + S.perm[DGB_CONN_PERM(cn) * NFP + m]];
        const bool in_ghost = GH && nb >= E;
        const long long pstride = (in_ghost ? G : E) * NP;
        const double* pbase = (in_ghost ? ghost : q) + (in_ghost ? nb - E : nb) * NP + jp;
#pragma unroll
        for (int c = 0; c < C; ++c) qp[k][c] = pbase[c * pstride];
      }
    }

    // ---- volume flux -> contravariant operand rows, wave speed ---------------------------------
    constexpr int PWU = DGB_EULER_PW_UNROLL;
#pragma unroll PWU
    for (int n0 = 0; n0 < KW * NP; n0 += 32) {
      const int n = n0 + lane;
      const int e = n / NP, j = n - e * NP;
      if (n < KW * NP && e < nel) {
        double qq[C];
#pragma unroll
        for (int c = 0; c < C; ++c) qq[c] = W.Qs[(c * KW + e) * NP + j];
        Prim<DIM> s;
        make_prim<DIM>(qq, ph.gamma, s);
        double F[DIM][C];
        inviscid_flux<DIM>(s, F);
#pragma unroll
        for (int r = 0; r < DIM; ++r) {
          double mm[DIM];
#pragma unroll
          for (int x = 0; x < DIM; ++x) mm[x] = M.drdx[r * DIM + x][e];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            double acc = mm[0] * F[0][c];
#pragma unroll
            for (int x = 1; x < DIM; ++x) acc += mm[x] * F[x][c];
            W.Ts[(c * KW + e) * EL::LDV + r * EL::NPK + j] = acc;
          }
        }
        W.Lam[n] = wavespeed<DIM>(s, ph.gamma);
      }
    }
    __syncwarp();

    // ---- face phase from the gathered states ----------------------------------------------------
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      if (cnk[k] >= 0) {
        const int flk = S.flc[k * 32 + lane];
        const int e = flk & 3, f = (flk >> 2) & 3, jm = (flk >> 8) & 255, fm = (flk >> 16) & 255;
        const int bc = DGB_CONN_BC(cnk[k]);
        double qm[C], nrm[DIM];
#pragma unroll
        for (int c = 0; c < C; ++c) qm[c] = W.Qs[(c * KW + e) * NP + jm];
#pragma unroll
        for (int x = 0; x < DIM; ++x) nrm[x] = M.nrm[x][e][f];
        if (bc != 0) bc_state<DIM, false>(bc, qm, nrm, ph, qp[k]);
        Prim<DIM> sp_;
        make_prim<DIM>(qp[k], ph.gamma, sp_);
        double fnp[C];
        inviscid_normal_flux<DIM>(sp_, nrm, fnp);
        const double fs_ = M.fsc[e][f];
        const double pen = fmax(W.Lam[e * NP + jm], wavespeed<DIM>(sp_, ph.gamma));
        double* fsrow = W.Fs + e * EL::LDF + fm;
#pragma unroll
        for (int c = 0; c < C; ++c) fsrow[c * (KW * EL::LDF)] = -0.5 * fs_ * (fnp[c] + pen * (qm[c] - qp[k][c]));
      }
    }
    __syncwarp();                        // Qs and this block's geometry are no longer needed ...

    // ... so the next block's rows start their trip now and land during the contraction
    if (nel1 > 0) euler4_stage<DIM, P, KW>(W.Qs, W.geo[buf ^ 1], d, q, ebeg + wb_next * KW, nel1, lane);
    cp_async_commit();
    if (DGB_L2_PREFETCH_BLOCKS > 0) {
      const long long wbp = wb_next + DGB_L2_PREFETCH_BLOCKS;
      if (wbp < nwblocks) {
        const long long epf = ebeg + wbp * KW;
        prefetch_block_rows<NP, KW>(q, C, E * NP, q, 0, 0, epf,
                                    (int)((eend - epf) < (long long)KW ? (eend - epf) : (long long)KW), lane);
      }
    }

    // ---- tensor-core contraction + (RK-fused) store ----------------------------------------------
    double acc[WS::NTILE][EL::NI][2];
#pragma unroll
    for (int mt = 0; mt < WS::NTILE; ++mt)
#pragma unroll
      for (int ni = 0; ni < EL::NI; ++ni) { acc[mt][ni][0] = 0.0; acc[mt][ni][1] = 0.0; }
    mma_block<EL::NI, WS::NTILE>(acc, W.Ts, EL::LDV, S.Wv, EL::LDV, EL::KV / 4, lane);
    mma_block<EL::NI, WS::NTILE>(acc, W.Fs, EL::LDF, S.Wl, EL::LDF, EL::KF / 4, lane);
    store_block<NP, KW, WS::NCOL, WS::NTILE, EL::NI>(ep, acc, E, e0, nel, lane);
    __syncwarp();                        // operand rows free for the next block
    if (nel1 == 0) break;
    wb = wb_next;
  }
  cp_async_wait<0>();
}

}  // namespace dgb
