// C ABI of the B200 DG right-hand-side path: discretisation handle, kernel dispatch, halo
// packing.  See include/dgb200.h for the contract and the reference interfaces replaced.
#include "dgb_internal.h"
#include "dgb_kernels_async.cuh"
#include "dgb_kernels_warp.cuh"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {
thread_local std::string g_err;
}  // namespace

int dgb_fail(int code, const std::string& msg) { g_err = msg; return code; }

int dgb_num_sms() {
  static int n[64] = {};
  int dev = 0; cudaGetDevice(&dev);
  int& v = n[dev & 63];
  if (!v) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

// SMs left free by the persistent kernels while a halo exchange is in flight, so that the NCCL send/recv
// kernel on the communication stream can start at once instead of waiting for a CTA to retire
static int g_sm_reserve = 0;
int dgb_grid_sms() { const int n = dgb_num_sms() - g_sm_reserve; return n < 1 ? 1 : n; }
extern "C" int dgb_set_sm_reserve(int nsm) {
  if (nsm < 0 || nsm >= dgb_num_sms()) return dgb_fail(DGB_ERR_INVALID, "SM reserve outside [0, number of SMs)");
  g_sm_reserve = nsm;
  return DGB_OK;
}

namespace {
int fail(int code, const std::string& msg) { return dgb_fail(code, msg); }
int num_sms() { return dgb_num_sms(); }
}  // namespace

// {{{ connectivity compression / expansion

namespace {

__global__ void k_build_conn(const long long* __restrict__ vm, const long long* __restrict__ vp,
                             const long long* __restrict__ bc, const int* __restrict__ tables,
                             long long E, long long G, int Np, int Nf, int Nfp, int nperm,
                             long long* __restrict__ conn, int* __restrict__ err) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= E * Nf) return;
  const long long e = idx / Nf;
  const int f = (int)(idx - e * Nf);
  const int* fn = tables;
  const int* perm = tables + Nf * Nfp;
  const long long base = idx * Nfp;
  const long long limit = (E + G) * Np;
  bool oob = false, bad = false;
  for (int m = 0; m < Nfp; ++m) {
    const long long a = vm[base + m], b = vp[base + m];
    if (a < 0 || a >= E * (long long)Np || b < 0 || b >= limit) oob = true;
    if (a != e * Np + fn[f * Nfp + m]) bad = true;
  }
  if (oob) { atomicMax(err, DGB_ERR_OUT_OF_BOUNDS + 100); return; }
  const long long bck = bc[idx];
  if (bck < 0 || bck > 2) bad = true;
  long long packed = 0;
  if (!bad && bck != 0) {
    for (int m = 0; m < Nfp; ++m) if (vp[base + m] != vm[base + m]) bad = true;
    packed = dgb::conn_pack(e, f, 0, (int)bck);
  } else if (!bad) {
    const long long nb = vp[base] / Np;
    bool found = false;
    for (int nf = 0; nf < Nf && !found; ++nf)
      for (int p = 0; p < nperm && !found; ++p) {
        bool ok = true;
        for (int m = 0; m < Nfp; ++m)
          if (vp[base + m] != nb * Np + fn[nf * Nfp + perm[p * Nfp + m]]) { ok = false; break; }
        if (ok) { found = true; packed = dgb::conn_pack(nb, nf, p, 0); }
      }
    if (!found) bad = true;
  }
  if (bad) { atomicMax(err, DGB_ERR_BAD_MAP); return; }
  conn[idx] = packed;
}

// the validated int64 neighbour map of the API narrowed to 32 bits: what the lean face phases gather through
__global__ void k_build_gidx(const long long* __restrict__ vp, long long n, unsigned* __restrict__ gidx) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) gidx[i] = (unsigned)vp[i];
}

__global__ void k_expand_conn(const long long* __restrict__ conn, const int* __restrict__ tables,
                              long long E, int Np, int Nf, int Nfp,
                              long long* __restrict__ vm, long long* __restrict__ vp) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= E * Nf * Nfp) return;
  const long long ef = n / Nfp;
  const int m = (int)(n - ef * Nfp);
  const long long e = ef / Nf;
  const int f = (int)(ef - e * Nf);
  const int* fn = tables;
  const int* perm = tables + Nf * Nfp;
  const long long c = conn[ef];
  const long long own = e * Np + fn[f * Nfp + m];
  vm[n] = own;
  vp[n] = DGB_CONN_BC(c) ? own
                         : DGB_CONN_NB(c) * Np + fn[DGB_CONN_NF(c) * Nfp + perm[DGB_CONN_PERM(c) * Nfp + m]];
}

__global__ void k_pack_elements(double* __restrict__ dst, const double* __restrict__ src,
                                const long long* __restrict__ elems, long long ncomp, long long nsrc,
                                long long nsel, long long ndofs) {
  const long long total = ncomp * nsel * ndofs;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    const long long j = n % ndofs, ci = n / ndofs;
    const long long i = ci % nsel, c = ci / nsel;
    dst[n] = src[(c * nsrc + elems[i]) * ndofs + j];
  }
}

// halo rows straight into a (peer-mapped) ghost array: dst[(c*ndst + slot0 + i)*ndofs + j] = src[(c*nsrc + elems[i])*ndofs + j]
__global__ void k_pack_elements_to(double* __restrict__ dst, long long ndst, long long slot0,
                                   const double* __restrict__ src, const long long* __restrict__ elems,
                                   long long ncomp, long long nsrc, long long nsel, long long ndofs) {
  const long long total = ncomp * nsel * ndofs;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    const long long j = n % ndofs, ci = n / ndofs;
    const long long i = ci % nsel, c = ci / nsel;
    dst[(c * ndst + slot0 + i) * ndofs + j] = src[(c * nsrc + elems[i]) * ndofs + j];
  }
}

// stream-ordered flags in (peer-mapped) device memory: everything enqueued before dgb_flag_signal on the
// stream is visible system-wide before the flag takes its value; dgb_flag_wait holds the stream until then
__global__ void k_flag_signal(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

__global__ void k_flag_wait(const unsigned long long* flag, unsigned long long value) {
  // bounded: a neighbour that never signals (crashed rank) must not wedge the GPU -- after ~20 s of
  // polling the kernel traps and the stream reports an error instead of hanging
  unsigned long long v;
  for (long long it = 0;; ++it) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= value) return;
    if (it > 40000000LL) __trap();
    __nanosleep(500);
  }
}

}  // namespace

// }}}

// {{{ launch configuration per (dim, order)

namespace {

// launch configuration of the warp-autonomous kernels (dgb_kernels_warp.cuh), the default path:
// KW elements per warp (C*KW columns padded to whole 8-column tiles), as many warps per SM as fit
#ifndef DGB_GRAD_WARPS
#define DGB_GRAD_WARPS 16
#endif
#ifndef DGB_RHS_WARPS
#define DGB_RHS_WARPS 12
#endif
constexpr int kSmemBudget = 232448 - 1024;   // 227 KB usable per CTA minus the 1 KB system reserve
constexpr int fit_warps(size_t fixed, size_t per_warp, int cap) {
  int n = (int)((kSmemBudget - fixed) / per_warp);
  return n < 1 ? 1 : (n > cap ? cap : n);
}
template <int DIM, int P> struct Cfg3 {
  static constexpr int KW = DIM == 3 ? 3 : 4;
  static constexpr size_t rhs_per = sizeof(dgb::Rhs3Warp<DIM, P, KW>);
  static constexpr size_t rhs_fixed = sizeof(dgb::Rhs3Smem<DIM, P, KW, 1>) - rhs_per;
  static constexpr int NW = fit_warps(rhs_fixed, rhs_per, DGB_RHS_WARPS);
  static constexpr size_t grad_per = sizeof(dgb::Grad3Warp<DIM, P, KW>);
  static constexpr size_t grad_fixed = sizeof(dgb::Grad3Smem<DIM, P, KW, 1>) - grad_per;
  static constexpr int NWG = fit_warps(grad_fixed, grad_per, DGB_GRAD_WARPS);
};

template <int DIM, int P, bool VISCOUS>
int launch_rhs3(const dgb_disc* d, const double* q, const double* gq, const double* ghost, const double* gghost,
                const dgb::Epilogue& ep, const dgb::Phys& ph, cudaStream_t st, long long ebeg = 0, long long eend = -1) {
  using C = Cfg3<DIM, P>;
  auto kern = dgb::k_rhs3<DIM, P, C::KW, C::NW, VISCOUS>;
  const size_t smem = sizeof(dgb::Rhs3Smem<DIM, P, C::KW, C::NW>);
  if (eend < 0) eend = d->dev.E;
  const long long nwb = (eend - ebeg + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured;
  if (!configured()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured() = true; }
  const long long need = (nwb + C::NW - 1) / C::NW;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters + 1, 0, sizeof(unsigned long long), st));
  kern<<<grid, C::NW * 32, smem, st>>>(d->dev, q, gq, ghost, gghost, ep, ph, nwb, d->counters + 1, ebeg, eend);
  {
    cudaError_t e_ = cudaGetLastError();
    if (e_ != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      return fail(DGB_ERR_CUDA, std::string("k_rhs3 launch: ") + cudaGetErrorString(e_) + " (regs=" +
                  std::to_string(fa.numRegs) + " maxThreads=" + std::to_string(fa.maxThreadsPerBlock) + " threads=" +
                  std::to_string(C::NW * 32) + " smem=" + std::to_string(smem) + " static=" +
                  std::to_string(fa.sharedSizeBytes) + " local=" + std::to_string(fa.localSizeBytes) + ")");
    }
  }
  return DGB_OK;
}

template <int DIM, int P>
int launch_grad3(const dgb_disc* d, const double* q, const double* ghost, double* grad, const dgb::Phys& ph,
                 cudaStream_t st) {
  using C = Cfg3<DIM, P>;
  auto kern = dgb::k_grad3<DIM, P, C::KW, C::NWG>;
  const size_t smem = sizeof(dgb::Grad3Smem<DIM, P, C::KW, C::NWG>);
  const long long nwb = (d->dev.E + C::KW - 1) / C::KW;
  if (nwb == 0) return DGB_OK;
  static DgbPerDevice configured;
  if (!configured()) { DGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); configured() = true; }
  const long long need = (nwb + C::NWG - 1) / C::NWG;
  const int grid = (int)(need < dgb_grid_sms() ? need : dgb_grid_sms());
  DGB_CUDA(cudaMemsetAsync(d->counters, 0, sizeof(unsigned long long), st));
  kern<<<grid, C::NWG * 32, smem, st>>>(d->dev, q, ghost, grad, ph, nwb, d->counters);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

#ifdef DGB_ONLY_3D_P3   // fast kernel-tuning builds (scripts/ab_variants.py)
#define DGB_FOR_EACH_ELEMENT(X) X(3, 3)
#else
#define DGB_FOR_EACH_ELEMENT(X) X(2, 1) X(2, 2) X(2, 3) X(2, 4) X(3, 1) X(3, 2) X(3, 3) X(3, 4)
#endif

int dispatch_rhs(const dgb_disc* d, bool viscous, const double* q, const double* gq, const double* ghost,
                 const double* gghost, const dgb::Epilogue& ep, const dgb::Phys& ph, cudaStream_t st,
                 long long ebeg = 0, long long eend = -1) {
  // Euler: k_euler4 (dgb_kernels_flux.cuh) unless DGB_EULER_KERNEL=3 asks for k_rhs3<inviscid>
  static int euler_kernel = -1;
  if (euler_kernel < 0) { const char* e = getenv("DGB_EULER_KERNEL"); euler_kernel = e ? atoi(e) : 4; }
  if (!viscous && euler_kernel == 4) return dgb_launch_euler4(d, q, ghost, ep, ph, ebeg, eend, st);
#define X(DIM, P)                                                                              \
  if (d->dim == DIM && d->order == P)                                                          \
    return viscous ? launch_rhs3<DIM, P, true>(d, q, gq, ghost, gghost, ep, ph, st, ebeg, eend)   \
                   : launch_rhs3<DIM, P, false>(d, q, gq, ghost, gghost, ep, ph, st, ebeg, eend);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

int dispatch_grad(const dgb_disc* d, const double* q, const double* ghost, double* grad, const dgb::Phys& ph,
                  cudaStream_t st) {
#define X(DIM, P) if (d->dim == DIM && d->order == P) return launch_grad3<DIM, P>(d, q, ghost, grad, ph, st);
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  return fail(DGB_ERR_INVALID, "unsupported (dim, order)");
}

template <int DIM, int P>
void fill_padded(const double* Sw, const double* lift, const int64_t* face_nodes, std::vector<double>& Wv,
                 std::vector<double>& Wl, std::vector<double>& Wq, std::vector<double>& Wf, std::vector<double>& Wv2) {
  using EL = dgb::ElemT<DIM, P>;
  Wv.assign((size_t)EL::NPR * EL::LDV, 0.0);
  Wl.assign((size_t)EL::NPR * EL::LDF, 0.0);
  Wq.assign((size_t)DIM * EL::NPR * EL::LDQ, 0.0);
  Wf.assign((size_t)EL::NF * EL::NPR * EL::LDL, 0.0);
  for (int r = 0; r < DIM; ++r)
    for (int i = 0; i < EL::NP; ++i)
      for (int j = 0; j < EL::NP; ++j) {
        const double v = Sw[((size_t)r * EL::NP + i) * EL::NP + j];
        Wv[(size_t)i * EL::LDV + r * EL::NPK + j] = v;
        Wq[((size_t)r * EL::NPR + i) * EL::LDQ + j] = v;
      }
  for (int i = 0; i < EL::NP; ++i)
    for (int f = 0; f < EL::NF; ++f)
      for (int m = 0; m < EL::NFP; ++m) {
        const double v = lift[(size_t)i * EL::NFT + f * EL::NFP + m];
        Wl[(size_t)i * EL::LDF + f * EL::NFP + m] = v;
        Wf[((size_t)f * EL::NPR + i) * EL::LDL + m] = v;
      }
  // flux arrangement: sJ F-.n at face node (f, m) is sum_r a[f][r] T[r][fn[f][m]] with a[0][r] = 1,
  // a[f][r] = -delta(r, f-1); the numerical flux contains half of it, which therefore folds into
  // the volume matrix:  Wv2[i][r, j] = Sw_r[i][j] - 1/2 sum_{(f,m): fn[f][m] = j} a[f][r] lift[i][f, m]
  Wv2 = Wv;
  for (int i = 0; i < EL::NP; ++i)
    for (int f = 0; f < EL::NF; ++f)
      for (int m = 0; m < EL::NFP; ++m) {
        const int j = (int)face_nodes[f * EL::NFP + m];
        if (j < 0 || j >= EL::NP) continue;          // rejected by dgb_disc_create right after this
        const double v = lift[(size_t)i * EL::NFT + f * EL::NFP + m];
        for (int r = 0; r < DIM; ++r) {
          const double a = f == 0 ? 1.0 : (r == f - 1 ? -1.0 : 0.0);
          Wv2[(size_t)i * EL::LDV + r * EL::NPK + j] -= 0.5 * a * v;
        }
      }
}

template <int DIM, int P> void elem_sizes(int* Np, int* Nf, int* Nfp, int* nperm) {
  using EL = dgb::ElemT<DIM, P>;
  *Np = EL::NP; *Nf = EL::NF; *Nfp = EL::NFP; *nperm = EL::NPERM;
}

template <typename T>
int upload(T** dev, const std::vector<T>& host, cudaStream_t st) {
  DGB_CUDA(cudaMalloc((void**)dev, host.size() * sizeof(T)));
  DGB_CUDA(cudaMemcpyAsync(*dev, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return DGB_OK;
}

void make_phys(dgb::Phys& ph, int C, const double* qfar, const double* phys) {
  ph.gamma = phys ? phys[0] : 1.4; ph.mu = phys ? phys[1] : 0.0; ph.kappa = phys ? phys[2] : 0.0;
  ph.rgas = phys ? phys[3] : 1.0;
  for (int c = 0; c < 5; ++c) ph.qfar[c] = (qfar && c < C) ? qfar[c] : 0.0;
}

}  // namespace

// }}}

extern "C" {

const char* dgb_last_error(void) { return g_err.c_str(); }
int dgb_version(void) { return 100; }

int dgb_malloc(void** dev, size_t bytes) { DGB_CUDA(cudaMalloc(dev, bytes ? bytes : 1)); return DGB_OK; }
int dgb_free(void* dev) { DGB_CUDA(cudaFree(dev)); return DGB_OK; }
int dgb_host_alloc(void** host, size_t bytes) { DGB_CUDA(cudaMallocHost(host, bytes ? bytes : 1)); return DGB_OK; }
int dgb_host_free(void* host) { DGB_CUDA(cudaFreeHost(host)); return DGB_OK; }
int dgb_memcpy_h2d(void* dev, const void* host, size_t bytes, void* stream) {
  DGB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream)); return DGB_OK;
}
int dgb_memcpy_d2h(void* host, const void* dev, size_t bytes, void* stream) {
  DGB_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream)); return DGB_OK;
}
int dgb_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  DGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream)); return DGB_OK;
}
int dgb_stream_sync(void* stream) { DGB_CUDA(cudaStreamSynchronize((cudaStream_t)stream)); return DGB_OK; }

int dgb_disc_create(dgb_disc** out, int dim, int order, int64_t E, int64_t G, const double* Sw_host,
                    const double* lift_host, const int64_t* face_nodes_host, const int64_t* face_perms_host,
                    const double* drdx_dev, const double* normals_dev, const double* fscale_dev,
                    const int64_t* vmap_m_dev, const int64_t* vmap_p_dev, const int64_t* bc_kind_dev,
                    void* stream) {
  if (!out) return fail(DGB_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (E < 0 || G < 0 || E + G >= (1LL << 31)) return fail(DGB_ERR_INVALID, "element count out of range");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> Wv, Wl, Wq, Wf, Wv2;
  int Np = 0, Nf = 0, Nfp = 0, nperm = 0;
  bool ok = false;
#define X(DIM, P)                                                        \
  if (dim == DIM && order == P) {                                        \
    fill_padded<DIM, P>(Sw_host, lift_host, face_nodes_host, Wv, Wl, Wq, Wf, Wv2); \
    elem_sizes<DIM, P>(&Np, &Nf, &Nfp, &nperm);                          \
    ok = true;                                                           \
  }
  DGB_FOR_EACH_ELEMENT(X)
#undef X
  if (!ok) return fail(DGB_ERR_INVALID, "unsupported (dim, order): dim in {2,3}, order in 1..4");
  std::vector<int> tables((size_t)Nf * Nfp + (size_t)nperm * Nfp);
  for (int n = 0; n < Nf * Nfp; ++n) {
    if (face_nodes_host[n] < 0 || face_nodes_host[n] >= Np) return fail(DGB_ERR_OUT_OF_BOUNDS, "face node table out of range");
    tables[n] = (int)face_nodes_host[n];
  }
  for (int n = 0; n < nperm * Nfp; ++n) {
    if (face_perms_host[n] < 0 || face_perms_host[n] >= Nfp) return fail(DGB_ERR_OUT_OF_BOUNDS, "face permutation table out of range");
    tables[(size_t)Nf * Nfp + n] = (int)face_perms_host[n];
  }
  dgb_disc* d = new dgb_disc();
  d->dim = dim; d->order = order; d->Np = Np; d->Nf = Nf; d->Nfp = Nfp; d->nperm = nperm;
  int rc;
  if ((rc = upload(&d->Wv, Wv, st)) || (rc = upload(&d->Wl, Wl, st)) || (rc = upload(&d->Wq, Wq, st)) ||
      (rc = upload(&d->Wf, Wf, st)) || (rc = upload(&d->Wv2, Wv2, st)) || (rc = upload(&d->tables, tables, st))) { dgb_disc_destroy(d); return rc; }
  int* err_dev = nullptr;
  cudaError_t ce = cudaMalloc((void**)&d->conn, sizeof(long long) * (size_t)(E * Nf ? E * Nf : 1));
  if (ce == cudaSuccess) ce = cudaMalloc((void**)&err_dev, sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemsetAsync(err_dev, 0, sizeof(int), st);
  if (ce != cudaSuccess) { dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, cudaGetErrorString(ce)); }
  int err_host = 0;
  if (E > 0) {
    const long long n = E * Nf;
    k_build_conn<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        (const long long*)vmap_m_dev, (const long long*)vmap_p_dev, (const long long*)bc_kind_dev, d->tables,
        E, G, Np, Nf, Nfp, nperm, d->conn, err_dev);
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&err_host, err_dev, sizeof(int), cudaMemcpyDeviceToHost, st);
  }
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  cudaFree(err_dev);
  if (ce != cudaSuccess) { dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, cudaGetErrorString(ce)); }
  if (err_host >= 100) { dgb_disc_destroy(d); return fail(DGB_ERR_OUT_OF_BOUNDS, "face index map leaves [0, (E+G)*Np)"); }
  if (err_host) { dgb_disc_destroy(d); return fail(DGB_ERR_BAD_MAP, "face index maps are not a conforming simplex face map"); }
  if (E > 0 && (E + G) * Np < (1LL << 32)) {
    const long long n = E * Nf * Nfp;
    if (cudaMalloc((void**)&d->gidx, sizeof(unsigned) * (size_t)n) != cudaSuccess) { dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, "gather map"); }
    k_build_gidx<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const long long*)vmap_p_dev, n, d->gidx);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) { dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, "gather map kernel"); }
  }
  if (cudaMalloc((void**)&d->timing, sizeof(long long) * 8 * 4096) != cudaSuccess ||
      cudaMemsetAsync(d->timing, 0, sizeof(long long) * 8 * 4096, st) != cudaSuccess) {
    dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, "timing buffer");
  }
  d->dev.timing = d->timing;
  if (cudaMalloc((void**)&d->counters, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    dgb_disc_destroy(d); return fail(DGB_ERR_CUDA, "work counters");
  }
  d->dev.E = E; d->dev.G = G;
  d->dev.Wv = d->Wv; d->dev.Wl = d->Wl; d->dev.Wq = d->Wq; d->dev.Wf = d->Wf; d->dev.Wv2 = d->Wv2;
  d->dev.drdx = drdx_dev; d->dev.normals = normals_dev; d->dev.fscale = fscale_dev;
  d->dev.conn = d->conn; d->dev.tables = d->tables; d->dev.gidx = d->gidx;
  d->bc_kind = bc_kind_dev;
  *out = d;
  return DGB_OK;
}

int dgb_disc_destroy(dgb_disc* d) {
  if (!d) return DGB_OK;
  dgb_disc_free_jacobian(d);
  cudaFree(d->Wv2); cudaFree(d->Wv); cudaFree(d->Wl); cudaFree(d->Wq); cudaFree(d->Wf); cudaFree(d->conn); cudaFree(d->gidx); cudaFree(d->tables); cudaFree(d->timing); cudaFree(d->counters);
  delete d;
  return DGB_OK;
}

int dgb_debug_phase_cycles(const dgb_disc* d, long long* out8_host) {
  // sum of the per-CTA phase cycle counters (only filled by builds with -DDGB_PHASE_TIMING); resets them
  if (!d) return fail(DGB_ERR_INVALID, "null handle");
  std::vector<long long> h(8 * 4096);
  DGB_CUDA(cudaMemcpy(h.data(), d->timing, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost));
  DGB_CUDA(cudaMemset(d->timing, 0, sizeof(long long) * h.size()));
  for (int k = 0; k < 8; ++k) { out8_host[k] = 0; for (int b = 0; b < 4096; ++b) out8_host[k] += h[b * 8 + k]; }
  return DGB_OK;
}

int dgb_disc_expand_maps(const dgb_disc* d, int64_t* vm, int64_t* vp, void* stream) {
  if (!d) return fail(DGB_ERR_INVALID, "null handle");
  const long long n = d->dev.E * d->Nf * d->Nfp;
  if (n == 0) return DGB_OK;
  k_expand_conn<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      d->conn, d->tables, d->dev.E, d->Np, d->Nf, d->Nfp, (long long*)vm, (long long*)vp);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

static int check_ghost(const dgb_disc* d, const void* ghost) {
  if (!d) return fail(DGB_ERR_INVALID, "null handle");
  if (d->dev.G > 0 && !ghost) return fail(DGB_ERR_INVALID, "discretisation has ghost elements but no ghost array was given");
  return DGB_OK;
}

int dgb_euler_rhs(const dgb_disc* d, const double* q, const double* ghost, double* rhs, const double* qfar,
                  const double* phys, void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return dispatch_rhs(d, false, q, nullptr, ghost, nullptr, ep, ph, (cudaStream_t)stream);
}

int dgb_euler_rhs_range(const dgb_disc* d, const double* q, const double* ghost, double* rhs, const double* qfar,
                        const double* phys, int64_t ebegin, int64_t eend, void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  if (ebegin < 0 || eend > d->dev.E || ebegin > eend) return fail(DGB_ERR_INVALID, "element range outside [0, E]");
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return dispatch_rhs(d, false, q, nullptr, ghost, nullptr, ep, ph, (cudaStream_t)stream, ebegin, eend);
}

int dgb_ns_grad(const dgb_disc* d, const double* q, const double* ghost, double* gradq, const double* qfar,
                void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, nullptr);
  return dispatch_grad(d, q, ghost, gradq, ph, (cudaStream_t)stream);
}

int dgb_ns_rhs(const dgb_disc* d, const double* q, const double* gradq, const double* ghost, const double* gghost,
               double* rhs, const double* qfar, const double* phys, void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  if ((rc = check_ghost(d, gghost))) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
  dgb::Epilogue ep{nullptr, rhs, nullptr, nullptr, 0.0, 1.0, 0.0, 0.0};
  return dispatch_rhs(d, true, q, gradq, ghost, gghost, ep, ph, (cudaStream_t)stream);
}

static int make_epilogue(dgb::Epilogue& ep, const double* q, const double* x1, double* out1, const double* x2,
                         double* out2, const double* rk) {
  if (!out1 || !rk) return fail(DGB_ERR_INVALID, "out1 and rk are required");
  if (out1 == q || (out2 && out2 == q) || (x2 && out1 == x2))
    return fail(DGB_ERR_INVALID, "RK outputs must not alias the stage input q (neighbours still read it)");
  if (out2 && !x2) return fail(DGB_ERR_INVALID, "out2 needs x2");
  // the epilogue loads and stores node pairs (double2) when Np is even
  if ((((uintptr_t)x1) | ((uintptr_t)out1) | ((uintptr_t)x2) | ((uintptr_t)out2)) & 15)
    return fail(DGB_ERR_INVALID, "RK operands and outputs must be 16-byte aligned");
  ep = dgb::Epilogue{x1, out1, x2, out2, rk[0], rk[1], rk[2], rk[3]};
  return DGB_OK;
}

int dgb_euler_rhs_rk(const dgb_disc* d, const double* q, const double* ghost, const double* x1, double* out1,
                     const double* x2, double* out2, const double* rk, const double* qfar, const double* phys,
                     void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
  dgb::Epilogue ep; if ((rc = make_epilogue(ep, q, x1, out1, x2, out2, rk))) return rc;
  return dispatch_rhs(d, false, q, nullptr, ghost, nullptr, ep, ph, (cudaStream_t)stream);
}

int dgb_ns_rhs_rk(const dgb_disc* d, const double* q, const double* gradq, const double* ghost,
                  const double* gghost, const double* x1, double* out1, const double* x2, double* out2,
                  const double* rk, const double* qfar, const double* phys, void* stream) {
  int rc = check_ghost(d, ghost); if (rc) return rc;
  if ((rc = check_ghost(d, gghost))) return rc;
  dgb::Phys ph; make_phys(ph, d->dim + 2, qfar, phys);
  dgb::Epilogue ep; if ((rc = make_epilogue(ep, q, x1, out1, x2, out2, rk))) return rc;
  return dispatch_rhs(d, true, q, gradq, ghost, gghost, ep, ph, (cudaStream_t)stream);
}

int dgb_pack_elements(double* dst, const double* src, const int64_t* elems, int64_t ncomp, int64_t nsrc,
                      int64_t nsel, int64_t ndofs, void* stream) {
  const long long total = ncomp * nsel * ndofs;
  if (total == 0) return DGB_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pack_elements<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst, src, (const long long*)elems, ncomp,
                                                                       nsrc, nsel, ndofs);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

int dgb_pack_elements_to(double* dst, int64_t ndst_elems, int64_t dst_slot0, const double* src, const int64_t* elems,
                         int64_t ncomp, int64_t nsrc, int64_t nsel, int64_t ndofs, void* stream) {
  const long long total = ncomp * nsel * ndofs;
  if (total == 0) return DGB_OK;
  if (dst_slot0 < 0 || dst_slot0 + nsel > ndst_elems) return fail(DGB_ERR_OUT_OF_BOUNDS, "halo slots outside the ghost array");
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pack_elements_to<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst, ndst_elems, dst_slot0, src,
                                                                          (const long long*)elems, ncomp, nsrc, nsel, ndofs);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

int dgb_ipc_alloc(void** dev, size_t bytes, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  DGB_CUDA(cudaMalloc(dev, bytes ? bytes : 8));
  DGB_CUDA(cudaMemset(*dev, 0, bytes ? bytes : 8));
  // the zero fill must have HAPPENED before a neighbour can map the array and store into it (cudaMemset
  // is asynchronous and would queue behind this rank's pending kernels, wiping a flag set meanwhile)
  DGB_CUDA(cudaDeviceSynchronize());
  DGB_CUDA(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle64, *dev));
  return DGB_OK;
}

int dgb_ipc_open(void** dev, const void* handle64) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  DGB_CUDA(cudaIpcOpenMemHandle(dev, h, cudaIpcMemLazyEnablePeerAccess));
  return DGB_OK;
}

int dgb_ipc_close(void* dev) { DGB_CUDA(cudaIpcCloseMemHandle(dev)); return DGB_OK; }

int dgb_flag_signal(uint64_t* flag_dev, uint64_t value, void* stream) {
  k_flag_signal<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long*)flag_dev, (unsigned long long)value);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

int dgb_flag_wait(const uint64_t* flag_dev, uint64_t value, void* stream) {
  k_flag_wait<<<1, 1, 0, (cudaStream_t)stream>>>((const unsigned long long*)flag_dev, (unsigned long long)value);
  DGB_CUDA(cudaGetLastError());
  return DGB_OK;
}

}  // extern "C"
