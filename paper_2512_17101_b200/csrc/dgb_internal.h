// Internals shared by the translation units of libdgb200.so (not part of the C ABI).
#pragma once
#include "../../include/dgb200.h"
#include "dgb_kernels.cuh"

#include <string>

#define DGB_HIDDEN __attribute__((visibility("hidden")))   // shared between translation units, not exported

int dgb_fail(int code, const std::string& msg);   // records the message for dgb_last_error()
int dgb_num_sms();                                // SMs of the CURRENT device
int dgb_grid_sms();                               // SMs a persistent kernel may occupy: dgb_num_sms() minus the reserve (dgb_set_sm_reserve)

// "done once" flags of the launch configuration (cudaFuncSetAttribute) are per DEVICE, not per process
struct DgbPerDevice {
  bool done[64] = {};
  bool& operator()() { int dev = 0; cudaGetDevice(&dev); return done[dev & 63]; }
};

#define DGB_CUDA(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return dgb_fail(DGB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));        \
  } while (0)

struct dgb_disc {
  int dim = 0, order = 0, Np = 0, Nf = 0, Nfp = 0, nperm = 0;
  dgb::DiscDev dev{};
  double *Wv = nullptr, *Wl = nullptr, *Wq = nullptr, *Wf = nullptr, *Wv2 = nullptr;
  long long* conn = nullptr;
  unsigned* gidx = nullptr;                 // 32-bit gather map (DiscDev::gidx)
  long long* timing = nullptr;
  unsigned long long* counters = nullptr;   // work counters: [0] gradient / flux pass, [1] divergence pass
  int* tables = nullptr;
  const int64_t* bc_kind = nullptr;
  double *sj = nullptr, *rj = nullptr;      // flux arrangement: face Jacobians (E, Nf), 1/J (E)
};

// dgb_nsflux.cu
int dgb_disc_free_jacobian(dgb_disc* d);
// single-pass Euler kernel of the flux-arrangement family (k_euler4); eend < 0 = all elements
int dgb_launch_euler4(const dgb_disc* d, const double* q, const double* ghost, const dgb::Epilogue& ep,
                      const dgb::Phys& ph, long long ebeg, long long eend, cudaStream_t st);
