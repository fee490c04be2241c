// FP64 peak microbenchmarks for B200 (sm_100a): decides DMMA-vs-DFMA for the DG
// contraction kernels.  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// 1. register-only DFMA, 16 independent chains per thread
__global__ void __launch_bounds__(256) k_dfma_reg(double* out, int iters, double b, double c) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 2. register-only DMMA m8n8k4, NACC independent accumulator tiles per warp
template <int NACC>
__global__ void __launch_bounds__(256) k_dmma_reg(double* out, int iters, double a, double b) {
  double c0[NACC], c1[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c0[i] = threadIdx.x * 1e-3 + i; c1[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma884(c0[i], c1[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3. matvec, thread per column, W in __constant__ memory, K=100, 20 outputs
__constant__ double cW[100 * 20];   // [k][i]
__global__ void __launch_bounds__(256) k_dfma_const(double* out, const double* __restrict__ xin, int iters) {
  __shared__ double xs[20][256];  // [k%20][col]  (256 cols)
  for (int k = 0; k < 20; ++k) xs[k][threadIdx.x] = xin[(k * 256 + threadIdx.x) % 4096];
  __syncthreads();
  double tot = 0;
  for (int it = 0; it < iters; ++it) {
    double acc[20];
#pragma unroll
    for (int i = 0; i < 20; ++i) acc[i] = 0;
#pragma unroll
    for (int k = 0; k < 100; ++k) {
      double x = xs[k % 20][threadIdx.x];
#pragma unroll
      for (int i = 0; i < 20; ++i) acc[i] = fma(cW[k * 20 + i], x, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < 20; ++i) tot += acc[i];
    xs[it % 20][threadIdx.x] = tot * 1e-30;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

// 4. matvec, thread handles NC columns, W from smem broadcast (LDS.128), K=100, 20 outputs
template <int NC>
__global__ void __launch_bounds__(256) k_dfma_smem(double* out, const double* __restrict__ win,
                                                    const double* __restrict__ xin, int iters) {
  __shared__ __align__(16) double ws[100 * 20];        // [k][i]
  __shared__ double xs[10][256];                       // [k%10][thread]
  for (int i = threadIdx.x; i < 2000; i += 256) ws[i] = win[i];
  for (int k = 0; k < 10; ++k) xs[k][threadIdx.x] = xin[(k * 256 + threadIdx.x) % 4096];
  __syncthreads();
  double tot = 0;
  for (int it = 0; it < iters; ++it) {
    double acc[NC][20];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < 20; ++i) acc[c][i] = 0;
#pragma unroll 4
    for (int k = 0; k < 100; ++k) {
      double x[NC];
      x[0] = xs[k % 10][threadIdx.x];
      if (NC > 1) x[1] = xs[(k + 3) % 10][threadIdx.x];
      const double2* wr = reinterpret_cast<const double2*>(&ws[k * 20]);
#pragma unroll
      for (int i2 = 0; i2 < 10; ++i2) {
        double2 w = wr[i2];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          acc[c][2 * i2] = fma(w.x, x[c], acc[c][2 * i2]);
          acc[c][2 * i2 + 1] = fma(w.y, x[c], acc[c][2 * i2 + 1]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < 20; ++i) tot += acc[c][i];
    xs[it % 10][threadIdx.x] = tot * 1e-30;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

// 5. DMMA matvec from smem: out[col][i] = sum_k W[i][k] X[col][k]; per warp NT column tiles (8 cols each),
//    3 i-tiles (24 rows, 20 useful), K=100 (25 k-steps).  X_s[col][XS] row stride XS doubles.
template <int NT>
__global__ void __launch_bounds__(256) k_dmma_smem(double* out, const double* __restrict__ win,
                                                    const double* __restrict__ xin, int iters) {
  constexpr int KK = 100, XS = 100;           // X stride in doubles
  constexpr int WS = 100;                     // W row stride
  extern __shared__ __align__(16) double sm[];
  double* ws = sm;                            // [24][WS]
  double* xs = sm + 24 * WS;                  // [8 warps * NT * 8 cols][XS]
  const int ncols = 8 * NT * 8;
  for (int i = threadIdx.x; i < 24 * WS; i += 256) ws[i] = (i < 20 * WS) ? win[i % 2000] : 0.0;
  for (int i = threadIdx.x; i < ncols * XS; i += 256) xs[i] = xin[i % 4096];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  double tot = 0;
  for (int it = 0; it < iters; ++it) {
    double c0[3][NT], c1[3][NT];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) { c0[m][n] = 0; c1[m][n] = 0; }
#pragma unroll 5
    for (int ks = 0; ks < KK / 4; ++ks) {
      double a[3], b[NT];
#pragma unroll
      for (int m = 0; m < 3; ++m) a[m] = ws[(m * 8 + r) * WS + ks * 4 + q];
#pragma unroll
      for (int n = 0; n < NT; ++n) b[n] = xs[((warp * NT + n) * 8 + r) * XS + ks * 4 + q];
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma884(c0[m][n], c1[m][n], a[m], b[n]);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) tot += c0[m][n] + c1[m][n];
    xs[(warp * NT * 8 + r) * XS + (it % 25) * 4 + q] = tot * 1e-30;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

// 7. concurrent DMMA + DFMA: even warps run DMMA chains, odd warps DFMA chains (are the pipes shared?)
__global__ void __launch_bounds__(256) k_mixed(double* out, int iters_mma, int iters_fma, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  } else {
    double c0[8], c1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c0[i] = threadIdx.x * 1e-3 + i; c1[i] = i; }
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma884(c0[i], c1[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c0[i] + c1[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 6. HBM copy (double2 grid-stride) for a local bandwidth reference
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename F>
static double time_ms(F f, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  int sustained = argc > 1 ? atoi(argv[1]) : 0;   // seconds of sustained DFMA/DMMA to sample clocks
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  const int grid = p.multiProcessorCount * 8, block = 256;
  double *out, *win, *xin;
  CK(cudaMalloc(&out, sizeof(double) * grid * block));
  CK(cudaMalloc(&win, sizeof(double) * 4096)); CK(cudaMalloc(&xin, sizeof(double) * 4096));
  double h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 1.0 / (1 + i % 97);
  CK(cudaMemcpy(win, h, sizeof(h), cudaMemcpyHostToDevice)); CK(cudaMemcpy(xin, h, sizeof(h), cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(cW, h, sizeof(double) * 2000));
  const double nthreads = (double)grid * block;

  { int iters = 20000; double ms = time_ms([&] { k_dfma_reg<<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5);
    printf("dfma_reg        : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads * iters * 16 * 2 / ms * 1e-9); }
  { int iters = 20000; double ms = time_ms([&] { k_dmma_reg<4><<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5);
    printf("dmma_reg<4>     : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads / 32 * iters * 4 * 512.0 / ms * 1e-9); }
  { int iters = 20000; double ms = time_ms([&] { k_dmma_reg<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5);
    printf("dmma_reg<8>     : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads / 32 * iters * 8 * 512.0 / ms * 1e-9); }
  { int iters = 20000; double ms = time_ms([&] { k_dmma_reg<16><<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5);
    printf("dmma_reg<16>    : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads / 32 * iters * 16 * 512.0 / ms * 1e-9); }
  { int iters = 200; double ms = time_ms([&] { k_dfma_const<<<grid, block>>>(out, xin, iters); }, 5);
    printf("dfma_const K100 : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads * iters * 2000.0 * 2 / ms * 1e-9); }
  { int iters = 200; double ms = time_ms([&] { k_dfma_smem<1><<<grid, block>>>(out, win, xin, iters); }, 5);
    printf("dfma_smem<1col> : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads * iters * 2000.0 * 2 / ms * 1e-9); }
  { int iters = 200; double ms = time_ms([&] { k_dfma_smem<2><<<grid, block>>>(out, win, xin, iters); }, 5);
    printf("dfma_smem<2col> : %8.3f ms  %7.2f TFLOP/s\n", ms, nthreads * iters * 4000.0 * 2 / ms * 1e-9); }
  {
    int iters = 400; constexpr int NT = 2; size_t smem = sizeof(double) * (24 * 100 + 8 * NT * 8 * 100);
    CK(cudaFuncSetAttribute(k_dmma_smem<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    double ms = time_ms([&] { k_dmma_smem<NT><<<p.multiProcessorCount * 2, block, smem>>>(out, win, xin, iters); }, 5);
    double useful = (double)p.multiProcessorCount * 2 * 8 * NT * 8 * iters * 2000.0 * 2;
    printf("dmma_smem<NT=2> : %8.3f ms  %7.2f TFLOP/s useful (x1.2 issued)\n", ms, useful / ms * 1e-9); }
  {
    int iters = 400; constexpr int NT = 4; size_t smem = sizeof(double) * (24 * 100 + 8 * NT * 8 * 100);
    CK(cudaFuncSetAttribute(k_dmma_smem<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    double ms = time_ms([&] { k_dmma_smem<NT><<<p.multiProcessorCount, block, smem>>>(out, win, xin, iters); }, 5);
    double useful = (double)p.multiProcessorCount * 8 * NT * 8 * iters * 2000.0 * 2;
    printf("dmma_smem<NT=4> : %8.3f ms  %7.2f TFLOP/s useful (x1.2 issued)\n", ms, useful / ms * 1e-9); }
  {
    // each alone (half the warps idle), then together
    int im = 20000, ifm = 20000;
    double t_m = time_ms([&] { k_mixed<<<grid, block>>>(out, im, 0, 1.0000001, 1e-9); }, 5);
    double t_f = time_ms([&] { k_mixed<<<grid, block>>>(out, 0, ifm, 1.0000001, 1e-9); }, 5);
    double t_b = time_ms([&] { k_mixed<<<grid, block>>>(out, im, ifm, 1.0000001, 1e-9); }, 5);
    double fl_m = nthreads / 2 / 32 * im * 8 * 512.0, fl_f = nthreads / 2 * ifm * 32.0;
    printf("mixed: dmma alone %8.3f ms (%6.2f TF)  dfma alone %8.3f ms (%6.2f TF)  together %8.3f ms (%6.2f TF total)\n",
           t_m, fl_m / t_m * 1e-9, t_f, fl_f / t_f * 1e-9, t_b, (fl_m + fl_f) / t_b * 1e-9);
  }
  {
    size_t n = (size_t)1 << 27;  // 2 GiB each
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); CK(cudaMemset(a, 1, n * 16));
    double ms = time_ms([&] { k_copy<<<p.multiProcessorCount * 16, 512>>>(a, b, n); }, 5);
    printf("copy 2GiB       : %8.3f ms  %7.1f GB/s (r+w)\n", ms, 2.0 * n * 16 / ms * 1e-6);
    double ms2 = time_ms([&] { cudaMemcpyAsync(b, a, n * 16, cudaMemcpyDeviceToDevice); }, 5);
    printf("cudaMemcpy D2D  : %8.3f ms  %7.1f GB/s (r+w)\n", ms2, 2.0 * n * 16 / ms2 * 1e-6);
    cudaFree(a); cudaFree(b);
  }
  if (sustained > 0) {
    // sustained loops so nvidia-smi sampling sees clocks under FP64 load
    int iters = 20000;
    double t = 0; int n = 0;
    while (t < sustained * 1000.0) { double ms = time_ms([&] { k_dfma_reg<<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5); t += ms * 6; ++n;
      if (n % 20 == 0) printf("sustained dfma_reg : %7.2f TFLOP/s\n", nthreads * iters * 32 / ms * 1e-9); }
    t = 0; n = 0;
    while (t < sustained * 1000.0) { double ms = time_ms([&] { k_dmma_reg<8><<<grid, block>>>(out, iters, 1.0000001, 1e-9); }, 5); t += ms * 6; ++n;
      if (n % 20 == 0) printf("sustained dmma_reg8: %7.2f TFLOP/s\n", nthreads / 32 * iters * 8 * 512.0 / ms * 1e-9); }
  }
  return 0;
}
