// Generic device array ops behind the array-context namespace (frontend.py:257-302): elementwise
// with trailing-aligned broadcast, where, strided copy, gather, einsum.  These are glue for code
// outside the fused DG functions (RK arithmetic, diagnostics); they are bandwidth-bound
// grid-stride kernels, not the hot path.
#include "../../include/dgb200.h"

#include <cuda_runtime.h>
#include <string>

int dgb_fail(int code, const std::string& msg);   // dgb200.cu: records the message for dgb_last_error()

namespace {

struct Dims {
  int rank;
  int ma, mb, mc;          // per operand: 0 = general strides, 1 = dense (offset == flat index), 2 = scalar (offset 0)
  long long ext[8];
  long long sa[8], sb[8], sc[8];
};

__device__ __forceinline__ double ld_f64(const void* p, int dt, long long off) {
  switch (dt) {
    case DGB_F64: return static_cast<const double*>(p)[off];
    case DGB_I64: return (double)static_cast<const long long*>(p)[off];
    default: return (double)static_cast<const unsigned char*>(p)[off];
  }
}
__device__ __forceinline__ long long ld_i64(const void* p, int dt, long long off) {
  switch (dt) {
    case DGB_F64: return (long long)static_cast<const double*>(p)[off];
    case DGB_I64: return static_cast<const long long*>(p)[off];
    default: return (long long)static_cast<const unsigned char*>(p)[off];
  }
}
__device__ __forceinline__ void st_any(void* p, int dt, long long off, double fv, long long iv, bool is_float) {
  switch (dt) {
    case DGB_F64: static_cast<double*>(p)[off] = is_float ? fv : (double)iv; break;
    case DGB_I64: static_cast<long long*>(p)[off] = is_float ? (long long)fv : iv; break;
    default: static_cast<unsigned char*>(p)[off] = is_float ? (fv != 0.0) : (iv != 0); break;
  }
}

__device__ __forceinline__ void offsets(const Dims& d, long long n, long long& oa, long long& ob, long long& oc) {
  // most elementwise ops of an array program combine same-shape dense arrays and scalars: no index decoding
  if (d.ma && d.mb && d.mc) {
    oa = d.ma == 1 ? n : 0; ob = d.mb == 1 ? n : 0; oc = d.mc == 1 ? n : 0;
    return;
  }
  const long long n0 = n;
  oa = ob = oc = 0;
#pragma unroll 1
  for (int k = d.rank - 1; k >= 0; --k) {
    const long long i = n % d.ext[k];
    n /= d.ext[k];
    oa += i * d.sa[k]; ob += i * d.sb[k]; oc += i * d.sc[k];
  }
  if (d.ma) oa = d.ma == 1 ? n0 : 0;
  if (d.mb) ob = d.mb == 1 ? n0 : 0;
  if (d.mc) oc = d.mc == 1 ? n0 : 0;
}

__device__ __forceinline__ long long floordiv_i(long long a, long long b) {
  if (b == 0) return 0;   // numpy: 0 with a warning
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

__global__ void k_binary(int op, void* out, int odt, const void* a, int adt, const void* b, int bdt, Dims d,
                         long long total, bool fcomp) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    long long oa, ob, oc;
    offsets(d, n, oa, ob, oc);
    double fr = 0.0; long long ir = 0; bool res_float = fcomp;
    if (fcomp) {
      const double x = ld_f64(a, adt, oa), y = ld_f64(b, bdt, ob);
      switch (op) {
        case DGB_ADD: fr = x + y; break;
        case DGB_SUB: fr = x - y; break;
        case DGB_MUL: fr = x * y; break;
        case DGB_TRUEDIV: fr = x / y; break;
        case DGB_FLOORDIV: fr = floor(x / y); break;
        case DGB_MOD: { fr = fmod(x, y); if (fr != 0.0 && ((fr < 0) != (y < 0))) fr += y; } break;
        case DGB_POW: fr = pow(x, y); break;
        case DGB_MIN: fr = (x != x || y != y) ? (x + y) : fmin(x, y); break;
        case DGB_MAX: fr = (x != x || y != y) ? (x + y) : fmax(x, y); break;
        case DGB_LT: ir = x < y; res_float = false; break;
        case DGB_LE: ir = x <= y; res_float = false; break;
        case DGB_GT: ir = x > y; res_float = false; break;
        case DGB_GE: ir = x >= y; res_float = false; break;
        case DGB_EQ: ir = x == y; res_float = false; break;
        default: ir = x != y; res_float = false; break;
      }
    } else {
      const long long x = ld_i64(a, adt, oa), y = ld_i64(b, bdt, ob);
      switch (op) {
        case DGB_ADD: ir = x + y; break;
        case DGB_SUB: ir = x - y; break;
        case DGB_MUL: ir = x * y; break;
        case DGB_TRUEDIV: fr = (double)x / (double)y; res_float = true; break;
        case DGB_FLOORDIV: ir = floordiv_i(x, y); break;
        case DGB_MOD: ir = y == 0 ? 0 : x - floordiv_i(x, y) * y; break;
        case DGB_POW: { long long r = 1, bb = x, ee = y; if (ee < 0) { r = 0; } else { while (ee) { if (ee & 1) r *= bb; bb *= bb; ee >>= 1; } } ir = r; } break;
        case DGB_MIN: ir = x < y ? x : y; break;
        case DGB_MAX: ir = x > y ? x : y; break;
        case DGB_LT: ir = x < y; break;
        case DGB_LE: ir = x <= y; break;
        case DGB_GT: ir = x > y; break;
        case DGB_GE: ir = x >= y; break;
        case DGB_EQ: ir = x == y; break;
        default: ir = x != y; break;
      }
    }
    st_any(out, odt, n, fr, ir, res_float);
  }
}

__global__ void k_unary(int op, void* out, int odt, const void* a, int adt, long long total) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    if (odt == DGB_F64) {
      const double x = ld_f64(a, adt, n);
      double r;
      switch (op) {
        case DGB_NEG: r = -x; break;
        case DGB_ABS: r = fabs(x); break;
        case DGB_SQRT: r = sqrt(x); break;
        case DGB_EXP: r = exp(x); break;
        default: r = log(x); break;
      }
      static_cast<double*>(out)[n] = r;
    } else {
      const long long x = ld_i64(a, adt, n);
      st_any(out, odt, n, 0.0, op == DGB_NEG ? -x : (x < 0 ? -x : x), false);
    }
  }
}

__global__ void k_where(void* out, int odt, const void* c, int cdt, const void* a, int adt, const void* b, int bdt,
                        Dims d, long long total) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    long long oa, ob, oc;
    offsets(d, n, oa, ob, oc);
    const bool cond = cdt == DGB_F64 ? (static_cast<const double*>(c)[oc] != 0.0) : (ld_i64(c, cdt, oc) != 0);
    if (odt == DGB_F64) static_cast<double*>(out)[n] = cond ? ld_f64(a, adt, oa) : ld_f64(b, bdt, ob);
    else st_any(out, odt, n, 0.0, cond ? ld_i64(a, adt, oa) : ld_i64(b, bdt, ob), false);
  }
}

__global__ void k_copy_strided(void* out, int odt, const void* a, int adt, Dims d, long long total) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    long long oa, ob, oc;
    offsets(d, n, oa, ob, oc);
    if (odt == DGB_F64) static_cast<double*>(out)[n] = ld_f64(a, adt, oa);
    else st_any(out, odt, n, 0.0, ld_i64(a, adt, oa), false);
  }
}

__global__ void k_copy_scatter(void* out, int odt, const void* a, int adt, Dims d, long long total) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    long long oa, ob, oc;
    offsets(d, n, oa, ob, oc);   // sb carries the output strides
    if (odt == DGB_F64) static_cast<double*>(out)[ob] = ld_f64(a, adt, oa);
    else st_any(out, odt, ob, 0.0, ld_i64(a, adt, oa), false);
  }
}

template <typename T>
__global__ void k_take(T* __restrict__ out, const T* __restrict__ a, const long long* __restrict__ idx,
                       long long outer, long long extent, long long inner, long long nidx, int* err) {
  const long long total = outer * nidx * inner;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < total;
       n += (long long)gridDim.x * blockDim.x) {
    const long long i = n % inner, ok = n / inner;
    const long long k = ok % nidx, o = ok / nidx;
    const long long src = idx[k];
    if (src < 0 || src >= extent) { *err = 1; continue; }
    out[n] = a[(o * extent + src) * inner + i];
  }
}

struct EinsumDesc {
  int nops, nout, nletters;
  long long ext[8];
  long long stride[3][8];
};

__global__ void k_einsum(double* __restrict__ out, const double* a, const double* b, const double* c, EinsumDesc d,
                         long long nout_total, long long nred_total) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nout_total;
       n += (long long)gridDim.x * blockDim.x) {
    long long o0 = 0, o1 = 0, o2 = 0, rem = n;
    for (int k = d.nout - 1; k >= 0; --k) {
      const long long i = rem % d.ext[k]; rem /= d.ext[k];
      o0 += i * d.stride[0][k]; o1 += i * d.stride[1][k]; o2 += i * d.stride[2][k];
    }
    double acc = 0.0;
    // ascending, outer-letter-first accumulation (expr.py:344-364).  The reduced letters are walked
    // with an odometer (last letter fastest) and incremental offsets -- the same order of terms as
    // decoding r by division, without two 64-bit divisions per letter and term.
    int idx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) idx[k] = 0;
    long long p0 = o0, p1 = o1, p2 = o2;
    for (long long r = 0; r < nred_total; ++r) {
      double v = a[p0];
      if (d.nops > 1) v *= b[p1];
      if (d.nops > 2) v *= c[p2];
      acc += v;
      bool carry = true;
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        if (carry && k >= d.nout && k < d.nletters) {
          ++idx[k];
          p0 += d.stride[0][k]; p1 += d.stride[1][k]; p2 += d.stride[2][k];
          if (idx[k] < d.ext[k]) {
            carry = false;
          } else {
            p0 -= d.ext[k] * d.stride[0][k]; p1 -= d.ext[k] * d.stride[1][k]; p2 -= d.ext[k] * d.stride[2][k];
            idx[k] = 0;
          }
        }
      }
    }
    out[n] = acc;
  }
}

// Few outputs, long reductions (norms, conservation sums: actx.np.sum over 1e8 values): the reduction range
// of every output is cut into segments of kEinsumSeg consecutive terms, one thread per (output, segment)
// sums its segment in the order above, and a second kernel adds the partial sums of an output in
// ascending segment order.  Fixed segment size and fixed order: deterministic, independent of the grid;
// the rounding differs from the single sequential sum of the reference interpreter in the last bits.
constexpr long long kEinsumSeg = 4096;

__global__ void k_einsum_seg(double* __restrict__ part, const double* a, const double* b, const double* c, EinsumDesc d,
                             long long nout_total, long long nred_total, long long nseg) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nout_total * nseg;
       t += (long long)gridDim.x * blockDim.x) {
    const long long n = t / nseg, sg = t - n * nseg;
    long long p0 = 0, p1 = 0, p2 = 0, rem = n;
    for (int k = d.nout - 1; k >= 0; --k) {
      const long long i = rem % d.ext[k]; rem /= d.ext[k];
      p0 += i * d.stride[0][k]; p1 += i * d.stride[1][k]; p2 += i * d.stride[2][k];
    }
    const long long r0 = sg * kEinsumSeg, r1 = r0 + kEinsumSeg < nred_total ? r0 + kEinsumSeg : nred_total;
    int idx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) idx[k] = 0;
    rem = r0;                               // odometer position of the segment's first term
    for (int k = d.nletters - 1; k >= d.nout; --k) {
      const long long i = rem % d.ext[k]; rem /= d.ext[k];
      idx[k] = (int)i;
      p0 += i * d.stride[0][k]; p1 += i * d.stride[1][k]; p2 += i * d.stride[2][k];
    }
    double acc = 0.0;
    for (long long r = r0; r < r1; ++r) {
      double v = a[p0];
      if (d.nops > 1) v *= b[p1];
      if (d.nops > 2) v *= c[p2];
      acc += v;
      bool carry = true;
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        if (carry && k >= d.nout && k < d.nletters) {
          ++idx[k];
          p0 += d.stride[0][k]; p1 += d.stride[1][k]; p2 += d.stride[2][k];
          if (idx[k] < d.ext[k]) {
            carry = false;
          } else {
            p0 -= d.ext[k] * d.stride[0][k]; p1 -= d.ext[k] * d.stride[1][k]; p2 -= d.ext[k] * d.stride[2][k];
            idx[k] = 0;
          }
        }
      }
    }
    part[t] = acc;
  }
}

__global__ void k_einsum_fold(double* __restrict__ out, const double* __restrict__ part, long long nout_total, long long nseg) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < nout_total;
       n += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long sg = 0; sg < nseg; ++sg) acc += part[n * nseg + sg];
    out[n] = acc;
  }
}

// ---- fused elementwise programs (dgb_ew_program) -------------------------------------------------
// The effect of the reference's loop fusion + array contraction (ir_passes.py:189-284) for chains of
// elementwise operations: the context records such a chain as a small register program (one
// instruction per array operation, in the order the program issued them) and this kernel interprets
// it once per output element -- every leaf array is read once, every requested result written once,
// no intermediate array touches HBM.  Each instruction applies exactly the scalar code of
// k_binary / k_unary / k_where above (same conversions, same IEEE operations, nothing contracted across
// instructions), so results are bit-identical to the op-by-op kernels.
__device__ __forceinline__ double reg_f64(unsigned long long v, int dt) {
  return dt == DGB_F64 ? __longlong_as_double((long long)v) : (double)(long long)v;
}
__device__ __forceinline__ long long reg_i64(unsigned long long v, int dt) {
  return dt == DGB_F64 ? (long long)__longlong_as_double((long long)v) : (long long)v;
}
__device__ __forceinline__ unsigned long long reg_store(int odt, double fv, long long iv, bool is_float) {
  switch (odt) {
    case DGB_F64: return (unsigned long long)__double_as_longlong(is_float ? fv : (double)iv);
    case DGB_I64: return (unsigned long long)(is_float ? (long long)fv : iv);
    default: return (unsigned long long)(is_float ? (fv != 0.0) : (iv != 0));
  }
}

__global__ void __launch_bounds__(256) k_ew_program(dgb_ew_prog pg) {
  unsigned long long r[DGB_EW_MAX_REGS];
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < pg.total;
       n += (long long)gridDim.x * blockDim.x) {
    long long idx[8];
    if (pg.need_index) {
      long long rem = n;
#pragma unroll 1
      for (int k = pg.rank - 1; k >= 0; --k) { idx[k] = rem % pg.ext[k]; rem /= pg.ext[k]; }
    }
#pragma unroll 1
    for (int i = 0; i < pg.nins; ++i) {
      const dgb_ew_ins in = pg.ins[i];
      unsigned long long res;
      switch (in.kind) {
        case DGB_EW_LOAD: {
          const dgb_ew_leaf& lf = pg.leaf[in.a];
          long long off = 0;
          if (lf.mode == 1) off = n;
          else if (lf.mode == 0) {
#pragma unroll 1
            for (int k = 0; k < pg.rank; ++k) off += idx[k] * lf.stride[k];
          }
          switch (lf.dtype) {
            case DGB_F64: res = (unsigned long long)static_cast<const long long*>(lf.dev)[off]; break;
            case DGB_I64: res = (unsigned long long)static_cast<const long long*>(lf.dev)[off]; break;
            default: res = (unsigned long long)static_cast<const unsigned char*>(lf.dev)[off]; break;
          }
        } break;
        case DGB_EW_CONST: res = pg.consts[in.a]; break;
        case DGB_EW_BINARY: {
          double fr = 0.0; long long ir = 0; bool res_float = in.fcomp != 0;
          if (in.fcomp) {
            const double x = reg_f64(r[in.a], in.adt), y = reg_f64(r[in.b], in.bdt);
            switch (in.op) {
              case DGB_ADD: fr = x + y; break;
              case DGB_SUB: fr = x - y; break;
              case DGB_MUL: fr = x * y; break;
              case DGB_TRUEDIV: fr = x / y; break;
              case DGB_FLOORDIV: fr = floor(x / y); break;
              case DGB_MOD: { fr = fmod(x, y); if (fr != 0.0 && ((fr < 0) != (y < 0))) fr += y; } break;
              case DGB_POW: fr = pow(x, y); break;
              case DGB_MIN: fr = (x != x || y != y) ? (x + y) : fmin(x, y); break;
              case DGB_MAX: fr = (x != x || y != y) ? (x + y) : fmax(x, y); break;
              case DGB_LT: ir = x < y; res_float = false; break;
              case DGB_LE: ir = x <= y; res_float = false; break;
              case DGB_GT: ir = x > y; res_float = false; break;
              case DGB_GE: ir = x >= y; res_float = false; break;
              case DGB_EQ: ir = x == y; res_float = false; break;
              default: ir = x != y; res_float = false; break;
            }
          } else {
            const long long x = reg_i64(r[in.a], in.adt), y = reg_i64(r[in.b], in.bdt);
            switch (in.op) {
              case DGB_ADD: ir = x + y; break;
              case DGB_SUB: ir = x - y; break;
              case DGB_MUL: ir = x * y; break;
              case DGB_TRUEDIV: fr = (double)x / (double)y; res_float = true; break;
              case DGB_FLOORDIV: ir = floordiv_i(x, y); break;
              case DGB_MOD: ir = y == 0 ? 0 : x - floordiv_i(x, y) * y; break;
              case DGB_POW: { long long rr = 1, bb = x, ee = y; if (ee < 0) { rr = 0; } else { while (ee) { if (ee & 1) rr *= bb; bb *= bb; ee >>= 1; } } ir = rr; } break;
              case DGB_MIN: ir = x < y ? x : y; break;
              case DGB_MAX: ir = x > y ? x : y; break;
              case DGB_LT: ir = x < y; break;
              case DGB_LE: ir = x <= y; break;
              case DGB_GT: ir = x > y; break;
              case DGB_GE: ir = x >= y; break;
              case DGB_EQ: ir = x == y; break;
              default: ir = x != y; break;
            }
          }
          res = reg_store(in.odt, fr, ir, res_float);
        } break;
        case DGB_EW_UNARY: {
          if (in.odt == DGB_F64) {
            const double x = reg_f64(r[in.a], in.adt);
            double v;
            switch (in.op) {
              case DGB_NEG: v = -x; break;
              case DGB_ABS: v = fabs(x); break;
              case DGB_SQRT: v = sqrt(x); break;
              case DGB_EXP: v = exp(x); break;
              default: v = log(x); break;
            }
            res = (unsigned long long)__double_as_longlong(v);
          } else {
            const long long x = reg_i64(r[in.a], in.adt);
            res = reg_store(in.odt, 0.0, in.op == DGB_NEG ? -x : (x < 0 ? -x : x), false);
          }
        } break;
        default: {   // DGB_EW_WHERE: a = value if true, b = value if false, c = condition
          const bool cond = in.cdt == DGB_F64 ? (__longlong_as_double((long long)r[in.c]) != 0.0) : ((long long)r[in.c] != 0);
          if (in.odt == DGB_F64) res = (unsigned long long)__double_as_longlong(cond ? reg_f64(r[in.a], in.adt) : reg_f64(r[in.b], in.bdt));
          else res = reg_store(in.odt, 0.0, cond ? reg_i64(r[in.a], in.adt) : reg_i64(r[in.b], in.bdt), false);
        } break;
      }
      r[in.dst] = res;
    }
#pragma unroll 1
    for (int o = 0; o < pg.nouts; ++o) {
      const unsigned long long v = r[pg.out[o].reg];
      if (pg.out[o].dtype == DGB_BOOL) static_cast<unsigned char*>(pg.out[o].dev)[n] = (unsigned char)v;
      else static_cast<unsigned long long*>(pg.out[o].dev)[n] = v;
    }
  }
}

int grid_for(long long total) {
  long long b = (total + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

int fill_dims(Dims& d, int rank, const int64_t* shape, const int64_t* sa, const int64_t* sb, const int64_t* sc,
              long long* total) {
  if (rank < 0 || rank > 8) return DGB_ERR_INVALID;
  d.rank = rank;
  long long t = 1;
  for (int k = 0; k < 8; ++k) {
    d.ext[k] = k < rank ? shape[k] : 1;
    d.sa[k] = (k < rank && sa) ? sa[k] : 0;
    d.sb[k] = (k < rank && sb) ? sb[k] : 0;
    d.sc[k] = (k < rank && sc) ? sc[k] : 0;
    if (k < rank) t *= shape[k];
  }
  *total = t;
  // classify each operand: dense (strides of a row-major array of this shape; extent-1 axes are free),
  // scalar (all strides 0), or general
  auto mode = [&](const long long* st, bool present) -> int {
    if (!present) return 2;
    bool dense = true, scalar = true;
    long long run = 1;
    for (int k = rank - 1; k >= 0; --k) {
      if (d.ext[k] != 1) {
        if (st[k] != run) dense = false;
        if (st[k] != 0) scalar = false;
      }
      run *= d.ext[k];
    }
    return dense ? 1 : (scalar ? 2 : 0);
  };
  d.ma = mode(d.sa, sa != nullptr); d.mb = mode(d.sb, sb != nullptr); d.mc = mode(d.sc, sc != nullptr);
  return DGB_OK;
}

}  // namespace

#define DGB_CHECK_LAUNCH()                                                                                   \
  do { cudaError_t e_ = cudaGetLastError();                                                                  \
       if (e_ != cudaSuccess) return dgb_fail(DGB_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); } while (0)
#define DGB_BAD_DIMS() dgb_fail(DGB_ERR_INVALID, "rank outside [0, 8]")

extern "C" {

int dgb_ew_binary(int op, void* out, int odt, const void* a, int adt, const int64_t* sa, const void* b, int bdt,
                  const int64_t* sb, int rank, const int64_t* shape, void* stream) {
  Dims d; long long total;
  if (fill_dims(d, rank, shape, sa, sb, nullptr, &total)) return DGB_BAD_DIMS();
  if (total == 0) return DGB_OK;
  const bool fcomp = adt == DGB_F64 || bdt == DGB_F64;
  k_binary<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(op, out, odt, a, adt, b, bdt, d, total, fcomp);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_ew_unary(int op, void* out, int odt, const void* a, int adt, int64_t n, void* stream) {
  if (n == 0) return DGB_OK;
  k_unary<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(op, out, odt, a, adt, n);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_ew_where(void* out, int odt, const void* c, int cdt, const int64_t* sc, const void* a, int adt,
                 const int64_t* sa, const void* b, int bdt, const int64_t* sb, int rank, const int64_t* shape,
                 void* stream) {
  Dims d; long long total;
  if (fill_dims(d, rank, shape, sa, sb, sc, &total)) return DGB_BAD_DIMS();
  if (total == 0) return DGB_OK;
  k_where<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(out, odt, c, cdt, a, adt, b, bdt, d, total);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_copy_strided(void* out, int odt, const void* a, int adt, const int64_t* sa, int rank, const int64_t* shape,
                     void* stream) {
  Dims d; long long total;
  if (fill_dims(d, rank, shape, sa, nullptr, nullptr, &total)) return DGB_BAD_DIMS();
  if (total == 0) return DGB_OK;
  k_copy_strided<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(out, odt, a, adt, d, total);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_copy_scatter(void* out, int odt, const int64_t* so, const void* a, int adt, const int64_t* sa, int rank,
                     const int64_t* shape, void* stream) {
  Dims d; long long total;
  if (fill_dims(d, rank, shape, sa, so, nullptr, &total)) return DGB_BAD_DIMS();
  if (total == 0) return DGB_OK;
  k_copy_scatter<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(out, odt, a, adt, d, total);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_take(void* out, const void* a, int dtype, const int64_t* idx, int64_t outer, int64_t extent, int64_t inner,
             int64_t nidx, void* stream) {
  const long long total = outer * nidx * inner;
  if (total == 0) return DGB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* err = nullptr;
  if (cudaMalloc((void**)&err, sizeof(int)) != cudaSuccess) return dgb_fail(DGB_ERR_CUDA, "dgb_take: cudaMalloc of the error flag failed");
  cudaMemsetAsync(err, 0, sizeof(int), st);
  if (dtype == DGB_BOOL)
    k_take<unsigned char><<<grid_for(total), 256, 0, st>>>((unsigned char*)out, (const unsigned char*)a,
                                                           (const long long*)idx, outer, extent, inner, nidx, err);
  else
    k_take<long long><<<grid_for(total), 256, 0, st>>>((long long*)out, (const long long*)a, (const long long*)idx,
                                                       outer, extent, inner, nidx, err);
  int h = 0;
  cudaError_t ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  cudaFree(err);
  if (ce != cudaSuccess) return dgb_fail(DGB_ERR_CUDA, std::string("dgb_take: ") + cudaGetErrorString(ce));
  return h ? dgb_fail(DGB_ERR_OUT_OF_BOUNDS, "index array leaves [0, extent)") : DGB_OK;
}

int dgb_take_deferred(void* out, const void* a, int dtype, const int64_t* idx, int64_t outer, int64_t extent,
                      int64_t inner, int64_t nidx, int* err_dev, void* stream) {
  // same gather, but an out-of-range index only raises *err_dev (checked by the caller at its next
  // synchronisation point): no allocation, no host synchronisation, capturable in a CUDA graph
  const long long total = outer * nidx * inner;
  if (total == 0) return DGB_OK;
  if (!err_dev) return dgb_fail(DGB_ERR_INVALID, "dgb_take_deferred needs a device error flag");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == DGB_BOOL)
    k_take<unsigned char><<<grid_for(total), 256, 0, st>>>((unsigned char*)out, (const unsigned char*)a,
                                                           (const long long*)idx, outer, extent, inner, nidx, err_dev);
  else
    k_take<long long><<<grid_for(total), 256, 0, st>>>((long long*)out, (const long long*)a, (const long long*)idx,
                                                       outer, extent, inner, nidx, err_dev);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_einsum(double* out, int nops, const double* const* ops, const int64_t* op_strides, int nout, int nletters,
               const int64_t* ext, void* stream) {
  if (nops < 1 || nops > 3 || nletters > 8 || nout > nletters)
    return dgb_fail(DGB_ERR_INVALID, "dgb_einsum: 1-3 operands, at most 8 letters, nout <= nletters");
  EinsumDesc d; d.nops = nops; d.nout = nout; d.nletters = nletters;
  long long no = 1, nr = 1;
  for (int k = 0; k < 8; ++k) {
    d.ext[k] = k < nletters ? ext[k] : 1;
    for (int o = 0; o < 3; ++o) d.stride[o][k] = (o < nops && k < nletters) ? op_strides[o * nletters + k] : 0;
    if (k < nout) no *= d.ext[k]; else if (k < nletters) nr *= d.ext[k];
  }
  if (no == 0) return DGB_OK;
  if (nr >= 8 * kEinsumSeg && no <= 4096) {
    // long reductions into few outputs: segmented, fixed-order (see k_einsum_seg)
    const long long nseg = (nr + kEinsumSeg - 1) / kEinsumSeg;
    double* part = nullptr;
    if (cudaMallocAsync((void**)&part, sizeof(double) * (size_t)(no * nseg), (cudaStream_t)stream) != cudaSuccess)
      return dgb_fail(DGB_ERR_CUDA, "dgb_einsum: allocation of the partial sums failed");
    k_einsum_seg<<<grid_for(no * nseg), 256, 0, (cudaStream_t)stream>>>(part, ops[0], nops > 1 ? ops[1] : nullptr,
                                                                        nops > 2 ? ops[2] : nullptr, d, no, nr, nseg);
    k_einsum_fold<<<grid_for(no), 256, 0, (cudaStream_t)stream>>>(out, part, no, nseg);
    cudaFreeAsync(part, (cudaStream_t)stream);
    DGB_CHECK_LAUNCH();
    return DGB_OK;
  }
  k_einsum<<<grid_for(no), 256, 0, (cudaStream_t)stream>>>(out, ops[0], nops > 1 ? ops[1] : nullptr,
                                                           nops > 2 ? ops[2] : nullptr, d, no, nr);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

int dgb_ew_program(const dgb_ew_prog* prog, void* stream) {
  if (!prog) return dgb_fail(DGB_ERR_INVALID, "dgb_ew_program: null program");
  const dgb_ew_prog& p = *prog;
  if (p.nins < 1 || p.nins > DGB_EW_MAX_INS || p.nleaves < 0 || p.nleaves > DGB_EW_MAX_LEAVES || p.nouts < 1 ||
      p.nouts > DGB_EW_MAX_OUTS || p.rank < 0 || p.rank > 8)
    return dgb_fail(DGB_ERR_INVALID, "dgb_ew_program: program exceeds the instruction / leaf / output / rank limits");
  for (int i = 0; i < p.nins; ++i) {
    const dgb_ew_ins& in = p.ins[i];
    const bool regs_ok = in.dst < DGB_EW_MAX_REGS && (in.kind <= DGB_EW_CONST || in.a < DGB_EW_MAX_REGS) &&
                         (in.kind != DGB_EW_BINARY && in.kind != DGB_EW_WHERE || in.b < DGB_EW_MAX_REGS) &&
                         (in.kind != DGB_EW_WHERE || in.c < DGB_EW_MAX_REGS);
    if (in.kind > DGB_EW_WHERE || !regs_ok || (in.kind == DGB_EW_LOAD && in.a >= p.nleaves) ||
        (in.kind == DGB_EW_CONST && in.a >= DGB_EW_MAX_CONSTS))
      return dgb_fail(DGB_ERR_INVALID, "dgb_ew_program: malformed instruction " + std::to_string(i));
  }
  for (int o = 0; o < p.nouts; ++o)
    if (p.out[o].reg < 0 || p.out[o].reg >= DGB_EW_MAX_REGS || !p.out[o].dev)
      return dgb_fail(DGB_ERR_INVALID, "dgb_ew_program: bad output");
  if (p.total == 0) return DGB_OK;
  k_ew_program<<<grid_for(p.total), 256, 0, (cudaStream_t)stream>>>(p);
  DGB_CHECK_LAUNCH();
  return DGB_OK;
}

}  // extern "C"
