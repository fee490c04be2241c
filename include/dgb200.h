/*
 * dgb200.h -- C ABI of the B200-native DG right-hand-side path.
 *
 * This is the drop-in boundary.  The reference is a pure-Python package
 * and has no FFI of its own; what this library replaces is the *executor* behind the
 * reference's array context for the outlined DG functions and the array ops they are
 * written in.  Each entry point cites the reference interface it stands in for
 * (paths relative to /root/reference/pkg/src/laze/).  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - every function returns a dgb_status (0 = ok); dgb_last_error() gives the text.
 *     The Python shim maps codes to the reference's exception classes (errors.py:11-119).
 *   - all `dev` pointers are CUDA device pointers of the current device; `host` pointers
 *     are ordinary host memory.  No torch / framework types cross this boundary.
 *   - arrays are dense row-major (scalar_ir.py:147-151, backend.py:222-231), FP64 unless
 *     stated, index maps int64 (adfg.py:540-541).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream); all work
 *     is enqueued asynchronously on it.
 *   - inputs are never modified and never aliased by outputs (adfg.py:341-348 ownership).
 */
#ifndef DGB200_H
#define DGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DGB_OK = 0,
  DGB_ERR_CUDA = 1,            /* CUDA runtime failure                       -> LazeError              */
  DGB_ERR_INVALID = 2,         /* bad argument / unsupported (dim, order)    -> ShapeMismatch          */
  DGB_ERR_OUT_OF_BOUNDS = 3,   /* gather index outside [0, extent)           -> OutOfBoundsIndex       */
  DGB_ERR_BAD_MAP = 4,         /* index map is not a conforming face map     -> BindingMismatch        */
  DGB_ERR_DTYPE = 5            /* unsupported element type                   -> DTypeMismatch          */
} dgb_status;

/* element types, adfg.py:39-45 */
typedef enum { DGB_F64 = 0, DGB_I64 = 1, DGB_BOOL = 2 } dgb_dtype;

const char* dgb_last_error(void);
int dgb_version(void);

/* ---- device memory + transfers: ArrayContext.from_numpy / to_numpy (frontend.py:327-343) ---- */
int dgb_malloc(void** dev, size_t bytes);
int dgb_free(void* dev);
int dgb_host_alloc(void** host, size_t bytes);                 /* pinned host staging */
int dgb_host_free(void* host);
int dgb_memcpy_h2d(void* dev, const void* host, size_t bytes, void* stream);
int dgb_memcpy_d2h(void* host, const void* dev, size_t bytes, void* stream);
int dgb_memcpy_d2d(void* dst_dev, const void* src_dev, size_t bytes, void* stream);
int dgb_stream_sync(void* stream);

/* ---- discretisation handle ------------------------------------------------------------------
 * Uploads the reference matrices and binds the per-mesh device arrays that the outlined DG
 * functions receive as arguments.  The int64 face maps (`vmap_m`, `vmap_p`: flat indices into
 * u.reshape(E*Np), used through Indexing, adfg.py:502-560) are range-checked ONCE here
 * (backend.py:59-68 checks on every load) and compressed to (neighbour element, neighbour
 * face, vertex permutation, bc) per face; dgb_disc_expand_maps() regenerates the int64 maps
 * from the compressed form so that bit-exactness can be asserted.
 *
 *   Sw_host      (dim, Np, Np)      weak reference-derivative matrices
 *   lift_host    (Np, Nf*Nfp)
 *   face_nodes_host (Nf, Nfp) int64, face_perms_host (dim!, Nfp) int64
 *   drdx_dev     (dim, dim, E)   [r, x, e]
 *   normals_dev  (dim, E, Nf)
 *   fscale_dev   (E, Nf)
 *   vmap_m_dev, vmap_p_dev (E*Nf*Nfp) int64; entries of vmap_p in [E*Np, (E+G)*Np) address
 *                ghost elements (halo copies of remote elements, G may be 0)
 *   bc_kind_dev  (E, Nf) int64: 0 interior, 1 far-field, 2 wall
 * The device arrays must stay alive (and unchanged) for the life of the handle.
 */
typedef struct dgb_disc dgb_disc;

int dgb_disc_create(dgb_disc** out, int dim, int order, int64_t nelements, int64_t nghost,
                    const double* Sw_host, const double* lift_host,
                    const int64_t* face_nodes_host, const int64_t* face_perms_host,
                    const double* drdx_dev, const double* normals_dev, const double* fscale_dev,
                    const int64_t* vmap_m_dev, const int64_t* vmap_p_dev,
                    const int64_t* bc_kind_dev, void* stream);
int dgb_disc_destroy(dgb_disc* disc);
int dgb_disc_expand_maps(const dgb_disc* disc, int64_t* vmap_m_dev, int64_t* vmap_p_dev, void* stream);
/* debug: per-phase cycle counters summed over CTAs (filled only by -DDGB_PHASE_TIMING builds); resets them */
int dgb_debug_phase_cycles(const dgb_disc* disc, long long* out8_host);

/* ---- the outlined DG functions (operators.py; reference boundary: a Call to a
 *      FunctionDefinition, adfg.py:722-803, executed as a CallStep, backend.py:90-96) ----------
 *   q      (C, E, Np)          conserved state [rho, rho E, rho u...]
 *   ghost  (C, G, Np) or NULL  halo elements
 *   gradq  (dim, C, E, Np), gghost (dim, C, G, Np) or NULL
 *   qfar_host (C)  far-field state;  phys_host (4) = gamma, mu, kappa, R
 *   rhs    (C, E, Np)
 */
int dgb_euler_rhs(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* rhs_dev,
                  const double* qfar_host, const double* phys_host, void* stream);
int dgb_ns_grad(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* gradq_dev,
                const double* qfar_host, void* stream);
int dgb_ns_rhs(const dgb_disc* disc, const double* q_dev, const double* gradq_dev,
               const double* ghost_dev, const double* gghost_dev, double* rhs_dev,
               const double* qfar_host, const double* phys_host, void* stream);

/* Same right-hand sides with the Runge-Kutta stage update fused into the epilogue (north-star
 * item 3): instead of rhs, writes
 *     out1 = a1 * x1 + b1 * rhs      (x1 may equal q; out1 must not alias q or x2)
 *     out2 = a2 * x2 + b2 * rhs      (out2 may be NULL; out2 may alias x2)
 * all (C, E, Np).  rk = {a1, b1, a2, b2} on the host.
 */
int dgb_euler_rhs_rk(const dgb_disc* disc, const double* q_dev, const double* ghost_dev,
                     const double* x1_dev, double* out1_dev, const double* x2_dev, double* out2_dev,
                     const double* rk_host, const double* qfar_host, const double* phys_host, void* stream);
int dgb_ns_rhs_rk(const dgb_disc* disc, const double* q_dev, const double* gradq_dev,
                  const double* ghost_dev, const double* gghost_dev,
                  const double* x1_dev, double* out1_dev, const double* x2_dev, double* out2_dev,
                  const double* rk_host, const double* qfar_host, const double* phys_host, void* stream);

/* ---- Navier-Stokes in the flux arrangement (operators.py: dg_ns_flux + dg_ns_div; the default
 *      of NavierStokesOperator.rhs).  Same reference boundary as above (a Call to a
 *      FunctionDefinition, adfg.py:722-803).  dgb_disc_set_jacobian binds the volume Jacobian
 *      jac (E) the two functions take as an argument and derives the face Jacobians
 *      fscale*jac and 1/jac on the device; call it once per handle before dgb_ns_flux.
 *   T      ((dim+1)*C + 1, E, Np)   planes r*C + c (r < dim): sum_x jac*drdx[r,x] * (F_inv - F_visc)[x][c] with the BR1
 *                               gradient of pass 1 folded in; last plane: wave speed |u| + c
 *   Tghost ((dim+1)*C + 1, G, Np) or NULL: the same planes of the halo elements (already scaled by
 *                               the sender's Jacobian, so no remote geometry is needed)
 *   all device arrays 16-byte aligned.
 */
int dgb_disc_set_jacobian(dgb_disc* disc, const double* jac_dev, void* stream);
int dgb_ns_flux(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* T_dev,
                const double* qfar_host, const double* phys_host, void* stream);
int dgb_ns_div(const dgb_disc* disc, const double* q_dev, const double* T_dev,
               const double* ghost_dev, const double* Tghost_dev, double* rhs_dev,
               const double* qfar_host, const double* phys_host, void* stream);
int dgb_ns_div_rk(const dgb_disc* disc, const double* q_dev, const double* T_dev,
                  const double* ghost_dev, const double* Tghost_dev,
                  const double* x1_dev, double* out1_dev, const double* x2_dev, double* out2_dev,
                  const double* rk_host, const double* qfar_host, const double* phys_host, void* stream);

/* ---- element sub-ranges: the same three right-hand-side kernels restricted to the elements
 *      [ebegin, eend) of the mesh (outputs of other elements are not touched).  A partitioned
 *      mesh orders its elements [interior | adjacent to a partition boundary]; the interior range
 *      needs no halo data and runs while the exchange (Send / Receive, adfg.py:380-399,834-869) is
 *      in flight on another stream -- the overlap the reference lists as missing.
 */
int dgb_euler_rhs_range(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* rhs_dev,
                        const double* qfar_host, const double* phys_host,
                        int64_t ebegin, int64_t eend, void* stream);
int dgb_ns_flux_range(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* T_dev,
                      const double* qfar_host, const double* phys_host,
                      int64_t ebegin, int64_t eend, void* stream);
int dgb_ns_div_range(const dgb_disc* disc, const double* q_dev, const double* T_dev,
                     const double* ghost_dev, const double* Tghost_dev, double* rhs_dev,
                     const double* qfar_host, const double* phys_host,
                     int64_t ebegin, int64_t eend, void* stream);
/* dgb_ns_div_rk on a sub-range: the partitioned right-hand side with the RK stage update fused into the store of
 * pass 2 (north-star items 3 and 4 together; halo.py: HaloExchange.ns_rhs_rk); eend < 0 = all elements */
int dgb_ns_div_rk_range(const dgb_disc* disc, const double* q_dev, const double* T_dev,
                        const double* ghost_dev, const double* Tghost_dev,
                        const double* x1_dev, double* out1_dev, const double* x2_dev, double* out2_dev,
                        const double* rk_host, const double* qfar_host, const double* phys_host,
                        int64_t ebegin, int64_t eend, void* stream);

/* ---- multi-species reactive Navier-Stokes (BASELINE configs[4]): the outlined functions dg_ms_flux / dg_ms_div of
 *      multispecies.py (Call nodes of the reference: adfg.py:722-803; op families: IndexLambda with exp / truediv,
 *      /root/reference/pkg/src/laze/expr.py:265-289, Einsum adfg.py:563-608, Indexing :502-560) on the same fused
 *      kernels instantiated for C = dim + 2 + ns fields, ns = 2, 3 or 4 (DGB_ERR_INVALID otherwise).  q: (C, E, Np); T: ((dim+1)*C + 1, E, Np) plane groups as
 *      in dgb_ns_flux; transport_host = [mu, kappa, D]; mixture_host = [ns, R[ns], cv[ns], h0[ns], A, Ta,
 *      reactant, product]; boundary faces take qfar_host (C values) as exterior state; eend < 0 = all elements. ---- */
int dgb_ms_flux_range(const dgb_disc* disc, const double* q_dev, const double* ghost_dev, double* T_dev,
                      const double* qfar_host, const double* transport_host, const double* mixture_host,
                      int64_t ebegin, int64_t eend, void* stream);
int dgb_ms_div_range(const dgb_disc* disc, const double* q_dev, const double* T_dev,
                     const double* ghost_dev, const double* Tghost_dev, double* rhs_dev,
                     const double* qfar_host, const double* transport_host, const double* mixture_host,
                     int64_t ebegin, int64_t eend, void* stream);

/* the same with the RK stage update fused into the store (north-star item 3), like dgb_ns_div_rk */
int dgb_ms_div_rk(const dgb_disc* disc, const double* q_dev, const double* T_dev,
                  const double* ghost_dev, const double* Tghost_dev,
                  const double* x1_dev, double* out1_dev, const double* x2_dev, double* out2_dev, const double* rk_host,
                  const double* qfar_host, const double* transport_host, const double* mixture_host, void* stream);

/* ---- halo packing: element rows <-> contiguous message (Send / Receive payloads,
 *      adfg.py:380-399,834-869).  dst[c, i, :] = src[c, elems[i], :]                        ---- */
int dgb_pack_elements(double* dst_dev, const double* src_dev, const int64_t* elems_dev,
                      int64_t ncomp, int64_t nsrc_elems, int64_t nsel, int64_t ndofs, void* stream);

/* ---- peer-memory halo transport (optional alternative to NCCL send/recv for the messages of
 *      adfg.py:380-399,834-869): each rank allocates its ghost arrays with dgb_ipc_alloc and publishes the
 *      64-byte handle; a neighbour maps it (dgb_ipc_open) and its pack kernel stores the halo rows
 *      straight into it over NVLink -- pack and transfer are one kernel, no staging buffer, no
 *      communication kernel competing for SMs.  Ordering: stream-ordered flags in peer-mapped memory
 *      (signal = system-scope release after everything enqueued before it; wait holds the stream).   ---- */
int dgb_ipc_alloc(void** dev, size_t bytes, void* handle64_out);         /* zero-filled */
int dgb_ipc_open(void** dev, const void* handle64);
int dgb_ipc_close(void* dev);
int dgb_pack_elements_to(double* dst_dev, int64_t ndst_elems, int64_t dst_slot0, const double* src_dev,
                         const int64_t* elems_dev, int64_t ncomp, int64_t nsrc_elems, int64_t nsel,
                         int64_t ndofs, void* stream);
/* Leave `nsm` SMs free in every persistent kernel launched from now on (0 = use all).  halo.py sets it while a
 * halo batch is in flight on the communication stream, so that the transport's own kernels (NCCL send/recv)
 * start at once and the exchange overlaps the interior range -- the reference's executor has no overlap
 * (distpart.py:430-560 runs the batches back to back). */
int dgb_set_sm_reserve(int nsm);
int dgb_flag_signal(uint64_t* flag_dev, uint64_t value, void* stream);
int dgb_flag_wait(const uint64_t* flag_dev, uint64_t value, void* stream);

/* ---- generic array ops of the context (frontend.py:257-302), for glue outside the fused
 *      functions.  Shapes are given after broadcasting: `rank`, `shape[rank]`, and per-operand
 *      element strides (0 on broadcast axes).  Outputs are dense row-major.                 ---- */
/* binary: ops in the order of expr.py:265-281 */
typedef enum { DGB_ADD = 0, DGB_SUB, DGB_MUL, DGB_TRUEDIV, DGB_FLOORDIV, DGB_MOD, DGB_POW, DGB_MIN,
               DGB_MAX, DGB_LT, DGB_LE, DGB_GT, DGB_GE, DGB_EQ, DGB_NE } dgb_binop;
typedef enum { DGB_NEG = 0, DGB_ABS, DGB_SQRT, DGB_EXP, DGB_LOG } dgb_unop;   /* expr.py:283-289 */

int dgb_ew_binary(int op, void* out_dev, int out_dtype,
                  const void* a_dev, int a_dtype, const int64_t* a_strides,
                  const void* b_dev, int b_dtype, const int64_t* b_strides,
                  int rank, const int64_t* shape, void* stream);
int dgb_ew_unary(int op, void* out_dev, int out_dtype, const void* a_dev, int a_dtype,
                 int64_t n, void* stream);
int dgb_ew_where(void* out_dev, int out_dtype,
                 const void* c_dev, int c_dtype, const int64_t* c_strides,
                 const void* a_dev, int a_dtype, const int64_t* a_strides,
                 const void* b_dev, int b_dtype, const int64_t* b_strides,
                 int rank, const int64_t* shape, void* stream);

/* Fused elementwise program: a chain of the elementwise operations above evaluated in ONE pass --
 * the hand-written counterpart of the reference's loop fusion + array contraction for pointwise
 * chains (ir_passes.py:189-284: fuse_loops, contract_arrays).  `ins` is a register program in issue
 * order; LOAD reads leaf `a` (trailing-aligned broadcast strides over `ext`, like dgb_ew_binary), CONST
 * reads `consts[a]` (raw 64-bit pattern of a double / int64 / 0-1 bool), BINARY / UNARY / WHERE apply
 * `op` to registers a, b, c (WHERE: a if c else b) with the operand dtypes adt / bdt / cdt and the
 * result dtype odt exactly as dgb_ew_binary / dgb_ew_unary / dgb_ew_where would (fcomp: the binary
 * operation is carried out in f64).  Outputs are dense arrays of `total` elements.  Results are
 * bit-identical to issuing the operations one by one. */
enum { DGB_EW_MAX_INS = 96, DGB_EW_MAX_REGS = 32, DGB_EW_MAX_LEAVES = 12, DGB_EW_MAX_OUTS = 4, DGB_EW_MAX_CONSTS = 24 };
typedef enum { DGB_EW_LOAD = 0, DGB_EW_CONST = 1, DGB_EW_BINARY = 2, DGB_EW_UNARY = 3, DGB_EW_WHERE = 4 } dgb_ew_kind;
typedef struct { uint8_t kind, op, dst, a, b, c, adt, bdt, cdt, odt, fcomp, pad_; } dgb_ew_ins;
typedef struct { const void* dev; int32_t dtype; int32_t mode; /* 0 strided, 1 dense, 2 scalar */ int64_t stride[8]; } dgb_ew_leaf;
typedef struct { void* dev; int32_t dtype; int32_t reg; } dgb_ew_out;
typedef struct {
  int32_t nins, nleaves, nouts, rank, need_index, pad_;
  int64_t total;
  int64_t ext[8];
  uint64_t consts[DGB_EW_MAX_CONSTS];
  dgb_ew_leaf leaf[DGB_EW_MAX_LEAVES];
  dgb_ew_out out[DGB_EW_MAX_OUTS];
  dgb_ew_ins ins[DGB_EW_MAX_INS];
} dgb_ew_prog;
int dgb_ew_program(const dgb_ew_prog* prog, void* stream);

/* strided copy / cast (reshape of views, slices, stack, concatenate): out dense */
int dgb_copy_strided(void* out_dev, int out_dtype, const void* a_dev, int a_dtype,
                     const int64_t* a_strides, int rank, const int64_t* shape, void* stream);
/* same with explicit element strides on the output (writes into a slice: concatenate / stack) */
int dgb_copy_scatter(void* out_dev, int out_dtype, const int64_t* out_strides, const void* a_dev, int a_dtype,
                     const int64_t* a_strides, int rank, const int64_t* shape, void* stream);
/* gather along one axis, array viewed as (outer, extent, inner): out[o, k, i] = a[o, idx[k], i];
 * every index is range-checked, DGB_ERR_OUT_OF_BOUNDS otherwise (frontend.py:121-136) */
int dgb_take(void* out_dev, const void* a_dev, int dtype, const int64_t* idx_dev,
             int64_t outer, int64_t extent, int64_t inner, int64_t nidx, void* stream);
/* the same gather for use inside a captured CUDA graph (CompiledFunction(graph=True)): no host
 * synchronisation; an out-of-range index sets *err_dev != 0, which the context checks at its next
 * synchronisation point */
int dgb_take_deferred(void* out_dev, const void* a_dev, int dtype, const int64_t* idx_dev,
                      int64_t outer, int64_t extent, int64_t inner, int64_t nidx, int* err_dev, void* stream);
/* einsum with up to 3 FP64 operands: loop extents `ext[nletters]` (output letters first, then
 * summed letters, ascending accumulation like expr.py:344-364), per-operand strides per letter */
int dgb_einsum(double* out_dev, int nops, const double* const* ops_dev, const int64_t* op_strides,
               int nout_letters, int nletters, const int64_t* ext, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DGB200_H */
