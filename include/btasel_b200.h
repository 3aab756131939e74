/*
 * btasel_b200 -- C ABI of the B200-native fused BT/BTA selected inversion (SI)
 * and selected quadratic solution (SQ) solver.
 *
 * Drop-in boundary for the reference `btasel` package (arXiv 2601.04904,
 * /root/reference/pkg/src/btasel).  The reference is pure Python/NumPy and has
 * no FFI of its own; each entry point below replaces the Python function cited
 * next to it, and the Python facade in paper_2601_04904_b200/ binds them with
 * ctypes exactly like the reference functions are called.
 *
 * Conventions
 *  - All matrix pointers are DEVICE pointers (CUDA global memory) unless the
 *    function name says `_host`.
 *  - complex128 is stored interleaved (re, im) as two IEEE doubles, blocks
 *    row-major, block lists stacked contiguously: exactly the numpy layout of
 *    a list of C-contiguous complex128 blocks and the BTA1 payload order
 *    (fileio.py:37-49), so host <-> device is one memcpy per array.
 *  - No exception crosses the ABI: every call returns a bsel_code_t and fills
 *    the optional status struct (code, index, message).
 *  - Calls are stream-ordered on the context's stream; they return after
 *    enqueueing except where noted ("synchronizes").
 */
#ifndef BTASEL_B200_H
#define BTASEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSEL_ABI_VERSION 3

typedef enum {
  BSEL_OK = 0,
  BSEL_ERR_SHAPE = 1,    /* -> ShapeMismatchError      (errors.py:8)      */
  BSEL_ERR_SINGULAR = 2, /* -> SingularBlockError(index) (errors.py:12-24) */
  BSEL_ERR_CUDA = 3,     /* -> RuntimeError                                 */
  BSEL_ERR_ARG = 4,      /* -> ValueError                                   */
  BSEL_ERR_INTERNAL = 5
} bsel_code_t;

typedef struct {
  int32_t code;
  int32_t reserved;
  int64_t index; /* singular: global diagonal block index (n for the tip) or
                    pivot row for bsel_block_inverse; -1 otherwise          */
  char message[256];
} bsel_status_t;

/* BtaMatrix (matrix.py:35-72) as stacked device arrays.  a == 0: BT. */
typedef struct {
  int64_t n, b, a;
  double* diag;      /* [n][b][b]                                  */
  double* lower;     /* [n-1][b][b]  block (i+1, i)                */
  double* upper;     /* [n-1][b][b]  block (i, i+1)                */
  double* arrow_row; /* [n][a][b]    block (t, i)                  */
  double* arrow_col; /* [n][b][a]    block (i, t)                  */
  double* tip;       /* [a][a]                                     */
} bsel_bta_t;

/* RgfFactors (rgf.py:37-61) as device arrays. */
typedef struct {
  int64_t n, b, a;
  int32_t fused; /* 1 = "siq", 0 = "si" */
  int32_t reserved;
  double* s_a;              /* [n][b][b]   inverted updated pivots          */
  double* s_b;              /* [n-1][b][b] quadratic Schur blocks (fused)   */
  double* b_diag_last;      /* [b][b]      (fused)                          */
  double* tip_inv;          /* [a][a]      tip_schur_inv                    */
  double* b_tip;            /* [a][a]      (fused)                          */
  double* arrow_row_elim;   /* [n][a][b]   strips as seen at elimination    */
  double* arrow_col_elim;   /* [n][b][a]                                    */
  double* b_arrow_row_elim; /* [n][a][b]   (fused)                          */
  double* b_arrow_col_elim; /* [n][b][a]   (fused)                          */
  /* Optional (NULL = recomputed by the backward): elimination products the
   * forward step of block i forms anyway, retained for the backward step of
   * block i (no reference counterpart):
   *   elim_f = A(j,i) S_i, elim_g = AR_i S_i,
   *   elim_q = Bd_i elim_f^H - B(i,j), elim_k = Bd_i elim_g^H - BC_i.        */
  double* elim_f;           /* [n][b][b]                                    */
  double* elim_g;           /* [n][a][b]                                    */
  double* elim_q;           /* [n][b][b]   (fused)                          */
  double* elim_k;           /* [n][b][a]   (fused)                          */
  double* elim_h;           /* [n][b][b]   S_i A(i,j)                       */
  double* elim_ha;          /* [n][b][a]   S_i AC_i                         */
  double* elim_eq;          /* [n][b][b]   -S_i elim_q      (fused)         */
  double* elim_ek;          /* [n][b][a]   -S_i elim_k      (fused)         */
} bsel_factors_t;

typedef struct bsel_context bsel_context_t;

/* ---- context ------------------------------------------------------------ */
int bsel_abi_version(void);
int bsel_context_create(int device, bsel_context_t** out, bsel_status_t* st);
int bsel_context_destroy(bsel_context_t* ctx);
/* Run subsequent calls on `cuda_stream` (cudaStream_t; NULL = legacy default). */
int bsel_context_set_stream(bsel_context_t* ctx, void* cuda_stream);
/* CTAs of the persistent block inverse on this context (0 = default: 64 or
 * BSEL_INV_GRID), for the sweeps and bsel_block_inverse.  Contexts sweeping
 * concurrently on one GPU (in-GPU partitions) use fewer so the chains leave
 * SMs to each other's GEMMs.                                                */
int bsel_context_set_inverse_grid(bsel_context_t* ctx, int ctas);
/* Symmetry of the right-hand side B.  Every forward entry point checks B
 * EXACTLY on its pattern (B = B^H, B = -B^H) while staging it; when B = s B^H
 * the backward sweep uses X_B = s X_B^H (fewer products, same result to
 * rounding).  mode: +1 / -1 force that path, 0 forces the general path,
 * 2 (default) = from this context's own last check.  A partitioned solve
 * must decide for the WHOLE B: OR the partitions' flags and force the mode.
 * flags: bit 0 = B is not Hermitian, bit 1 = B is not anti-Hermitian
 * (3 if nothing was checked since the last forward began).               */
int bsel_context_set_b_symmetry(bsel_context_t* ctx, int mode);
/* Forward sweeps on this context keep SMs [0, n) free of their throughput
 * (aux-stream) GEMM levels, so the Schur chain's inverse runs on SMs of its
 * own (one partition per GPU: the chain is the critical path).  0 = off.  */
int bsel_context_set_aux_avoid_sms(bsel_context_t* ctx, int n);
int bsel_context_b_symmetry(bsel_context_t* ctx, int* flags, int* mode);
/* Synchronizes; reports deferred device errors (singular pivots). */
int bsel_synchronize(bsel_context_t* ctx, bsel_status_t* st);
/* Device time of the last forward / backward sweep in ms (synchronizes). */
int bsel_last_timings(bsel_context_t* ctx, double* forward_ms, double* backward_ms);

/* ---- kernels (kernels.py) ----------------------------------------------- */
/* block_multiply_acc (kernels.py:106-154):
 *   d = beta*c + alpha*op(a) @ op(b), op = identity or conjugate transpose.
 *   op(a) is m x k, op(b) is k x n; c may be NULL (then beta is ignored);
 *   d may alias c.  alpha/beta are complex (re, im).                        */
int bsel_block_multiply_acc(bsel_context_t* ctx, double* d, int64_t ldd, const double* c, int64_t ldc,
                            const double* a, int64_t lda, int trans_a, const double* b, int64_t ldb,
                            int trans_b, int64_t m, int64_t n, int64_t k, double alpha_re, double alpha_im,
                            double beta_re, double beta_im, bsel_status_t* st);
/* block_inverse (kernels.py:220-236): out = a^-1 (n x n).  Exactly singular
 * (partial pivoting meets a zero pivot) -> BSEL_ERR_SINGULAR, index = pivot
 * row.  Synchronizes.                                                       */
int bsel_block_inverse(bsel_context_t* ctx, const double* a, int64_t lda, double* out, int64_t ldo,
                       int64_t n, bsel_status_t* st);

/* ---- sequential solver (rgf.py) ----------------------------------------- */
/* bt_forward / bta_forward (rgf.py:79, :207): a_work (and b_work, NULL for
 * "si") are working copies mutated in place; factors are written to `f`
 * (whose *_elim pointers must alias the working arrow strips or be copies
 * filled afterwards by the caller).  Synchronizes; singular pivot ->
 * BSEL_ERR_SINGULAR with the global block index (n for the tip).           */
int bsel_bta_forward(bsel_context_t* ctx, const bsel_bta_t* a_work, const bsel_bta_t* b_work,
                     const bsel_factors_t* f, bsel_status_t* st);
/* bt_backward / bta_backward (rgf.py:127, :401): reads the factors and the
 * original off-diagonal blocks of a (and b); writes x_a (and x_b).         */
int bsel_bta_backward(bsel_context_t* ctx, const bsel_factors_t* f, const bsel_bta_t* a, const bsel_bta_t* b,
                      const bsel_bta_t* x_a, const bsel_bta_t* x_b, int diagonal_only, bsel_status_t* st);
/* Device workspace (bytes) needed by bsel_solve_selected. */
int bsel_solve_workspace_size(int64_t n, int64_t b, int64_t a, int fused, size_t* bytes);
/* solve_selected (rgf.py:497-531): non-destructive forward + backward.
 * `b`, `x_b` NULL for "si".  workspace: >= bsel_solve_workspace_size bytes
 * of device memory (NULL: the context allocates it).  Synchronizes.        */
int bsel_solve_selected(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b, const bsel_bta_t* x_a,
                        const bsel_bta_t* x_b, int diagonal_only, void* workspace, size_t workspace_bytes,
                        bsel_status_t* st);

/* ---- distributed scheme (dist.py) --------------------------------------- */
/* LocalFactors (dist.py:134-151) of the partition [lo, hi), block i stored
 * at index i - lo.  fill_* (middle partitions): couplings A'(lo,i)/A'(i,lo)
 * seen when block i is eliminated; index hi-lo-1 = final coupling pair.   */
typedef struct {
  int64_t lo, hi;
  int32_t kind; /* 0 first, 1 middle, 2 last (plan_partitions kinds)  */
  int32_t fused;
  double* s_a;        /* [len][b][b]                                     */
  double* s_b;        /* [len][b][b]  (fused)                            */
  double* fill_row;   /* [len][b][b]  (middle)                           */
  double* fill_col;   /* [len][b][b]  (middle)                           */
  double* b_fill_row; /* [len][b][b]  (middle, fused)                    */
  double* b_fill_col; /* [len][b][b]  (middle, fused)                    */
  /* Optional elimination products (see bsel_factors_t); middle partitions
   * also elim_fr = fill_row S_i and elim_qr = Bd_i elim_fr^H - b_fill_col.  */
  double* elim_f;     /* [len][b][b]                                     */
  double* elim_g;     /* [len][a][b]                                     */
  double* elim_q;     /* [len][b][b]  (fused)                            */
  double* elim_k;     /* [len][b][a]  (fused)                            */
  double* elim_fr;    /* [len][b][b]  (middle)                           */
  double* elim_qr;    /* [len][b][b]  (middle, fused)                    */
  double* elim_h;     /* [len][b][b]  S_i U_i (U = the coupling eliminated along) */
  double* elim_ha;    /* [len][b][a]  S_i AC_i                           */
  double* elim_eq;    /* [len][b][b]  -S_i elim_q   (fused)              */
  double* elim_ek;    /* [len][b][a]  -S_i elim_k   (fused)              */
} bsel_local_factors_t;
/* Optional end-to-end mode (no reference counterpart; the reference moves
 * whole matrices with cupy before/after its sweeps): the full-size matrices
 * stay in (pinned) host memory and move in chunks of chunk_blocks partition
 * blocks on the context's copy stream, overlapped with the sweeps.
 * local_forward reads a/b (host inputs; copy_tip = this partition also
 * moves the tips) -- the device a/b then only provide storage for the
 * couplings and tip, their diag/arrow arrays are not read; local_backward
 * writes x_a/x_b (host outputs; the tip when write_tip).  copy_stream
 * (cudaStream_t, NULL = the context's own): partitions running
 * concurrently on one GPU should share one input copy stream -- the chunks
 * are queued a few chunks ahead of each sweep, so a shared stream
 * interleaves them in progress order (separate streams are drained one
 * after the other by the copy engine).  The calling stream waits for every
 * copy.  NULL io = no host transfers.                                      */
typedef struct {
  const bsel_bta_t* a;   /* host inputs  (local_forward)  */
  const bsel_bta_t* b;
  const bsel_bta_t* x_a; /* host outputs (local_backward) */
  const bsel_bta_t* x_b;
  int64_t chunk_blocks;
  int32_t copy_tip;
  int32_t reserved;
  void* copy_stream;
} bsel_host_io_t;

/* local_forward (dist.py:172-416): a, b = full original matrices (read
 * only); a_work/b_work = partition working arrays (n = hi-lo; diag, arrow
 * strips; tip receives the rank's tip contribution).  Afterwards the work
 * arrays hold the retained strips and the boundary payload.  Synchronizes;
 * singular pivot -> BSEL_ERR_SINGULAR with the global block index.        */
int bsel_local_forward(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b, const bsel_bta_t* a_work,
                       const bsel_bta_t* b_work, const bsel_local_factors_t* f, const bsel_host_io_t* io,
                       bsel_status_t* st);
/* local_backward (dist.py:542-744): seeded from the reduced solution
 * (x_red, z_red; boundary indices k_top/k_bot), writes this partition's
 * pattern blocks of the full-size outputs x_a/x_b (and the tip if
 * write_tip).                                                              */
int bsel_local_backward(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b,
                        const bsel_local_factors_t* f, const bsel_bta_t* a_work, const bsel_bta_t* b_work,
                        const bsel_bta_t* x_red, const bsel_bta_t* z_red, int64_t k_top, int64_t k_bot,
                        int write_tip, const bsel_bta_t* x_a, const bsel_bta_t* x_b,
                        const bsel_host_io_t* io, bsel_status_t* st);

/* ---- synthetic inputs (matrix.py) --------------------------------------- */
/* generate_dd_bta (matrix.py:224-284) written straight into device arrays:
 * bit-identical splitmix64 stream; the dominance shift sums |row| entries
 * left to right (the host uses pairwise sums: last-bit differences on the
 * shifted diagonal are possible).                                          */
int bsel_generate_dd_bta(bsel_context_t* ctx, const bsel_bta_t* out, uint64_t seed, double dominance,
                         bsel_status_t* st);
/* hermitianize (matrix.py:337-354) in place: m <- (m + m^H)/2 on the pattern. */
int bsel_hermitianize(bsel_context_t* ctx, const bsel_bta_t* m, bsel_status_t* st);
/* Boundary publication over peer memory (the distributed scheme's all_gather,
 * dist.py:436, as one kernel of NVLink P2P stores): copy nblocks (<= 16)
 * device blocks src[i] of elems[i] complex elements to complex offset
 * dst_off[i] of EVERY destination buffer dst[d] (ndst <= 8: the group's
 * symmetric-memory receive buffers, this rank's included, mapped into this
 * process), plus the 4-double slot header at complex offset hdr_off.  The
 * caller orders it with a device-side group barrier before the receivers
 * read.  Replaces: collectives.py:136-158 ThreadCollectives.all_gather
 * (TorchCollectives(symmetric=True)).                                      */
int bsel_publish(bsel_context_t* ctx, const void* const* src, const int64_t* elems, const int64_t* dst_off,
                 int nblocks, void* const* dst, int ndst, int64_t hdr_off, const double* hdr, bsel_status_t* st);
/* Number of CUDA kernels this library has launched in this process.        */
uint64_t bsel_kernel_launches(void);

/* ---- instrumentation ------------------------------------------------------ */
typedef struct {
  int64_t gemm_launches; /* grouped DMMA GEMM launches (outside inverses)   */
  double gemm_flops;     /* sum of 8*M*N*K over their products            */
  double gemm_ms;        /* sum of their CUDA-event durations              */
  int64_t inverse_calls; /* block inverses                                  */
  double inverse_ms;     /* sum of their CUDA-event durations              */
  double gemm_bytes;     /* compulsory bytes of the GEMM launches: every  */
                         /* operand read once, outputs written once       */
  double gemm_busy_ms;   /* union of the GEMM launches' [start, end] spans */
                         /* (launches on concurrent streams overlap)      */
  double inverse_busy_ms;/* union of the inverses' spans                   */
  double inverse_flops;  /* sum of 8*n^3 over the inverses                 */
  double gemm_exec_flops;/* tensor-pipe flops the GEMM launches executed:   */
                         /* 6*M*N*K per product in the 3M kernel, 8*M*N*K */
                         /* in the real-embedding kernel                   */
} bsel_profile_t;
/* Bracket every launch with CUDA events on its stream until _end (which
 * synchronizes the device and returns the totals).                        */
int bsel_profile_begin(void);
int bsel_profile_end(bsel_profile_t* out);

#ifdef __cplusplus
}
#endif
#endif /* BTASEL_B200_H */
