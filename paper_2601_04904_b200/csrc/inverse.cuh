// Complex128 block inverse for the RGF pivots (replaces block_inverse /
// _lu_packed, pkg/src/btasel/kernels.py:169-236, and _invert_pivot,
// pkg/src/btasel/rgf.py:64-71).
//
// Fast path: blocked Gauss-Jordan with kLeaf-wide panels.  Each panel's
// diagonal leaf is inverted with partial pivoting inside one CTA (shared
// memory, no physical row swaps); the panel is then applied to the whole
// matrix with the grouped DMMA GEMM (zgemm.cuh).  This is exact block
// Gauss-Jordan, stable for the (block) diagonally dominant pivots the RGF
// produces.  Drop-in semantics of the reference (error iff LAPACK-style
// partial pivoting meets an exactly zero pivot) are preserved by an exact
// fallback: when a leaf meets an exactly zero pivot, a full-column
// partial-pivoting Gauss-Jordan of the untouched input runs on device and
// only it decides singularity.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bsel {

constexpr int kLeaf = 32;

// Debug: when non-null (device buffer of 8*panels u64), the persistent
// inverse records per-panel globaltimer stamps there.
extern unsigned long long* g_inverse_trace;

// Instrumented builds (-DBSEL_INV_STATS=1, run with BSEL_INV_STATS=1): the
// marks the chain's kernels use to measure the gap between one chain kernel's
// end and the next one's start (printed with the inverse statistics); null
// otherwise.  One lane per process (the marks are per process).
unsigned long long* chain_marks();

// Workspace (complex elements) needed by launch_block_inverse for one n x n.
// It must be ZERO when first used (its head holds the dataflow kernel's
// epoch-tagged ready flags, which are never reset).
int64_t block_inverse_workspace(int n);

// Y = inv(X) for one n x n matrix (X untouched, Y must not alias X).
//  work   : block_inverse_workspace(n) complex elements
//  flag   : one device int, 0 on entry; 1 = leaf met a zero pivot (fallback ran),
//           2 + row = exactly singular at pivot row `row`
//  status : optional device u64; on exact singularity atomicMin(status, key)
//  grid   : CTAs of the persistent kernel (0 = default, BSEL_INV_GRID or 64)
cudaError_t launch_block_inverse(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n,
                                 double2* work, int* flag, unsigned long long* status,
                                 unsigned long long key, cudaStream_t stream, int grid = 0);

// Fused Schur step of the forward sweeps (one persistent launch):
//   Sout = D^-1, H = D^-1 U, F = L D^-1, C <- C - L D^-1 U   (all b x b)
// by Gauss-Jordan on [[D, U], [L, C]] with pivots in D only: the chain's two
// GEMMs become part of the panel updates.  H may be null (not kept).  Same
// singularity semantics as launch_block_inverse (exact fallback recomputes
// everything from the untouched D, U, L, C).  b > kLeaf only.
int64_t schur_step_workspace(int b);
bool schur_step_supported(int b);
cudaError_t launch_schur_step(const double2* D, int64_t ldd, const double2* U, int64_t ldu, const double2* L,
                              int64_t ldl, double2* C, int64_t ldc, double2* S, int64_t lds, double2* H,
                              int64_t ldh, double2* F, int64_t ldf, int b, double2* work, int* flag,
                              unsigned long long* status, unsigned long long key, cudaStream_t stream,
                              int grid = 0);

// Batched small inverses (n <= kLeaf) in one launch: Y_b = inv(X_b).
cudaError_t launch_leaf_inverse_batched(const double2* X, int64_t ldx, int64_t strideX, double2* Y,
                                        int64_t ldy, int64_t strideY, int n, int batch, int* flags,
                                        cudaStream_t stream);

}  // namespace bsel
