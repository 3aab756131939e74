// Exact (anti-)Hermitian detection of the right-hand side B and conjugate
// transposes for the symmetric backward path (steps.cuh BackSweep).
//
// X_B = A^-1 B A^-H inherits B^H = s B (s = +1 Hermitian, e.g. the bench
// protocol's hermitianize(B) (cli.py:273-277); s = -1 anti-Hermitian, the
// physical lesser/greater self-energies).  The check is EXACT on the pattern:
// diag blocks D = s D^H, lower_i = s upper_i^H, arrow_row_i = s arrow_col_i^H,
// tip = s tip^H.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace bsel {

// flags bit 0: some entry violates B = B^H; bit 1: some entry violates B = -B^H.
enum : int { kNotHermitian = 1, kNotSkew = 2 };

// Check `count` block pairs X (r x c, stride sx) against Y (c x r, stride sy):
// X == s Y^H entrywise; OR the violations into *flags.  `same`: X and Y are
// the same blocks (diag, tip).  dX / dY (optional, same layout) receive a copy
// of X / Y, so the working-copy staging of B costs no extra pass.
struct SymJob {
  const double2* X = nullptr;
  const double2* Y = nullptr;
  double2* dX = nullptr;
  double2* dY = nullptr;
  int r = 0, c = 0;
  int64_t sx = 0, sy = 0, count = 0;
  bool same = false;
};
cudaError_t launch_sym_check(const SymJob& j, int* flags, cudaStream_t s);

// dst (c x r) = sign * src^H for up to 3 blocks (src r x c).
struct TransJob {
  const double2* src = nullptr;
  double2* dst = nullptr;
  int64_t lds = 0, ldd = 0;
  int r = 0, c = 0;
};
cudaError_t launch_conj_transpose(const TransJob* jobs, int njobs, int sign, cudaStream_t s);

// A (n x n): A[r][c] = sign * conj(A[c][r]) for c > r (the strict upper
// triangle from the lower one; pairs with Level::lower_only()).
cudaError_t launch_mirror_lower(double2* A, int64_t ld, int n, int sign, cudaStream_t s);

}  // namespace bsel
