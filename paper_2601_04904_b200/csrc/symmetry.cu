// See symmetry.cuh.  Both kernels are HBM-bound tile transposes: a 32 x 32
// complex tile and its mirror are staged through shared memory so that every
// global access is a coalesced 16-byte row segment.
#include <algorithm>

#include "symmetry.cuh"
#include "zgemm.cuh"

namespace bsel {

namespace {
constexpr int kT = 32, kRows = 8;

__global__ void __launch_bounds__(kT * kRows) sym_check_kernel(SymJob j, int* flags) {
  const int tj = blockIdx.x, ti = blockIdx.y;
  if (j.same && ti > tj) return;
  __shared__ double2 sx[kT][kT + 1], sy[kT][kT + 1];
  __shared__ int s_done;
  if (!j.dX) {
    // one read of the flags word decides the early exit for the whole block
    // (other blocks may be OR-ing it concurrently)
    if (threadIdx.x == 0 && threadIdx.y == 0)
      s_done = *reinterpret_cast<volatile int*>(flags) == (kNotHermitian | kNotSkew);
    __syncthreads();
    if (s_done) return;
  }
  const int64_t blk = blockIdx.z;
  const double2* X = j.X + blk * j.sx;
  const double2* Y = j.Y + blk * j.sy;
  double2* dX = j.dX ? j.dX + blk * j.sx : nullptr;
  double2* dY = j.dY ? j.dY + blk * j.sy : nullptr;
  const int tx = threadIdx.x;
  const bool mirror_copy = dY && !(j.same && ti == tj);
  for (int e = threadIdx.y; e < kT; e += kRows) {
    // X tile: rows ti*32.., cols tj*32..  (X is r x c)
    int row = ti * kT + e, col = tj * kT + tx;
    if (row < j.r && col < j.c) {
      const double2 v = X[(int64_t)row * j.c + col];
      sx[e][tx] = v;
      if (dX) dX[(int64_t)row * j.c + col] = v;
    }
    // Y tile: rows tj*32.., cols ti*32..  (Y is c x r)
    row = tj * kT + e, col = ti * kT + tx;
    if (row < j.c && col < j.r) {
      const double2 v = Y[(int64_t)row * j.r + col];
      sy[e][tx] = v;
      if (mirror_copy) dY[(int64_t)row * j.r + col] = v;
    }
  }
  __syncthreads();
  int bad = 0;
  for (int e = threadIdx.y; e < kT; e += kRows) {
    const int row = ti * kT + e, col = tj * kT + tx;  // X[row][col] vs Y[col][row]
    if (row < j.r && col < j.c) {
      const double2 x = sx[e][tx], y = sy[tx][e];
      if (x.x != y.x || x.y != -y.y) bad |= kNotHermitian;
      if (x.x != -y.x || x.y != y.y) bad |= kNotSkew;
    }
  }
  const int h = __syncthreads_or(bad & kNotHermitian), k = __syncthreads_or(bad & kNotSkew);
  if (threadIdx.x == 0 && threadIdx.y == 0 && (h || k)) atomicOr(flags, (h ? kNotHermitian : 0) | (k ? kNotSkew : 0));
}

struct TransBatch {
  TransJob j[3];
  int n;
  int sign;
};

__global__ void __launch_bounds__(kT * kRows) conj_transpose_kernel(TransBatch b) {
  int t = blockIdx.x;
  int q = 0;
  for (; q < b.n; ++q) {
    const int tiles = ((b.j[q].r + kT - 1) / kT) * ((b.j[q].c + kT - 1) / kT);
    if (t < tiles) break;
    t -= tiles;
  }
  if (q == b.n) return;
  const TransJob& J = b.j[q];
  const int tc = (J.c + kT - 1) / kT;
  const int ti = t / tc, tj = t % tc;  // src tile (rows ti, cols tj)
  __shared__ double2 s[kT][kT + 1];
  const int tx = threadIdx.x;
  for (int e = threadIdx.y; e < kT; e += kRows) {
    const int row = ti * kT + e, col = tj * kT + tx;
    if (row < J.r && col < J.c) s[e][tx] = J.src[(int64_t)row * J.lds + col];
  }
  __syncthreads();
  const double sg = (double)b.sign;
  for (int e = threadIdx.y; e < kT; e += kRows) {
    const int row = tj * kT + e, col = ti * kT + tx;  // dst[row][col] = sign * conj(src[col][row])
    if (row < J.c && col < J.r) {
      const double2 v = s[tx][e];
      J.dst[(int64_t)row * J.ldd + col] = make_double2(sg * v.x, -sg * v.y);
    }
  }
}
__global__ void __launch_bounds__(kT * kRows) mirror_lower_kernel(double2* A, int64_t ld, int n, int sign) {
  // pair index -> (tj, ti), ti <= tj: the upper tile (ti, tj) is written from
  // the lower tile (tj, ti)
  const int l = blockIdx.x;
  int tj = (int)((sqrt(8.0 * l + 1.0) - 1.0) * 0.5);
  while ((tj + 1) * (tj + 2) / 2 <= l) ++tj;
  while (tj * (tj + 1) / 2 > l) --tj;
  const int ti = l - tj * (tj + 1) / 2;
  __shared__ double2 s[kT][kT + 1];
  const int tx = threadIdx.x;
  for (int e = threadIdx.y; e < kT; e += kRows) {  // lower tile rows tj*32.., cols ti*32..
    const int row = tj * kT + e, col = ti * kT + tx;
    if (row < n && col < n) s[e][tx] = A[(int64_t)row * ld + col];
  }
  __syncthreads();
  const double sg = (double)sign;
  for (int e = threadIdx.y; e < kT; e += kRows) {  // upper element (ti*32+e, tj*32+tx) <- s[tx][e]
    const int row = ti * kT + e, col = tj * kT + tx;
    if (row < n && col < n && col > row) {
      const double2 v = s[tx][e];
      A[(int64_t)row * ld + col] = make_double2(sg * v.x, -sg * v.y);
    }
  }
}
}  // namespace

cudaError_t launch_mirror_lower(double2* A, int64_t ld, int n, int sign, cudaStream_t s) {
  if (n <= 1) return cudaSuccess;
  const int nt = (n + kT - 1) / kT;
  mirror_lower_kernel<<<nt * (nt + 1) / 2, dim3(kT, kRows), 0, s>>>(A, ld, n, sign);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sym_check(const SymJob& j, int* flags, cudaStream_t s) {
  if (j.r <= 0 || j.c <= 0) return cudaSuccess;
  for (int64_t b0 = 0; b0 < j.count; b0 += 65535) {  // gridDim.z limit
    SymJob part = j;
    part.count = std::min<int64_t>(65535, j.count - b0);
    part.X += b0 * j.sx;
    part.Y += b0 * j.sy;
    if (part.dX) part.dX += b0 * j.sx;
    if (part.dY) part.dY += b0 * j.sy;
    dim3 grid((j.c + kT - 1) / kT, (j.r + kT - 1) / kT, (unsigned)part.count);
    sym_check_kernel<<<grid, dim3(kT, kRows), 0, s>>>(part, flags);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_conj_transpose(const TransJob* jobs, int njobs, int sign, cudaStream_t s) {
  TransBatch b{};
  int tiles = 0;
  for (int q = 0; q < njobs; ++q) {
    if (jobs[q].r <= 0 || jobs[q].c <= 0) continue;
    b.j[b.n++] = jobs[q];
    tiles += ((jobs[q].r + kT - 1) / kT) * ((jobs[q].c + kT - 1) / kT);
  }
  if (tiles == 0) return cudaSuccess;
  b.sign = sign;
  conj_transpose_kernel<<<tiles, dim3(kT, kRows), 0, s>>>(b);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsel
