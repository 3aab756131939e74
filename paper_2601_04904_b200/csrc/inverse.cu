// Complex128 block inverse (see inverse.cuh).
#include "inverse.cuh"
#include "zgemm.cuh"

namespace bsel {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 crecip(double2 a) {
  // Smith's algorithm (no spurious overflow/underflow).
  if (fabs(a.x) >= fabs(a.y)) {
    double r = a.y / a.x, d = a.x + a.y * r;
    return make_double2(1.0 / d, -r / d);
  }
  double r = a.x / a.y, d = a.y + a.x * r;
  return make_double2(r / d, -1.0 / d);
}
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }

// In-place Gauss-Jordan with partial pivoting and *virtual* row interchanges
// (rows are never moved: piv[k] is the physical pivot row of step k).  After
// n steps the storage S satisfies inv(A)[r][piv[k]] = S[piv[r]][k].
// Pivot choice: max |re|+|im| among unused rows (LAPACK izamax), lowest
// index on ties.  Two barriers per elimination step.
template <int NB, int THREADS>
__global__ void __launch_bounds__(THREADS)
    leaf_inverse_kernel(const double2* __restrict__ X, int64_t ldx, int64_t sx, double2* __restrict__ Y,
                        int64_t ldy, int64_t sy, int n, int* flags, int64_t flag_stride) {
  __shared__ double2 a[NB][NB + 1];
  __shared__ double2 fcol[NB];
  __shared__ double2 prow[NB];
  __shared__ int piv[NB];
  __shared__ int used[NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  X += blockIdx.x * sx;
  Y += blockIdx.x * sy;
  int* flag = flags + blockIdx.x * flag_stride;

  for (int e = tid; e < NB * NB; e += THREADS) {
    int i = e / NB, j = e % NB;
    if (i < n && j < n) a[i][j] = X[(int64_t)i * ldx + j];
  }
  for (int i = tid; i < NB; i += THREADS) used[i] = 0;
  __syncthreads();

  bool any_zero = false;
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int bi = NB;
      for (int i = lane; i < n; i += 32) {
        if (!used[i]) {
          double v = cabs1(a[i][k]);
          if (v > best) {
            best = v;
            bi = i;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      const bool zero = !(best > 0.0);
      int p = bi;
      if (p >= n) p = k;  // only reachable for NaN columns
      double2 inv = zero ? make_double2(1.0, 0.0) : crecip(a[p][k]);
      for (int i = lane; i < n; i += 32) fcol[i] = (i == p) ? make_double2(0.0, 0.0) : a[i][k];
      for (int j = lane; j < n; j += 32) prow[j] = (j == k) ? inv : cmul(a[p][j], inv);
      if (lane == 0) {
        piv[k] = p;
        used[p] = 1;
      }
      any_zero |= zero;
    }
    __syncthreads();
    const int p = piv[k];
    for (int e = tid; e < NB * NB; e += THREADS) {
      int i = e / NB, j = e % NB;
      if (i >= n || j >= n) continue;
      double2 pr = prow[j];
      if (i == p) {
        a[i][j] = pr;
      } else {
        double2 f = fcol[i];
        double2 v = (j == k) ? make_double2(0.0, 0.0) : a[i][j];
        v.x -= f.x * pr.x - f.y * pr.y;
        v.y -= f.x * pr.y + f.y * pr.x;
        a[i][j] = v;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && any_zero) atomicMax(flag, 1);
  for (int e = tid; e < NB * NB; e += THREADS) {
    int r = e / NB, k = e % NB;
    if (r < n && k < n) Y[(int64_t)r * ldy + piv[k]] = a[piv[r]][k];
  }
}

// Exact fallback: full-column partial-pivoting Gauss-Jordan in global memory
// (one CTA).  Runs only when the fast path flagged a zero leaf pivot.
__global__ void __launch_bounds__(1024)
    exact_inverse_kernel(const double2* __restrict__ X, int64_t ldx, double2* __restrict__ Y, int64_t ldy,
                         int n, double2* __restrict__ S, int* flag, unsigned long long* status,
                         unsigned long long key) {
  if (*flag != 1) return;  // only after a fast-path zero pivot
  extern __shared__ unsigned char smem_raw[];
  double2* fcol = reinterpret_cast<double2*>(smem_raw);
  double2* prow = fcol + n;
  int* piv = reinterpret_cast<int*>(prow + n);
  int* used = piv + n;
  __shared__ double s_best[32];
  __shared__ int s_bi[32];
  __shared__ int s_p;
  __shared__ double2 s_inv;
  __shared__ int s_zero;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int64_t e = tid; e < (int64_t)n * n; e += blockDim.x) {
    int i = (int)(e / n), j = (int)(e % n);
    S[e] = X[(int64_t)i * ldx + j];
  }
  for (int i = tid; i < n; i += blockDim.x) used[i] = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = tid; i < n; i += blockDim.x) {
      if (!used[i]) {
        double v = cabs1(S[(int64_t)i * n + k]);
        if (v > best || (v == best && i < bi)) {
          best = v;
          bi = i;
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, off);
      int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_best[warp] = best;
      s_bi[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double bb = -1.0;
      int b2 = n;
      for (int w = 0; w < nw; ++w)
        if (s_best[w] > bb || (s_best[w] == bb && s_bi[w] < b2)) {
          bb = s_best[w];
          b2 = s_bi[w];
        }
      s_zero = !(bb > 0.0);
      s_p = (b2 < n) ? b2 : k;
      if (!s_zero) s_inv = crecip(S[(int64_t)s_p * n + k]);
    }
    __syncthreads();
    if (s_zero) {
      if (tid == 0) {
        *flag = 2 + k;
        if (status) atomicMin(status, key);
      }
      return;
    }
    const int p = s_p;
    const double2 inv = s_inv;
    for (int i = tid; i < n; i += blockDim.x) fcol[i] = (i == p) ? make_double2(0.0, 0.0) : S[(int64_t)i * n + k];
    for (int j = tid; j < n; j += blockDim.x) prow[j] = (j == k) ? inv : cmul(S[(int64_t)p * n + j], inv);
    if (tid == 0) {
      piv[k] = p;
      used[p] = 1;
    }
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)n * n; e += blockDim.x) {
      int i = (int)(e / n), j = (int)(e % n);
      double2 pr = prow[j];
      if (i == p) {
        S[e] = pr;
      } else {
        double2 f = fcol[i];
        double2 v = (j == k) ? make_double2(0.0, 0.0) : S[e];
        v.x -= f.x * pr.x - f.y * pr.y;
        v.y -= f.x * pr.y + f.y * pr.x;
        S[e] = v;
      }
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < (int64_t)n * n; e += blockDim.x) {
    int r = (int)(e / n), k = (int)(e % n);
    Y[(int64_t)r * ldy + piv[k]] = S[(int64_t)piv[r] * n + k];
  }
  if (tid == 0) *flag = 0;  // fast path failed, exact path succeeded
}

constexpr int kLeafThreads = 256;

GemmTerm term(const double2* A, int64_t lda, uint8_t opA, const double2* B, int64_t ldb, uint8_t opB,
              int K, int sign) {
  GemmTerm t{};
  t.A = A;
  t.B = B;
  t.lda = lda;
  t.ldb = ldb;
  t.K = K;
  t.opA = opA;
  t.opB = opB;
  t.sign = static_cast<int8_t>(sign);
  return t;
}

}  // namespace

int64_t block_inverse_workspace(int n) { return (int64_t)n * n; }

cudaError_t launch_leaf_inverse_batched(const double2* X, int64_t ldx, int64_t strideX, double2* Y,
                                        int64_t ldy, int64_t strideY, int n, int batch, int* flags,
                                        cudaStream_t stream) {
  if (n <= 0 || batch <= 0) return cudaSuccess;
  if (n > kLeaf) return cudaErrorInvalidValue;
  leaf_inverse_kernel<kLeaf, kLeafThreads>
      <<<batch, kLeafThreads, 0, stream>>>(X, ldx, strideX, Y, ldy, strideY, n, flags, 1);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_inverse(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n,
                                 double2* work, int* flag, unsigned long long* status,
                                 unsigned long long key, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  const int panels = (n + kLeaf - 1) / kLeaf;
  // Ping-pong so that the last panel writes Y and X is never written.
  const double2* R = X;
  int64_t ldr = ldx;
  for (int s = 0; s < panels; ++s) {
    double2* W = ((panels - 1 - s) % 2 == 0) ? Y : work;
    const int64_t ldw = (W == Y) ? ldy : n;
    const int j0 = s * kLeaf;
    const int jb = (n - j0 < kLeaf) ? n - j0 : kLeaf;
    const int j1 = j0 + jb;
    // 1. leaf: W[J,J] = inv(R[J,J])
    leaf_inverse_kernel<kLeaf, kLeafThreads><<<1, kLeafThreads, 0, stream>>>(
        R + (int64_t)j0 * ldr + j0, ldr, 0, W + (int64_t)j0 * ldw + j0, ldw, 0, jb, flag, 0);
    count_launch();
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    if (panels == 1) break;
    const double2* Dinv = W + (int64_t)j0 * ldw + j0;
    // 2. row panel: W[J,K] = Dinv . R[J,K]  for K != J
    {
      GemmBatch b{};
      int np = 0;
      const int cols[2][2] = {{0, j0}, {j1, n}};
      for (auto& c : cols) {
        if (c[1] <= c[0]) continue;
        GemmProblem& P = b.p[np++];
        P.D = W + (int64_t)j0 * ldw + c[0];
        P.ldd = ldw;
        P.M = jb;
        P.N = c[1] - c[0];
        P.nterms = 1;
        P.naddends = 0;
        P.term[0] = term(Dinv, ldw, kOpN, R + (int64_t)j0 * ldr + c[0], ldr, kOpN, jb, +1);
      }
      b.nproblems = np;
      if ((err = launch_gemm_batch(b, stream)) != cudaSuccess) return err;
    }
    // 3. rank-jb update of the other rows:
    //    W[I,K] = R[I,K] - R[I,J] . W[J,K]   (K != J)
    //    W[I,J] = -R[I,J] . Dinv
    {
      GemmBatch b{};
      int np = 0;
      const int rows[2][2] = {{0, j0}, {j1, n}};
      const int cols[3][2] = {{0, j0}, {j1, n}, {j0, j1}};
      for (auto& r : rows) {
        if (r[1] <= r[0]) continue;
        for (int ci = 0; ci < 3; ++ci) {
          const int* c = cols[ci];
          if (c[1] <= c[0]) continue;
          GemmProblem& P = b.p[np++];
          P.D = W + (int64_t)r[0] * ldw + c[0];
          P.ldd = ldw;
          P.M = r[1] - r[0];
          P.N = c[1] - c[0];
          P.nterms = 1;
          const double2* RIJ = R + (int64_t)r[0] * ldr + j0;
          if (ci < 2) {
            P.naddends = 1;
            P.add[0].X = R + (int64_t)r[0] * ldr + c[0];
            P.add[0].ldx = ldr;
            P.add[0].sign = +1;
            P.term[0] = term(RIJ, ldr, kOpN, W + (int64_t)j0 * ldw + c[0], ldw, kOpN, jb, -1);
          } else {
            P.naddends = 0;
            P.term[0] = term(RIJ, ldr, kOpN, Dinv, ldw, kOpN, jb, -1);
          }
        }
      }
      b.nproblems = np;
      if ((err = launch_gemm_batch(b, stream)) != cudaSuccess) return err;
    }
    R = W;
    ldr = ldw;
  }
  // Exact fallback (no-op unless a leaf met an exactly zero pivot).
  const size_t smem = (size_t)n * (2 * sizeof(double2) + 2 * sizeof(int));
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    cudaFuncSetAttribute(exact_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  exact_inverse_kernel<<<1, 1024, smem, stream>>>(X, ldx, Y, ldy, n, work, flag, status, key);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsel
