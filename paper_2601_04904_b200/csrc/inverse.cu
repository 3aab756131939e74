// Complex128 block inverse (see inverse.cuh).
#include <cstdlib>

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

// 1/z via one correctly rounded reciprocal of |z|^2 (operands here are O(1)
// pivots of diagonally dominant blocks; the exact fallback handles the rest).
__device__ __forceinline__ double2 crecip_fast(double2 z) {
  const double r = __drcp_rn(fma(z.x, z.x, z.y * z.y));
  return make_double2(z.x * r, -z.y * r);
}

// 32 x 32 Gauss-Jordan with partial pivoting by 256 threads.  Thread t owns
// row t/8, columns 4*(t%8) .. +3 IN REGISTERS for the whole elimination;
// per pivot step only the pivot column (for the search and the row
// multipliers) and the pivot row go through shared memory (the row buffer is
// skewed so the 4 reads per thread are conflict-free broadcasts).  Pivot
// search by every warp: redux.sync on the high word of |re|+|im| (monotone
// for non-negative doubles), lowest row on ties; virtual row interchanges
// tracked in a register bitmask.  Input in a (rows/cols < n); on return a
// holds S with inv(A)[r][piv[k]] = S[piv[r]][k].
struct Leaf32 {
  double2 a[32][33];  // input, then (after the elimination) the result S
  double2 col[2][32];
  double2 row[2][32];
  int piv[32];
};

__device__ __forceinline__ int row_slot(int c) { return (c & 3) * 8 + (c >> 2); }

__device__ bool gj_leaf32(Leaf32& L, int n) {
  const int t = threadIdx.x, lane = t & 31;
  const int i = t >> 3, c0 = (t & 7) * 4;
  double2 v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    v[q] = (i < n && c0 + q < n) ? L.a[i][c0 + q] : make_double2(0.0, 0.0);
  if ((t & 7) == 0) L.col[0][i] = v[0];
  __syncthreads();
  unsigned used = 0u;
  bool any_zero = false;
  for (int k = 0; k < n; ++k) {
    const int buf = k & 1;
    const bool cand = lane < n && !((used >> lane) & 1u);
    const unsigned key = cand ? (unsigned)__double2hiint(cabs1(L.col[buf][lane])) + 1u : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned ball = __ballot_sync(0xffffffffu, cand && key == kmax);
    const int p = __ffs(ball) - 1;
    const bool zero = kmax <= 1u;  // all candidates zero (or subnormal): let the exact path decide
    any_zero |= zero;
    used |= 1u << p;
    if (t == 0) L.piv[k] = p;
    if (i == p) {
#pragma unroll
      for (int q = 0; q < 4; ++q) L.row[buf][row_slot(c0 + q)] = v[q];
    }
    const double2 inv = zero ? make_double2(1.0, 0.0) : crecip_fast(L.col[buf][p]);
    const double2 m = cmul(L.col[buf][i], inv);
    __syncthreads();
    // pivot row: a'[p][c] = inv * a[p][c]; other rows: a'[i][c] = a[i][c] - m a[p][c];
    // column k: inv resp. -m.  One complex FMA per entry: a' = base + coef * a[p][c].
    const bool prow = i == p;
    const double2 coef = prow ? inv : make_double2(-m.x, -m.y);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + q;
      const double2 pr = L.row[buf][row_slot(c)];
      const double bx = prow ? 0.0 : v[q].x, by = prow ? 0.0 : v[q].y;
      double2 nv;
      nv.x = fma(coef.x, pr.x, fma(-coef.y, pr.y, bx));
      nv.y = fma(coef.x, pr.y, fma(coef.y, pr.x, by));
      if (c == k) nv = coef;
      if (c < n && i < n) v[q] = nv;
    }
    const int q1 = k + 1 - c0;  // publish column k+1 (static selects keep v[] in registers)
    if (q1 >= 0 && q1 < 4) L.col[buf ^ 1][i] = q1 == 0 ? v[0] : q1 == 1 ? v[1] : q1 == 2 ? v[2] : v[3];
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) L.a[i][c0 + q] = v[q];
  __syncthreads();
  return any_zero;
}

// One CTA (256 threads) per matrix, n <= 32.
__global__ void __launch_bounds__(256)
    leaf_inverse_kernel(const double2* __restrict__ X, int64_t ldx, int64_t sx, double2* __restrict__ Y,
                        int64_t ldy, int64_t sy, int n, int* flags, int64_t flag_stride) {
  __shared__ Leaf32 L;
  const int tid = threadIdx.x;
  X += blockIdx.x * sx;
  Y += blockIdx.x * sy;
  int* flag = flags + blockIdx.x * flag_stride;
  for (int e = tid; e < 32 * 32; e += 256) {
    int i = e >> 5, j = e & 31;
    if (i < n && j < n) L.a[i][j] = X[(int64_t)i * ldx + j];
  }
  __syncthreads();
  const bool any_zero = gj_leaf32(L, n);
  if (tid == 0 && any_zero) atomicMax(flag, 1);
  const double2 (*S)[33] = L.a;
  for (int e = tid; e < 32 * 32; e += 256) {
    int r = e >> 5, k = e & 31;
    if (r < n && k < n) Y[(int64_t)r * ldy + L.piv[k]] = S[L.piv[r]][k];
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

// ---------------------------------------------------------------------------
// Persistent blocked Gauss-Jordan: ONE cooperative launch per inverse.
//
// For each 32-wide panel J: CTA 0 inverts the diagonal tile W[J,J] with
// partial pivoting (gj_leaf) and publishes Dinv; after a grid barrier every
// CTA updates its 32x32 output tiles with DMMA from shared memory:
//   W'[J,J] = Dinv, W'[J,K] = Dinv W[J,K], W'[I,J] = -W[I,J] Dinv,
//   W'[I,K] = W[I,K] - W[I,J] (Dinv W[J,K]),
// ping-ponging between two n x n buffers (the last panel writes Y).  Global
// reads of the ping-pong buffers use ld.global.cg (L2) because other SMs
// rewrote them since this SM may have cached them in L1.
// ---------------------------------------------------------------------------

constexpr int kT = 32;
constexpr int kTLD = kT + 2;  // 544-byte rows: conflict-free DMMA fragment loads

struct PinvSmem;
struct PinvSmem {
  double2 d[kT][kTLD];  // Dinv
  double2 x[kT][kTLD];  // row-panel tile W[J,K] -> R = Dinv W[J,K]
  double2 c[kT][kTLD];  // column-panel tile W[I,J]
  double2 r[kT][kTLD];
};

static_assert(sizeof(Leaf32) <= 2 * sizeof(double2) * kT * kTLD, "leaf scratch must fit in PinvSmem::x and ::c");

__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      if (v < target) __nanosleep(64);
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// Load a kT x kT tile (rows x cols valid, zero elsewhere) into smem.
__device__ __forceinline__ void load_tile(double2 (*dst)[kTLD], const double2* src, int64_t ld, int rows, int cols) {
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e / kT, j = e % kT;
    dst[i][j] = (i < rows && j < cols) ? ldcg2(src + (int64_t)i * ld + j) : make_double2(0.0, 0.0);
  }
}

// acc (warp tile 8 x 16 complex) = sA (32 x 32) . sB (32 x 32), DMMA.
__device__ __forceinline__ void tile_mma(double (&acc)[4][2], const double2 (*sA)[kTLD], const double2 (*sB)[kTLD]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mg = warp & 3, nh = warp >> 2;
  const unsigned maskB = ((lane & 1) == 1 && ((lane >> 2) & 1) == 0) ? 0x80000000u : 0u;
  const double* A = reinterpret_cast<const double*>(&sA[mg * 8 + (lane >> 2)][0]);
  const int kc0 = (lane & 3) >> 1, part = lane & 1;
  const int comp = (lane & 1) ^ ((lane >> 2) & 1);
  const int col0 = nh * 16 + ((lane >> 2) >> 1);
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < kT / 2; ++kk) {
    const int kc = 2 * kk + kc0;
    const double af = A[kc * 2 + part];
    const double* Brow = reinterpret_cast<const double*>(&sB[kc][0]);
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      double bf = Brow[(col0 + jn * 4) * 2 + comp];
      int hi = __double2hiint(bf) ^ (int)maskB;
      bf = __hiloint2double(hi, __double2loint(bf));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[jn][0]), "+d"(acc[jn][1])
                   : "d"(af), "d"(bf));
    }
  }
}

// Warp-tile coordinates of acc[jn]: row, col inside the 32 x 32 tile.
__device__ __forceinline__ int acc_row() { return ((threadIdx.x >> 5) & 3) * 8 + ((threadIdx.x & 31) >> 2); }
__device__ __forceinline__ int acc_col(int jn) { return ((threadIdx.x >> 5) >> 2) * 16 + jn * 4 + (threadIdx.x & 3); }

// CTA-wide: invert the diagonal tile W[j0:j0+jb, j0:j0+jb] and publish the
// zero-padded 32 x 32 Dinv to gDp.
__device__ void leaf_publish(Leaf32& L, const double2* W, int64_t ld, int j0, int jb, double2* gDp, int* flag) {
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e >> 5, j = e & 31;
    L.a[i][j] = (i < jb && j < jb) ? ldcg2(W + (int64_t)(j0 + i) * ld + j0 + j) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const bool zero = gj_leaf32(L, jb);
  if (threadIdx.x == 0 && zero) atomicMax(flag, 1);
  const double2 (*S)[33] = L.a;
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int r = e >> 5, k = e & 31;
    if (r < jb && k < jb)
      gDp[r * kT + L.piv[k]] = S[L.piv[r]][k];
    else
      gDp[r * kT + k] = make_double2(0.0, 0.0);
  }
  __syncthreads();
}

struct TileCtx {
  int n, nt, p, j0, jb;
  const double2* Wc;
  int64_t ldc;
  double2* Wn;
  int64_t ldn;
  int r_tk;  // column tile whose R = Dinv W[J,K] is cached in S.r
};

// One 32 x 32 output tile of the Gauss-Jordan update of panel p.
__device__ void gj_tile(PinvSmem& S, TileCtx& T, int t) {
  const int tk = t / T.nt, ti = t % T.nt, p = T.p;
  const int i0 = ti * kT, k0 = tk * kT;
  const int ib = min(kT, T.n - i0), kb = min(kT, T.n - k0);
  double acc[4][2];
  double2* out = T.Wn + (int64_t)i0 * T.ldn + k0;
  const int orow = acc_row();
  if (ti == p && tk == p) {
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
      const int i = e >> 5, j = e & 31;
      if (i < ib && j < kb) out[(int64_t)i * T.ldn + j] = S.d[i][j];
    }
    return;
  }
  if (tk != p && T.r_tk != tk) {  // R = Dinv . W[J,K]
    __syncthreads();
    load_tile(S.x, T.Wc + (int64_t)T.j0 * T.ldc + k0, T.ldc, T.jb, kb);
    __syncthreads();
    tile_mma(acc, S.d, S.x);
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) S.r[orow][acc_col(jn)] = make_double2(acc[jn][0], acc[jn][1]);
    __syncthreads();
    T.r_tk = tk;
  }
  if (ti == p) {  // W'[J,K] = R
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
      const int i = e >> 5, j = e & 31;
      if (i < ib && j < kb) out[(int64_t)i * T.ldn + j] = S.r[i][j];
    }
    return;
  }
  __syncthreads();
  load_tile(S.c, T.Wc + (int64_t)i0 * T.ldc + T.j0, T.ldc, ib, T.jb);
  __syncthreads();
  tile_mma(acc, S.c, tk == p ? S.d : S.r);
#pragma unroll
  for (int jn = 0; jn < 4; ++jn) {
    const int oc = acc_col(jn);
    if (orow < ib && oc < kb) {
      double2 v = make_double2(-acc[jn][0], -acc[jn][1]);
      if (tk != p) {
        const double2 w = ldcg2(T.Wc + (int64_t)(i0 + orow) * T.ldc + k0 + oc);
        v.x += w.x;
        v.y += w.y;
      }
      out[(int64_t)orow * T.ldn + oc] = v;
    }
  }
}

// Lookahead: during panel p, CTA 0 first computes the next diagonal tile
// W'[p+1,p+1], immediately factors it and publishes Dinv_{p+1} (double-
// buffered gD) while the other CTAs update the rest -> one grid barrier per
// panel, the leaf latency hidden behind the update.
__global__ void __launch_bounds__(256, 1)
    persistent_inverse_kernel(const double2* __restrict__ X, int64_t ldx, double2* Y, int64_t ldy, int n,
                              double2* work, double2* gD, unsigned* barrier, int* flag,
                              unsigned long long* trace) {
  // trace (debug, may be null): per panel p, [8p+0] CTA0 start, [+1] after the
  // lookahead tile, [+2] after the leaf, [+3] CTA0 at barrier, [+4] CTA1 done
  // with its tiles, [+5] CTA1 after barrier (globaltimer ns).
  auto stamp = [&](int slot) {
    if (trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[slot] = t;
    }
  };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PinvSmem& S = *reinterpret_cast<PinvSmem*>(smem_raw);
  Leaf32& L = *reinterpret_cast<Leaf32*>(&S.x[0][0]);  // spans x and c
  const int nt = (n + kT - 1) / kT, ntiles = nt * nt, G = gridDim.x;
  unsigned target = 0;
  if (blockIdx.x == 0) leaf_publish(L, X, ldx, 0, min(kT, n), gD, flag);
  target += G;
  grid_barrier(barrier, target);
  TileCtx T;
  T.n = n;
  T.nt = nt;
  T.Wc = X;
  T.ldc = ldx;
  const int workers = G > 1 ? G - 1 : 1, wid = G > 1 ? (int)blockIdx.x - 1 : 0;
  for (int p = 0; p < nt; ++p) {
    T.p = p;
    T.j0 = p * kT;
    T.jb = min(kT, n - T.j0);
    T.Wn = ((nt - 1 - p) % 2 == 0) ? Y : work;
    T.ldn = (T.Wn == Y) ? ldy : n;
    T.r_tk = -1;
    load_tile(S.d, gD + (p & 1) * kT * kT, kT, kT, kT);
    __syncthreads();
    const int sp = (p + 1 < nt) ? (p + 1) * nt + (p + 1) : -1;
    if (blockIdx.x == 0) stamp(8 * p + 0);
    if (blockIdx.x == 0 && sp >= 0) {
      gj_tile(S, T, sp);
      __syncthreads();
      stamp(8 * p + 1);
      leaf_publish(L, T.Wn, T.ldn, (p + 1) * kT, min(kT, n - (p + 1) * kT), gD + ((p + 1) & 1) * kT * kT, flag);
      stamp(8 * p + 2);
    }
    if (G == 1 || blockIdx.x > 0) {
      const int chunk = (ntiles + workers - 1) / workers;
      const int t0 = wid * chunk, t1 = min(ntiles, t0 + chunk);
      for (int t = t0; t < t1; ++t)
        if (t != sp || G == 1) gj_tile(S, T, t);
    }
    if (blockIdx.x == 0) stamp(8 * p + 3);
    if (blockIdx.x == 1) stamp(8 * p + 4);
    target += G;
    grid_barrier(barrier, target);
    if (blockIdx.x == 1) stamp(8 * p + 5);
    T.Wc = T.Wn;
    T.ldc = T.ldn;
  }
}

}  // namespace

// work: n*n ping-pong buffer (also the exact fallback's scratch), then the
// published Dinv tiles (2 x kT*kT, double-buffered) and the grid-barrier counter.
unsigned long long* g_inverse_trace = nullptr;

int64_t block_inverse_workspace(int n) { return (int64_t)n * n + 2 * kT * kT + 1; }

namespace {
// CTAs of the persistent inverse.  Default 64: fewer CTAs become co-resident
// sooner while the aux stream's GEMM tiles hold SMs (measured on cfg4: 64
// beats 148/96/32).  BSEL_INV_GRID overrides.
int inverse_grid_cap() {
  static const int cap = [] {
    const char* e = getenv("BSEL_INV_GRID");
    int c = e ? atoi(e) : 64;
    return (c <= 0 || c > device_sm_count()) ? device_sm_count() : c;
  }();
  return cap;
}

int coop_grid_limit() {
  static const int limit = [] {
    int dev = 0, coop = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (cudaFuncSetAttribute(persistent_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(PinvSmem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persistent_inverse_kernel, 256,
                                                      sizeof(PinvSmem)) != cudaSuccess)
      per_sm = 0;
    return coop ? per_sm * device_sm_count() : 0;
  }();
  return limit;
}
}  // namespace

cudaError_t launch_leaf_inverse_batched(const double2* X, int64_t ldx, int64_t strideX, double2* Y,
                                        int64_t ldy, int64_t strideY, int n, int batch, int* flags,
                                        cudaStream_t stream) {
  if (n <= 0 || batch <= 0) return cudaSuccess;
  if (n > kLeaf) return cudaErrorInvalidValue;
  leaf_inverse_kernel<<<batch, kLeafThreads, 0, stream>>>(X, ldx, strideX, Y, ldy, strideY, n, flags, 1);
  count_launch();
  return cudaGetLastError();
}

namespace {

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

// Multi-launch variant (no cooperative launch available): per panel one leaf
// kernel and two grouped GEMM launches.
cudaError_t levels_inverse(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n, double2* work,
                           int* flag, cudaStream_t stream) {
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
    leaf_inverse_kernel<<<1, kLeafThreads, 0, stream>>>(
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
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_block_inverse(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n,
                                 double2* work, int* flag, unsigned long long* status,
                                 unsigned long long key, cudaStream_t stream, int grid_req) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  const int panels = (n + kLeaf - 1) / kLeaf;
  const int limit = coop_grid_limit();
  if (panels > 1 && limit > 0) {
    double2* gD = work + (int64_t)n * n;
    unsigned* barrier = reinterpret_cast<unsigned*>(gD + 2 * kT * kT);
    if ((err = cudaMemsetAsync(barrier, 0, sizeof(unsigned), stream)) != cudaSuccess) return err;
    int grid = panels * panels < limit ? panels * panels : limit;
    const int cap = grid_req > 0 ? grid_req : inverse_grid_cap();
    if (grid > cap) grid = cap;
    unsigned long long* trace = g_inverse_trace;
    void* args[] = {(void*)&X, (void*)&ldx, (void*)&Y, (void*)&ldy, (void*)&n,
                    (void*)&work, (void*)&gD, (void*)&barrier, (void*)&flag, (void*)&trace};
    err = cudaLaunchCooperativeKernel((const void*)persistent_inverse_kernel, grid, 256, args, sizeof(PinvSmem),
                                      stream);
    count_launch();
  } else {
    err = levels_inverse(X, ldx, Y, ldy, n, work, flag, stream);
  }
  if (err != cudaSuccess) return err;
  // Exact fallback (no-op unless a leaf met an exactly zero pivot).
  const size_t smem = (size_t)n * (2 * sizeof(double2) + 2 * sizeof(int));
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static const cudaError_t smem_attr =  // thread-safe one-time init, sized for n <= 2048
      cudaFuncSetAttribute(exact_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (smem_attr != cudaSuccess) return smem_attr;
  exact_inverse_kernel<<<1, 1024, smem, stream>>>(X, ldx, Y, ldy, n, work, flag, status, key);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsel
