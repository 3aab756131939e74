// Complex128 block inverse (see inverse.cuh).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>

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

// 32 x 32 Gauss-Jordan with partial pivoting by 256 threads, blocked in four
// sub-panels of 8 columns.  Thread t owns row i = t/8 and the columns
// t%8 + 8s (one per sub-panel s) IN REGISTERS for the whole elimination.
// A pivot step only updates the current sub-panel (one complex FMA per
// thread); the sub-panel is republished to shared memory after every step
// (double buffered), so pivot column, pivot row and multipliers all come
// from one buffer and a step needs a single __syncthreads.  After the 8
// steps of a sub-panel the other 24 columns receive the whole sub-panel at
// once: with G = G_8..G_1 the sub-panel's elementary transforms and P its
// pivot rows, x' = zero_rows_P(x) + G[:, P] x[P], and G[:, p_j] is exactly
// the sub-panel column j after its 8 steps.  Pivot search by every warp:
// redux.sync on the high word of |re|+|im| (monotone for non-negative
// doubles), lowest row on ties; virtual row interchanges tracked in a
// register bitmask.  Input in a (rows/cols < n); on return a holds S with
// inv(A)[r][piv[k]] = S[piv[r]][k].
constexpr int kSub = 8;               // sub-panel width
// BSEL_LEAF_UNROLL: unroll factor of a sub-panel's pivot steps (code size:
// fully unrolled, the leaf is ~7k instructions per call site)
#ifndef BSEL_LEAF_UNROLL
#define BSEL_LEAF_UNROLL 2
#endif
constexpr int kLeafUnroll = BSEL_LEAF_UNROLL;
constexpr int kPanLd = kSub + 1;      // padded: column reads hit 8 distinct bank groups
struct Leaf32 {
  double2 a[32][33];                  // input, then (after the elimination) the result S
  double2 pan[2][32][kPanLd];         // current sub-panel, double buffered
  double2 prow[kSub][3][kSub];        // pivot rows of the other three sub-panels
  int piv[32];
  int rowstep[32];                    // warp leaf: step of the sub-panel row i was pivot of, else -1
  int pstep[kSub];                    // warp leaf: pivot row of each step of the sub-panel
};

#ifndef BSEL_LEAF_NOINLINE
#define BSEL_LEAF_NOINLINE 0
#endif
#if BSEL_LEAF_NOINLINE
__device__ __noinline__
#else
__device__
#endif
bool gj_leaf32(Leaf32& L, int n, long long* trace = nullptr) {
  const int t = threadIdx.x, lane = t & 31;
  const int i = t >> 3, cl = t & 7;
  double2 v[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int c = cl + kSub * s;
    v[s] = (i < n && c < n) ? L.a[i][c] : make_double2(0.0, 0.0);
  }
  unsigned used = 0u;
  bool any_zero = false;
  int buf = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k0 = kSub * s;
    if (k0 >= n) break;
    if (trace && t == 0) trace[3 * s] = clock64();
    L.pan[buf][i][cl] = v[s];
    __syncthreads();
    const int steps = min(kSub, n - k0);
    int jp = -1;  // this row's step within the sub-panel if it was chosen as a pivot row
#pragma unroll kLeafUnroll
    for (int j = 0; j < kSub; ++j) {
      if (j >= steps) break;
      const int k = k0 + j;
      const double2 cv = L.pan[buf][lane][j];  // column k, row `lane`
      const bool cand = lane < n && !((used >> lane) & 1u);
      // Pivot key in integer ops only (no FP64 latency on the search): the
      // max-norm max(|re|, |im|) from the sign-cleared high words (monotone
      // for non-negative doubles), 5 low bits traded for the row so that ONE
      // redux.max yields the pivot row (lowest row among near-equal keys).
      const unsigned mag = max((unsigned)__double2hiint(cv.x) & 0x7fffffffu, (unsigned)__double2hiint(cv.y) & 0x7fffffffu);
      const unsigned key = cand ? (((mag >> 5) + 1u) << 5) | (31u - (unsigned)lane) : 0u;
      // Off the critical path: every lane inverts its own candidate while the
      // search runs; the pivot's reciprocal is then one shuffle away.
      const double2 rl = crecip_fast(cv);
      const double2 ci = make_double2(__shfl_sync(0xffffffffu, cv.x, i), __shfl_sync(0xffffffffu, cv.y, i));
      const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
      const int p = 31 - (int)(kmax & 31u);
      const bool zero = (kmax >> 5) <= 1u;  // all candidates zero (or subnormal): let the exact path decide
      any_zero |= zero;
      used |= 1u << p;
      if (p == i) jp = j;
      if (t == 0) L.piv[k] = p;
      const double2 pr = L.pan[buf][p][cl];
      const double2 rp = make_double2(__shfl_sync(0xffffffffu, rl.x, p), __shfl_sync(0xffffffffu, rl.y, p));
      const double2 inv = zero ? make_double2(1.0, 0.0) : rp;
      const double2 m = cmul(ci, inv);
      // pivot row: a'[p][c] = inv * a[p][c]; other rows: a'[i][c] = a[i][c] - m a[p][c];
      // column k: inv resp. -m.  One complex FMA per entry: a' = base + coef * a[p][c].
      const bool prow_ = i == p;
      const double2 coef = prow_ ? inv : make_double2(-m.x, -m.y);
      const double bx = prow_ ? 0.0 : v[s].x, by = prow_ ? 0.0 : v[s].y;
      double2 nv;
      nv.x = fma(coef.x, pr.x, fma(-coef.y, pr.y, bx));
      nv.y = fma(coef.x, pr.y, fma(coef.y, pr.x, by));
      if (cl == j) nv = coef;
      if (i < n && cl + k0 < n) v[s] = nv;
      buf ^= 1;
      L.pan[buf][i][cl] = v[s];
      __syncthreads();
    }
    if (trace && t == 0) trace[3 * s + 1] = clock64();
    // Lazy update of the other sub-panels: x' = zero_rows_P(x) + W x[P].
    // Unconditional 8-term sums (the loads pipeline): a short last
    // sub-panel has zero columns in pan and zero-filled pivot rows here.
    if (steps < kSub) {
      double2* pf = &L.prow[0][0][0];
      for (int e = t; e < kSub * 3 * kSub; e += blockDim.x)
        if (e / (3 * kSub) >= steps) pf[e] = make_double2(0.0, 0.0);
    }
    if (jp >= 0) {
#pragma unroll
      for (int o = 0, s2 = 0; s2 < 4; ++s2)
        if (s2 != s) L.prow[jp][o++][cl] = v[s2];
    }
    __syncthreads();
    double2 w[kSub];
#pragma unroll
    for (int j = 0; j < kSub; ++j) w[j] = L.pan[buf][i][j];
#pragma unroll
    for (int o = 0, s2 = 0; s2 < 4; ++s2) {
      if (s2 == s) continue;
      double2 acc = jp >= 0 ? make_double2(0.0, 0.0) : v[s2];
#pragma unroll
      for (int j = 0; j < kSub; ++j) {
        const double2 x = L.prow[j][o][cl];
        acc.x = fma(w[j].x, x.x, fma(-w[j].y, x.y, acc.x));
        acc.y = fma(w[j].x, x.y, fma(w[j].y, x.x, acc.y));
      }
      if (i < n && cl + kSub * s2 < n) v[s2] = acc;
      ++o;
    }
    buf ^= 1;  // next sub-panel starts in the other buffer (the lazy update still read this one)
    if (trace && t == 0) trace[3 * s + 2] = clock64();
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) L.a[i][cl + kSub * s] = v[s];
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
// Returns false (flag = 2 + row, status updated) if exactly singular.
__device__ bool exact_gj(const double2* __restrict__ X, int64_t ldx, double2* __restrict__ Y, int64_t ldy,
                         int n, double2* __restrict__ S, int* flag, unsigned long long* status,
                         unsigned long long key) {
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
      return false;
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
  __syncthreads();
  return true;
}

__global__ void __launch_bounds__(1024)
    exact_inverse_kernel(const double2* __restrict__ X, int64_t ldx, double2* __restrict__ Y, int64_t ldy,
                         int n, double2* __restrict__ S, int* flag, unsigned long long* status,
                         unsigned long long key) {
  if (*flag != 1) return;  // only after a fast-path zero pivot
  if (exact_gj(X, ldx, Y, ldy, n, S, flag, status, key) && threadIdx.x == 0) *flag = 0;
}

// Schur step fallback: exact inverse, then H = S U, F = L S, C -= F U by plain
// loops (one CTA; only runs when a leaf met an exactly zero pivot, in which
// case the fast kernel left C untouched).
__global__ void __launch_bounds__(1024)
    exact_schur_kernel(const double2* __restrict__ D, int64_t ldd, const double2* __restrict__ U, int64_t ldu,
                       const double2* __restrict__ Lm, int64_t ldl, double2* C, int64_t ldc, double2* Sout,
                       int64_t lds, double2* H, int64_t ldh, double2* F, int64_t ldf, int n, double2* scratch,
                       int* flag, unsigned long long* status, unsigned long long key) {
  if (*flag != 1) return;
  if (!exact_gj(D, ldd, Sout, lds, n, scratch, flag, status, key)) return;
  __threadfence_block();
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    double2 h = make_double2(0.0, 0.0), f = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) {
      const double2 s1 = Sout[(int64_t)r * lds + k], u = U[(int64_t)k * ldu + c];
      const double2 l = Lm[(int64_t)r * ldl + k], s2 = Sout[(int64_t)k * lds + c];
      h.x += s1.x * u.x - s1.y * u.y, h.y += s1.x * u.y + s1.y * u.x;
      f.x += l.x * s2.x - l.y * s2.y, f.y += l.x * s2.y + l.y * s2.x;
    }
    H[(int64_t)r * ldh + c] = h;
    F[(int64_t)r * ldf + c] = f;
  }
  __threadfence_block();
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    double2 v = C[(int64_t)r * ldc + c];
    for (int k = 0; k < n; ++k) {
      const double2 f = F[(int64_t)r * ldf + k], u = U[(int64_t)k * ldu + c];
      v.x -= f.x * u.x - f.y * u.y, v.y -= f.x * u.y + f.y * u.x;
    }
    C[(int64_t)r * ldc + c] = v;
  }
  if (threadIdx.x == 0) *flag = 0;
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

// grid-barrier poll back-off in ns (0 = spin)
#ifndef BSEL_BARRIER_SLEEP
#define BSEL_BARRIER_SLEEP 64
#endif
// DMMA accumulator sets per tile product (2: even / odd k steps, half-length
// chains -- measured neutral-to-slower in the cfg4 step, profiles/sweeps_r02.md)
#ifndef BSEL_TILE_ACC
#define BSEL_TILE_ACC 1
#endif
constexpr int kT = 32;
constexpr int kTLD = kT + 2;  // 544-byte rows: conflict-free DMMA fragment loads
// largest |re| + |im| of a block Gauss-Jordan multiplier accepted without the
// exact fallback (threshold pivoting with tau ~ 1/16)
constexpr double kMultMax = 16.0;

// Operand tiles double buffered: the next tile's loads fly while the
// current one computes (3 buffers, or the addend tile via smem, measured
// slower: 1 CTA/SM either way, more bytes in flight per SM).
struct PinvSmem {
  double2 d[kT][kTLD];     // Dinv
  double2 x[2][kT][kTLD];  // row-panel tiles W[J,K]; R = Dinv W[J,K] is formed from them
  double2 c[2][kT][kTLD];  // column-panel tiles W[I,J]
  double2 r[kT][kTLD];     // R of the current column
};

static_assert(sizeof(Leaf32) <= sizeof(PinvSmem::x), "leaf scratch must fit in PinvSmem::x");
static_assert(2048 * (2 * sizeof(double2) + 2 * sizeof(int)) <= sizeof(PinvSmem),
              "the dataflow kernel's in-kernel exact fallback (n <= 2048) must fit its shared memory");

__device__ __forceinline__ void inv_cp16(void* smem, const void* gmem, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void inv_cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void inv_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Asynchronous (L2, cp.async.cg) load of a kT x kT tile; zero-fill outside rows x cols.
__device__ __forceinline__ void load_tile_async(double2 (*dst)[kTLD], const double2* src, int64_t ld, int rows,
                                                int cols) {
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e / kT, j = e % kT;
    const bool ok = i < rows && j < cols;
    inv_cp16(&dst[i][j], ok ? src + (int64_t)i * ld + j : src, ok);
  }
}

__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
#if BSEL_BARRIER_SLEEP > 0
      if (v < target) __nanosleep(BSEL_BARRIER_SLEEP);
#endif
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// Dataflow flags (epoch-tagged u64, never reset): spin until *p >= target.
// Bounded: a flag that never arrives traps (a launch error) instead of
// hanging the GPU.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Publish a flag after the CTA's stores (callers: __syncthreads, then one
// thread): the release store is cumulative over the stores the barrier
// ordered before it (a preceding __threadfence, or fence.acq_rel + relaxed
// store, measured the same).
__device__ __forceinline__ void publish_flag(unsigned long long* p, unsigned long long v) { st_release(p, v); }
// Several flags after the CTA's stores: ONE fence, then relaxed stores (the
// release pattern; a release store per flag costs a MEMBAR each).
__device__ __forceinline__ void release_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Poll back-off: 32 ns (0 / 256 ns and relaxed polling with one final
// acquire measured the same, tools/build_sweep.sh).
__device__ __noinline__ void wait_ge_slow(const unsigned long long* p, unsigned long long target) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire(p) < target) {
    __nanosleep(32);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();  // 4 s: a lost flag, not a slow peer
  }
}
__device__ __forceinline__ void wait_ge(const unsigned long long* p, unsigned long long target) {
  if (ld_acquire(p) < target) wait_ge_slow(p, target);
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
  // BSEL_TILE_ACC independent accumulator sets (k steps round robin): the
  // latency-bound tiles of the inverse (lookahead tile, panel updates) see
  // dependent DMMA chains of 16 / BSEL_TILE_ACC steps (the DMMA dependent
  // latency is ~90 ns on B200, tools/inv_micro lookahead trace)
  constexpr int NA = BSEL_TILE_ACC;
  double accs[NA][4][2];
#pragma unroll
  for (int q = 0; q < NA; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) accs[q][j][0] = accs[q][j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kT / 2; ++kk) {
    const int kc = 2 * kk + kc0;
    const double af = A[kc * 2 + part];
    const double* Brow = reinterpret_cast<const double*>(&sB[kc][0]);
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      double bf = Brow[(col0 + jn * 4) * 2 + comp];
      int hi = __double2hiint(bf) ^ (int)maskB;
      bf = __hiloint2double(hi, __double2loint(bf));
      double(&c)[2] = accs[kk % NA][jn];
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[0]), "+d"(c[1])
                   : "d"(af), "d"(bf));
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[j][0] = accs[0][j][0];
    acc[j][1] = accs[0][j][1];
#pragma unroll
    for (int q = 1; q < NA; ++q) acc[j][0] += accs[q][j][0], acc[j][1] += accs[q][j][1];
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

// A square matrix of 1 x 1 or 2 x 2 quadrants of b x b blocks at separate
// addresses (quadrant (r, c) at index 2r + c).  Tile (ti, tk) of the tile grid
// (nq*ntq x nq*ntq, ntq = ceil(b/32) tiles per quadrant side) never straddles
// quadrants; edge tiles of each quadrant are partial.
struct Quad {
  double2* p[4];
  int64_t ld[4];
};

// As leaf_publish, with the diagonal tile already in shared memory.
__device__ void leaf_publish_smem(Leaf32& L, const double2 (*src)[kTLD], int jb, double2* gDp, int* flag,
                                  double2 (*dsmem)[kTLD] = nullptr, long long* trace = nullptr) {
  if (trace && threadIdx.x == 0) {
    trace[12] = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace[16]));
  }
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int i = e >> 5, j = e & 31;
    L.a[i][j] = (i < jb && j < jb) ? src[i][j] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[13] = clock64();
  const bool zero = gj_leaf32(L, jb, trace);
  if (trace && threadIdx.x == 0) trace[14] = clock64();
  if (threadIdx.x == 0 && zero) atomicMax(flag, 1);
  const double2 (*Sx)[33] = L.a;
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int r = e >> 5, k = e & 31;
    const int c = (r < jb && k < jb) ? L.piv[k] : k;
    const double2 v = (r < jb && k < jb) ? Sx[L.piv[r]][k] : make_double2(0.0, 0.0);
    gDp[r * kT + c] = v;
    if (dsmem) dsmem[r][c] = v;  // the publishing CTA keeps its copy (no reload through L2)
  }
  __syncthreads();
  if (trace && threadIdx.x == 0) {
    trace[15] = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace[17]));
  }
}

struct TileCtx {
  int b, ntq, nt, p, j0, jb;
  const Quad* Wc;  // current (in the __grid_constant__ kernel parameters)
  const Quad* Wn;  // next
  bool final_;      // this panel writes the caller's outputs
  bool skip_c;      // final: leave quadrant 3 untouched (fallback recomputes it)
  bool keep;        // lookahead tile: also leave the result in S.r for the leaf
  int r_tk;  // column tile whose R = Dinv W[J,K] is cached in S.r
  unsigned long long* trace;  // debug (may be null)
  int* flag;  // exact-fallback request (growth check, below)
  __device__ int quad(int ti, int tk) const { return 2 * (ti / ntq) + (tk / ntq); }
  __device__ int ext(int t) const { return min(kT, b - (t % ntq) * kT); }  // valid rows / cols of tile t
  __device__ double2* at(const Quad* Q, int ti, int tk) const {
    const int q = quad(ti, tk);
    return Q->p[q] + (int64_t)((ti % ntq) * kT) * Q->ld[q] + (tk % ntq) * kT;
  }
  __device__ int64_t ld(const Quad* Q, int ti, int tk) const { return Q->ld[quad(ti, tk)]; }
};

// Issue the asynchronous operand loads of output tile t into buffer `buf`:
// the column-panel tile W[I,J] and, at the first tile of a new column K,
// the row-panel tile W[J,K] that R = Dinv W[J,K] is formed from.
struct TileIssue {
  bool has_x;
  double2 w[4];  // epilogue operands W[I,K] of this thread's outputs (in flight)
};
__device__ __forceinline__ TileIssue issue_tile(PinvSmem& S, const TileCtx& T, int t, int buf, int& issued_r_tk) {
  const int tk = t / T.nt, ti = t % T.nt, p = T.p;
  const int ib = T.ext(ti), kb = T.ext(tk);
  TileIssue is;
  is.has_x = false;
  // Epilogue operands first: their L2 latency overlaps everything until the
  // tile's DMMA is done.
  const bool addend = ti != p && tk != p;
  const int orow = acc_row();
  const double2* wik = T.at(T.Wc, ti, tk);
  const int64_t ldik = T.ld(T.Wc, ti, tk);
#pragma unroll
  for (int jn = 0; jn < 4; ++jn) {
    const int oc = acc_col(jn);
    is.w[jn] = (addend && orow < ib && oc < kb) ? ldcg2(wik + (int64_t)orow * ldik + oc) : make_double2(0.0, 0.0);
  }
  if (!(ti == p && tk == p)) {
    if (tk != p && tk != issued_r_tk) {
      load_tile_async(S.x[buf], T.at(T.Wc, p, tk), T.ld(T.Wc, p, tk), T.jb, kb);
      is.has_x = true;
      issued_r_tk = tk;
    }
    if (ti != p) load_tile_async(S.c[buf], T.at(T.Wc, ti, p), T.ld(T.Wc, ti, p), ib, T.jb);
  }
  inv_cp_commit();
  return is;
}

// Compute output tile t from buffer `buf` (its loads have landed).
template <bool DF>
__device__ __forceinline__ void compute_tile(PinvSmem& S, TileCtx& T, int t, int buf, const TileIssue& is) {
  const int tk = t / T.nt, ti = t % T.nt, p = T.p;
  const int ib = T.ext(ti), kb = T.ext(tk);
  const int q = T.quad(ti, tk);
  double2* out = T.at(T.Wn, ti, tk);
  const int64_t ldn = T.ld(T.Wn, ti, tk);
  // final panel: quadrant 2 receives -(-L D^-1) = L D^-1; quadrant 3 is kept
  // when the exact fallback will recompute it
  const bool skip = T.final_ && T.skip_c && q == 3;
  const double sg = (T.final_ && q == 2) ? -1.0 : 1.0;
  const int orow = acc_row();
  double acc[4][2];
  if (ti == p && tk == p) {
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
      const int i = e >> 5, j = e & 31;
      if (i < ib && j < kb) out[(int64_t)i * ldn + j] = S.d[i][j];
    }
    return;
  }
  if (is.has_x) {  // R = Dinv . W[J,K]
    tile_mma(acc, S.d, S.x[buf]);
    if (T.trace && T.keep && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      T.trace[16 * T.p + 12] = v;
    }
    __syncthreads();  // previous readers of S.r are done
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) S.r[orow][acc_col(jn)] = make_double2(acc[jn][0], acc[jn][1]);
    __syncthreads();
    T.r_tk = tk;
  }
  if (ti == p) {  // W'[J,K] = R
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
      const int i = e >> 5, j = e & 31;
      if (i < ib && j < kb) out[(int64_t)i * ldn + j] = S.r[i][j];
    }
    return;
  }
  tile_mma(acc, S.c[buf], tk == p ? S.d : S.r);
  if (tk == p && ti > p && q == 0) {
    // Growth check (threshold pivoting): acc = W[I,p] Dinv_p are the
    // multipliers of rows not yet pivotal (pivot candidates of a full-column
    // search) against this panel's in-tile pivots.  Partial pivoting keeps
    // them <= 1; if any exceeds kMultMax the in-tile pivot was small for its
    // column and the exact full-column partial-pivoting inverse takes over
    // (same flag as an exactly zero leaf pivot).  Diagonally dominant pivots
    // (the RGF recursion's) give multipliers << 1.
    bool big = false;
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) big |= fabs(acc[jn][0]) + fabs(acc[jn][1]) > kMultMax;
    if (__syncthreads_or(big) && threadIdx.x == 0) atomicMax(T.flag, 1);
  }
  if (T.keep) {  // the next leaf reads this tile from shared memory, not back through L2
    __syncthreads();  // every warp is done reading S.r
#pragma unroll
    for (int jn = 0; jn < 4; ++jn)
      S.r[orow][acc_col(jn)] = make_double2(is.w[jn].x - acc[jn][0], is.w[jn].y - acc[jn][1]);
  }
  if (skip || (DF && T.keep)) return;  // dataflow: the lookahead tile lives in S.r only
#pragma unroll
  for (int jn = 0; jn < 4; ++jn) {
    const int oc = acc_col(jn);
    if (orow < ib && oc < kb)
      out[(int64_t)orow * ldn + oc] = make_double2(sg * (is.w[jn].x - acc[jn][0]), sg * (is.w[jn].y - acc[jn][1]));
  }
}

// One pipeline stage: wait for tile t's operands (slot B), start tile tn's
// loads into slot B ^ 1, compute t.  B is a template constant so the two
// in-flight TileIssue register sets never have to be copied (a copy would
// wait for the in-flight epilogue loads).
template <int B, bool DF = false>
__device__ __forceinline__ void gj_stage(PinvSmem& S, TileCtx& T, int t, int tn, int t1, int t0,
                                         const TileIssue& cur, TileIssue& nxt, int& issued_r_tk) {
  const bool lk = T.trace && T.keep && blockIdx.x == 0 && threadIdx.x == 0;  // debug: lookahead phases
  auto gt = [] {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  };
  if (lk) T.trace[16 * T.p + 8] = gt();
  if (tn < t1) {
    nxt = issue_tile(S, T, tn, B ^ 1, issued_r_tk);
    inv_cp_wait<1>();
  } else {
    inv_cp_wait<0>();
  }
  __syncthreads();
  if (lk) T.trace[16 * T.p + 9] = gt();
  const bool tr = T.trace && blockIdx.x == 1 && threadIdx.x == 0 && t == t0;  // debug stamps
  unsigned long long g0 = 0, g1 = 0;
  if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  compute_tile<DF>(S, T, t, B, cur);
  __syncthreads();  // slot B is refilled by the next stage's issue
  if (lk) T.trace[16 * T.p + 10] = gt();
  if (tr) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    T.trace[16 * T.p + 6] = g0, T.trace[16 * T.p + 7] = g1;
  }
}

// Output tiles [t0, t1) of the Gauss-Jordan update of panel p (tile `skip`
// excluded), software pipelined: the operands of the next tile stream in
// (cp.async, double buffered) while the current one computes.
template <bool DF = false>
__device__ void gj_tiles(PinvSmem& S, TileCtx& T, int t0, int t1, int skip) {
  auto next = [&](int t) { ++t; return t == skip ? t + 1 : t; };
  int t = t0 == skip ? t0 + 1 : t0;
  if (t >= t1) return;
  int issued_r_tk = T.r_tk;
  __syncthreads();  // smem buffers free (previous panel / leaf)
  TileIssue a, b;
  if (T.trace && T.keep && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    T.trace[16 * T.p + 11] = v;
  }
  a = issue_tile(S, T, t, 0, issued_r_tk);
  b.has_x = false;
  while (true) {
    int tn = next(t);
    gj_stage<0, DF>(S, T, t, tn, t1, t0, a, b, issued_r_tk);
    if (tn >= t1) break;
    t = tn;
    tn = next(t);
    gj_stage<1, DF>(S, T, t, tn, t1, t0, b, a, issued_r_tk);
    if (tn >= t1) break;
    t = tn;
  }
}

// Dataflow variant of gj_tiles: the tiles of [t0, t1) (minus `skip`) in two
// passes -- first the "hot" ones (row / column p+1 and the tile (p+2, p+2):
// the sources of the next panel and of CTA 0's next lookahead tile), then the
// rest -- one software pipeline across both passes.  After the last hot tile
// ONE fence publishes all hot tiles' ready flags (ver[t] = done).  Positions
// k in [0, 2 len): pass k / len, tile t0 + k % len.
__device__ void gj_tiles_df(PinvSmem& S, TileCtx& T, int t0, int t1, int skip, unsigned long long* ver,
                            unsigned long long done) {
  const int len = t1 - t0, p = T.p, nt = T.nt;
  auto hot = [&](int t) {
    const int tk = t / nt, ti = t % nt;
    return ti == p + 1 || tk == p + 1 || (ti == p + 2 && tk == p + 2);
  };
  auto tile = [&](int k) { return t0 + (k >= len ? k - len : k); };
  auto next = [&](int k) {  // next position whose tile belongs to its pass
    for (++k; k < 2 * len; ++k) {
      const int t = tile(k);
      if (t != skip && hot(t) == (k < len)) break;
    }
    return k;
  };
  int k = next(-1);
  if (k >= 2 * len) return;
  const bool flags = ver != nullptr;
  int issued_r_tk = T.r_tk;
  __syncthreads();  // smem buffers free (previous panel)
  TileIssue a, b;
  a = issue_tile(S, T, tile(k), 0, issued_r_tk);
  b.has_x = false;
  auto publish_hot = [&](int kk, int kn) {  // after the last hot tile: flags of every hot tile
    if (flags && kk < len && kn >= len && threadIdx.x == 0) {
      release_fence();  // orders every hot tile's stores (ordered before it by the stage's barrier)
      for (int t = t0; t < t1; ++t)
        if (t != skip && hot(t)) st_relaxed(ver + t, done);
    }
  };
  constexpr int kNone = 1 << 30;
  while (true) {
    int kn = next(k);
    gj_stage<0, true>(S, T, tile(k), kn < 2 * len ? tile(kn) : kNone, kNone, -1, a, b, issued_r_tk);
    publish_hot(k, kn);
    if (kn >= 2 * len) break;
    k = kn;
    kn = next(k);
    gj_stage<1, true>(S, T, tile(k), kn < 2 * len ? tile(kn) : kNone, kNone, -1, b, a, issued_r_tk);
    publish_hot(k, kn);
    if (kn >= 2 * len) break;
    k = kn;
  }
}

// Persistent blocked Gauss-Jordan over the pivot columns of quadrant 0:
// nq = 1: Y = inv(X).  nq = 2: the Schur step of the forward sweep,
//   [[D, U], [L, C]] -> [[D^-1, D^-1 U], [L D^-1, C - L D^-1 U]]
// (pivot rows and columns only in D; the L rows and U columns are eliminated
// along, so the chain's two GEMMs f = L S, C -= f U become part of the GJ
// panel updates, which overlap the latency-bound leaf factorizations).
// Buffers: panel 0 reads IN; the last panel writes OUT; the panels before it
// alternate between B (last-but-one) and A.  A may share quadrants with OUT
// except the one OUT shares with IN (C, updated in place).
// Lookahead: during panel p, CTA 0 first computes the next diagonal tile
// W'[p+1,p+1], immediately factors it and publishes Dinv_{p+1} (double-
// buffered gD) while the other CTAs update the rest -> one grid barrier per
// panel, the leaf latency hidden behind the update.
// launch_bounds(256, 2): <= 128 registers, so a CTA can share an SM with a
// GEMM CTA of the concurrent sweeps.
struct GjArgs {
  Quad in, out, a, bq;
  int b, nq;
  double2* gD;
  unsigned* barrier;
  int* flag;
  unsigned long long* trace;
  unsigned long long* stats;  // BSEL_INV_STATS: phase totals (ns) over all launches, may be null
};

#if BSEL_INV_STATS
#define LEAF_TRACE_DECL __shared__ long long s_leaf_tr[18];
#define LEAF_TRACE (g.stats ? s_leaf_tr : nullptr)
#define LEAF_TRACE_ACC                                                              \
  if (g.stats && threadIdx.x == 0)                                                  \
    for (int q = 0; q < 4; ++q) {                                                   \
      atomicAdd(g.stats + kStSteps, (unsigned long long)(s_leaf_tr[3 * q + 1] - s_leaf_tr[3 * q])); \
      atomicAdd(g.stats + kStLazy, (unsigned long long)(s_leaf_tr[3 * q + 2] - s_leaf_tr[3 * q + 1])); \
      if (q == 0) {                                                                 \
        atomicAdd(g.stats + kStPro, (unsigned long long)(s_leaf_tr[13] - s_leaf_tr[12])); \
        atomicAdd(g.stats + kStCore, (unsigned long long)(s_leaf_tr[14] - s_leaf_tr[13])); \
        atomicAdd(g.stats + kStEpi, (unsigned long long)(s_leaf_tr[15] - s_leaf_tr[14])); \
        atomicAdd(g.stats + kStLeafNs, (unsigned long long)(s_leaf_tr[17] - s_leaf_tr[16])); \
      }                                                                             \
    }
#else
#define LEAF_TRACE_DECL
#define LEAF_TRACE nullptr
#define LEAF_TRACE_ACC
#endif
// Build with -DBSEL_INV_STATS=1 and run with BSEL_INV_STATS=1: slots (summed over launches, globaltimer ns): CTA 0 per panel
// lookahead tile / leaf / wait at the barrier, CTA 1 tile updates / wait,
// whole kernel (CTA 0 first stamp -> exit), launches, panels.
#ifndef BSEL_INV_STATS
#define BSEL_INV_STATS 0
#endif
enum InvStat { kStLook = 0, kStLeaf, kStWait0, kStTiles1, kStWait1, kStKernel, kStLaunches, kStPanels, kStPub, kStCoLoc, kStSteps, kStLazy, kStPro, kStCore, kStEpi, kStLeafNs,
               kStMark = 280, kStFirst = 298, kStLast, kStSpread, kStCta0Late, kStCta0LateSum,
               kStSm = 16, kStN = 304 };

__global__ void __launch_bounds__(256, 2) persistent_gj_kernel(const __grid_constant__ GjArgs g) {
  // trace (debug, may be null): per panel p, [8p+0] CTA0 start, [+1] after the
  // lookahead tile, [+2] after the leaf, [+3] CTA0 at barrier, [+4] CTA1 done
  // with its tiles, [+5] CTA1 after barrier (globaltimer ns).
  auto stamp = [&](int slot) {
    if (g.trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g.trace[slot] = t;
    }
  };
  auto now = [] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
#if BSEL_INV_STATS
  const bool st = g.stats && threadIdx.x == 0 && blockIdx.x < 2;
#else
  constexpr bool st = false;  // instrumentation compiled out (it costs registers)
#endif
  unsigned long long st_t = st ? now() : 0;
  auto lap = [&](int slot) {  // time since the previous lap into `slot`
    if (st) {
      const unsigned long long t = now();
      atomicAdd(g.stats + slot, t - st_t);
      st_t = t;
    }
  };
  if (st && blockIdx.x == 0) {
    atomicAdd(g.stats + kStKernel, 0ull - st_t);
    atomicAdd(g.stats + kStLaunches, 1ull);
    atomicAdd(g.stats + kStPanels, (unsigned long long)((g.b + kT - 1) / kT));
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PinvSmem& S = *reinterpret_cast<PinvSmem*>(smem_raw);
  Leaf32& L = *reinterpret_cast<Leaf32*>(&S.x[0][0][0]);  // spans x[0] and x[1]
  LEAF_TRACE_DECL
  const int b = g.b, ntq = (b + kT - 1) / kT, nt = g.nq * ntq, ntiles = nt * nt, G = gridDim.x;
  unsigned target = 0;
  if (blockIdx.x == 0) leaf_publish(L, g.in.p[0], g.in.ld[0], 0, min(kT, b), g.gD, g.flag);
  target += G;
  grid_barrier(g.barrier, target);
  TileCtx T;
  T.keep = false;
  T.trace = g.trace;
  T.flag = g.flag;
  T.b = b;
  T.ntq = ntq;
  T.nt = nt;
  T.Wc = &g.in;
  const int workers = G > 1 ? G - 1 : 1, wid = G > 1 ? (int)blockIdx.x - 1 : 0;
  for (int p = 0; p < ntq; ++p) {
    T.p = p;
    T.j0 = p * kT;
    T.jb = min(kT, b - T.j0);
    const int rem = ntq - 1 - p;  // panels after this one
    T.final_ = rem == 0;
    T.Wn = rem == 0 ? &g.out : (rem % 2 == 1 ? &g.bq : &g.a);
    // every leaf (the last one was factored during panel ntq-2) has reported
    T.skip_c = T.final_ && g.nq == 2 && *reinterpret_cast<volatile int*>(g.flag) != 0;
    T.r_tk = -1;
    // CTA 0 (with other CTAs updating the tiles) already holds Dinv_p in
    // S.d: it factored the leaf itself (lookahead) and kept the result
    if (!(blockIdx.x == 0 && G > 1 && p > 0)) load_tile(S.d, g.gD + (p & 1) * kT * kT, kT, kT, kT);
    __syncthreads();
    const int sp = (p + 1 < ntq) ? (p + 1) * nt + (p + 1) : -1;
    if (blockIdx.x == 0) stamp(16 * p + 0);
    lap(blockIdx.x == 0 ? kStWait0 : kStWait1);
    if (blockIdx.x == 0 && sp >= 0) {
      T.keep = true;
      gj_tiles(S, T, sp, sp + 1, -1);
      T.keep = false;
      T.r_tk = -1;  // S.r now holds the tile, not an R
      __syncthreads();
      stamp(16 * p + 1);
      lap(kStLook);
      // S.d is free once the lookahead tile is done (CTA 0 updates no other
      // tiles when G > 1): keep Dinv_{p+1} there for the next panel
      leaf_publish_smem(L, S.r, min(kT, b - (p + 1) * kT), g.gD + ((p + 1) & 1) * kT * kT, g.flag,
                        G > 1 ? S.d : nullptr, LEAF_TRACE);
      LEAF_TRACE_ACC
      stamp(16 * p + 2);
      lap(kStLeaf);
    }
    if (G == 1 || blockIdx.x > 0) {
      const int chunk = (ntiles + workers - 1) / workers;
      const int t0 = wid * chunk, t1 = min(ntiles, t0 + chunk);
      gj_tiles(S, T, t0, t1, G == 1 ? -1 : sp);
    }
    if (blockIdx.x == 0) stamp(16 * p + 3);
    if (blockIdx.x == 1) stamp(16 * p + 4);
    if (blockIdx.x == 1) lap(kStTiles1);
    target += G;
    grid_barrier(g.barrier, target);
    if (blockIdx.x == 1) stamp(16 * p + 5);
    T.Wc = T.Wn;
  }
  lap(blockIdx.x == 0 ? kStWait0 : kStWait1);
  if (st && blockIdx.x == 0) atomicAdd(g.stats + kStKernel, st_t);
}


// ---------------------------------------------------------------------------
// Dataflow persistent Gauss-Jordan (nq = 1, the chain's block inverse): the
// per-panel grid barrier of persistent_gj_kernel replaced by ready flags.
//
// Measured (BSEL_INV_STATS, b = 512): with the barrier every panel costs
// max(CTA 0's lookahead tile + leaf, the slowest worker's tiles) + barrier;
// under the concurrent GEMM levels the workers' tiles (22 us per panel on
// one GPU with two lanes) and the leaf path (20 us) alternate as the
// slower side, and neither overlaps the other's panel.  Here:
//  * CTA 0 runs ahead: lookahead tile (p+1, p+1) (its three source tiles'
//    flags), leaf, publish Dinv_{p+1} into its own slot (one slot per
//    panel: no reuse), flag dv = p + 2 -- it never waits for the bulk of
//    panel p.
//  * Workers (fixed tile ranges) start panel p once Dinv_p is out, wait per
//    tile for the flags of its two foreign source tiles (row-panel (p, K),
//    column-panel (I, p)), do their "hot" tiles (the next panel's sources)
//    first and publish them with one fence, then the rest.
//  * Three rotating n x n buffers (panel p reads R(p) = W(p-1), writes
//    W(p); the last panel writes Y, R(0) = X).  W(p) reuses W(p-3)'s
//    buffer, last read during panel p-2: a worker starts panel p only when
//    every worker has reported panel p-2 done (per-CTA progress flags; CTA
//    0's reads of R(p-2) precede its publication of Dinv_p).
// Flags are u64 = epoch * 256 + version (epoch: a process-wide launch
// counter) in a zero-initialised sync area at the start of the workspace,
// so they are never reset.
// ---------------------------------------------------------------------------
constexpr int kSyncTiles = 4096;  // (2048 / kT)^2 tile flags: b <= 2048
constexpr int kSyncCtas = 256;
constexpr int64_t kSyncElems = (kSyncTiles + 1 + kSyncCtas + 1) / 2;  // in double2 units

struct DfArgs {
  unsigned long long* stats;  // BSEL_INV_STATS (instrumented builds), may be null
  Quad in, y, s1, s2;  // nq = 1 quads (p[0], ld[0])
  double2* dinv;       // ntq slots of kT x kT
  unsigned long long* ver;   // tile flags [nt * nt]
  unsigned long long* dv;    // Dinv_p published: *dv >= base + p + 1
  unsigned long long* prog;  // per-CTA progress: panel p done -> base + p + 1
  unsigned long long base;   // epoch * 256
  int b;
  int* flag;
  unsigned long long* status;  // exact fallback (in-kernel): singular -> atomicMin(status, key)
  unsigned long long key;
};

__global__ void __launch_bounds__(256, 2) dataflow_gj_kernel(const __grid_constant__ DfArgs g) {
  // Programmatic dependent launch (launch_dataflow): the CTAs may be placed
  // while the previous kernel of the stream (the chain GEMM producing X)
  // still runs; nothing is read before it has completed and flushed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PinvSmem& S = *reinterpret_cast<PinvSmem*>(smem_raw);
  Leaf32& L = *reinterpret_cast<Leaf32*>(&S.x[0][0][0]);  // spans x[0] and x[1]
  LEAF_TRACE_DECL
  const int b = g.b, nt = (b + kT - 1) / kT, ntiles = nt * nt, G = gridDim.x;
  const unsigned long long base = g.base;
  // instrumentation (-DBSEL_INV_STATS=1): CTA 0 source waits / lookahead /
  // leaf, CTA 1 wait phase / tiles (the InvStat slots)
#if BSEL_INV_STATS
  const bool st = g.stats && threadIdx.x == 0 && blockIdx.x < 2;
#else
  constexpr bool st = false;
#endif
  unsigned long long st_t = 0;
  auto lap = [&](int slot) {
    if (st) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (slot >= 0) atomicAdd(g.stats + slot, t - st_t);
      st_t = t;
    }
  };
  lap(-1);
#if BSEL_INV_STATS
  if (g.stats && threadIdx.x == 0) {  // CTA start spread of this launch (one lane per process only)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) {  // gap since the previous chain kernel ended (marks: [0] end, [4] gap, [5] count)
      const unsigned long long prev = atomicAdd(g.stats + kStMark, 0ull);
      if (prev && t > prev && t - prev < 10000000ull) {
        atomicAdd(g.stats + kStMark + 4, t - prev);
        atomicAdd(g.stats + kStMark + 5, 1ull);
      }
    }
    atomicMin(g.stats + kStFirst, t);
    atomicMax(g.stats + kStLast, t);
    if (blockIdx.x == 0) atomicExch(g.stats + kStCta0Late, t);
  }
  if (g.stats && threadIdx.x == 0) {  // CTAs per SM of this launch (co-location check)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    atomicAdd(g.stats + kStSm + (smid & 255), 1ull);
    if (blockIdx.x == 0) atomicExch(g.stats + kStCoLoc, (unsigned long long)smid);
  }
#endif
  if (st && blockIdx.x == 0) {
    atomicAdd(g.stats + kStKernel, 0ull - st_t);
    atomicAdd(g.stats + kStLaunches, 1ull);
    atomicAdd(g.stats + kStPanels, (unsigned long long)((g.b + kT - 1) / kT));
  }
  // W(p): the last panel writes Y, earlier ones rotate backwards over Y, s1, s2
  auto wbuf = [&](int p) -> const Quad* {
    const int r = (nt - 1 - p) % 3;
    return r == 0 ? &g.y : r == 1 ? &g.s1 : &g.s2;
  };
  TileCtx T;
  T.trace = nullptr;
  T.flag = g.flag;
  T.b = b;
  T.ntq = nt;
  T.nt = nt;
  T.skip_c = false;
  if (blockIdx.x == 0) {
    // ---- CTA 0: leaf 0, then per panel the lookahead tile + leaf ----
    leaf_publish(L, g.in.p[0], g.in.ld[0], 0, min(kT, b), g.dinv, g.flag);
    // keep Dinv_0 in S.d for the first lookahead
    for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) S.d[e >> 5][e & 31] = ldcg2(g.dinv + e);
    __syncthreads();
    if (threadIdx.x == 0) publish_flag(g.dv, base + 1);
    lap(kStLeaf);
    for (int p = 0; p + 1 < nt; ++p) {
      T.p = p;
      T.j0 = p * kT;
      T.jb = min(kT, b - T.j0);
      T.final_ = false;
      T.Wc = p == 0 ? &g.in : wbuf(p - 1);
      T.Wn = wbuf(p);
      T.r_tk = -1;
      T.keep = true;
      const int sp = (p + 1) * nt + (p + 1);
      // sources of the lookahead tile at version p (panel 0 reads the input):
      // (p+1, p+1), row-panel (p, p+1), column-panel (p+1, p)
      if (p > 0 && threadIdx.x < 3) {
        const int src = threadIdx.x == 0 ? sp : threadIdx.x == 1 ? (p + 1) * nt + p : p * nt + (p + 1);
        wait_ge(g.ver + src, base + p);
      }
      __syncthreads();
      lap(kStWait0);
      gj_tiles<true>(S, T, sp, sp + 1, -1);
      T.keep = false;
      __syncthreads();
      lap(kStLook);
      leaf_publish_smem(L, S.r, min(kT, b - (p + 1) * kT), g.dinv + (int64_t)(p + 1) * kT * kT, g.flag,
                        S.d, LEAF_TRACE);
      LEAF_TRACE_ACC
      lap(kStLeaf);
      if (threadIdx.x == 0) publish_flag(g.dv, base + p + 2);
      lap(kStPub);
    }
    // Exact fallback in-kernel (no separate launch per inverse: under the
    // concurrent GEMM levels a 1024-thread fallback CTA waited for an SM on
    // every chain step).  Once every worker is past its last panel (growth
    // flags are raised during the panels, the last one wrote Y), a flagged
    // inverse is recomputed from X by full-column partial pivoting.
    if (threadIdx.x >= 1 && threadIdx.x < G) wait_ge(g.prog + threadIdx.x, base + nt);
    __syncthreads();
    int fl;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(fl) : "l"(g.flag) : "memory");
    if (fl == 1 && exact_gj(g.in.p[0], g.in.ld[0], g.y.p[0], g.y.ld[0], b, g.s1.p[0], g.flag, g.status, g.key) &&
        threadIdx.x == 0)
      *g.flag = 0;
    if (st) atomicAdd(g.stats + kStKernel, st_t);
#if BSEL_INV_STATS
    if (g.stats && threadIdx.x == 0) {  // every CTA has started (all reported their last panel)
      const unsigned long long f = atomicExch(g.stats + kStFirst, ~0ull), l = atomicExch(g.stats + kStLast, 0ull);
      atomicAdd(g.stats + kStSpread, l - f);
      const unsigned long long c0 = atomicAdd(g.stats + kStCta0Late, 0ull);
      atomicAdd(g.stats + kStCta0LateSum, c0 - f);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(g.stats + kStMark, t);
    }
#endif
    return;
  }
  // ---- workers: fixed tile ranges ----
  const int workers = G - 1, wid = blockIdx.x - 1;
  const int chunk = (ntiles + workers - 1) / workers;
  const int t0 = min(ntiles, wid * chunk), t1 = min(ntiles, t0 + chunk);
  for (int p = 0; p < nt; ++p) {
    const int sp = (p + 1 < nt) ? (p + 1) * nt + (p + 1) : -1;
    // One wait phase per panel (each flag polled by one thread, released to
    // the CTA by the barrier): W(p) reuses the buffer read during panel p-2
    // (every CTA must be past it); Dinv_p; the source tiles of this range at
    // version p -- column-panel (ti, p) per tile, row-panel (p, tk) per column.
    const int tid = threadIdx.x;
    // (CTA 0 has no progress flag: Dinv_p -- waited for below -- is published
    // after its lookahead of panel p-1, i.e. after its reads of R(p-2))
    if (p >= 2 && tid > 0 && tid < G) wait_ge(g.prog + tid, base + p - 1);
    if (tid == 255) wait_ge(g.dv, base + p + 1);
    if (p > 0 && tid >= 128 && tid < 160) {
      for (int j = tid - 128; j < t1 - t0; j += 32) {
        const int t = t0 + j, tk = t / nt, ti = t % nt;
        if (ti != p && t != sp) wait_ge(g.ver + p * nt + ti, base + p);
        // (also when the column's first tile here is the skipped lookahead
        // tile: the column's other tiles form R from (p, tk))
        if ((j == 0 || ti == 0) && tk != p) wait_ge(g.ver + tk * nt + p, base + p);
      }
    }
    __syncthreads();
    // Dinv_p arrives asynchronously with the first tile's operands (its
    // cp.async group completes before that tile computes)
    load_tile_async(S.d, g.dinv + (int64_t)p * kT * kT, kT, kT, kT);
    inv_cp_commit();
    if (blockIdx.x == 1) lap(kStWait1);
    T.p = p;
    T.j0 = p * kT;
    T.jb = min(kT, b - T.j0);
    T.final_ = p == nt - 1;
    T.Wc = p == 0 ? &g.in : wbuf(p - 1);
    T.Wn = wbuf(p);
    T.r_tk = -1;
    T.keep = false;
    gj_tiles_df(S, T, t0, t1, sp, T.final_ ? nullptr : g.ver, base + p + 1);
    inv_cp_wait<0>();  // (a range without tiles never waited for its Dinv copy)
    __syncthreads();
    if (threadIdx.x == 0) st_release(g.prog + blockIdx.x, base + p + 1);
    if (blockIdx.x == 1) lap(kStTiles1);
  }
}
}  // namespace

// work: n*n ping-pong buffer (also the exact fallback's scratch), then the
// published Dinv tiles (2 x kT*kT, double-buffered) and the grid-barrier counter.
unsigned long long* g_inverse_trace = nullptr;

namespace {
// BSEL_INV_STATS=1: per-phase totals of every persistent inverse of the
// process, printed to stderr at exit (one buffer per process, device 0 of
// the first launch; the analysis tool, not a product path).
unsigned long long* inverse_stats() {
  static unsigned long long* buf = [] {
    const char* e = getenv("BSEL_INV_STATS");
    unsigned long long* p = nullptr;
    if (!(e && atoi(e) != 0)) return p;
    if (cudaMallocManaged(&p, kStN * sizeof(unsigned long long)) != cudaSuccess) return (unsigned long long*)nullptr;
    memset(p, 0, kStN * sizeof(unsigned long long));
    p[kStFirst] = ~0ull;
    atexit([] {
      unsigned long long* q = inverse_stats();
      if (!q || cudaDeviceSynchronize() != cudaSuccess) return;
      const double n = q[kStLaunches] ? (double)q[kStLaunches] : 1.0;
      int multi = 0, used = 0;
      for (int k = 0; k < 256; ++k) used += q[kStSm + k] > 0, multi += q[kStSm + k] > q[kStLaunches];
      fprintf(stderr, "[inverse stats] chain gaps: before an inverse %.1f us (%llu), before a chain GEMM %.1f us (%llu)\n",
              q[kStMark + 5] ? q[kStMark + 4] / (double)q[kStMark + 5] / 1e3 : 0.0, q[kStMark + 5],
              q[kStMark + 3] ? q[kStMark + 2] / (double)q[kStMark + 3] / 1e3 : 0.0, q[kStMark + 3]);
      fprintf(stderr, "[inverse stats] CTA start spread per launch %.1f us (CTA 0 after the first CTA by %.1f us)\n",
              q[kStSpread] / n / 1e3, q[kStCta0LateSum] / n / 1e3);
      fprintf(stderr, "[inverse stats] leaf per launch: pivot steps %.0f kcycles, lazy updates %.0f kcycles | "
              "prologue %.0f, core %.0f, epilogue %.0f kcycles; leaf_publish_smem %.1f us (globaltimer)\n",
              q[kStSteps] / n / 1e3, q[kStLazy] / n / 1e3, q[kStPro] / n / 1e3, q[kStCore] / n / 1e3,
              q[kStEpi] / n / 1e3, q[kStLeafNs] / n / 1e3);
      fprintf(stderr, "[inverse stats] SMs used %d, SMs hosting > 1 CTA per launch on average %d, CTA0's last SM %llu "
              "hosted %.2f CTAs per launch\n", used, multi, q[kStCoLoc], q[kStSm + (q[kStCoLoc] & 255)] / n);
      fprintf(stderr,
              "[inverse stats] launches %llu panels/launch %.1f | per launch us: kernel %.1f | CTA0 lookahead %.1f "
              "leaf %.1f wait %.1f publish %.1f | CTA1 tiles %.1f wait %.1f\n",
              q[kStLaunches], q[kStPanels] / n, q[kStKernel] / n / 1e3, q[kStLook] / n / 1e3, q[kStLeaf] / n / 1e3,
              q[kStWait0] / n / 1e3, q[kStPub] / n / 1e3, q[kStTiles1] / n / 1e3, q[kStWait1] / n / 1e3);
    });
    return p;
  }();
  return buf;
}
}  // namespace

unsigned long long* chain_marks() {
#if BSEL_INV_STATS
  unsigned long long* q = inverse_stats();
  return q ? q + kStMark : nullptr;
#else
  return nullptr;
#endif
}

// Layout: [sync area: kSyncElems (zero at allocation, epoch-tagged flags of
// the dataflow kernel)][scratch].  Scratch: dataflow kernel s1, s2 (n x n
// each) + Dinv slots (ntq x kT x kT); barrier kernel: n x n ping-pong, 2 Dinv
// tiles, barrier counter; exact fallback: n x n.
int64_t block_inverse_workspace(int n) {
  const int64_t ntq = (n + kT - 1) / kT;
  return kSyncElems + std::max<int64_t>(2 * (int64_t)n * n + ntq * kT * kT, (int64_t)n * n + 2 * kT * kT + 1);
}


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
  return per_device([] {
    int dev = 0, coop = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (cudaFuncSetAttribute(persistent_gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(PinvSmem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persistent_gj_kernel, 256,
                                                      sizeof(PinvSmem)) != cudaSuccess)
      per_sm = 0;
    return coop ? per_sm * device_sm_count() : 0;
  });
}

Quad quad1(const double2* p, int64_t ld) {
  Quad q{};
  q.p[0] = const_cast<double2*>(p);
  q.ld[0] = ld;
  return q;
}

// BSEL_INV_DATAFLOW=0 selects the barrier kernel for the block inverse
// (A/B experiments); default: the dataflow kernel.
bool dataflow_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSEL_INV_DATAFLOW");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

std::atomic<unsigned long long> g_inverse_epoch{0};

// BSEL_INV_PDL=1 (experiment): launch the dataflow kernel as a programmatic
// dependent of the previous kernel.  Measured slower (2 GPUs 495 vs 466 ms,
// 1 GPU 810 vs 781): the launch gap before the inverse drops from ~62 to
// ~15 us, but its early-placed CTAs slow the inverse itself and the GEMMs.
bool dataflow_pdl() {
  static const bool on = [] {
    const char* e = getenv("BSEL_INV_PDL");
    return e && atoi(e) != 0;
  }();
  return on;
}

// BSEL_INV_DF_COOP=1: cooperative launch of the dataflow kernel (experiment).
bool dataflow_coop() {
  static const bool on = [] {
    const char* e = getenv("BSEL_INV_DF_COOP");
    return e && atoi(e) != 0;
  }();
  return on;
}

cudaError_t launch_dataflow(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n, double2* sync,
                            double2* scratch, int* flag, unsigned long long* status, unsigned long long key,
                            int grid, cudaStream_t stream) {
  const cudaError_t attr = per_device([] {
    return cudaFuncSetAttribute(dataflow_gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(PinvSmem));
  });
  if (attr != cudaSuccess) return attr;
  const int ntq = (n + kT - 1) / kT;
  DfArgs g{};
  g.in = quad1(const_cast<double2*>(X), ldx);
  g.y = quad1(Y, ldy);
  g.s1 = quad1(scratch, n);
  g.s2 = quad1(scratch + (int64_t)n * n, n);
  g.dinv = scratch + 2 * (int64_t)n * n;
  unsigned long long* f = reinterpret_cast<unsigned long long*>(sync);
  g.ver = f;
  g.dv = f + kSyncTiles;
  g.prog = f + kSyncTiles + 1;
  g.base = (g_inverse_epoch.fetch_add(1) + 1) << 8;
  g.b = n;
  g.flag = flag;
  g.status = status;
  g.key = key;
  g.stats = inverse_stats();
  (void)ntq;
  cudaError_t err;
  if (dataflow_coop()) {
    void* args[] = {(void*)&g};
    err = cudaLaunchCooperativeKernel((const void*)dataflow_gj_kernel, grid, 256, args, sizeof(PinvSmem), stream);
  } else {
    // Under the concurrent GEMM levels the inverse starts ~62 us after the
    // previous chain GEMM ended (2 GPUs, chain marks of the instrumented
    // build: its CTAs need 104 KB of shared memory on SMs the persistent
    // aux-level GEMM CTAs hold).  BSEL_INV_PDL=1 launches it as a
    // programmatic dependent of that GEMM (which signals launch_dependents
    // on entry) -- measured slower, see dataflow_pdl.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = sizeof(PinvSmem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = dataflow_pdl() ? 1 : 0;
    err = cudaLaunchKernelEx(&cfg, dataflow_gj_kernel, g);
  }
  count_launch();
  return err;
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

namespace {

cudaError_t launch_gj(GjArgs& g, int grid, cudaStream_t stream) {
  // (A warp-resident leaf measured 2x slower -- 22.6 vs 11.0 us per 32x32
  // leaf, profiles/inverse_leaf_r02.md -- and was removed in round 2: its
  // runtime switch tripled the kernels' code.)
  g.stats = inverse_stats();
  if ((cudaError_t)cudaMemsetAsync(g.barrier, 0, sizeof(unsigned), stream) != cudaSuccess) return cudaGetLastError();
  // The CTAs wait on one another (grid barrier), so the launch is
  // cooperative: co-residency of the whole grid is guaranteed.  Cooperative
  // launches from different streams are serialized by the driver, which
  // makes the inverses of concurrent lanes wait for each other (SI, 2 lanes:
  // 454 us per inverse with plain launches vs 666 us cooperative; SI+SQ
  // forward 564 vs 578 ms).  BSEL_INV_COOP=0 (experiment) uses a plain launch:
  // all CTAs still become resident in practice (grid <= occupancy limit and
  // the concurrent GEMM levels never wait on the inverse) but nothing
  // guarantees it.
  static const bool coop = [] {
    const char* e = getenv("BSEL_INV_COOP");
    return !(e && atoi(e) == 0);
  }();
  // BSEL_INV_SMEM (bytes, experiment): request more shared memory per CTA
  // than the kernel uses, so that no GEMM CTA can share an SM with it.
  const size_t smem = per_device([] {
    const char* e = getenv("BSEL_INV_SMEM");
    size_t v = e ? (size_t)atoll(e) : 0;
    if (v < sizeof(PinvSmem)) v = sizeof(PinvSmem);
    if (v != sizeof(PinvSmem)) cudaFuncSetAttribute(persistent_gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v);
    return v;
  });
  cudaError_t err;
  if (coop) {
    void* args[] = {(void*)&g};
    err = cudaLaunchCooperativeKernel((const void*)persistent_gj_kernel, grid, 256, args, smem, stream);
  } else {
    persistent_gj_kernel<<<grid, 256, smem, stream>>>(g);
    err = cudaGetLastError();
  }
  count_launch();
  return err;
}

cudaError_t launch_exact_fallback_attr() {
  return per_device([] {  // thread-safe one-time init per device, sized for n <= 2048
    const cudaError_t a1 =
        cudaFuncSetAttribute(exact_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const cudaError_t a2 =
        cudaFuncSetAttribute(exact_schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return a1 != cudaSuccess ? a1 : a2;
  });
}
}  // namespace

cudaError_t launch_block_inverse(const double2* X, int64_t ldx, double2* Y, int64_t ldy, int n,
                                 double2* work, int* flag, unsigned long long* status,
                                 unsigned long long key, cudaStream_t stream, int grid_req) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  double2* sync = work;
  work += kSyncElems;
  const int panels = (n + kLeaf - 1) / kLeaf;
  const int limit = coop_grid_limit();
  if (panels > 1 && limit > 0) {
    int grid = panels * panels < limit ? panels * panels : limit;
    const int cap = grid_req > 0 ? grid_req : inverse_grid_cap();
    if (grid > cap) grid = cap;
    if (dataflow_enabled() && grid >= 2 && grid <= kSyncCtas && panels * panels <= kSyncTiles) {
      // the exact fallback runs inside the dataflow kernel (n <= 2048: its
      // n * 40 B of shared memory fit the kernel's)
      return launch_dataflow(X, ldx, Y, ldy, n, sync, work, flag, status, key, grid, stream);
    }
    GjArgs g{};
    g.in = quad1(X, ldx);
    g.out = g.a = quad1(Y, ldy);
    g.bq = quad1(work, n);
    g.b = n;
    g.nq = 1;
    g.gD = work + (int64_t)n * n;
    g.barrier = reinterpret_cast<unsigned*>(g.gD + 2 * kT * kT);
    g.flag = flag;
    g.trace = g_inverse_trace;
    err = launch_gj(g, grid, stream);
  } else {
    err = levels_inverse(X, ldx, Y, ldy, n, work, flag, stream);
  }
  if (err != cudaSuccess) return err;
  // Exact fallback (no-op unless a leaf met an exactly zero pivot).
  const size_t smem = (size_t)n * (2 * sizeof(double2) + 2 * sizeof(int));
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if ((err = launch_exact_fallback_attr()) != cudaSuccess) return err;
  exact_inverse_kernel<<<1, 1024, smem, stream>>>(X, ldx, Y, ldy, n, work, flag, status, key);
  count_launch();
  return cudaGetLastError();
}

int64_t schur_step_workspace(int b) { return kSyncElems + 6 * (int64_t)b * b + 2 * kT * kT + 1; }

bool schur_step_supported(int b) { return b > kLeaf && coop_grid_limit() > 0; }

cudaError_t launch_schur_step(const double2* D, int64_t ldd, const double2* U, int64_t ldu, const double2* Lm,
                              int64_t ldl, double2* C, int64_t ldc, double2* Sout, int64_t lds, double2* H,
                              int64_t ldh, double2* F, int64_t ldf, int b, double2* work, int* flag,
                              unsigned long long* status, unsigned long long key, cudaStream_t stream,
                              int grid_req) {
  if (!schur_step_supported(b)) return cudaErrorInvalidValue;
  const int64_t bb = (int64_t)b * b;
  work += kSyncElems;  // the sync area belongs to the dataflow inverse
  double2* w = work;  // w0..w3 (B buffer), wc (A's C quadrant), wh (H if none given)
  if (!H) H = w + 5 * bb, ldh = b;
  GjArgs g{};
  const double2* inp[4] = {D, U, Lm, C};
  const int64_t inl[4] = {ldd, ldu, ldl, ldc};
  double2* outp[4] = {Sout, H, F, C};
  const int64_t outl[4] = {lds, ldh, ldf, ldc};
  for (int q = 0; q < 4; ++q) {
    g.in.p[q] = const_cast<double2*>(inp[q]), g.in.ld[q] = inl[q];
    g.out.p[q] = outp[q], g.out.ld[q] = outl[q];
    g.a.p[q] = q == 3 ? w + 4 * bb : outp[q], g.a.ld[q] = q == 3 ? b : outl[q];
    g.bq.p[q] = w + q * bb, g.bq.ld[q] = b;
  }
  g.b = b;
  g.nq = 2;
  g.gD = w + 6 * bb;
  g.barrier = reinterpret_cast<unsigned*>(g.gD + 2 * kT * kT);
  g.flag = flag;
  g.trace = g_inverse_trace;
  const int ntq = (b + kT - 1) / kT;
  int grid = std::min(4 * ntq * ntq, coop_grid_limit());
  static const int cap_env = [] {
    const char* e = getenv("BSEL_SCHUR_GRID");
    return e ? atoi(e) : 128;
  }();
  const int cap = grid_req > 0 ? grid_req : cap_env;
  if (cap > 0 && grid > cap) grid = cap;
  cudaError_t err = launch_gj(g, grid, stream);
  if (err != cudaSuccess) return err;
  const size_t smem = (size_t)b * (2 * sizeof(double2) + 2 * sizeof(int));
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if ((err = launch_exact_fallback_attr()) != cudaSuccess) return err;
  exact_schur_kernel<<<1, 1024, smem, stream>>>(D, ldd, U, ldu, Lm, ldl, C, ldc, Sout, lds, H, ldh, F, ldf, b, w,
                                                 flag, status, key);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsel
