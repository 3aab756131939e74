// Device generator for the reference's synthetic inputs (matrix.py:192-284).
//
// The splitmix64 stream is a pure function of (seed, position), so every
// complex entry is generated independently: entry e of the concatenated
// stream diag | lower | upper | arrow_row | arrow_col | tip uses positions
// 2e+1 (re) and 2e+2 (im).  This is bit-identical to the host generator.
// The dominance shift needs |row| sums across blocks; they are accumulated
// in numpy's pairwise order with numpy's rounding of the shift (see
// pairwise_abs / shift_entry) and numpy's complex absolute (cabs_), so the
// shifted diagonal matches the host generator bit for bit.
#include <cstdint>

#include "generate.cuh"
#include "zgemm.cuh"

namespace bsel {

namespace {

__device__ __forceinline__ double splitmix_uniform(uint64_t seed, uint64_t pos) {
  uint64_t z = seed + pos * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1.0p-52 - 1.0;
}

__global__ void fill_uniform_kernel(double2* out, int64_t count, uint64_t seed, uint64_t first_entry) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = 2 * (first_entry + (uint64_t)e);
    out[e] = make_double2(splitmix_uniform(seed, p + 1), splitmix_uniform(seed, p + 2));
  }
}

// |z| exactly as numpy's SIMD complex absolute (numpy 2.x, AVX2 / AVX-512
// hosts) computes it: larger * sqrt(fma(r, r, 1)) with r = smaller / larger
// (checked bit for bit against np.abs on 2e5 random entries; libm hypot
// differs from it in ~35 % of the last bits).
__device__ __forceinline__ double cabs_(double2 z) {
  const double ax = fabs(z.x), ay = fabs(z.y);
  const double mx = fmax(ax, ay), mn = fmin(ax, ay);
  if (mx == 0.0) return 0.0;
  const double r = __ddiv_rn(mn, mx);
  return __dmul_rn(mx, __dsqrt_rn(__fma_rn(r, r, 1.0)));
}

// numpy's pairwise summation (umath loops_utils pairwise_sum) of |x_j| over
// a contiguous run of n complex entries: below 8 a plain loop, up to 128
// eight interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// plus the tail, above that the two halves (first half rounded down to a
// multiple of 8) summed recursively.  The reference's np.abs(X).sum(axis=1)
// row sums (matrix.py:262-282) therefore come out with numpy's rounding.
__device__ double pairwise_abs(const double2* x, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, cabs_(x[i]));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = cabs_(x[j]);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], cabs_(x[i + j]));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, cabs_(x[i]));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_abs(x, n2), pairwise_abs(x + n2, n - n2));
}

// d + dominance (rs + 1) phase(d), evaluated as numpy does: phase = d / |d|
// by numpy's complex division (Smith's form: d * (1/|d|) for a real
// divisor), then a real x complex product and a complex add, each rounded
// separately (no FMA contraction).
__device__ __forceinline__ double2 shift_entry(double2 v, double rs, double dominance) {
  const double mag = cabs_(v);
  double px = 1.0, py = 0.0;
  if (mag > 0) {
    const double scl = __drcp_rn(mag);
    px = __dmul_rn(v.x, scl);
    py = __dmul_rn(v.y, scl);
  }
  const double shift = __dmul_rn(dominance, __dadd_rn(rs, 1.0));
  return make_double2(__dadd_rn(v.x, __dmul_rn(shift, px)), __dadd_rn(v.y, __dmul_rn(shift, py)));
}

// One thread per global diagonal row r = i*b + row: the reference's
// off-diagonal |row| sum (rs = sum(|diag row|) - |d|, then + lower[i-1] row,
// + upper[i] row, + arrow_col[i] row, matrix.py:271-279), then the shift.
__global__ void dominance_rows_kernel(BtaDevView m, double dominance) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m.n * m.b) return;
  const int64_t i = r / m.b, row = r % m.b, b = m.b, a = m.a;
  const double2* d = m.diag + i * b * b + row * b;
  double s = __dadd_rn(pairwise_abs(d, b), -cabs_(d[row]));
  if (i > 0) s = __dadd_rn(s, pairwise_abs(m.lower + (i - 1) * b * b + row * b, b));
  if (i < m.n - 1) s = __dadd_rn(s, pairwise_abs(m.upper + i * b * b + row * b, b));
  if (a > 0) s = __dadd_rn(s, pairwise_abs(m.arrow_col + i * b * a + row * a, a));
  double2* dd = m.diag + i * b * b + row * b + row;
  *dd = shift_entry(*dd, s, dominance);
}

__global__ void dominance_tip_kernel(BtaDevView m, double dominance) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t a = m.a, b = m.b;
  if (row >= a) return;
  const double2* t = m.tip + row * a;
  double s = __dadd_rn(pairwise_abs(t, a), -cabs_(t[row]));
  for (int64_t i = 0; i < m.n; ++i) s = __dadd_rn(s, pairwise_abs(m.arrow_row + i * a * b + row * b, b));
  double2* dd = m.tip + row * a + row;
  *dd = shift_entry(*dd, s, dominance);
}

// (X + X^H)/2 on the pattern (matrix.py:337-354); out-of-place pairs.
__global__ void herm_pair_kernel(double2* x, double2* y, int64_t count, int r, int c) {
  // x: [count][r][c], y: [count][c][r]; x' = (x + y^H)/2, y' = (y + x^H)/2
  const int64_t total = count * (int64_t)r * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)r * c), rem = e % ((int64_t)r * c);
    const int64_t i = rem / c, j = rem % c;
    double2* px = x + k * r * c + i * c + j;
    double2* py = y + k * r * c + j * r + i;
    if (x == y && j < i) continue;  // same array (square diagonal blocks): handle each pair once
    const double2 u = *px, w = *py;
    *px = make_double2(0.5 * (u.x + w.x), 0.5 * (u.y - w.y));
    if (px != py) *py = make_double2(0.5 * (w.x + u.x), 0.5 * (w.y - u.y));
  }
}

int blocks_for(int64_t count) {
  int64_t b = (count + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t generate_dd_bta_device(const BtaDevView& m, uint64_t seed, double dominance, cudaStream_t s) {
  const int64_t n = m.n, b = m.b, a = m.a;
  struct Seg {
    double2* p;
    int64_t count;
  } segs[6] = {{m.diag, n * b * b},         {m.lower, (n - 1) * b * b}, {m.upper, (n - 1) * b * b},
               {m.arrow_row, n * a * b}, {m.arrow_col, n * b * a},  {m.tip, a * a}};
  uint64_t entry = 0;
  for (auto& sg : segs) {
    if (sg.count > 0) {
      fill_uniform_kernel<<<blocks_for(sg.count), 256, 0, s>>>(sg.p, sg.count, seed, entry);
      count_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    entry += (uint64_t)sg.count;
  }
  dominance_rows_kernel<<<(unsigned)((n * b + 127) / 128), 128, 0, s>>>(m, dominance);
  if (a > 0) dominance_tip_kernel<<<(unsigned)((a + 127) / 128), 128, 0, s>>>(m, dominance);
  return cudaGetLastError();
}

cudaError_t hermitianize_device(const BtaDevView& m, cudaStream_t s) {
  const int64_t n = m.n, b = m.b, a = m.a;
  herm_pair_kernel<<<blocks_for(n * b * b), 256, 0, s>>>(m.diag, m.diag, n, (int)b, (int)b);
  if (n > 1)
    herm_pair_kernel<<<blocks_for((n - 1) * b * b), 256, 0, s>>>(m.upper, m.lower, n - 1, (int)b, (int)b);
  if (a > 0) {
    herm_pair_kernel<<<blocks_for(n * a * b), 256, 0, s>>>(m.arrow_row, m.arrow_col, n, (int)a, (int)b);
    herm_pair_kernel<<<blocks_for(a * a), 256, 0, s>>>(m.tip, m.tip, 1, (int)a, (int)a);
  }
  return cudaGetLastError();
}

}  // namespace bsel
