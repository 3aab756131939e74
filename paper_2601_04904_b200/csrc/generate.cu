// Device generator for the reference's synthetic inputs (matrix.py:192-284).
//
// The splitmix64 stream is a pure function of (seed, position), so every
// complex entry is generated independently: entry e of the concatenated
// stream diag | lower | upper | arrow_row | arrow_col | tip uses positions
// 2e+1 (re) and 2e+2 (im).  This is bit-identical to the host generator.
// The dominance shift needs |row| sums across blocks; they are accumulated
// left-to-right in double (the host uses numpy pairwise sums, so the shifted
// diagonal can differ from the host generator in the last bit).
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

__device__ __forceinline__ double cabs_(double2 z) { return hypot(z.x, z.y); }

// One thread per global diagonal row r = i*b + row: off-diagonal |row| sum
// (diag block without its diagonal entry, lower[i-1], upper[i], arrow_col[i]),
// then push the diagonal entry along its phase.
__global__ void dominance_rows_kernel(BtaDevView m, double dominance) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m.n * m.b) return;
  const int64_t i = r / m.b, row = r % m.b, b = m.b, a = m.a;
  const double2* d = m.diag + i * b * b + row * b;
  double s = 0.0;
  for (int64_t j = 0; j < b; ++j)
    if (j != row) s += cabs_(d[j]);
  if (i > 0) {
    const double2* l = m.lower + (i - 1) * b * b + row * b;
    for (int64_t j = 0; j < b; ++j) s += cabs_(l[j]);
  }
  if (i < m.n - 1) {
    const double2* u = m.upper + i * b * b + row * b;
    for (int64_t j = 0; j < b; ++j) s += cabs_(u[j]);
  }
  if (a > 0) {
    const double2* c = m.arrow_col + i * b * a + row * a;
    for (int64_t j = 0; j < a; ++j) s += cabs_(c[j]);
  }
  double2* dd = m.diag + i * b * b + row * b + row;
  const double2 v = *dd;
  const double mag = cabs_(v);
  const double px = mag > 0 ? v.x / mag : 1.0, py = mag > 0 ? v.y / mag : 0.0;
  const double shift = dominance * (s + 1.0);
  *dd = make_double2(v.x + shift * px, v.y + shift * py);
}

__global__ void dominance_tip_kernel(BtaDevView m, double dominance) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t a = m.a, b = m.b;
  if (row >= a) return;
  double s = 0.0;
  for (int64_t j = 0; j < a; ++j)
    if (j != row) s += cabs_(m.tip[row * a + j]);
  for (int64_t i = 0; i < m.n; ++i) {
    const double2* r = m.arrow_row + i * a * b + row * b;
    for (int64_t j = 0; j < b; ++j) s += cabs_(r[j]);
  }
  double2* dd = m.tip + row * a + row;
  const double2 v = *dd;
  const double mag = cabs_(v);
  const double px = mag > 0 ? v.x / mag : 1.0, py = mag > 0 ? v.y / mag : 0.0;
  const double shift = dominance * (s + 1.0);
  *dd = make_double2(v.x + shift * px, v.y + shift * py);
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
