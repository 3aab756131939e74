// Per-phase clock64 profile of the register-resident 32x32 leaf (debug).
#include "../paper_2601_04904_b200/csrc/zgemm.cu"
#include "../paper_2601_04904_b200/csrc/inverse.cu"
#include <cstdio>
namespace bsel {
__global__ void leaf_phases(const double2* X, int n, long long* out) {
  __shared__ Leaf32 L;
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    int i = e >> 5, j = e & 31;
    if (i < n && j < n) L.a[i][j] = X[i * n + j];
  }
  __syncthreads();
  const int t = threadIdx.x, lane = t & 31;
  const int i = t >> 3, c0 = (t & 7) * 4;
  double2 v[4];
  for (int q = 0; q < 4; ++q) v[q] = (i < n && c0 + q < n) ? L.a[i][c0 + q] : make_double2(0.0, 0.0);
  if ((t & 7) == 0) L.col[0][i] = v[0];
  __syncthreads();
  unsigned used = 0u;
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  for (int k = 0; k < n; ++k) {
    long long c_0 = clock64();
    const int buf = k & 1;
    const bool cand = lane < n && !((used >> lane) & 1u);
    const unsigned key = cand ? (unsigned)__double2hiint(cabs1(L.col[buf][lane])) + 1u : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned ball = __ballot_sync(0xffffffffu, cand && key == kmax);
    const int p = __ffs(ball) - 1;
    used |= 1u << p;
    long long c_1 = clock64();
    if (i == p) for (int q = 0; q < 4; ++q) L.row[buf][row_slot(c0 + q)] = v[q];
    const double2 inv = crecip_fast(L.col[buf][p]);
    const double2 m = cmul(L.col[buf][i], inv);
    asm volatile("" :: "d"(m.x), "d"(inv.x));
    long long c_2 = clock64();
    __syncthreads();
    long long c_3 = clock64();
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
    const int q1 = k + 1 - c0;
    if (q1 >= 0 && q1 < 4) L.col[buf ^ 1][i] = q1 == 0 ? v[0] : q1 == 1 ? v[1] : q1 == 2 ? v[2] : v[3];
    asm volatile("" :: "d"(v[0].x), "d"(v[3].y));
    long long c_4 = clock64();
    __syncthreads();
    long long c_5 = clock64();
    acc[0] += c_1 - c_0; acc[1] += c_2 - c_1; acc[2] += c_3 - c_2; acc[3] += c_4 - c_3; acc[4] += c_5 - c_4;
  }
  if (threadIdx.x == 0 || threadIdx.x == 255)
    for (int j = 0; j < 5; ++j) out[(threadIdx.x == 255) * 8 + j] = acc[j];
}
}
int main() {
  const int n = 32;
  double2 h[n * n];
  for (int i = 0; i < n * n; ++i) h[i] = make_double2((i % 7) * 0.1, (i % 5) * 0.1 - 0.2);
  for (int i = 0; i < n; ++i) h[i * n + i].x += 3 * n;
  double2* d; long long* s; long long hs[16];
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&s, 128);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) bsel::leaf_phases<<<1, 256>>>(d, n, s);
  cudaMemcpy(hs, s, 128, cudaMemcpyDeviceToHost);
  for (int w = 0; w < 2; ++w)
    printf("{\"thread\": %d, \"pivot\": %.0f, \"rcp_m\": %.0f, \"sync1\": %.0f, \"update\": %.0f, \"sync2\": %.0f}\n", w ? 255 : 0,
           hs[w * 8 + 0] / 32.0, hs[w * 8 + 1] / 32.0, hs[w * 8 + 2] / 32.0, hs[w * 8 + 3] / 32.0, hs[w * 8 + 4] / 32.0);
  return 0;
}
