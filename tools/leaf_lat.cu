// Latency of one 32x32 leaf (gj_leaf32) in isolation: one CTA, repeated
// calls on freshly loaded input, clock64 per call.
#include "../paper_2601_04904_b200/csrc/zgemm.cu"
#include "../paper_2601_04904_b200/csrc/inverse.cu"
#include <cstdio>
namespace bsel {
__global__ void leaf_lat(const double2* X, int n, int reps, long long* out, double2* Y) {
  __shared__ Leaf32 L;
  long long best = 1LL << 60, total = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      int i = e >> 5, j = e & 31;
      L.a[i][j] = (i < n && j < n) ? X[i * n + j] : make_double2(0, 0);
    }
    __syncthreads();
    long long c0 = clock64();
    gj_leaf32(L, n, r == reps - 1 ? out + 2 : nullptr);
    long long c1 = clock64();
    best = min(best, c1 - c0);
    total += c1 - c0;
  }
  if (threadIdx.x == 0) {
    out[0] = best;
    out[1] = total / reps;
  }
  for (int e = threadIdx.x; e < 32 * 32; e += 256) Y[e] = L.a[e >> 5][e & 31];
}
// Instrumented copy of one sub-panel's steps (phase clocks, thread 0).
__global__ void step_phases(const double2* X, long long* out) {
  __shared__ Leaf32 L;
  const int t = threadIdx.x, lane = t & 31;
  const int i = t >> 3, cl = t & 7;
  double2 v = X[i * 32 + cl];
  long long acc[5] = {0, 0, 0, 0, 0};
  unsigned used = 0u;
  int buf = 0;
  L.pan[buf][i][cl] = v;
  __syncthreads();
  for (int rep = 0; rep < 4; ++rep) {
    used = 0u;
    for (int j = 0; j < 8; ++j) {
      long long c0 = clock64();
      const double2 cv = L.pan[buf][lane][j];
      const bool cand = !((used >> lane) & 1u);
      const unsigned key = cand ? (unsigned)__double2hiint(cabs1(cv)) + 1u : 0u;
      const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
      const unsigned ball = __ballot_sync(0xffffffffu, cand && key == kmax);
      const int p = __ffs(ball) - 1;
      used |= 1u << p;
      asm volatile("" ::"r"(p));
      long long c1 = clock64();
      const double2 z = make_double2(__shfl_sync(0xffffffffu, cv.x, p), __shfl_sync(0xffffffffu, cv.y, p));
      const double2 ci = make_double2(__shfl_sync(0xffffffffu, cv.x, i), __shfl_sync(0xffffffffu, cv.y, i));
      const double2 pr = L.pan[buf][p][cl];
      const double2 inv = crecip_fast(z);
      asm volatile("" ::"d"(inv.x), "d"(inv.y));
      long long c2 = clock64();
      const double2 m = cmul(ci, inv);
      const bool prow_ = i == p;
      const double2 coef = prow_ ? inv : make_double2(-m.x, -m.y);
      const double bx = prow_ ? 0.0 : v.x, by = prow_ ? 0.0 : v.y;
      double2 nv;
      nv.x = fma(coef.x, pr.x, fma(-coef.y, pr.y, bx));
      nv.y = fma(coef.x, pr.y, fma(coef.y, pr.x, by));
      if (cl == j) nv = coef;
      v = nv;
      buf ^= 1;
      L.pan[buf][i][cl] = v;
      asm volatile("" ::"d"(v.x));
      long long c3 = clock64();
      __syncthreads();
      long long c4 = clock64();
      acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3; acc[4] += c4 - c0;
    }
  }
  if (t == 0 || t == 255)
    for (int k = 0; k < 5; ++k) out[(t == 255) * 5 + k] = acc[k] / 32;
}
}  // namespace bsel
int main() {
  const int n = 32;
  double2 h[n * n];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = make_double2((i == j ? 40.0 : 0.0) + ((i * 7 + j * 13) % 11) * 0.1 - 0.5, ((i * 5 + j * 3) % 7) * 0.1 - 0.3);
  double2 *X, *Y;
  long long* o;
  cudaMalloc(&X, sizeof(h));
  cudaMalloc(&Y, sizeof(h));
  cudaMalloc(&o, 16 * 8);
  cudaMemcpy(X, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int nn : {8, 16, 24}) {
    bsel::leaf_lat<<<1, 256>>>(X, nn, 50, o, Y);
    long long q[2];
    cudaMemcpy(q, o, 16, cudaMemcpyDeviceToHost);
    printf("{\"n\": %d, \"leaf_cycles_best\": %lld}\n", nn, q[0]);
  }
  bsel::leaf_lat<<<1, 256>>>(X, n, 200, o, Y);
  long long r[2];
  cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
  long long* ph;
  cudaMalloc(&ph, 80);
  bsel::step_phases<<<1, 256>>>(X, ph);
  long long hp[10];
  cudaMemcpy(hp, ph, 80, cudaMemcpyDeviceToHost);
  for (int w = 0; w < 2; ++w)
    printf("{\"thread\": %d, \"search\": %lld, \"shfl_rcp\": %lld, \"update_sts\": %lld, \"bar\": %lld, \"step\": %lld}\n",
           w ? 255 : 0, hp[w * 5], hp[w * 5 + 1], hp[w * 5 + 2], hp[w * 5 + 3], hp[w * 5 + 4]);
  long long tr[14];
  cudaMemcpy(tr, o, sizeof(tr), cudaMemcpyDeviceToHost);
  for (int sp = 0; sp < 4; ++sp)
    printf("{\"subpanel\": %d, \"steps\": %lld, \"lazy\": %lld}\n", sp, tr[2 + 3 * sp + 1] - tr[2 + 3 * sp],
           tr[2 + 3 * sp + 2] - tr[2 + 3 * sp + 1]);
  printf("{\"leaf_cycles_best\": %lld, \"leaf_cycles_mean\": %lld, \"per_step\": %.0f, \"err\": \"%s\"}\n", r[0], r[1],
         r[0] / 32.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
