// Microbenchmark of the block-inverse kernels (links the library objects):
// event-timed persistent inverse for several n and a per-panel phase trace.
#include <cstdio>
#include <vector>
#include "../paper_2601_04904_b200/csrc/inverse.cuh"
#include "../paper_2601_04904_b200/csrc/zgemm.cuh"

__global__ void fill(double2* a, int n, unsigned seed) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  int i = e / n, j = e % n;
  unsigned h = (unsigned)(e * 2654435761u) ^ seed;
  double x = ((h & 0xffff) / 65536.0) - 0.5, y = (((h >> 16) & 0xffff) / 65536.0) - 0.5;
  if (i == j) x += 3.0 * n;
  a[e] = make_double2(x, y);
}

__global__ void clock_probe(double* mhz) {
  unsigned long long g0, g1;
  long long c0 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  while (true) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (g1 - g0 > 2000000) break;
  }
  long long c1 = clock64();
  *mhz = (double)(c1 - c0) / (double)(g1 - g0) * 1e3;
}

static double sm_mhz() {
  double* d;
  double h = 0;
  cudaMalloc(&d, 8);
  clock_probe<<<1, 1>>>(d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  {  // warm the clocks up: ~2 s of back-to-back inverses
    const int n = 512;
    double2 *X, *Y, *W;
    int* flag;
    cudaMalloc(&X, (size_t)n * n * 16);
    cudaMalloc(&Y, (size_t)n * n * 16);
    cudaMalloc(&W, (size_t)bsel::block_inverse_workspace(n) * 16);
    cudaMemset(W, 0, (size_t)bsel::block_inverse_workspace(n) * 16);
    cudaMalloc(&flag, 4);
    cudaMemset(flag, 0, 4);
    fill<<<(n * n + 255) / 256, 256>>>(X, n, 7);
    printf("{\"sm_mhz_idle\": %.0f}\n", sm_mhz());
    for (int r = 0; r < 3000; ++r) bsel::launch_block_inverse(X, n, Y, n, n, W, flag, nullptr, 0, s);
    cudaStreamSynchronize(s);
    printf("{\"sm_mhz_after_warmup\": %.0f}\n", sm_mhz());
    cudaFree(X); cudaFree(Y); cudaFree(W); cudaFree(flag);
  }
  for (int n : {32, 64, 128, 256, 512, 1024}) {
    double2 *X, *Y, *W;
    int* flag;
    cudaMalloc(&X, (size_t)n * n * 16);
    cudaMalloc(&Y, (size_t)n * n * 16);
    cudaMalloc(&W, (size_t)bsel::block_inverse_workspace(n) * 16);
    cudaMemset(W, 0, (size_t)bsel::block_inverse_workspace(n) * 16);
    cudaMalloc(&flag, 4);
    cudaMemset(flag, 0, 4);
    fill<<<(n * n + 255) / 256, 256>>>(X, n, 7);
    for (int r = 0; r < 3; ++r) bsel::launch_block_inverse(X, n, Y, n, n, W, flag, nullptr, 0, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) bsel::launch_block_inverse(X, n, Y, n, n, W, flag, nullptr, 0, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"n\": %d, \"inverse_us\": %.1f, \"err\": \"%s\"}\n", n, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
    if (n == 512) {
      const int nt = n / 32;
      unsigned long long* tr;
      cudaMalloc(&tr, 16 * nt * 8);
      cudaMemset(tr, 0, 16 * nt * 8);
      bsel::g_inverse_trace = tr;
      bsel::launch_block_inverse(X, n, Y, n, n, W, flag, nullptr, 0, s);
      cudaStreamSynchronize(s);
      bsel::g_inverse_trace = nullptr;
      std::vector<unsigned long long> h(16 * nt);
      cudaMemcpy(h.data(), tr, 16 * nt * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = h[0];
      for (int p = 0; p < nt; ++p) {
        auto d = [&](int k) { return h[16 * p + k] ? (double)(h[16 * p + k] - t0) / 1e3 : -1.0; };
        printf("panel %2d: cta0 start %7.2f  tile %7.2f  leaf %7.2f  atbar %7.2f | cta1 first-tile %7.2f..%7.2f done %7.2f  past-bar %7.2f us\n",
               p, d(0), d(1), d(2), d(3), d(6), d(7), d(4), d(5));
        printf("          lookahead: issue %7.2f  stage-begin %7.2f  landed %7.2f  R-done %7.2f  tile-done %7.2f\n",
               d(11), d(8), d(9), d(12), d(10));
      }
    }
    cudaFree(X); cudaFree(Y); cudaFree(W); cudaFree(flag);
  }
  return 0;
}
