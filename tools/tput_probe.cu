// FP64 non-tensor throughput per SM (one CTA of 256 or 1024 threads, 8 chains).
#include <cstdio>
template <int CH>
__global__ void dfma_tput(double* out, long long* cyc, int iters, double b) {
  double c[CH];
  for (int j = 0; j < CH; ++j) c[j] = threadIdx.x + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = fma(c[j], b, 1e-7);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < CH; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main(int argc, char** argv) {
  double* d; long long* c; long long h[148];
  cudaMalloc(&d, 148 * 1024 * 8); cudaMalloc(&c, 148 * 8);
  const int iters = 2048;
  for (int threads : {256, 512, 1024}) {
    for (int r = 0; r < 2; ++r) dfma_tput<8><<<1, threads>>>(d, c, iters, argc > 5 ? 1.0 : 0.9999999);
    cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * 8 * iters;
    printf("{\"threads\": %d, \"dfma_per_clk_per_SM\": %.2f}\n", threads, ops / h[0]);
  }
  // full chip
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_tput<8><<<148 * 4, 256>>>(d, c, iters, 0.9999999);
  cudaEventRecord(e0);
  dfma_tput<8><<<148 * 4, 256>>>(d, c, iters, 0.9999999);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"chip_dfma_tflops\": %.2f}\n", 2.0 * 148 * 4 * 256 * 8.0 * iters / ms / 1e9);
  return 0;
}
