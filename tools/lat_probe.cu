// Latency probes on B200 (sm_100a): dependent-chain latencies of DFMA, DMUL,
// MUFU.RCP64H-based reciprocal, LDS, redux.sync, __syncthreads (8 warps).
#include <cstdio>
__global__ void probe(double* out, long long* cyc, int iters) {
  __shared__ double sm[256];
  __shared__ int si[256];
  sm[threadIdx.x] = threadIdx.x * 0.5;
  si[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  double x = threadIdx.x * 1e-3 + 1.0, y = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = x * y;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = __drcp_rn(x) + 1e-300;
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) idx = si[idx];
  long long t4 = clock64();
  unsigned v = threadIdx.x;
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v + i);
  long long t5 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t6 = clock64();
  double z = x;
  for (int i = 0; i < iters; ++i) z = z + 1e-300;
  long long t7 = clock64();
  unsigned b = 0;
  for (int i = 0; i < iters; ++i) b += __ballot_sync(0xffffffffu, (v >> (i & 7)) & 1);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
    cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x + idx + v + z + b;
}
int main() {
  double* d; long long* c; long long h[8];
  cudaMalloc(&d, 4096); cudaMalloc(&c, 64);
  const int iters = 4096;
  for (int w = 0; w < 3; ++w) probe<<<1, 256>>>(d, c, iters);
  cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* names[8] = {"dfma", "dmul", "drcp_rn", "lds_chase", "redux_max", "syncthreads_8warps", "dadd", "ballot"};
  printf("{");
  for (int i = 0; i < 8; ++i) printf("%s\"%s_cycles\": %.1f", i ? ", " : "", names[i], (double)h[i] / iters);
  printf("}\n");
  return 0;
}
