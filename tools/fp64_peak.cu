// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync f64) and DFMA
// register-resident loops, plus cuBLAS Dgemm/Zgemm as yardsticks only (the
// solver never calls cuBLAS). Prints one JSON line.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma16_loop(double* out, int iters) {
  // m16n8k16: A 8 regs, B 4 regs, C 4 regs per thread
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 2e-3 + i;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0)); f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int nsm = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  const int iters = 4096;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f", p.name, nsm, clk_khz / 1e3);
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = nsm * 4;
    float ms = time_it([&] { dmma_loop<8><<<blocks, threads>>>(out, iters); }, 5);
    double fl = 512.0 * 8 * iters * (double)blocks * wpb;
    printf(", \"dmma_m8n8k4_w%d_tflops\": %.2f", wpb, fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = nsm * 4;
    float ms = time_it([&] { dmma16_loop<4><<<blocks, threads>>>(out, iters / 4); }, 5);
    double fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)blocks * 8;
    printf(", \"dmma_m16n8k16_tflops\": %.2f", fl / ms / 1e9);
  }
  {
    int threads = 256, blocks = nsm * 8;
    float ms = time_it([&] { dfma_loop<16><<<blocks, threads>>>(out, iters); }, 5);
    double fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf(", \"dfma_tflops\": %.2f", fl / ms / 1e9);
  }
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {512, 1024, 4096}) {
    size_t bytes = (size_t)n * n * 16;
    void *A, *B, *C; CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    CK(cudaMemset(A, 0, bytes)); CK(cudaMemset(B, 0, bytes));
    cuDoubleComplex one = {1, 0}, zero = {0, 0};
    float ms = time_it([&] { cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, (cuDoubleComplex*)A, n, (cuDoubleComplex*)B, n, &zero, (cuDoubleComplex*)C, n); }, 10);
    printf(", \"cublas_zgemm_%d_tflops\": %.2f", n, 8.0 * n * n * (double)n / ms / 1e9);
    double d1 = 1, d0 = 0;
    ms = time_it([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &d1, (double*)A, n, (double*)B, n, &d0, (double*)C, n); }, 10);
    printf(", \"cublas_dgemm_%d_tflops\": %.2f", n, 2.0 * n * n * (double)n / ms / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  printf("}\n");
  return 0;
}
