// Cycles of one 32x32x32 complex tile_mma (the inverse's tile product) on
// one SM, 256 threads; DMMA floor = 64 DMMA/warp x 2 warps/SMSP x 16 clk.
#include "../paper_2601_04904_b200/csrc/zgemm.cu"
#include "../paper_2601_04904_b200/csrc/inverse.cu"
#include <cstdio>
namespace bsel {
__global__ void probe(long long* out, double* sink) {
  __shared__ double2 A[kT][kTLD], B[kT][kTLD];
  for (int e = threadIdx.x; e < kT * kTLD; e += blockDim.x) {
    (&A[0][0])[e] = make_double2(e * 1e-3, 1.0);
    (&B[0][0])[e] = make_double2(1.0, e * 1e-3);
  }
  __syncthreads();
  double acc[4][2];
  double s = 0;
  long long best = 1LL << 60;
  for (int r = 0; r < 50; ++r) {
    __syncthreads();
    long long c0 = clock64();
    tile_mma(acc, A, B);
    s += acc[0][0] + acc[3][1];
    __syncthreads();
    long long c1 = clock64();
    best = min(best, c1 - c0);
  }
  if (threadIdx.x == 0) out[0] = best;
  sink[threadIdx.x] = s;
}
}  // namespace bsel
int main() {
  long long* o;
  double* sk;
  cudaMalloc(&o, 8);
  cudaMalloc(&sk, 256 * 8);
  bsel::probe<<<1, 256>>>(o, sk);
  long long h;
  cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  printf("{\"tile_mma_cycles\": %lld, \"floor_cycles\": 2048, \"err\": \"%s\"}\n", h, cudaGetErrorString(cudaGetLastError()));
}
