// Grouped multi-term complex128 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
// One launch evaluates up to kMaxProblems independent block products
//
//     D = sum_a  s_a * X_a  +  sum_t  s_t * op(A_t) @ op(B_t)      (s = +-1)
//
// with op in {N, C} (C = conjugate transpose, never materialised: the
// transposition is folded into the shared-memory staging addresses and the
// conjugation into a sign-bit XOR on the fragment registers).  This is the
// B200 replacement for every `mm(...)` / `block_multiply_acc` call of the
// reference (pkg/src/btasel/kernels.py:106-166) and for the elementwise
// +/- combinations around them (e.g. rgf.py:113-118, rgf.py:258-280): the
// K-concatenated terms share one accumulator tile, the addends are fused
// into the epilogue.
//
// Complex arithmetic uses the real 2x2 embedding: an interleaved complex row
// of length K is a real row of length 2K, and
//     C_re = A_il . [B_re ; -B_im],   C_im = A_il . [B_im ; B_re]
// so each mma.sync.m8n8k4.f64 computes an 8 x 4 (complex) tile over 2
// complex k.  No flops are wasted (8 real flops per complex MAC).
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace bsel {

// Value computed once PER DEVICE (f() runs with that device current): kernel
// attributes such as the dynamic shared-memory opt-in and occupancy-derived
// limits are per device, and one process may drive several GPUs.  Each call
// site (lambda type) gets its own cache.
constexpr int kMaxDevices = 64;
template <class F>
auto per_device(F&& f) -> decltype(f()) {
  using T = decltype(f());
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  static T val[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return f();
  std::lock_guard<std::mutex> lock(mu);
  if (!done[dev]) {
    val[dev] = f();
    done[dev] = true;
  }
  return val[dev];
}

enum : uint8_t { kOpN = 0, kOpC = 1 };

constexpr int kMaxTerms = 6;
constexpr int kMaxAddends = 3;
constexpr int kMaxProblems = 16;

struct GemmTerm {
  const double2* A;   // op(A) is M x K
  const double2* B;   // op(B) is K x N
  int64_t lda;        // leading dimension of the STORED A (complex elements)
  int64_t ldb;
  int32_t K;
  uint8_t opA, opB;
  int8_t sign;        // +1 / -1
  uint8_t pad_;
  uint32_t tmaA, tmaB;  // TMA descriptor slots (filled by the 3M launcher)
};

struct GemmAddend {
  const double2* X;   // M x N
  int64_t ldx;
  int32_t sign;
  int32_t pad_;
};

struct GemmProblem {
  double2* D;         // M x N output (may alias an addend, never a term operand)
  int64_t ldd;
  int32_t M, N;
  int32_t nterms, naddends;
  int32_t tiles_n;    // filled by the launcher
  int32_t tile_begin; // filled by the launcher
  int32_t lower_only; // M == N: only tiles on / below the tile diagonal are computed
  int32_t pad_;
  GemmAddend add[kMaxAddends];
  GemmTerm term[kMaxTerms];
};

struct GemmBatch {
  int32_t nproblems;
  int32_t total_tiles;
  // > 0: launch at most max_ctas CTAs that loop over the tiles (leaves SMs
  // free for a concurrent latency-critical chain); 0: one CTA per tile
  int32_t max_ctas;
  // > 0: CTAs landing on SMs with id < avoid_sms exit at once and the others
  // fetch tiles dynamically from tile_counter[0] (tile_counter[1] counts the
  // CTAs that left; both zeroed by the launcher):
  // those SMs stay free for a concurrent latency-critical kernel
  int32_t avoid_sms;
  unsigned* tile_counter;
  const void* tma_table;  // device table of CUtensorMap descriptors (3M launcher)
  // instrumented builds (-DBSEL_INV_STATS=1) only: chain launch-gap marks
  // (inverse.cuh chain_marks), null otherwise
  unsigned long long* chain_mark;
  GemmProblem p[kMaxProblems];
};

// Tile configurations (complex tile BM x BN).
// kTileAuto: 64x64 tiles once a launch has >= 2 waves of them; kTileAutoWide:
// already from 128 of them (BSEL_GEMM_MIN_TILES64_WIDE): the middle
// partitions' k = 3 back-substitution, measured best there.  kTileAutoFwd:
// the forward sweeps' aux levels, which run beside the Schur chain (3M tile
// policy without the BK 32 variant, zgemm3m.cu).
enum TileCfg : int { kTile64 = 0, kTile32 = 1, kTileAuto = 2, kTileAutoWide = 3, kTileAutoFwd = 4,
                     // forced kernel variants (microbenchmarks / A-B tests)
                     kTile3m64 = 10, kTile3m6432 = 11, kTile3m32 = 12, kTile3m64k32 = 13, kTile3m6432k32 = 14,
                     kTile4m64 = 20, kTile4m32 = 21 };

// Launch one grouped batch on `stream`.  Problems with M==0 or N==0 are
// dropped.  Returns cudaSuccess or the launch error.
cudaError_t launch_gemm_batch(GemmBatch& batch, cudaStream_t stream, int tile_cfg = kTileAuto);
// The 3-multiplication bulk-async kernel (zgemm3m.cu) behind launch_gemm_batch.
cudaError_t launch_gemm_batch_3m(GemmBatch& batch, cudaStream_t stream, int tile_cfg);

// Boundary publication to peers' symmetric-memory buffers (publish.cu).
cudaError_t launch_publish(const double2* const* src, const int64_t* elems, const int64_t* dst_off, int nblocks,
                           double2* const* dst, int ndst, int64_t hdr_off, const double* hdr, cudaStream_t s);

// Number of SMs of the current device (cached).
int device_sm_count();

// Process-wide count of kernels launched by this library (bench evidence).
void count_launch(uint64_t k = 1);
uint64_t launch_count();

// Optional per-launch device timing (CUDA events on the launching stream),
// used by bench.py to measure the dominant kernel live.  kind 0 = grouped
// GEMM launch (flops = sum 8*M*N*K), kind 1 = one whole block inverse.
struct ProfileTotals {
  int64_t gemm_launches;
  double gemm_flops;
  double gemm_ms;
  int64_t inverse_calls;
  double inverse_ms;
  double gemm_bytes;
  double gemm_busy_ms, inverse_busy_ms, inverse_flops;
  double gemm_exec_flops;  // executed tensor-pipe flops (3M: 6MNK, real embedding: 8MNK)
};
void profile_begin();
ProfileTotals profile_end();
bool profiling();
void profile_suspend(bool on);  // temporarily ignore GEMM launches (inside an inverse)
int profile_open(cudaStream_t s);                          // returns record id (or -1)
void profile_close(int id, cudaStream_t s, int kind, double flops, double bytes = 0.0, double exec_flops = -1.0);

}  // namespace bsel
