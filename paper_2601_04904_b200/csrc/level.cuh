// Host-side builder for one "level" of independent block products, launched
// as grouped DMMA GEMMs (zgemm.cuh).  The sweeps (sweeps.cu) are written as
// sequences of levels; each level lists the products whose inputs are ready.
#pragma once
#include <stdexcept>
#include <string>

#include "zgemm.cuh"

namespace bsel {

struct ShapeError : std::runtime_error {
  explicit ShapeError(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// A (rows x cols) block view of a row-major complex128 array.
struct Mat {
  double2* p = nullptr;
  int64_t ld = 0;
  int r = 0, c = 0;
};

// i-th block of a stacked [count][r][c] array.
inline Mat blk(double2* base, int64_t i, int r, int c) {
  return Mat{base + i * (int64_t)r * c, c, r, c};
}
inline Mat blk(const double2* base, int64_t i, int r, int c) {
  return blk(const_cast<double2*>(base), i, r, c);
}

enum : char { N = 'N', H = 'H' };

class Level {
 public:
  explicit Level(cudaStream_t s, int tile_cfg = kTileAuto, int max_ctas = 0) : s_(s), cfg_(tile_cfg) {
    b_.nproblems = 0;
    b_.max_ctas = max_ctas;
    b_.avoid_sms = 0;
    b_.tile_counter = nullptr;
    b_.chain_mark = nullptr;
  }
  // Instrumented builds: record this level's launches as chain kernels
  // (launch-gap statistics, inverse.cuh chain_marks).
  Level& chain_mark(unsigned long long* m) {
    b_.chain_mark = m;
    return *this;
  }
  // Keep SMs [0, n) free of this level's CTAs (zgemm.cuh avoid_sms); counter:
  // a device u32 owned by this level's stream.
  Level& avoid_sms(int n, unsigned* counter) {
    b_.avoid_sms = counter ? n : 0;
    b_.tile_counter = counter;
    return *this;
  }
  ~Level() noexcept(false) {}

  // Start a new output D = (addends) + (terms).
  Level& out(Mat D) {
    if (b_.nproblems == kMaxProblems) flush();
    cur_ = &b_.p[b_.nproblems++];
    *cur_ = GemmProblem{};
    cur_->D = D.p;
    cur_->ldd = D.ld;
    cur_->M = D.r;
    cur_->N = D.c;
    return *this;
  }
  Level& add(int sign, Mat X) {
    if (!cur_) throw ShapeError("add() before out()");
    if (X.r != cur_->M || X.c != cur_->N)
      throw ShapeError("addend shape mismatch: " + dims(X.r, X.c) + " vs " + dims(cur_->M, cur_->N));
    if (cur_->M == 0 || cur_->N == 0) return *this;
    if (cur_->naddends == kMaxAddends) throw ShapeError("too many addends");
    GemmAddend& a = cur_->add[cur_->naddends++];
    a.X = X.p;
    a.ldx = X.ld;
    a.sign = sign;
    return *this;
  }
  // Only the tiles on / below the tile diagonal of the (square) output are
  // computed (a Hermitian result mirrored afterwards).
  Level& lower_only() {
    if (!cur_ || cur_->M != cur_->N) throw ShapeError("lower_only() needs a square output");
    cur_->lower_only = 1;
    return *this;
  }
  // D += sign * op(A) @ op(B); op 'N' or 'H' (conjugate transpose).
  Level& mm(int sign, Mat A, char oa, Mat B, char ob) {
    if (!cur_) throw ShapeError("mm() before out()");
    const int am = (oa == N) ? A.r : A.c, ak = (oa == N) ? A.c : A.r;
    const int bk = (ob == N) ? B.r : B.c, bn = (ob == N) ? B.c : B.r;
    if (am != cur_->M || bn != cur_->N || ak != bk)
      throw ShapeError("product shape mismatch: op(A) " + dims(am, ak) + ", op(B) " + dims(bk, bn) +
                       ", D " + dims(cur_->M, cur_->N));
    if (ak == 0 || cur_->M == 0 || cur_->N == 0) return *this;
    if (cur_->nterms == kMaxTerms) throw ShapeError("too many terms");
    GemmTerm& t = cur_->term[cur_->nterms++];
    t.A = A.p;
    t.B = B.p;
    t.lda = A.ld;
    t.ldb = B.ld;
    t.K = ak;
    t.opA = (oa == N) ? kOpN : kOpC;
    t.opB = (ob == N) ? kOpN : kOpC;
    t.sign = static_cast<int8_t>(sign);
    return *this;
  }
  void flush() {
    if (b_.nproblems > 0) cuda_check(launch_gemm_batch(b_, s_, cfg_), "grouped zgemm launch");
    b_.nproblems = 0;
    cur_ = nullptr;
  }

 private:
  static std::string dims(int r, int c) { return "(" + std::to_string(r) + "x" + std::to_string(c) + ")"; }
  cudaStream_t s_;
  int cfg_;
  GemmBatch b_{};
  GemmProblem* cur_ = nullptr;
};

}  // namespace bsel
