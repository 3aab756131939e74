// Device-side sequential RGF solver: forward Schur sweep, fused SI+SQ
// backward sweep, arrowhead tip update (pkg/src/btasel/rgf.py) and the
// distributed partition kernels (pkg/src/btasel/dist.py), expressed as
// stream-ordered levels of grouped DMMA GEMMs plus block inverses.
#pragma once
#include <cstdint>
#include <vector>

#include "level.cuh"
#include "symmetry.cuh"

namespace bsel {

// Stacked BT(A) matrix in device memory (see include/btasel_b200.h).
struct BtaDev {
  int64_t n = 0, b = 0, a = 0;
  double2* diag = nullptr;       // [n][b][b]
  double2* lower = nullptr;      // [n-1][b][b]   block (i+1, i)
  double2* upper = nullptr;      // [n-1][b][b]   block (i, i+1)
  double2* arrow_row = nullptr;  // [n][a][b]     block (t, i)
  double2* arrow_col = nullptr;  // [n][b][a]     block (i, t)
  double2* tip = nullptr;        // [a][a]
  Mat D(int64_t i) const { return blk(diag, i, (int)b, (int)b); }
  Mat L(int64_t i) const { return blk(lower, i, (int)b, (int)b); }
  Mat U(int64_t i) const { return blk(upper, i, (int)b, (int)b); }
  Mat AR(int64_t i) const { return blk(arrow_row, i, (int)a, (int)b); }
  Mat AC(int64_t i) const { return blk(arrow_col, i, (int)b, (int)a); }
  Mat T() const { return Mat{tip, a, (int)a, (int)a}; }
};

// RgfFactors (rgf.py:37-61) in device memory.
struct FactorsDev {
  int64_t n = 0, b = 0, a = 0;
  bool fused = false;
  double2* s_a = nullptr;             // [n][b][b]
  double2* s_b = nullptr;             // [n-1][b][b]           (fused)
  double2* b_diag_last = nullptr;     // [b][b]                (fused)
  double2* tip_inv = nullptr;         // [a][a]                (a > 0)
  double2* b_tip = nullptr;           // [a][a]                (fused, a > 0)
  double2* arrow_row_elim = nullptr;  // [n][a][b]
  double2* arrow_col_elim = nullptr;  // [n][b][a]
  double2* b_arrow_row_elim = nullptr;
  double2* b_arrow_col_elim = nullptr;
  // optional retained elimination products (bsel_factors_t elim_*)
  double2* elim_f = nullptr;  // [n][b][b]  A(j,i) S_i
  double2* elim_g = nullptr;  // [n][a][b]  AR_i S_i
  double2* elim_q = nullptr;  // [n][b][b]  Bd_i f^H - B(i,j)
  double2* elim_k = nullptr;  // [n][b][a]  Bd_i g^H - BC_i
  double2* elim_h = nullptr;   // [n][b][b]  S_i A(i,j)
  double2* elim_ha = nullptr;  // [n][b][a]  S_i AC_i
  double2* elim_eq = nullptr;  // [n][b][b]  -S_i elim_q
  double2* elim_ek = nullptr;  // [n][b][a]  -S_i elim_k
  Mat EH(int64_t i) const { return elim_h ? blk(elim_h, i, (int)b, (int)b) : Mat{}; }
  Mat EHA(int64_t i) const { return elim_ha ? blk(elim_ha, i, (int)b, (int)a) : Mat{}; }
  Mat EEQ(int64_t i) const { return elim_eq ? blk(elim_eq, i, (int)b, (int)b) : Mat{}; }
  Mat EEK(int64_t i) const { return elim_ek ? blk(elim_ek, i, (int)b, (int)a) : Mat{}; }
  Mat EF(int64_t i) const { return elim_f ? blk(elim_f, i, (int)b, (int)b) : Mat{}; }
  Mat EG(int64_t i) const { return elim_g ? blk(elim_g, i, (int)a, (int)b) : Mat{}; }
  Mat EQ(int64_t i) const { return elim_q ? blk(elim_q, i, (int)b, (int)b) : Mat{}; }
  Mat EK(int64_t i) const { return elim_k ? blk(elim_k, i, (int)b, (int)a) : Mat{}; }
  Mat SA(int64_t i) const { return blk(s_a, i, (int)b, (int)b); }
  Mat SB(int64_t i) const { return blk(s_b, i, (int)b, (int)b); }
  Mat ARe(int64_t i) const { return blk(arrow_row_elim, i, (int)a, (int)b); }
  Mat ACe(int64_t i) const { return blk(arrow_col_elim, i, (int)b, (int)a); }
  Mat BRe(int64_t i) const { return blk(b_arrow_row_elim, i, (int)a, (int)b); }
  Mat BCe(int64_t i) const { return blk(b_arrow_col_elim, i, (int)b, (int)a); }
};

struct SingularInfo {
  bool singular = false;
  int64_t index = -1;
};

class Context {
 public:
  // Status + symmetry flags published by a kernel into mapped pinned host
  // memory: a copy-engine D2H would wait behind any multi-GiB D2H in flight
  // on another stream (tools/ce_starve_probe.py), a kernel store does not.
  struct HostFlags {
    unsigned long long status;
    int sym;
  };
  explicit Context(int device);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  void set_stream(cudaStream_t s) { user_stream_ = s; }
  // CTAs of the persistent block inverse (0 = library default).  Fewer when
  // several contexts run sweeps concurrently on one GPU.
  void set_inverse_grid(int ctas) { inv_grid_ = ctas; }
  int inverse_grid() const { return inv_grid_; }
  cudaStream_t stream() const { return user_stream_; }
  cudaStream_t aux() const { return aux_; }
  // High-priority stream for the latency-critical Schur chain (pivot
  // inverse -> elimination factors -> next pivot); its CTAs are scheduled
  // ahead of the aux stream's throughput work as SMs free up.
  cudaStream_t chain() const { return chain_; }
  // Low-priority stream for work that runs ahead of both chains (the
  // backward sweep's per-step prologue).
  cudaStream_t side() const { return side_; }
  int device() const { return device_; }

  // Scratch: `count` temporaries of (r x c) complex, grow-only.
  double2* scratch(int64_t elems);
  // Temporary block slot k of size (r x c) inside the slot pool.
  Mat tmp(int slot, int r, int c);
  void reserve_slots(int nslots, int64_t slot_elems);
  double2* inv_work(int64_t elems);

  // Symmetry of the right-hand side B (symmetry.cuh).  sym_reset() clears
  // the device flags, sym_check() ORs a block-pair check into them (stream
  // ordered), read_status() brings them to the host.  b_symmetry(): the
  // backward path to take, +1 / -1 (B = +-B^H exactly), 0 = general; forced
  // by set_b_symmetry(+1 / -1 / 0) (the partitioned solves decide globally),
  // or kSymAuto = from this context's own last check.
  static constexpr int kSymAuto = 2;
  void sym_reset(cudaStream_t s);
  void sym_check(const SymJob& j, cudaStream_t s);
  void set_b_symmetry(int mode) { sym_mode_ = mode; }
  int b_symmetry() const;
  int sym_flags() const { return sym_checked_ ? sym_flags_ : 3; }
  // Synchronize the stream and read the flags of the checks queued so far;
  // returns +1 / -1 when THAT data is exactly (anti-)Hermitian, else 0.  The
  // forward of a partition may use its own data's symmetry (its recursion
  // never reads another partition's blocks); set_forward_symmetry() passes it
  // to the forward steps.
  int sym_now(cudaStream_t s);
  void set_forward_symmetry(int s) { fwd_sym_ = s; }
  // Forward aux-stream levels keep SMs [0, n) free for the Schur chain's
  // inverse (zgemm.cuh avoid_sms); 0 = off.  aux_counter(): their tile counter.
  void set_aux_avoid_sms(int n) { aux_avoid_ = n; }
  int aux_avoid_sms() const { return aux_avoid_; }
  unsigned* aux_counter() const { return d_aux_counter_; }
  int forward_symmetry() const { return fwd_sym_; }

  // Singularity bookkeeping (device side, checked at synchronize()).
  void reset_status();
  void invert(Mat X, Mat Y, uint64_t order, int64_t index, cudaStream_t s);
  // Fused Schur step (inverse.cuh launch_schur_step): S = D^-1, H = D^-1 U
  // (H.p may be null), F = L D^-1, C -= L D^-1 U.  schur_ok(b): available.
  bool schur_ok(int b) const;
  void schur(Mat D, Mat U, Mat L, Mat C, Mat S, Mat H, Mat F, uint64_t order, int64_t index, cudaStream_t s);
  SingularInfo read_status();  // synchronizes the user stream

  // Copy stream for host<->device transfers overlapped with the sweeps and
  // a pool of ordering events for them (created on first use).
  cudaStream_t xfer();
  cudaEvent_t xfer_event(int i);
  // Events for cross-stream ordering: 0..15 fork/join and the forward ring,
  // kBackEvents.. the backward sweep's ring.
  static constexpr int kBackEvents = 16;
  cudaEvent_t event(int i);
  cudaEvent_t timer(int i);

  float last_forward_ms = 0.f, last_backward_ms = 0.f;

 private:
  int device_;
  cudaStream_t user_stream_ = nullptr;
  cudaStream_t aux_ = nullptr;
  cudaStream_t chain_ = nullptr;
  cudaStream_t side_ = nullptr;
  double2* slots_ = nullptr;
  int64_t slot_elems_ = 0;
  int nslots_ = 0;
  double2* inv_work_ = nullptr;
  int64_t inv_work_elems_ = 0;
  int* d_flag_ = nullptr;
  int* d_sym_ = nullptr;
  unsigned* d_aux_counter_ = nullptr;
  int aux_avoid_ = 0;
  int sym_flags_ = 3, sym_mode_ = kSymAuto, fwd_sym_ = 0;
  bool sym_checked_ = false;
  unsigned long long* d_status_ = nullptr;
  HostFlags* h_flags_ = nullptr;
  HostFlags* d_hflags_ = nullptr;
  void publish_flags(cudaStream_t s);
  std::vector<cudaEvent_t> events_;
  std::vector<cudaEvent_t> xfer_events_;
  cudaStream_t xfer_ = nullptr;
  int inv_grid_ = 0;
  cudaEvent_t timers_[4] = {nullptr, nullptr, nullptr, nullptr};
};

// Symmetry checks of a right-hand side (Context::sym_check).  Strips: diag
// blocks and arrow pairs of global blocks [g0, g1) of `src` (whose block 0 is
// global block src_lo), optionally copied to `dst` (block 0 = dst_lo);
// couplings: lower/upper pairs [e0, e1); tip: optionally copied to dst_tip.
void sym_check_strips(Context& ctx, const BtaDev& src, int64_t src_lo, int64_t g0, int64_t g1, const BtaDev* dst,
                      int64_t dst_lo, cudaStream_t s);
void sym_check_couplings(Context& ctx, const BtaDev& src, int64_t e0, int64_t e1, cudaStream_t s);
void sym_check_tip(Context& ctx, const BtaDev& src, double2* dst_tip, cudaStream_t s);

// rgf.py:79 bt_forward / rgf.py:207 bta_forward.  `A`, `B` are working
// copies mutated in place (diag, arrow strips, tip); B may be null (SI).
void bta_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F);
// rgf.py:127 bt_backward / rgf.py:401 bta_backward.
void bta_backward(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B, const BtaDev& XA,
                  const BtaDev* XB, bool diagonal_only);

}  // namespace bsel
