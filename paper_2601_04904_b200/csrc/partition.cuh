// Partition kernels of the distributed scheme (dist.py:172-416, 542-744).
#pragma once
#include "solver.cuh"

namespace bsel {

enum PartKind : int { kFirst = 0, kMiddle = 1, kLast = 2 };

// LocalFactors (dist.py:134-151) in device memory; block i of the partition
// [lo, hi) is stored at index i - lo.  fill_* (middle only) hold the fill
// couplings A'(lo, i) / A'(i, lo) as seen when block i is eliminated; index
// len-1 receives the final coupling pair (the AllGather payload).
struct LocalFactorsDev {
  int64_t lo = 0, hi = 0, b = 0, a = 0;
  int kind = kFirst;
  bool fused = false;
  double2* s_a = nullptr;         // [len][b][b]
  double2* s_b = nullptr;         // [len][b][b]   (fused)
  double2* fill_row = nullptr;    // [len][b][b]   (middle)
  double2* fill_col = nullptr;    // [len][b][b]   (middle)
  double2* b_fill_row = nullptr;  // [len][b][b]   (middle, fused)
  double2* b_fill_col = nullptr;  // [len][b][b]   (middle, fused)
  // optional retained elimination products (bsel_local_factors_t elim_*)
  double2* elim_f = nullptr;
  double2* elim_g = nullptr;
  double2* elim_q = nullptr;
  double2* elim_k = nullptr;
  double2* elim_fr = nullptr;
  double2* elim_qr = nullptr;
  double2* elim_h = nullptr;
  double2* elim_ha = nullptr;
  double2* elim_eq = nullptr;
  double2* elim_ek = nullptr;
  Mat EH(int64_t k) const { return elim_h ? blk(elim_h, k, (int)b, (int)b) : Mat{}; }
  Mat EHA(int64_t k) const { return elim_ha ? blk(elim_ha, k, (int)b, (int)a) : Mat{}; }
  Mat EEQ(int64_t k) const { return elim_eq ? blk(elim_eq, k, (int)b, (int)b) : Mat{}; }
  Mat EEK(int64_t k) const { return elim_ek ? blk(elim_ek, k, (int)b, (int)a) : Mat{}; }
  Mat EF(int64_t k) const { return elim_f ? blk(elim_f, k, (int)b, (int)b) : Mat{}; }
  Mat EG(int64_t k) const { return elim_g ? blk(elim_g, k, (int)a, (int)b) : Mat{}; }
  Mat EQ(int64_t k) const { return elim_q ? blk(elim_q, k, (int)b, (int)b) : Mat{}; }
  Mat EK(int64_t k) const { return elim_k ? blk(elim_k, k, (int)b, (int)a) : Mat{}; }
  Mat EFR(int64_t k) const { return elim_fr ? blk(elim_fr, k, (int)b, (int)b) : Mat{}; }
  Mat EQR(int64_t k) const { return elim_qr ? blk(elim_qr, k, (int)b, (int)b) : Mat{}; }
  Mat SA(int64_t k) const { return blk(s_a, k, (int)b, (int)b); }
  Mat SB(int64_t k) const { return blk(s_b, k, (int)b, (int)b); }
  Mat FR(int64_t k) const { return blk(fill_row, k, (int)b, (int)b); }
  Mat FC(int64_t k) const { return blk(fill_col, k, (int)b, (int)b); }
  Mat BFR(int64_t k) const { return blk(b_fill_row, k, (int)b, (int)b); }
  Mat BFC(int64_t k) const { return blk(b_fill_col, k, (int)b, (int)b); }
};

// Optional end-to-end mode: the full-size matrices live in (pinned) host
// memory and move chunk by chunk on the context's copy stream, overlapped
// with the sweeps.  A chunk = `chunk` consecutive partition blocks in
// processing order (first/middle partitions ascending from lo, last
// partition descending from hi-1).  local_forward: chunk c's diag / arrow
// strips go straight into the work arrays and its couplings into A/B (device
// storage; their diag/arrow arrays are not read), each sweep step waits for
// its chunk.  local_backward: after backward steps [c*chunk, (c+1)*chunk)
// (chunk 0 also the seeds, the last chunk everything) the finished output
// blocks are copied to hx_a/hx_b.  The calling stream waits for every copy.
struct HostIo {
  const BtaDev* ha = nullptr;   // host inputs (forward)
  const BtaDev* hb = nullptr;
  const BtaDev* hxa = nullptr;  // host outputs (backward)
  const BtaDev* hxb = nullptr;
  int64_t chunk = 0;
  bool copy_tip = false;                // forward: this partition moves the input tips
  cudaStream_t copy_stream = nullptr;   // shared copy stream (nullptr: the context's own)
};

// dist.py:172-416.  A, B: full original matrices (read only).  WA/WB: the
// partition's working copies (n = hi - lo blocks; diag / arrow strips; tip
// receives this rank's tip contribution).  After the call WA/WB hold the
// eliminated strips and the updated boundary blocks (the payload).
void local_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const BtaDev& WA, const BtaDev* WB,
                   const LocalFactorsDev& F, const HostIo* io = nullptr);

// dist.py:542-744.  XR/ZR: reduced solution; k_top/k_bot: reduced indices of
// this partition's boundaries; XA/XB: full-size outputs (only this rank's
// pattern blocks are written; rank 0 also writes the tip).
void local_backward(Context& ctx, const BtaDev& A, const BtaDev* B, const LocalFactorsDev& F, const BtaDev& WA,
                    const BtaDev* WB, const BtaDev& XR, const BtaDev* ZR, int64_t k_top, int64_t k_bot,
                    bool write_tip, const BtaDev& XA, const BtaDev* XB, const HostIo* io = nullptr);

}  // namespace bsel
