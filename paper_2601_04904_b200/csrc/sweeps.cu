// Sequential RGF sweeps on device (rgf.py:79-489), BT and BTA, SI and SI+SQ.
//
// Every step is a short sequence of "levels" (Level, level.cuh): each level
// is ONE grouped DMMA GEMM launch containing all block products whose inputs
// are ready, with multi-term K-concatenation and fused +/- addends.  The
// forward sweep runs the A-side Schur chain (inverse -> f,g -> next pivot) on
// the main stream and the B-side (quadratic) updates on an auxiliary stream,
// so the latency-bound pivot inverse of step i+1 overlaps the quadratic
// updates of step i.  Temporaries live in a double-buffered slot ring.
#include <algorithm>
#include <cstring>

#include "inverse.cuh"
#include "solver.cuh"

namespace bsel {

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------

Context::Context(int device) : device_(device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking), "aux stream");
  cuda_check(cudaMalloc(&d_flag_, sizeof(int)), "flag");
  cuda_check(cudaMalloc(&d_status_, sizeof(unsigned long long)), "status");
  events_.resize(8);
  for (auto& e : events_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (auto& t : timers_) cuda_check(cudaEventCreate(&t), "timer");
  reset_status();
  cuda_check(cudaStreamSynchronize(user_stream_), "init sync");
}

Context::~Context() {
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  if (slots_) cudaFree(slots_);
  if (inv_work_) cudaFree(inv_work_);
  if (d_flag_) cudaFree(d_flag_);
  if (d_status_) cudaFree(d_status_);
  for (auto& e : events_) cudaEventDestroy(e);
  for (auto& t : timers_) cudaEventDestroy(t);
  if (aux_) cudaStreamDestroy(aux_);
}

void Context::reserve_slots(int nslots, int64_t slot_elems) {
  if (nslots <= nslots_ && slot_elems <= slot_elems_) return;
  cuda_check(cudaStreamSynchronize(user_stream_), "sync before realloc");
  cuda_check(cudaStreamSynchronize(aux_), "sync before realloc");
  if (slots_) cudaFree(slots_);
  nslots_ = std::max(nslots, nslots_);
  slot_elems_ = std::max(slot_elems, slot_elems_);
  cuda_check(cudaMalloc(&slots_, (size_t)nslots_ * slot_elems_ * sizeof(double2)), "slot pool");
}

Mat Context::tmp(int slot, int r, int c) {
  if (slot >= nslots_ || (int64_t)r * c > slot_elems_) throw ShapeError("temporary slot out of range");
  return Mat{slots_ + (int64_t)slot * slot_elems_, c, r, c};
}

double2* Context::inv_work(int64_t elems) {
  if (elems > inv_work_elems_) {
    cuda_check(cudaStreamSynchronize(user_stream_), "sync before realloc");
    if (inv_work_) cudaFree(inv_work_);
    cuda_check(cudaMalloc(&inv_work_, (size_t)elems * sizeof(double2)), "inverse workspace");
    inv_work_elems_ = elems;
  }
  return inv_work_;
}

void Context::reset_status() {
  cuda_check(cudaMemsetAsync(d_flag_, 0, sizeof(int), user_stream_), "memset flag");
  cuda_check(cudaMemsetAsync(d_status_, 0xff, sizeof(unsigned long long), user_stream_), "memset status");
}

void Context::invert(Mat X, Mat Y, uint64_t order, int64_t index, cudaStream_t s) {
  if (X.r != X.c || Y.r != X.r || Y.c != X.c) throw ShapeError("inverse needs square blocks");
  const unsigned long long key = (order << 32) | (uint64_t)(uint32_t)index;
  double2* work = inv_work(std::max<int64_t>(block_inverse_workspace(X.r), 1));
  // Inner GEMM launches of the inverse are attributed to the inverse, not the GEMM kernel.
  const bool prof = profiling();
  int id = prof ? profile_open(s) : -1;
  if (prof) profile_suspend(true);
  cudaError_t e = launch_block_inverse(X.p, X.ld, Y.p, Y.ld, X.r, work, d_flag_, d_status_, key, s);
  if (prof) profile_suspend(false);
  profile_close(id, s, 1, 8.0 * X.r * (double)X.r * X.r);
  cuda_check(e, "block inverse");
}

SingularInfo Context::read_status() {
  unsigned long long st = 0;
  cuda_check(cudaMemcpyAsync(&st, d_status_, sizeof(st), cudaMemcpyDeviceToHost, user_stream_), "status d2h");
  cuda_check(cudaStreamSynchronize(user_stream_), "status sync");
  SingularInfo info;
  if (st != ~0ull) {
    info.singular = true;
    info.index = (int64_t)(uint32_t)(st & 0xffffffffu);
  }
  return info;
}

cudaEvent_t Context::event(int i) { return events_.at(i); }
cudaEvent_t Context::timer(int i) { return timers_[i]; }

namespace {

inline Mat cm(const double2* p, int r, int c) { return Mat{const_cast<double2*>(p), c, r, c}; }

// Copy a block (elementwise level with a single addend).
void copy_block(Level& L, Mat dst, Mat src) { L.out(dst).add(+1, src); }

// ---------------------------------------------------------------------------
// Forward sweeps
// ---------------------------------------------------------------------------

// rgf.py:79-124 (Alg. 1), BT.
void bt_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F) {
  const int n = (int)A.n, b = (int)A.b;
  cudaStream_t sA = ctx.stream(), sB = ctx.aux();
  const bool fused = B != nullptr;
  ctx.reserve_slots(8, (int64_t)b * b);
  for (int i = 0; i < n - 1; ++i) {
    const int r = (i & 1) * 4;
    Mat S = F.SA(i), t1 = ctx.tmp(r + 0, b, b);
    ctx.invert(A.D(i), S, i, i, sA);
    if (fused && i >= 2) cuda_check(cudaStreamWaitEvent(sA, ctx.event(2 + (i & 1)), 0), "wait B");
    {
      Level L(sA);
      L.out(t1).mm(+1, A.L(i), N, S, N);
      L.flush();
    }
    if (fused) cuda_check(cudaEventRecord(ctx.event(i & 1), sA), "record A");
    {
      Level L(sA);
      L.out(A.D(i + 1)).add(+1, A.D(i + 1)).mm(-1, t1, N, A.U(i), N);
      L.flush();
    }
    if (fused) {
      cuda_check(cudaStreamWaitEvent(sB, ctx.event(i & 1), 0), "wait A");
      Mat w = ctx.tmp(r + 1, b, b), v = ctx.tmp(r + 2, b, b), sb = F.SB(i);
      Level L(sB);
      L.out(w).mm(+1, S, N, B->D(i), N);
      L.flush();
      L.out(sb).mm(+1, w, N, S, H);
      L.flush();
      L.out(v).mm(+1, A.L(i), N, sb, N);
      L.flush();
      L.out(B->D(i + 1))
          .add(+1, B->D(i + 1))
          .mm(+1, v, N, A.L(i), H)
          .mm(-1, B->L(i), N, t1, H)
          .mm(-1, t1, N, B->U(i), N);
      L.flush();
      cuda_check(cudaEventRecord(ctx.event(2 + (i & 1)), sB), "record B");
    }
  }
  ctx.invert(A.D(n - 1), F.SA(n - 1), n - 1, n - 1, sA);
  if (fused) {
    Level L(sB);
    copy_block(L, cm(F.b_diag_last, b, b), B->D(n - 1));
    L.flush();
  }
}

// rgf.py:207-319, BTA (a > 0).
void bta_forward_arrow(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F) {
  const int n = (int)A.n, b = (int)A.b, a = (int)A.a;
  cudaStream_t sA = ctx.stream(), sB = ctx.aux();
  const bool fused = B != nullptr;
  const int mx = std::max(a, b);
  ctx.reserve_slots(16, (int64_t)mx * mx);
  for (int i = 0; i < n - 1; ++i) {
    Mat S = F.SA(i);
    ctx.invert(A.D(i), S, i, i, sA);
    if (!fused) {
      // rgf.py:281-288: right-hand temporaries.
      Mat t1 = ctx.tmp(0, b, b), t2 = ctx.tmp(1, b, a);
      Level L(sA);
      L.out(t1).mm(+1, S, N, A.U(i), N);
      L.out(t2).mm(+1, S, N, A.AC(i), N);
      L.flush();
      L.out(A.D(i + 1)).add(+1, A.D(i + 1)).mm(-1, A.L(i), N, t1, N);
      L.out(A.AR(i + 1)).add(+1, A.AR(i + 1)).mm(-1, A.AR(i), N, t1, N);
      L.out(A.AC(i + 1)).add(+1, A.AC(i + 1)).mm(-1, A.L(i), N, t2, N);
      L.out(A.T()).add(+1, A.T()).mm(-1, A.AR(i), N, t2, N);
      L.flush();
      continue;
    }
    // rgf.py:246-280, fused.
    const int r = (i & 1) * 8;
    Mat f = ctx.tmp(r + 0, b, b), g = ctx.tmp(r + 1, a, b), w = ctx.tmp(r + 2, b, b);
    Mat p = ctx.tmp(r + 3, a, b), k = ctx.tmp(r + 4, b, a), v = ctx.tmp(r + 5, b, b);
    Mat sb = F.SB(i);
    if (i >= 2) cuda_check(cudaStreamWaitEvent(sA, ctx.event(2 + (i & 1)), 0), "wait B");
    {
      Level L(sA);
      L.out(f).mm(+1, A.L(i), N, S, N);
      L.out(g).mm(+1, A.AR(i), N, S, N);
      L.flush();
    }
    cuda_check(cudaEventRecord(ctx.event(i & 1), sA), "record A");
    {
      Level L(sA);
      L.out(A.D(i + 1)).add(+1, A.D(i + 1)).mm(-1, f, N, A.U(i), N);
      L.out(A.AR(i + 1)).add(+1, A.AR(i + 1)).mm(-1, g, N, A.U(i), N);
      L.out(A.AC(i + 1)).add(+1, A.AC(i + 1)).mm(-1, f, N, A.AC(i), N);
      L.out(A.T()).add(+1, A.T()).mm(-1, g, N, A.AC(i), N);
      L.flush();
    }
    cuda_check(cudaStreamWaitEvent(sB, ctx.event(i & 1), 0), "wait A");
    {
      Level L(sB);
      L.out(w).mm(+1, S, N, B->D(i), N);
      L.out(p).mm(+1, g, N, B->D(i), N);
      L.out(k).mm(+1, B->D(i), N, g, H);
      L.flush();
      L.out(sb).mm(+1, w, N, S, H);
      L.flush();
      L.out(v).mm(+1, A.L(i), N, sb, N);
      L.out(B->AR(i + 1))
          .add(+1, B->AR(i + 1))
          .mm(-1, g, N, B->U(i), N)
          .mm(+1, p, N, f, H)
          .mm(-1, B->AR(i), N, f, H);
      L.out(B->AC(i + 1))
          .add(+1, B->AC(i + 1))
          .mm(-1, f, N, B->AC(i), N)
          .mm(-1, B->L(i), N, g, H)
          .mm(+1, f, N, k, N);
      L.out(B->T())
          .add(+1, B->T())
          .mm(-1, g, N, B->AC(i), N)
          .mm(-1, B->AR(i), N, g, H)
          .mm(+1, p, N, g, H);
      L.flush();
      L.out(B->D(i + 1))
          .add(+1, B->D(i + 1))
          .mm(+1, v, N, A.L(i), H)
          .mm(-1, B->L(i), N, f, H)
          .mm(-1, f, N, B->U(i), N);
      L.flush();
    }
    cuda_check(cudaEventRecord(ctx.event(2 + (i & 1)), sB), "record B");
  }
  // Epilogue (rgf.py:290-318): eliminate block n-1 into the tip, invert it.
  const int i = n - 1;
  Mat S = F.SA(i);
  ctx.invert(A.D(i), S, i, i, sA);
  if (!fused) {
    Mat t2 = ctx.tmp(0, b, a);
    Level L(sA);
    L.out(t2).mm(+1, S, N, A.AC(i), N);
    L.flush();
    L.out(A.T()).add(+1, A.T()).mm(-1, A.AR(i), N, t2, N);
    L.flush();
  } else {
    const int r = (i & 1) * 8;
    Mat g = ctx.tmp(r + 1, a, b), p = ctx.tmp(r + 3, a, b);
    if (i >= 2) cuda_check(cudaStreamWaitEvent(sA, ctx.event(2 + (i & 1)), 0), "wait B");
    Level L(sA);
    L.out(g).mm(+1, A.AR(i), N, S, N);
    L.flush();
    cuda_check(cudaEventRecord(ctx.event(i & 1), sA), "record A");
    L.out(A.T()).add(+1, A.T()).mm(-1, g, N, A.AC(i), N);
    L.flush();
    cuda_check(cudaStreamWaitEvent(sB, ctx.event(i & 1), 0), "wait A");
    Level LB(sB);
    LB.out(p).mm(+1, g, N, B->D(i), N);
    copy_block(LB, cm(F.b_diag_last, b, b), B->D(i));
    LB.flush();
    LB.out(B->T())
        .add(+1, B->T())
        .mm(-1, g, N, B->AC(i), N)
        .mm(-1, B->AR(i), N, g, H)
        .mm(+1, p, N, g, H);
    LB.flush();
    copy_block(LB, cm(F.b_tip, a, a), B->T());
    LB.flush();
  }
  ctx.invert(A.T(), cm(F.tip_inv, a, a), n, n, sA);
}

// ---------------------------------------------------------------------------
// Backward sweeps
// ---------------------------------------------------------------------------

// rgf.py:127-199 (Alg. 2), BT.
void bt_backward(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B, const BtaDev& XA,
                 const BtaDev* XB, bool diag_only) {
  const int n = (int)A.n, b = (int)A.b;
  cudaStream_t s = ctx.stream();
  const bool fused = B != nullptr;
  ctx.reserve_slots(16, (int64_t)b * b);
  Level L(s);
  copy_block(L, XA.D(n - 1), F.SA(n - 1));
  if (fused) {
    Mat w = ctx.tmp(0, b, b);
    L.out(w).mm(+1, F.SA(n - 1), N, cm(F.b_diag_last, b, b), N);
    L.flush();
    L.out(XB->D(n - 1)).mm(+1, w, N, F.SA(n - 1), H);
  }
  L.flush();
  for (int i = n - 2; i >= 0; --i) {
    Mat S = F.SA(i), Xp = XA.D(i + 1);
    Mat tA1 = ctx.tmp(0, b, b), tA2 = ctx.tmp(1, b, b);
    Mat xlo = diag_only ? ctx.tmp(2, b, b) : XA.L(i);
    Mat xup = diag_only ? ctx.tmp(3, b, b) : XA.U(i);
    L.out(tA1).mm(+1, S, N, A.U(i), N);
    L.out(tA2).mm(+1, Xp, N, A.L(i), N);
    Mat sbu = ctx.tmp(4, b, b), xbl = ctx.tmp(5, b, b);
    if (fused) {
      L.out(sbu).mm(+1, S, N, B->U(i), N);
      L.out(xbl).mm(+1, Xp, N, B->L(i), N);
    }
    L.flush();
    L.out(xlo).mm(-1, tA2, N, S, N);
    L.out(xup).mm(-1, tA1, N, Xp, N);
    Mat tB1 = ctx.tmp(6, b, b), tB2 = ctx.tmp(7, b, b), tB3 = ctx.tmp(8, b, b);
    Mat tB4 = ctx.tmp(9, b, b), tB5 = ctx.tmp(10, b, b);
    Mat Zp, sb;
    if (fused) {
      Zp = XB->D(i + 1);
      sb = F.SB(i);
      L.out(tB1).mm(+1, Zp, N, tA1, H);
      L.out(tB2).mm(+1, sb, N, tA2, H);
      L.out(tB3).mm(+1, tA2, N, sb, N);
      L.out(tB4).mm(+1, sbu, N, Xp, H);
      L.out(tB5).mm(+1, xbl, N, S, H);
    }
    L.flush();
    L.out(XA.D(i)).add(+1, S).mm(-1, tA1, N, xlo, N);
    if (fused) {
      Mat xbup = diag_only ? ctx.tmp(11, b, b) : XB->U(i);
      Mat xblo = diag_only ? ctx.tmp(12, b, b) : XB->L(i);
      L.out(xbup).add(+1, tB4).add(-1, tB2).mm(-1, tA1, N, Zp, N);
      L.out(xblo).add(-1, tB1).add(-1, tB3).add(+1, tB5);
      L.out(XB->D(i))
          .add(+1, sb)
          .mm(+1, tA1, N, tB1, N)
          .mm(+1, tA1, N, tB3, N)
          .mm(+1, tB2, N, tA1, H)
          .mm(-1, tA1, N, tB5, N)
          .mm(-1, tB4, N, tA1, H);
    }
    L.flush();
  }
}

// rgf.py:322-398 (_backstep, k = 1 and k = 2) driven by rgf.py:401-489.
void bta_backward_arrow(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B,
                        const BtaDev& XA, const BtaDev* XB, bool diag_only) {
  const int n = (int)A.n, b = (int)A.b, a = (int)A.a;
  cudaStream_t s = ctx.stream();
  const bool fused = B != nullptr;
  const int mx = std::max(a, b);
  ctx.reserve_slots(24, (int64_t)mx * mx);
  Mat Xtt = cm(F.tip_inv, a, a);
  Mat Ztt;
  Level L(s);
  copy_block(L, XA.T(), Xtt);
  if (fused) {
    Mat w = ctx.tmp(0, a, a);
    L.out(w).mm(+1, Xtt, N, cm(F.b_tip, a, a), N);
    L.flush();
    L.out(XB->T()).mm(+1, w, N, Xtt, H);
    Ztt = XB->T();
  }
  L.flush();

  // ---- i = n-1: one trailing coupling (the tip) ----
  {
    const int i = n - 1;
    Mat g = F.SA(i), ACe = F.ACe(i), ARe = F.ARe(i);
    Mat RA = ctx.tmp(0, b, a), CA = ctx.tmp(1, a, b), phi = ctx.tmp(2, b, b);
    L.out(RA).mm(+1, ACe, N, Xtt, N);
    L.out(CA).mm(+1, Xtt, N, ARe, N);
    Mat RZ = ctx.tmp(3, b, a), CZ = ctx.tmp(4, a, b), sct = ctx.tmp(5, b, b), sc = ctx.tmp(6, b, b);
    Mat quad = ctx.tmp(7, b, b), e0 = ctx.tmp(8, b, a), f0 = ctx.tmp(9, a, b);
    Mat acc1 = ctx.tmp(10, b, b), acc2 = ctx.tmp(11, b, b), gq = ctx.tmp(12, b, b);
    if (fused) {
      L.out(RZ).mm(+1, ACe, N, Ztt, N);
      L.out(CZ).mm(+1, Ztt, N, ACe, H);
      L.out(sct).mm(+1, g, N, cm(F.b_diag_last, b, b), N);
    }
    L.flush();
    Mat xrow = XA.AC(i), xcol = XA.AR(i);
    L.out(xrow).mm(-1, g, N, RA, N);
    L.out(xcol).mm(-1, CA, N, g, N);
    if (fused) {
      L.out(sc).mm(+1, sct, N, g, H);
      L.out(quad).mm(+1, ACe, N, CZ, N);
    }
    L.flush();
    L.out(phi).mm(-1, xrow, N, ARe, N);
    if (fused) {
      Mat BCe = F.BCe(i), BRe = F.BRe(i);
      L.out(e0).mm(+1, g, N, BCe, N).mm(-1, sc, N, ARe, H);
      L.out(f0).mm(+1, BRe, N, g, H).mm(-1, ARe, N, sc, N);
      L.out(acc1).mm(+1, BCe, N, xrow, H);
      L.out(acc2).mm(+1, xrow, N, BRe, N);
      L.out(gq).mm(+1, g, N, quad, N);
    }
    L.flush();
    L.out(XA.D(i)).add(+1, g).mm(+1, phi, N, g, N);
    if (fused) {
      L.out(XB->AC(i)).mm(+1, e0, N, Xtt, H).mm(-1, g, N, RZ, N);
      L.out(XB->AR(i)).mm(+1, Xtt, N, f0, N).mm(-1, CZ, N, g, H);
      L.out(XB->D(i))
          .add(+1, sc)
          .mm(+1, phi, N, sc, N)
          .mm(+1, sc, N, phi, H)
          .mm(+1, g, N, acc1, N)
          .mm(+1, acc2, N, g, H)
          .mm(+1, gq, N, g, H);
    }
    L.flush();
  }

  // ---- i = n-2 .. 0: two trailing couplings (next diagonal block, tip) ----
  for (int i = n - 2; i >= 0; --i) {
    Mat g = F.SA(i), U = A.U(i), Lo = A.L(i), ACe = F.ACe(i), ARe = F.ARe(i);
    Mat Ydd = XA.D(i + 1), Ydt = XA.AC(i + 1), Ytd = XA.AR(i + 1), Ytt = Xtt;
    Mat RA0 = ctx.tmp(0, b, b), RA1 = ctx.tmp(1, b, a), CA0 = ctx.tmp(2, b, b), CA1 = ctx.tmp(3, a, b);
    L.out(RA0).mm(+1, U, N, Ydd, N).mm(+1, ACe, N, Ytd, N);
    L.out(RA1).mm(+1, U, N, Ydt, N).mm(+1, ACe, N, Ytt, N);
    L.out(CA0).mm(+1, Ydd, N, Lo, N).mm(+1, Ydt, N, ARe, N);
    L.out(CA1).mm(+1, Ytd, N, Lo, N).mm(+1, Ytt, N, ARe, N);
    Mat RZ0 = ctx.tmp(4, b, b), RZ1 = ctx.tmp(5, b, a), CZ0 = ctx.tmp(6, b, b), CZ1 = ctx.tmp(7, a, b);
    Mat e0 = ctx.tmp(8, b, b), e1 = ctx.tmp(9, b, a), f0 = ctx.tmp(10, b, b), f1 = ctx.tmp(11, a, b);
    Mat Zdd, Zdt, Ztd, sc, BU, BL, BCe, BRe;
    if (fused) {
      Zdd = XB->D(i + 1);
      Zdt = XB->AC(i + 1);
      Ztd = XB->AR(i + 1);
      sc = F.SB(i);
      BU = B->U(i);
      BL = B->L(i);
      BCe = F.BCe(i);
      BRe = F.BRe(i);
      L.out(RZ0).mm(+1, U, N, Zdd, N).mm(+1, ACe, N, Ztd, N);
      L.out(RZ1).mm(+1, U, N, Zdt, N).mm(+1, ACe, N, Ztt, N);
      L.out(CZ0).mm(+1, Zdd, N, U, H).mm(+1, Zdt, N, ACe, H);
      L.out(CZ1).mm(+1, Ztd, N, U, H).mm(+1, Ztt, N, ACe, H);
      L.out(e0).mm(+1, g, N, BU, N).mm(-1, sc, N, Lo, H);
      L.out(e1).mm(+1, g, N, BCe, N).mm(-1, sc, N, ARe, H);
      L.out(f0).mm(+1, BL, N, g, H).mm(-1, Lo, N, sc, N);
      L.out(f1).mm(+1, BRe, N, g, H).mm(-1, ARe, N, sc, N);
    }
    L.flush();
    Mat xr0 = diag_only ? ctx.tmp(12, b, b) : XA.U(i);
    Mat xc0 = diag_only ? ctx.tmp(13, b, b) : XA.L(i);
    Mat xr1 = XA.AC(i), xc1 = XA.AR(i);
    L.out(xr0).mm(-1, g, N, RA0, N);
    L.out(xr1).mm(-1, g, N, RA1, N);
    L.out(xc0).mm(-1, CA0, N, g, N);
    L.out(xc1).mm(-1, CA1, N, g, N);
    Mat quad = ctx.tmp(14, b, b);
    if (fused) {
      Mat zr0 = diag_only ? ctx.tmp(15, b, b) : XB->U(i);
      Mat zc0 = diag_only ? ctx.tmp(16, b, b) : XB->L(i);
      L.out(zr0).mm(+1, e0, N, Ydd, H).mm(+1, e1, N, Ydt, H).mm(-1, g, N, RZ0, N);
      L.out(XB->AC(i)).mm(+1, e0, N, Ytd, H).mm(+1, e1, N, Ytt, H).mm(-1, g, N, RZ1, N);
      L.out(zc0).mm(+1, Ydd, N, f0, N).mm(+1, Ydt, N, f1, N).mm(-1, CZ0, N, g, H);
      L.out(XB->AR(i)).mm(+1, Ytd, N, f0, N).mm(+1, Ytt, N, f1, N).mm(-1, CZ1, N, g, H);
      L.out(quad).mm(+1, U, N, CZ0, N).mm(+1, ACe, N, CZ1, N);
    }
    L.flush();
    Mat phi = ctx.tmp(17, b, b), acc1 = ctx.tmp(18, b, b), acc2 = ctx.tmp(19, b, b), gq = ctx.tmp(20, b, b);
    L.out(phi).mm(-1, xr0, N, Lo, N).mm(-1, xr1, N, ARe, N);
    if (fused) {
      L.out(acc1).mm(+1, BU, N, xr0, H).mm(+1, BCe, N, xr1, H);
      L.out(acc2).mm(+1, xr0, N, BL, N).mm(+1, xr1, N, BRe, N);
      L.out(gq).mm(+1, g, N, quad, N);
    }
    L.flush();
    L.out(XA.D(i)).add(+1, g).mm(+1, phi, N, g, N);
    if (fused) {
      L.out(XB->D(i))
          .add(+1, sc)
          .mm(+1, phi, N, sc, N)
          .mm(+1, sc, N, phi, H)
          .mm(+1, g, N, acc1, N)
          .mm(+1, acc2, N, g, H)
          .mm(+1, gq, N, g, H);
    }
    L.flush();
  }
}

}  // namespace

void bta_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F) {
  if (A.n < 1 || A.b < 1 || A.a < 0) throw ShapeError("invalid shape parameters");
  if (B && (B->n != A.n || B->b != A.b || B->a != A.a))
    throw ShapeError("right-hand side shape differs from system shape");
  cudaStream_t s = ctx.stream();
  ctx.reset_status();
  cuda_check(cudaEventRecord(ctx.timer(0), s), "timer");
  cuda_check(cudaEventRecord(ctx.event(4), s), "fork");
  cuda_check(cudaStreamWaitEvent(ctx.aux(), ctx.event(4), 0), "fork wait");
  if (A.a == 0)
    bt_forward(ctx, A, B, F);
  else
    bta_forward_arrow(ctx, A, B, F);
  cuda_check(cudaEventRecord(ctx.event(5), ctx.aux()), "join");
  cuda_check(cudaStreamWaitEvent(s, ctx.event(5), 0), "join wait");
  cuda_check(cudaEventRecord(ctx.timer(1), s), "timer");
}

void bta_backward(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B, const BtaDev& XA,
                  const BtaDev* XB, bool diagonal_only) {
  if (A.n != F.n || A.b != F.b || A.a != F.a) throw ShapeError("system shape disagrees with factors");
  if (F.fused && !B) throw ShapeError("fused factors require the right-hand side");
  if (!F.fused) {
    B = nullptr;
    XB = nullptr;
  }
  cudaStream_t s = ctx.stream();
  cuda_check(cudaEventRecord(ctx.timer(2), s), "timer");
  if (A.a == 0)
    bt_backward(ctx, F, A, B, XA, XB, diagonal_only);
  else
    bta_backward_arrow(ctx, F, A, B, XA, XB, diagonal_only);
  cuda_check(cudaEventRecord(ctx.timer(3), s), "timer");
}

}  // namespace bsel
