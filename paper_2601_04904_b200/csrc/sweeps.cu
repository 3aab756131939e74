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
#include <cstdlib>
#include <cstring>

#include "inverse.cuh"
#include "solver.cuh"
#include "steps.cuh"
#include "symmetry.cuh"

namespace bsel {

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------

Context::Context(int device) : device_(device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  int least = 0, greatest = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&aux_, cudaStreamNonBlocking, least), "aux stream");
  cuda_check(cudaStreamCreateWithPriority(&chain_, cudaStreamNonBlocking, greatest), "chain stream");
  cuda_check(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, least), "side stream");
  cuda_check(cudaMalloc(&d_flag_, sizeof(int)), "flag");
  cuda_check(cudaMalloc(&d_status_, sizeof(unsigned long long)), "status");
  cuda_check(cudaMalloc(&d_sym_, sizeof(int)), "symmetry flags");
  cuda_check(cudaMalloc(&d_aux_counter_, 2 * sizeof(unsigned)), "aux tile counter");
  cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&h_flags_), sizeof(HostFlags), cudaHostAllocMapped),
             "mapped flags");
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hflags_), h_flags_, 0), "mapped flags pointer");
  events_.resize(64);
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
  if (d_sym_) cudaFree(d_sym_);
  if (d_aux_counter_) cudaFree(d_aux_counter_);
  if (h_flags_) cudaFreeHost(h_flags_);
  for (auto& e : events_) cudaEventDestroy(e);
  for (auto& t : timers_) cudaEventDestroy(t);
  for (auto& e : xfer_events_) cudaEventDestroy(e);
  if (xfer_) cudaStreamDestroy(xfer_);
  if (aux_) cudaStreamDestroy(aux_);
  if (chain_) cudaStreamDestroy(chain_);
  if (side_) cudaStreamDestroy(side_);
}

cudaStream_t Context::xfer() {
  if (!xfer_) cuda_check(cudaStreamCreateWithFlags(&xfer_, cudaStreamNonBlocking), "copy stream");
  return xfer_;
}

cudaEvent_t Context::xfer_event(int i) {
  while ((int)xfer_events_.size() <= i) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    xfer_events_.push_back(e);
  }
  return xfer_events_[i];
}

void Context::reserve_slots(int nslots, int64_t slot_elems) {
  if (nslots <= nslots_ && slot_elems <= slot_elems_) return;
  cuda_check(cudaStreamSynchronize(user_stream_), "sync before realloc");
  cuda_check(cudaStreamSynchronize(aux_), "sync before realloc");
  cuda_check(cudaStreamSynchronize(chain_), "sync before realloc");
  cuda_check(cudaStreamSynchronize(side_), "sync before realloc");
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
    cuda_check(cudaStreamSynchronize(chain_), "sync before realloc");
    if (inv_work_) cudaFree(inv_work_);
    cuda_check(cudaMalloc(&inv_work_, (size_t)elems * sizeof(double2)), "inverse workspace");
    // the inverse's sync area (epoch-tagged flags, never reset) starts at zero
    cuda_check(cudaMemset(inv_work_, 0, (size_t)elems * sizeof(double2)), "inverse workspace init");
    cuda_check(cudaDeviceSynchronize(), "inverse workspace init");
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
  cudaError_t e = launch_block_inverse(X.p, X.ld, Y.p, Y.ld, X.r, work, d_flag_, d_status_, key, s, inv_grid_);
  if (prof) profile_suspend(false);
  profile_close(id, s, 1, 8.0 * X.r * (double)X.r * X.r);
  cuda_check(e, "block inverse");
}

void Context::sym_reset(cudaStream_t s) {
  cuda_check(cudaMemsetAsync(d_sym_, 0, sizeof(int), s), "memset symmetry flags");
  sym_checked_ = false;
}

void Context::sym_check(const SymJob& j, cudaStream_t s) {
  cuda_check(launch_sym_check(j, d_sym_, s), "symmetry check");
  sym_checked_ = true;
}

__global__ void publish_flags_kernel(const unsigned long long* status, const int* sym,
                                     volatile Context::HostFlags* out) {
  out->status = *status;
  out->sym = *sym;
  __threadfence_system();
}

void Context::publish_flags(cudaStream_t s) {
  publish_flags_kernel<<<1, 1, 0, s>>>(d_status_, d_sym_, d_hflags_);
  cuda_check(cudaGetLastError(), "publish flags");
  cuda_check(cudaStreamSynchronize(s), "flags sync");
}

int Context::sym_now(cudaStream_t s) {
  publish_flags(s);
  const int f = reinterpret_cast<volatile HostFlags*>(h_flags_)->sym;
  if (!sym_checked_) return 0;
  sym_flags_ = f;
  return !(f & kNotHermitian) ? +1 : !(f & kNotSkew) ? -1 : 0;
}

int Context::b_symmetry() const {
  if (sym_mode_ != kSymAuto) return sym_mode_;
  if (!sym_checked_) return 0;
  if (!(sym_flags_ & kNotHermitian)) return +1;
  if (!(sym_flags_ & kNotSkew)) return -1;
  return 0;
}

// The fused Schur step is opt-in (BSEL_SCHUR=1, read per call): alone it
// beats inverse + 2 GEMMs (SI chain 422 vs 453 us per step at b=512), but its
// 4x larger rank-32 panel updates lose more under the quadratic solve's
// concurrent GEMM levels (cfg4, 2 lanes: forward 700 vs 565 ms).
bool Context::schur_ok(int b) const {
  const char* e = getenv("BSEL_SCHUR");
  return e && atoi(e) != 0 && schur_step_supported(b);
}

void Context::schur(Mat D, Mat U, Mat L, Mat C, Mat S, Mat H, Mat F, uint64_t order, int64_t index,
                    cudaStream_t s) {
  const int b = D.r;
  for (const Mat* m : {&D, &U, &L, &C, &S, &F})
    if (m->r != b || m->c != b) throw ShapeError("Schur step needs square blocks of one size");
  if (H.p && (H.r != b || H.c != b)) throw ShapeError("Schur step H shape");
  const unsigned long long key = (order << 32) | (uint64_t)(uint32_t)index;
  double2* work = inv_work(schur_step_workspace(b));
  int id = profiling() ? profile_open(s) : -1;
  // executed: the inverse and the three products it absorbs (L S, S U, (L S) U)
  cudaError_t e = launch_schur_step(D.p, D.ld, U.p, U.ld, L.p, L.ld, C.p, C.ld, S.p, S.ld, H.p, H.ld, F.p, F.ld,
                                    b, work, d_flag_, d_status_, key, s, inv_grid_ > 0 ? 2 * inv_grid_ : 0);
  profile_close(id, s, 1, 32.0 * b * (double)b * b);
  cuda_check(e, "Schur step");
}

SingularInfo Context::read_status() {
  publish_flags(user_stream_);
  const unsigned long long st = reinterpret_cast<volatile HostFlags*>(h_flags_)->status;
  sym_flags_ = reinterpret_cast<volatile HostFlags*>(h_flags_)->sym;
  SingularInfo info;
  if (st != ~0ull) {
    info.singular = true;
    info.index = (int64_t)(uint32_t)(st & 0xffffffffu);
  }
  return info;
}

void sym_check_strips(Context& ctx, const BtaDev& src, int64_t src_lo, int64_t g0, int64_t g1, const BtaDev* dst,
                      int64_t dst_lo, cudaStream_t s) {
  if (g1 <= g0) return;
  const int64_t b = src.b, a = src.a, o = g0 - src_lo, od = g0 - dst_lo;
  SymJob d;
  d.X = d.Y = src.diag + o * b * b;
  d.r = d.c = (int)b;
  d.sx = d.sy = b * b;
  d.count = g1 - g0;
  d.same = true;
  if (dst) d.dX = d.dY = dst->diag + od * b * b;
  ctx.sym_check(d, s);
  if (a == 0) return;
  SymJob r;
  r.X = src.arrow_row + o * a * b;
  r.Y = src.arrow_col + o * b * a;
  r.r = (int)a, r.c = (int)b;
  r.sx = r.sy = a * b;
  r.count = g1 - g0;
  if (dst) r.dX = dst->arrow_row + od * a * b, r.dY = dst->arrow_col + od * b * a;
  ctx.sym_check(r, s);
}

void sym_check_couplings(Context& ctx, const BtaDev& src, int64_t e0, int64_t e1, cudaStream_t s) {
  if (e1 <= e0) return;
  const int64_t b = src.b;
  SymJob j;
  j.X = src.lower + e0 * b * b;
  j.Y = src.upper + e0 * b * b;
  j.r = j.c = (int)b;
  j.sx = j.sy = b * b;
  j.count = e1 - e0;
  ctx.sym_check(j, s);
}

void sym_check_tip(Context& ctx, const BtaDev& src, double2* dst_tip, cudaStream_t s) {
  if (src.a == 0) return;
  SymJob j;
  j.X = j.Y = src.tip;
  j.r = j.c = (int)src.a;
  j.count = 1;
  j.same = true;
  j.dX = j.dY = dst_tip;
  ctx.sym_check(j, s);
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
  cudaStream_t sA = ctx.chain(), sB = ctx.aux();
  const bool fused = B != nullptr;
  ctx.reserve_slots(8, (int64_t)b * b);
  for (int i = 0; i < n - 1; ++i) {
    const int r = (i & 1) * 4;
    Mat S = F.SA(i), t1 = F.elim_f ? F.EF(i) : ctx.tmp(r + 0, b, b);
    if (fused && i >= 2) cuda_check(cudaStreamWaitEvent(sA, ctx.event(2 + (i & 1)), 0), "wait B");
    if (ctx.schur_ok(b)) {
      // inverse, t1 = L S and D(i+1) -= t1 U in one persistent launch
      ctx.schur(A.D(i), A.U(i), A.L(i), A.D(i + 1), S, F.EH(i), t1, i, i, sA);
      if (fused) cuda_check(cudaEventRecord(ctx.event(i & 1), sA), "record A");
    } else {
      ctx.invert(A.D(i), S, i, i, sA);
      Level L(sA);
      L.out(t1).mm(+1, A.L(i), N, S, N);
      L.flush();
      if (fused) cuda_check(cudaEventRecord(ctx.event(i & 1), sA), "record A");
      L.out(A.D(i + 1)).add(+1, A.D(i + 1)).mm(-1, t1, N, A.U(i), N);
      L.flush();
    }
    if (fused) {
      cuda_check(cudaStreamWaitEvent(sB, ctx.event(i & 1), 0), "wait A");
      // v L^H - t1 BU = L S_B L^H - t1 BU = t1 (Bd t1^H - BU): two levels,
      // one product fewer than rgf.py:113-118.
      Mat w = ctx.tmp(r + 1, b, b), q = F.elim_q ? F.EQ(i) : ctx.tmp(r + 2, b, b), sb = F.SB(i);
      Level L(sB, kTileAutoFwd);
      L.out(w).mm(+1, S, N, B->D(i), N);
      L.out(q).add(-1, B->U(i)).mm(+1, B->D(i), N, t1, H);
      L.flush();
      L.out(sb).mm(+1, w, N, S, H);
      L.out(B->D(i + 1)).add(+1, B->D(i + 1)).mm(+1, t1, N, q, N).mm(-1, B->L(i), N, t1, H);
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

// rgf.py:207-319, BTA (a > 0): n-1 elimination steps (steps.cu end_step),
// then the last block is eliminated into the tip and the tip is inverted.
void bta_forward_arrow(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F) {
  const int n = (int)A.n, b = (int)A.b, a = (int)A.a;
  cudaStream_t sA = ctx.chain(), sB = ctx.aux();
  const bool fused = B != nullptr;
  const int mx = std::max(a, b);
  ctx.reserve_slots(64, (int64_t)mx * mx);
  for (int i = 0; i < n - 1; ++i) {
    EndStep st;  // (end_step waits for the ring slot after its inverse)
    st.Lk = A.L(i), st.Uk = A.U(i);
    st.ad_i = A.D(i), st.ad_j = A.D(i + 1), st.ar_i = A.AR(i), st.ar_j = A.AR(i + 1);
    st.ac_i = A.AC(i), st.ac_j = A.AC(i + 1), st.tipA = A.T();
    st.S = F.SA(i);
    if (fused) {
      st.BL = B->L(i), st.BU = B->U(i);
      st.bd_i = B->D(i), st.bd_j = B->D(i + 1), st.br_i = B->AR(i), st.br_j = B->AR(i + 1);
      st.bc_i = B->AC(i), st.bc_j = B->AC(i + 1), st.tipB = B->T();
      st.sb = F.SB(i);
      st.f_out = F.EF(i), st.g_out = F.EG(i), st.q_out = F.EQ(i), st.k_out = F.EK(i);
      if (fwd_backward_products()) st.eq_out = F.EEQ(i), st.ek_out = F.EEK(i);
    }
    // SI: h = S U and S AC_i are the forward's own temporaries; fused: only
    // with the Schur step (h) or BSEL_FWD_BWD_PRODUCTS
    const bool extra = !fused || fwd_backward_products();
    if (extra || ctx.schur_ok(b)) st.h_out = F.EH(i);
    if (extra) st.ha_out = F.EHA(i);
    end_step(ctx, st, fused, i, i, fwd_slot(i));
  }
  // Epilogue (rgf.py:290-318).  The last block's arrow strips and the tip
  // were updated on the aux stream: the chain waits for the last step's aux.
  const int i = n - 1;
  if (n >= 2) cuda_check(cudaStreamWaitEvent(sA, ring_b_event(ctx, fwd_slot(n - 2)), 0), "aux done");
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
    const int r = fwd_slot(i) * 8;
    Mat g = ctx.tmp(r + 1, a, b), p = ctx.tmp(r + 3, a, b);
    ring_wait(ctx, i);
    Level L(sA);
    L.out(g).mm(+1, A.AR(i), N, S, N);
    L.flush();
    cuda_check(cudaEventRecord(ring_a_event(ctx, fwd_slot(i)), sA), "record A");
    L.out(A.T()).add(+1, A.T()).mm(-1, g, N, A.AC(i), N);
    L.flush();
    cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, fwd_slot(i)), 0), "wait A");
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

// rgf.py:127-199 (Alg. 2), BT: the generic back step with k = 1 (rs = U,
// qs = L), i.e. X_up = -(S U) X+, X_lo = -X+ (L S), X_dd = S - X_up (L S)
// and the same re-association of the quadratic terms (steps.cuh).
void bt_backward(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B, const BtaDev& XA,
                 const BtaDev* XB, bool diag_only) {
  const int n = (int)A.n, b = (int)A.b;
  cudaStream_t s = ctx.stream();
  const bool fused = B != nullptr;
  ctx.reserve_slots(back_sweep_slots(), (int64_t)b * b);
  Level L(s);
  copy_block(L, XA.D(n - 1), F.SA(n - 1));
  if (fused) {
    Mat w = ctx.tmp(0, b, b);
    L.out(w).mm(+1, F.SA(n - 1), N, cm(F.b_diag_last, b, b), N);
    L.flush();
    L.out(XB->D(n - 1)).mm(+1, w, N, F.SA(n - 1), H);
  }
  L.flush();
  BackSweep sweep(ctx);
  sweep.begin();
  for (int i = n - 2; i >= 0; --i) {
    BackStep st;
    st.k = 1;
    st.g = F.SA(i);
    st.rs[0] = A.U(i), st.qs[0] = A.L(i);
    st.ya[0][0] = XA.D(i + 1);
    if (!diag_only) st.row[0] = XA.U(i), st.col[0] = XA.L(i);
    st.diag = XA.D(i);
    if (fused) {
      st.sc = F.SB(i);
      st.ss[0] = B->U(i), st.ws[0] = B->L(i);
      st.cpre[0] = F.EF(i), st.qpre[0] = F.EQ(i);
      if (ctx.schur_ok(b)) st.hpre[0] = F.EH(i);
      st.yb[0][0] = XB->D(i + 1);
      if (!diag_only) st.zrow[0] = XB->U(i), st.zcol[0] = XB->L(i);
      st.zdiag = XB->D(i);
    }
    sweep.step(st);
  }
  sweep.end();
}

// rgf.py:401-489: generic _backstep (steps.cu BackSweep) with k = 1 at the
// last block (tip coupling only) and k = 2 elsewhere (next block, tip).
void bta_backward_arrow(Context& ctx, const FactorsDev& F, const BtaDev& A, const BtaDev* B,
                        const BtaDev& XA, const BtaDev* XB, bool diag_only) {
  const int n = (int)A.n, b = (int)A.b, a = (int)A.a;
  cudaStream_t s = ctx.stream();
  const bool fused = B != nullptr;
  const int mx = std::max(a, b);
  ctx.reserve_slots(back_sweep_slots(), (int64_t)mx * mx);
  Mat Xtt = cm(F.tip_inv, a, a);
  Mat Ztt, sc_last;
  Level L(s);
  copy_block(L, XA.T(), Xtt);
  if (fused) {
    Mat w = ctx.tmp(0, a, a), sct = ctx.tmp(1, b, b);
    sc_last = ctx.tmp(2, b, b);
    L.out(w).mm(+1, Xtt, N, cm(F.b_tip, a, a), N);
    L.out(sct).mm(+1, F.SA(n - 1), N, cm(F.b_diag_last, b, b), N);
    L.flush();
    L.out(XB->T()).mm(+1, w, N, Xtt, H);
    L.out(sc_last).mm(+1, sct, N, F.SA(n - 1), H);
    Ztt = XB->T();
  }
  L.flush();
  BackSweep sweep(ctx);
  sweep.begin();
  for (int i = n - 1; i >= 0; --i) {
    BackStep st;
    st.g = F.SA(i);
    if (i == n - 1) {
      st.k = 1;
      st.rs[0] = F.ACe(i), st.qs[0] = F.ARe(i), st.ya[0][0] = Xtt;
      st.row[0] = XA.AC(i), st.col[0] = XA.AR(i);
      if (fused) {
        st.sc = sc_last;
        st.ss[0] = F.BCe(i), st.ws[0] = F.BRe(i), st.yb[0][0] = Ztt;
        st.zrow[0] = XB->AC(i), st.zcol[0] = XB->AR(i);
      }
    } else {
      st.k = 2;
      st.rs[0] = A.U(i), st.rs[1] = F.ACe(i);
      st.qs[0] = A.L(i), st.qs[1] = F.ARe(i);
      st.ya[0][0] = XA.D(i + 1), st.ya[0][1] = XA.AC(i + 1), st.ya[1][0] = XA.AR(i + 1), st.ya[1][1] = Xtt;
      if (!diag_only) st.row[0] = XA.U(i), st.col[0] = XA.L(i);
      st.row[1] = XA.AC(i), st.col[1] = XA.AR(i);
      {  // retained by the forward (see bta_forward_arrow)
        const bool extra = !fused || fwd_backward_products();
        if (extra || ctx.schur_ok(b)) st.hpre[0] = F.EH(i);
        if (extra) st.hpre[1] = F.EHA(i);
      }
      if (fused) {
        st.sc = F.SB(i);
        st.cpre[0] = F.EF(i), st.cpre[1] = F.EG(i), st.qpre[0] = F.EQ(i), st.qpre[1] = F.EK(i);
        if (fwd_backward_products()) st.epre[0] = F.EEQ(i), st.epre[1] = F.EEK(i);
        st.ss[0] = B->U(i), st.ss[1] = F.BCe(i);
        st.ws[0] = B->L(i), st.ws[1] = F.BRe(i);
        st.yb[0][0] = XB->D(i + 1), st.yb[0][1] = XB->AC(i + 1), st.yb[1][0] = XB->AR(i + 1);
        st.yb[1][1] = Ztt;
        if (!diag_only) st.zrow[0] = XB->U(i), st.zcol[0] = XB->L(i);
        st.zrow[1] = XB->AC(i), st.zcol[1] = XB->AR(i);
      }
    }
    st.diag = XA.D(i);
    if (fused) st.zdiag = XB->D(i);
    sweep.step(st);
  }
  sweep.end();
}

}  // namespace

void bta_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const FactorsDev& F) {
  if (A.n < 1 || A.b < 1 || A.a < 0) throw ShapeError("invalid shape parameters");
  if (B && (B->n != A.n || B->b != A.b || B->a != A.a))
    throw ShapeError("right-hand side shape differs from system shape");
  cudaStream_t s = ctx.stream();
  ctx.reset_status();
  cuda_check(cudaEventRecord(ctx.timer(0), s), "timer");
  streams_fork(ctx);
  if (A.a == 0)
    bt_forward(ctx, A, B, F);
  else
    bta_forward_arrow(ctx, A, B, F);
  streams_join(ctx);
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
