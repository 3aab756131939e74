// Generic elimination / back-substitution steps (see steps.cuh).
//
// Stream discipline of the fused forward steps: the A-side Schur chain
// (pivot inverse, elimination factors, A updates) is issued on the
// high-priority chain stream, the quadratic B-side updates on the aux
// stream.  Temporaries of step k live in ring slot k % kFwdDepth; before the
// A side rewrites a slot it waits for the B side of step k - kFwdDepth
// (ring_wait), so the B side may lag the A chain by kFwdDepth - 1 steps: the
// latency-bound chain runs ahead and the B-side GEMM levels fill the SMs it
// leaves idle.
#include "steps.cuh"

namespace bsel {

namespace {
constexpr int kRing = 8;        // temporaries per forward ring slot
constexpr int kBackBase = 16;   // first slot used by back_step (2 x kBackSlots)
// The forward ring (kFwdDepth x kRing slots) overlaps the backward slots:
// forward and backward never run concurrently on one context.
static_assert(kFwdDepth * kRing <= 64, "forward ring exceeds the slot pool");
Mat rt(Context& ctx, int slot, int k, int r, int c) { return ctx.tmp(slot * kRing + k, r, c); }
}  // namespace

cudaEvent_t ring_a_event(Context& ctx, int slot) { return ctx.event(8 + slot); }
cudaEvent_t ring_b_event(Context& ctx, int slot) { return ctx.event(8 + kFwdDepth + slot); }

void streams_fork(Context& ctx) {
  cuda_check(cudaEventRecord(ctx.event(4), ctx.stream()), "fork");
  cuda_check(cudaStreamWaitEvent(ctx.aux(), ctx.event(4), 0), "fork wait");
  cuda_check(cudaStreamWaitEvent(ctx.chain(), ctx.event(4), 0), "fork wait");
}

void streams_join(Context& ctx) {
  cuda_check(cudaEventRecord(ctx.event(5), ctx.aux()), "join");
  cuda_check(cudaStreamWaitEvent(ctx.stream(), ctx.event(5), 0), "join wait");
  cuda_check(cudaEventRecord(ctx.event(6), ctx.chain()), "join");
  cuda_check(cudaStreamWaitEvent(ctx.stream(), ctx.event(6), 0), "join wait");
}

void ring_wait(Context& ctx, int step) {
  if (step >= kFwdDepth)
    cuda_check(cudaStreamWaitEvent(ctx.chain(), ring_b_event(ctx, fwd_slot(step)), 0), "ring wait");
}

// Critical chain of a step: pivot inverse -> f = Lk S -> ad_j -= f Uk (the
// next inverse needs nothing else).  Every other update -- arrow strips, tip,
// the whole B side -- runs on the aux stream, which may lag the chain by
// kFwdDepth - 1 steps.  Each output keeps the reference's expression and
// term order, so results do not depend on the stream split.
void end_step(Context& ctx, const EndStep& st, bool fused, uint64_t order, int64_t index, int slot) {
  cudaStream_t sA = ctx.chain(), sB = ctx.aux();
  const int b = st.ad_i.r, a = st.ar_i.r;
  ctx.invert(st.ad_i, st.S, order, index, sA);
  const Mat& S = st.S;
  if (!fused) {
    // rgf.py:283-288 / dist.py:252-257: right-hand temporaries.
    Mat t1 = rt(ctx, slot, 0, b, b), t2 = rt(ctx, slot, 1, b, a);
    Level L(sA);
    L.out(t1).mm(+1, S, N, st.Uk, N);
    L.flush();
    cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    L.out(st.ad_j).add(+1, st.ad_j).mm(-1, st.Lk, N, t1, N);
    L.flush();
    cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
    Level LB(sB);
    LB.out(t2).mm(+1, S, N, st.ac_i, N);
    LB.out(st.ar_j).add(+1, st.ar_j).mm(-1, st.ar_i, N, t1, N);
    LB.flush();
    LB.out(st.ac_j).add(+1, st.ac_j).mm(-1, st.Lk, N, t2, N);
    LB.out(st.tipA).add(+1, st.tipA).mm(-1, st.ar_i, N, t2, N);
    LB.flush();
    cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
    return;
  }
  Mat f = rt(ctx, slot, 0, b, b), g = rt(ctx, slot, 1, a, b), w = rt(ctx, slot, 2, b, b);
  Mat p = rt(ctx, slot, 3, a, b), k = rt(ctx, slot, 4, b, a), q = rt(ctx, slot, 5, b, b);
  {
    Level L(sA);
    L.out(f).mm(+1, st.Lk, N, S, N);
    L.flush();
    cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    L.out(st.ad_j).add(+1, st.ad_j).mm(-1, f, N, st.Uk, N);
    L.flush();
  }
  // Aux: A-side arrow/tip updates and the B side in three levels.  v Lk^H =
  // Lk S_B Lk^H = f (Bd f^H) = f q removes the reference's serial chain
  // w -> S_B -> v -> Bd (same product count).
  cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
  Level L(sB);
  L.out(g).mm(+1, st.ar_i, N, S, N);
  L.out(w).mm(+1, S, N, st.bd_i, N);
  L.out(q).mm(+1, st.bd_i, N, f, H);
  L.out(st.ac_j).add(+1, st.ac_j).mm(-1, f, N, st.ac_i, N);
  L.flush();
  L.out(st.ar_j).add(+1, st.ar_j).mm(-1, g, N, st.Uk, N);
  L.out(st.tipA).add(+1, st.tipA).mm(-1, g, N, st.ac_i, N);
  L.out(p).mm(+1, g, N, st.bd_i, N);
  L.out(k).mm(+1, st.bd_i, N, g, H);
  L.out(st.sb).mm(+1, w, N, S, H);
  L.out(st.bd_j).add(+1, st.bd_j).mm(+1, f, N, q, N).mm(-1, st.BL, N, f, H).mm(-1, f, N, st.BU, N);
  L.flush();
  L.out(st.br_j).add(+1, st.br_j).mm(-1, g, N, st.BU, N).mm(+1, p, N, f, H).mm(-1, st.br_i, N, f, H);
  L.out(st.bc_j).add(+1, st.bc_j).mm(-1, f, N, st.bc_i, N).mm(-1, st.BL, N, g, H).mm(+1, f, N, k, N);
  L.out(st.tipB).add(+1, st.tipB).mm(-1, g, N, st.bc_i, N).mm(-1, st.br_i, N, g, H).mm(+1, p, N, g, H);
  L.flush();
  cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
}

// Middle step: the chain is inverse -> fn = L S -> ad_n -= fn U; fill-in,
// lo-boundary, arrow, tip and B-side updates run on the aux stream.
void middle_step(Context& ctx, const MiddleStep& st, bool fused, uint64_t order, int64_t index, int slot) {
  cudaStream_t sA = ctx.chain(), sB = ctx.aux();
  const int b = st.ad_i.r, a = st.ar_i.r;
  ctx.invert(st.ad_i, st.S, order, index, sA);
  const Mat& S = st.S;
  Mat fn = rt(ctx, slot, 0, b, b), fr = rt(ctx, slot, 1, b, b), g = rt(ctx, slot, 2, a, b);
  {
    Level L(sA);
    L.out(fn).mm(+1, st.L, N, S, N);
    L.flush();
    cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    L.out(st.ad_n).add(+1, st.ad_n).mm(-1, fn, N, st.U, N);
    L.flush();
  }
  cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
  Level L(sB);
  L.out(fr).mm(+1, st.fill_r, N, S, N);
  L.out(g).mm(+1, st.ar_i, N, S, N);
  L.out(st.nfill_c).mm(-1, fn, N, st.fill_c, N);
  L.out(st.ac_n).add(+1, st.ac_n).mm(-1, fn, N, st.ac_i, N);
  Mat w, qn, qr, p, kk;
  if (fused) {
    // v_n = L S_B, v_0 = fill_r S_B enter only as v_x y^H = f_x (Bd f_y^H):
    // two levels instead of the reference's w -> S_B -> v -> update chain.
    w = rt(ctx, slot, 3, b, b), qn = rt(ctx, slot, 4, b, b), qr = rt(ctx, slot, 5, b, b);
    p = rt(ctx, slot, 6, a, b), kk = rt(ctx, slot, 7, b, a);
    L.out(w).mm(+1, S, N, st.bd_i, N);
    L.out(qn).mm(+1, st.bd_i, N, fn, H);
  }
  L.flush();
  L.out(st.nfill_r).mm(-1, fr, N, st.U, N);
  L.out(st.ad_lo).add(+1, st.ad_lo).mm(-1, fr, N, st.fill_c, N);
  L.out(st.ar_n).add(+1, st.ar_n).mm(-1, g, N, st.U, N);
  L.out(st.ar_lo).add(+1, st.ar_lo).mm(-1, g, N, st.fill_c, N);
  L.out(st.ac_lo).add(+1, st.ac_lo).mm(-1, fr, N, st.ac_i, N);
  L.out(st.tipA).add(+1, st.tipA).mm(-1, g, N, st.ac_i, N);
  if (!fused) {
    L.flush();
    cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
    return;
  }
  L.out(p).mm(+1, g, N, st.bd_i, N);
  L.out(qr).mm(+1, st.bd_i, N, fr, H);
  L.out(kk).mm(+1, st.bd_i, N, g, H);
  L.out(st.sb).mm(+1, w, N, S, H);
  L.out(st.bd_n).add(+1, st.bd_n).mm(-1, fn, N, st.BU, N).mm(-1, st.BL, N, fn, H).mm(+1, fn, N, qn, N);
  L.flush();
  L.out(st.br_n).add(+1, st.br_n).mm(-1, g, N, st.BU, N).mm(-1, st.br_i, N, fn, H).mm(+1, p, N, fn, H);
  L.out(st.br_lo).add(+1, st.br_lo).mm(-1, g, N, st.bfill_c, N).mm(-1, st.br_i, N, fr, H).mm(+1, p, N, fr, H);
  L.out(st.tipB).add(+1, st.tipB).mm(-1, g, N, st.bc_i, N).mm(-1, st.br_i, N, g, H).mm(+1, p, N, g, H);
  L.out(st.nbfill_c).mm(-1, fn, N, st.bfill_c, N).mm(-1, st.BL, N, fr, H).mm(+1, fn, N, qr, N);
  L.out(st.nbfill_r).mm(-1, fr, N, st.BU, N).mm(-1, st.bfill_r, N, fn, H).mm(+1, fr, N, qn, N);
  L.out(st.bd_lo).add(+1, st.bd_lo).mm(-1, fr, N, st.bfill_c, N).mm(-1, st.bfill_r, N, fr, H).mm(+1, fr, N, qr, N);
  L.out(st.bc_n).add(+1, st.bc_n).mm(-1, fn, N, st.bc_i, N).mm(-1, st.BL, N, g, H).mm(+1, fn, N, kk, N);
  L.out(st.bc_lo).add(+1, st.bc_lo).mm(-1, fr, N, st.bc_i, N).mm(-1, st.bfill_r, N, g, H).mm(+1, fr, N, kk, N);
  L.flush();
  cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
}

namespace {
constexpr int kBackSlots = 24;  // per parity half
bool any_late_col(const BackStep& st, int j) {  // ya[l][j] for some l
  for (int l = 0; l < st.k; ++l)
    if (st.late[l][j]) return true;
  return false;
}
bool any_late_row(const BackStep& st, int j) {  // ya[j][l] for some l
  for (int l = 0; l < st.k; ++l)
    if (st.late[j][l]) return true;
  return false;
}
}  // namespace

// L1 of one step: the problems that only read inputs and trailing blocks.
// `late_pass` selects which half is emitted.
static void back_l1(Context& ctx, Level& L, const BackStep& st, int parity, bool late_pass, Mat* RA, Mat* CA,
                    Mat* RZ, Mat* CZ, Mat* e, Mat* f) {
  const int k = st.k, b = st.g.r;
  const bool fused = st.sc.p != nullptr;
  const int base = kBackBase + parity * kBackSlots;
  for (int j = 0; j < k; ++j) {
    const int dj = st.rs[j].c;
    RA[j] = ctx.tmp(base + 6 * j + 0, b, dj);
    CA[j] = ctx.tmp(base + 6 * j + 1, dj, b);
    if (any_late_col(st, j) == late_pass) {
      L.out(RA[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, st.rs[l], N, st.ya[l][j], N);
    }
    if (any_late_row(st, j) == late_pass) {
      L.out(CA[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, st.ya[j][l], N, st.qs[l], N);
    }
    if (!fused) continue;
    RZ[j] = ctx.tmp(base + 6 * j + 2, b, dj);
    CZ[j] = ctx.tmp(base + 6 * j + 3, dj, b);
    e[j] = ctx.tmp(base + 6 * j + 4, b, dj);
    f[j] = ctx.tmp(base + 6 * j + 5, dj, b);
    if (any_late_col(st, j) == late_pass) {
      L.out(RZ[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, st.rs[l], N, st.yb[l][j], N);
    }
    if (any_late_row(st, j) == late_pass) {
      L.out(CZ[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, st.yb[j][l], N, st.rs[l], H);
    }
    if (!late_pass) {
      L.out(e[j]).mm(+1, st.g, N, st.ss[j], N).mm(-1, st.sc, N, st.qs[j], H);
      L.out(f[j]).mm(+1, st.ws[j], N, st.g, H).mm(-1, st.qs[j], N, st.sc, N);
    }
  }
}

void BackPipe::early(Level& L, const BackStep& st, int parity) {
  back_l1(ctx_, L, st, parity, false, RA, CA, RZ, CZ, e, f);
}

void BackPipe::rest(Level& L, const BackStep& st, int parity) {
  const int k = st.k, b = st.g.r;
  const bool fused = st.sc.p != nullptr;
  back_l1(ctx_, L, st, parity, true, RA, CA, RZ, CZ, e, f);
  L.flush();
  // L2: row/column blocks of X_A and X_B, and the quadratic coupling.
  const int base = kBackBase + parity * kBackSlots + 18;
  Mat quad = ctx_.tmp(base + 0, b, b);
  for (int j = 0; j < k; ++j) {
    L.out(st.row[j]).mm(-1, st.g, N, RA[j], N);
    L.out(st.col[j]).mm(-1, CA[j], N, st.g, N);
    if (fused) {
      L.out(st.zrow[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, e[l], N, st.ya[j][l], H);
      L.mm(-1, st.g, N, RZ[j], N);
      L.out(st.zcol[j]);
      for (int l = 0; l < k; ++l) L.mm(+1, st.ya[j][l], N, f[l], N);
      L.mm(-1, CZ[j], N, st.g, H);
    }
  }
  if (fused) {
    L.out(quad);
    for (int l = 0; l < k; ++l) L.mm(+1, st.rs[l], N, CZ[l], N);
  }
  L.flush();
  // L3
  Mat phi = ctx_.tmp(base + 1, b, b), acc1 = ctx_.tmp(base + 2, b, b), acc2 = ctx_.tmp(base + 3, b, b);
  Mat gq = ctx_.tmp(base + 4, b, b);
  L.out(phi);
  for (int l = 0; l < k; ++l) L.mm(-1, st.row[l], N, st.qs[l], N);
  if (fused) {
    L.out(acc1);
    for (int l = 0; l < k; ++l) L.mm(+1, st.ss[l], N, st.row[l], H);
    L.out(acc2);
    for (int l = 0; l < k; ++l) L.mm(+1, st.row[l], N, st.ws[l], N);
    L.out(gq).mm(+1, st.g, N, quad, N);
  }
  L.flush();
  // L4 (left pending: the caller adds the next step's early L1 before flushing)
  L.out(st.diag).add(+1, st.g).mm(+1, phi, N, st.g, N);
  if (fused) {
    L.out(st.zdiag)
        .add(+1, st.sc)
        .mm(+1, phi, N, st.sc, N)
        .mm(+1, st.sc, N, phi, H)
        .mm(+1, st.g, N, acc1, N)
        .mm(+1, acc2, N, st.g, H)
        .mm(+1, gq, N, st.g, H);
  }
}

void back_step(Context& ctx, cudaStream_t s, const BackStep& st) {
  BackPipe pipe(ctx);
  Level L(s);
  pipe.early(L, st, 0);
  pipe.rest(L, st, 0);
  L.flush();
}

}  // namespace bsel
