// Generic elimination / back-substitution steps (see steps.cuh).
//
// Stream discipline of the fused forward steps: the A-side Schur chain
// (pivot inverse, elimination factors, A updates) is issued on the
// high-priority chain stream, the quadratic B-side updates on the aux
// stream.  Temporaries of step k live in ring slot k % kFwdDepth; before the
// A side rewrites a slot it waits for the B side of step k - kFwdDepth
// (ring_wait), so the B side may lag the A chain by kFwdDepth - 1 steps: the
// latency-bound chain runs ahead and the B-side GEMM levels fill the SMs it
// leaves idle.  The wait is enqueued AFTER the step's inverse (which touches
// no ring slot), so the inverse directly follows the previous step's last
// chain GEMM in the stream and is launched as its programmatic dependent
// (inverse.cu launch_dataflow: its CTAs are placed while that GEMM runs).
#include <cstdlib>

#include "steps.cuh"
#include "inverse.cuh"

namespace bsel {

namespace {
constexpr int kRing = 8;        // temporaries per forward ring slot
constexpr int kBackBase = 16;   // first slot used by back_step (2 x kBackSlots)
// The forward ring (kFwdDepth x kRing slots) overlaps the backward slots:
// forward and backward never run concurrently on one context.
static_assert(kFwdDepth * kRing <= 64, "forward ring exceeds the slot pool");
static_assert(8 + 2 * kFwdDepth <= 64, "forward ring events");
Mat rt(Context& ctx, int slot, int k, int r, int c) { return ctx.tmp(slot * kRing + k, r, c); }
// CTA cap of the forward's aux-stream levels (BSEL_AUX_CTAS, 0 = none): a
// capped level loops its tiles over fewer CTAs and leaves SMs to the chain.
int aux_ctas() {
  static const int cap = [] {
    const char* e = getenv("BSEL_AUX_CTAS");
    return e ? atoi(e) : 0;
  }();
  return cap;
}
// Tile configuration of the chain's two products (BSEL_CHAIN_TILE: auto
// (default), 6432 = 64x32 / BK 32, 64, 32) -- experiment knob.
int chain_tile() {
  static const int cfg = [] {
    const char* e = getenv("BSEL_CHAIN_TILE");
    const int v = e ? atoi(e) : 0;
    return v == 6432 ? (int)kTile3m6432k32 : v == 64 ? (int)kTile3m64 : v == 32 ? (int)kTile3m32 : (int)kTileAuto;
  }();
  return cfg;
}

// BSEL_AUX_AFTER_CHAIN=1: a step's aux levels start after BOTH chain
// products (not after f): the chain's second product then runs without the
// step's own aux level competing for the SMs (experiment).
bool aux_after_chain() {
  static const bool on = [] {
    const char* e = getenv("BSEL_AUX_AFTER_CHAIN");
    return e && atoi(e) != 0;
  }();
  return on;
}
}  // namespace

bool fwd_backward_products() {
  static const bool on = [] {
    const char* e = getenv("BSEL_FWD_BWD_PRODUCTS");
    return e && atoi(e) != 0;
  }();
  return on;
}

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
  const bool schur = ctx.schur_ok(b);
  const Mat& S = st.S;
  if (!fused) {
    // rgf.py:283-288 / dist.py:252-257: right-hand temporaries.
    Mat t1 = st.h_out.p ? st.h_out : rt(ctx, slot, 0, b, b), t2 = st.ha_out.p ? st.ha_out : rt(ctx, slot, 1, b, a);
    if (schur) {  // S, t1 = S Uk and ad_j -= Lk t1 in one launch
      ring_wait(ctx, (int)order);
      ctx.schur(st.ad_i, st.Uk, st.Lk, st.ad_j, S, t1, st.f_out.p ? st.f_out : rt(ctx, slot, 2, b, b), order, index,
                sA);
      cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    } else {
      ctx.invert(st.ad_i, st.S, order, index, sA);
      ring_wait(ctx, (int)order);  // after the inverse: it touches no ring slot (PDL launch)
      Level L(sA);
      L.out(t1).mm(+1, S, N, st.Uk, N);
      L.flush();
      cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
      L.out(st.ad_j).add(+1, st.ad_j).mm(-1, st.Lk, N, t1, N);
      L.flush();
    }
    cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
    Level LB(sB, kTileAutoFwd, aux_ctas());
    LB.avoid_sms(ctx.aux_avoid_sms(), ctx.aux_counter());
    LB.out(t2).mm(+1, S, N, st.ac_i, N);
    LB.out(st.ar_j).add(+1, st.ar_j).mm(-1, st.ar_i, N, t1, N);
    LB.flush();
    LB.out(st.ac_j).add(+1, st.ac_j).mm(-1, st.Lk, N, t2, N);
    LB.out(st.tipA).add(+1, st.tipA).mm(-1, st.ar_i, N, t2, N);
    LB.flush();
    cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
    return;
  }
  auto keep = [&](const Mat& m, int k_, int r, int c) { return m.p ? m : rt(ctx, slot, k_, r, c); };
  Mat f = keep(st.f_out, 0, b, b), g = keep(st.g_out, 1, a, b), w = rt(ctx, slot, 2, b, b);
  Mat k = keep(st.k_out, 4, b, a), q = keep(st.q_out, 5, b, b);
  if (schur) {  // S, f = Lk S and ad_j -= f Uk (and h = S Uk) in one launch
    ring_wait(ctx, (int)order);
    ctx.schur(st.ad_i, st.Uk, st.Lk, st.ad_j, S, st.h_out, f, order, index, sA);
    cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
  } else {
    ctx.invert(st.ad_i, st.S, order, index, sA);
    ring_wait(ctx, (int)order);  // after the inverse: it touches no ring slot (PDL launch)
    Level L(sA, chain_tile());
    L.chain_mark(chain_marks());
    L.out(f).mm(+1, st.Lk, N, S, N);
    L.flush();
    if (!aux_after_chain()) cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    L.out(st.ad_j).add(+1, st.ad_j).mm(-1, f, N, st.Uk, N);
    L.flush();
    if (aux_after_chain()) cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
  }
  // Aux: A-side arrow/tip updates and the B side in three levels.  The
  // reference's quadratic updates (rgf.py:257-280) are re-associated so each
  // output is two products: with q = Bd f^H - BU and k = Bd g^H - BC_i,
  //   v Lk^H - BL f^H - f BU        = f q - BL f^H        (v = Lk S_B)
  //   -g BU + p f^H - BR_i f^H      = g q - BR_i f^H      (p = g Bd)
  //   -f BC_i - BL g^H + f (Bd g^H) = f k - BL g^H
  //   -g BC_i - BR_i g^H + p g^H    = g k - BR_i g^H
  // which also removes the reference's serial chain w -> S_B -> v -> Bd.
  cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
  Level L(sB, kTileAutoFwd, aux_ctas());
  L.avoid_sms(ctx.aux_avoid_sms(), ctx.aux_counter());
  L.out(g).mm(+1, st.ar_i, N, S, N);
  L.out(w).mm(+1, S, N, st.bd_i, N);
  L.out(q).add(-1, st.BU).mm(+1, st.bd_i, N, f, H);
  L.out(st.ac_j).add(+1, st.ac_j).mm(-1, f, N, st.ac_i, N);
  // the backward step's h_l (g rs_l) formed here, where the chain-bound
  // forward leaves the SMs room, instead of in the throughput-bound backward
  if (st.h_out.p && !schur) L.out(st.h_out).mm(+1, S, N, st.Uk, N);
  if (st.ha_out.p) L.out(st.ha_out).mm(+1, S, N, st.ac_i, N);
  L.flush();
  L.out(st.ar_j).add(+1, st.ar_j).mm(-1, g, N, st.Uk, N);
  L.out(st.tipA).add(+1, st.tipA).mm(-1, g, N, st.ac_i, N);
  L.out(k).add(-1, st.bc_i).mm(+1, st.bd_i, N, g, H);
  // B = s B^H (this partition's data, checked before the sweep): S_B and the
  // updated B diagonal stay (anti-)Hermitian -> lower-triangle tiles + mirror,
  // and the arrow column is the (conjugate) transpose of the arrow row.
  const int sym = ctx.forward_symmetry();
  L.out(st.sb).mm(+1, w, N, S, H);
  if (sym) L.lower_only();
  L.out(st.bd_j).add(+1, st.bd_j).mm(+1, f, N, q, N).mm(-1, st.BL, N, f, H);
  if (sym) L.lower_only();
  L.out(st.br_j).add(+1, st.br_j).mm(+1, g, N, q, N).mm(-1, st.br_i, N, f, H);
  if (st.eq_out.p) L.out(st.eq_out).mm(-1, S, N, q, N);  // the backward's e_0 = -g q
  L.flush();
  if (sym) {
    cuda_check(launch_mirror_lower(st.sb.p, st.sb.ld, st.sb.r, sym, sB), "mirror");
    cuda_check(launch_mirror_lower(st.bd_j.p, st.bd_j.ld, st.bd_j.r, sym, sB), "mirror");
    TransJob tj;
    tj.src = st.br_j.p, tj.lds = st.br_j.ld, tj.r = st.br_j.r, tj.c = st.br_j.c;
    tj.dst = st.bc_j.p, tj.ldd = st.bc_j.ld;
    cuda_check(launch_conj_transpose(&tj, 1, sym, sB), "conjugate transpose");
  } else {
    L.out(st.bc_j).add(+1, st.bc_j).mm(+1, f, N, k, N).mm(-1, st.BL, N, g, H);
  }
  L.out(st.tipB).add(+1, st.tipB).mm(+1, g, N, k, N).mm(-1, st.br_i, N, g, H);
  if (st.ek_out.p) L.out(st.ek_out).mm(-1, S, N, k, N);  // the backward's e_1 = -g k
  L.flush();
  cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
}

// Middle step: the chain is inverse -> fn = L S -> ad_n -= fn U; fill-in,
// lo-boundary, arrow, tip and B-side updates run on the aux stream.
void middle_step(Context& ctx, const MiddleStep& st, bool fused, uint64_t order, int64_t index, int slot) {
  cudaStream_t sA = ctx.chain(), sB = ctx.aux();
  const int b = st.ad_i.r, a = st.ar_i.r;
  const Mat& S = st.S;
  auto keep = [&](const Mat& m, int k_, int r, int c) { return m.p ? m : rt(ctx, slot, k_, r, c); };
  Mat fn = keep(st.fn_out, 0, b, b), fr = keep(st.fr_out, 1, b, b), g = keep(st.g_out, 2, a, b);
  if (ctx.schur_ok(b)) {  // S, fn = L S and ad_n -= fn U (and h = S U) in one launch
    ring_wait(ctx, (int)order);
    ctx.schur(st.ad_i, st.U, st.L, st.ad_n, S, st.h_out, fn, order, index, sA);
    cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
  } else {
    ctx.invert(st.ad_i, st.S, order, index, sA);
    ring_wait(ctx, (int)order);  // after the inverse: it touches no ring slot (PDL launch)
    Level L(sA, chain_tile());
    L.chain_mark(chain_marks());
    L.out(fn).mm(+1, st.L, N, S, N);
    L.flush();
    if (!aux_after_chain()) cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
    L.out(st.ad_n).add(+1, st.ad_n).mm(-1, fn, N, st.U, N);
    L.flush();
    if (aux_after_chain()) cuda_check(cudaEventRecord(ring_a_event(ctx, slot), sA), "record A");
  }
  cuda_check(cudaStreamWaitEvent(sB, ring_a_event(ctx, slot), 0), "wait A");
  Level L(sB, kTileAutoFwd, aux_ctas());
  L.avoid_sms(ctx.aux_avoid_sms(), ctx.aux_counter());
  L.out(fr).mm(+1, st.fill_r, N, S, N);
  L.out(g).mm(+1, st.ar_i, N, S, N);
  L.out(st.nfill_c).mm(-1, fn, N, st.fill_c, N);
  L.out(st.ac_n).add(+1, st.ac_n).mm(-1, fn, N, st.ac_i, N);
  Mat w, qn, qr, kk;
  if (fused) {
    // Re-associated quadratic updates (see end_step): with
    //   qn = Bd fn^H - BU, qr = Bd fr^H - BFC, kk = Bd g^H - BC_i
    // every B-side output of dist.py:360-396 is two products.
    w = rt(ctx, slot, 3, b, b), qn = keep(st.qn_out, 4, b, b), qr = keep(st.qr_out, 5, b, b);
    kk = keep(st.kk_out, 7, b, a);
    L.out(w).mm(+1, S, N, st.bd_i, N);
    L.out(qn).add(-1, st.BU).mm(+1, st.bd_i, N, fn, H);
    // the backward step's h for the U and arrow couplings (see end_step)
    if (st.h_out.p && !ctx.schur_ok(b)) L.out(st.h_out).mm(+1, S, N, st.U, N);
    if (st.ha_out.p) L.out(st.ha_out).mm(+1, S, N, st.ac_i, N);
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
  L.out(qr).add(-1, st.bfill_c).mm(+1, st.bd_i, N, fr, H);
  L.out(kk).add(-1, st.bc_i).mm(+1, st.bd_i, N, g, H);
  // B = s B^H (see end_step): Hermitian blocks as lower-triangle tiles +
  // mirror, column-side blocks (bc_n, bc_lo, the new column fill) as
  // transposes of their row-side partners.
  const int sym = ctx.forward_symmetry();
  L.out(st.sb).mm(+1, w, N, S, H);
  if (sym) L.lower_only();
  L.out(st.bd_n).add(+1, st.bd_n).mm(+1, fn, N, qn, N).mm(-1, st.BL, N, fn, H);
  if (sym) L.lower_only();
  L.out(st.br_n).add(+1, st.br_n).mm(+1, g, N, qn, N).mm(-1, st.br_i, N, fn, H);
  L.out(st.nbfill_r).mm(+1, fr, N, qn, N).mm(-1, st.bfill_r, N, fn, H);
  if (st.eq_out.p) L.out(st.eq_out).mm(-1, S, N, qn, N);
  L.flush();
  if (st.ek_out.p) L.out(st.ek_out).mm(-1, S, N, kk, N);
  L.out(st.br_lo).add(+1, st.br_lo).mm(+1, g, N, qr, N).mm(-1, st.br_i, N, fr, H);
  L.out(st.tipB).add(+1, st.tipB).mm(+1, g, N, kk, N).mm(-1, st.br_i, N, g, H);
  L.out(st.bd_lo).add(+1, st.bd_lo).mm(+1, fr, N, qr, N).mm(-1, st.bfill_r, N, fr, H);
  if (sym) {
    L.lower_only();
  } else {
    L.out(st.nbfill_c).mm(+1, fn, N, qr, N).mm(-1, st.BL, N, fr, H);
    L.out(st.bc_n).add(+1, st.bc_n).mm(+1, fn, N, kk, N).mm(-1, st.BL, N, g, H);
    L.out(st.bc_lo).add(+1, st.bc_lo).mm(+1, fr, N, kk, N).mm(-1, st.bfill_r, N, g, H);
  }
  L.flush();
  if (sym) {
    for (const Mat* m : {&st.sb, &st.bd_n, &st.bd_lo})
      cuda_check(launch_mirror_lower(m->p, m->ld, m->r, sym, sB), "mirror");
    TransJob tj[3];
    const Mat* src[3] = {&st.br_n, &st.br_lo, &st.nbfill_r};
    const Mat* dst[3] = {&st.bc_n, &st.bc_lo, &st.nbfill_c};
    for (int q = 0; q < 3; ++q) {
      tj[q].src = src[q]->p, tj[q].lds = src[q]->ld, tj[q].r = src[q]->r, tj[q].c = src[q]->c;
      tj[q].dst = dst[q]->p, tj[q].ldd = dst[q]->ld;
    }
    cuda_check(launch_conj_transpose(tj, 3, sym, sB), "conjugate transpose");
  }
  cuda_check(cudaEventRecord(ring_b_event(ctx, slot), sB), "record B");
}

// ---------------------------------------------------------------------------
// Backward sweep engine (see steps.cuh for the re-associated step).
// Ring slot r = t % kBackDepth holds step t's prologue temporaries and the
// outputs the caller left empty; its events: pre done, X_A level 1 done,
// X_B done.  The prologue of step t (side stream) reuses the slot of step
// t - kBackDepth, whose blocks are last read by X_B(t - kBackDepth + 1)
// (carried couplings of a middle partition), so it waits for that step.
// ---------------------------------------------------------------------------
namespace {
constexpr int kBackRingBase = 16;  // slots 0..15 stay free for the callers' prologues
constexpr int kBackPerStep = 16;   // h, c, e, f (3 each) + 4 ring-allocated outputs
cudaEvent_t ev_pre(Context& ctx, int64_t t) { return ctx.event(Context::kBackEvents + (int)(t % kBackDepth)); }
cudaEvent_t ev_a1(Context& ctx, int64_t t) {
  return ctx.event(Context::kBackEvents + kBackDepth + (int)(t % kBackDepth));
}
cudaEvent_t ev_b(Context& ctx, int64_t t) {
  return ctx.event(Context::kBackEvents + 2 * kBackDepth + (int)(t % kBackDepth));
}
cudaEvent_t ev_fork(Context& ctx) { return ctx.event(Context::kBackEvents + 3 * kBackDepth); }
cudaEvent_t ev_join(Context& ctx, int i) { return ctx.event(Context::kBackEvents + 3 * kBackDepth + 1 + i); }
static_assert(Context::kBackEvents + 3 * kBackDepth + 3 <= 64, "event pool");
}  // namespace

int back_sweep_slots() { return kBackRingBase + kBackPerStep * kBackDepth; }

BackSweep::BackSweep(Context& ctx, int tile_cfg) : ctx_(ctx), cfg_(tile_cfg), sym_(ctx.b_symmetry()) {}

Mat BackSweep::ring(int64_t t, int k, int r, int c) {
  return ctx_.tmp(kBackRingBase + (int)(t % kBackDepth) * kBackPerStep + k, r, c);
}

void BackSweep::begin() {
  cuda_check(cudaEventRecord(ev_fork(ctx_), ctx_.stream()), "back fork");
  for (cudaStream_t s : {ctx_.side(), ctx_.chain(), ctx_.aux()})
    cuda_check(cudaStreamWaitEvent(s, ev_fork(ctx_), 0), "back fork wait");
}

void BackSweep::fence() {
  // X_B(t) follows X_A level 1 (t), the prologue precedes both; the chain's
  // last diagonal block is joined separately.
  cuda_check(cudaEventRecord(ev_join(ctx_, 0), ctx_.aux()), "back join");
  cuda_check(cudaEventRecord(ev_join(ctx_, 1), ctx_.chain()), "back join");
  cuda_check(cudaStreamWaitEvent(ctx_.stream(), ev_join(ctx_, 0), 0), "back join wait");
  cuda_check(cudaStreamWaitEvent(ctx_.stream(), ev_join(ctx_, 1), 0), "back join wait");
}

void BackSweep::step(BackStep& st) {
  const int64_t t = t_++;
  const int k = st.k, b = st.g.r;
  const bool fused = st.sc.p != nullptr;
  const int sym = fused ? sym_ : 0;
  if (k < 1 || k > 3) throw ShapeError("back step needs 1..3 couplings");
  // Ring-allocate the outputs the caller left empty.
  int spare = 12;
  auto own = [&](Mat& m, int r, int c) {
    if (m.p) return;
    if (spare == kBackPerStep) throw ShapeError("too many ring-allocated back-step outputs");
    m = ring(t, spare++, r, c);
  };
  for (int j = 0; j < k; ++j) {
    const int dj = st.rs[j].c;
    own(st.row[j], b, dj);
    own(st.col[j], dj, b);
    if (fused) {
      own(st.zrow[j], b, dj);
      own(st.zcol[j], dj, b);
    }
  }
  Mat h[3], c[3], e[3], f[3];
  for (int l = 0; l < k; ++l) {
    const int dl = st.rs[l].c;
    h[l] = ring(t, l, b, dl);
    c[l] = ring(t, 3 + l, dl, b);
    if (fused) e[l] = ring(t, 6 + l, b, dl), f[l] = sym ? Mat{} : ring(t, 9 + l, dl, b);
  }
  // Prologue (side stream): forward factors and couplings only.
  {
    cudaStream_t sp = ctx_.side();
    if (t >= kBackDepth - 1) cuda_check(cudaStreamWaitEvent(sp, ev_b(ctx_, t - kBackDepth + 1), 0), "ring wait");
    Level P(sp, cfg_);
    for (int l = 0; l < k; ++l) {
      if (st.hpre[l].p) h[l] = st.hpre[l];
      else P.out(h[l]).mm(+1, st.g, N, st.rs[l], N);
      if (st.cpre[l].p) c[l] = st.cpre[l];
      else P.out(c[l]).mm(+1, st.qs[l], N, st.g, N);
      if (fused) {
        // e_l = g ss_l - sc qs_l^H = -g (Bd c_l^H - ss_l)  (sc = g Bd g^H)
        if (st.epre[l].p) e[l] = st.epre[l];
        else if (st.qpre[l].p) P.out(e[l]).mm(-1, st.g, N, st.qpre[l], N);
        else P.out(e[l]).mm(+1, st.g, N, st.ss[l], N).mm(-1, st.sc, N, st.qs[l], H);
        if (!sym) P.out(f[l]).mm(+1, st.ws[l], N, st.g, H).mm(-1, st.qs[l], N, st.sc, N);
      }
    }
    P.flush();
    cuda_check(cudaEventRecord(ev_pre(ctx_, t), sp), "pre record");
  }
  // X_A chain (chain stream): row / col, then the diagonal block.
  {
    cudaStream_t sa = ctx_.chain();
    cuda_check(cudaStreamWaitEvent(sa, ev_pre(ctx_, t), 0), "pre wait");
    Level A(sa, cfg_);
    for (int j = 0; j < k; ++j) {
      A.out(st.row[j]);
      for (int l = 0; l < k; ++l) A.mm(-1, h[l], N, st.ya[l][j], N);
      A.out(st.col[j]);
      for (int l = 0; l < k; ++l) A.mm(-1, st.ya[j][l], N, c[l], N);
    }
    A.flush();
    cuda_check(cudaEventRecord(ev_a1(ctx_, t), sa), "a1 record");
    A.out(st.diag).add(+1, st.g);
    for (int l = 0; l < k; ++l) A.mm(-1, st.row[l], N, c[l], N);
    A.flush();
  }
  if (!fused) {
    cuda_check(cudaEventRecord(ev_b(ctx_, t), ctx_.chain()), "b record");
    return;
  }
  // X_B chain (aux stream), one step behind at most kBackDepth - 1.
  {
    cudaStream_t sb = ctx_.aux();
    cuda_check(cudaStreamWaitEvent(sb, ev_a1(ctx_, t), 0), "a1 wait");
    Level B(sb, cfg_);
    for (int j = 0; j < k; ++j) {
      B.out(st.zrow[j]);
      for (int l = 0; l < k; ++l) B.mm(+1, e[l], N, st.ya[j][l], H);
      for (int l = 0; l < k; ++l) B.mm(-1, h[l], N, st.yb[l][j], N);
      if (sym) continue;
      B.out(st.zcol[j]);
      for (int l = 0; l < k; ++l) B.mm(+1, st.ya[j][l], N, f[l], N);
      for (int l = 0; l < k; ++l) B.mm(-1, st.yb[j][l], N, h[l], H);
    }
    B.flush();
    B.out(st.zdiag).add(+1, st.sc);
    if (sym) B.lower_only();  // X_B(i,i) = s X_B(i,i)^H: lower tiles, then mirrored
    for (int l = 0; l < k; ++l) {
      if (sym) B.mm(sym, st.row[l], N, e[l], H);  // f_l = s e_l^H
      else B.mm(+1, st.row[l], N, f[l], N);
    }
    for (int l = 0; l < k; ++l) B.mm(-1, st.zrow[l], N, h[l], H);
    B.flush();
    if (sym) {
      cuda_check(launch_mirror_lower(st.zdiag.p, st.zdiag.ld, st.zdiag.r, sym, sb), "mirror");
      // zcol_j = X_B(trail_j, i) = s X_B(i, trail_j)^H
      TransJob tj[3];
      for (int j = 0; j < k; ++j) {
        tj[j].src = st.zrow[j].p, tj[j].lds = st.zrow[j].ld, tj[j].r = st.zrow[j].r, tj[j].c = st.zrow[j].c;
        tj[j].dst = st.zcol[j].p, tj[j].ldd = st.zcol[j].ld;
        if (st.zcol[j].r != st.zrow[j].c || st.zcol[j].c != st.zrow[j].r) throw ShapeError("zcol shape");
      }
      cuda_check(launch_conj_transpose(tj, k, sym, sb), "conjugate transpose");
    }
    cuda_check(cudaEventRecord(ev_b(ctx_, t), sb), "b record");
  }
}

}  // namespace bsel
