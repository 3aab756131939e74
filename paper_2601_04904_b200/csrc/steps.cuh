// Generic elimination / back-substitution steps shared by the sequential BTA
// sweep (rgf.py:237-288, 322-398) and the partition kernels of the
// distributed scheme (dist.py:211-397, 595-742).
#pragma once
#include "solver.cuh"

namespace bsel {

// One downward/upward elimination step of block i into its neighbour j
// (rgf.py:246-288; dist.py:216-257 first, 265-306 last).
//   Lk = A(j,i), Uk = A(i,j), BL = B(j,i), BU = B(i,j).
// Updates ad_j, ar_j, ac_j, tipA (and the B-side counterparts); writes S
// (and sb).  The A-side chain runs on ctx.stream(), the B side on ctx.aux().
struct EndStep {
  Mat Lk, Uk, BL, BU;
  Mat ad_i, ad_j, ar_i, ar_j, ac_i, ac_j, tipA;
  Mat bd_i, bd_j, br_i, br_j, bc_i, bc_j, tipB;
  Mat S, sb;
  // optional: retain f = Lk S, g = AR_i S, q = Bd_i f^H - BU, k = Bd_i g^H - BC_i
  // here (the backward step of block i reuses them) instead of ring slots
  Mat f_out, g_out, q_out, k_out;
  Mat h_out;  // optional: h = S Uk (the backward's h_0), free with the fused Schur step
  // optional, formed on the aux stream for the backward step of this block
  // (which then has no prologue): ha = S AC_i, eq = -S q, ek = -S k
  Mat ha_out, eq_out, ek_out;
};
// Forward ring: temporaries of step k live in ring slot fwd_slot(k); the
// B side (aux stream) may lag the A chain by up to kFwdDepth - 1 steps.
#ifndef BSEL_FWD_DEPTH
#define BSEL_FWD_DEPTH 4
#endif
constexpr int kFwdDepth = BSEL_FWD_DEPTH;
inline int fwd_slot(int64_t step) { return (int)(step % kFwdDepth); }
cudaEvent_t ring_a_event(Context& ctx, int slot);  // A side of the slot's step reached its B fork
cudaEvent_t ring_b_event(Context& ctx, int slot);  // B side of the slot's step done
void end_step(Context& ctx, const EndStep& st, bool fused, uint64_t order, int64_t index, int slot);

// One interior step of a middle partition with fill-in to its top boundary
// lo (dist.py:315-396).  fill_* are the couplings before the step, nfill_*
// receive the updated ones.
struct MiddleStep {
  Mat L, U, BL, BU;              // A(i+1,i), A(i,i+1), B(i+1,i), B(i,i+1)
  Mat ad_i, ad_n, ad_lo, ar_i, ar_n, ar_lo, ac_i, ac_n, ac_lo, tipA;
  Mat bd_i, bd_n, bd_lo, br_i, br_n, br_lo, bc_i, bc_n, bc_lo, tipB;
  Mat fill_r, fill_c, bfill_r, bfill_c;
  Mat nfill_r, nfill_c, nbfill_r, nbfill_c;
  Mat S, sb;
  // optional retained products (see EndStep): fn = L S, fr = fill_r S,
  // g = AR_i S, qn = Bd fn^H - BU, qr = Bd fr^H - bfill_c, kk = Bd g^H - BC_i
  Mat fn_out, fr_out, g_out, qn_out, qr_out, kk_out;
  Mat h_out;  // optional: h = S U
  Mat ha_out, eq_out, ek_out;  // optional: S AC_i, -S qn, -S kk (see EndStep)
};
void middle_step(Context& ctx, const MiddleStep& st, bool fused, uint64_t order, int64_t index, int slot);

// BSEL_FWD_BWD_PRODUCTS=1: the fused forward also forms the backward step's
// h and e products (EndStep/MiddleStep ha_out, eq_out, ek_out, h_out) on its
// aux stream.  Off by default: the chain-bound forward absorbs them only at
// the cost of more contention on its chain (config 4: 1 GPU 1057 vs 1055 ms,
// 2 GPUs 626 vs 684 ms).
bool fwd_backward_products();

// Wait for the B side of the step that last used ring slot `parity` (call
// before reusing it) and join both streams at the end of a sweep.
void ring_wait(Context& ctx, int step);
void streams_fork(Context& ctx);
void streams_join(Context& ctx);

// Generic Takahashi back-substitution step with k <= 3 trailing couplings
// (rgf.py:322-398).  sc.p == nullptr -> selected inversion only.
// Outputs left empty (p == nullptr) are allocated by BackSweep in its ring
// (diagonal_only drops, carried middle-partition couplings); step() fills
// them in so the caller can read the block back.
struct BackStep {
  int k = 0;
  Mat g, sc;
  Mat rs[3], qs[3], ss[3], ws[3];
  Mat ya[3][3], yb[3][3];
  // optional products retained by the forward step of this block:
  // cpre[l] = qs_l g, qpre[l] = Bd (qs_l g)^H - ss_l  (then e_l = -g qpre[l])
  Mat cpre[3], qpre[3];
  Mat hpre[3];  // optional: h_l = g rs_l (retained by the forward)
  Mat epre[3];  // optional: e_l (retained by the forward)
  // outputs
  Mat row[3], col[3], diag;
  Mat zrow[3], zcol[3], zdiag;
};

// Backward sweep engine.  The reference's _backstep is re-associated so that
// every product involving the trailing solution is ONE level deep:
//   h_l = g rs_l,  c_l = qs_l g,  e_l = g ss_l - sc qs_l^H,  f_l = ws_l g^H - qs_l sc
//   row_j = -sum_l h_l ya[l][j]             col_j = -sum_l ya[j][l] c_l
//   diag  = g - sum_l row_l c_l
//   zrow_j = sum_l e_l ya[j][l]^H - sum_l h_l yb[l][j]
//   zcol_j = sum_l ya[j][l] f_l - sum_l yb[j][l] h_l^H
//   zdiag = sc + sum_l (row_l f_l - zrow_l h_l^H)
// (algebraically identical to rgf.py:342-397: phi g = -sum row_l c_l, and
// g quad g^H + g acc1 + sc phi^H fold into -sum zrow_l h_l^H).
// When B = s B^H exactly (s = +-1, Context::b_symmetry()), X_B = s X_B^H and
// f_l = s e_l^H: the prologue skips f, zcol_j = s zrow_j^H is a transposed
// copy and zdiag uses s row_l e_l^H (a quarter fewer products per step).
// Three streams: the per-step prologue (h, c, e, f: forward factors only)
// runs ahead on the side stream, the X_A chain (2 levels per step) on the
// high-priority chain stream, the X_B chain (2 levels per step, lagging) on
// the aux stream; a ring of kBackDepth steps bounds the lag.
#ifndef BSEL_BACK_DEPTH
#define BSEL_BACK_DEPTH 4
#endif
constexpr int kBackDepth = BSEL_BACK_DEPTH;
// Slots of the context pool a backward sweep uses (reserve before begin()).
int back_sweep_slots();
class BackSweep {
 public:
  explicit BackSweep(Context& ctx, int tile_cfg = kTileAuto);
  // Fork the three streams from ctx.stream() (everything queued there so far
  // precedes the sweep).
  void begin();
  void step(BackStep& st);
  // Make ctx.stream() wait for every step issued so far (outputs complete).
  void fence();
  void end() { fence(); }

 private:
  Context& ctx_;
  int cfg_;
  int sym_;  // b_symmetry() at construction: +1 / -1 / 0
  int64_t t_ = 0;
  Mat ring(int64_t t, int k, int r, int c);
};

}  // namespace bsel
