// Partition kernels of the distributed scheme (dist.py:172-416, 542-744):
// local elimination of one contiguous block range (first: downward into
// hi-1, last: upward into lo, middle: downward with fill-in to lo) and the
// seeded local back-substitution.  The collectives between the two phases
// live in the host layer (NCCL through torch.distributed).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "partition.cuh"
#include "steps.cuh"

namespace bsel {

namespace {

inline Mat cm(const double2* p, int r, int c) { return Mat{const_cast<double2*>(p), c, r, c}; }

void copy_blocks(Context& ctx, double2* dst, const double2* src, int64_t elems) {
  if (elems > 0)
    cuda_check(cudaMemcpyAsync(dst, src, (size_t)elems * sizeof(double2), cudaMemcpyDeviceToDevice,
                               ctx.stream()),
               "partition copy");
}

void copy_async(cudaStream_t s, double2* dst, const double2* src, int64_t elems) {
  if (elems > 0)
    cuda_check(cudaMemcpyAsync(dst, src, (size_t)elems * sizeof(double2), cudaMemcpyDefault, s), "host copy");
}

// Blocks [g0, g1) and couplings [e0, e1) of one transfer chunk.
struct ChunkRange {
  int64_t g0, g1, e0, e1;
};

// Forward chunk c: processing positions [c*C, (c+1)*C) and the couplings of
// the same blocks (all the sweep touches up to position (c+1)*C - 1).
ChunkRange in_chunk(PartKind kind, int64_t lo, int64_t hi, int64_t n, int64_t C, int64_t c) {
  const int64_t len = hi - lo, p0 = c * C, p1 = std::min((c + 1) * C, len);
  ChunkRange r;
  if (kind == kLast) r.g0 = hi - p1, r.g1 = hi - p0;
  else r.g0 = lo + p0, r.g1 = lo + p1;
  r.e0 = r.g0, r.e1 = std::min(r.g1, n - 1);
  return r;
}

// Backward chunk c of nc: the outputs final after backward steps
// [c*C, (c+1)*C).  Backward position q: block hi-1-q (first / middle,
// descending) or lo+q (last, ascending; its couplings lag one step).
ChunkRange out_chunk(PartKind kind, int64_t lo, int64_t hi, int64_t n, int64_t C, int64_t c, int64_t nc) {
  const int64_t len = hi - lo;
  const bool last = c == nc - 1;
  const int64_t q0 = c == 0 ? 0 : c * C + 1, q1 = last ? len - 1 : std::min((c + 1) * C, len - 1);
  ChunkRange r;
  if (kind == kLast) {
    r.g0 = lo + q0, r.g1 = lo + q1 + 1;
    r.e0 = lo + c * C, r.e1 = lo + (last ? len - 1 : (c + 1) * C);
  } else {
    r.g0 = hi - 1 - q1, r.g1 = hi - q0;
    r.e0 = r.g0, r.e1 = r.g1;
  }
  r.e1 = std::min(r.e1, n - 1);
  return r;
}

// Copy the diag / arrow strips (dst indexed from block strip_lo: work arrays
// start at the partition) and / or the couplings of one chunk.
void copy_chunk(cudaStream_t s, const BtaDev& dst, const BtaDev& src, const ChunkRange& r, int64_t strip_lo,
                bool strips, bool couplings) {
  const int64_t b = src.b, a = src.a, nb = r.g1 - r.g0, d0 = r.g0 - strip_lo, s0 = r.g0;
  if (strips) {
    copy_async(s, dst.diag + d0 * b * b, src.diag + s0 * b * b, nb * b * b);
    copy_async(s, dst.arrow_row + d0 * a * b, src.arrow_row + s0 * a * b, nb * a * b);
    copy_async(s, dst.arrow_col + d0 * b * a, src.arrow_col + s0 * b * a, nb * b * a);
  }
  if (couplings && r.e1 > r.e0) {
    copy_async(s, dst.lower + r.e0 * b * b, src.lower + r.e0 * b * b, (r.e1 - r.e0) * b * b);
    copy_async(s, dst.upper + r.e0 * b * b, src.upper + r.e0 * b * b, (r.e1 - r.e0) * b * b);
  }
}

}  // namespace

void local_forward(Context& ctx, const BtaDev& A, const BtaDev* B, const BtaDev& WA, const BtaDev* WB,
                   const LocalFactorsDev& F, const HostIo* io) {
  const int64_t lo = F.lo, hi = F.hi, len = hi - lo, b = A.b, a = A.a;
  const bool fused = B != nullptr;
  if (len < 2 || lo < 0 || hi > A.n) throw ShapeError("invalid partition range");
  if (WA.n != len || WA.b != b || WA.a != a) throw ShapeError("partition workspace shape");
  const int mx = (int)std::max(a, b);
  ctx.reserve_slots(64, (int64_t)mx * mx);
  ctx.reset_status();
  ctx.sym_reset(ctx.stream());
  // Working copies of the partition (dist.py:194-202) and zeroed tip deltas.
  // B's strips are staged by the symmetry check (one pass), which also checks
  // this partition's couplings and the tip (the partitions' flags are OR-ed
  // by the host layer: together they cover every pattern block of B).
  auto stage = [&](const BtaDev& src, const BtaDev& w, bool check) {
    if (check) {
      sym_check_strips(ctx, src, 0, lo, hi, &w, lo, ctx.stream());
      sym_check_couplings(ctx, src, lo, std::min(hi, A.n - 1), ctx.stream());
      sym_check_tip(ctx, src, nullptr, ctx.stream());
    } else {
      copy_blocks(ctx, w.diag, src.diag + lo * b * b, len * b * b);
      copy_blocks(ctx, w.arrow_row, src.arrow_row + lo * a * b, len * a * b);
      copy_blocks(ctx, w.arrow_col, src.arrow_col + lo * b * a, len * b * a);
    }
    if (a > 0) cuda_check(cudaMemsetAsync(w.tip, 0, (size_t)(a * a) * sizeof(double2), ctx.stream()), "tip");
  };
  // End-to-end mode: input chunks are queued on the copy stream a few
  // chunks ahead of the sweep's launches (so partitions sharing one copy
  // stream interleave their chunks in progress order instead of one
  // partition's whole input arriving first); the chain waits for chunk c
  // before the first step that touches it.
  const bool streamed = io && io->ha && io->chunk > 0;
  if (streamed && (fused != (io->hb != nullptr))) throw ShapeError("host right-hand side disagrees with factors");
  const int64_t C = streamed ? io->chunk : 1, n_in = streamed ? (len + C - 1) / C : 0;
  constexpr int64_t kLookahead = 3;  // chunks queued ahead of the sweep
  cudaStream_t xs = streamed ? (io->copy_stream ? io->copy_stream : ctx.xfer()) : nullptr;
  // BSEL_XFER_TRACE=1: print chunk arrival vs. chain progress (debug only).
  static const bool trace = getenv("BSEL_XFER_TRACE") != nullptr;
  std::vector<cudaEvent_t> tin, tstep;
  auto tev = [](std::vector<cudaEvent_t>& v, cudaStream_t st) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "trace event");
    cuda_check(cudaEventRecord(e, st), "trace event");
    v.push_back(e);
  };
  if (trace) tev(tstep, ctx.stream());
  int64_t issued = 0;
  auto issue = [&](int64_t upto) {  // queue input chunks [issued, upto]
    for (; streamed && issued <= std::min(upto, n_in - 1); ++issued) {
      const int64_t c = issued;
      const ChunkRange r = in_chunk((PartKind)F.kind, lo, hi, A.n, C, c);
      copy_chunk(xs, WA, *io->ha, r, lo, true, false);
      copy_chunk(xs, A, *io->ha, r, 0, false, true);
      if (fused) {
        copy_chunk(xs, *WB, *io->hb, r, lo, true, false);
        copy_chunk(xs, *B, *io->hb, r, 0, false, true);
        // symmetry of the chunk as it lands (before the sweep mutates it)
        sym_check_strips(ctx, *WB, lo, r.g0, r.g1, nullptr, 0, xs);
        sym_check_couplings(ctx, *B, r.e0, r.e1, xs);
      }
      if (c == 0 && io->copy_tip && a > 0) {
        copy_async(xs, A.tip, io->ha->tip, a * a);
        if (fused) {
          copy_async(xs, B->tip, io->hb->tip, a * a);
          sym_check_tip(ctx, *B, nullptr, xs);
        }
      }
      cuda_check(cudaEventRecord(ctx.xfer_event((int)c), xs), "chunk record");
      if (trace) tev(tin, xs);
    }
  };
  int waited = -1;  // last input chunk the chain stream waited for
  auto need = [&](cudaStream_t s, int64_t pos) {
    if (!streamed) return;
    const int c = (int)std::min<int64_t>(pos / C, n_in - 1);
    issue(c + kLookahead);
    for (int k = waited + 1; k <= c; ++k) cuda_check(cudaStreamWaitEvent(s, ctx.xfer_event(k), 0), "chunk wait");
    waited = std::max(waited, c);
  };
  if (streamed) {
    cuda_check(cudaEventRecord(ctx.event(7), ctx.stream()), "xfer fork");
    cuda_check(cudaStreamWaitEvent(xs, ctx.event(7), 0), "xfer fork");  // buffers free
    issue(kLookahead);
    for (auto* w : {&WA, WB})
      if (w && a > 0) cuda_check(cudaMemsetAsync(w->tip, 0, (size_t)(a * a) * sizeof(double2), ctx.stream()), "tip");
  } else {
    stage(A, WA, false);
    if (fused) stage(*B, *WB, true);
  }
  // Device-resident inputs: the staging check of this partition's B is known
  // before the sweep starts (streamed chunks are checked only as they land).
  ctx.set_forward_symmetry(fused && !streamed ? ctx.sym_now(ctx.stream()) : 0);
  cuda_check(cudaEventRecord(ctx.timer(0), ctx.stream()), "timer");
  auto d = [&](const BtaDev& w, int64_t i) { return w.D(i - lo); };
  auto ar = [&](const BtaDev& w, int64_t i) { return w.AR(i - lo); };
  auto ac = [&](const BtaDev& w, int64_t i) { return w.AC(i - lo); };

  if (F.kind == kMiddle) {
    need(ctx.stream(), 1);
    waited = -1;  // the chain stream still has to wait for itself
    Level L(ctx.stream());
    L.out(F.FR(1)).add(+1, A.U(lo));
    L.out(F.FC(1)).add(+1, A.L(lo));
    if (fused) {
      L.out(F.BFR(1)).add(+1, B->U(lo));
      L.out(F.BFC(1)).add(+1, B->L(lo));
    }
    L.flush();
  }
  streams_fork(ctx);
  if (F.kind == kFirst || F.kind == kLast) {
    const bool down = F.kind == kFirst;
    for (int64_t s = 0; s < len - 1; ++s) {
      const int64_t i = down ? lo + s : hi - 1 - s;
      const int64_t j = down ? i + 1 : i - 1;
      const int64_t e = down ? i : i - 1;  // index of the coupling pair
      need(ctx.chain(), s + 1);
      EndStep st;
      st.Lk = down ? A.L(e) : A.U(e);
      st.Uk = down ? A.U(e) : A.L(e);
      st.ad_i = d(WA, i), st.ad_j = d(WA, j), st.ar_i = ar(WA, i), st.ar_j = ar(WA, j);
      st.ac_i = ac(WA, i), st.ac_j = ac(WA, j), st.tipA = WA.T();
      st.S = F.SA(i - lo);
      if (fused) {
        st.BL = down ? B->L(e) : B->U(e);
        st.BU = down ? B->U(e) : B->L(e);
        st.bd_i = d(*WB, i), st.bd_j = d(*WB, j), st.br_i = ar(*WB, i), st.br_j = ar(*WB, j);
        st.bc_i = ac(*WB, i), st.bc_j = ac(*WB, j), st.tipB = WB->T();
        st.sb = F.SB(i - lo);
        st.f_out = F.EF(i - lo), st.g_out = F.EG(i - lo), st.q_out = F.EQ(i - lo), st.k_out = F.EK(i - lo);
        if (fwd_backward_products()) st.eq_out = F.EEQ(i - lo), st.ek_out = F.EEK(i - lo);
      }
      const bool extra = !fused || fwd_backward_products();
      if (extra || ctx.schur_ok((int)b)) st.h_out = F.EH(i - lo);
      if (extra) st.ha_out = F.EHA(i - lo);
      end_step(ctx, st, fused, (uint64_t)s, i, fwd_slot(s));
      if (trace && (s + 1) % C == 0) tev(tstep, ctx.chain());
    }
  } else {
    for (int64_t i = lo + 1; i < hi - 1; ++i) {
      const int64_t s = i - lo - 1;
      need(ctx.chain(), i + 1 - lo);
      MiddleStep st;
      st.L = A.L(i), st.U = A.U(i);
      st.ad_i = d(WA, i), st.ad_n = d(WA, i + 1), st.ad_lo = d(WA, lo);
      st.ar_i = ar(WA, i), st.ar_n = ar(WA, i + 1), st.ar_lo = ar(WA, lo);
      st.ac_i = ac(WA, i), st.ac_n = ac(WA, i + 1), st.ac_lo = ac(WA, lo), st.tipA = WA.T();
      st.fill_r = F.FR(i - lo), st.fill_c = F.FC(i - lo);
      st.nfill_r = F.FR(i - lo + 1), st.nfill_c = F.FC(i - lo + 1);
      st.S = F.SA(i - lo);
      if (fused) {
        st.BL = B->L(i), st.BU = B->U(i);
        st.bd_i = d(*WB, i), st.bd_n = d(*WB, i + 1), st.bd_lo = d(*WB, lo);
        st.br_i = ar(*WB, i), st.br_n = ar(*WB, i + 1), st.br_lo = ar(*WB, lo);
        st.bc_i = ac(*WB, i), st.bc_n = ac(*WB, i + 1), st.bc_lo = ac(*WB, lo), st.tipB = WB->T();
        st.bfill_r = F.BFR(i - lo), st.bfill_c = F.BFC(i - lo);
        st.nbfill_r = F.BFR(i - lo + 1), st.nbfill_c = F.BFC(i - lo + 1);
        st.sb = F.SB(i - lo);
        st.fn_out = F.EF(i - lo), st.fr_out = F.EFR(i - lo), st.g_out = F.EG(i - lo);
        st.qn_out = F.EQ(i - lo), st.qr_out = F.EQR(i - lo), st.kk_out = F.EK(i - lo);
        // middles: the backward's h / e products are formed here -- a middle
        // partition's forward finishes early (4 GPUs: 175 vs 218 ms for the
        // ends) while its k = 3 backward is the longest
        st.ha_out = F.EHA(i - lo), st.eq_out = F.EEQ(i - lo), st.ek_out = F.EEK(i - lo);
      }
      if (fused || ctx.schur_ok((int)b)) st.h_out = F.EH(i - lo);
      middle_step(ctx, st, fused, (uint64_t)s, i, fwd_slot(s));
    }
  }
  streams_join(ctx);
  if (streamed) {
    issue(n_in - 1);
    cuda_check(cudaStreamWaitEvent(ctx.stream(), ctx.xfer_event((int)n_in - 1), 0), "copies done");
  }
  if (trace) {
    tev(tstep, ctx.stream());
    cuda_check(cudaStreamSynchronize(ctx.stream()), "trace sync");
    fprintf(stderr, "[xfer] part lo=%lld kind=%d: chunk arrival / chain step-block done (ms)\n", (long long)lo, F.kind);
    for (size_t k = 1; k < std::max(tin.size() + 1, tstep.size()); ++k) {
      float a_ms = -1, s_ms = -1;
      if (k - 1 < tin.size()) cudaEventElapsedTime(&a_ms, tstep[0], tin[k - 1]);
      if (k < tstep.size()) cudaEventElapsedTime(&s_ms, tstep[0], tstep[k]);
      fprintf(stderr, "[xfer] %zu %.2f %.2f\n", k - 1, a_ms, s_ms);
    }
    for (auto e : tin) cudaEventDestroy(e);
    for (auto e : tstep) cudaEventDestroy(e);
  }
  cuda_check(cudaEventRecord(ctx.timer(1), ctx.stream()), "timer");
}

void local_backward(Context& ctx, const BtaDev& A, const BtaDev* B, const LocalFactorsDev& F, const BtaDev& WA,
                    const BtaDev* WB, const BtaDev& XR, const BtaDev* ZR, int64_t k_top, int64_t k_bot,
                    bool write_tip, const BtaDev& XA, const BtaDev* XB, const HostIo* io) {
  const int64_t lo = F.lo, hi = F.hi, len = hi - lo, b = A.b, a = A.a;
  const bool fused = F.fused;
  if (fused && (!B || !WB || !ZR || !XB)) throw ShapeError("fused factors require the right-hand side");
  const int mx = (int)std::max(a, b);
  ctx.reserve_slots(back_sweep_slots(), (int64_t)mx * mx);
  cudaStream_t s = ctx.stream();
  cuda_check(cudaEventRecord(ctx.timer(2), s), "timer");
  // first / last partitions: the common 2-wave 64x64 threshold (2 GPUs:
  // backward 294 vs 305 ms); middles (k = 3, larger levels): the wide one
  BackSweep sweep(ctx, F.kind == kMiddle ? kTileAutoWide : kTileAuto);
  // End-to-end mode: move each chunk of finished outputs to the host on the
  // copy stream while the sweep continues.
  const bool streamed = io && io->hxa && io->chunk > 0;
  if (streamed && fused && !io->hxb) throw ShapeError("host output for the quadratic solution missing");
  const int64_t C = streamed ? io->chunk : 1, n_out = std::max<int64_t>(1, (len - 1 + C - 1) / C);
  int64_t sent = 0;  // chunks queued
  auto send = [&](int64_t steps, bool final) {  // backward steps [0, steps) are complete
    if (!streamed) return;
    sweep.fence();
    while (sent < n_out && (final || (sent + 1) * C <= steps) && (final || sent < n_out - 1)) {
      cudaEvent_t ev = ctx.xfer_event((int)sent);
      cuda_check(cudaEventRecord(ev, s), "chunk record");
      cudaStream_t xs = ctx.xfer();
      cuda_check(cudaStreamWaitEvent(xs, ev, 0), "chunk wait");
      const ChunkRange r = out_chunk((PartKind)F.kind, lo, hi, A.n, C, sent, n_out);
      copy_chunk(xs, *io->hxa, XA, r, 0, true, true);
      if (fused) copy_chunk(xs, *io->hxb, *XB, r, 0, true, true);
      if (sent == 0 && write_tip && a > 0) {
        copy_async(xs, io->hxa->tip, XA.tip, a * a);
        if (fused) copy_async(xs, io->hxb->tip, XB->tip, a * a);
      }
      ++sent;
    }
    if (final) {
      cuda_check(cudaEventRecord(ctx.event(7), ctx.xfer()), "copies done");
      cuda_check(cudaStreamWaitEvent(s, ctx.event(7), 0), "copies done");
    }
  };
  const Mat ytt = XR.T();
  const Mat ztt = fused ? ZR->T() : Mat{};
  Level L(s, kTileAutoWide);
  if (write_tip) {
    L.out(XA.T()).add(+1, XR.T());
    if (fused) L.out(XB->T()).add(+1, ZR->T());
  }
  auto seed = [&](int64_t k, int64_t g) {
    L.out(XA.D(g)).add(+1, XR.D(k));
    L.out(XA.AC(g)).add(+1, XR.AC(k));
    L.out(XA.AR(g)).add(+1, XR.AR(k));
    if (fused) {
      L.out(XB->D(g)).add(+1, ZR->D(k));
      L.out(XB->AC(g)).add(+1, ZR->AC(k));
      L.out(XB->AR(g)).add(+1, ZR->AR(k));
    }
  };
  auto separator = [&](int64_t k) {
    L.out(XA.L(hi - 1)).add(+1, XR.L(k));
    L.out(XA.U(hi - 1)).add(+1, XR.U(k));
    if (fused) {
      L.out(XB->L(hi - 1)).add(+1, ZR->L(k));
      L.out(XB->U(hi - 1)).add(+1, ZR->U(k));
    }
  };
  auto el = [&](const BtaDev& w, int64_t i, bool row) { return row ? w.AR(i - lo) : w.AC(i - lo); };

  if (F.kind == kFirst || F.kind == kLast) {
    const bool down = F.kind == kFirst;
    if (down) {
      seed(k_bot, hi - 1);
      if (hi < A.n) separator(k_bot);
    } else {
      seed(k_top, lo);
    }
    L.flush();
    sweep.begin();
    for (int64_t t = 0; t < len - 1; ++t) {
      const int64_t i = down ? hi - 2 - t : lo + 1 + t;
      const int64_t p = down ? i + 1 : i - 1;  // previously solved neighbour
      const int64_t e = down ? i : i - 1;
      BackStep st;
      st.k = 2;
      st.g = F.SA(i - lo);
      st.rs[0] = down ? A.U(e) : A.L(e), st.rs[1] = el(WA, i, false);
      st.qs[0] = down ? A.L(e) : A.U(e), st.qs[1] = el(WA, i, true);
      st.ya[0][0] = XA.D(p), st.ya[0][1] = XA.AC(p), st.ya[1][0] = XA.AR(p), st.ya[1][1] = ytt;
      st.row[0] = down ? XA.U(e) : XA.L(e), st.row[1] = XA.AC(i);
      st.col[0] = down ? XA.L(e) : XA.U(e), st.col[1] = XA.AR(i);
      {  // retained by the forward (see local_forward)
        const bool extra = !fused || fwd_backward_products();
        if (extra || ctx.schur_ok((int)b)) st.hpre[0] = F.EH(i - lo);
        if (extra) st.hpre[1] = F.EHA(i - lo);
      }
      st.diag = XA.D(i);
      if (fused) {
        st.sc = F.SB(i - lo);
        st.cpre[0] = F.EF(i - lo), st.cpre[1] = F.EG(i - lo), st.qpre[0] = F.EQ(i - lo), st.qpre[1] = F.EK(i - lo);
        if (fwd_backward_products()) st.epre[0] = F.EEQ(i - lo), st.epre[1] = F.EEK(i - lo);
        st.ss[0] = down ? B->U(e) : B->L(e), st.ss[1] = el(*WB, i, false);
        st.ws[0] = down ? B->L(e) : B->U(e), st.ws[1] = el(*WB, i, true);
        st.yb[0][0] = XB->D(p), st.yb[0][1] = XB->AC(p), st.yb[1][0] = XB->AR(p), st.yb[1][1] = ztt;
        st.zrow[0] = down ? XB->U(e) : XB->L(e), st.zrow[1] = XB->AC(i);
        st.zcol[0] = down ? XB->L(e) : XB->U(e), st.zcol[1] = XB->AR(i);
        st.zdiag = XB->D(i);
      }
      sweep.step(st);
      if (streamed && (t + 1) % C == 0) send(t + 1, false);
    }
  } else {
    seed(k_top, lo);
    seed(k_bot, hi - 1);
    if (hi < A.n) separator(k_bot);
    // X(lo, hi-1) / X(hi-1, lo) from the reduced system's fill coupling.
    Mat yfr = XR.U(k_top), yfc = XR.L(k_top);
    Mat zfr = fused ? ZR->U(k_top) : Mat{}, zfc = fused ? ZR->L(k_top) : Mat{};
    if (len == 2) {
      L.out(XA.U(lo)).add(+1, yfr);
      L.out(XA.L(lo)).add(+1, yfc);
      if (fused) {
        L.out(XB->U(lo)).add(+1, zfr);
        L.out(XB->L(lo)).add(+1, zfc);
      }
    }
    L.flush();
    sweep.begin();
    for (int64_t i = hi - 2; i > lo; --i) {
      const bool last_step = i == lo + 1;
      BackStep st;
      st.k = 3;
      st.g = F.SA(i - lo);
      st.rs[0] = F.FC(i - lo), st.rs[1] = A.U(i), st.rs[2] = el(WA, i, false);
      st.qs[0] = F.FR(i - lo), st.qs[1] = A.L(i), st.qs[2] = el(WA, i, true);
      const Mat y00 = XA.D(lo), y0t = XA.AC(lo), yt0 = XA.AR(lo);
      st.ya[0][0] = y00, st.ya[0][1] = yfr, st.ya[0][2] = y0t;
      st.ya[1][0] = yfc, st.ya[1][1] = XA.D(i + 1), st.ya[1][2] = XA.AC(i + 1);
      st.ya[2][0] = yt0, st.ya[2][1] = XA.AR(i + 1), st.ya[2][2] = ytt;
      // row[0] = X(i, lo), col[0] = X(lo, i): carried to the next step (ring-allocated).
      if (last_step) st.row[0] = XA.L(lo), st.col[0] = XA.U(lo);
      st.row[1] = XA.U(i), st.row[2] = XA.AC(i);
      st.col[1] = XA.L(i), st.col[2] = XA.AR(i);
      st.diag = XA.D(i);
      if (fused) {
        st.sc = F.SB(i - lo);
        st.cpre[0] = F.EFR(i - lo), st.cpre[1] = F.EF(i - lo), st.cpre[2] = F.EG(i - lo);
        st.qpre[0] = F.EQR(i - lo), st.qpre[1] = F.EQ(i - lo), st.qpre[2] = F.EK(i - lo);
        st.hpre[1] = F.EH(i - lo), st.hpre[2] = F.EHA(i - lo);  // formed by the middle forward
        st.epre[1] = F.EEQ(i - lo), st.epre[2] = F.EEK(i - lo);
        st.ss[0] = F.BFC(i - lo), st.ss[1] = B->U(i), st.ss[2] = el(*WB, i, false);
        st.ws[0] = F.BFR(i - lo), st.ws[1] = B->L(i), st.ws[2] = el(*WB, i, true);
        const Mat z00 = XB->D(lo), z0t = XB->AC(lo), zt0 = XB->AR(lo);
        st.yb[0][0] = z00, st.yb[0][1] = zfr, st.yb[0][2] = z0t;
        st.yb[1][0] = zfc, st.yb[1][1] = XB->D(i + 1), st.yb[1][2] = XB->AC(i + 1);
        st.yb[2][0] = zt0, st.yb[2][1] = XB->AR(i + 1), st.yb[2][2] = ztt;
        if (last_step) st.zrow[0] = XB->L(lo), st.zcol[0] = XB->U(lo);
        st.zrow[1] = XB->U(i), st.zrow[2] = XB->AC(i);
        st.zcol[1] = XB->L(i), st.zcol[2] = XB->AR(i);
        st.zdiag = XB->D(i);
      }
      sweep.step(st);
      const int64_t t = hi - 2 - i;
      if (streamed && (t + 1) % C == 0) send(t + 1, false);
      yfr = st.col[0], yfc = st.row[0];
      if (fused) zfr = st.zcol[0], zfc = st.zrow[0];
    }
  }
  L.flush();
  sweep.end();
  send(len - 1, true);
  cuda_check(cudaEventRecord(ctx.timer(3), s), "timer");
}

}  // namespace bsel
