// C ABI (include/btasel_b200.h): status mapping, workspace management and the
// non-destructive solve facade.  No exception crosses this boundary.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/btasel_b200.h"
#include "generate.cuh"
#include "inverse.cuh"
#include "partition.cuh"
#include "steps.cuh"
#include "solver.cuh"

struct bsel_context {
  std::unique_ptr<bsel::Context> impl;
  void* solve_ws = nullptr;
  size_t solve_ws_bytes = 0;
  double2* mm_tmp = nullptr;
  size_t mm_tmp_elems = 0;
};

namespace {

using namespace bsel;

struct SingularError : std::runtime_error {
  int64_t index;
  SingularError(const std::string& m, int64_t i) : std::runtime_error(m), index(i) {}
};
struct ArgError : std::runtime_error {
  explicit ArgError(const std::string& m) : std::runtime_error(m) {}
};

void fill(bsel_status_t* st, int code, int64_t index, const char* msg) {
  if (!st) return;
  st->code = code;
  st->reserved = 0;
  st->index = index;
  std::snprintf(st->message, sizeof(st->message), "%s", msg ? msg : "");
}

template <class F>
int guarded(bsel_status_t* st, F&& f) {
  try {
    f();
    fill(st, BSEL_OK, -1, "");
    return BSEL_OK;
  } catch (const SingularError& e) {
    fill(st, BSEL_ERR_SINGULAR, e.index, e.what());
    return BSEL_ERR_SINGULAR;
  } catch (const ShapeError& e) {
    fill(st, BSEL_ERR_SHAPE, -1, e.what());
    return BSEL_ERR_SHAPE;
  } catch (const ArgError& e) {
    fill(st, BSEL_ERR_ARG, -1, e.what());
    return BSEL_ERR_ARG;
  } catch (const CudaError& e) {
    fill(st, BSEL_ERR_CUDA, -1, e.what());
    return BSEL_ERR_CUDA;
  } catch (const std::exception& e) {
    fill(st, BSEL_ERR_INTERNAL, -1, e.what());
    return BSEL_ERR_INTERNAL;
  }
}

inline double2* dp(double* p) { return reinterpret_cast<double2*>(p); }
inline const double2* dp(const double* p) { return reinterpret_cast<const double2*>(p); }

BtaDev to_dev(const bsel_bta_t& m) {
  BtaDev d;
  d.n = m.n;
  d.b = m.b;
  d.a = m.a;
  d.diag = dp(m.diag);
  d.lower = dp(m.lower);
  d.upper = dp(m.upper);
  d.arrow_row = dp(m.arrow_row);
  d.arrow_col = dp(m.arrow_col);
  d.tip = dp(m.tip);
  return d;
}

FactorsDev to_dev(const bsel_factors_t& f) {
  FactorsDev d;
  d.n = f.n;
  d.b = f.b;
  d.a = f.a;
  d.fused = f.fused != 0;
  d.s_a = dp(f.s_a);
  d.s_b = dp(f.s_b);
  d.b_diag_last = dp(f.b_diag_last);
  d.tip_inv = dp(f.tip_inv);
  d.b_tip = dp(f.b_tip);
  d.arrow_row_elim = dp(f.arrow_row_elim);
  d.arrow_col_elim = dp(f.arrow_col_elim);
  d.b_arrow_row_elim = dp(f.b_arrow_row_elim);
  d.b_arrow_col_elim = dp(f.b_arrow_col_elim);
  d.elim_f = dp(f.elim_f);
  d.elim_g = dp(f.elim_g);
  d.elim_q = dp(f.elim_q);
  d.elim_k = dp(f.elim_k);
  d.elim_h = dp(f.elim_h);
  d.elim_ha = dp(f.elim_ha);
  d.elim_eq = dp(f.elim_eq);
  d.elim_ek = dp(f.elim_ek);
  return d;
}

void check_shape(const bsel_bta_t* m, const char* what) {
  if (!m) throw ArgError(std::string(what) + " is NULL");
  if (m->n < 1 || m->b < 1 || m->a < 0)
    throw ShapeError(std::string("invalid shape parameters for ") + what);
}

void check_same(const bsel_bta_t* x, const bsel_bta_t* y) {
  if (x->n != y->n || x->b != y->b || x->a != y->a)
    throw ShapeError("right-hand side shape differs from system shape");
}

void raise_if_singular(Context& ctx, int64_t n) {
  SingularInfo info = ctx.read_status();
  if (!info.singular) return;
  char msg[256];
  if (info.index >= n)
    std::snprintf(msg, sizeof msg, "singular updated arrow tip (input not diagonally dominant?)");
  else
    std::snprintf(msg, sizeof msg, "singular pivot at diagonal block %lld (input not diagonally dominant?)",
                  (long long)info.index);
  throw SingularError(msg, info.index);
}

__global__ void axpby_kernel(double2* d, int64_t ldd, const double2* x, int64_t ldx, double2 alpha,
                             const double2* c, int64_t ldc, double2 beta, int64_t m, int64_t n) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  int64_t i = e / n, j = e % n;
  double2 v = x[i * ldx + j];
  double2 r = make_double2(alpha.x * v.x - alpha.y * v.y, alpha.x * v.y + alpha.y * v.x);
  if (c) {
    double2 w = c[i * ldc + j];
    r.x += beta.x * w.x - beta.y * w.y;
    r.y += beta.x * w.y + beta.y * w.x;
  }
  d[i * ldd + j] = r;
}

struct SolveLayout {
  size_t off[21];
  size_t total;
};

// Workspace: working copies of the mutated arrays (diag, arrow strips, tip)
// of A (and B) plus the factors.  Off-diagonal blocks are read in place.
SolveLayout solve_layout(int64_t n, int64_t b, int64_t a, bool fused) {
  SolveLayout L{};
  size_t cur = 0;
  auto take = [&](int slot, int64_t elems) {
    cur = (cur + 255) & ~size_t(255);
    L.off[slot] = cur;
    cur += (size_t)std::max<int64_t>(elems, 0) * sizeof(double2);
  };
  take(0, n * b * b);  // A diag
  take(1, n * a * b);  // A arrow_row
  take(2, n * b * a);  // A arrow_col
  take(3, a * a);      // A tip
  take(4, n * b * b);  // s_a
  take(5, a * a);      // tip_inv
  if (fused) {
    take(6, n * b * b);        // B diag
    take(7, n * a * b);        // B arrow_row
    take(8, n * b * a);        // B arrow_col
    take(9, a * a);            // B tip
    take(10, (n - 1) * b * b); // s_b
    take(11, b * b);           // b_diag_last
    take(12, a * a);           // b_tip
    take(15, n * b * b);       // elim_q
    take(16, n * b * a);       // elim_k
  }
  take(13, n * b * b);  // elim_f
  take(14, n * a * b);  // elim_g
  take(17, n * b * b);  // elim_h
  const bool extra = fwd_backward_products();
  if (extra || !fused) take(18, n * b * a);  // elim_ha
  if (fused && extra) {
    take(19, n * b * b);  // elim_eq
    take(20, n * b * a);  // elim_ek
  }
  L.total = cur + 256;
  return L;
}

}  // namespace

extern "C" {

int bsel_abi_version(void) { return BSEL_ABI_VERSION; }

int bsel_context_create(int device, bsel_context_t** out, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!out) throw ArgError("out is NULL");
    auto* c = new bsel_context;
    try {
      c->impl.reset(new Context(device));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int bsel_context_destroy(bsel_context_t* ctx) {
  if (!ctx) return BSEL_OK;
  if (ctx->solve_ws) cudaFree(ctx->solve_ws);
  if (ctx->mm_tmp) cudaFree(ctx->mm_tmp);
  delete ctx;
  return BSEL_OK;
}

int bsel_context_set_stream(bsel_context_t* ctx, void* cuda_stream) {
  if (!ctx) return BSEL_ERR_ARG;
  ctx->impl->set_stream(static_cast<cudaStream_t>(cuda_stream));
  return BSEL_OK;
}

int bsel_context_set_inverse_grid(bsel_context_t* ctx, int ctas) {
  if (!ctx || ctas < 0) return BSEL_ERR_ARG;
  ctx->impl->set_inverse_grid(ctas);
  return BSEL_OK;
}

int bsel_context_set_b_symmetry(bsel_context_t* ctx, int mode) {
  if (!ctx || mode < -1 || mode > Context::kSymAuto) return BSEL_ERR_ARG;
  ctx->impl->set_b_symmetry(mode);
  return BSEL_OK;
}

int bsel_context_set_aux_avoid_sms(bsel_context_t* ctx, int n) {
  if (!ctx || n < 0 || n >= device_sm_count()) return BSEL_ERR_ARG;
  ctx->impl->set_aux_avoid_sms(n);
  return BSEL_OK;
}

int bsel_context_b_symmetry(bsel_context_t* ctx, int* flags, int* mode) {
  if (!ctx) return BSEL_ERR_ARG;
  if (flags) *flags = ctx->impl->sym_flags();
  if (mode) *mode = ctx->impl->b_symmetry();
  return BSEL_OK;
}

int bsel_synchronize(bsel_context_t* ctx, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    cuda_check(cudaStreamSynchronize(ctx->impl->stream()), "synchronize");
    cuda_check(cudaStreamSynchronize(ctx->impl->aux()), "synchronize aux");
  });
}

int bsel_last_timings(bsel_context_t* ctx, double* forward_ms, double* backward_ms) {
  if (!ctx) return BSEL_ERR_ARG;
  Context& c = *ctx->impl;
  if (cudaEventSynchronize(c.timer(3)) != cudaSuccess) return BSEL_ERR_CUDA;
  float f = 0.f, b = 0.f;
  if (cudaEventElapsedTime(&f, c.timer(0), c.timer(1)) != cudaSuccess) f = 0.f;
  if (cudaEventElapsedTime(&b, c.timer(2), c.timer(3)) != cudaSuccess) b = 0.f;
  if (forward_ms) *forward_ms = f;
  if (backward_ms) *backward_ms = b;
  return BSEL_OK;
}

int bsel_block_multiply_acc(bsel_context_t* ctx, double* d, int64_t ldd, const double* c, int64_t ldc,
                            const double* a, int64_t lda, int trans_a, const double* b, int64_t ldb,
                            int trans_b, int64_t m, int64_t n, int64_t k, double alpha_re, double alpha_im,
                            double beta_re, double beta_im, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    if (m < 0 || n < 0 || k < 0) throw ShapeError("negative dimension");
    if (m == 0 || n == 0) return;
    Context& cx = *ctx->impl;
    cudaStream_t s = cx.stream();
    const bool simple_alpha = alpha_im == 0.0 && (alpha_re == 1.0 || alpha_re == -1.0);
    const bool simple_beta = !c || (beta_re == 1.0 && beta_im == 0.0) || (beta_re == 0.0 && beta_im == 0.0);
    const int ra = trans_a ? (int)k : (int)m, ca = trans_a ? (int)m : (int)k;
    const int rb = trans_b ? (int)n : (int)k, cb = trans_b ? (int)k : (int)n;
    Mat A{const_cast<double2*>(dp(a)), lda, ra, ca}, B{const_cast<double2*>(dp(b)), ldb, rb, cb};
    Mat D{dp(d), ldd, (int)m, (int)n};
    if (simple_alpha && simple_beta) {
      Level L(s);
      L.out(D);
      if (c && beta_re == 1.0) L.add(+1, Mat{const_cast<double2*>(dp(c)), ldc, (int)m, (int)n});
      if (k > 0) L.mm(alpha_re > 0 ? +1 : -1, A, trans_a ? H : N, B, trans_b ? H : N);
      L.flush();
    } else {
      const size_t elems = (size_t)m * n;
      if (elems > ctx->mm_tmp_elems) {
        cuda_check(cudaStreamSynchronize(s), "sync");
        if (ctx->mm_tmp) cudaFree(ctx->mm_tmp);
        cuda_check(cudaMalloc(&ctx->mm_tmp, elems * sizeof(double2)), "tmp");
        ctx->mm_tmp_elems = elems;
      }
      Mat T{ctx->mm_tmp, n, (int)m, (int)n};
      Level L(s);
      L.out(T);
      if (k > 0) L.mm(+1, A, trans_a ? H : N, B, trans_b ? H : N);
      L.flush();
      const int64_t tot = m * n;
      axpby_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
          dp(d), ldd, ctx->mm_tmp, n, make_double2(alpha_re, alpha_im), c ? dp(c) : nullptr, ldc,
          make_double2(beta_re, beta_im), m, n);
      cuda_check(cudaGetLastError(), "axpby");
    }
  });
}

int bsel_block_inverse(bsel_context_t* ctx, const double* a, int64_t lda, double* out, int64_t ldo, int64_t n,
                       bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    if (n < 0) throw ShapeError("negative dimension");
    if (n == 0) return;
    Context& cx = *ctx->impl;
    cudaStream_t s = cx.stream();
    int* flag = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s), "flag");
    cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), s), "flag");
    double2* work = cx.inv_work(block_inverse_workspace((int)n));
    cudaError_t e = launch_block_inverse(dp(a), lda, dp(out), ldo, (int)n, work, flag, nullptr, 0, s,
                                         cx.inverse_grid());
    int h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(flag, s);
    cuda_check(e, "block inverse");
    if (h >= 2) {
      char msg[128];
      std::snprintf(msg, sizeof msg, "exactly singular pivot at row %d", h - 2);
      throw SingularError(msg, h - 2);
    }
  });
}

int bsel_bta_forward(bsel_context_t* ctx, const bsel_bta_t* a_work, const bsel_bta_t* b_work,
                     const bsel_factors_t* f, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx || !f) throw ArgError("NULL argument");
    check_shape(a_work, "a");
    if (b_work) check_same(a_work, b_work);
    if ((f->fused != 0) != (b_work != nullptr)) throw ArgError("factors mode disagrees with right-hand side");
    BtaDev A = to_dev(*a_work), B;
    Context& cx = *ctx->impl;
    if (b_work) {
      B = to_dev(*b_work);
      cx.sym_reset(cx.stream());
      sym_check_strips(cx, B, 0, 0, B.n, nullptr, 0, cx.stream());
      sym_check_couplings(cx, B, 0, B.n - 1, cx.stream());
      sym_check_tip(cx, B, nullptr, cx.stream());
    }
    cx.set_forward_symmetry(b_work ? cx.sym_now(cx.stream()) : 0);
    bta_forward(cx, A, b_work ? &B : nullptr, to_dev(*f));
    raise_if_singular(*ctx->impl, a_work->n);
  });
}

int bsel_bta_backward(bsel_context_t* ctx, const bsel_factors_t* f, const bsel_bta_t* a, const bsel_bta_t* b,
                      const bsel_bta_t* x_a, const bsel_bta_t* x_b, int diagonal_only, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx || !f) throw ArgError("NULL argument");
    check_shape(a, "a");
    check_shape(x_a, "x_a");
    if (f->fused && (!b || !x_b)) throw ShapeError("fused factors require the right-hand side");
    BtaDev A = to_dev(*a), XA = to_dev(*x_a), B, XB;
    if (f->fused) {
      B = to_dev(*b);
      XB = to_dev(*x_b);
    }
    bta_backward(*ctx->impl, to_dev(*f), A, f->fused ? &B : nullptr, XA, f->fused ? &XB : nullptr,
                 diagonal_only != 0);
    cuda_check(cudaGetLastError(), "backward");
  });
}

int bsel_solve_workspace_size(int64_t n, int64_t b, int64_t a, int fused, size_t* bytes) {
  if (!bytes || n < 1 || b < 1 || a < 0) return BSEL_ERR_ARG;
  *bytes = solve_layout(n, b, a, fused != 0).total;
  return BSEL_OK;
}

int bsel_solve_selected(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b, const bsel_bta_t* x_a,
                        const bsel_bta_t* x_b, int diagonal_only, void* workspace, size_t workspace_bytes,
                        bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    check_shape(a, "a");
    check_shape(x_a, "x_a");
    check_same(a, x_a);
    const bool fused = b != nullptr;
    if (fused) {
      check_same(a, b);
      if (!x_b) throw ArgError("x_b is NULL in fused mode");
      check_same(a, x_b);
    }
    const int64_t n = a->n, bs = a->b, as = a->a;
    SolveLayout lay = solve_layout(n, bs, as, fused);
    char* ws = static_cast<char*>(workspace);
    Context& cx = *ctx->impl;
    cudaStream_t s = cx.stream();
    if (!ws || workspace_bytes < lay.total) {
      if (ctx->solve_ws_bytes < lay.total) {
        cuda_check(cudaStreamSynchronize(s), "sync");
        if (ctx->solve_ws) cudaFree(ctx->solve_ws);
        ctx->solve_ws = nullptr;
        cuda_check(cudaMalloc(&ctx->solve_ws, lay.total), "solve workspace");
        ctx->solve_ws_bytes = lay.total;
      }
      ws = static_cast<char*>(ctx->solve_ws);
    }
    ws = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    auto at = [&](int slot) { return reinterpret_cast<double2*>(ws + lay.off[slot]); };
    auto cp = [&](double2* dst, const double* src, int64_t elems) {
      if (elems > 0)
        cuda_check(cudaMemcpyAsync(dst, src, (size_t)elems * sizeof(double2), cudaMemcpyDeviceToDevice, s),
                   "input copy");
    };
    // Working copies (rgf.py:520-521: the facade never mutates its inputs).
    BtaDev A = to_dev(*a);
    A.diag = at(0);
    A.arrow_row = at(1);
    A.arrow_col = at(2);
    A.tip = at(3);
    cp(A.diag, a->diag, n * bs * bs);
    cp(A.arrow_row, a->arrow_row, n * as * bs);
    cp(A.arrow_col, a->arrow_col, n * bs * as);
    cp(A.tip, a->tip, as * as);
    FactorsDev F;
    F.n = n;
    F.b = bs;
    F.a = as;
    F.fused = fused;
    F.s_a = at(4);
    F.tip_inv = at(5);
    F.arrow_row_elim = A.arrow_row;
    F.arrow_col_elim = A.arrow_col;
    F.elim_f = at(13);
    F.elim_g = as > 0 ? at(14) : nullptr;
    F.elim_h = at(17);
    const bool extra = fwd_backward_products();
    F.elim_ha = as > 0 && (extra || !fused) ? at(18) : nullptr;
    if (fused && extra) {
      F.elim_eq = at(19);
      F.elim_ek = as > 0 ? at(20) : nullptr;
    }
    BtaDev B;
    if (fused) {
      B = to_dev(*b);
      B.diag = at(6);
      B.arrow_row = at(7);
      B.arrow_col = at(8);
      B.tip = at(9);
      // Working copies of B, staged by the symmetry check (one pass).
      const BtaDev Bin = to_dev(*b);
      cx.sym_reset(s);
      sym_check_strips(cx, Bin, 0, 0, n, &B, 0, s);
      sym_check_couplings(cx, Bin, 0, n - 1, s);
      sym_check_tip(cx, Bin, B.tip, s);
      F.s_b = at(10);
      F.b_diag_last = at(11);
      F.b_tip = at(12);
      F.b_arrow_row_elim = B.arrow_row;
      F.b_arrow_col_elim = B.arrow_col;
      F.elim_q = at(15);
      F.elim_k = as > 0 ? at(16) : nullptr;
    }
    cx.set_forward_symmetry(fused ? cx.sym_now(s) : 0);
    bta_forward(cx, A, fused ? &B : nullptr, F);
    raise_if_singular(cx, n);
    BtaDev XA = to_dev(*x_a), XB;
    if (fused) XB = to_dev(*x_b);
    // Original off-diagonals are read in place (never modified by the sweep).
    bta_backward(cx, F, A, fused ? &B : nullptr, XA, fused ? &XB : nullptr, diagonal_only != 0);
    cuda_check(cudaStreamSynchronize(s), "solve");
  });
}

static LocalFactorsDev to_dev(const bsel_local_factors_t& f, int64_t b, int64_t a) {
  LocalFactorsDev d;
  d.lo = f.lo;
  d.hi = f.hi;
  d.b = b;
  d.a = a;
  d.kind = f.kind;
  d.fused = f.fused != 0;
  d.s_a = dp(f.s_a);
  d.s_b = dp(f.s_b);
  d.fill_row = dp(f.fill_row);
  d.fill_col = dp(f.fill_col);
  d.b_fill_row = dp(f.b_fill_row);
  d.b_fill_col = dp(f.b_fill_col);
  d.elim_f = dp(f.elim_f);
  d.elim_g = dp(f.elim_g);
  d.elim_q = dp(f.elim_q);
  d.elim_k = dp(f.elim_k);
  d.elim_fr = dp(f.elim_fr);
  d.elim_qr = dp(f.elim_qr);
  d.elim_h = dp(f.elim_h);
  d.elim_ha = dp(f.elim_ha);
  d.elim_eq = dp(f.elim_eq);
  d.elim_ek = dp(f.elim_ek);
  return d;
}

// Host end-to-end descriptors (pointers are host memory; shapes must match).
struct HostIoArgs {
  BtaDev a, b, xa, xb;
  HostIo io;
};

static const HostIo* to_io(const bsel_host_io_t* h, const bsel_bta_t* like, HostIoArgs& out) {
  if (!h) return nullptr;
  if (h->chunk_blocks <= 0) throw ArgError("chunk_blocks must be positive");
  auto one = [&](const bsel_bta_t* m, BtaDev& d, const char* what) -> const BtaDev* {
    if (!m) return nullptr;
    check_same(like, m);
    (void)what;
    d = to_dev(*m);
    return &d;
  };
  out.io.ha = one(h->a, out.a, "a");
  out.io.hb = one(h->b, out.b, "b");
  out.io.hxa = one(h->x_a, out.xa, "x_a");
  out.io.hxb = one(h->x_b, out.xb, "x_b");
  out.io.chunk = h->chunk_blocks;
  out.io.copy_tip = h->copy_tip != 0;
  out.io.copy_stream = static_cast<cudaStream_t>(h->copy_stream);
  return &out.io;
}

int bsel_local_forward(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b, const bsel_bta_t* a_work,
                       const bsel_bta_t* b_work, const bsel_local_factors_t* f, const bsel_host_io_t* io,
                       bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx || !f) throw ArgError("NULL argument");
    check_shape(a, "a");
    check_shape(a_work, "a_work");
    if (f->kind < 0 || f->kind > 2) throw ArgError("invalid partition kind");
    if ((f->fused != 0) != (b != nullptr) || (b != nullptr) != (b_work != nullptr))
      throw ArgError("factors mode disagrees with right-hand side");
    if (b) check_same(a, b);
    BtaDev A = to_dev(*a), WA = to_dev(*a_work), B, WB;
    if (b) {
      B = to_dev(*b);
      WB = to_dev(*b_work);
    }
    HostIoArgs hio;
    local_forward(*ctx->impl, A, b ? &B : nullptr, WA, b ? &WB : nullptr, to_dev(*f, a->b, a->a), to_io(io, a, hio));
    raise_if_singular(*ctx->impl, a->n);
  });
}

int bsel_local_backward(bsel_context_t* ctx, const bsel_bta_t* a, const bsel_bta_t* b,
                        const bsel_local_factors_t* f, const bsel_bta_t* a_work, const bsel_bta_t* b_work,
                        const bsel_bta_t* x_red, const bsel_bta_t* z_red, int64_t k_top, int64_t k_bot,
                        int write_tip, const bsel_bta_t* x_a, const bsel_bta_t* x_b,
                        const bsel_host_io_t* io, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx || !f) throw ArgError("NULL argument");
    check_shape(a, "a");
    check_shape(x_a, "x_a");
    check_shape(x_red, "x_red");
    const bool fused = f->fused != 0;
    if (fused && (!b || !b_work || !z_red || !x_b)) throw ShapeError("fused factors require the right-hand side");
    BtaDev A = to_dev(*a), WA = to_dev(*a_work), XR = to_dev(*x_red), XA = to_dev(*x_a), B, WB, ZR, XB;
    HostIoArgs hio;
    const HostIo* hp = to_io(io, a, hio);
    if (fused) {
      B = to_dev(*b);
      WB = to_dev(*b_work);
      ZR = to_dev(*z_red);
      XB = to_dev(*x_b);
    }
    local_backward(*ctx->impl, A, fused ? &B : nullptr, to_dev(*f, a->b, a->a), WA, fused ? &WB : nullptr, XR,
                   fused ? &ZR : nullptr, k_top, k_bot, write_tip != 0, XA, fused ? &XB : nullptr, hp);
    cuda_check(cudaGetLastError(), "local backward");
  });
}

int bsel_generate_dd_bta(bsel_context_t* ctx, const bsel_bta_t* out, uint64_t seed, double dominance,
                         bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    check_shape(out, "out");
    if (dominance < 1.0) throw ArgError("dominance must be >= 1");
    cuda_check(generate_dd_bta_device(to_dev(*out), seed, dominance, ctx->impl->stream()), "generate");
  });
}

int bsel_hermitianize(bsel_context_t* ctx, const bsel_bta_t* m, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx) throw ArgError("ctx is NULL");
    check_shape(m, "m");
    cuda_check(hermitianize_device(to_dev(*m), ctx->impl->stream()), "hermitianize");
  });
}

int bsel_publish(bsel_context_t* ctx, const void* const* src, const int64_t* elems, const int64_t* dst_off,
                 int nblocks, void* const* dst, int ndst, int64_t hdr_off, const double* hdr, bsel_status_t* st) {
  return guarded(st, [&] {
    if (!ctx || (nblocks > 0 && (!src || !elems || !dst_off)) || !dst || !hdr) throw ArgError("NULL argument");
    cuda_check(launch_publish(reinterpret_cast<const double2* const*>(src), elems, dst_off, nblocks,
                              reinterpret_cast<double2* const*>(dst), ndst, hdr_off, hdr, ctx->impl->stream()),
               "publish");
  });
}

uint64_t bsel_kernel_launches(void) { return launch_count(); }

int bsel_profile_begin(void) {
  profile_begin();
  return BSEL_OK;
}

int bsel_profile_end(bsel_profile_t* out) {
  ProfileTotals t = profile_end();
  if (out) {
    out->gemm_launches = t.gemm_launches;
    out->gemm_flops = t.gemm_flops;
    out->gemm_ms = t.gemm_ms;
    out->inverse_calls = t.inverse_calls;
    out->inverse_ms = t.inverse_ms;
    out->gemm_bytes = t.gemm_bytes;
    out->gemm_busy_ms = t.gemm_busy_ms;
    out->inverse_busy_ms = t.inverse_busy_ms;
    out->inverse_flops = t.inverse_flops;
    out->gemm_exec_flops = t.gemm_exec_flops;
  }
  return BSEL_OK;
}

}  // extern "C"
