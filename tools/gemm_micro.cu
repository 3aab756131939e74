// Grouped DMMA ZGEMM microbenchmark on the real level shapes of the cfg4
// (b=512, a=256) sweeps: event-timed TFLOP/s per level type.
#include <cstdio>
#include <vector>

#include "../paper_2601_04904_b200/csrc/zgemm.cuh"

using namespace bsel;

struct Buf {
  double2* p;
  int r, c;
};

static GemmTerm T(Buf A, uint8_t oa, Buf B, uint8_t ob, int sign = 1) {
  GemmTerm t{};
  t.A = A.p;
  t.B = B.p;
  t.lda = A.c;
  t.ldb = B.c;
  t.K = oa == kOpN ? A.c : A.r;
  t.opA = oa;
  t.opB = ob;
  t.sign = (int8_t)sign;
  return t;
}

static void P(GemmBatch& b, Buf D, std::initializer_list<GemmTerm> terms, Buf* add = nullptr) {
  GemmProblem& p = b.p[b.nproblems++];
  p = GemmProblem{};
  p.D = D.p;
  p.ldd = D.c;
  p.M = D.r;
  p.N = D.c;
  for (auto& t : terms) p.term[p.nterms++] = t;
  if (add) {
    p.add[0].X = add->p;
    p.add[0].ldx = add->c;
    p.add[0].sign = 1;
    p.naddends = 1;
  }
}

static double flops(const GemmBatch& b) {
  double f = 0;
  for (int i = 0; i < b.nproblems; ++i)
    for (int t = 0; t < b.p[i].nterms; ++t) f += 8.0 * b.p[i].M * (double)b.p[i].N * b.p[i].term[t].K;
  return f;
}

int main() {
  const int bs = 512, as = 256;
  std::vector<Buf> pool;
  auto mk = [&](int r, int c) {
    Buf x{nullptr, r, c};
    cudaMalloc(&x.p, (size_t)r * c * 16);
    cudaMemset(x.p, 0, (size_t)r * c * 16);
    pool.push_back(x);
    return x;
  };
  Buf g = mk(bs, bs), U = mk(bs, bs), Lo = mk(bs, bs), ACe = mk(bs, as), ARe = mk(as, bs), Ydd = mk(bs, bs),
      Ydt = mk(bs, as), Ytd = mk(as, bs), Ytt = mk(as, as), sc = mk(bs, bs), BU = mk(bs, bs), BL = mk(bs, bs),
      BCe = mk(bs, as), BRe = mk(as, bs);
  Buf o[20];
  for (int i = 0; i < 20; ++i) o[i] = mk(bs, bs);
  Buf oa[8];
  for (int i = 0; i < 8; ++i) oa[i] = mk(bs, as);
  Buf ob[8];
  for (int i = 0; i < 8; ++i) ob[i] = mk(as, bs);

  struct Lvl {
    const char* name;
    GemmBatch b;
  };
  std::vector<Lvl> lv;
  {  // backward L1 (12 problems)
    Lvl l{"bwd_L1", {}};
    GemmBatch& b = l.b;
    P(b, o[0], {T(U, kOpN, Ydd, kOpN), T(ACe, kOpN, Ytd, kOpN)});
    P(b, oa[0], {T(U, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, o[1], {T(Ydd, kOpN, Lo, kOpN), T(Ydt, kOpN, ARe, kOpN)});
    P(b, ob[0], {T(Ytd, kOpN, Lo, kOpN), T(Ytt, kOpN, ARe, kOpN)});
    P(b, o[2], {T(U, kOpN, Ydd, kOpN), T(ACe, kOpN, Ytd, kOpN)});
    P(b, oa[1], {T(U, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, o[3], {T(Ydd, kOpN, U, kOpC), T(Ydt, kOpN, ACe, kOpC)});
    P(b, ob[1], {T(Ytd, kOpN, U, kOpC), T(Ytt, kOpN, ACe, kOpC)});
    P(b, o[4], {T(g, kOpN, BU, kOpN), T(sc, kOpN, Lo, kOpC, -1)});
    P(b, oa[2], {T(g, kOpN, BCe, kOpN), T(sc, kOpN, ARe, kOpC, -1)});
    P(b, o[5], {T(BL, kOpN, g, kOpC), T(Lo, kOpN, sc, kOpN, -1)});
    P(b, ob[2], {T(BRe, kOpN, g, kOpC), T(ARe, kOpN, sc, kOpN, -1)});
    lv.push_back(l);
  }
  {  // backward L3 (4 problems)
    Lvl l{"bwd_L3", {}};
    GemmBatch& b = l.b;
    P(b, o[6], {T(o[0], kOpN, Lo, kOpN, -1), T(oa[0], kOpN, ARe, kOpN, -1)});
    P(b, o[7], {T(BU, kOpN, o[0], kOpC), T(BCe, kOpN, oa[0], kOpC)});
    P(b, o[8], {T(o[0], kOpN, BL, kOpN), T(oa[0], kOpN, BRe, kOpN)});
    P(b, o[9], {T(g, kOpN, o[1], kOpN)});
    lv.push_back(l);
  }
  {  // backward L4 + next early L1 (pipelined level)
    Lvl l{"bwd_L4+early", {}};
    GemmBatch& b = l.b;
    P(b, o[10], {T(o[6], kOpN, g, kOpN)}, &g);
    P(b, o[11], {T(o[6], kOpN, sc, kOpN), T(sc, kOpN, o[6], kOpC), T(g, kOpN, o[7], kOpN), T(o[8], kOpN, g, kOpC),
                 T(o[9], kOpN, g, kOpC)}, &sc);
    P(b, oa[3], {T(U, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, ob[3], {T(Ytd, kOpN, Lo, kOpN), T(Ytt, kOpN, ARe, kOpN)});
    P(b, oa[4], {T(U, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, ob[4], {T(Ytd, kOpN, U, kOpC), T(Ytt, kOpN, ACe, kOpC)});
    P(b, o[12], {T(g, kOpN, BU, kOpN), T(sc, kOpN, Lo, kOpC, -1)});
    P(b, oa[5], {T(g, kOpN, BCe, kOpN), T(sc, kOpN, ARe, kOpC, -1)});
    P(b, o[13], {T(BL, kOpN, g, kOpC), T(Lo, kOpN, sc, kOpN, -1)});
    P(b, ob[5], {T(BRe, kOpN, g, kOpC), T(ARe, kOpN, sc, kOpN, -1)});
    lv.push_back(l);
  }
  {  // forward chain GEMM (single 512^3) and square 2048
    Lvl l{"chain_512^3", {}};
    P(l.b, o[14], {T(Lo, kOpN, g, kOpN)});
    lv.push_back(l);
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  // warm clocks
  for (int r = 0; r < 200; ++r) {
    GemmBatch b = lv[0].b;
    launch_gemm_batch(b, s);
  }
  cudaStreamSynchronize(s);
  printf("{");
  for (size_t li = 0; li < lv.size(); ++li) {
    for (int cfg : {kTileAuto, kTile64, kTile32}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = 20;
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) {
        GemmBatch b = lv[li].b;
        launch_gemm_batch(b, s, cfg);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* cn = cfg == kTileAuto ? "auto" : cfg == kTile64 ? "t64" : "t32";
      printf("%s\"%s_%s_tflops\": %.2f", (li || cfg != kTileAuto) ? ", " : "", lv[li].name, cn,
             flops(lv[li].b) * reps / ms / 1e9);
    }
  }
  // Concurrent: the same level on 3 streams at once (tails overlap, as in
  // the real sweeps where chain / aux / other partition overlap).
  cudaStream_t cs[3];
  for (auto& x : cs) cudaStreamCreate(&x);
  for (size_t li = 0; li < lv.size(); ++li) {
    for (int cfg : {kTile64, kTile32}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = 20;
      cudaDeviceSynchronize();
      cudaEventRecord(e0, cs[0]);
      cudaStreamWaitEvent(cs[1], e0, 0);
      cudaStreamWaitEvent(cs[2], e0, 0);
      for (int r = 0; r < reps; ++r)
        for (auto& x : cs) {
          GemmBatch b = lv[li].b;
          launch_gemm_batch(b, x, cfg);
        }
      for (int k = 1; k < 3; ++k) {
        cudaEvent_t ek;
        cudaEventCreate(&ek);
        cudaEventRecord(ek, cs[k]);
        cudaStreamWaitEvent(cs[0], ek, 0);
      }
      cudaEventRecord(e1, cs[0]);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf(", \"%s_%s_x3_tflops\": %.2f", lv[li].name, cfg == kTile64 ? "t64" : "t32",
             flops(lv[li].b) * reps * 3 / ms / 1e9);
    }
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
