// Grouped complex128 GEMM microbenchmark on the cfg4 (b=512, a=256) level
// shapes: the 3M bulk-async kernel (zgemm3m.cu) variants vs the round-1
// real-embedding cp.async kernel (4m) vs cuBLAS ZGEMM (yardstick only; one
// cublasZgemm per problem), event-timed, plus the 3M-vs-4M result deviation.
// Prints one JSON object.  TFLOP/s are ALGORITHMIC (8 M N K per complex
// product), so the 3M kernel can exceed the 37.15 TF DMMA peak by up to 4/3.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gemm3m_micro.cu \
//        paper_2601_04904_b200/csrc/build/zgemm.o paper_2601_04904_b200/csrc/build/zgemm3m.o -lcublas -o tools/gemm3m_micro
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <cublas_v2.h>

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

int main(int argc, char** argv) {
  const int bs = 512, as = 256;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U1(-1.0, 1.0);
  auto mk = [&](int r, int c) {
    Buf x{nullptr, r, c};
    cudaMalloc(&x.p, (size_t)r * c * 16);
    std::vector<double2> h((size_t)r * c);
    for (auto& v : h) v = make_double2(U1(rng), U1(rng));
    cudaMemcpy(x.p, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    return x;
  };
  Buf g = mk(bs, bs), Uu = mk(bs, bs), Lo = mk(bs, bs), ACe = mk(bs, as), ARe = mk(as, bs), Ydd = mk(bs, bs),
      Ydt = mk(bs, as), Ytd = mk(as, bs), Ytt = mk(as, as), sc = mk(bs, bs), BU = mk(bs, bs), BL = mk(bs, bs),
      BCe = mk(bs, as), BRe = mk(as, bs);
  Buf o[20], oa[8], ob[8];
  for (auto& x : o) x = mk(bs, bs);
  for (auto& x : oa) x = mk(bs, as);
  for (auto& x : ob) x = mk(as, bs);
  Buf big[3];
  for (auto& x : big) x = mk(1024, 1024);
  Buf o2 = mk(1024, 1024);

  struct Lvl {
    std::string name;
    GemmBatch b;
  };
  std::vector<Lvl> lv;
  {
    Lvl l{"bwd_L1_12p", {}};
    GemmBatch& b = l.b;
    P(b, o[0], {T(Uu, kOpN, Ydd, kOpN), T(ACe, kOpN, Ytd, kOpN)});
    P(b, oa[0], {T(Uu, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, o[1], {T(Ydd, kOpN, Lo, kOpN), T(Ydt, kOpN, ARe, kOpN)});
    P(b, ob[0], {T(Ytd, kOpN, Lo, kOpN), T(Ytt, kOpN, ARe, kOpN)});
    P(b, o[2], {T(Uu, kOpN, Ydd, kOpN), T(ACe, kOpN, Ytd, kOpN)});
    P(b, oa[1], {T(Uu, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, o[3], {T(Ydd, kOpN, Uu, kOpC), T(Ydt, kOpN, ACe, kOpC)});
    P(b, ob[1], {T(Ytd, kOpN, Uu, kOpC), T(Ytt, kOpN, ACe, kOpC)});
    P(b, o[4], {T(g, kOpN, BU, kOpN), T(sc, kOpN, Lo, kOpC, -1)});
    P(b, oa[2], {T(g, kOpN, BCe, kOpN), T(sc, kOpN, ARe, kOpC, -1)});
    P(b, o[5], {T(BL, kOpN, g, kOpC), T(Lo, kOpN, sc, kOpN, -1)});
    P(b, ob[2], {T(BRe, kOpN, g, kOpC), T(ARe, kOpN, sc, kOpN, -1)});
    lv.push_back(l);
  }
  {
    Lvl l{"bwd_L3_4p", {}};
    GemmBatch& b = l.b;
    P(b, o[6], {T(o[0], kOpN, Lo, kOpN, -1), T(oa[0], kOpN, ARe, kOpN, -1)});
    P(b, o[7], {T(BU, kOpN, o[0], kOpC), T(BCe, kOpN, oa[0], kOpC)});
    P(b, o[8], {T(o[0], kOpN, BL, kOpN), T(oa[0], kOpN, BRe, kOpN)});
    P(b, o[9], {T(g, kOpN, o[1], kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"bwd_L4_early_10p", {}};
    GemmBatch& b = l.b;
    P(b, o[10], {T(o[6], kOpN, g, kOpN)}, &g);
    P(b, o[11], {T(o[6], kOpN, sc, kOpN), T(sc, kOpN, o[6], kOpC), T(g, kOpN, o[7], kOpN), T(o[8], kOpN, g, kOpC),
                 T(o[9], kOpN, g, kOpC)}, &sc);
    P(b, oa[3], {T(Uu, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, ob[3], {T(Ytd, kOpN, Lo, kOpN), T(Ytt, kOpN, ARe, kOpN)});
    P(b, oa[4], {T(Uu, kOpN, Ydt, kOpN), T(ACe, kOpN, Ytt, kOpN)});
    P(b, ob[4], {T(Ytd, kOpN, Uu, kOpC), T(Ytt, kOpN, ACe, kOpC)});
    P(b, o[12], {T(g, kOpN, BU, kOpN), T(sc, kOpN, Lo, kOpC, -1)});
    P(b, oa[5], {T(g, kOpN, BCe, kOpN), T(sc, kOpN, ARe, kOpC, -1)});
    P(b, o[13], {T(BL, kOpN, g, kOpC), T(Lo, kOpN, sc, kOpN, -1)});
    P(b, ob[5], {T(BRe, kOpN, g, kOpC), T(ARe, kOpN, sc, kOpN, -1)});
    lv.push_back(l);
  }
  const char* ops[4] = {"NN", "NC", "CN", "CC"};
  for (int q = 0; q < 4; ++q) {
    Lvl l{std::string("sq512_") + ops[q], {}};
    P(l.b, o[14], {T(Lo, q & 2 ? kOpC : kOpN, g, q & 1 ? kOpC : kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"256x512x512_NN", {}};
    P(l.b, ob[6], {T(ARe, kOpN, g, kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"512x256x512_NN", {}};
    P(l.b, o[15], {T(ACe, kOpN, ARe, kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"512x512x256_NN", {}};
    P(l.b, oa[6], {T(Lo, kOpN, ACe, kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"sq1024_NN", {}};
    P(l.b, o2, {T(big[0], kOpN, big[1], kOpN)});
    lv.push_back(l);
  }
  {
    Lvl l{"lower_only_512", {}};
    P(l.b, o[16], {T(g, kOpN, sc, kOpC)});
    l.b.p[0].lower_only = 1;
    lv.push_back(l);
  }

  cudaStream_t s;
  cudaStreamCreate(&s);
  if (argc > 3) {  // profiling mode: <level index> <tile cfg code> <reps>
    const int li = atoi(argv[1]), cfg = atoi(argv[2]), reps = atoi(argv[3]);
    for (int r = 0; r < reps; ++r) {
      GemmBatch b = lv[li].b;
      launch_gemm_batch(b, s, cfg);
    }
    cudaStreamSynchronize(s);
    printf("{\"level\": \"%s\", \"err\": \"%s\"}\n", lv[li].name.c_str(), cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  cublasHandle_t h;
  cublasCreate(&h);
  cublasSetStream(h, s);
  for (int r = 0; r < 200; ++r) {  // warm clocks
    GemmBatch b = lv[0].b;
    launch_gemm_batch(b, s, kTile4m64);
  }
  cudaStreamSynchronize(s);
  std::vector<double2> r4, r3;
  auto fetch = [&](const GemmBatch& b, std::vector<double2>& out) {
    out.clear();
    for (int i = 0; i < b.nproblems; ++i) {
      std::vector<double2> t((size_t)b.p[i].M * b.p[i].N);
      cudaMemcpy2D(t.data(), b.p[i].N * 16, b.p[i].D, b.p[i].ldd * 16, b.p[i].N * 16, b.p[i].M,
                   cudaMemcpyDeviceToHost);
      out.insert(out.end(), t.begin(), t.end());
    }
  };
  auto timeit = [&](const GemmBatch& b0, int cfg, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    {
      GemmBatch b = b0;
      launch_gemm_batch(b, s, cfg);
    }
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) {
      GemmBatch b = b0;
      launch_gemm_batch(b, s, cfg);
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return flops(b0) * reps / ms / 1e9;
  };
  auto cublas_time = [&](const GemmBatch& b0, int reps) {
    // D = op(A) op(B) per problem per term (beta accumulates); row-major via C^T = B^T A^T
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const cuDoubleComplex one = make_cuDoubleComplex(1, 0);
    auto run = [&]() {
      for (int i = 0; i < b0.nproblems; ++i) {
        const GemmProblem& p = b0.p[i];
        for (int t = 0; t < p.nterms; ++t) {
          const GemmTerm& tt = p.term[t];
          const cuDoubleComplex beta = make_cuDoubleComplex(t ? 1 : 0, 0);
          cublasZgemm(h, tt.opB == kOpC ? CUBLAS_OP_C : CUBLAS_OP_N, tt.opA == kOpC ? CUBLAS_OP_C : CUBLAS_OP_N,
                      p.N, p.M, tt.K, &one, (const cuDoubleComplex*)tt.B, (int)tt.ldb,
                      (const cuDoubleComplex*)tt.A, (int)tt.lda, &beta, (cuDoubleComplex*)p.D, (int)p.ldd);
        }
      }
    };
    run();
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return flops(b0) * reps / ms / 1e9;
  };
  printf("{\"unit\": \"algorithmic TFLOP/s (8MNK)\"");
  const int cfgs[] = {kTile4m64, kTile4m32, kTile3m64, kTile3m6432, kTile3m32, kTileAuto, kTile3m64k32,
                      kTile3m6432k32};
  const char* cn[] = {"4m64", "4m32", "3m64", "3m6432", "3m32", "auto3m", "3m64k32", "3m6432k32"};
  const int ncfg = 8;
  for (auto& l : lv) {
    const int reps = 20;
    printf(",\n \"%s\": {", l.name.c_str());
    for (int c = 0; c < ncfg; ++c) {
      printf("%s\"%s\": %.2f", c ? ", " : "", cn[c], timeit(l.b, cfgs[c], reps));
    }
    if (!l.b.p[0].lower_only) printf(", \"cublas\": %.2f", cublas_time(l.b, reps));
    // deviation 3M (auto) vs 4M (64): max |d| / max |ref|
    {
      GemmBatch b = l.b;
      launch_gemm_batch(b, s, kTile4m64);
      cudaStreamSynchronize(s);
      fetch(l.b, r4);
      for (int c : {kTile3m64, kTile3m6432, kTile3m32}) {
        GemmBatch b2 = l.b;
        launch_gemm_batch(b2, s, c);
        cudaStreamSynchronize(s);
        fetch(l.b, r3);
        double md = 0, mr = 0;
        for (size_t i = 0; i < r4.size(); ++i) {
          if (l.b.p[0].lower_only) {  // only the lower triangle is defined
            const int row = (int)(i / l.b.p[0].N), col = (int)(i % l.b.p[0].N);
            if (col > row) continue;
          }
          md = std::max(md, std::hypot(r4[i].x - r3[i].x, r4[i].y - r3[i].y));
          mr = std::max(mr, std::hypot(r4[i].x, r4[i].y));
        }
        printf(", \"dev_%d\": %.3e", c, md / mr);
      }
    }
    printf("}");
  }
  // concurrent: 3 streams (steady state of the sweeps)
  cudaStream_t cs[3];
  for (auto& x : cs) cudaStreamCreate(&x);
  for (int li = 0; li < 3; ++li) {
    for (int c = 0; c < ncfg; ++c) {
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
          launch_gemm_batch(b, x, cfgs[c]);
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
      printf(",\n \"%s_x3_%s\": %.2f", lv[li].name.c_str(), cn[c], flops(lv[li].b) * reps * 3 / ms / 1e9);
    }
  }
  printf(",\n \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
