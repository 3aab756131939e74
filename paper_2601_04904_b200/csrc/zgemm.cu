// Grouped multi-term complex128 DMMA GEMM (see zgemm.cuh for the contract).
//
// Kernel anatomy (one CTA per output tile, tiles of all problems of a batch
// flattened into one grid, heaviest problems first):
//   * multi-stage cp.async pipeline (LDGSTS, zero-fill for ragged edges)
//     staging op(A) as sA[m][k] and op(B) as sB[k][n] in padded,
//     bank-conflict-free layouts; conjugate transposes are handled by the
//     staging addresses (16-byte complex elements are the copy unit);
//   * warp tiles of (BM/WM) x (BN/WN) complex held in registers as DMMA
//     8x8 real accumulators (one complex value per thread per tile);
//   * conjugation / term sign / the -B_im of the real embedding are sign-bit
//     XORs on the ALU pipe, never FP64 multiplies;
//   * epilogue fuses the +-addends (the reference's elementwise +/-).
#include <cstdlib>

#include "zgemm.cuh"

#include <algorithm>
#include <vector>
#include <atomic>
#include <cstdio>
#include <deque>
#include <mutex>
#include <string>

namespace bsel {

namespace {

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_, int BK_ = 8>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = BK_;               // complex k per stage
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int WTM = BM / WM;          // warp tile rows (complex)
  static constexpr int WTN = BN / WN;          // warp tile cols (complex)
  static constexpr int FM = WTM / 8;           // DMMA row fragments per warp
  static constexpr int FN = WTN / 4;           // DMMA col fragments per warp (4 complex cols)
  static constexpr int SA_LD = BK + 2;         // 160 / 288 B rows (== 32 mod 128): conflict-free A fragments
  static constexpr int SB_LD = BN + 2;         // == 32 mod 128 B: conflict-free B fragments
  static constexpr int SA_ELEMS = BM * SA_LD;
  static constexpr int SB_ELEMS = BK * SB_LD;
  static constexpr int A_PER_THREAD = BM * BK / THREADS;
  static constexpr int B_PER_THREAD = BK * BN / THREADS;
  static constexpr int SMEM = STAGES * (SA_ELEMS + SB_ELEMS) * 16;
  static_assert(A_PER_THREAD * THREADS == BM * BK, "A tile split");
  static_assert(B_PER_THREAD * THREADS == BK * BN, "B tile split");
  static_assert(FM * 8 == WTM && FN * 4 == WTN, "warp tile");
};

// 64x64 tiles: 8 warps (32x16 warp tiles), BK 8 x 4 stages, 2 CTAs/SM.
// Measured on the cfg4 level shapes (tools/gemm_micro, 3 concurrent
// streams): 31.5 TF/s vs 31.3 for BK 16 x 3 stages, 32.2 for 4 warps with
// 32x32 warp tiles (which loses 25 % on single launches: 3 CTAs/SM quantize
// worse); whole solve 1972 vs 1989 ms.
using Cfg64 = Cfg<64, 64, 2, 4, 4, 2, 8>;
// 32x32 tiles, 4 warps: latency-critical and small levels (forward sweeps).
// 32x64 / 64x32 tiles with 4 warps measured no better on the whole solve.
using Cfg32 = Cfg<32, 32, 2, 2, 4, 4>;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double xor_sign(double x, unsigned mask) {
  int hi = __double2hiint(x) ^ static_cast<int>(mask);
  return __hiloint2double(hi, __double2loint(x));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Chunk iterator over the K-concatenation of the terms of one problem.
struct ChunkIter {
  int t;   // term index
  int k0;  // complex k offset within the term
};

template <class C>
__device__ __forceinline__ void load_chunk(const GemmProblem& P, const ChunkIter& it, int m0, int n0,
                                           double2* sA, double2* sB, int tid) {
  const GemmTerm& T = P.term[it.t];
  const int K = T.K, M = P.M, N = P.N, k0 = it.k0;
  const double2* A = T.A;
  const double2* B = T.B;
  const int64_t lda = T.lda, ldb = T.ldb;
  if (T.opA == kOpN) {
#pragma unroll
    for (int j = 0; j < C::A_PER_THREAD; ++j) {
      int e = tid + j * C::THREADS;
      int row = e / C::BK, kc = e % C::BK;
      bool ok = (m0 + row < M) && (k0 + kc < K);
      const double2* src = ok ? A + (int64_t)(m0 + row) * lda + (k0 + kc) : A;
      cp_async16(&sA[row * C::SA_LD + kc], src, ok);
    }
  } else {
#pragma unroll
    for (int j = 0; j < C::A_PER_THREAD; ++j) {
      int e = tid + j * C::THREADS;
      int kc = e / C::BM, row = e % C::BM;
      bool ok = (m0 + row < M) && (k0 + kc < K);
      const double2* src = ok ? A + (int64_t)(k0 + kc) * lda + (m0 + row) : A;
      cp_async16(&sA[row * C::SA_LD + kc], src, ok);
    }
  }
  if (T.opB == kOpN) {
#pragma unroll
    for (int j = 0; j < C::B_PER_THREAD; ++j) {
      int e = tid + j * C::THREADS;
      int kc = e / C::BN, col = e % C::BN;
      bool ok = (n0 + col < N) && (k0 + kc < K);
      const double2* src = ok ? B + (int64_t)(k0 + kc) * ldb + (n0 + col) : B;
      cp_async16(&sB[kc * C::SB_LD + col], src, ok);
    }
  } else {
#pragma unroll
    for (int j = 0; j < C::B_PER_THREAD; ++j) {
      int e = tid + j * C::THREADS;
      int col = e / C::BK, kc = e % C::BK;
      bool ok = (n0 + col < N) && (k0 + kc < K);
      const double2* src = ok ? B + (int64_t)(n0 + col) * ldb + (k0 + kc) : B;
      cp_async16(&sB[kc * C::SB_LD + col], src, ok);
    }
  }
}

__device__ __forceinline__ void advance(const GemmProblem& P, ChunkIter& it, int bk) {
  it.k0 += bk;
  if (it.k0 >= P.term[it.t].K) {
    it.k0 = 0;
    ++it.t;
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    zgemm_grouped_kernel(const __grid_constant__ GemmBatch batch) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sA_all = reinterpret_cast<double2*>(smem_raw);
  double2* sB_all = sA_all + C::STAGES * C::SA_ELEMS;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp / C::WN;
  const int wn = warp % C::WN;

  const bool dyn = batch.avoid_sms > 0;
  __shared__ int s_tile;
  if (dyn) {
    // CTAs on avoided SMs leave at once, except the grid's last CTA to
    // leave, which then works off whatever no other CTA took (a small launch
    // on an idle GPU may land entirely on the avoided SMs).
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid < batch.avoid_sms) {
      if (tid == 0) s_tile = (int)atomicAdd(batch.tile_counter + 1, 1u);
      __syncthreads();
      if (s_tile != (int)gridDim.x - 1) return;
      __syncthreads();
    }
    if (tid == 0) s_tile = (int)atomicAdd(batch.tile_counter, 1u);
    __syncthreads();
  }
  for (int bid = dyn ? s_tile : (int)blockIdx.x; bid < batch.total_tiles;) {
  // Locate the problem / tile of this CTA.
  int pi = 0;
  while (pi + 1 < batch.nproblems && bid >= batch.p[pi + 1].tile_begin) ++pi;
  const GemmProblem& P = batch.p[pi];
  const int local = bid - P.tile_begin;
  int m0 = (local / P.tiles_n) * C::BM;
  int n0 = (local % P.tiles_n) * C::BN;
  if (P.lower_only) {  // local = tr (tr + 1) / 2 + tc, tc <= tr
    int tr = (int)((sqrt(8.0 * local + 1.0) - 1.0) * 0.5);
    while ((tr + 1) * (tr + 2) / 2 <= local) ++tr;
    while (tr * (tr + 1) / 2 > local) --tr;
    m0 = tr * C::BM;
    n0 = (local - tr * (tr + 1) / 2) * C::BN;
  }

  int nchunks = 0;
  for (int t = 0; t < P.nterms; ++t) nchunks += (P.term[t].K + C::BK - 1) / C::BK;

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Skip empty-K terms at the front.
  ChunkIter ld_it{0, 0};
  while (ld_it.t < P.nterms && P.term[ld_it.t].K <= 0) ++ld_it.t;
  ChunkIter cp_it = ld_it;

  // Prologue: fill STAGES-1 stages.
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nchunks) {
      load_chunk<C>(P, ld_it, m0, n0, sA_all + s * C::SA_ELEMS, sB_all + s * C::SB_ELEMS, tid);
      advance(P, ld_it, C::BK);
      while (ld_it.t < P.nterms && P.term[ld_it.t].K <= 0) ++ld_it.t;
    }
    cp_async_commit();
  }

  // Per-thread fragment coordinates (constant over the K loop).
  const int a_row = wm * C::WTM + (lane >> 2);       // + im*8
  const int a_kc = (lane & 3) >> 1;                  // + kk*2
  const int a_part = lane & 1;
  const int b_kc = (lane & 3) >> 1;                  // + kk*2
  const int b_col = wn * C::WTN + ((lane >> 2) >> 1);  // + jn*4
  const int b_r = lane & 1, b_s = (lane >> 2) & 1;
  const int b_comp = b_r ^ b_s;

  int cur_term = -1;
  unsigned maskA = 0, maskB = 0;

  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nc = c + C::STAGES - 1;
      if (nc < nchunks) {
        const int st = nc % C::STAGES;
        load_chunk<C>(P, ld_it, m0, n0, sA_all + st * C::SA_ELEMS, sB_all + st * C::SB_ELEMS, tid);
        advance(P, ld_it, C::BK);
        while (ld_it.t < P.nterms && P.term[ld_it.t].K <= 0) ++ld_it.t;
      }
      cp_async_commit();
    }
    if (cp_it.t != cur_term) {
      cur_term = cp_it.t;
      const GemmTerm& T = P.term[cur_term];
      const unsigned SIGN = 0x80000000u;
      maskA = (T.sign < 0 ? SIGN : 0u) ^ ((T.opA == kOpC && a_part) ? SIGN : 0u);
      // Real embedding of op(B): rows (2k+r), cols (2n+s); value Re if r==s
      // else Im; negative for (r,s)=(1,0) [op N] or (0,1) [op C: Im -> -Im].
      if (T.opB == kOpN)
        maskB = (b_r == 1 && b_s == 0) ? SIGN : 0u;
      else
        maskB = (b_r == 0 && b_s == 1) ? SIGN : 0u;
    }
    const int st = c % C::STAGES;
    const double* sAd = reinterpret_cast<const double*>(sA_all + st * C::SA_ELEMS);
    const double* sBd = reinterpret_cast<const double*>(sB_all + st * C::SB_ELEMS);
#pragma unroll
    for (int kk = 0; kk < C::BK / 2; ++kk) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int im = 0; im < C::FM; ++im)
        af[im] = xor_sign(sAd[((a_row + im * 8) * C::SA_LD + kk * 2 + a_kc) * 2 + a_part], maskA);
#pragma unroll
      for (int jn = 0; jn < C::FN; ++jn)
        bf[jn] = xor_sign(sBd[((kk * 2 + b_kc) * C::SB_LD + b_col + jn * 4) * 2 + b_comp], maskB);
#pragma unroll
      for (int im = 0; im < C::FM; ++im)
#pragma unroll
        for (int jn = 0; jn < C::FN; ++jn) dmma(acc[im][jn], af[im], bf[jn]);
    }
    advance(P, cp_it, C::BK);
    while (cp_it.t < P.nterms && P.term[cp_it.t].K <= 0) ++cp_it.t;
  }
  cp_async_wait<0>();

  // Epilogue: D = acc + sum of signed addends.
  const int e_row = wm * C::WTM + (lane >> 2);
  const int e_col = wn * C::WTN + (lane & 3);
#pragma unroll
  for (int im = 0; im < C::FM; ++im) {
    const int m = m0 + e_row + im * 8;
    if (m >= P.M) continue;
#pragma unroll
    for (int jn = 0; jn < C::FN; ++jn) {
      const int n = n0 + e_col + jn * 4;
      if (n >= P.N) continue;
      double re = acc[im][jn][0], imv = acc[im][jn][1];
      for (int a = 0; a < P.naddends; ++a) {
        const GemmAddend& X = P.add[a];
        double2 x = X.X[(int64_t)m * X.ldx + n];
        if (X.sign > 0) {
          re += x.x;
          imv += x.y;
        } else {
          re -= x.x;
          imv -= x.y;
        }
      }
      P.D[(int64_t)m * P.ldd + n] = make_double2(re, imv);
    }
  }
  // next tile (the barrier also orders this tile's stage reads before the
  // next tile's prologue overwrites the stages)
  if (dyn) {
    __syncthreads();
    if (tid == 0) s_tile = (int)atomicAdd(batch.tile_counter, 1u);
    __syncthreads();
    bid = s_tile;
    if (bid >= batch.total_tiles) {  // leaving: count it (see above)
      __syncthreads();
      if (tid == 0) s_tile = (int)atomicAdd(batch.tile_counter + 1, 1u);
      __syncthreads();
      if (s_tile != (int)gridDim.x - 1) break;
      // the last CTA to leave: take what is left (nothing, since this CTA
      // fetched until the tiles ran out)
      break;
    }
  } else {
    bid += gridDim.x;
    __syncthreads();
  }
  }  // tile loop
}

template <class C>
cudaError_t launch_cfg(GemmBatch& batch, cudaStream_t stream) {
  // thread-safe one-time init per device (partitions may launch from several threads)
  const cudaError_t attr = per_device([] {
    return cudaFuncSetAttribute(zgemm_grouped_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  if (attr != cudaSuccess) return attr;
  int tiles = 0;
  for (int i = 0; i < batch.nproblems; ++i) {
    GemmProblem& P = batch.p[i];
    P.tiles_n = (P.N + C::BN - 1) / C::BN;
    P.tile_begin = tiles;
    if (P.lower_only && (P.M != P.N || C::BM != C::BN)) return cudaErrorInvalidValue;
    tiles += P.lower_only ? P.tiles_n * (P.tiles_n + 1) / 2 : ((P.M + C::BM - 1) / C::BM) * P.tiles_n;
  }
  batch.total_tiles = tiles;
  if (tiles == 0) return cudaSuccess;
  int prof = -1;
  double flops = 0.0, bytes = 0.0;
  if (profiling()) {
    // flops: 8 real flops per complex MAC; bytes: every operand read once,
    // D written once (the compulsory DRAM traffic of the launch).
    for (int i = 0; i < batch.nproblems; ++i) {
      const GemmProblem& P = batch.p[i];
      const double tn = P.tiles_n;
      const double frac = P.lower_only ? (tn + 1.0) / (2.0 * tn) : 1.0;  // share of tiles computed
      const double M = P.M * frac, N = P.N;
      bytes += 16.0 * M * N * (1 + P.naddends);
      for (int t = 0; t < P.nterms; ++t) {
        flops += 8.0 * M * N * P.term[t].K;
        bytes += 16.0 * (M + N) * P.term[t].K;
      }
    }
    prof = profile_open(stream);
  }
  const int grid = batch.max_ctas > 0 && batch.max_ctas < tiles ? batch.max_ctas : tiles;
  if (batch.avoid_sms > 0) {
    if (!batch.tile_counter) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(batch.tile_counter, 0, 2 * sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
  }
  zgemm_grouped_kernel<C><<<grid, C::THREADS, C::SMEM, stream>>>(batch);
  count_launch();
  profile_close(prof, stream, 0, flops, bytes);
  return cudaGetLastError();
}

int64_t problem_weight(const GemmProblem& P) {
  int64_t k = 0;
  for (int t = 0; t < P.nterms; ++t) k += P.term[t].K;
  return k;
}

}  // namespace

namespace {
std::atomic<uint64_t> g_launches{0};
struct ProfRec {
  cudaEvent_t t0, t1;
  cudaStream_t stream;
  int kind;
  double flops;
  double bytes;
  double exec_flops;
};
// Partitions of one solve may run in concurrent host threads (dist.py
// _Lanes): records are appended under a mutex (deque: stable references),
// the suspend flag is per thread.
bool g_prof_on = false;
thread_local bool g_prof_suspended = false;
std::deque<ProfRec> g_prof;
size_t g_prof_used = 0;
std::mutex g_prof_mu;
}  // namespace

cudaEvent_t g_prof_base = nullptr;
void profile_begin() {
  cudaDeviceSynchronize();
  if (!g_prof_base) cudaEventCreate(&g_prof_base);
  cudaEventRecord(g_prof_base, 0);
  g_prof_on = true;
  g_prof_used = 0;
}
bool profiling() { return g_prof_on && !g_prof_suspended; }
void profile_suspend(bool on) { g_prof_suspended = on; }
int profile_open(cudaStream_t s) {
  if (!g_prof_on || g_prof_suspended) return -1;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (g_prof_used == g_prof.size()) {
    ProfRec r{};
    cudaEventCreate(&r.t0);
    cudaEventCreate(&r.t1);
    g_prof.push_back(r);
  }
  const int id = (int)g_prof_used++;
  g_prof[id].stream = s;
  cudaEventRecord(g_prof[id].t0, s);
  return id;
}
void profile_close(int id, cudaStream_t s, int kind, double flops, double bytes, double exec_flops) {
  if (id < 0) return;
  std::lock_guard<std::mutex> lock(g_prof_mu);
  g_prof[id].kind = kind;
  g_prof[id].flops = flops;
  g_prof[id].bytes = bytes;
  g_prof[id].exec_flops = exec_flops < 0.0 ? flops : exec_flops;
  cudaEventRecord(g_prof[id].t1, s);
}
ProfileTotals profile_end() {
  ProfileTotals t{};
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lock(g_prof_mu);
  // Spans relative to the base event; busy time = union of the spans of one
  // kind (launches of concurrent streams overlap).
  std::vector<std::pair<float, float>> spans[2];
  // BSEL_PROFILE_DUMP=path: every launch as "kind,stream,start_ms,end_ms,flops,exec_flops" (timeline analysis)
  static const char* dump_path = getenv("BSEL_PROFILE_DUMP");
  FILE* dump = dump_path ? fopen(dump_path, "w") : nullptr;
  for (size_t i = 0; i < g_prof_used; ++i) {
    float ms = 0.f, s0 = 0.f, s1 = 0.f;
    cudaEventElapsedTime(&ms, g_prof[i].t0, g_prof[i].t1);
    cudaEventElapsedTime(&s0, g_prof_base, g_prof[i].t0);
    cudaEventElapsedTime(&s1, g_prof_base, g_prof[i].t1);
    const int kind = g_prof[i].kind == 0 ? 0 : 1;
    spans[kind].emplace_back(s0, s1);
    if (dump)
      fprintf(dump, "%d,%p,%.4f,%.4f,%.6g,%.6g\n", kind, (void*)g_prof[i].stream, s0, s1, g_prof[i].flops,
              g_prof[i].exec_flops);
    if (kind == 0) {
      ++t.gemm_launches;
      t.gemm_flops += g_prof[i].flops;
      t.gemm_exec_flops += g_prof[i].exec_flops;
      t.gemm_bytes += g_prof[i].bytes;
      t.gemm_ms += ms;
    } else {
      ++t.inverse_calls;
      t.inverse_ms += ms;
      t.inverse_flops += g_prof[i].flops;
    }
  }
  double busy[2] = {0.0, 0.0};
  for (int k = 0; k < 2; ++k) {
    auto& v = spans[k];
    std::sort(v.begin(), v.end());
    double cur0 = -1.0, cur1 = -1.0;
    for (auto& sp : v) {
      if (sp.first > cur1) {
        if (cur1 > cur0) busy[k] += cur1 - cur0;
        cur0 = sp.first, cur1 = sp.second;
      } else if (sp.second > cur1) {
        cur1 = sp.second;
      }
    }
    if (cur1 > cur0) busy[k] += cur1 - cur0;
  }
  if (dump) fclose(dump);
  t.gemm_busy_ms = busy[0];
  t.inverse_busy_ms = busy[1];
  g_prof_on = false;
  g_prof_used = 0;
  return t;
}
void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int device_sm_count() {
  return per_device([] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  });
}

cudaError_t launch_gemm_batch(GemmBatch& batch, cudaStream_t stream, int tile_cfg) {
  // Drop empty problems; heaviest (longest K-concatenation) first so the
  // long tiles start in the first wave.
  int w = 0;
  for (int i = 0; i < batch.nproblems; ++i)
    if (batch.p[i].M > 0 && batch.p[i].N > 0) {
      if (w != i) batch.p[w] = batch.p[i];
      ++w;
    }
  batch.nproblems = w;
  if (w == 0) return cudaSuccess;
  std::stable_sort(batch.p, batch.p + w, [](const GemmProblem& x, const GemmProblem& y) {
    return problem_weight(x) > problem_weight(y);
  });
  // Kernel choice.  The 3M TMA kernel (zgemm3m.cu) forms each complex
  // product from three real products: 25 % fewer tensor-pipe flops, but the
  // pre-added operands (Re + Im) round, so even a product with an exactly
  // real / identity factor is no longer exact.  Products of small blocks
  // (any of M, N, K below BSEL_GEMM3M_MIN, default 32 complex) cost little
  // and keep the exact real-embedding form (this kernel): the reference's
  // exact small-system answers (identity systems: X_B == B bit for bit,
  // pkg/tests/test_rgf.py:64-72) stay exact.  BSEL_GEMM=4m / 3m forces one
  // kernel everywhere.
  static const int mode = [] {
    const char* e = getenv("BSEL_GEMM");
    return !e ? 0 : std::string(e) == "4m" ? 4 : std::string(e) == "3m" ? 3 : 0;
  }();
  static const int min3 = [] {
    const char* e = getenv("BSEL_GEMM3M_MIN");
    return e ? atoi(e) : 32;
  }();
  if (tile_cfg == kTile4m64 || tile_cfg == kTile4m32) {
    tile_cfg = tile_cfg == kTile4m64 ? kTile64 : kTile32;
  } else if (tile_cfg >= kTile3m64 && tile_cfg <= kTile3m6432k32) {
    return launch_gemm_batch_3m(batch, stream, tile_cfg);
  } else if (mode != 4) {
    bool big = true;
    for (int i = 0; i < w && big; ++i) {
      const GemmProblem& P = batch.p[i];
      big = P.M >= min3 && P.N >= min3;
      for (int t = 0; t < P.nterms && big; ++t) big = P.term[t].K >= min3;
    }
    if (mode == 3 || big) return launch_gemm_batch_3m(batch, stream, tile_cfg);
  }
  if (tile_cfg == kTileAuto || tile_cfg == kTileAutoWide || tile_cfg == kTileAutoFwd) {
    int64_t tiles64 = 0;
    for (int i = 0; i < w; ++i)
      tiles64 += (int64_t)((batch.p[i].M + 63) / 64) * ((batch.p[i].N + 63) / 64);
    // 64x64 tiles (8 warps) run the DMMA pipe hotter than 32x32 (4 warps)
    // but leave SMs idle when there are too few of them.
    static const int64_t min64 = [] {
      const char* e = getenv("BSEL_GEMM_MIN_TILES64");
      return e ? (int64_t)atoll(e) : (int64_t)2 * device_sm_count();
    }();
    // middle partitions' k = 3 backward levels (4 GPUs: middles' backward
    // 214 ms with 128 vs 252 ms with 2 waves)
    static const int64_t min64_wide = [] {
      const char* e = getenv("BSEL_GEMM_MIN_TILES64_WIDE");
      return e ? (int64_t)atoll(e) : (int64_t)128;
    }();
    tile_cfg = (tiles64 >= (tile_cfg == kTileAutoWide ? min64_wide : min64)) ? kTile64 : kTile32;
  }
  if (tile_cfg == kTile64) return launch_cfg<Cfg64>(batch, stream);
  return launch_cfg<Cfg32>(batch, stream);
}

}  // namespace bsel
