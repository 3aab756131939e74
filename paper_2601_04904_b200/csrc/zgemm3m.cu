// Grouped multi-term complex128 GEMM, 3-multiplication form, bulk-async
// (TMA engine) staged, warp specialized (see zgemm.cuh for the contract).
//
// Arithmetic.  Every complex product is formed from THREE real products
// (the Gauss / "3M" scheme):
//     P1 = Re A . Re B,   P2 = Im A . Im B,   P3 = (Re A + Im A) . (Re B + Im B)
//     Re C = P1 - P2,     Im C = P3 - P1 - P2
// so one 8 x 8 complex output tile over 4 complex k is three DMMA.8x8x4
// (mma.sync.m8n8k4.f64) instead of the four the real 2x2 embedding needs:
// 6 real flops per complex MAC instead of 8, 25 % less tensor-pipe time for
// the same block product.  Its error bound is a small multiple of the
// classical one (|Re C| and |Im C| are each bounded by eps-multiples of
// sum |a||b|-like terms), far inside the 1e-10 parity tolerance.
//
// Staging.  One producer thread moves operand tiles global -> shared with
// TMA tensor copies (cp.async.bulk.tensor.2d, SASS UTMALDG) into 128-byte
// swizzled boxes, completing on a per-stage mbarrier with expect_tx byte
// counts; the consumer warps wait on that barrier, compute, and release the
// stage through a second mbarrier.  A box is 8 complex (128 B) wide: the
// k-contiguous operands (op(A) = A, op(B) = B^H) arrive as BK/8 boxes of
// BM (BN) rows, the k-strided ones (op(A) = A^H, op(B) = B) as BM/8 (BN/8)
// boxes of BK rows.  With the hardware's 128 B swizzle and the DMMA
// fragment rows/columns permuted (pi below), every 16-byte fragment load of
// a quarter warp hits 8 distinct bank groups in both layouts.  Conjugate
// transposes are never materialised; conjugation and term signs are
// sign-bit XORs on the fragment registers.  The descriptors (one per
// operand block, 2-D: the block's own rows x columns, so TMA zero-fills
// every ragged edge) are encoded once on the host and cached in a
// device-resident table; the kernel parameters carry slot indices.
//
// Tiles of all problems of a launch are processed by a persistent grid;
// the producer runs ahead into the next tile while the consumers finish
// the current one (epilogue overlapped with the next tile's loads).
// Boxes entirely outside a block are not issued; k beyond K within the
// last chunk of a term is masked to zero on the fragment registers.
#include <cstdlib>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <shared_mutex>
#include <unordered_map>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "zgemm.cuh"

namespace bsel {

namespace {

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg3 {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int CONS_WARPS = WM * WN;
  static constexpr int THREADS = 32 * (CONS_WARPS + 1);  // + 1 producer warp
  static constexpr int WTM = BM / WM, WTN = BN / WN;     // warp tile (complex)
  static constexpr int FM = WTM / 8, FN = WTN / 8;       // 8x8 complex DMMA tiles per warp
  static constexpr int A_BYTES = BM * BK * 16;         // BK/8 boxes of BM x 128 B, or BM/8 of BK x 128 B
  static constexpr int B_BYTES = BN * BK * 16;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // multiple of 1024 (swizzle atom)
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + STAGES * 16 + STAGES * 4 + 16;  // + alignment slack
  static_assert(FM * 8 == WTM && FN * 8 == WTN, "warp tile must be a multiple of 8x8");
  static_assert(BK % 4 == 0, "BK multiple of the DMMA k (4)");
  static_assert(BK % 8 == 0 && BM % 8 == 0 && BN % 8 == 0, "8-complex (128 B) boxes");
  static_assert(STAGE_BYTES % 1024 == 0, "stages stay 1024-B aligned");
};

// 64x64 tiles, 8 consumer warps of 32x16, BK 16 x 4 stages, 1 CTA / SM.
using C3_64 = Cfg3<64, 64, 16, 2, 4, 4, 1>;
// 64x32 tiles, 4 consumer warps of 32x16, BK 16 x 4 stages, 2 CTAs / SM.
using C3_6432 = Cfg3<64, 32, 16, 2, 2, 4, 2>;
// 32x32 tiles, 4 consumer warps of 16x16, BK 16 x 4 stages (small / chain levels).
using C3_32 = Cfg3<32, 32, 16, 2, 2, 4, 3>;
// BK 32 variants (half the barrier round trips per flop); 64x32 / BK 32 is the default for levels
// that fill a wave (launch_gemm_batch_3m)
using C3_64_K32 = Cfg3<64, 64, 32, 2, 4, 3, 1>;
using C3_6432_K32 = Cfg3<64, 32, 32, 2, 2, 2, 2>;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 2-D TMA tensor copy global -> shared (box at element coordinates c0, c1),
// completing on `bar`
__device__ __forceinline__ void tma_load_2d(unsigned dst, const void* desc, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dst),
      "l"(desc), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_desc_acquire(const void* desc) {
  // the table is written by host copies (generic proxy) before the launch
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(desc) : "memory");
}

__device__ __forceinline__ double xor_hi(double x, unsigned mask) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(mask), __double2loint(x));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// DMMA row (or column) r of an 8-group -> tile row: quarter warps then read
// rows r and r^4, which sit 64 B apart in bank space.
__device__ __forceinline__ int pi8(int r) { return (r >> 1) | ((r & 1) << 2); }

struct TileLoc {
  int pi, m0, n0;
};

template <class C>
__device__ __forceinline__ TileLoc locate(const GemmBatch& batch, int bid) {
  int pi = 0;
  while (pi + 1 < batch.nproblems && bid >= batch.p[pi + 1].tile_begin) ++pi;
  const GemmProblem& P = batch.p[pi];
  int local = bid - P.tile_begin;
  int m0, n0;
  if (P.lower_only) {
    // tiles meeting the lower triangle: row band tr has min(tiles_n, ((tr+1)BM-1)/BN + 1) tiles
    int tr = 0;
    for (;;) {
      int cnt = ((tr + 1) * C::BM - 1) / C::BN + 1;
      if (cnt > P.tiles_n) cnt = P.tiles_n;
      if (local < cnt) break;
      local -= cnt;
      ++tr;
    }
    m0 = tr * C::BM;
    n0 = local * C::BN;
  } else {
    m0 = (local / P.tiles_n) * C::BM;
    n0 = (local % P.tiles_n) * C::BN;
  }
  return TileLoc{pi, m0, n0};
}

// One staged chunk: BK/4 DMMA k-steps of the warp's FM x FN 8x8 complex
// tiles, three accumulators each (3M).  Fragment address of 8-group i and
// k-step kk:  base + i * step8 + (kk >> 1) * k2 + (kk & 1) * k1 + (x0 ^ ((kk & 1) << 6))
// (x0: the thread's swizzled 16-B chunk).  TAIL: k beyond kv masked to zero.
struct Frag {
  unsigned base, step8, k2, k1;
};

template <class C, bool TAIL>
__device__ __forceinline__ void chunk_mma(double (&acc)[C::FM][C::FN][3][2], Frag fa, Frag fb, unsigned x0,
                                          unsigned mAr, unsigned mAi, unsigned mBi, int tq, int kv) {
#pragma unroll
  for (int kk = 0; kk < C::BK / 4; ++kk) {
    const bool kok = !TAIL || kk * 4 + tq < kv;
    const unsigned xo = x0 ^ ((kk & 1) << 6);
    double br[C::FN], bi[C::FN], bs[C::FN];
#pragma unroll
    for (int jn = 0; jn < C::FN; ++jn) {
      double2 v = lds128(fb.base + jn * fb.step8 + (kk >> 1) * fb.k2 + (kk & 1) * fb.k1 + xo);
      if (TAIL && !kok) v = make_double2(0.0, 0.0);
      br[jn] = v.x;
      bi[jn] = xor_hi(v.y, mBi);
      bs[jn] = br[jn] + bi[jn];
    }
#pragma unroll
    for (int im = 0; im < C::FM; ++im) {
      double2 v = lds128(fa.base + im * fa.step8 + (kk >> 1) * fa.k2 + (kk & 1) * fa.k1 + xo);
      if (TAIL && !kok) v = make_double2(0.0, 0.0);
      const double ar = xor_hi(v.x, mAr), ai = xor_hi(v.y, mAi);
      const double as = ar + ai;
#pragma unroll
      for (int jn = 0; jn < C::FN; ++jn) {
        dmma(acc[im][jn][0], ar, br[jn]);
        dmma(acc[im][jn][1], ai, bi[jn]);
        dmma(acc[im][jn][2], as, bs[jn]);
      }
    }
  }
}

// Fragment addressing of one operand tile in a stage.  in_k: k-contiguous
// boxes (BK/8 boxes of R rows x 128 B); else k-strided (R/8 boxes of BK rows).
// r0: the thread's first tile row (or column) of its warp, incl. pi.
template <class C>
__device__ __forceinline__ Frag frag_of(unsigned s, bool in_k, int R, int w0, int p, int tq) {
  if (in_k) return Frag{s + (unsigned)(w0 + p) * 128u, 1024u, (unsigned)R * 128u, 0u};
  return Frag{s + (unsigned)(w0 / 8) * (C::BK * 128u) + (unsigned)tq * 128u, C::BK * 128u, 1024u, 512u};
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) zgemm3m_kernel(const __grid_constant__ GemmBatch batch) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128-B swizzled TMA boxes need 1024-B aligned destinations
  const unsigned sraw = smem_u32(smem_raw);
  const unsigned sbase = (sraw + 1023u) & ~1023u;
  unsigned char* smem = smem_raw + (sbase - sraw);
  const unsigned full0 = sbase + C::BAR_OFF;           // full[s]  = full0 + 16 s
  const unsigned empty0 = full0 + 8;                    // empty[s] = empty0 + 16 s
  int* stage_tile = reinterpret_cast<int*>(smem + C::BAR_OFF + C::STAGES * 16);
  __shared__ int s_tile;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // A programmatic dependent of this launch (the chain's block inverse,
  // inverse.cu launch_dataflow) may be placed from now on; it waits for this
  // grid's completion (griddepcontrol.wait) before reading its output.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if BSEL_INV_STATS
  // chain launch-gap statistics (inverse.cuh chain_marks): [0] last chain
  // kernel end, [2]/[3] gap sum / count before chain GEMMs
  if (batch.chain_mark && blockIdx.x == 0 && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long prev = atomicAdd(batch.chain_mark, 0ull);
    if (prev && t > prev && t - prev < 10000000ull) {
      atomicAdd(batch.chain_mark + 2, t - prev);
      atomicAdd(batch.chain_mark + 3, 1ull);
    }
  }
#endif

  // ---- SM avoidance (zgemm.cuh avoid_sms): leave at once, except the grid's
  // last CTA to leave, which then works off whatever is left
  const bool dyn = batch.avoid_sms > 0;
  if (dyn) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if ((int)smid < batch.avoid_sms) {
      if (tid == 0) s_tile = (int)atomicAdd(batch.tile_counter + 1, 1u);
      __syncthreads();
      if (s_tile != (int)gridDim.x - 1) return;
      __syncthreads();
    }
  }
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full0 + 16 * s, 1);
      mbar_init(empty0 + 16 * s, C::CONS_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == C::CONS_WARPS) {
    // ======================= producer (one thread) =======================
    if (lane != 0) return;
    const char* table = static_cast<const char*>(batch.tma_table);
    int stage = 0;
    unsigned phase = 0;
    int tile = dyn ? (int)atomicAdd(batch.tile_counter, 1u) : (int)blockIdx.x;
    while (tile < batch.total_tiles) {
      const TileLoc L = locate<C>(batch, tile);
      const GemmProblem& P = batch.p[L.pi];
      bool any = false;
      for (int t = 0; t < P.nterms; ++t) any |= P.term[t].K > 0;
      if (!any) {  // addends only: one stage without data carries the tile
        mbar_wait(empty0 + 16 * stage, phase ^ 1u);
        stage_tile[stage] = tile;
        mbar_arrive(full0 + 16 * stage);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      for (int t = 0; t < P.nterms; ++t) {
        const GemmTerm& T = P.term[t];
        if (T.K <= 0) continue;
        const void* dA = table + (size_t)T.tmaA * 128;
        const void* dB = table + (size_t)T.tmaB * 128;
        tma_desc_acquire(dA);
        tma_desc_acquire(dB);
        // boxes inside the blocks (rows / columns beyond M / N only feed discarded outputs)
        const int mbox = min(C::BM / 8, (P.M - L.m0 + 7) / 8), nbox = min(C::BN / 8, (P.N - L.n0 + 7) / 8);
        for (int k0 = 0; k0 < T.K; k0 += C::BK) {
          const int kbox = min(C::BK / 8, (T.K - k0 + 7) / 8);
          mbar_wait(empty0 + 16 * stage, phase ^ 1u);
          const unsigned sA = sbase + stage * C::STAGE_BYTES;
          const unsigned sB = sA + C::A_BYTES;
          const unsigned full = full0 + 16 * stage;
          const unsigned txA = T.opA == kOpN ? kbox * C::BM * 128u : mbox * C::BK * 128u;
          const unsigned txB = T.opB == kOpC ? kbox * C::BN * 128u : nbox * C::BK * 128u;
          stage_tile[stage] = tile;
          mbar_arrive_expect_tx(full, txA + txB);
          if (T.opA == kOpN)  // A (M x K): boxes of 8 k x BM rows
            for (int h = 0; h < kbox; ++h) tma_load_2d(sA + h * (C::BM * 128), dA, 2 * (k0 + 8 * h), L.m0, full);
          else  // A^H stored K x M: boxes of 8 m x BK rows
            for (int j = 0; j < mbox; ++j) tma_load_2d(sA + j * (C::BK * 128), dA, 2 * (L.m0 + 8 * j), k0, full);
          if (T.opB == kOpC)  // B^H stored N x K: boxes of 8 k x BN rows
            for (int h = 0; h < kbox; ++h) tma_load_2d(sB + h * (C::BN * 128), dB, 2 * (k0 + 8 * h), L.n0, full);
          else  // B stored K x N: boxes of 8 n x BK rows
            for (int j = 0; j < nbox; ++j) tma_load_2d(sB + j * (C::BK * 128), dB, 2 * (L.n0 + 8 * j), k0, full);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      tile = dyn ? (int)atomicAdd(batch.tile_counter, 1u) : tile + (int)gridDim.x;
    }
    // end marker
    mbar_wait(empty0 + 16 * stage, phase ^ 1u);
    stage_tile[stage] = -1;
    mbar_arrive(full0 + 16 * stage);
    return;
  }

  // ======================= consumer warps =======================
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int g = lane >> 2, tq = lane & 3;
  const int prow = pi8(g);  // this thread's A row / B column within an 8-group
  const unsigned x0 = (unsigned)((tq ^ prow) << 4);
  int stage = 0;
  unsigned phase = 0;
  const unsigned SIGN = 0x80000000u;
  for (;;) {
    mbar_wait(full0 + 16 * stage, phase);
    const int tile = stage_tile[stage];
    if (tile < 0) break;
    const TileLoc L = locate<C>(batch, tile);
    const GemmProblem& P = batch.p[L.pi];

    double acc[C::FM][C::FN][3][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j)
#pragma unroll
        for (int q = 0; q < 3; ++q) acc[i][j][q][0] = acc[i][j][q][1] = 0.0;

    bool first = true;
    for (int t = 0; t < P.nterms; ++t) {
      const GemmTerm& T = P.term[t];
      const unsigned sgn = T.sign < 0 ? SIGN : 0u;
      const unsigned mAr = sgn, mAi = sgn ^ (T.opA == kOpC ? SIGN : 0u);
      const unsigned mBi = T.opB == kOpC ? SIGN : 0u;
      const bool a_in = T.opA == kOpN, b_in = T.opB == kOpC;
      for (int k0 = 0; k0 < T.K; k0 += C::BK) {
        if (!first) mbar_wait(full0 + 16 * stage, phase);
        first = false;
        const int kv = min(C::BK, T.K - k0);
        const unsigned sA = sbase + stage * C::STAGE_BYTES;
        const unsigned sB = sA + C::A_BYTES;
        const Frag fa = frag_of<C>(sA, a_in, C::BM, wm * C::WTM, prow, tq);
        const Frag fb = frag_of<C>(sB, b_in, C::BN, wn * C::WTN, prow, tq);
        if (kv == C::BK)
          chunk_mma<C, false>(acc, fa, fb, x0, mAr, mAi, mBi, tq, kv);
        else
          chunk_mma<C, true>(acc, fa, fb, x0, mAr, mAi, mBi, tq, kv);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 16 * stage);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    if (first) {  // addends only: release the data-less stage that carried the tile
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 16 * stage);
      if (++stage == C::STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }

    // ---- epilogue: D = (P1 - P2, P3 - P1 - P2) + sum of signed addends
#pragma unroll
    for (int im = 0; im < C::FM; ++im) {
      const int m = L.m0 + wm * C::WTM + im * 8 + prow;
      if (m >= P.M) continue;
#pragma unroll
      for (int jn = 0; jn < C::FN; ++jn) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = L.n0 + wn * C::WTN + jn * 8 + tq + 4 * e;
          if (n >= P.N) continue;
          const double p1 = acc[im][jn][0][e], p2 = acc[im][jn][1][e], p3 = acc[im][jn][2][e];
          double re = p1 - p2, imv = (p3 - p1) - p2;
          for (int a = 0; a < P.naddends; ++a) {
            const GemmAddend& X = P.add[a];
            const double2 x = X.X[(int64_t)m * X.ldx + n];
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
    }
  }
#if BSEL_INV_STATS
  if (batch.chain_mark && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(batch.chain_mark, t);
  }
#endif
}

// ---------------------------------------------------------------------------
// Host side: TMA descriptor table (one per device)
// ---------------------------------------------------------------------------

// A descriptor describes one stored operand block: rows x cols complex at
// leading dimension ld, read in boxes of 8 complex x box_rows rows.
struct TmaKey {
  const void* p;
  int64_t ld;
  int32_t rows, cols, box_rows;
  bool operator==(const TmaKey& o) const {
    return p == o.p && ld == o.ld && rows == o.rows && cols == o.cols && box_rows == o.box_rows;
  }
};
struct TmaKeyHash {
  size_t operator()(const TmaKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.p) * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)k.ld * 0xBF58476D1CE4E5B9ull + (uint64_t)k.rows * 0x94D049BB133111EBull +
         ((uint64_t)k.cols << 20) + ((uint64_t)k.box_rows << 40);
    return (size_t)(h ^ (h >> 31));
  }
};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// Descriptors are encoded once per distinct operand block and kept in a
// device table (append-only; the kernel parameters carry slot indices, so a
// launch stays a few KB).  New slots are uploaded with one copy per launch
// before any kernel can reference them.  When the table fills, the device
// is synchronised and the table restarts (launches hold the shared side of
// `rw` from slot lookup to kernel launch).
class TmaTable {
 public:
  static constexpr uint32_t kMaxCap = 1u << 18;  // 32 MiB of descriptors per device
  // BSEL_TMA_TABLE_CAP (>= 64) shrinks the table (tests exercise the reset path)
  static uint32_t cap() {
    static const uint32_t c = [] {
      const char* e = getenv("BSEL_TMA_TABLE_CAP");
      const long v = e ? atol(e) : 0;
      return v >= 64 && v < (long)kMaxCap ? (uint32_t)v : kMaxCap;
    }();
    return c;
  }

  static TmaTable& current() {
    static std::mutex mu;
    static std::unique_ptr<TmaTable> tables[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!tables[dev]) tables[dev].reset(new TmaTable());
    return *tables[dev];
  }

  cudaError_t init() {
    if (dev_) return cudaSuccess;
    if (!encode_fn()) return cudaErrorNotSupported;
    cudaError_t e;
    if ((e = cudaMalloc(&dev_, (size_t)cap() * 128)) != cudaSuccess) return e;
    if ((e = cudaHostAlloc(&host_, (size_t)cap() * 128, cudaHostAllocDefault)) != cudaSuccess) return e;
    return cudaStreamCreateWithFlags(&up_, cudaStreamNonBlocking);
  }

  // Fill tmaA / tmaB of every term; the caller holds rw (shared).
  cudaError_t resolve(GemmBatch& b, int BM, int BN, int BK, bool* full) {
    std::lock_guard<std::mutex> lock(mu_);
    cudaError_t e = init();
    if (e != cudaSuccess) return e;
    const uint32_t first = next_;
    for (int i = 0; i < b.nproblems; ++i) {
      GemmProblem& P = b.p[i];
      for (int t = 0; t < P.nterms; ++t) {
        GemmTerm& T = P.term[t];
        if (T.K <= 0) continue;
        // A: op N -> stored M x K (boxes of BM rows); op C -> stored K x M (boxes of BK rows)
        const TmaKey ka = T.opA == kOpN ? TmaKey{T.A, T.lda, P.M, T.K, BM} : TmaKey{T.A, T.lda, T.K, P.M, BK};
        // B: op N -> stored K x N (boxes of BK rows); op C -> stored N x K (boxes of BN rows)
        const TmaKey kb = T.opB == kOpN ? TmaKey{T.B, T.ldb, T.K, P.N, BK} : TmaKey{T.B, T.ldb, P.N, T.K, BN};
        if ((e = slot(ka, &T.tmaA, full)) != cudaSuccess || (e = slot(kb, &T.tmaB, full)) != cudaSuccess)
          return e;
        if (*full) return cudaSuccess;
      }
    }
    if (next_ > first) {  // publish the new descriptors before any launch can use them
      if ((e = cudaMemcpyAsync(dev_ + (size_t)first * 128, host_ + (size_t)first * 128,
                               (size_t)(next_ - first) * 128, cudaMemcpyHostToDevice, up_)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(up_)) != cudaSuccess) return e;
      for (uint32_t s = first; s < next_; ++s) map_.emplace(pending_[s - first], s);
      pending_.clear();
    }
    b.tma_table = dev_;
    return cudaSuccess;
  }

  void reset() {  // caller holds rw exclusively
    std::lock_guard<std::mutex> lock(mu_);
    cudaDeviceSynchronize();
    map_.clear();
    pending_.clear();
    next_ = 0;
  }

  std::shared_mutex rw;

 private:
  cudaError_t slot(const TmaKey& k, uint32_t* id, bool* full) {
    auto it = map_.find(k);
    if (it != map_.end()) {
      *id = it->second;
      return cudaSuccess;
    }
    for (size_t j = 0; j < pending_.size(); ++j)  // new in this launch already
      if (pending_[j] == k) {
        *id = next_ - (uint32_t)pending_.size() + (uint32_t)j;
        return cudaSuccess;
      }
    if (next_ == cap()) {
      *full = true;
      pending_.clear();
      return cudaSuccess;
    }
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(host_ + (size_t)next_ * 128);
    const cuuint64_t dims[2] = {(cuuint64_t)k.cols * 2, (cuuint64_t)k.rows};  // doubles, rows
    const cuuint64_t strides[1] = {(cuuint64_t)k.ld * 16};
    const cuuint32_t box[2] = {16, (cuuint32_t)k.box_rows};  // 8 complex = 128 B
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(k.p), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      fprintf(stderr, "bsel: cuTensorMapEncodeTiled failed (%d): rows %d cols %d ld %lld box %d\n", (int)r, k.rows,
              k.cols, (long long)k.ld, k.box_rows);
      return cudaErrorInvalidValue;
    }
    pending_.push_back(k);
    *id = next_++;
    return cudaSuccess;
  }

  std::mutex mu_;
  std::unordered_map<TmaKey, uint32_t, TmaKeyHash> map_;
  std::vector<TmaKey> pending_;
  char* dev_ = nullptr;
  char* host_ = nullptr;
  cudaStream_t up_ = nullptr;
  uint32_t next_ = 0;
};

template <class C>
int tiles_of(GemmProblem& P) {
  P.tiles_n = (P.N + C::BN - 1) / C::BN;
  const int tm = (P.M + C::BM - 1) / C::BM;
  if (!P.lower_only) return tm * P.tiles_n;
  int cnt = 0;
  for (int tr = 0; tr < tm; ++tr) cnt += std::min(P.tiles_n, ((tr + 1) * C::BM - 1) / C::BN + 1);
  return cnt;
}

template <class C>
cudaError_t launch3(GemmBatch& batch, cudaStream_t stream, bool no_persist = false) {
  const cudaError_t attr = per_device([] {
    return cudaFuncSetAttribute(zgemm3m_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  if (attr != cudaSuccess) return attr;
  const int resident = per_device([] {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zgemm3m_kernel<C>, C::THREADS, C::SMEM) !=
        cudaSuccess)
      per_sm = 1;
    return std::max(1, per_sm) * device_sm_count();
  });
  int tiles = 0;
  for (int i = 0; i < batch.nproblems; ++i) {
    GemmProblem& P = batch.p[i];
    P.tile_begin = tiles;
    tiles += tiles_of<C>(P);
  }
  batch.total_tiles = tiles;
  if (tiles == 0) return cudaSuccess;
  int prof = -1;
  double flops = 0.0, bytes = 0.0;
  if (profiling()) {
    for (int i = 0; i < batch.nproblems; ++i) {
      const GemmProblem& P = batch.p[i];
      const double frac = P.lower_only ? (double)tiles_of<C>(const_cast<GemmProblem&>(P)) /
                                             (double)(((P.M + C::BM - 1) / C::BM) * P.tiles_n)
                                       : 1.0;
      const double M = P.M * frac, N = P.N;
      bytes += 16.0 * M * N * (1 + P.naddends);
      for (int t = 0; t < P.nterms; ++t) {
        flops += 8.0 * M * N * P.term[t].K;  // algorithmic (complex) flops; the 3M form executes 3/4
        bytes += 16.0 * (M + N) * P.term[t].K;
      }
    }
    prof = profile_open(stream);
  }
  TmaTable& tab = TmaTable::current();
  std::shared_lock<std::shared_mutex> hold(tab.rw);
  for (;;) {
    bool full = false;
    const cudaError_t e = tab.resolve(batch, C::BM, C::BN, C::BK, &full);
    if (e != cudaSuccess) return e;
    if (!full) break;
    hold.unlock();
    {
      std::unique_lock<std::shared_mutex> excl(tab.rw);
      tab.reset();
    }
    hold.lock();
  }
  // persistent grid (one wave of CTAs looping over the tiles; the producer
  // overlaps the next tile's loads with the epilogue) or, with
  // BSEL_GEMM3M_PERSIST=0, one CTA per tile (the CTA scheduler can then slot
  // a higher-priority stream's CTAs in between tiles)
  static const bool persist = [] {
    const char* e = getenv("BSEL_GEMM3M_PERSIST");
    return !(e && atoi(e) == 0);
  }();
  int grid = (persist && !no_persist) ? std::min(tiles, resident) : tiles;
  if (batch.max_ctas > 0 && batch.max_ctas < grid) grid = batch.max_ctas;
  if (batch.avoid_sms > 0) {
    if (!batch.tile_counter) return cudaErrorInvalidValue;
    grid = std::min(tiles, resident);
    const cudaError_t e = cudaMemsetAsync(batch.tile_counter, 0, 2 * sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
  }
  zgemm3m_kernel<C><<<grid, C::THREADS, C::SMEM, stream>>>(batch);
  count_launch();
  profile_close(prof, stream, 0, flops, bytes, 0.75 * flops);
  return cudaGetLastError();
}

}  // namespace

// Variant selection (tile counts of the launch).  BSEL_GEMM3M_CFG forces one:
// 64 (64x64), 6432 (64x32), 643232 (64x32, BK 32), 32 (32x32).
cudaError_t launch_gemm_batch_3m(GemmBatch& batch, cudaStream_t stream, int tile_cfg) {
  static const int forced = [] {
    const char* e = getenv("BSEL_GEMM3M_CFG");
    return e ? atoi(e) : 0;
  }();
  int cfg = forced;
  if (tile_cfg == kTile3m64) cfg = 64;
  if (tile_cfg == kTile3m6432) cfg = 6432;
  if (tile_cfg == kTile3m32) cfg = 32;
  if (tile_cfg == kTile3m64k32) return launch3<C3_64_K32>(batch, stream);
  if (tile_cfg == kTile3m6432k32) return launch3<C3_6432_K32>(batch, stream);
  if (!cfg) {
    int64_t t64 = 0, t6432 = 0;
    for (int i = 0; i < batch.nproblems; ++i) {
      const GemmProblem& P = batch.p[i];
      t64 += (int64_t)((P.M + 63) / 64) * ((P.N + 63) / 64);
      t6432 += (int64_t)((P.M + 63) / 64) * ((P.N + 31) / 32);
    }
    const int64_t sms = device_sm_count();
    if (tile_cfg == kTile32)
      cfg = 32;
    else if (tile_cfg == kTile64)
      cfg = 64;
    else if (tile_cfg == kTileAutoFwd)
      // Forward aux levels share the SMs with the Schur chain (block inverse
      // + two chain products on the priority stream): the BK 16 variants,
      // 64x64 from two waves.  With the BK 32 tiles here the single-lane
      // chain of a 2-GPU rank ran 328 vs 274 ms (profiles/sweeps_r02.md).
      cfg = t64 >= 2 * sms ? 64 : t6432 >= sms ? 6432 : 32;
    else if (t6432 >= sms)
      // 64x32 tiles with BK 32 (2 CTAs/SM) whenever they fill one wave: on
      // the concurrent backward levels they beat 64x64 (43.1 vs 41.9 TFLOP/s
      // algorithmic, 3 streams) and match it on 1024^3 (35.9 vs 35.8);
      // profiles/gemm3m_micro_r02b.json.
      cfg = 643232;
    else
      cfg = 32;
  }
  // BSEL_FWD_AUX_PERSIST=0 (experiment): the forward aux levels launch one
  // CTA per tile, so the chain's next kernel can take SMs between tiles
  static const bool fwd_np = [] {
    const char* e = getenv("BSEL_FWD_AUX_PERSIST");
    return e && atoi(e) == 0;
  }();
  const bool np = fwd_np && tile_cfg == kTileAutoFwd;
  if (cfg == 64) return launch3<C3_64>(batch, stream, np);
  if (cfg == 6432) return launch3<C3_6432>(batch, stream, np);
  if (cfg == 643232) return launch3<C3_6432_K32>(batch, stream, np);
  return launch3<C3_32>(batch, stream, np);
}

}  // namespace bsel
