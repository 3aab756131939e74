// Boundary publication over NVLink peer memory (bsel_publish, btasel_b200.h).
//
// The distributed scheme's one all_gather (dist.py:436) moves every rank's
// boundary payload -- its updated boundary diagonal blocks, arrow strips and
// (middle partitions) fill-in couplings -- to every rank.  Instead of packing
// the blocks into a send slot and calling NCCL, one kernel reads each block
// where the elimination left it and stores it straight into the payload
// slot of this rank in EVERY rank's receive buffer (symmetric memory: the
// peers' buffers are mapped into this process, so the stores travel over
// NVLink / NVSwitch as 16-byte P2P writes).  The caller brackets it with a
// device-side barrier over the group (torch symmetric memory signal pads).
// HBM / NVLink bound: bytes per rank = payload x world.
#include <algorithm>
#include <cstdint>

#include "zgemm.cuh"

namespace bsel {

namespace {
constexpr int kMaxPubBlocks = 16, kMaxPubDst = 8;

struct PublishArgs {
  const double2* src[kMaxPubBlocks];
  int64_t elems[kMaxPubBlocks];    // complex elements of block i
  int64_t dst_off[kMaxPubBlocks];  // complex offset of block i in every destination buffer
  double2* dst[kMaxPubDst];
  int nblocks, ndst;
  int64_t hdr_off;                 // complex offset of the 2-complex (4-double) header
  double hdr[4];
};

__global__ void __launch_bounds__(256) publish_kernel(const __grid_constant__ PublishArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t0 < 2)
    for (int d = 0; d < a.ndst; ++d) a.dst[d][a.hdr_off + t0] = make_double2(a.hdr[2 * t0], a.hdr[2 * t0 + 1]);
  for (int i = 0; i < a.nblocks; ++i) {
    const double2* s = a.src[i];
    for (int64_t e = t0; e < a.elems[i]; e += stride) {
      const double2 v = __ldcs(s + e);  // read once, streamed
#pragma unroll 1
      for (int d = 0; d < a.ndst; ++d) a.dst[d][a.dst_off[i] + e] = v;
    }
  }
}
}  // namespace

cudaError_t launch_publish(const double2* const* src, const int64_t* elems, const int64_t* dst_off, int nblocks,
                           double2* const* dst, int ndst, int64_t hdr_off, const double* hdr, cudaStream_t s) {
  if (nblocks < 0 || nblocks > kMaxPubBlocks || ndst < 1 || ndst > kMaxPubDst) return cudaErrorInvalidValue;
  PublishArgs a{};
  int64_t total = 0;
  for (int i = 0; i < nblocks; ++i) {
    a.src[i] = src[i];
    a.elems[i] = elems[i];
    a.dst_off[i] = dst_off[i];
    total += elems[i];
  }
  for (int d = 0; d < ndst; ++d) a.dst[d] = dst[d];
  a.nblocks = nblocks;
  a.ndst = ndst;
  a.hdr_off = hdr_off;
  for (int k = 0; k < 4; ++k) a.hdr[k] = hdr[k];
  const int grid = (int)std::min<int64_t>(4 * (int64_t)device_sm_count(), std::max<int64_t>(1, (total + 255) / 256));
  publish_kernel<<<grid, 256, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bsel
