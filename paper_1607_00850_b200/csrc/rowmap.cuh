// Device-side addressing of the z lines a RowMap describes (kernels.cuh),
// shared by the fused z pass (kernels.cu) and the generic-length kernels
// (kernels_gen.cu).
#pragma once

#include "kernels.cuh"

namespace sdns_dev {

// Offset of element kz of z line ri: `ro` = zrow_off for unsegmented maps.
__device__ __forceinline__ long long zel(const RowMap& rm, long long ro, int ri, int k) {
  if (rm.cstride) return ro + static_cast<long long>(k >> 3) * rm.cstride + (k & 7);
  if (rm.nseg == 0) return ro + k;
  int sg = 0;
  while (sg + 1 < rm.nseg && k >= rm.seg_k0[sg + 1]) ++sg;
  return rm.seg_base[sg] + static_cast<long long>(ri) * rm.seg_pitch[sg] + (k - rm.seg_k0[sg]);
}

__device__ __forceinline__ long long zrow_off(const RowMap& rm, int ri) {
  if (rm.cstride) {
    const int x = ri / rm.rpp, y = ri - x * rm.rpp;
    return static_cast<long long>(x) * rm.xplane + static_cast<long long>(y) * 8;
  }
  if (rm.blk == 0) {
    const int pl = ri / rm.rpp, r = ri - pl * rm.rpp;
    return (static_cast<long long>(pl) * rm.prow + r) * rm.pitch;
  }
  const int xl = ri / rm.ny, y = ri - xl * rm.ny;
  const int q = y / rm.blk, yl = y - q * rm.blk;
  return (static_cast<long long>(q * rm.blk + xl) * rm.prow + yl) * rm.pitch;
}

// Output element (ri, kz k) of a peer-direct z pass and its destination's
// component stride (see z_fused_to).
struct ZDst {
  long long el, cs;
};
__device__ __forceinline__ ZDst zdst(const RowMap& rmo, int ri, int k) {
  int sg = 0;
  while (sg + 1 < rmo.nseg && k >= rmo.seg_k0[sg + 1]) ++sg;
  return ZDst{rmo.seg_base[sg] + static_cast<long long>(ri) * rmo.seg_pitch[sg] +
                  (k - rmo.seg_k0[sg]),
              rmo.seg_cs[sg]};
}

}  // namespace sdns_dev
