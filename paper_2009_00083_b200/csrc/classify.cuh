// classify.cuh -- extremum classification stencil (reference critical.py:95-119,
// _kernels.py:106-156) fused with the steepest-ascent / -descent pointers used
// by region discovery.
//
// Per vertex the kernel builds two K-bit masks over the Freudenthal stencil
// (valid neighbours, upper neighbours).  Minimum <=> no lower neighbour,
// maximum <=> no upper neighbour (critical.py:117-119 with counts of 0).  The
// reference's link component counts are exact functions of the side masks, so
// they come from a 2^K lookup table built from the reference's own link-pair
// table (triangulation.py:52-78 -- over-connected):
// lower = LUT[valid & ~upper], upper = LUT[upper].
#pragma once
#include "lts_common.cuh"

namespace lts {

enum { PTR_NONE = 0, PTR_ASC = 1, PTR_DESC = 2 };

template <int NDIM, bool COUNTS, int PTR>
__global__ void __launch_bounds__(256) k_classify(Grid g, const int32_t *__restrict__ rank,
                                                  uint8_t *__restrict__ flags,
                                                  int16_t *__restrict__ lower,
                                                  int16_t *__restrict__ upper,
                                                  const uint8_t *__restrict__ lut,
                                                  int32_t *__restrict__ ptr) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  const int n = (int)g.n;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int x, y, z;
    coords(g, v, x, y, z);
    const int rv = __ldg(rank + v);
    unsigned up = 0, valid = 0;
    int best = v;
    int brank = PTR == PTR_ASC ? -1 : 0x7fffffff;
#pragma unroll
    for (int k = 0; k < K; k++) {
      int u = nbr_at(g, x, y, z, k);
      if (u < 0) continue;
      valid |= 1u << k;
      int ru = __ldg(rank + u);
      if (ru > rv) {
        up |= 1u << k;
        if (PTR == PTR_ASC && ru > brank) {
          brank = ru;
          best = u;
        }
      } else if (PTR == PTR_DESC && ru < brank) {
        brank = ru;
        best = u;
      }
    }
    unsigned lo = valid & ~up;
    if (flags) flags[v] = (uint8_t)((up == 0 ? FL_MAX : 0) | (lo == 0 ? FL_MIN : 0));
    if (COUNTS) {
      lower[v] = (int16_t)__ldg(lut + lo);
      upper[v] = (int16_t)__ldg(lut + up);
    }
    if (PTR != PTR_NONE) ptr[v] = best;
  }
}

inline void launch_classify(const Grid &g, const int32_t *rank, uint8_t *flags, int16_t *lower,
                            int16_t *upper, const uint8_t *lut, int32_t *ptr, int ptr_kind,
                            cudaStream_t s) {
  int blocks = grid_blocks(g.n, 256, 148 * 8);
  bool counts = lower != nullptr;
#define LTS_CL(ND, C, P) k_classify<ND, C, P><<<blocks, 256, 0, s>>>(g, rank, flags, lower, upper, lut, ptr)
  if (g.ndim == 2) {
    if (counts) LTS_CL(2, true, PTR_NONE);
    else if (ptr_kind == PTR_ASC) LTS_CL(2, false, PTR_ASC);
    else if (ptr_kind == PTR_DESC) LTS_CL(2, false, PTR_DESC);
    else LTS_CL(2, false, PTR_NONE);
  } else {
    if (counts) LTS_CL(3, true, PTR_NONE);
    else if (ptr_kind == PTR_ASC) LTS_CL(3, false, PTR_ASC);
    else if (ptr_kind == PTR_DESC) LTS_CL(3, false, PTR_DESC);
    else LTS_CL(3, false, PTR_NONE);
  }
#undef LTS_CL
  g_launches++;
}

}  // namespace lts
