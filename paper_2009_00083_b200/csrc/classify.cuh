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
//
// Memory layout: a CTA owns a 32 x 8 (x, y) column of the grid and marches in
// z; three (8+2) x (32+2) rank planes with halo live in shared memory, so each
// rank is read from HBM about 1.3 times (halo) and every output is written
// once, coalesced.  No integer division: coordinates come from the launch grid.
#pragma once
#include "lts_common.cuh"

namespace lts {

enum { PTR_NONE = 0, PTR_ASC = 1, PTR_DESC = 2 };

constexpr int CL_TX = 32, CL_TY = 8, CL_ZC = 16;
constexpr int CL_PX = CL_TX + 2, CL_PY = CL_TY + 2;

// compile-time copy of the reference offset tables (triangulation.py:32-45)
template <int NDIM>
struct Stencil {
  static constexpr int K = NDIM == 2 ? 6 : 14;
  __host__ __device__ static constexpr int dx(int k) {
    constexpr int a2[6] = {1, 0, 1, -1, 0, -1};
    constexpr int a3[14] = {1, 0, 0, 1, 1, 0, 1, -1, 0, 0, -1, -1, 0, -1};
    return NDIM == 2 ? a2[k] : a3[k];
  }
  __host__ __device__ static constexpr int dy(int k) {
    constexpr int a2[6] = {0, 1, 1, 0, -1, -1};
    constexpr int a3[14] = {0, 1, 0, 1, 0, 1, 1, 0, -1, 0, -1, 0, -1, -1};
    return NDIM == 2 ? a2[k] : a3[k];
  }
  __host__ __device__ static constexpr int dz(int k) {
    constexpr int a3[14] = {0, 0, 1, 0, 1, 1, 1, 0, 0, -1, 0, -1, -1, -1};
    return NDIM == 2 ? 0 : a3[k];
  }
};

template <int NDIM, bool COUNTS, int PTR>
__global__ void __launch_bounds__(CL_TX *CL_TY) k_classify_tile(Grid g, const int32_t *__restrict__ rank,
                                                             uint8_t *__restrict__ flags,
                                                             int16_t *__restrict__ lower,
                                                             int16_t *__restrict__ upper,
                                                             const uint8_t *__restrict__ lut,
                                                             int32_t *__restrict__ ptr) {
  using St = Stencil<NDIM>;
  constexpr int K = St::K;
  constexpr int NP = NDIM == 2 ? 1 : 3;
  __shared__ int pl[NP][CL_PY * CL_PX];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * CL_TX + tx;
  const int x0 = blockIdx.x * CL_TX, y0 = blockIdx.y * CL_TY;
  const int x = x0 + tx, y = y0 + ty;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t sxy = (int64_t)nx * ny;
  // each thread owns <= 2 halo-tile elements; plane z+1 is prefetched into
  // registers one iteration ahead so HBM latency overlaps the stencil work
  constexpr int NE = CL_PY * CL_PX, NT = CL_TX * CL_TY;
  int gofs[2];
  bool gin[2];
#pragma unroll
  for (int e = 0; e < 2; e++) {
    int i = tid + e * NT;
    int py = i / CL_PX, px = i - py * CL_PX;
    int gx = x0 + px - 1, gy = y0 + py - 1;
    gin[e] = i < NE && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    gofs[e] = gin[e] ? gy * nx + gx : 0;
  }
  auto fetch = [&](int z, int *reg) {
#pragma unroll
    for (int e = 0; e < 2; e++)
      reg[e] = (gin[e] && z >= 0 && z < nz) ? __ldg(rank + (int64_t)z * sxy + gofs[e]) : -1;
  };
  auto put = [&](int buf, const int *reg) {
#pragma unroll
    for (int e = 0; e < 2; e++)
      if (tid + e * NT < NE) pl[buf][tid + e * NT] = reg[e];
  };
  const int zb = NDIM == 2 ? 0 : blockIdx.z * CL_ZC;
  const int ze = NDIM == 2 ? 1 : min(nz, zb + CL_ZC);
  int nxt[2], nx2[2], nx3[2];
  if (NDIM == 3) {
    int a[2];
    fetch(zb - 1, a);
    put(0, a);
    fetch(zb, a);
    put(1, a);
    fetch(zb + 1, nxt);
    fetch(zb + 2, nx2);
    fetch(zb + 3, nx3);
  } else {
    int a[2];
    fetch(0, a);
    put(0, a);
  }
  const int c = (ty + 1) * CL_PX + (tx + 1);
  int r3 = 0;  // (z - zb) % 3
  for (int z = zb; z < ze; z++) {
    // ring buffer: plane z-1 in slot r3, z in r3+1, z+1 in r3+2 (mod 3)
    const int s1 = r3 == 2 ? 0 : r3 + 1;
    const int s2 = s1 == 2 ? 0 : s1 + 1;
    if (NDIM == 3) {
      put(s2, nxt);
      __syncthreads();
      // three planes in flight per thread
#pragma unroll
      for (int e = 0; e < 2; e++) {
        nxt[e] = nx2[e];
        nx2[e] = nx3[e];
      }
      if (z + 3 < ze) fetch(z + 4, nx3);
    } else {
      __syncthreads();
    }
    const int *pm = pl[NDIM == 2 ? 0 : r3];
    const int *p0 = pl[NDIM == 2 ? 0 : s1];
    const int *pp = pl[NDIM == 2 ? 0 : s2];
    if (x < nx && y < ny) {
      const int rv = p0[c];
      const int64_t v = (int64_t)z * sxy + (int64_t)y * nx + x;
      if (COUNTS) {
        unsigned up = 0, valid = 0;
#pragma unroll
        for (int k = 0; k < K; k++) {
          const int *P = St::dz(k) < 0 ? pm : (St::dz(k) > 0 ? pp : p0);
          const int ru = P[c + St::dy(k) * CL_PX + St::dx(k)];
          valid |= (unsigned)(ru >= 0) << k;
          up |= (unsigned)(ru > rv) << k;
        }
        const unsigned lo = valid & ~up;
        if (flags) flags[v] = (uint8_t)((up == 0 ? FL_MAX : 0) | (lo == 0 ? FL_MIN : 0));
        lower[v] = (int16_t)__ldg(lut + lo);
        upper[v] = (int16_t)__ldg(lut + up);
      } else {
        // invalid neighbours hold -1: never the signed max, always the
        // unsigned max.  Packing (rank << 4 | k) keeps the arg of the extremum.
        int hi = -1;
        unsigned lo = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < K; k++) {
          const int *P = St::dz(k) < 0 ? pm : (St::dz(k) > 0 ? pp : p0);
          const int ru = P[c + St::dy(k) * CL_PX + St::dx(k)];
          if (PTR == PTR_NONE) {
            hi = max(hi, ru);
            lo = min(lo, (unsigned)ru);
          } else {
            const int pk = (ru << 4) | k;  // ru < 2^27 (n < 2^27 for PTR kernels)
            hi = max(hi, ru < 0 ? -1 : pk);
            lo = min(lo, ru < 0 ? 0xffffffffu : (unsigned)pk);
          }
        }
        const int hr = PTR == PTR_NONE ? hi : (hi < 0 ? -1 : (hi >> 4));
        const unsigned lr = PTR == PTR_NONE ? lo : (lo == 0xffffffffu ? lo : (lo >> 4));
        const bool ismax = hr < rv, ismin = lr > (unsigned)rv;
        if (flags) flags[v] = (uint8_t)((ismax ? FL_MAX : 0) | (ismin ? FL_MIN : 0));
        if (PTR != PTR_NONE) {
          const bool self = PTR == PTR_ASC ? ismax : ismin;
          const int kb = PTR == PTR_ASC ? (hi & 15) : (int)(lo & 15u);
          int64_t d = 0;
#pragma unroll
          for (int k = 0; k < K; k++)
            if (kb == k) d = St::dx(k) + (int64_t)nx * St::dy(k) + sxy * St::dz(k);
          ptr[v] = (int)(self ? v : v + d);
        }
      }
    }
    r3 = s1;
    __syncthreads();
  }
}

inline void launch_classify(const Grid &g, const int32_t *rank, uint8_t *flags, int16_t *lower,
                            int16_t *upper, const uint8_t *lut, int32_t *ptr, int ptr_kind,
                            cudaStream_t s) {
  dim3 blk(CL_TX, CL_TY);
  dim3 grd((g.nx + CL_TX - 1) / CL_TX, (g.ny + CL_TY - 1) / CL_TY,
           g.ndim == 2 ? 1 : (g.nz + CL_ZC - 1) / CL_ZC);
  bool counts = lower != nullptr;
#define LTS_CL(ND, C, P) k_classify_tile<ND, C, P><<<grd, blk, 0, s>>>(g, rank, flags, lower, upper, lut, ptr)
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
