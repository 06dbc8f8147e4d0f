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
// Memory layout: a CTA owns a 32 x 32 (x, y) column of the grid and marches in
// z; a ring of (32+2) x (32+4) rank planes with halo lives in shared memory, so
// each rank is read from HBM once (halos hit L2) and every output is written
// once, coalesced.  No integer division: coordinates come from the launch grid.
// 3-D grids with nx % 4 == 0 take the TMA-fed register-marching kernel of
// classify_zreg.cuh instead (flags / pointer variants).
#pragma once
#include <cstdlib>

#include "lts_common.cuh"

namespace lts {

enum { PTR_NONE = 0, PTR_ASC = 1, PTR_DESC = 2 };

constexpr int CL_TX = 32, CL_TY = 8, CL_VY = 2, CL_ZC = 16;  // thread owns CL_VY rows
constexpr int CL_PX = CL_TX + 2, CL_PY = CL_TY * CL_VY + 2;

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
  // (d(k) + 1) in bits 2k..2k+1
  __host__ __device__ static constexpr unsigned packed_dx() {
    unsigned p = 0;
    for (int k = 0; k < K; k++) p |= (unsigned)(dx(k) + 1) << (2 * k);
    return p;
  }
  __host__ __device__ static constexpr unsigned packed_dy() {
    unsigned p = 0;
    for (int k = 0; k < K; k++) p |= (unsigned)(dy(k) + 1) << (2 * k);
    return p;
  }
  __host__ __device__ static constexpr unsigned packed_dz() {
    unsigned p = 0;
    for (int k = 0; k < K; k++) p |= (unsigned)(dz(k) + 1) << (2 * k);
    return p;
  }
};

// Thread layout: 16 x 16 threads, each owns the voxel pair (x, x+1) of one
// row of a 32 x 16 (x, y) tile and marches in z.  Shared-memory rows are
// padded so the pair sits at an even index: one 64-bit load fetches both
// centres / both same-column neighbours, and the 14-neighbour stencil of the
// pair needs 7 paired + 8 scalar loads.  Flags use 3-input min/max
// (VIMNMX3): invalid neighbours hold -1, which is never the signed max and
// always the unsigned max; packing (rank << 4 | k) keeps the arg-extremum.
constexpr int CP_TX = 16, CP_TY = 16, CP_RY = 2, CP_ZC = 16;  // thread: 2 x-pairs rows
constexpr int CP_W = 2 * CP_TX;           // tile width (voxels)
constexpr int CP_PITCH = CP_W + 4;         // padded smem row: [pad, x0-1 .. x0+32, pad]
constexpr int CP_ROWS = CP_TY * CP_RY + 2;
constexpr int CP_RING = 5;  // planes z-1..z+1 read, z+2 written: one barrier per plane

struct Nb2 {  // the 14 stencil values of one voxel, reference offset order
  int v[14];
};

template <int NDIM, bool COUNTS, int PTR>
__device__ __forceinline__ void classify_emit(const Nb2 &A, const Nb2 &B, int2 c0, int x, int y, int z,
                                              int nx, int64_t sxy, uint8_t *__restrict__ flags,
                                              int16_t *__restrict__ lower, int16_t *__restrict__ upper,
                                              const uint8_t *__restrict__ lut, int32_t *__restrict__ ptr);

// classification of the voxel pair (x, x+1) of row y in plane z; c = index of
// (x, y) in the padded plane rows; p0 / pm / pp = planes z, z-1, z+1
template <int NDIM, bool COUNTS, int PTR, int PITCH>
__device__ __forceinline__ void classify_pair(const int *__restrict__ p0, const int *__restrict__ pm,
                                              const int *__restrict__ pp, int c, int x, int y, int z,
                                              int nx, int64_t sxy, uint8_t *__restrict__ flags,
                                              int16_t *__restrict__ lower, int16_t *__restrict__ upper,
                                              const uint8_t *__restrict__ lut, int32_t *__restrict__ ptr) {
  using St = Stencil<NDIM>;
  constexpr int CP_PITCH = PITCH;
  {
      // plane z rows y-1, y, y+1
      const int2 c0 = *reinterpret_cast<const int2 *>(p0 + c);
      const int a0m = p0[c - 1], a0p = p0[c + 2];
      const int2 u0 = *reinterpret_cast<const int2 *>(p0 + c + CP_PITCH);
      const int u0p = p0[c + CP_PITCH + 2];
      const int2 d0 = *reinterpret_cast<const int2 *>(p0 + c - CP_PITCH);
      const int d0m = p0[c - CP_PITCH - 1];
      Nb2 A, B;
      // reference offset order (triangulation.py:32-45)
      A.v[0] = c0.y;  B.v[0] = a0p;            // (1,0,0)
      A.v[1] = u0.x;  B.v[1] = u0.y;           // (0,1,0)
      if (NDIM == 2) {
        A.v[2] = u0.y;  B.v[2] = u0p;          // (1,1)
        A.v[3] = a0m;   B.v[3] = c0.x;         // (-1,0)
        A.v[4] = d0.x;  B.v[4] = d0.y;         // (0,-1)
        A.v[5] = d0m;   B.v[5] = d0.x;         // (-1,-1)
      } else {
        const int2 cp = *reinterpret_cast<const int2 *>(pp + c);
        const int cpp = pp[c + 2];
        const int2 up = *reinterpret_cast<const int2 *>(pp + c + CP_PITCH);
        const int upp = pp[c + CP_PITCH + 2];
        const int2 cm = *reinterpret_cast<const int2 *>(pm + c);
        const int cmm = pm[c - 1];
        const int2 dm = *reinterpret_cast<const int2 *>(pm + c - CP_PITCH);
        const int dmm = pm[c - CP_PITCH - 1];
        A.v[2] = cp.x;   B.v[2] = cp.y;        // (0,0,1)
        A.v[3] = u0.y;   B.v[3] = u0p;         // (1,1,0)
        A.v[4] = cp.y;   B.v[4] = cpp;         // (1,0,1)
        A.v[5] = up.x;   B.v[5] = up.y;        // (0,1,1)
        A.v[6] = up.y;   B.v[6] = upp;         // (1,1,1)
        A.v[7] = a0m;    B.v[7] = c0.x;        // (-1,0,0)
        A.v[8] = d0.x;   B.v[8] = d0.y;        // (0,-1,0)
        A.v[9] = cm.x;   B.v[9] = cm.y;        // (0,0,-1)
        A.v[10] = d0m;   B.v[10] = d0.x;       // (-1,-1,0)
        A.v[11] = cmm;   B.v[11] = cm.x;       // (-1,0,-1)
        A.v[12] = dm.x;  B.v[12] = dm.y;       // (0,-1,-1)
        A.v[13] = dmm;   B.v[13] = dm.x;       // (-1,-1,-1)
      }
      classify_emit<NDIM, COUNTS, PTR>(A, B, c0, x, y, z, nx, sxy, flags, lower, upper, lut, ptr);
  }
}

// classification outputs of the voxel pair (x, x+1) from its two neighbour
// vectors (reference offset order) and centre ranks c0
template <int NDIM, bool COUNTS, int PTR>
__device__ __forceinline__ void classify_emit(const Nb2 &A, const Nb2 &B, int2 c0, int x, int y, int z,
                                              int nx, int64_t sxy, uint8_t *__restrict__ flags,
                                              int16_t *__restrict__ lower, int16_t *__restrict__ upper,
                                              const uint8_t *__restrict__ lut, int32_t *__restrict__ ptr) {
  using St = Stencil<NDIM>;
  constexpr int K = St::K;
  {
      const int64_t vA = (int64_t)z * sxy + (int64_t)y * nx + x;
      uint8_t fl[2] = {0, 0};
      int pv[2] = {0, 0};
      const bool two = x + 1 < nx;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const Nb2 &N = h == 0 ? A : B;
        const int rv = h == 0 ? c0.x : c0.y;
        const int64_t v = vA + h;
        if (h == 1 && !two) break;
        if (COUNTS) {
          unsigned upm = 0, valid = 0;
#pragma unroll
          for (int k = 0; k < K; k++) {
            valid |= (unsigned)(N.v[k] >= 0) << k;
            upm |= (unsigned)(N.v[k] > rv) << k;
          }
          const unsigned lo = valid & ~upm;
          if (flags) flags[v] = (uint8_t)((upm == 0 ? FL_MAX : 0) | (lo == 0 ? FL_MIN : 0));
          lower[v] = (int16_t)__ldg(lut + lo);
          upper[v] = (int16_t)__ldg(lut + upm);
        } else {
          // One side is a packed arg-extremum reduction (three-input
          // VIMNMX3, quarter-rate XU pipe); the other side is only a yes/no
          // test, done as an ISETP chain on the ALU pipe so the two pipes
          // share the work.  Invalid neighbours hold -1: never the signed
          // max, always the unsigned max.
          constexpr bool DESC = PTR == PTR_DESC;
          int ext = -1;
          unsigned ulo = 0xffffffffu;
          bool other = true;
#pragma unroll
          for (int k = 0; k < K; k += 2) {
            int a = N.v[k], b = N.v[k + 1];
            if (DESC) other = other & (a < rv) & (b < rv);  // no upper neighbour
            else other = other & ((unsigned)a > (unsigned)rv) & ((unsigned)b > (unsigned)rv);  // no lower
            if (PTR != PTR_NONE) {  // ru < 2^27 (n <= 2^27)
              a = a < 0 ? -1 : ((a << 4) | k);
              b = b < 0 ? -1 : ((b << 4) | (k + 1));
            }
            if (DESC) ulo = __vimin3_u32(ulo, (unsigned)a, (unsigned)b);
            else ext = __vimax3_s32(ext, a, b);
          }
          int hi = ext;
          unsigned lo = ulo;
          bool ismax, ismin;
          if (DESC) {
            ismax = other;
            ismin = (lo == 0xffffffffu ? lo : (lo >> 4)) > (unsigned)rv;
          } else {
            ismax = (PTR == PTR_NONE ? hi : (hi < 0 ? -1 : (hi >> 4))) < rv;
            ismin = other;
          }
          fl[h] = (uint8_t)((ismax ? FL_MAX : 0) | (ismin ? FL_MIN : 0));
          if (PTR != PTR_NONE) {
            const bool self = PTR == PTR_ASC ? ismax : ismin;
            const int kb = PTR == PTR_ASC ? (hi & 15) : (int)(lo & 15u);
            // offset of stencil entry kb from 2-bit packed (d+1) tables
            const int ddx = (int)((St::packed_dx() >> (2 * kb)) & 3u) - 1;
            const int ddy = (int)((St::packed_dy() >> (2 * kb)) & 3u) - 1;
            const int ddz = (int)((St::packed_dz() >> (2 * kb)) & 3u) - 1;
            const int d = ddx + nx * ddy + (int)sxy * ddz;  // n <= 2^27
            pv[h] = self ? (int)v : (int)v + d;
          }
        }
      }
      if (!COUNTS) {
        // paired stores when the pair is 2-element aligned (nx even)
        const bool paired = two && (nx & 1) == 0;
        if (flags) {
          if (paired) *reinterpret_cast<uint16_t *>(flags + vA) = (uint16_t)(fl[0] | (fl[1] << 8));
          else {
            flags[vA] = fl[0];
            if (two) flags[vA + 1] = fl[1];
          }
        }
        if (PTR != PTR_NONE) {
          if (paired) *reinterpret_cast<int2 *>(ptr + vA) = make_int2(pv[0], pv[1]);
          else {
            ptr[vA] = pv[0];
            if (two) ptr[vA + 1] = pv[1];
          }
        }
      }
  }
}

template <int NDIM, bool COUNTS, int PTR>
__global__ void __launch_bounds__(CP_TX *CP_TY) k_classify_tile(Grid g, const int32_t *__restrict__ rank,
                                                             uint8_t *__restrict__ flags,
                                                             int16_t *__restrict__ lower,
                                                             int16_t *__restrict__ upper,
                                                             const uint8_t *__restrict__ lut,
                                                             int32_t *__restrict__ ptr) {
  using St = Stencil<NDIM>;
  constexpr int NP = NDIM == 2 ? 1 : CP_RING;
  __shared__ __align__(16) int pl[NP][CP_ROWS * CP_PITCH];
  const int tid = threadIdx.y * CP_TX + threadIdx.x;
  const int x0 = blockIdx.x * CP_W, y0 = blockIdx.y * (CP_TY * CP_RY);
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t sxy = (int64_t)nx * ny;
  constexpr int NE = CP_ROWS * (CP_W + 2), NT = CP_TX * CP_TY, NEPT = (NE + NT - 1) / NT;
  int gofs[NEPT], sofs[NEPT];
  bool gin[NEPT], sin_[NEPT];
#pragma unroll
  for (int e = 0; e < NEPT; e++) {
    int i = tid + e * NT;
    int py = i / (CP_W + 2), px = i - py * (CP_W + 2);
    int gx = x0 + px - 1, gy = y0 + py - 1;
    sin_[e] = i < NE;
    gin[e] = sin_[e] && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    gofs[e] = gin[e] ? gy * nx + gx : 0;
    sofs[e] = py * CP_PITCH + px + 1;
  }
  auto fetch = [&](int z, int *reg) {
#pragma unroll
    for (int e = 0; e < NEPT; e++)
      reg[e] = (gin[e] && z >= 0 && z < nz) ? __ldg(rank + (int64_t)z * sxy + gofs[e]) : -1;
  };
  auto put = [&](int buf, const int *reg) {
#pragma unroll
    for (int e = 0; e < NEPT; e++)
      if (sin_[e]) pl[buf][sofs[e]] = reg[e];
  };
  const int zb = NDIM == 2 ? 0 : blockIdx.z * CP_ZC;
  const int ze = NDIM == 2 ? 1 : min(nz, zb + CP_ZC);
  int nxt[NEPT];
  {
    int a[NEPT];
    if (NDIM == 3) {
      fetch(zb - 1, a);
      put(0, a);
      fetch(zb, a);
      put(1, a);
      fetch(zb + 1, a);
      put(2, a);
      fetch(zb + 2, nxt);
    } else {
      fetch(0, a);
      put(0, a);
    }
  }
  const int tx = threadIdx.x;
  int sm = 0;  // ring slot of plane z-1
  for (int z = zb; z < ze; z++) {
    const int s1 = sm + 1 >= CP_RING ? sm + 1 - CP_RING : sm + 1;
    const int s2 = s1 + 1 >= CP_RING ? s1 + 1 - CP_RING : s1 + 1;
    const int s3 = s2 + 1 >= CP_RING ? s2 + 1 - CP_RING : s2 + 1;
    if (NDIM == 3) {
      // plane z+2 goes to a slot nobody reads this iteration; prefetch z+3
      put(s3, nxt);
      if (z + 3 < ze + 1) fetch(z + 3, nxt);
    }
    __syncthreads();
    const int r3 = sm;
    const int *p0 = pl[NDIM == 2 ? 0 : s1];
    const int *pm = pl[NDIM == 2 ? 0 : r3];
    const int *pp = pl[NDIM == 2 ? 0 : s2];
#pragma unroll
    for (int ry = 0; ry < CP_RY; ry++) {
    const int ty = threadIdx.y + ry * CP_TY;
    const int x = x0 + 2 * tx, y = y0 + ty;
    const int c = (ty + 1) * CP_PITCH + 2 * tx + 2;
    if (y < ny && x < nx)
      classify_pair<NDIM, COUNTS, PTR, CP_PITCH>(p0, pm, pp, c, x, y, z, nx, sxy, flags, lower, upper, lut, ptr);
    }
    sm = s1;
    if (NDIM == 2) __syncthreads();
  }
}

inline bool launch_classify_zreg(const Grid &g, const int32_t *rank, uint8_t *flags, int32_t *ptr, int ptr_kind,
                                 cudaStream_t s);
// 2-D strip kernel (classify_2d.cuh); false = not applicable
inline bool launch_classify_2d(const Grid &g, const int32_t *rank, uint8_t *flags, int32_t *ptr, int ptr_kind,
                               cudaStream_t s);

inline void launch_classify(const Grid &g, const int32_t *rank, uint8_t *flags, int16_t *lower,
                            int16_t *upper, const uint8_t *lut, int32_t *ptr, int ptr_kind,
                            cudaStream_t s) {
  if (lower == nullptr && launch_classify_zreg(g, rank, flags, ptr, ptr_kind, s)) return;
  if (lower == nullptr && launch_classify_2d(g, rank, flags, ptr, ptr_kind, s)) return;
  dim3 blk(CP_TX, CP_TY);
  dim3 grd((g.nx + CP_W - 1) / CP_W, (g.ny + CP_TY * CP_RY - 1) / (CP_TY * CP_RY),
           g.ndim == 2 ? 1 : (g.nz + CP_ZC - 1) / CP_ZC);
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
