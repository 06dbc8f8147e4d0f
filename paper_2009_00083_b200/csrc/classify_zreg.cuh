// classify_zreg.cuh -- 3-D extremum classification (reference critical.py:95-119,
// _kernels.py:128-156; extremum <=> empty lower / upper link) fused with the
// steepest-ascent / -descent pointers, fed by TMA and marching z in registers.
//
// A CTA owns a 32 x 32 (x, y) column of the grid and a chunk of z.  Each
// plane z arrives as ONE cp.async.bulk.tensor box of (32+8) x (32+2) ranks
// (x from x0-4 so rows are 16-byte aligned) in a CZ_RING-deep shared ring,
// CZ_RING-1 planes ahead of the plane being loaded, completion tracked per
// slot by an mbarrier.  A thread owns a 4-voxel x strip of one row: per plane
// it loads the 16 ranks its strip's stencil touches in that plane (three
// 128-bit rows; the x-1 / x+4 halo comes from the neighbouring lane by
// shuffle) into registers and keeps the last three planes there, so every
// rank is read from shared memory once per thread instead of once per use.
// TMA zero-fills out-of-grid cells; the thread knows statically which of its
// 16 cells lie outside the grid in x / y and substitutes -1 (the "no
// neighbour" rank).  The planes z = -1 and z = nz are not loaded: the CTA
// fills their slot with -1 and completes the slot's mbarrier phase by a plain
// arrive, so every plane is read the same way.
//
// Pointers: the arg-extremum of the 14 neighbours must name its direction.
// Every loaded rank is packed once as r*8 + h, h = (i + 2j) mod 8 for the cell
// at offset (i, j) from the thread's strip origin (only the owning thread
// compares these values, so h can be strip-relative and a constant): the
// six in-plane offsets (dx + 2dy in +-{1,2,3}) and the four per adjacent plane
// ({0..3} or {0,-1,-2,-3}) are distinct mod 8 within their plane, and the
// plane of the winner comes from comparing the overall extremum with the two
// per-plane extrema.  Invalid neighbours pack to negative values: never the
// signed max, always the unsigned max.  Needs n <= 2^28 (r*8 < 2^31).
#pragma once
#include "classify.cuh"
#include "tma.cuh"

#include <algorithm>

namespace lts {

constexpr int CZ_TX = 8, CZ_TY = 32, CZ_T = CZ_TX * CZ_TY;  // 8 strips of 4 voxels x 32 rows
constexpr int CZ_W = 4 * CZ_TX;                              // tile width, voxels
constexpr int CZ_BX = CZ_W + 8, CZ_BY = CZ_TY + 2;          // TMA box 40 x 34 int32
constexpr int CZ_PLANE = CZ_BX * CZ_BY;
constexpr int CZ_SLOT = (CZ_PLANE * 4 + 127) / 128 * 32;    // 128-byte aligned destinations
constexpr int CZ_RING = 6;
#ifndef LTS_CZ_MINB
#define LTS_CZ_MINB 4
#endif

// the 16 stencil cells of a 4-voxel strip in one plane: row y-1 at x-1..x+3,
// row y at x-1..x+4, row y+1 at x..x+4
struct ZPl {
  int d[5], c[6], u[5];
};

enum { ZE_XM = 1, ZE_XP = 2, ZE_YM = 4, ZE_YP = 8 };

template <int PTR>
__device__ __forceinline__ void zreg_load(ZPl &P, const int *__restrict__ slot, int so, int tx, unsigned edge) {
  const int4 dv = *reinterpret_cast<const int4 *>(slot + so - CZ_BX);
  const int4 cv = *reinterpret_cast<const int4 *>(slot + so);
  const int4 uv = *reinterpret_cast<const int4 *>(slot + so + CZ_BX);
  int cm1 = __shfl_up_sync(0xffffffffu, cv.w, 1);
  int dm1 = __shfl_up_sync(0xffffffffu, dv.w, 1);
  int c4 = __shfl_down_sync(0xffffffffu, cv.x, 1);
  int u4 = __shfl_down_sync(0xffffffffu, uv.x, 1);
  if (tx == 0) {
    cm1 = slot[so - 1];
    dm1 = slot[so - CZ_BX - 1];
  }
  if (tx == CZ_TX - 1) {
    c4 = slot[so + 4];
    u4 = slot[so + CZ_BX + 4];
  }
  P.d[0] = dm1, P.d[1] = dv.x, P.d[2] = dv.y, P.d[3] = dv.z, P.d[4] = dv.w;
  P.c[0] = cm1, P.c[1] = cv.x, P.c[2] = cv.y, P.c[3] = cv.z, P.c[4] = cv.w, P.c[5] = c4;
  P.u[0] = uv.x, P.u[1] = uv.y, P.u[2] = uv.z, P.u[3] = uv.w, P.u[4] = u4;
  if (edge) {
    if (edge & ZE_XM) P.d[0] = -1, P.c[0] = -1;
    if (edge & ZE_XP) P.c[5] = -1, P.u[4] = -1;
    if (edge & ZE_YM) {
#pragma unroll
      for (int e = 0; e < 5; e++) P.d[e] = -1;
    }
    if (edge & ZE_YP) {
#pragma unroll
      for (int e = 0; e < 5; e++) P.u[e] = -1;
    }
  }
  if (PTR != PTR_NONE) {
    // pack r*8 + h, h of the cell at strip offset (i, j) = (i + 2j) mod 8
#pragma unroll
    for (int e = 0; e < 5; e++) P.d[e] = P.d[e] * 8 + ((e - 1 - 2 + 8) & 7);
#pragma unroll
    for (int e = 0; e < 6; e++) P.c[e] = P.c[e] * 8 + ((e - 1 + 8) & 7);
#pragma unroll
    for (int e = 0; e < 5; e++) P.u[e] = P.u[e] * 8 + ((e + 2) & 7);
  }
}

__device__ __forceinline__ int smax3(int a, int b, int c) { return __vimax3_s32(a, b, c); }
__device__ __forceinline__ unsigned umin3(unsigned a, unsigned b, unsigned c) { return __vimin3_u32(a, b, c); }

// classify the 4 voxels of plane z (planes: m = z-1, o = z, p = z+1)
template <int PTR>
__device__ __forceinline__ void zreg_plane(const ZPl &m, const ZPl &o, const ZPl &p, int64_t v0, bool store,
                                           const int *__restrict__ lut,
                                           uint8_t *__restrict__ flags, int32_t *__restrict__ ptr) {
  unsigned fl = 0;
  int pv[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int rv = o.c[i + 1];
    // neighbours: plane z (6), z+1 (4), z-1 (4)
    const int a0 = o.c[i + 2], a1 = o.u[i], a2 = o.u[i + 1], a3 = o.c[i], a4 = o.d[i + 1], a5 = o.d[i];
    const int b0 = p.c[i + 1], b1 = p.c[i + 2], b2 = p.u[i], b3 = p.u[i + 1];
    const int c0 = m.c[i + 1], c1 = m.c[i], c2 = m.d[i + 1], c3 = m.d[i];
    bool ismax, ismin;
    if (PTR == PTR_DESC) {
      const unsigned Mp = umin3(umin3(b0, b1, b2), b3, 0xffffffffu);
      const unsigned Mm = umin3(umin3(c0, c1, c2), c3, 0xffffffffu);
      const unsigned M = umin3(umin3(umin3(a0, a1, a2), a3, a4), umin3(a5, Mp, Mm), 0xffffffffu);
      const int X = smax3(smax3(smax3(a0, a1, a2), smax3(a3, a4, a5), smax3(b0, b1, b2)),
                          smax3(b3, c0, c1), smax3(c2, c3, -1));
      ismin = M > (unsigned)rv;
      ismax = X < rv;
      const int pc = M == Mp ? 8 : (M == Mm ? 16 : 0);
      pv[i] = ismin ? 0 : lut[pc + (((int)M - i) & 7)];
    } else if (PTR == PTR_ASC) {
      const int Mp = smax3(smax3(b0, b1, b2), b3, -1);
      const int Mm = smax3(smax3(c0, c1, c2), c3, -1);
      const int M = smax3(smax3(smax3(a0, a1, a2), a3, a4), smax3(a5, Mp, Mm), -1);
      const unsigned X = umin3(umin3(umin3(a0, a1, a2), umin3(a3, a4, a5), umin3(b0, b1, b2)),
                               umin3(b3, c0, c1), umin3(c2, c3, 0xffffffffu));
      ismax = M < rv;
      ismin = X > (unsigned)rv;
      const int pc = M == Mp ? 8 : (M == Mm ? 16 : 0);
      pv[i] = ismax ? 0 : lut[pc + ((M - i) & 7)];
    } else {
      const int M = smax3(smax3(smax3(a0, a1, a2), smax3(a3, a4, a5), smax3(b0, b1, b2)), smax3(b3, c0, c1),
                          smax3(c2, c3, -1));
      const unsigned X = umin3(umin3(umin3(a0, a1, a2), umin3(a3, a4, a5), umin3(b0, b1, b2)),
                               umin3(b3, c0, c1), umin3(c2, c3, 0xffffffffu));
      ismax = M < rv;
      ismin = X > (unsigned)rv;
    }
    fl |= ((ismax ? (unsigned)FL_MAX : 0u) | (ismin ? (unsigned)FL_MIN : 0u)) << (8 * i);
  }
  if (store) {
    if (flags) *reinterpret_cast<uint32_t *>(flags + v0) = fl;
    if (PTR != PTR_NONE) {
      const int v = (int)v0;
      *reinterpret_cast<int4 *>(ptr + v0) = make_int4(v + pv[0], v + 1 + pv[1], v + 2 + pv[2], v + 3 + pv[3]);
    }
  }
}

template <int PTR>
__global__ void __launch_bounds__(CZ_T, LTS_CZ_MINB) k_classify_zreg(const __grid_constant__ CUtensorMap map, Grid g,
                                                                  int zc, uint8_t *__restrict__ flags,
                                                                  int32_t *__restrict__ ptr) {
  extern __shared__ __align__(128) int ring[];  // CZ_RING planes, barriers, offset table
  uint64_t *bar = reinterpret_cast<uint64_t *>(ring + CZ_RING * CZ_SLOT);
  int *lut = reinterpret_cast<int *>(bar + CZ_RING);
  const int tid = threadIdx.x, tx = tid & (CZ_TX - 1), ty = tid / CZ_TX;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t sxy = (int64_t)nx * ny;
  const int x0 = blockIdx.x * CZ_W, y0 = blockIdx.y * CZ_TY;
  const int zb = blockIdx.z * zc, ze = min(nz, zb + zc);
  const int npl = ze - zb + 2;  // planes zb-1 .. ze
  const int x = x0 + 4 * tx, y = y0 + ty;
  auto zin = [&](int j) { return zb - 1 + j >= 0 && zb - 1 + j < nz; };  // plane j inside the grid
  if (tid < 24) {
    // neighbour offset by (plane code, (dx + 2dy) mod 8): plane z, z+1, z-1
    const int s = tid & 7, pc = tid >> 3;
    const int sg = s >= 5 ? -1 : 1, a = s >= 5 ? 8 - s : s;
    const int dz = pc == 1 ? 1 : (pc == 2 ? -1 : 0);
    lut[tid] = sg * ((a & 1) + nx * (a >> 1)) + (int)sxy * dz;
  }
  if (tid == 0) {
    tma_prefetch_desc(&map);
    for (int r = 0; r < CZ_RING; r++) mbar_init(&bar[r], 1);
    fence_mbar_init();
    for (int j = 0; j < min(CZ_RING, npl); j++) {
      if (zin(j)) {
        mbar_expect_tx(&bar[j], CZ_PLANE * 4);
        tma_load_3d(ring + j * CZ_SLOT, &map, &bar[j], x0 - 4, y0 - 1, zb - 1 + j);
      }
    }
  }
  for (int j = 0; j < min(CZ_RING, npl); j++)
    if (!zin(j))
      for (int e = tid; e < CZ_PLANE; e += CZ_T) ring[j * CZ_SLOT + e] = -1;
  unsigned edge = 0;
  if (x == 0) edge |= ZE_XM;
  if (x + 4 >= nx) edge |= ZE_XP;
  if (y == 0) edge |= ZE_YM;
  if (y + 1 >= ny) edge |= ZE_YP;
  const bool store = x < nx && y < ny;
  const int so = (ty + 1) * CZ_BX + 4 * tx + 4;
  __syncthreads();  // barriers initialised, offset table and out-of-grid planes written
  if (tid == 0)
    for (int j = 0; j < min(CZ_RING, npl); j++)
      if (!zin(j)) mbar_arrive(&bar[j]);

  auto fetch = [&](ZPl &P, int j) {  // plane j = z - (zb - 1) into registers
    const int slot = j % CZ_RING;
    mbar_wait(&bar[slot], (unsigned)(j / CZ_RING) & 1u);
    zreg_load<PTR>(P, ring + slot * CZ_SLOT, so, tx, edge);
  };
  auto refill = [&](int j) {  // after a barrier: slot of plane j takes plane j + CZ_RING
    const int jn = j + CZ_RING, slot = j % CZ_RING;
    if (jn >= npl) return;
    if (zin(jn)) {
      if (tid == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar[slot], CZ_PLANE * 4);
        tma_load_3d(ring + slot * CZ_SLOT, &map, &bar[slot], x0 - 4, y0 - 1, zb - 1 + jn);
      }
    } else {  // read after at least one more barrier (CZ_RING > 2)
      for (int e = tid; e < CZ_PLANE; e += CZ_T) ring[slot * CZ_SLOT + e] = -1;
      if (tid == 0) mbar_arrive(&bar[slot]);
    }
  };
  ZPl A, B, C;
  fetch(A, 0);
  fetch(B, 1);
  __syncthreads();
  refill(0);
  refill(1);
  const int cnt = ze - zb;
  int64_t v0 = (int64_t)zb * sxy + (int64_t)y * nx + x;
  auto step = [&](const ZPl &m, const ZPl &o, ZPl &p, int i) {
    fetch(p, i + 2);
    __syncthreads();
    refill(i + 2);
    zreg_plane<PTR>(m, o, p, v0, store, lut, flags, ptr);
    v0 += sxy;
  };
  int i = 0;
  for (; i + 3 <= cnt; i += 3) {
    step(A, B, C, i);
    step(B, C, A, i + 1);
    step(C, A, B, i + 2);
  }
  if (i < cnt) step(A, B, C, i);
  if (i + 1 < cnt) step(B, C, A, i + 1);
}

inline int classify_zreg_zc(const Grid &g) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("LTS_CZ_ZC");
    env = e ? atoi(e) : 0;
  }
  if (env > 0) return env;
  // z-chunk: enough CTAs to fill ~3 resident per SM twice over, chunks >= 8
  const int64_t cols = (int64_t)((g.nx + CZ_W - 1) / CZ_W) * ((g.ny + CZ_TY - 1) / CZ_TY);
  int zc = 64;
  while (zc > 8 && cols * ((g.nz + zc - 1) / zc) < 148 * 3 * 2) zc >>= 1;
  return zc;
}

inline bool launch_classify_zreg(const Grid &g, const int32_t *rank, uint8_t *flags, int32_t *ptr, int ptr_kind,
                                 cudaStream_t s) {
  static int disabled = -1;
  if (disabled < 0) {
    const char *e = getenv("LTS_NO_TMA");
    disabled = e && e[0] == '1';
  }
  if (disabled || g.ndim != 3 || g.n > (int64_t(1) << 28) || (g.nx & 3)) return false;
  CUtensorMap map;
  if (!tma_map_3d_i32(&map, rank, g.nx, g.ny, g.nz, CZ_BX, CZ_BY, 1)) return false;
  const size_t smem = CZ_RING * CZ_SLOT * 4 + CZ_RING * 8 + 24 * 4;
  static int per_sm[3] = {0, 0, 0}, nsm = 0;  // occupancy (set-up once per kernel)
  const int kind = ptr_kind == PTR_ASC ? 1 : (ptr_kind == PTR_DESC ? 2 : 0);
  if (!per_sm[kind]) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    auto setup = [&](const void *fn) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, CZ_T, smem);
      return b > 0 ? b : 1;
    };
    per_sm[kind] = kind == 1 ? setup((const void *)k_classify_zreg<PTR_ASC>)
                   : kind == 2 ? setup((const void *)k_classify_zreg<PTR_DESC>)
                               : setup((const void *)k_classify_zreg<PTR_NONE>);
  }
  const int zc = classify_zreg_zc(g);
  dim3 grd((g.nx + CZ_W - 1) / CZ_W, (g.ny + CZ_TY - 1) / CZ_TY, (g.nz + zc - 1) / zc);
  if (kind == 1) k_classify_zreg<PTR_ASC><<<grd, CZ_T, smem, s>>>(map, g, zc, flags, ptr);
  else if (kind == 2) k_classify_zreg<PTR_DESC><<<grd, CZ_T, smem, s>>>(map, g, zc, flags, ptr);
  else k_classify_zreg<PTR_NONE><<<grd, CZ_T, smem, s>>>(map, g, zc, flags, ptr);
  g_launches++;
  return true;
}

}  // namespace lts
