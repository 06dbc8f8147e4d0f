// classify_2d.cuh -- extremum flags (and steepest pointers) of a 2-D grid.
//
// The 2-D Freudenthal stencil has six neighbours (reference
// triangulation.py:32-38): (1,0) (0,1) (1,1) (-1,0) (0,-1) (-1,-1).  A CTA of
// 32 x 8 threads owns a 128 x 32 tile: the ranks of the tile and its one-pixel
// halo are staged in shared memory with 16-byte loads (rows of the grid are
// contiguous, so every load is a full sector), each thread then classifies a
// 4-pixel strip of four consecutive rows, sliding three rows through
// registers.  Flags leave as one 32-bit store per strip, pointers as one
// 128-bit store.  Semantics are those of the tile kernel (classify.cuh):
// out-of-grid neighbours hold -1, never the signed maximum and always the
// unsigned maximum; the pointer of a vertex is itself at an extremum of its
// kind, else its highest (PTR_ASC) / lowest (PTR_DESC) neighbour.
// HBM-bound: 4 B read and 1 B (flags) + 4 B (pointer) written per pixel.
#pragma once
#include "classify.cuh"

namespace lts {

constexpr int C2_TX = 32, C2_TY = 8, C2_RY = 4;
constexpr int C2_W = 4 * C2_TX, C2_H = C2_TY * C2_RY;  // 128 x 32 tile
constexpr int C2_PITCH = C2_W + 8;                      // [x0-4 .. x0+131]
constexpr int C2_ROWS = C2_H + 2;

struct C2Row {
  int c[6];  // x-1 .. x+4
};

__device__ __forceinline__ void c2_load(C2Row &R, const int *row, int col) {
  const int4 v = *reinterpret_cast<const int4 *>(row + col);
  R.c[0] = row[col - 1];
  R.c[1] = v.x;
  R.c[2] = v.y;
  R.c[3] = v.z;
  R.c[4] = v.w;
  R.c[5] = row[col + 4];
}

template <int PTR>
__global__ void __launch_bounds__(C2_TX * C2_TY) k_classify_2d(Grid g, const int32_t *__restrict__ rank,
                                                              uint8_t *__restrict__ flags,
                                                              int32_t *__restrict__ ptr) {
  __shared__ __align__(16) int sm[C2_ROWS][C2_PITCH];
  const int nx = g.nx, ny = g.ny;
  const int x0 = blockIdx.x * C2_W, y0 = blockIdx.y * C2_H;
  const int tid = threadIdx.y * C2_TX + threadIdx.x;
  constexpr int G4 = C2_PITCH / 4;  // 16-byte groups per staged row
  for (int i = tid; i < C2_ROWS * G4; i += C2_TX * C2_TY) {
    const int r = i / G4, q = i - r * G4;
    const int gy = y0 - 1 + r, gx = x0 - 4 + 4 * q;
    int4 v = make_int4(-1, -1, -1, -1);
    if (gy >= 0 && gy < ny && gx >= 0 && gx < nx) v = *reinterpret_cast<const int4 *>(rank + (int64_t)gy * nx + gx);
    *reinterpret_cast<int4 *>(&sm[r][4 * q]) = v;
  }
  __syncthreads();
  const int x = x0 + 4 * threadIdx.x;
  const int col = 4 + 4 * threadIdx.x;
  const int yb = y0 + C2_RY * threadIdx.y;
  if (x >= nx) return;
  C2Row D, C, U;
  c2_load(D, sm[C2_RY * threadIdx.y], col);
  c2_load(C, sm[C2_RY * threadIdx.y + 1], col);
#pragma unroll
  for (int j = 0; j < C2_RY; j++) {
    const int y = yb + j;
    c2_load(U, sm[C2_RY * threadIdx.y + j + 2], col);
    if (y < ny) {
      unsigned fl = 0;
      int pv[4];
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int rv = C.c[i + 1];
        // reference offset order: (1,0) (0,1) (1,1) (-1,0) (0,-1) (-1,-1)
        int a0 = C.c[i + 2], a1 = U.c[i + 1], a2 = U.c[i + 2], a3 = C.c[i], a4 = D.c[i + 1], a5 = D.c[i];
        bool ismax, ismin;
        if (PTR == PTR_NONE) {
          const int hi = __vimax3_s32(__vimax3_s32(a0, a1, a2), __vimax3_s32(a3, a4, a5), -1);
          const unsigned lo = __vimin3_u32(__vimin3_u32((unsigned)a0, (unsigned)a1, (unsigned)a2),
                                           __vimin3_u32((unsigned)a3, (unsigned)a4, (unsigned)a5), 0xffffffffu);
          ismax = hi < rv;
          ismin = lo > (unsigned)rv;
        } else {
          // packed (rank << 3 | slot): ranks stay below 2^27 (n <= 2^27)
          const int p0 = a0 < 0 ? -1 : (a0 << 3), p1 = a1 < 0 ? -1 : ((a1 << 3) | 1),
                    p2 = a2 < 0 ? -1 : ((a2 << 3) | 2), p3 = a3 < 0 ? -1 : ((a3 << 3) | 3),
                    p4 = a4 < 0 ? -1 : ((a4 << 3) | 4), p5 = a5 < 0 ? -1 : ((a5 << 3) | 5);
          const int hi = __vimax3_s32(__vimax3_s32(p0, p1, p2), __vimax3_s32(p3, p4, p5), -1);
          const unsigned lo = __vimin3_u32(__vimin3_u32((unsigned)p0, (unsigned)p1, (unsigned)p2),
                                           __vimin3_u32((unsigned)p3, (unsigned)p4, (unsigned)p5), 0xffffffffu);
          ismax = (hi < 0 ? -1 : (hi >> 3)) < rv;
          ismin = (lo == 0xffffffffu ? lo : (lo >> 3)) > (unsigned)rv;
          const bool self = PTR == PTR_ASC ? ismax : ismin;
          const int kb = PTR == PTR_ASC ? (hi & 7) : (int)(lo & 7u);
          // slot -> offset: +1, +nx, +nx+1, -1, -nx, -nx-1
          const int sg = kb >= 3 ? -1 : 1, ka = kb >= 3 ? kb - 3 : kb;
          const int d = sg * ((ka != 1 ? 1 : 0) + (ka != 0 ? nx : 0));
          pv[i] = self ? 0 : d;
        }
        fl |= ((ismax ? (unsigned)FL_MAX : 0u) | (ismin ? (unsigned)FL_MIN : 0u)) << (8 * i);
      }
      const int64_t v0 = (int64_t)y * nx + x;
      if (flags) *reinterpret_cast<uint32_t *>(flags + v0) = fl;
      if (PTR != PTR_NONE) {
        const int v = (int)v0;
        *reinterpret_cast<int4 *>(ptr + v0) = make_int4(v + pv[0], v + 1 + pv[1], v + 2 + pv[2], v + 3 + pv[3]);
      }
    }
    D = C;
    C = U;
  }
}

// 2-D grids of a million pixels or more (smaller ones do not fill the GPU
// with 128 x 32 tiles; the pair kernel is faster there), rows a multiple of
// four pixels, 16-byte aligned arrays
inline bool launch_classify_2d(const Grid &g, const int32_t *rank, uint8_t *flags, int32_t *ptr, int ptr_kind,
                               cudaStream_t s) {
  if (g.ndim != 2 || (g.nx & 3) || g.n > (int64_t(1) << 27) || g.n < (int64_t(1) << 20)) return false;
  if (((uintptr_t)rank & 15) || ((uintptr_t)flags & 3) || ((uintptr_t)ptr & 15)) return false;
  dim3 blk(C2_TX, C2_TY), grd((g.nx + C2_W - 1) / C2_W, (g.ny + C2_H - 1) / C2_H);
  if (ptr_kind == PTR_ASC) k_classify_2d<PTR_ASC><<<grd, blk, 0, s>>>(g, rank, flags, ptr);
  else if (ptr_kind == PTR_DESC) k_classify_2d<PTR_DESC><<<grd, blk, 0, s>>>(g, rank, flags, ptr);
  else k_classify_2d<PTR_NONE><<<grd, blk, 0, s>>>(g, rank, flags, ptr);
  g_launches++;
  return true;
}

}  // namespace lts
