// lts_common.cuh -- shared device helpers for the sm_100a LTS path.
//
// Grid conventions follow the reference (triangulation.py:8): vertex ids are
// x-fastest, id = x + nx*(y + ny*z); the Freudenthal stencil is the
// reference's offset table (triangulation.py:32-45): 6 neighbours in 2D, 14 in
// 3D, clipped at the boundary.  Vertex ids and ranks are int32 on the device
// (SURVEY D11); every config has n < 2^31.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lts_sm100.h"

#define LTS_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return lts_set_cuda_error(e_, #call, __FILE__, __LINE__); \
  } while (0)

int lts_set_cuda_error(cudaError_t e, const char *what, const char *file, int line);
int lts_set_error(int code, const char *msg);

#define GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

namespace lts {

constexpr int kMaxK = 14;
constexpr uint8_t FL_MIN = 1;   // no lower neighbour  (lower link empty)
constexpr uint8_t FL_MAX = 2;   // no upper neighbour  (upper link empty)
constexpr uint8_t PM_MIN = 1;   // preserved minimum mark
constexpr uint8_t PM_MAX = 2;   // preserved maximum mark

// The mesh: a regular 2D/3D Freudenthal grid (ndim 2/3, implicit stencil) or
// an explicit triangle mesh (ndim 0: symmetric CSR adjacency cptr/cidx, as the
// reference's Triangulation.indptr/indices, triangulation.py:81-125).
struct Grid {
  int nx, ny, nz;  // nz == 1 in 2D; explicit mesh: nx = n, ny = nz = 1
  int ndim, K;
  int64_t n;
  const int *cptr, *cidx;  // explicit mesh only
};

// stencil offsets, x/y/z per neighbour (reference triangulation.py:32-45)
__constant__ int8_t c_off[3][kMaxK];  // single translation unit (unity build)

__device__ __forceinline__ void coords(const Grid &g, int v, int &x, int &y, int &z) {
  x = v % g.nx;
  int r = v / g.nx;
  y = r % g.ny;
  z = r / g.ny;
}

// neighbour k of (x,y,z) or -1 if clipped
__device__ __forceinline__ int nbr_at(const Grid &g, int x, int y, int z, int k) {
  int a = x + c_off[0][k], b = y + c_off[1][k], c = z + c_off[2][k];
  if ((unsigned)a >= (unsigned)g.nx || (unsigned)b >= (unsigned)g.ny || (unsigned)c >= (unsigned)g.nz)
    return -1;
  return a + g.nx * (b + g.ny * c);
}

#ifndef LTS_CSR_K
#define LTS_CSR_K 16
#endif
constexpr int kCsrK = LTS_CSR_K;  // largest vertex degree of explicit meshes

// neighbour slots per vertex: 6 / 14 grid stencil entries, kCsrK CSR entries
template <int NDIM>
struct KOf {
  static constexpr int value = NDIM == 2 ? 6 : (NDIM == 3 ? 14 : kCsrK);
};

// the neighbours of one vertex, slot k = 0..K-1 (-1: no neighbour in that slot)
template <int NDIM>
struct Nb {
  int a, b, c;  // grid: x, y, z; explicit mesh: row start, degree
  __device__ __forceinline__ Nb(const Grid &g, int v) {
    if (NDIM == 0) {
      a = g.cptr[v];
      b = g.cptr[v + 1] - a;
      c = 0;
    } else {
      coords(g, v, a, b, c);
    }
  }
  __device__ __forceinline__ int operator()(const Grid &g, int k) const {
    if (NDIM == 0) return k < b ? g.cidx[a + k] : -1;
    return nbr_at(g, a, b, c, k);
  }
};

// effective rank of the current pass: the minima pass runs the maxima
// machinery on the reversed order n-1-rank (reference order.py:54-56)
__device__ __forceinline__ int eff_rank(const int *rank, int v, int rev, int n) {
  int r = rank[v];
  return rev ? (n - 1 - r) : r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// warp-aggregated atomic increment; returns this lane's slot
__device__ __forceinline__ int warp_alloc(int *counter, bool want) {
  unsigned m = __ballot_sync(__activemask(), want);
  if (!want) return -1;
  int leader = __ffs(m) - 1;
  int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(m, base, leader);
  return base + __popc(m & lanemask_lt());
}

inline int grid_blocks(int64_t n, int threads, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

}  // namespace lts
