// prims.cuh -- device-wide scan and small utility kernels.
#pragma once
#include "lts_common.cuh"

namespace lts {

extern int64_t g_launches;

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_IPT;

__device__ __forceinline__ int block_scan_excl_int(int x, int *s_w, int *total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? s_w[lane] : 0;
    int ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < nw) s_w[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  int r = s_w[w] + inc - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const int *__restrict__ in, int64_t n,
                                                              int *bsum) {
  __shared__ int s_w[32];
  __shared__ int s_tot;
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int acc = 0;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; j++) {
    int64_t i = base + j * SCAN_THREADS + threadIdx.x;
    if (i < n) acc += in[i];
  }
  block_scan_excl_int(acc, s_w, &s_tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s_tot;
}

__global__ void __launch_bounds__(1024) k_scan_bsums(int *bsum, int nb, int *total_out) {
  __shared__ int s_w[32];
  __shared__ int s_tot;
  int carry = 0;
  for (int c = 0; c < nb; c += 1024) {
    int i = c + threadIdx.x;
    int x = i < nb ? bsum[i] : 0;
    int e = block_scan_excl_int(x, s_w, &s_tot);
    if (i < nb) bsum[i] = carry + e;
    carry += s_tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// out[i] = exclusive (or inclusive) prefix sum of in; in and out may alias.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(const int *in, int *out, int64_t n,
                                                            const int *__restrict__ bsum,
                                                            int inclusive) {
  __shared__ int s_w[32];
  __shared__ int s_tot;
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  int x[SCAN_IPT];
  int acc = 0;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; j++) {
    int64_t i = base + j;
    x[j] = i < n ? in[i] : 0;
    acc += x[j];
  }
  int e = block_scan_excl_int(acc, s_w, &s_tot) + bsum[blockIdx.x];
#pragma unroll
  for (int j = 0; j < SCAN_IPT; j++) {
    int64_t i = base + j;
    int nx = e + x[j];
    if (i < n) out[i] = inclusive ? nx : e;
    e = nx;
  }
}

// exclusive/inclusive scan with the grand total written to *total (device)
inline int scan_int(const int *in, int *out, int64_t n, int *bsum, int *total, bool inclusive,
                    cudaStream_t s) {
  if (n <= 0) {
    if (total) LTS_CUDA(cudaMemsetAsync(total, 0, sizeof(int), s));
    return 0;
  }
  int nb = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
  k_scan_reduce<<<nb, SCAN_THREADS, 0, s>>>(in, n, bsum);
  k_scan_bsums<<<1, 1024, 0, s>>>(bsum, nb, total);
  k_scan_down<<<nb, SCAN_THREADS, 0, s>>>(in, out, n, bsum, inclusive ? 1 : 0);
  g_launches += 3;
  return 0;
}

__global__ void k_fill_int(int *a, int64_t n, int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void k_iota(int *a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

__global__ void k_int_to_i64(const int *a, int64_t *b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// inverse[rank[v]] = v (order_from_ranks, reference order.py:94-99)
__global__ void k_scatter_inverse(const int *__restrict__ rank, int *inverse, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    inverse[rank[v]] = (int)v;
}

// order_from_ranks with validation: inverse must be pre-filled with -1; a rank
// outside [0, n) or a rank taken twice (so `rank` is not a bijection) sets *bad
__global__ void k_scatter_inverse_checked(const int *__restrict__ rank, int *inverse, int64_t n, int *bad) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int r = rank[v];
    if (r < 0 || (int64_t)r >= n) {
      atomicOr(bad, 1);
      continue;
    }
    if (atomicExch(inverse + r, (int)v) != -1) atomicOr(bad, 1);
  }
}

// ScalarField finiteness (reference order.py:35-36) for callers that bring
// their own order field: NaN or +-inf sets *bad
__global__ void k_nonfinite(const float *__restrict__ f, int64_t n, int *bad) {
  bool b = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b |= (__float_as_uint(f[i]) & 0x7f800000u) == 0x7f800000u;
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

}  // namespace lts
