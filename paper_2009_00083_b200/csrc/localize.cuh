// localize.cuh -- localized simplification of every region (reference
// localize_regions / _localize_one, _kernels.py:424-591).
//
// One warp per region, regions claimed largest-first from an atomic queue so
// the long floods start early and the many small regions fill in behind them.
// Within a region the alternating descending / ascending priority floods are
// exact (distinct keys, unique extraction order): lane 0 owns a binary heap
// (shared memory for small regions, the region's slice of a global scratch heap
// otherwise) while the lanes resolve the <=14 stencil neighbours of each
// extracted vertex in parallel (membership: region id + local index maps).
// Period-2 cycles are detected by comparing the state after flood t
// with the state after flood t-2 and jumping straight to the capped state, which
// is bit-identical to running the remaining floods (contract D5).
#pragma once
#include "lts_common.cuh"

namespace lts {

extern int64_t g_launches;

constexpr int LOC_WARPS = 4;                 // warps per block
constexpr int LOC_SMEM_HEAP = 1024;          // heap entries per warp in smem
constexpr uint8_t SF_INHEAP = 1, SF_OUT = 2, SF_MIN = 4;

struct LocArgs {
  Grid g;
  const int *rank;
  int rev;
  const int *order;   // regions, largest first
  int R;
  const int *rptr;    // R+1 slot offsets
  const int *verts;   // slots: vertex ids, saddle first
  const int *slot_of;  // vertex -> its slot in `verts` (claimed vertices), -1 otherwise
  int *buf0, *buf1, *buf2;  // slot arrays: rotating flood states
  int *out;                 // slot array: final local order
  unsigned long long *gheap;  // slot array: global heap scratch
  uint8_t *sfl;             // slot array: flags
  int *n_iters, *status;
  int max_iter;
  int *queue;
  int qbase;          // first entry of `order` handled by this launch
};

__device__ __forceinline__ void heap_push(unsigned long long *h, int &size, unsigned long long x) {
  int i = size++;
  while (i > 0) {
    int p = (i - 1) >> 1;
    unsigned long long y = h[p];
    if ((long long)y >= (long long)x) break;
    h[i] = y;
    i = p;
  }
  h[i] = x;
}

__device__ __forceinline__ unsigned long long heap_pop(unsigned long long *h, int &size) {
  unsigned long long top = h[0];
  size--;
  if (size > 0) {
    unsigned long long x = h[size];
    int i = 0;
    for (;;) {
      int l = 2 * i + 1;
      if (l >= size) break;
      int b = l;
      unsigned long long yl = h[l];
      if (l + 1 < size) {
        unsigned long long yr = h[l + 1];
        if ((long long)yr > (long long)yl) {
          b = l + 1;
          yl = yr;
        }
      }
      if ((long long)x >= (long long)yl) break;
      h[i] = yl;
      i = b;
    }
    h[i] = x;
  }
  return top;
}

__device__ __forceinline__ unsigned long long hkey(int key, int p) {
  return ((unsigned long long)(unsigned)key << 32) | (unsigned)p;
}

// local index of vertex u within the region of slots [lo, lo + k) (saddle s at
// index 0), or -1: one read of the vertex's global slot (k_place)
__device__ __forceinline__ int member(const LocArgs &A, int u, int lo, int k, int s) {
  if (u < 0) return -1;
  if (u == s) return 0;
  const int d = A.slot_of[u] - lo;
  return d > 0 && d < k ? d : -1;
}

// One exact priority flood.  desc: source = saddle, max-key first, label
// k-1-e.  asc: sources = admissible minima (SF_MIN & SF_OUT), min-key first,
// label e.  cin/cout: slot arrays of this region (already offset).
template <int NDIM>
__device__ void flood(const LocArgs &A, bool asc, int rid, int s, int k, const int *verts,
                      const int *cin, int *cout, uint8_t *sfl, unsigned long long *heap) {
  constexpr int K = KOf<NDIM>::value;
  const int lane = threadIdx.x & 31;
  for (int p = lane; p < k; p += 32) sfl[p] &= (uint8_t)~SF_INHEAP;
  __syncwarp();
  int size = 0;
  if (!asc) {
    if (lane == 0) {
      heap_push(heap, size, hkey(cin[0], 0));
      sfl[0] |= SF_INHEAP;
    }
  } else {
    for (int p0 = 1; p0 < k; p0 += 32) {
      int p = p0 + lane;
      bool src = p < k && (sfl[p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT);
      unsigned m = __ballot_sync(0xffffffffu, src);
      int key = src ? -cin[p] : 0;
      if (src) sfl[p] |= SF_INHEAP;
      while (m) {
        int b = __ffs(m) - 1;
        m &= m - 1;
        int kb = __shfl_sync(0xffffffffu, key, b);
        if (lane == 0) heap_push(heap, size, hkey(kb, p0 + b));
      }
    }
    // no admissible minimum: the reference's flood extracts nothing and its
    // label buffer keeps the previous flood's output (_kernels.py:531-552)
    if (__shfl_sync(0xffffffffu, size, 0) == 0)
      for (int p = lane; p < k; p += 32) cout[p] = cin[p];
  }
  __syncwarp();
  int e = 0;
  for (;;) {
    int p = -1;
    if (lane == 0 && size > 0) p = (int)(unsigned)(heap_pop(heap, size) & 0xffffffffull);
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p < 0) break;
    if (lane == 0) cout[p] = asc ? e : (k - 1 - e);
    e++;
    int v = verts[p];
    int q = -1, key = 0;
    if (lane < K) {
      const Nb<NDIM> nb(A.g, v);
      int u = nb(A.g, lane);
      q = member(A, u, (int)(verts - A.verts), k, s);
      if (q >= 0) {
        if (sfl[q] & SF_INHEAP) {
          q = -1;
        } else {
          sfl[q] |= SF_INHEAP;
          key = asc ? -cin[q] : cin[q];
        }
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, q >= 0);
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      int kb = __shfl_sync(0xffffffffu, key, b);
      int qb = __shfl_sync(0xffffffffu, q, b);
      if (lane == 0) heap_push(heap, size, hkey(kb, qb));
    }
    __syncwarp();
  }
  __syncwarp();
}

// after a descending flood: marks local minima (SF_MIN); returns true if an
// unauthorized minimum (no outside neighbour) exists (_kernels.py:512-526)
template <int NDIM>
__device__ bool check_minima(const LocArgs &A, int rid, int s, int k, const int *verts,
                             const int *cur, uint8_t *sfl) {
  constexpr int K = KOf<NDIM>::value;
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int p = 1 + lane; p < k; p += 32) {
    int v = verts[p];
    const Nb<NDIM> nb(A.g, v);
    int c = cur[p];
    bool mn = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = member(A, nb(A.g, kk), (int)(verts - A.verts), k, s);
      if (q >= 0 && cur[q] < c) {
        mn = false;
        break;
      }
    }
    uint8_t f = sfl[p];
    f = mn ? (f | SF_MIN) : (f & (uint8_t)~SF_MIN);
    sfl[p] = f;
    if (mn && !(f & SF_OUT)) bad = true;
  }
  return __any_sync(0xffffffffu, bad);
}

// after an ascending flood: true if some vertex other than the saddle is a
// local maximum (_kernels.py:554-568)
template <int NDIM>
__device__ bool check_maxima(const LocArgs &A, int rid, int s, int k, const int *verts,
                             const int *cur) {
  constexpr int K = KOf<NDIM>::value;
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int p = 1 + lane; p < k; p += 32) {
    int v = verts[p];
    const Nb<NDIM> nb(A.g, v);
    int c = cur[p];
    bool mx = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = member(A, nb(A.g, kk), (int)(verts - A.verts), k, s);
      if (q >= 0 && cur[q] > c) {
        mx = false;
        break;
      }
    }
    if (mx) bad = true;
  }
  return __any_sync(0xffffffffu, bad);
}

__device__ __forceinline__ bool states_equal(const int *a, const int *b, int k) {
  const int lane = threadIdx.x & 31;
  bool diff = false;
  for (int p = lane; p < k; p += 32)
    if (a[p] != b[p]) diff = true;
  return !__any_sync(0xffffffffu, diff);
}

template <int NDIM>
__global__ void __launch_bounds__(32 * LOC_WARPS) k_localize(LocArgs A) {
  constexpr int K = KOf<NDIM>::value;
  __shared__ unsigned long long s_heap[LOC_WARPS][LOC_SMEM_HEAP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = (int)A.g.n;
  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(A.queue, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi + A.qbase >= A.R) break;
    const int rid = A.order[A.qbase + qi];
    const int lo = A.rptr[rid];
    const int k = A.rptr[rid + 1] - lo;
    const int *verts = A.verts + lo;
    uint8_t *sfl = A.sfl + lo;
    int *bufs[3] = {A.buf0 + lo, A.buf1 + lo, A.buf2 + lo};
    unsigned long long *heap = k <= LOC_SMEM_HEAP ? s_heap[w] : A.gheap + lo;
    const int s = verts[0];
    const int srank = eff_rank(A.rank, s, A.rev, n);
    // has_outside: a neighbour below the saddle (_kernels.py:460-468)
    int v0 = 0x7fffffff;
    for (int p = lane; p < k; p += 32) {
      bool out = false;
      if (p >= 1) {
        const Nb<NDIM> nb(A.g, verts[p]);
#pragma unroll
        for (int kk = 0; kk < K; kk++) {
          int u = nb(A.g, kk);
          if (u >= 0 && eff_rank(A.rank, u, A.rev, n) < srank) {
            out = true;
            break;
          }
        }
      }
      sfl[p] = out ? SF_OUT : 0;
      if (out && p < v0) v0 = p;
      bufs[0][p] = p;
    }
    v0 = __reduce_min_sync(0xffffffffu, v0);
    __syncwarp();
    if (v0 == 0x7fffffff) {  // no admissible boundary minimum (status 1)
      if (lane == 0) {
        A.status[rid] = 1;
        A.n_iters[rid] = 0;
      }
      for (int p = lane; p < k; p += 32) A.out[lo + p] = p;
      continue;
    }
    if (lane == 0) {
      bufs[0][0] = 0x7fffffff;   //  BIG
      bufs[0][v0] = (int)0x80000000;  // -BIG
    }
    __syncwarp();
    int t = 0, status = 0, fin = 0;
    for (;;) {
      // descending flood from the saddle
      flood<NDIM>(A, false, rid, s, k, verts, bufs[t % 3], bufs[(t + 1) % 3], sfl, heap);
      t++;
      bool bad = check_minima<NDIM>(A, rid, s, k, verts, bufs[t % 3], sfl);
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && states_equal(bufs[t % 3], bufs[(t + 1) % 3], k)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
      // ascending flood from the admissible minima
      flood<NDIM>(A, true, rid, s, k, verts, bufs[t % 3], bufs[(t + 1) % 3], sfl, heap);
      t++;
      bad = check_maxima<NDIM>(A, rid, s, k, verts, bufs[t % 3]);
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && states_equal(bufs[t % 3], bufs[(t + 1) % 3], k)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
    }
    const int *fb = bufs[fin % 3];
    for (int p = lane; p < k; p += 32) A.out[lo + p] = fb[p];
    if (lane == 0) {
      A.status[rid] = status;
      A.n_iters[rid] = t;
    }
    __syncwarp();
  }
}

}  // namespace lts
