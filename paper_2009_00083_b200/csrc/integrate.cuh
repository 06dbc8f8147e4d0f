// integrate.cuh -- order integration,
// numeric realization (contract D1), verification and restoration
// (SURVEY A11/A12).
//
// Integration without a sort.  Keys: non-region vertex (rank,0,0); region
// vertex (rank s, local, topseed); saddle (rank s, +inf, +inf).  With
// delta[t] = -1 if the vertex of rank t is claimed, +sum(region sizes) if it is
// a saddle, 0 otherwise, and D = inclusive scan(delta):
//   non-claimed v of rank t:       G = t + D[t]
//   region vertex (local l):       G = t_s + D[t_s] - delta[t_s] + sib(l)
// where sib(l) = l for a region whose saddle is not shared, else
// sum_j min(l, k_j-1) + #{j : top_j < top_r, l <= k_j-2} over the sibling
// regions j sharing the saddle (k_j = size incl. saddle).
#pragma once
#include <math_constants.h>

#include "lts_common.cuh"

namespace lts {

extern int64_t g_launches;

__global__ void k_delta_claimed(const uint32_t *__restrict__ sval, int C, const int *__restrict__ rank,
                                int rev, int n, int *delta) {
  GRID_STRIDE(j, C) delta[eff_rank(rank, (int)sval[j], rev, n)] = -1;
}

__global__ void k_delta_saddles(const int *__restrict__ rsad, const int *__restrict__ rsize, int R,
                                int *delta) {
  GRID_STRIDE(r, R) atomicAdd(delta + rsad[r], rsize[r]);
}

// regions whose saddle is shared: delta[t_s] != own size
__global__ void k_count_shared(const int *__restrict__ rsad, const int *__restrict__ rsize, int R,
                               const int *__restrict__ delta, int *nshared) {
  GRID_STRIDE(r, R) if (delta[rsad[r]] != rsize[r]) atomicAdd(nshared, 1);
}

__device__ __forceinline__ void write_g(int v, int gp, int rev, int n, int *G, int *Ginv) {
  int gr = rev ? (n - 1 - gp) : gp;
  G[v] = gr;
  Ginv[gr] = v;
}

// rank order: inverse and prefix are read coalesced, the claimed test is a
// bit-set probe, new inverses land in ascending (coalesced) order
__global__ void k_integrate_plain(const int *__restrict__ inv, int rev, int n,
                                  const uint32_t *__restrict__ cbits, const int *__restrict__ D,
                                  int *G, int *Ginv) {
  GRID_STRIDE(t, n) {
    int v = inv[rev ? (n - 1 - t) : t];
    if ((__ldg(cbits + (v >> 5)) >> (v & 31)) & 1u) continue;
    write_g(v, (int)t + D[t], rev, n, G, Ginv);
  }
}

// sorted sibling groups: sib_rid sorted by saddle rank (stable), pos_of[rid].
// Every region sharing a saddle holds one of the saddle's neighbours, so a
// group has at most K members (14 on grids, 16 on meshes): the loop is O(K).
__device__ __forceinline__ int sib_offset(int l, int rid, int top_r, const int *rsad,
                                          const int *rsize, const int *rtop, const int *sib_rid,
                                          const int *pos_of, int R) {
  int p = pos_of[rid];
  int ts = rsad[rid];
  int a = p;
  while (a > 0 && rsad[sib_rid[a - 1]] == ts) a--;
  int acc = 0;
  for (int i = a; i < R; i++) {
    int j = sib_rid[i];
    if (rsad[j] != ts) break;
    int kj = rsize[j] + 1;
    acc += l < kj - 1 ? l : kj - 1;
    if (j != rid && rtop[j] < top_r && l <= kj - 2) acc++;
  }
  return acc;
}

__global__ void k_integrate_regions(const uint32_t *__restrict__ skey, const uint32_t *__restrict__ sval,
                                    int C, const int *__restrict__ rptr, const int *__restrict__ local,
                                    const int *__restrict__ rsad, const int *__restrict__ rsize,
                                    const int *__restrict__ rtop, const int *__restrict__ delta,
                                    const int *__restrict__ D, const int *__restrict__ sib_rid,
                                    const int *__restrict__ pos_of, int R, int shared, int rev,
                                    int n, int *G, int *Ginv) {
  GRID_STRIDE(j, C) {
    int rid = (int)skey[j];
    int v = (int)sval[j];
    int slot = (int)j + rid + 1;
    int l = local[slot];
    int ts = rsad[rid];
    int base = ts + D[ts] - delta[ts];
    int off = l;
    if (shared && delta[ts] != rsize[rid])
      off = sib_offset(l, rid, rtop[rid], rsad, rsize, rtop, sib_rid, pos_of, R);
    write_g(v, base + off, rev, n, G, Ginv);
  }
}

__global__ void k_pos_of(const uint32_t *__restrict__ sorted_rid, int R, int *sib_rid, int *pos_of) {
  GRID_STRIDE(i, R) {
    int r = (int)sorted_rid[i];
    sib_rid[i] = r;
    pos_of[r] = (int)i;
  }
}

// contract D1: every claimed vertex takes its region saddle's value (the
// saddle is never claimed in its own pass, so the update is in place)
__global__ void k_realize(const uint32_t *__restrict__ skey, const uint32_t *__restrict__ sval, int C,
                          const int *__restrict__ rptr, const int *__restrict__ verts, float *g) {
  GRID_STRIDE(j, C) {
    int rid = (int)skey[j];
    int s = verts[rptr[rid]];
    g[sval[j]] = g[s];
  }
}

// g = f with -0.0 canonicalised to +0.0 (D10); copies preserve the sign bit
__global__ void k_copy_canon(const float *__restrict__ f, float *g, int64_t n) {
  GRID_STRIDE(i, n) {
    float x = f[i];
    g[i] = x == 0.0f ? 0.0f : x;
  }
}

// verify_constraints: counts [extra_max, lost_max,
// extra_min, lost_min]
__global__ void k_verify(const uint8_t *__restrict__ flags, const uint8_t *__restrict__ pmark,
                         int64_t n, int *cnt) {
  GRID_STRIDE(v, n) {
    uint8_t f = flags[v], p = pmark[v];
    bool ismax = f & FL_MAX, ismin = f & FL_MIN;
    bool pmax = p & PM_MAX, pmin = p & PM_MIN;
    int e0 = ismax && !pmax, e1 = pmax && !ismax, e2 = ismin && !pmin, e3 = pmin && !ismin;
    unsigned act = __activemask();
    unsigned b0 = __ballot_sync(act, e0), b1 = __ballot_sync(act, e1);
    unsigned b2 = __ballot_sync(act, e2), b3 = __ballot_sync(act, e3);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
      if (b0) atomicAdd(cnt + 0, __popc(b0));
      if (b1) atomicAdd(cnt + 1, __popc(b1));
      if (b2) atomicAdd(cnt + 2, __popc(b2));
      if (b3) atomicAdd(cnt + 3, __popc(b3));
    }
  }
}

// lost preserved extrema (kind 0 minima, 1 maxima) -> list (unordered)
__global__ void k_lost(const uint8_t *__restrict__ flags, const uint8_t *__restrict__ pmark,
                       int64_t n, int kind, int *list, int *count) {
  GRID_STRIDE(v, n) {
    bool lost = kind == 0 ? ((pmark[v] & PM_MIN) && !(flags[v] & FL_MIN))
                          : ((pmark[v] & PM_MAX) && !(flags[v] & FL_MAX));
    if (lost) list[atomicAdd(count, 1)] = (int)v;
  }
}

// restore one lost extremum x (D6): target rank of the lowest (highest)
// neighbour; scal[0] = rx, scal[1] = ry, scal[2] = apply
template <int NDIM>
__global__ void k_restore_target(Grid g, const int *__restrict__ rank, int x, int kind, int *scal) {
  constexpr int K = KOf<NDIM>::value;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Nb<NDIM> nb(g, x);
  int rx = rank[x];
  int ry = kind == 0 ? 0x7fffffff : -1;
  for (int k = 0; k < K; k++) {
    int u = nb(g, k);
    if (u < 0) continue;
    int ru = rank[u];
    if (kind == 0 ? ru < ry : ru > ry) ry = ru;
  }
  scal[0] = rx;
  scal[1] = ry;
  scal[2] = kind == 0 ? (ry < rx) : (ry > rx);
}

__global__ void k_restore_shift(int *rank, int64_t n, int x, int kind, const int *__restrict__ scal) {
  if (!scal[2]) return;
  int rx = scal[0], ry = scal[1];
  GRID_STRIDE(v, n) {
    int r = rank[v];
    if (v == x) {
      rank[v] = ry;
    } else if (kind == 0) {
      if (r >= ry && r < rx) rank[v] = r + 1;
    } else {
      if (r > rx && r <= ry) rank[v] = r - 1;
    }
  }
}

// Literal realize_sweep (reference _kernels.py:84-99) in float64: walk the
// order from the top; a vertex that violates it under (value, id)
// tie-breaking takes g[prev] - zeta (nextafter(g[prev], -inf) when that does
// not decrease).  Inherently sequential: one CTA, the values of a chunk of
// RZ_C positions gathered in parallel into shared memory, the chain run by
// thread 0 over the chunk, the results scattered back in parallel.
constexpr int RZ_T = 256, RZ_C = 2048;

__global__ void __launch_bounds__(RZ_T) k_realize_sweep(double *g, const int *__restrict__ inverse, int64_t n,
                                                        double zeta) {
  __shared__ double s_val[RZ_C];
  __shared__ int s_id[RZ_C];
  __shared__ double s_prev_val;
  __shared__ int s_prev;
  if (threadIdx.x == 0) {
    s_prev = inverse[n - 1];
    s_prev_val = g[s_prev];
  }
  // positions n-2 .. 0 in chunks, top chunk first
  for (int64_t hi = n - 2; hi >= 0; hi -= RZ_C) {
    const int64_t lo = hi - RZ_C + 1 > 0 ? hi - RZ_C + 1 : 0;
    const int cnt = (int)(hi - lo + 1);
    for (int j = threadIdx.x; j < cnt; j += RZ_T) {  // j = 0 is position hi
      const int v = inverse[hi - j];
      s_id[j] = v;
      s_val[j] = g[v];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int prev = s_prev;
      double pv = s_prev_val;
      for (int j = 0; j < cnt; j++) {
        const int v = s_id[j];
        double x = s_val[j];
        if (x > pv || (x == pv && v > prev)) {
          double nv = pv - zeta;
          if (nv >= pv) nv = nextafter(pv, -CUDART_INF);
          x = nv;
          s_val[j] = x;
        }
        prev = v;
        pv = x;
      }
      s_prev = prev;
      s_prev_val = pv;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += RZ_T) g[s_id[j]] = s_val[j];
    __syncthreads();
  }
}

}  // namespace lts
