// discover.cuh -- region discovery (reference discover_sweep, _kernels.py:194-303)
// as a schedule-free data-parallel computation.
//
// The reference sweeps one global max-heap; its result is characterised
// exactly: v is CLAIMED iff the component of
// {u : rank u >= rank v} that contains v has all its maxima in the seed set D;
// regions are the connected components of claimed vertices; a region's saddle
// is its highest unclaimed neighbour; topseed is its highest rank.
//
// B200 formulation (no priority queue, no sequential sweep):
//  1. steepest-ascent forest (fused into classification) compressed to the
//     ascending-manifold maximum M(v) of every vertex;
//  2. cross-manifold edges (a=M(u), b=M(v), w=min(rank u, rank v)) form the
//     maxima graph; the join-tree connectivity of superlevel sets equals its
//     connectivity through edges of weight >= t;
//  3. tau(m) = bottleneck from maximum m to a preserved maximum, computed by
//     Boruvka rounds: every non-preserved component hooks along its heaviest
//     edge; chains reaching preserved territory are final (tau = edge weight,
//     non-decreasing along the chain), chains ending in 2-cycles contract;
//  4. claimed(v) <=> M(v) in D and rank v > tau(M(v)); saddle = vertex of
//     rank tau; regions = union-find over edges between claimed endpoints.
// Parity with the reference sweep is checked in tests/test_gpu_parity.py.
#pragma once
#include <cooperative_groups.h>

#include "lts_common.cuh"
#include "classify.cuh"  // Stencil

namespace lts {
namespace cg = cooperative_groups;

extern int64_t g_launches;

// root of a pointer forest by path halving; concurrent callers only ever
// write ancestors, so races are benign
__device__ __forceinline__ int forest_root(int *p, int x) {
  for (;;) {
    int q = ((volatile int *)p)[x];
    if (q == x) return x;
    int r = ((volatile int *)p)[q];
    if (r != q) p[x] = r;
    x = q;
  }
}

// pointer jumping round (in place: any ancestor is a valid pointer)
__global__ void k_jump(int *ptr, int64_t n) {
  GRID_STRIDE(v, n) {
    int p = ptr[v];
    int q = ptr[p];
    ptr[v] = ptr[q];
  }
}

// path halving on the ascent forest (writes only ancestors) ...
__global__ void k_compress(int *ptr, int64_t n) {
  GRID_STRIDE(v, n) forest_root(ptr, (int)v);
}

// ... then read-only root lookup into a separate array: a halving write by a
// concurrent thread could otherwise overwrite a final root with an ancestor
__global__ void k_roots(const int *__restrict__ ptr, int64_t n, int *root) {
  GRID_STRIDE(v, n) {
    int x = ptr[v];
    for (int q = ptr[x]; q != x; q = ptr[x]) x = q;
    root[v] = x;
  }
}

// vertex class: 1 = discarded maximum (seed, in D), 2 = preserved maximum (P)
__global__ void k_mark_maxima(const uint8_t *__restrict__ flags, const uint8_t *__restrict__ pmark,
                              int kind, int64_t n, uint8_t *vcls, uint8_t *cst, int *mlist,
                              int *counts /* [0]=maxima [1]=D (one u64) */, int *comp, int *par,
                              int *acc, int *rpar, unsigned long long *bestP) {
  GRID_STRIDE(v, n) {
    uint8_t fl = flags[v];
    bool ext = kind == 0 ? (fl & FL_MAX) : (fl & FL_MIN);
    bool pres = kind == 0 ? (pmark[v] & PM_MAX) : (pmark[v] & PM_MIN);
    uint8_t c = ext ? (pres ? 2 : 1) : 0;
    vcls[v] = c;
    unsigned act = __activemask();
    unsigned md = __ballot_sync(act, c == 1);
    unsigned mp = __ballot_sync(act, c == 2);
    unsigned mm = md | mp;
    int lane = threadIdx.x & 31;
    int leader = __ffs(act) - 1;
    int base = 0;
    if (lane == leader && mm) {  // one 64-bit atomic: D count high, all maxima low
      const unsigned long long add = ((unsigned long long)__popc(md) << 32) | (unsigned)__popc(mm);
      base = (int)(unsigned)(atomicAdd(reinterpret_cast<unsigned long long *>(counts), add) & 0xffffffffull);
    }
    base = __shfl_sync(act, base, leader);
    if (c) {
      mlist[base + __popc(mm & lanemask_lt())] = (int)v;
      cst[v] = c == 2 ? 1 : 0;
      comp[v] = (int)v;
      par[v] = (int)v;
      acc[v] = 0x7fffffff;
      rpar[v] = (int)v;
      bestP[v] = 0ull;
    }
  }
}

// Boruvka edge key: heavier first, ties by the other component id
__device__ __forceinline__ unsigned long long bv_pack(int w, int c) {
  return ((unsigned long long)(unsigned)(w + 1) << 32) | (unsigned)c;
}

// De-duplicating edge table: one slot per unordered manifold pair, holding the
// heaviest weight (the only copy any bottleneck or region test can use).
// Linear probing; keys are written once by CAS, weights by atomicMax.
struct EdgeHash {
  unsigned long long *key;  // ~0 = empty
  int *w;                   // -1 = empty
  int bits;                 // 0 = list mode (no table)
  int *count, *overflow;
};

__device__ __forceinline__ void eh_insert(const EdgeHash &H, int a, int b, int w) {
  const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
  const unsigned long long key = ((unsigned long long)lo << 32) | hi;
  const unsigned long long mask = (1ull << H.bits) - 1;
  unsigned long long h = (key * 0x9E3779B97F4A7C15ull) >> (64 - H.bits);
  for (int probe = 0; probe < 64; probe++, h = (h + 1) & mask) {
    unsigned long long k = *(volatile unsigned long long *)(H.key + h);
    if (k == ~0ull) {
      k = atomicCAS(H.key + h, ~0ull, key);
      if (k == ~0ull) {
        if (atomicAdd(H.count, 1) >= (1 << (H.bits - 1))) atomicOr(H.overflow, 1);
        k = key;
      }
    }
    if (k == key) {
      if (*(volatile int *)(H.w + h) < w) atomicMax(H.w + h, w);
      return;
    }
  }
  atomicOr(H.overflow, 1);
}

// table -> edge list (a < b); order is irrelevant to every consumer
__global__ void k_hash_compact(EdgeHash H, int *ea, int *eb, int *ew, int *cnt) {
  const int64_t hc = 1ll << H.bits;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < hc; i0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = i0 + threadIdx.x;
    unsigned long long k = i < hc ? H.key[i] : ~0ull;
    bool has = k != ~0ull;
    unsigned bal = __ballot_sync(0xffffffffu, has);
    if (!bal) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(cnt, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (has) {
      int slot = base + __popc(bal & ((1u << lane) - 1));
      ea[slot] = (int)(k >> 32);
      eb[slot] = (int)(unsigned)(k & 0xffffffffull);
      ew[slot] = H.w[i];
    }
  }
}

// Cross-manifold edges of the maxima graph.  Every grid edge is visited once,
// from its endpoint with the forward stencil offset, with the weight of its
// lower endpoint's rank; a vertex emits one edge per DISTINCT neighbouring
// manifold (its heaviest), so duplicates cannot change any bottleneck.  A CTA owns a
// 32 x 16 (x, y) column of the grid and marches in z (8-plane chunks) (one z plane for 2D grids); the manifold labels M and the
// ranks of planes z-1..z+1 sit in a 5-slot shared-memory ring with halo, so
// the 14-neighbour tests never touch L1/L2.  Edges found by the CTA are
// combined in a shared hash table (one slot per manifold pair, heaviest
// weight) and flushed to the global table / bestP once it fills and at the
// end: a manifold boundary crossing the tile costs one global update instead
// of one per boundary vertex.
#ifndef LTS_ET_ZC
#define LTS_ET_ZC 8
#endif
#ifndef LTS_ET_TY
#define LTS_ET_TY 16
#endif
constexpr int ET_TX = 32, ET_TY = LTS_ET_TY, ET_ZC = LTS_ET_ZC, ET_RING = 5;
constexpr int ET_PX = ET_TX + 2, ET_PY = ET_TY + 2, ET_PL = ET_PX * ET_PY;
constexpr int ET_NT = ET_TX * ET_TY, ET_NEPT = (ET_PL + ET_NT - 1) / ET_NT;
constexpr int ET_HT = 2048, ET_FLUSH = 1024;  // shared table slots / flush level

__device__ __forceinline__ void edge_global(const EdgeHash &H, const uint8_t *__restrict__ vcls,
                                            unsigned long long *bestP, int *ea, int *eb, int *ew,
                                            int *ecount, int a, int b, int w) {
  const bool pa = vcls[a] == 2, pb = vcls[b] == 2;
  if (pa && pb) return;  // preserved-preserved: never needed
  if (pa != pb) {
    const int d = pa ? b : a, pm = pa ? a : b;
    atomicMax(bestP + d, bv_pack(w, pm));
  } else if (H.bits) {
    eh_insert(H, a, b, w);
  } else {
    const int slot = atomicAdd(ecount, 1);
    ea[slot] = a;
    eb[slot] = b;
    ew[slot] = w;
  }
}

// shared edge table insert (one slot per unordered manifold pair, max
// weight); a full probe window sends the edge straight to the global table
__device__ __forceinline__ void et_insert(unsigned long long *hkey, int *hw, int *hcount,
                                          const EdgeHash &H, const uint8_t *__restrict__ vcls,
                                          unsigned long long *bestP, int *ea, int *eb, int *ew,
                                          int *ecount, int a, int b, int w) {
  const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
  const unsigned long long key = ((unsigned long long)lo << 32) | hi;
  unsigned h = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 53) & (ET_HT - 1);
  bool done = false;
  for (int probe = 0; probe < 32 && !done; probe++, h = (h + 1) & (ET_HT - 1)) {
    unsigned long long kk = hkey[h];
    if (kk == ~0ull) {
      kk = atomicCAS(hkey + h, ~0ull, key);
      if (kk == ~0ull) {
        atomicAdd(hcount, 1);
        kk = key;
      }
    }
    if (kk == key) {
      if (hw[h] < w) atomicMax(hw + h, w);
      done = true;
    }
  }
  if (!done) edge_global(H, vcls, bestP, ea, eb, ew, ecount, (int)lo, (int)hi, w);
}

template <int NDIM>
__global__ void __launch_bounds__(ET_NT) k_edges_tile(Grid g, const int *__restrict__ rank, int rev,
                                                    const int *__restrict__ M,
                                                    const uint8_t *__restrict__ vcls, int *ea, int *eb,
                                                    int *ew, int *ecount, unsigned long long *bestP,
                                                    EdgeHash H) {
  using St = Stencil<NDIM>;
  constexpr int K = St::K;
  constexpr int NP = NDIM == 2 ? 1 : ET_RING;
  __shared__ int sM[NP][ET_PL], sR[NP][ET_PL];
  __shared__ unsigned long long hkey[ET_HT];
  __shared__ int hw[ET_HT];
  __shared__ int hcount;
  const int tid = threadIdx.y * ET_TX + threadIdx.x;
  const int x0 = blockIdx.x * ET_TX, y0 = blockIdx.y * ET_TY;
  const int nx = g.nx, ny = g.ny, nz = g.nz, n = (int)g.n;
  const int64_t sxy = (int64_t)nx * ny;
  for (int i = tid; i < ET_HT; i += ET_NT) {
    hkey[i] = ~0ull;
    hw[i] = -1;
  }
  if (tid == 0) hcount = 0;
  // rank planes hold effective ranks (rev applied); -1 / M = -1 outside
  auto fetch = [&](int z, int *rm, int *rr) {
#pragma unroll
    for (int e = 0; e < ET_NEPT; e++) {
      const int i = tid + e * ET_NT;
      const int py = i / ET_PX, px = i - py * ET_PX;
      const int gx = x0 + px - 1, gy = y0 + py - 1;
      const bool in = i < ET_PL && z >= 0 && z < nz && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
      const int64_t gv = (int64_t)z * sxy + (int64_t)gy * nx + gx;
      rm[e] = in ? __ldg(M + gv) : -1;
      const int r = in ? __ldg(rank + gv) : 0;
      rr[e] = rev ? n - 1 - r : r;
    }
  };
  auto put = [&](int slot, const int *rm, const int *rr) {
#pragma unroll
    for (int e = 0; e < ET_NEPT; e++) {
      const int i = tid + e * ET_NT;
      if (i < ET_PL) {
        sM[slot][i] = rm[e];
        sR[slot][i] = rr[e];
      }
    }
  };
  auto flush = [&]() {
    __syncthreads();
    for (int i = tid; i < ET_HT; i += ET_NT) {
      const unsigned long long kk = hkey[i];
      if (kk != ~0ull) {
        edge_global(H, vcls, bestP, ea, eb, ew, ecount, (int)(kk >> 32), (int)(unsigned)(kk & 0xffffffffu), hw[i]);
        hkey[i] = ~0ull;
        hw[i] = -1;
      }
    }
    __syncthreads();
    if (tid == 0) hcount = 0;
    __syncthreads();
  };
  const int zb = NDIM == 2 ? 0 : blockIdx.z * ET_ZC;
  const int ze = NDIM == 2 ? 1 : min(nz, zb + ET_ZC);
  int nm[ET_NEPT], nr[ET_NEPT];
  {
    int am[ET_NEPT], ar[ET_NEPT];
    if (NDIM == 3) {
      fetch(zb - 1, am, ar);
      put(0, am, ar);
      fetch(zb, am, ar);
      put(1, am, ar);
      fetch(zb + 1, am, ar);
      put(2, am, ar);
      fetch(zb + 2, nm, nr);
    } else {
      fetch(0, am, ar);
      put(0, am, ar);
    }
  }
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const int c = (threadIdx.y + 1) * ET_PX + threadIdx.x + 1;
  int sm = 0;
  for (int z = zb; z < ze; z++) {
    const int s1 = sm + 1 >= ET_RING ? sm + 1 - ET_RING : sm + 1;
    const int s2 = s1 + 1 >= ET_RING ? s1 + 1 - ET_RING : s1 + 1;
    const int s3 = s2 + 1 >= ET_RING ? s2 + 1 - ET_RING : s2 + 1;
    if (NDIM == 3) {
      put(s3, nm, nr);
      if (z + 3 < ze + 1) fetch(z + 3, nm, nr);
    }
    // one barrier per plane; it also carries the (uniform) flush decision
    if (__syncthreads_or(tid == 0 && hcount > ET_FLUSH)) flush();
    const int *m0 = sM[NDIM == 2 ? 0 : s1], *mm = sM[NDIM == 2 ? 0 : sm], *mp = sM[NDIM == 2 ? 0 : s2];
    const int *r0 = sR[NDIM == 2 ? 0 : s1], *rm_ = sR[NDIM == 2 ? 0 : sm], *rp = sR[NDIM == 2 ? 0 : s2];
    int a = -1, rv = -1;
    // Every grid edge is visited once, from its endpoint with the forward
    // stencil offset (the first K/2 offsets): weight = the lower endpoint's
    // rank.  Up to three distinct neighbouring manifolds are kept per vertex
    // with their heaviest edge; further ones go straight to the shared table.
    int d0 = -1, d1 = -1, d2 = -1, w0 = -1, w1 = -1, w2 = -1;
    if (x < nx && y < ny) {
      a = m0[c];
      rv = r0[c];
#pragma unroll
      for (int k = 0; k < K / 2; k++) {
        const int dz = St::dz(k);
        const int o = c + St::dx(k) + ET_PX * St::dy(k);
        const int *mk = dz == 0 ? m0 : mp;
        const int *rk = dz == 0 ? r0 : rp;
        const int b = mk[o];
        if (b == a || b < 0) continue;
        const int w = min(rv, rk[o]);
        if (b == d0) w0 = max(w0, w);
        else if (b == d1) w1 = max(w1, w);
        else if (b == d2) w2 = max(w2, w);
        else if (d0 < 0) { d0 = b; w0 = w; }
        else if (d1 < 0) { d1 = b; w1 = w; }
        else if (d2 < 0) { d2 = b; w2 = w; }
        else et_insert(hkey, hw, &hcount, H, vcls, bestP, ea, eb, ew, ecount, a, b, w);  // rare
      }
    }
    // warp aggregation (32 consecutive x voxels usually border the same
    // manifolds): one shared-table update per distinct pair and warp
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int b = i == 0 ? d0 : (i == 1 ? d1 : d2);
      const int w = i == 0 ? w0 : (i == 1 ? w1 : w2);
      const bool has = b >= 0;
      if (!__any_sync(0xffffffffu, has)) break;
      const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
      const unsigned long long key = has ? (((unsigned long long)lo << 32) | hi) : ~0ull;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int best = __reduce_max_sync(peers, w);
      const unsigned top = __ballot_sync(0xffffffffu, has && w == best) & peers;
      if (has && (threadIdx.x & 31) == __ffs(top) - 1)
        et_insert(hkey, hw, &hcount, H, vcls, bestP, ea, eb, ew, ecount, a, b, w);
    }
    sm = s1;
  }
  flush();
}

// ---- Boruvka rounds over the maxima graph --------------------------------


__device__ __forceinline__ void bv_reset(int *mlist, int nm, unsigned long long *best) {
  GRID_STRIDE(i, nm) best[mlist[i]] = 0ull;
}

// each thread scans a run of consecutive edges (edges are emitted per vertex,
// so runs share endpoints) and only issues an atomic when its endpoint changes
constexpr int BV_RUN = 8;
// every active component starts a round from its members' heaviest edges
// into preserved territory
__device__ __forceinline__ void bv_pmax(int *mlist, int nm, int *comp,
                          uint8_t *cst, uint8_t *vcls,
                          unsigned long long *bestP, unsigned long long *best) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (vcls[m] != 1) continue;
    int c = comp[m];
    unsigned long long b = bestP[m];
    if (cst[c] == 0 && b) atomicMax(best + c, b);
  }
}

__device__ __forceinline__ void bv_best(int *ea, int *eb,
                          int *ew, int ne, int *comp,
                          uint8_t *cst, unsigned long long *best) {
  const int64_t nrun = ((int64_t)ne + BV_RUN - 1) / BV_RUN;
  GRID_STRIDE(r, nrun) {
    int64_t i0 = r * BV_RUN, i1 = min((int64_t)ne, i0 + BV_RUN);
    int cur_a = -1, cur_b = -1;
    unsigned long long best_a = 0ull, best_b = 0ull;
    for (int64_t i = i0; i < i1; i++) {
      int ca = comp[ea[i]], cb = comp[eb[i]];
      if (ca == cb) continue;
      int w = ew[i];
      if (ca != cur_a) {
        if (cur_a >= 0 && best_a) atomicMax(best + cur_a, best_a);
        cur_a = ca;
        best_a = 0ull;
      }
      if (cb != cur_b) {
        if (cur_b >= 0 && best_b) atomicMax(best + cur_b, best_b);
        cur_b = cb;
        best_b = 0ull;
      }
      if (cst[ca] == 0) best_a = max(best_a, bv_pack(w, cb));
      if (cst[cb] == 0) best_b = max(best_b, bv_pack(w, ca));
    }
    if (cur_a >= 0 && best_a) atomicMax(best + cur_a, best_a);
    if (cur_b >= 0 && best_b) atomicMax(best + cur_b, best_b);
  }
}

// active root: comp[m] == m && cst[m] == 0
__device__ __forceinline__ void bv_hook(int *mlist, int nm, int *comp,
                          uint8_t *cst, unsigned long long *best,
                          int *par, int *wc, int *err) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (comp[m] != m || cst[m] != 0) continue;
    unsigned long long b = best[m];
    if (b == 0ull) {  // isolated pure component: no preserved maximum reachable
      atomicOr(err, 1);
      par[m] = m;
      wc[m] = -1;
      continue;
    }
    par[m] = (int)(unsigned)(b & 0xffffffffull);
    wc[m] = (int)(b >> 32) - 1;
  }
}

__device__ __forceinline__ void bv_cycle(int *mlist, int nm, int *comp,
                           uint8_t *cst, int *par) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (comp[m] != m || cst[m] != 0) continue;
    int q = par[m];
    if (q != m && cst[q] == 0 && comp[q] == q && par[q] == m && m < q) par[m] = m;
  }
}

__device__ __forceinline__ void bv_jump(int *mlist, int nm, int *comp,
                          uint8_t *cst, int *par) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (comp[m] != m || cst[m] != 0) continue;
    forest_root(par, m);
  }
}

__device__ __forceinline__ void bv_roots(int *mlist, int nm, int *comp,
                           uint8_t *cst, int *par, int *rt) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (comp[m] != m || cst[m] != 0) continue;
    int x = par[m];
    for (int q = par[x]; q != x; q = par[x]) x = q;
    rt[m] = x;
  }
}

// members: tau accumulator and new component; comp is read through a snapshot
// of the round's roots (par of the old root), so the update order is irrelevant
__device__ __forceinline__ void bv_members(int *mlist, int nm, int *comp,
                             uint8_t *cst, int *rt,
                             int *wc, int *acc) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    int c = comp[m];
    if (cst[c] != 0) continue;  // preserved or already final
    int w = wc[c];
    if (w < acc[m]) acc[m] = w;
    comp[m] = rt[c];  // chain root of the old component (bv_roots)
  }
}

// after members moved: roots that reached preserved territory become final;
// count remaining active roots (2-cycle roots)
__device__ __forceinline__ void bv_settle(int *mlist, int nm, int *comp,
                            uint8_t *cst, int *active) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (cst[m] != 0) continue;
    int c = comp[m];
    if (c != m) {
      // m is no longer a root; its component state follows its root
      if (cst[c] != 0) cst[m] = 1;
      continue;
    }
    atomicAdd(active, 1);
  }
}

// All Boruvka rounds in one cooperative launch: the phases of a round are
// separated by grid-wide barriers instead of kernel boundaries, and the
// "still active" test is read on the device instead of by a host readback per
// round.  state[0] = active roots of the last round, state[1] = rounds run.
struct BvArgs {
  int *mlist;
  int nm;
  int *comp, *par, *wc, *rt, *acc, *err;
  uint8_t *cst, *vcls;
  unsigned long long *bestP, *best;
  int *ea, *eb, *ew;
  const int *ne;  // device: edge count written by the edge kernels (no host readback)
  int *state;
};

__global__ void __launch_bounds__(256) k_bv_coop(BvArgs a) {
  cg::grid_group grid = cg::this_grid();
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int ne = *a.ne;
  for (int round = 0; round < 64; round++) {
    bv_reset(a.mlist, a.nm, a.best);
    if (lead) a.state[0] = 0;
    grid.sync();
    bv_pmax(a.mlist, a.nm, a.comp, a.cst, a.vcls, a.bestP, a.best);
    if (ne > 0) bv_best(a.ea, a.eb, a.ew, ne, a.comp, a.cst, a.best);
    grid.sync();
    bv_hook(a.mlist, a.nm, a.comp, a.cst, a.best, a.par, a.wc, a.err);
    grid.sync();
    bv_cycle(a.mlist, a.nm, a.comp, a.cst, a.par);
    grid.sync();
    bv_jump(a.mlist, a.nm, a.comp, a.cst, a.par);
    grid.sync();
    bv_roots(a.mlist, a.nm, a.comp, a.cst, a.par, a.rt);
    grid.sync();
    bv_members(a.mlist, a.nm, a.comp, a.cst, a.rt, a.wc, a.acc);
    grid.sync();
    bv_settle(a.mlist, a.nm, a.comp, a.cst, a.state);
    grid.sync();
    const int act = *(volatile int *)a.state, bad = *(volatile int *)a.err;
    if (lead) a.state[1] = round + 1;
    if (act == 0 || bad) break;
    grid.sync();  // every thread has read state[0] before the next round clears it
  }
}

// ---- claimed set and regions -----------------------------------------------

__device__ __forceinline__ int uf_find(int *p, int x) { return forest_root(p, x); }

__device__ __forceinline__ void uf_union(int *p, int a, int b) {
  for (;;) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a > b) {
      int t = a;
      a = b;
      b = t;
    }
    // hook the larger root under the smaller
    if (atomicCAS(p + b, b, a) == b) return;
  }
}

__global__ void k_region_union(const int *__restrict__ ea, const int *__restrict__ eb,
                               const int *__restrict__ ew, const int *__restrict__ ne_dev,
                               const uint8_t *__restrict__ vcls, const int *__restrict__ acc, int *rpar) {
  const int ne = *ne_dev;
  GRID_STRIDE(i, ne) {
    int a = ea[i], b = eb[i];
    if (vcls[a] != 1 || vcls[b] != 1) continue;
    if (ew[i] <= acc[a]) continue;  // an endpoint at or below the saddle level
    uf_union(rpar, a, b);
  }
}

__global__ void k_region_roots(const int *__restrict__ mlist, int nm, const uint8_t *__restrict__ vcls,
                               const int *__restrict__ acc, const int *__restrict__ rank, int rev,
                               int n, int *rpar, int *ridx, int *nreg, int *rsad, int *rtop,
                               int *rsize) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (vcls[m] != 1) continue;
    int r = uf_find(rpar, m);
    if (r == m) {
      int id = atomicAdd(nreg, 1);
      ridx[m] = id;
      rsad[id] = acc[m];  // saddle rank (effective order)
      rtop[id] = -1;
      rsize[id] = 0;
    }
  }
}

__global__ void k_region_tops(const int *__restrict__ mlist, int nm, const uint8_t *__restrict__ vcls,
                              const int *__restrict__ rank, int rev, int n, int *rpar,
                              const int *__restrict__ ridx, int *rtop) {
  GRID_STRIDE(i, nm) {
    int m = mlist[i];
    if (vcls[m] != 1) continue;
    int r = uf_find(rpar, m);
    atomicMax(rtop + ridx[r], eff_rank(rank, m, rev, n));
  }
}

// claimed <=> M(v) is a seed and rank v > tau(M(v)); label and count
__global__ void k_region_label(const int *__restrict__ rank, int rev, int n,
                               const int *__restrict__ M, const uint8_t *__restrict__ vcls,
                               const int *__restrict__ acc, int *rpar, const int *__restrict__ ridx,
                               int *reg_of, int *rsize, uint32_t *cbits) {
  GRID_STRIDE(v, n) {
    int m = M[v];
    int rid = -1;
    if (vcls[m] == 1 && eff_rank(rank, (int)v, rev, n) > acc[m]) rid = ridx[uf_find(rpar, m)];
    reg_of[v] = rid;
    unsigned act = __activemask();
    // claimed bit set: warps cover 32 consecutive, 32-aligned vertices
    unsigned cb = __ballot_sync(act, rid >= 0);
    if ((threadIdx.x & 31) == __ffs(act) - 1) cbits[v >> 5] = cb;
    unsigned peers = __match_any_sync(act, rid);
    if (rid >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(rsize + rid, __popc(peers));
  }
}

// flag[t] = 1 if the vertex of effective rank t is claimed (for rank-ordered
// compaction)
__device__ __forceinline__ bool claimed_bit(const uint32_t *cbits, int v) {
  return (__ldg(cbits + (v >> 5)) >> (v & 31)) & 1u;
}

// Claimed vertices in rank order as (region, vertex) pairs, in one pass:
// each thread tests 16 consecutive ranks, a block scan orders the CTA's tile,
// and a decoupled look-back over the tiles' published counts gives the tile's
// output offset (replaces flags + a three-kernel scan + compaction).
// st[0] = tile ticket counter, st[1 + tile] = status (2 flag bits | count).
#ifndef LTS_CC_IPT
#define LTS_CC_IPT 8
#endif
constexpr int CC_T = 256, CC_IPT = LTS_CC_IPT, CC_TILE = CC_T * CC_IPT;
constexpr int CC_AGG = 1 << 30, CC_PRE = (int)(2u << 30), CC_VAL = (1 << 30) - 1;

__global__ void __launch_bounds__(CC_T) k_claimed_compact_lb(const int *__restrict__ inv, int rev, int n,
                                                           const uint32_t *__restrict__ cbits,
                                                           const int *__restrict__ reg_of, uint32_t *ckey,
                                                           uint32_t *cval, int *st, int *total) {
  __shared__ int s_tile, s_base, s_wsum[CC_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(st, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = (int64_t)tile * CC_TILE + (int64_t)tid * CC_IPT;
  int v[CC_IPT];
  unsigned fl = 0;
#pragma unroll
  for (int j = 0; j < CC_IPT; j++) {
    const int64_t t = t0 + j;
    v[j] = t < n ? __ldg(inv + (rev ? (n - 1 - t) : t)) : 0;
    if (t < n && claimed_bit(cbits, v[j])) fl |= 1u << j;
  }
  const int c = __popc(fl);
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_wsum[warp] = inc;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < CC_T / 32; w++) {
    const int x = s_wsum[w];
    pre += w < warp ? x : 0;
    tot += x;
  }
  if (warp == 0) {
    // decoupled look-back, 32 predecessors per round trip: publish the tile
    // aggregate, then sum predecessors back to the nearest inclusive prefix
    volatile int *S = st + 1;
    int base = 0;
    if (tile == 0) {
      if (lane == 0) S[0] = CC_PRE | tot;
    } else {
      if (lane == 0) S[tile] = CC_AGG | tot;
      int acc = 0;
      int64_t hi = (int64_t)tile - 1;  // newest predecessor of the window
      for (;;) {
        const int64_t p = hi - lane;
        const int sv = p >= 0 ? (int)S[p] : (int)CC_PRE;
        const int flag = sv & ~CC_VAL;
        if (__any_sync(0xffffffffu, flag == 0)) continue;  // someone in the window has not published
        const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == CC_PRE);
        const int stop = pre_mask ? __ffs(pre_mask) - 1 : 31;  // nearest inclusive prefix
        int v = lane <= stop ? (sv & CC_VAL) : 0;
        v = __reduce_add_sync(0xffffffffu, v);
        acc += v;
        if (pre_mask) break;
        hi -= 32;
      }
      base = acc;
      if (lane == 0) S[tile] = CC_PRE | (acc + tot);
    }
    if (lane == 0) {
      s_base = base;
      if ((int64_t)(tile + 1) * CC_TILE >= n) *total = base + tot;
    }
  }
  __syncthreads();
  int p = s_base + pre + inc - c;
#pragma unroll
  for (int j = 0; j < CC_IPT; j++)
    if (fl >> j & 1u) {
      ckey[p] = (uint32_t)reg_of[v[j]];
      cval[p] = (uint32_t)v[j];
      p++;
    }
}

// region sizes (+1 for the saddle) -> scan input
__global__ void k_region_slots(const int *__restrict__ rsize, int R, int *tmp) {
  GRID_STRIDE(i, R) tmp[i] = rsize[i] + 1;
}

__global__ void k_place(const uint32_t *__restrict__ skey, const uint32_t *__restrict__ sval, int C,
                        const int *__restrict__ rptr, int *verts, int *slot_of) {
  // slot_of is the region-label array: claimed vertices trade their region id
  // for their slot (>= 1), unclaimed ones keep -1
  GRID_STRIDE(j, C) {
    int rid = (int)skey[j];
    int v = (int)sval[j];
    int slot = (int)j + rid + 1;
    verts[slot] = v;
    slot_of[v] = slot;
  }
}

__global__ void k_place_saddles(const int *__restrict__ inv, int rev, int n,
                                const int *__restrict__ rsad, int R, const int *__restrict__ rptr,
                                int *verts) {
  GRID_STRIDE(r, R) {
    int t = rsad[r];
    verts[rptr[r]] = inv[rev ? (n - 1 - t) : t];
  }
}

}  // namespace lts
