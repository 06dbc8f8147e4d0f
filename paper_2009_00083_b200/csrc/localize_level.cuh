// localize_level.cuh -- exact priority floods of large regions by level-parallel
// decomposition (no sequential extraction loop).
//
// A max-first priority flood from a source b over a vertex set C with distinct
// keys (_kernels.py:491-552) factors exactly:
//   * let beta(v) be the vertex of smallest key on the maximin (bottleneck)
//     path from b to v inside C (b itself excluded; b counts as +infinity);
//   * the "trunk" {t : beta(t) = t} is the sequence of record lows of the
//     flood; the classes {v : beta(v) = t} are extracted contiguously, in
//     decreasing key(t), each one starting with t;
//   * inside a class the order is the same flood started at t, with t's own
//     adjacency and t counted as +infinity.
// So the extraction order is the preorder of a forest F (parent of v = the
// trunk vertex of the level at which v became a trunk vertex's class member,
// i.e. the source of the flood task in which v is a record low) with children
// visited in decreasing key, and the subtree sizes of F are the class sizes.
// Bottleneck paths are paths of a maximum spanning tree under the edge weight
// min(key u, key v), so the flood of all flagged regions is data-parallel, one
// cooperative kernel (k_lv_coop) with grid barriers between its phases:
//   1. once per flood, the Boruvka maximum spanning forest R of the region
//      graphs, kept rooted at each region's source (a hooking component
//      reverses the path from its hook vertex to its old root; the source's
//      component never hooks);
//   2. levels: R is never re-rooted.  A class is a connected piece of R and the
//      spanning forest of a later task lies inside R's edges plus the edges
//      from the task's source set to the class, so beta of a level is a
//      multi-source bottleneck on R restricted to the class (lv_pins, two
//      pointer-doubling sweeps); trunk vertices are placed, the others move to
//      the task of their class's trunk vertex (lv_classes_list);
//   3. before the sweeps every task places a prefix of its exact order with a
//      one-warp flood (lv_prefix), so a climb through a bumpy field crosses
//      many bumps per level.
// Levels repeat until every vertex is placed; a final stable sort by F-parent, a
// segmented prefix of the class sizes and pointer jumping over F give every
// vertex its extraction index.  Ascending floods (many sources, min-first) are
// the same flood on reversed keys from a virtual root adjacent to every
// source.  The decomposition was checked against heap floods of the reference
// on the regions of the BASELINE configs (2-D and 3-D, single and multi
// source) and is covered bit-exactly by the parity tests (both flood paths
// forced in turn, randomised sweeps, the full-size digests).
//
// Everything is indexed in "key space": j = jb(region) + key, keys in [0, k],
// jb = bpre[qi] + qi; within a region j is monotone in the key, so keys are
// compared through j.  The neighbour keys of every key come from k_big_setup
// (BigArgs::nrowkey), as for the CTA floods.
#pragma once
#include <cooperative_groups.h>

#include "localize_big.cuh"

namespace lts {

namespace cg = cooperative_groups;

constexpr int LV_DONE = -1;
constexpr unsigned LV_NONE = 0xffffffffu;
constexpr int LV_INTERIOR = -(1 << 30);  // lvl mark during the forest rounds
constexpr int LV_CHAIN = 1 << 29;        // lvl of a prefix vertex: LV_CHAIN | its place after the source
enum { LVC_HOOKS = 0, LVC_CHANGED = 1, LVC_ACTIVE = 2, LVC_N = 16 };

struct LvArgs {
  int *task;    // j: source (j index) of the flood task the vertex belongs to, LV_DONE when placed
  unsigned *fp; // j: F-parent (j index), LV_NONE for sources / non-vertices
  int *par;     // j: parent in the rooted spanning forest
  int *comp;    // j: component label (= j of the component's tree root) at round start
  int *link;    // labels: hook target of this round
  int *csize;   // j: class size (F-subtree size) of a trunk vertex
  int *lvl;     // j: level at which the vertex was placed (-2: not yet; sources: 0)
  int *skey, *sval, *oval;  // final sort / scan buffers; during the levels skey = chain end of a source,
                            // sval = task whose root component a placed chain vertex / ascending source joins
  unsigned long long *best;  // labels: best outgoing edge (min j, max j | INF)
  unsigned long long *pm;    // j: (value, ancestor) pairs of the two pointer-jumping phases
  int *ctr;
  int nj;
  int level;
  const int *alist;  // vertices still active at this level (nullptr: scan the whole key space)
  int na;
};

struct LvRef {
  int qi, rid, lo, k, jb, t;
  bool active, asc;
};

__device__ __forceinline__ LvRef lv_ref(const LocArgs &A, const BigArgs &Bg, int j) {
  int lo = 0, hi = Bg.nbig - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (Bg.bpre[mid] + mid <= j) lo = mid;
    else hi = mid - 1;
  }
  LvRef R;
  R.qi = lo;
  R.jb = Bg.bpre[lo] + lo;
  R.rid = A.order[Bg.qbase + lo];
  R.lo = A.rptr[R.rid];
  R.k = A.rptr[R.rid + 1] - R.lo;
  const int *st = Bg.st + lo * BST_W;
  R.t = st[BST_T];
  R.active = st[BST_ACTIVE] != 0 && st[BST_LEVEL] != 0;
  R.asc = R.t & 1;
  return R;
}

__device__ __forceinline__ unsigned long long lv_pack(unsigned hi, unsigned lo) {
  return ((unsigned long long)hi << 32) | lo;
}

// Every phase is a device function over the key space, strided by the caller:
// a kernel of its own on the host-driven path, a stage between grid barriers
// in the cooperative kernel.
#define LV_FOR(j, L) for (int j = t0; j < (L).nj; j += nt)
// over the level's active list
#define LV_ACT(j, L)                                                                    \
  for (int i_ = t0, j = 0, lim_ = (L).alist ? (L).na : (L).nj;                          \
       i_ < lim_ && ((j = (L).alist ? (L).alist[i_] : i_), true); i_ += nt)

template <int K>
__device__ __forceinline__ void lv_load_row(const BigArgs &Bg, const LvRef &R, int j, int (&q)[K]) {
  const int2 *row = reinterpret_cast<const int2 *>(Bg.nrowkey + ((size_t)R.lo + R.rid + (j - R.jb)) * K);
#pragma unroll
  for (int h = 0; h < K / 2; h++) {
    const int2 v = row[h];
    q[2 * h] = v.x;
    q[2 * h + 1] = v.y;
  }
}

// sources of the coming ascending flood, per region (flat over big-region slots)
__device__ __forceinline__ void lv_nsrc(const LocArgs &A, const BigArgs &Bg, int t0, int nt) {
  for (int i = t0; i < Bg.bslots; i += nt) {
    const int qi = big_locate(Bg, i);
    int *st = Bg.st + qi * BST_W;
    if (!st[BST_ACTIVE] || !st[BST_LEVEL] || !(st[BST_T] & 1)) continue;
    const BigRef R = big_ref(A, Bg, qi);
    const int p = i - Bg.bpre[qi];
    if (p >= 1 && (A.sfl[R.lo + p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT)) atomicAdd(st + BST_NSRC, 1);
  }
}

// tasks of level 1: every vertex of a flooding region belongs to the task of
// the region's source (desc) or virtual root (asc, at the unused key k)
__device__ __forceinline__ void lv_init(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, int *active_ctr, int t0,
                                        int nt) {
  int mine = 0;
  LV_FOR(j, L) {
    int task = LV_DONE, lvl = -2, csz = 0, croot = -1;
    const LvRef R = lv_ref(A, Bg, j);
    if (R.active) {
      const int kap = j - R.jb;
      const int *cin = big_buf(A, R.t) + R.lo;
      if (R.asc) {
        // an empty ascending flood keeps the labels; key k is the virtual root
        if (Bg.st[R.qi * BST_W + BST_NSRC] != 0 && kap != R.k) {
          const int p = Bg.inv[R.lo + R.rid + kap];
          task = R.jb + R.k;
          if (p >= 1 && (A.sfl[R.lo + p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT)) croot = task;
          mine++;
        }
      } else {
        const int unused = R.t == 0 ? Bg.v0[R.qi] : R.k;
        const int src = flood_key(cin[0], false, R.k);
        if (kap == src) {
          lvl = 0;
          csz = R.k;  // a source with a class: its ascent chain is contracted at level 1
        } else if (kap != unused) {
          task = R.jb + src;
          mine++;
        }
      }
    }
    L.task[j] = task;
    L.fp[j] = LV_NONE;
    L.lvl[j] = lvl;
    L.csize[j] = csz;
    L.sval[j] = croot;
    L.skey[j] = j;
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(active_ctr, mine);
}

// Ascent contraction.  The flood of a task starts at its source p with the
// highest member neighbour z1 of p, and continues z1 < z2 < ... as long as the
// highest unplaced member neighbour of the last vertex is higher than it (it
// then beats every older frontier key).  The chain is placed at once: F-parent
// of z(i+1) is z(i), and the rest of the task floods from the sources
// {p, z1, .., zm} together (they all count as +infinity).  One thread per task.
template <int K>
__device__ __forceinline__ void lv_chain(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, const int *plist,
                                         int np, int t0, int nt) {
  // candidates: the vertices active at the previous level (plist), or every key
  for (int i_ = t0, lim_ = plist ? np : L.nj; i_ < lim_; i_ += nt) {
    const int p = plist ? plist[i_] : i_;
    if (L.lvl[p] != L.level - 1 || L.csize[p] <= 1 || L.task[p] != LV_DONE) continue;
    const LvRef R = lv_ref(A, Bg, p);
    int cur = p, last = -1;
    for (;;) {
      int q[K];
      lv_load_row<K>(Bg, R, cur, q);
      int z = -1;
#pragma unroll
      for (int kk = 0; kk < K; kk++) {
        if (q[kk] < 0) continue;
        const int u = R.jb + q[kk];
        if (u > z && L.task[u] == p) z = u;
      }
      if (z < 0 || z < last) break;
      L.task[z] = LV_DONE;
      L.fp[z] = (unsigned)cur;
      L.lvl[z] = L.level;
      L.csize[z] = 1;
      L.sval[z] = p;
      last = cur = z;
    }
    L.skey[p] = cur;
  }
}

// Flood prefix (cooperative path).  Any prefix of a task's exact extraction
// order can be placed up front as a chain in F, the rest of the task flooding
// from the source plus that prefix.  One warp per task source runs the plain
// priority flood with its frontier in shared memory: as long as it climbs
// (every step of an ascent is free: the chain rule above), and otherwise for a
// budget of steps proportional to the task's size (at least 32 for tasks of
// 1 K vertices: about the latency of a level's barriers), so that the
// sequential prefix costs about as much as the level's sweeps over the task.  On a climb
// through a bumpy field a level then crosses many bumps instead of one.
constexpr int LV_FCAP = 704;    // frontier entries per warp (static shared memory: 16 x 704 ints)
constexpr int LV_WARPS = 16;    // warps per block of the cooperative kernel
#ifndef LTS_LV_MINB
#define LTS_LV_MINB 32
#endif
#ifndef LTS_LV_MINB_SIZE
#define LTS_LV_MINB_SIZE 1024
#endif
constexpr int LV_MINB = LTS_LV_MINB, LV_MINB_SIZE = LTS_LV_MINB_SIZE;  // least prefix budget of tasks of that size

__device__ __forceinline__ void lv_sources(const LvArgs &L, const int *plist, int np, int *srclist, int *nsrc,
                                           int t0, int nt) {
  for (int i_ = t0, lim_ = plist ? np : L.nj; i_ < lim_; i_ += nt) {
    const int p = plist ? plist[i_] : i_;
    if (L.lvl[p] != L.level - 1 || L.csize[p] <= 1 || L.task[p] != LV_DONE) continue;
    srclist[atomicAdd(nsrc, 1)] = p;
  }
}

template <int K>
__device__ __forceinline__ void lv_prefix(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, const int *srclist,
                                          int ns, int (*fr_all)[LV_FCAP], int t0, int nt) {
  static_assert(K <= 32, "one lane per neighbour slot");
  const int lane = threadIdx.x & 31;
  int *fr = fr_all[threadIdx.x >> 5];
  const int mark = -(3 + L.level);  // "in the frontier of this level's prefix"
  for (int si = t0 >> 5; si < ns; si += nt >> 5) {
    const int p = srclist[si];
    const LvRef R = lv_ref(A, Bg, p);
    const int budget = min(4096, max(L.csize[p] >> 13, L.csize[p] >= LV_MINB_SIZE ? LV_MINB : 0));
    int nf = 0, cur = p, last = -1, prev = p, steps = 0;
    for (;;) {
      // the unplaced member neighbours of the vertex just placed join the frontier
      int u = -1;
      if (lane < K) {
        const int q = Bg.nrowkey[((size_t)R.lo + R.rid + (cur - R.jb)) * K + lane];
        if (q >= 0) {
          u = R.jb + q;
          if (L.task[u] != p || L.lvl[u] == mark) u = -1;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, u >= 0);
      if (u >= 0) {
        L.lvl[u] = mark;
        fr[nf + __popc(m & lanemask_lt())] = u;
      }
      nf += __popc(m);
      __syncwarp();
      if (nf == 0) break;
      int best = -1, bi = 0;
      for (int i = lane; i < nf; i += 32) {
        const int x = fr[i];
        if (x > best) {
          best = x;
          bi = i;
        }
      }
      const int z = __reduce_max_sync(0xffffffffu, best);
      if (z < last && steps >= budget) break;
      if (nf - 1 + K > LV_FCAP) break;  // no room for the next vertex's neighbours
      const unsigned own = __ballot_sync(0xffffffffu, best == z);
      bi = __shfl_sync(0xffffffffu, bi, __ffs(own) - 1);
      if (lane == 0) {
        fr[bi] = fr[nf - 1];
        // the i-th prefix vertex sits i places after the source: it hangs off p
        // directly with that offset, so the prefix adds no depth to F
        L.task[z] = LV_DONE;
        L.fp[z] = (unsigned)p;
        L.lvl[z] = LV_CHAIN | (steps + 1);
        L.csize[z] = 1;
        L.sval[z] = p;
      }
      nf--;
      __syncwarp();
      prev = last = cur = z;
      steps++;
    }
    if (lane == 0) L.skey[p] = prev;
  }
}

// per level: singleton components, no tree edges; the sources of an ascending
// flood start inside the (virtual) root's component
__device__ __forceinline__ void lv_prep(const LvArgs &L, int t0, int nt) {
  LV_FOR(j, L) {
    const int tk = L.task[j];
    if (tk < 0) continue;
    int c = j, p = -1;
    if (L.sval[j] == tk) c = p = tk;
    L.comp[j] = c;
    L.link[j] = j;
    L.par[j] = p;
    L.best[j] = 0ull;
    L.csize[j] = 0;
    L.comp[tk] = tk;
    L.link[tk] = tk;
  }
}

// Boruvka round, step 1: every vertex outside its task's root component offers
// its heaviest edge leaving its component (weight: (min j, max j), the root
// counting as +infinity) to the component's label
template <int K>
__device__ __forceinline__ void lv_scan(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, int t0, int nt) {
  LV_FOR(j, L) {
    const int tk = L.task[j];
    if (tk < 0) continue;
    const int c = L.comp[j];
    if (c == tk) continue;
    // a vertex whose neighbours all share its component stays interior for the
    // rest of the forest (components only merge): skipped from then on
    if (L.lvl[j] == LV_INTERIOR) continue;
    const LvRef R = lv_ref(A, Bg, j);
    int q[K];
    lv_load_row<K>(Bg, R, j, q);
    unsigned long long b = 0ull;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      if (q[kk] < 0) continue;
      // the forest is built on the level-1 graph: every neighbour row entry is a
      // member of the same task, or the region's source itself
      const int u = R.jb + q[kk];
      unsigned long long w;
      if (u == tk) {
        w = lv_pack((unsigned)j, LV_NONE);
      } else {
        if (L.comp[u] == c) continue;
        w = lv_pack((unsigned)min(u, j), (unsigned)max(u, j));
      }
      b = max(b, w);
    }
    if (b) atomicMax(L.best + c, b);
    else L.lvl[j] = LV_INTERIOR;
  }
}

// step 2: every component outside the root's hooks along its best edge: the
// tree path from the hook vertex to the old root is reversed, so the merged
// tree stays rooted at the target's root.  Two components choosing the same
// edge: the larger label hooks.
__device__ __forceinline__ void lv_hook(const LvArgs &L, int *hook_ctr, int t0, int nt) {
  int hooks = 0;
  LV_FOR(c, L) {
    const int tk = L.task[c];
    if (tk < 0 || L.comp[c] != c) continue;
    const unsigned long long e = L.best[c];
    if (e == 0ull) continue;
    const int x = (int)(e >> 32);
    const unsigned hi = (unsigned)(e & 0xffffffffu);
    const int y = hi == LV_NONE ? tk : (int)hi;
    const int cx = L.comp[x];
    const int cy = y == tk ? tk : L.comp[y];
    int a, b, c2;
    if (cx == c) {
      a = x; b = y; c2 = cy;
    } else {
      a = y; b = x; c2 = cx;
    }
    if (c2 != tk && c < c2 && L.best[c2] == e) continue;
    int prev = b, cur = a;
    while (cur >= 0) {
      const int nxt = L.par[cur];
      L.par[cur] = prev;
      prev = cur;
      cur = nxt;
    }
    L.link[c] = c2;
    hooks++;
  }
  hooks = __reduce_add_sync(0xffffffffu, hooks);
  if ((threadIdx.x & 31) == 0 && hooks) atomicAdd(hook_ctr, hooks);
}

// step 3: labels of the merged components (the label is the tree root)
__device__ __forceinline__ void lv_jump(const LvArgs &L, int t0, int nt) {
  LV_FOR(j, L) {
    if (L.task[j] < 0) continue;
    const int c = L.comp[j];
    int r = c, nx;
    while ((nx = L.link[r]) != r) r = nx;
    int cur = c;
    while (cur != r) {  // shorten the chain for the threads that follow
      nx = L.link[cur];
      if (nx != r) L.link[cur] = r;
      cur = nx;
    }
    L.comp[j] = r;
    L.best[j] = 0ull;
  }
}

// ---- beta of a level on the static tree -------------------------------------
// The spanning forest R is built once per flood (level 1 graph: only the
// region's source counts as +infinity) and never re-rooted: a class is a
// connected piece of R, and the maximum spanning forest of a later task lies
// inside R's edges plus the edges from the task's source set S to the class.
// So beta(v) is a multi-source bottleneck on R restricted to the class:
//     H(v) = max over pins z of min key on the R-path z..v,
// pins = members adjacent to S.  Two sweeps of exact pointer doubling over the
// parent pointers (segments [v, anc) with their minimum):
//   up:   g(a) = max over pins z below a of pathmin(z..a)   (pushed, atomicMax)
//   down: H(v) = max over ancestors a of min(g(a), pathmin(v..a))   (pulled)
// max / min are idempotent, so the in-place updates of g need no ordering
// beyond the barrier between rounds; the doubling tables are double-buffered.
constexpr unsigned LV_NIL = 0xffffffffu;
#ifndef LTS_LV_HOPS
#define LTS_LV_HOPS 3
#endif
constexpr int LV_HOPS = LTS_LV_HOPS;  // ancestors visited per round (3: radix-4 doubling, 7: radix-8)

// MARKS: the flood prefix (lv_prefix) has pushed every member neighbour of a
// task's source set into its frontier and marked it: the pins are the marked
// vertices that stayed unplaced, no neighbour row is read.  Without the prefix
// (host-driven path: plain ascent chains) every member scans its neighbours.
template <int K, bool MARKS>
__device__ __forceinline__ void lv_pins(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, unsigned long long *J,
                                        int t0, int nt) {
  const int mark = -(3 + L.level);
  LV_ACT(j, L) {
    const int tk = L.task[j];
    if (tk < 0) continue;
    bool pin = L.sval[j] == tk;  // a source of an ascending flood (virtual root)
    if (MARKS) {
      pin = pin || L.lvl[j] == mark;
    } else if (!pin) {
      const LvRef R = lv_ref(A, Bg, j);
      int q[K];
      lv_load_row<K>(Bg, R, j, q);
#pragma unroll
      for (int kk = 0; kk < K; kk++) {
        if (q[kk] < 0) continue;
        const int u = R.jb + q[kk];
        if (u == tk || (L.task[u] < 0 && L.sval[u] == tk)) pin = true;
      }
    }
    L.comp[j] = pin ? j : -1;  // g, then H
    L.csize[j] = 0;
    const int pa = L.par[j];
    const bool in = pa >= 0 && L.task[pa] == tk;
    J[j] = lv_pack((unsigned)j, in ? (unsigned)pa : LV_NIL);
  }
}

// the doubling pair of j before any jump: ([j, parent), parent), parent NIL outside the task
__device__ __forceinline__ unsigned long long lv_j0(const LvArgs &L, int j, int tk) {
  const int pa = L.par[j];
  const bool in = pa >= 0 && L.task[pa] == tk;
  return lv_pack((unsigned)j, in ? (unsigned)pa : LV_NIL);
}

// One doubling round.  FIRST: the pairs are read from the parent pointers (the
// downward sweep restarts the doubling without an initialisation phase).  With
// HOPS = 3 the round jumps four segments instead of two (it pushes to / pulls
// from the ancestors at one, two and three segment lengths): half the rounds,
// i.e. half the grid barriers of the small floods and half the passes over
// the pair arrays of the large ones (cfg4 276 -> 251 ms against HOPS = 1).
// The round reports whether any vertex still has an ancestor to jump to.
template <bool UP, bool FIRST, int HOPS>
__device__ __forceinline__ void lv_sweep_round(const LvArgs &L, const unsigned long long *Jc, unsigned long long *Jn,
                                               int *changed, int t0, int nt) {
  int ch = 0;
  int *g = L.comp;
  LV_ACT(j, L) {
    const int tk = L.task[j];
    if (tk < 0) continue;
    const unsigned long long a = FIRST ? lv_j0(L, j, tk) : Jc[j];
    unsigned anc = (unsigned)(a & 0xffffffffu);
    if (anc == LV_NIL) {
      Jn[j] = a;
      continue;
    }
    int pmin = (int)(a >> 32);  // smallest j in [j, anc)
    const int gv = UP ? g[j] : 0;
    int hv = UP ? 0 : g[j];
    const int hv0 = hv;
#pragma unroll
    for (int hop = 0; hop < HOPS; hop++) {
      if (UP) {
        if (gv >= 0) atomicMax(g + anc, min(min(gv, pmin), (int)anc));
      } else {
        hv = max(hv, min(pmin, g[anc]));
      }
      const unsigned long long b = FIRST ? lv_j0(L, (int)anc, tk) : Jc[anc];
      pmin = min(pmin, (int)(b >> 32));
      anc = (unsigned)(b & 0xffffffffu);
      if (anc == LV_NIL) break;
    }
    if (!UP && hv > hv0) g[j] = hv;
    Jn[j] = lv_pack((unsigned)pmin, anc);
    if (anc != LV_NIL) ch = 1;
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// classes of this level: trunk vertices are placed (F-parent = the end of the
// task source's chain), the others join the task of their class's trunk vertex
__device__ __forceinline__ void lv_classes(const LvArgs &L, int *active_ctr, int t0, int nt) {
  int act = 0;
  const int lim = L.alist ? L.na : L.nj;
  for (int i0 = t0 - (int)(threadIdx.x & 31); i0 < lim; i0 += nt) {
    const int i = i0 + (threadIdx.x & 31);
    const int j = i < lim ? (L.alist ? L.alist[i] : i) : -1;
    const int tk = j >= 0 ? L.task[j] : -1;
    int beta = -1;
    if (tk >= 0) {
      beta = L.comp[j];
      if (beta == j) {
        L.fp[j] = (unsigned)L.skey[tk];
        L.lvl[j] = L.level;
        L.task[j] = LV_DONE;
      } else {
        L.task[j] = beta;
        act++;
      }
    }
    // one atomic per class and warp
    const unsigned peers = __match_any_sync(0xffffffffu, beta);
    if (beta >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(L.csize + beta, __popc(peers));
  }
  if (active_ctr) {
    act = __reduce_add_sync(0xffffffffu, act);
    if ((threadIdx.x & 31) == 0 && act) atomicAdd(active_ctr, act);
  }
}

// classes and the active list of the next level in one phase (cooperative
// path): a block takes tiles of the current list (level 1: of the key space),
// and the vertices still unplaced are appended tile by tile, in order, so the
// phases that follow stay coalesced; *cursor ends as the active count
__device__ __forceinline__ void lv_classes_list(const LvArgs &L, int *list, int *cursor) {
  __shared__ int wsum[32], wbeta[32], wcnt[32];
  __shared__ int base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lim = L.alist ? L.na : L.nj;
  for (int tile = blockIdx.x * blockDim.x; tile < lim; tile += gridDim.x * blockDim.x) {
    const int i = tile + threadIdx.x;
    const int j = i < lim ? (L.alist ? L.alist[i] : i) : -1;
    const int tk = j >= 0 ? L.task[j] : -1;
    int beta = -1;
    bool on = false;
    if (tk >= 0) {
      beta = L.comp[j];
      if (beta == j) {
        L.fp[j] = (unsigned)L.skey[tk];
        L.lvl[j] = L.level;
        L.task[j] = LV_DONE;
      } else {
        L.task[j] = beta;
        on = true;
      }
    }
    // class sizes: one atomic per class and warp, and the warps' first classes
    // (a giant class fills whole tiles) merged once more across the block
    const unsigned peers = __match_any_sync(0xffffffffu, beta);
    const unsigned valid = __ballot_sync(0xffffffffu, beta >= 0);
    const int first = valid ? __ffs(valid) - 1 : -1;
    const bool infirst = first >= 0 && ((peers >> first) & 1u);
    if (beta >= 0 && !infirst && lane == __ffs(peers) - 1) atomicAdd(L.csize + beta, __popc(peers));
    if (lane == (first < 0 ? 0 : first)) {
      wbeta[warp] = first < 0 ? -1 : beta;
      wcnt[warp] = first < 0 ? 0 : __popc(peers);
    }
    const unsigned m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      const int b = lane < nw ? wbeta[lane] : -1;
      const int c = lane < nw ? wcnt[lane] : 0;
      const unsigned same = __match_any_sync(0xffffffffu, b);
      const int tot = __reduce_add_sync(same, c);
      if (b >= 0 && lane == __ffs(same) - 1) atomicAdd(L.csize + b, tot);
    }
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < nw; w++) {
        const int c = wsum[w];
        wsum[w] = tot;
        tot += c;
      }
      base = tot ? atomicAdd(cursor, tot) : 0;
    }
    __syncthreads();
    if (on) list[base + wsum[warp] + __popc(m & lanemask_lt())] = j;
    __syncthreads();
  }
}

// ---- extraction indices: preorder of F, children in decreasing key ----------
__device__ __forceinline__ void lv_sortkeys(const LvArgs &L, int t0, int nt) {
  LV_FOR(i, L) {
    const int j = L.nj - 1 - i;
    const unsigned f = L.fp[j];
    L.skey[i] = f == LV_NONE ? L.nj : (int)f;
    L.sval[i] = j;
  }
}

__device__ __forceinline__ void lv_gather(const LvArgs &L, int t0, int nt) {
  LV_FOR(i, L) {
    const int j = L.oval[i];
    L.skey[i] = L.fp[j] == LV_NONE ? 0 : L.csize[j];
  }
}

// cum = exclusive prefix of the class sizes in sorted order (in sval); the
// first child of every parent records the parent's base
__device__ __forceinline__ void lv_heads(const LvArgs &L, int t0, int nt) {
  LV_FOR(i, L) {
    const unsigned f = L.fp[L.oval[i]];
    if (f == LV_NONE) continue;
    if (i == 0 || L.fp[L.oval[i - 1]] != f) L.par[f] = L.sval[i];
  }
}

__device__ __forceinline__ void lv_off(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, int t0, int nt) {
  LV_FOR(i, L) {
    const int j = L.oval[i];
    const unsigned f = L.fp[j];
    if (f == LV_NONE) continue;
    int acc = L.sval[i] - L.par[f] + 1;
    const int lv = L.lvl[j];
    if (lv >= LV_CHAIN) acc = lv - LV_CHAIN;  // prefix vertex: its place after the source
    else if (L.fp[f] == LV_NONE && lv_ref(A, Bg, j).asc) acc--;  // children of the virtual root start at 0
    L.pm[j] = lv_pack((unsigned)acc, f);
  }
}

__device__ __forceinline__ void lv_pos_round(const LvArgs &L, int *changed, int t0, int nt) {
  int ch = 0;
  LV_FOR(j, L) {
    if (L.fp[j] == LV_NONE) continue;
    unsigned long long a = L.pm[j];
    unsigned acc = (unsigned)(a >> 32), anc = (unsigned)(a & 0xffffffffu);
    if (L.fp[anc] == LV_NONE) continue;
    // up to three jumps per round: every pair read is a consistent (offset,
    // ancestor) snapshot, so any number of hops keeps the invariant
#pragma unroll
    for (int hop = 0; hop < 3; hop++) {
      const unsigned long long b = L.pm[anc];
      acc += (unsigned)(b >> 32);
      anc = (unsigned)(b & 0xffffffffu);
      if (L.fp[anc] == LV_NONE) break;
    }
    L.pm[j] = lv_pack(acc, anc);
    ch = 1;
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// state t+1 of every level-flooded region
__device__ __forceinline__ void lv_write(const LocArgs &A, const BigArgs &Bg, const LvArgs &L, int t0, int nt) {
  LV_FOR(j, L) {
    const LvRef R = lv_ref(A, Bg, j);
    if (!R.active) continue;
    const int kap = j - R.jb;
    const int unused = R.t == 0 ? Bg.v0[R.qi] : R.k;
    if (kap == unused) continue;
    const int p = Bg.inv[R.lo + R.rid + kap];
    const int *cin = big_buf(A, R.t) + R.lo;
    int *cout = big_buf(A, R.t + 1) + R.lo;
    if (R.asc && Bg.st[R.qi * BST_W + BST_NSRC] == 0) {
      cout[p] = cin[p];
      continue;
    }
    const int e = L.fp[j] == LV_NONE ? 0 : (int)(L.pm[j] >> 32);
    cout[p] = R.asc ? e : R.k - 1 - e;
    if (p == 0) atomicAdd(Bg.work, (unsigned long long)R.k);
  }
}

#define LV_T0 (int)(blockIdx.x * blockDim.x + threadIdx.x)
#define LV_NT (int)(gridDim.x * blockDim.x)
__global__ void __launch_bounds__(256) k_lv_nsrc(LocArgs A, BigArgs Bg) { lv_nsrc(A, Bg, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_init(LocArgs A, BigArgs Bg, LvArgs L) {
  lv_init(A, Bg, L, L.ctr + LVC_ACTIVE, LV_T0, LV_NT);
}
template <int K>
__global__ void __launch_bounds__(256) k_lv_chain(LocArgs A, BigArgs Bg, LvArgs L) {
  lv_chain<K>(A, Bg, L, nullptr, 0, LV_T0, LV_NT);
}
__global__ void __launch_bounds__(256) k_lv_prep(LvArgs L) { lv_prep(L, LV_T0, LV_NT); }
template <int K>
__global__ void __launch_bounds__(256) k_lv_scan(LocArgs A, BigArgs Bg, LvArgs L) { lv_scan<K>(A, Bg, L, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_hook(LvArgs L) { lv_hook(L, L.ctr + LVC_HOOKS, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_jump(LvArgs L) { lv_jump(L, LV_T0, LV_NT); }
template <int K>
__global__ void __launch_bounds__(256) k_lv_pins(LocArgs A, BigArgs Bg, LvArgs L, unsigned long long *J) {
  lv_pins<K, false>(A, Bg, L, J, LV_T0, LV_NT);
}
template <bool UP, bool FIRST>
__global__ void __launch_bounds__(256) k_lv_sweep(LvArgs L, const unsigned long long *Jc, unsigned long long *Jn) {
  lv_sweep_round<UP, FIRST, 1>(L, Jc, Jn, L.ctr + LVC_CHANGED, LV_T0, LV_NT);
}
__global__ void __launch_bounds__(256) k_lv_classes(LvArgs L) { lv_classes(L, L.ctr + LVC_ACTIVE, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_sortkeys(LvArgs L) { lv_sortkeys(L, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_gather(LvArgs L) { lv_gather(L, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_heads(LvArgs L) { lv_heads(L, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_off(LocArgs A, BigArgs Bg, LvArgs L) { lv_off(A, Bg, L, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_pos_round(LvArgs L) { lv_pos_round(L, L.ctr + LVC_CHANGED, LV_T0, LV_NT); }
__global__ void __launch_bounds__(256) k_lv_write(LocArgs A, BigArgs Bg, LvArgs L) { lv_write(A, Bg, L, LV_T0, LV_NT); }

// All levels of one flood in one cooperative launch: the phases are separated
// by grid barriers and the loop conditions are read on the device.  A counter
// slot is cleared only after every thread has read it and passed a barrier:
// the hook counter alternates between two slots (read before the round's last
// barrier), the changed flag rotates over three (read after its barrier), the
// active count alternates by level.
enum { LVK_HOOKS = 0, LVK_CHANGED = 2, LVK_ACTIVE = 5, LVK_INIT = 7, LVK_LEVELS = 8, LVK_ROUNDS = 9, LVK_NSRC = 10,
       LVK_ERR = 12 };  // LVK_ERR: a loop hit its round limit (the host turns it into an error)

// phase clocks of the lead thread (LTS_LEVEL_VERBOSE): chain, prep, scan, hook, jump, beta, classes
__device__ long long d_lvclk[8];
__device__ long long d_lvlog[128][4];  // per level (LTS_LEVEL_VERBOSE): active, sweep rounds, sweep cycles, level cycles
#define LV_TICK(i)                 \
  if (lead) {                      \
    const long long tn = clock64(); \
    d_lvclk[i] += tn - tq;         \
    tq = tn;                       \
  }

template <int K>
__global__ void __launch_bounds__(32 * LV_WARPS) k_lv_coop(LocArgs A, BigArgs Bg, LvArgs L) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int s_front[LV_WARPS][LV_FCAP];
  const int t0 = LV_T0, nt = LV_NT;
  const bool lead = t0 == 0;
  long long tq = clock64();
  int *ctr = L.ctr;  // zeroed by the host
  lv_nsrc(A, Bg, t0, nt);
  grid.sync();
  lv_init(A, Bg, L, ctr + LVK_INIT, t0, nt);
  grid.sync();
  int active = *(volatile int *)(ctr + LVK_INIT);
  int rounds = 0, cslot = 0;
  // the spanning forest R of the whole flood, rooted at the sources
  if (active > 0) {
    L.level = 1;
    lv_prep(L, t0, nt);
    grid.sync();
    LV_TICK(1)
    for (int round = 0; round < 64; round++, rounds++) {
      const int hp = round & 1;
      lv_scan<K>(A, Bg, L, t0, nt);
      if (lead) ctr[LVK_HOOKS + (hp ^ 1)] = 0;
      grid.sync();
      LV_TICK(2)
      lv_hook(L, ctr + LVK_HOOKS + hp, t0, nt);
      grid.sync();
      LV_TICK(3)
      lv_jump(L, t0, nt);
      const int h = *(volatile int *)(ctr + LVK_HOOKS + hp);
      grid.sync();
      LV_TICK(4)
      if (h == 0) break;
      if (round == 63 && lead) ctr[LVK_ERR] = 1;
    }
  }
  L.level = 0;
  unsigned long long *Ja = L.pm, *Jb = L.best;
  // The active list of a level is built at the end of the previous one, the
  // two buffers (link, oval: both free once the forest stands) alternating;
  // level 1 runs over the whole key space.  The list a level ran over holds
  // the trunk vertices it placed: the chain candidates of the next level.
  int *bufs[2] = {L.link, L.oval};
  const int *plist = nullptr;
  int np = 0;
  L.alist = nullptr;
  L.na = active;
  while (active > 0) {
    L.level++;
    const int apar = L.level & 1;
    const long long lv_t0 = clock64();
    long long lv_ts = 0;
    int lv_rounds = 0;
    lv_sources(L, plist, np, (int *)Jb, ctr + LVK_NSRC + apar, t0, nt);
    grid.sync();
    lv_prefix<K>(A, Bg, L, (const int *)Jb, *(volatile int *)(ctr + LVK_NSRC + apar), s_front, t0, nt);
    grid.sync();
    LV_TICK(0)
    lv_pins<K, true>(A, Bg, L, Ja, t0, nt);
    if (lead) {
      ctr[LVK_ACTIVE + apar] = 0;
      ctr[LVK_NSRC + (apar ^ 1)] = 0;
    }
    grid.sync();
    lv_ts = clock64();
    for (int sweep = 0; sweep < 2; sweep++) {
      unsigned long long *Jc = Ja, *Jn = Jb;
      for (int it = 0; it < 40; it++) {
        lv_rounds++;
        cslot = cslot == 2 ? 0 : cslot + 1;
        if (lead) ctr[LVK_CHANGED + (cslot == 2 ? 0 : cslot + 1)] = 0;
        int *chg = ctr + LVK_CHANGED + cslot;
        if (sweep == 0) lv_sweep_round<true, false, LV_HOPS>(L, Jc, Jn, chg, t0, nt);
        else if (it == 0) lv_sweep_round<false, true, LV_HOPS>(L, Jc, Jn, chg, t0, nt);
        else lv_sweep_round<false, false, LV_HOPS>(L, Jc, Jn, chg, t0, nt);
        grid.sync();
        unsigned long long *tmp = Jc;
        Jc = Jn;
        Jn = tmp;
        if (*(volatile int *)chg == 0) break;
        if (it == 39 && lead) ctr[LVK_ERR] = 1;
      }
    }
    LV_TICK(5)
    lv_ts = clock64() - lv_ts;
    int *lnext = bufs[apar];
    lv_classes_list(L, lnext, ctr + LVK_ACTIVE + apar);
    grid.sync();
    LV_TICK(6)
    if (lead && L.level <= 128) {
      d_lvlog[L.level - 1][0] = L.na;
      d_lvlog[L.level - 1][1] = lv_rounds;
      d_lvlog[L.level - 1][2] = lv_ts;
      d_lvlog[L.level - 1][3] = clock64() - lv_t0;
    }
    active = *(volatile int *)(ctr + LVK_ACTIVE + apar);
    plist = L.alist;
    np = L.na;
    L.alist = lnext;
    L.na = active;
  }
  if (lead) {
    ctr[LVK_LEVELS] = L.level;
    ctr[LVK_ROUNDS] = rounds;
  }
}

// positions by pointer jumping over F, all rounds in one cooperative launch
// (ctr[LVK_CHANGED..+2] zeroed by the host)
__global__ void __launch_bounds__(512) k_lv_pos_coop(LvArgs L) {
  cg::grid_group grid = cg::this_grid();
  const int t0 = LV_T0, nt = LV_NT;
  int cslot = 0;
  for (int it = 0; it < 64; it++) {
    cslot = cslot == 2 ? 0 : cslot + 1;
    if (t0 == 0) L.ctr[LVK_CHANGED + (cslot == 2 ? 0 : cslot + 1)] = 0;
    lv_pos_round(L, L.ctr + LVK_CHANGED + cslot, t0, nt);
    grid.sync();
    if (*(volatile int *)(L.ctr + LVK_CHANGED + cslot) == 0) break;
    if (it == 63 && t0 == 0) L.ctr[LVK_ERR] = 1;
  }
}

}  // namespace lts
