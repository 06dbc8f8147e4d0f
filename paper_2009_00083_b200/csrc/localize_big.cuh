// localize_big.cuh -- exact priority floods of large regions, one CTA each,
// extracting many vertices per synchronisation step.
//
// A priority flood's extraction order depends only on which vertices are in
// the frontier F when each extraction happens.  Let f1 > f2 > ... be F sorted
// by key and let new_i be the unseen neighbours exposed by extracting f1..fi.
// Then f1..fj are the next j extractions, in that order, iff
//     max key(new_1 u ... u new_i) < key(f_{i+1})   for every i < j.
// Each step therefore takes the top-B keys of F, computes the exposure maxima
// of all candidates in parallel (B x K neighbour probes), cuts the prefix at
// the first preemption and commits it.  On the cfg3 regions a flood needs
// ~1% as many steps as extractions.
//
// Keys are a permutation of a small integer range (the region's local order),
// so F is a bit set over key space kept as a 32-ary bit tree in shared memory
// (the leaf level spills to global memory for very large regions).  The top-B
// keys come from a descending walk of the tree; key -> local index is an
// inverse array rebuilt per flood; "seen" is a bit set over local indices.
// Region adjacency is resolved once per region into rows of local indices so
// every flood and check touches one row per vertex.
// Semantics follow _localize_one (_kernels.py:443-575) exactly, including the
// empty-ascending-flood case and the period-2 cycle jump (contract D5).
#pragma once
#include "localize.cuh"

namespace lts {

#ifndef LTS_BIG_T
#define LTS_BIG_T 1024
#endif
constexpr int BIG_T = LTS_BIG_T;
#ifndef LTS_BIG_B
#define LTS_BIG_B 256
#endif
constexpr int BIG_B = LTS_BIG_B;              // max candidates per step
constexpr int BIG_SMEM_WORDS = 10 * 1024;     // bit-set words in shared memory (rest of the SM is L1)
constexpr int BIG_XMAX = 512;                 // climb continuation list (index fits 9 bits)
static_assert(BIG_XMAX <= 512, "packed climb argmax");
constexpr int BIG_HOPS = 16;                  // sequential hops per step
constexpr int BIG_THRESHOLD = 256;            // regions with k > this use this kernel

struct BigArgs {
  int *v0;           // per big region: first admissible boundary minimum
  int *inv;          // key -> local index, S + R entries (region base lo + rid)
  uint32_t *gbits;   // spill space for leaf / seen bit sets
  int *nrow;         // per slot: K local neighbour indices (-1 = not a member)
  int *nrowkey;      // per key: K neighbour keys of the current flood (rows in key order)
  int qbase, nbig;   // regions order[qbase .. qbase+nbig)
  int *queue;
};

// optional per-region instrumentation (lts_debug_big_stats): big-queue slot i
// records [k, steps, candidates, committed, flood cycles, check cycles, init
// cycles, n_iters]
constexpr int DBG_MAX = 256, DBG_W = 24;
__device__ long long d_dbg[DBG_MAX * DBG_W];
__device__ int d_dbg_on;

// Frontier F as a counted bit set over key space [0, k]: leaf bits plus, per
// block of 32^(l+1) keys, the number of keys in F (levels 1..top).  The top
// level has <= 32 blocks, so one warp reads it in one step.
struct CTree {
  uint32_t *leaf;
  int nw0;          // leaf words
  int *cnt[6];      // cnt[l][i], l = 1..top: keys in block i of level l
  int nb[6];        // blocks per level (nb[0] = nw0)
  int top;
};

__device__ __forceinline__ uint32_t mask_le(int b) { return b >= 31 ? 0xffffffffu : ((2u << b) - 1u); }

__device__ __forceinline__ void ct_insert(const CTree &T, int key) {
  atomicOr(T.leaf + (key >> 5), 1u << (key & 31));
  for (int l = 1; l <= T.top; l++) atomicAdd(T.cnt[l] + (key >> (5 * (l + 1))), 1);
}

__device__ __forceinline__ void ct_remove(const CTree &T, int key) {
  atomicAnd(T.leaf + (key >> 5), ~(1u << (key & 31)));
  for (int l = 1; l <= T.top; l++) atomicSub(T.cnt[l] + (key >> (5 * (l + 1))), 1);
}

// warp-aggregated count updates: the upper levels have few blocks, so per-key
// shared atomics would serialise on a handful of addresses
__device__ __forceinline__ void ct_update_warp(const CTree &T, int key, bool valid, int delta) {
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  if (valid) {
    if (delta > 0) atomicOr(T.leaf + (key >> 5), 1u << (key & 31));
    else atomicAnd(T.leaf + (key >> 5), ~(1u << (key & 31)));
  }
  for (int l = 1; l <= T.top; l++) {
    int idx = valid ? (key >> (5 * (l + 1))) : -1;
    unsigned peers = __match_any_sync(act, idx);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(T.cnt[l] + idx, delta * __popc(peers));
  }
}

// leaf-only frontier updates; the highest non-empty chunk (BIG_T leaf words)
// is tracked with one warp-aggregated atomicMax per insertion batch
__device__ __forceinline__ void leaf_remove(uint32_t *leaf, int key, bool valid) {
  if (valid) atomicAnd(leaf + (key >> 5), ~(1u << (key & 31)));
}

__device__ __forceinline__ void leaf_insert(uint32_t *leaf, int *hi_chunk, int key, bool valid,
                                            int chunk_shift) {
  if (valid) atomicOr(leaf + (key >> 5), 1u << (key & 31));
  const unsigned act = __activemask();
  const int m = __reduce_max_sync(act, valid ? (key >> chunk_shift) : -1);
  if (m >= 0 && (threadIdx.x & 31) == __ffs(act) - 1) atomicMax(hi_chunk, m);
}

// warp 0: the `need`-th largest key of F (need clamped to |F|).  Returns the
// threshold key tau (-1 if F is empty) and the clamped need.
__device__ __forceinline__ int ct_threshold(const CTree &T, int want, int &need_out) {
  const int lane = threadIdx.x & 31;
  int l = T.top, base = 0, nel = T.nb[T.top];
  int need = want;
  bool first = true;
  for (;;) {
    int e = base + nel - 1 - lane;
    int c = 0;
    if (lane < nel) c = l == 0 ? __popc(T.leaf[e]) : T.cnt[l][e];
    int P = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, P, o);
      if (lane >= o) P += y;
    }
    if (first) {
      int total = __shfl_sync(0xffffffffu, P, 31);
      need = min(need, total);
      need_out = need;
      if (need == 0) return -1;
      first = false;
    }
    unsigned hit = __ballot_sync(0xffffffffu, P >= need);
    int src = __ffs(hit) - 1;
    int before = __shfl_sync(0xffffffffu, P - c, src);
    int es = base + nel - 1 - src;
    need -= before;
    if (l == 0) {
      uint32_t w = T.leaf[es];
      // need-th highest set bit of w
      int b = 31;
      for (int r = 0;; b--) {
        if ((w >> b) & 1u) {
          if (++r == need) break;
        }
      }
      return (es << 5) + b;
    }
    base = es << 5;
    nel = min(32, T.nb[l - 1] - base);
    l--;
  }
}

struct BigSmem {
  int cand_key[BIG_B];
  int newmax[BIG_B];
  int pair_key[BIG_B * kMaxK];
  int wsum[BIG_T / 32 + 1];
  int ncand, cut, nsrc, red, v0, qi, tau, carry, hi_chunk;
  int xcnt, enew;           // climb continuation: exposures above the window
  int xkey[BIG_XMAX];
  CTree T;          // frontier descriptor (uniform; kept out of local memory)
  uint32_t *seen;   // bit set over keys
  uint32_t bits[BIG_SMEM_WORDS];
};

struct BigRegion {
  int rid, lo, k, s;
  const int *verts;
  const int *row;   // k*K local neighbour indices, by local index
  int *krow;        // (k+1)*K neighbour keys of the current flood, by key (-1: not a member)
  uint8_t *sfl;
  int *inv;
};

__device__ __forceinline__ bool seen_test(const uint32_t *seen, int q) {
  return (seen[q >> 5] >> (q & 31)) & 1u;
}

// desc floods map the sentinels +BIG -> k, -BIG -> 0; asc floods reverse
__device__ __forceinline__ int flood_key(int c, bool asc, int k) {
  if (asc) return k - 1 - c;
  if (c == 0x7fffffff) return k;
  if (c == (int)0x80000000) return 0;
  return c;
}

// block-wide exclusive scan (BIG_T threads) with one barrier: warp scans,
// then every warp scans the warp totals itself.  The caller must barrier
// before wsum is written again.
__device__ __forceinline__ int big_scan_excl(int x, int *wsum, int &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  const int v = lane < BIG_T / 32 ? wsum[lane] : 0;
  int p = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, p, o);
    if (lane >= o) p += y;
  }
  total = __shfl_sync(0xffffffffu, p, 31);
  return __shfl_sync(0xffffffffu, p - v, warp) + inc - x;
}

template <int K>
__device__ void big_flood(BigSmem &S, BigRegion &G, bool asc, const int *cin, int *cout, int &Beff,
                          long long *dbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = G.k;
  const CTree &T = S.T;
  uint32_t *const seen = S.seen;
  const int seen_words = T.nw0;
  for (int i = tid; i < T.nw0; i += BIG_T) T.leaf[i] = 0u;
  for (int l = 1; l <= T.top; l++)
    for (int i = tid; i < T.nb[l]; i += BIG_T) T.cnt[l][i] = 0;
  for (int i = tid; i < seen_words; i += BIG_T) seen[i] = 0u;
  if (tid == 0) {
    S.nsrc = 0;
    S.hi_chunk = -1;
  }
  __syncthreads();
  auto key_of = [&](int p) -> int { return flood_key(cin[p], asc, k); };
  for (int p = tid; p < k; p += BIG_T) G.inv[key_of(p)] = p;
  // neighbour keys of this flood, one row per KEY: the flood never needs a
  // local index except to write its label
  for (int i = tid; i < k * K; i += BIG_T) {
    const int p = i / K, kk = i - p * K;
    const int q = G.row[i];
    G.krow[key_of(p) * K + kk] = q >= 0 ? key_of(q) : -1;
  }
  constexpr int CHUNK_SHIFT = BIG_T == 1024 ? 15 : BIG_T == 512 ? 14 : 13;  // BIG_T leaf words per chunk
  static_assert((32 * BIG_T) == (1 << CHUNK_SHIFT), "chunk = BIG_T leaf words");
  if (!asc) {
    if (warp == 0) {
      const bool src = lane == 0;
      const int key = key_of(0);
      if (src) {
        atomicOr(seen + (key >> 5), 1u << (key & 31));
        S.nsrc = 1;
      }
      leaf_insert(T.leaf, &S.hi_chunk, key, src, CHUNK_SHIFT);
    }
  } else {
    for (int p0 = 1; p0 < k; p0 += BIG_T) {
      const int p = p0 + tid;
      const bool src = p < k && (G.sfl[p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT);
      const int key = src ? key_of(p) : 0;
      if (src) {
        atomicOr(seen + (key >> 5), 1u << (key & 31));
        atomicAdd(&S.nsrc, 1);
      }
      leaf_insert(T.leaf, &S.hi_chunk, key, src, CHUNK_SHIFT);
    }
  }
  __syncthreads();
  if (S.nsrc == 0) {  // empty ascending flood keeps the previous labels
    for (int p = tid; p < k; p += BIG_T) cout[p] = cin[p];
    __syncthreads();
    return;
  }
  int e = 0;
  // instrumentation accumulates in registers (a global += per tick would
  // stall thread 0 on a load and perturb the barriers being measured)
  long long tacc[DBG_W];
#pragma unroll
  for (int i = 0; i < DBG_W; i++) tacc[i] = 0;
  long long tq = clock64(), tn;
#define BIG_TICK(slot)                          \
  if (dbg && tid == 0) {                        \
    tn = clock64();                             \
    dbg[slot] += tn - tq;                       \
    tq = tn;                                    \
  }
  for (;;) {
    BIG_TICK(8)
    if (tid == 0) S.xcnt = 0;
    // (a) candidates = the top Beff keys of F.  The CTA scans leaf words in
    // chunks of BIG_T words (one word per thread, thread 0 = highest word),
    // skipping empty chunks with the level-2 counts; a block scan of the
    // popcounts gives every key its descending rank.
    int nc = 0;
    {
      const int hi = S.hi_chunk;
      int top_found = -1;
      for (int ch = hi; ch >= 0 && nc < Beff; ch--) {
        const int w = ch * BIG_T + (BIG_T - 1 - tid);
        uint32_t word = w < T.nw0 ? T.leaf[w] : 0u;
        int tot;
        int r = nc + big_scan_excl(__popc(word), S.wsum, tot);
        if (dbg && tid == 0) {
          tn = clock64();
          tacc[16] += 1;
          tacc[17] += tn - tq;
          tq = tn;
        }
        while (word && r < Beff) {
          int b = 31 - __clz(word);
          word &= ~(1u << b);
          S.newmax[r] = -1;
          S.cand_key[r++] = (w << 5) + b;
        }
        if (tot > 0 && top_found < 0) top_found = ch;
        nc = min(Beff, nc + tot);
        __syncthreads();
        if (dbg && tid == 0) {
          tn = clock64();
          tacc[18] += tn - tq;
          tq = tn;
        }
      }
      // chunks above the first non-empty one are empty: start lower next time
      if (tid == 0) S.hi_chunk = top_found;
    }
    BIG_TICK(9)
    if (nc == 0) break;
    if (tid == 0) S.cut = nc;
    // the label slot of candidate tid, in flight until the commit (BIG_B <= BIG_T)
    const int cand_p = tid < nc ? G.inv[S.cand_key[tid]] : 0;
    BIG_TICK(10)
    // (b) exposure maxima of every candidate: all row loads issued first
    {
      constexpr int PPT = (BIG_B * K + BIG_T - 1) / BIG_T;
      int nk[PPT];
#pragma unroll
      for (int t = 0; t < PPT; t++) {
        const int i = tid + t * BIG_T;
        nk[t] = -1;
        if (i < nc * K) {
          const int c = i / K;
          nk[t] = G.krow[S.cand_key[c] * K + (i - c * K)];
        }
      }
#pragma unroll
      for (int t = 0; t < PPT; t++) {
        const int i = tid + t * BIG_T;
        if (i < nc * K) {
          int q = nk[t];
          if (q >= 0 && !seen_test(seen, q)) atomicMax(&S.newmax[i / K], q);
          else q = -1;
          S.pair_key[i] = q;
        }
      }
    }
    __syncthreads();
    BIG_TICK(11)
    // (c) prefix max and first preemption: warp 0, 8 candidates per lane
    if (warp == 0) {
      constexpr int PER = BIG_B / 32;
      int loc[PER];
      int m = -1;
#pragma unroll
      for (int t = 0; t < PER; t++) {
        int i = lane * PER + t;
        int v = i < nc ? S.newmax[i] : -1;
        m = max(m, v);
        loc[t] = m;
      }
      int P = m;  // inclusive scan of lane maxima
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, P, o);
        if (lane >= o) P = max(P, y);
      }
      int carry = __shfl_up_sync(0xffffffffu, P, 1);
      if (lane == 0) carry = -1;
      int first = 0x7fffffff;
#pragma unroll
      for (int t = 0; t < PER; t++) {
        int i = lane * PER + t;
        if (i + 1 < nc && max(carry, loc[t]) > S.cand_key[i + 1] && first == 0x7fffffff) first = i + 1;
      }
      first = __reduce_min_sync(0xffffffffu, first);
      if (lane == 0 && first != 0x7fffffff) S.cut = first;
    }
    __syncthreads();
    BIG_TICK(12)
    const int j = S.cut;
    // (d) commit the prefix: labels, leave F; its exposures join F
    {
      const bool v = tid < j;
      if (v) cout[cand_p] = asc ? (e + tid) : (k - 1 - (e + tid));
      leaf_remove(T.leaf, v ? S.cand_key[tid] : 0, v);
    }
    BIG_TICK(13)
    const int kappa = S.cand_key[nc - 1];  // every key of F above kappa is known
    for (int i0 = 0; i0 < j * K; i0 += BIG_T) {
      int i = i0 + tid;
      int q = i < j * K ? S.pair_key[i] : -1;
      bool ins = false;
      if (q >= 0) {
        uint32_t bit = 1u << (q & 31);
        ins = !(atomicOr(seen + (q >> 5), bit) & bit);
      }
      leaf_insert(T.leaf, &S.hi_chunk, ins ? q : 0, ins, CHUNK_SHIFT);
      if (ins && q > kappa) {
        int x = atomicAdd(&S.xcnt, 1);
        if (x < BIG_XMAX) S.xkey[x] = q;
      }
    }
    e += j;
    if (dbg && tid == 0) {
      tacc[1] += 1;
      tacc[2] += nc;
      tacc[3] += j;
    }
    if (j == nc && nc == Beff && Beff < BIG_B) Beff *= 2;
    else if (j * 4 < Beff && Beff > 8) Beff >>= 1;
    __syncthreads();
    BIG_TICK(14)
    // (e) climb continuation (warp 0): while the largest known exposure beats
    // the next candidate, it IS the next extraction; follow it with one row
    // load per hop instead of a full CTA step.  Exposures above kappa join
    // the known list; everything else stays in the bit set.
    const int xc = S.xcnt;
    if (j <= 4 && xc > 0 && xc <= BIG_XMAX) {  // block-uniform: climbs only
      if (dbg && tid == 0) tacc[19] += 1;
      if (warp == 0) {
        const int bound = j < nc ? S.cand_key[j] : kappa;
        int m = xc, ee = e;
        for (int hop = 0; hop < BIG_HOPS && m > 0; hop++) {
          // argmax of the known list (keys are distinct): one packed
          // (key, index) reduction when keys fit in 23 bits
          int bk = -1, bi = 0x7fffffff;
          if (k < (1 << 22)) {
            unsigned pk = 0u;
            for (int i = lane; i < m; i += 32) pk = max(pk, ((unsigned)(S.xkey[i] + 1) << 9) | (unsigned)i);
            pk = __reduce_max_sync(0xffffffffu, pk);
            bk = (int)(pk >> 9) - 1;
            bi = (int)(pk & 511u);
          } else {
            for (int i = lane; i < m; i += 32) bk = max(bk, S.xkey[i]);
            bk = __reduce_max_sync(0xffffffffu, bk);
            for (int i = lane; i < m; i += 32)
              if (S.xkey[i] == bk) bi = i;
            bi = __reduce_min_sync(0xffffffffu, bi);
          }
          if (bk <= bound) break;
          const int key2 = lane < K ? G.krow[bk * K + lane] : -1;
          __syncwarp();
          if (lane == 0) {
            cout[G.inv[bk]] = asc ? ee : (k - 1 - ee);
            S.xkey[bi] = S.xkey[m - 1];
          }
          leaf_remove(T.leaf, bk, lane == 0);
          ee++;
          m--;
          __syncwarp();
          bool ins = false;
          if (key2 >= 0) {
            uint32_t bit = 1u << (key2 & 31);
            ins = !(atomicOr(seen + (key2 >> 5), bit) & bit);
          }
          leaf_insert(T.leaf, &S.hi_chunk, ins ? key2 : 0, ins, CHUNK_SHIFT);
          const bool add = ins && key2 > kappa;
          const unsigned am = __ballot_sync(0xffffffffu, add);
          if (m + __popc(am) > BIG_XMAX) break;  // list full: leave the rest to the CTA
          if (add) S.xkey[m + __popc(am & lanemask_lt())] = key2;
          m += __popc(am);
          __syncwarp();
        }
        if (lane == 0) S.enew = ee;
      }
      __syncthreads();
      if (dbg && tid == 0) tacc[15] += S.enew - e;
      e = S.enew;
    }
  }
#undef BIG_TICK
  if (dbg && tid == 0) {
#pragma unroll
    for (int i = 1; i < DBG_W; i++)
      if (i < 4 || i > 7) dbg[i] += tacc[i];
  }
}

// after a descending flood: SF_MIN marks, true if an unauthorized minimum
template <int K>
__device__ bool big_check_minima(BigSmem &S, BigRegion &G, const int *cur) {
  if (threadIdx.x == 0) S.red = 0;
  __syncthreads();
  bool bad = false;
  for (int p = 1 + threadIdx.x; p < G.k; p += BIG_T) {
    const int *row = G.row + p * K;
    int c = cur[p];
    bool mn = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = row[kk];
      if (q >= 0 && cur[q] < c) mn = false;
    }
    uint8_t f = G.sfl[p];
    f = mn ? (f | SF_MIN) : (f & (uint8_t)~SF_MIN);
    G.sfl[p] = f;
    if (mn && !(f & SF_OUT)) bad = true;
  }
  if (bad) atomicOr(&S.red, 1);
  __syncthreads();
  bool r = S.red != 0;
  __syncthreads();
  return r;
}

// after an ascending flood: true if a vertex other than the saddle is a max
template <int K>
__device__ bool big_check_maxima(BigSmem &S, BigRegion &G, const int *cur) {
  if (threadIdx.x == 0) S.red = 0;
  __syncthreads();
  bool bad = false;
  for (int p = 1 + threadIdx.x; p < G.k; p += BIG_T) {
    const int *row = G.row + p * K;
    int c = cur[p];
    bool mx = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = row[kk];
      if (q >= 0 && cur[q] > c) mx = false;
    }
    if (mx) bad = true;
  }
  if (bad) atomicOr(&S.red, 1);
  __syncthreads();
  bool r = S.red != 0;
  __syncthreads();
  return r;
}

__device__ bool big_states_equal(BigSmem &S, const int *a, const int *b, int k) {
  if (threadIdx.x == 0) S.red = 0;
  __syncthreads();
  bool diff = false;
  for (int p = threadIdx.x; p < k; p += BIG_T)
    if (a[p] != b[p]) diff = true;
  if (diff) atomicOr(&S.red, 1);
  __syncthreads();
  bool r = S.red == 0;
  __syncthreads();
  return r;
}

// Region adjacency rows, has_outside flags, identity initial order and v0 for
// every large region, computed by the whole GPU before the flood kernel
// (_kernels.py:453-481).  grid.y = big-region index, grid.x = slot chunks.
template <int NDIM>
__global__ void __launch_bounds__(256) k_big_rows(LocArgs A, BigArgs Bg) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  const int qi = blockIdx.y;
  const int rid = A.order[Bg.qbase + qi];
  const int lo = A.rptr[rid];
  const int k = A.rptr[rid + 1] - lo;
  const int n = (int)A.g.n;
  const int s = A.verts[lo];
  const int srank = eff_rank(A.rank, s, A.rev, n);
  int mine = 0x7fffffff;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < k; p += gridDim.x * blockDim.x) {
    int x, y, z;
    coords(A.g, A.verts[lo + p], x, y, z);
    bool out = false;
    int *row = Bg.nrow + ((size_t)lo + p) * K;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int u = nbr_at(A.g, x, y, z, kk);
      row[kk] = member(A, u, rid, s);
      if (p >= 1 && u >= 0 && eff_rank(A.rank, u, A.rev, n) < srank) out = true;
    }
    A.sfl[lo + p] = out ? SF_OUT : 0;
    if (out && p < mine) mine = p;
    A.buf0[lo + p] = p;
  }
  mine = __reduce_min_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine != 0x7fffffff) atomicMin(Bg.v0 + qi, mine);
}

template <int NDIM>
__global__ void __launch_bounds__(BIG_T) k_localize_big(LocArgs A, BigArgs Bg) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  extern __shared__ __align__(16) unsigned char smraw[];
  BigSmem &S = *reinterpret_cast<BigSmem *>(smraw);
  const int tid = threadIdx.x;
  const int n = (int)A.g.n;
  for (;;) {
    if (tid == 0) S.qi = atomicAdd(Bg.queue, 1);
    __syncthreads();
    const int qi = S.qi;
    __syncthreads();
    if (qi >= Bg.nbig) break;
    BigRegion G;
    G.rid = A.order[Bg.qbase + qi];
    G.lo = A.rptr[G.rid];
    G.k = A.rptr[G.rid + 1] - G.lo;
    G.verts = A.verts + G.lo;
    G.sfl = A.sfl + G.lo;
    G.inv = Bg.inv + G.lo + G.rid;
    G.row = Bg.nrow + (size_t)G.lo * K;
    G.krow = Bg.nrowkey + ((size_t)G.lo + G.rid) * K;
    G.s = G.verts[0];
    const int k = G.k, rid = G.rid, lo = G.lo;
    int *const b0 = A.buf0 + lo, *const b1 = A.buf1 + lo, *const b2 = A.buf2 + lo;
#define BUF(i) ((i) % 3 == 0 ? b0 : ((i) % 3 == 1 ? b1 : b2))
    // shared-memory layout: counts, leaf bits (if they fit), seen bits
    if (tid == 0) {
      CTree &T = S.T;
      T.nw0 = (k + 1 + 31) >> 5;
      T.nb[0] = T.nw0;
      int l = 0;
      while (T.nb[l] > 32) {
        T.nb[l + 1] = (T.nb[l] + 31) >> 5;
        l++;
      }
      T.top = l;
      uint32_t *sp = S.bits;
      int used = 0;
      const int seen_words = T.nw0;
      uint32_t *gp = Bg.gbits + 3 * (((size_t)lo + rid + 31) >> 5) + 8 * (size_t)rid;
      int ncnt = 0;
      for (int i = 1; i <= T.top; i++) ncnt += T.nb[i];
      const bool cnt_smem = ncnt <= BIG_SMEM_WORDS;  // else every level in global
      for (int i = 1; i <= T.top; i++) {
        if (cnt_smem) {
          T.cnt[i] = (int *)sp;
          sp += T.nb[i];
          used += T.nb[i];
        } else {
          T.cnt[i] = (int *)gp;
          gp += T.nb[i];
        }
      }
      if (used + T.nw0 <= BIG_SMEM_WORDS) {
        T.leaf = sp;
        sp += T.nw0;
        used += T.nw0;
      } else {
        T.leaf = gp;
        gp += T.nw0;
      }
      S.seen = (used + seen_words <= BIG_SMEM_WORDS) ? sp : gp;
    }
    __syncthreads();
    const int qa = Bg.qbase + qi;  // absolute big-queue position
    long long *dbg = (d_dbg_on && qa < DBG_MAX) ? d_dbg + qa * DBG_W : nullptr;
    long long c0 = clock64(), c1;
    // rows, has_outside and v0 were produced by k_big_rows (grid-wide)
    if (tid == 0) S.v0 = Bg.v0[qa];
    __syncthreads();
    const int v0 = S.v0;
    if (v0 == 0x7fffffff) {
      for (int p = tid; p < k; p += BIG_T) A.out[lo + p] = p;
      if (tid == 0) {
        A.status[rid] = 1;
        A.n_iters[rid] = 0;
      }
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      b0[0] = 0x7fffffff;
      b0[v0] = (int)0x80000000;
      if (dbg) dbg[0] = k;
    }
    __syncthreads();
    c1 = clock64();
    if (dbg && tid == 0) dbg[6] += c1 - c0;
    int t = 0, status = 0, fin = 0, Beff = 32;
    for (;;) {
      c1 = clock64();
      big_flood<K>(S, G, false, BUF(t), BUF(t + 1), Beff, dbg);
      c0 = clock64();
      if (dbg && tid == 0) dbg[4] += c0 - c1;
      t++;
      bool bad = big_check_minima<K>(S, G, BUF(t));
      c1 = clock64();
      if (dbg && tid == 0) dbg[5] += c1 - c0;
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && big_states_equal(S, BUF(t), BUF(t + 1), k)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
      c1 = clock64();
      big_flood<K>(S, G, true, BUF(t), BUF(t + 1), Beff, dbg);
      c0 = clock64();
      if (dbg && tid == 0) dbg[4] += c0 - c1;
      t++;
      bad = big_check_maxima<K>(S, G, BUF(t));
      c1 = clock64();
      if (dbg && tid == 0) dbg[5] += c1 - c0;
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && big_states_equal(S, BUF(t), BUF(t + 1), k)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
    }
    const int *fb = BUF(fin);
#undef BUF
    for (int p = tid; p < k; p += BIG_T) A.out[lo + p] = fb[p];
    if (tid == 0) {
      A.status[rid] = status;
      A.n_iters[rid] = t;
      if (dbg) dbg[7] = t;
    }
    __syncthreads();
  }
}

}  // namespace lts
