// localize_big.cuh -- exact priority floods of large regions, one CTA each,
// extracting many vertices per synchronisation step.
//
// A priority flood's extraction order depends only on which vertices are in
// the frontier F when each extraction happens.  Let f1 > f2 > ... be F sorted
// by key and let new_i be the unseen neighbours exposed by extracting f_i.
// Then f1..fj are the next j extractions, in that order, iff
//     max key(new_1 u ... u new_i) < key(f_{i+1})   for every i < j.
// Each step therefore takes the top-B keys of F (B = one per thread), every
// thread loads its candidate's neighbour row and computes its exposure
// maximum, one block-wide prefix-max scan finds the first preemption, and the
// prefix is committed.  On the cfg3 regions a flood needs ~1% as many steps as
// extractions, so the step's latency is the kernel's cost: a step is one
// L2 round trip (the candidates' rows) plus shared-memory scans and four
// barriers of BIG_T/32 warps.
//
// Keys are a permutation of a small integer range (the region's local order),
// so F is a bit set over key space ("leaf" words, in shared memory unless the
// region is very large); the top-B keys come from a descending chunked scan
// of the leaf words, starting at the highest non-empty chunk.  "seen" is a bit
// set over keys.  The neighbour rows of the flood are indexed by key and the
// key -> local index map is rebuilt per flood by k_big_setup (grid-wide).
// Semantics follow _localize_one (_kernels.py:443-575) exactly, including the
// empty-ascending-flood case and the period-2 cycle jump (contract D5).
#pragma once
#include "localize.cuh"

namespace lts {

#ifndef LTS_BIG_T
#define LTS_BIG_T 256
#endif
constexpr int BIG_T = LTS_BIG_T;              // threads per flood CTA
constexpr int BIG_B = BIG_T;                  // candidates per step: one per thread
constexpr int BIG_NW = BIG_T / 32;
#ifndef LTS_BIG_WPT
#define LTS_BIG_WPT 4
#endif
constexpr int BIG_WPT = LTS_BIG_WPT;          // leaf words per thread in the candidate scan
constexpr int BIG_CHUNK = BIG_T * BIG_WPT;    // leaf words per scan chunk
constexpr int BIG_CHUNK_SHIFT = BIG_CHUNK == 512 ? 14 : BIG_CHUNK == 1024 ? 15 : BIG_CHUNK == 2048 ? 16 : 17;
static_assert((32 * BIG_CHUNK) == (1 << BIG_CHUNK_SHIFT), "chunk = BIG_CHUNK leaf words");
constexpr int BIG_SMEM_WORDS = 16 * 1024;     // bit-set words in shared memory (rest of the SM is L1)
#ifndef LTS_BIG_THRESHOLD
#define LTS_BIG_THRESHOLD 256
#endif
constexpr int BIG_THRESHOLD = LTS_BIG_THRESHOLD;  // regions with k > this use this kernel

#ifndef LTS_LEVEL_NMAX
#define LTS_LEVEL_NMAX 256
#endif

struct BigArgs {
  int *v0;           // per big region: first admissible boundary minimum
  int *inv;          // key -> local index, S + R entries (region base lo + rid)
  uint32_t *gbits;   // spill space for leaf / seen bit sets
  int *nrow;         // per slot: K local neighbour indices (-1 = not a member)
  int *nrowkey;      // per key: K neighbour keys of the current flood (rows in key order)
  int qbase, nbig;   // regions order[qbase .. qbase+nbig)
  int *queue;
  int *st;           // per big region: BST_W ints of flood state (below)
  int *nactive;      // regions still flooding after the last decide
  unsigned long long *work;  // sum of the region sizes flooded (report)
  const int *bpre;   // nbig + 1: exclusive prefix of the big-region sizes (queue order)
  int bslots;        // bpre[nbig]: slots of all big regions
};

// big-queue index of flat big-region slot i (largest qi with bpre[qi] <= i)
__device__ __forceinline__ int big_locate(const BigArgs &Bg, int i) {
  int lo = 0, hi = Bg.nbig - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (Bg.bpre[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// per-region flood state, kept in global memory between the grid-wide
// setup / check kernels and the one-CTA-per-region flood kernel
// BST_NSRC: sources of the coming ascending flood; BST_LEVEL: the region floods
// level-parallel (localize_level.cuh) instead of in k_big_flood
// BST_NMAX: local maxima of the region's initial order (its roughness)
enum { BST_T = 0, BST_ACTIVE, BST_FIN, BST_STATUS, BST_BAD, BST_DIFF, BST_NSRC, BST_LEVEL, BST_NMAX, BST_W = 12 };

// optional per-region instrumentation (lts_debug_big_stats): big-queue slot i
// records [k, frontier steps, candidates, committed, flood cycles, global-rule
// steps, global-rule commits, n_iters, frontier-rule gather, probe, cut,
// commit cycles, steps with j <= 8, j <= 32, sum ceil(j/32), unpreempted
// steps, warp-mode steps, global-rule cycles, global-rule attempts, warp-mode
// cycles, warp-step gather / probe / cut+commit cycles]
constexpr int DBG_MAX = 256, DBG_W = 24;
__device__ long long d_dbg[DBG_MAX * DBG_W];
__device__ int d_dbg_on;

struct BigSmem {
  int pref[BIG_T];
  int wsum[BIG_NW];
  int wmax[BIG_NW];
  int cutbuf[2], hi_chunk, nw, nw4;  // cut: first failing candidate (double-buffered per step)
  int ghi_chunk, gblock;  // global rule: highest possibly unextracted chunk, blocking key
  int hi_sw, nsw4;        // frontier summary: highest possibly non-empty summary word, words
  int hw;                 // highest possibly non-empty leaf word (warp mode)
  int keep_sum;           // the summary is maintained (large regions only)
  int wmode, ew;          // warp mode on; extraction count handed back by warp 0
  uint32_t *leaf;   // frontier bit set over keys
  uint32_t *seen;   // bit set over keys
  uint32_t *sum;    // frontier summary: bit w set iff leaf word w is non-zero
  __align__(16) uint32_t bits[BIG_SMEM_WORDS];
};

struct BigRegion {
  int rid, lo, k, s;
  const int *verts;
  const int *row;   // k*K local neighbour indices, by local index
  int *krow;        // (k+1)*K neighbour keys of the current flood, by key (-1: not a member)
  uint8_t *sfl;
  int *inv;
};

// desc floods map the sentinels +BIG -> k, -BIG -> 0; asc floods reverse
__device__ __forceinline__ int flood_key(int c, bool asc, int k) {
  if (asc) return k - 1 - c;
  if (c == 0x7fffffff) return k;
  if (c == (int)0x80000000) return 0;
  return c;
}

// block-wide exclusive sum over threads in tid order, one barrier; the caller
// barriers before wsum is written again
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
  int pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < BIG_NW; w++) {
    const int v = wsum[w];
    pre += w < warp ? v : 0;
    tot += v;
  }
  total = tot;
  return pre + inc - x;
}

// Top-BIG_B set bits of a key-space bit set, descending, one per thread.
// word4(b) returns the four words b..b+3 (zero past the key range); hi_chunk
// (shared) is an upper bound of the highest non-empty chunk and is lowered to
// the highest chunk found non-empty.  A chunk of leaf words (thread 0 owns the
// highest BIG_WPT words) is popcounted and scanned once; then candidate slot i
// binary-searches the per-thread prefix for the owner of its key and selects
// the bit, so every thread does the same small amount of work however the
// keys cluster.  Returns the candidate count (block-uniform); key = -1 for
// threads without a candidate.
template <class W4>
__device__ __forceinline__ int big_gather(BigSmem &S, int &hi_chunk, W4 word4, int &key, int *iters = nullptr) {
  const int tid = threadIdx.x;
  int nc = 0;
  key = -1;
  const int hi = hi_chunk;
  int top_found = -1, nit = 0;
  for (int ch = hi; ch >= 0 && nc < BIG_B; ch--, nit++) {
    const int base = ch * BIG_CHUNK + (BIG_T - 1 - tid) * BIG_WPT;
    const uint4 w = word4(base);
    const int cnt = __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
    int tot;
    const int r = big_scan_excl(cnt, S.wsum, tot);
    S.pref[tid] = r;
    __syncthreads();
    const int want = tid - nc;
    if (want >= 0 && want < tot) {
      int lo = 0, up = BIG_T - 1;  // owner: the last thread with pref <= want
#pragma unroll
      for (int it = 0; it < 16 && lo < up; it++) {
        const int mid = (lo + up + 1) >> 1;
        if (S.pref[mid] <= want) lo = mid;
        else up = mid - 1;
      }
      int rem = want - S.pref[lo];
      const int b0 = ch * BIG_CHUNK + (BIG_T - 1 - lo) * BIG_WPT;
      const uint4 ow = word4(b0);
      const uint32_t ws[4] = {ow.w, ow.z, ow.y, ow.x};  // highest word first
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const int c = __popc(ws[h]);
        if (rem < c) {
          const uint32_t x = ws[h];
          const int need = rem + 1;  // need-th highest set bit of x
          int bpos = 0;
#pragma unroll
          for (int sft = 16; sft >= 1; sft >>= 1)
            if (__popc(x >> (bpos + sft)) >= need) bpos += sft;
          key = ((b0 + 3 - h) << 5) + bpos;
          break;
        }
        rem -= c;
      }
    }
    if (tot > 0 && top_found < 0) top_found = ch;
    nc = min(BIG_B, nc + tot);
  }
  // chunks above top_found are empty (when the loop ran no chunk, hi < 0 and
  // the value written is unchanged, so no barrier is needed against readers)
  if (tid == 0) hi_chunk = top_found;
  if (iters) *iters = nit;
  return nc;
}

__device__ __forceinline__ bool big_bit(const uint32_t *b, int x) { return (b[x >> 5] >> (x & 31)) & 1u; }

// rem-th highest set bit of x (rem < popc(x))
__device__ __forceinline__ int big_nth_high(uint32_t x, int rem) {
  const int need = rem + 1;
  int bpos = 0;
#pragma unroll
  for (int sft = 16; sft >= 1; sft >>= 1)
    if (__popc(x >> (bpos + sft)) >= need) bpos += sft;
  return bpos;
}

// ---- frontier summary -----------------------------------------------------
// sum bit w is set whenever leaf word w gains a key and cleared lazily by the
// warp gather when it finds the word empty.  A stale set bit only costs a
// look; a cleared bit over a non-empty word cannot happen because bits are
// cleared only by the gathering warp while no other warp commits.
#ifndef LTS_BIG_SUM_MIN_WORDS
#define LTS_BIG_SUM_MIN_WORDS 4096  // regions with fewer leaf words scan without a summary
#endif
__device__ __forceinline__ void big_front_add(BigSmem &S, int x, bool ks) {
  atomicOr(S.leaf + (x >> 5), 1u << (x & 31));
  if (ks) atomicOr(S.sum + (x >> 10), 1u << ((x >> 5) & 31));
}

template <int K>
__device__ __forceinline__ void big_row(const BigRegion &G, int key, int (&q)[K]) {
  const int2 *row = reinterpret_cast<const int2 *>(G.krow + (size_t)key * K);
#pragma unroll
  for (int h = 0; h < K / 2; h++) {
    const int2 v = row[h];
    q[2 * h] = v.x;
    q[2 * h + 1] = v.y;
  }
}

// largest lane u with v_u <= t for a lane-ascending (non-decreasing) v
__device__ __forceinline__ int warp_owner(int v, int t) {
  int lo = 0;
#pragma unroll
  for (int sft = 16; sft >= 1; sft >>= 1)
    if (__shfl_sync(0xffffffffu, v, lo + sft) <= t) lo += sft;
  return lo;
}

__device__ __forceinline__ int warp_incl_sum(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Highest non-empty leaf word <= w0 (or -1), for the single warp: the
// summary words are read 32 at a time from w0's downward; a set summary bit
// whose leaf word turns out empty (stale: the summary is only ever set on
// insert) is cleared by the caller, which then asks again.
__device__ __forceinline__ int big_warp_next_word(BigSmem &S, int w0) {
  const int lane = threadIdx.x & 31;
  const uint32_t *const sum = S.sum;
  for (int s0 = w0 >> 5; s0 >= 0; s0 -= 32) {
    const int sw = s0 - lane;
    uint32_t m = sw >= 0 ? sum[sw] : 0u;
    if (sw == (w0 >> 5)) m &= (w0 & 31) == 31 ? 0xffffffffu : ((2u << (w0 & 31)) - 1u);
    const unsigned nz = __ballot_sync(0xffffffffu, m != 0u);
    if (nz) {
      const int l = __ffs(nz) - 1;
      const uint32_t ml = __shfl_sync(0xffffffffu, m, l);
      return (s0 - l) * 32 + 31 - __clz(ml);
    }
  }
  return -1;
}

// Frontier keys for the single-warp step, descending, lane i gets the i-th
// (-1 past the count): every frontier key of the 32 leaf words below the
// highest non-empty one (at most 32 of them).  Any exact prefix of the
// frontier order is a valid candidate list, so a sparse window simply yields
// fewer candidates -- and rough floods commit only a few keys per step
// anyway.  Lowers hw to the top non-empty word.
__device__ int big_warp_gather(BigSmem &S, int &key) {
  const int lane = threadIdx.x & 31;
  volatile uint32_t *const leaf = S.leaf;
  key = -1;
  int hw = S.hw;
  int nc = 0;
  while (hw >= 0) {
    const int w = hw - lane;
    const uint32_t lw = w >= 0 ? leaf[w] : 0u;
    const unsigned nz = __ballot_sync(0xffffffffu, lw != 0u);
    if (nz == 0u && !S.keep_sum) {  // small region: no summary, step down a window
      hw -= 32;
      continue;
    }
    if (nz == 0u) {
      // an empty window: clear its (stale) summary bits, then jump to the
      // next non-empty word the summary knows of
      if (lane == 0) {
        const int lo = max(hw - 31, 0);
        for (int sw = hw >> 5; sw >= (lo >> 5); sw--) {
          const int a = max(lo, sw * 32) - sw * 32, b = min(hw, sw * 32 + 31) - sw * 32;
          const uint32_t mask = (b == 31 ? 0xffffffffu : ((2u << b) - 1u)) & ~((1u << a) - 1u);
          atomicAnd(S.sum + sw, ~mask);
        }
      }
      __syncwarp();
      hw = big_warp_next_word(S, hw - 32);
      continue;
    }
    const int top = __ffs(nz) - 1;  // lanes run from the highest word down
    const int c = __popc(lw);
    const int inc = warp_incl_sum(c);
    const int tot = __shfl_sync(0xffffffffu, inc, 31);
    const int ex = inc - c;
    const int o = warp_owner(ex, lane);
    const uint32_t lwo = __shfl_sync(0xffffffffu, lw, o);
    const int eo = __shfl_sync(0xffffffffu, ex, o);
    if (lane < tot) key = ((hw - o) << 5) + big_nth_high(lwo, lane - eo);
    nc = min(32, tot);
    hw -= top;
    break;
  }
  if (lane == 0) S.hw = hw;
  __syncwarp();
  return nc;
}

#ifndef LTS_BIG_HW_FROM_BLOCK
#define LTS_BIG_HW_FROM_BLOCK 1
#endif
#ifndef LTS_BIG_WARP_ENTER
#define LTS_BIG_WARP_ENTER 24  // a block step committing fewer keys enters warp mode
#endif
#ifndef LTS_BIG_WARP_EXIT
#define LTS_BIG_WARP_EXIT 28   // a warp step committing this many returns to block mode
#endif
#ifndef LTS_BIG_WARP_FREE
#define LTS_BIG_WARP_FREE 8    // ... or this many with no preemption
#endif

// One exact priority flood of a large region (the e-th extraction gets label
// k-1-e for descending floods, e for ascending ones).  Each iteration commits
// an exact prefix of the extraction order by one of two rules:
//  (g) global rule: let x_1 > x_2 > ... be the unextracted keys.  x_i is the
//      i-th next extraction iff x_1..x_i are each in the frontier, or have a
//      higher neighbour (which is then an earlier x_j), or an extracted
//      neighbour: the frontier max is then always the largest unextracted
//      key.  So the longest prefix of the top-B unextracted keys whose members
//      pass that local test is committed at once.  Floods after the first
//      (where the order is already nearly monotone) commit most of a region
//      this way.  The first failing key is an unreached local maximum; the
//      rule is skipped until that vertex enters the frontier.
//  (f) frontier rule: with f1 > f2 > ... the frontier and new_i the unseen
//      neighbours exposed by f_i, f1..fj are the next j extractions iff
//      max key(new_1 u ... u new_i) < key(f_{i+1}) for every i < j.
// Keys are a permutation of [0, k] minus one unused key (the region's local
// order with the +-BIG sentinels of the first flood mapped to k and 0), so
// the frontier ("leaf") and the seen set are bit sets over key space;
// extracted = seen and not leaf.
// The frontier rule runs in one of two modes.  Block mode: B = BIG_T
// candidates from a chunk scan of the leaf words, block-wide scans (smooth
// floods commit tens to hundreds of keys per step).  Warp mode: warp 0 alone
// takes the top 32 keys through the frontier summary and runs the whole step
// with shuffles and no block barrier (rough floods commit a few keys per
// step, so the step latency is what counts).
template <int K>
__device__ void big_flood(BigSmem &S, BigRegion &G, bool asc, const int *cin, int *cout, int unused_key,
                          long long *dbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = G.k;
  uint32_t *const leaf = S.leaf;
  uint32_t *const seen = S.seen;
  const int nw = S.nw4;
  const int nwv = S.nw;                       // words holding keys 0..k
  const uint32_t lastmask = ((k + 1) & 31) ? ((1u << ((k + 1) & 31)) - 1u) : 0xffffffffu;
  for (int i = tid; i < nw; i += BIG_T) {
    leaf[i] = 0u;
    seen[i] = 0u;
  }
  for (int i = tid; i < S.nsw4; i += BIG_T) S.sum[i] = 0u;
  const bool ks = S.nw4 > LTS_BIG_SUM_MIN_WORDS;
  if (tid == 0) {
    S.keep_sum = ks;
    S.hi_sw = -1;
    S.hw = -1;
    S.wmode = 0;
    S.hi_chunk = -1;
    S.ghi_chunk = k >> BIG_CHUNK_SHIFT;
    S.gblock = -1;
    S.cutbuf[0] = S.cutbuf[1] = 0x7fffffff;
  }
  __syncthreads();
  // the one key no slot maps to counts as extracted
  if (tid == 0) seen[unused_key >> 5] |= 1u << (unused_key & 31);
  // sources: the saddle (desc) or every admissible boundary minimum (asc)
  int mine = 0;
  if (!asc) {
    if (tid == 0) {
      const int key = flood_key(cin[0], false, k);
      seen[key >> 5] |= 1u << (key & 31);
      big_front_add(S, key, ks);
      S.hi_chunk = key >> BIG_CHUNK_SHIFT;
      S.hi_sw = key >> 10;
      S.hw = key >> 5;
      mine = 1;
    }
  } else {
    int mch = -1;
    for (int p = 1 + tid; p < k; p += BIG_T) {
      if ((G.sfl[p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT)) {
        const int key = flood_key(cin[p], true, k);
        atomicOr(seen + (key >> 5), 1u << (key & 31));
        big_front_add(S, key, ks);
        mch = max(mch, key >> 5);
        mine = 1;
      }
    }
    mch = __reduce_max_sync(0xffffffffu, mch);
    if (lane == 0 && mch >= 0) {
      atomicMax(&S.hw, mch);
      atomicMax(&S.hi_sw, mch >> 5);
      atomicMax(&S.hi_chunk, mch >> (BIG_CHUNK_SHIFT - 5));
    }
  }
  if (__syncthreads_or(mine) == 0) {  // empty ascending flood keeps the previous labels
    for (int p = tid; p < k; p += BIG_T) cout[p] = cin[p];
    __syncthreads();
    return;
  }
  const auto leaf4 = [&](int b) -> uint4 {
    return b < nw ? *reinterpret_cast<const uint4 *>(leaf + b) : make_uint4(0u, 0u, 0u, 0u);
  };
  const auto unext4 = [&](int b) -> uint4 {  // unextracted = not seen, or in the frontier
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int i = b + j;
      uint32_t x = i < nwv ? (~seen[i] | leaf[i]) : 0u;
      if (i == nwv - 1) x &= lastmask;
      w[j] = x;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  };
  int e = 0, par = 0;
  long long nst = 0, ncand = 0, ngs = 0, ngc = 0, nga = 0, nws = 0;
  long long tq = 0, tn;
  if (dbg && tid == 0) tq = clock64();
#define BIG_TICK(i)         \
  if (dbg && tid == 0) {    \
    tn = clock64();         \
    dbg[i] += tn - tq;      \
    tq = tn;                \
  }
  while (e < k) {
    int key, q[K];
    int *const cut = &S.cutbuf[par];
    // ---- (g) global rule ---------------------------------------------------
    int j = 0;
    const int gb = S.gblock;
    if (gb < 0 || big_bit(seen, gb)) {
      nga++;
      const int ng = big_gather(S, S.ghi_chunk, unext4, key);
      const bool isc = tid < ng;
      int cand_p = 0;
      if (isc) {
        cand_p = G.inv[key];
        big_row<K>(G, key, q);
        bool ok = big_bit(leaf, key);
#pragma unroll
        for (int kk = 0; kk < K; kk++) {
          const int x = q[kk];
          if (x > key) ok = true;                                               // a higher neighbour
          else if (x >= 0 && big_bit(seen, x) && !big_bit(leaf, x)) ok = true;  // an extracted one
          if (x < 0 || big_bit(seen, x)) q[kk] = -1;                           // keep the exposures
        }
        const unsigned bad = __ballot_sync(__activemask(), !ok);
        if (bad && lane == __ffs(bad) - 1) atomicMin(cut, tid);
      }
      __syncthreads();
      j = min(*cut, ng);
      if (j < ng && tid == j) S.gblock = key;  // first failing key: an unreached local maximum
      if (j == ng && tid == 0) S.gblock = -1;
      if (j > 0) {
        int mch = -1;
        if (tid < j) {
          cout[cand_p] = asc ? (e + tid) : (k - 1 - (e + tid));
          atomicOr(seen + (key >> 5), 1u << (key & 31));
#pragma unroll
          for (int kk = 0; kk < K; kk++) {
            const int x = q[kk];
            if (x >= 0) {
              atomicOr(seen + (x >> 5), 1u << (x & 31));
              big_front_add(S, x, ks);
              mch = max(mch, x >> 5);
            }
          }
        }
        mch = __reduce_max_sync(0xffffffffu, mch);
        if (lane == 0 && mch >= 0) {
          atomicMax(&S.hw, mch);
          atomicMax(&S.hi_sw, mch >> 5);
          atomicMax(&S.hi_chunk, mch >> (BIG_CHUNK_SHIFT - 5));
        }
        __syncthreads();
        if (tid < j) atomicAnd(leaf + (key >> 5), ~(1u << (key & 31)));
        e += j;
        ngs++;
        ngc += j;
      }
      if (tid == 0) S.cutbuf[par ^ 1] = 0x7fffffff;
      par ^= 1;
      __syncthreads();
      BIG_TICK(17)
      if (j > 0) continue;
    }
    // ---- (f) frontier rule, warp mode ---------------------------------------
    if (S.wmode) {
      if (warp == 0) {
        int ew = e;
        long long wt = dbg ? clock64() : 0, wn;
#define WARP_TICK(i)                         \
  if (dbg) {                                 \
    wn = clock64();                          \
    if (lane == 0) dbg[i] += wn - wt;        \
    wt = wn;                                 \
  }
        for (;;) {
          int wkey;
          const int nc = big_warp_gather(S, wkey);
          WARP_TICK(20)
          if (nc == 0) break;
          int wq[K], cand_p = 0;
          if (lane < nc) {
            cand_p = G.inv[wkey];
            big_row<K>(G, wkey, wq);
          } else {
#pragma unroll
            for (int kk = 0; kk < K; kk++) wq[kk] = -1;
          }
          int nm = -1;
#pragma unroll
          for (int kk = 0; kk < K; kk++) {
            const int x = wq[kk];
            if (x >= 0 && !((((volatile uint32_t *)seen)[x >> 5] >> (x & 31)) & 1u)) nm = max(nm, x);
            else wq[kk] = -1;
          }
          int inc = nm;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc = max(inc, y);
          }
          WARP_TICK(21)
          int ex = __shfl_up_sync(0xffffffffu, inc, 1);
          const unsigned bal = __ballot_sync(0xffffffffu, lane > 0 && lane < nc && ex > wkey);
          const int jw = bal ? __ffs(bal) - 1 : nc;
          int mch = -1;
          if (lane < jw) {
            cout[cand_p] = asc ? (ew + lane) : (k - 1 - (ew + lane));
            atomicAnd(leaf + (wkey >> 5), ~(1u << (wkey & 31)));
#pragma unroll
            for (int kk = 0; kk < K; kk++) {
              const int x = wq[kk];
              if (x >= 0) {
                atomicOr(seen + (x >> 5), 1u << (x & 31));
                big_front_add(S, x, ks);
                mch = max(mch, x >> 5);
              }
            }
          }
          mch = __reduce_max_sync(0xffffffffu, mch);
          if (lane == 0 && mch >= 0) {
            S.hw = max(S.hw, mch);
            S.hi_sw = max(S.hi_sw, mch >> 5);
            S.hi_chunk = max(S.hi_chunk, mch >> (BIG_CHUNK_SHIFT - 5));
          }
          __syncwarp();  // orders the commit's shared / global updates before the next gather
          WARP_TICK(22)
          ew += jw;
          nws++;
          // back to block mode once the flood commits (nearly) a whole warp's
          // candidates, or commits every candidate of a window without a
          // preemption (a smooth phase in a sparse frontier: block steps
          // would commit more keys per step)
          if (ew >= k || jw >= LTS_BIG_WARP_EXIT || (jw == nc && nc >= LTS_BIG_WARP_FREE)) break;
          const int gbw = S.gblock;
          if (gbw >= 0 && ((((volatile uint32_t *)seen)[gbw >> 5] >> (gbw & 31)) & 1u)) break;
        }
#undef WARP_TICK
        if (lane == 0) {
          S.ew = ew;
          S.wmode = 0;
        }
      }
      __syncthreads();
      e = S.ew;
      BIG_TICK(19)
      continue;
    }
    // ---- (f) frontier rule, block mode --------------------------------------
    int *const cutf = &S.cutbuf[par];
    const int nc = big_gather(S, S.hi_chunk, leaf4, key);
    BIG_TICK(8)
    if (nc == 0) break;
    // the top frontier word bounds the warp gather's start (the commit below
    // raises it for higher exposures, after the cut's barriers)
#if LTS_BIG_HW_FROM_BLOCK
    if (tid == 0) S.hw = key >> 5;
#endif
    const bool isc = tid < nc;
    int cand_p = 0;
    if (isc) {
      cand_p = G.inv[key];
      big_row<K>(G, key, q);
    } else {
#pragma unroll
      for (int kk = 0; kk < K; kk++) q[kk] = -1;
    }
    int nm = -1;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      const int x = q[kk];
      if (x >= 0 && !big_bit(seen, x)) nm = max(nm, x);
      else q[kk] = -1;
    }
    BIG_TICK(9)
    // first preemption: exclusive prefix max of the exposures in candidate
    // order against the candidate's own key
    {
      int inc = nm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = max(inc, y);
      }
      if (lane == 31) S.wmax[warp] = inc;
      __syncthreads();
      int pre = -1;
#pragma unroll
      for (int w = 0; w < BIG_NW; w++)
        if (w < warp) pre = max(pre, S.wmax[w]);
      int ex = __shfl_up_sync(0xffffffffu, inc, 1);
      ex = lane == 0 ? pre : max(pre, ex);
      const unsigned bal = __ballot_sync(0xffffffffu, isc && tid > 0 && ex > key);
      if (lane == 0 && bal) atomicMin(cutf, warp * 32 + __ffs(bal) - 1);
      __syncthreads();
    }
    j = min(*cutf, nc);
    BIG_TICK(10)
    // commit the prefix: labels, leave F; its exposures join F (setting a bit
    // twice is harmless, so the updates need no return value)
    int mch = -1;
    if (tid < j) {
      cout[cand_p] = asc ? (e + tid) : (k - 1 - (e + tid));
      atomicAnd(leaf + (key >> 5), ~(1u << (key & 31)));
#pragma unroll
      for (int kk = 0; kk < K; kk++) {
        const int x = q[kk];
        if (x >= 0) {
          atomicOr(seen + (x >> 5), 1u << (x & 31));
          big_front_add(S, x, ks);
          mch = max(mch, x >> 5);
        }
      }
    }
    mch = __reduce_max_sync(0xffffffffu, mch);
    if (lane == 0 && mch >= 0) {
      atomicMax(&S.hw, mch);
      atomicMax(&S.hi_sw, mch >> 5);
      atomicMax(&S.hi_chunk, mch >> (BIG_CHUNK_SHIFT - 5));
    }
    e += j;
    nst++;
    ncand += nc;
    if (dbg && tid == 0) {  // commit-size histogram (lts_debug_big_stats)
      dbg[12] += j <= 8;
      dbg[13] += j <= 32;
      dbg[14] += (j + 31) / 32;
      dbg[15] += j == nc;
    }
    if (tid == 0) {
      S.cutbuf[par ^ 1] = 0x7fffffff;
      if (j < LTS_BIG_WARP_ENTER) S.wmode = 1;  // few keys committed: warp mode
    }
    par ^= 1;
    __syncthreads();
    BIG_TICK(11)
  }
#undef BIG_TICK
  if (dbg && tid == 0) {
    dbg[1] += nst;
    dbg[2] += ncand;
    dbg[3] += e;
    dbg[5] += ngs;
    dbg[6] += ngc;
    dbg[16] += nws;
    dbg[18] += nga;
  }
}

// Region adjacency rows, has_outside flags, identity initial order and v0 for
// every large region, computed by the whole GPU before the flood kernel
// (_kernels.py:453-481).  grid.y = big-region index, grid.x = slot chunks.
template <int NDIM>
__global__ void __launch_bounds__(256) k_big_rows(LocArgs A, BigArgs Bg) {
  constexpr int K = KOf<NDIM>::value;
  const int n = (int)A.g.n;
  const int lane = threadIdx.x & 31;
  // flat over the slots of all big regions; warps stay converged so the
  // per-region minimum is reduced over the lanes of the same region
  for (int b0 = blockIdx.x * blockDim.x; b0 < Bg.bslots; b0 += gridDim.x * blockDim.x) {
    const int i = b0 + threadIdx.x;
    const int qi = i < Bg.bslots ? big_locate(Bg, i) : -1;
    int mine = 0x7fffffff;
    bool ismax = false;
    if (qi >= 0) {
      const int rid = A.order[Bg.qbase + qi];
      const int lo = A.rptr[rid];
      const int p = i - Bg.bpre[qi];
      const int s = A.verts[lo];
      const int srank = eff_rank(A.rank, s, A.rev, n);
      const Nb<NDIM> nb(A.g, A.verts[lo + p]);
      bool out = false, top = p >= 1;
      int *row = Bg.nrow + ((size_t)lo + p) * K;
#pragma unroll
      for (int kk = 0; kk < K; kk++) {
        int u = nb(A.g, kk);
        const int q = member(A, u, lo, A.rptr[rid + 1] - lo, s);
        row[kk] = q;
        if (q > p) top = false;
        if (p >= 1 && u >= 0 && eff_rank(A.rank, u, A.rev, n) < srank) out = true;
      }
      A.sfl[lo + p] = out ? SF_OUT : 0;
      if (out) mine = p;
      ismax = top;
      A.buf0[lo + p] = p;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, qi);
    const int m = __reduce_min_sync(peers, mine);
    const int nm = __popc(__ballot_sync(0xffffffffu, ismax) & peers);
    if (qi >= 0 && lane == __ffs(peers) - 1) {
      if (m != 0x7fffffff) atomicMin(Bg.v0 + qi, m);
      if (nm) atomicAdd(Bg.st + qi * BST_W + BST_NMAX, nm);
    }
  }
}

// exclusive prefix of the big-region sizes in queue order (one block)
__global__ void __launch_bounds__(1024) k_big_prefix(LocArgs A, BigArgs Bg, int *bpre) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < Bg.nbig; b0 += 1024) {
    const int qi = b0 + threadIdx.x;
    int x = 0;
    if (qi < Bg.nbig) {
      const int rid = A.order[Bg.qbase + qi];
      x = A.rptr[rid + 1] - A.rptr[rid];
    }
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int pre = carry;
    for (int w = 0; w < warp; w++) pre += wsum[w];
    if (qi < Bg.nbig) bpre[qi] = pre + inc - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry = pre + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) bpre[Bg.nbig] = carry;
}

// The big-region floods run as an iteration of four launches over all large
// regions at once, so the per-flood work that is not the priority flood
// itself (relabelling the neighbour rows, the constraint checks) is spread
// over the whole GPU instead of one SM per region:
//   k_big_setup   (grid-wide)  key -> local index and neighbour keys of flood t
//   k_big_flood   (CTA/region) the exact batched priority flood t -> t+1
//   k_big_check   (grid-wide)  unauthorized extrema of state t+1, and whether
//                              state t+1 equals state t-1 (period-2 cycle)
//   k_big_decide  (per region) _localize_one's stopping rules
// The host repeats the iteration while a region is still flooding.

__device__ __forceinline__ int *big_buf(const LocArgs &A, int i) {
  const int m = i % 3;
  return m == 0 ? A.buf0 : (m == 1 ? A.buf1 : A.buf2);
}

struct BigRef {
  int rid, lo, k;
};

__device__ __forceinline__ BigRef big_ref(const LocArgs &A, const BigArgs &Bg, int qi) {
  BigRef r;
  r.rid = A.order[Bg.qbase + qi];
  r.lo = A.rptr[r.rid];
  r.k = A.rptr[r.rid + 1] - r.lo;
  return r;
}

// per region: v0 from k_big_rows; no admissible minimum -> status 1
__global__ void k_big_init(LocArgs A, BigArgs Bg, int level_min, int level_ratio, int level_giant, int *nlevel) {
  GRID_STRIDE(qi, Bg.nbig) {
    const BigRef R = big_ref(A, Bg, (int)qi);
    const int v0 = Bg.v0[qi];
    int *st = Bg.st + qi * BST_W;
    st[BST_T] = 0;
    st[BST_BAD] = 0;
    st[BST_DIFF] = 0;
    st[BST_NSRC] = 0;
    // rough regions flood level-parallel (many local maxima per vertex, or many
    // in absolute terms: the CTA flood needs about one step per ascent), and
    // so do the regions whose bit sets would not fit its shared memory
    const int nmax = st[BST_NMAX];
    const int lev = level_min >= 0 && R.k >= level_min &&
                    ((long long)nmax * level_ratio >= R.k || nmax >= LTS_LEVEL_NMAX || R.k >= level_giant) ? 1 : 0;
    st[BST_LEVEL] = lev;
    if (lev) atomicAdd(nlevel, 1);
    if (v0 == 0x7fffffff) {
      st[BST_ACTIVE] = 0;
      st[BST_FIN] = -1;
      st[BST_STATUS] = 1;
    } else {
      st[BST_ACTIVE] = 1;
      st[BST_FIN] = 0;
      st[BST_STATUS] = 0;
      A.buf0[R.lo] = 0x7fffffff;
      A.buf0[R.lo + v0] = (int)0x80000000;
    }
  }
}

// flat over big-region slots: inverse and neighbour keys of the next flood.
// One row per thread, the K label gathers of a row independent of each other.
template <int NDIM>
__global__ void __launch_bounds__(256) k_big_setup(LocArgs A, BigArgs Bg) {
  constexpr int K = KOf<NDIM>::value;
  static_assert(K % 2 == 0, "rows are read and written as int2");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Bg.bslots; i += gridDim.x * blockDim.x) {
    const int qi = big_locate(Bg, i);
    const int *st = Bg.st + qi * BST_W;
    if (!st[BST_ACTIVE]) continue;
    const int t = st[BST_T];
    const bool asc = t & 1;
    const BigRef R = big_ref(A, Bg, qi);
    const int k = R.k;
    const int p = i - Bg.bpre[qi];
    const int *cin = big_buf(A, t) + R.lo;
    const int kp = flood_key(cin[p], asc, k);
    Bg.inv[R.lo + R.rid + kp] = p;
    const int2 *row = reinterpret_cast<const int2 *>(Bg.nrow + ((size_t)R.lo + p) * K);
    int q[K], c[K];
#pragma unroll
    for (int h = 0; h < K / 2; h++) {
      const int2 v = row[h];
      q[2 * h] = v.x;
      q[2 * h + 1] = v.y;
    }
#pragma unroll
    for (int kk = 0; kk < K; kk++) c[kk] = q[kk] >= 0 ? cin[q[kk]] : 0;
    int2 *dst = reinterpret_cast<int2 *>(Bg.nrowkey + ((size_t)R.lo + R.rid + kp) * K);
#pragma unroll
    for (int h = 0; h < K / 2; h++)
      dst[h] = make_int2(q[2 * h] >= 0 ? flood_key(c[2 * h], asc, k) : -1,
                         q[2 * h + 1] >= 0 ? flood_key(c[2 * h + 1], asc, k) : -1);
  }
}

// one CTA per region (grid = regions, largest first): flood t -> t+1
template <int NDIM>
__global__ void __launch_bounds__(BIG_T) k_big_flood(LocArgs A, BigArgs Bg) {
  constexpr int K = KOf<NDIM>::value;
  extern __shared__ __align__(16) unsigned char smraw[];
  BigSmem &S = *reinterpret_cast<BigSmem *>(smraw);
  const int tid = threadIdx.x;
  const int qi = blockIdx.x;
  int *st = Bg.st + qi * BST_W;
  if (!st[BST_ACTIVE] || st[BST_LEVEL]) return;
  const int t = st[BST_T];
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
  // bit sets in shared memory when they fit (the leaf words first: the
  // candidate scan reads them every step), else in the region's spill space
  if (tid == 0) {
    const int nw = (k + 1 + 31) >> 5;
    // spill space: leaf, seen and summary words of every region fit in
    // 3 (k+1)/32 + 16 words per region (gbits holds 6n + 64 words)
    uint32_t *gp = Bg.gbits + ((3 * (((size_t)lo + rid) >> 5) + 16 * (size_t)rid + 3) & ~(size_t)3);
    const int nw4 = (nw + 3) & ~3;  // leaf read as uint4; padding stays zero
    const int nsw4 = (((nw + 31) >> 5) + 3) & ~3;
    S.nsw4 = nsw4;
    S.nw = nw;
    S.nw4 = nw4;
    // shared memory in order of use per step: summary, leaf, seen
    int used = 0;
    S.sum = nsw4 <= BIG_SMEM_WORDS ? S.bits : gp + 2 * nw4;
    if (nsw4 <= BIG_SMEM_WORDS) used = nsw4;
    S.leaf = used + nw4 <= BIG_SMEM_WORDS ? S.bits + used : gp;
    if (used + nw4 <= BIG_SMEM_WORDS) used += nw4;
    S.seen = used + nw4 <= BIG_SMEM_WORDS ? S.bits + used : gp + nw4;
  }
  __syncthreads();
  const int qa = Bg.qbase + qi;  // absolute big-queue position
  long long *dbg = (d_dbg_on && qa < DBG_MAX) ? d_dbg + qa * DBG_W : nullptr;
  if (dbg && tid == 0) dbg[0] = k;
  if (tid == 0) atomicAdd(Bg.work, (unsigned long long)k);
  const long long c0 = clock64();
  // the key no slot maps to: v0's index in the first flood (its slot maps to
  // key 0 and the saddle's to k), k in every later one
  const int unused_key = t == 0 ? Bg.v0[qi] : k;
  big_flood<K>(S, G, t & 1, big_buf(A, t) + lo, big_buf(A, t + 1) + lo, unused_key, dbg);
  if (dbg && tid == 0) dbg[4] += clock64() - c0;
}

// flat over big-region slots: constraint check of state t+1 (desc flood: local
// minima get SF_MIN, unauthorized if not SF_OUT; asc flood: any local maximum
// besides the saddle) and, from t+1 >= 3 on, state t+1 != state t-1
template <int NDIM>
__global__ void __launch_bounds__(256) k_big_check(LocArgs A, BigArgs Bg) {
  constexpr int K = KOf<NDIM>::value;
  const int lane = threadIdx.x & 31;
  for (int b0 = blockIdx.x * blockDim.x; b0 < Bg.bslots; b0 += gridDim.x * blockDim.x) {
    const int i = b0 + threadIdx.x;
    int qi = i < Bg.bslots ? big_locate(Bg, i) : -1;
    int *st = qi >= 0 ? Bg.st + qi * BST_W : nullptr;
    if (st && !st[BST_ACTIVE]) qi = -1;
    bool bad = false, diff = false;
    if (qi >= 0) {
      const int t1 = st[BST_T] + 1;
      const bool desc = (t1 & 1) == 1;  // flood t1-1 was descending
      const BigRef R = big_ref(A, Bg, qi);
      const int p = i - Bg.bpre[qi];
      const int *cur = big_buf(A, t1) + R.lo;
      const int *old = big_buf(A, t1 + 1) + R.lo;  // state t1-2
      const int c = cur[p];
      if (t1 >= 3 && c != old[p]) diff = true;
      if (p >= 1) {
        const int2 *row = reinterpret_cast<const int2 *>(Bg.nrow + ((size_t)R.lo + p) * K);
        int q[K];
#pragma unroll
        for (int h = 0; h < K / 2; h++) {
          const int2 v = row[h];
          q[2 * h] = v.x;
          q[2 * h + 1] = v.y;
        }
        bool ext = true;
#pragma unroll
        for (int kk = 0; kk < K; kk++)
          if (q[kk] >= 0 && (desc ? cur[q[kk]] < c : cur[q[kk]] > c)) ext = false;
        if (desc) {
          uint8_t *sfl = A.sfl + R.lo;
          uint8_t f = sfl[p];
          f = ext ? (f | SF_MIN) : (f & (uint8_t)~SF_MIN);
          sfl[p] = f;
          if (ext && !(f & SF_OUT)) bad = true;
        } else if (ext) {
          bad = true;
        }
      }
    }
    // one atomic per region and warp
    const unsigned peers = __match_any_sync(0xffffffffu, qi);
    const unsigned bb = __ballot_sync(0xffffffffu, bad) & peers;
    const unsigned dd = __ballot_sync(0xffffffffu, diff) & peers;
    if (qi >= 0 && lane == __ffs(peers) - 1) {
      if (bb) atomicOr(st + BST_BAD, 1);
      if (dd) atomicOr(st + BST_DIFF, 1);
    }
  }
}

// per region: the stopping rules of _localize_one (_kernels.py:491-571) with
// the period-2 cycle jump (contract D5); counts the regions still flooding
__global__ void k_big_decide(LocArgs A, BigArgs Bg) {
  GRID_STRIDE(qi, Bg.nbig) {
    int *st = Bg.st + qi * BST_W;
    if (!st[BST_ACTIVE]) continue;
    int t = st[BST_T] + 1;
    const bool bad = st[BST_BAD] != 0, diff = st[BST_DIFF] != 0;
    st[BST_BAD] = 0;
    st[BST_DIFF] = 0;
    st[BST_NSRC] = 0;
    bool done = true;
    if (!bad) {
      st[BST_FIN] = t;
    } else if (t >= A.max_iter) {
      st[BST_STATUS] = 2;
      st[BST_FIN] = t;
    } else if (t >= 3 && !diff) {
      st[BST_STATUS] = 2;
      st[BST_FIN] = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
      t = A.max_iter;
    } else {
      done = false;
    }
    st[BST_T] = t;
    if (done) st[BST_ACTIVE] = 0;
    else atomicAdd(Bg.nactive, 1);
  }
}

// flat over big-region slots: final local order, status and flood count
__global__ void __launch_bounds__(256) k_big_final(LocArgs A, BigArgs Bg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Bg.bslots; i += gridDim.x * blockDim.x) {
    const int qi = big_locate(Bg, i);
    const int *st = Bg.st + qi * BST_W;
    const BigRef R = big_ref(A, Bg, qi);
    const int p = i - Bg.bpre[qi];
    const int fin = st[BST_FIN];
    A.out[R.lo + p] = fin >= 0 ? big_buf(A, fin)[R.lo + p] : p;
    if (p == 0) {
      A.status[R.rid] = st[BST_STATUS];
      A.n_iters[R.rid] = st[BST_T];
      const int qa = Bg.qbase + qi;
      if (d_dbg_on && qa < DBG_MAX) d_dbg[qa * DBG_W + 7] = st[BST_T];
    }
  }
}

}  // namespace lts
