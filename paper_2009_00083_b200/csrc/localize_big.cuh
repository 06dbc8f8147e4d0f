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
// ~0.5-0.75% as many steps as extractions (measured with the oracle).
//
// Keys are a permutation of a small integer range (the region's local order),
// so F is a bit set over key space kept as a 32-ary bit tree (levels in shared
// memory; the leaf level spills to global memory for very large regions).
// The top-B keys come from a descending walk of the tree; key -> local index
// is an inverse array rebuilt per flood; "seen" is a per-slot epoch stamp.
// Semantics follow _localize_one (_kernels.py:443-575) exactly, including the
// empty-ascending-flood case and the period-2 cycle jump (contract D5).
#pragma once
#include "localize.cuh"

namespace lts {

constexpr int BIG_T = 512;
constexpr int BIG_B = 256;                    // max candidates per step
constexpr int BIG_SMEM_WORDS = 36 * 1024;     // bit-tree words in shared memory
constexpr int BIG_THRESHOLD = 1024;           // regions with k > this use this kernel

struct BigArgs {
  int *inv;          // key -> local index, S + R entries (region base lo + rid)
  uint32_t *gbits;   // spill space for the leaf level
  uint32_t *seenw;   // per slot: epoch of the last flood that saw it
  int qbase, nbig;   // regions order[qbase .. qbase+nbig)
  int *queue;
};

struct BitTree {
  uint32_t *L[6];
  int nw[6];
  int top;
};

__device__ __forceinline__ uint32_t mask_le(int b) { return b >= 31 ? 0xffffffffu : ((2u << b) - 1u); }

// largest set key <= x, or -1
__device__ int bt_prev(const BitTree &T, int x) {
  int l = 0, pos = x;
  for (;;) {
    if (pos < 0) return -1;
    int w = pos >> 5;
    uint32_t m = ((volatile uint32_t *)T.L[l])[w] & mask_le(pos & 31);
    if (m) {
      pos = (w << 5) + 31 - __clz(m);
      break;
    }
    if (l == T.top) {
      pos = (w << 5) - 1;
      continue;
    }
    pos = w - 1;
    l++;
  }
  while (l > 0) {
    l--;
    uint32_t m = ((volatile uint32_t *)T.L[l])[pos];
    pos = (pos << 5) + 31 - __clz(m);
  }
  return pos;
}

__device__ __forceinline__ void bt_insert(const BitTree &T, int key) {
  int idx = key;
  for (int l = 0; l <= T.top; l++) {
    uint32_t old = atomicOr(T.L[l] + (idx >> 5), 1u << (idx & 31));
    if (old != 0) break;  // word was already non-empty: ancestors are set
    idx >>= 5;
  }
}

template <int NDIM>
__device__ __forceinline__ int nbr_member(const LocArgs &A, int v, int kk, int rid, int s) {
  int x, y, z;
  coords(A.g, v, x, y, z);
  return member(A, nbr_at(A.g, x, y, z, kk), rid, s);
}

// smem layout for the big kernel (dynamic)
struct BigSmem {
  int cand_key[BIG_B];
  int cand_p[BIG_B];
  int cand_v[BIG_B];
  int newmax[BIG_B];
  int pair_q[BIG_B * kMaxK];
  int pair_key[BIG_B * kMaxK];
  int ncand, cut, nsrc, red;
  uint32_t bits[BIG_SMEM_WORDS];
};

template <int NDIM>
__device__ void big_flood(const LocArgs &A, const BigArgs &Bg, BigSmem &S, BitTree &T, bool asc,
                          int rid, int s, int lo, int k, const int *verts, const int *cin, int *cout,
                          const uint8_t *sfl, uint32_t epoch, int *inv, int &Beff) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K1 = k + 1;
  uint32_t *seen = Bg.seenw + lo;
  // key of local index p: desc floods map the sentinels +BIG -> k, -BIG -> 0
  auto keyof = [&](int p) -> int {
    int c = cin[p];
    if (asc) return k - 1 - c;
    if (c == 0x7fffffff) return k;
    if (c == (int)0x80000000) return 0;
    return c;
  };
  for (int l = 0; l <= T.top; l++)
    for (int i = tid; i < T.nw[l]; i += BIG_T) T.L[l][i] = 0u;
  if (tid == 0) S.nsrc = 0;
  __syncthreads();
  for (int p = tid; p < k; p += BIG_T) inv[keyof(p)] = p;
  // sources
  if (!asc) {
    if (tid == 0) {
      seen[0] = epoch;
      bt_insert(T, keyof(0));
      S.nsrc = 1;
    }
  } else {
    for (int p = 1 + tid; p < k; p += BIG_T)
      if ((sfl[p] & (SF_MIN | SF_OUT)) == (SF_MIN | SF_OUT)) {
        seen[p] = epoch;
        bt_insert(T, keyof(p));
        atomicAdd(&S.nsrc, 1);
      }
  }
  __syncthreads();
  if (S.nsrc == 0) {  // empty ascending flood keeps the previous labels
    for (int p = tid; p < k; p += BIG_T) cout[p] = cin[p];
    __syncthreads();
    return;
  }
  int e = 0;
  int pos = K1 - 1;  // no key above the current top can re-enter F except via exposure
  for (;;) {
    // (a) candidates: top keys of F in descending order (warp 0)
    if (warp == 0) {
      int nc = 0;
      int x = K1 - 1;
      while (nc < Beff) {
        int key0 = 0;
        if (lane == 0) key0 = bt_prev(T, x);
        key0 = __shfl_sync(0xffffffffu, key0, 0);
        if (key0 < 0) break;
        int w = key0 >> 5;
        uint32_t word = ((volatile uint32_t *)T.L[0])[w] & mask_le(key0 & 31);
        int c = __popc(word);
        int take = min(c, Beff - nc);
        if ((word >> lane) & 1u) {
          int r = __popc(word & ~mask_le(lane));  // set bits above this one
          if (r < take) {
            int key = (w << 5) + lane;
            int p = inv[key];
            S.cand_key[nc + r] = key;
            S.cand_p[nc + r] = p;
            S.cand_v[nc + r] = verts[p];
            S.newmax[nc + r] = -1;
          }
        }
        nc += take;
        x = (w << 5) - 1;
      }
      if (lane == 0) {
        S.ncand = nc;
        S.cut = nc;
      }
    }
    __syncthreads();
    const int nc = S.ncand;
    if (nc == 0) break;
    // (b) exposure maxima of every candidate
    for (int i = tid; i < nc * K; i += BIG_T) {
      int c = i / K, kk = i - c * K;
      int q = nbr_member<NDIM>(A, S.cand_v[c], kk, rid, s);
      int key = -1;
      if (q >= 0 && ((volatile uint32_t *)seen)[q] != epoch) {
        key = keyof(q);
        atomicMax(&S.newmax[c], key);
      } else {
        q = -1;
      }
      S.pair_q[i] = q;
      S.pair_key[i] = key;
    }
    __syncthreads();
    // (c) prefix max and first preemption (warp 0)
    if (warp == 0) {
      int run = -1;
      for (int b0 = 0; b0 < nc; b0 += 32) {
        int i = b0 + lane;
        int v = i < nc ? S.newmax[i] : -1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v = max(v, y);
        }
        v = max(v, run);
        bool pre = (i + 1 < nc) && v > S.cand_key[i + 1];
        unsigned bm = __ballot_sync(0xffffffffu, pre);
        if (bm) {
          if (lane == 0) S.cut = b0 + __ffs(bm);  // commit candidates [0, i] (i+1 of them)
          break;
        }
        run = __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    const int j = S.cut;
    // (d) commit: labels, remove from F
    for (int i = tid; i < j; i += BIG_T) {
      int p = S.cand_p[i];
      cout[p] = asc ? (e + i) : (k - 1 - (e + i));
      int key = S.cand_key[i];
      atomicAnd(T.L[0] + (key >> 5), ~(1u << (key & 31)));
    }
    __syncthreads();
    for (int l = 0; l < T.top; l++) {
      for (int i = tid; i < j; i += BIG_T) {
        int idx = S.cand_key[i] >> (5 * (l + 1));  // word index at level l
        if (((volatile uint32_t *)T.L[l])[idx] == 0u)
          atomicAnd(T.L[l + 1] + (idx >> 5), ~(1u << (idx & 31)));
      }
      __syncthreads();
    }
    // exposures of the committed prefix join F
    for (int i = tid; i < j * K; i += BIG_T) {
      int q = S.pair_q[i];
      if (q >= 0 && atomicMax(seen + q, epoch) != epoch) bt_insert(T, S.pair_key[i]);
    }
    e += j;
    if (j == nc && nc == Beff && Beff < BIG_B) Beff *= 2;
    else if (j * 4 < Beff && Beff > 8) Beff >>= 1;
    __syncthreads();
  }
  (void)pos;
}

template <int NDIM>
__device__ bool big_check_minima(const LocArgs &A, int rid, int s, int k, const int *verts,
                                 const int *cur, uint8_t *sfl, int *red) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  if (threadIdx.x == 0) *red = 0;
  __syncthreads();
  bool bad = false;
  for (int p = 1 + threadIdx.x; p < k; p += BIG_T) {
    int v = verts[p];
    int x, y, z;
    coords(A.g, v, x, y, z);
    int c = cur[p];
    bool mn = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = member(A, nbr_at(A.g, x, y, z, kk), rid, s);
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
  if (bad) atomicOr(red, 1);
  __syncthreads();
  bool r = *red != 0;
  __syncthreads();
  return r;
}

template <int NDIM>
__device__ bool big_check_maxima(const LocArgs &A, int rid, int s, int k, const int *verts,
                                 const int *cur, int *red) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  if (threadIdx.x == 0) *red = 0;
  __syncthreads();
  bool bad = false;
  for (int p = 1 + threadIdx.x; p < k; p += BIG_T) {
    int v = verts[p];
    int x, y, z;
    coords(A.g, v, x, y, z);
    int c = cur[p];
    bool mx = true;
#pragma unroll
    for (int kk = 0; kk < K; kk++) {
      int q = member(A, nbr_at(A.g, x, y, z, kk), rid, s);
      if (q >= 0 && cur[q] > c) {
        mx = false;
        break;
      }
    }
    if (mx) bad = true;
  }
  if (bad) atomicOr(red, 1);
  __syncthreads();
  bool r = *red != 0;
  __syncthreads();
  return r;
}

__device__ bool big_states_equal(const int *a, const int *b, int k, int *red) {
  if (threadIdx.x == 0) *red = 0;
  __syncthreads();
  bool diff = false;
  for (int p = threadIdx.x; p < k; p += BIG_T)
    if (a[p] != b[p]) diff = true;
  if (diff) atomicOr(red, 1);
  __syncthreads();
  bool r = *red == 0;
  __syncthreads();
  return r;
}

template <int NDIM>
__global__ void __launch_bounds__(BIG_T) k_localize_big(LocArgs A, BigArgs Bg) {
  constexpr int K = NDIM == 2 ? 6 : 14;
  extern __shared__ __align__(16) unsigned char smraw[];
  BigSmem &S = *reinterpret_cast<BigSmem *>(smraw);
  __shared__ int s_qi, s_v0;
  const int tid = threadIdx.x;
  const int n = (int)A.g.n;
  for (;;) {
    if (tid == 0) s_qi = atomicAdd(Bg.queue, 1);
    __syncthreads();
    const int qi = s_qi;
    if (qi >= Bg.nbig) break;
    const int rid = A.order[Bg.qbase + qi];
    const int lo = A.rptr[rid];
    const int k = A.rptr[rid + 1] - lo;
    const int *verts = A.verts + lo;
    uint8_t *sfl = A.sfl + lo;
    int *bufs[3] = {A.buf0 + lo, A.buf1 + lo, A.buf2 + lo};
    int *inv = Bg.inv + lo + rid;
    const int s = verts[0];
    const int srank = eff_rank(A.rank, s, A.rev, n);
    // bit tree geometry over key space [0, k]
    BitTree T;
    {
      int words = (k + 1 + 31) >> 5;
      int l = 0;
      T.nw[0] = words;
      while (T.nw[l] > 32) {
        T.nw[l + 1] = (T.nw[l] + 31) >> 5;
        l++;
      }
      T.top = l;
      int upper = 0;
      for (int i = 1; i <= T.top; i++) upper += T.nw[i];
      bool leaf_smem = upper + T.nw[0] <= BIG_SMEM_WORDS;
      uint32_t *sp = S.bits;
      if (leaf_smem) {
        T.L[0] = sp;
        sp += T.nw[0];
      } else {
        T.L[0] = Bg.gbits + ((lo + rid + 31) >> 5) + rid;
      }
      for (int i = 1; i <= T.top; i++) {
        T.L[i] = sp;
        sp += T.nw[i];
      }
    }
    if (tid == 0) s_v0 = 0x7fffffff;
    __syncthreads();
    for (int p = tid; p < k; p += BIG_T) {
      bool out = false;
      if (p >= 1) {
        int x, y, z;
        coords(A.g, verts[p], x, y, z);
#pragma unroll
        for (int kk = 0; kk < K; kk++) {
          int u = nbr_at(A.g, x, y, z, kk);
          if (u >= 0 && eff_rank(A.rank, u, A.rev, n) < srank) {
            out = true;
            break;
          }
        }
      }
      sfl[p] = out ? SF_OUT : 0;
      if (out) atomicMin(&s_v0, p);
      bufs[0][p] = p;
      Bg.seenw[lo + p] = 0u;
    }
    __syncthreads();
    const int v0 = s_v0;
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
      bufs[0][0] = 0x7fffffff;
      bufs[0][v0] = (int)0x80000000;
    }
    __syncthreads();
    int t = 0, status = 0, fin = 0, Beff = 32;
    for (;;) {
      big_flood<NDIM>(A, Bg, S, T, false, rid, s, lo, k, verts, bufs[t % 3], bufs[(t + 1) % 3], sfl,
                      (uint32_t)(t + 1), inv, Beff);
      t++;
      bool bad = big_check_minima<NDIM>(A, rid, s, k, verts, bufs[t % 3], sfl, &S.red);
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && big_states_equal(bufs[t % 3], bufs[(t + 1) % 3], k, &S.red)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
      big_flood<NDIM>(A, Bg, S, T, true, rid, s, lo, k, verts, bufs[t % 3], bufs[(t + 1) % 3], sfl,
                      (uint32_t)(t + 1), inv, Beff);
      t++;
      bad = big_check_maxima<NDIM>(A, rid, s, k, verts, bufs[t % 3], &S.red);
      if (!bad) { fin = t; break; }
      if (t >= A.max_iter) { status = 2; fin = t; break; }
      if (t >= 3 && big_states_equal(bufs[t % 3], bufs[(t + 1) % 3], k, &S.red)) {
        status = 2;
        fin = ((A.max_iter - t) % 2 == 0) ? t : t - 1;
        t = A.max_iter;
        break;
      }
    }
    const int *fb = bufs[fin % 3];
    for (int p = tid; p < k; p += BIG_T) A.out[lo + p] = fb[p];
    if (tid == 0) {
      A.status[rid] = status;
      A.n_iters[rid] = t;
    }
    __syncthreads();
  }
}

}  // namespace lts
