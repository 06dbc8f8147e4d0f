// sort.cuh -- onesweep LSD radix sort (uint32 keys, uint32 payload).
//
// Replaces the order field's np.argsort(kind="stable") (reference
// order.py:86-91) and serves the region assembly / scheduling sorts.
// Design (Adinets & Merrill "Onesweep"): one upfront histogram kernel for all
// digit passes, then one kernel per 8-bit digit that ranks a 4096-key tile with
// warp-level multisplit (__match_any_sync), publishes per-digit tile counts
// through a decoupled look-back status array, and scatters through shared
// memory so global writes are digit-contiguous.  Tiles are claimed from an
// atomic counter so look-back always waits on resident blocks.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "lts_common.cuh"

namespace lts {
namespace rs {

constexpr int RADIX = 256;
#ifndef LTS_OS_T
#define LTS_OS_T 256
#endif
#ifndef LTS_OS_KPT
#define LTS_OS_KPT 16
#endif
constexpr int THREADS = LTS_OS_T;
constexpr int WARPS = THREADS / 32;
constexpr int KPT = LTS_OS_KPT;
constexpr int TILE = THREADS * KPT;  // 4096 keys per tile (256 threads x 16, 4 CTAs per SM)
static_assert(THREADS >= RADIX && WARPS <= 32, "one thread per digit");
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_PRE = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;

// float32 -> order-preserving uint32; -0.0 is canonicalised to +0.0 so that
// ties between the two zeros break by vertex id.
__device__ __forceinline__ uint32_t float_key(uint32_t u) {
  if ((u & 0x7fffffffu) == 0) u = 0;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <bool FLOATKEY>
__global__ void __launch_bounds__(256) k_hist(const uint32_t *__restrict__ keys, int64_t n,
                                              int npasses, uint32_t *hist, int *nonfinite) {
  __shared__ uint32_t sh[4][RADIX];
  for (int i = threadIdx.x; i < 4 * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  bool bad = false;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // the caller's array may start at any 4-byte boundary (a view with a
  // storage offset): the first `head` keys are read one by one, the rest as
  // 16-byte vectors
  const int64_t head = min(n, (int64_t)(((16u - ((uint32_t)(uintptr_t)keys & 15u)) & 15u) >> 2));
  const int64_t n4 = (n - head) / 4;
  const uint4 *k4 = reinterpret_cast<const uint4 *>(keys + head);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < head; i += stride) {
    uint32_t x = keys[i];
    if (FLOATKEY) {
      if ((x & 0x7f800000u) == 0x7f800000u) bad = true;
      x = float_key(x);
    }
    for (int p = 0; p < npasses; p++) atomicAdd(&sh[p][(x >> (8 * p)) & 255], 1u);
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint4 q = __ldg(k4 + i);
    uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; e++) {
      uint32_t x = u[e];
      if (FLOATKEY) {
        if ((x & 0x7f800000u) == 0x7f800000u) bad = true;
        x = float_key(x);
      }
      for (int p = 0; p < npasses; p++) atomicAdd(&sh[p][(x >> (8 * p)) & 255], 1u);
    }
  }
  for (int64_t i = head + n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t x = keys[i];
    if (FLOATKEY) {
      if ((x & 0x7f800000u) == 0x7f800000u) bad = true;
      x = float_key(x);
    }
    for (int p = 0; p < npasses; p++) atomicAdd(&sh[p][(x >> (8 * p)) & 255], 1u);
  }
  if (FLOATKEY && bad) atomicOr(nonfinite, 1);
  __syncthreads();
  for (int i = threadIdx.x; i < npasses * RADIX; i += blockDim.x) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// exclusive scan of each pass's 256 bins (one block of 256 threads per pass)
__global__ void k_hist_scan(uint32_t *hist) {
  __shared__ uint32_t s[RADIX];
  uint32_t *h = hist + blockIdx.x * RADIX;
  s[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int d = 0; d < RADIX; d++) {
      uint32_t c = s[d];
      s[d] = acc;
      acc += c;
    }
  }
  __syncthreads();
  h[threadIdx.x] = s[threadIdx.x];
}

// block-wide exclusive scan over 256 values held one per thread (256 threads)
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t *warp_tot) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  uint32_t off = 0;
  for (int i = 0; i < w; i++) off += warp_tot[i];
  return off + inc - x;
}

__device__ long long d_sort_dbg[8];
__device__ int d_sort_dbg_on;

#ifndef LTS_OS_MATCH
#define LTS_OS_MATCH 0
#endif
#ifndef LTS_OS_MINB
#define LTS_OS_MINB 4
#endif
template <bool FLOATKEY, bool HAS_VALS, bool WRITE_KEYS, bool WRITE_RANK>
__global__ void __launch_bounds__(THREADS, LTS_OS_MINB) k_onesweep(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int32_t *__restrict__ rank_out, int64_t n, int shift,
    const uint32_t *__restrict__ offs, uint32_t *status, uint32_t *tile_ctr) {
  __shared__ uint32_t s_tile;
  __shared__ uint16_t s_wh[WARPS][RADIX];
  __shared__ uint32_t s_excl[RADIX];
  __shared__ uint32_t s_start[RADIX];
  __shared__ uint32_t s_wtot[RADIX / 32];
  __shared__ uint32_t s_hist[RADIX];
  __shared__ uint32_t s_keys[TILE];
  __shared__ uint32_t s_vals[TILE];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long t_prev = clock64();
#define SORT_TICK(i)                                              \
  if (d_sort_dbg_on && tid == 0) {                                \
    long long t_now = clock64();                                  \
    atomicAdd((unsigned long long *)&d_sort_dbg[i], (unsigned long long)(t_now - t_prev)); \
    t_prev = t_now;                                               \
  }
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < WARPS * RADIX / 2; i += THREADS) reinterpret_cast<uint32_t *>(&s_wh[0][0])[i] = 0;
  if (tid < RADIX) s_hist[tid] = 0;
  __syncthreads();
  SORT_TICK(1);
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * TILE;

  uint32_t k[KPT], v[KPT];
  uint32_t r[KPT];
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    int64_t idx = base + warp * 32 * KPT + j * 32 + lane;
    if (idx < n) {
      uint32_t u = kin[idx];
      if (FLOATKEY) u = float_key(u);
      k[j] = u;
      v[j] = HAS_VALS ? vin[idx] : (uint32_t)idx;
    } else {
      k[j] = 0xffffffffu;
      v[j] = 0;
    }
  }
  // tile histogram first (shared atomics) so the aggregate is published
  // before the expensive ranking: successors' look-backs rarely spin
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    int64_t idx = base + warp * 32 * KPT + j * 32 + lane;
    if (idx < n) atomicAdd(&s_hist[(k[j] >> shift) & 255u], 1u);
  }
  __syncthreads();
  SORT_TICK(2);
  volatile uint32_t *st = status;
  if (tid < RADIX) {
    uint32_t c = s_hist[tid];
    if (tile == 0) st[tid] = FLAG_PRE | (offs[tid] + c);
    else st[(int64_t)tile * RADIX + tid] = FLAG_AGG | c;
  }
  // warp-level multisplit: peers with the same 8-bit digit from 8 ballots;
  // stable rank among same-digit keys of this warp (chunks of 32 consecutive
  // keys processed in input order)
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    const uint32_t d = (k[j] >> shift) & 255u;
#if LTS_OS_MATCH
    const unsigned peers = __match_any_sync(0xffffffffu, d);
#else
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
      unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
#endif
    const int leader = __ffs(peers) - 1;
    uint32_t cnt = 0;
    if (lane == leader) {
      cnt = s_wh[warp][d];
      s_wh[warp][d] = (uint16_t)(cnt + __popc(peers));
    }
    cnt = __shfl_sync(0xffffffffu, cnt, leader);
    r[j] = cnt + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  SORT_TICK(3);
  // per digit (threads 0..255): exclusive offsets across warps; decoupled
  // look-back over predecessors, four status words per round trip
  uint32_t sum = 0;
  if (tid < RADIX) {
    const int d = tid;
#pragma unroll
    for (int w = 0; w < WARPS; w++) {
      uint32_t c = s_wh[w][d];
      s_wh[w][d] = (uint16_t)sum;
      sum += c;
    }
    uint32_t excl;
    if (tile == 0) {
      excl = offs[d];
    } else {
      uint32_t acc = 0;
      int64_t t = (int64_t)tile - 1;
      bool done = false;
      while (!done) {
        uint32_t sv[4];
#pragma unroll
        for (int q = 0; q < 4; q++) sv[q] = (t - q >= 0) ? st[(t - q) * RADIX + d] : (FLAG_PRE | 0u);
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (done) break;
          uint32_t f = sv[q] & ~VAL_MASK;
          if (f == 0) break;  // not yet published: re-read from here
          acc += sv[q] & VAL_MASK;
          t--;
          if (f == FLAG_PRE) done = true;
        }
      }
      excl = acc;
      st[(int64_t)tile * RADIX + d] = FLAG_PRE | (acc + sum);
    }
    s_excl[d] = excl;
  }
  // tile-local digit starts: exclusive scan of the 256 digit totals
  {
    uint32_t inc = sum;
    if (tid < RADIX) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_wtot[warp] = inc;
    }
    __syncthreads();
    if (tid < RADIX) {
      uint32_t off = 0;
#pragma unroll
      for (int i = 0; i < RADIX / 32; i++)
        if (i < warp) off += s_wtot[i];
      s_start[tid] = off + inc - sum;
    }
  }
  __syncthreads();
  SORT_TICK(4);
#pragma unroll
  for (int j = 0; j < KPT; j++) {
    uint32_t d = (k[j] >> shift) & 255u;
    uint32_t pos = s_start[d] + s_wh[warp][d] + r[j];
    s_keys[pos] = k[j];
    s_vals[pos] = v[j];
  }
  __syncthreads();
  SORT_TICK(5);
  int64_t rem = n - base;
  int valid = rem < TILE ? (int)rem : TILE;
#pragma unroll 4
  for (int i = tid; i < valid; i += THREADS) {
    uint32_t key = s_keys[i];
    uint32_t d = (key >> shift) & 255u;
    uint32_t gpos = s_excl[d] + (uint32_t)i - s_start[d];
    uint32_t val = s_vals[i];
    if (WRITE_KEYS) kout[gpos] = key;
    vout[gpos] = val;
    if (WRITE_RANK) rank_out[val] = (int32_t)gpos;
  }
  SORT_TICK(6);
#undef SORT_TICK
}

// ---------------------------------------------------------------------------
// rank[id] = position, from the sorted ids (inverse), without a random 4-byte
// scatter over the whole rank array: (1) the inverse is partitioned into RB
// buckets by id high bits (bucket b = ids [b*W, (b+1)*W): exactly W entries,
// so each bucket's region is known), staged through shared memory so every
// tile writes one contiguous run per bucket; (2) the pairs are placed bucket
// after bucket, so the rank window being written (n/RB ids) stays in L2 and
// leaves it as full lines.
// ---------------------------------------------------------------------------
#ifndef LTS_RB_BITS
#define LTS_RB_BITS 6
#endif
constexpr int RB_BITS = LTS_RB_BITS, RB = 1 << RB_BITS;

__global__ void __launch_bounds__(THREADS) k_rank_bucket(const uint32_t *__restrict__ inv, int64_t n, int bshift,
                                                        uint32_t *__restrict__ pos_out,
                                                        uint32_t *__restrict__ id_out, uint32_t *ctr) {
  __shared__ uint32_t s_pos[TILE], s_id[TILE];
  __shared__ uint32_t s_wc[WARPS][RB];
  static_assert(RB <= 64 && WARPS * RB <= 2 * THREADS, "bucket counters");
  __shared__ uint32_t s_start[RB], s_base[RB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * TILE;
    for (int i = tid; i < WARPS * RB; i += THREADS) (&s_wc[0][0])[i] = 0;
    __syncthreads();
    uint32_t id[KPT], r[KPT];
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      const int64_t idx = base + warp * 32 * KPT + j * 32 + lane;
      id[j] = idx < n ? inv[idx] : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      const bool ok = id[j] != 0xffffffffu;
      const uint32_t b = ok ? (id[j] >> bshift) : 0u;
      unsigned peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int t = 0; t < RB_BITS; t++) {
        const unsigned bal = __ballot_sync(0xffffffffu, (b >> t) & 1u);
        peers &= ((b >> t) & 1u) ? bal : ~bal;
      }
      const int leader = __ffs(peers) - 1;
      uint32_t cnt = 0;
      if (ok && lane == leader) {
        cnt = s_wc[warp][b];
        s_wc[warp][b] = cnt + __popc(peers);
      }
      cnt = __shfl_sync(0xffffffffu, cnt, leader < 0 ? 0 : leader);
      r[j] = cnt + __popc(peers & lanemask_lt());
      __syncwarp();
    }
    __syncthreads();
    __shared__ uint32_t s_half;
    uint32_t sum = 0, inc = 0;
    if (tid < RB) {  // per bucket: warp offsets, tile total, global slot run
#pragma unroll
      for (int w = 0; w < WARPS; w++) {
        const uint32_t c = s_wc[w][tid];
        s_wc[w][tid] = sum;
        sum += c;
      }
      s_base[tid] = sum ? atomicAdd(ctr + tid, sum) : 0u;
      inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (tid == 31) s_half = inc;
    }
    __syncthreads();
    if (tid < RB) s_start[tid] = inc - sum + (tid >= 32 ? s_half : 0u);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      if (id[j] == 0xffffffffu) continue;
      const uint32_t b = id[j] >> bshift;
      const uint32_t p = s_start[b] + s_wc[warp][b] + r[j];
      s_id[p] = id[j];
      s_pos[p] = (uint32_t)(base + warp * 32 * KPT + j * 32 + lane);
    }
    __syncthreads();
    const int valid = (int)min((int64_t)TILE, n - base);
    for (int i = tid; i < valid; i += THREADS) {
      const uint32_t v = s_id[i];
      const uint32_t b = v >> bshift;
      const int64_t g = ((int64_t)b << bshift) + s_base[b] + (uint32_t)i - s_start[b];
      id_out[g] = v;
      pos_out[g] = s_pos[i];
    }
    __syncthreads();
  }
}

__global__ void k_rank_place(const uint32_t *__restrict__ pos, const uint32_t *__restrict__ id, int64_t n,
                             int32_t *__restrict__ rank) {
  GRID_STRIDE(i, n) rank[__ldcs(id + i)] = (int32_t)__ldcs(pos + i);
}

struct Bufs {
  uint32_t *k1, *v1, *k2, *v2;  // ping-pong, n each
  uint32_t *status;             // ceil(n/TILE)*256
  uint32_t *hist;               // 4*256
  uint32_t *ctr;                // 4
  int *nonfinite;               // 1
};

inline int64_t status_elems(int64_t n) { return ((n + TILE - 1) / TILE + 1) * RADIX; }

}  // namespace rs

extern int64_t g_launches;

// Stable LSD radix sort of n (key, value) pairs by the low `bits` key bits.
// keys_in: uint32 keys, or float32 bits when floatkey (transformed on the fly).
// vals_in: may be NULL (values = input index).  keys_out may be NULL.
// rank_out (may be NULL): rank_out[value] = sorted position (last pass).
inline int radix_sort(const uint32_t *keys_in, const uint32_t *vals_in, int64_t n, int bits,
                      bool floatkey, uint32_t *keys_out, uint32_t *vals_out, int32_t *rank_out,
                      rs::Bufs &b, cudaStream_t s) {
  using namespace rs;
  if (n <= 0) return 0;
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  if (passes > 4) passes = 4;
  int64_t ntiles = (n + TILE - 1) / TILE;
  // rank via id buckets when the rank array would not stay in L2 (random
  // 4-byte writes then cost a DRAM read-modify-write each)
  static int rb_env = -2;
  if (rb_env == -2) {
    const char *e = getenv("LTS_RANK_BUCKET");
    rb_env = e ? atoi(e) : -1;
  }
  const bool bucket_rank = rank_out != nullptr && vals_out != nullptr && n >= (1 << RB_BITS) &&
                           (rb_env >= 0 ? rb_env == 1 : n * 4 > (int64_t)96 << 20);
  LTS_CUDA(cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * 4 * RADIX, s));
  LTS_CUDA(cudaMemsetAsync(b.ctr, 0, sizeof(uint32_t) * 4, s));
  int hb = grid_blocks(n / 4 + 1, 256, 148 * 4);
  if (floatkey)
    k_hist<true><<<hb, 256, 0, s>>>(keys_in, n, passes, b.hist, b.nonfinite);
  else
    k_hist<false><<<hb, 256, 0, s>>>(keys_in, n, passes, b.hist, b.nonfinite);
  k_hist_scan<<<passes, RADIX, 0, s>>>(b.hist);
  g_launches += 2;
  const uint32_t *ck = keys_in, *cv = vals_in;
  for (int p = 0; p < passes; p++) {
    bool last = p == passes - 1;
    uint32_t *ok = last ? keys_out : (p % 2 == 0 ? b.k1 : b.k2);
    uint32_t *ov = last ? vals_out : (p % 2 == 0 ? b.v1 : b.v2);
    LTS_CUDA(cudaMemsetAsync(b.status, 0, sizeof(uint32_t) * ntiles * RADIX, s));
    const uint32_t *offs = b.hist + p * RADIX;
    int sh = 8 * p;
    dim3 grid((unsigned)ntiles);
    bool fk = floatkey && p == 0;
    bool hv = cv != nullptr;
    bool wk = ok != nullptr;
    bool wr = last && rank_out != nullptr && !bucket_rank;
#define LTS_OS(FK, HV, WK, WR) \
  k_onesweep<FK, HV, WK, WR><<<grid, THREADS, 0, s>>>(ck, cv, ok, ov, rank_out, n, sh, offs, b.status, b.ctr + p)
    if (fk) {
      if (wr) { if (wk) LTS_OS(true, false, true, true); else LTS_OS(true, false, false, true); }
      else LTS_OS(true, false, true, false);
    } else if (hv) {
      if (wr) { if (wk) LTS_OS(false, true, true, true); else LTS_OS(false, true, false, true); }
      else { if (wk) LTS_OS(false, true, true, false); else LTS_OS(false, true, false, false); }
    } else {
      if (wr) { if (wk) LTS_OS(false, false, true, true); else LTS_OS(false, false, false, true); }
      else { if (wk) LTS_OS(false, false, true, false); else LTS_OS(false, false, false, false); }
    }
#undef LTS_OS
    g_launches++;
    ck = ok;
    cv = ov;
  }
  if (bucket_rank) {
    int lg = 0;
    while ((int64_t(1) << lg) < n) lg++;
    const int bshift = lg > RB_BITS ? lg - RB_BITS : 0;
    LTS_CUDA(cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * RB, s));
    const int nb = (int)std::min<int64_t>(ntiles, 148 * 4);
    k_rank_bucket<<<nb, THREADS, 0, s>>>(vals_out, n, bshift, b.k2, b.v2, b.hist);
    k_rank_place<<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(b.k2, b.v2, n, rank_out);
    g_launches += 2;
  }
  return 0;
}

}  // namespace lts
