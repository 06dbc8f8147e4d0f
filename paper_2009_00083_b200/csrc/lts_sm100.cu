// lts_sm100.cu -- C ABI and device-resident orchestration of the LTS hot path
// on B200 (sm_100a).  Unity build: every kernel header is included here so the
// stencil tables live in one __constant__ bank.
//
// Pipeline:
//   order field (onesweep radix sort)          reference order.py:86-91
//   classification stencil                     critical.py:95-112
//   repeat {maxima pass, minima pass,          _kernels.py:194-303, 578-591,
//           restore, verify}
//   realization by saddle-value gathers        contract D1
// Host code only sequences launches on the caller's stream and reads back a
// handful of scalars (counts) per pass; all arrays stay in HBM.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lts_common.cuh"
#include "prims.cuh"
#include "sort.cuh"
#include "classify.cuh"
#include "classify_zreg.cuh"
#include "classify_2d.cuh"
#include "discover.cuh"
#include "localize.cuh"
#include "localize_big.cuh"
#include "localize_level.cuh"
#include "integrate.cuh"
#include "persistence.cuh"
#include "csr.cuh"

namespace lts {
int64_t g_launches = 0;
}
#ifndef LTS_PEEL_ROUNDS
#define LTS_PEEL_ROUNDS 16  // leaf-peeling rounds of the persistence forest before the sweep
#endif
#ifndef LTS_JUMPS
#define LTS_JUMPS 3  // pointer-jumping launches on the ascent forest before path halving
#endif
#ifndef LTS_BV_COOP_PER_SM
#define LTS_BV_COOP_PER_SM 1
#endif

using namespace lts;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

int lts_set_error(int code, const char *msg) {
  g_err = msg;
  return code;
}

int lts_set_cuda_error(cudaError_t e, const char *what, const char *file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, what);
  g_err = buf;
  return LTS_E_CUDA;
}

#define LTS_TRY(x)          \
  do {                      \
    int rc_ = (x);          \
    if (rc_ != 0) return rc_; \
  } while (0)
#define LTS_KCHECK() LTS_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// stencil tables: offsets (triangulation.py:32-45) and the reference link-pair
// table restated from _face_triple (triangulation.py:52-75), folded
// into per-mask component-count LUTs.
// ---------------------------------------------------------------------------
static const int8_t H_OFF2[6][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {-1, 0, 0}, {0, -1, 0}, {-1, -1, 0}};
static const int8_t H_OFF3[14][3] = {{1, 0, 0},  {0, 1, 0},   {0, 0, 1},   {1, 1, 0},  {1, 0, 1},
                                     {0, 1, 1},  {1, 1, 1},   {-1, 0, 0},  {0, -1, 0}, {0, 0, -1},
                                     {-1, -1, 0}, {-1, 0, -1}, {0, -1, -1}, {-1, -1, -1}};

__device__ uint8_t d_lut2[1 << 6];
__device__ uint8_t d_lut3[1 << 14];

static bool is01(const int *d, int nd) {
  for (int a = 0; a < nd; a++)
    if (d[a] != 0 && d[a] != 1) return false;
  return true;
}

static bool face_triple(const int8_t *a, const int8_t *b, int nd) {
  int z[3] = {0, 0, 0}, A[3], B[3];
  for (int i = 0; i < 3; i++) {
    A[i] = a[i];
    B[i] = b[i];
  }
  const int *seq[6][3] = {{z, A, B}, {z, B, A}, {A, z, B}, {B, z, A}, {A, B, z}, {B, A, z}};
  for (auto &s : seq) {
    int d1[3], d2[3];
    for (int i = 0; i < nd; i++) {
      d1[i] = s[1][i] - s[0][i];
      d2[i] = s[2][i] - s[1][i];
    }
    if (is01(d1, nd) && is01(d2, nd)) return true;
  }
  return false;
}

static void build_lut(int ndim, std::vector<uint8_t> &lut) {
  int K = ndim == 2 ? 6 : 14;
  const int8_t(*off)[3] = ndim == 2 ? H_OFF2 : H_OFF3;
  std::vector<std::pair<int, int>> pairs;
  for (int i = 0; i < K; i++)
    for (int j = i + 1; j < K; j++)
      if (face_triple(off[i], off[j], ndim)) pairs.emplace_back(i, j);
  lut.assign(1u << K, 0);
  for (unsigned m = 0; m < (1u << K); m++) {
    int p[14];
    for (int i = 0; i < K; i++) p[i] = i;
    auto find = [&](int x) {
      while (p[x] != x) x = p[x] = p[p[x]];
      return x;
    };
    for (auto &e : pairs)
      if ((m >> e.first & 1) && (m >> e.second & 1)) {
        int a = find(e.first), b = find(e.second);
        if (a != b) p[b] = a;
      }
    int c = 0;
    for (int i = 0; i < K; i++)
      if ((m >> i & 1) && find(i) == i) c++;
    lut[m] = (uint8_t)c;
  }
}

// ---------------------------------------------------------------------------
// Per-device state.  __constant__ / __device__ symbols, streams, events and
// function attributes belong to one device, so everything the library caches
// is kept per device (indexed by cudaGetDevice), and every C ABI entry point
// holds g_mu for its duration (one call at a time per process; the calls are
// synchronous on their stream anyway).
// ---------------------------------------------------------------------------
constexpr int LTS_MAX_DEV = 64;
struct DevState {
  bool tables_ready = false;
  int off_ndim = 0;
  int *h_scal = nullptr;  // pinned scalar readback slots
  std::vector<cudaEvent_t> events;
  size_t ev_next = 0;
  cudaStream_t side = nullptr, side2 = nullptr, copys = nullptr;
  cudaEvent_t g_ready = nullptr, g_copied = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, lfork = nullptr, ljoin = nullptr;
  bool big_attr = false;
  int coop_blocks = 0, coop_per = 0;  // SMs and resident CTAs per SM of k_bv_coop
  int coop_ok = -1;  // cudaDevAttrCooperativeLaunch
  int lv_blocks[4] = {0, 0, 0, 0}, lv_per[4] = {0, 0, 0, 0};  // cooperative grid of the level floods, per ndim
};
static DevState g_dev[LTS_MAX_DEV];
static DevState *g_cur = &g_dev[0];
static std::recursive_mutex g_mu;
#define LTS_LOCK std::lock_guard<std::recursive_mutex> lts_lock_(g_mu)

static int select_device() {
  int d = 0;
  LTS_CUDA(cudaGetDevice(&d));
  if (d < 0 || d >= LTS_MAX_DEV) return lts_set_error(LTS_E_INVALID, "device index out of range");
  g_cur = &g_dev[d];
  return 0;
}

static int init_tables() {
  if (g_cur->tables_ready) return 0;
  std::vector<uint8_t> l2, l3;
  build_lut(2, l2);
  build_lut(3, l3);
  LTS_CUDA(cudaMemcpyToSymbol(d_lut2, l2.data(), l2.size()));
  LTS_CUDA(cudaMemcpyToSymbol(d_lut3, l3.data(), l3.size()));
  g_cur->tables_ready = true;
  return 0;
}

static int set_offsets(int ndim, cudaStream_t s) {
  if (g_cur->off_ndim == ndim) return 0;
  int8_t off[3][kMaxK] = {};
  int K = ndim == 2 ? 6 : 14;
  for (int k = 0; k < K; k++)
    for (int a = 0; a < 3; a++) off[a][k] = ndim == 2 ? H_OFF2[k][a] : H_OFF3[k][a];
  LTS_CUDA(cudaMemcpyToSymbolAsync(c_off, off, sizeof(off), 0, cudaMemcpyHostToDevice, s));
  LTS_CUDA(cudaStreamSynchronize(s));
  g_cur->off_ndim = ndim;
  return 0;
}

static const uint8_t *lut_ptr(int ndim) {
  void *p = nullptr;
  cudaError_t e = ndim == 2 ? cudaGetSymbolAddress(&p, d_lut2) : cudaGetSymbolAddress(&p, d_lut3);
  if (e != cudaSuccess) return nullptr;
  return (const uint8_t *)p;
}

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
struct WS {
  // n-sized int32
  int *rankA, *invA, *rankB, *invB, *ptr, *M, *rt, *acc, *comp, *par, *wc, *rpar, *ridx, *reg_of, *loc_of,
      *delta, *D, *flagscan, *mlist;
  uint32_t *ckey, *cval, *skey, *sval;
  // region-sized (n+1) int32
  int *rsize, *rtop, *rsad, *order, *nit, *st, *rtmp, *rptr, *sib_rid, *pos_of, *lost, *okey;
  uint32_t *oval, *okey2;
  int64_t *rptr64;
  unsigned long long *best, *bestP;
  uint8_t *flags, *pmark, *vcls, *cst;
  int *ea, *eb, *ew;
  int64_t emax;
  char *ebuf;  // 12 * emax bytes: list-mode ea/eb/ew, or hash table + unique list
  // slots (2n)
  int *verts, *buf0, *buf1, *buf2, *out;
  unsigned long long *gheap;
  uint8_t *sfl;
  int *binv, *nrow, *nrowkey, *bigv0, *bst, *bpre;
  uint32_t *cbits;
  uint32_t *gbits;
  rs::Bufs sb;
  int *bsum;
  // level-parallel floods (localize_level.cuh): key-space arrays and their own sort / scan scratch
  LvArgs lv;
  rs::Bufs lsb;
  int *lbsum;
  int *scal;  // 64 device scalars
  int *pstats;  // 4 per reported pass: N_I max, capped, status-1 regions, largest
  size_t bytes;
};

enum {
  SC_COUNTS = 0,   // 2: all maxima, discarded maxima (one 64-bit counter)
  SC_ECOUNT = 4,
  SC_ACTIVE = 5,
  SC_ERR = 6,
  SC_NREG = 7,
  SC_S = 8,
  SC_C = 9,
  SC_NSHARED = 10,
  SC_QUEUE = 11,
  SC_STATS = 12,   // 4: nit max, capped, status1, largest
  SC_VERIFY = 16,  // 4
  SC_LOST = 20,
  SC_BADPRES = 21,
  SC_RESTORE = 24, // 3
  SC_TMP = 28,
  SC_NBIG = 29,
  SC_BIGQ = 30,
  SC_LARGEST = 31,
  SC_BIGACT = 32,
  SC_BIGWORK = 34,  // 2 ints: 64-bit sum of region sizes flooded by k_big_flood
  SC_BIGSLOTS = 36, // = SC_NBIG + 7: slots of the big regions
  SC_BVSTATE = 40,  // 2: active roots of the last Boruvka round, rounds run
  SC_LV = 44,       // LVC_N (16) counters of the level-parallel floods
  SC_LVTMP = 60,
  SC_N = 64
};

static int64_t carve(WS *w, char *base, int ndim, int64_t n) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char * {
    off = (off + 255) & ~(size_t)255;
    char *p = base ? base + off : nullptr;
    off += bytes;
    return p;
  };
  auto i32 = [&](int64_t cnt) { return (int *)take(sizeof(int) * (size_t)cnt); };
  auto u32 = [&](int64_t cnt) { return (uint32_t *)take(sizeof(uint32_t) * (size_t)cnt); };
  int64_t n1 = n + 1, s2 = 2 * n + 2;
  // maxima-graph edge capacity per vertex (explicit meshes: one per mesh edge end)
  int KH = ndim == 2 ? 3 : (ndim == 3 ? 7 : kCsrK);
  w->rankA = i32(n); w->invA = i32(n); w->rankB = i32(n); w->invB = i32(n);
  w->ptr = i32(n); w->M = i32(n); w->rt = i32(n); w->acc = i32(n); w->comp = i32(n); w->par = i32(n); w->wc = i32(n);
  w->rpar = i32(n); w->ridx = i32(n); w->reg_of = i32(n); w->loc_of = i32(n);
  w->delta = i32(n); w->D = i32(n); w->flagscan = i32(n); w->mlist = i32(n);
  w->ckey = u32(n); w->cval = u32(n); w->skey = u32(n); w->sval = u32(n);
  w->rsize = i32(n1); w->rtop = i32(n1); w->rsad = i32(n1); w->order = i32(n1); w->nit = i32(n1);
  w->st = i32(n1); w->rtmp = i32(n1); w->rptr = i32(n1); w->sib_rid = i32(n1); w->pos_of = i32(n1);
  w->lost = i32(n1); w->okey = i32(n1); w->oval = u32(n1); w->okey2 = u32(n1);
  w->rptr64 = (int64_t *)take(sizeof(int64_t) * (size_t)n1);
  w->best = (unsigned long long *)take(sizeof(unsigned long long) * (size_t)n);
  w->bestP = (unsigned long long *)take(sizeof(unsigned long long) * (size_t)n);
  w->flags = (uint8_t *)take((size_t)n); w->pmark = (uint8_t *)take((size_t)n);
  w->vcls = (uint8_t *)take((size_t)n); w->cst = (uint8_t *)take((size_t)n);
  w->emax = (int64_t)KH * n;
  w->ebuf = take(12 * (size_t)w->emax);
  w->ea = (int *)w->ebuf; w->eb = w->ea + w->emax; w->ew = w->eb + w->emax;
  w->verts = i32(s2); w->buf0 = i32(s2); w->buf1 = i32(s2); w->buf2 = i32(s2); w->out = i32(s2);
  w->gheap = (unsigned long long *)take(sizeof(unsigned long long) * (size_t)s2);
  w->sfl = (uint8_t *)take((size_t)s2);
  w->binv = i32(3 * n + 8);
  w->bigv0 = i32(n1);
  w->bst = i32(BST_W * (n1 / BIG_THRESHOLD + 2));  // regions with k > BIG_THRESHOLD
  w->bpre = i32(n1 / BIG_THRESHOLD + 4);
  w->cbits = u32(n / 32 + 64);
  w->gbits = u32(6 * n + 64);
  const int KR = ndim == 2 ? 6 : (ndim == 3 ? 14 : kCsrK);  // neighbour slots per region slot
  w->nrow = i32(KR * s2);
  w->nrowkey = i32(KR * s2);
  w->sb.k1 = u32(n); w->sb.v1 = u32(n); w->sb.k2 = u32(n); w->sb.v2 = u32(n);
  w->sb.status = u32(rs::status_elems(n));
  w->sb.hist = u32(4 * 256);
  w->sb.ctr = u32(8);
  w->sb.nonfinite = i32(4);
  w->bsum = i32(n / SCAN_TILE + 2);
  {
    // key space of the large regions: one entry per slot plus one per region.
    // The maxima-graph edge buffer is idle between discover and the next pass:
    // the level arrays live in it as far as they fit.
    const int64_t nj = s2 + n1 / BIG_THRESHOLD + 8;
    size_t eoff = 0;
    const size_t ecap = 12 * (size_t)w->emax;
    auto etake = [&](size_t bytes) -> char * {
      const size_t at = (eoff + 255) & ~(size_t)255;
      if (at + bytes > ecap) return take(bytes);
      eoff = at + bytes;
      return base ? w->ebuf + at : nullptr;
    };
    auto ei32 = [&](int64_t cnt) { return (int *)etake(sizeof(int) * (size_t)cnt); };
    w->lv.best = (unsigned long long *)etake(sizeof(unsigned long long) * (size_t)nj);
    w->lv.pm = (unsigned long long *)etake(sizeof(unsigned long long) * (size_t)nj);
    w->lv.task = ei32(nj); w->lv.fp = (unsigned *)ei32(nj); w->lv.par = ei32(nj); w->lv.comp = ei32(nj);
    w->lv.link = ei32(nj); w->lv.csize = ei32(nj); w->lv.lvl = ei32(nj); w->lv.skey = ei32(nj);
    w->lv.sval = ei32(nj); w->lv.oval = ei32(nj);
    // the final sort runs after the levels: its ping-pong buffers reuse the Boruvka arrays
    w->lsb.k1 = (uint32_t *)w->lv.comp; w->lsb.v1 = (uint32_t *)w->lv.link;
    w->lsb.k2 = (uint32_t *)w->lv.best; w->lsb.v2 = w->lsb.k2 ? w->lsb.k2 + nj : nullptr;
    w->lsb.status = u32(rs::status_elems(nj));
    w->lsb.hist = u32(4 * 256);
    w->lsb.ctr = u32(8);
    w->lsb.nonfinite = i32(4);
    w->lbsum = i32(nj / SCAN_TILE + 2);
  }
  w->scal = i32(SC_N);
  w->pstats = i32(4 * LTS_MAX_REPORT_PASSES + 4);
  w->bytes = off + 256;
  return (int64_t)w->bytes;
}

// ---------------------------------------------------------------------------
// context, scalar readback, timing
// ---------------------------------------------------------------------------
struct Ctx {
  Grid g;
  int64_t n;
  WS w;
  cudaStream_t s;
  const uint8_t *lut;
  int *h_scal;  // pinned
  bool timing;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  int64_t flood_launches = 0, flood_slots = 0;
  // host-buffer call (lts_simplify_host): g goes to the host as soon as a minima pass has
  // realised it, beside that pass's floods; G at the end
  float *g_host = nullptr;
  int32_t *G_host = nullptr;
  bool g_copy_valid = false, g_copy_pending = false;
  const int *lptr = nullptr, *la = nullptr, *lb = nullptr;  // explicit mesh: link edges (counts only)
};

// classification of the pass's order: stencil kernels on grids, the CSR
// kernel on explicit meshes
static void classify_any(Ctx &c, const int32_t *rank, uint8_t *flags, int16_t *lower, int16_t *upper,
                         const uint8_t *lut, int32_t *ptr, int ptr_kind, cudaStream_t s) {
  if (c.g.ndim == 0) launch_classify_csr(c.g, rank, flags, lower, upper, c.lptr, c.la, c.lb, ptr, ptr_kind, s);
  else launch_classify(c.g, rank, flags, lower, upper, lut, ptr, ptr_kind, s);
}

static cudaEvent_t next_event() {
  DevState &d = *g_cur;
  if (d.ev_next >= d.events.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    d.events.push_back(e);
  }
  return d.events[d.ev_next++];
}

struct Phase {
  Ctx &c;
  int id;
  cudaEvent_t a;
  Phase(Ctx &c_, int id_) : c(c_), id(id_), a(nullptr) {
    if (c.timing) {
      a = next_event();
      cudaEventRecord(a, c.s);
    }
  }
  ~Phase() {
    if (c.timing) {
      cudaEvent_t b = next_event();
      cudaEventRecord(b, c.s);
      c.marks.push_back({id, {a, b}});
    }
  }
};

static int readback(Ctx &c, int first, int count) {
  LTS_CUDA(cudaMemcpyAsync(c.h_scal + first, c.w.scal + first, sizeof(int) * count,
                           cudaMemcpyDeviceToHost, c.s));
  LTS_CUDA(cudaStreamSynchronize(c.s));
  return 0;
}

static int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 32 && ((int64_t)1 << b) <= maxval) b++;
  return b;
}

static int setup_common(Ctx &c, void *ws, size_t ws_bytes, void *stream) {
  c.s = (cudaStream_t)stream;
  LTS_TRY(select_device());
  int64_t need = carve(&c.w, nullptr, c.g.ndim, c.n);
  if (ws != nullptr) {
    if ((size_t)need > ws_bytes) return lts_set_error(LTS_E_WORKSPACE, "workspace too small");
    carve(&c.w, (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255), c.g.ndim, c.n);
  }
  LTS_TRY(init_tables());
  if (!g_cur->h_scal) LTS_CUDA(cudaHostAlloc((void **)&g_cur->h_scal, sizeof(int) * SC_N, cudaHostAllocDefault));
  c.h_scal = g_cur->h_scal;
  c.timing = false;
  g_cur->ev_next = 0;
  return 0;
}

// An explicit triangle mesh: n vertices, symmetric CSR
// adjacency (device int32 indptr[n+1], indices[nnz]), every degree <= kCsrK.
static int setup_csr(Ctx &c, int64_t n, const int32_t *indptr, const int32_t *indices, void *ws, size_t ws_bytes,
                     void *stream) {
  if (n < 1 || n > ((int64_t)1 << 30)) return lts_set_error(LTS_E_BAD_DIMS, "mesh needs 1 <= n <= 2^30 vertices");
  if (!indptr || !indices) return lts_set_error(LTS_E_INVALID, "indptr and indices are required");
  c.g.nx = (int)n;
  c.g.ny = 1;
  c.g.nz = 1;
  c.g.ndim = 0;
  c.g.K = kCsrK;
  c.g.n = n;
  c.g.cptr = indptr;
  c.g.cidx = indices;
  c.n = n;
  LTS_TRY(setup_common(c, ws, ws_bytes, stream));
  c.lut = nullptr;
  if (ws) {  // the device rows hold kCsrK neighbours per vertex
    LTS_CUDA(cudaMemsetAsync(c.w.scal + SC_TMP, 0, sizeof(int), c.s));
    k_max_degree<<<grid_blocks(n, 256), 256, 0, c.s>>>(indptr, n, c.w.scal + SC_TMP);
    g_launches++;
    LTS_TRY(readback(c, SC_TMP, 1));
    if (c.h_scal[SC_TMP] > kCsrK) return lts_set_error(LTS_E_BAD_DIMS, "a vertex has more than LTS_CSR_K (16) neighbours");
  }
  return 0;
}

static int setup(Ctx &c, int ndim, const int64_t *dims, void *ws, size_t ws_bytes, void *stream) {
  c.g.cptr = c.g.cidx = nullptr;
  if (ndim == 1) {  // a plain vertex list (order field of an explicit mesh)
    if (dims[0] < 1 || dims[0] > ((int64_t)1 << 30)) return lts_set_error(LTS_E_BAD_DIMS, "need 1 <= n <= 2^30 vertices");
    c.g.nx = (int)dims[0];
    c.g.ny = c.g.nz = 1;
    c.g.ndim = 1;
    c.g.K = 0;
    c.g.n = c.n = dims[0];
    return setup_common(c, ws, ws_bytes, stream);
  }
  if (ndim != 2 && ndim != 3) return lts_set_error(LTS_E_BAD_DIMS, "grid must be 2D or 3D");
  int64_t n = 1;
  for (int a = 0; a < ndim; a++) {
    if (dims[a] < 2) return lts_set_error(LTS_E_BAD_DIMS, "every grid axis needs at least 2 vertices");
    n *= dims[a];
  }
  // ranks are packed as (rank << 4 | stencil index) in 32-bit words by the
  // classification kernel: n <= 2^27 (512^3) keeps that exact
  if (n > (int64_t)1 << 27) return lts_set_error(LTS_E_BAD_DIMS, "grid too large (n > 2^27)");
  c.g.nx = (int)dims[0];
  c.g.ny = (int)dims[1];
  c.g.nz = ndim == 3 ? (int)dims[2] : 1;
  c.g.ndim = ndim;
  c.g.K = ndim == 2 ? 6 : 14;
  c.g.n = n;
  c.n = n;
  c.s = (cudaStream_t)stream;
  LTS_TRY(select_device());
  int64_t need = carve(&c.w, nullptr, ndim, n);
  if (ws != nullptr) {
    if ((size_t)need > ws_bytes) return lts_set_error(LTS_E_WORKSPACE, "workspace too small");
    carve(&c.w, (char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255), ndim, n);
  }
  LTS_TRY(init_tables());
  LTS_TRY(set_offsets(ndim, c.s));
  c.lut = lut_ptr(ndim);
  if (!c.lut) return lts_set_error(LTS_E_CUDA, "cudaGetSymbolAddress failed for the link LUT");
  if (!g_cur->h_scal) LTS_CUDA(cudaHostAlloc((void **)&g_cur->h_scal, sizeof(int) * SC_N, cudaHostAllocDefault));
  c.h_scal = g_cur->h_scal;
  c.timing = false;
  g_cur->ev_next = 0;
  return 0;
}

#define NB(nn) grid_blocks((nn), 256)

// ---------------------------------------------------------------------------
// one removal pass (maxima pass, or minima pass on the reversed order)
// ---------------------------------------------------------------------------
__global__ void k_loc_stats(const int *nit, const int *st, const int *rsize, int R, int *out) {
  GRID_STRIDE(r, R) {
    atomicMax(out + 0, nit[r]);
    if (st[r] == 2) atomicAdd(out + 1, 1);
    if (st[r] == 1) atomicAdd(out + 2, 1);
    atomicMax(out + 3, rsize[r] + 1);
  }
}

// out[0] = regions with k > th, out[2] = largest k (saddle included)
// out[0] = #regions with k > th, out[2] = largest k
// out[7] = slots of the regions with k > th
__global__ void k_count_big(const int *rsize, int R, int th, int *out) {
  GRID_STRIDE(r, R) {
    if (rsize[r] + 1 > th) {
      atomicAdd(out, 1);
      atomicAdd(out + 7, rsize[r] + 1);
    }
    atomicMax(out + 2, rsize[r] + 1);
  }
}

static cudaStream_t g_bigs = nullptr;  // stream of the current call's large-region floods
static cudaStream_t g_lvs = nullptr;   // stream of their level-parallel part (beside the CTA floods)

static int big_stream_fork(cudaStream_t s) {
  DevState &d = *g_cur;
  if (!d.side) {
    LTS_CUDA(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking));
    LTS_CUDA(cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming));
    LTS_CUDA(cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming));
    LTS_CUDA(cudaStreamCreateWithFlags(&d.side2, cudaStreamNonBlocking));
    LTS_CUDA(cudaEventCreateWithFlags(&d.lfork, cudaEventDisableTiming));
    LTS_CUDA(cudaEventCreateWithFlags(&d.ljoin, cudaEventDisableTiming));
  }
  if (!d.big_attr) {
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmem)));
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmem)));
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmem)));
    // leave the rest of the unified L1/shared array to L1: the floods re-read
    // region rows and keys that fit there
    int carve = (int)((sizeof(BigSmem) * 100 + 227 * 1024 - 1) / (228 * 1024)) + 1;
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<2>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<3>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    LTS_CUDA(cudaFuncSetAttribute(k_big_flood<0>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    d.big_attr = true;
  }
  // LTS_BIG_SERIAL (diagnostic): run the large-region floods on the main
  // stream, alone on the GPU
  static const bool serial = getenv("LTS_BIG_SERIAL") != nullptr;
  g_bigs = serial ? s : d.side;
  g_lvs = serial ? s : d.side2;
  if (serial) return 0;
  LTS_CUDA(cudaEventRecord(d.fork, s));
  LTS_CUDA(cudaStreamWaitEvent(g_bigs, d.fork, 0));
  return 0;
}

static int big_stream_join(cudaStream_t s) {
  if (g_bigs == s) return 0;
  LTS_CUDA(cudaEventRecord(g_cur->join, g_bigs));
  LTS_CUDA(cudaStreamWaitEvent(s, g_cur->join, 0));
  return 0;
}

// one flood of every large region still flooding: grid-wide relabelling,
// one CTA per region for the flood, grid-wide checks, per-region decision
static int big_level_flood(Ctx &c, const LocArgs &A, const BigArgs &B);
// Flood policy: a large region floods level-parallel (localize_level.cuh) when it
// is rough, i.e. has at least k / ratio local maxima in its initial order (or
// LTS_LEVEL_NMAX of them), or when it has at least `giant` slots.  Small smooth
// regions keep the batched CTA flood, which commits long monotone runs per
// step; the two paths run side by side on two streams, so the few largest
// smooth regions go level-parallel and the many mid-sized ones to the CTAs
// (16 K measured best on cfg3: 11.5 -> 10.7 ms per pass).
// LTS_LEVEL_MIN=-1 disables the level path; LTS_LEVEL_RATIO / LTS_LEVEL_GIANT
// move the thresholds.
static int g_level_min = 0, g_level_ratio = 32, g_level_giant = 16384;
static int g_nlevel = 0;  // level-flooded regions of the current pass

static int big_iteration(Ctx &c, const LocArgs &A, const BigArgs &B, int gx) {
  const int rg = gx;
  LTS_CUDA(cudaMemsetAsync(B.nactive, 0, sizeof(int), g_bigs));
  if (c.g.ndim == 2) k_big_setup<2><<<rg, 256, 0, g_bigs>>>(A, B);
  else if (c.g.ndim == 3) k_big_setup<3><<<rg, 256, 0, g_bigs>>>(A, B);
  else k_big_setup<0><<<rg, 256, 0, g_bigs>>>(A, B);
  // device time of the flood kernel itself (report slot LTS_PH_FLOOD_KERNEL)
  cudaEvent_t fa = nullptr, fb = nullptr;
  if (c.timing) {
    fa = next_event();
    LTS_CUDA(cudaEventRecord(fa, g_bigs));
  }
  const bool lev = g_nlevel > 0;
  if (lev && g_lvs != g_bigs) {  // the level-parallel floods run beside the CTA floods
    LTS_CUDA(cudaEventRecord(g_cur->lfork, g_bigs));
    LTS_CUDA(cudaStreamWaitEvent(g_lvs, g_cur->lfork, 0));
  }
  if (g_nlevel < B.nbig) {
    if (c.g.ndim == 2) k_big_flood<2><<<B.nbig, BIG_T, sizeof(BigSmem), g_bigs>>>(A, B);
    else if (c.g.ndim == 3) k_big_flood<3><<<B.nbig, BIG_T, sizeof(BigSmem), g_bigs>>>(A, B);
    else k_big_flood<0><<<B.nbig, BIG_T, sizeof(BigSmem), g_bigs>>>(A, B);
  }
  if (lev) {
    LTS_TRY(big_level_flood(c, A, B));
    if (g_lvs != g_bigs) {
      LTS_CUDA(cudaEventRecord(g_cur->ljoin, g_lvs));
      LTS_CUDA(cudaStreamWaitEvent(g_bigs, g_cur->ljoin, 0));
    }
  }
  if (c.timing) {
    fb = next_event();
    LTS_CUDA(cudaEventRecord(fb, g_bigs));
    c.marks.push_back({LTS_PH_FLOOD_KERNEL, {fa, fb}});
    c.flood_launches++;
  }
  if (c.g.ndim == 2) k_big_check<2><<<rg, 256, 0, g_bigs>>>(A, B);
  else if (c.g.ndim == 3) k_big_check<3><<<rg, 256, 0, g_bigs>>>(A, B);
  else k_big_check<0><<<rg, 256, 0, g_bigs>>>(A, B);
  k_big_decide<<<NB(B.nbig), 256, 0, g_bigs>>>(A, B);
  g_launches += 4;
  LTS_KCHECK();
  return 0;
}

// Level-parallel flood t -> t+1 of every large region flagged BST_LEVEL
// (localize_level.cuh), between k_big_setup and k_big_check.  The host drives
// the level / Boruvka-round / pointer-jumping loops from three counters read
// back on the flood stream.
static int lv_read(Ctx &c, int first, int count) {
  LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_LV + first, c.w.scal + SC_LV + first, sizeof(int) * count,
                           cudaMemcpyDeviceToHost, g_lvs));
  LTS_CUDA(cudaStreamSynchronize(g_lvs));
  return 0;
}

static int big_level_flood(Ctx &c, const LocArgs &A, const BigArgs &B) {
  WS &w = c.w;
  LvArgs L = w.lv;
  L.ctr = w.scal + SC_LV;
  L.nj = B.bslots + B.nbig;
  L.level = 0;
  L.alist = nullptr;
  L.na = 0;
  cudaStream_t s = g_lvs;
  const int gj = (int)std::min<int64_t>(((int64_t)L.nj + 255) / 256, 148 * 8);
  const int gs = (int)std::min<int64_t>(((int64_t)B.bslots + 255) / 256, 148 * 8);
  int *hc = c.h_scal + SC_LV;
  int levels = 0, rounds_total = 0, lv_grid = 1;
  LTS_CUDA(cudaMemsetAsync(L.ctr, 0, sizeof(int) * LVC_N, s));
  bool host_loop = getenv("LTS_LEVEL_HOST") != nullptr;  // debugging: one launch per phase
  {
    // devices without cooperative launches take the host-driven loop as well
    DevState &d = *g_cur;
    if (d.coop_ok < 0) {
      int dev = 0, ok = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
      d.coop_ok = ok ? 1 : 0;
    }
    if (!d.coop_ok) host_loop = true;
  }
  const int nd = c.g.ndim;
  if (!host_loop) {
    // every level in one cooperative launch
    DevState &d = *g_cur;
    const void *fn = nd == 2 ? (const void *)k_lv_coop<6> : nd == 3 ? (const void *)k_lv_coop<14>
                                                                   : (const void *)k_lv_coop<kCsrK>;
    if (!d.lv_blocks[nd]) {
      int dev = 0, nsm = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      LTS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 512, 0));
      d.lv_blocks[nd] = nsm;
      d.lv_per[nd] = std::max(1, per);
    }
    // one block per SM keeps the grid barriers short; large key spaces take
    // more blocks for memory parallelism
    {
      static int per_env = -1;  // LTS_LV_PER: CTAs per SM of the cooperative grid (tuning)
      if (per_env < 0) {
        const char *e = getenv("LTS_LV_PER");
        per_env = e ? atoi(e) : 0;
      }
      const int want = per_env > 0 ? per_env : (L.nj >= (1 << 20) ? 2 : 1);
      lv_grid = d.lv_blocks[nd] * std::min(d.lv_per[nd], want);
    }
    lv_grid = (int)std::max<int64_t>(1, std::min<int64_t>(lv_grid, ((int64_t)L.nj + 511) / 512));
    void *kargs[] = {(void *)&A, (void *)&B, (void *)&L};
    LTS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(lv_grid), dim3(512), kargs, 0, s));
    g_launches++;
  } else {
    k_lv_nsrc<<<gs, 256, 0, s>>>(A, B);
    k_lv_init<<<gj, 256, 0, s>>>(A, B, L);
    g_launches += 2;
    LTS_TRY(lv_read(c, LVC_ACTIVE, 1));
    int active = hc[LVC_ACTIVE];
    if (active > 0) {  // the spanning forest of the flood
      L.level = 1;
      k_lv_prep<<<gj, 256, 0, s>>>(L);
      g_launches++;
      for (int round = 0;; round++) {
        if (round >= 64) return lts_set_error(LTS_E_CUDA, "level flood: spanning forest did not converge");
        LTS_CUDA(cudaMemsetAsync(L.ctr + LVC_HOOKS, 0, sizeof(int), s));
        if (nd == 2) k_lv_scan<6><<<gj, 256, 0, s>>>(A, B, L);
        else if (nd == 3) k_lv_scan<14><<<gj, 256, 0, s>>>(A, B, L);
        else k_lv_scan<kCsrK><<<gj, 256, 0, s>>>(A, B, L);
        k_lv_hook<<<gj, 256, 0, s>>>(L);
        k_lv_jump<<<gj, 256, 0, s>>>(L);
        g_launches += 3;
        rounds_total++;
        LTS_TRY(lv_read(c, LVC_HOOKS, 1));
        if (hc[LVC_HOOKS] == 0) break;
      }
    }
    while (active > 0) {
      L.level = ++levels;
      if (nd == 2) k_lv_chain<6><<<gj, 256, 0, s>>>(A, B, L);
      else if (nd == 3) k_lv_chain<14><<<gj, 256, 0, s>>>(A, B, L);
      else k_lv_chain<kCsrK><<<gj, 256, 0, s>>>(A, B, L);
      if (nd == 2) k_lv_pins<6><<<gj, 256, 0, s>>>(A, B, L, L.pm);
      else if (nd == 3) k_lv_pins<14><<<gj, 256, 0, s>>>(A, B, L, L.pm);
      else k_lv_pins<kCsrK><<<gj, 256, 0, s>>>(A, B, L, L.pm);
      g_launches += 2;
      for (int sweep = 0; sweep < 2; sweep++) {
        unsigned long long *Jc = L.pm, *Jn = L.best;
        for (int it = 0;; it++) {
          if (it >= 40) return lts_set_error(LTS_E_CUDA, "level flood: sweep did not converge");
          LTS_CUDA(cudaMemsetAsync(L.ctr + LVC_CHANGED, 0, sizeof(int), s));
          if (sweep == 0) k_lv_sweep<true, false><<<gj, 256, 0, s>>>(L, Jc, Jn);
          else if (it == 0) k_lv_sweep<false, true><<<gj, 256, 0, s>>>(L, Jc, Jn);
          else k_lv_sweep<false, false><<<gj, 256, 0, s>>>(L, Jc, Jn);
          g_launches++;
          std::swap(Jc, Jn);
          LTS_TRY(lv_read(c, LVC_CHANGED, 1));
          if (hc[LVC_CHANGED] == 0) break;
        }
      }
      LTS_CUDA(cudaMemsetAsync(L.ctr + LVC_ACTIVE, 0, sizeof(int), s));
      k_lv_classes<<<gj, 256, 0, s>>>(L);
      g_launches++;
      LTS_TRY(lv_read(c, LVC_ACTIVE, 1));
      if (hc[LVC_ACTIVE] >= active) return lts_set_error(LTS_E_CUDA, "level flood: no progress");
      active = hc[LVC_ACTIVE];
    }
  }
  // extraction index = preorder of F, children in decreasing key
  k_lv_sortkeys<<<gj, 256, 0, s>>>(L);
  LTS_TRY(radix_sort((const uint32_t *)L.skey, (const uint32_t *)L.sval, L.nj, bits_for(L.nj), false, nullptr,
                     (uint32_t *)L.oval, nullptr, w.lsb, s));
  k_lv_gather<<<gj, 256, 0, s>>>(L);
  LTS_TRY(scan_int(L.skey, L.sval, L.nj, w.lbsum, w.scal + SC_LVTMP, false, s));
  k_lv_heads<<<gj, 256, 0, s>>>(L);
  k_lv_off<<<gj, 256, 0, s>>>(A, B, L);
  g_launches += 4;
  if (!host_loop) {
    LTS_CUDA(cudaMemsetAsync(L.ctr + LVK_CHANGED, 0, sizeof(int) * 3, s));
    void *kargs[] = {(void *)&L};
    LTS_CUDA(cudaLaunchCooperativeKernel((const void *)k_lv_pos_coop, dim3(lv_grid), dim3(512), kargs, 0, s));
    g_launches++;
  } else {
    for (int it = 0;; it++) {
      if (it >= 40) return lts_set_error(LTS_E_CUDA, "level flood: positions did not converge");
      LTS_CUDA(cudaMemsetAsync(L.ctr + LVC_CHANGED, 0, sizeof(int), s));
      k_lv_pos_round<<<gj, 256, 0, s>>>(L);
      k_lv_pos_round<<<gj, 256, 0, s>>>(L);
      g_launches += 2;
      LTS_TRY(lv_read(c, LVC_CHANGED, 1));
      if (hc[LVC_CHANGED] == 0) break;
    }
  }
  k_lv_write<<<gj, 256, 0, s>>>(A, B, L);
  g_launches++;
  static const bool verbose = getenv("LTS_LEVEL_VERBOSE") != nullptr;
  if (verbose) {
    if (!host_loop) {
      LTS_TRY(lv_read(c, LVK_LEVELS, 2));
      levels = hc[LVK_LEVELS];
      rounds_total = hc[LVK_ROUNDS];
    }
    long long clk[8];
    cudaMemcpyFromSymbol(clk, d_lvclk, sizeof(clk));
    fprintf(stderr, "[lts] level flood: nj %d levels %d boruvka rounds %d | Mcyc chain %.2f prep %.2f scan %.2f hook %.2f "
            "jump %.2f beta %.2f classes %.2f\n", L.nj, levels, rounds_total, clk[0] / 1e6, clk[1] / 1e6, clk[2] / 1e6,
            clk[3] / 1e6, clk[4] / 1e6, clk[5] / 1e6, clk[6] / 1e6);
    memset(clk, 0, sizeof(clk));
    cudaMemcpyToSymbol(d_lvclk, clk, sizeof(clk));
    if (getenv("LTS_LEVEL_LOG") && levels >= 20) {  // per level: active, sweep rounds, sweep kcycles, level kcycles
      static long long lg[128][4];
      cudaMemcpyFromSymbol(lg, d_lvlog, sizeof(lg));
      for (int i = 0; i < std::min(levels, 128); i++)
        fprintf(stderr, "[lts]   level %d: active %lld rounds %lld sweep %lld kcyc level %lld kcyc\n", i + 1, lg[i][0],
                lg[i][1], lg[i][2] / 1000, lg[i][3] / 1000);
    }
  }
  LTS_KCHECK();
  return 0;
}

__global__ void k_order_keys(const int *rsize, int R, uint32_t *key) {
  GRID_STRIDE(r, R) key[r] = 0x7fffffffu - (uint32_t)rsize[r];
}

// classified: w.flags / w.ptr already hold this pass's classification of rank
static int run_pass(Ctx &c, int kind, const int *rank, const int *inv, const uint8_t *pmark,
                    int max_iter, int *new_rank, int *new_inv, float *g, lts_pass_report_t *rep,
                    lts_regions_view_t *view, bool classified = false, int *pstats = nullptr,
                    bool list_mode = false) {
  WS &w = c.w;
  const int64_t n = c.n;
  const int ni = (int)n;
  const int rev = kind;
  cudaStream_t s = c.s;
  lts_pass_report_t r{};
  r.kind = kind;
  int R = 0, C = 0, S = 0, nshared = 0;
  {
    Phase ph(c, LTS_PH_CLASSIFY);
    if (!classified)
      classify_any(c, rank, w.flags, nullptr, nullptr, c.lut, w.ptr, kind == 0 ? PTR_ASC : PTR_DESC, s);
    LTS_KCHECK();
  }
  {
    Phase ph(c, LTS_PH_DISCOVER);
    LTS_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(int) * SC_N, s));
    k_mark_maxima<<<NB(n), 256, 0, s>>>(w.flags, pmark, kind, n, w.vcls, w.cst, w.mlist,
                                         w.scal + SC_COUNTS, w.comp, w.par, w.acc, w.rpar, w.bestP);
    g_launches++;
    LTS_KCHECK();
    LTS_TRY(readback(c, SC_COUNTS, 2));
    const int nm = c.h_scal[SC_COUNTS], nD = c.h_scal[SC_COUNTS + 1], nP = nm - nD;
    r.seeds = nD;
    if (nD == 0) {
      LTS_CUDA(cudaMemcpyAsync(new_rank, rank, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
      LTS_CUDA(cudaMemcpyAsync(new_inv, inv, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
      if (rep) *rep = r;
      if (view) memset(view, 0, sizeof(*view));
      return 0;
    }
    if (nP == 0) return lts_set_error(LTS_E_NO_SADDLE, "every extremum of this kind is discarded: no saddle");
    for (int j = 0; j < LTS_JUMPS; j++) k_jump<<<NB(n), 256, 0, s>>>(w.ptr, n);
    k_compress<<<NB(n), 256, 0, s>>>(w.ptr, n);
    k_roots<<<NB(n), 256, 0, s>>>(w.ptr, n, w.M);
    g_launches += 3;
    g_launches += 3;
    // maxima-graph edges, de-duplicated per manifold pair in a hash table
    // sized from the maxima count; list mode if the table would overflow
    static const bool force_list_env = getenv("LTS_FORCE_EDGE_LIST") != nullptr;  // test hook
    const bool force_list = force_list_env || list_mode;
    int hbits = 12;
    while (hbits < 30 && (1ll << hbits) < 64ll * nm) hbits++;
    while (hbits > 10 && 18ll << hbits > 12 * w.emax) hbits--;
    EdgeHash H{(unsigned long long *)w.ebuf, (int *)(w.ebuf + (8ll << hbits)), hbits,
               w.scal + SC_ECOUNT, w.scal + SC_ACTIVE};
    int *ea = w.ea, *eb = w.eb, *ew = w.ew;
    // One attempt (hash table, or list mode when forced): the edge count
    // stays on the device and the table overflow flag is read back together
    // with the Boruvka / region results below; an overflow reruns the pass in
    // list mode (the inputs are untouched until then).
    {
      const int mode = force_list ? 1 : 0;
      if (mode == 0) {
        ea = (int *)(w.ebuf + (12ll << hbits));
        eb = ea + (1ll << (hbits - 1));
        ew = eb + (1ll << (hbits - 1));
        LTS_CUDA(cudaMemsetAsync(w.ebuf, 0xff, 12ull << hbits, s));
      } else {
        H.bits = 0;
        ea = w.ea; eb = w.eb; ew = w.ew;
        LTS_CUDA(cudaMemsetAsync(w.scal + SC_ECOUNT, 0, sizeof(int) * 2, s));
        LTS_CUDA(cudaMemsetAsync(w.bestP, 0, sizeof(unsigned long long) * n, s));
      }
      if (c.g.ndim == 0) {
        k_edges_csr<<<NB(n), 256, 0, s>>>(c.g, rank, rev, w.M, w.vcls, ea, eb, ew, w.scal + SC_ECOUNT, w.bestP, H);
      } else {
        dim3 eg((c.g.nx + ET_TX - 1) / ET_TX, (c.g.ny + ET_TY - 1) / ET_TY,
                c.g.ndim == 2 ? 1 : (c.g.nz + ET_ZC - 1) / ET_ZC);
        dim3 eb3(ET_TX, ET_TY);
        if (c.g.ndim == 2)
          k_edges_tile<2><<<eg, eb3, 0, s>>>(c.g, rank, rev, w.M, w.vcls, ea, eb, ew, w.scal + SC_ECOUNT, w.bestP, H);
        else
          k_edges_tile<3><<<eg, eb3, 0, s>>>(c.g, rank, rev, w.M, w.vcls, ea, eb, ew, w.scal + SC_ECOUNT, w.bestP, H);
      }
      g_launches++;
      if (mode == 0) {
        k_hash_compact<<<NB(1ll << hbits), 256, 0, s>>>(H, ea, eb, ew, w.scal + SC_TMP);
        g_launches++;
      }
      LTS_KCHECK();
    }
    // Boruvka rounds: tau(m) = bottleneck to preserved maxima, all rounds in
    // one cooperative launch (grid barriers between phases); one readback
    {
      // one CTA per SM keeps the grid barriers short; graphs with many maxima
      // (hundreds of edges per thread and round) take four
      int &coop_sm = g_cur->coop_blocks, &coop_per = g_cur->coop_per;
      if (!coop_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&coop_per, k_bv_coop, 256, 0);
        coop_per = std::max(1, coop_per);
      }
      const int coop_blocks = coop_sm * std::min(coop_per, nm >= (1 << 16) ? 4 : LTS_BV_COOP_PER_SM);
      BvArgs ba{w.mlist, nm, w.comp, w.par, w.wc, w.rt, w.acc, w.scal + SC_ERR, w.cst, w.vcls, w.bestP, w.best,
                ea, eb, ew, w.scal + SC_ECOUNT, w.scal + SC_BVSTATE};
      void *kargs[] = {&ba};
      LTS_CUDA(cudaLaunchCooperativeKernel((const void *)k_bv_coop, dim3(coop_blocks), dim3(256), kargs, 0, s));
      g_launches++;
      LTS_KCHECK();
    }
    // regions: union-find over edges between claimed endpoints
    k_region_union<<<148 * 8, 256, 0, s>>>(ea, eb, ew, w.scal + SC_ECOUNT, w.vcls, w.acc, w.rpar);
    k_region_roots<<<NB(nm), 256, 0, s>>>(w.mlist, nm, w.vcls, w.acc, rank, rev, ni, w.rpar, w.ridx,
                                           w.scal + SC_NREG, w.rsad, w.rtop, w.rsize);
    k_region_tops<<<NB(nm), 256, 0, s>>>(w.mlist, nm, w.vcls, rank, rev, ni, w.rpar, w.ridx, w.rtop);
    k_region_label<<<NB(n), 256, 0, s>>>(rank, rev, ni, w.M, w.vcls, w.acc, w.rpar, w.ridx, w.reg_of, w.rsize, w.cbits);
    g_launches += 4;
    LTS_KCHECK();
    // one readback for the edge count / table overflow, Boruvka state and
    // the region count
    LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_BVSTATE, w.scal + SC_BVSTATE, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    LTS_TRY(readback(c, SC_ECOUNT, SC_NREG + 1 - SC_ECOUNT));
    if (!force_list && c.h_scal[SC_ACTIVE])  // hash table overflow: rerun in list mode
      return run_pass(c, kind, rank, inv, pmark, max_iter, new_rank, new_inv, g, rep, view, true, pstats, true);
    if (c.h_scal[SC_ERR]) return lts_set_error(LTS_E_NO_SADDLE, "a discarded extremum cannot reach a preserved one");
    r.maxima_edges = c.h_scal[SC_ECOUNT];
    r.boruvka_rounds = c.h_scal[SC_BVSTATE + 1];
    R = c.h_scal[SC_NREG];
  }
  {
    Phase ph(c, LTS_PH_ASSEMBLE);
    k_region_slots<<<NB(R), 256, 0, s>>>(w.rsize, R, w.rtmp);
    g_launches++;
    LTS_TRY(scan_int(w.rtmp, w.rptr, R, w.bsum, w.scal + SC_S, false, s));
    {
      const int cc_tiles = (int)((n + CC_TILE - 1) / CC_TILE);
      LTS_CUDA(cudaMemsetAsync(w.flagscan, 0, sizeof(int) * (cc_tiles + 1), s));
      LTS_CUDA(cudaMemsetAsync(w.scal + SC_C, 0, sizeof(int), s));
      if (cc_tiles > 0)
        k_claimed_compact_lb<<<cc_tiles, CC_T, 0, s>>>(inv, rev, ni, w.cbits, w.reg_of, w.ckey, w.cval,
                                                     w.flagscan, w.scal + SC_C);
      g_launches++;
    }
    // regions are ordered largest first: the first nbig (k > BIG_THRESHOLD) go
    // to the CTA-batched flood on a side stream, the rest to warp floods
    k_count_big<<<NB(R), 256, 0, s>>>(w.rsize, R, BIG_THRESHOLD, w.scal + SC_NBIG);
    g_launches++;
    LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_NBIG, w.scal + SC_NBIG, sizeof(int) * 8, cudaMemcpyDeviceToHost, s));
    LTS_TRY(readback(c, SC_S, 2));
    S = c.h_scal[SC_S];
    C = c.h_scal[SC_C];
    LTS_CUDA(cudaMemcpyAsync(w.rptr + R, w.scal + SC_S, sizeof(int), cudaMemcpyDeviceToDevice, s));
    LTS_TRY(radix_sort(w.ckey, w.cval, C, bits_for(R - 1), false, w.skey, w.sval, nullptr, w.sb, s));
    k_place<<<NB(C), 256, 0, s>>>(w.skey, w.sval, C, w.rptr, w.verts, w.reg_of);
    k_place_saddles<<<NB(R), 256, 0, s>>>(inv, rev, ni, w.rsad, R, w.rptr, w.verts);
    // schedule: largest region first (stable by region id)
    k_order_keys<<<NB(R), 256, 0, s>>>(w.rsize, R, (uint32_t *)w.okey);
    g_launches += 3;
    LTS_TRY(radix_sort((uint32_t *)w.okey, nullptr, R, 31, false, w.okey2, (uint32_t *)w.order, nullptr, w.sb, s));
    LTS_KCHECK();
  }
  {
    Phase ph(c, LTS_PH_LOCALIZE);
    LocArgs A;
    A.g = c.g; A.rank = rank; A.rev = rev; A.order = w.order; A.R = R; A.rptr = w.rptr;
    A.verts = w.verts; A.slot_of = w.reg_of; A.buf0 = w.buf0; A.buf1 = w.buf1;
    A.buf2 = w.buf2; A.out = w.out; A.gheap = w.gheap; A.sfl = w.sfl; A.n_iters = w.nit;
    A.status = w.st; A.max_iter = max_iter; A.queue = w.scal + SC_QUEUE; A.qbase = 0;
    const int nbig = c.h_scal[SC_NBIG];
    r.big_regions = nbig;
    BigArgs B{};
    int big_gx = 1;
    if (nbig > 0) {
      LTS_TRY(big_stream_fork(s));
      B.inv = w.binv; B.gbits = w.gbits; B.nrow = w.nrow; B.nrowkey = w.nrowkey; B.qbase = 0; B.nbig = nbig;
      B.queue = w.scal + SC_BIGQ;
      B.v0 = w.bigv0;
      B.st = w.bst;
      B.nactive = w.scal + SC_BIGACT;
      B.work = reinterpret_cast<unsigned long long *>(w.scal + SC_BIGWORK);
      k_fill_int<<<NB(nbig), 256, 0, g_bigs>>>(w.bigv0, nbig, 0x7fffffff);
      LTS_CUDA(cudaMemsetAsync(w.bst, 0, sizeof(int) * BST_W * (size_t)nbig, g_bigs));
      k_big_prefix<<<1, 1024, 0, g_bigs>>>(A, B, w.bpre);
      B.bpre = w.bpre;
      B.bslots = c.h_scal[SC_BIGSLOTS];
      // flat kernels over all big-region slots
      big_gx = (int)std::min<int64_t>((B.bslots + 255) / 256, 148 * 8);
      if (c.g.ndim == 2) k_big_rows<2><<<big_gx, 256, 0, g_bigs>>>(A, B);
      else if (c.g.ndim == 3) k_big_rows<3><<<big_gx, 256, 0, g_bigs>>>(A, B);
      else k_big_rows<0><<<big_gx, 256, 0, g_bigs>>>(A, B);
      {
        const char *e = getenv("LTS_LEVEL_MIN");
        g_level_min = e ? atoi(e) : 0;
        e = getenv("LTS_LEVEL_RATIO");
        g_level_ratio = e ? atoi(e) : 32;
        e = getenv("LTS_LEVEL_GIANT");
        g_level_giant = e ? atoi(e) : 16384;
      }
      LTS_CUDA(cudaMemsetAsync(w.scal + SC_BIGACT + 1, 0, sizeof(int), g_bigs));
      k_big_init<<<NB(nbig), 256, 0, g_bigs>>>(A, B, g_level_min, g_level_ratio, g_level_giant, w.scal + SC_BIGACT + 1);
      if (getenv("LTS_LEVEL_VERBOSE")) {  // the largest regions: slots, local maxima, path chosen
        int hb[4 * BST_W], hp[5];
        const int m = std::min(nbig, 4);
        cudaMemcpyAsync(hb, w.bst, sizeof(int) * BST_W * m, cudaMemcpyDeviceToHost, g_bigs);
        cudaMemcpyAsync(hp, w.bpre, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost, g_bigs);
        cudaStreamSynchronize(g_bigs);
        for (int i = 0; i < m; i++)
          fprintf(stderr, "[lts] big region %d: k %d local maxima %d level %d\n", i, hp[i + 1] - hp[i],
                  hb[i * BST_W + BST_NMAX], hb[i * BST_W + BST_LEVEL]);
      }
      g_launches += 4;
      // which regions flood level-parallel is decided on the device: one readback,
      // then the first flood of every large region is queued before the main
      // stream's work so the long floods start first
      LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_BIGACT + 1, w.scal + SC_BIGACT + 1, sizeof(int), cudaMemcpyDeviceToHost,
                               g_bigs));
      LTS_CUDA(cudaStreamSynchronize(g_bigs));
      g_nlevel = c.h_scal[SC_BIGACT + 1];
      LTS_TRY(big_iteration(c, A, B, big_gx));
      // A cooperative flood over millions of keys pays for every grid barrier
      // with the slowest CTA: sharing the SMs with the warp floods below slows
      // it by far more than those take (cfg5: 600 vs 370 ms), so the main
      // stream waits for the first flood of large key spaces.
      static int solo = -1;  // LTS_LEVEL_SOLO: key-space size from which the main stream waits
      if (solo < 0) {
        const char *e = getenv("LTS_LEVEL_SOLO");
        solo = e ? atoi(e) : (4 << 20);
      }
      if (g_nlevel > 0 && g_bigs != s && B.bslots >= solo) {
        LTS_CUDA(cudaEventRecord(g_cur->join, g_bigs));
        LTS_CUDA(cudaStreamWaitEvent(s, g_cur->join, 0));
      }
    }
    A.qbase = nbig;
    if (R > nbig) {
      int blocks = (R - nbig + LOC_WARPS - 1) / LOC_WARPS;
      if (blocks > 148 * 8) blocks = 148 * 8;
      if (c.g.ndim == 2) k_localize<2><<<blocks, 32 * LOC_WARPS, 0, s>>>(A);
      else if (c.g.ndim == 3) k_localize<3><<<blocks, 32 * LOC_WARPS, 0, s>>>(A);
      else k_localize<0><<<blocks, 32 * LOC_WARPS, 0, s>>>(A);
      g_launches++;
    }
    // Work that does not need the local orders runs while the large-region
    // floods finish on the side stream: the integration prefix, the ranks of
    // every unclaimed vertex (k_integrate_plain) and the numeric realization.
    LTS_CUDA(cudaMemsetAsync(w.delta, 0, sizeof(int) * n, s));
    k_delta_claimed<<<NB(C), 256, 0, s>>>(w.sval, C, rank, rev, ni, w.delta);
    k_delta_saddles<<<NB(R), 256, 0, s>>>(w.rsad, w.rsize, R, w.delta);
    k_count_shared<<<NB(R), 256, 0, s>>>(w.rsad, w.rsize, R, w.delta, w.scal + SC_NSHARED);
    g_launches += 3;
    LTS_TRY(scan_int(w.delta, w.D, n, w.bsum, w.scal + SC_TMP, true, s));
    LTS_TRY(readback(c, SC_NSHARED, 1));
    nshared = c.h_scal[SC_NSHARED];
    r.shared_saddles = nshared;
    if (nshared) {
      k_iota<<<NB(R), 256, 0, s>>>(w.okey, R);  // reuse as values
      g_launches++;
      LTS_TRY(radix_sort((const uint32_t *)w.rsad, (const uint32_t *)w.okey, R, bits_for(n - 1), false,
                         w.okey2, w.oval, nullptr, w.sb, s));
      k_pos_of<<<NB(R), 256, 0, s>>>(w.oval, R, w.sib_rid, w.pos_of);
      g_launches++;
    }
    k_integrate_plain<<<NB(n), 256, 0, s>>>(inv, rev, ni, w.cbits, w.D, new_rank, new_inv);
    g_launches++;
    if (g) {
      if (c.g_host && c.g_copy_pending) {  // an earlier copy of g still reads it
        LTS_CUDA(cudaStreamWaitEvent(s, g_cur->g_copied, 0));
        c.g_copy_pending = false;
      }
      k_realize<<<NB(C), 256, 0, s>>>(w.skey, w.sval, C, w.rptr, w.verts, g);
      g_launches++;
      c.g_copy_valid = false;
      if (c.g_host && kind == 1) {
        // g is final unless another outer iteration follows: copy it out now,
        // beside this pass's floods
        DevState &d = *g_cur;
        LTS_CUDA(cudaEventRecord(d.g_ready, s));
        LTS_CUDA(cudaStreamWaitEvent(d.copys, d.g_ready, 0));
        LTS_CUDA(cudaMemcpyAsync(c.g_host, g, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost, d.copys));
        LTS_CUDA(cudaEventRecord(d.g_copied, d.copys));
        c.g_copy_valid = c.g_copy_pending = true;
      }
    }
    if (nbig > 0) {
      // the remaining floods of the large regions; every other localize-phase
      // launch is already queued on the main stream
      for (;;) {
        LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_BIGACT, w.scal + SC_BIGACT, 4 * sizeof(int), cudaMemcpyDeviceToHost, g_bigs));
        LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_LV + LVK_ERR, w.scal + SC_LV + LVK_ERR, sizeof(int), cudaMemcpyDeviceToHost,
                                 g_bigs));
        LTS_CUDA(cudaStreamSynchronize(g_bigs));
        if (g_nlevel > 0 && c.h_scal[SC_LV + LVK_ERR])
          return lts_set_error(LTS_E_CUDA, "level flood: a loop hit its round limit");
        if (c.h_scal[SC_BIGACT] == 0) {
          c.flood_slots += *reinterpret_cast<const long long *>(c.h_scal + SC_BIGWORK);
          break;
        }
        LTS_TRY(big_iteration(c, A, B, big_gx));
      }
      k_big_final<<<big_gx, 256, 0, g_bigs>>>(A, B);
      g_launches++;
      LTS_TRY(big_stream_join(s));
    }
    // per-pass N_I / capped / status-1 / largest: into the caller's device
    // slots (read back once at the end of lts_simplify), else read now
    k_loc_stats<<<NB(R), 256, 0, s>>>(w.nit, w.st, w.rsize, R, pstats ? pstats : w.scal + SC_STATS);
    g_launches += 1;
    LTS_KCHECK();
    if (!pstats) {
      LTS_TRY(readback(c, SC_STATS, 4));
      r.n_iter_max = c.h_scal[SC_STATS];
      r.capped = c.h_scal[SC_STATS + 1];
      r.largest = c.h_scal[SC_STATS + 3];
      if (c.h_scal[SC_STATS + 2]) return lts_set_error(LTS_E_LOCALIZE_NO_MIN, "region without an admissible boundary minimum (status 1)");
    }
  }
  {
    Phase ph(c, LTS_PH_INTEGRATE);
    k_integrate_regions<<<NB(C), 256, 0, s>>>(w.skey, w.sval, C, w.rptr, w.out, w.rsad, w.rsize, w.rtop,
                                              w.delta, w.D, w.sib_rid, w.pos_of, R, nshared, rev, ni,
                                              new_rank, new_inv);
    g_launches++;
    LTS_KCHECK();
  }
  r.regions = R;
  r.claimed = C;
  if (rep) *rep = r;
  if (view) {
    k_int_to_i64<<<NB(R + 1), 256, 0, s>>>(w.rptr, w.rptr64, R + 1);
    g_launches++;
    view->regions = R;
    view->slots = S;
    view->region_ptr = w.rptr64;
    view->region_verts = w.verts;
    view->local_rank = w.out;
    view->n_iters = w.nit;
    view->status = w.st;
    view->topseed = w.rtop;
  }
  return 0;
}

// A caller-supplied order field F (simplify_field(order=F), remove_extrema,
// lts_extremum_pairs): copied to rankA with its inverse in invA.  F must be a
// bijection onto [0, n) (else LTS_E_INVALID) and f, when given, must be
// finite (reference ScalarField, order.py:35-36; else LTS_E_FIELD_NONFINITE).
static int install_order(Ctx &c, const float *f, const int32_t *order) {
  WS &w = c.w;
  const int64_t n = c.n;
  cudaStream_t s = c.s;
  LTS_CUDA(cudaMemcpyAsync(w.rankA, order, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  LTS_CUDA(cudaMemsetAsync(w.invA, 0xff, sizeof(int) * n, s));
  LTS_CUDA(cudaMemsetAsync(w.scal + SC_TMP, 0, sizeof(int) * 2, s));
  k_scatter_inverse_checked<<<NB(n), 256, 0, s>>>(w.rankA, w.invA, n, w.scal + SC_TMP);
  g_launches++;
  if (f) {
    k_nonfinite<<<grid_blocks(n, 256, 148 * 8), 256, 0, s>>>(f, n, w.scal + SC_TMP + 1);
    g_launches++;
  }
  LTS_KCHECK();
  LTS_TRY(readback(c, SC_TMP, 2));
  if (c.h_scal[SC_TMP + 1]) return lts_set_error(LTS_E_FIELD_NONFINITE, "scalar field contains NaN or infinite values");
  if (c.h_scal[SC_TMP]) return lts_set_error(LTS_E_INVALID, "order is not a permutation of 0..n-1");
  return 0;
}

// ---------------------------------------------------------------------------
// preserve marks
// ---------------------------------------------------------------------------
__global__ void k_set_pmark(const int64_t *ids, int64_t cnt, int64_t n, uint8_t bit, uint8_t *pmark, int *bad) {
  GRID_STRIDE(i, cnt) {
    int64_t v = ids[i];
    if (v < 0 || v >= n) {
      atomicOr(bad, 1);
      continue;
    }
    atomicOr((unsigned *)(pmark + (v & ~(int64_t)3)), (unsigned)bit << (8 * (v & 3)));
  }
}

__global__ void k_set_global(const int *inv, int64_t n, int which, uint8_t *pmark) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int v = which == 0 ? inv[0] : inv[n - 1];
    pmark[v] |= which == 0 ? PM_MIN : PM_MAX;
  }
}

__global__ void k_check_pres(const uint8_t *flags, const uint8_t *pmark, int64_t n, int *bad) {
  GRID_STRIDE(v, n) {
    uint8_t p = pmark[v], f = flags[v];
    if (((p & PM_MAX) && !(f & FL_MAX)) || ((p & PM_MIN) && !(f & FL_MIN))) atomicOr(bad, 1);
  }
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *lts_version(void) { return "lts_sm100 1.0 (sm_100a)"; }
const char *lts_last_error(void) { return g_err.c_str(); }
int64_t lts_kernel_launches(void) { return g_launches; }

// Kernel micro-benchmarks for the roofline report: each rep flushes L2 with a
// 256 MiB memset, then times one kernel (or kernel group) with events placed
// directly around it on `stream`.  out_ms[0] order-field sort (histogram +
// 4 onesweep passes + rank scatter), [1] classification (flags), [2]
// classification + ascent pointer, [3] mean onesweep pass.  Averages over reps.
// ---------------------------------------------------------------------------
// persistence-driven mode: extremum-saddle pairs (persistence.cuh)
// ---------------------------------------------------------------------------
static int order_field_impl(Ctx &c, const float *f, int32_t *rank, int32_t *inverse, bool defer_check = false);

static int pairs_impl(Ctx &c, const float *f, const int *rank, const int *inv, int kind, double eps,
                      int32_t *ext_out, int32_t *sad_out, int64_t *count_out) {
  WS &w = c.w;
  const int64_t n = c.n;
  const int ni = (int)n;
  const int rev = kind;
  cudaStream_t s = c.s;
  // every extremum of the polarity is a seed: no preserve marks
  LTS_CUDA(cudaMemsetAsync(w.pmark, 0, (size_t)n, s));
  LTS_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(int) * SC_N, s));
  classify_any(c, rank, w.flags, nullptr, nullptr, c.lut, w.ptr, kind == 0 ? PTR_ASC : PTR_DESC, s);
  k_mark_maxima<<<NB(n), 256, 0, s>>>(w.flags, w.pmark, kind, n, w.vcls, w.cst, w.mlist, w.scal + SC_COUNTS,
                                       w.comp, w.par, w.acc, w.rpar, w.bestP);
  for (int j = 0; j < LTS_JUMPS; j++) k_jump<<<NB(n), 256, 0, s>>>(w.ptr, n);
  k_compress<<<NB(n), 256, 0, s>>>(w.ptr, n);
  k_roots<<<NB(n), 256, 0, s>>>(w.ptr, n, w.M);
  g_launches += 7;
  LTS_KCHECK();
  LTS_TRY(readback(c, SC_COUNTS, 2));
  const int nm = c.h_scal[SC_COUNTS];
  *count_out = nm;
  if (nm == 0) return 0;
  // extrema in ascending vertex order = node order
  LTS_TRY(radix_sort((const uint32_t *)w.mlist, nullptr, nm, bits_for(ni - 1), false, w.ckey, w.cval, nullptr,
                     w.sb, s));
  int *idx = w.delta, *nrank = w.rt, *comp = w.comp, *par = w.par, *pair = w.acc, *rt = w.wc;
  k_pn_index<<<NB(nm), 256, 0, s>>>(w.ckey, nm, idx, rank, rev, ni, nrank, comp, pair);
  g_launches++;
  // maxima-graph edges (hash-deduplicated per manifold pair; list fallback)
  int hbits = 12;
  while (hbits < 30 && (1ll << hbits) < 64ll * nm) hbits++;
  while (hbits > 10 && 18ll << hbits > 12 * w.emax) hbits--;
  EdgeHash H{(unsigned long long *)w.ebuf, (int *)(w.ebuf + (8ll << hbits)), hbits, w.scal + SC_ECOUNT,
             w.scal + SC_ACTIVE};
  int *ea = w.ea, *eb = w.eb, *ew = w.ew;
  for (int mode = 0; mode < 2; mode++) {
    if (mode == 0) {
      ea = (int *)(w.ebuf + (12ll << hbits));
      eb = ea + (1ll << (hbits - 1));
      ew = eb + (1ll << (hbits - 1));
      LTS_CUDA(cudaMemsetAsync(w.ebuf, 0xff, 12ull << hbits, s));
    } else {
      H.bits = 0;
      ea = w.ea; eb = w.eb; ew = w.ew;
      LTS_CUDA(cudaMemsetAsync(w.scal + SC_ECOUNT, 0, sizeof(int) * 2, s));
    }
    dim3 eg((c.g.nx + ET_TX - 1) / ET_TX, (c.g.ny + ET_TY - 1) / ET_TY,
            c.g.ndim == 2 ? 1 : (c.g.nz + ET_ZC - 1) / ET_ZC);
    dim3 eb3(ET_TX, ET_TY);
    if (c.g.ndim == 2)
      k_edges_tile<2><<<eg, eb3, 0, s>>>(c.g, rank, rev, w.M, w.vcls, ea, eb, ew, w.scal + SC_ECOUNT, w.bestP, H);
    else
      k_edges_tile<3><<<eg, eb3, 0, s>>>(c.g, rank, rev, w.M, w.vcls, ea, eb, ew, w.scal + SC_ECOUNT, w.bestP, H);
    g_launches++;
    if (mode == 0) {
      k_hash_compact<<<NB(1ll << hbits), 256, 0, s>>>(H, ea, eb, ew, w.scal + SC_TMP);
      g_launches++;
    }
    LTS_KCHECK();
    LTS_TRY(readback(c, SC_ECOUNT, 2));
    if (mode == 0 && c.h_scal[SC_ACTIVE] == 0) break;
  }
  const int ne = c.h_scal[SC_ECOUNT];
  int *ia = w.nrowkey, *ib = w.nrowkey + w.emax, *mst = w.nrow;
  if (ne > 0) {
    k_pn_edges<<<NB(ne), 256, 0, s>>>(ea, eb, ne, idx, ia, ib, mst);
    g_launches++;
  }
  // maximum spanning forest (Boruvka)
  for (int round = 0; round < 64 && ne > 0; round++) {
    LTS_CUDA(cudaMemsetAsync(w.scal + SC_ACTIVE, 0, sizeof(int), s));
    k_pn_reset<<<NB(nm), 256, 0, s>>>(nm, w.best);
    k_pn_best<<<NB(ne), 256, 0, s>>>(ia, ib, ew, ne, comp, w.best);
    k_pn_hook<<<NB(nm), 256, 0, s>>>(nm, comp, w.best, ia, ib, par, mst, w.scal + SC_ACTIVE);
    k_pn_cycle<<<NB(nm), 256, 0, s>>>(nm, comp, par);
    k_pn_roots<<<NB(nm), 256, 0, s>>>(nm, comp, par, rt);
    k_pn_relabel<<<NB(nm), 256, 0, s>>>(nm, comp, rt);
    g_launches += 6;
    LTS_KCHECK();
    LTS_TRY(readback(c, SC_ACTIVE, 1));
    if (c.h_scal[SC_ACTIVE] == 0) break;
  }
  // forest edges by decreasing weight, then the Elder-rule sweep
  int cnt = 0;
  if (ne > 0) {
    LTS_CUDA(cudaMemsetAsync(w.scal + SC_TMP, 0, sizeof(int), s));
    k_pn_mst_keys<<<NB(ne), 256, 0, s>>>(mst, ew, ne, ni, (uint32_t *)w.rtmp, (uint32_t *)w.okey,
                                         w.scal + SC_TMP);
    g_launches++;
    LTS_TRY(readback(c, SC_TMP, 1));
    cnt = c.h_scal[SC_TMP];
  }
  if (cnt > 0) {
    // leaf peeling: leaves lower than their only neighbour die at that edge
    int *pa = w.buf0, *pb = w.buf1, *pw = w.buf2;
    int *alive = w.flagscan, *deg = w.ridx, *deg0 = w.reg_of, *map = w.loc_of, *nrank2 = w.wc;
    LTS_CUDA(cudaMemsetAsync(deg, 0, sizeof(int) * (size_t)nm, s));
    LTS_CUDA(cudaMemsetAsync(w.scal + SC_BVSTATE, 0, sizeof(int) * 2, s));
    k_pn_leaf_init<<<NB(cnt), 256, 0, s>>>((const uint32_t *)w.okey, cnt, ia, ib, ew, pa, pb, pw, alive, deg);
    g_launches++;
    for (int round = 0; round < LTS_PEEL_ROUNDS; round++) {
      k_pn_copy<<<NB(nm), 256, 0, s>>>(deg, nm, deg0);
      k_pn_peel<<<NB(cnt), 256, 0, s>>>(pa, pb, pw, cnt, nrank, deg0, deg, alive, (int *)w.skey, (int *)w.sval,
                                        w.scal + SC_BVSTATE);
      g_launches += 2;
    }
    LTS_KCHECK();
    LTS_TRY(readback(c, SC_BVSTATE, 1));
    const int rem = cnt - c.h_scal[SC_BVSTATE];
    if (rem > 0) {
      // the rest by the sequential Elder-rule sweep, in decreasing weight
      LTS_CUDA(cudaMemsetAsync(w.scal + SC_TMP, 0, sizeof(int), s));
      k_pn_rest_keys<<<NB(cnt), 256, 0, s>>>(alive, pw, cnt, ni, (uint32_t *)w.rtmp, (uint32_t *)w.okey,
                                             w.scal + SC_TMP);
      k_pn_remap<<<NB(nm), 256, 0, s>>>(deg, nm, nrank, map, nrank2, w.scal + SC_BVSTATE + 1);
      g_launches += 2;
      LTS_TRY(readback(c, SC_BVSTATE, 2));
      const int nm2 = c.h_scal[SC_BVSTATE + 1];
      LTS_TRY(radix_sort((const uint32_t *)w.rtmp, (const uint32_t *)w.okey, rem, bits_for(ni - 1), false,
                         w.okey2, w.oval, nullptr, w.sb, s));
      int *sa = w.verts, *sb2 = w.out, *sw = (int *)w.gheap;
      k_pn_gather_rest<<<NB(rem), 256, 0, s>>>(w.oval, rem, pa, pb, pw, map, sa, sb2, sw);
      const size_t shm = sizeof(int) * (size_t)nm2;
      // LTS_PAIRS_FORCE_GLOBAL (test hook): run the global-memory branch of
      // the sweep on fields whose forest would fit in shared memory
      const int use_smem = shm <= 220 * 1024 && getenv("LTS_PAIRS_FORCE_GLOBAL") == nullptr;
      if (use_smem)
        LTS_CUDA(cudaFuncSetAttribute(k_pn_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
      k_pn_sweep<<<1, 256, use_smem ? shm : 0, s>>>(sa, sb2, sw, rem, nrank2, nm2, par, use_smem, (int *)w.skey,
                                                    (int *)w.sval);
      g_launches += 2;
    }
    k_pn_pairs<<<NB(cnt), 256, 0, s>>>((const int *)w.skey, (const int *)w.sval, cnt, inv, rev, ni, f, eps, idx,
                                       pair);
    g_launches++;
  }
  k_pn_out<<<NB(nm), 256, 0, s>>>(w.ckey, pair, nm, ext_out, sad_out);
  g_launches++;
  LTS_KCHECK();
  return 0;
}

int lts_extremum_pairs(const float *f, const int32_t *order, int ndim, const int64_t *dims, int kind, double epsilon,
                       int32_t *extrema_out, int32_t *saddle_out, int64_t *count_out, void *ws, size_t ws_bytes,
                       void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  if (kind != 0 && kind != 1) return lts_set_error(LTS_E_INVALID, "kind must be 0 (maxima) or 1 (minima)");
  if (!(epsilon >= 0)) return lts_set_error(LTS_E_INVALID, "epsilon must be >= 0");
  WS &w = c.w;
  if (order) {
    LTS_TRY(install_order(c, f, order));
  } else {
    LTS_TRY(order_field_impl(c, f, w.rankA, w.invA));
  }
  LTS_TRY(pairs_impl(c, f, w.rankA, w.invA, kind, epsilon, extrema_out, saddle_out, count_out));
  LTS_CUDA(cudaStreamSynchronize(c.s));
  return 0;
}

int lts_bench_kernels(const float *f, int ndim, const int64_t *dims, int reps, double *out_ms, void *ws,
                      size_t ws_bytes, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  WS &w = c.w;
  cudaStream_t s = c.s;
  const size_t flush_bytes = (size_t)256 << 20;
  char *flush = (char *)w.nrow;  // scratch: >= 256 MiB for n >= 2^21
  size_t nrow_bytes = sizeof(int) * (size_t)(ndim == 2 ? 6 : 14) * (size_t)(2 * c.n + 2);
  size_t fb = flush_bytes < nrow_bytes ? flush_bytes : nrow_bytes;
  cudaEvent_t a = next_event(), b = next_event();
  double acc[4] = {0, 0, 0, 0};
  for (int r = 0; r < reps; r++) {
    float ms;
    // sort
    LTS_CUDA(cudaMemsetAsync(flush, r & 0xff, fb, s));
    LTS_CUDA(cudaEventRecord(a, s));
    LTS_TRY(radix_sort((const uint32_t *)f, nullptr, c.n, 32, true, nullptr, (uint32_t *)w.invA, w.rankA, w.sb, s));
    LTS_CUDA(cudaEventRecord(b, s));
    LTS_CUDA(cudaEventSynchronize(b));
    LTS_CUDA(cudaEventElapsedTime(&ms, a, b));
    acc[0] += ms;
    // classification, flags only
    LTS_CUDA(cudaMemsetAsync(flush, r & 0xff, fb, s));
    LTS_CUDA(cudaEventRecord(a, s));
    classify_any(c, w.rankA, w.flags, nullptr, nullptr, c.lut, nullptr, PTR_NONE, s);
    LTS_CUDA(cudaEventRecord(b, s));
    LTS_CUDA(cudaEventSynchronize(b));
    LTS_CUDA(cudaEventElapsedTime(&ms, a, b));
    acc[1] += ms;
    // classification + ascent pointer
    LTS_CUDA(cudaMemsetAsync(flush, r & 0xff, fb, s));
    LTS_CUDA(cudaEventRecord(a, s));
    classify_any(c, w.rankA, w.flags, nullptr, nullptr, c.lut, w.ptr, PTR_ASC, s);
    LTS_CUDA(cudaEventRecord(b, s));
    LTS_CUDA(cudaEventSynchronize(b));
    LTS_CUDA(cudaEventElapsedTime(&ms, a, b));
    acc[2] += ms;
  }
  LTS_KCHECK();
  for (int i = 0; i < 3; i++) out_ms[i] = acc[i] / (reps > 0 ? reps : 1);
  out_ms[3] = 0;
  return 0;
}

// diagnostics: enable/read the per-region counters of the CTA flood kernel
int lts_debug_big_stats(int enable, int64_t *out, int nregions) {
  LTS_LOCK;
  int on = enable ? 1 : 0;
  LTS_CUDA(cudaMemcpyToSymbol(d_dbg_on, &on, sizeof(int)));
  if (enable) {
    std::vector<long long> z(DBG_MAX * DBG_W, 0);
    LTS_CUDA(cudaMemcpyToSymbol(d_dbg, z.data(), z.size() * sizeof(long long)));
  }
  if (out && nregions > 0) {
    int m = nregions < DBG_MAX ? nregions : DBG_MAX;
    LTS_CUDA(cudaMemcpyFromSymbol(out, d_dbg, sizeof(long long) * m * DBG_W));
  }
  if (nregions < 0) {  // sort phase counters: enable = -nregions-1 ... read into out[0..7]
    int on = enable ? 1 : 0;
    LTS_CUDA(cudaMemcpyToSymbol(rs::d_sort_dbg_on, &on, sizeof(int)));
    if (enable) {
      long long z[8] = {0};
      LTS_CUDA(cudaMemcpyToSymbol(rs::d_sort_dbg, z, sizeof(z)));
    } else if (out) {
      LTS_CUDA(cudaMemcpyFromSymbol(out, rs::d_sort_dbg, sizeof(long long) * 8));
    }
  }
  return 0;
}

int lts_workspace_size(int ndim, const int64_t *dims, size_t *bytes) {
  if (ndim != 2 && ndim != 3) return lts_set_error(LTS_E_BAD_DIMS, "grid must be 2D or 3D");
  int64_t n = 1;
  for (int a = 0; a < ndim; a++) {
    if (dims[a] < 2) return lts_set_error(LTS_E_BAD_DIMS, "every grid axis needs at least 2 vertices");
    n *= dims[a];
  }
  WS w;
  *bytes = (size_t)carve(&w, nullptr, ndim, n) + 256;
  return 0;
}

// defer_check: the caller reads w.sb.nonfinite back later (with its own
// readback) instead of synchronising here
static int order_field_impl(Ctx &c, const float *f, int32_t *rank, int32_t *inverse, bool defer_check) {
  WS &w = c.w;
  Phase ph(c, LTS_PH_ORDER);
  LTS_CUDA(cudaMemsetAsync(w.sb.nonfinite, 0, sizeof(int), c.s));
  uint32_t *inv_out = inverse ? (uint32_t *)inverse : w.sval;
  LTS_TRY(radix_sort((const uint32_t *)f, nullptr, c.n, 32, true, nullptr, inv_out, rank, w.sb, c.s));
  LTS_KCHECK();
  if (defer_check) return 0;
  LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_TMP, w.sb.nonfinite, sizeof(int), cudaMemcpyDeviceToHost, c.s));
  LTS_CUDA(cudaStreamSynchronize(c.s));
  if (c.h_scal[SC_TMP]) return lts_set_error(LTS_E_FIELD_NONFINITE, "scalar field contains NaN or infinite values");
  return 0;
}

int lts_check_field(const float *f, int64_t n, void *stream) {
  LTS_LOCK;
  LTS_TRY(select_device());
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (!g_cur->h_scal) LTS_CUDA(cudaHostAlloc((void **)&g_cur->h_scal, sizeof(int) * SC_N, cudaHostAllocDefault));
  int *d = nullptr;
  LTS_CUDA(cudaMallocAsync((void **)&d, sizeof(int), s));
  LTS_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  k_nonfinite<<<grid_blocks(n, 256, 148 * 8), 256, 0, s>>>(f, n, d);
  g_launches++;
  LTS_KCHECK();
  LTS_CUDA(cudaMemcpyAsync(g_cur->h_scal + SC_TMP, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  LTS_CUDA(cudaFreeAsync(d, s));
  LTS_CUDA(cudaStreamSynchronize(s));
  if (g_cur->h_scal[SC_TMP]) return lts_set_error(LTS_E_FIELD_NONFINITE, "scalar field contains NaN or infinite values");
  return 0;
}

int lts_realize_numeric(double *g, const int32_t *inverse, int64_t n, double zeta, void *stream) {
  LTS_LOCK;
  LTS_TRY(select_device());
  if (!(zeta >= 0)) return lts_set_error(LTS_E_INVALID, "zeta must be >= 0");
  if (n < 2) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_realize_sweep<<<1, RZ_T, 0, s>>>(g, inverse, n, zeta);
  g_launches++;
  LTS_KCHECK();
  LTS_CUDA(cudaStreamSynchronize(s));
  return 0;
}

int lts_order_field(const float *f, int ndim, const int64_t *dims, int32_t *rank, int32_t *inverse,
                    void *ws, size_t ws_bytes, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  return order_field_impl(c, f, rank, inverse);
}

int lts_classify(const int32_t *rank, int ndim, const int64_t *dims, uint8_t *flags, int16_t *lower,
                 int16_t *upper, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, nullptr, 0, stream));
  if ((lower == nullptr) != (upper == nullptr)) return lts_set_error(LTS_E_INVALID, "lower and upper go together");
  classify_any(c, rank, flags, lower, upper, c.lut, nullptr, PTR_NONE, c.s);
  LTS_KCHECK();
  return 0;
}

int lts_remove_pass(int kind, const int32_t *rank, const int32_t *inverse, const uint8_t *pmark, int ndim,
                    const int64_t *dims, int32_t max_iterations, int32_t *new_rank, int32_t *new_inverse,
                    float *g, lts_pass_report_t *rep, lts_regions_view_t *view, void *ws, size_t ws_bytes,
                    void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  if (kind != 0 && kind != 1) return lts_set_error(LTS_E_INVALID, "kind must be 0 (maxima) or 1 (minima)");
  if (max_iterations < 1) max_iterations = 100;
  return run_pass(c, kind, rank, inverse, pmark, max_iterations, new_rank, new_inverse, g, rep, view);
}

static int simplify_impl(Ctx &c, const float *f, const int64_t *pres_max, int64_t n_max, const int64_t *pres_min,
                         int64_t n_min, const int32_t *order, float *g, int32_t *G, lts_report_t *rep,
                         const lts_options_t *opt, void *ws) {
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  if ((f == nullptr) != (g == nullptr)) return lts_set_error(LTS_E_INVALID, "f and g go together");
  if (!f && !order) return lts_set_error(LTS_E_INVALID, "f is required unless an order field is given");
  lts_options_t o{};
  o.max_iterations = 100;
  o.restore_interior_extrema = 1;
  if (opt) o = *opt;
  if (o.max_iterations < 1) o.max_iterations = 100;
  c.timing = o.collect_timing != 0;
  lts_report_t R{};
  WS &w = c.w;
  const int64_t n = c.n;
  cudaStream_t s = c.s;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (c.timing) {
    t0 = next_event();
    cudaEventRecord(t0, s);
  }
  // A1/A2: order field F
  if (order) {
    LTS_TRY(install_order(c, f, order));
  } else {
    LTS_TRY(order_field_impl(c, f, w.rankA, w.invA, true));
  }
  // preserve marks and validation
  LTS_CUDA(cudaMemsetAsync(w.pmark, 0, (size_t)n, s));
  LTS_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(int) * SC_N, s));
  if (n_max > 0) k_set_pmark<<<NB(n_max), 256, 0, s>>>(pres_max, n_max, n, PM_MAX, w.pmark, w.scal + SC_BADPRES);
  else k_set_global<<<1, 32, 0, s>>>(w.invA, n, 1, w.pmark);
  if (n_min > 0) k_set_pmark<<<NB(n_min), 256, 0, s>>>(pres_min, n_min, n, PM_MIN, w.pmark, w.scal + SC_BADPRES);
  else k_set_global<<<1, 32, 0, s>>>(w.invA, n, 0, w.pmark);
  {
    // extrema of F; the ascent pointers are the first maxima pass's input
    Phase ph(c, LTS_PH_CLASSIFY);
    classify_any(c, w.rankA, w.flags, nullptr, nullptr, c.lut, w.ptr, PTR_ASC, s);
  }
  k_check_pres<<<NB(n), 256, 0, s>>>(w.flags, w.pmark, n, w.scal + SC_BADPRES);
  if (g) k_copy_canon<<<NB(n), 256, 0, s>>>(f, g, n);
  g_launches += g ? 4 : 3;
  LTS_KCHECK();
  // one readback: the order field's finiteness flag and the preserve check
  c.h_scal[SC_TMP] = 0;
  if (!order) LTS_CUDA(cudaMemcpyAsync(c.h_scal + SC_TMP, w.sb.nonfinite, sizeof(int), cudaMemcpyDeviceToHost, s));
  LTS_TRY(readback(c, SC_BADPRES, 1));
  if (c.h_scal[SC_TMP]) return lts_set_error(LTS_E_FIELD_NONFINITE, "scalar field contains NaN or infinite values");
  if (c.h_scal[SC_BADPRES]) return lts_set_error(LTS_E_CONSTRAINT_NOT_EXTREMUM, "a preserved vertex is not an extremum of the input order (ConstraintNotExtremum)");

  int *cr = w.rankA, *ci = w.invA, *nr = w.rankB, *ni = w.invB;
  bool ok = false;
  int it = 0;
  LTS_CUDA(cudaMemsetAsync(w.pstats, 0, sizeof(int) * (4 * LTS_MAX_REPORT_PASSES + 4), s));
  for (it = 1; it <= o.max_iterations; it++) {
    for (int kind = 0; kind < 2; kind++) {
      lts_pass_report_t pr{};
      const int slot = std::min(R.n_passes, LTS_MAX_REPORT_PASSES);  // the last slot collects the overflow
      LTS_TRY(run_pass(c, kind, cr, ci, w.pmark, o.max_iterations, nr, ni, g, &pr, nullptr,
                       it == 1 && kind == 0, w.pstats + 4 * slot));
      if (R.n_passes < LTS_MAX_REPORT_PASSES) R.passes[R.n_passes++] = pr;
      if (o.region_ni_out && pr.regions > 0) {  // per-region N_I
        const int64_t room = o.region_ni_capacity - R.region_ni_count;
        const int64_t cnt = std::min<int64_t>(room, pr.regions);
        if (cnt > 0)
          LTS_CUDA(cudaMemcpyAsync(o.region_ni_out + R.region_ni_count, w.nit, sizeof(int) * cnt,
                                   cudaMemcpyDeviceToDevice, s));
        R.region_ni_count += pr.regions;
      }
      std::swap(cr, nr);
      std::swap(ci, ni);
    }
    // restore (D6) and verify
    Phase ph(c, LTS_PH_VERIFY);
    classify_any(c, cr, w.flags, nullptr, nullptr, c.lut, nullptr, PTR_NONE, s);
    LTS_CUDA(cudaMemsetAsync(w.scal + SC_VERIFY, 0, sizeof(int) * 4, s));
    k_verify<<<NB(n), 256, 0, s>>>(w.flags, w.pmark, n, w.scal + SC_VERIFY);
    g_launches++;
    LTS_KCHECK();
    LTS_TRY(readback(c, SC_VERIFY, 4));
    int lost = c.h_scal[SC_VERIFY + 1] + c.h_scal[SC_VERIFY + 3];
    if (lost && o.restore_interior_extrema) {
      for (int kind = 0; kind < 2; kind++) {  // minima first, then maxima
        LTS_CUDA(cudaMemsetAsync(w.scal + SC_LOST, 0, sizeof(int), s));
        k_lost<<<NB(n), 256, 0, s>>>(w.flags, w.pmark, n, kind, w.lost, w.scal + SC_LOST);
        g_launches++;
        LTS_TRY(readback(c, SC_LOST, 1));
        int nl = c.h_scal[SC_LOST];
        if (!nl) continue;
        std::vector<int> ids(nl);
        LTS_CUDA(cudaMemcpyAsync(ids.data(), w.lost, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
        LTS_CUDA(cudaStreamSynchronize(s));
        std::sort(ids.begin(), ids.end());
        for (int x : ids) {
          if (c.g.ndim == 0) k_restore_target<0><<<1, 32, 0, s>>>(c.g, cr, x, kind, w.scal + SC_RESTORE);
          else if (c.g.ndim == 2) k_restore_target<2><<<1, 32, 0, s>>>(c.g, cr, x, kind, w.scal + SC_RESTORE);
          else k_restore_target<3><<<1, 32, 0, s>>>(c.g, cr, x, kind, w.scal + SC_RESTORE);
          k_restore_shift<<<NB(n), 256, 0, s>>>(cr, n, x, kind, w.scal + SC_RESTORE);
          g_launches += 2;
        }
        R.restored += nl;
      }
      k_scatter_inverse<<<NB(n), 256, 0, s>>>(cr, ci, n);
      classify_any(c, cr, w.flags, nullptr, nullptr, c.lut, nullptr, PTR_NONE, s);
      LTS_CUDA(cudaMemsetAsync(w.scal + SC_VERIFY, 0, sizeof(int) * 4, s));
      k_verify<<<NB(n), 256, 0, s>>>(w.flags, w.pmark, n, w.scal + SC_VERIFY);
      g_launches += 2;
      LTS_KCHECK();
      LTS_TRY(readback(c, SC_VERIFY, 4));
    }
    R.extra_max = c.h_scal[SC_VERIFY];
    R.lost_max = c.h_scal[SC_VERIFY + 1];
    R.extra_min = c.h_scal[SC_VERIFY + 2];
    R.lost_min = c.h_scal[SC_VERIFY + 3];
    if (R.extra_max == 0 && R.lost_max == 0 && R.extra_min == 0 && R.lost_min == 0) {
      ok = true;
      break;
    }
  }
  if (it > o.max_iterations) it = o.max_iterations;
  if (c.G_host) {
    LTS_CUDA(cudaMemcpyAsync(c.G_host, cr, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    if (!c.g_copy_valid) LTS_CUDA(cudaMemcpyAsync(c.g_host, g, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    if (c.g_copy_pending) LTS_CUDA(cudaStreamWaitEvent(s, g_cur->g_copied, 0));
  } else {
    LTS_CUDA(cudaMemcpyAsync(G, cr, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  }
  R.ok = ok ? 1 : 0;
  R.outer_iterations = it;
  if (c.timing) {
    t1 = next_event();
    cudaEventRecord(t1, s);
  }
  std::vector<int> pst(4 * LTS_MAX_REPORT_PASSES + 4);
  LTS_CUDA(cudaMemcpyAsync(pst.data(), w.pstats, sizeof(int) * pst.size(), cudaMemcpyDeviceToHost, s));
  LTS_CUDA(cudaStreamSynchronize(s));
  bool status1 = false;
  for (int i = 0; i < R.n_passes; i++) {
    if (R.passes[i].regions == 0) continue;
    const int *q = pst.data() + 4 * i;
    R.passes[i].n_iter_max = q[0];
    R.passes[i].capped = q[1];
    R.passes[i].largest = q[3];
    status1 |= q[2] != 0;
  }
  if (status1) return lts_set_error(LTS_E_LOCALIZE_NO_MIN, "region without an admissible boundary minimum (status 1)");
  if (c.timing) {
    for (auto &m : c.marks) {
      float ms = 0;
      cudaEventElapsedTime(&ms, m.second.first, m.second.second);
      if (m.first >= 0 && m.first < LTS_NUM_PHASES) R.phase_ms[m.first] += ms;
    }
    float tot = 0;
    cudaEventElapsedTime(&tot, t0, t1);
    R.phase_ms[LTS_PH_TOTAL] = tot;
    R.phase_ms[LTS_PH_FLOOD_LAUNCHES] = (double)c.flood_launches;
    R.phase_ms[LTS_PH_FLOOD_SLOTS] = (double)c.flood_slots;
  }
  if (rep) *rep = R;
  if (!ok) return lts_set_error(LTS_E_VERIFY_FAILED_AT_CAP, "verify_constraints still failing after maxIterations outer iterations");
  return 0;
}

int lts_simplify(const float *f, int ndim, const int64_t *dims, const int64_t *pres_max, int64_t n_max,
                 const int64_t *pres_min, int64_t n_min, const int32_t *order, float *g, int32_t *G,
                 lts_report_t *rep, const lts_options_t *opt, void *ws, size_t ws_bytes, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  return simplify_impl(c, f, pres_max, n_max, pres_min, n_min, order, g, G, rep, opt, ws);
}

// Host-buffer form: the caller's arrays live in (pinned) host memory, as the
// reference's numpy arrays do.  `dev` is device scratch for f, g and the
// preserve lists; g leaves for the host while the last pass still floods.
static size_t host_scratch_layout(int64_t n, int64_t n_max, int64_t n_min, size_t *of, size_t *og, size_t *opm,
                                  size_t *opn) {
  size_t off = 0;
  auto take = [&](size_t b) {
    off = (off + 255) & ~(size_t)255;
    const size_t at = off;
    off += b;
    return at;
  };
  *of = take(sizeof(float) * (size_t)n);
  *og = take(sizeof(float) * (size_t)n);
  *opm = take(sizeof(int64_t) * (size_t)std::max<int64_t>(n_max, 1));
  *opn = take(sizeof(int64_t) * (size_t)std::max<int64_t>(n_min, 1));
  return off + 256;
}

int lts_host_scratch_size(int ndim, const int64_t *dims, int64_t n_max, int64_t n_min, size_t *bytes) {
  if (!dims || !bytes || n_max < 0 || n_min < 0) return lts_set_error(LTS_E_INVALID, "null argument");
  int64_t n = 1;
  for (int a = 0; a < ndim; a++) n *= dims[a];
  size_t a, b, c2, d;
  *bytes = host_scratch_layout(n, n_max, n_min, &a, &b, &c2, &d);
  return 0;
}

int lts_simplify_host(const float *f_host, int ndim, const int64_t *dims, const int64_t *pres_max_host, int64_t n_max,
                      const int64_t *pres_min_host, int64_t n_min, float *g_host, int32_t *G_host,
                      lts_report_t *rep, const lts_options_t *opt, void *dev, size_t dev_bytes, void *ws,
                      size_t ws_bytes, void *stream) {
  LTS_LOCK;
  if (!f_host || !g_host || !G_host || !dev) return lts_set_error(LTS_E_INVALID, "null argument");
  if (n_max < 0 || n_min < 0 || (n_max && !pres_max_host) || (n_min && !pres_min_host))
    return lts_set_error(LTS_E_INVALID, "bad preserve lists");
  Ctx c;
  LTS_TRY(setup(c, ndim, dims, ws, ws_bytes, stream));
  size_t of, og, opm, opn;
  if (host_scratch_layout(c.n, n_max, n_min, &of, &og, &opm, &opn) > dev_bytes)
    return lts_set_error(LTS_E_WORKSPACE, "device scratch too small (lts_host_scratch_size)");
  char *base = (char *)(((uintptr_t)dev + 255) & ~(uintptr_t)255);
  float *f_d = (float *)(base + of), *g_d = (float *)(base + og);
  int64_t *pm_d = (int64_t *)(base + opm), *pn_d = (int64_t *)(base + opn);
  DevState &d = *g_cur;
  if (!d.copys) {
    LTS_CUDA(cudaStreamCreateWithFlags(&d.copys, cudaStreamNonBlocking));
    LTS_CUDA(cudaEventCreateWithFlags(&d.g_ready, cudaEventDisableTiming));
    LTS_CUDA(cudaEventCreateWithFlags(&d.g_copied, cudaEventDisableTiming));
  }
  cudaStream_t s = c.s;
  LTS_CUDA(cudaMemcpyAsync(f_d, f_host, sizeof(float) * (size_t)c.n, cudaMemcpyHostToDevice, s));
  if (n_max) LTS_CUDA(cudaMemcpyAsync(pm_d, pres_max_host, sizeof(int64_t) * (size_t)n_max, cudaMemcpyHostToDevice, s));
  if (n_min) LTS_CUDA(cudaMemcpyAsync(pn_d, pres_min_host, sizeof(int64_t) * (size_t)n_min, cudaMemcpyHostToDevice, s));
  c.g_host = g_host;
  c.G_host = G_host;
  return simplify_impl(c, f_d, pm_d, n_max, pn_d, n_min, nullptr, g_d, nullptr, rep, opt, ws);
}

// ---------------------------------------------------------------------------
// explicit triangle meshes: the same pass over a CSR mesh
// ---------------------------------------------------------------------------
int lts_workspace_size_csr(int64_t n, size_t *bytes) {
  if (n < 1 || n > ((int64_t)1 << 30)) return lts_set_error(LTS_E_BAD_DIMS, "mesh needs 1 <= n <= 2^30 vertices");
  WS w;
  *bytes = (size_t)carve(&w, nullptr, 0, n) + 256;
  return 0;
}

int lts_classify_csr(const int32_t *rank, int64_t n, const int32_t *indptr, const int32_t *indices,
                     const int32_t *link_ptr, const int32_t *link_a, const int32_t *link_b, uint8_t *flags,
                     int16_t *lower, int16_t *upper, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup_csr(c, n, indptr, indices, nullptr, 0, stream));
  if ((lower == nullptr) != (upper == nullptr)) return lts_set_error(LTS_E_INVALID, "lower and upper go together");
  if (lower && !(link_ptr && link_a && link_b))
    return lts_set_error(LTS_E_INVALID, "link_ptr / link_a / link_b are required for the component counts");
  c.lptr = link_ptr;
  c.la = link_a;
  c.lb = link_b;
  classify_any(c, rank, flags, lower, upper, nullptr, nullptr, PTR_NONE, c.s);
  LTS_KCHECK();
  return 0;
}

int lts_remove_pass_csr(int kind, const int32_t *rank, const int32_t *inverse, const uint8_t *pmark, int64_t n,
                        const int32_t *indptr, const int32_t *indices, int32_t max_iterations, int32_t *new_rank,
                        int32_t *new_inverse, float *g, lts_pass_report_t *rep, lts_regions_view_t *view, void *ws,
                        size_t ws_bytes, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup_csr(c, n, indptr, indices, ws, ws_bytes, stream));
  if (!ws) return lts_set_error(LTS_E_WORKSPACE, "workspace required");
  if (kind != 0 && kind != 1) return lts_set_error(LTS_E_INVALID, "kind must be 0 (maxima) or 1 (minima)");
  if (max_iterations < 1) max_iterations = 100;
  return run_pass(c, kind, rank, inverse, pmark, max_iterations, new_rank, new_inverse, g, rep, view);
}

int lts_simplify_csr(const float *f, int64_t n, const int32_t *indptr, const int32_t *indices,
                     const int64_t *pres_max, int64_t n_max, const int64_t *pres_min, int64_t n_min,
                     const int32_t *order, float *g, int32_t *G, lts_report_t *rep, const lts_options_t *opt,
                     void *ws, size_t ws_bytes, void *stream) {
  LTS_LOCK;
  Ctx c;
  LTS_TRY(setup_csr(c, n, indptr, indices, ws, ws_bytes, stream));
  return simplify_impl(c, f, pres_max, n_max, pres_min, n_min, order, g, G, rep, opt, ws);
}

}  // extern "C"
