// api.cu - the C ABI of libsten.so (include/sten.h): operator setup, workspace,
// TMA descriptors, the BiCGStab driver (CUDA graphs of whole iterations), the
// z-slab halo exchange and the fp32 scalar all-reduce (NCCL over NVLink).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "sten_internal.cuh"

using namespace sten;

// ------------------------------------------------------------ errors --
static thread_local std::string g_err;
static int set_err(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return set_err(STEN_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
  } while (0)
#define RC_TRY(expr)                 \
  do {                               \
    int rc_ = (expr);                \
    if (rc_ != STEN_OK) return rc_;  \
  } while (0)
#define KLAUNCH(expr)                                                                              \
  do {                                                                                             \
    int e_ = (expr);                                                                               \
    if (e_ != 0)                                                                                   \
      return set_err(STEN_ECUDA, "%s:%d launch %s: %s", __FILE__, __LINE__, #expr,                \
                     cudaGetErrorString((cudaError_t)e_));                                         \
  } while (0)

// ------------------------------------------------------------- NCCL --
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;
static int nccl_load() {
  if (g_nccl.h) return STEN_OK;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_err(STEN_ENCCL, "cannot dlopen libnccl.so.2: %s", dlerror());
#define SYM(field, name)                                                               \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));             \
  if (!g_nccl.field) return set_err(STEN_ENCCL, "libnccl.so.2 lacks %s", name);
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(AllReduce, "ncclAllReduce");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g_nccl.h = h;
  return STEN_OK;
}
#define NCCL_TRY(expr)                                                                          \
  do {                                                                                          \
    ncclResult_t r_ = (expr);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      return set_err(STEN_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr, g_nccl.GetErrorString(r_)); \
  } while (0)

struct sten_comm {
  ncclComm_t comm = nullptr;  // NULL: peer-memory-only communicator (no NCCL)
  int nranks = 1, rank = 0, device = 0;
};

// -------------------------------------------------- tensor-map encoding --
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;
static int load_encode() {
  if (g_encode) return STEN_OK;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return set_err(STEN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  return STEN_OK;
}
// 3D map over an array of `planes` planes of (ny rows x pitch elements, `pstride`
// elements apart), logical width nx; `promo` = L2 promotion (0 none, 1 64 B, 2 128 B, 3 256 B).
static int make_map_p(CUtensorMap *m, void *base, int elem, int nx, int ny, int planes, int pitch, long long pstride,
                      int promo, int boxx, int boxy) {
  RC_TRY(load_encode());
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * elem, (cuuint64_t)pstride * elem};
  cuuint32_t box[3] = {(cuuint32_t)boxx, (cuuint32_t)boxy, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  CUresult r = g_encode(m, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base,
                        dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        pr[promo & 3], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(STEN_ECUDA, "cuTensorMapEncodeTiled failed (%d): dims %d %d %d box %d %d", (int)r, nx, ny, planes,
                   boxx, boxy);
  return STEN_OK;
}

// ------------------------------------------------------------ handle --
struct Tiling {
  int rows = 0;  // 1: full-row strips (k_rows), 0: BX-wide tiles with an x halo (k_stencil)
  int bx = 0, by = 0, zc = 0, stages = 0, threads = 0;
  int cstages = 0;  // > 0: coefficient (+ rhat) tiles by TMA into a ring of this depth (k_stencil)
  int zc2 = 0;      // z chunk of H2 (0: zc; H1 and the apply use zc)
};
static int zc_of(const Tiling &t, int mode) { return mode == MODE_H2 && t.zc2 > 0 ? t.zc2 : t.zc; }

// SR schedule buffers (R19): two halo planes per side, because the
// sweep's y' = A(A p') reaches two planes into the z-neighbour's data.
constexpr int kSrHalo = 2;
struct SrBufs {
  bool ready = false, maps_ok = false;
  void *x = nullptr, *rh = nullptr;
  void *vec[2][5] = {};           // ping-pong sets of r, p, v, q, y
  CUtensorMap m_vec[2][5], m_c[6], m_x, m_rh;
};

struct PrecBufs {
  bool ready = false;
  void *x = nullptr, *r = nullptr, *rh = nullptr, *p[2] = {nullptr, nullptr}, *v[2] = {nullptr, nullptr};
  void *s = nullptr, *t = nullptr, *bw = nullptr;
  // tensor maps (rebuilt when the tiling changes)
  bool maps_ok = false;
  CUtensorMap m_r, m_p[2], m_v[2], m_s, m_x, m_rh, m_c[6];
};

struct Slab {
  int nz = 0;                     // planes of this slab
  long long z_first = 0;          // first plane within this rank's part
  float *c32[6] = {};             // interior plane 0 (one halo plane below it: c32b)
  __half *c16[6] = {};
  float *c32b[6] = {};            // allocations: nz + 2 planes, halo planes 0 and nz+1
  __half *c16b[6] = {};
  double *aP = nullptr;
  int has_below = 0, has_above = 0;  // a z-neighbour slab (this rank or the next) exists
  PrecBufs pb[2];
  SrBufs sr[2];
};

struct GraphKey {
  int prec, chunk, timing, sched;
  bool operator<(const GraphKey &o) const {
    return std::tie(prec, chunk, timing, sched) < std::tie(o.prec, o.chunk, o.timing, o.sched);
  }
};
struct SrTiling {
  int by = 0, stages = 0, cstages = 0, zc = 0;
  int zc_tail = 0, tail = 0;  // the last `tail` planes in chunks of zc_tail (0: none)
  int pack = 16;              // bytes per thread vector (16, or 8: twice the threads per tile)
};
struct GraphRec {
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;
  std::vector<cudaEvent_t> ev;  // [chunk][3][2] when timing
};

struct sten_stencil {
  int nx = 0, ny = 0, nz = 0, pitch = 0;
  long long plane = 0;
  int nslabs = 1;
  std::vector<Slab> slabs;
  sten_comm *comm = nullptr;
  bool has_diag = false;
  int sm = 148;
  Tiling tiling[2];
  SrTiling srt[2];
  int schedule = STEN_SCHED_CLASSIC;
  DevState *st = nullptr;       // device
  DevState *st_host = nullptr;  // pinned mirror
  float *partials = nullptr;
  int partials_cap = 0;
  unsigned *counter = nullptr;
  float *slab_sums = nullptr;   // [nslabs * kMaxDots]
  float *red_total = nullptr;   // [kMaxDots] (NCCL path)
  double *hist = nullptr;
  float *ahist = nullptr, *whist = nullptr;
  int hist_cap = 0;
  cudaStream_t cap = nullptr;   // capture stream
  std::map<GraphKey, GraphRec> graphs;
  bool timing = false;
  int coef_pf = 0;              // L2 prefetch distance of coefficient tiles (STEN_OPT_COEF_PREFETCH)
  int tma_promo = 3;            // TMA L2 promotion of every tensor map (STEN_OPT_TMA_L2_PROMOTION)
  int ew_bps = 64;              // element-wise kernels: CTAs per SM (STEN_OPT_EW_CTAS_PER_SM)
  bool sr_light = true;         // SR, one slab: last sweep without its SpMVs (STEN_OPT_SR_LIGHT_LAST)
  bool cls_overlap = true;      // classic, decomposed: halo exchange overlapped with the interior (STEN_OPT_CLASSIC_OVERLAP)
  bool cls_fuse = false;        // classic, decomposed: fused peer-memory exchange + all-reduce (STEN_OPT_CLASSIC_FUSED)
  bool cls_const = true;        // constant operator: classic kernels with scalar couplings (STEN_OPT_CLASSIC_CONST)
  void (*barrier_fn)(void *) = nullptr;  // host lockstep of several ranks on ONE GPU (sten_set_host_barrier)
  void *barrier_ctx = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  sten_stats stats{};
  std::vector<float> iter_ms;   // [it][3] per-iteration phase ms of the last timed bicgstab_solve
  long long launches = 0;       // kernel launches (direct + graph nodes) of the current call
  void *stage = nullptr;        // contiguous device staging for pitched host copies
  size_t stage_bytes = 0;
  unsigned *ir_amax = nullptr;  // refinement: max|r| (float bits), sigma
  float *ir_sigma = nullptr;
  int sr_l2pf = 0;              // SR: L2 prefetch distance (STEN_OPT_SR_L2_PREFETCH)
  bool sr_overlap = true;       // SR, decomposed: halo exchange overlapped with the interior chunks
  bool sr_p2p = true;           // SR, decomposed: fused halo stores + peer-memory all-reduce (sten_set_sr_exchange)
  bool p2p_ranks = false;       // ... across ranks too (after sten_p2p_import: CUDA IPC peers)
  float *p2p_sums = nullptr;    // own inbox: [slots][kMaxDots]
  unsigned *p2p_flags = nullptr;  // [slots]
  unsigned *p2p_seq = nullptr;  // sweeps finalised so far (persistent sequence number)
  int p2p_slots = 0;
  std::vector<P2PBox> p2p_remote;           // other ranks' inboxes (IPC)
  void *p2p_lo[2][2][5] = {}, *p2p_hi[2][2][5] = {};  // [prec][set][vec]: the z-neighbour ranks' buffers (IPC)
  void *cls_lo[2][5] = {}, *cls_hi[2][5] = {};  // [prec][r, p0, p1, v0, v1]: classic buffers of the z-neighbour ranks (IPC)
  std::vector<void *> ipc_opened;
  std::map<std::string, void *> ipc_map;  // IPC handle bytes -> mapped pointer
  cudaStream_t side = nullptr;  // capture side stream (exchange + boundary chunks)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  float *partials2 = nullptr;   // reduction scratch of the concurrent interior launch
  int partials2_cap = 0;
  unsigned *counter2 = nullptr;
  bool cc = false;              // constant-coefficient operator (stencil_create_const)
  bool half_dots = false;       // mixed SR sweeps accumulate the sums in fp16 pencils (R22)
  double cscaled[6] = {};       // its couplings A_d / a_P (fp64)
  // bicgstab_solve_batch: copy stream, double-buffered dense staging of b / x
  cudaStream_t io = nullptr;
  void *bstage[2] = {}, *xstage[2] = {};
  size_t io_bytes = 0;
  cudaEvent_t ev_in[2] = {}, ev_used[2] = {}, ev_out[2] = {}, ev_dn[2] = {};
};

static bool decomposed(const sten_stencil *st) { return st->nslabs > 1 || st->comm != nullptr; }
// several ranks, no NCCL: only the fused SR path (CUDA IPC peer memory) moves data between them
static bool p2p_only(const sten_stencil *st) { return st->comm && st->comm->nranks > 1 && !st->comm->comm; }
static bool nccl_ranks(const sten_stencil *st) { return st->comm && st->comm->nranks > 1 && st->comm->comm; }
// tensor map over one of the handle's z-major arrays (planes st->plane elements apart)
static int make_map(const sten_stencil *st, CUtensorMap *m, void *base, int elem, int nx, int ny, int planes,
                    int pitch, int boxx, int boxy) {
  return make_map_p(m, base, elem, nx, ny, planes, pitch, st->plane, st->tma_promo, boxx, boxy);
}
static int esize(int prec) { return prec == STEN_FP32 ? 4 : 2; }

static int rows_thr(int prec, int nx, int by) {
  return prec == STEN_FP32 ? rows_threads<float>(nx, by) : rows_threads<__half>(nx, by);
}

// Default: 256-B-wide tiles x 16 rows, 4 TMA stages (2 CTAs/SM).  Measured on
// B200 at 600x595x1536 (profiles/): 102.9 Gpoint-iter/s vs
// 99.9 for the best full-row strip (by 2, 3 stages) - the strips need more
// CTAs in flight than their shared-memory footprint allows.  Strips remain
// selectable with sten_set_tiling(bx >= nx).
// z-chunk length for a small mesh: enough chunks that the grid fills ~2 waves of
// the SMs (a 32^3 mesh has 2 xy tiles; one chunk each would leave the GPU idle
// and the z-march latency-bound), never below 4 planes
static int small_mesh_zc(const sten_stencil *st, int bx, int by, int nzs, int zc, int ctas_per_sm, int zmin = 4) {
  const long long tiles = (long long)((st->nx + bx - 1) / bx) * ((st->ny + by - 1) / by);
  const long long want = 2LL * st->sm * ctas_per_sm;
  const long long chunks = (want + tiles - 1) / tiles;
  if (chunks <= 1) return zc;
  int z = (int)((nzs + chunks - 1) / chunks);
  if (z < zmin) z = zmin;
  return z < zc ? z : zc;
}

static void default_tiling(sten_stencil *st, int prec) {
  Tiling &t = st->tiling[prec];
  int nzs = st->slabs[0].nz;
  // z chunks (config 3, paired runs, tools/zc_sweep.sh): H1 1.94 ms at 16-24 planes vs 2.07 at 64
  // (2.15 at 128, 2.31 at 1536: neighbouring tiles march together for a shorter time, so fewer
  // of their shared halo rows miss L2); H2 1.63 ms at 40-48 planes vs 1.66 at 16-20
  // fp32 fields (planes twice the bytes): H1 4.05 ms at 32 planes vs 4.07-4.08 at 20 and 4.10-4.11 at 16
  // (tools/fp32_zc.sh); H2 3.39-3.40 at 40-48.  fp32 constant operator (scalar couplings,
  // tools/fp32c_zc.sh): H1 2.075 ms at 20 vs 2.30 at 32; H2 1.48 at 64 vs 1.54 at 32
  const bool f32 = prec == STEN_FP32;
  const int zc1 = f32 && !st->cc ? 32 : 20, zc2 = f32 && st->cc ? 64 : 40;
  t.zc = nzs < zc1 ? nzs : zc1;
  t.zc2 = nzs < zc2 ? nzs : zc2;
  t.rows = 0;
  t.bx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();
  t.by = 16;
  const int zs = small_mesh_zc(st, t.bx, t.by, nzs, 64, 2);
  if (zs < t.zc) t.zc = zs;
  if (zs < t.zc2) t.zc2 = zs;
  // coefficient (+ rhat) tiles by TMA, 2 input + 2 coefficient stages (2 CTAs/SM): H1 2.12 ms vs
  // 2.31 ms with per-thread coefficient loads, which straddle sectors on unpadded rows
  t.stages = 2;
  t.cstages = 2;
  t.threads = prec == STEN_FP32 ? stencil_threads<float>(t.by) : stencil_threads<__half>(t.by);
}

static int ensure_maps(sten_stencil *st, int prec) {
  const Tiling &t = st->tiling[prec];
  const int e = esize(prec);
  const int H = prec == STEN_FP32 ? 4 : 8;
  for (Slab &sl : st->slabs) {
    PrecBufs &b = sl.pb[prec];
    if (b.maps_ok) continue;
    const int planes = sl.nz + 2;
    const int hx = t.rows ? kRowBoxElems : t.bx + 2 * H, hy = t.by + 2;
    const int ix = t.rows ? kRowBoxElems : t.bx;  // interior box (coefficient / rhat prefetch)
    RC_TRY(make_map(st, &b.m_r, b.r, e, st->nx, st->ny, planes, st->pitch, hx, hy));
    for (int i = 0; i < 2; ++i) {
      RC_TRY(make_map(st, &b.m_p[i], b.p[i], e, st->nx, st->ny, planes, st->pitch, hx, hy));
      RC_TRY(make_map(st, &b.m_v[i], b.v[i], e, st->nx, st->ny, planes, st->pitch, hx, hy));
    }
    RC_TRY(make_map(st, &b.m_s, b.s, e, st->nx, st->ny, planes, st->pitch, hx, hy));
    RC_TRY(make_map(st, &b.m_x, b.x, e, st->nx, st->ny, planes, st->pitch, hx, hy));
    RC_TRY(make_map(st, &b.m_rh, b.rh, e, st->nx, st->ny, planes, st->pitch, ix, t.by));
    for (int d = 0; d < 6; ++d) {
      void *c = prec == STEN_FP32 ? (void *)sl.c32[d] : (void *)sl.c16[d];
      RC_TRY(make_map(st, &b.m_c[d], c, e, st->nx, st->ny, sl.nz, st->pitch, ix, t.by));
    }
    b.maps_ok = true;
  }
  return STEN_OK;
}

static void drop_graphs(sten_stencil *st);
static int ew_grid(sten_stencil *st, long long nvec);
static int ensure_bufs(sten_stencil *st, int prec) {
  const size_t vbytes = (size_t)st->plane * esize(prec);
  for (Slab &sl : st->slabs) {
    PrecBufs &b = sl.pb[prec];
    if (b.ready) continue;
    const size_t bytes = vbytes * (sl.nz + 2);
    void **all[] = {&b.x, &b.r, &b.rh, &b.p[0], &b.p[1], &b.v[0], &b.v[1], &b.s, &b.t, &b.bw};
    for (void **pp : all) {
      cudaError_t e = cudaMalloc(pp, bytes);
      if (e != cudaSuccess) return set_err(STEN_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
      CUDA_TRY(cudaMemset(*pp, 0, bytes));  // halo planes and row padding stay zero
    }
    b.ready = true;
    b.maps_ok = false;
  }
  if (st->tiling[prec].bx == 0) default_tiling(st, prec);
  RC_TRY(ensure_maps(st, prec));
  // partial-sum buffer: one slot per CTA of the largest grid of ANY reducing
  // kernel - stencil tiles and the element-wise kernels (checked at launch too)
  int need = 0;
  for (Slab &sl : st->slabs) {
    const Tiling &t = st->tiling[prec];
    const int zmin = t.zc2 > 0 && t.zc2 < t.zc ? t.zc2 : t.zc;
    int g = ((st->nx + t.bx - 1) / t.bx) * ((st->ny + t.by - 1) / t.by) * ((sl.nz + zmin - 1) / zmin);
    if (g > need) need = g;
    const int ge = ew_grid(st, (long long)st->plane * sl.nz / 4);  // vec = 4 gives the larger grid
    if (ge > need) need = ge;
  }
  if (need < st->sm * 16) need = st->sm * 16;
  if (need > st->partials_cap) {
    if (st->partials) cudaFree(st->partials);
    CUDA_TRY(cudaMalloc(&st->partials, (size_t)need * kMaxDots * sizeof(float)));
    st->partials_cap = need;
    drop_graphs(st);
  }
  if (decomposed(st) && st->partials2_cap < st->partials_cap) {  // concurrent interior launches
    if (st->partials2) cudaFree(st->partials2);
    CUDA_TRY(cudaMalloc(&st->partials2, (size_t)st->partials_cap * kMaxDots * sizeof(float)));
    st->partials2_cap = st->partials_cap;
    drop_graphs(st);
  }
  return STEN_OK;
}

// --------------------------------------------------------- launch helpers --
static Reduce make_red(sten_stencil *st, int slab) {
  Reduce r;
  r.partials = st->partials;
  r.counter = st->counter;
  r.slab_out = decomposed(st) ? st->slab_sums + slab * kMaxDots : nullptr;
  r.st = st->st;
  return r;
}

// fused exchange: the slab's sums go straight into every participant's inbox (slot = global slab)
static void fused_red(sten_stencil *st, int slab, Reduce &r) {
  const int ns = (int)st->slabs.size();
  r.slab_out = nullptr;
  r.p2p_slot = (st->comm ? st->comm->rank : 0) * ns + slab;
  r.p2p_nslots = st->p2p_slots;
  r.p2p_seq = st->p2p_seq;
  r.p2p[0] = P2PBox{st->p2p_sums, st->p2p_flags};
  r.p2p_n = 1;
  for (const P2PBox &b : st->p2p_remote) r.p2p[r.p2p_n++] = b;
}
// classic buffers in the IPC record order (r, p0, p1, v0, v1)
static void *cls_buf(PrecBufs &b, int i) {
  void *q[5] = {b.r, b.p[0], b.p[1], b.v[0], b.v[1]};
  return q[i];
}
// the lower / upper z-neighbour's halo plane of classic buffer i for slab `slab` (null: none)
static void *cls_peer(sten_stencil *st, int prec, int slab, int i, bool lower) {
  const size_t pb = (size_t)st->plane * esize(prec);
  const int ns = (int)st->slabs.size();
  Slab &sl = st->slabs[slab];
  if (lower) {
    if (slab > 0) {
      Slab &n = st->slabs[slab - 1];
      return (char *)cls_buf(n.pb[prec], i) + (size_t)(n.nz + 1) * pb;
    }
    return st->cls_lo[prec][i] ? (char *)st->cls_lo[prec][i] + (size_t)(sl.nz + 1) * pb : nullptr;  // equal slabs
  }
  if (slab + 1 < ns) return cls_buf(st->slabs[slab + 1].pb[prec], i);
  return st->cls_hi[prec][i];
}

// part: CLS_ALL planes [0, nz) of the slab; CLS_INTERIOR [1, nz-1) (no halo plane
// read), CLS_BOTTOM plane 0, CLS_TOP plane nz-1 (decomposed, overlapped exchange:
// each part deposits its sums in slot 3*slab + part - 1, CLS_INTERIOR with the
// second reduction scratch because it runs concurrently with the other two)
enum { CLS_ALL = 0, CLS_INTERIOR = 1, CLS_BOTTOM = 2, CLS_TOP = 3 };
static int launch_stencil(sten_stencil *st, int prec, int mode, int slab, int parity, cudaStream_t s,
                          int part = CLS_ALL, bool capture = false, bool fused = false) {
  Slab &sl = st->slabs[slab];
  PrecBufs &b = sl.pb[prec];
  const Tiling &t = st->tiling[prec];
  StencilArgs a;
  memset(&a, 0, sizeof a);
  const int cur = parity, nxt = parity ^ 1;
  if (mode == MODE_APPLY) {
    a.tm_in[0] = b.m_s;  // apply reads the s buffer
    a.out0 = b.t;
  } else if (mode == MODE_H1) {
    a.tm_in[0] = b.m_r;
    a.tm_in[1] = b.m_p[cur];
    a.tm_in[2] = b.m_v[cur];
    a.tm_aux = b.m_rh;
    a.aux = b.rh;
    a.out0 = b.v[nxt];
    a.out1 = b.p[nxt];
  } else {
    a.tm_in[0] = b.m_r;
    a.tm_in[1] = b.m_v[nxt];
    a.out0 = b.t;
    a.out1 = b.s;
  }
  for (int d = 0; d < 6; ++d) {
    a.tm_c[d] = b.m_c[d];
    a.cptr[d] = prec == STEN_FP32 ? (const void *)sl.c32[d] : (const void *)sl.c16[d];
  }
  a.g = Geom{st->nx, st->ny, sl.nz, st->pitch, st->plane};
  a.zc = (prec == STEN_MIXED && st->half_dots) ? t.zc : zc_of(t, mode);  // half dots: one plan for all phases
  a.zlo = part == CLS_INTERIOR ? 1 : (part == CLS_TOP ? sl.nz - 1 : 0);
  a.zhi = part == CLS_INTERIOR ? sl.nz - 1 : (part == CLS_BOTTOM ? 1 : sl.nz);
  if (part == CLS_BOTTOM || part == CLS_TOP) a.zc = 1;
  a.pf = st->coef_pf;
  a.tiles_x = t.rows ? 1 : (st->nx + t.bx - 1) / t.bx;
  a.tiles_y = (st->ny + t.by - 1) / t.by;
  if (a.zhi > a.zlo && (long long)a.tiles_x * a.tiles_y * ((a.zhi - a.zlo + a.zc - 1) / a.zc) > st->partials_cap)
    return set_err(STEN_ECUDA, "internal: stencil grid exceeds the partial-sum buffer");
  a.red = make_red(st, slab);
  if (capture) a.red.slab_out = st->slab_sums + slab * kMaxDots;  // raw sums (sten_classic_phase)
  if (part != CLS_ALL) {
    a.red.slab_out = st->slab_sums + (3 * slab + part - 1) * kMaxDots;
    if (part == CLS_INTERIOR) {
      a.red.partials = st->partials2;
      a.red.counter = st->counter2;
    }
  }
  if (fused) {
    fused_red(st, slab, a.red);
    if (mode == MODE_H1) {  // p', v' boundary planes into the neighbours' halo planes
      const int nxt = parity ^ 1;
      for (int i = 0; i < 2; ++i) {
        const int idx = i == 0 ? 3 + nxt : 1 + nxt;  // out0 = v[nxt], out1 = p[nxt]
        a.peer_lo[i] = cls_peer(st, prec, slab, idx, true);
        a.peer_hi[i] = cls_peer(st, prec, slab, idx, false);
      }
    }
  }
  if (a.zhi <= a.zlo) return STEN_OK;
  // constant operator (NEXT-4): the couplings as scalars, no coefficient tiles (17 instead of 29 passes
  // per iteration); the default tile geometry only - any other tiling reads the coefficient arrays
  if (st->cc && st->cls_const && !t.rows && t.by == 16 && t.stages == 2 && t.cstages == 2 &&
      !(prec == STEN_MIXED && st->half_dots && mode != MODE_APPLY)) {
    a.cc = 1;
    for (int d = 0; d < 6; ++d) {  // the same roundings as k_create_coeffs: fp64 quotient, RN once
      a.cf32[d] = (float)st->cscaled[d];
      __half_raw hr = __half(__double2half(st->cscaled[d]));
      a.cf16[d] = hr.x;
    }
  }
  if (prec == STEN_MIXED && st->half_dots && mode != MODE_APPLY) {  // half dots (R22, R28): one chunk plan
    if (t.rows || fused) return set_err(STEN_EUNSUPPORTED, "half dots: the tile kernels without the fused exchange");
    KLAUNCH(stencil_launch_half(mode, a, t.by, t.stages, t.cstages, s));
    st->launches++;
    return STEN_OK;
  }
  if (fused && mode == MODE_H1 && (a.peer_lo[0] || a.peer_hi[0])) {
    if (t.rows) return set_err(STEN_EUNSUPPORTED, "the fused classic exchange needs the tile kernels");
    if (prec == STEN_FP32) KLAUNCH(stencil_launch_fused<float>(a, t.by, t.stages, t.cstages, s));
    else KLAUNCH(stencil_launch_fused<__half>(a, t.by, t.stages, t.cstages, s));
    st->launches++;
    return STEN_OK;
  }
  if (t.rows) {
    if (prec == STEN_FP32) KLAUNCH(rows_launch<float>(mode, a, t.by, t.stages, s));
    else KLAUNCH(rows_launch<__half>(mode, a, t.by, t.stages, s));
  } else {
    if (prec == STEN_FP32) KLAUNCH(stencil_launch<float>(mode, a, t.by, t.stages, t.cstages, s));
    else KLAUNCH(stencil_launch<__half>(mode, a, t.by, t.stages, t.cstages, s));
  }
  st->launches++;
  return STEN_OK;
}

// Element-wise grid: 64 CTAs of 256 threads per SM (measured best for the H3
// stream, 1.33 -> 1.29 ms at 600x595x1536 vs 8/SM), capped by the work so a
// small mesh does not launch idle CTAs (STEN_OPT_EW_CTAS_PER_SM).
static int ew_grid(sten_stencil *st, long long nvec) {
  const int bps = st->ew_bps;
  long long need = (nvec + 511) / 512;  // two vectors per thread
  long long g = (long long)st->sm * bps;
  if (need < g) g = need;
  return (int)(g < 1 ? 1 : g);
}

static int launch_h3(sten_stencil *st, int prec, int slab, int parity, cudaStream_t s, bool fused = false) {
  Slab &sl = st->slabs[slab];
  PrecBufs &b = sl.pb[prec];
  const int e = esize(prec), vec = prec == STEN_FP32 ? 4 : 8;
  const size_t off = (size_t)st->plane * e;  // interior starts at plane 1
  auto in = [&](void *p) { return (const void *)((char *)p + off); };
  EwArgs a;
  memset(&a, 0, sizeof a);
  a.x = in(b.x);
  a.p = in(b.p[parity ^ 1]);
  a.s = in(b.s);
  a.t = in(b.t);
  a.rhat = in(b.rh);
  a.xo = (char *)b.x + off;
  a.ro = (char *)b.r + off;
  a.rows = (long long)st->ny * sl.nz;
  a.vpr = (st->nx + vec - 1) / vec;
  a.pitch = st->pitch;
  a.nvec = (long long)st->plane * sl.nz / vec;  // linear over whole planes (padding holds zeros)
  a.red = make_red(st, slab);
  if (fused) {  // r's boundary planes into the neighbours' halo planes, sums into the inboxes
    fused_red(st, slab, a.red);
    a.peer_lo_r = cls_peer(st, prec, slab, 0, true);
    a.peer_hi_r = cls_peer(st, prec, slab, 0, false);
    a.plane_elems = st->plane;
    a.nzp = sl.nz;
  }
  if (prec == STEN_MIXED && st->half_dots) {  // half dots (R28): H3 marches the H1 / H2 chunk plan
    const Tiling &t = st->tiling[prec];
    H3zArgs h;
    memset(&h, 0, sizeof h);
    h.x = a.x;
    h.p = a.p;
    h.s = a.s;
    h.t = a.t;
    h.rh = a.rhat;
    h.xo = a.xo;
    h.ro = a.ro;
    h.g = Geom{st->nx, st->ny, sl.nz, st->pitch, st->plane};
    h.zc = t.zc;
    h.tiles_x = (st->nx + t.bx - 1) / t.bx;
    h.tiles_y = (st->ny + t.by - 1) / t.by;
    h.red = a.red;
    if (h3z_half_grid(st->sm, h) > st->partials_cap)
      return set_err(STEN_ECUDA, "internal: H3 grid exceeds the partial-sum buffer");
    KLAUNCH(h3z_half_launch(h, t.by, s));
    st->launches++;
    return STEN_OK;
  }
  if (ew_grid(st, a.nvec) > st->partials_cap)
    return set_err(STEN_ECUDA, "internal: element-wise grid exceeds the partial-sum buffer");
  if (prec == STEN_FP32) KLAUNCH(h3_launch<float>(a, ew_grid(st, a.nvec), 256, s));
  else KLAUNCH(h3_launch<__half>(a, ew_grid(st, a.nvec), 256, s));
  st->launches++;
  return STEN_OK;
}

static int launch_init(sten_stencil *st, int prec, int slab, bool with_ax, cudaStream_t s, bool scale = true) {
  Slab &sl = st->slabs[slab];
  PrecBufs &b = sl.pb[prec];
  const int e = esize(prec), vec = prec == STEN_FP32 ? 4 : 8;
  const size_t off = (size_t)st->plane * e;
  EwArgs a;
  memset(&a, 0, sizeof a);
  a.bw = (char *)b.bw + off;
  a.aP = (scale && st->has_diag) ? sl.aP : nullptr;
  a.ax = with_ax ? (const void *)((char *)b.t + off) : nullptr;
  a.r = (char *)b.r + off;
  a.rh = (char *)b.rh + off;
  a.p0 = (char *)b.p[0] + off;
  a.v0 = (char *)b.v[0] + off;
  a.rows = (long long)st->ny * sl.nz;
  a.vpr = (st->nx + vec - 1) / vec;
  a.pitch = st->pitch;
  a.nvec = (long long)st->plane * sl.nz / vec;  // linear over whole planes (padding holds zeros)
  a.red = make_red(st, slab);
  if (ew_grid(st, a.nvec) > st->partials_cap)
    return set_err(STEN_ECUDA, "internal: element-wise grid exceeds the partial-sum buffer");
  if (prec == STEN_FP32) KLAUNCH(init_launch<float>(a, ew_grid(st, a.nvec), 256, s));
  else KLAUNCH(init_launch<__half>(a, ew_grid(st, a.nvec), 256, s));
  st->launches++;
  return STEN_OK;
}

// One halo plane to each z-neighbour, for the array selected by `pick`.
template <typename Pick>
static int exchange(sten_stencil *st, int prec, Pick pick, cudaStream_t s) {
  const size_t pb = (size_t)st->plane * esize(prec);
  const int ns = (int)st->slabs.size();
  for (int k = 0; k + 1 < ns; ++k) {  // local neighbours: device copies
    char *lo = (char *)pick(st->slabs[k].pb[prec]);
    char *hi = (char *)pick(st->slabs[k + 1].pb[prec]);
    const int nzl = st->slabs[k].nz;
    CUDA_TRY(cudaMemcpyAsync(hi, lo + (size_t)nzl * pb, pb, cudaMemcpyDeviceToDevice, s));        // top -> halo 0
    CUDA_TRY(cudaMemcpyAsync(lo + (size_t)(nzl + 1) * pb, hi + pb, pb, cudaMemcpyDeviceToDevice, s));  // bottom -> halo top
  }
  if (p2p_only(st) && st->p2p_ranks) {
    // peer memory (CUDA IPC): push this rank's boundary planes into the z-neighbour ranks' halo
    // planes; the caller's host barrier then orders them before any rank's stencil reads them
    const int R = st->comm->nranks, me = st->comm->rank;
    PrecBufs &bb = st->slabs[0].pb[prec], &tb = st->slabs[ns - 1].pb[prec];
    char *bot = (char *)pick(bb), *top = (char *)pick(tb);
    int idx = -1;
    const void *cand[5] = {bb.r, bb.p[0], bb.p[1], bb.v[0], bb.v[1]};
    for (int i = 0; i < 5; ++i)
      if (cand[i] == (void *)bot) idx = i;
    if (idx < 0) return set_err(STEN_EUNSUPPORTED, "internal: peer-memory exchange of an unexported buffer");
    const int nzt = st->slabs[ns - 1].nz;
    if (me > 0) {  // our bottom interior plane -> the lower rank's top halo plane
      if (!st->cls_lo[prec][idx]) return set_err(STEN_EUNSUPPORTED, "internal: classic peer buffers not imported");
      CUDA_TRY(cudaMemcpyAsync((char *)st->cls_lo[prec][idx] + (size_t)(nzt + 1) * pb, bot + pb, pb,
                               cudaMemcpyDeviceToDevice, s));
    }
    if (me + 1 < R) {  // our top interior plane -> the upper rank's bottom halo plane
      if (!st->cls_hi[prec][idx]) return set_err(STEN_EUNSUPPORTED, "internal: classic peer buffers not imported");
      CUDA_TRY(cudaMemcpyAsync((char *)st->cls_hi[prec][idx], top + (size_t)nzt * pb, pb, cudaMemcpyDeviceToDevice, s));
    }
    return STEN_OK;
  }
  if (nccl_ranks(st)) {
    const int R = st->comm->nranks, me = st->comm->rank;
    char *bot = (char *)pick(st->slabs[0].pb[prec]);
    char *top = (char *)pick(st->slabs[ns - 1].pb[prec]);
    const int nzt = st->slabs[ns - 1].nz;
    NCCL_TRY(g_nccl.GroupStart());
    if (me > 0) {
      NCCL_TRY(g_nccl.Send(bot + pb, pb, ncclUint8, me - 1, st->comm->comm, s));
      NCCL_TRY(g_nccl.Recv(bot, pb, ncclUint8, me - 1, st->comm->comm, s));
    }
    if (me + 1 < R) {
      NCCL_TRY(g_nccl.Send(top + (size_t)nzt * pb, pb, ncclUint8, me + 1, st->comm->comm, s));
      NCCL_TRY(g_nccl.Recv(top + (size_t)(nzt + 1) * pb, pb, ncclUint8, me + 1, st->comm->comm, s));
    }
    NCCL_TRY(g_nccl.GroupEnd());
  }
  return STEN_OK;
}

// Decomposed solve: slab sums -> (NCCL fp32 all-reduce) -> scalar step.
static int host_barrier(sten_stencil *st, cudaStream_t s);
// Host lockstep (sten_set_host_barrier): before a peer-memory all-reduce's
// waiting kernel, finish this rank's work and meet the other ranks, so that the
// waiting kernel finds every flag already set and never spins on a kernel of
// another process (several ranks on one GPU: such waits are not guaranteed to
// make progress).  Not allowed inside a graph capture.
static int host_barrier(sten_stencil *st, cudaStream_t s) {
  if (!st->barrier_fn || !p2p_only(st)) return STEN_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return set_err(STEN_ECUDA, "internal: host barrier inside a graph capture");
  CUDA_TRY(cudaStreamSynchronize(s));
  st->barrier_fn(st->barrier_ctx);
  return STEN_OK;
}

static int reduce_scalars(sten_stencil *st, int phase, cudaStream_t s, int nslots = 0) {
  if (!decomposed(st)) return STEN_OK;
  const int ns = nslots > 0 ? nslots : (int)st->slabs.size();
  if (p2p_only(st)) {  // peer-memory all-reduce: deposit this rank's slab sums, wait for every rank's
    if (phase == PH_SR || nslots > 0 || !st->p2p_ranks)
      return set_err(STEN_EUNSUPPORTED, "internal: peer-memory reduction of phase %d", phase);
    std::vector<P2PBox> boxes{P2PBox{st->p2p_sums, st->p2p_flags}};
    for (const P2PBox &b : st->p2p_remote) boxes.push_back(b);
    KLAUNCH(p2p_put_launch(st->slab_sums, ns, st->comm->rank * ns, st->p2p_slots, boxes.data(), (int)boxes.size(),
                           st->p2p_seq, s));
    RC_TRY(host_barrier(st, s));
    KLAUNCH(p2p_fin_launch(phase, P2PBox{st->p2p_sums, st->p2p_flags}, st->p2p_slots, st->p2p_seq, st->st, s));
    st->launches += 2;
    return STEN_OK;
  }
  if (nccl_ranks(st)) {
    KLAUNCH(slabsum_launch(st->slab_sums, ns, st->red_total, s));
    NCCL_TRY(g_nccl.AllReduce(st->red_total, st->red_total, kMaxDots, ncclFloat32, ncclSum, st->comm->comm, s));
    KLAUNCH(scalars_launch(phase, st->red_total, 1, st->st, s));
    st->launches += 2;
  } else {
    KLAUNCH(scalars_launch(phase, st->slab_sums, ns, st->st, s));
    st->launches += 1;
  }
  return STEN_OK;
}

// One BiCGStab iteration (Alg. 1 l.176-184); iteration parity selects the
// ping-pong p/v buffers.  evs: optional [3][2] events around H1, H2, H3.
// Decomposed and overlapped (north_star (4)): the interior planes [1, nz-1) of
// every slab on the solve's stream while a side stream exchanges the halo
// planes and then runs the two boundary planes; the three parts' sums meet in
// the phase's reduction.
template <typename Xchg>
static int overlapped_phase(sten_stencil *st, int prec, int mode, int parity, cudaStream_t s, Xchg xchg,
                            bool finalize = true) {
  const int ns = (int)st->slabs.size();
  CUDA_TRY(cudaEventRecord(st->ev_fork, s));
  CUDA_TRY(cudaStreamWaitEvent(st->side, st->ev_fork, 0));
  for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, mode, k, parity, s, CLS_INTERIOR));
  RC_TRY(xchg(st->side));
  for (int k = 0; k < ns; ++k) {
    RC_TRY(launch_stencil(st, prec, mode, k, parity, st->side, CLS_BOTTOM));
    RC_TRY(launch_stencil(st, prec, mode, k, parity, st->side, CLS_TOP));
  }
  CUDA_TRY(cudaEventRecord(st->ev_join, st->side));
  CUDA_TRY(cudaStreamWaitEvent(s, st->ev_join, 0));
  return finalize ? reduce_scalars(st, mode == MODE_H1 ? PH_H1 : PH_H2, s, 3 * ns) : STEN_OK;
}

// classic fused exchange (STEN_OPT_CLASSIC_FUSED): loopback slabs, 1-rank communicators, or
// ranks whose classic buffers were imported (sten_p2p_import)
static bool cls_fused(const sten_stencil *st) {
  if (!decomposed(st) || !st->cls_fuse) return false;
  return !st->comm || st->comm->nranks == 1 || st->p2p_ranks;
}
static bool cls_overlapped(const sten_stencil *st) {
  if (!decomposed(st) || !st->cls_overlap || p2p_only(st) || cls_fused(st)) return false;
  for (const Slab &sl : st->slabs)
    if (sl.nz < 3) return false;
  return true;
}

// peer all-reduce wait of a fused phase: (host lockstep: all ranks' deposits first) the 1-thread kernel
static int fused_fin(sten_stencil *st, int phase, cudaStream_t s) {
  RC_TRY(host_barrier(st, s));
  KLAUNCH(p2p_fin_launch(phase, P2PBox{st->p2p_sums, st->p2p_flags}, st->p2p_slots, st->p2p_seq, st->st, s));
  st->launches++;
  return STEN_OK;
}

static int enqueue_iteration(sten_stencil *st, int prec, int parity, cudaStream_t s, cudaEvent_t *evs) {
  const int ns = (int)st->slabs.size();
  const bool dec = decomposed(st);
  if (cls_fused(st)) {  // compute + collective in the phase kernels themselves (STEN_OPT_CLASSIC_FUSED)
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, MODE_H1, k, parity, s, CLS_ALL, false, true));
    RC_TRY(fused_fin(st, PH_H1, s));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[2], s, cudaEventRecordExternal));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, MODE_H2, k, parity, s, CLS_ALL, false, true));
    RC_TRY(fused_fin(st, PH_H2, s));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[3], s, cudaEventRecordExternal));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[4], s, cudaEventRecordExternal));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_h3(st, prec, k, parity, s, true));
    RC_TRY(fused_fin(st, PH_H3, s));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[5], s, cudaEventRecordExternal));
    return STEN_OK;
  }
  if (cls_overlapped(st)) {
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
    RC_TRY(overlapped_phase(st, prec, MODE_H1, parity, s, [&](cudaStream_t ss) {
      RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.r; }, ss));
      RC_TRY(exchange(st, prec, [parity](PrecBufs &b) { return b.p[parity]; }, ss));
      return exchange(st, prec, [parity](PrecBufs &b) { return b.v[parity]; }, ss);
    }));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[2], s, cudaEventRecordExternal));
    RC_TRY(overlapped_phase(st, prec, MODE_H2, parity, s, [&](cudaStream_t ss) {
      return exchange(st, prec, [parity](PrecBufs &b) { return b.v[parity ^ 1]; }, ss);
    }));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[3], s, cudaEventRecordExternal));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[4], s, cudaEventRecordExternal));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_h3(st, prec, k, parity, s));
    RC_TRY(reduce_scalars(st, PH_H3, s));
    if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[5], s, cudaEventRecordExternal));
    return STEN_OK;
  }
  // H1: halos of r (new from H3), p, v (new from the previous H1)
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
  if (dec) {
    RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.r; }, s));
    RC_TRY(exchange(st, prec, [parity](PrecBufs &b) { return b.p[parity]; }, s));
    RC_TRY(exchange(st, prec, [parity](PrecBufs &b) { return b.v[parity]; }, s));
    RC_TRY(host_barrier(st, s));  // peer memory: every rank's halo pushes have landed
  }
  for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, MODE_H1, k, parity, s));
  RC_TRY(reduce_scalars(st, PH_H1, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
  // H2: halo of the new v
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[2], s, cudaEventRecordExternal));
  if (dec) {
    RC_TRY(exchange(st, prec, [parity](PrecBufs &b) { return b.v[parity ^ 1]; }, s));
    RC_TRY(host_barrier(st, s));
  }
  for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, MODE_H2, k, parity, s));
  RC_TRY(reduce_scalars(st, PH_H2, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[3], s, cudaEventRecordExternal));
  // H3
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[4], s, cudaEventRecordExternal));
  for (int k = 0; k < ns; ++k) RC_TRY(launch_h3(st, prec, k, parity, s));
  RC_TRY(reduce_scalars(st, PH_H3, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[5], s, cudaEventRecordExternal));
  return STEN_OK;
}

// ============================================== SR schedule (R19) ==
// Coefficient halo planes: the z-neighbour slab's boundary plane of each of
// the 12 coefficient arrays (6 x fp32, 6 x fp16).  Device copies between the
// slabs of this rank, NCCL send/recv between ranks; once, at create.
static int fill_coef_halos(sten_stencil *st, cudaStream_t s) {
  const int ns = (int)st->slabs.size();
  for (int pr = 0; pr < 2; ++pr) {
    const size_t pb = (size_t)st->plane * (pr == 0 ? 4 : 2);
    auto base = [&](Slab &sl, int d) -> char * { return pr == 0 ? (char *)sl.c32b[d] : (char *)sl.c16b[d]; };
    for (int k = 0; k + 1 < ns; ++k) {
      Slab &lo = st->slabs[k], &hi = st->slabs[k + 1];
      for (int d = 0; d < 6; ++d) {
        CUDA_TRY(cudaMemcpyAsync(base(hi, d), base(lo, d) + (size_t)lo.nz * pb, pb, cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(base(lo, d) + (size_t)(lo.nz + 1) * pb, base(hi, d) + pb, pb, cudaMemcpyDeviceToDevice, s));
      }
    }
    if (nccl_ranks(st)) {
      const int R = st->comm->nranks, me = st->comm->rank;
      Slab &bot = st->slabs[0], &top = st->slabs[ns - 1];
      NCCL_TRY(g_nccl.GroupStart());
      for (int d = 0; d < 6; ++d) {
        if (me > 0) {
          NCCL_TRY(g_nccl.Send(base(bot, d) + pb, pb, ncclUint8, me - 1, st->comm->comm, s));
          NCCL_TRY(g_nccl.Recv(base(bot, d), pb, ncclUint8, me - 1, st->comm->comm, s));
        }
        if (me + 1 < R) {
          NCCL_TRY(g_nccl.Send(base(top, d) + (size_t)top.nz * pb, pb, ncclUint8, me + 1, st->comm->comm, s));
          NCCL_TRY(g_nccl.Recv(base(top, d) + (size_t)(top.nz + 1) * pb, pb, ncclUint8, me + 1, st->comm->comm, s));
        }
      }
      NCCL_TRY(g_nccl.GroupEnd());
    }
  }
  return STEN_OK;
}

// Default SR geometry: 16-row tiles, 2 input stages, 2 coefficient stages (one
// 256-thread CTA per SM), 160-plane chunks with a 320-plane tail of 64-plane chunks.
static void default_sr_tiling(sten_stencil *st, int prec) {
  SrTiling &t = st->srt[prec];
  // measured at 600x595x1536: mixed 16-row tiles, 160-plane
  // chunks + 64-plane tail chunks; fp32 uniform 64-plane chunks (73.7 vs 70.2);
  // the constant-coefficient mixed sweep 8-row tiles with 3 input stages (192.7 vs 186.5)
  int by = 16, stg = 2, cst = 2, zc = 160, zct = 64, tail = 320, pack = 16;
  if (prec == STEN_FP32) {
    zc = 64;
    tail = 0;
  } else if (st->cc) {
    by = 8;
    stg = 3;
  }
  t.pack = pack;
  t.by = by;
  t.stages = stg;
  t.cstages = cst;
  const int nzs = st->slabs[0].nz;
  t.zc = zc < nzs ? zc : nzs;
  t.zc_tail = zct > 0 ? zct : t.zc;
  t.tail = tail > 0 ? tail : 0;
  const int bx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();
  // Small meshes: uniform short chunks.  HBM-bound ones: enough chunks to fill ~2 waves
  // (chunks down to 2 planes).  L2-resident ones (the sweep's ~15 arrays within 2x L2): at
  // most one wave, which balances the z-halo overhead of short chunks against parallelism
  // (config 2, 128^3 fp32, 16 tiles: 36 us per iteration at 15- or 16-plane chunks / 144 or 128
  // CTAs, 42 at 8 / 256, 51 at 32 / 64; config 1, 32^3: 2-plane chunks / 32 CTAs, 12 us).
  const long long tiles = (long long)((st->nx + bx - 1) / bx) * ((st->ny + t.by - 1) / t.by);
  const double ws = 15.0 * (double)st->nx * st->ny * nzs * esize(prec);
  int zs;
  if (ws <= 2.0 * 126e6) {
    const long long chunks = st->sm / tiles > 1 ? st->sm / tiles : 1;
    zs = (int)((nzs + chunks - 1) / chunks);
    if (zs < 2) zs = 2;
  } else {
    zs = small_mesh_zc(st, bx, t.by, nzs, t.zc, 1, 2);
  }
  if (zs < t.zc) {
    t.zc = t.zc_tail = zs;
    t.tail = 0;
  }
}

// chunk plan of a slab: nbig chunks of zc planes, then zc_tail-plane chunks to
// the end (the short chunks come last in launch order and even out the final
// wave; the long ones keep the per-chunk halo planes and pipeline fill rare)
static void sr_chunks(const SrTiling &t, int nzs, int *nbig, int *zct) {
  int big = nzs - (t.tail < nzs ? t.tail : 0);
  *nbig = big / t.zc;
  *zct = t.zc_tail;
  if (*nbig * t.zc == nzs) *zct = t.zc;  // no tail left
}

static int sr_grid(const sten_stencil *st, int prec, int nzs) {
  const SrTiling &t = st->srt[prec];
  const int bx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();
  int nbig, zct;
  sr_chunks(t, nzs, &nbig, &zct);
  const int nch = nbig + (nzs - nbig * t.zc + zct - 1) / zct;
  return ((st->nx + bx - 1) / bx) * ((st->ny + t.by - 1) / t.by) * nch;
}

static int ensure_sr(sten_stencil *st, int prec) {
  for (const Slab &sl : st->slabs)  // the two-plane halos come from the z-neighbour's own planes
    if (decomposed(st) && sl.nz < kSrHalo)
      return set_err(STEN_EINVAL, "the SR schedule needs >= %d planes per slab (slab of %d)", kSrHalo, sl.nz);
  if (st->srt[prec].by == 0) default_sr_tiling(st, prec);
  const SrTiling &t = st->srt[prec];
  if (!sr_config_ok(t.by, t.stages, t.cstages, t.pack) || t.zc <= 0)
    return set_err(STEN_EINVAL, "unsupported SR tiling by=%d stages=%d cstages=%d zc=%d pack=%d", t.by, t.stages,
                   t.cstages, t.zc, t.pack);
  if (prec == STEN_MIXED && st->half_dots) {  // R22: general operator, 16-B packs, no fused exchange
    if (st->cc) return set_err(STEN_EUNSUPPORTED, "half dots: not with the constant-coefficient operator");
    if (st->sr_p2p && decomposed(st))
      return set_err(STEN_EUNSUPPORTED, "half dots: not with the fused peer-memory exchange (STEN_XCHG_FUSED)");
    if (!sr_hd_config_ok(t.by, t.stages, t.cstages, t.pack))
      return set_err(STEN_EUNSUPPORTED, "half dots: SR tiling by=%d stages=%d cstages=%d pack=%d not built", t.by,
                     t.stages, t.cstages, t.pack);
  }
  const int e = esize(prec);
  const size_t vb = (size_t)st->plane * e;
  const int H = 16 / e, bx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();  // 16-B x halo pad
  for (Slab &sl : st->slabs) {
    SrBufs &b = sl.sr[prec];
    if (!b.ready) {
      const size_t bytes = vb * (sl.nz + 2 * kSrHalo);
      void **all[12] = {&b.x, &b.rh};
      int n = 2;
      for (int k = 0; k < 2; ++k)
        for (int i = 0; i < 5; ++i) all[n++] = &b.vec[k][i];
      for (void **pp : all) {
        cudaError_t ce = cudaMalloc(pp, bytes);
        if (ce != cudaSuccess) return set_err(STEN_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(ce));
        CUDA_TRY(cudaMemset(*pp, 0, bytes));  // halo planes and row padding stay zero
      }
      b.ready = true;
      b.maps_ok = false;
    }
    if (!b.maps_ok) {
      for (int k = 0; k < 2; ++k)
        for (int i = 0; i < 5; ++i)
#ifndef STEN_SR_DIAG
#define STEN_SR_DIAG 0
#endif
          RC_TRY(make_map(st, &b.m_vec[k][i], b.vec[k][i], e, st->nx, st->ny, sl.nz + 2 * kSrHalo, st->pitch,
                          bx + ((STEN_SR_DIAG & 1) ? 0 : 2 * H), t.by + ((STEN_SR_DIAG & 2) ? 0 : 4)));
      for (int d = 0; d < 6; ++d) {
        void *c = prec == STEN_FP32 ? (void *)sl.c32b[d] : (void *)sl.c16b[d];
        RC_TRY(make_map(st, &b.m_c[d], c, e, st->nx, st->ny, sl.nz + 2, st->pitch, bx + ((STEN_SR_DIAG & 4) ? 0 : 2 * H),
                        t.by + ((STEN_SR_DIAG & 4) ? 0 : 2)));
      }
      RC_TRY(make_map(st, &b.m_x, b.x, e, st->nx, st->ny, sl.nz + 2 * kSrHalo, st->pitch, bx, t.by));
      RC_TRY(make_map(st, &b.m_rh, b.rh, e, st->nx, st->ny, sl.nz + 2 * kSrHalo, st->pitch, bx, t.by));
      b.maps_ok = true;
    }
    const int g = sr_grid(st, prec, sl.nz);
    if (g > st->partials_cap) {
      if (st->partials) cudaFree(st->partials);
      CUDA_TRY(cudaMalloc(&st->partials, (size_t)g * kMaxDots * sizeof(float)));
      st->partials_cap = g;
      drop_graphs(st);
    }
    if (decomposed(st) && !st->partials2) {
      CUDA_TRY(cudaMalloc(&st->partials2, (size_t)st->partials_cap * kMaxDots * sizeof(float)));
      st->partials2_cap = st->partials_cap;
    }
    if (decomposed(st) && st->partials2_cap < st->partials_cap) {
      cudaFree(st->partials2);
      CUDA_TRY(cudaMalloc(&st->partials2, (size_t)st->partials_cap * kMaxDots * sizeof(float)));
      st->partials2_cap = st->partials_cap;
      drop_graphs(st);
    }
  }
  return STEN_OK;
}

static char *sr_interior(void *base, const sten_stencil *st, int prec) {
  return (char *)base + (size_t)kSrHalo * st->plane * esize(prec);
}

// one sweep of slab `slab`: reads set `set`, writes set `set ^ 1`.
// part: SR_ALL chunks, SR_INTERIOR (input planes all inside the slab: no halo
// needed) or SR_BOUNDARY (the rest).  capture: deposit the raw sums in
// slab_sums (slot 2*slab + (part == SR_INTERIOR)) instead of finalising.
enum { SR_ALL = 0, SR_INTERIOR = 1, SR_BOUNDARY = 2 };
// fused (peer-memory) halo + all-reduce path for decomposed SR sweeps
static bool sr_fused(const sten_stencil *st) {
  if (!decomposed(st) || !st->sr_p2p) return false;
  return !st->comm || st->comm->nranks == 1 || st->p2p_ranks;
}
static void sr_chunk_z(const SrTiling &t, int nbig, int zct, int c, int *z0) {
  *z0 = c < nbig ? c * t.zc : nbig * t.zc + (c - nbig) * zct;
}
static int launch_sr(sten_stencil *st, int prec, int slab, int set, bool capture, cudaStream_t s, int part = SR_ALL,
                     bool fused = false) {
  Slab &sl = st->slabs[slab];
  SrBufs &b = sl.sr[prec];
  const SrTiling &t = st->srt[prec];
  SrArgs a;
  memset(&a, 0, sizeof a);
  for (int i = 0; i < 5; ++i) {
    a.tm_in[i] = b.m_vec[set][i];
    a.out[i] = sr_interior(b.vec[set ^ 1][i], st, prec);
  }
  for (int d = 0; d < 6; ++d) a.tm_c[d] = b.m_c[d];
  a.tm_x = b.m_x;
  a.tm_rh = b.m_rh;
  a.x = sr_interior(b.x, st, prec);
  a.rh = sr_interior(b.rh, st, prec);
  a.g = Geom{st->nx, st->ny, sl.nz, st->pitch, st->plane};
  a.zc = t.zc;
  sr_chunks(t, sl.nz, &a.nbig, &a.zc_tail);
  const int ntot = a.nbig + (sl.nz - a.nbig * t.zc + a.zc_tail - 1) / a.zc_tail;
  // interior chunks: [clo, chi), those whose staged planes z0-2 .. z1+1 lie in the slab
  int clo = 0, chi = 0;
  for (int c = 0; c < ntot; ++c) {
    int z0c, z0n;
    sr_chunk_z(t, a.nbig, a.zc_tail, c, &z0c);
    sr_chunk_z(t, a.nbig, a.zc_tail, c + 1, &z0n);
    const bool in = z0c >= 2 && (z0n < sl.nz ? z0n : sl.nz) <= sl.nz - 2;
    if (in && chi == clo) clo = chi = c;
    if (in) chi = c + 1;
  }
  if (part == SR_ALL) { a.nch = ntot; a.ch_lo_n = 0; a.ch_hi0 = 0; }
  else if (part == SR_INTERIOR) { a.nch = chi - clo; a.ch_lo_n = 0; a.ch_hi0 = clo; }
  else { a.nch = ntot - (chi - clo); a.ch_lo_n = clo; a.ch_hi0 = chi; }
  const int bx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();
  a.tiles_x = (st->nx + bx - 1) / bx;
  a.tiles_y = (st->ny + t.by - 1) / t.by;
  if (sr_grid(st, prec, sl.nz) > st->partials_cap)
    return set_err(STEN_ECUDA, "internal: SR grid exceeds the partial-sum buffer");
  a.red = make_red(st, slab);
  if (capture) a.red.slab_out = st->slab_sums + slab * kMaxDots;
  if (part != SR_ALL) {
    a.red.slab_out = st->slab_sums + (2 * slab + (part == SR_INTERIOR)) * kMaxDots;
    if (part == SR_INTERIOR) {
      a.red.partials = st->partials2;
      a.red.counter = st->counter2;
    }
  }
  a.l2pf = st->sr_l2pf;
  if (fused) {
    // halo planes straight into the z-neighbours' next-set buffers ...
    const size_t pb = (size_t)st->plane * esize(prec);
    const int ns = (int)st->slabs.size();
    for (int i = 0; i < 5; ++i) {
      void *lo = nullptr, *hi = nullptr;
      if (slab > 0) {
        Slab &n = st->slabs[slab - 1];
        lo = (char *)n.sr[prec].vec[set ^ 1][i] + (size_t)(n.nz + kSrHalo) * pb;
      } else if (st->p2p_lo[prec][set ^ 1][i]) {
        lo = (char *)st->p2p_lo[prec][set ^ 1][i] + (size_t)(sl.nz + kSrHalo) * pb;  // equal slabs on every rank
      }
      if (slab + 1 < ns) hi = st->slabs[slab + 1].sr[prec].vec[set ^ 1][i];
      else if (st->p2p_hi[prec][set ^ 1][i]) hi = st->p2p_hi[prec][set ^ 1][i];
      a.peer_lo[i] = lo;
      a.peer_hi[i] = hi;
    }
    // ... and the sums into every participant's inbox, slot = global slab index
    a.red.slab_out = nullptr;
    a.red.p2p_slot = (st->comm ? st->comm->rank : 0) * ns + slab;
    a.red.p2p_nslots = st->p2p_slots;
    a.red.p2p_seq = st->p2p_seq;
    a.red.p2p[0] = P2PBox{st->p2p_sums, st->p2p_flags};
    a.red.p2p_n = 1;
    for (const P2PBox &b2 : st->p2p_remote) a.red.p2p[a.red.p2p_n++] = b2;
  }
  if (st->cc) {  // the same roundings as k_create_coeffs: fp64 quotient, RN to fp32 / fp16
    for (int d = 0; d < 6; ++d) {
      a.cf32[d] = (float)st->cscaled[d];
      __half_raw hr = __half(__double2half(st->cscaled[d]));
      a.cf16[d] = hr.x;
    }
    a.has_below = sl.has_below;
    a.has_above = sl.has_above;
  }
  if (a.nch == 0) return STEN_OK;
  if (prec == STEN_FP32) KLAUNCH(sr_launch<float>(a, t.by, t.stages, t.cstages, t.pack, st->cc, false, s));
  else KLAUNCH(sr_launch<__half>(a, t.by, t.stages, t.cstages, t.pack, st->cc, st->half_dots, s));
  st->launches++;
  return STEN_OK;
}

// two halo planes of r, p, v, q, y (set `set`) to each z-neighbour
static int sr_exchange(sten_stencil *st, int prec, int set, cudaStream_t s) {
  const size_t pb = (size_t)st->plane * esize(prec), hb = pb * kSrHalo;
  const int ns = (int)st->slabs.size();
  for (int i = 0; i < 5; ++i) {
    for (int k = 0; k + 1 < ns; ++k) {
      char *lo = (char *)st->slabs[k].sr[prec].vec[set][i];
      char *hi = (char *)st->slabs[k + 1].sr[prec].vec[set][i];
      const int nzl = st->slabs[k].nz;
      CUDA_TRY(cudaMemcpyAsync(hi, lo + (size_t)nzl * pb, hb, cudaMemcpyDeviceToDevice, s));  // top 2 -> low halo
      CUDA_TRY(cudaMemcpyAsync(lo + (size_t)(nzl + kSrHalo) * pb, hi + hb, hb, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (p2p_only(st)) {
    // no NCCL: PULL the z-neighbour ranks' boundary planes into our halo planes
    // through peer memory (their init, which wrote them, finished before the
    // init's peer-memory all-reduce completed; nothing writes them again before
    // our first sweep's sums have been deposited)
    if (!st->p2p_ranks) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: call sten_p2p_import first");
    const int R = st->comm->nranks, me = st->comm->rank;
    for (int i = 0; i < 5; ++i) {
      char *bot = (char *)st->slabs[0].sr[prec].vec[set][i];
      char *top = (char *)st->slabs[ns - 1].sr[prec].vec[set][i];
      const int nzt = st->slabs[ns - 1].nz;  // equal slabs on every rank
      if (me > 0)
        CUDA_TRY(cudaMemcpyAsync(bot, (char *)st->p2p_lo[prec][set][i] + (size_t)nzt * pb, hb, cudaMemcpyDefault, s));
      if (me + 1 < R)
        CUDA_TRY(cudaMemcpyAsync(top + (size_t)(nzt + kSrHalo) * pb, (char *)st->p2p_hi[prec][set][i] + hb, hb,
                                 cudaMemcpyDefault, s));
    }
  }
  if (nccl_ranks(st)) {
    const int R = st->comm->nranks, me = st->comm->rank;
    NCCL_TRY(g_nccl.GroupStart());
    for (int i = 0; i < 5; ++i) {
      char *bot = (char *)st->slabs[0].sr[prec].vec[set][i];
      char *top = (char *)st->slabs[ns - 1].sr[prec].vec[set][i];
      const int nzt = st->slabs[ns - 1].nz;
      if (me > 0) {
        NCCL_TRY(g_nccl.Send(bot + hb, hb, ncclUint8, me - 1, st->comm->comm, s));
        NCCL_TRY(g_nccl.Recv(bot, hb, ncclUint8, me - 1, st->comm->comm, s));
      }
      if (me + 1 < R) {
        NCCL_TRY(g_nccl.Send(top + (size_t)nzt * pb, hb, ncclUint8, me + 1, st->comm->comm, s));
        NCCL_TRY(g_nccl.Recv(top + (size_t)(nzt + kSrHalo) * pb, hb, ncclUint8, me + 1, st->comm->comm, s));
      }
    }
    NCCL_TRY(g_nccl.GroupEnd());
  }
  return STEN_OK;
}

// one SR iteration: halos of the input set, the sweep of every slab, the
// cross-slab / cross-rank scalar step.  evs: optional [2] events.
static int enqueue_sr_sweep(sten_stencil *st, int prec, int set, cudaStream_t s, cudaEvent_t *evs) {
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
  const int ns = (int)st->slabs.size();
  if (sr_fused(st)) {
    // one kernel per slab does the sweep, its halo exchange (stores into the
    // neighbours' buffers) and its share of the all-reduce (inbox deposits);
    // a 1-thread kernel waits for every slot and runs the scalar step
    for (int k = 0; k < ns; ++k) RC_TRY(launch_sr(st, prec, k, set, false, s, SR_ALL, true));
    RC_TRY(host_barrier(st, s));
    KLAUNCH(p2p_fin_launch(PH_SR, P2PBox{st->p2p_sums, st->p2p_flags}, st->p2p_slots, st->p2p_seq, st->st, s));
    st->launches++;
  } else if (decomposed(st) && st->sr_overlap) {
    // the halo exchange and the chunks that read halo planes on a side
    // stream, concurrent with the interior chunks (north_star: halos
    // "overlapped with interior compute"); both deposit slab sums
    CUDA_TRY(cudaMemsetAsync(st->slab_sums, 0, sizeof(float) * kMaxDots * 2 * ns, s));
    CUDA_TRY(cudaEventRecord(st->ev_fork, s));
    CUDA_TRY(cudaStreamWaitEvent(st->side, st->ev_fork, 0));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_sr(st, prec, k, set, false, s, SR_INTERIOR));
    RC_TRY(sr_exchange(st, prec, set, st->side));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_sr(st, prec, k, set, false, st->side, SR_BOUNDARY));
    CUDA_TRY(cudaEventRecord(st->ev_join, st->side));
    CUDA_TRY(cudaStreamWaitEvent(s, st->ev_join, 0));
    RC_TRY(reduce_scalars(st, PH_SR, s, 2 * ns));
  } else {
    if (decomposed(st)) RC_TRY(sr_exchange(st, prec, set, s));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_sr(st, prec, k, set, false, s));
    RC_TRY(reduce_scalars(st, PH_SR, s));
  }
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
  return STEN_OK;
}

static int get_graph(sten_stencil *st, int prec, int chunk, GraphRec **out) {
  GraphKey key{prec, chunk, st->timing ? 1 : 0, st->schedule};
  auto it = st->graphs.find(key);
  if (it != st->graphs.end()) {
    *out = &it->second;
    return STEN_OK;
  }
  GraphRec rec;
  if (st->timing) {
    rec.ev.resize((size_t)chunk * 6);
    for (auto &e : rec.ev) CUDA_TRY(cudaEventCreate(&e));
  }
  const long long l0 = st->launches;
  CUDA_TRY(cudaStreamBeginCapture(st->cap, cudaStreamCaptureModeThreadLocal));
  int rc = STEN_OK;
  for (int j = 0; j < chunk && rc == STEN_OK; ++j)
    rc = st->schedule == STEN_SCHED_SR
             ? enqueue_sr_sweep(st, prec, j & 1, st->cap, st->timing ? &rec.ev[(size_t)j * 6] : nullptr)
             : enqueue_iteration(st, prec, j & 1, st->cap, st->timing ? &rec.ev[(size_t)j * 6] : nullptr);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(st->cap, &g);
  if (rc != STEN_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess) return set_err(STEN_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&rec.exec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return set_err(STEN_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
  rec.kernels = st->launches - l0;
  st->launches = l0;
  auto ins = st->graphs.emplace(key, rec);
  *out = &ins.first->second;
  return STEN_OK;
}

static void drop_graphs(sten_stencil *st) {
  for (auto &kv : st->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    for (auto e : kv.second.ev) cudaEventDestroy(e);
  }
  st->graphs.clear();
}

// dense (nz,ny,nx) user array <-> internal array (rows of `pitch`, planes of
// `plane` elements, halo planes): one 3D copy per slab, a 1D copy when the
// internal layout has no padding at all.
static int ptr_on_device(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}
// Host <-> device copies of a pitched layout go through a contiguous device
// staging buffer: one full-speed linear PCIe transfer, then the pitched copy
// on the device (a pitched host transfer runs at a fraction of the link rate).
static cudaError_t stage_buffer(sten_stencil *st, size_t bytes, void **out) {
  if (bytes > st->stage_bytes) {
    if (st->stage) cudaFree(st->stage);
    st->stage = nullptr;
    st->stage_bytes = 0;
    cudaError_t e = cudaMalloc(&st->stage, bytes);
    if (e != cudaSuccess) return e;
    st->stage_bytes = bytes;
  }
  *out = st->stage;
  return cudaSuccess;
}
static cudaError_t copy3d(sten_stencil *st, void *dst, size_t dpitch, size_t dysize, const void *src, size_t spitch,
                          size_t sysize, size_t wbytes, size_t h, size_t d, cudaStream_t s) {
  if (dpitch == wbytes && spitch == wbytes && dysize == h && sysize == h)
    return cudaMemcpyAsync(dst, src, wbytes * h * d, cudaMemcpyDefault, s);
  const bool dev_src = ptr_on_device(src), dev_dst = ptr_on_device(dst);
  if (dev_src != dev_dst) {
    void *stg = nullptr;
    cudaError_t e = stage_buffer(st, wbytes * h * d, &stg);
    if (e != cudaSuccess) return e;
    if (!dev_src) {  // host (dense rows) -> staging -> pitched device
      e = cudaMemcpyAsync(stg, src, wbytes * h * d, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return e;
      return copy3d(st, dst, dpitch, dysize, stg, wbytes, h, wbytes, h, d, s);
    }
    e = copy3d(st, stg, wbytes, h, src, spitch, sysize, wbytes, h, d, s);  // pitched device -> staging
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(dst, stg, wbytes * h * d, cudaMemcpyDeviceToHost, s);
  }
  if (dev_src && dev_dst) {  // device <-> device: the row-copy stream (falls back for odd alignment)
    const int e = copy_rows_launch(dst, dpitch, dysize, src, spitch, sysize, wbytes, h, d, st->sm, s);
    if (e == (int)cudaSuccess) st->launches++;
    if (e != (int)cudaErrorNotSupported) return (cudaError_t)e;
  }
  cudaMemcpy3DParms p;
  memset(&p, 0, sizeof p);
  p.srcPtr = make_cudaPitchedPtr(const_cast<void *>(src), spitch, wbytes, sysize);
  p.dstPtr = make_cudaPitchedPtr(dst, dpitch, wbytes, dysize);
  p.extent = make_cudaExtent(wbytes, h, d);
  p.kind = cudaMemcpyDefault;
  return cudaMemcpy3DAsync(&p, s);
}
static int copy_in(sten_stencil *st, int prec, void *(*sel)(PrecBufs &), const void *src, cudaStream_t s) {
  const int e = esize(prec);
  for (Slab &sl : st->slabs) {
    char *dst = (char *)sel(sl.pb[prec]) + (size_t)st->plane * e;
    const char *sp = (const char *)src + (size_t)sl.z_first * st->nx * st->ny * e;
    CUDA_TRY(copy3d(st, dst, (size_t)st->pitch * e, (size_t)(st->plane / st->pitch), sp, (size_t)st->nx * e,
                    (size_t)st->ny, (size_t)st->nx * e, (size_t)st->ny, (size_t)sl.nz, s));
  }
  return STEN_OK;
}
static int copy_out(sten_stencil *st, int prec, void *(*sel)(PrecBufs &), void *dst, cudaStream_t s) {
  const int e = esize(prec);
  for (Slab &sl : st->slabs) {
    const char *src = (const char *)sel(sl.pb[prec]) + (size_t)st->plane * e;
    char *dp = (char *)dst + (size_t)sl.z_first * st->nx * st->ny * e;
    CUDA_TRY(copy3d(st, dp, (size_t)st->nx * e, (size_t)st->ny, src, (size_t)st->pitch * e,
                    (size_t)(st->plane / st->pitch), (size_t)st->nx * e, (size_t)st->ny, (size_t)sl.nz, s));
  }
  return STEN_OK;
}
// the same for SR buffers (kSrHalo halo planes); base(slab) -> allocation
template <typename Base>
static int sr_copy_in(sten_stencil *st, int prec, Base base, const void *src, cudaStream_t s) {
  const int e = esize(prec);
  for (Slab &sl : st->slabs) {
    char *dst = sr_interior(base(sl), st, prec);
    const char *sp = (const char *)src + (size_t)sl.z_first * st->nx * st->ny * e;
    CUDA_TRY(copy3d(st, dst, (size_t)st->pitch * e, (size_t)(st->plane / st->pitch), sp, (size_t)st->nx * e,
                    (size_t)st->ny, (size_t)st->nx * e, (size_t)st->ny, (size_t)sl.nz, s));
  }
  return STEN_OK;
}
template <typename Base>
static int sr_copy_out(sten_stencil *st, int prec, Base base, void *dst, cudaStream_t s) {
  const int e = esize(prec);
  for (Slab &sl : st->slabs) {
    const char *src = sr_interior(base(sl), st, prec);
    char *dp = (char *)dst + (size_t)sl.z_first * st->nx * st->ny * e;
    CUDA_TRY(copy3d(st, dp, (size_t)st->nx * e, (size_t)st->ny, src, (size_t)st->pitch * e,
                    (size_t)(st->plane / st->pitch), (size_t)st->nx * e, (size_t)st->ny, (size_t)sl.nz, s));
  }
  return STEN_OK;
}

// S1 for the SR schedule: b_hat, r0 = b_hat - A x0, rhat = p = r0, v = 0 into
// SR set 0 (k_init), q = y = 0.
static int launch_init_sr(sten_stencil *st, int prec, int slab, bool with_ax, cudaStream_t s, bool scale = true) {
  Slab &sl = st->slabs[slab];
  PrecBufs &b = sl.pb[prec];
  SrBufs &r = sl.sr[prec];
  const int e = esize(prec), vec = prec == STEN_FP32 ? 4 : 8;
  const size_t off = (size_t)st->plane * e;
  EwArgs a;
  memset(&a, 0, sizeof a);
  a.bw = (char *)b.bw + off;
  a.aP = (scale && st->has_diag) ? sl.aP : nullptr;
  a.ax = with_ax ? (const void *)((char *)b.t + off) : nullptr;
  a.r = sr_interior(r.vec[0][0], st, prec);
  a.rh = sr_interior(r.rh, st, prec);
  a.p0 = sr_interior(r.vec[0][1], st, prec);
  a.v0 = sr_interior(r.vec[0][2], st, prec);
  a.rows = (long long)st->ny * sl.nz;
  a.vpr = (st->nx + vec - 1) / vec;
  a.pitch = st->pitch;
  a.nvec = (long long)st->plane * sl.nz / vec;
  a.red = make_red(st, slab);
  if (ew_grid(st, a.nvec) > st->partials_cap)
    return set_err(STEN_ECUDA, "internal: element-wise grid exceeds the partial-sum buffer");
  const size_t all = (size_t)st->plane * e * (sl.nz + 2 * kSrHalo);
  CUDA_TRY(cudaMemsetAsync(r.vec[0][3], 0, all, s));
  CUDA_TRY(cudaMemsetAsync(r.vec[0][4], 0, all, s));
  if (prec == STEN_FP32) KLAUNCH(init_launch<float>(a, ew_grid(st, a.nvec), 256, s));
  else KLAUNCH(init_launch<__half>(a, ew_grid(st, a.nvec), 256, s));
  st->launches++;
  return STEN_OK;
}

static void *sel_x(PrecBufs &b) { return b.x; }
static void *sel_s(PrecBufs &b) { return b.s; }
static void *sel_t(PrecBufs &b) { return b.t; }
static void *sel_bw(PrecBufs &b) { return b.bw; }

// ============================================================== C ABI ==
extern "C" {

int sten_version(void) { return STEN_VERSION; }
const char *sten_last_error(void) { return g_err.c_str(); }

int sten_comm_unique_id(void *id_out) {
  if (!id_out) return set_err(STEN_EINVAL, "id_out is NULL");
  RC_TRY(nccl_load());
  ncclUniqueId id;
  NCCL_TRY(g_nccl.GetUniqueId(&id));
  memcpy(id_out, &id, sizeof id);
  return STEN_OK;
}

int sten_comm_create(const void *unique_id, int nranks, int rank, int cuda_device, sten_comm **out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_err(STEN_EINVAL, "bad comm arguments (nranks=%d rank=%d)", nranks, rank);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev)
    return set_err(STEN_EINVAL, "cuda_device %d not in 0..%d", cuda_device, ndev - 1);
  CUDA_TRY(cudaSetDevice(cuda_device));
  sten_comm *c = new sten_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  if (!unique_id) {  // peer-memory only: the data plane comes from sten_p2p_import
    *out = c;
    return STEN_OK;
  }
  int rc = nccl_load();
  if (rc != STEN_OK) {
    delete c;
    return rc;
  }
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof id);
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_err(STEN_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  }
  *out = c;
  return STEN_OK;
}

void sten_comm_destroy(sten_comm *c) {
  if (!c) return;
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  delete c;
}

static int is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // extern "C"

// cconst (host, 7 doubles: a_P, A_xm .. A_zp) selects a constant operator;
// else coeffs[] are the per-point fields
static int create_impl(int nx, int ny, int nz_global, const void *const coeffs[7], int coeff_dtype,
                       const double *cconst, int nslabs, sten_comm *comm, void *cuda_stream, sten_stencil **out) {
  if (!out) return set_err(STEN_EINVAL, "out is NULL");
  if (nx <= 0 || ny <= 0 || nz_global <= 0)
    return set_err(STEN_EINVAL, "mesh %d x %d x %d must be positive", nx, ny, nz_global);
  // slab convention: rank r of R owns planes [r nz/R, (r+1) nz/R)
  const int R_ = comm ? comm->nranks : 1;
  if (nz_global % R_ != 0)
    return set_err(STEN_EINVAL, "nz_global=%d not divisible by %d ranks", nz_global, R_);
  const int nz = nz_global / R_;
  if (comm) {
    int dev = -1;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev != comm->device)
      return set_err(STEN_EINVAL, "current CUDA device %d is not the communicator's device %d", dev, comm->device);
  }
  if (nslabs < 1 || nz % nslabs != 0) return set_err(STEN_EINVAL, "nz=%d not divisible into nslabs=%d", nz, nslabs);
  if (cconst) {
    for (int d = 0; d < 7; ++d)
      if (!std::isfinite(cconst[d])) return set_err(STEN_EINVAL, "constant coefficient %d is not finite", d);
    if (cconst[0] == 0.0) return set_err(STEN_EINVAL, "constant diagonal is zero");
    coeffs = nullptr;
    coeff_dtype = STEN_DT_F64;
  } else {
    if (!coeffs) return set_err(STEN_EINVAL, "coeffs is NULL");
    for (int d = 1; d < 7; ++d)
      if (!coeffs[d]) return set_err(STEN_EINVAL, "coeffs[%d] is NULL", d);
    if (coeff_dtype != STEN_DT_F64 && coeff_dtype != STEN_DT_F32)
      return set_err(STEN_EINVAL, "coeff_dtype %d unsupported", coeff_dtype);
  }
  if (nx > (1 << 20) || ny > (1 << 20)) return set_err(STEN_EINVAL, "nx, ny too large");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  sten_stencil *st = new sten_stencil;
  st->nx = nx;
  st->ny = ny;
  st->nz = nz;  // this rank's planes
  // Layout: rows of `pitch` elements, a multiple of
  // 8 (16-B vectors), planes a multiple of 64 elements.  Unpadded rows move
  // no padding bytes: the SR sweep (the bench's schedule) is 1.9% faster with
  // them at nx = 600 (144.0 vs 141.5 Gpoint-iter/s); with their coefficient tiles by
  // TMA the classic kernels are fastest unpadded too (107.1 vs 103.4 on 128-B rows).
  {
    const int align = 8;
    st->pitch = (nx + align - 1) / align * align;
    int nyp = ny;
    while (((long long)st->pitch * nyp) % 64) ++nyp;
    st->plane = (long long)st->pitch * nyp;
  }
  st->nslabs = nslabs;
  st->comm = comm;
  st->has_diag = cconst ? true : coeffs[0] != nullptr;
  if (cconst) {
    st->cc = true;
    for (int d = 0; d < 6; ++d) st->cscaled[d] = cconst[1 + d] / cconst[0];  // fp64, as k_create_coeffs
  }
  st->sm = device_sm_count();
  st->slabs.resize(nslabs);
  auto fail = [&](int rc) {
    stencil_destroy(st);
    return rc;
  };
  const int ein = coeff_dtype == STEN_DT_F64 ? 8 : 4;
  const size_t nin = (size_t)nx * ny * nz;
  // stage host inputs on the device
  std::vector<void *> staged(8, nullptr);
  const void *dev_in[7] = {};
  double *dconst = nullptr;
  if (cconst) {
    if (cudaMalloc(&staged[7], 7 * sizeof(double)) != cudaSuccess)
      return fail(set_err(STEN_ENOMEM, "constant staging failed"));
    dconst = (double *)staged[7];
    cudaMemcpyAsync(dconst, cconst, 7 * sizeof(double), cudaMemcpyHostToDevice, s);
  }
  for (int d = 0; d < 7 && coeffs; ++d) {
    dev_in[d] = coeffs[d];
    if (coeffs[d] && !is_device_ptr(coeffs[d])) {
      if (cudaMalloc(&staged[d], nin * ein) != cudaSuccess) {
        for (void *p : staged) cudaFree(p);
        return fail(set_err(STEN_ENOMEM, "staging coefficients failed"));
      }
      cudaMemcpyAsync(staged[d], coeffs[d], nin * ein, cudaMemcpyHostToDevice, s);
      dev_in[d] = staged[d];
    }
  }
  int rc = STEN_OK;
  const int nzs = nz / nslabs;
  const int R = comm ? comm->nranks : 1, me = comm ? comm->rank : 0;
  for (int k = 0; k < nslabs && rc == STEN_OK; ++k) {
    Slab &sl = st->slabs[k];
    sl.nz = nzs;
    sl.z_first = (long long)k * nzs;
    // one halo plane below and above (zero at the global mesh boundary, the
    // z-neighbour's plane at slab interfaces; read only by the SR sweep)
    const size_t cb32 = (size_t)st->plane * (nzs + 2) * 4, cb16 = (size_t)st->plane * (nzs + 2) * 2;
    for (int d = 0; d < 6 && rc == STEN_OK; ++d) {
      if (cudaMalloc(&sl.c32b[d], cb32) != cudaSuccess || cudaMalloc(&sl.c16b[d], cb16) != cudaSuccess) {
        rc = set_err(STEN_ENOMEM, "coefficient allocation failed");
        break;
      }
      cudaMemsetAsync(sl.c32b[d], 0, cb32, s);
      cudaMemsetAsync(sl.c16b[d], 0, cb16, s);
      sl.c32[d] = sl.c32b[d] + st->plane;
      sl.c16[d] = sl.c16b[d] + st->plane;
    }
    if (rc == STEN_OK && st->has_diag && cudaMalloc(&sl.aP, (size_t)st->plane * nzs * 8) != cudaSuccess)
      rc = set_err(STEN_ENOMEM, "diagonal allocation failed");
    if (rc != STEN_OK) break;
    const size_t soff = (size_t)sl.z_first * nx * ny * ein;
    const void *off[6] = {};
    for (int d = 0; d < 6 && !cconst; ++d) off[d] = (const char *)dev_in[d + 1] + soff;
    const void *dg = dev_in[0] ? (const char *)dev_in[0] + soff : nullptr;
    Geom g{nx, ny, nzs, st->pitch, st->plane};
    const int below = k > 0 || me > 0, above = k + 1 < nslabs || me + 1 < R;
    sl.has_below = below;
    sl.has_above = above;
    int e = create_coeffs_launch(coeff_dtype, dg, off, g, below, above, sl.c32, sl.c16, sl.aP, dconst, s);
    if (e) rc = set_err(STEN_ECUDA, "coefficient kernel: %s", cudaGetErrorString((cudaError_t)e));
  }
  if (rc == STEN_OK) rc = fill_coef_halos(st, s);
  if (rc == STEN_OK) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = set_err(STEN_ECUDA, "stencil_create: %s", cudaGetErrorString(e));
  }
  for (void *p : staged)
    if (p) cudaFree(p);
  if (rc != STEN_OK) return fail(rc);
  if (cudaMalloc(&st->st, sizeof(DevState)) != cudaSuccess ||
      cudaMallocHost(&st->st_host, sizeof(DevState)) != cudaSuccess ||
      cudaMalloc(&st->counter, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc(&st->slab_sums, sizeof(float) * kMaxDots * 3 * nslabs) != cudaSuccess ||
      cudaMalloc(&st->counter2, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc(&st->red_total, sizeof(float) * kMaxDots) != cudaSuccess)
    return fail(set_err(STEN_ENOMEM, "state allocation failed"));
  st->p2p_slots = nslabs * (comm ? comm->nranks : 1);  // x 2: double-buffered by sequence parity
  if (cudaMalloc(&st->p2p_sums, sizeof(float) * kMaxDots * 2 * st->p2p_slots) != cudaSuccess ||
      cudaMalloc(&st->p2p_flags, sizeof(unsigned) * 2 * st->p2p_slots) != cudaSuccess ||
      cudaMalloc(&st->p2p_seq, sizeof(unsigned)) != cudaSuccess)
    return fail(set_err(STEN_ENOMEM, "inbox allocation failed"));
  cudaMemset(st->p2p_sums, 0, sizeof(float) * kMaxDots * 2 * st->p2p_slots);
  cudaMemset(st->p2p_flags, 0, sizeof(unsigned) * 2 * st->p2p_slots);
  cudaMemset(st->p2p_seq, 0, sizeof(unsigned));
  cudaMemset(st->counter, 0, sizeof(unsigned));
  cudaMemset(st->counter2, 0, sizeof(unsigned));
  cudaMemset(st->st, 0, sizeof(DevState));
  cudaMemset(st->slab_sums, 0, sizeof(float) * kMaxDots * 3 * nslabs);
  cudaMemset(st->red_total, 0, sizeof(float) * kMaxDots);
  if (cudaStreamCreateWithFlags(&st->cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&st->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&st->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreate(&st->ev_a) != cudaSuccess || cudaEventCreate(&st->ev_b) != cudaSuccess)
    return fail(set_err(STEN_ECUDA, "stream/event creation failed"));
  *out = st;
  return STEN_OK;
}

extern "C" {

int stencil_create(int nx, int ny, int nz, const void *const coeffs[7], int coeff_dtype, int nslabs,
                   sten_comm *comm, void *cuda_stream, sten_stencil **out) {
  return create_impl(nx, ny, nz, coeffs, coeff_dtype, nullptr, nslabs, comm, cuda_stream, out);
}

int stencil_create_const(int nx, int ny, int nz, const double coeffs[7], int nslabs, sten_comm *comm,
                         void *cuda_stream, sten_stencil **out) {
  if (!coeffs) return set_err(STEN_EINVAL, "coeffs is NULL");
  return create_impl(nx, ny, nz, nullptr, STEN_DT_F64, coeffs, nslabs, comm, cuda_stream, out);
}

void stencil_destroy(sten_stencil *st) {
  if (!st) return;
  drop_graphs(st);
  for (Slab &sl : st->slabs) {
    for (int d = 0; d < 6; ++d) {
      cudaFree(sl.c32b[d]);
      cudaFree(sl.c16b[d]);
    }
    cudaFree(sl.aP);
    for (PrecBufs &b : sl.pb) {
      void *all[] = {b.x, b.r, b.rh, b.p[0], b.p[1], b.v[0], b.v[1], b.s, b.t, b.bw};
      for (void *p : all) cudaFree(p);
    }
    for (SrBufs &b : sl.sr) {
      cudaFree(b.x);
      cudaFree(b.rh);
      for (int k = 0; k < 2; ++k)
        for (int i = 0; i < 5; ++i) cudaFree(b.vec[k][i]);
    }
  }
  cudaFree(st->st);
  if (st->st_host) cudaFreeHost(st->st_host);
  cudaFree(st->partials);
  cudaFree(st->partials2);
  for (void *p : st->ipc_opened) cudaIpcCloseMemHandle(p);
  cudaFree(st->p2p_sums);
  cudaFree(st->p2p_flags);
  cudaFree(st->p2p_seq);
  cudaFree(st->counter);
  cudaFree(st->counter2);
  if (st->side) cudaStreamDestroy(st->side);
  if (st->io) cudaStreamDestroy(st->io);
  for (int k = 0; k < 2; ++k) {
    cudaFree(st->bstage[k]);
    cudaFree(st->xstage[k]);
    for (cudaEvent_t e : {st->ev_in[k], st->ev_used[k], st->ev_out[k], st->ev_dn[k]})
      if (e) cudaEventDestroy(e);
  }
  if (st->ev_fork) cudaEventDestroy(st->ev_fork);
  if (st->ev_join) cudaEventDestroy(st->ev_join);
  cudaFree(st->slab_sums);
  cudaFree(st->red_total);
  cudaFree(st->hist);
  cudaFree(st->ahist);
  cudaFree(st->whist);
  cudaFree(st->stage);
  cudaFree(st->ir_amax);
  cudaFree(st->ir_sigma);
  if (st->cap) cudaStreamDestroy(st->cap);
  if (st->ev_a) cudaEventDestroy(st->ev_a);
  if (st->ev_b) cudaEventDestroy(st->ev_b);
  delete st;
}

int sten_set_tiling(sten_stencil *st, int prec, int bx, int by, int zc, int stages) {
  if (!st || (prec != STEN_FP32 && prec != STEN_MIXED)) return set_err(STEN_EINVAL, "bad handle/precision");
  if (st->slabs[0].pb[prec].ready == false && st->tiling[prec].bx == 0) default_tiling(st, prec);
  Tiling t = st->tiling[prec];
  const int tbx = prec == STEN_FP32 ? tile_bx<float>() : tile_bx<__half>();
  if (bx == tbx) {
    t.rows = 0;
    t.bx = tbx;
  } else if (bx >= st->nx) {
    t.rows = 1;
    t.bx = st->pitch;
  } else if (bx != 0) {
    return set_err(STEN_EINVAL, "bx must be 0, %d (tiles) or >= nx=%d (full-row strips)", tbx, st->nx);
  }
  if (by) t.by = by;
  if (zc) t.zc = t.zc2 = zc;
  if (stages) {  // an explicit pipeline depth selects the per-thread coefficient loads (3 or 4 stages)
    t.stages = stages;
    t.cstages = 0;
  } else if (t.rows || (t.cstages && !stencil_config_ok(t.by, t.stages, t.cstages))) {
    t.stages = 4;  // row strips, or a tile height without a coefficient-TMA instance
    t.cstages = 0;
  }
  if (t.rows) {
    if (t.zc <= 0 || !rows_config_ok(t.by, t.stages) || rows_thr(prec, st->nx, t.by) > 512 ||
        rows_smem_bytes(MODE_H1, esize(prec), st->pitch, t.by, t.stages) > 227 * 1024)
      return set_err(STEN_EINVAL, "unsupported row-strip tiling by=%d zc=%d stages=%d", t.by, t.zc, t.stages);
    t.threads = rows_thr(prec, st->nx, t.by);
  } else {
    if (t.zc <= 0 || !stencil_config_ok(t.by, t.stages, t.cstages))
      return set_err(STEN_EINVAL, "unsupported tiling by=%d zc=%d stages=%d (by 4/8/16, stages 3/4)", t.by, t.zc,
                     t.stages);
    t.threads = prec == STEN_FP32 ? stencil_threads<float>(t.by) : stencil_threads<__half>(t.by);
  }
  st->tiling[prec] = t;
  for (Slab &sl : st->slabs) sl.pb[prec].maps_ok = false;
  drop_graphs(st);
  if (st->slabs[0].pb[prec].ready) RC_TRY(ensure_bufs(st, prec));
  return STEN_OK;
}

int sten_set_host_barrier(sten_stencil *st, void (*fn)(void *ctx), void *ctx) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  st->barrier_fn = fn;
  st->barrier_ctx = ctx;
  drop_graphs(st);
  return STEN_OK;
}

int sten_set_option(sten_stencil *st, int option, int value) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  switch (option) {
    case STEN_OPT_TMA_L2_PROMOTION:
      if (value < 0 || value > 3) return set_err(STEN_EINVAL, "TMA L2 promotion %d not in 0..3", value);
      st->tma_promo = value;
      for (Slab &sl : st->slabs)
        for (int p = 0; p < 2; ++p) {
          sl.pb[p].maps_ok = false;
          sl.sr[p].maps_ok = false;
        }
      break;
    case STEN_OPT_EW_CTAS_PER_SM:
      if (value < 1 || value > 64) return set_err(STEN_EINVAL, "element-wise CTAs per SM %d not in 1..64", value);
      st->ew_bps = value;
      break;
    case STEN_OPT_COEF_PREFETCH:
      if (value < 0 || value > 16) return set_err(STEN_EINVAL, "coefficient prefetch distance %d not in 0..16", value);
      st->coef_pf = value;
      break;
    case STEN_OPT_SR_L2_PREFETCH:
      if (value < 0 || value > 16) return set_err(STEN_EINVAL, "SR L2 prefetch distance %d not in 0..16", value);
      st->sr_l2pf = value;
      break;
    case STEN_OPT_SR_LIGHT_LAST:
      if (value != 0 && value != 1) return set_err(STEN_EINVAL, "SR light last sweep must be 0 or 1 (got %d)", value);
      st->sr_light = value != 0;
      break;
    case STEN_OPT_CLASSIC_OVERLAP:
      if (value != 0 && value != 1) return set_err(STEN_EINVAL, "classic overlap must be 0 or 1 (got %d)", value);
      st->cls_overlap = value != 0;
      break;
    case STEN_OPT_CLASSIC_FUSED:
      if (value != 0 && value != 1) return set_err(STEN_EINVAL, "classic fused exchange must be 0 or 1 (got %d)", value);
      st->cls_fuse = value != 0;
      break;
    case STEN_OPT_CLASSIC_CONST:
      if (value != 0 && value != 1) return set_err(STEN_EINVAL, "classic constant couplings must be 0 or 1 (got %d)", value);
      st->cls_const = value != 0;
      break;
    default:
      return set_err(STEN_EINVAL, "unknown option %d", option);
  }
  drop_graphs(st);
  return STEN_OK;
}

int sten_get_option(sten_stencil *st, int option, int *value) {
  if (!st || !value) return set_err(STEN_EINVAL, "NULL argument");
  switch (option) {
    case STEN_OPT_TMA_L2_PROMOTION: *value = st->tma_promo; break;
    case STEN_OPT_EW_CTAS_PER_SM: *value = st->ew_bps; break;
    case STEN_OPT_COEF_PREFETCH: *value = st->coef_pf; break;
    case STEN_OPT_SR_L2_PREFETCH: *value = st->sr_l2pf; break;
    case STEN_OPT_SR_LIGHT_LAST: *value = st->sr_light ? 1 : 0; break;
    case STEN_OPT_CLASSIC_OVERLAP: *value = st->cls_overlap ? 1 : 0; break;
    case STEN_OPT_CLASSIC_FUSED: *value = st->cls_fuse ? 1 : 0; break;
    case STEN_OPT_CLASSIC_CONST: *value = st->cls_const ? 1 : 0; break;
    default: return set_err(STEN_EINVAL, "unknown option %d", option);
  }
  return STEN_OK;
}

int sten_set_timing(sten_stencil *st, int enable) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  st->timing = enable != 0;
  return STEN_OK;
}

int sten_get_stats(sten_stencil *st, sten_stats *out) {
  if (!st || !out) return set_err(STEN_EINVAL, "NULL argument");
  *out = st->stats;
  return STEN_OK;
}

int stencil_apply(sten_stencil *st, int prec, const void *x, void *y, void *cuda_stream) {
  if (!st || !x || !y) return set_err(STEN_EINVAL, "NULL argument");
  if (p2p_only(st)) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: stencil_apply needs NCCL");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  RC_TRY(ensure_bufs(st, prec));
  st->launches = 0;
  RC_TRY(copy_in(st, prec, sel_s, x, s));
  if (decomposed(st)) RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.s; }, s));
  for (int k = 0; k < (int)st->slabs.size(); ++k) RC_TRY(launch_stencil(st, prec, MODE_APPLY, k, 0, s));
  RC_TRY(copy_out(st, prec, sel_t, y, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return STEN_OK;
}

// The solve proper (Alg. 1 / SR) on a right-hand side already in the working
// precision's bw buffer and (with_x0) an initial guess in the classic x
// buffer.  scale_rhs: b_hat = b / a_P (R3) - off for the refinement's inner
// solves, whose right-hand side is already a residual of the scaled system.
struct SolveOut {
  DevState fin;
  int chunk = 0;
  long long kernels = 0;
  double ph_ms[3] = {0, 0, 0};
  long long ph_n[3] = {0, 0, 0};
  std::vector<float> iter_ms;  // device ms of each timed iteration: [it][H1, H2, H3] (SR: [it][sweep, 0, 0])
};
static int solve_core(sten_stencil *st, int prec, bool with_x0, bool scale_rhs, double tol, int maxit, cudaStream_t s,
                      SolveOut *out) {
  const bool sr = st->schedule == STEN_SCHED_SR;
  if (!sr && prec == STEN_MIXED && st->half_dots) {  // R28: one slab, the tile kernels, field operator
    const Tiling &t = st->tiling[prec];
    if (decomposed(st) || st->cc || (t.bx != 0 && (t.rows || !(t.by == 16 && t.stages == 2 && t.cstages == 2))))
      return set_err(STEN_EUNSUPPORTED, "half dots in the classic schedule: one slab, field coefficients, the "
                                        "default tile kernels");
  }
  if (p2p_only(st)) {  // no NCCL: peer memory moves the data between ranks (after sten_p2p_import)
    if (!st->p2p_ranks || (sr && !st->sr_p2p))
      return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: a solve needs sten_p2p_import (and, for the SR "
                                        "schedule, the fused exchange)");
    if (with_x0) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: x0 must be NULL");
    if (!sr && !st->barrier_fn)
      return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: the classic schedule runs in host lockstep "
                                        "(sten_set_host_barrier)");
  }
  RC_TRY(ensure_bufs(st, prec));
  if (sr) RC_TRY(ensure_sr(st, prec));
  if (maxit + 2 > st->hist_cap) {
    cudaFree(st->hist);
    cudaFree(st->ahist);
    cudaFree(st->whist);
    st->hist_cap = maxit + 2 < 64 ? 64 : maxit + 2;
    CUDA_TRY(cudaMalloc(&st->hist, sizeof(double) * st->hist_cap));
    CUDA_TRY(cudaMalloc(&st->ahist, sizeof(float) * st->hist_cap));
    CUDA_TRY(cudaMalloc(&st->whist, sizeof(float) * st->hist_cap));
  }
  // device state
  DevState h;
  memset(&h, 0, sizeof h);
  h.tol = tol;
  h.maxit = maxit;
  h.status = -1;
  h.ev = -1;
  h.half = prec == STEN_MIXED;
  h.hist = st->hist;
  h.ahist = st->ahist;
  h.whist = st->whist;
  // SR on one slab: the last sweep without its SpMVs (k_sr_last)
  const bool light = sr && !decomposed(st) && !(prec == STEN_MIXED && st->half_dots) && st->sr_light;
  h.light = light ? 1 : 0;
  *st->st_host = h;
  CUDA_TRY(cudaMemcpyAsync(st->st, st->st_host, sizeof h, cudaMemcpyHostToDevice, s));
  // S1: b_hat, r0, rhat, p0 (Alg. 1 l.174; R1, R3)
  if (with_x0) {
    // A x0 through the apply path: input buffer s, output t
    for (Slab &sl : st->slabs) {
      const size_t vb = (size_t)st->plane * esize(prec);
      CUDA_TRY(cudaMemcpyAsync((char *)sl.pb[prec].s + vb, (char *)sl.pb[prec].x + vb, vb * sl.nz,
                               cudaMemcpyDeviceToDevice, s));
    }
    if (decomposed(st)) RC_TRY(exchange(st, prec, [](PrecBufs &bb) { return bb.s; }, s));
    for (int k = 0; k < (int)st->slabs.size(); ++k) RC_TRY(launch_stencil(st, prec, MODE_APPLY, k, 0, s));
    if (sr)
      for (Slab &sl : st->slabs) {
        const size_t vb = (size_t)st->plane * esize(prec);
        CUDA_TRY(cudaMemcpyAsync(sr_interior(sl.sr[prec].x, st, prec), (char *)sl.pb[prec].x + vb, vb * sl.nz,
                                 cudaMemcpyDeviceToDevice, s));
      }
  } else {
    for (Slab &sl : st->slabs) {
      const size_t vb = (size_t)st->plane * esize(prec);
      if (sr) CUDA_TRY(cudaMemsetAsync(sr_interior(sl.sr[prec].x, st, prec), 0, vb * sl.nz, s));
      else CUDA_TRY(cudaMemsetAsync((char *)sl.pb[prec].x + vb, 0, vb * sl.nz, s));
    }
  }
  for (int k = 0; k < (int)st->slabs.size(); ++k)
    RC_TRY(sr ? launch_init_sr(st, prec, k, with_x0, s, scale_rhs) : launch_init(st, prec, k, with_x0, s, scale_rhs));
  RC_TRY(reduce_scalars(st, PH_INIT, s));
  // fused SR: every sweep writes the halos of the set the next one reads; the
  // first sweep's (set 0, from the init) are exchanged here once
  if (sr && sr_fused(st)) RC_TRY(sr_exchange(st, prec, 0, s));
  // fused classic: H1 and H3 write the halos the next phases read; the first H1's (r, p0, v0 from
  // the init) are exchanged here once
  if (!sr && cls_fused(st)) {
    RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.r; }, s));
    RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.p[0]; }, s));
    RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.v[0]; }, s));
    RC_TRY(host_barrier(st, s));
  }
  // iterations: CUDA graphs of `chunk` iterations (even, so the ping-pong
  // parity of p/v is the same at every replay)
  const int nsteps = sr ? maxit + 1 : maxit;  // SR: sweep i computes x_i, r_i (i = 0..maxit)
  if (nsteps > 0) {
    const bool lockstep = st->barrier_fn && p2p_only(st);
    int chunk = tol > 0.0 ? 8 : ((nsteps + 1) / 2) * 2;
    if (chunk > 2048) chunk = 2048;
    if (lockstep) chunk = 0;
    out->chunk = chunk;
    // host lockstep (several ranks on one GPU): sweep by sweep, no graph; every
    // rank runs the same sweeps because every rank takes the same scalar decisions
    for (int i = 0; lockstep && i < nsteps; ++i) {
      RC_TRY(sr ? enqueue_sr_sweep(st, prec, i & 1, s, nullptr) : enqueue_iteration(st, prec, i & 1, s, nullptr));
      CUDA_TRY(cudaMemcpyAsync(st->st_host, st->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      if (st->st_host->stop || st->st_host->it >= maxit) break;
    }
    GraphRec *gr = nullptr;
    if (!lockstep) RC_TRY(get_graph(st, prec, chunk, &gr));
    const int nrep = lockstep ? 0 : (nsteps + chunk - 1) / chunk;
    for (int rep = 0; rep < nrep; ++rep) {
      CUDA_TRY(cudaGraphLaunch(gr->exec, s));
      out->kernels += gr->kernels;
      const bool poll = tol > 0.0 || st->timing;
      if (poll) {
        CUDA_TRY(cudaMemcpyAsync(st->st_host, st->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (st->timing) {
          const int done_it = st->st_host->it;
          const int first = rep * chunk;
          for (int j = 0; j < chunk; ++j) {
            if (sr ? first + j > done_it : first + j >= done_it) break;  // later kernels were no-ops
            float it_ms[3] = {0.f, 0.f, 0.f};
            for (int p = 0; p < (sr ? 1 : 3); ++p) {
              float ms = 0.f;
              cudaError_t te =
                  cudaEventElapsedTime(&ms, gr->ev[(size_t)j * 6 + 2 * p], gr->ev[(size_t)j * 6 + 2 * p + 1]);
              if (te != cudaSuccess)
                return set_err(STEN_ECUDA, "cudaEventElapsedTime(iter %d, phase %d): %s", j, p,
                               cudaGetErrorString(te));
              out->ph_ms[p] += ms;
              out->ph_n[p] += 1;
              it_ms[p] = ms;
            }
            out->iter_ms.insert(out->iter_ms.end(), it_ms, it_ms + 3);
          }
        }
        if (st->st_host->stop || st->st_host->it >= maxit) break;
      }
    }
    if (light) {  // sweep maxit (a no-op unless the solve got there)
      Slab &sl = st->slabs[0];
      SrBufs &b = sl.sr[prec];
      const int set = maxit & 1, vec = prec == STEN_FP32 ? 4 : 8;
      SrLastArgs la;
      memset(&la, 0, sizeof la);
      la.x = sr_interior(b.x, st, prec);
      la.rh = sr_interior(b.rh, st, prec);
      la.r = sr_interior(b.vec[set][0], st, prec);
      la.p = sr_interior(b.vec[set][1], st, prec);
      la.v = sr_interior(b.vec[set][2], st, prec);
      la.q = sr_interior(b.vec[set][3], st, prec);
      la.y = sr_interior(b.vec[set][4], st, prec);
      la.nvec = (long long)st->plane * sl.nz / vec;
      la.red = make_red(st, 0);
      const int g = ew_grid(st, la.nvec);
      if (g > st->partials_cap) return set_err(STEN_ECUDA, "internal: last-sweep grid exceeds the partial-sum buffer");
      if (prec == STEN_FP32) KLAUNCH(sr_last_launch<float>(la, g, s));
      else KLAUNCH(sr_last_launch<__half>(la, g, s));
      out->kernels += 1;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(st->st_host, st->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  out->fin = *st->st_host;
  if (out->fin.zero_x)
    for (Slab &sl : st->slabs) {
      const size_t vb = (size_t)st->plane * esize(prec);
      if (sr) CUDA_TRY(cudaMemsetAsync(sr_interior(sl.sr[prec].x, st, prec), 0, vb * sl.nz, s));
      else CUDA_TRY(cudaMemsetAsync((char *)sl.pb[prec].x + vb, 0, vb * sl.nz, s));
    }
  return STEN_OK;
}

// device pointer of slab `k`'s solution (interior plane 0) after solve_core
static char *solution_ptr(sten_stencil *st, int prec, Slab &sl) {
  if (st->schedule == STEN_SCHED_SR) return sr_interior(sl.sr[prec].x, st, prec);
  return (char *)sl.pb[prec].x + (size_t)st->plane * esize(prec);
}

int bicgstab_solve(sten_stencil *st, int prec, const void *b, const void *x0, double tol, int maxit, void *x_out,
                   int *iters, double *res_hist, int *status, void *cuda_stream) {
  if (!st || !b || !x_out || !iters || !res_hist || !status) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (!(tol >= 0.0) || maxit < 0) return set_err(STEN_EINVAL, "tol=%g maxit=%d invalid", tol, maxit);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const bool sr = st->schedule == STEN_SCHED_SR;
  RC_TRY(ensure_bufs(st, prec));
  if (sr) RC_TRY(ensure_sr(st, prec));
  st->launches = 0;
  memset(&st->stats, 0, sizeof st->stats);
  CUDA_TRY(cudaEventRecord(st->ev_a, s));
  RC_TRY(copy_in(st, prec, sel_bw, b, s));
  if (x0) RC_TRY(copy_in(st, prec, sel_x, x0, s));
  SolveOut so;
  RC_TRY(solve_core(st, prec, x0 != nullptr, true, tol, maxit, s, &so));
  CUDA_TRY(cudaEventRecord(st->ev_b, s));
  const DevState &fin = so.fin;
  if (sr) RC_TRY(sr_copy_out(st, prec, [prec](Slab &sl) { return sl.sr[prec].x; }, x_out, s));
  else RC_TRY(copy_out(st, prec, sel_x, x_out, s));
  CUDA_TRY(cudaMemcpyAsync(res_hist, st->hist, sizeof(double) * (fin.it + 1), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  *iters = fin.it;
  *status = fin.stop ? fin.status : (fin.ev >= 0 ? fin.ev : STEN_MAXIT);
  float solve_ms = 0.f;
  cudaEventElapsedTime(&solve_ms, st->ev_a, st->ev_b);
  st->stats.solve_ms = solve_ms;
  for (int p = 0; p < 3; ++p) {
    st->stats.phase_ms[p] = so.ph_ms[p];
    st->stats.phase_launches[p] = so.ph_n[p];
  }
  st->stats.kernel_launches = st->launches + so.kernels;
  st->stats.event_iter = fin.ev >= 0 ? fin.ev_it : 0;
  st->stats.graph_chunk = so.chunk;
  st->iter_ms = so.iter_ms;
  return STEN_OK;
}

int sten_iter_ms(sten_stencil *st, int phase, float *out, int cap, int *n) {
  if (!st || !n || (cap > 0 && !out)) return set_err(STEN_EINVAL, "NULL argument");
  if (phase < -1 || phase > 2) return set_err(STEN_EINVAL, "phase %d not in -1..2", phase);
  *n = (int)(st->iter_ms.size() / 3);
  for (int i = 0; i < cap && i < *n; ++i) {
    const float *m = &st->iter_ms[(size_t)i * 3];
    out[i] = phase < 0 ? m[0] + m[1] + m[2] : m[phase];
  }
  return STEN_OK;
}

// Many right-hand sides: the host<->device copies of solve i+1 / i-1 run on a
// copy stream during solve i (double-buffered dense staging).
static int ensure_io(sten_stencil *st, size_t bytes) {
  if (!st->io) {  // events first, the stream last: a half-made set is retried on the next call
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t *e : {&st->ev_in[k], &st->ev_used[k], &st->ev_out[k], &st->ev_dn[k]})
        if (!*e) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    cudaStream_t io = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&io, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {st->ev_in[k], st->ev_used[k], st->ev_out[k], st->ev_dn[k]})
        CUDA_TRY(cudaEventRecord(e, io));  // "done" before first use
    st->io = io;
  }
  if (bytes > st->io_bytes) {
    CUDA_TRY(cudaStreamSynchronize(st->io));
    for (int k = 0; k < 2; ++k) {
      cudaFree(st->bstage[k]);
      cudaFree(st->xstage[k]);
      st->bstage[k] = st->xstage[k] = nullptr;
      st->io_bytes = 0;
      if (cudaMalloc(&st->bstage[k], bytes) != cudaSuccess || cudaMalloc(&st->xstage[k], bytes) != cudaSuccess)
        return set_err(STEN_ENOMEM, "bicgstab_solve_batch: staging of 4 x %zu bytes", bytes);
    }
    st->io_bytes = bytes;
  }
  return STEN_OK;
}

int bicgstab_solve_batch(sten_stencil *st, int prec, int n, const void *const *b, void *const *x_out, double tol,
                         int maxit, int *iters, double *res_hist, int *status, void *cuda_stream) {
  if (!st || n < 0 || (n > 0 && (!b || !x_out || !iters || !res_hist || !status)))
    return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (!(tol >= 0.0) || maxit < 0) return set_err(STEN_EINVAL, "tol=%g maxit=%d invalid", tol, maxit);
  for (int i = 0; i < n; ++i)
    if (!b[i] || !x_out[i]) return set_err(STEN_EINVAL, "NULL vector %d", i);
  if (n == 0) return STEN_OK;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const bool sr = st->schedule == STEN_SCHED_SR;
  RC_TRY(ensure_bufs(st, prec));
  if (sr) RC_TRY(ensure_sr(st, prec));
  long long pts = 0;
  for (const Slab &sl : st->slabs) pts += (long long)sl.nz;
  const size_t bytes = (size_t)pts * st->nx * st->ny * esize(prec);
  RC_TRY(ensure_io(st, bytes));
  // every exit (errors included) waits for the copy stream: no copy into or out of the
  // caller's buffers may still be in flight when the call returns
  struct IoDrain {
    cudaStream_t io;
    ~IoDrain() { cudaStreamSynchronize(io); }
  } drain{st->io};
  st->launches = 0;
  memset(&st->stats, 0, sizeof st->stats);
  CUDA_TRY(cudaEventRecord(st->ev_a, s));
  // H2D of b[i] into slot i&1 once the solve of i-2 has consumed that slot
  auto upload = [&](int i) -> int {
    const int k = i & 1;
    if (ptr_on_device(b[i])) return STEN_OK;
    CUDA_TRY(cudaStreamWaitEvent(st->io, st->ev_used[k], 0));
    CUDA_TRY(cudaMemcpyAsync(st->bstage[k], b[i], bytes, cudaMemcpyHostToDevice, st->io));
    CUDA_TRY(cudaEventRecord(st->ev_in[k], st->io));
    return STEN_OK;
  };
  RC_TRY(upload(0));
  long long kernels = 0;
  for (int i = 0; i < n; ++i) {
    const int k = i & 1;
    if (i + 1 < n) RC_TRY(upload(i + 1));
    const bool bdev = ptr_on_device(b[i]), xdev = ptr_on_device(x_out[i]);
    if (!bdev) CUDA_TRY(cudaStreamWaitEvent(s, st->ev_in[k], 0));
    RC_TRY(copy_in(st, prec, sel_bw, bdev ? b[i] : st->bstage[k], s));
    if (!bdev) CUDA_TRY(cudaEventRecord(st->ev_used[k], s));
    SolveOut so;
    RC_TRY(solve_core(st, prec, false, true, tol, maxit, s, &so));
    kernels += so.kernels;
    const DevState &fin = so.fin;
    if (!xdev) CUDA_TRY(cudaStreamWaitEvent(s, st->ev_dn[k], 0));  // the D2H of solve i-2 left the slot
    void *xd = xdev ? x_out[i] : st->xstage[k];
    if (sr) RC_TRY(sr_copy_out(st, prec, [prec](Slab &sl) { return sl.sr[prec].x; }, xd, s));
    else RC_TRY(copy_out(st, prec, sel_x, xd, s));
    CUDA_TRY(cudaMemcpyAsync(res_hist + (size_t)i * (maxit + 1), st->hist, sizeof(double) * (fin.it + 1),
                             cudaMemcpyDeviceToHost, s));
    for (int j = fin.it + 1; j <= maxit; ++j) res_hist[(size_t)i * (maxit + 1) + j] = NAN;
    if (!xdev) {
      CUDA_TRY(cudaEventRecord(st->ev_out[k], s));
      CUDA_TRY(cudaStreamWaitEvent(st->io, st->ev_out[k], 0));
      CUDA_TRY(cudaMemcpyAsync(x_out[i], st->xstage[k], bytes, cudaMemcpyDeviceToHost, st->io));
      CUDA_TRY(cudaEventRecord(st->ev_dn[k], st->io));
    }
    iters[i] = fin.it;
    status[i] = fin.stop ? fin.status : (fin.ev >= 0 ? fin.ev : STEN_MAXIT);
  }
  CUDA_TRY(cudaStreamSynchronize(st->io));
  CUDA_TRY(cudaEventRecord(st->ev_b, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, st->ev_a, st->ev_b);
  st->stats.solve_ms = ms;
  st->stats.kernel_launches = st->launches + kernels;
  return STEN_OK;
}

// ------------------------------------------ iterative refinement (R21) --
static int ir_grid(sten_stencil *st, long long n) {
  long long g = (n + 255) / 256;
  if (g > (long long)st->sm * 8) g = st->sm * 8;
  return (int)(g < 1 ? 1 : g);
}

// r = b_hat - A x (fp32) on every slab; returns ||r||^2 (all slabs / ranks) and
// leaves max|r| in ir_amax.  x_zero: x = 0, so r = b_hat exactly and no SpMV runs.
static int ir_residual(sten_stencil *st, cudaStream_t s, double *rr, bool x_zero = false) {
  const int F = STEN_FP32;
  const size_t vb = (size_t)st->plane * 4;
  if (!x_zero) {
    if (decomposed(st)) RC_TRY(exchange(st, F, [](PrecBufs &bb) { return bb.s; }, s));
    for (int k = 0; k < (int)st->slabs.size(); ++k) RC_TRY(launch_stencil(st, F, MODE_APPLY, k, 0, s));
  }
  CUDA_TRY(cudaMemsetAsync(st->ir_amax, 0, sizeof(unsigned), s));
  for (int k = 0; k < (int)st->slabs.size(); ++k) {
    Slab &sl = st->slabs[k];
    PrecBufs &b = sl.pb[F];
    IrArgs a;
    memset(&a, 0, sizeof a);
    a.b = (const float *)((char *)b.rh + vb);  // b_hat
    a.ax = x_zero ? nullptr : (const float *)((char *)b.t + vb);
    a.r = (float *)((char *)b.r + vb);
    a.amax = st->ir_amax;
    a.n = (long long)st->plane * sl.nz;
    a.red = make_red(st, k);
    a.red.slab_out = st->slab_sums + k * kMaxDots;
    const int g = ir_grid(st, a.n);
    if (g > st->partials_cap) return set_err(STEN_ECUDA, "internal: refinement grid exceeds the partial-sum buffer");
    KLAUNCH(ir_launch(IR_RESID, a, g, s));
    st->launches++;
  }
  KLAUNCH(slabsum_launch(st->slab_sums, (int)st->slabs.size(), st->red_total, s));
  if (nccl_ranks(st)) {
    NCCL_TRY(g_nccl.AllReduce(st->red_total, st->red_total, 1, ncclFloat32, ncclSum, st->comm->comm, s));
    NCCL_TRY(g_nccl.AllReduce(st->ir_amax, st->ir_amax, 1, ncclUint32, ncclMax, st->comm->comm, s));
  }
  float h = 0.f;
  CUDA_TRY(cudaMemcpyAsync(&h, st->red_total, sizeof h, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *rr = (double)h;
  return STEN_OK;
}

int bicgstab_refine(sten_stencil *st, const void *b, const void *x0, double tol, int outer_maxit, double inner_tol,
                    int inner_maxit, void *x_out, int *outer_iters, int *inner_iters, double *res_hist, int *status,
                    void *cuda_stream) {
  if (!st || !b || !x_out || !outer_iters || !inner_iters || !res_hist || !status)
    return set_err(STEN_EINVAL, "NULL argument");
  if (p2p_only(st)) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: bicgstab_refine needs NCCL");
  if (!(tol > 0.0) || !(inner_tol >= 0.0) || outer_maxit < 0 || inner_maxit < 1)
    return set_err(STEN_EINVAL, "tol=%g inner_tol=%g outer_maxit=%d inner_maxit=%d invalid", tol, inner_tol,
                   outer_maxit, inner_maxit);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int F = STEN_FP32, M = STEN_MIXED;
  RC_TRY(ensure_bufs(st, F));
  RC_TRY(ensure_bufs(st, M));
  if (st->schedule == STEN_SCHED_SR) RC_TRY(ensure_sr(st, M));
  if (!st->ir_amax) {
    CUDA_TRY(cudaMalloc(&st->ir_amax, sizeof(unsigned)));
    CUDA_TRY(cudaMalloc(&st->ir_sigma, sizeof(float)));
  }
  st->launches = 0;
  memset(&st->stats, 0, sizeof st->stats);
  CUDA_TRY(cudaEventRecord(st->ev_a, s));
  const size_t v4 = (size_t)st->plane * 4, v2 = (size_t)st->plane * 2;
  // b_hat (fp32, R3) into the fp32 rh buffer; the iterate x lives in the fp32 s buffer
  RC_TRY(copy_in(st, F, sel_bw, b, s));
  for (Slab &sl : st->slabs) {
    PrecBufs &pb = sl.pb[F];
    IrArgs a;
    memset(&a, 0, sizeof a);
    a.b = (const float *)((char *)pb.bw + v4);
    a.aP = st->has_diag ? sl.aP : nullptr;
    a.r = (float *)((char *)pb.rh + v4);
    a.n = (long long)st->plane * sl.nz;
    KLAUNCH(ir_launch(IR_BHAT, a, ir_grid(st, a.n), s));
    st->launches++;
    CUDA_TRY(cudaMemsetAsync((char *)pb.s + v4, 0, v4 * sl.nz, s));
  }
  double bb = 0.0;
  RC_TRY(ir_residual(st, s, &bb, true));  // x = 0: r = b_hat
  const double nb = sqrt(bb);
  const bool zero_b = nb == 0.0;  // b = 0: x = 0 is exact, whatever x0 is
  if (x0 && !zero_b) RC_TRY(copy_in(st, F, sel_s, x0, s));
  int k = 0, inner = 0, stat = STEN_MAXIT, stale = 0;
  double best = 0.0;
  // the first stagnation switches the inner schedule, classic <-> SR (R21);
  // the handle's schedule is restored on every return
  struct SchedRestore {
    sten_stencil *st;
    int sched;
    ~SchedRestore() { st->schedule = sched; }
  } restore{st, st->schedule};
  st->stats.handover = -1;
  for (;; ++k) {
    if (zero_b) {
      res_hist[0] = 0.0;
      stat = STEN_CONVERGED;
      break;
    }
    double rr = bb;
    if (x0 || k > 0) RC_TRY(ir_residual(st, s, &rr));
    const double res = sqrt(rr) / nb;
    res_hist[k] = res;
    if (!std::isfinite(res)) { stat = STEN_NONFINITE; break; }
    if (res <= tol) { stat = STEN_CONVERGED; break; }
    // stagnation (R21): three consecutive steps without a 1% gain on the best residual
    if (k == 0 || res < 0.99 * best) {
      best = (k == 0 || res < best) ? res : best;
      stale = 0;
    } else if (++stale >= 3) {
      const int other = st->schedule == STEN_SCHED_SR ? STEN_SCHED_CLASSIC : STEN_SCHED_SR;
      // (the classic buffers exist, ensure_bufs above; SR ones are made here - a handle
      // whose configuration has no SR sweep stops instead)
      if (st->stats.handover >= 0 || (other == STEN_SCHED_SR && ensure_sr(st, M) != STEN_OK)) {
        stat = STEN_BREAKDOWN;
        break;
      }
      st->schedule = other;
      st->stats.handover = k;
      stale = 0;
    }
    if (k == outer_maxit) { stat = STEN_MAXIT; break; }
    // inner right-hand side: r / sigma in fp16 (sigma = 2^e >= max|r|)
    for (Slab &sl : st->slabs) {
      IrArgs a;
      memset(&a, 0, sizeof a);
      a.r = (float *)((char *)sl.pb[F].r + v4);
      a.r16 = (__half *)((char *)sl.pb[M].bw + v2);
      a.amax = st->ir_amax;
      a.sigma = st->ir_sigma;
      a.n = (long long)st->plane * sl.nz;
      KLAUNCH(ir_launch(IR_SCALE, a, ir_grid(st, a.n), s));
      st->launches++;
    }
    SolveOut so;
    RC_TRY(solve_core(st, M, false, false, inner_tol, inner_maxit, s, &so));
    inner += so.fin.it;
    st->launches += so.kernels;
    const int ist = so.fin.stop ? so.fin.status : (so.fin.ev >= 0 ? so.fin.ev : STEN_MAXIT);
    if (ist == STEN_NONFINITE) {  // R21: a diverged inner solve adds nothing; the cap halves
      inner_maxit = std::max(1, inner_maxit / 2);
      continue;
    }
    for (Slab &sl : st->slabs) {
      IrArgs a;
      memset(&a, 0, sizeof a);
      a.d16 = (const __half *)solution_ptr(st, M, sl);
      a.x = (float *)((char *)sl.pb[F].s + v4);
      a.sigma = st->ir_sigma;
      a.n = (long long)st->plane * sl.nz;
      KLAUNCH(ir_launch(IR_UPDATE, a, ir_grid(st, a.n), s));
      st->launches++;
    }
  }
  CUDA_TRY(cudaEventRecord(st->ev_b, s));
  RC_TRY(copy_out(st, F, sel_s, x_out, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  *outer_iters = k;
  *inner_iters = inner;
  *status = stat;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, st->ev_a, st->ev_b);
  st->stats.solve_ms = ms;
  st->stats.kernel_launches = st->launches;
  return STEN_OK;
}

int sten_scalar_history(sten_stencil *st, int n, double *alpha, double *omega) {
  if (!st || n < 0 || (n > 0 && (!alpha || !omega))) return set_err(STEN_EINVAL, "bad arguments");
  if (n + 1 > st->hist_cap) return set_err(STEN_EINVAL, "n=%d exceeds the last solve", n);
  std::vector<float> a(n + 1), w(n + 1);
  CUDA_TRY(cudaMemcpy(a.data(), st->ahist, sizeof(float) * (n + 1), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(w.data(), st->whist, sizeof(float) * (n + 1), cudaMemcpyDeviceToHost));
  for (int i = 1; i <= n; ++i) {
    alpha[i - 1] = a[i];
    omega[i - 1] = w[i];
  }
  return STEN_OK;
}

int sten_set_dot_precision(sten_stencil *st, int dots) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  if (dots != STEN_DOTS_MIXED && dots != STEN_DOTS_HALF) return set_err(STEN_EINVAL, "unknown dot precision %d", dots);
  if (st->half_dots != (dots == STEN_DOTS_HALF)) drop_graphs(st);
  st->half_dots = dots == STEN_DOTS_HALF;
  return STEN_OK;
}

int sten_classic_segments(sten_stencil *st, int prec, int *z0, int cap, int *n) {
  if (!st || !n) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (st->tiling[prec].bx == 0) default_tiling(st, prec);
  const Tiling &t = st->tiling[prec];
  int cnt = 0;
  for (const Slab &sl : st->slabs) {
    std::vector<int> starts;
    for (int mode : {MODE_H1, MODE_H2}) {  // the union of the H1 (= apply) and H2 plans
      const int zc = (prec == STEN_MIXED && st->half_dots) ? t.zc : zc_of(t, mode);  // half dots: one plan
      if (cls_overlapped(st)) {  // plane 0, the interior in zc chunks from plane 1, plane nz-1
        starts.push_back(0);
        for (int z = 1; z < sl.nz - 1; z += zc) starts.push_back(z);
        starts.push_back(sl.nz - 1);
      } else {
        for (int z = 0; z < sl.nz; z += zc) starts.push_back(z);
      }
    }
    std::sort(starts.begin(), starts.end());
    starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
    for (int z : starts) {
      if (z0 && cnt < cap) z0[cnt] = (int)sl.z_first + z;
      ++cnt;
    }
  }
  *n = cnt;
  if (z0 && cnt > cap) return set_err(STEN_EINVAL, "%d segments, room for %d", cnt, cap);
  return STEN_OK;
}

int sten_sr_segments(sten_stencil *st, int prec, int *z0, int cap, int *n) {
  if (!st || !n) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (st->srt[prec].by == 0) default_sr_tiling(st, prec);
  const SrTiling &t = st->srt[prec];
  int cnt = 0;
  for (const Slab &sl : st->slabs) {
    int nbig, zct;
    sr_chunks(t, sl.nz, &nbig, &zct);
    const int nch = nbig + (sl.nz - nbig * t.zc + zct - 1) / zct;
    for (int c = 0; c < nch; ++c, ++cnt) {
      int zc0;
      sr_chunk_z(t, nbig, zct, c, &zc0);
      if (z0 && cnt < cap) z0[cnt] = (int)sl.z_first + zc0;
    }
  }
  *n = cnt;
  if (z0 && cnt > cap) return set_err(STEN_EINVAL, "%d segments, room for %d", cnt, cap);
  return STEN_OK;
}

int sten_set_schedule(sten_stencil *st, int schedule) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  if (schedule != STEN_SCHED_CLASSIC && schedule != STEN_SCHED_SR)
    return set_err(STEN_EINVAL, "unknown schedule %d", schedule);
  st->schedule = schedule;
  return STEN_OK;
}

// ------------------------------------------- peer memory across ranks --
// export: IPC handles of this rank's bottom-slab and top-slab SR buffers
// (2 sets x 5 vectors each), of its inbox (sums, flags) and of the bottom- and
// top-slab coefficient arrays (6 fp32 + 6 fp16 each: a p2p-only communicator
// fills the coefficient halo planes from them at import)
constexpr int kIpcN = 56;  // SR vecs 2 x 10, inbox 2, coefficients 2 x 12, classic r p0 p1 v0 v1 2 x 5
int sten_p2p_export(sten_stencil *st, int prec, void *out, size_t *bytes) {
  if (!st || !bytes) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  const size_t need = sizeof(cudaIpcMemHandle_t) * kIpcN;
  if (!out) {
    *bytes = need;
    return STEN_OK;
  }
  if (*bytes < need) return set_err(STEN_EINVAL, "export buffer of %zu bytes, need %zu", *bytes, need);
  RC_TRY(ensure_bufs(st, prec));
  RC_TRY(ensure_sr(st, prec));
  cudaIpcMemHandle_t *h = (cudaIpcMemHandle_t *)out;
  int n = 0;
  for (Slab *sl : {&st->slabs.front(), &st->slabs.back()})
    for (int set = 0; set < 2; ++set)
      for (int i = 0; i < 5; ++i) CUDA_TRY(cudaIpcGetMemHandle(&h[n++], sl->sr[prec].vec[set][i]));
  CUDA_TRY(cudaIpcGetMemHandle(&h[n++], st->p2p_sums));
  CUDA_TRY(cudaIpcGetMemHandle(&h[n++], st->p2p_flags));
  for (Slab *sl : {&st->slabs.front(), &st->slabs.back()}) {
    for (int d = 0; d < 6; ++d) CUDA_TRY(cudaIpcGetMemHandle(&h[n++], sl->c32b[d]));
    for (int d = 0; d < 6; ++d) CUDA_TRY(cudaIpcGetMemHandle(&h[n++], sl->c16b[d]));
  }
  for (Slab *sl : {&st->slabs.front(), &st->slabs.back()}) {  // classic schedule: the halo'd vectors
    PrecBufs &b = sl->pb[prec];
    for (void *q : {b.r, b.p[0], b.p[1], b.v[0], b.v[1]}) CUDA_TRY(cudaIpcGetMemHandle(&h[n++], q));
  }
  *bytes = need;
  return STEN_OK;
}

// import: every rank's export in rank order (nranks x bytes_per_rank); opens the
// z-neighbours' buffers and the other ranks' inboxes, then selects the fused
// exchange across ranks
int sten_p2p_import(sten_stencil *st, int prec, const void *all, size_t bytes_per_rank) {
  if (!st || !all) return set_err(STEN_EINVAL, "NULL argument");
  if (!st->comm || st->comm->nranks < 2) return set_err(STEN_EINVAL, "p2p import needs a multi-rank communicator");
  if (bytes_per_rank < sizeof(cudaIpcMemHandle_t) * kIpcN) return set_err(STEN_EINVAL, "short export record");
  const int R = st->comm->nranks, me = st->comm->rank;
  if (R > kMaxPeers) return set_err(STEN_EUNSUPPORTED, "at most %d ranks in the peer-memory all-reduce", kMaxPeers);
  auto rec = [&](int r) { return (const cudaIpcMemHandle_t *)((const char *)all + (size_t)r * bytes_per_rank); };
  auto open = [&](const cudaIpcMemHandle_t &h, void **p) -> int {  // each handle opened once per handle
    std::string key((const char *)&h, sizeof h);
    auto it = st->ipc_map.find(key);
    if (it != st->ipc_map.end()) {
      *p = it->second;
      return STEN_OK;
    }
    cudaError_t e = cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_err(STEN_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    st->ipc_opened.push_back(*p);
    st->ipc_map[key] = *p;
    return STEN_OK;
  };
  for (int set = 0; set < 2; ++set)
    for (int i = 0; i < 5; ++i) {
      if (me > 0) RC_TRY(open(rec(me - 1)[10 + set * 5 + i], &st->p2p_lo[prec][set][i]));   // its top slab
      if (me + 1 < R) RC_TRY(open(rec(me + 1)[set * 5 + i], &st->p2p_hi[prec][set][i]));  // its bottom slab
    }
  for (int i = 0; i < 5; ++i) {  // classic: the lower rank's top slab, the upper rank's bottom slab
    if (me > 0) RC_TRY(open(rec(me - 1)[51 + i], &st->cls_lo[prec][i]));
    if (me + 1 < R) RC_TRY(open(rec(me + 1)[46 + i], &st->cls_hi[prec][i]));
  }
  st->p2p_remote.clear();
  for (int r = 0; r < R; ++r) {
    if (r == me) continue;
    P2PBox b;
    RC_TRY(open(rec(r)[20], (void **)&b.sums));
    RC_TRY(open(rec(r)[21], (void **)&b.flags));
    st->p2p_remote.push_back(b);
  }
  if (p2p_only(st)) {  // coefficient halo planes (NCCL fills them at create otherwise)
    const int ns = (int)st->slabs.size();
    Slab &bot = st->slabs[0], &top = st->slabs[ns - 1];
    for (int pr = 0; pr < 2; ++pr) {
      const size_t pb = (size_t)st->plane * (pr == 0 ? 4 : 2);
      for (int d = 0; d < 6; ++d) {
        const int k = pr * 6 + d;
        char *mine_b = pr == 0 ? (char *)bot.c32b[d] : (char *)bot.c16b[d];
        char *mine_t = pr == 0 ? (char *)top.c32b[d] : (char *)top.c16b[d];
        void *peer = nullptr;
        if (me > 0) {  // the lower rank's top slab: its top interior plane -> our bottom halo plane
          RC_TRY(open(rec(me - 1)[34 + k], &peer));
          CUDA_TRY(cudaMemcpy(mine_b, (char *)peer + (size_t)top.nz * pb, pb, cudaMemcpyDefault));
        }
        if (me + 1 < R) {  // the upper rank's bottom slab: its bottom interior plane -> our top halo plane
          RC_TRY(open(rec(me + 1)[22 + k], &peer));
          CUDA_TRY(cudaMemcpy(mine_t + (size_t)(top.nz + 1) * pb, (char *)peer + pb, pb, cudaMemcpyDefault));
        }
      }
    }
  }
  st->p2p_ranks = true;
  st->sr_p2p = true;
  drop_graphs(st);
  return STEN_OK;
}

int sten_set_sr_exchange(sten_stencil *st, int mode) {
  if (!st || mode < STEN_XCHG_SERIAL || mode > STEN_XCHG_FUSED) return set_err(STEN_EINVAL, "bad exchange mode");
  st->sr_p2p = mode == STEN_XCHG_FUSED;
  st->sr_overlap = mode == STEN_XCHG_OVERLAP;
  drop_graphs(st);
  return STEN_OK;
}

int sten_set_sr_chunks(sten_stencil *st, int prec, int zc, int tail_planes, int zc_tail) {
  if (!st || (prec != STEN_FP32 && prec != STEN_MIXED)) return set_err(STEN_EINVAL, "bad handle/precision");
  if (zc < 1 || tail_planes < 0 || (tail_planes > 0 && zc_tail < 1))
    return set_err(STEN_EINVAL, "bad SR chunk plan zc=%d tail_planes=%d zc_tail=%d", zc, tail_planes, zc_tail);
  if (st->srt[prec].by == 0) default_sr_tiling(st, prec);
  SrTiling &t = st->srt[prec];
  t.zc = zc;
  t.tail = tail_planes;
  t.zc_tail = tail_planes > 0 ? zc_tail : zc;
  drop_graphs(st);
  return ensure_bufs(st, prec) == STEN_OK ? ensure_sr(st, prec) : STEN_ECUDA;  // partial-sum capacity
}

int sten_set_sr_tiling(sten_stencil *st, int prec, int by, int stages, int cstages, int zc, int pack) {
  if (!st || (prec != STEN_FP32 && prec != STEN_MIXED)) return set_err(STEN_EINVAL, "bad handle/precision");
  if (st->srt[prec].by == 0) default_sr_tiling(st, prec);
  SrTiling t = st->srt[prec];
  if (by) t.by = by;
  if (stages) t.stages = stages;
  if (cstages) t.cstages = cstages;
  if (pack) t.pack = pack;
  if (zc) {  // an explicit chunk length: uniform chunks
    t.zc = zc;
    t.zc_tail = zc;
    t.tail = 0;
  }
  if (!sr_config_ok(t.by, t.stages, t.cstages, t.pack) || t.zc <= 0)
    return set_err(STEN_EINVAL, "unsupported SR tiling by=%d stages=%d cstages=%d zc=%d pack=%d", t.by, t.stages,
                   t.cstages, t.zc, t.pack);
  st->srt[prec] = t;
  for (Slab &sl : st->slabs) sl.sr[prec].maps_ok = false;
  drop_graphs(st);
  return STEN_OK;
}

int sten_classic_phase(sten_stencil *st, int prec, int phase, double alpha, double omega, double beta,
                       const void *r, const void *p, const void *v, const void *rh, void *out0, void *out1,
                       float *dots, void *cuda_stream) {
  if (!st || !r || !v || !out0 || !out1 || !dots) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (phase != 1 && phase != 2) return set_err(STEN_EINVAL, "phase %d is not 1 (H1) or 2 (H2)", phase);
  if (phase == 1 && (!p || !rh)) return set_err(STEN_EINVAL, "H1 needs p and rh");
  if (p2p_only(st)) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: sten_classic_phase needs NCCL");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  RC_TRY(ensure_bufs(st, prec));
  st->launches = 0;
  DevState h;
  memset(&h, 0, sizeof h);
  h.alpha = (float)alpha;
  h.omega = (float)omega;
  h.beta = (float)beta;
  h.maxit = 1;
  h.ev = -1;
  h.half = prec == STEN_MIXED;
  *st->st_host = h;
  CUDA_TRY(cudaMemcpyAsync(st->st, st->st_host, sizeof h, cudaMemcpyHostToDevice, s));
  const int ns = (int)st->slabs.size();
  const int mode = phase == 1 ? MODE_H1 : MODE_H2;
  RC_TRY(copy_in(st, prec, [](PrecBufs &b) -> void * { return b.r; }, r, s));
  if (phase == 1) {
    RC_TRY(copy_in(st, prec, [](PrecBufs &b) -> void * { return b.p[0]; }, p, s));
    RC_TRY(copy_in(st, prec, [](PrecBufs &b) -> void * { return b.v[0]; }, v, s));
    RC_TRY(copy_in(st, prec, [](PrecBufs &b) -> void * { return b.rh; }, rh, s));
  } else {
    RC_TRY(copy_in(st, prec, [](PrecBufs &b) -> void * { return b.v[1]; }, v, s));
  }
  auto xchg = [&](cudaStream_t ss) {
    if (phase == 1) {
      RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.r; }, ss));
      RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.p[0]; }, ss));
      return exchange(st, prec, [](PrecBufs &b) { return b.v[0]; }, ss);
    }
    // H2 also reads r at the neighbours (s = r - alpha v); a solve exchanged it before H1
    RC_TRY(exchange(st, prec, [](PrecBufs &b) { return b.r; }, ss));
    return exchange(st, prec, [](PrecBufs &b) { return b.v[1]; }, ss);
  };
  int nslots = ns;
  if (cls_overlapped(st)) {
    RC_TRY(overlapped_phase(st, prec, mode, 0, s, xchg, false));
    nslots = 3 * ns;
  } else {
    if (decomposed(st)) RC_TRY(xchg(s));
    for (int k = 0; k < ns; ++k) RC_TRY(launch_stencil(st, prec, mode, k, 0, s, CLS_ALL, true));
  }
  KLAUNCH(slabsum_launch(st->slab_sums, nslots, st->red_total, s));
  if (nccl_ranks(st))
    NCCL_TRY(g_nccl.AllReduce(st->red_total, st->red_total, kMaxDots, ncclFloat32, ncclSum, st->comm->comm, s));
  if (phase == 1) {
    RC_TRY(copy_out(st, prec, [](PrecBufs &b) -> void * { return b.p[1]; }, out0, s));
    RC_TRY(copy_out(st, prec, [](PrecBufs &b) -> void * { return b.v[1]; }, out1, s));
  } else {
    RC_TRY(copy_out(st, prec, sel_s, out0, s));
    RC_TRY(copy_out(st, prec, sel_t, out1, s));
  }
  CUDA_TRY(cudaMemcpyAsync(dots, st->red_total, sizeof(float) * (phase == 1 ? 1 : 2), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return STEN_OK;
}

int sten_sr_sweep(sten_stencil *st, int prec, double alpha, double omega, double beta, const void *rh, void *x,
                  void *r, void *p, void *v, void *q, void *y, float *dots, void *cuda_stream) {
  if (!st || !rh || !x || !r || !p || !v || !q || !y || !dots) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (p2p_only(st)) return set_err(STEN_EUNSUPPORTED, "p2p-only communicator: sten_sr_sweep needs NCCL");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  RC_TRY(ensure_bufs(st, prec));
  RC_TRY(ensure_sr(st, prec));
  st->launches = 0;
  DevState h;
  memset(&h, 0, sizeof h);
  h.alpha = (float)alpha;
  h.omega = (float)omega;
  h.beta = (float)beta;
  h.maxit = 1;
  h.ev = -1;
  h.half = prec == STEN_MIXED;
  *st->st_host = h;
  CUDA_TRY(cudaMemcpyAsync(st->st, st->st_host, sizeof h, cudaMemcpyHostToDevice, s));
  void *user[5] = {r, p, v, q, y};
  for (int i = 0; i < 5; ++i)
    RC_TRY(sr_copy_in(st, prec, [prec, i](Slab &sl) { return sl.sr[prec].vec[0][i]; }, user[i], s));
  RC_TRY(sr_copy_in(st, prec, [prec](Slab &sl) { return sl.sr[prec].x; }, x, s));
  RC_TRY(sr_copy_in(st, prec, [prec](Slab &sl) { return sl.sr[prec].rh; }, rh, s));
  if (decomposed(st)) RC_TRY(sr_exchange(st, prec, 0, s));
  const int ns = (int)st->slabs.size();
  for (int k = 0; k < ns; ++k) RC_TRY(launch_sr(st, prec, k, 0, true, s));
  float *sums = st->slab_sums;
  if (nccl_ranks(st)) {
    KLAUNCH(slabsum_launch(st->slab_sums, ns, st->red_total, s));
    NCCL_TRY(g_nccl.AllReduce(st->red_total, st->red_total, kMaxDots, ncclFloat32, ncclSum, st->comm->comm, s));
    sums = st->red_total;
  } else if (ns > 1) {
    KLAUNCH(slabsum_launch(st->slab_sums, ns, st->red_total, s));
    sums = st->red_total;
  }
  for (int i = 0; i < 5; ++i)
    RC_TRY(sr_copy_out(st, prec, [prec, i](Slab &sl) { return sl.sr[prec].vec[1][i]; }, user[i], s));
  RC_TRY(sr_copy_out(st, prec, [prec](Slab &sl) { return sl.sr[prec].x; }, x, s));
  CUDA_TRY(cudaMemcpyAsync(dots, sums, sizeof(float) * 12, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  return STEN_OK;
}

}  // extern "C"

// ====================================================== 2D 9-point SpMV ==
// NEXT-3 of SURVEY §8(f): the paper's second kernel, its
// tiled output-halo form (R24) and BiCGStab around it (R25).
struct Bufs2 {
  bool ready = false;
  void *x = nullptr, *r = nullptr, *rh = nullptr, *p[2] = {}, *v[2] = {}, *s = nullptr, *t = nullptr, *bw = nullptr;
  CUtensorMap m_x, m_r, m_p[2], m_v[2];
  CUtensorMap m_pa[2], m_sa;  // the tiled solve's SpMV inputs p', s (k_apply9 boxes)
};
struct sten_stencil2d {
  int nx = 0, ny = 0, pitch = 0;
  int sm = 148;
  bool has_diag = false;
  float *c32[8] = {};
  __half *c16[8] = {};
  double *aP = nullptr;            // a_P per point (padding 1) when a diagonal was given (R3)
  void *v[2] = {}, *u[2] = {};     // stencil2d_apply, per precision: pitched input / output
  bool maps_ok[2] = {false, false};
  CUtensorMap m_v[2];
  // tiled (output-halo) SpMV, R24
  int TX = 1, TY = 1, HS = 0, WS = 0;
  unsigned char *xm = nullptr, *ym = nullptr;
  void *ring = nullptr;
  // bicgstab2d_solve
  Bufs2 sb[2];
  DevState *st = nullptr, *st_host = nullptr;
  float *partials = nullptr;
  int partials_cap = 0;
  unsigned *counter = nullptr;
  double *hist = nullptr;
  float *ahist = nullptr, *whist = nullptr;
  int hist_cap = 0;
  cudaStream_t cap = nullptr;
  std::map<GraphKey, GraphRec> graphs;
  bool timing = false;
  double ph_ms[3] = {0, 0, 0};
  long long ph_n = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double last_ms = 0.0;
};

static int bx2d(int prec) { return prec == STEN_FP32 ? 64 : 128; }

static int create2d_impl(int nx, int ny, const void *const coeffs[9], int dtype, cudaStream_t s,
                         sten_stencil2d **out) {
  if (!out || !coeffs) return set_err(STEN_EINVAL, "NULL argument");
  if (nx <= 0 || ny <= 0 || nx > (1 << 24) || ny > (1 << 24)) return set_err(STEN_EINVAL, "bad 2D mesh %d x %d", nx, ny);
  for (int d = 1; d < 9; ++d)
    if (!coeffs[d]) return set_err(STEN_EINVAL, "coeffs[%d] is NULL", d);
  if (dtype != STEN_DT_F64 && dtype != STEN_DT_F32) return set_err(STEN_EINVAL, "coeff_dtype %d unsupported", dtype);
  sten_stencil2d *st = new sten_stencil2d;
  st->nx = nx;
  st->ny = ny;
  st->pitch = (nx + 63) / 64 * 64;  // 128-B rows (fp16), like the 3D layout
  st->has_diag = coeffs[0] != nullptr;
  st->sm = device_sm_count();
  auto fail = [&](int rc) {
    stencil2d_destroy(st);
    return rc;
  };
  const size_t n = (size_t)nx * ny, ein = dtype == STEN_DT_F64 ? 8 : 4;
  const size_t cells = (size_t)st->pitch * ny;
  std::vector<void *> staged(9, nullptr);
  const void *dev[9];
  for (int d = 0; d < 9; ++d) {
    dev[d] = coeffs[d];
    if (coeffs[d] && !ptr_on_device(coeffs[d])) {
      if (cudaMalloc(&staged[d], n * ein) != cudaSuccess) {
        for (void *p : staged) cudaFree(p);
        return fail(set_err(STEN_ENOMEM, "staging 2D coefficients failed"));
      }
      cudaMemcpyAsync(staged[d], coeffs[d], n * ein, cudaMemcpyHostToDevice, s);
      dev[d] = staged[d];
    }
  }
  Coef9In in;
  Coef9Out co;
  int rc = STEN_OK;
  for (int d = 0; d < 8 && rc == STEN_OK; ++d) {
    in.off[d] = dev[d + 1];
    if (cudaMalloc(&st->c32[d], cells * 4) != cudaSuccess || cudaMalloc(&st->c16[d], cells * 2) != cudaSuccess)
      rc = set_err(STEN_ENOMEM, "2D coefficient allocation failed");
    co.c32[d] = st->c32[d];
    co.c16[d] = st->c16[d];
  }
  if (rc == STEN_OK && st->has_diag && cudaMalloc(&st->aP, cells * 8) != cudaSuccess)
    rc = set_err(STEN_ENOMEM, "2D a_P allocation failed");
  if (rc == STEN_OK) {
    int e = create9_launch(dtype, dev[0], in, nx, ny, st->pitch, co, st->aP, s);
    if (e) rc = set_err(STEN_ECUDA, "2D coefficient kernel: %s", cudaGetErrorString((cudaError_t)e));
  }
  if (rc == STEN_OK && cudaStreamSynchronize(s) != cudaSuccess) rc = set_err(STEN_ECUDA, "stencil2d_create sync failed");
  for (void *p : staged) cudaFree(p);
  if (rc != STEN_OK) return fail(rc);
  if (cudaEventCreate(&st->e0) != cudaSuccess || cudaEventCreate(&st->e1) != cudaSuccess)
    return fail(set_err(STEN_ECUDA, "event creation failed"));
  *out = st;
  return STEN_OK;
}

static void drop_graphs2d(sten_stencil2d *st) {
  for (auto &kv : st->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    for (auto e : kv.second.ev) cudaEventDestroy(e);
  }
  st->graphs.clear();
}

// one (nx, ny) map over a pitched plane, box (BX + 2H) x (BY + 2)
static constexpr int kApply9BY = 32;  // rows per k_apply9 tile (apply9_launch)
static int map2d(const sten_stencil2d *st, CUtensorMap *m, void *base, int prec, int by) {
  const int e = esize(prec), H = 16 / e;
  return make_map_p(m, base, e, st->nx, st->ny, 1, st->pitch, (long long)st->pitch * st->ny, 3, bx2d(prec) + 2 * H,
                    by + 2);
}

// The apply path's SpMV: gather (1 x 1 tiles) or the tiled output-halo form.
static int launch_apply2d(sten_stencil2d *st, int prec, const CUtensorMap &mv, const void *v, void *u,
                          cudaStream_t s) {
  Apply9Args a;
  memset(&a, 0, sizeof a);
  a.tm_v = mv;
  for (int d = 0; d < 8; ++d) a.c[d] = prec == STEN_FP32 ? (const void *)st->c32[d] : (const void *)st->c16[d];
  a.u = u;
  a.nx = st->nx;
  a.ny = st->ny;
  a.pitch = st->pitch;
  a.tiles_x = (st->nx + bx2d(prec) - 1) / bx2d(prec);
  const bool tiled = st->TX * st->TY > 1;
  if (tiled) {
    a.xm = st->xm;
    a.ym = st->ym;
  }
  if (prec == STEN_FP32) KLAUNCH(apply9_launch<float>(a, s));
  else KLAUNCH(apply9_launch<__half>(a, s));
  if (!tiled) return STEN_OK;
  Ring9Args r;
  memset(&r, 0, sizeof r);
  for (int d = 0; d < 8; ++d) r.c[d] = a.c[d];
  r.v = v;
  r.u = u;
  r.ring = st->ring;
  r.nx = st->nx;
  r.ny = st->ny;
  r.pitch = st->pitch;
  r.TX = st->TX;
  r.TY = st->TY;
  r.HS = st->HS;
  r.WS = st->WS;
  if (prec == STEN_FP32) KLAUNCH(ring9_launch<float>(r, s));
  else KLAUNCH(ring9_launch<__half>(r, s));
  for (int dir = 0; dir < 2; ++dir) {
    if ((dir == 0 ? st->TX : st->TY) == 1) continue;
    if (prec == STEN_FP32) KLAUNCH(round9_launch<float>(r, dir, s));
    else KLAUNCH(round9_launch<__half>(r, dir, s));
  }
  return STEN_OK;
}

// ----------------------------------------------------- 2D solve plumbing --
static int ensure2d(sten_stencil2d *st, int prec) {
  Bufs2 &b = st->sb[prec];
  const size_t bytes = (size_t)st->pitch * st->ny * esize(prec);
  if (!b.ready) {
    void **all[] = {&b.x, &b.r, &b.rh, &b.p[0], &b.p[1], &b.v[0], &b.v[1], &b.s, &b.t, &b.bw};
    for (void **pp : all) {
      if (!*pp) {
        cudaError_t e = cudaMalloc(pp, bytes);
        if (e != cudaSuccess) return set_err(STEN_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
      }
      CUDA_TRY(cudaMemset(*pp, 0, bytes));  // row padding stays zero (the element-wise kernels stream it)
    }
    RC_TRY(map2d(st, &b.m_x, b.x, prec, kApply9BY));  // A x0 by k_apply9
    RC_TRY(map2d(st, &b.m_r, b.r, prec, kBicg9BY));
    for (int k = 0; k < 2; ++k) {
      RC_TRY(map2d(st, &b.m_p[k], b.p[k], prec, kBicg9BY));
      RC_TRY(map2d(st, &b.m_v[k], b.v[k], prec, kBicg9BY));
      RC_TRY(map2d(st, &b.m_pa[k], b.p[k], prec, kApply9BY));
    }
    RC_TRY(map2d(st, &b.m_sa, b.s, prec, kApply9BY));
    b.ready = true;
  }
  if (!st->st) {
    CUDA_TRY(cudaMalloc(&st->st, sizeof(DevState)));
    CUDA_TRY(cudaMallocHost(&st->st_host, sizeof(DevState)));
    CUDA_TRY(cudaMalloc(&st->counter, 2 * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(st->counter, 0, 2 * sizeof(unsigned)));
    CUDA_TRY(cudaStreamCreateWithFlags(&st->cap, cudaStreamNonBlocking));
  }
  const int tiles = ((st->nx + bx2d(STEN_FP32) - 1) / bx2d(STEN_FP32)) * ((st->ny + kBicg9BY - 1) / kBicg9BY);
  int need = tiles > st->sm * 64 ? tiles : st->sm * 64;  // the stencil grid and the element-wise grid
  if (need > st->partials_cap) {
    cudaFree(st->partials);
    st->partials = nullptr;
    CUDA_TRY(cudaMalloc(&st->partials, (size_t)need * kMaxDots * sizeof(float)));
    st->partials_cap = need;
    drop_graphs2d(st);
  }
  return STEN_OK;
}

static Reduce red2d(sten_stencil2d *st) {
  Reduce r;
  memset(&r, 0, sizeof r);
  r.partials = st->partials;
  r.counter = st->counter;
  r.st = st->st;
  return r;
}

static int ew_grid2d(const sten_stencil2d *st, long long nvec) {
  long long need = (nvec + 511) / 512, g = (long long)st->sm * 64;
  if (need < g) g = need;
  return (int)(g < 1 ? 1 : g);
}

static int ew2d(sten_stencil2d *st, int prec, EwArgs &a) {
  a.rows = st->ny;
  a.vpr = (st->nx + (prec == STEN_FP32 ? 4 : 8) - 1) / (prec == STEN_FP32 ? 4 : 8);
  a.pitch = st->pitch;
  a.nvec = (long long)st->pitch * st->ny / (prec == STEN_FP32 ? 4 : 8);
  a.red = red2d(st);
  return ew_grid2d(st, a.nvec);
}

// one iteration of Alg. 1: H1, H2 (k_bicg9), H3 (k_h3); p / v ping-pong on `parity`
// the tiled solve's iteration (TX x TY > 1): unfused updates and dots around the tiled SpMV
static int enqueue_iter2d_tiled(sten_stencil2d *st, int prec, int parity, cudaStream_t s, cudaEvent_t *evs) {
  Bufs2 &b = st->sb[prec];
  const int cur = parity, nxt = parity ^ 1;
  const long long nvec = (long long)st->pitch * st->ny / (prec == STEN_FP32 ? 4 : 8);
  const int g = ew_grid2d(st, nvec);
  Upd9Args u;
  Dot9Args d;
  memset(&u, 0, sizeof u);
  memset(&d, 0, sizeof d);
  u.nvec = d.nvec = nvec;
  u.st = st->st;
  d.red = red2d(st);
  // H1: p' = r + beta (p - omega v), v' = A p' (tiled), (rhat, v')
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
  u.r = b.r;
  u.p = b.p[cur];
  u.v = b.v[cur];
  u.out = b.p[nxt];
  if (prec == STEN_FP32) KLAUNCH(upd9_launch<float>(MODE_H1, u, g, s));
  else KLAUNCH(upd9_launch<__half>(MODE_H1, u, g, s));
  RC_TRY(launch_apply2d(st, prec, b.m_pa[nxt], b.p[nxt], b.v[nxt], s));
  d.a0 = b.rh;
  d.b0 = b.v[nxt];
  if (prec == STEN_FP32) KLAUNCH(dot9_launch<float>(MODE_H1, d, g, s));
  else KLAUNCH(dot9_launch<__half>(MODE_H1, d, g, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
  // H2: s = r - alpha v', t = A s (tiled), (t, s), (t, t)
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[2], s, cudaEventRecordExternal));
  u.p = nullptr;
  u.v = b.v[nxt];
  u.out = b.s;
  if (prec == STEN_FP32) KLAUNCH(upd9_launch<float>(MODE_H2, u, g, s));
  else KLAUNCH(upd9_launch<__half>(MODE_H2, u, g, s));
  RC_TRY(launch_apply2d(st, prec, b.m_sa, b.s, b.t, s));
  d.a0 = b.t;
  d.b0 = b.s;
  if (prec == STEN_FP32) KLAUNCH(dot9_launch<float>(MODE_H2, d, g, s));
  else KLAUNCH(dot9_launch<__half>(MODE_H2, d, g, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[3], s, cudaEventRecordExternal));
  // H3: the element-wise x, r updates and (rhat, r), (r, r)
  EwArgs e;
  memset(&e, 0, sizeof e);
  e.x = b.x;
  e.p = b.p[nxt];
  e.s = b.s;
  e.t = b.t;
  e.rhat = b.rh;
  e.xo = b.x;
  e.ro = b.r;
  const int g3 = ew2d(st, prec, e);
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[4], s, cudaEventRecordExternal));
  if (prec == STEN_FP32) KLAUNCH(h3_launch<float>(e, g3, 256, s));
  else KLAUNCH(h3_launch<__half>(e, g3, 256, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[5], s, cudaEventRecordExternal));
  return STEN_OK;
}

static int enqueue_iter2d(sten_stencil2d *st, int prec, int parity, cudaStream_t s, cudaEvent_t *evs) {
  if (st->TX * st->TY > 1) return enqueue_iter2d_tiled(st, prec, parity, s, evs);
  Bufs2 &b = st->sb[prec];
  const int cur = parity, nxt = parity ^ 1;
  Bicg9Args a;
  memset(&a, 0, sizeof a);
  for (int d = 0; d < 8; ++d) a.c[d] = prec == STEN_FP32 ? (const void *)st->c32[d] : (const void *)st->c16[d];
  a.nx = st->nx;
  a.ny = st->ny;
  a.pitch = st->pitch;
  a.tiles_x = (st->nx + bx2d(prec) - 1) / bx2d(prec);
  a.tiles_y = (st->ny + kBicg9BY - 1) / kBicg9BY;
  a.red = red2d(st);
  // H1
  a.tm_in[0] = b.m_r;
  a.tm_in[1] = b.m_p[cur];
  a.tm_in[2] = b.m_v[cur];
  a.rh = b.rh;
  a.out0 = b.v[nxt];
  a.out1 = b.p[nxt];
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[0], s, cudaEventRecordExternal));
  if (prec == STEN_FP32) KLAUNCH(bicg9_launch<float>(MODE_H1, a, s));
  else KLAUNCH(bicg9_launch<__half>(MODE_H1, a, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[1], s, cudaEventRecordExternal));
  // H2
  a.tm_in[0] = b.m_r;
  a.tm_in[1] = b.m_v[nxt];
  a.rh = nullptr;
  a.out0 = b.t;
  a.out1 = b.s;
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[2], s, cudaEventRecordExternal));
  if (prec == STEN_FP32) KLAUNCH(bicg9_launch<float>(MODE_H2, a, s));
  else KLAUNCH(bicg9_launch<__half>(MODE_H2, a, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[3], s, cudaEventRecordExternal));
  // H3
  EwArgs e;
  memset(&e, 0, sizeof e);
  e.x = b.x;
  e.p = b.p[nxt];
  e.s = b.s;
  e.t = b.t;
  e.rhat = b.rh;
  e.xo = b.x;
  e.ro = b.r;
  const int g = ew2d(st, prec, e);
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[4], s, cudaEventRecordExternal));
  if (prec == STEN_FP32) KLAUNCH(h3_launch<float>(e, g, 256, s));
  else KLAUNCH(h3_launch<__half>(e, g, 256, s));
  if (evs) CUDA_TRY(cudaEventRecordWithFlags(evs[5], s, cudaEventRecordExternal));
  return STEN_OK;
}

static int graph2d(sten_stencil2d *st, int prec, int chunk, GraphRec **out) {
  GraphKey key{prec, chunk, st->timing ? 1 : 0, st->TX * st->TY > 1 ? 1 : 0};
  auto it = st->graphs.find(key);
  if (it != st->graphs.end()) {
    *out = &it->second;
    return STEN_OK;
  }
  GraphRec rec;
  if (st->timing) {
    rec.ev.resize((size_t)chunk * 6);
    for (auto &e : rec.ev) CUDA_TRY(cudaEventCreate(&e));
  }
  CUDA_TRY(cudaStreamBeginCapture(st->cap, cudaStreamCaptureModeThreadLocal));
  int rc = STEN_OK;
  for (int j = 0; j < chunk && rc == STEN_OK; ++j)
    rc = enqueue_iter2d(st, prec, j & 1, st->cap, st->timing ? &rec.ev[(size_t)j * 6] : nullptr);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(st->cap, &g);
  if (rc != STEN_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess) return set_err(STEN_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&rec.exec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return set_err(STEN_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
  rec.kernels = 3LL * chunk;
  auto ins = st->graphs.emplace(key, rec);
  *out = &ins.first->second;
  return STEN_OK;
}

static int copy2d_in(sten_stencil2d *st, int prec, void *dst, const void *src, cudaStream_t s) {
  const size_t e = esize(prec);
  CUDA_TRY(cudaMemcpy2DAsync(dst, st->pitch * e, src, st->nx * e, st->nx * e, st->ny, cudaMemcpyDefault, s));
  return STEN_OK;
}
static int copy2d_out(sten_stencil2d *st, int prec, void *dst, const void *src, cudaStream_t s) {
  const size_t e = esize(prec);
  CUDA_TRY(cudaMemcpy2DAsync(dst, st->nx * e, src, st->pitch * e, st->nx * e, st->ny, cudaMemcpyDefault, s));
  return STEN_OK;
}

extern "C" {

int stencil2d_create(int nx, int ny, const void *const coeffs[9], int coeff_dtype, void *cuda_stream,
                     sten_stencil2d **out) {
  return create2d_impl(nx, ny, coeffs, coeff_dtype, (cudaStream_t)cuda_stream, out);
}

void stencil2d_destroy(sten_stencil2d *st) {
  if (!st) return;
  if (st->st) cudaDeviceSynchronize();  // graphs / kernels of this handle may still run
  drop_graphs2d(st);
  for (int d = 0; d < 8; ++d) {
    cudaFree(st->c32[d]);
    cudaFree(st->c16[d]);
  }
  cudaFree(st->aP);
  for (int p = 0; p < 2; ++p) {
    cudaFree(st->v[p]);
    cudaFree(st->u[p]);
    Bufs2 &b = st->sb[p];
    for (void *q : {b.x, b.r, b.rh, b.p[0], b.p[1], b.v[0], b.v[1], b.s, b.t, b.bw}) cudaFree(q);
  }
  cudaFree(st->xm);
  cudaFree(st->ym);
  cudaFree(st->ring);
  cudaFree(st->st);
  if (st->st_host) cudaFreeHost(st->st_host);
  cudaFree(st->partials);
  cudaFree(st->counter);
  cudaFree(st->hist);
  cudaFree(st->ahist);
  cudaFree(st->whist);
  if (st->cap) cudaStreamDestroy(st->cap);
  if (st->e0) cudaEventDestroy(st->e0);
  if (st->e1) cudaEventDestroy(st->e1);
  delete st;
}

int stencil2d_set_tiles(sten_stencil2d *st, int tiles_x, int tiles_y) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  if (tiles_x < 1 || tiles_y < 1 || tiles_x > st->nx || tiles_y > st->ny)
    return set_err(STEN_EINVAL, "tiles %d x %d: need 1 <= tiles_x <= nx = %d, 1 <= tiles_y <= ny = %d", tiles_x, tiles_y,
                   st->nx, st->ny);
  CUDA_TRY(cudaDeviceSynchronize());
  drop_graphs2d(st);  // captured solves hold the old tiling's pointers
  cudaFree(st->xm);
  cudaFree(st->ym);
  cudaFree(st->ring);
  st->xm = st->ym = nullptr;
  st->ring = nullptr;
  st->TX = st->TY = 1;
  if (tiles_x * (long long)tiles_y == 1) return STEN_OK;
  // per column / row: is the -1 (bit 0) / +1 (bit 1) neighbour in the same tile (R24)
  auto flags = [](int n, int t, int len) {
    std::vector<unsigned char> f((size_t)len, 0);
    for (int a = 0; a < t; ++a) {
      const int lo = (int)((long long)a * n / t), hi = (int)((long long)(a + 1) * n / t);
      for (int x = lo; x < hi; ++x) f[x] = (unsigned char)((x - 1 >= lo ? 1 : 0) | (x + 1 < hi ? 2 : 0));
    }
    return f;
  };
  const std::vector<unsigned char> fx = flags(st->nx, tiles_x, st->pitch), fy = flags(st->ny, tiles_y, st->ny);
  const int HS = (st->ny + tiles_y - 1) / tiles_y + 2, WS = (st->nx + tiles_x - 1) / tiles_x;
  const size_t ring_elems = (size_t)tiles_x * tiles_y * (2 * (size_t)HS + 2 * (size_t)WS);
  if (cudaMalloc(&st->xm, fx.size()) != cudaSuccess || cudaMalloc(&st->ym, fy.size()) != cudaSuccess ||
      cudaMalloc(&st->ring, ring_elems * 4) != cudaSuccess)
    return set_err(STEN_ENOMEM, "tile masks / output-halo ring (%zu elements)", ring_elems);
  CUDA_TRY(cudaMemcpy(st->xm, fx.data(), fx.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(st->ym, fy.data(), fy.size(), cudaMemcpyHostToDevice));
  st->TX = tiles_x;
  st->TY = tiles_y;
  st->HS = HS;
  st->WS = WS;
  return STEN_OK;
}

int stencil2d_apply(sten_stencil2d *st, int prec, const void *x, void *y, void *cuda_stream) {
  if (!st || !x || !y) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int e = esize(prec);
  const size_t bytes = (size_t)st->pitch * st->ny * e;
  if (!st->v[prec]) {
    CUDA_TRY(cudaMalloc(&st->v[prec], bytes));
    CUDA_TRY(cudaMalloc(&st->u[prec], bytes));
    CUDA_TRY(cudaMemset(st->v[prec], 0, bytes));  // padding columns stay zero
  }
  if (!st->maps_ok[prec]) {
    RC_TRY(map2d(st, &st->m_v[prec], st->v[prec], prec, kApply9BY));
    st->maps_ok[prec] = true;
  }
  RC_TRY(copy2d_in(st, prec, st->v[prec], x, s));
  CUDA_TRY(cudaEventRecord(st->e0, s));
  RC_TRY(launch_apply2d(st, prec, st->m_v[prec], st->v[prec], st->u[prec], s));
  CUDA_TRY(cudaEventRecord(st->e1, s));
  RC_TRY(copy2d_out(st, prec, y, st->u[prec], s));
  CUDA_TRY(cudaStreamSynchronize(s));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, st->e0, st->e1));
  st->last_ms = ms;
  return STEN_OK;
}

int stencil2d_last_ms(sten_stencil2d *st, double *ms) {
  if (!st || !ms) return set_err(STEN_EINVAL, "NULL argument");
  *ms = st->last_ms;
  return STEN_OK;
}

int stencil2d_set_timing(sten_stencil2d *st, int enable) {
  if (!st) return set_err(STEN_EINVAL, "NULL handle");
  st->timing = enable != 0;
  return STEN_OK;
}

int stencil2d_phase_ms(sten_stencil2d *st, double ms[3], long long *iterations) {
  if (!st || !ms || !iterations) return set_err(STEN_EINVAL, "NULL argument");
  for (int p = 0; p < 3; ++p) ms[p] = st->ph_n ? st->ph_ms[p] / (double)st->ph_n : 0.0;
  *iterations = st->ph_n;
  return STEN_OK;
}

int bicgstab2d_solve(sten_stencil2d *st, int prec, const void *b, const void *x0, double tol, int maxit, void *x_out,
                     int *iters, double *res_hist, int *status, void *cuda_stream) {
  if (!st || !b || !x_out || !iters || !res_hist || !status) return set_err(STEN_EINVAL, "NULL argument");
  if (prec != STEN_FP32 && prec != STEN_MIXED) return set_err(STEN_EINVAL, "bad precision %d", prec);
  if (!(tol >= 0.0) || !std::isfinite(tol) || maxit < 0) return set_err(STEN_EINVAL, "tol=%g maxit=%d invalid", tol, maxit);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  RC_TRY(ensure2d(st, prec));
  Bufs2 &bf = st->sb[prec];
  if (maxit + 2 > st->hist_cap) {
    cudaFree(st->hist);
    cudaFree(st->ahist);
    cudaFree(st->whist);
    st->hist = nullptr;
    st->ahist = st->whist = nullptr;
    st->hist_cap = maxit + 2 < 64 ? 64 : maxit + 2;
    CUDA_TRY(cudaMalloc(&st->hist, sizeof(double) * st->hist_cap));
    CUDA_TRY(cudaMalloc(&st->ahist, sizeof(float) * st->hist_cap));
    CUDA_TRY(cudaMalloc(&st->whist, sizeof(float) * st->hist_cap));
  }
  DevState h;
  memset(&h, 0, sizeof h);
  h.tol = tol;
  h.maxit = maxit;
  h.status = -1;
  h.ev = -1;
  h.half = prec == STEN_MIXED;
  h.hist = st->hist;
  h.ahist = st->ahist;
  h.whist = st->whist;
  *st->st_host = h;
  CUDA_TRY(cudaMemcpyAsync(st->st, st->st_host, sizeof h, cudaMemcpyHostToDevice, s));
  RC_TRY(copy2d_in(st, prec, bf.bw, b, s));
  CUDA_TRY(cudaEventRecord(st->e0, s));
  // S1 (Alg. 1 l.174, R1, R3): r0 = b_hat - A x0, rhat = p0 = r0, v0 = 0
  if (x0) {
    RC_TRY(copy2d_in(st, prec, bf.x, x0, s));
    RC_TRY(launch_apply2d(st, prec, bf.m_x, bf.x, bf.t, s));  // A x0 into t (the handle's SpMV form)
  } else {
    CUDA_TRY(cudaMemsetAsync(bf.x, 0, (size_t)st->pitch * st->ny * esize(prec), s));
  }
  EwArgs e;
  memset(&e, 0, sizeof e);
  e.bw = bf.bw;
  e.aP = st->aP;
  e.ax = x0 ? bf.t : nullptr;
  e.r = bf.r;
  e.rh = bf.rh;
  e.p0 = bf.p[0];
  e.v0 = bf.v[0];
  const int g = ew2d(st, prec, e);
  if (g > st->partials_cap) return set_err(STEN_ECUDA, "internal: element-wise grid exceeds the partial-sum buffer");
  if (prec == STEN_FP32) KLAUNCH(init_launch<float>(e, g, 256, s));
  else KLAUNCH(init_launch<__half>(e, g, 256, s));
  // iterations: graphs of `chunk` iterations (even: the p / v parity repeats)
  if (maxit > 0) {
    int chunk = tol > 0.0 ? 8 : ((maxit + 1) / 2) * 2;
    if (chunk > 2048) chunk = 2048;
    GraphRec *gr = nullptr;
    RC_TRY(graph2d(st, prec, chunk, &gr));
    if (st->timing) {
      st->ph_ms[0] = st->ph_ms[1] = st->ph_ms[2] = 0.0;
      st->ph_n = 0;
    }
    const int nrep = (maxit + chunk - 1) / chunk;
    for (int rep = 0; rep < nrep; ++rep) {
      CUDA_TRY(cudaGraphLaunch(gr->exec, s));
      if (tol > 0.0 || st->timing) {
        CUDA_TRY(cudaMemcpyAsync(st->st_host, st->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (st->timing) {
          const int done = st->st_host->it;
          for (int j = 0; j < chunk && rep * chunk + j < done; ++j) {
            for (int p = 0; p < 3; ++p) {
              float ms = 0.f;
              CUDA_TRY(cudaEventElapsedTime(&ms, gr->ev[(size_t)j * 6 + 2 * p], gr->ev[(size_t)j * 6 + 2 * p + 1]));
              st->ph_ms[p] += ms;
            }
            st->ph_n += 1;
          }
        }
        if (st->st_host->stop || st->st_host->it >= maxit) break;
      }
    }
  }
  CUDA_TRY(cudaEventRecord(st->e1, s));
  CUDA_TRY(cudaMemcpyAsync(st->st_host, st->st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const DevState fin = *st->st_host;
  if (fin.zero_x) CUDA_TRY(cudaMemsetAsync(bf.x, 0, (size_t)st->pitch * st->ny * esize(prec), s));
  RC_TRY(copy2d_out(st, prec, x_out, bf.x, s));
  CUDA_TRY(cudaMemcpyAsync(res_hist, st->hist, sizeof(double) * (fin.it + 1), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaGetLastError());
  *iters = fin.it;
  *status = fin.stop ? fin.status : (fin.ev >= 0 ? fin.ev : STEN_MAXIT);
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, st->e0, st->e1));
  st->last_ms = ms;
  return STEN_OK;
}

}  // extern "C"
