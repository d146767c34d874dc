// C ABI of the B200 RANS step path (declared in include/citywind_b200.h).
// Host orchestration: one context per grid owns the workspace, the operator
// code field, the device report ring and the error latch; cw_step enqueues
// whole steps (no host synchronisation inside a step or between steps).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/citywind_b200.h"
#include "cw_common.cuh"
#include "cw_pcg.cuh"
#include "cw_step.cuh"
#include "cw_aux.cuh"

using namespace cw;

static thread_local std::string g_err;
static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CW_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(CW_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

static constexpr int TX = PCG_TX, TY = PCG_TY;
static constexpr int RING = 4096;

struct cw_ctx {
  int prec = 4;
  int device = 0;
  int num_sms = 148;
  Dims d{};
  cw_grid grid{};
  size_t esz = 4;
  long long ncell = 0, nu_ = 0, nv_ = 0, nw_ = 0;
  int nxp = 0;                 // row pitch of the PCG vectors (multiple of 16 elements)
  long long ncellp = 0;
  void* xw = nullptr;          // pitched PCG solution vector
  CUtensorMap tm[9];           // z, p0, p1, x, ap, r0, r1, code, code_own
  size_t pcg_smem = 0;
  // workspace (context precision)
  void *tk = nullptr, *tw = nullptr, *speed = nullptr;
  void *ahead[3] = {nullptr, nullptr, nullptr}, *adv[3] = {nullptr, nullptr, nullptr};
  void *clip_mn[3] = {nullptr, nullptr, nullptr}, *clip_mx[3] = {nullptr, nullptr, nullptr};   // MacCormack clip range
  void *r0 = nullptr, *r1 = nullptr, *p0 = nullptr, *p1 = nullptr, *z = nullptr, *Ap = nullptr;
  void *lut = nullptr, *uzx = nullptr, *uzy = nullptr;
  uint8_t* code = nullptr;
  double* part = nullptr;
  unsigned* tags = nullptr;    // [2][part_stride] per-unit publication tags (k_pcg flag-in-data folds)
  int chunk0 = 0, nchunk_g = 1;   // this context's first chunk / chunks of the whole z-slab solve
  unsigned* bar = nullptr;
  int* gate = nullptr;
  DevReport* rep = nullptr;
  double* reg_part = nullptr;   // region partials
  long long* reg_cnt = nullptr;
  double* reg_out = nullptr;
  long long* reg_cout = nullptr;
  // per-step region-speed accumulation (cw_step_regions): after every step
  // the region means are added to reg_sums (the trailing window of
  // evaluate_objective, optimize.py:93-99), no host round trip
  int reg_n = 0;
  RegionBoxes reg_boxes{};
  double* reg_sums = nullptr;
  long long* reg_counts = nullptr;
  int* flag = nullptr;
  // operator
  bool have_op = false;
  double omega = 1.65, tol_default = 0.0;
  double tol_kind[3] = {1e-8, 0.0, 0.0};   // default_projection_tol per preconditioner kind
  int precond = 2;
  int max_iter = 10000;        // project(max_iter=10_000), solver.py:249; cw_set_max_iter
  long long n_unknown = 0;
  double op_sum[2] = {0.0, 0.0};   // owned-plane sums of diag(W) (AI1) and 1/d (Jacobi)
  long long op_n = 0;
  bool op_outlet = false;
  int U = 0, ntx = 0, nty = 0, zc = 1, pcg_blocks = 0, part_stride = 0;
  int max_blocks = 0;          // co-resident PCG blocks on this device
  // z-slab solve across devices (cw_slab_attach): this slab's place and the
  // neighbours' / root's buffers (device pointers valid on this device)
  int nslab = 1, slab = 0;
  cw_slab_buffers lower{}, upper{}, root{};
  unsigned* xbar = nullptr;    // this context's cross-slab barrier (used when it is the root)
  double* xval = nullptr;
  void* slab_args = nullptr;   // device array of per-slab kernel arguments (group launches)
  // grow-only device scratch of cw_voxelize (cw_internal_scratch slots)
  void* vscr[32] = {};
  size_t vscr_n[32] = {};
  // painted-porosity layer for cw_voxelize (device buffers owned by the caller)
  const uint8_t* paint = nullptr;
  const uint8_t* paint_mask = nullptr;
  int paint_kmax = 0;
  double paint_lad = 1.0;
  // pending reports: steps write rep_live, and the step's last kernel commits
  // it to rep[*slot_dev] (the device's count of committed reports, equal to
  // head in stream order) -- no report pointer is baked into a captured step
  int head = 0;
  DevReport* rep_live = nullptr;
  int* slot_dev = nullptr;
  // CUDA-graph replay of whole steps (cw_step): captured once per (fields,
  // params, tolerance, regions) key on a private stream, replayed on the
  // caller's stream.  Off by default (CW_GRAPHS=1 enables): measured at C3 the
  // step's kernels already run back to back (4.482 vs 4.483 ms per steady
  // step), and every design evaluation brings new state buffers, i.e. a new
  // capture (channel_opt: 0.52 s vs 0.17 s per evaluation)
  bool graphs = false;
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    std::string key;
    cudaGraphExec_t exec;
    long long kernels;
  };
  std::vector<GraphEntry> gcache;
  std::vector<double> slot_dt;
  // inlet cache
  cw_inlet inl_cache{};
  bool inl_valid = false;
  // boundary-write lists (k_bc_*_list), built for the labels array at bc_lab
  const void* bc_lab = nullptr;
  long long bc_ver = 0;
  BcEntry* bc_list[7] = {};   // 6 outlet sides in the reference's order, then inlet/wall
  int bc_n[7] = {};
  int* bc_count = nullptr;
  // their composition (k_bc_compose_*): one k_bc_replay launch per pass;
  // bc_nf < 0: not composed (CW_BC_COMPOSE=0, or too many ordered writes)
  BcOp* bc_ops = nullptr;     // bc_nf independent writes, then bc_no ordered ones
  int bc_nf = -1, bc_no = 0;
  size_t bc_cap[7] = {}, bc_ops_cap = 0;   // grow-only capacities (bytes)
  void* bc_held = nullptr;    // > 256 * BC_ORD_PER_THREAD ordered writes: their values (k_bc_ord_gather)
  size_t bc_held_cap = 0;
  // stage timing
  bool timing = false;
  // one-shot waits of the next enqueued step (cw_step_defer): first use of nu_t / p
  cudaEvent_t wait_nut = nullptr, wait_p = nullptr;
  cudaEvent_t wait_kw = nullptr;      // cw_step_defer_kw: k, omega
  cudaEvent_t ev[8] = {};
  bool ev_made = false;
  float stage_ms[7] = {0, 0, 0, 0, 0, 0, 0};
  long long launches = 0;             // kernels enqueued (evidence for the bench's gpu_launches)
  // per-launch device time of the PCG kernel (bench roofline), when enabled
  std::vector<cudaEvent_t> pev;
  int pcg_timed = 0;
  // advection kernels (bench roofline): before predict, after predict, after correct
  std::vector<cudaEvent_t> aev;
  int adv_timed = 0;
};

extern "C" int cw_abi_version(void) { return CW_ABI_VERSION; }

// shared with cw_voxel.cu
int cw_internal_fail(int code, const char* msg) { return fail(code, msg); }
void* cw_internal_scratch(cw_ctx* c, int slot, size_t bytes) {
  if (slot < 0 || slot >= 32) return nullptr;
  if (c->vscr_n[slot] < bytes) {
    if (c->vscr[slot]) cudaFree(c->vscr[slot]);
    c->vscr[slot] = nullptr;
    c->vscr_n[slot] = 0;
    const size_t grow = bytes + bytes / 4;   // a little headroom: designs change the object extents
    if (cudaMalloc(&c->vscr[slot], grow) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    c->vscr_n[slot] = grow;
  }
  return c->vscr[slot];
}
int cw_internal_device(cw_ctx* c, int* nx, int* ny, int* nz, double* h, double* origin) {
  if (c->d.kg0 != 0 || c->d.nz != c->d.nzg)
    return fail(CW_ERR_INVALID, "voxelize on a whole-grid context and copy the slab's window");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(CW_ERR_CUDA, cudaGetErrorString(e));
  *nx = c->d.nx; *ny = c->d.ny; *nz = c->d.nz;
  h[0] = c->grid.dx; h[1] = c->grid.dy; h[2] = c->grid.dz;
  for (int a = 0; a < 3; ++a) origin[a] = c->grid.origin[a];
  return CW_OK;
}
void cw_internal_paint(cw_ctx* c, const uint8_t** image, const uint8_t** mask, int* kmax, double* tree_lad) {
  *image = c->paint;
  *mask = c->paint_mask;
  *kmax = c->paint_kmax;
  *tree_lad = c->paint_lad;
}
extern "C" const char* cw_last_error(void) { return g_err.c_str(); }

extern "C" int cw_set_paint(cw_ctx* c, const unsigned char* d_image, const unsigned char* d_tree_mask, int kmax,
                            double tree_lad) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  if (d_image && (kmax < 0 || kmax > c->d.nz)) return fail(CW_ERR_INVALID, "kmax must lie in [0, nz]");
  c->paint = d_image;
  c->paint_mask = d_image ? d_tree_mask : nullptr;
  c->paint_kmax = d_image ? kmax : 0;
  c->paint_lad = tree_lad;
  return CW_OK;
}

static int alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return fail(CW_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  e = cudaMemset(*p, 0, bytes);
  if (e != cudaSuccess) return fail(CW_ERR_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
  return CW_OK;
}

template <typename T>
static int pcg_occupancy(int* blocks_per_sm, size_t* smem) {
  *smem = pcg_smem_bytes<T>();
  cudaError_t e = cudaFuncSetAttribute(k_pcg<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pcg<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pcg_slabs<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  if (e != cudaSuccess) return fail(CW_ERR_CUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_pcg<T, false>, PCG_THREADS, *smem);
  int b1 = 0, b2 = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_pcg<T, true>, PCG_THREADS, *smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_pcg_slabs<T>, PCG_THREADS, *smem);
  *blocks_per_sm = std::min(*blocks_per_sm, std::min(b1, b2));
  if (e != cudaSuccess) return fail(CW_ERR_CUDA, std::string("occupancy: ") + cudaGetErrorString(e));
  return CW_OK;
}

// TMA descriptors for the pitched PCG vectors (3D: x, y, z; OOB -> zero fill)
static int make_tmap(CUtensorMap* m, CUtensorMapDataType dt, size_t esz, void* base, const cw_ctx* c,
                     unsigned bx, unsigned by) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return fail(CW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint64_t dims[3] = {(cuuint64_t)c->d.nx, (cuuint64_t)c->d.ny, (cuuint64_t)c->d.nz};
  cuuint64_t strides[2] = {(cuuint64_t)c->nxp * esz, (cuuint64_t)c->nxp * c->d.ny * esz};
  cuuint32_t box[3] = {bx, by, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CW_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return CW_OK;
}

// PCG work decomposition: tiles TX x TY over (x, y), z-chunks of zc planes;
// each co-resident block streams ceil(U/B) units of zc+2 planes: minimise
// that critical path (halo planes included).  At most CW_PCG_MAXG (chunk,
// 32-tile group) items (the in-kernel fold keeps one sum per item).  CW_PCG_ZC
// overrides.
static int choose_zc(int tiles, int nown, int maxb) {
  const int ng = (tiles + 31) / 32;   // (chunk, 32-tile group) items of the fold must fit CW_PCG_MAXG
  const int maxc = std::max(1, CW_PCG_MAXG / ng);
  const int zmin = std::max(1, (nown + maxc - 1) / maxc);
  int best_zc = nown, best_cost = 1 << 30;
  for (int zc = zmin; zc <= nown; ++zc) {
    const int U = tiles * ((nown + zc - 1) / zc);
    const int B = std::min(U, maxb);
    const int m = (U + B - 1) / B;
    const int cost = m * (zc + 2);
    if (cost < best_cost) { best_cost = cost; best_zc = zc; }
  }
  if (const char* ev = std::getenv("CW_PCG_ZC")) best_zc = std::max(zmin, std::min(nown, std::atoi(ev)));
  return best_zc;
}

static void plan_units(cw_ctx* c) {
  const int nown = c->d.o1 - c->d.o0;
  const int nchunk = (nown + c->zc - 1) / c->zc;
  c->U = c->ntx * c->nty * nchunk;
  c->pcg_blocks = std::min(c->U, c->max_blocks);
  if (const char* eb = std::getenv("CW_PCG_BLOCKS")) c->pcg_blocks = std::max(1, std::min(c->pcg_blocks, std::atoi(eb)));
  c->chunk0 = 0;
  c->nchunk_g = nchunk;
}

static void drop_graphs(cw_ctx* c);

static int alloc_partials(cw_ctx* c) {
  drop_graphs(c);   // captured PCG launches carry the partition and the partial buffers
  const int need = std::max(c->U, c->max_blocks);
  if (c->part && c->part_stride >= need) return CW_OK;
  if (c->part) { cudaFree(c->part); c->part = nullptr; }
  if (c->tags) { cudaFree(c->tags); c->tags = nullptr; }
  c->part_stride = need;
  int rc = alloc((void**)&c->part, 6 * (size_t)need * sizeof(double));
  rc |= alloc((void**)&c->tags, 2 * (size_t)need * sizeof(unsigned));
  return rc;
}

// A context over the local grid g (a whole grid, or a z-slab window: global
// planes [kg0, kg0 + g->nz) of nzg, owning local planes [own0, own1)).
static int ctx_create(const cw_grid* g, int kg0, int nzg, int own0, int own1, int precision, int device,
                      cw_ctx** out) {
  if (!g || !out) return fail(CW_ERR_INVALID, "null argument");
  if (precision != 4 && precision != 8) return fail(CW_ERR_INVALID, "precision must be 4 or 8");
  if (g->nx < 1 || g->ny < 1 || g->nz < 1) return fail(CW_ERR_INVALID, "cell counts must be >= 1");
  if (!(g->dx > 0 && g->dy > 0 && g->dz > 0)) return fail(CW_ERR_INVALID, "cell spacings must be > 0");
  CW_CUDA(cudaSetDevice(device));
  cw_ctx* c = new cw_ctx();
  c->prec = precision;
  c->esz = precision;
  c->device = device;
  c->grid = *g;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  Dims& d = c->d;
  d.nx = g->nx; d.ny = g->ny; d.nz = g->nz;
  d.dx = (float)g->dx; d.dy = (float)g->dy; d.dz = (float)g->dz;
  d.ddx = g->dx; d.ddy = g->dy; d.ddz = g->dz;
  {
    const double hh[3] = {g->dx, g->dy, g->dz};
    for (int a = 0; a < 3; ++a) {
      d.drh[a] = 1.0 / hh[a];
      d.drh2[a] = 1.0 / (hh[a] * hh[a]);
      d.rh[a] = (float)d.drh[a];
      d.rh2[a] = (float)d.drh2[a];
    }
  }
  d.is2d = g->nz == 1;
  d.o0 = own0; d.o1 = own1; d.kg0 = kg0; d.nzg = nzg;
  c->ncell = d.ncell();
  c->nu_ = (long long)(d.nx + 1) * d.ny * d.nz;
  c->nv_ = (long long)d.nx * (d.ny + 1) * d.nz;
  c->nw_ = (long long)d.nx * d.ny * (d.nz + 1);
  if (std::max(std::max(c->nu_, c->nv_), c->nw_) >= (1LL << 31) || d.nz > 65535) {   // 32-bit gathers, 3-D grids
    cw_ctx_destroy(c);
    return fail(CW_ERR_INVALID, "grid too large for one device context (face arrays must hold < 2^31 cells, nz <= 65535)");
  }
  const size_t cb = c->ncell * c->esz;
  size_t fb[3] = {c->nu_ * c->esz, c->nv_ * c->esz, c->nw_ * c->esz};
  int rc = CW_OK;
  rc |= alloc(&c->tk, cb); rc |= alloc(&c->tw, cb); rc |= alloc(&c->speed, cb);
  for (int a = 0; a < 3; ++a) { rc |= alloc(&c->ahead[a], fb[a]); rc |= alloc(&c->adv[a], fb[a]); }
#if CW_MAC_CLIP
  for (int a = 0; a < 3; ++a) { rc |= alloc(&c->clip_mn[a], fb[a]); rc |= alloc(&c->clip_mx[a], fb[a]); }
#endif
  c->nxp = (d.nx + 15) / 16 * 16;
  c->ncellp = (long long)c->nxp * d.ny * d.nz;
  const size_t pb = c->ncellp * c->esz;
  rc |= alloc(&c->r0, c->ncellp * sizeof(double)); rc |= alloc(&c->r1, c->ncellp * sizeof(double));
  rc |= alloc(&c->p0, pb); rc |= alloc(&c->p1, pb); rc |= alloc(&c->z, pb); rc |= alloc(&c->Ap, pb);
  rc |= alloc(&c->xw, pb);
  rc |= alloc(&c->lut, 64 * 4 * c->esz);
  rc |= alloc(&c->uzx, d.nz * c->esz); rc |= alloc(&c->uzy, d.nz * c->esz);
  rc |= alloc((void**)&c->code, c->ncellp);
  rc |= alloc((void**)&c->bar, 64 * sizeof(unsigned));
  rc |= alloc((void**)&c->gate, sizeof(int));
  rc |= alloc((void**)&c->flag, 4 * sizeof(int));
  rc |= alloc((void**)&c->rep, RING * sizeof(DevReport));
  rc |= alloc((void**)&c->rep_live, sizeof(DevReport));
  rc |= alloc((void**)&c->slot_dev, sizeof(int));
  if (const char* eg = std::getenv("CW_GRAPHS")) c->graphs = std::atoi(eg) != 0;
  if (rc != CW_OK) { cw_ctx_destroy(c); return CW_ERR_CUDA; }
  // PCG work decomposition: tiles TX x TY over (x, y), z-chunks of zc planes;
  // each co-resident block owns at most one unit when the grid allows it.
  int per_sm = 0;
  rc = precision == 4 ? pcg_occupancy<float>(&per_sm, &c->pcg_smem) : pcg_occupancy<double>(&per_sm, &c->pcg_smem);
  if (rc != CW_OK || per_sm < 1) { cw_ctx_destroy(c); return rc != CW_OK ? rc : fail(CW_ERR_CUDA, "pcg kernel cannot be resident"); }
  const int maxb = per_sm * c->num_sms;
  c->max_blocks = maxb;
  c->ntx = (d.nx + TX - 1) / TX;
  c->nty = (d.ny + TY - 1) / TY;
  const int tiles = c->ntx * c->nty;
  c->zc = choose_zc(tiles, d.o1 - d.o0, maxb);
  plan_units(c);
  {
    const CUtensorMapDataType tdt = precision == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    const size_t e = c->esz;
    const unsigned hbw = precision == 4 ? Halo<float>::BW : Halo<double>::BW;
    int r2 = make_tmap(&c->tm[0], tdt, e, c->z, c, hbw, BOX_Y);
    r2 |= make_tmap(&c->tm[1], tdt, e, c->p0, c, hbw, BOX_Y);
    r2 |= make_tmap(&c->tm[2], tdt, e, c->p1, c, hbw, BOX_Y);
    r2 |= make_tmap(&c->tm[3], tdt, e, c->xw, c, TX, TY);
    r2 |= make_tmap(&c->tm[4], tdt, e, c->Ap, c, hbw, BOX_Y);
    r2 |= make_tmap(&c->tm[5], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, c->r0, c, Halo<double>::BW, BOX_Y);
    r2 |= make_tmap(&c->tm[6], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, c->r1, c, Halo<double>::BW, BOX_Y);
    r2 |= make_tmap(&c->tm[7], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, c->code, c, Halo<uint8_t>::BW, BOX_Y);
    r2 |= make_tmap(&c->tm[8], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, c->code, c, TX, TY);
    if (r2 != CW_OK) { cw_ctx_destroy(c); return CW_ERR_CUDA; }
  }
  rc = alloc_partials(c);
  rc |= alloc((void**)&c->xbar, 64 * sizeof(unsigned));
  rc |= alloc((void**)&c->xval, 6 * (size_t)CW_MAX_CHUNKS * sizeof(double));
  rc |= alloc(&c->slab_args, (size_t)CW_MAX_SLABS * sizeof(PcgArgs<double>));
  rc |= alloc((void**)&c->reg_part, (size_t)1024 * 64 * sizeof(double));
  rc |= alloc((void**)&c->reg_cnt, (size_t)1024 * 64 * sizeof(long long));
  rc |= alloc((void**)&c->reg_out, 64 * sizeof(double));
  rc |= alloc((void**)&c->reg_cout, 64 * sizeof(long long));
  if (rc != CW_OK) { cw_ctx_destroy(c); return CW_ERR_CUDA; }
  c->slot_dt.assign(RING, 0.0);
  *out = c;
  return CW_OK;
}

extern "C" int cw_ctx_create(const cw_grid* g, int precision, int device, cw_ctx** out) {
  if (!g) return fail(CW_ERR_INVALID, "null argument");
  return ctx_create(g, 0, g->nz, 0, g->nz, precision, device, out);
}

extern "C" int cw_ctx_create_slab(const cw_grid* g, int k_lo, int k_hi, int halo, int precision, int device,
                                  cw_ctx** out) {
  if (!g || !out) return fail(CW_ERR_INVALID, "null argument");
  if (!(0 <= k_lo && k_lo < k_hi && k_hi <= g->nz)) return fail(CW_ERR_INVALID, "slab planes must satisfy 0 <= k_lo < k_hi <= nz");
  if (halo < 2) return fail(CW_ERR_INVALID, "slab halo must be >= 2 planes");
  const int kb = std::max(k_lo - halo, 0), ke = std::min(k_hi + halo, g->nz);
  cw_grid loc = *g;
  loc.nz = ke - kb;   // origin stays the global one: heights use the global plane index
  return ctx_create(&loc, kb, g->nz, k_lo - kb, k_hi - kb, precision, device, out);
}

extern "C" int cw_slab_info(cw_ctx* c, int* kg0, int* nz_local, int* own0, int* own1) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  if (kg0) *kg0 = c->d.kg0;
  if (nz_local) *nz_local = c->d.nz;
  if (own0) *own0 = c->d.o0;
  if (own1) *own1 = c->d.o1;
  return CW_OK;
}

extern "C" void cw_ctx_destroy(cw_ctx* c) {
  if (!c) return;
  for (int q = 0; q < 32; ++q)
    if (c->vscr[q]) cudaFree(c->vscr[q]);
  for (auto& e : c->gcache) cudaGraphExecDestroy(e.exec);
  c->gcache.clear();
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  cudaSetDevice(c->device);
  void* ptrs[] = {c->tk, c->tw, c->speed, c->ahead[0], c->ahead[1], c->ahead[2], c->clip_mn[0], c->clip_mn[1], c->clip_mn[2], c->clip_mx[0], c->clip_mx[1], c->clip_mx[2], c->adv[0], c->adv[1],
                  c->adv[2], c->r0, c->r1, c->p0, c->p1, c->z, c->Ap, c->xw, c->lut, c->uzx, c->uzy, c->code,
                  c->part, c->tags, c->bar, c->gate, c->rep, c->rep_live, c->slot_dev, c->reg_part, c->reg_cnt, c->reg_out, c->reg_cout,
                  c->flag, c->xbar, c->xval, c->slab_args};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int q = 0; q < 7; ++q)
    if (c->bc_list[q]) cudaFree(c->bc_list[q]);
  if (c->bc_count) cudaFree(c->bc_count);
  if (c->bc_ops) cudaFree(c->bc_ops);
  if (c->bc_held) cudaFree(c->bc_held);
  if (c->ev_made)
    for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->pev) cudaEventDestroy(e);
  for (auto& e : c->aev) cudaEventDestroy(e);
  delete c;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline dim3 g3(int ex, int ey, int ez) {   // 3-D stage-kernel grid (cw_step.cuh CW_IJK)
  return dim3((unsigned)((ex + ST_BX - 1) / ST_BX), (unsigned)((ey + ST_BY - 1) / ST_BY),
              (unsigned)((ez + ST_BZ - 1) / ST_BZ));
}
static const dim3 B3(ST_BX, ST_BY, ST_BZ);
// z-coarsened stage kernels (CW_ZT planes per thread)
static inline dim3 g3z(int ex, int ey, int ez) {
  return dim3((unsigned)((ex + ST_BX - 1) / ST_BX), (unsigned)((ey + ST_BY - 1) / ST_BY),
              (unsigned)((ez + CW_ZT - 1) / CW_ZT));
}
// owned-plane max reduction (k_div_max): each block strides
// over the planes, about 2048 blocks in all, one atomic per block
static inline dim3 g3r(int ex, int ey, int nz) {
  const int bx = (ex + ST_BX - 1) / ST_BX, by = (ey + 7) / 8;
  return dim3((unsigned)bx, (unsigned)by, (unsigned)std::max(1, std::min(nz, 2048 / std::max(1, bx * by))));
}
static const dim3 B3R(ST_BX, 8, 1);
static inline int nblk(long long n, int bs = 256) {
  long long b = (n + bs - 1) / bs;
  return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 32));
}

// ---------------------------------------------------------------------------
// operator setup

extern "C" int cw_set_operator(cw_ctx* c, const signed char* lab, double ai_omega, long long* n_unknown,
                               double* tol_default, void* stream) {
  if (!c || !lab) return fail(CW_ERR_INVALID, "null argument");
  if (!(ai_omega > 0.0 && ai_omega < 2.0)) return fail(CW_ERR_INVALID, "omega must lie in (0, 2)");
  CW_CUDA(cudaSetDevice(c->device));
  const Dims& d = c->d;
  const double w[3] = {1.0 / (c->grid.dx * c->grid.dx), 1.0 / (c->grid.dy * c->grid.dy),
                       1.0 / (c->grid.dz * c->grid.dz)};
  // LUT: d, 1/d, s*omega with s = (2-omega)*omega/d, and omega/d for each
  // neighbour-bit pattern (the PCG's W r: y = (2-omega) omega q + s omega sum w q_-,
  // z = y + (omega/d) sum w y_+, cw_pcg.cuh).
  // Neighbour order +x,-x,+y,-y,+z,-z (ref linalg.py:20 offsets order).
  std::vector<double> lut(64 * 4, 0.0);
  for (int b = 1; b < 64; ++b) {
    double dd = 0.0;
    for (int q = 0; q < 6; ++q)
      if (b & (1 << q)) dd += w[q / 2];
    lut[b * 4 + 0] = dd;
    lut[b * 4 + 1] = 1.0 / dd;
    lut[b * 4 + 2] = (2.0 - ai_omega) * ai_omega / dd * ai_omega;
    lut[b * 4 + 3] = ai_omega / dd;
  }
  if (c->prec == 4) {
    std::vector<float> lf(lut.begin(), lut.end());
    CW_CUDA(cudaMemcpyAsync(c->lut, lf.data(), lf.size() * 4, cudaMemcpyHostToDevice, S(stream)));
  } else {
    CW_CUDA(cudaMemcpyAsync(c->lut, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, S(stream)));
  }
  CW_CUDA(cudaMemsetAsync(c->flag, 0, 4 * sizeof(int), S(stream)));
  const int nb = std::min(nblk(c->ncell), 1024);
  (k_build_code<<<nb, 256, 0, S(stream)>>>(d, c->nxp, (const int8_t*)lab, c->code, c->flag), ++c->launches);
  CW_CUDA(cudaGetLastError());
  (k_wdiag_partials<<<nb, 256, 0, S(stream)>>>(d, c->nxp, c->code, w[0], w[1], w[2], ai_omega, c->reg_part, c->reg_cnt,
                                               c->reg_part + 1024), ++c->launches);
  CW_CUDA(cudaGetLastError());
  std::vector<double> parts(nb), jparts(nb);
  std::vector<long long> cnts(nb);
  int flags[4];
  CW_CUDA(cudaMemcpyAsync(parts.data(), c->reg_part, nb * sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaMemcpyAsync(jparts.data(), c->reg_part + 1024, nb * sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaMemcpyAsync(cnts.data(), c->reg_cnt, nb * sizeof(long long), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaMemcpyAsync(flags, c->flag, sizeof(flags), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  double sum = 0.0, jsum = 0.0;
  long long n = 0;
  for (int b = 0; b < nb; ++b) { sum += parts[b]; jsum += jparts[b]; n += cnts[b]; }
  const bool slab = d.kg0 != 0 || d.nz != d.nzg;
  c->op_sum[0] = sum; c->op_sum[1] = jsum; c->op_n = n; c->op_outlet = flags[0] != 0;
  // a z-slab's operator checks are global: the caller combines cw_operator_partials
  if (n == 0 && !slab) return fail(CW_ERR_INVALID, "no flow cells to solve for");
  if (flags[0] == 0 && !slab) return fail(CW_ERR_SINGULAR, "no outlet cells: pressure defined only up to a constant");
  if (flags[1] != 0) return fail(CW_ERR_INVALID, "AI preconditioner requires a positive diagonal");
  c->omega = ai_omega;
  c->n_unknown = n;
  const double mean = n > 0 ? sum / (double)n : 0.0;
  c->tol_kind[0] = 1e-8;                                           // no W: mscale 1
  c->tol_kind[1] = 1e-8 * std::max(n > 0 ? jsum / (double)n : 0.0, 1e-300);   // Jacobi W = diag(1/d)
  c->tol_kind[2] = 1e-8 * std::max(mean, 1e-300);                  // AI1
  c->tol_default = c->tol_kind[c->precond];
  c->have_op = true;
  if (n_unknown) *n_unknown = n;
  if (tol_default) *tol_default = c->tol_default;
  return CW_OK;
}

extern "C" int cw_operator_partials(cw_ctx* c, double* wdiag_sum, double* jacobi_sum, long long* n_unknown,
                                    int* has_outlet) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  if (!c->have_op) return fail(CW_ERR_INVALID, "cw_set_operator first");
  if (wdiag_sum) *wdiag_sum = c->op_sum[0];
  if (jacobi_sum) *jacobi_sum = c->op_sum[1];
  if (n_unknown) *n_unknown = c->op_n;
  if (has_outlet) *has_outlet = c->op_outlet ? 1 : 0;
  return CW_OK;
}

// ---------------------------------------------------------------------------
// drag coefficient

extern "C" int cw_drag_coefficient(cw_ctx* c, const double* phi, const double* lad, const signed char* lab,
                                   const cw_params* prm, void* g, int* has_drag, void* stream) {
  if (!c || !phi || !lad || !lab || !prm || !g) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  CW_CUDA(cudaMemsetAsync(c->flag, 0, sizeof(int), S(stream)));
  if (c->prec == 4)
    (k_drag_coef<float><<<nblk(c->ncell), 256, 0, S(stream)>>>(c->ncell, phi, lad, (const int8_t*)lab, *prm, (float*)g, c->flag), ++c->launches);
  else
    (k_drag_coef<double><<<nblk(c->ncell), 256, 0, S(stream)>>>(c->ncell, phi, lad, (const int8_t*)lab, *prm, (double*)g, c->flag), ++c->launches);
  CW_CUDA(cudaGetLastError());
  int f = 0;
  CW_CUDA(cudaMemcpyAsync(&f, c->flag, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  if (has_drag) *has_drag = f != 0;
  return CW_OK;
}

// ---------------------------------------------------------------------------
// boundary conditions

static int upload_inlet(cw_ctx* c, const cw_inlet* inl, cudaStream_t st) {
  if (c->inl_valid && std::memcmp(&c->inl_cache, inl, sizeof(cw_inlet)) == 0) return CW_OK;
  const int nz = c->d.nz;
  std::vector<double> ux(nz), uy(nz);
  for (int k = 0; k < nz; ++k) {
    const double zc = c->grid.origin[2] + ((double)(k + c->d.kg0) + 0.5) * c->grid.dz;   // solver.py:384
    double s;
    if (inl->kind == 0) s = inl->speed;
    else s = zc > inl->z0 ? inl->u_star / inl->kappa * std::log(zc / inl->z0) : 0.0;   // solver.py:75-82
    ux[k] = s * inl->dir_x;
    uy[k] = s * inl->dir_y;
  }
  if (c->prec == 4) {
    std::vector<float> fx(ux.begin(), ux.end()), fy(uy.begin(), uy.end());
    CW_CUDA(cudaMemcpyAsync(c->uzx, fx.data(), nz * 4, cudaMemcpyHostToDevice, st));
    CW_CUDA(cudaMemcpyAsync(c->uzy, fy.data(), nz * 4, cudaMemcpyHostToDevice, st));
    CW_CUDA(cudaStreamSynchronize(st));   // host vectors go out of scope
  } else {
    CW_CUDA(cudaMemcpyAsync(c->uzx, ux.data(), nz * 8, cudaMemcpyHostToDevice, st));
    CW_CUDA(cudaMemcpyAsync(c->uzy, uy.data(), nz * 8, cudaMemcpyHostToDevice, st));
    CW_CUDA(cudaStreamSynchronize(st));
  }
  c->inl_cache = *inl;
  c->inl_valid = true;
  return CW_OK;
}

// Enumerate the boundary writes of this labels array (once per labels
// pointer; labels are fixed while a context steps them).  0 on success.
static void drop_graphs(cw_ctx* c) {
  for (auto& e : c->gcache) cudaGraphExecDestroy(e.exec);
  c->gcache.clear();
}

static void compose_bc(cw_ctx* c, cudaStream_t st);

// grow-only device buffer (the boundary lists and their composition are
// rebuilt for every design's labels: no cudaFree / cudaMalloc churn)
static bool grow(void** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return true;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const size_t n = need + need / 4;
  if (cudaMalloc(p, n) != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return false;
  }
  *cap = n;
  return true;
}

static int build_bc_lists(cw_ctx* c, const int8_t* lab, long long ver, cudaStream_t st) {
  const Dims& d = c->d;
  drop_graphs(c);   // captured steps reference the lists rebuilt below
  c->bc_nf = -1;
  for (int q = 0; q < 7; ++q) c->bc_n[q] = 0;
  c->bc_lab = nullptr;
  if (!c->bc_count && alloc((void**)&c->bc_count, 8 * sizeof(int)) != CW_OK) return 1;
  const int sides = d.is2d ? 4 : 6;
  auto side_launch = [&](int s, BcEntry* out, int cap) {
    const int axis = s / 2;
    const int ext = axis == 0 ? d.nx : (axis == 1 ? d.ny : d.nz);
    const int pos = (s & 1) ? ext - 1 : 0;
    const int e1 = axis == 0 ? d.ny : d.nx, e2 = axis == 2 ? d.ny : d.nz;
    k_bc_outlet_list<<<nblk((long long)(e1 + 1) * (e2 + 1)), 256, 0, st>>>(d, axis, pos, lab, out, c->bc_count + s, cap);
  };
  // pass 1: counts
  if (cudaMemsetAsync(c->bc_count, 0, 8 * sizeof(int), st) != cudaSuccess) return 1;
  for (int s = 0; s < sides; ++s) side_launch(s, nullptr, 0);
  k_bc_inlet_wall_list<<<g3(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(d, lab, nullptr, c->bc_count + 6, 0);
  int cnt[8];
  if (cudaMemcpyAsync(cnt, c->bc_count, sizeof(cnt), cudaMemcpyDeviceToHost, st) != cudaSuccess) return 1;
  if (cudaStreamSynchronize(st) != cudaSuccess) return 1;
  // pass 2: the entries
  for (int q = 0; q < 7; ++q)
    if (cnt[q] > 0 && !grow((void**)&c->bc_list[q], &c->bc_cap[q], (size_t)cnt[q] * sizeof(BcEntry))) return 1;
  if (cudaMemsetAsync(c->bc_count, 0, 8 * sizeof(int), st) != cudaSuccess) return 1;
  for (int s = 0; s < sides; ++s)
    if (cnt[s] > 0) side_launch(s, c->bc_list[s], cnt[s]);
  if (cnt[6] > 0)
    k_bc_inlet_wall_list<<<g3(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(d, lab, c->bc_list[6], c->bc_count + 6, cnt[6]);
  if (cudaGetLastError() != cudaSuccess) return 1;
  for (int q = 0; q < 7; ++q) c->bc_n[q] = cnt[q];
  c->bc_lab = lab;
  c->bc_ver = ver;
  compose_bc(c, st);   // on failure the ordered list launches stay in use
  return 0;
}

// The lists' composition for k_bc_replay (see k_bc_compose_expand).  Sets
// bc_ops / bc_nf / bc_no, or leaves bc_nf = -1.
static void compose_bc(cw_ctx* c, cudaStream_t st) {
  c->bc_nf = -1;
  c->bc_no = 0;
  const char* env = getenv("CW_BC_COMPOSE");
  if (env && env[0] == '0') return;
  long long base[7], tot = 0;
  for (int q = 0; q < 7; ++q) {
    base[q] = tot;
    tot += 4LL * c->bc_n[q];
  }
  if (tot == 0) {
    c->bc_nf = 0;
    return;
  }
  BcFieldOff fo;
  const long long sz[7] = {c->nu_, c->nv_, c->nw_, c->ncell, c->ncell, c->ncell, c->ncell};
  fo.off[0] = 0;
  for (int f = 0; f < 7; ++f) fo.off[f + 1] = fo.off[f] + sz[f];
  constexpr int ORD_CAP = 256 * BC_ORD_PER_THREAD;
  // temporaries in the context's grow-only scratch (slots 24..29; cw_voxelize uses the low slots)
  int* wmap = (int*)cw_internal_scratch(c, 29, (size_t)fo.off[7] * sizeof(int));
  BcOp* ops = (BcOp*)cw_internal_scratch(c, 28, (size_t)tot * sizeof(BcOp));
  BcOp* outp = (BcOp*)cw_internal_scratch(c, 27, 2 * (size_t)tot * sizeof(BcOp));
  uint8_t* flag = (uint8_t*)cw_internal_scratch(c, 26, (size_t)tot);
  if (!wmap || !ops || !outp || !flag) return;
  int nc[2] = {0, 0};
  bool ok = cudaMemsetAsync(wmap, 0xff, (size_t)fo.off[7] * sizeof(int), st) == cudaSuccess &&
            cudaMemsetAsync(c->bc_count, 0, 2 * sizeof(int), st) == cudaSuccess;
  const int grid = 4 * c->num_sms;
  for (int q = 0; ok && q < 7; ++q) {
    if (c->bc_n[q] == 0) continue;
    k_bc_compose_expand<<<std::min(nblk(c->bc_n[q]), grid), 256, 0, st>>>(c->bc_list[q], c->bc_n[q], q == 6, ops,
                                                                          base[q], wmap, fo);
    k_bc_compose_claim<<<std::min(nblk(4LL * c->bc_n[q]), grid), 256, 0, st>>>(ops, base[q], 4LL * c->bc_n[q], wmap,
                                                                              fo);
  }
  k_bc_compose_final<<<std::min(nblk(tot), grid), 256, 0, st>>>(ops, tot, wmap, fo, flag);
  k_bc_compose_conflict<<<std::min(nblk(tot), grid), 256, 0, st>>>(ops, tot, wmap, fo, flag);
  k_bc_compose_compact<<<std::min(nblk(tot), grid), 256, 0, st>>>(ops, tot, flag, outp, outp + tot, (int)tot,
                                                                   c->bc_count);
  ok = ok && cudaGetLastError() == cudaSuccess &&
       cudaMemcpyAsync(nc, c->bc_count, sizeof(nc), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
       cudaStreamSynchronize(st) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return;
  }
  // more ordered writes than block 0 of the replay holds: a gather launch first
  if (nc[1] > ORD_CAP && !grow(&c->bc_held, &c->bc_held_cap, (size_t)nc[1] * sizeof(double))) return;
  if (getenv("CW_BC_DEBUG"))
    fprintf(stderr, "cw: boundary pass composed: %d independent writes, %d ordered (%s)\n", nc[0], nc[1],
            nc[1] > ORD_CAP ? "gather launch" : "replay block 0");
  const int n = nc[0];
  if (n + nc[1] > 0) {
    ok = grow((void**)&c->bc_ops, &c->bc_ops_cap, (size_t)(n + nc[1]) * sizeof(BcOp)) &&
         cudaMemcpyAsync(c->bc_ops + n, outp + tot, (size_t)nc[1] * sizeof(BcOp), cudaMemcpyDeviceToDevice, st) ==
             cudaSuccess;
    if (ok && n > 0) {   // the independent writes sorted by (field, destination): coalesced replay
      size_t tmp_n = 0;
      ok = cub::DeviceRadixSort::SortPairs(nullptr, tmp_n, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                           (int*)nullptr, (int*)nullptr, n, 0, 35, st) == cudaSuccess;
      unsigned long long* keys = (unsigned long long*)cw_internal_scratch(c, 25, 2 * (size_t)n * sizeof(unsigned long long));
      int* idx = (int*)cw_internal_scratch(c, 24, 2 * (size_t)n * sizeof(int));
      void* tmp = cw_internal_scratch(c, 23, std::max<size_t>(tmp_n, 16));
      ok = ok && keys && idx && tmp;
      if (ok) {
        k_bc_compose_keys<<<std::min(nblk(n), grid), 256, 0, st>>>(outp, n, keys, idx);
        ok = cub::DeviceRadixSort::SortPairs(tmp, tmp_n, keys, keys + n, idx, idx + n, n, 0, 35, st) == cudaSuccess;
        k_bc_compose_gather<<<std::min(nblk(n), grid), 256, 0, st>>>(outp, idx + n, n, c->bc_ops);
        ok = ok && cudaGetLastError() == cudaSuccess;
      }
    }
  }
  if (ok) {
    c->bc_nf = n;
    c->bc_no = nc[1];
  }
  cudaGetLastError();
}

// the boundary lists of (lab, ver) are built (and composed when enabled)
static bool have_bc_lists(cw_ctx* c, const int8_t* lab, long long ver, cudaStream_t st) {
  return ver != 0 && ((c->bc_lab == lab && c->bc_ver == ver) || build_bc_lists(c, lab, ver, st) == 0);
}

constexpr unsigned BC_ALL = 0x7fu, BC_UVWP = 0x47u, BC_KWN = 0x38u;   // fields u v w k omega nu_t p = bits 0..6

// fmask != BC_ALL only with composed lists (callers check c->bc_nf >= 0)
template <typename T>
static void launch_bc(cw_ctx* c, BcFields<T> F, const int8_t* lab, long long ver, const cw_params* prm,
                      cudaStream_t st, unsigned fmask = BC_ALL, unsigned gate_pass = 0) {
  const Dims& d = c->d;
  if (have_bc_lists(c, lab, ver, st)) {
    if (c->bc_nf >= 0) {   // the composed pass: one launch (two with a large ordered set)
      const T k_in = (T)prm->k_in, om_in = (T)prm->omega_in, nut_in = (T)(prm->k_in / prm->omega_in);
      const BcOp* oops = c->bc_ops + c->bc_nf;
      T* held = nullptr;
      if (c->bc_no > 256 * BC_ORD_PER_THREAD) {
        held = (T*)c->bc_held;
        (k_bc_ord_gather<T><<<std::min(nblk(c->bc_no), 8 * c->num_sms), 256, 0, st>>>(
             F, oops, c->bc_no, (const T*)c->uzx, (const T*)c->uzy, k_in, om_in, nut_in, fmask, held, c->gate,
             gate_pass),
         ++c->launches);
      }
      if (c->bc_nf + c->bc_no > 0)
        (k_bc_replay<T><<<1 + std::max(1, std::min(nblk(c->bc_nf), 8 * c->num_sms)), 256, 0, st>>>(
             F, c->bc_ops, c->bc_nf, oops, c->bc_no, (const T*)c->uzx, (const T*)c->uzy, k_in, om_in, nut_in, fmask,
             c->gate, held, gate_pass),
         ++c->launches);
      return;
    }
    for (int q = 0; q < 6; ++q)
      if (c->bc_n[q] > 0)
        (k_bc_copy_list<T><<<nblk(c->bc_n[q]), 256, 0, st>>>(F, c->bc_list[q], c->bc_n[q], c->gate), ++c->launches);
    if (c->bc_n[6] > 0)
      (k_bc_set_list<T><<<nblk(c->bc_n[6]), 256, 0, st>>>(F, c->bc_list[6], c->bc_n[6], (const T*)c->uzx,
                                                         (const T*)c->uzy, (T)prm->k_in, (T)prm->omega_in,
                                                         (T)(prm->k_in / prm->omega_in), c->gate),
       ++c->launches);
    return;
  }
  cudaGetLastError();   // list build failed: the full-volume kernels below
  const int sides = d.is2d ? 4 : 6;
  for (int s = 0; s < sides; ++s) {
    const int axis = s / 2;
    const int ext = axis == 0 ? d.nx : (axis == 1 ? d.ny : d.nz);
    const int pos = (s & 1) ? ext - 1 : 0;
    const int e1 = axis == 0 ? d.ny : d.nx, e2 = axis == 2 ? d.ny : d.nz;
    (k_bc_outlet_side<T><<<nblk((long long)(e1 + 1) * (e2 + 1)), 256, 0, st>>>(d, axis, pos, F, lab, c->gate), ++c->launches);
  }
  (k_bc_inlet_wall<T><<<g3(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(d, F, lab, (const T*)c->uzx, (const T*)c->uzy, (T)prm->k_in,
                                              (T)prm->omega_in, (T)(prm->k_in / prm->omega_in), c->gate), ++c->launches);
}

extern "C" int cw_apply_boundary(cw_ctx* c, const cw_fields* f, const cw_params* prm, const cw_inlet* inl,
                                 void* stream) {
  if (!c || !f || !prm || !inl) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  int rc = upload_inlet(c, inl, S(stream));
  if (rc) return rc;
  if (c->prec == 4) {
    BcFields<float> F{(float*)f->u, (float*)f->v, (float*)f->w, (float*)f->p, (float*)f->k, (float*)f->omega, (float*)f->nu_t};
    launch_bc<float>(c, F, (const int8_t*)f->labels, f->labels_version, prm, S(stream));
  } else {
    BcFields<double> F{(double*)f->u, (double*)f->v, (double*)f->w, (double*)f->p, (double*)f->k, (double*)f->omega, (double*)f->nu_t};
    launch_bc<double>(c, F, (const int8_t*)f->labels, f->labels_version, prm, S(stream));
  }
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

// ---------------------------------------------------------------------------
// the step

template <typename T>
static void fill_pcg_args(PcgArgs<T>& A, cw_ctx* c, const cw_fields* f, DevReport* rep, double dt, double tol) {
  A.tm_z = c->tm[0]; A.tm_p0 = c->tm[1]; A.tm_p1 = c->tm[2]; A.tm_x = c->tm[3]; A.tm_ap = c->tm[4];
  A.tm_r0 = c->tm[5]; A.tm_r1 = c->tm[6]; A.tm_code = c->tm[7]; A.tm_code_own = c->tm[8];
  A.d = c->d;
  A.nxp = c->nxp;
  A.code = c->code;
  A.state_p = (T*)f->p;
  A.u = (const T*)f->u; A.v = (const T*)f->v; A.w = (const T*)f->w;
  A.r0 = (double*)c->r0; A.r1 = (double*)c->r1; A.p0 = (T*)c->p0; A.p1 = (T*)c->p1; A.z = (T*)c->z; A.Ap = (T*)c->Ap;
  A.x = (T*)c->xw;
  A.part = c->part;
  A.tags = c->tags;
  A.PS = c->part_stride;
  A.tiles = c->ntx * c->nty;
  A.nchunk = c->U / A.tiles;
  A.chunk0 = c->chunk0;
  A.nchunk_g = c->nchunk_g;
  A.bar = c->bar;
  A.gate = c->gate;
  A.rep = rep;
  A.lut = (const T*)c->lut;
  A.wx = (T)(1.0 / (c->grid.dx * c->grid.dx));
  A.wy = (T)(1.0 / (c->grid.dy * c->grid.dy));
  A.wz = c->d.is2d ? (T)0 : (T)(1.0 / (c->grid.dz * c->grid.dz));
  A.om = (T)c->omega;
  A.dt = dt;
  A.tol = tol;
  A.res_factor = std::pow(10.0, -4.5);   // DIV_REDUCTION_TARGET, solver.py:232
  A.max_iter = c->max_iter;              // project(max_iter=10_000) by default, solver.py:249
  A.precond = c->precond;
  A.ntx = c->ntx; A.nty = c->nty; A.zc = c->zc; A.U = c->U;
  A.o0 = c->d.o0; A.o1 = c->d.o1;
  A.nslab = 1; A.slab = 0;
  A.lo = PcgPeer<T>{}; A.hi = PcgPeer<T>{};
  A.xbar = nullptr; A.xval = nullptr;
  A.timeout_ns = 20LL * 1000 * 1000 * 1000;
  A.probe_mode = 0;
  A.probe_iters = 0;
  if (const char* pe = std::getenv("CW_PCG_PROBE")) {   // developer timing probe "mode,iters"
    A.probe_mode = std::atoi(pe);
    const char* comma = std::strchr(pe, 0x2c);
    A.probe_iters = comma ? std::atoi(comma + 1) : 100;
  }
}

template <typename T>
static PcgPeer<T> peer_of(const cw_slab_buffers& b, int plane, long long pplane) {
  PcgPeer<T> q{};
  if (!b.z) return q;
  q.r0 = (double*)b.r0; q.r1 = (double*)b.r1;
  q.p0 = (T*)b.p0; q.p1 = (T*)b.p1; q.z = (T*)b.z; q.Ap = (T*)b.Ap;
  q.plane_off = (long long)plane * pplane;
  return q;
}

// this context's slab within an attached multi-device solve
template <typename T>
static void set_slab_peers(PcgArgs<T>& A, const cw_ctx* c) {
  const long long pplane = (long long)c->nxp * c->d.ny;
  A.nslab = c->nslab;
  A.slab = c->slab;
  A.lo = peer_of<T>(c->lower, c->lower.o1, pplane);       // their halo plane above their slab
  A.hi = peer_of<T>(c->upper, c->upper.o0 - 1, pplane);   // their halo plane below their slab
  A.xbar = (unsigned*)c->root.xbar;
  A.xval = (double*)c->root.xval;
}

template <typename T>
static int launch_pcg(cw_ctx* c, const cw_fields* f, DevReport* rep, double dt, double tol, cudaStream_t st) {
  PcgArgs<T> A;
  fill_pcg_args<T>(A, c, f, rep, dt, tol);
  if (c->nslab > 1) set_slab_peers<T>(A, c);
  CW_CUDA(cudaMemsetAsync(c->bar, 0, 64 * sizeof(unsigned), st));
  CW_CUDA(cudaMemsetAsync(c->tags, 0, 2 * (size_t)c->part_stride * sizeof(unsigned), st));
  void* args[] = {&A};
  const void* kfn = c->nslab > 1 ? (const void*)k_pcg<T, true> : (const void*)k_pcg<T, false>;
  CW_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(c->pcg_blocks), dim3(PCG_THREADS), args, c->pcg_smem, st));
  return CW_OK;
}

// stage building blocks ------------------------------------------------------
template <typename T>
struct StepPtrs {
  T *u, *v, *w, *p, *k, *om, *nut;
  const int8_t* lab;
  long long lab_ver;
  const T* g;
};

template <typename T>
static double nu_stable(const cw_ctx* c, double dt) {   // turbulence.py:18-23
  double s = 1.0 / (c->grid.dx * c->grid.dx) + 1.0 / (c->grid.dy * c->grid.dy);
  if (!c->d.is2d) s += 1.0 / (c->grid.dz * c->grid.dz);
  return 1.0 / (2.0 * dt * s);
}

// upwind k/omega into (kout, wout); MacCormack u, v, w into the adv buffers
// acell != nullptr (cw_step_defer_kw): the predictor saves the cell-centred
// old velocity there instead of running the upwind step
template <typename T>
static void st_advect(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, T* kout, T* wout, cudaStream_t st,
                      T* acell = nullptr) {
  const Dims& d = c->d;
  const T dt = (T)prm->dt;
  const bool turb = prm->turbulence != 0;    // upwind k, omega ride along in the predictor launch
  const bool timed = c->adv_timed < (int)c->aev.size() / 3;
  if (timed) cudaEventRecord(c->aev[3 * c->adv_timed], st);
  const MacClip<T> clip{{(T*)c->clip_mn[0], (T*)c->clip_mn[1], (T*)c->clip_mn[2]},
                        {(T*)c->clip_mx[0], (T*)c->clip_mx[1], (T*)c->clip_mx[2]}};
  const dim3 gp((d.nx + 1 + ST_BX - 1) / ST_BX, (d.ny + 1 + ST_BY - 1) / ST_BY, (d.nz + 1 + ZT_MAC - 1) / ZT_MAC);
  if (acell)
    (k_mac_predict<T, true><<<gp, B3, 0, st>>>(d, P.u, P.v, P.w, (T*)c->ahead[0], (T*)c->ahead[1], (T*)c->ahead[2],
                                               dt, (const T*)P.k, (const T*)P.om, (T*)nullptr, (T*)nullptr, clip,
                                               c->gate, acell),
     ++c->launches);
  else
    (k_mac_predict<T><<<gp, B3, 0, st>>>(
         d, P.u, P.v, P.w, (T*)c->ahead[0], (T*)c->ahead[1], (T*)c->ahead[2], dt, (const T*)P.k, (const T*)P.om,
         turb ? kout : (T*)nullptr, turb ? wout : (T*)nullptr, clip, c->gate), ++c->launches);
  if (timed) cudaEventRecord(c->aev[3 * c->adv_timed + 1], st);
  (k_mac_correct<T><<<dim3((d.nx + 1 + ST_BX - 1) / ST_BX, (d.ny + 1 + ST_BY - 1) / ST_BY, (d.nz + 1 + ZT_MAC - 1) / ZT_MAC), B3, 0, st>>>(
       d, P.u, P.v, P.w, (const T*)c->ahead[0], (const T*)c->ahead[1], (const T*)c->ahead[2], (T*)c->adv[0],
       (T*)c->adv[1], (T*)c->adv[2], dt, clip, c->gate), ++c->launches);
  if (timed) cudaEventRecord(c->aev[3 * c->adv_timed++ + 2], st);
}

template <typename T>
static void st_diffuse(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, cudaStream_t st) {
  const Dims& d = c->d;
  T* cu[3] = {P.u, P.v, P.w};
  double cap = nu_stable<T>(c, prm->dt) - prm->nu;
  if (cap <= 0) cap = 0.0;                               // solver.py:195-201
#ifdef CW_DIFFUSE_GENERIC   // developer comparison: the per-axis-loop kernel
  (k_diffuse<T><<<g3z(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(
       d, (const T*)c->adv[0], (const T*)c->adv[1], (const T*)c->adv[2], cu[0], cu[1], cu[2], P.nut, (T)prm->dt,
       (T)prm->nu, (T)cap, c->gate), ++c->launches);
#else
  (k_diffuse_c<T><<<g3z(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(
       d, (const T*)c->adv[0], (const T*)c->adv[1], (const T*)c->adv[2], cu[0], cu[1], cu[2], P.nut, (T)prm->dt,
       (T)prm->nu, (T)cap, c->gate), ++c->launches);
#endif
}

template <typename T>
static void st_drag(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, int has_drag, cudaStream_t st) {
  if (!has_drag) return;                                 // solver.py:157-158
  const Dims& d = c->d;
  T* cu[3] = {P.u, P.v, P.w};
  (k_cell_speed<T><<<g3(d.nx, d.ny, d.nz), B3, 0, st>>>(d, P.u, P.v, P.w, (T*)c->speed, c->gate), ++c->launches);
  (k_drag<T><<<g3z(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(d, cu[0], cu[1], cu[2], P.g, (const T*)c->speed,
                                                                (T)prm->dt, c->gate), ++c->launches);
}

template <typename T>
static void st_project_tail(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, DevReport* rep, cudaStream_t st);

template <typename T>
static int st_project(cw_ctx* c, const StepPtrs<T>& P, const cw_fields* f, const cw_params* prm, double tol,
                      DevReport* rep, cudaStream_t st) {
  T* cu[3] = {P.u, P.v, P.w};
  const bool tpcg = c->pcg_timed < (int)c->pev.size() / 2;
  if (tpcg) cudaEventRecord(c->pev[2 * c->pcg_timed], st);
  int rc = launch_pcg<T>(c, f, rep, prm->dt, tol, st);
  ++c->launches;
  if (tpcg) cudaEventRecord(c->pev[2 * c->pcg_timed++ + 1], st);
  if (rc) return rc;
  st_project_tail<T>(c, P, prm, rep, st);
  return CW_OK;
}

// after the PCG: pressure-gradient update and max |div| (solver.py:282-304)
template <typename T>
static void st_project_tail(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, DevReport* rep, cudaStream_t st) {
  const Dims& d = c->d;
  T* cu[3] = {P.u, P.v, P.w};
  (k_gradient<T><<<g3z(d.nx + 1, d.ny + 1, d.nz + 1), B3, 0, st>>>(d, cu[0], cu[1], cu[2], P.p, P.lab, (T)prm->dt,
                                                                    c->gate), ++c->launches);
  (k_div_max<T><<<g3r(d.nx, d.ny, d.o1 - d.o0), B3R, 0, st>>>(d, P.u, P.v, P.w, P.lab, rep, SLOT_DIV_AFTER, c->gate), ++c->launches);
}

template <typename T>
static void st_turb(cw_ctx* c, const StepPtrs<T>& P, const cw_params* prm, const T* kin, const T* win,
                    DevReport* rep, cudaStream_t st) {
  StepConsts sc;
  const double nus = nu_stable<T>(c, prm->dt);
  sc.dt = prm->dt; sc.nu = prm->nu; sc.cap_diffuse = 0.0;
  sc.cap_turb = std::max(nus - prm->nu, 0.0);            // turbulence.py:110
  sc.c_mu = prm->c_mu; sc.alpha = prm->alpha; sc.beta = prm->beta;
  sc.sigma = prm->sigma; sc.sigma_star = prm->sigma_star; sc.c_lim = prm->c_lim;
  sc.lim_scale = (double)((T)2 / (T)prm->c_mu);   // the kernel's former per-cell (T)2 / (T)c_mu, bit for bit
  sc.k_in = prm->k_in; sc.om_in = prm->omega_in; sc.nut_in = prm->k_in / prm->omega_in;
#ifdef CW_TURB_PERCELL   // developer comparison: the per-cell kernel
  (k_turbulence<T><<<dim3((c->d.nx + ST_BX - 1) / ST_BX, (c->d.ny + ST_BY - 1) / ST_BY,
                          (c->d.nz + ZT_TURB - 1) / ZT_TURB), B3, 0, st>>>(c->d, P.u, P.v, P.w, kin, win, P.k, P.om, P.nut, (T*)c->speed, sc, rep, c->gate), ++c->launches);
#elif defined(CW_TURB_ZMARCH)   // developer comparison: the z-march kernel
  (k_turbulence_z<T><<<dim3((c->d.nx + 31) / 32, (c->d.ny + 7) / 8, (c->d.nz + TURB_CZ - 1) / TURB_CZ), dim3(32, 8), 0,
                       st>>>(c->d, P.u, P.v, P.w, kin, win, P.k, P.om, P.nut, (T*)c->speed, sc, rep, c->gate),
   ++c->launches);
#else
  (k_turbulence_c<T><<<dim3((c->d.nx + ST_BX - 1) / ST_BX, (c->d.ny + ST_BY - 1) / ST_BY,
                            (c->d.nz + TURB_ZT - 1) / TURB_ZT), B3, 0, st>>>(c->d, P.u, P.v, P.w, kin, win, P.k, P.om, P.nut,
                                                                   (T*)c->speed, sc, rep, c->gate),
   ++c->launches);
#endif
  (k_turb_check<<<1, 1, 0, st>>>(rep, c->gate), ++c->launches);
}

template <typename T>
static StepPtrs<T> ptrs_of(const cw_fields* f) {
  StepPtrs<T> P;
  P.u = (T*)f->u; P.v = (T*)f->v; P.w = (T*)f->w; P.p = (T*)f->p;
  P.k = (T*)f->k; P.om = (T*)f->omega; P.nut = (T*)f->nu_t;
  P.lab = (const int8_t*)f->labels; P.lab_ver = f->labels_version; P.g = (const T*)f->g;
  return P;
}

// region means of the current state (k_region_partials + a fold): into
// reg_out / reg_cout, or (accumulate) added to reg_sums in step order
template <typename T>
static void launch_regions(cw_ctx* c, const cw_fields* f, bool accumulate, cudaStream_t st) {
  const RegionBoxes& B = c->reg_boxes;
  const int nb = std::min(nblk(c->ncell), 1024);
  (k_region_partials<T><<<nb, 256, 0, st>>>(c->d, c->grid.origin[0], c->grid.origin[1], c->grid.origin[2],
      (const T*)f->u, (const T*)f->v, (const T*)f->w, (const int8_t*)f->labels, B, c->reg_part, c->reg_cnt),
   ++c->launches);
  if (accumulate)
    (k_region_accum<<<1, 64, 0, st>>>(nb, B.n, c->reg_part, c->reg_cnt, c->reg_sums, c->reg_counts, c->gate),
     ++c->launches);
  else
    (k_region_fold<<<1, 64, 0, st>>>(nb, B.n, c->reg_part, c->reg_cnt, c->reg_out, c->reg_cout), ++c->launches);
}

// one full step (solver.py:407-461): no copies, stage temporaries chained
template <typename T>
static int enqueue_step(cw_ctx* c, const cw_fields* f, const cw_params* prm, double tol, cudaStream_t st) {
  DevReport* rep = c->rep_live;
  const StepPtrs<T> P = ptrs_of<T>(f);
  const bool turb = prm->turbulence != 0;
  auto mark = [&](int i) { if (c->timing) cudaEventRecord(c->ev[i], st); };
  (k_report_init<<<1, 1, 0, st>>>(rep), ++c->launches);
  // cw_step_defer_kw: k, omega arrive during the projection (their first
  // readers, the upwind step and the first boundary pass's k / omega / nu_t
  // writes, move behind it); without composed lists the step waits here
  T* acell = nullptr;
  bool defer_kw = false;
  if (c->wait_kw) {
    defer_kw = have_bc_lists(c, P.lab, P.lab_ver, st) && c->bc_nf >= 0;
    if (defer_kw && turb) {
      acell = (T*)cw_internal_scratch(c, 22, 3 * (size_t)c->ncell * sizeof(T));
      defer_kw = acell != nullptr;
    }
    if (!defer_kw) {
      CW_CUDA(cudaStreamWaitEvent(st, c->wait_kw, 0));
      c->wait_kw = nullptr;
    }
  }
  mark(0);
  st_advect<T>(c, P, prm, (T*)c->tk, (T*)c->tw, st, acell);  // "advect"
  mark(1);
  if (c->wait_nut) {   // nu_t is first read by the diffusion
    CW_CUDA(cudaStreamWaitEvent(st, c->wait_nut, 0));
    c->wait_nut = nullptr;
  }
  st_diffuse<T>(c, P, prm, st);                               // "diffuse"
  mark(2);
  st_drag<T>(c, P, prm, f->has_drag, st);                     // "drag"
  mark(3);
  StepPtrs<T> B = P;                                          // k, omega after upwind live in tk, tw
  if (turb) { B.k = (T*)c->tk; B.om = (T*)c->tw; }
  BcFields<T> F1{B.u, B.v, B.w, B.p, B.k, B.om, B.nut};
  if (c->wait_p) {     // p is first touched by the boundary writes (outlet copies)
    CW_CUDA(cudaStreamWaitEvent(st, c->wait_p, 0));
    c->wait_p = nullptr;
  }
  launch_bc<T>(c, F1, P.lab, P.lab_ver, prm, st, defer_kw ? BC_UVWP : BC_ALL);   // "boundary"
  mark(4);
  int rc = st_project<T>(c, P, f, prm, tol, rep, st);         // "project"
  if (rc) return rc;
  if (defer_kw) {   // the deferred k / omega part of the step, same writes
    // it also runs after a failed projection (device status 1 or 4): the
    // reference has advected k, omega and written their boundary values
    // before project() raises
    constexpr unsigned PASS = (1u << 1) | (1u << 4);
    CW_CUDA(cudaStreamWaitEvent(st, c->wait_kw, 0));
    c->wait_kw = nullptr;
    if (turb)
      (k_upwind_saved<T><<<g3(c->d.nx, c->d.ny, c->d.nz), B3, 0, st>>>(c->d, acell, P.k, P.om, (T*)c->tk, (T*)c->tw,
                                                                       (T)prm->dt, c->gate, PASS), ++c->launches);
    launch_bc<T>(c, F1, P.lab, P.lab_ver, prm, st, BC_KWN, PASS);
  }
  mark(5);
  if (turb) st_turb<T>(c, P, prm, B.k, B.om, rep, st);        // "turbulence"
  mark(6);
  BcFields<T> F2{P.u, P.v, P.w, P.p, P.k, P.om, P.nut};
  launch_bc<T>(c, F2, P.lab, P.lab_ver, prm, st);                        // "boundary2"
  (k_speed_max_flat<T><<<4 * 148, B3R, 0, st>>>(c->d, P.u, P.v, P.w, rep, c->gate),
   ++c->launches);
  mark(7);
  if (c->reg_n > 0) launch_regions<T>(c, f, true, st);        // trailing-window region sums
  (k_report_commit<<<1, 1, 0, st>>>(c->rep_live, c->rep, c->slot_dev), ++c->launches);
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

// a single reference stage function on a state (tests / stage-level API)
template <typename T>
static int enqueue_stage(cw_ctx* c, const cw_fields* f, const cw_params* prm, int stage, double tol, int slot,
                         cudaStream_t st) {
  DevReport* rep = c->rep + slot;
  const StepPtrs<T> P = ptrs_of<T>(f);
  const Dims& d = c->d;
  const size_t cb = c->ncell * sizeof(T);
  const size_t fb[3] = {c->nu_ * sizeof(T), c->nv_ * sizeof(T), c->nw_ * sizeof(T)};
  T* cu[3] = {P.u, P.v, P.w};
  const int ncomp = d.is2d ? 2 : 3;
  (k_report_init<<<1, 1, 0, st>>>(rep), ++c->launches);
  switch (stage) {
    case CW_STAGE_ADVECT:
      st_advect<T>(c, P, prm, (T*)c->tk, (T*)c->tw, st);
      if (prm->turbulence) {
        CW_CUDA(cudaMemcpyAsync(P.k, c->tk, cb, cudaMemcpyDeviceToDevice, st));
        CW_CUDA(cudaMemcpyAsync(P.om, c->tw, cb, cudaMemcpyDeviceToDevice, st));
      }
      for (int a = 0; a < ncomp; ++a) CW_CUDA(cudaMemcpyAsync(cu[a], c->adv[a], fb[a], cudaMemcpyDeviceToDevice, st));
      break;
    case CW_STAGE_DIFFUSE:
      for (int a = 0; a < ncomp; ++a) CW_CUDA(cudaMemcpyAsync(c->adv[a], cu[a], fb[a], cudaMemcpyDeviceToDevice, st));
      st_diffuse<T>(c, P, prm, st);
      break;
    case CW_STAGE_DRAG:
      st_drag<T>(c, P, prm, f->has_drag, st);
      break;
    case CW_STAGE_BOUNDARY: {
      BcFields<T> F{P.u, P.v, P.w, P.p, P.k, P.om, P.nut};
      launch_bc<T>(c, F, P.lab, P.lab_ver, prm, st);
      break;
    }
    case CW_STAGE_PROJECT: {
      if (!c->have_op) return fail(CW_ERR_INVALID, "cw_set_operator has not been called");
      int rc = st_project<T>(c, P, f, prm, tol, rep, st);
      if (rc) return rc;
      break;
    }
    case CW_STAGE_PRE: {        // step() up to the projection; k, omega stay in tk, tw until POST
      const bool turb = prm->turbulence != 0;
      if (d.kg0 > 0 || d.kg0 + d.nz < d.nzg) {   // a z-slab window: does the step's reach fit its halo?
        (k_wmax_window<T><<<std::min(nblk(c->nw_), 4 * c->num_sms), 256, 0, st>>>(c->nw_, P.w, rep, c->gate),
         ++c->launches);
        (k_halo_gate<T><<<1, 1, 0, st>>>(d, prm->dt, rep, c->gate), ++c->launches);
      }
      st_advect<T>(c, P, prm, (T*)c->tk, (T*)c->tw, st);
      st_diffuse<T>(c, P, prm, st);
      st_drag<T>(c, P, prm, f->has_drag, st);
      StepPtrs<T> B = P;
      if (turb) { B.k = (T*)c->tk; B.om = (T*)c->tw; }
      BcFields<T> F1{B.u, B.v, B.w, B.p, B.k, B.om, B.nut};
      launch_bc<T>(c, F1, P.lab, P.lab_ver, prm, st);
      break;
    }
    case CW_STAGE_SOLVE: {
      if (!c->have_op) return fail(CW_ERR_INVALID, "cw_set_operator has not been called");
      const bool tpcg = c->pcg_timed < (int)c->pev.size() / 2;
      if (tpcg) cudaEventRecord(c->pev[2 * c->pcg_timed], st);
      int rc = launch_pcg<T>(c, f, rep, prm->dt, tol, st);
      ++c->launches;
      if (tpcg) cudaEventRecord(c->pev[2 * c->pcg_timed++ + 1], st);
      if (rc) return rc;
      break;
    }
    case CW_STAGE_POST: {       // step() after the projection
      st_project_tail<T>(c, P, prm, rep, st);
      if (prm->turbulence) st_turb<T>(c, P, prm, (const T*)c->tk, (const T*)c->tw, rep, st);
      BcFields<T> F2{P.u, P.v, P.w, P.p, P.k, P.om, P.nut};
      launch_bc<T>(c, F2, P.lab, P.lab_ver, prm, st);
      (k_speed_max_flat<T><<<4 * 148, B3R, 0, st>>>(d, P.u, P.v, P.w, rep, c->gate),
       ++c->launches);
      break;
    }
    case CW_STAGE_TURBULENCE:
      CW_CUDA(cudaMemcpyAsync(c->tk, P.k, cb, cudaMemcpyDeviceToDevice, st));
      CW_CUDA(cudaMemcpyAsync(c->tw, P.om, cb, cudaMemcpyDeviceToDevice, st));
      st_turb<T>(c, P, prm, (const T*)c->tk, (const T*)c->tw, rep, st);
      break;
    default:
      return fail(CW_ERR_INVALID, "unknown stage");
  }
  (k_slot_bump<<<1, 1, 0, st>>>(c->slot_dev), ++c->launches);   // this report went to rep[slot] directly
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

// ---------------------------------------------------------------------------
// probes and streamlines (run_simulation probes, scenario.py:473-478;
// trace_streamlines, solver.py:488-532)

static Frame frame_of(const cw_ctx* c) {
  Frame fr;
  const double h[3] = {c->grid.dx, c->grid.dy, c->grid.dz};
  const int n[3] = {c->d.nx, c->d.ny, c->d.nz};
  for (int a = 0; a < 3; ++a) {
    fr.o[a] = c->grid.origin[a];
    fr.h[a] = h[a];
    fr.lo[a] = c->grid.origin[a];
    fr.hi[a] = c->grid.origin[a] + h[a] * n[a];   // GridSpec.extent(): lo + spacing * shape
  }
  return fr;
}

extern "C" int cw_probe(cw_ctx* c, const cw_fields* f, int n, const double* pts, double* out, void* stream) {
  if (!c || !f || (n > 0 && (!pts || !out))) return fail(CW_ERR_INVALID, "null argument");
  if (c->d.kg0 != 0 || c->d.nz != c->d.nzg) return fail(CW_ERR_INVALID, "probes need a whole-grid context");
  if (n == 0) return CW_OK;
  CW_CUDA(cudaSetDevice(c->device));
  const Frame fr = frame_of(c);
  if (c->prec == 4)
    (k_probe<float><<<(n + 127) / 128, 128, 0, S(stream)>>>(c->d, fr, (const float*)f->u, (const float*)f->v,
                                                            (const float*)f->w, pts, n, out), ++c->launches);
  else
    (k_probe<double><<<(n + 127) / 128, 128, 0, S(stream)>>>(c->d, fr, (const double*)f->u, (const double*)f->v,
                                                             (const double*)f->w, pts, n, out), ++c->launches);
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

extern "C" int cw_streamlines(cw_ctx* c, const cw_fields* f, int nseeds, const double* seeds, double step_len,
                              int max_steps, double min_speed, double* paths, int* len, void* stream) {
  if (!c || !f || (nseeds > 0 && (!seeds || !paths || !len))) return fail(CW_ERR_INVALID, "null argument");
  if (max_steps < 0) return fail(CW_ERR_INVALID, "max_steps < 0");
  if (c->d.kg0 != 0 || c->d.nz != c->d.nzg) return fail(CW_ERR_INVALID, "streamlines need a whole-grid context");
  if (nseeds == 0) return CW_OK;
  CW_CUDA(cudaSetDevice(c->device));
  const Frame fr = frame_of(c);
  const int nb = (nseeds + 63) / 64;
  if (c->prec == 4)
    (k_streamlines<float><<<nb, 64, 0, S(stream)>>>(c->d, fr, (const float*)f->u, (const float*)f->v,
                                                    (const float*)f->w, seeds, nseeds, step_len, max_steps,
                                                    min_speed, paths, len), ++c->launches);
  else
    (k_streamlines<double><<<nb, 64, 0, S(stream)>>>(c->d, fr, (const double*)f->u, (const double*)f->v,
                                                     (const double*)f->w, seeds, nseeds, step_len, max_steps,
                                                     min_speed, paths, len), ++c->launches);
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

// ---------------------------------------------------------------------------
// z-slab solves

extern "C" int cw_slab_buffers_get(cw_ctx* c, cw_slab_buffers* out) {
  if (!c || !out) return fail(CW_ERR_INVALID, "null argument");
  out->r0 = c->r0; out->r1 = c->r1; out->p0 = c->p0; out->p1 = c->p1; out->z = c->z; out->Ap = c->Ap;
  out->xbar = c->xbar; out->xval = c->xval;
  out->o0 = c->d.o0; out->o1 = c->d.o1;
  return CW_OK;
}

extern "C" int cw_pcg_chunk_of(const cw_grid* g, int precision, int device, int* zc) {
  if (!g || !zc || (precision != 4 && precision != 8)) return fail(CW_ERR_INVALID, "bad argument");
  CW_CUDA(cudaSetDevice(device));
  int per_sm = 0, sms = 0;
  size_t smem = 0;
  const int rc = precision == 4 ? pcg_occupancy<float>(&per_sm, &smem) : pcg_occupancy<double>(&per_sm, &smem);
  if (rc != CW_OK) return rc;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int tiles = ((g->nx + TX - 1) / TX) * ((g->ny + TY - 1) / TY);
  *zc = choose_zc(tiles, g->nz, std::max(1, per_sm * sms));
  return CW_OK;
}

extern "C" int cw_set_pcg_chunk(cw_ctx* c, int zc) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  const int nown = c->d.o1 - c->d.o0;
  if (zc < 1 || (nown + zc - 1) / zc * ((c->ntx * c->nty + 31) / 32) > CW_PCG_MAXG)
    return fail(CW_ERR_INVALID, "bad PCG chunk size");
  c->zc = std::min(zc, nown);
  plan_units(c);
  return alloc_partials(c);
}

extern "C" int cw_slab_chunks(cw_ctx* c, int chunk0, int nchunk_g) {
  if (!c || chunk0 < 0 || nchunk_g < 1 || nchunk_g * ((c->ntx * c->nty + 31) / 32) > CW_MAX_CHUNKS ||
      chunk0 + c->U / (c->ntx * c->nty) > nchunk_g)
    return fail(CW_ERR_INVALID, "bad chunk range");
  c->chunk0 = chunk0;
  c->nchunk_g = nchunk_g;
  return CW_OK;
}

extern "C" int cw_pcg_chunks(cw_ctx* c, int* zc, int* nchunk) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  if (zc) *zc = c->zc;
  if (nchunk) *nchunk = c->U / (c->ntx * c->nty);
  return CW_OK;
}

extern "C" int cw_slab_attach(cw_ctx* c, int slab, int nslab, const cw_slab_buffers* lower,
                              const cw_slab_buffers* upper, const cw_slab_buffers* root) {
  if (!c || !root) return fail(CW_ERR_INVALID, "null argument");
  if (nslab < 1 || nslab > CW_MAX_SLABS || slab < 0 || slab >= nslab) return fail(CW_ERR_INVALID, "bad slab index");
  const bool has_lo = c->d.kg0 + c->d.o0 > 0, has_hi = c->d.kg0 + c->d.o1 < c->d.nzg;
  if (has_lo != (lower && lower->z != nullptr) || has_hi != (upper && upper->z != nullptr))
    return fail(CW_ERR_INVALID, "neighbour buffers must be given exactly for interior slab faces");
  if ((lower && lower->z && lower->o1 < 1) || (upper && upper->z && upper->o0 < 1))
    return fail(CW_ERR_INVALID, "neighbour slab has no halo plane");
  c->slab = slab;
  c->nslab = nslab;
  c->lower = lower ? *lower : cw_slab_buffers{};
  c->upper = upper ? *upper : cw_slab_buffers{};
  c->root = *root;
  return CW_OK;
}

template <typename T>
static int group_pcg(cw_ctx** cs, const cw_fields* fs, int n, const cw_params* prm, double pcg_tol,
                     cudaStream_t st) {
  cw_ctx* c0 = cs[0];
  // blocks per slab: every slab gets the same share of the co-resident blocks
  int umax = 0;
  for (int s = 0; s < n; ++s) umax = std::max(umax, cs[s]->U);
  const int bps = std::max(1, std::min(c0->max_blocks / n, umax));
  std::vector<PcgArgs<T>> args(n);
  int nchunk_g = 0;
  for (int s = 0; s < n; ++s) nchunk_g += cs[s]->U / (cs[s]->ntx * cs[s]->nty);
  if (nchunk_g * ((c0->ntx * c0->nty + 31) / 32) > CW_MAX_CHUNKS)
    return fail(CW_ERR_INVALID, "too many PCG fold items over the slabs");
  for (int s = 0, ch = 0; s < n; ++s) {
    cw_ctx* c = cs[s];
    c->chunk0 = ch;
    c->nchunk_g = nchunk_g;
    ch += c->U / (c->ntx * c->nty);
    const double tol = pcg_tol < 0 || std::isnan(pcg_tol) ? c->tol_default : pcg_tol;
    const int slot = c->head++;
    c->slot_dt[slot] = prm->dt;
    DevReport* rep = c->rep + slot;
    (k_report_init<<<1, 1, 0, st>>>(rep), ++c->launches);
    fill_pcg_args<T>(args[s], c, &fs[s], rep, prm->dt, tol);
    args[s].probe_mode = 0;   // timing probes assume one slab
    cw_slab_buffers lo{}, hi{}, root{};
    if (s > 0) cw_slab_buffers_get(cs[s - 1], &lo);
    if (s + 1 < n) cw_slab_buffers_get(cs[s + 1], &hi);
    cw_slab_buffers_get(c0, &root);
    const long long pplane = (long long)c->nxp * c->d.ny;
    args[s].nslab = n;
    args[s].slab = s;
    args[s].lo = peer_of<T>(lo, lo.o1, pplane);
    args[s].hi = peer_of<T>(hi, hi.o0 - 1, pplane);
    args[s].xbar = c0->xbar;
    args[s].xval = c0->xval;
    CW_CUDA(cudaMemsetAsync(c->bar, 0, 64 * sizeof(unsigned), st));
    CW_CUDA(cudaMemsetAsync(c->tags, 0, 2 * (size_t)c->part_stride * sizeof(unsigned), st));
  }
  CW_CUDA(cudaMemsetAsync(c0->xbar, 0, 64 * sizeof(unsigned), st));
  CW_CUDA(cudaMemcpyAsync(c0->slab_args, args.data(), n * sizeof(PcgArgs<T>), cudaMemcpyHostToDevice, st));
  const PcgArgs<T>* dargs = (const PcgArgs<T>*)c0->slab_args;
  int ibps = bps;
  void* kargs[] = {(void*)&dargs, (void*)&ibps};
  CW_CUDA(cudaLaunchCooperativeKernel((const void*)k_pcg_slabs<T>, dim3(n * bps), dim3(PCG_THREADS), kargs,
                                      c0->pcg_smem, st));
  ++c0->launches;
  for (int s = 0; s < n; ++s) (k_slot_bump<<<1, 1, 0, st>>>(cs[s]->slot_dev), ++cs[s]->launches);
  CW_CUDA(cudaStreamSynchronize(st));   // the host argument array goes out of scope
  return CW_OK;
}

extern "C" int cw_slab_group_pcg(cw_ctx** cs, const cw_fields* fs, int n, const cw_params* prm, double pcg_tol,
                                 void* stream) {
  if (!cs || !fs || !prm || n < 1) return fail(CW_ERR_INVALID, "null argument");
  if (n > CW_MAX_SLABS) return fail(CW_ERR_INVALID, "too many slabs");
  for (int s = 0; s < n; ++s) {
    cw_ctx* c = cs[s];
    if (!c) return fail(CW_ERR_INVALID, "null context");
    if (!c->have_op) return fail(CW_ERR_INVALID, "cw_set_operator has not been called");
    if (c->device != cs[0]->device || c->prec != cs[0]->prec || c->d.nx != cs[0]->d.nx ||
        c->d.ny != cs[0]->d.ny || c->d.nzg != cs[0]->d.nzg)
      return fail(CW_ERR_INVALID, "slabs must share device, precision and global grid");
    const int lo = c->d.kg0 + c->d.o0, hi = c->d.kg0 + c->d.o1;
    if ((s == 0 && lo != 0) || (s + 1 == n && hi != c->d.nzg) ||
        (s > 0 && cs[s - 1]->d.kg0 + cs[s - 1]->d.o1 != lo))
      return fail(CW_ERR_INVALID, "slabs must tile the global grid in z order");
    if (c->head + 1 > RING) return fail(CW_ERR_INVALID, "report ring full: call cw_read_reports");
  }
  CW_CUDA(cudaSetDevice(cs[0]->device));
  return cs[0]->prec == 4 ? group_pcg<float>(cs, fs, n, prm, pcg_tol, S(stream))
                          : group_pcg<double>(cs, fs, n, prm, pcg_tol, S(stream));
}

extern "C" int cw_ipc_get(void* p, unsigned char handle[64]) {
  if (!p || !handle) return fail(CW_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  CW_CUDA(cudaIpcGetMemHandle(&h, p));
  std::memcpy(handle, &h, 64);
  return CW_OK;
}

extern "C" int cw_ipc_open(const unsigned char handle[64], int device, void** p) {
  if (!handle || !p) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CW_CUDA(cudaIpcOpenMemHandle(p, h, cudaIpcMemLazyEnablePeerAccess));
  return CW_OK;
}

extern "C" int cw_ipc_close(void* p) {
  if (!p) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaIpcCloseMemHandle(p));
  return CW_OK;
}

extern "C" int cw_run_stage(cw_ctx* c, const cw_fields* f, const cw_params* prm, const cw_inlet* inl, int stage,
                            double pcg_tol, void* stream) {
  if (!c || !f || !prm || !inl) return fail(CW_ERR_INVALID, "null argument");
  if (c->head + 1 > RING) return fail(CW_ERR_INVALID, "report ring full: call cw_read_reports");
  if (stage == CW_STAGE_DRAG && f->has_drag && !f->g) return fail(CW_ERR_INVALID, "has_drag without g");
  CW_CUDA(cudaSetDevice(c->device));
  int rc = upload_inlet(c, inl, S(stream));
  if (rc) return rc;
  const double tol = pcg_tol < 0 || std::isnan(pcg_tol) ? c->tol_default : pcg_tol;
  const int slot = c->head++;
  c->slot_dt[slot] = prm->dt;
  return c->prec == 4 ? enqueue_stage<float>(c, f, prm, stage, tol, slot, S(stream))
                      : enqueue_stage<double>(c, f, prm, stage, tol, slot, S(stream));
}

// One step as a CUDA-graph replay: the key is everything the captured
// kernels bake in (field pointers, labels version, parameters, tolerance,
// trailing-window regions).  The boundary-write lists are built first (their
// construction synchronises), outside the capture.  Returns -1 when this step
// cannot be captured (graphs then stay off for the context).
static int graph_step(cw_ctx* c, const cw_fields* f, const cw_params* prm, double tol, cudaStream_t st) {
  if (f->labels_version != 0 && !(c->bc_lab == f->labels && c->bc_ver == f->labels_version)) {
    if (build_bc_lists(c, (const int8_t*)f->labels, f->labels_version, st) != 0) { cudaGetLastError(); return -1; }
  }
  std::string key;
  key.append((const char*)f, sizeof(cw_fields));
  key.append((const char*)prm, sizeof(cw_params));
  key.append((const char*)&tol, sizeof(double));
  key.append((const char*)&c->reg_n, sizeof(int));
  if (c->reg_n > 0) {
    key.append((const char*)&c->reg_boxes, sizeof(RegionBoxes));
    key.append((const char*)&c->reg_sums, sizeof(void*));
    key.append((const char*)&c->reg_counts, sizeof(void*));
  }
  cw_ctx::GraphEntry* hit = nullptr;
  for (auto& e : c->gcache)
    if (e.key == key) { hit = &e; break; }
  if (!hit) {
    if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      c->graphs = false;
      return -1;
    }
    const long long l0 = c->launches;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      c->graphs = false;
      return -1;
    }
    const int rc = c->prec == 4 ? enqueue_step<float>(c, f, prm, tol, c->cap_stream)
                                : enqueue_step<double>(c, f, prm, tol, c->cap_stream);
    const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &g);
    const long long nk = c->launches - l0;   // the step's kernels (gpu_launches evidence), counted per replay
    c->launches = l0;
    cudaGraphExec_t ex = nullptr;
    if (rc != CW_OK || ec != cudaSuccess || !g || cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      c->graphs = false;
      return -1;
    }
    cudaGraphDestroy(g);
    if (c->gcache.size() >= 8) {
      cudaGraphExecDestroy(c->gcache.front().exec);
      c->gcache.erase(c->gcache.begin());
    }
    c->gcache.push_back(cw_ctx::GraphEntry{key, ex, nk});
    hit = &c->gcache.back();
  }
  CW_CUDA(cudaGraphLaunch(hit->exec, st));
  c->launches += hit->kernels;
  return CW_OK;
}

extern "C" int cw_step(cw_ctx* c, const cw_fields* f, const cw_params* prm, const cw_inlet* inl, double pcg_tol,
                       int nsteps, void* stream) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  // the one-shot waits of cw_step_defer belong to this call only: cleared on
  // every exit (the first enqueued step consumes them)
  struct DeferGuard {
    cw_ctx* c;
    ~DeferGuard() { c->wait_nut = nullptr; c->wait_p = nullptr; c->wait_kw = nullptr; }
  } defer_guard{c};
  if (!f || !prm || !inl) return fail(CW_ERR_INVALID, "null argument");
  if (!c->have_op) return fail(CW_ERR_INVALID, "cw_set_operator has not been called");
  if (nsteps < 0) return fail(CW_ERR_INVALID, "nsteps < 0");
  if (c->head + nsteps > RING) return fail(CW_ERR_INVALID, "report ring full: call cw_read_reports");
  if (f->has_drag && !f->g) return fail(CW_ERR_INVALID, "has_drag without a drag-coefficient buffer");
  CW_CUDA(cudaSetDevice(c->device));
  int rc = upload_inlet(c, inl, S(stream));
  if (rc) return rc;
  if (c->timing && !c->ev_made) {
    for (auto& e : c->ev) CW_CUDA(cudaEventCreate(&e));
    c->ev_made = true;
  }
  const double tol = pcg_tol < 0 || std::isnan(pcg_tol) ? c->tol_default : pcg_tol;
  for (int s = 0; s < nsteps; ++s) {
    const int slot = c->head++;
    c->slot_dt[slot] = prm->dt;
    const bool timed = c->timing || c->pcg_timed < (int)c->pev.size() / 2 || c->adv_timed < (int)c->aev.size() / 3;
    if (c->graphs && !timed && !c->wait_nut && !c->wait_p && !c->wait_kw) {
      rc = graph_step(c, f, prm, tol, S(stream));
      if (rc == CW_OK) continue;
      if (rc != -1) return rc;   // -1: capture not possible here, run the step directly
    }
    rc = c->prec == 4 ? enqueue_step<float>(c, f, prm, tol, S(stream))
                      : enqueue_step<double>(c, f, prm, tol, S(stream));
    if (rc) return rc;
  }
  return CW_OK;
}

extern "C" int cw_read_reports(cw_ctx* c, cw_report* out, int n, int* n_out, void* stream) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  const int m = std::min(n, c->head);
  std::vector<DevReport> dr(std::max(c->head, 1));
  if (c->head > 0)
    CW_CUDA(cudaMemcpy(dr.data(), c->rep, c->head * sizeof(DevReport), cudaMemcpyDeviceToHost));
  if (c->timing && c->ev_made && c->head > 0) {
    for (int i = 0; i < 7; ++i) cudaEventElapsedTime(&c->stage_ms[i], c->ev[i], c->ev[i + 1]);
  }
  const double hmin = std::min(c->grid.dx, std::min(c->grid.dy, c->grid.dz));
  int first_err = CW_OK;
  for (int i = 0; i < c->head; ++i) {
    const DevReport& r = dr[i];
    cw_report o{};
    o.iterations = r.iterations;
    o.converged = r.converged;
    o.criterion = r.criterion;
    double smax, db, da;
    if (c->prec == 4) {
      float t;
      std::memcpy(&t, &r.fmax[SLOT_SPEED], 4); smax = t;
      std::memcpy(&t, &r.fmax[SLOT_DIV_BEFORE], 4); db = t;
      std::memcpy(&t, &r.fmax[SLOT_DIV_AFTER], 4); da = t;
    } else {
      std::memcpy(&smax, &r.dmax[SLOT_SPEED], 8);
      std::memcpy(&db, &r.dmax[SLOT_DIV_BEFORE], 8);
      std::memcpy(&da, &r.dmax[SLOT_DIV_AFTER], 8);
    }
    o.cfl = std::max(smax, 1e-300) * c->slot_dt[i] / hmin;
    o.div_before = db;
    o.div_after = da;
    o.bad_cell = -1;
    switch (r.status) {
      case 0: o.status = CW_OK; break;
      case 1: o.status = CW_ERR_PCG; break;
      case 2:
        o.status = CW_ERR_NONFINITE;
        o.bad_field = r.bad_index[0] != 0x7fffffffffffffffLL ? 0 : 1;
        o.bad_cell = r.bad_index[o.bad_field];
        break;
      case 3: o.status = CW_ERR_TIMEOUT; break;
      case 4: o.status = CW_ERR_RHS; break;
      case 5: o.status = CW_ERR_HALO; o.bad_cell = r.halo_need; break;
      default: o.status = CW_ERR_CUDA; break;
    }
    if (o.status != CW_OK && first_err == CW_OK) first_err = o.status;
    if (i < m && out) out[i] = o;
  }
  if (n_out) *n_out = m;
  c->head = 0;
  CW_CUDA(cudaMemset(c->slot_dev, 0, sizeof(int)));
  CW_CUDA(cudaMemset(c->gate, 0, sizeof(int)));
  CW_CUDA(cudaMemset(c->bar, 0, 64 * sizeof(unsigned)));
  if (first_err != CW_OK) {
    const char* what = first_err == CW_ERR_PCG ? "pressure solve did not converge"
                       : first_err == CW_ERR_NONFINITE ? "turbulence update produced non-finite values"
                       : first_err == CW_ERR_RHS ? "right-hand side contains non-finite entries"
                       : first_err == CW_ERR_TIMEOUT ? "device grid barrier timed out"
                       : first_err == CW_ERR_HALO ? "z-slab halo too shallow for the step's reach"
                                                     : "device error";
    g_err = what;
  }
  return first_err;
}

extern "C" int cw_set_preconditioner(cw_ctx* c, int kind, double* tol_default) {
  if (!c || kind < 0 || kind > 2) return fail(CW_ERR_INVALID, "preconditioner kind must be 0, 1 or 2");
  c->precond = kind;
  c->tol_default = c->tol_kind[kind];
  if (tol_default) *tol_default = c->tol_default;
  return CW_OK;
}

extern "C" int cw_pcg_timing(cw_ctx* c, int max_launches) {
  if (!c || max_launches < 0) return fail(CW_ERR_INVALID, "bad argument");
  CW_CUDA(cudaSetDevice(c->device));
  for (auto& e : c->pev) cudaEventDestroy(e);
  c->pev.assign(2 * (size_t)max_launches, nullptr);
  for (auto& e : c->pev) CW_CUDA(cudaEventCreate(&e));
  c->pcg_timed = 0;
  for (auto& e : c->aev) cudaEventDestroy(e);
  c->aev.assign(3 * (size_t)max_launches, nullptr);
  for (auto& e : c->aev) CW_CUDA(cudaEventCreate(&e));
  c->adv_timed = 0;
  return CW_OK;
}

extern "C" int cw_read_pcg_timing(cw_ctx* c, float* ms, int n, int* n_out) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  const int m = std::min(n, c->pcg_timed);
  for (int i = 0; i < m; ++i) {
    CW_CUDA(cudaEventSynchronize(c->pev[2 * i + 1]));
    CW_CUDA(cudaEventElapsedTime(&ms[i], c->pev[2 * i], c->pev[2 * i + 1]));
  }
  if (n_out) *n_out = m;
  c->pcg_timed = 0;
  return CW_OK;
}

extern "C" int cw_read_adv_timing(cw_ctx* c, float* predict_ms, float* correct_ms, int n, int* n_out) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  const int m = std::min(n, c->adv_timed);
  for (int i = 0; i < m; ++i) {
    CW_CUDA(cudaEventSynchronize(c->aev[3 * i + 2]));
    CW_CUDA(cudaEventElapsedTime(&predict_ms[i], c->aev[3 * i], c->aev[3 * i + 1]));
    CW_CUDA(cudaEventElapsedTime(&correct_ms[i], c->aev[3 * i + 1], c->aev[3 * i + 2]));
  }
  if (n_out) *n_out = m;
  c->adv_timed = 0;
  return CW_OK;
}

extern "C" long long cw_launch_count(cw_ctx* c, int reset) {
  if (!c) return -1;
  const long long v = c->launches;
  if (reset) c->launches = 0;
  return v;
}

extern "C" int cw_turb_rollback(cw_ctx* c, const cw_fields* f, void* stream) {
  if (!c || !f) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  const int nb = std::min(nblk(c->ncell), 4 * c->num_sms * 8);
  if (c->prec == 4)
    (k_turb_rollback<float><<<nb, 256, 0, S(stream)>>>(c->ncell, (const float*)c->tk, (const float*)c->tw,
        (const float*)c->speed, (float*)f->k, (float*)f->omega, (float*)f->nu_t), ++c->launches);
  else
    (k_turb_rollback<double><<<nb, 256, 0, S(stream)>>>(c->ncell, (const double*)c->tk, (const double*)c->tw,
        (const double*)c->speed, (double*)f->k, (double*)f->omega, (double*)f->nu_t), ++c->launches);
  CW_CUDA(cudaGetLastError());
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  return CW_OK;
}

extern "C" int cw_proj_rollback(cw_ctx* c, const cw_fields* f, int turbulence, void* stream) {
  if (!c || !f) return fail(CW_ERR_INVALID, "null argument");
  CW_CUDA(cudaSetDevice(c->device));
  if (turbulence) {   // k, omega as advected this step (their boundary values written); nu_t untouched
    const int nb = std::min(nblk(c->ncell), 4 * c->num_sms * 8);
    if (c->prec == 4)
      (k_turb_rollback<float><<<nb, 256, 0, S(stream)>>>(c->ncell, (const float*)c->tk, (const float*)c->tw, nullptr,
                                                          (float*)f->k, (float*)f->omega, (float*)f->nu_t),
       ++c->launches);
    else
      (k_turb_rollback<double><<<nb, 256, 0, S(stream)>>>(c->ncell, (const double*)c->tk, (const double*)c->tw,
                                                           nullptr, (double*)f->k, (double*)f->omega,
                                                           (double*)f->nu_t),
       ++c->launches);
    CW_CUDA(cudaGetLastError());
  }
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  return CW_OK;
}

extern "C" int cw_ref_layout(cw_ctx* c, int direction, int field, const void* src, void* dst, void* stream) {
  if (!c || !src || !dst || direction < 0 || direction > 1 || field < 0 || field > 3)
    return fail(CW_ERR_INVALID, "cw_ref_layout: bad argument");
  CW_CUDA(cudaSetDevice(c->device));
  int ex = c->d.nx, ey = c->d.ny, ez = c->d.nz;
  if (field < 3) comp_extent(c->d, field, ex, ey, ez);
  const dim3 blk(32, 8);
  if (direction == 0) {
    const dim3 grd((ez + 31) / 32, (ex + 31) / 32, ey);
    if (c->prec == 4) (k_ref_to_dev<float><<<grd, blk, 0, S(stream)>>>((const double*)src, (float*)dst, ex, ey, ez), ++c->launches);
    else (k_ref_to_dev<double><<<grd, blk, 0, S(stream)>>>((const double*)src, (double*)dst, ex, ey, ez), ++c->launches);
  } else {
    const dim3 grd((ex + 31) / 32, (ez + 31) / 32, ey);
    if (c->prec == 4) (k_dev_to_ref<float><<<grd, blk, 0, S(stream)>>>((const float*)src, (double*)dst, ex, ey, ez), ++c->launches);
    else (k_dev_to_ref<double><<<grd, blk, 0, S(stream)>>>((const double*)src, (double*)dst, ex, ey, ez), ++c->launches);
  }
  CW_CUDA(cudaGetLastError());
  return CW_OK;
}

extern "C" int cw_set_max_iter(cw_ctx* c, int max_iter) {
  if (!c || max_iter < 0) return fail(CW_ERR_INVALID, "max_iter must be >= 0");
  c->max_iter = max_iter;
  return CW_OK;
}

extern "C" int cw_step_defer(cw_ctx* c, void* nu_t_ready, void* p_ready) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  c->wait_nut = (cudaEvent_t)nu_t_ready;
  c->wait_p = (cudaEvent_t)p_ready;
  return CW_OK;
}

extern "C" int cw_step_defer_kw(cw_ctx* c, void* k_omega_ready) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  c->wait_kw = (cudaEvent_t)k_omega_ready;
  return CW_OK;
}

extern "C" int cw_set_stage_timing(cw_ctx* c, int enabled) {
  if (!c) return fail(CW_ERR_INVALID, "null argument");
  c->timing = enabled != 0;
  return CW_OK;
}

extern "C" int cw_read_stage_timings(cw_ctx* c, float out_ms[7]) {
  if (!c || !out_ms) return fail(CW_ERR_INVALID, "null argument");
  for (int i = 0; i < 7; ++i) out_ms[i] = c->stage_ms[i];
  return CW_OK;
}

// ---------------------------------------------------------------------------
// region averages

extern "C" int cw_region_speed(cw_ctx* c, const cw_fields* f, int n, const double* lo, const double* hi,
                               double* mean_out, long long* count_out, void* stream) {
  if (!c || !f || n < 1 || n > 16 || !lo || !hi) return fail(CW_ERR_INVALID, "bad region arguments (1..16 boxes)");
  CW_CUDA(cudaSetDevice(c->device));
  const RegionBoxes keep = c->reg_boxes;
  RegionBoxes& B = c->reg_boxes;
  B.n = n;
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < 3; ++a) { B.lo[b][a] = lo[3 * b + a]; B.hi[b][a] = hi[3 * b + a]; }
  if (c->prec == 4) launch_regions<float>(c, f, false, S(stream));
  else launch_regions<double>(c, f, false, S(stream));
  c->reg_boxes = keep;   // a pending cw_step_regions set stays in force
  CW_CUDA(cudaGetLastError());
  CW_CUDA(cudaMemcpyAsync(mean_out, c->reg_out, n * sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaMemcpyAsync(count_out, c->reg_cout, n * sizeof(long long), cudaMemcpyDeviceToHost, S(stream)));
  CW_CUDA(cudaStreamSynchronize(S(stream)));
  return CW_OK;
}

extern "C" int cw_step_regions(cw_ctx* c, int n, const double* lo, const double* hi, double* sums_dev,
                               long long* counts_dev) {
  if (!c || n < 0 || n > 16) return fail(CW_ERR_INVALID, "bad region arguments (0..16 boxes)");
  if (n > 0 && (!lo || !hi || !sums_dev || !counts_dev)) return fail(CW_ERR_INVALID, "null argument");
  c->reg_n = n;
  c->reg_boxes.n = n;
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < 3; ++a) { c->reg_boxes.lo[b][a] = lo[3 * b + a]; c->reg_boxes.hi[b][a] = hi[3 * b + a]; }
  c->reg_sums = sums_dev;
  c->reg_counts = counts_dev;
  return CW_OK;
}
