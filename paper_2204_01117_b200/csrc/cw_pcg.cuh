// Pressure projection: one persistent cooperative kernel runs the whole
// warm-started PCG of project() (solver.py:246-280) / pcg_solve()
// (linalg.py:310-368) on the device, with no host round trip per iteration.
//
// Operators are matrix-free on the x-fastest grid:
//   A p  : 7-point negated Laplacian, diagonal d_i = sum of 1/h^2 over
//          neighbours that are unknowns or outlets (linalg.py:81-112).
//   W r  : untruncated AI1 preconditioner W = K^T K (linalg.py:201-232),
//          applied as two 4-point sweeps  y = s (r + w * sum_a w_a q_{i-e_a}),
//          z = y + (w/d) sum_a w_a y_{i+e_a}  with q = r/d, s = (2-w) w / d.
// Both read a 1-byte per-cell code (bit 6: unknown; bits 0..5: neighbour
// +x,-x,+y,-y,+z,-z is an unknown or an outlet) and a 64-entry table of
// (d, 1/d, s w, w/d) -- no CSR, no stored coefficients.
//
// Data movement (B200): the PCG vectors live on a pitched copy of the grid
// (row pitch nxp = nx rounded up to 16 elements, exact zeros off the
// unknowns) so that every (x,y)-tile-with-halo of one z-plane is a single
// TMA box (cp.async.bulk.tensor.3d; out-of-range elements are zero-filled by
// the hardware, which is exactly the operator's boundary rule).  Each block
// marches 32x32 tiles through z (4 rows per thread); one thread keeps a
// DEPTH-stage shared-memory ring of planes in flight (mbarrier complete_tx).
//
// Each PCG iteration is two grid phases separated by a grid barrier that
// also completes a deterministic fp64 reduction:
//   phase A: p' = z + beta p  (recomputed on the tile halo), x += alpha_prev p,
//            Ap = A p', partial p'.Ap
//   phase B: r' = r - alpha Ap (recomputed on the halo), z = W r',
//            partials r'.z and max|r'|
// Storage: p, z, Ap, x in the state precision; r in float64 (a float32
// recursive residual drifts by ~eps*|b| per iteration, several percent of the
// max-norm target 10^-4.5 max|b|, which flips stopping decisions); A p is
// evaluated in float64 arithmetic.  Partials are kept per block over a fixed
// unit->block map and every block folds them in the same fixed order: all
// blocks agree bit-for-bit on alpha/beta and runs are deterministic.
#pragma once
#include <cuda.h>

#include "cw_common.cuh"
#include "cw_step.cuh"

namespace cw {

constexpr int PCG_TX = 32, PCG_TY = 32;                 // tile (cells)
#ifndef CW_PCG_THREADS
#define CW_PCG_THREADS 256
#endif
#ifndef CW_PCG_MINB
#define CW_PCG_MINB 2
#endif
constexpr int PCG_THREADS = CW_PCG_THREADS;
constexpr int PCG_RSTEP = PCG_THREADS / PCG_TX;         // 8 rows per thread sweep
constexpr int PCG_RPT = PCG_TY / PCG_RSTEP;             // 4 rows per thread
constexpr int BOX_Y = PCG_TY + 2;
constexpr int HW = PCG_TX + 2, HH = PCG_TY + 2;         // halo tile (34 x 34)
constexpr int YW = PCG_TX + 1, YH = PCG_TY + 1;         // y tile (33 x 33)

// Halo box geometry per element type.  A TMA box must START on a 16-byte
// boundary in x, so the box begins SH elements left of the tile (SH = 16 B /
// element) and is BW elements wide; halo column hx (hx = 0 is x = i0-1)
// lives at box column hx + OFF.
template <typename E>
struct Halo {
  static constexpr int SH = 16 / (int)sizeof(E);
  static constexpr int BW = ((SH + PCG_TX + 1) + SH - 1) / SH * SH;
  static constexpr int OFF = SH - 1;
  static constexpr unsigned BYTES = (unsigned)(BW * BOX_Y * (int)sizeof(E));
  __device__ __forceinline__ static int at(int hy, int hx) { return hy * BW + hx + OFF; }
};

// z-slab neighbour: the pitched PCG vectors of the slab below or above, and
// the element offset of the plane of theirs that mirrors our boundary plane
// (their halo plane).  Null pointers: no neighbour on that side.
template <typename T>
struct PcgPeer {
  double* r0; double* r1;
  T* p0; T* p1; T* z; T* Ap;
  long long plane_off;
};

template <typename T>
struct PcgArgs {
  CUtensorMap tm_z, tm_p0, tm_p1, tm_x, tm_ap, tm_r0, tm_r1, tm_code, tm_code_own;
  Dims d;
  int nxp;                   // row pitch of the PCG vectors
  const uint8_t* code;       // pitched
  T* state_p;                // state pressure (unpitched): warm start in, solution out
  const T* u; const T* v; const T* w;
  double* r0; double* r1;    // pitched, float64
  T* p0; T* p1; T* z; T* Ap; T* x;   // pitched
  double* part;              // [2][3][PS] per-unit partials (two alternating sets)
  unsigned* tags;            // [2][PS] phase number of each unit's published partials (flag in data)
  int tiles, nchunk;         // (x, y) tiles per plane; z-chunks of this launch (U = tiles * nchunk)
  int chunk0, nchunk_g;      // global index of this slab's first chunk; chunks of the whole grid
  unsigned int* bar;         // [0] arrival count, [32] generation
  int* gate;
  DevReport* rep;
  const T* lut;              // [64][4] = d, 1/d, s, 0
  T wx, wy, wz, om;
  double dt, tol, res_factor;
  int max_iter;
  int precond;               // 0 identity, 1 jacobi (diag(1/d)), 2 AI1 (K^T K)
  int ntx, nty, zc, U;
  int PS;                    // partial-slot stride, >= max(U, blocks serving the slab)
  int o0, o1;                // owned planes [o0, o1) of the local grid (a z-slab window)
  // z-slab decomposition (nslab > 1): boundary planes are pushed into the
  // neighbours' halo planes as they are written; the slabs meet at the root
  // slab's barrier, where each slab's folded partials are published
  int nslab, slab;
  PcgPeer<T> lo, hi;
  unsigned int* xbar;        // root slab: [0] arrivals, [32] generation (system scope)
  double* xval;              // root slab: [2 sets][3 values][nchunk_g * groups] item sums
  long long timeout_ns;
  int probe_mode, probe_iters;   // developer timing probe (CW_PCG_PROBE), 0 = off
};

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "CW_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra CW_WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* b, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
      : "memory");
}
// L2 residency: the vectors re-read in the very next phase (z: B -> A, Ap:
// A -> B), x (own tile only, read and written once per iteration) and the
// operator codes are stored / loaded evict_last so they stay in the 126 MB L2
// (55 MB at C3); p and r (re-read an iteration later, r in fp64) are
// evict_first.  Measured at C3 (5 steady steps, k_pcg per step): this 3836 us,
// x evict_first 3868, everything evict_last 3869, r also kept 3846, p also
// kept 3895, no hints 3913.  CW_L2HINT=0 drops the hints (developer comparison).
#ifndef CW_L2HINT
#define CW_L2HINT 1
#endif
// which streams are evict_last (bits: 1 z, 2 p, 4 x, 8 codes, 16 r, 32 Ap);
// the rest evict_first (developer comparisons: CW_L2KEEP=63 keeps all)
#ifndef CW_L2KEEP
#define CW_L2KEEP 45
#endif
template <int BIT>
__device__ __forceinline__ uint64_t l2_pol(uint64_t keep, uint64_t drop) {
  return (CW_L2KEEP & BIT) ? keep : drop;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* b, int x, int y, int z,
                                                 uint64_t pol) {
#if CW_L2HINT
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b)), "l"(pol)
      : "memory");
#else
  tma_load_3d(dst, map, b, x, y, z);
#endif
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef CW_BAR_NS
#define CW_BAR_NS 32   // back-off between polls of the arrival counter (ns)
#endif
// Grid barrier for a cooperative launch (all blocks co-resident).  The
// arrival counter only grows during a launch (zeroed before it): barrier e
// (0-based, counted per block in `epoch`) completes when it reaches
// (e+1)*nblocks.  Arrival is one release reduction, waiting is acquire loads:
// no counter reset and no generation word on the critical path.  Times out
// (status 3) instead of hanging if the co-residency assumption is ever broken.
__device__ __forceinline__ void grid_barrier(unsigned* bar, int* gate, DevReport* rep, long long timeout_ns,
                                             unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    unsigned* count = bar;
    const unsigned target = epoch * nblocks;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    if (ld_acquire(count) < target) {
      const unsigned long long t0 = globaltimer();
      unsigned spins = 0;
      while (ld_acquire(count) < target) {
        if (CW_BAR_NS > 0) __nanosleep(CW_BAR_NS);
        if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > timeout_ns) {
          rep->status = 3;
          *gate = 3;
          break;
        }
      }
    }
    fence_proxy_async();   // the next phase's TMA (async proxy) reads see this phase's writes
  }
  __syncthreads();
}

// Fold n partials in a fixed order; every block computes the same bits.
// mode 0: sum, 1: max.  Result broadcast to all threads.
__device__ __forceinline__ double fold_partials(const double* part, int n, int mode, double* sh) {
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int q = threadIdx.x; q < n; q += 32) {
      const double v = __ldcg(part + q);
      if (mode == 0) a += v;
      else a = (v > a || v != v) ? v : a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b = __shfl_down_sync(0xffffffffu, a, o);
      if (mode == 0) a += b;
      else a = (b > a || b != b) ? b : a;
    }
    if (threadIdx.x == 0) sh[0] = a;
  }
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Fold up to three partial arrays part[q*stride + 0..n) at once with the
// whole block (one L2 round trip): per-thread strided sums, warp trees, then
// the warp results in warp order.  A fixed order: every block gets the same
// bits.  Bit q of maxmask: max (non-negative values, NaN wins) instead of sum.
__device__ __forceinline__ void fold_multi(const double* part, int n, int stride, int nval, unsigned maxmask,
                                           double* out, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (q < nval) {
      const bool mx = (maxmask >> q) & 1u;
      double a = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = __ldcg(part + (size_t)q * stride + i);
        a = mx ? ((v > a || v != v) ? v : a) : a + v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double b = __shfl_down_sync(0xffffffffu, a, o);
        a = mx ? ((b > a || b != b) ? b : a) : a + b;
      }
      if (lane == 0) sh[q * 32 + wid] = a;
    }
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (q < nval) {
      const bool mx = (maxmask >> q) & 1u;
      double a = sh[q * 32];
      for (int w = 1; w < nw; ++w) {
        const double b = sh[q * 32 + w];
        a = mx ? ((b > a || b != b) ? b : a) : a + b;
      }
      out[q] = a;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Per-unit reductions.  Each unit (tile x z-chunk) publishes its partials and
// then, with release semantics, the phase number in its tag (fold_chunks can
// acquire the tags instead of a grid barrier; measured slower at C3: 65K
// acquiring polls per phase against one counter, so phase_end keeps the
// barrier).  The fold is the same fixed tree wherever a chunk is folded -- one warp per
// chunk, lane l summing tiles l, l+32, ... in order, a shuffle tree, lane 0's
// result -- and the chunk sums are added in global chunk order.  So a whole
// grid and any split into z-slabs whose boundaries fall on chunk boundaries
// produce the same bits (slab_reduce publishes chunk sums, not slab sums).
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef CW_PCG_TAGS
#define CW_PCG_TAGS 0   // 1: publish per-unit tags (for fold_chunks(wait=true)); a release store per unit and phase
#endif
template <typename T>
__device__ __forceinline__ void publish_unit(const PcgArgs<T>& A, double* part, int set, int unit, int nval,
                                             const double* v, unsigned seq) {
  for (int q = 0; q < nval; ++q) part[(size_t)q * A.PS + unit] = v[q];
  if (CW_PCG_TAGS) st_release_u32(A.tags + (size_t)set * A.PS + unit, seq);
}

template <typename T>
__device__ __forceinline__ bool wait_tag(const PcgArgs<T>& A, const unsigned* tag, unsigned seq) {
  if ((int)(ld_acquire(tag) - seq) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  while ((int)(ld_acquire(tag) - seq) < 0) {
    __nanosleep(32);
    if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > A.timeout_ns) {
      A.rep->status = 3;
      *A.gate = 3;
      return false;
    }
  }
  return true;
}

// Item sums of this launch's units into S.grp.  An item is (chunk c, group
// g): tiles 32g .. 32g+31 of chunk c, items numbered c * ng + g (ng groups
// per chunk).  One warp per item (lane l: tile 32g + l, a shuffle tree, lane
// 0's result); items spread over the block's warps.  Returns after a
// __syncthreads.  wait: acquire every unit's tag first.
template <typename T, typename Sh>
__device__ __forceinline__ void fold_chunks(const PcgArgs<T>& A, const double* part, int set, unsigned seq, int nval,
                                            unsigned maxmask, bool wait, Sh& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  const unsigned* tags = A.tags + (size_t)set * A.PS;
  const int ng = (A.tiles + 31) >> 5;
  const bool flat = (A.tiles & 31) == 0;   // items are runs of 32 consecutive units
  for (int it = wid; it < A.nchunk * ng; it += nw) {
    int u, i;
    if (flat) {
      u = it * 32 + lane;
      i = 0;
    } else {
      const int c = it / ng;
      i = (it - c * ng) * 32 + lane;
      u = c * A.tiles + i;
    }
    double a[3] = {0.0, 0.0, 0.0};
    if (i < A.tiles) {
      if (wait) wait_tag<T>(A, tags + u, seq);
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < nval) a[q] = __ldcg(part + (size_t)q * A.PS + u);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q < nval) {
        const bool mx = (maxmask >> q) & 1u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double b = __shfl_xor_sync(0xffffffffu, a[q], o);
          a[q] = mx ? ((b > a[q] || b != b) ? b : a[q]) : a[q] + b;
        }
        if (lane == 0) S.grp[q][it] = a[q];
      }
    }
  }
  __syncthreads();
}

// the totals: all items in item order (one thread per value), broadcast
// through shared memory -- the same sequence the z-slab root table sums
template <typename T, typename Sh>
__device__ __forceinline__ void sum_items(const PcgArgs<T>& A, Sh& S, int nval, unsigned maxmask, double* out) {
  if (threadIdx.x < (unsigned)nval) {
    const int q = threadIdx.x, n = A.nchunk * ((A.tiles + 31) >> 5);
    const bool mx = (maxmask >> q) & 1u;
    double a = S.grp[q][0];
    for (int it = 1; it < n; ++it) {
      const double b = S.grp[q][it];
      a = mx ? ((b > a || b != b) ? b : a) : a + b;
    }
    S.vals[q] = a;
  }
  __syncthreads();
  for (int q = 0; q < nval; ++q) out[q] = S.vals[q];
}

// ---------------------------------------------------------------------------
// shared memory layout

__host__ __device__ constexpr int align128(int b) { return (b + 127) & ~127; }

template <typename T>
struct StageLayout {
  // phase A: z, p (halo boxes), x and code (own boxes)
  static constexpr int A_Z = 0;
  static constexpr int A_P = align128((int)Halo<T>::BYTES);
  static constexpr int A_X = A_P + align128((int)Halo<T>::BYTES);
  static constexpr int A_C = A_X + align128(PCG_TX * PCG_TY * (int)sizeof(T));
  static constexpr int A_END = A_C + align128(PCG_TX * PCG_TY);
  // phase B: r (float64), Ap, code (halo boxes)
  static constexpr int B_R = 0;
  static constexpr int B_AP = align128((int)Halo<double>::BYTES);
  static constexpr int B_C = B_AP + align128((int)Halo<T>::BYTES);
  static constexpr int B_END = B_C + align128((int)Halo<uint8_t>::BYTES);
  static constexpr int STAGE = A_END > B_END ? A_END : B_END;
#ifndef CW_PCG_DEPTH
#define CW_PCG_DEPTH 4
#endif
  static constexpr int DEPTH = sizeof(T) == 4 ? CW_PCG_DEPTH : 3;
  static constexpr unsigned BYTES_A_HALO = 2u * Halo<T>::BYTES;
  static constexpr unsigned BYTES_A_X = PCG_TX * PCG_TY * (sizeof(T) + 1);   // x + code, own box
  static constexpr unsigned BYTES_B = Halo<double>::BYTES + Halo<T>::BYTES + Halo<uint8_t>::BYTES;
};

// phase-B work planes.  q tile: halo column hx at PCG_QOFF + hx, so the own
// quads (hx = 1 + 4 tx) start on 16-byte boundaries; y tile: column x at x.
constexpr int PCG_QOFF = 3, PCG_QW = 40, PCG_YP = 36;
template <typename T>
struct PcgWork {
  alignas(16) T qb[4][HH][PCG_QW];   // q = r'/d on the halo tile, planes kk, kk-1 (+2 hazard-free)
  alignas(16) T yb[2][YH][PCG_YP];   // y on the y tile, planes kk and kk-1
};

#ifndef CW_PCG_MAXG
#define CW_PCG_MAXG 128  // (z-chunk, 32-tile group) items per launch (the context picks zc to fit)
#endif
template <typename T>
struct PcgShared {
  T lut[64 * 4];
  union {
    T pa[2][HH][HW];      // phase 0 planes
    PcgWork<T> wk;        // phase B
  };
  double red[32];
  double bc[4];
  double vals[4];           // slab_reduce results
  double fold[3 * 32];      // fold_multi warp results
  double grp[3][CW_PCG_MAXG];     // fold_chunks: (chunk, 32-tile group) sums, combined in order
  unsigned last, gen0;      // slab_reduce: this block arrived last; generation seen
  unsigned long long pt[3]; // timing probe (modes 13-16): phase start, first stage landed, jobs done
  alignas(8) uint64_t full[8];
};

template <typename T>
__host__ __device__ constexpr size_t pcg_smem_bytes() {
  return 128 + (size_t)StageLayout<T>::STAGE * StageLayout<T>::DEPTH + sizeof(PcgShared<T>);
}

struct Unit {
  int i0, j0, k0, k1;
};

// This block's place among the blocks serving its slab (the whole grid when
// there is one slab per launch).
struct Blk {
  int id, n;
};

template <typename T>
__device__ __forceinline__ Unit unit_of(const PcgArgs<T>& A, int u) {
  const int per = A.ntx * A.nty;
  const int tz = u / per, rem = u - tz * per;
  Unit t;
  t.i0 = (rem % A.ntx) * PCG_TX;
  t.j0 = (rem / A.ntx) * PCG_TY;
  t.k0 = A.o0 + tz * A.zc;
  t.k1 = min(t.k0 + A.zc, A.o1);
  return t;
}

// Jobs of one ring phase for this block: its units in order (unit
// blk.id + m*blk.n), each contributing planes k0-1 .. k1.
struct JobCursor {
  int unit, nb;
  Unit t;
  int kk;
};

template <typename T>
__device__ __forceinline__ bool cursor_begin(const PcgArgs<T>& A, const Blk& blk, JobCursor& c) {
  c.unit = blk.id;
  c.nb = blk.n;
  if (c.unit >= A.U) return false;
  c.t = unit_of<T>(A, c.unit);
  c.kk = c.t.k0 - 1;
  return true;
}
template <typename T>
__device__ __forceinline__ bool cursor_next(const PcgArgs<T>& A, JobCursor& c) {
  if (c.kk < c.t.k1) { ++c.kk; return true; }
  c.unit += c.nb;
  if (c.unit >= A.U) return false;
  c.t = unit_of<T>(A, c.unit);
  c.kk = c.t.k0 - 1;
  return true;
}

// Producer: thread 0 issues job `ticket` (numbered across the whole kernel,
// which fixes every stage's mbarrier parity).
template <typename T>
__device__ __forceinline__ void issue_A(const PcgArgs<T>& A, uint8_t* ring, uint64_t* full, unsigned ticket,
                                        const JobCursor& c, const CUtensorMap* tp) {
  using L = StageLayout<T>;
  const int s = ticket % L::DEPTH;
  uint8_t* st = ring + (size_t)s * L::STAGE;
  const bool own = c.kk >= c.t.k0 && c.kk < c.t.k1;
  mbar_expect_tx(&full[s], L::BYTES_A_HALO + (own ? L::BYTES_A_X : 0u));
  const uint64_t keep = l2_evict_last(), drop = l2_evict_first();
  tma_load_3d_hint(st + L::A_Z, &A.tm_z, &full[s], c.t.i0 - Halo<T>::SH, c.t.j0 - 1, c.kk, l2_pol<1>(keep, drop));
  tma_load_3d_hint(st + L::A_P, tp, &full[s], c.t.i0 - Halo<T>::SH, c.t.j0 - 1, c.kk, l2_pol<2>(keep, drop));
  if (own) {
    tma_load_3d_hint(st + L::A_X, &A.tm_x, &full[s], c.t.i0, c.t.j0, c.kk, l2_pol<4>(keep, drop));
    tma_load_3d_hint(st + L::A_C, &A.tm_code_own, &full[s], c.t.i0, c.t.j0, c.kk, l2_pol<8>(keep, drop));
  }
}

template <typename T>
__device__ __forceinline__ void issue_B(const PcgArgs<T>& A, uint8_t* ring, uint64_t* full, unsigned ticket,
                                        const JobCursor& c, const CUtensorMap* tr) {
  using L = StageLayout<T>;
  const int s = ticket % L::DEPTH;
  uint8_t* st = ring + (size_t)s * L::STAGE;
  mbar_expect_tx(&full[s], L::BYTES_B);
  const uint64_t keep = l2_evict_last(), drop = l2_evict_first();
  tma_load_3d_hint(st + L::B_R, tr, &full[s], c.t.i0 - Halo<double>::SH, c.t.j0 - 1, c.kk, l2_pol<16>(keep, drop));
  tma_load_3d_hint(st + L::B_AP, &A.tm_ap, &full[s], c.t.i0 - Halo<T>::SH, c.t.j0 - 1, c.kk, l2_pol<32>(keep, drop));
  tma_load_3d_hint(st + L::B_C, &A.tm_code, &full[s], c.t.i0 - Halo<uint8_t>::SH, c.t.j0 - 1, c.kk,
                   l2_pol<8>(keep, drop));
}

// A p' per cell.  float32 state: the difference form sum_a w_a (p_i - p_a)
// over the neighbours a that are unknowns or outlets (p_a = 0 at an outlet).
// The 7-point combination of a smooth p cancels d*p almost entirely, so the
// direct form d*p - sum w p_a needs float64; in the difference form the
// cancellation happens inside the differences, which are exact in float32
// when neighbours are within a factor of two (Sterbenz) and otherwise carry
// no cancellation, so float32 arithmetic keeps ~eps*|A p| accuracy.  float64
// state: the direct form in float64.  The +z term is added once the next
// plane lands (ap_finish).
template <typename T> struct ApAccT { typedef double type; };
template <> struct ApAccT<float> { typedef float type; };
template <typename T> using ApAcc = typename ApAccT<T>::type;

template <typename T>
__device__ __forceinline__ ApAcc<T> ap_partial(uint8_t cd, T d, T pc, T pxp, T pxm, T pyp, T pym, T pzm, T wx, T wy,
                                               T wz) {
  if constexpr (sizeof(T) == 4) {
    float a = 0.f;
    if (cd & 1) a += wx * (pc - pxp);
    if (cd & 2) a += wx * (pc - pxm);
    if (cd & 4) a += wy * (pc - pyp);
    if (cd & 8) a += wy * (pc - pym);
    if (cd & 32) a += wz * (pc - pzm);
    return a;
  } else {   // 0 off the unknowns (code 0), like the difference form
    if (!(cd & 64)) return 0.0;
    return (double)d * (double)pc - ((double)wx * ((double)pxm + (double)pxp) +
                                     (double)wy * ((double)pym + (double)pyp) + (double)wz * (double)pzm);
  }
}

template <typename T>
__device__ __forceinline__ double ap_finish(ApAcc<T> part, T wz, T pc, T pzp, bool zp) {
  if constexpr (sizeof(T) == 4) {
    return (double)(zp ? part + wz * (pc - pzp) : part);
  } else {
    return zp ? part - (double)wz * (double)pzp : part;   // p = 0 on a +z neighbour that is not an unknown
  }
}

// ---------------------------------------------------------------------------
// Ring phases.  Thread layout: QX = 8 threads across x, each owning an x quad
// (4 consecutive cells of one row), times 32 rows: one 32 x 32 plane per
// block sweep.  Own quads move as 128-bit shared and global accesses; the x
// neighbours come from the adjacent lanes of the row (shuffles), the tile
// edges from the halo columns (every lane loads its edge cell, no divergent
// path), the y neighbours from the rows above and below (128-bit loads), the
// z neighbours from registers carried through the z march.  The march is
// unrolled by two so the carried planes alternate between two register sets.
// Shared offsets are fixed per thread; global offsets are 32-bit (pitched
// fields hold < 2^31 elements, cw_capi.cu).
constexpr int QX = PCG_TX / 4;
#ifndef CW_ABL
#define CW_ABL 0   // developer ablations (timing only; results are wrong when set): B ring 1, B y edge 2, B stores 4, B pass 2 8, A stores 16
#endif
static_assert(PCG_THREADS == QX * PCG_TY, "one thread per x quad of a 32 x 32 plane");
static_assert(PCG_THREADS - (2 * (PCG_TX + 2) + 2 * PCG_TY) >= (PCG_TX + 1) + PCG_TY,
              "the q ring and the y-tile edge run on disjoint warps");

__device__ __forceinline__ float fmat(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename E>
__device__ __forceinline__ void ld4(const E* p, E (&v)[4]) {   // p: 16-byte aligned
  if constexpr (sizeof(E) == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}
template <typename E>
__device__ __forceinline__ void st4(E* p, const E (&v)[4]) {
  if constexpr (sizeof(E) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
  }
}
// global quad store: float64 quads go out as one 256-bit store (STG.E.ENL2.256),
// so a warp instruction covers whole 32-byte sectors (two 128-bit halves would
// each write half of every sector); p: 32-byte aligned for float64
template <typename E>
__device__ __forceinline__ void stg4(E* p, const E (&v)[4]) {
  if constexpr (sizeof(E) == 8) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
  } else {
    st4<E>(p, v);
  }
}
// the same with an L2 eviction policy (l2_evict_first / l2_evict_last)
template <typename E>
__device__ __forceinline__ void stg4h(E* p, const E (&v)[4], uint64_t pol) {
#if CW_L2HINT
  if constexpr (sizeof(E) == 8) {
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(v[0]), "d"(v[1]),
                 "d"(v[2]), "d"(v[3]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "l"(pol)
                 : "memory");
  }
#else
  stg4<E>(p, v);
#endif
}
// the neighbouring lane of the same 8-lane row (a lane at the row's end gets its own value)
template <typename E>
__device__ __forceinline__ E from_left(E v) { return __shfl_up_sync(0xffffffffu, v, 1, QX); }
template <typename E>
__device__ __forceinline__ E from_right(E v) { return __shfl_down_sync(0xffffffffu, v, 1, QX); }

// operator table row of a code byte: d, 1/d, s*w, w/d (cw_set_operator)
template <typename T>
__device__ __forceinline__ T lut_at(const T* lut, unsigned cd, int which) { return lut[(cd & 63u) * 4 + which]; }

// y = s (r' + w sum_a w_a q_{i-e_a}) with s r' = (2-w) w q:  c0 q + (s w) (sum_a w_a q_{i-e_a})
template <typename T>
__device__ __forceinline__ T y_of(T c0, T q, T sw, T wx, T qxm, T wy, T qym, T wz, T qzm) {
  return fmat(c0, q, sw * fmat(wx, qxm, fmat(wy, qym, wz * qzm)));
}
// z = y + (w/d) sum_a w_a y_{i+e_a}
template <typename T>
__device__ __forceinline__ T z_of(T y, T wd, T wx, T yxp, T wy, T yyp, T wz, T yzp) {
  return fmat(wd, fmat(wx, yxp, fmat(wy, yyp, wz * yzp)), y);
}

// Producer side of a ring phase: thread 0 keeps DEPTH stages in flight.
template <typename T, typename Issue>
__device__ __forceinline__ void ring_fill(const PcgArgs<T>& A, JobCursor& prod, bool& more, unsigned& issued,
                                          unsigned upto, Issue issue) {
  while (more && issued < upto) {
    issue(issued, prod);
    ++issued;
    more = cursor_next<T>(A, prod);
  }
}

// ---- phase 0: b = -div/dt, r0 = b - A x0 with x0 = p on the unknowns ------
// (once per projection; plain loads).  x quads like the ring phases: plane k's
// halo tile of x0 goes to a shared double buffer (own quads plus the 132-cell
// ring), the z neighbours are the own quads of planes k-1, k+1 in registers.
template <typename T, bool SLABS>
__device__ void phase0(const PcgArgs<T>& A, double* part, int set, unsigned seq, int unit, PcgShared<T>& S) {
  const Dims& d = A.d;
  const Unit t = unit_of<T>(A, unit);
  const int tx = threadIdx.x % QX, ty = threadIdx.x / QX;
  const bool lft = tx == 0, rgt = tx == QX - 1;
  const int hy = ty + 1, hx0 = 1 + 4 * tx;
  const int i = t.i0 + 4 * tx, jj = t.j0 + ty;
  const int plane = d.nx * d.ny, pplane = A.nxp * d.ny;
  // x0 = state p on the unknowns, 0 elsewhere and outside the grid: the code
  // byte and p are loaded independently (clamped address), then selected
  auto x0_at = [&](int kk, int gi, int gj) -> T {
    const bool in = kk >= 0 && kk < d.nz && gi >= 0 && gi < d.nx && gj >= 0 && gj < d.ny;
    const int ck = in ? kk : 0, ci = in ? gi : 0, cj = in ? gj : 0;
    const uint8_t cd = __ldg(A.code + (ck * pplane + cj * A.nxp + ci));
    const T pv = __ldg(A.state_p + (ck * plane + cj * d.nx + ci));
    return (in && (cd & 64)) ? pv : (T)0;
  };
  auto x0_quad = [&](int kk, T (&q)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) q[c] = x0_at(kk, i + c, jj);
  };
  // the tile's ring cell of this thread (the last 132 threads, as in phase B)
  const int rt = (int)threadIdx.x - (PCG_THREADS - (2 * HW + 2 * PCG_TY));
  const bool ring_t = rt >= 0;
  const int ry = rt < HW ? 0 : (rt < 2 * HW ? HH - 1 : (rt < 2 * HW + PCG_TY ? rt - 2 * HW + 1 : rt - 2 * HW - PCG_TY + 1));
  const int rx = rt < HW ? rt : (rt < 2 * HW ? rt - HW : (rt < 2 * HW + PCG_TY ? 0 : HW - 1));
  constexpr int QPL = HH * PCG_QW;
  T* tile = &S.wk.qb[0][0][0];                  // two planes of the phase-B q ring (free here)
  const int q_own = hy * PCG_QW + hx0 + PCG_QOFF;
  const int q_e = hy * PCG_QW + PCG_QOFF + (lft ? 0 : (rgt ? PCG_TX + 1 : hx0));
  const int ro_q = ry * PCG_QW + rx + PCG_QOFF;
  const bool rows = jj < d.ny && i < A.nxp;
  const double rdt = 1.0 / A.dt;
  const double wx = (double)A.wx, wy = (double)A.wy, wz = (double)A.wz;
  double b2 = 0.0, bmax = 0.0, dmax = 0.0;
  T xm[4], xc[4], xn[4];
  x0_quad(t.k0 - 1, xm);
  x0_quad(t.k0, xc);
  for (int k = t.k0; k < t.k1; ++k) {
    T* tl = tile + (k & 1) * QPL;
    st4<T>(tl + q_own, xc);
    if (ring_t) tl[ro_q] = x0_at(k, t.i0 + rx - 1, t.j0 + ry - 1);
    x0_quad(k + 1, xn);                         // the next plane's own quad, in flight over the barrier
    __syncthreads();
    T ym[4], yp[4];
    ld4<T>(tl + q_own - PCG_QW, ym);
    ld4<T>(tl + q_own + PCG_QW, yp);
    const T xe = tl[q_e];
    T left = from_left(xc[3]), right = from_right(xc[0]);
    left = lft ? xe : left;
    right = rgt ? xe : right;
    if (rows) {
      const int g = k * pplane + jj * A.nxp + i;   // pitched, quad-aligned
      const uint32_t cw4 = *reinterpret_cast<const uint32_t*>(A.code + g);
      const int ui = (k * d.ny + jj) * (d.nx + 1) + i;
      const int vi = (k * (d.ny + 1) + jj) * d.nx + i;
      const int c0 = k * plane + jj * d.nx + i;
      double rv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        rv[c] = 0.0;
        const unsigned cd = (cw4 >> (8 * c)) & 0xffu;   // 0 beyond the grid's x extent (pitched padding)
        if (cd & 64u) {
          // divergence and A x0 in float64 from the stored fields
          double div = ((double)A.u[ui + c + 1] - (double)A.u[ui + c]) * d.drh[0] +
                       ((double)A.v[vi + c + d.nx] - (double)A.v[vi + c]) * d.drh[1];
          if (!d.is2d) div = div + ((double)A.w[c0 + c + plane] - (double)A.w[c0 + c]) * d.drh[2];
          const double b = -div * rdt;
          const double ax = (double)lut_at(S.lut, cd, 0) * (double)xc[c] -
                            (wx * ((double)(c == 0 ? left : xc[c - 1]) + (double)(c == 3 ? right : xc[c + 1])) +
                             wy * ((double)ym[c] + (double)yp[c]) + wz * ((double)xm[c] + (double)xn[c]));
          rv[c] = b - ax;
          b2 += b * b;
          const double ab = fabs(b), ad = fabs(div);
          bmax = (ab > bmax || ab != ab) ? ab : bmax;
          dmax = (ad > dmax || ad != ad) ? ad : dmax;
        }
      }
      stg4<double>(A.r0 + g, rv);
      stg4<T>(A.x + g, xc);
      if (SLABS && k == A.o0 && A.lo.r0) stg4<double>(A.lo.r0 + A.lo.plane_off + (g - k * pplane), rv);   // z-slab halo push
      if (SLABS && k == A.o1 - 1 && A.hi.r0) stg4<double>(A.hi.r0 + A.hi.plane_off + (g - k * pplane), rv);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) { xm[c] = xc[c]; xc[c] = xn[c]; }
  }
  const double s0 = block_sum(b2, S.red);
  __syncthreads();
  const double m1 = block_max(bmax, S.red);
  __syncthreads();
  const double m2 = block_max(dmax, S.red);
  if (threadIdx.x == 0) {
    const double v[3] = {s0, m1, m2};
    publish_unit<T>(A, part, set, unit, 3, v, seq);
  }
  __syncthreads();
}

// ---- phase A: p' = z + beta p, x += alpha_prev p, Ap = A p' ---------------
// (first iteration: the p box is read from z and beta = 0, so p' = z)
// UPDX: x += alpha_prev p (every iteration but the first); STREAM: timing
// probe that only streams the stages (CW_PCG_PROBE modes 4, 7)
template <typename T, bool SLABS, bool UPDX, bool STREAM>
__device__ void phaseA(const PcgArgs<T>& A, const Blk& blk, double* part, int set, unsigned seq, PcgShared<T>& S,
                       uint8_t* ring, unsigned& ticket, bool first, T beta, T alpha_prev, int pin_sel) {
  constexpr bool upd_x = UPDX;
  using L = StageLayout<T>;
  using H = Halo<T>;
  const Dims& d = A.d;
  const CUtensorMap* tp = first ? &A.tm_z : (pin_sel == 0 ? &A.tm_p0 : &A.tm_p1);
  const T b = first ? (T)0 : beta;
  T* __restrict__ pout = pin_sel == 0 ? A.p1 : A.p0;
  T* __restrict__ apout = A.Ap;
  T* __restrict__ xout = A.x;
  const T wx = A.wx, wy = A.wy, wz = A.wz;
  const uint64_t keep = l2_evict_last(), drop = l2_evict_first();
  const int tx = threadIdx.x % QX, ty = threadIdx.x / QX;
  const bool lft = tx == 0, rgt = tx == QX - 1;
  const int o_c = H::at(ty + 1, 1 + 4 * tx), o_dn = o_c - H::BW, o_up = o_c + H::BW;
  const int o_e = H::at(ty + 1, lft ? 0 : (rgt ? PCG_TX + 1 : 1 + 4 * tx));
  const int o_own = ty * PCG_TX + 4 * tx;      // own boxes: x (elements), code (bytes)
  const int nxp = A.nxp, ny = d.ny, pplane = nxp * ny;
  const bool timing = A.probe_mode >= 13;
  if (timing && threadIdx.x == 0) S.pt[0] = S.pt[1] = S.pt[2] = globaltimer();
  JobCursor prod, cons;
  double acc = 0.0;
  if (cursor_begin<T>(A, blk, cons)) {
    const int last_unit = blk.id + (A.U - 1 - blk.id) / blk.n * blk.n;
    prod = cons;
    const unsigned t0 = ticket;
    unsigned issued = 0;
    bool more = true;   // producer state, meaningful in thread 0 only
    auto issue = [&](unsigned n, const JobCursor& c) { issue_A<T>(A, ring, S.full, t0 + n, c, tp); };
    if (threadIdx.x == 0) ring_fill<T>(A, prod, more, issued, (unsigned)L::DEPTH, issue);
    unsigned j = 0;     // consumer job number in this phase
    // plane kk-1's pending result (A p' without its +z term, p', new x),
    // finished once plane kk lands
    T pcur[4], xn[4];
    ApAcc<T> pap[4];
    unsigned pzb = 0;   // bit c: cell c's +z neighbour is an unknown or an outlet
    bool pend = false;
    T pa[4] = {(T)0, (T)0, (T)0, (T)0}, pb[4];   // p' of the previous / this plane (alternating)
    auto plane = [&](const T (&pm)[4], T (&pn)[4]) -> bool {
      const unsigned tk = t0 + j;
      const int s = tk % L::DEPTH;
      const uint8_t* st = ring + s * L::STAGE;
      mbar_wait(&S.full[s], (tk / L::DEPTH) & 1u);
      if (timing && j == 0 && threadIdx.x == 0) S.pt[1] = globaltimer();
      const int kk = cons.kk;
      const Unit u = cons.t;
      if (!STREAM) {
        const T* zz = reinterpret_cast<const T*>(st + L::A_Z);
        const T* pp = reinterpret_cast<const T*>(st + L::A_P);
        const int jj = u.j0 + ty, i = u.i0 + 4 * tx;
        const bool rows = jj < ny && i < nxp;
        const int e = jj * nxp + i;
        T zc[4], pc[4];
        ld4<T>(zz + o_c, zc);
        ld4<T>(pp + o_c, pc);
#pragma unroll
        for (int c = 0; c < 4; ++c) pn[c] = fmat(b, pc[c], zc[c]);
        if (pend) {   // finish plane kk-1: add the +z neighbour (this plane) and store
          T apv[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double ap = ap_finish<T>(pap[c], wz, pcur[c], pn[c], (pzb >> c) & 1u);
            apv[c] = (T)ap;
            acc += (double)pcur[c] * ap;
          }
          if (rows && !(CW_ABL & 16)) {
            const int g = (kk - 1) * pplane + e;
            stg4h<T>(pout + g, pcur, l2_pol<2>(keep, drop));
            stg4h<T>(apout + g, apv, l2_pol<32>(keep, drop));
            if (upd_x) stg4h<T>(xout + g, xn, l2_pol<4>(keep, drop));
            if (SLABS && A.nslab > 1) {   // boundary planes go to the neighbours' halo planes
              if (kk - 1 == A.o0 && A.lo.Ap) {
                stg4<T>((pin_sel == 0 ? A.lo.p1 : A.lo.p0) + A.lo.plane_off + e, pcur);
                stg4<T>(A.lo.Ap + A.lo.plane_off + e, apv);
              }
              if (kk - 1 == A.o1 - 1 && A.hi.Ap) {
                stg4<T>((pin_sel == 0 ? A.hi.p1 : A.hi.p0) + A.hi.plane_off + e, pcur);
                stg4<T>(A.hi.Ap + A.hi.plane_off + e, apv);
              }
            }
          }
          pend = false;
        }
        if (kk >= u.k0 && kk < u.k1) {
          T zd[4], pd[4], zu[4], pu[4], pym[4], pyp[4];
          ld4<T>(zz + o_dn, zd);
          ld4<T>(pp + o_dn, pd);
          ld4<T>(zz + o_up, zu);
          ld4<T>(pp + o_up, pu);
          const T pe = fmat(b, pp[o_e], zz[o_e]);
          const uint32_t cw4 = *reinterpret_cast<const uint32_t*>(st + L::A_C + o_own);
          T xv[4];
          if (upd_x) ld4<T>(reinterpret_cast<const T*>(st + L::A_X) + o_own, xv);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            pym[c] = fmat(b, pd[c], zd[c]);
            pyp[c] = fmat(b, pu[c], zu[c]);
          }
          T left = from_left(pn[3]), right = from_right(pn[0]);
          left = lft ? pe : left;
          right = rgt ? pe : right;
          pzb = 0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const unsigned cd = (cw4 >> (8 * c)) & 0xffu;   // 0 off the unknowns: A p' = 0 there
            pap[c] = ap_partial<T>((uint8_t)cd, lut_at(S.lut, cd, 0), pn[c], c == 3 ? right : pn[c + 1],
                                   c == 0 ? left : pn[c - 1], pyp[c], pym[c], pm[c], wx, wy, wz);
            pzb |= ((cd >> 4) & 1u) << c;
            pcur[c] = pn[c];
            if (upd_x) xn[c] = fmat(alpha_prev, pc[c], xv[c]);
          }
          pend = true;
        }
      }
      if (kk == u.k1 && cons.unit + cons.nb < A.U) {   // a unit done and another follows: publish it now
        const double sum = block_sum(acc, S.red);
        if (threadIdx.x == 0) publish_unit<T>(A, part, set, cons.unit, 1, &sum, seq);
        acc = 0.0;
      }
      const bool live = cursor_next<T>(A, cons);
      ++j;
      return live;
    };
    // two planes per block barrier: their dependent chains interleave (the
    // second plane's stage is waited for before the first one is computed)
    for (;;) {
      const bool live = plane(pa, pb);
      const bool live2 = live && plane(pb, pa);
      __syncthreads();   // every thread is done with these jobs' stages: refill them
      if (threadIdx.x == 0) ring_fill<T>(A, prod, more, issued, j + L::DEPTH, issue);
      if (!live2) break;
    }
    if (timing && threadIdx.x == 0) S.pt[2] = globaltimer();
    ticket = t0 + j;
    const double sum = block_sum(acc, S.red);   // the block's last unit
    if (threadIdx.x == 0) publish_unit<T>(A, part, set, last_unit, 1, &sum, seq);
  }
}

// ---- phase B: r' = r - alpha Ap, z = W r' ----------------------------------
// Per landed plane kk: pass 1 computes q = r'/d on the 34 x 34 halo tile
// (own quads plus the 132-cell ring) into a 3-plane shared ring; after one
// barrier pass 2 computes y(kk) on the 33 x 33 y tile and the own cells
// finish z on plane kk-1 from y(kk-1) (shared) and y(kk) (registers).
template <typename T>
struct PlaneB {           // one plane's own-quad values carried to the next plane
  double r[4];            // r'
  T q[4], y[4], wd[4];    // q = r'/d, y, w/d
};

// USE_AP: r' = r - alpha Ap, written back (false: z0 = W r0 from phase 0's
// r0, nothing but z written); STREAM: timing probe, stages only (mode 7).
// Partials: r'.z and a flag for |r'| > res_target anywhere (NaN included),
// the max-norm half of pcg_solve's stopping rule (linalg.py:332-337).
template <typename T, bool SLABS, bool USE_AP, bool STREAM>
__device__ void phaseB(const PcgArgs<T>& A, const Blk& blk, double* part, int set, unsigned seq, PcgShared<T>& S,
                       uint8_t* ring, unsigned& ticket, double alpha, double res_target, int rin_sel) {
  constexpr bool use_ap = USE_AP, write_r = USE_AP;
  using L = StageLayout<T>;
  using H = Halo<T>;
  using HD = Halo<double>;
  using HC = Halo<uint8_t>;
  const Dims& d = A.d;
  const CUtensorMap* tr = rin_sel == 0 ? &A.tm_r0 : &A.tm_r1;
  double* __restrict__ rout = rin_sel == 0 ? A.r1 : A.r0;
  T* __restrict__ zout = A.z;
  const T om = A.om;
  const T c0 = ((T)2 - om) * om;          // s * d
  const T wx = A.wx, wy = A.wy, wz = A.wz;
  const int precond = A.precond;
  const double na = -alpha;
  const uint64_t keep = l2_evict_last(), drop = l2_evict_first();
  const int tx = threadIdx.x % QX, ty = threadIdx.x / QX;
  const bool lft = tx == 0, rgt = tx == QX - 1;
  const int hy = ty + 1, hx0 = 1 + 4 * tx;
  const int o_r = HD::at(hy, hx0), o_a = H::at(hy, hx0), o_c = HC::at(hy, hx0);
  const int q_own = hy * PCG_QW + hx0 + PCG_QOFF, q_dn = q_own - PCG_QW, q_e = hy * PCG_QW + PCG_QOFF;
  const int y_own = ty * PCG_YP + 4 * tx, y_up = y_own + PCG_YP, y_e = ty * PCG_YP + PCG_TX;
  // ring cell of q (pass 1): rows 0 and 33, columns 0 and 33, on the last 132
  // threads (warps 3-7); the y-tile edge of pass 2 runs on warps 0-2, so no
  // warp carries extra work in both passes
  const int t = threadIdx.x;
  const int rt = t - (PCG_THREADS - (2 * HW + 2 * PCG_TY));
  const bool ring_t = rt >= 0;
  const int ry = rt < HW ? 0 : (rt < 2 * HW ? HH - 1 : (rt < 2 * HW + PCG_TY ? rt - 2 * HW + 1 : rt - 2 * HW - PCG_TY + 1));
  const int rx = rt < HW ? rt : (rt < 2 * HW ? rt - HW : (rt < 2 * HW + PCG_TY ? 0 : HW - 1));
  const int ro_r = HD::at(ry, rx), ro_a = H::at(ry, rx), ro_c = HC::at(ry, rx), ro_q = ry * PCG_QW + rx + PCG_QOFF;
  // y-tile row 32 and column 32 (threads < 65)
  const bool yh_t = t < YW + PCG_TY;
  const int yy = t < YW ? PCG_TY : t - YW, yx = t < YW ? t : PCG_TX;
  const int yo = yy * PCG_YP + yx, yq = (yy + 1) * PCG_QW + yx + 1 + PCG_QOFF, yc = HC::at(yy + 1, yx + 1);
  const int nxp = A.nxp, ny = d.ny, pplane = nxp * ny;
  const bool timing = A.probe_mode >= 13;
  PcgWork<T>& W = S.wk;
  T* qb = &W.qb[0][0][0];
  T* yb = &W.yb[0][0][0];
  constexpr int QPL = HH * PCG_QW, YPL = YH * PCG_YP;   // plane strides of the q and y rings
  if (timing && threadIdx.x == 0) S.pt[0] = S.pt[1] = S.pt[2] = globaltimer();
  JobCursor prod, cons;
  double acc = 0.0;
  bool exceed = false;
  if (cursor_begin<T>(A, blk, cons)) {
    const int last_unit = blk.id + (A.U - 1 - blk.id) / blk.n * blk.n;
    prod = cons;
    const unsigned t0 = ticket;
    unsigned issued = 0;
    bool more = true;
    auto issue = [&](unsigned n, const JobCursor& c) { issue_B<T>(A, ring, S.full, t0 + n, c, tr); };
    if (threadIdx.x == 0) ring_fill<T>(A, prod, more, issued, (unsigned)L::DEPTH, issue);
    unsigned j = 0;
    PlaneB<T> pa, pb;
#pragma unroll
    for (int c = 0; c < 4; ++c) { pa.r[c] = 0.0; pa.q[c] = pa.y[c] = pa.wd[c] = (T)0; }
    auto plane = [&](const PlaneB<T>& pv, PlaneB<T>& cu) -> bool {
      const unsigned tk = t0 + j;
      const int s = tk % L::DEPTH;
      const uint8_t* st = ring + s * L::STAGE;
      mbar_wait(&S.full[s], (tk / L::DEPTH) & 1u);
      if (timing && j == 0 && threadIdx.x == 0) S.pt[1] = globaltimer();
      const int kk = cons.kk;
      const Unit u = cons.t;
      constexpr bool probe_stream = STREAM;
      T* qcur = qb + (j & 3) * QPL;               // q planes kk, kk-1 (ring of 4)
      const T* qprv = qb + ((j + 3) & 3) * QPL;
      T* ycur = yb + (j & 1) * YPL;               // y planes kk, kk-1 (ring of 2)
      const T* yprv = yb + ((j + 1) & 1) * YPL;
      const double* rr = reinterpret_cast<const double*>(st + L::B_R);
      const T* aa = reinterpret_cast<const T*>(st + L::B_AP);
      const uint8_t* cc = st + L::B_C;
      const int jj = u.j0 + ty, i = u.i0 + 4 * tx;
      const bool rows = jj < ny && i < nxp;
      const int e = jj * nxp + i;
      T sw[4], iv[4];
      if (!probe_stream) {
        // pass 1: own quad r', 1/d, s w, w/d, q; the halo ring of q
        const uint32_t cw4 = *reinterpret_cast<const uint32_t*>(cc + o_c);
        double r4[4];
        ld4<double>(rr + o_r, r4);
        T a4[4];
        if (use_ap) ld4<T>(aa + o_a, a4);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const unsigned cd = (cw4 >> (8 * c)) & 0xffu;   // 0 off the unknowns: q = y = z = 0 there
          cu.r[c] = use_ap ? fmat(na, (double)a4[c], r4[c]) : r4[c];
          iv[c] = lut_at(S.lut, cd, 1);
          sw[c] = lut_at(S.lut, cd, 2);
          cu.wd[c] = lut_at(S.lut, cd, 3);
          cu.q[c] = (T)cu.r[c] * iv[c];
        }
        if (precond == 2) {
          st4<T>(qcur + q_own, cu.q);
          if (ring_t && !(CW_ABL & 1)) {
            double r = rr[ro_r];
            if (use_ap) r = fmat(na, (double)aa[ro_a], r);
            qcur[ro_q] = (T)r * lut_at(S.lut, cc[ro_c], 1);
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && j > 0) ring_fill<T>(A, prod, more, issued, j + L::DEPTH, issue);   // stage j-1 is free
      if (!probe_stream) {
        if (precond == 2) {
          // pass 2: y(kk) on the y tile (own quads in registers and shared, plus row 32 and column 32)
          if (kk >= u.k0 && !(CW_ABL & 8)) {
            T qym[4];
            ld4<T>(qcur + q_dn, qym);
            const T qe = qcur[q_e];
            T left = from_left(cu.q[3]);
            left = lft ? qe : left;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              cu.y[c] = y_of<T>(c0, cu.q[c], sw[c], wx, c == 0 ? left : cu.q[c - 1], wy, qym[c], wz, pv.q[c]);
            st4<T>(ycur + y_own, cu.y);
            if (yh_t && !(CW_ABL & 2))
              ycur[yo] = y_of<T>(c0, qcur[yq], lut_at(S.lut, cc[yc], 2), wx, qcur[yq - 1], wy, qcur[yq - PCG_QW], wz,
                                 qprv[yq]);
          }
          // z on plane kk-1 (own cells): y(kk-1) from the previous plane, y(kk) own
          if (kk >= u.k0 + 1 && !(CW_ABL & 8)) {
            T yyp[4], zv[4];
            ld4<T>(yprv + y_up, yyp);
            const T ye = yprv[y_e];
            T right = from_right(pv.y[0]);
            right = rgt ? ye : right;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              zv[c] = z_of<T>(pv.y[c], pv.wd[c], wx, c == 3 ? right : pv.y[c + 1], wy, yyp[c], wz, cu.y[c]);
              acc = fmat(pv.r[c], (double)zv[c], acc);
              exceed |= !(fabs(pv.r[c]) <= res_target);
            }
            if (rows && !(CW_ABL & 4)) {
              const int g = (kk - 1) * pplane + e;
              stg4h<T>(zout + g, zv, l2_pol<1>(keep, drop));
              if (write_r) stg4h<double>(rout + g, pv.r, l2_pol<16>(keep, drop));
              if (SLABS && A.nslab > 1) {   // boundary planes go to the neighbours' halo planes
                if (kk - 1 == A.o0 && A.lo.z) {
                  stg4<T>(A.lo.z + A.lo.plane_off + e, zv);
                  if (write_r) stg4<double>((rin_sel == 0 ? A.lo.r1 : A.lo.r0) + A.lo.plane_off + e, pv.r);
                }
                if (kk - 1 == A.o1 - 1 && A.hi.z) {
                  stg4<T>(A.hi.z + A.hi.plane_off + e, zv);
                  if (write_r) stg4<double>((rin_sel == 0 ? A.hi.r1 : A.hi.r0) + A.hi.plane_off + e, pv.r);
                }
              }
            }
          }
        } else if (kk >= u.k0 && kk < u.k1) {
          // identity / Jacobi: z = r' or r'/d on this plane
          T zv[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            zv[c] = precond == 1 ? (T)cu.r[c] * iv[c] : (T)cu.r[c];
            acc = fmat(cu.r[c], (double)zv[c], acc);
            exceed |= !(fabs(cu.r[c]) <= res_target);
          }
          if (rows) {
            const int g = kk * pplane + e;
            stg4<T>(zout + g, zv);
            if (write_r) stg4<double>(rout + g, cu.r);
            if (SLABS && A.nslab > 1) {
              if (kk == A.o0 && A.lo.z) {
                stg4<T>(A.lo.z + A.lo.plane_off + e, zv);
                if (write_r) stg4<double>((rin_sel == 0 ? A.lo.r1 : A.lo.r0) + A.lo.plane_off + e, cu.r);
              }
              if (kk == A.o1 - 1 && A.hi.z) {
                stg4<T>(A.hi.z + A.hi.plane_off + e, zv);
                if (write_r) stg4<double>((rin_sel == 0 ? A.hi.r1 : A.hi.r0) + A.hi.plane_off + e, cu.r);
              }
            }
          }
        }
      }
      if (kk == u.k1 && cons.unit + cons.nb < A.U) {   // a unit done and another follows: publish it now
        const double sm = block_sum(acc, S.red);
        __syncthreads();
        const double mx = __syncthreads_or(exceed) ? 1.0 : 0.0;
        if (threadIdx.x == 0) {
          const double v[2] = {sm, mx};
          publish_unit<T>(A, part, set, cons.unit, 2, v, seq);
        }
        acc = 0.0;
        exceed = false;
      }
      const bool live = cursor_next<T>(A, cons);
      ++j;
      return live;
    };
    while (plane(pa, pb) && plane(pb, pa)) {
    }
    if (timing && threadIdx.x == 0) S.pt[2] = globaltimer();
    ticket = t0 + j;
    const double sm = block_sum(acc, S.red);   // the block's last unit
    __syncthreads();
    const double mx = __syncthreads_or(exceed) ? 1.0 : 0.0;
    if (threadIdx.x == 0) {
      const double v[2] = {sm, mx};
      publish_unit<T>(A, part, set, last_unit, 2, v, seq);
    }
  }
  __syncthreads();
}

// final, after a converged solve: state p = x (+ alpha p pending) on the
// unknowns and 0 elsewhere (project() replaces p, solver.py:278-280); a solve
// that does not converge leaves p as it was (project() raises first)
template <typename T>
__device__ void finish_x(const PcgArgs<T>& A, int unit, T alpha, const T* __restrict__ p, bool zero) {
  const Dims& d = A.d;
  const Unit t = unit_of<T>(A, unit);
  const int tx = threadIdx.x % QX, ty = threadIdx.x / QX;
  const int i = t.i0 + 4 * tx, j = t.j0 + ty;
  if (i >= d.nx || j >= d.ny) return;
  const int plane = d.nx * d.ny, pplane = A.nxp * d.ny;
#pragma unroll 4
  for (int k = t.k0; k < t.k1; ++k) {
    const int g = k * pplane + j * A.nxp + i;   // pitched PCG vectors: quad-aligned
    const int c = k * plane + j * d.nx + i;      // state pressure (unpitched)
    const uint32_t cw4 = *reinterpret_cast<const uint32_t*>(A.code + g);
    T xv[4], pv[4];
    ld4<T>(A.x + g, xv);
    if (alpha != (T)0) ld4<T>(p + g, pv);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i + q >= d.nx) break;
      if (zero || !((cw4 >> (8 * q + 6)) & 1u)) A.state_p[c + q] = (T)0;
      else A.state_p[c + q] = alpha != (T)0 ? xv[q] + alpha * pv[q] : xv[q];
    }
  }
}

// ---------------------------------------------------------------------------
// Phase end for z-slab solves (nslab > 1).  The last block of this slab to
// arrive folds the slab's partials (fixed order), publishes them in the root
// slab's value table and meets the other slabs at the root's counter (system
// scope: slabs may live on different GPUs, reached over NVLink); then it
// releases its own slab.  Every block then combines the slab values in slab
// order, so all blocks of all slabs hold the same bits.
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ void slab_reduce(const PcgArgs<T>& A, const Blk& blk, const double* part, int pset, unsigned seq, int nval,
                            unsigned maxmask, double* out, PcgShared<T>& S) {
  __syncthreads();
  unsigned* count = A.bar;
  unsigned* gen = A.bar + 32;
  if (threadIdx.x == 0) {
    S.gen0 = ld_acquire(gen);
    __threadfence_system();   // this block's writes (and its pushes into peer slabs) before the arrival
    S.last = atomicAdd(count, 1u) == (unsigned)blk.n - 1;
    if (S.last) __threadfence();
  }
  __syncthreads();
  if (S.last) {
    // this slab's chunk sums (the same tree as the whole grid's), published
    // at their global chunk index in the root's table
    fold_chunks<T>(A, part, pset, seq, nval, maxmask, false, S);
    const int ng = (A.tiles + 31) >> 5, ni = A.nchunk * ng, nig = A.nchunk_g * ng;
    for (int e = threadIdx.x; e < nval * ni; e += blockDim.x) {   // item sums at their global item index
      const int q = e / ni, it = e - q * ni;
      A.xval[((size_t)pset * 3 + q) * nig + A.chunk0 * ng + it] = S.grp[q][it];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned* xc = A.xbar;
      unsigned* xg = A.xbar + 32;
      const unsigned g = ld_acquire_sys(xg);
      __threadfence_system();
      if (atomicAdd_system(xc, 1u) == (unsigned)A.nslab - 1) {
        atomicExch_system(xc, 0u);
        __threadfence_system();
        atomicAdd_system(xg, 1u);
      } else {
        const unsigned long long t0 = globaltimer();
        unsigned spins = 0;
        while (ld_acquire_sys(xg) == g) {
          __nanosleep(64);
          if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > A.timeout_ns) {
            A.rep->status = 3;
            *A.gate = 3;
            break;
          }
        }
      }
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    }
  } else if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    unsigned spins = 0;
    while (ld_acquire(gen) == S.gen0) {
      __nanosleep(32);
      if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > A.timeout_ns) {
        A.rep->status = 3;
        *A.gate = 3;
        break;
      }
    }
  }
  if (threadIdx.x == 0) {
    __threadfence_system();
    fence_proxy_async();   // the next phase's TMA reads see the pushed halo planes
  }
  __syncthreads();
  if (threadIdx.x < nval) {   // all global items in item order (volatile: peers write the table)
    const int q = threadIdx.x, nig = A.nchunk_g * ((A.tiles + 31) >> 5);
    const bool mx = (maxmask >> q) & 1u;
    const volatile double* xv = A.xval + ((size_t)pset * 3 + q) * nig;
    double v = xv[0];
    for (int c = 1; c < nig; ++c) {
      const double w = xv[c];
      v = mx ? ((w > v || w != w) ? w : v) : v + w;
    }
    S.vals[q] = v;
  }
  __syncthreads();
  for (int q = 0; q < nval; ++q) out[q] = S.vals[q];
  __syncthreads();
}

// Phase end: the reduced values out[0..nval) (thread-local; bit q of maxmask:
// max instead of sum) over the units' partials of set pset, published with
// tag seq.  One launch: wait for every unit's tag (no separate grid barrier)
// and fold; z-slabs: slab_reduce.
template <typename T, bool SLABS>
__device__ __forceinline__ void phase_end(const PcgArgs<T>& A, const Blk& blk, const double* part, int pset,
                                          unsigned seq, int nval, unsigned maxmask, double* out, PcgShared<T>& S,
                                          unsigned& epoch) {
  if (SLABS && A.nslab > 1) {
    slab_reduce<T>(A, blk, part, pset, seq, nval, maxmask, out, S);
    return;
  }
  // a grid barrier (one arrival counter: measured faster than every block
  // acquiring every unit's tag), then the chunk-structured fold
  grid_barrier(A.bar, A.gate, A.rep, A.timeout_ns, (unsigned)blk.n, epoch);
#ifdef CW_PCG_FOLD_MULTI   // developer comparison: the block-wide fold (not slab-split invariant)
  fold_multi(part, A.U, A.PS, nval, maxmask, out, S.fold);
#else
  fold_chunks<T>(A, part, pset, seq, nval, maxmask, false, S);
  sum_items<T>(A, S, nval, maxmask, out);   // S.grp / S.vals are next written a phase later
#endif
}

template <typename T, bool SLABS>
__device__ __forceinline__ void pcg_body(const PcgArgs<T>& A, const Blk& blk, uint8_t* smem_raw) {
  // dynamic smem is the only shared allocation of this kernel, so it starts
  // at the (1 KB aligned) base of the block's window; keep every access on
  // this array so the compiler emits LDS/STS rather than generic loads
  uint8_t* ring = smem_raw;
  PcgShared<T>& S =
      *reinterpret_cast<PcgShared<T>*>(smem_raw + (size_t)StageLayout<T>::STAGE * StageLayout<T>::DEPTH);
  if (*(volatile int*)A.gate) return;  // uniform across blocks: set before launch
  if ((smem_u32(smem_raw) & 127u) != 0u) {   // TMA destinations need 128-byte alignment
    if (threadIdx.x == 0) { A.rep->status = 3; *A.gate = 3; }
    return;
  }
  for (int e = threadIdx.x; e < 64 * 4; e += blockDim.x) S.lut[e] = A.lut[e];
  if (threadIdx.x == 0) {
    for (int s = 0; s < StageLayout<T>::DEPTH; ++s) mbar_init(&S.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  __syncthreads();
  DevReport* rep = A.rep;
  const int U = A.U;
  const int B = blk.n;
  const bool lead = blk.id == 0 && threadIdx.x == 0;
  unsigned ticket = 0;
  unsigned epoch = 0;    // grid barriers passed (every thread keeps the count)
  unsigned seq = 0;      // phases started: the tag the units publish (tags zeroed before the launch)
  // two partial sets, alternated by phase: a unit's slot is rewritten only
  // after every block has folded it
  double* P[2] = {A.part, A.part + 3 * A.PS};
  double red[3];

  if ((A.probe_mode == 8 || (A.probe_mode >= 13 && A.probe_mode <= 15)) && lead) rep->criterion = 0.0;
  if (A.probe_mode == 16 && lead) rep->criterion = 1e30;
  ++seq;
  for (int u = blk.id; u < U; u += B) phase0<T, SLABS>(A, P[0], 0, seq, u, S);
  phase_end<T, SLABS>(A, blk, P[0], 0, seq, 3, 6u, red, S, epoch);
  const double b2 = red[0], bmax = red[1], divmax = red[2];
  if (lead) report_max<T>(rep, SLOT_DIV_BEFORE, (T)divmax);
  if (*(volatile int*)A.gate == 3) {
    if (lead) rep->status = 3;
    return;
  }
  if (!isfinite(bmax)) {                     // pcg_solve raises on a non-finite rhs
    if (lead) { rep->status = 4; *A.gate = 4; }
    return;
  }
  if (b2 == 0.0) {                           // linalg.py:329-330: x = 0, 0 iterations
    for (int u = blk.id; u < U; u += B) finish_x<T>(A, u, (T)0, A.p0, true);
    if (lead) { rep->iterations = 0; rep->converged = 1; rep->criterion = 0.0; }
    return;
  }
  const double res_target = A.res_factor * bmax;   // solver.py:266 (b.any() holds: b2 > 0)
  const double tol = A.tol;

  // z = W r0, rz, max|r0|  (pcg_solve:342-345)
  ++seq;
  phaseB<T, SLABS, false, false>(A, blk, P[1], 1, seq, S, ring, ticket, 0.0, res_target, 0);
  phase_end<T, SLABS>(A, blk, P[1], 1, seq, 2, 2u, red, S, epoch);
  double rz = red[0];
  double rmax = red[1];
  double crit = rz / b2;
  int it = 0, converged = 0, status = 0;
  bool finished = false;
  if (A.probe_mode) {
    unsigned long long wait_ns = 0;
    // timing probe: repeat one phase (1: A, 2: B, 3: barrier only) with its
    // grid barrier; the state's p is not meaningful afterwards
    for (int q = 0; q < A.probe_iters; ++q) {
      // 6, 7: phase A and phase B alternate as in the solve (7: stream only)
      const bool pa = A.probe_mode == 1 || A.probe_mode == 4 || (A.probe_mode >= 6 && A.probe_mode < 17 && !(q & 1));
      const bool pb = A.probe_mode == 2 || (A.probe_mode >= 6 && A.probe_mode < 17 && (q & 1));
      const bool stream = A.probe_mode == 4 || A.probe_mode == 7;
      if (pa && stream) phaseA<T, SLABS, true, true>(A, blk, P[0], 0, 0u, S, ring, ticket, false, (T)0.5, (T)0.0, (q >> 1) & 1);
      if (pa && !stream) phaseA<T, SLABS, true, false>(A, blk, P[0], 0, 0u, S, ring, ticket, false, (T)0.5, (T)0.0, (q >> 1) & 1);
      if (pb && A.probe_mode == 7) phaseB<T, SLABS, true, true>(A, blk, P[1], 1, 0u, S, ring, ticket, 0.0, res_target, (q >> 1) & 1);
      if (pb && A.probe_mode != 7) phaseB<T, SLABS, true, false>(A, blk, P[1], 1, 0u, S, ring, ticket, 0.0, res_target, (q >> 1) & 1);
      if (A.probe_mode >= 13 && threadIdx.x == 0)
        wait_ns += A.probe_mode == 13 ? S.pt[1] - S.pt[0] : S.pt[2] - S.pt[0];
      const unsigned long long ta = globaltimer();
      grid_barrier(A.bar, A.gate, rep, A.timeout_ns, (unsigned)B, epoch);
      if (A.probe_mode < 13) wait_ns += globaltimer() - ta;
      if (A.probe_mode == 5) {   // barrier plus phase B's two folds
        rz += fold_partials(P[1], B, 0, S.bc);
        rmax = fold_partials(P[1] + A.PS, B, 1, S.bc);
      }
      if (A.probe_mode == 17) {   // barrier plus the chunk-structured fold of two values
        fold_chunks<T>(A, P[1], 1, 0u, 2, 2u, false, S);
        sum_items<T>(A, S, 2, 2u, red);
        rz += red[0];
      }
      if (A.probe_mode == 18) {   // barrier plus fold_multi of two values
        fold_multi(P[1], A.U, A.PS, 2, 2u, red, S.fold);
        rz += red[0];
      }
    }
    // 8: report the mean grid-barrier wait per block and phase (us) as the criterion
    if (A.probe_mode == 8 && threadIdx.x == 0) atomicAdd(&rep->criterion, (double)wait_ns * 1e-3 / (B * A.probe_iters));
    // 13: mean time to the first landed stage, 14: mean time to the end of the
    // jobs (per block and phase, us); 15 / 16: max / min over blocks of the latter
    if (A.probe_mode >= 13 && threadIdx.x == 0) {
      const double us = (double)wait_ns * 1e-3 / A.probe_iters;
      if (A.probe_mode <= 14) atomicAdd(&rep->criterion, us / B);
      else if (A.probe_mode == 15) atomic_max_nonneg(&rep->criterion, us);
      else atomicMin(reinterpret_cast<unsigned long long*>(&rep->criterion), (unsigned long long)__double_as_longlong(us));
    }
    if (lead) { rep->iterations = A.probe_iters; rep->converged = 1; }
    return;
  }
  if (0.0 <= crit && crit < tol && rmax == 0.0) { converged = 1; finished = true; }   // rmax: the |r| > res_target flag
  else if (rz < 0.0) { finished = true; }
  int rsel = 0;       // r lives in r0 (0) or r1 (1)
  int psel = 1;       // previous p lives in p0 (0) or p1 (1); the first pass ignores it
  double alpha = 0.0, beta = 0.0;
  while (!finished) {
    if (it >= A.max_iter) break;
    ++it;
    const bool first = it == 1;
    ++seq;
    if (first) phaseA<T, SLABS, false, false>(A, blk, P[0], 0, seq, S, ring, ticket, true, (T)0, (T)0, psel);
    else phaseA<T, SLABS, true, false>(A, blk, P[0], 0, seq, S, ring, ticket, false, (T)beta, (T)alpha, psel);
    phase_end<T, SLABS>(A, blk, P[0], 0, seq, 1, 0u, red, S, epoch);
    const double pAp = red[0];
    psel ^= 1;                                // the new p went to the other buffer
    if (*(volatile int*)A.gate == 3) { status = 3; alpha = 0.0; break; }
    if (pAp <= 0.0) { it -= 1; alpha = 0.0; break; }   // linalg.py:354-355
    alpha = rz / pAp;
    ++seq;
    phaseB<T, SLABS, true, false>(A, blk, P[1], 1, seq, S, ring, ticket, alpha, res_target, rsel);
    phase_end<T, SLABS>(A, blk, P[1], 1, seq, 2, 2u, red, S, epoch);
    const double rz_new = red[0];
    rmax = red[1];
    rsel ^= 1;
    crit = rz_new / b2;
    if (*(volatile int*)A.gate == 3) { status = 3; break; }
    if (0.0 <= crit && crit < tol && rmax == 0.0) { converged = 1; break; }
    if (rz_new < 0.0) break;                  // linalg.py:364-365
    beta = rz_new / rz;
    rz = rz_new;
  }
  // state p = x, plus the alpha p of the last completed iteration if pending
  const T* plast = psel == 0 ? A.p0 : A.p1;
  if (converged)
    for (int u = blk.id; u < U; u += B) finish_x<T>(A, u, (T)alpha, plast, false);
  if (lead) {
    rep->iterations = it;
    rep->converged = converged;
    rep->criterion = crit;
    if (status) rep->status = status;
    else if (!converged) { rep->status = 1; *A.gate = 1; }
  }
}

// One slab per launch (the whole grid, or this GPU's slab of a multi-GPU solve).
// SLABS = false: a whole grid; the z-slab code paths are compiled out.
template <typename T, bool SLABS>
__global__ void __launch_bounds__(PCG_THREADS, CW_PCG_MINB) k_pcg(const __grid_constant__ PcgArgs<T> A) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  pcg_body<T, SLABS>(A, Blk{(int)blockIdx.x, (int)gridDim.x}, smem_raw);
}

// All slabs of a z-slab solve on one device in one cooperative launch: blocks
// [s*bps, (s+1)*bps) serve slab s, whose arguments sit in global memory.
template <typename T>
__global__ void __launch_bounds__(PCG_THREADS, CW_PCG_MINB) k_pcg_slabs(const PcgArgs<T>* __restrict__ all, int bps) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int s = blockIdx.x / bps;
  pcg_body<T, true>(all[s], Blk{(int)(blockIdx.x - s * bps), bps}, smem_raw);
}

}  // namespace cw
