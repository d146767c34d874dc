// Porosity voxelizer on the device, bit-exact with the reference
// (grid.py:133-325, geometry.py:145-241, scenario.py:351-360, grid.py:473-478).
//
// Pipeline per design:
//   host  : per-object constants -- candidate cell ranges, sub-sample
//           coordinates, per-triangle edge/determinant data (O(#triangles),
//           same float64 expressions as the reference's numpy code)
//   device: k_vox_columns  one thread per (x,y) sample column of a mesh object:
//                          +z ray against every triangle, even-odd parity per
//                          z sample, ambiguity detection (grid.py:144-202)
//           k_vox_points   ambiguous columns: primary-direction point casts
//                          (geometry.py:145-192, 204-233)
//           k_vox_merge    one thread per cell: objects in order, uniform
//                          sample state (boxes), numpy pairwise sample mean
//           k_vox_complex  one warp per cell touched by a mesh: per-sample
//                          state across objects, pairwise mean
// All float64 arithmetic uses explicitly rounded intrinsics (no FMA
// contraction), mirroring numpy's evaluation order: einsum 3-term dot
// products are (x0*y0 + x2*y2) + x1*y1, np.cross and np.linalg.norm as written.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/citywind_b200.h"
#include "cw_common.cuh"

namespace cwv {

using namespace cw;

#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DMUL __dmul_rn
#define DDIV __ddiv_rn

constexpr double EPS_BARY = 1e-10, EPS_T = 1e-9, EPS_PAR = 1e-10;
constexpr int MAX_CROSS = 64;

struct ColTri {      // column-cast data per triangle (grid.py:153-164)
  double v0x, v0y, v0z, e1x, e1y, e1z, e2x, e2y, e2z, sdet, xlo, xhi, ylo, yhi;
  int vertical;
};
struct PtTri {       // point-cast data per non-degenerate triangle (geometry.py:152-166)
  double v0[3], e1[3], e2[3], nrm[3], area2, pvec[3], sdet;
  int parallel;
};
struct MeshObj {
  int a0[3], n[3];           // candidate cell ranges (start, count) per axis
  int NS[3];                 // sample counts per axis (n * subdiv)
  int tri_off, ntri;         // into ColTri array
  int pt_off, npt;           // into PtTri array
  int xs_off, ys_off, zs_off;
  long long bits_off;        // into the bit lattice (uint32 words)
  int zwords;                // words per column
  double lo[3], hi[3];       // AABB expanded by EPS_T (points_in_mesh)
};
struct VoxObj {
  int kind, is_mesh, mesh;   // mesh: index into MeshObj
  double phi, lad;
  double lo[3], hi[3];       // box
};
struct VoxGrid {
  int nx, ny, nz, sd, nsamp;
  double ox, oy, oz, hx, hy, hz;
  // painted-porosity base layer (grid.py:337-377), or paint == nullptr
  const uint8_t* paint;      // (ny, nx) raster, row 0 = min-y row: pixel (j, i) at j*nx + i
  const uint8_t* tmask;      // tree mask of the same shape, or nullptr
  int kmax;                  // planes [0, kmax) carry the paint
  double tree_lad;
};

// numpy pairwise summation (loops_utils.h.src pairwise_sum), n <= 512
__device__ double pw_block(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = DADD(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = DADD(r[j], a[i + j]);
  double res = DADD(DADD(DADD(r[0], r[1]), DADD(r[2], r[3])), DADD(DADD(r[4], r[5]), DADD(r[6], r[7])));
  for (; i < n; ++i) res = DADD(res, a[i]);
  return res;
}
__device__ double pw_sum(const double* a, int n) {   // recursion unrolled for n <= 512
  if (n <= 128) return pw_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  auto half = [](const double* b, int m) -> double {
    if (m <= 128) return pw_block(b, m);
    int m2 = m / 2;
    m2 -= m2 % 8;
    auto q = [](const double* c, int k) -> double {
      if (k <= 128) return pw_block(c, k);
      int k2 = k / 2;
      k2 -= k2 % 8;
      return DADD(pw_block(c, k2), pw_block(c + k2, k - k2));
    };
    return DADD(q(b, m2), q(b + m2, m - m2));
  };
  return DADD(half(a, n2), half(a + n2, n - n2));
}
// pairwise sum of n copies of v (uniform sample state), same association
__device__ double pw_const(double v, int n) {
  double buf[8];
  for (int j = 0; j < 8; ++j) buf[j] = v;
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = DADD(r, v);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = v;
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = DADD(r[j], v);
    double res = DADD(DADD(DADD(r[0], r[1]), DADD(r[2], r[3])), DADD(DADD(r[4], r[5]), DADD(r[6], r[7])));
    for (; i < n; ++i) res = DADD(res, v);
    return res;
  }
  (void)buf;
  int n2 = n / 2;
  n2 -= n2 % 8;
  return DADD(pw_const(v, n2), pw_const(v, n - n2));
}

__device__ __forceinline__ double axis_center(double o, int i, double h) {
  return DADD(o, DMUL(DADD((double)i, 0.5), h));       // grid.py:70-73
}

// exact covered fraction along one axis (grid.py:221-227)
__device__ __forceinline__ double cover_frac(double o, int i, double h, double lo, double hi) {
  const double c = axis_center(o, i, h);
  const double cl = DSUB(c, DMUL(0.5, h));
  const double ov = DSUB(fmin(hi, DADD(cl, h)), fmax(lo, cl));
  double f = DDIV(ov, h);
  f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
  return f;
}

__device__ __forceinline__ double dot3(const double* x, const double* y) {   // einsum order
  return DADD(DADD(DMUL(x[0], y[0]), DMUL(x[2], y[2])), DMUL(x[1], y[1]));
}

// ---- +z column casts (grid.py:144-202) -------------------------------------
__global__ void k_vox_columns(MeshObj m, const ColTri* __restrict__ tris, const double* __restrict__ xs,
                              const double* __restrict__ ys, const double* __restrict__ zs,
                              uint32_t* __restrict__ bits, uint8_t* __restrict__ amb, int* err) {
  const long long ncol = (long long)m.NS[0] * m.NS[1];
  for (long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x; col < ncol;
       col += (long long)gridDim.x * blockDim.x) {
    const int xi = (int)(col / m.NS[1]), yi = (int)(col % m.NS[1]);
    const double px = xs[m.xs_off + xi], py = ys[m.ys_off + yi];
    double cr[MAX_CROSS];
    int nc = 0;
    bool ambiguous = false;
    for (int t = 0; t < m.ntri; ++t) {
      const ColTri T = tris[m.tri_off + t];
      if (T.vertical) {
        if (px >= DSUB(T.xlo, EPS_T) && px <= DADD(T.xhi, EPS_T) && py >= DSUB(T.ylo, EPS_T) &&
            py <= DADD(T.yhi, EPS_T))
          ambiguous = true;
        continue;
      }
      const double rx = DSUB(px, T.v0x), ry = DSUB(py, T.v0y);
      const double u = DDIV(DSUB(DMUL(rx, T.e2y), DMUL(ry, T.e2x)), T.sdet);
      const double v = DDIV(DSUB(DMUL(ry, T.e1x), DMUL(rx, T.e1y)), T.sdet);
      const double w = DSUB(DSUB(1.0, u), v);
      const bool loose = u >= -EPS_BARY && v >= -EPS_BARY && w >= -EPS_BARY;
      if (!loose) continue;
      if (u <= EPS_BARY || v <= EPS_BARY || w <= EPS_BARY) ambiguous = true;
      const double zc = DADD(DADD(T.v0z, DMUL(u, T.e1z)), DMUL(v, T.e2z));
      if (nc < MAX_CROSS) cr[nc++] = zc;
      else ambiguous = true;
    }
    uint32_t* out = bits + m.bits_off + col * m.zwords;
    for (int q = 0; q < m.zwords; ++q) out[q] = 0u;
    if (!ambiguous) {
      for (int a = 1; a < nc; ++a) {            // insertion sort (np.sort)
        const double key = cr[a];
        int b = a - 1;
        while (b >= 0 && cr[b] > key) { cr[b + 1] = cr[b]; --b; }
        cr[b + 1] = key;
      }
      for (int zi = 0; zi < m.NS[2] && !ambiguous; ++zi) {
        const double z = zs[m.zs_off + zi];
        for (int a = 0; a < nc; ++a)
          if (fabs(DSUB(cr[a], z)) <= EPS_T) { ambiguous = true; break; }
      }
    }
    if (ambiguous) { amb[col] = 1; continue; }
    amb[col] = 0;
    for (int zi = 0; zi < m.NS[2]; ++zi) {
      const double z = zs[m.zs_off + zi];
      int idx = 0;                               // searchsorted(cr, z, 'left')
      while (idx < nc && cr[idx] < z) ++idx;
      if (((nc - idx) & 1) == 1) out[zi >> 5] |= 1u << (zi & 31);
    }
  }
  (void)err;
}

// ---- primary-direction point casts (geometry.py:145-192, 204-233) ----------
__global__ void k_vox_points(MeshObj m, const PtTri* __restrict__ tris, const double* __restrict__ xs,
                             const double* __restrict__ ys, const double* __restrict__ zs,
                             const int* __restrict__ cols, int ncols, double dx, double dy, double dz,
                             uint32_t* __restrict__ bits, int* err) {
  const long long n = (long long)ncols * m.NS[2];
  const double dir[3] = {dx, dy, dz};
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const int cidx = (int)(q / m.NS[2]), zi = (int)(q % m.NS[2]);
    const int col = cols[cidx];
    const int xi = col / m.NS[1], yi = col % m.NS[1];
    const double p[3] = {xs[m.xs_off + xi], ys[m.ys_off + yi], zs[m.zs_off + zi]};
    bool inside = false;
    const bool active = p[0] >= m.lo[0] && p[0] <= m.hi[0] && p[1] >= m.lo[1] && p[1] <= m.hi[1] &&
                        p[2] >= m.lo[2] && p[2] <= m.hi[2];
    if (active) {
      long long hits = 0;
      bool amb = false;
      for (int t = 0; t < m.npt; ++t) {
        const PtTri& T = tris[m.pt_off + t];
        const double tv[3] = {DSUB(p[0], T.v0[0]), DSUB(p[1], T.v0[1]), DSUB(p[2], T.v0[2])};
        const double u = DDIV(dot3(tv, T.pvec), T.sdet);
        const double qv[3] = {DSUB(DMUL(tv[1], T.e1[2]), DMUL(tv[2], T.e1[1])),
                              DSUB(DMUL(tv[2], T.e1[0]), DMUL(tv[0], T.e1[2])),
                              DSUB(DMUL(tv[0], T.e1[1]), DMUL(tv[1], T.e1[0]))};
        const double v = DDIV(dot3(qv, dir), T.sdet);
        const double tt = DDIV(dot3(qv, T.e2), T.sdet);
        const double w = DSUB(DSUB(1.0, u), v);
        const bool loose = u >= -EPS_BARY && v >= -EPS_BARY && w >= -EPS_BARY;
        if (!T.parallel) {
          if (loose && tt > EPS_T) ++hits;
          if (loose && (u <= EPS_BARY || v <= EPS_BARY || w <= EPS_BARY || fabs(tt) <= EPS_T)) amb = true;
        } else {
          const double pd = DDIV(fabs(dot3(tv, T.nrm)), T.area2);
          if (pd <= EPS_T) amb = true;
        }
      }
      if (amb) atomicOr(err, 1);   // would need the seeded re-casts (geometry.py:222-233)
      inside = (hits & 1) == 1;
    }
    if (inside) atomicOr(bits + m.bits_off + (long long)col * m.zwords + (zi >> 5), 1u << (zi & 31));
  }
}

// ---- per-cell merge ---------------------------------------------------------
struct CellAcc {
  double kphi;
  int kind;     // 0 = no entry in cell_kind
};

__device__ __forceinline__ void note_kind(CellAcc& a, double ophi, int kind, int* nwarn) {
  if (a.kind == 0 || ophi < a.kphi) {     // grid.py:256-265 (strict: first object wins ties)
    if (a.kind != 0 && a.kind != kind && nwarn) atomicAdd(nwarn, 1);
    a.kphi = ophi;
    a.kind = kind;
  }
}

__device__ __forceinline__ bool mesh_covers(const MeshObj& m, const uint32_t* bits, int sd, int i, int j, int k,
                                            int sx, int sy, int sz) {
  const int xi = (i - m.a0[0]) * sd + sx, yi = (j - m.a0[1]) * sd + sy, zi = (k - m.a0[2]) * sd + sz;
  const long long col = (long long)xi * m.NS[1] + yi;
  return (bits[m.bits_off + col * m.zwords + (zi >> 5)] >> (zi & 31)) & 1u;
}
__device__ __forceinline__ bool in_range(const MeshObj& m, int i, int j, int k) {
  return i >= m.a0[0] && i < m.a0[0] + m.n[0] && j >= m.a0[1] && j < m.a0[1] + m.n[1] && k >= m.a0[2] &&
         k < m.a0[2] + m.n[2];
}

// the base layer under the objects at cell c: open air, or the painted
// raster extruded over planes [0, kmax) (decode_painted_porosity, grid.py:337-377)
__device__ __forceinline__ void base_layer(const VoxGrid& g, long long c, int8_t& blab, double& bphi, double& blad) {
  blab = AIR;
  bphi = 1.0;
  blad = 0.0;
  if (!g.paint) return;
  const long long plane = (long long)g.nx * g.ny;
  const long long k = c / plane;
  if (k >= g.kmax) return;
  const long long p = c - k * plane;
  const bool tree = g.tmask != nullptr && g.tmask[p] != 0;
  bphi = DDIV((double)g.paint[p], 255.0);                 // image / 255.0 (float64)
  blab = tree ? (int8_t)TREE : ((bphi < 1.0) ? (int8_t)BUILDING : (int8_t)AIR);
  blad = tree ? g.tree_lad : 0.0;
}

// final label/phi/lad of one cell: combine_porosity(base, objects)
// (scenario.py:351-360) and overlay under the boundary frame (grid.py:473-478)
__device__ __forceinline__ void write_cell(const VoxGrid& g, long long c, int8_t bnd, double phi, double lad,
                                           const CellAcc& a, int8_t* labels, double* ophi, double* olad) {
  int8_t lab = AIR;
  if (a.kind != 0 && (phi < DSUB(1.0, 1e-12) || lad > 0.0)) lab = (int8_t)a.kind;   // grid.py:320-324
  int8_t blab;
  double bphi, blad;
  base_layer(g, c, blab, bphi, blad);
  int8_t comb = phi < bphi ? lab : blab;                  // take = add.phi < base.phi
  if (lab == TREE && comb == AIR) comb = TREE;
  ophi[c] = phi < bphi ? phi : bphi;                      // np.minimum
  olad[c] = lad > blad ? lad : blad;                      // np.maximum
  labels[c] = (bnd == AIR && comb != AIR) ? comb : bnd;
}

__global__ void k_vox_merge(VoxGrid g, const VoxObj* __restrict__ objs, int nobj, const MeshObj* __restrict__ meshes,
                            const uint32_t* __restrict__ bits, const int8_t* __restrict__ bnd, int8_t* labels,
                            double* ophi, double* olad, int* complex_list, int* ncomplex, int* nwarn) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny), k = (int)(c / ((long long)g.nx * g.ny));
    double sp = 1.0, sl = 0.0;
    bool phi_e = false, lad_e = false, complex_cell = false;
    CellAcc a{0.0, 0};
    for (int o = 0; o < nobj && !complex_cell; ++o) {
      const VoxObj& ob = objs[o];
      const double eff = ob.kind == TREE ? 1.0 : ob.phi;
      if (ob.is_mesh) {
        const MeshObj& m = meshes[ob.mesh];
        if (!in_range(m, i, j, k)) continue;
        bool any = false;
        for (int s = 0; s < g.nsamp && !any; ++s) {
          const int sx = s / (g.sd * g.sd), sy = (s / g.sd) % g.sd, sz = s % g.sd;
          any = mesh_covers(m, bits, g.sd, i, j, k, sx, sy, sz);
        }
        if (any) complex_cell = true;
        continue;
      }
      const double fx = cover_frac(g.ox, i, g.hx, ob.lo[0], ob.hi[0]);
      const double fy = cover_frac(g.oy, j, g.hy, ob.lo[1], ob.hi[1]);
      const double fz = cover_frac(g.oz, k, g.hz, ob.lo[2], ob.hi[2]);
      const double cov = DMUL(DMUL(fx, fy), fz);
      if (!(cov > 0.0)) continue;
      phi_e = true;
      sp = DMUL(sp, DSUB(1.0, DMUL(cov, DSUB(1.0, eff))));   // grid.py:306-307
      if (ob.kind == TREE && ob.lad > 0.0) {
        lad_e = true;
        sl = DADD(sl, DMUL(ob.lad, cov));
      }
      note_kind(a, eff, ob.kind, nwarn);
    }
    if (complex_cell) {
      complex_list[atomicAdd(ncomplex, 1)] = (int)c;
      continue;
    }
    const double phi = phi_e ? DDIV(pw_const(sp, g.nsamp), (double)g.nsamp) : 1.0;
    const double lad = lad_e ? DDIV(pw_const(sl, g.nsamp), (double)g.nsamp) : 0.0;
    write_cell(g, c, bnd[c], phi, lad, a, labels, ophi, olad);
  }
}

// one warp per mesh-touched cell: per-sample state, objects in order
__global__ void k_vox_complex(VoxGrid g, const VoxObj* __restrict__ objs, int nobj,
                              const MeshObj* __restrict__ meshes, const uint32_t* __restrict__ bits,
                              const int8_t* __restrict__ bnd, const int* __restrict__ list, int nlist,
                              int8_t* labels, double* ophi, double* olad, int* nwarn) {
  extern __shared__ double wbuf[];   // [warps][2][512]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* sbuf = wbuf + (size_t)wib * 1024;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
  for (int q = gw; q < nlist; q += nw) {
    const long long c = list[q];
    const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny), k = (int)(c / ((long long)g.nx * g.ny));
    double sp[16], sl[16];
    for (int t = 0; t < 16; ++t) { sp[t] = 1.0; sl[t] = 0.0; }
    bool phi_e = false, lad_e = false;
    CellAcc a{0.0, 0};
    for (int o = 0; o < nobj; ++o) {
      const VoxObj& ob = objs[o];
      const double eff = ob.kind == TREE ? 1.0 : ob.phi;
      if (ob.is_mesh) {
        const MeshObj& m = meshes[ob.mesh];
        if (!in_range(m, i, j, k)) continue;
        bool ins[16];
        bool any = false;
        for (int t = 0; t < 16; ++t) {
          const int s = lane + 32 * t;
          ins[t] = false;
          if (s < g.nsamp) {
            const int sx = s / (g.sd * g.sd), sy = (s / g.sd) % g.sd, sz = s % g.sd;
            ins[t] = mesh_covers(m, bits, g.sd, i, j, k, sx, sy, sz);
            any |= ins[t];
          }
        }
        if (!__any_sync(0xffffffffu, any)) continue;       // not covered (grid.py:288)
        phi_e = true;
        const bool lad_on = ob.kind == TREE && ob.lad > 0.0;
        if (lad_on) lad_e = true;
        for (int t = 0; t < 16; ++t) {
          const double cand = ins[t] ? eff : 1.0;
          sp[t] = fmin(sp[t], cand);                          // np.minimum (no NaN here)
          if (lad_on) sl[t] = fmax(sl[t], ins[t] ? ob.lad : 0.0);
        }
        note_kind(a, eff, ob.kind, lane == 0 ? nwarn : nullptr);
        continue;
      }
      const double fx = cover_frac(g.ox, i, g.hx, ob.lo[0], ob.hi[0]);
      const double fy = cover_frac(g.oy, j, g.hy, ob.lo[1], ob.hi[1]);
      const double fz = cover_frac(g.oz, k, g.hz, ob.lo[2], ob.hi[2]);
      const double cov = DMUL(DMUL(fx, fy), fz);
      if (!(cov > 0.0)) continue;
      phi_e = true;
      const double tgt = DSUB(1.0, DMUL(cov, DSUB(1.0, eff)));
      const bool lad_on = ob.kind == TREE && ob.lad > 0.0;
      if (lad_on) lad_e = true;
      const double add = DMUL(ob.lad, cov);
      for (int t = 0; t < 16; ++t) {
        sp[t] = DMUL(sp[t], tgt);
        if (lad_on) sl[t] = DADD(sl[t], add);
      }
      note_kind(a, eff, ob.kind, lane == 0 ? nwarn : nullptr);
    }
    // pairwise means in sample order (sx, sy, sz) row-major
    for (int t = 0; t < 16; ++t) {
      const int s = lane + 32 * t;
      if (s < g.nsamp) { sbuf[s] = sp[t]; sbuf[512 + s] = sl[t]; }
    }
    __syncwarp();
    if (lane == 0) {
      const double phi = phi_e ? DDIV(pw_sum(sbuf, g.nsamp), (double)g.nsamp) : 1.0;
      const double lad = lad_e ? DDIV(pw_sum(sbuf + 512, g.nsamp), (double)g.nsamp) : 0.0;
      write_cell(g, c, bnd[c], phi, lad, a, labels, ophi, olad);
    }
    __syncwarp();
  }
}

}  // namespace cwv

// ---------------------------------------------------------------------------
// host side

using namespace cwv;

static thread_local std::string v_err;
extern "C" const char* cw_last_error(void);

namespace {
struct HostTri {
  double v0[3], v1[3], v2[3];
};
double axis_center_h(double o, int i, double h) { return o + ((double)i + 0.5) * h; }
double dot3_h(const double* x, const double* y) { return (x[0] * y[0] + x[2] * y[2]) + x[1] * y[1]; }
void cross_h(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
}  // namespace

// fixed primary cast direction after normalisation (geometry.py:22-23)
static const double PRIMARY[3] = {0x1.2470b1aa2db79p-2, 0x1.24c01e97c27f3p-1, 0x1.89c714ad8027ap-1};

struct cw_ctx;
extern int cw_internal_fail(int code, const char* msg);
extern int cw_internal_device(cw_ctx* c, int* nx, int* ny, int* nz, double* h, double* origin);
extern void cw_internal_paint(cw_ctx* c, const uint8_t** image, const uint8_t** mask, int* kmax, double* tree_lad);
extern void* cw_internal_scratch(cw_ctx* c, int slot, size_t bytes);

#define VCUDA(call)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return cw_internal_fail(CW_ERR_CUDA, (std::string(#call) + ": " + cudaGetErrorString(e_)).c_str()); \
  } while (0)

extern "C" int cw_voxelize(cw_ctx* ctx, const cw_object* objs, int n_obj, const double* verts, const int* tris,
                           int subdiv, const signed char* d_bnd, signed char* d_labels, double* d_phi,
                           double* d_lad, int* n_overlap, void* stream) {
  if (!ctx || (n_obj > 0 && !objs) || !d_bnd || !d_labels || !d_phi || !d_lad)
    return cw_internal_fail(CW_ERR_INVALID, "null argument");
  if (subdiv < 1 || subdiv > 8) return cw_internal_fail(CW_ERR_INVALID, "subdiv must be in [1, 8]");
  int nx, ny, nz;
  double h[3], org[3];
  int rc = cw_internal_device(ctx, &nx, &ny, &nz, h, org);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int dims[3] = {nx, ny, nz};
  const int sd = subdiv;

  std::vector<VoxObj> vobj(n_obj);
  std::vector<MeshObj> meshes;
  std::vector<ColTri> ctri;
  std::vector<PtTri> ptri;
  std::vector<double> xs, ys, zs;
  long long nbits = 0;
  for (int o = 0; o < n_obj; ++o) {
    const cw_object& ob = objs[o];
    if (ob.kind != BUILDING && ob.kind != TREE) return cw_internal_fail(CW_ERR_INVALID, "object kind must be 1 or 2");
    VoxObj& v = vobj[o];
    v.kind = ob.kind;
    v.phi = ob.phi;
    v.lad = ob.lad;
    v.is_mesh = ob.shape == 1;
    v.mesh = -1;
    for (int a = 0; a < 3; ++a) { v.lo[a] = ob.lo[a]; v.hi[a] = ob.hi[a]; }
    if (!v.is_mesh) continue;
    if (!verts || !tris || ob.n_verts < 1 || ob.n_tris < 1) return cw_internal_fail(CW_ERR_INVALID, "empty mesh");
    const double* V = verts + 3LL * ob.vert_offset;
    const int* TI = tris + 3LL * ob.tri_offset;
    double bmin[3], bmax[3];
    for (int a = 0; a < 3; ++a) { bmin[a] = V[a]; bmax[a] = V[a]; }
    for (int q = 1; q < ob.n_verts; ++q)
      for (int a = 0; a < 3; ++a) { bmin[a] = std::min(bmin[a], V[3 * q + a]); bmax[a] = std::max(bmax[a], V[3 * q + a]); }
    MeshObj m{};
    bool empty = false;
    for (int a = 0; a < 3; ++a) {       // _candidate_ranges (grid.py:133-141)
      const double pad = 0.5 * h[a];
      const double lo = bmin[a] - pad, hi = bmax[a] + pad;
      int first = -1, last = -2;
      for (int i = 0; i < dims[a]; ++i) {
        const double c = axis_center_h(org[a], i, h[a]);
        if (c >= lo && c <= hi) { if (first < 0) first = i; last = i; }
      }
      if (first < 0) { empty = true; break; }
      m.a0[a] = first;
      m.n[a] = last - first + 1;
      m.NS[a] = m.n[a] * sd;
    }
    if (empty) { v.is_mesh = 1; v.mesh = -2; continue; }   // skipped entirely (grid.py:285)
    for (int a = 0; a < 3; ++a) { m.lo[a] = bmin[a] - 1e-9; m.hi[a] = bmax[a] + 1e-9; }
    // sub-sample coordinates (grid.py:267-271)
    std::vector<double>* dst[3] = {&xs, &ys, &zs};
    int* offs[3] = {&m.xs_off, &m.ys_off, &m.zs_off};
    for (int a = 0; a < 3; ++a) {
      *offs[a] = (int)dst[a]->size();
      for (int ci = 0; ci < m.n[a]; ++ci) {
        const double base = org[a] + (double)(m.a0[a] + ci) * h[a];
        for (int s = 0; s < sd; ++s) dst[a]->push_back(base + (((double)s + 0.5) * h[a]) / (double)sd);
      }
    }
    // triangles
    m.tri_off = (int)ctri.size();
    m.pt_off = (int)ptri.size();
    for (int t = 0; t < ob.n_tris; ++t) {
      HostTri T;
      for (int a = 0; a < 3; ++a) {
        T.v0[a] = V[3 * TI[3 * t + 0] + a];
        T.v1[a] = V[3 * TI[3 * t + 1] + a];
        T.v2[a] = V[3 * TI[3 * t + 2] + a];
      }
      double e1[3], e2[3];
      for (int a = 0; a < 3; ++a) { e1[a] = T.v1[a] - T.v0[a]; e2[a] = T.v2[a] - T.v0[a]; }
      ColTri C;
      C.v0x = T.v0[0]; C.v0y = T.v0[1]; C.v0z = T.v0[2];
      C.e1x = e1[0]; C.e1y = e1[1]; C.e1z = e1[2]; C.e2x = e2[0]; C.e2y = e2[1]; C.e2z = e2[2];
      const double det = e1[0] * e2[1] - e1[1] * e2[0];
      const double scale = std::max(std::fabs(e1[0] * e2[1]) + std::fabs(e1[1] * e2[0]), 1e-300);
      C.vertical = std::fabs(det) <= 1e-12 * scale;
      C.sdet = C.vertical ? 1.0 : det;
      C.xlo = std::min(std::min(T.v0[0], T.v1[0]), T.v2[0]);
      C.xhi = std::max(std::max(T.v0[0], T.v1[0]), T.v2[0]);
      C.ylo = std::min(std::min(T.v0[1], T.v1[1]), T.v2[1]);
      C.yhi = std::max(std::max(T.v0[1], T.v1[1]), T.v2[1]);
      ctri.push_back(C);
      // point-cast data (geometry.py:152-166), degenerate triangles dropped
      double nrm[3];
      cross_h(e1, e2, nrm);
      const double area2 = std::sqrt((nrm[0] * nrm[0] + nrm[1] * nrm[1]) + nrm[2] * nrm[2]);
      if (!(area2 * 0.5 > 1e-12)) continue;
      PtTri P;
      for (int a = 0; a < 3; ++a) { P.v0[a] = T.v0[a]; P.e1[a] = e1[a]; P.e2[a] = e2[a]; P.nrm[a] = nrm[a]; }
      P.area2 = area2;
      cross_h(PRIMARY, e2, P.pvec);
      const double d2 = dot3_h(e1, P.pvec);
      P.parallel = std::fabs(d2) <= 1e-10 * area2;
      P.sdet = P.parallel ? 1.0 : d2;
      ptri.push_back(P);
    }
    m.ntri = (int)ctri.size() - m.tri_off;
    m.npt = (int)ptri.size() - m.pt_off;
    m.zwords = (m.NS[2] + 31) / 32;
    m.bits_off = nbits;
    nbits += (long long)m.NS[0] * m.NS[1] * m.zwords;
    v.mesh = (int)meshes.size();
    meshes.push_back(m);
  }
  // objects skipped for empty candidate ranges do not take part at all
  std::vector<VoxObj> live;
  for (auto& v : vobj)
    if (!(v.is_mesh && v.mesh == -2)) live.push_back(v);

  // device scratch from the context's grow-only arena (one slot per buffer):
  // no cudaMalloc / cudaFree per design evaluation
  int slot_n = 0;
  auto dalloc = [&](void** p, size_t b) -> cudaError_t {
    *p = cw_internal_scratch(ctx, slot_n++, std::max<size_t>(b, 16));
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  };
  VoxObj* d_obj = nullptr;
  MeshObj* d_mesh = nullptr;
  ColTri* d_ct = nullptr;
  PtTri* d_pt = nullptr;
  double *d_xs = nullptr, *d_ys = nullptr, *d_zs = nullptr;
  uint32_t* d_bits = nullptr;
  uint8_t* d_amb = nullptr;
  int *d_err = nullptr, *d_list = nullptr, *d_cols = nullptr;
  const long long ncell = (long long)nx * ny * nz;
  VCUDA(dalloc((void**)&d_obj, live.size() * sizeof(VoxObj)));
  VCUDA(dalloc((void**)&d_mesh, meshes.size() * sizeof(MeshObj)));
  VCUDA(dalloc((void**)&d_ct, ctri.size() * sizeof(ColTri)));
  VCUDA(dalloc((void**)&d_pt, ptri.size() * sizeof(PtTri)));
  VCUDA(dalloc((void**)&d_xs, xs.size() * 8));
  VCUDA(dalloc((void**)&d_ys, ys.size() * 8));
  VCUDA(dalloc((void**)&d_zs, zs.size() * 8));
  VCUDA(dalloc((void**)&d_bits, nbits * 4));
  VCUDA(dalloc((void**)&d_err, 4 * sizeof(int)));
  VCUDA(dalloc((void**)&d_list, ncell * sizeof(int)));
  VCUDA(cudaMemsetAsync(d_err, 0, 4 * sizeof(int), st));
  if (!live.empty()) VCUDA(cudaMemcpyAsync(d_obj, live.data(), live.size() * sizeof(VoxObj), cudaMemcpyHostToDevice, st));
  if (!meshes.empty()) VCUDA(cudaMemcpyAsync(d_mesh, meshes.data(), meshes.size() * sizeof(MeshObj), cudaMemcpyHostToDevice, st));
  if (!ctri.empty()) VCUDA(cudaMemcpyAsync(d_ct, ctri.data(), ctri.size() * sizeof(ColTri), cudaMemcpyHostToDevice, st));
  if (!ptri.empty()) VCUDA(cudaMemcpyAsync(d_pt, ptri.data(), ptri.size() * sizeof(PtTri), cudaMemcpyHostToDevice, st));
  if (!xs.empty()) VCUDA(cudaMemcpyAsync(d_xs, xs.data(), xs.size() * 8, cudaMemcpyHostToDevice, st));
  if (!ys.empty()) VCUDA(cudaMemcpyAsync(d_ys, ys.data(), ys.size() * 8, cudaMemcpyHostToDevice, st));
  if (!zs.empty()) VCUDA(cudaMemcpyAsync(d_zs, zs.data(), zs.size() * 8, cudaMemcpyHostToDevice, st));
  // 1) column casts of every mesh, one read-back of all ambiguous-column
  // flags, 2) point casts of the ambiguous columns of every mesh
  std::vector<long long> col_off(meshes.size() + 1, 0);
  for (size_t mi = 0; mi < meshes.size(); ++mi)
    col_off[mi + 1] = col_off[mi] + (long long)meshes[mi].NS[0] * meshes[mi].NS[1];
  const long long ncol_all = std::max(col_off.back(), 1LL);
  VCUDA(dalloc((void**)&d_amb, ncol_all));
  VCUDA(dalloc((void**)&d_cols, ncol_all * sizeof(int)));
  for (size_t mi = 0; mi < meshes.size(); ++mi) {
    const MeshObj& m = meshes[mi];
    const long long ncol = col_off[mi + 1] - col_off[mi];
    const int nb = (int)std::min<long long>((ncol + 127) / 128, 4096);
    k_vox_columns<<<nb, 128, 0, st>>>(m, d_ct, d_xs, d_ys, d_zs, d_bits, d_amb + col_off[mi], d_err);
    VCUDA(cudaGetLastError());
  }
  if (!meshes.empty()) {
    std::vector<uint8_t> amb(col_off.back());
    VCUDA(cudaMemcpyAsync(amb.data(), d_amb, col_off.back(), cudaMemcpyDeviceToHost, st));
    VCUDA(cudaStreamSynchronize(st));
    std::vector<int> cols;
    std::vector<long long> cbeg(meshes.size() + 1, 0);
    for (size_t mi = 0; mi < meshes.size(); ++mi) {
      for (long long q = col_off[mi]; q < col_off[mi + 1]; ++q)
        if (amb[q]) cols.push_back((int)(q - col_off[mi]));
      cbeg[mi + 1] = (long long)cols.size();
    }
    if (!cols.empty()) {
      VCUDA(cudaMemcpyAsync(d_cols, cols.data(), cols.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      for (size_t mi = 0; mi < meshes.size(); ++mi) {
        const long long nc = cbeg[mi + 1] - cbeg[mi];
        if (nc == 0) continue;
        const MeshObj& m = meshes[mi];
        const long long np = nc * m.NS[2];
        k_vox_points<<<(int)std::min<long long>((np + 127) / 128, 4096), 128, 0, st>>>(
            m, d_pt, d_xs, d_ys, d_zs, d_cols + cbeg[mi], (int)nc, PRIMARY[0], PRIMARY[1], PRIMARY[2], d_bits, d_err);
        VCUDA(cudaGetLastError());
      }
    }
  }
  // 3) merge
  VoxGrid g{nx, ny, nz, sd, sd * sd * sd, org[0], org[1], org[2], h[0], h[1], h[2], nullptr, nullptr, 0, 0.0};
  cw_internal_paint(ctx, &g.paint, &g.tmask, &g.kmax, &g.tree_lad);
  k_vox_merge<<<(int)std::min<long long>((ncell + 255) / 256, 148LL * 16), 256, 0, st>>>(
      g, d_obj, (int)live.size(), d_mesh, d_bits, (const int8_t*)d_bnd, (int8_t*)d_labels, d_phi, d_lad, d_list,
      d_err + 1, d_err + 2);
  VCUDA(cudaGetLastError());
  int h_err[4];
  VCUDA(cudaMemcpyAsync(h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, st));
  VCUDA(cudaStreamSynchronize(st));
  if (h_err[1] > 0) {
    const int warps = 4;
    k_vox_complex<<<(h_err[1] + warps - 1) / warps, 32 * warps, warps * 1024 * sizeof(double), st>>>(
        g, d_obj, (int)live.size(), d_mesh, d_bits, (const int8_t*)d_bnd, d_list, h_err[1], (int8_t*)d_labels, d_phi,
        d_lad, d_err + 2);
    VCUDA(cudaGetLastError());
    VCUDA(cudaMemcpyAsync(h_err, d_err, sizeof(h_err), cudaMemcpyDeviceToHost, st));
    VCUDA(cudaStreamSynchronize(st));
  }
  if (n_overlap) *n_overlap = h_err[2];
  if (h_err[0]) return cw_internal_fail(CW_ERR_GEOMETRY, "point unclassifiable by the primary cast (needs re-casts)");
  return CW_OK;
}
