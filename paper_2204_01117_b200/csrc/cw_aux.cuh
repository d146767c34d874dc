// Small per-design / per-scenario kernels: operator code, W-diagonal mean,
// drag coefficient, region averages, report initialisation.
#pragma once
#include "../../include/citywind_b200.h"
#include "cw_common.cuh"
#include "cw_step.cuh"

namespace cw {

__global__ void k_report_init(DevReport* r) {
  r->iterations = 0;
  r->converged = 0;
  r->status = 0;
  r->halo_need = 0;
  r->criterion = 0.0;
  for (int s = 0; s < 4; ++s) { r->fmax[s] = 0u; r->dmax[s] = 0ull; }
  r->bad_index[0] = 0x7fffffffffffffffLL;
  r->bad_index[1] = 0x7fffffffffffffffLL;
}

// the step's report (written to rep_live by its kernels) into the ring slot
// the device counts; enqueue_stage / slab solves write their slot directly
// and only advance the count
__global__ void k_report_commit(const DevReport* live, DevReport* ring, int* slot) {
  ring[*slot] = *live;
  *slot += 1;
}
__global__ void k_slot_bump(int* slot) { *slot += 1; }

// Per-cell operator code (build_pressure_matrix, linalg.py:67-112):
// bit 6 = unknown (interior_mask, grid.py:481-484); bit q (q = 0..5 for
// +x,-x,+y,-y,+z,-z) = that neighbour is an unknown (off-diagonal -1/h^2 and
// +1/h^2 on the diagonal) or an outlet (Dirichlet: +1/h^2 on the diagonal).
// flag[0]: some unknown touches an outlet; flag[1]: an unknown has d = 0.
__global__ void k_build_code(Dims d, int nxp, const int8_t* __restrict__ lab, uint8_t* __restrict__ code,
                             int* flag) {
  const long long n = d.ncell();
  CW_GRID_STRIDE(c, n) {
    const int8_t l = lab[c];
    const int i = (int)(c % d.nx), j = (int)((c / d.nx) % d.ny), k = (int)(c / ((long long)d.nx * d.ny));
    const long long pc = ((long long)k * d.ny + j) * nxp + i;   // pitched (PCG layout)
    if (!is_unknown(l)) { code[pc] = 0; continue; }
    const int pos[3] = {i, j, k}, ext[3] = {d.nx, d.ny, d.nz};
    const long long str[3] = {1, d.nx, (long long)d.nx * d.ny};
    uint8_t cd = 64;
    bool outl = false;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int ax = q >> 1, sg = (q & 1) ? -1 : 1;
      const int np = pos[ax] + sg;
      if (np < 0 || np >= ext[ax]) continue;
      const int8_t nl = lab[c + sg * str[ax]];
      if (is_unknown(nl)) cd |= (uint8_t)(1 << q);
      else if (nl == OUTLET) { cd |= (uint8_t)(1 << q); outl = true; }
    }
    code[pc] = cd;
    if (outl) atomicOr(&flag[0], 1);
    if ((cd & 63) == 0 && k >= d.o0 && k < d.o1) atomicOr(&flag[1], 1);   // owned planes (z-slab halos are partial)
  }
}

__device__ __forceinline__ double code_d(uint8_t cd, double wx, double wy, double wz) {
  double s = 0.0;
  const double w[3] = {wx, wy, wz};
#pragma unroll
  for (int q = 0; q < 6; ++q)
    if (cd & (1 << q)) s += w[q >> 1];
  return s;
}

// sum over unknowns of diag(W) (closed form of K^T K) for
// default_projection_tol (solver.py:235-243); fixed grid => deterministic.
__global__ void k_wdiag_partials(Dims d, int nxp, const uint8_t* __restrict__ code, double wx, double wy, double wz,
                                 double om, double* part, long long* cnt, double* jpart) {
  __shared__ double red[32];
  const long long plane = (long long)d.nx * d.ny;
  double acc = 0.0, jacc = 0.0;
  long long m = 0;
  const double w[3] = {wx, wy, wz};
  for (long long c0 = d.o0 * plane + (long long)blockIdx.x * blockDim.x + threadIdx.x; c0 < d.o1 * plane;
       c0 += (long long)gridDim.x * blockDim.x) {   // owned planes
    const int pos[3] = {(int)(c0 % d.nx), (int)((c0 / d.nx) % d.ny), (int)(c0 / ((long long)d.nx * d.ny))};
    const long long c = ((long long)pos[2] * d.ny + pos[1]) * nxp + pos[0];
    const uint8_t cd = code[c];
    if (!(cd & 64)) continue;
    const int ext[3] = {d.nx, d.ny, d.nz};
    const long long str[3] = {1, nxp, (long long)nxp * d.ny};
    const double di = code_d(cd, wx, wy, wz);
    jacc += 1.0 / di;
    double wii = (2.0 - om) * om / di;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (pos[ax] + 1 >= ext[ax]) continue;
      const uint8_t cn = code[c + str[ax]];
      if (!(cn & 64)) continue;
      const double sn = (2.0 - om) * om / code_d(cn, wx, wy, wz);
      const double f = w[ax] * om / di;
      wii += sn * f * f;
    }
    acc += wii;
    ++m;
  }
  const double s = block_sum(acc, red);
  __syncthreads();
  const double mm = block_sum((double)m, red);
  __syncthreads();
  const double js = block_sum(jacc, red);
  if (threadIdx.x == 0) { part[blockIdx.x] = s; cnt[blockIdx.x] = (long long)mm; jpart[blockIdx.x] = js; }
}

// drag_factor_cells (solver.py:123-135) in float64, stored in the step precision
template <typename T>
__global__ void k_drag_coef(long long n, const double* __restrict__ phi, const double* __restrict__ lad,
                            const int8_t* __restrict__ lab, cw_params prm, T* __restrict__ g, int* any) {
  CW_GRID_STRIDE(c, n) {
    double v = 0.0;
    if (lab[c] == BUILDING) {
      const double ratio = (1.0 - phi[c]) / (phi[c] + prm.drag_eps);
      v = prm.cd_building * prm.drag_a * pow(ratio, prm.drag_b);
    } else if (lab[c] == TREE) {
      v = prm.cd_tree * lad[c];
    }
    g[c] = (T)v;
    if (v != 0.0) atomicOr(any, 1);
  }
}

struct RegionBoxes {
  int n;
  double lo[16][3], hi[16][3];
};

// region_average_speed (solver.py:535-549): per-block partial sums and counts
template <typename T>
__global__ void k_region_partials(Dims d, double ox, double oy, double oz, const T* __restrict__ u,
                                  const T* __restrict__ v, const T* __restrict__ w,
                                  const int8_t* __restrict__ lab, RegionBoxes B, double* part,
                                  long long* cnt) {
  __shared__ double red[32];
  double s[16];
  long long m[16];
  for (int b = 0; b < 16; ++b) { s[b] = 0.0; m[b] = 0; }
  const long long plane = (long long)d.nx * d.ny;
  for (long long c = d.o0 * plane + (long long)blockIdx.x * blockDim.x + threadIdx.x; c < d.o1 * plane;
       c += (long long)gridDim.x * blockDim.x) {   // owned planes
    if (lab[c] != AIR) continue;
    const int i = (int)(c % d.nx), j = (int)((c / d.nx) % d.ny), k = (int)(c / ((long long)d.nx * d.ny));
    const double cx = ox + ((double)i + 0.5) * d.ddx;
    const double cy = oy + ((double)j + 0.5) * d.ddy;
    const double cz = oz + ((double)(k + d.kg0) + 0.5) * d.ddz;   // global plane index
    bool anyb = false;
    for (int b = 0; b < B.n; ++b)
      anyb |= cx >= B.lo[b][0] && cx <= B.hi[b][0] && cy >= B.lo[b][1] && cy <= B.hi[b][1] &&
              cz >= B.lo[b][2] && cz <= B.hi[b][2];
    if (!anyb) continue;
    const long long ui = ((long long)k * d.ny + j) * (d.nx + 1) + i;
    const long long vi = ((long long)k * (d.ny + 1) + j) * d.nx + i;
    const T uc = (T)0.5 * (u[ui] + u[ui + 1]);
    const T vc = (T)0.5 * (v[vi] + v[vi + d.nx]);
    const T wc = (T)0.5 * (w[c] + w[c + (long long)d.nx * d.ny]);
    const double sp = (double)sqrt(uc * uc + vc * vc + wc * wc);
    for (int b = 0; b < B.n; ++b)
      if (cx >= B.lo[b][0] && cx <= B.hi[b][0] && cy >= B.lo[b][1] && cy <= B.hi[b][1] &&
          cz >= B.lo[b][2] && cz <= B.hi[b][2]) { s[b] += sp; m[b] += 1; }
  }
  for (int b = 0; b < B.n; ++b) {
    const double t = block_sum(s[b], red);
    __syncthreads();
    const double mm = block_sum((double)m[b], red);
    __syncthreads();
    if (threadIdx.x == 0) { part[blockIdx.x * 16 + b] = t; cnt[blockIdx.x * 16 + b] = (long long)mm; }
  }
}

__global__ void k_region_fold(int nblocks, int n, const double* part, const long long* cnt, double* out,
                              long long* cout) {
  const int b = threadIdx.x;
  if (b >= n) return;
  double s = 0.0;
  long long m = 0;
  for (int q = 0; q < nblocks; ++q) { s += part[q * 16 + b]; m += cnt[q * 16 + b]; }
  out[b] = m > 0 ? s / (double)m : 0.0;
  cout[b] = m;
}

// ---------------------------------------------------------------------------
// Reference layout <-> device layout (the drop-in binding of refbind.py).
// The reference's FlowState arrays are float64, C-order (ex, ey, ez) with x
// slowest (grid.py:492-571); device fields are x-fastest (ez, ey, ex) in the
// context precision.  For every y the (x, z) plane is a 2-D transpose: 32 x 32
// tiles through shared memory, both global sides coalesced.  blockIdx.z = y.
template <typename T>
__global__ void k_ref_to_dev(const double* __restrict__ src, T* __restrict__ dst, int ex, int ey, int ez) {
  __shared__ double tile[32][33];
  const int y = blockIdx.z;
  const int z0 = blockIdx.x * 32, x0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {          // read rows x, contiguous z
    const int x = x0 + r, z = z0 + threadIdx.x;
    if (x < ex && z < ez) tile[r][threadIdx.x] = src[((long long)x * ey + y) * ez + z];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {          // write rows z, contiguous x
    const int z = z0 + r, x = x0 + threadIdx.x;
    if (x < ex && z < ez) dst[((long long)z * ey + y) * ex + x] = (T)tile[threadIdx.x][r];
  }
}

template <typename T>
__global__ void k_dev_to_ref(const T* __restrict__ src, double* __restrict__ dst, int ex, int ey, int ez) {
  __shared__ double tile[32][33];
  const int y = blockIdx.z;
  const int z0 = blockIdx.y * 32, x0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {          // read rows z, contiguous x
    const int z = z0 + r, x = x0 + threadIdx.x;
    if (x < ex && z < ez) tile[r][threadIdx.x] = (double)src[((long long)z * ey + y) * ex + x];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {          // write rows x, contiguous z
    const int x = x0 + r, z = z0 + threadIdx.x;
    if (x < ex && z < ez) dst[((long long)x * ey + y) * ez + z] = tile[threadIdx.x][r];
  }
}

// the same fold, added to running sums in step order (the reference's
// sums[ri] += region_average_speed(...), optimize.py:96-99); counts keep the
// latest step's air-cell count (labels are fixed: the same every step)
__global__ void k_region_accum(int nblocks, int n, const double* part, const long long* cnt, double* sums,
                               long long* counts, const int* gate) {
  if (*gate) return;
  const int b = threadIdx.x;
  if (b >= n) return;
  double s = 0.0;
  long long m = 0;
  for (int q = 0; q < nblocks; ++q) { s += part[q * 16 + b]; m += cnt[q * 16 + b]; }
  sums[b] += m > 0 ? s / (double)m : 0.0;
  counts[b] = m;
}

}  // namespace cw

namespace cw {

// ---------------------------------------------------------------------------
// Velocity samples at arbitrary points, float64 (Advector.sample/velocity_at,
// advection.py:49-111: trilinear with clamped indices on the staggered grids)
template <typename T>
__device__ __forceinline__ double sample64(const T* __restrict__ a, int ex, int ey, int ez, double fx, double fy,
                                           double fz) {
  int i0 = (int)floor(fx), j0 = (int)floor(fy), k0 = (int)floor(fz);
  const int im = ex - 2 > 0 ? ex - 2 : 0, jm = ey - 2 > 0 ? ey - 2 : 0, km = ez - 2 > 0 ? ez - 2 : 0;
  i0 = i0 < 0 ? 0 : (i0 > im ? im : i0);
  j0 = j0 < 0 ? 0 : (j0 > jm ? jm : j0);
  k0 = k0 < 0 ? 0 : (k0 > km ? km : k0);
  double tx = fx - i0, ty = fy - j0, tz = fz - k0;
  tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);
  ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
  tz = tz < 0.0 ? 0.0 : (tz > 1.0 ? 1.0 : tz);
  const long long sx = ex > 1 ? 1 : 0, sy = ey > 1 ? ex : 0, sz = ez > 1 ? (long long)ex * ey : 0;
  const long long b = ((long long)k0 * ey + j0) * ex + i0;
  const double c000 = a[b], c100 = a[b + sx], c010 = a[b + sy], c110 = a[b + sx + sy];
  const double c001 = a[b + sz], c101 = a[b + sx + sz], c011 = a[b + sy + sz], c111 = a[b + sx + sy + sz];
  const double ox = 1.0 - tx, oy = 1.0 - ty, oz = 1.0 - tz;
  const double c00 = c000 * ox + c100 * tx, c10 = c010 * ox + c110 * tx;
  const double c01 = c001 * ox + c101 * tx, c11 = c011 * ox + c111 * tx;
  const double c0 = c00 * oy + c10 * ty, c1 = c01 * oy + c11 * ty;
  return c0 * oz + c1 * tz;
}

// velocity at grid coordinates (X, Y, Z) = (p - origin) / h
template <typename T>
__device__ __forceinline__ void velocity64(const Dims& d, const T* u, const T* v, const T* w, double X, double Y,
                                           double Z, double& us, double& vs, double& ws) {
  us = sample64<T>(u, d.nx + 1, d.ny, d.nz, X, Y - 0.5, Z - 0.5);
  vs = sample64<T>(v, d.nx, d.ny + 1, d.nz, X - 0.5, Y, Z - 0.5);
  ws = sample64<T>(w, d.nx, d.ny, d.nz + 1, X - 0.5, Y - 0.5, Z);
}

struct Frame {
  double o[3], h[3], lo[3], hi[3];
};

template <typename T>
__global__ void k_probe(Dims d, Frame fr, const T* __restrict__ u, const T* __restrict__ v,
                        const T* __restrict__ w, const double* __restrict__ pts, int n, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double us, vs, ws;
  velocity64<T>(d, u, v, w, (pts[3 * q] - fr.o[0]) / fr.h[0], (pts[3 * q + 1] - fr.o[1]) / fr.h[1],
                (pts[3 * q + 2] - fr.o[2]) / fr.h[2], us, vs, ws);
  out[3 * q] = us;
  out[3 * q + 1] = vs;
  out[3 * q + 2] = ws;
}

__device__ __forceinline__ bool outside(const Frame& fr, const double* p) {
  return p[0] < fr.lo[0] || p[1] < fr.lo[1] || p[2] < fr.lo[2] || p[0] > fr.hi[0] || p[1] > fr.hi[1] ||
         p[2] > fr.hi[2];
}

// trace_streamlines (solver.py:488-532): one thread per seed, RK2 midpoint steps
template <typename T>
__global__ void k_streamlines(Dims d, Frame fr, const T* __restrict__ u, const T* __restrict__ v,
                              const T* __restrict__ w, const double* __restrict__ seeds, int nseeds,
                              double step_len, int max_steps, double min_speed, double* __restrict__ paths,
                              int* __restrict__ len) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseeds) return;
  double* out = paths + (size_t)s * (max_steps + 1) * 3;
  double p[3] = {seeds[3 * s], seeds[3 * s + 1], seeds[3 * s + 2]};
  if (outside(fr, p)) { len[s] = 0; return; }
  int m = 0;
  for (int a = 0; a < 3; ++a) out[a] = p[a];
  ++m;
  auto vel = [&](const double* x, double* vv) {
    velocity64<T>(d, u, v, w, (x[0] - fr.o[0]) / fr.h[0], (x[1] - fr.o[1]) / fr.h[1], (x[2] - fr.o[2]) / fr.h[2],
                  vv[0], vv[1], vv[2]);
  };
  for (int it = 0; it < max_steps; ++it) {
    double v1[3], v2[3], mid[3];
    vel(p, v1);
    const double s1 = sqrt((v1[0] * v1[0] + v1[1] * v1[1]) + v1[2] * v1[2]);
    if (s1 < min_speed) break;
    for (int a = 0; a < 3; ++a) mid[a] = p[a] + 0.5 * step_len * v1[a] / s1;
    if (outside(fr, mid)) break;
    vel(mid, v2);
    const double s2 = sqrt((v2[0] * v2[0] + v2[1] * v2[1]) + v2[2] * v2[2]);
    if (s2 < min_speed) break;
    for (int a = 0; a < 3; ++a) p[a] = p[a] + step_len * v2[a] / s2;
    if (outside(fr, p)) break;
    for (int a = 0; a < 3; ++a) out[3 * m + a] = p[a];
    ++m;
  }
  len[s] = m;
}

}  // namespace cw
