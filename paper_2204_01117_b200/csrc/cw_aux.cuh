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
  r->criterion = 0.0;
  for (int s = 0; s < 4; ++s) { r->fmax[s] = 0u; r->dmax[s] = 0ull; }
  r->bad_index[0] = 0x7fffffffffffffffLL;
  r->bad_index[1] = 0x7fffffffffffffffLL;
}

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

}  // namespace cw
