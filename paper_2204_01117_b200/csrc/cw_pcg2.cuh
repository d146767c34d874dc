// Pressure projection, second implementation: the same persistent PCG
// (same barriers, partials and stopping logic as k_pcg) but every phase is a
// sync-free per-warp z-march with L1-cached neighbour loads:
//   * a block is a 32x8 tile of (x, y) columns, one thread per column;
//   * in-plane neighbours come through L1 (the sibling threads load the same
//     lines); z-neighbours live in registers as the thread marches up;
//   * no shared memory and no __syncthreads inside a phase, so each warp
//     streams independently and occupancy is limited by registers only.
// W r' is applied in one pass as the 13-point footprint of K^T K: q = r'/d
// is evaluated on the fly at the 7 new points a column needs per plane and
// y = s (r' + w sum w_a q_{-a}) at the 3 upper neighbours, with the z-window
// rolled in registers.  Global data written by other blocks in the previous
// phase is visible after the grid barrier (its gpu-scope fence invalidates
// L1).
#pragma once
#include "cw_pcg.cuh"

namespace cw {

constexpr int P2_TX = 32, P2_TY = 8, P2_THREADS = P2_TX * P2_TY;

struct P2Unit {
  int i, j, k0, k1;   // this thread's column and the unit's z-range
  bool col;           // column inside the grid
};

template <typename T>
__device__ __forceinline__ P2Unit p2_unit(const PcgArgs<T>& A, int u) {
  const int per = A.ntx * A.nty;
  const int tz = u / per, rem = u - tz * per;
  P2Unit t;
  t.i = (rem % A.ntx) * P2_TX + (int)(threadIdx.x % P2_TX);
  t.j = (rem / A.ntx) * P2_TY + (int)(threadIdx.x / P2_TX);
  t.k0 = tz * A.zc;
  t.k1 = min(t.k0 + A.zc, A.d.nz);
  t.col = t.i < A.d.nx && t.j < A.d.ny;
  return t;
}

// ---- phase 0: b = -div/dt, r0 = b - A x0, x = x0 (masked p) --------------
template <typename T>
__device__ void p2_phase0(const PcgArgs<T>& A, double* part, int unit, double* red) {
  const Dims& d = A.d;
  const P2Unit t = p2_unit<T>(A, unit);
  const long long plane = (long long)d.nx * d.ny, pplane = (long long)A.nxp * d.ny;
  auto x0 = [&](int i, int j, int k) -> double {   // masked warm start
    if (i < 0 || i >= d.nx || j < 0 || j >= d.ny || k < 0 || k >= d.nz) return 0.0;
    if (!(A.code[k * pplane + (long long)j * A.nxp + i] & 64)) return 0.0;
    return (double)A.state_p[k * plane + (long long)j * d.nx + i];
  };
  double b2 = 0.0, bmax = 0.0, dmax = 0.0;
  if (t.col) {
    const int i = t.i, j = t.j;
    double xm = x0(i, j, t.k0 - 1), xc = x0(i, j, t.k0);
    for (int k = t.k0; k < t.k1; ++k) {
      const double xn = x0(i, j, k + 1);
      const long long c = k * plane + (long long)j * d.nx + i;
      const long long pc = k * pplane + (long long)j * A.nxp + i;
      const uint8_t cd = A.code[pc];
      if (cd & 64) {
        const long long ui = ((long long)k * d.ny + j) * (d.nx + 1) + i;
        const long long vi = ((long long)k * (d.ny + 1) + j) * d.nx + i;
        double div = ((double)A.u[ui + 1] - (double)A.u[ui]) / d.ddx +
                     ((double)A.v[vi + d.nx] - (double)A.v[vi]) / d.ddy;
        if (!d.is2d) div = div + ((double)A.w[c + plane] - (double)A.w[c]) / d.ddz;
        const double b = -div / A.dt;
        const double ax = (double)A.lut[(cd & 63) * 4] * xc -
                          ((double)A.wx * (x0(i - 1, j, k) + x0(i + 1, j, k)) +
                           (double)A.wy * (x0(i, j - 1, k) + x0(i, j + 1, k)) + (double)A.wz * (xm + xn));
        A.r0[pc] = b - ax;
        A.x[pc] = (T)xc;
        b2 += b * b;
        const double ab = fabs(b), ad = fabs(div);
        bmax = (ab > bmax || ab != ab) ? ab : bmax;
        dmax = (ad > dmax || ad != ad) ? ad : dmax;
      }
      xm = xc;
      xc = xn;
    }
  }
  const double s0 = block_sum(b2, red);
  __syncthreads();
  const double m1 = block_max(bmax, red);
  __syncthreads();
  const double m2 = block_max(dmax, red);
  if (threadIdx.x == 0) {
    part[unit] = s0;
    part[A.U + unit] = m1;
    part[2 * A.U + unit] = m2;
  }
  __syncthreads();
}

// zero the state pressure off the unknowns (project() sets p = 0 there); a
// separate pass because phase 0 reads p at neighbours
template <typename T>
__device__ void p2_zero_frame(const PcgArgs<T>& A, int unit) {
  const Dims& d = A.d;
  const P2Unit t = p2_unit<T>(A, unit);
  if (!t.col) return;
  const long long plane = (long long)d.nx * d.ny, pplane = (long long)A.nxp * d.ny;
  for (int k = t.k0; k < t.k1; ++k)
    if (!(A.code[k * pplane + (long long)t.j * A.nxp + t.i] & 64)) A.state_p[k * plane + (long long)t.j * d.nx + t.i] = (T)0;
}

// ---- phase A: p' = z + beta p, x += alpha_prev p, Ap = A p' ---------------
template <typename T>
__device__ double p2_phaseA(const PcgArgs<T>& A, int unit, bool first, T beta, bool upd_x, T alpha_prev,
                            const T* __restrict__ pin, T* __restrict__ pout) {
  const Dims& d = A.d;
  const P2Unit t = p2_unit<T>(A, unit);
  if (!t.col) return 0.0;
  const long long pplane = (long long)A.nxp * d.ny;
  const int i = t.i, j = t.j;
  auto pn = [&](int ii, int jj, int kk) -> T {      // p' at a cell (0 outside the grid)
    if (ii < 0 || ii >= d.nx || jj < 0 || jj >= d.ny || kk < 0 || kk >= d.nz) return (T)0;
    const long long q = kk * pplane + (long long)jj * A.nxp + ii;
    const T zz = A.z[q];
    return first ? zz : zz + beta * pin[q];
  };
  double acc = 0.0;
  T pm = pn(i, j, t.k0 - 1), pc = pn(i, j, t.k0);
  for (int k = t.k0; k < t.k1; ++k) {
    const T pnx = pn(i, j, k + 1);
    const long long q = k * pplane + (long long)j * A.nxp + i;
    const uint8_t cd = A.code[q];
    if (cd & 64) {
      const double ap = (double)A.lut[(cd & 63) * 4] * (double)pc -
                        ((double)A.wx * ((double)pn(i - 1, j, k) + (double)pn(i + 1, j, k)) +
                         (double)A.wy * ((double)pn(i, j - 1, k) + (double)pn(i, j + 1, k)) +
                         (double)A.wz * ((double)pm + (double)pnx));
      pout[q] = pc;
      A.Ap[q] = (T)ap;
      if (upd_x) A.x[q] = A.x[q] + alpha_prev * pin[q];
      acc += (double)pc * ap;
    }
    pm = pc;
    pc = pnx;
  }
  return acc;
}

// ---- phase B: r' = r - alpha Ap, z = W r' (13-point, one pass) ------------
template <typename T>
__device__ void p2_phaseB(const PcgArgs<T>& A, int unit, bool use_ap, double alpha, const double* __restrict__ rin,
                          double* __restrict__ rout, bool write_r, double& acc, double& rmax) {
  const Dims& d = A.d;
  const P2Unit t = p2_unit<T>(A, unit);
  if (!t.col) return;
  const long long pplane = (long long)A.nxp * d.ny;
  const int i = t.i, j = t.j;
  const T om = A.om, c0 = ((T)2 - om) * om;
  auto rv = [&](long long q) -> double {
    double r = rin[q];
    if (use_ap) r = r - alpha * (double)A.Ap[q];
    return r;
  };
  auto qv = [&](int ii, int jj, int kk) -> T {      // q = r'/d (0 outside / off the unknowns)
    if (ii < 0 || ii >= d.nx || jj < 0 || jj >= d.ny || kk < 0 || kk >= d.nz) return (T)0;
    const long long q = kk * pplane + (long long)jj * A.nxp + ii;
    return (T)rv(q) * A.lut[(A.code[q] & 63) * 4 + 1];
  };
  auto sv = [&](int ii, int jj, int kk) -> T {      // s = (2-w) w / d (0 off the unknowns)
    if (ii < 0 || ii >= d.nx || jj < 0 || jj >= d.ny || kk < 0 || kk >= d.nz) return (T)0;
    return A.lut[(A.code[kk * pplane + (long long)jj * A.nxp + ii] & 63) * 4 + 2];
  };
  // y = s (r' + w sum_a w_a q_{-a}) with s r' = c0 q  (all zero off the unknowns)
  auto yv = [&](T q0, T qxm, T qym, T qzm, T s) -> T {
    return c0 * q0 + s * (om * (A.wx * qxm + A.wy * qym + A.wz * qzm));
  };
  // z-window: plane k-1 (m), k (c), k+1 (n)
  const int k0 = t.k0;
  T q_c = qv(i, j, k0), q_xm_c = qv(i - 1, j, k0), q_ym_c = qv(i, j - 1, k0);
  T q_m = qv(i, j, k0 - 1), q_xp_m = qv(i + 1, j, k0 - 1), q_yp_m = qv(i, j + 1, k0 - 1);
  T y_c = yv(q_c, q_xm_c, q_ym_c, q_m, sv(i, j, k0));
  double r_c = 0.0;
  {
    const long long q = k0 * pplane + (long long)j * A.nxp + i;
    if (k0 < d.nz) r_c = rv(q);
  }
  for (int k = k0; k < t.k1; ++k) {
    // new points on plane k (P+x, P+y, P+x-y, P-x+y) and k+1 (P, P-x, P-y)
    const T q_xp = qv(i + 1, j, k), q_yp = qv(i, j + 1, k);
    const T q_xpym = qv(i + 1, j - 1, k), q_xmyp = qv(i - 1, j + 1, k);
    const T q_n = qv(i, j, k + 1), q_xm_n = qv(i - 1, j, k + 1), q_ym_n = qv(i, j - 1, k + 1);
    const T y_xp = yv(q_xp, q_c, q_xpym, q_xp_m, sv(i + 1, j, k));
    const T y_yp = yv(q_yp, q_xmyp, q_c, q_yp_m, sv(i, j + 1, k));
    const T y_n = yv(q_n, q_xm_n, q_ym_n, q_c, sv(i, j, k + 1));
    const long long q = k * pplane + (long long)j * A.nxp + i;
    const uint8_t cd = A.code[q];
    double r_n = 0.0;
    if (k + 1 < d.nz) r_n = rv(q + pplane);
    if (cd & 64) {
      T zv;
      const T invd = A.lut[(cd & 63) * 4 + 1];
      if (A.precond == 2) zv = y_c + om * invd * (A.wx * y_xp + A.wy * y_yp + A.wz * y_n);
      else if (A.precond == 1) zv = (T)r_c * invd;
      else zv = (T)r_c;
      A.z[q] = zv;
      if (write_r) rout[q] = r_c;
      acc += r_c * (double)zv;
      const double ar = fabs(r_c);
      rmax = (ar > rmax || ar != ar) ? ar : rmax;
    }
    // roll the window up one plane
    q_m = q_c; q_xp_m = q_xp; q_yp_m = q_yp;
    q_c = q_n; q_xm_c = q_xm_n; q_ym_c = q_ym_n;
    y_c = y_n;
    r_c = r_n;
  }
  (void)q_xm_c;
  (void)q_ym_c;
}

template <typename T>
__device__ void p2_finish_x(const PcgArgs<T>& A, int unit, T alpha, const T* __restrict__ p, bool zero) {
  const Dims& d = A.d;
  const P2Unit t = p2_unit<T>(A, unit);
  if (!t.col) return;
  const long long plane = (long long)d.nx * d.ny, pplane = (long long)A.nxp * d.ny;
  for (int k = t.k0; k < t.k1; ++k) {
    const long long c = k * plane + (long long)t.j * d.nx + t.i;
    const long long q = k * pplane + (long long)t.j * A.nxp + t.i;
    if (zero) { A.state_p[c] = (T)0; continue; }
    if (A.code[q] & 64) A.state_p[c] = alpha != (T)0 ? A.x[q] + alpha * p[q] : A.x[q];
  }
}

template <typename T>
__global__ void __launch_bounds__(P2_THREADS, 3) k_pcg2(const __grid_constant__ PcgArgs<T> A) {
  __shared__ double red[32];
  __shared__ double bc[4];
  if (*(volatile int*)A.gate) return;
  DevReport* rep = A.rep;
  const int U = A.U, B = gridDim.x;
  double* P[2] = {A.part, A.part + 3 * U};

  for (int u = blockIdx.x; u < U; u += B) p2_phase0<T>(A, P[0], u, red);
  grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
  for (int u = blockIdx.x; u < U; u += B) p2_zero_frame<T>(A, u);
  const double b2 = fold_partials(P[0], U, 0, bc);
  const double bmax = fold_partials(P[0] + U, U, 1, bc);
  const double divmax = fold_partials(P[0] + 2 * U, U, 1, bc);
  if (blockIdx.x == 0 && threadIdx.x == 0) report_max<T>(rep, SLOT_DIV_BEFORE, (T)divmax);
  if (*(volatile int*)A.gate == 3) {
    if (blockIdx.x == 0 && threadIdx.x == 0) rep->status = 3;
    return;
  }
  if (!isfinite(bmax)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { rep->status = 4; *A.gate = 4; }
    return;
  }
  if (b2 == 0.0) {
    for (int u = blockIdx.x; u < U; u += B) p2_finish_x<T>(A, u, (T)0, A.p0, true);
    if (blockIdx.x == 0 && threadIdx.x == 0) { rep->iterations = 0; rep->converged = 1; rep->criterion = 0.0; }
    return;
  }
  const double res_target = A.res_factor * bmax;
  const double tol = A.tol;
  auto phaseB = [&](double* part, bool use_ap, double alpha, const double* rin, double* rout, bool wr) {
    double acc = 0.0, rmax = 0.0;
    for (int u = blockIdx.x; u < U; u += B) p2_phaseB<T>(A, u, use_ap, alpha, rin, rout, wr, acc, rmax);
    const double s = block_sum(acc, red);
    __syncthreads();
    const double m = block_max(rmax, red);
    if (threadIdx.x == 0) { part[blockIdx.x] = s; part[U + blockIdx.x] = m; }
    __syncthreads();
  };
  auto phaseA = [&](double* part, bool first, T beta, bool upd, T alpha_prev, const T* pin, T* pout) {
    double acc = 0.0;
    for (int u = blockIdx.x; u < U; u += B) acc += p2_phaseA<T>(A, u, first, beta, upd, alpha_prev, pin, pout);
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    __syncthreads();
  };

  phaseB(P[1], false, 0.0, A.r0, A.r0, false);
  grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
  double rz = fold_partials(P[1], B, 0, bc);
  double rmax = fold_partials(P[1] + U, B, 1, bc);
  double crit = rz / b2;
  int it = 0, converged = 0, status = 0;
  bool finished = false;
  if (0.0 <= crit && crit < tol && rmax <= res_target) { converged = 1; finished = true; }
  else if (rz < 0.0) { finished = true; }
  if (A.probe_mode && !finished) {
    for (int q = 0; q < A.probe_iters; ++q) {
      if (A.probe_mode == 1) phaseA(P[0], false, (T)0.5, true, (T)0.0, (q & 1) ? A.p1 : A.p0, (q & 1) ? A.p0 : A.p1);
      if (A.probe_mode == 2) phaseB(P[1], true, 0.0, (q & 1) ? A.r1 : A.r0, (q & 1) ? A.r0 : A.r1, true);
      grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { rep->iterations = A.probe_iters; rep->converged = 1; }
    return;
  }
  const double* rc = A.r0;
  double* rn = A.r1;
  const T* pc = A.p1;
  T* pn = A.p0;
  double alpha = 0.0, beta = 0.0;
  while (!finished) {
    if (it >= A.max_iter) break;
    ++it;
    const bool first = it == 1;
    phaseA(P[0], first, (T)beta, !first, (T)alpha, pc, pn);
    grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
    const double pAp = fold_partials(P[0], B, 0, bc);
    { const T* tmp = pc; pc = pn; pn = const_cast<T*>(tmp); }
    if (*(volatile int*)A.gate == 3) { status = 3; alpha = 0.0; break; }
    if (pAp <= 0.0) { it -= 1; alpha = 0.0; break; }
    alpha = rz / pAp;
    phaseB(P[1], true, alpha, rc, rn, true);
    grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
    const double rz_new = fold_partials(P[1], B, 0, bc);
    rmax = fold_partials(P[1] + U, B, 1, bc);
    { const double* tmp = rc; rc = rn; rn = const_cast<double*>(tmp); }
    crit = rz_new / b2;
    if (*(volatile int*)A.gate == 3) { status = 3; break; }
    if (0.0 <= crit && crit < tol && rmax <= res_target) { converged = 1; break; }
    if (rz_new < 0.0) break;
    beta = rz_new / rz;
    rz = rz_new;
  }
  for (int u = blockIdx.x; u < U; u += B) p2_finish_x<T>(A, u, (T)alpha, pc, false);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rep->iterations = it;
    rep->converged = converged;
    rep->criterion = crit;
    if (status) rep->status = status;
    else if (!converged) { rep->status = 1; *A.gate = 1; }
  }
}

}  // namespace cw
