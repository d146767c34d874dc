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
// (d, 1/d, s) -- no CSR, no stored coefficients.
//
// PCG vectors live on the full grid with exact zeros at non-unknown cells,
// so stencils need no masks.  Each iteration is two grid phases separated
// by a grid barrier that also completes a deterministic fp64 reduction:
//   phase A: p' = z + beta p  (recomputed on the tile halo), x += alpha_prev p,
//            Ap = A p', partial p'.Ap
//   phase B: r' = r - alpha Ap (recomputed on the halo), z = W r',
//            partials r'.z and max|r'|
// (x's update is deferred by one phase so phase B streams 16 B/unknown and
// phase A 24 B/unknown in fp32.)  Partial sums are kept per work unit and
// every block folds them in the same fixed order, so all blocks agree
// bit-for-bit on alpha/beta and the result is run-to-run deterministic.
#pragma once
#include "cw_common.cuh"
#include "cw_step.cuh"

namespace cw {

template <typename T>
struct PcgArgs {
  Dims d;
  const uint8_t* code;
  T* x;                      // state p (in: warm start, out: solution; 0 off the unknowns)
  const T* u; const T* v; const T* w;
  T* r0; T* r1; T* p0; T* p1; T* z; T* Ap;
  double* part;              // [2][3][U] per-unit partials (two alternating sets)
  unsigned int* bar;         // [0] arrival count, [32] generation
  int* gate;
  DevReport* rep;
  const T* lut;              // [64][4] = d, 1/d, s, 0
  T wx, wy, wz, om;
  double dt, tol, res_factor;
  int max_iter;
  int precond;               // 0 identity, 1 jacobi (diag(1/d)), 2 AI1 (K^T K)
  int ntx, nty, zc, U;
  long long timeout_ns;
};

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

// Grid barrier for a cooperative launch (all blocks co-resident).  Times out
// (status 3) instead of hanging if the co-residency assumption is ever broken.
__device__ __forceinline__ void grid_barrier(unsigned* bar, int* gate, DevReport* rep,
                                             long long timeout_ns) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* count = bar;
    unsigned* gen = bar + 32;
    const unsigned g = ld_acquire(gen);
    __threadfence();
    const unsigned prev = atomicAdd(count, 1u);
    if (prev == gridDim.x - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      const unsigned long long t0 = globaltimer();
      unsigned spins = 0;
      while (ld_acquire(gen) == g) {
        __nanosleep(64);
        if ((++spins & 1023u) == 0 && (long long)(globaltimer() - t0) > timeout_ns) {
          rep->status = 3;
          *gate = 3;
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Fold U per-unit partials in a fixed order; every block computes the same
// bits.  mode 0: sum, 1: max.  Result broadcast to all threads.
__device__ __forceinline__ double fold_partials(const double* part, int U, int mode, double* sh) {
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int q = threadIdx.x; q < U; q += 32) {
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

template <typename T, int TX, int TY>
struct PcgSmem {
  T lut[64 * 4];
  T pa[3][TY + 2][TX + 2];
  T rb[2][TY + 2][TX + 2];
  T qb[2][TY + 2][TX + 2];
  uint8_t cb[2][TY + 2][TX + 2];
  T yb[2][TY + 1][TX + 1];
  double red[32];
  T redt[32];
  double bc[4];
};

struct Unit {
  int i0, j0, k0, k1;
};

template <typename T, int TX, int TY>
__device__ __forceinline__ Unit unit_of(const PcgArgs<T>& A, int u) {
  const int per = A.ntx * A.nty;
  const int tz = u / per, rem = u - tz * per;
  Unit t;
  t.i0 = (rem % A.ntx) * TX;
  t.j0 = (rem / A.ntx) * TY;
  t.k0 = tz * A.zc;
  t.k1 = min(t.k0 + A.zc, A.d.nz);
  return t;
}

// ---- phase 0: b = -div/dt, r0 = b - A x0 with x0 = p on the unknowns ------
template <typename T, int TX, int TY>
__device__ void phase0(const PcgArgs<T>& A, double* part, int unit, PcgSmem<T, TX, TY>& S) {
  const Dims& d = A.d;
  const Unit t = unit_of<T, TX, TY>(A, unit);
  const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
  const int i = t.i0 + lx, j = t.j0 + ly;
  const bool own = i < d.nx && j < d.ny;
  const long long plane = (long long)d.nx * d.ny;
  auto load = [&](int kk, int b) {
    for (int e = threadIdx.x; e < (TX + 2) * (TY + 2); e += TX * TY) {
      const int hx = e % (TX + 2), hy = e / (TX + 2);
      const int gi = t.i0 + hx - 1, gj = t.j0 + hy - 1;
      T val = (T)0;
      if (kk >= 0 && kk < d.nz && gi >= 0 && gi < d.nx && gj >= 0 && gj < d.ny) {
        const long long c = kk * plane + (long long)gj * d.nx + gi;
        if (A.code[c] & 64) val = __ldcg(A.x + c);
      }
      S.pa[b][hy][hx] = val;
    }
  };
  double b2 = 0.0, bmax = 0.0, dmax = 0.0;
  T pm = (T)0;
  if (own && t.k0 - 1 >= 0) {
    const long long c = (t.k0 - 1) * plane + (long long)j * d.nx + i;
    pm = (A.code[c] & 64) ? __ldcg(A.x + c) : (T)0;
  }
  int bc = 0, bn = 1;
  load(t.k0, bc);
  for (int k = t.k0; k < t.k1; ++k) {
    load(k + 1, bn);
    __syncthreads();
    if (own) {
      const long long c = k * plane + (long long)j * d.nx + i;
      const uint8_t cd = A.code[c];
      const T pc = S.pa[bc][ly + 1][lx + 1];
      const T pn = S.pa[bn][ly + 1][lx + 1];
      if (cd & 64) {
        const long long ui = ((long long)k * d.ny + j) * (d.nx + 1) + i;
        const long long vi = ((long long)k * (d.ny + 1) + j) * d.nx + i;
        T div = (A.u[ui + 1] - A.u[ui]) / (T)d.dx + (A.v[vi + d.nx] - A.v[vi]) / (T)d.dy;
        if (!d.is2d) div = div + (A.w[c + plane] - A.w[c]) / (T)d.dz;
        const T b = -div / (T)A.dt;
        const T ax = S.lut[(cd & 63) * 4] * pc -
                     (A.wx * (S.pa[bc][ly + 1][lx] + S.pa[bc][ly + 1][lx + 2]) +
                      A.wy * (S.pa[bc][ly][lx + 1] + S.pa[bc][ly + 2][lx + 1]) + A.wz * (pm + pn));
        A.r0[c] = b - ax;
        b2 += (double)b * (double)b;
        const double ab = fabs((double)b), ad = fabs((double)div);
        bmax = (ab > bmax || ab != ab) ? ab : bmax;
        dmax = (ad > dmax || ad != ad) ? ad : dmax;
      } else {
        A.x[c] = (T)0;
      }
      pm = pc;
    }
    // rotate: next plane becomes current; the old current buffer is free
    // once every thread has passed the barrier at the top of the next pass
    __syncthreads();
    const int tmp = bc; bc = bn; bn = tmp;
  }
  const double s0 = block_sum(b2, S.red);
  __syncthreads();
  const double m1 = block_max(bmax, S.red);
  __syncthreads();
  const double m2 = block_max(dmax, S.red);
  if (threadIdx.x == 0) {
    part[unit] = s0;
    part[A.U + unit] = m1;
    part[2 * A.U + unit] = m2;
  }
}

// ---- phase A: p' = z + beta p, x += alpha_prev p, Ap = A p' ---------------
template <typename T, int TX, int TY>
__device__ void phaseA(const PcgArgs<T>& A, double* part, int unit, PcgSmem<T, TX, TY>& S, bool first, T beta,
                       bool upd_x, T alpha_prev, const T* __restrict__ pin, T* __restrict__ pout) {
  const Dims& d = A.d;
  const Unit t = unit_of<T, TX, TY>(A, unit);
  const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
  const int i = t.i0 + lx, j = t.j0 + ly;
  const bool own = i < d.nx && j < d.ny;
  const long long plane = (long long)d.nx * d.ny;
  auto pnew = [&](long long c) -> T {
    const T zz = __ldcg(A.z + c);
    return first ? zz : zz + beta * __ldcg(pin + c);
  };
  auto load = [&](int kk, int b) {
    for (int e = threadIdx.x; e < (TX + 2) * (TY + 2); e += TX * TY) {
      const int hx = e % (TX + 2), hy = e / (TX + 2);
      const int gi = t.i0 + hx - 1, gj = t.j0 + hy - 1;
      T val = (T)0;
      if (kk >= 0 && kk < d.nz && gi >= 0 && gi < d.nx && gj >= 0 && gj < d.ny)
        val = pnew(kk * plane + (long long)gj * d.nx + gi);
      S.pa[b][hy][hx] = val;
    }
  };
  double acc = 0.0;
  T pm = (T)0;
  if (own && t.k0 - 1 >= 0) pm = pnew((t.k0 - 1) * plane + (long long)j * d.nx + i);
  int bc = 0, bn = 1;
  load(t.k0, bc);
  for (int k = t.k0; k < t.k1; ++k) {
    load(k + 1, bn);
    __syncthreads();
    if (own) {
      const long long c = k * plane + (long long)j * d.nx + i;
      const uint8_t cd = A.code[c];
      const T pc = S.pa[bc][ly + 1][lx + 1];
      const T pn = S.pa[bn][ly + 1][lx + 1];
      if (cd & 64) {
        const T ap = S.lut[(cd & 63) * 4] * pc -
                     (A.wx * (S.pa[bc][ly + 1][lx] + S.pa[bc][ly + 1][lx + 2]) +
                      A.wy * (S.pa[bc][ly][lx + 1] + S.pa[bc][ly + 2][lx + 1]) + A.wz * (pm + pn));
        pout[c] = pc;
        A.Ap[c] = ap;
        if (upd_x) A.x[c] += alpha_prev * __ldcg(pin + c);
        acc += (double)pc * (double)ap;
      }
      pm = pc;
    }
    __syncthreads();
    const int tmp = bc; bc = bn; bn = tmp;
  }
  const double s = block_sum(acc, S.red);
  if (threadIdx.x == 0) part[unit] = s;
}

// ---- phase B: r' = r - alpha Ap, z = W r' ----------------------------------
template <typename T, int TX, int TY>
__device__ void phaseB(const PcgArgs<T>& A, double* part, int unit, PcgSmem<T, TX, TY>& S, bool use_ap, T alpha,
                       const T* __restrict__ rin, T* __restrict__ rout) {
  const Dims& d = A.d;
  const Unit t = unit_of<T, TX, TY>(A, unit);
  const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
  const int i = t.i0 + lx, j = t.j0 + ly;
  const bool own = i < d.nx && j < d.ny;
  const long long plane = (long long)d.nx * d.ny;
  const T om = A.om;
  auto load = [&](int kk, int b) {
    for (int e = threadIdx.x; e < (TX + 2) * (TY + 2); e += TX * TY) {
      const int hx = e % (TX + 2), hy = e / (TX + 2);
      const int gi = t.i0 + hx - 1, gj = t.j0 + hy - 1;
      T rr = (T)0;
      uint8_t cd = 0;
      if (kk >= 0 && kk < d.nz && gi >= 0 && gi < d.nx && gj >= 0 && gj < d.ny) {
        const long long c = kk * plane + (long long)gj * d.nx + gi;
        cd = A.code[c];
        rr = __ldcg(rin + c);
        if (use_ap) rr = rr - alpha * __ldcg(A.Ap + c);
      }
      S.rb[b][hy][hx] = rr;
      S.qb[b][hy][hx] = rr * S.lut[(cd & 63) * 4 + 1];
      S.cb[b][hy][hx] = cd;
    }
  };
  double acc = 0.0, rmax = 0.0;
  T rprev = (T)0;
  for (int kk = t.k0 - 1; kk <= t.k1; ++kk) {
    const int b = kk & 1, bp = (kk - 1) & 1;
    load(kk, b);
    __syncthreads();
    const T rown = S.rb[b][ly + 1][lx + 1];
    if (kk >= t.k0) {
      for (int e = threadIdx.x; e < (TX + 1) * (TY + 1); e += TX * TY) {
        const int hx = e % (TX + 1), hy = e / (TX + 1);
        const uint8_t cd = S.cb[b][hy + 1][hx + 1];
        const T s = S.lut[(cd & 63) * 4 + 2];
        S.yb[b][hy][hx] = s * (S.rb[b][hy + 1][hx + 1] +
                               om * (A.wx * S.qb[b][hy + 1][hx] + A.wy * S.qb[b][hy][hx + 1] +
                                     A.wz * S.qb[bp][hy + 1][hx + 1]));
      }
    }
    __syncthreads();
    if (kk >= t.k0 + 1 && own) {
      const int k = kk - 1;
      const long long c = k * plane + (long long)j * d.nx + i;
      const uint8_t cd = S.cb[bp][ly + 1][lx + 1];
      if (cd & 64) {
        T zv;
        if (A.precond == 2)
          zv = S.yb[bp][ly][lx] + om * S.lut[(cd & 63) * 4 + 1] *
               (A.wx * S.yb[bp][ly][lx + 1] + A.wy * S.yb[bp][ly + 1][lx] + A.wz * S.yb[b][ly][lx]);
        else if (A.precond == 1)
          zv = S.qb[bp][ly + 1][lx + 1];
        else
          zv = rprev;
        A.z[c] = zv;
        if (use_ap) rout[c] = rprev;
        acc += (double)rprev * (double)zv;
        const double ar = fabs((double)rprev);
        rmax = (ar > rmax || ar != ar) ? ar : rmax;
      }
    }
    rprev = rown;
  }
  const double s = block_sum(acc, S.red);
  __syncthreads();
  const double m = block_max(rmax, S.red);
  if (threadIdx.x == 0) {
    part[unit] = s;
    part[A.U + unit] = m;
  }
}

template <typename T, int TX, int TY>
__device__ void x_update(const PcgArgs<T>& A, int unit, T alpha, const T* __restrict__ p) {
  const Dims& d = A.d;
  const Unit t = unit_of<T, TX, TY>(A, unit);
  const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
  const int i = t.i0 + lx, j = t.j0 + ly;
  if (i >= d.nx || j >= d.ny) return;
  const long long plane = (long long)d.nx * d.ny;
  for (int k = t.k0; k < t.k1; ++k) {
    const long long c = k * plane + (long long)j * d.nx + i;
    if (A.code[c] & 64) A.x[c] += alpha * __ldcg(p + c);
  }
}

template <typename T, int TX, int TY>
__device__ void x_zero(const PcgArgs<T>& A, int unit) {
  const Dims& d = A.d;
  const Unit t = unit_of<T, TX, TY>(A, unit);
  const int lx = threadIdx.x % TX, ly = threadIdx.x / TX;
  const int i = t.i0 + lx, j = t.j0 + ly;
  if (i >= d.nx || j >= d.ny) return;
  const long long plane = (long long)d.nx * d.ny;
  for (int k = t.k0; k < t.k1; ++k) A.x[k * plane + (long long)j * d.nx + i] = (T)0;
}

template <typename T, int TX, int TY>
__global__ void __launch_bounds__(TX * TY) k_pcg(PcgArgs<T> A) {
  __shared__ PcgSmem<T, TX, TY> S;
  if (*(volatile int*)A.gate) return;  // uniform across blocks: set before launch
  for (int e = threadIdx.x; e < 64 * 4; e += blockDim.x) S.lut[e] = A.lut[e];
  __syncthreads();
  DevReport* rep = A.rep;
  const int U = A.U;
  // two partial sets, alternated by phase, so one barrier per phase suffices
  double* P[2] = {A.part, A.part + 3 * U};

  for (int u = blockIdx.x; u < U; u += gridDim.x) phase0<T, TX, TY>(A, P[0], u, S);
  grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
  const double b2 = fold_partials(P[0], U, 0, S.bc);
  const double bmax = fold_partials(P[0] + U, U, 1, S.bc);
  const double divmax = fold_partials(P[0] + 2 * U, U, 1, S.bc);
  if (blockIdx.x == 0 && threadIdx.x == 0) report_max<T>(rep, SLOT_DIV_BEFORE, (T)divmax);
  if (*(volatile int*)A.gate == 3) { if (blockIdx.x == 0 && threadIdx.x == 0) rep->status = 3; return; }
  if (!isfinite(bmax)) {                     // pcg_solve raises on a non-finite rhs
    if (blockIdx.x == 0 && threadIdx.x == 0) { rep->status = 4; *A.gate = 4; }
    return;
  }
  if (b2 == 0.0) {                           // linalg.py:329-330: x = 0, 0 iterations
    for (int u = blockIdx.x; u < U; u += gridDim.x) x_zero<T, TX, TY>(A, u);
    if (blockIdx.x == 0 && threadIdx.x == 0) { rep->iterations = 0; rep->converged = 1; rep->criterion = 0.0; }
    return;
  }
  const double res_target = A.res_factor * bmax;   // solver.py:266 (b.any() holds: b2 > 0)
  const double tol = A.tol;

  // z = W r0, rz, max|r0|  (pcg_solve:342-345)
  for (int u = blockIdx.x; u < U; u += gridDim.x)
    phaseB<T, TX, TY>(A, P[1], u, S, false, (T)0, A.r0, A.r0);
  grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
  double rz = fold_partials(P[1], U, 0, S.bc);
  double rmax = fold_partials(P[1] + U, U, 1, S.bc);
  double crit = rz / b2;
  int it = 0, converged = 0, status = 0;
  bool finished = false;
  if (0.0 <= crit && crit < tol && rmax <= res_target) { converged = 1; finished = true; }
  else if (rz < 0.0) { finished = true; }
  T* rc = A.r0; T* rn = A.r1;
  T* pc = A.p1; T* pn = A.p0;     // pc: previous direction (unused on the first pass)
  double alpha = 0.0, beta = 0.0;
  while (!finished) {
    if (it >= A.max_iter) break;
    ++it;
    const bool first = it == 1;
    for (int u = blockIdx.x; u < U; u += gridDim.x)
      phaseA<T, TX, TY>(A, P[0], u, S, first, (T)beta, !first, (T)alpha, pc, pn);
    grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
    const double pAp = fold_partials(P[0], U, 0, S.bc);
    { T* tmp = pc; pc = pn; pn = tmp; }      // pc now holds this iteration's p
    if (*(volatile int*)A.gate == 3) { status = 3; alpha = 0.0; break; }
    if (pAp <= 0.0) { it -= 1; alpha = 0.0; break; }   // linalg.py:354-355
    alpha = rz / pAp;
    for (int u = blockIdx.x; u < U; u += gridDim.x)
      phaseB<T, TX, TY>(A, P[1], u, S, true, (T)alpha, rc, rn);
    grid_barrier(A.bar, A.gate, rep, A.timeout_ns);
    const double rz_new = fold_partials(P[1], U, 0, S.bc);
    rmax = fold_partials(P[1] + U, U, 1, S.bc);
    { T* tmp = rc; rc = rn; rn = tmp; }
    crit = rz_new / b2;
    if (*(volatile int*)A.gate == 3) { status = 3; break; }
    if (0.0 <= crit && crit < tol && rmax <= res_target) { converged = 1; break; }
    if (rz_new < 0.0) break;                  // linalg.py:364-365
    beta = rz_new / rz;
    rz = rz_new;
  }
  // x += alpha p of the last completed iteration is still pending
  if (alpha != 0.0)
    for (int u = blockIdx.x; u < U; u += gridDim.x) x_update<T, TX, TY>(A, u, (T)alpha, pc);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rep->iterations = it;
    rep->converged = converged;
    rep->criterion = crit;
    if (status) rep->status = status;
    else if (!converged) { rep->status = 1; *A.gate = 1; }
  }
}

}  // namespace cw
