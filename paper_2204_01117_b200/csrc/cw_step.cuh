// Per-stage kernels of one RANS step (everything except the pressure solve).
// Each kernel restates one reference stage on the x-fastest device layout;
// the reference file:line each one follows is given at the kernel.
#pragma once
#include "cw_common.cuh"

namespace cw {

struct StepConsts {
  double dt, nu, cap_diffuse, cap_turb;   // cap_diffuse: solver.py:195-201; cap_turb: turbulence.py:110
  double c_mu, alpha, beta, sigma, sigma_star, c_lim;
  double k_in, om_in, nut_in;             // inlet turbulence (turbulence.py:26-33)
  double lim_scale;                       // c_lim / (c_mu / 2), the limiter's factor (turbulence.py:93-97)
};

// Per-step device report (one slot per step in a batch).
struct DevReport {
  int iterations;
  int converged;
  int status;            // 0 ok, 1 pcg not converged, 2 non-finite turbulence, 3 barrier timeout, 4 non-finite rhs,
                         // 5 z-slab halo too shallow for this step's reach
  int halo_need;         // status 5: planes the window needs per interior face (criterion = max|w| dt/dz)
  double criterion;
  unsigned int fmax[4];  // float max slots: 0 div_before, 1 div_after, 2 max|vel| (bit patterns)
  unsigned long long dmax[4];
  long long bad_index[2];  // first non-finite k / omega cell, reference C order (i*ny+j)*nz+k
};

enum MaxSlot { SLOT_DIV_BEFORE = 0, SLOT_DIV_AFTER = 1, SLOT_SPEED = 2, SLOT_WMAX = 3 };

template <typename T> __device__ __forceinline__ void report_max(DevReport* r, int slot, T v);
template <> __device__ __forceinline__ void report_max<float>(DevReport* r, int slot, float v) {
  atomicMax(&r->fmax[slot], __float_as_uint(v));
}
template <> __device__ __forceinline__ void report_max<double>(DevReport* r, int slot, double v) {
  atomicMax(&r->dmax[slot], (unsigned long long)__double_as_longlong(v));
}

#define CW_GRID_STRIDE(idx, n) \
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (n); \
       idx += (long long)gridDim.x * blockDim.x)

// Stage kernels run on a 3-D grid: blockDim (32, 8), grid (ceil(ex/32),
// ceil(ey/8), ez) -- the element's (i, j, k) come from the launch, no
// per-element 64-bit division.
#ifndef CW_ST_BY
#define CW_ST_BY 8
#endif
#ifndef CW_ST_BZ
#define CW_ST_BZ 1
#endif
// blocks span ST_BZ planes so that z-neighbour reads hit the block's own L1
constexpr int ST_BX = 32, ST_BY = CW_ST_BY, ST_BZ = CW_ST_BZ;
#define CW_IJK(ex, ey, ez, inb)                                  \
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x);         \
  const int j = (int)(blockIdx.y * ST_BY + threadIdx.y);         \
  const int k = (int)(blockIdx.z * ST_BZ + threadIdx.z);         \
  const bool inb = i < (ex) && j < (ey) && k < (ez)
// z-coarsened stage kernels (diffuse, drag, gradient, turbulence): a thread
// handles CW_ZT consecutive planes, so loads of several planes are in flight
// per thread; grid (ceil(ex/32), ceil(ey/ST_BY), ceil(ez/CW_ZT)), ST_BZ = 1.
#ifndef CW_ZT
#define CW_ZT 4
#endif
static_assert(ST_BZ == 1, "z-coarsened kernels take one plane per block row");
#ifndef CW_ZT_TURB
#define CW_ZT_TURB 1
#endif
constexpr int ZT_TURB = CW_ZT_TURB;   // k_turbulence planes per thread (2 and 4 measured slower: 90 -> 98 / 100 us at C3)
#ifndef CW_ZT_MAC
#define CW_ZT_MAC 2
#endif
constexpr int ZT_MAC = CW_ZT_MAC;   // MacCormack predictor / corrector

__device__ __forceinline__ int clampi(int a, int lo, int hi) { return a < lo ? lo : (a > hi ? hi : a); }

// ---------------------------------------------------------------------------
// upwind k and omega (advection.py:154-173), old velocity, axes x,y,z in turn
// the upwind update of cell (i, j, k) given its cell-centred velocity a
template <typename T>
__device__ __forceinline__ void upwind_cell_a(const Dims& d, const T (&a)[3], const T* __restrict__ kin,
                                              const T* __restrict__ win, T* __restrict__ kout, T* __restrict__ wout,
                                              T dt, int i, int j, int k) {
  {
    const int c = d.cidx32(i, j, k);
    const int pos[3] = {i, j, k};
    const int ext[3] = {d.nx, d.ny, d.nz};
    const int str[3] = {1, d.nx, (int)d.nx * d.ny};
    const T rh[3] = {inv_h<T>(d, 0), inv_h<T>(d, 1), inv_h<T>(d, 2)};
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const T* fld = f ? win : kin;
      const T fc = fld[c];
      T out = fc;
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (ext[ax] == 1) continue;
        const T bwd = pos[ax] > 0 ? (fc - fld[c - str[ax]]) * rh[ax] : (T)0;
        const T fwd = pos[ax] < ext[ax] - 1 ? (fld[c + str[ax]] - fc) * rh[ax] : (T)0;
        const T ap = a[ax] > (T)0 ? a[ax] : (T)0;
        const T am = a[ax] < (T)0 ? a[ax] : (T)0;
        out -= dt * (ap * bwd + am * fwd);
      }
      (f ? wout : kout)[c] = out;
    }
  }
}

// cell-centred velocity of cell (i, j, k) (grid.py:561-566)
template <typename T>
__device__ __forceinline__ void cell_vel_a(const Dims& d, const T* __restrict__ u, const T* __restrict__ v,
                                           const T* __restrict__ w, int i, int j, int k, T (&a)[3]) {
  const int c = d.cidx32(i, j, k);
  a[0] = (T)0.5 * (u[((int)k * d.ny + j) * (d.nx + 1) + i] + u[((int)k * d.ny + j) * (d.nx + 1) + i + 1]);
  a[1] = (T)0.5 * (v[((int)k * (d.ny + 1) + j) * d.nx + i] + v[((int)k * (d.ny + 1) + j + 1) * d.nx + i]);
  a[2] = (T)0.5 * (w[c] + w[c + (int)d.nx * d.ny]);
}

template <typename T>
__device__ __forceinline__ void upwind_cell(const Dims& d, const T* __restrict__ u, const T* __restrict__ v,
                                            const T* __restrict__ w, const T* __restrict__ kin,
                                            const T* __restrict__ win, T* __restrict__ kout, T* __restrict__ wout,
                                            T dt, int i, int j, int k) {
  if (i < d.nx && j < d.ny && k < d.nz) {
    T a[3];
    cell_vel_a<T>(d, u, v, w, i, j, k, a);
    upwind_cell_a<T>(d, a, kin, win, kout, wout, dt, i, j, k);
  }
}

// the upwind step from a saved cell-centred velocity (cw_step_defer_kw)
// gate_pass: device statuses (bit s) the launch runs through -- the
// deferred k / omega part runs after a failed projection too, so the state
// ends as the reference leaves it when project() raises (advected k, omega)
__device__ __forceinline__ bool gated(const int* gate, unsigned gate_pass) {
  const int g = *gate;
  return g != 0 && !((gate_pass >> (g & 31)) & 1u);
}

template <typename T>
__global__ void k_upwind_saved(Dims d, const T* __restrict__ acell, const T* __restrict__ kin,
                               const T* __restrict__ win, T* __restrict__ kout, T* __restrict__ wout, T dt,
                               const int* gate, unsigned gate_pass = 0) {
  if (gated(gate, gate_pass)) return;
  CW_IJK(d.nx, d.ny, d.nz, inb);
  if (!inb) return;
  const long long ncell = (long long)d.nx * d.ny * d.nz;
  const int c = d.cidx32(i, j, k);
  const T a[3] = {acell[c], acell[ncell + c], acell[2 * ncell + c]};
  upwind_cell_a<T>(d, a, kin, win, kout, wout, dt, i, j, k);
}

// ---------------------------------------------------------------------------
// MacCormack predictor / corrector (advection.py:125-142)
__device__ __forceinline__ void comp_offset(int comp, float& ox, float& oy, float& oz) {
  ox = comp == 0 ? 0.f : 0.5f;
  oy = comp == 1 ? 0.f : 0.5f;
  oz = comp == 2 ? 0.f : 0.5f;
}

// Velocity of the pre-advection field at the face point of component `comp`
// with integer index (i, j, k) (advection.py:16-21, 49-101).  The point sits at
// fixed half-cell offsets from every velocity grid, so the trilinear weights are
// 0, 1/2 or 1: a weight-1/2 pair is an exact average, and at the domain edge the
// clamped pair averages a value with itself (exact).  This equals the general
// trilinear gather bit for bit (x, then y, then z, as gather_at) with 9 loads
// and straight-line index arithmetic.
template <typename T>
__device__ __forceinline__ T avg2(T a, T b) { return a * (T)0.5 + b * (T)0.5; }

template <typename T>
__device__ __forceinline__ void face_velocity(const Dims& d, int comp, const T* __restrict__ u,
                                              const T* __restrict__ v, const T* __restrict__ w, int i, int j, int k,
                                              T& us, T& vs, T& ws) {
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int uy = nx + 1, uz = (nx + 1) * ny;     // u strides
  const int vy = nx, vz = nx * (ny + 1);         // v strides
  const int wy = nx, wz = nx * ny;               // w strides
  if (comp == 0) {           // u face: i in 0..nx, j < ny, k < nz
    const int im = max(i - 1, 0), ip = min(i, nx - 1);
    us = u[k * uz + j * uy + i];
    const T* vr = v + k * vz + j * vy;           // rows j, j+1 of v on plane k
    vs = avg2(avg2(vr[im], vr[ip]), avg2(vr[vy + im], vr[vy + ip]));
    const T* wr = w + k * wz + j * wy;           // planes k, k+1 of w on row j
    ws = avg2(avg2(wr[im], wr[ip]), avg2(wr[wz + im], wr[wz + ip]));
  } else if (comp == 1) {    // v face: i < nx, j in 0..ny, k < nz
    const int jm = max(j - 1, 0), jp = min(j, ny - 1);
    vs = v[k * vz + j * vy + i];
    const T* ur = u + k * uz + i;
    us = avg2(avg2(ur[jm * uy], ur[jm * uy + 1]), avg2(ur[jp * uy], ur[jp * uy + 1]));
    const T* wr = w + k * wz + i;
    ws = avg2(avg2(wr[jm * wy], wr[jp * wy]), avg2(wr[wz + jm * wy], wr[wz + jp * wy]));
  } else {                   // w face: i < nx, j < ny, k in 0..nz
    const int km = max(k - 1, 0), kp = min(k, nz - 1);
    ws = w[k * wz + j * wy + i];
    const T* ur = u + j * uy + i;
    us = avg2(avg2(ur[km * uz], ur[km * uz + 1]), avg2(ur[kp * uz], ur[kp * uz + 1]));
    const T* vr = v + j * vy + i;
    vs = avg2(avg2(vr[km * vz], vr[km * vz + vy]), avg2(vr[kp * vz], vr[kp * vz + vy]));
  }
}

// The velocities of a thread whose (i, j, k) is inside all three face extents
// and the cell grid (3-D): the u, v and w face points and the cell centre need
// 6 distinct values of each velocity array (18 loads, against 39 when
// face_velocity runs per component and the upwind step loads its own);
// every average is the same expression on the same values, bit for bit.
template <typename T>
struct VelNbhd {
  T fu[3], fv[3], fw[3];   // velocity (u, v, w) at the face point of component c
  T a[3];                  // cell-centred velocity (upwind step)
};

template <typename T>
__device__ __forceinline__ void vel_nbhd(const Dims& d, const T* __restrict__ u, const T* __restrict__ v,
                                         const T* __restrict__ w, int i, int j, int k, VelNbhd<T>& n) {
  const int nx = d.nx, ny = d.ny;
  const int uy = nx + 1, uz = (nx + 1) * ny;
  const int vy = nx, vz = nx * (ny + 1);
  const int wy = nx, wz = nx * ny;
  const int im = max(i - 1, 0), jm = max(j - 1, 0), km = max(k - 1, 0);
  const T* ur = u + k * uz + j * uy + i;
  const T U0 = ur[0], U1 = ur[1];                                   // u(i..i+1, j, k)
  const T U2 = u[k * uz + jm * uy + i], U3 = u[k * uz + jm * uy + i + 1];   // u(i..i+1, jm, k)
  const T U4 = u[km * uz + j * uy + i], U5 = u[km * uz + j * uy + i + 1];   // u(i..i+1, j, km)
  const T V0 = v[k * vz + j * vy + i], V1 = v[k * vz + (j + 1) * vy + i];   // v(i, j..j+1, k)
  const T V2 = v[k * vz + j * vy + im], V3 = v[k * vz + (j + 1) * vy + im]; // v(im, j..j+1, k)
  const T V4 = v[km * vz + j * vy + i], V5 = v[km * vz + (j + 1) * vy + i]; // v(i, j..j+1, km)
  const T W0 = w[k * wz + j * wy + i], W1 = w[(k + 1) * wz + j * wy + i];   // w(i, j, k..k+1)
  const T W2 = w[k * wz + j * wy + im], W3 = w[(k + 1) * wz + j * wy + im]; // w(im, j, k..k+1)
  const T W4 = w[k * wz + jm * wy + i], W5 = w[(k + 1) * wz + jm * wy + i]; // w(i, jm, k..k+1)
  // u face (face_velocity comp 0: ip = i)
  n.fu[0] = U0;
  n.fv[0] = avg2(avg2(V2, V0), avg2(V3, V1));
  n.fw[0] = avg2(avg2(W2, W0), avg2(W3, W1));
  // v face (comp 1: jp = j)
  n.fu[1] = avg2(avg2(U2, U3), avg2(U0, U1));
  n.fv[1] = V0;
  n.fw[1] = avg2(avg2(W4, W0), avg2(W5, W1));
  // w face (comp 2: kp = k)
  n.fu[2] = avg2(avg2(U4, U5), avg2(U0, U1));
  n.fv[2] = avg2(avg2(V4, V5), avg2(V0, V1));
  n.fw[2] = W0;
  // cell centre (upwind_cell)
  n.a[0] = (T)0.5 * (U0 + U1);
  n.a[1] = (T)0.5 * (V0 + V1);
  n.a[2] = (T)0.5 * (W0 + W1);
}

// The clip range of each face: the predictor's gather already visits the 8
// corners whose min / max the corrector clips to (advection.py:130-134 takes
// `ahead, mn, mx` from that one sample), so it stores them (CW_MAC_CLIP=1) and
// the corrector reads two values instead of gathering the same corners again.
#ifndef CW_MAC_CLIP
#define CW_MAC_CLIP 1
#endif
template <typename T>
struct MacClip {
  T* mn[3];
  T* mx[3];
};

// the predictor for one face given the face-point velocity
template <typename T>
__device__ __forceinline__ void mac_predict_face_v(const Dims& d, int comp, const T* arr, T* ahead, T dt, int i,
                                                   int j, int k, T us, T vs, T ws, const MacClip<T>& clip) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  float fox, foy, foz;
  comp_offset(comp, fox, foy, foz);
  const T ox = (T)fox, oy = (T)foy, oz = (T)foz;
  const int c = ((int)k * ey + j) * ex + i;
  const T X = (T)i + ox, Y = (T)j + oy, Z = (T)(k + d.kg0) + oz;   // global z (z-slab windows)
#if CW_MAC_CLIP
  // the corrector's expressions for the trace (X - s with s rounded on its own)
  const T sx = dt * us * inv_h<T>(d, 0), sy = dt * vs * inv_h<T>(d, 1), sz = dt * ws * inv_h<T>(d, 2);
  const T bx = X - sx, by = Y - sy, bz = Z - sz;
  T mn, mx;
  ahead[c] = gather<T>(arr, ex, ey, ez, bx - ox, by - oy, bz - oz, &mn, &mx, d.kg0);
  clip.mn[comp][c] = mn;
  clip.mx[comp][c] = mx;
#else
  const T bx = X - dt * us * inv_h<T>(d, 0), by = Y - dt * vs * inv_h<T>(d, 1), bz = Z - dt * ws * inv_h<T>(d, 2);
  ahead[c] = gather<T>(arr, ex, ey, ez, bx - ox, by - oy, bz - oz, nullptr, nullptr, d.kg0);
#endif
}

// One thread per (i, j, k) of the union of the face extents handles the u, v
// and w faces there (all three read the same pre-advection velocity).
template <typename T>
__device__ __forceinline__ void mac_predict_face(const Dims& d, int comp, const T* u, const T* v, const T* w,
                                                 T* ahead, T dt, int i, int j, int k, const MacClip<T>& clip) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  if (i >= ex || j >= ey || k >= ez) return;
  const T* arr = comp == 0 ? u : (comp == 1 ? v : w);
  T us, vs, ws;
  face_velocity<T>(d, comp, u, v, w, i, j, k, us, vs, ws);
  mac_predict_face_v<T>(d, comp, arr, ahead, dt, i, j, k, us, vs, ws, clip);
}

// the predictor launch also runs the upwind step of k and omega (cells,
// advection.py:154-173) when kout != nullptr: both read the old velocity
#ifndef CW_MAC_PRED_MINB
#define CW_MAC_PRED_MINB 8
#endif
// 8 resident blocks per SM (<= 32 registers): measured 102 us at C3, against
// 106 us at 6 blocks and 223 us uncapped
// SAVE_A (cw_step_defer_kw): instead of the upwind step, store the cell-centred
// old velocity (the upwind step's input) in acell[0..2]; k_upwind_saved runs
// the upwind step from it later
template <typename T, bool SAVE_A = false>
__global__ void __launch_bounds__(256, CW_MAC_PRED_MINB) k_mac_predict(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                              const T* __restrict__ w, T* __restrict__ a0, T* __restrict__ a1,
                              T* __restrict__ a2, T dt, const T* __restrict__ kin, const T* __restrict__ win,
                              T* __restrict__ kout, T* __restrict__ wout, MacClip<T> clip, const int* gate,
                              T* __restrict__ acell = nullptr) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i > d.nx || j > d.ny) return;
  const long long ncell = (long long)d.nx * d.ny * d.nz;
#pragma unroll
  for (int kz = 0; kz < ZT_MAC; ++kz) {
    const int k = (int)blockIdx.z * ZT_MAC + kz;
    if (k > d.nz) break;
    if (!d.is2d && i < d.nx && j < d.ny && k < d.nz) {   // interior: shared velocity loads
      VelNbhd<T> n;
      vel_nbhd<T>(d, u, v, w, i, j, k, n);
      if (SAVE_A) {
        const int c = d.cidx32(i, j, k);
        acell[c] = n.a[0];
        acell[ncell + c] = n.a[1];
        acell[2 * ncell + c] = n.a[2];
      } else if (kout) {
        upwind_cell_a<T>(d, n.a, kin, win, kout, wout, dt, i, j, k);
      }
      mac_predict_face_v<T>(d, 0, u, a0, dt, i, j, k, n.fu[0], n.fv[0], n.fw[0], clip);
      mac_predict_face_v<T>(d, 1, v, a1, dt, i, j, k, n.fu[1], n.fv[1], n.fw[1], clip);
      mac_predict_face_v<T>(d, 2, w, a2, dt, i, j, k, n.fu[2], n.fv[2], n.fw[2], clip);
      continue;
    }
    if (SAVE_A) {
      if (i < d.nx && j < d.ny && k < d.nz) {
        T a[3];
        cell_vel_a<T>(d, u, v, w, i, j, k, a);
        const int c = d.cidx32(i, j, k);
        acell[c] = a[0];
        acell[ncell + c] = a[1];
        acell[2 * ncell + c] = a[2];
      }
    } else if (kout) {
      upwind_cell<T>(d, u, v, w, kin, win, kout, wout, dt, i, j, k);
    }
    mac_predict_face<T>(d, 0, u, v, w, a0, dt, i, j, k, clip);
    mac_predict_face<T>(d, 1, u, v, w, a1, dt, i, j, k, clip);
    if (!d.is2d) mac_predict_face<T>(d, 2, u, v, w, a2, dt, i, j, k, clip);
  }
}

// the corrector for one face given the face-point velocity
template <typename T>
__device__ __forceinline__ void mac_correct_face_v(const Dims& d, int comp, const T* arr, const T* ahead, T* out,
                                                   T dt, int i, int j, int k, T us, T vs, T ws, T self,
                                                   const MacClip<T>& clip) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  float fox, foy, foz;
  comp_offset(comp, fox, foy, foz);
  const T ox = (T)fox, oy = (T)foy, oz = (T)foz;
  const int c = ((int)k * ey + j) * ex + i;
  const T X = (T)i + ox, Y = (T)j + oy, Z = (T)(k + d.kg0) + oz;   // global z (z-slab windows)
  T mn, mx;
  const T sx = dt * us * inv_h<T>(d, 0), sy = dt * vs * inv_h<T>(d, 1), sz = dt * ws * inv_h<T>(d, 2);
#if CW_MAC_CLIP
  mn = clip.mn[comp][c];
  mx = clip.mx[comp][c];
  (void)arr;
#else
  const T bx = X - sx, by = Y - sy, bz = Z - sz;
  (void)gather<T>(arr, ex, ey, ez, bx - ox, by - oy, bz - oz, &mn, &mx, d.kg0);
#endif
  const T fx = X + sx, fy = Y + sy, fz = Z + sz;
  const T back = gather<T>(ahead, ex, ey, ez, fx - ox, fy - oy, fz - oz, nullptr, nullptr, d.kg0);
  T cor = ahead[c] + (T)0.5 * (self - back);   // self = arr[c]
  cor = cor < mn ? mn : cor;
  cor = cor > mx ? mx : cor;
  out[c] = cor;
}

template <typename T>
__device__ __forceinline__ void mac_correct_face(const Dims& d, int comp, const T* u, const T* v, const T* w,
                                                 const T* ahead, T* out, T dt, int i, int j, int k,
                                                 const MacClip<T>& clip) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  if (i >= ex || j >= ey || k >= ez) return;
  const T* arr = comp == 0 ? u : (comp == 1 ? v : w);
  T us, vs, ws;
  face_velocity<T>(d, comp, u, v, w, i, j, k, us, vs, ws);
  mac_correct_face_v<T>(d, comp, arr, ahead, out, dt, i, j, k, us, vs, ws, arr[((int)k * ey + j) * ex + i], clip);
}

#ifndef CW_MAC_CORR_MINB
#define CW_MAC_CORR_MINB 5
#endif
// 5 resident blocks per SM (<= 51 registers): the gathers are latency-bound,
// occupancy beats the few reloads the register cap costs (141 us uncapped at
// 72 registers, 108 us at 5 or 6 blocks)
template <typename T>
__global__ void __launch_bounds__(256, CW_MAC_CORR_MINB) k_mac_correct(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                              const T* __restrict__ w, const T* __restrict__ a0, const T* __restrict__ a1,
                              const T* __restrict__ a2, T* __restrict__ o0, T* __restrict__ o1,
                              T* __restrict__ o2, T dt, MacClip<T> clip, const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i > d.nx || j > d.ny) return;
#pragma unroll
  for (int kz = 0; kz < ZT_MAC; ++kz) {
    const int k = (int)blockIdx.z * ZT_MAC + kz;
    if (k > d.nz) break;
    if (!d.is2d && i < d.nx && j < d.ny && k < d.nz) {   // interior: shared velocity loads
      VelNbhd<T> n;
      vel_nbhd<T>(d, u, v, w, i, j, k, n);
      mac_correct_face_v<T>(d, 0, u, a0, o0, dt, i, j, k, n.fu[0], n.fv[0], n.fw[0], n.fu[0], clip);
      mac_correct_face_v<T>(d, 1, v, a1, o1, dt, i, j, k, n.fu[1], n.fv[1], n.fw[1], n.fv[1], clip);
      mac_correct_face_v<T>(d, 2, w, a2, o2, dt, i, j, k, n.fu[2], n.fv[2], n.fw[2], n.fw[2], clip);
      continue;
    }
    mac_correct_face<T>(d, 0, u, v, w, a0, o0, dt, i, j, k, clip);
    mac_correct_face<T>(d, 1, u, v, w, a1, o1, dt, i, j, k, clip);
    if (!d.is2d) mac_correct_face<T>(d, 2, u, v, w, a2, o2, dt, i, j, k, clip);
  }
}

// ---------------------------------------------------------------------------
// explicit diffusion with the capped eddy viscosity (solver.py:175-208)
template <typename T>
__device__ __forceinline__ T nu_eff(const T* nut, int c, T nu, T cap) {
  T t = nut[c];
  t = t < (T)0 ? (T)0 : t;
  t = t > cap ? cap : t;
  return nu + t;
}

template <typename T>
__device__ __forceinline__ void diffuse_face(const Dims& d, int comp, const T* __restrict__ src,
                                             T* __restrict__ dst, const T* __restrict__ nut, T dt, T nu, T cap,
                                             int i, int j, int k) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  const int ext[3] = {ex, ey, ez};
  const int str[3] = {1, ex, (int)ex * ey};
  const T rh2[3] = {inv_h2<T>(d, 0), inv_h2<T>(d, 1), inv_h2<T>(d, 2)};
  if (i < ex && j < ey && k < ez) {
    const int c = ((int)k * ey + j) * ex + i;
    const int pos[3] = {i, j, k};
    const T mid = src[c];
    T lap = (T)0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (ext[ax] == 1 || (d.is2d && ax == 2)) continue;
      const T lo = pos[ax] > 0 ? src[c - str[ax]] : mid;
      const T hi = pos[ax] < ext[ax] - 1 ? src[c + str[ax]] : mid;
      lap += (lo - (T)2 * mid + hi) * rh2[ax];
    }
    // face viscosity along the component's own axis, edge faces copy the cell
    int ci[3] = {pos[0], pos[1], pos[2]};
    const int nc = comp == 0 ? d.nx : (comp == 1 ? d.ny : d.nz);
    const int f = pos[comp];
    ci[comp] = clampi(f - 1, 0, nc - 1);
    const T a = nu_eff(nut, d.cidx32(ci[0], ci[1], ci[2]), nu, cap);
    ci[comp] = clampi(f, 0, nc - 1);
    const T b = nu_eff(nut, d.cidx32(ci[0], ci[1], ci[2]), nu, cap);
    dst[c] = mid + dt * ((T)0.5 * (a + b)) * lap;
  }
}

// all components in one launch over the union of the face extents
template <typename T>
__global__ void k_diffuse(Dims d, const T* __restrict__ s0, const T* __restrict__ s1, const T* __restrict__ s2,
                          T* __restrict__ d0, T* __restrict__ d1, T* __restrict__ d2, const T* __restrict__ nut,
                          T dt, T nu, T cap, const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i > d.nx || j > d.ny) return;
#pragma unroll
  for (int kz = 0; kz < CW_ZT; ++kz) {
    const int k = (int)blockIdx.z * CW_ZT + kz;
    if (k > d.nz) break;
    diffuse_face<T>(d, 0, s0, d0, nut, dt, nu, cap, i, j, k);
    diffuse_face<T>(d, 1, s1, d1, nut, dt, nu, cap, i, j, k);
    if (!d.is2d) diffuse_face<T>(d, 2, s2, d2, nut, dt, nu, cap, i, j, k);
  }
}

// The same diffusion with straight-line access: the edge-replicated
// neighbours are clamped indices (a clamped neighbour is the face itself:
// (mid - 2 mid) + hi == hi - mid exactly, as the generic per-axis loop
// computes), the three components of one (i, j, k) share the capped cell
// viscosities they read (cells (i,j,k), (i-1,j,k), (i,j-1,k), (i,j,k-1)).
// Same arithmetic as diffuse_face, axis sums in x, y, z order.
template <typename T>
__device__ __forceinline__ T lap_face(const T* __restrict__ a, int c, T mid, int sxm, int sxp, int sym, int syp,
                                      int szm, int szp, T r20, T r21, T r22, bool hx, bool hy, bool hz) {
  T lap = (T)0;
  if (hx) lap += (a[c - sxm] - (T)2 * mid + a[c + sxp]) * r20;
  if (hy) lap += (a[c - sym] - (T)2 * mid + a[c + syp]) * r21;
  if (hz) lap += (a[c - szm] - (T)2 * mid + a[c + szp]) * r22;
  return lap;
}

template <typename T>
__global__ void k_diffuse_c(Dims d, const T* __restrict__ s0, const T* __restrict__ s1, const T* __restrict__ s2,
                            T* __restrict__ d0, T* __restrict__ d1, T* __restrict__ d2, const T* __restrict__ nut,
                            T dt, T nu, T cap, const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  if (i > nx || j > ny) return;
  const T r20 = inv_h2<T>(d, 0), r21 = inv_h2<T>(d, 1), r22 = inv_h2<T>(d, 2);
  const bool z3 = !d.is2d;
#pragma unroll
  for (int kz = 0; kz < CW_ZT; ++kz) {
    const int k = (int)blockIdx.z * CW_ZT + kz;
    if (k > nz) break;
    // capped viscosities of the cells around (i, j, k), clamped to the grid
    const int ci = min(i, nx - 1), cj = min(j, ny - 1), ck = min(k, nz - 1);
    const T n0 = nu_eff(nut, d.cidx32(ci, cj, ck), nu, cap);
    if (i < nx + 1 && j < ny && k < nz) {           // u face (nx+1, ny, nz)
      const int ex = nx + 1, ey = ny;
      const int c = (k * ey + j) * ex + i;
      const T mid = s0[c];
      const T lap = lap_face<T>(s0, c, mid, i > 0 ? 1 : 0, i < ex - 1 ? 1 : 0, j > 0 ? ex : 0, j < ey - 1 ? ex : 0,
                                k > 0 ? ex * ey : 0, k < nz - 1 ? ex * ey : 0, r20, r21, r22, ex > 1, ey > 1,
                                z3 && nz > 1);
      const T a = nu_eff(nut, d.cidx32(max(i - 1, 0), j, k), nu, cap);
      const T b = i < nx ? n0 : nu_eff(nut, d.cidx32(nx - 1, j, k), nu, cap);
      d0[c] = mid + dt * ((T)0.5 * (a + b)) * lap;
    }
    if (i < nx && j < ny + 1 && k < nz) {           // v face (nx, ny+1, nz)
      const int ex = nx, ey = ny + 1;
      const int c = (k * ey + j) * ex + i;
      const T mid = s1[c];
      const T lap = lap_face<T>(s1, c, mid, i > 0 ? 1 : 0, i < ex - 1 ? 1 : 0, j > 0 ? ex : 0, j < ey - 1 ? ex : 0,
                                k > 0 ? ex * ey : 0, k < nz - 1 ? ex * ey : 0, r20, r21, r22, ex > 1, ey > 1,
                                z3 && nz > 1);
      const T a = nu_eff(nut, d.cidx32(i, max(j - 1, 0), k), nu, cap);
      const T b = j < ny ? n0 : nu_eff(nut, d.cidx32(i, ny - 1, k), nu, cap);
      d1[c] = mid + dt * ((T)0.5 * (a + b)) * lap;
    }
    if (z3 && i < nx && j < ny && k < nz + 1) {     // w face (nx, ny, nz+1)
      const int ex = nx, ey = ny, ez = nz + 1;
      const int c = (k * ey + j) * ex + i;
      const T mid = s2[c];
      const T lap = lap_face<T>(s2, c, mid, i > 0 ? 1 : 0, i < ex - 1 ? 1 : 0, j > 0 ? ex : 0, j < ey - 1 ? ex : 0,
                                k > 0 ? ex * ey : 0, k < ez - 1 ? ex * ey : 0, r20, r21, r22, ex > 1, ey > 1, ez > 1);
      const T a = nu_eff(nut, d.cidx32(i, j, max(k - 1, 0)), nu, cap);
      const T b = k < nz ? n0 : nu_eff(nut, d.cidx32(i, j, nz - 1), nu, cap);
      d2[c] = mid + dt * ((T)0.5 * (a + b)) * lap;
    }
  }
}

// ---------------------------------------------------------------------------
// porosity drag (solver.py:123-168)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// |u| at the centre of cell (i, j, k) (solver.py:160-161), roundings explicit
template <typename T>
__device__ __forceinline__ T cell_speed_at(const Dims& d, const T* __restrict__ u, const T* __restrict__ v,
                                           const T* __restrict__ w, int i, int j, int k) {
  const int c = d.cidx32(i, j, k);
  const int ui = ((int)k * d.ny + j) * (d.nx + 1) + i;
  const int vi = ((int)k * (d.ny + 1) + j) * d.nx + i;
  const T uc = (T)0.5 * (u[ui] + u[ui + 1]);
  const T vc = (T)0.5 * (v[vi] + v[vi + d.nx]);
  const T wc = (T)0.5 * (w[c] + w[c + (int)d.nx * d.ny]);
  // np.sum(vel * vel, axis=-1) with the two fused multiply-adds nvcc chose
  // for uc*uc + vc*vc + wc*wc (the arithmetic the parity runs validated)
  return sqrt(fma_rn(wc, wc, fma_rn(vc, vc, mul_rn(uc, uc))));
}

template <typename T>
__global__ void k_cell_speed(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                             const T* __restrict__ w, T* __restrict__ speed, const int* gate) {
  if (*gate) return;
  CW_IJK(d.nx, d.ny, d.nz, inb);
  if (inb) speed[d.cidx32(i, j, k)] = cell_speed_at<T>(d, u, v, w, i, j, k);
}

// max(0, 1 - dt g_face s_face) with the roundings nvcc chose for the plain
// expression (dt*g rounded, then one fused multiply-add)
template <typename T>
__device__ __forceinline__ T drag_fac(T gf, T sf, T dt) {
  const T fac = fma_rn(sf, -mul_rn(dt, gf), (T)1);
  return fac > (T)0 ? fac : (T)0;
}

template <typename T>
__device__ __forceinline__ void drag_face(const Dims& d, int comp, T* __restrict__ arr, const T* __restrict__ g,
                                          const T* __restrict__ speed, T dt, int i, int j, int k) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  const int nc = comp == 0 ? d.nx : (comp == 1 ? d.ny : d.nz);
  if (i < ex && j < ey && k < ez) {
    const int c = ((int)k * ey + j) * ex + i;
    int p[3] = {i, j, k};
    const int f = p[comp];
    p[comp] = clampi(f - 1, 0, nc - 1);
    const int lo = d.cidx32(p[0], p[1], p[2]);
    p[comp] = clampi(f, 0, nc - 1);
    const int hi = d.cidx32(p[0], p[1], p[2]);
    arr[c] *= drag_fac<T>((T)0.5 * (g[lo] + g[hi]), (T)0.5 * (speed[lo] + speed[hi]), dt);
  }
}

template <typename T>
__global__ void k_drag(Dims d, T* __restrict__ u, T* __restrict__ v, T* __restrict__ w, const T* __restrict__ g,
                       const T* __restrict__ speed, T dt, const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i > d.nx || j > d.ny) return;
#pragma unroll
  for (int kz = 0; kz < CW_ZT; ++kz) {
    const int k = (int)blockIdx.z * CW_ZT + kz;
    if (k > d.nz) break;
    drag_face<T>(d, 0, u, g, speed, dt, i, j, k);
    drag_face<T>(d, 1, v, g, speed, dt, i, j, k);
    if (!d.is2d) drag_face<T>(d, 2, w, g, speed, dt, i, j, k);
  }
}

// ---------------------------------------------------------------------------
// boundary conditions (solver.py:330-400): ordered outlet copies, one launch
// per domain side in the reference's side order, then inlet and wall writes.
template <typename T>
struct BcFields {
  T* u; T* v; T* w; T* p; T* k; T* om; T* nut;
};

template <typename T>
__global__ void k_bc_outlet_side(Dims d, int axis, int pos, BcFields<T> F,
                                 const int8_t* __restrict__ lab, const int* gate) {
  if (*gate) return;
  const int ext[3] = {d.nx, d.ny, d.nz};
  const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;   // in-plane axes
  const int n1 = ext[a1] + 1, n2 = ext[a2] + 1;
  const int inner = pos == 0 ? pos + 1 : pos - 1;
  const int n = n1 * n2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int q1 = t % n1, q2 = t / n1;
    int c[3];
    // cells (scalars) and the normal velocity component
    if (q1 < ext[a1] && q2 < ext[a2]) {
      c[axis] = pos; c[a1] = q1; c[a2] = q2;
      const int cc = d.cidx32(c[0], c[1], c[2]);
      if (lab[cc] == OUTLET) {
        c[axis] = inner;
        const int ci = d.cidx32(c[0], c[1], c[2]);
        F.k[cc] = F.k[ci]; F.om[cc] = F.om[ci]; F.nut[cc] = F.nut[ci]; F.p[cc] = F.p[ci];
        if (!(d.is2d && axis == 2)) {
          int ex, ey, ez;
          comp_extent(d, axis, ex, ey, ez);
          int f[3];
          f[a1] = q1; f[a2] = q2;
          f[axis] = pos > 0 ? pos + 1 : 0;
          const int fo = ((int)f[2] * ey + f[1]) * ex + f[0];
          f[axis] = pos > 0 ? pos : 1;
          const int fs = ((int)f[2] * ey + f[1]) * ex + f[0];
          T* arr = axis == 0 ? F.u : (axis == 1 ? F.v : F.w);
          arr[fo] = arr[fs];
        }
      }
    }
    // tangential components: face index q along its own axis, mask = either
    // adjacent outlet-slab cell is an outlet (_face_adjacent_mask)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int caxis = s == 0 ? a1 : a2;
      if (d.is2d && caxis == 2) continue;
      const int qa = s == 0 ? q1 : q2, qb = s == 0 ? q2 : q1;
      const int oth = s == 0 ? a2 : a1;
      if (qa > ext[caxis] || qb >= ext[oth]) continue;
      c[axis] = pos; c[oth] = qb;
      c[caxis] = clampi(qa - 1, 0, ext[caxis] - 1);
      bool m = lab[d.cidx32(c[0], c[1], c[2])] == OUTLET;
      c[caxis] = clampi(qa, 0, ext[caxis] - 1);
      m = m || lab[d.cidx32(c[0], c[1], c[2])] == OUTLET;
      if (!m) continue;
      int ex, ey, ez;
      comp_extent(d, caxis, ex, ey, ez);
      int f[3];
      f[axis] = pos; f[caxis] = qa; f[oth] = qb;
      const int fo = ((int)f[2] * ey + f[1]) * ex + f[0];
      f[axis] = inner;
      const int fs = ((int)f[2] * ey + f[1]) * ex + f[0];
      T* arr = caxis == 0 ? F.u : (caxis == 1 ? F.v : F.w);
      arr[fo] = arr[fs];
    }
  }
}

// inlet scalars, inlet face velocities, then walls zero all touching faces.
// One thread per (i, j, k) of the union of the cell and face extents.
template <typename T>
__device__ __forceinline__ void bc_face(const Dims& d, int comp, T* arr, const int8_t* lab, int i, int j, int k,
                                        const T* uz_dirx, const T* uz_diry) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  if (i >= ex || j >= ey || k >= ez) return;
  const int ext[3] = {d.nx, d.ny, d.nz};
  int p[3] = {i, j, k};
  const int f = p[comp];
  p[comp] = clampi(f - 1, 0, ext[comp] - 1);
  const int8_t la = lab[d.cidx32(p[0], p[1], p[2])];
  p[comp] = clampi(f, 0, ext[comp] - 1);
  const int8_t lb = lab[d.cidx32(p[0], p[1], p[2])];
  const int r = ((int)k * ey + j) * ex + i;
  if (la == SOLID_WALL || lb == SOLID_WALL) {
    arr[r] = (T)0;
  } else if (la == INLET || lb == INLET) {
    arr[r] = comp == 0 ? uz_dirx[p[2]] : (comp == 1 ? uz_diry[p[2]] : (T)0);
  }
}

template <typename T>
__global__ void k_bc_inlet_wall(Dims d, BcFields<T> F, const int8_t* __restrict__ lab,
                                const T* __restrict__ uz_dirx, const T* __restrict__ uz_diry,
                                T k_in, T om_in, T nut_in, const int* gate) {
  if (*gate) return;
  CW_IJK(d.nx + 1, d.ny + 1, d.nz + 1, inb);
  if (!inb) return;
  if (i < d.nx && j < d.ny && k < d.nz) {
    const int t = d.cidx32(i, j, k);
    if (lab[t] == INLET) { F.k[t] = k_in; F.om[t] = om_in; F.nut[t] = nut_in; }
  }
  bc_face<T>(d, 0, F.u, lab, i, j, k, uz_dirx, uz_diry);
  bc_face<T>(d, 1, F.v, lab, i, j, k, uz_dirx, uz_diry);
  if (!d.is2d) bc_face<T>(d, 2, F.w, lab, i, j, k, uz_dirx, uz_diry);
}

// ---------------------------------------------------------------------------
// The same boundary writes from precomputed lists.  The labels fix which
// locations each write touches, so they are enumerated once per labels array
// (k_bc_outlet_list / k_bc_inlet_wall_list, the predicates of the kernels
// above) and every step replays them with O(boundary) threads.  Within one
// side's list, and within the inlet/wall list, every (array, dst) is written
// by one entry and no entry reads another's dst, so entries run in any order;
// the sides still run in the reference's order (one launch each).
struct BcEntry {
  int arr;   // 0 u, 1 v, 2 w; 3: the four scalars k, omega, nu_t, p (copy) / k, omega, nu_t (inlet)
  int dst;
  int src;   // copy: source index; set: inlet profile row (>= 0) or -1 for a zero (wall)
};

__device__ __forceinline__ void bc_emit(BcEntry* out, int* count, int cap, int arr, int dst, int src) {
  const int q = atomicAdd(count, 1);
  if (out && q < cap) out[q] = BcEntry{arr, dst, src};
}

__global__ void k_bc_outlet_list(Dims d, int axis, int pos, const int8_t* __restrict__ lab, BcEntry* out, int* count,
                                 int cap) {
  const int ext[3] = {d.nx, d.ny, d.nz};
  const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;
  const int n1 = ext[a1] + 1, n2 = ext[a2] + 1;
  const int inner = pos == 0 ? pos + 1 : pos - 1;
  const int n = n1 * n2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int q1 = t % n1, q2 = t / n1;
    int c[3];
    if (q1 < ext[a1] && q2 < ext[a2]) {
      c[axis] = pos; c[a1] = q1; c[a2] = q2;
      const int cc = d.cidx32(c[0], c[1], c[2]);
      if (lab[cc] == OUTLET) {
        c[axis] = inner;
        bc_emit(out, count, cap, 3, cc, d.cidx32(c[0], c[1], c[2]));
        if (!(d.is2d && axis == 2)) {
          int ex, ey, ez;
          comp_extent(d, axis, ex, ey, ez);
          int f[3];
          f[a1] = q1; f[a2] = q2;
          f[axis] = pos > 0 ? pos + 1 : 0;
          const int fo = ((int)f[2] * ey + f[1]) * ex + f[0];
          f[axis] = pos > 0 ? pos : 1;
          bc_emit(out, count, cap, axis, fo, ((int)f[2] * ey + f[1]) * ex + f[0]);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int caxis = s == 0 ? a1 : a2;
      if (d.is2d && caxis == 2) continue;
      const int qa = s == 0 ? q1 : q2, qb = s == 0 ? q2 : q1;
      const int oth = s == 0 ? a2 : a1;
      if (qa > ext[caxis] || qb >= ext[oth]) continue;
      c[axis] = pos; c[oth] = qb;
      c[caxis] = clampi(qa - 1, 0, ext[caxis] - 1);
      bool m = lab[d.cidx32(c[0], c[1], c[2])] == OUTLET;
      c[caxis] = clampi(qa, 0, ext[caxis] - 1);
      m = m || lab[d.cidx32(c[0], c[1], c[2])] == OUTLET;
      if (!m) continue;
      int ex, ey, ez;
      comp_extent(d, caxis, ex, ey, ez);
      int f[3];
      f[axis] = pos; f[caxis] = qa; f[oth] = qb;
      const int fo = ((int)f[2] * ey + f[1]) * ex + f[0];
      f[axis] = inner;
      bc_emit(out, count, cap, caxis, fo, ((int)f[2] * ey + f[1]) * ex + f[0]);
    }
  }
}

__device__ __forceinline__ void bc_face_list(const Dims& d, int comp, const int8_t* lab, int i, int j, int k,
                                             BcEntry* out, int* count, int cap) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  if (i >= ex || j >= ey || k >= ez) return;
  const int ext[3] = {d.nx, d.ny, d.nz};
  int p[3] = {i, j, k};
  const int f = p[comp];
  p[comp] = clampi(f - 1, 0, ext[comp] - 1);
  const int8_t la = lab[d.cidx32(p[0], p[1], p[2])];
  p[comp] = clampi(f, 0, ext[comp] - 1);
  const int8_t lb = lab[d.cidx32(p[0], p[1], p[2])];
  const int r = ((int)k * ey + j) * ex + i;
  if (la == SOLID_WALL || lb == SOLID_WALL) bc_emit(out, count, cap, comp, r, -1);
  else if (la == INLET || lb == INLET) bc_emit(out, count, cap, comp, r, p[2]);
}

__global__ void k_bc_inlet_wall_list(Dims d, const int8_t* __restrict__ lab, BcEntry* out, int* count, int cap) {
  CW_IJK(d.nx + 1, d.ny + 1, d.nz + 1, inb);
  if (!inb) return;
  if (i < d.nx && j < d.ny && k < d.nz) {
    const int t = d.cidx32(i, j, k);
    if (lab[t] == INLET) bc_emit(out, count, cap, 3, t, 0);
  }
  bc_face_list(d, 0, lab, i, j, k, out, count, cap);
  bc_face_list(d, 1, lab, i, j, k, out, count, cap);
  if (!d.is2d) bc_face_list(d, 2, lab, i, j, k, out, count, cap);
}

template <typename T>
__global__ void k_bc_copy_list(BcFields<T> F, const BcEntry* __restrict__ e, int n, const int* gate) {
  if (*gate) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const BcEntry x = e[t];
    if (x.arr == 3) {
      F.k[x.dst] = F.k[x.src]; F.om[x.dst] = F.om[x.src]; F.nut[x.dst] = F.nut[x.src]; F.p[x.dst] = F.p[x.src];
    } else {
      T* a = x.arr == 0 ? F.u : (x.arr == 1 ? F.v : F.w);
      a[x.dst] = a[x.src];
    }
  }
}

template <typename T>
__global__ void k_bc_set_list(BcFields<T> F, const BcEntry* __restrict__ e, int n, const T* __restrict__ uz_dirx,
                              const T* __restrict__ uz_diry, T k_in, T om_in, T nut_in, const int* gate) {
  if (*gate) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const BcEntry x = e[t];
    if (x.arr == 3) {
      F.k[x.dst] = k_in; F.om[x.dst] = om_in; F.nut[x.dst] = nut_in;
    } else {
      T* a = x.arr == 0 ? F.u : (x.arr == 1 ? F.v : F.w);
      a[x.dst] = x.src < 0 ? (T)0 : (x.arr == 0 ? uz_dirx[x.src] : (x.arr == 1 ? uz_diry[x.src] : (T)0));
    }
  }
}

// ---------------------------------------------------------------------------
// One boundary pass as ONE launch.  The lists above are replayed in order
// (sides, then inlet/wall), so a later side can overwrite an earlier side's
// write or read it (edges and corners where two outlet sides meet).  Their
// composition is fixed by the labels: every location a pass writes ends up
// holding either the pass-start value of one location, a zero, an inlet
// profile value or an inlet scalar.  k_bc_compose_* derive that composition
// once per labels array (per list, in the reference's order: resolve each
// entry's source through the writer table of the lists before it, then claim
// its destinations); k_bc_replay then performs only the final writes.  A
// final write whose source location is itself finally written (or whose
// destination is such a source) must read before the other writes: those
// few (edge lines) go to block 0, which loads all their values, barriers and
// stores; every other write is independent of all the rest.  Pure copies and
// constants: the fields equal the ordered replay bit for bit.
// Expanded op: one field per op (fields 0 u, 1 v, 2 w, 3 k, 4 omega, 5 nu_t, 6 p).
enum BcKind { BK_ORIG = 0, BK_ZERO = 1, BK_INX = 2, BK_INY = 3, BK_KIN = 4, BK_OMIN = 5, BK_NUTIN = 6 };
struct BcOp {
  int fk;    // field | kind << 3; -1: unused slot
  int dst;
  int src;   // BK_ORIG: source index in the same field; BK_INX / BK_INY: profile row
};
struct BcFieldOff {
  long long off[8];   // writer-table offset of each field (off[7] = table size)
};

// expand list entries (4 op slots per entry) and resolve their sources
// through the writers of the earlier lists
__global__ void k_bc_compose_expand(const BcEntry* __restrict__ e, int n, bool set_list, BcOp* ops, long long base,
                                    const int* __restrict__ wmap, BcFieldOff fo) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const BcEntry x = e[t];
    BcOp* o = ops + base + 4 * (long long)t;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      BcOp op{-1, x.dst, 0};
      int f = -1, kind = BK_ORIG, src = x.src;
      if (x.arr < 3) {
        if (s == 0) {
          f = x.arr;
          if (set_list) {
            kind = x.src < 0 || x.arr == 2 ? BK_ZERO : (x.arr == 0 ? BK_INX : BK_INY);
            src = x.src < 0 ? 0 : x.src;
          }
        }
      } else if (!set_list) {
        f = s == 0 ? 3 : (s == 1 ? 4 : (s == 2 ? 5 : 6));   // k, omega, nu_t, p copied together
      } else if (s < 3) {
        f = 3 + s;
        kind = BK_KIN + s;
        src = 0;
      }
      if (f >= 0) {
        if (kind == BK_ORIG) {
          const int w = wmap[fo.off[f] + src];
          if (w >= 0) {   // the source was written by an earlier list: take that write's value
            const BcOp prev = ops[w];
            kind = prev.fk >> 3;
            src = prev.src;
          }
        }
        op.fk = f | (kind << 3);
        op.src = src;
      }
      o[s] = op;
    }
  }
}

// the list's ops become the latest writers of their destinations
__global__ void k_bc_compose_claim(const BcOp* __restrict__ ops, long long base, long long n, int* wmap, BcFieldOff fo) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const BcOp op = ops[base + t];
    if (op.fk >= 0) wmap[fo.off[op.fk & 7] + op.dst] = (int)(base + t);
  }
}

// 1 = final write (last writer, not an identity copy), 2 = final and ordered
// (reads a location another final write changes, or writes one that a final
// write reads)
__global__ void k_bc_compose_final(const BcOp* __restrict__ ops, long long n, const int* __restrict__ wmap, BcFieldOff fo,
                                   uint8_t* flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const BcOp op = ops[t];
    uint8_t fl = 0;
    if (op.fk >= 0) {
      const int f = op.fk & 7;
      const bool ident = (op.fk >> 3) == BK_ORIG && op.src == op.dst;
      fl = (wmap[fo.off[f] + op.dst] == (int)t && !ident) ? 1 : 0;
    }
    flag[t] = fl;
  }
}
__global__ void k_bc_compose_conflict(const BcOp* __restrict__ ops, long long n, const int* __restrict__ wmap, BcFieldOff fo,
                                      uint8_t* flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const BcOp op = ops[t];
    if (op.fk < 0 || (op.fk >> 3) != BK_ORIG || (flag[t] & 1) == 0) continue;
    const int w = wmap[fo.off[op.fk & 7] + op.src];
    if (w >= 0 && (flag[w] & 1)) {   // both orders matter: same value stored by every racer
      flag[t] = 3;
      flag[w] = 3;
    }
  }
}
// compaction: final writes to `free_ops` (from the front) or `ord_ops`
__global__ void k_bc_compose_compact(const BcOp* __restrict__ ops, long long n, const uint8_t* __restrict__ flag,
                                     BcOp* free_ops, BcOp* ord_ops, int ord_cap, int* counts) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const uint8_t fl = flag[t];
    if (fl == 1) {
      free_ops[atomicAdd(&counts[0], 1)] = ops[t];
    } else if (fl == 3) {
      const int q = atomicAdd(&counts[1], 1);
      if (q < ord_cap) ord_ops[q] = ops[t];
    }
  }
}

// the independent writes in (field, destination) order: coalesced replay
__global__ void k_bc_compose_keys(const BcOp* __restrict__ ops, int n, unsigned long long* keys, int* idx) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    keys[t] = ((unsigned long long)(ops[t].fk & 7) << 32) | (unsigned)ops[t].dst;
    idx[t] = t;
  }
}
__global__ void k_bc_compose_gather(const BcOp* __restrict__ ops, const int* __restrict__ idx, int n, BcOp* out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) out[t] = ops[idx[t]];
}

template <typename T>
__device__ __forceinline__ T* bc_field(const BcFields<T>& F, int f) {
  switch (f) {
    case 0: return F.u;
    case 1: return F.v;
    case 2: return F.w;
    case 3: return F.k;
    case 4: return F.om;
    case 5: return F.nut;
    default: return F.p;
  }
}
template <typename T>
__device__ __forceinline__ T bc_value(const BcFields<T>& F, const BcOp& op, const T* __restrict__ uzx,
                                      const T* __restrict__ uzy, T k_in, T om_in, T nut_in) {
  switch (op.fk >> 3) {
    case BK_ORIG: return bc_field<T>(F, op.fk & 7)[op.src];
    case BK_INX: return uzx[op.src];
    case BK_INY: return uzy[op.src];
    case BK_KIN: return k_in;
    case BK_OMIN: return om_in;
    case BK_NUTIN: return nut_in;
    default: return (T)0;
  }
}

constexpr int BC_ORD_PER_THREAD = 8;   // block 0: up to 256 * 8 ordered writes
// more ordered writes than block 0 holds: their values are read by a launch
// of their own first (k_bc_ord_gather into `held`), and k_bc_replay stores them
template <typename T>
__global__ void k_bc_ord_gather(BcFields<T> F, const BcOp* __restrict__ oops, int no, const T* __restrict__ uzx,
                                const T* __restrict__ uzy, T k_in, T om_in, T nut_in, unsigned fmask, T* held,
                                const int* gate, unsigned gate_pass = 0) {
  if (gated(gate, gate_pass)) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < no; t += gridDim.x * blockDim.x)
    if (fmask >> (oops[t].fk & 7) & 1u) held[t] = bc_value<T>(F, oops[t], uzx, uzy, k_in, om_in, nut_in);
}

// fmask: the fields (bit f) this launch writes -- a pass split by field
// (cw_step_defer_kw) is the same writes: every op reads its own field only
template <typename T>
__global__ void __launch_bounds__(256) k_bc_replay(BcFields<T> F, const BcOp* __restrict__ fops, int nf,
                                                   const BcOp* __restrict__ oops, int no, const T* __restrict__ uzx,
                                                   const T* __restrict__ uzy, T k_in, T om_in, T nut_in,
                                                   unsigned fmask, const int* gate, const T* __restrict__ held = nullptr,
                                                   unsigned gate_pass = 0) {
  if (gated(gate, gate_pass)) return;
  if (held) {   // the ordered writes' values were read by k_bc_ord_gather
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < no; t += gridDim.x * blockDim.x) {
      const BcOp op = oops[t];
      if (fmask >> (op.fk & 7) & 1u) bc_field<T>(F, op.fk & 7)[op.dst] = held[t];
    }
  } else if (blockIdx.x == 0) {
    T v[BC_ORD_PER_THREAD];
#pragma unroll
    for (int s = 0; s < BC_ORD_PER_THREAD; ++s) {
      const int t = (int)threadIdx.x + s * 256;
      if (t < no && (fmask >> (oops[t].fk & 7) & 1u)) v[s] = bc_value<T>(F, oops[t], uzx, uzy, k_in, om_in, nut_in);
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < BC_ORD_PER_THREAD; ++s) {
      const int t = (int)threadIdx.x + s * 256;
      if (t < no) {
        const BcOp op = oops[t];
        if (fmask >> (op.fk & 7) & 1u) bc_field<T>(F, op.fk & 7)[op.dst] = v[s];
      }
    }
    return;
  }
  const int b0 = held ? 0 : 1;   // without `held`, block 0 took the ordered writes
  for (int t = (blockIdx.x - b0) * blockDim.x + threadIdx.x; t < nf; t += (gridDim.x - b0) * blockDim.x) {
    const BcOp op = fops[t];
    if (fmask >> (op.fk & 7) & 1u) bc_field<T>(F, op.fk & 7)[op.dst] = bc_value<T>(F, op, uzx, uzy, k_in, om_in, nut_in);
  }
}

// ---------------------------------------------------------------------------
// pressure-gradient update (solver.py:282-303)
template <typename T>
__device__ __forceinline__ void gradient_face(const Dims& d, int comp, T* __restrict__ arr, const T* __restrict__ p,
                                              const int8_t* __restrict__ lab, T dt, int i, int j, int k) {
  int ex, ey, ez;
  comp_extent(d, comp, ex, ey, ez);
  const T rh = inv_h<T>(d, comp);
  const int nc = comp == 0 ? d.nx : (comp == 1 ? d.ny : d.nz);
  if (i < ex && j < ey && k < ez) {
    const int c = ((int)k * ey + j) * ex + i;
    int q[3] = {i, j, k};
    const int f = q[comp];
    if (f < 1 || f > nc - 1) return;
    q[comp] = f - 1;
    const int lo = d.cidx32(q[0], q[1], q[2]);
    q[comp] = f;
    const int hi = d.cidx32(q[0], q[1], q[2]);
    const int8_t la = lab[lo], lb = lab[hi];
    const T plo = p[lo], phi = p[hi], a = arr[c];   // not gated on the labels: one memory round trip
    const bool au = is_unknown(la), bu = is_unknown(lb);
    T grad = (T)0;
    if (au && bu) grad = (phi - plo) * rh;
    else if (au && lb == OUTLET) grad = -plo * rh;
    else if (bu && la == OUTLET) grad = phi * rh;
    else return;
    arr[c] = a - dt * grad;
  }
}

template <typename T>
__global__ void k_gradient(Dims d, T* __restrict__ u, T* __restrict__ v, T* __restrict__ w, const T* __restrict__ p,
                           const int8_t* __restrict__ lab, T dt, const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i > d.nx || j > d.ny) return;
#pragma unroll
  for (int kz = 0; kz < CW_ZT; ++kz) {
    const int k = (int)blockIdx.z * CW_ZT + kz;
    if (k > d.nz) break;
    gradient_face<T>(d, 0, u, p, lab, dt, i, j, k);
    gradient_face<T>(d, 1, v, p, lab, dt, i, j, k);
    if (!d.is2d) gradient_face<T>(d, 2, w, p, lab, dt, i, j, k);
  }
}

// max |div| over unknown cells (solver.py:215-229)
template <typename T>
__global__ void k_div_max(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                          const T* __restrict__ w, const int8_t* __restrict__ lab,
                          DevReport* rep, int slot, const int* gate) {
  if (*gate) return;
  __shared__ T scratch[32];
  T m = (T)0;
  // planes d.o0 + blockIdx.z, + gridDim.z, ...: a few blocks per column, one atomic each
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * 8 + threadIdx.y);
  if (i < d.nx && j < d.ny) {
    // the label does not gate the loads (one memory round trip per plane, not two)
#pragma unroll 2
    for (int k = d.o0 + (int)blockIdx.z; k < d.o1; k += (int)gridDim.z) {
      const int c = d.cidx32(i, j, k);
      const bool unk = is_unknown(lab[c]);
      const int ui = ((int)k * d.ny + j) * (d.nx + 1) + i;
      const int vi = ((int)k * (d.ny + 1) + j) * d.nx + i;
      T div = (u[ui + 1] - u[ui]) * inv_h<T>(d, 0) + (v[vi + d.nx] - v[vi]) * inv_h<T>(d, 1);
      if (!d.is2d) div = div + (w[c + (int)d.nx * d.ny] - w[c]) * inv_h<T>(d, 2);
      const T a = fabs(div);
      if (unk) m = (a > m || a != a) ? a : m;
    }
  }
  m = block_max_2d(m, scratch);
  if (threadIdx.x == 0 && threadIdx.y == 0) report_max<T>(rep, slot, m);
}

// max |u|,|v|,|w| for the CFL number (solver.py:456-458), over the owned
// planes (a w face shared with the slab above is counted by both, which a
// max does not notice).
// The owned part of each face array is one contiguous run of planes (u, v:
// planes o0..o1-1; w: faces o0..o1), so the CFL max runs over three flat
// ranges with 16-byte vector loads, grid-stride over a few blocks per SM.
template <typename T>
__device__ __forceinline__ T amax1(T m, T x) {
  const T a = fabs(x);
  return (a > m || a != a) ? a : m;   // NaN sticks (numpy max)
}
template <typename T> struct Vec16;
template <> struct Vec16<float> { typedef float4 type; static constexpr int n = 4; };
template <> struct Vec16<double> { typedef double2 type; static constexpr int n = 2; };

template <typename T>
__device__ __forceinline__ T absmax_run(const T* __restrict__ a, long long lo, long long hi, T m, long long gt,
                                        long long gs) {
  const T* p = a + lo;
  long long n = hi - lo;
  long long head = (long long)(((16u - ((uintptr_t)p & 15u)) & 15u) / sizeof(T));
  head = head < n ? head : n;
  for (long long e = gt; e < head; e += gs) m = amax1(m, p[e]);
  p += head;
  n -= head;
  using V = Vec16<T>;
  const long long nv = n / V::n;
  const typename V::type* pv = reinterpret_cast<const typename V::type*>(p);
  for (long long e = gt; e < nv; e += gs) {
    const typename V::type q = __ldcs(pv + e);
    const T* qq = reinterpret_cast<const T*>(&q);
#pragma unroll
    for (int c = 0; c < V::n; ++c) m = amax1(m, qq[c]);
  }
  for (long long e = nv * V::n + gt; e < n; e += gs) m = amax1(m, p[e]);
  return m;
}

template <typename T>
__global__ void k_speed_max_flat(Dims d, const T* __restrict__ u, const T* __restrict__ v, const T* __restrict__ w,
                                 DevReport* rep, const int* gate) {
  if (*gate) return;
  __shared__ T scratch[32];
  const long long gs = (long long)gridDim.x * blockDim.x * blockDim.y;
  const long long gt = (long long)blockIdx.x * blockDim.x * blockDim.y + threadIdx.y * blockDim.x + threadIdx.x;
  const long long pu = (long long)(d.nx + 1) * d.ny, pv = (long long)d.nx * (d.ny + 1), pw = (long long)d.nx * d.ny;
  T m = (T)0;
  m = absmax_run<T>(u, d.o0 * pu, d.o1 * pu, m, gt, gs);
  m = absmax_run<T>(v, d.o0 * pv, d.o1 * pv, m, gt, gs);
  m = absmax_run<T>(w, d.o0 * pw, (d.o1 + 1) * pw, m, gt, gs);
  m = block_max_2d(m, scratch);
  if (threadIdx.x == 0 && threadIdx.y == 0) report_max<T>(rep, SLOT_SPEED, m);
}

// ---------------------------------------------------------------------------
// k-omega sources, diffusion, limiter (turbulence.py:36-132)
template <typename T>
__device__ __forceinline__ T cell_vel(const Dims& d, int comp, const T* u, const T* v, const T* w,
                                      int i, int j, int k) {
  if (comp == 0) {
    const int ui = ((int)k * d.ny + j) * (d.nx + 1) + i;
    return (T)0.5 * (u[ui] + u[ui + 1]);
  }
  if (comp == 1) {
    const int vi = ((int)k * (d.ny + 1) + j) * d.nx + i;
    return (T)0.5 * (v[vi] + v[vi + d.nx]);
  }
  const int c = d.cidx32(i, j, k);
  return (T)0.5 * (w[c] + w[c + (int)d.nx * d.ny]);
}

// np.gradient of the cell-centred component `comp` along `ax` (edge_order 1)
template <typename T>
__device__ __forceinline__ T cgrad(const Dims& d, int comp, int ax, const T* u, const T* v,
                                   const T* w, int i, int j, int k) {
  const int n = ax == 0 ? d.nx : (ax == 1 ? d.ny : d.nz);
  if (n == 1) return (T)0;
  const int q = ax == 0 ? i : (ax == 1 ? j : k);
  const T rh = inv_h<T>(d, ax);
  int p0[3] = {i, j, k}, p1[3] = {i, j, k};
  if (q == 0) { p1[ax] = 1; p0[ax] = 0; }
  else if (q == n - 1) { p1[ax] = n - 1; p0[ax] = n - 2; }
  else { p1[ax] = q + 1; p0[ax] = q - 1; }
  const T f1 = cell_vel(d, comp, u, v, w, p1[0], p1[1], p1[2]);
  const T f0 = cell_vel(d, comp, u, v, w, p0[0], p0[1], p0[2]);
  if (q == 0 || q == n - 1) return (f1 - f0) * rh;
  return (f1 - f0) * ((T)0.5 * rh);
}

template <typename T>
__device__ __forceinline__ T pad_lap(const Dims& d, const T* f, int c, int i, int j, int k) {
  const int pos[3] = {i, j, k}, ext[3] = {d.nx, d.ny, d.nz};
  const int str[3] = {1, d.nx, (int)d.nx * d.ny};
  const T fc = f[c];
  T out = (T)0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const int n = ext[ax];
    if (n == 1) continue;
    const T r2 = inv_h2<T>(d, ax);
    if (pos[ax] == 0) out += (f[c + str[ax]] - fc) * r2;
    else if (pos[ax] == n - 1) out += (f[c - str[ax]] - fc) * r2;
    else out += (f[c - str[ax]] - (T)2 * fc + f[c + str[ax]]) * r2;
  }
  return out;
}

template <typename T>
__global__ void k_turbulence(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                             const T* __restrict__ w, const T* __restrict__ kin,
                             const T* __restrict__ win, T* __restrict__ kout, T* __restrict__ wout,
                             T* __restrict__ nut, T* __restrict__ nut_prev, StepConsts sc, DevReport* rep,
                             const int* gate) {
  if (*gate) return;
  const T dt = (T)sc.dt, nu = (T)sc.nu, cap = (T)sc.cap_turb;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i >= d.nx || j >= d.ny) return;
  for (int kz = 0; kz < ZT_TURB; ++kz) {
    const int k = (int)blockIdx.z * ZT_TURB + kz;
    if (k >= d.nz) break;
    const int c = d.cidx32(i, j, k);
    const int ui = ((int)k * d.ny + j) * (d.nx + 1) + i;
    const int vi = ((int)k * (d.ny + 1) + j) * d.nx + i;
    const T dudx = (u[ui + 1] - u[ui]) * inv_h<T>(d, 0);
    const T dvdy = (v[vi + d.nx] - v[vi]) * inv_h<T>(d, 1);
    const T dwdz = (w[c + (int)d.nx * d.ny] - w[c]) * inv_h<T>(d, 2);
    const T dudy = cgrad(d, 0, 1, u, v, w, i, j, k), dudz = cgrad(d, 0, 2, u, v, w, i, j, k);
    const T dvdx = cgrad(d, 1, 0, u, v, w, i, j, k), dvdz = cgrad(d, 1, 2, u, v, w, i, j, k);
    const T dwdx = cgrad(d, 2, 0, u, v, w, i, j, k), dwdy = cgrad(d, 2, 1, u, v, w, i, j, k);
    const T a = dudy + dvdx, b = dudz + dwdx, e = dvdz + dwdy;
    const T s2 = (dudx * dudx + dvdy * dvdy + dwdz * dwdz) + (T)0.5 * (a * a + b * b + e * e);
    const T nt = nut[c];
    const T kc = kin[c], wc = win[c];
    const T pk = (T)2 * nt * s2;
    T sk = (T)sc.sigma_star * nt; sk = sk < cap ? sk : cap;
    T sw = (T)sc.sigma * nt; sw = sw < cap ? sw : cap;
    const T dk = nu + sk, dw = nu + sw;
    const T kn = (kc + dt * (pk + dk * pad_lap(d, kin, c, i, j, k))) / ((T)1 + dt * (T)sc.c_mu * wc);
    const T wn = (wc + dt * ((T)2 * (T)sc.alpha * s2 + dw * pad_lap(d, win, c, i, j, k)))
                 / ((T)1 + dt * (T)sc.beta * wc);
    if (k >= d.o0 && k < d.o1) {   // reference C order over the global grid
      const long long ref = ((long long)i * d.ny + j) * d.nzg + (k + d.kg0);
      if (!isfinite(kn)) atomicMin(&rep->bad_index[0], ref);
      if (!isfinite(wn)) atomicMin(&rep->bad_index[1], ref);
    }
    const T kf = kn > (T)1e-12 ? kn : (T)1e-12;
    const T wf = wn > (T)1e-8 ? wn : (T)1e-8;
    T omt = (T)sc.c_lim * sqrt(s2) * (T)sc.lim_scale;
    omt = wf > omt ? wf : omt;
    omt = omt > (T)1e-8 ? omt : (T)1e-8;
    kout[c] = kf;
    wout[c] = wf;
    nut_prev[c] = nt;   // kept for cw_turb_rollback (the reference raises before it assigns)
    nut[c] = kf / omt;
  }
}

// The same k-omega update as a z march (one launch of (32, 8)-thread blocks,
// each thread a column (i, j) through TURB_CZ planes).  Per plane a thread
// loads its own cell once -- the six faces, k, omega, nu_t -- and forms the
// cell-centred velocities; x and y neighbours come from a shared plane tile
// (edge threads fill the one-cell halo), z neighbours from registers carried
// down the column.  Three shared planes rotate, so one barrier per plane
// suffices.  The arithmetic is the per-cell kernel's expression for
// expression: np.gradient (central, one-sided at the array ends) of the
// cell velocities, the edge-padded Laplacians of k and omega, the Patankar
// update, floors and limiter (turbulence.py:36-132).  ~530 instructions per
// cell in k_turbulence (ncu), most of them index arithmetic of the
// neighbour loads.
#ifndef CW_TURB_CZ
#define CW_TURB_CZ 8
#endif
constexpr int TURB_CZ = CW_TURB_CZ;

template <typename T>
struct TurbCell {
  T uc, vc, wc, k, om;
};

// np.gradient along one axis at position q of n (edge_order 1)
template <typename T>
__device__ __forceinline__ T grad3(T fm, T f0, T fp, int q, int n, T rh) {
  if (n == 1) return (T)0;
  if (q == 0) return (fp - f0) * rh;
  if (q == n - 1) return (f0 - fm) * rh;
  return (fp - fm) * ((T)0.5 * rh);
}
// one axis of the edge-padded Laplacian (turbulence.py:36-63)
template <typename T>
__device__ __forceinline__ T lap3(T fm, T f0, T fp, int q, int n, T r2) {
  if (n == 1) return (T)0;
  if (q == 0) return (fp - f0) * r2;
  if (q == n - 1) return (fm - f0) * r2;
  return (fm - (T)2 * f0 + fp) * r2;
}

template <typename T>
__device__ __forceinline__ TurbCell<T> turb_cell(const Dims& d, const T* __restrict__ u, const T* __restrict__ v,
                                                 const T* __restrict__ w, const T* __restrict__ kin,
                                                 const T* __restrict__ win, int i, int j, int k) {
  TurbCell<T> q;
  const int c = d.cidx32(i, j, k);
  const int ui = (k * d.ny + j) * (d.nx + 1) + i;
  const int vi = (k * (d.ny + 1) + j) * d.nx + i;
  q.uc = (T)0.5 * (u[ui] + u[ui + 1]);
  q.vc = (T)0.5 * (v[vi] + v[vi + d.nx]);
  q.wc = (T)0.5 * (w[c] + w[c + d.nx * d.ny]);
  q.k = kin[c];
  q.om = win[c];
  return q;
}

template <typename T>
__global__ void __launch_bounds__(256) k_turbulence_z(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                                                      const T* __restrict__ w, const T* __restrict__ kin,
                                                      const T* __restrict__ win, T* __restrict__ kout,
                                                      T* __restrict__ wout, T* __restrict__ nut,
                                                      T* __restrict__ nut_prev, StepConsts sc, DevReport* rep,
                                                      const int* gate) {
  if (*gate) return;
  // [rotating plane][quantity uc, vc, wc, k, om][row j0-1 .. j0+8][column i0-1 .. i0+32]
  __shared__ T tile[3][5][10][34];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = (int)blockIdx.x * 32 + tx, j = (int)blockIdx.y * 8 + ty;
  const int kb = (int)blockIdx.z * TURB_CZ, ke = min(kb + TURB_CZ, d.nz);
  const bool in = i < d.nx && j < d.ny;
  const T dt = (T)sc.dt, nu = (T)sc.nu, cap = (T)sc.cap_turb;
  const T rh0 = inv_h<T>(d, 0), rh1 = inv_h<T>(d, 1), rh2 = inv_h<T>(d, 2);
  const T r20 = inv_h2<T>(d, 0), r21 = inv_h2<T>(d, 1), r22 = inv_h2<T>(d, 2);
  const int m0 = max(kb - 1, 0), m1 = min(ke, d.nz - 1);   // planes whose cells the chunk reads
  TurbCell<T> qm{}, q0{}, qp{};   // planes m-2, m-1, m of this column
  auto put = [&](T (*t)[10][34], int r, int cl, const TurbCell<T>& q) {
    t[0][r][cl] = q.uc; t[1][r][cl] = q.vc; t[2][r][cl] = q.wc; t[3][r][cl] = q.k; t[4][r][cl] = q.om;
  };
  for (int m = m0; m <= m1 + 1; ++m) {
    if (m <= m1) {
      T (*t)[10][34] = tile[m % 3];
      if (in) {
        qp = turb_cell<T>(d, u, v, w, kin, win, i, j, m);
        put(t, ty + 1, tx + 1, qp);
        // the one-cell halo of the tile (not at the grid's ends)
        if (tx == 0 && i > 0) put(t, ty + 1, 0, turb_cell<T>(d, u, v, w, kin, win, i - 1, j, m));
        if ((tx == 31 || i == d.nx - 1) && i + 1 < d.nx)
          put(t, ty + 1, tx + 2, turb_cell<T>(d, u, v, w, kin, win, i + 1, j, m));
        if (ty == 0 && j > 0) put(t, 0, tx + 1, turb_cell<T>(d, u, v, w, kin, win, i, j - 1, m));
        if ((ty == 7 || j == d.ny - 1) && j + 1 < d.ny)
          put(t, ty + 2, tx + 1, turb_cell<T>(d, u, v, w, kin, win, i, j + 1, m));
      }
    }
    __syncthreads();
    const int k = m - 1;   // the plane whose update is complete: m-2, m-1, m are in hand
    if (in && k >= kb && k < ke) {
      const T (*t)[10][34] = tile[k % 3];
      const int r = ty + 1, cl = tx + 1;
      const int c = d.cidx32(i, j, k);
      const int ui = (k * d.ny + j) * (d.nx + 1) + i;
      const int vi = (k * (d.ny + 1) + j) * d.nx + i;
      const T dudx = (u[ui + 1] - u[ui]) * rh0;
      const T dvdy = (v[vi + d.nx] - v[vi]) * rh1;
      const T dwdz = (w[c + d.nx * d.ny] - w[c]) * rh2;
      const TurbCell<T>& zc = q0;   // this cell (plane k)
      const TurbCell<T>& zm = k > 0 ? qm : q0;
      const TurbCell<T>& zp = k < d.nz - 1 ? qp : q0;
      const T dudy = grad3<T>(t[0][r - 1][cl], t[0][r][cl], t[0][r + 1][cl], j, d.ny, rh1);
      const T dudz = grad3<T>(zm.uc, zc.uc, zp.uc, k, d.nz, rh2);
      const T dvdx = grad3<T>(t[1][r][cl - 1], t[1][r][cl], t[1][r][cl + 1], i, d.nx, rh0);
      const T dvdz = grad3<T>(zm.vc, zc.vc, zp.vc, k, d.nz, rh2);
      const T dwdx = grad3<T>(t[2][r][cl - 1], t[2][r][cl], t[2][r][cl + 1], i, d.nx, rh0);
      const T dwdy = grad3<T>(t[2][r - 1][cl], t[2][r][cl], t[2][r + 1][cl], j, d.ny, rh1);
      const T a = dudy + dvdx, b = dudz + dwdx, e = dvdz + dwdy;
      const T s2 = (dudx * dudx + dvdy * dvdy + dwdz * dwdz) + (T)0.5 * (a * a + b * b + e * e);
      T lk = (T)0, lw = (T)0;
      lk += lap3<T>(t[3][r][cl - 1], zc.k, t[3][r][cl + 1], i, d.nx, r20);
      lw += lap3<T>(t[4][r][cl - 1], zc.om, t[4][r][cl + 1], i, d.nx, r20);
      lk += lap3<T>(t[3][r - 1][cl], zc.k, t[3][r + 1][cl], j, d.ny, r21);
      lw += lap3<T>(t[4][r - 1][cl], zc.om, t[4][r + 1][cl], j, d.ny, r21);
      lk += lap3<T>(zm.k, zc.k, zp.k, k, d.nz, r22);
      lw += lap3<T>(zm.om, zc.om, zp.om, k, d.nz, r22);
      const T nt = nut[c];
      const T kc = zc.k, wc = zc.om;
      const T pk = (T)2 * nt * s2;
      T sk = (T)sc.sigma_star * nt; sk = sk < cap ? sk : cap;
      T sw = (T)sc.sigma * nt; sw = sw < cap ? sw : cap;
      const T dk = nu + sk, dw = nu + sw;
      const T kn = (kc + dt * (pk + dk * lk)) / ((T)1 + dt * (T)sc.c_mu * wc);
      const T wn = (wc + dt * ((T)2 * (T)sc.alpha * s2 + dw * lw)) / ((T)1 + dt * (T)sc.beta * wc);
      if (k >= d.o0 && k < d.o1) {   // reference C order over the global grid
        const long long refi = ((long long)i * d.ny + j) * d.nzg + (k + d.kg0);
        if (!isfinite(kn)) atomicMin(&rep->bad_index[0], refi);
        if (!isfinite(wn)) atomicMin(&rep->bad_index[1], refi);
      }
      const T kf = kn > (T)1e-12 ? kn : (T)1e-12;
      const T wf = wn > (T)1e-8 ? wn : (T)1e-8;
      T omt = (T)sc.c_lim * sqrt(s2) * (T)sc.lim_scale;
      omt = wf > omt ? wf : omt;
      omt = omt > (T)1e-8 ? omt : (T)1e-8;
      kout[c] = kf;
      wout[c] = wf;
      nut_prev[c] = nt;
      nut[c] = kf / omt;
    }
    qm = q0;
    q0 = qp;
  }
}

// The k-omega update per cell with straight-line neighbour access: the
// array-end rules of np.gradient and the edge-padded Laplacian become clamped
// neighbour indices (a clamped neighbour equals the cell itself, and
// (f - 2 f) + f_p == f_p - f exactly), so the interior and the edges run the
// same instructions; the one-sided gradient keeps its 1/h, the central one
// its 1/(2h).  Same arithmetic as k_turbulence, far fewer instructions.
#ifndef CW_TURB_ZT
#define CW_TURB_ZT 1
#endif
constexpr int TURB_ZT = CW_TURB_ZT;   // planes per thread of k_turbulence_c

template <typename T>
__global__ void __launch_bounds__(256) k_turbulence_c(Dims d, const T* __restrict__ u, const T* __restrict__ v,
                                                      const T* __restrict__ w, const T* __restrict__ kin,
                                                      const T* __restrict__ win, T* __restrict__ kout,
                                                      T* __restrict__ wout, T* __restrict__ nut,
                                                      T* __restrict__ nut_prev, StepConsts sc, DevReport* rep,
                                                      const int* gate) {
  if (*gate) return;
  const int i = (int)(blockIdx.x * ST_BX + threadIdx.x), j = (int)(blockIdx.y * ST_BY + threadIdx.y);
  if (i >= d.nx || j >= d.ny) return;
#pragma unroll
  for (int kz = 0; kz < TURB_ZT; ++kz) {
  const int k = (int)blockIdx.z * TURB_ZT + kz;
  if (k >= d.nz) break;
  const T dt = (T)sc.dt, nu = (T)sc.nu, cap = (T)sc.cap_turb;
  const T rh0 = inv_h<T>(d, 0), rh1 = inv_h<T>(d, 1), rh2 = inv_h<T>(d, 2);
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int im = max(i - 1, 0), ip = min(i + 1, nx - 1);
  const int jm = max(j - 1, 0), jp = min(j + 1, ny - 1);
  const int km = max(k - 1, 0), kp = min(k + 1, nz - 1);
  const T gx = (ip - im == 2) ? (T)0.5 * rh0 : rh0;   // central / one-sided (n == 1: both 0, any scale)
  const T gy = (jp - jm == 2) ? (T)0.5 * rh1 : rh1;
  const T gz = (kp - km == 2) ? (T)0.5 * rh2 : rh2;
  const int uy = nx + 1, uz = (nx + 1) * ny;   // u strides
  const int vy = nx, vz = nx * (ny + 1);       // v strides
  const int cy = nx, cz = nx * ny;             // cell / w strides
  const int c = k * cz + j * cy + i;
  // own faces
  const T* ur = u + k * uz + j * uy;
  const T* vr = v + k * vz + j * vy;
  const T u0 = ur[i], u1 = ur[i + 1];
  const T v0 = vr[i], v1 = vr[i + vy];
  const T w0 = w[c], w1 = w[c + cz];
  const T dudx = (u1 - u0) * rh0;
  const T dvdy = (v1 - v0) * rh1;
  const T dwdz = (w1 - w0) * rh2;
  // cell-centred velocities of the neighbours (cell_vel: 0.5 * (a + b))
  const T* urm = u + k * uz + jm * uy; const T* urp = u + k * uz + jp * uy;       // rows jm, jp
  const T* uzm = u + km * uz + j * uy; const T* uzp = u + kp * uz + j * uy;       // planes km, kp
  const T uc_jm = (T)0.5 * (urm[i] + urm[i + 1]), uc_jp = (T)0.5 * (urp[i] + urp[i + 1]);
  const T uc_km = (T)0.5 * (uzm[i] + uzm[i + 1]), uc_kp = (T)0.5 * (uzp[i] + uzp[i + 1]);
  const T vc_im = (T)0.5 * (vr[im] + vr[im + vy]), vc_ip = (T)0.5 * (vr[ip] + vr[ip + vy]);
  const T* vzm = v + km * vz + j * vy; const T* vzp = v + kp * vz + j * vy;
  const T vc_km = (T)0.5 * (vzm[i] + vzm[i + vy]), vc_kp = (T)0.5 * (vzp[i] + vzp[i + vy]);
  const T* wr = w + k * cz + j * cy;
  const T wc_im = (T)0.5 * (wr[im] + wr[im + cz]), wc_ip = (T)0.5 * (wr[ip] + wr[ip + cz]);
  const T* wrm = w + k * cz + jm * cy; const T* wrp = w + k * cz + jp * cy;
  const T wc_jm = (T)0.5 * (wrm[i] + wrm[i + cz]), wc_jp = (T)0.5 * (wrp[i] + wrp[i + cz]);
  const T dudy = (uc_jp - uc_jm) * gy, dudz = (uc_kp - uc_km) * gz;
  const T dvdx = (vc_ip - vc_im) * gx, dvdz = (vc_kp - vc_km) * gz;
  const T dwdx = (wc_ip - wc_im) * gx, dwdy = (wc_jp - wc_jm) * gy;
  const T a = dudy + dvdx, b = dudz + dwdx, e = dvdz + dwdy;
  const T s2 = (dudx * dudx + dvdy * dvdy + dwdz * dwdz) + (T)0.5 * (a * a + b * b + e * e);
  // edge-padded Laplacians (pad_lap): clamped neighbours
  const T r20 = inv_h2<T>(d, 0), r21 = inv_h2<T>(d, 1), r22 = inv_h2<T>(d, 2);
  const int cxm = k * cz + j * cy + im, cxp = k * cz + j * cy + ip;
  const int cym = k * cz + jm * cy + i, cyp = k * cz + jp * cy + i;
  const int czm = km * cz + j * cy + i, czp = kp * cz + j * cy + i;
  const T kc = kin[c], wc = win[c];
  T lk = (T)0, lw = (T)0;
  if (nx > 1) { lk += (kin[cxm] - (T)2 * kc + kin[cxp]) * r20; lw += (win[cxm] - (T)2 * wc + win[cxp]) * r20; }
  if (ny > 1) { lk += (kin[cym] - (T)2 * kc + kin[cyp]) * r21; lw += (win[cym] - (T)2 * wc + win[cyp]) * r21; }
  if (nz > 1) { lk += (kin[czm] - (T)2 * kc + kin[czp]) * r22; lw += (win[czm] - (T)2 * wc + win[czp]) * r22; }
  const T nt = nut[c];
  const T pk = (T)2 * nt * s2;
  T sk = (T)sc.sigma_star * nt; sk = sk < cap ? sk : cap;
  T sw = (T)sc.sigma * nt; sw = sw < cap ? sw : cap;
  const T dk = nu + sk, dw = nu + sw;
  const T kn = (kc + dt * (pk + dk * lk)) / ((T)1 + dt * (T)sc.c_mu * wc);
  const T wn = (wc + dt * ((T)2 * (T)sc.alpha * s2 + dw * lw)) / ((T)1 + dt * (T)sc.beta * wc);
  const bool bad_k = !isfinite(kn), bad_w = !isfinite(wn);
  if ((bad_k || bad_w) && k >= d.o0 && k < d.o1) {   // reference C order over the global grid
    const long long refi = ((long long)i * d.ny + j) * d.nzg + (k + d.kg0);
    if (bad_k) atomicMin(&rep->bad_index[0], refi);
    if (bad_w) atomicMin(&rep->bad_index[1], refi);
  }
  const T kf = kn > (T)1e-12 ? kn : (T)1e-12;
  const T wf = wn > (T)1e-8 ? wn : (T)1e-8;
  T omt = (T)sc.c_lim * sqrt(s2) * (T)sc.lim_scale;
  omt = wf > omt ? wf : omt;
  omt = omt > (T)1e-8 ? omt : (T)1e-8;
  kout[c] = kf;
  wout[c] = wf;
  nut_prev[c] = nt;
  nut[c] = kf / omt;
  }
}

// After a non-finite k / omega (status 2) the reference has raised before it
// assigned anything (turbulence.py:121-131): the state keeps the advected
// k, omega (still in the step's upwind buffers) and the previous nu_t
// (k_turbulence saved it).  Launched by cw_turb_rollback on the error path only.
template <typename T>
__global__ void k_turb_rollback(long long n, const T* __restrict__ k_adv, const T* __restrict__ w_adv,
                                const T* __restrict__ nut_prev, T* __restrict__ k, T* __restrict__ w,
                                T* __restrict__ nut) {
  CW_GRID_STRIDE(c, n) {
    k[c] = k_adv[c];
    w[c] = w_adv[c];
    if (nut_prev) nut[c] = nut_prev[c];
  }
}

// ---------------------------------------------------------------------------
// z-slab reach check (SURVEY 7 hard part 4).  A window stores `halo` planes
// beyond its owned planes on each interior face; the step's stages read
// across planes, so the owned planes come out as in the whole-grid step only
// if the chain's reach fits.  The MacCormack backtrace and forward trace each
// reach floor(S) + 1 planes (S = max|w| dt / dz, unbounded: the scheme is
// unconditionally stable), diffusion and the drag's cell speeds one more
// each: 2 floor(S) + 4 planes (S < 1: 4, the z-slab tests' measured minimum
// for bitwise equality).  max|w| over the window before the step; too
// shallow a halo fails the step loudly instead of corrupting the owned planes.
template <typename T>
__global__ void k_wmax_window(long long n, const T* __restrict__ w, DevReport* rep, const int* gate) {
  if (*gate) return;
  __shared__ T scratch[32];
  T m = (T)0;
  CW_GRID_STRIDE(c, n) {
    const T a = fabs(w[c]);
    m = (a > m || a != a) ? a : m;
  }
  m = block_max(m, scratch);
  if (threadIdx.x == 0) report_max<T>(rep, SLOT_WMAX, m);
}

template <typename T>
__global__ void k_halo_gate(Dims d, double dt, DevReport* rep, int* gate) {
  if (*gate) return;
  double wmax;
  if (sizeof(T) == 4) wmax = (double)__uint_as_float(rep->fmax[SLOT_WMAX]);
  else wmax = __longlong_as_double((long long)rep->dmax[SLOT_WMAX]);
  const double S = wmax * dt / d.ddz;
  const int need = S != S ? 1 << 30 : 2 * (int)floor(fmin(S, 1e6)) + 4;
  const int lo = d.kg0 > 0 ? d.o0 : (1 << 30);                      // interior faces only: at the
  const int hi = d.kg0 + d.nz < d.nzg ? d.nz - d.o1 : (1 << 30);    // grid's ends the clamp is the grid's
  if (need > (lo < hi ? lo : hi)) {
    rep->status = 5;
    rep->halo_need = need;
    rep->criterion = S;
    *gate = 5;
  }
}

// turbulence error latch: runs after k_turbulence, sets the step status/gate
__global__ void k_turb_check(DevReport* rep, int* gate) {
  if (*gate) return;
  if (rep->bad_index[0] != 0x7fffffffffffffffLL || rep->bad_index[1] != 0x7fffffffffffffffLL) {
    rep->status = 2;
    *gate = 2;
  }
}

}  // namespace cw
