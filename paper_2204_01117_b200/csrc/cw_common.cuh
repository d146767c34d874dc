// Common device helpers for the citywind B200 step path.
//
// Layout: every field is x-fastest.  A cell field is (nz, ny, nx); the
// staggered velocity components are u (nz, ny, nx+1), v (nz, ny+1, nx),
// w (nz+1, ny, nx).  This is the reference's F-order / unknown numbering
// (linalg.py:53-54), so pressure unknowns keep the reference's order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cw {

enum Label : int8_t { AIR = 0, BUILDING = 1, TREE = 2, INLET = 3, OUTLET = 4, SOLID_WALL = 5 };

__host__ __device__ inline bool is_unknown(int8_t l) { return l == AIR || l == BUILDING || l == TREE; }

struct Dims {
  int nx, ny, nz;
  float dx, dy, dz;        // spacings in the arithmetic type used by kernels
  double ddx, ddy, ddz;    // float64 spacings for host-side derived constants
  int is2d;
  // reciprocal spacings 1/h and 1/h^2 per axis (host-computed in float64):
  // kernels multiply instead of dividing by the constant spacings
  float rh[3], rh2[3];
  double drh[3], drh2[3];
  // z-slab window: the local grid holds global planes [kg0, kg0 + nz) of a
  // grid with nzg planes and owns local planes [o0, o1) (reductions and
  // reports cover the owned planes only).  A whole grid: 0, nz, 0, nz.
  int o0, o1, kg0, nzg;
  __host__ __device__ inline long long ncell() const { return (long long)nx * ny * nz; }
  __host__ __device__ inline long long cidx(int i, int j, int k) const {
    return ((long long)k * ny + j) * nx + i;
  }
  // 32-bit cell index (contexts hold < 2^31 cells per field, cw_capi.cu)
  __host__ __device__ inline int cidx32(int i, int j, int k) const { return (k * ny + j) * nx + i; }
};

template <typename T> __host__ __device__ inline T inv_h(const Dims& d, int ax);
template <> __host__ __device__ inline float inv_h<float>(const Dims& d, int ax) { return d.rh[ax]; }
template <> __host__ __device__ inline double inv_h<double>(const Dims& d, int ax) { return d.drh[ax]; }
template <typename T> __host__ __device__ inline T inv_h2(const Dims& d, int ax);
template <> __host__ __device__ inline float inv_h2<float>(const Dims& d, int ax) { return d.rh2[ax]; }
template <> __host__ __device__ inline double inv_h2<double>(const Dims& d, int ax) { return d.drh2[ax]; }

// Extents of component arrays: comp 0 = u, 1 = v, 2 = w, 3 = cell.
__host__ __device__ inline void comp_extent(const Dims& d, int comp, int& ex, int& ey, int& ez) {
  ex = d.nx + (comp == 0);
  ey = d.ny + (comp == 1);
  ez = d.nz + (comp == 2);
}

// ---------------------------------------------------------------------------
// Trilinear gather with clamped indices (advection.py:49-101, _kernels.py:25-58)
// Arrays hold < 2^31 elements (checked at context creation): 32-bit indices.
template <typename T>
__device__ __forceinline__ T gather_at(const T* __restrict__ a, int ex, int ey, int ez, int i0, int j0, int k0,
                                       T tx, T ty, T tz, T* mn, T* mx) {
  const int sx = ex > 1 ? 1 : 0, sy = ey > 1 ? ex : 0, sz = ez > 1 ? ex * ey : 0;
  const int b = (k0 * ey + j0) * ex + i0;
  const T c000 = a[b], c100 = a[b + sx], c010 = a[b + sy], c110 = a[b + sx + sy];
  const T c001 = a[b + sz], c101 = a[b + sx + sz], c011 = a[b + sy + sz], c111 = a[b + sx + sy + sz];
  const T ox = (T)1 - tx, oy = (T)1 - ty, oz = (T)1 - tz;
  const T c00 = c000 * ox + c100 * tx, c10 = c010 * ox + c110 * tx;
  const T c01 = c001 * ox + c101 * tx, c11 = c011 * ox + c111 * tx;
  const T c0 = c00 * oy + c10 * ty, c1 = c01 * oy + c11 * ty;
  if (mn) {   // the stencil's min / max (finite values: order-independent, one FMNMX each)
    *mn = fmin(fmin(fmin(c000, c100), fmin(c010, c110)), fmin(fmin(c001, c101), fmin(c011, c111)));
    *mx = fmax(fmax(fmax(c000, c100), fmax(c010, c110)), fmax(fmax(c001, c101), fmax(c011, c111)));
  }
  return c0 * oz + c1 * tz;
}

// fz is a GLOBAL z coordinate and the array's plane 0 is global plane kg0 (a
// z-slab window; 0 for a whole grid): the floor and the weight are taken in
// global coordinates, so a slab rounds exactly like the whole grid (a local
// coordinate k + 0.5 - s rounds differently from kg0 + k + 0.5 - s), and the
// index is clamped to the stored planes
template <typename T>
__device__ __forceinline__ T gather(const T* __restrict__ a, int ex, int ey, int ez,
                                    T fx, T fy, T fz, T* mn, T* mx, int kg0 = 0) {
  int i0 = (int)floor(fx), j0 = (int)floor(fy), k0 = (int)floor(fz);
  const int im = ex - 2 > 0 ? ex - 2 : 0, jm = ey - 2 > 0 ? ey - 2 : 0, km = ez - 2 > 0 ? ez - 2 : 0;
  i0 = i0 < 0 ? 0 : (i0 > im ? im : i0);
  j0 = j0 < 0 ? 0 : (j0 > jm ? jm : j0);
  k0 = k0 < kg0 ? kg0 : (k0 > kg0 + km ? kg0 + km : k0);
  T tx = fx - (T)i0, ty = fy - (T)j0, tz = fz - (T)k0;
  tx = tx < (T)0 ? (T)0 : (tx > (T)1 ? (T)1 : tx);
  ty = ty < (T)0 ? (T)0 : (ty > (T)1 ? (T)1 : ty);
  tz = tz < (T)0 ? (T)0 : (tz > (T)1 ? (T)1 : tz);
  return gather_at<T>(a, ex, ey, ez, i0, j0, k0 - kg0, tx, ty, tz, mn, mx);
}


// ---------------------------------------------------------------------------
// Order-independent max reductions on non-negative values (bit patterns of
// non-negative IEEE floats order like unsigned integers; NaN sorts above inf,
// so a NaN anywhere propagates exactly like numpy's max).
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (w > v || w != w) ? w : v;
  }
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide reductions with a fixed tree: deterministic for a fixed block
// shape.  `scratch` must hold blockDim/32 entries.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in thread 0
}

template <typename T>
__device__ __forceinline__ T block_max(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T t = (T)0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : (T)0;
    t = warp_max(t);
  }
  return t;  // valid in thread 0
}

// block_max for 2-D blocks (linear thread id x + y * blockDim.x); result in thread (0, 0)
template <typename T>
__device__ __forceinline__ T block_max_2d(T v, T* scratch) {
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = (blockDim.x * blockDim.y + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T t = (T)0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : (T)0;
    t = warp_max(t);
  }
  return t;
}

}  // namespace cw
