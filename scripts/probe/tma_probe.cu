// Standalone probe of the TMA/mbarrier helpers used by k_pcg.
#include <cstdio>
#include <vector>
#include <cudaTypedefs.h>
#include "../../paper_2204_01117_b200/csrc/cw_pcg.cuh"
using namespace cw;

struct Args { CUtensorMap tm; int mode; int cx, cy, cz; };

__global__ void probe(const __grid_constant__ Args a, float* out, const CUtensorMap* gtm) {
  extern __shared__ uint8_t dyn[];
  uint8_t* base = reinterpret_cast<uint8_t*>(((uintptr_t)dyn + 127) & ~(uintptr_t)127);
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (a.mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.mode & 2) fence_proxy_async();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, BOX_X * BOX_Y * 4);
    const CUtensorMap* m = (a.mode & 4) ? gtm : &a.tm;
    const int c0 = (a.mode & 8) ? 0 : -1;
    (void)c0;
    if (a.mode & 16) asm volatile("prefetch.tensormap [%0];" :: "l"((unsigned long long)m) : "memory");
    tma_load_3d(base, m, &bar, a.cx, a.cy, a.cz);
  }
  mbar_wait(&bar, 0);
  const float* f = reinterpret_cast<const float*>(base);
  for (int e = threadIdx.x; e < BOX_X * BOX_Y; e += blockDim.x) out[e] = f[e];
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 3;
  const int nx = 48, ny = 16, nz = 4, nxp = 48;
  std::vector<float> h(nxp * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  Args a; a.mode = mode; a.cx = atoi(argv[2]); a.cy = atoi(argv[3]); a.cz = atoi(argv[4]);
  cuuint64_t dims[3] = {nx, ny, nz};
  cuuint64_t str[2] = {nxp * 4, (cuuint64_t)nxp * ny * 4};
  cuuint32_t box[3] = {BOX_X, BOX_Y, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  CUtensorMap* g; cudaMalloc(&g, sizeof(CUtensorMap));
  cudaMemcpy(g, &a.tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  printf("sizeof Args %zu align %zu\n", sizeof(Args), alignof(Args));
  probe<<<1, 128, 8192>>>(a, o, g);
  cudaError_t e = cudaDeviceSynchronize();
  printf("coords %d %d %d: %s\n", a.cx, a.cy, a.cz, cudaGetErrorString(e));
  std::vector<float> ho(BOX_X * BOX_Y);
  cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
  printf("row0: %g %g %g ... row1: %g %g\n", ho[0], ho[1], ho[2], ho[BOX_X], ho[BOX_X + 1]);
  return 0;
}
