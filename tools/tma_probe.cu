// Probe: which 3-D TMA tile configurations the B200 accepts (box width,
// negative start coordinates).  nvcc -arch=sm_100a tools/tma_probe.cu -o /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, int x, int y, int z, int bytes, int* out) {
  extern __shared__ __align__(128) unsigned char s[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sa(s)), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(sa(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
    out[0] = ((uint16_t*)s)[0];
  }
}

int main() {
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  uint16_t* d; cudaMalloc(&d, 64 << 20);
  int* out; cudaMalloc(&out, 4);
  int widths[] = {48, 56, 64, 96, 104, 112, 128};
  int coords[][3] = {{0, 0, 0}, {-8, 0, 0}, {0, -1, 0}, {0, 0, -1}, {-8, -1, -1}, {184, 60, 63}};
  for (int w : widths)
    for (auto& c : coords) {
      CUtensorMap map;
      cuuint64_t dims[3] = {192, 64, 64};
      cuuint64_t st[2] = {384, 384 * 64};
      cuuint32_t box[3] = {(cuuint32_t)w, 18, 2};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      int bytes = w * 18 * 2 * 2;
      k<<<1, 32, 16384>>>(map, c[0], c[1], c[2], bytes, out);
      cudaError_t e = cudaDeviceSynchronize();
      printf("w=%3d coords=(%d,%d,%d) encode=%d run=%s\n", w, c[0], c[1], c[2], (int)r, cudaGetErrorString(e));
      if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, 64 << 20); cudaMalloc(&out, 4); }
    }
}
