// Stand-alone probe of the TMA row load used by k_step (debug aid):
// 3-D FP64 map {pitch, ny, 8} with box {NT, 1, 4} + 2-D u8 mask map, one
// mbarrier, loads one row and copies the staged smem back to global.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int NT = 128;
__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
constexpr int MW = NT + 16;  // mask box: starts at a 16-column boundary
__global__ void k_probe(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tm,
                        int c0, int row, int plane0, double* out, unsigned char* outm) {
  __shared__ __align__(128) double q[4][NT];
  __shared__ __align__(128) unsigned char m[MW];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                 "r"(4u * NT * 8u + MW)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(&q[0][0])),
        "l"(reinterpret_cast<unsigned long long>(&tq)), "r"(c0), "r"(row), "r"(plane0),
        "r"(su32(&bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(su32(&m[0])),
        "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(c0 & ~15), "r"(row), "r"(su32(&bar))
        : "memory");
  }
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(&bar)), "r"(0u)
        : "memory");
  } while (!done);
  for (int p = 0; p < 4; p++) out[p * NT + threadIdx.x] = q[p][threadIdx.x];
  outm[threadIdx.x] = m[(c0 & 15) + threadIdx.x];
}

int main() {
  const int pitch = 256, ny = 64;
  const size_t plane = (size_t)pitch * ny;
  double* d;
  cudaMalloc(&d, (8 * plane + 4) * sizeof(double));
  double* base = d + 2;
  double* h = (double*)malloc(8 * plane * sizeof(double));
  for (size_t i = 0; i < 8 * plane; i++) h[i] = (double)i;
  cudaMemcpy(base, h, 8 * plane * sizeof(double), cudaMemcpyHostToDevice);
  unsigned char* dm;
  cudaMalloc(&dm, plane);
  unsigned char* hm = (unsigned char*)malloc(plane);
  for (size_t i = 0; i < plane; i++) hm[i] = (unsigned char)(i % 251);
  cudaMemcpy(dm, hm, plane, cudaMemcpyHostToDevice);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tq, tm;
  cuuint64_t qdim[3] = {(cuuint64_t)pitch, (cuuint64_t)ny, 8};
  cuuint64_t qstr[2] = {(cuuint64_t)pitch * 8, plane * 8};
  cuuint32_t qbox[3] = {NT, 1, 4};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&tq, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, qdim, qstr, qbox, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode q: %d\n", (int)r);
  cuuint64_t mdim[2] = {(cuuint64_t)pitch, (cuuint64_t)ny};
  cuuint64_t mstr[1] = {(cuuint64_t)pitch};
  cuuint32_t mbox[2] = {MW, 1};
  r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dm, mdim, mstr, mbox, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode m: %d\n", (int)r);
  double* out;
  unsigned char* outm;
  cudaMalloc(&out, 4 * NT * 8);
  cudaMalloc(&outm, NT);
  int cases[6][3] = {{0, 5, 0}, {124, 7, 4}, {200, -2, 4}, {0, 63, 0}, {248, 3, 0}, {62, 1, 1}};
  for (auto& cs : cases) {
    k_probe<<<1, NT>>>(tq, tm, cs[0], cs[1], cs[2], out, outm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("case c0=%d row=%d plane=%d: %s\n", cs[0], cs[1], cs[2], cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    double ho[4 * NT];
    unsigned char hmo[NT];
    cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
    cudaMemcpy(hmo, outm, NT, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int p = 0; p < 4; p++)
      for (int t = 0; t < NT; t++) {
        int col = cs[0] + t, row = cs[1];
        double want = (col < pitch && row >= 0 && row < ny) ? h[(cs[2] + p) * plane + (size_t)row * pitch + col] : 0.0;
        if (ho[p * NT + t] != want) bad++;
      }
    for (int t = 0; t < NT; t++) {
      int col = cs[0] + t, row = cs[1];
      unsigned char want = (col < pitch && row >= 0 && row < ny) ? hm[(size_t)row * pitch + col] : 0;
      if (hmo[t] != want) bad++;
    }
    printf("  mismatches: %d\n", bad);
  }
  return 0;
}
