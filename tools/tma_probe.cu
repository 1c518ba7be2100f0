// standalone probe of the level kernels' tensor-map copies
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define EBCC_CH 8
namespace ebcc { namespace fused {
constexpr int CH = 8, KB = 4, TW = 224;
} }
struct alignas(64) TMaps { CUtensorMap pk4, pk1, ll4, ll1, orig; };
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_box(uint32_t dst, const CUtensorMap* tm, int x, int y, int z, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(dst), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory");
}
struct Big { int a[300]; };
__global__ void k(Big big, unsigned long long* out, int x, int y, int z, int mode, const __grid_constant__ TMaps tm) {
  __shared__ __align__(128) unsigned long long d[4][128];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) mbar_expect_tx(smem_u32(&bar), 4 * 128 * 8);
    __syncwarp();
    if (mode == 0) { if (lane == 0) tma_box(smem_u32(&d[0][0]), big.a[5] ? &tm.ll4 : &tm.pk4, x, y, z, smem_u32(&bar)); }
    else if (lane < 4) tma_box(smem_u32(&d[lane][0]), lane == 0 ? &tm.pk1 : (big.a[7] ? &tm.ll1 : &tm.pk1), x, y + lane, z, smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = d[i / 128][i % 128];
}
typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  printf("entry %d %d %p\n", (int)e, (int)qr, fn);
  Encode enc = (Encode)fn;
  const uint64_t cols = 22, rows = 16, F = 3;
  std::vector<unsigned long long> h(cols * rows * F);
  for (size_t i = 0; i < h.size(); i++) h[i] = i;
  unsigned long long *dbuf, *dout;
  cudaMalloc(&dbuf, h.size() * 8); cudaMalloc(&dout, 512 * 8);
  cudaMemcpy(dbuf, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  TMaps tm; Big big; for (int i = 0; i < 300; i++) big.a[i] = 0;
  for (int b1 : {4, 1}) {
    cuuint64_t gdim[3] = {cols, rows, F}; cuuint64_t gstr[2] = {cols * 8, cols * rows * 8};
    cuuint32_t box[3] = {128, (cuuint32_t)b1, 1}; cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(b1 == 4 ? &tm.pk4 : &tm.pk1, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, dbuf, gdim, gstr, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode b1=%d -> %d\n", b1, (int)r);
  }
  for (int mode = 0; mode < 2; mode++) {
    int x = 0, y = 4, z = 2;
    k<<<1, 256>>>(big, dout, x, y, z, mode, tm);
    e = cudaDeviceSynchronize();
    printf("mode %d sync: %s\n", mode, cudaGetErrorString(e));
    unsigned long long o[512]; cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int u = 0; u < 4; u++) for (int c = 0; c < 128; c++) {
      unsigned long long want = (unsigned long long)z * cols * rows + (y + u) * cols + x + c;
      if (x + c >= (int)cols) want = 0;
      if (o[u * 128 + c] != want) bad++;
    }
    printf("mode %d mismatches %d (o[0]=%llu)\n", mode, bad, o[0]);
  }
  // edge: box beyond the right border and the last rows
  k<<<1, 256>>>(big, dout, 11, 14, 2, 0, tm);
  e = cudaDeviceSynchronize();
  printf("edge sync: %s\n", cudaGetErrorString(e));
  return 0;
}
