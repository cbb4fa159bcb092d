// Experiment (not product code): DRAM throughput of K3-like TMA box streams.
// A [C][2H][2W] f32 plane; items = (tile, channel) in row-major tile order,
// each item loads 4 boxes (BW x BH floats) from the four subband quadrants,
// like k_level<true>, and does no compute.  Reports GB/s of box bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_pattern tma_pattern.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int BW, int BH>
__global__ void __launch_bounds__(128) k(const __grid_constant__ CUtensorMap tm, int bw, int bh, int ntx, int ntiles, int C, int TXs, int TYs, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  constexpr int SLOT = ((BW * BH * 4 + 127) / 128) * 128;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0, acc = 0;
  const int n = ntiles * C;
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const int tile = it / C, c = it - tile * C;
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int ox = max(tx * TXs - 4, 0), oy = max(ty * TYs - 2, 0);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(4u * BW * BH * 4u) : "memory");
      const int xs[4] = {ox, bw + ox, ox, bw + ox}, ys[4] = {oy, oy, bh + oy, bh + oy};
      for (int q = 0; q < 4; ++q)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su(smem + q * SLOT)), "l"((uint64_t)&tm), "r"(xs[q]), "r"(ys[q]), "r"(c), "r"(su(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(su(&bar)), "r"(phase) : "memory");
    }
    phase ^= 1;
    acc += ((const uint32_t*)smem)[threadIdx.x];
    __syncthreads();
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const int W = 4096 * 2, H = 4096 * 2, C = 3;   // level-1 plane of an 8K frame: subbands 4096^2
  const int bw = W / 2, bh = H / 2;
  float* d;
  size_t bytes = (size_t)C * H * W * 4;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  unsigned* sink; cudaMalloc(&sink, 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int BW, int BH, int TXs, int TYs, int occ) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C};
    cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    cuuint32_t box[3] = {(cuuint32_t)BW, (cuuint32_t)BH, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int ntx = (bw + TXs - 1) / TXs, nty = (bh + TYs - 1) / TYs, nt = ntx * nty;
    const int slot = ((BW * BH * 4 + 127) / 128) * 128, sm = 4 * slot;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const int grid = sms * occ;
    for (int rep = 0; rep < 2; ++rep) kern<<<grid, 128, sm>>>(tm, bw, bh, ntx, nt, C, TXs, TYs, sink);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) kern<<<grid, 128, sm>>>(tm, bw, bh, ntx, nt, C, TXs, TYs, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    const double useful = (double)nt * C * 4 * TXs * TYs * 4;       // subband bytes covered
    const double boxb = (double)nt * C * 4 * BW * BH * 4;           // box bytes moved into smem
    printf("box %dx%d tile %dx%d occ %d: %.1f us  useful %.0f GB/s  box %.0f GB/s  err=%s\n", BW, BH, TXs, TYs, occ,
           ms * 1e3, useful / ms / 1e6, boxb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int occ : {4, 8, 12}) {
    run(k<36, 36>, 36, 36, 28, 32, occ);
    run(k<64, 36>, 64, 36, 56, 32, occ);
    run(k<128, 20>, 128, 20, 120, 16, occ);
    run(k<40, 36>, 40, 36, 32, 32, occ);
  }
  return 0;
}
