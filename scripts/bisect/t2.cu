#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
// layout: dynamic smem only; bar at 0, box at dst_off
__global__ void ktma(const __grid_constant__ CUtensorMap m, float* out, int dst_off, int x, int y, int dims3){
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar=(uint64_t*)sm;
  if(threadIdx.x==0){
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if(threadIdx.x==0){
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)),"r"(32*32*4):"memory");
    if(dims3) asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(sa(sm+dst_off)),"l"(reinterpret_cast<uint64_t>(&m)),"r"(x),"r"(y),"r"(0),"r"(sa(bar)):"memory");
    else asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(sa(sm+dst_off)),"l"(reinterpret_cast<uint64_t>(&m)),"r"(x),"r"(y),"r"(sa(bar)):"memory");
  }
  uint32_t done=0;
  while(!done){ asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" :"=r"(done):"r"(sa(bar)),"r"(0):"memory"); }
  out[threadIdx.x]=((float*)(sm+dst_off))[threadIdx.x];
}
int main(){
  void* fn; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",&fn,cudaEnableDefault,&q);
  auto enc=(PFN_cuTensorMapEncodeTiled_v12000)fn;
  float* g; cudaMalloc(&g, 64*64*3*4); cudaMemset(g,0,64*64*3*4); float* out; cudaMalloc(&out, 4096);
  for(int d3=0; d3<2; ++d3){
    CUtensorMap m; cuuint64_t dims[3]={64,64,3}; cuuint64_t str[2]={256,256*64}; cuuint32_t box[3]={32,32,1}, es[3]={1,1,1};
    CUresult r=enc(&m,CU_TENSOR_MAP_DATA_TYPE_FLOAT32,d3?3:2,g,dims,str,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("dims%d enc %d\n", d3?3:2, r);
    int offs[2]={128,1024}; int coords[6][2]={{0,0},{0,30},{0,1},{4,0},{2,0},{30,0}};
    for(int o=0;o<1;++o) for(int c=0;c<6;++c){
      ktma<<<1,32,8192>>>(m,out,offs[o],coords[c][0],coords[c][1],d3);
      cudaError_t e=cudaDeviceSynchronize();
      printf("  off %d coord %d,%d: %s\n", offs[o], coords[c][0], coords[c][1], cudaGetErrorString(e));
      if(e!=cudaSuccess) return 1;
    }
  }
  { // tensor smaller than box
    CUtensorMap m; cuuint64_t dims[3]={16,16,3}; cuuint64_t str[2]={64,64*16}; cuuint32_t box[3]={32,32,1}, es[3]={1,1,1};
    CUresult r=enc(&m,CU_TENSOR_MAP_DATA_TYPE_FLOAT32,3,g,dims,str,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("small enc %d\n", r);
    ktma<<<1,32,8192>>>(m,out,128,0,0,1); printf("small: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
