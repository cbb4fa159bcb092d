#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
__global__ void kf2(float2* a){ float2 x=a[threadIdx.x]; float2 t=__fmul2_rn(x, make_float2(2.f,3.f)); t=__fadd2_rn(t,x); a[threadIdx.x]=t; }
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
template<int MODE>
__global__ void ktma(const __grid_constant__ CUtensorMap m, float* out){
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if(threadIdx.x==0){
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    if (MODE>=1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if(threadIdx.x==0){
    if (MODE>=2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),"r"(36*36*4):"memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(sa(sm)),"l"(reinterpret_cast<uint64_t>(&m)),"r"(-2),"r"(-2),"r"(0),"r"(sa(&bar)):"memory");
  }
  uint32_t done=0;
  while(!done){ asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" :"=r"(done):"r"(sa(&bar)),"r"(0):"memory"); }
  out[threadIdx.x]=((float*)sm)[threadIdx.x];
}
int main(){
  float2* a; cudaMalloc(&a, 1024); kf2<<<1,32>>>(a); printf("f2: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  void* fn; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",&fn,cudaEnableDefault,&q);
  auto enc=(PFN_cuTensorMapEncodeTiled_v12000)fn;
  float* g; cudaMalloc(&g, 64*64*3*4); cudaMemset(g,0,64*64*3*4); float* out; cudaMalloc(&out, 4096);
  CUtensorMap m; cuuint64_t dims[3]={64,64,3}; cuuint64_t str[2]={256,256*64}; cuuint32_t box[3]={36,36,1}, es[3]={1,1,1};
  CUresult r=enc(&m,CU_TENSOR_MAP_DATA_TYPE_FLOAT32,3,g,dims,str,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_L2_128B,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("enc %d\n", r);
  ktma<0><<<1,32,8192>>>(m,out); printf("tma0: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  ktma<1><<<1,32,8192>>>(m,out); printf("tma1: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  ktma<2><<<1,32,8192>>>(m,out); printf("tma2: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
