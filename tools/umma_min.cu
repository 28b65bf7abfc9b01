#include <cstdio>
#include <cstdint>
__device__ inline uint32_t su(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__global__ void k(float* out, int variant){
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar; __shared__ uint32_t tbase;
  float* A=(float*)sm; float* B=(float*)(sm+65536);
  int tid=threadIdx.x;
  for(int e=tid;e<128*8;e+=128) A[e]=1.f;   // 128 rows x 8 k: K-major interleave: core 8x4 (128B); rows 16B apart
  for(int e=tid;e<32*8;e+=128) B[e]=1.f;
  if(tid<32){asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"::"r"(su(&tbase)),"r"(64));
             asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");}
  if(tid==0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(su(&bar)),"r"(1));
  asm volatile("fence.proxy.async.shared::cta;":::"memory");
  asm volatile("fence.mbarrier_init.release.cluster;":::"memory");
  asm volatile("tcgen05.fence::before_thread_sync;":::"memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;":::"memory");
  uint32_t tb=tbase;
  int w=tid>>5;
  if(variant==0){ // st/ld roundtrip
    uint32_t v=__float_as_uint(1.0f+tid);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};"::"r"(tb+((32*w)<<16)),"r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;":::"memory");
  } else if(tid==0){
    // A: 128 x 8 K-major: core matrices 8 rows x 16B at 128B each; SBO = 8-row group stride; LBO = K chunk stride
    uint32_t aA=su(A), aB=su(B);
    uint64_t lboA = 16*128, sboA=128;   // A: 16 row-groups of 128B contiguous => SBO=128; 2nd K chunk after 2048B
    uint64_t lboB = 4*128, sboB=128;    // B: N=32 -> 4 groups
    uint64_t da = ((aA>>4)&0x3fff) | ((lboA>>4)<<16) | ((sboA>>4)<<32) | (1ull<<46);
    uint64_t db = ((aB>>4)&0x3fff) | ((lboB>>4)<<16) | ((sboB>>4)<<32) | (1ull<<46);
    uint32_t id = (1u<<4)|(2u<<7)|(2u<<10)|((uint32_t)((variant-1)&1)<<15)|((uint32_t)(((variant-1)>>1)&1)<<16)|((32u>>3)<<17)|((128u>>4)<<24);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"::"r"(tb),"l"(da),"l"(db),"r"(id),"r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"::"r"(su(&bar)):"memory");
    asm volatile("{\n .reg .pred q;\n W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W;\n}\n"::"r"(su(&bar)),"r"(0):"memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;":::"memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;":::"memory");
  uint32_t r0,r1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];":"=r"(r0),"=r"(r1):"r"(tb+((32*w)<<16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;":::"memory");
  out[tid*2]=__uint_as_float(r0); out[tid*2+1]=__uint_as_float(r1);
  __syncthreads();
  if(tid<32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"::"r"(tb),"r"(64));
}
int main(){
  float* d; cudaMalloc(&d,256*4); float h[256];
  cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,80*1024);
  for(int v=0;v<5;v++){ cudaMemset(d,0,1024); k<<<1,128,80*1024>>>(d,v); cudaError_t e=cudaDeviceSynchronize();
    cudaMemcpy(h,d,1024,cudaMemcpyDeviceToHost); printf("variant %d err=%s: %g %g %g %g ... %g\n",v,cudaGetErrorString(e),h[0],h[1],h[2],h[3],h[254]); }
}
